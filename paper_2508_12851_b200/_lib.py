"""ctypes binding of libmoeplace_b200.so (include/moeplace_b200.h).

There is no fallback: if the shared library is missing or does not export
the ABI, importing the GPU path raises.  Error codes map onto the reference's
exception types (reference pkg/src/moeplace/domain.py:32-37, cost.py:34-35).
"""

from __future__ import annotations

import ctypes
from ctypes import POINTER, Structure, c_char_p, c_int, c_int32, c_int64, c_void_p
from pathlib import Path

from .errors import DimensionMismatch, InfeasibleError, UnplacedExpertError

LIB_PATH = Path(__file__).resolve().parent / "libmoeplace_b200.so"
ABI_VERSION = 3
MAX_GROUPS = 128

MP_OK = 0
MP_E_ARG = -1
MP_E_SHAPE = -2
MP_E_CAPACITY = -3
MP_E_UNPLACED = -4
MP_E_CUDA = -5
MP_E_PEER = -6

MP_SCORE_TOPK_SOFTMAX = 0
MP_SCORE_SOFTMAX_TOPK = 1
NUM_STAGE_EVENTS = 13
MAIN_STAGE_EVENTS = 11  # 11, 12: side-chain start / end (side stream, split plan only)
# Intervals between consecutive stage events.  The count exchange and the dispatch / return
# waits are folded into the router, permute, GEMM and combine kernels (PeerSync), so their
# intervals only hold event overhead; "shared_expert" is empty when the plan fuses it into K3.
STAGES = ("router", "unused", "unused", "permute_dispatch", "shared_expert", "unused",
          "gemm1_swiglu", "gemm2", "unused", "combine_return")
GEMM_START, GEMM1_END, GEMM_END = 6, 7, 8
CFG_KEYS = {"pair_routed": 0, "split_m": 1, "small_grid": 2, "fuse_shared": 3}

# Every symbol the header declares (checked by tests/test_abi.py).
EXPORTED_SYMBOLS = (
    "mp_abi_version", "mp_last_error", "mp_router_packed_bytes", "mp_router_pack", "mp_router_topk_hist",
    "mp_router_topk_logits", "mp_grouped_gemm",
    "mp_layer_create", "mp_layer_destroy", "mp_layer_get_ptrs", "mp_layer_export_handles",
    "mp_layer_open_peers", "mp_layer_set_routes", "mp_layer_prepare_router", "mp_layer_forward",
    "mp_layer_forward_timed", "mp_layer_route", "mp_layer_permute", "mp_layer_experts", "mp_layer_combine_gather",
    "mp_layer_last_launches", "mp_layer_config", "mp_layer_read_counts", "mp_layer_check", "mp_layer_migrate",
    "mp_layer_peer_probe", "mp_layer_sync_state",
)


class LayerDesc(Structure):
    _fields_ = [
        ("rank", c_int32), ("world", c_int32), ("device", c_int32), ("max_tokens", c_int32),
        ("d", c_int32), ("f", c_int32), ("E", c_int32), ("top_k", c_int32),
        ("score_mode", c_int32), ("renorm", c_int32), ("n_slots", c_int32),
        ("shared_f", c_int32), ("shared_gate", c_int32),
    ]


class LayerPtrs(Structure):
    _fields_ = [
        ("pool", c_void_p), ("wg", c_void_p), ("bias", c_void_p),
        ("w13_shared", c_void_p), ("w2_shared", c_void_p), ("idx", c_void_p), ("w", c_void_p),
        ("pos_dst", c_void_p), ("pos_row", c_void_p), ("recv", c_void_p), ("h", c_void_p), ("ret", c_void_p),
        ("recv_src", c_void_p),
        ("hist", c_void_p), ("counts", c_void_p),
        ("shared_gate", c_void_p), ("batch_counts", c_void_p), ("recv_cap", c_int64), ("slot_bytes", c_int64),
    ]


class CopyOp(Structure):
    _fields_ = [("src_rank", c_int32), ("src_slot", c_int32), ("dst_slot", c_int32)]


_lib = None


def load(path: Path | str | None = None) -> ctypes.CDLL:
    """Load (once) and type the library; raises if it is absent or stale."""
    global _lib
    if _lib is not None:
        return _lib
    p = Path(path) if path else LIB_PATH
    if not p.exists():
        raise RuntimeError(
            f"{p} is missing: the B200 CUDA library has not been built "
            "(run `python -c 'import __graft_entry__ as g; g.build()'`); there is no CPU fallback")
    lib = ctypes.CDLL(str(p))
    for name in EXPORTED_SYMBOLS:
        if not hasattr(lib, name):
            raise RuntimeError(f"{p} does not export {name}")
    V, I, I64 = c_void_p, c_int, c_int64
    sig = {
        "mp_abi_version": ([], I),
        "mp_last_error": ([c_char_p, I], I),
        "mp_router_pack": ([V, I, I, V, V], I),
        "mp_router_packed_bytes": ([I, I], ctypes.c_size_t),
        "mp_router_topk_hist": ([V, V, V, I, I, I, I, I, I, I, V, V, V, V, V], I),
        "mp_router_topk_logits": ([V, I, V, I, I, I, I, I, V, V, V, V], I),
        "mp_grouped_gemm": ([V, I64, V, I64, V, V, I, I, V, I, I, V], I),
        "mp_layer_create": ([POINTER(LayerDesc), POINTER(c_void_p)], I),
        "mp_layer_destroy": ([V], I),
        "mp_layer_get_ptrs": ([V, POINTER(LayerPtrs)], I),
        "mp_layer_export_handles": ([V, V], I),
        "mp_layer_open_peers": ([V, V], I),
        "mp_layer_set_routes": ([V, V, V, V], I),
        "mp_layer_prepare_router": ([V, V], I),
        "mp_layer_forward": ([V, V, V, I, V], I),
        "mp_layer_forward_timed": ([V, V, V, I, V, POINTER(c_void_p)], I),
        "mp_layer_route": ([V, V, I, V], I),
        "mp_layer_permute": ([V, V, I, V, V, V], I),
        "mp_layer_experts": ([V, V, I, V, V], I),
        "mp_layer_combine_gather": ([V, V, I, V, V], I),
        "mp_layer_last_launches": ([V], I),
        "mp_layer_config": ([V, I], I),
        "mp_layer_read_counts": ([V, V, V], I),
        "mp_layer_sync_state": ([V, V, V], I),
        "mp_layer_check": ([V, V], I),
        "mp_layer_migrate": ([V, POINTER(CopyOp), I, V, V], I),
        "mp_layer_peer_probe": ([V, I, I64, I, V, POINTER(ctypes.c_float)], I),
    }
    for name, (args, res) in sig.items():
        fn = getattr(lib, name)
        fn.argtypes = args
        fn.restype = res
    if lib.mp_abi_version() != ABI_VERSION:
        raise RuntimeError(f"{p}: ABI version {lib.mp_abi_version()} != {ABI_VERSION}")
    _lib = lib
    return lib


def last_error() -> str:
    buf = ctypes.create_string_buffer(1024)
    load().mp_last_error(buf, 1024)
    return buf.value.decode(errors="replace")


def check(code: int, what: str = "") -> None:
    """Raise the reference-typed exception for a non-zero ABI return code."""
    if code == MP_OK:
        return
    msg = f"{what}: {last_error()}" if what else last_error()
    if code == MP_E_SHAPE:
        raise DimensionMismatch(msg)
    if code == MP_E_CAPACITY:
        raise InfeasibleError(msg)
    if code == MP_E_UNPLACED:
        raise UnplacedExpertError(msg)
    if code == MP_E_ARG:
        raise ValueError(msg)
    raise RuntimeError(msg)
