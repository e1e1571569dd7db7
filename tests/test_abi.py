"""The C-ABI library (CPU checks: load, exports, errors -- no compute calls without a GPU)."""

import ctypes
import re
from pathlib import Path

import pytest

REPO = Path(__file__).resolve().parent.parent


def header_symbols():
    text = (REPO / "include" / "moeplace_b200.h").read_text()
    return sorted(set(re.findall(r"^(?:int|size_t) (mp_\w+)\(", text, flags=re.M)))


def test_header_and_binding_agree():
    from paper_2508_12851_b200 import _lib
    assert sorted(_lib.EXPORTED_SYMBOLS) == header_symbols()


def test_library_loads_and_exports_every_symbol():
    from paper_2508_12851_b200 import _lib
    lib = _lib.load()
    raw = ctypes.CDLL(str(_lib.LIB_PATH))
    for name in header_symbols():
        assert hasattr(raw, name), name
    assert lib.mp_abi_version() == _lib.ABI_VERSION


def test_sm100a_code_in_library():
    import shutil
    import subprocess
    from paper_2508_12851_b200 import _lib
    if not shutil.which("cuobjdump"):
        pytest.skip("cuobjdump not available")
    out = subprocess.run(["cuobjdump", "-lelf", str(_lib.LIB_PATH)], capture_output=True, text=True).stdout
    assert "sm_100a" in out


def test_invalid_desc_maps_to_reference_exceptions():
    from paper_2508_12851_b200 import DimensionMismatch, InfeasibleError, _lib
    lib = _lib.load()
    h = ctypes.c_void_p()
    bad = _lib.LayerDesc(rank=0, world=9, device=0, max_tokens=16, d=512, f=512, E=8, top_k=2)
    rc = lib.mp_layer_create(ctypes.byref(bad), ctypes.byref(h))
    assert rc == _lib.MP_E_SHAPE
    assert "world=9" in _lib.last_error()
    with pytest.raises(DimensionMismatch):
        _lib.check(rc)
    bad2 = _lib.LayerDesc(rank=0, world=1, device=0, max_tokens=16, d=512, f=512, E=8, top_k=2, n_slots=-1)
    rc = lib.mp_layer_create(ctypes.byref(bad2), ctypes.byref(h))
    with pytest.raises(InfeasibleError):
        _lib.check(rc)
    assert lib.mp_layer_forward(None, None, None, 0, None) == _lib.MP_E_ARG
    with pytest.raises(ValueError):
        _lib.check(_lib.MP_E_ARG)


def test_no_banned_copy_apis_in_sources():
    """Batched-copy APIs are off limits on this B200 pool (B200_PROFILING.md)."""
    banned = re.compile(r"(cuda|cu)Memcpy(3D)?Batch" + "Async")
    for p in list((REPO / "paper_2508_12851_b200" / "csrc").glob("*")) + [REPO / "include" / "moeplace_b200.h"]:
        assert not banned.search(p.read_text()), p
