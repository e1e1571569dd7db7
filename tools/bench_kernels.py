"""Per-kernel micro-benchmarks through the C ABI (CUDA events, warm, back-to-back).

usage: python tools/bench_kernels.py [--config mixtral] [--T 4096] [--iters 50] [--only router]
Prints achieved GB/s (HBM-bound kernels) or TFLOP/s (GEMM) per kernel.
"""

import argparse
import ctypes
import json
import sys
from pathlib import Path

REPO = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(REPO))

import torch  # noqa: E402

from paper_2508_12851_b200 import _lib, workload as wl  # noqa: E402
from paper_2508_12851_b200.shapes import get_shape  # noqa: E402


def vp(t):
    return ctypes.c_void_p(t.data_ptr())


def timeit(fn, iters):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(iters):
        fn()
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) / iters * 1e3  # us


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="mixtral")
    ap.add_argument("--T", type=int, default=4096)
    ap.add_argument("--iters", type=int, default=50)
    ap.add_argument("--only", default="")
    args = ap.parse_args()
    shape = get_shape(args.config)
    lib = _lib.load()
    dev = torch.device("cuda", 0)
    st = ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)
    T, d, E, k = args.T, shape.d, shape.E, shape.k
    res = {}
    E_tot = E + shape.shared_gate
    if not args.only or args.only == "router":
        # 16 rotating batches (> L2) so every call reads its x cold from HBM, as inside a layer step
        xs_ = [wl.tokens(T, d, dev, batch=b) for b in range(16)]
        x = xs_[0]
        wg = wl.router_weights(E_tot, d, dev)
        packed = torch.empty(lib.mp_router_packed_bytes(E_tot, d), device=dev, dtype=torch.uint8)
        _lib.check(lib.mp_router_pack(vp(wg), E_tot, d, vp(packed), st))
        bias = wl.origin_bias(0, E).to(dev)
        idx = torch.empty(T, k, dtype=torch.int32, device=dev)
        w = torch.empty(T, k, dtype=torch.float32, device=dev)
        g = torch.empty(T, dtype=torch.float32, device=dev)
        hist = torch.zeros(E, dtype=torch.int32, device=dev)
        rot = [0]

        def nxt():
            rot[0] = (rot[0] + 1) % len(xs_)
            return xs_[rot[0]]
        call = lambda: _lib.check(lib.mp_router_topk_hist(vp(nxt()), vp(packed), vp(bias), T, d, E, shape.shared_gate, k,
                                                          shape.score_mode, 0, vp(idx), vp(w), vp(g), vp(hist), st))
        us = timeit(call, args.iters)
        byts = T * d * 2 + T * k * 8
        res["router"] = {"us": us, "GB/s": byts / us / 1e3, "fma_TF/s": 2 * T * E_tot * d / us / 1e6}
    if not args.only or args.only == "gemm":
        M = T * k // E
        groups = torch.tensor([[i * M, M, i, i * M] for i in range(E)], dtype=torch.int32, device=dev).reshape(-1)
        ng = torch.tensor([E], dtype=torch.int32, device=dev)
        a = wl.tokens(T * k, d, dev)
        b13 = (torch.randn(E * 2 * shape.f, d, device=dev) / d ** 0.5).bfloat16()
        h = torch.empty(T * k, shape.f, device=dev, dtype=torch.bfloat16)
        us = timeit(lambda: _lib.check(lib.mp_grouped_gemm(vp(a), T * k, vp(b13), E * 2 * shape.f, vp(groups), vp(ng),
                                                           2 * shape.f, d, vp(h), shape.f, 1, st)), args.iters)
        fl = 2.0 * T * k * d * 2 * shape.f
        res["gemm1_uniform"] = {"us": us, "TFLOP/s": fl / us / 1e6}
        b2 = (torch.randn(E * d, shape.f, device=dev) / shape.f ** 0.5).bfloat16()
        y = torch.empty(T * k, d, device=dev, dtype=torch.bfloat16)
        us = timeit(lambda: _lib.check(lib.mp_grouped_gemm(vp(h), T * k, vp(b2), E * d, vp(groups), vp(ng), d, shape.f,
                                                           vp(y), d, 0, st)), args.iters)
        res["gemm2_uniform"] = {"us": us, "TFLOP/s": fl / 2 / us / 1e6}
        # the same expert FLOPs through cuBLAS (torch.bmm over the E groups, no SwiGLU / scatter):
        # a same-box, same-clock yardstick for the tcgen05 kernels above
        a3 = a.view(E, M, d)
        w13 = b13.view(E, 2 * shape.f, d).transpose(1, 2)
        h3 = torch.empty(E, M, 2 * shape.f, device=dev, dtype=torch.bfloat16)
        us = timeit(lambda: torch.bmm(a3, w13, out=h3), args.iters)
        res["cublas_bmm1"] = {"us": us, "TFLOP/s": fl / us / 1e6}
        hh = h.view(E, M, shape.f)
        w2 = b2.view(E, d, shape.f).transpose(1, 2)
        y3 = torch.empty(E, M, d, device=dev, dtype=torch.bfloat16)
        us = timeit(lambda: torch.bmm(hh, w2, out=y3), args.iters)
        res["cublas_bmm2"] = {"us": us, "TFLOP/s": fl / 2 / us / 1e6}
    print(json.dumps({"config": shape.name, "T": T, **res}))


if __name__ == "__main__":
    main()
