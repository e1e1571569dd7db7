"""Floating-point tolerances of the GPU parity tests (stated once, used everywhere).

Both sides compute in fp32 from bf16-exact inputs and round the same
intermediates to bf16 (h = bf16(silu(g) * u), y = bf16(h W2^T), out =
bf16(sum_j w_j y_j (+ g_sh y_sh))); they differ only in the fp32 summation
order inside the GEMMs, which can flip a bf16 rounding by one unit in the last
place (an ulp is 2^-8..2^-7 of the value).  The per-element bound is the
a-priori error of those flips, relative to the magnitude of the terms each
element is made of -- NOT to the element itself, which can be a cancelled sum:

* layer output   |out - ref| <= 2^-7 * (mag2 + 2 mag) + 1e-5 * max|ref|,
                 mag  = sum_j |w_j y_j| (+ |g_sh y_sh|)           one ulp of y_j and of out;
                 mag2 = sum_j |w_j| (|h_j| |W2|^T) (+ shared)     one ulp of every h element
                                                                  feeding GEMM2 (worst case);
                 (OracleResult.mag / mag2, tests/torch_ref.py at full size);
                 relative Frobenius error <= 3e-3;
* GEMM (+SwiGLU) |got - ref| <= 2^-6 * |ref| + 1e-3 * max|ref| per element
                 (two bf16 ulps of the fp32 result plus an accumulation-order
                 floor for cancelled sums); relative Frobenius error <= 3e-3.
"""

from __future__ import annotations

import numpy as np

LAYER_ULP = 2.0 ** -7
LAYER_ABS_FLOOR = 1e-5
GEMM_REL = 2.0 ** -6
GEMM_ABS_FLOOR = 1e-3
RTOL_FRO = 3e-3


def check_layer_close(got, ref, mag, mag2, what: str = "") -> dict:
    got = np.asarray(got, dtype=np.float32)
    ref = np.asarray(ref, dtype=np.float32)
    if ref.size == 0:
        assert got.size == 0, what
        return {}
    mag = np.asarray(mag, dtype=np.float32)
    mag2 = np.asarray(mag2, dtype=np.float32)
    err = np.abs(got - ref)
    scale = float(np.abs(ref).max())
    bound = LAYER_ULP * (mag2 + 2.0 * mag) + LAYER_ABS_FLOOR * scale
    bad = err > bound
    rel = float(np.linalg.norm(got - ref) / max(np.linalg.norm(ref), 1e-30))
    used = float((err / bound).max())
    assert not bad.any(), (f"{what}: {int(bad.sum())} of {bad.size} elements outside 2^-7*(mag2+2mag); "
                           f"max err {float(err.max())} max err/bound {used} scale {scale}")
    assert rel <= RTOL_FRO, f"{what}: relative Frobenius error {rel}"
    return {"max_err": float(err.max()), "max_err_over_bound": used, "rel_fro": rel,
            "mean_bound_over_scale": float(bound.mean() / max(scale, 1e-30))}


def check_gemm_close(got, ref, what: str = "") -> dict:
    got = np.asarray(got, dtype=np.float32)
    ref = np.asarray(ref, dtype=np.float32)
    err = np.abs(got - ref)
    scale = float(np.abs(ref).max())
    bad = err > GEMM_REL * np.abs(ref) + GEMM_ABS_FLOOR * scale
    rel = float(np.linalg.norm(got - ref) / max(np.linalg.norm(ref), 1e-30))
    assert not bad.any(), f"{what}: {int(bad.sum())} of {bad.size} elements out of bound; max err {float(err.max())}"
    assert rel <= RTOL_FRO, f"{what}: relative Frobenius error {rel}"
    return {"max_err": float(err.max()), "rel_fro": rel}
