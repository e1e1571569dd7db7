"""Floating-point tolerances of the GPU parity tests (stated once, used everywhere).

Both sides compute in fp32 from bf16-exact inputs and round the same
intermediates to bf16 (h = bf16(silu(g) * u), y = bf16(h W2^T), out =
bf16(sum_j w_j y_j (+ g_sh y_sh))); they differ only in the fp32 summation
order inside the GEMMs, which can flip a bf16 rounding of h, y or out by one
unit in the last place.  The bounds are therefore relative to the magnitude of
the terms each element is made of, in bf16 ulps (2^-8..2^-7 of a value):

* layer output   |out - ref| <= 2^-6 * mag + 1e-5 * max|ref|   per element,
                 mag = sum_j |w_j y_j| (+ |g_sh y_sh|)  (OracleResult.mag),
                 i.e. two to four bf16 ulps of the contributing terms;
                 relative Frobenius error <= 3e-3;
* GEMM (+SwiGLU) |got - ref| <= 2^-6 * |ref| + 1e-3 * max|ref| per element
                 (two bf16 ulps of the fp32 result plus an accumulation-order
                 floor for cancelled sums); relative Frobenius error <= 3e-3.
"""

from __future__ import annotations

import numpy as np

LAYER_REL_MAG = 2.0 ** -6
LAYER_ABS_FLOOR = 1e-5
GEMM_REL = 2.0 ** -6
GEMM_ABS_FLOOR = 1e-3
RTOL_FRO = 3e-3


def check_layer_close(got, ref, mag, what: str = "") -> dict:
    got = np.asarray(got, dtype=np.float32)
    ref = np.asarray(ref, dtype=np.float32)
    if ref.size == 0:
        assert got.size == 0, what
        return {}
    mag = np.asarray(mag, dtype=np.float32)
    err = np.abs(got - ref)
    scale = float(np.abs(ref).max())
    bound = LAYER_REL_MAG * mag + LAYER_ABS_FLOOR * scale
    bad = err > bound
    rel = float(np.linalg.norm(got - ref) / max(np.linalg.norm(ref), 1e-30))
    worst = float((err / np.maximum(mag, 1e-30)).max())
    assert not bad.any(), (f"{what}: {int(bad.sum())} of {bad.size} elements outside 2^-6*mag; "
                           f"max err {float(err.max())} max err/mag {worst} scale {scale}")
    assert rel <= RTOL_FRO, f"{what}: relative Frobenius error {rel}"
    return {"max_err": float(err.max()), "max_err_over_mag": worst, "rel_fro": rel}


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
