"""GPU parity of the individual kernels through the C ABI.

* K3 grouped GEMM (tcgen05): against a plain PyTorch fp32 reference of the
  same op on identical bf16 inputs (floating-point kernel).
* K1 router: against the CPU oracle -- indices and histogram bit-exact,
  gate weights within 1e-5 (fp32 exp differences only).
"""

import ctypes

import numpy as np
import pytest

from oracle import moe_oracle as orc
from tolerance import check_gemm_close

torch = pytest.importorskip("torch")

pytestmark = pytest.mark.gpu


def _lib():
    from paper_2508_12851_b200 import _lib as L
    return L, L.load()


def _vp(t):
    return ctypes.c_void_p(t.data_ptr())


def _stream():
    return ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)


def _groups(ms, slots, a_offsets=None):
    rows, arr = 0, []
    for i, (m, s) in enumerate(zip(ms, slots)):
        a = rows if a_offsets is None else a_offsets[i]
        arr.append([a, m, s, a])
        rows = a + m
    g = torch.tensor(arr, dtype=torch.int32, device="cuda").reshape(-1)
    n = torch.tensor([len(ms)], dtype=torch.int32, device="cuda")
    return g, n, rows


def _ref_gemm(a, b, ms, slots, N, swiglu):
    outs, r = [], 0
    for m, s in zip(ms, slots):
        acc = a[r:r + m].float() @ b[s * N:(s + 1) * N].float().T
        if swiglu:
            nb = N // 256
            acc = acc.view(m, nb, 2, 128)
            g, u = acc[:, :, 0, :].reshape(m, -1), acc[:, :, 1, :].reshape(m, -1)
            acc = torch.nn.functional.silu(g) * u
        outs.append(acc)
        r += m
    return torch.cat(outs)


@pytest.mark.parametrize("pair", [0, 1], ids=["cta1", "cta_pair"])
@pytest.mark.parametrize("swiglu", [0, 1])
@pytest.mark.parametrize("ms,K,N", [([128], 64, 256), ([300, 5, 128, 0 + 1], 512, 512), ([1000, 37], 2048, 768),
                                    ([257, 511, 256], 256, 512)])
def test_grouped_gemm_matches_torch(swiglu, ms, K, N, pair, monkeypatch):
    monkeypatch.setenv("MP_GEMM_PAIR", str(pair))
    L, lib = _lib()
    torch.manual_seed(0)
    S = len(ms) + 1
    slots = [(i * 2 + 1) % S for i in range(len(ms))]
    rows = sum(ms)
    a = (torch.randn(rows + 7, K, device="cuda") / 4).bfloat16()
    b = (torch.randn(S * N, K, device="cuda") / np.sqrt(K)).bfloat16()
    g, n, _ = _groups(ms, slots)
    out_ld = N // 2 if swiglu else N
    out = torch.full((rows + 7, out_ld), float("nan"), device="cuda", dtype=torch.bfloat16)
    rc = lib.mp_grouped_gemm(_vp(a), a.shape[0], _vp(b), b.shape[0], _vp(g), _vp(n), N, K, _vp(out), out_ld, swiglu,
                             _stream())
    L.check(rc, "mp_grouped_gemm")
    torch.cuda.synchronize()
    ref = _ref_gemm(a, b, ms, slots, N, swiglu)
    got = out[:rows].float()
    assert torch.isfinite(got).all()
    check_gemm_close(got.cpu().numpy(), ref.cpu().numpy())
    # rows outside every group are untouched
    assert torch.isnan(out[rows:].float()).all()


@pytest.mark.parametrize("pair", [0, 1], ids=["cta1", "cta_pair"])
def test_grouped_gemm_large_k_many_tiles(pair, monkeypatch):
    """More tiles than SMs (persistent loop + TMEM double buffer + smem ring wrap)."""
    monkeypatch.setenv("MP_GEMM_PAIR", str(pair))
    L, lib = _lib()
    torch.manual_seed(1)
    ms, K, N = [2048, 1500, 900], 1024, 1024
    slots = [0, 2, 1]
    rows = sum(ms)
    a = (torch.randn(rows, K, device="cuda") / 4).bfloat16()
    b = (torch.randn(3 * N, K, device="cuda") / np.sqrt(K)).bfloat16()
    g, n, _ = _groups(ms, slots)
    out = torch.empty(rows, N, device="cuda", dtype=torch.bfloat16)
    L.check(lib.mp_grouped_gemm(_vp(a), rows, _vp(b), 3 * N, _vp(g), _vp(n), N, K, _vp(out), N, 0, _stream()))
    torch.cuda.synchronize()
    ref = _ref_gemm(a, b, ms, slots, N, 0)
    rel = ((out.float() - ref).norm() / ref.norm()).item()
    assert rel < 1e-2, rel


def _run_router(x, wg, bias, E, k, mode, gate):
    """mp_router_pack + mp_router_topk_hist (the tensor-core exact-integer router)."""
    L, lib = _lib()
    T, d = x.shape
    xt = torch.from_numpy(x).cuda().bfloat16()
    wgt = torch.from_numpy(wg).cuda().bfloat16()
    packed = torch.empty(lib.mp_router_packed_bytes(E + gate, d), device="cuda", dtype=torch.uint8)
    L.check(lib.mp_router_pack(_vp(wgt), E + gate, d, _vp(packed), _stream()))
    bt = torch.from_numpy(bias).cuda()
    idx = torch.empty(T, k, dtype=torch.int32, device="cuda")
    w = torch.empty(T, k, dtype=torch.float32, device="cuda")
    go = torch.empty(T, dtype=torch.float32, device="cuda")
    hist = torch.zeros(E, dtype=torch.int32, device="cuda")
    L.check(lib.mp_router_topk_hist(_vp(xt), _vp(packed), _vp(bt), T, d, E, gate, k, mode, 0, _vp(idx), _vp(w),
                                    _vp(go) if gate else None, _vp(hist), _stream()))
    torch.cuda.synchronize()
    return idx.cpu().numpy(), w.cpu().numpy(), hist.cpu().numpy(), go.cpu().numpy()


@pytest.mark.parametrize("split", ["", "1", "2", "4"])
@pytest.mark.parametrize("E,k,mode,d", [(8, 2, 0, 512), (64, 6, 1, 256), (16, 4, 0, 4096), (60, 4, 1, 2048),
                                        (8, 2, 0, 3072)])
def test_router_ties_go_to_the_lower_expert(E, k, mode, d, split, monkeypatch):
    """Exact logit ties (duplicated router rows + biases, all-zero tokens whose logits are the
    biases alone) resolve to the lower expert id, bit-exact with the oracle -- for every K split
    of the tensor-core router ("" = the default; the integer logits cannot depend on it)."""
    if split:
        monkeypatch.setenv("MP_ROUTER_SPLIT", split)
    T = 96
    x = orc.synthetic_tokens(0, T, d, seed=7)
    x[::3] = 0.0                       # every third token: logits == bias
    wg = orc.synthetic_router(E, d, seed=7)
    bias = orc.origin_bias(0, E, seed=7)
    for a, b in [(2, 5), (1, E - 1)]:  # identical experts
        wg[b] = wg[a]
        bias[b] = bias[a]
    bias[3] = bias[4] = bias[6] = np.float32(bias.max())   # three-way tie among the biases
    lg = orc.router_logits(x, wg, bias)
    idx_ref, w_ref = orc.topk_route(lg, E, k, mode)
    idx, w, hist, _ = _run_router(x, wg, bias, E, k, mode, 0)
    assert np.array_equal(idx, idx_ref)
    assert np.array_equal(hist, orc.histogram(idx_ref, E))
    np.testing.assert_allclose(w, w_ref, rtol=1e-5, atol=1e-6)
    for row in idx[::3]:               # zero tokens: 3 < 4 < 6 when tied at the top
        pos = {int(e): i for i, e in enumerate(row)}
        for lo, hi in [(3, 4), (4, 6), (2, 5)]:
            if lo in pos and hi in pos:
                assert pos[lo] < pos[hi], row


@pytest.mark.parametrize("E,k,mode,gate,d,T", [(8, 2, 0, 0, 512, 333), (64, 6, 1, 0, 256, 200), (60, 4, 1, 1, 512, 64),
                                               (8, 2, 0, 0, 4096, 48), (16, 4, 0, 0, 4096, 100),
                                               (64, 6, 1, 1, 2048, 1000), (33, 3, 0, 0, 768, 129),
                                               (64, 8, 1, 1, 1024, 77), (1, 1, 0, 0, 512, 5), (48, 2, 0, 1, 256, 1)])
def test_router_bit_exact(E, k, mode, gate, d, T):
    """The tensor-core router against oracle.router_logits: every N instantiation (E + gate up to
    65 rows -> N = 80), partial tiles, K ranges of uneven length (d = 768), rows on tiny and on
    dominated grids."""
    x = orc.synthetic_tokens(0, T, d, seed=3)
    if T > 6:
        x[5] *= np.float32(2.0 ** -90)     # a row on a tiny grid
        x[6, 11] = np.float32(3.0e4)       # a row whose maximum dwarfs the rest
    wg = orc.synthetic_router(E + gate, d, seed=3)
    bias = orc.origin_bias(1, E, seed=3)
    lg = orc.router_logits(x, wg, bias)
    idx_ref, w_ref = orc.topk_route(lg, E, k, mode)
    hist_ref = orc.histogram(idx_ref, E)
    idx, w, hist, go = _run_router(x, wg, bias, E, k, mode, gate)
    assert np.array_equal(idx, idx_ref)
    assert np.array_equal(hist, hist_ref)
    np.testing.assert_allclose(w, w_ref, rtol=1e-5, atol=1e-6)
    if gate:
        g_ref = 1.0 / (1.0 + np.exp(-lg[:, E].astype(np.float64)))
        np.testing.assert_allclose(go, g_ref, rtol=1e-5, atol=1e-6)


@pytest.mark.parametrize("E,k,mode,renorm", [(8, 2, 0, 0), (64, 6, 1, 0), (60, 4, 1, 1), (33, 8, 1, 0), (1, 1, 0, 0)])
def test_router_logits_in_selection(E, k, mode, renorm):
    """mp_router_topk_logits: K1's selection stage from given logits -- random logits plus rows
    of exact ties (all equal, pairs, a tied top) -- indices and histogram bit-exact, weights to
    fp32 rounding, against the oracle's selection rule."""
    L, lib = _lib()
    rng = np.random.default_rng(E * 10 + k)
    T = 257
    lg = rng.standard_normal((T, E)).astype(np.float32)
    lg[1] = 0.5                                  # all tied: lowest ids first
    lg[2, 1::2] = lg[2, 0::2][: lg[2, 1::2].size]  # adjacent pairs tied
    lg[3, -1] = lg[3, 0] = np.float32(lg[3].max() + 1)  # tied top: 0 before E-1
    bias = rng.standard_normal(E).astype(np.float32) * np.float32(0.1)
    bias[-1] = bias[0]
    ref_lg = (lg + bias[None, :]).astype(np.float32)
    idx_ref, w_ref = orc.topk_route(ref_lg, E, k, mode, renorm)
    ld = E + 3
    buf = np.zeros((T, ld), np.float32)
    buf[:, :E] = lg
    lt = torch.from_numpy(buf).cuda()
    bt = torch.from_numpy(bias).cuda()
    idx = torch.empty(T, k, dtype=torch.int32, device="cuda")
    w = torch.empty(T, k, dtype=torch.float32, device="cuda")
    hist = torch.zeros(E, dtype=torch.int32, device="cuda")
    L.check(lib.mp_router_topk_logits(_vp(lt), ld, _vp(bt), T, E, k, mode, renorm, _vp(idx), _vp(w), _vp(hist),
                                      _stream()))
    torch.cuda.synchronize()
    assert np.array_equal(idx.cpu().numpy(), idx_ref)
    assert np.array_equal(hist.cpu().numpy(), orc.histogram(idx_ref, E))
    np.testing.assert_allclose(w.cpu().numpy(), w_ref, rtol=1e-5, atol=1e-6)


@pytest.mark.parametrize("E,k,d", [(8, 2, 512), (64, 6, 2048)])
def test_router_extreme_rows_bit_exact(E, k, d):
    """Rows at the edges of the grid rule on the GPU: all-zero tokens, tokens below the E = -100
    clamp, huge tokens, single-element tokens, constant tokens, a tiny and a duplicated expert --
    indices, histogram and weights against the oracle."""
    rng = np.random.default_rng(E + d)
    T = 160
    x = orc.synthetic_tokens(0, T, d, seed=21)
    x[0::8] = 0.0
    x[1::8] = orc.bf16_round(x[1::8] * np.float32(2.0 ** -120))
    x[2::8] = orc.bf16_round(x[2::8] * np.float32(2.0 ** 60))
    x[3::8] = 0.0
    x[3::8, 5] = np.float32(-2.5)
    x[4::8] = np.float32(0.25)
    wg = orc.synthetic_router(E, d, seed=21)
    wg[1] = orc.bf16_round(wg[1] * np.float32(2.0 ** -110))
    wg[E - 1] = wg[0]
    bias = orc.origin_bias(0, E, seed=21)
    lg = orc.router_logits(x, wg, bias)
    idx_ref, w_ref = orc.topk_route(lg, E, k, 0)
    idx, w, hist, _ = _run_router(x, wg, bias, E, k, 0, 0)
    assert np.array_equal(idx, idx_ref)
    assert np.array_equal(hist, orc.histogram(idx_ref, E))
    np.testing.assert_allclose(w, w_ref, rtol=1e-5, atol=1e-6)
