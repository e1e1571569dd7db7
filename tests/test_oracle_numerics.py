"""Oracle self-consistency (CPU): router order contract, permutation, layer algebra."""

import numpy as np
import pytest

from oracle import moe_oracle as orc


def test_bf16_round_matches_torch():
    torch = pytest.importorskip("torch")
    a = np.random.default_rng(0).standard_normal(10000).astype(np.float32) * 100
    ref = torch.from_numpy(a).bfloat16().float().numpy()
    np.testing.assert_array_equal(orc.bf16_round(a), ref)


def _rne_f32(v: int) -> float:
    a = abs(v)
    if a == 0:
        return 0.0
    drop = max(a.bit_length() - 24, 0)
    m, rem = a >> drop, a & ((1 << drop) - 1)
    if drop and (rem > (1 << (drop - 1)) or (rem == (1 << (drop - 1)) and m & 1)):
        m += 1
    return float(m * 2 ** drop) * (-1 if v < 0 else 1)


def test_router_logits_contract():
    """Each row on its own integer grid, the exact integer dot product, one rounding to fp32, the
    power-of-two rescale -- restated with Python integers -- and close to the real dot product."""
    rng = np.random.default_rng(1)
    d = 512
    x = orc.bf16_round(rng.standard_normal((3, d)).astype(np.float32))
    w = orc.bf16_round(rng.standard_normal((5, d)).astype(np.float32))
    x[1] *= np.float32(2.0 ** -70)
    x[2, 3] = np.float32(-5.0e3)
    got = orc.router_logits(x, w)

    def grid(row, win):
        m = max(abs(float(v)) for v in row)
        ef = 0 if m == 0 else int(np.frexp(np.float32(m))[1]) + 126   # bf16 exponent field
        e = max(ef - 126, -100)
        return [int(np.rint(float(v) * 2.0 ** (win - e))) for v in row], e

    for t in range(3):
        qx, ex = grid(x[t], 21)
        assert max(abs(q) for q in qx) <= 2 ** 21
        for e in range(5):
            qw, ew = grid(w[e], 14)
            assert max(abs(q) for q in qw) <= 2 ** 14
            s = sum(a * b for a, b in zip(qx, qw))
            want = np.float32(_rne_f32(s) * 2.0 ** (ex + ew - 35))
            assert got[t, e] == want
    ref = x.astype(np.float64) @ w.astype(np.float64).T
    scale = np.abs(x).max(axis=1, keepdims=True) * np.abs(w).max(axis=1)[None, :] * d
    assert (np.abs(got - ref) <= 2.0 ** -14 * scale + 1e-30).all()


def test_exact_int_matmul_and_rounding():
    rng = np.random.default_rng(5)
    q = rng.integers(-2 ** 21, 2 ** 21 + 1, size=(7, 4096))
    r = rng.integers(-2 ** 21, 2 ** 21 + 1, size=(3, 4096))
    s = orc.exact_int_matmul(q, r)
    for i in range(7):
        for j in range(3):
            assert int(s[i, j]) == sum(int(a) * int(b) for a, b in zip(q[i], r[j]))
    vals = np.concatenate([rng.integers(-2 ** 62, 2 ** 62, size=5000), [0, 1, -1, 2 ** 24 + 1, 2 ** 24 + 3,
                                                                         2 ** 25 + 2, 2 ** 25 + 6, -(2 ** 25 + 6)]])
    got = orc.rne_f32_of_int(vals)
    assert all(got[i] == _rne_f32(int(v)) for i, v in enumerate(vals))


def test_topk_ties_go_to_lower_id():
    lg = np.array([[1.0, 3.0, 3.0, 2.0, 3.0]], dtype=np.float32)
    idx, w = orc.topk_route(lg, 5, 3, 0)
    assert idx.tolist() == [[1, 2, 4]]
    np.testing.assert_allclose(w.sum(), 1.0, rtol=1e-6)


def test_softmax_modes():
    lg = np.array([[0.0, 1.0, 2.0, 3.0]], dtype=np.float32)
    idx, w = orc.topk_route(lg, 4, 2, 1)
    p = np.exp(lg[0] - 3) / np.exp(lg[0] - 3).sum()
    assert idx.tolist() == [[3, 2]]
    np.testing.assert_allclose(w[0], p[[3, 2]], rtol=1e-6)
    _, wr = orc.topk_route(lg, 4, 2, 1, renorm=1)
    np.testing.assert_allclose(wr[0].sum(), 1.0, rtol=1e-6)


def test_pair_positions_stable_and_dense():
    rng = np.random.default_rng(2)
    G, E, k, T = 3, 8, 2, 50
    idxs = [np.stack([rng.choice(E, k, replace=False) for _ in range(T)]) for _ in range(G)]
    counts = np.stack([orc.histogram(i, E) for i in idxs])
    route = rng.integers(0, G, (G, E)).astype(np.int32)
    M, gb, send = orc.receive_layout(counts, route)
    for D in range(G):
        seen = []
        for s in range(G):
            dst, rows = orc.pair_positions(idxs[s], route[s], send[s])
            # stable: within (s, e) rows increase in (token, slot) order
            for e in range(E):
                r = rows[idxs[s] == e]
                assert np.all(np.diff(r) == 1)
            seen += list(rows[dst == D])
        assert sorted(seen) == list(range(int(M[D].sum())))


def test_layer_linear_in_gate_weights_and_empty_batch():
    from paper_2508_12851_b200.shapes import LayerShape
    shape = LayerShape("t", d=256, f=256, E=4, k=2)
    experts = {e: orc.synthetic_expert(e, 256, 256) for e in range(4)}
    wg = orc.synthetic_router(4, 256)
    x = orc.synthetic_tokens(0, 0, 256)
    r = orc.moe_layer_forward(shape, [x], wg, [None], np.zeros((1, 4), np.int32), experts)
    assert r.out[0].shape == (0, 256) and r.counts.sum() == 0


def test_router_contract_extreme_rows():
    """Rows at the edges of the grid rule -- all zero, subnormal-range bf16 values (E(a) clamped
    at -100), huge magnitudes, a single non-zero element, ties -- against the Python-integer
    restatement, and the logits are finite."""
    rng = np.random.default_rng(11)
    d = 256
    x = orc.bf16_round(rng.standard_normal((6, d)).astype(np.float32))
    w = orc.bf16_round(rng.standard_normal((4, d)).astype(np.float32) / np.float32(16.0))
    x[0] = 0.0
    x[1] = orc.bf16_round(x[1] * np.float32(2.0 ** -120))      # below the clamp: E = -100
    x[2] = orc.bf16_round(x[2] * np.float32(2.0 ** 60))        # huge
    x[3] = 0.0
    x[3, 17] = np.float32(-3.0)                                 # one element
    x[4] = orc.bf16_round(np.full(d, 0.5, np.float32))          # constant row
    w[1] = orc.bf16_round(w[1] * np.float32(2.0 ** -110))
    w[2] = w[0]                                                 # duplicated expert
    got = orc.router_logits(x, w)
    assert np.isfinite(got).all()

    def grid(row, win):
        m = max(abs(float(v)) for v in row)
        ef = 0 if m == 0 else int(np.frexp(np.float32(m))[1]) + 126
        e = max(ef - 126, -100)
        return [int(np.rint(float(v) * 2.0 ** (win - e))) for v in row], e

    for t in range(x.shape[0]):
        qx, ex = grid(x[t], 21)
        for e in range(w.shape[0]):
            qw, ew = grid(w[e], 14)
            s = sum(a * b for a, b in zip(qx, qw))
            assert got[t, e] == np.float32(_rne_f32(s) * 2.0 ** (ex + ew - 35)), (t, e)
    assert (got[:, 0] == got[:, 2]).all()
    assert (got[0] == 0).all() and (got[3, :] == got[3, :]).all()
