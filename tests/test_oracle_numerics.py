"""Oracle self-consistency (CPU): router order contract, permutation, layer algebra."""

import numpy as np
import pytest

from oracle import moe_oracle as orc


def test_bf16_round_matches_torch():
    torch = pytest.importorskip("torch")
    a = np.random.default_rng(0).standard_normal(10000).astype(np.float32) * 100
    ref = torch.from_numpy(a).bfloat16().float().numpy()
    np.testing.assert_array_equal(orc.bf16_round(a), ref)


def test_router_logits_contract():
    """32 lane chains over 8-wide k slices strided by 256, then the butterfly tree."""
    rng = np.random.default_rng(1)
    d = 512
    x = orc.bf16_round(rng.standard_normal((3, d)).astype(np.float32))
    w = orc.bf16_round(rng.standard_normal((5, d)).astype(np.float32))
    got = orc.router_logits(x, w)
    for t in range(3):
        for e in range(5):
            p = []
            for lane in range(32):
                acc = np.float32(0)
                for s in range(d // 256):
                    for j in range(8):
                        k = 256 * s + 8 * lane + j
                        acc = np.float32(acc + np.float32(x[t, k] * w[e, k]))
                p.append(acc)
            for o in (16, 8, 4, 2, 1):
                p = [np.float32(p[i] + p[i + o]) for i in range(o)]
            assert got[t, e] == p[0]
    np.testing.assert_allclose(got, x @ w.T, rtol=1e-4, atol=1e-3)


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
