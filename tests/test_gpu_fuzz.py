"""Randomised layer shapes against the oracle (G = 1).

Each seed draws a layer shape (hidden width, FFN width, expert count, top-k,
router mode, renormalisation, shared expert with or without its sigmoid gate),
a token count and a routing skew, then checks the whole forward the same way as
test_gpu_layer.py: routing indices, histogram, count table, per-pair receive
positions and received rows bit-exact; the output within the stated tolerance.
The shapes cover every K3 plan (1-CTA only, CTA pairs, small-group side chain,
fused shared expert) and every router variant.
"""

import os

import numpy as np
import pytest

from oracle import moe_oracle as orc
from tolerance import check_layer_close

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu


def _draw(seed):
    from paper_2508_12851_b200.shapes import LayerShape
    r = np.random.default_rng(1000 + seed)
    E = int(r.choice([4, 8, 16, 24, 32, 60, 64]))
    k = int(r.integers(1, min(8, E) + 1))
    d = int(r.choice([256, 512, 768, 1024, 2048, 3072, 4096]))  # 1..8 router K ranges, odd k-block counts
    f = int(r.choice([128, 256, 384, 512, 640]))
    mode = int(r.integers(0, 2))
    renorm = int(r.integers(0, 2)) if mode == 1 else 0
    shared_f = int(r.choice([0, 0, 256, 512]))
    gate = int(r.integers(0, 2)) if shared_f else 0
    T = int(r.integers(1, 700))
    alpha = float(r.choice([0.1, 0.3, 1.0]))
    shape = LayerShape(f"fuzz{seed}", d=d, f=f, E=E, k=k, score_mode=mode, renorm=renorm, shared_f=shared_f,
                       shared_gate=gate)
    return shape, T, alpha


# MP_FUZZ_SEEDS=a:b widens the sweep for a dedicated fuzz run (the suite default: 40 seeds)
_SEEDS = range(*map(int, os.environ.get("MP_FUZZ_SEEDS", "0:40").split(":")))


@pytest.mark.parametrize("seed", _SEEDS)
def test_random_layer_matches_oracle(seed):
    from paper_2508_12851_b200.layer import B200MoELayer
    shape, T, alpha = _draw(seed)
    E = shape.E
    experts = {e: orc.synthetic_expert(e, shape.d, shape.f, seed) for e in range(E)}
    shared = orc.synthetic_expert(999, shape.d, shape.shared_f, seed) if shape.shared_f else None
    wg = orc.synthetic_router(E + shape.shared_gate, shape.d, seed)
    p = np.random.default_rng(seed).dirichlet(np.full(E, alpha))
    bias = np.log(p * (1 - 1e-9) + 1e-9 / E).astype(np.float32)
    x = orc.synthetic_tokens(0, T, shape.d, seed=seed)

    layer = B200MoELayer(shape, max_tokens=T, cap_slots=E)
    layer.set_router(torch.from_numpy(wg[:E]), torch.from_numpy(bias),
                     torch.from_numpy(wg[E]) if shape.shared_gate else None)
    if shared is not None:
        layer.set_shared(*(torch.from_numpy(w) for w in shared))
    layer.set_placement_sets([list(range(E))], lambda e: tuple(torch.from_numpy(w) for w in experts[e]))
    out = layer.forward(torch.from_numpy(x).cuda().bfloat16())
    torch.cuda.synchronize()
    layer.check()

    route = np.zeros((1, E), dtype=np.int32)
    ref = orc.moe_layer_forward(shape, [x], wg[:E], [bias], route, experts, shared,
                                wg[E] if shape.shared_gate else None)
    tag = f"{shape} T={T} plan={layer.exec_plan()}"
    assert np.array_equal(layer.idx[:T].cpu().numpy(), ref.idx[0]), tag
    assert np.array_equal(layer.activation_counts(), ref.hist[0]), tag
    assert np.array_equal(layer.read_counts(), ref.counts), tag
    assert np.array_equal(layer.pos_row[:T].cpu().numpy(), ref.pos_row[0]), tag
    rows = ref.pos_row[0].ravel()
    recv = layer.recv[: rows.max() + 1].float().cpu().numpy()
    np.testing.assert_array_equal(recv[rows], np.repeat(x, shape.k, axis=0))
    check_layer_close(out.float().cpu().numpy(), ref.out[0], ref.mag[0], ref.mag2[0], tag)
    layer.close()
