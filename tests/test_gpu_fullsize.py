"""Full BASELINE.json sizes on one B200: every token checked, no sampling.

Sizes: Mixtral-8x7B (d 4096, f 14336, E 8, k 2) at T = 4096 (the bench
workload), Qwen1.5-MoE-A2.7B at T = 4096 and DeepSeek-V2-Lite (E 64, k 6,
2 shared) at T = 4096 and at the maximum T = 16384.
  * routing: every token's indices bit-exact and weights to fp32 rounding
    against oracle.router_logits / topk_route (the exact-integer contract is
    cheap in numpy at these sizes); histogram == bincount;
  * permutation: the receive rows of all (token, slot) pairs are a dense
    permutation of 0..T*k-1 equal to the oracle's positions, and every
    received row equals its token's x row;
  * outputs: every element against the GPU fp32 restatement
    (tests/torch_ref.py: the oracle's arithmetic in torch fp32, bf16 h / y /
    out) within tests/tolerance.py's bound;
  * determinism: a second forward is bit-identical.
"""

import numpy as np
import pytest

from oracle import moe_oracle as orc
from tolerance import check_layer_close

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu


def _run(shape, T, seed=0):
    from paper_2508_12851_b200 import workload as wl
    from paper_2508_12851_b200.layer import B200MoELayer
    from torch_ref import layer_reference
    dev = torch.device("cuda", 0)
    E, k = shape.E, shape.k
    wg = wl.router_weights(E + shape.shared_gate, shape.d, dev, seed)
    bias = wl.origin_bias(0, E, seed)
    layer = B200MoELayer(shape, max_tokens=T, cap_slots=E, staging_slots=0)
    layer.set_router(wg[:E], bias, wg[E] if shape.shared_gate else None)
    shared = wl.shared_weights(shape.d, shape.shared_f, dev, seed) if shape.shared_f else None
    if shared is not None:
        layer.set_shared(*shared)
    src = lambda e: wl.expert_weights(e, shape.d, shape.f, dev, seed)
    layer.set_placement_sets([list(range(E))], src)
    x = wl.tokens(T, shape.d, dev, seed, 0, batch=7)
    out = layer.forward(x)
    out2 = layer.forward(x)
    torch.cuda.synchronize()
    layer.check()

    # determinism
    assert torch.equal(out, out2)
    # routing, every token, bit-exact against the oracle's contract
    x_np = x.float().cpu().numpy()
    lg = orc.router_logits(x_np, wg.float().cpu().numpy(), bias.numpy())
    idx_ref, w_ref = orc.topk_route(lg, E, k, shape.score_mode, shape.renorm)
    idx = layer.idx[:T].cpu().numpy()
    assert np.array_equal(idx, idx_ref)
    np.testing.assert_allclose(layer.gate_w[:T].cpu().numpy(), w_ref, rtol=1e-5, atol=1e-6)
    hist = layer.activation_counts() // 2          # two forwards
    assert np.array_equal(hist, orc.histogram(idx_ref, E))
    gate = None
    if shape.shared_gate:
        gate = (1.0 / (1.0 + np.exp(-lg[:, E].astype(np.float64)))).astype(np.float32)
        np.testing.assert_allclose(layer.shared_gate[:T].cpu().numpy(), gate, rtol=1e-5, atol=1e-6)
    # permutation: oracle positions, dense, and every received row is its token's row
    route = np.zeros((1, E), np.int32)
    _, _, send = orc.receive_layout(orc.histogram(idx_ref, E)[None], route)
    _, rows_ref = orc.pair_positions(idx_ref, route[0], send[0])
    rows = layer.pos_row[:T].cpu().numpy()
    assert np.array_equal(rows, rows_ref)
    assert np.array_equal(np.sort(rows.ravel()), np.arange(T * k))
    rows_d = torch.from_numpy(rows.ravel()).long().to(dev)
    assert torch.equal(layer.recv[rows_d], x.repeat_interleave(k, dim=0))
    # every output element against the GPU fp32 restatement
    ref, mag, mag2 = layer_reference(x, idx_ref, w_ref, src, shared, gate)
    stats = check_layer_close(out.float().cpu().numpy(), ref.cpu().numpy(), mag.cpu().numpy(), mag2.cpu().numpy(),
                              shape.name)
    print(f"{shape.name} T={T} plan={layer.exec_plan()} {stats}")
    layer.close()


def test_mixtral_full_size_T4096():
    from paper_2508_12851_b200.shapes import MIXTRAL
    _run(MIXTRAL, 4096)


def test_deepseek_full_size_T4096():
    from paper_2508_12851_b200.shapes import DEEPSEEK
    _run(DEEPSEEK, 4096)


def test_deepseek_full_size_max_tokens():
    from paper_2508_12851_b200.shapes import DEEPSEEK
    _run(DEEPSEEK, 16384)


def test_qwen_full_size_T4096():
    from paper_2508_12851_b200.shapes import QWEN
    _run(QWEN, 4096)
