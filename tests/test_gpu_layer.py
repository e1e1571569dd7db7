"""Single-GPU parity of the whole MoE-layer forward (G = 1) against the oracle.

Bit-exact: routed indices, histogram, per-pair receive positions, count table.
Tolerance (floating point, stated in tests/tolerance.py): per element
|out - ref| <= 2^-7 * (mag2 + 2 mag) + 1e-5 * max|ref| (one bf16 ulp of every
term the element is made of) and relative Frobenius error <= 3e-3.
"""

import numpy as np
import pytest

from oracle import moe_oracle as orc

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

from tolerance import check_layer_close


def _shape(name):
    from paper_2508_12851_b200.shapes import LayerShape
    small = {
        "toy": LayerShape("toy", d=512, f=2048, E=8, k=2),
        "qwen_small": LayerShape("qwen_small", d=256, f=256, E=60, k=4, score_mode=1, shared_f=512, shared_gate=1),
        "ds_small": LayerShape("ds_small", d=256, f=384, E=64, k=6, score_mode=1, shared_f=256),
        "mixtral_narrow": LayerShape("mixtral_narrow", d=4096, f=512, E=8, k=2),
    }
    return small[name]


def _weights(shape, seed=0):
    experts = {e: orc.synthetic_expert(e, shape.d, shape.f, seed) for e in range(shape.E)}
    shared = orc.synthetic_expert(999, shape.d, shape.shared_f, seed) if shape.shared_f else None
    wg = orc.synthetic_router(shape.E + shape.shared_gate, shape.d, seed)
    return experts, shared, wg


def _build_layer(shape, T, experts, shared, wg, bias, cap=None):
    from paper_2508_12851_b200.layer import B200MoELayer
    layer = B200MoELayer(shape, max_tokens=T, cap_slots=cap or shape.E)
    E = shape.E
    layer.set_router(torch.from_numpy(wg[:E]), torch.from_numpy(bias),
                     torch.from_numpy(wg[E]) if shape.shared_gate else None)
    if shared is not None:
        layer.set_shared(*(torch.from_numpy(w) for w in shared))
    src = lambda e: tuple(torch.from_numpy(w) for w in experts[e])
    layer.set_placement_sets([list(range(E))], src)
    return layer


def _check_close(got, ref, mag, mag2):
    check_layer_close(got, ref, mag, mag2)


@pytest.mark.parametrize("pair", ["0", "1"], ids=["cta1", "cta_pair"])
@pytest.mark.parametrize("name,T", [("toy", 256), ("toy", 77), ("qwen_small", 200), ("ds_small", 300),
                                    ("mixtral_narrow", 130)])
def test_layer_g1_matches_oracle(name, T, pair, monkeypatch):
    monkeypatch.setenv("MP_GEMM_PAIR", pair)
    shape = _shape(name)
    experts, shared, wg = _weights(shape)
    x = orc.synthetic_tokens(0, T, shape.d, seed=5)
    bias = orc.origin_bias(0, shape.E, seed=5)
    layer = _build_layer(shape, max(T, 64), experts, shared, wg, bias)
    out = layer.forward(torch.from_numpy(x).cuda().bfloat16())
    torch.cuda.synchronize()
    layer.check()

    route = np.zeros((1, shape.E), dtype=np.int32)
    ref = orc.moe_layer_forward(shape, [x], wg[:shape.E], [bias], route, experts, shared,
                                wg[shape.E] if shape.shared_gate else None)
    # bit-exact routing / dispatch
    assert np.array_equal(layer.idx[:T].cpu().numpy(), ref.idx[0])
    assert np.array_equal(layer.activation_counts(), ref.hist[0])
    assert np.array_equal(layer.read_counts(), ref.counts)
    assert np.array_equal(layer.pos_dst[:T].cpu().numpy(), ref.pos_dst[0])
    assert np.array_equal(layer.pos_row[:T].cpu().numpy(), ref.pos_row[0])
    # received rows are exactly the permuted token rows
    rows = ref.pos_row[0].ravel()
    recv = layer.recv[: rows.max() + 1].float().cpu().numpy()
    np.testing.assert_array_equal(recv[rows], np.repeat(x, shape.k, axis=0))
    _check_close(out.float().cpu().numpy(), ref.out[0], ref.mag[0], ref.mag2[0])
    acc = layer.dispatch_accounting()
    assert acc["remote_invocations"] == 0 and acc["local_ratio"] == 1.0
    layer.close()


def test_layer_repeated_forwards_accumulate_histogram():
    shape = _shape("toy")
    experts, shared, wg = _weights(shape)
    T = 128
    x = orc.synthetic_tokens(1, T, shape.d, seed=2)
    bias = orc.origin_bias(2, shape.E, seed=2)
    layer = _build_layer(shape, T, experts, shared, wg, bias)
    xt = torch.from_numpy(x).cuda().bfloat16()
    o1 = layer.forward(xt).clone()
    o2 = layer.forward(xt)
    torch.cuda.synchronize()
    assert torch.equal(o1, o2)  # deterministic
    idx = orc.topk_route(orc.router_logits(x, wg, bias), shape.E, shape.k, 0)[0]
    assert np.array_equal(layer.activation_counts(), 2 * orc.histogram(idx, shape.E))
    assert layer.last_launches() >= 5
    # the router's last-CTA ticket and batch-count accumulator are back at zero between
    # forwards (mp_layer_sync_state [3], [7]); no peer protocol at G = 1
    st = layer.sync_state()
    assert st[3] == 0 and st[7] == 0 and st[6] == 0, st
    layer.close()


def test_layer_empty_batch():
    shape = _shape("toy")
    experts, shared, wg = _weights(shape)
    layer = _build_layer(shape, 64, experts, shared, wg, np.zeros(shape.E, np.float32))
    x = torch.empty(0, shape.d, device="cuda", dtype=torch.bfloat16)
    out = layer.forward(x)
    torch.cuda.synchronize()
    assert out.shape == (0, shape.d)
    assert layer.activation_counts().sum() == 0
    layer.close()


def test_route_to_unplaced_expert_raises():
    from paper_2508_12851_b200 import UnplacedExpertError
    shape = _shape("toy")
    experts, shared, wg = _weights(shape)
    layer = _build_layer(shape, 64, experts, shared, wg, np.zeros(shape.E, np.float32))
    bad_slots = layer.slot_of.copy()
    bad_slots[3] = -1
    with pytest.raises(UnplacedExpertError):
        layer.set_routes(np.zeros((1, shape.E), np.int32), bad_slots)
    layer.close()


@pytest.mark.parametrize("depth", [1, 2, 3])
def test_host_pipeline_matches_device_forward(depth):
    """HostPipeline (the bench's e2e path): pinned host batches in, host outputs out, copies on
    their own streams with `depth` device buffers -- every host output equals the device-side
    forward of the same batch."""
    from paper_2508_12851_b200.layer import HostPipeline
    shape = _shape("toy")
    T = 96
    experts, shared, wg = _weights(shape)
    bias = orc.origin_bias(0, shape.E, seed=2)
    layer = _build_layer(shape, T, experts, shared, wg, bias)
    xs = [torch.from_numpy(orc.synthetic_tokens(0, T, shape.d, seed=20 + i)).bfloat16() for i in range(5)]
    ref = [layer.forward(x.cuda()).cpu() for x in xs]
    xh = [x.pin_memory() for x in xs]
    oh = [torch.empty(T, shape.d, dtype=torch.bfloat16).pin_memory() for _ in xs]
    pipe = HostPipeline(layer, T, depth=depth)
    for x, o in zip(xh, oh):
        pipe.submit(x, o)
    pipe.drain()
    torch.cuda.synchronize()
    for i in range(len(xs)):
        assert torch.equal(oh[i], ref[i]), i
    layer.close()


def test_large_batch_block_scan_from_global():
    """T large enough that the router's [blocks][E] count matrix (1250 x 64 ints) no longer
    fits the last CTA's shared memory: the block scan reads it from global memory instead.
    Routing, counts and receive positions stay bit-exact."""
    from paper_2508_12851_b200.shapes import LayerShape
    shape = LayerShape("wide_batch", d=256, f=128, E=64, k=6, score_mode=1)
    T = 40_000
    experts, shared, wg = _weights(shape)
    x = orc.synthetic_tokens(0, T, shape.d, seed=8)
    bias = orc.origin_bias(0, shape.E, seed=8)
    layer = _build_layer(shape, T, experts, shared, wg, bias)
    out = layer.forward(torch.from_numpy(x).cuda().bfloat16())
    torch.cuda.synchronize()
    layer.check()
    route = np.zeros((1, shape.E), dtype=np.int32)
    ref = orc.moe_layer_forward(shape, [x], wg[:shape.E], [bias], route, experts, shared, None)
    assert np.array_equal(layer.idx[:T].cpu().numpy(), ref.idx[0])
    assert np.array_equal(layer.read_counts(), ref.counts)
    assert np.array_equal(layer.pos_row[:T].cpu().numpy(), ref.pos_row[0])
    _check_close(out.float().cpu().numpy(), ref.out[0], ref.mag[0], ref.mag2[0])
    layer.close()


@pytest.mark.parametrize("name,T", [("toy", 200), ("ds_small", 300), ("qwen_small", 150)])
def test_stage_entries_match_fused_forward(name, T):
    """The stage entries (mp_layer_route / _permute / _experts / _combine_gather, the kernels of
    the host-driven NCCL transport) reproduce the fused forward bit for bit at G = 1."""
    from paper_2508_12851_b200.nccl_path import NcclForward
    shape = _shape(name)
    experts, shared, wg = _weights(shape)
    x = orc.synthetic_tokens(0, T, shape.d, seed=6)
    bias = orc.origin_bias(0, shape.E, seed=6)
    layer = _build_layer(shape, T, experts, shared, wg, bias)
    xt = torch.from_numpy(x).cuda().bfloat16()
    fused = layer.forward(xt).clone()
    pos = layer.pos_row[:T].clone()
    staged = NcclForward(layer).forward(xt)
    torch.cuda.synchronize()
    assert torch.equal(staged, fused)
    assert torch.equal(layer.pos_row[:T], pos)
    layer.close()
