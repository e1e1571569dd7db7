"""Shared expert fused into the routed CTA-pair launches (K3 plan `fuse_shared`).

The fused launch only reschedules whole 256x256 tiles (aux tiles round-robin,
routed tiles round-robin with a deficit tail for the clusters that drew fewer
aux tiles); each tile's k-loop order is unchanged, so the layer output must be BIT-IDENTICAL to the unfused plan (shared
expert in its own two launches) for every token count and cluster count.  The
unfused plan itself is checked against the oracle in test_gpu_layer.py.
"""

import numpy as np
import pytest

from oracle import moe_oracle as orc

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu


def _shape(name):
    from paper_2508_12851_b200.shapes import LayerShape
    return {
        "qwen_small": LayerShape("qwen_small", d=256, f=256, E=60, k=4, score_mode=1, shared_f=512, shared_gate=1),
        "ds_mid": LayerShape("ds_mid", d=1024, f=384, E=64, k=6, score_mode=1, shared_f=768),
    }[name]


def _run(shape, T, env, monkeypatch):
    from paper_2508_12851_b200.layer import B200MoELayer
    env = {"MP_STREAM_ROWS": "0", **env}  # these tests pin the split / fused plan at every T
    for k, v in env.items():
        monkeypatch.setenv(k, v)
    experts = {e: orc.synthetic_expert(e, shape.d, shape.f, 0) for e in range(shape.E)}
    shared = orc.synthetic_expert(999, shape.d, shape.shared_f, 0)
    wg = orc.synthetic_router(shape.E + shape.shared_gate, shape.d, 0)
    bias = orc.origin_bias(0, shape.E, seed=3)
    layer = B200MoELayer(shape, max_tokens=max(T, 64), cap_slots=shape.E)
    E = shape.E
    layer.set_router(torch.from_numpy(wg[:E]), torch.from_numpy(bias),
                     torch.from_numpy(wg[E]) if shape.shared_gate else None)
    layer.set_shared(*(torch.from_numpy(w) for w in shared))
    layer.set_placement_sets([list(range(E))], lambda e: tuple(torch.from_numpy(w) for w in experts[e]))
    x = torch.from_numpy(orc.synthetic_tokens(0, T, shape.d, seed=9)).cuda().bfloat16()
    out = layer.forward(x)
    torch.cuda.synchronize()
    layer.check()
    plan = layer.exec_plan()
    res = out.cpu()
    layer.close()
    for k in env:
        monkeypatch.delenv(k)
    return res, plan


@pytest.mark.parametrize("name", ["qwen_small", "ds_mid"])
@pytest.mark.parametrize("T", [1, 130, 600, 2048])
def test_fused_shared_bit_identical(name, T, monkeypatch):
    shape = _shape(name)
    ref, p0 = _run(shape, T, {"MP_FUSE_SHARED": "0"}, monkeypatch)
    assert p0["fuse_shared"] == 0
    got, p1 = _run(shape, T, {}, monkeypatch)
    assert p1["fuse_shared"] == 1 and p1["pair_routed"] == 1
    assert torch.equal(got, ref)
    # different cluster counts for the big chain change every cluster's range
    for grid in ("8", "40"):
        g, p = _run(shape, T, {"MP_GEMM_SMALL_GRID": grid}, monkeypatch)
        assert p["small_grid"] == int(grid)
        assert torch.equal(g, ref), grid


@pytest.mark.parametrize("name", ["qwen_small", "ds_mid"])
@pytest.mark.parametrize("T", [64, 700])
def test_stream_plan_matches_split_plan(name, T, monkeypatch):
    """Small batches stream every group over all SMs (1-CTA kernel, shared expert as its aux
    problem) instead of the split / pair-fused plan: same products, different tile shapes,
    equal within bf16 rounding of the tensor-core accumulation."""
    shape = _shape(name)
    ref, p0 = _run(shape, T, {}, monkeypatch)
    got, p1 = _run(shape, T, {"MP_STREAM_ROWS": "1000000"}, monkeypatch)
    assert p0["split_m"] > 0 and p1["split_m"] == 0 and p1["pair_routed"] == 0
    assert p1["fuse_shared"] == 1      # the shared expert rides in the 1-CTA routed launches
    r, g = ref.float(), got.float()
    assert ((g - r).abs().max() <= 1e-2 * r.abs().max() + 1e-3).item()
    assert ((g - r).norm() / r.norm()).item() <= 5e-3


@pytest.mark.parametrize("T", [1, 200, 1000])
def test_stream_plan_fused_shared_matches_separate(T, monkeypatch):
    """Stream plan: the shared expert as the aux problem of the 1-CTA launches against its own
    launches (MP_FUSE_SHARED=0)."""
    shape = _shape("qwen_small")
    env = {"MP_STREAM_ROWS": "1000000"}
    ref, p0 = _run(shape, T, {**env, "MP_FUSE_SHARED": "0"}, monkeypatch)
    got, p1 = _run(shape, T, env, monkeypatch)
    assert p0["fuse_shared"] == 0 and p1["fuse_shared"] == 1 and p1["pair_routed"] == 0
    r, g = ref.float(), got.float()
    assert ((g - r).abs().max() <= 1e-2 * r.abs().max() + 1e-3).item()
    assert ((g - r).norm() / r.norm()).item() <= 5e-3
