"""Trace export (F4) and measured-cost calibration (F1) against the reference (CPU)."""

import numpy as np
import pytest

from oracle import moe_oracle as orc
from paper_2508_12851_b200.calibrate import calibrated_time_model, fit_linear_cost, remote_penalty_seconds
from paper_2508_12851_b200.errors import import_moeplace
from paper_2508_12851_b200.trace import counts_from_records, trace_records, write_trace


def _idx(seed, T=300, E=16, k=3):
    x = orc.synthetic_tokens(seed, T, 256, seed)
    wg = orc.synthetic_router(E, 256, seed)
    return orc.topk_route(orc.router_logits(x, wg, orc.origin_bias(seed, E, seed)), E, k, 1)[0]


def test_trace_records_reproduce_histogram():
    idx = _idx(1)
    recs = trace_records(idx, server=2, layer=1, t=5.0)
    c = counts_from_records(recs, 3, (16, 16))
    assert np.array_equal(c[2, 1], orc.histogram(idx, 16))
    assert sum(r["tokens"] for r in recs) == idx.shape[0]


def test_trace_roundtrip_through_reference_parse_trace(tmp_path):
    mp = import_moeplace()
    if mp is None:
        pytest.skip("reference not importable")
    from moeplace.cli import parse_trace
    idxs = {s: _idx(s) for s in range(3)}
    path = str(tmp_path / "trace.jsonl")
    for s, idx in idxs.items():
        write_trace(path, trace_records(idx, s, 0, t=float(s)), append=s > 0)
    model = mp.ModelSpec(1, (16,), 3, 1e6, 256)
    events = parse_trace(path, model, 3)
    stats = mp.ActivationStats(3, (16,))
    for ev in events:
        stats.ingest(ev)
    for s, idx in idxs.items():
        assert np.array_equal(stats.counts[s, 0].astype(np.int64), orc.histogram(idx, 16))


def test_fit_linear_cost():
    t = np.array([256, 1024, 4096, 16384])
    base, per = fit_linear_cost(t, 20e-6 + 0.5e-6 * t)
    assert base == pytest.approx(20e-6, rel=1e-6) and per == pytest.approx(0.5e-6, rel=1e-9)
    with pytest.raises(ValueError):
        fit_linear_cost([5, 5], [1, 1])


def test_calibrated_time_model_prices_like_the_reference():
    mp = import_moeplace()
    if mp is None:
        pytest.skip("reference not importable")
    from paper_2508_12851_b200.shapes import MIXTRAL, cluster_spec, model_spec
    cluster, model = cluster_spec(MIXTRAL, 4), model_spec(MIXTRAL)
    samples = [[(1024, 1e-4 + 1024 * 2.5e-7), (4096, 1e-4 + 4096 * 2.5e-7)] for _ in range(4)]
    tm = calibrated_time_model(cluster, samples, link_bandwidth=770e9, link_latency=3e-6)
    assert mp.comp_time(tm, 0, 2048) == pytest.approx(1e-4 + 2048 * 2.5e-7)
    # comm_time with the measured link (cost.py:139-149)
    assert mp.comm_time(tm, 0, 1, 1, model) == pytest.approx(3e-6 + 2 * 4096 * 2 / 770e9)
    assert remote_penalty_seconds(4096, 770e9) == pytest.approx(2 * 4096 * 2 / 770e9)
