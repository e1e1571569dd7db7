"""Measured-cost feedback into the reference's decision layer.

The reference prices placements with an analytic TimeModel: compute
`(comp_base + comp_per_token * tokens) * load` (cost.py:132-136) and transfers
`latency + 2 * payload / bandwidth` (cost.py:139-149), with defaults of 2 ms,
50 us/token and a 500 Mbps network (cost.py:68-78).  On a B200
box those constants are measurable: this module fits them from layer timings
and builds the reference TimeModel / CostSnapshot inputs from real numbers.
"""

from __future__ import annotations

import numpy as np


def fit_linear_cost(tokens, seconds) -> tuple[float, float]:
    """Least-squares fit seconds ~= base + per_token * tokens (base, per_token >= 0)."""
    t = np.asarray(tokens, dtype=float)
    s = np.asarray(seconds, dtype=float)
    if t.size < 2 or np.ptp(t) == 0:
        raise ValueError("need at least two distinct token counts")
    A = np.stack([np.ones_like(t), t], axis=1)
    (base, per_tok), *_ = np.linalg.lstsq(A, s, rcond=None)
    if per_tok < 0:
        per_tok = 0.0
        base = float(s.mean())
    return max(0.0, float(base)), float(per_tok)


def calibrated_time_model(cluster, comp_samples, link_bandwidth: float | None = None,
                          link_latency: float | None = None):
    """A reference TimeModel whose constants come from B200 measurements.

    comp_samples: per server, a list of (tokens, seconds) pairs of expert compute
    (e.g. the K3 stage time at several batch sizes); link_bandwidth / latency:
    measured NVLink figures replacing the cluster's link matrices.
    """
    from .errors import import_moeplace

    mp = import_moeplace()
    if mp is None:
        raise RuntimeError("the reference package moeplace is not importable")
    G = cluster.num_servers
    bases, per = [], []
    for n in range(G):
        b, p = fit_linear_cost([t for t, _ in comp_samples[n]], [s for _, s in comp_samples[n]])
        bases.append(b)
        per.append(p)
    bw = np.array(cluster.link_bandwidth, dtype=float)
    lat = np.array(cluster.link_latency, dtype=float)
    if link_bandwidth is not None:
        bw = np.full((G, G), float(link_bandwidth))
    if link_latency is not None:
        lat = np.full((G, G), float(link_latency))
        np.fill_diagonal(lat, 0.0)
    return mp.TimeModel(np.array(bases), np.array(per), bw, lat)


def observed_remote_penalty(step_s_a: float, remote_a: float, step_s_b: float, remote_b: float) -> float:
    """Measured mean extra seconds per remote (token, expert) invocation: the step-time difference
    of two runs of the same batch size whose placements send different numbers of invocations
    remote, over that difference -- the quantity the reference accumulates per remote invocation
    as `penalty_seconds / penalty_volume` (sim.py:455-456, 469) and hands to CostSnapshot
    (cost.py:195-214) as avg_remote_penalty_seconds."""
    dr = float(remote_b) - float(remote_a)
    if abs(dr) < 1.0:
        return 0.0
    return max(0.0, (float(step_s_b) - float(step_s_a)) / dr)


def invocations_of(counts, route, layer: int = 0):
    """The forward as the reference's ExpertInvocation records (cost.py:89-101): one per (origin,
    expert) with the origin's routed tokens, target = route[origin][expert]."""
    from .errors import import_moeplace

    mp = import_moeplace()
    counts = np.asarray(counts)
    return [mp.ExpertInvocation(int(s), int(route[s][e]), 0, layer, int(e), int(counts[s, e]))
            for s in range(counts.shape[0]) for e in range(counts.shape[1]) if counts[s, e] > 0]


def predicted_layer_latency(time_model, placement, model_spec, counts, route) -> dict:
    """The reference's latency model on a measured forward: `layer_latency` (cost.py:152-168, the
    max rule over independent invocations) and, since one GPU runs all of its groups in one
    grouped GEMM, the same model with every GPU's rows as one batch (comp_time of the GPU's total
    rows + the slowest remote transfer into it)."""
    from .errors import import_moeplace

    mp = import_moeplace()
    counts = np.asarray(counts)
    inv = invocations_of(counts, route)
    per_inv = mp.layer_latency(inv, placement, time_model, model_spec)
    G = counts.shape[0]
    rows = np.zeros(G, dtype=np.int64)
    worst_comm = np.zeros(G)
    for s in range(G):
        for e in range(counts.shape[1]):
            if counts[s, e] <= 0:
                continue
            D = int(route[s][e])
            rows[D] += counts[s, e]
            worst_comm[D] = max(worst_comm[D], mp.comm_time(time_model, s, D, int(counts[s, e]), model_spec))
    agg = max(worst_comm[D] + mp.comp_time(time_model, D, int(rows[D])) for D in range(G) if rows[D] > 0)
    return {"layer_latency_per_invocation_s": float(per_inv), "layer_latency_per_gpu_batch_s": float(agg),
            "rows_per_gpu": rows.tolist()}


def remote_penalty_seconds(d: int, link_bandwidth: float, bpe: int = 2) -> float:
    """Mean extra seconds one remote (token, expert) invocation costs: activations out and
    results back over the link (the bandwidth term of comm_time, cost.py:148), per token-unit --
    the `avg_remote_penalty_seconds` of a CostSnapshot (cost.py:194-214)."""
    return 2.0 * d * bpe / float(link_bandwidth)
