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


def remote_penalty_seconds(d: int, link_bandwidth: float, bpe: int = 2) -> float:
    """Mean extra seconds one remote (token, expert) invocation costs: activations out and
    results back over the link (the bandwidth term of comm_time, cost.py:148), per token-unit --
    the `avg_remote_penalty_seconds` of a CostSnapshot (cost.py:194-214)."""
    return 2.0 * d * bpe / float(link_bandwidth)
