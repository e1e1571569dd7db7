"""Host-side route tables: the reference's target rule, evaluated once per placement.

`_EventLoop._choose_target` (reference pkg/src/moeplace/sim.py:433-439) picks,
per (origin, layer, expert) invocation, the origin itself when it holds the
expert, else the holder with the smallest `comm_time` (cost.py:139-149), ties
to the lowest server id, and raises when no server holds the expert.  The B200
path folds that rule into a [G, E] table per layer, uploaded to every GPU, so
the permute kernel only reads `route[origin][expert]`.

Placements are the reference's `Placement` objects (domain.py:222-319), used
through their public API only (`server_experts`, `holders`, `gpu_sets`), or a
placement document in the reference JSON format (`Placement.to_dict`,
domain.py:281-289).
"""

from __future__ import annotations

import numpy as np

from .errors import DimensionMismatch, InfeasibleError


def _comm_time(src: int, dst: int, tokens: int, latency, bandwidth, d: int, bpe: int) -> float:
    if src == dst:
        return 0.0
    payload = float(max(1, int(tokens))) * d * bpe
    return float(latency[src][dst] + 2.0 * payload / bandwidth[src][dst])


def server_expert_sets(placement, layer: int = 0) -> list[frozenset]:
    """Per-server expert sets of one layer (Placement.server_experts, domain.py:246-250)."""
    if isinstance(placement, dict):
        entry = next(e for e in placement["layers"] if e["layer"] == layer)
        servers = sorted(entry["servers"], key=lambda s: s["server"])
        return [frozenset(e for gpu in s["gpus"] for e in gpu) for s in servers]
    return [frozenset(placement.server_experts(n, layer)) for n in range(placement.num_servers)]


def gpu_expert_sets(placement, layer: int = 0) -> list[list[int]]:
    """Experts held by GPU 0 of every server for one layer (servers have one GPU each here)."""
    if isinstance(placement, dict):
        entry = next(e for e in placement["layers"] if e["layer"] == layer)
        servers = sorted(entry["servers"], key=lambda s: s["server"])
        out = []
        for s in servers:
            if len(s["gpus"]) != 1:
                raise DimensionMismatch(f"server {s['server']} has {len(s['gpus'])} GPUs; the B200 path maps one GPU per server")
            out.append(sorted(int(e) for e in s["gpus"][0]))
        return out
    out = []
    for n, srv in enumerate(placement.gpu_sets):
        if len(srv) != 1:
            raise DimensionMismatch(f"server {n} has {len(srv)} GPUs; the B200 path maps one GPU per server")
        out.append(sorted(e for (l, e) in srv[0] if l == layer))
    return out


def route_table(server_sets, E: int, link_latency, link_bandwidth, d: int, bpe: int = 2,
                tokens: int = 1) -> np.ndarray:
    """route[s, e] per `_choose_target` (sim.py:433-439); tokens = 1 per routed token."""
    G = len(server_sets)
    holders = {e: [n for n in range(G) if e in server_sets[n]] for e in range(E)}
    route = np.empty((G, E), dtype=np.int32)
    for s in range(G):
        for e in range(E):
            if e in server_sets[s]:
                route[s, e] = s
                continue
            if not holders[e]:
                raise RuntimeError(f"expert {e} of layer is placed nowhere")
            route[s, e] = min(holders[e], key=lambda n: (_comm_time(s, n, tokens, link_latency, link_bandwidth, d, bpe), n))
    return route


def route_table_for(placement, cluster, E: int, d: int, bpe: int = 2, layer: int = 0) -> np.ndarray:
    """Route table from a reference Placement + ClusterSpec (link matrices domain.py:73-107)."""
    return route_table(server_expert_sets(placement, layer), E, cluster.link_latency, cluster.link_bandwidth, d, bpe)


def uniform_links(G: int, latency: float = 3e-6, bandwidth: float = 770e9):
    lat = np.full((G, G), latency)
    np.fill_diagonal(lat, 0.0)
    return lat, np.full((G, G), bandwidth)


def slot_map(experts: list[int], E: int, n_slots: int) -> np.ndarray:
    """slot_of[e] for one GPU: its experts in ascending id -> slots 0..n-1, -1 elsewhere."""
    if len(experts) > n_slots:
        raise InfeasibleError(f"{len(experts)} experts do not fit in {n_slots} slots")
    slot_of = np.full(E, -1, dtype=np.int32)
    for i, e in enumerate(sorted(experts)):
        slot_of[e] = i
    return slot_of


def pair_matrix(counts: np.ndarray, route: np.ndarray) -> np.ndarray:
    """pairs[s, D]: (token, expert) invocations origin s sends to GPU D."""
    G, E = counts.shape
    P = np.zeros((G, G), dtype=np.int64)
    for s in range(G):
        np.add.at(P[s], route[s], counts[s])
    return P


def dispatch_accounting(counts: np.ndarray, route: np.ndarray, d: int, bpe: int = 2) -> dict:
    """Reference accounting of one forward from the exchanged count table.

    * remote invocations and `remote_bytes += 2 * token_payload_bytes` per
      remote invocation (sim.py:452-456, domain.py:193-194);
    * token-weighted local ratio (Metrics.local_ratio, sim.py:281-299);
    * wire bytes actually crossing NVLink: rows out + expert outputs back.
    """
    P = pair_matrix(np.asarray(counts, dtype=np.int64), np.asarray(route))
    total = int(P.sum())
    local = int(np.trace(P))
    remote = total - local
    return {
        "invocations": total,
        "remote_invocations": remote,
        "remote_bytes": 2.0 * remote * d * bpe,
        "wire_bytes": 2 * remote * d * bpe,
        "local_ratio": local / total if total else 0.0,
        "pairs": P.tolist(),
    }


def receive_layout(counts: np.ndarray, route: np.ndarray):
    """Host mirror of the GPU layout kernel (csrc/dispatch.cu): per-GPU receive groups.

    Returns (M[D][e] rows GPU D computes for expert e, send_base[s][e] first
    row of origin s's expert-e rows in GPU route[s][e]'s receive buffer).
    Receive buffers are ordered by expert, then source GPU, then (token, slot).
    """
    counts = np.asarray(counts, dtype=np.int64)
    G, E = counts.shape
    M = np.zeros((G, E), dtype=np.int64)
    for s in range(G):
        np.add.at(M, (route[s], np.arange(E)), counts[s])
    base = np.zeros((G, E), dtype=np.int64)
    base[:, 1:] = np.cumsum(M, axis=1)[:, :-1]
    send = np.zeros((G, E), dtype=np.int64)
    seen = np.zeros((G, E), dtype=np.int64)
    for s in range(G):
        for e in range(E):
            D = route[s, e]
            send[s, e] = base[D, e] + seen[D, e]
            seen[D, e] += counts[s, e]
    return M, send
