"""CPU restatement of the distributed MoE-layer forward -- TEST INFRASTRUCTURE ONLY.

This module is the parity oracle for the B200 path.  Only `tests/`,
`__graft_entry__.smoke()` and `bench.py`'s `cpu_baseline` / `--impl reference`
legs may import it; the product package never does (it fails loudly when its
CUDA library is missing instead of falling back here).

What is pinned by the reference (`moeplace`, /root/reference/pkg/src/moeplace)
and what is not:

* routing target        -- restates `_EventLoop._choose_target`
                           (reference sim.py:433-439) with `comm_time`
                           (cost.py:139-149) and `Placement.has_local/holders`
                           (domain.py:249-266).  PINNED: tests/golden/ holds the
                           reference's own choices (tests/golden/make_golden.py).
* histogram             -- restates `ActivationStats.ingest` (stats.py:82-96)
                           with one event per token (token_count = 1).  PINNED.
* dispatch accounting   -- remote pairs / `remote_volume` (cost.py:120-129) and
                           remote bytes `2 * token_payload_bytes` per remote
                           invocation (sim.py:452-456, domain.py:193-194).  PINNED.
* migration plan        -- slot diff of `migration_cost` (cost.py:171-191) on
                           `Placement.slots` (domain.py:268-276).  PINNED.
* synthetic skew        -- `_selection_dists` / `generate_workload`
                           (sim.py:153-191): Dirichlet(0.3) per server from
                           `default_rng([n, seed + n])` (WorkloadSpec.synthetic
                           sim.py:124-138), floored by 1e-9/E.  PINNED (same
                           numpy PCG64 stream; numpy version recorded).
* router math, SwiGLU, combine -- NOT in the reference: restated
                           from the public Mixtral / Qwen1.5-MoE /
                           DeepSeek-V2 model definitions.  Parity unpinned by the
                           reference; the GPU path is checked against this
                           restatement bit-exactly for indices/counts and within
                           the stated tolerance for activations.

Numerics contract shared with the CUDA kernels:
  logits[t,e] = f32( rn_f32(S) * 2^(E(x_t) + E(w_e) - 35) ) + bias[e], with
                S = sum_k qx[t,k] qw[e,k] EXACT, q = rint(a * 2^(win - E(a))) per
                row (win 21 for x, 14 for Wg) and E(a) = max(ef(max|a|) - 126, -100)
                (router_logits).
  top-k       = k largest logits, descending, ties -> lower expert id.
  h           = bf16( silu(g) * u ) with g, u the fp32 GEMM accumulators.
  y           = bf16( h @ W2^T ) (fp32 accumulate).
  out[t]      = bf16( sum_j w[t,j] * y[t,j] (+ gate[t] * ysh[t]) ), j ascending.
"""

from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np

# ----------------------------------------------------------------------------- bf16


def bf16_round(a: np.ndarray) -> np.ndarray:
    """Round float32 values to the nearest bf16 (ties to even), returned as float32."""
    a = np.ascontiguousarray(a, dtype=np.float32)
    u = a.view(np.uint32).astype(np.uint64)
    u = (u + 0x7FFF + ((u >> 16) & 1)) & 0xFFFF0000
    return u.astype(np.uint32).view(np.float32).reshape(a.shape)


def bf16_bits(a: np.ndarray) -> np.ndarray:
    """bf16 bit patterns (uint16) of float32 values that are already bf16-exact."""
    return (np.ascontiguousarray(a, dtype=np.float32).view(np.uint32) >> 16).astype(np.uint16)


def from_bf16_bits(b: np.ndarray) -> np.ndarray:
    return (np.asarray(b, dtype=np.uint16).astype(np.uint32) << 16).view(np.float32)


# ----------------------------------------------------------------------------- shapes


@dataclass(frozen=True)
class LayerShape:
    """Geometry of one MoE layer (ModelSpec plus what ModelSpec cannot express).

    ModelSpec (reference domain.py:158-219) carries E, top_k, hidden width and
    a uniform expert byte size; the FFN width, router convention and shared
    experts live here (SURVEY §5 "Config / flags").
    """

    name: str
    d: int
    f: int
    E: int
    k: int
    score_mode: int = 0        # 0: top-k then softmax over k (Mixtral); 1: softmax over E then top-k
    renorm: int = 0
    shared_f: int = 0          # shared experts concatenated along the FFN width
    shared_gate: int = 0       # 1: sigmoid(x . w_sg) scales the shared output (Qwen)

    @property
    def expert_bytes(self) -> int:
        """m_e = 3 * d * f * 2 (W1, W3, W2 in bf16) -- ModelSpec.expert_size."""
        return 3 * self.d * self.f * 2


# ----------------------------------------------------------------------------- synthetic skew


def origin_expert_dist(origin: int, E: int, seed: int = 0, alpha: float = 0.3) -> np.ndarray:
    """Per-server expert distribution exactly as the reference's synthetic workload.

    WorkloadSpec.synthetic gives server n the seed `seed + n` (sim.py:134-137);
    generate_workload draws from default_rng([n, sw.seed]) (sim.py:172) and
    _selection_dists takes a Dirichlet(alpha) draw, floored by 1e-9/E and
    renormalised (sim.py:161-164).  Layer 0's vector is the first draw.
    """
    rng = np.random.default_rng([origin, seed + origin])
    p = rng.dirichlet(np.full(E, alpha))
    p = p * (1.0 - 1e-9) + 1e-9 / E
    return p / p.sum()


def origin_bias(origin: int, E: int, seed: int = 0, alpha: float = 0.3) -> np.ndarray:
    """Routing skew as a logit bias: log p (fp32)."""
    return np.log(origin_expert_dist(origin, E, seed, alpha)).astype(np.float32)


def synthetic_tokens(origin: int, T: int, d: int, seed: int = 0) -> np.ndarray:
    """x ~ N(0,1) rounded to bf16, from a numpy PCG64 stream per (seed, origin)."""
    rng = np.random.default_rng([1000 + seed, origin])
    return bf16_round(rng.standard_normal((T, d), dtype=np.float32))


def synthetic_router(E_tot: int, d: int, seed: int = 0) -> np.ndarray:
    rng = np.random.default_rng([2000 + seed])
    return bf16_round(rng.standard_normal((E_tot, d), dtype=np.float32) / np.float32(np.sqrt(d)))


def synthetic_expert(expert: int, d: int, f: int, seed: int = 0, layer: int = 0):
    """(W1 [f,d], W3 [f,d], W2 [d,f]) bf16-exact float32, seeded per (seed, layer, expert)."""
    rng = np.random.default_rng([3000 + seed, layer, expert])
    w1 = bf16_round(rng.standard_normal((f, d), dtype=np.float32) / np.float32(np.sqrt(d)))
    w3 = bf16_round(rng.standard_normal((f, d), dtype=np.float32) / np.float32(np.sqrt(d)))
    w2 = bf16_round(rng.standard_normal((d, f), dtype=np.float32) / np.float32(np.sqrt(f)))
    return w1, w3, w2


# ----------------------------------------------------------------------------- routing target


def comm_time(src: int, dst: int, tokens: int, link_latency, link_bandwidth, d: int, bpe: int = 2) -> float:
    """cost.py:139-149: zero locally, else latency + 2 * payload / bandwidth."""
    if src == dst:
        return 0.0
    payload = float(max(1, int(tokens))) * d * bpe  # ModelSpec.token_payload_bytes, domain.py:193-194
    return float(link_latency[src][dst] + 2.0 * payload / link_bandwidth[src][dst])


def route_table(server_experts, link_latency, link_bandwidth, d: int, bpe: int = 2, tokens: int = 1) -> np.ndarray:
    """route[s][e] restating `_choose_target` (sim.py:433-439).

    server_experts[s] = set of experts server s holds for this layer
    (Placement.server_experts, domain.py:246-250).  Origin if it holds e, else
    argmin over holders of (comm_time, server id); raises if no holder.
    The GPU path evaluates the rule once per placement at token granularity
    (tokens = 1: one invocation per routed token).
    """
    E = 1 + max((max(s) for s in server_experts if s), default=-1)
    return route_table_E(server_experts, E, link_latency, link_bandwidth, d, bpe, tokens)


def route_table_E(server_experts, E, link_latency, link_bandwidth, d, bpe=2, tokens=1) -> np.ndarray:
    G = len(server_experts)
    route = np.full((G, E), -1, dtype=np.int32)
    holders = {e: [s for s in range(G) if e in server_experts[s]] for e in range(E)}
    for s in range(G):
        for e in range(E):
            if e in server_experts[s]:
                route[s, e] = s
                continue
            if not holders[e]:
                raise RuntimeError(f"expert {e} of layer 0 is placed nowhere")
            route[s, e] = min(holders[e], key=lambda n: (comm_time(s, n, tokens, link_latency, link_bandwidth, d, bpe), n))
    return route


def slot_assignment(gpu_experts) -> dict:
    """Expert -> local slot: experts held by one GPU in ascending id order."""
    return {e: i for i, e in enumerate(sorted(gpu_experts))}


# ----------------------------------------------------------------------------- router


ROUTER_WIN_X = 21      # token rows: |q| <= 2^21 on each row's integer grid
ROUTER_WIN_W = 14      # router-weight rows: |q| <= 2^14
ROUTER_MIN_EXP = -100  # floor of the row exponent


def router_row_exponent(a: np.ndarray) -> np.ndarray:
    """E(a) per row of a bf16-exact array: max(ef - 126, -100) with ef the bf16 exponent field of
    the row's largest magnitude, so every |a_k| < 2^E(a) (csrc/router.cu row_exponent)."""
    bits = (np.ascontiguousarray(a, dtype=np.float32).view(np.uint32) >> 16) & 0x7FFF
    ef = (bits.max(axis=1) >> 7).astype(np.int64)
    return np.maximum(ef - 126, ROUTER_MIN_EXP)


def router_quantise(a: np.ndarray, win: int):
    """Integer grid of each row: q = rint(a * 2^(win - E(a))) (round half to even), exact in fp64."""
    e = router_row_exponent(a)
    q = np.rint(np.asarray(a, dtype=np.float64) * np.exp2(win - e)[:, None]).astype(np.int64)
    return q, e


def exact_int_matmul(q: np.ndarray, r: np.ndarray) -> np.ndarray:
    """q @ r.T exactly for |q|, |r| <= 2^21 and rows up to 16384 long: 11-bit halves through
    fp64 GEMMs, each of whose partial sums is an integer below 2^53 (so any summation order
    is exact), recombined in int64."""
    qh, ql = q >> 11, q & 2047
    rh, rl = r >> 11, r & 2047
    mm = lambda a, b: np.rint(a.astype(np.float64) @ b.astype(np.float64).T).astype(np.int64)
    return (mm(qh, rh) << 22) + ((mm(qh, rl) + mm(ql, rh)) << 11) + mm(ql, rl)


def rne_f32_of_int(s: np.ndarray) -> np.ndarray:
    """Round int64 values to the nearest fp32 (ties to even), exactly (returned as float64)."""
    s = np.asarray(s, dtype=np.int64)
    a = np.abs(s).astype(np.uint64)
    nb = np.zeros(a.shape, dtype=np.int64)            # bit length of |s|
    for sh in (32, 16, 8, 4, 2, 1):
        big = (a >> np.uint64(sh)) >> nb.astype(np.uint64) != 0
        nb = np.where(big, nb + sh, nb)
    nb = np.where(a != 0, nb + 1, 0)
    drop = np.maximum(nb - 24, 0).astype(np.uint64)
    m = a >> drop
    rem = a - (m << drop)
    half = np.where(drop > 0, np.uint64(1) << np.maximum(drop, np.uint64(1)) - np.uint64(1), np.uint64(0))
    up = (drop > 0) & ((rem > half) | ((rem == half) & ((m & np.uint64(1)) == 1)))
    m = m + up.astype(np.uint64)
    v = m.astype(np.float64) * np.exp2(drop.astype(np.float64))
    return np.where(s < 0, -v, v)


def router_logits(x: np.ndarray, wg: np.ndarray, bias: np.ndarray | None = None) -> np.ndarray:
    """Router logits under K1's exact-integer contract (csrc/router.cu).

    Each row is quantised on its own grid, q = rint(a * 2^(win - E(a))), win = 21 for token
    rows and 14 for router-weight rows; S[t,e] = sum_k qx[t,k] qw[e,k] is an exact integer;
    logits = f32(f64(rn_f32(S)) * 2^(E(x_t) + E(w_e) - 35)), then + bias[e] in fp32.  The GPU
    computes S with 8-bit limb MMAs on the tensor cores; exactness makes it independent of
    any summation order.
    """
    x = np.asarray(x, dtype=np.float32)
    wg = np.asarray(wg, dtype=np.float32)
    if x.shape[1] % 256:
        raise ValueError("router contract needs d % 256 == 0")
    qx, ex = router_quantise(x, ROUTER_WIN_X)
    qw, ew = router_quantise(wg, ROUTER_WIN_W)
    S = exact_int_matmul(qx, qw)
    logits = rne_f32_of_int(S) * np.exp2((ex[:, None] + ew[None, :] - ROUTER_WIN_X - ROUTER_WIN_W).astype(np.float64))
    logits = np.ascontiguousarray(logits.astype(np.float32))
    if bias is not None:
        logits[:, :bias.shape[0]] += np.asarray(bias, dtype=np.float32)[None, :]
    return logits


def topk_route(logits: np.ndarray, E: int, k: int, score_mode: int, renorm: int = 0):
    """Top-k by logit (descending, ties -> lower id) and gate weights."""
    lg = logits[:, :E].astype(np.float64)
    # stable sort on -logit keeps lower ids first among equal logits
    order = np.argsort(-logits[:, :E], axis=1, kind="stable")
    idx = order[:, :k].astype(np.int32)
    sel = np.take_along_axis(lg, idx, axis=1)
    mx = sel[:, :1]
    if score_mode == 0:
        ex = np.exp(sel - mx)
        w = ex / ex.sum(axis=1, keepdims=True)
    else:
        z = np.exp(lg - mx).sum(axis=1, keepdims=True)
        w = np.exp(sel - mx) / z
        if renorm:
            w = w / w.sum(axis=1, keepdims=True)
    return idx, w.astype(np.float32)


def histogram(idx: np.ndarray, E: int) -> np.ndarray:
    """Per-expert token counts: ActivationStats.ingest with token_count 1 per token (stats.py:82-96)."""
    return np.bincount(np.asarray(idx).ravel(), minlength=E).astype(np.int64)


# ----------------------------------------------------------------------------- dispatch layout


def receive_layout(counts: np.ndarray, route: np.ndarray):
    """Per-GPU receive groups and per-origin send bases.

    counts[s][e] = pairs origin s routes to expert e; route[s][e] = target GPU.
    Receive buffer of GPU D: experts ascending, then source ascending.
    Returns (M[D][e], group_base[D][e], send_base[s][e]).
    """
    G, E = counts.shape
    M = np.zeros((G, E), dtype=np.int64)
    for s in range(G):
        for e in range(E):
            M[route[s, e], e] += counts[s, e]
    gbase = np.zeros((G, E), dtype=np.int64)
    gbase[:, 1:] = np.cumsum(M, axis=1)[:, :-1]
    send = np.zeros((G, E), dtype=np.int64)
    for s in range(G):
        for e in range(E):
            D = route[s, e]
            send[s, e] = gbase[D, e] + sum(counts[q, e] for q in range(s) if route[q, e] == D)
    return M, gbase, send


def pair_positions(idx: np.ndarray, route_row: np.ndarray, send_base: np.ndarray):
    """(target GPU, receive row) for every (token, slot) pair of one origin.

    Stable counting sort: inside an expert, pairs keep (token, slot) order --
    the grouping of `_dispatch_layer` (sim.py:446-457) at token granularity.
    """
    T, k = idx.shape
    flat = idx.ravel()
    order = np.argsort(flat, kind="stable")
    rank = np.empty_like(order)
    sorted_e = flat[order]
    starts = np.searchsorted(sorted_e, sorted_e, side="left")
    rank[order] = np.arange(flat.size) - starts
    rows = send_base[flat] + rank
    dst = route_row[flat]
    return dst.reshape(T, k).astype(np.int32), rows.reshape(T, k).astype(np.int64)


# ----------------------------------------------------------------------------- expert FFN


def silu(x):
    return x / (1.0 + np.exp(-x))


def swiglu_ffn(xrows: np.ndarray, w1: np.ndarray, w3: np.ndarray, w2: np.ndarray, with_terms: bool = False):
    """bf16( bf16(silu(x W1^T) * (x W3^T)) W2^T ), fp32 accumulation.  with_terms: also return
    |h| |W2|^T, the magnitude of GEMM2's terms (what a one-ulp change of every h can move y by)."""
    g = xrows @ w1.T
    u = xrows @ w3.T
    h = bf16_round((silu(g) * u).astype(np.float32))
    y = bf16_round((h @ w2.T).astype(np.float32))
    if with_terms:
        return y, (np.abs(h) @ np.abs(w2).T).astype(np.float32)
    return y


# ----------------------------------------------------------------------------- full layer


@dataclass
class OracleResult:
    out: list                     # per origin [T, d] float32 (bf16-exact)
    idx: list                     # per origin [T, k] int32
    w: list                       # per origin [T, k] float32
    hist: list                    # per origin [E] int64
    counts: np.ndarray            # [G, E]
    route: np.ndarray             # [G, E]
    pos_dst: list = field(default_factory=list)
    pos_row: list = field(default_factory=list)
    recv_M: np.ndarray | None = None
    shared_gate: list = field(default_factory=list)
    mag: list = field(default_factory=list)   # per origin [T, d]: sum_j |w_j y_j| (+ |g ysh|)
    mag2: list = field(default_factory=list)  # per origin [T, d]: sum_j |w_j| (|h_j| |W2|^T) (+ shared):
                                              # GEMM2 term magnitude (tests/tolerance.py's bound)


def moe_layer_forward(shape: LayerShape, xs, wg, biases, route, experts, shared=None, wsg=None) -> OracleResult:
    """Whole distributed MoE-layer forward, all origins.

    xs[s]      [T_s, d] bf16-exact float32 tokens of origin s
    wg         [E, d] router weights; wsg [d] shared gate row (Qwen) or None
    biases[s]  [E] fp32 skew of origin s (or None)
    route      [G, E] target GPU table (route_table)
    experts    dict e -> (w1, w3, w2)  (weights of every expert; copies are identical)
    shared     (w1, w3, w2) of the concatenated shared experts or None
    """
    G = len(xs)
    E, k = shape.E, shape.k
    wg_full = wg if wsg is None else np.concatenate([wg, wsg[None, :]], axis=0)
    idxs, ws, hists, gates = [], [], [], []
    counts = np.zeros((G, E), dtype=np.int64)
    for s in range(G):
        lg = router_logits(xs[s], wg_full, biases[s] if biases is not None else None)
        idx, w = topk_route(lg, E, k, shape.score_mode, shape.renorm)
        idxs.append(idx)
        ws.append(w)
        h = histogram(idx, E)
        hists.append(h)
        counts[s] = h
        gates.append((1.0 / (1.0 + np.exp(-lg[:, E].astype(np.float64)))).astype(np.float32) if wsg is not None else None)
    M, gbase, send = receive_layout(counts, route)
    pos_dst, pos_row = [], []
    for s in range(G):
        dst, rows = pair_positions(idxs[s], route[s], send[s])
        pos_dst.append(dst)
        pos_row.append(rows)
    # expert outputs per (origin, token, slot)
    outs, mags, mags2 = [], [], []
    for s in range(G):
        T = xs[s].shape[0]
        y = np.zeros((T, k, shape.d), dtype=np.float32)
        yt = np.zeros((T, k, shape.d), dtype=np.float32)
        for e in np.unique(idxs[s]):
            sel = np.nonzero(idxs[s] == e)
            y[sel], yt[sel] = swiglu_ffn(xs[s][sel[0]], *experts[int(e)], with_terms=True)
        acc = np.zeros((T, shape.d), dtype=np.float32)
        mag = np.zeros((T, shape.d), dtype=np.float32)
        mag2 = np.zeros((T, shape.d), dtype=np.float32)
        for j in range(k):
            acc = acc + ws[s][:, j:j + 1] * y[:, j, :]
            mag = mag + np.abs(ws[s][:, j:j + 1] * y[:, j, :])
            mag2 = mag2 + np.abs(ws[s][:, j:j + 1]) * yt[:, j, :]
        if shared is not None:
            ysh, ysht = swiglu_ffn(xs[s], *shared, with_terms=True)
            g = gates[s][:, None] if wsg is not None else np.float32(1.0)
            acc = acc + g * ysh
            mag = mag + np.abs(g * ysh)
            mag2 = mag2 + np.abs(g) * ysht
        outs.append(bf16_round(acc.astype(np.float32)))
        mags.append(mag)
        mags2.append(mag2)
    return OracleResult(outs, idxs, ws, hists, counts, route, pos_dst, pos_row, M, gates, mags, mags2)


# ----------------------------------------------------------------------------- accounting


def pair_matrix(counts: np.ndarray, route: np.ndarray) -> np.ndarray:
    """pairs[s][D]: (token, expert) invocations origin s sends to GPU D."""
    G, E = counts.shape
    P = np.zeros((G, G), dtype=np.int64)
    for s in range(G):
        for e in range(E):
            P[s, route[s, e]] += counts[s, e]
    return P


def remote_pairs(counts: np.ndarray, route: np.ndarray) -> int:
    P = pair_matrix(counts, route)
    return int(P.sum() - np.trace(P))


def reference_remote_bytes(counts: np.ndarray, route: np.ndarray, d: int, bpe: int = 2) -> float:
    """sim.py:452-456: remote_bytes += 2 * token_payload_bytes(tokens) per remote invocation."""
    return 2.0 * remote_pairs(counts, route) * d * bpe


def remote_volume(counts: np.ndarray, server_experts) -> float:
    """cost.py:120-129 on counts (G, E): token-weighted activations of experts absent locally."""
    total = 0.0
    for n in range(counts.shape[0]):
        row = counts[n]
        total += float(row.sum() - sum(row[i] for i in server_experts[n]))
    return total


def local_ratio(counts: np.ndarray, route: np.ndarray) -> float:
    """Metrics.local_ratio (sim.py:281-299) at token granularity."""
    P = pair_matrix(counts, route)
    tot = P.sum()
    return float(np.trace(P) / tot) if tot > 0 else 0.0


# ----------------------------------------------------------------------------- migration


def slots_of(gpu_sets) -> set:
    """Placement.slots (domain.py:268-276) for single-GPU servers, layer 0: {(n, 0, 0, e)}."""
    return {(n, 0, 0, e) for n, experts in enumerate(gpu_sets) for e in experts}


def migration_plan(old_sets, new_sets):
    """(added, removed) slot sets, restating migration_cost's diff (cost.py:186-187)."""
    old, new = slots_of(old_sets), slots_of(new_sets)
    return sorted(new - old), sorted(old - new)


def migration_seconds(old_sets, new_sets, expert_size: float, load_bw, mode: str = "literal") -> float:
    """migration_cost (cost.py:171-191) with per-GPU load bandwidth load_bw[n]."""
    if mode not in ("literal", "loads-only"):
        raise ValueError(f"unknown migration cost mode {mode!r}")
    added, removed = migration_plan(old_sets, new_sets)
    changed = added if mode == "loads-only" else added + removed
    return float(sum(expert_size / load_bw[n] for n, _g, _l, _e in changed))


def should_migrate(cost_old: float, cost_new: float, transfer: float) -> bool:
    """Eq. 4 (cost.py:233): adopt iff cost_new + transfer < cost_old, strictly."""
    return cost_new + transfer < cost_old
