"""Generate golden fixtures from the REFERENCE implementation (`moeplace`).

Run in the build container (where /root/reference exists):

    python tests/golden/make_golden.py

It imports the reference package from /root/reference/pkg/src (read-only; run
from a copy so hypothesis/pycache never touch it) and records what the
reference itself computes for the hot path's pinned quantities:

  route_golden.json      `_EventLoop._choose_target` (sim.py:433-439) for every
                         (origin, expert) of random placements, with uniform and
                         random link matrices;
  dispatch_golden.json   `_EventLoop._dispatch_layer` (sim.py:441-463) run on
                         per-token requests (tokens = 1) whose expert sets come
                         from the oracle router on seeded synthetic tokens:
                         per-invocation targets, remote_bytes, window counts,
                         remote_volume / proxy_cost of the placement;
  migration_golden.json  `migration_cost` (cost.py:171-191) literal / loads-only
                         and `should_migrate` (cost.py:217-248) decisions;
  skew_golden.json       `_selection_dists` (sim.py:153-165) Dirichlet(0.3)
                         vectors for the synthetic workload's servers;
  placements/*.json      `build_placement("ours")` documents for the bench
                         configs (fallback when moeplace is absent on a box).

The fixtures are small JSON files; nothing at GPU-test or bench time reads
/root/reference.
"""

from __future__ import annotations

import json
import shutil
import sys
import tempfile
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
REPO = HERE.parent.parent
sys.path.insert(0, str(REPO))

REF_SRC = Path("/root/reference/pkg/src")


def import_reference():
    tmp = Path(tempfile.mkdtemp(prefix="moeplace_ref_"))
    shutil.copytree(REF_SRC / "moeplace", tmp / "moeplace")
    sys.path.insert(0, str(tmp))
    import moeplace  # noqa: F401
    return moeplace


def single_gpu_cluster(mp, caps, expert_size, bw, lat, load_bw=5e8):
    servers = tuple(mp.ServerSpec(n, (mp.GpuSpec(float(c * expert_size), load_bw),)) for n, c in enumerate(caps))
    return mp.ClusterSpec(servers, np.asarray(bw, float), np.asarray(lat, float))


def make_loop(mp, cluster, model, placement):
    """A reference event loop whose placement is `placement` (the constructor's own
    initial placement is built on a roomy copy of the cluster and then replaced)."""
    from moeplace.sim import _EventLoop, SchedulerPolicy
    stats = mp.ActivationStats(cluster.num_servers, model.experts_per_layer)
    roomy = mp.ClusterSpec(
        tuple(mp.ServerSpec(n, (mp.GpuSpec(float(model.total_experts * model.expert_size), 5e8),))
              for n in range(cluster.num_servers)), cluster.link_bandwidth, cluster.link_latency)
    loop = _EventLoop(roomy, model, "uniform", [], mp.TimeModel.from_cluster(cluster),
                      SchedulerPolicy(migration_enabled=False), stats, 0)
    loop.placement = placement
    return loop


def placement_sets(placement, layer=0):
    return [sorted(e for (l, e) in srv[0] if l == layer) for srv in placement.gpu_sets]


def gen_routes(mp, rng):
    cases = []
    for case in range(24):
        G = int(rng.integers(1, 9))
        E = int(rng.choice([4, 8, 16, 60, 64]))
        d = int(rng.choice([512, 2048, 4096]))
        # random coverage-valid placement with replication
        sets = [set() for _ in range(G)]
        for e in range(E):
            sets[int(rng.integers(G))].add(e)
        for g in range(G):
            extra = rng.choice(E, size=int(rng.integers(0, max(1, E // 2))), replace=False)
            sets[g].update(int(e) for e in extra)
        caps = [max(1, len(s)) for s in sets]
        if case % 2 == 0:
            bw = np.full((G, G), 770e9)
            lat = np.full((G, G), 3e-6)
        else:
            bw = rng.uniform(1e8, 1e12, (G, G))
            lat = rng.uniform(0, 1e-3, (G, G))
        np.fill_diagonal(lat, 0.0)
        model = mp.ModelSpec(1, (E,), min(2, E), 1e6, d)
        cluster = single_gpu_cluster(mp, caps, 1e6, bw, lat)
        placement = mp.Placement(tuple((frozenset((0, e) for e in s),) for s in sets), 1)
        loop = make_loop(mp, cluster, model, placement)
        route = [[int(loop._choose_target(s, 0, e, 1)) for e in range(E)] for s in range(G)]
        cases.append({"G": G, "E": E, "d": d, "sets": [sorted(s) for s in sets], "bw": bw.tolist(),
                      "lat": lat.tolist(), "route": route})
    return cases


def gen_dispatch(mp):
    from oracle import moe_oracle as orc
    from moeplace.sim import RequestTrace

    out = []
    configs = [("toy", 3, 512, 8, 2, 0, 64, [4, 4, 4]), ("ds_like", 4, 256, 64, 6, 1, 48, [20, 20, 18, 18]),
               ("qwen_like", 8, 256, 60, 4, 1, 40, [12, 10, 8, 8, 8, 6, 6, 6])]
    for name, G, d, E, k, mode, T, caps in configs:
        seed = 11
        wg = orc.synthetic_router(E, d, seed)
        idxs = []
        for s in range(G):
            x = orc.synthetic_tokens(s, T, d, seed)
            lg = orc.router_logits(x, wg, orc.origin_bias(s, E, seed))
            idxs.append(orc.topk_route(lg, E, k, mode)[0])
        counts = np.stack([orc.histogram(i, E) for i in idxs]).astype(float)
        expert_size = float(3 * d * 256 * 2)
        model = mp.ModelSpec(1, (E,), k, expert_size, d)
        bw = np.full((G, G), 770e9)
        lat = np.full((G, G), 3e-6)
        np.fill_diagonal(lat, 0.0)
        cluster = single_gpu_cluster(mp, caps, expert_size, bw, lat)
        stats = mp.ActivationStats.from_counts(counts[:, None, :], (E,))
        placement = mp.build_placement("ours", cluster, model, stats, 0)
        assert mp.validate_placement(placement, cluster, model).ok
        loop = make_loop(mp, cluster, model, placement)
        reqs = []
        rid = 0
        for s in range(G):
            for t in range(T):
                reqs.append(RequestTrace(rid, s, 0.0, 1, (tuple(sorted(int(e) for e in idxs[s][t])),)))
                rid += 1
        loop.requests = reqs
        loop.by_id = {r.request_id: r for r in reqs}
        loop.remote_per_request = {r.request_id: 0 for r in reqs}
        for r in reqs:
            loop._dispatch_layer(0.0, r.request_id, 0)
        inv = [[i.origin, i.target, i.expert] for i in loop.inv_log]
        out.append({
            "name": name, "G": G, "d": d, "E": E, "k": k, "score_mode": mode, "T": T, "seed": seed, "caps": caps,
            "idx": [i.tolist() for i in idxs],
            "placement": placement.to_dict(),
            "invocations": inv,
            "remote_bytes": loop.remote_bytes,
            "window_counts": loop.window_stats.counts[:, 0, :].tolist(),
            "remote_volume": mp.remote_volume(placement, stats),
            "proxy_cost": mp.proxy_cost(placement, stats),
        })
    return out


def gen_migration(mp, rng):
    cases = []
    for case in range(16):
        G = int(rng.integers(2, 6))
        E = int(rng.choice([4, 8, 16]))
        expert_size = float(rng.uniform(1e8, 1e9))
        load_bw = rng.uniform(1e8, 1e10, G)
        servers = tuple(mp.ServerSpec(n, (mp.GpuSpec(1e15, float(load_bw[n])),)) for n in range(G))
        cluster = mp.ClusterSpec(servers, np.full((G, G), 1e9), np.zeros((G, G)))
        model = mp.ModelSpec(1, (E,), 1, expert_size, 512)

        def rand_sets():
            sets = [set() for _ in range(G)]
            for e in range(E):
                sets[int(rng.integers(G))].add(e)
            for g in range(G):
                sets[g].update(int(e) for e in rng.choice(E, size=int(rng.integers(0, E)), replace=False))
            return sets

        a, b = rand_sets(), rand_sets()
        pa = mp.Placement(tuple((frozenset((0, e) for e in s),) for s in a), 1)
        pb = mp.Placement(tuple((frozenset((0, e) for e in s),) for s in b), 1)
        counts = rng.integers(0, 50, (G, 1, E)).astype(float)
        stats = mp.ActivationStats.from_counts(counts, (E,))
        penalty = float(rng.uniform(0, 1e-2))
        snap = mp.CostSnapshot(stats, penalty, 0.0, 1.0)
        rec = {"G": G, "E": E, "expert_size": expert_size, "load_bw": load_bw.tolist(),
               "old": [sorted(s) for s in a], "new": [sorted(s) for s in b], "counts": counts[:, 0, :].tolist(),
               "penalty": penalty,
               "literal": mp.migration_cost(pa, pb, cluster, model, "literal"),
               "loads_only": mp.migration_cost(pa, pb, cluster, model, "loads-only"),
               "added": sorted([list(x) for x in (pb.slots - pa.slots)]),
               "removed": sorted([list(x) for x in (pa.slots - pb.slots)])}
        for mode in ("literal", "loads-only"):
            dec, ledger = mp.should_migrate(pa, pb, snap, cluster, model, mode)
            rec[f"decision_{mode}"] = bool(dec)
            rec[f"cost_old_{mode}"] = ledger["cost_current_seconds"]
            rec[f"cost_new_{mode}"] = ledger["cost_candidate_seconds"]
        cases.append(rec)
    return cases


def gen_skew(mp):
    from moeplace.sim import ServerWorkload, _selection_dists
    out = []
    for E in (8, 60, 64):
        model = mp.ModelSpec(1, (E,), 2, 1e6, 512)
        for seed in (0, 11):
            for n in range(8):
                sw = ServerWorkload(1.0, 1, 1, dirichlet_alpha=0.3, seed=seed + n)
                rng = np.random.default_rng([n, sw.seed])
                p = _selection_dists(sw, model, rng)[0]
                out.append({"E": E, "seed": seed, "server": n, "p": p.tolist()})
    return {"numpy": np.__version__, "cases": out}


def gen_bench_placements(mp):
    """'ours' placements for the bench configs from expected counts T*k*p (fallback documents)."""
    from paper_2508_12851_b200.shapes import MIXTRAL, QWEN, DEEPSEEK, TOY, cluster_spec, model_spec, slot_caps
    from paper_2508_12851_b200.workload import origin_dist
    docs = {}
    for shape in (TOY, MIXTRAL, QWEN, DEEPSEEK):
        for G in (2, 3, 4, 8):
            caps = slot_caps(shape, G)
            cluster = cluster_spec(shape, G, caps)
            model = model_spec(shape)
            counts = np.stack([4096 * shape.k * origin_dist(s, shape.E, 0) for s in range(G)])
            stats = mp.ActivationStats.from_counts(counts[:, None, :], (shape.E,))
            for strat in ("ours", "uniform", "eplb"):
                try:
                    p = mp.build_placement(strat, cluster, model, stats, 0)
                except mp.InfeasibleError:
                    continue
                docs[f"{shape.name}_G{G}_{strat}"] = {"caps": caps, "placement": p.to_dict()}
    return docs


def main():
    mp = import_reference()
    rng = np.random.default_rng(20250812)
    (HERE / "route_golden.json").write_text(json.dumps(gen_routes(mp, rng)))
    (HERE / "dispatch_golden.json").write_text(json.dumps(gen_dispatch(mp)))
    (HERE / "migration_golden.json").write_text(json.dumps(gen_migration(mp, rng)))
    (HERE / "skew_golden.json").write_text(json.dumps(gen_skew(mp)))
    pdir = REPO / "paper_2508_12851_b200" / "placements"
    pdir.mkdir(exist_ok=True)
    (pdir / "bench_placements.json").write_text(json.dumps(gen_bench_placements(mp)))
    for p in sorted(HERE.glob("*.json")):
        print(p.name, p.stat().st_size)


if __name__ == "__main__":
    main()
