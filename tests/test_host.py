"""Host-side logic of the drop-in (CPU): shapes, route tables from reference placements,
accounting, migration planning, the bench placement fallback documents."""

import json
from pathlib import Path

import numpy as np
import pytest

from paper_2508_12851_b200 import routing
from paper_2508_12851_b200.errors import import_moeplace
from paper_2508_12851_b200.migration import added_cells, plan_rounds
from paper_2508_12851_b200.shapes import DEEPSEEK, MIXTRAL, QWEN, SHAPES, TOY, get_shape, slot_caps

REPO = Path(__file__).resolve().parent.parent


def test_shapes_expert_bytes_and_flops():
    assert MIXTRAL.expert_bytes == 352_321_536
    assert QWEN.expert_bytes == DEEPSEEK.expert_bytes == 17_301_504
    assert MIXTRAL.flops_per_token() == 704_643_072
    assert QWEN.flops_per_token() == DEEPSEEK.flops_per_token() == 138_412_032
    for s in SHAPES.values():
        assert s.d % 256 == 0 and s.f % 128 == 0 and s.shared_f % 128 == 0
    assert get_shape("ds") is DEEPSEEK


@pytest.mark.parametrize("shape", [TOY, MIXTRAL, QWEN, DEEPSEEK], ids=lambda s: s.name)
@pytest.mark.parametrize("G", [1, 2, 4, 8])
def test_caps_cover_all_experts(shape, G):
    caps = slot_caps(shape, G)
    assert len(caps) == G and sum(caps) >= shape.E
    if shape is QWEN and G == 8:
        assert caps == [12, 10, 8, 8, 8, 6, 6, 6]
    if shape is MIXTRAL and G == 8:
        assert caps == [2] * 8


def test_route_table_from_placement_document():
    doc = {"layers": [{"layer": 0, "servers": [{"server": 0, "gpus": [[0, 1, 2]]},
                                                 {"server": 1, "gpus": [[2, 3]]}]}]}
    lat, bw = routing.uniform_links(2)
    r = routing.route_table(routing.server_expert_sets(doc), 4, lat, bw, 512)
    assert r.tolist() == [[0, 0, 0, 1], [0, 0, 1, 1]]
    assert routing.gpu_expert_sets(doc) == [[0, 1, 2], [2, 3]]


def test_route_table_from_reference_placement_object():
    mp = import_moeplace()
    if mp is None:
        pytest.skip("reference not importable")
    p = mp.Placement(((frozenset({(0, 0), (0, 1)}),), (frozenset({(0, 1), (0, 2), (0, 3)}),)), 1)
    servers = tuple(mp.ServerSpec(n, (mp.GpuSpec(4e6, 5e8),)) for n in range(2))
    lat, bw = routing.uniform_links(2)
    cluster = mp.ClusterSpec(servers, bw, lat)
    r = routing.route_table_for(p, cluster, 4, 512)
    assert r.tolist() == [[0, 0, 1, 1], [0, 1, 1, 1]]


def test_slot_map_and_capacity():
    from paper_2508_12851_b200 import InfeasibleError
    assert routing.slot_map([5, 1], 8, 3).tolist() == [-1, 0, -1, -1, -1, 1, -1, -1]
    with pytest.raises(InfeasibleError):
        routing.slot_map([1, 2, 3], 8, 2)


def test_dispatch_accounting_reference_formula():
    counts = np.array([[5, 3, 0, 2], [1, 1, 1, 1]])
    route = np.array([[0, 0, 1, 1], [0, 0, 1, 1]])
    acc = routing.dispatch_accounting(counts, route, 4096)
    assert acc["remote_invocations"] == 2 + 2
    assert acc["remote_bytes"] == 2.0 * 4 * 4096 * 2   # sim.py:454, payload d*bpe per token
    assert acc["local_ratio"] == pytest.approx((8 + 2) / 14)


def test_plan_rounds_uses_lowest_current_holder():
    old = [[0, 1, 2], [2, 3], [0, 3]]
    new = [[0, 1, 3], [1, 2, 3], [0, 2]]
    rounds = plan_rounds(old, new, [4, 4, 4])
    assert len(rounds) == 1
    assert sorted((p.expert, p.src_rank, p.dst_rank) for p in rounds[0].pulls) == [(1, 0, 1), (2, 0, 2), (3, 1, 0)]
    assert [list(s) for s in rounds[0].sets_after] == new
    assert added_cells(rounds) == [(0, 0, 0, 3), (1, 0, 0, 1), (2, 0, 0, 2)]


def _check_rounds(old, new, phys):
    rounds = plan_rounds(old, new, phys)
    cur = [set(s) for s in old]
    E = set().union(*map(set, old))
    for r in rounds:
        for p in r.pulls:                       # sources hold the expert when the round starts
            assert p.expert in cur[p.src_rank] and p.expert not in cur[p.dst_rank]
        during = [cur[g] | {p.expert for p in r.pulls if p.dst_rank == g} for g in range(len(old))]
        assert all(len(during[g]) <= phys[g] for g in range(len(old)))   # old copies retire after
        after = [set(s) for s in r.sets_after]
        assert set().union(*after) == E                                  # coverage at every swap
        assert all(after[g] <= during[g] for g in range(len(old)))
        cur = after
    assert [sorted(c) for c in cur] == [sorted(s) for s in new]
    return rounds


def test_plan_rounds_full_gpus_swap_through_one_staging_slot():
    # every GPU exactly full (cap = 3): swapping whole blocks takes one round per expert
    old = [[0, 1, 2], [3, 4, 5]]
    new = [[3, 4, 5], [0, 1, 2]]
    rounds = _check_rounds(old, new, [4, 4])
    assert len(rounds) == 3
    assert all(len(r.pulls) == 2 for r in rounds)


def test_plan_rounds_random_heterogeneous_caps():
    rng = np.random.default_rng(7)
    for _ in range(300):
        G = int(rng.integers(2, 9))
        E = int(rng.choice([8, 16, 60, 64]))
        caps = [-(-E // G) + int(rng.integers(0, 3)) for _ in range(G)]

        def place():
            sets = [set() for _ in range(G)]
            for e in rng.permutation(E):
                g = int(rng.choice([g for g in range(G) if len(sets[g]) < caps[g]]))
                sets[g].add(int(e))
            for g in range(G):
                while len(sets[g]) < caps[g] and rng.random() < 0.6:
                    sets[g].add(int(rng.integers(E)))
            return [sorted(s) for s in sets]
        _check_rounds(place(), place(), [c + 1 for c in caps])


def test_plan_rounds_rejects_over_cap_and_unheld():
    from paper_2508_12851_b200 import InfeasibleError
    with pytest.raises(InfeasibleError):
        plan_rounds([[0, 1]], [[0, 1, 2]], [2])
    with pytest.raises(InfeasibleError):
        plan_rounds([[0], [1]], [[0, 2], [1]], [3, 3])


def test_bench_placement_documents_are_valid():
    docs = json.loads((REPO / "paper_2508_12851_b200" / "placements" / "bench_placements.json").read_text())
    assert any(k.startswith("mixtral-8x7b_G8_ours") for k in docs)
    for key, d in docs.items():
        name, G, strat = key.rsplit("_", 2)
        shape = get_shape(name)
        sets = routing.gpu_expert_sets(d["placement"])
        assert len(sets) == int(G[1:])
        assert set().union(*map(set, sets)) == set(range(shape.E)), key          # coverage
        assert all(len(s) <= c for s, c in zip(sets, d["caps"])), key           # memory caps


def test_interleave_w13_layout():
    torch = pytest.importorskip("torch")
    from paper_2508_12851_b200.layer import interleave_w13
    f, d = 256, 8
    w1 = torch.arange(f * d).reshape(f, d).float()
    w3 = -w1
    w13 = interleave_w13(w1, w3)
    assert torch.equal(w13[0:128], w1[0:128]) and torch.equal(w13[128:256], w3[0:128])
    assert torch.equal(w13[256:384], w1[128:256]) and torch.equal(w13[384:512], w3[128:256])


@pytest.mark.parametrize("penalty,expect", [(2.5e-8, False), (1e-4, True)])
def test_migration_controller_check_is_the_reference_decision(penalty, expect):
    """MigrationController.check == build_placement + should_migrate of the reference on the
    same window statistics (_migration_check, sim.py:465-481), for a drifted window."""
    mp = import_moeplace()
    if mp is None:
        pytest.skip("reference package not importable")
    from types import SimpleNamespace

    from paper_2508_12851_b200 import workload as wl
    from paper_2508_12851_b200.controller import MigrationController
    from paper_2508_12851_b200.shapes import cluster_spec, model_spec

    shape, G = DEEPSEEK, 4
    caps = slot_caps(shape, G)
    cluster, model = cluster_spec(shape, G, caps), model_spec(shape)
    T, k = 4096, shape.k
    counts_a = np.stack([np.rint(T * k * wl.origin_dist(g, shape.E)) for g in range(G)]).astype(np.int64)
    counts_b = np.stack([np.roll(c, shape.E // 2) for c in counts_a])
    stats_a = mp.ActivationStats.from_counts(counts_a[:, None, :].astype(float), (shape.E,))
    current = mp.build_placement("ours", cluster, model, stats_a, 0)
    fake = SimpleNamespace(gathered_counts=lambda group=None: counts_b, shape=shape, world=1,
                           reset_counts=lambda: None)
    window = 0.05
    ctl = MigrationController(fake, cluster, model, current, penalty_seconds=penalty)
    adopt, ledger, cand = ctl.check(window)
    stats_b = mp.ActivationStats.from_counts(counts_b[:, None, :].astype(float), (shape.E,))
    ref_cand = mp.build_placement("ours", cluster, model, stats_b, 0)
    ref_adopt, ref_ledger = mp.should_migrate(current, ref_cand, mp.CostSnapshot(stats_b, penalty, 0.0, window),
                                              cluster, model, "loads-only")
    assert adopt == bool(ref_adopt) == expect
    assert ledger == ref_ledger
    assert routing.gpu_expert_sets(cand, 0) == routing.gpu_expert_sets(ref_cand, 0)
