"""Multi-GPU parity worker (one process per GPU, launched by torchrun from test_gpu_multi.py).

Every rank builds the same G-origin problem, runs its own origin through the
B200 layer (count exchange + NVLink dispatch + tcgen05 experts + NVLink return)
and checks against the CPU oracle computed for all origins:
  * bit-exact: routed indices, the exchanged count table, per-pair target GPU
    and receive row, reference-accounted remote bytes;
  * tolerance: layer output (tests/tolerance.py, same bound as the single-GPU tests).
Then it executes a migration (NVLink peer copies on a side stream, route swap
after completion) and checks the new placement the same way.
"""

import os
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))

import numpy as np
import torch
import torch.distributed as dist

from oracle import moe_oracle as orc
from tolerance import check_layer_close
from paper_2508_12851_b200.layer import B200MoELayer
from paper_2508_12851_b200.routing import route_table, uniform_links
from paper_2508_12851_b200.shapes import LayerShape


NCCL_GROUP = None


def assert_protocol_quiescent(layer, G, tag):
    """Between forwards the NVLink flag protocol is at rest on every rank: one epoch
    everywhere, every flag of every window equal to it, arrival tickets / router count
    accumulator / timeout bits zero (mp_layer_sync_state)."""
    st = [int(v) for v in layer.sync_state()]
    allst = [None] * G
    dist.all_gather_object(allst, st)
    ep = allst[0][0]
    for r, s in enumerate(allst):
        assert s[0] == ep, f"{tag}: rank {r} epoch {s[0]} != {ep}"
        assert s[8:8 + G] == [ep] * G, f"{tag}: rank {r} flags {s[8:8 + G]} != {ep}"
        assert s[3:8] == [0] * 5, f"{tag}: rank {r} tickets / accumulator / err {s[3:8]}"


def run_case(shape, G, rank, sets, sets2, T_list, seed, caps=None, expect=None, expect_rounds=0, staging=1):
    """expect: K3 plan keys (B200MoELayer.exec_plan) the first forward must have run, so the
    production plans -- CTA-pair tiles with the NVLink-scatter GEMM2 epilogue; the split plan
    with the pair-fused shared expert and the small-group side chain -- meet the oracle at G > 1."""
    dev = torch.device("cuda", torch.cuda.current_device())
    E = shape.E
    experts = {e: orc.synthetic_expert(e, shape.d, shape.f, seed) for e in range(E)}
    shared = orc.synthetic_expert(999, shape.d, shape.shared_f, seed) if shape.shared_f else None
    wg = orc.synthetic_router(E + shape.shared_gate, shape.d, seed)
    biases = [orc.origin_bias(s, E, seed) for s in range(G)]
    xs = [orc.synthetic_tokens(s, T_list[s], shape.d, seed) for s in range(G)]
    lat, bw = uniform_links(G)

    cap = max(len(s) for s in sets + sets2) if caps is None else caps[rank]
    layer = B200MoELayer(shape, rank=rank, world=G, max_tokens=max(T_list), cap_slots=cap, staging_slots=staging)
    layer.open_peers()
    layer.set_router(torch.from_numpy(wg[:E]), torch.from_numpy(biases[rank]),
                     torch.from_numpy(wg[E]) if shape.shared_gate else None)
    if shared is not None:
        layer.set_shared(*(torch.from_numpy(w) for w in shared))
    src = lambda e: tuple(torch.from_numpy(w) for w in experts[e])
    layer.set_placement_sets(sets, src)
    x = torch.from_numpy(xs[rank]).to(dev).bfloat16().contiguous()

    def check(route, tag):
        out = layer.forward(x)
        torch.cuda.synchronize()
        layer.check()
        dist.barrier()
        ref = orc.moe_layer_forward(shape, xs, wg[:E], biases, route, experts, shared,
                                    wg[E] if shape.shared_gate else None)
        T = T_list[rank]
        assert np.array_equal(layer.idx[:T].cpu().numpy(), ref.idx[rank]), f"{tag}: idx"
        assert np.array_equal(layer.read_counts(), ref.counts), f"{tag}: counts"
        assert np.array_equal(layer.pos_dst[:T].cpu().numpy(), ref.pos_dst[rank]), f"{tag}: pos_dst"
        assert np.array_equal(layer.pos_row[:T].cpu().numpy(), ref.pos_row[rank]), f"{tag}: pos_row"
        acc = layer.dispatch_accounting()
        assert acc["remote_bytes"] == orc.reference_remote_bytes(ref.counts, route, shape.d), f"{tag}: bytes"
        check_layer_close(out.float().cpu().numpy(), ref.out[rank], ref.mag[rank], ref.mag2[rank], tag)
        return out, ref

    route1 = route_table([frozenset(s) for s in sets], E, lat, bw, shape.d)
    assert np.array_equal(layer.route, route1)
    out_a, ref_a = check(route1, "placement A")
    out_a = out_a.clone()
    if expect:
        plan = layer.exec_plan()
        assert all(plan[k] == v for k, v in expect.items()), f"{shape.name}: plan {plan}, expected {expect}"
    # repeated forwards reuse the parity-double-buffered count tables
    check(route1, "placement A again")
    # CUDA-graph replay across GPUs (device-side barrier epochs / count parity)
    from paper_2508_12851_b200.layer import capture_graph
    gout = torch.empty_like(x)
    g = capture_graph(lambda: layer.forward(x, gout))
    for _ in range(3):
        g.replay()
    torch.cuda.synchronize()
    layer.check()
    dist.barrier()
    assert torch.equal(gout, out_a), "graph replay differs from eager forward"
    assert_protocol_quiescent(layer, G, "after graph replay")
    # the NCCL all-to-all-v transport (the K4 A/B arm) runs the same kernels as stages with NCCL
    # moving the rows: bit-identical outputs and routing
    from paper_2508_12851_b200.nccl_path import NcclForward
    nf = NcclForward(layer, group=NCCL_GROUP)
    out_n = nf.forward(x)
    torch.cuda.synchronize()
    assert torch.equal(out_n, out_a), "NCCL transport differs from the fused NVLink forward"
    assert np.array_equal(layer.pos_row[:T_list[rank]].cpu().numpy(), ref_a.pos_row[rank]), "NCCL path pos_row"
    assert np.array_equal(layer.read_counts(), orc.moe_layer_forward(
        shape, xs, wg[:E], biases, route1, experts, shared, wg[E] if shape.shared_gate else None).counts)
    del g

    # ---- migration A -> B in cap-respecting rounds (cap + 1 staging slot per GPU, coverage at
    # every instant): NVLink pulls on a side stream with forwards in flight, route swap per round
    phys = [(caps[g] if caps is not None else cap) + staging for g in range(G)]
    fwd_out = torch.empty_like(x)
    res = layer.migrate(sets, sets2, phys_slots=phys, stream=torch.cuda.Stream(dev),
                        while_copying=lambda: (layer.forward(x, fwd_out), 1)[1])
    route2 = route_table([frozenset(s) for s in sets2], E, lat, bw, shape.d)
    assert np.array_equal(layer.route, route2)
    assert int((layer.slot_of >= 0).sum()) == len(sets2[rank]) <= phys[rank] - staging
    if expect_rounds:
        assert res["rounds"] >= expect_rounds, res["rounds"]
    # migrated weights are bit-identical to the source copies
    for e, _ in res["adds"]:
        w1, w3, w2 = layer.read_slot(int(layer.slot_of[e]))
        assert np.array_equal(w1.float().cpu().numpy(), experts[e][0]), f"migrated W1 of expert {e}"
        assert np.array_equal(w2.float().cpu().numpy(), experts[e][2]), f"migrated W2 of expert {e}"
    layer.check()
    check(route2, "placement B (after migration)")
    assert_protocol_quiescent(layer, G, "end of case")
    layer.close()


def main():
    dist.init_process_group("gloo")
    rank, G = dist.get_rank(), dist.get_world_size()
    # one rank per GPU, never more: the layer kernels spin on flags raised by the peers'
    # kernels, which co-resident processes on one GPU cannot guarantee to schedule
    local = int(os.environ.get("LOCAL_RANK", rank))
    if local >= torch.cuda.device_count():
        raise SystemExit(f"rank {rank}: LOCAL_RANK {local} but only {torch.cuda.device_count()} GPUs")
    torch.cuda.set_device(local)
    global NCCL_GROUP
    NCCL_GROUP = dist.new_group(backend="nccl")
    only = os.environ.get("MGPU_CASES")  # optional subset, e.g. "prod" (production plans only)

    if only == "rand":  # randomised cases only, seeds from MGPU_RAND_SEEDS (a fuzz run)
        random_cases(G, rank, [int(v) for v in os.environ.get("MGPU_RAND_SEEDS", "11,12").split(",")])
    else:
        if only != "prod":
            small_cases(G, rank)
            tight_cap_case(G, rank)
        production_cases(G, rank)

    dist.barrier()
    if rank == 0:
        print(f"mgpu ok: G={G}")
    dist.destroy_process_group()


def production_cases(G, rank):
    """The K3 plans the BASELINE shapes run at G > 1, at sizes the oracle finishes in seconds."""
    # (a) Mixtral-like: 8 experts top-2, G*T*k >= 512*E -> routed experts on CTA pairs (256-row
    # tiles); GEMM2's epilogue scatters each output row to its origin GPU over NVLink
    shape = LayerShape("mixtral_like", d=512, f=512, E=8, k=2)
    sets = [sorted({(g * 8 // G + i) % 8 for i in range(-(-8 // G))}) for g in range(G)]
    sets2 = [sorted({(g * 8 // G + i + 1) % 8 for i in range(-(-8 // G) + 1)}) for g in range(G)]
    run_case(shape, G, rank, sets, sets2, [-(-2304 // G) + 40 * s for s in range(G)], seed=21,
             expect={"pair_routed": 1, "split_m": 0})
    # (b) DeepSeek-like split plan: groups >= 256 rows on CTA pairs with the shared expert fused
    # into the same launches, groups < 256 rows on the 1-CTA side chain over 20 SMs
    # (256 <= G*T*k/E < 1024 rows per expert on average)
    shape = LayerShape("ds_like", d=256, f=256, E=64, k=6, score_mode=1, shared_f=512)
    per = -(-64 // G)
    own = [set(range(g * per, min(64, (g + 1) * per))) for g in range(G)]
    sets = [sorted(own[g] | {(g * per + per) % 64}) for g in range(G)]
    sets2 = [sorted(own[g] | {(g * per + per + 1) % 64, (g * per + 2 * per + 5) % 64}) for g in range(G)]
    T = -(-4096 // G)  # avg rows per expert = G*T*6/64 = 384
    run_case(shape, G, rank, sets, sets2, [T + 24 * s for s in range(G)], seed=22,
             expect={"pair_routed": 1, "split_m": 256, "small_grid": 20, "fuse_shared": 1})
    # (c) the same plan with >= 1024 rows per expert on average: the side chain gets 8 SMs
    T = -(-11264 // G)  # G*T*6/64 = 1056
    run_case(shape, G, rank, sets, sets, [T] * G, seed=23,
             expect={"pair_routed": 1, "split_m": 256, "small_grid": 8, "fuse_shared": 1})
    # (d) Qwen-like split plan with the sigmoid-gated shared expert (avg rows 256..1024)
    shape = LayerShape("qwen_like", d=256, f=384, E=60, k=4, score_mode=1, shared_f=512, shared_gate=1)
    per = -(-60 // G)
    sets = [sorted(set(range(g * per, min(60, (g + 1) * per)))) for g in range(G)]
    sets2 = [sorted(set(range(g * per, min(60, (g + 1) * per))) | {(g * per + per + 2) % 60}) for g in range(G)]
    T = -(-5120 // G)  # G*T*4/60 = 341
    run_case(shape, G, rank, sets, sets2, [T + 16 * s for s in range(G)], seed=24,
             expect={"pair_routed": 1, "split_m": 256, "small_grid": 20, "fuse_shared": 1})


def tight_cap_case(G, rank):
    """Heterogeneous, exactly-full caps (Qwen-like 60 experts, caps in the ratio of the Qwen
    config's [12,10,8,8,8,6,6,6]): every GPU holds cap experts and swaps a block of them, so the
    migration needs several rounds through the single staging slot."""
    shape = LayerShape("qwen_tight", d=256, f=256, E=60, k=4, score_mode=1, shared_f=256, shared_gate=1)
    het = np.array([12, 10, 8, 8, 8, 6, 6, 6][:G], dtype=float)
    sizes = np.floor(60 * het / het.sum()).astype(int)
    sizes[0] += 60 - int(sizes.sum())
    starts = np.concatenate([[0], np.cumsum(sizes)[:-1]])
    sets = [list(range(int(a), int(a + n))) for a, n in zip(starts, sizes)]
    shift = max(3, 60 // (3 * G))
    sets2 = [sorted((e + shift) % 60 for e in s) for s in sets]
    run_case(shape, G, rank, sets, sets2, [160 + 8 * s for s in range(G)], seed=31, caps=[int(n) for n in sizes],
             expect_rounds=2)


def small_cases(G, rank):
    # case 1: toy-like shape, replicated experts; origins with different T (ragged)
    shape = LayerShape("toy_small", d=512, f=512, E=8, k=2)
    sets = [sorted({(g * 8 // G + i) % 8 for i in range(8 // G + 1)}) for g in range(G)]
    sets2 = [sorted({(g * 8 // G + i + 3) % 8 for i in range(8 // G + 1)}) for g in range(G)]
    run_case(shape, G, rank, sets, sets2, [200 + 37 * s for s in range(G)], seed=1)

    # case 2: DeepSeek-like routing (64 experts, top-6, shared experts), one GPU holding few experts
    shape = LayerShape("ds_small", d=256, f=256, E=64, k=6, score_mode=1, shared_f=512)
    per = -(-64 // G)
    own = [set(range(g * per, min(64, (g + 1) * per))) for g in range(G)]
    sets = [sorted(own[g] | {(g * per + per) % 64}) for g in range(G)]
    sets2 = [sorted(own[g] | {(g * per + per + 1) % 64, (g * per + 2 * per + 5) % 64}) for g in range(G)]
    run_case(shape, G, rank, sets, sets2, [150] * G, seed=2)

    # case 3: Qwen-like (softmax-top4 + sigmoid-gated shared expert)
    shape = LayerShape("qwen_small", d=256, f=384, E=60, k=4, score_mode=1, shared_f=512, shared_gate=1)
    per = -(-60 // G)
    sets = [sorted(set(range(g * per, min(60, (g + 1) * per)))) for g in range(G)]
    sets2 = [sorted(set(range(g * per, min(60, (g + 1) * per))) | {(g * per + per + 2) % 60}) for g in range(G)]
    run_case(shape, G, rank, sets, sets2, [96 + 16 * s for s in range(G)], seed=3)

    # case 4: an idle origin (T = 0 on rank 0: no router / permute launched there; it still
    # publishes zero counts and its flags) next to busy ones, DeepSeek-like plan (fused shared)
    shape = LayerShape("ds_small", d=256, f=256, E=64, k=6, score_mode=1, shared_f=512)
    per = -(-64 // G)
    sets = [sorted(set(range(g * per, min(64, (g + 1) * per))) | {(g * per + per) % 64}) for g in range(G)]
    run_case(shape, G, rank, sets, sets, [0] + [120] * (G - 1), seed=4)

    # case 5: a GPU with no expert memory at all (cap 0 -> no slots, no K3 launches; it still
    # raises its return flag) while it keeps originating tokens
    shape = LayerShape("toy_small", d=512, f=512, E=8, k=2)
    holders = list(range(G - 1))
    sets = [sorted(e for e in range(8) if e % len(holders) == g) if g < G - 1 else [] for g in range(G)]
    caps = [max(len(x) for x in sets)] * (G - 1) + [0]
    run_case(shape, G, rank, sets, sets, [100 + 20 * s for s in range(G)], seed=5, caps=caps, staging=0)

    random_cases(G, rank, (11, 12))


def random_cases(G, rank, seeds):
    # case 6: randomised shapes and placements (every rank draws the same ones): replicated
    # experts, ragged T including empty origins, migration between two random placements
    for seed in seeds:
        r = np.random.default_rng(seed * 100 + G)
        E = int(r.choice([8, 16, 60, 64]))
        k = int(r.integers(1, min(6, E) + 1))
        shared_f = int(r.choice([0, 256]))
        shape = LayerShape(f"rand{seed}", d=int(r.choice([256, 512])), f=int(r.choice([128, 256, 384])), E=E, k=k,
                           score_mode=int(r.integers(0, 2)), shared_f=shared_f,
                           shared_gate=int(r.integers(0, 2)) if shared_f else 0)

        def random_sets():
            held = [set() for _ in range(G)]
            for e in range(E):
                for g in r.choice(G, size=int(r.integers(1, min(2, G) + 1)), replace=False):
                    held[int(g)].add(e)
            return [sorted(h) for h in held]
        sets, sets2 = random_sets(), random_sets()
        # seeds >= 100 draw batches up to 3000 tokens, so the CTA-pair / split plans run too
        T_list = [int(t) for t in r.integers(0, 3000 if seed >= 100 else 300, size=G)]
        T_list[int(r.integers(0, G))] = max(1, T_list[0])
        run_case(shape, G, rank, sets, sets2, T_list, seed=seed)


if __name__ == "__main__":
    main()
