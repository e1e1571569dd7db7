"""N > 1 host logic on CPU with gloo process groups of 2 and 8 ranks.

Covers what the ranks agree on before the NVLink kernels run: identical route
tables from one placement, the handle all-gather of B200MoELayer.open_peers,
the count all-gather feeding the reference solver, the receive layout each
rank derives independently (must equal the oracle), and consistent migration
plans (every rank derives the same cap-respecting migration rounds; every
pulled expert is held by its source when its round starts).  The 8-rank case
covers the G = 8 host side that no 4-GPU box can run (the layer's kernels must
never share a GPU between ranks).
"""

import os
import socket

import numpy as np
import pytest

torch = pytest.importorskip("torch")
import torch.distributed as dist  # noqa: E402
import torch.multiprocessing as tmp  # noqa: E402


def _port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from oracle import moe_oracle as orc
        from paper_2508_12851_b200 import routing
        from paper_2508_12851_b200.migration import plan_rounds

        E, k, d, T = 16, 2, 256, 64
        sets = [[e for e in range(E) if e % world == r or e == 0] for r in range(world)]
        lat, bw = routing.uniform_links(world)
        route = routing.route_table([frozenset(s) for s in sets], E, lat, bw, d)
        # 1. every rank built the same route table
        allr = [None] * world
        dist.all_gather_object(allr, route.tolist())
        assert all(r == allr[0] for r in allr)
        # 2. handle exchange as in open_peers (128 opaque bytes per rank)
        mine = bytes([rank]) * 128
        hs = [None] * world
        dist.all_gather_object(hs, mine)
        assert b"".join(hs) == b"".join(bytes([r]) * 128 for r in range(world))
        # 3. counts all-gather -> identical count table; local layout == oracle layout
        wg = orc.synthetic_router(E, d, 4)
        x = orc.synthetic_tokens(rank, T, d, 4)
        idx, _ = orc.topk_route(orc.router_logits(x, wg, orc.origin_bias(rank, E, 4)), E, k, 0)
        h = torch.from_numpy(orc.histogram(idx, E))
        gath = [torch.zeros_like(h) for _ in range(world)]
        dist.all_gather(gath, h)
        counts = torch.stack(gath).numpy()
        M, send = routing.receive_layout(counts, route)
        M_o, _, send_o = orc.receive_layout(counts, route)
        assert np.array_equal(M, M_o) and np.array_equal(send, send_o)
        dst, rows = orc.pair_positions(idx, route[rank], send[rank])
        mine_rows = torch.tensor([int((dst == D).sum()) for D in range(world)])
        tot = mine_rows.clone()
        dist.all_reduce(tot)
        assert tot.tolist() == [int(M[D].sum()) for D in range(world)]
        # 4. migration rounds are identical on every rank and move exactly the slot diff
        new = [[e for e in range(E) if e % world == (r + 1) % world or e == 1] for r in range(world)]
        phys = [max(len(a), len(b)) + 1 for a, b in zip(sets, new)]
        rounds = plan_rounds(sets, new, phys)
        plan = [[(p.expert, p.src_rank, p.dst_rank) for p in r.pulls] for r in rounds]
        allp = [None] * world
        dist.all_gather_object(allp, plan)
        assert all(p == allp[0] for p in allp)
        cur = [set(x) for x in sets]
        for r in rounds:
            for p in r.pulls:
                assert p.expert in cur[p.src_rank]
            cur = [set(x) for x in r.sets_after]
        assert [sorted(c) for c in cur] == [sorted(x) for x in new]
        mine = {p.expert for r in rounds for p in r.pulls if p.dst_rank == rank}
        assert mine == set(new[rank]) - set(sets[rank])
        q.put((rank, "ok"))
    except Exception as ex:  # pragma: no cover - reported to the parent
        q.put((rank, repr(ex)))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 8])
def test_multi_rank_host_logic_gloo(world):
    ctx = tmp.get_context("spawn")
    q = ctx.Queue()
    port = _port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=180) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
    assert sorted(res) == [(r, "ok") for r in range(world)], res


def _agree_worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import bench

        # loop counts a rank derives from its own clock (settle length, e2e pre-batches) differ
        # across ranks; bench.agree_max makes every rank run the same number of forwards
        n = bench.agree_max(3 + 4 * rank, world, torch.device("cpu"))
        go = bench.agree_max(rank == world - 1, world, torch.device("cpu"))
        q.put((rank, n, go))
    finally:
        dist.destroy_process_group()


def test_bench_loop_counts_agree_gloo():
    world, port = 2, _port()
    ctx = tmp.get_context("spawn")
    q = ctx.Queue()
    ps = [ctx.Process(target=_agree_worker, args=(r, world, port, q)) for r in range(world)]
    for p in ps:
        p.start()
    for p in ps:
        p.join(120)
        assert p.exitcode == 0
    got = sorted(q.get() for _ in range(world))
    assert got == [(0, 7, 1), (1, 7, 1)]
