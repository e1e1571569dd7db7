"""Soak test of the NVLink flag protocol: chunks of forwards, then every rank's protocol
state is gathered and checked (same epoch everywhere, every flag equal to it, arrival
tickets and the router accumulator back at zero, no timeout bits).  Stops at the first
chunk that breaks an invariant and prints every rank's state.

  python -m torch.distributed.run --nproc-per-node 4 --master-addr 127.0.0.1 \
      tools/soak.py --gpus 4 --config deepseek --steps 6000 --chunk 250
"""

import json
import sys
import time
from pathlib import Path

REPO = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(REPO))

import bench  # noqa: E402


def main():
    bench_argv = [a for a in sys.argv[1:] if not a.startswith("--chunk") and a != "--events"]
    chunk = 250
    use_events = "--events" in sys.argv[1:]  # per-forward stage events, as bench.py's timed loop
    for a in sys.argv[1:]:
        if a.startswith("--chunk="):
            chunk = int(a.split("=")[1])
    sys.argv = [sys.argv[0]] + bench_argv
    args = bench.parse()
    b = bench.setup_bench_layer(args)
    torch, dist, layer, xs, out, world, rank = b.torch, b.dist, b.layer, b.xs, b.out, b.world, b.rank
    n_rot = len(xs)
    done, t0, bad = 0, time.time(), None
    while done < args.steps:
        n = min(chunk, args.steps - done)
        evs = [None] * n
        if use_events:
            NS, lib = b._lib.NUM_STAGE_EVENTS, b._lib
            which = {0, lib.GEMM_START, lib.GEMM1_END, lib.GEMM_END, lib.MAIN_STAGE_EVENTS - 1}
            evs = [[torch.cuda.Event(enable_timing=True) if j in which else None for j in range(NS)]
                   for _ in range(n)]
            for row in evs:
                for ev in row:
                    if ev is not None:
                        ev.record()
            torch.cuda.synchronize()
        for i in range(n):
            layer.forward(xs[(done + i) % n_rot], out, events=evs[i])
        done += n
        st = torch.tensor(layer.sync_state().astype("int64"), device=b.dev)
        allst = [torch.zeros_like(st) for _ in range(world)]
        dist.all_gather(allst, st) if world > 1 else allst.__setitem__(0, st)
        S = [a.cpu().tolist() for a in allst]
        ep = {s[0] for s in S}
        flags_ok = all(s[8 + p] == s[0] for s in S for p in range(world)) if world > 1 else True
        zero_ok = all(s[3] == 0 and s[4] == 0 and s[5] == 0 and s[6] == 0 and s[7] == 0 for s in S)
        if rank == 0 and (done // n) % 50 == 0:
            print(json.dumps({"progress": done, "epoch": S[0][0]}), flush=True)
        if len(ep) != 1 or not flags_ok or not zero_ok:
            bad = S
            break
    res = {"soak": b.shape.name, "G": world, "forwards": done, "seconds": round(time.time() - t0, 1),
           "ok": bad is None}
    if bad is not None:
        res["states"] = bad
    if rank == 0:
        print(json.dumps(res), flush=True)
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()
    sys.exit(0 if bad is None else 1)


if __name__ == "__main__":
    main()
