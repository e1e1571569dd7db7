"""Host <-> device copy bandwidth per GPU, alone and with every rank copying at once.

usage: torchrun --nproc-per-node N tools/host_bw.py [--mb 16] [--iters 50]
Measures, per rank, pinned-host -> device, device -> pinned-host and both directions
concurrently (two streams), after NUMA binding like bench.py.  This is the ceiling of
the bench's `e2e` figure, whose timed region carries x in and the output back per step.
"""

import argparse
import json
import os
import sys
from pathlib import Path

import torch
import torch.distributed as dist

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--mb", type=int, default=16)
    ap.add_argument("--iters", type=int, default=50)
    args = ap.parse_args()
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    from paper_2508_12851_b200 import numa
    numa.bind_to_gpu_node(local)
    if world > 1:
        dist.init_process_group("gloo")
    n = args.mb * 2**20
    h_src = torch.empty(n, dtype=torch.uint8).pin_memory()
    h_dst = torch.empty(n, dtype=torch.uint8).pin_memory()
    d_a = torch.empty(n, dtype=torch.uint8, device="cuda")
    d_b = torch.empty(n, dtype=torch.uint8, device="cuda")
    s_in, s_out = torch.cuda.Stream(), torch.cuda.Stream()

    def run(h2d, d2h):
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        s_in.wait_stream(torch.cuda.current_stream())
        s_out.wait_stream(torch.cuda.current_stream())
        for _ in range(args.iters):
            if h2d:
                with torch.cuda.stream(s_in):
                    d_a.copy_(h_src, non_blocking=True)
            if d2h:
                with torch.cuda.stream(s_out):
                    h_dst.copy_(d_b, non_blocking=True)
        torch.cuda.current_stream().wait_stream(s_in)
        torch.cuda.current_stream().wait_stream(s_out)
        e1.record()
        torch.cuda.synchronize()
        return n * args.iters / (e0.elapsed_time(e1) * 1e-3) / 1e9

    run(True, True)  # warm-up
    res = {"rank": rank, "world": world, "h2d_GBs": run(True, False), "d2h_GBs": run(False, True)}
    both = run(True, True)
    res["duplex_GBs_each_direction"] = both
    out = [None] * world
    if world > 1:
        dist.all_gather_object(out, res)
    else:
        out = [res]
    if rank == 0:
        print(json.dumps(out))
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
