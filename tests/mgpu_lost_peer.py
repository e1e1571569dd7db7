"""Lost-peer worker (G = 2, launched by test_gpu_multi.py with MP_PEER_TIMEOUT_MS=2000).

Rank 1 stops calling forward after two good forwards (a lost GPU, as seen by its peer).  Rank 0
runs one more forward: every wait for rank 1 must time out -- bounded, with no kernel trap, so
the CUDA context stays usable -- the error word must name rank 1, and the NEXT forward must
refuse to launch (MP_E_PEER -> RuntimeError), as INTEGRATION.md documents.
"""

import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))

import torch
import torch.distributed as dist

from paper_2508_12851_b200 import workload as wl
from paper_2508_12851_b200.layer import B200MoELayer
from paper_2508_12851_b200.shapes import get_shape


def main():
    import os
    rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
    torch.cuda.set_device(rank)
    dev = torch.device("cuda", rank)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    shape = get_shape("toy")
    T = 256
    layer = B200MoELayer(shape, rank=rank, world=world, device=rank, max_tokens=T, cap_slots=shape.E)
    layer.open_peers()
    wg = wl.router_weights(shape.E + shape.shared_gate, shape.d, dev)
    layer.set_router(wg[:shape.E], wl.origin_bias(rank, shape.E).to(dev),
                     wg[shape.E] if shape.shared_gate else None)
    src = lambda e: wl.expert_weights(e, shape.d, shape.f, dev)
    layer.set_placement_sets([list(range(shape.E))[r::world] for r in range(world)], src)
    x = wl.tokens(T, shape.d, dev, origin=rank)
    for _ in range(2):
        layer.forward(x)
    torch.cuda.synchronize()
    layer.check()
    dist.barrier()
    if rank == 0:
        t0 = time.time()
        layer.forward(x)           # rank 1 never joins this forward
        torch.cuda.synchronize()   # bounded waits, no trap: the context is still usable
        waited = time.time() - t0
        try:
            layer.check()
            raise AssertionError("check() did not report the lost peer")
        except RuntimeError as e:
            assert "0x2" in str(e), str(e)
        try:
            layer.forward(x)
            raise AssertionError("forward launched after a peer was lost")
        except RuntimeError as e:
            assert "timed out" in str(e) or "peer" in str(e).lower(), str(e)
        torch.zeros(1, device=dev).add_(1).item()  # the CUDA context is alive
        print(f"lost-peer ok: waited {waited:.1f} s", flush=True)
    dist.barrier()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
