"""Router time under layer conditions: K1 alone (mp_layer_route) timed with CUDA events between full
layer forwards of rotating batches (so L2 holds what a real step leaves behind), and back to back.

usage: python tools/router_probe.py [--config deepseek] [--T 4096] [--iters 30]
"""
import argparse
import ctypes
import json
import sys
from pathlib import Path

REPO = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(REPO))

import torch  # noqa: E402

from paper_2508_12851_b200 import workload as wl  # noqa: E402
from paper_2508_12851_b200.layer import B200MoELayer  # noqa: E402
from paper_2508_12851_b200.shapes import get_shape  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="deepseek")
    ap.add_argument("--T", type=int, default=4096)
    ap.add_argument("--iters", type=int, default=30)
    args = ap.parse_args()
    shape = get_shape(args.config)
    dev = torch.device("cuda", 0)
    T, E = args.T, shape.E
    layer = B200MoELayer(shape, max_tokens=T, cap_slots=E, staging_slots=0)
    wg = wl.router_weights(E + shape.shared_gate, shape.d, dev)
    layer.set_router(wg[:E], wl.origin_bias(0, E), wg[E] if shape.shared_gate else None)
    if shape.shared_f:
        layer.set_shared(*wl.shared_weights(shape.d, shape.shared_f, dev))
    layer.set_placement_sets([list(range(E))], lambda e: wl.expert_weights(e, shape.d, shape.f, dev))
    xs = [wl.tokens(T, shape.d, dev, batch=b) for b in range(8)]
    out = torch.empty_like(xs[0])
    st = ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)
    res = {}
    for mode in ("after_forward", "back_to_back"):
        ts = []
        for i in range(args.iters + 3):
            x = xs[i % 8]
            if mode == "after_forward":
                layer.forward(xs[(i + 3) % 8], out)
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record()
            layer.lib.mp_layer_route(layer._h, x.data_ptr(), T, st)
            b.record()
            ts.append((a, b))
        torch.cuda.synchronize()
        ms = sorted(a.elapsed_time(b) for a, b in ts[3:])
        res[mode] = {"median_us": ms[len(ms) // 2] * 1e3, "min_us": ms[0] * 1e3}
    print(json.dumps({"config": shape.name, "T": T, **res}))
    layer.close()


if __name__ == "__main__":
    main()
