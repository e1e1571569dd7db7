"""One layer forward of the bench workload, for ncu captures of its kernels (no timing here).

  ncu --set full --clock-control none -k regex:grouped_gemm -o k3 python tools/ncu_step.py --config mixtral
The layer is built as bench.py builds it (same placement, weights and inputs), with two
untimed forwards first so the launch of interest sees the steady-state plan.
"""
import sys
from pathlib import Path

REPO = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(REPO))

import bench  # noqa: E402


def main():
    sys.argv += ["--warmup", "0"]
    args = bench.parse()
    b = bench.setup_bench_layer(args)
    for i in range(3):
        b.layer.forward(b.xs[i % len(b.xs)], b.out)
    b.torch.cuda.synchronize()
    b.layer.check()


if __name__ == "__main__":
    main()
