"""Online placement control over a running B200MoELayer.

Mirrors the reference event loop's migration logic, one call per decision point:
  * `_migration_check` (reference pkg/src/moeplace/sim.py:465-481): window
    statistics -> `build_placement(strategy, ...)` candidate ->
    `should_migrate(current, candidate, CostSnapshot, cluster, model, mode)`
    (cost.py:217-248), adopt iff C(P') + T_mig < C(P);
  * `migration_complete` (sim.py:520-525): the new placement takes effect only
    after every GPU's weight copies landed, then the window statistics reset.

The statistics are the GPU router's histograms (`B200MoELayer.gathered_counts`,
token_count 1 per token), the remote penalty and the copy bandwidth are measured
on the box (`calibrate.py`), and the copies are NVLink pulls on a side stream
(`B200MoELayer.migrate_async`), so traffic keeps flowing on the old placement
while the weights move.  SPMD: every rank calls every method.
"""

from __future__ import annotations

import numpy as np
import torch

from .errors import import_moeplace
from .routing import gpu_expert_sets


class MigrationController:
    def __init__(self, layer, cluster, model, placement, *, strategy: str = "ours", seed: int = 0,
                 mode: str = "loads-only", penalty_seconds: float = 0.0, group=None):
        self.mp = import_moeplace()
        if self.mp is None:
            raise RuntimeError("the reference package moeplace is not importable")
        self.layer, self.cluster, self.model = layer, cluster, model
        self.placement = placement
        self.strategy, self.seed, self.mode = strategy, seed, mode
        self.penalty_seconds = penalty_seconds
        self.group = group
        self.history: list[dict] = []

    # ---------------------------------------------------------------- statistics
    def window_stats(self):
        """ActivationStats of the current window (all origins' GPU histograms)."""
        counts = self.layer.gathered_counts(self.group).astype(float)
        return self.mp.ActivationStats.from_counts(counts[:, None, :], (self.layer.shape.E,))

    def reset_window(self) -> None:
        self.layer.reset_counts()

    # ---------------------------------------------------------------- decision
    def check(self, window_seconds: float):
        """One `_migration_check`: returns (adopt, ledger, candidate placement)."""
        stats = self.window_stats()
        candidate = self.mp.build_placement(self.strategy, self.cluster, self.model, stats, self.seed)
        snapshot = self.mp.CostSnapshot(stats, self.penalty_seconds, 0.0, window_seconds)
        adopt, ledger = self.mp.should_migrate(self.placement, candidate, snapshot, self.cluster, self.model,
                                               self.mode)
        return bool(adopt), ledger, candidate

    # ---------------------------------------------------------------- execution
    def migrate(self, candidate, side_stream: torch.cuda.Stream | None = None, while_copying=None) -> dict:
        """Execute an adopted plan: NVLink pulls on `side_stream` in cap-respecting rounds
        (migration.plan_rounds: at most cap + 1 resident experts per GPU, every expert covered at
        every instant), `while_copying()` (e.g. a few forwards on the current placement) overlapped
        with each round's copies, the route swap after each round (`migration_complete`), then a
        fresh statistics window.  Returns copy accounting."""
        import torch.distributed as dist

        layer = self.layer
        world = layer.world
        old_sets = gpu_expert_sets(self.placement, 0)
        new_sets = gpu_expert_sets(candidate, 0)
        # physical slots of every GPU: the reference's per-GPU cap (packable_capacity,
        # domain.py:395-401) plus the staging slot(s) every layer reserves
        phys = [int(self.mp.packable_capacity(self.cluster, n, self.model)) + layer.staging_slots
                for n in range(world)]
        lat = np.asarray(self.cluster.link_latency, dtype=float)
        bw = np.asarray(self.cluster.link_bandwidth, dtype=float)
        res = layer.migrate(old_sets, new_sets, phys_slots=phys, stream=side_stream, while_copying=while_copying,
                            link_latency=lat, link_bandwidth=bw, group=self.group)
        self.placement = candidate
        self.reset_window()
        n_add, t_copy = len(res["adds"]), res["copy_ms"]
        if world > 1:
            dev = layer.device if dist.get_backend(self.group) == "nccl" else "cpu"
            a = torch.tensor([float(n_add)], dtype=torch.float64, device=dev)
            b = torch.tensor([t_copy], dtype=torch.float64, device=dev)
            dist.all_reduce(a, group=self.group)
            dist.all_reduce(b, op=dist.ReduceOp.MAX, group=self.group)
            n_add, t_copy = int(a.item()), float(b.item())
        rec = {"slots_copied": n_add, "bytes_copied": n_add * layer.shape.expert_bytes, "copy_ms_max_gpu": t_copy,
               "rounds": res["rounds"], "forwards_during_copy": res["forwards_during_copy"]}
        self.history.append(rec)
        return rec

    def step(self, window_seconds: float, side_stream=None, while_copying=None):
        """check() and, if adopted, migrate(): returns (ledger, copy record or None)."""
        adopt, ledger, candidate = self.check(window_seconds)
        rec = self.migrate(candidate, side_stream, while_copying) if adopt else None
        return ledger, rec
