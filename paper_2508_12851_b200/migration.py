"""Host side of expert migration (K6): plan the slot diff, then execute it with peer copies.

The reference decides *whether* to migrate with `should_migrate` (reference
cost.py:217-248: adopt iff C(P') + T_mig < C(P), strictly) and prices the
transfer with `migration_cost` (cost.py:171-191), whose slot diff
`new.slots - old.slots` (cost.py:186) is exactly the set of weight copies the
GPUs must perform.  The event loop keeps serving with the old placement until
`migration_complete` (sim.py:520-525) swaps it in; old copies retire only after
the new ones land.

Here every GPU pulls each expert it gains from the lowest-id GPU that held it
in the old placement, into a free (staging) slot, on a side stream; the route
tables swap on all GPUs only after every GPU's copies completed.
"""

from __future__ import annotations

from dataclasses import dataclass

from .errors import InfeasibleError


@dataclass(frozen=True)
class Pull:
    expert: int
    src_rank: int
    dst_slot: int


def plan_pulls(rank: int, old_sets, new_sets, free_slots) -> list[Pull]:
    """Copies GPU `rank` performs to go from old_sets to new_sets (per-GPU expert lists)."""
    mine_old = set(old_sets[rank])
    free = sorted(free_slots)
    pulls = []
    for e in sorted(set(new_sets[rank]) - mine_old):
        holders = [n for n in range(len(old_sets)) if e in old_sets[n]]
        if not holders:
            raise RuntimeError(f"expert {e} has no holder in the old placement")
        if not free:
            raise InfeasibleError(f"GPU {rank}: no free slot to stage expert {e}")
        pulls.append(Pull(e, holders[0], free.pop(0)))
    return pulls


def slot_diff(old_sets, new_sets):
    """(added, removed) (server, gpu, layer, expert) cells -- Placement.slots diff (domain.py:268-276)."""
    old = {(n, 0, 0, e) for n, s in enumerate(old_sets) for e in s}
    new = {(n, 0, 0, e) for n, s in enumerate(new_sets) for e in s}
    return sorted(new - old), sorted(old - new)


def transfer_seconds(old_sets, new_sets, expert_bytes: float, load_bandwidth, mode: str = "literal") -> float:
    """migration_cost (cost.py:171-191) for single-GPU servers with per-GPU load bandwidth."""
    if mode not in ("literal", "loads-only"):
        raise ValueError(f"unknown migration cost mode {mode!r}")
    added, removed = slot_diff(old_sets, new_sets)
    changed = added if mode == "loads-only" else added + removed
    return float(sum(expert_bytes / load_bandwidth[n] for n, _g, _l, _e in changed))
