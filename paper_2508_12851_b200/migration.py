"""Host side of expert migration (K6): the slot diff, ordered into rounds that respect the caps.

The reference decides *whether* to migrate with `should_migrate` (reference
cost.py:217-248: adopt iff C(P') + T_mig < C(P), strictly) and prices the
transfer with `migration_cost` (cost.py:171-191), whose slot diff
`new.slots - old.slots` (cost.py:186) is exactly the set of weight copies the
GPUs perform.  Traffic keeps the old placement until `migration_complete`
(sim.py:520-525) swaps the new one in, and old copies retire only after the
new ones land.  Coverage -- every expert held somewhere
(domain.py:376-380) -- must hold at every instant.

On a GPU the cap is physical: GpuSpec.memory // m_e expert slots
(domain.py:395-401) plus ONE staging slot (stated in DESIGN.md), so a GPU can
hold at most cap + 1 experts while a migration is in flight.  `plan_rounds`
orders the diff so that bound and coverage hold throughout:

  each round  every GPU with experts still to gain pulls as many as it has free
              slots, each from the lowest-id GPU holding it at that moment
              (first the experts whose only copy sits on a GPU that must drop
              it -- they unblock evictions elsewhere);
  then        once every GPU's copies of the round landed, the route tables swap
              to the round's intermediate placement, in which every GPU drops
              the experts it does not keep that are now held elsewhere; their
              slots are free for the next round.

The union of the rounds' pulls is the reference slot diff (added cells); the
intermediate placements are valid placements (coverage, caps + staging).  A
round that cannot progress (a cycle of full GPUs each holding the only copy
another one needs) raises InfeasibleError instead of breaking coverage.
"""

from __future__ import annotations

from dataclasses import dataclass

from .errors import InfeasibleError


@dataclass(frozen=True)
class Pull:
    expert: int
    src_rank: int   # GPU holding the expert when the round starts (lowest id)
    dst_rank: int


@dataclass(frozen=True)
class Round:
    pulls: tuple[Pull, ...]
    sets_after: tuple[tuple[int, ...], ...]   # placement in effect after the round's route swap


def plan_rounds(old_sets, new_sets, phys_slots) -> list[Round]:
    """Migration rounds from `old_sets` to `new_sets` (per-GPU expert lists) with at most
    phys_slots[g] experts resident on GPU g at any instant."""
    G = len(old_sets)
    if len(new_sets) != G or len(phys_slots) != G:
        raise ValueError("old_sets, new_sets and phys_slots need one entry per GPU")
    cur = [set(int(e) for e in s) for s in old_sets]
    new = [set(int(e) for e in s) for s in new_sets]
    for g in range(G):
        if len(cur[g]) > phys_slots[g] or len(new[g]) > phys_slots[g]:
            raise InfeasibleError(f"GPU {g}: placement exceeds its {phys_slots[g]} physical slots")
    for e in set().union(*new):
        if not any(e in c for c in cur):
            raise InfeasibleError(f"expert {e} has no holder in the old placement")
    rounds: list[Round] = []
    while any(cur[g] != new[g] for g in range(G)):
        holders = {}
        for g in range(G):
            for e in cur[g]:
                holders.setdefault(e, []).append(g)
        # experts whose only copy sits on a GPU that drops it: pulling them first frees that GPU
        blocking = {e for e, hs in holders.items() if len(hs) == 1 and e not in new[hs[0]]}
        pulls = []
        for g in range(G):
            free = phys_slots[g] - len(cur[g])
            want = sorted(new[g] - cur[g], key=lambda e: (e not in blocking, e))
            for e in want[:max(0, free)]:
                pulls.append(Pull(e, min(holders[e]), g))
        for p in pulls:
            cur[p.dst_rank].add(p.expert)
        evicted = 0
        for g in range(G):
            for e in sorted(cur[g] - new[g]):
                if any(e in cur[h] for h in range(G) if h != g):
                    cur[g].discard(e)
                    evicted += 1
        if not pulls and not evicted:
            raise InfeasibleError(
                "migration cannot progress with one staging slot per GPU: full GPUs hold the only copies "
                "of each other's missing experts " + str([sorted(c) for c in cur]))
        rounds.append(Round(tuple(pulls), tuple(tuple(sorted(c)) for c in cur)))
    return rounds


def added_cells(rounds) -> list[tuple[int, int, int, int]]:
    """(server, gpu, layer, expert) cells the rounds add -- equals `new.slots - old.slots` of
    migration_cost (cost.py:186-187) for single-GPU servers, layer 0."""
    return sorted((p.dst_rank, 0, 0, p.expert) for r in rounds for p in r.pulls)
