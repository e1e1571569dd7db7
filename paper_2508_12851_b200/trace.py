"""Export GPU routing decisions as the reference's activation trace (JSON lines).

`moeplace` reads traces with `parse_trace` (reference cli.py:91-135): one JSON
object per line with fields t, server, layer, experts, tokens; each record is an
`ActivationEvent` whose token_count is added to every listed expert
(`ActivationStats.ingest`, stats.py:82-96).  Tokens that chose the same expert
SET are aggregated into one record, so replaying the file through the reference
reproduces the GPU histogram exactly while keeping expert co-occurrence.
"""

from __future__ import annotations

import json
from collections import Counter

import numpy as np


def trace_records(idx: np.ndarray, server: int, layer: int, t: float = 0.0) -> list[dict]:
    """Records for one forward's routed indices idx [T, k] of one origin GPU."""
    sets = Counter(tuple(sorted(int(e) for e in row)) for row in np.asarray(idx))
    return [{"t": float(t), "server": int(server), "layer": int(layer), "experts": list(k), "tokens": int(n)}
            for k, n in sorted(sets.items())]


def write_trace(path: str, records, append: bool = False) -> int:
    """Write records as JSON lines; returns the number written."""
    n = 0
    with open(path, "a" if append else "w", encoding="utf-8") as fh:
        for r in records:
            fh.write(json.dumps(r, sort_keys=True) + "\n")
            n += 1
    return n


def counts_from_records(records, num_servers: int, experts_per_layer) -> np.ndarray:
    """Token-weighted counts [servers, layers, Emax] as the reference would ingest them."""
    L = len(experts_per_layer)
    c = np.zeros((num_servers, L, max(experts_per_layer)), dtype=np.int64)
    for r in records:
        for e in r["experts"]:
            c[r["server"], r["layer"], e] += r["tokens"]
    return c
