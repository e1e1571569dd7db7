"""Synthetic inputs of the benchmark configs (data = "synthetic").

* Routing skew: the reference's synthetic workload gives server n a
  Dirichlet(alpha = 0.3) expert distribution drawn from
  `default_rng([n, seed + n])` (WorkloadSpec.synthetic, reference sim.py:124-138;
  generate_workload sim.py:172; _selection_dists sim.py:161-164).  The B200 path
  has a real router, so the same distribution enters as a per-origin logit bias
  log p; the workload-shift run rolls it by E/2 (the acceptance suite's drift,
  reference tests/test_acceptance.py:67-68, uses np.roll).
* Tokens, router and expert weights: N(0,1) / sqrt(fan_in) in bf16, generated
  on the GPU from per-(seed, layer, expert) generators, so every copy of an
  expert is bit-identical on every GPU without any transfer.
"""

from __future__ import annotations

import numpy as np
import torch


def origin_dist(origin: int, E: int, seed: int = 0, alpha: float = 0.3) -> np.ndarray:
    rng = np.random.default_rng([origin, seed + origin])
    p = rng.dirichlet(np.full(E, alpha))
    p = p * (1.0 - 1e-9) + 1e-9 / E
    return p / p.sum()


def origin_bias(origin: int, E: int, seed: int = 0, shift: int = 0) -> torch.Tensor:
    """log p of origin `origin` (fp32 [E]); `shift` rolls the distribution (workload drift)."""
    p = origin_dist(origin, E, seed)
    if shift:
        p = np.roll(p, shift)
    return torch.from_numpy(np.log(p).astype(np.float32))


def _gen(device, *key: int) -> torch.Generator:
    g = torch.Generator(device=device)
    h = 1469598103934665603
    for k in key:
        h = ((h ^ (k & 0xFFFFFFFF)) * 1099511628211) & ((1 << 63) - 1)
    g.manual_seed(h)
    return g


def tokens(T: int, d: int, device, seed: int = 0, origin: int = 0, batch: int = 0) -> torch.Tensor:
    g = _gen(device, 11, seed, origin, batch)
    return torch.randn(T, d, device=device, generator=g, dtype=torch.float32).to(torch.bfloat16)


def router_weights(E_tot: int, d: int, device, seed: int = 0) -> torch.Tensor:
    g = _gen(device, 13, seed)
    return (torch.randn(E_tot, d, device=device, generator=g) / d ** 0.5).to(torch.bfloat16)


def expert_weights(e: int, d: int, f: int, device, seed: int = 0, layer: int = 0):
    """(W1 [f, d], W3 [f, d], W2 [d, f]) bf16 of expert e."""
    g = _gen(device, 17, seed, layer, e)
    w1 = (torch.randn(f, d, device=device, generator=g) / d ** 0.5).to(torch.bfloat16)
    w3 = (torch.randn(f, d, device=device, generator=g) / d ** 0.5).to(torch.bfloat16)
    w2 = (torch.randn(d, f, device=device, generator=g) / f ** 0.5).to(torch.bfloat16)
    return w1, w3, w2


def shared_weights(d: int, f_shared: int, device, seed: int = 0, layer: int = 0):
    return expert_weights(1_000_003, d, f_shared, device, seed, layer)
