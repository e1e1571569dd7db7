"""Layer geometries of the BASELINE.json configs and their per-GPU slot caps.

`ModelSpec` (reference domain.py:158-219) carries L, experts_per_layer, top_k,
a uniform expert byte size and the hidden width; it has no field for the FFN
width, the router convention or shared experts, so those live in
`LayerShape`.  `model_spec()` / `cluster_spec()` build the reference value
objects for a shape so the reference placement solver can run on it.
"""

from __future__ import annotations

from dataclasses import dataclass

TOPK_SOFTMAX = 0   # Mixtral: top-k logits, softmax over the k
SOFTMAX_TOPK = 1   # Qwen1.5-MoE / DeepSeek-V2-Lite: softmax over E, top-k, no renorm


@dataclass(frozen=True)
class LayerShape:
    name: str
    d: int            # hidden width (ModelSpec.hidden_width)
    f: int            # routed expert FFN width
    E: int            # routed experts (ModelSpec.experts_per_layer[0])
    k: int            # ModelSpec.top_k
    score_mode: int = TOPK_SOFTMAX
    renorm: int = 0
    shared_f: int = 0     # shared experts, concatenated along the FFN width
    shared_gate: int = 0  # 1: shared output scaled by sigmoid(x . w_sg)

    @property
    def expert_bytes(self) -> int:
        """m_e = 3*d*f*2: W1, W3 [f, d] and W2 [d, f] in bf16."""
        return 3 * self.d * self.f * 2

    def flops_per_token(self) -> int:
        """Routed + shared expert FLOPs per token (2 * 3 * d * f per (token, expert))."""
        return 6 * self.d * (self.k * self.f + self.shared_f)


TOY = LayerShape("toy", d=512, f=2048, E=8, k=2)
MIXTRAL = LayerShape("mixtral-8x7b", d=4096, f=14336, E=8, k=2)
QWEN = LayerShape("qwen1.5-moe-a2.7b", d=2048, f=1408, E=60, k=4, score_mode=SOFTMAX_TOPK,
                  shared_f=5632, shared_gate=1)
DEEPSEEK = LayerShape("deepseek-v2-lite", d=2048, f=1408, E=64, k=6, score_mode=SOFTMAX_TOPK,
                      shared_f=2 * 1408)

SHAPES = {s.name: s for s in (TOY, MIXTRAL, QWEN, DEEPSEEK)}
ALIASES = {"toy": "toy", "mixtral": "mixtral-8x7b", "qwen": "qwen1.5-moe-a2.7b", "deepseek": "deepseek-v2-lite",
           "ds": "deepseek-v2-lite"}


def get_shape(name: str) -> LayerShape:
    return SHAPES[ALIASES.get(name, name)]


def slot_caps(shape: LayerShape, G: int) -> list[int]:
    """Per-GPU expert slot caps (GpuSpec.memory // m_e) used by the configs.

    * Mixtral: ceil(E/G) + 1 (2 slots at G=8);
    * Qwen: heterogeneous [12,10,8,8,8,6,6,6] at G=8, scaled for smaller G;
    * DeepSeek-V2-Lite and toy: ceil(E/G) + 4.
    """
    base = -(-shape.E // G)
    if shape.name == MIXTRAL.name:
        return [base + 1] * G
    if shape.name == QWEN.name:
        het = [12, 10, 8, 8, 8, 6, 6, 6]
        if G == 8:
            return het
        scale = 8 / G
        caps = [max(base + 2, int(round(het[i] * scale))) for i in range(G)]
        return caps
    return [min(shape.E, base + 4)] * G


def model_spec(shape: LayerShape):
    """The reference ModelSpec for one MoE layer of this shape."""
    from .errors import import_moeplace

    mp = import_moeplace()
    if mp is None:
        raise RuntimeError("the reference package moeplace is not importable")
    return mp.ModelSpec(num_layers=1, experts_per_layer=(shape.E,), top_k=shape.k,
                        expert_size=float(shape.expert_bytes), hidden_width=shape.d, bytes_per_element=2)


def cluster_spec(shape: LayerShape, G: int, caps: list[int] | None = None,
                 link_bandwidth: float = 770e9, link_latency: float = 3e-6, load_bandwidth: float = 770e9):
    """Reference ClusterSpec: G single-GPU servers joined by uniform NVLink 5.

    Link figures are the measured B200 NVLink peer-copy bandwidth (770 GB/s per
    direction, B200_PROFILING.md) and a few-microsecond latency; with uniform
    links `_choose_target` (sim.py:433-439) picks the lowest-id holder.
    """
    import numpy as np

    from .errors import import_moeplace

    mp = import_moeplace()
    if mp is None:
        raise RuntimeError("the reference package moeplace is not importable")
    caps = caps or slot_caps(shape, G)
    servers = tuple(mp.ServerSpec(n, (mp.GpuSpec(float(caps[n] * shape.expert_bytes), load_bandwidth),))
                    for n in range(G))
    bw = np.full((G, G), link_bandwidth)
    lat = np.full((G, G), link_latency)
    np.fill_diagonal(lat, 0.0)
    return mp.ClusterSpec(servers, bw, lat)
