"""GPU fp32 restatement of the MoE-layer expert math -- TEST INFRASTRUCTURE ONLY.

The numpy oracle (oracle/moe_oracle.py) is the parity reference; at BASELINE
sizes (Mixtral d 4096 x f 14336 at T = 4096) its CPU GEMMs are too slow for a
test, so the full-size tests restate the same arithmetic in plain PyTorch fp32
on the GPU (TF32 off): per routed (token, slot) pair
    h = bf16(silu(x W1^T) * (x W3^T)),  y = bf16(h W2^T)
and out = bf16(sum_j w_j y_j (+ g_sh y_sh)), j ascending -- the contract of
moe_oracle.moe_layer_forward.  Routing (idx, w, gate) comes from the oracle.
"""

from __future__ import annotations

import torch


def _ffn(x: torch.Tensor, w1: torch.Tensor, w3: torch.Tensor, w2: torch.Tensor):
    """(y, |h| |W2|^T): the output and the magnitude of GEMM2's terms."""
    g = x @ w1.float().T
    u = x @ w3.float().T
    h = (torch.nn.functional.silu(g) * u).bfloat16().float()
    w2f = w2.float()
    return (h @ w2f.T).bfloat16().float(), h.abs() @ w2f.abs().T


def layer_reference(x: torch.Tensor, idx, w, expert_src, shared=None, gate=None):
    """x [T, d] bf16 (device); idx [T, k] int, w [T, k] fp32 (numpy or torch); expert_src(e) ->
    (W1 [f, d], W3 [f, d], W2 [d, f]) bf16 device tensors; shared (W1, W3, W2) or None; gate [T]
    (sigmoid shared gate) or None.  Returns (out [T, d] fp32 bf16-exact, mag, mag2) with
    mag = sum_j |w_j y_j| (+ |g y_sh|) and mag2 = sum_j |w_j| (|h_j| |W2|^T) (+ shared), the
    magnitudes tests/tolerance.py's bound is relative to."""
    prev = torch.backends.cuda.matmul.allow_tf32
    torch.backends.cuda.matmul.allow_tf32 = False
    try:
        dev = x.device
        idx = torch.as_tensor(idx, device=dev).long()
        w = torch.as_tensor(w, device=dev).float()
        T, k = idx.shape
        xf = x.float()
        y = torch.zeros(T, k, x.shape[1], device=dev)
        yt = torch.zeros_like(y)
        for e in torch.unique(idx).tolist():
            t, j = torch.nonzero(idx == e, as_tuple=True)
            y[t, j], yt[t, j] = _ffn(xf[t], *expert_src(e))
        acc = torch.zeros(T, x.shape[1], device=dev)
        mag = torch.zeros_like(acc)
        mag2 = torch.zeros_like(acc)
        for j in range(k):
            term = w[:, j:j + 1] * y[:, j]
            acc = acc + term
            mag = mag + term.abs()
            mag2 = mag2 + w[:, j:j + 1].abs() * yt[:, j]
        if shared is not None:
            ysh, ysht = _ffn(xf, *shared)
            g = torch.as_tensor(gate, device=dev).float()[:, None] if gate is not None else 1.0
            acc = acc + g * ysh
            mag = mag + (g * ysh).abs()
            mag2 = mag2 + (g.abs() if gate is not None else 1.0) * ysht
        return acc.bfloat16().float(), mag, mag2
    finally:
        torch.backends.cuda.matmul.allow_tf32 = prev
