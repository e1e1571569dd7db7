"""The NCCL all-to-all-v transport for the layer forward (the A/B arm of K4).

SURVEY §5 / the north star name NCCL send/recv for the dispatch and the return
of non-local tokens (the reference prices that exchange analytically,
`comm_time` cost.py:139-149, remote bytes sim.py:452-456).  The product path
(`B200MoELayer.forward`) fuses both transfers into its kernels as NVLink peer
stores; this module runs the SAME kernels as separate stages with NCCL moving
the rows in between, so the two transports can be compared on one box:

  K1  mp_layer_route          router + histogram, this origin's batch counts
      all_gather (NCCL)       the G x E count table, then ONE host sync: NCCL
                              needs the chunk sizes on the host
  K2  mp_layer_permute        own rows into recv, rows for GPU D into the
                              sender's image of D's receive layout
      send/recv (NCCL group)  one chunk per (source, expert) pair, same
                              offsets on both sides
  K3  mp_layer_experts        grouped SwiGLU over recv, outputs in place
      send/recv (NCCL group)  every chunk back to its origin's image
  K5  mp_layer_combine_gather gather-combine from recv / the return images

Every rank calls `forward` (SPMD), with a NCCL process group.
"""

from __future__ import annotations

import ctypes

import numpy as np
import torch
import torch.distributed as dist

from . import _lib
from .routing import receive_layout


class NcclForward:
    STAGES = ("route+counts", "permute", "dispatch", "experts", "return", "combine")

    def __init__(self, layer, group=None, timing: bool = False):
        self.layer = layer
        self.timing = timing
        self.events = []
        self.group = group
        self.lib = layer.lib
        G, E, d = layer.world, layer.shape.E, layer.shape.d
        cap = int(layer._ptrs.recv_cap)
        dev = layer.device
        self.cap = cap
        self.counts = torch.zeros(G * E, dtype=torch.int32, device=dev)
        self.batch_counts = layer.batch_counts
        # images of every peer's receive layout (own entry unused): dispatch out, return in
        self.staging = torch.empty(G * cap, d, dtype=torch.bfloat16, device=dev) if G > 1 else None
        self.ret_stage = torch.empty(G * cap, d, dtype=torch.bfloat16, device=dev) if G > 1 else None
        self.last = {}

    def _stream(self):
        return ctypes.c_void_p(torch.cuda.current_stream(self.layer.device).cuda_stream)

    def forward(self, x: torch.Tensor, out: torch.Tensor | None = None) -> torch.Tensor:
        layer, lib = self.layer, self.lib
        G, E, rank = layer.world, layer.shape.E, layer.rank
        T = x.shape[0]
        if out is None:
            out = torch.empty_like(x)
        st = self._stream()
        ev = []

        def mark():
            if self.timing:
                e = torch.cuda.Event(enable_timing=True)
                e.record()
                ev.append(e)
        mark()
        _lib.check(lib.mp_layer_route(layer._h, x.data_ptr(), T, st), "mp_layer_route")
        if G > 1:
            dist.all_gather_into_tensor(self.counts, self.batch_counts, group=self.group)
        else:
            self.counts.copy_(self.batch_counts)
        counts = self.counts.view(G, E).cpu().numpy()          # host sync: NCCL needs the sizes
        mark()
        stg = self.staging.data_ptr() if G > 1 else None
        _lib.check(lib.mp_layer_permute(layer._h, x.data_ptr(), T, self.counts.data_ptr(), stg, st),
                   "mp_layer_permute")
        mark()
        # (peer, first row in the receive layout, rows) per (source, expert) chunk
        chunks_out, chunks_in = chunk_plan(counts, layer.route, rank) if G > 1 else ([], [])
        if G > 1:
            self._exchange([(self.staging, D * self.cap + a, n, D) for D, a, n in chunks_out],
                           [(layer.recv, a, n, s) for s, a, n in chunks_in])
        mark()
        _lib.check(lib.mp_layer_experts(layer._h, x.data_ptr(), T, self.counts.data_ptr(), st), "mp_layer_experts")
        mark()
        if G > 1:
            self._exchange([(layer.recv, a, n, s) for s, a, n in chunks_in],
                           [(self.ret_stage, D * self.cap + a, n, D) for D, a, n in chunks_out])
        mark()
        rs = self.ret_stage.data_ptr() if G > 1 else None
        _lib.check(lib.mp_layer_combine_gather(layer._h, rs, T, out.data_ptr(), st), "mp_layer_combine_gather")
        mark()
        if self.timing:
            self.events.append(ev)
        row_b = layer.shape.d * 2
        self.last = {"chunks_out": len(chunks_out), "chunks_in": len(chunks_in),
                     "dispatch_bytes": sum(n for _, _, n in chunks_out) * row_b,
                     "return_bytes": sum(n for _, _, n in chunks_in) * row_b}
        return out

    __call__ = forward

    def stage_ms(self) -> dict:
        """Mean per-stage milliseconds of the timed forwards (timing=True; synchronises)."""
        torch.cuda.synchronize(self.layer.device)
        if not self.events:
            return {}
        per = np.array([[ev[i].elapsed_time(ev[i + 1]) for i in range(len(ev) - 1)] for ev in self.events])
        self.events = []
        return dict(zip(self.STAGES, per.mean(axis=0).tolist()))

    def _exchange(self, sends, recvs):
        """One NCCL group of point-to-point ops; chunks to / from one peer are posted in the
        same (expert ascending) order on both sides, so they match pairwise."""
        ops = [dist.P2POp(dist.isend, buf[a:a + n], peer, group=self.group) for buf, a, n, peer in sends]
        ops += [dist.P2POp(dist.irecv, buf[a:a + n], peer, group=self.group) for buf, a, n, peer in recvs]
        if not ops:
            return
        for w in dist.batch_isend_irecv(ops):
            w.wait()


def chunk_plan(counts: np.ndarray, route: np.ndarray, rank: int):
    """(outgoing, incoming) chunk lists of one rank: (peer, first row in the receiving GPU's layout
    (routing.receive_layout), rows) per (source, expert) pair whose rows cross GPUs, expert
    ascending per peer -- the order both sides post their NCCL ops in."""
    G, E = counts.shape
    _, send = receive_layout(counts, route)
    out = [(int(route[rank, e]), int(send[rank, e]), int(counts[rank, e])) for e in range(E)
           if route[rank, e] != rank and counts[rank, e] > 0]
    inc = [(s, int(send[s, e]), int(counts[s, e])) for s in range(G) if s != rank for e in range(E)
           if route[s, e] == rank and counts[s, e] > 0]
    return out, inc
