"""`B200MoELayer`: the GPU drop-in for the reference's per-layer dispatch.

One object per (process, GPU).  It owns an `mp_layer` of the C ABI
(include/moeplace_b200.h) and exposes the reference-facing operations:

* `set_placement(placement, cluster)` -- route table by `_choose_target`'s rule
  (sim.py:433-439) + expert slots filled from a weight source;
* `forward(x)` -- one MoE-layer forward, the counterpart of `_dispatch_layer`
  (sim.py:441-463), all kernels hand-written for sm_100a;
* `activation_counts()` / `activation_stats()` -- the fused GPU histogram as
  reference `ActivationStats.from_counts` (stats.py:67-80);
* `dispatch_accounting()` -- remote invocations / bytes of the last forward in
  the reference's accounting (sim.py:452-456);
* `migrate(...)` -- executes `migration_cost`'s slot diff (cost.py:186-187)
  with NVLink peer copies on a side stream, in rounds that keep every GPU
  within its cap + one staging slot and every expert covered, swapping routes
  only after each round's copies landed (sim.py:520-525).

PyTorch is used for device memory views, streams and `torch.distributed`
plumbing only; every kernel on the path lives in the CUDA library.
"""

from __future__ import annotations

import ctypes
from ctypes import byref, c_void_p

import numpy as np
import torch

from . import _lib
from .errors import InfeasibleError
from .migration import Round, plan_rounds
from .routing import dispatch_accounting, gpu_expert_sets, route_table, route_table_for, uniform_links
from .shapes import LayerShape


class _CudaBuf:
    """Minimal __cuda_array_interface__ exporter for library-owned memory."""

    def __init__(self, ptr: int, shape, typestr: str):
        self.__cuda_array_interface__ = {"shape": tuple(shape), "typestr": typestr, "data": (int(ptr), False),
                                         "version": 3, "strides": None}


def _view(ptr: int, shape, dtype: torch.dtype, device: torch.device) -> torch.Tensor:
    typestr = {torch.bfloat16: "<i2", torch.float32: "<f4", torch.int32: "<i4"}[dtype]
    t = torch.as_tensor(_CudaBuf(ptr, shape, typestr), device=device)
    return t.view(torch.bfloat16) if dtype is torch.bfloat16 else t


def interleave_w13(w1: torch.Tensor, w3: torch.Tensor) -> torch.Tensor:
    """[2f, d]: per 128-row block b, gate rows W1[128b:128b+128] then up rows W3[...]."""
    f, d = w1.shape
    return torch.stack([w1.reshape(f // 128, 128, d), w3.reshape(f // 128, 128, d)], dim=1).reshape(2 * f, d)


class B200MoELayer:
    def __init__(self, shape: LayerShape, *, rank: int = 0, world: int = 1, device: int | None = None,
                 max_tokens: int = 4096, cap_slots: int | None = None, staging_slots: int = 1):
        """cap_slots = floor(GpuSpec.memory / m_e) (domain.py:395-401) expert slots plus
        `staging_slots` (default ONE) that hold incoming experts while a migration is in flight,
        so old copies retire only after new ones land -- the physical pool is
        cap + 1 slots; `migrate` orders the copies into rounds within that bound."""
        self.lib = _lib.load()
        self.shape = shape
        self.rank, self.world = rank, world
        self.device = torch.device("cuda", torch.cuda.current_device() if device is None else device)
        self.max_tokens = max_tokens
        self.cap_slots = shape.E if cap_slots is None else int(cap_slots)
        self.staging_slots = int(staging_slots)
        n_phys = self.cap_slots + self.staging_slots
        desc = _lib.LayerDesc(rank=rank, world=world, device=self.device.index, max_tokens=max_tokens, d=shape.d,
                              f=shape.f, E=shape.E, top_k=shape.k, score_mode=shape.score_mode, renorm=shape.renorm,
                              n_slots=n_phys, shared_f=shape.shared_f, shared_gate=shape.shared_gate)
        h = c_void_p()
        _lib.check(self.lib.mp_layer_create(byref(desc), byref(h)), "mp_layer_create")
        self._h = h
        p = _lib.LayerPtrs()
        _lib.check(self.lib.mp_layer_get_ptrs(h, byref(p)), "mp_layer_get_ptrs")
        self._ptrs = p
        d, f, E, k, T = shape.d, shape.f, shape.E, shape.k, max_tokens
        dev = self.device
        self.n_phys_slots = n_phys
        self.slot_elems = int(p.slot_bytes) // 2
        self.pool = _view(p.pool, (n_phys, self.slot_elems), torch.bfloat16, dev) if n_phys else None
        self.wg = _view(p.wg, (E + shape.shared_gate, d), torch.bfloat16, dev)
        self.bias = _view(p.bias, (E,), torch.float32, dev)
        self.idx = _view(p.idx, (T, k), torch.int32, dev)
        self.gate_w = _view(p.w, (T, k), torch.float32, dev)
        self.pos_dst = _view(p.pos_dst, (T, k), torch.int32, dev)
        self.pos_row = _view(p.pos_row, (T, k), torch.int32, dev)
        self.recv = _view(p.recv, (p.recv_cap, d), torch.bfloat16, dev)
        self.ret = _view(p.ret, (T * k, d), torch.bfloat16, dev)          # expert outputs, (token, slot) order
        self.recv_src = _view(p.recv_src, (p.recv_cap,), torch.int32, dev)
        self.hist = _view(p.hist, (E,), torch.int32, dev)
        self.batch_counts = _view(p.batch_counts, (E,), torch.int32, dev)
        self.w13_shared = _view(p.w13_shared, (2 * shape.shared_f, d), torch.bfloat16, dev) if shape.shared_f else None
        self.w2_shared = _view(p.w2_shared, (d, shape.shared_f), torch.bfloat16, dev) if shape.shared_f else None
        self.shared_gate = _view(p.shared_gate, (T,), torch.float32, dev) if shape.shared_gate else None
        self.slot_of = np.full(E, -1, dtype=np.int32)     # expert -> physical slot on this GPU
        self.route = None
        self._free = list(range(n_phys))
        self._peers_open = world == 1
        self._stream = lambda: ctypes.c_void_p(torch.cuda.current_stream(self.device).cuda_stream)

    # ------------------------------------------------------------------ lifecycle
    def close(self) -> None:
        if getattr(self, "_h", None):
            self.lib.mp_layer_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def open_peers(self, group=None) -> None:
        """Exchange CUDA IPC handles of the NVLink window / weight pool with all ranks."""
        if self.world == 1:
            return
        import torch.distributed as dist

        buf = (ctypes.c_uint8 * 128)()
        _lib.check(self.lib.mp_layer_export_handles(self._h, buf), "mp_layer_export_handles")
        mine = bytes(buf)
        gathered = [None] * self.world
        dist.all_gather_object(gathered, mine, group=group)
        allh = b"".join(gathered)
        _lib.check(self.lib.mp_layer_open_peers(self._h, allh), "mp_layer_open_peers")
        dist.barrier(group=group)
        self._peers_open = True

    # ------------------------------------------------------------------ weights
    def set_router(self, wg: torch.Tensor, bias: torch.Tensor | None = None, w_shared_gate: torch.Tensor | None = None):
        """Router weights Wg [E, d] (+ shared gate row [d]) and the per-origin logit bias [E]."""
        E = self.shape.E
        with torch.no_grad():
            self.wg[:E].copy_(wg.to(self.device, torch.bfloat16))
            if self.shape.shared_gate:
                if w_shared_gate is None:
                    raise ValueError("this shape needs the shared-expert gate row")
                self.wg[E].copy_(w_shared_gate.to(self.device, torch.bfloat16))
            self.bias.copy_(bias.to(self.device, torch.float32) if bias is not None else torch.zeros(E))
        _lib.check(self.lib.mp_layer_prepare_router(self._h, self._stream()), "mp_layer_prepare_router")

    def write_slot(self, slot: int, w1: torch.Tensor, w3: torch.Tensor, w2: torch.Tensor) -> None:
        d, f = self.shape.d, self.shape.f
        with torch.no_grad():
            s = self.pool[slot]
            s[: 2 * f * d].view(2 * f, d).copy_(interleave_w13(w1.to(self.device, torch.bfloat16),
                                                               w3.to(self.device, torch.bfloat16)))
            s[2 * f * d:].view(d, f).copy_(w2.to(self.device, torch.bfloat16))

    def read_slot(self, slot: int):
        d, f = self.shape.d, self.shape.f
        s = self.pool[slot]
        w13 = s[: 2 * f * d].view(f // 128, 2, 128, d)
        return w13[:, 0].reshape(f, d), w13[:, 1].reshape(f, d), s[2 * f * d:].view(d, f)

    def set_shared(self, w1: torch.Tensor, w3: torch.Tensor, w2: torch.Tensor) -> None:
        with torch.no_grad():
            self.w13_shared.copy_(interleave_w13(w1.to(self.device, torch.bfloat16), w3.to(self.device, torch.bfloat16)))
            self.w2_shared.copy_(w2.to(self.device, torch.bfloat16))

    # ------------------------------------------------------------------ placement
    def set_routes(self, route: np.ndarray, slot_of: np.ndarray) -> None:
        route = np.ascontiguousarray(route, dtype=np.int32)
        slot_of = np.ascontiguousarray(slot_of, dtype=np.int32)
        if route.shape != (self.world, self.shape.E):
            raise ValueError(f"route table shape {route.shape} != ({self.world}, {self.shape.E})")
        _lib.check(self.lib.mp_layer_set_routes(self._h, route.ctypes.data, slot_of.ctypes.data, self._stream()),
                   "mp_layer_set_routes")
        self.route = route.copy()
        self.slot_of = slot_of.copy()

    def load_experts(self, experts, weight_source) -> np.ndarray:
        """Place `experts` into free slots (those not yet resident); returns slot_of."""
        if len(experts) > self.cap_slots:
            raise InfeasibleError(f"GPU {self.rank}: {len(experts)} experts exceed its {self.cap_slots} slots")
        slot_of = self.slot_of.copy()
        keep = set(int(e) for e in experts)
        for e in range(self.shape.E):
            if slot_of[e] >= 0 and e not in keep:
                self._free.append(int(slot_of[e]))
                slot_of[e] = -1
        self._free.sort()
        for e in sorted(keep):
            if slot_of[e] < 0:
                s = self._free.pop(0)
                self.write_slot(s, *weight_source(e))
                slot_of[e] = s
        return slot_of

    def set_placement(self, placement, cluster, weight_source, layer: int = 0) -> None:
        """Adopt a reference Placement: route table + resident expert slots."""
        route = route_table_for(placement, cluster, self.shape.E, self.shape.d, 2, layer)
        mine = gpu_expert_sets(placement, layer)[self.rank]
        slot_of = self.load_experts(mine, weight_source)
        torch.cuda.synchronize(self.device)
        self.set_routes(route, slot_of)

    def set_placement_sets(self, gpu_sets, weight_source, link_latency=None, link_bandwidth=None) -> None:
        """Same as set_placement from plain per-GPU expert lists (uniform links by default)."""
        G, E = self.world, self.shape.E
        if link_latency is None or link_bandwidth is None:
            link_latency, link_bandwidth = uniform_links(G)
        route = route_table([frozenset(s) for s in gpu_sets], E, link_latency, link_bandwidth, self.shape.d)
        slot_of = self.load_experts(gpu_sets[self.rank], weight_source)
        torch.cuda.synchronize(self.device)
        self.set_routes(route, slot_of)

    # ------------------------------------------------------------------ forward
    def forward(self, x: torch.Tensor, out: torch.Tensor | None = None, events=None) -> torch.Tensor:
        """One MoE-layer forward of this GPU's tokens.  `events`: optional list of
        _lib.NUM_STAGE_EVENTS torch.cuda.Event(enable_timing=True) (None = skip) recorded
        at the stage boundaries (see include/moeplace_b200.h)."""
        if x.dtype != torch.bfloat16 or x.device != self.device or not x.is_contiguous():
            raise ValueError("x must be a contiguous bf16 tensor on the layer's device")
        if x.dim() != 2 or x.shape[1] != self.shape.d:
            from .errors import DimensionMismatch
            raise DimensionMismatch(f"x has shape {tuple(x.shape)}, layer hidden width is {self.shape.d}")
        T = x.shape[0]
        if out is None:
            out = torch.empty_like(x)
        if events is None:
            rc = self.lib.mp_layer_forward(self._h, x.data_ptr(), out.data_ptr(), T, self._stream())
        else:
            if any(ev is not None and ev.cuda_event == 0 for ev in events):
                raise ValueError("stage events must be created (recorded once) before use")
            arr = (c_void_p * _lib.NUM_STAGE_EVENTS)(*[c_void_p(ev.cuda_event if ev is not None else 0)
                                                       for ev in events])
            rc = self.lib.mp_layer_forward_timed(self._h, x.data_ptr(), out.data_ptr(), T, self._stream(), arr)
        _lib.check(rc, "mp_layer_forward")
        return out

    __call__ = forward

    def last_launches(self) -> int:
        return int(self.lib.mp_layer_last_launches(self._h))

    def exec_plan(self) -> dict:
        """Execution plan the C ABI chose for this layer (mp_layer_config)."""
        return {k: int(self.lib.mp_layer_config(self._h, v)) for k, v in _lib.CFG_KEYS.items()}

    def peer_probe(self, peer: int, nbytes: int, reps: int = 20) -> float:
        """Seconds per `nbytes` copy from `peer` over NVLink (mp_layer_peer_probe; overwrites the
        receive buffer -- call between forwards)."""
        ms = ctypes.c_float()
        _lib.check(self.lib.mp_layer_peer_probe(self._h, peer, int(nbytes), reps, self._stream(), byref(ms)),
                   "mp_layer_peer_probe")
        return ms.value * 1e-3

    def check(self) -> None:
        _lib.check(self.lib.mp_layer_check(self._h, self._stream()), "mp_layer_check")

    def sync_state(self) -> np.ndarray:
        """Flag-protocol state at a quiescent point (synchronises): see mp_layer_sync_state."""
        out = np.zeros(16, dtype=np.uint32)
        _lib.check(self.lib.mp_layer_sync_state(self._h, out.ctypes.data_as(ctypes.c_void_p), self._stream()),
                   "mp_layer_sync_state")
        return out

    # ------------------------------------------------------------------ statistics / accounting
    def activation_counts(self) -> np.ndarray:
        """Cumulative per-expert token counts of this origin (fused router histogram)."""
        return self.hist.cpu().numpy().astype(np.int64)

    def gathered_counts(self, group=None) -> np.ndarray:
        """[G, E] cumulative histograms of all origins (all-gather over torch.distributed)."""
        h = self.hist.clone()
        if self.world == 1:
            return h[None].cpu().numpy().astype(np.int64)
        import torch.distributed as dist
        src = h if dist.get_backend(group) == "nccl" else h.cpu()
        parts = [torch.zeros_like(src) for _ in range(self.world)]
        dist.all_gather(parts, src, group=group)
        return torch.stack([p.cpu() for p in parts]).numpy().astype(np.int64)

    def activation_stats(self, group=None):
        """The GPU histogram as reference ActivationStats (stats.py:67-80); token_count 1 per token."""
        from .errors import import_moeplace
        mp = import_moeplace()
        if mp is None:
            raise RuntimeError("the reference package moeplace is not importable")
        counts = self.gathered_counts(group).astype(float)
        return mp.ActivationStats.from_counts(counts[:, None, :], (self.shape.E,))

    def trace_records(self, T: int, layer: int = 0, t: float = 0.0, server: int | None = None) -> list[dict]:
        """The last forward's routing of this origin as reference trace records (cli.py:91-135);
        server defaults to this GPU's rank."""
        from .trace import trace_records
        return trace_records(self.idx[:T].cpu().numpy(), self.rank if server is None else server, layer, t)

    def reset_counts(self) -> None:
        self.hist.zero_()

    def read_counts(self) -> np.ndarray:
        """Exchanged count table C[src][e] of the last forward (G x E)."""
        buf = np.zeros((self.world, self.shape.E), dtype=np.int32)
        _lib.check(self.lib.mp_layer_read_counts(self._h, buf.ctypes.data, self._stream()), "mp_layer_read_counts")
        return buf

    def dispatch_accounting(self) -> dict:
        """Reference-accounted remote invocations / bytes of the last forward (all origins)."""
        return dispatch_accounting(self.read_counts(), self.route, self.shape.d)

    # ------------------------------------------------------------------ migration
    def plan_migration(self, old_sets, new_sets, phys_slots=None) -> list[Round]:
        """Rounds of the slot diff `new.slots - old.slots` (migration_cost, cost.py:186-187) that keep
        every GPU within its physical slots (cap + staging) and every expert covered
        (migration.plan_rounds).  Every rank computes the same plan; phys_slots defaults to this
        layer's own count on every GPU."""
        phys = phys_slots if phys_slots is not None else [self.n_phys_slots] * self.world
        return plan_rounds(old_sets, new_sets, phys)

    def migrate_round_async(self, rnd: Round, peer_slot_of, stream: torch.cuda.Stream, event: torch.cuda.Event):
        """Issue this GPU's pulls of one round on `stream` (peer_slot_of[n][e] = slot of e on GPU n);
        returns [(expert, destination slot)]."""
        mine = [p for p in rnd.pulls if p.dst_rank == self.rank]
        if len(mine) > len(self._free):
            raise InfeasibleError(f"GPU {self.rank}: {len(mine)} pulls but {len(self._free)} free slots")
        arr = (_lib.CopyOp * max(1, len(mine)))()
        adds = []
        for i, p in enumerate(mine):
            dst = self._free[i]
            arr[i] = _lib.CopyOp(p.src_rank, int(peer_slot_of[p.src_rank][p.expert]), dst)
            adds.append((p.expert, dst))
        with torch.cuda.stream(stream):
            _lib.check(self.lib.mp_layer_migrate(self._h, arr, len(mine), c_void_p(stream.cuda_stream), None),
                       "mp_layer_migrate")
            event.record(stream)  # torch-side record: the CUDA event is created lazily by torch
        for _, dst in adds:
            self._free.remove(dst)
        return adds

    def finish_round(self, rnd: Round, adds, link_latency=None, link_bandwidth=None) -> None:
        """After every GPU's copies of the round landed: the added experts become resident, the
        experts this GPU drops in the round's placement retire, routes swap to that placement
        (migration_complete, sim.py:520-525, one round at a time)."""
        G, E = self.world, self.shape.E
        slot_of = self.slot_of.copy()
        for e, dst in adds:
            slot_of[e] = dst
        keep = set(rnd.sets_after[self.rank])
        for e in range(E):
            if slot_of[e] >= 0 and e not in keep:
                self._free.append(int(slot_of[e]))
                slot_of[e] = -1
        self._free.sort()
        if link_latency is None or link_bandwidth is None:
            link_latency, link_bandwidth = uniform_links(G)
        route = route_table([frozenset(s) for s in rnd.sets_after], E, link_latency, link_bandwidth, self.shape.d)
        self.set_routes(route, slot_of)

    def migrate(self, old_sets, new_sets, *, phys_slots=None, stream: torch.cuda.Stream | None = None,
                while_copying=None, link_latency=None, link_bandwidth=None, group=None) -> dict:
        """Execute an adopted plan (SPMD: every rank calls it): per round, NVLink pulls on the side
        `stream` while `while_copying()` (e.g. forwards on the current placement) keeps traffic
        flowing, then -- after every GPU's copies landed -- the route swap.  Returns accounting
        (this GPU's adds, rounds, copy time)."""
        import torch.distributed as dist
        rounds = self.plan_migration(old_sets, new_sets, phys_slots)
        side = stream or torch.cuda.Stream(self.device)
        main = torch.cuda.current_stream(self.device)
        copy_ms, n_overlap, all_adds = 0.0, 0, []
        for rnd in rounds:
            if self.world > 1:
                slot_maps = [None] * self.world
                dist.all_gather_object(slot_maps, self.slot_of.tolist(), group=group)
            else:
                slot_maps = [self.slot_of.tolist()]
            # the slots freed by the previous round may still be read by forwards queued before its swap
            side.wait_stream(main)
            t0, done = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            t0.record(side)
            adds = self.migrate_round_async(rnd, slot_maps, side, done)
            if while_copying is not None:
                n_overlap += while_copying() or 0
            done.synchronize()
            copy_ms += t0.elapsed_time(done)
            if self.world > 1:
                dist.barrier(group=group)  # every GPU's copies of this round landed
            self.finish_round(rnd, adds, link_latency, link_bandwidth)
            if self.world > 1:
                dist.barrier(group=group)  # every GPU swapped before the next round overwrites slots
            all_adds += adds
        return {"rounds": len(rounds), "adds": all_adds, "copy_ms": copy_ms, "forwards_during_copy": n_overlap}


class HostPipeline:
    """Streams token batches from pinned host memory through a B200MoELayer.

    Serving-style end-to-end path: batch i's host->device copy runs on a copy-in
    stream while batch i-1 is in the layer and batch i-2's output drains on a
    copy-out stream (PCIe is full duplex), with `depth` device buffers per
    direction so a slow copy of one batch does not stall the next batch's layer.
    Each batch still crosses the host boundary in full: x in, layer output out.
    """

    def __init__(self, layer: B200MoELayer, T: int, depth: int = 2):
        self.layer = layer
        dev = layer.device
        d = layer.shape.d
        self.depth = depth  # device buffers per direction (batches in flight)
        self.xd = [torch.empty(T, d, device=dev, dtype=torch.bfloat16) for _ in range(depth)]
        self.od = [torch.empty(T, d, device=dev, dtype=torch.bfloat16) for _ in range(depth)]
        self.s_in = torch.cuda.Stream(dev)
        self.s_out = torch.cuda.Stream(dev)
        self.compute = torch.cuda.current_stream(dev)
        self.ev_in = [torch.cuda.Event() for _ in range(depth)]
        self.ev_comp = [torch.cuda.Event() for _ in range(depth)]
        self.ev_out = [torch.cuda.Event() for _ in range(depth)]
        self.n = 0

    def submit(self, x_host: torch.Tensor, out_host: torch.Tensor, start_event=None) -> None:
        """Enqueue one batch: x_host [T, d] pinned bf16 -> layer -> out_host [T, d] pinned bf16.
        start_event: recorded on the copy-in stream right before this batch's copy starts."""
        b = self.n % self.depth
        if self.n >= self.depth:
            self.s_in.wait_event(self.ev_comp[b])      # xd[b] free once batch n-depth left the layer
        if start_event is not None:
            start_event.record(self.s_in)
        with torch.cuda.stream(self.s_in):
            self.xd[b].copy_(x_host, non_blocking=True)
            self.ev_in[b].record(self.s_in)
        self.compute.wait_event(self.ev_in[b])
        if self.n >= self.depth:
            self.compute.wait_event(self.ev_out[b])    # od[b] drained to the host
        with torch.cuda.stream(self.compute):
            self.layer.forward(self.xd[b], self.od[b])
            self.ev_comp[b].record(self.compute)
        self.s_out.wait_event(self.ev_comp[b])
        with torch.cuda.stream(self.s_out):
            out_host.copy_(self.od[b], non_blocking=True)
            self.ev_out[b].record(self.s_out)
        self.n += 1

    def drain(self) -> None:
        self.s_out.synchronize()
        self.compute.synchronize()


def capture_graph(fn, warmup: int = 1):
    """Capture fn() (a sequence of layer forwards on static buffers) into a CUDA graph.

    The forward is graph-safe: no host synchronisation, flag epochs and
    count-table parity live on the device, every tensor map is bound to a
    static buffer.  Warm-up calls run eagerly first (attribute setup).
    """
    for _ in range(warmup):
        fn()
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        fn()
    return g


class MoEStack:
    """Several MoE layers applied in sequence -- ModelSpec.num_layers > 1.

    The reference walks a request through its layers strictly in order
    (sim.py:500-505); each layer has its own placement, expert weights and
    activation statistics (one B200MoELayer per layer).  Non-MoE compute
    between layers is outside the path (modelled as a constant).
    """

    def __init__(self, layers: list[B200MoELayer]):
        if not layers:
            raise ValueError("a stack needs at least one layer")
        self.layers = layers
        d = layers[0].shape.d
        if any(l.shape.d != d for l in layers):
            raise ValueError("all layers of a stack share the hidden width")
        self._bufs = {}

    def forward(self, x: torch.Tensor, out: torch.Tensor | None = None) -> torch.Tensor:
        key = (x.shape[0], x.device)
        if key not in self._bufs:
            self._bufs[key] = [torch.empty_like(x), torch.empty_like(x)]
        bufs = self._bufs[key]
        cur = x
        for i, layer in enumerate(self.layers):
            dst = out if (i == len(self.layers) - 1 and out is not None) else bufs[i & 1]
            cur = layer.forward(cur, dst)
        return cur

    __call__ = forward

    def capture(self, x: torch.Tensor, out: torch.Tensor, warmup: int = 1):
        """CUDA graph of the whole stack on static x / out buffers (replay with g.replay())."""
        return capture_graph(lambda: self.forward(x, out), warmup)
