#!/usr/bin/env python
"""Benchmark of the B200 MoE-layer forward (BASELINE.json metric).

Metric: MoE-layer tokens/s (whole job, all GPUs) with p50 batch latency and
remote-dispatch bytes.  One "step" = one MoE-layer forward of T tokens per GPU
(weak scaling: T fixed per GPU).  Default workload (N=1): the Mixtral-8x7B
layer shape (BASELINE.json configs[1]), T = 4096 tokens per GPU,
activation-aware placement ("ours") from the reference solver.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config mixtral] [--impl b200|reference]

N > 1 is launched by torchrun (one process per GPU; RANK/LOCAL_RANK/WORLD_SIZE
from the env).  Rank 0 prints one JSON line.
"""

from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time
from pathlib import Path

import numpy as np

REPO = Path(__file__).resolve().parent
sys.path.insert(0, str(REPO))

METRIC = "MoE-layer tokens/s (p50 batch latency, remote-dispatch bytes)"
UNIT = "tokens/s"
PEAKS_FALLBACK = {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0, "bf16_tflops_sustained": 1400.0}
N_ROTATE = 8  # distinct input batches cycled through the timed region


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=200)
    ap.add_argument("--warmup", type=int, default=10)
    ap.add_argument("--config", default="mixtral")
    ap.add_argument("--tokens", type=int, default=4096, help="tokens per GPU per step")
    ap.add_argument("--strategy", default="ours")
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--seed", type=int, default=0)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--cpu-tokens", type=int, default=256, help="tokens per CPU-baseline sample")
    ap.add_argument("--cpu-seconds", type=float, default=10.0)
    ap.add_argument("--stages", action="store_true", help="print the per-stage table on stderr")
    ap.add_argument("--layers", type=int, default=4, help="--scenario stack: MoE layers in the stack")
    ap.add_argument("--scenario", default="steady", choices=["steady", "shift", "stack", "transport", "calibrate"],
                    help="shift: BASELINE config 5, drifting routing + expert migration vs static placement")
    return ap.parse_args()


# ----------------------------------------------------------------------------- dist helpers
def dist_env():
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return rank, local, world


def load_peaks():
    p = REPO / "MEASURED_PEAKS.json"
    if p.exists():
        d = json.loads(p.read_text())
        return d, "measured"
    return PEAKS_FALLBACK, "fallback"


def init_dist_quiet(dev):
    """NCCL process group; keep stdout to the single JSON line (the NCCL version banner is
    printed on the first communicator creation, so fd 1 is silenced until then)."""
    import torch.distributed as dist
    os.environ["NCCL_DEBUG"] = "WARN"
    sys.stdout.flush()
    saved = os.dup(1)
    devnull = os.open(os.devnull, os.O_WRONLY)
    os.dup2(devnull, 1)
    try:
        dist.init_process_group("nccl", device_id=dev)
        dist.barrier()
    finally:
        sys.stdout.flush()
        os.dup2(saved, 1)
        os.close(saved)
        os.close(devnull)


# ----------------------------------------------------------------------------- clocks
def agree_max(v, world: int, dev) -> int:
    """max of an int (or bool) over the ranks: loop counts that decide how many layer
    forwards a rank runs must agree, since each forward is a lock-step of every rank."""
    v = int(v)
    if world > 1:
        import torch
        import torch.distributed as dist
        t = torch.tensor([v], dtype=torch.int64, device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        v = int(t.item())
    return v


class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled DURING the timed region."""

    FIELDS = ("timestamp,index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, device_index: int):
        self.dev = device_index
        self.proc = None
        self.lines = []
        self.window = None  # (start, end) host datetimes of the timed region; samples outside are dropped

    def mark(self, which: str):
        import datetime
        now = datetime.datetime.now()
        self.window = (now, None) if which == "start" else (self.window[0] if self.window else now, now)

    def start(self):
        if os.environ.get("MP_BENCH_NO_CLOCKS") == "1":  # diagnostics: no nvidia-smi sampler
            return
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits", "-lms", "100",
                 "-i", str(self.dev)], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self._t = threading.Thread(target=self._read, daemon=True)
            self._t.start()
        except Exception:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def stop(self) -> dict:
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        time.sleep(0.25)
        self.proc.terminate()
        try:
            self.proc.wait(timeout=2)
        except Exception:
            self.proc.kill()
        self._t.join(timeout=1)
        sm, mx, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        import datetime

        def collect(before_s, after_s=0.1):
            sm, mx, reasons = [], [], set()
            for ln in self.lines:
                parts = [p.strip() for p in ln.split(",")]
                if len(parts) < 10:
                    continue
                try:
                    ts = datetime.datetime.strptime(parts[0], "%Y/%m/%d %H:%M:%S.%f")
                    if self.window and self.window[1] is not None and not (
                            self.window[0] - datetime.timedelta(seconds=before_s) <= ts
                            <= self.window[1] + datetime.timedelta(seconds=after_s)):
                        continue
                    sm.append(float(parts[2]))
                    mx.append(float(parts[3]))
                except ValueError:
                    continue
                for nm, v in zip(names, parts[6:10]):
                    if v.lower() == "active":
                        reasons.add(nm)
            return sm, mx, reasons

        # samples every 100 ms: a short timed region may hold one or none, so widen the window
        # backwards into the loaded settle phase (never forwards: the GPU idles after the region)
        sm, mx, reasons = collect(0.1)
        if len(sm) < 2:
            sm, mx, reasons = collect(0.3)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": sorted(reasons), "samples": len(sm)}


def stage_roofline(shape, T, rows, stage_ms, hbm_gbs):
    """Algorithmic HBM bytes of the memory-bound stages over their diagnostic-pass
    time (event-bounded, so launch gaps are included: a lower bound on the kernel's own rate)."""
    d, k = shape.d, shape.k
    algo = {
        "router": T * d * 2 + T * k * 8,                           # x once + idx/w out
        "permute_dispatch": T * d * 2 + T * k * d * 2 + T * k * 8,  # x once, k row copies, positions
        "combine_return": T * k * d * 2 + T * k * 4 + T * d * 2 + (T * d * 2 if shape.shared_f else 0),
    }
    out = {}
    for name, b in algo.items():
        ms = stage_ms.get(name, 0.0)
        gbs = b / (ms * 1e-3) / 1e9 if ms > 0 else None
        out[name] = {"bytes": b, "ms": ms, "GB/s": gbs, "frac_hbm": gbs / hbm_gbs if gbs else None}
    # the router's exact logits are nine 8-bit limb GEMMs on the tensor cores (kind::i8):
    # their integer ops over the time, next to the HBM view above
    n_pad = max(16, (shape.E + shape.shared_gate + 15) // 16 * 16)
    r_ms = stage_ms.get("router", 0.0)
    if r_ms > 0:
        ops = 9 * 2.0 * T * n_pad * d
        out["router"].update({"i8_OP": ops, "i8_TOP/s": ops / (r_ms * 1e-3) / 1e12})
    return out


# ----------------------------------------------------------------------------- placement
def build_placement_sets(shape, G, counts, strategy, seed):
    """Per-GPU expert lists from the reference placement solver (build_placement,
    reference placement.py:541-566) on the GPU-measured activation counts."""
    from paper_2508_12851_b200.errors import import_moeplace
    from paper_2508_12851_b200.shapes import cluster_spec, model_spec, slot_caps
    from paper_2508_12851_b200.routing import gpu_expert_sets

    caps = slot_caps(shape, G)
    if G == 1:
        return [list(range(shape.E))], caps, "all-local (G=1)"
    mp = import_moeplace()
    if mp is None:
        # documents produced offline by the same solver on the expected counts T*k*p
        # (tests/golden/make_golden.py); used only when moeplace is absent on the box
        docs = json.loads((REPO / "paper_2508_12851_b200" / "placements" / "bench_placements.json").read_text())
        key = f"{shape.name}_G{G}_{strategy}"
        if key not in docs:
            raise RuntimeError(f"moeplace not importable and no stored placement {key}")
        return gpu_expert_sets(docs[key]["placement"], 0), docs[key]["caps"], f"stored build_placement({strategy!r})"
    cluster = cluster_spec(shape, G, caps)
    model = model_spec(shape)
    stats = mp.ActivationStats.from_counts(np.asarray(counts, dtype=float)[:, None, :], (shape.E,))
    placement = mp.build_placement(strategy, cluster, model, stats, seed)
    rep = mp.validate_placement(placement, cluster, model)
    if not rep.ok:
        raise RuntimeError(f"invalid placement: {rep}")
    return gpu_expert_sets(placement, 0), caps, f"moeplace.build_placement({strategy!r})"


def uniform_sets(shape, G):
    """place_uniform's round-robin partition (reference placement.py:407-422), for the naive comparison."""
    sets = [[] for _ in range(G)]
    for e in range(shape.E):
        sets[e % G].append(e)
    return sets


# ----------------------------------------------------------------------------- CPU baseline
def cpu_layer_sample(shape, T_cpu, seed, weights_cpu, wg_np, bias_np):
    """One oracle forward of T_cpu tokens (G=1, all experts local)."""
    from oracle import moe_oracle as orc
    x = orc.synthetic_tokens(0, T_cpu, shape.d, seed)
    route = np.zeros((1, shape.E), dtype=np.int32)
    shared = weights_cpu.get("shared")
    wsg = wg_np[shape.E] if shape.shared_gate else None
    orc.moe_layer_forward(shape, [x], wg_np[:shape.E], [bias_np], route, weights_cpu["experts"], shared, wsg)


def cpu_weights(shape, seed, expert_src):
    """fp32 host copies of the expert weights (the same values the GPU holds)."""
    import torch
    from paper_2508_12851_b200 import workload as wl
    experts = {}
    for e in range(shape.E):
        w1, w3, w2 = expert_src(e)
        experts[e] = (w1.float().cpu().numpy(), w3.float().cpu().numpy(), w2.float().cpu().numpy())
    out = {"experts": experts}
    if shape.shared_f:
        dev = torch.device("cuda", torch.cuda.current_device())
        s = wl.shared_weights(shape.d, shape.shared_f, dev, seed)
        out["shared"] = tuple(w.float().cpu().numpy() for w in s)
    return out


def cpu_threads() -> tuple[int, dict]:
    """Use every host core for the oracle's numpy BLAS (threadpoolctl sets OpenBLAS' pool; torch's
    setting does not govern it) and report what actually runs."""
    import torch
    threads = len(os.sched_getaffinity(0)) if hasattr(os, "sched_getaffinity") else (os.cpu_count() or 1)
    torch.set_num_threads(threads)
    info = {"cpu_model": None, "blas": None}
    try:
        from threadpoolctl import threadpool_info, threadpool_limits
        threadpool_limits(threads)
        pools = [p for p in threadpool_info() if p.get("user_api") == "blas"]
        if pools:
            info["blas"] = f"{pools[0].get('internal_api')} {pools[0].get('version')}, {pools[0].get('num_threads')} threads"
            threads = int(pools[0].get("num_threads", threads))
    except Exception:
        pass
    try:
        for ln in open("/proc/cpuinfo"):
            if ln.startswith("model name"):
                info["cpu_model"] = ln.split(":", 1)[1].strip()
                break
    except OSError:
        pass
    return threads, info


def time_cpu_baseline(shape, seed, T_cpu, budget_s, weights_cpu, wg_np, bias_np, min_reps=1):
    threads, _ = cpu_threads()
    cpu_layer_sample(shape, min(T_cpu, 32), seed, weights_cpu, wg_np, bias_np)  # warm (BLAS init)
    reps, t0 = 0, time.perf_counter()
    while True:
        cpu_layer_sample(shape, T_cpu, seed, weights_cpu, wg_np, bias_np)
        reps += 1
        el = time.perf_counter() - t0
        if el >= budget_s or reps >= 1000 or (reps >= min_reps and el * (reps + 1) / reps > 3 * budget_s):
            break
    el = time.perf_counter() - t0
    return reps * T_cpu / el, reps, el, threads


# ----------------------------------------------------------------------------- main (B200 arm)
def setup_bench_layer(args):
    """Process group, weights, the reference solver's placement on GPU-measured counts, the layer
    and its warm-up (shared by the steady and transport scenarios)."""
    import torch
    import torch.distributed as dist
    from paper_2508_12851_b200 import _lib, workload as wl
    from paper_2508_12851_b200.layer import B200MoELayer, HostPipeline
    from paper_2508_12851_b200.routing import dispatch_accounting, route_table, uniform_links
    from paper_2508_12851_b200.shapes import get_shape

    rank, local, world = dist_env()
    if world != args.gpus:
        raise SystemExit(f"--gpus {args.gpus} but WORLD_SIZE={world}")
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        from paper_2508_12851_b200.numa import bind_to_gpu_node
        bind_to_gpu_node(local)  # host buffers of the e2e path stay on the GPU's NUMA node
        init_dist_quiet(dev)
    shape = get_shape(args.config)
    T, G, seed = args.tokens, world, args.seed

    # ---- router weights + per-origin skew (the reference's Dirichlet recipe)
    wg = wl.router_weights(shape.E + shape.shared_gate, shape.d, dev, seed)
    bias = wl.origin_bias(rank, shape.E, seed)
    expert_src = lambda e: wl.expert_weights(e, shape.d, shape.f, dev, seed)

    # ---- activation counts of a warm-up batch (GPU router kernel) -> placement
    lib = _lib.load()
    import ctypes
    packed = torch.empty(lib.mp_router_packed_bytes(shape.E + shape.shared_gate, shape.d), device=dev,
                         dtype=torch.uint8)
    st = ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)
    _lib.check(lib.mp_router_pack(ctypes.c_void_p(wg.data_ptr()), shape.E + shape.shared_gate, shape.d,
                                  ctypes.c_void_p(packed.data_ptr()), st))
    xw = wl.tokens(T, shape.d, dev, seed, rank, batch=10_000)
    idx = torch.empty(T, shape.k, dtype=torch.int32, device=dev)
    wtmp = torch.empty(T, shape.k, dtype=torch.float32, device=dev)
    hist = torch.zeros(shape.E, dtype=torch.int32, device=dev)
    bias_d = bias.to(dev)
    _lib.check(lib.mp_router_topk_hist(ctypes.c_void_p(xw.data_ptr()), ctypes.c_void_p(packed.data_ptr()),
                                       ctypes.c_void_p(bias_d.data_ptr()), T, shape.d, shape.E, shape.shared_gate,
                                       shape.k, shape.score_mode, shape.renorm, ctypes.c_void_p(idx.data_ptr()),
                                       ctypes.c_void_p(wtmp.data_ptr()), None, ctypes.c_void_p(hist.data_ptr()), st))
    if world > 1:
        allh = [torch.zeros_like(hist) for _ in range(world)]
        dist.all_gather(allh, hist)
        counts = torch.stack(allh).cpu().numpy()
    else:
        counts = hist[None].cpu().numpy()
    sets, caps, solver = build_placement_sets(shape, G, counts, args.strategy, seed)

    # ---- the layer
    layer = B200MoELayer(shape, rank=rank, world=world, device=local, max_tokens=T, cap_slots=caps[rank])
    layer.open_peers()
    layer.set_router(wg[:shape.E], bias, wg[shape.E] if shape.shared_gate else None)
    if shape.shared_f:
        layer.set_shared(*wl.shared_weights(shape.d, shape.shared_f, dev, seed))
    layer.set_placement_sets(sets, expert_src)
    del xw, idx, wtmp
    torch.cuda.synchronize()

    # rotating input batches (+ weights) exceed L2: 8 x T x d bf16 + all expert slots
    xs = [wl.tokens(T, shape.d, dev, seed, rank, batch=b) for b in range(N_ROTATE)]
    out = torch.empty(T, shape.d, device=dev, dtype=torch.bfloat16)
    stream = torch.cuda.current_stream()

    def barrier():
        if world > 1:
            dist.barrier()

    for i in range(args.warmup):
        layer.forward(xs[i % N_ROTATE], out)
    torch.cuda.synchronize()
    layer.check()
    from types import SimpleNamespace
    return SimpleNamespace(torch=torch, dist=dist, _lib=_lib, rank=rank, local=local, world=world, dev=dev,
                           shape=shape, T=T, G=G, seed=seed, layer=layer, xs=xs, out=out, stream=stream,
                           barrier=barrier, sets=sets, caps=caps, solver=solver, wg=wg, bias=bias,
                           expert_src=expert_src, lib=lib)


def main_b200(args):
    import torch
    import torch.distributed as dist
    from paper_2508_12851_b200 import _lib
    from paper_2508_12851_b200.layer import HostPipeline
    from paper_2508_12851_b200.routing import dispatch_accounting, route_table, uniform_links

    b = setup_bench_layer(args)
    rank, local, world, dev = b.rank, b.local, b.world, b.dev
    shape, T, G, seed, layer, xs, out, stream, barrier = b.shape, b.T, b.G, b.seed, b.layer, b.xs, b.out, b.stream, b.barrier
    sets, caps, solver, wg, bias, expert_src = b.sets, b.caps, b.solver, b.wg, b.bias, b.expert_src

    # ---- timed region (device time, CUDA events).  Inside it only the K3 (grouped GEMM)
    # boundaries are recorded per step -- the roofline's kernel duration; the full per-stage
    # breakdown comes from a separate diagnostic pass below.
    K = args.steps
    NS = _lib.NUM_STAGE_EVENTS

    def make_events(n, which):
        rows = []
        for _ in range(n):
            row = [torch.cuda.Event(enable_timing=True) if j in which else None for j in range(NS)]
            for ev in row:
                if ev is not None:
                    ev.record(stream)  # torch creates the CUDA event lazily on first record
            rows.append(row)
        return rows

    g0, g1, g2 = _lib.GEMM_START, _lib.GEMM1_END, _lib.GEMM_END
    evs = make_events(K, {0, g0, g1, g2, _lib.MAIN_STAGE_EVENTS - 1})
    torch.cuda.synchronize()
    sampler = ClockSampler(local)
    sampler.start()
    # settle: the sampler's start and the event setup left the GPU idle; keep it busy for
    # ~150 ms (untimed, extra warm-up) so the timed steps start from the loaded power / clock
    # state instead of ramping out of idle inside a short timed region
    # (in chunks of 8 whose continuation every rank agrees on: at G > 1 each forward is a
    # lock-step of all ranks, so every rank must run the same number of them)
    t_settle = time.time()
    i_settle = 0
    while True:
        for _ in range(8):
            layer.forward(xs[i_settle % N_ROTATE], out)
            i_settle += 1
        torch.cuda.synchronize()
        if not agree_max(time.time() - t_settle < 0.15, world, dev):
            break
    barrier()
    torch.cuda.synchronize()
    sampler.mark("start")
    start = torch.cuda.Event(enable_timing=True)
    end = torch.cuda.Event(enable_timing=True)
    start.record(stream)
    h0 = time.perf_counter()
    for i in range(K):
        layer.forward(xs[i % N_ROTATE], out, events=evs[i])
    end.record(stream)
    host_enqueue_ms = (time.perf_counter() - h0) * 1e3 / K  # host time to enqueue one forward
    torch.cuda.synchronize()
    sampler.mark("end")
    barrier()
    clocks = sampler.stop()
    layer.check()
    t_ms = start.elapsed_time(end)
    step_ms = [evs[i][0].elapsed_time(evs[i][_lib.MAIN_STAGE_EVENTS - 1]) for i in range(K)]
    gemm1_ms = np.array([evs[i][g0].elapsed_time(evs[i][g1]) for i in range(K)])
    gemm2_ms = np.array([evs[i][g1].elapsed_time(evs[i][g2]) for i in range(K)])

    # ---- diagnostic pass (not timed for `value`): every stage boundary
    n_diag = min(K, 50)
    dev_ = make_events(n_diag, set(range(NS)))
    torch.cuda.synchronize()
    barrier()
    for i in range(n_diag):
        layer.forward(xs[i % N_ROTATE], out, events=dev_[i])
    torch.cuda.synchronize()
    barrier()
    NM = _lib.MAIN_STAGE_EVENTS
    stage_ms = np.array([[dev_[i][j].elapsed_time(dev_[i][j + 1]) for j in range(NM - 1)] for i in range(n_diag)])
    side_ms = None
    if layer.exec_plan()["split_m"] > 0:
        # the small-group chain on the side stream: its span and its offset from GEMM start
        side_ms = [float(np.mean([dev_[i][NM].elapsed_time(dev_[i][NM + 1]) for i in range(n_diag)])),
                   float(np.mean([dev_[i][_lib.GEMM_START].elapsed_time(dev_[i][NM + 1]) for i in range(n_diag)]))]
    launches = layer.last_launches() * K
    exec_plan = layer.exec_plan()
    acc_ours = layer.dispatch_accounting()
    counts_last = layer.read_counts()
    recv_rows = int(np.sum([counts_last[s, e] for s in range(G) for e in range(shape.E) if layer.route[s, e] == rank]))
    # expert slots this GPU streamed per step (groups with rows) -- the weight bytes of K3
    active_local = int(sum(1 for e in range(shape.E)
                           if sum(counts_last[s, e] for s in range(G) if layer.route[s, e] == rank) > 0))
    # K4 wire bytes of this GPU: token rows it dispatched to peers (inside the permute kernel)
    # and expert-output rows it returned to peers (inside its GEMM2 epilogue)
    sent_rows = int(sum(counts_last[rank, e] for e in range(shape.E) if layer.route[rank, e] != rank))
    ret_rows = int(sum(counts_last[s, e] for s in range(G) for e in range(shape.E)
                       if s != rank and layer.route[s, e] == rank))

    # ---- e2e: the same forward through the public API with HOST buffers: every step copies its
    # x from pinned host memory and its output back (HostPipeline overlaps the copies of
    # neighbouring batches with the layer on separate streams)
    xh = [x.cpu().pin_memory() for x in xs]
    oh = [torch.empty(T, shape.d, dtype=torch.bfloat16).pin_memory() for _ in range(N_ROTATE)]
    pipe = HostPipeline(layer, T)
    torch.cuda.synchronize()
    barrier()
    # steady state of a serving stream: the warm-up batches flow straight into the timed ones
    # (no drain in between); the region runs from the first timed batch's host->device copy
    # (recorded when its buffer frees up) to the last timed batch's device->host copy, so it
    # holds all K batches' copies in both directions and their K forwards
    # (>= 150 ms of them, like the device-timed region's settle phase, so the timed batches run
    # in the loaded power state)
    n_pre = max(2, min(args.warmup, 4), min(64, int(np.ceil(150.0 / max(t_ms / K, 1e-3)))))
    n_pre = agree_max(n_pre, world, dev)  # the same number of forwards on every rank
    for i in range(n_pre):
        pipe.submit(xh[i % N_ROTATE], oh[i % N_ROTATE])
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    for i in range(K):
        pipe.submit(xh[i % N_ROTATE], oh[i % N_ROTATE], start_event=e0 if i == 0 else None)
    pipe.s_out.wait_stream(pipe.compute)
    e1.record(pipe.s_out)
    torch.cuda.synchronize()
    barrier()
    e2e_ms = e0.elapsed_time(e1)
    layer.check()
    # the host copy of the last output is the layer's output
    assert torch.equal(oh[(K - 1) % N_ROTATE], pipe.od[(pipe.n - 1) % pipe.depth].cpu())

    # ---- max over ranks
    vals = torch.tensor([t_ms, e2e_ms, float(np.median(step_ms))], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(vals, op=dist.ReduceOp.MAX)
    t_ms, e2e_ms, p50_ms = vals.tolist()
    stage_mean = stage_ms.mean(axis=0)
    stage_t = torch.tensor(stage_mean, dtype=torch.float64, device=dev)
    gemm_local = float(gemm1_ms.mean() + gemm2_ms.mean())
    stage_local = dict(zip(_lib.STAGES, stage_mean.tolist()))
    rank_t = torch.tensor([recv_rows, gemm_local, active_local, sent_rows, ret_rows,
                           stage_local["permute_dispatch"], float(gemm2_ms.mean())], dtype=torch.float64,
                          device=dev)
    if world > 1:
        dist.all_reduce(stage_t, op=dist.ReduceOp.MAX)
        parts = [torch.zeros_like(rank_t) for _ in range(world)]
        dist.all_gather(parts, rank_t)
        per_rank = [(int(p[0].item()), float(p[1].item())) for p in parts]
        active_list = [int(p[2].item()) for p in parts]
        k4_rank = [p[3:].tolist() for p in parts]
    else:
        per_rank = [(recv_rows, gemm_local)]
        active_list = [active_local]
        k4_rank = [[sent_rows, ret_rows, stage_local["permute_dispatch"], float(gemm2_ms.mean())]]
    # K4 over NVLink: dispatch wire rate = a GPU's outgoing token rows / its permute-kernel time
    # (rows are stored to the peers' receive buffers by that kernel); the return rides the GEMM2
    # epilogue, so its rate is bounded by the GEMM, reported as bytes / GEMM2 time
    nvl_peak = 770.0
    k4 = None
    peer_bw = measure_peer_copy(layer, G, rank) / 1e9 if G > 1 else None
    peer_lat = measure_peer_latency(layer, rank, G) if G > 1 else None
    if G > 1:
        row_b = shape.d * 2
        disp = [r[0] * row_b / (r[2] * 1e-3) / 1e9 if r[2] > 0 else 0.0 for r in k4_rank]
        retr = [r[1] * row_b / (r[3] * 1e-3) / 1e9 if r[3] > 0 else 0.0 for r in k4_rank]
        k4 = {"dispatch_bytes_per_gpu": [int(r[0] * row_b) for r in k4_rank],
              "return_bytes_per_gpu": [int(r[1] * row_b) for r in k4_rank],
              "dispatch_GBps_per_gpu": disp, "return_GBps_per_gpu": retr,
              "dispatch_frac_of_peer_copy": max(disp) / nvl_peak, "peak_GBps": nvl_peak,
              "peak_source": "measured peer copy per direction (B200_PROFILING.md)",
              "peer_copy_GBps_this_box": peer_bw, "small_copy_latency_s_this_box": peer_lat,
              "note": "dispatch = outgoing rows / permute kernel time (the kernel also writes the local rows); "
                      "return = rows sent back / GEMM2 time (the stores ride the GEMM epilogue)"}
    rows_list = [r for r, _ in per_rank]

    # naive placement accounting on the same counts (counts do not depend on placement)
    lat, bw = uniform_links(G)
    naive_route = route_table([frozenset(s) for s in uniform_sets(shape, G)], shape.E, lat, bw, shape.d)
    acc_naive = dispatch_accounting(counts_last, naive_route, shape.d)

    # ---- roofline of the dominant kernel: grouped_gemm_kernel (GEMM1 SwiGLU + GEMM2), every GPU;
    # the headline figure is the GPU with the most routed rows (it sets the step time)
    peaks, peaks_src = load_peaks()
    # algorithmic: 6*d*f per routed (token, expert) pair, plus 6*d*f_shared per token when the
    # shared expert rides in the same launches (fused plan)
    shared_flops = 2.0 * T * 3 * shape.d * shape.shared_f if exec_plan["fuse_shared"] else 0.0
    per_rank_tf = [(2.0 * r * 3 * shape.d * shape.f + shared_flops) / (ms * 1e-3) / 1e12 if ms > 0 else 0.0
                   for r, ms in per_rank]
    hot = int(np.argmax(rows_list))
    flops = 2.0 * rows_list[hot] * 3 * shape.d * shape.f + shared_flops
    achieved_tflops = per_rank_tf[hot]
    # the denominator matches the regime the timed region ran in: it follows >= 150 ms of load
    # (settle phase), so under the 1 kW cap (SM clock well below max, sw_power_cap) K3 runs in
    # the regime of the sustained figure; at full clock, the burst figure.  Both fractions are
    # reported.
    peak_burst = float(peaks.get("bf16_tflops"))
    peak_sus = float(peaks.get("bf16_tflops_sustained", peak_burst))
    capped = bool(clocks.get("sm_mhz") and clocks.get("sm_max_mhz")
                  and clocks["sm_mhz"] < 0.92 * clocks["sm_max_mhz"])
    peak = peak_sus if capped else peak_burst
    peak_regime = "sustained (power-capped clocks in the timed region)" if capped else "burst (full clocks)"
    # the same launches seen from HBM: every active expert slot's weights are streamed once
    # (+ the shared expert's when fused); small batches are bound by this, not by the tensor pipe
    w_bytes = active_list[hot] * shape.expert_bytes + (3 * shape.d * shape.shared_f * 2 if exec_plan["fuse_shared"]
                                                        else 0)
    w_gbs = w_bytes / (per_rank[hot][1] * 1e-3) / 1e9 if per_rank[hot][1] > 0 else None
    hbm_peak = float(peaks.get("hbm_gbs", 6546.6))
    ridge = peak * 1e12 / (hbm_peak * 1e9)  # flop/B where the two roofs meet
    bound = "tensor" if flops / max(w_bytes, 1) >= ridge else "hbm"
    traffic = None
    tf = REPO / "profiles" / "traffic.json"
    if tf.exists():
        try:
            traffic = json.loads(tf.read_text()).get(f"{shape.name}_G{G}_T{T}")
        except Exception:
            traffic = None

    if rank != 0:
        if world > 1:
            dist.barrier()
            dist.destroy_process_group()
        layer.close()
        return

    # ---- CPU baseline (rank 0, N=1 only)
    cpu = None
    if not args.no_cpu_baseline and world == 1:
        wcpu = cpu_weights(shape, seed, expert_src)
        wg_np = wg.float().cpu().numpy()
        rate, reps, el, thr = time_cpu_baseline(shape, seed, args.cpu_tokens, args.cpu_seconds, wcpu, wg_np,
                                                bias.numpy())
        cpu = {"value": rate, "unit": UNIT, "cores": thr, "kind": "port", **cpu_threads()[1],
               "sample": f"oracle/moe_oracle.py numpy fp32 layer forward, {shape.name} shape, {args.cpu_tokens} "
                         f"tokens x {reps} reps ({el:.1f} s), all experts local, {thr} threads"}

    tokens_total = G * T * K
    value = tokens_total / (t_ms * 1e-3)
    line = {
        "metric": METRIC,
        "value": value,
        "unit": UNIT,
        "n_gpus": G,
        "steps": K,
        "warmup": args.warmup,
        "ms_per_step": t_ms / K,
        "p50_batch_latency_ms": p50_ms,
        "higher_is_better": True,
        "scaling": "weak",
        "vs_baseline": None,
        "dtype": "bf16",
        "data": "synthetic (N(0,1) tokens, random-init expert/router weights, Dirichlet(0.3) routing skew "
                "per origin as in the reference's WorkloadSpec.synthetic)",
        "config": {"workload": f"{shape.name} MoE layer, {T} tokens/GPU, placement {solver}",
                   "model": shape.name, "d": shape.d, "ffn": shape.f, "experts": shape.E, "top_k": shape.k,
                   "shared_ffn": shape.shared_f, "tokens_per_gpu": T, "global_batch": G * T,
                   "slot_caps": caps, "parallelism": f"ep{G}+dp{G}", "k3_plan": exec_plan,
                   "l2": f"{N_ROTATE} rotating input batches ({N_ROTATE * T * shape.d * 2 / 2**20:.0f} MiB) + "
                         f"{sum(len(s) for s in sets) * shape.expert_bytes / 2**30:.2f} GiB resident expert weights "
                         "streamed per step exceed the 126 MB L2"},
        "dispatch": {
            "ours": {k: acc_ours[k] for k in ("remote_invocations", "remote_bytes", "wire_bytes", "local_ratio")},
            "uniform": {k: acc_naive[k] for k in ("remote_invocations", "remote_bytes", "wire_bytes", "local_ratio")},
            "recv_rows_per_gpu": rows_list,
            "gpus_active": int(sum(1 for r in rows_list if r > 0)),
            "k4_nvlink": k4,
        },
        "stages_ms": {name: float(v) for name, v in zip(_lib.STAGES, stage_t.tolist()) if name != "unused"},
        "host_enqueue_ms_per_step": host_enqueue_ms,
        "stage_roofline": stage_roofline(shape, T, rows_list[hot], dict(zip(_lib.STAGES, stage_t.tolist())),
                                         float(peaks.get("hbm_gbs"))),
        "side_chain_ms": side_ms,
        "stages_note": "side_chain_ms = [span of the small-group chain on the side stream, GEMM start -> its end]; "
                       "per-stage means from a diagnostic pass with events at every boundary (max over ranks); "
                       "the timed region records only the K3 boundaries",
        "roofline": {"bound": bound,
                     "kernel": ("grouped_gemm_2sm_kernel" if exec_plan["pair_routed"] else "grouped_gemm_kernel")
                               + f" (GEMM1+SwiGLU, GEMM2), rank {hot} (most routed rows)"
                               + ("; small groups on grouped_gemm_kernel over a side stream"
                                  if exec_plan["split_m"] else "")
                                                  + ("; shared expert fused into the same launches"
                                                     if exec_plan["fuse_shared"] else ""),
                     "achieved_per_rank": per_rank_tf,
                     **({"achieved": achieved_tflops, "peak": peak, "unit": "TFLOP/s",
                         "frac": achieved_tflops / peak if peak else None, "peak_regime": peak_regime,
                         "peak_burst": peak_burst, "frac_burst": achieved_tflops / peak_burst,
                         "peak_sustained": peak_sus, "frac_sustained": achieved_tflops / peak_sus}
                        if bound == "tensor" else
                        {"achieved": w_gbs, "peak": hbm_peak, "unit": "GB/s",
                         "frac": w_gbs / hbm_peak if w_gbs else None,
                         "tensor_view": {"achieved": achieved_tflops, "peak": peak, "unit": "TFLOP/s"}}),
                     "traffic": traffic,
                     "peak_source": f"{peaks_src}: bf16_tflops (burst, best of 10 8192^3 matmuls) or "
                                    "bf16_tflops_sustained (4 s back to back, power-capped), chosen by the "
                                    "SM clock sampled in the timed region (peak_regime)",
                     "flops_per_step": flops,
                     "weights": {"bytes_per_step": w_bytes, "GB/s": w_gbs, "peak_GB/s": hbm_peak,
                                 "frac": w_gbs / hbm_peak if w_gbs else None,
                                 "note": "active expert slots' weights streamed by the same K3 launches; "
                                         "'bound' is hbm when flops/weight-bytes is below the ridge "
                                         f"({ridge:.0f} flop/B)"}},
        "cpu_baseline": cpu,
        "e2e": {"value": tokens_total / (e2e_ms * 1e-3), "unit": UNIT,
                "h2d_bytes_per_step": T * shape.d * 2, "d2h_bytes_per_step": T * shape.d * 2,
                "path": "HostPipeline over B200MoELayer.forward (C ABI mp_layer_forward): pinned host x -> device "
                        "and out -> host every step, copies overlapped with the neighbouring batches' compute"},
        "gpu_launches": launches,
        "clocks": clocks,
    }
    print(json.dumps(line), flush=True)
    if args.stages:
        for name, v in zip(_lib.STAGES, stage_mean):
            sys.stderr.write(f"{name:18s} {v * 1e3:9.1f} us\n")
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()
    layer.close()


# ----------------------------------------------------------------------------- reference arm
def time_reference_package(shape, G: int, seed: int, budget_s: float = 8.0) -> dict | None:
    """The reference package's own hot-path Python, single-threaded as written (BASELINE.md CPU
    plan item 2): `sim.run` on a synthetic workload of this shape over G servers (its
    `_dispatch_layer` invocations/s, sim.py:441-463 -- analytic comm/comp, no layer arithmetic),
    `stats_from_requests` (sim.py:194-205 -> ActivationStats.ingest, stats.py:82-96) and
    `build_placement("ours")` (placement.py:541-566)."""
    from paper_2508_12851_b200.errors import import_moeplace
    from paper_2508_12851_b200.shapes import cluster_spec, model_spec, slot_caps
    mp = import_moeplace()
    if mp is None:
        return None
    import moeplace.sim as msim
    Gs = max(G, 3 if shape.E == 8 and shape.d == 512 else 2)
    cluster = cluster_spec(shape, Gs, slot_caps(shape, Gs))
    model = model_spec(shape)
    tm = mp.TimeModel.from_cluster(cluster)
    policy = msim.SchedulerPolicy(migration_enabled=False)
    n_req = 200
    while True:
        wl = msim.WorkloadSpec.synthetic(Gs, 0.05, n_req, tokens=64, seed=seed)
        reqs = msim.generate_workload(wl, model)
        t0 = time.perf_counter()
        stats = msim.stats_from_requests(reqs, model, Gs)
        t_stats = time.perf_counter() - t0
        t0 = time.perf_counter()
        placement = mp.build_placement("ours", cluster, model, stats, seed)
        t_place = time.perf_counter() - t0
        t0 = time.perf_counter()
        m = msim.run(cluster, model, "ours", reqs, tm, policy, initial_stats=stats, seed=seed)
        t_run = time.perf_counter() - t0
        if t_run >= budget_s / 4 or n_req >= 20000:
            break
        n_req = min(20000, int(n_req * max(2.0, budget_s / 4 / max(t_run, 1e-3))))
    inv = len(reqs) * model.num_layers * model.top_k
    toks = sum(int(r.tokens) for r in reqs)
    del placement, m
    return {"what": "reference moeplace package, 1 thread as written: sim.run (analytic comm/comp -- it "
                    "simulates the layer, no arithmetic), stats_from_requests, build_placement('ours')",
            "servers": Gs, "requests": len(reqs), "tokens_per_request": 64,
            "sim_run_s": t_run, "sim_invocations_per_s": inv / t_run, "sim_tokens_per_s": toks / t_run,
            "stats_from_requests_ms": t_stats * 1e3, "build_placement_ms": t_place * 1e3}


def main_reference(args):
    """The reference's CPU path for this workload: the oracle port (the reference itself has no
    layer arithmetic -- SPEC.md:8 -- so its CPU implementation is the restatement in oracle/)."""
    rank, local, world = dist_env()
    if rank != 0:
        return
    import torch
    from oracle import moe_oracle as orc
    from paper_2508_12851_b200.shapes import get_shape

    shape = get_shape(args.config)
    seed = args.seed
    threads, cinfo = cpu_threads()
    T_cpu = args.cpu_tokens
    oshape = orc.LayerShape(shape.name, shape.d, shape.f, shape.E, shape.k, shape.score_mode, shape.renorm,
                            shape.shared_f, shape.shared_gate)
    # weights: only experts the sample can reach are materialised lazily
    wg = orc.synthetic_router(shape.E + shape.shared_gate, shape.d, seed)
    bias = orc.origin_bias(0, shape.E, seed)
    x = orc.synthetic_tokens(0, T_cpu, shape.d, seed)
    idx, _ = orc.topk_route(orc.router_logits(x, wg, bias), shape.E, shape.k, shape.score_mode)
    experts = {int(e): orc.synthetic_expert(int(e), shape.d, shape.f, seed) for e in np.unique(idx)}
    shared = orc.synthetic_expert(999, shape.d, shape.shared_f, seed) if shape.shared_f else None
    route = np.zeros((1, shape.E), dtype=np.int32)
    wsg = wg[shape.E] if shape.shared_gate else None

    def step():
        orc.moe_layer_forward(oshape, [x], wg[:shape.E], [bias], route, experts, shared, wsg)

    # bound the whole run to ~2 minutes: shrink the per-step sample if one step is slow
    t0 = time.perf_counter()
    step()
    one = time.perf_counter() - t0
    budget = 120.0 / max(1, args.steps + args.warmup)
    if one > budget:
        T_cpu = max(8, int(T_cpu * budget / one))
        x = x[:T_cpu]
    for _ in range(args.warmup):
        step()
    t0 = time.perf_counter()
    for _ in range(args.steps):
        step()
    el = time.perf_counter() - t0
    value = args.steps * T_cpu / el
    try:
        ref_pkg = time_reference_package(shape, max(1, args.gpus), seed)
    except Exception as ex:  # reported, never fatal for the arm
        ref_pkg = {"error": repr(ex)}
    line = {
        "impl": "reference",
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": args.gpus, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": el / args.steps * 1e3, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "f32", "data": "synthetic",
        "config": {"workload": f"{shape.name} MoE layer on the host CPU, {T_cpu} tokens per step (bounded sample)",
                   "model": shape.name, "tokens_per_step": T_cpu},
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": threads, "kind": "port", **cinfo,
                         "sample": f"oracle/moe_oracle.py numpy fp32, {T_cpu} tokens/step x {args.steps} steps"},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "reference_package": ref_pkg,
    }
    print(json.dumps(line), flush=True)


# ----------------------------------------------------------------------------- workload-shift scenario
def main_shift(args):
    """BASELINE config 5: routing drifts (p -> roll(p, E/2), as the reference acceptance suite's
    drift, tests/test_acceptance.py:67-68); the migration check mirrors `_migration_check`
    (sim.py:465-481): window stats -> build_placement -> should_migrate (cost.py:217-248) with a
    measured remote penalty and measured peer-copy bandwidth; an adopted plan executes as NVLink
    peer copies on a side stream while traffic keeps the old placement, then routes swap
    (migration_complete, sim.py:520-525).  Reports phase throughput and local ratio for the
    static control and the migrated placement."""
    import torch
    import torch.distributed as dist
    from paper_2508_12851_b200 import workload as wl
    from paper_2508_12851_b200.errors import import_moeplace
    from paper_2508_12851_b200.layer import B200MoELayer
    from paper_2508_12851_b200.routing import dispatch_accounting, gpu_expert_sets
    from paper_2508_12851_b200.shapes import cluster_spec, get_shape, model_spec, slot_caps

    rank, local, world = dist_env()
    if world < 2:
        raise SystemExit("the shift scenario needs >= 2 GPUs (with one GPU nothing is remote)")
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    init_dist_quiet(dev)
    mp = import_moeplace()
    if mp is None:
        raise SystemExit("the shift scenario needs the reference solver (moeplace)")
    shape = get_shape(args.config)
    T, G, seed, E = args.tokens, world, args.seed, shape.E
    caps = slot_caps(shape, G)
    cluster0 = cluster_spec(shape, G, caps)
    model = model_spec(shape)
    wg = wl.router_weights(E + shape.shared_gate, shape.d, dev, seed)
    expert_src = lambda e: wl.expert_weights(e, shape.d, shape.f, dev, seed)
    layer = B200MoELayer(shape, rank=rank, world=world, device=local, max_tokens=T, cap_slots=caps[rank])
    layer.open_peers()
    if shape.shared_f:
        layer.set_shared(*wl.shared_weights(shape.d, shape.shared_f, dev, seed))
    xs = [wl.tokens(T, shape.d, dev, seed, rank, batch=b) for b in range(N_ROTATE)]
    out = torch.empty(T, shape.d, device=dev, dtype=torch.bfloat16)
    stream = torch.cuda.current_stream()

    def all_counts():
        return layer.gathered_counts()

    def set_phase(shift):
        layer.set_router(wg[:E], wl.origin_bias(rank, E, seed, shift=shift), wg[E] if shape.shared_gate else None)

    def run(steps):
        """steps forwards; returns (tokens/s over all GPUs, max-over-ranks seconds)"""
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(stream)
        for i in range(steps):
            layer.forward(xs[i % N_ROTATE], out)
        b.record(stream)
        torch.cuda.synchronize()
        ms = torch.tensor([a.elapsed_time(b)], dtype=torch.float64, device=dev)
        if world > 1:
            dist.all_reduce(ms, op=dist.ReduceOp.MAX)
        layer.check()
        return G * T * steps / (ms.item() * 1e-3), ms.item() * 1e-3

    def placement_from(counts):
        stats = mp.ActivationStats.from_counts(np.asarray(counts, float)[:, None, :], (E,))
        return mp.build_placement("ours", cluster0, model, stats, seed), stats

    # ---- phase A: placement fit to phase-A traffic (warm-up histogram)
    set_phase(0)
    # warm-up counts with a provisional all-covering placement (uniform round robin)
    prov = [[e for e in range(E) if e % G == r] for r in range(G)]
    layer.set_placement_sets(prov, expert_src)
    layer.reset_counts()
    run(args.warmup)
    pa, _ = placement_from(all_counts())
    sets_a = gpu_expert_sets(pa, 0)
    layer.set_placement_sets(sets_a, expert_src)
    layer.reset_counts()
    tps_a, _ = run(args.steps)
    acc_a = dispatch_accounting(all_counts(), layer.route, shape.d)

    # ---- phase B with the static placement (the control): drifted routing
    set_phase(E // 2)
    layer.reset_counts()
    tps_b_static, win_s = run(args.steps)
    acc_b_static = dispatch_accounting(all_counts(), layer.route, shape.d)

    # ---- migration check (sim.py:465-481) with measured costs
    # remote penalty per token-unit: wire time of one remote invocation (activations out, results
    # back, comm_time's bandwidth term cost.py:148) at the measured peer bandwidth (probe copy below)
    bw_probe = measure_peer_copy(layer, world, rank) if world > 1 else 770e9
    from paper_2508_12851_b200.calibrate import observed_remote_penalty, remote_penalty_seconds
    # observed per-invocation penalty (sim.py:455-456, 469): the step-time difference of phase A
    # and static phase B (same batch size, placement A) over their remote-invocation difference
    penalty_analytic = remote_penalty_seconds(shape.d, bw_probe)
    per_step = lambda tps: G * T / tps
    penalty = observed_remote_penalty(per_step(tps_a), acc_a["remote_invocations"] / args.steps,
                                      per_step(tps_b_static), acc_b_static["remote_invocations"] / args.steps)
    if penalty <= 0.0:
        penalty = penalty_analytic
    cluster = cluster_spec(shape, G, caps, link_bandwidth=bw_probe, load_bandwidth=bw_probe)
    from paper_2508_12851_b200.controller import MigrationController
    ctl = MigrationController(layer, cluster, model, pa, strategy="ours", seed=seed, mode="loads-only",
                              penalty_seconds=penalty)
    adopt, ledger, candidate = ctl.check(win_s)      # window = the static phase-B run
    mig = {"decision": ledger["decision"], "cost_current_seconds": ledger["cost_current_seconds"],
           "cost_candidate_seconds": ledger["cost_candidate_seconds"],
           "migration_seconds_model": ledger["migration_seconds"], "penalty_seconds_per_token": penalty,
           "penalty_source": "observed: (step_B_static - step_A) / (remote_B - remote_A) per step",
           "penalty_analytic_2dbpe_over_bw": penalty_analytic,
           "peer_copy_GBps": bw_probe / 1e9}
    tps_b_mig, acc_b_mig = None, None
    if adopt:
        # traffic keeps flowing on the old placement while the weights move (a fixed number of
        # forwards on every rank: the layer is SPMD across GPUs)
        def overlap():
            for i in range(3):
                layer.forward(xs[i % N_ROTATE], out)
            return 3
        mig.update(ctl.migrate(candidate, torch.cuda.Stream(dev), overlap))
        tps_b_mig, _ = run(args.steps)
        acc_b_mig = dispatch_accounting(all_counts(), layer.route, shape.d)

    # ---- parity of the forward on the final placement (after the migration when adopted): 32
    # tokens per rank against the fp32 restatement of the layer math (tests/torch_ref.py) under
    # the stated tolerance (tests/tolerance.py), routing taken from the layer's own router
    chk = torch.empty_like(out)
    layer.forward(xs[0], chk)
    torch.cuda.synchronize()
    sys.path.insert(0, str(REPO / "tests"))
    from tolerance import check_layer_close
    from torch_ref import layer_reference
    n_chk = min(32, T)
    shared_w = wl.shared_weights(shape.d, shape.shared_f, dev, seed) if shape.shared_f else None
    gate = layer.shared_gate[:n_chk] if shape.shared_gate else None
    ref, mag, mag2 = layer_reference(xs[0][:n_chk], layer.idx[:n_chk], layer.gate_w[:n_chk], expert_src, shared_w, gate)
    try:
        st = check_layer_close(chk[:n_chk].float().cpu().numpy(), ref.cpu().numpy(), mag.cpu().numpy(),
                               mag2.cpu().numpy(), "post-migration forward")
        used, ok = st["max_err_over_bound"], 1.0
    except AssertionError:
        used, ok = float("inf"), 0.0
    pv = torch.tensor([used if used != float("inf") else 1e30, -ok], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(pv, op=dist.ReduceOp.MAX)
    parity = {"tokens_per_rank": n_chk, "placement": "migrated" if tps_b_mig is not None else "static",
              "max_err_over_bound": pv[0].item(), "ok": pv[1].item() == -1.0,
              "reference": "fp32 restatement (tests/torch_ref.py), bound of tests/tolerance.py"}

    if rank == 0:
        keep = ("remote_invocations", "remote_bytes", "local_ratio")
        line = {"scenario": "workload-shift (BASELINE config 5)", "metric": METRIC, "unit": UNIT, "n_gpus": G,
                "config": {"model": shape.name, "tokens_per_gpu": T, "steps_per_phase": args.steps,
                           "slot_caps": caps, "drift": f"p -> roll(p, {E // 2})"},
                "phase_a": {"value": tps_a, **{k: acc_a[k] for k in keep}},
                "phase_b_static": {"value": tps_b_static, **{k: acc_b_static[k] for k in keep}},
                "migration": mig,
                "phase_b_migrated": None if tps_b_mig is None else
                {"value": tps_b_mig, **{k: acc_b_mig[k] for k in keep}},
                "parity": parity}
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()
    layer.close()


def main_stack(args):
    """F3: an L-layer MoEStack (ModelSpec.num_layers > 1, the reference walks a request through
    its layers in order, sim.py:500-505), each layer with its own router, expert weights and
    placement, run eagerly and as one captured CUDA graph (device-side flag epochs and count
    parity make the forward replayable).  Reports tokens/s through the whole stack both ways."""
    import torch
    import torch.distributed as dist
    from paper_2508_12851_b200 import workload as wl
    from paper_2508_12851_b200.layer import B200MoELayer, MoEStack
    from paper_2508_12851_b200.shapes import get_shape

    rank, local, world = dist_env()
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        init_dist_quiet(dev)
    shape = get_shape(args.config)
    T, G, L = args.tokens, world, args.layers
    layers = []
    for l in range(L):
        seed = args.seed + 101 * l
        wg = wl.router_weights(shape.E + shape.shared_gate, shape.d, dev, seed)
        src = (lambda s: lambda e: wl.expert_weights(e, shape.d, shape.f, dev, s, layer=l))(seed)
        # placement of layer l: the reference solver on this layer's warm-up histogram
        prov = [[e for e in range(shape.E) if e % G == r] for r in range(G)]
        caps = [max(len(p) for p in prov)] * G if G > 1 else [shape.E]
        probe = B200MoELayer(shape, rank=rank, world=world, device=local, max_tokens=T,
                             cap_slots=max(caps[rank], max(len(p) for p in prov)))
        probe.open_peers()
        probe.set_router(wg[:shape.E], wl.origin_bias(rank, shape.E, seed), wg[shape.E] if shape.shared_gate else None)
        if shape.shared_f:
            probe.set_shared(*wl.shared_weights(shape.d, shape.shared_f, dev, seed, layer=l))
        probe.set_placement_sets(prov, src)
        probe.forward(wl.tokens(T, shape.d, dev, seed, rank, batch=10_000))
        torch.cuda.synchronize()
        counts = probe.gathered_counts()
        probe.close()
        sets, caps, _ = build_placement_sets(shape, G, counts, args.strategy, seed)
        layer = B200MoELayer(shape, rank=rank, world=world, device=local, max_tokens=T, cap_slots=caps[rank])
        layer.open_peers()
        layer.set_router(wg[:shape.E], wl.origin_bias(rank, shape.E, seed), wg[shape.E] if shape.shared_gate else None)
        if shape.shared_f:
            layer.set_shared(*wl.shared_weights(shape.d, shape.shared_f, dev, seed, layer=l))
        layer.set_placement_sets(sets, src)
        layers.append(layer)
    stack = MoEStack(layers)
    x = wl.tokens(T, shape.d, dev, args.seed, rank, batch=0)
    out = torch.empty_like(x)
    stream = torch.cuda.current_stream()

    def timed(fn, steps):
        for _ in range(args.warmup):
            fn()
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(stream)
        for _ in range(steps):
            fn()
        b.record(stream)
        torch.cuda.synchronize()
        ms = torch.tensor([a.elapsed_time(b) / steps], dtype=torch.float64, device=dev)
        if world > 1:
            dist.all_reduce(ms, op=dist.ReduceOp.MAX)
        return ms.item()

    eager_ms = timed(lambda: stack.forward(x, out), args.steps)
    eager_out = out.clone()
    graph = stack.capture(x, out)
    graph_ms = timed(graph.replay, args.steps)
    torch.cuda.synchronize()
    for layer in layers:
        layer.check()
    same = bool(torch.equal(out, eager_out))
    launches = sum(layer.last_launches() for layer in layers)
    if rank == 0:
        line = {"scenario": "multi-layer stack (F3)", "metric": METRIC, "unit": UNIT, "n_gpus": G,
                "config": {"model": shape.name, "layers": L, "tokens_per_gpu": T, "steps": args.steps},
                "eager": {"value": G * T / (eager_ms * 1e-3), "ms_per_stack_forward": eager_ms},
                "cuda_graph": {"value": G * T / (graph_ms * 1e-3), "ms_per_stack_forward": graph_ms},
                "graph_output_equals_eager": same, "kernel_launches_per_stack_forward": launches}
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()
    del graph
    for layer in layers:
        layer.close()


def main_transport(args):
    """K4 A/B (north star (4)): the same layer, placement and inputs run through the
    fused NVLink transport (B200MoELayer.forward: peer stores inside the permute kernel and the
    GEMM2 epilogue, flag protocol inside the kernels) and through the NCCL all-to-all-v transport
    (nccl_path.NcclForward: the same kernels as stages, NCCL send/recv of every (source, expert)
    chunk, one host sync for the chunk sizes).  Reports tokens/s of both (max over ranks), the
    NCCL dispatch / return wire rates, and the measured peer-copy bandwidth."""
    from paper_2508_12851_b200.nccl_path import NcclForward
    b = setup_bench_layer(args)
    torch, dist = b.torch, b.dist
    layer, xs, out, stream, G, T, rank, dev = b.layer, b.xs, b.out, b.stream, b.G, b.T, b.rank, b.dev

    def timed(fn, steps):
        for i in range(args.warmup):
            fn(xs[i % N_ROTATE])
        torch.cuda.synchronize()
        b.barrier()
        a, z = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(stream)
        for i in range(steps):
            fn(xs[i % N_ROTATE])
        z.record(stream)
        torch.cuda.synchronize()
        b.barrier()
        ms = torch.tensor([a.elapsed_time(z)], dtype=torch.float64, device=dev)
        if G > 1:
            dist.all_reduce(ms, op=dist.ReduceOp.MAX)
        return ms.item()

    fused_ms = timed(lambda x: layer.forward(x, out), args.steps)
    fused_out = out.clone()
    layer.check()
    nf = NcclForward(layer, group=None)
    nccl_ms = timed(lambda x: nf.forward(x, out), args.steps)
    same = bool(torch.equal(out, fused_out))
    nf.timing = True
    for i in range(min(args.steps, 20)):
        nf.forward(xs[i % N_ROTATE], out)
    st_ms = nf.stage_ms()
    vals = torch.tensor([st_ms.get(k, 0.0) for k in NcclForward.STAGES] +
                        [nf.last["dispatch_bytes"], nf.last["return_bytes"]], dtype=torch.float64, device=dev)
    parts = [torch.zeros_like(vals) for _ in range(G)]
    if G > 1:
        dist.all_gather(parts, vals)
    else:
        parts = [vals]
    per_rank = [p.tolist() for p in parts]
    peer_bw = measure_peer_copy(layer, G, rank) if G > 1 else None
    if rank == 0:
        ns = len(NcclForward.STAGES)
        disp = [p[ns] / (p[2] * 1e-3) / 1e9 if p[2] > 0 else None for p in per_rank]
        retr = [p[ns + 1] / (p[4] * 1e-3) / 1e9 if p[4] > 0 else None for p in per_rank]
        line = {"scenario": "transport A/B (K4: fused NVLink peer stores vs NCCL all-to-all-v)", "metric": METRIC,
                "unit": UNIT, "n_gpus": G, "steps": args.steps,
                "config": {"model": b.shape.name, "tokens_per_gpu": T, "placement": b.solver, "slot_caps": b.caps},
                "fused": {"value": G * T * args.steps / (fused_ms * 1e-3), "ms_per_step": fused_ms / args.steps},
                "nccl": {"value": G * T * args.steps / (nccl_ms * 1e-3), "ms_per_step": nccl_ms / args.steps,
                         "stages_ms_per_rank": [dict(zip(NcclForward.STAGES, p[:ns])) for p in per_rank],
                         "dispatch_bytes_per_rank": [int(p[ns]) for p in per_rank],
                         "return_bytes_per_rank": [int(p[ns + 1]) for p in per_rank],
                         "dispatch_GBps_per_rank": disp, "return_GBps_per_rank": retr},
                "fused_over_nccl": nccl_ms / fused_ms, "outputs_bit_identical": same,
                "peer_copy_GBps": peer_bw / 1e9 if peer_bw else None, "nvlink_peak_GBps": 770.0,
                "decision": "fused" if fused_ms <= nccl_ms else "nccl"}
        print(json.dumps(line), flush=True)
    if G > 1:
        dist.barrier()
        dist.destroy_process_group()
    layer.close()


def measure_peer_latency(layer, rank, world, reps: int = 200) -> float:
    """Seconds per small (4 KB) NVLink copy from the next GPU's window (mp_layer_peer_probe) --
    the link latency term of comm_time (cost.py:139-149); max over ranks."""
    import torch
    import torch.distributed as dist
    dist.barrier()
    lat = layer.peer_probe((rank + 1) % world, 4096, reps)
    t = torch.tensor([lat], dtype=torch.float64, device=layer.device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    dist.barrier()
    return float(t.item())


def main_calibrate(args):
    """F1: measured-cost feedback into the reference's decision layer.  The analytic TimeModel
    (cost.py:39-85: comp_base 2 ms, comp_per_token 50 us, link matrices) and the remote penalty of
    CostSnapshot (cost.py:195-214, accumulated per remote invocation at sim.py:455-456, 469) get
    their numbers from this box: a batch-size sweep of the expert GEMMs (K3 time vs routed rows per
    GPU, least squares per GPU), the measured NVLink peer-copy bandwidth and small-copy latency, and
    the observed penalty (step time of the same batch under the uniform vs the activation-aware
    placement over their remote-invocation difference).  The reference's layer model
    (`layer_latency`, cost.py:152-168) then predicts the measured forward."""
    import numpy as np
    from paper_2508_12851_b200 import calibrate as cal
    from paper_2508_12851_b200.errors import import_moeplace
    from paper_2508_12851_b200.routing import dispatch_accounting
    from paper_2508_12851_b200.shapes import cluster_spec, model_spec
    b = setup_bench_layer(args)
    torch, dist, _lib = b.torch, b.dist, b._lib
    layer, xs, out, stream, G, T, rank, dev, shape = b.layer, b.xs, b.out, b.stream, b.G, b.T, b.rank, b.dev, b.shape
    mp = import_moeplace()
    NS = _lib.NUM_STAGE_EVENTS

    def run(Tn, steps):
        """(mean step ms max over ranks, this GPU's mean K3 ms, rows this GPU computed, counts)"""
        evs = []
        for _ in range(steps):
            row = [torch.cuda.Event(enable_timing=True) if j in (0, _lib.GEMM_START, _lib.GEMM_END,
                                                                  _lib.MAIN_STAGE_EVENTS - 1) else None
                   for j in range(NS)]
            for ev in row:
                if ev is not None:
                    ev.record(stream)
            evs.append(row)
        for i in range(args.warmup):
            layer.forward(xs[i % N_ROTATE][:Tn], out[:Tn])
        torch.cuda.synchronize()
        b.barrier()
        for i in range(steps):
            layer.forward(xs[i % N_ROTATE][:Tn], out[:Tn], events=evs[i])
        torch.cuda.synchronize()
        b.barrier()
        layer.check()
        step = float(np.median([e[0].elapsed_time(e[_lib.MAIN_STAGE_EVENTS - 1]) for e in evs]))
        k3 = float(np.mean([e[_lib.GEMM_START].elapsed_time(e[_lib.GEMM_END]) for e in evs]))
        st = torch.tensor([step], dtype=torch.float64, device=dev)
        if G > 1:
            dist.all_reduce(st, op=dist.ReduceOp.MAX)
        counts = layer.read_counts()
        rows = int(sum(counts[s, e] for s in range(G) for e in range(shape.E) if layer.route[s, e] == rank))
        return st.item(), k3, rows, counts

    sweep = sorted({max(256, T // 8), max(256, T // 4), max(256, T // 2), T})
    samples = []
    for Tn in sweep:
        step_ms, k3_ms, rows, counts = run(Tn, args.steps)
        samples.append((rows, k3_ms * 1e-3))
    allsamp = [None] * G
    if G > 1:
        dist.all_gather_object(allsamp, samples)
    else:
        allsamp = [samples]
    step_ours, _, _, counts_ours = run(T, args.steps)
    acc_ours = dispatch_accounting(counts_ours, layer.route, shape.d)
    penalty, step_uni, acc_uni = None, None, None
    bw, lat = 770e9, 3e-6
    if G > 1:
        bw = measure_peer_copy(layer, G, rank)
        lat = measure_peer_latency(layer, rank, G)
        uni = uniform_sets(shape, G)
        if all(len(uni[g]) <= layer.cap_slots for g in range(G)):
            layer.set_placement_sets(uni, b.expert_src)
            step_uni, _, _, counts_uni = run(T, args.steps)
            acc_uni = dispatch_accounting(counts_uni, layer.route, shape.d)
            penalty = cal.observed_remote_penalty(step_ours * 1e-3, acc_ours["remote_invocations"],
                                                  step_uni * 1e-3, acc_uni["remote_invocations"])
            layer.set_placement_sets(b.sets, b.expert_src)
    pred = None
    if rank == 0 and mp is not None:
        cluster = cluster_spec(shape, G, b.caps, link_bandwidth=bw, link_latency=lat, load_bandwidth=bw)
        model = model_spec(shape)
        tm = cal.calibrated_time_model(cluster, allsamp, link_bandwidth=bw, link_latency=lat)
        placement = mp.placement_from_server_sets([[s] for s in b.sets], cluster, model)
        pred = cal.predicted_layer_latency(tm, placement, model, counts_ours, layer.route)
        default_tm = mp.TimeModel.from_cluster(cluster)
        pred_default = cal.predicted_layer_latency(default_tm, placement, model, counts_ours, layer.route)
        line = {"scenario": "calibration (F1: measured TimeModel / CostSnapshot inputs)", "n_gpus": G,
                "config": {"model": shape.name, "tokens_per_gpu": T, "sweep_tokens": sweep, "steps": args.steps},
                "comp_fit": {"comp_base_s": tm.comp_base.tolist(), "comp_per_token_s": tm.comp_per_token.tolist(),
                             "samples_rows_seconds": allsamp},
                "link": {"peer_copy_GBps": bw / 1e9, "small_copy_latency_s": lat},
                "penalty": {"observed_s_per_remote_invocation": penalty,
                            "analytic_2dbpe_over_bw_s": cal.remote_penalty_seconds(shape.d, bw),
                            "step_ms_ours": step_ours, "step_ms_uniform": step_uni,
                            "remote_invocations_ours": acc_ours["remote_invocations"],
                            "remote_invocations_uniform": acc_uni["remote_invocations"] if acc_uni else None},
                "measured_step_ms": step_ours,
                "predicted_calibrated": {k: (v * 1e3 if k.endswith("_s") else v) for k, v in pred.items()},
                "predicted_reference_defaults": {k: (v * 1e3 if k.endswith("_s") else v)
                                                 for k, v in pred_default.items()},
                "units": "predicted_* latencies in ms (reference layer_latency, cost.py:152-168)"}
        print(json.dumps(line), flush=True)
    if G > 1:
        dist.barrier()
        dist.destroy_process_group()
    layer.close()


def measure_peer_copy(layer, world, rank):
    """NVLink pull bandwidth from the next GPU's window (mp_layer_peer_probe, up to 64 MiB per
    copy); min over ranks."""
    import torch
    import torch.distributed as dist
    dist.barrier()
    cap = int(layer._ptrs.recv_cap) * layer.shape.d * 2
    nbytes = min(cap, 64 << 20)
    sec = layer.peer_probe((rank + 1) % world, nbytes, 5)
    bw = torch.tensor([nbytes / sec], dtype=torch.float64, device=layer.device)
    dist.all_reduce(bw, op=dist.ReduceOp.MIN)
    dist.barrier()
    return float(bw.item())


def self_launch(args) -> int:
    """`python bench.py --gpus N` without a torchrun environment: re-exec this script under
    torch.distributed.run with one process per GPU (127.0.0.1 rendezvous); rank 0's single JSON
    line comes through on stdout."""
    import socket
    sock = socket.socket()
    sock.bind(("127.0.0.1", 0))
    port = sock.getsockname()[1]
    sock.close()
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr", "127.0.0.1", "--master-port", str(port), str(Path(__file__).resolve()), *sys.argv[1:]]
    env = dict(os.environ, OMP_NUM_THREADS=os.environ.get("OMP_NUM_THREADS", "1"))
    return subprocess.run(cmd, env=env).returncode


if __name__ == "__main__":
    a = parse()
    if a.gpus > 1 and "WORLD_SIZE" not in os.environ and a.impl != "reference":
        raise SystemExit(self_launch(a))
    if a.scenario == "shift" and a.impl != "reference":
        main_shift(a)
        raise SystemExit(0)
    if a.scenario == "stack" and a.impl != "reference":
        main_stack(a)
        raise SystemExit(0)
    if a.scenario == "transport" and a.impl != "reference":
        main_transport(a)
        raise SystemExit(0)
    if a.scenario == "calibrate" and a.impl != "reference":
        main_calibrate(a)
        raise SystemExit(0)
    if a.impl == "reference":
        # keep the whole --steps K run within minutes: clamp the sample size for the big shapes
        main_reference(a)
    else:
        main_b200(a)
