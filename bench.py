#!/usr/bin/env python
"""Benchmark of the dense view-synthesis hot path (BASELINE.json metric:
synthesized virtual views/s at 1080p; per-rig-frame latency).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config cfg4] [--impl b200|reference]

One step = a batch of F independent rig frames of the live stream per rank
(--frames-in-flight, default auto = 6 / 3 / 1, the most that fit a quarter of HBM; F > 1 run concurrently on forked streams inside one
CUDA graph): every dense view of every camera gap (recursive midpoints,
server/pipeline.py:254-271) plus every cluster frame (server/pipeline.py:273-292).
The per-rig-frame latency (one frame in flight) is measured separately and
reported as config.rig_frame_latency_ms.  Default workload = BASELINE config 4 (8-camera
1080p YUV420 rig, 7 gaps x 15 views = 105 views, 8 cluster frames), which
fits one B200.  Multi-GPU: one process per GPU (torchrun), each rank owns
its own rig frames (frame sharding, weak scaling) and the cluster frames are
gathered to the encoder-feeding rank 0 with NCCL send/recv.

`--impl reference` times the reference algorithm's CPU implementation (the
oracle port in oracle/, all host threads) on a bounded sample of the same
workload: each step = one interpolate() at the config's resolution.
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

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

CONFIGS = {
    "cfg1": dict(desc="single camera pair 256x448 RGB, 1 midpoint virtual view", W=448, H=256, fmt=2,
                 cams=2, stages=1, vps=0),
    "cfg2": dict(desc="single camera pair 1920x1080, 7 dense intermediate views per pair", W=1920, H=1080,
                 fmt=1, cams=2, stages=3, vps=0),
    "cfg3": dict(desc="4-camera linear rig 1920x1080, 3 pairs x 15 intermediate views, tiled output frame",
                 W=1920, H=1080, fmt=1, cams=4, stages=4, vps=16),
    "cfg4": dict(desc="8-camera arc rig 1920x1080, 7 pairs x 15 views, pairs sharded across B200s",
                 W=1920, H=1080, fmt=1, cams=8, stages=4, vps=16),
    "cfg5": dict(desc="16-camera rig 3840x2160, 15 pairs x 31 views, batched multi-frame live stream",
                 W=3840, H=2160, fmt=1, cams=16, stages=5, vps=32),
}
FMT_NAME = {0: "gray8", 1: "yuv420", 2: "rgb8"}
METRIC = "synthesized virtual views/sec at 1080p"


# ---------------------------------------------------------------------------
# synthetic multi-view input (deterministic parallax scene, numpy)
# ---------------------------------------------------------------------------
def _texture(rng, h, w):
    from scipy.ndimage import gaussian_filter
    t = gaussian_filter(rng.random((h, w)), 6.0) * 0.6 + gaussian_filter(rng.random((h, w)), 1.5) * 0.4
    t = (t - t.min()) / (np.ptp(t) + 1e-12)
    return 28.0 + 190.0 * t


def synth_rig(W, H, fmt, cams, seed=42):
    """cams packed frames of a planar-parallax scene: far background plus two
    near sprites, disparities growing with camera index."""
    rng = np.random.default_rng(seed)
    d_bg, d_sp = max(1, round(1.5 * W / 640)), [round(6 * W / 640), round(4 * W / 640)]
    pad = (cams + 1) * max(d_sp) + 8
    bg = _texture(rng, H, W + pad)
    sprites = []
    for k, d in enumerate(d_sp):
        sh, sw = H // (3 + k), W // (5 + k)
        sprites.append((_texture(rng, sh, sw) * 0.8 + 30, d, H // 4 + k * H // 3, W // 4 + k * W // 3))
    frames = []
    for c in range(cams):
        y = bg[:, c * d_bg:c * d_bg + W].copy()
        for tex, d, top, left in sprites:
            x0 = left - c * d
            sh, sw = tex.shape
            xs, xe = max(0, x0), min(W, x0 + sw)
            if xe > xs:
                y[top:top + sh, xs:xe] = tex[:, xs - x0:xe - x0]
        yp = np.clip(np.rint(y), 0, 255).astype(np.uint8)
        if fmt == 0:
            frames.append(yp.reshape(-1))
        elif fmt == 2:
            rgb = np.stack([yp, np.clip(yp.astype(int) + 20, 0, 255), 255 - yp], -1).astype(np.uint8)
            frames.append(rgb.reshape(-1))
        else:
            c2 = yp[::2, ::2].astype(np.int32)
            u = np.clip(128 + (c2 - 128) // 5, 0, 255).astype(np.uint8)
            v = np.clip(128 - (c2 - 128) // 6, 0, 255).astype(np.uint8)
            frames.append(np.concatenate([yp.reshape(-1), u.reshape(-1), v.reshape(-1)]))
    return np.stack(frames)


# ---------------------------------------------------------------------------
# clocks during the timed region (B200_PROFILING.md clocks line)
# ---------------------------------------------------------------------------
class ClockSampler:
    Q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")

    def __init__(self, index=0):
        self.index = index
        self.samples = []
        self.proc = None

    def start(self):
        try:
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.Q}",
                                          "--format=csv,noheader,nounits", "-lms", "50"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.thread = threading.Thread(target=self._read, daemon=True)
            self.thread.start()
        except FileNotFoundError:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            parts = [p.strip() for p in line.split(",")]
            if len(parts) == 6:
                self.samples.append(parts)

    def stop(self):
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        time.sleep(0.12)
        self.proc.terminate()
        try:
            self.proc.wait(timeout=2)
        except subprocess.TimeoutExpired:
            self.proc.kill()
        self.thread.join(timeout=2)
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        sm = [float(s[0]) for s in self.samples if s[0].replace(".", "").isdigit()]
        mx = [float(s[1]) for s in self.samples if s[1].replace(".", "").isdigit()]
        reasons = sorted({names[i] for s in self.samples for i in range(4) if s[2 + i] == "Active"})
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(self.samples)}


# ---------------------------------------------------------------------------
# algorithmic work per kernel class
# ---------------------------------------------------------------------------
def kernel_figures(cfg, npairs_total):
    """{class: (bound, unit, algorithmic amount over all launches of one step)}"""
    W, H, fmt = cfg["W"], cfg["H"], cfg["fmt"]
    bframe = {0: 1.0, 1: 1.5, 2: 3.0}[fmt] * W * H
    r = (12, 4, 2)
    lv = [(W // 4, H // 4), (W // 2, H // 2), (W, H)]
    sad = [2 * (2 * r[s] + 1) ** 2 * lv[s][0] * lv[s][1] * npairs_total for s in range(3)]
    return {
        "k_sad<0>": ("int", "Gop/s", sad[0]),
        "k_sad<1>": ("int", "Gop/s", sad[1]),
        "k_sad<2>": ("int", "Gop/s", sad[2]),
        # warp + mask + blend: 2 source frames read, 1 view written (compulsory)
        "k_mask_cols": ("hbm", "GB/s", 2 * bframe * npairs_total),
        "k_scan_carry": ("hbm", "GB/s", 2 * W * H * npairs_total),
        "k_blend": ("hbm", "GB/s", bframe * npairs_total),
        "k_warpq<2>": ("hbm", "GB/s", (2 * W * H + 2 * 2 * W * H + 16 * W * H / 4) * npairs_total),
    }


def measured_peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            return json.load(f), "measured"
    except OSError:
        return {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0, "sm_max_mhz": 1965.0}, "fallback"


# ---------------------------------------------------------------------------
# CPU reference (oracle port) -- cpu_baseline and --impl reference
# ---------------------------------------------------------------------------
def cpu_interp_rate(cfg, budget_s=10.0, min_reps=1):
    from oracle import oracle as O
    O.set_threads(os.cpu_count() or 1)
    W, H, fmt = cfg["W"], cfg["H"], cfg["fmt"]
    fr = synth_rig(W, H, fmt, 2, seed=7)
    O.interpolate(fr[0], fr[1], W, H, fmt)  # warm (first-touch, thread pool)
    n, t0 = 0, time.perf_counter()
    while n < min_reps or time.perf_counter() - t0 < budget_s:
        O.interpolate(fr[0], fr[1], W, H, fmt)
        n += 1
    dt = time.perf_counter() - t0
    return n / dt, n, dt, O.num_threads()


def run_reference(args, cfg, rank, world):
    if rank != 0:
        return 0
    from oracle import oracle as O
    O.set_threads(os.cpu_count() or 1)
    W, H, fmt = cfg["W"], cfg["H"], cfg["fmt"]
    fr = synth_rig(W, H, fmt, 2, seed=7)
    for _ in range(args.warmup):
        O.interpolate(fr[0], fr[1], W, H, fmt)
    t0 = time.perf_counter()
    for _ in range(args.steps):
        O.interpolate(fr[0], fr[1], W, H, fmt)
    dt = time.perf_counter() - t0
    rate = args.steps / dt
    sample = f"{args.steps} x interpolate() {W}x{H} {FMT_NAME[fmt]} (one view each) from {args.config}"
    line = {
        "metric": METRIC, "value": rate, "unit": "views/s", "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": dt / args.steps * 1e3, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "u8/i32/f64", "data": "synthetic",
        "impl": "reference",
        "config": {"workload": args.config, "desc": cfg["desc"], "width": W, "height": H,
                   "format": FMT_NAME[fmt], "step": "one interpolate() per step (bounded CPU sample)"},
        "cpu_baseline": {"value": rate, "unit": "views/s", "cores": O.num_threads(), "kind": "port",
                         "sample": sample},
        "e2e": {"value": rate, "unit": "views/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line))
    return 0


# ---------------------------------------------------------------------------
# B200 arm
# ---------------------------------------------------------------------------
def run_b200(args, cfg, rank, world, local_rank):
    import ctypes

    import torch
    import torch.distributed as dist
    from paper_2112_10603_b200 import _lib
    from paper_2112_10603_b200.cluster import rig_cluster_sizes, rig_clusters
    from paper_2112_10603_b200.interp import Interpolator

    torch.cuda.set_device(local_rank)
    dev = torch.device("cuda", local_rank)
    W, H, fmt, C, S, vps = cfg["W"], cfg["H"], cfg["fmt"], cfg["cams"], cfg["stages"], cfg["vps"]
    step_views = (C - 1) * ((1 << S) - 1)
    total_views = (C - 1) * (1 << S) + 1
    max_pairs = (C - 1) * (1 << (S - 1))
    npairs_total = step_views  # interpolations per rig frame
    # frames in flight: --frames-in-flight N, or 0 = auto (the largest of 6 / 3 / 1 whose rig
    # frames' engines, views and clusters take under a quarter of HBM: cfg1-4 run 6, cfg5's 48 GB
    # engines stay single; r2 v8 sweep F = 1 / 3 / 6 / 10: cfg1 7151 / 19314 / 35543 / 49381,
    # cfg2 7485 / 9337 / 10489 / 10693, cfg3 10273 / 11034 / 11253 / 11273 views/s at the same
    # per-frame latency)
    F_req = args.frames_in_flight
    F = max(1, F_req) if F_req > 0 else 6
    engines, cams_l, views_l, clusters_l, hosts = [], [], [], [], []
    i = 0
    while i < F:
        if F_req <= 0 and i == 1:
            per = engines[0].workspace_bytes + views_l[0].numel() + (clusters_l[0].numel() if vps else 0)
            quarter = 0.25 * torch.cuda.get_device_properties(dev).total_memory
            F = next(f for f in (6, 3, 1) if f == 1 or f * per <= quarter)
            if F == 1:
                break
        e = Interpolator(W, H, fmt, max_pairs=max_pairs, device=dev)
        h = torch.from_numpy(synth_rig(W, H, fmt, C, seed=42 + rank * 8 + i)).pin_memory()
        engines.append(e)
        hosts.append(h)
        cams_l.append(h.to(dev))
        views_l.append(torch.empty((total_views, e.frame_bytes), dtype=torch.uint8, device=dev))
        if vps:
            sizes = rig_cluster_sizes(W, H, fmt, C, S, vps)
            clusters_l.append(torch.empty(sum(sizes), dtype=torch.uint8, device=dev))
        i += 1
    eng, cams, views = engines[0], cams_l[0], views_l[0]
    clusters = clusters_l[0] if vps else None
    results = clusters_l if vps else views_l
    host_out = [torch.empty(r.shape, dtype=torch.uint8).pin_memory() for r in results]

    def compute_one(i):
        engines[i].rig(cams_l[i], S, views_l[i])
        if vps:
            rig_clusters(views_l[i], W, H, fmt, C, S, vps, out=clusters_l[i])

    stream = torch.cuda.Stream(device=dev)
    side = [torch.cuda.Stream(device=dev) for _ in range(F)]

    def compute_all():
        # F independent rig frames of the live stream, forked onto F streams and joined
        if F == 1:
            compute_one(0)
            return
        cur = torch.cuda.current_stream()
        fork = torch.cuda.Event()
        fork.record(cur)
        joins = []
        for i in range(F):
            side[i].wait_event(fork)
            with torch.cuda.stream(side[i]):
                compute_one(i)
                ev = torch.cuda.Event()
                ev.record(side[i])
                joins.append(ev)
        for ev in joins:
            cur.wait_event(ev)

    from paper_2112_10603_b200.shard import gather_to_root
    gather_bufs = [[torch.empty_like(r) for _ in range(world - 1)] for r in results] \
        if world > 1 and rank == 0 else None

    def gather():
        # cluster frames of every rank -> the encoder-feeding rank 0 (NCCL over NVLink)
        if world > 1:
            for i, r in enumerate(results):
                gather_to_root(r, rank, world, out=gather_bufs[i] if gather_bufs else None)

    torch.cuda.synchronize()
    # capture the step (F rig frames) and a single rig frame as CUDA graphs
    graph = graph1 = None
    if not args.no_graph:
        with torch.cuda.stream(stream):
            compute_all()  # first run outside capture (lazy attributes, allocator)
        torch.cuda.synchronize()
        graph = torch.cuda.CUDAGraph()
        with torch.cuda.graph(graph, stream=stream):
            compute_all()
        graph1 = torch.cuda.CUDAGraph()
        with torch.cuda.graph(graph1, stream=stream):
            compute_one(0)
        torch.cuda.synchronize()

    def step():
        if graph is not None:
            graph.replay()
        else:
            compute_all()
        gather()

    with torch.cuda.stream(stream):
        for _ in range(max(args.warmup, 3)):
            step()
    torch.cuda.synchronize()

    def barrier():
        if world > 1:
            dist.barrier()

    def max_over_ranks(v):
        if world == 1:
            return v
        t = torch.tensor([v], dtype=torch.float64, device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    # ---- timed region: device-resident inputs --------------------------------
    clocks = ClockSampler(local_rank)
    barrier()
    torch.cuda.synchronize()
    clocks.start()
    with torch.cuda.stream(stream):
        t_start = torch.cuda.Event(enable_timing=True)
        t_end = torch.cuda.Event(enable_timing=True)
        t_start.record(stream)
        for _ in range(args.steps):
            step()
        t_end.record(stream)
    torch.cuda.synchronize()
    clk = clocks.stop()
    barrier()
    ms = max_over_ranks(t_start.elapsed_time(t_end))
    ms_per_step = ms / args.steps
    value = world * F * step_views * args.steps / (ms / 1e3)

    # ---- single rig frame in flight: per-rig-frame latency ------------------
    with torch.cuda.stream(stream):
        l0 = torch.cuda.Event(enable_timing=True)
        l1 = torch.cuda.Event(enable_timing=True)
        l0.record(stream)
        for _ in range(max(3, args.steps // 3)):
            graph1.replay() if graph1 is not None else compute_one(0)
        l1.record(stream)
    torch.cuda.synchronize()
    latency_ms = max_over_ranks(l0.elapsed_time(l1)) / max(3, args.steps // 3)

    # ---- e2e: host buffers through the public API (RigPipeline.stream_ticks), ---
    # H2D of every tick's cameras and D2H of its cluster frames inside the region,
    # overlapped with synthesis as a live stream would run them
    e2e_steps = max(3, args.steps)  # as many ticks as timed steps: the slots' fill and drain amortised alike
    E2E_SLOTS = int(os.environ.get("FVV_E2E_SLOTS", "4"))  # r2: 2 / 3 / 4 slots = 10700 / 10726 / 10765 views/s e2e
    e2e_detail = {}
    if vps and world == 1:
        from paper_2112_10603_b200.pipeline import RigPipeline
        # slots bounded by free HBM (cfg5: ~48 GB of engine workspace per slot)
        per_slot = engines[0].workspace_bytes + views_l[0].numel() + clusters_l[0].numel()
        E2E_SLOTS = max(1, min(E2E_SLOTS, int(0.95 * torch.cuda.mem_get_info(dev)[0]) // max(1, per_slot)))
        pipe = RigPipeline(W, H, fmt, C, S, vps, device=dev)
        hins = [hosts[t % F] for t in range(e2e_steps + 2)]
        houts = [torch.empty(pipe.clusters.numel(), dtype=torch.uint8).pin_memory() for _ in range(2)]
        pipe.stream_ticks(hins[:E2E_SLOTS], houts, slots=E2E_SLOTS)  # warm every slot (graph capture)
        torch.cuda.synchronize()
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record(pipe.stream)
        pipe.stream_ticks(hins[:e2e_steps], [houts[t % 2] for t in range(e2e_steps)], slots=E2E_SLOTS)
        e1.record(pipe.stream)
        torch.cuda.synchronize()
        e2e_ms = e0.elapsed_time(e1)
        e2e_value = step_views * e2e_steps / (e2e_ms / 1e3)
        h2d, d2h = hosts[0].numel(), pipe.clusters.numel()
        e2e_detail = {"api": "RigPipeline.stream_ticks (%d slots: copies and consecutive ticks overlapped)" % E2E_SLOTS}
        del pipe
    else:
        # double-buffered: H2D of step t+1 and D2H of step t-1 run on a copy stream
        # while step t computes (device staging slots; the captured graph keeps its
        # fixed buffers, fed and drained by D2D copies at HBM speed)
        cs = torch.cuda.Stream(device=dev)
        st_in = [[torch.empty_like(c) for c in cams_l] for _ in range(2)]
        st_out = [[torch.empty_like(r) for r in results] for _ in range(2)]
        ev_in = [torch.cuda.Event() for _ in range(2)]     # slot's H2D landed
        ev_used = [torch.cuda.Event() for _ in range(2)]   # slot's inputs consumed by compute
        ev_done = [torch.cuda.Event() for _ in range(2)]   # slot's outputs ready for D2H
        ev_out = [torch.cuda.Event() for _ in range(2)]    # slot's D2H finished

        def h2d_issue(t):
            k = t % 2
            with torch.cuda.stream(cs):
                if t >= 2:
                    cs.wait_event(ev_used[k])
                for i in range(F):
                    st_in[k][i].copy_(hosts[i], non_blocking=True)
                ev_in[k].record(cs)
        barrier()
        torch.cuda.synchronize()
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        cs.wait_event(e0)
        h2d_issue(0)
        for t in range(e2e_steps):
            k = t % 2
            if t + 1 < e2e_steps:
                h2d_issue(t + 1)
            with torch.cuda.stream(stream):
                stream.wait_event(ev_in[k])
                for i in range(F):
                    cams_l[i].copy_(st_in[k][i], non_blocking=True)
                ev_used[k].record(stream)
                if t >= 2:
                    stream.wait_event(ev_out[k])  # st_out[k] drained
                step()
                for i in range(F):
                    st_out[k][i].copy_(results[i], non_blocking=True)
                ev_done[k].record(stream)
            with torch.cuda.stream(cs):
                cs.wait_event(ev_done[k])
                for i in range(F):
                    host_out[i].copy_(st_out[k][i], non_blocking=True)
                ev_out[k].record(cs)
        stream.wait_stream(cs)
        e1.record(stream)
        torch.cuda.synchronize()
        barrier()
        e2e_ms = max_over_ranks(e0.elapsed_time(e1))
        e2e_value = world * F * step_views * e2e_steps / (e2e_ms / 1e3)
        h2d = sum(h.numel() for h in hosts)
        d2h = sum(h.numel() for h in host_out)
        e2e_detail = {"api": "Interpolator.rig (+ rig_clusters), copies double-buffered on a copy stream"}

    if rank != 0:
        return 0

    roofline, launches_per_step = kernel_roofline(
        args, cfg, eng, lambda: compute_one(0), npairs_total, clk, stream,
        (lambda: rig_clusters(views, W, H, fmt, C, S, vps, out=clusters)) if vps else None)
    gpu_launches = launches_per_step * F * args.steps

    # CPU baseline: oracle port on this box's host cores, bounded sample
    rate, reps, dt, threads = cpu_interp_rate(cfg, budget_s=args.cpu_budget)
    cpu = {"value": rate, "unit": "views/s", "cores": threads, "kind": "port",
           "sample": f"{reps} x interpolate() {W}x{H} {FMT_NAME[fmt]} in {dt:.1f}s (oracle/, C port of "
                     f"the reference path, {threads} threads)"}

    line = {
        "metric": METRIC, "value": value, "unit": "views/s", "n_gpus": world, "steps": args.steps,
        "warmup": max(args.warmup, 3), "ms_per_step": ms_per_step, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "u8/i32/f64", "data": "synthetic",
        "config": {"workload": args.config, "desc": cfg["desc"], "width": W, "height": H,
                   "format": FMT_NAME[fmt], "cameras": C, "stages": S, "views_per_side": vps,
                   "views_per_rig_frame": step_views, "rig_frames_per_step": F,
                   "rig_frame_latency_ms": latency_ms,
                   "parallelism": f"frame-sharded x{world}, {F} rig frames in flight per rank" +
                                  (" + NCCL gather to rank 0" if world > 1 else ""),
                   "cuda_graph": graph is not None,
                   "l2": "working set > L2 (views %.0f MB + workspace %.0f MB per rank)" % (
                       views.numel() / 1e6, eng.workspace_bytes / 1e6)},
        "roofline": roofline,
        "cpu_baseline": cpu,
        "e2e": {"value": e2e_value, "unit": "views/s", "h2d_bytes_per_step": h2d,
                "d2h_bytes_per_step": d2h, "ms_per_step": e2e_ms / e2e_steps, **e2e_detail},
        "gpu_launches": gpu_launches,
        "clocks": clk,
    }
    if not args.no_direct:
        try:
            line["direct_t"] = run_direct(cfg, eng, cams, views, clusters, stream, steps=max(3, args.steps // 2))
        except Exception as exc:
            line["direct_t"] = {"error": f"{type(exc).__name__}: {exc}"}
    if vps and fmt != 2 and not args.no_encoder:
        try:
            # a second rig frame (another scene) so consecutive P records carry real residuals
            cams2 = torch.from_numpy(synth_rig(W, H, fmt, C, seed=4242)).to(dev)
            clusters2 = torch.empty_like(clusters)
            with torch.cuda.stream(stream):
                eng.rig(cams2, S, views)
                rig_clusters(views, W, H, fmt, C, S, vps, out=clusters2)
            torch.cuda.synchronize()
            line["encoder"] = run_encoder(cfg, dev, [clusters, clusters2], stream)
        except Exception as exc:  # the headline line must survive a failure of the secondary stage
            line["encoder"] = {"error": f"{type(exc).__name__}: {exc}"}
    if not args.no_vinet and rank == 0 and min(W, H) >= 64:
        try:
            line["vinet"] = run_vinet(cfg, dev, use_graph=not args.no_graph)
        except Exception as exc:  # the headline line must survive a failure of the secondary path
            line["vinet"] = {"error": f"{type(exc).__name__}: {exc}"}
    print(json.dumps(line))
    return 0


def kernel_roofline(args, cfg, eng, run_once, npairs_total, clk, stream, tile_fn=None):
    """Live per-kernel CUDA-event timing of one rig frame's stage kernels
    (C-ABI profiling hook) -> the bench line's roofline object for the
    dominant kernel, and the kernel launches of one rig frame."""
    import ctypes

    import torch
    from paper_2112_10603_b200 import _lib
    W, H = cfg["W"], cfg["H"]
    prof_steps = 3
    L = _lib.load()
    _lib.check(L.fvv_profile_enable(eng._h, 4096))
    with torch.cuda.stream(stream):
        for _ in range(prof_steps):
            run_once()
    torch.cuda.synchronize()
    n = 11  # FVV_NUM_KERNEL_CLASSES
    ms_k = (ctypes.c_double * n)()
    cnt_k = (ctypes.c_int * n)()
    _lib.check(L.fvv_profile_read(eng._h, ms_k, cnt_k, n))
    L.fvv_profile_enable(eng._h, 0)
    per_class = {L.fvv_kernel_class_name(i).decode(): (ms_k[i] / prof_steps, cnt_k[i] // prof_steps)
                 for i in range(n)}
    tile_ms = 0.0
    if tile_fn is not None:
        with torch.cuda.stream(stream):
            a = torch.cuda.Event(enable_timing=True)
            b = torch.cuda.Event(enable_timing=True)
            a.record(stream)
            for _ in range(prof_steps):
                tile_fn()
            b.record(stream)
        torch.cuda.synchronize()
        tile_ms = a.elapsed_time(b) / prof_steps
        per_class["k_rig_clusters"] = (tile_ms, 1)
    step_kernel_ms = sum(v[0] for v in per_class.values())
    figs = kernel_figures(cfg, npairs_total)
    dom = max((k for k in per_class if k in figs), key=lambda k: per_class[k][0])
    bound, unit, amount = figs[dom]
    peaks, peak_src = measured_peaks()
    dom_ms = per_class[dom][0]
    if bound == "hbm":
        achieved = amount / (dom_ms / 1e3) / 1e9
        peak = float(peaks["hbm_gbs"])
        peak_note = f"{peak_src} HBM copy bandwidth (MEASURED_PEAKS.json)"
    else:
        achieved = amount / (dom_ms / 1e3) / 1e9
        sm_mhz = clk.get("sm_mhz") or float(peaks.get("sm_max_mhz", 1965.0))
        # issue-rate ceiling for packed-u16 SAD: 148 SMs x 128 lanes/clk x 2 diffs per lane
        peak = 148 * 128 * 2 * sm_mhz * 1e6 / 1e9
        peak_note = ("derived: 148 SMs x 128 lanes x 2 (u16x2) abs-diffs/clk at the median SM clock "
                     "under load; no measured INT peak in MEASURED_PEAKS.json")
    # DRAM bytes and warp instructions per step of the dominant kernel class,
    # from the committed ncu launch list (profiles/traffic.json)
    traffic, issue = None, None
    try:
        with open(os.path.join(ROOT, "profiles", "traffic.json")) as f:
            t = json.load(f).get(args.config, {}).get(dom)
        if t:
            traffic = t["dram_bytes_per_pair"] * npairs_total
            sm_mhz = clk.get("sm_mhz") or float(peaks.get("sm_max_mhz", 1965.0))
            ach = t["warp_inst_per_pair"] * npairs_total / (dom_ms / 1e3) / 1e9
            pk = 148 * 4 * sm_mhz * 1e6 / 1e9  # 4 schedulers x 1 warp-instruction per clock per SM
            issue = {"achieved": ach, "peak": pk, "unit": "G warp-instr/s", "frac": ach / pk,
                     "note": "the path's exact integer/f64 arithmetic makes this kernel issue-bound; "
                             "ncu instruction count x live kernel time vs 148 SMs x 4 issue/clk"}
    except (OSError, KeyError, ValueError):
        pass
    roofline = {"bound": bound, "kernel": dom, "achieved": achieved, "peak": peak, "unit": unit,
                "frac": achieved / peak, "traffic": traffic, "traffic_unit": "bytes per rig frame (ncu dram read+write)",
                "peak_source": peak_note, "issue": issue,
                "kernel_ms_per_step": dom_ms, "kernel_share_of_step": dom_ms / step_kernel_ms,
                "per_kernel_ms_per_step": {k: round(v[0], 4) for k, v in per_class.items()},
                "kernel_timing_unit": "one rig frame (its stage kernels timed alone with CUDA events; "
                                      "traffic from the ncu launch list is per rig frame too)"}

    launches_per_step = sum(v[1] for v in per_class.values())
    # SAD classes launch a second (ragged-column) kernel when the level width is not a multiple of 8
    for s, (lw, _lh) in enumerate([(W // 4, H // 4), (W // 2, H // 2), (W, H)]):
        if lw % 8:
            launches_per_step += per_class[f"k_sad<{s}>"][1]
    return roofline, launches_per_step



def vinet_conv_flops(W, H):
    """Useful convolution FLOPs of one VINet forward (vinet_params.LAYERS on the 64-aligned canvas)."""
    from paper_2112_10603_b200.vinet_params import BLOCK_IN
    Wp, Hp = (W + 63) // 64 * 64, (H + 63) // 64 * 64
    tot = 0
    for i in range(3):
        w, h = Wp >> (2 - i), Hp >> (2 - i)
        tot += 2 * (w // 2) * (h // 2) * 128 * 9 * BLOCK_IN[i]     # c0
        tot += 2 * (w // 4) * (h // 4) * 256 * 9 * 128             # c1
        tot += 6 * 2 * (w // 4) * (h // 4) * 256 * 9 * 256         # r1..r6
        tot += 2 * (w // 2) * (h // 2) * 128 * 4 * 256             # u0: 2x2 taps per output phase
        tot += 2 * w * h * 5 * 4 * 128                             # u1
    return tot


def vinet_dominant_conv(W, H, npairs, dev, reps=10):
    """Live CUDA-event timing of the network's dominant kernel: one 256->256 3x3 residual
    layer (k_conv_tc<256,128>) of the full-resolution block at 1/4 of the 64-aligned canvas,
    all pairs of the rig in one launch, through the public fvv_conv2d_bf16."""
    import torch
    from paper_2112_10603_b200 import convtc
    Wp, Hp = (W + 63) // 64 * 64, (H + 63) // 64 * 64
    w4, h4 = Wp // 4, Hp // 4
    g = torch.Generator(device=dev).manual_seed(5)
    x = (torch.randn((npairs, h4, w4, 256), generator=g, device=dev) * 0.5).to(torch.bfloat16)
    wt = torch.randn((256, 256, 3, 3), generator=g, device=dev) * (2.0 / 2304) ** 0.5
    wp = convtc.pack_conv(wt, 256, 256)
    b = torch.zeros(256, device=dev)
    out = torch.empty((npairs, h4, w4, 256), dtype=torch.bfloat16, device=dev)
    for _ in range(3):
        convtc.conv2d(x, wp, b, 256, 3, 1, 1, out=out, ntile=256)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        convtc.conv2d(x, wp, b, 256, 3, 1, 1, out=out, ntile=256)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / reps
    flop = 2.0 * npairs * h4 * w4 * 256 * 256 * 9
    peaks, src = measured_peaks()
    burst = float(peaks.get("bf16_tflops", 1701.7))                 # a kernel timed alone: burst peak
    sustained = float(peaks.get("bf16_tflops_sustained", burst))
    ach = flop / (ms / 1e3) / 1e12
    return {"kernel": "k_conv_tc<256,128> (3x3 256->256, %d x %dx%d)" % (npairs, h4, w4), "bound": "tensor",
            "achieved": ach, "peak": burst, "unit": "TFLOP/s", "frac": ach / burst,
            "frac_vs_sustained": ach / sustained, "flop_per_launch": flop, "ms_per_launch": ms,
            "peak_source": "%s cuBLAS bf16 8192^3, burst (kernel timed alone, %d back-to-back launches)" % (src, reps)}


def run_vinet(cfg, dev, steps=10, warmup=3, use_graph=True):
    """The north-star CNN path on the same rig: VINet flows once per camera gap
    + direct-t synthesis of all views of the gap in one pass (tcgen05 convs),
    written into the global views buffer, then the cluster frames."""
    import torch
    from paper_2112_10603_b200.cluster import rig_cluster_sizes, rig_clusters
    from paper_2112_10603_b200.vinet import VINet
    W, H, fmt, C, S, vps = cfg["W"], cfg["H"], cfg["fmt"], cfg["cams"], cfg["stages"], cfg["vps"]
    npairs, nviews = C - 1, (1 << S) - 1
    cams = torch.from_numpy(synth_rig(W, H, fmt, C, seed=42)).to(dev)
    net = VINet(W, H, fmt, seed=0, max_pairs=npairs, device=dev)
    views = net.rig(cams, S)
    tiled = bool(vps) and fmt != 2
    clusters = torch.empty(max(1, sum(rig_cluster_sizes(W, H, fmt, C, S, vps))) if tiled else 1,
                           dtype=torch.uint8, device=dev)
    L, R = cams[:-1].contiguous(), cams[1:].contiguous()
    flows = net.flows(L, R)

    def step():  # fused: the synthesis epilogue writes the quarter tiles (fvv_vinet_rig_clusters)
        if tiled:
            net.rig_clusters(cams, S, vps, views=views, out=clusters)
        else:
            net.rig(cams, S, views=views)

    def step_unfused():  # fvv_vinet_rig + fvv_rig_clusters (views re-read for the tiles)
        net.rig(cams, S, views=views)
        if tiled:
            rig_clusters(views, W, H, fmt, C, S, vps, out=clusters)
    def flows_only():
        net.flows(L, R, out=flows)
    for _ in range(warmup):
        step()
        step_unfused()
        flows_only()
    torch.cuda.synchronize()
    # one CUDA graph per variant: the ~150 launches of a rig frame replay without host work
    graphs, graph_note = {}, None
    if use_graph:
        try:
            for name, fn in (("fused", step), ("flows", flows_only), ("unfused", step_unfused)):
                g = torch.cuda.CUDAGraph()
                with torch.cuda.graph(g):
                    fn()
                graphs[name] = g
            torch.cuda.synchronize()
        except Exception as ex:  # keep the eager numbers rather than none
            graphs, graph_note = {}, f"capture failed, eager: {type(ex).__name__}: {ex}"

    def run(name, fn):
        if name in graphs:
            graphs[name].replay()
        else:
            fn()
    for name, fn in (("fused", step), ("flows", flows_only), ("unfused", step_unfused)):
        run(name, fn)
    torch.cuda.synchronize()
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(4)]
    ev[0].record()
    for _ in range(steps):
        run("fused", step)
    ev[1].record()
    for _ in range(steps):
        run("flows", flows_only)
    ev[2].record()
    for _ in range(steps):
        run("unfused", step_unfused)
    ev[3].record()
    torch.cuda.synchronize()
    unfused_ms = ev[2].elapsed_time(ev[3]) / steps
    rig_ms, fl_ms = ev[0].elapsed_time(ev[1]) / steps, ev[1].elapsed_time(ev[2]) / steps
    dom = vinet_dominant_conv(W, H, npairs, dev)
    flops = vinet_conv_flops(W, H) * npairs
    try:
        refine = run_refine(cfg, dev, net, cams, flows, steps=3, use_graph=use_graph)
    except Exception as exc:  # keep the VINet numbers if the refinement stage fails
        refine = {"error": f"{type(exc).__name__}: {exc}"}
    peaks, src = measured_peaks()
    peak = float(peaks.get("bf16_tflops_sustained", peaks.get("bf16_tflops", 1401.6)))
    ach = flops / (fl_ms / 1e3) / 1e12
    return {
        "path": "VINet (north-star CNN: 3 VIBlocks x 10 tcgen05 conv layers, seeded random-init weights), "
                "direct-t synthesis of every view of a gap from one flow field, cluster tiles fused into its epilogue",
        "value": npairs * nviews / (rig_ms / 1e3), "unit": "views/s",
        "ms_per_step": rig_ms, "flows_ms": fl_ms, "synth_and_tiling_ms": rig_ms - fl_ms,
        "unfused_ms_per_step": unfused_ms, "tiling": "fused into the synthesis epilogue" if tiled else "none",
        "cuda_graph": bool(graphs), **({"graph_note": graph_note} if graph_note else {}),
        "pairs": npairs, "views_per_pair": nviews, "dtype": "bf16 convs, fp32 accumulate / warps",
        "roofline": {"bound": "tensor", "achieved": ach, "peak": peak, "unit": "TFLOP/s", "frac": ach / peak,
                     "traffic": None, "flop_per_step": flops,
                     "note": "useful conv FLOPs / whole flow-network time (pyramid, block inputs and "
                             "residual kernels included); peak = sustained cuBLAS bf16 (%s)" % src},
        "dominant_kernel": dom,
        "synthesis": synth_roofline(cfg, rig_ms - fl_ms, npairs, nviews, tiled, peaks, src),
        "parity": "fp32 torch oracle (oracle/vinet_ref.py): flows within 3 % max-abs, synthesis within "
                  "1 level, end-to-end PSNR >= 50 dB (tests/test_gpu_vinet.py)",
        "refine": refine,
    }


def run_direct(cfg, eng, cams, views, clusters, stream, steps=10):
    """Direct-t mode of the SAD path (fvv_rig_views_mode FVV_DENSE_DIRECT): per gap
    one interpolation (its t = 1/2 view bit-exact with the reference) plus the
    other views synthesized from its flows and mask, then the cluster frames;
    the same rig frame as the headline, as one CUDA graph."""
    import torch
    from paper_2112_10603_b200.cluster import rig_clusters
    W, H, fmt, C, S, vps = cfg["W"], cfg["H"], cfg["fmt"], cfg["cams"], cfg["stages"], cfg["vps"]
    step_views = (C - 1) * ((1 << S) - 1)

    def frame():
        eng.rig(cams, S, views, mode=1)
        if vps:
            rig_clusters(views, W, H, fmt, C, S, vps, out=clusters)
    with torch.cuda.stream(stream):
        frame()
        torch.cuda.synchronize()
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=stream):
            frame()
        for _ in range(3):
            g.replay()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(stream)
        for _ in range(steps):
            g.replay()
        b.record(stream)
    torch.cuda.synchronize()
    ms = a.elapsed_time(b) / steps
    return {"path": "SAD flows, direct-t: one interpolation per camera gap (t = 1/2 bit-exact vs interp.py:131-132) "
                    "+ the other views of the gap synthesized from its flows and mask in one pass, cluster frames",
            "value": step_views / (ms / 1e3), "unit": "views/s", "ms_per_step": ms, "interpolations_per_step": C - 1,
            "cuda_graph": True,
            "parity": "t = 1/2 views bit-exact vs the oracle; other views within 1 level of the fp32 direct-t "
                      "restatement (oracle/vinet_ref.synth) on the oracle's flows and mask (tests/test_gpu_timed_path.py)"}


def run_encoder(cfg, dev, cluster_bufs, stream, ticks=4):
    """The encoder hand-off: FVT1 records of every
    tile of every cluster frame of the rig frame (server/pipeline.py:294-318),
    transform stage and DEFLATE (zlib-identical, deflate_kernels.cu) on the
    device (encoder.RigEncoder), record framing on the host.  gop 30
    (PipelineConfig default): tick 0 is intra, the rest P.  One tick is also
    timed with DEFLATE on the host thread pool (the previous design)."""
    import time

    import torch
    from paper_2112_10603_b200.cluster import build_layouts
    from paper_2112_10603_b200.encoder import RigEncoder
    from paper_2112_10603_b200.viewmodel import ViewIndexModel
    W, H, fmt, C, S, vps = cfg["W"], cfg["H"], cfg["fmt"], cfg["cams"], cfg["stages"], cfg["vps"]
    threads = os.cpu_count() or 8
    enc = RigEncoder(build_layouts(ViewIndexModel(C, S), vps), W, H, fmt, quality=75, gop=30, device=dev,
                     threads=threads)
    with torch.cuda.stream(stream):
        enc.encode(cluster_bufs[0])  # intra tick (warm-up)
        torch.cuda.synchronize()
        nbytes = 0
        recs0 = None
        walls = []
        for k in range(ticks):
            t0 = time.perf_counter()
            recs = enc.encode(cluster_bufs[(k + 1) % len(cluster_bufs)])
            walls.append(time.perf_counter() - t0)
            recs0 = recs if recs0 is None else recs0
            nbytes += sum(len(r) for c in recs for r in c)
        wall = statistics.median(walls)  # per tick; host-side hiccups do not skew it
        # device transform stage alone (blocks + tokens kernels), CUDA events
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        import ctypes
        from paper_2112_10603_b200 import _lib
        L = _lib.load()
        jt = enc._last_jobs
        a.record(stream)
        for _ in range(ticks):
            _lib.check(L.fvv_encode_blocks(ctypes.c_void_p(jt.data_ptr()), enc._last_njobs, enc.nblocks,
                                           int(enc.lossless), ctypes.c_void_p(enc.zz.data_ptr()),
                                           ctypes.c_void_p(enc.ntok.data_ptr()), ctypes.c_void_p(stream.cuda_stream)))
        b.record(stream)
        torch.cuda.synchronize()
        dev_ms_blocks = a.elapsed_time(b) / ticks
        # device DEFLATE alone (all plane token streams of the last tick), CUDA events
        from paper_2112_10603_b200.deflate import deflate_streams
        po = enc._last_plane_offs
        tok = enc.tokens[:po[-1]]
        a.record(stream)
        for _ in range(ticks):
            deflate_streams(tok, po, stream=stream)
        b.record(stream)
        torch.cuda.synchronize()
        zd_ms = a.elapsed_time(b) / ticks
        # the previous design: DEFLATE with zlib on the host threads (one P tick)
        enc_h = RigEncoder(build_layouts(ViewIndexModel(C, S), vps), W, H, fmt, quality=75, gop=30, device=dev,
                           threads=threads, deflate="host")
        enc_h.encode(cluster_bufs[0])
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        recs_h = enc_h.encode(cluster_bufs[1 % len(cluster_bufs)])
        host_ms = (time.perf_counter() - t0) * 1e3
    dev_ms = dev_ms_blocks
    tiles = sum(len(t) for t in enc.tiles)
    return {"path": "FVT1 tile records (codec.TileEncoder-identical bytes) of every tile of the rig frame's "
                    "cluster frames: 8x8 DCT / quant / reconstruction / zigzag / tokens and DEFLATE "
                    "(zlib level 6, byte-identical) on the device, record framing on the host",
            "tiles_per_rig_frame": tiles, "quality": 75, "gop": 30, "record": "P (closed loop, device-resident "
            "reconstruction)", "ms_per_rig_frame": wall * 1e3, "device_transform_ms": dev_ms,
            "device_deflate_ms": zd_ms, "token_bytes_per_rig_frame": int(po[-1]),
            "host_deflate_ms_per_rig_frame": host_ms, "host_deflate_threads": threads,
            "records_identical_device_vs_host_zlib": recs_h == recs0,
            "bytes_per_rig_frame": nbytes / ticks,
            "parity": "byte-identical records vs reference-generated goldens, lossy I/P and lossless "
                      "(tests/test_gpu_encoder.py)"}


def synth_roofline(cfg, ms, npairs, nviews, tiled, peaks, src):
    """HBM roofline of the direct-t synthesis (+ fused tiling): per pair both source
    frames read once, every view written, plus its quarter tile when tiled."""
    W, H, fmt = cfg["W"], cfg["H"], cfg["fmt"]
    fb = {0: 1.0, 1: 1.5, 2: 3.0}[fmt] * W * H
    nbytes = npairs * (2 * fb + nviews * fb * (1 + (1 / 16 if tiled else 0)))
    ach = nbytes / (ms / 1e3) / 1e9 if ms > 0 else 0.0
    peak = float(peaks["hbm_gbs"])
    return {"bound": "hbm", "achieved": ach, "peak": peak, "unit": "GB/s", "frac": ach / peak,
            "bytes_per_step": nbytes, "ms_per_step": ms,
            "note": "algorithmic bytes (2 frames read + views written per pair) / synthesis + tiling time; "
                    "the 15 views of a pixel reuse its source taps from L1/L2, so the kernel is "
                    "instruction-bound well below this (DESIGN.md sec. 9); peak: %s HBM copy bandwidth" % src}


def refine_conv_flops(W, H, nviews, npairs=1):
    """Useful conv FLOPs of RefineNet (per view) + ContextNet (per pair, 2 images) on the 64-aligned canvas."""
    from paper_2112_10603_b200.vinet_params import CONTEXT_LAYERS, REFINE_LAYERS
    Wp, Hp = (W + 63) // 64 * 64, (H + 63) // 64 * 64
    ctx, h, w = 0, Hp, Wp
    for _, stride, cin, cout in CONTEXT_LAYERS:
        h, w = h // stride, w // stride
        ctx += 2 * cin * cout * 9 * h * w
    un, h, w = 0, Hp, Wp
    for _, kind, cin, cout in REFINE_LAYERS:
        if kind == "conv_s2":
            h, w = h // 2, w // 2
        if kind == "convT":
            h, w = h * 2, w * 2
            un += 2 * cin * cout * 4 * h * w
        else:
            un += 2 * cin * cout * 9 * h * w
    return npairs * (2 * ctx + nviews * un)


def run_refine(cfg, dev, net, cams, flows, steps=5, use_graph=True):
    """RefineNet + ContextNet on every direct-t view of the rig:
    context once per pair, U-Net per view (15 views of a gap per batch)."""
    import torch
    from paper_2112_10603_b200.refine import RefineNet
    W, H, fmt, C, S = cfg["W"], cfg["H"], cfg["fmt"], cfg["cams"], cfg["stages"]
    npairs, nviews = C - 1, (1 << S) - 1
    ref = RefineNet(W, H, fmt, seed=1, max_views=min(nviews, 8), device=dev)
    L, R = cams[:-1].contiguous(), cams[1:].contiguous()
    out = torch.empty((npairs, nviews, ref.frame_bytes), dtype=torch.uint8, device=dev)

    def step():
        net.flows(L, R, out=flows)
        ref.views(L, R, flows, nviews, out=out)

    def refine_only():
        ref.views(L, R, flows, nviews, out=out)
    for _ in range(2):
        step()
    torch.cuda.synchronize()
    graphs = {}
    if use_graph:
        for name, fn in (("step", step), ("refine", refine_only)):
            g = torch.cuda.CUDAGraph()
            with torch.cuda.graph(g):
                fn()
            graphs[name] = g
        torch.cuda.synchronize()
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(3)]
    ev[0].record()
    for _ in range(steps):
        graphs["step"].replay() if graphs else step()
    ev[1].record()
    for _ in range(steps):
        graphs["refine"].replay() if graphs else refine_only()
    ev[2].record()
    torch.cuda.synchronize()
    step_ms, ref_ms = ev[0].elapsed_time(ev[1]) / steps, ev[1].elapsed_time(ev[2]) / steps
    flops = refine_conv_flops(W, H, nviews, npairs)
    peaks, src = measured_peaks()
    peak = float(peaks.get("bf16_tflops_sustained", peaks.get("bf16_tflops", 1401.6)))
    ach = flops / (ref_ms / 1e3) / 1e12
    return {"path": "VINet flows + RefineNet/ContextNet-refined direct-t views (21 tcgen05 conv layers per view, "
                    "context features once per pair), seeded random-init weights",
            "value": npairs * nviews / (step_ms / 1e3), "unit": "views/s", "ms_per_step": step_ms,
            "refine_ms": ref_ms, "cuda_graph": bool(graphs),
            "roofline": {"bound": "tensor", "achieved": ach, "peak": peak, "unit": "TFLOP/s", "frac": ach / peak,
                         "flop_per_step": flops,
                         "note": "useful RefineNet + ContextNet conv FLOPs / refine time (input, warp, skip and "
                                 "output kernels included); peak = sustained cuBLAS bf16 (%s)" % src},
            "parity": "fp32 torch oracle (oracle/vinet_ref.py refine_view): PSNR >= 50 dB (tests/test_gpu_refine.py)"}


def run_b200_gap(args, cfg, rank, world, local_rank):
    """Gap-sharded rig frame (SURVEY.md sec. 8(e) option 2; cfg3/cfg4 "pairs
    sharded across B200s"): ONE rig frame per step split over the ranks by
    contiguous camera gaps (shard.GapShardedRig).  Per step: each rank's dense
    views + outgoing halo tiles (graph), the halo exchange (NCCL P2P), its
    cluster frames (graph), the gather of every cluster frame to the
    encoder-feeding rank 0 (NCCL P2P).  Total work per step is fixed, so the
    per-rig-frame latency drops with N (scaling "strong")."""
    import torch
    import torch.distributed as dist
    from paper_2112_10603_b200.shard import GapShardedRig, gap_plan

    torch.cuda.set_device(local_rank)
    dev = torch.device("cuda", local_rank)
    W, H, fmt, C, S, vps = cfg["W"], cfg["H"], cfg["fmt"], cfg["cams"], cfg["stages"], cfg["vps"]
    step_views = (C - 1) * ((1 << S) - 1)
    rig = GapShardedRig(W, H, fmt, C, S, vps, rank, world, device=dev)
    p = rig.plan
    all_cams = synth_rig(W, H, fmt, C, seed=42)
    host_cams = torch.from_numpy(all_cams[p.cams.start:p.cams.stop] if p.active else all_cams[:1]).pin_memory()
    ncam_local = len(p.cams)
    if p.active:
        rig.cams[:ncam_local].copy_(host_cams)
    total_cluster_bytes = sum(rig.sizes_by_rank)
    gathered = torch.empty(total_cluster_bytes, dtype=torch.uint8, device=dev) if rank == 0 else None
    host_out = torch.empty(total_cluster_bytes, dtype=torch.uint8).pin_memory() if rank == 0 else None
    stream = torch.cuda.Stream(device=dev)

    def barrier():
        if world > 1:
            dist.barrier()

    barrier()  # communicators up before any rank-specific P2P

    g_compute = g_stitch = None
    if not args.no_graph and p.active:  # a rank without gaps (more GPUs than gaps) has nothing to capture
        with torch.cuda.stream(stream):
            rig.compute()
            rig.exchange()
            rig.stitch()
        torch.cuda.synchronize()
        g_compute, g_stitch = torch.cuda.CUDAGraph(), torch.cuda.CUDAGraph()
        with torch.cuda.graph(g_compute, stream=stream):
            rig.compute()
        with torch.cuda.graph(g_stitch, stream=stream):
            rig.stitch()
        torch.cuda.synchronize()

    def step(h2d=False, d2h=False):
        if h2d and p.active:
            rig.cams[:ncam_local].copy_(host_cams, non_blocking=True)
        g_compute.replay() if g_compute is not None else rig.compute()
        rig.exchange()
        g_stitch.replay() if g_stitch is not None else rig.stitch()
        res = rig.gather(out=gathered)
        if d2h and rank == 0:
            host_out.copy_(res[:total_cluster_bytes], non_blocking=True)

    with torch.cuda.stream(stream):
        for _ in range(max(args.warmup, 3)):
            step()
    torch.cuda.synchronize()

    def all_reduce(v, op="sum"):
        t = torch.tensor([v], dtype=torch.float64, device=dev)
        if world > 1:
            dist.all_reduce(t, op=dist.ReduceOp.MAX if op == "max" else dist.ReduceOp.SUM)
        return float(t.item())

    def max_over_ranks(v):
        return all_reduce(v, "max")

    clocks = ClockSampler(local_rank)
    barrier()
    torch.cuda.synchronize()
    clocks.start()
    t0, t1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with torch.cuda.stream(stream):
        t0.record(stream)
        for _ in range(args.steps):
            step()
        t1.record(stream)
    torch.cuda.synchronize()
    clk = clocks.stop()
    barrier()
    ms = max_over_ranks(t0.elapsed_time(t1))
    ms_per_step = ms / args.steps
    value = step_views * args.steps / (ms / 1e3)

    # e2e: each rank's camera frames H2D from pinned host memory, rank 0's
    # cluster frames D2H, every step, inside the timed region
    e2e_steps = max(3, args.steps // 2)
    barrier()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with torch.cuda.stream(stream):
        e0.record(stream)
        for _ in range(e2e_steps):
            step(h2d=True, d2h=True)
        e1.record(stream)
    torch.cuda.synchronize()
    barrier()
    e2e_ms = max_over_ranks(e0.elapsed_time(e1))
    h2d = int(all_reduce(host_cams.numel() if p.active else 0))

    # per-rank kernel share (rank 0's gaps), profiled outside the timed region
    roofline, launches = None, 0
    if p.active:
        npairs_rank = len(p.gaps) * ((1 << S) - 1)
        roofline, launches = kernel_roofline(args, cfg, rig.engine, rig.compute, npairs_rank, clk, stream,
                                             rig.stitch)
    launches_all = int(all_reduce(launches))
    if rank != 0:
        return 0
    gaps_per_rank = [len(gap_plan(C, S, vps, r, world).gaps) for r in range(world)]
    line = {
        "metric": METRIC, "value": value, "unit": "views/s", "n_gpus": world, "steps": args.steps,
        "warmup": max(args.warmup, 3), "ms_per_step": ms_per_step, "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": "u8/i32/f64", "data": "synthetic",
        "config": {"workload": args.config, "desc": cfg["desc"], "width": W, "height": H,
                   "format": FMT_NAME[fmt], "cameras": C, "stages": S, "views_per_side": vps,
                   "views_per_rig_frame": step_views, "rig_frames_per_step": 1,
                   "rig_frame_latency_ms": ms_per_step,
                   "parallelism": f"gap-sharded x{world} (gaps per rank {gaps_per_rank}), halo quarter tiles "
                                  "+ cluster gather to rank 0 over NCCL P2P",
                   "cuda_graph": not args.no_graph,
                   "l2": "working set > L2 (views %.0f MB + workspace %.0f MB on rank 0)" % (
                       rig.views.numel() / 1e6, rig.engine.workspace_bytes / 1e6 if rig.engine else 0)},
        "roofline": roofline,
        "cpu_baseline": None,
        "e2e": {"value": step_views * e2e_steps / (e2e_ms / 1e3), "unit": "views/s", "h2d_bytes_per_step": h2d,
                "d2h_bytes_per_step": total_cluster_bytes, "ms_per_step": e2e_ms / e2e_steps,
                "api": "shard.GapShardedRig (compute / exchange / stitch / gather), copies not overlapped"},
        "gpu_launches": launches_all * args.steps,
        "clocks": clk,
    }
    print(json.dumps(line))
    return 0


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=50)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--config", default="cfg4", choices=sorted(CONFIGS))
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--no-graph", action="store_true")
    ap.add_argument("--frames-in-flight", type=int, default=0,
                    help="independent rig frames of the live stream processed concurrently per step "
                         "(0 = auto: 3 when they fit a quarter of HBM, else 1)")
    ap.add_argument("--cpu-budget", type=float, default=12.0)
    ap.add_argument("--no-vinet", action="store_true", help="skip the VINet (CNN path) section")
    ap.add_argument("--no-encoder", action="store_true", help="skip the encoder hand-off section")
    ap.add_argument("--no-direct", action="store_true", help="skip the direct-t SAD-path section")
    ap.add_argument("--shard", default="auto", choices=["auto", "gap", "frame"],
                    help="N>1 partition: gap = one rig frame split by camera gaps (latency; default for "
                         "tiled rigs that fit, cfg3/cfg4), frame = whole rig frames per rank (throughput, cfg5)")
    args = ap.parse_args()
    cfg = CONFIGS[args.config]
    if "WORLD_SIZE" not in os.environ and args.gpus > 1:
        # one process per GPU: re-exec under torchrun (the driver's own launch form)
        import socket
        sock = socket.socket()
        sock.bind(("127.0.0.1", 0))
        port = sock.getsockname()[1]
        sock.close()
        cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
               "--master-addr", "127.0.0.1", "--master-port", str(port), os.path.abspath(__file__), *sys.argv[1:]]
        return subprocess.call(cmd)
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local_rank = int(os.environ.get("LOCAL_RANK", "0"))
    if world != args.gpus:
        print(f"bench.py: --gpus {args.gpus} but WORLD_SIZE {world}", file=sys.stderr)
        return 2
    if args.impl == "reference":
        return run_reference(args, cfg, rank, world)
    shard = args.shard
    if shard == "auto":
        shard = "gap" if cfg["vps"] and args.config != "cfg5" else "frame"
    if world > 1:
        import torch
        import torch.distributed as dist
        torch.cuda.set_device(local_rank)
        dist.init_process_group("nccl", device_id=torch.device("cuda", local_rank))
    try:
        if shard == "gap" and (world > 1 or args.shard == "gap"):
            return run_b200_gap(args, cfg, rank, world, local_rank)
        return run_b200(args, cfg, rank, world, local_rank)
    finally:
        if world > 1:
            import torch.distributed as dist
            dist.destroy_process_group()


if __name__ == "__main__":
    sys.exit(main())
