#!/usr/bin/env python
"""bench.py -- LinPrim (arXiv 2501.16312) training-step benchmark on B200.

Workload (BASELINE.json configs[4], the config its metric "fwd+bwd Mpixel/s and train iters/s at
1/2/4/8 B200" is quoted on): 1M octahedra, SH degree 3, a batch of 8 views at 1600x1060.  One step
is paper_2501_16312_b200.step.TrainStep: lp_preprocess of the local views; per view lp_bin_sort ->
lp_render_fwd -> lp_loss_grad (3DGS L1 + SSIM) -> lp_raster_bwd (views over --streams CUDA
streams); lp_preprocess_bwd_assign over the local views; N > 1: ONE NCCL all_reduce of the flat
fp32 gradient (north_star; --sharded: reduce-scatter + sharded Adam + all-gather instead); the
fused Adam (learning rates P:1169-1185).  Views are sharded views[r::N] over ranks (strong
scaling of the fixed global batch of 8).

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
      --gpus N > 1 without WORLD_SIZE in the environment re-launches itself through
      torch.distributed.run with N ranks (127.0.0.1); under torchrun --gpus must equal WORLD_SIZE.
  python bench.py --gpus 2 --dry-run      (CPU: spawns the ranks over gloo and reports them; no GPU)

--impl reference times the CPU oracle (oracle/, plain C fp64) on a bounded pixel sample of the
same workload on the host cores (rank 0 only).
"""
from __future__ import annotations

import argparse
import json
import math
import os
import socket
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

WORKLOAD = "C5"
METRIC = "fwd+bwd Mpixel/s (C5 training step: 8 views, fwd+bwd+allreduce+Adam)"
PAPER_FPS_CONTEXT = "paper (RTX 3090, forward only): octahedra 14.6 ms ScanNet++ 1752x1168, 34.6 ms Mip-NeRF360"


def parse(argv=None):
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--n", type=int, default=None, help="override the primitive count (debug)")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--sharded", action="store_true",
                    help="N > 1: reduce-scatter + Adam on 1/N of the parameters + all-gather instead of the "
                         "single allreduce + replicated Adam")
    ap.add_argument("--dry-run", action="store_true",
                    help="launch the ranks and check the process group over gloo on CPU; no GPU work")
    ap.add_argument("--seed", type=int, default=0)
    ap.add_argument("--loss", default="l1ssim", choices=["l1ssim", "l1"],
                    help="training loss: 3DGS (1-0.2) L1 + 0.2 (1-SSIM) (P:212) or L1 only")
    ap.add_argument("--exact", action="store_true",
                    help="the paper's no-ray-space variant (App. D) instead of the EWA ray-space method")
    ap.add_argument("--streams", type=int, default=8, help="CUDA streams the views of a step are spread over")
    ap.add_argument("--wave", type=int, default=4,
                    help="with --split-pre: views in the first preprocess launch (their binning starts early)")
    ap.add_argument("--ar-chunks", type=int, default=4,
                    help="N > 1: the gradient allreduce as this many in-order async chunks, Adam per chunk")
    ap.add_argument("--assign", action=argparse.BooleanOptionalAction, default=True,
                    help="preprocess backward SETS the step's gradient (lp_preprocess_bwd_assign) instead of "
                         "accumulating into a zeroed one")
    ap.add_argument("--split-pre", action=argparse.BooleanOptionalAction, default=False,
                    help="preprocess the first --wave views in their own launch so their binning overlaps "
                         "the preprocess of the others (off by default: one K1 launch over all local views, "
                         "one stream per view, measured faster on C5)")
    ap.add_argument("--dist-backend", default="nccl", choices=["nccl", "gloo"], help=argparse.SUPPRESS)
    ap.add_argument("--shared-gpu", action="store_true", help=argparse.SUPPRESS)   # code-path check: all ranks on cuda:0
    ap.add_argument("--profile-step", action="store_true",
                    help="after warm-up run ONE step between cudaProfilerStart/Stop (ncu --profile-from-start off) and exit")
    return ap.parse_args(argv)


# ------------------------------------------------------------------------------ clocks sampler

class ClockSampler:
    FIELDS = "clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,clocks_event_reasons.hw_slowdown," \
             "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown," \
             "clocks_event_reasons.sw_power_cap"

    def __init__(self, gpu_index):
        self.idx = gpu_index
        self.rows = []
        self.proc = None
        self.thread = None

    def start(self):
        try:
            self.proc = subprocess.Popen(["nvidia-smi", f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits",
                                          "-i", str(self.idx), "-lms", "100"], stdout=subprocess.PIPE,
                                         stderr=subprocess.DEVNULL, text=True)
        except OSError:
            self.proc = None
            return
        self.thread = threading.Thread(target=self._read, daemon=True)
        self.thread.start()

    def _read(self):
        for line in self.proc.stdout:
            parts = [p.strip() for p in line.split(",")]
            if len(parts) >= 8:
                self.rows.append(parts)

    def stop(self):
        if self.proc is not None:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except subprocess.TimeoutExpired:
                self.proc.kill()
        if self.thread is not None:
            self.thread.join(timeout=2)

    def summary(self):
        if not self.rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unavailable"]}
        sm = [float(r[0]) for r in self.rows if r[0].replace(".", "").isdigit()]
        mx = [float(r[1]) for r in self.rows if r[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = set()
        for r in self.rows:
            for k, nm in enumerate(names):
                if r[4 + k].lower() == "active":
                    reasons.add(nm)
        load = [s for s in sm if s > 0.5 * max(sm)] if sm else []
        return {"sm_mhz": statistics.median(load) if load else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": sorted(reasons), "samples": len(self.rows)}


# ------------------------------------------------------------------------------ work models
#
# Algorithmic work per launch.  Each raster kernel's fraction is reported under two
# models side by side; `frac` is SURVEY §8(d)'s:
#   K3 forward (lane instr.): §8(d) 28 I + 9 X (octa) / 16 I + 9 X (tetra);  builder 6 I + 24 B + 11 X (tetra 19 B)
#   K4 backward:              §8(d) 36 I_b + 50 X + 32 W_h + 20 A with I_b = I (the pairs a reverse walk of
#                             the processed lists visits);  builder 6 I + 30 B + 61 X (tetra 25 B)
#   I iterated, B in-bbox, X intersected (pixel, entry) pairs; W_h (warp, entry) and A (tile, entry) pairs
#   with a hit -- all counted by the untimed count_stats pass (LP_CNT_*).
# HBM kernels (bytes per launch): K1 N F + v (24 N + 4 RW V_vis); K5 4 N v + 4 RG V_vis v + 3 N F (v views
#   of the launch); K2 (lp_bin_sort, per view) §8(d) (24 + 24 P) E + 24 N with P = ceil(key bits / 8) 8-bit
#   passes of the (tile|depth) key; Adam 28 B per parameter (32 without --assign).

def raster_work(kind, c, backward, model):
    I, B, X, Wh, A = c["I"], c["B"], c["X"], c["Wh"], c["A"]
    if model == "survey":
        if not backward:
            return (28 if kind == 0 else 16) * I + 9 * X
        return 36 * I + 50 * X + 32 * Wh + 20 * A
    chord = 24 if kind == 0 else 19
    if not backward:
        return 6 * I + chord * B + 11 * X
    return 6 * I + (chord + 6) * B + 61 * X


def load_json(path):
    try:
        return json.load(open(path))
    except Exception:
        return {}


# ------------------------------------------------------------------------------ our implementation

def run_ours(args, rank, world, local_rank):
    import torch
    import torch.distributed as dist

    from paper_2501_16312_b200 import linprim as L
    from paper_2501_16312_b200 import render, scenegen, step as S, train

    torch.cuda.set_device(local_rank)
    dev = torch.device("cuda", local_rank)
    scene, cams = scenegen.make_scene(WORKLOAD, seed=args.seed, n=args.n)
    n_views = len(cams)
    W, H = cams[0]["width"], cams[0]["height"]
    my_views = train.shard_views(n_views, rank, world)
    my_cams = [cams[v] for v in my_views]
    kappa = 0.0 if args.exact else 0.1
    ds = S.device_scene(scene, dev, world, args.sharded)

    # synthetic targets: the same scene with jittered centres, rendered once at setup
    rng = np.random.default_rng(1234)
    tgt_scene = dict(scene)
    tgt_scene["pos"] = (scene["pos"] + rng.normal(0, 0.01, scene["pos"].shape) *
                        scene["dist"].mean(0, keepdims=True)).astype(np.float32)
    tds = render.DeviceScene(tgt_scene, device=dev)
    targets_render = render.Renderer(tds, my_cams, exact=args.exact, aa_kernel=kappa).forward()
    # training targets are 8-bit images (the datasets' PNG / JPEG frames): quantised once here; both the
    # device-timed loop and the e2e loop train on the same 8-bit targets, e2e ships them as bytes and
    # expands them on the device (lp_image_from_u8)
    targets_u8 = (targets_render.clamp(0.0, 1.0) * 255.0).round().to(torch.uint8)
    targets = torch.empty_like(targets_render)
    L.lp_image_from_u8(targets_u8, targets, torch.cuda.current_stream(dev))
    torch.cuda.synchronize()
    del tds, targets_render

    # counters pass (untimed): per view E, I, B, X, W_h, A, visible primitives
    rr = render.Renderer(ds, my_cams, count_stats=True, exact=args.exact, aa_kernel=kappa)
    rr.forward()
    torch.cuda.synchronize()
    stats = [rr.counters(i) for i in range(len(my_views))]
    del rr
    u64 = lambda s, k: int(s[k]) | (int(s[k + 1]) << 32)
    cnt = {"E": [int(s[L.LP_CNT_ENTRIES]) for s in stats], "I": [u64(s, L.LP_CNT_ITERATED) for s in stats],
           "X": [u64(s, L.LP_CNT_INTERSECTED) for s in stats], "B": [u64(s, L.LP_CNT_INBOX) for s in stats],
           "Wh": [int(s[L.LP_CNT_WARP_HITS]) for s in stats], "A": [int(s[L.LP_CNT_TILE_HITS]) for s in stats],
           "vis": [int(s[L.LP_CNT_VISIBLE]) for s in stats], "frustum": [int(s[L.LP_CNT_FRUSTUM]) for s in stats]}

    ts = S.TrainStep(ds, my_cams, n_views, targets=targets, loss=args.loss, streams=args.streams,
                     split_pre=args.split_pre, assign=args.assign, exact=args.exact,
                     capacity=int(max(cnt["E"]) * 1.3) + 4096, world=world, rank=rank, sharded=args.sharded,
                     loss_slots=2 * (args.warmup + 3 * args.steps) + 64, ar_chunks=args.ar_chunks, wave=args.wave)
    st = ts.st
    n_local = ts.n_local
    total_steps = args.warmup + args.steps

    def barrier():
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()

    def check_overflow(where):
        assert not ts.overflowed(), f"tile-list capacity overflow ({where})"

    for s in range(args.warmup):
        ts.run(s)
    barrier()
    if args.profile_step:
        torch.cuda.profiler.start()
        ts.run(args.warmup)
        torch.cuda.synchronize()
        torch.cuda.profiler.stop()
        return None, None
    check_overflow("warm-up")

    vis = [s for s in os.environ.get("CUDA_VISIBLE_DEVICES", "").split(",") if s.strip().isdigit()]
    clocks = ClockSampler(int(vis[local_rank]) if local_rank < len(vis) else local_rank)
    t0 = torch.cuda.Event(enable_timing=True)
    t1 = torch.cuda.Event(enable_timing=True)
    clocks.start()
    time.sleep(0.3)
    barrier()
    wall0 = time.perf_counter()
    t0.record(st)
    for k in range(args.steps):
        ts.run(args.warmup + k)
    t1.record(st)
    barrier()
    wall = time.perf_counter() - wall0
    clocks.stop()
    check_overflow("timed loop")     # Adam moved the scene during the timed steps
    ms_t = torch.tensor([t0.elapsed_time(t1)], device=dev)
    if world > 1:
        dist.all_reduce(ms_t, op=dist.ReduceOp.MAX)
    ms_step = float(ms_t.item()) / args.steps

    # ---------------- attribution: the same K steps with the views serialised on one stream and CUDA
    # events around every stage (per view: sort, fwd, loss, raster bwd; per step: pre, pbwd, collective, adam)
    ev_names = ["sort", "fwd", "loss", "rbwd"]
    evs = [[[torch.cuda.Event(enable_timing=True) for _ in range(5)] for _ in range(n_local)] +
           [[torch.cuda.Event(enable_timing=True) for _ in range(5)]] for _ in range(args.steps)]
    barrier()
    for k in range(args.steps):
        ts.run(total_steps + k, t=args.warmup + k + 1, events=evs[k], serial=True)
    barrier()
    check_overflow("attribution loop")
    stage = {nm: [] for nm in ev_names}
    pre, pb, ar, ad = [], [], [], []
    for k in range(args.steps):
        for i in range(n_local):
            e = evs[k][i]
            for j, nm in enumerate(ev_names):
                stage[nm].append(e[j].elapsed_time(e[j + 1]))
        Sv = evs[k][n_local]
        pre.append(Sv[0].elapsed_time(Sv[1]))
        pb.append(evs[k][n_local - 1][4].elapsed_time(Sv[2]))
        ar.append(Sv[2].elapsed_time(Sv[3]))
        ad.append(Sv[3].elapsed_time(Sv[4]))
    stage_ms = {nm: statistics.mean(vals) for nm, vals in stage.items()}
    stage_ms["pre_all_views"] = statistics.mean(pre)
    stage_ms["pbwd_all_views"] = statistics.mean(pb)
    stage_ms["collective"] = statistics.mean(ar)
    stage_ms["adam"] = statistics.mean(ad)
    serial_step_ms = statistics.mean(evs[k][n_local][0].elapsed_time(evs[k][n_local][4]) for k in range(args.steps))

    # ---------------- standalone all-reduce busbw probe of the step's gradient buffer (N > 1)
    probe = None
    if world > 1:
        buf = torch.empty_like(ds.grad_padded)
        buf.fill_(1.0)
        for _ in range(3):
            dist.all_reduce(buf)
        barrier()
        a0, a1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        reps = 20
        a0.record(st)
        for _ in range(reps):
            dist.all_reduce(buf)
        a1.record(st)
        barrier()
        t = torch.tensor([a0.elapsed_time(a1) / reps], device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        sec = float(t.item()) * 1e-3
        nbytes = buf.numel() * 4
        algbw = nbytes / sec / 1e9
        probe = {"bytes": nbytes, "ms": round(sec * 1e3, 4), "algbw_gbs": round(algbw, 1),
                 "busbw_gbs": round(algbw * 2 * (world - 1) / world, 1), "nvlink_peak_gbs": 900.0,
                 "step_collective_ms": round(stage_ms["collective"], 4)}
        del buf

    # ---------------- rooflines: per LAUNCH algorithmic work / per-launch time
    kind = ds.kind
    peaks = load_json(os.path.join(ROOT, "MEASURED_PEAKS.json"))
    hbm_peak = float(peaks.get("hbm_gbs", 6550.0))
    clk_max = float(peaks.get("sm_max_mhz", 1965.0))
    alu_peak = 148 * 128 * clk_max * 1e6 / 1e12            # T FP32 lane-instr/s (nominal: unit counts x max clock)
    ncu_db = load_json(os.path.join(ROOT, "profiles", "round2", "ncu_kernels.json"))
    K = ds.K
    RG, RW = (20, 20) if kind == 0 else (24, 28)
    ncoef = (ds.sh_degree + 1) ** 2
    Fb = 4 * (3 + 4 + K + 1 + 3 * ncoef)                    # feature bytes per primitive
    n = ds.n
    mean = lambda k: statistics.mean(cnt[k])
    per_view = {k: mean(k) for k in ("I", "B", "X", "Wh", "A", "E", "vis")}
    tiles = ts.frames[0].c.tiles_x * ts.frames[0].c.tiles_y
    key_bits = 32 + max(1, math.ceil(math.log2(tiles)))
    P = math.ceil(key_bits / 8)
    n_pre_launch = 2 if (args.split_pre and n_local > ts.wave) else math.ceil(n_local / 8)
    n_k5_launch = math.ceil(n_local / 4)
    v_pre, v_k5 = n_local / n_pre_launch, n_local / n_k5_launch
    params = ts.chunk if ts.sharded else ds.flat.numel()
    # (kernel, bound, per-launch amount [§8(d)], per-launch amount [builder] or None, per-launch ms, launches/step)
    work = {
        "rbwd": ("k_raster_bwd", "alu", raster_work(kind, per_view, True, "survey"),
                 raster_work(kind, per_view, True, "builder"), stage_ms["rbwd"], n_local),
        "fwd": ("k_raster_fwd", "alu", raster_work(kind, per_view, False, "survey"),
                raster_work(kind, per_view, False, "builder"), stage_ms["fwd"], n_local),
        "pre_all_views": ("k_preprocess", "hbm", n * Fb + v_pre * (n * 24 + per_view["vis"] * 4 * RW), None,
                          stage_ms["pre_all_views"] / n_pre_launch, n_pre_launch),
        "pbwd_all_views": ("k_preprocess_bwd", "hbm", 4 * n * v_k5 + per_view["vis"] * v_k5 * 4 * RG + n * 3 * Fb,
                           None, stage_ms["pbwd_all_views"] / n_k5_launch, n_k5_launch),
        "sort": ("lp_bin_sort (K2)", "hbm", (24 + 24 * P) * per_view["E"] + 24 * n, None, stage_ms["sort"], n_local),
        "adam": ("k_adam", "hbm", (28 if args.assign else 32) * params, None, stage_ms["adam"], 1),
        "loss": (("lp_loss_grad (k_ssim_maps + k_ssim_grad)", "alu", 206 * 3 * W * H, None, stage_ms["loss"], n_local)
                 if args.loss == "l1ssim"
                 else ("k_l1_grad", "hbm", 12 * 3 * W * H, None, stage_ms["loss"], n_local)),
    }
    rooflines = {}
    for key, (kname, bound, amount, amount_b, ms_l, nl) in work.items():
        sec = ms_l * 1e-3
        if bound == "alu":
            ach, pk, unit = amount / sec / 1e12, alu_peak, "T FP32 lane-instr/s"
        else:
            ach, pk, unit = amount / sec / 1e9, hbm_peak, "GB/s"
        nc = ncu_db.get(kname.split(" ")[0], {})
        r = {"kernel": kname, "bound": bound, "achieved": round(ach, 3), "peak": round(pk, 3), "unit": unit,
             "frac": round(ach / pk, 4), "traffic": nc.get("traffic_bytes"), "ms": round(ms_l, 4),
             "algorithmic_per_launch": int(amount), "launches_per_step": nl,
             "ms_per_step": round(ms_l * nl, 4)}
        if amount_b is not None:
            r["frac_builder_model"] = round(amount_b / sec / 1e12 / pk, 4)
        if nc.get("thread_inst_executed") and bound == "alu":
            r["frac_ncu_executed"] = round(nc["thread_inst_executed"] / sec / 1e12 / pk, 4)
        if bound == "hbm" and nc.get("traffic_bytes"):
            r["traffic_over_algorithmic"] = round(nc["traffic_bytes"] / amount, 3)
        rooflines[key] = r
    dom = max(rooflines, key=lambda k: rooflines[k]["ms_per_step"])

    mpix = n_views * W * H / 1e6
    value = mpix / (ms_step * 1e-3)

    # ---------------- e2e: host (pinned) targets copied in and the loss read back every step
    e2e = None
    if not args.no_e2e:
        host_t = torch.empty(targets_u8.shape, dtype=torch.uint8, pin_memory=True)
        host_t.copy_(targets_u8)
        dev_u8 = [torch.empty_like(targets_u8), torch.empty_like(targets_u8)]
        dev_t = [torch.empty_like(targets), torch.empty_like(targets)]
        # uploads on a high-priority stream (its expansion kernel gets SMs as soon as raster CTAs retire
        # instead of queueing behind them; measured: 8.35 vs 8.55 ms per step with per-view copies)
        cp = torch.cuda.Stream(dev, priority=torch.cuda.Stream.priority_range()[1])
        copied = [[torch.cuda.Event() for _ in range(n_local)] for _ in range(2)]
        freed = [torch.cuda.Event(), torch.cuda.Event()]
        loss_host = torch.zeros(args.steps, dtype=torch.float32, pin_memory=True)
        read = [torch.cuda.Event() for _ in range(args.steps)]
        done = [torch.cuda.Event() for _ in range(args.steps)]
        rb = torch.cuda.Stream(dev)   # the loss readback, off the step stream (no copy between two steps)
        base = total_steps + args.steps
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)

        def copy_in(b):   # the whole batch: one DMA, one expansion kernel
            with torch.cuda.stream(cp):
                dev_u8[b].copy_(host_t, non_blocking=True)
                L.lp_image_from_u8(dev_u8[b], dev_t[b], cp)
                for i in range(n_local):
                    copied[b][i].record(cp)

        barrier()
        e0.record(st)
        cp.wait_stream(st)
        copy_in(0)
        losses = []
        for k in range(args.steps):
            b = k & 1
            ts.run(base + k, t=args.warmup + args.steps + k + 1, tgt=dev_t[b], tgt_ready=copied[b])
            freed[b].record(st)
            if k + 1 < args.steps:
                # the next step's targets, once this step's middle view has rendered (uploads issued
                # right after the preprocess slowed the step by ~0.25 ms, mid-step ones by ~0.06), into
                # the buffer the previous step has released
                cp.wait_event(ts.mid_done)
                if k >= 1:
                    cp.wait_event(freed[1 - b])
                copy_in(1 - b)
            done[k].record(st)
            rb.wait_event(done[k])
            with torch.cuda.stream(rb):
                loss_host[k:k + 1].copy_(ts.loss_buf[base + k:base + k + 1], non_blocking=True)
            read[k].record(rb)
            if k >= 1:
                read[k - 1].synchronize()
                losses.append(float(loss_host[k - 1]))
        st.wait_stream(rb)
        e1.record(st)
        read[args.steps - 1].synchronize()
        losses.append(float(loss_host[args.steps - 1]))
        barrier()
        check_overflow("e2e loop")
        t = torch.tensor([e0.elapsed_time(e1)], device=dev)
        if world > 1:
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
        e2e_step = float(t.item()) / args.steps
        assert all(math.isfinite(x) for x in losses)
        e2e = {"value": round(mpix / (e2e_step * 1e-3), 3), "unit": "Mpixel/s",
               "h2d_bytes_per_step": int(host_t.numel() * host_t.element_size() * world), "d2h_bytes_per_step": 4 * world,
               "h2d_format": "8-bit target channels, expanded on the device (lp_image_from_u8)",
               "ms_per_step": round(e2e_step, 3), "loss_last": losses[-1]}

    mode = ("sharded Adam (reduce-scatter / all-gather)" if ts.sharded else "one NCCL all_reduce + replicated Adam") \
        if world > 1 else "single GPU"
    out = {
        "metric": METRIC,
        "value": round(value, 3), "unit": "Mpixel/s", "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": round(ms_step, 3), "higher_is_better": True, "scaling": "strong", "vs_baseline": None,
        "dtype": "f32", "data": "synthetic (seeded scenegen, BASELINE configs[4] shape; random-init features)",
        "iters_per_s": round(1000.0 / ms_step, 3),
        "config": {"workload": "C5: 1M octahedra, SH deg 3, 8 views 1600x1060, training step (views sharded)",
                   "loss": "3DGS 0.8 L1 + 0.2 (1 - SSIM)" if args.loss == "l1ssim" else "L1",
                   "projection": "no ray space (App. D)" if args.exact else "EWA ray space",
                   "n_primitives": n, "kind": "octahedron", "sh_degree": 3, "global_batch_views": n_views,
                   "views_per_gpu": n_local, "width": W, "height": H,
                   "parallelism": f"dp{world} (views), {mode}",
                   "l2": "inputs larger than L2: features+grads+Adam state = %.2f GB touched per step"
                         % (ds.flat.numel() * 4 * 5 / 1e9),
                   "tile_list_entries_per_view": cnt["E"],
                   "iterated_pairs_per_px": round(sum(cnt["I"]) / (n_local * W * H), 2),
                   "intersected_pairs_per_px": round(sum(cnt["X"]) / (n_local * W * H), 2),
                   "in_bbox_pairs_per_px": round(sum(cnt["B"]) / (n_local * W * H), 2),
                   "warp_hit_pairs_per_view": cnt["Wh"], "tile_hit_pairs_per_view": cnt["A"],
                   "frustum_primitives_per_view": cnt["frustum"], "capacity": [f.capacity for f in ts.frames]},
        "streams": ts.n_str,
        "stages_ms_per_view": {k: round(v, 4) for k, v in stage_ms.items()},
        "serial_step_ms": round(serial_step_ms, 3),
        "roofline": dict(rooflines[dom], peak_source=(
            "measured HBM copy (MEASURED_PEAKS.json)" if rooflines[dom]["bound"] == "hbm" else
            "nominal: 148 SM x 128 FP32 lanes x %.0f MHz (B200_PROFILING unit counts; no measured FP32 peak)" % clk_max)),
        "rooflines": rooflines,
        "allreduce_probe": probe,
        "e2e": e2e, "gpu_launches": ts.kernel_launches() * args.steps, "wall_s_timed": round(wall, 3),
        "context": PAPER_FPS_CONTEXT,
    }
    out["clocks"] = clocks.summary()
    return out, (scene, cams, my_views)


# ------------------------------------------------------------------------------ oracle (CPU) legs

def oracle_sample(scene, cam, rows, seed=0):
    """Oracle fwd+bwd of the pixel band rows[0]:rows[1] of one view; returns (seconds, pixels)."""
    import oracle
    from paper_2501_16312_b200 import scenegen
    W, H = cam["width"], cam["height"]
    y0, y1 = rows
    pix = (np.arange(y0, y1)[:, None] * W + np.arange(W)[None, :]).reshape(-1).astype(np.int32)
    gx = (W + 15) // 16
    mask = np.zeros(gx * ((H + 15) // 16), np.uint8)
    for ty in range(y0 // 16, (y1 - 1) // 16 + 1):
        mask[ty * gx:(ty + 1) * gx] = 1
    G = scenegen.upstream_grad(W, H, seed=seed)[0]
    osc = oracle.Scene(scene["kind"], scene["pos"], scene["rot"], scene["dist"], scene["opacity"], scene["sh"],
                       scene["sh_degree"])
    t = time.perf_counter()
    oracle.forward_backward(osc, cam, G, pix=pix, tile_mask=mask)
    return time.perf_counter() - t, len(pix)


def cpu_baseline(scene, cams, budget_s=15.0):
    import oracle
    oracle.build()
    H = cams[0]["height"]
    secs, npx = oracle_sample(scene, cams[0], (512, 528))          # one tile row to size the sample
    rows = int(min(H - 512, max(16, 16 * round((budget_s / max(secs, 1e-3)) * 16 / 16 / 1.0))))
    rows = max(16, min(rows, 256))
    secs, npx = oracle_sample(scene, cams[0], (512 - rows // 2, 512 - rows // 2 + rows))
    return {"value": round(npx / secs / 1e6, 6), "unit": "Mpixel/s", "cores": os.cpu_count(), "kind": "oracle",
            "sample": f"fwd+bwd of rows {512 - rows // 2}..{512 - rows // 2 + rows} ({npx} px) of view 0 of the C5 "
                      f"workload incl. preprocess of all 1M primitives and binning of the band; {secs:.1f} s"}


def run_reference(args, rank, world):
    """--impl reference: the oracle as it stands, on a bounded sample per step (rank 0 only)."""
    if rank != 0:
        return None
    from paper_2501_16312_b200 import scenegen
    import oracle
    oracle.build()
    scene, cams = scenegen.make_scene(WORKLOAD, seed=args.seed, n=args.n)
    band = 16
    for s in range(args.warmup):
        oracle_sample(scene, cams[s % len(cams)], (512, 512 + band))
    tot_s, tot_px = 0.0, 0
    for s in range(args.steps):
        secs, npx = oracle_sample(scene, cams[s % len(cams)], (512, 512 + band))
        tot_s += secs
        tot_px += npx
    value = tot_px / tot_s / 1e6
    return {"impl": "reference", "metric": "fwd+bwd Mpixel/s (C5 training step: 8 views, fwd+bwd+allreduce+Adam)",
            "value": round(value, 6), "unit": "Mpixel/s", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": round(1000 * tot_s / args.steps, 3), "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {"workload": "C5: 1M octahedra, SH deg 3, 8 views 1600x1060, training step (views sharded)",
                       "sample_per_step": f"{band} rows x 1600 px of one view (fwd+bwd; a seeded upstream gradient "
                                          f"stands in for the loss gradient), views round-robin"},
            "cpu_baseline": {"value": round(value, 6), "unit": "Mpixel/s", "cores": os.cpu_count(),
                             "kind": "oracle", "sample": f"{band}-row band per step, {args.steps} steps"},
            "e2e": {"value": round(value, 6), "unit": "Mpixel/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}


def free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def relaunch(args):
    """--gpus N > 1 outside torchrun: run this script under torch.distributed.run with N ranks."""
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr=127.0.0.1", f"--master-port={free_port()}", os.path.abspath(__file__)] + sys.argv[1:]
    env = dict(os.environ, OMP_NUM_THREADS=os.environ.get("OMP_NUM_THREADS", "4"))
    return subprocess.call(cmd, env=env)


def dry_run(args, rank, world):
    """Process-group check without GPU work: every rank joins over gloo and contributes its rank."""
    import torch
    import torch.distributed as dist
    if world > 1:
        dist.init_process_group("gloo")
    t = torch.zeros(world, dtype=torch.int64)
    t[rank] = 1 + rank
    if world > 1:
        dist.all_reduce(t)
    from paper_2501_16312_b200 import train
    out = {"dry_run": True, "n_gpus": world, "ranks_seen": [int(x) - 1 for x in t.tolist()],
           "views_per_rank": [train.shard_views(8, r, world) for r in range(world)]}
    if world > 1:
        dist.destroy_process_group()
    if rank == 0:
        print(json.dumps(out), flush=True)


def main():
    args = parse()
    env_world = os.environ.get("WORLD_SIZE")
    if env_world is None and args.gpus > 1:
        sys.exit(relaunch(args))
    world = int(env_world or "1")
    rank = int(os.environ.get("RANK", "0"))
    local_rank = int(os.environ.get("LOCAL_RANK", "0"))
    if world != args.gpus:
        print(json.dumps({"error": f"--gpus {args.gpus} but WORLD_SIZE={world}: refusing to report a number "
                                   f"for a different GPU count"}), flush=True)
        sys.exit(2)
    if args.dry_run:
        return dry_run(args, rank, world)
    if args.impl == "reference":
        out = run_reference(args, rank, world)
        if out is not None:
            print(json.dumps(out), flush=True)
        return
    import torch
    if args.shared_gpu:
        # code-path check only (gloo, every rank on cuda:0): the number it prints is not a bench value
        local_rank = 0
    if torch.cuda.device_count() < local_rank + 1:
        raise SystemExit(f"rank {rank}: {torch.cuda.device_count()} visible GPUs, local rank {local_rank} has none")
    if world > 1:
        import torch.distributed as dist
        if rank == 0:                      # NCCL init lines (rank count, NVLS / ring) on stderr
            os.environ.setdefault("NCCL_DEBUG", "INFO")
            os.environ.setdefault("NCCL_DEBUG_SUBSYS", "INIT")
            os.environ.setdefault("NCCL_DEBUG_FILE", "/dev/stderr")
        torch.cuda.set_device(local_rank)
        if args.dist_backend == "nccl":
            dist.init_process_group("nccl", device_id=torch.device("cuda", local_rank))
        else:
            dist.init_process_group("gloo")
    out, ctx = run_ours(args, rank, world, local_rank)
    if world > 1:
        import torch.distributed as dist
        dist.barrier()
        dist.destroy_process_group()
    if out is None:
        return
    if rank == 0:
        if world == 1 and not args.no_cpu_baseline:
            scene, cams, _ = ctx
            out["cpu_baseline"] = cpu_baseline(scene, cams)
        if args.shared_gpu:
            out["config"]["code_path_check"] = "all ranks on one GPU over gloo: not a bench value"
        print(json.dumps(out), flush=True)


if __name__ == "__main__":
    main()
