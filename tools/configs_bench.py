"""Per-config measurement of the single-view configs C1-C4 (SURVEY §8d "per-config reporting").

For each config: one view, the C-ABI calls of the hot path timed separately with CUDA events on the
launching stream, L2 flushed (a 2 x L2 write) before every iteration, median over --iters after
--warmup:

  fwd      = lp_preprocess + lp_bin_sort + lp_render_fwd              (render-only frame)
  fwd+bwd  = fwd + lp_raster_bwd + lp_preprocess_bwd                  (seeded upstream G ~ N(0,1)/(3HW))

Prints one JSON line per config (Mpixel/s, FPS, per-call ms, the tile-list / pair counters, the
raster kernels' ALU-model fraction as in bench.py) and with --out appends them to a file.

  python tools/configs_bench.py [C1 C2 C3 C4] [--iters 20] [--warmup 5] [--exact] [--size-mult 0.5 1 2]
                                [--out FILE]
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

import bench  # noqa: E402  (work model, clock sampler)
from paper_2501_16312_b200 import linprim as L  # noqa: E402
from paper_2501_16312_b200 import render, scenegen  # noqa: E402

RENDER_ONLY = {"C4"}        # BASELINE configs[3]: "render-only FPS"


def run(name, iters, warmup, exact, size_mult=1.0, sort_method=None):
    dev = torch.device("cuda", 0)
    scene, cams = scenegen.make_scene(name, seed=0, size_scale=scenegen.DEFAULT_SIZE_SCALE * size_mult)
    cam = cams[0]
    W, H = cam["width"], cam["height"]
    ds = render.DeviceScene(scene, device=dev)
    kw = dict(exact=exact, aa_kernel=0.0 if exact else 0.1)
    # counters pass (untimed)
    rr = render.Renderer(ds, [cam], count_stats=True, **kw)
    rr.forward()
    torch.cuda.synchronize()
    s = rr.counters(0)
    E = int(s[L.LP_CNT_ENTRIES])
    I_ = int(s[8]) | (int(s[9]) << 32)
    X_ = int(s[10]) | (int(s[11]) << 32)
    B_ = int(s[12]) | (int(s[13]) << 32)
    vis = int(s[L.LP_CNT_VISIBLE])
    Wh, A_ = int(s[L.LP_CNT_WARP_HITS]), int(s[L.LP_CNT_TILE_HITS])
    del rr
    rend = render.Renderer(ds, [cam], capacity=int(E * 1.3) + 4096, sync_capacity=False, sort_method=sort_method, **kw)
    st = torch.cuda.current_stream(dev)
    img = torch.empty((1, 3, H, W), dtype=torch.float32, device=dev)
    G = torch.from_numpy(scenegen.upstream_grad(W, H, seed=0)).to(dev).reshape(1, 3, H, W).contiguous()
    l2 = torch.cuda.get_device_properties(dev).L2_cache_size
    flush = torch.empty(2 * l2 // 4 + 1024, dtype=torch.float32, device=dev)
    ca = rend._cams([0])
    fa = render.frames_array(rend.frames)
    bwd = name not in RENDER_ONLY
    names = ["pre", "sort", "fwd"] + (["rbwd", "pbwd"] if bwd else [])

    def once(ev=None, upto=None):
        st = torch.cuda.current_stream(dev)   # the capture stream inside torch.cuda.graph

        def rec(j):
            if ev is not None:
                ev[j].record(st)
        rec(0)
        L.lp_preprocess(ds.prims, ca, rend.cfg, fa, st)
        rec(1)
        if upto == "pre":
            return
        L.lp_bin_sort(ca, fa, st, None)
        rec(2)
        if upto == "sort":
            return
        L.lp_render_fwd(ca, rend.cfg, fa, img[0], st)
        rec(3)
        if upto == "fwd":
            return
        if bwd:
            L.lp_raster_bwd(ca, rend.cfg, fa, G[0], st)
            rec(4)
            L.lp_preprocess_bwd(ds.prims, ca, rend.cfg, fa, ds.grads, st)
            rec(5)

    for _ in range(warmup):
        flush.fill_(1.0)
        once()
    torch.cuda.synchronize()
    c = L.lp_frame_counters(rend.frames[0].c, st)
    assert c[L.LP_CNT_OVERFLOW] == 0, "tile-list capacity overflow"
    evs = [[torch.cuda.Event(enable_timing=True) for _ in range(len(names) + 1)] for _ in range(iters)]
    clocks = bench.ClockSampler(0)
    clocks.start()
    for k in range(iters):
        flush.fill_(1.0)
        once(evs[k])
        ds.grad.zero_()
    torch.cuda.synchronize()
    clocks.stop()
    per = {nm: statistics.median(e[j].elapsed_time(e[j + 1]) for e in evs) for j, nm in enumerate(names)}
    fwd_ms = statistics.median(e[0].elapsed_time(e[3]) for e in evs)
    out = {"workload": name, "kind": "octahedron" if ds.kind == 0 else "tetrahedron", "n_primitives": ds.n,
           "sh_degree": ds.sh_degree, "width": W, "height": H,
           "projection": "no ray space (App. D)" if exact else "EWA ray space", "size_mult": size_mult,
           "l2": "flushed (2 x L2 write) before every iteration", "iters": iters, "warmup": warmup,
           "fwd_ms": round(fwd_ms, 4), "fwd_mpix_s": round(W * H / (fwd_ms * 1e-3) / 1e6, 2),
           "render_fps": round(1000.0 / fwd_ms, 1)}
    if bwd:
        fb_ms = statistics.median(e[0].elapsed_time(e[5]) for e in evs)
        out.update({"fwd_bwd_ms": round(fb_ms, 4), "fwd_bwd_mpix_s": round(W * H / (fb_ms * 1e-3) / 1e6, 2),
                    "iters_per_s": round(1000.0 / fb_ms, 1)})
    out["calls_ms"] = {k: round(v, 4) for k, v in per.items()}
    # the same frame replayed as a CUDA graph (launch gaps of the latency-bound small configs shrink):
    # medians of --iters replays after an L2 flush, graphs of pre | pre+sort | fwd (| fwd+bwd)
    gms = {}
    for upto in ("pre", "sort", "fwd") + (("all",) if bwd else ()):
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g):
            once(upto=None if upto == "all" else upto)
        times = []
        for k in range(iters + 3):
            flush.fill_(1.0)
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(st)
            g.replay()
            e1.record(st)
            torch.cuda.synchronize()
            if k >= 3:
                times.append(e0.elapsed_time(e1))
            ds.grad.zero_()
        gms[upto] = statistics.median(times)
        del g
    out["graph_ms"] = {"pre": round(gms["pre"], 4), "sort": round(gms["sort"] - gms["pre"], 4),
                       "fwd_total": round(gms["fwd"], 4), "fwd_mpix_s": round(W * H / (gms["fwd"] * 1e-3) / 1e6, 2),
                       "sort_share_of_fwd": round((gms["sort"] - gms["pre"]) / gms["fwd"], 3)}
    if bwd:
        out["graph_ms"].update({"fwd_bwd_total": round(gms["all"], 4),
                                "fwd_bwd_mpix_s": round(W * H / (gms["all"] * 1e-3) / 1e6, 2)})
    alu_peak = 148 * 128 * 1965.0 * 1e6
    cnt = {"I": I_, "B": B_, "X": X_, "Wh": Wh, "A": A_}
    # the raster kernels' fractions of the nominal ALU peak under SURVEY §8(d)'s work model and the
    # builder's (bench.raster_work), side by side
    for key, b in (("fwd", False), ("rbwd", True)):
        if key == "rbwd" and not bwd:
            continue
        sec = per[key] * 1e-3
        out[f"raster_{'bwd' if b else 'fwd'}_alu_frac"] = round(bench.raster_work(ds.kind, cnt, b, "survey") / sec / alu_peak, 4)
        out[f"raster_{'bwd' if b else 'fwd'}_alu_frac_builder"] = round(
            bench.raster_work(ds.kind, cnt, b, "builder") / sec / alu_peak, 4)
    out["sort_share_of_fwd"] = round(per["sort"] / fwd_ms, 3)
    out["counters"] = {"tile_list_entries": E, "visible_primitives": vis,
                       "iterated_pairs_per_px": round(I_ / (W * H), 2),
                       "in_bbox_pairs_per_px": round(B_ / (W * H), 2),
                       "intersected_pairs_per_px": round(X_ / (W * H), 2),
                       "warp_hit_pairs": Wh, "tile_hit_pairs": A_}
    out["clocks"] = clocks.summary()
    return out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("configs", nargs="*", default=["C1", "C2", "C3", "C4"])
    ap.add_argument("--iters", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--exact", action="store_true")
    ap.add_argument("--out", default=None)
    ap.add_argument("--sort", default="auto", choices=["auto", "radix", "bucket"],
                    help="lp_frame.sort_method (auto: lp_frame_init's size-based default)")
    ap.add_argument("--size-mult", type=float, nargs="*", default=[1.0],
                    help="primitive size scale multipliers (SURVEY §8d sensitivity sweep: 0.5 1 2)")
    a = ap.parse_args()
    torch.cuda.set_device(0)
    for name in a.configs:
        for sm in a.size_mult:
            r = run(name, a.iters, a.warmup, a.exact, sm,
                    sort_method={"auto": None, "bucket": L.LP_SORT_BUCKET, "radix": L.LP_SORT_RADIX}[a.sort])
            r["sort_method"] = a.sort
            line = json.dumps(r)
            print(line, flush=True)
            if a.out:
                with open(a.out, "a") as f:
                    f.write(line + "\n")
            torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
