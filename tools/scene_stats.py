"""Scene statistics for calibrating the synthetic generator against the paper's counters
(275M iterated / 52M intersected pairs over 1752x1168 -> ~134 / ~25 per pixel).
Runs the CUDA path with count_stats; prints E, iterated and intersected pairs per pixel."""
import argparse
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

from paper_2501_16312_b200 import render, scenegen  # noqa: E402


def stats(cfg, size_scale, opacity_mu, seed=0, views=1):
    scene, cams = scenegen.make_scene(cfg, seed=seed, size_scale=size_scale, opacity_mu=opacity_mu)
    ds = render.DeviceScene(scene)
    r = render.Renderer(ds, cams[:views], count_stats=True)
    img = r.forward()
    torch.cuda.synchronize()
    out = []
    for v in range(views):
        c = r.counters(v)
        W, H = cams[v]["width"], cams[v]["height"]
        it = int(c[8]) | (int(c[9]) << 32)
        hit = int(c[10]) | (int(c[11]) << 32)
        out.append({"E": int(c[0]), "E_per_tile": round(int(c[0]) / r.frames[v].c.tiles_x / r.frames[v].c.tiles_y, 1),
                    "frustum": int(c[3]), "visible": int(c[4]), "iter_px": round(it / (W * H), 2),
                    "hit_px": round(hit / (W * H), 2), "mean_T": round(float(r.frames[v].buf("T_final", W * H, torch.float32).mean()), 3)})
    return out


if __name__ == "__main__":
    ap = argparse.ArgumentParser()
    ap.add_argument("--cfg", default="C5")
    ap.add_argument("--views", type=int, default=1)
    ap.add_argument("--sweep", action="store_true")
    a = ap.parse_args()
    grid = [(s, m) for s in (0.12, 0.15, 0.18, 0.22) for m in (-3.0, -2.0, -1.5, -1.0)] if a.sweep else [(0.5, 0.0)]
    for s, m in grid:
        t = time.time()
        print(json.dumps({"cfg": a.cfg, "size_scale": s, "opacity_mu": m, "views": stats(a.cfg, s, m, views=a.views),
                          "s": round(time.time() - t, 1)}), flush=True)
