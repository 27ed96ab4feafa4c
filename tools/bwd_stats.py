"""Warp-level event counts of the raster backward on C5 view 0 (needs a -DLP_BWD_STATS build)."""
import ctypes
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2501_16312_b200 import linprim as L, render, scenegen  # noqa: E402

scene, cams = scenegen.make_scene(sys.argv[1] if len(sys.argv) > 1 else "C5", seed=0)
ds = render.DeviceScene(scene, device=torch.device("cuda", 0))
r = render.Renderer(ds, cams[:1])
print("scene ready", flush=True)
img = r.forward()
torch.cuda.synchronize()
print("forward done", flush=True)
g = torch.rand_like(img)
f = L._lib.lp_debug_bwd_stats
out = (ctypes.c_ulonglong * 48)()
torch.cuda.synchronize()
f(out, 1)
r.backward(g)
torch.cuda.synchronize()
f(out, 0)
px = cams[0]["width"] * cams[0]["height"]
warps = px / 64
names = ["sublist", "any_bbox", "hit", "hit_lanes", "smem_red", "bbox_lanes"]
for i, n in enumerate(names):
    print(f"{n:12s} {out[i]:>14d}  per-warp {out[i] / warps:10.1f}")
print("hit lanes per reduction", out[3] / max(out[2], 1), " smem share", out[4] / max(out[2], 1))
print("reductions with both pixel rows hit", out[6] / max(out[2], 1), " hit pixels per reduction", out[7] / max(out[2], 1))
print("8x8 warps: (warp, entry) iterations", out[2], " active pixel rows (of 2)", out[2] + out[6])
print("16x8 halves, 4 pixels per lane: iterations", out[41], " active pixel rows (of 4)", out[42],
      " rows per iteration", out[42] / max(out[41], 1))
hist = [out[8 + h] for h in range(33)]
tot = max(sum(hist), 1)
print("h histogram (share of reductions):", " ".join(f"{h}:{hist[h] / tot:.3f}" for h in range(1, 33)))
