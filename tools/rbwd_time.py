"""Kernel-variant timing (measurement tool, run under gpurun): C5 view(s), one forward, then the
raster forward and the raster backward each timed alone with CUDA events (20 reps after 3 warm-up,
L2 not flushed between reps).  LP_LIB selects the library build; prints one JSON line."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2501_16312_b200 import linprim as L, render, scenegen  # noqa: E402

cfgname = sys.argv[1] if len(sys.argv) > 1 else "C5"
nv = int(sys.argv[2]) if len(sys.argv) > 2 else 2
scene, cams = scenegen.make_scene(cfgname, seed=0)
ds = render.DeviceScene(scene, device=torch.device("cuda", 0))
r = render.Renderer(ds, cams[:nv])
img = r.forward()
g = torch.randn_like(img) / img[0].numel()
st = r.stream()


def timeit(fn, reps=20):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(st)
    for _ in range(reps):
        fn()
    e1.record(st)
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps


out = {"lib": os.path.basename(os.environ.get("LP_LIB", "liblinprim.so")), "cfg": cfgname, "views": nv}
views = list(range(nv))
fa = render.frames_array(r.frames)
out["rbwd_ms_per_view"] = round(timeit(lambda: L.lp_raster_bwd(r._cams(views), r.cfg, fa, g, st)) / nv, 4)
out["fwd_ms_per_view"] = round(timeit(lambda: r.render_views(img, views)) / nv, 4)
print(json.dumps(out))
