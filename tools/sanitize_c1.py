"""One C1 forward + backward (ray space, deterministic, no-ray-space) and one small C5 TrainStep,
for compute-sanitizer (memcheck / racecheck / synccheck) runs: profiles/round2/sanitizer_*.txt."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2501_16312_b200 import render, scenegen, step as S  # noqa: E402

scene, cams = scenegen.make_scene("C1", seed=0)
G = torch.from_numpy(scenegen.upstream_grad(128, 128, seed=0)).cuda()
for kw in (dict(), dict(deterministic=True), dict(exact=True, aa_kernel=0.0)):
    ds = render.DeviceScene(scene)
    r = render.Renderer(ds, cams, count_stats=True, **kw)
    img = r.forward(depth=True, alpha=True)[0]
    r.backward(G)
    torch.cuda.synchronize()
    print(kw, "image sum", float(img.sum()), "grad |max|", float(ds.grad.abs().max()))
sc, cc = scenegen.make_scene("C5", seed=0, n=2000)
f = np.float32(32 / np.tan(np.deg2rad(30.0)))
cc = [dict(c, width=64, height=48, cx=np.float32(32), cy=np.float32(24), fx=f, fy=f) for c in cc]
ds = S.device_scene(sc, "cuda")
ts = S.TrainStep(ds, cc, 8, targets=torch.rand((8, 3, 48, 64), device="cuda"))
ts.run(0)
torch.cuda.synchronize()
print("train step ok, loss", float(ts.loss_buf[0]))
