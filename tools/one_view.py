"""One forward + backward of view 0 of a config (default C5) -- the driver for single-kernel ncu captures."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2501_16312_b200 import render, scenegen  # noqa: E402

scene, cams = scenegen.make_scene(sys.argv[1] if len(sys.argv) > 1 else "C5", seed=0)
ds = render.DeviceScene(scene, device=torch.device("cuda", 0))
r = render.Renderer(ds, cams[:1])
for _ in range(2):
    img = r.forward()
    r.backward(torch.rand_like(img))
torch.cuda.synchronize()
print("ok", float(img.mean()))
