"""Drive lp_loss_grad on the C5 image batch (8 x 3 x 1060 x 1600) -- for kernel profiling / timing; the fused
kernel by default, the split path (a G-map workspace) with LOSS_SPLIT=1."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2501_16312_b200 import linprim as L  # noqa: E402

V, H, W = 8, 1060, 1600
x = torch.rand(V, 3, H, W, device="cuda")
y = (0.5 * x + 0.5 * torch.rand_like(x)).contiguous()
d = torch.empty_like(x)
ws = torch.empty(3 * x.numel(), device="cuda") if os.environ.get("LOSS_SPLIT") == "1" else None
loss = torch.zeros(1, device="cuda")
st = torch.cuda.current_stream()
for _ in range(3):
    L.lp_loss_grad(x, y, d, loss, 0.2, 1.0 / x.numel(), st, workspace=ws)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record(st)
for _ in range(20):
    L.lp_loss_grad(x, y, d, loss, 0.2, 1.0 / x.numel(), st, workspace=ws)
e1.record(st)
torch.cuda.synchronize()
print("loss kernel ms per 8-view batch", e0.elapsed_time(e1) / 20)
x1, y1, d1 = x[:1].contiguous(), y[:1].contiguous(), d[:1].contiguous()
for _ in range(3):
    L.lp_loss_grad(x1, y1, d1, loss, 0.2, 1.0 / x1.numel(), st, workspace=ws)
e0.record(st)
for _ in range(50):
    L.lp_loss_grad(x1, y1, d1, loss, 0.2, 1.0 / x1.numel(), st, workspace=ws)
e1.record(st)
torch.cuda.synchronize()
print("loss kernel ms per view (3 planes)", e0.elapsed_time(e1) / 50)
