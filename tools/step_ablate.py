"""Marginal cost of each stage inside the overlapped C5 step (measurement tool, run under gpurun):
the TrainStep timed as is, then with one C-ABI call replaced by a no-op (after warm-up, so the frames
keep valid lists).  The differences say how much of each stage is exposed; the ablated numbers are
not bench values."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2501_16312_b200 import linprim as L, render, scenegen, step as S  # noqa: E402

scene, cams = scenegen.make_scene("C5", seed=0)
dev = torch.device("cuda", 0)
ds = S.device_scene(scene, dev)
rr = render.Renderer(ds, cams, count_stats=True)
tg = rr.forward().clone()
E = max(int(rr.counters(i)[L.LP_CNT_ENTRIES]) for i in range(len(cams)))
del rr
ts = S.TrainStep(ds, cams, len(cams), targets=tg, capacity=int(E * 1.3) + 4096, loss_slots=512)
st = ts.st


snap = (ds.flat.clone(), ts.m.clone(), ts.v.clone())


def timed(k=10, w=3, tag=""):
    # every measurement starts from the same scene and optimizer state (Adam moves the scene, and
    # the step time with it)
    ds.flat.copy_(snap[0])
    ts.m.copy_(snap[1])
    ts.v.copy_(snap[2])
    for i in range(w):
        ts.run(i % 256)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(st)
    for i in range(k):
        ts.run((w + i) % 256)
    e1.record(st)
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / k


# binning: record each frame's sorted-list pointers during a real step, replay them when ablated
_sorted = {}
_real_bin_sort = L.lp_bin_sort


def _recording_bin_sort(cams, frames, stream, n_entries=None):
    r = _real_bin_sort(cams, frames, stream, n_entries)
    _sorted[id(frames)] = (frames[0].sorted_tile, frames[0].sorted_val)
    return r


def _skipped_bin_sort(cams, frames, stream, n_entries=None):
    frames[0].sorted_tile, frames[0].sorted_val = _sorted[id(frames)]
    return 0


L.lp_bin_sort = _recording_bin_sort
timed()
names = [a for a in sys.argv[1:] if a != "none"] if sys.argv[1:] else ["lp_bin_sort", "lp_loss_grad", "lp_raster_bwd", "lp_preprocess", "lp_preprocess_bwd_assign",
                         "lp_adam_step"]
res = {"full": []}
for rep in range(3):   # interleaved repeats, minimum kept (the step time drifts by ~0.5 ms between runs)
    res["full"].append(timed(k=20))
    for nm in names:
        orig = getattr(L, nm)
        setattr(L, nm, _skipped_bin_sort if nm == "lp_bin_sort" else (lambda *a, **k: 0))
        try:
            res.setdefault("no_" + nm, []).append(timed(k=20))
        finally:
            setattr(L, nm, orig)
out = {k: round(min(v), 4) for k, v in res.items()}
out.update({"spread_full": [round(x, 3) for x in res["full"]]})
print(json.dumps(out))
