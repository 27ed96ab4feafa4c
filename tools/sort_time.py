"""Binning-method timing (measurement tool, run under gpurun): per config and sort method, the
preprocess alone and preprocess + lp_bin_sort of view 0, CUDA events, median of 20 reps after 3
warm-up (stream launches, L2 not flushed).  LP_LIB selects the library build; one JSON line each."""
import json
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2501_16312_b200 import linprim as L, render, scenegen  # noqa: E402

for cfgname in (sys.argv[1:] or ["C3", "C5"]):
    scene, cams = scenegen.make_scene(cfgname, seed=0)
    ds = render.DeviceScene(scene, device=torch.device("cuda", 0))
    for method in (L.LP_SORT_BUCKET, L.LP_SORT_RADIX):
        r = render.Renderer(ds, cams[:1], sort_method=method)
        img = r.forward()
        st = r.stream()
        ca = r._cams([0])

        def pre():
            fa = render.frames_array([r.frames[0]])
            L.lp_preprocess(ds.prims, ca, r.cfg, fa, st)
            render._store_back([r.frames[0]], fa)

        def pre_sort():
            fa = render.frames_array([r.frames[0]])
            L.lp_preprocess(ds.prims, ca, r.cfg, fa, st)
            L.lp_bin_sort(ca, fa, st, None)
            render._store_back([r.frames[0]], fa)

        def pre_sort_fwd():
            pre_sort()
            r.render_views(img2, [0])

        img2 = torch.empty_like(img)
        res = {}
        for name, fn in (("pre", pre), ("pre_sort", pre_sort), ("pre_sort_fwd", pre_sort_fwd)):
            ts = []
            for k in range(23):
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record(st)
                fn()
                e1.record(st)
                torch.cuda.synchronize()
                if k >= 3:
                    ts.append(e0.elapsed_time(e1))
            res[name] = statistics.median(ts)
        # correctness of the timed frame: the forward after the last binning still renders the same image
        r.render_views(img2, [0])
        torch.cuda.synchronize()
        same = bool(torch.equal(img, img2))
        print(json.dumps({"lib": os.path.basename(os.environ.get("LP_LIB", "liblinprim.so")), "cfg": cfgname,
                          "method": ["bucket", "radix"][method],
                          "pre_ms": round(res["pre"], 4), "sort_ms": round(res["pre_sort"] - res["pre"], 4),
                          "sort_fwd_ms": round(res["pre_sort_fwd"] - res["pre"], 4),
                          "E": int(r.counters(0)[0]), "image_unchanged": same}), flush=True)
        del r
