"""GPU-vs-oracle parity helpers (test-only).  Both sides get the same seeded inputs; the oracle
supplies the decision margins used for masking."""
from __future__ import annotations

import numpy as np

import oracle
from tests.helpers import oscene

STOP_MARGIN = 1e-4      # |ln(T/t_stop)| below this: the stop index may flip -> pixel masked
FACE_MARGIN = 2e-5      # min barycentric below this: entry/exit face may switch -> primitive flagged
IMG_TOL = 1e-4          # north_star: images within 1e-4 max abs (fp32)
GRAD_RTOL = 1e-3        # north_star: gradients within 1e-3 relative ...
GRAD_ATOL_REL = 1e-5    # ... or 1e-5 absolute, in units of the group's largest |gradient|
MAX_FLAGGED_FRAC = 2e-2  # face-switch-flagged primitives allowed (FACE_MARGIN 2e-5 flags 0.5-1.4 % at full size)
MAX_MASKED_FRAC = 2e-3   # stop-margin pixels allowed (SURVEY §8c-5 expects ~2e-4 of terminating pixels)


LOG = []    # parity counts of this session (printed by tests/conftest.py)


def log(name, **kw):
    LOG.append(dict(test=name, **kw))


def gpu_run(scene, cams, G=None, kappa=0.1, t_stop=1e-3, bg=(0.0, 0.0, 0.0), with_canon=True, capacity=None,
            count_stats=True, filter3d=None, sort_method=None, exact=False, deterministic=False):
    import torch

    from paper_2501_16312_b200 import render
    ds = render.DeviceScene(scene, filter3d=filter3d)
    r = render.Renderer(ds, cams, aa_kernel=kappa, t_stop=t_stop, bg=bg, with_canon=with_canon,
                        capacity=capacity, count_stats=count_stats, sort_method=sort_method, exact=exact,
                        deterministic=deterministic)
    img = r.forward()
    if G is not None:
        r.backward(torch.as_tensor(G, device="cuda").reshape(img.shape))
    torch.cuda.synchronize()
    return ds, r, img


def frame_arrays(r, v, n, K):
    f = r.frames[v]
    import torch
    W, H = f.c.width, f.c.height
    cnt = r.counters(v)
    E = int(cnt[0])
    out = {
        "tiles_touched": f.buf("tiles_touched", n, torch.int32).cpu().numpy().view(np.uint32),
        "rect": f.buf("rect", 4 * n, torch.int16).cpu().numpy().view(np.uint16).reshape(n, 4).astype(np.int32),
        "depth_key": f.buf("depth_key", n, torch.int32).cpu().numpy().view(np.uint32),
        "E": E,
        "sorted_val": f.buf("sorted_val", E, torch.int32).cpu().numpy().view(np.uint32),
        "sorted_tile": f.buf("sorted_tile", E, torch.int32).cpu().numpy().view(np.uint32),
        "ranges": f.buf("ranges", 2 * f.c.tiles_x * f.c.tiles_y, torch.int32).cpu().numpy().view(np.uint32).reshape(-1, 2),
        "T_final": f.buf("T_final", W * H, torch.float32).cpu().numpy().reshape(H, W),
        "n_proc": f.buf("n_proc", W * H, torch.int32).cpu().numpy().reshape(H, W),
        "counters": cnt,
    }
    if f.c.canon:
        out["canon"] = f.buf("canon", n * (2 + 3 * K), torch.float32).cpu().numpy().reshape(n, 2 + 3 * K)
    return out


def grad_close(name, got, ref, flagged=None, rtol=GRAD_RTOL, atol_rel=GRAD_ATOL_REL, loose=1e-1, bound=None,
               exclude=None):
    """Element-wise |got - ref| <= rtol |ref| + atol_rel * max|ref| (+ bound: the oracle's first-order
    fp32 conditioning error of that element); flagged primitives (last axis) only at the
    loose bound; excluded elements (a decision within rounding, both outcomes valid) are not compared.
    Returns (ok, worst ratio, report, elements that needed the conditioning term)."""
    got = np.asarray(got, np.float64)
    ref = np.asarray(ref, np.float64)
    scale = np.abs(ref).max() if ref.size else 0.0
    if scale == 0.0:
        return (np.abs(got).max() == 0.0 if got.size else True), 0.0, f"{name}: all zero", 0
    base = rtol * np.abs(ref) + atol_rel * scale
    tol = base if bound is None else base + np.asarray(bound, np.float64)
    err = np.abs(got - ref)
    ratio = err / tol
    n_cond = int(((err > base) & (err <= tol)).sum())
    if flagged is not None and flagged.any():
        lt = loose * (np.abs(ref) + 1e-2 * scale)
        ratio[..., flagged] = (err / lt)[..., flagged]
    if exclude is not None:
        ratio[exclude] = 0.0
    worst = float(ratio.max())
    idx = np.unravel_index(int(np.argmax(ratio)), ratio.shape)
    return worst <= 1.0, worst, (f"{name}: worst {worst:.3g} at {idx} got {got[idx]:.6g} ref {ref[idx]:.6g} "
                                 f"scale {scale:.3g} bound {0.0 if bound is None else np.asarray(bound)[idx]:.3g}"), n_cond


# ray-space centre / offsets this far from the pixels (in pixels): the fp32 pixel offsets r - c_r of the
# primitive carry >= 2^-10 px of rounding, which its moment -> vertex chain (M^-1 of offsets ~1e5 px)
# amplifies; such primitives (near the camera plane, off-screen centres) are flagged
SCREEN_SCALE = 8192.0


def screen_flags(pre, exact=False):
    """Primitives whose ray-space geometry spans >= SCREEN_SCALE pixels (ray-space mode only)."""
    if exact:
        return np.zeros(len(pre.flag), bool)
    K = (pre.geom.shape[1] - 3) // 3
    xy = [np.abs(pre.geom[:, 0]), np.abs(pre.geom[:, 1])]
    for j in range(K):
        xy += [np.abs(pre.geom[:, 3 + 3 * j]), np.abs(pre.geom[:, 4 + 3 * j])]
    return (np.max(xy, axis=0) >= SCREEN_SCALE) & (pre.flag == 0)


CLAMP_MARGIN = 1e-6     # |SH colour before max(0, .)| below this: the clamp may flip in fp32 (both valid; seen: 9.5e-9)


def check_gradients(gd, g, gb, pre, flagged, loose=1e-1, clamp=None):
    """All five feature-gradient groups of the CUDA path (gd, torch) against the oracle's (g), with
    the oracle's conditioning bounds gb (oracle.feature_bounds, or None).  A colour channel whose
    clamp decision is within rounding of 0 is excluded from the SH comparison and its primitive
    flagged (the SH direction term of its position gradient flips with it).
    Returns (worst ratio per group, report strings, elements that needed the conditioning term,
    clamp-margin channels); asserts nothing.  clamp: precomputed [n, 3] clamp-margin mask (a multi-view
    step: the union over views), else taken from pre.rgb_raw."""
    if clamp is None:
        clamp = np.abs(pre.rgb_raw) < CLAMP_MARGIN
        clamp &= (pre.flag == 0)[:, None]
    fl = flagged | clamp.any(1)
    worst, reps, n_cond = {}, [], 0
    ok_all = True
    for name, fgrp in (("pos", fl), ("rot", fl), ("dist", fl), ("opacity", None), ("sh", None)):
        ref = getattr(g, name)
        got = gd[name].cpu().numpy().reshape(ref.shape)
        bnd = getattr(gb, name) if gb is not None else None
        excl = np.broadcast_to(clamp.T[None], ref.shape) if name == "sh" else None
        ok, worst[name], rep, nc = grad_close(name, got, ref, fgrp, loose=loose, bound=bnd, exclude=excl)
        ok_all &= ok
        reps.append(rep)
        n_cond += nc
    return ok_all, worst, reps, n_cond, int(clamp.sum())
