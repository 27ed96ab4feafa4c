"""CPU oracle of the population-control inputs on the hot path -- TEST
INFRASTRUCTURE, fp64 NumPy.  Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s oracle
legs may import this.

* 3D smoothing filter size ("limit how small primitives can become based on visibility
  from the training views", reading 26):
      s_3d = kappa * min over training cameras that see the primitive of (camera-space depth / fx),
  a camera "sees" the centre c when p = W c + t has p_z > znear and its projection
  (fx p_x/p_z + cx, fy p_y/p_z + cy) lies inside [0, width] x [0, height]; a primitive no camera
  sees takes kappa |p| / fx of the camera nearest to it (smallest |p|).
* densification statistics ("primitives that have large view-space positional
  gradients"): per view, |dL/d c_r.xy| -- the norm of the gradient with respect to the ray-space
  centre's screen position, i.e. of the sum over the vertices of the ray-space vertex gradients
  (the vertices are c_r + offsets) -- and a visibility count (views with tiles_touched > 0).
"""
from __future__ import annotations

import numpy as np


def camera_space(pos, cam):
    """p = W c + t for all centres (pos [3, n]) -> [3, n] fp64."""
    W = np.asarray(cam["W"], np.float64).reshape(3, 3)
    t = np.asarray(cam["t"], np.float64).reshape(3, 1)
    return W @ np.asarray(pos, np.float64) + t


def sees(pos, cam):
    p = camera_space(pos, cam)
    z = p[2]
    ok = z > float(cam["znear"])
    zs = np.where(ok, z, 1.0)
    u = float(cam["fx"]) * p[0] / zs + float(cam["cx"])
    v = float(cam["fy"]) * p[1] / zs + float(cam["cy"])
    return ok & (u >= 0) & (u <= float(cam["width"])) & (v >= 0) & (v <= float(cam["height"])), p


def filter3d(pos, cams, kappa):
    """s_3d [n] (fp64) for centres pos [3, n] and a list of camera dicts."""
    n = np.asarray(pos).shape[1]
    best = np.full(n, np.inf)
    near_d = np.full(n, np.inf)
    near_v = np.zeros(n)
    for cam in cams:
        vis, p = sees(pos, cam)
        fx = float(cam["fx"])
        best = np.where(vis, np.minimum(best, p[2] / fx), best)
        dist = np.sqrt((p * p).sum(0))
        closer = dist < near_d
        near_v = np.where(closer, dist / fx, near_v)
        near_d = np.where(closer, dist, near_d)
    return kappa * np.where(np.isfinite(best), best, near_v)


def mean2d_norm(dv):
    """|dL/d c_r.xy| per primitive from ray-space vertex gradients dv [n, V, 3] of ONE view."""
    g = np.asarray(dv, np.float64)[:, :, :2].sum(axis=1)
    return np.sqrt((g * g).sum(axis=1))
