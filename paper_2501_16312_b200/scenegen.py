"""Seeded synthetic scenes and cameras.

This module is the ONLY code shared by the CUDA path's tests/bench and the oracle:
it draws random numbers and lays them out as the primitive-feature SoA; it holds
none of the method's arithmetic (no projection, no Eq. 1, no SH evaluation).

Feature layout (fp32, component-major, N contiguous per component), P:111-139:
    pos [3][N], rot [4][N] (w,x,y,z, unnormalised), dist [3|4][N] (raw, > 0),
    opacity [N] (logit), sh [(deg+1)^2][3][N].
Rotations q ~ N(0, I4) are uniform on SO(3) ("uniformly random rotation").
"""
from __future__ import annotations

import math

import numpy as np

OCTA, TETRA = 0, 1

# name: (kind, N, sh_degree, width, height, shape, n_views)   -- BASELINE.json configs[0..4]
CONFIGS = {
    "C1": (OCTA, 1_000, 0, 128, 128, "uniform", 1),
    "C2": (TETRA, 100_000, 3, 1280, 720, "scene", 1),
    "C3": (OCTA, 1_000_000, 3, 1600, 1060, "scene", 1),
    "C4": (TETRA, 3_000_000, 3, 1957, 1091, "scene", 1),
    "C5": (OCTA, 1_000_000, 3, 1600, 1060, "ring", 8),
}

# Calibration knobs: projected size scale and opacity-logit mean.
SIZE_LO, SIZE_HI = 0.002, 0.03
# Calibrated on C5 view 0 (tools/scene_stats.py sweep on B200) to the paper's only published
# counters, ~134 iterated and ~25 intersected (pixel, primitive) pairs per pixel:
# size 0.22 / mu -1.5 gave 152 / 23, size 0.22 / mu -1.0 gave 122 / 19.
DEFAULT_SIZE_SCALE = 0.23
DEFAULT_OPACITY_MU = -1.4


def pinhole(width, height, W=None, t=None, fov_x_deg=60.0, znear=0.2):
    f = (width / 2.0) / math.tan(math.radians(fov_x_deg) / 2.0)
    return {"W": np.eye(3, dtype=np.float32) if W is None else np.asarray(W, np.float32),
            "t": np.zeros(3, np.float32) if t is None else np.asarray(t, np.float32),
            "fx": np.float32(f), "fy": np.float32(f), "cx": np.float32(width / 2.0),
            "cy": np.float32(height / 2.0), "znear": np.float32(znear),
            "width": int(width), "height": int(height)}


def look_at(eye, target, up=(0.0, -1.0, 0.0)):
    """World->camera rotation W and translation t (x_cam = W x + t); camera looks along +z,
    image y grows downward (so world up maps to -y)."""
    eye = np.asarray(eye, np.float64)
    fwd = np.asarray(target, np.float64) - eye
    fwd /= np.linalg.norm(fwd)
    right = np.cross(fwd, np.asarray(up, np.float64))
    right /= np.linalg.norm(right)
    down = np.cross(fwd, right)
    Wm = np.stack([right, down, fwd])          # rows: camera x, y, z axes in world coords
    t = -Wm @ eye
    return Wm.astype(np.float32), t.astype(np.float32)


def ring_cameras(width, height, n_views=8, radius=4.0, elevation_deg=10.0, center=(0.0, 0.0, 0.0)):
    cams = []
    el = math.radians(elevation_deg)
    for v in range(n_views):
        az = 2.0 * math.pi * v / n_views
        eye = np.array(center) + radius * np.array([math.cos(el) * math.sin(az), -math.sin(el),
                                                    -math.cos(el) * math.cos(az)])
        W, t = look_at(eye, center)
        cams.append(pinhole(width, height, W=W, t=t))
    return cams


def _log_uniform(rng, lo, hi, size):
    return np.exp(rng.uniform(math.log(lo), math.log(hi), size))


def _in_frustum(rng, n, cam, z0, z1):
    z = rng.uniform(z0, z1, n)
    sx = rng.uniform(0, cam["width"], n)
    sy = rng.uniform(0, cam["height"], n)
    x = (sx - float(cam["cx"])) * z / float(cam["fx"])
    y = (sy - float(cam["cy"])) * z / float(cam["fy"])
    return np.stack([x, y, z]), z


def _features(rng, kind, n, sh_degree, size, opacity_mu, aniso=3.0):
    K = 3 if kind == OCTA else 4
    rot = rng.standard_normal((4, n))
    a = _log_uniform(rng, 1.0 / aniso, aniso, (K, n))          # per-axis anisotropy, max/min <= aniso^2
    dist = size[None, :] * a
    opacity = rng.normal(opacity_mu, 2.0, n)
    ncoef = (sh_degree + 1) ** 2
    sh = np.zeros((ncoef, 3, n))
    sh[0] = rng.uniform(-1.7, 1.7, (3, n))                       # DC: colour spread over [0, 1]
    for l in range(1, sh_degree + 1):
        sh[l * l:(l + 1) * (l + 1)] = rng.normal(0.0, 0.2 / (l + 1), ((2 * l + 1), 3, n))
    return rot, dist, opacity, sh


def make_scene(name_or_tuple, seed=0, size_scale=DEFAULT_SIZE_SCALE, opacity_mu=DEFAULT_OPACITY_MU, n=None):
    """Return (scene dict, list of camera dicts) for a BASELINE config (C1..C5)."""
    kind, N, deg, W, H, shape, nv = CONFIGS[name_or_tuple] if isinstance(name_or_tuple, str) else name_or_tuple
    if n is not None:
        N = n
    rng = np.random.Generator(np.random.PCG64(seed))
    if shape == "uniform":
        cam = pinhole(W, H)
        pos, _ = _in_frustum(rng, N, cam, 3.0, 8.0)
        K = 3 if kind == OCTA else 4
        rot = rng.standard_normal((4, N))
        dist = _log_uniform(rng, 0.03, 0.3, (K, N))
        opacity = rng.normal(opacity_mu, 2.0, N)
        ncoef = (deg + 1) ** 2
        sh = np.zeros((ncoef, 3, N))
        sh[0] = rng.uniform(-1.7, 1.7, (3, N))
        for l in range(1, deg + 1):
            sh[l * l:(l + 1) * (l + 1)] = rng.normal(0.0, 0.2 / (l + 1), ((2 * l + 1), 3, N))
        cams = [cam]
    elif shape == "scene":
        cam = pinhole(W, H)
        n_obj = int(round(0.6 * N))
        centre = np.array([0.0, 0.0, 6.0])
        obj = centre[:, None] + 0.8 * rng.standard_normal((3, n_obj))
        bgp, _ = _in_frustum(rng, N - n_obj, cam, 8.0, 30.0)
        pos = np.concatenate([obj, bgp], axis=1)
        perm = rng.permutation(N)
        pos = pos[:, perm]
        depth = np.maximum(pos[2], 0.5)
        size = _log_uniform(rng, SIZE_LO, SIZE_HI, N) * depth * size_scale
        rot, dist, opacity, sh = _features(rng, kind, N, deg, size, opacity_mu)
        cams = [cam]
    elif shape == "ring":
        n_obj = int(round(0.6 * N))
        obj = 0.8 * rng.standard_normal((3, n_obj))
        nb = N - n_obj
        dirs = rng.standard_normal((3, nb))
        dirs /= np.linalg.norm(dirs, axis=0, keepdims=True)
        bgp = dirs * rng.uniform(8.0, 30.0, nb)[None, :]
        pos = np.concatenate([obj, bgp], axis=1)[:, rng.permutation(N)]
        depth = np.linalg.norm(pos, axis=0) + 4.0
        size = _log_uniform(rng, SIZE_LO, SIZE_HI, N) * depth * size_scale
        rot, dist, opacity, sh = _features(rng, kind, N, deg, size, opacity_mu)
        cams = ring_cameras(W, H, nv)
    else:
        raise ValueError(shape)
    scene = {"kind": kind, "sh_degree": deg,
             "pos": pos.astype(np.float32), "rot": rot.astype(np.float32),
             "dist": dist.astype(np.float32), "opacity": opacity.astype(np.float32),
             "sh": sh.astype(np.float32)}
    return scene, cams


def small_scene(kind, n, seed=0, width=64, height=48, sh_degree=3, depth=(3.0, 8.0), size=(0.05, 0.4),
                opacity_mu=0.0, aniso=3.0):
    """Random small scene for parity / finite-difference tests (well in front of the camera)."""
    rng = np.random.Generator(np.random.PCG64(seed))
    cam = pinhole(width, height)
    pos, z = _in_frustum(rng, n, cam, *depth)
    sz = _log_uniform(rng, size[0], size[1], n)
    rot, dist, opacity, sh = _features(rng, kind, n, sh_degree, sz, opacity_mu, aniso=aniso)
    scene = {"kind": kind, "sh_degree": sh_degree,
             "pos": pos.astype(np.float32), "rot": rot.astype(np.float32),
             "dist": dist.astype(np.float32), "opacity": opacity.astype(np.float32),
             "sh": sh.astype(np.float32)}
    return scene, cam


def edge_scene(kind, seed=0, width=77, height=45, sh_degree=1):
    """Edge cases for binning parity: tile-border stragglers, off-screen, behind the camera,
    sub-pixel, huge, alpha ~ 0, exact duplicate depths, zero quaternion, d <= 0, NaN."""
    scene, cam = small_scene(kind, 64, seed=seed, width=width, height=height, sh_degree=sh_degree)
    K = 3 if kind == OCTA else 4
    rng = np.random.Generator(np.random.PCG64(seed + 1000))
    p, q, d, o = scene["pos"], scene["rot"], scene["dist"], scene["opacity"]
    f = float(cam["fx"])
    # primitives centred exactly on tile borders (x = 16k, y = 16m) at depth 5
    for j, (sx, sy) in enumerate([(16, 16), (32, 16), (48, 32), (64, 16), (0, 0)]):
        p[:, j] = [(sx - float(cam["cx"])) * 5.0 / f, (sy - float(cam["cy"])) * 5.0 / f, 5.0]
    p[:, 5] = [50.0, 0.0, 5.0]             # far off-screen right
    p[:, 6] = [0.0, 0.0, -3.0]             # behind the camera
    p[:, 7] = [0.0, 0.0, 0.19]             # inside znear
    d[:, 8] = 1e-4                          # sub-pixel
    d[:, 9] = 10.0                          # huge (covers every tile)
    p[:, 9] = [0.0, 0.0, 12.0]
    o[10] = -40.0                           # alpha ~ 0
    p[:, 12] = p[:, 11]                     # exact duplicate depth (tie broken by id)
    q[:, 13] = 0.0                          # zero quaternion -> invalid
    d[0, 14] = 0.0                          # d <= 0 -> invalid
    d[1, 15] = -1.0
    p[0, 16] = np.nan                       # NaN -> invalid
    q[:, 17] = [1.0, 0.0, 0.0, 0.0]         # identity rotation (axis-aligned faces)
    q[:, 18] = [math.cos(math.pi / 8), 0.0, math.sin(math.pi / 8), 0.0]   # 45 deg about y
    return scene, cam


def upstream_grad(width, height, seed=0, n_views=1):
    """Seeded dL/dimage ~ N(0,1)/(3HW)."""
    rng = np.random.Generator(np.random.PCG64(seed + 7))
    g = rng.standard_normal((n_views, 3, height, width)) / (3.0 * width * height)
    return g.astype(np.float32)
