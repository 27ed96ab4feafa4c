"""CPU oracle for the LinPrim tile rasterizer (arXiv 2501.16312) -- TEST INFRASTRUCTURE.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s ``cpu_baseline`` /
``--impl reference`` legs may import this package.  The product path
(``paper_2501_16312_b200``) never imports it and shares no code with it.

This module is argument marshalling over ``liblpo.so`` (oracle/lpo.c, plain C,
fp64) plus ``build()``.  Every numeric step lives in lpo.c and cites PAPER.md.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess
from dataclasses import dataclass

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SO = os.path.join(_HERE, "liblpo.so")
_SRCS = [os.path.join(_HERE, f) for f in ("lpo.c", "lpo.h", "lpo_geom.inc")]

OCTA, TETRA = 0, 1
TILE = 16


def build(force: bool = False) -> str:
    """Compile liblpo.so (gcc, IEEE fp32/fp64, no FMA contraction, OpenMP)."""
    newest = max(os.path.getmtime(s) for s in _SRCS)
    if force or not os.path.exists(_SO) or os.path.getmtime(_SO) < newest:
        cmd = ["gcc", "-O2", "-std=c11", "-ffp-contract=off", "-fno-fast-math", "-fexcess-precision=standard",
               "-msse2", "-mfpmath=sse", "-fopenmp", "-fPIC", "-shared", "-Wall", "-Wno-unused-function",
               "-o", _SO + ".tmp", os.path.join(_HERE, "lpo.c"), "-lm"]
        subprocess.run(cmd, check=True)
        os.replace(_SO + ".tmp", _SO)
    return _SO


_lib = None


def lib():
    global _lib
    if _lib is None:
        build()
        _lib = C.CDLL(_SO)
        _lib.lpo_preprocess.restype = C.c_int
        _lib.lpo_bin.restype = C.c_int64
        _lib.lpo_render.restype = C.c_int
        _lib.lpo_preprocess_bwd.restype = C.c_int
    return _lib


class _Scene(C.Structure):
    _fields_ = [("kind", C.c_int32), ("n", C.c_int32), ("sh_degree", C.c_int32),
                ("pos", C.c_void_p), ("rot", C.c_void_p), ("dist", C.c_void_p),
                ("opacity", C.c_void_p), ("sh", C.c_void_p), ("filter3d", C.c_void_p)]


class _Camera(C.Structure):
    _fields_ = [("W", C.c_float * 9), ("t", C.c_float * 3), ("fx", C.c_float), ("fy", C.c_float),
                ("cx", C.c_float), ("cy", C.c_float), ("znear", C.c_float),
                ("width", C.c_int32), ("height", C.c_int32)]


class _Pre(C.Structure):
    _fields_ = [("flag", C.c_void_p), ("tiles_touched", C.c_void_p), ("rect", C.c_void_p),
                ("depth_key", C.c_void_p), ("geom", C.c_void_p), ("canon", C.c_void_p),
                ("sigma", C.c_void_p), ("sigma_den", C.c_void_p), ("rgb", C.c_void_p), ("rgb_raw", C.c_void_p)]


class _RenderCfg(C.Structure):
    _fields_ = [("bg", C.c_float * 3), ("t_stop", C.c_float), ("brute", C.c_int32), ("exact", C.c_int32)]


def _ptr(a):
    return None if a is None else a.ctypes.data


def _f32(a):
    return None if a is None else np.ascontiguousarray(a, dtype=np.float32)


class Scene:
    """Host copy of a primitive-feature SoA (all fp32, component-major)."""

    def __init__(self, kind, pos, rot, dist, opacity, sh, sh_degree, filter3d=None):
        self.kind = int(kind)
        self.pos, self.rot, self.dist = _f32(pos), _f32(rot), _f32(dist)
        self.opacity, self.sh, self.filter3d = _f32(opacity), _f32(sh), _f32(filter3d)
        self.sh_degree = int(sh_degree)
        self.n = self.pos.shape[-1]
        K = 3 if self.kind == OCTA else 4
        ncoef = (self.sh_degree + 1) ** 2
        assert self.pos.shape == (3, self.n) and self.rot.shape == (4, self.n)
        assert self.dist.shape == (K, self.n) and self.opacity.shape == (self.n,)
        assert self.sh.shape == (ncoef, 3, self.n)

    def c(self):
        s = _Scene()
        s.kind, s.n, s.sh_degree = self.kind, self.n, self.sh_degree
        s.pos, s.rot, s.dist = _ptr(self.pos), _ptr(self.rot), _ptr(self.dist)
        s.opacity, s.sh, s.filter3d = _ptr(self.opacity), _ptr(self.sh), _ptr(self.filter3d)
        return s


def camera(cam) -> _Camera:
    """cam: dict with W (3x3), t (3), fx, fy, cx, cy, znear, width, height."""
    c = _Camera()
    c.W[:] = [float(v) for v in np.asarray(cam["W"], np.float32).reshape(9)]
    c.t[:] = [float(v) for v in np.asarray(cam["t"], np.float32).reshape(3)]
    for k in ("fx", "fy", "cx", "cy", "znear"):
        setattr(c, k, float(np.float32(cam[k])))
    c.width, c.height = int(cam["width"]), int(cam["height"])
    return c


@dataclass
class Pre:
    flag: np.ndarray
    tiles_touched: np.ndarray
    rect: np.ndarray
    depth_key: np.ndarray
    geom: np.ndarray
    canon: np.ndarray
    sigma: np.ndarray
    sigma_den: np.ndarray
    rgb: np.ndarray
    rgb_raw: np.ndarray = None     # SH colour before the clamp (clamp-decision margins in the parity tests)

    def c(self):
        p = _Pre()
        for f in ("flag", "tiles_touched", "rect", "depth_key", "geom", "canon", "sigma", "sigma_den", "rgb",
                  "rgb_raw"):
            setattr(p, f, _ptr(getattr(self, f)))
        return p


def preprocess(scene: Scene, cam, kappa=0.1, mode=0, den_override=None, exact=False) -> Pre:
    """Per-primitive geometry (mode 0 canonical fp32, 1 fp64), Eq. 1 sigma and SH colour.
    exact: the "no ray space" variant (App. D): camera-space geometry, perspective bbox, no 2D filter."""
    n = scene.n
    K = 3 if scene.kind == OCTA else 4
    out = Pre(flag=np.zeros(n, np.int32), tiles_touched=np.zeros(n, np.uint32),
              rect=np.zeros((n, 4), np.int32), depth_key=np.zeros(n, np.uint32),
              geom=np.zeros((n, 3 + 3 * K), np.float64), canon=np.zeros((n, 2 + 3 * K), np.float32),
              sigma=np.zeros(n, np.float64), sigma_den=np.zeros(n, np.float64),
              rgb=np.zeros((n, 3), np.float64), rgb_raw=np.zeros((n, 3), np.float64))
    den = None if den_override is None else np.ascontiguousarray(den_override, np.float64)
    s, c, p = scene.c(), camera(cam), out.c()
    rc = lib().lpo_preprocess(C.byref(s), C.byref(c), C.c_float(kappa), C.c_int32(mode), C.c_int32(1 if exact else 0),
                              C.c_void_p(_ptr(den)), C.byref(p))
    assert rc == 0
    return out


def bin_tiles(pre: Pre, width, height, tile_mask=None):
    """(tile|depth, id) binning and ordering.  Returns keys (u64), vals (u32), ranges [T,2] (i64)."""
    n = pre.flag.shape[0]
    gx, gy = (width + TILE - 1) // TILE, (height + TILE - 1) // TILE
    T = gx * gy
    mask = None if tile_mask is None else np.ascontiguousarray(tile_mask, np.uint8)
    ranges = np.zeros((T, 2), np.int64)
    cap = 0
    while True:
        keys = np.zeros(max(cap, 1), np.uint64)
        vals = np.zeros(max(cap, 1), np.uint32)
        E = lib().lpo_bin(C.c_int32(n), C.c_void_p(_ptr(pre.tiles_touched)), C.c_void_p(_ptr(pre.rect)),
                          C.c_void_p(_ptr(pre.depth_key)), C.c_int32(width), C.c_int32(height),
                          C.c_void_p(_ptr(mask)), C.c_void_p(_ptr(keys)), C.c_void_p(_ptr(vals)),
                          C.c_int64(cap), C.c_void_p(_ptr(ranges)))
        if E >= 0:
            return keys[:E], vals[:E], ranges
        if E == -1 and cap > 0:
            raise MemoryError("lpo_bin")
        cap = -E


@dataclass
class RenderOut:
    image: np.ndarray
    T_final: np.ndarray
    n_proc: np.ndarray
    m_stop: np.ndarray
    m_face: np.ndarray
    counters: np.ndarray
    dv: np.ndarray = None
    dsigma: np.ndarray = None
    drgb: np.ndarray = None
    face_margin: np.ndarray = None
    depth: np.ndarray = None       # depth mode: entry distance at cumulative opacity > 0.5, else 0
    m_depth: np.ndarray = None     # min |ln(T_after / 0.5)| over the pixel's hits
    alpha: np.ndarray = None       # alpha mode: 1 - T_final
    # conditioning bounds (bounds=True): first-order fp32 error of drgb / dsigma / dv (lpo.h)
    bnd_rgb: np.ndarray = None
    bnd_sigma: np.ndarray = None
    bnd_dv: np.ndarray = None


def render(scene: Scene, cam, pre: Pre, vals, ranges, bg=(0.0, 0.0, 0.0), t_stop=1e-3,
           pix=None, dL_dimage=None, brute=False, exact=False, bounds=False) -> RenderOut:
    """MTIA rasterisation of the requested pixels (all when pix is None), optional backward."""
    W, H = int(cam["width"]), int(cam["height"])
    n = scene.n
    NV = 6 if scene.kind == OCTA else 4
    cfg = _RenderCfg()
    cfg.bg[:] = [float(b) for b in bg]
    cfg.t_stop = float(t_stop)
    cfg.brute = 1 if brute else 0
    cfg.exact = 1 if exact else 0
    out = RenderOut(image=np.zeros((3, H, W), np.float64), T_final=np.zeros((H, W), np.float64),
                    n_proc=np.zeros((H, W), np.int32), m_stop=np.full((H, W), np.inf),
                    m_face=np.full((H, W), np.inf), counters=np.zeros(2, np.int64),
                    depth=np.zeros((H, W), np.float64), m_depth=np.full((H, W), np.inf))
    pix_a = None if pix is None else np.ascontiguousarray(pix, np.int32)
    npix = 0 if pix_a is None else pix_a.shape[0]
    g = None
    if dL_dimage is not None:
        g = np.ascontiguousarray(dL_dimage, np.float32).reshape(3, H, W)
        out.dv = np.zeros((n, NV, 3), np.float64)
        out.dsigma = np.zeros(n, np.float64)
        out.drgb = np.zeros((n, 3), np.float64)
        out.face_margin = np.full(n, np.inf)
        if bounds:
            out.bnd_rgb = np.zeros((n, 3), np.float64)
            out.bnd_sigma = np.zeros(n, np.float64)
            out.bnd_dv = np.zeros((n, NV, 3), np.float64)
    vals = np.ascontiguousarray(vals, np.uint32)
    ranges = np.ascontiguousarray(ranges, np.int64)
    s, c, p = scene.c(), camera(cam), pre.c()
    rc = lib().lpo_render(C.byref(s), C.byref(c), C.byref(p), C.c_void_p(_ptr(vals)), C.c_void_p(_ptr(ranges)),
                          C.byref(cfg), C.c_void_p(_ptr(pix_a)), C.c_int64(npix),
                          C.c_void_p(_ptr(out.image)), C.c_void_p(_ptr(out.T_final)),
                          C.c_void_p(_ptr(out.n_proc)), C.c_void_p(_ptr(out.m_stop)),
                          C.c_void_p(_ptr(out.m_face)), C.c_void_p(_ptr(g)),
                          C.c_void_p(_ptr(out.dv)), C.c_void_p(_ptr(out.dsigma)),
                          C.c_void_p(_ptr(out.drgb)), C.c_void_p(_ptr(out.face_margin)),
                          C.c_void_p(_ptr(out.counters)), C.c_void_p(_ptr(out.depth)),
                          C.c_void_p(_ptr(out.m_depth)), C.c_void_p(_ptr(out.bnd_rgb)),
                          C.c_void_p(_ptr(out.bnd_sigma)), C.c_void_p(_ptr(out.bnd_dv)))
    assert rc == 0
    out.alpha = 1.0 - out.T_final
    return out


@dataclass
class Grads:
    pos: np.ndarray
    rot: np.ndarray
    dist: np.ndarray
    opacity: np.ndarray
    sh: np.ndarray


def preprocess_bwd(scene: Scene, cam, pre: Pre, r: RenderOut, den_override=None, exact=False) -> Grads:
    n = scene.n
    g = Grads(pos=np.zeros((3, n)), rot=np.zeros((4, n)), dist=np.zeros(scene.dist.shape),
              opacity=np.zeros(n), sh=np.zeros(scene.sh.shape))
    den = None if den_override is None else np.ascontiguousarray(den_override, np.float64)
    s, c, p = scene.c(), camera(cam), pre.c()
    rc = lib().lpo_preprocess_bwd(C.byref(s), C.byref(c), C.byref(p), C.c_int32(1 if exact else 0),
                                  C.c_void_p(_ptr(den)),
                                  C.c_void_p(_ptr(r.dv)), C.c_void_p(_ptr(r.dsigma)), C.c_void_p(_ptr(r.drgb)),
                                  C.c_void_p(_ptr(g.pos)), C.c_void_p(_ptr(g.rot)), C.c_void_p(_ptr(g.dist)),
                                  C.c_void_p(_ptr(g.opacity)), C.c_void_p(_ptr(g.sh)))
    assert rc == 0
    return g


def sh_basis(d):
    """Y[16] and dY/ddir [16,3] of the 3DGS SH basis at unit direction d."""
    Y = np.zeros(16)
    dY = np.zeros((16, 3))
    lib().lpo_sh_basis(C.c_double(d[0]), C.c_double(d[1]), C.c_double(d[2]),
                       C.c_void_p(Y.ctypes.data), C.c_void_p(dY.ctypes.data))
    return Y, dY


# ---------------------------------------------------------------- convenience pipelines

@dataclass
class Forward:
    pre: Pre
    keys: np.ndarray
    vals: np.ndarray
    ranges: np.ndarray
    out: RenderOut


def forward(scene, cam, kappa=0.1, mode=0, bg=(0, 0, 0), t_stop=1e-3, pix=None, den_override=None,
            dL_dimage=None, tile_mask=None, brute=False, exact=False, bounds=False) -> Forward:
    pre = preprocess(scene, cam, kappa=kappa, mode=mode, den_override=den_override, exact=exact)
    keys, vals, ranges = bin_tiles(pre, cam["width"], cam["height"], tile_mask=tile_mask)
    out = render(scene, cam, pre, vals, ranges, bg=bg, t_stop=t_stop, pix=pix, dL_dimage=dL_dimage,
                 brute=brute, exact=exact, bounds=bounds)
    return Forward(pre, keys, vals, ranges, out)


def forward_backward(scene, cam, dL_dimage, kappa=0.1, mode=0, bg=(0, 0, 0), t_stop=1e-3, pix=None,
                     den_override=None, tile_mask=None, exact=False, bounds=False):
    f = forward(scene, cam, kappa=kappa, mode=mode, bg=bg, t_stop=t_stop, pix=pix,
                den_override=den_override, dL_dimage=dL_dimage, tile_mask=tile_mask, exact=exact,
                bounds=bounds)
    g = preprocess_bwd(scene, cam, f.pre, f.out, den_override=den_override, exact=exact)
    return f, g


def mtia(A, B, C_, r):
    """(hit, u, v, d, depth) of the 2-D Moller-Trumbore test for the vertical ray through r."""
    out = np.zeros(4)
    A, B, C_ = (np.ascontiguousarray(x, np.float64) for x in (A, B, C_))
    hit = lib().lpo_mtia(C.c_void_p(A.ctypes.data), C.c_void_p(B.ctypes.data), C.c_void_p(C_.ctypes.data),
                         C.c_double(r[0]), C.c_double(r[1]), C.c_void_p(out.ctypes.data))
    return bool(hit), out[0], out[1], out[2], out[3]


def mtia_grad(A, B, C_, r, u, v, d):
    """App. E: d(depth)/d(v_k) for the three corners, [3][3]."""
    di = np.zeros((3, 3))
    A, B, C_ = (np.ascontiguousarray(x, np.float64) for x in (A, B, C_))
    lib().lpo_mtia_grad(C.c_void_p(A.ctypes.data), C.c_void_p(B.ctypes.data), C.c_void_p(C_.ctypes.data),
                        C.c_double(r[0]), C.c_double(r[1]), C.c_double(u), C.c_double(v), C.c_double(d),
                        C.c_void_p(di.ctypes.data))
    return di


def mtia3(A, B, C_, r):
    """(hit, u, v, det, t) of the 3-D Moller-Trumbore test of the ray t r (origin 0), App. D mode."""
    out = np.zeros(4)
    A, B, C_, r = (np.ascontiguousarray(x, np.float64) for x in (A, B, C_, r))
    hit = lib().lpo_mtia3(C.c_void_p(A.ctypes.data), C.c_void_p(B.ctypes.data), C.c_void_p(C_.ctypes.data),
                          C.c_void_p(r.ctypes.data), C.c_void_p(out.ctypes.data))
    return bool(hit), out[0], out[1], out[2], out[3]


def mtia3_grad(A, B, C_, r):
    """d t / d(A, B, C) [3][3] of the 3-D hit (zeros on a miss)."""
    dt = np.zeros((3, 3))
    A, B, C_, r = (np.ascontiguousarray(x, np.float64) for x in (A, B, C_, r))
    lib().lpo_mtia3_grad(C.c_void_p(A.ctypes.data), C.c_void_p(B.ctypes.data), C.c_void_p(C_.ctypes.data),
                         C.c_void_p(r.ctypes.data), C.c_void_p(dt.ctypes.data))
    return dt


def feature_bounds(scene: Scene, cam, pre: Pre, r: RenderOut, exact=False) -> Grads:
    """Conditioning bounds of the feature gradients (test tolerances only): the render's
    bnd_rgb / bnd_sigma / bnd_dv chained to the features by the same preprocess backward, in
    absolute value."""
    b = RenderOut(image=None, T_final=None, n_proc=None, m_stop=None, m_face=None, counters=None,
                  dv=r.bnd_dv, dsigma=r.bnd_sigma, drgb=r.bnd_rgb)
    g = preprocess_bwd(scene, cam, pre, b, exact=exact)
    return Grads(*(np.abs(getattr(g, k)) for k in ("pos", "rot", "dist", "opacity", "sh")))
