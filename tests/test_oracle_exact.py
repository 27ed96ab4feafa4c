"""Pins for the oracle's "no ray space" variant (App. D): per-pixel
perspective rays r = ((x+0.5-cx)/fx, (y+0.5-cy)/fy, 1) against the camera-space faces.

* closed form: an axis-aligned octahedron centred on the optical axis at depth Z, ray (a, b, 1):
  |t a|/dx + |t b|/dy + |t - Z|/dz <= 1 gives t_in = (Z - dz)/(1 - k dz), t_out = (Z + dz)/(1 + k dz)
  with k = |a|/dx + |b|/dy, chord = (t_out - t_in)|r|;
* on the optical axis the chord is 2 min d, so the centre pixel's alpha is 0.99 alpha;
* a regular tetrahedron with a face squarely towards the camera: depth (entry distance) =
  (Z - d/3)|r| over its whole silhouette;
* 3-D Moller-Trumbore against the plane intersection and its gradient against finite differences;
* the full backward against central finite differences of the fp64 forward (every feature);
* tiling exactness: the tiled render equals the brute-force (no tiles) render;
* ray-space vertex error against the exact projection falls with log-log slope 2 (S:761 #10).
"""
import math

import numpy as np
import pytest

import oracle
from paper_2501_16312_b200 import scenegen
from tests.helpers import cam, concat, one_prim, oscene

OCTA, TETRA = oracle.OCTA, oracle.TETRA


def render(scene, c, **kw):
    kw.setdefault("kappa", 0.0)
    kw.setdefault("mode", 1)
    kw.setdefault("t_stop", 0.0)
    return oracle.forward(oscene(scene), c, exact=True, **kw)


def test_axis_aligned_octahedron_closed_form():
    c = cam(64, 48)
    Z, d = 4.0, (0.5, 0.4, 0.3)
    s = one_prim(OCTA, (0, 0, Z), (1, 0, 0, 0), d, logit=-1.0)
    f = render(s, c)
    sig = f.pre.sigma[0]
    chord = -np.log(f.out.T_final) / sig
    fx, fy, cx, cy = (float(c[k]) for k in ("fx", "fy", "cx", "cy"))
    ys, xs = np.mgrid[0:48, 0:64] + 0.5
    a, b = (xs - cx) / fx, (ys - cy) / fy
    dx, dy, dz = (float(np.float32(v)) for v in d)
    k = np.abs(a) / dx + np.abs(b) / dy
    t_in = (Z - dz) / (1 - k * dz)
    t_out = (Z + dz) / (1 + k * dz)
    ref = np.where((1 - k * dz > 0) & (t_out > t_in), (t_out - t_in) * np.sqrt(a * a + b * b + 1), 0.0)
    assert (ref > 0).sum() > 50
    assert np.abs(chord - ref).max() < 1e-12


def test_optical_axis_alpha():
    """one axis-aligned octahedron on the optical axis: centre-pixel alpha = 0.99 alpha."""
    c = dict(cam(64, 48), cx=np.float32(32.5), cy=np.float32(24.5))
    s = one_prim(OCTA, (0, 0, 5.0), (1, 0, 0, 0), (0.4, 0.5, 0.2), logit=0.3)
    T = float(render(s, c).out.T_final[24, 32])
    assert math.isclose(1 - T, 0.99 / (1 + math.exp(-float(np.float32(0.3)))), rel_tol=1e-12)


def test_tetra_face_on_depth():
    c = cam(64, 48)
    Z, d = 5.0, 0.6
    u = np.array([1.0, 1.0, 1.0]) / math.sqrt(3)
    v = np.array([0.0, 0.0, 1.0])
    axis = np.cross(u, v)
    ang = math.atan2(np.linalg.norm(axis), u @ v)
    axis /= np.linalg.norm(axis)
    q = np.array([math.cos(ang / 2), *(math.sin(ang / 2) * axis)])
    s = one_prim(TETRA, (0, 0, Z), q, (d, d, d, d), logit=6.0)
    out = render(s, c).out
    crossed = out.T_final < 0.5
    assert crossed.sum() > 30
    fx, fy, cx, cy = (float(c[k]) for k in ("fx", "fy", "cx", "cy"))
    ys, xs = np.mgrid[0:48, 0:64] + 0.5
    rn = np.sqrt(((xs - cx) / fx) ** 2 + ((ys - cy) / fy) ** 2 + 1)
    assert np.abs(out.depth[crossed] - ((Z - d / 3) * rn)[crossed]).max() < 3e-6


@pytest.mark.parametrize("seed", range(5))
def test_mtia3_plane_and_gradient(seed):
    rng = np.random.default_rng(seed)
    A, B, C_ = (rng.normal(0, 0.3, 3) + np.array([0, 0, 4.0]) for _ in range(3))
    cen = (A + B + C_) / 3
    r = cen / cen[2] + rng.normal(0, 0.0005, 3) * np.array([1, 1, 0])
    hit, u, v, det, t = oracle.mtia3(A, B, C_, r)
    assert hit
    n = np.cross(B - A, C_ - A)
    assert math.isclose(t, (n @ A) / (n @ r), rel_tol=1e-12)
    P = t * r
    assert np.allclose(P, (1 - u - v) * A + u * B + v * C_, atol=1e-12)
    g = oracle.mtia3_grad(A, B, C_, r)
    h = 1e-6
    for k, V in enumerate((A, B, C_)):
        for a in range(3):
            Vp, Vm = V.copy(), V.copy()
            Vp[a] += h
            Vm[a] -= h
            args_p = [A, B, C_]
            args_m = [A, B, C_]
            args_p[k], args_m[k] = Vp, Vm
            fd = (oracle.mtia3(*args_p, r)[4] - oracle.mtia3(*args_m, r)[4]) / (2 * h)
            assert abs(fd - g[k, a]) < 1e-6 * max(1.0, abs(fd)), (k, a, fd, g[k, a])


def _loss(scene, c, G, den, t_stop, bg):
    f = oracle.forward(oscene(scene), c, kappa=0.0, mode=1, t_stop=t_stop, bg=bg, den_override=den, exact=True)
    return float(np.sum(G.astype(np.float64) * f.out.image))


@pytest.mark.parametrize("kind", [OCTA, TETRA])
@pytest.mark.parametrize("seed", [0, 1])
def test_fd_full_backward_exact(kind, seed):
    scene, c = scenegen.small_scene(kind, 5, seed=seed, width=32, height=24, sh_degree=1,
                                    depth=(3.0, 9.0), size=(0.15, 0.5), opacity_mu=0.5)
    G = scenegen.upstream_grad(32, 24, seed=seed)[0]
    bg = (0.1, 0.2, 0.3)
    sc = oscene(scene)
    den = oracle.preprocess(sc, c, kappa=0.0, mode=1, exact=True).sigma_den.copy()
    f, g = oracle.forward_backward(sc, c, G, kappa=0.0, mode=1, t_stop=0.0, bg=bg, den_override=den, exact=True)
    worst = {}
    for name in ("pos", "rot", "dist", "opacity", "sh"):
        arr = scene[name]
        an = getattr(g, name)
        scale = np.abs(an).max()
        flat = arr.reshape(-1)
        errs = []
        for idx in range(flat.size):
            th = float(flat[idx])
            h = max(1e-5 * abs(th), 1e-6)
            old = flat[idx]
            flat[idx] = np.float32(th + h)
            hp = float(flat[idx]) - th
            lp = _loss(scene, c, G, den, 0.0, bg)
            flat[idx] = np.float32(th - h)
            hm = th - float(flat[idx])
            lm = _loss(scene, c, G, den, 0.0, bg)
            flat[idx] = old
            fd = (lp - lm) / (hp + hm)
            a = an.reshape(-1)[idx]
            errs.append(abs(fd - a) / (abs(a) + 1e-4 * scale + 1e-300))
        worst[name] = max(errs)
    assert max(worst.values()) < 2e-5, worst


@pytest.mark.parametrize("kind", [OCTA, TETRA])
def test_tiling_is_exact(kind):
    scene, c = scenegen.small_scene(kind, 200, seed=4, width=80, height=56)
    sc = oscene(scene)
    a = oracle.forward(sc, c, kappa=0.0, mode=0, t_stop=1e-3, exact=True).out
    b = oracle.forward(sc, c, kappa=0.0, mode=0, t_stop=1e-3, exact=True, brute=True).out
    assert np.array_equal(a.image, b.image)


def test_ray_space_vertex_error_is_second_order():
    """S:761 criterion 10: the ray-space vertex c_r + J(v - p) against the exact projection phi(v)
    of the exact-mode camera-space vertex v = p + oc: the screen error falls with log-log slope 2
    as the primitive shrinks (first-order Taylor expansion of phi at p)."""
    c = cam(64, 48)
    fx, fy, cx, cy = (float(c[k]) for k in ("fx", "fy", "cx", "cy"))
    errs = []
    sizes = (0.4, 0.2, 0.1, 0.05)
    for sz in sizes:
        s = one_prim(OCTA, (0.6, -0.3, 3.0), (0.9, 0.3, 0.2, -0.1), (sz, 0.8 * sz, 0.6 * sz), logit=0.5)
        gr = oracle.preprocess(oscene(s), c, kappa=0.0, mode=1).geom[0]
        ge = oracle.preprocess(oscene(s), c, kappa=0.0, mode=1, exact=True).geom[0]
        e = 0.0
        for j in range(3):
            for sgn in (1, -1):
                vr = gr[:2] + sgn * gr[3 + 3 * j:5 + 3 * j]
                v = ge[:3] + sgn * ge[3 + 3 * j:6 + 3 * j]
                ve = np.array([fx * v[0] / v[2] + cx, fy * v[1] / v[2] + cy])
                e = max(e, float(np.abs(vr - ve).max()))
        errs.append(e)
    slopes = [math.log(errs[i] / errs[i + 1]) / math.log(2) for i in range(3)]
    assert all(abs(sl - 2) < 0.2 for sl in slopes), (errs, slopes)


@pytest.mark.parametrize("kind", [OCTA, TETRA])
def test_exact_canonical_matches_numpy_arbiter(kind):
    """The exact-mode canonical fp32 geometry: oracle == NumPy float32, bit for bit."""
    from tests.canonical_np import canonical
    scene, c = scenegen.small_scene(kind, 3000, seed=8, width=123, height=77, depth=(0.6, 9.0), size=(0.05, 1.2))
    pre = oracle.preprocess(oscene(scene), c, kappa=0.0, mode=0, exact=True)
    ref = canonical(scene, c, kappa=0.0, exact=True)
    assert np.array_equal(pre.flag, ref["flag"])
    assert np.array_equal(pre.tiles_touched, ref["tiles_touched"])
    assert np.array_equal(pre.rect, ref["rect"])
    assert np.array_equal(pre.depth_key, ref["depth_key"])
    assert np.array_equal(pre.canon.view(np.uint32), ref["canon"].view(np.uint32))
    # the whole-screen case occurs
    full = (pre.flag == 0) & (pre.tiles_touched == ((123 + 15) // 16) * ((77 + 15) // 16))
    assert full.sum() > 0
