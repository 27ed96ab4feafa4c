"""Pins for the oracle's rasterisation: MTIA chords against closed forms, Eq. 1, compositing
algebra and invariants, tiling exactness."""
import math

import numpy as np
import pytest

import oracle
from paper_2501_16312_b200 import scenegen
from tests.helpers import cam, concat, one_prim, oscene

OCTA, TETRA = oracle.OCTA, oracle.TETRA


def render_one(scene, c, kappa=0.0, mode=1, t_stop=0.0, bg=(0, 0, 0), pix=None):
    return oracle.forward(oscene(scene), c, kappa=kappa, mode=mode, t_stop=t_stop, bg=bg, pix=pix)


def chord_image(scene, c):
    """chord = -ln(T)/sigma for a single primitive (T = exp(-sigma chord))."""
    f = render_one(scene, c)
    sig = f.pre.sigma[0]
    return -np.log(f.out.T_final.astype(np.float64)) / sig, f


# ---------------------------------------------------------------- Eq. 1

def test_density_examples():
    # S:82-84 (value corrected: -ln(0.505)/2 = 0.3415984, S:83 prints 0.341549)
    s = one_prim(OCTA, (0, 0, 5), (1, 0, 0, 0), (1.0, 2.0, 3.0), logit=0.0)   # alpha = 0.5, min d = 1
    pre = oracle.preprocess(oscene(s), cam(), kappa=0.0, mode=1)
    assert math.isclose(pre.sigma[0], -math.log(1 - 0.99 * 0.5) / 2.0, rel_tol=1e-14)
    assert math.isclose(pre.sigma[0], 0.3415984, abs_tol=5e-8)
    s = one_prim(OCTA, (0, 0, 5), (1, 0, 0, 0), (0.5, 0.7, 0.9), logit=40.0)  # alpha -> 1, min d = 0.5
    pre = oracle.preprocess(oscene(s), cam(), kappa=0.0, mode=1)
    assert math.isclose(pre.sigma[0], 4.605170, rel_tol=1e-6)
    s = one_prim(OCTA, (0, 0, 5), (1, 0, 0, 0), (0.5, 0.7, 0.9), logit=-80.0)  # alpha -> 0
    pre = oracle.preprocess(oscene(s), cam(), kappa=0.0, mode=1)
    assert pre.sigma[0] < 1e-30


def test_density_scale_covariant():
    s1 = one_prim(TETRA, (0, 0, 5), (1, 0, 0, 0), (0.3, 0.4, 0.5, 0.6), logit=0.7)
    s2 = one_prim(TETRA, (0, 0, 5), (1, 0, 0, 0), (0.6, 0.8, 1.0, 1.2), logit=0.7)
    p1 = oracle.preprocess(oscene(s1), cam(), mode=1)
    p2 = oracle.preprocess(oscene(s2), cam(), mode=1)
    assert math.isclose(p1.sigma[0], 2 * p2.sigma[0], rel_tol=1e-12)


# ---------------------------------------------------------------- chord closed forms

@pytest.mark.parametrize("d", [(0.3, 0.2, 0.25), (0.1, 0.4, 0.15), (0.05, 0.05, 0.3)])
def test_chord_axis_aligned_octahedron(d):
    """On-axis octahedron, identity rotation, depth Z:
    chord(r) = 2 d_z max(0, 1 - |r_x - cx| Z/(fx d_x) - |r_y - cy| Z/(fy d_y))."""
    c = cam(64, 48)
    Z = 4.0
    s = one_prim(OCTA, (0, 0, Z), (1, 0, 0, 0), d, logit=-1.0)
    ch, f = chord_image(s, c)
    fx, fy, cx, cy = (float(c[k]) for k in ("fx", "fy", "cx", "cy"))
    ys, xs = np.mgrid[0:48, 0:64] + 0.5
    ref = 2 * d[2] * np.maximum(0, 1 - np.abs(xs - cx) * Z / (fx * np.float32(d[0]))
                                - np.abs(ys - cy) * Z / (fy * np.float32(d[1])))
    ref *= np.float32(d[2]) / d[2]
    assert np.abs(ch - ref).max() < 1e-6 * 2 * d[2]   # T is stored in fp32


def test_chord_regular_tetrahedron():
    """Regular tetrahedron (equal d, identity rotation): chord = 2 max(0, d/sqrt3 - max(|dx| Z/fx, |dy| Z/fy))."""
    c = cam(64, 48)
    Z, d = 4.0, 0.35
    s = one_prim(TETRA, (0, 0, Z), (1, 0, 0, 0), (d, d, d, d), logit=-1.0)
    ch, f = chord_image(s, c)
    fx, fy, cx, cy = (float(c[k]) for k in ("fx", "fy", "cx", "cy"))
    ys, xs = np.mgrid[0:48, 0:64] + 0.5
    dd = float(np.float32(d))
    ref = 2 * np.maximum(0, dd / math.sqrt(3) - np.maximum(np.abs(xs - cx) * Z / fx, np.abs(ys - cy) * Z / fy))
    assert np.abs(ch - ref).max() < 2e-6 * dd


@pytest.mark.parametrize("seed", range(8))
def test_chord_through_centre_any_rotation(seed):
    """A ray through an octahedron's centre with direction u in its frame: chord = 2 / sum |u_i|/d_i.
    The ray-space centre pixel ray is the camera ray p/|p| (|J^-1 e3| = 1)."""
    rng = np.random.default_rng(seed)
    W, t = scenegen.look_at(rng.normal(0, 1, 3), [0, 0, 6])
    c = cam(64, 48, W=W, t=t)
    Wd, td = np.asarray(W, np.float64), np.asarray(t, np.float64)
    # place the centre exactly on the ray of pixel (20, 30): camera-space p = s * (x, y, 1)
    px, py, depth = 20.5, 30.5, 5.0 + rng.uniform()
    pc = depth * np.array([(px - float(c["cx"])) / float(c["fx"]), (py - float(c["cy"])) / float(c["fy"]), 1.0])
    centre = Wd.T @ (pc - td)
    q = rng.standard_normal(4)
    d = rng.uniform(0.1, 0.3, 3)
    s = one_prim(OCTA, centre.astype(np.float32), q, d, logit=-1.0)
    # recompute the fp32-rounded inputs the oracle actually sees
    cen32 = np.asarray(s["pos"][:, 0], np.float64)
    p = Wd @ cen32 + td
    ch, f = chord_image(s, c)
    qq = np.asarray(s["rot"][:, 0], np.float64)
    qq /= np.linalg.norm(qq)
    w, x, y, z = qq
    R = np.array([[1 - 2 * (y * y + z * z), 2 * (x * y - w * z), 2 * (x * z + w * y)],
                  [2 * (x * y + w * z), 1 - 2 * (x * x + z * z), 2 * (y * z - w * x)],
                  [2 * (x * z - w * y), 2 * (y * z + w * x), 1 - 2 * (x * x + y * y)]])
    u = R.T @ (Wd.T @ (p / np.linalg.norm(p)))
    d32 = np.asarray(s["dist"][:, 0], np.float64)
    ref = 2.0 / np.sum(np.abs(u) / d32)
    # the pixel centre is ~1e-5 px off the fp32 centre: compare with slack for that offset
    assert abs(ch[30, 20] - ref) < 1e-4 * ref


def test_eq1_identity_centre_pixel():
    """a ray through the centre along d_z = min d gives chord 2 min d, hence o = 0.99 alpha."""
    c = dict(cam(64, 48), cx=np.float32(32.5), cy=np.float32(24.5))   # optical axis through pixel (32, 24)
    alpha_logit = 0.3
    s = one_prim(OCTA, (0, 0, 5.0), (1, 0, 0, 0), (0.4, 0.5, 0.2), logit=alpha_logit)
    f = render_one(s, c)
    T = float(f.out.T_final[24, 32])
    alpha = 1 / (1 + math.exp(-alpha_logit))
    assert math.isclose(1 - T, 0.99 * alpha, rel_tol=1e-6)


# ---------------------------------------------------------------- compositing

def test_single_and_two_primitive_algebra():
    c = cam(64, 48)
    a = one_prim(OCTA, (0, 0, 4.0), (1, 0, 0, 0), (0.3, 0.3, 0.2), logit=0.5, rgb_dc=(1.0, -0.5, 0.2))
    b = one_prim(OCTA, (0, 0, 6.0), (1, 0, 0, 0), (0.45, 0.45, 0.3), logit=1.5, rgb_dc=(-1.0, 0.7, 0.4))
    bg = (0.2, 0.3, 0.4)
    fa = render_one(a, c, bg=(0, 0, 0))
    Ta = fa.out.T_final.astype(np.float64)
    rgb_a = fa.pre.rgb[0]
    # one primitive over black: pixel = o c
    assert np.allclose(fa.out.image, (1 - Ta)[None] * rgb_a[:, None, None], atol=1e-7)
    fab = render_one(concat([a, b]), c, bg=bg)
    fb = render_one(b, c)
    o1, o2 = 1 - Ta, 1 - fb.out.T_final.astype(np.float64)
    ref = (o1[None] * rgb_a[:, None, None] + ((1 - o1) * o2)[None] * fab.pre.rgb[1][:, None, None]
           + ((1 - o1) * (1 - o2))[None] * np.asarray(bg)[:, None, None])
    assert np.allclose(fab.out.image, ref, atol=2e-7)


@pytest.mark.parametrize("kind", [OCTA, TETRA])
def test_transmittance_bounds_and_zero_opacity_noop(kind):
    sc, c = scenegen.small_scene(kind, 40, seed=3, width=48, height=40)
    f = oracle.forward(oscene(sc), c, t_stop=0.0)
    assert np.all(f.out.T_final >= 0) and np.all(f.out.T_final <= 1)
    # add 10 zero-opacity primitives: image unchanged
    extra, _ = scenegen.small_scene(kind, 10, seed=4, width=48, height=40)
    extra["opacity"][:] = -200.0
    g = oracle.forward(oscene(concat([sc, extra])), c, t_stop=0.0)
    assert np.allclose(f.out.image, g.out.image, rtol=0, atol=1e-80)    # alpha = sigmoid(-200) ~ 1e-87
    assert np.array_equal(f.out.T_final, g.out.T_final)


@pytest.mark.parametrize("kind", [OCTA, TETRA])
def test_tiling_is_exact(kind):
    """Binning by the canonical tile rect drops no hit: tiled == every primitive per pixel."""
    sc, c = scenegen.small_scene(kind, 60, seed=5, width=70, height=52)
    f = oracle.forward(oscene(sc), c, t_stop=1e-3)
    b = oracle.forward(oscene(sc), c, t_stop=1e-3, brute=True)
    assert np.array_equal(f.out.image, b.out.image)
    assert np.array_equal(f.out.T_final, b.out.T_final)


@pytest.mark.parametrize("kind", [OCTA, TETRA])
def test_early_stop_bound(kind):
    """stopping at T < 1e-3 changes each channel by < 1e-3 (residual transmittance bound)."""
    sc, c = scenegen.small_scene(kind, 80, seed=6, width=48, height=40, opacity_mu=3.0, size=(0.2, 0.6))
    a = oracle.forward(oscene(sc), c, t_stop=1e-3)
    b = oracle.forward(oscene(sc), c, t_stop=0.0)
    assert (a.out.T_final < 1e-3).any()         # the stop is exercised
    assert np.abs(a.out.image - b.out.image).max() < 1e-3


def test_order_only_through_key():
    """Relabelling primitives (a permutation of ids) with distinct keys leaves the image unchanged."""
    sc, c = scenegen.small_scene(OCTA, 50, seed=7, width=48, height=40)
    f = oracle.forward(oscene(sc), c)
    perm = np.random.default_rng(0).permutation(50)
    sp = dict(sc)
    for k in ("pos", "rot", "dist", "sh"):
        sp[k] = sc[k][..., perm]
    sp["opacity"] = sc["opacity"][perm]
    g = oracle.forward(oscene(sp), c)
    assert np.array_equal(f.out.image, g.out.image)


# ---------------------------------------------------------------- binning

def test_binning_worked_examples():
    c = cam(64, 48)
    fx = float(c["fx"])
    # one primitive inside one tile -> 1 entry; one spanning a 2x2 block -> 4 entries
    small = one_prim(OCTA, ((8 - 32) * 5 / fx, (8 - 24) * 5 / fx, 5.0), (1, 0, 0, 0), (0.05, 0.05, 0.05))
    cross = one_prim(OCTA, ((32 - 32) * 6 / fx, (32 - 24) * 6 / fx, 6.0), (1, 0, 0, 0), (0.1, 0.1, 0.1))
    pre = oracle.preprocess(oscene(concat([small, cross])), c, mode=0)
    assert list(pre.tiles_touched) == [1, 4]
    keys, vals, ranges = oracle.bin_tiles(pre, 64, 48)
    assert len(keys) == 5
    # same tile, depths 3 and 5 -> order (3, 5)
    a = one_prim(OCTA, ((8 - 32) * 5 / fx, (8 - 24) * 5 / fx, 5.0), (1, 0, 0, 0), (0.05, 0.05, 0.05))
    b = one_prim(OCTA, ((8 - 32) * 3 / fx, (8 - 24) * 3 / fx, 3.0), (1, 0, 0, 0), (0.05, 0.05, 0.05))
    pre = oracle.preprocess(oscene(concat([a, b])), c, mode=0)
    keys, vals, ranges = oracle.bin_tiles(pre, 64, 48)
    assert list(vals) == [1, 0]


@pytest.mark.parametrize("kind", [OCTA, TETRA])
def test_binning_invariants(kind):
    sc, c = scenegen.edge_scene(kind)
    pre = oracle.preprocess(oscene(sc), c, mode=0)
    keys, vals, ranges = oracle.bin_tiles(pre, c["width"], c["height"])
    assert len(keys) == int(pre.tiles_touched.sum())
    assert np.all(np.diff(keys.astype(np.float64)) >= 0)                 # keys non-decreasing
    k2 = keys[1:] == keys[:-1]
    assert np.all(vals[1:][k2] > vals[:-1][k2])                           # ties by id
    # ranges partition [0, E)
    nz = ranges[ranges[:, 1] > ranges[:, 0]]
    assert nz[0, 0] == 0 and nz[-1, 1] == len(keys) and np.all(nz[1:, 0] == nz[:-1, 1])
    # brute-force enumeration of (primitive, tile) overlaps from the rects
    gx = (c["width"] + 15) // 16
    got = sorted(((int(k >> 32), int(v)) for k, v in zip(keys, vals)))
    ref = sorted((ty * gx + tx, i) for i in range(sc["pos"].shape[1]) if pre.tiles_touched[i]
                 for ty in range(pre.rect[i, 1], pre.rect[i, 3] + 1)
                 for tx in range(pre.rect[i, 0], pre.rect[i, 2] + 1))
    assert got == ref


def test_counters_and_pixel_subset():
    sc, c = scenegen.small_scene(TETRA, 60, seed=9, width=50, height=40)
    full = oracle.forward(oscene(sc), c)
    assert full.out.counters[1] <= full.out.counters[0]      # intersected <= iterated
    assert full.out.counters[0] == int(full.out.n_proc.sum())
    pix = np.array([0, 17, 399, 1234, 1999], np.int32)
    sub = oracle.forward(oscene(sc), c, pix=pix)
    for p in pix:
        y, x = divmod(int(p), 50)
        assert np.array_equal(sub.out.image[:, y, x], full.out.image[:, y, x])
        assert sub.out.n_proc[y, x] == full.out.n_proc[y, x]


# ---------------------------------------------------------------- conditioning bounds

def test_conditioning_bound_closed_form_and_silhouette_growth():
    """The oracle's first-order fp32 error of drgb (test tolerances only): on the centre ray of an
    on-axis octahedron the entry / exit are at -d_z / +d_z from the centre and the depth extent is
    d_z, so dc = 2^-20 (d_z + d_z + 2 d_z) and bnd_rgb_c = |G_c| sigma E dc exactly (T = 1 in
    front, no error carried).  Near the silhouette the bound relative to the pixel's own colour
    gradient grows like 1 / chord (the chord is a difference of two depths that do not shrink)."""
    c = dict(cam(64, 48), cx=np.float32(32.5), cy=np.float32(24.5))
    dz = 0.5
    s = one_prim(OCTA, (0, 0, 5.0), (1, 0, 0, 0), (0.4, 0.6, dz), logit=0.3)
    G = np.zeros((3, 48, 64), np.float32)
    G[:, 24, 32] = (0.5, -1.0, 2.0)
    f, g = oracle.forward_backward(oscene(s), c, G, kappa=0.0, mode=1, t_stop=0.0, bounds=True)
    sig = f.pre.sigma[0]
    chord = 2 * dz
    E = math.exp(-sig * chord)
    dc = 2.0 ** -20 * 4 * dz
    np.testing.assert_allclose(f.out.bnd_rgb[0], np.abs(G[:, 24, 32]) * sig * E * dc, rtol=1e-9)
    assert np.all(f.out.bnd_rgb >= 0) and np.all(f.out.bnd_sigma >= 0) and np.all(f.out.bnd_dv >= 0)
    # relative bound |bnd_rgb / drgb| at the centre vs at a pixel near the footprint's edge
    rel = []
    for x in (32, None):
        G2 = np.zeros((3, 48, 64), np.float32)
        if x is None:   # the last pixel of row 24 still hit (smallest chord along the row)
            ch = chord_image(s, c)[0][24]
            x = int(np.nonzero(ch > 0)[0].max())
        G2[:, 24, x] = 1.0
        f2, _ = oracle.forward_backward(oscene(s), c, G2, kappa=0.0, mode=1, t_stop=0.0, bounds=True)
        rel.append(f2.out.bnd_rgb[0, 0] / abs(f2.out.drgb[0, 0]))
    assert rel[1] > 3 * rel[0]
