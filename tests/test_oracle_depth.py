"""Pins for the oracle's depth / alpha modes (App. B: "the predicted depth
is defined as the distance to the first primitive along the viewing ray where cumulative opacity
exceeds 0.5"; reading 24).  Closed forms from elementary geometry:
  * axis-aligned octahedron on the optical axis: entry depth Z - d_z (1 - |dx| Z/(fx d_x) - |dy| Z/(fy d_y));
  * a regular tetrahedron / octahedron turned so one face squarely faces the camera: the entry
    depth is the face's distance, Z - d/3 (tetrahedron inradius) or Z - d/sqrt(3) (octahedron);
  * the 0.5 rule picks the FIRST primitive after which 1 - T > 0.5, never an earlier one.
"""
import math

import numpy as np
import pytest

import oracle
from tests.helpers import cam, concat, one_prim, oscene

OCTA, TETRA = oracle.OCTA, oracle.TETRA


def render(scene, c, t_stop=0.0):
    return oracle.forward(oscene(scene), c, kappa=0.0, mode=1, t_stop=t_stop).out


def quat_turning(u, v):
    """Unit quaternion (w, x, y, z) of the rotation taking unit vector u to unit vector v."""
    u = np.asarray(u, np.float64) / np.linalg.norm(u)
    v = np.asarray(v, np.float64) / np.linalg.norm(v)
    axis = np.cross(u, v)
    s = np.linalg.norm(axis)
    ang = math.atan2(s, float(u @ v))
    axis /= s
    return np.array([math.cos(ang / 2), *(math.sin(ang / 2) * axis)])


def test_axis_aligned_octahedron_entry_depth():
    c = cam(64, 48)
    Z, d = 4.0, (0.3, 0.25, 0.2)
    s = one_prim(OCTA, (0, 0, Z), (1, 0, 0, 0), d, logit=6.0)
    out = render(s, c)
    fx, fy, cx, cy = (float(c[k]) for k in ("fx", "fy", "cx", "cy"))
    ys, xs = np.mgrid[0:48, 0:64] + 0.5
    d32 = [float(np.float32(x)) for x in d]
    w = 1 - np.abs(xs - cx) * Z / (fx * d32[0]) - np.abs(ys - cy) * Z / (fy * d32[1])
    ref = Z - d32[2] * w
    crossed = out.T_final < 0.5
    assert crossed.sum() > 10 and (~crossed & (w > 0)).sum() > 0      # both regimes present
    assert np.abs(out.depth[crossed] - ref[crossed]).max() < 1e-6
    assert np.all(out.depth[~crossed] == 0.0)                           # invalid marker (reading 24)
    # alpha mode = 1 - T_final
    assert np.array_equal(out.alpha, 1.0 - out.T_final)


@pytest.mark.parametrize("kind", [TETRA, OCTA])
def test_face_on_entry_depth(kind):
    """Regular primitive with a face turned squarely towards the camera.  Tetrahedron: every ray that
    enters, enters through that face (its silhouette).  Octahedron: the rays through the front
    triangle (incircle radius d/sqrt6 around the axis) do; the others enter through a side face."""
    c = cam(64, 48)
    Z, d = 5.0, 0.6
    if kind == TETRA:
        # vertex b_0 = (1,1,1)/sqrt3 turned to +z: the opposite face (inradius d/3) faces the camera
        q = quat_turning((1, 1, 1), (0, 0, 1))
        s = one_prim(TETRA, (0, 0, Z), q, (d, d, d, d), logit=6.0)
        r_in = d / 3.0
    else:
        q = quat_turning((1, 1, 1), (0, 0, -1))      # face normal (1,1,1)/sqrt3 -> towards the camera
        s = one_prim(OCTA, (0, 0, Z), q, (d, d, d), logit=6.0)
        r_in = d / math.sqrt(3.0)
    out = render(s, c)
    crossed = out.T_final < 0.5
    assert crossed.sum() > 30
    if kind == OCTA:
        ys, xs = np.mgrid[0:48, 0:64] + 0.5
        rad = np.hypot(xs - float(c["cx"]), ys - float(c["cy"])) * Z / float(c["fx"])
        inner = rad < 0.95 * d / math.sqrt(6.0)
        assert (crossed & inner).sum() >= 8
        assert np.all(out.depth[crossed & ~inner] > Z - r_in - 2e-6)   # side faces are further away
        sel = crossed & inner
    else:
        sel = crossed
    # fp32 quaternion / distances: the face is flat to ~1e-7 relative
    assert np.abs(out.depth[sel] - (Z - r_in)).max() < 2e-6
    assert np.all(out.depth[~crossed] == 0.0)


def test_first_primitive_past_half_is_chosen():
    """Front primitive with o < 0.5 everywhere, back one opaque: depth is the BACK primitive's entry
    wherever the pair crosses 0.5; where only the front is hit it never crosses."""
    c = cam(64, 48)
    fx, fy, cx, cy = (float(c[k]) for k in ("fx", "fy", "cx", "cy"))
    Zf, df = 3.0, (0.5, 0.5, 0.2)
    Zb, db = 6.0, (0.4, 0.35, 0.3)
    front = one_prim(OCTA, (0, 0, Zf), (1, 0, 0, 0), df, logit=-0.5)      # alpha 0.38: o <= 0.99 alpha < 0.5
    back = one_prim(OCTA, (0, 0, Zb), (1, 0, 0, 0), db, logit=6.0)
    out = render(concat([front, back]), c)
    only_front = render(front, c)
    assert np.all(only_front.T_final > 0.5) and np.all(only_front.depth == 0.0)
    ys, xs = np.mgrid[0:48, 0:64] + 0.5
    b32 = [float(np.float32(x)) for x in db]
    wb = 1 - np.abs(xs - cx) * Zb / (fx * b32[0]) - np.abs(ys - cy) * Zb / (fy * b32[1])
    ref = Zb - b32[2] * wb
    crossed = out.T_final < 0.5
    assert crossed.sum() > 20
    assert np.abs(out.depth[crossed] - ref[crossed]).max() < 1e-6
    assert np.all(out.depth[~crossed] == 0.0)


def test_depth_margin_and_early_stop_independence():
    """m_depth = min |ln(T_after/0.5)|; the 0.999 stop (T < 1e-3) happens after the 0.5 crossing, so
    depth is the same with and without early stopping."""
    from paper_2501_16312_b200 import scenegen
    scene, c = scenegen.small_scene(OCTA, n=300, width=64, height=48, seed=3)
    a = oracle.forward(oscene(scene), c, kappa=0.1, mode=1, t_stop=1e-3).out
    b = oracle.forward(oscene(scene), c, kappa=0.1, mode=1, t_stop=0.0).out
    assert np.array_equal(a.depth, b.depth)
    assert np.all(a.m_depth >= 0)
    crossed = a.T_final < 0.5
    assert np.all(a.depth[crossed] > 0) and np.all(a.depth[~crossed] == 0)
