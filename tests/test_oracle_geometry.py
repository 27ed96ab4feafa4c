"""Pins for the oracle's preprocess geometry."""
import math

import numpy as np
import pytest

import oracle
from paper_2501_16312_b200 import scenegen
from tests.canonical_np import canonical
from tests.helpers import cam, one_prim, oscene

OCTA, TETRA = oracle.OCTA, oracle.TETRA
H = 0.5 * float(np.float32(0.1))   # the kernel is an fp32 input; half of it per side


def geom(scene, c, kappa=0.0, mode=1):
    return oracle.preprocess(oscene(scene), c, kappa=kappa, mode=mode)


def recover_R(q, Z=10.0):
    """On the optical axis with W = I, J = diag(fx/Z, fy/Z, 1), so o_j = J d_j R e_j."""
    c = cam()
    pre = geom(one_prim(OCTA, (0, 0, Z), q, (1, 1, 1)), c)
    off = pre.geom[0, 3:].reshape(3, 3)
    scale = np.array([Z / float(c["fx"]), Z / float(c["fy"]), 1.0])
    return np.stack([off[j] * scale for j in range(3)], axis=1)


@pytest.mark.parametrize("seed", range(5))
def test_rotation_orthonormal_and_sign_invariant(seed):
    q = np.random.default_rng(seed).standard_normal(4)
    R = recover_R(q)
    assert np.allclose(R @ R.T, np.eye(3), atol=1e-12)
    assert math.isclose(np.linalg.det(R), 1.0, abs_tol=1e-12)
    assert np.allclose(recover_R(-q), R, atol=1e-12)          # q and -q: same rotation
    assert np.allclose(recover_R(3.7 * q), R, atol=1e-12)     # normalisation


def test_rotation_worked_examples():
    # (2,0,0,0) -> identity; (1,1,1,1) -> 120 deg about (1,1,1): x->y->z->x
    assert np.allclose(recover_R((2, 0, 0, 0)), np.eye(3), atol=1e-12)
    assert np.allclose(recover_R((1, 1, 1, 1)), [[0, 0, 1], [1, 0, 0], [0, 1, 0]], atol=1e-12)
    # 90 deg about z maps +x to +y
    R = recover_R((math.cos(math.pi / 4), 0, 0, math.sin(math.pi / 4)))
    assert np.allclose(R[:, 0], [0, 1, 0], atol=1e-12)


def test_octahedron_vertices_axis_aligned():
    # identity rotation, d = (1,2,3) -> vertices c +- d_i e_i (mapped by J on the axis)
    c = cam()
    Z = 10.0
    pre = geom(one_prim(OCTA, (0, 0, Z), (1, 0, 0, 0), (1, 2, 3)), c)
    off = pre.geom[0, 3:].reshape(3, 3)
    fx, fy = float(c["fx"]), float(c["fy"])
    assert np.allclose(off, [[fx * 1 / Z, 0, 0], [0, fy * 2 / Z, 0], [0, 0, 3]], atol=1e-12)
    assert np.allclose(pre.geom[0, :3], [float(c["cx"]), float(c["cy"]), Z], atol=1e-12)


def test_tetrahedron_basis():
    # S:66 + S:102: identity rotation, d = 1 -> the canonical basis (pairwise dot -1/3, sum 0)
    c = cam()
    Z = 10.0
    pre = geom(one_prim(TETRA, (0, 0, Z), (1, 0, 0, 0), (1, 1, 1, 1)), c)
    off = pre.geom[0, 3:].reshape(4, 3)
    b = off * np.array([Z / float(c["fx"]), Z / float(c["fy"]), 1.0])
    assert np.allclose(np.linalg.norm(b, axis=1), 1.0, atol=1e-12)
    G = b @ b.T
    assert np.allclose(G[~np.eye(4, dtype=bool)], -1.0 / 3.0, atol=1e-12)
    assert np.allclose(b.sum(0), 0.0, atol=1e-12)
    s3 = 1 / math.sqrt(3)
    assert np.allclose(b, s3 * np.array([[1, 1, 1], [1, -1, -1], [-1, 1, -1], [-1, -1, 1]]), atol=1e-12)


def test_ray_space_map_examples():
    # p = (0,0,z) -> (cx, cy, z); fx=fy=100, cx=cy=0, p=(1,0,1) -> (100, 0, sqrt 2)
    c = cam()
    pre = geom(one_prim(OCTA, (0, 0, 7.0), (1, 0, 0, 0), (0.1, 0.1, 0.1)), c)
    assert np.allclose(pre.geom[0, :3], [float(c["cx"]), float(c["cy"]), 7.0], atol=1e-12)
    c2 = dict(c, fx=np.float32(100), fy=np.float32(100), cx=np.float32(0), cy=np.float32(0))
    pre = geom(one_prim(OCTA, (1, 0, 1), (1, 0, 0, 0), (0.01, 0.01, 0.01)), c2)
    assert np.allclose(pre.geom[0, :3], [100.0, 0.0, math.sqrt(2)], atol=1e-12)


def _phi(p, c):
    """phi(p) from its definition: (fx px/pz + cx, fy py/pz + cy, |p|)."""
    return np.array([float(c["fx"]) * p[0] / p[2] + float(c["cx"]),
                     float(c["fy"]) * p[1] / p[2] + float(c["cy"]), np.linalg.norm(p)])


@pytest.mark.parametrize("seed", range(6))
def test_jacobian_matches_finite_differences_of_phi(seed):
    """Offsets o_j = J(p) W (d_j e_j): compare with central differences of phi."""
    rng = np.random.default_rng(seed)
    W, t = scenegen.look_at(rng.normal(0, 2, 3), rng.normal(0, 1, 3) + [0, 0, 6])
    c = cam(W=W, t=t)
    centre = rng.normal(0, 1, 3) + [0, 0, 6]
    d = 1e-4 * np.array([1.0, 2.0, 3.0])
    pre = geom(one_prim(OCTA, centre, (1, 0, 0, 0), d), c)
    off = pre.geom[0, 3:].reshape(3, 3)
    Wd, td = np.asarray(W, np.float64), np.asarray(t, np.float64)
    p = Wd @ np.asarray(centre, np.float32).astype(np.float64) + td
    for j in range(3):
        e = np.zeros(3)
        e[j] = np.float32(d[j])
        fd = (_phi(p + Wd @ e, c) - _phi(p - Wd @ e, c)) / 2.0
        assert np.allclose(off[j], fd, rtol=1e-6, atol=1e-10 * np.abs(fd).max())


@pytest.mark.parametrize("seed", range(6))
def test_det_J(seed):
    """det J = fx fy |p| / p_z^3 > 0 (orientation preserving)."""
    rng = np.random.default_rng(seed)
    W, t = scenegen.look_at(rng.normal(0, 2, 3), [0, 0, 6])
    c = cam(W=W, t=t)
    centre = rng.normal(0, 1, 3) + [0, 0, 6]
    d = np.array([0.3, 0.2, 0.1])
    pre = geom(one_prim(OCTA, centre, (1, 0, 0, 0), d), c)
    M = pre.geom[0, 3:].reshape(3, 3).T
    p = np.asarray(W, np.float64) @ np.asarray(centre, np.float32).astype(np.float64) + np.asarray(t, np.float64)
    detJ = float(c["fx"]) * float(c["fy"]) * np.linalg.norm(p) / p[2] ** 3
    detW = np.linalg.det(np.asarray(W, np.float64))   # fp32 W is orthonormal only to ~1e-7
    assert math.isclose(np.linalg.det(M) / (detW * np.prod(np.float32(d).astype(np.float64))), detJ, rel_tol=1e-9)


def test_2d_filter_octahedron_axis_aligned():
    # S:277-279 / P:1193: kernel 0.1 -> the ray-space vector moves by 0.05, bbox grows by 0.1
    c = cam()
    s = one_prim(OCTA, (0, 0, 10.0), (1, 0, 0, 0), (0.2, 0.1, 0.3))
    a = geom(s, c, kappa=0.0).geom[0, 3:].reshape(3, 3)
    b = geom(s, c, kappa=0.1).geom[0, 3:].reshape(3, 3)
    delta = b - a
    assert math.isclose(delta[0, 0], H, abs_tol=1e-12)    # x-extremal axis
    assert math.isclose(delta[1, 1], H, abs_tol=1e-12)    # y-extremal axis
    delta[0, 0] = delta[1, 1] = 0.0
    assert np.all(delta == 0.0)                              # nothing else moves


def test_2d_filter_tetrahedron_extremes():
    c = cam()
    s = one_prim(TETRA, (0.1, 0.05, 10.0), (0.9, 0.2, -0.3, 0.1), (0.2, 0.25, 0.15, 0.3))
    a = geom(s, c, kappa=0.0).geom[0, 3:].reshape(4, 3)
    b = geom(s, c, kappa=0.1).geom[0, 3:].reshape(4, 3)
    for ax in range(2):
        assert math.isclose(b[:, ax].max() - a[:, ax].max(), H, abs_tol=1e-12)
        assert math.isclose(a[:, ax].min() - b[:, ax].min(), H, abs_tol=1e-12)
    assert np.all(b[:, 2] == a[:, 2])


@pytest.mark.parametrize("kind", [OCTA, TETRA])
@pytest.mark.parametrize("seed", range(3))
def test_canonical_fp32_matches_numpy_arbiter(kind, seed):
    """The oracle's mode-0 geometry equals an independent NumPy float32 evaluation bit for bit."""
    for sc, c in (scenegen.small_scene(kind, 3000, seed=seed, width=333, height=211),
                  scenegen.edge_scene(kind, seed=seed)):
        pre = oracle.preprocess(oscene(sc), c, kappa=0.1, mode=0)
        ref = canonical(sc, c, kappa=0.1)
        assert np.array_equal(pre.flag, ref["flag"])
        assert np.array_equal(pre.tiles_touched, ref["tiles_touched"])
        assert np.array_equal(pre.rect, ref["rect"])
        assert np.array_equal(pre.depth_key, ref["depth_key"])
        assert np.array_equal(pre.canon.view(np.uint32), ref["canon"].view(np.uint32))


def test_edge_scene_flags():
    for kind in (OCTA, TETRA):
        sc, c = scenegen.edge_scene(kind)
        pre = oracle.preprocess(oscene(sc), c, kappa=0.1, mode=0)
        assert pre.flag[6] == 2 and pre.flag[7] == 2                 # behind camera / inside znear
        assert pre.flag[13] == 1 and pre.flag[14] == 1 and pre.flag[15] == 1 and pre.flag[16] == 1
        assert pre.tiles_touched[5] == 0                             # off-screen
        gx, gy = (c["width"] + 15) // 16, (c["height"] + 15) // 16
        assert pre.tiles_touched[9] == gx * gy                       # huge primitive covers every tile
        assert pre.depth_key[11] == pre.depth_key[12]
