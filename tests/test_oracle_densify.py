"""Pins for oracle/densify.py.

* S:545-548 worked examples: kappa = 0 -> 0; one camera at depth 10, focal 1000, kappa 0.2 ->
  s_3d = 0.002;
* the minimum is over the cameras that SEE the centre (a nearer camera looking away does not count);
* a centre no camera sees takes kappa |p| / fx of the nearest camera;
* mean2d_norm: the gradient with respect to the ray-space centre is the sum of the vertex gradients
  (all vertices move with c_r) -- checked on a hand-made dv, and by finite differences of the
  principal point: phi_x = fx p_x/p_z + cx, so moving cx moves c_r.x of every primitive by the same
  amount and leaves J (the offsets) unchanged; with one primitive dL/dcx = dL/dc_r.x exactly.
"""
import math

import numpy as np

from oracle import densify as OD
from paper_2501_16312_b200 import scenegen


def cam_at(z_eye, f=1000.0, W=None, t=None, width=640, height=480):
    c = scenegen.pinhole(width, height, W=W, t=t)
    c["fx"] = c["fy"] = np.float32(f)
    return c


def test_spec_examples():
    pos = np.array([[0.0], [0.0], [10.0]])
    c = cam_at(0.0)
    assert OD.filter3d(pos, [c], 0.0)[0] == 0.0
    assert math.isclose(OD.filter3d(pos, [c], 0.2)[0], 0.002, rel_tol=1e-12)


def test_min_over_seeing_cameras_only():
    pos = np.array([[0.0], [0.0], [10.0]])
    far = cam_at(0.0)                                          # depth 10, sees it
    near = cam_at(0.0, t=np.array([0.0, 0.0, -7.0], np.float32))  # depth 3, sees it
    behind = cam_at(0.0, t=np.array([0.0, 0.0, -12.0], np.float32))  # depth -2: does not see
    side = cam_at(0.0, t=np.array([5.0, 0.0, -9.0], np.float32))    # depth 1, projects off-image
    s = OD.filter3d(pos, [far, near, behind, side], 0.5)[0]
    assert math.isclose(s, 0.5 * 3.0 / 1000.0, rel_tol=1e-12)


def test_unseen_uses_nearest_camera():
    pos = np.array([[0.0], [0.0], [-4.0]])                      # behind every camera below
    c1 = cam_at(0.0)                                            # |p| = 4
    c2 = cam_at(0.0, t=np.array([0.0, 0.0, 6.0], np.float32), f=500.0)   # p_z = 2 > znear: sees it
    assert math.isclose(OD.filter3d(pos, [c1, c2], 1.0)[0], 2.0 / 500.0, rel_tol=1e-12)
    c3 = cam_at(0.0, t=np.array([0.0, 0.0, -3.0], np.float32), f=250.0)  # |p| = 7, unseen
    assert math.isclose(OD.filter3d(pos, [c1, c3], 1.0)[0], 4.0 / 1000.0, rel_tol=1e-12)
    assert math.isclose(OD.filter3d(pos, [c3], 1.0)[0], 7.0 / 250.0, rel_tol=1e-12)


def test_mean2d_norm_is_centre_gradient():
    dv = np.zeros((2, 6, 3))
    dv[0, :, 0] = [1, -2, 0.5, 0.5, 0, 1]        # sum 1
    dv[0, :, 1] = [0, 0, 3, -3, 2, 2]            # sum 4
    dv[0, :, 2] = 100.0                          # depth components do not count
    dv[1] = 0.0
    m = OD.mean2d_norm(dv)
    assert math.isclose(m[0], math.hypot(1.0, 4.0), rel_tol=1e-14) and m[1] == 0.0


def test_mean2d_against_principal_point_fd():
    import oracle
    from tests.helpers import cam, one_prim, oscene
    c = cam(64, 48)
    s = one_prim(oracle.OCTA, (0.1, -0.05, 4.0), (0.9, 0.2, -0.3, 0.1), (0.35, 0.25, 0.3), logit=0.4,
                 rgb_dc=(0.8, 0.3, 0.5))
    G = np.random.default_rng(0).normal(0, 1, (3, 48, 64)).astype(np.float32)
    f, _ = oracle.forward_backward(oscene(s), c, G, kappa=0.0, mode=1, t_stop=0.0)
    g = f.out.dv[0, :, :2].sum(0)

    def loss(dcx, dcy):
        cc = dict(c, cx=np.float32(float(c["cx"]) + dcx), cy=np.float32(float(c["cy"]) + dcy))
        return float((oracle.forward(oscene(s), cc, kappa=0.0, mode=1, t_stop=0.0).out.image * G).sum())
    h = 1.0 / 4096      # exact in fp32 at cx ~ 32; small so few pixel centres cross a face edge
    fd = np.array([(loss(h, 0) - loss(-h, 0)) / (2 * h), (loss(0, h) - loss(0, -h)) / (2 * h)])
    assert np.abs(fd - g).max() <= 2e-3 * np.abs(g).max(), (fd, g)
    assert math.isclose(OD.mean2d_norm(f.out.dv)[0], float(np.hypot(*g)), rel_tol=1e-12)
