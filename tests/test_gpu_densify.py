"""GPU parity of the f4 inputs to population control against oracle/densify.py:
lp_filter3d (3D smoothing filter size from training cameras) and the densification statistics
accumulated by the preprocess backward (lp_grads.mean2d_abs, lp_grads.vis_count)."""
import numpy as np
import pytest

import oracle
from oracle import densify as OD
from paper_2501_16312_b200 import scenegen
from tests import parity as PT
from tests.helpers import oscene

pytestmark = pytest.mark.gpu

OCTA, TETRA = scenegen.OCTA, scenegen.TETRA


@pytest.fixture(scope="module", autouse=True)
def _cuda():
    import torch
    assert torch.cuda.is_available(), "gpu tests need CUDA"
    from paper_2501_16312_b200 import _build
    _build.build()
    torch.cuda.set_device(0)


def borderline(pos, cams, tol=1e-3):
    """Primitives whose 'camera sees centre' decision is within tol of flipping for some camera."""
    bad = np.zeros(pos.shape[1], bool)
    for c in cams:
        p = OD.camera_space(pos, c)
        z = p[2]
        zs = np.where(np.abs(z) > 1e-9, z, 1e-9)
        u = float(c["fx"]) * p[0] / zs + float(c["cx"])
        v = float(c["fy"]) * p[1] / zs + float(c["cy"])
        bad |= np.abs(z - float(c["znear"])) < tol
        for a, lim in ((u, 0.0), (u, float(c["width"])), (v, 0.0), (v, float(c["height"]))):
            bad |= (z > 0) & (np.abs(a - lim) < tol)
    return bad


@pytest.mark.parametrize("n_cams", [1, 8, 100])
def test_filter3d_vs_oracle(n_cams):
    import torch

    from paper_2501_16312_b200 import render
    scene, cams = scenegen.make_scene("C2", seed=1, n=20000)
    rng = np.random.default_rng(5)
    ring = scenegen.ring_cameras(320, 240, n_views=n_cams, radius=4.0)
    # some centres far outside every view (fallback branch) and some behind the cameras
    pos = scene["pos"].copy()
    pos[:, :500] = rng.uniform(-30, 30, (3, 500)).astype(np.float32)
    scene = dict(scene, pos=pos)
    ds = render.DeviceScene(scene)
    got = ds.set_filter3d(ring, 0.2).cpu().numpy()
    torch.cuda.synchronize()
    ref = OD.filter3d(pos, ring, 0.2)
    ok = ~borderline(pos, ring)
    assert ok.mean() > 0.97
    rel = np.abs(got - ref) / np.maximum(np.abs(ref), 1e-30)
    assert rel[ok].max() < 2e-6, rel[ok].max()
    # the fallback branch was exercised
    seen = np.zeros(pos.shape[1], bool)
    for c in ring:
        seen |= OD.sees(pos, c)[0]
    assert (~seen).sum() > 10


@pytest.mark.parametrize("kind", [OCTA, TETRA])
def test_densification_statistics(kind):
    import torch

    from paper_2501_16312_b200 import render
    scene, cam = scenegen.small_scene(kind, n=500, seed=21, width=96, height=72)
    # three views of the same scene: the original and two shifted principal points
    cams = [cam, dict(cam, cx=np.float32(float(cam["cx"]) + 7.0)), dict(cam, cy=np.float32(float(cam["cy"]) - 5.0))]
    W, H = cam["width"], cam["height"]
    ds = render.DeviceScene(scene)
    ds.track_mean2d()
    r = render.Renderer(ds, cams)
    img = r.forward()
    G = np.stack([scenegen.upstream_grad(W, H, seed=30 + v)[0] for v in range(3)])
    r.backward(torch.as_tensor(G, device="cuda").reshape(img.shape))
    torch.cuda.synchronize()
    m2d = ds.mean2d.cpu().numpy()
    cnt = ds.vis_count.cpu().numpy()
    ref_m, ref_c, flagged = np.zeros(500), np.zeros(500), np.zeros(500, bool)
    for v, c in enumerate(cams):
        fb, _ = oracle.forward_backward(oscene(scene), c, G[v])
        ref_m += OD.mean2d_norm(fb.out.dv)
        ref_c += (fb.pre.tiles_touched > 0)
        flagged |= fb.out.face_margin < PT.FACE_MARGIN
        assert (fb.out.m_stop < PT.STOP_MARGIN).mean() < 0.01
    assert np.array_equal(cnt, ref_c)
    ok, worst, rep, _ = PT.grad_close("mean2d_abs", m2d, ref_m, flagged)
    assert ok, rep
