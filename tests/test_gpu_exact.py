"""GPU parity of the "no ray space" variant (lp_raster_cfg.exact = 1) against the
oracle's exact mode: bit-exact tiles / rects / keys / canonical camera-space geometry / sorted lists,
images within 1e-4, gradients within the north_star bar, depth / alpha."""
import numpy as np
import pytest

import oracle
from paper_2501_16312_b200 import scenegen
from tests import parity as PT
from tests.helpers import oscene
from tests.test_gpu_parity import full_parity

pytestmark = pytest.mark.gpu

OCTA, TETRA = scenegen.OCTA, scenegen.TETRA


@pytest.fixture(scope="module", autouse=True)
def _cuda():
    import torch
    assert torch.cuda.is_available(), "gpu tests need CUDA"
    from paper_2501_16312_b200 import _build
    _build.build()
    torch.cuda.set_device(0)


@pytest.mark.parametrize("kind", [OCTA, TETRA])
@pytest.mark.parametrize("seed", range(4))
def test_exact_random_small_scenes(kind, seed):
    scene, cam = scenegen.small_scene(kind, n=300 + 200 * seed, seed=40 + seed, width=80 + 16 * seed,
                                      height=64 + 8 * seed)
    full_parity(scene, cam, kappa=0.0, exact=True)


@pytest.mark.parametrize("kind", [OCTA, TETRA])
def test_exact_no_stop(kind):
    scene, cam = scenegen.small_scene(kind, n=500, seed=77, width=96, height=64)
    full_parity(scene, cam, kappa=0.0, t_stop=0.0, exact=True)


def test_exact_c1():
    scene, cams = scenegen.make_scene("C1", seed=0)
    full_parity(scene, cams[0], kappa=0.0, exact=True)


@pytest.mark.parametrize("kind", [OCTA, TETRA])
def test_exact_near_camera_whole_screen_rect(kind):
    """Large primitives straddling the camera plane: the rect is the whole screen on both sides and the
    chord is 0 where the entry is behind the camera (reading 27)."""
    scene, cam = scenegen.small_scene(kind, n=120, seed=5, width=64, height=48, depth=(0.5, 3.0), size=(0.2, 1.5))
    pre = oracle.preprocess(oscene(scene), cam, kappa=0.0, mode=1, exact=True)
    K = 3 if kind == OCTA else 4
    off_z = pre.geom[:, 5::3][:, :K]
    vz = pre.geom[:, 2:3] + (np.concatenate([off_z, -off_z], 1) if kind == OCTA else off_z)
    behind = (pre.flag == 0) & (vz <= 0).any(1)
    assert behind.sum() >= 2 and np.all(pre.tiles_touched[behind] == 4 * 3)   # whole screen (4 x 3 tiles)
    full_parity(scene, cam, kappa=0.0, exact=True, max_flagged=0.25)  # few, large primitives: many edge pixels each


@pytest.mark.parametrize("kind", [OCTA, TETRA])
def test_exact_depth_alpha(kind):
    import torch

    from paper_2501_16312_b200 import render
    scene, cam = scenegen.small_scene(kind, n=600, seed=13, width=96, height=72, opacity_mu=0.5)
    ds = render.DeviceScene(scene)
    r = render.Renderer(ds, [cam], aa_kernel=0.0, exact=True)
    img, dep, alp = r.forward(depth=True, alpha=True)
    torch.cuda.synchronize()
    o = oracle.forward(oscene(scene), cam, kappa=0.0, exact=True).out
    mask = (o.m_stop < PT.STOP_MARGIN) | (o.m_depth < 1e-4)
    assert mask.mean() < 0.02
    assert np.abs(alp[0].cpu().numpy() - o.alpha)[~mask].max() <= PT.IMG_TOL
    d = dep[0].cpu().numpy()
    assert np.abs(d - o.depth)[~mask].max() <= 1e-4
    assert (o.depth > 0).sum() > 100


def test_exact_differs_from_ray_space():
    """The variant is really different (not the ray-space path with a flag ignored)."""
    import torch

    from paper_2501_16312_b200 import render
    scene, cam = scenegen.small_scene(OCTA, n=300, seed=2, width=64, height=48, size=(0.3, 0.8))
    ds = render.DeviceScene(scene)
    a = render.Renderer(ds, [cam], aa_kernel=0.0).forward().cpu().numpy()
    b = render.Renderer(ds, [cam], aa_kernel=0.0, exact=True).forward().cpu().numpy()
    torch.cuda.synchronize()
    assert np.abs(a - b).max() > 1e-3


@pytest.mark.parametrize("kind", [OCTA, TETRA])
@pytest.mark.parametrize("seed", range(3))
def test_exact_edge_scenes(kind, seed):
    """The ray-space edge cases (tile-border stragglers, off-screen, behind the camera, inside znear,
    sub-pixel, huge, alpha ~ 0, duplicate depths, invalid inputs, axis-aligned faces; image size not a
    multiple of 16) through the no-ray-space variant."""
    scene, cam = scenegen.edge_scene(kind, seed=seed)
    full_parity(scene, cam, kappa=0.0, seed=seed, exact=True, max_flagged=0.1)


def test_exact_empty_and_single():
    import torch
    scene, cam = scenegen.small_scene(OCTA, 50, seed=1, width=40, height=30)
    scene["pos"][2] = -5.0
    ds, r, img = PT.gpu_run(scene, [cam], G=np.ones((3, 30, 40), np.float32), bg=(0.25, 0.5, 0.75), kappa=0.0,
                            exact=True)
    assert torch.allclose(img[0, 0], torch.full_like(img[0, 0], 0.25))
    assert float(ds.grad.abs().max()) == 0.0
    scene, cam = scenegen.small_scene(TETRA, 1, seed=2, width=1, height=1)
    full_parity(scene, cam, kappa=0.0, seed=1, exact=True)
