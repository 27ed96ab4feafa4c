"""GPU parity of the depth / alpha render modes (lp_render_fwd_aux) against the oracle.

depth: entry distance of the first primitive after which 1 - T > 0.5, 0 if never
(reading 24); tolerance 1e-4 world units (S:759 criterion 8).  Pixels whose 0.5 decision
is within DEPTH_MARGIN of flipping (oracle m_depth) or whose stop index may flip (m_stop) are masked
and counted.  alpha = 1 - T_final within the image tolerance.  The colour image must be bitwise
unchanged by the extra outputs.
"""
import numpy as np
import pytest

import oracle
from paper_2501_16312_b200 import scenegen
from tests import parity as PT
from tests.helpers import oscene

pytestmark = pytest.mark.gpu

OCTA, TETRA = scenegen.OCTA, scenegen.TETRA
DEPTH_TOL = 1e-4
DEPTH_MARGIN = 1e-4


@pytest.fixture(scope="module", autouse=True)
def _cuda():
    import torch
    assert torch.cuda.is_available(), "gpu tests need CUDA"
    from paper_2501_16312_b200 import _build
    _build.build()
    torch.cuda.set_device(0)


def run_aux(scene, cams, kappa=0.1, t_stop=1e-3):
    import torch

    from paper_2501_16312_b200 import render
    ds = render.DeviceScene(scene)
    r = render.Renderer(ds, cams, aa_kernel=kappa, t_stop=t_stop)
    img0 = r.forward()
    img, dep, alp = r.forward(depth=True, alpha=True)
    torch.cuda.synchronize()
    return img0.cpu().numpy(), img.cpu().numpy(), dep.cpu().numpy(), alp.cpu().numpy()


def check(scene, cam, kappa=0.1, t_stop=1e-3, max_masked=0.02):
    img0, img, dep, alp = run_aux(scene, [cam], kappa=kappa, t_stop=t_stop)
    assert np.array_equal(img0.view(np.uint32), img.view(np.uint32)), "colour image changed by the aux outputs"
    f = oracle.forward(oscene(scene), cam, kappa=kappa, t_stop=t_stop)
    o = f.out
    mask = (o.m_stop < PT.STOP_MARGIN) | (o.m_depth < DEPTH_MARGIN)
    assert mask.mean() <= max_masked, f"masked {mask.mean()}"
    a_err = np.abs(alp[0] - o.alpha)[~mask]
    assert a_err.max(initial=0.0) <= PT.IMG_TOL, f"alpha err {a_err.max()}"
    d_ok = ~mask
    d_err = np.abs(dep[0] - o.depth)[d_ok]
    assert d_err.max(initial=0.0) <= DEPTH_TOL, f"depth err {d_err.max()}"
    # both sides agree on where the depth is defined
    assert np.array_equal(dep[0][d_ok] == 0, o.depth[d_ok] == 0)
    return int((o.depth > 0).sum())


@pytest.mark.parametrize("kind", [OCTA, TETRA])
@pytest.mark.parametrize("seed", range(4))
def test_depth_alpha_random_scenes(kind, seed):
    scene, cam = scenegen.small_scene(kind, n=400 + 300 * seed, seed=100 + seed, width=96 + 16 * seed,
                                      height=64 + 8 * seed, opacity_mu=0.5)
    defined = check(scene, cam)
    assert defined > 100


@pytest.mark.parametrize("kind", [OCTA, TETRA])
def test_depth_alpha_no_stop_and_filter(kind):
    scene, cam = scenegen.small_scene(kind, n=600, seed=7, width=80, height=72)
    check(scene, cam, kappa=0.5, t_stop=0.0)


def test_depth_alpha_c1():
    scene, cams = scenegen.make_scene("C1", seed=0)
    check(scene, cams[0])


def test_depth_empty_scene():
    scene, cam = scenegen.small_scene(OCTA, n=50, seed=1, width=48, height=40)
    scene = dict(scene)
    scene["opacity"] = np.full_like(scene["opacity"], -80.0)     # alpha -> 0: nothing crosses 0.5
    img0, img, dep, alp = run_aux(scene, [cam])
    assert np.all(dep == 0.0)
    assert np.abs(alp).max() < 1e-6
