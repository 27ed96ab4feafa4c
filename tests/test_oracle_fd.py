"""Central finite differences of the oracle's fp64 forward pin its analytic backward
(App. E; blend backward P:215-216; Eq. 1 with frozen denominator P:1192;
S:387-401).  Geometry in fp64 (mode 1) so the loss is smooth away from visibility kinks."""
import numpy as np
import pytest

import oracle
from paper_2501_16312_b200 import scenegen
from tests.helpers import oscene

OCTA, TETRA = oracle.OCTA, oracle.TETRA


def _loss(scene, c, G, den, kappa, t_stop, bg, filter3d=None):
    f = oracle.forward(oscene(scene, filter3d), c, kappa=kappa, mode=1, t_stop=t_stop, bg=bg, den_override=den)
    return float(np.sum(G.astype(np.float64) * f.out.image))


def _fd_check(scene, c, G, kappa, t_stop, bg=(0.1, 0.2, 0.3), filter3d=None, rtol=2e-5, groups=None):
    sc = oscene(scene, filter3d)
    pre = oracle.preprocess(sc, c, kappa=kappa, mode=1)
    den = pre.sigma_den.copy()
    f, g = oracle.forward_backward(sc, c, G, kappa=kappa, mode=1, t_stop=t_stop, bg=bg, den_override=den)
    worst = {}
    for name in groups or ("pos", "rot", "dist", "opacity", "sh"):
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
            lp = _loss(scene, c, G, den, kappa, t_stop, bg, filter3d)
            flat[idx] = np.float32(th - h)
            hm = th - float(flat[idx])
            lm = _loss(scene, c, G, den, kappa, t_stop, bg, filter3d)
            flat[idx] = old
            fd = (lp - lm) / (hp + hm)
            a = an.reshape(-1)[idx]
            err = abs(fd - a) / (abs(a) + 1e-4 * scale + 1e-300)
            errs.append(err)
        worst[name] = max(errs) if errs else 0.0
    bad = {k: v for k, v in worst.items() if v > rtol}
    assert not bad, f"FD mismatch (relative, worst per group): {worst}"
    return f, g


@pytest.mark.parametrize("kind", [OCTA, TETRA])
@pytest.mark.parametrize("kappa", [0.0, 0.1])
@pytest.mark.parametrize("seed", [0, 1])
def test_fd_full_backward(kind, kappa, seed):
    """S:752 acceptance 1 (fp64 variant): every feature of a few-primitive scene."""
    scene, c = scenegen.small_scene(kind, 5, seed=seed, width=32, height=24, sh_degree=3 if seed == 0 else 1,
                                    depth=(3.0, 9.0), size=(0.15, 0.5), opacity_mu=0.5)
    G = scenegen.upstream_grad(32, 24, seed=seed)[0]
    _fd_check(scene, c, G, kappa, t_stop=0.0)


@pytest.mark.parametrize("kind", [OCTA, TETRA])
def test_fd_with_3d_filter(kind):
    scene, c = scenegen.small_scene(kind, 4, seed=11, width=32, height=24, sh_degree=0,
                                    depth=(3.0, 9.0), size=(0.15, 0.5))
    f3 = np.full(4, 0.05, np.float32)
    G = scenegen.upstream_grad(32, 24, seed=11)[0]
    _fd_check(scene, c, G, 0.1, t_stop=0.0, filter3d=f3, groups=("pos", "rot", "dist", "opacity"))


@pytest.mark.parametrize("kind", [OCTA, TETRA])
def test_fd_with_early_stop(kind):
    """With the 0.999 stop active, away from stop-index flips (margin checked)."""
    scene, c = scenegen.small_scene(kind, 8, seed=21, width=24, height=20, sh_degree=1,
                                    depth=(3.0, 6.0), size=(0.4, 0.9), opacity_mu=4.0)
    G = scenegen.upstream_grad(24, 20, seed=21)[0]
    sc = oscene(scene)
    f = oracle.forward(sc, c, kappa=0.1, mode=1, t_stop=1e-3)
    assert (f.out.T_final < 1e-3).any()
    # zero the upstream gradient at pixels within 1e-3 (log-margin) of a stop decision
    G = G * (f.out.m_stop > 1e-3)[None].astype(np.float32)
    _fd_check(scene, c, G, 0.1, t_stop=1e-3, groups=("pos", "dist", "opacity"))


def test_background_gradient_is_final_transmittance():
    """dC/d(bg) = T_final exactly (C is affine in bg)."""
    scene, c = scenegen.small_scene(OCTA, 12, seed=3, width=32, height=24)
    sc = oscene(scene)
    a = oracle.forward(sc, c, bg=(0.0, 0.0, 0.0), mode=1)
    b = oracle.forward(sc, c, bg=(1.0, 0.0, 0.0), mode=1)
    assert np.allclose(b.out.image[0] - a.out.image[0], a.out.T_final, atol=1e-15)


@pytest.mark.parametrize("kind", [OCTA, TETRA])
def test_partition_of_unity(kind):
    """for one pixel, sum_k dC/drgb_k + T_final = 1 (with dL/dC = 1 on one channel)."""
    scene, c = scenegen.small_scene(kind, 30, seed=4, width=32, height=24, size=(0.3, 0.8))
    sc = oscene(scene)
    f0 = oracle.forward(sc, c, mode=1, t_stop=0.0)
    ys, xs = np.nonzero(f0.out.T_final < 0.9)
    y, x = int(ys[0]), int(xs[0])
    G = np.zeros((3, 24, 32), np.float32)
    G[1, y, x] = 1.0
    f = oracle.forward(sc, c, mode=1, t_stop=0.0, dL_dimage=G)
    assert abs(f.out.drgb[:, 1].sum() + f.out.T_final[y, x] - 1.0) < 1e-12


@pytest.mark.parametrize("kind", [OCTA, TETRA])
def test_quaternion_gradient_orthogonal_to_q(kind):
    """the normalisation projects the rotation gradient orthogonal to q."""
    scene, c = scenegen.small_scene(kind, 10, seed=5, width=32, height=24)
    G = scenegen.upstream_grad(32, 24, seed=5)[0]
    f, g = oracle.forward_backward(oscene(scene), c, G, mode=1)
    q = scene["rot"].astype(np.float64)
    dots = np.abs((g.rot * q).sum(0))
    assert np.all(dots <= 1e-12 * (np.abs(g.rot).sum(0) * np.abs(q).sum(0) + 1e-300))


def test_zero_opacity_primitive_has_no_geometry_gradient():
    scene, c = scenegen.small_scene(OCTA, 6, seed=6, width=32, height=24)
    scene["opacity"][2] = -300.0
    G = scenegen.upstream_grad(32, 24, seed=6)[0]
    f, g = oracle.forward_backward(oscene(scene), c, G, mode=1)
    assert np.all(np.abs(g.pos[:, 2]) < 1e-100) and np.all(np.abs(g.dist[:, 2]) < 1e-100)
