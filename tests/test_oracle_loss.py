"""Pins for the loss oracle (oracle/loss.py).

* definition identities: SSIM(x, x) = 1 -> loss 0 and gradient 0 (lam = 1); lam = 0 -> pure L1;
* closed form: constant images a, b have S = (2ab + C1) / (a^2 + b^2 + C1) wherever the window
  lies inside the image (zero variance, A2 / B2 = C2 / C2);
* an independent library routine: SciPy's gaussian_filter (mode 'constant', radius 5, sigma 1.5)
  gives the same window sums, hence the same SSIM map, on random images;
* the analytic gradient against central finite differences of the loss (fp64).
"""
import math

import numpy as np
import pytest

from oracle import loss as OL


def rand_imgs(seed, C=3, H=20, W=23):
    rng = np.random.default_rng(seed)
    x = rng.uniform(0, 1, (C, H, W))
    y = np.clip(x + rng.normal(0, 0.2, x.shape), 0, 1)
    return x, y


def test_window_is_normalised_gaussian():
    w = OL.window()
    assert w.shape == (11, 11) and math.isclose(w.sum(), 1.0, rel_tol=1e-14)
    assert math.isclose(w[5, 6] / w[5, 5], math.exp(-1 / (2 * 1.5 ** 2)), rel_tol=1e-12)
    assert np.allclose(w, w.T) and np.allclose(w, w[::-1, ::-1])


def test_identical_images():
    x, _ = rand_imgs(0)
    L, g = OL.loss_and_grad(x, x, lam=1.0)
    assert abs(L) < 1e-12 and np.abs(g).max() < 1e-12
    assert math.isclose(OL.ssim(x, x), 1.0, rel_tol=1e-12)


def test_lambda_zero_is_l1():
    x, y = rand_imgs(1)
    L, g = OL.loss_and_grad(x, y, lam=0.0)
    assert math.isclose(L, np.abs(x - y).mean(), rel_tol=1e-13)
    assert np.allclose(g, np.sign(x - y) / x.size)


@pytest.mark.parametrize("a,b", [(0.2, 0.7), (0.5, 0.5), (0.9, 0.1)])
def test_constant_images_closed_form(a, b):
    H, W = 25, 27
    x, y = np.full((1, H, W), a), np.full((1, H, W), b)
    t = OL.ssim_terms(x[0], y[0], OL.window())
    inner = t["S"][5:H - 5, 5:W - 5]
    assert np.allclose(inner, (2 * a * b + OL.C1) / (a * a + b * b + OL.C1), rtol=1e-12)


@pytest.mark.parametrize("seed", range(3))
def test_ssim_map_matches_scipy_gaussian_filter(seed):
    from scipy.ndimage import gaussian_filter
    x, y = rand_imgs(seed, C=1, H=31, W=26)

    def gf(a):
        return gaussian_filter(a, sigma=1.5, mode="constant", cval=0.0, truncate=5.0 / 1.5)
    mx, my = gf(x[0]), gf(y[0])
    vx, vy, cxy = gf(x[0] ** 2) - mx ** 2, gf(y[0] ** 2) - my ** 2, gf(x[0] * y[0]) - mx * my
    S = ((2 * mx * my + OL.C1) * (2 * cxy + OL.C2)) / ((mx ** 2 + my ** 2 + OL.C1) * (vx + vy + OL.C2))
    t = OL.ssim_terms(x[0], y[0], OL.window())
    assert np.abs(t["S"] - S).max() < 1e-12


@pytest.mark.parametrize("lam", [0.2, 1.0])
def test_gradient_finite_differences(lam):
    x, y = rand_imgs(5, C=2, H=14, W=17)
    _, g = OL.loss_and_grad(x, y, lam)
    rng = np.random.default_rng(9)
    h = 1e-6
    for _ in range(40):
        c, i, j = rng.integers(2), rng.integers(14), rng.integers(17)
        if abs(x[c, i, j] - y[c, i, j]) < 1e-4:
            continue                      # stay away from the L1 kink
        xp, xm = x.copy(), x.copy()
        xp[c, i, j] += h
        xm[c, i, j] -= h
        fd = (OL.loss_and_grad(xp, y, lam)[0] - OL.loss_and_grad(xm, y, lam)[0]) / (2 * h)
        assert abs(fd - g[c, i, j]) <= 1e-6 * np.abs(g).max() + 1e-7 * abs(fd), (c, i, j, fd, g[c, i, j])


def test_batch_is_mean_of_views():
    x1, y1 = rand_imgs(2)
    x2, y2 = rand_imgs(3)
    L, G = OL.batch_loss_and_grad(np.stack([x1, x2]), np.stack([y1, y2]))
    La, ga = OL.loss_and_grad(x1, y1)
    Lb, gb = OL.loss_and_grad(x2, y2)
    assert math.isclose(L, (La + Lb) / 2, rel_tol=1e-14)
    assert np.allclose(G[0], ga / 2) and np.allclose(G[1], gb / 2)
