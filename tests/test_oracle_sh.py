"""Pins for the SH colour (3DGS convention)."""
import math

import numpy as np
import pytest
from scipy.special import sph_harm_y

import oracle
from tests.helpers import cam, one_prim, oscene


def _sphere_quadrature(nt=24, nph=48):
    x, w = np.polynomial.legendre.leggauss(nt)          # cos(theta)
    ph = 2 * np.pi * np.arange(nph) / nph
    ct, PH = np.meshgrid(x, ph, indexing="ij")
    st = np.sqrt(1 - ct ** 2)
    dirs = np.stack([st * np.cos(PH), st * np.sin(PH), ct], -1).reshape(-1, 3)
    wts = (w[:, None] * np.full(nph, 2 * np.pi / nph)[None]).reshape(-1)
    return dirs, wts


def test_basis_orthonormal_on_sphere():
    dirs, wts = _sphere_quadrature()
    Y = np.stack([oracle.sh_basis(d)[0] for d in dirs])
    G = (Y * wts[:, None]).T @ Y
    assert np.abs(G - np.eye(16)).max() < 1e-12


def _real_sh(l, m, d):
    theta = np.arccos(np.clip(d[:, 2], -1, 1))
    phi = np.arctan2(d[:, 1], d[:, 0])
    if m == 0:
        return sph_harm_y(l, 0, theta, phi).real
    if m > 0:
        return math.sqrt(2) * (-1) ** m * sph_harm_y(l, m, theta, phi).real
    return math.sqrt(2) * (-1) ** m * sph_harm_y(l, -m, theta, phi).imag


def test_basis_is_textbook_real_sh_up_to_sign():
    """Each 3DGS basis function equals +-1 times a textbook real SH of the same degree
    (the sign table itself is the 3DGS convention, parity-unpinned: DESIGN.md)."""
    rng = np.random.default_rng(0)
    d = rng.standard_normal((200, 3))
    d /= np.linalg.norm(d, axis=1, keepdims=True)
    Y = np.stack([oracle.sh_basis(v)[0] for v in d])
    for l in range(4):
        ref = [_real_sh(l, m, d) for m in range(-l, l + 1)]
        for k in range(l * l, (l + 1) ** 2):
            best = min(min(np.abs(Y[:, k] - r).max(), np.abs(Y[:, k] + r).max()) for r in ref)
            assert best < 1e-12, (l, k)


def test_basis_gradient_finite_differences():
    rng = np.random.default_rng(1)
    for _ in range(10):
        d = rng.standard_normal(3)
        Y, dY = oracle.sh_basis(d)
        h = 1e-6
        for a in range(3):
            e = np.zeros(3)
            e[a] = h
            fd = (oracle.sh_basis(d + e)[0] - oracle.sh_basis(d - e)[0]) / (2 * h)
            assert np.allclose(dY[:, a], fd, atol=1e-8)


def test_colour_examples():
    c = cam()
    # all-zero coefficients -> 0.5
    s = one_prim(oracle.OCTA, (0.3, 0.2, 5.0), (1, 0, 0, 0), (0.1, 0.1, 0.1), sh_degree=3, rgb_dc=(0, 0, 0))
    pre = oracle.preprocess(oscene(s), c, mode=1)
    assert np.allclose(pre.rgb[0], 0.5, atol=1e-15)
    # DC only -> max(0, C0 c + 0.5)
    s = one_prim(oracle.OCTA, (0.3, 0.2, 5.0), (1, 0, 0, 0), (0.1, 0.1, 0.1), sh_degree=2, rgb_dc=(1.0, -0.5, -3.0))
    pre = oracle.preprocess(oscene(s), c, mode=1)
    C0 = 1.0 / (2.0 * math.sqrt(math.pi))
    assert np.allclose(pre.rgb[0], [C0 * 1.0 + 0.5, -0.5 * C0 + 0.5, 0.0], atol=1e-15)


def test_degree_gating():
    """degree 0 -> colour independent of the viewing direction."""
    s = one_prim(oracle.OCTA, (0.3, 0.2, 5.0), (1, 0, 0, 0), (0.1, 0.1, 0.1), sh_degree=0, rgb_dc=(0.3, 0.2, 0.1))
    a = oracle.preprocess(oscene(s), cam(), mode=1).rgb[0]
    b = oracle.preprocess(oscene(s), cam(t=(1.0, -2.0, 0.5)), mode=1).rgb[0]
    assert np.array_equal(a, b)
