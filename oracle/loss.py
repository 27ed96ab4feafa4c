"""CPU oracle of the training loss -- TEST INFRASTRUCTURE, fp64 NumPy.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s oracle legs may import this.

P:212 "we use the loss formulation of 3DGS, consisting of L1 and SSIM terms"; S:436 fixes it as
    L = (1 - lam) L1 + lam (1 - SSIM),   lam = 0.2,
SSIM with an 11 x 11 Gaussian window (sigma 1.5), C1 = 0.01^2, C2 = 0.03^2, averaged over channels
and pixels; the window is applied with zero padding so the SSIM map has the image's size (the
3DGS convention, reading 25).  Over a batch of V views the loss is the mean of the per-view
losses.  Everything below is the definition written out: the 2-D window sum is the plain
121-term sum (no separable factorisation), and the gradient is the chain rule through it.
"""
from __future__ import annotations

import numpy as np

C1 = 0.01 ** 2
C2 = 0.03 ** 2
WIN = 11
SIGMA = 1.5
LAMBDA = 0.2


def window(size=WIN, sigma=SIGMA):
    """Normalised 2-D Gaussian window w[i, j] = g[i] g[j], g[k] ~ exp(-(k - r)^2 / (2 sigma^2))."""
    r = size // 2
    g = np.exp(-((np.arange(size) - r) ** 2) / (2.0 * sigma * sigma))
    g /= g.sum()
    return np.outer(g, g)


def wsum(img, w):
    """out[p] = sum_{i,j} w[i,j] img[p + (i - r, j - r)], zero outside the image (same size)."""
    H, W = img.shape
    r = w.shape[0] // 2
    pad = np.zeros((H + 2 * r, W + 2 * r))
    pad[r:r + H, r:r + W] = img
    out = np.zeros((H, W))
    for i in range(w.shape[0]):
        for j in range(w.shape[1]):
            out += w[i, j] * pad[i:i + H, j:j + W]
    return out


def ssim_terms(x, y, w):
    """Per-channel window statistics and the SSIM map (one [H, W] channel)."""
    mx, my = wsum(x, w), wsum(y, w)
    exx, eyy, exy = wsum(x * x, w), wsum(y * y, w), wsum(x * y, w)
    vx, vy, cxy = exx - mx * mx, eyy - my * my, exy - mx * my
    A1, A2 = 2 * mx * my + C1, 2 * cxy + C2
    B1, B2 = mx * mx + my * my + C1, vx + vy + C2
    S = (A1 * A2) / (B1 * B2)
    return dict(mx=mx, my=my, A1=A1, A2=A2, B1=B1, B2=B2, S=S)


def ssim(x, y):
    """Mean SSIM of two [C, H, W] images."""
    w = window()
    return float(np.mean([ssim_terms(x[c], y[c], w)["S"].mean() for c in range(x.shape[0])]))


def loss_and_grad(x, y, lam=LAMBDA):
    """L = (1 - lam) mean|x - y| + lam (1 - mean SSIM(x, y)) over one [C, H, W] image and dL/dx.

    Gradient: with m_x = w*x, e_xx = w*(x^2), e_xy = w*(xy) (w* = zero-padded window sum), S depends
    on x only through them:
      dS/dm_x  = 2 m_y (A2 - A1) / (B1 B2) - 2 m_x S (1/B1 - 1/B2)
      dS/de_xy = 2 A1 / (B1 B2)
      dS/de_xx = -S / B2
    and the adjoint of the zero-padded window sum is the window sum with the mirrored window
    (w is symmetric), so dL/dx = -lam/N [w*(dS/dm_x) + y w*(dS/de_xy) + 2 x w*(dS/de_xx)]
    + (1 - lam)/N sign(x - y), N = C H W.
    """
    x = np.asarray(x, np.float64)
    y = np.asarray(y, np.float64)
    C, H, W = x.shape
    N = C * H * W
    w = window()
    wT = w[::-1, ::-1]
    L1 = np.abs(x - y).sum() / N
    Ssum = 0.0
    g = (1.0 - lam) * np.sign(x - y) / N
    for c in range(C):
        t = ssim_terms(x[c], y[c], w)
        Ssum += t["S"].sum()
        B1B2 = t["B1"] * t["B2"]
        d_mx = 2 * t["my"] * (t["A2"] - t["A1"]) / B1B2 - 2 * t["mx"] * t["S"] * (1 / t["B1"] - 1 / t["B2"])
        d_exy = 2 * t["A1"] / B1B2
        d_exx = -t["S"] / t["B2"]
        dS = wsum(d_mx, wT) + y[c] * wsum(d_exy, wT) + 2 * x[c] * wsum(d_exx, wT)
        g[c] += -lam * dS / N
    L = (1.0 - lam) * L1 + lam * (1.0 - Ssum / N)
    return L, g


def batch_loss_and_grad(X, Y, lam=LAMBDA):
    """Mean of the per-view losses over [V, C, H, W] batches and the gradient of that mean."""
    V = X.shape[0]
    Ls, Gs = zip(*(loss_and_grad(X[v], Y[v], lam) for v in range(V)))
    return float(np.mean(Ls)), np.stack(Gs) / V
