"""GPU parity of the L1 + SSIM loss kernels (lp_loss_grad: fused, or split through a workspace;
SURVEY §8 f1) against oracle/loss.py.

Tolerances: loss within 1e-5 relative; gradient |err| <= 1e-3 |g| + 1e-5 max|g| (north_star's
gradient bar), on sizes spanning several 32 x 32 tiles with ragged edges.
"""
import numpy as np
import pytest

from oracle import loss as OL
from tests import parity as PT

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module", autouse=True)
def _cuda():
    import torch
    assert torch.cuda.is_available(), "gpu tests need CUDA"
    from paper_2501_16312_b200 import _build
    _build.build()
    torch.cuda.set_device(0)


def images(V, H, W, seed):
    rng = np.random.default_rng(seed)
    x = rng.uniform(0, 1, (V, 3, H, W)).astype(np.float32)
    # structured target: smooth blobs + noise so SSIM is far from 0 and 1
    yy, xx = np.mgrid[0:H, 0:W]
    y = 0.5 + 0.4 * np.sin(xx / 7.0)[None, None] * np.cos(yy / 5.0)[None, None] + rng.normal(0, 0.05, x.shape)
    y = np.clip(0.6 * y + 0.4 * x, 0, 1).astype(np.float32)
    return x, y


def run(x, y, lam, split=False):
    """split: pass a G-map workspace (the two-kernel path; W % 4 == 0 only, else the fused kernel)."""
    import torch

    from paper_2501_16312_b200 import linprim as L
    X = torch.as_tensor(x, device="cuda")
    Y = torch.as_tensor(y, device="cuda")
    D = torch.empty_like(X)
    loss = torch.zeros(1, device="cuda")
    V, C, H, W = x.shape
    ws = torch.full((3 * X.numel(),), float("nan"), device="cuda") if split else None   # garbage in: must not leak
    L.lp_loss_grad(X, Y, D, loss, lam, 1.0 / (C * H * W * V), torch.cuda.current_stream(), workspace=ws)
    torch.cuda.synchronize()
    return float(loss.item()), D.cpu().numpy()


@pytest.mark.parametrize("V,H,W,seed", [(1, 32, 32, 0), (1, 45, 70, 1), (2, 96, 128, 2), (1, 100, 33, 3),
                                         (1, 7, 5, 4), (1, 470, 70, 5), (1, 217, 40, 6), (1, 252, 64, 7),
                                         (1, 33, 36, 8)])
@pytest.mark.parametrize("lam", [0.2, 1.0])
@pytest.mark.parametrize("split", [False, True])
def test_loss_and_grad_vs_oracle(V, H, W, seed, lam, split):
    x, y = images(V, H, W, seed)
    L_ref, G_ref = OL.batch_loss_and_grad(x.astype(np.float64), y.astype(np.float64), lam)
    L_got, G_got = run(x, y, lam, split)
    assert abs(L_got - L_ref) <= 1e-5 * abs(L_ref), (L_got, L_ref)
    ok, worst, rep, _ = PT.grad_close("dL/dimage", G_got, G_ref)
    assert ok, rep


@pytest.mark.parametrize("V,H,W,seed", [(1, 32, 32, 0), (2, 96, 128, 2), (1, 217, 40, 6), (1, 1060, 1600, 9),
                                         (3, 61, 100, 10)])
def test_split_path_is_bitwise_the_fused_kernel(V, H, W, seed):
    """The two-kernel path (G maps through the workspace) gives the fused kernel's dL/dx bit for bit
    (the same fp32 operations per output) and its loss within fp32 summation order."""
    x, y = images(V, H, W, seed)
    L0, G0 = run(x, y, 0.2, split=False)
    L1, G1 = run(x, y, 0.2, split=True)
    assert np.array_equal(G0, G1)
    assert abs(L1 - L0) <= 1e-6 * abs(L0)


def test_unaligned_workspace_falls_back_to_the_fused_kernel():
    """A workspace that is not 16-byte aligned (the TMA maps need it) runs the fused kernel: the same
    dL/dx bit for bit."""
    import torch

    from paper_2501_16312_b200 import linprim as L
    x, y = images(1, 96, 128, 11)
    X, Y = torch.as_tensor(x, device="cuda"), torch.as_tensor(y, device="cuda")
    outs = []
    for ws in (None, torch.empty(3 * X.numel() + 1, device="cuda")[1:]):
        D = torch.empty_like(X)
        loss = torch.zeros(1, device="cuda")
        L.lp_loss_grad(X, Y, D, loss, 0.2, 1.0 / X.numel(), torch.cuda.current_stream(), workspace=ws)
        torch.cuda.synchronize()
        outs.append(D.cpu().numpy())
    assert np.array_equal(outs[0], outs[1])


def test_lambda_zero_matches_l1_kernel():
    import torch

    from paper_2501_16312_b200 import linprim as L
    x, y = images(2, 50, 61, 7)
    _, G = run(x, y, 0.0)
    X, Y = torch.as_tensor(x, device="cuda"), torch.as_tensor(y, device="cuda")
    D = torch.empty_like(X)
    loss = torch.zeros(1, device="cuda")
    L.lp_l1_grad(X, Y, D, loss, 1.0 / x.size, torch.cuda.current_stream())
    torch.cuda.synchronize()
    assert np.array_equal(G, D.cpu().numpy())


def test_identical_images_zero_loss():
    x, _ = images(1, 40, 40, 3)
    L_got, G = run(x, x, 0.2)
    assert abs(L_got) < 1e-6 and np.abs(G).max() < 1e-9


def test_image_from_u8_is_numpy_division():
    """lp_image_from_u8 (the e2e path's 8-bit target staging): bitwise uint8 -> float32 / 255,
    vectorised body and scalar tail (odd lengths, unaligned tail)."""
    import torch

    from paper_2501_16312_b200 import linprim as L
    for n in (1, 15, 16, 17, 4099, 3 * 1060 * 1600):
        src = np.random.default_rng(n).integers(0, 256, n, dtype=np.uint8)
        s = torch.as_tensor(src, device="cuda")
        d = torch.empty(n, dtype=torch.float32, device="cuda")
        L.lp_image_from_u8(s, d, torch.cuda.current_stream())
        torch.cuda.synchronize()
        ref = src.astype(np.float32) / np.float32(255.0)
        assert np.array_equal(d.cpu().numpy().view(np.uint32), ref.view(np.uint32))
