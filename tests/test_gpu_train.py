"""GPU parity of the C5 training-step helpers against oracle/train.py:
the fused Adam (lp_adam_step) element by element, including groups shorter than one float4 and
groups that start or end off a 16-byte boundary."""
import numpy as np
import pytest

from oracle import train as otr

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module", autouse=True)
def _cuda():
    import torch
    assert torch.cuda.is_available()
    from paper_2501_16312_b200 import _build
    _build.build()


def _adam_case(n, groups, steps, zero_grad, seed=0, eps=1e-15):
    import torch

    from paper_2501_16312_b200 import linprim as L
    rng = np.random.default_rng(seed)
    p0 = rng.normal(size=n).astype(np.float32)
    m0 = (rng.normal(size=n) * 1e-4).astype(np.float32)
    v0 = rng.uniform(0, 1e-8, n).astype(np.float32)
    p, m, v = (torch.from_numpy(a.copy()).cuda() for a in (p0, m0, v0))
    pr, mr, vr = p0.astype(np.float64), m0.astype(np.float64), v0.astype(np.float64)
    st = torch.cuda.current_stream()
    for t in range(1, steps + 1):
        g0 = (rng.normal(size=n) * 10.0 ** rng.uniform(-7, -3, n)).astype(np.float32)
        g = torch.from_numpy(g0).cuda()
        before = p.clone()
        L.lp_adam_step(p, g, m, v, groups, 0.9, 0.999, eps, t, st, zero_grad=zero_grad)
        torch.cuda.synchronize()
        # the oracle steps from the GPU's previous fp32 state (each step compared on its own)
        p_prev, m_prev, v_prev = (x.astype(np.float64) for x in (before.cpu().numpy(), mr, vr))
        # the ABI's betas are fp32: the oracle gets the same fp32 values (0.9f, 0.999f)
        pr, mr_new, vr_new = otr.adam_step(p_prev, g0, m_prev, v_prev, groups, t, b1=float(np.float32(0.9)),
                                           b2=float(np.float32(0.999)), eps=float(np.float32(eps)))
        got_p, got_m, got_v = p.cpu().numpy(), m.cpu().numpy(), v.cpu().numpy()
        upd = np.abs(pr - p_prev)
        tol = 2e-6 * upd + 2.0 ** -23 * np.abs(pr) + 1e-30
        assert np.all(np.abs(got_p - pr) <= tol), f"step {t}: worst {np.max(np.abs(got_p - pr) / tol):.3g}"
        # m = b1 m + (1 - b1) g may cancel: a few ulp of the two terms, not of the result
        tol_m = 2.0 ** -21 * (0.9 * np.abs(m_prev) + 0.1 * np.abs(g0.astype(np.float64))) + 1e-38
        assert np.all(np.abs(got_m - mr_new) <= tol_m), f"m: worst {np.max(np.abs(got_m - mr_new) / tol_m):.3g}"
        np.testing.assert_allclose(got_v, vr_new, rtol=1e-6, atol=1e-38)
        inside = np.zeros(n, bool)
        for b, e, _ in groups:
            inside[b:e] = True
        assert np.array_equal(got_p[~inside], p_prev[~inside].astype(np.float32)), "element outside every group changed"
        gnow = g.cpu().numpy()
        if zero_grad:
            assert np.all(gnow[inside] == 0) and np.array_equal(gnow[~inside], g0[~inside])
        else:
            assert np.array_equal(gnow, g0)
        mr, vr = got_m.astype(np.float64), got_v.astype(np.float64)


@pytest.mark.parametrize("zero_grad", [False, True])
def test_adam_small_and_unaligned_groups(zero_grad):
    """a group of 1-3 elements starting on a multiple of 4 was never updated."""
    groups = [(0, 3, 1e-3), (4, 6, 2e-2), (9, 10, 0.3), (13, 4113, 5e-4), (4113, 4116, 1e-2), (4120, 9000, 2.5e-3)]
    _adam_case(9003, groups, 3, zero_grad)


def test_adam_paper_groups_layout():
    """The paper's six groups over a C5-shaped flat buffer (1k primitives, SH degree 3)."""
    n = 1003
    groups = otr.lr_table(0, n, 3, extent=4.0)
    _adam_case(groups[-1][1] + 5, groups, 2, False, seed=4)
