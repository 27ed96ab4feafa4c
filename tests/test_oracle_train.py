"""Pins of oracle/train.py (the C5 step's Adam and learning-rate table)
against things other than itself: Adam's closed forms (Kingma & Ba, Alg. 1), torch.optim.Adam (a
library routine, fp64 on CPU), the paper's printed rates, and finite differences of the update."""
import numpy as np
import pytest

import oracle
from oracle import train as otr


def test_first_step_closed_form():
    """t = 1 from m = v = 0: m_hat = g, v_hat = g^2, so p -= lr g / (|g| + eps) (Alg. 1)."""
    rng = np.random.default_rng(0)
    p = rng.normal(size=50)
    g = rng.normal(size=50) * 10.0 ** rng.uniform(-8, 0, 50)
    p1, m1, v1 = otr.adam_step(p, g, np.zeros(50), np.zeros(50), [(0, 50, 0.01)], 1, eps=1e-8)
    np.testing.assert_allclose(p1, p - 0.01 * g / (np.abs(g) + 1e-8), rtol=0, atol=1e-15)
    np.testing.assert_allclose(m1, 0.1 * g, rtol=1e-14)
    np.testing.assert_allclose(v1, 0.001 * g * g, rtol=1e-14)


def test_constant_gradient_keeps_unit_steps():
    """A constant gradient gives m_hat = g and v_hat = g^2 at every t (the bias corrections are
    exact), so each step moves p by lr g / (|g| + eps)."""
    g = np.array([3e-4, -2.0, 5e-9])
    p = np.zeros(3)
    m = np.zeros(3)
    v = np.zeros(3)
    for t in range(1, 8):
        p, m, v = otr.adam_step(p, g, m, v, [(0, 3, 0.5)], t, eps=0.0)
    np.testing.assert_allclose(p, -7 * 0.5 * np.sign(g), rtol=1e-12)


def test_matches_torch_adam_with_groups():
    """Per-group learning rates, untouched elements outside every group, 5 steps: torch.optim.Adam
    (fp64, one param group per lr) gives the same parameters."""
    import torch
    rng = np.random.default_rng(1)
    n = 40
    groups = [(0, 3, 1e-3), (4, 6, 2e-2), (9, 10, 0.3), (12, 40, 5e-4)]
    p = rng.normal(size=n)
    m = np.zeros(n)
    v = np.zeros(n)
    tp = [torch.tensor(p[b:e], dtype=torch.float64, requires_grad=True) for b, e, _ in groups]
    opt = torch.optim.Adam([{"params": [t], "lr": lr} for t, (_, _, lr) in zip(tp, groups)], betas=(0.9, 0.999),
                           eps=1e-12)
    for t in range(1, 6):
        g = rng.normal(size=n) * 1e-3
        p, m, v = otr.adam_step(p, g, m, v, groups, t, eps=1e-12)
        for tt, (b, e, _) in zip(tp, groups):
            tt.grad = torch.tensor(g[b:e], dtype=torch.float64)
        opt.step()
    for tt, (b, e, _) in zip(tp, groups):
        np.testing.assert_allclose(p[b:e], tt.detach().numpy(), rtol=1e-13, atol=1e-15)
    outside = np.ones(n, bool)
    for b, e, _ in groups:
        outside[b:e] = False
    rng2 = np.random.default_rng(1)
    np.testing.assert_array_equal(p[outside], rng2.normal(size=n)[outside])


def test_lr_table_is_the_papers():
    """P:1169-1185 printed values; groups tile the flat buffer exactly."""
    n, deg = 10, 3
    g = otr.lr_table(oracle.OCTA, n, deg, extent=4.0)
    lrs = [lr for _, _, lr in g]
    assert lrs[1] == 1e-3 and lrs[3] == 2.5e-2 and lrs[4] == 2.5e-3 and lrs[5] == 1.25e-4
    assert lrs[2] == pytest.approx(4.0 * 1e-4 / 2.6) and lrs[0] == pytest.approx(4.0 * 1.6e-4)
    assert g[0][0] == 0 and all(g[k][1] == g[k + 1][0] for k in range(len(g) - 1))
    assert g[-1][1] == 3 * n + 4 * n + 3 * n + n + 16 * 3 * n
    assert g[4][1] - g[4][0] == 3 * n                        # DC coefficients: 3 per primitive


def test_update_sensitivity_by_finite_differences():
    rng = np.random.default_rng(3)
    n = 12
    groups = [(0, 12, 1e-2)]
    g = rng.normal(size=n) * 1e-4
    m = rng.normal(size=n) * 1e-4
    v = rng.uniform(1e-9, 1e-8, n)
    s = otr.adam_update_sensitivity(g, m, v, groups, 4, eps=1e-12)
    h = 1e-10
    pp = otr.adam_step(np.zeros(n), g + h, m, v, groups, 4, eps=1e-12)[0]
    pm = otr.adam_step(np.zeros(n), g - h, m, v, groups, 4, eps=1e-12)[0]
    np.testing.assert_allclose(np.abs((pp - pm) / (2 * h)), s, rtol=1e-5)


def test_c5_step_gradient_is_the_batch_loss_derivative():
    """c5_step's summed gradient (loss -> per-view dL/dimage -> render backward -> preprocess backward
    -> sum over views) equals central finite differences of the batch loss (the mean of the per-view
    3DGS losses) w.r.t. features, on a tiny two-view scene in fp64 geometry; and the returned
    parameters are adam_step of that gradient."""
    from oracle import loss as oloss
    from paper_2501_16312_b200 import scenegen
    from tests.helpers import oscene
    scene, cams = scenegen.make_scene("C5", seed=3, n=400)
    cams = [dict(c, width=24, height=20, cx=np.float32(12), cy=np.float32(10), fx=np.float32(14.0),
                 fy=np.float32(14.0)) for c in cams[:2]]
    osc = oscene(scene)
    imgs = np.stack([oracle.forward(osc, c, kappa=0.0, mode=1, t_stop=0.0).out.image for c in cams])
    rng = np.random.default_rng(0)
    targets = imgs + rng.choice([-1, 1], imgs.shape) * rng.uniform(0.05, 0.1, imgs.shape)
    n = scene["pos"].shape[1]
    groups = otr.lr_table(oracle.OCTA, n, 3, 4.0)
    z = np.zeros(groups[-1][1])
    r = otr.c5_step(osc, cams, targets, groups, z, z, 1, kappa=0.0, t_stop=0.0, mode=1)

    def batch_loss(sc):
        X = np.stack([oracle.forward(sc, c, kappa=0.0, mode=1, t_stop=0.0).out.image for c in cams])
        return oloss.batch_loss_and_grad(X, targets)[0]

    off = otr.offsets(oracle.OCTA, n, 3)
    go = np.abs(r["grad"][off["opacity"][0]:off["opacity"][1]])
    touched = np.argsort(-go)[:3]
    touched = touched[go[touched] > 0]
    assert touched.size >= 2
    checked = 0
    for i in touched:
        for name, comp in (("opacity", None), ("pos", 0), ("sh", 0)):
            sc = {k: np.array(v, copy=True) for k, v in scene.items() if isinstance(v, np.ndarray)}
            sc.update(kind=scene["kind"], sh_degree=scene["sh_degree"])
            arr = sc[name]
            idx = (i,) if comp is None else ((comp, i) if arr.ndim == 2 else (0, comp, i))
            h = 1e-3 if name != "pos" else 1e-4
            base = float(arr[idx])
            vals = []
            for sgn in (1, -1):
                arr[idx] = np.float32(base + sgn * h)
                vals.append(batch_loss(oscene(sc)))
            arr[idx] = np.float32(base)
            hh = (np.float64(np.float32(base + h)) - np.float64(np.float32(base - h))) / 2
            fd = (vals[0] - vals[1]) / (2 * hh)
            flat_i = off[name][0] + (np.ravel_multi_index(idx, arr.shape))
            an = r["grad"][flat_i]
            assert abs(fd - an) <= 2e-3 * abs(an) + 1e-9, (name, i, fd, an)
            checked += 1
    assert checked >= 6
    p1, _, _ = otr.adam_step(r["p0"], r["grad"], z, z, groups, 1)
    np.testing.assert_array_equal(p1, r["p"])
