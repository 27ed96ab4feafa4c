"""GPU parity of the C5 training step AS BENCH.PY TIMES IT (row a13): the
TrainStep object (8 views, one stream each -- bench.py's default -- or over 4 streams with the split
preprocess; lp_loss_grad 3DGS L1 + SSIM,
lp_raster_bwd, the two-pack lp_preprocess_bwd_assign, the fused Adam with the paper's learning
rates) against oracle/train.py.c5_step (oracle.forward -> oracle.loss -> oracle.render backward ->
oracle.preprocess_bwd -> sum -> Adam, fp64), at reduced N and resolution, element by element:
images, loss, dL/dimage, every feature-gradient group, and the post-step parameters, m and v.

Inputs: make_scene("C5", n=3000) with the 8 ring cameras at 96 x 64; targets = the ORACLE's
images + a seeded +-U(0.01, 0.05) offset per pixel (so no L1 sign sits within rounding of 0);
Adam state warm (t = 10, m and v seeded at the scale of the oracle's gradient) so the update is
a smooth function of the gradient."""
import numpy as np
import pytest

import oracle
from oracle import train as otr
from paper_2501_16312_b200 import scenegen
from tests import parity as PT
from tests.helpers import oscene

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module", autouse=True)
def _cuda():
    import torch
    assert torch.cuda.is_available()
    from paper_2501_16312_b200 import _build
    _build.build()


def _small_c5(seed, n=3000, W=96, H=64):
    scene, cams = scenegen.make_scene("C5", seed=seed, n=n)
    f = np.float32(W / 2 / np.tan(np.deg2rad(30.0)))
    cams = [dict(c, width=W, height=H, cx=np.float32(W / 2), cy=np.float32(H / 2), fx=f, fy=f) for c in cams]
    return scene, cams


@pytest.mark.parametrize("streams,split_pre", [(8, False), (4, True)])   # bench's default, the split variant
@pytest.mark.parametrize("loss", ["l1ssim", "l1"])
def test_c5_step_vs_oracle(loss, streams, split_pre, parity_log):
    import torch

    from paper_2501_16312_b200 import step as S
    scene, cams = _small_c5(seed=0)
    osc = oscene(scene)
    n = scene["pos"].shape[1]
    fwd0 = [oracle.forward(osc, c) for c in cams]
    masked = sum(int((f.out.m_stop < PT.STOP_MARGIN).sum()) for f in fwd0)
    assert masked == 0, "choose a scene without stop-margin pixels (the loss spreads them over a window)"
    X0 = np.stack([f.out.image for f in fwd0])
    rng = np.random.default_rng(7)
    targets = (X0 + rng.choice([-1.0, 1.0], X0.shape) * rng.uniform(0.01, 0.05, X0.shape)).astype(np.float32)
    lam = 0.2 if loss == "l1ssim" else 0.0
    groups = otr.lr_table(oracle.OCTA, n, 3, extent=4.0)
    P = groups[-1][1]
    # oracle gradient first (zero state), then the warm Adam state at its scale
    z = np.zeros(P)
    r = otr.c5_step(osc, cams, targets.astype(np.float64), groups, z, z, 1, lam=lam, bounds=True)
    g_o = r["grad"]
    m0 = np.zeros(P, np.float32)
    v0 = np.zeros(P, np.float32)
    for b, e, _ in groups:
        sc = np.abs(g_o[b:e]).max()
        m0[b:e] = (rng.normal(0, 0.3, e - b) * sc).astype(np.float32)
        v0[b:e] = (rng.uniform(0.5, 2.0, e - b) * sc * sc).astype(np.float32)
    t = 10
    b1, b2, eps = float(np.float32(0.9)), float(np.float32(0.999)), float(np.float32(1e-15))
    p_o, m_o, v_o = otr.adam_step(r["p0"], g_o, m0.astype(np.float64), v0.astype(np.float64), groups, t, b1, b2, eps)

    # ---- the CUDA step, exactly as bench.py runs it
    ds = S.device_scene(scene, "cuda")
    ts = S.TrainStep(ds, cams, len(cams), targets=torch.from_numpy(targets).cuda(), loss=loss, streams=streams,
                     split_pre=split_pre, assign=True)
    ts.m.copy_(torch.from_numpy(m0))
    ts.v.copy_(torch.from_numpy(v0))
    p_before = ds.flat.clone()
    ts.run(0, t=t)
    torch.cuda.synchronize()
    assert not ts.overflowed()
    assert torch.equal(p_before.cpu(), torch.from_numpy(r["p0"].astype(np.float32)))

    # images and loss
    img = ts.img.cpu().numpy()
    assert np.abs(img - r["images"]).max() <= PT.IMG_TOL
    loss_gpu = float(ts.loss_buf[0])
    assert abs(loss_gpu - r["loss"]) <= 1e-5 * abs(r["loss"]), (loss_gpu, r["loss"])
    # dL/dimage (scale = 1 / (3 H W V): the mean over views of the per-view means, like the oracle)
    ok, worst_dl, rep, _ = PT.grad_close("dL/dimage", ts.dL.cpu().numpy(), r["dL"])
    assert ok, rep
    # the step's gradient, every group (the second K5 pack accumulates onto the first's assignment)
    off = otr.offsets(oracle.OCTA, n, 3)
    shapes = {"pos": (3, n), "rot": (4, n), "dist": (3, n), "opacity": (n,), "sh": (16, 3, n)}

    class G:
        pass
    g, gb = G(), G()
    for k, (b, e) in off.items():
        setattr(g, k, g_o[b:e].reshape(shapes[k]))
        setattr(gb, k, r["bound"][b:e].reshape(shapes[k]))
    for f in r["fwd"]:
        r["flagged"] |= PT.screen_flags(f.pre) & (f.pre.tiles_touched > 0)
    ok, worst, reports, n_cond, n_clamp = PT.check_gradients(ds.grad_dict(), g, gb, None, r["flagged"],
                                                             clamp=r["clamp"])
    parity_log(f"c5 step ({loss}, {streams} streams{', split' if split_pre else ''})", views=len(cams), hit_prims=int(np.isfinite(r["fwd"][0].out.m_face).sum()),
               flagged=int(r["flagged"].sum()), clamp=n_clamp, cond_elems=n_cond, worst=dict(worst, dL=worst_dl))
    assert ok, "; ".join(reports)

    # post-step parameters, m, v: the oracle's Adam of the oracle's gradient; tolerance = the
    # gradient bar propagated through Adam (|d p / d g|) + fp32 rounding of the update and of p
    grad_tol = np.zeros(P)
    flag_el = np.zeros(P, bool)
    for k, (b, e) in off.items():
        ref = g_o[b:e]
        grad_tol[b:e] = PT.GRAD_RTOL * np.abs(ref) + PT.GRAD_ATOL_REL * np.abs(ref).max() + r["bound"][b:e]
        if k in ("pos", "rot", "dist"):
            fl = np.broadcast_to(r["flagged"] | r["clamp"].any(1), shapes[k]).reshape(-1)
            flag_el[b:e] = fl
        if k == "sh":
            flag_el[b:e] = np.broadcast_to(r["clamp"].T[None], shapes[k]).reshape(-1)
    sens = otr.adam_update_sensitivity(g_o, m0.astype(np.float64), v0.astype(np.float64), groups, t, b1, b2, eps)
    p_g = ds.flat.cpu().numpy().astype(np.float64)
    tol_p = sens * grad_tol + 4e-6 * np.abs(p_o - r["p0"]) + 2.0 ** -23 * np.abs(p_o) + 1e-30
    bad = (np.abs(p_g - p_o) > tol_p) & ~flag_el
    assert not bad.any(), f"{bad.sum()} parameters off; worst {np.max(np.abs(p_g - p_o)[~flag_el] / tol_p[~flag_el]):.3g}"
    m_g, v_g = ts.m.cpu().numpy().astype(np.float64), ts.v.cpu().numpy().astype(np.float64)
    tol_m = 0.1 * grad_tol + 2.0 ** -21 * (0.9 * np.abs(m0) + 0.1 * np.abs(g_o)) + 1e-38
    assert not ((np.abs(m_g - m_o) > tol_m) & ~flag_el).any()
    tol_v = 2e-3 * 2 * np.abs(g_o) * grad_tol + 2e-6 * v_o + 1e-38
    assert not ((np.abs(v_g - v_o) > tol_v) & ~flag_el).any()
    # the gradient left in the buffer is the step's (assign semantics: nothing zeroes it)
    assert float(ds.grad.abs().max()) > 0


def test_kernel_launch_claim_matches_profiler():
    """bench.py's gpu_launches claim (TrainStep.kernel_launches() per step) equals the liblinprim
    kernels a CUDA profiler sees in one full-size C5 step (bench's default launch configuration)."""
    import torch
    from torch.profiler import ProfilerActivity, profile

    from paper_2501_16312_b200 import linprim as L, render, step as S
    scene, cams = scenegen.make_scene("C5", seed=0)
    ds = S.device_scene(scene, "cuda")
    rr = render.Renderer(ds, cams, count_stats=True)
    tg = rr.forward().clone()
    E = max(int(rr.counters(i)[L.LP_CNT_ENTRIES]) for i in range(len(cams)))
    del rr
    ts = S.TrainStep(ds, cams, len(cams), targets=tg, capacity=int(E * 1.3) + 4096, loss_slots=16)
    for i in range(2):
        ts.run(i)
    torch.cuda.synchronize()
    with profile(activities=[ProfilerActivity.CUDA]) as prof:
        ts.run(5)
        torch.cuda.synchronize()
    ours = [e.name for e in prof.events()
            if e.device_type == torch.autograd.DeviceType.CUDA and "lp::k_" in e.name]
    assert len(ours) == ts.kernel_launches(), (len(ours), ts.kernel_launches())
