"""GPU parity: the CUDA path (through the C-ABI) against the CPU oracle on the same seeded inputs.

Bit-exact: tiles_touched, tile rect, depth key, canonical geometry bits, sorted (tile, id) list,
per-tile ranges.  Tolerances (north_star): image max |err| <= 1e-4; gradients |err| <= 1e-3 |g| +
1e-5 * max|g| per group.  Stop-index flips and entry/exit-face switches are masked / flagged from
the oracle's margins; the counts are asserted to stay small.
"""
import numpy as np
import pytest

import oracle
from paper_2501_16312_b200 import scenegen
from tests import parity as PT
from tests.canonical_np import canonical
from tests.helpers import oscene

pytestmark = pytest.mark.gpu

OCTA, TETRA = scenegen.OCTA, scenegen.TETRA
K_OF = {OCTA: 3, TETRA: 4}


@pytest.fixture(scope="module", autouse=True)
def _cuda():
    import torch
    assert torch.cuda.is_available(), "gpu tests need CUDA"
    from paper_2501_16312_b200 import _build
    _build.build()
    torch.cuda.set_device(0)


def check_preprocess(scene, cam, r, v=0, kappa=0.1, filter3d=None, exact=False):
    n = scene["pos"].shape[1]
    K = K_OF[scene["kind"]]
    got = PT.frame_arrays(r, v, n, K)
    pre = oracle.preprocess(oscene(scene, filter3d), cam, kappa=kappa, mode=0, exact=exact)
    assert np.array_equal(got["tiles_touched"], pre.tiles_touched), "tiles_touched"
    assert np.array_equal(got["rect"], pre.rect), "rect"
    assert np.array_equal(got["depth_key"], pre.depth_key), "depth key"
    if "canon" in got:
        assert np.array_equal(got["canon"].view(np.uint32), pre.canon.view(np.uint32)), "canonical geometry bits"
    c = got["counters"]
    assert c[2] == int((pre.flag == 1).sum()) and c[3] == int((pre.flag == 0).sum())
    assert c[4] == int((pre.tiles_touched > 0).sum())
    return got, pre


def check_binning(got, pre, cam):
    keys, vals, ranges = oracle.bin_tiles(pre, cam["width"], cam["height"])
    assert got["E"] == len(vals)
    assert np.array_equal(got["sorted_val"], vals), "sorted ids"
    assert np.array_equal(got["sorted_tile"].astype(np.uint64), keys >> np.uint64(32)), "sorted tiles"
    assert np.array_equal(got["ranges"].astype(np.int64), ranges), "ranges"
    # the full 64-bit (tile | depth) key of every entry, reconstructed
    k64 = (got["sorted_tile"].astype(np.uint64) << np.uint64(32)) | got["depth_key"][got["sorted_val"]].astype(np.uint64)
    assert np.array_equal(k64, keys)
    c = got["counters"]
    assert c[7] in (0, c[4]), "depth-sorted primitives = visible ones (radix method, n > 4096), else unused"
    return keys, vals, ranges


def full_parity(scene, cam, kappa=0.1, t_stop=1e-3, bg=(0.0, 0.0, 0.0), seed=0, grads=True, filter3d=None,
                max_masked=0.01, max_flagged=0.03, exact=False, loose=0.1, deterministic=False):
    W, H = cam["width"], cam["height"]
    osc = oscene(scene, filter3d)
    f0 = oracle.forward(osc, cam, kappa=kappa, t_stop=t_stop, bg=bg, exact=exact)
    mask = f0.out.m_stop < PT.STOP_MARGIN
    assert mask.mean() <= max_masked, f"too many stop-margin pixels {mask.mean()}"
    G = scenegen.upstream_grad(W, H, seed=seed)[0] * (~mask)[None].astype(np.float32) if grads else None
    ds, r, img = PT.gpu_run(scene, [cam], G=G, kappa=kappa, t_stop=t_stop, bg=bg, filter3d=filter3d, exact=exact,
                            deterministic=deterministic)
    got, pre = check_preprocess(scene, cam, r, kappa=kappa, filter3d=filter3d, exact=exact)
    check_binning(got, pre, cam)
    im = img[0].cpu().numpy()
    err = np.abs(im - f0.out.image)[:, ~mask]
    assert err.max(initial=0.0) <= PT.IMG_TOL, f"image max err {err.max()}"
    assert np.abs(got["T_final"] - f0.out.T_final)[~mask].max(initial=0.0) <= PT.IMG_TOL
    assert np.array_equal(got["n_proc"][~mask], f0.out.n_proc[~mask]), "n_proc"
    assert got["counters"][8] == int(f0.out.n_proc.sum()) or mask.any()
    if not grads:
        return
    fb, g = oracle.forward_backward(osc, cam, G, kappa=kappa, t_stop=t_stop, bg=bg, exact=exact, bounds=True)
    gb = oracle.feature_bounds(osc, cam, fb.pre, fb.out, exact=exact)
    touched = np.isfinite(fb.out.face_margin)
    flagged = (fb.out.face_margin < PT.FACE_MARGIN) | (PT.screen_flags(fb.pre, exact) & touched)
    assert flagged.sum() <= max(2, max_flagged * touched.sum()), f"flagged {flagged.sum()} of {touched.sum()}"
    ok, worst, reports, n_cond, n_clamp = PT.check_gradients(ds.grad_dict(), g, gb, fb.pre, flagged, loose=loose)
    import os
    PT.log(os.environ.get("PYTEST_CURRENT_TEST", "full_parity").split(" ")[0].split("::")[-1], pixels=W * H,
           masked_px=int(mask.sum()), hit_prims=int(touched.sum()), flagged=int(flagged.sum()), clamp=n_clamp,
           cond_elems=n_cond, worst=worst)
    assert ok, "; ".join(reports)
    return reports


# ------------------------------------------------------------------------------------------------

def test_c1_full_forward_backward():
    """configs[0]: 1k random octahedra, SH deg 0, 128x128, fwd+bwd vs the oracle."""
    scene, cams = scenegen.make_scene("C1", seed=0)
    full_parity(scene, cams[0])


@pytest.mark.parametrize("kind", [OCTA, TETRA])
@pytest.mark.parametrize("seed", range(6))
def test_random_small_scenes(kind, seed):
    scene, cam = scenegen.small_scene(kind, 300, seed=seed, width=96, height=72, sh_degree=seed % 4,
                                      opacity_mu=0.5 * (seed % 3))
    full_parity(scene, cam, seed=seed, bg=(0.1, 0.2, 0.3) if seed % 2 else (0, 0, 0))


@pytest.mark.parametrize("kind", [OCTA, TETRA])
@pytest.mark.parametrize("kappa,t_stop", [(0.0, 1e-3), (0.1, 0.0), (0.5, 1e-2)])
def test_filter_and_stop_variants(kind, kappa, t_stop):
    scene, cam = scenegen.small_scene(kind, 250, seed=11, width=80, height=64, sh_degree=2, opacity_mu=1.0)
    full_parity(scene, cam, kappa=kappa, t_stop=t_stop, seed=3)


@pytest.mark.parametrize("kind", [OCTA, TETRA])
def test_3d_filter(kind):
    scene, cam = scenegen.small_scene(kind, 200, seed=12, width=64, height=48, sh_degree=1)
    f3 = np.random.default_rng(0).uniform(0.0, 0.05, 200).astype(np.float32)
    full_parity(scene, cam, filter3d=f3, seed=4)


@pytest.mark.parametrize("kind", [OCTA, TETRA])
@pytest.mark.parametrize("seed", range(3))
def test_edge_scenes(kind, seed):
    """Tile-border stragglers, off-screen, behind camera, znear, sub-pixel, huge, alpha ~ 0,
    duplicate depths, zero quaternion, d <= 0, NaN; image size not a multiple of 16."""
    scene, cam = scenegen.edge_scene(kind, seed=seed)
    full_parity(scene, cam, seed=seed)


def test_canonical_matches_numpy_arbiter_on_gpu():
    scene, cam = scenegen.small_scene(OCTA, 5000, seed=5, width=333, height=211)
    ds, r, img = PT.gpu_run(scene, [cam])
    got = PT.frame_arrays(r, 0, 5000, 3)
    ref = canonical(scene, cam, kappa=0.1)
    assert np.array_equal(got["canon"].view(np.uint32), ref["canon"].view(np.uint32))
    assert np.array_equal(got["tiles_touched"], ref["tiles_touched"])


def test_empty_and_degenerate_inputs():
    import torch
    # all primitives culled
    scene, cam = scenegen.small_scene(OCTA, 50, seed=1, width=40, height=30)
    scene["pos"][2] = -5.0
    ds, r, img = PT.gpu_run(scene, [cam], G=np.ones((3, 30, 40), np.float32), bg=(0.25, 0.5, 0.75))
    assert torch.allclose(img[0, 0], torch.full_like(img[0, 0], 0.25))
    assert float(ds.grad.abs().max()) == 0.0
    # a single primitive, 1x1 image
    scene, cam = scenegen.small_scene(TETRA, 1, seed=2, width=1, height=1)
    full_parity(scene, cam, seed=1)


@pytest.mark.parametrize("culled", ["all", "half"])
def test_radix_depth_sort_drops_invisible(culled):
    """The multi-block radix path (n > 4096): the first depth pass drops the invisible primitives and
    the later passes, the scan and the emission run over the kept ones only (LP_CNT_SORTED); with every
    primitive culled the list is empty and the image is the background."""
    import torch

    from paper_2501_16312_b200 import linprim as L
    n = 6000
    scene, cam = scenegen.small_scene(OCTA, n, seed=31, width=120, height=90)
    behind = np.arange(n) % 2 == 0 if culled == "half" else np.ones(n, bool)
    scene["pos"][2][behind] = -5.0
    ds, r, img = PT.gpu_run(scene, [cam], sort_method=L.LP_SORT_RADIX, capacity=1 << 16, bg=(0.25, 0.5, 0.75))
    got = PT.frame_arrays(r, 0, n, K_OF[OCTA])
    pre = oracle.preprocess(oscene(scene), cam)
    vis = int((pre.tiles_touched > 0).sum())
    assert got["counters"][7] == vis and (vis == 0) == (culled == "all")
    check_binning(got, pre, cam)
    if culled == "all":
        assert got["E"] == 0 and torch.allclose(img[0, 2], torch.full_like(img[0, 2], 0.75))
    else:   # the same lists as the bucket path -> the same image, bit for bit
        _, _, img_b = PT.gpu_run(scene, [cam], sort_method=L.LP_SORT_BUCKET, bg=(0.25, 0.5, 0.75))
        assert torch.equal(img, img_b)


def test_multi_view_call_and_accumulation():
    """Two views in one Renderer: gradients accumulate (+=) over views."""
    import torch
    scene, cams = scenegen.make_scene("C5", seed=0, n=3000)
    cams = [dict(c, width=96, height=64, cx=np.float32(48), cy=np.float32(32),
                 fx=np.float32(83.1), fy=np.float32(83.1)) for c in cams[:2]]
    G = scenegen.upstream_grad(96, 64, seed=0, n_views=2)
    ds, r, img = PT.gpu_run(scene, cams, G=G)
    osc = oscene(scene)
    tot = None
    for v in range(2):
        f, g = oracle.forward_backward(osc, cams[v], G[v])
        assert np.abs(img[v].cpu().numpy() - f.out.image).max() <= PT.IMG_TOL
        tot = g.opacity if tot is None else tot + g.opacity
    ok, worst, rep, _ = PT.grad_close("opacity", ds.grad_dict()["opacity"].cpu().numpy(), tot)
    assert ok, rep


@pytest.mark.parametrize("n_views", [1, 6])
def test_preprocess_bwd_assign_equals_zeroed_accumulate(n_views):
    """lp_preprocess_bwd_assign (every primitive's feature gradient SET, the old contents never read;
    6 views = two view packs: the second one accumulates) gives bit for bit what lp_preprocess_bwd
    gives on a zeroed gradient, from the same raster moments; densification statistics accumulate."""
    import torch
    from paper_2501_16312_b200 import linprim as L
    from paper_2501_16312_b200 import render
    scene, cams = scenegen.make_scene("C5", seed=1, n=4000)
    cams = [dict(c, width=80, height=64, cx=np.float32(40), cy=np.float32(32),
                 fx=np.float32(69.3), fy=np.float32(69.3)) for c in cams[:n_views]]
    ds = render.DeviceScene(scene)
    ds.track_mean2d()
    r = render.Renderer(ds, cams)
    img = r.forward()
    G = torch.from_numpy(scenegen.upstream_grad(80, 64, seed=2, n_views=n_views)).cuda().contiguous()
    st = torch.cuda.current_stream()
    fa = render.frames_array(r.frames)
    ca = r._cams(list(range(n_views)))
    L.lp_raster_bwd(ca, r.cfg, fa, G, st)
    ds.grad.zero_()
    L.lp_preprocess_bwd(ds.prims, ca, r.cfg, fa, ds.grads, st)
    ref = ds.grad.clone()
    m2d_ref = ds.mean2d.clone()
    ds.grad.fill_(7.0)                      # stale garbage: must be overwritten, never read
    L.lp_preprocess_bwd_assign(ds.prims, ca, r.cfg, fa, ds.grads, st)
    torch.cuda.synchronize()
    assert torch.equal(ds.grad, ref)
    # the statistics accumulated over both calls (equal up to the summation order of the packs)
    assert torch.allclose(ds.mean2d, 2 * m2d_ref, rtol=1e-6, atol=0)
    assert img.shape[0] == n_views and float(ref.abs().sum()) > 0


def test_capacity_error_and_async_overflow_flag():
    import ctypes as C

    import torch

    from paper_2501_16312_b200 import linprim as L
    from paper_2501_16312_b200 import render
    scene, cam = scenegen.small_scene(OCTA, 400, seed=3, width=64, height=48)
    ds = render.DeviceScene(scene)
    fr = render.Frame(ds.kind, ds.n, 64, 48, capacity=16)
    cams = L.cameras([cam])
    cfg = L.raster_cfg()
    fa = render.frames_array([fr])
    st = torch.cuda.current_stream()
    L.lp_preprocess(ds.prims, cams, cfg, fa, st)
    ne = (C.c_int64 * 1)()
    assert L.lp_bin_sort(cams, fa, st, ne) == L.LP_ERR_CAPACITY
    pre = oracle.preprocess(oscene(scene), cam)
    assert ne[0] == int(pre.tiles_touched.sum())
    L.lp_preprocess(ds.prims, cams, cfg, fa, st)
    L.lp_bin_sort(cams, fa, st, None)                     # async: no truncation is silent
    cnt = L.lp_frame_counters(fa[0], st)
    assert cnt[L.LP_CNT_OVERFLOW] == 1 and cnt[L.LP_CNT_ENTRIES] == ne[0]


def test_l1_grad_and_adam_vs_torch():
    import torch

    from paper_2501_16312_b200 import linprim as L
    g = torch.Generator(device="cuda").manual_seed(0)
    a = torch.rand(3 * 37 * 29 + 3, device="cuda", generator=g)
    b = torch.rand(a.numel(), device="cuda", generator=g)
    dL = torch.empty_like(a)
    loss = torch.zeros(1, device="cuda")
    st = torch.cuda.current_stream()
    L.lp_l1_grad(a, b, dL, loss, 0.5, st)
    assert torch.equal(dL, 0.5 * torch.sign(a - b))
    assert torch.allclose(loss, 0.5 * (a - b).abs().sum(), rtol=1e-5)
    p = torch.randn(1000, device="cuda", generator=g)
    gr = torch.randn(1000, device="cuda", generator=g)
    m = torch.zeros_like(p)
    v = torch.zeros_like(p)
    p_ref, m_ref, v_ref = p.clone(), m.clone(), v.clone()
    groups = [(0, 300, 1e-3), (300, 900, 2.5e-2)]
    for step in (1, 2, 3):
        L.lp_adam_step(p, gr, m, v, groups, 0.9, 0.999, 1e-15, step, st)
        m_ref = 0.9 * m_ref + 0.1 * gr
        v_ref = 0.999 * v_ref + 0.001 * gr * gr
        for b0, e0, lr in groups:
            mh = m_ref[b0:e0] / (1 - 0.9 ** step)
            vh = v_ref[b0:e0] / (1 - 0.999 ** step)
            p_ref[b0:e0] -= lr * mh / (vh.sqrt() + 1e-15)
        m_ref[900:] = 0
        v_ref[900:] = 0
    assert torch.allclose(p, p_ref, rtol=1e-5, atol=1e-6)
    assert torch.equal(p[900:], p_ref[900:])


@pytest.mark.parametrize("kind", [OCTA, TETRA])
def test_radix_and_bucket_sort_agree(kind):
    """Both lp_bin_sort methods produce the oracle's (tile, depth, id) order bit for bit."""
    from paper_2501_16312_b200 import linprim as L
    scene, cam = scenegen.small_scene(kind, 3000, seed=21, width=200, height=150)
    outs = []
    for method in (L.LP_SORT_RADIX, L.LP_SORT_BUCKET):
        ds, r, img = PT.gpu_run(scene, [cam], sort_method=method)
        got = PT.frame_arrays(r, 0, 3000, K_OF[kind])
        pre = oracle.preprocess(oscene(scene), cam)
        check_binning(got, pre, cam)
        outs.append(img.cpu().numpy())
    assert np.array_equal(outs[0], outs[1])


def test_oversize_tile_bucket_uses_global_network():
    """A tile list longer than the shared-memory capacity (4096) is sorted in place in global memory."""
    from paper_2501_16312_b200 import linprim as L
    # primitives of a few pixels (smaller ones at the image centre would fall between pixel centres
    # and touch no tile at all)
    scene, cam = scenegen.small_scene(OCTA, 5000, seed=22, width=16, height=16, size=(0.3, 0.6))
    scene["pos"][2] = np.random.default_rng(0).uniform(3.0, 8.0, 5000).astype(np.float32)
    scene["pos"][0] = 0.0
    scene["pos"][1] = 0.0
    scene["pos"][2][10] = scene["pos"][2][11]            # a depth tie inside the big bucket
    pre = oracle.preprocess(oscene(scene), cam)
    assert int(pre.tiles_touched.sum()) > 4096           # one tile list beyond the shared-memory capacity
    ds, r, img = PT.gpu_run(scene, [cam], sort_method=L.LP_SORT_BUCKET)
    check_binning(PT.frame_arrays(r, 0, 5000, K_OF[OCTA]), pre, cam)
    full_parity(scene, cam, seed=5, grads=False, max_masked=0.05)   # image / T / n_proc (default method)


@pytest.mark.parametrize("which", ["C1", "small_octa", "small_tetra", "edge"])
def test_small_frame_binning_path(which):
    """Frames with n <= 4096 and capacity <= 8192 bin in one CTA per step (k_small_depth_scan,
    k_small_tile_sort): the sorted lists, ranges and image equal the oracle's and the multi-block
    path's bit for bit, and the (deterministic-mode) gradients are identical too."""
    from paper_2501_16312_b200 import linprim as L
    if which == "C1":
        scene, cams = scenegen.make_scene("C1", seed=0)
        cam = cams[0]
    elif which == "edge":
        scene, cam = scenegen.edge_scene(TETRA, seed=1)
    else:
        scene, cam = scenegen.small_scene(OCTA if which == "small_octa" else TETRA, 1500, seed=7, width=150,
                                          height=100)
    G = scenegen.upstream_grad(cam["width"], cam["height"], seed=3)[0]
    pre = oracle.preprocess(oscene(scene), cam)
    E = int(pre.tiles_touched.astype(np.int64).sum())
    assert E + 16 <= 8192
    outs = []
    for cap in (E + 16, 1 << 16):        # small path, then the multi-block path
        ds, r, img = PT.gpu_run(scene, [cam], G=G, capacity=cap, deterministic=True,   # bitwise gradients
                                sort_method=L.LP_SORT_RADIX)
        got = PT.frame_arrays(r, 0, scene["pos"].shape[1], K_OF[scene["kind"]])
        check_binning(got, pre, cam)
        outs.append((img.cpu().numpy(), ds.grad.cpu().numpy()))
    assert np.array_equal(outs[0][0], outs[1][0]) and np.array_equal(outs[0][1], outs[1][1])


@pytest.mark.parametrize("kind", [OCTA, TETRA])
@pytest.mark.parametrize("n_views", [2, 3, 4, 5])
def test_multi_view_preprocess_equals_single_view_calls(kind, n_views):
    """One lp_preprocess call over several views (the view-interleaved K1 grid) writes every frame
    output (tile counts, rects, depth keys, records, canonical geometry) bitwise as one single-view
    call per view does; the 3D filter and an invalid primitive included."""
    import torch
    from paper_2501_16312_b200 import linprim as L
    from paper_2501_16312_b200 import render
    n = 5000
    if kind == OCTA:
        scene, cams = scenegen.make_scene("C5", seed=2, n=n)
        cams = [dict(c, width=80, height=64, cx=np.float32(40), cy=np.float32(32),
                     fx=np.float32(69.3), fy=np.float32(69.3)) for c in cams[:n_views]]
    else:   # one tetrahedron scene seen through shifted principal points
        scene, cams = scenegen.make_scene("C2", seed=2, n=n)
        cams = [dict(cams[0], width=80, height=64, cx=np.float32(40 + 7 * v), cy=np.float32(32 - 3 * v),
                     fx=np.float32(69.3), fy=np.float32(69.3)) for v in range(n_views)]
    scene["pos"][0][7] = np.nan
    f3 = np.random.default_rng(0).uniform(0.0, 0.05, n).astype(np.float32)
    ds = render.DeviceScene(scene, filter3d=f3)
    multi = render.Renderer(ds, cams, with_canon=True)
    singles = [render.Renderer(ds, [c], with_canon=True) for c in cams]
    st = multi.stream()
    fa = render.frames_array(multi.frames)
    L.lp_preprocess(ds.prims, multi._cams(list(range(n_views))), multi.cfg, fa, st)
    for s_ in singles:
        fs_ = render.frames_array(s_.frames)
        L.lp_preprocess(ds.prims, s_._cams([0]), s_.cfg, fs_, st)
    torch.cuda.synchronize()
    K = K_OF[scene["kind"]]
    assert int((multi.frames[0].buf("tiles_touched", n, torch.int32) > 0).sum()) > 100
    for v in range(n_views):
        fm_, fs1 = multi.frames[v], singles[v].frames[0]
        for field, cnt, dt in (("tiles_touched", n, torch.int32), ("rect", 4 * n, torch.int16),
                               ("depth_key", n, torch.int32), ("record", n * fm_.c.record_words, torch.int32),
                               ("canon", n * (2 + 3 * K), torch.int32)):
            a = fm_.buf(field, cnt, dt).cpu().numpy()
            b = fs1.buf(field, cnt, dt).cpu().numpy()
            if field == "record":   # records of invisible primitives are not written: compare visible rows
                vis = fm_.buf("tiles_touched", n, torch.int32).cpu().numpy() > 0
                a = a.reshape(n, -1)[vis]
                b = b.reshape(n, -1)[vis]
            assert np.array_equal(a, b), (field, v)
