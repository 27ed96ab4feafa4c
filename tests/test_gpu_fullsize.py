"""Full-size parity on BASELINE.json configs[1..4] (C2 100k tetra 1280x720, C3 1M octa 1600x1060,
C4 3M tetra 1957x1091, C5 view 0 of the 8-view ring) in the launch configuration bench.py times.

The oracle preprocesses and bins ALL primitives (bit-exact per-primitive outputs), orders the lists
of a sample of tiles, and renders + backpropagates the pixels of those tiles; the GPU runs the whole
frame with dL/dC non-zero only on the sampled tiles, so every per-primitive gradient is comparable.
Global properties (E, range partition, key order) are checked on the full GPU list."""
import numpy as np
import pytest

import oracle
from paper_2501_16312_b200 import scenegen
from tests import parity as PT
from tests.helpers import oscene

pytestmark = pytest.mark.gpu

K_OF = {0: 3, 1: 4}


@pytest.fixture(scope="module", autouse=True)
def _cuda():
    import torch
    assert torch.cuda.is_available()
    from paper_2501_16312_b200 import _build
    _build.build()


def _sample_tiles(gx, gy, k, seed):
    rng = np.random.default_rng(seed)
    return np.sort(rng.choice(gx * gy, size=min(k, gx * gy), replace=False))


@pytest.mark.parametrize("cfg,exact,view", [("C2", False, 0), ("C3", False, 0), ("C4", False, 0)] +
                         [("C5", False, v) for v in range(8)] + [("C3", True, 0), ("C2", True, 0)])
def test_fullsize_sampled_parity(cfg, exact, view, parity_log):
    """exact: the no-ray-space variant (f3) at the same full size, no 2D filter; view: which camera of
    the configuration (C5: all eight ring cameras the bench step renders)."""
    import torch
    scene, cams = scenegen.make_scene(cfg, seed=0)
    cam = cams[view]
    W, H = cam["width"], cam["height"]
    n = scene["pos"].shape[1]
    K = K_OF[scene["kind"]]
    gx, gy = (W + 15) // 16, (H + 15) // 16
    tiles = _sample_tiles(gx, gy, 24, seed=len(cfg) + n % 97 + 7 * view)
    mask_t = np.zeros(gx * gy, np.uint8)
    mask_t[tiles] = 1
    # pixels of the sampled tiles
    pix = []
    for t in tiles:
        ty, tx = divmod(int(t), gx)
        ys = np.arange(ty * 16, min(ty * 16 + 16, H))
        xs = np.arange(tx * 16, min(tx * 16 + 16, W))
        pix.append((ys[:, None] * W + xs[None, :]).reshape(-1))
    pix = np.concatenate(pix).astype(np.int32)

    osc = oscene(scene)
    kappa = 0.0 if exact else 0.1
    pre = oracle.preprocess(osc, cam, kappa=kappa, mode=0, exact=exact)
    keys, vals, ranges = oracle.bin_tiles(pre, W, H, tile_mask=mask_t)
    f0 = oracle.render(osc, cam, pre, vals, ranges, pix=pix, exact=exact)
    stop_mask = np.zeros((H, W), bool)
    stop_mask.reshape(-1)[pix] = f0.m_stop.reshape(-1)[pix] < PT.STOP_MARGIN
    G = np.zeros((3, H, W), np.float32)
    Gs = scenegen.upstream_grad(W, H, seed=1)[0]
    sel = np.zeros(H * W, bool)
    sel[pix] = True
    sel &= ~stop_mask.reshape(-1)
    G.reshape(3, -1)[:, sel] = Gs.reshape(3, -1)[:, sel]

    ds, r, img = PT.gpu_run(scene, [cam], G=G, kappa=kappa, exact=exact)
    got = PT.frame_arrays(r, 0, n, K)
    # ---- per-primitive outputs, all primitives, bit-exact
    assert np.array_equal(got["tiles_touched"], pre.tiles_touched)
    assert np.array_equal(got["rect"], pre.rect)
    assert np.array_equal(got["depth_key"], pre.depth_key)
    assert np.array_equal(got["canon"].view(np.uint32), pre.canon.view(np.uint32))
    # ---- global list properties
    E = got["E"]
    assert E == int(pre.tiles_touched.astype(np.int64).sum())
    # radix-binned frames (the default above LP_BUCKET_MAX_N primitives): the depth sort kept exactly
    # the visible primitives (its first pass drops the others)
    if r.frames[0].c.sort_method == 1:   # LP_SORT_RADIX
        assert got["counters"][7] == int((pre.tiles_touched > 0).sum()) < n
    st = got["sorted_tile"].astype(np.int64)
    assert np.all(np.diff(st) >= 0)
    k64 = (st.astype(np.uint64) << np.uint64(32)) | got["depth_key"][got["sorted_val"]].astype(np.uint64)
    same = st[1:] == st[:-1]
    assert np.all(k64[1:][same] >= k64[:-1][same])
    tie = same & (k64[1:] == k64[:-1])
    assert np.all(got["sorted_val"][1:][tie] > got["sorted_val"][:-1][tie])
    rg = got["ranges"].astype(np.int64)
    nz = rg[rg[:, 1] > rg[:, 0]]
    assert nz[0, 0] == 0 and nz[-1, 1] == E and np.all(nz[1:, 0] == nz[:-1, 1])
    # ---- sampled tiles: bit-exact lists
    for t in tiles:
        a, b = rg[t]
        oa, ob = ranges[t]
        assert np.array_equal(got["sorted_val"][a:b], vals[oa:ob]), f"tile {t}"
    # ---- image on the sampled pixels
    im = img[0].cpu().numpy().reshape(3, -1)[:, pix]
    ref = f0.image.reshape(3, -1)[:, pix]
    ok = ~stop_mask.reshape(-1)[pix]
    assert np.abs(im - ref)[:, ok].max() <= PT.IMG_TOL
    assert np.array_equal(got["n_proc"].reshape(-1)[pix][ok], f0.n_proc.reshape(-1)[pix][ok])
    # ---- gradients (dL/dC non-zero only on the sampled pixels)
    fb = oracle.render(osc, cam, pre, vals, ranges, pix=pix, dL_dimage=G, exact=exact, bounds=True)
    g = oracle.preprocess_bwd(osc, cam, pre, fb, exact=exact)
    gb = oracle.feature_bounds(osc, cam, pre, fb, exact=exact)
    touched = np.isfinite(fb.face_margin)
    screen = PT.screen_flags(pre, exact) & touched
    flagged = (fb.face_margin < PT.FACE_MARGIN) | screen
    ok, worst, reports, n_cond, n_clamp = PT.check_gradients(ds.grad_dict(), g, gb, pre, flagged)
    parity_log(f"fullsize {cfg}{' exact' if exact else ''} view {view}", pixels=int(pix.size),
               masked_px=int(stop_mask.sum()), hit_prims=int(touched.sum()), flagged=int(flagged.sum()),
               screen_flagged=int(screen.sum()), clamp=n_clamp, cond_elems=n_cond, worst=worst)
    assert ok, "; ".join(reports)
    # SURVEY §8c-5 expects ~7e-4 of the primitives flagged; bound it so a drift in the geometry
    # cannot hide behind the loose bound
    nf = int((fb.face_margin < PT.FACE_MARGIN).sum())
    assert nf <= max(3, PT.MAX_FLAGGED_FRAC * touched.sum()), f"face-flagged {nf} of {touched.sum()}"
    assert screen.sum() <= max(3, PT.MAX_FLAGGED_FRAC * touched.sum()), f"screen-flagged {screen.sum()} of {touched.sum()}"
    assert stop_mask.sum() <= PT.MAX_MASKED_FRAC * pix.size, f"masked {stop_mask.sum()} of {pix.size}"
    torch.cuda.empty_cache()


@pytest.mark.parametrize("cfg", ["C2", "C3", "C4", "C5"])
def test_forward_warp_masks_drop_no_hit(cfg):
    """The forward's per-record warp masks (footprint strips) only skip records that hit
    no pixel of the warp: the timed forward (masks) and the counting forward (bbox sub-list + per-pixel
    bbox test, count_stats) give bit-identical image, T_final, n_proc and forward-to-backward hit bits
    at full size -- so the backward gets bit-identical inputs from either."""
    import torch
    from paper_2501_16312_b200 import linprim as L
    from paper_2501_16312_b200 import render
    scene, cams = scenegen.make_scene(cfg, seed=0)
    cam = cams[0]
    W, H = cam["width"], cam["height"]
    ds = render.DeviceScene(scene)
    outs = []
    for stats in (False, True):
        r = render.Renderer(ds, [cam], count_stats=stats)
        img = r.forward()
        torch.cuda.synchronize()
        f = r.frames[0]
        E = int(r.counters(0)[L.LP_CNT_ENTRIES])
        words = (f.capacity + 31) // 32
        hm = f.buf("hitmask", 4 * words, torch.int32).reshape(4, words)[:, :(E + 31) // 32]
        outs.append((f.buf("T_final", W * H, torch.float32).cpu().numpy(),
                     f.buf("n_proc", W * H, torch.int32).cpu().numpy(), hm.cpu().numpy(), img.cpu().numpy()))
    for a, b, name in zip(outs[0], outs[1], ("T_final", "n_proc", "hit bits", "image")):
        assert np.array_equal(a, b), f"{cfg}: {name} differs between the masked and the counting forward"
