"""The C5 training iteration: the launch sequence of one step over this
rank's views -- host-side sequencing of C-ABI calls only (streams, events, the one collective).

Per step:
  lp_preprocess of all local views (one launch for up to 8 views; two with split_pre so the first
  `wave` views bin early)
  per local view, round-robin over `streams` CUDA streams (default: one per view):
      lp_bin_sort -> lp_render_fwd -> lp_loss_grad (3DGS L1 + SSIM) | lp_l1_grad -> lp_raster_bwd
  lp_preprocess_bwd_assign over all local views (the step's gradient is SET: no zeroing pass)
  N > 1: ONE NCCL all_reduce(SUM) of the flat fp32 gradient (north_star; issued as ar_chunks
         in-order asynchronous chunks so the replicated fused Adam of chunk k (lp_adam_step, groups
         clipped to the chunk) overlaps the transfer of chunk k + 1) -- or, with sharded=True,
         reduce_scatter + Adam on this rank's chunk + all_gather of the parameters (same wire bytes,
         1/N of the Adam work)
bench.py times exactly this object; tests/test_gpu_step.py compares one step of it with
oracle/train.py.c5_step.
"""
from __future__ import annotations

import torch

from . import linprim as L
from . import render, train


def device_scene(scene, device, world=1, sharded=False):
    """DeviceScene padded for the sharded optimizer when it is used (world * chunk elements)."""
    total = sum(sz for _, sz in train.section_sizes(scene["kind"], scene["pos"].shape[1], scene["sh_degree"]))
    _, _, chunk = train.shard_range(total, 0, world)
    return render.DeviceScene(scene, device=device, pad_to=world * chunk if sharded and world > 1 else 0)


class TrainStep:
    """One training iteration of LinPrim over the local views `cams` of a global batch of
    `n_views_total` views (views[r::N] on rank r)."""

    def __init__(self, ds: render.DeviceScene, cams, n_views_total, *, targets=None, loss="l1ssim", lam=0.2,
                 streams=8, split_pre=False, assign=True, exact=False, capacity=None, world=1, rank=0,
                 sharded=False, extent=4.0, betas=(0.9, 0.999), eps=1e-15, loss_slots=256, aa_kernel=None,
                 deterministic=False, ar_chunks=4, wave=4):
        dev = ds.flat.device
        self.ds, self.dev = ds, dev
        self.n_local = len(cams)
        self.world, self.rank = world, rank
        self.sharded = bool(sharded) and world > 1
        self.loss_kind, self.lam = loss, lam
        self.assign, self.split_pre = assign, split_pre
        self.betas, self.eps = betas, eps
        W, H = cams[0]["width"], cams[0]["height"]
        self.W, self.H = W, H
        kappa = (0.0 if exact else 0.1) if aa_kernel is None else aa_kernel
        self.rend = render.Renderer(ds, cams, capacity=capacity, exact=exact, aa_kernel=kappa, sync_capacity=False,
                                    deterministic=deterministic)
        self.img = torch.empty((self.n_local, 3, H, W), dtype=torch.float32, device=dev)
        self.dL = torch.empty_like(self.img)
        # the split L1 + SSIM path's G-map workspace, one per view (views on different streams run concurrently)
        self.loss_ws = (torch.empty((self.n_local, 3 * 3 * H * W), dtype=torch.float32, device=dev)
                        if loss != "l1" else None)
        self.targets = targets
        self.loss_buf = torch.zeros(loss_slots, dtype=torch.float32, device=dev)
        self.scale = 1.0 / (3.0 * W * H * n_views_total)       # mean over views of the per-view means
        groups = train.lr_groups(ds.offsets, ds.n, extent=extent)
        self.groups = groups
        if self.sharded:
            lo, hi, chunk = train.shard_range(ds.total, rank, world)
            self.chunk = chunk
            self.sgroups = train.shard_groups(groups, lo, hi)
            self.m = torch.zeros(chunk, dtype=torch.float32, device=dev)
            self.gshard = torch.zeros(chunk, dtype=torch.float32, device=dev)
        else:
            self.m = torch.zeros(ds.flat.numel(), dtype=torch.float32, device=dev)
        self.v = torch.zeros_like(self.m)
        # N > 1, single allreduce: issued as `ar_chunks` in-order chunks, each chunk's Adam (groups
        # clipped to it) waiting only for its own chunk, so the optimizer overlaps the remaining transfer
        self.ar_bounds = (train.chunk_bounds(ds.total, ar_chunks) if world > 1 and not self.sharded and ar_chunks > 1
                          else [])
        self.ar_groups = [train.shard_groups(groups, lo, hi) for lo, hi in self.ar_bounds]
        st = torch.cuda.current_stream(dev)
        self.st = st
        n = self.n_local
        rend = self.rend
        self.fa_all = render.frames_array(rend.frames)
        self.ca_all = rend._cams(list(range(n)))
        self.fa_view = [render.frames_array([rend.frames[i]]) for i in range(n)]
        self.ca_view = [rend._cams([i]) for i in range(n)]
        self.n_str = max(1, min(streams, n))
        self.streams = [st] + [torch.cuda.Stream(dev) for _ in range(self.n_str - 1)]
        self.fork, self.fork2 = torch.cuda.Event(), torch.cuda.Event()
        # recorded on the main stream once the step's preprocess launches are enqueued: a caller's
        # host -> device copies for the NEXT step wait for it (copies under K1's HBM traffic slow it)
        self.pre_done = torch.cuda.Event()
        # recorded after the forward of the middle local view: where a caller's uploads for the NEXT step
        # cost least (measured: right after the preprocess they slow the step's start; see bench.py)
        self.mid_done = torch.cuda.Event()
        self.joins = [torch.cuda.Event() for _ in self.streams[1:]]
        self.aux = [torch.cuda.Stream(dev) for _ in range(self.n_str)] if split_pre else []
        self.joins_aux = [torch.cuda.Event() for _ in self.aux]
        # binning of every local view on its own stream, enqueued before any raster work: the sorts
        # are chains of small latency-bound kernels and overlap the raster kernels of earlier views
        # instead of queueing behind them (C5 step 9.61 -> 9.48 ms)
        # (high priority: the block scheduler hands them SMs as raster CTAs retire, ahead of the queued
        # raster CTAs, so their short kernels do not wait for a whole raster kernel to drain)
        lo, hi = torch.cuda.Stream.priority_range()
        self.sort_streams = [torch.cuda.Stream(dev, priority=hi) for _ in range(n)] if streams > 1 else []
        self.sorted = [torch.cuda.Event() for _ in range(n)]
        self.joins_sort = [torch.cuda.Event() for _ in self.sort_streams]
        # split_pre: the first `wave` views are preprocessed in their own launch, so their binning starts
        # while the second launch runs
        ns = self.wave = min(wave, n)
        self.pre_cams = [rend._cams(list(range(ns))), rend._cams(list(range(ns, n)))]
        self.pre_frames = [render.frames_array([rend.frames[i] for i in range(ns)]),
                           render.frames_array([rend.frames[i] for i in range(ns, n)])]

    # ------------------------------------------------------------------------------------------
    @property
    def frames(self):
        return self.rend.frames

    def counters(self, i):
        return self.rend.counters(i)

    def overflowed(self):
        """True if any local view's tile list overflowed its capacity (async binning; synchronises)."""
        return any(int(self.counters(i)[L.LP_CNT_OVERFLOW]) != 0 for i in range(self.n_local))

    def kernel_launches(self):
        """Launches of liblinprim kernels one step enqueues (bench.py's gpu_launches claim)."""
        import math
        F = self.rend.frames[0].c
        tiles = F.tiles_x * F.tiles_y
        tile_passes = math.ceil(max(1, math.ceil(math.log2(tiles))) / 8)
        # depth sort | scan | emit | tile sort (the emission writes its first histogram) | ranges | fwd | loss | rbwd
        loss = 2 if (self.loss_ws is not None and self.W % 4 == 0) else 1     # the split L1 + SSIM path: 2 kernels
        per_view = 4 * 3 + 3 + 1 + (3 * tile_passes - 1) + 1 + 1 + loss + 1
        n_pre = 2 if (self.split_pre and self.n_local > self.wave) else math.ceil(self.n_local / 8)
        return self.n_local * per_view + n_pre + math.ceil(self.n_local / 4) + 1

    # ------------------------------------------------------------------------------------------
    def run(self, si, t=None, tgt=None, events=None, serial=False, tgt_ready=None):
        """Enqueue one step on the current stream.  si: loss slot; t: Adam step (default si + 1);
        tgt: [n_local,3,H,W] device targets (default self.targets); events: per-view + step events
        (bench attribution); serial: all views on one stream; tgt_ready: per-view events the loss
        waits for (e2e host copies)."""
        L_ = L
        st = self.st
        n_local = self.n_local
        tg = self.targets if tgt is None else tgt
        t = si + 1 if t is None else t
        S = events[n_local] if events is not None else None

        def rec(evl, j, stream):
            if evl is not None:
                evl[j].record(stream)

        rec(S, 0, st)
        for i in range(n_local):
            self.fa_all[i] = self.fa_view[i][0]
        strs = [st] if serial else self.streams
        split = not serial and self.split_pre and n_local > self.wave
        if split:
            nf = self.wave
            L_.lp_preprocess(self.ds.prims, self.pre_cams[0], self.rend.cfg, self.pre_frames[0], st)
            self.fork.record(st)
            L_.lp_preprocess(self.ds.prims, self.pre_cams[1], self.rend.cfg, self.pre_frames[1], st)
            self.fork2.record(st)
            for i in range(n_local):
                self.fa_view[i][0] = self.pre_frames[0][i] if i < nf else self.pre_frames[1][i - nf]
        else:
            L_.lp_preprocess(self.ds.prims, self.ca_all, self.rend.cfg, self.fa_all, st)
            for i in range(n_local):
                self.fa_view[i][0] = self.fa_all[i]
        rec(S, 1, st)
        self.pre_done.record(st)
        if len(strs) > 1 and not split:
            self.fork.record(st)
            for s_ in strs[1:]:
                s_.wait_event(self.fork)
        early = not serial and len(self.sort_streams) == n_local
        if early:
            for i in range(n_local):
                ss = self.sort_streams[i]
                ss.wait_event(self.fork if (not split or i < self.wave) else self.fork2)
                ev = events[i] if events is not None else None
                rec(ev, 0, ss)
                L_.lp_bin_sort(self.ca_view[i], self.fa_view[i], ss, None)
                rec(ev, 1, ss)
                self.sorted[i].record(ss)
        for i in range(n_local):
            sx = strs[i % len(strs)]
            if split:
                sx = self.aux[i % len(self.aux)]
                sx.wait_event(self.fork if i < self.wave else self.fork2)
            ca, fa = self.ca_view[i], self.fa_view[i]
            ev = events[i] if events is not None else None
            if early:
                sx.wait_event(self.sorted[i])
            else:
                rec(ev, 0, sx)
                L_.lp_bin_sort(ca, fa, sx, None)
                rec(ev, 1, sx)
            L_.lp_render_fwd(ca, self.rend.cfg, fa, self.img[i], sx)
            rec(ev, 2, sx)
            if i == (n_local - 1) // 2:
                self.mid_done.record(sx)
            if tgt_ready is not None:
                sx.wait_event(tgt_ready[i])
            if self.loss_kind == "l1":
                L_.lp_l1_grad(self.img[i], tg[i], self.dL[i], self.loss_buf[si:si + 1], self.scale, sx)
            else:
                L_.lp_loss_grad(self.img[i], tg[i], self.dL[i], self.loss_buf[si:si + 1], self.lam, self.scale, sx,
                                workspace=self.loss_ws[i])
            rec(ev, 3, sx)
            L_.lp_raster_bwd(ca, self.rend.cfg, fa, self.dL[i], sx)
            rec(ev, 4, sx)
            self.fa_all[i] = fa[0]
        if early:
            for j, s_ in enumerate(self.sort_streams):
                self.joins_sort[j].record(s_)
                st.wait_event(self.joins_sort[j])
        if split:
            for j, s_ in enumerate(self.aux):
                self.joins_aux[j].record(s_)
                st.wait_event(self.joins_aux[j])
        elif len(strs) > 1:
            for j, s_ in enumerate(strs[1:]):
                self.joins[j].record(s_)
                st.wait_event(self.joins[j])
        ds = self.ds
        (L_.lp_preprocess_bwd_assign if self.assign else L_.lp_preprocess_bwd)(ds.prims, self.ca_all, self.rend.cfg,
                                                                               self.fa_all, ds.grads, st)
        rec(S, 2, st)
        b1, b2 = self.betas
        if self.sharded:
            train.reduce_scatter_gradients(ds.grad_padded, self.gshard, self.world)
            if not self.assign:
                ds.grad_padded.zero_()
            rec(S, 3, st)
            c = self.chunk
            L_.lp_adam_step(ds.flat_padded[self.rank * c:(self.rank + 1) * c], self.gshard, self.m, self.v,
                            self.sgroups, b1, b2, self.eps, t, st, zero_grad=False)
            train.all_gather_params(ds.flat_padded, self.rank, c)
        elif self.ar_bounds and not serial:
            works = train.allreduce_gradients_chunked(ds.grad, self.world, self.ar_bounds)
            rec(S, 3, st)
            for (lo, hi), grp, work in zip(self.ar_bounds, self.ar_groups, works):
                work.wait()   # the current stream waits for this chunk's collective only
                L_.lp_adam_step(ds.flat[lo:hi], ds.grad[lo:hi], self.m[lo:hi], self.v[lo:hi], grp, b1, b2,
                                self.eps, t, st, zero_grad=not self.assign)
        else:
            train.allreduce_gradients(ds.grad, self.world)
            rec(S, 3, st)
            L_.lp_adam_step(ds.flat, ds.grad, self.m, self.v, self.groups, b1, b2, self.eps, t, st,
                            zero_grad=not self.assign)
        rec(S, 4, st)
