"""Device-resident scene + frame management around the C-ABI (marshalling and memory only).

PyTorch provides device memory and streams; every computation is a liblinprim kernel.
Features (and their gradients) live in ONE flat fp32 buffer laid out
[pos 3N | rot 4N | dist KN | opacity N | sh (deg+1)^2*3N] so the C5 step can allreduce and Adam
it as a single tensor.
"""
from __future__ import annotations

import ctypes as C

import numpy as np
import torch

from . import linprim as L
from .train import section_sizes


class DeviceScene:
    """Primitive features + gradient sinks in flat device buffers."""

    def __init__(self, scene: dict, device="cuda", filter3d=None, pad_to: int = 0):
        self.kind = int(scene["kind"])
        self.sh_degree = int(scene["sh_degree"])
        self.n = int(scene["pos"].shape[1])
        self.K = 3 if self.kind == L.LP_OCTAHEDRON else 4
        secs = section_sizes(self.kind, self.n, self.sh_degree)
        total = sum(s for _, s in secs)
        self.total = total
        # pad_to: allocate the flat buffers padded (sharded optimizer: world * chunk elements); the
        # padding is zero and never read by the kernels
        alloc = max(total, int(pad_to))
        self.flat_padded = torch.zeros(alloc, dtype=torch.float32, device=device)
        self.grad_padded = torch.zeros(alloc, dtype=torch.float32, device=device)
        self.flat = self.flat_padded[:total]
        self.grad = self.grad_padded[:total]
        self.offsets = {}
        o = 0
        for name, size in secs:
            self.offsets[name] = (o, o + size)
            src = torch.from_numpy(np.ascontiguousarray(scene[name], np.float32).reshape(-1))
            self.flat[o:o + size].copy_(src)
            o += size
        self.filter3d = None if filter3d is None else torch.as_tensor(filter3d, dtype=torch.float32, device=device)
        self.mean2d = None
        self.vis_count = None
        self._rebuild()

    def view(self, name, grad=False):
        b, e = self.offsets[name]
        return (self.grad if grad else self.flat)[b:e]

    def _rebuild(self):
        v = {k: self.view(k) for k in self.offsets}
        self.prims = L.prims_struct(self.kind, self.n, self.sh_degree, v["pos"], v["rot"], v["dist"], v["opacity"],
                                    v["sh"], self.filter3d)
        g = {k: self.view(k, grad=True) for k in self.offsets}
        self.grads = L.grads_struct(g["pos"], g["rot"], g["dist"], g["opacity"], g["sh"], self.mean2d,
                                    self.vis_count)

    def track_mean2d(self):
        """Accumulate the densification statistics (lp_grads.mean2d_abs / vis_count) from now on."""
        self.mean2d = torch.zeros(self.n, dtype=torch.float32, device=self.flat.device)
        self.vis_count = torch.zeros(self.n, dtype=torch.float32, device=self.flat.device)
        self._rebuild()

    def set_filter3d(self, cams, kappa):
        """s_3d from training cameras (lp_filter3d, f4) -> lp_prims.filter3d for the following calls."""
        arr = L.cameras(cams)
        raw = torch.frombuffer(bytearray(bytes(arr)), dtype=torch.uint8).to(self.flat.device)
        out = torch.empty(self.n, dtype=torch.float32, device=self.flat.device)
        b, e = self.offsets["pos"]
        L.lp_filter3d(self.flat[b:e], self.n, raw, len(cams), kappa, out, torch.cuda.current_stream(self.flat.device))
        self.filter3d = out
        self._rebuild()
        return out

    def grad_dict(self):
        return {k: self.view(k, grad=True) for k in self.offsets}


class Frame:
    """One view's scratch: a device workspace carved by lp_frame_init."""

    def __init__(self, kind, n, width, height, capacity, device="cuda", with_canon=False, deterministic=False):
        flags = (L.LP_FRAME_CANON if with_canon else 0) | (L.LP_FRAME_DETERMINISTIC if deterministic else 0)
        self.args = (kind, n, width, height, int(capacity), flags)
        nbytes = L.lp_frame_bytes(*self.args)
        if nbytes == 0:
            raise L.LinPrimError("lp_frame_bytes: invalid frame arguments")
        self.ws = torch.empty(nbytes + 256, dtype=torch.uint8, device=device)
        base = self.ws.data_ptr()
        self.shift = (-base) % 256
        self.c = L.lp_frame()
        L._check(L._lib.lp_frame_init(C.byref(self.c), C.c_void_p(base + self.shift), nbytes, *self.args),
                 "lp_frame_init")

    @property
    def capacity(self):
        return self.c.capacity

    def buf(self, field, count, dtype=torch.int32):
        """Torch view of a frame buffer (device pointer inside the workspace)."""
        ptr = getattr(self.c, field)
        if ptr is None:
            return None
        off = ptr - self.ws.data_ptr()
        item = torch.empty((), dtype=dtype).element_size()
        return self.ws[off:off + count * item].view(dtype)


def frames_array(frames):
    arr = (L.lp_frame * len(frames))()
    for i, f in enumerate(frames):
        arr[i] = f.c
    return arr


def _store_back(frames, arr):
    for i, f in enumerate(frames):
        f.c = arr[i]


def estimate_capacity(n, width, height):
    return max(1 << 16, 8 * n + 4 * width * height)


class Renderer:
    """Forward / backward of the LinPrim tile rasterizer over a list of views (C-ABI calls only)."""

    def __init__(self, scene: DeviceScene, cams, aa_kernel=0.1, t_stop=1e-3, bg=(0.0, 0.0, 0.0), capacity=None,
                 with_canon=False, count_stats=False, sync_capacity=True, sort_method=None, exact=False,
                 deterministic=False):
        self.scene = scene
        self.sort_method = None if sort_method is None else int(sort_method)   # None: lp_frame_init's default
        self.cam_dicts = list(cams)
        self.cams = L.cameras(self.cam_dicts)
        # exact: the "no ray space" variant (App. D, lp_raster_cfg.exact)
        self.cfg = L.raster_cfg(aa_kernel, t_stop, bg, count_stats, exact)
        self.with_canon = with_canon
        # deterministic: bitwise reproducible backward (LP_FRAME_DETERMINISTIC frames)
        self.deterministic = deterministic
        self.sync_capacity = sync_capacity
        dev = scene.flat.device
        self.frames = []
        for c in self.cam_dicts:
            cap = capacity or estimate_capacity(scene.n, c["width"], c["height"])
            self.frames.append(self._new_frame(c, cap))
        self.sizes = [3 * c["width"] * c["height"] for c in self.cam_dicts]

    def _new_frame(self, cam, capacity):
        f = Frame(self.scene.kind, self.scene.n, cam["width"], cam["height"], capacity, self.scene.flat.device,
                  self.with_canon, self.deterministic)
        if self.sort_method is not None:
            f.c.sort_method = self.sort_method
        return f

    def stream(self):
        return torch.cuda.current_stream(self.scene.flat.device)

    def _cams(self, views):
        arr = (L.lp_camera * len(views))()
        for i, v in enumerate(views):
            arr[i] = self.cams[v]
        return arr

    def preprocess_and_sort(self, views=None):
        views = list(range(len(self.frames))) if views is None else list(views)
        st = self.stream()
        for v in views:
            cams = self._cams([v])
            while True:
                fa = frames_array([self.frames[v]])
                L.lp_preprocess(self.scene.prims, cams, self.cfg, fa, st)
                if self.sync_capacity:
                    ne = (C.c_int64 * 1)()
                    status = L.lp_bin_sort(cams, fa, st, ne)
                    _store_back([self.frames[v]], fa)
                    if status == L.LP_ERR_CAPACITY:
                        self.frames[v] = self._new_frame(self.cam_dicts[v], int(ne[0] * 1.25) + 1024)
                        continue
                else:
                    L.lp_bin_sort(cams, fa, st, None)
                    _store_back([self.frames[v]], fa)
                break

    def render_views(self, image, views=None, depth=None, alpha=None):
        """Forward raster of the views into image[i] (and depth[i] / alpha[i] when given, the
        depth / alpha render modes, lp_render_fwd_aux)."""
        views = list(range(len(self.frames))) if views is None else list(views)
        st = self.stream()
        for i, v in enumerate(views):
            fa = frames_array([self.frames[v]])
            if depth is None and alpha is None:
                L.lp_render_fwd(self._cams([v]), self.cfg, fa, image[i], st)
            else:
                L.lp_render_fwd_aux(self._cams([v]), self.cfg, fa, image[i],
                                    None if depth is None else depth[i], None if alpha is None else alpha[i], st)
            _store_back([self.frames[v]], fa)

    def forward(self, views=None, image=None, depth=False, alpha=False):
        """Render the views; returns image [V,3,H,W], or (image, depth [V,H,W] | None, alpha [V,H,W] | None)
        when depth or alpha is requested."""
        views = list(range(len(self.frames))) if views is None else list(views)
        c = self.cam_dicts[views[0]]
        dev = self.scene.flat.device
        if image is None:
            image = torch.empty((len(views), 3, c["height"], c["width"]), dtype=torch.float32, device=dev)
        dmap = torch.empty((len(views), c["height"], c["width"]), dtype=torch.float32, device=dev) if depth else None
        amap = torch.empty((len(views), c["height"], c["width"]), dtype=torch.float32, device=dev) if alpha else None
        self.preprocess_and_sort(views)
        self.render_views(image, views, depth=dmap, alpha=amap)
        if depth or alpha:
            return image, dmap, amap
        return image

    def backward(self, dL_dimage, views=None):
        views = list(range(len(self.frames))) if views is None else list(views)
        st = self.stream()
        dL_dimage = dL_dimage.contiguous()
        # one call for all views: the raster backward runs per view, the preprocess backward is
        # fused over the views (feature / SH gradients read-modified-written once)
        fa = frames_array([self.frames[v] for v in views])
        L.lp_render_bwd(self.scene.prims, self._cams(views), self.cfg, fa, dL_dimage, self.scene.grads, st)

    def counters(self, v=0):
        return L.lp_frame_counters(self.frames[v].c, self.stream())
