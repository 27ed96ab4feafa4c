"""Thin ctypes binding of liblinprim.so (include/linprim.h) -- argument marshalling only.

Every step of the hot path runs in the CUDA kernels behind the C-ABI; this module only turns
torch tensors / dicts into the C structs and calls the entry points with the same names.
There is NO CPU fallback: importing this module without the built library raises.
"""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
# LP_LIB: an alternative build of the same library (tests only: liblinprim_checked.so, bounds checks)
LIB_PATH = os.environ.get("LP_LIB") or os.path.join(_HERE, "liblinprim.so")
if not os.path.exists(LIB_PATH):
    raise ImportError(f"{LIB_PATH} is not built; run `python -c 'import __graft_entry__ as g; g.build()'` "
                      "(no CPU fallback exists)")
_lib = C.CDLL(LIB_PATH)

LP_OK, LP_ERR_ARG, LP_ERR_CAPACITY, LP_ERR_CUDA, LP_ERR_UNSUPPORTED = range(5)
LP_OCTAHEDRON, LP_TETRAHEDRON = 0, 1
LP_TILE = 16
LP_CNT_ENTRIES, LP_CNT_OVERFLOW, LP_CNT_INVALID, LP_CNT_FRUSTUM, LP_CNT_VISIBLE = 0, 1, 2, 3, 4
LP_CNT_WARP_HITS, LP_CNT_TILE_HITS, LP_CNT_SORTED = 5, 6, 7
LP_CNT_ITERATED, LP_CNT_INTERSECTED, LP_CNT_INBOX, LP_NUM_COUNTERS = 8, 10, 12, 16
LP_SORT_BUCKET, LP_SORT_RADIX = 0, 1
LP_FRAME_CANON, LP_FRAME_DETERMINISTIC = 1, 2
LP_ABI_VERSION = 6            # include/linprim.h; the loaded library must match the structs below

_p = C.c_void_p


class lp_prims(C.Structure):
    _fields_ = [("kind", C.c_int32), ("n", C.c_int32), ("sh_degree", C.c_int32),
                ("pos", _p), ("rot", _p), ("dist", _p), ("opacity", _p), ("sh", _p), ("filter3d", _p)]


class lp_camera(C.Structure):
    _fields_ = [("W", C.c_float * 9), ("t", C.c_float * 3), ("fx", C.c_float), ("fy", C.c_float),
                ("cx", C.c_float), ("cy", C.c_float), ("znear", C.c_float),
                ("width", C.c_int32), ("height", C.c_int32)]


class lp_raster_cfg(C.Structure):
    _fields_ = [("aa_kernel", C.c_float), ("t_stop", C.c_float), ("bg", C.c_float * 3),
                ("count_stats", C.c_int32), ("exact", C.c_int32)]


class lp_frame(C.Structure):
    _fields_ = [("kind", C.c_int32), ("n", C.c_int32), ("width", C.c_int32), ("height", C.c_int32),
                ("tiles_x", C.c_int32), ("tiles_y", C.c_int32), ("capacity", C.c_int64),
                ("record_words", C.c_int32), ("rgrad_words", C.c_int32)] + \
        [(f, _p) for f in ("tiles_touched", "rect", "depth_key", "record", "prim_key", "prim_key_alt",
                           "prim_order", "prim_order_alt", "offsets", "tile_key", "tile_key_alt", "entry_val",
                           "entry_val_alt", "sorted_tile", "sorted_val", "ranges", "sort_hist", "scan_tmp",
                           "counters", "T_final", "n_proc", "rgrad", "canon", "tile_diff", "tile_cursor")] + \
        [("sort_method", C.c_int32), ("hitmask", _p), ("T_last", _p), ("deterministic", C.c_int32),
         ("emit_prim", _p), ("emit_pos", _p), ("prim_emit", _p), ("part", _p), ("T_ckpt", _p)]


class lp_adam_group(C.Structure):
    _fields_ = [("begin", C.c_int64), ("end", C.c_int64), ("lr", C.c_float)]


class lp_grads(C.Structure):
    _fields_ = [(f, _p) for f in ("pos", "rot", "dist", "opacity", "sh", "mean2d_abs", "vis_count")]


_sig = {
    "lp_abi_version": (C.c_int32, []),
    "lp_status_string": (C.c_char_p, [C.c_int]),
    "lp_frame_bytes": (C.c_size_t, [C.c_int32, C.c_int32, C.c_int32, C.c_int32, C.c_int64, C.c_int32]),
    "lp_frame_init": (C.c_int, [C.POINTER(lp_frame), _p, C.c_size_t, C.c_int32, C.c_int32, C.c_int32, C.c_int32,
                                C.c_int64, C.c_int32]),
    "lp_preprocess": (C.c_int, [C.POINTER(lp_prims), C.POINTER(lp_camera), C.c_int32, C.POINTER(lp_raster_cfg),
                                C.POINTER(lp_frame), _p]),
    "lp_bin_sort": (C.c_int, [C.POINTER(lp_camera), C.c_int32, C.POINTER(lp_frame), C.POINTER(C.c_int64), _p]),
    "lp_render_fwd": (C.c_int, [C.POINTER(lp_camera), C.c_int32, C.POINTER(lp_raster_cfg), C.POINTER(lp_frame),
                                _p, _p]),
    "lp_render_fwd_aux": (C.c_int, [C.POINTER(lp_camera), C.c_int32, C.POINTER(lp_raster_cfg),
                                    C.POINTER(lp_frame), _p, _p, _p, _p]),
    "lp_render_bwd": (C.c_int, [C.POINTER(lp_prims), C.POINTER(lp_camera), C.c_int32, C.POINTER(lp_raster_cfg),
                                C.POINTER(lp_frame), _p, C.POINTER(lp_grads), _p]),
    "lp_raster_bwd": (C.c_int, [C.POINTER(lp_camera), C.c_int32, C.POINTER(lp_raster_cfg), C.POINTER(lp_frame),
                                _p, _p]),
    "lp_preprocess_bwd": (C.c_int, [C.POINTER(lp_prims), C.POINTER(lp_camera), C.c_int32,
                                    C.POINTER(lp_raster_cfg), C.POINTER(lp_frame), C.POINTER(lp_grads), _p]),
    "lp_preprocess_bwd_assign": (C.c_int, [C.POINTER(lp_prims), C.POINTER(lp_camera), C.c_int32,
                                    C.POINTER(lp_raster_cfg), C.POINTER(lp_frame), C.POINTER(lp_grads), _p]),
    "lp_frame_counters": (C.c_int, [C.POINTER(lp_frame), C.POINTER(C.c_uint32), _p]),
    "lp_l1_grad": (C.c_int, [_p, _p, _p, _p, C.c_int64, C.c_float, _p]),
    "lp_filter3d": (C.c_int, [_p, C.c_int32, _p, C.c_int32, C.c_float, _p, _p]),
    "lp_image_from_u8": (C.c_int, [_p, _p, C.c_int64, _p]),
    "lp_loss_grad": (C.c_int, [_p, _p, _p, _p, C.c_int32, C.c_int32, C.c_int32, C.c_float, C.c_float, _p, _p]),
    "lp_adam_step": (C.c_int, [_p, _p, _p, _p, C.POINTER(lp_adam_group), C.c_int32, C.c_float, C.c_float,
                               C.c_float, C.c_int32, C.c_int32, _p]),
}
for _name, (_res, _args) in _sig.items():
    _f = getattr(_lib, _name)
    _f.restype = _res
    _f.argtypes = _args

EXPORTS = tuple(_sig)
if _lib.lp_abi_version() != LP_ABI_VERSION:
    raise ImportError(f"{LIB_PATH} has ABI {_lib.lp_abi_version()}, this binding expects {LP_ABI_VERSION}; rebuild")


class LinPrimError(RuntimeError):
    pass


def _check(status, what):
    if status != LP_OK:
        raise LinPrimError(f"{what}: {lp_status_string(status)} ({status})")
    return status


def _ptr(t):
    return None if t is None else C.c_void_p(t.data_ptr())


def _stream(stream):
    return C.c_void_p(stream) if isinstance(stream, int) else C.c_void_p(stream.cuda_stream)


# ------------------------------------------------------------------ raw entry points (same names)

def lp_abi_version() -> int:
    return _lib.lp_abi_version()


def lp_status_string(s) -> str:
    return _lib.lp_status_string(int(s)).decode()


def lp_frame_bytes(kind, n, width, height, capacity, flags=0) -> int:
    return int(_lib.lp_frame_bytes(kind, n, width, height, capacity, flags))


def lp_frame_init(frame, workspace, nbytes, kind, n, width, height, capacity, flags=0):
    return _check(_lib.lp_frame_init(C.byref(frame), _ptr(workspace), nbytes, kind, n, width, height, capacity,
                                     flags), "lp_frame_init")


def lp_preprocess(prims, cams, cfg, frames, stream):
    return _check(_lib.lp_preprocess(C.byref(prims), cams, len(cams), C.byref(cfg), frames, _stream(stream)),
                  "lp_preprocess")


def lp_bin_sort(cams, frames, stream, n_entries=None):
    """n_entries: None (async) or a ctypes c_int64 array of len(cams) (synchronising, capacity checked)."""
    st = _lib.lp_bin_sort(cams, len(cams), frames, n_entries, _stream(stream))
    if st == LP_ERR_CAPACITY:
        return st
    return _check(st, "lp_bin_sort")


def lp_render_fwd(cams, cfg, frames, image, stream):
    return _check(_lib.lp_render_fwd(cams, len(cams), C.byref(cfg), frames, _ptr(image), _stream(stream)),
                  "lp_render_fwd")


def lp_render_fwd_aux(cams, cfg, frames, image, depth, alpha, stream):
    return _check(_lib.lp_render_fwd_aux(cams, len(cams), C.byref(cfg), frames, _ptr(image), _ptr(depth),
                                         _ptr(alpha), _stream(stream)), "lp_render_fwd_aux")


def lp_render_bwd(prims, cams, cfg, frames, dL_dimage, grads, stream):
    return _check(_lib.lp_render_bwd(C.byref(prims), cams, len(cams), C.byref(cfg), frames, _ptr(dL_dimage),
                                     C.byref(grads), _stream(stream)), "lp_render_bwd")


def lp_raster_bwd(cams, cfg, frames, dL_dimage, stream):
    return _check(_lib.lp_raster_bwd(cams, len(cams), C.byref(cfg), frames, _ptr(dL_dimage), _stream(stream)),
                  "lp_raster_bwd")


def lp_preprocess_bwd(prims, cams, cfg, frames, grads, stream):
    return _check(_lib.lp_preprocess_bwd(C.byref(prims), cams, len(cams), C.byref(cfg), frames, C.byref(grads),
                                         _stream(stream)), "lp_preprocess_bwd")


def lp_preprocess_bwd_assign(prims, cams, cfg, frames, grads, stream):
    return _check(_lib.lp_preprocess_bwd_assign(C.byref(prims), cams, len(cams), C.byref(cfg), frames, C.byref(grads),
                                         _stream(stream)), "lp_preprocess_bwd_assign")


def lp_frame_counters(frame, stream) -> np.ndarray:
    out = (C.c_uint32 * LP_NUM_COUNTERS)()
    _check(_lib.lp_frame_counters(C.byref(frame), out, _stream(stream)), "lp_frame_counters")
    return np.frombuffer(out, dtype=np.uint32).copy()


def lp_l1_grad(image, target, dL, loss_sum, scale, stream):
    return _check(_lib.lp_l1_grad(_ptr(image), _ptr(target), _ptr(dL), _ptr(loss_sum), image.numel(),
                                  C.c_float(scale), _stream(stream)), "lp_l1_grad")


def lp_image_from_u8(src_u8, dst, stream):
    """8-bit target channels -> fp32 / 255 on the device (C5 input staging)."""
    assert src_u8.numel() == dst.numel()
    return _check(_lib.lp_image_from_u8(_ptr(src_u8), _ptr(dst), src_u8.numel(), _stream(stream)),
                  "lp_image_from_u8")


def lp_filter3d(pos, n, cams_dev, n_cams, kappa, out, stream):
    """pos: device [3, n] fp32; cams_dev: device uint8 tensor holding n_cams lp_camera structs."""
    return _check(_lib.lp_filter3d(_ptr(pos), int(n), _ptr(cams_dev), int(n_cams), C.c_float(kappa), _ptr(out),
                                   _stream(stream)), "lp_filter3d")


def lp_loss_grad(image, target, dL, loss_sum, lam, scale, stream, workspace=None):
    """image / target / dL: contiguous [..., H, W] fp32 tensors (all leading dims are planes);
    workspace: None or a contiguous fp32 tensor of >= 3 * image.numel() elements (the split path)."""
    H, W = image.shape[-2], image.shape[-1]
    planes = image.numel() // (H * W) if H * W else 0
    if workspace is not None and workspace.numel() < 3 * image.numel():
        raise ValueError("lp_loss_grad workspace needs 3 floats per image element")
    return _check(_lib.lp_loss_grad(_ptr(image), _ptr(target), _ptr(dL), _ptr(loss_sum), planes, H, W,
                                    C.c_float(lam), C.c_float(scale), _ptr(workspace), _stream(stream)),
                  "lp_loss_grad")


def lp_adam_step(param, grad, m, v, groups, beta1, beta2, eps, step, stream, zero_grad=False):
    arr = (lp_adam_group * len(groups))(*[lp_adam_group(int(b), int(e), float(lr)) for b, e, lr in groups])
    return _check(_lib.lp_adam_step(_ptr(param), _ptr(grad), _ptr(m), _ptr(v), arr, len(groups), C.c_float(beta1),
                                    C.c_float(beta2), C.c_float(eps), int(step), 1 if zero_grad else 0,
                                    _stream(stream)), "lp_adam_step")


# ------------------------------------------------------------------ struct builders

def camera(cam) -> lp_camera:
    c = lp_camera()
    c.W[:] = [float(v) for v in np.asarray(cam["W"], np.float32).reshape(9)]
    c.t[:] = [float(v) for v in np.asarray(cam["t"], np.float32).reshape(3)]
    for k in ("fx", "fy", "cx", "cy", "znear"):
        setattr(c, k, float(np.float32(cam[k])))
    c.width, c.height = int(cam["width"]), int(cam["height"])
    return c


def cameras(cams):
    arr = (lp_camera * len(cams))()
    for i, c in enumerate(cams):
        arr[i] = camera(c)
    return arr


def raster_cfg(aa_kernel=0.1, t_stop=1e-3, bg=(0.0, 0.0, 0.0), count_stats=False, exact=False) -> lp_raster_cfg:
    c = lp_raster_cfg()
    c.aa_kernel, c.t_stop = float(aa_kernel), float(t_stop)
    c.bg[:] = [float(b) for b in bg]
    c.count_stats = 1 if count_stats else 0
    c.exact = 1 if exact else 0
    return c


def prims_struct(kind, n, sh_degree, pos, rot, dist, opacity, sh, filter3d=None) -> lp_prims:
    p = lp_prims()
    p.kind, p.n, p.sh_degree = int(kind), int(n), int(sh_degree)
    p.pos, p.rot, p.dist, p.opacity, p.sh = (t.data_ptr() for t in (pos, rot, dist, opacity, sh))
    p.filter3d = None if filter3d is None else filter3d.data_ptr()
    return p


def grads_struct(pos=None, rot=None, dist=None, opacity=None, sh=None, mean2d_abs=None,
                 vis_count=None) -> lp_grads:
    g = lp_grads()
    for f, t in (("pos", pos), ("rot", rot), ("dist", dist), ("opacity", opacity), ("sh", sh),
                 ("mean2d_abs", mean2d_abs), ("vis_count", vis_count)):
        setattr(g, f, None if t is None else t.data_ptr())
    return g
