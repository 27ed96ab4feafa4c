/*
 * include/linprim.h -- C-ABI of liblinprim.so, the B200 (sm_100a) implementation of
 * LinPrim's differentiable tile rasterizer for transparent octahedra and tetrahedra
 * (arXiv 2501.16312).  P:n = PAPER.md line n, S:n = SPEC.md line n.
 *
 * Conventions for every entry point
 *   - extern "C", plain pointers and sizes; no C++ or torch types cross the ABI.
 *   - Device pointers are CUDA device memory owned by the CALLER (PyTorch tensors in the
 *     binding).  The library allocates no persistent memory and keeps no global mutable
 *     state; a frame's scratch lives in a caller-provided workspace (lp_frame_init).
 *   - Every call enqueues asynchronously on the given stream (cudaStream_t passed as void*;
 *     NULL = legacy default stream).  Only lp_bin_sort with a non-NULL n_entries and
 *     lp_frame_counters synchronise that stream.
 *   - Arguments are validated BEFORE anything is enqueued; on LP_ERR_ARG nothing ran.
 *     LP_ERR_CUDA reports a launch error (cudaGetLastError); asynchronous faults surface at
 *     the caller's next synchronisation.
 *   - Per-primitive bad data (non-finite features, |q| = 0, any distance <= 0) is not an
 *     error: such primitives are culled, get zero gradient and are counted (#23).
 *   - Gradients ACCUMULATE (+=) so views and calls sum; the caller zeroes them.
 *   - Images are fp32, channel-major [3][H][W] per view (CHW).
 */
#ifndef LINPRIM_H
#define LINPRIM_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define LP_ABI_VERSION 6
#define LP_TILE 16            /* 16 x 16 pixel tiles */

typedef enum {
  LP_OK = 0,
  LP_ERR_ARG = 1,             /* null / inconsistent argument; nothing enqueued */
  LP_ERR_CAPACITY = 2,        /* tile list longer than the frame's capacity (never truncate silently) */
  LP_ERR_CUDA = 3,            /* CUDA launch / runtime error */
  LP_ERR_UNSUPPORTED = 4      /* valid request this build does not implement */
} lp_status;

typedef enum { LP_OCTAHEDRON = 0, LP_TETRAHEDRON = 1 } lp_kind;

/* Primitive features, device fp32, structure-of-arrays, component-major (N contiguous per
 * component).  P:111-139: octahedron 11 floats (c, q, d_x d_y d_z, opacity), tetrahedron 12
 * (c, q, d_0..d_3, opacity), plus (deg+1)^2 x 3 SH coefficients (48 at degree 3). */
typedef struct {
  int32_t kind;               /* lp_kind */
  int32_t n;                  /* number of primitives, >= 0 */
  int32_t sh_degree;          /* 0..3: storage AND evaluation degree */
  const float *pos;           /* [3][n] world centre c */
  const float *rot;           /* [4][n] quaternion (w,x,y,z), need not be unit (normalised inside) */
  const float *dist;          /* [3][n] octa | [4][n] tetra, raw world distances > 0 (reading 2) */
  const float *opacity;       /* [n] logit; alpha = sigmoid (reading 1) */
  const float *sh;            /* [(deg+1)^2][3][n] SH coefficients, 3DGS basis order */
  const float *filter3d;      /* [n] 3D smoothing filter size s (d -> sqrt(d^2+s^2)) or NULL */
} lp_prims;

/* Pinhole camera, host POD passed by value to the kernels.  x_cam = W x_world + t. */
typedef struct {
  float W[9];                 /* world->camera rotation, row-major */
  float t[3];
  float fx, fy, cx, cy;       /* pixels; pixel (x, y) has its centre at (x + 0.5, y + 0.5) (reading 12) */
  float znear;                /* cull iff p_z <= znear (reading 5) */
  int32_t width, height;      /* > 0 */
} lp_camera;

typedef struct {
  float aa_kernel;            /* 2D anti-aliasing filter kernel kappa in pixels (0.1), 0 disables */
  float t_stop;               /* stop once transmittance T < t_stop (1e-3); values below 2^-100 (0
                                 included) act as 2^-100, where no fp32 image changes any more (DESIGN.md
                                 reading 28) */
  float bg[3];                /* background colour (reading 14) */
  int32_t count_stats;        /* 1: count iterated / intersected pairs into the frame counters */
  int32_t exact;              /* 0: EWA ray space (the method); 1: the "no ray space" variant
                                 (App. D, #27): per-pixel perspective rays against
                                 the camera-space faces, perspective tile bbox, no 2D filter.  Must be the
                                 same for every call on a frame. */
} lp_raster_cfg;

/* Per-view scratch carved from one caller-allocated device workspace by lp_frame_init.
 * All pointers are device pointers into that workspace; callers treat them as read-only
 * results (the layout is the library's). */
typedef struct {
  int32_t kind, n, width, height, tiles_x, tiles_y;
  int64_t capacity;           /* maximum tile-list entries */
  int32_t record_words;       /* record stride in floats (24 octa, 28 tetra) */
  int32_t rgrad_words;        /* rgrad row stride in floats (20 octa: dsigma, drgb, 16 moments; 24 tetra: 18 moments + pad) */
  uint32_t *tiles_touched;    /* [n] */
  uint16_t *rect;             /* [n][4] tile rect tx0, ty0, tx1, ty1 (inclusive), zeros if none */
  uint32_t *depth_key;        /* [n] float bits of l = |p| (0 if culled / invalid) */
  float    *record;           /* [n][record_words] raster records */
  uint32_t *prim_key, *prim_key_alt;     /* [n] depth-sort keys */
  uint32_t *prim_order, *prim_order_alt; /* [n] depth-sorted primitive ids */
  uint32_t *offsets;          /* [n + 1] exclusive scan of tiles_touched in depth order */
  uint32_t *tile_key, *tile_key_alt;     /* [capacity] */
  uint32_t *entry_val, *entry_val_alt;   /* [capacity] */
  uint32_t *sorted_tile;      /* [E] after lp_bin_sort: tile of each entry, ascending (points into the above) */
  uint32_t *sorted_val;       /* [E] after lp_bin_sort: primitive id of each entry */
  uint32_t *ranges;           /* [tiles][2] [start, end) into the sorted list */
  uint32_t *sort_hist;        /* radix-sort histogram scratch */
  uint32_t *scan_tmp;         /* scan scratch */
  uint32_t *counters;         /* [16] device counters, see LP_CNT_* */
  float    *T_final;          /* [H][W] final transmittance */
  uint32_t *n_proc;           /* [H][W] tile-list entries processed per pixel (from the tile's start) */
  float    *rgrad;            /* [n][rgrad_words] raster-gradient scratch of the backward, one row per primitive */
  float    *canon;            /* [n][2 + 3K] canonical fp32 cr_x, cr_y, offsets (debug; NULL unless requested) */
  int32_t  *tile_diff;        /* [(tiles_y+1)][(tiles_x+1)] 2-D difference counts of the tile rects (bucket sort) */
  uint32_t *tile_cursor;      /* [tiles] bucket fill cursors (bucket sort) */
  int32_t   sort_method;      /* LP_SORT_BUCKET or LP_SORT_RADIX; lp_frame_init picks BUCKET for n <= 300000 (launch-
                                 latency-bound frames) and RADIX above it and for deterministic frames; the caller
                                 may change it before lp_preprocess (K1 fills the bucket method's rect grid only
                                 when selected; deterministic frames require RADIX) */
  uint32_t *hitmask;          /* [4][capacity/32 + 2] per warp of a tile, one bit per tile-list entry: the forward
                                 sets it when the entry intersected one of the warp's pixels; the backward
                                 replays only those entries */
  float    *T_last;           /* [H][W] T in front of the entry that stopped the pixel (= T_final if it never
                                 stopped): the backward's first recovered T, never divided by a tiny E */
  int32_t   deterministic;    /* 1 (frame created with LP_FRAME_DETERMINISTIC): the backward's raster moments are
                                 written per (tile-list entry, warp) and summed per primitive in a fixed order
                                 (bitwise reproducible gradients); 0: RED.F32 atomics */
  uint32_t *emit_prim;        /* [capacity] deterministic frames: primitive of every emitted entry (emission order) */
  uint32_t *emit_pos;         /* [capacity] deterministic frames: sorted position of every emitted entry */
  uint32_t *prim_emit;        /* [n] deterministic frames: first emitted entry of every primitive */
  float    *part;             /* [capacity][4 warps][rgrad_words] deterministic frames: per (entry, warp) moment sums */
  float    *T_ckpt;           /* [tiles + capacity/128 + 2][128][2] the pixels' T in front of every 128-entry
                                 batch of their tile list after the first (forward); the backward restarts its
                                 T = T_after / E recovery from these, so no division chain spans two batches */
} lp_frame;

/* lp_bin_sort methods; both produce the identical (tile, depth, id) order. */
enum {
  LP_SORT_BUCKET = 0,         /* 2-D difference histogram of the rects -> per-tile buckets -> per-tile bitonic sort */
  LP_SORT_RADIX = 1           /* depth sort of the primitives -> emission in depth order -> stable radix sort by tile */
};

enum {
  LP_CNT_ENTRIES = 0,         /* E, tile-list length */
  LP_CNT_OVERFLOW = 1,        /* 1 if E > capacity (entries beyond capacity were not written) */
  LP_CNT_INVALID = 2,         /* primitives with invalid features */
  LP_CNT_FRUSTUM = 3,         /* primitives with p_z > znear and valid features */
  LP_CNT_VISIBLE = 4,         /* primitives with tiles_touched > 0 */
  LP_CNT_WARP_HITS = 5,       /* (warp, entry) pairs with a hit: the backward's replayed (warp, primitive) pairs
                                 W_h (count_stats; from lp_render_fwd's hit bits) */
  LP_CNT_TILE_HITS = 6,       /* (tile, entry) pairs hit by any pixel of the tile: A (count_stats) */
  LP_CNT_SORTED = 7,          /* primitives in lp_bin_sort's depth order (the visible ones; radix method, n > 4096) */
  LP_CNT_ITERATED = 8,        /* words 8-9: u64 (pixel, entry) pairs evaluated by the forward (count_stats) */
  LP_CNT_INTERSECTED = 10,    /* words 10-11: u64 pairs with chord > 0 (count_stats) */
  LP_CNT_INBOX = 12,          /* words 12-13: u64 pairs inside the primitive's screen bbox (count_stats) */
  LP_NUM_COUNTERS = 16
};

/* C5 helpers: per-parameter-group learning rates for the fused Adam. */
typedef struct {
  int64_t begin, end;         /* element range [begin, end) of the flat parameter buffer */
  float lr;
} lp_adam_group;

/* Gradient sinks, device fp32, same layout as lp_prims; += semantics.  Any may be NULL. */
typedef struct {
  float *pos, *rot, *dist, *opacity, *sh;
  float *mean2d_abs;          /* [n] += |dL/d c_ray.xy| per view, pixel units (densification statistic,
                                 P:252-260, #26) or NULL */
  float *vis_count;           /* [n] += number of the call's views with tiles_touched > 0 (the statistic's
                                 denominator) or NULL */
} lp_grads;

int32_t     lp_abi_version(void);
const char *lp_status_string(lp_status s);

/* lp_frame_bytes / lp_frame_init flags */
enum {
  LP_FRAME_CANON = 1,         /* keep the canonical fp32 geometry (lp_frame.canon; parity tests) */
  LP_FRAME_DETERMINISTIC = 2  /* deterministic backward (lp_frame.deterministic): + capacity x (8 + 16 rgrad_words) B */
};

/* Bytes of device workspace for one frame (256-byte aligned inside); flags: LP_FRAME_* bits. */
size_t lp_frame_bytes(int32_t kind, int32_t n, int32_t width, int32_t height, int64_t capacity,
                      int32_t flags);

/* Carve a frame out of `workspace` (device, >= lp_frame_bytes, 256-byte aligned). Host-only. */
lp_status lp_frame_init(lp_frame *frame, void *workspace, size_t bytes, int32_t kind, int32_t n,
                        int32_t width, int32_t height, int64_t capacity, int32_t flags);

/* a1-a3: per primitive, for each view v:
 * vertices from features, view transform, EWA ray space, 2D filter, bbox -> tile rect,
 * depth key, raster record (slab / plane form), sigma (Eq. 1) and SH colour.
 * Also resets the frame's counters and its backward scratch (rgrad).  frames[v].n must equal
 * prims->n. */
lp_status lp_preprocess(const lp_prims *prims, const lp_camera *cams, int32_t n_views,
                        const lp_raster_cfg *cfg, lp_frame *frames, void *stream);

/* a4-a7: depth sort of the primitives, exclusive scan of tiles_touched, emission
 * of (tile, id) entries in depth order, stable radix sort by tile, per-tile ranges.
 * n_entries: NULL -> fully asynchronous (overflow is flagged in LP_CNT_OVERFLOW and must be
 * checked by the caller after synchronising); non-NULL [n_views] host array -> the stream is
 * synchronised after the scan, E is written per view and LP_ERR_CAPACITY is returned (with
 * nothing truncated and the sort not run) if any E exceeds its frame's capacity. */
lp_status lp_bin_sort(const lp_camera *cams, int32_t n_views, lp_frame *frames, int64_t *n_entries,
                      void *stream);

/* a8-a9: per-pixel chord through each primitive of the pixel's
 * tile list (slab / Cyrus-Beck form of the ray-face intersection), opacity
 * 1 - exp(-sigma chord), front-to-back compositing with include-then-stop at T < t_stop.
 * image: device [n_views][3][H][W]; T_final / n_proc are kept in the frame for the backward. */
lp_status lp_render_fwd(const lp_camera *cams, int32_t n_views, const lp_raster_cfg *cfg,
                        lp_frame *frames, float *image, void *stream);

/* lp_render_fwd plus the depth and alpha render modes, from the same pass:
 * depth (App. B): per pixel the entry distance i1 (ray-space, i.e. camera distance
 *   |p| of the centre plus the entry offset along the ray) of the FIRST composited primitive
 *   after which the cumulative opacity 1 - T exceeds 0.5; 0 where it never does (#24).
 * alpha: 1 - T_final.
 * depth, alpha: device [n_views][H][W] fp32 or NULL (each independently). */
lp_status lp_render_fwd_aux(const lp_camera *cams, int32_t n_views, const lp_raster_cfg *cfg,
                            lp_frame *frames, float *image, float *depth, float *alpha, void *stream);

/* a10-a12 (App. E): reverse replay of each tile list, blend backward,
 * chord -> entry/exit -> slab/plane moments reduced per (warp, primitive) -> rgrad, then the
 * preprocess backward to world features (+= into grads).  Requires the frames filled by
 * lp_preprocess / lp_bin_sort / lp_render_fwd with the same prims, cams and cfg.
 * dL_dimage: device [n_views][3][H][W]. */
lp_status lp_render_bwd(const lp_prims *prims, const lp_camera *cams, int32_t n_views,
                        const lp_raster_cfg *cfg, lp_frame *frames, const float *dL_dimage,
                        const lp_grads *grads, void *stream);

/* The two halves of lp_render_bwd, exported separately so callers can time / overlap them:
 * lp_raster_bwd  (a10-a11): reverse replay -> += rgrad moments (rgrad is zeroed by lp_preprocess).
 * lp_preprocess_bwd (a12): rgrad moments -> world features (+= into grads). */
lp_status lp_raster_bwd(const lp_camera *cams, int32_t n_views, const lp_raster_cfg *cfg, lp_frame *frames,
                        const float *dL_dimage, void *stream);
lp_status lp_preprocess_bwd(const lp_prims *prims, const lp_camera *cams, int32_t n_views,
                            const lp_raster_cfg *cfg, lp_frame *frames, const lp_grads *grads, void *stream);

/* lp_preprocess_bwd with ASSIGN semantics for the feature gradients: grads.pos/rot/dist/opacity/sh
 * are SET to the sum over these n_views (every primitive written, zero where no view has a raster
 * gradient; the old contents are never read), so a training step that starts with this call needs no
 * gradient zeroing (lp_adam_step with zero_grad = 0).  grads.mean2d_abs / vis_count still accumulate.
 * Same arguments, layout and errors as lp_preprocess_bwd. */
lp_status lp_preprocess_bwd_assign(const lp_prims *prims, const lp_camera *cams, int32_t n_views,
                                   const lp_raster_cfg *cfg, lp_frame *frames, const lp_grads *grads, void *stream);

/* Copy the frame's counters to host (synchronises the stream). */
lp_status lp_frame_counters(const lp_frame *frame, uint32_t *host_counters /* [LP_NUM_COUNTERS] words */,
                            void *stream);

/* C5 (north_star): L1 loss gradient dL/dC = scale * sign(C - target) over n elements
 * (written, not accumulated) and loss_sum[0] += scale * sum |C - target| (device float). */
lp_status lp_l1_grad(const float *image, const float *target, float *dL_dimage, float *loss_sum,
                     int64_t n, float scale, void *stream);

/* f4 (#26): 3D smoothing filter size per primitive from the training
 * cameras, s_3d = kappa * min over the cameras that see the centre (p_z > znear, projection inside
 * [0, W] x [0, H]) of p_z / fx, or kappa |p| / fx of the nearest camera when none sees it.
 * pos: device [3][n] world centres; cams_dev: DEVICE array of n_cams lp_camera (unlike the other
 * entry points, so any number of training cameras fits); filter3d: device [n] fp32, written.
 * Feed the result to lp_prims.filter3d (d -> sqrt(d^2 + s^2)). */
lp_status lp_filter3d(const float *pos, int32_t n, const lp_camera *cams_dev, int32_t n_cams, float kappa,
                      float *filter3d, void *stream);

/* f1 (#25): the 3DGS loss L = (1 - lambda) L1 + lambda (1 - SSIM) of
 * n_planes fp32 image planes [n_planes][height][width] (n_views * 3 channels, CHW per view) and its
 * gradient.  SSIM: 11 x 11 Gaussian window (sigma 1.5) with zero padding, C1 = 0.01^2, C2 = 0.03^2.
 * dL_dimage = scale * [(1 - lambda) sign(x - y) - lambda dSumS/dx] (written, not accumulated);
 * loss_sum[0] += scale * sum_p [(1 - lambda)|x_p - y_p| + lambda (1 - S_p)] (device float).
 * scale = 1 / (3 H W n_views) makes both the mean over views of the per-view losses.
 * lambda = 0 reduces to lp_l1_grad.
 * workspace: NULL, or device fp32 scratch of 3 * n_planes * height * width floats (16-byte aligned,
 * caller-owned, contents undefined on return): with it (and width % 4 == 0) the loss runs as two
 * kernels -- the SSIM maps on each 32 x 32 tile's core into the workspace, then their window sums --
 * instead of one kernel that recomputes the maps on a 42 x 42 halo region per tile; dL_dimage is
 * bitwise the same either way, loss_sum differs only in fp32 summation order. */
lp_status lp_loss_grad(const float *image, const float *target, float *dL_dimage, float *loss_sum,
                       int32_t n_planes, int32_t height, int32_t width, float lambda, float scale,
                       float *workspace, void *stream);

/* C5 input staging (not part of the method): training images arrive as 8-bit channels (the
 * datasets' PNG / JPEG targets); dst[i] = src[i] / 255 (IEEE fp32 division, so bitwise
 * numpy's uint8 -> float32 / 255) for n elements.  src, dst: device pointers; dst written. */
lp_status lp_image_from_u8(const uint8_t *src, float *dst, int64_t n, void *stream);

/* C5: one fused Adam step over a flat fp32 parameter buffer with per-group learning
 * rates; elements outside every group are left unchanged.  step >= 1 (bias correction). */
lp_status lp_adam_step(float *param, float *grad, float *m, float *v,
                       const lp_adam_group *groups, int32_t n_groups, float beta1, float beta2,
                       float eps, int32_t step, int32_t zero_grad /* 1: grad = 0 after use */,
                       void *stream);

#ifdef __cplusplus
}
#endif
#endif /* LINPRIM_H */
