// lp_kernels.h -- internal launch wrappers (host side) of liblinprim; not part of the C-ABI.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include "../../include/linprim.h"
#include "lp_check.cuh"

namespace lp {

// words per warp row of lp_frame.hitmask (one bit per tile-list entry, +2 so a 128-entry batch at
// any bit offset stays inside the row)
__host__ __device__ inline int64_t hit_words(int64_t capacity) { return (capacity + 31) / 32 + 2; }

// K1 / K5 (lp_preprocess.cu)
// exact: the no-ray-space variant (App. D, reading 27)
void launch_preprocess(const lp_prims &P, const lp_camera *cams, float kappa, const lp_frame *frames, int n_views,
                       bool exact, cudaStream_t st);
// fused over the views of one call (chunks of 8): feature / SH gradients written once per chunk
void launch_preprocess_bwd(const lp_prims &P, const lp_camera *cams, float kappa, const lp_frame *frames, int n_views,
                           const lp_grads &G, bool exact, bool assign, cudaStream_t st);

// K2 (lp_sort.cu)
constexpr int SORT_THREADS = 256;
#ifndef LP_SORT_ITEMS
#define LP_SORT_ITEMS 8      // keys per thread of a radix block (measurement knob -DLP_SORT_ITEMS)
#endif
constexpr int SORT_ITEMS = LP_SORT_ITEMS;
constexpr int SORT_TILE = SORT_THREADS * SORT_ITEMS;   // keys per radix block
constexpr int SCAN_TILE = 2048;                        // elements per scan block
size_t radix_hist_words(int64_t max_items);
size_t scan_tmp_words(int64_t max_items);
// stable LSD radix sort of (key, val) u32 pairs over key bits [0, bits); n from n_dev if non-null
// else n_host; returns 1 if the result lives in the *_alt buffers.  kept (non-null): the first pass
// drops every pair whose key is RADIX_DROP_KEY and writes the number kept to *kept; the later
// passes (and the caller) sort / use only those (n_dev is then ignored).
constexpr uint32_t RADIX_DROP_KEY = 0xFFFFFFFFu;
int radix_sort_pairs(uint32_t *keys, uint32_t *keys_alt, uint32_t *vals, uint32_t *vals_alt, int64_t n_max,
                     const uint32_t *n_dev, int bits, uint32_t *hist, cudaStream_t st, uint32_t *kept = nullptr,
                     bool hist0_ready = false);   // hist0_ready: the first pass's histogram is already in hist
// n: the host bound; n_dev (nullable): the device count of depth-sorted primitives (<= n)
void launch_scan_tiles(const lp_frame &F, int n, const uint32_t *n_dev, cudaStream_t st);   // offsets + E -> counters
// hist0: also write the first tile-sort pass's per-block histogram to F.sort_hist (returns hist0)
bool launch_emit(const lp_frame &F, int n, const uint32_t *n_dev, int64_t max_entries, bool hist0, cudaStream_t st);
void launch_ranges(const lp_frame &F, const uint32_t *sorted_tile, int tiles, cudaStream_t st);
// small frames (n <= 4096, capacity <= 8192): one-CTA depth sort + scan and tile sort + ranges
bool small_bin_ok(const lp_frame &F);
void launch_small_depth_scan(const lp_frame &F, cudaStream_t st);
void launch_small_tile_sort(const lp_frame &F, int bits, int tiles, cudaStream_t st);
// deterministic frames: emission positions + sorted values back to primitive ids (after the tile sort)
void launch_det_fixup(const lp_frame &F, uint32_t *sorted_val, cudaStream_t st);
// deterministic frames: per-primitive raster moments summed in a fixed order from the (entry, warp) partials
void launch_det_gather(const lp_frame &F, cudaStream_t st);
// LP_SORT_BUCKET path
void launch_tile_counts(const lp_frame &F, cudaStream_t st);
void launch_bucket(const lp_frame &F, cudaStream_t st);
void launch_tile_sort(const lp_frame &F, cudaStream_t st);

// K3 / K4 (lp_raster.cu)
// depth / alpha: optional [H][W] outputs (depth mode P:840-841, alpha = 1 - T_final), may be null
void launch_raster_fwd(const lp_frame &F, const lp_camera &cam, const lp_raster_cfg &cfg, float *image, float *depth,
                       float *alpha, cudaStream_t st);
void launch_raster_bwd(const lp_frame &F, const lp_camera &cam, const lp_raster_cfg &cfg, const float *dL_dimage,
                       cudaStream_t st);

// C5 helpers (lp_train.cu)
void launch_l1_grad(const float *img, const float *tgt, float *dL, float *loss, int64_t n, float scale,
                    cudaStream_t st);
// f4 (lp_train.cu): 3D smoothing filter size; cams in device memory
void launch_filter3d(const float *pos, int n, const lp_camera *cams, int nc, float kappa, float *out,
                     cudaStream_t st);
// f1 (lp_loss.cu): fused L1 + SSIM loss and gradient over n_planes [H][W] planes
// ws (nullable): [3][n_planes][H][W] fp32 G-map workspace -> the two-kernel split path
void launch_loss_ssim(const float *img, const float *tgt, float *dL, float *loss_sum, int n_planes, int H, int W,
                      float lam, float scale, float *ws, cudaStream_t st);
void launch_image_from_u8(const uint8_t *src, float *dst, int64_t n, cudaStream_t st);
void launch_adam(float *p, float *g, float *m, float *v, const lp_adam_group *groups, int ng, float b1,
                 float b2, float eps, int step, bool zero_grad, cudaStream_t st);

}  // namespace lp
