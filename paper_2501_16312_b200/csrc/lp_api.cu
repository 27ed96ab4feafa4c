// lp_api.cu -- the C-ABI of liblinprim.so (include/linprim.h): argument validation, frame
// workspace layout, and the per-view launch sequences of the four hot-path calls.
#include <cuda_runtime.h>
#include <stdint.h>
#include <string.h>

#include "../../include/linprim.h"
#include "lp_device.cuh"
#include "lp_kernels.h"

namespace {

using namespace lp;

constexpr size_t ALIGN = 256;
constexpr int32_t LP_BUCKET_MAX_N = 300000;   // default sort method switch (lp_frame_init)
inline size_t up(size_t x) { return (x + ALIGN - 1) / ALIGN * ALIGN; }

// record stride (words): room for both the ray-space and the exact-mode record
inline int record_words(int kind) { return kind == LP_OCTAHEDRON ? Kind<LP_OCTAHEDRON>::RS : Kind<LP_TETRAHEDRON>::RS; }
inline int rgrad_words(int kind) {   // row stride of the [n][rgrad_words] scratch
  return kind == LP_OCTAHEDRON ? lp_rgs<LP_OCTAHEDRON>() : lp_rgs<LP_TETRAHEDRON>();
}
inline int offsets_k(int kind) { return kind == LP_OCTAHEDRON ? 3 : 4; }

struct Layout {
  size_t tiles_touched, rect, depth_key, record, prim_key, prim_key_alt, prim_order, prim_order_alt, offsets, tile_key,
      tile_key_alt, entry_val, entry_val_alt, ranges, sort_hist, scan_tmp, counters, T_final, n_proc, rgrad, canon,
      tile_diff, tile_cursor, hitmask, T_last, T_ckpt, emit_prim, emit_pos, prim_emit, part, total;
};

Layout layout(int kind, int64_t n, int w, int h, int64_t cap, int flags) {
  const bool canon = (flags & LP_FRAME_CANON) != 0, det = (flags & LP_FRAME_DETERMINISTIC) != 0;
  Layout L;
  const int64_t tiles = (int64_t)((w + LP_TILE - 1) / LP_TILE) * ((h + LP_TILE - 1) / LP_TILE);
  const int64_t hw = (int64_t)w * h;
  const int64_t nn = n > 0 ? n : 1, cc = cap > 0 ? cap : 1;
  size_t o = 0;
  auto take = [&](size_t bytes) { const size_t at = o; o += up(bytes); return at; };
  L.tiles_touched = take(4 * nn);
  L.rect = take(8 * nn);
  L.depth_key = take(4 * nn);
  L.record = take(4 * (size_t)record_words(kind) * nn);
  L.prim_key = take(4 * nn);
  L.prim_key_alt = take(4 * nn);
  L.prim_order = take(4 * nn);
  L.prim_order_alt = take(4 * nn);
  L.offsets = take(4 * (nn + 1));
  L.tile_key = take(4 * cc);
  L.tile_key_alt = take(4 * cc);
  L.entry_val = take(4 * cc);
  L.entry_val_alt = take(4 * cc);
  L.ranges = take(8 * tiles);
  L.sort_hist = take(4 * radix_hist_words(nn > cc ? nn : cc));
  L.scan_tmp = take(4 * scan_tmp_words(nn));
  L.counters = take(4 * LP_NUM_COUNTERS);
  L.T_final = take(4 * hw);
  L.n_proc = take(4 * hw);
  L.rgrad = take(4 * (size_t)rgrad_words(kind) * nn);
  L.canon = canon ? take(4 * (size_t)(2 + 3 * offsets_k(kind)) * nn) : 0;
  const int64_t gx = (w + LP_TILE - 1) / LP_TILE, gy = (h + LP_TILE - 1) / LP_TILE;
  L.tile_diff = take(4 * (gx + 1) * (gy + 1));
  L.tile_cursor = take(4 * tiles);
  L.hitmask = take(4 * 4 * hit_words(cc));
  L.T_last = take(4 * hw);
  L.T_ckpt = take(8 * 128 * (size_t)ckpt_slots(tiles, cc));
  L.emit_prim = det ? take(4 * cc) : 0;
  L.emit_pos = det ? take(4 * cc) : 0;
  L.prim_emit = det ? take(4 * nn) : 0;
  L.part = det ? take(4 * 4 * (size_t)rgrad_words(kind) * cc) : 0;
  L.total = o;
  return L;
}

bool valid_kind(int k) { return k == LP_OCTAHEDRON || k == LP_TETRAHEDRON; }

bool valid_cam(const lp_camera &c) {
  return c.width > 0 && c.height > 0 && c.width <= 65535 * LP_TILE && c.height <= 65535 * LP_TILE &&
         c.fx > 0.f && c.fy > 0.f;
}

bool frame_matches(const lp_frame &F, const lp_camera &c) {
  return F.counters && F.width == c.width && F.height == c.height;
}

lp_status check_prims(const lp_prims *P) {
  if (!P || !valid_kind(P->kind) || P->n < 0 || P->sh_degree < 0 || P->sh_degree > 3) return LP_ERR_ARG;
  if (P->n > 0 && (!P->pos || !P->rot || !P->dist || !P->opacity || !P->sh)) return LP_ERR_ARG;
  return LP_OK;
}

lp_status last_error() { return cudaGetLastError() == cudaSuccess ? LP_OK : LP_ERR_CUDA; }

int bits_for(int64_t v) {   // bits needed to represent values in [0, v)
  int b = 1;
  while ((int64_t(1) << b) < v) ++b;
  return b;
}

}  // namespace

extern "C" {

int32_t lp_abi_version(void) { return LP_ABI_VERSION; }

const char *lp_status_string(lp_status s) {
  switch (s) {
    case LP_OK: return "ok";
    case LP_ERR_ARG: return "invalid argument";
    case LP_ERR_CAPACITY: return "tile list exceeds frame capacity";
    case LP_ERR_CUDA: return "CUDA error";
    case LP_ERR_UNSUPPORTED: return "unsupported";
  }
  return "unknown status";
}

size_t lp_frame_bytes(int32_t kind, int32_t n, int32_t width, int32_t height, int64_t capacity, int32_t flags) {
  if (!valid_kind(kind) || n < 0 || width <= 0 || height <= 0 || capacity < 0 || (flags & ~3)) return 0;
  return layout(kind, n, width, height, capacity, flags).total;
}

lp_status lp_frame_init(lp_frame *F, void *workspace, size_t bytes, int32_t kind, int32_t n, int32_t width,
                        int32_t height, int64_t capacity, int32_t flags) {
  if (!F || !workspace || !valid_kind(kind) || n < 0 || width <= 0 || height <= 0 || capacity < 0 || (flags & ~3))
    return LP_ERR_ARG;
  const bool with_canon = (flags & LP_FRAME_CANON) != 0, det = (flags & LP_FRAME_DETERMINISTIC) != 0;
  if ((reinterpret_cast<uintptr_t>(workspace) & (ALIGN - 1)) != 0) return LP_ERR_ARG;
  if (capacity > (int64_t)0xFFFFFFF0u) return LP_ERR_ARG;   // entries are indexed with u32
  const Layout L = layout(kind, n, width, height, capacity, flags);
  if (bytes < L.total) return LP_ERR_ARG;
  char *b = static_cast<char *>(workspace);
  memset(F, 0, sizeof(*F));
  F->kind = kind;
  F->n = n;
  F->width = width;
  F->height = height;
  F->tiles_x = (width + LP_TILE - 1) / LP_TILE;
  F->tiles_y = (height + LP_TILE - 1) / LP_TILE;
  F->capacity = capacity;
  F->record_words = record_words(kind);
  F->rgrad_words = rgrad_words(kind);
  F->tiles_touched = reinterpret_cast<uint32_t *>(b + L.tiles_touched);
  F->rect = reinterpret_cast<uint16_t *>(b + L.rect);
  F->depth_key = reinterpret_cast<uint32_t *>(b + L.depth_key);
  F->record = reinterpret_cast<float *>(b + L.record);
  F->prim_key = reinterpret_cast<uint32_t *>(b + L.prim_key);
  F->prim_key_alt = reinterpret_cast<uint32_t *>(b + L.prim_key_alt);
  F->prim_order = reinterpret_cast<uint32_t *>(b + L.prim_order);
  F->prim_order_alt = reinterpret_cast<uint32_t *>(b + L.prim_order_alt);
  F->offsets = reinterpret_cast<uint32_t *>(b + L.offsets);
  F->tile_key = reinterpret_cast<uint32_t *>(b + L.tile_key);
  F->tile_key_alt = reinterpret_cast<uint32_t *>(b + L.tile_key_alt);
  F->entry_val = reinterpret_cast<uint32_t *>(b + L.entry_val);
  F->entry_val_alt = reinterpret_cast<uint32_t *>(b + L.entry_val_alt);
  F->sorted_tile = nullptr;
  F->sorted_val = nullptr;
  F->ranges = reinterpret_cast<uint32_t *>(b + L.ranges);
  F->sort_hist = reinterpret_cast<uint32_t *>(b + L.sort_hist);
  F->scan_tmp = reinterpret_cast<uint32_t *>(b + L.scan_tmp);
  F->counters = reinterpret_cast<uint32_t *>(b + L.counters);
  F->T_final = reinterpret_cast<float *>(b + L.T_final);
  F->n_proc = reinterpret_cast<uint32_t *>(b + L.n_proc);
  F->rgrad = reinterpret_cast<float *>(b + L.rgrad);
  F->canon = with_canon ? reinterpret_cast<float *>(b + L.canon) : nullptr;
  F->tile_diff = reinterpret_cast<int32_t *>(b + L.tile_diff);
  F->tile_cursor = reinterpret_cast<uint32_t *>(b + L.tile_cursor);
  // default binning method by size (measured): the per-tile bucket sort needs ~4 launches
  // and wins while launch latency dominates (C1: 0.079 -> 0.028 ms, C2: 0.127 -> 0.056 ms); the
  // depth-first radix path wins at 1M primitives (K1's rect-grid atomics grow with the rect sizes);
  // deterministic frames need the radix path's emission order
  F->sort_method = (!det && n <= LP_BUCKET_MAX_N) ? LP_SORT_BUCKET : LP_SORT_RADIX;
  F->hitmask = reinterpret_cast<uint32_t *>(b + L.hitmask);
  F->T_last = reinterpret_cast<float *>(b + L.T_last);
  F->T_ckpt = reinterpret_cast<float *>(b + L.T_ckpt);
  F->deterministic = det ? 1 : 0;
  F->emit_prim = det ? reinterpret_cast<uint32_t *>(b + L.emit_prim) : nullptr;
  F->emit_pos = det ? reinterpret_cast<uint32_t *>(b + L.emit_pos) : nullptr;
  F->prim_emit = det ? reinterpret_cast<uint32_t *>(b + L.prim_emit) : nullptr;
  F->part = det ? reinterpret_cast<float *>(b + L.part) : nullptr;
  return LP_OK;
}

lp_status lp_preprocess(const lp_prims *prims, const lp_camera *cams, int32_t n_views, const lp_raster_cfg *cfg,
                        lp_frame *frames, void *stream) {
  if (check_prims(prims) != LP_OK || !cams || !cfg || !frames || n_views < 0) return LP_ERR_ARG;
  if (!(cfg->aa_kernel >= 0.f) || (cfg->exact != 0 && cfg->exact != 1)) return LP_ERR_ARG;
  for (int v = 0; v < n_views; ++v) {
    if (!valid_cam(cams[v]) || !frame_matches(frames[v], cams[v])) return LP_ERR_ARG;
    if (frames[v].kind != prims->kind || frames[v].n != prims->n) return LP_ERR_ARG;
  }
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  for (int v = 0; v < n_views; ++v) {
    lp_frame &F = frames[v];
    F.sorted_tile = F.sorted_val = nullptr;
    cudaMemsetAsync(F.counters, 0, 4 * LP_NUM_COUNTERS, st);
    // (the backward's raster-moment scratch rows are zeroed by k_preprocess itself)
    if (F.sort_method == LP_SORT_BUCKET)
      cudaMemsetAsync(F.tile_diff, 0, 4 * (size_t)(F.tiles_x + 1) * (F.tiles_y + 1), st);
  }
  // one launch per 8 views: each primitive's features are read once for all of them
  launch_preprocess(*prims, cams, cfg->aa_kernel, frames, n_views, cfg->exact != 0, st);
  return last_error();
}

lp_status lp_bin_sort(const lp_camera *cams, int32_t n_views, lp_frame *frames, int64_t *n_entries, void *stream) {
  if (!cams || !frames || n_views < 0) return LP_ERR_ARG;
  for (int v = 0; v < n_views; ++v)
    if (!valid_cam(cams[v]) || !frame_matches(frames[v], cams[v])) return LP_ERR_ARG;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  lp_status status = LP_OK;
  for (int v = 0; v < n_views; ++v) {
    lp_frame &F = frames[v];
    const int n = F.n;
    if (F.sort_method == LP_SORT_BUCKET && F.deterministic) return LP_ERR_UNSUPPORTED;   // emission order needs radix
    if (F.sort_method == LP_SORT_BUCKET) {
      // counts (2-D prefix of the rect difference grid K1 filled) -> ranges, cursors, E
      launch_tile_counts(F, st);
      if (n_entries) {
        uint32_t e32 = 0;
        cudaMemcpyAsync(&e32, F.counters + LP_CNT_ENTRIES, 4, cudaMemcpyDeviceToHost, st);
        if (cudaStreamSynchronize(st) != cudaSuccess) return LP_ERR_CUDA;
        n_entries[v] = e32;
        if ((int64_t)e32 > F.capacity) {
          status = LP_ERR_CAPACITY;
          continue;
        }
      }
      launch_bucket(F, st);
      launch_tile_sort(F, st);
      F.sorted_tile = F.tile_key;
      F.sorted_val = F.entry_val;
      continue;
    }
    // LP_SORT_RADIX
    // small frames: steps 1-2 and 4-5 each in one CTA (3 launches instead of ~23)
    const bool small = small_bin_ok(F);
    lp_frame Fv = F;
    if (small) {
      launch_small_depth_scan(F, st);
    } else {
      // 1. depth sort of the primitives (stable: ties keep ascending id, reading 11); the first pass
      //    drops the invisible ones (key 0xFFFFFFFF, K1), the other three sort the visible ones only
      const int flip = radix_sort_pairs(F.prim_key, F.prim_key_alt, F.prim_order, F.prim_order_alt, n, nullptr, 32,
                                        F.sort_hist, st, F.counters + LP_CNT_SORTED);
      if (flip) {
        Fv.prim_key = F.prim_key_alt;
        Fv.prim_order = F.prim_order_alt;
      }
      // 2. exclusive scan of tiles_touched in depth order -> offsets, E
      launch_scan_tiles(Fv, n, F.counters + LP_CNT_SORTED, st);
    }
    int64_t E_host = -1;
    if (n_entries) {
      uint32_t e32 = 0;
      cudaMemcpyAsync(&e32, F.counters + LP_CNT_ENTRIES, 4, cudaMemcpyDeviceToHost, st);
      if (cudaStreamSynchronize(st) != cudaSuccess) return LP_ERR_CUDA;
      E_host = e32;
      n_entries[v] = E_host;
      if (E_host > F.capacity) {
        status = LP_ERR_CAPACITY;
        continue;
      }
    }
    // 3. emission in depth order
    const int64_t nmax = E_host >= 0 ? E_host : F.capacity;
    const bool hist0 = launch_emit(Fv, n, small ? nullptr : F.counters + LP_CNT_SORTED, nmax, !small, st);
    // 4. stable sort by tile id
    const int tiles = F.tiles_x * F.tiles_y;
    if (small) {   // + 5. ranges, in the same CTA
      launch_small_tile_sort(F, bits_for(tiles), tiles, st);
      F.sorted_tile = F.tile_key;
      F.sorted_val = F.entry_val;
      if (F.deterministic) launch_det_fixup(F, F.sorted_val, st);
      continue;
    }
    const uint32_t *ndev = E_host >= 0 ? nullptr : F.counters + LP_CNT_ENTRIES;
    const int tflip = radix_sort_pairs(F.tile_key, F.tile_key_alt, F.entry_val, F.entry_val_alt, nmax, ndev,
                                       bits_for(tiles), F.sort_hist, st, nullptr, hist0);
    F.sorted_tile = tflip ? F.tile_key_alt : F.tile_key;
    F.sorted_val = tflip ? F.entry_val_alt : F.entry_val;
    if (F.deterministic) launch_det_fixup(F, F.sorted_val, st);
    // 5. ranges
    lp_frame Fr = F;
    if (E_host >= 0) Fr.capacity = E_host;
    launch_ranges(Fr, F.sorted_tile, tiles, st);
  }
  const lp_status e = last_error();
  return status != LP_OK ? status : e;
}

lp_status lp_render_fwd_aux(const lp_camera *cams, int32_t n_views, const lp_raster_cfg *cfg, lp_frame *frames,
                            float *image, float *depth, float *alpha, void *stream) {
  if (!cams || !cfg || !frames || !image || n_views < 0) return LP_ERR_ARG;
  for (int v = 0; v < n_views; ++v)
    if (!valid_cam(cams[v]) || !frame_matches(frames[v], cams[v]) || !frames[v].sorted_val) return LP_ERR_ARG;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  size_t off = 0;
  for (int v = 0; v < n_views; ++v) {
    const size_t hw = (size_t)cams[v].width * cams[v].height;
    launch_raster_fwd(frames[v], cams[v], *cfg, image + 3 * off, depth ? depth + off : nullptr, alpha ? alpha + off : nullptr,
                      st);
    off += hw;
  }
  return last_error();
}

lp_status lp_render_fwd(const lp_camera *cams, int32_t n_views, const lp_raster_cfg *cfg, lp_frame *frames,
                        float *image, void *stream) {
  return lp_render_fwd_aux(cams, n_views, cfg, frames, image, nullptr, nullptr, stream);
}

lp_status lp_render_bwd(const lp_prims *prims, const lp_camera *cams, int32_t n_views, const lp_raster_cfg *cfg,
                        lp_frame *frames, const float *dL_dimage, const lp_grads *grads, void *stream) {
  if (check_prims(prims) != LP_OK || !cams || !cfg || !frames || !dL_dimage || !grads || n_views < 0) return LP_ERR_ARG;
  for (int v = 0; v < n_views; ++v) {
    if (!valid_cam(cams[v]) || !frame_matches(frames[v], cams[v]) || !frames[v].sorted_val) return LP_ERR_ARG;
    if (frames[v].kind != prims->kind || frames[v].n != prims->n) return LP_ERR_ARG;
  }
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  size_t off = 0;
  for (int v = 0; v < n_views; ++v) {
    launch_raster_bwd(frames[v], cams[v], *cfg, dL_dimage + off, st);
    off += (size_t)3 * cams[v].width * cams[v].height;
  }
  launch_preprocess_bwd(*prims, cams, cfg->aa_kernel, frames, n_views, *grads, cfg->exact != 0, false, st);
  return last_error();
}

lp_status lp_raster_bwd(const lp_camera *cams, int32_t n_views, const lp_raster_cfg *cfg, lp_frame *frames,
                        const float *dL_dimage, void *stream) {
  if (!cams || !cfg || !frames || !dL_dimage || n_views < 0) return LP_ERR_ARG;
  for (int v = 0; v < n_views; ++v)
    if (!valid_cam(cams[v]) || !frame_matches(frames[v], cams[v]) || !frames[v].sorted_val) return LP_ERR_ARG;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  size_t off = 0;
  for (int v = 0; v < n_views; ++v) {
    const lp_frame &F = frames[v];
    launch_raster_bwd(F, cams[v], *cfg, dL_dimage + off, st);
    off += (size_t)3 * cams[v].width * cams[v].height;
  }
  return last_error();
}

static lp_status preprocess_bwd(const lp_prims *prims, const lp_camera *cams, int32_t n_views, const lp_raster_cfg *cfg,
                                lp_frame *frames, const lp_grads *grads, bool assign, void *stream) {
  if (check_prims(prims) != LP_OK || !cams || !cfg || !frames || !grads || n_views < 0) return LP_ERR_ARG;
  for (int v = 0; v < n_views; ++v) {
    if (!valid_cam(cams[v]) || !frame_matches(frames[v], cams[v]) || !frames[v].sorted_val) return LP_ERR_ARG;
    if (frames[v].kind != prims->kind || frames[v].n != prims->n) return LP_ERR_ARG;
  }
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  launch_preprocess_bwd(*prims, cams, cfg->aa_kernel, frames, n_views, *grads, cfg->exact != 0, assign, st);
  return last_error();
}

lp_status lp_preprocess_bwd(const lp_prims *prims, const lp_camera *cams, int32_t n_views, const lp_raster_cfg *cfg,
                            lp_frame *frames, const lp_grads *grads, void *stream) {
  return preprocess_bwd(prims, cams, n_views, cfg, frames, grads, false, stream);
}

lp_status lp_preprocess_bwd_assign(const lp_prims *prims, const lp_camera *cams, int32_t n_views,
                                   const lp_raster_cfg *cfg, lp_frame *frames, const lp_grads *grads, void *stream) {
  return preprocess_bwd(prims, cams, n_views, cfg, frames, grads, true, stream);
}

lp_status lp_frame_counters(const lp_frame *F, uint32_t *host, void *stream) {
  if (!F || !F->counters || !host) return LP_ERR_ARG;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  if (cudaMemcpyAsync(host, F->counters, 4 * LP_NUM_COUNTERS, cudaMemcpyDeviceToHost, st) != cudaSuccess)
    return LP_ERR_CUDA;
  return cudaStreamSynchronize(st) == cudaSuccess ? LP_OK : LP_ERR_CUDA;
}

lp_status lp_l1_grad(const float *image, const float *target, float *dL_dimage, float *loss_sum, int64_t n,
                     float scale, void *stream) {
  if (!image || !target || !dL_dimage || !loss_sum || n < 0) return LP_ERR_ARG;
  launch_l1_grad(image, target, dL_dimage, loss_sum, n, scale, static_cast<cudaStream_t>(stream));
  return last_error();
}

lp_status lp_image_from_u8(const uint8_t *src, float *dst, int64_t n, void *stream) {
  if (n < 0 || (n > 0 && (!src || !dst))) return LP_ERR_ARG;
  launch_image_from_u8(src, dst, n, static_cast<cudaStream_t>(stream));
  return last_error();
}

lp_status lp_filter3d(const float *pos, int32_t n, const lp_camera *cams_dev, int32_t n_cams, float kappa,
                      float *filter3d, void *stream) {
  if (n < 0 || n_cams < 1 || !cams_dev || !filter3d || (n > 0 && !pos) || !(kappa >= 0.f)) return LP_ERR_ARG;
  launch_filter3d(pos, n, cams_dev, n_cams, kappa, filter3d, static_cast<cudaStream_t>(stream));
  return last_error();
}

lp_status lp_loss_grad(const float *image, const float *target, float *dL_dimage, float *loss_sum, int32_t n_planes,
                       int32_t height, int32_t width, float lambda, float scale, float *workspace, void *stream) {
  if (!image || !target || !dL_dimage || !loss_sum || n_planes < 0 || height < 0 || width < 0 || n_planes > 65535 ||
      !(lambda >= 0.f && lambda <= 1.f))
    return LP_ERR_ARG;
  launch_loss_ssim(image, target, dL_dimage, loss_sum, n_planes, height, width, lambda, scale, workspace,
                   static_cast<cudaStream_t>(stream));
  return last_error();
}

lp_status lp_adam_step(float *param, float *grad, float *m, float *v, const lp_adam_group *groups,
                       int32_t n_groups, float beta1, float beta2, float eps, int32_t step, int32_t zero_grad,
                       void *stream) {
  if (!param || !grad || !m || !v || (n_groups > 0 && !groups) || n_groups < 0 || step < 1) return LP_ERR_ARG;
  for (int g = 0; g < n_groups; ++g)
    if (groups[g].begin < 0 || groups[g].end < groups[g].begin) return LP_ERR_ARG;
  launch_adam(param, grad, m, v, groups, n_groups, beta1, beta2, eps, step, zero_grad != 0,
              static_cast<cudaStream_t>(stream));
  return last_error();
}

}  // extern "C"
