// lp_raster.cu -- K3 forward raster (rows a8-a9) and K4 backward raster (rows a10-a11).
//
// One CTA per 16x16 tile.  A CTA walks its tile's sorted list in batches of NT records: each
// thread stages one record (80 B octa / 112 B tetra, gathered by primitive id) into shared
// memory and marks which of the four 8x8 warp rectangles its footprint reaches; each warp then
// evaluates its sub-list of the batch for its pixels (2 per thread), reading each record with
// broadcast LDS.128.  The per-pair work is the slab / Cyrus-Beck chord:
// ~26 FP32 instructions per (pixel, octahedron), ~19 per (pixel, tetrahedron), plus ~10 per
// intersected pair for the opacity and compositing.
//
// Backward: the same lists in reverse.  Per (pixel, entry) with chord > 0 it recovers T_k = T/E,
// runs the blend backward and the chord backward (App. E, in slab/plane
// moment form) into its lane's compacted shared-memory row (<= 22 moments; one 16-byte
// read-modify-write per entry / exit plane), then a column sum over the hit lanes and one
// RED.F32 per moment per (warp, primitive) into the primitive's rgrad row rgrad[n][lp_rgs].
#include <cuda_runtime.h>
#include <stdint.h>

#include "lp_device.cuh"
#include "lp_kernels.h"

namespace lp {

// pixel (x, y) of thread `tid`, slot k, inside the 16x16 tile (warps cover compact squares)
template <int NT>
__device__ __forceinline__ void pixel_of(int tid, int k, int &x, int &y) {
  const int w = tid >> 5, lane = tid & 31;
  if (NT == 128) {          // PPT 2: warp = 8x8 square, lane = 8x4, second pixel 4 rows down
    x = (w & 1) * 8 + (lane & 7);
    y = (w >> 1) * 8 + (lane >> 3) + 4 * k;
  } else if (NT == 64) {    // PPT 4: warp = 16x8, lane = 16x2, pixels 2 rows apart
    x = lane & 15;
    y = w * 8 + (lane >> 4) + 2 * k;
  } else {                  // PPT 1 (NT 256): warp = 8x4
    x = (w & 1) * 8 + (lane & 7);
    y = (w >> 1) * 4 + (lane >> 3);
  }
}

// the warp's pixel-centre rectangle (absolute pixel coordinates + 0.5), for the warp-uniform reject
template <int NT>
__device__ __forceinline__ void warp_rect(int w, int tx, int ty, float &x0, float &x1, float &y0, float &y1) {
  int ox, oy, wx, wy;
  if (NT == 128) { ox = (w & 1) * 8; oy = (w >> 1) * 8; wx = 8; wy = 8; }
  else if (NT == 64) { ox = 0; oy = w * 8; wx = 16; wy = 8; }
  else { ox = (w & 1) * 8; oy = (w >> 1) * 4; wx = 8; wy = 4; }
  x0 = (float)(tx * LP_TILE + ox) + 0.5f;
  x1 = x0 + (float)(wx - 1);
  y0 = (float)(ty * LP_TILE + oy) + 0.5f;
  y1 = y0 + (float)(wy - 1);
}

// does the primitive's screen bbox reach the warp's pixel-centre rectangle?
__device__ __forceinline__ bool rect_hits_bbox(const float4 &bb, float x0, float x1, float y0, float y1) {
  return bb.x - bb.z <= x1 && bb.x + bb.z >= x0 && bb.y - bb.w <= y1 && bb.y + bb.w >= y0;
}

// Build the warp's ordered sub-list of batch records [0, cnt) whose bbox reaches its rectangle.
// Lane l tests records l, l+32, ...; returns the list length (warp-uniform).
// WM: the records' per-warp masks s_wm (octahedron_ / tetrahedron_warp_mask) replace the bbox test.
template <int NT, int RW4, bool WM>
__device__ __forceinline__ int warp_sublist(const float4 *s_rec, const unsigned char *s_wm, int cnt, float x0,
                                            float x1, float y0, float y1, unsigned char *list) {
  const int lane = threadIdx.x & 31;
  const unsigned lt = (1u << lane) - 1u;
  int n = 0;
#pragma unroll
  for (int r = 0; r < NT; r += 32) {
    const int j = r + lane;
    const bool ov = j < cnt && (WM ? ((s_wm[j] >> (threadIdx.x >> 5)) & 1u) != 0
                                   : rect_hits_bbox(s_rec[j * RW4], x0, x1, y0, y1));
    const unsigned m = __ballot_sync(0xffffffffu, ov);
    if (ov) list[n + __popc(m & lt)] = (unsigned char)j;
    n += __popc(m);
  }
  __syncwarp();
  return n;
}

// Which of the CTA's four 8x8 warp rectangles (NT = 128: warp w at (8 (w & 1), 8 (w >> 1)) in the
// tile) the octahedron's screen footprint can reach: the record's bbox against each rectangle, then
// the separating-axis test against the six strips that bound the footprint,
//   chord(D) > 0  =>  |(b_s - b_t) D.x + (g_s - g_t) D.y| < h_s + h_t   for every slab pair {s, t}
// (min_s (L_s + h_s) > max_t (L_t - h_t) with L = b D.x + g D.y, D relative to the centre).  A
// rectangle with centre D_c and half-size 3.5 misses strip {s, t} if |a . D_c| > h_s + h_t +
// 3.5 (|a.x| + |a.y|); the bound is widened by 1e-4 relative plus 1e-5 of the evaluated terms so fp32
// rounding never drops a record with a hit.  Computed once per staged record by its staging thread
// (instead of a bbox test per warp): on C5 about half of the bbox sub-list entries hit no pixel of
// the warp.
__device__ __forceinline__ unsigned octahedron_warp_mask(const float4 *r, int tx, int ty) {
  const float4 bb = r[0];
  const float b[4] = {r[1].x, r[1].w, r[2].z, r[3].y};
  const float g[4] = {r[1].y, r[2].x, r[2].w, r[3].z};
  const float h[4] = {r[1].z, r[2].y, r[3].x, r[3].w};
  const float dcx = (float)(tx * LP_TILE) + 4.f - bb.x, dcy = (float)(ty * LP_TILE) + 4.f - bb.y;
  unsigned m = 0u;
#pragma unroll
  for (int w = 0; w < 4; ++w) {
    const float ox = (w & 1) ? 8.f : 0.f, oy = (w & 2) ? 8.f : 0.f;
    if (fabsf(dcx + ox) <= bb.z + 3.5f && fabsf(dcy + oy) <= bb.w + 3.5f) m |= 1u << w;
  }
  const float K = 1e-5f * (fabsf(dcx) + fabsf(dcy) + 16.f);
#pragma unroll
  for (int s = 0; s < 4; ++s)
#pragma unroll
    for (int t = s + 1; t < 4; ++t) {
      const float ax = b[s] - b[t], ay = g[s] - g[t], aa = fabsf(ax) + fabsf(ay);
      const float e = fmaf(aa, K, (h[s] + h[t] + 3.5f * aa) * 1.0001f);
      const float v0 = fmaf(ax, dcx, ay * dcy), v1 = fmaf(8.f, ax, v0), v2 = fmaf(8.f, ay, v0), v3 = fmaf(8.f, ay, v1);
      m &= (fabsf(v0) <= e ? 1u : 0u) | (fabsf(v1) <= e ? 2u : 0u) | (fabsf(v2) <= e ? 4u : 0u) |
           (fabsf(v3) <= e ? 8u : 0u);
    }
  return m;
}

// The same for a tetrahedron: chord(D) > 0 needs every back plane above every front plane,
//   (A_b - A_f) + (B_b - B_f) D.x + (C_b - C_f) D.y > 0   (front slots 0-2, back slots 3-5),
// so a rectangle misses the footprint if for some pair the maximum of that plane over it is < 0.
__device__ __forceinline__ unsigned tetrahedron_warp_mask(const float4 *r, int tx, int ty) {
  const float4 bb = r[0];
  const float cx = r[1].x, cy = r[1].y;
  const float w_[24] = {r[1].z, r[1].w, r[2].x, r[2].y, r[2].z, r[2].w, r[3].x, r[3].y, r[3].z, r[3].w, r[4].x,
                        r[4].y, r[4].z, r[4].w, r[5].x, r[5].y, r[5].z, r[5].w, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f};
  const float X = (float)(tx * LP_TILE) + 4.f, Y = (float)(ty * LP_TILE) + 4.f;
  const float dbx = X - bb.x, dby = Y - bb.y, dcx = X - cx, dcy = Y - cy;
  unsigned m = 0u;
#pragma unroll
  for (int w = 0; w < 4; ++w) {
    const float ox = (w & 1) ? 8.f : 0.f, oy = (w & 2) ? 8.f : 0.f;
    if (fabsf(dbx + ox) <= bb.z + 3.5f && fabsf(dby + oy) <= bb.w + 3.5f) m |= 1u << w;
  }
  const float K = 1e-5f * (fabsf(dcx) + fabsf(dcy) + 16.f);
#pragma unroll
  for (int f = 0; f < 3; ++f)
#pragma unroll
    for (int bk = 3; bk < 6; ++bk) {
      const float dA = w_[3 * bk] - w_[3 * f], dB = w_[3 * bk + 1] - w_[3 * f + 1], dC = w_[3 * bk + 2] - w_[3 * f + 2];
      const float aa = fabsf(dB) + fabsf(dC);
      const float tol = fmaf(aa, K, 1e-4f * (fabsf(w_[3 * bk]) + fabsf(w_[3 * f]) + 3.5f * aa));
      const float lim = -(dA + 3.5f * aa + tol);   // keep warp w if dB D.x + dC D.y >= lim at its centre
      const float v0 = fmaf(dB, dcx, dC * dcy), v1 = fmaf(8.f, dB, v0), v2 = fmaf(8.f, dC, v0), v3 = fmaf(8.f, dC, v1);
      m &= (v0 >= lim ? 1u : 0u) | (v1 >= lim ? 2u : 0u) | (v2 >= lim ? 4u : 0u) | (v3 >= lim ? 8u : 0u);
    }
  return m;
}

// 16-byte global -> shared copies that bypass the registers (cp.async, L2 only): the backward
// stages the next batch's records while it processes the current one
__device__ __forceinline__ void cp_async16(void *smem, const void *gmem) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(static_cast<uint32_t>(__cvta_generic_to_shared(smem))),
               "l"(gmem)
               : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
__device__ __forceinline__ void cp_async_wait_all() { asm volatile("cp.async.wait_all;" ::: "memory"); }

// resident CTAs per SM the backward asks the register allocator for (LP_BWD_BLOCKS overrides at
// build time): 6 x 128 threads allows 80 registers (measured on C5 with the shared-row moments:
// 6 -> 0.613 ms, 7 (72 registers) -> 0.616, 8 (64) -> 0.616)
#ifndef LP_BWD_BLOCKS
#define LP_BWD_BLOCKS 6
#endif
// (tetrahedra: 29.7 KB of shared memory per CTA fits at most 7 per SM)
#define BWD_MIN_BLOCKS(kind, nt) \
  ((nt) == 128 ? ((kind) == LP_OCTAHEDRON || LP_BWD_BLOCKS < 7 ? LP_BWD_BLOCKS : 7) : 1)

#ifdef LP_BWD_STATS
// measurement build only (-DLP_BWD_STATS): warp-level event counts of the backward
// [0] sublist records, [1] records with a lane in bbox, [2] records with a hit lane, [3] sum of hit lanes,
// [5] in-bbox lane tests, [6] reductions where both pixel rows of the warp hit, [7] hit pixels,
// [8 + h] reductions with h hit lanes (h = 1..32), [41] / [42] (16x8 half, record) iterations and their
// active pixel rows under a 2-warps-per-tile, 4-pixels-per-lane mapping
__device__ unsigned long long g_bwd_stats[48];
extern "C" int lp_debug_bwd_stats(unsigned long long *out, int reset) {
  cudaMemcpyFromSymbol(out, g_bwd_stats, sizeof(g_bwd_stats));
  if (reset) {
    unsigned long long z[48] = {};
    cudaMemcpyToSymbol(g_bwd_stats, z, sizeof(z));
  }
  return 0;
}
// counted per CTA in shared memory (s_bst), flushed once per CTA: same-address global atomics from every
// warp of the grid stall the kernel
#define BWD_STAT(i, v) do { if ((threadIdx.x & 31) == 0) atomicAdd(&s_bst[i], (unsigned)(v)); } while (0)
#else
#define BWD_STAT(i, v) do { } while (0)
#endif

// the forward's hit bits of 32 consecutive entries [bit0, bit0 + 32) into warp row w of the hit mask
// (once per batch; kept out of line so its 64-bit address math does not occupy registers across the
// record loop)
__device__ __noinline__ void write_hit_word(uint32_t *hitmask, int64_t capacity, int w, uint32_t bit0, uint32_t m) {
  uint32_t *row = hitmask + (size_t)w * hit_words(capacity);
  const uint32_t wd = bit0 >> 5, sh = bit0 & 31u;
  LP_CHECK((int64_t)wd + (sh ? 1 : 0) < hit_words(capacity));
  atomicOr(row + wd, m << sh);
  if (sh) atomicOr(row + wd + 1, m >> (32u - sh));
}

// =============================================================================================
// K3 forward
// =============================================================================================
// AUX: also the depth (entry distance of the first primitive after which the cumulative
// opacity 1 - T exceeds 0.5, 0 if never; reading 24) and alpha (1 - T_final) images,
// either pointer may be null.
//
// 128 threads, 2 pixels per thread: pixel k = 0 / 1 of a thread are (x, y) and (x, y + 4), so they
// share dx, and their chords are ONE paired evaluation (chord2: FFMA2 / FADD2
// lanes, bitwise the scalar chord the backward replays).
// EXACT: the no-ray-space variant (App. D, reading 27): per-pixel perspective rays
// r = ((x+0.5-cx)/fx, (y+0.5-cy)/fy, 1) against the record's camera-space planes.
// LP_FWD_BLOCKS (measurement knob): resident CTAs per SM asked of the register allocator.  Unset, the
// bound names no minimum: ptxas then allocates 64 registers (an explicit minimum of 1 gives 90)
#ifdef LP_FWD_BLOCKS
#define LP_FWD_BOUNDS __launch_bounds__(128, LP_FWD_BLOCKS)
#else
#define LP_FWD_BOUNDS __launch_bounds__(128)
#endif
template <int KIND, bool STATS, bool AUX, bool EXACT>
__global__ void LP_FWD_BOUNDS k_raster_fwd(lp_frame F, lp_camera cam, lp_raster_cfg cfg,
                                                    float *__restrict__ image, float *__restrict__ depth,
                                                    float *__restrict__ alpha) {
  constexpr int NT = 128, PPT = 2;
  using KD = Kind<KIND>;
  using ER = ExactRec<KIND>;
  constexpr int RW = EXACT ? ER::W : KD::RW, RW4 = RW / 4, RS = KD::RS;
  constexpr int SIGMA = EXACT ? ER::SIGMA : KD::SIGMA, RGB = EXACT ? ER::RGB : KD::RGB;
  __shared__ float4 s_rec[NT * RW4];
  __shared__ unsigned char s_list[NT / 32][NT];
  __shared__ unsigned char s_wm[NT];
  __shared__ unsigned char s_hit[NT / 32][NT];   // per warp: batch record j hit one of its pixels
  __shared__ unsigned long long s_stat[3];
  // per-record warp masks (footprint strips) in ray space; the bbox test in the counting and the
  // no-ray-space variants
  constexpr bool WM = !EXACT && !STATS && NT == 128;

  const int tile = blockIdx.x;
  const int tx = tile % F.tiles_x, ty = tile / F.tiles_x;
  const uint32_t start = F.ranges[2 * tile], end = F.ranges[2 * tile + 1];
  const int W = F.width, H = F.height;
  if (threadIdx.x < 3) s_stat[threadIdx.x] = 0ull;
  for (int i = threadIdx.x; i < NT * (NT / 32); i += NT) (&s_hit[0][0])[i] = 0;

  float fy[PPT], dep[PPT], tlast[PPT];
  float2 T2 = make_float2(1.f, 1.f), C2[3];   // transmittance and colour of the two pixels (lane k = pixel k)
  uint32_t nproc[PPT];
  const float tstop = effective_t_stop(cfg.t_stop);
  bool done[PPT], inside[PPT], dset[PPT];
  uint32_t nhit = 0, nbox = 0;
  float fx;
#pragma unroll
  for (int k = 0; k < PPT; ++k) {
    int x, y;
    pixel_of<NT>(threadIdx.x, k, x, y);
    x += tx * LP_TILE;
    y += ty * LP_TILE;
    inside[k] = x < W && y < H;
    fx = (float)x + 0.5f;
    fy[k] = (float)y + 0.5f;
    done[k] = !inside[k];
    nproc[k] = end - start;
    dep[k] = 0.f;
    tlast[k] = 1.f;
    dset[k] = false;
  }
#pragma unroll
  for (int c = 0; c < 3; ++c) C2[c] = make_float2(0.f, 0.f);
  // exact mode: the pixel rays (r_x shared by the pair, r_z = 1), their lengths and exact offsets
  ExactRay RY;
  if (EXACT) RY = make_ray(cam, fx, fy[0], fy[1]);
  const float2 rn2 = EXACT ? RY.rn2 : make_float2(1.f, 1.f);
  float wx0, wx1, wy0, wy1;
  warp_rect<NT>(threadIdx.x >> 5, tx, ty, wx0, wx1, wy0, wy1);

  for (uint32_t b = start; b < end; b += NT) {
    if (__syncthreads_and(done[0] && done[1])) break;   // also protects s_rec from the previous batch
    // the pixels' T in front of this batch: the backward restarts its T recovery here
    if (b > start) {
      LP_CHECK_CKPT(F, tile, start, b);
      *(ckpt_at(F.T_ckpt, tile, start, b) + threadIdx.x) = T2;
    }
    const uint32_t e = b + threadIdx.x;
    if (e < end) {
      LP_CHECK((int64_t)e < F.capacity);
      const uint32_t v = F.sorted_val[e];
      LP_CHECK(v < (uint32_t)F.n && F.tiles_touched[v] > 0);
      const float4 *src = reinterpret_cast<const float4 *>(F.record + (size_t)v * RS);
      float4 rv[RW4];
#pragma unroll
      for (int w = 0; w < RW4; ++w) rv[w] = __ldg(src + w);
#pragma unroll
      for (int w = 0; w < RW4; ++w) s_rec[threadIdx.x * RW4 + w] = rv[w];
      if constexpr (WM && KIND == LP_OCTAHEDRON) s_wm[threadIdx.x] = (unsigned char)octahedron_warp_mask(rv, tx, ty);
      if constexpr (WM && KIND == LP_TETRAHEDRON) s_wm[threadIdx.x] = (unsigned char)tetrahedron_warp_mask(rv, tx, ty);
    }
    __syncthreads();
    if (__all_sync(0xffffffffu, done[0] && done[1])) continue;
    const int cnt = (int)min((uint32_t)NT, end - b);
    const int wrp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    uint32_t hitw = 0u;                                 // lane L < NT/32: the warp's hit bits of records 32L..
    // per-warp sub-list: the batch records whose footprint (WM) or bbox reaches the warp's pixels, in
    // list order (convexity: outside the footprint / vertex bbox the chord is <= 0)
    const int nl = warp_sublist<NT, RW4, WM>(s_rec, s_wm, cnt, wx0, wx1, wy0, wy1, s_list[wrp]);
    for (int q = 0; q < nl; ++q) {
      const int j = s_list[wrp][q];
      bool test[PPT];
      if (STATS || EXACT) {
        // per-pixel bbox test (the in-bbox counter; exact mode: degenerate records are marked by an
        // empty bbox only)
        const float4 bb = s_rec[j * RW4];
        const bool inx = fabsf(fx - bb.x) <= bb.z;
#pragma unroll
        for (int k = 0; k < PPT; ++k) test[k] = !done[k] && inx && fabsf(fy[k] - bb.y) <= bb.w;
        if (!__any_sync(0xffffffffu, test[0] || test[1])) continue;
      } else {
        // ray space: no per-pixel bbox test -- the record's bbox reaches the warp's pixel rectangle
        // (sub-list), and outside the primitive the chord is <= 0 (the backward's hit test is
        // chord > 0 alone); a warp whose pixels all stopped skips the compositing and leaves at the
        // next batch
#pragma unroll
        for (int k = 0; k < PPT; ++k) test[k] = !done[k];
      }
      const float *rec = reinterpret_cast<const float *>(&s_rec[j * RW4]);
      float2 ch2, en2;
      if constexpr (EXACT) {
        PlanesE2 P;
        planesE2<KIND>(rec, RY, P);
        float2 ex2;
        const float pz = rec[ER::P + 2];
        const float2 cht = chordE2_of(P, pz, en2, ex2);
        ch2 = fmul2(cht, rn2);                         // Euclidean chord (negative: no hit)
        en2 = fmul2(fadd2(en2, bc(pz)), rn2);          // entry distance from the camera
      } else {
        const float dx = fs(fx, rec[KD::CX]);
        const float2 dy2 = fsub2(make_float2(fy[0], fy[1]), bc(rec[KD::CX + 1]));
        ch2 = chord2<KIND>(rec, dx, dy2, en2);
      }
      const float enk[PPT] = {en2.x, en2.y};
      bool hk[PPT];
#pragma unroll
      for (int k = 0; k < PPT; ++k) hk[k] = test[k] && lane_k(ch2, k) > 0.f;
      if (STATS) nbox += (uint32_t)test[0] + (uint32_t)test[1];
      // the forward's hits of this record -> the warp's hit flags (one byte per batch record; lane 0
      // writes it, the batch's words are built by ballots after the sub-list)
      if (!__any_sync(0xffffffffu, hk[0] || hk[1])) continue;
      if (lane == 0) s_hit[wrp][j] = 1;
      // both pixels composited as f32x2 pairs; a pixel this record does not hit gets chord 0 ->
      // x = 0, E = 1, o = 0, leaving its T and colour bitwise unchanged
      const float2 Tin = T2;
      {
        const float sig = rec[SIGMA];
        const float2 X = make_float2(hk[0] ? optical_depth(sig, ch2.x) : 0.f, hk[1] ? optical_depth(sig, ch2.y) : 0.f);
        const float2 E = make_float2(transmit_x(X.x), transmit_x(X.y));
        const float2 wgt = fmul2(T2, opacity_x2(X, E));
#pragma unroll
        for (int c = 0; c < 3; ++c) C2[c] = ffma2(wgt, bc(rec[RGB + c]), C2[c]);
        T2 = fmul2(T2, E);
      }
      if (AUX) {
#pragma unroll
        for (int k = 0; k < PPT; ++k) {
          if (hk[k] && !dset[k] && lane_k(T2, k) < 0.5f) {   // cumulative opacity 1 - T > 0.5 (once per pixel)
            dset[k] = true;
            if (EXACT) {
              dep[k] = enk[k];
            } else {
              const uint32_t id = F.sorted_val[b + (uint32_t)j];
              dep[k] = fa(__uint_as_float(F.depth_key[id]), enk[k]);
            }
          }
        }
      }
      if (STATS) nhit += (uint32_t)hk[0] + (uint32_t)hk[1];
      // include-then-stop (readings 9, 28): a pixel stops at most once, so the common path is one
      // predicate test per pixel pair
      const bool st0 = hk[0] && T2.x < tstop, st1 = hk[1] && T2.y < tstop;
      if (__any_sync(0xffffffffu, st0 || st1)) {   // warp-uniform: the compiler would predicate a lane branch
#pragma unroll
        for (int k = 0; k < PPT; ++k) {
          if (k == 0 ? st0 : st1) {
            done[k] = true;
            nproc[k] = b + (uint32_t)j - start + 1;
            tlast[k] = lane_k(Tin, k);   // T in front of the stopping entry (the backward's start)
          }
        }
        // every pixel of the warp stopped: the rest of its sub-list cannot change them
        if (__all_sync(0xffffffffu, done[0] && done[1])) break;
      }
    }
    // this batch's hit bits of the warp -> the global per-warp bit row (entry index = bit index)
    __syncwarp();
#pragma unroll
    for (int i = 0; i < NT / 32; ++i) {
      const unsigned m = __ballot_sync(0xffffffffu, s_hit[wrp][32 * i + lane] != 0);
      if (lane == i) hitw = m;
      s_hit[wrp][32 * i + lane] = 0;
    }
    if (hitw) write_hit_word(F.hitmask, F.capacity, wrp, b + 32u * (uint32_t)lane, hitw);
  }

  const size_t HW = (size_t)W * H;
  unsigned long long it = 0;
#pragma unroll
  for (int k = 0; k < PPT; ++k) {
    if (!inside[k]) continue;
    const int x = (int)fx, y = (int)fy[k];
    const size_t p = (size_t)y * W + x;
    const float Tk = lane_k(T2, k);
    image[p] = fmaf(Tk, cfg.bg[0], lane_k(C2[0], k));
    image[HW + p] = fmaf(Tk, cfg.bg[1], lane_k(C2[1], k));
    image[2 * HW + p] = fmaf(Tk, cfg.bg[2], lane_k(C2[2], k));
    F.T_final[p] = Tk;
    F.T_last[p] = Tk < tstop ? tlast[k] : Tk;
    F.n_proc[p] = nproc[k];
    if (AUX) {
      if (depth) depth[p] = dep[k];
      if (alpha) alpha[p] = 1.f - Tk;
    }
    it += nproc[k];
  }
  if (STATS) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      it += __shfl_xor_sync(0xffffffffu, it, o);
      nhit += __shfl_xor_sync(0xffffffffu, nhit, o);
      nbox += __shfl_xor_sync(0xffffffffu, nbox, o);
    }
    __syncthreads();
    if ((threadIdx.x & 31) == 0) {
      atomicAdd(&s_stat[0], it);
      atomicAdd(&s_stat[1], (unsigned long long)nhit);
      atomicAdd(&s_stat[2], (unsigned long long)nbox);
    }
    __syncthreads();
    if (threadIdx.x == 0) {
      atomicAdd(reinterpret_cast<unsigned long long *>(F.counters + LP_CNT_ITERATED), s_stat[0]);
      atomicAdd(reinterpret_cast<unsigned long long *>(F.counters + LP_CNT_INTERSECTED), s_stat[1]);
      atomicAdd(reinterpret_cast<unsigned long long *>(F.counters + LP_CNT_INBOX), s_stat[2]);
    }
  }
}

// =============================================================================================
// K4 backward
// =============================================================================================
// EXACT: the no-ray-space variant; per plane f the moments are (dL/dm_f, dL/dn_f) with
// t = (m -+ 1)/k or m/k, k = n . r:  dt/dm = 1/k, dt/dn = -t r / k  (reading 27).
template <int KIND, int NT, bool EXACT>
__global__ void __launch_bounds__(NT, BWD_MIN_BLOCKS(KIND, NT)) k_raster_bwd(lp_frame F, lp_camera cam,
                                                                      lp_raster_cfg cfg,
                                                                      const float *__restrict__ dL) {
  static_assert(NT == 128, "paired pixel evaluation assumes 2 pixels per thread");
  using KD = Kind<KIND>;
  using ER = ExactRec<KIND>;
  constexpr int RW = EXACT ? ER::W : KD::RW, RW4 = RW / 4, PPT = 256 / NT, RG = KD::RG, RS = KD::RS;
  constexpr int SIGMA = EXACT ? ER::SIGMA : KD::SIGMA, RGB = EXACT ? ER::RGB : KD::RGB;
  constexpr int RGP = RG == 20 ? 20 : 28;      // padded row: 16-byte stores, conflict-free (RGP/4 odd)
  __shared__ float4 s_rec2[2][NT * RW4];   // double-buffered batch records (cp.async)
  __shared__ __align__(16) float s_red[NT / 32][32][RGP];
  __shared__ uint32_t s_id2[2][NT];
  __shared__ uint32_t s_last;
#ifdef LP_BWD_STATS
  __shared__ unsigned s_bst[48];
  __shared__ unsigned char s_pairs[4][NT];   // per warp and batch record: hit row-pair mask
  if (threadIdx.x < 48) s_bst[threadIdx.x] = 0u;
  for (int q = threadIdx.x; q < 4 * NT; q += NT) (&s_pairs[0][0])[q] = 0;
#endif

  const int tile = blockIdx.x;
  const int tx = tile % F.tiles_x, ty = tile / F.tiles_x;
  const uint32_t start = F.ranges[2 * tile], end = F.ranges[2 * tile + 1];
  if (end <= start) return;
  const int W = F.width, H = F.height;
  const size_t HW = (size_t)W * H;
  const int lane = threadIdx.x & 31;
  if (threadIdx.x == 0) s_last = start;
  __syncthreads();

  float fx[PPT], fy[PPT], T[PPT], S[PPT][3], G[PPT][3];
  uint32_t last[PPT];
  // T[k]: the pixel's transmittance in front of the hit entry processed last (the next one in list
  // order); fresh[k]: T[k] is already the T in front of the upcoming hit (no division).  A stopped
  // pixel starts from T_last (T in front of its stopping entry), every other one from T_final.
  bool fresh[PPT];
  const float tstop = effective_t_stop(cfg.t_stop);
#pragma unroll
  for (int k = 0; k < PPT; ++k) {
    int x, y;
    pixel_of<NT>(threadIdx.x, k, x, y);
    x += tx * LP_TILE;
    y += ty * LP_TILE;
    const bool in = x < W && y < H;
    fx[k] = (float)x + 0.5f;
    fy[k] = (float)y + 0.5f;
    const size_t p = in ? (size_t)y * W + x : 0;
    const float tf = in ? F.T_final[p] : 1.f;
    fresh[k] = tf < tstop;                          // stopped (include-then-stop)
    T[k] = fresh[k] ? F.T_last[p] : tf;
    last[k] = in ? start + F.n_proc[p] : start;     // entries [start, last) were processed
#pragma unroll
    for (int c = 0; c < 3; ++c) {
      S[k][c] = cfg.bg[c];
      G[k][c] = in ? dL[c * HW + p] : 0.f;
    }
    if (last[k] > start) atomicMax(&s_last, last[k]);
  }
  __syncthreads();
  const uint32_t lmax = s_last;
  float wx0, wx1, wy0, wy1;
  warp_rect<NT>(threadIdx.x >> 5, tx, ty, wx0, wx1, wy0, wy1);
  // exact mode: the pixel rays (bitwise the forward's)
  ExactRay RY;
  if (EXACT) RY = make_ray(cam, fx[0], fy[0], fy[1]);
  const float rx = EXACT ? RY.rx : 0.f;
  const float2 ry2 = EXACT ? RY.ry2 : make_float2(0.f, 0.f);
  const float2 rn2 = EXACT ? RY.rn2 : make_float2(1.f, 1.f);

  // batches walk the list backwards, aligned with the forward's (entries [start + 128 i, start +
  // 128 (i + 1)), the top one cut at lmax): batch [bstart(bend), bend), the next one ends at bstart
  auto bstart_of = [&](uint32_t be) { return be > start ? start + (((be - 1u - start) / NT) * NT) : start; };
  // this thread's entry of the batch ending at `be` (its primitive id; false if none)
  auto entry_of = [&](uint32_t be, uint32_t &v) {
    if (be <= start) return false;
    const uint32_t e = bstart_of(be) + threadIdx.x;
    if (e >= be) return false;
    LP_CHECK((int64_t)e < F.capacity);
    v = F.sorted_val[e];
    LP_CHECK(v < (uint32_t)F.n);
    return true;
  };
  auto stage = [&](int bf, uint32_t v) {
    s_id2[bf][threadIdx.x] = v;
    const float4 *src = reinterpret_cast<const float4 *>(F.record + (size_t)v * RS);
#pragma unroll
    for (int w = 0; w < RW4; ++w) cp_async16(&s_rec2[bf][threadIdx.x * RW4 + w], src + w);
  };
  // prologue: the first batch in flight, the second batch's primitive id loaded
  uint32_t vcur = 0, vnext = 0;
  if (entry_of(lmax, vcur)) stage(0, vcur);
  cp_async_commit();
  bool has_next = entry_of(bstart_of(lmax), vnext);
  int buf = 0;
  for (uint32_t bend = lmax; bend > start; bend = bstart_of(bend), buf ^= 1) {
    const uint32_t bstart = bstart_of(bend);
    cp_async_wait_all();
    __syncthreads();   // this batch landed for every thread; every thread is done with the other buffer
#ifdef LP_BWD_STATS
    // the previous batch's (16x8 half, record) iterations [41] and their active pixel rows [42] under a
    // 2-warps-per-tile, 4-pixels-per-lane mapping (halves = warps 0|1 and 2|3)
    if (threadIdx.x < NT) {
      const int j = threadIdx.x;
      const unsigned h0 = s_pairs[0][j] | s_pairs[1][j], h1 = s_pairs[2][j] | s_pairs[3][j];
      const unsigned it = (h0 != 0u) + (h1 != 0u), rows = __popc(h0) + __popc(h1);
      if (it) atomicAdd(&s_bst[41], it);
      if (rows) atomicAdd(&s_bst[42], rows);
    }
    __syncthreads();
    for (int q = threadIdx.x; q < 4 * NT; q += NT) (&s_pairs[0][0])[q] = 0;
#endif
    // the next batch's records into the other buffer (their ids were loaded one batch ago), and
    // the id of the batch after it
    if (has_next) stage(buf ^ 1, vnext);
    cp_async_commit();
    has_next = bstart > start && entry_of(bstart_of(bstart), vnext);
    const float4 *s_rec = s_rec2[buf];
    const uint32_t *s_id = s_id2[buf];
    bool act = false, after = false;
#pragma unroll
    for (int k = 0; k < PPT; ++k) {
      act = act || (last[k] > bstart);
      after = after || (last[k] > bend);
    }
    if (!__any_sync(0xffffffffu, act)) continue;
    // re-anchor the T recovery at the forward's checkpoint in front of the next batch: the
    // divisions T / E never chain across more than one 128-entry batch
    if (after) {
      LP_CHECK_CKPT(F, tile, start, bend);
      const float2 c = *(ckpt_at(F.T_ckpt, tile, start, bend) + threadIdx.x);
#pragma unroll
      for (int k = 0; k < PPT; ++k)
        if (last[k] > bend) {
          T[k] = lane_k(c, k);
          fresh[k] = false;
        }
    }
    const int w = threadIdx.x >> 5;
    // the entries of this batch that hit one of the warp's pixels in the forward (its hit bits):
    // no rect / bbox tests and no chord evaluation of entries that miss every pixel of the warp
    uint32_t hb[NT / 32];
    {
      const uint32_t *row = F.hitmask + (size_t)w * hit_words(F.capacity);
      uint32_t mine = 0u;
      if (lane < NT / 32) {
        const uint32_t bit0 = bstart + 32u * lane, wd = bit0 >> 5, sh = bit0 & 31u;
        mine = row[wd] >> sh;
        if (sh) mine |= row[wd + 1] << (32u - sh);
        const int rem = (int)(bend - bstart) - 32 * lane;   // records of this word inside the batch
        if (rem < 32) mine = rem <= 0 ? 0u : (mine & ((1u << rem) - 1u));
      }
#pragma unroll
      for (int i = 0; i < NT / 32; ++i) hb[i] = __shfl_sync(0xffffffffu, mine, i);
    }
    BWD_STAT(0, __popc(hb[0]) + __popc(hb[1]) + __popc(hb[2]) + __popc(hb[3]));

#pragma unroll 1
    for (int wi = NT / 32 - 1; wi >= 0; --wi) {
    uint32_t bits = hb[0];
#pragma unroll
    for (int i = 1; i < NT / 32; ++i)
      if (wi == i) bits = hb[i];
    while (bits) {
      const int bt = 31 - __clz(bits);
      bits &= ~(1u << bt);
      const int j = 32 * wi + bt;
      const uint32_t ej = bstart + (uint32_t)j;
      // a pixel outside the primitive has chord <= 0; the forward stopped pixel k after last[k].  (No
      // vote to skip the entry: the forward set its hit bit for a pixel that had not stopped, so some
      // pixel of the warp has ej < last.)
      bool test[PPT], any = false;
#pragma unroll
      for (int k = 0; k < PPT; ++k) {
        test[k] = ej < last[k];
        any = any || test[k];
      }
#ifdef LP_CHECKED
      LP_CHECK(__any_sync(0xffffffffu, any));
#endif
      (void)any;
      BWD_STAT(1, 1);
#ifdef LP_BWD_STATS
      {
        unsigned nb = 0;
        for (int k = 0; k < PPT; ++k) nb += __popc(__ballot_sync(0xffffffffu, test[k]));
        BWD_STAT(5, nb);
      }
#endif
      const float *rec = reinterpret_cast<const float *>(&s_rec[j * RW4]);
      // the warp's pixels this entry hits (chord > 0 before the forward's stop): their lanes get a
      // compacted shared-memory row [dsigma, drgb | per-plane moments] that the pixels update in
      // place (one 16-byte read-modify-write per entry / exit plane, no per-plane selects)
      float2 ch2, en2, ex2;
      float dx = 0.f, dxp = 0.f;
      float2 dy2 = make_float2(0.f, 0.f), dyp2 = make_float2(0.f, 0.f);
      PlanesE2 PE;
      Planes2<KIND> PR;
      if (EXACT) {
        planesE2<KIND>(rec, RY, PE);
        ch2 = fmul2(chordE2_of(PE, rec[ER::P + 2], en2, ex2), rn2);
        exact_d<KIND>(rec, RY, dxp, dyp2);
      } else {
        dx = fs(fx[0], rec[KD::CX]);
        dy2 = fsub2(make_float2(fy[0], fy[1]), bc(rec[KD::CX + 1]));
        planes2<KIND>(rec, dx, dy2, PR);
        ch2 = chord2_of<KIND>(PR, en2, ex2);
      }
      bool hk[PPT], hit = false;
#pragma unroll
      for (int k = 0; k < PPT; ++k) {
        hk[k] = test[k] && lane_k(ch2, k) > 0.f;
        hit = hit || hk[k];
      }
      // (hm != 0: the chord is bitwise the forward's, which set this entry's hit bit; were it 0, the
      // entry would only add zero column sums)
      const unsigned hm = __ballot_sync(0xffffffffu, hit);
      LP_CHECK(hm != 0u);
      BWD_STAT(2, 1);
      BWD_STAT(3, __popc(hm));
      BWD_STAT(8 + __popc(hm), 1);
#ifdef LP_BWD_STATS
      {
        const bool a0 = __any_sync(0xffffffffu, hk[0]), a1 = __any_sync(0xffffffffu, hk[1]);
        const unsigned np = __popc(__ballot_sync(0xffffffffu, hk[0])) + __popc(__ballot_sync(0xffffffffu, hk[1]));
        BWD_STAT(6, a0 && a1);
        BWD_STAT(7, np);
        // row pairs {0,1}, {2,3}, {4,5}, {6,7} of the warp's 8x8 pixels with a hit (a 4-pixels-per-lane
        // mapping's pixel rows), kept per batch record for the 16x8 half-tile accounting below
        const unsigned b0 = __ballot_sync(0xffffffffu, hk[0]), b1 = __ballot_sync(0xffffffffu, hk[1]);
        unsigned pm = 0u;
#pragma unroll
        for (int r = 0; r < 8; ++r) {
          const unsigned rowbits = ((r < 4 ? b0 : b1) >> (8 * (r & 3))) & 0xFFu;
          if (rowbits) pm |= 1u << (r >> 1);
        }
        if (lane == 0) s_pairs[w][j] = (unsigned char)pm;
      }
#endif
      float *row = &s_red[w][__popc(hm & ((1u << lane) - 1u))][0];
      // sigma and colour into registers once per entry, by every lane (one broadcast load; inside
      // the hit lanes' loop the compiler re-reads them after every shared store to the rows)
      float sig, rgbv[3];
      if constexpr (SIGMA % 4 == 0 && RGB == SIGMA + 1) {
        const float4 v = reinterpret_cast<const float4 *>(rec)[SIGMA / 4];
        sig = v.x;
        rgbv[0] = v.y;
        rgbv[1] = v.z;
        rgbv[2] = v.w;
      } else {
        sig = rec[SIGMA];
#pragma unroll
        for (int c = 0; c < 3; ++c) rgbv[c] = rec[RGB + c];
      }
      if (hit) {
#pragma unroll
        for (int a = 1; a < RGP / 4; ++a) reinterpret_cast<float4 *>(row)[a] = make_float4(0.f, 0.f, 0.f, 0.f);
        float4 tail = make_float4(0.f, 0.f, 0.f, 0.f);   // dsigma, dr, dg, db
#pragma unroll
        for (int k = 0; k < PPT; ++k) {
          if (!hk[k]) continue;
          const float ch = lane_k(ch2, k), te = lane_k(en2, k), tx_ = lane_k(ex2, k);
          int se, sx;
          if (EXACT) trackE_k(PE, k, te, tx_, se, sx);
          else track_k<KIND>(PR, k, te, tx_, se, sx);
          const float x = optical_depth(sig, ch);
          const float E = transmit_x(x);
          const float o = opacity_x(x, E);
          const float Tk = fresh[k] ? T[k] : T[k] * rcp_ftz(E);   // transmittance in front of this entry
          fresh[k] = false;
          float dLdo = 0.f;
          tail.y = fmaf(Tk * o, G[k][0], tail.y);           // dL/drgb
          tail.z = fmaf(Tk * o, G[k][1], tail.z);
          tail.w = fmaf(Tk * o, G[k][2], tail.w);
#pragma unroll
          for (int c = 0; c < 3; ++c) {
            dLdo = fmaf(rgbv[c] - S[k][c], G[k][c], dLdo);
            S[k][c] = fmaf(o, rgbv[c], E * S[k][c]);        // colour behind the previous entry
          }
          dLdo *= Tk;
          T[k] = Tk;
          const float gE = E * dLdo;
          tail.x = fmaf(ch, gE, tail.x);                    // dL/dsigma = chord E dL/do
          float4 *slot = reinterpret_cast<float4 *>(row + 4);
          if (EXACT) {
            // centred moments: dL/dm = dL/dt / k and dL/dn = -dL/dt (q - p) / k with
            // q - p = tau r - d (tau = t - p_z, d = p - p_z r)
            const float ry = lane_k(ry2, k), dyp = lane_k(dyp2, k);
            const float wt = sig * gE * lane_k(rn2, k);    // dL/dt_exit = wt, dL/dt_entry = -wt
            const float ax = wt * plane_ik<KIND>(rec, sx, rx, ry), ae = -wt * plane_ik<KIND>(rec, se, rx, ry);
            const float qx0 = fmaf(tx_, rx, -dxp), qx1 = fmaf(tx_, ry, -dyp);
            const float qe0 = fmaf(te, rx, -dxp), qe1 = fmaf(te, ry, -dyp);
            {   // exit then entry plane, one read-modify-write each in order (no branch: se == sx sums too)
              float4 m = slot[sx];
              m.x += ax;
              m.y -= ax * qx0;
              m.z -= ax * qx1;
              m.w -= ax * tx_;
              slot[sx] = m;
              float4 n = slot[se];
              n.x += ae;
              n.y -= ae * qe0;
              n.z -= ae * qe1;
              n.w -= ae * te;
              slot[se] = n;
            }
          } else if (KIND == OCTA) {
            // slab s: (dL/da, dL/db, dL/dc, dL/dhalf) += (w dx, w dy, w, u) with w = gx - gn, u = gx + gn
            const float g = sig * gE, dy = lane_k(dy2, k);   // dL/d exit = g, dL/d entry = -g
            {   // exit then entry slab, one read-modify-write each in order (no branch: se == sx sums too)
              float4 m = slot[sx];
              m.x = fmaf(g, dx, m.x);
              m.y = fmaf(g, dy, m.y);
              m.z += g;
              m.w += g;
              slot[sx] = m;
              float4 n = slot[se];
              n.x = fmaf(-g, dx, n.x);
              n.y = fmaf(-g, dy, n.y);
              n.z -= g;
              n.w += g;
              slot[se] = n;
            }
          } else {
            const float g = sig * gE, dy = lane_k(dy2, k);
            float *px = row + 4 + 3 * sx, *pe = row + 4 + 3 * se;
            const float x0 = px[0], x1 = px[1], x2 = px[2], e0 = pe[0], e1 = pe[1], e2 = pe[2];
            px[0] = x0 + g;
            px[1] = fmaf(g, dx, x1);
            px[2] = fmaf(g, dy, x2);
            pe[0] = e0 - g;
            pe[1] = fmaf(-g, dx, e1);
            pe[2] = fmaf(-g, dy, e2);
          }
        }
        reinterpret_cast<float4 *>(row)[0] = tail;
      }
      // per-(warp, primitive) reduction of the <= 22 moments, one RED.F32 per moment: lane m < RG
      // sums column m over the h rows (2 instructions per row, 4 independent partial sums)
      const uint32_t id = s_id[j];
      const int h = __popc(hm);
      __syncwarp();
      if (lane < RG) {
        const float *col = &s_red[w][0][lane];
        float s0 = 0.f, s1 = 0.f, s2 = 0.f, s3 = 0.f;
        int q = 0;
        for (; q + 4 <= h; q += 4) {
          s0 += col[(q + 0) * RGP];
          s1 += col[(q + 1) * RGP];
          s2 += col[(q + 2) * RGP];
          s3 += col[(q + 3) * RGP];
        }
        if (q + 0 < h) s0 += col[(q + 0) * RGP];
        if (q + 1 < h) s1 += col[(q + 1) * RGP];
        if (q + 2 < h) s2 += col[(q + 2) * RGP];
        const float sum = (s0 + s1) + (s2 + s3);
        // the shared row's layout is the rgrad row's (dsigma, drgb | moments): the h-row column sums
        // land in one primitive's 80 / 96-byte row (3 sectors per RED instruction); deterministic
        // frames store the (entry, warp) partial instead, summed per primitive in a fixed order by
        // k_det_gather
        LP_CHECK((int64_t)ej < F.capacity && id < (uint32_t)F.n);
        if (F.deterministic) F.part[((size_t)ej * 4 + w) * lp_rgs<KIND>() + lane] = sum;
        // (zero column sums are added too: a branch around them diverged inside the 20 lanes and cost
        // more issue slots than the RED traffic it saved)
        else atomicAdd(F.rgrad + (size_t)id * lp_rgs<KIND>() + lane, sum);
      }
      __syncwarp();
    }
    }
  }
#ifdef LP_BWD_STATS
  __syncthreads();
  if (threadIdx.x < NT) {
    const int j = threadIdx.x;
    const unsigned h0 = s_pairs[0][j] | s_pairs[1][j], h1 = s_pairs[2][j] | s_pairs[3][j];
    const unsigned it = (h0 != 0u) + (h1 != 0u), rows = __popc(h0) + __popc(h1);
    if (it) atomicAdd(&s_bst[41], it);
    if (rows) atomicAdd(&s_bst[42], rows);
  }
  __syncthreads();
  if (threadIdx.x < 48 && s_bst[threadIdx.x]) atomicAdd(&g_bwd_stats[threadIdx.x], (unsigned long long)s_bst[threadIdx.x]);
#endif
}

// ---------------------------------------------------------------------------------------------
template <bool STATS, bool AUX, bool EXACT>
static void fwd_k(const lp_frame &F, const lp_camera &cam, const lp_raster_cfg &cfg, float *image, float *depth,
                  float *alpha, cudaStream_t st) {
  const int tiles = F.tiles_x * F.tiles_y;
  if (F.kind == LP_OCTAHEDRON)
    k_raster_fwd<LP_OCTAHEDRON, STATS, AUX, EXACT><<<tiles, 128, 0, st>>>(F, cam, cfg, image, depth, alpha);
  else k_raster_fwd<LP_TETRAHEDRON, STATS, AUX, EXACT><<<tiles, 128, 0, st>>>(F, cam, cfg, image, depth, alpha);
}

template <bool EXACT>
static void fwd_x(const lp_frame &F, const lp_camera &cam, const lp_raster_cfg &cfg, float *image, float *depth,
                  float *alpha, cudaStream_t st) {
  const bool aux = depth || alpha;
  if (cfg.count_stats) {
    if (aux) fwd_k<true, true, EXACT>(F, cam, cfg, image, depth, alpha, st);
    else fwd_k<true, false, EXACT>(F, cam, cfg, image, depth, alpha, st);
  } else {
    if (aux) fwd_k<false, true, EXACT>(F, cam, cfg, image, depth, alpha, st);
    else fwd_k<false, false, EXACT>(F, cam, cfg, image, depth, alpha, st);
  }
}

// count_stats: the backward's work counters from the forward's hit bits (SURVEY §8d K4 model):
// W_h = (warp, entry) pairs with a hit (popcount of the four warp rows), A = (tile, entry) pairs
// with a hit in any warp (popcount of their OR; entries of different tiles are disjoint)
__global__ void __launch_bounds__(256) k_hit_stats(const uint32_t *__restrict__ hitmask, int64_t words_per_row,
                                                   uint32_t *__restrict__ counters) {
  const int64_t nw = ((int64_t)min(counters[LP_CNT_ENTRIES], (uint32_t)(words_per_row - 2) * 32u) + 31) / 32;
  uint32_t wh = 0, a = 0;
  for (int64_t w = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; w < nw; w += (int64_t)gridDim.x * blockDim.x) {
    const uint32_t r0 = hitmask[w], r1 = hitmask[words_per_row + w], r2 = hitmask[2 * words_per_row + w],
                   r3 = hitmask[3 * words_per_row + w];
    wh += __popc(r0) + __popc(r1) + __popc(r2) + __popc(r3);
    a += __popc(r0 | r1 | r2 | r3);
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    wh += __shfl_xor_sync(0xffffffffu, wh, o);
    a += __shfl_xor_sync(0xffffffffu, a, o);
  }
  if ((threadIdx.x & 31) == 0) {
    atomicAdd(counters + LP_CNT_WARP_HITS, wh);
    atomicAdd(counters + LP_CNT_TILE_HITS, a);
  }
}

void launch_raster_fwd(const lp_frame &F, const lp_camera &cam, const lp_raster_cfg &cfg, float *image, float *depth,
                       float *alpha, cudaStream_t st) {
  cudaMemsetAsync(F.hitmask, 0, sizeof(uint32_t) * 4 * (size_t)hit_words(F.capacity), st);   // the backward's hit bits
  if (cfg.exact) fwd_x<true>(F, cam, cfg, image, depth, alpha, st);
  else fwd_x<false>(F, cam, cfg, image, depth, alpha, st);
  if (cfg.count_stats) {
    cudaMemsetAsync(F.counters + LP_CNT_WARP_HITS, 0, 8, st);
    k_hit_stats<<<148, 256, 0, st>>>(F.hitmask, hit_words(F.capacity), F.counters);
  }
}

// deterministic frames: every visible primitive's raster moments = the sum, over its
// emitted entries in emission order and the four warps in order, of the partials the backward stored
// for the (entry, warp) pairs the forward's hit bits mark -- a fixed summation order, so the
// gradients are bitwise reproducible.  One thread per primitive.
template <int KIND>
__global__ void __launch_bounds__(128) k_det_gather(lp_frame F) {
  constexpr int RG = Kind<KIND>::RG, RGS = lp_rgs<KIND>();
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= F.n) return;
  const uint32_t tt = F.tiles_touched[i];
  if (tt == 0) return;
  const uint32_t k0 = F.prim_emit[i];
  const int64_t hw = hit_words(F.capacity);
  float acc[RG];
#pragma unroll
  for (int a = 0; a < RG; ++a) acc[a] = 0.f;
  for (uint32_t t = 0; t < tt; ++t) {
    LP_CHECK((int64_t)k0 + t < F.capacity);
    const uint32_t e = F.emit_pos[k0 + t];
    LP_CHECK((int64_t)e < F.capacity);
#pragma unroll
    for (int w = 0; w < 4; ++w) {
      if (((F.hitmask[w * hw + (e >> 5)] >> (e & 31u)) & 1u) == 0u) continue;
      const float *row = F.part + ((size_t)e * 4 + w) * RGS;
#pragma unroll
      for (int a = 0; a < RG; ++a) acc[a] += row[a];
    }
  }
  float *dst = F.rgrad + (size_t)i * RGS;
#pragma unroll
  for (int a = 0; a < RGS; ++a) dst[a] = a < RG ? acc[a] : 0.f;
}

void launch_det_gather(const lp_frame &F, cudaStream_t st) {
  if (F.n <= 0 || !F.deterministic) return;
  if (F.kind == LP_OCTAHEDRON) k_det_gather<LP_OCTAHEDRON><<<(F.n + 127) / 128, 128, 0, st>>>(F);
  else k_det_gather<LP_TETRAHEDRON><<<(F.n + 127) / 128, 128, 0, st>>>(F);
}

void launch_raster_bwd(const lp_frame &F, const lp_camera &cam, const lp_raster_cfg &cfg, const float *dL,
                       cudaStream_t st) {
  const int tiles = F.tiles_x * F.tiles_y;
  if (cfg.exact) {
    if (F.kind == LP_OCTAHEDRON) k_raster_bwd<LP_OCTAHEDRON, 128, true><<<tiles, 128, 0, st>>>(F, cam, cfg, dL);
    else k_raster_bwd<LP_TETRAHEDRON, 128, true><<<tiles, 128, 0, st>>>(F, cam, cfg, dL);
  } else {
    if (F.kind == LP_OCTAHEDRON) k_raster_bwd<LP_OCTAHEDRON, 128, false><<<tiles, 128, 0, st>>>(F, cam, cfg, dL);
    else k_raster_bwd<LP_TETRAHEDRON, 128, false><<<tiles, 128, 0, st>>>(F, cam, cfg, dL);
  }
}

}  // namespace lp
