// lp_preprocess.cu -- K1 (forward preprocess, rows a1-a3) and K5 (preprocess backward, row a12).
//
// One thread per primitive.  Feature loads are SoA and coalesced across the warp (thread i reads
// element i of each component array).  HBM-bound: see DESIGN.md §7 for the algorithmic bytes.
#include <cuda_runtime.h>
#include <stdint.h>

#include "lp_device.cuh"
#include "lp_kernels.h"
#include "lp_sh.cuh"

namespace lp {

__device__ __forceinline__ void warp_count(uint32_t *ctr, bool pred) {
  const unsigned b = __ballot_sync(0xffffffffu, pred);
  if ((threadIdx.x & 31) == 0 && b) atomicAdd(ctr, (uint32_t)__popc(b));
}

// unclamped SH colour exactly as the forward computes it (fp32), shared by K1 and K5.  DEG is the
// compile-time SH degree: the (DEG+1)^2 x 3 coefficient loads are issued together, then summed in
// basis order (acc = 0.5 + sum_k sh_k Y_k, one FFMA per term).
template <int DEG>
__device__ __forceinline__ void sh_colour_fp32(const lp_prims &P, int i, const lp_camera &cam, const float c[3],
                                               float raw[3]) {
  constexpr int NC = (DEG + 1) * (DEG + 1);
  float shv[NC * 3];
#pragma unroll
  for (int q = 0; q < NC * 3; ++q) shv[q] = P.sh[(size_t)q * P.n + i];
  const float cpx = -(cam.W[0] * cam.t[0] + cam.W[3] * cam.t[1] + cam.W[6] * cam.t[2]);
  const float cpy = -(cam.W[1] * cam.t[0] + cam.W[4] * cam.t[1] + cam.W[7] * cam.t[2]);
  const float cpz = -(cam.W[2] * cam.t[0] + cam.W[5] * cam.t[1] + cam.W[8] * cam.t[2]);
  float vx = c[0] - cpx, vy = c[1] - cpy, vz = c[2] - cpz;
  const float inv = rsqrtf(vx * vx + vy * vy + vz * vz);
  vx *= inv;
  vy *= inv;
  vz *= inv;
  float Y[16];
  sh_basis<float>(DEG, vx, vy, vz, Y);
#pragma unroll
  for (int ch = 0; ch < 3; ++ch) {
    float acc = 0.5f;
#pragma unroll
    for (int k = 0; k < NC; ++k) acc += shv[k * 3 + ch] * Y[k];
    raw[ch] = acc;
  }
}

// =============================================================================================
// K1: features -> canonical geometry -> record, sigma (Eq. 1), SH colour
// =============================================================================================
// views preprocessed by one launch (features are read from HBM once, then L1/L2 for the others)
constexpr int LP_PRE_MAXV = 8;
struct PreViews {
  lp_camera cam[LP_PRE_MAXV];
  lp_frame frame[LP_PRE_MAXV];
  int nv;
};

template <int KIND, bool EXACT, int DEG>
__device__ __forceinline__ void preprocess_view(const lp_prims &P, const lp_camera &cam, float kappa,
                                                const lp_frame &F, int i);

// resident K1 blocks per SM asked of the register allocator (-DLP_PRE_MINB overrides): 4 x 256
// threads = 64 registers (70 unconstrained, 3 blocks)
#ifndef LP_PRE_MINB
#define LP_PRE_MINB 4
#endif
template <int KIND, bool EXACT, int DEG>
__global__ void __launch_bounds__(256, LP_PRE_MINB) k_preprocess(lp_prims P, float kappa, PreViews V) {
  // view-interleaved grid: the nv consecutive blocks of one primitive range run the nv views, so
  // the primitive features come from HBM once and from L2 for the other views
  const int v = blockIdx.x % V.nv;
  const int i = (blockIdx.x / V.nv) * blockDim.x + threadIdx.x;
  preprocess_view<KIND, EXACT, DEG>(P, V.cam[v], kappa, V.frame[v], i);
}

// exact-mode record planes (App. D, reading 27), fp64 from the canonical fp32 geometry
// returns false for a degenerate primitive (the caller empties its bbox)
template <int KIND>
__device__ __forceinline__ bool exact_planes(const Geom &g, float *rec) {
  using ER = ExactRec<KIND>;
  const double p[3] = {(double)g.crx, (double)g.cry, (double)g.cz};
  rec[ER::P] = g.crx;
  rec[ER::P + 1] = g.cry;
  rec[ER::P + 2] = g.cz;
  if (KIND == OCTA) {
    double M[3][3], G[3][3], det;
#pragma unroll
    for (int a = 0; a < 3; ++a)
#pragma unroll
      for (int j = 0; j < 3; ++j) M[a][j] = (double)g.off[j][a];
    inverse3(M, G, det);
    const bool ok = isfinite(det) && det != 0.0;
#pragma unroll
    for (int s = 0; s < 4; ++s) {
      float *n = rec + 4 + 3 * s;
#pragma unroll
      for (int c = 0; c < 3; ++c)
        n[c] = ok ? (float)(slab_sign(s, 0) * G[0][c] + slab_sign(s, 1) * G[1][c] + slab_sign(s, 2) * G[2][c]) : 0.f;
    }
    return ok;
  } else {
    double v[4][3];
#pragma unroll
    for (int k = 0; k < 4; ++k)
#pragma unroll
      for (int a = 0; a < 3; ++a) v[k][a] = p[a] + (double)g.off[k][a];
    bool ok = true;
    double nn[4][3], mm[4];
#pragma unroll
    for (int f = 0; f < 4; ++f) {
      const int ia = tetra_face(f, 0), ib = tetra_face(f, 1), ic = tetra_face(f, 2);
      const double e1[3] = {v[ib][0] - v[ia][0], v[ib][1] - v[ia][1], v[ib][2] - v[ia][2]};
      const double e2[3] = {v[ic][0] - v[ia][0], v[ic][1] - v[ia][1], v[ic][2] - v[ia][2]};
      nn[f][0] = e1[1] * e2[2] - e1[2] * e2[1];
      nn[f][1] = e1[2] * e2[0] - e1[0] * e2[2];
      nn[f][2] = e1[0] * e2[1] - e1[1] * e2[0];
      if (nn[f][0] == 0.0 && nn[f][1] == 0.0 && nn[f][2] == 0.0) ok = false;
      // m'_f = n_f . oc_a: the plane offset relative to the centre
      mm[f] = nn[f][0] * (double)g.off[ia][0] + nn[f][1] * (double)g.off[ia][1] + nn[f][2] * (double)g.off[ia][2];
    }
#pragma unroll
    for (int f = 0; f < 4; ++f) {
      float *pl = rec + 4 + 4 * f;
      pl[0] = ok ? (float)nn[f][0] : 0.f;
      pl[1] = ok ? (float)nn[f][1] : 0.f;
      pl[2] = ok ? (float)nn[f][2] : 1.f;
      pl[3] = ok ? (float)mm[f] : 0.f;
    }
    return ok;
  }
}

template <int KIND, bool EXACT, int DEG>
__device__ __forceinline__ void preprocess_view(const lp_prims &P, const lp_camera &cam, float kappa,
                                                const lp_frame &F, int i) {
  constexpr int K = Kind<KIND>::K, RW = Kind<KIND>::RW, RS = Kind<KIND>::RS;
  const bool inb = i < P.n;
  Geom g;
  float dh[4], q[4], c[3];
  g.flag = 1;
  g.tiles = 0;
  if (inb) canonical_geometry<KIND>(P, i, cam, kappa, g, dh, q, c, EXACT);
  warp_count(F.counters + LP_CNT_INVALID, inb && g.flag == 1);
  warp_count(F.counters + LP_CNT_FRUSTUM, inb && g.flag == 0);
  warp_count(F.counters + LP_CNT_VISIBLE, inb && g.tiles > 0);
  if (!inb) return;

  const bool ok = g.flag == 0;
  F.tiles_touched[i] = g.tiles;
  reinterpret_cast<ushort4 *>(F.rect)[i] =
      make_ushort4((unsigned short)g.rect[0], (unsigned short)g.rect[1], (unsigned short)g.rect[2],
                   (unsigned short)g.rect[3]);
  const uint32_t key = ok ? __float_as_uint(g.l) : 0u;
  F.depth_key[i] = key;
  F.prim_key[i] = g.tiles > 0 ? key : 0xFFFFFFFFu;   // invisible primitives sort last (emit nothing)
  F.prim_order[i] = (uint32_t)i;
  if (F.canon) {
    float *cn = F.canon + (size_t)i * (2 + 3 * K);
    cn[0] = ok ? g.crx : 0.f;
    cn[1] = ok ? g.cry : 0.f;
#pragma unroll
    for (int j = 0; j < K; ++j)
#pragma unroll
      for (int a = 0; a < 3; ++a) cn[2 + 3 * j + a] = ok ? g.off[j][a] : 0.f;
  }
  if (g.tiles == 0) return;   // only visible primitives need a record
  {
    // the backward's raster-moment row of this (primitive, view) starts at zero (only visible
    // primitives: K4 and K5 touch no other row).  Whole 32-byte sectors are written -- the row
    // plus the neighbours' bytes sharing its first / last sector (zeros as well, harmless) -- so
    // L2 never has to fetch a partially written sector from HBM.
    constexpr int RB = 4 * lp_rgs<KIND>();
    const size_t b0 = ((size_t)i * RB) & ~(size_t)31, b1 = ((size_t)i * RB + RB + 31) & ~(size_t)31;
    float4 *z = reinterpret_cast<float4 *>(reinterpret_cast<char *>(F.rgrad) + b0);
    const size_t zend = min(b1, (size_t)P.n * RB);
#pragma unroll
    for (int q = 0; q < (RB + 64) / 16; ++q)
      if (b0 + 16 * (size_t)q < zend) z[q] = make_float4(0.f, 0.f, 0.f, 0.f);
  }
  if (F.sort_method == LP_SORT_BUCKET) {
    // tile rect into the 2-D difference grid of the bucket sort (4 atomics instead of tiles_touched)
    const int cols = F.tiles_x + 1;
    atomicAdd(F.tile_diff + g.rect[1] * cols + g.rect[0], 1);
    atomicAdd(F.tile_diff + g.rect[1] * cols + g.rect[2] + 1, -1);
    atomicAdd(F.tile_diff + (g.rect[3] + 1) * cols + g.rect[0], -1);
    atomicAdd(F.tile_diff + (g.rect[3] + 1) * cols + g.rect[2] + 1, 1);
  }

  // ---- density, Eq. 1: sigma = -log(1 - 0.99 alpha) / (2 min dhat)
  const float alpha = 1.f / (1.f + expf(-P.opacity[i]));
  float md = dh[0];
#pragma unroll
  for (int a = 1; a < K; ++a) md = fminf(md, dh[a]);
  const float sigma = -log1pf(-0.99f * alpha) / (2.f * md);

  // ---- SH colour
  float rgb[3];
  sh_colour_fp32<DEG>(P, i, cam, c, rgb);
  // clamp max(0, .); a clamped channel is stored as -0.0 so the backward reads the clamp
  // decision from the record's sign bit instead of re-evaluating the SH colour
#pragma unroll
  for (int ch = 0; ch < 3; ++ch) rgb[ch] = rgb[ch] < 0.f ? -0.f : rgb[ch];

  // ---- raster record
  using KD = Kind<KIND>;
  if (EXACT) {
    using ER = ExactRec<KIND>;
    float rec[ER::W];
    const float hx = 0.5f * (g.bhi[0] - g.blo[0]), hy = 0.5f * (g.bhi[1] - g.blo[1]);
    rec[0] = 0.5f * (g.blo[0] + g.bhi[0]);
    rec[1] = 0.5f * (g.blo[1] + g.bhi[1]);
    rec[2] = hx * 1.0001f + 1e-3f;
    rec[3] = hy * 1.0001f + 1e-3f;
    if (!exact_planes<KIND>(g, rec)) rec[2] = rec[3] = -1.f;   // degenerate: no pixel passes the bbox test
    rec[ER::SIGMA] = sigma;
    rec[ER::RGB + 0] = rgb[0];
    rec[ER::RGB + 1] = rgb[1];
    rec[ER::RGB + 2] = rgb[2];
    rec[ER::W - 1] = 0.f;
    float4 *dst = reinterpret_cast<float4 *>(F.record + (size_t)i * RS);
#pragma unroll
    for (int w = 0; w < ER::W / 4; ++w)
      dst[w] = make_float4(rec[4 * w], rec[4 * w + 1], rec[4 * w + 2], rec[4 * w + 3]);
    return;
  }
  float rec[RW];
  // screen bbox of the (filtered) vertices, with a small slack (record word 0..3)
  float xlo = g.off[0][0], xhi = g.off[0][0], ylo = g.off[0][1], yhi = g.off[0][1];
#pragma unroll
  for (int j = 1; j < K; ++j) {
    xlo = fminf(xlo, g.off[j][0]); xhi = fmaxf(xhi, g.off[j][0]);
    ylo = fminf(ylo, g.off[j][1]); yhi = fmaxf(yhi, g.off[j][1]);
  }
  if (KIND == OCTA) {   // vertices c +- o_j: symmetric about c
    xhi = fmaxf(-xlo, xhi); xlo = -xhi;
    yhi = fmaxf(-ylo, yhi); ylo = -yhi;
  }
  const float hx = 0.5f * (xhi - xlo), hy = 0.5f * (yhi - ylo);
  rec[0] = g.crx + 0.5f * (xlo + xhi);
  rec[1] = g.cry + 0.5f * (ylo + yhi);
  rec[2] = hx * 1.0001f + 1e-3f;
  rec[3] = hy * 1.0001f + 1e-3f;
  rec[KD::CX] = g.crx;
  rec[KD::CX + 1] = g.cry;
  if (KIND == OCTA) {
    SlabRows S;
    octa_slabs(g.off, S);
#pragma unroll
    for (int s = 0; s < 4; ++s) {
      const double irz = 1.0 / S.r[s][2];   // one fp64 division per slab (K5 uses the same)
      rec[KD::SLAB + 3 * s] = S.ok ? (float)(-S.r[s][0] * irz) : 0.f;
      rec[KD::SLAB + 1 + 3 * s] = S.ok ? (float)(-S.r[s][1] * irz) : 0.f;
      rec[KD::SLAB + 2 + 3 * s] = S.ok ? (float)fabs(irz) : -1.f;   // h = -1: never intersected
    }
  } else {
    TetraPlanes T;
    tetra_planes(g.off, T);
#pragma unroll
    for (int s = 0; s < 6; ++s) {
      const int f = T.slot_face[s];
      rec[KD::SLAB + 3 * s] = T.ok ? (float)sel(T.A, f) : (s < 3 ? 1.f : -1.f);   // empty: entry 1 > exit -1
      rec[KD::SLAB + 1 + 3 * s] = T.ok ? (float)sel(T.B, f) : 0.f;
      rec[KD::SLAB + 2 + 3 * s] = T.ok ? (float)sel(T.C, f) : 0.f;
    }
  }
  rec[KD::SIGMA] = sigma;
  rec[KD::RGB + 0] = rgb[0];
  rec[KD::RGB + 1] = rgb[1];
  rec[KD::RGB + 2] = rgb[2];
  // the whole RS-word row (pad words zero): a partially written 32-byte sector would make L2 read it
  // from HBM first
  float4 *dst = reinterpret_cast<float4 *>(F.record + (size_t)i * RS);
#pragma unroll
  for (int w = 0; w < RS / 4; ++w)
    dst[w] = 4 * w < RW ? make_float4(rec[4 * w], rec[4 * w + 1], rec[4 * w + 2], rec[4 * w + 3])
                        : make_float4(0.f, 0.f, 0.f, 0.f);
}

// =============================================================================================
// K5: raster moments -> ray-space geometry -> world features
// One thread per primitive, looping over up to LP_MAXV views (the frames of one call): the
// feature gradients are accumulated in registers and written once per call, and a primitive
// invisible in one view usually has work in another (better SIMT utilisation).
// =============================================================================================
// views per K5 launch and resident K5 blocks per SM asked of the register allocator (measured on
// C5: 4 views x 8 blocks (128 registers, a few spills) beats 8 x 1 (196 registers, 40 KB smem)
// by 8 %; -DLP_K5_MAXV / -DLP_K5_MINB override)
#ifndef LP_K5_MAXV
#define LP_K5_MAXV 4
#endif
#ifndef LP_K5_MINB
#define LP_K5_MINB 8
#endif
constexpr int LP_MAXV = LP_K5_MAXV;
struct ViewPack {
  lp_camera cam[LP_MAXV];
  const float *rgrad[LP_MAXV];
  const uint32_t *tt[LP_MAXV];
  const float *rec[LP_MAXV];   // the view's raster records: the stored colour's sign bit is the clamp
  int nv;
};

// one view's contribution of primitive i (a visible primitive: finite geometry).
// EXACT: the no-ray-space moments (per plane: dL/dm, dL/dn) -> camera-space offsets and centre.
template <int KIND, bool EXACT>
__device__ __forceinline__ void view_feature_grad(const lp_prims &P, const lp_camera &cam, float kappa, int i,
                                                  const float *__restrict__ rgrad, float gpos[3], float grot[4],
                                                  float gdist[4], float &gop, float &m2d) {
  constexpr int K = Kind<KIND>::K, RG = Kind<KIND>::RG;
  const int n = P.n;
  // (no early exit on all-zero moments: the items are (primitive, view) pairs with a raster
  // gradient, and without a branch on the moments the feature loads below overlap theirs)
  // the primitive's rgrad row (dsigma, drgb | moments) -> m[moments..., dsigma, drgb]
  float m[RG];
  {
    const float4 *row = reinterpret_cast<const float4 *>(rgrad + (size_t)i * lp_rgs<KIND>());
    float t[4 * ((RG + 3) / 4)];
#pragma unroll
    for (int q = 0; q < (RG + 3) / 4; ++q) {
      const float4 x = row[q];
      t[4 * q] = x.x;
      t[4 * q + 1] = x.y;
      t[4 * q + 2] = x.z;
      t[4 * q + 3] = x.w;
    }
#pragma unroll
    for (int a = 0; a < RG; ++a) m[a] = a < RG - 4 ? t[a + 4] : t[a - (RG - 4)];
  }

  Geom g;
  float dhf[4], qf[4], cf[3];
  canonical_geometry<KIND>(P, i, cam, kappa, g, dhf, qf, cf, EXACT);

  // ---- raster moments -> d/d(ray-space offsets) and d/d(ray-space centre xy)
  double go[4][3] = {{0, 0, 0}, {0, 0, 0}, {0, 0, 0}, {0, 0, 0}};
  double gcr[2] = {0, 0};
  double gpc[3] = {0, 0, 0};   // exact mode: d/d(camera-space centre p)
  double dsig, drgb[3];
  if (EXACT) {
    // planes n . q = m (+-1 for slabs); moments per plane f: (dL/dm, dL/dn.x, dL/dn.y, dL/dn.z)
    if (KIND == OCTA) {
      double M[3][3], G[3][3], det;
#pragma unroll
      for (int a = 0; a < 3; ++a)
#pragma unroll
        for (int j = 0; j < 3; ++j) M[a][j] = (double)g.off[j][a];
      inverse3(M, G, det);
      double gG[3][3] = {{0, 0, 0}, {0, 0, 0}, {0, 0, 0}};
#pragma unroll
      for (int s = 0; s < 4; ++s) {
        double n3[3];
#pragma unroll
        for (int c = 0; c < 3; ++c)
          n3[c] = slab_sign(s, 0) * G[0][c] + slab_sign(s, 1) * G[1][c] + slab_sign(s, 2) * G[2][c];
        const double dm = m[4 * s];
        // centred moments: dL/dn_s (plane moving with p) and dL/dp += dm n_s
        const double dn[3] = {m[4 * s + 1], m[4 * s + 2], m[4 * s + 3]};
#pragma unroll
        for (int a = 0; a < 3; ++a) {
          gpc[a] += dm * n3[a];
          const double sa = slab_sign(s, a);
#pragma unroll
          for (int c = 0; c < 3; ++c) gG[a][c] += sa * dn[c];
        }
      }
      double t1[3][3];
#pragma unroll
      for (int a = 0; a < 3; ++a)
#pragma unroll
        for (int b = 0; b < 3; ++b) t1[a][b] = G[0][a] * gG[0][b] + G[1][a] * gG[1][b] + G[2][a] * gG[2][b];
#pragma unroll
      for (int a = 0; a < 3; ++a)
#pragma unroll
        for (int j = 0; j < 3; ++j) go[j][a] += -(t1[a][0] * G[j][0] + t1[a][1] * G[j][1] + t1[a][2] * G[j][2]);
    } else {
      // faces relative to the centre: n_f . (q - p) = m'_f, m'_f = n_f . oc_a, n_f = (oc_b - oc_a) x (oc_c - oc_a)
      double v[4][3];
#pragma unroll
      for (int k = 0; k < 4; ++k)
#pragma unroll
        for (int a = 0; a < 3; ++a) v[k][a] = (double)g.off[k][a];
#pragma unroll
      for (int f = 0; f < 4; ++f) {
        const double dm = m[4 * f];
        const int ia = tetra_face(f, 0), ib = tetra_face(f, 1), ic = tetra_face(f, 2);
        const double e1[3] = {v[ib][0] - v[ia][0], v[ib][1] - v[ia][1], v[ib][2] - v[ia][2]};
        const double e2[3] = {v[ic][0] - v[ia][0], v[ic][1] - v[ia][1], v[ic][2] - v[ia][2]};
        const double nf[3] = {e1[1] * e2[2] - e1[2] * e2[1], e1[2] * e2[0] - e1[0] * e2[2], e1[0] * e2[1] - e1[1] * e2[0]};
        // centred moments: dL/dn_f at fixed m'_f, plus m'_f = n_f . oc_a
        const double gn[3] = {m[4 * f + 1] + dm * v[ia][0], m[4 * f + 2] + dm * v[ia][1], m[4 * f + 3] + dm * v[ia][2]};
        const double ge1[3] = {e2[1] * gn[2] - e2[2] * gn[1], e2[2] * gn[0] - e2[0] * gn[2], e2[0] * gn[1] - e2[1] * gn[0]};
        const double ge2[3] = {gn[1] * e1[2] - gn[2] * e1[1], gn[2] * e1[0] - gn[0] * e1[2], gn[0] * e1[1] - gn[1] * e1[0]};
#pragma unroll
        for (int a = 0; a < 3; ++a) {
          go[ia][a] += dm * nf[a] - ge1[a] - ge2[a];
          go[ib][a] += ge1[a];
          go[ic][a] += ge2[a];
          gpc[a] += dm * nf[a];      // the plane moves with p
        }
      }
    }
    constexpr int RGK = Kind<KIND>::RG;
    dsig = m[RGK - 4];
    drgb[0] = m[RGK - 3]; drgb[1] = m[RGK - 2]; drgb[2] = m[RGK - 1];
    // densification statistic in pixel units at the centre's depth (reading 26/27)
    gcr[0] = gpc[0] * (double)g.cz / (double)cam.fx;
    gcr[1] = gpc[1] * (double)g.cz / (double)cam.fy;
  } else if (KIND == OCTA) {
    double M[3][3], G[3][3], det;
#pragma unroll
    for (int a = 0; a < 3; ++a)
#pragma unroll
      for (int j = 0; j < 3; ++j) M[a][j] = (double)g.off[j][a];
    inverse3(M, G, det);
    SlabRows S;
    octa_slabs(g.off, S);
    double gG[3][3] = {{0, 0, 0}, {0, 0, 0}, {0, 0, 0}};
#pragma unroll
    for (int s = 0; s < 4; ++s) {
      const double rx = S.r[s][0], ry = S.r[s][1], rz = S.r[s][2];
      const double irz = 1.0 / rz;                       // one fp64 division per slab
      const double b = -rx * irz, gg = -ry * irz;
      const double db = m[4 * s + 0], dg = m[4 * s + 1], mc = m[4 * s + 2], dhh = m[4 * s + 3];
      // L_s = b dx + g dy with dx = px - c.x: d/dc.x = -b (summed weights M_c)
      gcr[0] -= b * mc;
      gcr[1] -= gg * mc;
      // b = -rx/rz, g = -ry/rz, h = 1/|rz|
      const double drx = -db * irz, dry = -dg * irz;
      const double drz = ((db * rx + dg * ry) - dhh * (rz > 0 ? 1.0 : -1.0)) * irz * irz;
#pragma unroll
      for (int a = 0; a < 3; ++a) {
        const double sa = slab_sign(s, a);
        gG[a][0] += sa * drx;
        gG[a][1] += sa * dry;
        gG[a][2] += sa * drz;
      }
    }
    // G = M^-1  =>  dM = -G^T dG G^T
    double t1[3][3];
#pragma unroll
    for (int a = 0; a < 3; ++a)
#pragma unroll
      for (int b = 0; b < 3; ++b) t1[a][b] = G[0][a] * gG[0][b] + G[1][a] * gG[1][b] + G[2][a] * gG[2][b];
#pragma unroll
    for (int a = 0; a < 3; ++a)
#pragma unroll
      for (int j = 0; j < 3; ++j) {
        const double dM = -(t1[a][0] * G[j][0] + t1[a][1] * G[j][1] + t1[a][2] * G[j][2]);
        go[j][a] += dM;   // column j of M is offset j
      }
    dsig = m[16];
    drgb[0] = m[17]; drgb[1] = m[18]; drgb[2] = m[19];
  } else {
    TetraPlanes T;
    tetra_planes(g.off, T);
    double v[4][3];
#pragma unroll
    for (int k = 0; k < 4; ++k)
#pragma unroll
      for (int a = 0; a < 3; ++a) v[k][a] = (double)g.off[k][a];
    // slot moments -> per-face plane gradients (a face may fill several slots)
    double fA[4] = {0, 0, 0, 0}, fB[4] = {0, 0, 0, 0}, fC[4] = {0, 0, 0, 0};
#pragma unroll
    for (int s = 0; s < 6; ++s) {
      const int sf = T.slot_face[s];
#pragma unroll
      for (int f = 0; f < 4; ++f)
        if (f == sf) {
          fA[f] += m[3 * s];
          fB[f] += m[3 * s + 1];
          fC[f] += m[3 * s + 2];
        }
    }
#pragma unroll
    for (int f = 0; f < 4; ++f) {
      const double dA = fA[f], dB = fB[f], dC = fC[f];
      if (dA == 0.0 && dB == 0.0 && dC == 0.0) continue;
      constexpr int dummy = 0;
      (void)dummy;
      const int ia = tetra_face(f, 0), ib = tetra_face(f, 1), ic = tetra_face(f, 2);
      const double B = T.B[f], C = T.C[f];
      gcr[0] -= B * dA;
      gcr[1] -= C * dA;
      // A = va.z - B va.x - C va.y
      go[ia][2] += dA;
      go[ia][0] -= B * dA;
      go[ia][1] -= C * dA;
      const double dBt = dB - dA * v[ia][0], dCt = dC - dA * v[ia][1];
      const double nx = T.n[f][0], ny = T.n[f][1], nz = T.n[f][2];
      const double gn[3] = {-dBt / nz, -dCt / nz, dBt * nx / (nz * nz) + dCt * ny / (nz * nz)};
      const double e1[3] = {v[ib][0] - v[ia][0], v[ib][1] - v[ia][1], v[ib][2] - v[ia][2]};
      const double e2[3] = {v[ic][0] - v[ia][0], v[ic][1] - v[ia][1], v[ic][2] - v[ia][2]};
      // n = e1 x e2:  dL/de1 = e2 x gn,  dL/de2 = gn x e1
      const double ge1[3] = {e2[1] * gn[2] - e2[2] * gn[1], e2[2] * gn[0] - e2[0] * gn[2], e2[0] * gn[1] - e2[1] * gn[0]};
      const double ge2[3] = {gn[1] * e1[2] - gn[2] * e1[1], gn[2] * e1[0] - gn[0] * e1[2], gn[0] * e1[1] - gn[1] * e1[0]};
#pragma unroll
      for (int a = 0; a < 3; ++a) {
        go[ib][a] += ge1[a];
        go[ic][a] += ge2[a];
        go[ia][a] -= ge1[a] + ge2[a];
      }
    }
    dsig = m[18];
    drgb[0] = m[19]; drgb[1] = m[20]; drgb[2] = m[21];
  }
  m2d += (float)sqrt(gcr[0] * gcr[0] + gcr[1] * gcr[1]);

  // ---- the 2D filter adds constants (fixed extreme index): identity.
  using CT = float;   // the chain below is well conditioned: fp32 (the M^-1 / plane part above is fp64)
  // ---- o_j = J W (dh_j R b_j); c_ray = phi(p), p = W c + t  (fp64 chain)
  // (one division per distinct denominator -- |q|, p_z, |p| -- and products with its reciprocal:
  // IEEE divisions were ~a third of K5's instructions; this chain is tolerance-compared, not part
  // of the bit-exact canonical contract)
  CT q[4] = {qf[0], qf[1], qf[2], qf[3]};
  const CT nq = sqrtf(q[0] * q[0] + q[1] * q[1] + q[2] * q[2] + q[3] * q[3]);
  const CT inq = 1.0f / nq;
  const CT w = q[0] * inq, x = q[1] * inq, y = q[2] * inq, z = q[3] * inq;
  const CT R[3][3] = {{1 - 2 * (y * y + z * z), 2 * (x * y - w * z), 2 * (x * z + w * y)},
                          {2 * (x * y + w * z), 1 - 2 * (x * x + z * z), 2 * (y * z - w * x)},
                          {2 * (x * z - w * y), 2 * (y * z + w * x), 1 - 2 * (x * x + y * y)}};
  CT Wm[3][3];
#pragma unroll
  for (int r = 0; r < 3; ++r)
#pragma unroll
    for (int cc = 0; cc < 3; ++cc) Wm[r][cc] = cam.W[3 * r + cc];
  CT p[3];
#pragma unroll
  for (int r = 0; r < 3; ++r) p[r] = Wm[r][0] * cf[0] + Wm[r][1] * cf[1] + Wm[r][2] * cf[2] + (CT)cam.t[r];
  const CT l = sqrtf(p[0] * p[0] + p[1] * p[1] + p[2] * p[2]);
  const CT fx = cam.fx, fy = cam.fy, pz = p[2];
  const CT ipz = 1.0f / pz, ipz2 = ipz * ipz, ipz3 = ipz2 * ipz, il = 1.0f / l, il2 = il * il;
  const CT J[3][3] = {{fx * ipz, 0, -fx * p[0] * ipz2}, {0, fy * ipz, -fy * p[1] * ipz2}, {p[0] * il, p[1] * il, p[2] * il}};
  CT gJ[3][3] = {{0, 0, 0}, {0, 0, 0}, {0, 0, 0}}, gR[3][3] = {{0, 0, 0}, {0, 0, 0}, {0, 0, 0}};
  CT gdh[4] = {0, 0, 0, 0};
  const CT kk = 0.57735026918962576451f;
#pragma unroll
  for (int j = 0; j < K; ++j) {
    CT bj[3];
    if (KIND == OCTA) {
      bj[0] = j == 0; bj[1] = j == 1; bj[2] = j == 2;
    } else {
      bj[0] = (j == 0 || j == 1) ? kk : -kk;
      bj[1] = (j == 0 || j == 2) ? kk : -kk;
      bj[2] = (j == 0 || j == 3) ? kk : -kk;
    }
    CT Rb[3], ow[3], oc[3], goc[3], gow[3];
#pragma unroll
    for (int r = 0; r < 3; ++r) Rb[r] = R[r][0] * bj[0] + R[r][1] * bj[1] + R[r][2] * bj[2];
#pragma unroll
    for (int r = 0; r < 3; ++r) ow[r] = (CT)dhf[j] * Rb[r];
#pragma unroll
    for (int r = 0; r < 3; ++r) oc[r] = Wm[r][0] * ow[0] + Wm[r][1] * ow[1] + Wm[r][2] * ow[2];
    if (EXACT) {
#pragma unroll
      for (int a = 0; a < 3; ++a) goc[a] = (CT)go[j][a];
    } else {
#pragma unroll
      for (int a = 0; a < 3; ++a) goc[a] = J[0][a] * go[j][0] + J[1][a] * go[j][1] + J[2][a] * go[j][2];
#pragma unroll
      for (int r = 0; r < 3; ++r)
#pragma unroll
        for (int a = 0; a < 3; ++a) gJ[r][a] += go[j][r] * oc[a];
    }
#pragma unroll
    for (int a = 0; a < 3; ++a) gow[a] = Wm[0][a] * goc[0] + Wm[1][a] * goc[1] + Wm[2][a] * goc[2];
    gdh[j] = Rb[0] * gow[0] + Rb[1] * gow[1] + Rb[2] * gow[2];
#pragma unroll
    for (int r = 0; r < 3; ++r)
#pragma unroll
      for (int cc = 0; cc < 3; ++cc) gR[r][cc] += (CT)dhf[j] * gow[r] * bj[cc];
  }
  CT gp[3];
  if (EXACT) {
#pragma unroll
    for (int a = 0; a < 3; ++a) gp[a] = (CT)gpc[a];
  } else {
#pragma unroll
  for (int a = 0; a < 3; ++a) gp[a] = J[0][a] * gcr[0] + J[1][a] * gcr[1];   // c_ray.z gets no gradient
  gp[2] += gJ[0][0] * (-fx * ipz2);
  gp[0] += gJ[0][2] * (-fx * ipz2);
  gp[2] += gJ[0][2] * (2.0f * fx * p[0] * ipz3);
  gp[2] += gJ[1][1] * (-fy * ipz2);
  gp[1] += gJ[1][2] * (-fy * ipz2);
  gp[2] += gJ[1][2] * (2.0f * fy * p[1] * ipz3);
#pragma unroll
  for (int k = 0; k < 3; ++k)
#pragma unroll
    for (int mm = 0; mm < 3; ++mm) gp[mm] += gJ[2][k] * (((k == mm) ? 1.0f : 0.0f) - p[k] * p[mm] * il2) * il;
  }
  CT gc[3];
#pragma unroll
  for (int a = 0; a < 3; ++a) gc[a] = Wm[0][a] * gp[0] + Wm[1][a] * gp[1] + Wm[2][a] * gp[2];

  // ---- distances (through the optional 3D filter)
  {
#pragma unroll
    for (int j = 0; j < K; ++j) {
      CT gd = gdh[j];
      if (P.filter3d) gd *= (CT)P.dist[j * n + i] / (CT)dhf[j];
      gdist[j] += (float)gd;
    }
  }
  // ---- rotation: R(q_hat) -> q_hat -> q
  {
    const CT dR[4][3][3] = {
        {{0, -2 * z, 2 * y}, {2 * z, 0, -2 * x}, {-2 * y, 2 * x, 0}},
        {{0, 2 * y, 2 * z}, {2 * y, -4 * x, -2 * w}, {2 * z, 2 * w, -4 * x}},
        {{-4 * y, 2 * x, 2 * w}, {2 * x, 0, 2 * z}, {-2 * w, 2 * z, -4 * y}},
        {{-4 * z, -2 * w, 2 * x}, {2 * w, -4 * z, 2 * y}, {2 * x, 2 * y, 0}}};
    CT gq[4] = {0, 0, 0, 0};
#pragma unroll
    for (int a = 0; a < 4; ++a)
#pragma unroll
      for (int r = 0; r < 3; ++r)
#pragma unroll
        for (int cc = 0; cc < 3; ++cc) gq[a] += gR[r][cc] * dR[a][r][cc];
    const CT qh[4] = {w, x, y, z};
    const CT dot = qh[0] * gq[0] + qh[1] * gq[1] + qh[2] * gq[2] + qh[3] * gq[3];
#pragma unroll
    for (int a = 0; a < 4; ++a) grot[a] += (float)((gq[a] - qh[a] * dot) * inq);
  }
  // ---- opacity: Eq. 1 with the denominator frozen, alpha = sigmoid(logit)
  {
    const CT alpha = 1.0f / (1.0f + expf(-(CT)P.opacity[i]));
    CT md = dhf[0];
#pragma unroll
    for (int a = 1; a < K; ++a) md = fminf(md, (CT)dhf[a]);
    const CT dsda = 0.99f / ((1.0f - 0.99f * alpha) * 2.0f * md);
    gop += (float)(dsig * dsda * alpha * (1.0f - alpha));
  }
  // (SH coefficients and the view-direction term of the centre: sh_view_inputs)
#pragma unroll
  for (int a = 0; a < 3; ++a) gpos[a] += (float)gc[a];
}

// SH inputs of one (primitive, view) item: the clamp-masked colour gradient gr and the view
// direction dir (the SH coefficient gradient Y(dir) gr is expanded later by the primitive's
// owner lane), plus the view-direction term of the centre gradient.
template <int DEG>
__device__ __forceinline__ void sh_view_inputs(const lp_prims &P, const lp_camera &cam, int i,
                                               const float *__restrict__ rgrad, int rg_words,
                                               const float *__restrict__ rec_rgb, float gr[3], float dir[3],
                                               float gpos[3]) {
  constexpr int NC = (DEG + 1) * (DEG + 1);
  const int n = P.n;
  const float c[3] = {P.pos[i], P.pos[n + i], P.pos[2 * n + i]};
#pragma unroll
  for (int ch = 0; ch < 3; ++ch) gr[ch] = rgrad[(size_t)i * rg_words + 1 + ch];   // row: dsigma, drgb | moments
  // the forward's clamp decision, stored by K1 as the colour's sign bit (-0.0: clamped)
#pragma unroll
  for (int ch = 0; ch < 3; ++ch)
    if (signbit(rec_rgb[ch])) gr[ch] = 0.f;
  const float cpx = -(cam.W[0] * cam.t[0] + cam.W[3] * cam.t[1] + cam.W[6] * cam.t[2]);
  const float cpy = -(cam.W[1] * cam.t[0] + cam.W[4] * cam.t[1] + cam.W[7] * cam.t[2]);
  const float cpz = -(cam.W[2] * cam.t[0] + cam.W[5] * cam.t[1] + cam.W[8] * cam.t[2]);
  const float d[3] = {c[0] - cpx, c[1] - cpy, c[2] - cpz};
  const float nv = sqrtf(d[0] * d[0] + d[1] * d[1] + d[2] * d[2]);
  const float inv = 1.0f / nv;
  dir[0] = d[0] * inv;
  dir[1] = d[1] * inv;
  dir[2] = d[2] * inv;
  if constexpr (DEG == 0) return;
  if (gr[0] == 0.f && gr[1] == 0.f && gr[2] == 0.f) return;
  float wk[16];
#pragma unroll
  for (int k = 0; k < 16; ++k) {
    wk[k] = 0.f;
    if (k < NC) {
#pragma unroll
      for (int ch = 0; ch < 3; ++ch) wk[k] = fmaf(gr[ch], P.sh[((size_t)k * 3 + ch) * n + i], wk[k]);
    }
  }
  float gdir[3];
  sh_basis_grad_dot<float>(DEG, dir[0], dir[1], dir[2], wk, gdir);
  const float dd = dir[0] * gdir[0] + dir[1] * gdir[1] + dir[2] * gdir[2];
#pragma unroll
  for (int a = 0; a < 3; ++a) gpos[a] += (gdir[a] - dir[a] * dd) * inv;
}

// per-item result record in shared memory
struct ItemRes {
  static constexpr int POS = 0, ROT = 3, DIST = 7, OP = 11, M2D = 12, GR = 13, DIR = 16;
  static constexpr int N = 19;
};

// K5, one launch for up to LP_MAXV views.  A warp owns 32 consecutive primitives.  Phase A: their
// active (primitive, view) items -- raster gradient present -- are compacted into a warp-local list
// and evaluated 32 at a time (dense SIMT lanes; the per-view geometry chain is the expensive part),
// each writing a 19-float result to shared memory.  Phase B: lane l owns primitive l, sums its
// items (contiguous in the list), expands the SH gradient sum_v Y(dir_v) gr_v in registers, and
// read-modify-writes every feature gradient once.  No shared-memory float atomics (sm_100 has
// none: they compile to CAS loops).
template <int KIND, int DEG, bool EXACT>
// assign: the feature gradients are SET (=) instead of accumulated (+=): every primitive's gradient
// is written (zeros where no view has a raster gradient), no old gradient is read -- the first pack
// of a step whose optimizer consumed (and need not zero) the previous step's gradients.  The
// densification statistics (mean2d_abs, vis_count) accumulate either way.
__global__ void __launch_bounds__(64, LP_K5_MINB) k_preprocess_bwd(lp_prims P, float kappa, ViewPack V, int rg_words,
                                                       lp_grads Gs, bool assign) {
  constexpr int WARPS = 2, K = Kind<KIND>::K, NC = (DEG + 1) * (DEG + 1);
  __shared__ lp_camera s_cam[LP_MAXV];
  __shared__ const float *s_rg[LP_MAXV];
  __shared__ float s_res[WARPS][32 * LP_MAXV][ItemRes::N];
  __shared__ unsigned char s_items[WARPS][32 * LP_MAXV];
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x < V.nv) {
    s_cam[threadIdx.x] = V.cam[threadIdx.x];
    s_rg[threadIdx.x] = V.rgrad[threadIdx.x];
  }
  __syncthreads();
  const int n = P.n;
  const int base = (blockIdx.x * WARPS + w) * 32;
  const int i = base + lane;
  unsigned vm = 0;   // views with a raster gradient for this lane's primitive
  if (i < n) {
    // independent loads for all views first (a dependent chain per view would serialise latency)
    unsigned vis = 0;
#pragma unroll
    for (int v = 0; v < LP_MAXV; ++v)
      if (v < V.nv && V.tt[v][i] != 0) vis |= 1u << v;
    if (Gs.vis_count && vis) Gs.vis_count[i] += (float)__popc(vis);   // densification denominator
    // (gated by vis: K1 zeroes the raster rows of visible primitives only)
    float probe[LP_MAXV];
#pragma unroll
    for (int v = 0; v < LP_MAXV; ++v) {
      probe[v] = 0.f;
      if (v < V.nv && ((vis >> v) & 1u)) {
        const float4 rg = *reinterpret_cast<const float4 *>(V.rgrad[v] + (size_t)i * lp_rgs<KIND>());   // dsigma, drgb
        probe[v] = fabsf(rg.x) + fabsf(rg.y) + fabsf(rg.z) + fabsf(rg.w);
      }
    }
#pragma unroll
    for (int v = 0; v < LP_MAXV; ++v)
      if (probe[v] != 0.f) vm |= 1u << v;
  }
  const int c = __popc(vm);
  int incl = c;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const int y = __shfl_up_sync(0xffffffffu, incl, o);
    if (lane >= o) incl += y;
  }
  const int total = __shfl_sync(0xffffffffu, incl, 31);
  if (total == 0 && !assign) return;   // (assign: the warp's gradients are still written, as zeros)
  const int first = incl - c;   // this lane's items are [first, first + c)
  {
    int slot = first;
    for (unsigned m = vm; m; m &= m - 1) s_items[w][slot++] = (unsigned char)((lane << 3) | (__ffs(m) - 1));
  }
  __syncwarp();
  // ---- phase A: dense evaluation of the items
  for (int r = 0; r < total; r += 32) {
    const int it = r + lane;
    if (it < total) {
      const int item = s_items[w][it];
      const int pl = item >> 3, v = item & 7;
      const int ii = base + pl;
      LP_CHECK(ii < n && v < V.nv && it < 32 * LP_MAXV);
      float gpos[3] = {0.f, 0.f, 0.f}, grot[4] = {0.f, 0.f, 0.f, 0.f}, gdist[4] = {0.f, 0.f, 0.f, 0.f};
      float gop = 0.f, m2d = 0.f, gr[3] = {0.f, 0.f, 0.f}, dir[3] = {0.f, 0.f, 1.f};
      view_feature_grad<KIND, EXACT>(P, s_cam[v], kappa, ii, s_rg[v], gpos, grot, gdist, gop, m2d);
      if (Gs.sh || Gs.pos) {
        constexpr int RGBW = EXACT ? ExactRec<KIND>::RGB : Kind<KIND>::RGB;
        const float *rgb = V.rec[v] + (size_t)ii * Kind<KIND>::RS + RGBW;
        sh_view_inputs<DEG>(P, s_cam[v], ii, s_rg[v], rg_words, rgb, gr, dir, gpos);
      }
      float *res = s_res[w][it];
#pragma unroll
      for (int a = 0; a < 3; ++a) res[ItemRes::POS + a] = gpos[a];
#pragma unroll
      for (int a = 0; a < 4; ++a) res[ItemRes::ROT + a] = grot[a];
#pragma unroll
      for (int a = 0; a < 4; ++a) res[ItemRes::DIST + a] = gdist[a];
      res[ItemRes::OP] = gop;
      res[ItemRes::M2D] = m2d;
#pragma unroll
      for (int a = 0; a < 3; ++a) {
        res[ItemRes::GR + a] = gr[a];
        res[ItemRes::DIR + a] = dir[a];
      }
    }
  }
  __syncwarp();
  if (!vm) {
    if (assign && i < n) {
#pragma unroll
      for (int a = 0; a < 3; ++a)
        if (Gs.pos) Gs.pos[(size_t)a * n + i] = 0.f;
#pragma unroll
      for (int a = 0; a < 4; ++a)
        if (Gs.rot) Gs.rot[(size_t)a * n + i] = 0.f;
#pragma unroll
      for (int a = 0; a < K; ++a)
        if (Gs.dist) Gs.dist[(size_t)a * n + i] = 0.f;
      if (Gs.opacity) Gs.opacity[i] = 0.f;
      if (Gs.sh) {
#pragma unroll
        for (int q = 0; q < 3 * NC; ++q) Gs.sh[(size_t)q * n + i] = 0.f;
      }
    }
    return;
  }
  // ---- phase B: owner lane sums its items and writes its primitive's gradients once
  // the old values of the non-SH feature gradients, loaded up front (independent round trips; the
  // compiler cannot move these loads past the stores below, which may alias)
  float acc[ItemRes::M2D + 1];
#pragma unroll
  for (int a = 0; a < 3; ++a) acc[ItemRes::POS + a] = (Gs.pos && !assign) ? Gs.pos[(size_t)a * n + i] : 0.f;
#pragma unroll
  for (int a = 0; a < 4; ++a) acc[ItemRes::ROT + a] = (Gs.rot && !assign) ? Gs.rot[(size_t)a * n + i] : 0.f;
#pragma unroll
  for (int a = 0; a < 4; ++a)
    acc[ItemRes::DIST + a] = (Gs.dist && a < K && !assign) ? Gs.dist[(size_t)a * n + i] : 0.f;
  acc[ItemRes::OP] = (Gs.opacity && !assign) ? Gs.opacity[i] : 0.f;
  acc[ItemRes::M2D] = Gs.mean2d_abs ? Gs.mean2d_abs[i] : 0.f;
  float sum[ItemRes::M2D + 1];
#pragma unroll
  for (int a = 0; a <= ItemRes::M2D; ++a) sum[a] = 0.f;
  if (Gs.sh && !assign) {   // the SH gradient rows of the warp's primitives: on their way to L1 during the sums
#pragma unroll
    for (int q = 0; q < 3 * NC; ++q) asm volatile("prefetch.global.L1 [%0];" ::"l"(Gs.sh + (size_t)q * n + i));
  }
  float gs[3][NC];
#pragma unroll
  for (int ch = 0; ch < 3; ++ch)
#pragma unroll
    for (int k = 0; k < NC; ++k) gs[ch][k] = 0.f;
  for (int it = first; it < first + c; ++it) {
    const float *res = s_res[w][it];
#pragma unroll
    for (int a = 0; a <= ItemRes::M2D; ++a) sum[a] += res[a];
    const float gr[3] = {res[ItemRes::GR], res[ItemRes::GR + 1], res[ItemRes::GR + 2]};
    if (gr[0] == 0.f && gr[1] == 0.f && gr[2] == 0.f) continue;
    float Y[16];
    sh_basis<float>(DEG, res[ItemRes::DIR], res[ItemRes::DIR + 1], res[ItemRes::DIR + 2], Y);
#pragma unroll
    for (int ch = 0; ch < 3; ++ch)
#pragma unroll
      for (int k = 0; k < NC; ++k) gs[ch][k] = fmaf(Y[k], gr[ch], gs[ch][k]);
  }
  if (Gs.pos) {
#pragma unroll
    for (int a = 0; a < 3; ++a) Gs.pos[(size_t)a * n + i] = acc[ItemRes::POS + a] + sum[ItemRes::POS + a];
  }
  if (Gs.rot) {
#pragma unroll
    for (int a = 0; a < 4; ++a) Gs.rot[(size_t)a * n + i] = acc[ItemRes::ROT + a] + sum[ItemRes::ROT + a];
  }
  if (Gs.dist) {
#pragma unroll
    for (int a = 0; a < K; ++a) Gs.dist[(size_t)a * n + i] = acc[ItemRes::DIST + a] + sum[ItemRes::DIST + a];
  }
  if (Gs.opacity) Gs.opacity[i] = acc[ItemRes::OP] + sum[ItemRes::OP];
  if (Gs.mean2d_abs) Gs.mean2d_abs[i] = acc[ItemRes::M2D] + sum[ItemRes::M2D];
  if (Gs.sh) {
    // all loads first, then the stores (the compiler cannot reorder loads past stores that may alias)
    float old[3 * NC];
#pragma unroll
    for (int q = 0; q < 3 * NC; ++q) old[q] = assign ? 0.f : Gs.sh[(size_t)q * n + i];
#pragma unroll
    for (int k = 0; k < NC; ++k)
#pragma unroll
      for (int ch = 0; ch < 3; ++ch) Gs.sh[((size_t)k * 3 + ch) * n + i] = old[k * 3 + ch] + gs[ch][k];
  }
}

// ---------------------------------------------------------------------------------------------
template <int KIND, bool EXACT>
static void pre_deg(const lp_prims &P, float kappa, const PreViews &V, int grid, cudaStream_t st) {
  switch (P.sh_degree) {
    case 0: k_preprocess<KIND, EXACT, 0><<<grid, 256, 0, st>>>(P, kappa, V); break;
    case 1: k_preprocess<KIND, EXACT, 1><<<grid, 256, 0, st>>>(P, kappa, V); break;
    case 2: k_preprocess<KIND, EXACT, 2><<<grid, 256, 0, st>>>(P, kappa, V); break;
    default: k_preprocess<KIND, EXACT, 3><<<grid, 256, 0, st>>>(P, kappa, V); break;
  }
}

void launch_preprocess(const lp_prims &P, const lp_camera *cams, float kappa, const lp_frame *frames, int n_views,
                       bool exact, cudaStream_t st) {
  if (P.n == 0 || n_views <= 0) return;
  const int grid = (P.n + 255) / 256;
  for (int v0 = 0; v0 < n_views; v0 += LP_PRE_MAXV) {
    PreViews V;
    V.nv = n_views - v0 < LP_PRE_MAXV ? n_views - v0 : LP_PRE_MAXV;
    for (int v = 0; v < LP_PRE_MAXV; ++v) {
      const int s = v0 + (v < V.nv ? v : 0);
      V.cam[v] = cams[s];
      V.frame[v] = frames[s];
    }
    if (P.kind == LP_OCTAHEDRON) {
      if (exact) pre_deg<LP_OCTAHEDRON, true>(P, kappa, V, grid * V.nv, st);
      else pre_deg<LP_OCTAHEDRON, false>(P, kappa, V, grid * V.nv, st);
    } else {
      if (exact) pre_deg<LP_TETRAHEDRON, true>(P, kappa, V, grid * V.nv, st);
      else pre_deg<LP_TETRAHEDRON, false>(P, kappa, V, grid * V.nv, st);
    }
  }
}

template <int KIND, bool EXACT>
static void bwd_deg(const lp_prims &P, float kappa, const ViewPack &V, int rg, const lp_grads &G, bool assign,
                    cudaStream_t st) {
  const int grid = (P.n + 63) / 64;
  switch (P.sh_degree) {
    case 0: k_preprocess_bwd<KIND, 0, EXACT><<<grid, 64, 0, st>>>(P, kappa, V, rg, G, assign); break;
    case 1: k_preprocess_bwd<KIND, 1, EXACT><<<grid, 64, 0, st>>>(P, kappa, V, rg, G, assign); break;
    case 2: k_preprocess_bwd<KIND, 2, EXACT><<<grid, 64, 0, st>>>(P, kappa, V, rg, G, assign); break;
    default: k_preprocess_bwd<KIND, 3, EXACT><<<grid, 64, 0, st>>>(P, kappa, V, rg, G, assign); break;
  }
}

void launch_preprocess_bwd(const lp_prims &P, const lp_camera *cams, float kappa, const lp_frame *frames, int n_views,
                           const lp_grads &G, bool exact, bool assign, cudaStream_t st) {
  if (P.n == 0 || n_views <= 0) return;
  // deterministic frames: the raster moments from the (entry, warp) partials, in a fixed order
  for (int v = 0; v < n_views; ++v) launch_det_gather(frames[v], st);
  for (int v0 = 0; v0 < n_views; v0 += LP_MAXV) {
    ViewPack V;
    V.nv = n_views - v0 < LP_MAXV ? n_views - v0 : LP_MAXV;
    for (int v = 0; v < LP_MAXV; ++v) {
      const int s = v0 + (v < V.nv ? v : 0);
      V.cam[v] = cams[s];
      V.rgrad[v] = frames[s].rgrad;
      V.tt[v] = frames[s].tiles_touched;
      V.rec[v] = frames[s].record;
    }
    const int rg = frames[v0].rgrad_words;
    if (P.kind == LP_OCTAHEDRON) {
      if (exact) bwd_deg<LP_OCTAHEDRON, true>(P, kappa, V, rg, G, assign && v0 == 0, st);
      else bwd_deg<LP_OCTAHEDRON, false>(P, kappa, V, rg, G, assign && v0 == 0, st);
    } else {
      if (exact) bwd_deg<LP_TETRAHEDRON, true>(P, kappa, V, rg, G, assign && v0 == 0, st);
      else bwd_deg<LP_TETRAHEDRON, false>(P, kappa, V, rg, G, assign && v0 == 0, st);
    }
  }
}

}  // namespace lp
