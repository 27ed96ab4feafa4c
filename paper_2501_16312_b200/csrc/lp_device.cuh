// lp_device.cuh -- device-side building blocks shared by the liblinprim kernels (sm_100a).
//
//   * canonical_geometry<KIND>: the integer-producing preprocess geometry in the canonical fp32
//     op order of DESIGN.md §3 (one __f*_rn intrinsic per operation: no FMA contraction).
//   * build_record<KIND>: the raster record (slab form for octahedra, plane form for
//     tetrahedra) computed in fp64 from the canonical offsets, stored fp32.
//   * chord<KIND>: per-pixel entry/exit/chord from a record; the SAME function (bitwise) is used
//     by the forward and the backward raster so transmittance recovery is exact.
//
// P:n = PAPER.md line n.  This header is product code: it shares nothing with
// oracle/ (the CPU oracle implements the same paper independently).
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include "../../include/linprim.h"
#include "lp_x2.cuh"

#include "lp_check.cuh"

namespace lp {

constexpr int OCTA = LP_OCTAHEDRON;
constexpr int TETRA = LP_TETRAHEDRON;

template <int KIND> struct Kind;
// Raster records (fp32, 16-byte aligned, gathered per tile-list entry).  The first float4 is
// always the screen bounding box as (centre x, centre y, half width, half height): a pixel
// outside it cannot intersect the primitive (convexity), so the raster rejects the pair with
// ~6 instructions before the slab / plane evaluation.
//   octahedron (20 words): bx=cx by=cy hx hy | (b g h) x 4 slabs | sigma r g b
//   tetrahedron (28 words): bx by hx hy | cx cy | (A B C) x 6 slots | sigma r g b
// raster-gradient scratch row stride (floats): rgrad is [n][lp_rgs], one row per primitive laid out
// as the backward's shared-memory row: dsigma, drgb (3), then the RG - 4 plane moments, then padding.
// A (warp, primitive) reduction's <= 22 RED.F32 then land in 3 consecutive 32-byte sectors
// instead of one sector per moment.
template <int KIND> __host__ __device__ constexpr int lp_rgs() { return KIND == LP_OCTAHEDRON ? 20 : 24; }   // 80 B / 96 B rows
template <> struct Kind<LP_OCTAHEDRON> {
  static constexpr int K = 3;          // offset vectors (vertices are c +- o_j)
  static constexpr int RW = 20;        // record words (ray space)
  static constexpr int RS = 24;        // record stride in words (room for the exact-mode record)
  static constexpr int RG = 20;        // raster-gradient words: (Mb Mg Mc Mh)x4 dsigma drgb
  static constexpr int CX = 0, SLAB = 4, SIGMA = 16, RGB = 17;
};
template <> struct Kind<LP_TETRAHEDRON> {
  static constexpr int K = 4;          // vertices c + o_k
  static constexpr int RW = 28;        // record words (ray space)
  static constexpr int RS = 28;        // record stride in words
  static constexpr int RG = 22;        // (MA MB MC)x6 slots dsigma drgb
  static constexpr int CX = 4, SLAB = 6, SIGMA = 24, RGB = 25;
};

// Exact-mode ("no ray space", App. D) records, camera space.  For the pixel ray q = t r,
// r = ((x+0.5-cx)/fx, (y+0.5-cy)/fy, 1), k = n . r, and with the centre p the planes are
// evaluated relative to it: t = p_z + tau, tau = (c + n . d) / k, d = p - p_z r = (p_x - p_z r_x,
// p_y - p_z r_y, 0) (small: no cancellation between two depths ~ p_z in the chord):
//   octahedron (24 words): bbox(4) | 4 slabs x n_s(3) | p(3) | sigma | rgb | pad
//     slab s = {q : |n_s . (q - p)| <= 1}, n_s = s^T M^-1 of the camera-space offsets: c = -+1
//   tetrahedron (28 words): bbox(4) | 4 faces x (n_f, m'_f) | p(3) | sigma | rgb | pad
//     face f = {q : n_f . (q - p) <= m'_f} (outward n_f, m'_f = n_f . oc_a): c = m'_f, entering
//     when k < 0
//   chord = (min exit - max entry) |r|, no intersection unless the entry is in front (t > 0).
// The backward accumulates the plane moments relative to p (dL/dn = -sum dL/dt (q - p)/k).
template <int KIND> struct ExactRec;
template <> struct ExactRec<LP_OCTAHEDRON> {
  static constexpr int W = 24, N = 4, P = 16, SIGMA = 19, RGB = 20;
};
template <> struct ExactRec<LP_TETRAHEDRON> {
  static constexpr int W = 28, N = 4, P = 20, SIGMA = 23, RGB = 24;
};

__device__ __forceinline__ float fm(float a, float b) { return __fmul_rn(a, b); }
__device__ __forceinline__ float fa(float a, float b) { return __fadd_rn(a, b); }
__device__ __forceinline__ float fs(float a, float b) { return __fsub_rn(a, b); }
__device__ __forceinline__ float fdv(float a, float b) { return __fdiv_rn(a, b); }
__device__ __forceinline__ float fq(float a) { return __fsqrt_rn(a); }

// fp32(1/sqrt(3)) = 0x3F13CD3A (tetrahedron basis b_k = (+-1,+-1,+-1)/sqrt(3))
__device__ __forceinline__ float tetra_k() { return __uint_as_float(0x3F13CD3Au); }

struct Geom {
  int flag;                  // 0 in frustum, 1 invalid input, 2 culled by znear
  float crx, cry, l;         // ray-space centre (l = |p|, the depth key source); exact: p_x, p_y
  float cz;                  // exact mode: camera-space p_z
  float blo[2], bhi[2];      // exact mode: screen bbox of the projected vertices
  float off[4][3];           // post-filter ray-space offsets; exact mode: camera-space offsets
  uint32_t tiles;            // tiles_touched
  int rect[4];               // tx0 ty0 tx1 ty1
};

// Canonical fp32 geometry.  Also returns the fp32 inputs used downstream.
// exact: the "no ray space" variant (App. D, reading 27): camera-space
// offsets, tile bbox from the perspective projections of the vertices, no 2D filter.
__device__ __forceinline__ void rect_from_bbox(const lp_camera &cam, const float lo_[2], const float hi_[2], Geom &g);

template <int KIND>
__device__ __forceinline__ void canonical_geometry(const lp_prims &P, int i, const lp_camera &cam, float kappa,
                                                   Geom &g, float dh[4], float q_out[4], float c_out[3],
                                                   bool exact = false) {
  constexpr int K = Kind<KIND>::K;
  const int n = P.n;
  g.flag = 0;
  g.tiles = 0;
  g.rect[0] = g.rect[1] = g.rect[2] = g.rect[3] = 0;
  g.crx = g.cry = g.l = g.cz = 0.f;
  float c[3], q[4], d[4], op = P.opacity[i];
#pragma unroll
  for (int a = 0; a < 3; ++a) c[a] = P.pos[a * n + i];
#pragma unroll
  for (int a = 0; a < 4; ++a) q[a] = P.rot[a * n + i];
#pragma unroll
  for (int a = 0; a < K; ++a) d[a] = P.dist[a * n + i];
  bool fin = isfinite(c[0]) && isfinite(c[1]) && isfinite(c[2]) && isfinite(q[0]) && isfinite(q[1]) &&
             isfinite(q[2]) && isfinite(q[3]) && isfinite(op);
  bool pos_d = true;
#pragma unroll
  for (int a = 0; a < K; ++a) {
    fin = fin && isfinite(d[a]);
    pos_d = pos_d && (d[a] > 0.f);
  }
  float f3 = 0.f;
  if (P.filter3d) {
    f3 = P.filter3d[i];
    fin = fin && isfinite(f3);
  }
#pragma unroll
  for (int a = 0; a < 3; ++a) c_out[a] = c[a];
#pragma unroll
  for (int a = 0; a < 4; ++a) q_out[a] = q[a];
  if (!fin || !pos_d) { g.flag = 1; return; }
#pragma unroll
  for (int a = 0; a < K; ++a) dh[a] = P.filter3d ? fq(fa(fm(d[a], d[a]), fm(f3, f3))) : d[a];

  // quaternion -> R (3DGS w-first formula), canonical order
  const float n2 = fa(fa(fa(fm(q[0], q[0]), fm(q[1], q[1])), fm(q[2], q[2])), fm(q[3], q[3]));
  if (n2 == 0.f) { g.flag = 1; return; }
  const float nq = fq(n2);
  const float w = fdv(q[0], nq), x = fdv(q[1], nq), y = fdv(q[2], nq), z = fdv(q[3], nq);
  const float xx = fm(x, x), yy = fm(y, y), zz = fm(z, z);
  const float xy = fm(x, y), xz = fm(x, z), yz = fm(y, z), wx = fm(w, x), wy = fm(w, y), wz = fm(w, z);
  float R[3][3];
  R[0][0] = fs(1.f, fm(2.f, fa(yy, zz)));
  R[0][1] = fm(2.f, fs(xy, wz));
  R[0][2] = fm(2.f, fa(xz, wy));
  R[1][0] = fm(2.f, fa(xy, wz));
  R[1][1] = fs(1.f, fm(2.f, fa(xx, zz)));
  R[1][2] = fm(2.f, fs(yz, wx));
  R[2][0] = fm(2.f, fs(xz, wy));
  R[2][1] = fm(2.f, fa(yz, wx));
  R[2][2] = fs(1.f, fm(2.f, fa(xx, yy)));

  // view transform
  float p[3];
#pragma unroll
  for (int r = 0; r < 3; ++r)
    p[r] = fa(fa(fa(fm(cam.W[3 * r + 0], c[0]), fm(cam.W[3 * r + 1], c[1])), fm(cam.W[3 * r + 2], c[2])), cam.t[r]);
  if (!(p[2] > cam.znear)) { g.flag = 2; return; }

  // EWA ray space
  const float l = fq(fa(fa(fm(p[0], p[0]), fm(p[1], p[1])), fm(p[2], p[2])));
  g.l = l;
  g.crx = fa(fm(cam.fx, fdv(p[0], p[2])), cam.cx);
  g.cry = fa(fm(cam.fy, fdv(p[1], p[2])), cam.cy);
  const float pz2 = fm(p[2], p[2]);
  const float J00 = fdv(cam.fx, p[2]);
  const float J02 = -fdv(fm(cam.fx, p[0]), pz2);
  const float J11 = fdv(cam.fy, p[2]);
  const float J12 = -fdv(fm(cam.fy, p[1]), pz2);
  const float J20 = fdv(p[0], l), J21 = fdv(p[1], l), J22 = fdv(p[2], l);

  // world offsets -> camera -> ray space
#pragma unroll
  for (int j = 0; j < K; ++j) {
    float ow[3];
    if (KIND == OCTA) {
#pragma unroll
      for (int r = 0; r < 3; ++r) ow[r] = fm(dh[j], R[r][j]);
    } else {
      const float k = tetra_k();
      const float b0 = (j == 0 || j == 1) ? k : -k;
      const float b1 = (j == 0 || j == 2) ? k : -k;
      const float b2 = (j == 0 || j == 3) ? k : -k;
#pragma unroll
      for (int r = 0; r < 3; ++r) ow[r] = fm(dh[j], fa(fa(fm(R[r][0], b0), fm(R[r][1], b1)), fm(R[r][2], b2)));
    }
    float oc[3];
#pragma unroll
    for (int r = 0; r < 3; ++r)
      oc[r] = fa(fa(fm(cam.W[3 * r + 0], ow[0]), fm(cam.W[3 * r + 1], ow[1])), fm(cam.W[3 * r + 2], ow[2]));
    if (exact) {
      g.off[j][0] = oc[0];
      g.off[j][1] = oc[1];
      g.off[j][2] = oc[2];
    } else {
      g.off[j][0] = fa(fm(J00, oc[0]), fm(J02, oc[2]));
      g.off[j][1] = fa(fm(J11, oc[1]), fm(J12, oc[2]));
      g.off[j][2] = fa(fa(fm(J20, oc[0]), fm(J21, oc[1])), fm(J22, oc[2]));
    }
  }
  if (exact) {
    // camera space; bbox of the perspective projections of the vertices (whole screen if a vertex
    // is at or behind the camera plane)
    g.crx = p[0];
    g.cry = p[1];
    g.cz = p[2];
    constexpr int NV = KIND == OCTA ? 6 : 4;
    float lo[2] = {0.f, 0.f}, hi[2] = {0.f, 0.f};
    bool behind = false;
#pragma unroll
    for (int v = 0; v < NV; ++v) {
      float q[3];
#pragma unroll
      for (int r = 0; r < 3; ++r) {
        const float o = KIND == OCTA ? g.off[v >> 1][r] : g.off[v][r];
        q[r] = (KIND == OCTA && (v & 1)) ? fs(p[r], o) : fa(p[r], o);
      }
      behind = behind || !(q[2] > 0.f);
      const float u = fa(fm(cam.fx, fdv(q[0], q[2])), cam.cx);
      const float w = fa(fm(cam.fy, fdv(q[1], q[2])), cam.cy);
      lo[0] = v == 0 ? u : fminf(lo[0], u);
      hi[0] = v == 0 ? u : fmaxf(hi[0], u);
      lo[1] = v == 0 ? w : fminf(lo[1], w);
      hi[1] = v == 0 ? w : fmaxf(hi[1], w);
    }
    if (behind) {
      lo[0] = lo[1] = -2.f;
      hi[0] = (float)(cam.width + 2);
      hi[1] = (float)(cam.height + 2);
    }
    g.blo[0] = lo[0];
    g.blo[1] = lo[1];
    g.bhi[0] = hi[0];
    g.bhi[1] = hi[1];
    rect_from_bbox(cam, lo, hi, g);
    return;
  }

  // 2D anti-aliasing filter (readings 19-20)
  const float h = fm(0.5f, kappa);
#pragma unroll
  for (int ax = 0; ax < 2; ++ax) {
    if (KIND == OCTA) {
      // first argmax of |o_j| (value tracked in a register: no dynamic array indexing)
      int jm = 0;
      float am = fabsf(g.off[0][ax]), v = g.off[0][ax];
#pragma unroll
      for (int j = 1; j < 3; ++j)
        if (fabsf(g.off[j][ax]) > am) { am = fabsf(g.off[j][ax]); v = g.off[j][ax]; jm = j; }
      const float nv = fa(v, v >= 0.f ? h : -h);
#pragma unroll
      for (int j = 0; j < 3; ++j)
        if (j == jm) g.off[j][ax] = nv;
    } else {
      int kmin = 0, kmax = 0;
      float vmin = g.off[0][ax], vmax = g.off[0][ax];
#pragma unroll
      for (int k = 1; k < 4; ++k) {
        if (g.off[k][ax] < vmin) { vmin = g.off[k][ax]; kmin = k; }
        if (g.off[k][ax] > vmax) { vmax = g.off[k][ax]; kmax = k; }
      }
#pragma unroll
      for (int k = 0; k < 4; ++k)
        if (k == kmin) g.off[k][ax] = fs(g.off[k][ax], h);
#pragma unroll
      for (int k = 0; k < 4; ++k)
        if (k == kmax) g.off[k][ax] = fa(g.off[k][ax], h);
    }
  }

  // bbox -> pixel rect -> tile rect
  const float cr[2] = {g.crx, g.cry};
  float lo[2], hi[2];
#pragma unroll
  for (int ax = 0; ax < 2; ++ax) {
    if (KIND == OCTA) {
      float m = fabsf(g.off[0][ax]);
#pragma unroll
      for (int j = 1; j < 3; ++j) m = fabsf(g.off[j][ax]) > m ? fabsf(g.off[j][ax]) : m;
      lo[ax] = fs(cr[ax], m);
      hi[ax] = fa(cr[ax], m);
    } else {
      float mn = g.off[0][ax], mx = g.off[0][ax];
#pragma unroll
      for (int k = 1; k < 4; ++k) {
        mn = g.off[k][ax] < mn ? g.off[k][ax] : mn;
        mx = g.off[k][ax] > mx ? g.off[k][ax] : mx;
      }
      lo[ax] = fa(cr[ax], mn);
      hi[ax] = fa(cr[ax], mx);
    }
  }
  rect_from_bbox(cam, lo, hi, g);
}

// screen bbox -> clamped pixel rect -> tile rect; canonical fp32
__device__ __forceinline__ void rect_from_bbox(const lp_camera &cam, const float lo_[2], const float hi_[2], Geom &g) {
  const int dims[2] = {cam.width, cam.height};
  int pmin[2], pmax[2];
#pragma unroll
  for (int ax = 0; ax < 2; ++ax) {
    float a = fs(lo_[ax], 0.5f), b = fs(hi_[ax], 0.5f);
    const float top = (float)(dims[ax] + 2);
    a = a < -2.f ? -2.f : (a > top ? top : a);
    b = b < -2.f ? -2.f : (b > top ? top : b);
    const int i0 = (int)ceilf(a), i1 = (int)floorf(b);
    pmin[ax] = i0 < 0 ? 0 : i0;
    pmax[ax] = i1 > dims[ax] - 1 ? dims[ax] - 1 : i1;
  }
  if (pmin[0] > pmax[0] || pmin[1] > pmax[1]) return;
  g.rect[0] = pmin[0] >> 4;
  g.rect[1] = pmin[1] >> 4;
  g.rect[2] = pmax[0] >> 4;
  g.rect[3] = pmax[1] >> 4;
  g.tiles = (uint32_t)((g.rect[2] - g.rect[0] + 1) * (g.rect[3] - g.rect[1] + 1));
}

// ---------------------------------------------------------------------------------------------
// raster records
// ---------------------------------------------------------------------------------------------
// Octahedron = {c + M lam : |lam|_1 <= 1}, M = [o0 o1 o2] (post-filter ray-space offsets).
// |lam|_1 <= 1  <=>  |s . G (x - c)| <= 1 for the 4 sign vectors s (up to sign), G = M^-1.
// For the vertical pixel ray x = (r, c_z + t):  t in [L_s - h_s, L_s + h_s] with
// L_s = b_s dx + g_s dy,  b = -row.x/row.z,  g = -row.y/row.z,  h = 1/|row.z|,  row = s^T G.
// entry = max_s (L_s - h_s), exit = min_s (L_s + h_s)   (equals MTIA's i2 - i1).
// Compile-time tables (functions of unrolled loop constants fold to immediates: no local memory).
__host__ __device__ __forceinline__ constexpr int slab_sign(int s, int a) {   // (1,1,1) (1,1,-1) (1,-1,1) (-1,1,1)
  return (s == 0) ? 1 : (s == 1 ? (a == 2 ? -1 : 1) : (s == 2 ? (a == 1 ? -1 : 1) : (a == 0 ? -1 : 1)));
}
// Tetrahedron faces (1,3,2) (0,2,3) (0,3,1) (0,1,2), outward for the S:102 basis (DESIGN.md conventions).
__host__ __device__ __forceinline__ constexpr int tetra_face(int f, int c) {
  return f == 0 ? (c == 0 ? 1 : (c == 1 ? 3 : 2))
                : (f == 1 ? (c == 0 ? 0 : (c == 1 ? 2 : 3)) : (f == 2 ? (c == 0 ? 0 : (c == 1 ? 3 : 1)) : c));
}

__device__ __forceinline__ void inverse3(const double M[3][3], double G[3][3], double &det) {
  const double a00 = M[1][1] * M[2][2] - M[1][2] * M[2][1];
  const double a01 = M[0][2] * M[2][1] - M[0][1] * M[2][2];
  const double a02 = M[0][1] * M[1][2] - M[0][2] * M[1][1];
  const double a10 = M[1][2] * M[2][0] - M[1][0] * M[2][2];
  const double a11 = M[0][0] * M[2][2] - M[0][2] * M[2][0];
  const double a12 = M[0][2] * M[1][0] - M[0][0] * M[1][2];
  const double a20 = M[1][0] * M[2][1] - M[1][1] * M[2][0];
  const double a21 = M[0][1] * M[2][0] - M[0][0] * M[2][1];
  const double a22 = M[0][0] * M[1][1] - M[0][1] * M[1][0];
  det = M[0][0] * a00 + M[0][1] * a10 + M[0][2] * a20;
  const double id = 1.0 / det;
  G[0][0] = a00 * id; G[0][1] = a01 * id; G[0][2] = a02 * id;
  G[1][0] = a10 * id; G[1][1] = a11 * id; G[1][2] = a12 * id;
  G[2][0] = a20 * id; G[2][1] = a21 * id; G[2][2] = a22 * id;
}

// clamp a near-zero depth coefficient away from 0 (vertical face / slab seen edge-on): the
// slab/plane then acts as the lateral constraint in the limit
__device__ __forceinline__ double clamp_away(double qz, double lateral) {
  const double lim = 1e-25 * lateral + 1e-300;
  if (fabs(qz) < lim) return qz < 0.0 ? -lim : lim;
  return qz;
}

struct SlabRows {     // octahedron: rows r_s = s^T G (fp64) and the clamped row.z
  double r[4][3];
  bool ok;
};

__device__ __forceinline__ void octa_slabs(const float off[4][3], SlabRows &S) {
  double M[3][3], G[3][3], det;
#pragma unroll
  for (int a = 0; a < 3; ++a)
#pragma unroll
    for (int j = 0; j < 3; ++j) M[a][j] = (double)off[j][a];   // columns are the offsets
  inverse3(M, G, det);
  S.ok = isfinite(det) && det != 0.0;
#pragma unroll
  for (int s = 0; s < 4; ++s) {
#pragma unroll
    for (int c = 0; c < 3; ++c)
      S.r[s][c] = slab_sign(s, 0) * G[0][c] + slab_sign(s, 1) * G[1][c] + slab_sign(s, 2) * G[2][c];
    S.r[s][2] = clamp_away(S.r[s][2], fmax(fabs(S.r[s][0]), fabs(S.r[s][1])));
  }
}

// a[i] for a runtime index via unrolled selects (keeps small arrays in registers)
template <typename T, int N>
__device__ __forceinline__ T sel(const T (&a)[N], int i) {
  T r = a[0];
#pragma unroll
  for (int k = 1; k < N; ++k)
    if (i == k) r = a[k];
  return r;
}

struct TetraPlanes {  // plane of each face: z = A + B dx + C dy relative to the centre
  double n[4][3];     // face normals (outward, n.z clamped away from 0)
  double A[4], B[4], C[4];
  int slot_face[6];   // slots 0..2 front (entry), 3..5 back (exit)
  bool ok;
};

__device__ __forceinline__ void tetra_planes(const float off[4][3], TetraPlanes &T) {
  double v[4][3];
#pragma unroll
  for (int k = 0; k < 4; ++k)
#pragma unroll
    for (int a = 0; a < 3; ++a) v[k][a] = (double)off[k][a];
  int front = 0;
  T.ok = true;
#pragma unroll
  for (int f = 0; f < 4; ++f) {
    const double *pa = v[tetra_face(f, 0)], *pb = v[tetra_face(f, 1)], *pc = v[tetra_face(f, 2)];
    const double e1[3] = {pb[0] - pa[0], pb[1] - pa[1], pb[2] - pa[2]};
    const double e2[3] = {pc[0] - pa[0], pc[1] - pa[1], pc[2] - pa[2]};
    double nx = e1[1] * e2[2] - e1[2] * e2[1];
    double ny = e1[2] * e2[0] - e1[0] * e2[2];
    double nz = e1[0] * e2[1] - e1[1] * e2[0];
    if (nx == 0.0 && ny == 0.0 && nz == 0.0) T.ok = false;
    nz = clamp_away(nz, fmax(fabs(nx), fabs(ny)));
    T.n[f][0] = nx; T.n[f][1] = ny; T.n[f][2] = nz;
    T.B[f] = -nx / nz;
    T.C[f] = -ny / nz;
    T.A[f] = pa[2] - T.B[f] * pa[0] - T.C[f] * pa[1];
    if (nz < 0.0) front |= 1 << f;   // outward normal towards the camera = entry face
  }
  const int nf = __popc(front), nb = 4 - nf;
  if (nf == 0 || nb == 0) T.ok = false;
  // slot s (0..2) = the min(s, nf-1)-th front face; slot 3+s = the min(s, nb-1)-th back face
#pragma unroll
  for (int s = 0; s < 3; ++s) {
    int sf = 0, sb = 0;
    const int rf = s < nf ? s : nf - 1, rb = s < nb ? s : nb - 1;
#pragma unroll
    for (int f = 0; f < 4; ++f) {
      const bool isf = (front >> f) & 1;
      const int rank_f = __popc(front & ((1 << f) - 1));
      const int rank_b = f - rank_f;
      if (isf && rank_f == rf) sf = f;
      if (!isf && rank_b == rb) sb = f;
    }
    T.slot_face[s] = sf;
    T.slot_face[3 + s] = sb;
  }
}

// ---------------------------------------------------------------------------------------------
// chord evaluation (a8).  TRACK: also return the entry / exit slab (octa) or slot (tetra).
// ---------------------------------------------------------------------------------------------
// dx, dy: pixel centre minus the ray-space centre c_r (record word CX, CX+1), fs()-computed.
// Slab value L_s = fma(g_s, dy, b_s dx), plane depth z_s = fma(C_s, dy, fma(B_s, dx, A_s)): the
// dx part first, so the two pixels of a thread (same column, PPT 2) share it and the paired
// forward (chord2 below, FFMA2 / FADD2 lanes) is bitwise this scalar evaluation.
template <bool TRACK>
__device__ __forceinline__ float octa_chord(const float *rec, float dx, float dy, int &se, int &sx) {
  constexpr int B = Kind<LP_OCTAHEDRON>::SLAB;
  float L = __fmaf_rn(rec[B + 1], dy, fm(rec[B], dx));
  float en = fs(L, rec[B + 2]), ex = fa(L, rec[B + 2]);
  if (TRACK) { se = 0; sx = 0; }
#pragma unroll
  for (int s = 1; s < 4; ++s) {
    L = __fmaf_rn(rec[B + 1 + 3 * s], dy, fm(rec[B + 3 * s], dx));
    const float a = fs(L, rec[B + 2 + 3 * s]), b = fa(L, rec[B + 2 + 3 * s]);
    if (TRACK) {
      if (a > en) se = s;
      if (b < ex) sx = s;
    }
    en = fmaxf(en, a);
    ex = fminf(ex, b);
  }
  return fs(ex, en);
}

template <bool TRACK>
__device__ __forceinline__ float tetra_chord(const float *rec, float dx, float dy, int &se, int &sx) {
  constexpr int B = Kind<LP_TETRAHEDRON>::SLAB;
  float z[6];
#pragma unroll
  for (int s = 0; s < 6; ++s) z[s] = __fmaf_rn(rec[B + 2 + 3 * s], dy, __fmaf_rn(rec[B + 1 + 3 * s], dx, rec[B + 3 * s]));
  float en = z[0], ex = z[3];
  if (TRACK) { se = 0; sx = 3; }
#pragma unroll
  for (int s = 1; s < 3; ++s) {
    if (TRACK) {
      if (z[s] > en) se = s;
      if (z[3 + s] < ex) sx = 3 + s;
    }
    en = fmaxf(en, z[s]);
    ex = fminf(ex, z[3 + s]);
  }
  return fs(ex, en);
}

template <int KIND, bool TRACK>
__device__ __forceinline__ float chord(const float *rec, float dx, float dy, int &se, int &sx) {
  if (KIND == LP_OCTAHEDRON) return octa_chord<TRACK>(rec, dx, dy, se, sx);
  return tetra_chord<TRACK>(rec, dx, dy, se, sx);
}

// Paired entry / exit values of the thread's two pixels (same dx, dy2 = their two dy): lane k of
// en[s] / ex[s] is bitwise the scalar chord's value for slab s (octahedron: L - h, L + h) or for the
// front / back plane slot s (tetrahedron: z_s, z_{3+s}).
template <int KIND> struct Planes2 {
  static constexpr int N = KIND == LP_OCTAHEDRON ? 4 : 3;
  float2 en[N], ex[N];
};

template <int KIND>
__device__ __forceinline__ void planes2(const float *rec, float dx, float2 dy2, Planes2<KIND> &P) {
  if (KIND == LP_OCTAHEDRON) {
    constexpr int B = Kind<LP_OCTAHEDRON>::SLAB;
#pragma unroll
    for (int s = 0; s < 4; ++s) {
      const float2 L = ffma2(bc(rec[B + 1 + 3 * s]), dy2, bc(fm(rec[B + 3 * s], dx)));
      P.en[s] = fsub2(L, bc(rec[B + 2 + 3 * s]));
      P.ex[s] = fadd2(L, bc(rec[B + 2 + 3 * s]));
    }
  } else {
    constexpr int B = Kind<LP_TETRAHEDRON>::SLAB;
#pragma unroll
    for (int s = 0; s < 3; ++s) {
      P.en[s] = ffma2(bc(rec[B + 2 + 3 * s]), dy2, bc(__fmaf_rn(rec[B + 1 + 3 * s], dx, rec[B + 3 * s])));
      const int t = s + 3;
      P.ex[s] = ffma2(bc(rec[B + 2 + 3 * t]), dy2, bc(__fmaf_rn(rec[B + 1 + 3 * t], dx, rec[B + 3 * t])));
    }
  }
}

__device__ __forceinline__ float lane_k(float2 v, int k) { return k == 0 ? v.x : v.y; }

// max entry / min exit per pixel (FMNMX3 chains); chord = exit - entry as one FADD2
template <int KIND>
__device__ __forceinline__ float2 chord2_of(const Planes2<KIND> &P, float2 &en2, float2 &ex2) {
  constexpr int N = Planes2<KIND>::N;
  en2 = P.en[0];
  ex2 = P.ex[0];
#pragma unroll
  for (int s = 1; s < N; ++s) {
    en2.x = fmaxf(en2.x, P.en[s].x);
    en2.y = fmaxf(en2.y, P.en[s].y);
    ex2.x = fminf(ex2.x, P.ex[s].x);
    ex2.y = fminf(ex2.y, P.ex[s].y);
  }
  return fsub2(ex2, en2);
}

// Paired chord (forward): lane k is bitwise chord<KIND, false>(rec, dx, dy2[k]); en2 receives the
// entry offsets (depth mode).
template <int KIND>
__device__ __forceinline__ float2 chord2(const float *rec, float dx, float2 dy2, float2 &en2) {
  Planes2<KIND> P;
  planes2<KIND>(rec, dx, dy2, P);
  float2 ex2;
  return chord2_of<KIND>(P, en2, ex2);
}

// Entry / exit slab (octa) or slot (tetra: exit slots 3..5) of pixel k: the FIRST index attaining
// the max entry / min exit, the same choice chord<KIND, true> makes while scanning.
template <int KIND>
__device__ __forceinline__ void track_k(const Planes2<KIND> &P, int k, float en, float ex, int &se, int &sx) {
  constexpr int N = Planes2<KIND>::N;
  se = N - 1;
  sx = N - 1;
#pragma unroll
  for (int s = N - 2; s >= 0; --s) {
    if (lane_k(P.en[s], k) == en) se = s;
    if (lane_k(P.ex[s], k) == ex) sx = s;
  }
  if (KIND == LP_TETRAHEDRON) sx += 3;
}

// ---------------------------------------------------------------------------------------------
// exact mode (App. D): paired per-plane entry / exit parameters of the thread's two pixels
// (same r.x, ry2 = their two r.y); lane k of en[f] / ex[f] is this plane's entry / exit t.
// ---------------------------------------------------------------------------------------------
struct PlanesE2 {
  float2 en[4], ex[4];
};

__device__ __forceinline__ float rcp_approx(float x) {
  float y;
  asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));   // rcp(+-0) = +-inf: a plane parallel to the ray
  return y;
}

// plane normal of plane f in an exact record, and (tetra) its offset m_f
template <int KIND>
__device__ __forceinline__ const float *plane_n(const float *rec, int f) {
  return KIND == LP_OCTAHEDRON ? rec + 4 + 3 * f : rec + 4 + 4 * f;
}

// The thread's two pixel rays r = ((x+0.5-cx)/fx, (y+0.5-cy)/fy, 1) (same x), their lengths, and the
// screen offsets x+0.5-cx, y+0.5-cy as unevaluated sums hi + lo (exact): d below needs them to
// ~1e-7 px relative accuracy, not the ~6e-8 relative accuracy of a rounded r (a rounded r is off by
// ~1e-6 at depth 15 -- visible as 5e-4 transmittance on a 3 mm primitive with sigma 290).
struct ExactRay {
  float rx;
  float2 ry2, rn2;
  float sxh, sxl, syh[2], syl[2];
  float fxc, fyc, ifx, ify;
};

__device__ __forceinline__ void two_diff(float a, float b, float &s, float &e) {   // s + e = a - b exactly
  s = fs(a, b);
  const float bv = fs(s, a);          // = -b up to the rounding of s
  const float av = fs(s, bv);
  e = fa(fs(a, av), fs(-b, bv));
}

__device__ __forceinline__ ExactRay make_ray(const lp_camera &cam, float px, float py0, float py1) {
  ExactRay R;
  R.rx = __fdiv_rn(fs(px, cam.cx), cam.fx);
  R.ry2 = make_float2(__fdiv_rn(fs(py0, cam.cy), cam.fy), __fdiv_rn(fs(py1, cam.cy), cam.fy));
  R.rn2 = make_float2(sqrtf(fmaf(R.rx, R.rx, fmaf(R.ry2.x, R.ry2.x, 1.f))),
                      sqrtf(fmaf(R.rx, R.rx, fmaf(R.ry2.y, R.ry2.y, 1.f))));
  two_diff(px, cam.cx, R.sxh, R.sxl);
  two_diff(py0, cam.cy, R.syh[0], R.syl[0]);
  two_diff(py1, cam.cy, R.syh[1], R.syl[1]);
  R.fxc = cam.fx;
  R.fyc = cam.fy;
  R.ifx = __frcp_rn(cam.fx);
  R.ify = __frcp_rn(cam.fy);
  return R;
}

// (p_c f - p_z s) / f with the two products split exactly (FMA) and s = sh + sl: the offset
// p_c - p_z r_c of the centre from the pixel ray at the centre's depth, accurate to a few ulp of
// itself even though p_c f and p_z s nearly cancel
__device__ __forceinline__ float ray_offset(float pc, float pz, float f, float sh, float sl, float inv_f) {
  const float ah = fm(pc, f), al = __fmaf_rn(pc, f, -ah);
  const float bh = fm(pz, sh);
  float bl = __fmaf_rn(pz, sh, -bh);
  bl = __fmaf_rn(pz, sl, bl);
  return fm(fa(fs(ah, bh), fs(al, bl)), inv_f);
}

// per-pixel offsets of the centre from the pixel ray at depth p_z: d = p - p_z r (d_z = 0)
template <int KIND>
__device__ __forceinline__ void exact_d(const float *rec, const ExactRay &R, float &dx, float2 &dy2) {
  using ER = ExactRec<KIND>;
  const float px = rec[ER::P], py = rec[ER::P + 1], pz = rec[ER::P + 2];
  dx = ray_offset(px, pz, R.fxc, R.sxh, R.sxl, R.ifx);
  dy2 = make_float2(ray_offset(py, pz, R.fyc, R.syh[0], R.syl[0], R.ify),
                    ray_offset(py, pz, R.fyc, R.syh[1], R.syl[1], R.ify));
}

template <int KIND>
__device__ __forceinline__ void planesE2(const float *rec, const ExactRay &R, PlanesE2 &P) {
  const float rx = R.rx;
  const float2 ry2 = R.ry2;
  float dx;
  float2 dy2;
  exact_d<KIND>(rec, R, dx, dy2);
#pragma unroll
  for (int f = 0; f < 4; ++f) {
    const float *n = plane_n<KIND>(rec, f);
    const float2 k = ffma2(bc(n[1]), ry2, bc(__fmaf_rn(n[0], rx, n[2])));
    const float2 ik = make_float2(rcp_approx(k.x), rcp_approx(k.y));
    const float2 L = ffma2(bc(n[1]), dy2, bc(fm(n[0], dx)));          // n . d
    if (KIND == LP_OCTAHEDRON) {
      const float2 ta = fmul2(fsub2(L, bc(1.f)), ik), tb = fmul2(fadd2(L, bc(1.f)), ik);
      P.en[f] = make_float2(fminf(ta.x, tb.x), fminf(ta.y, tb.y));
      P.ex[f] = make_float2(fmaxf(ta.x, tb.x), fmaxf(ta.y, tb.y));
    } else {
      const float2 t = fmul2(fadd2(L, bc(n[3])), ik);
      P.en[f] = make_float2(k.x < 0.f ? t.x : -INFINITY, k.y < 0.f ? t.y : -INFINITY);
      P.ex[f] = make_float2(k.x > 0.f ? t.x : INFINITY, k.y > 0.f ? t.y : INFINITY);
    }
  }
}

// 1/k of plane f for one pixel, bitwise the paired evaluation above
template <int KIND>
__device__ __forceinline__ float plane_ik(const float *rec, int f, float rx, float ry) {
  const float *n = plane_n<KIND>(rec, f);
  return rcp_approx(__fmaf_rn(n[1], ry, __fmaf_rn(n[0], rx, n[2])));
}

// chord in ray parameter, ex - en (negative when there is no intersection in front of the camera,
// i.e. unless p_z + entry > 0); en2 / ex2 receive the entry / exit tau.  Euclidean chord = this |r|.
__device__ __forceinline__ float2 chordE2_of(const PlanesE2 &P, float pz, float2 &en2, float2 &ex2) {
  en2 = P.en[0];
  ex2 = P.ex[0];
#pragma unroll
  for (int f = 1; f < 4; ++f) {
    en2.x = fmaxf(en2.x, P.en[f].x);
    en2.y = fmaxf(en2.y, P.en[f].y);
    ex2.x = fminf(ex2.x, P.ex[f].x);
    ex2.y = fminf(ex2.y, P.ex[f].y);
  }
  float2 ch = fsub2(ex2, en2);
  if (!(fa(en2.x, pz) > 0.f)) ch.x = -1.f;   // entry behind the camera: the oracle's single-hit case (reading 27)
  if (!(fa(en2.y, pz) > 0.f)) ch.y = -1.f;
  return ch;
}

// first plane attaining the max entry / min exit of pixel k
__device__ __forceinline__ void trackE_k(const PlanesE2 &P, int k, float en, float ex, int &se, int &sx) {
  se = 3;
  sx = 3;
#pragma unroll
  for (int f = 2; f >= 0; --f) {
    if (lane_k(P.en[f], k) == en) se = f;
    if (lane_k(P.ex[f], k) == ex) sx = f;
  }
}

// slack of the bbox reject test: a pair rejected by it has chord <= 0 (up to fp32 rounding of
// the bbox itself, covered by the slack)
__device__ __forceinline__ bool in_bbox(const float4 &bb, float px, float py) {
  return fabsf(px - bb.x) <= bb.z && fabsf(py - bb.y) <= bb.w;
}

// MUFU approximations without the denormal range fix-ups (arguments and results stay normal here)
__device__ __forceinline__ float ex2_ftz(float x) {
  float y;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}
__device__ __forceinline__ float rcp_ftz(float x) {
  float y;
  asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}

// optical depth x = sigma chord of one (pixel, entry) pair, capped at 80 so E = exp(-x) stays a
// normal fp32 (>= 1.8e-35) and the backward can divide by it (T / E = T * rcp_ftz(E)); the cap
// changes o by < 1e-34.
__device__ __forceinline__ float optical_depth(float sigma, float chord) { return fminf(fm(sigma, chord), 80.f); }
// transmittance factor E = exp(-x); identical in forward and backward.  Same value as
// __expf (ex2.approx of x log2 e) minus its denormal-result handling, never needed above 2^-116.
__device__ __forceinline__ float transmit_x(float x) { return ex2_ftz(fm(-x, 1.44269504f)); }
__device__ __forceinline__ float transmit(float sigma, float chord) { return transmit_x(optical_depth(sigma, chord)); }

// opacity o = 1 - exp(-x) = -expm1(-x) to ~4e-6 relative for every x >= 0.  1 - E cancels
// for small x: an E near 1 carries ex2.approx's ~2^-22 relative error into o as 2^-22 / x (a
// primitive with x = 1e-4 got o wrong by 0.3 %, and its colour gradient sum_p T o G -- strongly
// cancelling under a random-sign upstream -- by the same factor).  Below x = 1/16, o is the Taylor
// series of -expm1(-x) to degree 4 in Horner form (truncation x^4 / 5! < 1.3e-7 relative); above
// it 1 - E loses at most E / o < 16 times E's relative error.
__device__ __forceinline__ float opacity_x(float x, float E) {
  float p = fmaf(x, -4.16666667e-02f, 1.66666667e-01f);   // -1/4!, 1/3!
  p = fmaf(x, p, -0.5f);
  p = fmaf(x, p, 1.f);
  return x < 0.0625f ? p * x : 1.f - E;
}
// the same for a pixel pair (FFMA2 lanes; each lane bitwise the scalar opacity_x)
__device__ __forceinline__ float2 opacity_x2(float2 x, float2 E) {
  float2 p = ffma2(x, bc(-4.16666667e-02f), bc(1.66666667e-01f));
  p = ffma2(x, p, bc(-0.5f));
  p = ffma2(x, p, bc(1.f));
  p = fmul2(p, x);
  const float2 q = fsub2(bc(1.f), E);
  return make_float2(x.x < 0.0625f ? p.x : q.x, x.y < 0.0625f ? p.y : q.y);
}

// smallest stop threshold the raster uses: t_stop below it is raised to it (reading 28).
// Every T the backward recovers is then >= 2^-100 (a normal fp32 far from underflow), except the
// stopping entry's own T_after, which the backward never divides (it starts from T_last).
#define LP_T_FLOOR 7.88860905e-31f   /* 2^-100 */
__host__ __device__ __forceinline__ float effective_t_stop(float t_stop) { return t_stop > LP_T_FLOOR ? t_stop : LP_T_FLOOR; }

// forward -> backward transmittance checkpoints: T of every pixel of a tile in front of batch i
// (entries [start + 128 i, ...)), i >= 1, stored at slot tile + start / 128 + i (unique per (tile,
// i): a list of n batches spans at least 128 (n - 1) + 1 entries); [slots][128 threads] float2
__host__ __device__ __forceinline__ int64_t ckpt_slots(int64_t tiles, int64_t capacity) { return tiles + capacity / 128 + 2; }
__device__ __forceinline__ float2 *ckpt_at(float *base, int tile, uint32_t start, uint32_t b) {
  return reinterpret_cast<float2 *>(base) + ((size_t)tile + (start >> 7) + ((b - start) >> 7)) * 128;
}
// checked builds: the slot of ckpt_at stays inside the frame's checkpoint buffer
#define LP_CHECK_CKPT(F, tile, start, b)                                                                  \
  LP_CHECK((int64_t)(tile) + ((start) >> 7) + (((b) - (start)) >> 7) <                                     \
           ckpt_slots((int64_t)(F).tiles_x * (F).tiles_y, (F).capacity > 0 ? (F).capacity : 1))

}  // namespace lp
