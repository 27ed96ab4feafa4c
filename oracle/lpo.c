/*
 * oracle/lpo.c -- CPU ORACLE for the LinPrim tile rasterizer (arXiv 2501.16312).
 *
 * TEST INFRASTRUCTURE ONLY: only tests/, __graft_entry__.smoke() and bench.py's
 * cpu_baseline / --impl reference legs may load it.  It shares no code with the
 * CUDA path.  Plain, slow, obviously-correct: fp64 everywhere except the
 * canonical fp32 geometry contract (lpo_geom.inc, mode 0).
 *
 * Build: gcc -O2 -std=c11 -ffp-contract=off -fno-fast-math -fopenmp -fPIC -shared
 *
 * Parity pins: every function below is pinned by tests/test_oracle_*.py
 * (closed forms, invariants, brute force, central finite differences).
 * Conventions the paper leaves open are listed in DESIGN.md "Readings".
 */
#define _GNU_SOURCE
#include "lpo.h"

#include <math.h>
#include <stdlib.h>
#include <string.h>
#include <float.h>
#ifdef _OPENMP
#include <omp.h>
#endif

/* 1/sqrt(3): tetrahedron basis b_k = (+-1, +-1, +-1)/sqrt(3) */
#define TETRA_K 0.57735026918962576451

/* ------------------------------------------------------------------ */
/* geometry: canonical fp32 (mode 0) and fp64 (mode 1) instantiations */
/* ------------------------------------------------------------------ */
#define REAL float
#define GTYPE geom_f
#define GFN geom_f32
#define GFN_RECT geom_rect_f32
#define RSQRT(x) sqrtf(x)
#define RCEIL(x) ceilf(x)
#define RFLOOR(x) floorf(x)
#define RABS(x) fabsf(x)
#include "lpo_geom.inc"
#undef REAL
#undef GTYPE
#undef GFN
#undef GFN_RECT
#undef RSQRT
#undef RCEIL
#undef RFLOOR
#undef RABS

#define REAL double
#define GTYPE geom_d
#define GFN geom_f64
#define GFN_RECT geom_rect_f64
#define RSQRT(x) sqrt(x)
#define RCEIL(x) ceil(x)
#define RFLOOR(x) floor(x)
#define RABS(x) fabs(x)
#include "lpo_geom.inc"
#undef REAL
#undef GTYPE
#undef GFN
#undef GFN_RECT
#undef RSQRT
#undef RCEIL
#undef RFLOOR
#undef RABS

/* ------------------------------------------------------------------ */
/* SH, 3DGS convention ("same approach described in 3DGS")   */
/* ------------------------------------------------------------------ */
static const double SH_C0 = 0.28209479177387814;
static const double SH_C1 = 0.4886025119029199;
static const double SH_C2[5] = {1.0925484305920792, -1.0925484305920792, 0.31539156525252005,
                                -1.0925484305920792, 0.5462742152960396};
static const double SH_C3[7] = {-0.5900435899266435, 2.890611442640554, -0.4570457994644658,
                                0.3731763325901154, -0.4570457994644658, 1.445305721320277,
                                -0.5900435899266435};

/* basis values Y[16] and gradients dY[16][3] at unit direction (x, y, z) */
static void sh_basis(double x, double y, double z, double Y[16], double dY[16][3])
{
  double xx = x * x, yy = y * y, zz = z * z, xy = x * y, yz = y * z, xz = x * z;
  memset(dY, 0, sizeof(double) * 48);
  Y[0] = SH_C0;
  Y[1] = -SH_C1 * y;  dY[1][1] = -SH_C1;
  Y[2] = SH_C1 * z;   dY[2][2] = SH_C1;
  Y[3] = -SH_C1 * x;  dY[3][0] = -SH_C1;
  Y[4] = SH_C2[0] * xy;                 dY[4][0] = SH_C2[0] * y;  dY[4][1] = SH_C2[0] * x;
  Y[5] = SH_C2[1] * yz;                 dY[5][1] = SH_C2[1] * z;  dY[5][2] = SH_C2[1] * y;
  Y[6] = SH_C2[2] * (2 * zz - xx - yy); dY[6][0] = -2 * SH_C2[2] * x; dY[6][1] = -2 * SH_C2[2] * y;
                                        dY[6][2] = 4 * SH_C2[2] * z;
  Y[7] = SH_C2[3] * xz;                 dY[7][0] = SH_C2[3] * z;  dY[7][2] = SH_C2[3] * x;
  Y[8] = SH_C2[4] * (xx - yy);          dY[8][0] = 2 * SH_C2[4] * x; dY[8][1] = -2 * SH_C2[4] * y;
  Y[9] = SH_C3[0] * y * (3 * xx - yy);
  dY[9][0] = 6 * SH_C3[0] * xy;         dY[9][1] = SH_C3[0] * (3 * xx - 3 * yy);
  Y[10] = SH_C3[1] * xy * z;
  dY[10][0] = SH_C3[1] * yz;            dY[10][1] = SH_C3[1] * xz;  dY[10][2] = SH_C3[1] * xy;
  Y[11] = SH_C3[2] * y * (4 * zz - xx - yy);
  dY[11][0] = -2 * SH_C3[2] * xy;       dY[11][1] = SH_C3[2] * (4 * zz - xx - 3 * yy);
  dY[11][2] = 8 * SH_C3[2] * yz;
  Y[12] = SH_C3[3] * z * (2 * zz - 3 * xx - 3 * yy);
  dY[12][0] = -6 * SH_C3[3] * xz;       dY[12][1] = -6 * SH_C3[3] * yz;
  dY[12][2] = SH_C3[3] * (6 * zz - 3 * xx - 3 * yy);
  Y[13] = SH_C3[4] * x * (4 * zz - xx - yy);
  dY[13][0] = SH_C3[4] * (4 * zz - 3 * xx - yy); dY[13][1] = -2 * SH_C3[4] * xy;
  dY[13][2] = 8 * SH_C3[4] * xz;
  Y[14] = SH_C3[5] * z * (xx - yy);
  dY[14][0] = 2 * SH_C3[5] * xz;        dY[14][1] = -2 * SH_C3[5] * yz;  dY[14][2] = SH_C3[5] * (xx - yy);
  Y[15] = SH_C3[6] * x * (xx - 3 * yy);
  dY[15][0] = SH_C3[6] * (3 * xx - 3 * yy); dY[15][1] = -6 * SH_C3[6] * xy;
}

/* exported for the pins: Y[16] (and dY[48]) at a unit direction */
void lpo_sh_basis(double x, double y, double z, double *Y, double *dY)
{
  double dd[16][3];
  sh_basis(x, y, z, Y, dd);
  if (dY) memcpy(dY, dd, sizeof(dd));
}

static void cam_pos(const lpo_camera *cam, double cp[3])
{
  /* x_cam = W x + t  =>  camera centre = -W^T t */
  for (int a = 0; a < 3; ++a)
    cp[a] = -((double)cam->W[0 * 3 + a] * cam->t[0] + (double)cam->W[1 * 3 + a] * cam->t[1]
              + (double)cam->W[2 * 3 + a] * cam->t[2]);
}

static int nverts(int kind) { return kind == LPO_OCTA ? 6 : 4; }
static int noffs(int kind) { return kind == LPO_OCTA ? 3 : 4; }

/* Eq. 1: sigma = -log(1 - 0.99 alpha) / (2 min(d)); alpha = sigmoid(logit) (reading 1) */
static double sigmoid(double x) { return 1.0 / (1.0 + exp(-x)); }

static double min_dhat(const lpo_scene *s, int i)
{
  int K = noffs(s->kind);
  double m = DBL_MAX;
  for (int a = 0; a < K; ++a) {
    double d = s->dist[a * s->n + i];
    if (s->filter3d) d = sqrt(d * d + (double)s->filter3d[i] * s->filter3d[i]);
    if (d < m) m = d;
  }
  return m;
}

int lpo_preprocess(const lpo_scene *s, const lpo_camera *cam, float kappa, int32_t mode, int32_t exact,
                   const double *den_override, lpo_pre *out)
{
  if (!s || !cam || !out || (s->kind != LPO_OCTA && s->kind != LPO_TETRA)) return -1;
  if (s->sh_degree < 0 || s->sh_degree > 3) return -1;
  const int n = s->n, K = noffs(s->kind), G = 3 + 3 * K, NC = 2 + 3 * K;
  const int ncoef = (s->sh_degree + 1) * (s->sh_degree + 1);
  double cp[3];
  cam_pos(cam, cp);
#pragma omp parallel for schedule(static)
  for (int i = 0; i < n; ++i) {
    int flag;
    uint32_t tt, key;
    int rect[4];
    double geo[15];
    if (mode == 0) {
      geom_f g;
      geom_f32(s, cam, i, kappa, exact, &g);
      flag = g.flag; tt = g.tiles_touched; key = g.depth_key;
      memcpy(rect, g.rect, sizeof(rect));
      geo[0] = g.cr_x; geo[1] = g.cr_y; geo[2] = exact ? g.cz : g.l;
      for (int j = 0; j < K; ++j)
        for (int a = 0; a < 3; ++a) geo[3 + 3 * j + a] = g.off[j][a];
      if (out->canon) {
        float *cn = out->canon + (size_t)i * NC;
        cn[0] = g.cr_x; cn[1] = g.cr_y;
        for (int j = 0; j < K; ++j)
          for (int a = 0; a < 3; ++a) cn[2 + 3 * j + a] = g.off[j][a];
      }
    } else {
      geom_d g;
      geom_f64(s, cam, i, kappa, exact, &g);
      flag = g.flag; tt = g.tiles_touched; key = g.depth_key;
      memcpy(rect, g.rect, sizeof(rect));
      geo[0] = g.cr_x; geo[1] = g.cr_y; geo[2] = exact ? g.cz : g.l;
      for (int j = 0; j < K; ++j)
        for (int a = 0; a < 3; ++a) geo[3 + 3 * j + a] = g.off[j][a];
      if (out->canon) memset(out->canon + (size_t)i * NC, 0, sizeof(float) * NC);
    }
    if (flag != 0) { tt = 0; memset(rect, 0, sizeof(rect)); memset(geo, 0, sizeof(geo)); }
    if (tt == 0) memset(rect, 0, sizeof(rect));
    out->flag[i] = flag;
    out->tiles_touched[i] = tt;
    memcpy(out->rect + 4 * (size_t)i, rect, sizeof(rect));
    out->depth_key[i] = flag ? 0u : key;
    memcpy(out->geom + (size_t)i * G, geo, sizeof(double) * G);

    /* density, Eq. 1, denominator frozen for the backward */
    double sig = 0.0, den = 0.0, rgb[3] = {0, 0, 0};
    if (flag == 0) {
      double alpha = sigmoid((double)s->opacity[i]);
      den = den_override ? den_override[i] : 2.0 * min_dhat(s, i);
      sig = -log1p(-0.99 * alpha) / den;
      /* view-dependent colour, dir = (c - campos)/|c - campos| (3DGS) */
      double v[3], nv = 0;
      for (int a = 0; a < 3; ++a) { v[a] = (double)s->pos[a * n + i] - cp[a]; nv += v[a] * v[a]; }
      nv = sqrt(nv);
      double Y[16], dY[16][3];
      sh_basis(v[0] / nv, v[1] / nv, v[2] / nv, Y, dY);
      for (int ch = 0; ch < 3; ++ch) {
        double acc = 0.0;
        for (int k = 0; k < ncoef; ++k) acc += (double)s->sh[((size_t)k * 3 + ch) * n + i] * Y[k];
        acc += 0.5;
        rgb[ch] = acc > 0.0 ? acc : 0.0;
        if (out->rgb_raw) out->rgb_raw[(size_t)i * 3 + ch] = acc;
      }
    }
    out->sigma[i] = sig;
    if (out->sigma_den) out->sigma_den[i] = den;
    for (int ch = 0; ch < 3; ++ch) out->rgb[(size_t)i * 3 + ch] = rgb[ch];
  }
  return 0;
}

/* ------------------------------------------------------------------ */
/* binning: one (tile|depth, id) entry per overlapped tile */
/* ------------------------------------------------------------------ */
typedef struct { uint64_t key; uint32_t id; } bin_entry;

static int cmp_entry(const void *a, const void *b)
{
  const bin_entry *x = (const bin_entry *)a, *y = (const bin_entry *)b;
  if (x->key != y->key) return x->key < y->key ? -1 : 1;
  if (x->id != y->id) return x->id < y->id ? -1 : 1;   /* ties by primitive id (reading 11) */
  return 0;
}

int64_t lpo_bin(int32_t n, const uint32_t *tiles_touched, const int32_t *rect,
                const uint32_t *depth_key, int32_t width, int32_t height,
                const uint8_t *tile_mask, uint64_t *keys, uint32_t *vals,
                int64_t capacity, int64_t *ranges)
{
  const int gx = (width + LPO_TILE - 1) / LPO_TILE, gy = (height + LPO_TILE - 1) / LPO_TILE;
  const int64_t T = (int64_t)gx * gy;
  int64_t E = 0;
  for (int i = 0; i < n; ++i) {
    if (tiles_touched[i] == 0) continue;
    for (int ty = rect[4 * i + 1]; ty <= rect[4 * i + 3]; ++ty)
      for (int tx = rect[4 * i + 0]; tx <= rect[4 * i + 2]; ++tx)
        if (!tile_mask || tile_mask[(int64_t)ty * gx + tx]) ++E;
  }
  if (E > capacity) return -E;
  bin_entry *buf = (bin_entry *)malloc(sizeof(bin_entry) * (size_t)(E > 0 ? E : 1));
  if (!buf) return -1;
  int64_t e = 0;
  for (int i = 0; i < n; ++i) {
    if (tiles_touched[i] == 0) continue;
    for (int ty = rect[4 * i + 1]; ty <= rect[4 * i + 3]; ++ty)
      for (int tx = rect[4 * i + 0]; tx <= rect[4 * i + 2]; ++tx) {
        int64_t t = (int64_t)ty * gx + tx;
        if (tile_mask && !tile_mask[t]) continue;
        buf[e].key = ((uint64_t)t << 32) | depth_key[i];
        buf[e].id = (uint32_t)i;
        ++e;
      }
  }
  qsort(buf, (size_t)E, sizeof(bin_entry), cmp_entry);
  for (int64_t t = 0; t < 2 * T; ++t) ranges[t] = 0;
  for (int64_t k = 0; k < E; ++k) {
    keys[k] = buf[k].key;
    vals[k] = buf[k].id;
    int64_t t = (int64_t)(buf[k].key >> 32);
    if (k == 0 || (buf[k - 1].key >> 32) != (uint64_t)t) ranges[2 * t] = k;
    ranges[2 * t + 1] = k + 1;
  }
  free(buf);
  (void)gy;
  return E;
}

/* ------------------------------------------------------------------ */
/* faces (windings outward)          */
/* ------------------------------------------------------------------ */
/* octahedron vertex 2j = c + o_j, 2j+1 = c - o_j; face f = 4[sx<0] + 2[sy<0] + [sz<0] */
static void octa_face(int f, int idx[3])
{
  int nx = (f >> 2) & 1, ny = (f >> 1) & 1, nz = f & 1;
  int a = 0 + nx, b = 2 + ny, c = 4 + nz;
  int neg = nx + ny + nz;   /* s_x s_y s_z > 0  <=>  even number of negative signs */
  idx[0] = a;
  if (neg % 2 == 0) { idx[1] = b; idx[2] = c; } else { idx[1] = c; idx[2] = b; }
}
static const int TETRA_FACES[4][3] = {{1, 3, 2}, {0, 2, 3}, {0, 3, 1}, {0, 1, 2}};

static void face_indices(int kind, int f, int idx[3])
{
  if (kind == LPO_OCTA) octa_face(f, idx);
  else { idx[0] = TETRA_FACES[f][0]; idx[1] = TETRA_FACES[f][1]; idx[2] = TETRA_FACES[f][2]; }
}

/* ray-space vertices of primitive i from its preprocess geometry (fp64) */
static void vertices(int kind, const double *geo, double V[6][3])
{
  if (kind == LPO_OCTA) {
    for (int j = 0; j < 3; ++j)
      for (int a = 0; a < 3; ++a) {
        V[2 * j][a] = geo[a] + geo[3 + 3 * j + a];
        V[2 * j + 1][a] = geo[a] - geo[3 + 3 * j + a];
      }
  } else {
    for (int k = 0; k < 4; ++k)
      for (int a = 0; a < 3; ++a) V[k][a] = geo[a] + geo[3 + 3 * k + a];
  }
}

/* 2-D Moller-Trumbore for the vertical ray through r (App. E).
 * d is the MT determinant e1 . (z x e2) = -(2-D cross) (reading 16).
 * Returns 1 on hit with barycentrics (u, v), determinant d and depth i. */
static int mtia(const double A[3], const double B[3], const double C[3], double rx, double ry,
                double *u, double *v, double *d, double *depth)
{
  double e1x = B[0] - A[0], e1y = B[1] - A[1];
  double e2x = C[0] - A[0], e2y = C[1] - A[1];
  double det = -(e1x * e2y - e1y * e2x);
  if (fabs(det) <= 1e-12) return 0;
  double sx = rx - A[0], sy = ry - A[1];
  double uu = (-sx * e2y + sy * e2x) / det;
  double vv = (sx * e1y - sy * e1x) / det;
  if (uu < 0.0 || vv < 0.0 || uu + vv > 1.0) return 0;
  *u = uu; *v = vv; *d = det;
  *depth = (1.0 - uu - vv) * A[2] + uu * B[2] + vv * C[2];
  return 1;
}

/* App. E: d i / d v_k for the three corners of a hit face.
 * v0 follows the printed formula; v1, v2 are "analogous" (derived in DESIGN.md). */
static void mtia_grad(const double A[3], const double B[3], const double C[3], double rx, double ry,
                      double u, double v, double d, double di[3][3])
{
  const double *v0 = A, *v1 = B, *v2 = C;
  double e1x = v1[0] - v0[0], e1y = v1[1] - v0[1];
  double e2x = v2[0] - v0[0], e2y = v2[1] - v0[1];
  double sx = rx - v0[0], sy = ry - v0[1];
  double du[3][2], dv[3][2];
  /* corner v0, as printed */
  du[0][0] = ((v2[1] - ry) - u * (v2[1] - v1[1])) / d;
  du[0][1] = ((rx - v2[0]) - u * (v1[0] - v2[0])) / d;
  dv[0][0] = ((ry - v1[1]) - v * (v2[1] - v1[1])) / d;
  dv[0][1] = ((v1[0] - rx) - v * (v1[0] - v2[0])) / d;
  /* corner v1 */
  du[1][0] = (u * e2y) / d;
  du[1][1] = (-u * e2x) / d;
  dv[1][0] = (-sy - v * (-e2y)) / d;
  dv[1][1] = (sx - v * e2x) / d;
  /* corner v2 */
  du[2][0] = (sy - u * e1y) / d;
  du[2][1] = (-sx - u * (-e1x)) / d;
  dv[2][0] = (-v * e1y) / d;
  dv[2][1] = (-v * (-e1x)) / d;
  const double w[3] = {1.0 - u - v, u, v};
  for (int k = 0; k < 3; ++k) {
    for (int a = 0; a < 2; ++a)
      di[k][a] = -(du[k][a] + dv[k][a]) * v0[2] + du[k][a] * v1[2] + dv[k][a] * v2[2];
    di[k][2] = w[k];
  }
}

/* 3-D Moller-Trumbore (the "no ray space" variant, App. D): ray t r from the camera centre
 * against triangle (A, B, C) in camera space.  Returns 1 on a hit with t > 0, barycentrics
 * (u, v), determinant d = e1 . (r x e2) and the ray parameter t (the camera-space depth, r_z = 1). */
static int mtia3(const double A[3], const double B[3], const double C[3], const double r[3],
                 double *u, double *v, double *d, double *t)
{
  double e1[3] = {B[0] - A[0], B[1] - A[1], B[2] - A[2]};
  double e2[3] = {C[0] - A[0], C[1] - A[1], C[2] - A[2]};
  double P[3] = {r[1] * e2[2] - r[2] * e2[1], r[2] * e2[0] - r[0] * e2[2], r[0] * e2[1] - r[1] * e2[0]};
  double det = e1[0] * P[0] + e1[1] * P[1] + e1[2] * P[2];
  double scale = (fabs(e1[0]) + fabs(e1[1]) + fabs(e1[2])) * (fabs(e2[0]) + fabs(e2[1]) + fabs(e2[2]));
  if (fabs(det) <= 1e-14 * scale) return 0;
  double T[3] = {-A[0], -A[1], -A[2]};
  double uu = (T[0] * P[0] + T[1] * P[1] + T[2] * P[2]) / det;
  double Q[3] = {T[1] * e1[2] - T[2] * e1[1], T[2] * e1[0] - T[0] * e1[2], T[0] * e1[1] - T[1] * e1[0]};
  double vv = (r[0] * Q[0] + r[1] * Q[1] + r[2] * Q[2]) / det;
  if (uu < 0.0 || vv < 0.0 || uu + vv > 1.0) return 0;
  double tt = (e2[0] * Q[0] + e2[1] * Q[1] + e2[2] * Q[2]) / det;
  if (!(tt > 0.0)) return 0;
  *u = uu; *v = vv; *d = det; *t = tt;
  return 1;
}

/* d t / d(A, B, C) of the hit above, from t = (n . A)/(n . r), n = (B - A) x (C - A):
 * with w = A - t r:  dt/dB = (e2 x w)/(n . r),  dt/dC = (w x e1)/(n . r),
 *                    dt/dA = (n - e2 x w - w x e1)/(n . r). */
static void mtia3_grad(const double A[3], const double B[3], const double C[3], const double r[3], double t,
                       double dt[3][3])
{
  double e1[3] = {B[0] - A[0], B[1] - A[1], B[2] - A[2]};
  double e2[3] = {C[0] - A[0], C[1] - A[1], C[2] - A[2]};
  double n[3] = {e1[1] * e2[2] - e1[2] * e2[1], e1[2] * e2[0] - e1[0] * e2[2], e1[0] * e2[1] - e1[1] * e2[0]};
  double D = n[0] * r[0] + n[1] * r[1] + n[2] * r[2];
  double w[3] = {A[0] - t * r[0], A[1] - t * r[1], A[2] - t * r[2]};
  double gB[3] = {e2[1] * w[2] - e2[2] * w[1], e2[2] * w[0] - e2[0] * w[2], e2[0] * w[1] - e2[1] * w[0]};
  double gC[3] = {w[1] * e1[2] - w[2] * e1[1], w[2] * e1[0] - w[0] * e1[2], w[0] * e1[1] - w[1] * e1[0]};
  for (int a = 0; a < 3; ++a) {
    dt[1][a] = gB[a] / D;
    dt[2][a] = gC[a] / D;
    dt[0][a] = (n[a] - gB[a] - gC[a]) / D;
  }
}

typedef struct {
  int32_t prim;
  double o, chord, E, T_before;
  int f_in, f_out;
  double u_in, v_in, d_in, u_out, v_out, d_out;
  double dc, eT;   /* conditioning (test tolerances only): fp32 chord error scale, relative T error in front */
} hit_rec;

/* exact (App. D): r = perspective ray of the pixel, depths are ray parameters t, and the chord
 * and entry are scaled by |r| to Euclidean lengths (r_z = 1). */
static void primitive_hit(int kind, const double *geo, double rx, double ry, double *chord,
                          int *f_in, double *u_in, double *v_in, double *d_in,
                          int *f_out, double *u_out, double *v_out, double *d_out, int *nhits,
                          double *entry, int exact, const double r[3])
{
  double V[6][3];
  vertices(kind, geo, V);
  int nf = kind == LPO_OCTA ? 8 : 4;
  double lo = DBL_MAX, hi = -DBL_MAX;
  int cnt = 0;
  for (int f = 0; f < nf; ++f) {
    int idx[3];
    face_indices(kind, f, idx);
    double u, v, d, dep;
    int hit = exact ? mtia3(V[idx[0]], V[idx[1]], V[idx[2]], r, &u, &v, &d, &dep)
                    : mtia(V[idx[0]], V[idx[1]], V[idx[2]], rx, ry, &u, &v, &d, &dep);
    if (!hit) continue;
    ++cnt;
    if (dep < lo) { lo = dep; *f_in = f; *u_in = u; *v_in = v; *d_in = d; }
    if (dep > hi) { hi = dep; *f_out = f; *u_out = u; *v_out = v; *d_out = d; }
  }
  *nhits = cnt;
  /* reading 4: chord = max - min over all hits if >= 2 hits, else 0 */
  double rn = exact ? sqrt(r[0] * r[0] + r[1] * r[1] + r[2] * r[2]) : 1.0;
  *chord = cnt >= 2 ? (hi - lo) * rn : 0.0;
  *entry = lo * rn;   /* i1, the entry depth (exact: Euclidean distance from the camera) */
  if (exact) { *d_in = lo; *d_out = hi; }   /* exact mode keeps the hit parameters t for the backward */
}

static void add_face_grad(int kind, const double *geo, int f, double u, double v, double d,
                          double rx, double ry, double dLdi, double *dvp, int exact, const double r[3],
                          int absval)
{
  double V[6][3];
  vertices(kind, geo, V);
  int idx[3];
  face_indices(kind, f, idx);
  double di[3][3];
  if (exact) {
    /* d is the hit parameter t here; chord = (t_out - t_in)|r| */
    double rn = sqrt(r[0] * r[0] + r[1] * r[1] + r[2] * r[2]);
    mtia3_grad(V[idx[0]], V[idx[1]], V[idx[2]], r, d, di);
    dLdi *= rn;
  } else {
    mtia_grad(V[idx[0]], V[idx[1]], V[idx[2]], rx, ry, u, v, d, di);
  }
  for (int k = 0; k < 3; ++k)
    for (int a = 0; a < 3; ++a) {
      double val = dLdi * di[k][a];
      if (absval) val = fabs(val);
#pragma omp atomic
      dvp[idx[k] * 3 + a] += val;
    }
}

static double bary_margin(double u, double v)
{
  double m = u;
  if (v < m) m = v;
  if (1.0 - u - v < m) m = 1.0 - u - v;
  return m;
}

typedef struct { int64_t start, end; } span;
typedef struct { uint32_t key; uint32_t id; } kid;
static int cmp_kid(const void *a, const void *b)
{
  const kid *x = (const kid *)a, *y = (const kid *)b;
  if (x->key != y->key) return x->key < y->key ? -1 : 1;
  return x->id < y->id ? -1 : (x->id > y->id);
}

int lpo_render(const lpo_scene *s, const lpo_camera *cam, const lpo_pre *pre,
               const uint32_t *sorted_vals, const int64_t *ranges,
               const lpo_render_cfg *cfg, const int32_t *pix, int64_t npix,
               double *image, double *T_final, int32_t *n_proc, double *m_stop, double *m_face,
               const float *dL_dimage, double *dv, double *dsigma, double *drgb,
               double *face_margin, int64_t *counters, double *depth, double *m_depth,
               double *bnd_rgb, double *bnd_sigma, double *bnd_dv)
{
  const int W = cam->width, H = cam->height, gx = (W + LPO_TILE - 1) / LPO_TILE;
  const int kind = s->kind, K = noffs(kind), G = 3 + 3 * K, NV = nverts(kind);
  const int64_t HW = (int64_t)W * H;
  const int64_t total = pix ? npix : HW;

  /* brute mode: every in-frustum primitive, ordered by (key, id) */
  uint32_t *bl = NULL;
  int64_t nb = 0;
  if (cfg->brute) {
    kid *tmp = (kid *)malloc(sizeof(kid) * (size_t)(s->n > 0 ? s->n : 1));
    for (int i = 0; i < s->n; ++i)
      if (pre->flag[i] == 0) { tmp[nb].key = pre->depth_key[i]; tmp[nb].id = (uint32_t)i; ++nb; }
    qsort(tmp, (size_t)nb, sizeof(kid), cmp_kid);
    bl = (uint32_t *)malloc(sizeof(uint32_t) * (size_t)(nb > 0 ? nb : 1));
    for (int64_t k = 0; k < nb; ++k) bl[k] = tmp[k].id;
    free(tmp);
  }
  int64_t it_total = 0, hit_total = 0;

#pragma omp parallel reduction(+ : it_total, hit_total)
  {
    int64_t cap = 256;
    hit_rec *hits = (hit_rec *)malloc(sizeof(hit_rec) * (size_t)cap);
#pragma omp for schedule(dynamic, 64)
    for (int64_t q = 0; q < total; ++q) {
      int64_t p = pix ? pix[q] : q;
      int px = (int)(p % W), py = (int)(p / W);
      double rx = px + 0.5, ry = py + 0.5;
      const double rv[3] = {(rx - (double)cam->cx) / (double)cam->fx, (ry - (double)cam->cy) / (double)cam->fy, 1.0};
      const int exact = cfg->exact;
      const uint32_t *list;
      int64_t cnt;
      if (cfg->brute) { list = bl; cnt = nb; }
      else {
        int64_t t = (int64_t)(py / LPO_TILE) * gx + px / LPO_TILE;
        list = sorted_vals + ranges[2 * t];
        cnt = ranges[2 * t + 1] - ranges[2 * t];
      }
      double T = 1.0, C[3] = {0, 0, 0}, ms = DBL_MAX, mf = DBL_MAX, dep = 0.0, md = DBL_MAX, eT = 0.0;
      int dep_set = 0;
      int64_t nh = 0, np = 0;
      for (int64_t e = 0; e < cnt; ++e) {
        int i = (int)list[e];
        np = e + 1;
        const double *geo = pre->geom + (size_t)i * G;
        double chord, u_in = 0, v_in = 0, d_in = 1, u_out = 0, v_out = 0, d_out = 1;
        int f_in = 0, f_out = 0, nhit;
        double i1;
        primitive_hit(kind, geo, rx, ry, &chord, &f_in, &u_in, &v_in, &d_in, &f_out, &u_out,
                      &v_out, &d_out, &nhit, &i1, exact, rv);
        if (!(chord > 0.0)) continue;
        /* opacity from the chord, App. E */
        double sig = pre->sigma[i];
        double E = exp(-sig * chord);
        double o = -expm1(-sig * chord);
        if (nh == cap) { cap *= 2; hits = (hit_rec *)realloc(hits, sizeof(hit_rec) * (size_t)cap); }
        hit_rec *h = &hits[nh++];
        h->prim = i; h->o = o; h->chord = chord; h->E = E; h->T_before = T;
        {
          /* Conditioning of the chord in fp32 (test tolerances only): an fp32
             evaluation of i2 - i1 from the primitive's centre-relative geometry carries an absolute
             error of a few units in the last place of the depths it subtracts, |i - z_c| and the
             primitive's own depth extent; 8 ulp (2^-20) of their sum.  eT: the relative error this
             puts on T of the entries behind (sum of sigma dc). */
          double zc, Z = 0.0;
          if (exact) {
            zc = sqrt(geo[0] * geo[0] + geo[1] * geo[1] + geo[2] * geo[2]);
            for (int j = 0; j < K; ++j) {
              const double *oj = geo + 3 + 3 * j;
              double nj = sqrt(oj[0] * oj[0] + oj[1] * oj[1] + oj[2] * oj[2]);
              if (nj > Z) Z = nj;
            }
          } else {
            zc = geo[2];
            for (int j = 0; j < K; ++j) if (fabs(geo[3 + 3 * j + 2]) > Z) Z = fabs(geo[3 + 3 * j + 2]);
          }
          h->dc = 0x1p-20 * (fabs(i1 - zc) + fabs(i1 + chord - zc) + 2.0 * Z);
          h->eT = eT;
          eT += sig * h->dc;
        }
        h->f_in = f_in; h->u_in = u_in; h->v_in = v_in; h->d_in = d_in;
        h->f_out = f_out; h->u_out = u_out; h->v_out = v_out; h->d_out = d_out;
        double m1 = bary_margin(u_in, v_in), m2 = bary_margin(u_out, v_out);
        if (m1 < mf) mf = m1;
        if (m2 < mf) mf = m2;
        /* front-to-back compositing */
        for (int ch = 0; ch < 3; ++ch) C[ch] += T * o * pre->rgb[(size_t)i * 3 + ch];
        T *= E;
        /* depth mode: first primitive after which cumulative opacity 1 - T > 0.5 */
        {
          double m = fabs(log(T / 0.5));
          if (m < md) md = m;
          if (!dep_set && 1.0 - T > 0.5) { dep = i1; dep_set = 1; }
        }
        {
          /* include-then-stop (reading 9); a threshold below 2^-100 (0 included) acts as 2^-100
             (reading 28: no fp32 image changes below it) */
          const double ts = cfg->t_stop > 0x1p-100f ? (double)cfg->t_stop : 0x1p-100;
          double m = fabs(log(T / ts));
          if (m < ms) ms = m;
          if (T < ts) break;
        }
      }
      for (int ch = 0; ch < 3; ++ch) C[ch] += T * cfg->bg[ch];
      it_total += np;
      hit_total += nh;
      if (image) for (int ch = 0; ch < 3; ++ch) image[ch * HW + p] = C[ch];
      if (T_final) T_final[p] = T;
      if (n_proc) n_proc[p] = (int32_t)np;
      if (m_stop) m_stop[p] = ms;
      if (m_face) m_face[p] = mf;
      if (depth) depth[p] = dep;
      if (m_depth) m_depth[p] = md;

      if (dL_dimage) {
        /* blend backward: S = colour behind k incl. background */
        double Gc[3] = {dL_dimage[p], dL_dimage[HW + p], dL_dimage[2 * HW + p]};
        double S[3] = {cfg->bg[0], cfg->bg[1], cfg->bg[2]}, eS[3] = {0, 0, 0};
        for (int64_t k = nh - 1; k >= 0; --k) {
          const hit_rec *h = &hits[k];
          const int i = h->prim;
          const double *rgb = pre->rgb + (size_t)i * 3;
          double dLdo = 0.0, edo = 0.0;
          const double eo = pre->sigma[i] * h->E * h->dc;   /* error of o from the chord's */
          for (int ch = 0; ch < 3; ++ch) {
            double val = h->T_before * h->o * Gc[ch];
#pragma omp atomic
            drgb[(size_t)i * 3 + ch] += val;
            dLdo += h->T_before * (rgb[ch] - S[ch]) * Gc[ch];
            edo += h->T_before * eS[ch] * fabs(Gc[ch]);
            if (bnd_rgb) {
              double b = h->T_before * fabs(Gc[ch]) * (eo + h->o * h->eT);
#pragma omp atomic
              bnd_rgb[(size_t)i * 3 + ch] += b;
            }
          }
          edo += fabs(dLdo) * h->eT;
          for (int ch = 0; ch < 3; ++ch) {
            eS[ch] = fabs(rgb[ch] - S[ch]) * eo + (1.0 - h->o) * eS[ch];
            S[ch] = h->o * rgb[ch] + (1.0 - h->o) * S[ch];
          }
          if (bnd_sigma) {
            double b = h->E * (fabs(dLdo) * h->dc * (1.0 + pre->sigma[i] * h->chord) + h->chord * edo);
#pragma omp atomic
            bnd_sigma[i] += b;
          }
          /* o = 1 - exp(-sigma (i2 - i1)) */
          double sig = pre->sigma[i];
          double ds = h->chord * h->E * dLdo;
#pragma omp atomic
          dsigma[i] += ds;
          double g = sig * h->E * dLdo;     /* dL/d i2 = g, dL/d i1 = -g */
          const double *geo = pre->geom + (size_t)i * G;
          double *dvp = dv + (size_t)i * NV * 3;
          add_face_grad(kind, geo, h->f_in, h->u_in, h->v_in, h->d_in, rx, ry, -g, dvp, exact, rv, 0);
          add_face_grad(kind, geo, h->f_out, h->u_out, h->v_out, h->d_out, rx, ry, g, dvp, exact, rv, 0);
          if (bnd_dv) {
            /* first-order error of g = sigma E dL/do from the chord and T errors */
            const double eg = sig * h->E * (fabs(dLdo) * sig * h->dc + edo);
            double *bvp = bnd_dv + (size_t)i * NV * 3;
            add_face_grad(kind, geo, h->f_in, h->u_in, h->v_in, h->d_in, rx, ry, eg, bvp, exact, rv, 1);
            add_face_grad(kind, geo, h->f_out, h->u_out, h->v_out, h->d_out, rx, ry, eg, bvp, exact, rv, 1);
          }
          if (face_margin) {
            double m = bary_margin(h->u_in, h->v_in), m2 = bary_margin(h->u_out, h->v_out);
            if (m2 < m) m = m2;
#pragma omp critical(lpo_fm)
            { if (m < face_margin[i]) face_margin[i] = m; }
          }
        }
      }
    }
    free(hits);
  }
  if (counters) { counters[0] += it_total; counters[1] += hit_total; }
  free(bl);
  return 0;
}

/* ------------------------------------------------------------------ */
/* preprocess backward, fp64          */
/* ------------------------------------------------------------------ */
int lpo_preprocess_bwd(const lpo_scene *s, const lpo_camera *cam, const lpo_pre *pre, int32_t exact,
                       const double *den_override, const double *dv, const double *dsigma,
                       const double *drgb, double *g_pos, double *g_rot, double *g_dist,
                       double *g_opacity, double *g_sh)
{
  const int n = s->n, kind = s->kind, K = noffs(kind), NV = nverts(kind);
  const int ncoef = (s->sh_degree + 1) * (s->sh_degree + 1);
  double cp[3];
  cam_pos(cam, cp);
  double Wm[3][3];
  for (int r = 0; r < 3; ++r)
    for (int c = 0; c < 3; ++c) Wm[r][c] = cam->W[3 * r + c];
  const double fx = cam->fx, fy = cam->fy;
#pragma omp parallel for schedule(static)
  for (int i = 0; i < n; ++i) {
    if (pre->flag[i] != 0) continue;
    const double *dvp = dv + (size_t)i * NV * 3;

    /* recompute the forward quantities in fp64 */
    double q[4], nq = 0;
    for (int a = 0; a < 4; ++a) { q[a] = s->rot[a * n + i]; nq += q[a] * q[a]; }
    nq = sqrt(nq);
    double w = q[0] / nq, x = q[1] / nq, y = q[2] / nq, z = q[3] / nq;
    double R[3][3] = {{1 - 2 * (y * y + z * z), 2 * (x * y - w * z), 2 * (x * z + w * y)},
                      {2 * (x * y + w * z), 1 - 2 * (x * x + z * z), 2 * (y * z - w * x)},
                      {2 * (x * z - w * y), 2 * (y * z + w * x), 1 - 2 * (x * x + y * y)}};
    double c[3], p[3];
    for (int a = 0; a < 3; ++a) c[a] = s->pos[a * n + i];
    for (int r = 0; r < 3; ++r) p[r] = Wm[r][0] * c[0] + Wm[r][1] * c[1] + Wm[r][2] * c[2] + cam->t[r];
    double l = sqrt(p[0] * p[0] + p[1] * p[1] + p[2] * p[2]);
    double J[3][3] = {{fx / p[2], 0, -fx * p[0] / (p[2] * p[2])},
                      {0, fy / p[2], -fy * p[1] / (p[2] * p[2])},
                      {p[0] / l, p[1] / l, p[2] / l}};
    double dh[4], dd[4];
    for (int a = 0; a < K; ++a) {
      dd[a] = s->dist[a * n + i];
      dh[a] = s->filter3d ? sqrt(dd[a] * dd[a] + (double)s->filter3d[i] * s->filter3d[i]) : dd[a];
    }
    double bvec[4][3];
    if (kind == LPO_OCTA) {
      for (int j = 0; j < 3; ++j)
        for (int a = 0; a < 3; ++a) bvec[j][a] = (a == j) ? 1.0 : 0.0;
    } else {
      const double kk = TETRA_K;
      const double B[4][3] = {{kk, kk, kk}, {kk, -kk, -kk}, {-kk, kk, -kk}, {-kk, -kk, kk}};
      memcpy(bvec, B, sizeof(B));
    }
    double ow[4][3], oc[4][3];
    for (int j = 0; j < K; ++j) {
      for (int r = 0; r < 3; ++r)
        ow[j][r] = dh[j] * (R[r][0] * bvec[j][0] + R[r][1] * bvec[j][1] + R[r][2] * bvec[j][2]);
      for (int r = 0; r < 3; ++r) oc[j][r] = Wm[r][0] * ow[j][0] + Wm[r][1] * ow[j][1] + Wm[r][2] * ow[j][2];
    }

    /* ray-space centre and offset gradients from the vertex gradients */
    double gcr[3] = {0, 0, 0}, go[4][3];
    for (int k = 0; k < NV; ++k)
      for (int a = 0; a < 3; ++a) gcr[a] += dvp[3 * k + a];
    if (kind == LPO_OCTA) {
      /* App. E: the negative-axis vertex gradient is negated onto the feature */
      for (int j = 0; j < 3; ++j)
        for (int a = 0; a < 3; ++a) go[j][a] = dvp[3 * (2 * j) + a] - dvp[3 * (2 * j + 1) + a];
    } else {
      for (int k = 0; k < 4; ++k)
        for (int a = 0; a < 3; ++a) go[k][a] = dvp[3 * k + a];
    }
    /* the 2D filter adds a constant (fixed index) -> identity */

    /* o_j = J oc_j, oc_j = W ow_j  (exact mode: the vertices are p +- oc_j, no J) */
    double gJ[3][3] = {{0}}, gp[3] = {0, 0, 0}, gR[3][3] = {{0}}, gdh[4] = {0, 0, 0, 0};
    for (int j = 0; j < K; ++j) {
      double goc[3], gow[3];
      for (int a = 0; a < 3; ++a)
        goc[a] = exact ? go[j][a] : J[0][a] * go[j][0] + J[1][a] * go[j][1] + J[2][a] * go[j][2];
      for (int r = 0; r < 3; ++r)
        for (int a = 0; a < 3; ++a) gJ[r][a] += go[j][r] * oc[j][a];
      for (int a = 0; a < 3; ++a)
        gow[a] = Wm[0][a] * goc[0] + Wm[1][a] * goc[1] + Wm[2][a] * goc[2];
      /* ow_j = dh_j R b_j */
      double Rb[3];
      for (int r = 0; r < 3; ++r) Rb[r] = R[r][0] * bvec[j][0] + R[r][1] * bvec[j][1] + R[r][2] * bvec[j][2];
      gdh[j] += Rb[0] * gow[0] + Rb[1] * gow[1] + Rb[2] * gow[2];
      for (int r = 0; r < 3; ++r)
        for (int cc = 0; cc < 3; ++cc) gR[r][cc] += dh[j] * gow[r] * bvec[j][cc];
    }
    /* centre: c_r = phi(p), d phi / dp = J  (exact mode: the centre is p itself) */
    if (exact) {
      for (int a = 0; a < 3; ++a) gp[a] += gcr[a];
    } else {
      for (int a = 0; a < 3; ++a) gp[a] += J[0][a] * gcr[0] + J[1][a] * gcr[1] + J[2][a] * gcr[2];
    }
    /* dJ/dp terms ("impact of the position on the ray space approximation"); gJ = 0 in exact mode */
    if (!exact) {
      double pz = p[2], pz2 = pz * pz, pz3 = pz2 * pz;
      gp[2] += gJ[0][0] * (-fx / pz2);
      gp[0] += gJ[0][2] * (-fx / pz2);
      gp[2] += gJ[0][2] * (2.0 * fx * p[0] / pz3);
      gp[2] += gJ[1][1] * (-fy / pz2);
      gp[1] += gJ[1][2] * (-fy / pz2);
      gp[2] += gJ[1][2] * (2.0 * fy * p[1] / pz3);
      for (int k = 0; k < 3; ++k)
        for (int m = 0; m < 3; ++m)
          gp[m] += gJ[2][k] * (((k == m) ? 1.0 : 0.0) - p[k] * p[m] / (l * l)) / l;
    }
    double gc[3];
    for (int a = 0; a < 3; ++a) gc[a] = Wm[0][a] * gp[0] + Wm[1][a] * gp[1] + Wm[2][a] * gp[2];

    /* distances (through the optional 3D filter) */
    for (int j = 0; j < K; ++j) g_dist[(size_t)j * n + i] += gdh[j] * (s->filter3d ? dd[j] / dh[j] : 1.0);

    /* R(q_hat) -> q_hat -> q */
    double dR[4][3][3] = {
      {{0, -2 * z, 2 * y}, {2 * z, 0, -2 * x}, {-2 * y, 2 * x, 0}},
      {{0, 2 * y, 2 * z}, {2 * y, -4 * x, -2 * w}, {2 * z, 2 * w, -4 * x}},
      {{-4 * y, 2 * x, 2 * w}, {2 * x, 0, 2 * z}, {-2 * w, 2 * z, -4 * y}},
      {{-4 * z, -2 * w, 2 * x}, {2 * w, -4 * z, 2 * y}, {2 * x, 2 * y, 0}}};
    double gqh[4] = {0, 0, 0, 0};
    for (int a = 0; a < 4; ++a)
      for (int r = 0; r < 3; ++r)
        for (int cc = 0; cc < 3; ++cc) gqh[a] += gR[r][cc] * dR[a][r][cc];
    double qh[4] = {w, x, y, z}, dot = 0;
    for (int a = 0; a < 4; ++a) dot += qh[a] * gqh[a];
    for (int a = 0; a < 4; ++a) g_rot[(size_t)a * n + i] += (gqh[a] - qh[a] * dot) / nq;

    /* opacity: Eq. 1 with the denominator frozen, alpha = sigmoid(logit) */
    double alpha = sigmoid((double)s->opacity[i]);
    double den = den_override ? den_override[i] : 2.0 * min_dhat(s, i);
    double dsig_dalpha = 0.99 / ((1.0 - 0.99 * alpha) * den);
    g_opacity[i] += dsigma[i] * dsig_dalpha * alpha * (1.0 - alpha);

    /* SH colour and its direction term */
    double v[3], nv = 0;
    for (int a = 0; a < 3; ++a) { v[a] = c[a] - cp[a]; nv += v[a] * v[a]; }
    nv = sqrt(nv);
    double dir[3] = {v[0] / nv, v[1] / nv, v[2] / nv};
    double Y[16], dY[16][3];
    sh_basis(dir[0], dir[1], dir[2], Y, dY);
    double gdir[3] = {0, 0, 0};
    for (int ch = 0; ch < 3; ++ch) {
      double raw = 0.5;
      for (int k = 0; k < ncoef; ++k) raw += (double)s->sh[((size_t)k * 3 + ch) * n + i] * Y[k];
      if (raw < 0.0) continue;   /* clamp max(0, .) */
      double gr = drgb[(size_t)i * 3 + ch];
      for (int k = 0; k < ncoef; ++k) {
        g_sh[((size_t)k * 3 + ch) * n + i] += Y[k] * gr;
        for (int a = 0; a < 3; ++a) gdir[a] += gr * (double)s->sh[((size_t)k * 3 + ch) * n + i] * dY[k][a];
      }
    }
    double dd_ = dir[0] * gdir[0] + dir[1] * gdir[1] + dir[2] * gdir[2];
    for (int a = 0; a < 3; ++a) gc[a] += (gdir[a] - dir[a] * dd_) / nv;

    for (int a = 0; a < 3; ++a) g_pos[(size_t)a * n + i] += gc[a];
  }
  return 0;
}

int lpo_mtia3(const double *A, const double *B, const double *C, const double *r, double *out)
{
  /* out = (u, v, det, t) */
  return mtia3(A, B, C, r, &out[0], &out[1], &out[2], &out[3]);
}

void lpo_mtia3_grad(const double *A, const double *B, const double *C, const double *r, double *dt)
{
  double u, v, d, t, g[3][3];
  if (!mtia3(A, B, C, r, &u, &v, &d, &t)) { memset(dt, 0, sizeof(g)); return; }
  mtia3_grad(A, B, C, r, t, g);
  memcpy(dt, g, sizeof(g));
}

/* ------------------------------------------------------------------ */
/* exported for the pins only: one MTIA evaluation and its App. E grads */
/* ------------------------------------------------------------------ */
int lpo_mtia(const double *A, const double *B, const double *C, double rx, double ry, double *out)
{
  /* out = (u, v, d, depth) */
  return mtia(A, B, C, rx, ry, &out[0], &out[1], &out[2], &out[3]);
}

void lpo_mtia_grad(const double *A, const double *B, const double *C, double rx, double ry,
                   double u, double v, double d, double *di /* [3][3] */)
{
  double g[3][3];
  mtia_grad(A, B, C, rx, ry, u, v, d, g);
  memcpy(di, g, sizeof(g));
}
