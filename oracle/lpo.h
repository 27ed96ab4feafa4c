/*
 * oracle/lpo.h -- CPU ORACLE for the LinPrim tile rasterizer (arXiv 2501.16312).
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and bench.py's
 * cpu_baseline / --impl reference legs may load this library.  The product path
 * (paper_2501_16312_b200/) never includes, links or calls it, and this file
 * shares no code with the CUDA path (no common headers, helpers or constants).
 *
 * Citation keys: P:n = PAPER.md line n, S:n = SPEC.md line n.
 *
 * What the oracle computes:
 *   - lpo_preprocess : per-primitive geometry in the canonical fp32
 *                      op order of DESIGN.md "Canonical fp32 contract" (mode 0),
 *                      or the same formulas in fp64 (mode 1, used only by the
 *                      finite-difference pins); sigma by Eq. 1 and
 *                      SH colour (3DGS convention) in fp64.
 *   - lpo_bin        : tile binning + (tile|depth, id) ordering.
 *   - lpo_render     : per pixel, 2-D Moller-Trumbore (MTIA) against every
 *                      triangular face, chord -> opacity
 *                      (P:1005-1007), front-to-back compositing with the
 *                      0.999 stop; optional backward by the
 *                      blend recursion and App. E.
 *   - lpo_preprocess_bwd : ray-space vertex gradients -> world features
 *                      (P:224-229), fp64.
 */
#ifndef LPO_H
#define LPO_H
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define LPO_OCTA  0
#define LPO_TETRA 1
#define LPO_TILE  16

typedef struct {
  int32_t kind, n, sh_degree;
  const float *pos;       /* [3][n] */
  const float *rot;       /* [4][n]  (w,x,y,z) */
  const float *dist;      /* [3|4][n] */
  const float *opacity;   /* [n] logit */
  const float *sh;        /* [(deg+1)^2][3][n] */
  const float *filter3d;  /* [n] or NULL */
} lpo_scene;

typedef struct {
  float W[9];   /* world->camera rotation, row-major: x_cam = W x + t */
  float t[3];
  float fx, fy, cx, cy, znear;
  int32_t width, height;
} lpo_camera;

/* Per-primitive preprocess outputs (caller allocates, n = scene->n, K = 3 octa / 4 tetra). */
typedef struct {
  int32_t  *flag;          /* [n] 0 = in frustum, 1 = invalid input, 2 = culled (p_z <= znear) */
  uint32_t *tiles_touched; /* [n] */
  int32_t  *rect;          /* [n][4] tx0, ty0, tx1, ty1 (inclusive); zeros when tiles_touched == 0 */
  uint32_t *depth_key;     /* [n] bits of the fp32 ray-space depth l = |p| */
  double   *geom;          /* [n][3 + 3K] c_r (x, y, l), then K post-filter ray-space offsets;
                              exact mode: camera-space centre p, then K camera-space offsets */
  float    *canon;         /* [n][2 + 3K] fp32 cr_x, cr_y, offsets (mode 0 only; may be NULL) */
  double   *sigma;         /* [n] Eq. 1 */
  double   *sigma_den;     /* [n] 2 * min(dhat), the frozen denominator */
  double   *rgb;           /* [n][3] clamped SH colour */
  double   *rgb_raw;       /* [n][3] SH colour before the clamp max(0, .) (may be NULL): parity tests use
                              it to find clamp decisions within rounding of 0 */
} lpo_pre;

/* Preprocess every primitive.  mode 0 = canonical fp32 geometry, 1 = fp64 geometry.
 * exact = 1: the "no ray space" variant (App. D): camera-space geometry, tile bbox
 * from the perspective projections of the vertices (whole screen if a vertex has p_z <= 0),
 * no 2D filter (kappa ignored); the depth key is still |p|.
 * den_override: NULL, or [n] frozen Eq. 1 denominators (finite-difference pins). */
int lpo_preprocess(const lpo_scene *s, const lpo_camera *cam, float kappa, int32_t mode, int32_t exact,
                   const double *den_override, lpo_pre *out);

/* Bin visible primitives to tiles and order every tile's list by (depth key, id).
 * tile_mask: NULL (all tiles) or [T] bytes; only tiles with mask != 0 get entries.
 * Returns E (number of entries written) or -(needed) if E > capacity.
 * keys[E] = (tile << 32) | depth_key, vals[E] = primitive id, ranges[2T] = [start, end). */
int64_t lpo_bin(int32_t n, const uint32_t *tiles_touched, const int32_t *rect,
                const uint32_t *depth_key, int32_t width, int32_t height,
                const uint8_t *tile_mask, uint64_t *keys, uint32_t *vals,
                int64_t capacity, int64_t *ranges);

typedef struct {
  float bg[3];
  float t_stop;           /* stop once T < t_stop (include-then-stop); below 2^-100 (0 included) it acts as
                             2^-100 (reading 28) */
  int32_t brute;          /* 1: ignore tiling, every valid primitive in (key, id) order */
  int32_t exact;          /* 1: geometry from lpo_preprocess(exact = 1); per-pixel perspective rays
                             r = ((x+0.5-cx)/fx, (y+0.5-cy)/fy, 1) against the camera-space faces by
                             3-D Moller-Trumbore, chord = (t_out - t_in) |r| (App. D) */
} lpo_render_cfg;

/* Render (and optionally backprop) a set of pixels.
 * pix: NULL (all pixels) or [npix] flat pixel indices y*W + x.
 * Outputs are full-image arrays; only the requested pixels are written.
 *   image[3][H][W] (fp64), T_final[H][W] (fp64), n_proc[H][W], m_stop[H][W] (min |ln(T/t_stop)| over hits),
 *   m_face[H][W] (min barycentric over the pixel's hit faces).
 * Backward (dL_dimage != NULL): accumulates (+=) into
 *   dv[n][V][3] (ray-space vertex gradients, V = 6 octa / 4 tetra), dsigma[n], drgb[n][3];
 *   face_margin[n] receives min barycentric over the primitive's hit faces (min-accumulate).
 * counters[2] (+=): iterated pairs, intersected pairs.
 * Depth mode (App. B "distance to the first primitive along the viewing ray where
 * cumulative opacity exceeds 0.5"): depth[H][W] = entry distance i1 (ray-space z of the entry
 * hit, whose scale is the camera distance |p|) of the first composited primitive after which
 * 1 - T > 0.5, else 0 (the invalid marker, reading 24); m_depth[H][W] = min over the pixel's
 * hits of |ln(T_after / 0.5)| (how far the 0.5 decision is from flipping).  Either may be NULL.
 * Conditioning bounds (test tolerances only; each may be NULL; += like the gradients):
 * bnd_rgb[n][3], bnd_sigma[n], bnd_dv[n][V][3] receive, per primitive, the first-order error that
 * an fp32 evaluation of the same method puts on drgb, dsigma and dv through the chord's rounding
 * (8 ulp of the centre-relative depths it subtracts) and the resulting T errors.
 * Returns 0 or -1. */
int lpo_render(const lpo_scene *s, const lpo_camera *cam, const lpo_pre *pre,
               const uint32_t *sorted_vals, const int64_t *ranges,
               const lpo_render_cfg *cfg, const int32_t *pix, int64_t npix,
               double *image, double *T_final, int32_t *n_proc, double *m_stop, double *m_face,
               const float *dL_dimage, double *dv, double *dsigma, double *drgb,
               double *face_margin, int64_t *counters, double *depth, double *m_depth,
               double *bnd_rgb, double *bnd_sigma, double *bnd_dv);

/* Chain ray-space gradients to the world features (+= into SoA fp64 gradients with the
 * same layout as the features).  Primitives with flag != 0 receive nothing.
 * exact = 1: dv are camera-space vertex gradients (render with cfg.exact = 1). */
int lpo_preprocess_bwd(const lpo_scene *s, const lpo_camera *cam, const lpo_pre *pre, int32_t exact,
                       const double *den_override, const double *dv, const double *dsigma,
                       const double *drgb, double *g_pos, double *g_rot, double *g_dist,
                       double *g_opacity, double *g_sh);

/* exported for the pins only: 3-D Moller-Trumbore of the ray t r (origin 0) against triangle
 * (A, B, C); out = (u, v, det, t); and d t / d(A, B, C) [3][3]. */
int lpo_mtia3(const double *A, const double *B, const double *C, const double *r, double *out);
void lpo_mtia3_grad(const double *A, const double *B, const double *C, const double *r, double *dt);

#ifdef __cplusplus
}
#endif
#endif
