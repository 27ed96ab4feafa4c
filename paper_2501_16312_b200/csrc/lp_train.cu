// lp_train.cu -- C5 helpers: L1 loss gradient and fused multi-group Adam.
// Both are HBM-bound elementwise kernels: float4 vectorised, grid-stride over 148 x k CTAs.
#include <cuda_runtime.h>
#include <stdint.h>

#include "lp_kernels.h"

namespace lp {

__global__ void __launch_bounds__(256) k_l1_grad(const float *__restrict__ img, const float *__restrict__ tgt,
                                                 float *__restrict__ dL, float *__restrict__ loss, int64_t n,
                                                 float scale) {
  float s = 0.f;
  const int64_t n4 = n / 4;
  const float4 *i4 = reinterpret_cast<const float4 *>(img);
  const float4 *t4 = reinterpret_cast<const float4 *>(tgt);
  float4 *d4 = reinterpret_cast<float4 *>(dL);
  const bool vec = ((reinterpret_cast<uintptr_t>(img) | reinterpret_cast<uintptr_t>(tgt) |
                     reinterpret_cast<uintptr_t>(dL)) & 15) == 0;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  int64_t i0 = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (vec) {
    for (int64_t i = i0; i < n4; i += stride) {
      const float4 a = i4[i], b = t4[i];
      const float dx = a.x - b.x, dy = a.y - b.y, dz = a.z - b.z, dw = a.w - b.w;
      s += fabsf(dx) + fabsf(dy) + fabsf(dz) + fabsf(dw);
      d4[i] = make_float4(scale * (float)((dx > 0.f) - (dx < 0.f)), scale * (float)((dy > 0.f) - (dy < 0.f)),
                          scale * (float)((dz > 0.f) - (dz < 0.f)), scale * (float)((dw > 0.f) - (dw < 0.f)));
    }
    i0 += n4 * 4;   // tail handled below
    for (int64_t i = n4 * 4 + (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride) {
      const float d = img[i] - tgt[i];
      s += fabsf(d);
      dL[i] = scale * (float)((d > 0.f) - (d < 0.f));
    }
  } else {
    for (int64_t i = i0; i < n; i += stride) {
      const float d = img[i] - tgt[i];
      s += fabsf(d);
      dL[i] = scale * (float)((d > 0.f) - (d < 0.f));
    }
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
  __shared__ float sw[8];
  if ((threadIdx.x & 31) == 0) sw[threadIdx.x >> 5] = s;
  __syncthreads();
  if (threadIdx.x == 0) {
    float t = 0.f;
    for (int w = 0; w < (int)(blockDim.x >> 5); ++w) t += sw[w];
    atomicAdd(loss, scale * t);
  }
}

void launch_l1_grad(const float *img, const float *tgt, float *dL, float *loss, int64_t n, float scale,
                    cudaStream_t st) {
  if (n <= 0) return;
  const int64_t want = (n / 4 + 255) / 256;
  const int grid = (int)(want < 148 * 8 ? (want > 0 ? want : 1) : 148 * 8);
  k_l1_grad<<<grid, 256, 0, st>>>(img, tgt, dL, loss, n, scale);
}

// ---------------------------------------------------------------------------------------------
// f4: 3D smoothing filter size from the training cameras (#26).
// One thread per primitive; the cameras are staged through shared memory 64 at a time.
__global__ void __launch_bounds__(256) k_filter3d(const float *__restrict__ pos, int n,
                                                  const lp_camera *__restrict__ cams, int nc, float kappa,
                                                  float *__restrict__ out) {
  __shared__ lp_camera s_cam[64];
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  float c[3] = {0.f, 0.f, 0.f};
  if (i < n) {
    c[0] = pos[i];
    c[1] = pos[n + i];
    c[2] = pos[2 * n + i];
  }
  float best = INFINITY, near_d = INFINITY, near_v = 0.f;
  for (int c0 = 0; c0 < nc; c0 += 64) {
    const int m = nc - c0 < 64 ? nc - c0 : 64;
    __syncthreads();
    if (threadIdx.x < m) s_cam[threadIdx.x] = cams[c0 + threadIdx.x];
    __syncthreads();
    for (int v = 0; v < m; ++v) {
      const lp_camera &cam = s_cam[v];
      float p[3];
#pragma unroll
      for (int r = 0; r < 3; ++r)
        p[r] = fmaf(cam.W[3 * r + 2], c[2], fmaf(cam.W[3 * r + 1], c[1], fmaf(cam.W[3 * r], c[0], cam.t[r])));
      if (p[2] > cam.znear) {
        const float u = fmaf(cam.fx, p[0] / p[2], cam.cx), w = fmaf(cam.fy, p[1] / p[2], cam.cy);
        if (u >= 0.f && u <= (float)cam.width && w >= 0.f && w <= (float)cam.height) best = fminf(best, p[2] / cam.fx);
      }
      const float d = sqrtf(fmaf(p[0], p[0], fmaf(p[1], p[1], p[2] * p[2])));
      if (d < near_d) {
        near_d = d;
        near_v = d / cam.fx;
      }
    }
  }
  if (i < n) out[i] = kappa * (best < INFINITY ? best : near_v);
}

void launch_filter3d(const float *pos, int n, const lp_camera *cams, int nc, float kappa, float *out,
                     cudaStream_t st) {
  if (n <= 0) return;
  k_filter3d<<<(n + 255) / 256, 256, 0, st>>>(pos, n, cams, nc, kappa, out);
}

// ---------------------------------------------------------------------------------------------
// C5: fused Adam over the flat parameter buffer, one CTA per ADAM_TILE-element tile of a
// group.  The bias corrections are folded on the host (the textbook update
//   p -= lr (m / bc1) / (sqrt(v / bc2) + eps)  ==  p -= step m / (sqrt(v) + eps_hat)
// with step = lr sqrt(bc2) / bc1 and eps_hat = eps sqrt(bc2), bc_i = 1 - beta_i^t), so an element
// costs 2 FFMA + 2 FMUL + sqrt + reciprocal.  Tiles never straddle groups: the float4 body covers
// the tile's 16-byte aligned part and threads 0-2 take its (at most 3 + 3) ragged elements.
constexpr int ADAM_THREADS = 256;
constexpr int ADAM_VEC = 4;                                   // float4 per thread per tile
constexpr int64_t ADAM_TILE = (int64_t)ADAM_THREADS * ADAM_VEC * 4;

struct AdamGroups {
  int64_t begin[8], end[8], tile0[9];                         // tile0: first tile of each group (prefix)
  float step[8], eps_hat[8];
  int n;
};

__device__ __forceinline__ float adam_elem(float p, float g, float &m, float &v, float b1, float b2, float om1,
                                           float om2, float step, float eps_hat) {
  m = fmaf(b1, m, om1 * g);
  v = fmaf(b2, v, om2 * g * g);
  return fmaf(-step, __fdividef(m, sqrtf(v) + eps_hat), p);
}

__global__ void __launch_bounds__(ADAM_THREADS) k_adam(float *__restrict__ p, float *__restrict__ g,
                                                       float *__restrict__ m, float *__restrict__ v,
                                                       const AdamGroups G, float b1, float b2, bool zero_grad) {
  const int64_t tile = blockIdx.x;
  int gi = 0;
  while (gi + 1 < G.n && tile >= G.tile0[gi + 1]) ++gi;       // block-uniform, <= 7 compares
  const int64_t b = G.begin[gi] + (tile - G.tile0[gi]) * ADAM_TILE;
  const int64_t e = min(b + ADAM_TILE, G.end[gi]);
  // 1 - beta is exact in fp32 for beta in [0.5, 1] (Sterbenz): the complement of the caller's fp32 beta
  const float step = G.step[gi], eh = G.eps_hat[gi], om1 = 1.f - b1, om2 = 1.f - b2;
  const int64_t b4 = (b + 3) & ~int64_t(3), e4 = e & ~int64_t(3);
  if (b4 < e4) {
    const int64_t q0 = b4 >> 2, nq = (e4 - b4) >> 2;
    float4 *p4 = reinterpret_cast<float4 *>(p) + q0, *g4 = reinterpret_cast<float4 *>(g) + q0;
    float4 *m4 = reinterpret_cast<float4 *>(m) + q0, *v4 = reinterpret_cast<float4 *>(v) + q0;
    float4 pp[ADAM_VEC], gg[ADAM_VEC], mm[ADAM_VEC], vv[ADAM_VEC];
#pragma unroll
    for (int k = 0; k < ADAM_VEC; ++k) {                     // all loads in flight first
      const int64_t i = threadIdx.x + (int64_t)k * ADAM_THREADS;
      if (i < nq) {
        pp[k] = p4[i];
        gg[k] = g4[i];
        mm[k] = m4[i];
        vv[k] = v4[i];
      }
    }
#pragma unroll
    for (int k = 0; k < ADAM_VEC; ++k) {
      const int64_t i = threadIdx.x + (int64_t)k * ADAM_THREADS;
      if (i < nq) {
        pp[k].x = adam_elem(pp[k].x, gg[k].x, mm[k].x, vv[k].x, b1, b2, om1, om2, step, eh);
        pp[k].y = adam_elem(pp[k].y, gg[k].y, mm[k].y, vv[k].y, b1, b2, om1, om2, step, eh);
        pp[k].z = adam_elem(pp[k].z, gg[k].z, mm[k].z, vv[k].z, b1, b2, om1, om2, step, eh);
        pp[k].w = adam_elem(pp[k].w, gg[k].w, mm[k].w, vv[k].w, b1, b2, om1, om2, step, eh);
        p4[i] = pp[k];
        m4[i] = mm[k];
        v4[i] = vv[k];
        if (zero_grad) g4[i] = make_float4(0.f, 0.f, 0.f, 0.f);
      }
    }
  }
  // ragged elements: [b, b4) and [e4, e) when the tile has an aligned body, else all of [b, e)
  int64_t i = -1;
  const int t = threadIdx.x;
  if (b4 < e4) {
    if (t < 3) i = b + t < b4 ? b + t : -1;
    else if (t < 6) i = e4 + (t - 3) < e ? e4 + (t - 3) : -1;
  } else if (t < 6) {
    i = b + t < e ? b + t : -1;
  }
  if (i >= 0) {
    float mm = m[i], vv = v[i];
    p[i] = adam_elem(p[i], g[i], mm, vv, b1, b2, om1, om2, step, eh);
    m[i] = mm;
    v[i] = vv;
    if (zero_grad) g[i] = 0.f;
  }
}

void launch_adam(float *p, float *g, float *m, float *v, const lp_adam_group *groups, int ng, float b1, float b2,
                 float eps, int step, bool zero_grad, cudaStream_t st) {
  // bias corrections in double on the host (Kingma & Ba, Alg. 1)
  const double bc1 = 1.0 - pow((double)b1, (double)step), bc2 = 1.0 - pow((double)b2, (double)step);
  for (int base = 0; base < ng; base += 8) {
    AdamGroups G;
    G.n = 0;
    int64_t tiles = 0;
    for (int k = 0; k < 8 && base + k < ng; ++k) {
      const lp_adam_group &gr = groups[base + k];
      if (gr.end <= gr.begin) continue;
      G.begin[G.n] = gr.begin;
      G.end[G.n] = gr.end;
      G.tile0[G.n] = tiles;
      G.step[G.n] = (float)((double)gr.lr * sqrt(bc2) / bc1);
      G.eps_hat[G.n] = (float)((double)eps * sqrt(bc2));
      tiles += (gr.end - gr.begin + ADAM_TILE - 1) / ADAM_TILE;
      ++G.n;
    }
    if (G.n == 0) continue;
    G.tile0[G.n] = tiles;
    k_adam<<<(unsigned)tiles, ADAM_THREADS, 0, st>>>(p, g, m, v, G, b1, b2, zero_grad);
  }
}

// 8-bit target channels -> fp32 in [0, 1] (16 bytes per thread per iteration)
__global__ void __launch_bounds__(256) k_image_from_u8(const uint8_t *__restrict__ src, float *__restrict__ dst,
                                                       int64_t n) {
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  const bool vec = ((reinterpret_cast<uintptr_t>(src) | reinterpret_cast<uintptr_t>(dst)) & 15) == 0;
  int64_t done = 0;
  if (vec) {
    const int64_t n16 = n / 16;
    const uint4 *s4 = reinterpret_cast<const uint4 *>(src);
    float4 *d4 = reinterpret_cast<float4 *>(dst);
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n16; i += stride) {
      const uint4 w = s4[i];
      const uint32_t ww[4] = {w.x, w.y, w.z, w.w};
#pragma unroll
      for (int q = 0; q < 4; ++q)
        d4[4 * i + q] = make_float4(__fdiv_rn((float)(ww[q] & 0xFFu), 255.f), __fdiv_rn((float)((ww[q] >> 8) & 0xFFu), 255.f),
                                    __fdiv_rn((float)((ww[q] >> 16) & 0xFFu), 255.f), __fdiv_rn((float)(ww[q] >> 24), 255.f));
    }
    done = n16 * 16;
  }
  for (int64_t i = done + (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride)
    dst[i] = __fdiv_rn((float)src[i], 255.f);
}

void launch_image_from_u8(const uint8_t *src, float *dst, int64_t n, cudaStream_t st) {
  if (n <= 0) return;
  const int64_t want = (n / 16 + 255) / 256;
  const int grid = (int)(want < 148 * 8 ? (want > 0 ? want : 1) : 148 * 8);
  k_image_from_u8<<<grid, 256, 0, st>>>(src, dst, n);
}

}  // namespace lp
