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

struct AdamGroups {
  int64_t begin[8], end[8];
  float lr[8];
  int n;
};

__global__ void __launch_bounds__(256) k_adam(float *__restrict__ p, float *__restrict__ g, float *__restrict__ m,
                                              float *__restrict__ v, AdamGroups G, float b1, float b2, float eps,
                                              float bc1, float bc2, bool zero_grad) {
  const int gi = blockIdx.y;
  const int64_t b = G.begin[gi], e = G.end[gi];
  const float lr = G.lr[gi];
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  const int64_t tid = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  auto upd = [&](float pp, float gg, float &mm, float &vv) {
    mm = fmaf(b1, mm, (1.f - b1) * gg);
    vv = fmaf(b2, vv, (1.f - b2) * gg * gg);
    return pp - lr * (mm / bc1) / (sqrtf(vv / bc2) + eps);
  };
  // float4 body over the 16-byte aligned part of [b, e), scalar head / tail
  const int64_t b4 = (b + 3) & ~int64_t(3), e4 = e & ~int64_t(3);
  if (b4 < e4) {
    float4 *p4 = reinterpret_cast<float4 *>(p + b4), *g4 = reinterpret_cast<float4 *>(g + b4);
    float4 *m4 = reinterpret_cast<float4 *>(m + b4), *v4 = reinterpret_cast<float4 *>(v + b4);
    const int64_t n4 = (e4 - b4) / 4;
    for (int64_t i = tid; i < n4; i += stride) {
      float4 pp = p4[i], gg = g4[i], mm = m4[i], vv = v4[i];
      pp.x = upd(pp.x, gg.x, mm.x, vv.x);
      pp.y = upd(pp.y, gg.y, mm.y, vv.y);
      pp.z = upd(pp.z, gg.z, mm.z, vv.z);
      pp.w = upd(pp.w, gg.w, mm.w, vv.w);
      p4[i] = pp;
      m4[i] = mm;
      v4[i] = vv;
      if (zero_grad) g4[i] = make_float4(0.f, 0.f, 0.f, 0.f);
    }
  }
  const int64_t head_end = b4 < e ? b4 : e;
  for (int64_t i = b + tid; i < head_end; i += stride) {
    float mm = m[i], vv = v[i];
    p[i] = upd(p[i], g[i], mm, vv);
    m[i] = mm;
    v[i] = vv;
    if (zero_grad) g[i] = 0.f;
  }
  for (int64_t i = (e4 > b ? (e4 > head_end ? e4 : head_end) : e) + tid; i < e; i += stride) {
    float mm = m[i], vv = v[i];
    p[i] = upd(p[i], g[i], mm, vv);
    m[i] = mm;
    v[i] = vv;
    if (zero_grad) g[i] = 0.f;
  }
}

// grid cap of the Adam kernel: blocks per SM and group (-DLP_ADAM_BPSM overrides)
#ifndef LP_ADAM_BPSM
#define LP_ADAM_BPSM 8
#endif
void launch_adam(float *p, float *g, float *m, float *v, const lp_adam_group *groups, int ng, float b1, float b2,
                 float eps, int step, bool zero_grad, cudaStream_t st) {
  for (int base = 0; base < ng; base += 8) {
    AdamGroups G;
    G.n = ng - base < 8 ? ng - base : 8;
    int64_t longest = 1;
    for (int k = 0; k < G.n; ++k) {
      G.begin[k] = groups[base + k].begin;
      G.end[k] = groups[base + k].end;
      G.lr[k] = groups[base + k].lr;
      if (G.end[k] - G.begin[k] > longest) longest = G.end[k] - G.begin[k];
    }
    for (int k = G.n; k < 8; ++k) { G.begin[k] = G.end[k] = 0; G.lr[k] = 0.f; }
    const float bc1 = 1.f - powf(b1, (float)step), bc2 = 1.f - powf(b2, (float)step);
    const int64_t want = (longest / 4 + 255) / 256 + 1;
    const int gx = (int)(want < 148 * LP_ADAM_BPSM ? want : 148 * LP_ADAM_BPSM);
    k_adam<<<dim3(gx, G.n), 256, 0, st>>>(p, g, m, v, G, b1, b2, eps, bc1, bc2, zero_grad);
  }
}

}  // namespace lp
