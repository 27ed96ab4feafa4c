// lp_loss.cu -- f1: the 3DGS training loss L = (1 - lam) L1 + lam (1 - SSIM) and its image gradient
// in ONE kernel (reading 25).
//
// SSIM uses an 11 x 11 Gaussian window (sigma 1.5) with zero padding.  With m = w*x, e = w*(xx),
// w* the zero-padded window sum, the map S depends on x through m_x, e_xx, e_xy only, and
//   dL/dx = scale [(1 - lam) sign(x - y) - lam (w*G_m + y w*G_xy + 2 x w*G_xx)]
//   G_m = 2 m_y (A2 - A1)/(B1 B2) - 2 m_x S (1/B1 - 1/B2),  G_xy = 2 A1/(B1 B2),  G_xx = -S/B2
// (the window is symmetric, so the adjoint of w* is w*).  A CTA owns a 32 x 32 core tile of one
// (image, channel) plane: it stages x and y with a 10-pixel halo in shared memory, runs the
// separable window (horizontal then vertical, register-blocked along the sliding direction) for
// the five products on the 42 x 42 region the core's gradient needs, forms S and the three G maps
// there (zero outside the image), runs the window again on the G maps for the core and writes
// dL/dx.  HBM traffic is the minimum 12 B per pixel-channel (read x, y; write dL/dx); the kernel
// is FP32-FMA bound (~290 FMA per pixel-channel).
#include <cuda_runtime.h>
#include <math.h>
#include <stdint.h>

#include "lp_kernels.h"
#include "lp_x2.cuh"

namespace lp {

namespace {
constexpr int TS = 32;               // core tile
constexpr int RAD = 5;               // window radius
constexpr int TAPS = 2 * RAD + 1;
constexpr int RA = TS + 2 * RAD;     // 42: region of S / G maps the core gradient needs
constexpr int RI = TS + 4 * RAD;     // 52: input region
constexpr int LT = 384;              // threads
constexpr float C1 = 0.01f * 0.01f, C2 = 0.03f * 0.03f;

struct Win {
  float g[TAPS];
};

struct LossSmem {
  float2 xy[RI][RI + 1];             // (x, y) pairs of the input region
  union {
    struct {
      float2 h01[RI][RA];            // stage 2: horizontal sums of (x, y)
      float2 h23[RI][RA];            //          (xx, yy)
      float h4[RI][RA];              //          xy
    } a;
    struct {
      float2 h01[RA][TS];            // stage 4: horizontal sums of (G_m, G_xy)
      float h2[RA][TS];              //          G_xx
    } b;
  } u;
  float2 g01[RA][RA + 1];            // (G_m, G_xy)
  float g2[RA][RA + 1];              // G_xx
  float red[LT / 32];
};
}  // namespace

// The window sums run on (x, y) and (xx, yy) as FFMA2 pairs (one instruction for two maps) and
// on xy as a scalar FFMA; pass 2 pairs (G_m, G_xy) and runs G_xx scalar.
__global__ void __launch_bounds__(LT, 2) k_loss_ssim(const float *__restrict__ img, const float *__restrict__ tgt,
                                                     float *__restrict__ dL, float *__restrict__ loss_sum, int H,
                                                     int W, int tiles_x, float lam, float scale, Win win) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  LossSmem &S = *reinterpret_cast<LossSmem *>(smem_raw);
  const int tid = threadIdx.x;
  const int tile = blockIdx.x;
  const int tx0 = (tile % tiles_x) * TS, ty0 = (tile / tiles_x) * TS;
  const size_t plane = (size_t)blockIdx.y * H * W;
  const float *X = img + plane, *Y = tgt + plane;
  float *D = dL + plane;

  // ---- stage 1: (x, y) on the 52 x 52 input region (zero outside the image); warp w loads rows
  // w, w + 12, ..., lanes the columns; all loads issued before the shared-memory stores
  {
    const int lane = tid & 31, warp = tid >> 5;
    constexpr int NW = LT / 32, NR = (RI + NW - 1) / NW;   // 5 row passes
    float ax[NR][2], ay[NR][2];
#pragma unroll
    for (int q = 0; q < NR; ++q) {
      const int r = warp + NW * q;
      const int gy = ty0 - 2 * RAD + r;
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int c = lane + 32 * h;
        const int gx = tx0 - 2 * RAD + c;
        const bool in = r < RI && c < RI && gy >= 0 && gy < H && gx >= 0 && gx < W;
        ax[q][h] = in ? __ldg(X + (size_t)gy * W + gx) : 0.f;
        ay[q][h] = in ? __ldg(Y + (size_t)gy * W + gx) : 0.f;
      }
    }
#pragma unroll
    for (int q = 0; q < NR; ++q) {
      const int r = warp + NW * q;
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int c = lane + 32 * h;
        if (r < RI && c < RI) S.xy[r][c] = make_float2(ax[q][h], ay[q][h]);
      }
    }
  }
  __syncthreads();

  // ---- stage 2: horizontal window sums of the five products, 52 rows x 42 cols, 6 cols per item
  {
    constexpr int CH = 6, NCH = RA / CH;   // 7 chunks per row
    for (int it = tid; it < RI * NCH; it += LT) {
      const int r = it / NCH, c0 = (it % NCH) * CH;
      float2 a01[CH], a23[CH];
      float a4[CH];
#pragma unroll
      for (int j = 0; j < CH; ++j) {
        a01[j] = a23[j] = make_float2(0.f, 0.f);
        a4[j] = 0.f;
      }
#pragma unroll
      for (int k = 0; k < CH + TAPS - 1; ++k) {
        const float2 v01 = S.xy[r][c0 + k];
        const float2 v23 = fmul2(v01, v01);
        const float v4 = v01.x * v01.y;
#pragma unroll
        for (int j = 0; j < CH; ++j) {
          const int t = k - j;
          if (t >= 0 && t < TAPS) {
            a01[j] = ffma2(bc(win.g[t]), v01, a01[j]);
            a23[j] = ffma2(bc(win.g[t]), v23, a23[j]);
            a4[j] = fmaf(win.g[t], v4, a4[j]);
          }
        }
      }
#pragma unroll
      for (int j = 0; j < CH; ++j) {
        S.u.a.h01[r][c0 + j] = a01[j];
        S.u.a.h23[r][c0 + j] = a23[j];
        S.u.a.h4[r][c0 + j] = a4[j];
      }
    }
  }
  __syncthreads();

  // ---- stage 3: vertical sums -> statistics -> S and the G maps on the 42 x 42 region
  float lsum = 0.f;
  {
    constexpr int CH = 6, NCH = RA / CH;   // 7 row chunks per column
    for (int it = tid; it < RA * NCH; it += LT) {
      const int c = it % RA, r0 = (it / RA) * CH;
      float2 a01[CH], a23[CH];
      float a4[CH];
#pragma unroll
      for (int j = 0; j < CH; ++j) {
        a01[j] = a23[j] = make_float2(0.f, 0.f);
        a4[j] = 0.f;
      }
#pragma unroll
      for (int k = 0; k < CH + TAPS - 1; ++k) {
        const float2 v01 = S.u.a.h01[r0 + k][c], v23 = S.u.a.h23[r0 + k][c];
        const float v4 = S.u.a.h4[r0 + k][c];
#pragma unroll
        for (int j = 0; j < CH; ++j) {
          const int t = k - j;
          if (t >= 0 && t < TAPS) {
            a01[j] = ffma2(bc(win.g[t]), v01, a01[j]);
            a23[j] = ffma2(bc(win.g[t]), v23, a23[j]);
            a4[j] = fmaf(win.g[t], v4, a4[j]);
          }
        }
      }
#pragma unroll
      for (int j = 0; j < CH; ++j) {
        const int r = r0 + j;
        const int gy = ty0 - RAD + r, gx = tx0 - RAD + c;
        float gmv = 0.f, gxy = 0.f, gxx = 0.f;
        if (gy >= 0 && gy < H && gx >= 0 && gx < W) {
          const float mx = a01[j].x, my = a01[j].y;
          const float vx = a23[j].x - mx * mx, vy = a23[j].y - my * my, cxy = a4[j] - mx * my;
          const float A1 = 2.f * mx * my + C1, A2 = 2.f * cxy + C2;
          const float B1 = mx * mx + my * my + C1, B2 = vx + vy + C2;
          const float iB1 = __fdividef(1.f, B1), iB2 = __fdividef(1.f, B2);   // B1, B2 >= C1, C2 > 0
          const float ssim = A1 * A2 * iB1 * iB2;
          gmv = 2.f * my * (A2 - A1) * iB1 * iB2 - 2.f * mx * ssim * (iB1 - iB2);
          gxy = 2.f * A1 * iB1 * iB2;
          gxx = -ssim * iB2;
          if (r >= RAD && r < RAD + TS && c >= RAD && c < RAD + TS) lsum += lam * (1.f - ssim);
        }
        S.g01[r][c] = make_float2(gmv, gxy);
        S.g2[r][c] = gxx;
      }
    }
  }
  __syncthreads();

  // ---- stage 4: horizontal window sums of the G maps, 42 rows x 32 core cols, 4 cols per item
  {
    constexpr int CH = 4, NCH = TS / CH;   // 8
    for (int it = tid; it < RA * NCH; it += LT) {
      const int r = it / NCH, c0 = (it % NCH) * CH;
      float2 a01[CH];
      float a2[CH];
#pragma unroll
      for (int j = 0; j < CH; ++j) {
        a01[j] = make_float2(0.f, 0.f);
        a2[j] = 0.f;
      }
#pragma unroll
      for (int k = 0; k < CH + TAPS - 1; ++k) {
        const float2 v01 = S.g01[r][c0 + k];
        const float v2 = S.g2[r][c0 + k];
#pragma unroll
        for (int j = 0; j < CH; ++j) {
          const int t = k - j;
          if (t >= 0 && t < TAPS) {
            a01[j] = ffma2(bc(win.g[t]), v01, a01[j]);
            a2[j] = fmaf(win.g[t], v2, a2[j]);
          }
        }
      }
#pragma unroll
      for (int j = 0; j < CH; ++j) {
        S.u.b.h01[r][c0 + j] = a01[j];
        S.u.b.h2[r][c0 + j] = a2[j];
      }
    }
  }
  __syncthreads();

  // ---- stage 5: vertical sums on the core, combine with L1, write dL/dx; 4 rows per item
  {
    constexpr int CH = 4, NCH = TS / CH;   // 8
    for (int it = tid; it < TS * NCH; it += LT) {
      const int c = it % TS, r0 = (it / TS) * CH;
      float2 a01[CH];
      float a2[CH];
#pragma unroll
      for (int j = 0; j < CH; ++j) {
        a01[j] = make_float2(0.f, 0.f);
        a2[j] = 0.f;
      }
#pragma unroll
      for (int k = 0; k < CH + TAPS - 1; ++k) {
        const float2 v01 = S.u.b.h01[r0 + k][c];
        const float v2 = S.u.b.h2[r0 + k][c];
#pragma unroll
        for (int j = 0; j < CH; ++j) {
          const int t = k - j;
          if (t >= 0 && t < TAPS) {
            a01[j] = ffma2(bc(win.g[t]), v01, a01[j]);
            a2[j] = fmaf(win.g[t], v2, a2[j]);
          }
        }
      }
#pragma unroll
      for (int j = 0; j < CH; ++j) {
        const int gy = ty0 + r0 + j, gx = tx0 + c;
        if (gy < H && gx < W) {
          const float2 p = S.xy[r0 + j + 2 * RAD][c + 2 * RAD];
          const float d = p.x - p.y;
          const float sg = (float)((d > 0.f) - (d < 0.f));
          const float dS = a01[j].x + p.y * a01[j].y + 2.f * p.x * a2[j];
          D[(size_t)gy * W + gx] = scale * ((1.f - lam) * sg - lam * dS);
          lsum += (1.f - lam) * fabsf(d);
        }
      }
    }
  }

  // ---- loss: scale * sum over the core of (1 - lam)|x - y| + lam (1 - S)
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) lsum += __shfl_xor_sync(0xffffffffu, lsum, o);
  if ((tid & 31) == 0) S.red[tid >> 5] = lsum;
  __syncthreads();
  if (tid == 0) {
    float t = 0.f;
#pragma unroll
    for (int w = 0; w < LT / 32; ++w) t += S.red[w];
    atomicAdd(loss_sum, scale * t);
  }
}

void launch_loss_ssim(const float *img, const float *tgt, float *dL, float *loss_sum, int n_planes, int H, int W,
                      float lam, float scale, cudaStream_t st) {
  if (n_planes <= 0 || H <= 0 || W <= 0) return;
  Win win;
  double g[TAPS], s = 0.0;
  for (int k = 0; k < TAPS; ++k) {
    g[k] = exp(-(double)((k - RAD) * (k - RAD)) / (2.0 * 1.5 * 1.5));
    s += g[k];
  }
  for (int k = 0; k < TAPS; ++k) win.g[k] = (float)(g[k] / s);
  const int tiles_x = (W + TS - 1) / TS, tiles_y = (H + TS - 1) / TS;
  const size_t smem = sizeof(LossSmem);
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(k_loss_ssim, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    attr = true;
  }
  dim3 grid(tiles_x * tiles_y, n_planes);
  k_loss_ssim<<<grid, LT, smem, st>>>(img, tgt, dL, loss_sum, H, W, tiles_x, lam, scale, win);
}

}  // namespace lp
