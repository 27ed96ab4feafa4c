// lp_loss.cu -- f1: the 3DGS training loss L = (1 - lam) L1 + lam (1 - SSIM) and its image gradient
// (reading 25): one fused kernel, or (given a workspace) the split pair
// k_ssim_maps + k_ssim_grad at the end of this file.
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
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>
#include <math.h>
#include <stdint.h>
#include <stdlib.h>

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
  // (g[t - 1], g[t]) for t = 0..TAPS (g outside [0, TAPS) is 0): the coefficient pair of two adjacent
  // outputs (o + 1, o) of the same input at tap t of output o, one FFMA2 for the scalar map's pair
  float2 gp[TAPS + 1];
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
  extern __shared__ __align__(128) unsigned char smem_raw[];
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


// ---------------------------------------------------------------------------------------------
// TMA-fed persistent variant (used when the image rows are 16-byte aligned, W % 4 == 0): one CTA
// loops over (plane, tile) work items; the x and y input boxes (10-pixel halo, zero fill outside
// the image done by the tensor-map OOB rule) arrive by cp.async.bulk.tensor into a double buffer,
// the next item's boxes in flight while the current one is computed.  The box starts 12 columns
// left of the tile (56 x 52): a TMA box's innermost start coordinate must be a multiple of
// 16 bytes when it is negative (measured: other negative x starts fault), so the 52-wide window
// sits at box column 2.
// ---------------------------------------------------------------------------------------------
namespace {
constexpr int BW = RI + 4;           // 56: box width (start 12 columns left of the tile)
constexpr int BX = 2;                // box column of window column 0
constexpr int BOXF = BW * RI;        // 2912 floats = 11648 B (a multiple of 128 B)
struct LossSmemT {
  float box[2][2][BOXF];             // [buffer][x | y]
  union {
    struct {
      float2 h01[RI][RA];
      float2 h23[RI][RA];
      float h4[RI][RA];
    } a;
    struct {
      float2 h01[RA][TS];
      float h2[RA][TS];
    } b;
  } u;
  float2 g01[RA][RA + 1];
  float g2[RA][RA + 1];
  unsigned long long bar[2];
  int meta[2][3];                    // per buffer: tile origin x, y and plane of the item it holds
  float red[LT / 32];
};

__device__ __forceinline__ uint32_t smem_u32(const void *p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(unsigned long long *bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}
__device__ __forceinline__ void mbar_expect_tx(unsigned long long *bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_wait(unsigned long long *bar, uint32_t parity) {
  asm volatile(
      "{\n\t.reg .pred p;\n"
      "WAIT_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
      "@!p bra WAIT_%=;\n}" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ void tma_load_3d(void *dst, const CUtensorMap *map, int c0, int c1, int c2,
                                            unsigned long long *bar) {
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], [%5];" ::"r"(
          smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(c2), "r"(smem_u32(bar))
      : "memory");
}
}  // namespace

__global__ void __launch_bounds__(LT, 2) k_loss_ssim_tma(const __grid_constant__ CUtensorMap map_x,
                                                         const __grid_constant__ CUtensorMap map_y,
                                                         float *__restrict__ dL, float *__restrict__ loss_sum, int H,
                                                         int W, int tiles_x, int tiles_per_plane, int items,
                                                         float lam, float scale, Win win) {
  extern __shared__ __align__(128) unsigned char smem_raw[];
  LossSmemT &S = *reinterpret_cast<LossSmemT *>(smem_raw);
  const int tid = threadIdx.x;
  constexpr uint32_t BOX_BYTES = BW * RI * 4;
  if (tid == 0) {
    mbar_init(&S.bar[0], 1);
    mbar_init(&S.bar[1], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  // (the item's tile origin and plane are computed once, by the issuing thread, and read from shared
  // memory by all: integer divisions by the runtime grid sizes were ~7 % of the instructions)
  auto issue = [&](int item, int buf) {
    const int plane = item / tiles_per_plane, tile = item % tiles_per_plane;
    const int tx0 = (tile % tiles_x) * TS, ty0 = (tile / tiles_x) * TS;
    S.meta[buf][0] = tx0;
    S.meta[buf][1] = ty0;
    S.meta[buf][2] = plane;
    mbar_expect_tx(&S.bar[buf], 2 * BOX_BYTES);
    tma_load_3d(S.box[buf][0], &map_x, tx0 - 2 * RAD - BX, ty0 - 2 * RAD, plane, &S.bar[buf]);
    tma_load_3d(S.box[buf][1], &map_y, tx0 - 2 * RAD - BX, ty0 - 2 * RAD, plane, &S.bar[buf]);
  };
  if (tid == 0 && (int)blockIdx.x < items) issue(blockIdx.x, 0);
  __syncthreads();   // the first item's metadata
  float lsum = 0.f;
  uint32_t phase[2] = {0u, 0u};
  int buf = 0;
  for (int item = blockIdx.x; item < items; item += gridDim.x, buf ^= 1) {
    if (tid == 0 && item + (int)gridDim.x < items) issue(item + gridDim.x, buf ^ 1);
    mbar_wait(&S.bar[buf], phase[buf]);
    phase[buf] ^= 1u;
    const float *X = S.box[buf][0], *Y = S.box[buf][1];
    const int tx0 = S.meta[buf][0], ty0 = S.meta[buf][1], plane = S.meta[buf][2];
    float *D = dL + (size_t)plane * H * W;

    // ---- stage 2: horizontal window sums of the five products, 52 rows x 42 cols
    {
      constexpr int CH = 6, NCH = RA / CH;
      for (int it = tid; it < RI * NCH; it += LT) {
        const int r = it / NCH, c0 = (it % NCH) * CH;
        float2 a01[CH], a23[CH], a4p[CH / 2];   // a4p[q] = xy sums of outputs (2q + 1, 2q)
#pragma unroll
        for (int j = 0; j < CH; ++j) a01[j] = a23[j] = make_float2(0.f, 0.f);
#pragma unroll
        for (int q = 0; q < CH / 2; ++q) a4p[q] = make_float2(0.f, 0.f);
#pragma unroll
        for (int k = 0; k < CH + TAPS - 1; ++k) {
          const float2 v01 = make_float2(X[r * BW + BX + c0 + k], Y[r * BW + BX + c0 + k]);
          const float2 v23 = fmul2(v01, v01);
          const float v4 = v01.x * v01.y;
#pragma unroll
          for (int j = 0; j < CH; ++j) {
            const int t = k - j;
            if (t >= 0 && t < TAPS) {
              a01[j] = ffma2(bc(win.g[t]), v01, a01[j]);
              a23[j] = ffma2(bc(win.g[t]), v23, a23[j]);
            }
          }
#pragma unroll
          for (int q = 0; q < CH / 2; ++q) {
            const int t = k - 2 * q;   // tap of output 2q (output 2q + 1 takes t - 1)
            if (t >= 0 && t <= TAPS) a4p[q] = ffma2(win.gp[t], bc(v4), a4p[q]);
          }
        }
#pragma unroll
        for (int j = 0; j < CH; ++j) {
          S.u.a.h01[r][c0 + j] = a01[j];
          S.u.a.h23[r][c0 + j] = a23[j];
          S.u.a.h4[r][c0 + j] = (j & 1) ? a4p[j / 2].x : a4p[j / 2].y;
        }
      }
    }
    __syncthreads();
    // ---- stage 3: vertical sums -> S and the G maps on the 42 x 42 region
    {
      constexpr int CH = 6, NCH = RA / CH;
      for (int it = tid; it < RA * NCH; it += LT) {
        const int c = it % RA, r0 = (it / RA) * CH;
        float2 a01[CH], a23[CH], a4p[CH / 2];   // a4p[q] = xy sums of rows (2q + 1, 2q)
#pragma unroll
        for (int j = 0; j < CH; ++j) a01[j] = a23[j] = make_float2(0.f, 0.f);
#pragma unroll
        for (int q = 0; q < CH / 2; ++q) a4p[q] = make_float2(0.f, 0.f);
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
            }
          }
#pragma unroll
          for (int q = 0; q < CH / 2; ++q) {
            const int t = k - 2 * q;
            if (t >= 0 && t <= TAPS) a4p[q] = ffma2(win.gp[t], bc(v4), a4p[q]);
          }
        }
        float a4[CH];
#pragma unroll
        for (int j = 0; j < CH; ++j) a4[j] = (j & 1) ? a4p[j / 2].x : a4p[j / 2].y;
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
            const float iB1 = __fdividef(1.f, B1), iB2 = __fdividef(1.f, B2);
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
    // ---- stage 4: horizontal window sums of the G maps
    {
      constexpr int CH = 4, NCH = TS / CH;
      for (int it = tid; it < RA * NCH; it += LT) {
        const int r = it / NCH, c0 = (it % NCH) * CH;
        float2 a01[CH], a2p[CH / 2];
#pragma unroll
        for (int j = 0; j < CH; ++j) a01[j] = make_float2(0.f, 0.f);
#pragma unroll
        for (int q = 0; q < CH / 2; ++q) a2p[q] = make_float2(0.f, 0.f);
#pragma unroll
        for (int k = 0; k < CH + TAPS - 1; ++k) {
          const float2 v01 = S.g01[r][c0 + k];
          const float v2 = S.g2[r][c0 + k];
#pragma unroll
          for (int j = 0; j < CH; ++j) {
            const int t = k - j;
            if (t >= 0 && t < TAPS) a01[j] = ffma2(bc(win.g[t]), v01, a01[j]);
          }
#pragma unroll
          for (int q = 0; q < CH / 2; ++q) {
            const int t = k - 2 * q;
            if (t >= 0 && t <= TAPS) a2p[q] = ffma2(win.gp[t], bc(v2), a2p[q]);
          }
        }
#pragma unroll
        for (int j = 0; j < CH; ++j) {
          S.u.b.h01[r][c0 + j] = a01[j];
          S.u.b.h2[r][c0 + j] = (j & 1) ? a2p[j / 2].x : a2p[j / 2].y;
        }
      }
    }
    __syncthreads();
    // ---- stage 5: vertical sums on the core, combine with L1, write dL/dx
    {
      constexpr int CH = 4, NCH = TS / CH;
      for (int it = tid; it < TS * NCH; it += LT) {
        const int c = it % TS, r0 = (it / TS) * CH;
        float2 a01[CH], a2p[CH / 2];
#pragma unroll
        for (int j = 0; j < CH; ++j) a01[j] = make_float2(0.f, 0.f);
#pragma unroll
        for (int q = 0; q < CH / 2; ++q) a2p[q] = make_float2(0.f, 0.f);
#pragma unroll
        for (int k = 0; k < CH + TAPS - 1; ++k) {
          const float2 v01 = S.u.b.h01[r0 + k][c];
          const float v2 = S.u.b.h2[r0 + k][c];
#pragma unroll
          for (int j = 0; j < CH; ++j) {
            const int t = k - j;
            if (t >= 0 && t < TAPS) a01[j] = ffma2(bc(win.g[t]), v01, a01[j]);
          }
#pragma unroll
          for (int q = 0; q < CH / 2; ++q) {
            const int t = k - 2 * q;
            if (t >= 0 && t <= TAPS) a2p[q] = ffma2(win.gp[t], bc(v2), a2p[q]);
          }
        }
        float a2[CH];
#pragma unroll
        for (int j = 0; j < CH; ++j) a2[j] = (j & 1) ? a2p[j / 2].x : a2p[j / 2].y;
#pragma unroll
        for (int j = 0; j < CH; ++j) {
          const int gy = ty0 + r0 + j, gx = tx0 + c;
          if (gy < H && gx < W) {
            const int bi = (r0 + j + 2 * RAD) * BW + BX + c + 2 * RAD;
            const float x = X[bi], y = Y[bi];
            const float d = x - y;
            const float sg = (float)((d > 0.f) - (d < 0.f));
            const float dS = a01[j].x + y * a01[j].y + 2.f * x * a2[j];
            D[(size_t)gy * W + gx] = scale * ((1.f - lam) * sg - lam * dS);
            lsum += (1.f - lam) * fabsf(d);
          }
        }
      }
    }
    __syncthreads();   // every thread is done with box[buf] and the stage buffers
  }
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


// ---------------------------------------------------------------------------------------------
// Split variant (two TMA-fed persistent kernels, with a workspace for the three G maps): the fused
// kernel above forms S and the G maps on the 42 x 42 region its core's gradient needs (the window
// sums of the five products on 52 x 42, halo included) -- 1.7x the core.  Here k_ssim_maps forms
// them on the 32 x 32 core only (window sums on 42 x 32) and stores G_m, G_xy, G_xx to the workspace;
// k_ssim_grad reads them back with their 5-pixel halo (zero outside the image: the tensor map's OOB
// fill, exactly the fused kernel's zero padding) and runs the window on them.  Every output is the
// same sequence of fp32 operations as in the fused kernel (bitwise the same dL/dx); the workspace
// round trip costs 24 B per pixel-channel of (mostly L2) traffic.
// ---------------------------------------------------------------------------------------------
namespace {
constexpr int SBW = 48;              // box width: columns tx0 - 8 .. tx0 + 39 (16-byte aligned start)
constexpr int SBX = 3;               // box column of window column 0 (tx0 - 5)
constexpr int SBF = SBW * RA;        // 2016 floats = 8064 B (63 x 128 B): rows ty0 - 5 .. ty0 + 36
#ifndef LP_SSIM_LT
#define LP_SSIM_LT 384
#endif
constexpr int SLT = LP_SSIM_LT;   // threads of the split kernels
#ifndef LP_SSIM_CHA
#define LP_SSIM_CHA 4        // outputs per thread of the horizontal (first) stage of the split kernels
#endif
#ifndef LP_SSIM_CHB
#define LP_SSIM_CHB 4        // outputs per thread of the vertical (second) stage
#endif
#ifndef LP_SSIM_MINB
#define LP_SSIM_MINB 3      // resident CTAs per SM of the split kernels (59 / 72 KB shared memory)
#endif
struct MapsSmem {
  float box[2][2][SBF];              // [buffer][x | y]
  float2 h01[RA][TS];                // horizontal window sums of (x, y) on the box rows, core columns
  float2 h23[RA][TS];                //                            (xx, yy)
  float h4[RA][TS];                  //                            xy
  unsigned long long bar[2];
  int meta[2][3];
  float red[SLT / 32];
};
struct GradSmem {
  float gbox[2][3][SBF];             // [buffer][G_m | G_xy | G_xx] with the 5-pixel halo
  float cbox[2][TS * TS];            // x | y of the current item's core (single buffer, own barrier)
  float2 h01[RA][TS];                // horizontal window sums of (G_m, G_xy)
  float h2[RA][TS];                  //                            G_xx
  unsigned long long bar[2], cbar;
  int meta[2][3];
  float red[SLT / 32];
};

__device__ __forceinline__ void block_loss_add(float lsum, float *red, float *loss_sum, float scale) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) lsum += __shfl_xor_sync(0xffffffffu, lsum, o);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = lsum;
  __syncthreads();
  if (threadIdx.x == 0) {
    float t = 0.f;
#pragma unroll
    for (int w = 0; w < SLT / 32; ++w) t += red[w];
    atomicAdd(loss_sum, scale * t);
  }
}
}  // namespace

// G maps (workspace [3][planes][H][W]: G_m, G_xy, G_xx) and the SSIM part of the loss
__global__ void __launch_bounds__(SLT, LP_SSIM_MINB) k_ssim_maps(const __grid_constant__ CUtensorMap map_x,
                                                      const __grid_constant__ CUtensorMap map_y,
                                                      float *__restrict__ gmaps, float *__restrict__ loss_sum, int H,
                                                      int W, int tiles_x, int tiles_per_plane, int items, float lam,
                                                      float scale, Win win) {
  extern __shared__ __align__(128) unsigned char smem_raw[];
  MapsSmem &S = *reinterpret_cast<MapsSmem *>(smem_raw);
  const int tid = threadIdx.x;
  constexpr uint32_t BOX_BYTES = SBF * 4;
  if (tid == 0) {
    mbar_init(&S.bar[0], 1);
    mbar_init(&S.bar[1], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  auto issue = [&](int item, int buf) {
    const int plane = item / tiles_per_plane, tile = item % tiles_per_plane;
    const int tx0 = (tile % tiles_x) * TS, ty0 = (tile / tiles_x) * TS;
    S.meta[buf][0] = tx0;
    S.meta[buf][1] = ty0;
    S.meta[buf][2] = plane;
    mbar_expect_tx(&S.bar[buf], 2 * BOX_BYTES);
    tma_load_3d(S.box[buf][0], &map_x, tx0 - RAD - SBX, ty0 - RAD, plane, &S.bar[buf]);
    tma_load_3d(S.box[buf][1], &map_y, tx0 - RAD - SBX, ty0 - RAD, plane, &S.bar[buf]);
  };
  if (tid == 0 && (int)blockIdx.x < items) issue(blockIdx.x, 0);
  __syncthreads();
  const size_t HW = (size_t)H * W, PHW = (size_t)(items / tiles_per_plane) * HW;
  float lsum = 0.f;
  uint32_t phase[2] = {0u, 0u};
  int buf = 0;
  for (int item = blockIdx.x; item < items; item += gridDim.x, buf ^= 1) {
    if (tid == 0 && item + (int)gridDim.x < items) issue(item + gridDim.x, buf ^ 1);
    mbar_wait(&S.bar[buf], phase[buf]);
    phase[buf] ^= 1u;
    const float *X = S.box[buf][0], *Y = S.box[buf][1];
    const int tx0 = S.meta[buf][0], ty0 = S.meta[buf][1], plane = S.meta[buf][2];
    // ---- horizontal window sums of the five products: 42 rows x the 32 core columns
    {
      constexpr int CH = LP_SSIM_CHA, NCH = TS / CH;
      for (int it = tid; it < RA * NCH; it += SLT) {
        const int r = it / NCH, c0 = (it % NCH) * CH;
        float2 a01[CH], a23[CH], a4p[CH / 2];   // a4p[q] = xy sums of outputs (2q + 1, 2q)
#pragma unroll
        for (int j = 0; j < CH; ++j) a01[j] = a23[j] = make_float2(0.f, 0.f);
#pragma unroll
        for (int q = 0; q < CH / 2; ++q) a4p[q] = make_float2(0.f, 0.f);
#pragma unroll
        for (int k = 0; k < CH + TAPS - 1; ++k) {
          const float2 v01 = make_float2(X[r * SBW + SBX + c0 + k], Y[r * SBW + SBX + c0 + k]);
          const float2 v23 = fmul2(v01, v01);
          const float v4 = v01.x * v01.y;
#pragma unroll
          for (int j = 0; j < CH; ++j) {
            const int t = k - j;
            if (t >= 0 && t < TAPS) {
              a01[j] = ffma2(bc(win.g[t]), v01, a01[j]);
              a23[j] = ffma2(bc(win.g[t]), v23, a23[j]);
            }
          }
#pragma unroll
          for (int q = 0; q < CH / 2; ++q) {
            const int t = k - 2 * q;
            if (t >= 0 && t <= TAPS) a4p[q] = ffma2(win.gp[t], bc(v4), a4p[q]);
          }
        }
#pragma unroll
        for (int j = 0; j < CH; ++j) {
          S.h01[r][c0 + j] = a01[j];
          S.h23[r][c0 + j] = a23[j];
          S.h4[r][c0 + j] = (j & 1) ? a4p[j / 2].x : a4p[j / 2].y;
        }
      }
    }
    __syncthreads();
    // ---- vertical sums -> S and the G maps on the core, stored to the workspace
    {
      constexpr int CH = LP_SSIM_CHB, NCH = TS / CH;
      for (int it = tid; it < TS * NCH; it += SLT) {
        const int c = it % TS, r0 = (it / TS) * CH;
        float2 a01[CH], a23[CH], a4p[CH / 2];
#pragma unroll
        for (int j = 0; j < CH; ++j) a01[j] = a23[j] = make_float2(0.f, 0.f);
#pragma unroll
        for (int q = 0; q < CH / 2; ++q) a4p[q] = make_float2(0.f, 0.f);
#pragma unroll
        for (int k = 0; k < CH + TAPS - 1; ++k) {
          const float2 v01 = S.h01[r0 + k][c], v23 = S.h23[r0 + k][c];
          const float v4 = S.h4[r0 + k][c];
#pragma unroll
          for (int j = 0; j < CH; ++j) {
            const int t = k - j;
            if (t >= 0 && t < TAPS) {
              a01[j] = ffma2(bc(win.g[t]), v01, a01[j]);
              a23[j] = ffma2(bc(win.g[t]), v23, a23[j]);
            }
          }
#pragma unroll
          for (int q = 0; q < CH / 2; ++q) {
            const int t = k - 2 * q;
            if (t >= 0 && t <= TAPS) a4p[q] = ffma2(win.gp[t], bc(v4), a4p[q]);
          }
        }
#pragma unroll
        for (int j = 0; j < CH; ++j) {
          const int gy = ty0 + r0 + j, gx = tx0 + c;
          if (gy < H && gx < W) {
            const float a4 = (j & 1) ? a4p[j / 2].x : a4p[j / 2].y;
            const float mx = a01[j].x, my = a01[j].y;
            const float vx = a23[j].x - mx * mx, vy = a23[j].y - my * my, cxy = a4 - mx * my;
            const float A1 = 2.f * mx * my + C1, A2 = 2.f * cxy + C2;
            const float B1 = mx * mx + my * my + C1, B2 = vx + vy + C2;
            const float iB1 = __fdividef(1.f, B1), iB2 = __fdividef(1.f, B2);
            const float ssim = A1 * A2 * iB1 * iB2;
            const size_t o = (size_t)plane * HW + (size_t)gy * W + gx;
            gmaps[o] = 2.f * my * (A2 - A1) * iB1 * iB2 - 2.f * mx * ssim * (iB1 - iB2);
            gmaps[PHW + o] = 2.f * A1 * iB1 * iB2;
            gmaps[2 * PHW + o] = -ssim * iB2;
            lsum += lam * (1.f - ssim);
          }
        }
      }
    }
    __syncthreads();   // every thread is done with box[buf] and the stage buffers
  }
  block_loss_add(lsum, S.red, loss_sum, scale);
}

// dL/dx from the G maps (window sums with their halo) and the L1 part of the loss
__global__ void __launch_bounds__(SLT, LP_SSIM_MINB) k_ssim_grad(const __grid_constant__ CUtensorMap map_gm,
                                                      const __grid_constant__ CUtensorMap map_gxy,
                                                      const __grid_constant__ CUtensorMap map_gxx,
                                                      const __grid_constant__ CUtensorMap map_cx,
                                                      const __grid_constant__ CUtensorMap map_cy,
                                                      float *__restrict__ dL, float *__restrict__ loss_sum, int H,
                                                      int W, int tiles_x, int tiles_per_plane, int items, float lam,
                                                      float scale, Win win) {
  extern __shared__ __align__(128) unsigned char smem_raw[];
  GradSmem &S = *reinterpret_cast<GradSmem *>(smem_raw);
  const int tid = threadIdx.x;
  constexpr uint32_t GBOX_BYTES = SBF * 4, CBOX_BYTES = TS * TS * 4;
  if (tid == 0) {
    mbar_init(&S.bar[0], 1);
    mbar_init(&S.bar[1], 1);
    mbar_init(&S.cbar, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  auto issue = [&](int item, int buf) {
    const int plane = item / tiles_per_plane, tile = item % tiles_per_plane;
    const int tx0 = (tile % tiles_x) * TS, ty0 = (tile / tiles_x) * TS;
    S.meta[buf][0] = tx0;
    S.meta[buf][1] = ty0;
    S.meta[buf][2] = plane;
    mbar_expect_tx(&S.bar[buf], 3 * GBOX_BYTES);
    tma_load_3d(S.gbox[buf][0], &map_gm, tx0 - RAD - SBX, ty0 - RAD, plane, &S.bar[buf]);
    tma_load_3d(S.gbox[buf][1], &map_gxy, tx0 - RAD - SBX, ty0 - RAD, plane, &S.bar[buf]);
    tma_load_3d(S.gbox[buf][2], &map_gxx, tx0 - RAD - SBX, ty0 - RAD, plane, &S.bar[buf]);
  };
  if (tid == 0 && (int)blockIdx.x < items) issue(blockIdx.x, 0);
  __syncthreads();
  float lsum = 0.f;
  uint32_t phase[2] = {0u, 0u}, cphase = 0u;
  int buf = 0;
  for (int item = blockIdx.x; item < items; item += gridDim.x, buf ^= 1) {
    if (tid == 0 && item + (int)gridDim.x < items) issue(item + gridDim.x, buf ^ 1);
    const int tx0 = S.meta[buf][0], ty0 = S.meta[buf][1], plane = S.meta[buf][2];
    if (tid == 0) {   // this item's core (x, y): needed by the last stage only
      mbar_expect_tx(&S.cbar, 2 * CBOX_BYTES);
      tma_load_3d(S.cbox[0], &map_cx, tx0, ty0, plane, &S.cbar);
      tma_load_3d(S.cbox[1], &map_cy, tx0, ty0, plane, &S.cbar);
    }
    mbar_wait(&S.bar[buf], phase[buf]);
    phase[buf] ^= 1u;
    const float *Gm = S.gbox[buf][0], *Gxy = S.gbox[buf][1], *Gxx = S.gbox[buf][2];
    float *D = dL + (size_t)plane * H * W;
    const float *X = S.cbox[0], *Y = S.cbox[1];
    // ---- horizontal window sums of the G maps: 42 rows x the 32 core columns
    {
      constexpr int CH = LP_SSIM_CHA, NCH = TS / CH;
      for (int it = tid; it < RA * NCH; it += SLT) {
        const int r = it / NCH, c0 = (it % NCH) * CH;
        float2 a01[CH], a2p[CH / 2];
#pragma unroll
        for (int j = 0; j < CH; ++j) a01[j] = make_float2(0.f, 0.f);
#pragma unroll
        for (int q = 0; q < CH / 2; ++q) a2p[q] = make_float2(0.f, 0.f);
#pragma unroll
        for (int k = 0; k < CH + TAPS - 1; ++k) {
          const int bi = r * SBW + SBX + c0 + k;
          const float2 v01 = make_float2(Gm[bi], Gxy[bi]);
          const float v2 = Gxx[bi];
#pragma unroll
          for (int j = 0; j < CH; ++j) {
            const int t = k - j;
            if (t >= 0 && t < TAPS) a01[j] = ffma2(bc(win.g[t]), v01, a01[j]);
          }
#pragma unroll
          for (int q = 0; q < CH / 2; ++q) {
            const int t = k - 2 * q;
            if (t >= 0 && t <= TAPS) a2p[q] = ffma2(win.gp[t], bc(v2), a2p[q]);
          }
        }
#pragma unroll
        for (int j = 0; j < CH; ++j) {
          S.h01[r][c0 + j] = a01[j];
          S.h2[r][c0 + j] = (j & 1) ? a2p[j / 2].x : a2p[j / 2].y;
        }
      }
    }
    __syncthreads();
    mbar_wait(&S.cbar, cphase);
    cphase ^= 1u;
    // ---- vertical sums on the core, combine with L1, write dL/dx
    {
      constexpr int CH = LP_SSIM_CHB, NCH = TS / CH;
      for (int it = tid; it < TS * NCH; it += SLT) {
        const int c = it % TS, r0 = (it / TS) * CH;
        float2 a01[CH], a2p[CH / 2];
#pragma unroll
        for (int j = 0; j < CH; ++j) a01[j] = make_float2(0.f, 0.f);
#pragma unroll
        for (int q = 0; q < CH / 2; ++q) a2p[q] = make_float2(0.f, 0.f);
#pragma unroll
        for (int k = 0; k < CH + TAPS - 1; ++k) {
          const float2 v01 = S.h01[r0 + k][c];
          const float v2 = S.h2[r0 + k][c];
#pragma unroll
          for (int j = 0; j < CH; ++j) {
            const int t = k - j;
            if (t >= 0 && t < TAPS) a01[j] = ffma2(bc(win.g[t]), v01, a01[j]);
          }
#pragma unroll
          for (int q = 0; q < CH / 2; ++q) {
            const int t = k - 2 * q;
            if (t >= 0 && t <= TAPS) a2p[q] = ffma2(win.gp[t], bc(v2), a2p[q]);
          }
        }
#pragma unroll
        for (int j = 0; j < CH; ++j) {
          const int gy = ty0 + r0 + j, gx = tx0 + c;
          if (gy < H && gx < W) {
            const float a2 = (j & 1) ? a2p[j / 2].x : a2p[j / 2].y;
            const float x = X[(r0 + j) * TS + c], y = Y[(r0 + j) * TS + c];
            const float d = x - y;
            const float sg = (float)((d > 0.f) - (d < 0.f));
            const float dS = a01[j].x + y * a01[j].y + 2.f * x * a2;
            D[(size_t)gy * W + gx] = scale * ((1.f - lam) * sg - lam * dS);
            lsum += (1.f - lam) * fabsf(d);
          }
        }
      }
    }
    __syncthreads();
  }
  block_loss_add(lsum, S.red, loss_sum, scale);
}

static bool make_box_map(CUtensorMap *map, const float *base, int planes, int H, int W, int bw = BW, int bh = RI) {
  static PFN_cuTensorMapEncodeTiled encode = nullptr;
  if (!encode) {
    cudaDriverEntryPointQueryResult q;
    void *fn = nullptr;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q) != cudaSuccess ||
        q != cudaDriverEntryPointSuccess || !fn) {
      cudaGetLastError();
      return false;
    }
    encode = reinterpret_cast<PFN_cuTensorMapEncodeTiled>(fn);
  }
  const cuuint64_t dims[3] = {(cuuint64_t)W, (cuuint64_t)H, (cuuint64_t)planes};
  const cuuint64_t strides[2] = {(cuuint64_t)W * 4, (cuuint64_t)W * H * 4};
  const cuuint32_t box[3] = {(cuuint32_t)bw, (cuuint32_t)bh, 1};
  const cuuint32_t estr[3] = {1, 1, 1};
  return encode(map, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 3, const_cast<float *>(base), dims, strides, box, estr,
                CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_128B,
                CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

void launch_loss_ssim(const float *img, const float *tgt, float *dL, float *loss_sum, int n_planes, int H, int W,
                      float lam, float scale, float *ws, cudaStream_t st) {
  if (n_planes <= 0 || H <= 0 || W <= 0) return;
  Win win;
  double g[TAPS], s = 0.0;
  for (int k = 0; k < TAPS; ++k) {
    g[k] = exp(-(double)((k - RAD) * (k - RAD)) / (2.0 * 1.5 * 1.5));
    s += g[k];
  }
  for (int k = 0; k < TAPS; ++k) win.g[k] = (float)(g[k] / s);
  for (int t = 0; t <= TAPS; ++t) win.gp[t] = make_float2(t >= 1 ? win.g[t - 1] : 0.f, t < TAPS ? win.g[t] : 0.f);
  const int tiles_x = (W + TS - 1) / TS, tiles_y = (H + TS - 1) / TS;
  // TMA path: rows 16-byte aligned (W % 4 == 0) and 16-byte aligned bases
  const bool aligned = (W % 4) == 0 && ((reinterpret_cast<uintptr_t>(img) | reinterpret_cast<uintptr_t>(tgt)) & 15) == 0;
  static const bool tma_off = getenv("LP_LOSS_NO_TMA") != nullptr;   // measurement knob
  CUtensorMap mx, my;
  if (ws && aligned && !tma_off && (reinterpret_cast<uintptr_t>(ws) & 15) == 0) {
    const size_t phw = (size_t)n_planes * H * W;
    CUtensorMap m[7];
    if (make_box_map(&m[0], img, n_planes, H, W, SBW, RA) && make_box_map(&m[1], tgt, n_planes, H, W, SBW, RA) &&
        make_box_map(&m[2], ws, n_planes, H, W, SBW, RA) && make_box_map(&m[3], ws + phw, n_planes, H, W, SBW, RA) &&
        make_box_map(&m[4], ws + 2 * phw, n_planes, H, W, SBW, RA) &&
        make_box_map(&m[5], img, n_planes, H, W, TS, TS) && make_box_map(&m[6], tgt, n_planes, H, W, TS, TS)) {
      static bool attr2 = false;
      if (!attr2) {
        cudaFuncSetAttribute(k_ssim_maps, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sizeof(MapsSmem));
        cudaFuncSetAttribute(k_ssim_grad, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sizeof(GradSmem));
        attr2 = true;
      }
      const int items = tiles_x * tiles_y * n_planes;
      int dev = 0, sms = 148;
      cudaGetDevice(&dev);
      cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
#ifndef LP_SSIM_GRID
#define LP_SSIM_GRID LP_SSIM_MINB   // persistent CTAs per SM in the grid (measurement knob)
#endif
      const int grid = items < LP_SSIM_GRID * sms ? items : LP_SSIM_GRID * sms;
      k_ssim_maps<<<grid, SLT, sizeof(MapsSmem), st>>>(m[0], m[1], ws, loss_sum, H, W, tiles_x, tiles_x * tiles_y,
                                                       items, lam, scale, win);
      k_ssim_grad<<<grid, SLT, sizeof(GradSmem), st>>>(m[2], m[3], m[4], m[5], m[6], dL, loss_sum, H, W, tiles_x,
                                                       tiles_x * tiles_y, items, lam, scale, win);
      return;
    }
  }
  if (aligned && !tma_off && make_box_map(&mx, img, n_planes, H, W) && make_box_map(&my, tgt, n_planes, H, W)) {
    const size_t smem = sizeof(LossSmemT);
    static bool attr = false;
    if (!attr) {
      cudaFuncSetAttribute(k_loss_ssim_tma, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
      attr = true;
    }
    const int items = tiles_x * tiles_y * n_planes;
    int dev = 0, sms = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    const int grid = items < 2 * sms ? items : 2 * sms;
    k_loss_ssim_tma<<<grid, LT, smem, st>>>(mx, my, dL, loss_sum, H, W, tiles_x, tiles_x * tiles_y, items, lam, scale,
                                            win);
    return;
  }
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
