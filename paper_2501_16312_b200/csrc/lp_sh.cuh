// lp_sh.cuh -- view-dependent colour from real SH up to degree 3, 3DGS convention
// ("following the same approach described in 3DGS"; constants and sign table in
// DESIGN.md §2).  rgb = max(0, sum_k sh_k Y_k(dir) + 0.5), dir = (c - campos)/|c - campos|.
#pragma once
#include <cuda_runtime.h>

namespace lp {

struct SHC {
  static constexpr float C0 = 0.28209479177387814f;
  static constexpr float C1 = 0.4886025119029199f;
  static constexpr float C2_0 = 1.0925484305920792f, C2_1 = -1.0925484305920792f, C2_2 = 0.31539156525252005f,
                         C2_3 = -1.0925484305920792f, C2_4 = 0.5462742152960396f;
  static constexpr float C3_0 = -0.5900435899266435f, C3_1 = 2.890611442640554f, C3_2 = -0.4570457994644658f,
                         C3_3 = 0.3731763325901154f, C3_4 = -0.4570457994644658f, C3_5 = 1.445305721320277f,
                         C3_6 = -0.5900435899266435f;
};

// Y[16] at unit direction (x,y,z); only the first (deg+1)^2 entries are meaningful.
template <typename T>
__device__ __forceinline__ void sh_basis(int deg, T x, T y, T z, T Y[16]) {
  Y[0] = (T)SHC::C0;
  if (deg < 1) return;
  Y[1] = -(T)SHC::C1 * y;
  Y[2] = (T)SHC::C1 * z;
  Y[3] = -(T)SHC::C1 * x;
  if (deg < 2) return;
  const T xx = x * x, yy = y * y, zz = z * z, xy = x * y, yz = y * z, xz = x * z;
  Y[4] = (T)SHC::C2_0 * xy;
  Y[5] = (T)SHC::C2_1 * yz;
  Y[6] = (T)SHC::C2_2 * (2 * zz - xx - yy);
  Y[7] = (T)SHC::C2_3 * xz;
  Y[8] = (T)SHC::C2_4 * (xx - yy);
  if (deg < 3) return;
  Y[9] = (T)SHC::C3_0 * y * (3 * xx - yy);
  Y[10] = (T)SHC::C3_1 * xy * z;
  Y[11] = (T)SHC::C3_2 * y * (4 * zz - xx - yy);
  Y[12] = (T)SHC::C3_3 * z * (2 * zz - 3 * xx - 3 * yy);
  Y[13] = (T)SHC::C3_4 * x * (4 * zz - xx - yy);
  Y[14] = (T)SHC::C3_5 * z * (xx - yy);
  Y[15] = (T)SHC::C3_6 * x * (xx - 3 * yy);
}

// gradient of sum_k w_k Y_k w.r.t. the (unnormalised-polynomial) direction components
template <typename T>
__device__ __forceinline__ void sh_basis_grad_dot(int deg, T x, T y, T z, const T w[16], T g[3]) {
  g[0] = g[1] = g[2] = 0;
  if (deg < 1) return;
  g[1] += -(T)SHC::C1 * w[1];
  g[2] += (T)SHC::C1 * w[2];
  g[0] += -(T)SHC::C1 * w[3];
  if (deg < 2) return;
  const T xx = x * x, yy = y * y, zz = z * z, xy = x * y, yz = y * z, xz = x * z;
  g[0] += (T)SHC::C2_0 * y * w[4];
  g[1] += (T)SHC::C2_0 * x * w[4];
  g[1] += (T)SHC::C2_1 * z * w[5];
  g[2] += (T)SHC::C2_1 * y * w[5];
  g[0] += -2 * (T)SHC::C2_2 * x * w[6];
  g[1] += -2 * (T)SHC::C2_2 * y * w[6];
  g[2] += 4 * (T)SHC::C2_2 * z * w[6];
  g[0] += (T)SHC::C2_3 * z * w[7];
  g[2] += (T)SHC::C2_3 * x * w[7];
  g[0] += 2 * (T)SHC::C2_4 * x * w[8];
  g[1] += -2 * (T)SHC::C2_4 * y * w[8];
  if (deg < 3) return;
  g[0] += (T)SHC::C3_0 * 6 * xy * w[9];
  g[1] += (T)SHC::C3_0 * (3 * xx - 3 * yy) * w[9];
  g[0] += (T)SHC::C3_1 * yz * w[10];
  g[1] += (T)SHC::C3_1 * xz * w[10];
  g[2] += (T)SHC::C3_1 * xy * w[10];
  g[0] += (T)SHC::C3_2 * (-2 * xy) * w[11];
  g[1] += (T)SHC::C3_2 * (4 * zz - xx - 3 * yy) * w[11];
  g[2] += (T)SHC::C3_2 * 8 * yz * w[11];
  g[0] += (T)SHC::C3_3 * (-6 * xz) * w[12];
  g[1] += (T)SHC::C3_3 * (-6 * yz) * w[12];
  g[2] += (T)SHC::C3_3 * (6 * zz - 3 * xx - 3 * yy) * w[12];
  g[0] += (T)SHC::C3_4 * (4 * zz - 3 * xx - yy) * w[13];
  g[1] += (T)SHC::C3_4 * (-2 * xy) * w[13];
  g[2] += (T)SHC::C3_4 * 8 * xz * w[13];
  g[0] += (T)SHC::C3_5 * 2 * xz * w[14];
  g[1] += (T)SHC::C3_5 * (-2 * yz) * w[14];
  g[2] += (T)SHC::C3_5 * (xx - yy) * w[14];
  g[0] += (T)SHC::C3_6 * (3 * xx - 3 * yy) * w[15];
  g[1] += (T)SHC::C3_6 * (-6 * xy) * w[15];
}

}  // namespace lp
