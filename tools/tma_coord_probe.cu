#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdint>
#include <cstdlib>
__device__ __forceinline__ uint32_t smem_u32(const void *p) { return static_cast<uint32_t>(__cvta_generic_to_shared(p)); }
__global__ void k(const __grid_constant__ CUtensorMap map_p, const CUtensorMap *map_g, float *out, int variant, int cx_, int cy_) {
  const CUtensorMap &map = variant >= 2 ? *map_g : map_p;
  extern __shared__ __align__(128) unsigned char smem[];
  const uint32_t base = smem_u32(smem);
  const uint32_t pad = (1024 - (base & 1023)) & 1023;
  float *box = reinterpret_cast<float *>(smem + pad);
  __shared__ __align__(8) unsigned long long bar;
  if (threadIdx.x == 0) printf("dyn smem base %u pad %u bar %u\n", base, pad, smem_u32(&bar));
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(&bar)), "r"(1));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(&bar)), "r"(52 * 52 * 4) : "memory");
    const int c0 = cx_, c1 = cy_;
    asm volatile("cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], [%5];"
                 ::"r"(smem_u32(box)), "l"(reinterpret_cast<uint64_t>(&map)), "r"(c0), "r"(c1), "r"(0), "r"(smem_u32(&bar)) : "memory");
  }
  asm volatile("{\n\t.reg .pred p;\nWAIT_%=:\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t@!p bra WAIT_%=;\n}" ::"r"(smem_u32(&bar)), "r"(0) : "memory");
  for (int i = threadIdx.x; i < 52 * 52; i += blockDim.x) out[i] = box[i];
}
int main(int argc, char **argv) {
  int W = 64, H = 48, P = 2;
  float *img; cudaMalloc(&img, W * H * P * 4);
  float *h = (float *)malloc(W * H * P * 4); for (int i = 0; i < W * H * P; ++i) h[i] = (float)i;
  cudaMemcpy(img, h, W * H * P * 4, cudaMemcpyHostToDevice);
  float *out; cudaMalloc(&out, 52 * 52 * 4);
  PFN_cuTensorMapEncodeTiled encode; cudaDriverEntryPointQueryResult q; void *fn;
  printf("entry %d\n", (int)cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q));
  encode = (PFN_cuTensorMapEncodeTiled)fn;
  CUtensorMap map;
  cuuint64_t dims[3] = {(cuuint64_t)W, (cuuint64_t)H, (cuuint64_t)P};
  cuuint64_t str[2] = {(cuuint64_t)W * 4, (cuuint64_t)W * H * 4};
  cuuint32_t box[3] = {52, 52, 1}, es[3] = {1, 1, 1};
  printf("encode %d\n", (int)encode(&map, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 3, img, dims, str, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                                 CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_128B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE));
  CUtensorMap *mg; cudaMalloc(&mg, sizeof(CUtensorMap)); cudaMemcpy(mg, &map, sizeof(map), cudaMemcpyHostToDevice);
  printf("sizeof map %zu align %zu\n", sizeof(CUtensorMap), alignof(CUtensorMap));
  {
    int variant = atoi(argv[1]);
    k<<<1, 128, 52 * 52 * 4 + 1024>>>(map, mg, out, variant, atoi(argv[2]), atoi(argv[3]));
    printf("variant %d: %s\n", variant, cudaGetErrorString(cudaDeviceSynchronize()));
    float o[52 * 52]; cudaMemcpy(o, out, sizeof(o), cudaMemcpyDeviceToHost);
    printf("  o[0]=%g o[10*52+10]=%g o[11*52+12]=%g\n", o[0], o[10 * 52 + 10], o[11 * 52 + 12]);
  }
}
