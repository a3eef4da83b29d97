// Microbenchmark: cost of issuing TMA loads from one thread (2-D tiled and 4-D im2col),
// measured with clock64 around the issue loop.  Build: nvcc -gencode arch=compute_100a,code=sm_100a
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdint>
#include <vector>

__device__ __forceinline__ uint32_t su32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

template <int MODE>
__global__ void kern(const __grid_constant__ CUtensorMap tm, int nloads, long long* out) {
  extern __shared__ __align__(1024) uint8_t sm[];
  __shared__ __align__(8) uint64_t bar;
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(&bar)));
    asm volatile("fence.mbarrier_init.release.cluster;");
    asm volatile("prefetch.tensormap [%0];" ::"l"((uint64_t)&tm));
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    const uint32_t bytes = 128 * 64;
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su32(&bar)), "r"(bytes * nloads));
    long long t0 = clock64();
    for (int i = 0; i < nloads; ++i) {
      uint8_t* dst = sm + (i % 16) * bytes;
      if (MODE == 0) {
        asm volatile("cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4}], [%2];"
                     ::"r"(su32(dst)), "l"((uint64_t)&tm), "r"(su32(&bar)), "r"(0), "r"((blockIdx.x * nloads + i) * 128) : "memory");
      } else {
        asm volatile("cp.async.bulk.tensor.4d.shared::cluster.global.im2col.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4, %5, %6}], [%2], {%7, %8};"
                     ::"r"(su32(dst)), "l"((uint64_t)&tm), "r"(su32(&bar)), "r"(0), "r"(-1), "r"(-1), "r"(blockIdx.x % 64),
                       "h"((uint16_t)(i % 3)), "h"((uint16_t)((i / 3) % 3)) : "memory");
      }
    }
    long long t1 = clock64();
    asm volatile("{\n.reg .pred P;\nW: mbarrier.try_wait.parity.shared::cta.b64 P, [%0], 0;\n@!P bra W;\n}" ::"r"(su32(&bar)));
    long long t2 = clock64();
    if (blockIdx.x == 0) { out[0] = t1 - t0; out[1] = t2 - t0; }
  }
}

int main() {
  void* fn = nullptr; cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q);
  auto encT = (PFN_cuTensorMapEncodeTiled_v12000)fn;
  cudaGetDriverEntryPoint("cuTensorMapEncodeIm2col", &fn, cudaEnableDefault, &q);
  auto encI = (PFN_cuTensorMapEncodeIm2col_v12000)fn;
  const size_t N = 64, H = 56, W = 56, C = 64;
  uint8_t* buf; cudaMalloc(&buf, N * H * W * C);
  cudaMemset(buf, 1, N * H * W * C);
  long long* out; cudaMalloc(&out, 16);
  CUtensorMap t2d, tim;
  {
    cuuint64_t dims[2] = {C, N * H * W}; cuuint64_t str[1] = {C}; cuuint32_t box[2] = {64, 128}; cuuint32_t es[2] = {1, 1};
    printf("enc2d %d\n", (int)encT(&t2d, CU_TENSOR_MAP_DATA_TYPE_UINT8, 2, buf, dims, str, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                                 CU_TENSOR_MAP_SWIZZLE_64B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE));
  }
  {
    cuuint64_t dims[4] = {C, W, H, N}; cuuint64_t str[3] = {C, C * W, C * W * H}; int lo[2] = {-1, -1}, hi[2] = {-1, -1};
    cuuint32_t es[4] = {1, 1, 1, 1};
    printf("encim %d\n", (int)encI(&tim, CU_TENSOR_MAP_DATA_TYPE_UINT8, 4, buf, dims, str, lo, hi, 64, 128, es,
                                  CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_64B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                                  CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE));
  }
  cudaFuncSetAttribute(kern<0>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
  cudaFuncSetAttribute(kern<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
  for (int grid : {1, 148}) for (int nl : {1, 4, 16}) {
    for (int mode = 0; mode < 2; ++mode) {
      long long h[2];
      for (int rep = 0; rep < 3; ++rep) {
        if (mode == 0) kern<0><<<grid, 32, 16 * 8192 + 1024>>>(t2d, nl, out); else kern<1><<<grid, 32, 16 * 8192 + 1024>>>(tim, nl, out);
        cudaDeviceSynchronize();
      }
      cudaMemcpy(h, out, 16, cudaMemcpyDeviceToHost);
      printf("grid %3d mode %s nloads %2d: issue %6lld cycles (%.0f/load)  complete %6lld\n", grid, mode ? "im2col" : "2d    ",
             nl, h[0], (double)h[0] / nl, h[1]);
    }
  }
  printf("err %s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
