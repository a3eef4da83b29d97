// Microbenchmark: HBM streaming bandwidth of (a) TMA 2-D tiled loads with 64-B or 128-B rows,
// (b) cp.async 16-B per thread (LDGSTS) by 4 warps, (c) TMA 2-D stores from smem.
// One persistent CTA per SM, a ring of `depth` 8 KB stages in flight.
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdint>

__device__ __forceinline__ uint32_t su32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void wait(uint64_t* b, uint32_t ph) {
  asm volatile("{\n.reg .pred P;\nW: mbarrier.try_wait.parity.shared::cta.b64 P, [%0], %1;\n@!P bra W;\n}" ::"r"(su32(b)), "r"(ph));
}

// MODE 0: TMA load rows of RB bytes (box {RB, 8192/RB}); MODE 1: cp.async by 128 threads; MODE 2: TMA store (box {RB, 8192/RB})
template <int MODE, int RB>
__global__ void __launch_bounds__(128) kern(const __grid_constant__ CUtensorMap tm, const uint8_t* src, long long tiles, int depth) {
  extern __shared__ __align__(1024) uint8_t sm[];
  __shared__ __align__(8) uint64_t bar[16];
  const int tid = threadIdx.x;
  if (tid == 0) {
    for (int i = 0; i < depth; ++i) asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(su32(&bar[i])), "r"(MODE == 1 ? 128 : 1));
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  __syncthreads();
  const int rows = 8192 / RB;
  long long it = 0;
  for (long long t = blockIdx.x; t < tiles; t += gridDim.x, ++it) {
    const int s = (int)(it % depth);
    const uint32_t ph = (uint32_t)((it / depth) & 1);
    if (MODE != 2 && it >= depth) wait(&bar[s], ph ^ 1);
    uint8_t* dst = sm + s * 8192;
    if (MODE == 0) {
      if (tid == 0) {
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], 8192;" ::"r"(su32(&bar[s])));
        asm volatile("cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4}], [%2];"
                     ::"r"(su32(dst)), "l"((uint64_t)&tm), "r"(su32(&bar[s])), "r"(0), "r"((int)(t * rows)) : "memory");
      }
    } else if (MODE == 1) {
      const uint8_t* g = src + t * 8192;
      #pragma unroll
      for (int i = 0; i < 4; ++i) {
        const int off = (i * 128 + tid) * 16;
        asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(su32(dst + off)), "l"(g + off) : "memory");
      }
      asm volatile("cp.async.mbarrier.arrive.noinc.shared::cta.b64 [%0];" ::"r"(su32(&bar[s])) : "memory");
    } else {
      if (tid == 0) {
        asm volatile("cp.async.bulk.tensor.2d.global.shared::cta.bulk_group [%0, {%2, %3}], [%1];"
                     ::"l"((uint64_t)&tm), "r"(su32(dst)), "r"(0), "r"((int)(t * rows)) : "memory");
        asm volatile("cp.async.bulk.commit_group;");
        asm volatile("cp.async.bulk.wait_group.read 7;" ::: "memory");
      }
    }
  }
  if (MODE == 2 && tid == 0) asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
  // drain
  if (MODE != 2) for (long long k = it - depth; k < it; ++k) if (k >= 0) wait(&bar[k % depth], (uint32_t)((k / depth) & 1));
}

int main() {
  void* fn = nullptr; cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q);
  auto encT = (PFN_cuTensorMapEncodeTiled_v12000)fn;
  const long long bytes = 1ll << 30;
  uint8_t* buf; cudaMalloc(&buf, bytes);
  cudaMemset(buf, 1, bytes);
  uint8_t* flush; cudaMalloc(&flush, 512 << 20);
  const long long tiles = bytes / 8192;
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  auto run = [&](const char* name, auto kernel, int rb, int depth) {
    CUtensorMap tm;
    cuuint64_t dims[2] = {(cuuint64_t)rb, (cuuint64_t)(bytes / rb)}; cuuint64_t str[1] = {(cuuint64_t)rb};
    cuuint32_t box[2] = {(cuuint32_t)rb, (cuuint32_t)(8192 / rb)}; cuuint32_t es[2] = {1, 1};
    encT(&tm, CU_TENSOR_MAP_DATA_TYPE_UINT8, 2, buf, dims, str, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
         rb == 128 ? CU_TENSOR_MAP_SWIZZLE_128B : (rb == 64 ? CU_TENSOR_MAP_SWIZZLE_64B : CU_TENSOR_MAP_SWIZZLE_32B),
         CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 16 * 8192 + 1024);
    float best = 1e9;
    for (int rep = 0; rep < 3; ++rep) {
      cudaMemset(flush, rep, 512 << 20);
      cudaEventRecord(a);
      kernel<<<148, 128, 16 * 8192 + 1024>>>(tm, buf, tiles, depth);
      cudaEventRecord(b); cudaEventSynchronize(b);
      float ms; cudaEventElapsedTime(&ms, a, b); if (ms < best) best = ms;
    }
    printf("%-28s rows %3d B depth %2d : %7.1f GB/s\n", name, rb, depth, bytes / (best * 1e-3) / 1e9);
  };
  for (int d : {4, 8, 16}) {
    run("TMA load", kern<0, 64>, 64, d);
    run("TMA load", kern<0, 128>, 128, d);
    run("TMA load", kern<0, 32>, 32, d);
    run("cp.async 16B x128 thr", kern<1, 64>, 64, d);
  }
  run("TMA store", kern<2, 64>, 64, 8);
  run("TMA store", kern<2, 128>, 128, 8);
  run("TMA store", kern<2, 32>, 32, 8);
  printf("err %s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
