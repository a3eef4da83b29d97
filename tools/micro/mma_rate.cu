// mma_rate.cu — microbenchmark: cycles per tcgen05.mma.kind::i8 (cta_group::1) vs M and N.
//
// One CTA per SM; one elected thread issues `iters` MMAs round-robin over `nacc` independent
// TMEM accumulators (so consecutive MMAs never depend on each other), then a commit + wait.
// A and B are zero-filled shared memory in the 128-B swizzle (values do not matter for timing).
// Prints cycles per MMA and the implied int8 TOPS per SM / per chip (148 SMs at the measured clock).
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/micro/mma_rate tools/micro/mma_rate.cu
#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

__device__ __forceinline__ uint64_t sdesc(uint32_t saddr) {   // K-major, 128-B rows, SW128
  uint64_t d = 0;
  d |= (uint64_t)((saddr & 0x3FFFFu) >> 4);
  d |= (uint64_t)1 << 16;
  d |= (uint64_t)((8u * 128u) >> 4) << 32;
  d |= (uint64_t)1 << 46;
  d |= (uint64_t)2 << 61;
  return d;
}

__global__ void __launch_bounds__(128, 1) mma_rate(int M, int N, int iters, int nacc, int nissuers, long long* out) {
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ uint32_t tmem_slot;
  __shared__ __align__(8) uint64_t bar;
  uint8_t* sa = smem + ((1024u - (smem_u32(smem) & 1023u)) & 1023u);
  uint8_t* sb = sa + 128 * 128;
  for (int i = threadIdx.x; i < (128 * 128 + 256 * 128) / 16; i += blockDim.x)
    reinterpret_cast<uint4*>(sa)[i] = make_uint4(0, 0, 0, 0);
  if (threadIdx.x < 32) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(smem_u32(&tmem_slot)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&bar)));
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  asm volatile("fence.proxy.async.shared::cta;");
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t tmem = tmem_slot;
  const uint32_t idesc = (2u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(M >> 4) << 24);
  const uint64_t ad = sdesc(smem_u32(sa)), bd = sdesc(smem_u32(sb));
  const uint32_t stride = 512u / (nacc * nissuers);
  // nissuers warps (lane 0 each) issue concurrently, each into its own accumulator subset
  const int wi = threadIdx.x >> 5;
  if ((threadIdx.x & 31) == 0 && wi < nissuers) {
    long long t0 = clock64();
    // tight loop: 4 MMAs per iteration into 4 precomputed accumulators (no index math per MMA)
    const uint32_t d0 = tmem + (uint32_t)(wi * 4 + 0) % (512u / stride) * stride;
    const uint32_t d1 = tmem + (uint32_t)(wi * 4 + (nacc > 1 ? 1 : 0)) % (512u / stride) * stride;
    const uint32_t d2 = tmem + (uint32_t)(wi * 4 + (nacc > 2 ? 2 : 0)) % (512u / stride) * stride;
    const uint32_t d3 = tmem + (uint32_t)(wi * 4 + (nacc > 3 ? 3 : (nacc > 1 ? 1 : 0))) % (512u / stride) * stride;
#pragma unroll 1
    for (int i = 0; i < iters; i += 4) {
      asm volatile(
          "tcgen05.mma.cta_group::1.kind::i8 [%0], %4, %5, %6, 1;\n\t"
          "tcgen05.mma.cta_group::1.kind::i8 [%1], %4, %5, %6, 1;\n\t"
          "tcgen05.mma.cta_group::1.kind::i8 [%2], %4, %5, %6, 1;\n\t"
          "tcgen05.mma.cta_group::1.kind::i8 [%3], %4, %5, %6, 1;\n\t" ::"r"(d0), "r"(d1), "r"(d2), "r"(d3),
          "l"(ad), "l"(bd), "r"(idesc));
    }
    if (wi == 0) {
      asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(&bar)));
      asm volatile(
          "{\n\t.reg .pred P1;\nW:\n\tmbarrier.try_wait.parity.shared::cta.b64 P1, [%0], 0;\n\t@P1 bra D;\n\tbra W;\nD:\n\t}" ::"r"(
              smem_u32(&bar)));
      long long t1 = clock64();
      if (blockIdx.x == 0) *out = t1 - t0;
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (threadIdx.x < 32) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tmem));
}

int main() {
  long long* d_out;
  cudaMalloc(&d_out, sizeof(long long));
  cudaFuncSetAttribute(mma_rate, cudaFuncAttributeMaxDynamicSharedMemorySize, 64 * 1024);
  int clk_khz = 0;
  cudaDeviceGetAttribute(&clk_khz, cudaDevAttrClockRate, 0);
  const int iters = 4096;
  printf("%4s %4s %5s %4s %12s %10s %14s\n", "M", "N", "nacc", "iss", "cycles/MMA", "MAC/clk", "TOPS(148 SM)");
  for (int nis : {1, 2})
  for (int M : {64, 128})
    for (int N : {32, 64, 128, 256})
      for (int nacc : {1, 2}) {
        if (512 / (nacc * nis) < N) continue;
        mma_rate<<<148, 128, 64 * 1024>>>(M, N, iters, nacc, nis, d_out);   // warm
        mma_rate<<<148, 128, 64 * 1024>>>(M, N, iters, nacc, nis, d_out);
        long long cyc = 0;
        cudaMemcpy(&cyc, d_out, sizeof(cyc), cudaMemcpyDeviceToHost);
        cudaError_t e = cudaGetLastError();
        if (e != cudaSuccess) {
          printf("error %s\n", cudaGetErrorString(e));
          return 1;
        }
        const double cpm = (double)cyc / (iters * nis);   // (issuer 0's window; others run concurrently)
        const double macs = (double)M * N * 32 / cpm;
        printf("%4d %4d %5d %4d %12.1f %10.0f %14.1f\n", M, N, nacc, nis, cpm, macs, macs * 2 * 148 * clk_khz * 1e3 / 1e12);
      }
  return 0;
}
