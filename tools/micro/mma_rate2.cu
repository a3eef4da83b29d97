// mma_rate2.cu — cycles per tcgen05.mma.kind::i8 (M=128, cta_group::1) vs swizzle mode of the K-major
// operands (32/64/128-B rows), operand contents (zeros vs random bytes) and N.  Each MMA reads a
// different 128-row A slice (walking a 64 KB ring, like the GEMM's pipeline stages).  shift = 1 starts
// each slice at a row offset that is not a multiple of the 8-row swizzle atom (the staged-row
// 3x3 path addresses filter taps that way).
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/micro/mma_rate2 tools/micro/mma_rate2.cu
#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

// K-major descriptor for rows of `rb` bytes (32/64/128) in the matching swizzle
__device__ __forceinline__ uint64_t sdesc(uint32_t saddr, int rb) {
  uint64_t d = 0;
  d |= (uint64_t)((saddr & 0x3FFFFu) >> 4);
  d |= (uint64_t)1 << 16;
  d |= (uint64_t)((8u * rb) >> 4) << 32;
  d |= (uint64_t)1 << 46;
  const uint64_t mode = rb == 128 ? 2 : rb == 64 ? 4 : 6;
  d |= mode << 61;
  return d;
}

__global__ void __launch_bounds__(128, 1) mma_rate(int N, int rb, int iters, int fill, int shift, long long* out) {
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ uint32_t tmem_slot;
  __shared__ __align__(8) uint64_t bar;
  uint8_t* sa = smem + ((1024u - (smem_u32(smem) & 1023u)) & 1023u);   // 64 KB A ring
  uint8_t* sb = sa + 65536;                                             // 32 KB B
  for (int i = threadIdx.x; i < (65536 + 32768) / 4; i += blockDim.x) {
    uint32_t v = fill ? (uint32_t)(i * 2654435761u) ^ 0x5bd1e995u * (uint32_t)(i >> 3) : 0u;
    reinterpret_cast<uint32_t*>(sa)[i] = v;
  }
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
  const uint32_t idesc = (2u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(128 >> 4) << 24);
  // A slices: 128 rows x rb bytes each; K=32 per MMA -> rb/32 MMAs per slice
  const int slice = 128 * rb, nslices = 65536 / slice / 2, kst = rb / 32;   // (half the ring: room for shifts)
  const int lk = __ffs(kst) - 1, smask = nslices - 1, kmask = kst - 1, lsl = __ffs(slice >> 4) - 1;
  if (threadIdx.x == 0) {
    const uint64_t a0 = sdesc(smem_u32(sa), rb), b0 = sdesc(smem_u32(sb), rb);
    long long t0 = clock64();
#pragma unroll 1
    for (int i = 0; i < iters; i += 4) {
      uint64_t ad[4], bd[4];
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        const int m = i + j, sl = (m >> lk) & smask, k = m & kmask;
        const uint32_t rsh = shift ? (uint32_t)((m >> lk) * 5 % 61) * rb : 0u;   // row shift, bytes
        ad[j] = a0 + ((uint32_t)sl << lsl) + (rsh >> 4) + 2 * k;
        bd[j] = b0 + 2 * k;
      }
      asm volatile(
          "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %9, 0;\n\t"
          "tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %8, p;\n\t"
          "tcgen05.mma.cta_group::1.kind::i8 [%0], %3, %4, %8, 1;\n\t"
          "tcgen05.mma.cta_group::1.kind::i8 [%0], %5, %6, %8, 1;\n\t"
          "tcgen05.mma.cta_group::1.kind::i8 [%0], %7, %10, %8, 1;\n\t}" ::"r"(tmem),
          "l"(ad[0]), "l"(bd[0]), "l"(ad[1]), "l"(bd[1]), "l"(ad[2]), "l"(bd[2]), "l"(ad[3]), "r"(idesc), "r"(i),
          "l"(bd[3]));
    }
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(&bar)));
    asm volatile(
        "{\n\t.reg .pred P1;\nW:\n\tmbarrier.try_wait.parity.shared::cta.b64 P1, [%0], 0;\n\t@P1 bra D;\n\tbra W;\nD:\n\t}" ::"r"(
            smem_u32(&bar)));
    long long t1 = clock64();
    if (blockIdx.x == 0) *out = t1 - t0;
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (threadIdx.x < 32) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tmem));
}

int main() {
  long long* d_out;
  cudaMalloc(&d_out, sizeof(long long));
  cudaFuncSetAttribute(mma_rate, cudaFuncAttributeMaxDynamicSharedMemorySize, 100 * 1024);
  const int iters = 8192;
  printf("%4s %4s %5s %5s %12s %12s\n", "N", "rowB", "fill", "shift", "cycles/MMA", "ideal(N/2)");
  for (int shift : {0, 1})
  for (int fill : {1})
    for (int rb : {32, 64, 128})
      for (int N : {32, 64, 128, 256}) {
        mma_rate<<<148, 128, 100 * 1024>>>(N, rb, iters, fill, shift, d_out);
        mma_rate<<<148, 128, 100 * 1024>>>(N, rb, iters, fill, shift, d_out);
        long long cyc = 0;
        cudaMemcpy(&cyc, d_out, sizeof(cyc), cudaMemcpyDeviceToHost);
        cudaError_t e = cudaGetLastError();
        if (e != cudaSuccess) {
          printf("error %s\n", cudaGetErrorString(e));
          return 1;
        }
        printf("%4d %4d %5d %5d %12.1f %12d\n", N, rb, fill, shift, (double)cyc / iters, N / 2);
      }
  return 0;
}
