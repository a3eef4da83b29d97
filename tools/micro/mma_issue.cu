// mma_issue.cu — is the single-thread tcgen05.mma issue rate bounded by how the issuing code is
// compiled?  mode 0: the loop runs in lane 0 only (divergent: descriptors live in regular
// registers and every UTCIMMA needs R2UR moves); mode 1: the whole warp runs the loop
// (warp-uniform, descriptors in uniform registers) and elect.sync picks the issuing lane per
// MMA group.  Descriptors advance by constant strides per MMA, as in the GEMM's issue loop.
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/micro/mma_issue tools/micro/mma_issue.cu
#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ uint64_t sdesc(uint32_t saddr) {   // K-major, 64-B rows, SW64
  uint64_t d = 0;
  d |= (uint64_t)((saddr & 0x3FFFFu) >> 4);
  d |= (uint64_t)1 << 16;
  d |= (uint64_t)((8u * 64u) >> 4) << 32;
  d |= (uint64_t)1 << 46;
  d |= (uint64_t)4 << 61;
  return d;
}
__device__ __forceinline__ bool elect_one() {
  uint32_t pred = 0;
  asm volatile("{\n\t.reg .pred P;\n\telect.sync _|P, 0xffffffff;\n\tselp.u32 %0, 1, 0, P;\n\t}" : "=r"(pred));
  return pred != 0;
}
__device__ __forceinline__ void mma(uint32_t d, uint64_t a, uint64_t b, uint32_t idesc, uint32_t acc) {
  asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\ttcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n\t}"
               ::"r"(d), "l"(a), "l"(b), "r"(idesc), "r"(acc));
}

template <int MODE>
__global__ void __launch_bounds__(128, 1) mma_issue(int N, int ntap, int reps, long long* out) {
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ uint32_t tmem_slot;
  __shared__ __align__(8) uint64_t bar;
  uint8_t* sa = smem + ((1024u - (smem_u32(smem) & 1023u)) & 1023u);   // 64 KB A rows
  uint8_t* sb = sa + 65536;                                             // 9 taps x 256 x 64 B of B
  for (int i = threadIdx.x; i < (65536 + 9 * 16384) / 4; i += blockDim.x)
    reinterpret_cast<uint32_t*>(sa)[i] = (uint32_t)(i * 2654435761u);
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
  const uint64_t a0 = sdesc(smem_u32(sa)), b0 = sdesc(smem_u32(sb));
  const uint32_t a_col16 = 64 >> 4, a_row16 = (58 * 64) >> 4, b_tap16 = (N * 64) >> 4;   // like layer1's a_rows
  long long t0 = 0;
  const int warp = __shfl_sync(0xffffffffu, (int)(threadIdx.x >> 5), 0);   // provably warp-uniform
  if (warp == 0) {
    if (MODE == 0) {
      if (threadIdx.x == 0) {
        t0 = clock64();
        for (int rep = 0; rep < reps; ++rep) {
          const uint32_t d = tmem + (uint32_t)(rep & 1) * 256;
          uint64_t ad_row = a0 + (uint64_t)((rep & 7) * 8), bd = b0;
          uint32_t acc = 0;
          for (int r = 0; r < ntap; ++r) {
            uint64_t ad = ad_row;
            for (int s = 0; s < ntap; ++s) {
#pragma unroll
              for (int k = 0; k < 2; ++k) mma(d, ad + 2 * k, bd + 2 * k, idesc, k ? 1u : acc);
              acc = 1;
              ad += a_col16;
              bd += b_tap16;
            }
            ad_row += a_row16;
          }
        }
      }
    } else {
      t0 = clock64();
      for (int rep = 0; rep < reps; ++rep) {
        const uint32_t d = tmem + (uint32_t)(rep & 1) * 256;
        uint64_t ad_row = a0 + (uint64_t)((rep & 7) * 8), bd = b0;
        uint32_t acc = 0;
        for (int r = 0; r < ntap; ++r) {
          uint64_t ad = ad_row;
          for (int s = 0; s < ntap; ++s) {
            if (elect_one()) {
              mma(d, ad, bd, idesc, acc);
              mma(d, ad + 2, bd + 2, idesc, 1u);
            }
            __syncwarp();
            acc = 1;
            ad += a_col16;
            bd += b_tap16;
          }
          ad_row += a_row16;
        }
      }
    }
    if (threadIdx.x == 0) {
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
  cudaFuncSetAttribute(mma_issue<0>, cudaFuncAttributeMaxDynamicSharedMemorySize, 215 * 1024);
  cudaFuncSetAttribute(mma_issue<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, 215 * 1024);
  const int reps = 256, ntap = 3;
  printf("%5s %4s %12s %12s\n", "mode", "N", "cycles/MMA", "ideal(N/2)");
  for (int mode : {0, 1})
    for (int N : {64, 128, 256}) {
      for (int w = 0; w < 2; ++w) {
        if (mode == 0) mma_issue<0><<<148, 128, 215 * 1024>>>(N, ntap, reps, d_out);
        else mma_issue<1><<<148, 128, 215 * 1024>>>(N, ntap, reps, d_out);
      }
      long long cyc = 0;
      cudaMemcpy(&cyc, d_out, sizeof(cyc), cudaMemcpyDeviceToHost);
      cudaError_t e = cudaGetLastError();
      if (e != cudaSuccess) { printf("error %s\n", cudaGetErrorString(e)); return 1; }
      printf("%5d %4d %12.1f %12d\n", mode, N, (double)cyc / (reps * ntap * ntap * 2), N / 2);
    }
  return 0;
}
