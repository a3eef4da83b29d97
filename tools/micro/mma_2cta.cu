// mma_2cta.cu — semantics probe for tcgen05.mma.cta_group::2 (kind::i8, M = 256, N = 256, K = 32)
// over a CTA pair: CTA r holds rows [128 r, +128) of A and rows [128 r, +128) of B (K-major,
// 32-byte rows, 32-B swizzle) at the same shared-memory offsets; the leader issues one MMA and a
// multicast commit; each CTA then reads its TMEM (128 lanes x 256 columns) and the host checks
// D[m][n] = sum_k A[m][k] B[n][k] for m in CTA r's half.  Prints OK / the first mismatch.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/micro/mma_2cta tools/micro/mma_2cta.cu
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t su32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ uint64_t sdesc32(uint32_t saddr) {   // K-major, 32-B rows, SW32
  uint64_t d = 0;
  d |= (uint64_t)((saddr & 0x3FFFFu) >> 4);
  d |= (uint64_t)1 << 16;
  d |= (uint64_t)((8u * 32u) >> 4) << 32;
  d |= (uint64_t)1 << 46;
  d |= (uint64_t)6 << 61;
  return d;
}

__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(128, 1)
    k2cta(const int8_t* A, const int8_t* B, int32_t* D) {
  __shared__ __align__(1024) uint8_t sa[128 * 32];
  __shared__ __align__(1024) uint8_t sb[128 * 32];
  __shared__ __align__(8) uint64_t bar;
  __shared__ uint32_t slot;
  uint32_t rank;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(rank));
  // rows of this CTA's halves, SW32: 16-B chunk c of row r at c ^ ((r >> 2) & 1)
  for (int i = threadIdx.x; i < 128 * 2; i += blockDim.x) {
    const int r = i >> 1, c = i & 1, cs = c ^ ((r >> 2) & 1);
    *reinterpret_cast<uint4*>(sa + r * 32 + cs * 16) = *reinterpret_cast<const uint4*>(A + (rank * 128 + r) * 32 + c * 16);
    *reinterpret_cast<uint4*>(sb + r * 32 + cs * 16) = *reinterpret_cast<const uint4*>(B + (rank * 128 + r) * 32 + c * 16);
  }
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(&bar)));
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  if (threadIdx.x < 32) {
    asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], 256;" ::"r"(su32(&slot)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;");
  }
  asm volatile("fence.proxy.async.shared::cta;");
  asm volatile("tcgen05.fence::before_thread_sync;");
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t tmem = slot;
  if (rank == 0 && threadIdx.x == 0) {
    const uint32_t idesc = (2u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(256 >> 3) << 17) | ((uint32_t)(256 >> 4) << 24);
    asm volatile("tcgen05.mma.cta_group::2.kind::i8 [%0], %1, %2, %3, 0;" ::"r"(tmem), "l"(sdesc32(su32(sa))),
                 "l"(sdesc32(su32(sb))), "r"(idesc));
    asm volatile("tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;"
                 ::"r"(su32(&bar)), "h"((uint16_t)3));
  }
  asm volatile("{\n\t.reg .pred P;\nW:\n\tmbarrier.try_wait.parity.shared::cta.b64 P, [%0], 0;\n\t@!P bra W;\n\t}" ::"r"(
                   su32(&bar)) : "memory");
  asm volatile("tcgen05.fence::after_thread_sync;");
  // warp w reads TMEM lanes [32 w, +32): 256 columns, 32 at a time
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  for (int c0 = 0; c0 < 256; c0 += 32) {
    uint32_t v[32];
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
        : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]), "=r"(v[8]),
          "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15]), "=r"(v[16]),
          "=r"(v[17]), "=r"(v[18]), "=r"(v[19]), "=r"(v[20]), "=r"(v[21]), "=r"(v[22]), "=r"(v[23]), "=r"(v[24]),
          "=r"(v[25]), "=r"(v[26]), "=r"(v[27]), "=r"(v[28]), "=r"(v[29]), "=r"(v[30]), "=r"(v[31])
        : "r"(tmem + ((uint32_t)(w * 32) << 16) + (uint32_t)c0));
    asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
    const int m = rank * 128 + w * 32 + lane;
    for (int i = 0; i < 32; ++i) D[m * 256 + c0 + i] = (int32_t)v[i];
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
  if (threadIdx.x < 32) asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, 256;" ::"r"(tmem));
}

int main() {
  const int M = 256, N = 256, K = 32;
  int8_t *hA = (int8_t*)malloc(M * K), *hB = (int8_t*)malloc(N * K);
  int32_t* hD = (int32_t*)malloc(M * N * 4);
  srand(1);
  for (int i = 0; i < M * K; ++i) hA[i] = (int8_t)(rand() % 255 - 127);
  for (int i = 0; i < N * K; ++i) hB[i] = (int8_t)(rand() % 255 - 127);
  int8_t *dA, *dB;
  int32_t* dD;
  cudaMalloc(&dA, M * K); cudaMalloc(&dB, N * K); cudaMalloc(&dD, M * N * 4);
  cudaMemcpy(dA, hA, M * K, cudaMemcpyHostToDevice);
  cudaMemcpy(dB, hB, N * K, cudaMemcpyHostToDevice);
  cudaMemset(dD, 0, M * N * 4);
  k2cta<<<2, 128>>>(dA, dB, dD);
  cudaError_t e = cudaDeviceSynchronize();
  if (e != cudaSuccess) { printf("error %s\n", cudaGetErrorString(e)); return 1; }
  cudaMemcpy(hD, dD, M * N * 4, cudaMemcpyDeviceToHost);
  int bad = 0;
  for (int m = 0; m < M && bad < 5; ++m)
    for (int n = 0; n < N && bad < 5; ++n) {
      int32_t ref = 0;
      for (int k = 0; k < K; ++k) ref += (int32_t)hA[m * K + k] * (int32_t)hB[n * K + k];
      if (ref != hD[m * N + n]) {
        printf("mismatch m %d n %d got %d want %d\n", m, n, hD[m * N + n], ref);
        ++bad;
      }
    }
  printf(bad ? "FAIL\n" : "OK: CTA r holds A rows and B rows [128 r, +128); its TMEM has D rows [128 r, +128) x all 256 columns\n");
  return 0;
}
