// tmem_layout.cu — which (TMEM lane, column) each thread receives from tcgen05.ld.16x256b.x2:
// TMEM is filled with (lane << 16 | column) through tcgen05.st.32x32b (lane = thread), then read
// back with the 16x256b shape at lane base 0 and 16.
#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>

__global__ void k(uint32_t* out) {
  __shared__ uint32_t slot;
  const int t = threadIdx.x;
  asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 32;" ::"r"(
      (uint32_t)__cvta_generic_to_shared(&slot)));
  asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncwarp();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t base = slot;
  uint32_t v[16];
  for (int c = 0; c < 16; ++c) v[c] = ((uint32_t)t << 16) | c;
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16};" ::"r"(base),
      "r"(v[0]), "r"(v[1]), "r"(v[2]), "r"(v[3]), "r"(v[4]), "r"(v[5]), "r"(v[6]), "r"(v[7]), "r"(v[8]), "r"(v[9]),
      "r"(v[10]), "r"(v[11]), "r"(v[12]), "r"(v[13]), "r"(v[14]), "r"(v[15]));
  asm volatile("tcgen05.wait::st.sync.aligned;");
  for (int h = 0; h < 2; ++h) {
    uint32_t r[8];
    asm volatile("tcgen05.ld.sync.aligned.16x256b.x2.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                 : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7])
                 : "r"(base + ((uint32_t)(16 * h) << 16)));
    asm volatile("tcgen05.wait::ld.sync.aligned;");
    for (int i = 0; i < 8; ++i) out[(h * 32 + t) * 8 + i] = r[i];
  }
  asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 32;" ::"r"(base));
}

int main() {
  uint32_t* d;
  cudaMalloc(&d, 2 * 32 * 8 * 4);
  k<<<1, 32>>>(d);
  uint32_t h[2 * 32 * 8];
  cudaError_t e = cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
  printf("%s\n", cudaGetErrorString(e));
  for (int hh = 0; hh < 2; ++hh)
    for (int t = 0; t < 32; t += 1) {
      printf("base %2d thread %2d:", 16 * hh, t);
      for (int i = 0; i < 8; ++i) printf(" (%2u,%2u)", h[(hh * 32 + t) * 8 + i] >> 16, h[(hh * 32 + t) * 8 + i] & 0xffff);
      printf("\n");
    }
  return 0;
}
