// launch_probe.cu — does a 576-thread CTA launch at 112 / 104 registers per thread (sm_100a)?
#include <cstdio>
#include <cuda_runtime.h>
template <int R>
__global__ void __maxnreg__(R) k(int* out) {
  if (threadIdx.x == 0 && out) out[blockIdx.x] = R;
}
template <int R>
void probe(int threads) {
  cudaFuncAttributes a;
  cudaFuncGetAttributes(&a, k<R>);
  k<R><<<1, threads>>>(nullptr);
  cudaError_t e = cudaDeviceSynchronize();
  if (e == cudaSuccess) e = cudaGetLastError();
  printf("maxnreg %d (numRegs %d) threads %d: %s\n", R, a.numRegs, threads, cudaGetErrorString(e));
  cudaGetLastError();
}
int main() {
  probe<112>(576);
  probe<104>(576);
  probe<112>(544);
  probe<96>(640);
  probe<128>(512);
  return 0;
}
