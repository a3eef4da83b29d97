// gemm_sm100_arows.cu — the staged-row (a_rows) variants of the pixel-major tcgen05 GEMM
// (gemm_sm100.cuh with AROWS = true): stride-1 convs whose input rows are staged once per
// channel chunk and whose filter taps are addressed through the MMA descriptor.  A separate
// instantiation so that neither path's code costs the other registers.
#include "gemm_sm100.cuh"

namespace qnn {

cudaError_t launch_gemm_arows(const CUtensorMap& tmA, const CUtensorMap& tmB, const CUtensorMap* tmC,
                              const GemmParams& p, int mode, bool clamp, int grid, cudaStream_t stream) {
  return launch_gemm_impl<false, false, true>(tmA, tmB, tmC, p, mode, clamp, grid, stream);
}

}  // namespace qnn
