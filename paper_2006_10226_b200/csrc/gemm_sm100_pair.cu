// gemm_sm100_pair.cu — the CTA-pair variants of the pixel-major tcgen05 GEMM (gemm_sm100.cuh
// with PAIR = true): clusters of 2 CTAs whose two M tiles form one cta_group::2 MMA (M = 256),
// each CTA staging its own A tile and half of the B tile -- 1.5x fewer operand bytes per SM per
// MAC for the streamed-weight layers.
#include "gemm_sm100.cuh"

namespace qnn {

cudaError_t launch_gemm_pair(const CUtensorMap& tmA, const CUtensorMap& tmB, const CUtensorMap* tmC,
                             const GemmParams& p, int mode, bool clamp, int grid, cudaStream_t stream) {
  return launch_gemm_impl<false, true, false>(tmA, tmB, tmC, p, mode, clamp, grid, stream);
}

}  // namespace qnn
