// gemm_sm100_split.cu — the split-weight variants of the pixel-major tcgen05 GEMM
// (gemm_sm100.cuh with SPLIT = true): weights packed as W - zp_W[k] in two s8 k-block sets, a
// second MMA per K step against the same activation tile, so Term 3 (zp_W * sum A) is
// computed by the tensor cores (reading R11, per-channel zero points).
#include "gemm_sm100.cuh"

namespace qnn {

cudaError_t launch_gemm_split(const CUtensorMap& tmA, const CUtensorMap& tmB, const CUtensorMap* tmC,
                              const GemmParams& p, int mode, bool clamp, int grid, cudaStream_t stream) {
  // (split weights on staged-row plans included: the AROWS path is a runtime choice there)
  return p.a_rows ? launch_gemm_impl<true, false, true>(tmA, tmB, tmC, p, mode, clamp, grid, stream)
                  : launch_gemm_impl<true, false, false>(tmA, tmB, tmC, p, mode, clamp, grid, stream);
}

}  // namespace qnn
