// gemm_sm100.cu — host side of the pixel-major tcgen05 GEMM (gemm_sm100.cuh): shared-memory
// sizing and the variant dispatch; the plain-weight kernel variants are instantiated here, the
// split-weight ones in gemm_sm100_split.cu (a second translation unit, compiled in parallel, so
// the plain kernels' code carries none of the split bookkeeping).
#include "gemm_sm100.cuh"

namespace qnn {

// b_res_kb > 0: the whole B operand (b_res_kb k-blocks) stays resident in smem and
// the pipeline stages carry A only.
// Each pipeline stage carries kps consecutive k-blocks (one barrier round trip, one
// commit per stage: amortises the per-stage synchronisation for narrow k-blocks).
size_t gemm_smem_bytes(int BK, int BN, int stages, int ncls, int b_res_kb, int kps, int raw_bytes,
                       int a_stage_bytes, int bparts, bool out_staging, bool pair) {
  // (bparts = 2: split weights, two B k-blocks per A k-block; b_res_kb then counts both parts;
  // pair: a CTA of a cta_group::2 pair stages half of each B k-block)
  const size_t a = a_stage_bytes ? (size_t)a_stage_bytes : (size_t)kGemmBM * BK * kps,
               b = (size_t)(pair ? BN / 2 : BN) * BK * bparts;
  const size_t ring = b_res_kb > 0 ? stages * a + (size_t)b_res_kb * (b / bparts) : stages * (a + b * kps);
  return 1024 + ring + (size_t)stages * raw_bytes + (out_staging ? kStageOutBytes : 0) + kParamBytes +
         off_table_bytes(ncls, BN) + 512;
}

int gemm_max_stages(int BK, int BN, int ncls, int b_res_kb, int kps, int raw_bytes, int a_stage_bytes, int bparts,
                    bool out_staging, bool pair) {
  const size_t budget = 227 * 1024;
  int s = 8;
  while (s > 2 &&
         gemm_smem_bytes(BK, BN, s, ncls, b_res_kb, kps, raw_bytes, a_stage_bytes, bparts, out_staging, pair) > budget)
    --s;
  return s;
}

cudaError_t launch_gemm(const CUtensorMap& tmA, const CUtensorMap& tmB, const CUtensorMap* tmC, const GemmParams& p,
                        int mode, bool clamp, int grid, cudaStream_t stream) {
  if (p.wsplit) return launch_gemm_split(tmA, tmB, tmC, p, mode, clamp, grid, stream);
  if (p.pair) return launch_gemm_pair(tmA, tmB, tmC, p, mode, clamp, grid, stream);
  if (p.a_rows) return launch_gemm_arows(tmA, tmB, tmC, p, mode, clamp, grid, stream);
  return launch_gemm_impl<false, false, false>(tmA, tmB, tmC, p, mode, clamp, grid, stream);
}

}  // namespace qnn
