// internal.h — parameter blocks and launcher declarations shared by the host
// ABI (abi.cu) and the kernel translation units.  Not part of the public ABI.
#pragma once

#include <cstddef>
#include <cstdint>
#include <cuda.h>
#include <cuda_runtime.h>

namespace qnn {

constexpr int kMaxChanParams = 4096;   // per-channel requantize multipliers in kernel params
constexpr int kMaxQuantParams = 2048;  // per-channel quantize/dequantize params in kernel params

// ---------------------------------------------------------------------------
// Tensor-core implicit-GEMM conv / dense (gemm_sm100.cu)
//   rows m  = output pixels (n, p, q) in NHWC order,   M = N*P*Q
//   cols k  = output channels,                          Nout = K
//   reduce  = (r, s, c-chunk) k-blocks of BK bytes,     num_kb = R*S*nchunks
// ---------------------------------------------------------------------------
struct GemmEpilogue {
  const int32_t* off;      // [ncls][Kpad]: bias - zpA*colsum_cls + zpA*zpW*Cg*nvalid_cls (int32 wrap)
  const int64_t* off64;    // [ncls][Kpad]: the same offsets, exact (folded into the UPWARD fast path)
  const int32_t* mult;     // [Kpad] fixed-point multiplier M_k
  const int32_t* rsh;      // [Kpad] right shift 31 - shift_k (1..62)
  const uint8_t* rowcls;   // [P] row border class (nullptr => class 0)
  const uint8_t* colcls;   // [Q] column border class
  const int32_t* rowsum;   // [M] Term-3 row sums (nullptr when zp_W == 0)
  void* out;
  long long out_pitch;     // elements between consecutive output pixels
  int ncls, ncc;           // number of border classes, of column classes
  int Kpad;
  int32_t zpW;
  int out_dtype;           // DT_U8 / DT_S8 / DT_S32
  int tma_store;           // 8-bit output through per-warp TMA stores (pitch % 16 == 0)
  int32_t zp_out, lo, hi;  // lo/hi already include ReLU, act clamp and dtype range
  // fused residual add (nullptr: none): + R((res - res_zp) * res_M * 2^-res_rsh) before the clamp
  const uint8_t* res;
  long long res_pitch;     // bytes between consecutive pixels of the residual
  int32_t res_M, res_rsh, res_zp, res_s8;
};

// Division by a runtime divisor d >= 1 for dividends in [0, 2^31): q = umulhi(x, mul) >> shr
// with p = 31 + ceil(log2 d), mul = ceil(2^p / d), shr = p - 32 (d == 1: mul = 0, identity).
struct FastDiv {
  uint32_t d, mul, shr;
};
inline FastDiv make_fastdiv(uint32_t d) {
  FastDiv f{d, 0, 0};
  if (d > 1) {
    uint32_t l = 0;
    while ((1ull << l) < d) ++l;
    const uint32_t p = 31 + l;
    f.mul = (uint32_t)(((1ull << p) + d - 1) / d);
    f.shr = p - 32;
  }
  return f;
}
#ifdef __CUDACC__
__device__ __forceinline__ uint32_t fdiv(uint32_t x, const FastDiv& f) {
  return f.d == 1 ? x : (__umulhi(x, f.mul) >> f.shr);
}
#endif

// Channel-major GEMM (gemm_t.cu): wide 1x1 convs, D^T = W * A^T with the output channels on
// the TMEM lanes (per-lane requantize constants in registers).
#ifndef QNN_T_BN
#define QNN_T_BN 256
#endif
constexpr int kGemmTBN = QNN_T_BN;   // pixels per channel-major tile (MMA N; 128 or 256)
struct GemmTParams {
  int BK, stages, num_kb, num_ch_tiles, num_px_tiles;
  int w_res;             // weight block resident (else streamed per stage)
  int Kout;              // output channels (a multiple of 128, or 64: half a block)
  int has_res;           // fused residual add (qnn_conv2d_packed_add): tmR + these
  int32_t res_M, res_rsh, res_zp, res_s8;
  uint32_t idesc;
  const int32_t* mult;   // [Kpad]
  const int32_t* rsh;    // [Kpad]
  const int64_t* off64;  // [Kpad] (single border class)
  int32_t zp_out, lo, hi;
  int stage_bufs;         // output staging buffers per column group (1 or 2)
  int wsplit;             // weights packed as W - zp_W[k] in two s8 parts: two A k-blocks per k-block
  int pair;               // CTA pairs (clusters of 2, cta_group::2): MMA M = 256 over the two channel
                          // blocks of a pair, each CTA staging half of every pixel tile
  int esets;              // 2: two epilogue sets of 8 warps take alternate tiles (no residual, not
                          // build mode), each warp 2 x 64 pixel columns; else all 16 warps per tile
  int out_rb;             // staging / TMA-store row bytes: 128 (min(K_out, 128) in build mode)
  // build mode (small-C stems, K_out <= 64): the B operand X'[pixel][s*C + c] (one 32-byte
  // k-block per filter row, width fold of P:259's zero-point-padded input) is built in shared
  // memory by the warps of the unused quads 2 and 3 from TMA-staged raw input rows
  int build;
  int b_W, b_C, b_S, b_sw, b_pl, b_rowlen, b_nr, b_H, b_slot_bytes, b_raw_bytes;
  int rstages;            // raw-row ring depth (build mode)
  uint32_t b_zp4;         // zp_A in all four bytes (written outside the image: one border class)
  int P, Q, sh, pt;
  FastDiv fdQ, fdP;
  int dbg;   // QNN_GEMM_DEBUG (instrumented builds only): 1 skips the epilogue math, 2 the TMA stores
  unsigned long long* trace;   // QNN_GEMM_TRACE (instrumented builds only): CTA 0 clock64 events
};
size_t gemm_t_smem_bytes(int BK, int num_kb, int stages, bool w_res, int stage_bufs, int build_raw_bytes = -1,
                         int rstages = 0, int out_rb = 128, int wparts = 1, bool pair = false);
int gemm_t_max_stages(int BK, int num_kb, bool w_res, int stage_bufs, int build_raw_bytes = -1, int rstages = 0,
                      int out_rb = 128, int wparts = 1, bool pair = false);
cudaError_t launch_gemm_t(const CUtensorMap& tmX, const CUtensorMap& tmW, const CUtensorMap& tmC,
                          const CUtensorMap& tmR, const GemmTParams& p, int mode, bool clamp, bool s8out, int grid,
                          cudaStream_t stream);

struct GemmParams {
  int M, Nout;
  int num_kb, nchunks, S, dil_h, dil_w;
  int BK, BN, stages;
  int num_m_tiles, num_n_tiles;
  int im2col;              // 1 => A via im2col TMA over NHWC, 0 => A is a 2-D [M][C] matrix
  int b_res;               // 1 => all of B resident in smem (single N tile, small weights)
  int kps;                 // k-blocks per pipeline stage
  const uint8_t* a_base;   // A operand base (for L2 prefetch), a_pitch bytes per pixel / row
  long long a_pitch;
  int H, W, a_halo;        // input geometry for the prefetch range (a_halo = (R-1)*dil_h)
  int dbg;                 // profiling knobs (QNN_GEMM_DEBUG): 1 no epilogue math, 2 no stores,
                           // 4 no A loads, 8 no MMAs, 16 no TMEM loads; results are then garbage
  unsigned long long* trace; // profiling: CTA 0 event timestamps (QNN_GEMM_TRACE), else nullptr
  int P, Q, sh, sw, pt, pl;
  FastDiv fdQ, fdPQ;       // output-row decode: /Q and /(P*Q)
  uint32_t idesc;
  // a_build: the A tiles of a width-folded conv (X'[n, h, q, s*C + c] = A[n, h, q*sw + s*dw - pl, c])
  // are built in shared memory by two builder warps straight from the raw NHWC input, instead of
  // materialising X' in HBM and reading it back with TMA (same bytes, same border classes)
  int a_build;
  int a_W, a_C, a_S, a_sw, a_pl;
  int a_rowlen;            // bytes of one input row (W * C, contiguous channels)
  int a_nr;                // output rows a 128-pixel tile can touch: raw rows staged per tile = a_nr * R
  int a_H, a_zpfill;       // a_zpfill: bytes outside the image are zp_A (single border class)
  uint32_t a_zp4;          // zp_A replicated into 4 bytes
  FastDiv fdP;
  int a_slot_bytes;        // one output row's R raw rows (R * a_rowlen rounded up to 128 B: TMA alignment)
  int a_raw_bytes;         // per-stage raw-row region (a_nr * a_slot_bytes)
  // a_rows (stride-1 convs with resident weights): per tile and channel chunk ONE tiled TMA box
  // brings the input rows the tile touches ([a_nri][a_Wp][BK], zero padded) and every tap (r, s)
  // is an MMA whose A descriptor starts (r*Wp + s) pixels further into it; GEMM rows are the
  // flattened (p, q) positions with pitch Wp = Q + S - 1 per image (q >= Q rows are discarded)
  int a_rows;
  int a_Wp, a_T, a_nri;    // flattened pitch, tiles per image, input rows per box
  int a_stage_bytes;       // A bytes per pipeline stage (a_rows: a_nri * a_Wp * BK rounded up)
  FastDiv fdT, fdWp;
  GemmEpilogue e;
  int wsplit; // weights packed as W - zp_W[k] in two s8 parts (Term 3 in the contraction)
  int out_staging;  // the epilogue's TMA-store staging region is allocated (0: direct stores only)
  int epi_sets;     // epilogue warp sets taking alternate tiles (0: gemm_epi_sets; single N tile only)
  int pair;         // CTA pairs (cta_group::2): consecutive M tiles of a cluster of 2 form one M = 256 MMA
};

// Launch with programmatic stream serialization (PDL) so the kernel's prologue (barrier init,
// TMEM allocation, descriptor prefetch, resident-weight loads) overlaps the previous kernel's
// tail; the kernel must call pdl_wait() before it reads or writes activations.  QNN_NO_PDL=1
// launches normally (A/B measurements).
bool pdl_enabled();
// cluster > 1: thread-block clusters of that many CTAs along x
template <typename... KArgs, typename... Args>
cudaError_t launch_ex(void (*kern)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t s, int cluster,
                      Args&&... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute at[2];
  int n = 0;
  if (pdl_enabled()) {
    at[n].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[n++].val.programmaticStreamSerializationAllowed = 1;
  }
  if (cluster > 1) {
    at[n].id = cudaLaunchAttributeClusterDimension;
    at[n].val.clusterDim.x = (unsigned)cluster;
    at[n].val.clusterDim.y = 1;
    at[n++].val.clusterDim.z = 1;
  }
  cfg.attrs = at;
  cfg.numAttrs = n;
  return cudaLaunchKernelEx(&cfg, kern, static_cast<Args&&>(args)...);
}
template <typename... KArgs, typename... Args>
cudaError_t launch_pdl(void (*kern)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t s, Args&&... args) {
  return launch_ex(kern, grid, block, smem, s, 1, static_cast<Args&&>(args)...);
}
// co-resident clusters of `cluster` CTAs of `kern` with `smem` dynamic bytes (0 on error)
template <typename... KArgs>
int max_active_clusters(void (*kern)(KArgs...), dim3 block, size_t smem, int cluster) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(cluster * 64);
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = (unsigned)cluster;
  at[0].val.clusterDim.y = 1;
  at[0].val.clusterDim.z = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  int n = 0;
  if (cudaOccupancyMaxActiveClusters(&n, kern, &cfg) != cudaSuccess) {
    cudaGetLastError();
    return 0;
  }
  return n;
}

constexpr int kGemmBM = 128;
constexpr int kGemmEpiWarps = 16;
// 20 warps: the register file is allocated per 4-warp group, so 18 warps would cost as much
// as 20 (measured: 576 threads x 112 registers does not launch)
constexpr int kGemmThreads = 128 + 32 * kGemmEpiWarps;  // + one warpgroup: 2 idle, producer, MMA/allocator
constexpr int kGemmRoleBase = kGemmEpiWarps + 2;

// TMEM accumulator buffers: 512 columns split into the largest power-of-two count
// (<= 8) of buffers at least BN wide, so narrow tiles keep more tiles in flight.
__host__ __device__ inline int gemm_acc_bufs(int BN) {
  int n = 8;
  while (n > 2 && 512 / n < BN) n >>= 1;
  return n;
}
// Epilogue warp sets: with fewer than four 32-column chunks per tile and a single N
// tile, the nepi epilogue warps split into sets that take alternate tiles (each set
// still covers all 128 rows: 4 quads x (nepi/4)/nsets column groups).  nepi is 16, or 8
// when half of them build A tiles (a_build).
__host__ __device__ inline int gemm_epi_sets(int BN, int num_n_tiles, int nepi = kGemmEpiWarps) {
  const int nchunk = BN / 32;
  if (num_n_tiles != 1 || nchunk >= 3) return 1;
  const int s = 4 / nchunk;   // 1 chunk -> 4 sets, 2 chunks -> 2 sets
  return s < nepi / 4 ? s : nepi / 4;
}

// epilogue variants: MODE 0 = requantize UPWARD, 1 = requantize TONEAREST, 2 = raw int32
// out_staging = false: no TMA-store staging region (plans whose epilogue stores directly);
// pair: CTA-pair plans (each CTA stages half of each B k-block)
size_t gemm_smem_bytes(int BK, int BN, int stages, int ncls, int b_res_kb, int kps, int raw_bytes = 0,
                       int a_stage_bytes = 0, int bparts = 1, bool out_staging = true, bool pair = false);
int gemm_max_stages(int BK, int BN, int ncls, int b_res_kb, int kps, int raw_bytes = 0, int a_stage_bytes = 0,
                    int bparts = 1, bool out_staging = true, bool pair = false);
cudaError_t launch_gemm(const CUtensorMap& tmA, const CUtensorMap& tmB, const CUtensorMap* tmC,
                        const GemmParams& p, int mode, bool clamp, int grid, cudaStream_t stream);
cudaError_t launch_gemm_split(const CUtensorMap& tmA, const CUtensorMap& tmB, const CUtensorMap* tmC,
                              const GemmParams& p, int mode, bool clamp, int grid, cudaStream_t stream);
cudaError_t launch_gemm_pair(const CUtensorMap& tmA, const CUtensorMap& tmB, const CUtensorMap* tmC,
                             const GemmParams& p, int mode, bool clamp, int grid, cudaStream_t stream);
cudaError_t launch_gemm_arows(const CUtensorMap& tmA, const CUtensorMap& tmB, const CUtensorMap* tmC,
                              const GemmParams& p, int mode, bool clamp, int grid, cudaStream_t stream);

// ---------------------------------------------------------------------------
// Prepack / auxiliary kernels (prep.cu)
// ---------------------------------------------------------------------------
struct ClassTable {
  int ncr, ncc;
  int r_lo[32], r_hi[32];  // valid filter-row range per row class
  int s_lo[32], s_hi[32];  // valid filter-col range per col class
};

cudaError_t launch_pack_weights(const void* W, void* Wp, int K, int RS, int C, int Cw, int Kpad,
                                cudaStream_t s, int perm32 = 0, int split = 0, int w_signed = 1,
                                const int32_t* zpv = nullptr);
cudaError_t launch_fold_offsets(const void* W, int w_signed, const int32_t* bias, int K, int R, int S, int C,
                                int32_t zpA, int32_t zpW, const ClassTable& ct, int32_t* off, int64_t* off64, int Kpad,
                                cudaStream_t s, const int32_t* zpv = nullptr);
cudaError_t launch_pack_dw_weights(const void* W, int w_signed, int32_t zpW, int16_t* Wd, int C, int RS,
                                   cudaStream_t s, const int32_t* zpv = nullptr);
cudaError_t launch_pad_channels(const void* in, long long in_cstride, void* out, int Cp, long long npix, int C,
                                cudaStream_t s);
cudaError_t launch_fold_width(const void* in, long long in_cstride, void* out, int N, int H, int W, int C, int Q, int S,
                              int sw, int pl, int dw, int Cf, cudaStream_t s);
cudaError_t launch_pixel_sums(const void* in, int a_signed, long long in_cstride, int C, long long npix,
                              int32_t* pixsum, cudaStream_t s);
cudaError_t launch_window_sums(const int32_t* pixsum, int N, int H, int W, int P, int Q, int R, int S, int sh,
                               int sw, int pt, int pl, int dh, int dw, int32_t* rowsum, cudaStream_t s);

// ---------------------------------------------------------------------------
// Depthwise conv (depthwise.cu): subtract-first lowering on CUDA cores
// ---------------------------------------------------------------------------
struct DwParams {
  const void* in;
  const int16_t* w;        // [R*S][C] holding W - zp_W
  const int32_t* bias;     // [C] or nullptr
  const int32_t* mult;     // [C]
  const int32_t* rsh;      // [C]
  void* out;
  long long in_cstride, out_cstride;
  int N, H, W, C, P, Q, R, S, sh, sw, pt, pl, dh, dw;
  int a_signed;
  int32_t zpA;
  int out_dtype, requant, mode;
  int32_t zp_out, lo, hi;
  int w_fits_s8;           // every W - zp_W in [-128, 127] (dp4a path)
  int qseg;                // dp4a path: column blocks per task (set by the launcher)
  int dwt_cs, dwt_wb, dwt_bp, dwt_stage_bytes;   // TMA-staged path: channel slice, box width, rows/band
};
cudaError_t launch_depthwise(const DwParams& p, cudaStream_t s);
bool launch_depthwise3(const DwParams& p, int clamp, cudaStream_t s);   // clamp: 0 none, 1 hi, 2 lo+hi
// 3x3 depthwise with TMA-staged input bands (depthwise_tma.cu): plan fills the dwt_* fields
bool dwtma_plan(DwParams& p);
cudaError_t launch_depthwise_tma(const CUtensorMap& tm, const DwParams& p, int clamp, cudaStream_t s);

// Tensor-core depthwise conv (depthwise_tc.cu): C % 16 == 0, s8 weights with zp_W == 0,
// stride 1 or 2, 8-bit requantized output.
struct DwTcParams {
  const uint8_t* wpk;       // [ceil(C/32)][R*S][1024] diagonal B tiles
  const int32_t* mult;      // [Cpad]
  const int32_t* rsh;       // [Cpad]
  const int32_t* off;       // [ncls][Cpad] bias - zp_A * sum_{valid taps} W (int32 wrap)
  const int64_t* off64;     // [ncls][Cpad] the same, exact
  const uint8_t* rowcls;    // [P] border row class
  const uint8_t* colcls;    // [Q] border column class
  uint8_t* out;             // NHWC, out_cs bytes per pixel
  long long out_cs;
  int N, C, Cpad, P, Q, R, S, sh, sw, pt, pl, ncls, ncc;
  int T, Wp, in_rows, nplanes, region_bytes, stage_bytes, tiles_per_item, nstrips, ncs, items, stages;
  uint32_t idesc;
  int32_t zp_out, lo, hi;
  unsigned long long* trace;   // profiling (QNN_DWTC_TRACE, instrumented builds): CTA 0 timestamps
};
bool dwtc_plan(DwTcParams& p);
cudaError_t launch_depthwise_tc(const CUtensorMap& tmA, const DwTcParams& p, int mode, bool clamp, bool s8out,
                                cudaStream_t s);
cudaError_t launch_pack_dwtc(const void* W, int C, int RS, void* wpk, cudaStream_t s);

// ---------------------------------------------------------------------------
// Elementwise (elementwise.cu)
// ---------------------------------------------------------------------------
struct RequantParams {
  const void* in;
  void* out;
  long long count, inner;
  int cext, nch;
  int in_dt, out_dt, mode;
  int32_t in_zp, out_zp, lo, hi;
  int32_t mult[kMaxChanParams];
  int8_t rsh[kMaxChanParams];
};
struct QuantParams {
  const void* in;
  void* out;
  long long count, inner;
  int cext, nch;
  int q_dt;               // quantized dtype (out of quantize / in of dequantize)
  int32_t lo, hi;
  float scale[kMaxQuantParams];
  int32_t zp[kMaxQuantParams];
};
cudaError_t launch_requantize(const RequantParams& p, cudaStream_t s);
cudaError_t launch_quantize(const QuantParams& p, cudaStream_t s);
cudaError_t launch_dequantize(const QuantParams& p, cudaStream_t s);

// ---------------------------------------------------------------------------
// Glue (glue.cu): qnn.add, pooling
// ---------------------------------------------------------------------------
struct AddParams {
  const void* a;
  const void* b;
  void* out;
  long long count;
  int vec;                      // 16-byte vector path (all three pointers 16-B aligned)
  bool a_s8, b_s8, o_s8;
  int32_t zp_a, zp_b, zp_out;
  int32_t Ma, Mb;               // fixed-point multipliers of s_a/s_out, s_b/s_out
  int ra, rb;                   // right shifts (31 - shift), 1..62
  int mode, relu;
};
cudaError_t launch_add(const AddParams& p, cudaStream_t s);
struct PoolParams {
  const void* in;
  void* out;
  long long in_cs, out_cs;
  int N, H, W, C, P, Q, R, S, sh, sw, pt, pl;
  bool s8, avg;
};
cudaError_t launch_pool(const PoolParams& p, cudaStream_t s);

// launch accounting (abi.cu)
void count_launch(int n = 1);

}  // namespace qnn
