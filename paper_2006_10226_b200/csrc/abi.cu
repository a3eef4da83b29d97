#include <cstdio>
// abi.cu — the C ABI of libqnn.so (include/qnn.h): argument validation, the
// host half of the paper's QNN canonicalisation — fixed-point
// multiplier derivation, border-class tables, compile-time folding plans —
// TMA descriptor encoding, and kernel launches.  No compute happens on the
// host: every step of the path runs in the kernels of this library.
#include <cudaTypedefs.h>

#include <algorithm>
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <map>
#include <mutex>
#include <vector>

#include "../../include/qnn.h"
#include "common.cuh"
#include "internal.h"

namespace qnn {

static thread_local uint64_t g_launches = 0;
void count_launch(int n) { g_launches += (uint64_t)n; }

bool pdl_enabled() {
  static const bool on = std::getenv("QNN_NO_PDL") == nullptr;
  return on;
}

static int sm_count() {
  static int cached[64] = {0};
  int dev = 0;
  cudaGetDevice(&dev);
  if (dev < 64 && cached[dev]) return cached[dev];
  int sms = 148;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  if (dev < 64) cached[dev] = sms;
  return sms;
}

// ---------------------------------------------------------------------------
// Driver entry points for TMA descriptor encoding (no link against libcuda)
// ---------------------------------------------------------------------------
static PFN_cuTensorMapEncodeTiled_v12000 p_encode_tiled = nullptr;
static PFN_cuTensorMapEncodeIm2col_v12000 p_encode_im2col = nullptr;
static int g_driver_version = 0;

static bool load_driver_entry_points() {
  static std::once_flag once;
  static bool ok = false;
  std::call_once(once, [] {
    cudaDriverEntryPointQueryResult q1 = cudaDriverEntryPointSymbolNotFound, q2 = cudaDriverEntryPointSymbolNotFound;
    void* f1 = nullptr;
    void* f2 = nullptr;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &f1, cudaEnableDefault, &q1) == cudaSuccess &&
        cudaGetDriverEntryPoint("cuTensorMapEncodeIm2col", &f2, cudaEnableDefault, &q2) == cudaSuccess &&
        q1 == cudaDriverEntryPointSuccess && q2 == cudaDriverEntryPointSuccess) {
      p_encode_tiled = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(f1);
      p_encode_im2col = reinterpret_cast<PFN_cuTensorMapEncodeIm2col_v12000>(f2);
      ok = true;
    }
    cudaDriverGetVersion(&g_driver_version);
  });
  return ok;
}

static CUtensorMapSwizzle swizzle_for(int row_bytes) {
  return row_bytes == 128 ? CU_TENSOR_MAP_SWIZZLE_128B
                          : (row_bytes == 64 ? CU_TENSOR_MAP_SWIZZLE_64B : CU_TENSOR_MAP_SWIZZLE_32B);
}

// Drivers up to 13.1 mis-handle a descriptor flag for tensors under 128 KiB;
// clear it as the CUDA tooling does for those drivers.
static void small_tensor_fixup(CUtensorMap* m, unsigned long long bytes) {
  if (g_driver_version <= 13010 && bytes < 131072ull) reinterpret_cast<uint64_t*>(m)[1] &= ~(1ull << 21);
}

static bool encode_2d(CUtensorMap* m, const void* base, uint64_t cols, uint64_t rows, uint64_t pitch_bytes,
                      uint32_t box_cols, uint32_t box_rows, bool swizzle = true) {
  const cuuint64_t dims[2] = {cols, rows};
  const cuuint64_t strides[1] = {pitch_bytes};
  const cuuint32_t box[2] = {box_cols, box_rows};
  const cuuint32_t estr[2] = {1, 1};
  CUresult r = p_encode_tiled(m, CU_TENSOR_MAP_DATA_TYPE_UINT8, 2, const_cast<void*>(base), dims, strides, box, estr,
                              CU_TENSOR_MAP_INTERLEAVE_NONE,
                              swizzle ? swizzle_for((int)box_cols) : CU_TENSOR_MAP_SWIZZLE_NONE,
                              CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  small_tensor_fixup(m, pitch_bytes * rows);
  return r == CUDA_SUCCESS;
}

static bool encode_im2col(CUtensorMap* m, const void* base, int C, int W, int H, int N, uint64_t pitch_bytes,
                          int lower_w, int lower_h, int upper_w, int upper_h, int BK, int sw, int sh) {
  const cuuint64_t dims[4] = {(cuuint64_t)C, (cuuint64_t)W, (cuuint64_t)H, (cuuint64_t)N};
  const cuuint64_t strides[3] = {pitch_bytes, pitch_bytes * W, pitch_bytes * W * H};
  const int lower[2] = {lower_w, lower_h};
  const int upper[2] = {upper_w, upper_h};
  const cuuint32_t estr[4] = {1, (cuuint32_t)sw, (cuuint32_t)sh, 1};
  CUresult r = p_encode_im2col(m, CU_TENSOR_MAP_DATA_TYPE_UINT8, 4, const_cast<void*>(base), dims, strides, lower,
                               upper, (cuuint32_t)BK, (cuuint32_t)kGemmBM, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                               swizzle_for(BK), CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  small_tensor_fixup(m, pitch_bytes * W * H * N);
  return r == CUDA_SUCCESS;
}

// ---------------------------------------------------------------------------
// Fixed-point multiplier (reading R2): from the IEEE-754 fields of m,
// M = round_half_away(significand * 2^31) with significand in [0.5, 1).
// ---------------------------------------------------------------------------
static bool derive_multiplier(double m, int32_t* M, int32_t* shift) {
  if (!(m > 0.0) || !std::isfinite(m)) return false;
  uint64_t bits;
  std::memcpy(&bits, &m, sizeof(bits));
  const int biased = (int)((bits >> 52) & 0x7FF);
  if (biased == 0) {  // subnormal: renormalise through frexp
    int e = 0;
    const double sig = std::frexp(m, &e);
    int64_t Mi = (int64_t)std::floor(std::ldexp(sig, 31) + 0.5);
    if (Mi == (int64_t)1 << 31) {
      Mi >>= 1;
      ++e;
    }
    *M = (int32_t)Mi;
    *shift = e;
    return true;
  }
  const uint64_t mant = (bits & ((1ull << 52) - 1)) | (1ull << 52);  // in [2^52, 2^53)
  int e = biased - 1023 + 1;                                          // m = (mant / 2^53) * 2^e
  uint64_t Mi = (mant + (1ull << 21)) >> 22;                          // round half up (= away, m > 0)
  if (Mi == (1ull << 31)) {
    Mi = 1ull << 30;
    ++e;
  }
  *M = (int32_t)Mi;
  *shift = e;
  return true;
}

// multiplier -> (M, right shift) for the kernels (reading R15).  Every product the kernels
// round is |x * M| < 2^63 (x = an int32 accumulator, an 8-bit code minus its zero point, or an
// int32 input minus its zero point, |x| <= 2^32 - 1; M < 2^31), so a right shift >= 64 rounds
// it to 0 in both modes and is replaced by M = 0.  rsh = 63 is kept: with int32 input and
// zp_in != 0, |x * M| reaches [2^62, 2^63) and rounds to +-1 (the 64-bit rq_round handles it).
static bool kernel_multiplier(double m, int32_t* M, int32_t* rsh) {
  int32_t Mi, sh;
  if (!derive_multiplier(m, &Mi, &sh)) return false;
  const int r = 31 - sh;
  if (r < 1) return false;  // m >= 2^30: unsupported (reading R15)
  if (r > 63) {
    *M = 0;
    *rsh = 1;
  } else {
    *M = Mi;
    *rsh = r;
  }
  return true;
}

static bool dtype_range(qnn_dtype_t dt, int64_t* lo, int64_t* hi) {
  switch (dt) {
    case QNN_S8: *lo = -128; *hi = 127; return true;
    case QNN_U8: *lo = 0; *hi = 255; return true;
    case QNN_S32: *lo = INT32_MIN; *hi = INT32_MAX; return true;
    default: return false;
  }
}
static bool is_8bit(qnn_dtype_t dt) { return dt == QNN_S8 || dt == QNN_U8; }
static bool zp_ok(qnn_dtype_t dt, int32_t zp) {
  int64_t lo, hi;
  return dtype_range(dt, &lo, &hi) && zp >= lo && zp <= hi;
}
static bool scale_ok(float s) { return std::isfinite(s) && s > 0.0f; }
static size_t align256(size_t x) { return (x + 255) & ~(size_t)255; }
static int round_up(int x, int m) { return (x + m - 1) / m * m; }

// ---------------------------------------------------------------------------
// Conv plan: everything the host derives from the descriptor
// ---------------------------------------------------------------------------
struct ConvPlan {
  bool depthwise = false;
  bool dwtc = false;       // depthwise on the tensor cores (weights packed for it)
  int P = 0, Q = 0;
  long long M = 0;
  int in_cs = 0, out_cs = 0;
  // tensor-core path
  bool pad_copy = false;
  bool fold = false;     // width fold: (s, c) -> channels of a copy, filter becomes R x 1 (small-C stems)
  bool a_build = false;  // fold done in shared memory by the GEMM's builder warps (no X' copy in HBM)
  int a_ib = 0, a_nr = 0, a_slot_bytes = 0, a_raw_bytes = 0;
  bool a_zpfill = false;  // a_build writes zp_A outside the image (single border class)
  bool a_rows = false;    // stride-1 convs: staged input rows + per-tap descriptor offsets
  bool pair = false;      // CTA pairs (cta_group::2): consecutive M tiles form one M = 256 MMA
  int a_Wp = 0, a_T = 0, a_nri = 0, a_stage_bytes = 0;
  int Ct = 0;            // channel count / pitch seen by TMA
  // geometry of the GEMM as the kernel sees it (differs from the descriptor when folded)
  int gW = 0, gS = 0, g_sw = 0, g_pl = 0, g_pr = 0, g_dw = 0;
  int BK = 0, nchunks = 0, Cw = 0, BN = 0, Kpad = 0, num_n = 0, num_m = 0, stages = 0, b_res_kb = 0, kps = 1;
  int grid = 0;   // persistent CTAs (a multiple of num_n when tiles > SMs)
  bool im2col = false;
  ClassTable ct{};
  std::vector<uint8_t> rowcls, colcls;
  // epilogue
  bool requant = false;
  int32_t lo = 0, hi = 0, zp_out = 0;
  int mode = 0;
  qnn_dtype_t out_dt = QNN_S32;
  // packed blob layout
  // channel-major GEMM (gemm_t.cu) for wide pointwise layers: chosen at plan time (its weights
  // are packed in the perm32 lane order as a second copy, pk_wt); at run time it also needs a
  // 16-B aligned output, else the pixel-major kernel runs on pk_w
  // weight zero points: per-channel vector (f4) or the scalar repeated; wsplit: Term 3 folded
  // into the contraction (weights packed as W - zp_W[k] in two s8 parts), else row sums
  std::vector<int32_t> zpv;
  bool zp_vec = false, any_zpw = false, wsplit = false;
  size_t pk_zpv = 0;
  bool trans = false, t_wres = false;
  int t_stages = 0, t_Kt = 0, t_bufs = 1;
  bool t_pair = false;   // CTA pairs (cta_group::2) over channel-block pairs: M = 256 per MMA
  // channel-major build mode (small-C stems with K_out <= 64): X' built in smem by the idle quads
  bool t_build = false;
  int t_ib = 0, t_nr = 0, t_slot = 0, t_raw = 0, t_rstages = 0;
  size_t pk_wt = 0;
  size_t pk_w = 0, pk_off = 0, pk_off64 = 0, pk_dwtc_w = 0, pk_mult = 0, pk_rsh = 0, pk_rowcls = 0, pk_colcls = 0, pk_bias = 0, pk_total = 0;
  // workspace layout
  size_t ws_pad = 0, ws_pixsum = 0, ws_rowsum = 0, ws_total = 0;
};

static qnn_status_t build_classes(int out, int in, int ksz, int stride, int pad, int dil, int* lo, int* hi, int* ncls,
                                  std::vector<uint8_t>& cls) {
  std::map<std::pair<int, int>, int> ids;
  cls.assign(out, 0);
  for (int p = 0; p < out; ++p) {
    int a = ksz, b = -1;
    for (int r = 0; r < ksz; ++r) {
      const long long h = (long long)p * stride + (long long)r * dil - pad;
      if (h >= 0 && h < in) {
        a = std::min(a, r);
        b = std::max(b, r);
      }
    }
    if (b < 0) {
      a = 0;
      b = -1;
    }
    auto key = std::make_pair(a, b);
    auto it = ids.find(key);
    int id;
    if (it == ids.end()) {
      id = (int)ids.size();
      if (id >= 32) return QNN_ERR_UNSUPPORTED;
      ids[key] = id;
      lo[id] = a;
      hi[id] = b;
    } else {
      id = it->second;
    }
    cls[p] = (uint8_t)id;
  }
  *ncls = (int)ids.size();
  return QNN_OK;
}

static qnn_status_t validate_output(const qnn_output_params_t* o, ConvPlan& pl) {
  if (!o) {
    pl.requant = false;
    pl.out_dt = QNN_S32;
    pl.lo = INT32_MIN;
    pl.hi = INT32_MAX;
    return QNN_OK;
  }
  if (!is_8bit(o->out_dtype)) return QNN_ERR_UNSUPPORTED;
  if (!scale_ok(o->output_scale) || !zp_ok(o->out_dtype, o->output_zero_point)) return QNN_ERR_INVALID_VALUE;
  if (o->rounding != QNN_ROUND_UPWARD && o->rounding != QNN_ROUND_TONEAREST) return QNN_ERR_INVALID_VALUE;
  int64_t qlo, qhi;
  dtype_range(o->out_dtype, &qlo, &qhi);
  int64_t lo = std::max<int64_t>(qlo, o->act_min);
  if (o->relu) lo = std::max<int64_t>(lo, o->output_zero_point);
  const int64_t hi = std::min<int64_t>(qhi, o->act_max);
  if (lo > hi) return QNN_ERR_INVALID_VALUE;
  pl.requant = true;
  pl.out_dt = o->out_dtype;
  pl.lo = (int32_t)lo;
  pl.hi = (int32_t)hi;
  pl.zp_out = o->output_zero_point;
  pl.mode = (int)o->rounding;
  return QNN_OK;
}

static qnn_status_t make_plan(const qnn_conv2d_desc_t* d, const qnn_output_params_t* o, ConvPlan& pl,
                             bool need_scales = true) {
  if (!d) return QNN_ERR_INVALID_VALUE;
  if (d->N <= 0 || d->H <= 0 || d->W <= 0 || d->C <= 0 || d->K <= 0 || d->R <= 0 || d->S <= 0)
    return QNN_ERR_INVALID_VALUE;
  if (d->stride_h <= 0 || d->stride_w <= 0 || d->dil_h <= 0 || d->dil_w <= 0 || d->groups <= 0)
    return QNN_ERR_INVALID_VALUE;
  if (d->pad_t < 0 || d->pad_l < 0 || d->pad_b < 0 || d->pad_r < 0) return QNN_ERR_INVALID_VALUE;
  if (!is_8bit(d->input_dtype) || !is_8bit(d->kernel_dtype)) return QNN_ERR_UNSUPPORTED;
  if (!zp_ok(d->input_dtype, d->input_zero_point) || !zp_ok(d->kernel_dtype, d->kernel_zero_point))
    return QNN_ERR_INVALID_VALUE;
  if (d->C % d->groups != 0 || d->K % d->groups != 0) return QNN_ERR_INVALID_VALUE;
  // weight zero points: scalar, or one per output channel (f4; reading R11)
  if (d->num_kernel_zero_points != 0) {
    if (d->num_kernel_zero_points != d->K || !d->kernel_zero_points) return QNN_ERR_INVALID_VALUE;
    pl.zp_vec = true;
    pl.zpv.assign(d->kernel_zero_points, d->kernel_zero_points + d->K);
    for (int32_t z : pl.zpv)
      if (!zp_ok(d->kernel_dtype, z)) return QNN_ERR_INVALID_VALUE;
  } else {
    pl.zpv.assign(d->K, d->kernel_zero_point);
  }
  for (int32_t z : pl.zpv) pl.any_zpw |= z != 0;
  pl.depthwise = d->groups > 1;
  if (pl.depthwise && !(d->groups == d->C && d->K == d->C)) return QNN_ERR_UNSUPPORTED;
  const long long Pn = ((long long)d->H + d->pad_t + d->pad_b - (long long)d->dil_h * (d->R - 1) - 1) / d->stride_h + 1;
  const long long Qn = ((long long)d->W + d->pad_l + d->pad_r - (long long)d->dil_w * (d->S - 1) - 1) / d->stride_w + 1;
  if (d->H + d->pad_t + d->pad_b < (long long)d->dil_h * (d->R - 1) + 1 ||
      d->W + d->pad_l + d->pad_r < (long long)d->dil_w * (d->S - 1) + 1 || Pn <= 0 || Qn <= 0)
    return QNN_ERR_INVALID_VALUE;
  pl.P = (int)Pn;
  pl.Q = (int)Qn;
  pl.M = (long long)d->N * Pn * Qn;
  if (pl.M > INT32_MAX) return QNN_ERR_UNSUPPORTED;
  pl.in_cs = d->in_cstride ? d->in_cstride : d->C;
  pl.out_cs = d->out_cstride ? d->out_cstride : d->K;
  if (pl.in_cs < d->C || pl.out_cs < d->K) return QNN_ERR_INVALID_VALUE;
  // reading R10: int32 exactness of the accumulator
  const long long KK = (long long)(d->C / d->groups) * d->R * d->S;
  if (KK * 255LL * 255LL > (long long)INT32_MAX) return QNN_ERR_UNSUPPORTED;
  // scales
  if (!scale_ok(d->input_scale)) return QNN_ERR_INVALID_VALUE;
  if (o && need_scales) {
    if (!d->kernel_scales || !(d->num_kernel_scales == 1 || d->num_kernel_scales == d->K)) return QNN_ERR_INVALID_VALUE;
    for (int i = 0; i < d->num_kernel_scales; ++i)
      if (!scale_ok(d->kernel_scales[i])) return QNN_ERR_INVALID_VALUE;
  }
  qnn_status_t st = validate_output(o, pl);
  if (st != QNN_OK) return st;

  if (pl.depthwise) {
    const int C = d->C, RS = d->R * d->S;
    size_t off = 0;
    pl.pk_w = off;
    off = align256(off + (size_t)RS * C * 2);
    pl.pk_bias = off;
    off = align256(off + (size_t)C * 4);
    pl.pk_mult = off;
    off = align256(off + (size_t)(C + 31) / 32 * 32 * 4);
    pl.pk_rsh = off;
    off = align256(off + (size_t)(C + 31) / 32 * 32 * 4);
    // tensor-core path (depthwise_tc.cu): diagonal B tiles, per-border-class folded offsets
    if (pl.zp_vec) {
      pl.pk_zpv = off;
      off = align256(off + (size_t)C * 4);
    }
    pl.dwtc = C % 16 == 0 && d->kernel_dtype == QNN_S8 && !pl.any_zpw && d->dil_h == 1 &&
              d->dil_w == 1 && (d->stride_h == 1 || d->stride_h == 2) && (d->stride_w == 1 || d->stride_w == 2) &&
              pl.in_cs % 16 == 0 && pl.out_cs % 16 == 0;
    if (pl.dwtc) {
      if (build_classes(pl.P, d->H, d->R, d->stride_h, d->pad_t, d->dil_h, pl.ct.r_lo, pl.ct.r_hi, &pl.ct.ncr,
                        pl.rowcls) != QNN_OK ||
          build_classes(pl.Q, d->W, d->S, d->stride_w, d->pad_l, d->dil_w, pl.ct.s_lo, pl.ct.s_hi, &pl.ct.ncc,
                        pl.colcls) != QNN_OK ||
          pl.ct.ncr * pl.ct.ncc > 64)
        pl.dwtc = false;
    }
    if (pl.dwtc) {
      const int Cpad = (C + 31) / 32 * 32, ncls = pl.ct.ncr * pl.ct.ncc;
      pl.Kpad = Cpad;
      pl.pk_dwtc_w = off;
      off = align256(off + (size_t)RS * Cpad * 32);
      pl.pk_off = off;
      off = align256(off + (size_t)ncls * Cpad * 4);
      pl.pk_off64 = off;
      off = align256(off + (size_t)ncls * Cpad * 8);
      pl.pk_rowcls = off;
      off = align256(off + (size_t)pl.P);
      pl.pk_colcls = off;
      off = align256(off + (size_t)pl.Q);
    }
    pl.pk_total = off;
    pl.ws_total = 0;
    return QNN_OK;
  }

  // ------------------------------------------------------------ tensor-core plan
  const bool tma_pitch_ok = (pl.in_cs % 16) == 0;
  pl.gW = d->W; pl.gS = d->S; pl.g_sw = d->stride_w; pl.g_pl = d->pad_l; pl.g_pr = d->pad_r; pl.g_dw = d->dil_w;
  pl.fold = (!tma_pitch_ok || d->C < 16) && d->S > 1 && d->S * d->C <= 128;
  if (pl.fold) {
    // X'[n, h, q, s*C + c] = A[n, h, q*sw + s*dw - pl, c] (0 outside): an R x 1 conv over X'
    pl.Ct = round_up(d->S * d->C, 16);
    pl.gW = (int)Qn; pl.gS = 1; pl.g_sw = 1; pl.g_pl = 0; pl.g_pr = 0; pl.g_dw = 1;
  } else {
    pl.pad_copy = !tma_pitch_ok;
    pl.Ct = pl.pad_copy ? round_up(d->C, 16) : d->C;
  }
  {
    int best_bk = 128, best = INT32_MAX;
    for (int bk : {128, 64, 32}) {
      const int n = (pl.Ct + bk - 1) / bk;
      if (n * bk < best) {
        best = n * bk;
        best_bk = bk;
      }
    }
    pl.BK = best_bk;
    pl.nchunks = (pl.Ct + best_bk - 1) / best_bk;
    pl.Cw = pl.nchunks * best_bk;
  }
  pl.num_m = (int)((pl.M + kGemmBM - 1) / kGemmBM);
  {
    // N tiling: fewest N tiles (BN <= 256) unless narrower tiles fill the persistent grid's last
    // round better -- cost ~ rounds x (BN + 32) (wave quantisation of the small-M deep layers,
    // e.g. ResNet-50 layer4 at batch 256: 196 tiles on 148 SMs).  With several N tiles and more
    // tiles than SMs the grid is a multiple of num_n, so every CTA keeps one N tile (tile t =
    // m * num_n + n, t += grid): its per-column epilogue parameters are staged once and its
    // weights can stay resident; rounds = ceil(num_m / (grid / num_n)).
    const int sms = sm_count();
    // QNN_NO_NSTAT=1: the plain persistent order (A/B measurements)
    static const bool no_nstat = std::getenv("QNN_NO_NSTAT") != nullptr;
    const int n0 = (d->K + 255) / 256;
    long long best = -1;
    for (int nn = n0; nn <= std::max(n0, (d->K + 63) / 64); ++nn) {
      const int bn = round_up((d->K + nn - 1) / nn, 32);
      if (bn < 64 && nn > n0) break;
      if (nn > sms) break;
      const long long tiles = (long long)pl.num_m * nn;
      const long long rounds = tiles <= sms ? 1
                               : no_nstat ? (tiles + sms - 1) / sms
                                          : (pl.num_m + sms / nn - 1) / (sms / nn);
      const long long cost = rounds * (bn + 32);
      if (best < 0 || cost < best) {
        best = cost;
        pl.num_n = nn;
        pl.BN = bn;
      }
    }
    const long long tiles = (long long)pl.num_m * pl.num_n;
    pl.grid = tiles <= sms ? (int)tiles : no_nstat ? sms : (sms / pl.num_n) * pl.num_n;
  }
  pl.Kpad = pl.num_n * pl.BN;
  pl.im2col = !(d->R == 1 && pl.gS == 1 && d->stride_h == 1 && pl.g_sw == 1 && d->pad_t == 0 && pl.g_pl == 0 &&
                 d->pad_b == 0 && pl.g_pr == 0);
  if (pl.im2col) {
    const int lw = -pl.g_pl, lh = -d->pad_t;
    const int uw = pl.g_pr - (pl.gS - 1) * pl.g_dw, uh = d->pad_b - (d->R - 1) * d->dil_h;
    if (lw < -128 || lh < -128 || uw < -128 || uh < -128 || uw > 127 || uh > 127) return QNN_ERR_UNSUPPORTED;
    if ((d->R - 1) * d->dil_h > 255 || (pl.gS - 1) * pl.g_dw > 255) return QNN_ERR_UNSUPPORTED;
    if (d->stride_h > 8 || pl.g_sw > 8) return QNN_ERR_UNSUPPORTED;
  }
  st = build_classes(pl.P, d->H, d->R, d->stride_h, d->pad_t, d->dil_h, pl.ct.r_lo, pl.ct.r_hi, &pl.ct.ncr, pl.rowcls);
  if (st != QNN_OK) return st;
  st = build_classes(pl.Q, d->W, d->S, d->stride_w, d->pad_l, d->dil_w, pl.ct.s_lo, pl.ct.s_hi, &pl.ct.ncc, pl.colcls);
  if (st != QNN_OK) return st;
  if (pl.ct.ncr * pl.ct.ncc > 255) return QNN_ERR_UNSUPPORTED;
  {
    // Term 3 (zp_W != 0) folded into the contraction when every channel's W - zp_W[k] range fits
    // two s8 parts ([-256, 254]: all u8 weights with zp >= 1, s8 weights with zp >= -127) and
    // the input is not width-folded; else the row-sum pass (scalar zp_W only).  QNN_NO_WSPLIT=1
    // keeps the row sums for a scalar zp_W (A/B measurements).
    // A scalar zp_W on a long reduction (KK >= 2048: the tensor-core-bound 3x3 layers, where
    // doubling the MMAs costs more than the row-sum pass; measured on ResNet-50 b256) keeps
    // the row sums.  (A width-folded input must also be built in smem: checked below.)
    static const bool no_wsplit = std::getenv("QNN_NO_WSPLIT") != nullptr;
    int64_t wlo, whi;
    dtype_range(d->kernel_dtype, &wlo, &whi);
    bool splittable = true;
    for (int32_t z : pl.zpv) splittable &= wlo - z >= -256 && whi - z <= 254;
    const long long KKs = (long long)(d->C / d->groups) * d->R * d->S;
    pl.wsplit = pl.any_zpw && splittable && (pl.zp_vec || (!no_wsplit && KKs < 2048));
    if (pl.zp_vec && pl.any_zpw && !pl.wsplit) return QNN_ERR_UNSUPPORTED;
  }
  const int bparts = pl.wsplit ? 2 : 1;
  {
    const int ncls = pl.ct.ncr * pl.ct.ncc;
    const int num_kb = d->R * pl.gS * pl.nchunks;
    // keep the whole weight operand resident when it is one N tile and leaves room for >= 4 A stages
    pl.b_res_kb = 0;
    // (several N tiles: each CTA keeps one, see the grid above)
    const bool one_n = pl.num_n == 1 || pl.grid % pl.num_n == 0;
    if (one_n && gemm_smem_bytes(pl.BK, pl.BN, 4, ncls, num_kb * bparts, 1, 0, 0, bparts) <= 227 * 1024)
      pl.b_res_kb = num_kb;
    // k-blocks per stage: about 32 KB of operands per barrier round trip, at least 3 stages
    const int per_kb = kGemmBM * pl.BK + (pl.b_res_kb ? 0 : pl.BN * pl.BK * bparts);
    pl.kps = std::max(1, std::min(num_kb, 32768 / per_kb));
    while (pl.kps > 1 && gemm_max_stages(pl.BK, pl.BN, ncls, pl.b_res_kb * bparts, pl.kps, 0, 0, bparts) < 3) --pl.kps;
    pl.stages = gemm_max_stages(pl.BK, pl.BN, ncls, pl.b_res_kb * bparts, pl.kps, 0, 0, bparts);
    if (gemm_smem_bytes(pl.BK, pl.BN, pl.stages, ncls, pl.b_res_kb * bparts, pl.kps, 0, 0, bparts) > 227 * 1024)
      return QNN_ERR_UNSUPPORTED;
  }

  // fold with one 32-byte k-block per filter row, resident weights and contiguous rows: the GEMM
  // kernel builds the X' tiles in shared memory from TMA-staged raw input rows instead of
  // materialising X' in HBM (QNN_NO_ABUILD=1 keeps the HBM copy, for A/B measurements)
  static const bool no_abuild = std::getenv("QNN_NO_ABUILD") != nullptr;
  {
    const long long rowlen = (long long)d->W * d->C;
    pl.a_build = !no_abuild && pl.num_n == 1 && pl.fold && pl.BK == 32 && pl.nchunks == 1 && pl.b_res_kb > 0 &&
                 d->S * d->C <= 32 && pl.in_cs == d->C && d->dil_w == 1 && rowlen % 16 == 0 &&
                 (long long)(d->R - 1) * d->dil_h + 1 <= 256;
    if (pl.a_build) {
      pl.a_ib = 0;
      for (int ib : {256, 128, 64, 32, 16})
        if (rowlen % ib == 0 && rowlen / ib <= 256) {
          pl.a_ib = ib;
          break;
        }
      pl.a_nr = 127 / pl.Q + 2;
      pl.a_slot_bytes = (int)((d->R * rowlen + 127) / 128 * 128);
      pl.a_raw_bytes = (pl.a_nr * pl.a_slot_bytes + 1023) / 1024 * 1024;   // keeps later regions 1 KB aligned
      const int ncls = pl.ct.ncr * pl.ct.ncc;
      const int num_kb = d->R;   // one k-block per filter row
      const int st = gemm_max_stages(pl.BK, pl.BN, ncls, pl.b_res_kb, num_kb, pl.a_raw_bytes);
      if (pl.a_ib == 0 || st < 2 ||
          gemm_smem_bytes(pl.BK, pl.BN, st, ncls, pl.b_res_kb, num_kb, pl.a_raw_bytes) > 227 * 1024) {
        pl.a_build = false;
      } else {
        pl.kps = num_kb;
        pl.stages = st;
      }
    }
    if (pl.a_build && (!pl.any_zpw || pl.wsplit)) {
      // the builders write zp_A (not 0) outside the image, so every tap is valid: one border
      // class, off = bias - zp_A * sum_taps W, and a per-class-free epilogue (zp_W == 0: no row sums)
      pl.a_zpfill = true;
      pl.ct.ncr = pl.ct.ncc = 1;
      pl.ct.r_lo[0] = 0; pl.ct.r_hi[0] = d->R - 1;
      pl.ct.s_lo[0] = 0; pl.ct.s_hi[0] = d->S - 1;
      pl.rowcls.assign(pl.P, 0);
      pl.colcls.assign(pl.Q, 0);
      pl.stages = gemm_max_stages(pl.BK, pl.BN, 1, pl.b_res_kb, pl.kps, pl.a_raw_bytes);
    }
  }
  if (pl.wsplit && pl.fold && !pl.a_build) {   // the HBM width-fold path keeps the row sums
    if (pl.zp_vec) return QNN_ERR_UNSUPPORTED;
    pl.wsplit = false;
  }
  // a_rows: stride-1 im2col convs with resident weights load the input rows a tile touches
  // once per channel chunk and address every tap through the MMA descriptor (no per-tap
  // im2col TMA); QNN_NO_AROWS=1 keeps the im2col path (A/B measurements).  Its epilogue
  // stores directly (no TMA-store staging), and those 32 KB are what let the weights of a
  // 128 x 128 x 3 x 3 layer (147 KB) stay resident beside two staged-row stages: the
  // streamed-weight im2col plan of such a layer is bound by the L2 -> SM feed (every tile
  // re-reads all weights and 9 im2col boxes).
  static const bool no_arows = std::getenv("QNN_NO_AROWS") != nullptr;
  if (!no_arows && pl.im2col && !pl.fold && !pl.pad_copy && !pl.a_build && d->stride_h == 1 && d->stride_w == 1 &&
      d->dil_h == 1 && d->dil_w == 1 && pl.num_n == 1 && d->C % pl.BK == 0) {
    const int Wp = pl.Q + d->S - 1;
    const long long flat = (long long)pl.P * Wp;
    const int T = (int)((flat + kGemmBM - 1) / kGemmBM);
    int nri = 0;
    for (int t = 0; t < T; ++t) {
      const long long f0 = (long long)t * kGemmBM, f1 = std::min(f0 + kGemmBM - 1, flat - 1);
      nri = std::max(nri, (int)(f1 / Wp - f0 / Wp) + d->R);
    }
    const long long a_stage = ((long long)(nri * Wp + d->S) * pl.BK + 1023) / 1024 * 1024;
    const int ncls = pl.ct.ncr * pl.ct.ncc;
    const int num_kb = d->R * d->S * pl.nchunks;
    if (Wp <= 256 && nri <= 256 && a_stage <= 96 * 1024) {
      // (stage count as if the staging region were there when that leaves >= 2 stages: deeper
      // rings measured no faster on ResNet-50 layer1; without it only when it is what fits)
      int st = gemm_max_stages(pl.BK, pl.BN, ncls, num_kb * bparts, d->R * d->S, 0, (int)a_stage, bparts, true);
      if (st < 2 || gemm_smem_bytes(pl.BK, pl.BN, st, ncls, num_kb * bparts, d->R * d->S, 0, (int)a_stage, bparts,
                                    true) > 227 * 1024)
        st = gemm_max_stages(pl.BK, pl.BN, ncls, num_kb * bparts, d->R * d->S, 0, (int)a_stage, bparts, false);
      static const int arows_cap = std::getenv("QNN_AROWS_STAGES") ? std::atoi(std::getenv("QNN_AROWS_STAGES")) : 0;
      if (arows_cap >= 2 && st > arows_cap) st = arows_cap;   // (A/B measurements of the ring depth)
      if (st >= 2 && gemm_smem_bytes(pl.BK, pl.BN, st, ncls, num_kb * bparts, d->R * d->S, 0, (int)a_stage, bparts,
                                     false) <= 227 * 1024) {
        pl.a_rows = true;
        pl.b_res_kb = num_kb;
        pl.a_Wp = Wp;
        pl.a_T = T;
        pl.a_nri = nri;
        pl.a_stage_bytes = (int)a_stage;
        pl.kps = d->R * d->S;
        pl.stages = st;
        pl.num_m = d->N * T;
        pl.grid = std::min(pl.num_m, sm_count());   // num_n == 1
      }
    }
  }
  {
    // wide pointwise layers: the channel-major GEMM keeps each output channel's requantize
    // constants in registers.  QNN_NO_TRANS=1 keeps the pixel-major kernel (A/B measurements).
    // K_out = 64 runs as half a 128-channel block: since the 16x256b epilogue, faster than the
    // pixel-major kernel (ResNet-50 b256 layer1 conv1 44 -> 34 us); QNN_TRANS_MINK=128 keeps
    // those layers pixel-major
    static const bool no_trans = std::getenv("QNN_NO_TRANS") != nullptr;
    static const int kTransMinK = std::getenv("QNN_TRANS_MINK") ? std::atoi(std::getenv("QNN_TRANS_MINK")) : 64;
    // (small M: when the channel-major grid of 256-pixel x 128-channel tiles would leave most
    // SMs idle and the pixel-major plan has more tiles, keep the pixel-major plan -- the
    // per-GPU batch 32 of 8-GPU strong scaling; QNN_TRANS_SMALLM=1 disables the check)
    static const bool small_ok = std::getenv("QNN_TRANS_SMALLM") != nullptr;
    const long long t_tiles = ((pl.M + kGemmTBN - 1) / kGemmTBN) * ((d->K + 127) / 128);
    const bool few = !small_ok && t_tiles < sm_count() / 2 && (long long)pl.num_m * pl.num_n > t_tiles;
    if (!no_trans && !few && !pl.im2col && !pl.fold && !pl.pad_copy && !pl.a_build && !pl.a_rows && d->groups == 1 &&
        (!pl.any_zpw || pl.wsplit) && (d->kernel_dtype == QNN_S8 || pl.wsplit) && pl.requant &&
        (pl.out_dt == QNN_U8 || pl.out_dt == QNN_S8) && (d->K % 128 == 0 || d->K == 64) && d->K >= kTransMinK &&
        pl.out_cs % 16 == 0 && pl.ct.ncr * pl.ct.ncc == 1) {
      const int num_kb = pl.nchunks;   // one tap
      // CTA pairs (cta_group::2, each CTA staging half of every pixel tile: operand bytes per SM
      // per MAC drop by 1.5x) where a single CTA would stream its weights and K_out >= 512 --
      // the layers bound by what an SM can take in (ResNet-50 layer4 conv1: -5..11%).  On
      // resident-weight and K_out = 256 layers the pair measured slower (the two CTAs' epilogues
      // and pipelines run in lockstep: conv3 +20-30%).  QNN_PAIR=0 / 1 forces it off / on where
      // the channel blocks pair up.
      static const int pair_env = std::getenv("QNN_PAIR") ? std::atoi(std::getenv("QNN_PAIR")) : -1;
      const bool can_pair = (round_up(d->K, 128) / 128) % 2 == 0;
      bool pair = false;
      if (can_pair && pair_env != 0) {
        if (pair_env == 1) {
          pair = true;
        } else if (d->K >= 512) {   // would a single CTA stream its weights?
          const int st_res = gemm_t_max_stages(pl.BK, num_kb, true, 1, -1, 0, 128, bparts);
          pair = !(st_res >= 3 && gemm_t_smem_bytes(pl.BK, num_kb, st_res, true, 1, -1, 0, 128, bparts) <= 226 * 1024);
        }
      }
      // preference: resident weights with a second output staging buffer per column group
      // (>= 4 stages), then resident weights with one, then streamed weights
      const int opts[3][2] = {{2, 1}, {1, 1}, {1, 0}};   // {buffers, weights resident}
      for (const auto& o : opts) {
        const int bufs = o[0];
        const bool w_res = o[1] != 0;
        const int stages = gemm_t_max_stages(pl.BK, num_kb, w_res, bufs, -1, 0, 128, bparts, pair);
        if (stages >= (bufs == 2 ? 4 : 3) &&
            gemm_t_smem_bytes(pl.BK, num_kb, stages, w_res, bufs, -1, 0, 128, bparts, pair) <= 226 * 1024) {
          pl.trans = true;
          pl.t_wres = w_res;
          pl.t_stages = stages;
          pl.t_bufs = bufs;
          pl.t_Kt = round_up(d->K, 128);
          pl.t_pair = pair;
          break;
        }
      }
    }
  }
  {
    // small-C stems with K_out <= 64 (ResNet-50 7x7x3, Inception-v3 / MobileNet-v2 3x3x3): the
    // channel-major GEMM in build mode -- its quads 2-3 (no output channels) build the X' tiles
    // and the epilogue keeps per-channel constants in registers.  Only where the pixel-major
    // builder (a_build, same zp_A fill, same single border class) is the fallback for a
    // misaligned output.  QNN_NO_TBUILD=1 keeps the pixel-major kernel (A/B measurements).
    static const bool no_tbuild = std::getenv("QNN_NO_TBUILD") != nullptr;
    const long long rowlen = (long long)d->W * d->C;
    if (!no_tbuild && pl.a_build && pl.a_zpfill && d->K <= 64 && d->K % 32 == 0 && d->dil_h == 1 &&
        (d->kernel_dtype == QNN_S8 || pl.wsplit) && (pl.out_dt == QNN_U8 || pl.out_dt == QNN_S8) &&
        pl.out_cs % 16 == 0 && d->R <= 16) {
      int ib = 0;
      for (int c : {256, 128, 64, 32, 16})
        if (rowlen % c == 0 && rowlen / c <= 256) {
          ib = c;
          break;
        }
      const int nr = (kGemmTBN - 1) / pl.Q + 2;
      const int slot = (int)((d->R * rowlen + 127) / 128 * 128);
      const int raw = (nr * slot + 1023) / 1024 * 1024;
      // two X' stages; the raw-row ring as deep as the rest of shared memory allows (<= 6)
      int rst = 0;
      for (int r = 6; r >= 2 && !rst; --r)
        if (gemm_t_smem_bytes(32, d->R, 2, true, 1, raw, r, d->K, pl.wsplit ? 2 : 1) <= 226 * 1024) rst = r;
      if (ib && rst) {
        pl.trans = pl.t_build = pl.t_wres = true;
        pl.t_stages = 2;
        pl.t_rstages = rst;
        pl.t_bufs = 1;
        pl.t_Kt = 128;
        pl.t_ib = ib;
        pl.t_nr = nr;
        pl.t_slot = slot;
        pl.t_raw = raw;
      }
    }
  }
  {
    // pixel-major CTA pairs (cta_group::2: each CTA of a cluster of 2 stages its own A tile and
    // half of the B tile, 1.5x fewer operand bytes per SM per MAC): only with QNN_PAIR=1.
    // Measured on the ResNet-50 b256 streamed-weight layers: layer3 3x3 -4..+3%, layer4 3x3 and
    // layer3.0.downsample +35% (the pair's two tiles, epilogues and pipelines run in lockstep,
    // and BN = 192 halves into 96-row B boxes), so the single-CTA plan stays the default.
    static const int pair_env = std::getenv("QNN_PAIR") ? std::atoi(std::getenv("QNN_PAIR")) : -1;
    const bool can = pair_env == 1 && !pl.trans && !pl.depthwise && !pl.a_rows && !pl.a_build && !pl.wsplit &&
                     pl.num_m >= 2 && pl.BN >= 64 && pl.BN % 16 == 0;
    if (can) {
      const int ncls = pl.ct.ncr * pl.ct.ncc;
      const int st = gemm_max_stages(pl.BK, pl.BN, ncls, pl.b_res_kb, pl.kps, pl.a_raw_bytes, pl.a_stage_bytes, 1, true,
                                     true);
      if (st >= 3 && gemm_smem_bytes(pl.BK, pl.BN, st, ncls, pl.b_res_kb, pl.kps, pl.a_raw_bytes, pl.a_stage_bytes, 1,
                                     true, true) <= 227 * 1024) {
        pl.pair = true;
        pl.stages = st;
        // grid in pairs: pair tiles = ceil(num_m / 2) x num_n, a pair keeps one N tile
        const long long ptiles = (long long)((pl.num_m + 1) / 2) * pl.num_n;
        const int maxp = sm_count() / 2;
        pl.grid = 2 * (int)(ptiles <= maxp ? ptiles : (long long)(maxp / pl.num_n) * pl.num_n);
        if (pl.grid <= 0) pl.pair = false;
      }
    }
  }
  const int taps = d->R * pl.gS;  // GEMM taps (R when folded)
  size_t off = 0;
  pl.pk_w = off;
  off = align256(off + (size_t)pl.Kpad * taps * pl.Cw * bparts);
  if (pl.trans) {
    pl.pk_wt = off;
    off = align256(off + (size_t)pl.t_Kt * taps * pl.Cw * bparts);
  }
  if (pl.any_zpw) {   // the per-channel zero points, for the packing and folding kernels
    pl.pk_zpv = off;
    off = align256(off + (size_t)d->K * 4);
  }
  pl.pk_off = off;
  off = align256(off + (size_t)pl.ct.ncr * pl.ct.ncc * pl.Kpad * 4);
  pl.pk_off64 = off;
  off = align256(off + (size_t)pl.ct.ncr * pl.ct.ncc * pl.Kpad * 8);
  pl.pk_mult = off;
  off = align256(off + (size_t)pl.Kpad * 4);
  pl.pk_rsh = off;
  off = align256(off + (size_t)pl.Kpad * 4);
  pl.pk_rowcls = off;
  off = align256(off + (size_t)pl.P);
  pl.pk_colcls = off;
  off = align256(off + (size_t)pl.Q);
  pl.pk_total = off;

  size_t w = 0;
  if (pl.pad_copy || (pl.fold && !pl.a_build)) {
    pl.ws_pad = w;
    w = align256(w + (size_t)d->N * d->H * pl.gW * pl.Ct);
  }
  if (pl.any_zpw && !pl.wsplit) {
    pl.ws_pixsum = w;
    w = align256(w + (size_t)d->N * d->H * d->W * 4);
    pl.ws_rowsum = w;
    w = align256(w + (size_t)pl.M * 4);
  }
  pl.ws_total = w;
  static const bool plan_trace = std::getenv("QNN_PLAN_TRACE") != nullptr;
  if (plan_trace)
    std::fprintf(stderr,
                 "[qnn plan] N%d C%d %dx%d K%d %dx%d s%d: BK%d BN%d num_m%d num_n%d chunks%d stages%d kps%d b_res%d "
                 "im2col%d fold%d pad_copy%d a_build%d a_rows%d (Wp%d T%d nri%d stage%dB) trans%d t_build%d "
                 "wsplit%d ppair%d (t: stages%d wres%d bufs%d Kt%d pair%d)\n",
                 d->N, d->C, d->H, d->W, d->K, d->R, d->S, d->stride_h, pl.BK, pl.BN, pl.num_m, pl.num_n,
                 pl.nchunks, pl.stages, pl.kps, pl.b_res_kb, (int)pl.im2col, (int)pl.fold, (int)pl.pad_copy,
                 (int)pl.a_build, (int)pl.a_rows, pl.a_Wp, pl.a_T, pl.a_nri, pl.a_stage_bytes, (int)pl.trans,
                 (int)pl.t_build, (int)pl.wsplit, (int)pl.pair, pl.t_stages, (int)pl.t_wres, pl.t_bufs, pl.t_Kt, (int)pl.t_pair);
  return QNN_OK;
}

static qnn_status_t cuda_status(cudaError_t e) { return e == cudaSuccess ? QNN_OK : QNN_ERR_CUDA; }

static qnn_status_t conv_prepack(const qnn_conv2d_desc_t* d, const void* kernel, const int32_t* bias,
                                 const qnn_output_params_t* o, void* packed, size_t packed_bytes, cudaStream_t s) {
  ConvPlan pl;
  qnn_status_t st = make_plan(d, o, pl);
  if (st != QNN_OK) return st;
  if (!kernel || !packed) return QNN_ERR_INVALID_VALUE;
  if (packed_bytes < pl.pk_total) return QNN_ERR_WORKSPACE;
  if (reinterpret_cast<uintptr_t>(packed) & 255) return QNN_ERR_MISALIGNED;
  uint8_t* pk = reinterpret_cast<uint8_t*>(packed);
  const int w_signed = d->kernel_dtype == QNN_S8;

  // per-channel multipliers m_k = s_A * s_W[k] / s_out (reading R3)
  const int nmult = pl.depthwise ? (pl.dwtc ? pl.Kpad : d->C) : pl.Kpad;
  // padding columns (k >= K) get M = 0 with a fast-path shift so they never force the generic epilogue
  std::vector<int32_t> mult(nmult, 0), rsh(nmult, 33);
  if (pl.requant) {
    for (int k = 0; k < d->K; ++k) {
      const double m = ((double)d->input_scale * (double)d->kernel_scales[d->num_kernel_scales == 1 ? 0 : k]) /
                       (double)o->output_scale;
      if (!kernel_multiplier(m, &mult[k], &rsh[k])) return QNN_ERR_UNSUPPORTED;
    }
  }
  cudaError_t e;
  // per-channel weight zero points on the device (packing / folding kernels read them)
  const int32_t* zpv_d = nullptr;
  if ((pl.depthwise && pl.zp_vec) || (!pl.depthwise && pl.any_zpw)) {
    e = cudaMemcpyAsync(pk + pl.pk_zpv, pl.zpv.data(), pl.zpv.size() * 4, cudaMemcpyHostToDevice, s);
    if (e != cudaSuccess) return QNN_ERR_CUDA;
    zpv_d = reinterpret_cast<const int32_t*>(pk + pl.pk_zpv);
  }
  if (pl.depthwise) {
    e = launch_pack_dw_weights(kernel, w_signed, d->kernel_zero_point, reinterpret_cast<int16_t*>(pk + pl.pk_w), d->C,
                               d->R * d->S, s, zpv_d);
    if (e != cudaSuccess) return QNN_ERR_CUDA;
    if (bias)
      e = cudaMemcpyAsync(pk + pl.pk_bias, bias, (size_t)d->C * 4, cudaMemcpyDeviceToDevice, s);
    else
      e = cudaMemsetAsync(pk + pl.pk_bias, 0, (size_t)d->C * 4, s);
    if (e != cudaSuccess) return QNN_ERR_CUDA;
    if (pl.dwtc) {
      e = launch_pack_dwtc(kernel, d->C, d->R * d->S, pk + pl.pk_dwtc_w, s);
      if (e != cudaSuccess) return QNN_ERR_CUDA;
      // per border class: bias - zp_A * sum of the valid taps (depthwise weights = C x R x S x 1)
      e = launch_fold_offsets(kernel, w_signed, bias, d->C, d->R, d->S, 1, d->input_zero_point, 0, pl.ct,
                              reinterpret_cast<int32_t*>(pk + pl.pk_off), reinterpret_cast<int64_t*>(pk + pl.pk_off64),
                              pl.Kpad, s);
      if (e != cudaSuccess) return QNN_ERR_CUDA;
      e = cudaMemcpyAsync(pk + pl.pk_rowcls, pl.rowcls.data(), pl.rowcls.size(), cudaMemcpyHostToDevice, s);
      if (e == cudaSuccess)
        e = cudaMemcpyAsync(pk + pl.pk_colcls, pl.colcls.data(), pl.colcls.size(), cudaMemcpyHostToDevice, s);
      if (e != cudaSuccess) return QNN_ERR_CUDA;
    }
  } else {
    // folded: each filter row r is one GEMM tap whose S*C channels are contiguous in OHWI;
    // wsplit: W - zp_W[k] in two s8 k-block sets (Term 3 in the contraction)
    const int sp = pl.wsplit ? 1 : 0;
    if (pl.fold)
      e = launch_pack_weights(kernel, pk + pl.pk_w, d->K, d->R, d->S * d->C, pl.Cw, pl.Kpad, s, 0, sp, w_signed, zpv_d);
    else
      e = launch_pack_weights(kernel, pk + pl.pk_w, d->K, d->R * d->S, d->C, pl.Cw, pl.Kpad, s, 0, sp, w_signed, zpv_d);
    if (e == cudaSuccess && pl.trans)
      e = pl.fold ? launch_pack_weights(kernel, pk + pl.pk_wt, d->K, d->R, d->S * d->C, pl.Cw, pl.t_Kt, s, /*perm32=*/1,
                                        sp, w_signed, zpv_d)
                  : launch_pack_weights(kernel, pk + pl.pk_wt, d->K, 1, d->C, pl.Cw, pl.t_Kt, s, /*perm32=*/1, sp,
                                        w_signed, zpv_d);
    if (e != cudaSuccess) return QNN_ERR_CUDA;
    e = launch_fold_offsets(kernel, w_signed, bias, d->K, d->R, d->S, d->C, d->input_zero_point, d->kernel_zero_point,
                            pl.ct, reinterpret_cast<int32_t*>(pk + pl.pk_off),
                            reinterpret_cast<int64_t*>(pk + pl.pk_off64), pl.Kpad, s, zpv_d);
    if (e != cudaSuccess) return QNN_ERR_CUDA;
    e = cudaMemcpyAsync(pk + pl.pk_rowcls, pl.rowcls.data(), pl.rowcls.size(), cudaMemcpyHostToDevice, s);
    if (e == cudaSuccess)
      e = cudaMemcpyAsync(pk + pl.pk_colcls, pl.colcls.data(), pl.colcls.size(), cudaMemcpyHostToDevice, s);
    if (e != cudaSuccess) return QNN_ERR_CUDA;
  }
  e = cudaMemcpyAsync(pk + pl.pk_mult, mult.data(), mult.size() * 4, cudaMemcpyHostToDevice, s);
  if (e == cudaSuccess) e = cudaMemcpyAsync(pk + pl.pk_rsh, rsh.data(), rsh.size() * 4, cudaMemcpyHostToDevice, s);
  if (e == cudaSuccess) e = cudaStreamSynchronize(s);  // host vectors die on return
  return cuda_status(e);
}

struct ResidualArgs {   // fused residual add (qnn_conv2d_packed_add)
  const void* ptr;
  qnn_dtype_t dtype;
  float scale;
  int32_t zp;
  int32_t cstride;
};

static qnn_status_t conv_packed(const qnn_conv2d_desc_t* d, const qnn_output_params_t* o, const void* packed,
                                const void* input, void* output, void* ws, size_t ws_bytes, cudaStream_t s,
                                const ResidualArgs* res = nullptr) {
  ConvPlan pl;
  qnn_status_t st = make_plan(d, o, pl, /*need_scales=*/false);
  if (st != QNN_OK) return st;
  if (!packed || !input || !output) return QNN_ERR_INVALID_VALUE;
  int32_t res_M = 0, res_rsh = 1;
  long long res_cs = 0;
  if (res) {
    if (!res->ptr || !o || !is_8bit(res->dtype) || !scale_ok(res->scale) || !zp_ok(res->dtype, res->zp))
      return QNN_ERR_INVALID_VALUE;
    res_cs = res->cstride ? res->cstride : d->K;
    if (res_cs < d->K) return QNN_ERR_INVALID_VALUE;
    if (pl.depthwise || d->K % 32 != 0) return QNN_ERR_UNSUPPORTED;
    if ((reinterpret_cast<uintptr_t>(res->ptr) & 15) || (res_cs % 16)) return QNN_ERR_MISALIGNED;
    if (!kernel_multiplier((double)res->scale / (double)o->output_scale, &res_M, &res_rsh))
      return QNN_ERR_UNSUPPORTED;
  }
  if (reinterpret_cast<uintptr_t>(packed) & 255) return QNN_ERR_MISALIGNED;
  if (pl.ws_total && (!ws || ws_bytes < pl.ws_total)) return QNN_ERR_WORKSPACE;
  if (ws && (reinterpret_cast<uintptr_t>(ws) & 255)) return QNN_ERR_MISALIGNED;
  const uint8_t* pk = reinterpret_cast<const uint8_t*>(packed);
  uint8_t* wsb = reinterpret_cast<uint8_t*>(ws);
  const int a_signed = d->input_dtype == QNN_S8;

  if (pl.depthwise) {
    // kernel choice: 3x3 TMA-staged (CUDA cores) > 3x3 register-blocked dp4a > tensor-core
    // path > generic CUDA-core kernel.  QNN_DW_IMPL=dp4a|tc|generic forces one of the others
    // (A/B measurements).
    static const char* dw_impl = std::getenv("QNN_DW_IMPL");
    const bool force_tc = dw_impl && std::strcmp(dw_impl, "tc") == 0;
    const bool force_generic = dw_impl && std::strcmp(dw_impl, "generic") == 0;
    const bool force_dp4a = dw_impl && std::strcmp(dw_impl, "dp4a") == 0;
    const bool no_dwtc = force_generic;
    DwParams p{};
    p.in = input;
    p.w = reinterpret_cast<const int16_t*>(pk + pl.pk_w);
    p.bias = reinterpret_cast<const int32_t*>(pk + pl.pk_bias);
    p.mult = reinterpret_cast<const int32_t*>(pk + pl.pk_mult);
    p.rsh = reinterpret_cast<const int32_t*>(pk + pl.pk_rsh);
    p.out = output;
    p.in_cstride = pl.in_cs;
    p.out_cstride = pl.out_cs;
    p.N = d->N; p.H = d->H; p.W = d->W; p.C = d->C; p.P = pl.P; p.Q = pl.Q; p.R = d->R; p.S = d->S;
    p.sh = d->stride_h; p.sw = d->stride_w; p.pt = d->pad_t; p.pl = d->pad_l; p.dh = d->dil_h; p.dw = d->dil_w;
    p.a_signed = a_signed;
    p.zpA = d->input_zero_point;
    p.out_dtype = pl.requant ? (int)pl.out_dt : DT_S32;
    p.requant = pl.requant;
    p.mode = pl.mode;
    p.zp_out = pl.zp_out; p.lo = pl.lo; p.hi = pl.hi;
    {
      int64_t wlo, whi;
      dtype_range(d->kernel_dtype, &wlo, &whi);
      p.w_fits_s8 = true;
      for (int32_t z : pl.zpv) p.w_fits_s8 = p.w_fits_s8 && wlo - z >= -128 && whi - z <= 127;
    }
    if (!force_tc && !force_generic && pl.requant) {
      int64_t qlo, qhi;
      dtype_range(pl.out_dt == DT_S8 ? QNN_S8 : (pl.out_dt == DT_U8 ? QNN_U8 : QNN_S32), &qlo, &qhi);
      const int clamp = pl.lo > qlo ? 2 : (pl.hi < qhi ? 1 : 0);   // the saturating pack covers the dtype range
      DwParams pt = p;
      if (!force_dp4a && dwtma_plan(pt) && load_driver_entry_points()) {
        // input (c, w, h, n); box = CS channels x Wb columns x band rows, zero outside the image
        alignas(64) CUtensorMap tm;
        const cuuint64_t dims[4] = {(cuuint64_t)d->C, (cuuint64_t)d->W, (cuuint64_t)d->H, (cuuint64_t)d->N};
        const cuuint64_t strides[3] = {(cuuint64_t)pl.in_cs, (cuuint64_t)pl.in_cs * d->W,
                                       (cuuint64_t)pl.in_cs * d->W * d->H};
        const cuuint32_t box[4] = {(cuuint32_t)pt.dwt_cs, (cuuint32_t)pt.dwt_wb,
                                   (cuuint32_t)((pt.dwt_bp - 1) * pt.sh + 3), 1};
        const cuuint32_t estr[4] = {1, 1, 1, 1};
        if (p_encode_tiled(&tm, CU_TENSOR_MAP_DATA_TYPE_UINT8, 4, const_cast<void*>(input), dims, strides, box, estr,
                           CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                           CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS) {
          small_tensor_fixup(&tm, (uint64_t)pl.in_cs * d->W * d->H * d->N);
          return cuda_status(launch_depthwise_tma(tm, pt, clamp, s));
        }
      }
      if (launch_depthwise3(p, clamp, s)) return cuda_status(cudaGetLastError());
    }
    if (pl.dwtc && !no_dwtc && pl.requant && (pl.out_dt == DT_U8 || pl.out_dt == DT_S8) &&
        ((reinterpret_cast<uintptr_t>(input) | reinterpret_cast<uintptr_t>(output)) & 15) == 0) {
      DwTcParams t{};
      t.wpk = pk + pl.pk_dwtc_w;
      t.mult = reinterpret_cast<const int32_t*>(pk + pl.pk_mult);
      t.rsh = reinterpret_cast<const int32_t*>(pk + pl.pk_rsh);
      t.off = reinterpret_cast<const int32_t*>(pk + pl.pk_off);
      t.off64 = reinterpret_cast<const int64_t*>(pk + pl.pk_off64);
      t.rowcls = pk + pl.pk_rowcls;
      t.colcls = pk + pl.pk_colcls;
      t.out = reinterpret_cast<uint8_t*>(output);
      t.out_cs = pl.out_cs;
      t.N = d->N; t.C = d->C; t.Cpad = pl.Kpad; t.P = pl.P; t.Q = pl.Q; t.R = d->R; t.S = d->S;
      t.sh = d->stride_h; t.sw = d->stride_w; t.pt = d->pad_t; t.pl = d->pad_l;
      t.ncls = pl.ct.ncr * pl.ct.ncc; t.ncc = pl.ct.ncc;
      t.idesc = make_idesc_i8(a_signed, 1, 128, 32);
      t.zp_out = pl.zp_out; t.lo = pl.lo; t.hi = pl.hi;
      static const char* tr_env = std::getenv("QNN_DWTC_TRACE");
      t.trace = tr_env ? reinterpret_cast<unsigned long long*>(std::strtoull(tr_env, nullptr, 0)) : nullptr;
      if (dwtc_plan(t) && load_driver_entry_points()) {
        // input as a 4-D tensor (c, w, h, n); box = one 32-channel slice x Wp x in_rows pixels with
        // element strides (sw, sh) for the phase planes; 32-B swizzle = the UMMA SW32 K-major layout
        alignas(64) CUtensorMap tm;
        const cuuint64_t dims[4] = {(cuuint64_t)d->C, (cuuint64_t)d->W, (cuuint64_t)d->H, (cuuint64_t)d->N};
        const cuuint64_t strides[3] = {(cuuint64_t)pl.in_cs, (cuuint64_t)pl.in_cs * d->W,
                                       (cuuint64_t)pl.in_cs * d->W * d->H};
        const cuuint32_t box[4] = {32, (cuuint32_t)(t.Wp * t.sw), (cuuint32_t)(t.in_rows * t.sh), 1};
        const cuuint32_t estr[4] = {1, (cuuint32_t)t.sw, (cuuint32_t)t.sh, 1};
        CUresult r = p_encode_tiled(&tm, CU_TENSOR_MAP_DATA_TYPE_UINT8, 4, const_cast<void*>(input), dims, strides, box,
                                    estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_32B,
                                    CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
        small_tensor_fixup(&tm, (uint64_t)pl.in_cs * d->W * d->H * d->N);
        if (r == CUDA_SUCCESS) {
          int64_t qlo, qhi;
          dtype_range(pl.out_dt == DT_S8 ? QNN_S8 : QNN_U8, &qlo, &qhi);
          const bool clamp = pl.lo > qlo || pl.hi < qhi;
          return cuda_status(launch_depthwise_tc(tm, t, pl.mode, clamp, pl.out_dt == DT_S8, s));
        }
      }
    }
    return cuda_status(launch_depthwise(p, s));
  }

  if (reinterpret_cast<uintptr_t>(input) & 15) return QNN_ERR_MISALIGNED;
  if (!load_driver_entry_points()) return QNN_ERR_CUDA;
  cudaError_t e;
  const void* A = input;
  long long a_pitch = pl.in_cs;
  if (pl.fold && !pl.a_build) {
    e = launch_fold_width(input, pl.in_cs, wsb + pl.ws_pad, d->N, d->H, d->W, d->C, pl.Q, d->S, d->stride_w, d->pad_l,
                          d->dil_w, pl.Ct, s);
    if (e != cudaSuccess) return QNN_ERR_CUDA;
    A = wsb + pl.ws_pad;
    a_pitch = pl.Ct;
  } else if (pl.pad_copy) {
    e = launch_pad_channels(input, pl.in_cs, wsb + pl.ws_pad, pl.Ct, (long long)d->N * d->H * d->W, d->C, s);
    if (e != cudaSuccess) return QNN_ERR_CUDA;
    A = wsb + pl.ws_pad;
    a_pitch = pl.Ct;
  }
  const int32_t* rowsum = nullptr;
  if (pl.any_zpw && !pl.wsplit) {
    int32_t* pixsum = reinterpret_cast<int32_t*>(wsb + pl.ws_pixsum);
    e = launch_pixel_sums(input, a_signed, pl.in_cs, d->C, (long long)d->N * d->H * d->W, pixsum, s);
    if (e != cudaSuccess) return QNN_ERR_CUDA;
    if (!pl.im2col) {
      rowsum = pixsum;  // 1x1 / stride 1 / no padding: one pixel per row
    } else {
      int32_t* rs = reinterpret_cast<int32_t*>(wsb + pl.ws_rowsum);
      e = launch_window_sums(pixsum, d->N, d->H, d->W, pl.P, pl.Q, d->R, d->S, d->stride_h, d->stride_w, d->pad_t,
                             d->pad_l, d->dil_h, d->dil_w, rs, s);
      if (e != cudaSuccess) return QNN_ERR_CUDA;
      rowsum = rs;
    }
  }

  // wide pointwise layers (plan: pl.trans): the channel-major GEMM (gemm_t.cu) on the perm32 weights
  if (pl.trans && (reinterpret_cast<uintptr_t>(output) & 15) == 0) {
    const int num_kb = pl.nchunks;   // one tap
    const bool w_res = pl.t_wres;
    const int stages = pl.t_stages;
    {
      alignas(64) CUtensorMap tmX, tmW, tmC, tmR;
      std::memset(&tmR, 0, sizeof(tmR));
      const int a_chan = d->C;
      bool okx;
      const int taps = d->R * pl.gS;
      // staging / store rows: one 128-channel block, or K_out (64 / 32) bytes in build mode
      const uint32_t out_rb = pl.t_build ? (uint32_t)d->K : 128u;
      if (pl.t_build) {
        // raw input rows as (ib bytes, W*C/ib, H, N): one box = the R filter rows of one output row
        const uint64_t rowlen = (uint64_t)d->W * d->C;
        const cuuint64_t dims[4] = {(cuuint64_t)pl.t_ib, rowlen / pl.t_ib, (cuuint64_t)d->H, (cuuint64_t)d->N};
        const cuuint64_t strides[3] = {(cuuint64_t)pl.t_ib, rowlen, rowlen * d->H};
        const cuuint32_t box[4] = {(cuuint32_t)pl.t_ib, (cuuint32_t)(rowlen / pl.t_ib), (cuuint32_t)d->R, 1};
        const cuuint32_t estr[4] = {1, 1, 1, 1};
        okx = p_encode_tiled(&tmX, CU_TENSOR_MAP_DATA_TYPE_UINT8, 4, const_cast<void*>(input), dims, strides, box, estr,
                             CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                             CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
        small_tensor_fixup(&tmX, rowlen * d->H * d->N);
      } else {
        okx = encode_2d(&tmX, A, (uint64_t)a_chan, (uint64_t)pl.M, (uint64_t)a_pitch, pl.BK,
                        pl.t_pair ? kGemmTBN / 2 : kGemmTBN);   // (pair: each CTA loads half a tile)
      }
      bool okt = okx &&
                 encode_2d(&tmW, pk + pl.pk_wt, (uint64_t)taps * pl.Cw * (pl.wsplit ? 2 : 1), (uint64_t)pl.t_Kt,
                           (uint64_t)taps * pl.Cw * (pl.wsplit ? 2 : 1), pl.BK,
                           128) &&
                 encode_2d(&tmC, output, (uint64_t)d->K, (uint64_t)pl.M, (uint64_t)pl.out_cs, out_rb, kGemmTBN / 4) &&
                 (!res || encode_2d(&tmR, res->ptr, (uint64_t)d->K, (uint64_t)pl.M, (uint64_t)res_cs, out_rb,
                                    kGemmTBN / 4));
      if (okt) {
        GemmTParams tp{};
        tp.BK = pl.BK;
        tp.stages = stages;
        tp.num_kb = num_kb;
        tp.w_res = w_res;
        tp.stage_bufs = pl.t_bufs;
        tp.out_rb = (int)out_rb;
        tp.num_ch_tiles = (d->K + 127) / 128;
        tp.Kout = d->K;
        if (res) {
          tp.has_res = 1;
          tp.res_M = res_M;
          tp.res_rsh = res_rsh;
          tp.res_zp = res->zp;
          tp.res_s8 = res->dtype == QNN_S8;
        }
        tp.num_px_tiles = (int)((pl.M + kGemmTBN - 1) / kGemmTBN);
        if (pl.t_build) {
          tp.build = 1;
          tp.num_kb = d->R;   // one 32-byte k-block (S*C bytes) per filter row
          tp.b_W = d->W; tp.b_C = d->C; tp.b_S = d->S; tp.b_sw = d->stride_w; tp.b_pl = d->pad_l;
          tp.b_rowlen = d->W * d->C;
          tp.b_nr = pl.t_nr;
          tp.b_H = d->H;
          tp.b_slot_bytes = pl.t_slot;
          tp.b_raw_bytes = pl.t_raw;
          tp.rstages = pl.t_rstages;
          tp.b_zp4 = 0x01010101u * (uint32_t)(d->input_zero_point & 0xFF);
          tp.P = pl.P; tp.Q = pl.Q; tp.sh = d->stride_h; tp.pt = d->pad_t;
          tp.fdQ = make_fastdiv((uint32_t)pl.Q);
          tp.fdP = make_fastdiv((uint32_t)pl.P);
        }
        // A = s8 weights (or split parts), B = activations; a pair's MMA has M = 256
        tp.idesc = make_idesc_i8(1, a_signed, pl.t_pair && !pl.t_build ? 256 : 128, kGemmTBN);
        tp.pair = pl.t_pair && !pl.t_build ? 1 : 0;
        tp.wsplit = pl.wsplit;
        static const bool one_set = std::getenv("QNN_TEPI_ONESET") != nullptr;   // (A/B measurements)
        tp.esets = (pl.t_build || one_set) ? 1 : 2;
        tp.mult = reinterpret_cast<const int32_t*>(pk + pl.pk_mult);
        tp.rsh = reinterpret_cast<const int32_t*>(pk + pl.pk_rsh);
        tp.off64 = reinterpret_cast<const int64_t*>(pk + pl.pk_off64);
        tp.zp_out = pl.zp_out;
        tp.lo = pl.lo;
        tp.hi = pl.hi;
#ifdef QNN_GEMM_INSTRUMENT
        {
          static const char* dbg_env = std::getenv("QNN_GEMM_DEBUG");
          tp.dbg = dbg_env ? std::atoi(dbg_env) : 0;
          static const char* tr_env = std::getenv("QNN_GEMM_TRACE");
          tp.trace = tr_env ? reinterpret_cast<unsigned long long*>(std::strtoull(tr_env, nullptr, 0)) : nullptr;
        }
#endif
        const int sms = sm_count();
        const int tiles = tp.num_ch_tiles * tp.num_px_tiles;
        const int grid = tiles <= sms ? tiles : std::max(1, sms / tp.num_ch_tiles) * tp.num_ch_tiles;
        int64_t qlo, qhi;
        dtype_range(pl.out_dt == DT_S8 ? QNN_S8 : QNN_U8, &qlo, &qhi);
        const bool clamp = pl.lo > qlo || pl.hi < qhi;
        return cuda_status(launch_gemm_t(tmX, tmW, tmC, tmR, tp, pl.mode, clamp, pl.out_dt == DT_S8, grid, s));
      }
    }
  }

  alignas(64) CUtensorMap tmA, tmB;
  bool ok;
  const int a_chan = (pl.pad_copy || pl.fold) ? pl.Ct : d->C;
  const int taps = d->R * pl.gS;
  if (pl.a_rows) {
    // input (c, w, h, n), box = one channel chunk x Wp columns x a_nri rows, swizzled like the
    // UMMA K-major layout of BK-byte rows; out-of-image pixels zero-filled (border classes)
    const cuuint64_t dims[4] = {(cuuint64_t)d->C, (cuuint64_t)d->W, (cuuint64_t)d->H, (cuuint64_t)d->N};
    const cuuint64_t strides[3] = {(cuuint64_t)pl.in_cs, (cuuint64_t)pl.in_cs * d->W,
                                   (cuuint64_t)pl.in_cs * d->W * d->H};
    const cuuint32_t box[4] = {(cuuint32_t)pl.BK, (cuuint32_t)pl.a_Wp, (cuuint32_t)pl.a_nri, 1};
    const cuuint32_t estr[4] = {1, 1, 1, 1};
    ok = p_encode_tiled(&tmA, CU_TENSOR_MAP_DATA_TYPE_UINT8, 4, const_cast<void*>(input), dims, strides, box, estr,
                        CU_TENSOR_MAP_INTERLEAVE_NONE, swizzle_for(pl.BK), CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                        CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
    small_tensor_fixup(&tmA, (uint64_t)pl.in_cs * d->W * d->H * d->N);
  } else if (pl.a_build) {
    // raw input rows as (ib bytes, W*C/ib, H, N): one box = R filter rows of one output row
    const uint64_t rowlen = (uint64_t)d->W * d->C;
    const cuuint64_t dims[4] = {(cuuint64_t)pl.a_ib, rowlen / pl.a_ib, (cuuint64_t)d->H, (cuuint64_t)d->N};
    const cuuint64_t strides[3] = {(cuuint64_t)pl.a_ib, rowlen, rowlen * d->H};
    const cuuint32_t box[4] = {(cuuint32_t)pl.a_ib, (cuuint32_t)(rowlen / pl.a_ib),
                               (cuuint32_t)((d->R - 1) * d->dil_h + 1), 1};
    const cuuint32_t estr[4] = {1, 1, (cuuint32_t)d->dil_h, 1};
    ok = p_encode_tiled(&tmA, CU_TENSOR_MAP_DATA_TYPE_UINT8, 4, const_cast<void*>(input), dims, strides, box, estr,
                        CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                        CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
    small_tensor_fixup(&tmA, rowlen * d->H * d->N);
  } else if (pl.im2col)
    ok = encode_im2col(&tmA, A, a_chan, pl.gW, d->H, d->N, (uint64_t)a_pitch, -pl.g_pl, -d->pad_t,
                       pl.g_pr - (pl.gS - 1) * pl.g_dw, d->pad_b - (d->R - 1) * d->dil_h, pl.BK, pl.g_sw,
                       d->stride_h);
  else
    ok = encode_2d(&tmA, A, (uint64_t)a_chan, (uint64_t)pl.M, (uint64_t)a_pitch, pl.BK, kGemmBM);
  if (!ok) return QNN_ERR_UNSUPPORTED;
  ok = encode_2d(&tmB, pk + pl.pk_w, (uint64_t)taps * pl.Cw * (pl.wsplit ? 2 : 1), (uint64_t)pl.Kpad,
                 (uint64_t)taps * pl.Cw * (pl.wsplit ? 2 : 1), pl.BK,
                 pl.pair ? pl.BN / 2 : pl.BN);
  if (!ok) return QNN_ERR_UNSUPPORTED;
  // 8-bit output through per-warp TMA stores when the output pitch allows it
  // one store box per epilogue column half: 32 rows x (that half's columns), swizzled to match
  // the staging layout (32/64/128-B rows), dense for 96-B rows
  alignas(64) CUtensorMap tmC[4];
  std::memset(tmC, 0, sizeof(tmC));
  static const bool no_tma_store = std::getenv("QNN_NO_TMA_STORE") != nullptr;   // profiling switch
  const bool tma_store = !no_tma_store && !pl.a_rows && pl.requant && (pl.out_cs % 16) == 0 &&
                         (reinterpret_cast<uintptr_t>(output) & 15) == 0;
  if (tma_store) {
    // column groups of one epilogue warp set (gemm_epi_sets): 4 / nsets
    const int nepi = pl.a_build ? 8 : kGemmEpiWarps;
    const int nchunk = pl.BN / 32, ng = (nepi / 4) / gemm_epi_sets(pl.BN, pl.num_n, nepi);
    for (int h = 0; h < ng; ++h) {
      const int width = ((h + 1) * nchunk / ng - h * nchunk / ng) * 32;
      const int wb = width ? width : 32;
      const bool swz = wb == 32 || wb == 64 || wb == 128;
      if (!encode_2d(&tmC[h], output, (uint64_t)d->K, (uint64_t)pl.M, (uint64_t)pl.out_cs, wb, 32, swz))
        return QNN_ERR_UNSUPPORTED;
    }
  }

  GemmParams p{};
  p.M = (int)pl.M;
  p.Nout = d->K;
  p.nchunks = pl.nchunks;
  p.num_kb = taps * pl.nchunks;
  p.S = pl.gS;
  p.dil_h = d->dil_h;
  p.dil_w = pl.g_dw;
  p.BK = pl.BK;
  p.BN = pl.BN;
  p.stages = pl.stages;
  p.num_m_tiles = pl.num_m;
  p.num_n_tiles = pl.num_n;
  p.im2col = pl.im2col;
  p.b_res = pl.b_res_kb > 0;
  p.kps = pl.kps;
  p.a_base = reinterpret_cast<const uint8_t*>(A);
  p.a_pitch = a_pitch;
  p.H = d->H;
  p.W = pl.gW;
  p.a_halo = (d->R - 1) * d->dil_h;
  {
    static const char* dbg_env = std::getenv("QNN_GEMM_DEBUG");
    p.dbg = dbg_env ? std::atoi(dbg_env) : 0;
    // QNN_GEMM_TRACE=<device address of a zeroed 64 KiB buffer>: CTA 0 records clock64 events
    static const char* tr_env = std::getenv("QNN_GEMM_TRACE");
    p.trace = tr_env ? reinterpret_cast<unsigned long long*>(std::strtoull(tr_env, nullptr, 0)) : nullptr;
  }
  p.P = pl.P; p.Q = pl.Q; p.sh = d->stride_h; p.sw = pl.g_sw; p.pt = d->pad_t; p.pl = pl.g_pl;
  p.fdQ = make_fastdiv((uint32_t)pl.Q);
  p.fdPQ = make_fastdiv((uint32_t)(pl.P * pl.Q));
  if (pl.a_rows) {
    p.a_rows = 1;
    p.a_Wp = pl.a_Wp;
    p.a_T = pl.a_T;
    p.a_nri = pl.a_nri;
    p.a_stage_bytes = pl.a_stage_bytes;
    p.fdT = make_fastdiv((uint32_t)pl.a_T);
    p.fdWp = make_fastdiv((uint32_t)pl.a_Wp);
  }
  if (pl.a_build) {
    p.a_build = 1;
    p.a_W = d->W; p.a_C = d->C; p.a_S = d->S; p.a_sw = d->stride_w; p.a_pl = d->pad_l;
    p.a_rowlen = d->W * d->C;
    p.a_nr = pl.a_nr;
    p.a_H = d->H;
    p.a_zpfill = pl.a_zpfill;
    p.a_zp4 = 0x01010101u * (uint32_t)(d->input_zero_point & 0xFF);
    p.fdP = make_fastdiv((uint32_t)pl.P);
    p.a_slot_bytes = pl.a_slot_bytes;
    p.a_raw_bytes = pl.a_raw_bytes;
  }
  // (split weights are s8 parts whatever the kernel dtype)
  p.idesc = make_idesc_i8(d->input_dtype == QNN_S8, d->kernel_dtype == QNN_S8 || pl.wsplit,
                          pl.pair ? 2 * kGemmBM : kGemmBM, pl.BN);   // (a pair's MMA has M = 256)
  p.wsplit = pl.wsplit;
  p.pair = pl.pair ? 1 : 0;
  {
    // staged-row plans store directly (no TMA store) and their epilogue is the bound: four warp
    // sets on alternate tiles (one quad each, every column chunk) keep four tiles' epilogues in
    // flight (ResNet-50 b256 layer2 3x3 s1 47 -> 39 us, layer1 3x3 58 -> 55 us; needs 4
    // accumulators: BN <= 128).  QNN_EPI_SETS=1/2/4 overrides (A/B measurements).
    static const int es_env = std::getenv("QNN_EPI_SETS") ? std::atoi(std::getenv("QNN_EPI_SETS")) : 0;
    const int es = es_env ? es_env : 4;
    if (pl.a_rows && pl.num_n == 1 && (es == 1 || es == 2 || es == 4) && pl.BN / 32 >= 4 / es &&
        gemm_acc_bufs(pl.BN) >= es)
      p.epi_sets = es;
  }
  GemmEpilogue& ep = p.e;
  ep.off = reinterpret_cast<const int32_t*>(pk + pl.pk_off);
  ep.off64 = reinterpret_cast<const int64_t*>(pk + pl.pk_off64);
  ep.mult = reinterpret_cast<const int32_t*>(pk + pl.pk_mult);
  ep.rsh = reinterpret_cast<const int32_t*>(pk + pl.pk_rsh);
  const bool one_class = pl.ct.ncr * pl.ct.ncc == 1;
  ep.rowcls = one_class ? nullptr : pk + pl.pk_rowcls;
  ep.colcls = one_class ? nullptr : pk + pl.pk_colcls;
  ep.ncc = pl.ct.ncc;
  ep.ncls = pl.ct.ncr * pl.ct.ncc;
  ep.tma_store = tma_store;
  p.out_staging = tma_store ? 1 : 0;   // a_rows plans are sized without the staging region
  ep.rowsum = rowsum;
  ep.zpW = pl.wsplit ? 0 : d->kernel_zero_point;
  ep.out = output;
  ep.out_pitch = pl.out_cs;
  ep.Kpad = pl.Kpad;
  ep.out_dtype = pl.requant ? (int)pl.out_dt : DT_S32;
  ep.zp_out = pl.zp_out;
  ep.lo = pl.lo;
  ep.hi = pl.hi;
  if (res) {
    ep.res = reinterpret_cast<const uint8_t*>(res->ptr);
    ep.res_pitch = res_cs;
    ep.res_M = res_M;
    ep.res_rsh = res_rsh;
    ep.res_zp = res->zp;
    ep.res_s8 = res->dtype == QNN_S8;
  }
  const int grid = pl.grid;
  int64_t qlo = INT32_MIN, qhi = INT32_MAX;
  if (pl.requant) dtype_range(pl.out_dt, &qlo, &qhi);
  // the residual can push the sum past [lo, hi] even when those are the dtype bounds, but
  // the saturating pack covers the dtype range; an explicit clamp is needed only inside it
  const bool clamp = pl.requant && (pl.lo > qlo || pl.hi < qhi);
  const int mode = pl.requant ? pl.mode : 2;
  return cuda_status(launch_gemm(tmA, tmB, tmC, p, mode, clamp, grid, s));
}

// dense -> 1x1 conv over an M x 1 x 1 "image batch"
static qnn_conv2d_desc_t dense_as_conv(const qnn_dense_desc_t* d) {
  qnn_conv2d_desc_t c{};
  c.N = d->M; c.H = 1; c.W = 1; c.C = d->K; c.K = d->N; c.R = 1; c.S = 1;
  c.stride_h = c.stride_w = 1; c.dil_h = c.dil_w = 1; c.groups = 1;
  c.in_cstride = d->lda; c.out_cstride = d->ldc;
  c.input_dtype = d->a_dtype; c.kernel_dtype = d->w_dtype;
  c.input_zero_point = d->zp_A; c.kernel_zero_point = d->zp_W;
  c.kernel_zero_points = d->zp_Ws; c.num_kernel_zero_points = d->n_zpW;
  c.input_scale = d->s_A; c.kernel_scales = d->s_W; c.num_kernel_scales = d->n_sW;
  return c;
}

static qnn_status_t shape_info(const int64_t* shape, int32_t ndim, int32_t axis, long long* count, long long* inner,
                               int* cext) {
  if (!shape || ndim < 1 || ndim > 8) return QNN_ERR_INVALID_VALUE;
  if (axis < 0) axis += ndim;
  if (axis < 0 || axis >= ndim) return QNN_ERR_INVALID_VALUE;
  long long c = 1, in = 1;
  for (int i = 0; i < ndim; ++i) {
    if (shape[i] < 0) return QNN_ERR_INVALID_VALUE;
    c *= shape[i];
    if (i > axis) in *= shape[i];
  }
  *count = c;
  *inner = in > 0 ? in : 1;
  *cext = (int)shape[axis];
  return QNN_OK;
}

}  // namespace qnn

using namespace qnn;

extern "C" {

const char* qnn_status_string(qnn_status_t st) {
  switch (st) {
    case QNN_OK: return "QNN_OK";
    case QNN_ERR_INVALID_VALUE: return "QNN_ERR_INVALID_VALUE";
    case QNN_ERR_UNSUPPORTED: return "QNN_ERR_UNSUPPORTED";
    case QNN_ERR_MISALIGNED: return "QNN_ERR_MISALIGNED";
    case QNN_ERR_WORKSPACE: return "QNN_ERR_WORKSPACE";
    case QNN_ERR_CUDA: return "QNN_ERR_CUDA";
  }
  return "QNN_ERR_UNKNOWN";
}

uint64_t qnn_launch_counter(void) { return g_launches; }
void qnn_launch_counter_reset(void) { g_launches = 0; }

qnn_status_t qnn_derive_multiplier(double m, int32_t* M, int32_t* shift) {
  if (!M || !shift) return QNN_ERR_INVALID_VALUE;
  return derive_multiplier(m, M, shift) ? QNN_OK : QNN_ERR_INVALID_VALUE;
}

qnn_status_t qnn_conv2d_prepack_size(const qnn_conv2d_desc_t* d, const qnn_output_params_t* o, size_t* bytes) {
  if (!bytes) return QNN_ERR_INVALID_VALUE;
  ConvPlan pl;
  qnn_status_t st = make_plan(d, o, pl, false);
  if (st == QNN_OK) *bytes = pl.pk_total;
  return st;
}

qnn_status_t qnn_conv2d_prepack(const qnn_conv2d_desc_t* d, const void* kernel, const int32_t* bias,
                                const qnn_output_params_t* o, void* packed, size_t packed_bytes, qnn_stream_t stream) {
  return conv_prepack(d, kernel, bias, o, packed, packed_bytes, (cudaStream_t)stream);
}

qnn_status_t qnn_conv2d_workspace_size(const qnn_conv2d_desc_t* d, const qnn_output_params_t* o, size_t* bytes) {
  if (!bytes) return QNN_ERR_INVALID_VALUE;
  ConvPlan pl;
  qnn_status_t st = make_plan(d, o, pl, false);
  if (st == QNN_OK) *bytes = pl.ws_total;
  return st;
}

qnn_status_t qnn_conv2d_packed(const qnn_conv2d_desc_t* d, const qnn_output_params_t* o, const void* packed,
                               const void* input, void* output, void* workspace, size_t workspace_bytes,
                               qnn_stream_t stream) {
  return conv_packed(d, o, packed, input, output, workspace, workspace_bytes, (cudaStream_t)stream);
}

qnn_status_t qnn_conv2d_packed_add(const qnn_conv2d_desc_t* d, const qnn_output_params_t* o, const void* packed,
                                   const void* input, const void* residual, qnn_dtype_t res_dtype, float res_scale,
                                   int32_t res_zero_point, int32_t res_cstride, void* output, void* workspace,
                                   size_t workspace_bytes, qnn_stream_t stream) {
  const ResidualArgs r{residual, res_dtype, res_scale, res_zero_point, res_cstride};
  return conv_packed(d, o, packed, input, output, workspace, workspace_bytes, (cudaStream_t)stream, &r);
}

qnn_status_t qnn_conv2d(const qnn_conv2d_desc_t* d, const void* input, const void* kernel, const int32_t* bias,
                        const qnn_output_params_t* o, void* output, void* workspace, size_t workspace_bytes,
                        qnn_stream_t stream) {
  ConvPlan pl;
  qnn_status_t st = make_plan(d, o, pl, true);
  if (st != QNN_OK) return st;
  const size_t pk = align256(pl.pk_total);
  if (!workspace || workspace_bytes < pk + pl.ws_total) return QNN_ERR_WORKSPACE;
  st = conv_prepack(d, kernel, bias, o, workspace, pk, (cudaStream_t)stream);
  if (st != QNN_OK) return st;
  uint8_t* rest = reinterpret_cast<uint8_t*>(workspace) + pk;
  return conv_packed(d, o, workspace, input, output, pl.ws_total ? rest : nullptr, workspace_bytes - pk,
                     (cudaStream_t)stream);
}

qnn_status_t qnn_depthwise_conv2d(const qnn_conv2d_desc_t* d, const void* input, const void* kernel,
                                  const int32_t* bias, const qnn_output_params_t* o, void* output, void* workspace,
                                  size_t workspace_bytes, qnn_stream_t stream) {
  if (!d) return QNN_ERR_INVALID_VALUE;
  if (!(d->groups == d->C && d->K == d->C && d->groups > 1)) return QNN_ERR_INVALID_VALUE;
  return qnn_conv2d(d, input, kernel, bias, o, output, workspace, workspace_bytes, stream);
}

qnn_status_t qnn_dense_prepack_size(const qnn_dense_desc_t* d, const qnn_output_params_t* o, size_t* bytes) {
  if (!d) return QNN_ERR_INVALID_VALUE;
  const qnn_conv2d_desc_t c = dense_as_conv(d);
  return qnn_conv2d_prepack_size(&c, o, bytes);
}
qnn_status_t qnn_dense_prepack(const qnn_dense_desc_t* d, const void* W, const int32_t* bias,
                               const qnn_output_params_t* o, void* packed, size_t packed_bytes, qnn_stream_t stream) {
  if (!d) return QNN_ERR_INVALID_VALUE;
  const qnn_conv2d_desc_t c = dense_as_conv(d);
  return qnn_conv2d_prepack(&c, W, bias, o, packed, packed_bytes, stream);
}
qnn_status_t qnn_dense_workspace_size(const qnn_dense_desc_t* d, const qnn_output_params_t* o, size_t* bytes) {
  if (!d) return QNN_ERR_INVALID_VALUE;
  const qnn_conv2d_desc_t c = dense_as_conv(d);
  return qnn_conv2d_workspace_size(&c, o, bytes);
}
qnn_status_t qnn_dense_packed(const qnn_dense_desc_t* d, const qnn_output_params_t* o, const void* packed,
                              const void* A, void* out, void* workspace, size_t workspace_bytes, qnn_stream_t stream) {
  if (!d) return QNN_ERR_INVALID_VALUE;
  const qnn_conv2d_desc_t c = dense_as_conv(d);
  return qnn_conv2d_packed(&c, o, packed, A, out, workspace, workspace_bytes, stream);
}
qnn_status_t qnn_dense(const qnn_dense_desc_t* d, const void* A, const void* W, const int32_t* bias,
                       const qnn_output_params_t* o, void* out, void* workspace, size_t workspace_bytes,
                       qnn_stream_t stream) {
  if (!d) return QNN_ERR_INVALID_VALUE;
  const qnn_conv2d_desc_t c = dense_as_conv(d);
  return qnn_conv2d(&c, A, W, bias, o, out, workspace, workspace_bytes, stream);
}

qnn_status_t qnn_requantize(const void* in, qnn_dtype_t in_dtype, void* out, qnn_dtype_t out_dtype,
                            const int64_t* shape, int32_t ndim, int32_t axis, const float* in_scales,
                            int32_t n_in_scales, int32_t in_zp, float out_scale, int32_t out_zp,
                            qnn_rounding_t rounding, qnn_stream_t stream) {
  static RequantParams p;  // large (20 KB): keep off the stack; guarded below
  static std::mutex mu;
  std::lock_guard<std::mutex> lock(mu);
  long long count, inner;
  int cext;
  qnn_status_t st = shape_info(shape, ndim, axis, &count, &inner, &cext);
  if (st != QNN_OK) return st;
  int64_t lo, hi;
  if (!dtype_range(in_dtype, &lo, &hi) || !dtype_range(out_dtype, &lo, &hi)) return QNN_ERR_UNSUPPORTED;
  if (!zp_ok(in_dtype, in_zp) || !zp_ok(out_dtype, out_zp)) return QNN_ERR_INVALID_VALUE;
  if (rounding != QNN_ROUND_UPWARD && rounding != QNN_ROUND_TONEAREST) return QNN_ERR_INVALID_VALUE;
  if (!in_scales || !(n_in_scales == 1 || n_in_scales == cext)) return QNN_ERR_INVALID_VALUE;
  if (n_in_scales > kMaxChanParams) return QNN_ERR_UNSUPPORTED;
  if (!scale_ok(out_scale)) return QNN_ERR_INVALID_VALUE;
  if (count > 0 && (!in || !out)) return QNN_ERR_INVALID_VALUE;
  for (int c = 0; c < n_in_scales; ++c) {
    if (!scale_ok(in_scales[c])) return QNN_ERR_INVALID_VALUE;
    int32_t M, r;
    if (!kernel_multiplier((double)in_scales[c] / (double)out_scale, &M, &r)) return QNN_ERR_UNSUPPORTED;
    p.mult[c] = M;
    p.rsh[c] = (int8_t)r;
  }
  if (count == 0) return QNN_OK;
  p.in = in;
  p.out = out;
  p.count = count;
  p.inner = inner;
  p.cext = cext;
  p.nch = n_in_scales;
  p.in_dt = (int)in_dtype;
  p.out_dt = (int)out_dtype;
  p.mode = (int)rounding;
  p.in_zp = in_zp;
  p.out_zp = out_zp;
  p.lo = (int32_t)lo;
  p.hi = (int32_t)hi;
  return cuda_status(launch_requantize(p, (cudaStream_t)stream));
}

static qnn_status_t quant_common(const void* in, void* out, qnn_dtype_t qdt, const int64_t* shape, int32_t ndim,
                                 int32_t axis, const float* scales, const int32_t* zps, int32_t n, bool quantize,
                                 cudaStream_t stream) {
  static QuantParams p;
  static std::mutex mu;
  std::lock_guard<std::mutex> lock(mu);
  long long count, inner;
  int cext;
  qnn_status_t st = shape_info(shape, ndim, axis, &count, &inner, &cext);
  if (st != QNN_OK) return st;
  int64_t lo, hi;
  if (!dtype_range(qdt, &lo, &hi)) return QNN_ERR_UNSUPPORTED;
  if (quantize && !is_8bit(qdt)) return QNN_ERR_UNSUPPORTED;
  if (!scales || !zps || !(n == 1 || n == cext)) return QNN_ERR_INVALID_VALUE;
  if (n > kMaxQuantParams) return QNN_ERR_UNSUPPORTED;
  for (int c = 0; c < n; ++c) {
    if (!scale_ok(scales[c]) || !zp_ok(qdt, zps[c])) return QNN_ERR_INVALID_VALUE;
    p.scale[c] = scales[c];
    p.zp[c] = zps[c];
  }
  if (count > 0 && (!in || !out)) return QNN_ERR_INVALID_VALUE;
  if (count == 0) return QNN_OK;
  p.in = in;
  p.out = out;
  p.count = count;
  p.inner = inner;
  p.cext = cext;
  p.nch = n;
  p.q_dt = (int)qdt;
  p.lo = (int32_t)lo;
  p.hi = (int32_t)hi;
  return cuda_status(quantize ? launch_quantize(p, stream) : launch_dequantize(p, stream));
}

qnn_status_t qnn_quantize(const float* in, void* out, qnn_dtype_t out_dtype, const int64_t* shape, int32_t ndim,
                          int32_t axis, const float* scales, const int32_t* zero_points, int32_t n_params,
                          qnn_stream_t stream) {
  return quant_common(in, out, out_dtype, shape, ndim, axis, scales, zero_points, n_params, true,
                      (cudaStream_t)stream);
}

qnn_status_t qnn_dequantize(const void* in, qnn_dtype_t in_dtype, float* out, const int64_t* shape, int32_t ndim,
                            int32_t axis, const float* scales, const int32_t* zero_points, int32_t n_params,
                            qnn_stream_t stream) {
  return quant_common(in, out, in_dtype, shape, ndim, axis, scales, zero_points, n_params, false,
                      (cudaStream_t)stream);
}

// page-locked host memory -> the device address kernels and copies use (UVA: usually the same
// pointer); nullptr for pageable or device memory
static void* pinned_device_ptr(const void* host) {
  cudaPointerAttributes at{};
  if (!host || cudaPointerGetAttributes(&at, host) != cudaSuccess) {
    cudaGetLastError();
    return nullptr;
  }
  if (at.type != cudaMemoryTypeHost || !at.devicePointer) return nullptr;
  return at.devicePointer;
}

qnn_status_t qnn_quantize_host(const float* host_in, float* staging, void* out, qnn_dtype_t out_dtype,
                               const int64_t* shape, int32_t ndim, int32_t axis, const float* scales,
                               const int32_t* zero_points, int32_t n_params, qnn_stream_t copy_stream,
                               qnn_stream_t stream) {
  if (!shape || ndim < 1 || ndim > 8 || !staging) return QNN_ERR_INVALID_VALUE;
  int64_t count = 1;
  for (int i = 0; i < ndim; ++i) {
    if (shape[i] < 0) return QNN_ERR_INVALID_VALUE;
    count *= shape[i];
  }
  if (count > 0 && !pinned_device_ptr(host_in)) return QNN_ERR_INVALID_VALUE;
  cudaStream_t cs = (cudaStream_t)copy_stream, s = (cudaStream_t)stream;
  if (count > 0) {
    if (cudaMemcpyAsync(staging, host_in, (size_t)count * 4, cudaMemcpyHostToDevice, cs) != cudaSuccess)
      return QNN_ERR_CUDA;
    if (cs != s) {
      // the quantize waits for the copy: one event per device, recorded and waited back to back
      // (a wait binds to the record that precedes it, so reuse is safe); serialised per process
      static std::mutex mu;
      static cudaEvent_t ev[64] = {};
      int dev = 0;
      cudaGetDevice(&dev);
      if (dev >= 64) return QNN_ERR_UNSUPPORTED;
      std::lock_guard<std::mutex> lk(mu);
      if (!ev[dev] && cudaEventCreateWithFlags(&ev[dev], cudaEventDisableTiming) != cudaSuccess) return QNN_ERR_CUDA;
      if (cudaEventRecord(ev[dev], cs) != cudaSuccess || cudaStreamWaitEvent(s, ev[dev], 0) != cudaSuccess)
        return QNN_ERR_CUDA;
    }
  }
  return quant_common(staging, out, out_dtype, shape, ndim, axis, scales, zero_points, n_params, true, s);
}

qnn_status_t qnn_dequantize_host(const void* in, qnn_dtype_t in_dtype, float* host_out, const int64_t* shape,
                                 int32_t ndim, int32_t axis, const float* scales, const int32_t* zero_points,
                                 int32_t n_params, qnn_stream_t stream) {
  if (!shape || ndim < 1 || ndim > 8) return QNN_ERR_INVALID_VALUE;
  int64_t count = 1;
  for (int i = 0; i < ndim; ++i) count *= shape[i] < 0 ? 0 : shape[i];
  float* dptr = static_cast<float*>(pinned_device_ptr(host_out));
  if (count > 0 && !dptr) return QNN_ERR_INVALID_VALUE;
  return quant_common(in, dptr, in_dtype, shape, ndim, axis, scales, zero_points, n_params, false,
                      (cudaStream_t)stream);
}

}  // extern "C"

// ---------------------------------------------------------------------------------- glue
extern "C" QNN_API qnn_status_t qnn_add(const void* a, qnn_dtype_t a_dtype, float s_a, int32_t zp_a, const void* b,
                                       qnn_dtype_t b_dtype, float s_b, int32_t zp_b, void* out,
                                       qnn_dtype_t out_dtype, float s_out, int32_t zp_out, int64_t count,
                                       qnn_rounding_t rounding, int32_t relu, qnn_stream_t stream) {
  using namespace qnn;
  if (!is_8bit(a_dtype) || !is_8bit(b_dtype) || !is_8bit(out_dtype)) return QNN_ERR_INVALID_VALUE;
  if (!scale_ok(s_a) || !scale_ok(s_b) || !scale_ok(s_out)) return QNN_ERR_INVALID_VALUE;
  if (!zp_ok(a_dtype, zp_a) || !zp_ok(b_dtype, zp_b) || !zp_ok(out_dtype, zp_out)) return QNN_ERR_INVALID_VALUE;
  if (rounding != QNN_ROUND_UPWARD && rounding != QNN_ROUND_TONEAREST) return QNN_ERR_INVALID_VALUE;
  if (count < 0) return QNN_ERR_INVALID_VALUE;
  if (count == 0) return QNN_OK;
  if (!a || !b || !out) return QNN_ERR_INVALID_VALUE;
  AddParams p{};
  if (!kernel_multiplier((double)s_a / (double)s_out, &p.Ma, &p.ra) ||
      !kernel_multiplier((double)s_b / (double)s_out, &p.Mb, &p.rb))
    return QNN_ERR_UNSUPPORTED;
  p.a = a; p.b = b; p.out = out; p.count = count;
  p.vec = ((reinterpret_cast<uintptr_t>(a) | reinterpret_cast<uintptr_t>(b) | reinterpret_cast<uintptr_t>(out)) &
           15) == 0;
  p.a_s8 = a_dtype == QNN_S8; p.b_s8 = b_dtype == QNN_S8; p.o_s8 = out_dtype == QNN_S8;
  p.zp_a = zp_a; p.zp_b = zp_b; p.zp_out = zp_out;
  p.mode = (int)rounding; p.relu = relu != 0;
  return cuda_status(launch_add(p, (cudaStream_t)stream));
}

extern "C" QNN_API qnn_status_t qnn_pool2d(const qnn_pool2d_desc_t* d, const void* in, void* out,
                                          qnn_stream_t stream) {
  using namespace qnn;
  if (!d) return QNN_ERR_INVALID_VALUE;
  if (d->N <= 0 || d->H <= 0 || d->W <= 0 || d->C <= 0 || d->R <= 0 || d->S <= 0 || d->stride_h <= 0 ||
      d->stride_w <= 0 || d->pad_t < 0 || d->pad_l < 0 || d->pad_b < 0 || d->pad_r < 0)
    return QNN_ERR_INVALID_VALUE;
  if (!is_8bit(d->dtype) || (d->mode != QNN_POOL_MAX && d->mode != QNN_POOL_AVG)) return QNN_ERR_INVALID_VALUE;
  if (d->pad_t >= d->R || d->pad_b >= d->R || d->pad_l >= d->S || d->pad_r >= d->S) return QNN_ERR_INVALID_VALUE;
  const long long Hp = (long long)d->H + d->pad_t + d->pad_b, Wp = (long long)d->W + d->pad_l + d->pad_r;
  if (Hp < d->R || Wp < d->S) return QNN_ERR_INVALID_VALUE;
  PoolParams p{};
  p.P = (int)((Hp - d->R) / d->stride_h + 1);
  p.Q = (int)((Wp - d->S) / d->stride_w + 1);
  p.in_cs = d->in_cstride ? d->in_cstride : d->C;
  p.out_cs = d->out_cstride ? d->out_cstride : d->C;
  if (p.in_cs < d->C || p.out_cs < d->C) return QNN_ERR_INVALID_VALUE;
  if (!in || !out) return QNN_ERR_INVALID_VALUE;
  p.in = in; p.out = out;
  p.N = d->N; p.H = d->H; p.W = d->W; p.C = d->C; p.R = d->R; p.S = d->S;
  p.sh = d->stride_h; p.sw = d->stride_w; p.pt = d->pad_t; p.pl = d->pad_l;
  p.s8 = d->dtype == QNN_S8;
  p.avg = d->mode == QNN_POOL_AVG;
  return cuda_status(launch_pool(p, (cudaStream_t)stream));
}
