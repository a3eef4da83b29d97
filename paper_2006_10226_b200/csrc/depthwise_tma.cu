// depthwise_tma.cu — 3x3 depthwise qnn.conv2d (stride 1 or 2) on the CUDA cores with the
// input staged in shared memory by TMA (the bandwidth-bound depthwise path;
// the arithmetic is the zero-point-expanded sum of P:189-217 per channel, then the fused
// requantize of Eq. 5).
//
// Work unit ("band"): one image n, BP consecutive output rows, one slice of CS channels.  The
// band's input rows, (BP-1)*SH + 3 of them, columns -pl .. (Q-1)*SH - pl + 2, arrive in one TMA
// box (zero outside the image) in a 2-stage ring, so a CTA always has the next band in flight
// while it computes the current one -- the memory-level parallelism the register-blocked dp4a
// kernel (depthwise.cu) lacks.  Items inside a band: (channel group g of 4 channels, output
// column q); lanes take consecutive g first, so one warp's shared-memory words are contiguous.
// An item sweeps its column downwards: each input row costs 3 LDS.32 (the pixels of its three
// taps), a 3x4 -> 4x3 byte transpose, and the rows' per-channel words are reused by the (up
// to) three output rows that read them (dp4a with the filter row (w0, w1, w2, 0)).
// Out-of-image taps read zp_A (select on the loaded word), so the per-channel constant
// bias - zp_A * sum(W) of the interior holds everywhere.  Weights, multipliers and the
// requantize constants of a thread's 4 channels stay in registers: the grid is a multiple of
// the slice count, so a CTA keeps one slice, and 256 is a multiple of CS/4, so a thread keeps
// one channel group.
#include <cstdint>

#include "common.cuh"
#include "internal.h"

namespace qnn {

namespace {

__device__ __forceinline__ void dwt_tma_load_4d(void* dst, const void* desc, uint64_t* bar, int c0, int c1, int c2,
                                                int c3) {
  asm volatile(
      "cp.async.bulk.tensor.4d.shared::cluster.global.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%3, %4, %5, %6}], [%2];" ::"r"(smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(desc)), "r"(smem_u32(bar)), "r"(c0), "r"(c1), "r"(c2), "r"(c3)
      : "memory");
}

template <bool ASIGNED>
__device__ __forceinline__ int32_t dwt_dp4a(uint32_t a, uint32_t w, int32_t c) {
  int32_t d;
  if (ASIGNED)
    asm("dp4a.s32.s32 %0, %1, %2, %3;" : "=r"(d) : "r"(a), "r"(w), "r"(c));
  else
    asm("dp4a.u32.s32 %0, %1, %2, %3;" : "=r"(d) : "r"(a), "r"(w), "r"(c));
  return d;
}

}  // namespace

#ifndef QNN_DWT_UNROLL
#define QNN_DWT_UNROLL 3   // (3: the three-row window rotation becomes register renaming)
#endif
constexpr int kDwtThreads = 256;

// One band of a stage: items (channel group g, output column q), lanes on consecutive g.  An
// item sweeps its column downwards: per input row 3 LDS.32 (its taps' pixels, zp_A outside the
// image), a 3x4 -> 4x3 byte transpose, and the per-channel words of the last three rows feed
// one output row (dp4a with the filter rows (w0, w1, w2, 0)).
// (Measured alternatives, all slower on the MobileNet-v2 b128 layers: column pairs per item
// with a shifted filter, vertical segments for load balance, a dedicated producer warp with
// zp_A written into the halo instead of selects, 2 CTAs/SM at 128 registers.)
template <int SH, int CLAMP, bool S8OUT, bool ASIGNED, bool FAST>
__device__ __forceinline__ void dwt_band(const DwParams& p, const uint8_t* __restrict__ st, int n, int p0, int np,
                                         int h0, int c0, int g, const uint32_t (&wr)[3][4], const int32_t (&Mc)[4],
                                         const int32_t (&Tc)[4], const int32_t (&Rc)[4], const long long (&Kc)[4],
                                         const int32_t (&off32)[4], uint32_t zfill) {
  const int cs = p.dwt_cs, lg = __ffs(cs >> 2) - 1;   // G = cs / 4 channel groups (a power of 2)
  const int items = p.Q << lg;
  const int rows = (np - 1) * SH + 3;
  const uint32_t row_bytes = (uint32_t)(p.dwt_wb * cs);
  const long long ostride = (long long)p.Q * p.out_cstride;   // one output row
  uint8_t* out = reinterpret_cast<uint8_t*>(p.out) + ((long long)n * p.P + p0) * ostride + c0;
  const uint32_t st_base = smem_u32(st) + 4u * (uint32_t)g;
  // band rows inside the image: ir in [ir_lo, ir_lo + nin) (one unsigned compare per row)
  const int ir_lo = max(0, -h0);
  const uint32_t nin = (uint32_t)max(0, min(rows, p.H - h0) - ir_lo);
  const int pl = p.pl, Wd = p.W;
  for (int it = threadIdx.x; it < items; it += kDwtThreads) {
    const int q = it >> lg;   // (it % G == g: kDwtThreads % G == 0)
    const int x = q * SH;     // box column of the first tap (box starts at input column -pl)
    // every tap's column checked against [0, W): with pl >= 2 (or a right pad >= 2) the middle
    // tap can fall outside the image too, and the TMA zero fill is not zp_A
    const bool c0ok = (unsigned)(x - pl) < (unsigned)Wd, c1ok = (unsigned)(x + 1 - pl) < (unsigned)Wd,
               c2ok = (unsigned)(x + 2 - pl) < (unsigned)Wd;
    uint32_t a = st_base + (uint32_t)(x * cs);
    uint8_t* dst = out + (long long)q * p.out_cstride;
    uint32_t T0[4], T1[4], T2[4];   // per-channel words of the last three input rows (bytes: 3 taps + junk)
#if defined(QNN_DWT_NO_UNROLL)
#pragma unroll 1
#else
#pragma unroll(SH == 1 ? 3 : 2)   // the window rotation becomes register renaming
#endif
    for (int ir = 0; ir < rows; ++ir, a += row_bytes) {
      const bool row_ok = (uint32_t)(ir - ir_lo) < nin;
      uint32_t wv[3];
      asm volatile("ld.shared.u32 %0, [%1];" : "=r"(wv[0]) : "r"(a));
      asm volatile("ld.shared.u32 %0, [%1];" : "=r"(wv[1]) : "r"(a + cs));
      asm volatile("ld.shared.u32 %0, [%1];" : "=r"(wv[2]) : "r"(a + 2 * cs));
      wv[0] = row_ok && c0ok ? wv[0] : zfill;
      wv[1] = row_ok && c1ok ? wv[1] : zfill;
      wv[2] = row_ok && c2ok ? wv[2] : zfill;
      // 3 pixels x 4 channels -> 4 channels x 3 pixels (byte 3 multiplies the filter's 0)
      const uint32_t t0 = __byte_perm(wv[0], wv[1], 0x5140), t1 = __byte_perm(wv[0], wv[1], 0x7362);
#pragma unroll
      for (int ch = 0; ch < 4; ++ch) {
        T0[ch] = T1[ch];
        T1[ch] = T2[ch];
      }
      T2[0] = __byte_perm(t0, wv[2], 0x4410);
      T2[1] = __byte_perm(t0, wv[2], 0x5532);
      T2[2] = __byte_perm(t1, wv[2], 0x6610);
      T2[3] = __byte_perm(t1, wv[2], 0x7732);
      if (ir < 2 || (SH == 2 && (ir & 1))) continue;
      int32_t y[4];
#pragma unroll
      for (int ch = 0; ch < 4; ++ch) {
        int32_t acc = dwt_dp4a<ASIGNED>(T0[ch], wr[0][ch], 0);
        acc = dwt_dp4a<ASIGNED>(T1[ch], wr[1][ch], acc);
        acc = dwt_dp4a<ASIGNED>(T2[ch], wr[2][ch], acc);
        int32_t v;
        if (FAST) {
          v = mad_hi64(acc, Mc[ch], Kc[ch]) >> Tc[ch];
        } else {
          const int32_t xv = (int32_t)((uint32_t)acc + (uint32_t)off32[ch]);
          v = rq_apply(xv, Mc[ch], Rc[ch], p.mode, p.zp_out, p.lo, p.hi);
        }
        if (CLAMP == 2) v = max(v, p.lo);
        if (CLAMP != 0) v = min(v, p.hi);
        y[ch] = v;
      }
      uint32_t word;
      if (S8OUT)
        asm("{\n\t.reg .u32 t;\n\tcvt.pack.sat.s8.s32.b32 t, %4, %3, 0;\n\tcvt.pack.sat.s8.s32.b32 %0, %2, %1, t;\n\t}"
            : "=r"(word) : "r"(y[0]), "r"(y[1]), "r"(y[2]), "r"(y[3]));
      else
        asm("{\n\t.reg .u32 t;\n\tcvt.pack.sat.u8.s32.b32 t, %4, %3, 0;\n\tcvt.pack.sat.u8.s32.b32 %0, %2, %1, t;\n\t}"
            : "=r"(word) : "r"(y[0]), "r"(y[1]), "r"(y[2]), "r"(y[3]));
      *reinterpret_cast<uint32_t*>(dst) = word;   // output row (ir - 2) / SH of the band
      dst += ostride;
    }
  }
}

template <int SH, int CLAMP, bool S8OUT, bool ASIGNED>
__global__ void __launch_bounds__(kDwtThreads, 3) dw3_tma_kernel(const __grid_constant__ CUtensorMap tm,
                                                                 const __grid_constant__ DwParams p) {
  pdl_wait();      // inputs are the previous kernel's output (PDL launch; no early trigger: the
                   // next kernel's CTAs would take this multi-wave grid's slots while waiting)
  extern __shared__ __align__(128) uint8_t dwt_smem[];
  __shared__ __align__(8) uint64_t full[2];
  const int CS = p.dwt_cs, G = CS >> 2;
  const int nsl = p.C / CS;
  const int PB = (p.P + p.dwt_bp - 1) / p.dwt_bp;
  const int nbands = p.N * PB * nsl;
  const int slice = blockIdx.x % nsl;   // fixed per CTA: gridDim.x % nsl == 0
  const int g = threadIdx.x % G;        // fixed per thread: kDwtThreads % G == 0
  const int c0 = slice * CS + 4 * g;
  const int stage_bytes = p.dwt_stage_bytes;
  const uint32_t box_bytes = (uint32_t)(((p.dwt_bp - 1) * SH + 3) * p.dwt_wb * CS);
  if (threadIdx.x == 0) {
    tma_prefetch_desc(&tm);
    mbar_init(&full[0], 1);
    mbar_init(&full[1], 1);
    fence_mbar_init();
  }
  __syncthreads();
  // band b = blockIdx.x + k * gridDim.x -> (slice = b % nsl, pb, n)
  auto issue = [&](int b, int stg) {
    const int rest = b / nsl;
    const int pb = rest % PB, n = rest / PB;
    mbar_arrive_expect_tx(&full[stg], box_bytes);
    dwt_tma_load_4d(dwt_smem + (size_t)stg * stage_bytes, &tm, &full[stg], slice * CS, -p.pl,
                    pb * p.dwt_bp * SH - p.pt, n);
  };
  if (threadIdx.x == 0) {
    if ((int)blockIdx.x < nbands) issue(blockIdx.x, 0);
    if ((int)(blockIdx.x + gridDim.x) < nbands) issue(blockIdx.x + gridDim.x, 1);
  }
  // per-thread channel constants (as depthwise3_kernel): filter rows (w0, w1, w2, 0) per channel
  uint32_t wr[3][4];
  long long wsum[4] = {0, 0, 0, 0};
#pragma unroll
  for (int ch = 0; ch < 4; ++ch)
#pragma unroll
    for (int r = 0; r < 3; ++r) {
      uint32_t word = 0;
#pragma unroll
      for (int s = 0; s < 3; ++s) {
        const int v = p.w[(r * 3 + s) * p.C + c0 + ch];
        wsum[ch] += v;
        word |= ((uint32_t)v & 0xFFu) << (8 * s);
      }
      wr[r][ch] = word;
    }
  int32_t Mc[4], Tc[4], Rc[4], off32[4];
  long long Kc[4];
  bool fast = p.mode == RND_UPWARD;
#pragma unroll
  for (int ch = 0; ch < 4; ++ch) {
    const int c = c0 + ch;
    const long long off = (p.bias ? (long long)p.bias[c] : 0) - (long long)p.zpA * wsum[ch];
    off32[ch] = (int32_t)(uint32_t)(unsigned long long)off;
    Mc[ch] = p.mult[c];
    const int r = p.rsh[c];
    Rc[ch] = r;
    Tc[ch] = 0;
    Kc[ch] = 0;
    if (r >= 33 && r <= 52) {
      const int t = r - 32;
      const unsigned long long c64 = (1ull << (t - 1)) + ((unsigned long long)(long long)p.zp_out << t);
      Kc[ch] = (long long)((unsigned long long)off * (unsigned long long)(long long)Mc[ch] + (c64 << 32));
      Tc[ch] = t;
    } else {
      fast = false;
    }
  }
  const uint32_t zfill = 0x01010101u * (uint32_t)(p.zpA & 0xFF);
  int k = 0;
  for (int b = blockIdx.x; b < nbands; b += gridDim.x, ++k) {
    const int stg = k & 1;
    const int rest = b / nsl;
    const int pb = rest % PB, n = rest / PB;
    const int p0 = pb * p.dwt_bp;
    const int np = min(p.dwt_bp, p.P - p0);
    mbar_wait(&full[stg], (uint32_t)((k >> 1) & 1));
    const uint8_t* st = dwt_smem + (size_t)stg * stage_bytes;
    if (fast)
      dwt_band<SH, CLAMP, S8OUT, ASIGNED, true>(p, st, n, p0, np, p0 * SH - p.pt, c0, g, wr, Mc, Tc, Rc, Kc, off32,
                                                 zfill);
    else
      dwt_band<SH, CLAMP, S8OUT, ASIGNED, false>(p, st, n, p0, np, p0 * SH - p.pt, c0, g, wr, Mc, Tc, Rc, Kc, off32,
                                                  zfill);
    __syncthreads();   // every thread is done with this stage: refill it
    if (threadIdx.x == 0 && b + 2 * (int)gridDim.x < nbands) issue(b + 2 * gridDim.x, stg);
  }
}

// Band geometry: CS (16/32/64 channels, dividing C), box width Wb, BP output rows per band
// (~32 KB stages); false if the shape is not eligible.
bool dwtma_plan(DwParams& p) {
  if (!(p.R == 3 && p.S == 3 && p.dh == 1 && p.dw == 1 && p.sh == p.sw && (p.sh == 1 || p.sh == 2))) return false;
  if (!p.requant || p.out_dtype == DT_S32 || !p.w_fits_s8) return false;
  if (p.C % 16 || p.in_cstride % 16 || p.out_cstride % 4) return false;
  if (((reinterpret_cast<uintptr_t>(p.in) & 15) | (reinterpret_cast<uintptr_t>(p.out) & 3)) != 0) return false;
  const int wb = (p.Q - 1) * p.sh + 3;
  if (wb > 256) return false;
  int cs = 64;
  while (cs > 16 && p.C % cs) cs >>= 1;
  const int rows_max = std::min(256, 32768 / (wb * cs));
  if (rows_max < 3) return false;
  const int bp = std::max(1, std::min(p.P, (rows_max - 3) / p.sh + 1));
  p.dwt_cs = cs;
  p.dwt_wb = wb;
  p.dwt_bp = bp;
  p.dwt_stage_bytes = (((bp - 1) * p.sh + 3) * wb * cs + 127) / 128 * 128;
  return true;
}

cudaError_t launch_depthwise_tma(const CUtensorMap& tm, const DwParams& p, int clamp, cudaStream_t s) {
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const size_t smem = 2 * (size_t)p.dwt_stage_bytes;
  const int per_sm = std::max(1, std::min(8, (int)((200 * 1024) / (smem + 1024))));
  const int nsl = p.C / p.dwt_cs;
  const long long nbands = (long long)p.N * ((p.P + p.dwt_bp - 1) / p.dwt_bp) * nsl;
  long long grid = std::min<long long>(nbands, (long long)sms * per_sm);
  grid = std::max<long long>(nsl, grid / nsl * nsl);   // a CTA keeps one channel slice
  const bool s8 = p.out_dtype == DT_S8;
#define QNN_DWT(SH_, C_, S_, A_)                                                                            \
  if (p.sh == SH_ && clamp == C_ && s8 == S_ && (p.a_signed != 0) == A_) {                                  \
    auto kern = dw3_tma_kernel<SH_, C_, S_, A_>;                                                            \
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);     \
    if (e != cudaSuccess) return e;                                                                          \
    launch_pdl(kern, dim3((int)grid), dim3(kDwtThreads), smem, s, tm, p);                                                        \
    count_launch();                                                                                          \
    return cudaGetLastError();                                                                               \
  }
#define QNN_DWT_A(SH_, C_, S_) QNN_DWT(SH_, C_, S_, false) QNN_DWT(SH_, C_, S_, true)
#define QNN_DWT_S(SH_, C_) QNN_DWT_A(SH_, C_, false) QNN_DWT_A(SH_, C_, true)
#define QNN_DWT_C(SH_) QNN_DWT_S(SH_, 0) QNN_DWT_S(SH_, 1) QNN_DWT_S(SH_, 2)
  QNN_DWT_C(1) QNN_DWT_C(2)
#undef QNN_DWT_C
#undef QNN_DWT_S
#undef QNN_DWT_A
#undef QNN_DWT
  return cudaErrorInvalidValue;
}

}  // namespace qnn
