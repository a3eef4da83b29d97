// gemm_t.cu — channel-major ("transposed") tcgen05 GEMM for wide pointwise convolutions
// (SURVEY §8 rows a3 + a4: the Term-1 contraction and the fused requantize of Eq. 5,
// P:273-281, for 1x1 / stride-1 / unpadded qnn.conv2d with K_out % 128 == 0, zp_W == 0).
//
// The pixel-major kernel (gemm_sm100.cu) puts output pixels on the TMEM lanes, so every
// epilogue lane needs every column's requantize constants: one shared-memory broadcast per
// (lane-row, column pair), and the wide 1x1 layers (K_out 256..2048 over a short reduction)
// are bound by that epilogue.  Here the MMA computes D^T = W * A^T: M = 128 output channels
// (A operand = the packed weights, resident in shared memory for the CTA's channel block),
// N = 256 pixels (B operand = the activation rows, streamed by TMA), so a TMEM lane is ONE
// output channel.  The weight rows are packed in the order perm32 (prep.cu): TMEM lane
// j + 8i of a 32-lane quadrant holds channel 4j + i, so the 16x256b TMEM load (thread
// (j = lane/4, u = lane%4) receives lanes j and j+8, or j+16 and j+24, at pixel columns
// 8r + 2u + {0, 1}) hands every thread four CONSECUTIVE output channels of a pixel: their
// four requantize constants live in its registers for the whole kernel, and each requantized
// group of four is one packed 32-bit word, stored with one STS.32 into a [64 pixels][32
// channels] staging tile that leaves by TMA store (previously one STS.U8 per output byte).
//
// Grid: a multiple of the channel-block count, so a CTA keeps one channel block (weights and
// constants loaded once; weights streamed per stage when the block does not fit); pixel
// tiles advance by grid / blocks.
// Warps: 0-15 epilogue (warp w: TMEM lanes 32*(w%4), pixel columns 64*(w/4)), 16 TMA
// producer, 17 MMA issuer + TMEM allocator (2 accumulators x 256 columns).
#include <cstdint>
#include <cstdio>
#include <cstdlib>

#include "epilogue.cuh"

// waits of the many-warp roles (epilogue, builders); QNN_EPI_SLEEP=1 at build time selects the
// sleeping poll (measured neutral on the ResNet-50 b256 layers, so off)
#ifdef QNN_EPI_SLEEP
#define QNN_EPI_WAIT mbar_wait_sleep
#else
#define QNN_EPI_WAIT mbar_wait
#endif
#include "internal.h"

namespace qnn {

namespace {

#ifdef QNN_GEMM_INSTRUMENT
constexpr bool kTInstrument = true;    // QNN_GEMM_DEBUG knobs compiled in (profiling builds only)
#else
constexpr bool kTInstrument = false;
#endif

constexpr int kTEpiWarps = 16;
constexpr int kTThreads = 32 * kTEpiWarps + 64;
constexpr int kTBM = 128;   // output channels per tile (MMA M)
constexpr int kTBN = kGemmTBN;          // pixels per tile (MMA N), internal.h
constexpr int kTNacc = 512 / kTBN;      // TMEM accumulator buffers (512 columns)
constexpr int kTCols = kTBN / 4;        // pixel columns per epilogue warp (4 column groups)
constexpr int kTHalves = kTCols / 32;   // 32-column steps per warp and tile
// output staging, per column group (the 4 warps of one group of pixel columns share it):
// [kTCols pixels][128 channels] in the TMA 128-B swizzle (16-B chunk c of row r at chunk
// c ^ (r % 8)), one TMA store of 128-B rows per group and tile; 1 or 2 buffers (host choice)
constexpr int kTGroupOut = kTCols * 128;
#ifdef QNN_T_SPIN
#define QNN_T_WAIT mbar_wait_spin
#else
#define QNN_T_WAIT mbar_wait
#endif

__device__ __forceinline__ void sts32(uint32_t addr, uint32_t v) {
  asm volatile("st.shared.u32 [%0], %1;" ::"r"(addr), "r"(v));
}
__device__ __forceinline__ uint32_t lds32(uint32_t addr) {
  uint32_t v;
  asm volatile("ld.shared.u32 %0, [%1];" : "=r"(v) : "r"(addr));
  return v;
}

// 16 TMEM lanes x 32 columns (16x256b.x4), not waited: thread (j, u) = (lane/4, lane%4)
// receives r[4k + e] = (lane base + j, column 8k + 2u + e), r[4k + 2 + e] = (base + 8 + j, same)
__device__ __forceinline__ void tmem_ld_16x256b_x4(uint32_t taddr, uint32_t (&r)[16]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.16x256b.x4.b32 "
      "{%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
        "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
      : "r"(taddr));
}
__device__ __forceinline__ void tmem_wait16x2(uint32_t (&a)[16], uint32_t (&b)[16]) {
  asm volatile("tcgen05.wait::ld.sync.aligned;"
               : "+r"(a[0]), "+r"(a[1]), "+r"(a[2]), "+r"(a[3]), "+r"(a[4]), "+r"(a[5]), "+r"(a[6]), "+r"(a[7]),
                 "+r"(a[8]), "+r"(a[9]), "+r"(a[10]), "+r"(a[11]), "+r"(a[12]), "+r"(a[13]), "+r"(a[14]),
                 "+r"(a[15]), "+r"(b[0]), "+r"(b[1]), "+r"(b[2]), "+r"(b[3]), "+r"(b[4]), "+r"(b[5]), "+r"(b[6]),
                 "+r"(b[7]), "+r"(b[8]), "+r"(b[9]), "+r"(b[10]), "+r"(b[11]), "+r"(b[12]), "+r"(b[13]),
                 "+r"(b[14]), "+r"(b[15])
               :
               : "memory");
}

// the residual byte requantized to the output scale with zero point 0 (reading R19: added
// to the conv's requantized value before the clamp)
template <int MODE>
__device__ __forceinline__ int32_t res_term(const GemmTParams& p, uint32_t word, int byte) {
  const uint32_t b = (word >> (8 * byte)) & 0xFFu;
  const int32_t x = (p.res_s8 ? (int32_t)(int8_t)b : (int32_t)b) - p.res_zp;
  return (int32_t)rq_round((int64_t)x * p.res_M, p.res_rsh, MODE);
}

// one thread's four channels: requantize constants in registers for the whole kernel
//   fast (UPWARD, rsh = 32 + t, t in [1, 20]): y = hi32(v * M + K) >> t with the 64-bit
//     K = off * M + (2^(t-1) + zp_out * 2^t) * 2^32 (modular int64: exact whenever the true
//     v + off fits int32, reading R10).  Written as 64-bit C++ so ptxas emits ONE IMAD.HI with
//     the persistent 64-bit K as its addend (an inline mad.wide became IMAD.WIDE + IMAD.X).
//   generic: exact 64-bit rounding of (v + off) * M by rsh (k holds off, t holds rsh)
struct TChan {
  int32_t M[4], t[4];
  long long k[4];
};

template <int MODE, bool FAST>
__device__ __forceinline__ int32_t tq1(const TChan& q, int i, uint32_t acc, int32_t zp_out) {
  if (FAST) return mad_hi64((int32_t)acc, q.M[i], q.k[i]) >> q.t[i];
  const long long z = rq_round(((long long)(int32_t)acc + q.k[i]) * q.M[i], q.t[i], MODE) + zp_out;
  return (int32_t)(z < INT32_MIN ? INT32_MIN : (z > INT32_MAX ? INT32_MAX : z));
}

// 32 of the warp's pixel columns x its quadrant's 32 channels: requantize, (residual), clamp,
// pack 4 channels per word, store into the staging tile [pixel][32 channels]
template <int MODE, bool FAST, bool CLAMP, bool S8OUT, bool RES>
__device__ __forceinline__ void t_epilogue(const GemmTParams& p, const TChan& q, const uint32_t (&va)[16],
                                           const uint32_t (&vb)[16], uint32_t st0, uint32_t st1) {
#pragma unroll
  for (int k = 0; k < 4; ++k) {
#pragma unroll
    for (int e = 0; e < 2; ++e) {
      // pixel column 8k + 2u + e of this 32-column step; channels 4j + i from lanes j, j+8 (va)
      // and j+16, j+24 (vb); the swizzled word address depends on e and the thread only
      const uint32_t a = (e ? st1 : st0) + (uint32_t)(8 * k * 128);
      int32_t y[4];
      y[0] = tq1<MODE, FAST>(q, 0, va[4 * k + e], p.zp_out);
      y[1] = tq1<MODE, FAST>(q, 1, va[4 * k + 2 + e], p.zp_out);
      y[2] = tq1<MODE, FAST>(q, 2, vb[4 * k + e], p.zp_out);
      y[3] = tq1<MODE, FAST>(q, 3, vb[4 * k + 2 + e], p.zp_out);
      if (RES) {
        const uint32_t rw = lds32(a);
#pragma unroll
        for (int i = 0; i < 4; ++i) y[i] += res_term<MODE>(p, rw, i);
      }
      if (CLAMP || !FAST) {
#pragma unroll
        for (int i = 0; i < 4; ++i) y[i] = min(max(y[i], p.lo), p.hi);
      }
      sts32(a, S8OUT ? pack4_s8(y[0], y[1], y[2], y[3]) : pack4_u8(y[0], y[1], y[2], y[3]));
    }
  }
}

}  // namespace

constexpr int kTSmemMax = 227 * 1024 - 1024;   // dynamic budget (the barriers are static)

// w_res: the CTA's weight block stays resident (num_kb blocks); otherwise each pipeline stage
// carries its weight k-block next to the activation k-block
size_t gemm_t_smem_bytes(int BK, int num_kb, int stages, bool w_res, int stage_bufs) {
  const size_t stage = (size_t)kTBN * BK + (w_res ? 0 : (size_t)kTBM * BK);
  return 1024 + (size_t)stages * stage + (w_res ? (size_t)num_kb * kTBM * BK : 0) +
         (size_t)4 * kTGroupOut * stage_bufs + 256;
}

int gemm_t_max_stages(int BK, int num_kb, bool w_res, int stage_bufs) {
  int s = 8;
  while (s > 2 && gemm_t_smem_bytes(BK, num_kb, s, w_res, stage_bufs) > (size_t)kTSmemMax) --s;
  return s;
}

template <int MODE, bool CLAMP, bool S8OUT, bool RES>
__global__ void __launch_bounds__(kTThreads, 1)
    qnn_gemm_t_kernel(const __grid_constant__ CUtensorMap tmX, const __grid_constant__ CUtensorMap tmW,
                      const __grid_constant__ CUtensorMap tmC, const __grid_constant__ CUtensorMap tmR,
                      const __grid_constant__ GemmTParams p) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = smem_raw + ((1024 - (smem_u32(smem_raw) & 1023)) & 1023);
  const int BK = p.BK, stages = p.stages, num_kb = p.num_kb;
  const uint32_t x_bytes = (uint32_t)kTBN * BK, w_bytes = (uint32_t)kTBM * BK;
  const bool w_res = p.w_res;
  uint8_t* sX = smem;                                  // stages x [256 pixels][BK]
  uint8_t* sW = sX + (size_t)stages * x_bytes;         // num_kb (resident) or stages x [128 channels][BK]
  uint8_t* sOut = sW + (size_t)(w_res ? num_kb : stages) * w_bytes;   // 16 x [64 pixels][32 channels]
  __shared__ __align__(8) uint64_t full[8], empty[8], tfull[kTNacc], tempty[kTNacc], wfull, rbar[4];
  __shared__ uint32_t tmem_slot;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  constexpr int kProdWarp = kTEpiWarps, kMmaWarp = kTEpiWarps + 1;
  const int nct = p.num_ch_tiles, npt = p.num_px_tiles;
  const int ch = blockIdx.x % nct;                  // fixed channel block (gridDim.x % nct == 0)
  const int px_first = blockIdx.x / nct, px_step = gridDim.x / nct;
  if (warp == kProdWarp && lane == 0) {
    tma_prefetch_desc(&tmX);
    tma_prefetch_desc(&tmW);
    tma_prefetch_desc(&tmC);
    if (RES) tma_prefetch_desc(&tmR);
    for (int s = 0; s < stages; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    for (int a = 0; a < kTNacc; ++a) {
      mbar_init(&tfull[a], 1);
      mbar_init(&tempty[a], kTEpiWarps);
    }
    mbar_init(&wfull, 1);
    for (int g = 0; g < 4; ++g) mbar_init(&rbar[g], 1);
    fence_mbar_init();
  }
  if (warp == kMmaWarp) tmem_alloc(&tmem_slot, 512);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = tmem_slot;

  if (warp == kProdWarp) {
    const bool leader = elect_one();
    if (leader && w_res && px_first < npt) {
      mbar_arrive_expect_tx(&wfull, (uint32_t)num_kb * w_bytes);
      for (int kb = 0; kb < num_kb; ++kb) tma_load_2d(sW + (size_t)kb * w_bytes, &tmW, &wfull, kb * BK, ch * kTBM);
    }
    int stage = 0;
    uint32_t phase = 0;
    for (int pt = px_first; pt < npt; pt += px_step) {
      for (int kb = 0; kb < num_kb; ++kb) {
        QNN_T_WAIT(&empty[stage], phase ^ 1);
        if (leader) {
          mbar_arrive_expect_tx(&full[stage], x_bytes + (w_res ? 0 : w_bytes));
          tma_load_2d(sX + (size_t)stage * x_bytes, &tmX, &full[stage], kb * BK, pt * kTBN);
          if (!w_res) tma_load_2d(sW + (size_t)stage * w_bytes, &tmW, &full[stage], kb * BK, ch * kTBM);
        }
        __syncwarp();
        if (++stage == stages) {
          stage = 0;
          phase ^= 1;
        }
      }
    }
  } else if (warp == kMmaWarp) {
    const bool leader = elect_one();
    const uint64_t wdesc0 = make_sdesc(smem_u32(sW), BK), xdesc0 = make_sdesc(smem_u32(sX), BK);
    const uint32_t idesc = p.idesc, w16 = w_bytes >> 4, x16 = x_bytes >> 4;
    const int ksteps = BK / 32;
    int stage = 0, it = 0;
    uint32_t phase = 0;
    if (w_res && px_first < npt) mbar_wait(&wfull, 0);
    for (int pt = px_first; pt < npt; pt += px_step, ++it) {
      const int acc = it % kTNacc;
      QNN_T_WAIT(&tempty[acc], ((it / kTNacc) & 1) ^ 1);
      tc_fence_after();
      const uint32_t d = tmem_base + (uint32_t)acc * kTBN;
      for (int kb = 0; kb < num_kb; ++kb) {
        QNN_T_WAIT(&full[stage], phase);
        tc_fence_after();
        if (leader) {
          const uint64_t wd = wdesc0 + (uint64_t)(w_res ? kb : stage) * w16, xd = xdesc0 + (uint64_t)stage * x16;
          for (int k = 0; k < ksteps; ++k) umma_i8(d, wd + 2 * k, xd + 2 * k, idesc, (kb | k) != 0);
          umma_commit(&empty[stage]);
        }
        __syncwarp();
        if (++stage == stages) {
          stage = 0;
          phase ^= 1;
        }
      }
      if (leader) umma_commit(&tfull[acc]);
      __syncwarp();
    }
  } else if (warp < kTEpiWarps) {
    // ---------------------------------------------------------------- epilogue
    const int quad = warp & 3, grp = warp >> 2;
    const int j = lane >> 2, u = lane & 3;
    // (K_out = 64: the upper half of the 128-channel block is zero weights; its quads compute
    // nothing and their stores fall outside the output tensor, which TMA drops)
    const bool quad_live = ch * kTBM + quad * 32 < p.Kout;
    TChan q;
    bool fast = MODE == 0;
    const int k0 = ch * kTBM + quad * 32 + 4 * j;   // this thread's channels k0 .. k0 + 3
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const int kk = k0 + i < p.Kout ? k0 + i : 0;
      const int32_t rsh = p.rsh[kk];
      const long long off = p.off64[kk];
      q.M[i] = p.mult[kk];
      if (MODE == 0 && rsh >= 33 && rsh <= 52) {
        const int t = rsh - 32;
        const unsigned long long c64 = (1ull << (t - 1)) + ((unsigned long long)(long long)p.zp_out << t);
        q.t[i] = t;
        q.k[i] = (long long)((unsigned long long)off * (unsigned long long)(long long)q.M[i] + (c64 << 32));
      } else {
        fast = false;
        q.t[i] = rsh;
        q.k[i] = off;
      }
    }
    const int dbg = kTInstrument ? p.dbg : 0;
    const bool all_fast = __all_sync(0xffffffffu, fast);
    // column group grp shares a [kTCols][128] staging tile (1 or 2 buffers) with the other 3
    // quads; its quad-0 lane 0 issues the group's TMA store (and residual load)
    const bool gleader = quad == 0 && lane == 0;
    const int nbufs = p.stage_bufs;
    uint8_t* const gstage = sOut + (size_t)grp * kTGroupOut * nbufs;
    // this thread's words (pixel rows 2u + e, e = 0/1; channel word 8 quad + j) in the 128-B swizzle
    const uint32_t ch16 = (uint32_t)(2 * quad + (j >> 2));
    const uint32_t st_off0 = (uint32_t)(2 * u) * 128 + ((ch16 ^ (uint32_t)(2 * u)) << 4) + (uint32_t)((j & 3) << 2);
    const uint32_t st_off1 = (uint32_t)(2 * u + 1) * 128 + ((ch16 ^ (uint32_t)(2 * u + 1)) << 4) +
                             (uint32_t)((j & 3) << 2);
    int it = 0;
    for (int pt = px_first; pt < npt; pt += px_step, ++it) {
      const int acc = it % kTNacc;
      uint8_t* const stage_out = gstage + (nbufs == 2 ? (it & 1) * kTGroupOut : 0);
      const uint32_t sbase = smem_u32(stage_out);
      if (gleader) {
        bulk_wait_read_dyn(nbufs - 1);   // the store that last used this buffer has read it
        if (RES) {
          // the residual tile (this group's pixels x 128 channels, same swizzle) lands in the
          // staging buffer; each thread reads its four channels' word per pixel and overwrites it
          mbar_arrive_expect_tx(&rbar[grp], kTGroupOut);
          tma_load_2d(stage_out, &tmR, &rbar[grp], ch * kTBM, pt * kTBN + grp * kTCols);
        }
      }
      named_bar_sync(1 + grp, 128);      // the buffer is free for every warp of the group
      QNN_EPI_WAIT(&tfull[acc], (it / kTNacc) & 1);
      tc_fence_after();
      const uint32_t tb = tmem_base + (uint32_t)acc * kTBN + ((uint32_t)(quad * 32) << 16) + (uint32_t)(grp * kTCols);
      if (RES) mbar_wait(&rbar[grp], (uint32_t)(it & 1));
      // steps of 32 pixel columns (register budget: 96 per thread at 18 warps)
#pragma unroll 1
      for (int h = 0; h < kTHalves; ++h) {
        uint32_t va[16], vb[16];
        tmem_ld_16x256b_x4(tb + 32 * h, va);                  // lanes j, j + 8
        tmem_ld_16x256b_x4(tb + 32 * h + (16u << 16), vb);    // lanes j + 16, j + 24
        tmem_wait16x2(va, vb);
        if (h == kTHalves - 1) {
          tc_fence_before();
          __syncwarp();
          if (lane == 0) mbar_arrive(&tempty[acc]);
        }
        const uint32_t rowb = sbase + (uint32_t)(h * 32 * 128);
        // (warp-uniform choice: a per-lane branch would be if-converted and issue both paths)
        if ((dbg & 1) || !quad_live) {
        } else if (all_fast) {
          t_epilogue<MODE, true, CLAMP, S8OUT, RES>(p, q, va, vb, rowb + st_off0, rowb + st_off1);
        } else {
          t_epilogue<MODE, false, CLAMP, S8OUT, RES>(p, q, va, vb, rowb + st_off0, rowb + st_off1);
        }
      }
      fence_proxy_async_smem();
      named_bar_sync(1 + grp, 128);      // every warp of the group has written its channels
      if (gleader && !(dbg & 2)) {
        tma_store_2d(&tmC, stage_out, ch * kTBM, pt * kTBN + grp * kTCols);
        bulk_commit();
      }
    }
    if (gleader) bulk_wait_all();
    __syncwarp();
  }
  tc_fence_before();
  __syncthreads();
  if (warp == kMmaWarp) {
    tc_fence_after();
    tmem_dealloc(tmem_base, 512);
  }
}

cudaError_t launch_gemm_t(const CUtensorMap& tmX, const CUtensorMap& tmW, const CUtensorMap& tmC,
                          const CUtensorMap& tmR, const GemmTParams& p, int mode, bool clamp, bool s8out, int grid,
                          cudaStream_t stream) {
  const bool res = p.has_res;
  const size_t smem = gemm_t_smem_bytes(p.BK, p.num_kb, p.stages, p.w_res, p.stage_bufs);
  if (smem > (size_t)kTSmemMax || p.stages > 8) return cudaErrorInvalidValue;
  int dev = 0;
  cudaGetDevice(&dev);
#define QNN_GT(M_, C_, S_, R_)                                                                             \
  if (mode == M_ && clamp == C_ && s8out == S_ && res == R_) {                                             \
    auto kern = qnn_gemm_t_kernel<M_, C_, S_, R_>;                                                         \
    static int attr_done[64] = {0};   /* per device: a process may drive several GPUs */                  \
    if (dev >= 64 || !attr_done[dev]) {                                                                    \
      cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, kTSmemMax);  \
      if (e != cudaSuccess) return e;                                                                      \
      if (dev < 64) attr_done[dev] = 1;                                                                    \
    }                                                                                                      \
    kern<<<grid, kTThreads, smem, stream>>>(tmX, tmW, tmC, tmR, p);                                        \
    count_launch();                                                                                        \
    const cudaError_t e = cudaGetLastError();                                                              \
    if (e != cudaSuccess && std::getenv("QNN_PLAN_TRACE"))                                                 \
      std::fprintf(stderr, "[qnn gemm_t] launch failed: %s\n", cudaGetErrorString(e));                    \
    return e;                                                                                              \
  }
#define QNN_GT_R(M_, C_, S_) QNN_GT(M_, C_, S_, false) QNN_GT(M_, C_, S_, true)
  QNN_GT_R(0, false, false) QNN_GT_R(0, false, true) QNN_GT_R(0, true, false) QNN_GT_R(0, true, true)
  QNN_GT_R(1, false, false) QNN_GT_R(1, false, true) QNN_GT_R(1, true, false) QNN_GT_R(1, true, true)
#undef QNN_GT_R
#undef QNN_GT
  return cudaErrorInvalidValue;
}

}  // namespace qnn
