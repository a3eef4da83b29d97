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
// output channel and its multiplier / shift / 64-bit constant live in that lane's registers
// for the whole kernel.  Bytes go to a [64 pixels][32 channels] staging tile with one STS.U8
// each and leave by TMA store.
//
// Grid: a multiple of the channel-block count, so a CTA keeps one channel block (weights and
// constants loaded once; weights streamed per stage when the block does not fit); pixel
// tiles advance by grid / blocks.
// Warps: 0-15 epilogue (warp w: TMEM lanes 32*(w%4) = its 32 channels, pixel columns
// 64*(w/4)), 16 TMA producer, 17 MMA issuer + TMEM allocator (2 accumulators x 256 columns).
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

constexpr int kTEpiWarps = 16;
constexpr int kTThreads = 32 * kTEpiWarps + 64;
constexpr int kTBM = 128;   // output channels per tile (MMA M)
constexpr int kTBN = 256;   // pixels per tile (MMA N)
constexpr int kTStageOut = 2048;   // per epilogue warp: 64 pixels x 32 channels

__device__ __forceinline__ void sts_u8(uint32_t addr, uint32_t v) {
  asm volatile("st.shared.u8 [%0], %1;" ::"r"(addr), "r"(v));
}

// two outputs of one channel (pixels j, j+1): clamp, saturate, one byte each into the
// [pixel][channel] staging tile
template <bool CLAMP, bool S8OUT>
__device__ __forceinline__ void store2(uint32_t a, int32_t y0, int32_t y1, int32_t lo, int32_t hi) {
  if (CLAMP) {
    y0 = min(max(y0, lo), hi);
    y1 = min(max(y1, lo), hi);
  }
  uint32_t b2;   // saturated bytes (y0, y1) in the low half-word
  if (S8OUT)
    asm("cvt.pack.sat.s8.s32.b32 %0, %2, %1, 0;" : "=r"(b2) : "r"(y0), "r"(y1));
  else
    asm("cvt.pack.sat.u8.s32.b32 %0, %2, %1, 0;" : "=r"(b2) : "r"(y0), "r"(y1));
  sts_u8(a, b2);
  sts_u8(a + 32, b2 >> 8);
}

__device__ __forceinline__ uint32_t lds_u8(uint32_t addr) {
  uint32_t v;
  asm volatile("ld.shared.u8 %0, [%1];" : "=r"(v) : "r"(addr));
  return v;
}

// the residual byte requantized to the output scale with zero point 0 (reading R19: added
// to the conv's requantized value before the clamp)
template <int MODE>
__device__ __forceinline__ int32_t res_term(const GemmTParams& p, uint32_t b) {
  const int32_t x = (p.res_s8 ? (int32_t)(int8_t)b : (int32_t)b) - p.res_zp;
  return (int32_t)rq_round((int64_t)x * p.res_M, p.res_rsh, MODE);
}

// hi32(v * M + K) (64-bit addend): one IMAD.WIDE
__device__ __forceinline__ int32_t madwide_hi(int32_t v, int32_t M, long long K) {
  long long d;
  asm("mad.wide.s32 %0, %1, %2, %3;" : "=l"(d) : "r"(v), "r"(M), "l"(K));
  return (int32_t)((unsigned long long)d >> 32);
}

}  // namespace

constexpr int kTSmemMax = 227 * 1024 - 1024;   // dynamic budget (the barriers are static)

// w_res: the CTA's weight block stays resident (num_kb blocks); otherwise each pipeline stage
// carries its weight k-block next to the activation k-block
size_t gemm_t_smem_bytes(int BK, int num_kb, int stages, bool w_res) {
  const size_t stage = (size_t)kTBN * BK + (w_res ? 0 : (size_t)kTBM * BK);
  return 1024 + (size_t)stages * stage + (w_res ? (size_t)num_kb * kTBM * BK : 0) +
         (size_t)kTEpiWarps * kTStageOut + 256;
}

int gemm_t_max_stages(int BK, int num_kb, bool w_res) {
  int s = 6;
  while (s > 2 && gemm_t_smem_bytes(BK, num_kb, s, w_res) > (size_t)kTSmemMax) --s;
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
  __shared__ __align__(8) uint64_t full[8], empty[8], tfull[2], tempty[2], wfull, rbar[kTEpiWarps];
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
    for (int a = 0; a < 2; ++a) {
      mbar_init(&tfull[a], 1);
      mbar_init(&tempty[a], kTEpiWarps);
    }
    mbar_init(&wfull, 1);
    for (int w = 0; w < kTEpiWarps; ++w) mbar_init(&rbar[w], 1);
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
        mbar_wait(&empty[stage], phase ^ 1);
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
      const int acc = it & 1;
      mbar_wait(&tempty[acc], ((it >> 1) & 1) ^ 1);
      tc_fence_after();
      const uint32_t d = tmem_base + (uint32_t)acc * kTBN;
      for (int kb = 0; kb < num_kb; ++kb) {
        mbar_wait(&full[stage], phase);
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
    const int k = ch * kTBM + quad * 32 + lane;   // this lane's output channel
    // (K_out = 64: the upper half of the 128-channel block is zero weights; its lanes compute
    // nothing and their stores fall outside the output tensor, which TMA drops)
    const bool quad_live = ch * kTBM + quad * 32 < p.Kout;
    const int kk = k < p.Kout ? k : 0;
    const int32_t M = p.mult[kk], rsh = p.rsh[kk];
    const long long off = p.off64[kk];
    const bool fast = MODE == 0 && rsh >= 33 && rsh <= 52;
    int t = 0;
    long long K = 0;
    if (fast) {
      t = rsh - 32;
      const unsigned long long c64 = (1ull << (t - 1)) + ((unsigned long long)(long long)p.zp_out << t);
      K = (long long)((unsigned long long)off * (unsigned long long)(long long)M + (c64 << 32));
    }
    const bool all_fast = __all_sync(0xffffffffu, fast);
    // 32-bit form of the fast path: with |acc| <= KK * 255 * 255 (any operand dtypes / zps) and
    // |off| below 2^31 minus that bound, acc + off is exact in int32, and since the rounding
    // constant c64 has no bits below 2^32,  hi64((acc + off) * M + c64 * 2^32) = hi32((acc + off) * M) + c64:
    // one IMAD.HI with a 32-bit addend instead of a 64-bit multiply-add with carry.
    const long long acc_bound = (long long)p.num_kb * p.BK * 65025LL;
    const bool fast32 = fast && (off < 0 ? -off : off) < (1LL << 31) - 1 - acc_bound;
    const int32_t off32 = (int32_t)off;
    const int32_t c32 = fast ? (int32_t)((1 << (t - 1)) + p.zp_out * (1 << t)) : 0;
    const bool all_fast32 = __all_sync(0xffffffffu, fast32) && !(p.dbg & 4);
    uint8_t* stage_out = sOut + warp * kTStageOut;
    const uint32_t st_lane = smem_u32(stage_out) + (uint32_t)lane;
    int it = 0;
    for (int pt = px_first; pt < npt; pt += px_step, ++it) {
      const int acc = it & 1;
      if (RES) {
        // the residual tile (this warp's 64 pixels x 32 channels) lands in the staging tile
        // itself; each lane then reads its channel's byte per pixel and overwrites it
        if (lane == 0) {
          bulk_wait_read<0>();   // the previous tile's store has read the staging tile
          if (quad_live) {
            mbar_arrive_expect_tx(&rbar[warp], kTStageOut);
            tma_load_2d(stage_out, &tmR, &rbar[warp], ch * kTBM + quad * 32, pt * kTBN + grp * 64);
          }
        }
        __syncwarp();
      }
      QNN_EPI_WAIT(&tfull[acc], (it >> 1) & 1);
      tc_fence_after();
      const uint32_t tb = tmem_base + (uint32_t)acc * kTBN + ((uint32_t)(quad * 32) << 16) + (uint32_t)(grp * 64);
      uint32_t va[32], vb[32];
      tmem_ld32_nowait(tb, va);
      tmem_ld32_nowait(tb + 32, vb);
      tmem_wait32(va);
      tmem_wait32(vb);
      tc_fence_before();
      __syncwarp();
      if (lane == 0) {
        mbar_arrive(&tempty[acc]);
        if (!RES) bulk_wait_read<0>();   // the previous tile's store has read the staging tile
      }
      __syncwarp();
      if (RES && quad_live) mbar_wait(&rbar[warp], (uint32_t)(it & 1));
      // (warp-uniform choice: a per-lane branch would be if-converted and issue both paths)
      if ((p.dbg & 1) || !quad_live) {
      } else if (all_fast32) {
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          const uint32_t* v = h ? vb : va;
#pragma unroll
          for (int j = 0; j < 32; j += 2) {
            const uint32_t a = st_lane + (uint32_t)((h * 32 + j) * 32);
            int32_t y0 = __mulhi((int32_t)v[j] + off32, M) + c32, y1 = __mulhi((int32_t)v[j + 1] + off32, M) + c32;
            y0 >>= t;
            y1 >>= t;
            if (RES) {
              y0 += res_term<MODE>(p, lds_u8(a));
              y1 += res_term<MODE>(p, lds_u8(a + 32));
            }
            store2<CLAMP, S8OUT>(a, y0, y1, p.lo, p.hi);
          }
        }
      } else if (all_fast) {
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          const uint32_t* v = h ? vb : va;
#pragma unroll
          for (int j = 0; j < 32; j += 2) {
            const uint32_t a = st_lane + (uint32_t)((h * 32 + j) * 32);
            int32_t y0 = madwide_hi((int32_t)v[j], M, K) >> t, y1 = madwide_hi((int32_t)v[j + 1], M, K) >> t;
            if (RES) {
              y0 += res_term<MODE>(p, lds_u8(a));
              y1 += res_term<MODE>(p, lds_u8(a + 32));
            }
            store2<CLAMP, S8OUT>(a, y0, y1, p.lo, p.hi);
          }
        }
      } else {
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          const uint32_t* v = h ? vb : va;
#pragma unroll
          for (int j = 0; j < 32; j += 2) {
            const uint32_t a = st_lane + (uint32_t)((h * 32 + j) * 32);
            int64_t z0, z1;   // exact: requantized value + zp_out (+ residual), clamped below
            if (fast) {
              z0 = (int32_t)(((unsigned long long)((long long)(int32_t)v[j] * M) + (unsigned long long)K) >> 32) >> t;
              z1 = (int32_t)(((unsigned long long)((long long)(int32_t)v[j + 1] * M) + (unsigned long long)K) >> 32) >>
                   t;
            } else {
              z0 = rq_round(((long long)(int32_t)v[j] + off) * M, rsh, MODE) + p.zp_out;
              z1 = rq_round(((long long)(int32_t)v[j + 1] + off) * M, rsh, MODE) + p.zp_out;
            }
            if (RES) {
              z0 += res_term<MODE>(p, lds_u8(a));
              z1 += res_term<MODE>(p, lds_u8(a + 32));
            }
            const int32_t y0 = (int32_t)(z0 < p.lo ? p.lo : (z0 > p.hi ? p.hi : z0));
            const int32_t y1 = (int32_t)(z1 < p.lo ? p.lo : (z1 > p.hi ? p.hi : z1));
            store2<false, S8OUT>(a, y0, y1, p.lo, p.hi);
          }
        }
      }
      fence_proxy_async_smem();
      __syncwarp();
      if (lane == 0 && quad_live && !(p.dbg & 2)) {
        tma_store_2d(&tmC, stage_out, ch * kTBM + quad * 32, pt * kTBN + grp * 64);
        bulk_commit();
      }
      __syncwarp();
    }
    if (lane == 0) bulk_wait_all();
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
  const size_t smem = gemm_t_smem_bytes(p.BK, p.num_kb, p.stages, p.w_res);
  if (smem > (size_t)kTSmemMax || p.stages > 8) return cudaErrorInvalidValue;
#define QNN_GT(M_, C_, S_, R_)                                                                             \
  if (mode == M_ && clamp == C_ && s8out == S_ && res == R_) {                                             \
    auto kern = qnn_gemm_t_kernel<M_, C_, S_, R_>;                                                         \
    static bool attr = false;                                                                              \
    if (!attr) {                                                                                           \
      cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, kTSmemMax);  \
      if (e != cudaSuccess) return e;                                                                      \
      attr = true;                                                                                         \
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
