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
#include <algorithm>
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

// CTA 0 event timestamps (instrumented builds): slot ranges per role, 64 tiles each
//   0: producer issue, 64: builder start (after its waits), 128: builder done, 192: MMA start,
//   256: MMA commit, 320: epilogue tfull wake (warp 0), 384: epilogue store issued (warp 0)
__device__ __forceinline__ void t_trace(const unsigned long long* tr, int slot, int it) {
  if (kTInstrument && tr && blockIdx.x == 0 && it < 64) const_cast<unsigned long long*>(tr)[slot + it] = clock64();
}

constexpr int kTEpiWarps = 16;
constexpr int kTThreads = 32 * kTEpiWarps + 64;
constexpr int kTBM = 128;   // output channels per tile (MMA M)
constexpr int kTBN = kGemmTBN;          // pixels per tile (MMA N), internal.h
constexpr int kTNacc = 512 / kTBN;      // TMEM accumulator buffers (512 columns)
// epilogue: warp (quad, grp) reads its quad's 32 TMEM lanes and pixel columns [grp * kTCols,
// +kTCols) of every tile (a variant with two warp sets taking alternate tiles, 128 columns
// per warp, measured 10-20% slower)
constexpr int kTCols = kTBN / 4;        // pixel columns per epilogue warp (4 column groups)
// output staging, per column group (the 4 warps of one group of pixel columns share it):
// [kTCols pixels][128 channels] in the TMA 128-B swizzle (16-B chunk c of row r at chunk
// c ^ (r % 8)), one TMA store of 128-B rows per group and tile; 1 or 2 buffers (host choice)
#ifdef QNN_T_SPIN
#define QNN_T_WAIT mbar_wait_spin
#else
#define QNN_T_WAIT mbar_wait
#endif
#ifdef QNN_T_EPI_SPIN
#define QNN_TEPI_WAIT mbar_wait_spin
#else
#define QNN_TEPI_WAIT QNN_EPI_WAIT
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

__device__ __forceinline__ void tma_load_4d_t(void* dst, const void* desc, uint64_t* bar, int c0, int c1, int c2,
                                              int c3) {
  asm volatile(
      "cp.async.bulk.tensor.4d.shared::cluster.global.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%3, %4, %5, %6}], [%2];" ::"r"(smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(desc)), "r"(smem_u32(bar)), "r"(c0), "r"(c1), "r"(c2), "r"(c3)
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
  // fused residual (reading R19), UPWARD fast form: R((r - zp_r) * M_r / 2^(32 + rt)) =
  // hi32((r - zp_r) * M_r + rk) >> rt with rk = 2^(rt - 1) * 2^32 (|r - zp_r| <= 255)
  int32_t rkh, rt;   // rk = rkh * 2^32
};

template <int MODE, bool FAST>
__device__ __forceinline__ int32_t tq1(const TChan& q, int i, uint32_t acc, int32_t zp_out) {
  if (FAST) return mad_hi64((int32_t)acc, q.M[i], q.k[i]) >> q.t[i];
  const long long z = rq_round(((long long)(int32_t)acc + q.k[i]) * q.M[i], q.t[i], MODE) + zp_out;
  return (int32_t)(z < INT32_MIN ? INT32_MIN : (z > INT32_MAX ? INT32_MAX : z));
}

// 32 of the warp's pixel columns x its quadrant's 32 channels: requantize, (residual), clamp,
// pack 4 channels per word, store into the staging tile [pixel][32 channels]
template <int MODE, bool FAST, bool CLAMP, bool S8OUT, bool RES, bool RESFAST = false>
__device__ __forceinline__ void t_epilogue(const GemmTParams& p, const TChan& q, const uint32_t (&va)[16],
                                           const uint32_t (&vb)[16], uint32_t st0, uint32_t st1, uint32_t rb) {
#pragma unroll
  for (int k = 0; k < 4; ++k) {
#pragma unroll
    for (int e = 0; e < 2; ++e) {
      // pixel column 8k + 2u + e of this 32-column step; channels 4j + i from lanes j, j+8 (va)
      // and j+16, j+24 (vb); the swizzled word address depends on e and the thread only
      const uint32_t a = (e ? st1 : st0) + (uint32_t)(8 * k) * rb;
      int32_t y[4];
      y[0] = tq1<MODE, FAST>(q, 0, va[4 * k + e], p.zp_out);
      y[1] = tq1<MODE, FAST>(q, 1, va[4 * k + 2 + e], p.zp_out);
      y[2] = tq1<MODE, FAST>(q, 2, vb[4 * k + e], p.zp_out);
      y[3] = tq1<MODE, FAST>(q, 3, vb[4 * k + 2 + e], p.zp_out);
      if (RES) {
        const uint32_t rw = lds32(a);
#pragma unroll
        for (int i = 0; i < 4; ++i) {
          if (RESFAST) {
            const uint32_t b = (rw >> (8 * i)) & 0xFFu;
            const int32_t x = (p.res_s8 ? (int32_t)(int8_t)b : (int32_t)b) - p.res_zp;
            y[i] += mad_hi64(x, p.res_M, (long long)q.rkh << 32) >> q.rt;
          } else {
            y[i] += res_term<MODE>(p, rw, i);
          }
        }
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
// carries its weight k-block next to the activation k-block.  build_raw_bytes >= 0: build mode,
// a stage holds all num_kb X' k-blocks of a tile plus its raw input rows (weights resident)
size_t gemm_t_smem_bytes(int BK, int num_kb, int stages, bool w_res, int stage_bufs, int build_raw_bytes,
                         int rstages, int out_rb, int wparts, bool pair) {
  // (wparts = 2: split weights, two weight k-blocks per activation k-block; pair: a CTA of a
  // cta_group::2 pair stages half of each pixel tile)
  const size_t stage = build_raw_bytes >= 0 ? (size_t)num_kb * kTBN * BK
                                            : (size_t)(pair ? kTBN / 2 : kTBN) * BK + (w_res ? 0 : (size_t)kTBM * BK * wparts);
  const size_t raw = build_raw_bytes >= 0 ? (size_t)rstages * build_raw_bytes : 0;
  return 1024 + (size_t)stages * stage + (w_res ? (size_t)num_kb * kTBM * BK * wparts : 0) + raw +
         (size_t)4 * kTCols * out_rb * stage_bufs + 256;
}

int gemm_t_max_stages(int BK, int num_kb, bool w_res, int stage_bufs, int build_raw_bytes, int rstages, int out_rb,
                      int wparts, bool pair) {
  int s = 8;
  while (s > 1 && gemm_t_smem_bytes(BK, num_kb, s, w_res, stage_bufs, build_raw_bytes, rstages, out_rb, wparts, pair) >
                      (size_t)kTSmemMax)
    --s;
  return s;
}

template <int MODE, bool CLAMP, bool S8OUT, bool RES, bool PAIR>
__global__ void __launch_bounds__(kTThreads, 1)
    qnn_gemm_t_kernel(const __grid_constant__ CUtensorMap tmX, const __grid_constant__ CUtensorMap tmW,
                      const __grid_constant__ CUtensorMap tmC, const __grid_constant__ CUtensorMap tmR,
                      const __grid_constant__ GemmTParams p) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = smem_raw + ((1024 - (smem_u32(smem_raw) & 1023)) & 1023);
  const int BK = p.BK, stages = p.stages, num_kb = p.num_kb;
  const bool build = p.build;
  // CTA pair (cta_group::2): the pair's two channel blocks form one M = 256 MMA; each CTA stages
  // half of every pixel tile (rows 128 r, +128) and its own weights; the leader (rank 0) issues
  // the MMAs; the TMA loads of both CTAs complete on the leader's barriers; the commits reach
  // both CTAs' barriers; every epilogue warp frees the accumulator on the leader's barrier
  // (a template parameter: kernels with cta_group::2 instructions must be launched as clusters)
  const bool pair = PAIR && !build;
  const uint32_t prank = pair ? cluster_rank() : 0u;
  const uint32_t x_bytes = (uint32_t)(pair ? kTBN / 2 : kTBN) * BK, w_bytes = (uint32_t)kTBM * BK;
  const bool w_res = p.w_res;
  const int wparts = p.wsplit ? 2 : 1;   // split weights (zp_W folded): two weight k-blocks per k-block
  // X: stages x [256 pixels][BK] (build mode: stages x num_kb x [256 pixels][32], built in smem)
  const size_t x_stage = build ? (size_t)num_kb * x_bytes : (size_t)x_bytes;
  uint8_t* sX = smem;
  uint8_t* sW = sX + (size_t)stages * x_stage;         // num_kb (resident) or stages x [128 channels][BK]
  uint8_t* sRaw = sW + (size_t)(w_res ? num_kb : stages) * w_bytes * wparts;   // build: stages x raw input rows
  uint8_t* sOut = sRaw + (build ? (size_t)p.rstages * p.b_raw_bytes : 0);   // 4 groups x [kTCols px][out_rb]
  const uint32_t out_rb = (uint32_t)p.out_rb;   // staging row bytes: 128, or 64 / 32 when K_out is 64 / 32
  // epilogue warps: the quads holding live channels (all 4, or K_out / 32 in build mode, whose
  // quads 2 and 3 build the X' tiles)
  const int ep_quads = build ? (p.Kout + 31) / 32 : 4;
  // two epilogue sets on alternate tiles: while one set waits on its TMEM loads or barriers the
  // other computes (one set of 16 warps on each tile leaves every SMSP idle at the same points)
  const bool sets2 = !RES && !build && p.esets == 2;
  __shared__ __align__(8) uint64_t full[8], empty[8], tfull[kTNacc], tempty[kTNacc], wfull, rbar[8], rawfull[8],
      rawempty[8];
  __shared__ uint32_t tmem_slot;
  // warp index through a shuffle: provably warp-uniform, so role branches keep their loop state
  // and UMMA / TMA operands in uniform registers (no R2UR per instruction)
  const int warp = __shfl_sync(0xffffffffu, (int)(threadIdx.x >> 5), 0), lane = threadIdx.x & 31;
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
      mbar_init(&full[s], build ? 8 : 1);   // build mode: one arrive per builder warp
      mbar_init(&empty[s], 1);
    }
    for (int s = 0; s < p.rstages; ++s) {
      mbar_init(&rawfull[s], 1);
      mbar_init(&rawempty[s], 8);   // build mode: every builder warp has read the raw rows
    }
    for (int a = 0; a < kTNacc; ++a) {
      mbar_init(&tfull[a], 1);
      // the tile's column groups x live quads (pair: the leader counts both CTAs' warps)
      mbar_init(&tempty[a], (sets2 ? 2 : 4) * ep_quads * (pair ? 2 : 1));
    }
    mbar_init(&wfull, 1);
    for (int g = 0; g < 8; ++g) mbar_init(&rbar[g], 1);   // per (group, staging buffer)
    fence_mbar_init();
  }
  if (warp == kMmaWarp) {
    if (pair)
      tmem_alloc2(&tmem_slot, 512);
    else
      tmem_alloc(&tmem_slot, 512);
  }
  tc_fence_before();
  __syncthreads();
  if (pair) cluster_sync_all();   // both CTAs' barriers initialised before any cross-CTA signal
  tc_fence_after();
  const uint32_t tmem_base = tmem_slot;
  // pair: the leader's barriers as cluster addresses (TMA completions, accumulator releases)
  const uint32_t full_l = pair ? cluster_addr(&full[0], 0) : 0u, wfull_l = pair ? cluster_addr(&wfull, 0) : 0u,
                 tempty_l = pair ? cluster_addr(&tempty[0], 0) : 0u;
  pdl_trigger();                        // the next layer's kernel may launch and run its prologue
  if (warp != kProdWarp) pdl_wait();    // (the producer waits after issuing the resident weights)

  if (warp == kProdWarp) {
    const bool leader = elect_one();
    if (leader && w_res && px_first < npt) {
      // (split weights: part a's num_kb k-blocks, then part b's; pair: both CTAs' weights on the
      // leader's barrier)
      if (prank == 0) mbar_arrive_expect_tx(&wfull, (uint32_t)(num_kb * wparts) * w_bytes * (pair ? 2u : 1u));
      for (int kb = 0; kb < num_kb * wparts; ++kb) {
        if (pair)
          tma_load_2d_pair(sW + (size_t)kb * w_bytes, &tmW, wfull_l, kb * BK, ch * kTBM);
        else
          tma_load_2d(sW + (size_t)kb * w_bytes, &tmW, &wfull, kb * BK, ch * kTBM);
      }
    }
    pdl_wait();   // activations are the previous kernel's output
    int stage = 0;
    uint32_t phase = 0;
    if (build) {
      // per tile: the R input rows of every output row the tile touches, one 4-D box each
      // (zero outside the image; the builders write zp_A there)
      // (raw rows have their own ring of rstages, deeper than the X' ring: the loads run ahead
      // of the builders by rstages tiles)
      const uint32_t bytes = (uint32_t)p.b_nr * num_kb * p.b_rowlen;
      for (int pt = px_first; pt < npt; pt += px_step) {
        const int r_first = (int)fdiv((uint32_t)(pt * kTBN), p.fdQ);
        QNN_T_WAIT(&rawempty[stage], phase ^ 1);
        if (leader) {
          t_trace(p.trace, 0, (pt - px_first) / px_step);
          mbar_arrive_expect_tx(&rawfull[stage], bytes);
          uint8_t* dst = sRaw + (size_t)stage * p.b_raw_bytes;
          for (int k = 0; k < p.b_nr; ++k) {
            const int ri = r_first + k, n = (int)fdiv((uint32_t)ri, p.fdP), pp = ri - n * p.P;
            tma_load_4d_t(dst + (size_t)k * p.b_slot_bytes, &tmX, &rawfull[stage], 0, 0, pp * p.sh - p.pt, n);
          }
        }
        __syncwarp();
        if (++stage == p.rstages) {
          stage = 0;
          phase ^= 1;
        }
      }
    }
    for (int pt = build ? npt : px_first; pt < npt; pt += px_step) {
      for (int kb = 0; kb < num_kb; ++kb) {
        QNN_T_WAIT(&empty[stage], phase ^ 1);
        if (leader && kb == 0) t_trace(p.trace, 0, (pt - px_first) / px_step);
        if (leader && pair) {
          const uint32_t fb = full_l + (uint32_t)stage * 8u;
          if (prank == 0) mbar_arrive_expect_tx(&full[stage], 2u * (x_bytes + (w_res ? 0 : w_bytes * wparts)));
          tma_load_2d_pair(sX + (size_t)stage * x_bytes, &tmX, fb, kb * BK, pt * kTBN + (int)prank * (kTBN / 2));
          if (!w_res) {
            tma_load_2d_pair(sW + (size_t)stage * w_bytes * wparts, &tmW, fb, kb * BK, ch * kTBM);
            if (wparts == 2)
              tma_load_2d_pair(sW + (size_t)stage * w_bytes * 2 + w_bytes, &tmW, fb, (num_kb + kb) * BK, ch * kTBM);
          }
        } else if (leader) {
          mbar_arrive_expect_tx(&full[stage], x_bytes + (w_res ? 0 : w_bytes * wparts));
          tma_load_2d(sX + (size_t)stage * x_bytes, &tmX, &full[stage], kb * BK, pt * kTBN);
          if (!w_res) {
            tma_load_2d(sW + (size_t)stage * w_bytes * wparts, &tmW, &full[stage], kb * BK, ch * kTBM);
            if (wparts == 2)
              tma_load_2d(sW + (size_t)stage * w_bytes * 2 + w_bytes, &tmW, &full[stage], (num_kb + kb) * BK,
                          ch * kTBM);
          }
        }
        __syncwarp();
        if (++stage == stages) {
          stage = 0;
          phase ^= 1;
        }
      }
    }
  } else if (warp == kMmaWarp && prank == 0) {   // (pair: the peer's MMA warp only allocates TMEM)
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
      if (!build && leader) t_trace(p.trace, 64, it);   // (non-build: slot 64 = accumulator free)
      const uint32_t d = tmem_base + (uint32_t)acc * kTBN;
      if (build) {
        // one stage = the whole tile: num_kb X' k-blocks (32 bytes = one K step each)
        QNN_T_WAIT(&full[stage], phase);
        tc_fence_after();
        if (leader) {
          t_trace(p.trace, 192, it);
          const uint64_t xd = xdesc0 + (uint64_t)((stage * x_stage) >> 4);
          for (int kb = 0; kb < num_kb; ++kb) {
            umma_i8(d, wdesc0 + (uint64_t)kb * w16, xd + (uint64_t)kb * x16, idesc, kb != 0);
            if (wparts == 2)   // split weights: part b, num_kb resident blocks on
              umma_i8(d, wdesc0 + (uint64_t)(num_kb + kb) * w16, xd + (uint64_t)kb * x16, idesc, 1u);
          }
          umma_commit(&empty[stage]);
          umma_commit(&tfull[acc]);
          t_trace(p.trace, 256, it);
        }
        __syncwarp();
        if (++stage == stages) {
          stage = 0;
          phase ^= 1;
        }
        continue;
      }
      for (int kb = 0; kb < num_kb; ++kb) {
        QNN_T_WAIT(&full[stage], phase);
        tc_fence_after();
        if (leader && kb == 0) t_trace(p.trace, 192, it);
        if (leader) {
          const uint64_t wd = wdesc0 + (uint64_t)(w_res ? kb : stage * wparts) * w16,
                         xd = xdesc0 + (uint64_t)((stage * x_stage) >> 4);
          // split weights: part b resident num_kb blocks on, or right after part a in the stage
          const uint64_t wsplit16 = wparts == 2 ? (uint64_t)(w_res ? num_kb : 1) * w16 : 0;
          if (pair) {
            for (int k = 0; k < ksteps; ++k) {
              umma_i8_pair(d, wd + 2 * k, xd + 2 * k, idesc, (kb | k) != 0);
              if (wparts == 2) umma_i8_pair(d, wd + wsplit16 + 2 * k, xd + 2 * k, idesc, 1u);
            }
            umma_commit_pair(&empty[stage]);   // both CTAs' producers may refill the stage
          } else {
            if (!(kTInstrument && (p.dbg & 8)))   // (instrumented builds: 8 skips the MMAs)
              for (int k = 0; k < ksteps; ++k) {
                umma_i8(d, wd + 2 * k, xd + 2 * k, idesc, (kb | k) != 0);
                if (wparts == 2) umma_i8(d, wd + wsplit16 + 2 * k, xd + 2 * k, idesc, 1u);
              }
            umma_commit(&empty[stage]);
          }
        }
        __syncwarp();
        if (++stage == stages) {
          stage = 0;
          phase ^= 1;
        }
      }
      if (leader) {
        if (pair)
          umma_commit_pair(&tfull[acc]);   // both CTAs' epilogues
        else
          umma_commit(&tfull[acc]);
        t_trace(p.trace, 256, it);
      }
      __syncwarp();
    }
  } else if (build && (warp & 3) >= 2) {
    // ---------------------------------------------------------------- X' builders (build mode)
    // thread bt (8 warps = 256 threads) owns pixel bt of every tile: for each filter row r the
    // S*C bytes of raw row (p, r) from column q*sw - pl on (zp_A outside the image), in the
    // 32-B swizzle of the UMMA K-major B operand.  Bytes past S*C are left as they come: the
    // packed weights are zero there.
    const int bt = ((warp >> 2) * 2 + ((warp & 3) - 2)) * 32 + lane;
    const int SC = p.b_S * p.b_C, rowlen = p.b_rowlen;
    const uint32_t swz = ((uint32_t)bt >> 2) & 1u;
    const uint32_t fill = p.b_zp4;
    int stage = 0, rstage = 0;
    uint32_t phase = 0, rphase = 0;
    for (int pt = px_first; pt < npt; pt += px_step) {
      const int m0 = pt * kTBN;
      const int r_first = (int)fdiv((uint32_t)m0, p.fdQ);
      const int row = m0 + bt;
      const int ri = (int)fdiv((uint32_t)row, p.fdQ), qq = row - ri * p.Q;
      const int o = (qq * p.b_sw - p.b_pl) * p.b_C;   // window start in the row (may be < 0)
      const int ab = o & ~3;
      const uint32_t sh8 = (uint32_t)(o - ab) * 8u;
      const bool border = o < 0 || o + SC > rowlen;
      uint32_t mk[8];
#pragma unroll
      for (int k = 0; k < 8; ++k) mk[k] = 0xFFFFFFFFu;
      if (border) {
        const int jlo = max(0, -o), jhi = min(SC, rowlen - o);
#pragma unroll
        for (int k = 0; k < 8; ++k) {
          const int l = min(max(jlo - 4 * k, 0), 4), h = min(max(jhi - 4 * k, 0), 4);
          const uint32_t mh = h == 4 ? 0xFFFFFFFFu : ((1u << (8 * h)) - 1u);
          const uint32_t ml = l == 4 ? 0xFFFFFFFFu : ((1u << (8 * l)) - 1u);
          mk[k] = h > l ? (mh & ~ml) : 0u;
        }
      }
      const int h0 = (ri - (int)fdiv((uint32_t)ri, p.fdP) * p.P) * p.sh - p.pt;   // input row of filter row 0
      QNN_EPI_WAIT(&empty[stage], phase ^ 1);
      QNN_EPI_WAIT(&rawfull[rstage], rphase);
      if (bt == 0) t_trace(p.trace, 64, (pt - px_first) / px_step);
      const uint8_t* rp0 = sRaw + (size_t)rstage * p.b_raw_bytes + (size_t)(ri - r_first) * p.b_slot_bytes + ab;
      uint8_t* dA = sX + (size_t)stage * x_stage + (size_t)bt * 32;
      // (measured: software-pipelining the row loads across rows does not help -- the stem is
      // bound by shared-memory bandwidth: raw-row reads, X' writes and the MMA's operand reads)
#pragma unroll 4
      for (int r = 0; r < num_kb; ++r) {
        // 9 aligned words around the window (addresses outside the row only feed masked bytes
        // and stay inside this CTA's shared memory)
        const uint32_t* wp = reinterpret_cast<const uint32_t*>(rp0 + (size_t)r * rowlen);
        uint32_t uw[9];
#pragma unroll
        for (int k = 0; k < 9; ++k) uw[k] = wp[k];
        uint32_t wv[8];
#pragma unroll
        for (int k = 0; k < 8; ++k) wv[k] = __funnelshift_r(uw[k], uw[k + 1], sh8);
        if (border) {
#pragma unroll
          for (int k = 0; k < 8; ++k) wv[k] = (wv[k] & mk[k]) | (fill & ~mk[k]);
        }
        const int hh = h0 + r;
        if (hh < 0 || hh >= p.b_H) {
#pragma unroll
          for (int k = 0; k < 8; ++k) wv[k] = fill;
        }
        uint8_t* rowdst = dA + (size_t)r * x_bytes;
        *reinterpret_cast<uint4*>(rowdst + (swz << 4)) = make_uint4(wv[0], wv[1], wv[2], wv[3]);
        *reinterpret_cast<uint4*>(rowdst + ((swz ^ 1u) << 4)) = make_uint4(wv[4], wv[5], wv[6], wv[7]);
      }
      fence_proxy_async_smem();
      __syncwarp();
      if (lane == 0) {
        if (bt == 0) t_trace(p.trace, 128, (pt - px_first) / px_step);
        mbar_arrive(&full[stage]);
        mbar_arrive(&rawempty[rstage]);
      }
      if (++stage == stages) {
        stage = 0;
        phase ^= 1;
      }
      if (++rstage == p.rstages) {
        rstage = 0;
        rphase ^= 1;
      }
    }
  } else if (warp < kTEpiWarps && (warp & 3) < ep_quads) {
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
    q.rt = 0;
    q.rkh = 0;
    if (RES && MODE == 0 && p.res_rsh >= 33 && p.res_rsh <= 52) {
      q.rt = p.res_rsh - 32;
      q.rkh = 1 << (q.rt - 1);
    }
    const int dbg = kTInstrument ? p.dbg : 0;
    const bool all_fast = __all_sync(0xffffffffu, fast);
    // column group grp shares a [kTCols][out_rb] staging tile (1 or 2 buffers) with the other
    // live quads; its quad-0 lane 0 issues the group's TMA store (and residual load)
    const bool gleader = quad == 0 && lane == 0;
    const int nbufs = p.stage_bufs;
    const uint32_t gbytes = (uint32_t)kTCols * out_rb;   // one group's staging buffer
    uint8_t* const gstage = sOut + (size_t)grp * gbytes * nbufs;
    // this thread's words (pixel rows 2u + e, e = 0/1; channel word 8 quad + j) in the TMA
    // swizzle of out_rb-byte rows: 16-B chunk c of row r sits at chunk c ^ (r / (128 / out_rb))
    // mod (out_rb / 16) -- for the rows 2u + e (+ 8k + 32h) of one store that is 2u + e at
    // 128 B, u at 64 B and u / 2 at 32 B
    const uint32_t ch16 = (uint32_t)(2 * quad + (j >> 2));
    const uint32_t sw0 = out_rb == 128 ? (uint32_t)(2 * u) : (out_rb == 64 ? (uint32_t)u : (uint32_t)(u >> 1));
    const uint32_t sw1 = out_rb == 128 ? (uint32_t)(2 * u + 1) : sw0;
    const uint32_t st_off0 = (uint32_t)(2 * u) * out_rb + ((ch16 ^ sw0) << 4) + (uint32_t)((j & 3) << 2);
    const uint32_t st_off1 = (uint32_t)(2 * u + 1) * out_rb + ((ch16 ^ sw1) << 4) + (uint32_t)((j & 3) << 2);
    if (sets2) {
      // set = grp / 2 takes the tiles it = set (mod 2), i.e. accumulator `set`; its two column
      // groups cover 128 pixels each, as two 64-pixel chunks (staging buffer c when there are two)
      const int set = grp >> 1, sg = grp & 1;
      int it = set;
      for (int pt = px_first + set * px_step; pt < npt; pt += 2 * px_step, it += 2) {
        const int acc = set;
        QNN_TEPI_WAIT(&tfull[acc], (it >> 1) & 1);
        tc_fence_after();
        if ((warp & 7) == 0 && lane == 0) t_trace(p.trace, 320, it);   // (warps 0 / 8: one per set)
#pragma unroll 1
        for (int c = 0; c < 2; ++c) {
          const int colrel = sg * (2 * kTCols) + c * kTCols;
          uint8_t* const stage_out = gstage + (nbufs == 2 ? c * gbytes : 0);
          const uint32_t sbase = smem_u32(stage_out);
          if (gleader) bulk_wait_read_dyn(nbufs - 1);   // the store that last used this buffer has read it
          named_bar_sync(1 + grp, 32 * ep_quads);
          const uint32_t tb = tmem_base + (uint32_t)acc * kTBN + ((uint32_t)(quad * 32) << 16) + (uint32_t)colrel;
          uint32_t va0[16], vb0[16], va1[16], vb1[16];
          if (!(dbg & 16)) {   // (instrumented builds: 16 skips the TMEM loads)
            tmem_ld_16x256b_x4(tb, va0);
            tmem_ld_16x256b_x4(tb + (16u << 16), vb0);
            tmem_ld_16x256b_x4(tb + 32, va1);
            tmem_ld_16x256b_x4(tb + 32 + (16u << 16), vb1);
            tmem_wait16x2(va0, vb0);
            tmem_wait16x2(va1, vb1);
          }
          tc_fence_before();
          __syncwarp();
          if (c == 1 && lane == 0) {   // this warp is done with the accumulator
            if (pair)
              mbar_arrive_cluster(tempty_l + (uint32_t)acc * 8u);
            else
              mbar_arrive(&tempty[acc]);
          }
          if (!quad_live || (dbg & 1)) {   // (instrumented builds: 1 skips the math)
          } else if (all_fast) {
            t_epilogue<MODE, true, CLAMP, S8OUT, false>(p, q, va0, vb0, sbase + st_off0, sbase + st_off1, out_rb);
            t_epilogue<MODE, true, CLAMP, S8OUT, false>(p, q, va1, vb1, sbase + 32 * out_rb + st_off0,
                                                        sbase + 32 * out_rb + st_off1, out_rb);
          } else {
            t_epilogue<MODE, false, CLAMP, S8OUT, false>(p, q, va0, vb0, sbase + st_off0, sbase + st_off1, out_rb);
            t_epilogue<MODE, false, CLAMP, S8OUT, false>(p, q, va1, vb1, sbase + 32 * out_rb + st_off0,
                                                         sbase + 32 * out_rb + st_off1, out_rb);
          }
          fence_proxy_async_smem();
          named_bar_sync(1 + grp, 32 * ep_quads);
          if (gleader && !(dbg & 2)) {   // (instrumented builds: 2 skips the stores)
            tma_store_2d(&tmC, stage_out, ch * kTBM, pt * kTBN + colrel);
            bulk_commit();
          }
        }
        if ((warp & 7) == 0 && lane == 0) t_trace(p.trace, 384, it);
      }
    }
    int it = 0;
    for (int pt = sets2 ? npt : px_first; pt < npt; pt += px_step, ++it) {
      const int acc = it % kTNacc;
      uint8_t* const stage_out = gstage + (nbufs == 2 ? (it & 1) * gbytes : 0);
      const uint32_t sbase = smem_u32(stage_out);
      const int col0 = pt * kTBN + grp * kTCols;
      // RES: the residual tile (this group's pixels x out_rb channels, same swizzle) lands in the
      // staging buffer; each thread reads its four channels' word per pixel and overwrites it.
      // With two buffers it is prefetched one tile ahead (issued while the previous tile
      // computes), else loaded here.
      const int b = nbufs == 2 ? (it & 1) : 0;
      if (gleader) {
        if (RES && nbufs == 2) {
          if (it == 0) {
            mbar_arrive_expect_tx(&rbar[grp * 2], gbytes);
            tma_load_2d(stage_out, &tmR, &rbar[grp * 2], ch * kTBM, col0);
          }
          if (pt + px_step < npt) {   // next tile's residual into the other buffer
            bulk_wait_read<0>();      // the store of tile it-1 has read that buffer
            uint8_t* nb = gstage + (size_t)(b ^ 1) * gbytes;
            mbar_arrive_expect_tx(&rbar[grp * 2 + (b ^ 1)], gbytes);
            tma_load_2d(nb, &tmR, &rbar[grp * 2 + (b ^ 1)], ch * kTBM, (pt + px_step) * kTBN + grp * kTCols);
          }
        } else {
          bulk_wait_read_dyn(nbufs - 1);   // the store that last used this buffer has read it
          if (RES) {
            mbar_arrive_expect_tx(&rbar[grp * 2], gbytes);
            tma_load_2d(stage_out, &tmR, &rbar[grp * 2], ch * kTBM, col0);
          }
        }
      }
      named_bar_sync(1 + grp, 32 * ep_quads);   // the buffer is free for every warp of the group
      QNN_TEPI_WAIT(&tfull[acc], (it / kTNacc) & 1);
      tc_fence_after();
      if (warp == 0 && lane == 0) t_trace(p.trace, 320, it);
      const uint32_t tb = tmem_base + (uint32_t)acc * kTBN + ((uint32_t)(quad * 32) << 16) + (uint32_t)(grp * kTCols);
      if (RES) mbar_wait(&rbar[grp * 2 + b], (uint32_t)(nbufs == 2 ? (it >> 1) & 1 : it & 1));
      // all four TMEM loads in flight at once, one wait, and the accumulator handed back to the
      // MMA warp before any math
      uint32_t va0[16], vb0[16], va1[16], vb1[16];
      if (!(dbg & 16)) {   // (instrumented builds: 16 skips the TMEM loads)
        tmem_ld_16x256b_x4(tb, va0);                         // lanes j, j + 8, columns 0..31
        tmem_ld_16x256b_x4(tb + (16u << 16), vb0);           // lanes j + 16, j + 24
        tmem_ld_16x256b_x4(tb + 32, va1);                    // columns 32..63
        tmem_ld_16x256b_x4(tb + 32 + (16u << 16), vb1);
        tmem_wait16x2(va0, vb0);
        tmem_wait16x2(va1, vb1);
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) {
        if (pair)
          mbar_arrive_cluster(tempty_l + (uint32_t)acc * 8u);
        else
          mbar_arrive(&tempty[acc]);
      }
      // (warp-uniform choice: a per-lane branch would be if-converted and issue both paths)
      if ((dbg & 1) || !quad_live) {
      } else if (all_fast && RES && q.rt > 0) {   // (q.rt is uniform: one per-tensor residual multiplier)
        t_epilogue<MODE, true, CLAMP, S8OUT, RES, true>(p, q, va0, vb0, sbase + st_off0, sbase + st_off1, out_rb);
        t_epilogue<MODE, true, CLAMP, S8OUT, RES, true>(p, q, va1, vb1, sbase + 32 * out_rb + st_off0,
                                                        sbase + 32 * out_rb + st_off1, out_rb);
      } else if (all_fast) {
        t_epilogue<MODE, true, CLAMP, S8OUT, RES>(p, q, va0, vb0, sbase + st_off0, sbase + st_off1, out_rb);
        t_epilogue<MODE, true, CLAMP, S8OUT, RES>(p, q, va1, vb1, sbase + 32 * out_rb + st_off0,
                                                  sbase + 32 * out_rb + st_off1, out_rb);
      } else {
        t_epilogue<MODE, false, CLAMP, S8OUT, RES>(p, q, va0, vb0, sbase + st_off0, sbase + st_off1, out_rb);
        t_epilogue<MODE, false, CLAMP, S8OUT, RES>(p, q, va1, vb1, sbase + 32 * out_rb + st_off0,
                                                   sbase + 32 * out_rb + st_off1, out_rb);
      }
      fence_proxy_async_smem();
      named_bar_sync(1 + grp, 32 * ep_quads);   // every warp of the group has written its channels
      if (gleader && !(dbg & 2)) {
        tma_store_2d(&tmC, stage_out, ch * kTBM, col0);
        bulk_commit();
      }
      if (warp == 0 && lane == 0) t_trace(p.trace, 384, it);
    }
    if (gleader) bulk_wait_all();
    __syncwarp();
  }
  tc_fence_before();
  __syncthreads();
  // (pair: the peer's last TMA completions, commits and releases target this CTA's barriers and
  // TMEM is allocated for the pair, so both CTAs leave together)
  if (pair) cluster_sync_all();
  if (warp == kMmaWarp) {
    tc_fence_after();
    if (pair)
      tmem_dealloc2(tmem_base, 512);
    else
      tmem_dealloc(tmem_base, 512);
  }
}

cudaError_t launch_gemm_t(const CUtensorMap& tmX, const CUtensorMap& tmW, const CUtensorMap& tmC,
                          const CUtensorMap& tmR, const GemmTParams& p, int mode, bool clamp, bool s8out, int grid,
                          cudaStream_t stream) {
  const bool res = p.has_res;
  const bool pair = p.pair != 0 && !p.build;
  const size_t smem = gemm_t_smem_bytes(p.BK, p.num_kb, p.stages, p.w_res, p.stage_bufs,
                                       p.build ? p.b_raw_bytes : -1, p.rstages, p.out_rb, p.wsplit ? 2 : 1, pair);
  if (smem > (size_t)kTSmemMax || p.stages > 8) return cudaErrorInvalidValue;
  int dev = 0;
  cudaGetDevice(&dev);
#define QNN_GT(M_, C_, S_, R_, P_)                                                                         \
  if (mode == M_ && clamp == C_ && s8out == S_ && res == R_ && pair == P_) {                               \
    auto kern = qnn_gemm_t_kernel<M_, C_, S_, R_, P_>;                                                     \
    static int attr_done[64] = {0};   /* per device: a process may drive several GPUs */                  \
    if (dev >= 64 || !attr_done[dev]) {                                                                    \
      cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, kTSmemMax);  \
      if (e != cudaSuccess) return e;                                                                      \
      if (dev < 64) attr_done[dev] = 1;                                                                    \
    }                                                                                                      \
    int g = grid;                                                                                          \
    if (pair) {   /* as many CTAs as pairs can be co-resident (GPCs with odd SM counts) */                  \
      static int maxc[64] = {0};                                                                           \
      static size_t maxc_smem[64] = {0};                                                                   \
      int m = 0;                                                                                           \
      if (dev < 64 && maxc_smem[dev] == smem) {                                                            \
        m = maxc[dev];                                                                                     \
      } else {                                                                                             \
        m = max_active_clusters(kern, dim3(kTThreads), smem, 2);                                           \
        if (dev < 64) { maxc[dev] = m; maxc_smem[dev] = smem; }                                            \
      }                                                                                                    \
      g = std::min(g, 2 * m);                                                                              \
      g -= g % p.num_ch_tiles;                                                                             \
      if (g <= 0) return cudaErrorInvalidValue;                                                            \
    }                                                                                                      \
    cudaError_t e = launch_ex(kern, dim3(g), dim3(kTThreads), smem, stream, pair ? 2 : 1, tmX, tmW, tmC,     \
                              tmR, p);                                                                     \
    count_launch();                                                                                        \
    if (e == cudaSuccess) e = cudaGetLastError();                                                          \
    if (e != cudaSuccess && std::getenv("QNN_PLAN_TRACE"))                                                 \
      std::fprintf(stderr, "[qnn gemm_t] launch failed: %s\n", cudaGetErrorString(e));                    \
    return e;                                                                                              \
  }
#define QNN_GT_P(M_, C_, S_, R_) QNN_GT(M_, C_, S_, R_, false) QNN_GT(M_, C_, S_, R_, true)
#define QNN_GT_R(M_, C_, S_) QNN_GT_P(M_, C_, S_, false) QNN_GT_P(M_, C_, S_, true)
  QNN_GT_R(0, false, false) QNN_GT_R(0, false, true) QNN_GT_R(0, true, false) QNN_GT_R(0, true, true)
  QNN_GT_R(1, false, false) QNN_GT_R(1, false, true) QNN_GT_R(1, true, false) QNN_GT_R(1, true, true)
#undef QNN_GT_R
#undef QNN_GT_P
#undef QNN_GT
  return cudaErrorInvalidValue;
}

}  // namespace qnn
