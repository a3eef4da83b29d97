// gemm_sm100.cuh — tcgen05 int8 implicit-GEMM for qnn.conv2d / qnn.dense (the pixel-major
// kernel template; instantiated by gemm_sm100.cu for plain weights and by gemm_sm100_split.cu
// for split weights, SPLIT = true: W - zp_W[k] in two s8 parts, Term 3 in the contraction).
//
// Computes, for output pixel m and output channel k:
//   acc  = sum_{kb} A_tile(m, kb) . W(k, kb)                    (Term 1, Eq. 3)
//   v    = acc + off[cls(m)][k] - zp_W * rowsum[m]              (Terms 2-4 folded, P:259/P:264;
//                                                                 Term 3; zp padding)
//   out  = clamp(zp_out + R(v * M_k * 2^(shift_k - 31)))        (Eq. 5 fused)
// with u8/s8 x s8/u8 operands on the 5th-generation tensor cores
// (tcgen05.mma.kind::i8, int32 accumulators in TMEM), operands staged by TMA
// (im2col mode for convolutions: zero fill outside the image, corrected by the
// per-border-class offsets), a persistent tile loop, and warp specialisation:
//   warps 0..15 : epilogue (TMEM -> registers -> requantize -> smem -> TMA store)
//   warp 18     : TMA producer (one elected lane issues)
//   warp 19     : MMA issuer (one elected lane issues) and TMEM allocator
// (warps 16 and 17 idle; 640 threads leave 96 registers per thread.)
// The TMEM accumulator is double-buffered (2 x 256 columns) so the epilogue of
// tile i overlaps the MMAs of tile i+1.
//
// Epilogue cost per output (fast path, rsh = 31 - shift in [33, 52], t = rsh - 32):
//   UPWARD: y = hi32((v - rterm)*M + K) >> t,   K = off*M + (2^(t-1) + zp_out*2^t)*2^32
// (one IMAD.WIDE + one SHF).  This equals floor(x*M/2^rsh + 1/2) + zp_out for the
// exact x = v + off - rterm: with x*M = hi*2^32 + lo, 0 <= lo < 2^32,
// floor((hi*2^32 + lo + 2^(rsh-1))/2^rsh) = floor((hi + 2^(t-1))/2^t) because the
// integer hi + 2^(t-1) cannot cross a multiple of 2^t by adding a fraction < 1.
// K is formed from the exact (int64) offset, and int64 arithmetic is modular, so
// the sum is exact whenever x fits in int32 (reading R10).  Saturation to u8/s8
// is done by cvt.pack.sat.  Per-column {M, t} and per-(class, column) K are staged
// once per N-tile in shared memory and read as broadcast LDS.128 (two columns each).
#pragma once
#include <algorithm>

#include "common.cuh"
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

// per-warp output staging for the TMA store, 32 rows x <= 64 B per buffer.  One buffer: the
// next tile's writes wait for the previous store to have read it (a few hundred cycles against
// tile periods of thousands), and the 32 KB saved buys a pipeline stage for the 48-KB-stage
// GEMMs (BK 128 x BN 256 with border classes: 2 -> 3 stages).  QNN_EPI_STAGE_BUFS=2 restores
// double buffering.
#ifndef QNN_EPI_STAGE_BUFS
#define QNN_EPI_STAGE_BUFS 1
#endif
constexpr int kEpiStageBufs = QNN_EPI_STAGE_BUFS;
constexpr int kStageOutBytes = kGemmEpiWarps * 2048 * kEpiStageBufs;
constexpr int kParamBytes = 256 * 8 + 256 * 8;            // per-column {M, t} and c

// per-class offset rows in smem: int64 K (UPWARD) or int32 off (TONEAREST / raw), pitch BN + 4
// entries: rows stay 16-B aligned and consecutive classes start in different banks
static __host__ __device__ inline size_t off_table_bytes(int ncls, int BN) { return (size_t)ncls * (BN + 4) * 8; }

#ifdef QNN_GEMM_INSTRUMENT
constexpr bool kInstrument = true;    // QNN_GEMM_DEBUG knobs and QNN_GEMM_TRACE timestamps compiled in
#else
constexpr bool kInstrument = false;
#endif

__device__ __forceinline__ void tma_load_4d(void* dst, const void* desc, uint64_t* bar, int c0, int c1, int c2,
                                            int c3) {
  asm volatile(
      "cp.async.bulk.tensor.4d.shared::cluster.global.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%3, %4, %5, %6}], [%2];" ::"r"(smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(desc)), "r"(smem_u32(bar)), "r"(c0), "r"(c1), "r"(c2), "r"(c3)
      : "memory");
}

__device__ __forceinline__ void trace_at(unsigned long long* tr, int slot) {
  if (kInstrument && tr && blockIdx.x == 0) tr[slot] = clock64();
}

// One stage's MMAs from a single thread, kept tight: the descriptors advance by constant
// strides (no per-MMA index math or parameter reloads), the K=32 steps of a k-block unrolled.
// Taps (r, s) of an R x S grid: A steps `a_col16` per s and `a_row16` per r, B `b_tap16` per
// tap (the plain k-block sequence is R = 1, S = nk).  The first MMA overwrites the accumulator
// unless `acc`.
// one tcgen05.mma / commit, single CTA or CTA pair (cta_group::2)
template <bool PAIR>
__device__ __forceinline__ void umma_x(uint32_t d, uint64_t a, uint64_t b, uint32_t idesc, uint32_t acc) {
  if (PAIR)
    umma_i8_pair(d, a, b, idesc, acc);
  else
    umma_i8(d, a, b, idesc, acc);
}
template <bool PAIR>
__device__ __forceinline__ void commit_x(uint64_t* bar) {
  if (PAIR)
    umma_commit_pair(bar);
  else
    umma_commit(bar);
}

// an epilogue warp hands the accumulator back (PAIR: on the leader's barrier)
template <bool PAIR>
__device__ __forceinline__ void release_acc(uint64_t* tempty, int acc, uint32_t tempty_l) {
  if (PAIR)
    mbar_arrive_cluster(tempty_l + (uint32_t)acc * 8u);
  else
    mbar_arrive(&tempty[acc]);
}

template <int KS, bool SPLIT, bool PAIR>
__device__ __forceinline__ void issue_mma_ks(uint32_t d, uint64_t ad_row, uint64_t bd, uint32_t idesc, int R, int S,
                                             uint32_t a_row16, uint32_t a_col16, uint32_t b_tap16, uint32_t acc,
                                             uint32_t bsplit16) {
  for (int r = 0; r < R; ++r) {
    uint64_t ad = ad_row;
    for (int s = 0; s < S; ++s) {
#pragma unroll
      for (int k = 0; k < KS; ++k) {
        umma_x<PAIR>(d, ad + 2 * k, bd + 2 * k, idesc, k ? 1u : acc);
        // split weights (zp_W folded): the second s8 part of W - zp_W against the same A
        if (SPLIT) umma_x<PAIR>(d, ad + 2 * k, bd + bsplit16 + 2 * k, idesc, 1u);
      }
      acc = 1;
      ad += a_col16;
      bd += b_tap16;
    }
    ad_row += a_row16;
  }
}

template <bool SPLIT, bool PAIR>
__device__ __forceinline__ void issue_mma(int ksteps, uint32_t d, uint64_t ad, uint64_t bd, uint32_t idesc, int R,
                                          int S, uint32_t a_row16, uint32_t a_col16, uint32_t b_tap16,
                                          uint32_t acc, uint32_t bsplit16) {
  if (ksteps == 4)
    issue_mma_ks<4, SPLIT, PAIR>(d, ad, bd, idesc, R, S, a_row16, a_col16, b_tap16, acc, bsplit16);
  else if (ksteps == 2)
    issue_mma_ks<2, SPLIT, PAIR>(d, ad, bd, idesc, R, S, a_row16, a_col16, b_tap16, acc, bsplit16);
  else if (ksteps == 1)
    issue_mma_ks<1, SPLIT, PAIR>(d, ad, bd, idesc, R, S, a_row16, a_col16, b_tap16, acc, bsplit16);
}

template <int MODE, bool HAS_CLS, bool CLAMP, bool S8OUT, bool RES, bool SPLIT, bool PAIR, bool AROWS>
__global__ void __launch_bounds__(kGemmThreads, 1)
    qnn_gemm_i8_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB,
                       const __grid_constant__ CUtensorMap tmC0, const __grid_constant__ CUtensorMap tmC1,
                       const __grid_constant__ CUtensorMap tmC2, const __grid_constant__ CUtensorMap tmC3,
                       const __grid_constant__ GemmParams p) {
  extern __shared__ uint8_t smem_raw[];
  // 1024-B aligned base (SW128 atoms); pointer arithmetic on the __shared__ array keeps the address space
  uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  const int BK = p.BK, BN = p.BN, stages = p.stages;
  const int nacc = gemm_acc_bufs(BN), acc_log = nacc == 8 ? 3 : (nacc == 4 ? 2 : 1);
  const uint32_t acc_cols = 512u / nacc;
  // a_build: warps 8..15 build A tiles, warps 0..7 run the epilogue
  const int nepi = p.a_build ? 8 : kGemmEpiWarps;
  const int nsets = p.epi_sets ? p.epi_sets : gemm_epi_sets(BN, p.num_n_tiles, nepi);
  // PAIR (cta_group::2, clusters of 2): the pair's two M tiles form one M = 256 MMA issued by the
  // leader (rank 0); each CTA stages its own A tile and half of the B tile (BN / 2 rows); TMA
  // loads of both CTAs complete on the leader's barriers, commits reach both CTAs, every
  // epilogue warp releases the accumulator on the leader's barrier
  const uint32_t prank = PAIR ? cluster_rank() : 0u;
  const uint32_t a_bytes = kGemmBM * BK, b_bytes = (PAIR ? BN / 2 : BN) * BK;
  const bool b_res = p.b_res;
  // SPLIT: weights packed as W - zp_W[k] in two s8 parts (Term 3 in the contraction), two B
  // k-blocks per A k-block.  A template parameter so the plain kernels carry none of it.
  constexpr int bparts = SPLIT ? 2 : 1;
  const int kps = p.kps;                   // k-blocks per pipeline stage
  uint8_t* sA = smem;
  const size_t a_stage = p.a_stage_bytes ? (size_t)p.a_stage_bytes : (size_t)kps * a_bytes;   // A bytes / stage
  uint8_t* sB = smem + (size_t)stages * a_stage;   // ring of B stages, or the resident B (num_kb blocks)
  uint8_t* sRaw = sB + (b_res ? (size_t)p.num_kb * b_bytes : (size_t)stages * kps * b_bytes) * bparts;   // a_build rows
  uint8_t* sOut = sRaw + (size_t)stages * p.a_raw_bytes;
  const bool tracing = kInstrument && p.trace != nullptr && blockIdx.x == 0;
  const int dbg = kInstrument ? p.dbg : 0;
  int2* sMT = reinterpret_cast<int2*>(sOut + (p.out_staging ? kStageOutBytes : 0));   // {M, t} per column
  int32_t* sCC = reinterpret_cast<int32_t*>(sMT + 256);               // c per column
  int32_t* sOff = sCC + 512;
  const int ncls = HAS_CLS ? p.e.ncls : 1;
  const int offp = BN + 4;
  uint64_t* full = reinterpret_cast<uint64_t*>(reinterpret_cast<uint8_t*>(sOff) + off_table_bytes(ncls, BN));
  uint64_t* empty = full + stages;
  uint64_t* tfull = empty + stages;
  uint64_t* tempty = tfull + 8;
  uint64_t* bres_full = tempty + 8;
  uint64_t* rawfull = bres_full + 1;   // a_build: raw input rows of a stage landed (TMA)
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(rawfull + 8);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  // Warp roles.  The warp scheduler favours higher warp ids, so the latency-critical
  // single-thread roles get the highest ids and are never starved by waiting epilogue warps.
  constexpr int kEpiW = kGemmEpiWarps;        // epilogue warps 0..15
  constexpr int kProdWarp = kGemmRoleBase;      // TMA producer
  constexpr int kMmaWarp = kGemmRoleBase + 1;   // MMA issuer
  constexpr int kAllocWarp = kMmaWarp;        // TMEM allocator (the MMA warp, before its loop)
  if (warp == kProdWarp && lane == 0) {
    tma_prefetch_desc(&tmA);
    tma_prefetch_desc(&tmB);
    if (p.e.tma_store) {
      tma_prefetch_desc(&tmC0);
      tma_prefetch_desc(&tmC1);
      tma_prefetch_desc(&tmC2);
      tma_prefetch_desc(&tmC3);
    }
    for (int s = 0; s < stages; ++s) {
      mbar_init(&full[s], p.a_build ? kEpiW - nepi : 1);   // a_build: one arrive per builder warp
      mbar_init(&empty[s], 1);
    }
    for (int a = 0; a < nacc; ++a) {
      mbar_init(&tfull[a], 1);
      mbar_init(&tempty[a], (nepi / nsets) * (PAIR ? 2 : 1));   // every warp of the set that owns the tile
    }
    mbar_init(bres_full, 1);
    for (int s = 0; s < stages; ++s) mbar_init(&rawfull[s], 1);
    fence_mbar_init();
  }
  if (tracing && threadIdx.x == 0) trace_at(p.trace, 6000);
  if (warp == kAllocWarp) {
    if (PAIR)
      tmem_alloc2(tmem_slot, 512);
    else
      tmem_alloc(tmem_slot, 512);
  }
  tc_fence_before();
  __syncthreads();
  if (PAIR) cluster_sync_all();   // both CTAs' barriers initialised before any cross-CTA signal
  if (tracing && threadIdx.x == 0) trace_at(p.trace, 6001);
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;
  pdl_trigger();                        // the next layer's kernel may launch and run its prologue
  if (warp != kProdWarp) pdl_wait();    // (the producer waits after issuing the resident weights)

  // (PAIR: tiles, CTAs and grid counted in pairs; CTA rank r computes M tile 2 m + r)
  const int num_tiles = (PAIR ? (p.num_m_tiles + 1) >> 1 : p.num_m_tiles) * p.num_n_tiles;
  const int vbx = PAIR ? (int)(blockIdx.x >> 1) : (int)blockIdx.x, vgx = PAIR ? (int)(gridDim.x >> 1) : (int)gridDim.x;
  const uint32_t full_l = PAIR ? cluster_addr(&full[0], 0) : 0u, bres_l = PAIR ? cluster_addr(bres_full, 0) : 0u,
                 tempty_l = PAIR ? cluster_addr(&tempty[0], 0) : 0u;
  // tile t = m_blk * nn + n_blk, visited t = blockIdx.x, += gridDim.x: (m_blk, n_blk) advanced without division
  const int nn = p.num_n_tiles;
  const int m_first = vbx / nn, n_first = vbx - m_first * nn;
  const int m_step = vgx / nn, n_step = vgx - m_step * nn;
#define QNN_NEXT_TILE()  \
  do {                   \
    n_blk += n_step;     \
    m_blk += m_step;     \
    if (n_blk >= nn) {   \
      n_blk -= nn;       \
      ++m_blk;           \
    }                    \
  } while (0)

  if (warp == kProdWarp) {
    // ------------------------------------------------------------ TMA producer
    // The whole warp runs the loop (warp-uniform control flow keeps coordinates and
    // descriptor addresses in uniform registers); one elected lane issues.
    const bool leader = elect_one();
    if (b_res && vbx < num_tiles) {
      // weights are shared by every tile of this CTA: load them once
      if (leader) {
        if (prank == 0) mbar_arrive_expect_tx(bres_full, (uint32_t)(p.num_kb * bparts) * b_bytes * (PAIR ? 2u : 1u));
        // (a CTA keeps one N tile for all its tiles: grid % num_n == 0, see the host plan;
        // split weights: part a's num_kb k-blocks, then part b's)
        for (int kb = 0; kb < p.num_kb * bparts; ++kb) {
          if (PAIR)
            tma_load_2d_pair(sB + kb * b_bytes, &tmB, bres_l, kb * BK, n_first * BN + (int)prank * (BN / 2));
          else
            tma_load_2d(sB + kb * b_bytes, &tmB, bres_full, kb * BK, n_first * BN);
        }
      }
      __syncwarp();
    }
    pdl_wait();   // activations are the previous kernel's output
    int stage = 0, it_p = 0;
    uint32_t phase = 0;
    const bool skip_a = dbg & 4;
    int m_blk = m_first, n_blk = n_first;
    if (AROWS) {
      // one box per (tile, channel chunk): input rows p_first - pt .. + a_nri, columns -pl .. + Wp
      const uint32_t bytes = (uint32_t)(p.a_nri * p.a_Wp * BK);
      for (int t = vbx; t < num_tiles; t += vgx) {
        const int n = (int)fdiv((uint32_t)m_blk, p.fdT), tt = m_blk - n * p.a_T;
        const int p_first = (int)fdiv((uint32_t)(tt * kGemmBM), p.fdWp);
        for (int kc = 0; kc < p.nchunks; ++kc) {
          if (tracing && leader && it_p < 256) trace_at(p.trace, 6300 + it_p);
          mbar_wait(&empty[stage], phase ^ 1);
          if (leader) {
            if (tracing && it_p < 2048) trace_at(p.trace, it_p);
            mbar_arrive_expect_tx(&full[stage], bytes);
            tma_load_4d(sA + (size_t)stage * a_stage, &tmA, &full[stage], kc * BK, -p.pl, p_first - p.pt, n);
            if (tracing && it_p < 256) trace_at(p.trace, 6600 + it_p);
          }
          __syncwarp();
          ++it_p;
          if (++stage == stages) {
            stage = 0;
            phase ^= 1;
          }
        }
        QNN_NEXT_TILE();
      }
    }
    if (p.a_build) {
      // raw input rows for the builders: per output row the tile touches, its R filter rows
      // (zero outside the image: TMA OOB fill), one 4-D box each
      const uint32_t bytes = (uint32_t)p.a_nr * p.num_kb * p.a_rowlen;
      for (int t = vbx; t < num_tiles; t += vgx) {
        const int r_first = (m_blk * kGemmBM) / p.Q;
        mbar_wait(&empty[stage], phase ^ 1);
        if (leader) {
          mbar_arrive_expect_tx(&rawfull[stage], bytes);
          uint8_t* dst = sRaw + (size_t)stage * p.a_raw_bytes;
          for (int k = 0; k < p.a_nr; ++k) {
            const int ri = r_first + k, n = ri / p.P, pp = ri - n * p.P;
            tma_load_4d(dst + (size_t)k * p.a_slot_bytes, &tmA, &rawfull[stage], 0, 0, pp * p.sh - p.pt, n);
          }
        }
        __syncwarp();
        if (++stage == stages) {
          stage = 0;
          phase ^= 1;
        }
        QNN_NEXT_TILE();
      }
    }
    for (int t = (p.a_build || AROWS) ? num_tiles : vbx; t < num_tiles; t += vgx) {   // done above
      const int m0 = (PAIR ? 2 * m_blk + (int)prank : m_blk) * kGemmBM;   // (PAIR: this CTA's M tile)
      int an = 0, ah = 0, aw = 0;
      if (p.im2col) {
        const int pq = p.P * p.Q;
        const int n0 = m0 / pq, rem = m0 - n0 * pq;
        const int p0 = rem / p.Q, q0 = rem - p0 * p.Q;
        an = n0;
        ah = p0 * p.sh - p.pt;
        aw = q0 * p.sw - p.pl;
      }
      // (filter row, filter col, channel chunk) of the next k-block, advanced by counters
      int kr = 0, ks = 0, kc = 0;
      for (int kb0 = 0; kb0 < p.num_kb; kb0 += kps) {
        const int nk = min(kps, p.num_kb - kb0);
        if (tracing && leader && it_p < 256) trace_at(p.trace, 6300 + it_p);
        mbar_wait(&empty[stage], phase ^ 1);
        if (leader) {
          if (tracing && it_p < 2048) trace_at(p.trace, it_p);
          if (prank == 0)   // (PAIR: the leader's barrier counts both CTAs' bytes)
            mbar_arrive_expect_tx(&full[stage], (uint32_t)nk * ((b_res ? 0 : b_bytes * bparts) + (skip_a ? 0 : a_bytes)) *
                                                    (PAIR ? 2u : 1u));
          const uint32_t fb = full_l + (uint32_t)stage * 8u;
          uint8_t* dA = sA + (size_t)stage * a_stage;
          uint8_t* dB = sB + (size_t)(stage * kps) * b_bytes * bparts;
          for (int t2 = 0; t2 < nk; ++t2, dA += a_bytes, dB += b_bytes * bparts) {
            const int kb = kb0 + t2;
            if (skip_a) {
            } else if (p.im2col) {
              if (PAIR)
                tma_load_im2col_4d_pair(dA, &tmA, fb, kc * BK, aw, ah, an, (uint16_t)(ks * p.dil_w),
                                        (uint16_t)(kr * p.dil_h));
              else
                tma_load_im2col_4d(dA, &tmA, &full[stage], kc * BK, aw, ah, an, (uint16_t)(ks * p.dil_w),
                                   (uint16_t)(kr * p.dil_h));
            } else {
              if (PAIR)
                tma_load_2d_pair(dA, &tmA, fb, kb * BK, m0);
              else
                tma_load_2d(dA, &tmA, &full[stage], kb * BK, m0);
            }
            if (!b_res) {
              if (PAIR) {
                tma_load_2d_pair(dB, &tmB, fb, kb * BK, n_blk * BN + (int)prank * (BN / 2));
              } else {
                tma_load_2d(dB, &tmB, &full[stage], kb * BK, n_blk * BN);
                if (SPLIT) tma_load_2d(dB + b_bytes, &tmB, &full[stage], (p.num_kb + kb) * BK, n_blk * BN);
              }
            }
            if (++kc == p.nchunks) {
              kc = 0;
              if (++ks == p.S) {
                ks = 0;
                ++kr;
              }
            }
          }
          if (tracing && it_p < 256) trace_at(p.trace, 6600 + it_p);
        }
        __syncwarp();
        ++it_p;
        if (++stage == stages) {
          stage = 0;
          phase ^= 1;
        }
      }
      QNN_NEXT_TILE();
    }
  } else if (p.a_build && warp >= nepi && warp < kEpiW) {
    // ------------------------------------------------------------ A-tile builders
    // Item (pixel mi, filter row r) of a tile: row mi of k-block r = X'[n, p*sh + r*dil_h - pt,
    // q, 0..32) for output pixel m0 + mi = (n, p, q): the S*C bytes of raw row (p, r) from
    // column q*sw - pl on (zero outside the row), in the 32-B swizzle of the UMMA descriptor.
    // Bytes past S*C are left as they come: the packed weights are zero there.  The raw rows
    // are in shared memory (TMA, see the producer): [output-row slot][r][W*C bytes].
    // 8 builder warps = 256 threads: thread bt owns pixel bt % 128 and the filter rows
    // r = bt / 128, +2, +4, ... (pixel decode once per tile)
    const int bt = (warp - nepi) * 32 + lane;
    const int mi = bt & (kGemmBM - 1), r0 = bt >> 7;
    const int SC = p.a_S * p.a_C;
    const int rowlen = p.a_rowlen;
    const uint32_t swz = ((uint32_t)mi >> 2) & 1u;   // 32-B swizzle of this row
    int stage = 0;
    uint32_t phase = 0;
    int m_blk = m_first, n_blk = n_first;
    for (int t = vbx; t < num_tiles; t += vgx) {
      const int m0 = m_blk * kGemmBM;
      const int r_first = (int)fdiv((uint32_t)m0, p.fdQ);
      const int row = m0 + mi;
      const int ri = (int)fdiv((uint32_t)row, p.fdQ), qq = row - ri * p.Q;
      const int o = (qq * p.a_sw - p.a_pl) * p.a_C;   // window start in the row (may be < 0)
      const int ab = o & ~3;
      const uint32_t sh8 = (uint32_t)(o - ab) * 8u;
      const bool border = o < 0 || o + SC > rowlen;
      // byte masks of the 8 window words (bytes outside the row take the fill): computed only
      // for the few border pixels (hoisted for every pixel, they cost ~150 instructions per tile)
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
      // a_zpfill: output row p of this pixel, for the filter rows that fall outside the image
      const int h0 = p.a_zpfill ? ((ri - (int)fdiv((uint32_t)ri, p.fdP) * p.P) * p.sh - p.pt) : 0;
      const uint32_t fill = p.a_zpfill ? p.a_zp4 : 0u;
      QNN_EPI_WAIT(&empty[stage], phase ^ 1);
      QNN_EPI_WAIT(&rawfull[stage], phase);
      const uint8_t* rp0 = sRaw + (size_t)stage * p.a_raw_bytes + (size_t)(ri - r_first) * p.a_slot_bytes + ab;
      uint8_t* dA = sA + (size_t)stage * a_stage + (size_t)mi * 32;
      for (int r = r0; r < p.num_kb; r += 2) {
        // 9 aligned words around the window (addresses outside the row only feed masked bytes
        // and stay inside this CTA's shared memory); bytes past S*C are left as they come:
        // the packed weights are zero there
        const uint32_t* wp = reinterpret_cast<const uint32_t*>(rp0 + (size_t)r * rowlen);
        uint32_t u[9];
#pragma unroll
        for (int k = 0; k < 9; ++k) u[k] = wp[k];
        uint32_t wv[8];
#pragma unroll
        for (int k = 0; k < 8; ++k) wv[k] = __funnelshift_r(u[k], u[k + 1], sh8);
        if (border) {
#pragma unroll
          for (int k = 0; k < 8; ++k) wv[k] = (wv[k] & mk[k]) | (fill & ~mk[k]);
        }
        if (p.a_zpfill) {
          const int hh = h0 + r * p.dil_h;
          if (hh < 0 || hh >= p.a_H) {
#pragma unroll
            for (int k = 0; k < 8; ++k) wv[k] = fill;
          }
        }
        uint8_t* rowdst = dA + (size_t)r * a_bytes;
        *reinterpret_cast<uint4*>(rowdst + (swz << 4)) = make_uint4(wv[0], wv[1], wv[2], wv[3]);
        *reinterpret_cast<uint4*>(rowdst + ((swz ^ 1u) << 4)) = make_uint4(wv[4], wv[5], wv[6], wv[7]);
      }
      fence_proxy_async_smem();
      __syncwarp();
      if (lane == 0) mbar_arrive(&full[stage]);
      if (++stage == stages) {
        stage = 0;
        phase ^= 1;
      }
      QNN_NEXT_TILE();
    }
  } else if (warp == kMmaWarp && prank == 0) {   // (PAIR: the peer's MMA warp only allocates TMEM)
    // ------------------------------------------------------------ MMA issuer
    // Warp-uniform loop; the elected lane issues every tcgen05.mma and its commits.
    const bool leader = elect_one();
    int stage = 0, it_m = 0;
    uint32_t phase = 0;
    int it = 0;
    const uint64_t adesc0 = make_sdesc(smem_u32(sA), BK);
    const uint64_t bdesc0 = make_sdesc(smem_u32(sB), BK);
    const int ksteps = (dbg & 8) ? 0 : BK / 32;
    // loop-invariant issue parameters in registers (tight issue loops: see issue_mma)
    const uint32_t idesc = p.idesc;
    constexpr bool a_rows = AROWS;
    const int nchunks = p.nchunks, num_kb = p.num_kb;
    const int S_taps = a_rows ? p.S : 1, R_taps = a_rows ? num_kb / (p.S * nchunks) : 1;
    const uint32_t a_col16 = (uint32_t)BK >> 4, a_row16 = (uint32_t)(p.a_Wp * BK) >> 4;
    const uint32_t b_tap16 = (uint32_t)(nchunks * b_bytes) >> 4;
    // split weights: part b sits num_kb k-blocks after part a when resident, right after it
    // (interleaved per k-block) when streamed
    const uint32_t bsplit16 = SPLIT ? (b_res ? ((uint32_t)num_kb * b_bytes) >> 4 : b_bytes >> 4) : 0u;
    if (b_res) mbar_wait(bres_full, 0);
    for (int t = vbx; t < num_tiles; t += vgx, ++it) {
      const int acc = it & (nacc - 1);
      const uint32_t acc_phase = (it >> acc_log) & 1;
      if (tracing && leader && it < 100) trace_at(p.trace, 7200 + it);
      mbar_wait(&tempty[acc], acc_phase ^ 1);
      if (tracing && leader && it < 100) trace_at(p.trace, 7300 + it);
      tc_fence_after();
      const uint32_t d_tmem = tmem_base + acc * acc_cols;
      if (a_rows) {
        // tap (r, s) of channel chunk kc: A starts (r*Wp + s) pixels into the staged input rows
        const int n = (int)fdiv((uint32_t)t, p.fdT), tt = t - n * p.a_T;   // num_n == 1 (resident B)
        const int p_first = (int)fdiv((uint32_t)(tt * kGemmBM), p.fdWp);
        const int off0 = tt * kGemmBM - p_first * p.a_Wp;
        for (int kc = 0; kc < nchunks; ++kc) {
          if (tracing && leader && it_m < 256) trace_at(p.trace, 6900 + it_m);
          mbar_wait(&full[stage], phase);
          tc_fence_after();
          if (leader) {
            if (tracing && it_m < 2048) trace_at(p.trace, 2048 + it_m);
            const uint64_t ad = adesc0 + (((uint32_t)(stage * a_stage) + (uint32_t)(off0 * BK)) >> 4);
            const uint64_t bd = bdesc0 + (((uint32_t)kc * b_bytes) >> 4);
            issue_mma<SPLIT, PAIR>(ksteps, d_tmem, ad, bd, idesc, R_taps, S_taps, a_row16, a_col16, b_tap16, kc != 0,
                                   bsplit16);
            if (tracing && it_m < 64) trace_at(p.trace, 6100 + it_m);   // all MMAs of the stage issued
            commit_x<PAIR>(&empty[stage]);
          }
          __syncwarp();
          ++it_m;
          if (++stage == stages) {
            stage = 0;
            phase ^= 1;
          }
        }
      }
      for (int kb0 = 0; kb0 < (a_rows ? 0 : num_kb); kb0 += kps) {
        const int nk = min(kps, num_kb - kb0);
        if (tracing && leader && it_m < 256) trace_at(p.trace, 6900 + it_m);
        mbar_wait(&full[stage], phase);
        tc_fence_after();
        if (leader) {
          if (tracing && it_m < 2048) trace_at(p.trace, 2048 + it_m);
          // descriptors advance by (byte offset >> 4) in the start-address field
          const uint64_t ad = adesc0 + (((uint32_t)(stage * a_stage)) >> 4);
          const uint64_t bd = bdesc0 + (((uint32_t)(b_res ? kb0 : stage * kps * bparts) * b_bytes) >> 4);
          issue_mma<SPLIT, PAIR>(ksteps, d_tmem, ad, bd, idesc, 1, nk, 0, a_bytes >> 4, (b_bytes * (b_res ? 1 : bparts)) >> 4,
                           kb0 != 0, bsplit16);
          commit_x<PAIR>(&empty[stage]);
        }
        __syncwarp();
        ++it_m;
        if (++stage == stages) {
          stage = 0;
          phase ^= 1;
        }
      }
      if (leader) commit_x<PAIR>(&tfull[acc]);   // (PAIR: both CTAs' epilogues)
      if (tracing && leader && it < 100) trace_at(p.trace, 7400 + it);
      __syncwarp();
    }
  } else if (warp < nepi) {
    // ------------------------------------------------------------ epilogue
    // 16 warps in nsets sets taking alternate tiles; within a set, warp w reads TMEM lanes
    // [32*(w%4), +32) (its quad of rows) and the contiguous chunk range of its column
    // group; one lane = one output row.
    const GemmEpilogue& e = p.e;
    const int et = threadIdx.x;
    const int ew = warp;
    const int quad = warp & 3;
    const int wps = nepi / nsets;                 // warps per set
    const int set = ew / wps;
    const int ngrp = wps >> 2;                    // column groups per set
    const int grp = (ew - set * wps) >> 2;
    const int nchunk = BN >> 5;
    const int c_begin = (grp * nchunk) / ngrp, c_end = ((grp + 1) * nchunk) / ngrp;
    const int pq = p.P * p.Q;
    const int32_t zp_out = e.zp_out, lo = e.lo, hi = e.hi;
    constexpr bool out8 = MODE != 2;   // requantize => 8-bit output, raw => int32 (abi guarantees it)
    const bool tma_st = e.tma_store;
    uint8_t* stage_base = sOut + ew * 2048 * kEpiStageBufs;
    int sbuf = 0;
    // staging row pitch = this group's column bytes; swizzle matches the store box (none for 96 B rows)
    const int row_bytes = (c_end - c_begin) * 32;
    const uint32_t swz_mask = row_bytes == 128 ? 7u : (row_bytes == 64 ? 3u : (row_bytes == 32 ? 1u : 0u));
    const CUtensorMap* tmC = grp == 0 ? &tmC0 : (grp == 1 ? &tmC1 : (grp == 2 ? &tmC2 : &tmC3));
    const int kEpiThreads = 32 * nepi;
    int cur_n = -1, tile_fast = 1;
    const bool has_rt = e.rowsum != nullptr;
    constexpr bool has_res = RES && MODE != 2;   // fused residual add: its own instantiation
    ResTerm rt_res{e.res_M, e.res_rsh, e.res_zp, MODE, e.res_s8};
    int m_blk = m_first, n_blk = n_first;
    if (nsets > 1) {   // single N tile: tile t is (t, 0)
      m_blk = vbx + set * vgx;
      n_blk = 0;
    }
    // the first N tile's parameters are staged before the loop by all 16 warps (a set may own
    // no tile at all); later N-tile changes only happen with one set, where all warps see them
    for (int t = vbx + set * vgx, it = set, first = 1; t < num_tiles || first;
         t += nsets * vgx, it += nsets, first = 0) {
      if (nsets > 1) m_blk = t;   // (several sets: single N tile, tile t is (t, 0); not carried)
      const int acc = it & (nacc - 1);
      const uint32_t acc_phase = (it >> acc_log) & 1;
      if (first || n_blk != cur_n) {
        const int nb = first ? n_first : n_blk;
        // stage this N-tile's per-column parameters (all epilogue warps)
        named_bar_sync(1, kEpiThreads);
        int ok = 1;
        for (int i = et; i < BN; i += kEpiThreads) {
          const int k = nb * BN + i;
          int32_t M = 0, c = 0, tt = 0;
          if (MODE != 2) {
            const int32_t r = e.rsh[k];
            M = e.mult[k];
            if (r >= 33 && r <= 52) {
              tt = r - 32;
              c = MODE == 0 ? (int32_t)((1u << (tt - 1)) + (uint32_t)zp_out * (1u << tt)) : (int32_t)(1u << (tt - 1));
            } else {
              tt = -r;  // generic 64-bit path
              ok = 0;
            }
          }
          sMT[i] = make_int2(M, tt);
          sCC[i] = c;
        }
        if (MODE == 0) {
          // K[cls][j] = off64*M + c*2^32 (modular int64), fast columns only
          long long* sK = reinterpret_cast<long long*>(sOff);
          for (int i = et; i < ncls * BN; i += kEpiThreads) {
            const int c = i / BN, j = i - c * BN;
            const int k = nb * BN + j;
            const int32_t r = e.rsh[k];
            unsigned long long K = 0;
            if (r >= 33 && r <= 52) {
              const int tt = r - 32;
              const unsigned long long c64 =
                  (1ull << (tt - 1)) + ((unsigned long long)(long long)zp_out << tt);
              K = (unsigned long long)e.off64[(size_t)c * e.Kpad + k] * (unsigned long long)(long long)e.mult[k] +
                  (c64 << 32);
            }
            sK[c * offp + j] = (long long)K;
          }
        } else {
          for (int i = et; i < ncls * BN; i += kEpiThreads) {
            const int c = i / BN, j = i - c * BN;
            sOff[c * offp + j] = e.off[(size_t)c * e.Kpad + nb * BN + j];
          }
        }
        tile_fast = named_bar_and(1, kEpiThreads, ok);
        cur_n = nb;
        if (t >= num_tiles) break;   // staged for the other sets only
      }
      const int row0 = (PAIR ? 2 * m_blk + (int)prank : m_blk) * kGemmBM + quad * 32;
      int row = row0 + lane;
      bool row_ok = row < p.M;
      int cls = 0;
      int32_t rterm = 0;
      if (AROWS) {
        // flattened (p, q) with pitch Wp per image: q >= Q (and rows past P) are discarded
        const int n = (int)fdiv((uint32_t)m_blk, p.fdT), tt = m_blk - n * p.a_T;
        const int f = tt * kGemmBM + quad * 32 + lane;
        const int pp = (int)fdiv((uint32_t)f, p.fdWp), qq = f - pp * p.a_Wp;
        row_ok = qq < p.Q && pp < p.P;
        row = (n * p.P + pp) * p.Q + qq;
        if (row_ok) {
          if (HAS_CLS) cls = (int)e.rowcls[pp] * e.ncc + (int)e.colcls[qq];
          if (has_rt) rterm = (int32_t)((uint32_t)e.zpW * (uint32_t)e.rowsum[row]);
        }
      } else if (row_ok) {
        if (HAS_CLS) {
          const int rem = row - (int)fdiv((uint32_t)row, p.fdPQ) * pq;
          const int pp = (int)fdiv((uint32_t)rem, p.fdQ), qq = rem - pp * p.Q;
          cls = (int)e.rowcls[pp] * e.ncc + (int)e.colcls[qq];
        }
        if (has_rt) rterm = (int32_t)((uint32_t)e.zpW * (uint32_t)e.rowsum[row]);
      }
      uint8_t* stage_out = stage_base + sbuf * 2048;
      if (tracing && warp == 0 && lane == 0 && it < 512) trace_at(p.trace, 4096 + it);
      QNN_EPI_WAIT(&tfull[acc], acc_phase);
      if (tracing && warp == 0 && lane == 0 && it < 512) trace_at(p.trace, 5120 + it);
      if (tracing && lane == 0 && it < 100) trace_at(p.trace, 9200 + it * 16 + warp);
      tc_fence_after();
      const uint32_t tbase = tmem_base + acc * acc_cols + ((uint32_t)(quad * 32) << 16);
      // common case (UPWARD fast path, TMA store, two chunks per warp, one epilogue set): both
      // TMEM loads in flight at once and the accumulator released before any math (measured:
      // a gain at BN 256, a 5-10% loss when several sets share the SM)
#ifdef QNN_EPI_NO_TWO
      const bool two = false;
#else
      const bool two = MODE == 0 && nsets == 1 && tile_fast && tma_st && !dbg && c_end - c_begin == 2 && !has_res;
#endif
      if (two) {
        uint32_t va[32], vb[32];
        tmem_ld32_nowait(tbase + c_begin * 32, va);
        tmem_ld32_nowait(tbase + c_begin * 32 + 32, vb);
        tmem_wait32(va);
        tmem_wait32(vb);
        if (tracing && warp == 0 && lane == 0 && it < 500) trace_at(p.trace, 12000 + it * 8 + 0);
        tc_fence_before();
        __syncwarp();
        if (lane == 0) release_acc<PAIR>(tempty, acc, tempty_l);
        if (tracing && lane == 0 && it < 100) trace_at(p.trace, 7500 + it * 16 + warp);
        if (lane == 0) bulk_wait_read<kEpiStageBufs - 1>();
        __syncwarp();
        if (tracing && warp == 0 && lane == 0 && it < 500) trace_at(p.trace, 12000 + it * 8 + 1);
        const long long* kbase = reinterpret_cast<const long long*>(sOff) + cls * offp + c_begin * 32;
        const int4* mt4 = reinterpret_cast<const int4*>(sMT + c_begin * 32);
        uint32_t w[8];
        const uint32_t l16 = (uint32_t)(lane * 64);   // 64-B staging rows, 128-B swizzle atoms
        const uint32_t sw = ((l16 >> 7) & 3u) << 4;
        if (has_rt)
          epi_chunk_up<CLAMP, S8OUT, true>(va, mt4, reinterpret_cast<const longlong2*>(kbase), rterm, lo, hi, w);
        else
          epi_chunk_up<CLAMP, S8OUT, false>(va, mt4, reinterpret_cast<const longlong2*>(kbase), rterm, lo, hi, w);
        *reinterpret_cast<uint4*>(stage_out + (l16 ^ sw)) = make_uint4(w[0], w[1], w[2], w[3]);
        *reinterpret_cast<uint4*>(stage_out + ((l16 + 16) ^ sw)) = make_uint4(w[4], w[5], w[6], w[7]);
        if (tracing && warp == 0 && lane == 0 && it < 500) trace_at(p.trace, 12000 + it * 8 + 2);
        if (has_rt)
          epi_chunk_up<CLAMP, S8OUT, true>(vb, mt4 + 16, reinterpret_cast<const longlong2*>(kbase + 32), rterm, lo,
                                           hi, w);
        else
          epi_chunk_up<CLAMP, S8OUT, false>(vb, mt4 + 16, reinterpret_cast<const longlong2*>(kbase + 32), rterm, lo,
                                            hi, w);
        *reinterpret_cast<uint4*>(stage_out + ((l16 + 32) ^ sw)) = make_uint4(w[0], w[1], w[2], w[3]);
        *reinterpret_cast<uint4*>(stage_out + ((l16 + 48) ^ sw)) = make_uint4(w[4], w[5], w[6], w[7]);
        if (tracing && warp == 0 && lane == 0 && it < 500) trace_at(p.trace, 12000 + it * 8 + 3);
      }
      if (dbg & 32) {   // (instrumented builds) no epilogue work: release the accumulator at once
        tc_fence_before();
        __syncwarp();
        if (lane == 0 && c_begin < c_end) release_acc<PAIR>(tempty, acc, tempty_l);
      }
#pragma unroll 1
      for (int j = (two || (dbg & 32)) ? c_end : c_begin; j < c_end; ++j) {
        uint32_t v[32];
        if (!(dbg & 16)) tmem_load32(tbase + j * 32, v);
        if (j == c_end - 1) {
          // accumulator fully read by this warp: hand the TMEM buffer back to the MMA warp
          tc_fence_before();
          __syncwarp();
          if (lane == 0) release_acc<PAIR>(tempty, acc, tempty_l);
          if (tracing && lane == 0 && it < 100) trace_at(p.trace, 7500 + it * 16 + warp);
        }
        const int k0 = n_blk * BN + j * 32;
        const int4* mt4 = reinterpret_cast<const int4*>(sMT + j * 32);      // 2 columns per int4
        uint32_t w[8];
        int32_t y[out8 ? 1 : 32];
        uint32_t rw[8] = {0, 0, 0, 0, 0, 0, 0, 0};   // residual bytes of this row's 32 columns
        if (has_res && row_ok && k0 < p.Nout) {
          const uint4* rp = reinterpret_cast<const uint4*>(e.res + (long long)row * e.res_pitch + k0);
          const uint4 r0 = __ldg(rp), r1 = __ldg(rp + 1);
          rw[0] = r0.x; rw[1] = r0.y; rw[2] = r0.z; rw[3] = r0.w;
          rw[4] = r1.x; rw[5] = r1.y; rw[6] = r1.z; rw[7] = r1.w;
        }
        if (MODE == 0) {
          if (tile_fast) {
            const longlong2* k2 = reinterpret_cast<const longlong2*>(reinterpret_cast<const long long*>(sOff) +
                                                                     cls * offp + j * 32);
            if (has_res) {
              if (has_rt)
                epi_chunk_up<CLAMP, S8OUT, true, true>(v, mt4, k2, rterm, lo, hi, w, rw, &rt_res);
              else
                epi_chunk_up<CLAMP, S8OUT, false, true>(v, mt4, k2, rterm, lo, hi, w, rw, &rt_res);
            } else if (has_rt) {
              epi_chunk_up<CLAMP, S8OUT, true>(v, mt4, k2, rterm, lo, hi, w);
            } else {
              epi_chunk_up<CLAMP, S8OUT, false>(v, mt4, k2, rterm, lo, hi, w);
            }
          } else {
            // generic 64-bit rounding (shifts outside [33, 52]): int32 offsets straight from global memory
            const int4* off4 = reinterpret_cast<const int4*>(e.off + (size_t)cls * e.Kpad + k0);
            if (has_res)
              epi_chunk<MODE, CLAMP, false, S8OUT, true>(v, off4, mt4, mt4, rterm, zp_out, lo, hi, w, y, rw, &rt_res);
            else
              epi_chunk<MODE, CLAMP, false, S8OUT>(v, off4, mt4, mt4, rterm, zp_out, lo, hi, w, y);
          }
        } else {
          const int4* off4 = reinterpret_cast<const int4*>(sOff + cls * offp + j * 32);
          const int4* c4 = reinterpret_cast<const int4*>(sCC + j * 32);
          if (has_res) {
            if (tile_fast)
              epi_chunk<MODE, CLAMP, true, S8OUT, true>(v, off4, mt4, c4, rterm, zp_out, lo, hi, w, y, rw, &rt_res);
            else
              epi_chunk<MODE, CLAMP, false, S8OUT, true>(v, off4, mt4, c4, rterm, zp_out, lo, hi, w, y, rw,
                                                         &rt_res);
          } else if (tile_fast) {
            epi_chunk<MODE, CLAMP, true, S8OUT>(v, off4, mt4, c4, rterm, zp_out, lo, hi, w, y);
          } else {
            epi_chunk<MODE, CLAMP, false, S8OUT>(v, off4, mt4, c4, rterm, zp_out, lo, hi, w, y);
          }
        }
        if (dbg & 2) {
        } else if constexpr (out8) {
          if (tma_st) {
            if (j == c_begin) {
              // the store issued two tiles ago from this buffer must have finished reading it
              if (lane == 0) bulk_wait_read<kEpiStageBufs - 1>();
              __syncwarp();
            }
            // staged in the TMA swizzle layout of this group's store box
            const uint32_t l16 = (uint32_t)(lane * row_bytes + (j - c_begin) * 32);
            const uint32_t s0 = l16 ^ (((l16 >> 7) & swz_mask) << 4);
            const uint32_t s1 = (l16 + 16) ^ ((((l16 + 16) >> 7) & swz_mask) << 4);
            *reinterpret_cast<uint4*>(stage_out + s0) = make_uint4(w[0], w[1], w[2], w[3]);
            *reinterpret_cast<uint4*>(stage_out + s1) = make_uint4(w[4], w[5], w[6], w[7]);
          } else if (row_ok) {
            uint8_t* o = reinterpret_cast<uint8_t*>(e.out) + (long long)row * e.out_pitch + k0;
            if (k0 + 32 <= p.Nout && ((reinterpret_cast<uintptr_t>(o) & 15) == 0)) {
              *reinterpret_cast<uint4*>(o) = make_uint4(w[0], w[1], w[2], w[3]);
              *reinterpret_cast<uint4*>(o + 16) = make_uint4(w[4], w[5], w[6], w[7]);
            } else {
#pragma unroll
              for (int i = 0; i < 32; ++i)
                if (k0 + i < p.Nout) o[i] = (uint8_t)(w[i >> 2] >> (8 * (i & 3)));
            }
          }
        } else if (row_ok) {
          int32_t* o = reinterpret_cast<int32_t*>(e.out) + (long long)row * e.out_pitch + k0;
          if (k0 + 32 <= p.Nout && ((reinterpret_cast<uintptr_t>(o) & 15) == 0)) {
#pragma unroll
            for (int i = 0; i < 32; i += 4)
              *reinterpret_cast<int4*>(o + i) =
                  make_int4(y[out8 ? 0 : i], y[out8 ? 0 : i + 1], y[out8 ? 0 : i + 2], y[out8 ? 0 : i + 3]);
          } else {
#pragma unroll
            for (int i = 0; i < 32; ++i)
              if (k0 + i < p.Nout) o[i] = y[out8 ? 0 : i];
          }
        }
      }
      if (tma_st && c_begin < c_end && !(dbg & 2)) {
        fence_proxy_async_smem();
        __syncwarp();
        if (lane == 0) {
          tma_store_2d(tmC, stage_out, n_blk * BN + c_begin * 32, row0);
          bulk_commit();
        }
        if (kEpiStageBufs == 2) sbuf ^= 1;
      }
      if (tracing && warp == 0 && lane == 0 && it < 512) trace_at(p.trace, 4608 + it);
      if (tracing && lane == 0 && it < 100) trace_at(p.trace, 10900 + it * 16 + warp);
      if (c_begin == c_end) {  // no columns for this warp: still release the accumulator
        tc_fence_before();
        __syncwarp();
        if (lane == 0) release_acc<PAIR>(tempty, acc, tempty_l);
      }
      if (nsets == 1) QNN_NEXT_TILE();
    }
    if (tma_st && lane == 0) bulk_wait_all();
    __syncwarp();
  }

#undef QNN_NEXT_TILE
  tc_fence_before();
  __syncthreads();
  if (tracing && threadIdx.x == 0) trace_at(p.trace, 6002);
  if (PAIR) cluster_sync_all();   // the peer's last signals target this CTA; TMEM is the pair's
  if (warp == kAllocWarp) {
    tc_fence_after();
    if (PAIR)
      tmem_dealloc2(tmem_base, 512);
    else
      tmem_dealloc(tmem_base, 512);
  }
}

template <int MODE, bool HAS_CLS, bool CLAMP, bool S8OUT, bool RES, bool SPLIT, bool PAIR, bool AROWS>
static cudaError_t launch_variant(const CUtensorMap& tmA, const CUtensorMap& tmB, const CUtensorMap* tmC,
                                  const GemmParams& p, int grid, cudaStream_t stream) {
  static int attr_done[64] = {0};
  int dev = 0;
  cudaGetDevice(&dev);
  auto kern = qnn_gemm_i8_kernel<MODE, HAS_CLS, CLAMP, S8OUT, RES, SPLIT, PAIR, AROWS>;
  if (dev >= 64 || !attr_done[dev]) {
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024);
    if (e != cudaSuccess) return e;
    if (dev < 64) attr_done[dev] = 1;
  }
  constexpr int bparts = SPLIT ? 2 : 1;
  const size_t smem = gemm_smem_bytes(p.BK, p.BN, p.stages, HAS_CLS ? p.e.ncls : 1, p.b_res ? p.num_kb * bparts : 0,
                                      p.kps, p.a_raw_bytes, p.a_stage_bytes, bparts, p.out_staging != 0, PAIR);
  if (smem > 227 * 1024) return cudaErrorInvalidValue;
  if (PAIR) {   // as many CTA pairs as can be co-resident (GPCs with odd SM counts), grid / 2 a multiple of num_n
    static int maxc[64] = {0};
    static size_t maxc_smem[64] = {0};
    int m = 0;
    if (dev < 64 && maxc_smem[dev] == smem) {
      m = maxc[dev];
    } else {
      m = max_active_clusters(kern, dim3(kGemmThreads), smem, 2);
      if (dev < 64) {
        maxc[dev] = m;
        maxc_smem[dev] = smem;
      }
    }
    int pairs = std::min(grid / 2, m);
    pairs -= pairs % p.num_n_tiles;
    if (pairs <= 0) return cudaErrorInvalidValue;
    grid = 2 * pairs;
  }
  cudaError_t e = launch_ex(kern, dim3(grid), dim3(kGemmThreads), smem, stream, PAIR ? 2 : 1, tmA, tmB, tmC[0],
                            tmC[1], tmC[2], tmC[3], p);
  count_launch();
  if (e == cudaSuccess) e = cudaGetLastError();
  static const bool trace_err = std::getenv("QNN_PLAN_TRACE") != nullptr;
  if (e != cudaSuccess && trace_err)
    std::fprintf(stderr, "[qnn gemm] launch failed: %s (grid %d, %d threads, %zu B smem)\n", cudaGetErrorString(e),
                 grid, kGemmThreads, smem);
  return e;
}

// one translation unit per (SPLIT, PAIR, AROWS) variant (gemm_sm100.cu, gemm_sm100_split.cu,
// gemm_sm100_pair.cu, gemm_sm100_arows.cu): compiled in parallel; each kernel carries only its
// own operand-staging path (the 96-register budget: code of another path costs spills)
template <bool SPLIT, bool PAIR, bool AROWS>
static cudaError_t launch_gemm_impl(const CUtensorMap& tmA, const CUtensorMap& tmB, const CUtensorMap* tmC,
                                    const GemmParams& p, int mode, bool clamp, int grid, cudaStream_t stream) {
  const bool cls = p.e.ncls > 1;
  const bool s8 = p.e.out_dtype == DT_S8;
  const bool res = p.e.res != nullptr && mode != 2;
#define QNN_GEMM_CASE(M_, C_, K_, S_, R_)                            \
  if (mode == M_ && cls == C_ && clamp == K_ && s8 == S_ && res == R_) \
    return launch_variant<M_, C_, K_, S_, R_, SPLIT, PAIR, AROWS>(tmA, tmB, tmC, p, grid, stream);
#define QNN_GEMM_CASES(M_, C_, K_)                                                            \
  QNN_GEMM_CASE(M_, C_, K_, false, false) QNN_GEMM_CASE(M_, C_, K_, true, false)              \
  QNN_GEMM_CASE(M_, C_, K_, false, true) QNN_GEMM_CASE(M_, C_, K_, true, true)
  QNN_GEMM_CASES(0, false, false)
  QNN_GEMM_CASES(0, false, true)
  QNN_GEMM_CASES(0, true, false)
  QNN_GEMM_CASES(0, true, true)
  QNN_GEMM_CASES(1, false, false)
  QNN_GEMM_CASES(1, false, true)
  QNN_GEMM_CASES(1, true, false)
  QNN_GEMM_CASES(1, true, true)
  QNN_GEMM_CASE(2, false, false, false, false)
  QNN_GEMM_CASE(2, true, false, false, false)
#undef QNN_GEMM_CASES
#undef QNN_GEMM_CASE
  return cudaErrorInvalidValue;
}

}  // namespace qnn
