// gemm_sm100.cu — tcgen05 int8 implicit-GEMM for qnn.conv2d / qnn.dense.
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
//   warp 0      : TMA producer (one elected lane)
//   warp 1      : MMA issuer   (one elected lane)
//   warp 2      : TMEM allocator
//   warps 4..11 : epilogue (TMEM -> registers -> requantize -> smem -> TMA store)
// The TMEM accumulator is double-buffered (2 x 256 columns) so the epilogue of
// tile i overlaps the MMAs of tile i+1.
//
// Epilogue cost per output (fast path, rsh = 31 - shift in [33, 52]):
//   UPWARD: y = (mulhi(v, M) + (2^(t-1) + zp_out*2^t)) >> t,  t = rsh - 32
// which equals floor(v*M/2^rsh + 1/2) + zp_out exactly: writing v*M = hi*2^32 + lo
// with 0 <= lo < 2^32, floor((hi*2^32 + lo + 2^(rsh-1))/2^rsh) =
// floor((hi + 2^(t-1) + lo/2^32)/2^t) = floor((hi + 2^(t-1))/2^t) because the
// integer hi + 2^(t-1) cannot cross a multiple of 2^t by adding a fraction < 1.
// Saturation to u8/s8 is done by cvt.pack.sat.  Per-column (M, c, t, off) are
// staged once per N-tile in shared memory and read as one broadcast LDS.128.
#include "common.cuh"
#include "internal.h"

namespace qnn {

constexpr int kStageOutBytes = kGemmEpiWarps * 2 * 1024;  // per-warp double-buffered 32x32 B staging
constexpr int kParamBytes = 256 * 16;                     // per-column {0, c, M, t}

// per-class offset rows in smem: pitch BN + 4 ints keeps rows 16-B aligned and spreads banks
static __host__ __device__ inline size_t off_table_bytes(int ncls, int BN) { return (size_t)ncls * (BN + 4) * 4; }

size_t gemm_smem_bytes(int BK, int BN, int stages, int ncls) {
  return 1024 + (size_t)stages * ((size_t)kGemmBM * BK + (size_t)BN * BK) + kStageOutBytes + kParamBytes +
         off_table_bytes(ncls, BN) + 256;
}

int gemm_max_stages(int BK, int BN, int ncls) {
  const size_t budget = 227 * 1024;
  int s = 8;
  while (s > 2 && gemm_smem_bytes(BK, BN, s, ncls) > budget) --s;
  return s;
}

__device__ __forceinline__ void named_bar_sync(int id, int n) {
  asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(n) : "memory");
}
__device__ __forceinline__ int named_bar_and(int id, int n, int pred) {
  int r;
  asm volatile(
      "{\n\t.reg .pred p, q;\n\t"
      "setp.ne.s32 q, %3, 0;\n\t"
      "bar.red.and.pred p, %1, %2, q;\n\t"
      "selp.s32 %0, 1, 0, p;\n\t}"
      : "=r"(r)
      : "r"(id), "r"(n), "r"(pred)
      : "memory");
  return r;
}
// TMEM -> registers: 32 lanes x 32 columns, waited in the same asm so no use of
// the registers can be scheduled before the load completes.
__device__ __forceinline__ void tmem_load32(uint32_t taddr, uint32_t (&r)[32]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 "
      "{%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
      "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];\n\t"
      "tcgen05.wait::ld.sync.aligned;"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
        "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15]),
        "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]),
        "=r"(r[23]), "=r"(r[24]), "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]),
        "=r"(r[30]), "=r"(r[31])
      : "r"(taddr));
}
__device__ __forceinline__ uint32_t pack4_u8(int a, int b, int c, int d) {
  uint32_t o;
  asm("{\n\t.reg .u32 t;\n\t"
      "cvt.pack.sat.u8.s32.b32 t, %4, %3, 0;\n\t"
      "cvt.pack.sat.u8.s32.b32 %0, %2, %1, t;\n\t}"
      : "=r"(o)
      : "r"(a), "r"(b), "r"(c), "r"(d));
  return o;
}
__device__ __forceinline__ uint32_t pack4_s8(int a, int b, int c, int d) {
  uint32_t o;
  asm("{\n\t.reg .u32 t;\n\t"
      "cvt.pack.sat.s8.s32.b32 t, %4, %3, 0;\n\t"
      "cvt.pack.sat.s8.s32.b32 %0, %2, %1, t;\n\t}"
      : "=r"(o)
      : "r"(a), "r"(b), "r"(c), "r"(d));
  return o;
}
__device__ __forceinline__ void tma_store_2d(const void* desc, const void* src, int c0, int c1) {
  asm volatile("cp.async.bulk.tensor.2d.global.shared::cta.bulk_group [%0, {%2, %3}], [%1];" ::"l"(
                   reinterpret_cast<uint64_t>(desc)),
               "r"(smem_u32(src)), "r"(c0), "r"(c1)
               : "memory");
}
__device__ __forceinline__ void bulk_commit() { asm volatile("cp.async.bulk.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void bulk_wait_read() {
  asm volatile("cp.async.bulk.wait_group.read %0;" ::"n"(N) : "memory");
}
__device__ __forceinline__ void bulk_wait_all() { asm volatile("cp.async.bulk.wait_group 0;" ::: "memory"); }
__device__ __forceinline__ void fence_proxy_async_smem() {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}

// Requantize 32 accumulators of one row (this lane) against 32 consecutive columns.
// prm[i] = {0, c, M, t}: the (0, c) pair is the 64-bit addend of IMAD.HI, so
// mulhi(v, M) + c is a single instruction.  offc: 32 per-column int32 offsets
// (16-B aligned, read 4 at a time).
template <int MODE, bool CLAMP, bool FAST>
__device__ __forceinline__ void requant_row32(const uint32_t (&acc)[32], const int4* __restrict__ prm,
                                              const int4* __restrict__ offc, int32_t rterm, int32_t zp_out,
                                              int32_t lo, int32_t hi, int32_t (&y)[32]) {
#pragma unroll
  for (int i4 = 0; i4 < 8; ++i4) {
    const int4 o4 = offc[i4];
    const int32_t offs[4] = {o4.x, o4.y, o4.z, o4.w};
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const int i = i4 * 4 + j;
      const int32_t v = (int32_t)(acc[i] + (uint32_t)offs[j] - (uint32_t)rterm);  // wrap-exact (reading R10)
      int32_t r;
      if (MODE == 2) {
        r = v;
      } else {
        const int4 q = prm[i];  // same address across the warp -> broadcast
        if (FAST) {
          if (MODE == 0) {
            r = (__mulhi(v, q.z) + q.y) >> q.w;
          } else {
            const uint32_t a = v < 0 ? (uint32_t)(-(int64_t)v) : (uint32_t)v;
            const int32_t m = (int32_t)((__umulhi(a, (uint32_t)q.z) + (uint32_t)q.y) >> q.w);
            r = (v < 0 ? -m : m) + zp_out;
          }
        } else {
          // generic 64-bit path (tile has a column outside the fast range); q.w holds
          // t = rsh - 32 for fast-range columns and -rsh for the others
          const int rsh = q.w > 0 ? q.w + 32 : -q.w;
          r = (int32_t)(rq_round((int64_t)v * q.z, rsh, MODE) + zp_out);
        }
        if (CLAMP) r = min(max(r, lo), hi);
      }
      y[i] = r;
    }
  }
}

template <int MODE, bool HAS_CLS, bool CLAMP>
__global__ void __launch_bounds__(kGemmThreads, 1)
    qnn_gemm_i8_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB,
                       const __grid_constant__ CUtensorMap tmC, const __grid_constant__ GemmParams p) {
  extern __shared__ uint8_t smem_raw[];
  // 1024-B aligned base (SW128 atoms); pointer arithmetic on the __shared__ array keeps the address space
  uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  const int BK = p.BK, BN = p.BN, stages = p.stages;
  const uint32_t a_bytes = kGemmBM * BK, b_bytes = BN * BK;
  uint8_t* sA = smem;
  uint8_t* sB = smem + stages * a_bytes;
  uint8_t* sOut = sB + stages * b_bytes;
  int4* sPrm = reinterpret_cast<int4*>(sOut + kStageOutBytes);
  int32_t* sOff = reinterpret_cast<int32_t*>(reinterpret_cast<uint8_t*>(sPrm) + kParamBytes);
  const int ncls = HAS_CLS ? p.e.ncls : 1;
  const int offp = BN + 4;
  uint64_t* full = reinterpret_cast<uint64_t*>(reinterpret_cast<uint8_t*>(sOff) + off_table_bytes(ncls, BN));
  uint64_t* empty = full + stages;
  uint64_t* tfull = empty + stages;
  uint64_t* tempty = tfull + 2;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + 2);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (warp == 0 && lane == 0) {
    tma_prefetch_desc(&tmA);
    tma_prefetch_desc(&tmB);
    if (p.e.tma_store) tma_prefetch_desc(&tmC);
    for (int s = 0; s < stages; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    for (int a = 0; a < 2; ++a) {
      mbar_init(&tfull[a], 1);
      mbar_init(&tempty[a], kGemmEpiWarps);
    }
    fence_mbar_init();
  }
  if (warp == 2) tmem_alloc(tmem_slot, 512);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;

  const int num_tiles = p.num_m_tiles * p.num_n_tiles;

  if (warp == 0) {
    // ------------------------------------------------------------ TMA producer
    if (lane == 0) {
      int stage = 0;
      uint32_t phase = 0;
      for (int t = blockIdx.x; t < num_tiles; t += gridDim.x) {
        const int m_blk = t / p.num_n_tiles, n_blk = t - m_blk * p.num_n_tiles;
        const int m0 = m_blk * kGemmBM;
        int an = 0, ah = 0, aw = 0;
        if (p.im2col) {
          const int pq = p.P * p.Q;
          const int n0 = m0 / pq, rem = m0 - n0 * pq;
          const int p0 = rem / p.Q, q0 = rem - p0 * p.Q;
          an = n0;
          ah = p0 * p.sh - p.pt;
          aw = q0 * p.sw - p.pl;
        }
        for (int kb = 0; kb < p.num_kb; ++kb) {
          mbar_wait(&empty[stage], phase ^ 1);
          mbar_arrive_expect_tx(&full[stage], a_bytes + b_bytes);
          uint8_t* dA = sA + stage * a_bytes;
          uint8_t* dB = sB + stage * b_bytes;
          if (p.im2col) {
            const int tap = kb / p.nchunks, ch = kb - tap * p.nchunks;
            const int r = tap / p.S, s = tap - r * p.S;
            tma_load_im2col_4d(dA, &tmA, &full[stage], ch * BK, aw, ah, an, (uint16_t)(s * p.dil_w),
                               (uint16_t)(r * p.dil_h));
          } else {
            tma_load_2d(dA, &tmA, &full[stage], kb * BK, m0);
          }
          tma_load_2d(dB, &tmB, &full[stage], kb * BK, n_blk * BN);
          if (++stage == stages) {
            stage = 0;
            phase ^= 1;
          }
        }
      }
    }
    __syncwarp();
  } else if (warp == 1) {
    // ------------------------------------------------------------ MMA issuer
    if (lane == 0) {
      int stage = 0;
      uint32_t phase = 0;
      int it = 0;
      for (int t = blockIdx.x; t < num_tiles; t += gridDim.x, ++it) {
        const int acc = it & 1;
        const uint32_t acc_phase = (it >> 1) & 1;
        mbar_wait(&tempty[acc], acc_phase ^ 1);
        tc_fence_after();
        const uint32_t d_tmem = tmem_base + acc * 256;
        for (int kb = 0; kb < p.num_kb; ++kb) {
          mbar_wait(&full[stage], phase);
          tc_fence_after();
          const uint32_t a_addr = smem_u32(sA + stage * a_bytes);
          const uint32_t b_addr = smem_u32(sB + stage * b_bytes);
          for (int k = 0; k < BK / 32; ++k) {
            umma_i8(d_tmem, make_sdesc(a_addr + k * 32, BK), make_sdesc(b_addr + k * 32, BK), p.idesc,
                    (kb | k) != 0);
          }
          umma_commit(&empty[stage]);
          if (++stage == stages) {
            stage = 0;
            phase ^= 1;
          }
        }
        umma_commit(&tfull[acc]);
      }
    }
    __syncwarp();
  } else if (warp >= 4) {
    // ------------------------------------------------------------ epilogue
    const GemmEpilogue& e = p.e;
    const int et = threadIdx.x - 128;   // 0..255
    const int ew = warp - 4;
    const int quad = warp & 3;          // TMEM lanes [32*quad, 32*quad+32) belong to this warp
    const int half = ew >> 2;
    const int nchunk = BN >> 5;
    const int split = (nchunk + 1) >> 1;
    const int c_begin = half ? split : 0, c_end = half ? nchunk : split;
    const int pq = p.P * p.Q;
    const int32_t zp_out = e.zp_out, lo = e.lo, hi = e.hi;
    const bool out8 = e.out_dtype != DT_S32;
    const bool is_s8 = e.out_dtype == DT_S8;
    uint8_t* stage_out = sOut + ew * 2048;
    int sbuf = 0;
    int cur_n = -1, tile_fast = 1;
    int it = 0;
    for (int t = blockIdx.x; t < num_tiles; t += gridDim.x, ++it) {
      const int acc = it & 1;
      const uint32_t acc_phase = (it >> 1) & 1;
      const int m_blk = t / p.num_n_tiles, n_blk = t - m_blk * p.num_n_tiles;
      if (n_blk != cur_n) {
        // stage this N-tile's per-column parameters (all 8 epilogue warps)
        named_bar_sync(1, 32 * kGemmEpiWarps);
        int ok = 1;
        for (int i = et; i < BN; i += 32 * kGemmEpiWarps) {
          const int k = n_blk * BN + i;
          int4 q = make_int4(0, 0, 0, 0);
          if (MODE != 2) {
            const int32_t M = e.mult[k], r = e.rsh[k];
            q.z = M;
            if (r >= 33 && r <= 52) {
              const int tt = r - 32;
              q.w = tt;
              q.y = MODE == 0 ? (int32_t)((1u << (tt - 1)) + (uint32_t)zp_out * (1u << tt)) : (int32_t)(1u << (tt - 1));
            } else {
              q.w = -r;  // generic 64-bit path
              ok = 0;
            }
          }
          sPrm[i] = q;
        }
        for (int i = et; i < ncls * BN; i += 32 * kGemmEpiWarps) {
          const int c = i / BN, j = i - c * BN;
          sOff[c * offp + j] = e.off[(size_t)c * e.Kpad + n_blk * BN + j];
        }
        tile_fast = named_bar_and(1, 32 * kGemmEpiWarps, ok);
        cur_n = n_blk;
      }
      const int row0 = m_blk * kGemmBM + quad * 32;
      const int row = row0 + lane;
      const bool row_ok = row < p.M;
      int cls = 0;
      int32_t rterm = 0;
      if (row_ok) {
        if (HAS_CLS) {
          const int rem = row % pq;
          const int pp = rem / p.Q, qq = rem - pp * p.Q;
          cls = (int)e.rowcls[pp] * e.ncc + (int)e.colcls[qq];
        }
        if (e.rowsum) rterm = (int32_t)((uint32_t)e.zpW * (uint32_t)e.rowsum[row]);
      }
      mbar_wait(&tfull[acc], acc_phase);
      tc_fence_after();
      for (int j = c_begin; j < c_end; ++j) {
        uint32_t v[32];
        tmem_load32(tmem_base + acc * 256 + j * 32 + ((uint32_t)(quad * 32) << 16), v);
        if (j == c_end - 1) {
          // accumulator fully read by this warp: hand the TMEM buffer back to the MMA warp
          tc_fence_before();
          __syncwarp();
          if (lane == 0) mbar_arrive(&tempty[acc]);
        }
        const int k0 = n_blk * BN + j * 32;
        int32_t y[32];
        const int4* prm = sPrm + j * 32;
        const int4* offc = reinterpret_cast<const int4*>(sOff + cls * offp + j * 32);
        if (tile_fast)
          requant_row32<MODE, CLAMP, true>(v, prm, offc, rterm, zp_out, lo, hi, y);
        else
          requant_row32<MODE, CLAMP, false>(v, prm, offc, rterm, zp_out, lo, hi, y);
        if (out8) {
          uint32_t w[8];
#pragma unroll
          for (int i = 0; i < 8; ++i)
            w[i] = is_s8 ? pack4_s8(y[4 * i], y[4 * i + 1], y[4 * i + 2], y[4 * i + 3])
                         : pack4_u8(y[4 * i], y[4 * i + 1], y[4 * i + 2], y[4 * i + 3]);
          if (e.tma_store) {
            // per-warp 32 rows x 32 B sub-tile -> smem -> TMA store (clips rows >= M, cols >= K)
            uint8_t* buf = stage_out + sbuf * 1024;
            if (lane == 0) bulk_wait_read<1>();
            __syncwarp();
            *reinterpret_cast<uint4*>(buf + lane * 32) = make_uint4(w[0], w[1], w[2], w[3]);
            *reinterpret_cast<uint4*>(buf + lane * 32 + 16) = make_uint4(w[4], w[5], w[6], w[7]);
            fence_proxy_async_smem();
            __syncwarp();
            if (lane == 0) {
              tma_store_2d(&tmC, buf, k0, row0);
              bulk_commit();
            }
            sbuf ^= 1;
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
              *reinterpret_cast<int4*>(o + i) = make_int4(y[i], y[i + 1], y[i + 2], y[i + 3]);
          } else {
#pragma unroll
            for (int i = 0; i < 32; ++i)
              if (k0 + i < p.Nout) o[i] = y[i];
          }
        }
      }
      if (c_begin == c_end) {  // no columns for this warp (BN == 32): still release the accumulator
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(&tempty[acc]);
      }
    }
    if (e.tma_store && lane == 0) bulk_wait_all();
    __syncwarp();
  }

  tc_fence_before();
  __syncthreads();
  if (warp == 2) {
    tc_fence_after();
    tmem_dealloc(tmem_base, 512);
  }
}

template <int MODE, bool HAS_CLS, bool CLAMP>
static cudaError_t launch_variant(const CUtensorMap& tmA, const CUtensorMap& tmB, const CUtensorMap& tmC,
                                  const GemmParams& p, int grid, cudaStream_t stream) {
  static int attr_done[64] = {0};
  int dev = 0;
  cudaGetDevice(&dev);
  auto kern = qnn_gemm_i8_kernel<MODE, HAS_CLS, CLAMP>;
  if (dev >= 64 || !attr_done[dev]) {
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024);
    if (e != cudaSuccess) return e;
    if (dev < 64) attr_done[dev] = 1;
  }
  const size_t smem = gemm_smem_bytes(p.BK, p.BN, p.stages, HAS_CLS ? p.e.ncls : 1);
  if (smem > 227 * 1024) return cudaErrorInvalidValue;
  kern<<<grid, kGemmThreads, smem, stream>>>(tmA, tmB, tmC, p);
  count_launch();
  return cudaGetLastError();
}

cudaError_t launch_gemm(const CUtensorMap& tmA, const CUtensorMap& tmB, const CUtensorMap& tmC, const GemmParams& p,
                        int mode, bool clamp, int grid, cudaStream_t stream) {
  const bool cls = p.e.ncls > 1;
#define QNN_GEMM_CASE(M_, C_, K_) \
  if (mode == M_ && cls == C_ && clamp == K_) return launch_variant<M_, C_, K_>(tmA, tmB, tmC, p, grid, stream);
  QNN_GEMM_CASE(0, false, false)
  QNN_GEMM_CASE(0, false, true)
  QNN_GEMM_CASE(0, true, false)
  QNN_GEMM_CASE(0, true, true)
  QNN_GEMM_CASE(1, false, false)
  QNN_GEMM_CASE(1, false, true)
  QNN_GEMM_CASE(1, true, false)
  QNN_GEMM_CASE(1, true, true)
  QNN_GEMM_CASE(2, false, false)
  QNN_GEMM_CASE(2, true, false)
#undef QNN_GEMM_CASE
  return cudaErrorInvalidValue;
}

}  // namespace qnn
