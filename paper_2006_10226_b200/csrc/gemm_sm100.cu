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
//   warps 4..11 : epilogue (TMEM -> registers -> requantize -> global)
// The TMEM accumulator is double-buffered (2 x 256 columns) so the epilogue of
// tile i overlaps the MMAs of tile i+1.
#include "common.cuh"
#include "internal.h"

namespace qnn {

size_t gemm_smem_bytes(int BK, int BN, int stages) {
  return 1024 + (size_t)stages * ((size_t)kGemmBM * BK + (size_t)BN * BK) + 256;
}

int gemm_max_stages(int BK, int BN) {
  const size_t budget = 227 * 1024;
  int s = 8;
  while (s > 2 && gemm_smem_bytes(BK, BN, s) > budget) --s;
  return s;
}

__global__ void __launch_bounds__(kGemmThreads, 1)
    qnn_gemm_i8_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB,
                       const __grid_constant__ GemmParams p) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  const int BK = p.BK, BN = p.BN, stages = p.stages;
  const uint32_t a_bytes = kGemmBM * BK, b_bytes = BN * BK;
  uint8_t* sA = smem;
  uint8_t* sB = smem + stages * a_bytes;
  uint64_t* full = reinterpret_cast<uint64_t*>(sB + stages * b_bytes);
  uint64_t* empty = full + stages;
  uint64_t* tfull = empty + stages;
  uint64_t* tempty = tfull + 2;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + 2);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (warp == 0 && lane == 0) {
    tma_prefetch_desc(&tmA);
    tma_prefetch_desc(&tmB);
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
    const int ew = warp - 4;
    const int quad = warp & 3;          // TMEM lanes [32*quad, 32*quad+32) belong to this warp
    const int half = ew >> 2;
    const int nchunk = BN >> 5;
    const int split = (nchunk + 1) >> 1;
    const int c_begin = half ? split : 0, c_end = half ? nchunk : split;
    const GemmEpilogue& e = p.e;
    const int pq = p.P * p.Q;
    int it = 0;
    for (int t = blockIdx.x; t < num_tiles; t += gridDim.x, ++it) {
      const int acc = it & 1;
      const uint32_t acc_phase = (it >> 1) & 1;
      const int m_blk = t / p.num_n_tiles, n_blk = t - m_blk * p.num_n_tiles;
      const int row = m_blk * kGemmBM + quad * 32 + lane;
      const bool row_ok = row < p.M;
      int cls = 0;
      int32_t rterm = 0;
      if (row_ok) {
        if (e.rowcls) {
          const int rem = row % pq;
          const int pp = rem / p.Q, qq = rem - pp * p.Q;
          cls = (int)e.rowcls[pp] * e.ncc + (int)e.colcls[qq];
        }
        if (e.rowsum) rterm = (int32_t)((uint32_t)e.zpW * (uint32_t)e.rowsum[row]);
      }
      const int32_t* offrow = e.off + (size_t)cls * e.Kpad;
      mbar_wait(&tfull[acc], acc_phase);
      tc_fence_after();
      for (int j = c_begin; j < c_end; ++j) {
        uint32_t v[32];
        tmem_ld_32x32b_x32(tmem_base + acc * 256 + j * 32 + ((uint32_t)(quad * 32) << 16), v);
        tmem_ld_wait();
        const int k0 = n_blk * BN + j * 32;
        int32_t y[32];
#pragma unroll
        for (int i = 0; i < 32; ++i) {
          const int k = k0 + i;
          // int32 wrap arithmetic is exact whenever the true result fits (reading R10)
          const int32_t val = (int32_t)(v[i] + (uint32_t)__ldg(&offrow[k]) - (uint32_t)rterm);
          if (e.requant)
            y[i] = rq_apply(val, __ldg(&e.mult[k]), __ldg(&e.rsh[k]), e.mode, e.zp_out, e.lo, e.hi);
          else
            y[i] = val;
        }
        if (!row_ok) continue;
        const bool full_chunk = k0 + 32 <= p.Nout;
        if (e.out_dtype == DT_S32) {
          int32_t* o = reinterpret_cast<int32_t*>(e.out) + (long long)row * e.out_pitch + k0;
          if (full_chunk && ((reinterpret_cast<uintptr_t>(o) & 15) == 0)) {
#pragma unroll
            for (int i = 0; i < 32; i += 4)
              *reinterpret_cast<int4*>(o + i) = make_int4(y[i], y[i + 1], y[i + 2], y[i + 3]);
          } else {
            for (int i = 0; i < 32 && k0 + i < p.Nout; ++i) o[i] = y[i];
          }
        } else {
          uint8_t* o = reinterpret_cast<uint8_t*>(e.out) + (long long)row * e.out_pitch + k0;
          uint32_t w[8];
#pragma unroll
          for (int i = 0; i < 8; ++i)
            w[i] = ((uint32_t)y[4 * i] & 0xFF) | (((uint32_t)y[4 * i + 1] & 0xFF) << 8) |
                   (((uint32_t)y[4 * i + 2] & 0xFF) << 16) | (((uint32_t)y[4 * i + 3] & 0xFF) << 24);
          if (full_chunk && ((reinterpret_cast<uintptr_t>(o) & 15) == 0)) {
            *reinterpret_cast<uint4*>(o) = make_uint4(w[0], w[1], w[2], w[3]);
            *reinterpret_cast<uint4*>(o + 16) = make_uint4(w[4], w[5], w[6], w[7]);
          } else {
            for (int i = 0; i < 32 && k0 + i < p.Nout; ++i) o[i] = (uint8_t)(w[i >> 2] >> (8 * (i & 3)));
          }
        }
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&tempty[acc]);
    }
  }

  tc_fence_before();
  __syncthreads();
  if (warp == 2) {
    tc_fence_after();
    tmem_dealloc(tmem_base, 512);
  }
}

cudaError_t launch_gemm(const CUtensorMap& tmA, const CUtensorMap& tmB, const GemmParams& p, int grid,
                        cudaStream_t stream) {
  static bool attr_set = false;
  if (!attr_set) {
    cudaError_t e = cudaFuncSetAttribute(qnn_gemm_i8_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         227 * 1024);
    if (e != cudaSuccess) return e;
    attr_set = true;
  }
  const size_t smem = gemm_smem_bytes(p.BK, p.BN, p.stages);
  qnn_gemm_i8_kernel<<<grid, kGemmThreads, smem, stream>>>(tmA, tmB, p);
  count_launch();
  return cudaGetLastError();
}

}  // namespace qnn
