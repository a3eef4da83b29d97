// depthwise_tc.cu — depthwise qnn.conv2d on the 5th-generation tensor cores
// (Eq. 3 with groups = C, zero-point padding P:259).
//
// out[n,p,q,c] = requantize( sum_{valid r,s} A[n, p*sh + r - pt, q*sw + s - pl, c] * W[c,r,s]
//                            + off[cls(p,q)][c] )
// off[cls][c] = bias[c] - zp_A * sum_{taps valid in border class cls} W[c,r,s] restores the
// zp_A padding that TMA's zero fill omits (reading R7; the GEMM uses the same classes).
//
// Layout.  Per work item (image n, 32-channel slice cs, strip of T output rows) one TMA
// box per phase plane brings the strip's input into shared memory: for stride s the
// input is split into sh x sw phase planes (plane (a,b) row i, column j = input pixel
// (sh*(p0 + i) + a - pt, sw*j + b - pl), TMA element strides (sw, sh)), each plane a
// [rows][Wp] array of 32-B pixels (the slice's 32 channels) in the 32-B swizzle.  With
// the flattened output index m = p_local*Wp + q, the A operand of tap (r,s) is the
// plane (r % sh, s % sw) starting at pixel m + (r / sh)*Wp + s / sw: a contiguous run of
// 32-B rows = the SW32 K-major UMMA layout.  So each tap is one tcgen05.mma
// (M = 128 flattened outputs, N = 32 channels, K = 32 channels) against a diagonal
// 32 x 32 B tile holding W[c,r,s] — the tensor core does the per-channel MAC.
// Flattened rows with q >= Q or beyond the strip are computed and discarded.
//
// Roles (18 warps): warps 0-15 epilogue (four sets of four taking every fourth tile),
// warp 16 TMA producer, warp 17 MMA issuer + TMEM allocator.
#include "common.cuh"
#include "epilogue.cuh"
#include "internal.h"

namespace qnn {

namespace {

constexpr int kDwSets = 4;
constexpr int kDwEpiWarps = 4 * kDwSets;
constexpr int kDwThreads = 32 * (kDwEpiWarps + 2);
constexpr int kDwNacc = 16;            // TMEM accumulator buffers of 32 columns
constexpr int kDwTmemCols = 512;
constexpr int kDwGroup = 4;            // tiles per MMA group (tap loop outside)

__device__ __forceinline__ void tma_load_4d(void* dst, const void* desc, uint64_t* bar, int c0, int c1, int c2,
                                            int c3) {
  asm volatile(
      "cp.async.bulk.tensor.4d.shared::cluster.global.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%3, %4, %5, %6}], [%2];" ::"r"(smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(desc)), "r"(smem_u32(bar)), "r"(c0), "r"(c1), "r"(c2), "r"(c3)
      : "memory");
}
__device__ __forceinline__ void bulk_load(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                   smem_u32(dst)),
               "l"(src), "r"(bytes), "r"(smem_u32(bar))
               : "memory");
}

// no-swizzle K-major UMMA shared-memory descriptor (for the diagonal B tiles)
__device__ __forceinline__ uint64_t sdesc_noswz(uint32_t saddr, uint32_t lbo_bytes, uint32_t sbo_bytes) {
  uint64_t d = 0;
  d |= (uint64_t)((saddr & 0x3FFFFu) >> 4);
  d |= (uint64_t)((lbo_bytes >> 4) & 0x3FFFu) << 16;
  d |= (uint64_t)((sbo_bytes >> 4) & 0x3FFFu) << 32;
  d |= (uint64_t)1 << 46;   // version; layout type 0 = SWIZZLE_NONE
  return d;
}

__device__ __forceinline__ void item_coords(const DwTcParams& p, int item, int& n, int& cs, int& strip) {
  strip = item % p.nstrips;
  const int t = item / p.nstrips;
  cs = t % p.ncs;
  n = t / p.ncs;
}

#ifdef QNN_DWTC_TRACE_BUILD
__device__ __forceinline__ void dtrace(const DwTcParams& p, int slot) {
  if (p.trace && blockIdx.x == 0 && slot < 8192) p.trace[slot] = clock64();
}
#else
__device__ __forceinline__ void dtrace(const DwTcParams&, int) {}
#endif

}  // namespace

size_t dwtc_param_bytes(int ncls) { return (size_t)kDwSets * (256 + 128 + (size_t)ncls * 32 * 8); }

template <int MODE, bool CLAMP, bool S8OUT>
__global__ void __launch_bounds__(kDwThreads, 1)
    depthwise_tc_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ DwTcParams p) {
  pdl_wait();      // inputs are the previous kernel's output (PDL launch; no early trigger: the
                   // next kernel's CTAs would take this multi-wave grid's slots while waiting)
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  uint8_t* stages = smem;                                           // p.stages x p.stage_bytes
  uint8_t* tail = stages + (size_t)p.stages * p.stage_bytes;
  const int ncls = p.ncls;
  const size_t set_bytes = 256 + 128 + (size_t)ncls * 32 * 8;       // {M,t}[32], c[32], K[ncls][32]
  uint64_t* full = reinterpret_cast<uint64_t*>(tail + kDwSets * set_bytes);
  uint64_t* empty = full + 4;
  uint64_t* tfull = empty + 4;
  uint64_t* tempty = tfull + kDwNacc;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + kDwNacc);

  const int warp = __shfl_sync(0xffffffffu, (int)(threadIdx.x >> 5), 0), lane = threadIdx.x & 31;
  constexpr int kProdWarp = kDwEpiWarps, kMmaWarp = kDwEpiWarps + 1;
  const int item_lo = (int)((long long)blockIdx.x * p.items / gridDim.x);
  const int item_hi = (int)((long long)(blockIdx.x + 1) * p.items / gridDim.x);

  if (threadIdx.x == 0) dtrace(p, 8000);
  if (warp == kProdWarp && lane == 0) {
    tma_prefetch_desc(&tmA);
    for (int s = 0; s < p.stages; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    for (int a = 0; a < kDwNacc; ++a) {
      mbar_init(&tfull[a], 1);
      mbar_init(&tempty[a], 4);
    }
    fence_mbar_init();
  }
  if (warp == kMmaWarp) tmem_alloc(tmem_slot, kDwTmemCols);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;
  const int RS = p.R * p.S;
  const uint32_t region = (uint32_t)p.region_bytes;
  const uint32_t b_off = (uint32_t)p.nplanes * region;   // B tiles after the input planes

  if (warp == kProdWarp) {
    // ------------------------------------------------------------ TMA producer
    if (lane == 0) {
      int stage = 0;
      uint32_t phase = 0;
      const uint32_t bytes = (uint32_t)p.nplanes * p.in_rows * p.Wp * 32u + (uint32_t)RS * 1024u;
      for (int item = item_lo; item < item_hi; ++item) {
        int n, cs, strip;
        item_coords(p, item, n, cs, strip);
        const int p0 = strip * p.T;
        dtrace(p, (item - item_lo) * 2);
        mbar_wait(&empty[stage], phase ^ 1);
        dtrace(p, (item - item_lo) * 2 + 1);
        uint8_t* sb = stages + (size_t)stage * p.stage_bytes;
        mbar_arrive_expect_tx(&full[stage], bytes);
        for (int plane = 0; plane < p.nplanes; ++plane) {
          const int a = plane / p.sw, b = plane - a * p.sw;
          tma_load_4d(sb + (size_t)plane * region, &tmA, &full[stage], cs * 32, b - p.pl, p.sh * p0 + a - p.pt, n);
        }
        bulk_load(sb + b_off, p.wpk + (size_t)cs * RS * 1024, (uint32_t)RS * 1024u, &full[stage]);
        if (++stage == p.stages) {
          stage = 0;
          phase ^= 1;
        }
      }
    }
  } else if (warp == kMmaWarp) {
    // ------------------------------------------------------------ MMA issuer
    const bool leader = elect_one();
    int stage = 0, it = 0;
    uint32_t phase = 0;
    for (int item = item_lo; item < item_hi; ++item) {
      mbar_wait(&full[stage], phase);
      tc_fence_after();
      const uint32_t sbase = smem_u32(stages + (size_t)stage * p.stage_bytes);
      // tiles in groups with the tap loop outside: consecutive MMAs write different accumulators
      for (int t0 = 0; t0 < p.tiles_per_item; t0 += kDwGroup) {
        const int ng = min(kDwGroup, p.tiles_per_item - t0);
        dtrace(p, 200 + 2 * (it & 1023));
        for (int g = 0; g < ng; ++g) mbar_wait(&tempty[(it + g) & (kDwNacc - 1)], (((it + g) >> 4) & 1) ^ 1);
        dtrace(p, 201 + 2 * (it & 1023));
        tc_fence_after();
        if (leader) {
          for (int tap = 0; tap < RS; ++tap) {
            const int r = tap / p.S, s = tap - r * p.S;
            const int plane = (r % p.sh) * p.sw + (s % p.sw);
            const int off = (r / p.sh) * p.Wp + s / p.sw;
            const uint64_t bd = sdesc_noswz(sbase + b_off + tap * 1024, 512, 128);
            for (int g = 0; g < ng; ++g) {
              const uint32_t a_addr = sbase + (uint32_t)plane * region + (uint32_t)((t0 + g) * 128 + off) * 32u;
              umma_i8(tmem_base + ((it + g) & (kDwNacc - 1)) * 32, make_sdesc(a_addr, 32), bd, p.idesc, tap > 0);
            }
          }
          for (int g = 0; g < ng; ++g) umma_commit(&tfull[(it + g) & (kDwNacc - 1)]);
        }
        __syncwarp();
        it += ng;
      }
      if (leader) umma_commit(&empty[stage]);
      __syncwarp();
      if (++stage == p.stages) {
        stage = 0;
        phase ^= 1;
      }
    }
  } else if (warp < kDwEpiWarps) {
    // ------------------------------------------------------------ epilogue
    const int set = warp >> 2, quad = warp & 3;
    const int st = threadIdx.x & 127;   // thread index within the set
    uint8_t* sp = tail + set * set_bytes;
    int2* mt = reinterpret_cast<int2*>(sp);                 // {M, t} per channel
    int32_t* cc = reinterpret_cast<int32_t*>(sp + 256);     // c per channel (TONEAREST)
    long long* kk = reinterpret_cast<long long*>(sp + 384); // [ncls][32] K (UPWARD) / int32 off (TONEAREST)
    int cur_cs = -1, fast = 1;
    int it = 0;
    for (int item = item_lo; item < item_hi; ++item) {
      int n, cs, strip;
      item_coords(p, item, n, cs, strip);
      const int p0 = strip * p.T;
      for (int t = 0; t < p.tiles_per_item; ++t, ++it) {
        if ((it & (kDwSets - 1)) != set) continue;
        if (cs != cur_cs) {
          // stage this slice's parameters (this set's four warps)
          named_bar_sync(1 + set, 128);
          int ok = 1;
          if (st < 32) {
            const int c = cs * 32 + st;
            const int32_t r = p.rsh[c], M = p.mult[c];
            int tt = -r;
            if (r >= 33 && r <= 52) {
              tt = r - 32;
              cc[st] = MODE == 0 ? 0 : (int32_t)(1u << (tt - 1));
            } else {
              ok = 0;
              cc[st] = 0;
            }
            mt[st] = make_int2(M, tt);
          }
          for (int i = st; i < ncls * 32; i += 128) {
            const int cl = i >> 5, j = i & 31, c = cs * 32 + j;
            if (MODE == 0) {
              const int32_t r = p.rsh[c];
              unsigned long long K = 0;
              if (r >= 33 && r <= 52) {
                const int tt = r - 32;
                const unsigned long long c64 = (1ull << (tt - 1)) + ((unsigned long long)(long long)p.zp_out << tt);
                K = (unsigned long long)p.off64[(size_t)cl * p.Cpad + c] * (unsigned long long)(long long)p.mult[c] +
                    (c64 << 32);
              }
              kk[i] = (long long)K;
            } else {
              reinterpret_cast<int32_t*>(kk)[i] = p.off[(size_t)cl * p.Cpad + c];
            }
          }
          fast = named_bar_and(1 + set, 128, ok);
          cur_cs = cs;
        }
        const int m = t * 128 + quad * 32 + lane;
        const int pl_ = m / p.Wp, q = m - pl_ * p.Wp;
        const int pp = p0 + pl_;
        const bool valid = q < p.Q && pl_ < p.T && pp < p.P;
        int cls = 0;
        if (ncls > 1 && valid) cls = (int)p.rowcls[pp] * p.ncc + (int)p.colcls[q];
        const int acc = it & (kDwNacc - 1);
        if (lane == 0 && quad == 0) dtrace(p, 1000 + 4 * (it & 1023));
        mbar_wait(&tfull[acc], (it >> 4) & 1);
        if (lane == 0 && quad == 0) dtrace(p, 1001 + 4 * (it & 1023));
        tc_fence_after();
        uint32_t v[32];
        tmem_load32(tmem_base + acc * 32 + ((uint32_t)(quad * 32) << 16), v);
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(&tempty[acc]);
        uint32_t w[8];
        int32_t y[1];
        const int4* mt4 = reinterpret_cast<const int4*>(mt);
        if (MODE == 0 && fast) {
          epi_chunk_up<CLAMP, S8OUT, false>(v, mt4, reinterpret_cast<const longlong2*>(kk + cls * 32), 0, p.lo, p.hi,
                                            w);
        } else if (MODE == 0) {
          epi_chunk<0, CLAMP, false, S8OUT>(v, reinterpret_cast<const int4*>(p.off + (size_t)cls * p.Cpad + cs * 32),
                                            mt4, mt4, 0, p.zp_out, p.lo, p.hi, w, y);
        } else {
          const int4* off4 = reinterpret_cast<const int4*>(reinterpret_cast<const int32_t*>(kk) + cls * 32);
          if (fast)
            epi_chunk<1, CLAMP, true, S8OUT>(v, off4, mt4, reinterpret_cast<const int4*>(cc), 0, p.zp_out, p.lo,
                                             p.hi, w, y);
          else
            epi_chunk<1, CLAMP, false, S8OUT>(v, off4, mt4, reinterpret_cast<const int4*>(cc), 0, p.zp_out, p.lo,
                                              p.hi, w, y);
        }
        if (valid) {
          uint8_t* o = p.out + (((long long)n * p.P + pp) * p.Q + q) * p.out_cs + cs * 32;
          *reinterpret_cast<uint4*>(o) = make_uint4(w[0], w[1], w[2], w[3]);
          if (cs * 32 + 16 < p.C) *reinterpret_cast<uint4*>(o + 16) = make_uint4(w[4], w[5], w[6], w[7]);
        }
        if (lane == 0 && quad == 0) dtrace(p, 1002 + 4 * (it & 1023));
      }
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == kMmaWarp) {
    tc_fence_after();
    tmem_dealloc(tmem_base, kDwTmemCols);
  }
}

// ---------------------------------------------------------------------------- host
size_t dwtc_smem_bytes(int stages, int stage_bytes, int ncls) {
  return 1024 + (size_t)stages * stage_bytes + dwtc_param_bytes(ncls) + 8 * (8 + 2 * kDwNacc) + 64;
}

// Plan the strip height T and the stage size; false if the shape does not fit.
bool dwtc_plan(DwTcParams& p) {
  p.nplanes = p.sh * p.sw;
  p.Wp = p.Q + (p.S - 1) / p.sw;
  if (p.Wp * p.sw > 256) return false;              // TMA box extent along W
  const int max_off = ((p.R - 1) / p.sh) * p.Wp + (p.S - 1) / p.sw;
  const int RS = p.R * p.S;
  for (int T = std::min(p.P, 64); T >= 1; --T) {
    const int in_rows = T + (p.R - 1) / p.sh;
    if (in_rows * p.sh > 256) continue;            // TMA box extent along H
    const int tiles = (T * p.Wp + 127) / 128;
    const int rows = std::max(in_rows * p.Wp, tiles * 128 + max_off);
    const int region = (rows * 32 + 1023) / 1024 * 1024;
    const int stage = p.nplanes * region + (RS * 1024 + 1023) / 1024 * 1024;
    int stages = 4;
    while (stages > 2 && dwtc_smem_bytes(stages, stage, p.ncls) > 220 * 1024) --stages;
    if (dwtc_smem_bytes(stages, stage, p.ncls) > 220 * 1024) continue;
    if (stages < 3 && T > 4) continue;             // prefer >= 3 stages of a shorter strip
    p.T = T;
    p.in_rows = in_rows;
    p.tiles_per_item = tiles;
    p.region_bytes = region;
    p.stage_bytes = stage;
    p.stages = stages;
    p.nstrips = (p.P + T - 1) / T;
    p.ncs = (p.C + 31) / 32;
    p.items = p.N * p.ncs * p.nstrips;
    return true;
  }
  return false;
}

template <int MODE, bool CLAMP, bool S8OUT>
static cudaError_t dwtc_launch_variant(const CUtensorMap& tmA, const DwTcParams& p, int grid, cudaStream_t s) {
  auto kern = depthwise_tc_kernel<MODE, CLAMP, S8OUT>;
  static int attr_done[64] = {0};
  int dev = 0;
  cudaGetDevice(&dev);
  if (dev >= 64 || !attr_done[dev]) {
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024);
    if (e != cudaSuccess) return e;
    if (dev < 64) attr_done[dev] = 1;
  }
  launch_pdl(kern, dim3(grid), dim3(kDwThreads), dwtc_smem_bytes(p.stages, p.stage_bytes, p.ncls), s, tmA, p);
  count_launch();
  return cudaGetLastError();
}

cudaError_t launch_depthwise_tc(const CUtensorMap& tmA, const DwTcParams& p, int mode, bool clamp, bool s8out,
                                cudaStream_t s) {
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const int grid = std::max(1, std::min(p.items, sms));
#define QNN_DWTC(M_, C_, S_) \
  if (mode == M_ && clamp == C_ && s8out == S_) return dwtc_launch_variant<M_, C_, S_>(tmA, p, grid, s);
  QNN_DWTC(0, false, false) QNN_DWTC(0, false, true) QNN_DWTC(0, true, false) QNN_DWTC(0, true, true)
  QNN_DWTC(1, false, false) QNN_DWTC(1, false, true) QNN_DWTC(1, true, false) QNN_DWTC(1, true, true)
#undef QNN_DWTC
  return cudaErrorInvalidValue;
}

// Diagonal B tiles: for slice cs and tap, a 32 x 32 (N x K) int8 tile holding W[32cs + n, tap]
// at (n, n) (0 for channels >= C), stored as no-swizzle K-major core matrices:
// byte (n / 8) * 128 + (k / 16) * 512 + (n % 8) * 16 + k % 16.
__global__ void pack_dwtc_kernel(const int8_t* __restrict__ W, int C, int RS, uint8_t* __restrict__ wpk) {
  const int ncs = (C + 31) / 32;
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < ncs * RS * 1024; i += gridDim.x * blockDim.x) {
    const int tile = i / 1024, e = i - tile * 1024;
    const int cs = tile / RS, tap = tile - cs * RS;
    const int kh = e / 512, rem = e - kh * 512, g = rem / 128, rem2 = rem - g * 128;
    const int n = g * 8 + rem2 / 16, k = kh * 16 + (rem2 % 16);
    const int c = cs * 32 + n;
    wpk[i] = (n == k && c < C) ? (uint8_t)W[c * RS + tap] : 0;
  }
}

cudaError_t launch_pack_dwtc(const void* W, int C, int RS, void* wpk, cudaStream_t s) {
  pack_dwtc_kernel<<<128, 256, 0, s>>>(reinterpret_cast<const int8_t*>(W), C, RS, reinterpret_cast<uint8_t*>(wpk));
  count_launch();
  return cudaGetLastError();
}

}  // namespace qnn
