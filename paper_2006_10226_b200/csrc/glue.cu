// glue.cu — inter-layer glue on the int8 path: qnn.add and pooling.
//
//   qnn.add   (reading R19): y = sat(max?(zp_out + R((a - zp_a) m_a) + R((b - zp_b) m_b)))
//             with m_x = s_x / s_out as fixed-point multipliers (Eq. 5).
//   pool2d    (reading R20): max, or rounding-division average, over the valid
//             taps of each window; input and output share (scale, zero point).
// Both are HBM-bound: 16-byte vector accesses, one warp instruction per contiguous span.
#include "common.cuh"
#include "internal.h"

namespace qnn {

namespace {

__device__ __forceinline__ uint32_t pack4_sat_u8(int a, int b, int c, int d) {
  uint32_t o;
  asm("{\n\t.reg .u32 t;\n\tcvt.pack.sat.u8.s32.b32 t, %4, %3, 0;\n\tcvt.pack.sat.u8.s32.b32 %0, %2, %1, t;\n\t}"
      : "=r"(o) : "r"(a), "r"(b), "r"(c), "r"(d));
  return o;
}
__device__ __forceinline__ uint32_t pack4_sat_s8(int a, int b, int c, int d) {
  uint32_t o;
  asm("{\n\t.reg .u32 t;\n\tcvt.pack.sat.s8.s32.b32 t, %4, %3, 0;\n\tcvt.pack.sat.s8.s32.b32 %0, %2, %1, t;\n\t}"
      : "=r"(o) : "r"(a), "r"(b), "r"(c), "r"(d));
  return o;
}
template <bool S8>
__device__ __forceinline__ int32_t byte_of(uint32_t w, int j) {
  const uint32_t b = (w >> (8 * j)) & 0xFFu;
  return S8 ? (int32_t)(int8_t)b : (int32_t)b;
}

// R((x - zp) * M * 2^-rsh): 64-bit fast form when rsh is in [11, 52] (|x - zp| < 2^9),
// else the generic rounding of common.cuh.
__device__ __forceinline__ int32_t rq_small(int32_t xz, int32_t M, int rsh, int mode) {
  return (int32_t)rq_round((int64_t)xz * M, rsh, mode);
}

}  // namespace

// --------------------------------------------------------------------------------- qnn.add
template <bool AS8, bool BS8, bool OS8>
__global__ void __launch_bounds__(256) add_kernel(const __grid_constant__ AddParams p) {
  pdl_wait();      // inputs are the previous kernel's output (PDL launch; no early trigger: the
                   // next kernel's CTAs would take this multi-wave grid's slots while waiting)
  const long long nthreads = (long long)gridDim.x * blockDim.x;
  const long long tid = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  const long long nvec = p.vec ? p.count >> 4 : 0;
  auto one = [&](int32_t a, int32_t b) -> int32_t {
    int32_t y = rq_small(a - p.zp_a, p.Ma, p.ra, p.mode) + rq_small(b - p.zp_b, p.Mb, p.rb, p.mode) + p.zp_out;
    if (p.relu) y = max(y, p.zp_out);
    return y;
  };
  for (long long v = tid; v < nvec; v += nthreads) {
    const uint4 av = __ldg(reinterpret_cast<const uint4*>(p.a) + v);
    const uint4 bv = __ldg(reinterpret_cast<const uint4*>(p.b) + v);
    const uint32_t aw[4] = {av.x, av.y, av.z, av.w}, bw[4] = {bv.x, bv.y, bv.z, bv.w};
    uint32_t ow[4];
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      int32_t y[4];
#pragma unroll
      for (int j = 0; j < 4; ++j) y[j] = one(byte_of<AS8>(aw[k], j), byte_of<BS8>(bw[k], j));
      ow[k] = OS8 ? pack4_sat_s8(y[0], y[1], y[2], y[3]) : pack4_sat_u8(y[0], y[1], y[2], y[3]);
    }
    reinterpret_cast<uint4*>(p.out)[v] = make_uint4(ow[0], ow[1], ow[2], ow[3]);
  }
  for (long long i = (nvec << 4) + tid; i < p.count; i += nthreads) {
    const uint8_t* a8 = reinterpret_cast<const uint8_t*>(p.a);
    const uint8_t* b8 = reinterpret_cast<const uint8_t*>(p.b);
    const int32_t a = AS8 ? (int32_t)(int8_t)a8[i] : (int32_t)a8[i];
    const int32_t b = BS8 ? (int32_t)(int8_t)b8[i] : (int32_t)b8[i];
    const int32_t y = min(max(one(a, b), OS8 ? -128 : 0), OS8 ? 127 : 255);
    reinterpret_cast<uint8_t*>(p.out)[i] = (uint8_t)y;
  }
}

cudaError_t launch_add(const AddParams& p, cudaStream_t s) {
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const long long work = p.vec ? (p.count + 15) / 16 : p.count;
  const int blocks = (int)std::max<long long>(1, std::min<long long>((work + 255) / 256, (long long)sms * 8));
#define QNN_ADD(A_, B_, O_) \
  if (p.a_s8 == A_ && p.b_s8 == B_ && p.o_s8 == O_) launch_pdl(add_kernel<A_, B_, O_>, dim3(blocks), dim3(256), 0, s, p);
  QNN_ADD(false, false, false) QNN_ADD(false, false, true) QNN_ADD(false, true, false) QNN_ADD(false, true, true)
  QNN_ADD(true, false, false) QNN_ADD(true, false, true) QNN_ADD(true, true, false) QNN_ADD(true, true, true)
#undef QNN_ADD
  count_launch();
  return cudaGetLastError();
}

// --------------------------------------------------------------------------------- pooling
// VEC channels per thread (16: one uint4 per tap, C % 16 == 0 and aligned pitches; else 1).
template <int VEC, bool S8, bool AVG>
__global__ void __launch_bounds__(256) pool_kernel(const __grid_constant__ PoolParams p) {
  pdl_wait();      // inputs are the previous kernel's output (PDL launch; no early trigger: the
                   // next kernel's CTAs would take this multi-wave grid's slots while waiting)
  const int G = p.C / VEC;
  const long long total = (long long)p.N * p.P * p.Q * G;
  const uint8_t* in = reinterpret_cast<const uint8_t*>(p.in);
  uint8_t* out = reinterpret_cast<uint8_t*>(p.out);
  for (long long idx = blockIdx.x * (long long)blockDim.x + threadIdx.x; idx < total;
       idx += (long long)gridDim.x * blockDim.x) {
    const int g = (int)(idx % G);
    const long long pix = idx / G;
    const int q = (int)(pix % p.Q);
    const long long t = pix / p.Q;
    const int pp = (int)(t % p.P), n = (int)(t / p.P);
    int32_t acc[VEC];
#pragma unroll
    for (int j = 0; j < VEC; ++j) acc[j] = AVG ? 0 : INT32_MIN;
    int cnt = 0;
    for (int r = 0; r < p.R; ++r) {
      const int h = pp * p.sh + r - p.pt;
      if (h < 0 || h >= p.H) continue;
      for (int s = 0; s < p.S; ++s) {
        const int w = q * p.sw + s - p.pl;
        if (w < 0 || w >= p.W) continue;
        ++cnt;
        const uint8_t* src = in + (((long long)n * p.H + h) * p.W + w) * p.in_cs + g * VEC;
        if (VEC == 16) {
          const uint4 v = __ldg(reinterpret_cast<const uint4*>(src));
          const uint32_t vw[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
          for (int j = 0; j < 16; ++j) {
            const int32_t x = byte_of<S8>(vw[j >> 2], j & 3);
            acc[j] = AVG ? acc[j] + x : max(acc[j], x);
          }
        } else {
          const int32_t x = S8 ? (int32_t)(int8_t)src[0] : (int32_t)src[0];
          acc[0] = AVG ? acc[0] + x : max(acc[0], x);
        }
      }
    }
    int32_t y[VEC];
#pragma unroll
    for (int j = 0; j < VEC; ++j) {
      if (AVG) {
        // sign(s) * floor((2|s| + n) / (2n)); all operands are small positive ints
        const int32_t a = acc[j] < 0 ? -acc[j] : acc[j];
        const int32_t m = cnt > 0 ? (2 * a + cnt) / (2 * cnt) : 0;
        y[j] = acc[j] < 0 ? -m : m;
      } else {
        y[j] = cnt > 0 ? acc[j] : 0;
      }
    }
    uint8_t* dst = out + (((long long)n * p.P + pp) * p.Q + q) * p.out_cs + g * VEC;
    if (VEC == 16) {
      uint32_t ow[4];
#pragma unroll
      for (int k = 0; k < 4; ++k)
        ow[k] = S8 ? pack4_sat_s8(y[4 * k], y[4 * k + 1], y[4 * k + 2], y[4 * k + 3])
                   : pack4_sat_u8(y[4 * k], y[4 * k + 1], y[4 * k + 2], y[4 * k + 3]);
      *reinterpret_cast<uint4*>(dst) = make_uint4(ow[0], ow[1], ow[2], ow[3]);
    } else {
      dst[0] = (uint8_t)y[0];
    }
  }
}

// Fast path (16 channels per thread, C % 16 == 0, 16-B aligned pitches): a thread owns TQ
// consecutive output columns of one output row and one 16-channel group, and loads each input
// column of their union window once per filter row ((TQ-1)*sw + S loads instead of TQ*S).
// Max: byte-parallel __vmaxu4 / __vmaxs4.  Average: sums in 16-bit lanes (<= 255 * 128 taps
// fits; s8 is biased by 128 into u8 and unbiased after), then the rounding division of R20 by
// an exact multiply-shift: floor(x / d) = (x * (2^32 / d + 1)) >> 32 for x < 2^16, d < 2^8.
// m = floor(2^32 / d) + 1 is computed once per output (d = 2 * count); x < 2^16 keeps the
// error x * (m - 2^32 / d) / 2^32 below 1/d, so the floor is exact
__device__ __forceinline__ uint32_t div_magic(uint32_t d) { return 0xFFFFFFFFu / d + 1u; }
__device__ __forceinline__ uint32_t div_small(uint32_t x, uint32_t m) {
  return (uint32_t)(((unsigned long long)x * m) >> 32);
}

template <bool S8, bool AVG, int TQ>
__global__ void __launch_bounds__(256) pool16_kernel(const __grid_constant__ PoolParams p, FastDiv fdG,
                                                      FastDiv fdQB, FastDiv fdP) {
  pdl_wait();      // inputs are the previous kernel's output (PDL launch; no early trigger: the
                   // next kernel's CTAs would take this multi-wave grid's slots while waiting)
  const int G = p.C >> 4;
  const int QB = (p.Q + TQ - 1) / TQ;
  const uint32_t total = (uint32_t)p.N * p.P * QB * G;
  const uint8_t* in = reinterpret_cast<const uint8_t*>(p.in);
  uint8_t* out = reinterpret_cast<uint8_t*>(p.out);
  const uint32_t bias = S8 ? 0x80808080u : 0u;   // s8 -> u8 (x + 128) for the byte-parallel ops
  for (uint32_t idx = blockIdx.x * blockDim.x + threadIdx.x; idx < total; idx += gridDim.x * blockDim.x) {
    const uint32_t rest0 = fdiv(idx, fdG);
    const int g = (int)(idx - rest0 * G);
    const uint32_t rest1 = fdiv(rest0, fdQB);
    const int qb = (int)(rest0 - rest1 * QB);
    const uint32_t n = fdiv(rest1, fdP);
    const int pp = (int)(rest1 - n * p.P);
    const int q0 = qb * TQ;
    // acc[t][k]: max -> 4 packed bytes per word (4 words = 16 channels); avg -> 2 x 16-bit
    // lanes per word (8 words: even bytes in [0..3], odd bytes in [4..7])
    uint32_t acc[TQ][8];
#pragma unroll
    for (int t = 0; t < TQ; ++t)
#pragma unroll
      for (int k = 0; k < 8; ++k) acc[t][k] = 0u;
    int rows = 0;
    const int w0 = q0 * p.sw - p.pl;
    const int ncols = (TQ - 1) * p.sw + p.S;
    for (int r = 0; r < p.R; ++r) {
      const int h = pp * p.sh + r - p.pt;
      if (h < 0 || h >= p.H) continue;
      ++rows;
      const uint8_t* rowp = in + (((long long)n * p.H + h) * p.W) * p.in_cs + g * 16;
      for (int c = 0; c < ncols; ++c) {
        const int w = w0 + c;
        if (w < 0 || w >= p.W) continue;
        const uint4 v4 = __ldg(reinterpret_cast<const uint4*>(rowp + (long long)w * p.in_cs));
        const uint32_t v[4] = {v4.x ^ bias, v4.y ^ bias, v4.z ^ bias, v4.w ^ bias};
#pragma unroll
        for (int t = 0; t < TQ; ++t) {
          const int sidx = c - t * p.sw;
          if (sidx < 0 || sidx >= p.S) continue;
#pragma unroll
          for (int k = 0; k < 4; ++k) {
            if (AVG) {
              acc[t][k] = __vadd2(acc[t][k], v[k] & 0x00FF00FFu);
              acc[t][k + 4] = __vadd2(acc[t][k + 4], (v[k] >> 8) & 0x00FF00FFu);
            } else {
              acc[t][k] = __vmaxu4(acc[t][k], v[k]);   // (biased s8 orders like u8)
            }
          }
        }
      }
    }
#pragma unroll
    for (int t = 0; t < TQ; ++t) {
      const int q = q0 + t;
      if (q >= p.Q) break;
      uint32_t ow[4];
      if (AVG) {
        int cols = 0;
        for (int sidx = 0; sidx < p.S; ++sidx) {
          const int w = q * p.sw + sidx - p.pl;
          cols += (w >= 0 && w < p.W) ? 1 : 0;
        }
        const int cnt = rows * cols;
        const uint32_t mag = div_magic(2u * (uint32_t)(cnt > 0 ? cnt : 1));
#pragma unroll
        for (int k = 0; k < 4; ++k) {
          uint32_t bytes = 0;
#pragma unroll
          for (int j = 0; j < 4; ++j) {
            const uint32_t word = j & 1 ? acc[t][k + 4] : acc[t][k];
            int32_t sum = (int32_t)((word >> (16 * (j >> 1))) & 0xFFFFu);
            if (S8) sum -= 128 * cnt;
            int32_t y = 0;
            if (cnt > 0) {
              // sign(s) * floor((2|s| + n) / (2n)): ties away from zero (reading R20)
              const uint32_t a = (uint32_t)(sum < 0 ? -sum : sum);
              const int32_t m = (int32_t)div_small(2u * a + (uint32_t)cnt, mag);
              y = sum < 0 ? -m : m;
            }
            bytes |= ((uint32_t)y & 0xFFu) << (8 * j);
          }
          ow[k] = bytes;
        }
      } else {
#pragma unroll
        for (int k = 0; k < 4; ++k) ow[k] = acc[t][k] ^ bias;
      }
      uint8_t* dst = out + (((long long)n * p.P + pp) * p.Q + q) * p.out_cs + g * 16;
      *reinterpret_cast<uint4*>(dst) = make_uint4(ow[0], ow[1], ow[2], ow[3]);
    }
  }
}


// 3x3 pooling with stride SH (1 or 2), separable: a thread owns 16 channels of one output
// column and sweeps a band of BP output rows; each input row is loaded once (3 x 16 B) and
// reduced across its 3 columns into 16-bit lanes (even / odd bytes: VIMNMX.U16x2 for max,
// VIADD.16x2 for sums, one instruction per 2 lanes), and an output row combines the row
// reductions of its 3 input rows -- kept in registers across output rows (stride 1 reuses 2
// of them, stride 2 one).  Same results as pool16_kernel (max of the valid taps; average =
// valid-tap sum / count rounded half away from zero, reading R20).
constexpr int kP3Band = 8;
__device__ __forceinline__ void p3_split(const uint4 v4, uint32_t bias, uint32_t (&lo)[4], uint32_t (&hi)[4]) {
  const uint32_t v[4] = {v4.x ^ bias, v4.y ^ bias, v4.z ^ bias, v4.w ^ bias};
#pragma unroll
  for (int k = 0; k < 4; ++k) {
    lo[k] = v[k] & 0x00FF00FFu;
    hi[k] = (v[k] >> 8) & 0x00FF00FFu;
  }
}
template <bool AVG>
__device__ __forceinline__ void p3_row(const uint8_t* rowp, long long cs, int w0, int W, bool rok, uint32_t bias,
                                       uint32_t (&red)[8]) {
#pragma unroll
  for (int k = 0; k < 8; ++k) red[k] = 0u;   // (max identity: 0 in the biased unsigned domain)
  if (!rok) return;
#pragma unroll
  for (int s = 0; s < 3; ++s) {
    const int w = w0 + s;
    if (w < 0 || w >= W) continue;
    uint32_t lo[4], hi[4];
    p3_split(__ldg(reinterpret_cast<const uint4*>(rowp + (long long)w * cs)), bias, lo, hi);
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      red[k] = AVG ? __vadd2(red[k], lo[k]) : __vmaxu2(red[k], lo[k]);
      red[k + 4] = AVG ? __vadd2(red[k + 4], hi[k]) : __vmaxu2(red[k + 4], hi[k]);
    }
  }
}

template <bool S8, bool AVG, int SH>
__global__ void __launch_bounds__(256) pool3_kernel(const __grid_constant__ PoolParams p, FastDiv fdG, FastDiv fdQ,
                                                    FastDiv fdB) {
  pdl_wait();      // inputs are the previous kernel's output (PDL launch; no early trigger)
  const int G = p.C >> 4;
  const int NB = (p.P + kP3Band - 1) / kP3Band;
  const uint32_t total = (uint32_t)p.N * NB * p.Q * G;
  const uint8_t* in = reinterpret_cast<const uint8_t*>(p.in);
  uint8_t* out = reinterpret_cast<uint8_t*>(p.out);
  const uint32_t bias = S8 ? 0x80808080u : 0u;
  for (uint32_t idx = blockIdx.x * blockDim.x + threadIdx.x; idx < total; idx += gridDim.x * blockDim.x) {
    const uint32_t r0 = fdiv(idx, fdG);
    const int g = (int)(idx - r0 * G);
    const uint32_t r1 = fdiv(r0, fdQ);
    const int q = (int)(r0 - r1 * p.Q);
    const uint32_t n = fdiv(r1, fdB);
    const int b = (int)(r1 - n * NB);
    const int p0 = b * kP3Band, p1 = min(p.P, p0 + kP3Band);
    const int w0 = q * SH - p.pl;
    int cols = 0;
#pragma unroll
    for (int s = 0; s < 3; ++s) cols += (w0 + s >= 0 && w0 + s < p.W) ? 1 : 0;
    const uint8_t* base = in + (long long)n * p.H * p.W * p.in_cs + g * 16;
    uint8_t* obase = out + ((long long)n * p.P * p.Q + q) * p.out_cs + g * 16;
    uint32_t R0[8], R1[8], R2[8];
    int h = p0 * SH - p.pt;   // first input row of output row p0
    bool v0 = (unsigned)h < (unsigned)p.H, v1 = (unsigned)(h + 1) < (unsigned)p.H,
         v2 = (unsigned)(h + 2) < (unsigned)p.H;
    p3_row<AVG>(base + (long long)h * p.W * p.in_cs, p.in_cs, w0, p.W, v0, bias, R0);
    p3_row<AVG>(base + (long long)(h + 1) * p.W * p.in_cs, p.in_cs, w0, p.W, v1, bias, R1);
    p3_row<AVG>(base + (long long)(h + 2) * p.W * p.in_cs, p.in_cs, w0, p.W, v2, bias, R2);
    for (int pp = p0; pp < p1; ++pp) {
      if (pp > p0) {   // slide the window SH input rows down
        h += SH;
        if (SH == 1) {
#pragma unroll
          for (int k = 0; k < 8; ++k) {
            R0[k] = R1[k];
            R1[k] = R2[k];
          }
          v0 = v1;
          v1 = v2;
          v2 = (unsigned)(h + 2) < (unsigned)p.H;
          p3_row<AVG>(base + (long long)(h + 2) * p.W * p.in_cs, p.in_cs, w0, p.W, v2, bias, R2);
        } else {
#pragma unroll
          for (int k = 0; k < 8; ++k) R0[k] = R2[k];
          v0 = v2;
          v1 = (unsigned)(h + 1) < (unsigned)p.H;
          v2 = (unsigned)(h + 2) < (unsigned)p.H;
          p3_row<AVG>(base + (long long)(h + 1) * p.W * p.in_cs, p.in_cs, w0, p.W, v1, bias, R1);
          p3_row<AVG>(base + (long long)(h + 2) * p.W * p.in_cs, p.in_cs, w0, p.W, v2, bias, R2);
        }
      }
      uint32_t ow[4];
      if (AVG) {
        const int cnt = ((int)v0 + (int)v1 + (int)v2) * cols;
        const uint32_t mag = div_magic(2u * (uint32_t)(cnt > 0 ? cnt : 1));
#pragma unroll
        for (int k = 0; k < 4; ++k) {
          const uint32_t slo = __vadd2(__vadd2(R0[k], R1[k]), R2[k]), shi = __vadd2(__vadd2(R0[k + 4], R1[k + 4]), R2[k + 4]);
          uint32_t bytes = 0;
#pragma unroll
          for (int j = 0; j < 4; ++j) {   // byte j of the word: lane j >> 1 of lo (even j) / hi (odd j)
            const uint32_t word = (j & 1) ? shi : slo;
            int32_t sum = (int32_t)((word >> (16 * (j >> 1))) & 0xFFFFu);
            if (S8) sum -= 128 * cnt;
            int32_t y = 0;
            if (cnt > 0) {
              const uint32_t a = (uint32_t)(sum < 0 ? -sum : sum);
              const int32_t m = (int32_t)div_small(2u * a + (uint32_t)cnt, mag);
              y = sum < 0 ? -m : m;
            }
            bytes |= ((uint32_t)y & 0xFFu) << (8 * j);
          }
          ow[k] = bytes;
        }
      } else {
#pragma unroll
        for (int k = 0; k < 4; ++k) {
          const uint32_t mlo = __vmaxu2(__vmaxu2(R0[k], R1[k]), R2[k]), mhi = __vmaxu2(__vmaxu2(R0[k + 4], R1[k + 4]), R2[k + 4]);
          ow[k] = (mlo | (mhi << 8)) ^ bias;
        }
      }
      *reinterpret_cast<uint4*>(obase + (long long)pp * p.Q * p.out_cs) = make_uint4(ow[0], ow[1], ow[2], ow[3]);
    }
  }
}

cudaError_t launch_pool(const PoolParams& p, cudaStream_t s) {
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const bool v16 = p.C % 16 == 0 && p.in_cs % 16 == 0 && p.out_cs % 16 == 0 &&
                   ((reinterpret_cast<uintptr_t>(p.in) | reinterpret_cast<uintptr_t>(p.out)) & 15) == 0;
  // fast path: every window has a valid tap (pad < window, checked by the ABI), sums of at
  // most 128 taps fit the 16-bit lanes, and the work-item count fits 32 bits
  constexpr int kTQ = 4;
  const long long items = (long long)p.N * p.P * ((p.Q + kTQ - 1) / kTQ) * (p.C / 16);
  // 3x3, stride 1 / 2 (ResNet-50 stem max pool, Inception-v3 max / branch average pools): the
  // separable row-reduction kernel (QNN_POOL_NO3=1 keeps pool16, A/B measurements)
  static const bool no3 = std::getenv("QNN_POOL_NO3") != nullptr;
  const long long items3 = (long long)p.N * ((p.P + kP3Band - 1) / kP3Band) * p.Q * (p.C / 16);
  if (!no3 && v16 && p.R == 3 && p.S == 3 && p.sh == p.sw && (p.sh == 1 || p.sh == 2) && items3 < (1ll << 31)) {
    const int blocks = (int)std::max<long long>(1, std::min<long long>((items3 + 255) / 256, (long long)sms * 16));
    const FastDiv fdG = make_fastdiv((uint32_t)(p.C / 16)), fdQ = make_fastdiv((uint32_t)p.Q),
                  fdB = make_fastdiv((uint32_t)((p.P + kP3Band - 1) / kP3Band));
#define QNN_POOL3(S_, A_, H_) \
  if (p.s8 == S_ && p.avg == A_ && p.sh == H_) launch_pdl(pool3_kernel<S_, A_, H_>, dim3(blocks), dim3(256), 0, s, p, fdG, fdQ, fdB);
    QNN_POOL3(false, false, 1) QNN_POOL3(false, true, 1) QNN_POOL3(true, false, 1) QNN_POOL3(true, true, 1)
    QNN_POOL3(false, false, 2) QNN_POOL3(false, true, 2) QNN_POOL3(true, false, 2) QNN_POOL3(true, true, 2)
#undef QNN_POOL3
    count_launch();
    return cudaGetLastError();
  }
  if (v16 && p.R * p.S <= 128 && items < (1ll << 31)) {
    const int blocks = (int)std::max<long long>(1, std::min<long long>((items + 255) / 256, (long long)sms * 16));
    const FastDiv fdG = make_fastdiv((uint32_t)(p.C / 16)), fdQB = make_fastdiv((uint32_t)((p.Q + kTQ - 1) / kTQ)),
                  fdP = make_fastdiv((uint32_t)p.P);
#define QNN_POOL16(S_, A_) \
  if (p.s8 == S_ && p.avg == A_) launch_pdl(pool16_kernel<S_, A_, kTQ>, dim3(blocks), dim3(256), 0, s, p, fdG, fdQB, fdP);
    QNN_POOL16(false, false) QNN_POOL16(false, true) QNN_POOL16(true, false) QNN_POOL16(true, true)
#undef QNN_POOL16
    count_launch();
    return cudaGetLastError();
  }
  const long long total = (long long)p.N * p.P * p.Q * (v16 ? p.C / 16 : p.C);
  const int blocks = (int)std::max<long long>(1, std::min<long long>((total + 255) / 256, (long long)sms * 16));
#define QNN_POOL(V_, S_, A_) \
  if ((v16 ? 16 : 1) == V_ && p.s8 == S_ && p.avg == A_) launch_pdl(pool_kernel<V_, S_, A_>, dim3(blocks), dim3(256), 0, s, p);
  QNN_POOL(16, false, false) QNN_POOL(16, false, true) QNN_POOL(16, true, false) QNN_POOL(16, true, true)
  QNN_POOL(1, false, false) QNN_POOL(1, false, true) QNN_POOL(1, true, false) QNN_POOL(1, true, true)
#undef QNN_POOL
  count_launch();
  return cudaGetLastError();
}

}  // namespace qnn
