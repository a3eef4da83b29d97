// elementwise.cu — standalone qnn.requantize / qnn.quantize / qnn.dequantize
// (SURVEY §8a rows a7, a8).  Bandwidth-bound: every thread moves 16 elements
// per iteration with 16-byte vector loads/stores (grid-stride, grid sized to
// the SM count), per-channel parameters staged in shared memory.
//
//   requantize (Eq. 5): y = clamp(R(m_c (x - zp_in)) + zp_out)
//   quantize   (Eq. 1 inverted, reading R14): q = clamp(round_half_away(x / s_c) + zp_c)
//   dequantize (Eq. 1): x = fl32(s_c (q - zp_c))
#include "common.cuh"
#include "internal.h"

namespace qnn {

template <int DT>
struct Elem;
template <>
struct Elem<DT_S8> {
  using T = int8_t;
  static constexpr int kBytes = 1;
};
template <>
struct Elem<DT_U8> {
  using T = uint8_t;
  static constexpr int kBytes = 1;
};
template <>
struct Elem<DT_S32> {
  using T = int32_t;
  static constexpr int kBytes = 4;
};

// Load / store 16 consecutive elements (vectorised when the pointer is 16-B aligned)
template <int DT>
__device__ __forceinline__ void load16(const void* base, long long i, int64_t (&v)[16]) {
  using T = typename Elem<DT>::T;
  const T* p = reinterpret_cast<const T*>(base) + i;
  if (Elem<DT>::kBytes == 1) {
    const uint4 u = __ldg(reinterpret_cast<const uint4*>(p));
    const uint32_t w[4] = {u.x, u.y, u.z, u.w};
#pragma unroll
    for (int j = 0; j < 16; ++j) {
      const uint32_t b = (w[j >> 2] >> (8 * (j & 3))) & 0xFF;
      v[j] = DT == DT_S8 ? (int64_t)(int8_t)b : (int64_t)b;
    }
  } else {
#pragma unroll
    for (int j = 0; j < 16; j += 4) {
      const int4 u = __ldg(reinterpret_cast<const int4*>(p) + j / 4);
      v[j] = u.x;
      v[j + 1] = u.y;
      v[j + 2] = u.z;
      v[j + 3] = u.w;
    }
  }
}

template <int DT>
__device__ __forceinline__ int64_t load1(const void* base, long long i) {
  return (int64_t)(reinterpret_cast<const typename Elem<DT>::T*>(base)[i]);
}

template <int DT>
__device__ __forceinline__ void store16(void* base, long long i, const int32_t (&y)[16]) {
  using T = typename Elem<DT>::T;
  T* p = reinterpret_cast<T*>(base) + i;
  if (Elem<DT>::kBytes == 1) {
    uint32_t w[4];
#pragma unroll
    for (int j = 0; j < 4; ++j)
      w[j] = ((uint32_t)y[4 * j] & 0xFF) | (((uint32_t)y[4 * j + 1] & 0xFF) << 8) |
             (((uint32_t)y[4 * j + 2] & 0xFF) << 16) | (((uint32_t)y[4 * j + 3] & 0xFF) << 24);
    *reinterpret_cast<uint4*>(p) = make_uint4(w[0], w[1], w[2], w[3]);
  } else {
#pragma unroll
    for (int j = 0; j < 16; j += 4) reinterpret_cast<int4*>(p)[j / 4] = make_int4(y[j], y[j + 1], y[j + 2], y[j + 3]);
  }
}

template <int DT>
__device__ __forceinline__ void store1(void* base, long long i, int32_t y) {
  reinterpret_cast<typename Elem<DT>::T*>(base)[i] = (typename Elem<DT>::T)y;
}

__device__ __forceinline__ int grid_threads() { return gridDim.x * blockDim.x; }

// ------------------------------------------------------------------ requantize
template <int IN, int OUT>
__global__ void __launch_bounds__(256) requantize_kernel(const __grid_constant__ RequantParams p) {
  pdl_wait();      // inputs are the previous kernel's output (PDL launch; no early trigger: the
                   // next kernel's CTAs would take this multi-wave grid's slots while waiting)
  __shared__ int32_t s_mult[kMaxChanParams];
  __shared__ int8_t s_rsh[kMaxChanParams];
  for (int c = threadIdx.x; c < p.nch; c += blockDim.x) {
    s_mult[c] = p.mult[c];
    s_rsh[c] = p.rsh[c];
  }
  __syncthreads();
  const bool vec = ((reinterpret_cast<uintptr_t>(p.in) | reinterpret_cast<uintptr_t>(p.out)) & 15) == 0;
  const long long nvec = vec ? p.count / 16 : 0;
  for (long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x; t < nvec; t += grid_threads()) {
    const long long i0 = t * 16;
    int64_t x[16];
    load16<IN>(p.in, i0, x);
    long long ci = 0, cj = 0;
    if (p.nch > 1) {
      ci = (i0 / p.inner) % p.cext;
      cj = i0 % p.inner;
    }
    int32_t y[16];
#pragma unroll
    for (int j = 0; j < 16; ++j) {
      const int c = (int)ci;
      y[j] = rq_apply(x[j] - p.in_zp, s_mult[c], s_rsh[c], p.mode, p.out_zp, p.lo, p.hi);
      if (p.nch > 1 && ++cj == p.inner) {
        cj = 0;
        if (++ci == p.cext) ci = 0;
      }
    }
    store16<OUT>(p.out, i0, y);
  }
  for (long long i = nvec * 16 + blockIdx.x * (long long)blockDim.x + threadIdx.x; i < p.count; i += grid_threads()) {
    const int c = p.nch > 1 ? (int)((i / p.inner) % p.cext) : 0;
    store1<OUT>(p.out, i, rq_apply(load1<IN>(p.in, i) - p.in_zp, s_mult[c], s_rsh[c], p.mode, p.out_zp, p.lo, p.hi));
  }
}

static int ew_blocks(long long work_items) {
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const long long want = (work_items + 255) / 256;
  return (int)std::max<long long>(1, std::min<long long>(want, (long long)sms * 8));
}

template <int IN>
static void dispatch_rq_out(const RequantParams& p, int blocks, cudaStream_t s) {
  switch (p.out_dt) {
    case DT_S8: launch_pdl(requantize_kernel<IN, DT_S8>, dim3(blocks), dim3(256), 0, s, p); break;
    case DT_U8: launch_pdl(requantize_kernel<IN, DT_U8>, dim3(blocks), dim3(256), 0, s, p); break;
    default: launch_pdl(requantize_kernel<IN, DT_S32>, dim3(blocks), dim3(256), 0, s, p); break;
  }
}

static cudaError_t launch_requantize_generic(const RequantParams& p, cudaStream_t s) {
  const int blocks = ew_blocks((p.count + 15) / 16);
  switch (p.in_dt) {
    case DT_S8: dispatch_rq_out<DT_S8>(p, blocks, s); break;
    case DT_U8: dispatch_rq_out<DT_U8>(p, blocks, s); break;
    default: dispatch_rq_out<DT_S32>(p, blocks, s); break;
  }
  count_launch();
  return cudaGetLastError();
}

// ------------------------------------------------------------------ quantize
__device__ __forceinline__ int32_t quant1(float x, float s, int32_t zp, int32_t lo, int32_t hi) {
  const float t = __fdiv_rn(x, s);  // IEEE fp32 division (reading R14)
  if (t != t) return zp;            // NaN -> zero point
  float r = roundf(t);              // half away from zero
  r = fminf(fmaxf(r, -4.0e9f), 4.0e9f);
  long long y = (long long)r + zp;
  y = y < lo ? lo : y;
  y = y > hi ? hi : y;
  return (int32_t)y;
}

template <int OUT>
__global__ void __launch_bounds__(256) quantize_kernel(const __grid_constant__ QuantParams p) {
  pdl_wait();      // inputs are the previous kernel's output (PDL launch; no early trigger: the
                   // next kernel's CTAs would take this multi-wave grid's slots while waiting)
  __shared__ float s_sc[kMaxQuantParams];
  __shared__ int32_t s_zp[kMaxQuantParams];
  for (int c = threadIdx.x; c < p.nch; c += blockDim.x) {
    s_sc[c] = p.scale[c];
    s_zp[c] = p.zp[c];
  }
  __syncthreads();
  const float* in = reinterpret_cast<const float*>(p.in);
  const bool vec = ((reinterpret_cast<uintptr_t>(p.in) | reinterpret_cast<uintptr_t>(p.out)) & 15) == 0;
  const long long nvec = vec ? p.count / 16 : 0;
  for (long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x; t < nvec; t += grid_threads()) {
    const long long i0 = t * 16;
    float x[16];
#pragma unroll
    for (int j = 0; j < 16; j += 4) {
      const float4 v = __ldg(reinterpret_cast<const float4*>(in + i0) + j / 4);
      x[j] = v.x;
      x[j + 1] = v.y;
      x[j + 2] = v.z;
      x[j + 3] = v.w;
    }
    long long ci = 0, cj = 0;
    if (p.nch > 1) {
      ci = (i0 / p.inner) % p.cext;
      cj = i0 % p.inner;
    }
    int32_t y[16];
#pragma unroll
    for (int j = 0; j < 16; ++j) {
      const int c = (int)ci;
      y[j] = quant1(x[j], s_sc[c], s_zp[c], p.lo, p.hi);
      if (p.nch > 1 && ++cj == p.inner) {
        cj = 0;
        if (++ci == p.cext) ci = 0;
      }
    }
    store16<OUT>(p.out, i0, y);
  }
  for (long long i = nvec * 16 + blockIdx.x * (long long)blockDim.x + threadIdx.x; i < p.count; i += grid_threads()) {
    const int c = p.nch > 1 ? (int)((i / p.inner) % p.cext) : 0;
    store1<OUT>(p.out, i, quant1(in[i], s_sc[c], s_zp[c], p.lo, p.hi));
  }
}

static cudaError_t launch_quantize_generic(const QuantParams& p, cudaStream_t s) {
  const int blocks = ew_blocks((p.count + 15) / 16);
  if (p.q_dt == DT_S8)
    launch_pdl(quantize_kernel<DT_S8>, dim3(blocks), dim3(256), 0, s, p);
  else
    launch_pdl(quantize_kernel<DT_U8>, dim3(blocks), dim3(256), 0, s, p);
  count_launch();
  return cudaGetLastError();
}

// ------------------------------------------------------------------ dequantize
template <int IN>
__device__ __forceinline__ float dequant1(int64_t q, float s, int32_t zp) {
  const int64_t d = q - zp;
  if (IN != DT_S32) {
    // |d| < 2^10: (float)d is exact, one rounding of the exact product
    return __fmul_rn((float)d, s);
  } else {
    // exact in double when |d| < 2^29; otherwise within 1 ulp of the single rounding
    return __double2float_rn(__dmul_rn((double)d, (double)s));
  }
}

template <int IN>
__global__ void __launch_bounds__(256) dequantize_kernel(const __grid_constant__ QuantParams p) {
  pdl_wait();      // inputs are the previous kernel's output (PDL launch; no early trigger: the
                   // next kernel's CTAs would take this multi-wave grid's slots while waiting)
  __shared__ float s_sc[kMaxQuantParams];
  __shared__ int32_t s_zp[kMaxQuantParams];
  for (int c = threadIdx.x; c < p.nch; c += blockDim.x) {
    s_sc[c] = p.scale[c];
    s_zp[c] = p.zp[c];
  }
  __syncthreads();
  float* out = reinterpret_cast<float*>(p.out);
  const bool vec = ((reinterpret_cast<uintptr_t>(p.in) | reinterpret_cast<uintptr_t>(p.out)) & 15) == 0;
  const long long nvec = vec ? p.count / 16 : 0;
  for (long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x; t < nvec; t += grid_threads()) {
    const long long i0 = t * 16;
    int64_t q[16];
    load16<IN>(p.in, i0, q);
    long long ci = 0, cj = 0;
    if (p.nch > 1) {
      ci = (i0 / p.inner) % p.cext;
      cj = i0 % p.inner;
    }
    float y[16];
#pragma unroll
    for (int j = 0; j < 16; ++j) {
      const int c = (int)ci;
      y[j] = dequant1<IN>(q[j], s_sc[c], s_zp[c]);
      if (p.nch > 1 && ++cj == p.inner) {
        cj = 0;
        if (++ci == p.cext) ci = 0;
      }
    }
#pragma unroll
    for (int j = 0; j < 16; j += 4)
      reinterpret_cast<float4*>(out + i0)[j / 4] = make_float4(y[j], y[j + 1], y[j + 2], y[j + 3]);
  }
  for (long long i = nvec * 16 + blockIdx.x * (long long)blockDim.x + threadIdx.x; i < p.count; i += grid_threads()) {
    const int c = p.nch > 1 ? (int)((i / p.inner) % p.cext) : 0;
    out[i] = dequant1<IN>(load1<IN>(p.in, i), s_sc[c], s_zp[c]);
  }
}

static cudaError_t launch_dequantize_generic(const QuantParams& p, cudaStream_t s) {
  const int blocks = ew_blocks((p.count + 15) / 16);
  switch (p.q_dt) {
    case DT_S8: launch_pdl(dequantize_kernel<DT_S8>, dim3(blocks), dim3(256), 0, s, p); break;
    case DT_U8: launch_pdl(dequantize_kernel<DT_U8>, dim3(blocks), dim3(256), 0, s, p); break;
    default: launch_pdl(dequantize_kernel<DT_S32>, dim3(blocks), dim3(256), 0, s, p); break;
  }
  count_launch();
  return cudaGetLastError();
}

// =========================================================================
// Fast paths.  Channel modes:
//   CM_TENSOR : one parameter set (registers)
//   CM_VEC    : inner % 16 == 0, so the 16 elements of a vector share one channel
//   CM_LAST   : inner == 1 and cext % 16 == 0 (channel is the fastest axis, e.g. NHWC
//               per-channel): each thread keeps the same 16 channels for its whole
//               grid-stride walk (grid * block is a multiple of cext / 16), so the 16
//               parameter sets live in registers.
// Anything else (or a shift outside the fast range) takes the generic kernels above.
// =========================================================================
enum { CM_TENSOR = 0, CM_VEC = 1, CM_LAST = 2 };

__device__ __forceinline__ uint32_t pack4_sat(int a, int b, int c, int d, bool s8) {
  uint32_t o;
  if (s8)
    asm("{\n\t.reg .u32 t;\n\tcvt.pack.sat.s8.s32.b32 t, %4, %3, 0;\n\tcvt.pack.sat.s8.s32.b32 %0, %2, %1, t;\n\t}"
        : "=r"(o) : "r"(a), "r"(b), "r"(c), "r"(d));
  else
    asm("{\n\t.reg .u32 t;\n\tcvt.pack.sat.u8.s32.b32 t, %4, %3, 0;\n\tcvt.pack.sat.u8.s32.b32 %0, %2, %1, t;\n\t}"
        : "=r"(o) : "r"(a), "r"(b), "r"(c), "r"(d));
  return o;
}

// raw input values (no zero point applied) of 16 consecutive elements
template <int DT>
__device__ __forceinline__ void load16_raw(const void* base, long long i, int32_t (&v)[16]) {
  if (DT == DT_S32) {
    const int4* p = reinterpret_cast<const int4*>(reinterpret_cast<const int32_t*>(base) + i);
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const int4 u = __ldg(p + j);
      v[4 * j] = u.x; v[4 * j + 1] = u.y; v[4 * j + 2] = u.z; v[4 * j + 3] = u.w;
    }
  } else {
    const uint4 u = __ldg(reinterpret_cast<const uint4*>(reinterpret_cast<const uint8_t*>(base) + i));
    const uint32_t w[4] = {u.x, u.y, u.z, u.w};
#pragma unroll
    for (int j = 0; j < 16; ++j) {
      const uint32_t b = (w[j >> 2] >> (8 * (j & 3))) & 0xFFu;
      v[j] = DT == DT_S8 ? (int32_t)(int8_t)b : (int32_t)b;
    }
  }
}

// 16 results -> 8-bit (saturating pack) or int32
template <int DT>
__device__ __forceinline__ void store16_sat(void* base, long long i, const int32_t (&y)[16]) {
  if (DT == DT_S32) {
    int4* p = reinterpret_cast<int4*>(reinterpret_cast<int32_t*>(base) + i);
#pragma unroll
    for (int j = 0; j < 4; ++j) p[j] = make_int4(y[4 * j], y[4 * j + 1], y[4 * j + 2], y[4 * j + 3]);
  } else {
    uint32_t w[4];
#pragma unroll
    for (int j = 0; j < 4; ++j) w[j] = pack4_sat(y[4 * j], y[4 * j + 1], y[4 * j + 2], y[4 * j + 3], DT == DT_S8);
    *reinterpret_cast<uint4*>(reinterpret_cast<uint8_t*>(base) + i) = make_uint4(w[0], w[1], w[2], w[3]);
  }
}

// Warp-interleaved 512-element units: lane t of a warp handles, for j = 0..3, the four
// consecutive elements u*512 + j*128 + 4t .. +3 (register v[4j + k]).  Every load and
// store instruction of the warp then covers one contiguous span (128 B for 8-bit data,
// 512 B for 32-bit data): whole sectors, no partial-sector writes.
// With W16 (8-bit in and out) lane t instead takes the 16 contiguous elements
// u*512 + 16t .. +15 (one 16-B access per lane, 512 B per warp instruction).
template <bool W16>
__device__ __forceinline__ long long il_elem(long long u, int j, int lane) {
  return W16 ? u * 512 + 16 * lane + 4 * j : u * 512 + j * 128 + 4 * lane;
}
template <int DT, bool W16 = false>
__device__ __forceinline__ void load_il(const void* base, long long u, int lane, int32_t (&v)[16]) {
  if (W16 && DT != DT_S32) {
    const uint4 w4 = __ldg(reinterpret_cast<const uint4*>(reinterpret_cast<const uint8_t*>(base) + u * 512 + 16 * lane));
    const uint32_t ws[4] = {w4.x, w4.y, w4.z, w4.w};
#pragma unroll
    for (int j = 0; j < 16; ++j) {
      const uint32_t b = (ws[j >> 2] >> (8 * (j & 3))) & 0xFFu;
      v[j] = DT == DT_S8 ? (int32_t)(int8_t)b : (int32_t)b;
    }
    return;
  }
#pragma unroll
  for (int j = 0; j < 4; ++j) {
    const long long e = u * 512 + j * 128 + 4 * lane;
    if (DT == DT_S32) {
      const int4 w = __ldg(reinterpret_cast<const int4*>(reinterpret_cast<const int32_t*>(base) + e));
      v[4 * j] = w.x; v[4 * j + 1] = w.y; v[4 * j + 2] = w.z; v[4 * j + 3] = w.w;
    } else {
      const uint32_t w = __ldg(reinterpret_cast<const uint32_t*>(reinterpret_cast<const uint8_t*>(base) + e));
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        const uint32_t b = (w >> (8 * k)) & 0xFFu;
        v[4 * j + k] = DT == DT_S8 ? (int32_t)(int8_t)b : (int32_t)b;
      }
    }
  }
}
template <int DT, bool W16 = false>
__device__ __forceinline__ void store_il_sat(void* base, long long u, int lane, const int32_t (&y)[16]) {
  if (W16 && DT != DT_S32) {
    uint32_t w[4];
#pragma unroll
    for (int j = 0; j < 4; ++j) w[j] = pack4_sat(y[4 * j], y[4 * j + 1], y[4 * j + 2], y[4 * j + 3], DT == DT_S8);
    *reinterpret_cast<uint4*>(reinterpret_cast<uint8_t*>(base) + u * 512 + 16 * lane) = make_uint4(w[0], w[1], w[2], w[3]);
    return;
  }
#pragma unroll
  for (int j = 0; j < 4; ++j) {
    const long long e = u * 512 + j * 128 + 4 * lane;
    if (DT == DT_S32)
      *reinterpret_cast<int4*>(reinterpret_cast<int32_t*>(base) + e) =
          make_int4(y[4 * j], y[4 * j + 1], y[4 * j + 2], y[4 * j + 3]);
    else
      *reinterpret_cast<uint32_t*>(reinterpret_cast<uint8_t*>(base) + e) =
          pack4_sat(y[4 * j], y[4 * j + 1], y[4 * j + 2], y[4 * j + 3], DT == DT_S8);
  }
}
__device__ __forceinline__ void load_il_f32(const float* base, long long u, int lane, float (&v)[16]) {
#pragma unroll
  for (int j = 0; j < 4; ++j) {
    const float4 w = __ldg(reinterpret_cast<const float4*>(base + u * 512 + j * 128 + 4 * lane));
    v[4 * j] = w.x; v[4 * j + 1] = w.y; v[4 * j + 2] = w.z; v[4 * j + 3] = w.w;
  }
}
__device__ __forceinline__ void store_il_f32(float* base, long long u, int lane, const float (&y)[16]) {
#pragma unroll
  for (int j = 0; j < 4; ++j)
    *reinterpret_cast<float4*>(base + u * 512 + j * 128 + 4 * lane) =
        make_float4(y[4 * j], y[4 * j + 1], y[4 * j + 2], y[4 * j + 3]);
}
// channel of element group j (CM_VEC: inner % 4 == 0, so the four elements share it)
template <bool W16 = false>
__device__ __forceinline__ int il_channel(long long u, int j, int lane, long long inner, int cext) {
  return (int)((il_elem<W16>(u, j, lane) / inner) % cext);
}

// ---- requantize: one channel's parameters for the 64-bit fast form.
//   UPWARD   : y = (x*M + c) >> rsh,   c = 2^(rsh-1) + zp_out*2^rsh - zp_in*M   (x raw)
//   TONEAREST: y = sign(d) * ((|d|*M + c) >> rsh) + zp_out,  d = x - zp_in, c = 2^(rsh-1)
// Both equal rq_apply exactly while no intermediate overflows: |x*M| < 2^62 and
// rsh <= 52 keep every sum below 2^63 (fast range checked on the host).
struct RqCh {
  int32_t M, rsh;
  long long c;
};
template <int MODE>
__device__ __forceinline__ RqCh rq_ch(const RequantParams& p, int ch) {
  RqCh q;
  q.M = p.mult[ch];
  q.rsh = p.rsh[ch];
  if (q.M == 0) q.rsh = 32;   // multiplier rounds to 0 (R15): y = zp_out
  const long long half = 1ll << (q.rsh - 1);
  q.c = MODE == RND_UPWARD ? half + (long long)p.out_zp * (1ll << q.rsh) - (long long)p.in_zp * q.M : half;
  return q;
}
template <int MODE>
__device__ __forceinline__ int32_t rq_fast(int32_t x, const RqCh& q, int32_t zp_in, int32_t zp_out) {
  if (MODE == RND_UPWARD) {
    return (int32_t)(((long long)x * q.M + q.c) >> q.rsh);
  } else {
    const int32_t d = x - zp_in;   // s32 inputs take this path only with zp_in == 0
    const uint32_t a = d < 0 ? 0u - (uint32_t)d : (uint32_t)d;
    const int32_t m = (int32_t)(((unsigned long long)a * (uint32_t)q.M + (unsigned long long)q.c) >> q.rsh);
    return (d < 0 ? -m : m) + zp_out;
  }
}

template <int IN, int OUT, int MODE, int CM>
__global__ void __launch_bounds__(256) requantize_fast_kernel(const __grid_constant__ RequantParams p) {
  pdl_wait();      // inputs are the previous kernel's output (PDL launch; no early trigger: the
                   // next kernel's CTAs would take this multi-wave grid's slots while waiting)
  const long long nthreads = (long long)gridDim.x * blockDim.x;
  const long long tid = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (CM == CM_LAST) {
    const int G = p.cext >> 4;
    const int g = (int)(tid % G);
    const long long rows = p.count / p.cext, rstride = nthreads / G;
    RqCh q[16];
#pragma unroll
    for (int j = 0; j < 16; ++j) q[j] = rq_ch<MODE>(p, g * 16 + j);
    for (long long r = tid / G; r < rows; r += rstride) {
      const long long i0 = r * p.cext + g * 16;
      int32_t x[16], y[16];
      load16_raw<IN>(p.in, i0, x);
#pragma unroll
      for (int j = 0; j < 16; ++j) y[j] = rq_fast<MODE>(x[j], q[j], p.in_zp, p.out_zp);
      store16_sat<OUT>(p.out, i0, y);
    }
    return;
  }
  const int lane = threadIdx.x & 31;
  const long long nunits = p.count >> 9, gw = tid >> 5, nw = nthreads >> 5;
  const RqCh q0 = rq_ch<MODE>(p, 0);
  constexpr bool W16 = IN != DT_S32 && OUT != DT_S32;
  // 8-bit inputs: two units per iteration, both loads issued before any math (one 16-B load
  // per lane per unit is too little memory-level parallelism for HBM at one resident wave)
  constexpr int UN = IN == DT_S32 ? 1 : 2;
  long long u = gw;
  for (; u + (UN - 1) * nw < nunits; u += UN * nw) {
    int32_t x[UN][16], y[16];
#pragma unroll
    for (int v = 0; v < UN; ++v) load_il<IN, W16>(p.in, u + v * nw, lane, x[v]);
#pragma unroll
    for (int v = 0; v < UN; ++v) {
      const long long uu = u + v * nw;
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        const RqCh q = CM == CM_VEC ? rq_ch<MODE>(p, il_channel<W16>(uu, j, lane, p.inner, p.cext)) : q0;
#pragma unroll
        for (int k = 0; k < 4; ++k) y[4 * j + k] = rq_fast<MODE>(x[v][4 * j + k], q, p.in_zp, p.out_zp);
      }
      store_il_sat<OUT, W16>(p.out, uu, lane, y);
    }
  }
  for (; u < nunits; u += nw) {
    int32_t x[16], y[16];
    load_il<IN, W16>(p.in, u, lane, x);
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const RqCh q = CM == CM_VEC ? rq_ch<MODE>(p, il_channel<W16>(u, j, lane, p.inner, p.cext)) : q0;
#pragma unroll
      for (int k = 0; k < 4; ++k) y[4 * j + k] = rq_fast<MODE>(x[4 * j + k], q, p.in_zp, p.out_zp);
    }
    store_il_sat<OUT, W16>(p.out, u, lane, y);
  }
  // tail: the last count % 512 elements, one per thread
  for (long long i = (nunits << 9) + tid; i < p.count; i += nthreads) {
    int32_t x;
    if (IN == DT_S32) x = reinterpret_cast<const int32_t*>(p.in)[i];
    else if (IN == DT_S8) x = reinterpret_cast<const int8_t*>(p.in)[i];
    else x = reinterpret_cast<const uint8_t*>(p.in)[i];
    const RqCh q = CM == CM_VEC ? rq_ch<MODE>(p, (int)((i / p.inner) % p.cext)) : q0;
    int32_t y = rq_fast<MODE>(x, q, p.in_zp, p.out_zp);
    if (OUT != DT_S32) y = min(max(y, p.lo), p.hi);
    store1<OUT>(p.out, i, y);
  }
}

// channel mode of an elementwise launch (-1: generic kernel)
static int channel_mode(long long count, long long inner, int cext, int nch, const void* in, const void* out) {
  const bool a16 = ((reinterpret_cast<uintptr_t>(in) | reinterpret_cast<uintptr_t>(out)) & 15) == 0;
  if (!a16) return -1;
  if (nch == 1) return CM_TENSOR;
  if (inner % 4 == 0) return CM_VEC;
  if (inner == 1 && cext % 16 == 0) return CM_LAST;
  return -1;
}

// grid for the fast kernels: ~4 waves of 256-thread blocks; CM_LAST needs a thread
// count that is a multiple of the channel-group count G = cext / 16
static int fast_blocks(long long vectors, int cm, int cext) {
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  // one resident wave (8 x 256 threads per SM at <= 32 registers); threads grid-stride
  long long b = std::max<long long>(1, std::min<long long>((vectors + 255) / 256, (long long)sms * 8));
  if (cm == CM_LAST) {
    const int G = cext / 16;
    int gg = G, t = 256;   // blocks must be a multiple of G / gcd(G, 256)
    while (t) { const int r = gg % t; gg = t; t = r; }
    const int unit = G / gg;
    b = (b + unit - 1) / unit * unit;
  }
  return (int)b;
}

template <int IN, int OUT, int MODE>
static void launch_rq_cm(const RequantParams& p, int cm, int blocks, cudaStream_t s) {
  if (cm == CM_TENSOR) launch_pdl(requantize_fast_kernel<IN, OUT, MODE, CM_TENSOR>, dim3(blocks), dim3(256), 0, s, p);
  else if (cm == CM_VEC) launch_pdl(requantize_fast_kernel<IN, OUT, MODE, CM_VEC>, dim3(blocks), dim3(256), 0, s, p);
  else launch_pdl(requantize_fast_kernel<IN, OUT, MODE, CM_LAST>, dim3(blocks), dim3(256), 0, s, p);
}
template <int IN, int OUT>
static void launch_rq_mode(const RequantParams& p, int cm, int blocks, cudaStream_t s) {
  if (p.mode == RND_UPWARD) launch_rq_cm<IN, OUT, RND_UPWARD>(p, cm, blocks, s);
  else launch_rq_cm<IN, OUT, RND_TONEAREST>(p, cm, blocks, s);
}
template <int IN>
static void launch_rq_out(const RequantParams& p, int cm, int blocks, cudaStream_t s) {
  if (p.out_dt == DT_S8) launch_rq_mode<IN, DT_S8>(p, cm, blocks, s);
  else if (p.out_dt == DT_U8) launch_rq_mode<IN, DT_U8>(p, cm, blocks, s);
  else launch_rq_mode<IN, DT_S32>(p, cm, blocks, s);
}

cudaError_t launch_requantize(const RequantParams& p, cudaStream_t s) {
  int cm = channel_mode(p.count, p.inner, p.cext, p.nch, p.in, p.out);
  // fast range: 8-bit inputs |x*M| < 2^40 need rsh >= 11 for an int32 result; int32 inputs
  // need zp_in == 0 and rsh >= 32; rsh <= 52 keeps zp_out*2^rsh small (see rq_ch)
  const int rmin = p.in_dt == DT_S32 ? 32 : 11;
  if (p.in_dt == DT_S32 && p.in_zp != 0) cm = -1;
  for (int c = 0; cm >= 0 && c < p.nch; ++c)
    if (p.mult[c] != 0 && (p.rsh[c] < rmin || p.rsh[c] > 52)) cm = -1;
  if (cm < 0) return launch_requantize_generic(p, s);
  const int blocks = fast_blocks(p.count / 16, cm, p.cext);
  switch (p.in_dt) {
    case DT_S8: launch_rq_out<DT_S8>(p, cm, blocks, s); break;
    case DT_U8: launch_rq_out<DT_U8>(p, cm, blocks, s); break;
    default: launch_rq_out<DT_S32>(p, cm, blocks, s); break;
  }
  count_launch();
  return cudaGetLastError();
}

// ---- quantize: q = sat(round_half_away(fl32(x / s)) + zp), NaN -> zp (reading R14).
// r + zp is exact in fp32 whenever the result can land inside the 8-bit range, larger
// magnitudes saturate either way; the f32 -> s32 conversion saturates (+-inf included).
// x / s correctly rounded from the correctly rounded reciprocal rs = RN(1/s) by one
// Markstein correction: q0 = RN(x*rs) is within 1 ulp of x/s, the remainder x - s*q0 is
// exact (FMA), and RN(q0 + rem*rs) = RN(x/s) (no overflow/underflow of the quotient;
// tiny or huge quotients round or saturate identically).  x = +-inf gives rem = NaN:
// keep q0 = +-inf.  x = NaN stays NaN -> zp.
__device__ __forceinline__ float div_rn_markstein(float x, float s, float rs) {
  const float q0 = __fmul_rn(x, rs);
  const float rem = __fmaf_rn(-q0, s, x);
  const float q = __fmaf_rn(rem, rs, q0);
  return q != q ? q0 : q;
}
__device__ __forceinline__ int32_t quant_fast(float x, float s, float rs, float zpf, int32_t zp) {
  const float t = div_rn_markstein(x, s, rs);
  const int32_t y = __float2int_rz(roundf(t) + zpf);
  return t != t ? zp : y;
}
template <int OUT, int CM>
__global__ void __launch_bounds__(256) quantize_fast_kernel(const __grid_constant__ QuantParams p) {
  pdl_wait();      // inputs are the previous kernel's output (PDL launch; no early trigger: the
                   // next kernel's CTAs would take this multi-wave grid's slots while waiting)
  const long long nthreads = (long long)gridDim.x * blockDim.x;
  const long long tid = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  const float* in = reinterpret_cast<const float*>(p.in);
  auto load = [&](long long i0, float (&x)[16]) {
#pragma unroll
    for (int j = 0; j < 16; j += 4) {
      const float4 v = __ldg(reinterpret_cast<const float4*>(in + i0) + j / 4);
      x[j] = v.x; x[j + 1] = v.y; x[j + 2] = v.z; x[j + 3] = v.w;
    }
  };
  if (CM == CM_LAST) {
    const int G = p.cext >> 4;
    const int g = (int)(tid % G);
    const long long rows = p.count / p.cext, rstride = nthreads / G;
    float sc[16], rs[16], zf[16];
    int32_t zp[16];
#pragma unroll
    for (int j = 0; j < 16; ++j) {
      sc[j] = p.scale[g * 16 + j];
      rs[j] = __frcp_rn(sc[j]);
      zp[j] = p.zp[g * 16 + j];
      zf[j] = (float)zp[j];
    }
    for (long long r = tid / G; r < rows; r += rstride) {
      const long long i0 = r * p.cext + g * 16;
      float x[16];
      int32_t y[16];
      load(i0, x);
#pragma unroll
      for (int j = 0; j < 16; ++j) y[j] = quant_fast(x[j], sc[j], rs[j], zf[j], zp[j]);
      store16_sat<OUT>(p.out, i0, y);
    }
    return;
  }
  const int lane = threadIdx.x & 31;
  const long long nunits = p.count >> 9, gw = tid >> 5, nw = nthreads >> 5;
  for (long long u = gw; u < nunits; u += nw) {
    float x[16];
    int32_t y[16];
    load_il_f32(in, u, lane, x);
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const int ch = CM == CM_VEC ? il_channel(u, j, lane, p.inner, p.cext) : 0;
      const float sc = p.scale[ch], rs = __frcp_rn(sc), zf = (float)p.zp[ch];
      const int32_t zp = p.zp[ch];
#pragma unroll
      for (int k = 0; k < 4; ++k) y[4 * j + k] = quant_fast(x[4 * j + k], sc, rs, zf, zp);
    }
    store_il_sat<OUT>(p.out, u, lane, y);
  }
  for (long long i = (nunits << 9) + tid; i < p.count; i += nthreads) {
    const int ch = CM == CM_VEC ? (int)((i / p.inner) % p.cext) : 0;
    const int32_t y = quant_fast(in[i], p.scale[ch], __frcp_rn(p.scale[ch]), (float)p.zp[ch], p.zp[ch]);
    store1<OUT>(p.out, i, min(max(y, p.lo), p.hi));
  }
}

cudaError_t launch_quantize(const QuantParams& p, cudaStream_t s) {
  const int cm = channel_mode(p.count, p.inner, p.cext, p.nch, p.in, p.out);
  if (cm < 0) return launch_quantize_generic(p, s);
  const int blocks = fast_blocks(p.count / 16, cm, p.cext);
#define QNN_QF(OUT_)                                                                        \
  if (cm == CM_TENSOR) launch_pdl(quantize_fast_kernel<OUT_, CM_TENSOR>, dim3(blocks), dim3(256), 0, s, p);     \
  else if (cm == CM_VEC) launch_pdl(quantize_fast_kernel<OUT_, CM_VEC>, dim3(blocks), dim3(256), 0, s, p);      \
  else launch_pdl(quantize_fast_kernel<OUT_, CM_LAST>, dim3(blocks), dim3(256), 0, s, p);
  if (p.q_dt == DT_S8) {
    QNN_QF(DT_S8)
  } else {
    QNN_QF(DT_U8)
  }
#undef QNN_QF
  count_launch();
  return cudaGetLastError();
}

// ---- dequantize (8-bit): x = fl32((q - zp) * s), one rounding of an exact product
template <int IN, int CM>
__global__ void __launch_bounds__(256) dequantize_fast_kernel(const __grid_constant__ QuantParams p) {
  pdl_wait();      // inputs are the previous kernel's output (PDL launch; no early trigger: the
                   // next kernel's CTAs would take this multi-wave grid's slots while waiting)
  const long long nthreads = (long long)gridDim.x * blockDim.x;
  const long long tid = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  float* out = reinterpret_cast<float*>(p.out);
  auto store = [&](long long i0, const float (&y)[16]) {
#pragma unroll
    for (int j = 0; j < 16; j += 4)
      reinterpret_cast<float4*>(out + i0)[j / 4] = make_float4(y[j], y[j + 1], y[j + 2], y[j + 3]);
  };
  if (CM == CM_LAST) {
    const int G = p.cext >> 4;
    const int g = (int)(tid % G);
    const long long rows = p.count / p.cext, rstride = nthreads / G;
    float sc[16];
    int32_t zp[16];
#pragma unroll
    for (int j = 0; j < 16; ++j) {
      sc[j] = p.scale[g * 16 + j];
      zp[j] = p.zp[g * 16 + j];
    }
    for (long long r = tid / G; r < rows; r += rstride) {
      const long long i0 = r * p.cext + g * 16;
      int32_t q[16];
      float y[16];
      load16_raw<IN>(p.in, i0, q);
#pragma unroll
      for (int j = 0; j < 16; ++j) y[j] = __fmul_rn((float)(q[j] - zp[j]), sc[j]);
      store(i0, y);
    }
    return;
  }
  const int lane = threadIdx.x & 31;
  const long long nunits = p.count >> 9, gw = tid >> 5, nw = nthreads >> 5;
  for (long long u = gw; u < nunits; u += nw) {
    int32_t q[16];
    float y[16];
    load_il<IN>(p.in, u, lane, q);
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const int ch = CM == CM_VEC ? il_channel(u, j, lane, p.inner, p.cext) : 0;
      const float sc = p.scale[ch];
      const int32_t zp = p.zp[ch];
#pragma unroll
      for (int k = 0; k < 4; ++k) y[4 * j + k] = __fmul_rn((float)(q[4 * j + k] - zp), sc);
    }
    store_il_f32(out, u, lane, y);
  }
  for (long long i = (nunits << 9) + tid; i < p.count; i += nthreads) {
    const int ch = CM == CM_VEC ? (int)((i / p.inner) % p.cext) : 0;
    const int32_t q = IN == DT_S8 ? (int32_t)reinterpret_cast<const int8_t*>(p.in)[i]
                                  : (int32_t)reinterpret_cast<const uint8_t*>(p.in)[i];
    out[i] = __fmul_rn((float)(q - p.zp[ch]), p.scale[ch]);
  }
}

cudaError_t launch_dequantize(const QuantParams& p, cudaStream_t s) {
  const int cm = p.q_dt == DT_S32 ? -1 : channel_mode(p.count, p.inner, p.cext, p.nch, p.in, p.out);
  if (cm < 0) return launch_dequantize_generic(p, s);
  const int blocks = fast_blocks(p.count / 16, cm, p.cext);
#define QNN_DQ(IN_)                                                                          \
  if (cm == CM_TENSOR) launch_pdl(dequantize_fast_kernel<IN_, CM_TENSOR>, dim3(blocks), dim3(256), 0, s, p);     \
  else if (cm == CM_VEC) launch_pdl(dequantize_fast_kernel<IN_, CM_VEC>, dim3(blocks), dim3(256), 0, s, p);      \
  else launch_pdl(dequantize_fast_kernel<IN_, CM_LAST>, dim3(blocks), dim3(256), 0, s, p);
  if (p.q_dt == DT_S8) {
    QNN_DQ(DT_S8)
  } else {
    QNN_DQ(DT_U8)
  }
#undef QNN_DQ
  count_launch();
  return cudaGetLastError();
}

}  // namespace qnn
