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
    case DT_S8: requantize_kernel<IN, DT_S8><<<blocks, 256, 0, s>>>(p); break;
    case DT_U8: requantize_kernel<IN, DT_U8><<<blocks, 256, 0, s>>>(p); break;
    default: requantize_kernel<IN, DT_S32><<<blocks, 256, 0, s>>>(p); break;
  }
}

cudaError_t launch_requantize(const RequantParams& p, cudaStream_t s) {
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

cudaError_t launch_quantize(const QuantParams& p, cudaStream_t s) {
  const int blocks = ew_blocks((p.count + 15) / 16);
  if (p.q_dt == DT_S8)
    quantize_kernel<DT_S8><<<blocks, 256, 0, s>>>(p);
  else
    quantize_kernel<DT_U8><<<blocks, 256, 0, s>>>(p);
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

cudaError_t launch_dequantize(const QuantParams& p, cudaStream_t s) {
  const int blocks = ew_blocks((p.count + 15) / 16);
  switch (p.q_dt) {
    case DT_S8: dequantize_kernel<DT_S8><<<blocks, 256, 0, s>>>(p); break;
    case DT_U8: dequantize_kernel<DT_U8><<<blocks, 256, 0, s>>>(p); break;
    default: dequantize_kernel<DT_S32><<<blocks, 256, 0, s>>>(p); break;
  }
  count_launch();
  return cudaGetLastError();
}

}  // namespace qnn
