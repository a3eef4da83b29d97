// depthwise.cu — quantized depthwise conv2d on CUDA cores.
//
// out[n,p,q,c] = requantize( sum_{valid r,s} (A[n,h,w,c] - zp_A) * (W[r,s,c] - zp_W) + bias[c] )
// using the paper's alternative "subtract zero points first" lowering,
// which is bit-identical to Eq. 3 and natural on CUDA cores (no tensor-core
// shape: each output reads only R*S inputs).  Padded taps contribute exactly 0,
// which is the zp_A padding of P:259.  W - zp_W is folded at prepack (int16).
// Each thread owns VEC consecutive channels of one output pixel (16-byte
// loads/stores when C % 16 == 0), threads of a warp walk consecutive channel
// groups, so every tap load is a coalesced row segment.  HBM-bound.
#include "common.cuh"
#include "internal.h"

namespace qnn {

template <int VEC>
struct VecLoad;
template <>
struct VecLoad<16> {
  __device__ static void load(const uint8_t* p, uint8_t (&b)[16]) {
    const uint4 v = __ldg(reinterpret_cast<const uint4*>(p));
    const uint32_t w[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
    for (int i = 0; i < 16; ++i) b[i] = (uint8_t)(w[i >> 2] >> (8 * (i & 3)));
  }
  __device__ static void store(uint8_t* p, const uint8_t (&b)[16]) {
    uint32_t w[4];
#pragma unroll
    for (int i = 0; i < 4; ++i)
      w[i] = (uint32_t)b[4 * i] | ((uint32_t)b[4 * i + 1] << 8) | ((uint32_t)b[4 * i + 2] << 16) |
             ((uint32_t)b[4 * i + 3] << 24);
    *reinterpret_cast<uint4*>(p) = make_uint4(w[0], w[1], w[2], w[3]);
  }
};
template <>
struct VecLoad<4> {
  __device__ static void load(const uint8_t* p, uint8_t (&b)[4]) {
    const uint32_t w = __ldg(reinterpret_cast<const uint32_t*>(p));
#pragma unroll
    for (int i = 0; i < 4; ++i) b[i] = (uint8_t)(w >> (8 * i));
  }
  __device__ static void store(uint8_t* p, const uint8_t (&b)[4]) {
    *reinterpret_cast<uint32_t*>(p) =
        (uint32_t)b[0] | ((uint32_t)b[1] << 8) | ((uint32_t)b[2] << 16) | ((uint32_t)b[3] << 24);
  }
};
template <>
struct VecLoad<1> {
  __device__ static void load(const uint8_t* p, uint8_t (&b)[1]) { b[0] = __ldg(p); }
  __device__ static void store(uint8_t* p, const uint8_t (&b)[1]) { p[0] = b[0]; }
};

template <int VEC>
__global__ void __launch_bounds__(256) depthwise_kernel(const __grid_constant__ DwParams p) {
  const int ngroups = p.C / VEC;
  const long long total = (long long)p.N * p.P * p.Q * ngroups;
  for (long long idx = blockIdx.x * (long long)blockDim.x + threadIdx.x; idx < total;
       idx += (long long)gridDim.x * blockDim.x) {
    const int g = (int)(idx % ngroups);
    long long pix = idx / ngroups;
    const int q = (int)(pix % p.Q);
    const long long t = pix / p.Q;
    const int pp = (int)(t % p.P);
    const int n = (int)(t / p.P);
    const int c0 = g * VEC;
    int32_t acc[VEC];
#pragma unroll
    for (int i = 0; i < VEC; ++i) acc[i] = 0;
    const uint8_t* in = reinterpret_cast<const uint8_t*>(p.in);
    for (int r = 0; r < p.R; ++r) {
      const int h = pp * p.sh + r * p.dh - p.pt;
      if (h < 0 || h >= p.H) continue;
      for (int s = 0; s < p.S; ++s) {
        const int w = q * p.sw + s * p.dw - p.pl;
        if (w < 0 || w >= p.W) continue;
        uint8_t b[VEC];
        VecLoad<VEC>::load(in + (((long long)n * p.H + h) * p.W + w) * p.in_cstride + c0, b);
        const int16_t* wt = p.w + (long long)(r * p.S + s) * p.C + c0;
#pragma unroll
        for (int i = 0; i < VEC; ++i) {
          const int32_t a = p.a_signed ? (int32_t)(int8_t)b[i] : (int32_t)b[i];
          acc[i] += (a - p.zpA) * (int32_t)__ldg(&wt[i]);
        }
      }
    }
    uint8_t ob[VEC];
    int32_t yv[VEC];
#pragma unroll
    for (int i = 0; i < VEC; ++i) {
      const int c = c0 + i;
      const int32_t v = acc[i] + (p.bias ? __ldg(&p.bias[c]) : 0);
      yv[i] = p.requant ? rq_apply(v, __ldg(&p.mult[c]), __ldg(&p.rsh[c]), p.mode, p.zp_out, p.lo, p.hi) : v;
      ob[i] = (uint8_t)yv[i];
    }
    if (p.out_dtype == DT_S32) {
      int32_t* o = reinterpret_cast<int32_t*>(p.out) + pix * p.out_cstride + c0;
#pragma unroll
      for (int i = 0; i < VEC; ++i) o[i] = yv[i];
    } else {
      VecLoad<VEC>::store(reinterpret_cast<uint8_t*>(p.out) + pix * p.out_cstride + c0, ob);
    }
  }
}

cudaError_t launch_depthwise(const DwParams& p, cudaStream_t s) {
  const bool a16 = (reinterpret_cast<uintptr_t>(p.in) & 15) == 0 && (reinterpret_cast<uintptr_t>(p.out) & 15) == 0;
  const bool a4 = (reinterpret_cast<uintptr_t>(p.in) & 3) == 0 && (reinterpret_cast<uintptr_t>(p.out) & 3) == 0;
  int vec = 1;
  if (p.C % 16 == 0 && p.in_cstride % 16 == 0 && p.out_cstride % 16 == 0 && a16 && p.out_dtype != DT_S32)
    vec = 16;
  else if (p.C % 4 == 0 && p.in_cstride % 4 == 0 && p.out_cstride % 4 == 0 && a4 && p.out_dtype != DT_S32)
    vec = 4;
  const long long total = (long long)p.N * p.P * p.Q * (p.C / vec);
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const int threads = 256;
  const long long want = (total + threads - 1) / threads;
  const int blocks = (int)std::max<long long>(1, std::min<long long>(want, (long long)sms * 8));
  if (vec == 16)
    depthwise_kernel<16><<<blocks, threads, 0, s>>>(p);
  else if (vec == 4)
    depthwise_kernel<4><<<blocks, threads, 0, s>>>(p);
  else
    depthwise_kernel<1><<<blocks, threads, 0, s>>>(p);
  count_launch();
  return cudaGetLastError();
}

}  // namespace qnn
