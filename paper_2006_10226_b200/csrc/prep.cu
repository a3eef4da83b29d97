// prep.cu — compile-time folding (weight prepack) and the auxiliary kernels of
// the conv path.
//
//  * pack_weights   : OHWI weights -> [Kpad][R*S][Cw] zero-padded, the B operand
//                     of the implicit GEMM (pad channels/rows are 0: reading R8).
//  * fold_offsets   : "term 2 and term 4 are compile-time constants" (P:259,
//                     P:264).  Per border class cls and channel k:
//                       off = bias[k] - zp_A * sum_{valid taps, c} W[k,r,s,c]
//                                     + zp_A * zp_W * C * nvalid_taps(cls)
//                     which also restores the zero-point padding that
//                     TMA's zero fill omits (reading R7).
//  * pixel_sums / window_sums : Term 3 ("sliding window reduction ... pool2d,
//                     reduce sum"): rowsum[n,p,q] = sum over valid taps
//                     of sum_c A.  Only launched when zp_W != 0.
//  * pad_channels   : copies an input whose pixel pitch is not a multiple of 16
//                     bytes into a zero-padded pitch the TMA can address.
#include "common.cuh"
#include "internal.h"

namespace qnn {

// perm32: row r of every 32-row group holds channel 4*(r % 8) + (r / 8) % 4 of that group -- the
// TMEM lane order of the channel-major GEMM (gemm_t.cu), whose 16x256b TMEM loads then hand a
// thread four consecutive output channels of one pixel.
// split (weight zero points, Term 3 folded into the contraction): row k holds W - zp_W[k] as two
// s8 k-block sets, [RS*Cw part a][RS*Cw part b] with a = clamp(W', -128, 127), b = W' - a, so
// sum_c A * (a + b) = sum_c A * (W - zp_W[k]) exactly (W' in [-256, 254], checked on the host)
__global__ void pack_weights_kernel(const uint8_t* __restrict__ W, uint8_t* __restrict__ Wp, int K, int RS, int C,
                                    int Cw, int Kpad, int perm32, int split, int w_signed,
                                    const int32_t* __restrict__ zpv) {
  const int row_w = (split ? 2 : 1) * RS * Cw;
  const long long total = (long long)Kpad * row_w;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < total;
       i += (long long)gridDim.x * blockDim.x) {
    const int col = (int)(i % row_w);
    const int row = (int)(i / row_w);
    const int part = col / (RS * Cw), cc = col - part * RS * Cw;
    const int c = cc % Cw, tap = cc / Cw;
    const int k = perm32 ? (row & ~31) | (4 * (row & 7) + ((row >> 3) & 3)) : row;
    uint8_t v = 0;
    if (k < K && c < C) {
      const uint8_t b = W[((long long)k * RS + tap) * C + c];
      if (split) {
        const int wv = (w_signed ? (int)(int8_t)b : (int)b) - zpv[k];
        const int a = min(max(wv, -128), 127);
        v = (uint8_t)(int8_t)(part == 0 ? a : wv - a);
      } else {
        v = b;
      }
    }
    Wp[i] = v;
  }
}

cudaError_t launch_pack_weights(const void* W, void* Wp, int K, int RS, int C, int Cw, int Kpad, cudaStream_t s,
                                int perm32, int split, int w_signed, const int32_t* zpv) {
  const long long total = (long long)Kpad * RS * Cw * (split ? 2 : 1);
  const int threads = 256;
  const int blocks = (int)std::min<long long>((total + threads - 1) / threads, 4096);
  pack_weights_kernel<<<blocks, threads, 0, s>>>((const uint8_t*)W, (uint8_t*)Wp, K, RS, C, Cw, Kpad, perm32, split,
                                                 w_signed, zpv);
  count_launch();
  return cudaGetLastError();
}

__global__ void fold_offsets_kernel(const uint8_t* __restrict__ W, int w_signed, const int32_t* __restrict__ bias,
                                    int K, int R, int S, int C, int32_t zpA, int32_t zpW_scalar, ClassTable ct,
                                    int32_t* __restrict__ off, int64_t* __restrict__ off64, int Kpad,
                                    const int32_t* __restrict__ zpv) {
  const int ncls = ct.ncr * ct.ncc;
  const int idx = blockIdx.x * blockDim.x + threadIdx.x;
  if (idx >= ncls * Kpad) return;
  const int cls = idx / Kpad, k = idx - cls * Kpad;
  if (k >= K) {
    off[idx] = 0;
    off64[idx] = 0;
    return;
  }
  const int rc = cls / ct.ncc, cc = cls - rc * ct.ncc;
  const int r0 = ct.r_lo[rc], r1 = ct.r_hi[rc], s0 = ct.s_lo[cc], s1 = ct.s_hi[cc];
  const long long zpW = zpv ? zpv[k] : zpW_scalar;   // per-channel weight zero point (f4)
  long long colsum = 0;
  int nvalid = 0;
  for (int r = r0; r <= r1; ++r)
    for (int s = s0; s <= s1; ++s) {
      ++nvalid;
      const uint8_t* w = W + (((long long)k * R + r) * S + s) * C;
      for (int c = 0; c < C; ++c) colsum += w_signed ? (long long)(int8_t)w[c] : (long long)w[c];
    }
  // int32 wrap is exact for the final sum (reading R10); compute in 64-bit then wrap.
  const long long v = (bias ? (long long)bias[k] : 0) - (long long)zpA * colsum +
                      (long long)zpA * zpW * (long long)C * nvalid;
  off[idx] = (int32_t)(uint32_t)(unsigned long long)v;
  off64[idx] = v;
}

cudaError_t launch_fold_offsets(const void* W, int w_signed, const int32_t* bias, int K, int R, int S, int C,
                                int32_t zpA, int32_t zpW, const ClassTable& ct, int32_t* off, int64_t* off64,
                                int Kpad, cudaStream_t s, const int32_t* zpv) {
  const int total = ct.ncr * ct.ncc * Kpad;
  fold_offsets_kernel<<<(total + 127) / 128, 128, 0, s>>>((const uint8_t*)W, w_signed, bias, K, R, S, C, zpA, zpW,
                                                         ct, off, off64, Kpad, zpv);
  count_launch();
  return cudaGetLastError();
}

// depthwise weights K x R x S x 1 (K == C) -> [R*S][C] int16 holding W - zp_W
__global__ void pack_dw_weights_kernel(const uint8_t* __restrict__ W, int w_signed, int32_t zpW,
                                       int16_t* __restrict__ Wd, int C, int RS, const int32_t* __restrict__ zpv) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= C * RS) return;
  const int tap = i / C, c = i - tap * C;
  const uint8_t b = W[(long long)c * RS + tap];
  const int v = w_signed ? (int)(int8_t)b : (int)b;
  Wd[i] = (int16_t)(v - (zpv ? zpv[c] : zpW));
}

cudaError_t launch_pack_dw_weights(const void* W, int w_signed, int32_t zpW, int16_t* Wd, int C, int RS,
                                   cudaStream_t s, const int32_t* zpv) {
  pack_dw_weights_kernel<<<(C * RS + 255) / 256, 256, 0, s>>>((const uint8_t*)W, w_signed, zpW, Wd, C, RS, zpv);
  count_launch();
  return cudaGetLastError();
}

__global__ void pad_channels_kernel(const uint8_t* __restrict__ in, long long in_cstride, uint8_t* __restrict__ out,
                                    int Cp, long long npix, int C) {
  const long long total = npix * Cp;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < total;
       i += (long long)gridDim.x * blockDim.x) {
    const long long pix = i / Cp;
    const int c = (int)(i - pix * Cp);
    out[i] = c < C ? in[pix * in_cstride + c] : (uint8_t)0;
  }
}

cudaError_t launch_pad_channels(const void* in, long long in_cstride, void* out, int Cp, long long npix, int C,
                                cudaStream_t s) {
  const long long total = npix * Cp;
  const int blocks = (int)std::min<long long>((total + 255) / 256, 148 * 16);
  pad_channels_kernel<<<blocks, 256, 0, s>>>((const uint8_t*)in, in_cstride, (uint8_t*)out, Cp, npix, C);
  count_launch();
  return cudaGetLastError();
}

// Width fold for small-C convolutions (e.g. the C = 3 stem): X'[n,h,q,j] with
// j = s*C + c holds A[n, h, q*sw + s*dw - pl, c] (0 outside the image and for
// j >= S*C), so the R x S conv becomes an R x 1 conv over S*C channels with
// far fewer, fuller tensor-core K steps.  Zero fill outside the image is
// corrected by the same border-class offsets as the TMA zero fill (reading R7).
__global__ void __launch_bounds__(256) fold_width_kernel(const uint8_t* __restrict__ in, long long in_cstride,
                                                         uint8_t* __restrict__ out, int N, int H, int W, int C, int Q,
                                                         int S, int sw, int pl, int dw, int Cf) {
  // one thread per 16-byte piece of a folded pixel; interior windows of a dense row read
  // their S*C contiguous bytes as aligned 32-bit words (L1-cached, neighbours overlap) and
  // funnel-shift them into place; border windows fall back to per-byte gathers
  __shared__ int tab_s[128], tab_c[128];   // folded channel j -> filter column s*dw (or a sentinel), channel c
  const int sc = S * C;
  for (int j = threadIdx.x; j < Cf; j += blockDim.x) {
    const int s = j / C;
    tab_s[j] = j < sc ? s * dw : -(1 << 20);
    tab_c[j] = j - s * C;
  }
  __syncthreads();
  const int pieces = Cf / 16;
  const bool dense = in_cstride == C && (reinterpret_cast<uintptr_t>(in) & 3) == 0 && ((W * C) & 3) == 0 && dw == 1;
  // 32-bit index arithmetic (the launcher guarantees N*H*Q*pieces < 2^31): 64-bit
  // division would dominate this bandwidth-bound kernel
  const uint32_t total = (uint32_t)((long long)N * H * Q * pieces);
  for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < total; i += gridDim.x * blockDim.x) {
    const uint32_t t32 = i / (uint32_t)pieces;
    const int pc = (int)(i - t32 * (uint32_t)pieces);
    const uint32_t nh32 = t32 / (uint32_t)Q;
    const int q = (int)(t32 - nh32 * (uint32_t)Q);
    const long long t = t32, nh = nh32;
    const int w0 = q * sw - pl;
    const uint8_t* rowp = in + nh * W * in_cstride;
    uint32_t wv[4] = {0, 0, 0, 0};
    if (dense && w0 >= 0 && w0 + S <= W) {
      const int base = w0 * C + pc * 16;
      const int valid = sc - pc * 16;   // bytes of this piece that are real folded channels
      if (valid > 0) {
        const uint32_t* rw = reinterpret_cast<const uint32_t*>(rowp);
        const int wa = base >> 2, shb = (base & 3) * 8;
        const int last = min(W * C / 4 - 1, wa + 4);   // never read past the row
        uint32_t x[5];
#pragma unroll
        for (int k = 0; k < 5; ++k) x[k] = __ldg(rw + min(wa + k, last));
#pragma unroll
        for (int k = 0; k < 4; ++k) wv[k] = shb ? __funnelshift_r(x[k], x[k + 1], shb) : x[k];
#pragma unroll
        for (int k = 0; k < 4; ++k) {
          const int nb = valid - 4 * k;
          wv[k] = nb >= 4 ? wv[k] : (nb <= 0 ? 0u : (wv[k] & ((1u << (8 * nb)) - 1u)));
        }
      }
    } else {
#pragma unroll
      for (int b = 0; b < 16; ++b) {
        const int j = pc * 16 + b;
        const int w = w0 + tab_s[j];
        if (w >= 0 && w < W) wv[b >> 2] |= (uint32_t)rowp[(long long)w * in_cstride + tab_c[j]] << (8 * (b & 3));
      }
    }
    *reinterpret_cast<uint4*>(out + t * Cf + pc * 16) = make_uint4(wv[0], wv[1], wv[2], wv[3]);
  }
}

cudaError_t launch_fold_width(const void* in, long long in_cstride, void* out, int N, int H, int W, int C, int Q, int S,
                              int sw, int pl, int dw, int Cf, cudaStream_t s) {
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const long long total = (long long)N * H * Q * (Cf / 16);
  if (total >= (1LL << 31)) return cudaErrorInvalidValue;
  const int grid = (int)std::max<long long>(1, std::min<long long>((total + 255) / 256, (long long)sms * 16));
  fold_width_kernel<<<grid, 256, 0, s>>>((const uint8_t*)in, in_cstride, (uint8_t*)out, N, H, W, C, Q, S, sw, pl, dw,
                                         Cf);
  count_launch();
  return cudaGetLastError();
}

// Term 3, step 1: per-pixel channel sums (one warp-cooperative pass over A).
__global__ void pixel_sums_kernel(const uint8_t* __restrict__ in, int a_signed, long long in_cstride, int C,
                                  long long npix, int32_t* __restrict__ pixsum) {
  const long long pix = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (pix >= npix) return;
  const uint8_t* a = in + pix * in_cstride;
  int32_t s = 0;
  int c = 0;
  if ((in_cstride & 15) == 0 && (reinterpret_cast<uintptr_t>(in) & 15) == 0) {
    for (; c + 16 <= C; c += 16) {
      const uint4 v = *reinterpret_cast<const uint4*>(a + c);
      const uint32_t w4[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        if (a_signed)
          s = __dp4a((int)w4[j], 0x01010101, s);
        else
          s = (int32_t)__dp4a(w4[j], 0x01010101u, (uint32_t)s);
      }
    }
  }
  for (; c < C; ++c) s += a_signed ? (int32_t)(int8_t)a[c] : (int32_t)a[c];
  pixsum[pix] = s;
}

// Coalesced variant for C % 16 == 0: gl = min(pow2floor(C/16), 32) consecutive
// lanes share one pixel (a warp reads 512 contiguous bytes per load when the pitch is C), each
// lane sums its 16-byte chunks with dp4a, and the group reduces with xor shuffles.  A block
// covers kPsUnroll x (256 / gl) pixels; each thread issues its kPsUnroll loads before any math
// (bytes in flight for HBM latency).
constexpr int kPsUnroll = 4;

__device__ __forceinline__ int32_t dp4a_sum4(uint4 v, int32_t s, int a_signed) {
  if (a_signed) {
    s = __dp4a((int)v.x, 0x01010101, s);
    s = __dp4a((int)v.y, 0x01010101, s);
    s = __dp4a((int)v.z, 0x01010101, s);
    return __dp4a((int)v.w, 0x01010101, s);
  }
  s = (int32_t)__dp4a(v.x, 0x01010101u, (uint32_t)s);
  s = (int32_t)__dp4a(v.y, 0x01010101u, (uint32_t)s);
  s = (int32_t)__dp4a(v.z, 0x01010101u, (uint32_t)s);
  return (int32_t)__dp4a(v.w, 0x01010101u, (uint32_t)s);
}

__global__ void pixel_sums_vec_kernel(const uint8_t* __restrict__ in, int a_signed, long long in_cstride, int G,
                                      int gl, long long npix, int32_t* __restrict__ pixsum) {
  const int per_pass = blockDim.x / gl;   // pixels per block per unroll step
  const int sub = threadIdx.x % gl;
  const long long pix0 = (long long)blockIdx.x * per_pass * kPsUnroll + threadIdx.x / gl;
  int32_t s[kPsUnroll];
  uint4 v[kPsUnroll];
#pragma unroll
  for (int u = 0; u < kPsUnroll; ++u) {
    s[u] = 0;
    v[u] = make_uint4(0u, 0u, 0u, 0u);
  }
  for (int k = sub; k < G; k += gl) {
#pragma unroll
    for (int u = 0; u < kPsUnroll; ++u) {
      const long long pix = pix0 + (long long)u * per_pass;
      if (pix < npix) v[u] = __ldg(reinterpret_cast<const uint4*>(in + pix * in_cstride) + k);
    }
#pragma unroll
    for (int u = 0; u < kPsUnroll; ++u) s[u] = dp4a_sum4(v[u], s[u], a_signed);
  }
#pragma unroll
  for (int u = 0; u < kPsUnroll; ++u) {
    for (int o = gl >> 1; o > 0; o >>= 1) s[u] += __shfl_xor_sync(0xffffffffu, s[u], o);
    const long long pix = pix0 + (long long)u * per_pass;
    if (sub == 0 && pix < npix) pixsum[pix] = s[u];
  }
}

cudaError_t launch_pixel_sums(const void* in, int a_signed, long long in_cstride, int C, long long npix,
                              int32_t* pixsum, cudaStream_t s) {
  const int G = C / 16;
  if (C % 16 == 0 && G > 0 && (in_cstride & 15) == 0 && (reinterpret_cast<uintptr_t>(in) & 15) == 0) {
    int gl = 1;   // lanes per pixel: the largest power of two <= min(G, 32) (lanes loop over the rest)
    while (gl * 2 <= G && gl < 32) gl *= 2;
    const long long per_block = (long long)(256 / gl) * kPsUnroll;
    pixel_sums_vec_kernel<<<(unsigned)((npix + per_block - 1) / per_block), 256, 0, s>>>((const uint8_t*)in, a_signed, in_cstride,
                                                                           G, gl, npix, pixsum);
  } else {
    pixel_sums_kernel<<<(unsigned)((npix + 255) / 256), 256, 0, s>>>((const uint8_t*)in, a_signed, in_cstride, C,
                                                                      npix, pixsum);
  }
  count_launch();
  return cudaGetLastError();
}

// Term 3, step 2: rowsum[n,p,q] = sum over in-image taps (r,s) of pixsum
// (zero-filled taps contribute 0; their zp part lives in the class offsets).
__global__ void window_sums_kernel(const int32_t* __restrict__ pixsum, int N, int H, int W, int P, int Q, int R,
                                   int S, int sh, int sw, int pt, int pl, int dh, int dw,
                                   int32_t* __restrict__ rowsum) {
  const long long m = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  const long long M = (long long)N * P * Q;
  if (m >= M) return;
  const int q = (int)(m % Q);
  const long long t = m / Q;
  const int p = (int)(t % P);
  const int n = (int)(t / P);
  int32_t s = 0;
  for (int r = 0; r < R; ++r) {
    const int h = p * sh + r * dh - pt;
    if (h < 0 || h >= H) continue;
    for (int c = 0; c < S; ++c) {
      const int w = q * sw + c * dw - pl;
      if (w < 0 || w >= W) continue;
      s += pixsum[((long long)n * H + h) * W + w];
    }
  }
  rowsum[m] = s;
}

cudaError_t launch_window_sums(const int32_t* pixsum, int N, int H, int W, int P, int Q, int R, int S, int sh,
                               int sw, int pt, int pl, int dh, int dw, int32_t* rowsum, cudaStream_t s) {
  const long long M = (long long)N * P * Q;
  window_sums_kernel<<<(unsigned)((M + 255) / 256), 256, 0, s>>>(pixsum, N, H, W, P, Q, R, S, sh, sw, pt, pl, dh,
                                                                  dw, rowsum);
  count_launch();
  return cudaGetLastError();
}

}  // namespace qnn
