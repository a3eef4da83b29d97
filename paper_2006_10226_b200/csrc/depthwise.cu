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
  pdl_wait();      // inputs are the previous kernel's output (PDL launch; no early trigger: the
                   // next kernel's CTAs would take this multi-wave grid's slots while waiting)
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
    launch_pdl(depthwise_kernel<16>, dim3(blocks), dim3(threads), 0, s, p);
  else if (vec == 4)
    launch_pdl(depthwise_kernel<4>, dim3(blocks), dim3(threads), 0, s, p);
  else
    launch_pdl(depthwise_kernel<1>, dim3(blocks), dim3(threads), 0, s, p);
  count_launch();
  return cudaGetLastError();
}

// ---------------------------------------------------------------------------
// 3x3 depthwise, stride 1 or 2, on CUDA cores with dp4a (the fast path).
//
// Each thread owns four channels (one 32-bit word of an NHWC pixel) and a register
// block of TP x TQ outputs.  Per input row it loads the (TQ-1)*SH + 3 pixel words it
// needs (out-of-image pixels read as zp_A, the P:259 padding), transposes them 4x4 with
// byte permutes so that each word holds four consecutive pixels of ONE channel, and
// then every (output, filter row, channel) term is a single
//     dp4a(window of 4 pixel bytes, (w0, w1, w2, 0))
// -- the three taps of a filter row in one instruction.  With zp_A padding every tap is
// valid, so  x = sum A*W - zp_A*sum W + bias  and the zero-point correction plus bias is
// one per-channel constant off[c], folded into the fixed-point requantize
//     y = hi32(acc*M + (off*M + (2^(t-1) + zp_out*2^t)*2^32)) >> t      (see epilogue.cuh)
// The thread's channel group is fixed for its whole grid-stride walk (grid size is a
// multiple of the group count), so weights and requantize parameters live in registers.
// Requires (checked per thread) W - zp_W in [-128, 127]; otherwise, and for shifts outside
// the fast range or TONEAREST, the exact int64 requantize is used.
// ---------------------------------------------------------------------------
template <bool ASIGNED>
__device__ __forceinline__ int32_t dp4a_aw(uint32_t a, uint32_t w, int32_t c) {
  int32_t d;
  if (ASIGNED)
    asm("dp4a.s32.s32 %0, %1, %2, %3;" : "=r"(d) : "r"(a), "r"(w), "r"(c));
  else
    asm("dp4a.u32.s32 %0, %1, %2, %3;" : "=r"(d) : "r"(a), "r"(w), "r"(c));
  return d;
}

// One thread's walk over its tasks for a fixed channel group.  A task is a row block of
// TP output rows and a run of up to p.qseg column blocks of TQ outputs, swept left to right:
// the input words a block shares with the previous one stay in registers, so each block loads
// only its TQ*SH new columns per input row.
template <int SH, int MODE, int CLAMP, bool S8OUT, bool ASIGNED, bool FAST>
__device__ __forceinline__ void dw3_items(const DwParams& p, int c0, int first, int step,
                                          const uint32_t (&wr)[3][4], const int32_t (&Mc)[4], const int32_t (&Tc)[4],
                                          const int32_t (&Rc)[4], const long long (&Kc)[4],
                                          const int32_t (&off32)[4]) {
  constexpr int TP = SH == 1 ? 2 : 1, TQ = 4;   // register block (stride 2: one row keeps it spill-free)
  constexpr int NW = (TQ - 1) * SH + 3;          // input pixel words per row
  constexpr int NT = (NW + 3) / 4;               // transposed words per channel
  constexpr int IR = (TP - 1) * SH + 3;          // input rows per block
  constexpr int STEP = TQ * SH;                  // input columns advanced per block
  const uint32_t zfill = 0x01010101u * (uint32_t)(p.zpA & 0xFF);
  const int PB = (p.P + TP - 1) / TP, QB = (p.Q + TQ - 1) / TQ;
  const int NS = (QB + p.qseg - 1) / p.qseg;     // column segments per row block
  const int tasks = p.N * PB * NS;
  const uint8_t* in = reinterpret_cast<const uint8_t*>(p.in);
  uint8_t* out = reinterpret_cast<uint8_t*>(p.out);
  const int pix = (int)p.in_cstride;
  for (int task = first; task < tasks; task += step) {
    const int seg = task % NS;
    const int t2 = task / NS;
    const int pb = t2 % PB;
    const int n = t2 / PB;
    const int p0 = pb * TP;
    const int qb_lo = seg * p.qseg, qb_hi = min(QB, qb_lo + p.qseg);
    const int h0 = p0 * SH - p.pt;
    const uint8_t* rowp[IR];
    uint32_t rowv = 0;
#pragma unroll
    for (int ir = 0; ir < IR; ++ir) {
      const int h = h0 + ir;
      const bool ok = h >= 0 && h < p.H;
      rowv |= (uint32_t)ok << ir;
      rowp[ir] = in + ((long long)n * p.H + (ok ? h : 0)) * p.W * pix + c0;
    }
    uint32_t x[IR][NT * 4];
    int w0 = qb_lo * STEP - p.pl;
    const bool rows_all = rowv == (1u << IR) - 1;
    auto load = [&](int ir, int j) -> uint32_t {
      const int w = w0 + j;
      const bool ok = ((rowv >> ir) & 1) && w >= 0 && w < p.W;
      const uint32_t v = __ldg(reinterpret_cast<const uint32_t*>(rowp[ir] + (ok ? w : 0) * pix));
      return ok ? v : zfill;
    };
#pragma unroll
    for (int ir = 0; ir < IR; ++ir)
#pragma unroll
      for (int j = 0; j < NT * 4; ++j) x[ir][j] = j < NW ? load(ir, j) : zfill;
    for (int qb = qb_lo; qb < qb_hi; ++qb) {
      if (qb > qb_lo) {
        w0 += STEP;
        if (rows_all && w0 + NW <= p.W) {
          // interior: all new columns are inside the image (w0 > 0 after the first block)
#pragma unroll
          for (int ir = 0; ir < IR; ++ir) {
            const uint8_t* base = rowp[ir] + w0 * pix;
#pragma unroll
            for (int j = 0; j < NW; ++j)
              x[ir][j] = j + STEP < NW ? x[ir][j + STEP]
                                       : __ldg(reinterpret_cast<const uint32_t*>(base + j * pix));
          }
        } else {
#pragma unroll
          for (int ir = 0; ir < IR; ++ir)
#pragma unroll
            for (int j = 0; j < NW; ++j) x[ir][j] = j + STEP < NW ? x[ir][j + STEP] : load(ir, j);
        }
      }
      const int q0 = qb * TQ;
      int32_t acc[TP][TQ][4];
#pragma unroll
      for (int a = 0; a < TP; ++a)
#pragma unroll
        for (int b = 0; b < TQ; ++b)
#pragma unroll
          for (int ch = 0; ch < 4; ++ch) acc[a][b][ch] = 0;
#pragma unroll
      for (int ir = 0; ir < IR; ++ir) {
        // 4x4 byte transposes: tw[ch][k] = pixels 4k..4k+3 of channel ch
        uint32_t tw[4][NT];
#pragma unroll
        for (int k = 0; k < NT; ++k) {
          const uint32_t a = x[ir][4 * k], b = x[ir][4 * k + 1], c = x[ir][4 * k + 2], d = x[ir][4 * k + 3];
          const uint32_t t0 = __byte_perm(a, b, 0x5140), t1 = __byte_perm(a, b, 0x7362);
          const uint32_t u0 = __byte_perm(c, d, 0x5140), u1 = __byte_perm(c, d, 0x7362);
          tw[0][k] = __byte_perm(t0, u0, 0x5410);
          tw[1][k] = __byte_perm(t0, u0, 0x7632);
          tw[2][k] = __byte_perm(t1, u1, 0x5410);
          tw[3][k] = __byte_perm(t1, u1, 0x7632);
        }
#pragma unroll
        for (int op = 0; op < TP; ++op) {
          const int r = ir - op * SH;
          if (r < 0 || r > 2) continue;
#pragma unroll
          for (int q = 0; q < TQ; ++q) {
            const int o = q * SH;                  // first pixel of the window
#pragma unroll
            for (int ch = 0; ch < 4; ++ch) {
              const uint32_t win = (o & 3) == 0 ? tw[ch][o >> 2]
                                                : __funnelshift_r(tw[ch][o >> 2], tw[ch][(o >> 2) + 1], 8 * (o & 3));
              acc[op][q][ch] = dp4a_aw<ASIGNED>(win, wr[r][ch], acc[op][q][ch]);
            }
          }
        }
      }
      // requantize + store (4 channels = one word per output pixel)
#pragma unroll
      for (int op = 0; op < TP; ++op) {
        const int pp = p0 + op;
        uint8_t* orow = out + ((long long)n * p.P + pp) * p.Q * p.out_cstride + c0;
#pragma unroll
        for (int q = 0; q < TQ; ++q) {
          const int qq = q0 + q;
          int32_t y[4];
#pragma unroll
          for (int ch = 0; ch < 4; ++ch) {
            int32_t v;
            if (FAST) {
              v = mad_hi64(acc[op][q][ch], Mc[ch], Kc[ch]) >> Tc[ch];
            } else {
              const int32_t xv = (int32_t)((uint32_t)acc[op][q][ch] + (uint32_t)off32[ch]);
              v = rq_apply(xv, Mc[ch], Rc[ch], p.mode, p.zp_out, p.lo, p.hi);
            }
            if (CLAMP == 2) v = max(v, p.lo);
            if (CLAMP != 0) v = min(v, p.hi);
            y[ch] = v;
          }
          uint32_t word;
          if (S8OUT)
            asm("{\n\t.reg .u32 t;\n\tcvt.pack.sat.s8.s32.b32 t, %4, %3, 0;\n\tcvt.pack.sat.s8.s32.b32 %0, %2, %1, t;\n\t}"
                : "=r"(word) : "r"(y[0]), "r"(y[1]), "r"(y[2]), "r"(y[3]));
          else
            asm("{\n\t.reg .u32 t;\n\tcvt.pack.sat.u8.s32.b32 t, %4, %3, 0;\n\tcvt.pack.sat.u8.s32.b32 %0, %2, %1, t;\n\t}"
                : "=r"(word) : "r"(y[0]), "r"(y[1]), "r"(y[2]), "r"(y[3]));
          if (pp < p.P && qq < p.Q) *reinterpret_cast<uint32_t*>(orow + (long long)qq * p.out_cstride) = word;
        }
      }
    }
  }
}

template <int SH, int MODE, int CLAMP, bool S8OUT, bool ASIGNED>
__global__ void __launch_bounds__(256, 2) depthwise3_kernel(const __grid_constant__ DwParams p) {
  pdl_wait();      // inputs are the previous kernel's output (PDL launch; no early trigger: the
                   // next kernel's CTAs would take this multi-wave grid's slots while waiting)
  const int G = p.C >> 2;
  const long long tid = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  const long long nthreads = (long long)gridDim.x * blockDim.x;
  const int g = (int)(tid % G);
  const int c0 = g * 4;
  // weights: per channel and filter row, (w0, w1, w2, 0) as s8 bytes (host checked the range)
  uint32_t wr[3][4];
  long long wsum[4] = {0, 0, 0, 0};
#pragma unroll
  for (int ch = 0; ch < 4; ++ch)
#pragma unroll
    for (int r = 0; r < 3; ++r) {
      uint32_t word = 0;
#pragma unroll
      for (int s = 0; s < 3; ++s) {
        const int v = p.w[(r * 3 + s) * p.C + c0 + ch];
        wsum[ch] += v;
        word |= ((uint32_t)v & 0xFFu) << (8 * s);
      }
      wr[r][ch] = word;
    }
  int32_t Mc[4], Tc[4], Rc[4], off32[4];
  long long Kc[4];
  bool fast = MODE == RND_UPWARD;
#pragma unroll
  for (int ch = 0; ch < 4; ++ch) {
    const int c = c0 + ch;
    const long long off = (p.bias ? (long long)p.bias[c] : 0) - (long long)p.zpA * wsum[ch];
    off32[ch] = (int32_t)(uint32_t)(unsigned long long)off;
    Mc[ch] = p.mult[c];
    const int r = p.rsh[c];
    Rc[ch] = r;
    Tc[ch] = 0;
    Kc[ch] = 0;
    if (r >= 33 && r <= 52) {
      const int t = r - 32;
      const unsigned long long c64 = (1ull << (t - 1)) + ((unsigned long long)(long long)p.zp_out << t);
      Kc[ch] = (long long)((unsigned long long)off * (unsigned long long)(long long)Mc[ch] + (c64 << 32));
      Tc[ch] = t;
    } else {
      fast = false;
    }
  }
  const int first = (int)(tid / G), step = (int)(nthreads / G);
  if (fast)
    dw3_items<SH, MODE, CLAMP, S8OUT, ASIGNED, true>(p, c0, first, step, wr, Mc, Tc, Rc, Kc, off32);
  else
    dw3_items<SH, MODE, CLAMP, S8OUT, ASIGNED, false>(p, c0, first, step, wr, Mc, Tc, Rc, Kc, off32);
}

// dispatch of the dp4a 3x3 kernel; false if the shape is not eligible
bool launch_depthwise3(const DwParams& p, int clamp, cudaStream_t s) {
  if (!(p.R == 3 && p.S == 3 && p.dh == 1 && p.dw == 1 && p.sh == p.sw && (p.sh == 1 || p.sh == 2))) return false;
  if (p.C % 4 || p.in_cstride % 4 || p.out_cstride % 4 || !p.requant || p.out_dtype == DT_S32) return false;
  if (((reinterpret_cast<uintptr_t>(p.in) | reinterpret_cast<uintptr_t>(p.out)) & 3) != 0) return false;
  if (!p.w_fits_s8) return false;
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const int G = p.C / 4;
  // tasks: row blocks x column segments; segments as long as the load balance allows (>= ~3
  // resident waves of threads), every extra block in a segment saves its halo loads
  const int TP = p.sh == 1 ? 2 : 1;
  const long long rowblocks = (long long)p.N * ((p.P + TP - 1) / TP);
  const int QB = (p.Q + 3) / 4;
  const long long want = (long long)sms * 2 * 256 * 3;   // thread slots x 3
  int qseg = QB;
  while (qseg > 1 && rowblocks * ((QB + qseg - 1) / qseg) * G < want) qseg = (qseg + 1) / 2;
  DwParams q = p;
  q.qseg = qseg;
  const long long tasks = rowblocks * ((QB + qseg - 1) / qseg);
  if (tasks * G > INT32_MAX) return false;
  long long blocks = std::max<long long>(1, std::min<long long>((tasks * G + 255) / 256, (long long)sms * 2));
  int gg = G, t = 256;
  while (t) { const int r = gg % t; gg = t; t = r; }
  const int unit = G / gg;
  blocks = (blocks + unit - 1) / unit * unit;
  const bool s8 = p.out_dtype == DT_S8;
#define QNN_DW3(SH_, M_, C_, S_, A_)                                                                      \
  if (p.sh == SH_ && p.mode == M_ && clamp == C_ && s8 == S_ && (p.a_signed != 0) == A_) {               \
    launch_pdl(depthwise3_kernel<SH_, M_, C_, S_, A_>, dim3((int)blocks), dim3(256), 0, s, q);                                  \
    count_launch();                                                                                        \
    return true;                                                                                           \
  }
#define QNN_DW3_A(SH_, M_, C_, S_) QNN_DW3(SH_, M_, C_, S_, false) QNN_DW3(SH_, M_, C_, S_, true)
#define QNN_DW3_S(SH_, M_, C_) QNN_DW3_A(SH_, M_, C_, false) QNN_DW3_A(SH_, M_, C_, true)
#define QNN_DW3_C(SH_, M_) QNN_DW3_S(SH_, M_, 0) QNN_DW3_S(SH_, M_, 1) QNN_DW3_S(SH_, M_, 2)
  QNN_DW3_C(1, 0) QNN_DW3_C(1, 1) QNN_DW3_C(2, 0) QNN_DW3_C(2, 1)
#undef QNN_DW3_C
#undef QNN_DW3_S
#undef QNN_DW3_A
#undef QNN_DW3
  return false;
}

}  // namespace qnn
