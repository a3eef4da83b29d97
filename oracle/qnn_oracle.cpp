/*
 * qnn_oracle.cpp — TEST INFRASTRUCTURE ONLY.
 *
 * A plain, slow, obviously-correct CPU implementation of what the QNN hot path
 * computes (arXiv 2006.10226, "Efficient Execution of Quantized Deep Learning
 * Models: A Compiler Approach").  Only tests/, __graft_entry__.smoke() and
 * bench.py's cpu_baseline / --impl reference legs may load this library.
 * The product path (paper_2006_10226_b200/) never includes, links or calls it,
 * and this file includes nothing from the product tree.
 *
 * Citations: "P:n" = line n of the paper's PAPER.md; "Eq. k" = the paper's
 * equation k (Eq.1, Eq.2, Eq.3, Eq.5).
 * Readings of ambiguous passages are listed in DESIGN.md §"Readings" (R1..).
 *
 * Layout: NCHW activations, OIHW weights (the paper's index names n,c,h,w /
 * k,c,r,s).  The test harness permutes to/from the kernel's NHWC/OHWI.
 *
 * Arithmetic: every accumulation is int64; requantize rounding is an exact
 * rational computed with __int128 numerators and floor division (no shifts),
 * so it shares no formulation with the GPU's shift-and-add epilogue.
 *
 * Parity status of each function: all pinned (see tests/test_oracle_*.py);
 * nothing here is "parity unpinned".
 */
#include <cstdint>
#include <cmath>
#include <cstring>
#include <climits>

extern "C" {

/* oracle dtype codes (private to the oracle; deliberately not shared with include/qnn.h) */
enum { OR_S8 = 0, OR_U8 = 1, OR_S32 = 2, OR_F32 = 3 };
/* rounding codes (R1): 0 = UPWARD (ties toward +inf), 1 = TONEAREST (ties away from zero) */
enum { OR_UPWARD = 0, OR_TONEAREST = 1 };

static inline int64_t load_q(const void* p, int dt, int64_t i) {
  switch (dt) {
    case OR_S8:  return (int64_t)((const int8_t*)p)[i];
    case OR_U8:  return (int64_t)((const uint8_t*)p)[i];
    case OR_S32: return (int64_t)((const int32_t*)p)[i];
    default:     return 0;
  }
}

static inline void dtype_range(int dt, int64_t* lo, int64_t* hi) {
  switch (dt) {
    case OR_S8:  *lo = -128; *hi = 127; break;
    case OR_U8:  *lo = 0; *hi = 255; break;
    default:     *lo = INT32_MIN; *hi = INT32_MAX; break;
  }
}

static inline void store_q(void* p, int dt, int64_t i, int64_t v) {
  switch (dt) {
    case OR_S8:  ((int8_t*)p)[i] = (int8_t)v; break;
    case OR_U8:  ((uint8_t*)p)[i] = (uint8_t)v; break;
    case OR_S32: ((int32_t*)p)[i] = (int32_t)v; break;
    default: break;
  }
}

/* ------------------------------------------------------------------------- *
 * Fixed-point multiplier ("fixed point multiplication as a proxy for
 * floating point multiplication"; reading R2 in DESIGN.md):
 *   (sig, e) = frexp(m), sig in [0.5, 1);  M = round_half_away(sig * 2^31);
 *   if M == 2^31 then M = 2^30, e += 1;    m ~= M * 2^(e - 31); shift := e.
 * Returns 0 on success, -1 if m is not a positive finite number.
 * ------------------------------------------------------------------------- */
int oracle_derive_multiplier(double m, int32_t* M, int32_t* shift) {
  if (!(m > 0.0) || !std::isfinite(m)) return -1;
  int e = 0;
  double sig = std::frexp(m, &e);          /* m = sig * 2^e, sig in [0.5,1) */
  double t = std::ldexp(sig, 31);          /* exact: scaling by a power of two */
  /* t in [2^30, 2^31) has ulp 2^-22, so t + 0.5 is exact; floor gives half-up,
     which for a positive value is half-away-from-zero. */
  int64_t Mi = (int64_t)std::floor(t + 0.5);
  if (Mi == (int64_t)1 << 31) { Mi = (int64_t)1 << 30; e += 1; }
  *M = (int32_t)Mi;
  *shift = (int32_t)e;
  return 0;
}

/* floor(a / b) for b > 0, on 128-bit integers */
static inline __int128 floor_div(__int128 a, __int128 b) {
  __int128 q = a / b;                       /* C truncates toward zero */
  if ((a % b) != 0 && a < 0) q -= 1;
  return q;
}

static inline int64_t sat64(__int128 v) {
  if (v > (__int128)INT64_MAX) return INT64_MAX;
  if (v < (__int128)INT64_MIN) return INT64_MIN;
  return (int64_t)v;
}

/* ------------------------------------------------------------------------- *
 * Round the exact rational  q = x * M / 2^(31 - shift)  to an integer
 * (Eq. 5's "(scale_A/scale_B) * (Q_A - zp_A)" with the fixed-point proxy of
 * P:281; reading R1 for the two rounding modes):
 *   UPWARD    : floor(q + 1/2)
 *   TONEAREST : sign(q) * floor(|q| + 1/2)
 * ------------------------------------------------------------------------- */
int64_t oracle_round_fixed(int64_t x, int32_t M, int32_t shift, int mode) {
  __int128 num = (__int128)x * (__int128)M;     /* |num| < 2^94 */
  int k = 31 - shift;                            /* q = num / 2^k */
  if (k <= 0) {
    /* q is an integer: num * 2^(-k); saturate if it leaves int64 */
    if (num == 0) return 0;
    if (-k >= 40) return num > 0 ? INT64_MAX : INT64_MIN;
    __int128 v = num;
    for (int i = 0; i < -k; ++i) v *= 2;
    return sat64(v);
  }
  if (k >= 120) return 0;                        /* |q| < 2^-25: rounds to 0 in both modes */
  __int128 den = (__int128)1 << k;
  if (mode == OR_UPWARD) {
    /* floor(num/den + 1/2) = floor((2*num + den) / (2*den)) */
    return sat64(floor_div(2 * num + den, 2 * den));
  } else {
    __int128 a = num < 0 ? -num : num;
    __int128 r = floor_div(2 * a + den, 2 * den);
    return sat64(num < 0 ? -r : r);
  }
}

/* Apply the requantize tail to one accumulator value: optional ReLU in the
 * int32 domain *before* requantize (the TFLite order of fig:tflite_conv2d,
 * conv -> bias_add -> clip -> requantize), fixed-point rescale,
 * + zp_out (Eq. 5), output-domain act clamp, saturation to the dtype (R5). */
static inline int64_t requant_tail(int64_t v, int32_t M, int32_t shift, int mode,
                                   int32_t zp_out, int relu, int32_t act_min,
                                   int32_t act_max, int out_dt) {
  if (relu && v < 0) v = 0;
  int64_t y = oracle_round_fixed(v, M, shift, mode);
  /* add zp_out without overflowing int64 */
  if (y > INT64_MAX / 2) y = INT64_MAX / 2;
  if (y < INT64_MIN / 2) y = INT64_MIN / 2;
  y += zp_out;
  if (y < act_min) y = act_min;
  if (y > act_max) y = act_max;
  int64_t lo, hi;
  dtype_range(out_dt, &lo, &hi);
  if (y < lo) y = lo;
  if (y > hi) y = hi;
  return y;
}

/* ------------------------------------------------------------------------- *
 * Direct quantized conv2d, Eq. 2 integer core with zero-point padding:
 *   acc[n,k,p,q] = sum_{c in group(k)} sum_{r,s}
 *                  (a(n, c, p*sh + r*dh - pt, q*sw + s*dw - pl) - zp_A)
 *                  * (W[k, c, r, s] - zp_W)            + bias[k]
 * where a(...) = zp_A outside the input ("padding a quantized input tensor
 * ... translates to padding the tensor with zero_point").  Eq. 3 is
 * written for stride 1 / no padding / groups 1; the general index
 * form is reading R9.  Output acc is int64, NKPQ.
 * ------------------------------------------------------------------------- */
static inline int64_t conv_one(int64_t n, int64_t k, int64_t p, int64_t q,
                               int C, int H, int W, int K, int R, int S,
                               int sh, int sw, int pt, int pl, int dh, int dw, int G,
                               int a_dt, const void* A, int w_dt, const void* Wt,
                               int32_t zpA, int32_t zpW, const int32_t* bias) {
  const int Cg = C / G, Kg = K / G;
  const int g = (int)(k / Kg);
  int64_t acc = 0;
  for (int c = 0; c < Cg; ++c) {
    const int64_t cin = (int64_t)g * Cg + c;
    for (int r = 0; r < R; ++r) {
      const int64_t h = p * sh + (int64_t)r * dh - pt;
      for (int s = 0; s < S; ++s) {
        const int64_t w = q * sw + (int64_t)s * dw - pl;
        int64_t a;
        if (h >= 0 && h < H && w >= 0 && w < W)
          a = load_q(A, a_dt, ((n * C + cin) * H + h) * W + w);
        else
          a = zpA;
        const int64_t wt = load_q(Wt, w_dt, ((k * Cg + c) * R + r) * S + s);
        acc += (a - zpA) * (wt - zpW);
      }
    }
  }
  if (bias) acc += bias[k];
  return acc;
}

static inline int out_dim(int in, int pad_lo, int pad_hi, int dil, int ksz, int stride) {
  return (in + pad_lo + pad_hi - dil * (ksz - 1) - 1) / stride + 1;
}

void oracle_conv2d_acc(int N, int C, int H, int W, int K, int R, int S,
                       int sh, int sw, int pt, int pl, int pb, int pr,
                       int dh, int dw, int G,
                       int a_dt, const void* A, int w_dt, const void* Wt,
                       int32_t zpA, int32_t zpW, const int32_t* bias,
                       int64_t* acc) {
  const int P = out_dim(H, pt, pb, dh, R, sh), Q = out_dim(W, pl, pr, dw, S, sw);
  #pragma omp parallel for collapse(2) schedule(dynamic)
  for (int n = 0; n < N; ++n)
    for (int k = 0; k < K; ++k)
      for (int p = 0; p < P; ++p)
        for (int q = 0; q < Q; ++q)
          acc[(((int64_t)n * K + k) * P + p) * Q + q] =
              conv_one(n, k, p, q, C, H, W, K, R, S, sh, sw, pt, pl, dh, dw, G,
                       a_dt, A, w_dt, Wt, zpA, zpW, bias);
}

/* Same definition, evaluated only at flat NKPQ indices idx[0..count) */
void oracle_conv2d_acc_at(int N, int C, int H, int W, int K, int R, int S,
                          int sh, int sw, int pt, int pl, int pb, int pr,
                          int dh, int dw, int G,
                          int a_dt, const void* A, int w_dt, const void* Wt,
                          int32_t zpA, int32_t zpW, const int32_t* bias,
                          const int64_t* idx, int64_t count, int64_t* acc) {
  (void)N;
  const int P = out_dim(H, pt, pb, dh, R, sh), Q = out_dim(W, pl, pr, dw, S, sw);
  #pragma omp parallel for schedule(dynamic, 64)
  for (int64_t i = 0; i < count; ++i) {
    int64_t t = idx[i];
    const int64_t q = t % Q; t /= Q;
    const int64_t p = t % P; t /= P;
    const int64_t k = t % K; t /= K;
    const int64_t n = t;
    acc[i] = conv_one(n, k, p, q, C, H, W, K, R, S, sh, sw, pt, pl, dh, dw, G,
                      a_dt, A, w_dt, Wt, zpA, zpW, bias);
  }
}

/* ------------------------------------------------------------------------- *
 * Eq. 3 evaluator (four terms, each summed separately over the zp-padded
 * input) — used ONLY by the oracle's self-tests to check Eq.2 == Eq.3.
 *   Q_C = sum QA*QW - sum zpA*QW - sum zpW*QA + sum zpA*zpW        (+ bias)
 * Term 4 sums over c,r,s of one group: zpA*zpW*Cg*R*S (reading R9).
 * ------------------------------------------------------------------------- */
void oracle_conv2d_eq3(int N, int C, int H, int W, int K, int R, int S,
                       int sh, int sw, int pt, int pl, int pb, int pr,
                       int dh, int dw, int G,
                       int a_dt, const void* A, int w_dt, const void* Wt,
                       int32_t zpA, int32_t zpW, const int32_t* bias,
                       int64_t* acc) {
  const int P = out_dim(H, pt, pb, dh, R, sh), Q = out_dim(W, pl, pr, dw, S, sw);
  const int Cg = C / G, Kg = K / G;
  #pragma omp parallel for collapse(2)
  for (int n = 0; n < N; ++n)
    for (int k = 0; k < K; ++k) {
      const int g = k / Kg;
      for (int p = 0; p < P; ++p)
        for (int q = 0; q < Q; ++q) {
          int64_t t1 = 0, t2 = 0, t3 = 0, t4 = 0;
          for (int c = 0; c < Cg; ++c) {
            const int64_t cin = (int64_t)g * Cg + c;
            for (int r = 0; r < R; ++r)
              for (int s = 0; s < S; ++s) {
                const int64_t h = (int64_t)p * sh + (int64_t)r * dh - pt;
                const int64_t w = (int64_t)q * sw + (int64_t)s * dw - pl;
                const int64_t qa = (h >= 0 && h < H && w >= 0 && w < W)
                    ? load_q(A, a_dt, (((int64_t)n * C + cin) * H + h) * W + w) : zpA;
                const int64_t qw = load_q(Wt, w_dt, (((int64_t)k * Cg + c) * R + r) * S + s);
                t1 += qa * qw;                 /* Term 1 */
                t2 += (int64_t)zpA * qw;       /* Term 2 */
                t3 += (int64_t)zpW * qa;       /* Term 3 */
                t4 += (int64_t)zpA * zpW;      /* Term 4 */
              }
          }
          int64_t v = t1 - t2 - t3 + t4;
          if (bias) v += bias[k];
          acc[(((int64_t)n * K + k) * P + p) * Q + q] = v;
        }
    }
}

/* ------------------------------------------------------------------------- *
 * Dense (qnn.dense): acc[m,n] = sum_k (A[m,k] - zp_A)(W[n,k] - zp_W) + bias[n]
 * (Eq. 2 with r = s = 1; the paper names "matmul" at P:294).
 * ------------------------------------------------------------------------- */
void oracle_dense_acc(int M, int Nn, int K, int a_dt, const void* A, int w_dt,
                      const void* Wt, int32_t zpA, int32_t zpW,
                      const int32_t* bias, int64_t* acc) {
  #pragma omp parallel for schedule(dynamic, 4)
  for (int m = 0; m < M; ++m)
    for (int n = 0; n < Nn; ++n) {
      int64_t s = 0;
      for (int k = 0; k < K; ++k)
        s += (load_q(A, a_dt, (int64_t)m * K + k) - zpA) *
             (load_q(Wt, w_dt, (int64_t)n * K + k) - zpW);
      if (bias) s += bias[n];
      acc[(int64_t)m * Nn + n] = s;
    }
}

void oracle_dense_acc_at(int M, int Nn, int K, int a_dt, const void* A, int w_dt,
                         const void* Wt, int32_t zpA, int32_t zpW,
                         const int32_t* bias, const int64_t* idx, int64_t count,
                         int64_t* acc) {
  (void)M;
  #pragma omp parallel for schedule(dynamic, 64)
  for (int64_t i = 0; i < count; ++i) {
    const int64_t m = idx[i] / Nn, n = idx[i] % Nn;
    int64_t s = 0;
    for (int k = 0; k < K; ++k)
      s += (load_q(A, a_dt, m * K + k) - zpA) * (load_q(Wt, w_dt, n * K + k) - zpW);
    if (bias) s += bias[n];
    acc[i] = s;
  }
}

/* Per-channel multipliers for a conv/dense output (reading R3):
 *   m_k = ((double)s_A * (double)s_W[k]) / (double)s_out   (Eq. 2: Q_C has
 *   scale s_A*s_W; Eq. 5 rescales it to s_out). n_sW is 1 or K. */
int oracle_conv_multipliers(float s_A, const float* s_W, int n_sW, int K,
                            float s_out, int32_t* M, int32_t* shift) {
  for (int k = 0; k < K; ++k) {
    const double m = ((double)s_A * (double)s_W[n_sW == 1 ? 0 : k]) / (double)s_out;
    if (oracle_derive_multiplier(m, &M[k], &shift[k]) != 0) return -1;
  }
  return 0;
}

/* Requantize an accumulator tensor (int64) whose channel index is
 * (i / inner) % Cext:  y = clamp(zp_out + R(relu(acc) * M_c * 2^(shift_c-31))).
 * n_ch is 1 (per-tensor) or Cext (per-channel). */
void oracle_requantize_acc(const int64_t* acc, int64_t count, int64_t inner, int Cext,
                           const int32_t* M, const int32_t* shift, int n_ch, int mode,
                           int32_t zp_out, int relu, int32_t act_min, int32_t act_max,
                           int out_dt, void* out) {
  #pragma omp parallel for schedule(static)
  for (int64_t i = 0; i < count; ++i) {
    const int c = n_ch == 1 ? 0 : (int)((i / inner) % Cext);
    store_q(out, out_dt, i,
            requant_tail(acc[i], M[c], shift[c], mode, zp_out, relu, act_min, act_max, out_dt));
  }
}

/* Standalone qnn.requantize (Eq. 5):
 *   Q_B = clamp( R( (s_A[c]/s_B) * (Q_A - zp_A) ) + zp_B )
 * with m_c = (double)s_in[c] / (double)s_out (R3) through the fixed-point
 * proxy (R2) and exact-rational rounding (R1).  x - zp_in is exact in int64.
 * Returns -1 if a multiplier cannot be derived. */
int oracle_requantize(const void* in, int in_dt, int64_t count, int64_t inner, int Cext,
                      const float* s_in, int n_s, int32_t zp_in, float s_out,
                      int32_t zp_out, int mode, int out_dt, void* out) {
  int32_t Ms[4096], Ss[4096];
  if (n_s > 4096) return -1;
  for (int c = 0; c < n_s; ++c)
    if (oracle_derive_multiplier((double)s_in[c] / (double)s_out, &Ms[c], &Ss[c]) != 0) return -1;
  #pragma omp parallel for schedule(static)
  for (int64_t i = 0; i < count; ++i) {
    const int c = n_s == 1 ? 0 : (int)((i / inner) % Cext);
    const int64_t x = load_q(in, in_dt, i) - (int64_t)zp_in;
    store_q(out, out_dt, i,
            requant_tail(x, Ms[c], Ss[c], mode, zp_out, 0, INT32_MIN, INT32_MAX, out_dt));
  }
  return 0;
}

/* qnn.quantize, Eq. 1 inverted (reading R14): t = fl32(x / s) (IEEE fp32
 * division), q = clamp(round_half_away(t) + zp).  NaN maps to zp. */
void oracle_quantize(const float* x, int64_t count, int64_t inner, int Cext,
                     const float* scales, const int32_t* zps, int n_p, int out_dt,
                     void* out) {
  int64_t lo, hi;
  dtype_range(out_dt, &lo, &hi);
  #pragma omp parallel for schedule(static)
  for (int64_t i = 0; i < count; ++i) {
    const int c = n_p == 1 ? 0 : (int)((i / inner) % Cext);
    volatile float t = x[i] / scales[c];        /* one IEEE fp32 division */
    float tv = t;
    int64_t q;
    if (std::isnan(tv)) {
      q = zps[c];
    } else {
      if (tv > 1e12f) tv = 1e12f;
      if (tv < -1e12f) tv = -1e12f;
      q = (int64_t)std::round(tv) + zps[c];      /* std::round: half away from zero */
    }
    if (q < lo) q = lo;
    if (q > hi) q = hi;
    store_q(out, out_dt, i, q);
  }
}

/* qnn.dequantize, Eq. 1: A_fp32 = scale * (Q - zp), a single fp32 rounding:
 * (q - zp) (< 2^33 in magnitude) times a 24-bit-significand scale needs at
 * most 57 significand bits, exact in x87 extended precision (64-bit
 * significand), so the final cast to float rounds exactly once. */
void oracle_dequantize(const void* q, int in_dt, int64_t count, int64_t inner, int Cext,
                       const float* scales, const int32_t* zps, int n_p, float* out) {
  #pragma omp parallel for schedule(static)
  for (int64_t i = 0; i < count; ++i) {
    const int c = n_p == 1 ? 0 : (int)((i / inner) % Cext);
    const long double d = (long double)(load_q(q, in_dt, i) - (int64_t)zps[c]) *
                          (long double)scales[c];
    out[i] = (float)d;
  }
}

/* ------------------------------------------------------------------------- *
 * Inter-layer glue (the paper's framework operators
 * "quantized_add", pooling).
 * ------------------------------------------------------------------------- */

/* qnn.add: each input is requantized (Eq. 5 with the fixed-point proxy, R2/R3)
 * to (s_out, zero point 0) as an exact integer, the two are summed, zp_out is
 * added, optional ReLU (lower bound zp_out), then saturation to the output
 * dtype (reading R19; SPEC canonicalize_add).  Returns -1 on a bad scale. */
int oracle_add(const void* a, int a_dt, float s_a, int32_t zp_a, const void* b, int b_dt, float s_b,
               int32_t zp_b, int64_t count, float s_out, int32_t zp_out, int mode, int relu, int out_dt,
               void* out) {
  int32_t Ma, Sa, Mb, Sb;
  if (oracle_derive_multiplier((double)s_a / (double)s_out, &Ma, &Sa) != 0) return -1;
  if (oracle_derive_multiplier((double)s_b / (double)s_out, &Mb, &Sb) != 0) return -1;
  int64_t lo, hi;
  dtype_range(out_dt, &lo, &hi);
  #pragma omp parallel for schedule(static)
  for (int64_t i = 0; i < count; ++i) {
    const int64_t ya = oracle_round_fixed(load_q(a, a_dt, i) - zp_a, Ma, Sa, mode);
    const int64_t yb = oracle_round_fixed(load_q(b, b_dt, i) - zp_b, Mb, Sb, mode);
    int64_t y = ya + yb + zp_out;
    if (relu && y < zp_out) y = zp_out;
    if (y < lo) y = lo;
    if (y > hi) y = hi;
    store_q(out, out_dt, i, y);
  }
  return 0;
}

/* Pooling on the quantized values, input and output sharing (scale, zero
 * point) as the frontend enforces (SPEC canonicalize_*_pool).  NCHW.
 * Padding taps are excluded (max: -inf; avg: not counted, reading R20).
 *   max: Q_out = max over the valid window (max commutes with the monotone
 *        affine map of Eq. 1).
 *   avg: s = sum of the valid taps (int64; the paper's int16 upcast cannot hold
 *        a sum of more than 128 u8 values, R17), n = number of valid taps,
 *        Q_out = sign(s) * floor((2|s| + n) / (2n))  (rounding division with ties
 *        away from zero, SPEC "ToNearestAway"). */
void oracle_pool2d(const void* in, int dt, int is_avg, int N, int C, int H, int W, int R, int S, int sh,
                   int sw, int pt, int pl, int P, int Q, void* out) {
  #pragma omp parallel for collapse(2) schedule(static)
  for (int n = 0; n < N; ++n)
    for (int c = 0; c < C; ++c)
      for (int p = 0; p < P; ++p)
        for (int q = 0; q < Q; ++q) {
          int64_t best = INT64_MIN, sum = 0, cnt = 0;
          for (int r = 0; r < R; ++r)
            for (int s = 0; s < S; ++s) {
              const int h = p * sh + r - pt, w = q * sw + s - pl;
              if (h < 0 || h >= H || w < 0 || w >= W) continue;
              const int64_t v = load_q(in, dt, (((int64_t)n * C + c) * H + h) * W + w);
              if (v > best) best = v;
              sum += v;
              ++cnt;
            }
          int64_t y = 0;
          if (is_avg) {
            if (cnt > 0) {
              const int64_t a = sum < 0 ? -sum : sum;
              const int64_t m = (2 * a + cnt) / (2 * cnt);
              y = sum < 0 ? -m : m;
            }
          } else {
            y = cnt > 0 ? best : 0;
          }
          store_q(out, dt, (((int64_t)n * C + c) * P + p) * Q + q, y);
        }
}

int oracle_num_threads(void);
void oracle_set_num_threads(int n);
}  /* extern "C" */

#ifdef _OPENMP
#include <omp.h>
extern "C" int oracle_num_threads(void) { return omp_get_max_threads(); }
// thread count of later parallel regions (timing only: the single-thread oracle rate)
extern "C" void oracle_set_num_threads(int n) { omp_set_num_threads(n > 0 ? n : 1); }
#else
extern "C" int oracle_num_threads(void) { return 1; }
extern "C" void oracle_set_num_threads(int) {}
#endif
