/*
 * qnn.h — C ABI of libqnn.so, the B200 (sm_100a) implementation of the QNN
 * pre-quantized operator hot path of arXiv 2006.10226 ("Efficient Execution of
 * Quantized Deep Learning Models: A Compiler Approach").
 *
 * Each entry point cites the passage of PAPER.md ("P:n" = line n) that defines
 * the operation; readings of ambiguous passages are numbered R1..R18 in
 * DESIGN.md.  The QNN operators carry "quantization scales, zero points and
 * data type"; the arguments below mirror those attributes.
 *
 * Conventions shared by every entry point
 * ---------------------------------------
 *  * Memory.  Tensor pointers are DEVICE pointers on the current CUDA device
 *    (set by the caller) unless a parameter says "host".  The caller owns every
 *    buffer; the library never allocates or frees device memory.  Host arrays
 *    (scales, zero points, shapes) are read before the call returns and may be
 *    freed afterwards.
 *  * Layout.  Activations are NHWC (channels innermost), conv weights OHWI
 *    (K x R x S x C/groups), dense operands row-major with the reduction axis
 *    innermost (A: M x K, W: N x K).
 *  * Asynchrony.  Work is enqueued on `stream` (a cudaStream_t; NULL = the
 *    legacy default stream) and the call returns before it completes, except
 *    the *_prepack calls, which block until the packed blob is complete.
 *    Calls that take only device pointers are CUDA-graph capturable.
 *  * Errors.  Arguments are validated before anything is enqueued; on any
 *    error nothing is enqueued and a non-zero qnn_status_t is returned.
 *    QNN_ERR_CUDA reports a failed launch.  No exception or abort crosses the
 *    ABI.  Thread-safe on distinct streams.
 *  * Arithmetic.  Integer results are bit-exact with the definition
 *    (P:169-188 for conv/dense, P:273-281 for requantize): int32
 *    accumulation is exact for KK*255*255 < 2^31 (reading R10), larger
 *    reductions are rejected with QNN_ERR_UNSUPPORTED.
 */
#ifndef QNN_H_
#define QNN_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#if defined(__GNUC__)
#define QNN_API __attribute__((visibility("default")))
#else
#define QNN_API
#endif

/* cudaStream_t without including CUDA headers */
typedef struct CUstream_st* qnn_stream_t;

typedef enum {
  QNN_S8 = 0,   /* int8  */
  QNN_U8 = 1,   /* uint8 */
  QNN_S32 = 2,  /* int32 */
  QNN_F32 = 3   /* float */
} qnn_dtype_t;

/* Rounding of the fixed-point product ("Different frameworks choose
 * different rounding methods"; reading R1; TVM's attribute names). */
typedef enum {
  QNN_ROUND_UPWARD = 0,    /* ties toward +inf:   floor(x + 1/2)            */
  QNN_ROUND_TONEAREST = 1  /* ties away from 0:   sign(x)*floor(|x| + 1/2)  */
} qnn_rounding_t;

typedef enum {
  QNN_OK = 0,
  QNN_ERR_INVALID_VALUE = 1, /* bad scale (<=0, NaN, inf), zp out of dtype range, bad shape */
  QNN_ERR_UNSUPPORTED = 2,   /* valid but not implemented (e.g. grouped conv, dilation on TC path) */
  QNN_ERR_MISALIGNED = 3,    /* pointer / pitch alignment the kernels need is not met */
  QNN_ERR_WORKSPACE = 4,     /* workspace or packed buffer too small */
  QNN_ERR_CUDA = 5           /* a CUDA launch or copy failed */
} qnn_status_t;

/* Output side of Eq. 5 fused into a conv/dense epilogue: bias is added to the
 * int32 Eq. 3 result, then (TFLite sequence, fig:tflite_conv2d)
 * ReLU, requantize by m_k = s_A*s_W[k]/output_scale (reading R3) through the
 * fixed-point multiplier (reading R2), + output_zero_point, clamp to
 * [act_min, act_max] in the output domain (reading R6), saturate (R5). */
typedef struct {
  float output_scale;          /* > 0, per-tensor (per-channel output scale unsupported) */
  int32_t output_zero_point;   /* within out_dtype's range                                */
  qnn_dtype_t out_dtype;       /* QNN_U8 or QNN_S8 (use NULL params for raw int32)       */
  qnn_rounding_t rounding;
  int32_t relu;                /* non-zero: lower clamp at output_zero_point (real 0.0)  */
  int32_t act_min, act_max;    /* output-domain clamp; INT32_MIN / INT32_MAX = none      */
} qnn_output_params_t;

/* Quantized conv2d attributes (Eq. 2 / Eq. 3; zp padding P:259).
 * groups == 1 runs the tensor-core implicit GEMM; groups == C == K runs the
 * depthwise kernel; other group counts return QNN_ERR_UNSUPPORTED. */
typedef struct {
  int32_t N, H, W, C;          /* input NHWC                                            */
  int32_t K, R, S;             /* output channels, filter height, width (OHWI weights)  */
  int32_t stride_h, stride_w;
  int32_t pad_t, pad_l, pad_b, pad_r;   /* padding value is input_zero_point    */
  int32_t dil_h, dil_w;
  int32_t groups;
  int32_t in_cstride;          /* channel pitch of the input (elements), 0 => C         */
  int32_t out_cstride;         /* channel pitch of the output (elements), 0 => K        */
  qnn_dtype_t input_dtype;     /* QNN_U8 or QNN_S8                                      */
  qnn_dtype_t kernel_dtype;    /* QNN_U8 or QNN_S8                                      */
  int32_t input_zero_point;    /* zp_A                                                   */
  int32_t kernel_zero_point;   /* zp_W, per-tensor (used when num_kernel_zero_points == 0) */
  float input_scale;           /* s_A                                                    */
  const float* kernel_scales;  /* host; 1 (per-tensor) or K (per-channel, axis 0) values*/
  int32_t num_kernel_scales;
  /* Per-channel weight zero points (the paper discusses per-channel
   * scales only, P:37, P:227 -- reading R11 extends Eq. 3 channel by channel):
   * host array of K values in the kernel dtype's range, or NULL with count 0.  Term 3 is
   * then zp_W[k] * rowsum, folded into the contraction (weights packed as W - zp_W[k],
   * split into two s8 k-blocks); channels whose W - zp_W[k] range is not inside
   * [-256, 254] (s8 weights with zp_W[k] = -128) give QNN_ERR_UNSUPPORTED. */
  const int32_t* kernel_zero_points;
  int32_t num_kernel_zero_points;   /* 0 (use kernel_zero_point) or K                      */
} qnn_conv2d_desc_t;

/* Quantized dense (qnn.dense; "matmul"): out[m,n] over A (M x K) and
 * W (N x K); the GEMM form of the conv path with R = S = 1. */
typedef struct {
  int32_t M, N, K;
  int32_t lda;                 /* row pitch of A in elements, 0 => K (must be a multiple of 16 bytes) */
  int32_t ldc;                 /* row pitch of out in elements, 0 => N                   */
  qnn_dtype_t a_dtype, w_dtype;
  int32_t zp_A, zp_W;
  float s_A;
  const float* s_W;            /* host; 1 or N values                                   */
  int32_t n_sW;
  const int32_t* zp_Ws;        /* host; per-output-channel weight zero points (N values), or NULL */
  int32_t n_zpW;               /* 0 (use zp_W) or N                                     */
} qnn_dense_desc_t;

QNN_API const char* qnn_status_string(qnn_status_t status);

/* Library / device diagnostics: number of kernels this library launched on
 * the calling thread since the last reset (used by the bench to report
 * gpu_launches); reset with qnn_launch_counter_reset(). */
QNN_API uint64_t qnn_launch_counter(void);
QNN_API void qnn_launch_counter_reset(void);

/* Fixed-point multiplier for a positive real m (reading R2):
 * M in [2^30, 2^31) and m ~= M * 2^(shift - 31).  Host only.
 * QNN_ERR_INVALID_VALUE if m <= 0, NaN or inf. */
QNN_API qnn_status_t qnn_derive_multiplier(double m, int32_t* M, int32_t* shift);

/* ------------------------------------------------------------------------- *
 * qnn.conv2d (+ bias + clip + requantize).
 *
 * Compile-time folding ("term 2 and term 4 are compile-time
 * constants"): qnn_conv2d_prepack packs the weights and folds Terms 2 and 4,
 * the bias and the zero-point padding corrections into per-(border class,
 * channel) int32 offsets, and derives the per-channel fixed-point
 * multipliers.  `o` NULL selects raw int32 output (Eq. 3 result + bias).
 * `kernel` and `bias` are device pointers (bias nullable: int32, scale
 * s_A*s_W[k], zero point 0 — reading R12).  `packed` must hold
 * qnn_conv2d_prepack_size() bytes, 256-byte aligned.  Blocks until done.
 * ------------------------------------------------------------------------- */
QNN_API qnn_status_t qnn_conv2d_prepack_size(const qnn_conv2d_desc_t* d, const qnn_output_params_t* o,
                                     size_t* bytes);
QNN_API qnn_status_t qnn_conv2d_prepack(const qnn_conv2d_desc_t* d, const void* kernel, const int32_t* bias,
                                const qnn_output_params_t* o, void* packed, size_t packed_bytes,
                                qnn_stream_t stream);

/* Per-call scratch for qnn_conv2d_packed (Term-3 row sums when zp_W != 0,
 * channel-padded input copy when C*elem is not a multiple of 16 bytes). */
QNN_API qnn_status_t qnn_conv2d_workspace_size(const qnn_conv2d_desc_t* d, const qnn_output_params_t* o,
                                       size_t* bytes);

/* The hot path: output = requantize(conv(input, W) with zp algebra + bias).
 * `input` NHWC with channel pitch in_cstride, base 16-byte aligned; `output`
 * NHWC with channel pitch out_cstride.  `d` and `o` must be the ones given to
 * qnn_conv2d_prepack (the scales inside are not re-read; o's zero point,
 * dtype, rounding, relu and act clamps are). */
QNN_API qnn_status_t qnn_conv2d_packed(const qnn_conv2d_desc_t* d, const qnn_output_params_t* o,
                               const void* packed, const void* input, void* output,
                               void* workspace, size_t workspace_bytes, qnn_stream_t stream);

/* qnn.conv2d fused with a residual qnn.add (reading R19): the conv's
 * int32 result requantized to (s_out, 0) plus the residual requantized to (s_out, 0), then
 * zp_out, ReLU (lower bound zp_out when o->relu), act clamps and saturation:
 *   out = sat(zp_out + R(acc * m_k) + R((res - res_zp) * res_scale / s_out))
 * `residual`: NHWC, N x P x Q x K (the conv output's shape), channel pitch res_cstride (0 => K),
 * 8-bit (res_dtype S8/U8), base and pitch 16-byte aligned.  Requires requantized output (o not
 * NULL), K % 32 == 0 and a non-depthwise conv (else UNSUPPORTED).  Everything else as
 * qnn_conv2d_packed. */
QNN_API qnn_status_t qnn_conv2d_packed_add(const qnn_conv2d_desc_t* d, const qnn_output_params_t* o,
                                           const void* packed, const void* input, const void* residual,
                                           qnn_dtype_t res_dtype, float res_scale, int32_t res_zero_point,
                                           int32_t res_cstride, void* output, void* workspace,
                                           size_t workspace_bytes, qnn_stream_t stream);

/* One-shot convenience: prepack into the front of `workspace`, then run.
 * workspace_bytes >= prepack_size (rounded up to 256) + workspace_size.
 * Not graph-capturable (prepack blocks). */
QNN_API qnn_status_t qnn_conv2d(const qnn_conv2d_desc_t* d, const void* input, const void* kernel,
                        const int32_t* bias, const qnn_output_params_t* o, void* output,
                        void* workspace, size_t workspace_bytes, qnn_stream_t stream);

/* Depthwise conv (groups == C == K, weights K x R x S x 1): the same calls
 * apply; this entry point only checks that `d` is depthwise and forwards to
 * qnn_conv2d.  CUDA-core kernel, subtract-first lowering. */
QNN_API qnn_status_t qnn_depthwise_conv2d(const qnn_conv2d_desc_t* d, const void* input, const void* kernel,
                                  const int32_t* bias, const qnn_output_params_t* o, void* output,
                                  void* workspace, size_t workspace_bytes, qnn_stream_t stream);

/* ------------------------------------------------------------------------- *
 * qnn.dense (+ bias + requantize).  Same prepack / packed / one-shot split.
 * ------------------------------------------------------------------------- */
QNN_API qnn_status_t qnn_dense_prepack_size(const qnn_dense_desc_t* d, const qnn_output_params_t* o,
                                    size_t* bytes);
QNN_API qnn_status_t qnn_dense_prepack(const qnn_dense_desc_t* d, const void* W, const int32_t* bias,
                               const qnn_output_params_t* o, void* packed, size_t packed_bytes,
                               qnn_stream_t stream);
QNN_API qnn_status_t qnn_dense_workspace_size(const qnn_dense_desc_t* d, const qnn_output_params_t* o,
                                      size_t* bytes);
QNN_API qnn_status_t qnn_dense_packed(const qnn_dense_desc_t* d, const qnn_output_params_t* o,
                              const void* packed, const void* A, void* out, void* workspace,
                              size_t workspace_bytes, qnn_stream_t stream);
QNN_API qnn_status_t qnn_dense(const qnn_dense_desc_t* d, const void* A, const void* W, const int32_t* bias,
                       const qnn_output_params_t* o, void* out, void* workspace,
                       size_t workspace_bytes, qnn_stream_t stream);

/* ------------------------------------------------------------------------- *
 * Standalone qnn.requantize (Eq. 5):
 *   out = clamp(R(m_c * (in - in_zp)) + out_zp),  m_c = in_scales[c] / out_scale
 * per-tensor (n_in_scales == 1) or per-channel along `axis` (n_in_scales ==
 * shape[axis], at most 4096).  in: S8/U8/S32, out: S8/U8/S32.  Each m_c must
 * be < 2^30.  `shape` is a host array of ndim (1..8) extents; axis < 0 counts
 * from the end.  Enqueue-only (multipliers travel as kernel parameters).
 * ------------------------------------------------------------------------- */
QNN_API qnn_status_t qnn_requantize(const void* in, qnn_dtype_t in_dtype, void* out, qnn_dtype_t out_dtype,
                            const int64_t* shape, int32_t ndim, int32_t axis, const float* in_scales,
                            int32_t n_in_scales, int32_t in_zp, float out_scale, int32_t out_zp,
                            qnn_rounding_t rounding, qnn_stream_t stream);

/* qnn.quantize (Eq. 1 inverted, reading R14): q = clamp(round_half_away(
 * fl32(x / s_c)) + zp_c); NaN -> zp_c.  in F32, out S8/U8.
 * qnn.dequantize (Eq. 1): x = fl32(s_c * (q - zp_c)), one rounding; in S8/U8/S32.
 * Per-tensor (n_params == 1) or per-channel along `axis` (<= 2048). */
QNN_API qnn_status_t qnn_quantize(const float* in, void* out, qnn_dtype_t out_dtype, const int64_t* shape,
                          int32_t ndim, int32_t axis, const float* scales, const int32_t* zero_points,
                          int32_t n_params, qnn_stream_t stream);
QNN_API qnn_status_t qnn_dequantize(const void* in, qnn_dtype_t in_dtype, float* out, const int64_t* shape,
                            int32_t ndim, int32_t axis, const float* scales, const int32_t* zero_points,
                            int32_t n_params, qnn_stream_t stream);

/* Host-buffer forms of quantize / dequantize: the end-to-end entry and exit of a network whose
 * input and output live in host memory (BASELINE configs[4]'s f32 images in, logits out).
 *
 * qnn_quantize_host: `host_in` is page-locked host memory (cudaHostAlloc / cudaHostRegister /
 *   torch pin_memory) holding the f32 tensor.  The call enqueues the host->device copy of
 *   prod(shape) * 4 bytes into `staging` (device memory, caller-owned, at least that size) on
 *   `copy_stream` (a copy engine: it runs alongside kernels on other streams), makes `stream` wait
 *   for that copy, then quantizes staging -> `out` (device) on `stream`, exactly as qnn_quantize.
 *   The caller orders `copy_stream` after the previous reader of `staging` (double buffering:
 *   two staging buffers, copy_stream waiting on an event recorded after the quantize that last
 *   read the buffer); copy_stream may equal stream (no overlap).
 * qnn_dequantize_host: `host_out` is page-locked host memory; the dequantize kernel writes the
 *   f32 result straight into it through its mapped device address (zero-copy over PCIe), so the
 *   values are on the host once `stream` passes the call.  Otherwise exactly qnn_dequantize.
 * Errors: QNN_ERR_INVALID_VALUE when the host pointer is not page-locked host memory (pageable
 * memory cannot be read or written by the device asynchronously) or when `staging` is null;
 * QNN_ERR_CUDA on a failed copy enqueue.  Enqueue-only. */
QNN_API qnn_status_t qnn_quantize_host(const float* host_in, float* staging, void* out, qnn_dtype_t out_dtype,
                               const int64_t* shape, int32_t ndim, int32_t axis, const float* scales,
                               const int32_t* zero_points, int32_t n_params, qnn_stream_t copy_stream,
                               qnn_stream_t stream);
QNN_API qnn_status_t qnn_dequantize_host(const void* in, qnn_dtype_t in_dtype, float* host_out, const int64_t* shape,
                                 int32_t ndim, int32_t axis, const float* scales, const int32_t* zero_points,
                                 int32_t n_params, qnn_stream_t stream);

/* -------------------------------------------------------------------------------------------
 * Inter-layer glue (the paper's framework operators quantized_add and
 * pooling).
 * ------------------------------------------------------------------------------------------- */

/* qnn.add (reading R19, SPEC canonicalize_add): each input is requantized (Eq. 5, fixed-point
 * multiplier of s_x / s_out, `rounding`) to (s_out, zero point 0), the two int32 values are
 * summed, zp_out is added, then max(., zp_out) if relu, then saturation to out_dtype:
 *   out[i] = sat(max?(zp_out + R((a[i]-zp_a) s_a/s_out) + R((b[i]-zp_b) s_b/s_out)))
 * a, b, out: `count` elements each, S8/U8 (device pointers, same element order).  Per-tensor
 * scales only.  Errors: INVALID_VALUE for a bad scale / zero point / dtype, UNSUPPORTED for a
 * scale ratio >= 2^30. */
QNN_API qnn_status_t qnn_add(const void* a, qnn_dtype_t a_dtype, float s_a, int32_t zp_a, const void* b,
                             qnn_dtype_t b_dtype, float s_b, int32_t zp_b, void* out, qnn_dtype_t out_dtype,
                             float s_out, int32_t zp_out, int64_t count, qnn_rounding_t rounding, int32_t relu,
                             qnn_stream_t stream);

typedef enum { QNN_POOL_MAX = 0, QNN_POOL_AVG = 1 } qnn_pool_mode_t;

/* Pooling on quantized NHWC values with input and output sharing (scale, zero point), as the
 * frontend enforces.  Padding taps are excluded (reading R20):
 *   MAX: out = max over the valid taps;
 *   AVG: s = sum over the valid taps (int32), n = their count,
 *        out = sign(s) * floor((2|s| + n) / (2n))   (rounding division, ties away from zero).
 * Output is N x P x Q x C with P = (H + pad_t + pad_b - R)/stride_h + 1 (likewise Q).
 * in_cstride / out_cstride: channel pitch of a pixel in elements (0 => C).  in, out: device. */
typedef struct {
  int32_t N, H, W, C, R, S;
  int32_t stride_h, stride_w, pad_t, pad_l, pad_b, pad_r;
  int32_t in_cstride, out_cstride;
  qnn_dtype_t dtype;            /* QNN_U8 or QNN_S8 */
  qnn_pool_mode_t mode;
} qnn_pool2d_desc_t;
QNN_API qnn_status_t qnn_pool2d(const qnn_pool2d_desc_t* d, const void* in, void* out, qnn_stream_t stream);

#ifdef __cplusplus
}
#endif
#endif /* QNN_H_ */
