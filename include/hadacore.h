/*
 * hadacore.h -- C ABI of the B200-native batched normalized Walsh-Hadamard transform
 * (the hot path of HadaCore, arXiv 2412.08832).
 *
 * Citations: "P:NN" = /root/reference/PAPER.md line NN [section].
 *
 * The operation (P:41 [Sec. 2.1]; P:87 [Sec. 2.4] "right-Hadamard transform"):
 *     out[i, :] = scale * H_n * in[i, :]        for every row i in [0, m)
 * where H_n is the n x n Walsh-Hadamard matrix in natural (Sylvester) order,
 * (H_n)[j][l] = (-1)^popcount(j & l), built by H(2k) = [[H, H], [H, -H]] (P:45
 * [Sec. 2.2]).  H_n is symmetric, so this equals the right multiply in * H_n.
 * `scale` is the WHOLE multiplier on the +-1 matrix: pass 1/sqrt(n) for the
 * normalized (orthonormal) transform of P:41 ("+-1/sqrt(d) ... when normalized").
 * n is a power of two in [2^7, 2^15] (the paper's range, P:97, P:128 [Sec. 3.2]) or in
 * [2, 2^6] (the strided entry points: [8, 2^6];
 * SPEC S:49's domain 2 <= d; fp32 register butterflies, DESIGN.md "Rows shorter
 * than 128").
 *
 * Layout: `in` and `out` are row-major m x n matrices of 16-bit floats (IEEE
 * binary16 or bfloat16; or binary32 for the HADACORE_F32 path), contiguous,
 * row pitch = n elements, in DEVICE memory of
 * the current CUDA device, 16-byte aligned.  in == out (in-place, P:264-274
 * [App. B]) is allowed and gives bit-identical results to out-of-place.
 *
 * Ownership: the caller owns both buffers; the library allocates nothing for
 * hadacore_fwht, keeps no reference after the call returns, and has no global
 * mutable state except a per-process cache of device attributes.  Buffers must
 * stay alive until the work queued on `stream` has completed.
 *
 * Errors: arguments are validated synchronously, before anything is queued; on a
 * validation error nothing is launched.  The launch is asynchronous on `stream`
 * (no host synchronisation; safe inside CUDA-graph capture).  A launch failure
 * returns HADACORE_ERR_CUDA and leaves the CUDA error for cudaGetLastError().
 * Faults during execution surface at the caller's next synchronisation.
 * No C++ exception crosses this ABI.  There is no CPU fallback: without a usable
 * sm_100 device the call returns HADACORE_ERR_CUDA.
 *
 * Numerics (n >= 128): the internal precision is fp16 (for fp16 data) or fp32
 * accumulate rounded to bf16 between factor stages (for bf16 data), the final factor
 * stage is accumulated in fp32, multiplied by `scale` (times an exact power of two) in
 * fp32 and rounded to nearest even; n < 128 and the fp32 path
 * compute in fp32 throughout with one final rounding.  Rows are independent: a
 * non-finite value in one row never affects another row.
 */
#ifndef HADACORE_H_
#define HADACORE_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* Opaque to keep this header free of CUDA headers: a cudaStream_t is passed as
 * this pointer type (cudaStream_t is itself a pointer; 0/NULL = legacy default). */
typedef struct CUstream_st* hadacore_stream_t;

typedef enum {
  HADACORE_F16 = 0,  /* IEEE 754 binary16 */
  HADACORE_BF16 = 1, /* bfloat16 */
  HADACORE_F32 = 2   /* IEEE 754 binary32: fp32 register butterflies (north_star's fp32 path, 1e-5) */
} hadacore_dtype_t;

/* Code formats of the fused quantized output (hadacore_fwht_quant). */
typedef enum {
  HADACORE_Q_E4M3 = 0, /* FP8 E4M3 ("e4m3fn": no infinities, max finite 448), RNE, saturating */
  HADACORE_Q_INT8 = 1, /* signed 8-bit integer, RNE, clamped to [-127, 127] */
  HADACORE_Q_INT4 = 2  /* signed 4-bit integer, RNE, clamped to [-7, 7]; two per byte, element 2j in the
                          low nibble of byte j (two's complement) */
} hadacore_qtype_t;

typedef enum {
  HADACORE_OK = 0,
  HADACORE_ERR_INVALID_N = 1,   /* n is not a power of two in [2, 32768] ([8, 32768] for the
                                   strided entry points) */
  HADACORE_ERR_INVALID_M = 2,   /* m < 0, or m * n * element size overflows int64 */
  HADACORE_ERR_NULL = 3,        /* in or out is NULL while m > 0 */
  HADACORE_ERR_MISALIGNED = 4,  /* in or out is not 16-byte aligned */
  HADACORE_ERR_OVERLAP = 5,     /* in != out and the two byte ranges overlap */
  HADACORE_ERR_DTYPE = 6,       /* unknown dtype */
  HADACORE_ERR_SCALE = 7,       /* scale is NaN, +-Inf, zero or negative (scale > 0) */
  HADACORE_ERR_CUDA = 8,        /* CUDA error (no device, launch failure, copy failure) */
  HADACORE_ERR_WORKSPACE = 9    /* hadacore_fwht_host: workspace NULL or too small */
} hadacore_status_t;

/*
 * out[i, :] = scale * H_n * in[i, :] for i in [0, m), on `stream` (device buffers).
 * n = 2..2^15.  m == 0 returns HADACORE_OK without launching anything.  Only the
 * buffer start must be 16-byte aligned: for n < 8 the total m * n * 2 bytes need
 * not be a multiple of 16 (bytes past the last row are never touched).
 */
hadacore_status_t hadacore_fwht(const void* in, void* out, int64_t m, int64_t n,
                                hadacore_dtype_t dtype, float scale, hadacore_stream_t stream);

/*
 * End-to-end variant on HOST buffers (the call a host-side user makes): copies row
 * blocks (<= 32 MiB) host->device into `workspace`, transforms them in place with the
 * same kernel, and copies them device->host into `out_host`, pipelined over up to
 * four workspace slots and internal streams so both copy directions overlap the
 * kernels (the four non-blocking streams and one event are created on the first call
 * of each host thread on each device and kept for the process).  Returns after the last
 * device->host copy has completed (synchronises `stream`).
 *   in_host / out_host: m x n row-major 16-bit matrices in host memory (pinned
 *     memory gives full PCIe bandwidth; pageable works but is slower).  May be equal.
 *   workspace: device buffer of workspace_bytes >= 2 * 2 * n bytes (two rows),
 *     16-byte aligned; larger workspaces mean larger copy blocks (for n < 8 the
 *     blocks hold multiples of 16 / (2 n) rows so that they stay 16-byte aligned).
 * Same validation and errors as hadacore_fwht, plus HADACORE_ERR_WORKSPACE.
 */
hadacore_status_t hadacore_fwht_host(const void* in_host, void* out_host, int64_t m, int64_t n,
                                     hadacore_dtype_t dtype, float scale, void* workspace,
                                     size_t workspace_bytes, hadacore_stream_t stream);

/*
 * Strided / multi-head rows: the same transform on the rows
 * of a 2-level grid, e.g. the Q (or K) heads inside a fused QKV projection
 * [tokens, 3, H, d] (m_outer = tokens, m_inner = H, stride_outer = 3*H*d,
 * stride_inner = d, n = d) rotated in place before FP8 attention.
 *     row (i, j), i < m_outer, j < m_inner:
 *         in  + i * in_stride_outer  + j * in_stride_inner     (element offsets)
 *         out + i * out_stride_outer + j * out_stride_inner
 * Strides are element counts, positive multiples of 8 (16 bytes) below 2^38; rows
 * may not overlap (stride_inner >= n when m_inner > 1; stride_outer >= (m_inner-1) *
 * stride_inner + n when m_outer > 1) -- else HADACORE_ERR_INVALID_M.  in == out
 * requires identical strides; otherwise the two extents may not overlap
 * (HADACORE_ERR_OVERLAP).  fp16/bf16 and n = 2^3..2^15 only (rows of >= 16 bytes: TMA
 * boxes).  Other rules as hadacore_fwht.
 */
hadacore_status_t hadacore_fwht_strided(const void* in, void* out, int64_t m_outer, int64_t m_inner,
                                        int64_t in_stride_outer, int64_t in_stride_inner,
                                        int64_t out_stride_outer, int64_t out_stride_inner, int64_t n,
                                        hadacore_dtype_t dtype, float scale, hadacore_stream_t stream);

/*
 * Fused transform + per-row symmetric quantization (the
 * paper's future work "fused Hadamard transform and quantization", P:207 [Sec. 5],
 * for its FP8-attention use, P:180 [Sec. 4.2]):
 *     y = scale * H_n * in[i, :]            (as hadacore_fwht, never written out)
 *     row_scale[i] = max_j |y_j| / Q        (Q = 448 E4M3, 127 INT8, 7 INT4; 1 if y == 0)
 *     out_q[i, j]  = round(y_j / row_scale[i])   (E4M3 saturating / INT8, INT4 clamped)
 * so out_q[i, j] * row_scale[i] ~= y_j.  A row containing Inf/NaN gets a non-finite
 * row_scale.  out_q: m x n bytes (m x n/2 for INT4), row-major, 16-byte aligned; row_scale: m floats
 * (fp32).  Neither may overlap `in`.  n = 2..2^15.  HBM traffic: 2 B read + 1 B
 * (INT4: 0.5 B) written per element.
 * Same validation, stream and error behaviour as hadacore_fwht; qtype outside the
 * enum, or dtype HADACORE_F32, returns HADACORE_ERR_DTYPE.
 */
hadacore_status_t hadacore_fwht_quant(const void* in, void* out_q, float* row_scale, int64_t m, int64_t n,
                                      hadacore_dtype_t dtype, hadacore_qtype_t qtype, float scale,
                                      hadacore_stream_t stream);

/*
 * Quantization-error lab (SPEC quant_lab S:397-440, the
 * paper's motivation P:24 [Sec. 1]: rotations "reduce the magnitude of outliers"):
 * the harness of the rotated-vs-plain experiment, whose rotations are
 * hadacore_fwht calls on fp32 rows.
 *
 * hadacore_fake_quant: symmetric quantize -> dequantize of fp32 rows,
 *     row_amax[i] = max_j |in[i, j]|          (per_tensor != 0: the max over the whole
 *                                             matrix, written to every row_amax[i])
 *     s_i = row_amax[i] / Q                   (Q = 448 E4M3, 127 INT8, 7 INT4; 1 if 0)
 *     out[i, j] = code(in[i, j] / s_i) * s_i  (E4M3 RNE satfinite; integers RNE, clamp +-Q)
 * in, out: m x n fp32 row-major device buffers (in == out allowed), row_amax: m
 * fp32; all 16-byte aligned; n a power of two in [2, 32768]; finite inputs (SPEC
 * S:420 "pre: finite input").  Asynchronous on `stream`; errors as hadacore_fwht,
 * HADACORE_ERR_DTYPE for a qtype outside the enum.
 *
 * hadacore_row_sq_error: out[i] = sum_j (a[i, j] - b[i, j])^2 accumulated in fp64,
 * for m x n fp32 row-major device buffers (4-byte aligned; out 8-byte aligned).
 */
hadacore_status_t hadacore_fake_quant(const float* in, float* out, float* row_amax, int64_t m, int64_t n,
                                      hadacore_qtype_t qtype, int per_tensor, hadacore_stream_t stream);
hadacore_status_t hadacore_row_sq_error(const float* a, const float* b, double* out, int64_t m, int64_t n,
                                        hadacore_stream_t stream);

/*
 * Strided rows + fused quantization (NEXT-1 x NEXT-3): the transform of the rows of a
 * 2-level grid (as hadacore_fwht_strided: row (i, j) at in + i * in_stride_outer +
 * j * in_stride_inner elements) fused with the per-row quantization of
 * hadacore_fwht_quant, codes and scales written CONTIGUOUSLY in row order (i, j):
 * out_q is [m_outer * m_inner, n] bytes ([.., n/2] for INT4), row_scale has
 * m_outer * m_inner floats -- e.g. the Q (or K) heads of a fused QKV projection
 * [tokens, 3, H, d] rotated and quantized to FP8 in one pass for FP8 attention
 * (P:24).  n = 2^3..2^15; stride rules as hadacore_fwht_strided; the input is
 * not modified; none of the three ranges may overlap.
 */
hadacore_status_t hadacore_fwht_quant_strided(const void* in, void* out_q, float* row_scale, int64_t m_outer,
                                              int64_t m_inner, int64_t in_stride_outer, int64_t in_stride_inner,
                                              int64_t n, hadacore_dtype_t dtype, hadacore_qtype_t qtype, float scale,
                                              hadacore_stream_t stream);

/* Static, human-readable description of a status code (never NULL). */
const char* hadacore_status_string(hadacore_status_t status);

/* Library version as 10000 * major + 100 * minor + patch. */
int hadacore_version(void);

/*
 * Number of kernel launches one hadacore_fwht call with these arguments makes
 * (0 when m == 0, else 1), for launch accounting in benchmarks.
 */
int hadacore_launches_per_call(int64_t m, int64_t n);

/* The same for a given dtype (every path is one launch in the default build; the
 * HC_F32_TWO_PASS build takes two for fp32 at n = 2^15). */
int hadacore_launches_per_call_dtype(int64_t m, int64_t n, hadacore_dtype_t dtype);

#ifdef __cplusplus
}
#endif

#endif /* HADACORE_H_ */
