/*
 * oracle/fwht_oracle.c -- plain, slow, obviously-correct fp64 CPU oracle for the
 * batched normalized Walsh-Hadamard transform of HadaCore (arXiv 2412.08832).
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and bench.py's
 * cpu_baseline / --impl reference legs may load this library.  It shares no code,
 * header, table or constant with the CUDA path (paper_2412_08832_b200/csrc) and
 * never includes or links anything from it.
 *
 * Citations: "P:NN" = /root/reference/PAPER.md line NN (section in brackets).
 *
 * What it computes (P:41 [Sec. 2.1 Hadamard Matrices]): for an m x n activation
 * matrix x (row-major, m rows, n = 2^k columns) and the n-sized Walsh-Hadamard
 * matrix H (entries +-1, built recursively by Sylvester's construction, P:45
 * [Sec. 2.2]), every row is replaced by  y_i = scale * H * x_i .  H is symmetric,
 * so this is also the "right-Hadamard transform" x * H (P:87 [Sec. 2.4]).
 * `scale` is the whole multiplier on the +-1 matrix; 1/sqrt(n) gives the
 * normalized (orthonormal) transform ("+-1/sqrt(d) ... when normalized").
 *
 * Two independent routes are provided:
 *  - oracle_fwht_f64: the FWHT listing of P:50-64 [Sec. 2.2], executed literally
 *    (h = 1, 2, 4, ...; butterflies a[j] = x + y, a[j+h] = x - y), except that the
 *    listing's per-iteration division by sqrt(2) is replaced by ONE
 *    multiplication by `scale` at the end (reading R3: identical in
 *    exact arithmetic, one rounding instead of k).
 *  - oracle_dense_entry_f64: the plain definition, one output at a time:
 *    y_l = scale * sum_j (-1)^popcount(j & l) * x_j   (the Sylvester sign rule,
 *    which the recursion H(2k) = [[H,H],[H,-H]] of P:45 produces).  O(n) per
 *    output; used to sample single outputs of full-size GPU runs.
 *
 * All arithmetic is IEEE fp64.  Rows are independent (P:77 [Sec. 2.3]) and are
 * split across POSIX threads; each row is processed by exactly one thread with the
 * same sequential loop, so the result does not depend on the thread count.
 */
#include <math.h>
#include <pthread.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

/* 0 on success, -1 if n is not a power of two >= 1. */
static int is_pow2(int64_t n) { return n >= 1 && (n & (n - 1)) == 0; }

/* The P:50-64 listing on one row a[0..n), in place, without the per-iteration
 * /sqrt(2); the caller applies `scale` once afterwards. */
static void fwht_listing_row(double* a, int64_t n) {
  for (int64_t h = 1; h < n; h *= 2) {              /* while h < len(a) */
    for (int64_t i = 0; i < n; i += 2 * h) {        /* range(0, len(a), 2h) */
      for (int64_t j = i; j < i + h; ++j) {         /* range(i, i + h) */
        double x = a[j];                            /* x = a[j] */
        double y = a[j + h];                        /* y = a[j + h] */
        a[j] = x + y;                               /* a[j] = x + y */
        a[j + h] = x - y;                           /* a[j + h] = x - y */
      }
    }
  }
}

typedef struct {
  const double* in;
  double* out;
  int64_t row_begin, row_end, n;
  double scale;
} job_t;

static void* worker(void* p) {
  job_t* jb = (job_t*)p;
  for (int64_t r = jb->row_begin; r < jb->row_end; ++r) {
    double* a = jb->out + r * jb->n;
    if (jb->in != jb->out) memcpy(a, jb->in + r * jb->n, (size_t)jb->n * sizeof(double));
    fwht_listing_row(a, jb->n);
    for (int64_t j = 0; j < jb->n; ++j) a[j] *= jb->scale;
  }
  return NULL;
}

/* out[i,:] = scale * H_n * in[i,:] for i in [0, m).  in may equal out.
 * threads <= 0 means "one thread".  Returns 0, or -1 on a bad argument. */
int oracle_fwht_f64(const double* in, double* out, int64_t m, int64_t n, double scale,
                    int threads) {
  if (m < 0 || !is_pow2(n) || (m > 0 && (!in || !out))) return -1;
  if (m == 0) return 0;
  if (threads < 1) threads = 1;
  if (threads > m) threads = (int)m;
  job_t* jobs = (job_t*)calloc((size_t)threads, sizeof(job_t));
  pthread_t* tids = (pthread_t*)calloc((size_t)threads, sizeof(pthread_t));
  if (!jobs || !tids) { free(jobs); free(tids); return -1; }
  for (int t = 0; t < threads; ++t) {
    jobs[t].in = in;
    jobs[t].out = out;
    jobs[t].n = n;
    jobs[t].scale = scale;
    jobs[t].row_begin = m * t / threads;
    jobs[t].row_end = m * (t + 1) / threads;
  }
  int spawned = 0;
  for (int t = 1; t < threads; ++t) {
    if (pthread_create(&tids[t], NULL, worker, &jobs[t]) != 0) break;
    spawned = t;
  }
  worker(&jobs[0]);
  for (int t = 1; t <= spawned; ++t) pthread_join(tids[t], NULL);
  /* rows of threads that failed to spawn are done here, sequentially */
  for (int t = spawned + 1; t < threads; ++t) worker(&jobs[t]);
  free(jobs);
  free(tids);
  return 0;
}

/* The definition, one output: scale * sum_j (-1)^popcount(j & l) * x[j]. */
double oracle_dense_entry_f64(const double* x, int64_t n, int64_t l, double scale) {
  double acc = 0.0;
  for (int64_t j = 0; j < n; ++j) {
    int odd = __builtin_popcountll((unsigned long long)(j & l)) & 1;
    acc += odd ? -x[j] : x[j];
  }
  return scale * acc;
}

/* The definition for a whole m x n matrix (O(m n^2); small n only). */
int oracle_dense_f64(const double* in, double* out, int64_t m, int64_t n, double scale) {
  if (m < 0 || !is_pow2(n) || (m > 0 && (!in || !out)) || in == out) return -1;
  for (int64_t r = 0; r < m; ++r)
    for (int64_t l = 0; l < n; ++l) out[r * n + l] = oracle_dense_entry_f64(in + r * n, n, l, scale);
  return 0;
}

/* ------------------------------------------------------------------------------
 * Symmetric per-row quantization of a transformed row (the
 * paper's stated future work "fused Hadamard transform and quantization"
 * [Sec. 5], and its FP8-attention use, P:180 [Sec. 4.2]).  SPEC S:423-431: scale =
 * max_abs / Q with Q = 448 (FP8 E4M3) or 127 (INT8); codes = round(x / scale);
 * an all-zero row has scale 1 and zero codes.
 *
 * qtype 0 = FP8 E4M3 (OCP "e4m3fn": bias 7, no infinities, 0x7F/0xFF = NaN, max
 *           finite 448): the code of the representable value nearest to x/scale,
 *           ties to the even code, magnitudes above 448 saturate to 448.
 * qtype 1 = INT8: round-half-to-even of x/scale, clamped to [-127, 127].
 * Everything in fp64; the e4m3 encoder enumerates the 127 non-negative finite codes.
 * ------------------------------------------------------------------------------ */
double oracle_e4m3_value(int code) {
  const int s = (code >> 7) & 1, e = (code >> 3) & 15, mant = code & 7;
  if (e == 15 && mant == 7) return NAN;
  double v = (e == 0) ? (mant / 8.0) * ldexp(1.0, -6) : (1.0 + mant / 8.0) * ldexp(1.0, e - 7);
  return s ? -v : v;
}

int oracle_e4m3_encode(double x) {
  if (x != x) return 0x7F;
  const int neg = x < 0;
  const double a = fabs(x);
  int best = 0;
  double best_err = INFINITY;
  for (int c = 0; c <= 0x7E; ++c) { /* non-negative finite codes in increasing order */
    const double err = fabs(oracle_e4m3_value(c) - a);
    if (err < best_err || (err == best_err && (c & 1) == 0)) {
      best = c;
      best_err = err;
    }
  }
  return (neg ? 0x80 : 0) | best; /* |x| > 448 lands on 0x7E (448): saturation */
}

/* qtype 2 = INT4 (SPEC quant_lab S:422 "Q = 7 (INT4)"): round-half-to-even of
 * x/scale, clamped to [-7, 7], one code per byte (two's complement). */
static double qmax_of(int qtype) { return qtype == 0 ? 448.0 : (qtype == 1 ? 127.0 : 7.0); }

static uint8_t encode(double v, int qtype) {
  if (qtype == 0) return (uint8_t)oracle_e4m3_encode(v);
  const double lim = qmax_of(qtype);
  double q = nearbyint(v); /* default rounding mode: to nearest, ties to even */
  if (q > lim) q = lim;
  if (q < -lim) q = -lim;
  return (uint8_t)(int8_t)q;
}

/* y: m x n fp64 (already transformed); codes: m x n bytes; scales: m doubles.
 * per_tensor = 0: one scale per row (SPEC "PerRow"); 1: one scale for the whole
 * matrix, max_abs over all m*n entries (SPEC "PerTensor"), repeated in
 * every scales[r]. */
int oracle_quantize_f64(const double* y, uint8_t* codes, double* scales, int64_t m, int64_t n, int qtype,
                        int per_tensor) {
  if (m < 0 || n < 1 || qtype < 0 || qtype > 2) return -1;
  const double qmax = qmax_of(qtype);
  double tmax = 0.0;
  if (per_tensor)
    for (int64_t i = 0; i < m * n; ++i) tmax = fmax(tmax, fabs(y[i]));
  for (int64_t r = 0; r < m; ++r) {
    const double* row = y + r * n;
    double amax = tmax;
    if (!per_tensor)
      for (int64_t j = 0; j < n; ++j) amax = fmax(amax, fabs(row[j]));
    const double s = amax > 0.0 ? amax / qmax : 1.0;
    scales[r] = s;
    for (int64_t j = 0; j < n; ++j) codes[r * n + j] = encode(amax > 0.0 ? row[j] / s : 0.0, qtype);
  }
  return 0;
}

int oracle_quantize_rows_f64(const double* y, uint8_t* codes, double* scales, int64_t m, int64_t n, int qtype) {
  return oracle_quantize_f64(y, codes, scales, m, n, qtype, 0);
}
