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
