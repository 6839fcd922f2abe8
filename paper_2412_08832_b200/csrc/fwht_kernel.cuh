// fwht_kernel.cuh -- sm_100a kernel for the batched normalized Walsh-Hadamard
// transform (HadaCore, arXiv 2412.08832).  "P:NN" = /root/reference/PAPER.md line.
//
// Design:
//  * Warp-specialized CTAs scheduled by cluster launch control (one CTA per tile; resident
//    CTAs cancel not-yet-launched ones and take their tiles).  One producer warp streams
//    row tiles HBM -> shared memory into a STAGES-deep mbarrier ring -- 1-D bulk copies
//    (SASS UBLKCP) for contiguous n <= 256, 3-D/5-D TMA tensor copies (UTMALDG) for row
//    grids and n >= 512 -- and, for n >= 512, stores finished tiles back with TMA tensor
//    stores (UTMASTG).  Every element is read once and written once (P:264 in place:
//    tiles are disjoint and read before written).
//  * The Kronecker factors H_16 (x) ... (P:150 [Sec. 3.4]) are contractions on the
//    tensor cores with register operands (mma.sync m16n8k16, SASS HMMA), as in the
//    paper's Sec. 3: a 256-element fragment lives in one warp, 8 elements per
//    lane.  Unlike the paper we never transpose with shuffles/movmatrix: putting the
//    CONSTANT in the A operand and the data in the B operand makes each stage return
//    D = K * X^T, i.e. the transpose comes free, and two such stages give
//    K_b * X * K_a in natural orientation (P:109's "transpose, H16, transpose back").
//  * Rows longer than 256 (P:120-129 [Sec. 3.2]): the TMA box lays each row out with the
//    hardware 128-byte swizzle; phase 1 applies H_256 to every 256-chunk in place, phase
//    2 gathers fragments across chunks with ldmatrix/stmatrix .trans (bank-conflict free
//    because of the swizzle) and applies H_{n/256} (residual 2^a factors as H_2^a (x) I
//    blocks, P:146 [Sec. 3.3]); the TMA store un-swizzles.  With fused quantization the
//    two factors run in the other order (they commute) so that H_256 comes last and its
//    fp32 results stay in registers until the row maximum is known.
//  * Normalization: every stage multiplies by an exact power of two
//    (+-2^-floor(h/2) entries); the last stage accumulates in fp32 and multiplies by
//    s_res = scale * 2^E before the single round-to-nearest-even to 16 bits.
//  * bf16 (P:294 [App. C]): fp32 accumulate, cvt.rn.bf16x2 between stages.
//    fp16: fp16 accumulate between stages, fp32 in the last stage.
//
// The lane/register slot algebra is modelled and checked in tools/fragment_model.py.
#pragma once
#include <cuda.h>
#include <cuda_fp16.h>
#include <type_traits>
#include <cuda_runtime.h>
#include <stdint.h>

namespace hadacore {

enum : int { DT_F16 = 0, DT_BF16 = 1 };

// ------------------------------------------------------------------ PTX helpers
__device__ __forceinline__ uint32_t smem_addr(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_addr(bar)), "r"(count) : "memory");
}

__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_addr(bar)), "r"(bytes)
               : "memory");
}

__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_addr(bar)) : "memory");
}

// HC_WAIT_HINT (ns): suspend-time hint of the try_wait loop -- a waiting warp sleeps
// until the phase completes or the hint expires instead of re-issuing the probe
// (tools/tune.py A/B; 0 = no hint)
#ifndef HC_WAIT_HINT
#define HC_WAIT_HINT 0
#endif
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
#if HC_WAIT_HINT > 0
  asm volatile(
      "{\n\t.reg .pred p;\n"
      "WAIT_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1, %2;\n\t"
      "@!p bra WAIT_%=;\n}" ::"r"(smem_addr(bar)),
      "r"(parity), "n"(HC_WAIT_HINT)
      : "memory");
#else
  asm volatile(
      "{\n\t.reg .pred p;\n"
      "WAIT_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
      "@!p bra WAIT_%=;\n}" ::"r"(smem_addr(bar)),
      "r"(parity)
      : "memory");
#endif
}

__device__ __forceinline__ uint64_t policy_evict_first() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
  return p;
}

// Bulk copy global -> shared, completion counted on `bar` (SASS: UBLKCP.S.G).
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar,
                                         uint64_t policy) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint"
      " [%0], [%1], %2, [%3], %4;" ::"r"(smem_addr(dst)),
      "l"(src), "r"(bytes), "r"(smem_addr(bar)), "l"(policy)
      : "memory");
}

// HC_TRACE builds (tools/trace_pipeline.py): %globaltimer stamps of pipeline events of
// the first CTAs, read back with hadacore_trace_read().
#ifdef HC_TRACE
constexpr int kTraceCtas = 4, kTraceTiles = 48, kTraceEv = 8;
__device__ uint64_t g_trace[kTraceCtas][kTraceTiles][kTraceEv];
__device__ uint64_t g_span[1024][3];  // per CTA: first load issued, last tile done (warp 0), tiles done
__device__ __forceinline__ uint64_t gtime() {
  uint64_t t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
__device__ __forceinline__ void trace(int it, int ev) {
  if (blockIdx.x < kTraceCtas && it < kTraceTiles) {
    uint64_t t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    g_trace[blockIdx.x][it][ev] = t;
  }
}
#else
__device__ __forceinline__ void trace(int, int) {}
#endif

// HC_JITTER (test build libhadacore_jitter.so, tests/test_gpu_jitter.py): random
// nanosleeps at the synchronization points of the multi-role / multi-CTA kernels, so
// that the barrier protocols are exercised under perturbed timing; results must stay
// bitwise identical to the product build.
#ifdef HC_JITTER
__device__ __forceinline__ void jitter(uint32_t site, uint32_t it) {
  uint32_t h = (blockIdx.x * 0x9E3779B1u) ^ (threadIdx.x * 0x85EBCA77u) ^ (it * 0xC2B2AE3Du) ^ (site * 0x27D4EB2Fu);
  h ^= h >> 15;
  h *= 0x2C1B3C6Du;
  h ^= h >> 12;
  if ((h & 3u) == 0u) __nanosleep((h >> 8) & 4095u);  // a quarter of the time, up to ~4 us
}
#else
__device__ __forceinline__ void jitter(uint32_t, uint32_t) {}
#endif

// Programmatic dependent launch: let the next kernel be scheduled early, and wait
// for the previous kernel's completion (and memory flush) before touching memory.
__device__ __forceinline__ void pdl_launch_dependents() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }

// ---- tile scheduling.  Default: Blackwell cluster launch control (CLC).  The grid has
// one CTA per tile; a running CTA's producer cancels a not-yet-launched CTA with
// clusterlaunchcontrol.try_cancel and processes its tile instead, so fast SMs take
// more tiles than slow ones (static round-robin leaves the grid waiting for the
// slowest SMs: profiles/r01_pipeline_trace_*).  HC_STATIC_SCHED = persistent grid
// with static round-robin tiles, for A/B.
#ifdef HC_STATIC_SCHED
constexpr bool kClc = false;
#else
constexpr bool kClc = true;
#endif
// Control block at the start of the barrier area: CLC response (16 B), its mbarrier,
// and the tile id of every ring stage (-1 = no more tiles).
struct SchedCtl {
  uint4 clc_resp;
  uint64_t clc_bar;
  uint64_t pad;
  int stage_tile[16];
};
static_assert(sizeof(SchedCtl) == 96, "SchedCtl layout");

__device__ __forceinline__ void clc_request(SchedCtl* ctl) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], 16;" ::"r"(smem_addr(&ctl->clc_bar)) : "memory");
  asm volatile("clusterlaunchcontrol.try_cancel.async.shared::cta.mbarrier::complete_tx::bytes.b128 [%0], [%1];" ::"r"(
                   smem_addr(&ctl->clc_resp)),
               "r"(smem_addr(&ctl->clc_bar))
               : "memory");
}
// Waits for the pending request; returns the cancelled CTA's blockIdx.x, or -1 when
// every remaining CTA is already running (then no further request may be made).
__device__ __forceinline__ int64_t clc_result(SchedCtl* ctl, uint32_t& phase) {
  asm volatile(
      "{\n\t.reg .pred p;\n"
      "WAITC_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
      "@!p bra WAITC_%=;\n}" ::"r"(smem_addr(&ctl->clc_bar)),
      "r"(phase)
      : "memory");
  phase ^= 1u;
  uint4 r;
  asm volatile("ld.shared.v4.b32 {%0, %1, %2, %3}, [%4];"
               : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w)
               : "r"(smem_addr(&ctl->clc_resp))
               : "memory");
  uint32_t ok, x;
  asm volatile(
      "{\n\t.reg .b128 R;\n\t.reg .pred P;\n\t"
      "mov.b128 R, {%2, %3};\n\t"
      "clusterlaunchcontrol.query_cancel.is_canceled.pred.b128 P, R;\n\t"
      "selp.b32 %0, 1, 0, P;\n\t"
      "clusterlaunchcontrol.query_cancel.get_first_ctaid::x.b32.b128 %1, R;\n\t}"
      : "=r"(ok), "=r"(x)
      : "l"((uint64_t(r.y) << 32) | r.x), "l"((uint64_t(r.w) << 32) | r.z)
      : "memory");
  return ok ? int64_t(x) : -1;
}

__device__ __forceinline__ void fence_proxy_async_smem() {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}

__device__ __forceinline__ void named_bar_sync(int id, int nthreads) {
  asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(nthreads) : "memory");
}

// Shared-memory accesses are plain C++ on pointers into the dynamic smem array so
// that the compiler may interleave independent work items (ILP); cross-warp order
// is provided by the mbarrier / named-barrier asm (memory clobbers).
__device__ __forceinline__ uint32_t lds32(const uint8_t* p) { return *reinterpret_cast<const uint32_t*>(p); }
__device__ __forceinline__ void sts32(uint8_t* p, uint32_t v) { *reinterpret_cast<uint32_t*>(p) = v; }
__device__ __forceinline__ void lds64(const uint8_t* p, uint32_t& a, uint32_t& b) {
  const uint2 v = *reinterpret_cast<const uint2*>(p);
  a = v.x;
  b = v.y;
}
__device__ __forceinline__ void lds128(const uint8_t* p, uint32_t& a, uint32_t& b, uint32_t& c, uint32_t& d) {
  const uint4 v = *reinterpret_cast<const uint4*>(p);
  a = v.x;
  b = v.y;
  c = v.z;
  d = v.w;
}
__device__ __forceinline__ void stg_sh128(uint8_t* p, const uint32_t v[4]) {
  *reinterpret_cast<uint4*>(p) = make_uint4(v[0], v[1], v[2], v[3]);
}
__device__ __forceinline__ void stg32(uint16_t* p, uint32_t v) { *reinterpret_cast<uint32_t*>(p) = v; }
#ifndef HC_QPACK_N
#define HC_QPACK_N 0  // fused quantization: the n whose phase-B results are held as packed 16-bit y
#endif
// HC_STORE_HINT (A/B builds): output stores marked evict-first in L2 (st.global.cs and the
// TMA store's L2::cache_hint), like the input loads
#ifndef HC_STORE_HINT
#define HC_STORE_HINT 1  // measured +0.2-0.3 % on the sweep, up to +1 % per n (profiles/r01_ab_store_hint.txt)
#endif
__device__ __forceinline__ void stg64(uint16_t* p, uint32_t a, uint32_t b) {
#if HC_STORE_HINT
  asm volatile("st.global.cs.v2.b32 [%0], {%1, %2};" ::"l"(p), "r"(a), "r"(b) : "memory");
#else
  *reinterpret_cast<uint2*>(p) = make_uint2(a, b);
#endif
}
__device__ __forceinline__ void stg128(uint16_t* p, uint32_t a, uint32_t b, uint32_t c, uint32_t d) {
#if HC_STORE_HINT
  asm volatile("st.global.cs.v4.b32 [%0], {%1, %2, %3, %4};" ::"l"(p), "r"(a), "r"(b), "r"(c), "r"(d) : "memory");
#else
  *reinterpret_cast<uint4*>(p) = make_uint4(a, b, c, d);
#endif
}

// ------------------------------------------------------------------ packing
template <int DT>
__device__ __forceinline__ uint32_t pack2(float lo, float hi) {
  uint32_t r;
  if constexpr (DT == DT_F16) {
    asm("cvt.rn.f16x2.f32 %0, %1, %2;" : "=r"(r) : "f"(hi), "f"(lo));
  } else {
    asm("cvt.rn.bf16x2.f32 %0, %1, %2;" : "=r"(r) : "f"(hi), "f"(lo));
  }
  return r;
}

// ------------------------------------------------------------------ mma wrappers
// D(f32 x4) = A(16x16, 4 regs) * B(16x8, 2 regs)
template <int DT>
__device__ __forceinline__ void mma_f32(const uint32_t a[4], uint32_t b0, uint32_t b1, float d[4]) {
#ifdef HC_NOCOMPUTE  // diagnostic build (tools/tune.py): data movement only
  d[0] = __uint_as_float(b0); d[1] = __uint_as_float(b0 ^ a[0]); d[2] = __uint_as_float(b1); d[3] = __uint_as_float(b1);
  return;
#endif
  if constexpr (DT == DT_F16) {
    asm(
        "mma.sync.aligned.m16n8k16.row.col.f32.f16.f16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, "
        "{%10,%10,%10,%10};"
        : "=f"(d[0]), "=f"(d[1]), "=f"(d[2]), "=f"(d[3])
        : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b0), "r"(b1), "f"(0.f));
  } else {
    asm(
        "mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, "
        "{%10,%10,%10,%10};"
        : "=f"(d[0]), "=f"(d[1]), "=f"(d[2]), "=f"(d[3])
        : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b0), "r"(b1), "f"(0.f));
  }
}

// D(2 packed 16-bit regs) = A * B: fp16 accumulates in fp16, bf16 in fp32 then RNE.
template <int DT>
__device__ __forceinline__ void mma_pk(const uint32_t a[4], uint32_t b0, uint32_t b1, uint32_t& d01,
                                       uint32_t& d23) {
#ifdef HC_NOCOMPUTE
  d01 = b0 ^ a[1];
  d23 = b1;
  return;
#endif
  if constexpr (DT == DT_F16) {
    asm(
        "mma.sync.aligned.m16n8k16.row.col.f16.f16.f16.f16 {%0,%1}, {%2,%3,%4,%5}, {%6,%7}, {%8,%8};"
        : "=r"(d01), "=r"(d23)
        : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b0), "r"(b1), "r"(0u));
  } else {
    float d[4];
    mma_f32<DT>(a, b0, b1, d);
    d01 = pack2<DT>(d[0], d[1]);
    d23 = pack2<DT>(d[2], d[3]);
  }
}

// ------------------------------------------------------------------ constants
// Entry (i, k) of the 16x16 Kronecker product over 4 index bits, bit q being H_2
// (unnormalized +-1) if (hmask >> q) & 1, else I_2.
__device__ __forceinline__ float kron_entry(uint32_t hmask, int i, int k) {
  int sgn = 0;
#ifdef HC_NEGCTL  // negative-control build (tests/test_gpu_edge.py): one sign of H_16 flipped
  if (hmask == 0xFu && i == 3 && k == 5) sgn = 1;
#endif
#pragma unroll
  for (int q = 0; q < 4; ++q) {
    const int bi = (i >> q) & 1, bk = (k >> q) & 1;
    if ((hmask >> q) & 1u) {
      sgn ^= bi & bk;
    } else if (bi != bk) {
      return 0.f;
    }
  }
  return sgn ? -1.f : 1.f;
}

__host__ __device__ constexpr int popc4(uint32_t m) {
  return int(m & 1u) + int((m >> 1) & 1u) + int((m >> 2) & 1u) + int((m >> 3) & 1u);
}
// exact per-stage normalization 2^-floor(h/2) (h = number of H_2 factors)
__host__ __device__ constexpr int stage_shift(uint32_t m) { return popc4(m) / 2; }

__device__ __forceinline__ uint32_t opaque(uint32_t v) {
  uint32_t r;
  asm volatile("mov.b32 %0, %1;" : "=r"(r) : "r"(v));
  return r;
}

// A-operand (row-major 16x16) registers of 2^-shift * K(hmask) for this lane.
template <int DT>
__device__ __forceinline__ void make_const_a(uint32_t hmask, uint32_t a[4]) {
  const int lane = threadIdx.x & 31, g = lane >> 2, t = lane & 3;
  const float s = ldexpf(1.f, -stage_shift(hmask));
  a[0] = pack2<DT>(s * kron_entry(hmask, g, 2 * t), s * kron_entry(hmask, g, 2 * t + 1));
  a[1] = pack2<DT>(s * kron_entry(hmask, g + 8, 2 * t), s * kron_entry(hmask, g + 8, 2 * t + 1));
  a[2] = pack2<DT>(s * kron_entry(hmask, g, 2 * t + 8), s * kron_entry(hmask, g, 2 * t + 9));
  a[3] = pack2<DT>(s * kron_entry(hmask, g + 8, 2 * t + 8), s * kron_entry(hmask, g + 8, 2 * t + 9));
#pragma unroll
  for (int i = 0; i < 4; ++i) a[i] = opaque(a[i]);
}

// B-operand (16x8, "col") registers of columns [8T, 8T+8) of 2^-shift * K(hmask).
template <int DT>
__device__ __forceinline__ void make_const_b(uint32_t hmask, int T, uint32_t b[2]) {
  const int lane = threadIdx.x & 31, g = lane >> 2, t = lane & 3;
  const float s = ldexpf(1.f, -stage_shift(hmask));
  const int n = 8 * T + g;
  b[0] = pack2<DT>(s * kron_entry(hmask, 2 * t, n), s * kron_entry(hmask, 2 * t + 1, n));
  b[1] = pack2<DT>(s * kron_entry(hmask, 2 * t + 8, n), s * kron_entry(hmask, 2 * t + 9, n));
  b[0] = opaque(b[0]);
  b[1] = opaque(b[1]);
}

// ------------------------------------------------------------------ stages
// "const-A" stage (P:101 two m16n8k16 mma per 16x16 fragment): tile T's B operand
// is (b_T0, b_T1); D = K * B, so the result comes back transposed for free.
// Outputs y0 = D_0 rows 0..7, y1 = D_0 rows 8..15, y2 = D_1 rows 0..7, y3 = D_1 rows 8..15.
template <int DT>
__device__ __forceinline__ void stage_ca(const uint32_t a[4], uint32_t b00, uint32_t b01, uint32_t b10,
                                         uint32_t b11, uint32_t y[4]) {
  mma_pk<DT>(a, b00, b01, y[0], y[1]);
  mma_pk<DT>(a, b10, b11, y[2], y[3]);
}
// Same with fp32 results d[0..3] = tile 0 (pairs y0, y1), d[4..7] = tile 1 (y2, y3).
template <int DT>
__device__ __forceinline__ void stage_ca_f32(const uint32_t a[4], uint32_t b00, uint32_t b01, uint32_t b10,
                                             uint32_t b11, float d[8]) {
  mma_f32<DT>(a, b00, b01, d);
  mma_f32<DT>(a, b10, b11, d + 4);
}
// "data-as-A" stage: D = X * Bc with X (4 regs) in the A layout; D has X's layout.
template <int DT>
__device__ __forceinline__ void stage_da_f32(const uint32_t x[4], const uint32_t bc0[2], const uint32_t bc1[2],
                                             float d[8]) {
  mma_f32<DT>(x, bc0[0], bc0[1], d);      // output columns 0..7  -> regs R0 (rows g), R1 (rows g+8)
  mma_f32<DT>(x, bc1[0], bc1[1], d + 4);  // output columns 8..15 -> R2, R3
}
// Packed fp32 butterfly on two adjacent pairs (SASS FADD2, sm_100): (a0, a1), (b0, b1) <-
// (a + b, a - b) element-wise, IEEE round-to-nearest like two scalar FADDs -- half the
// issue slots of the scalar butterflies (P:50-64 listing's x + y, x - y).
__device__ __forceinline__ void bfly2(float& a0, float& a1, float& b0, float& b1) {
#ifdef HC_SCALAR_BFLY  // A/B builds: scalar FADDs
  const float s0 = a0 + b0, s1 = a1 + b1, d0 = a0 - b0, d1 = a1 - b1;
  a0 = s0; a1 = s1; b0 = d0; b1 = d1;
#else
  asm("{.reg .b64 a, b, s, d;\n mov.b64 a, {%0,%1};\n mov.b64 b, {%2,%3};\n add.rn.f32x2 s, a, b;\n"
      " sub.rn.f32x2 d, a, b;\n mov.b64 {%0,%1}, s;\n mov.b64 {%2,%3}, d;}"
      : "+f"(a0), "+f"(a1), "+f"(b0), "+f"(b1));
#endif
}
// fp32 butterflies between two 8-value fragments (a chunk bit held across a lane's fragments)
__device__ __forceinline__ void bfly8(float a[8], float b[8]) {
#pragma unroll
  for (int e = 0; e < 8; e += 2) bfly2(a[e], a[e + 1], b[e], b[e + 1]);
}
// Two chunk-bit groups at once (n >= 8192): H_16 over the A fragment's column bits as a
// data-as-A stage (layout kept), then H_2 over the fragment's row-half bit (the ldmatrix
// matrix index bit j0: d[0..1], d[4..5] are rows g, d[2..3], d[6..7] rows g + 8) as fp32
// butterflies in registers -- 2 HMMA instead of two const-A stages (4 HMMA and a 16-bit
// intermediate).  HC_J0_MMA builds keep the const-A pair for A/B.
template <int DT>
__device__ __forceinline__ void stage_da_j0_f32(const uint32_t x[4], const uint32_t bc0[2], const uint32_t bc1[2],
                                                float d[8]) {
  stage_da_f32<DT>(x, bc0, bc1, d);
  bfly2(d[0], d[1], d[2], d[3]);
  bfly2(d[4], d[5], d[6], d[7]);
}
#ifdef HC_J0_MMA
constexpr bool kJ0Mma = true;
#else
constexpr bool kJ0Mma = false;
#endif

// fp32 epilogue: * s_res (exact normalization remainder), one RNE rounding to 16 bits.
// The multiplies are packed (mul.rn.f32x2, SASS FMUL2: IEEE-identical to two FMULs).
template <int DT>
__device__ __forceinline__ void scale_pack(const float d[8], float s_res, uint32_t y[4]) {
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    float a = d[2 * i], b = d[2 * i + 1];
#ifndef HC_SCALAR_BFLY
    asm("{.reg .b64 t, s;\n mov.b64 t, {%0,%1};\n mov.b64 s, {%2,%2};\n mul.rn.f32x2 t, t, s;\n mov.b64 {%0,%1}, t;}"
        : "+f"(a), "+f"(b)
        : "f"(s_res));
#else
    a *= s_res;
    b *= s_res;
#endif
    y[i] = pack2<DT>(a, b);
  }
}

// ------------------------------------------------------------------ SIMT ablation
// HC_SIMT builds replace every tensor-core stage by fp32 warp-shuffle butterflies
// on the same fragment (tools/tune.py "tuned-simt"), to measure whether the mma
// contractions beat shuffle butterflies (north_star).  Fragment value index
// i = 2*j + h (register X_j, half h); fragment bits: b0 = h, b1/b2 = lane bits 0/1,
// b3 = j bit 1, b4..b6 = lane bits 2..4, b7 = j bit 0.
template <int DT>
__device__ __forceinline__ void unpack8(const uint32_t x[4], float v[8]) {
#pragma unroll
  for (int j = 0; j < 4; ++j) {
    if constexpr (DT == DT_F16) {
      const float2 f = __half22float2(*reinterpret_cast<const __half2*>(&x[j]));
      v[2 * j] = f.x;
      v[2 * j + 1] = f.y;
    } else {
      v[2 * j] = __uint_as_float(x[j] << 16);
      v[2 * j + 1] = __uint_as_float(x[j] & 0xffff0000u);
    }
  }
}
// HC_SIMT_SCALAR: the round-1 scalar form (one SHFL + one FFMA per value and lane bit);
// default: packed f32x2 math -- in-register bits as FADD2 butterfly pairs, lane bits as
// two SHFL + one FFMA2 per value pair (SURVEY.md 7 variant V-B)
__device__ __forceinline__ void simt_butterflies(float v[8], uint32_t mask8) {
  const int lane = threadIdx.x & 31;
  constexpr int reg_bit[8] = {0, -1, -1, 2, -1, -1, -1, 1};   // b -> bit of the value index
  constexpr int lane_bit[8] = {-1, 0, 1, -1, 2, 3, 4, -1};    // b -> lane bit
#pragma unroll
  for (int b = 0; b < 8; ++b) {
    if (!((mask8 >> b) & 1u)) continue;
    if (reg_bit[b] >= 0) {
      const int st = 1 << reg_bit[b];
#ifdef HC_SIMT_SCALAR
#pragma unroll
      for (int i = 0; i < 8; ++i)
        if (!(i & st)) {
          const float p0 = v[i], p1 = v[i | st];
          v[i] = p0 + p1;
          v[i | st] = p0 - p1;
        }
#else
#pragma unroll
      for (int k = 0; k < 4; k += 2) {  // the k-th index with bit st clear: (k / st) * 2 st + k % st
        const int i0 = (k / st) * 2 * st + k % st, i1 = ((k + 1) / st) * 2 * st + (k + 1) % st;
        bfly2(v[i0], v[i1], v[i0 | st], v[i1 | st]);
      }
#endif
    } else {
      const int lb = 1 << lane_bit[b];
      const float sg = (lane & lb) ? -1.f : 1.f;
#ifdef HC_SIMT_SCALAR
#pragma unroll
      for (int i = 0; i < 8; ++i) v[i] = fmaf(v[i], sg, __shfl_xor_sync(0xffffffffu, v[i], lb));
#else
#pragma unroll
      for (int i = 0; i < 8; i += 2) {
        const float q0 = __shfl_xor_sync(0xffffffffu, v[i], lb), q1 = __shfl_xor_sync(0xffffffffu, v[i + 1], lb);
        float a = v[i], c = v[i + 1];
        asm("{.reg .b64 t, s, u;\n mov.b64 t, {%0,%1};\n mov.b64 s, {%2,%2};\n mov.b64 u, {%3,%4};\n"
            " fma.rn.f32x2 t, t, s, u;\n mov.b64 {%0,%1}, t;}"
            : "+f"(a), "+f"(c)
            : "f"(sg), "f"(q0), "f"(q1));
        v[i] = a;
        v[i + 1] = c;
      }
#endif
    }
  }
}
__device__ __forceinline__ void mul2(float& a, float& b, float m);
template <int DT>
__device__ __forceinline__ void simt_fwht_pack(const uint32_t x[4], uint32_t mask8, float mul, uint32_t z[4]) {
  float v[8];
  unpack8<DT>(x, v);
  simt_butterflies(v, mask8);
#pragma unroll
  for (int j = 0; j < 4; ++j) {
    mul2(v[2 * j], v[2 * j + 1], mul);
    z[j] = pack2<DT>(v[2 * j], v[2 * j + 1]);
  }
}

// ------------------------------------------------------------------ fused quantization
// NEXT-1 ("fused Hadamard transform and quantization"):
// per-row symmetric scale s = max|y| / Q (Q = 448 for FP8 E4M3, 127 for INT8; s = 1
// for an all-zero row), codes = RNE(y / s) (E4M3 saturating, INT8 clamped to +-127).
// A non-finite value in a row makes that row's scale non-finite.
enum : int { QT_NONE = -1, QT_E4M3 = 0, QT_INT8 = 1, QT_INT4 = 2 };
template <int QT>
__host__ __device__ constexpr float qmax_of() {
  return QT == QT_E4M3 ? 448.f : (QT == QT_INT8 ? 127.f : 7.f);
}
// INT4 codes ("Q = 7 (INT4)", QuaRot-style 4-bit activations): two
// per byte, element 2j in the low nibble of byte j (two's complement).  Bytes in
// b0..b3 hold the codes' two's-complement low bytes; returns the 4 nibbles in 16 bits.
__device__ __forceinline__ uint32_t nibbles4(uint32_t b0, uint32_t b1, uint32_t b2, uint32_t b3) {
  const uint32_t w = __byte_perm(__byte_perm(b0, b1, 0x0040), __byte_perm(b2, b3, 0x0040), 0x5410) & 0x0F0F0F0Fu;
  return __byte_perm(w | (w >> 4), 0u, 0x0020) & 0xFFFFu;  // bytes 0 and 2 of w | w >> 4
}
// max of |v| that propagates NaN (max.NaN, one FMNMX.NAN): a NaN anywhere in a row
// poisons the row's scale, an Inf makes it Inf
__device__ __forceinline__ float absmax_nan(float acc, float v) {
  float r;
  asm("max.NaN.f32 %0, %1, %2;" : "=f"(r) : "f"(acc), "f"(fabsf(v)));
  return r;
}
// warp-wide max of non-negative floats (or +NaN): their bit patterns order like
// unsigned integers (NaN > Inf > finite), so one redux.sync.max.u32 (REDUX) does it
__device__ __forceinline__ float warp_absmax(float v) {
  return __uint_as_float(__reduce_max_sync(0xffffffffu, __float_as_uint(v)));
}
template <int QT>
__device__ __forceinline__ uint32_t quant4(float a, float b, float c, float d) {
  if constexpr (QT == QT_E4M3) {
    uint16_t lo, hi;
    asm("cvt.rn.satfinite.e4m3x2.f32 %0, %1, %2;" : "=h"(lo) : "f"(b), "f"(a));
    asm("cvt.rn.satfinite.e4m3x2.f32 %0, %1, %2;" : "=h"(hi) : "f"(d), "f"(c));
    return uint32_t(lo) | (uint32_t(hi) << 16);
  } else if constexpr (QT == QT_INT4) {
    const float a2 = fminf(fmaxf(rintf(a), -7.f), 7.f), b2 = fminf(fmaxf(rintf(b), -7.f), 7.f);
    const float c2 = fminf(fmaxf(rintf(c), -7.f), 7.f), d2 = fminf(fmaxf(rintf(d), -7.f), 7.f);
    return nibbles4(uint32_t(int(a2)), uint32_t(int(b2)), uint32_t(int(c2)), uint32_t(int(d2)));
  } else {
    // RNE with saturation to [-128, 127]; -128 cannot occur because |v| <= Q (up to
    // the rounding of the reciprocal, which stays below 127.5)
    int qa, qb, qc, qd;
    asm("cvt.rni.sat.s8.f32 %0, %1;" : "=r"(qa) : "f"(a));
    asm("cvt.rni.sat.s8.f32 %0, %1;" : "=r"(qb) : "f"(b));
    asm("cvt.rni.sat.s8.f32 %0, %1;" : "=r"(qc) : "f"(c));
    asm("cvt.rni.sat.s8.f32 %0, %1;" : "=r"(qd) : "f"(d));
    return __byte_perm(__byte_perm(uint32_t(qa), uint32_t(qb), 0x0040), __byte_perm(uint32_t(qc), uint32_t(qd), 0x0040),
                       0x5410);
  }
}
// Fast path of the fused quantization (rows whose max lies in [2^-100, hi]: finite,
// non-zero, no NaN, no fp32-subnormal reciprocal): packed f32x2 math (FMUL2 / FFMA2)
// and, for INT8, round-to-nearest-even by the 1.5 * 2^23 trick -- one FFMA2 rounds
// the exact product v * m to an integer held in the low mantissa bits, so no F2I.
// |v * m| <= Q (1 + 2^-8)(1 + 2^-22) < 127.5 for the 16-bit image (RNE of y, which is
// <= amax (1 + 2^-8)) and the fp32 accumulators alike, so no clamp is needed.
__device__ __forceinline__ void mul2(float& a, float& b, float m) {
  asm("{.reg .b64 t, s;\n mov.b64 t, {%0,%1};\n mov.b64 s, {%2,%2};\n mul.rn.f32x2 t, t, s;\n mov.b64 {%0,%1}, t;}"
      : "+f"(a), "+f"(b)
      : "f"(m));
}
__device__ __forceinline__ void fma2(float& a, float& b, float m, float c) {
  asm("{.reg .b64 t, s, u;\n mov.b64 t, {%0,%1};\n mov.b64 s, {%2,%2};\n mov.b64 u, {%3,%3};\n"
      " fma.rn.f32x2 t, t, s, u;\n mov.b64 {%0,%1}, t;}"
      : "+f"(a), "+f"(b)
      : "f"(m), "f"(c));
}
__device__ __forceinline__ float rcp_ftz(float x) {
  float r;
  asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(x));
  return r;
}
__device__ __forceinline__ bool quant_fast_range(float amax, float hi) {
  return amax >= 0x1p-100f && amax <= hi;  // false for 0, NaN, Inf
}
template <int QT>
__device__ __forceinline__ uint32_t quant4_fast(float a, float b, float c, float d, float m) {
  if constexpr (QT == QT_E4M3) {
    fma2(a, b, m, 0.f);  // + 0: an exact zero codes as +0 (0x00) whatever the multiplier's sign
    fma2(c, d, m, 0.f);
    uint16_t lo, hi;
    asm("cvt.rn.satfinite.e4m3x2.f32 %0, %1, %2;" : "=h"(lo) : "f"(b), "f"(a));
    asm("cvt.rn.satfinite.e4m3x2.f32 %0, %1, %2;" : "=h"(hi) : "f"(d), "f"(c));
    return uint32_t(lo) | (uint32_t(hi) << 16);
  } else {
    if constexpr (QT == QT_INT4) {
      // |v m| <= 7 (1 + 2^-8)(1 + 2^-22) < 7.5.  Rounding with the addend 1.5 * 2^23 + 8
      // leaves r + 8 in [1, 15] in the low mantissa bits (above them only the 2^22
      // bit): an offset-binary nibble with clean neighbours, so a + 16 b + 256 c +
      // 4096 d (integer multiply-adds) assembles four of them, and XOR 8 per nibble
      // turns offset binary into two's complement.  Bits above 15 are not cleared
      // (callers keep the low 16 bits).
      fma2(a, b, m, 12582920.f);  // 1.5 * 2^23 + 8 (even: ties stay ties-to-even)
      fma2(c, d, m, 12582920.f);
      uint32_t t = __float_as_uint(a) + 16u * __float_as_uint(b);
      t += 256u * __float_as_uint(c);
      t += 4096u * __float_as_uint(d);
      return t ^ 0x8888u;
    }
    fma2(a, b, m, 12582912.f);  // 1.5 * 2^23
    fma2(c, d, m, 12582912.f);
    return __byte_perm(__byte_perm(__float_as_uint(a), __float_as_uint(b), 0x0040),
                       __byte_perm(__float_as_uint(c), __float_as_uint(d), 0x0040), 0x5410);
  }
}
__device__ __forceinline__ void stg16_if(void* p, uint32_t v, bool pred) {
  asm volatile("{.reg .pred q;\n .reg .b16 h;\n setp.ne.b32 q, %2, 0;\n cvt.u16.u32 h, %1;\n @q st.global.b16 [%0], h;}"
               ::"l"(p), "r"(v), "r"(int(pred))
               : "memory");
}
// predicated global stores (no divergent branch around the epilogue)
__device__ __forceinline__ void stg32_if(void* p, uint32_t v, bool pred) {
  asm volatile("{.reg .pred q;\n setp.ne.b32 q, %2, 0;\n @q st.global.b32 [%0], %1;}" ::"l"(p), "r"(v),
               "r"(int(pred))
               : "memory");
}
__device__ __forceinline__ void stg64_if(void* p, uint32_t a, uint32_t b, bool pred) {
  asm volatile("{.reg .pred q;\n setp.ne.b32 q, %3, 0;\n @q st.global.v2.b32 [%0], {%1, %2};}" ::"l"(p), "r"(a),
               "r"(b), "r"(int(pred))
               : "memory");
}
__device__ __forceinline__ void stf32_if(float* p, float v, bool pred) {
  asm volatile("{.reg .pred q;\n setp.ne.b32 q, %2, 0;\n @q st.global.f32 [%0], %1;}" ::"l"(p), "f"(v),
               "r"(int(pred))
               : "memory");
}

// row scale s = amax / Q and the code multiplier Q / amax (amax = max |y| >= 0, Inf or NaN)
template <int QT>
__device__ __forceinline__ void row_scale_of(float amax, float& scale, float& inv) {
  const bool pos = amax > 0.f;  // false for 0 and NaN
  scale = pos ? amax * (1.f / qmax_of<QT>()) : (amax == 0.f ? 1.f : amax);
  float r;
  asm("rcp.approx.f32 %0, %1;" : "=f"(r) : "f"(amax));  // MUFU.RCP; codes tolerate its ~1 ulp
  inv = pos ? qmax_of<QT>() * r : (amax == 0.f ? 0.f : amax);
}

__device__ __forceinline__ void ldsm_x4_t(uint32_t addr, uint32_t r[4]) {
  asm volatile("ldmatrix.sync.aligned.m8n8.x4.trans.shared.b16 {%0,%1,%2,%3}, [%4];"
               : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3])
               : "r"(addr)
               : "memory");
}
__device__ __forceinline__ void stsm_x4_t(uint32_t addr, const uint32_t r[4]) {
  asm volatile("stmatrix.sync.aligned.m8n8.x4.trans.shared.b16 [%0], {%1,%2,%3,%4};" ::"r"(addr), "r"(r[0]),
               "r"(r[1]), "r"(r[2]), "r"(r[3])
               : "memory");
}

// ------------------------------------------------------------------ per-n plans
template <int N>
__host__ __device__ constexpr int log2_n() {
  int k = 0;
  while ((1 << k) < N) ++k;
  return k;
}

// Phase 2 of rows with n = 256 * 2^Q (tools/fragment_model.py
// planL/check_rowL).  A phase-2 fragment is one ldmatrix.x4.trans: lane L = 8j + r
// supplies the address of a 16-byte granule (8 consecutive elements) for matrix j,
// row r.  Slot bits r0 r1 r2 j0 j1 (+ per-lane extra fragments x0 x1, + loop bits):
//   chunk bits -> slots in the order r0, r1, r2, j1, j0, x0, x1 (first Q);
//   granule bits -> the remaining slots (low bits first), loop bits on top.
// Contraction: M columns (h, t0, t1, j1) = (r0, r1, r2, j1) via data-as-A (one
// stage); j0 via a second const-A stage (Q >= 5); x0, x1 via fp32 butterflies
// across per-lane fragments (Q >= 6).  Swizzle: granule ^= chunk & (2^min(Q,3) - 1).
template <int Q>
struct PlanL {
  static constexpr int nx = Q > 5 ? Q - 5 : 0;           // extra per-lane fragments (log2)
  static constexpr bool two_stage = Q >= 5;              // j0 is a chunk bit
  static constexpr uint32_t mask_a = (Q >= 4) ? 0xFu : ((1u << Q) - 1u);
  static constexpr int nloop_bits = Q <= 4 ? Q : 5;      // granule bits on the loop index
  static constexpr uint32_t swz_mask = (1u << (Q < 3 ? Q : 3)) - 1u;
};

// exponent E of the exact power-of-two normalization applied by the constants
template <int N>
__host__ __device__ constexpr int total_shift() {
  if constexpr (N == 128) return stage_shift(0xFu) + stage_shift(0x7u);
  else if constexpr (N == 256) return 2 * stage_shift(0xFu);
  else return 2 * stage_shift(0xFu) + stage_shift(PlanL<log2_n<N>() - 8>::mask_a);
}

// ------------------------------------------------------------------ TMA tensor helpers
__device__ __forceinline__ void tma_prefetch(const void* tmap) {
  asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(tmap)) : "memory");
}
// 4-D tiled TMA load (SASS UTMALDG) with completion on an mbarrier.
__device__ __forceinline__ void tma_load_4d(void* dst, const void* tmap, int c0, int c1, int c2, int c3,
                                            uint64_t* bar, uint64_t policy) {
  asm volatile(
      "cp.async.bulk.tensor.4d.shared::cluster.global.tile.mbarrier::complete_tx::bytes.L2::cache_hint"
      " [%0], [%1, {%2, %3, %4, %5}], [%6], %7;" ::"r"(smem_addr(dst)),
      "l"(reinterpret_cast<uint64_t>(tmap)), "r"(c0), "r"(c1), "r"(c2), "r"(c3), "r"(smem_addr(bar)), "l"(policy)
      : "memory");
}
// 4-D tiled TMA store (SASS UTMASTG), bulk-group completion.
__device__ __forceinline__ void tma_store_4d(const void* tmap, int c0, int c1, int c2, int c3, const void* src) {
  asm volatile("cp.async.bulk.tensor.4d.global.shared::cta.tile.bulk_group [%0, {%1, %2, %3, %4}], [%5];" ::"l"(
                   reinterpret_cast<uint64_t>(tmap)),
               "r"(c0), "r"(c1), "r"(c2), "r"(c3), "r"(smem_addr(src))
               : "memory");
}
// 3-D / 5-D tiled TMA loads and 5-D store (the row-grid views of DESIGN.md "Row grids").
__device__ __forceinline__ void tma_load_3d(void* dst, const void* tmap, int c0, int c1, int c2, uint64_t* bar,
                                            uint64_t policy) {
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes.L2::cache_hint"
      " [%0], [%1, {%2, %3, %4}], [%5], %6;" ::"r"(smem_addr(dst)),
      "l"(reinterpret_cast<uint64_t>(tmap)), "r"(c0), "r"(c1), "r"(c2), "r"(smem_addr(bar)), "l"(policy)
      : "memory");
}
__device__ __forceinline__ void tma_store_3d(const void* tmap, int c0, int c1, int c2, const void* src) {
#if HC_STORE_HINT
  asm volatile("cp.async.bulk.tensor.3d.global.shared::cta.tile.bulk_group.L2::cache_hint [%0, {%1, %2, %3}], [%4], %5;" ::"l"(
                   reinterpret_cast<uint64_t>(tmap)),
               "r"(c0), "r"(c1), "r"(c2), "r"(smem_addr(src)), "l"(policy_evict_first())
               : "memory");
#else
  asm volatile("cp.async.bulk.tensor.3d.global.shared::cta.tile.bulk_group [%0, {%1, %2, %3}], [%4];" ::"l"(
                   reinterpret_cast<uint64_t>(tmap)),
               "r"(c0), "r"(c1), "r"(c2), "r"(smem_addr(src))
               : "memory");
#endif
}
__device__ __forceinline__ void tma_load_5d(void* dst, const void* tmap, int c0, int c1, int c2, int c3, int c4,
                                            uint64_t* bar, uint64_t policy) {
  asm volatile(
      "cp.async.bulk.tensor.5d.shared::cluster.global.tile.mbarrier::complete_tx::bytes.L2::cache_hint"
      " [%0], [%1, {%2, %3, %4, %5, %6}], [%7], %8;" ::"r"(smem_addr(dst)),
      "l"(reinterpret_cast<uint64_t>(tmap)), "r"(c0), "r"(c1), "r"(c2), "r"(c3), "r"(c4), "r"(smem_addr(bar)),
      "l"(policy)
      : "memory");
}
__device__ __forceinline__ void tma_store_5d(const void* tmap, int c0, int c1, int c2, int c3, int c4, const void* src) {
#if HC_STORE_HINT
  asm volatile("cp.async.bulk.tensor.5d.global.shared::cta.tile.bulk_group.L2::cache_hint [%0, {%1, %2, %3, %4, %5}], [%6], %7;" ::"l"(
                   reinterpret_cast<uint64_t>(tmap)),
               "r"(c0), "r"(c1), "r"(c2), "r"(c3), "r"(c4), "r"(smem_addr(src)), "l"(policy_evict_first())
               : "memory");
#else
  asm volatile("cp.async.bulk.tensor.5d.global.shared::cta.tile.bulk_group [%0, {%1, %2, %3, %4, %5}], [%6];" ::"l"(
                   reinterpret_cast<uint64_t>(tmap)),
               "r"(c0), "r"(c1), "r"(c2), "r"(c3), "r"(c4), "r"(smem_addr(src))
               : "memory");
#endif
}
__device__ __forceinline__ void bulk_commit() { asm volatile("cp.async.bulk.commit_group;" ::: "memory"); }
__device__ __forceinline__ void bulk_wait_read_all() { asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory"); }
__device__ __forceinline__ void bulk_wait_all() { asm volatile("cp.async.bulk.wait_group 0;" ::: "memory"); }
template <int PENDING>
__device__ __forceinline__ void bulk_wait_read() {
  asm volatile("cp.async.bulk.wait_group.read %0;" ::"n"(PENDING) : "memory");
}

// ------------------------------------------------------------------ row grids
// Rows are a 2-level grid (NEXT-3 "strided / multi-head layouts"): row (i, j), i <
// m_outer, j < m_inner, lives at base + i*stride_outer + j*stride_inner elements
// (contiguous m x n: m_outer = m, m_inner = 1).  A pipeline tile is a rectangle of
// bo outer x bi inner rows (bi a power of two, bi * bo = TILE_ROWS), matching the
// TMA box, numbered tile = outer_block * nib + inner_block; rows past either edge
// are zero-filled on load and skipped on store.
struct RowGrid {
  int64_t m_outer, m_inner;
  int64_t out_so, out_si;  // output strides in elements (16-bit outputs)
  int64_t nib;             // inner blocks = ceil(m_inner / bi)
  int64_t num_tiles;
  int32_t lbi, bo;         // log2(bi), bo
  // non-null when the input rows are one contiguous m x n block (m_inner = 1,
  // stride_outer = n): fwht_kernel then loads a tile with one 1-D bulk copy of its
  // valid rows instead of the 3-D tensor box, whose 256-byte box rows (n = 128)
  // measured 6-9 % slower (profiles/r01_ab_strided.txt)
  const uint16_t* flat_in;
  // non-null when the inner rows are contiguous (stride_inner = n, e.g. the Q and K heads
  // of a token): fwht_kernel then loads each of a tile's bo outer row blocks with one 1-D
  // bulk copy of its valid rows (row r = ob * bi + jj of the tile) instead of a 3-D box
  const uint16_t* rows_in;
  int64_t in_so;
  // fwht_small_kernel row grids: log2 of the n-element rows per grid row (the grid then
  // describes contiguous outer row blocks as pseudo-rows of 2^lp rows; 0 = rows of n)
  int32_t lp;
};
struct TileRows {
  int64_t i0, j0;
  int lbi;
  __device__ __forceinline__ TileRows(const RowGrid& g, int64_t tile) : lbi(g.lbi) {
    const int64_t ob = tile / g.nib, ib = tile - ob * g.nib;
    i0 = ob * g.bo;
    j0 = ib << g.lbi;
  }
  // tile row r -> (i, j); false if (i, j) is outside the grid
  __device__ __forceinline__ bool at(const RowGrid& g, int r, int64_t& i, int64_t& j) const {
    i = i0 + (r >> lbi);
    j = j0 + (r & ((1 << lbi) - 1));
    return i < g.m_outer && j < g.m_inner;
  }
};
// The same per tile, with the epilogue's per-row work reduced to 32-bit tests and one
// wide multiply-add: rows (r >> lbi, r & mask) of the box are valid below (ni, nj), and
// row r's linear index (i * m_inner + j: codes/scales) and output element offset
// (i * out_so + j * out_si) are bases plus small multiples.
struct TileRowsFast {
  int64_t lin0, off0;  // i0 * m_inner + j0, i0 * out_so + j0 * out_si
  int ni, nj, lbi;
  // whole inner rows per box (m_inner == bi, e.g. the Q and K heads of a token): row r of
  // the box is linear row lin0 + r, valid below ni * bi
  __device__ __forceinline__ bool linear_rows(const RowGrid& g) const {
    return g.nib == 1 && g.m_inner == (int64_t(1) << lbi);
  }
  __device__ __forceinline__ TileRowsFast(const RowGrid& g, int64_t tile) : lbi(g.lbi) {
    const int64_t ob = tile / g.nib, ib = tile - ob * g.nib;
    const int64_t i0 = ob * g.bo, j0 = ib << g.lbi;
    lin0 = i0 * g.m_inner + j0;
    off0 = i0 * g.out_so + j0 * g.out_si;
    const int64_t ri = g.m_outer - i0, rj = g.m_inner - j0;
    ni = int(ri < g.bo ? ri : g.bo);
    nj = int(rj < (int64_t(1) << g.lbi) ? rj : (int64_t(1) << g.lbi));
  }
  __device__ __forceinline__ bool valid(int r) const { return (r >> lbi) < ni && (r & ((1 << lbi) - 1)) < nj; }
  __device__ __forceinline__ int64_t lin(const RowGrid& g, int r) const {
    // m_inner <= 2^31 (validated): one 32 x 32 -> 64-bit multiply-add (IMAD.WIDE.U32)
    return lin0 + int64_t(uint64_t(uint32_t(r >> lbi)) * uint32_t(g.m_inner)) + (r & ((1 << lbi) - 1));
  }
  __device__ __forceinline__ int64_t off(const RowGrid& g, int r) const {
    return off0 + int64_t(r >> lbi) * g.out_so + int64_t(r & ((1 << lbi) - 1)) * g.out_si;
  }
};

// ------------------------------------------------------------------ kernel
// Template parameters: N (row length), DT (dtype), TILE_ROWS (rows per pipeline
// stage), STAGES (ring depth), NT (compute warps), P (warps per row team, n > 256),
// U (work items per warp processed together, for ILP), CTAS (resident CTAs per SM).
// FLAT: input and output are contiguous m x n (g.flat_in set, out_so = n): the
// epilogue addresses rows as out + row * n with a 32-bit bound, as before the row
// grids existed (the general (i, j) addressing costs n = 128 6-9 %).
template <int N, int DT, int TILE_ROWS, int STAGES, int NT, int P, int U, int CTAS, int QT, bool FLAT>
__global__ void __launch_bounds__((NT + 1) * 32, CTAS)
    fwht_kernel(const __grid_constant__ CUtensorMap tm_in, uint16_t* __restrict__ out, uint8_t* __restrict__ out_q,
                float* __restrict__ row_scale, const RowGrid g, float s_res) {
  constexpr int ROW_BYTES = 2 * N;
  constexpr int TILE_BYTES = TILE_ROWS * ROW_BYTES;
  static_assert(TILE_BYTES % 16 == 0, "bulk copy granularity");
  extern __shared__ __align__(1024) uint8_t smem[];
  SchedCtl* ctl = reinterpret_cast<SchedCtl*>(smem + STAGES * TILE_BYTES);
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + STAGES * TILE_BYTES + sizeof(SchedCtl));
  uint64_t* empty = full + STAGES;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t num_tiles = g.num_tiles;
  static_assert(STAGES <= 16, "SchedCtl holds 16 stages");

  if (threadIdx.x == 0) {
    mbar_init(&ctl->clc_bar, 1);
#pragma unroll
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], NT);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    fence_proxy_async_smem();
  }
  __syncthreads();

  pdl_launch_dependents();
  if (warp == NT) {
    // ---------------- producer: TMA loads (3-D row-grid box) of row tiles into the ring
    if (lane == 0) {
      if (!FLAT && g.rows_in == nullptr) tma_prefetch(&tm_in);
      pdl_wait();  // the previous kernel on the stream has completed; all our global traffic follows this
      const uint64_t pol = policy_evict_first();
      uint32_t clc_phase = 0;
      int64_t tile = blockIdx.x;
      for (int it = 0;; ++it) {
        const int s = it % STAGES;
        const uint32_t ph = (it / STAGES) & 1;
        mbar_wait(&empty[s], ph ^ 1);
        if (tile < 0 || tile >= num_tiles) {  // no more tiles: tell the consumers
          ctl->stage_tile[s] = -1;
          mbar_arrive(&full[s]);
          break;
        }
        ctl->stage_tile[s] = int(tile);
        if constexpr (kClc) clc_request(ctl);  // ask for the next tile while this one loads
        const TileRows tr(g, tile);
        if (FLAT) {
          const int64_t rem = g.m_outer - tr.i0;
          const uint32_t bytes = uint32_t(rem < TILE_ROWS ? rem : TILE_ROWS) * ROW_BYTES;
          mbar_arrive_expect_tx(&full[s], bytes);
          bulk_g2s(smem + s * TILE_BYTES, g.flat_in + tr.i0 * N, bytes, &full[s], pol);
        } else if (g.rows_in != nullptr) {
          // rows outside the grid are not loaded: their (stale) slots are computed but never stored
          const int bi = 1 << g.lbi;
          const int64_t rj = g.m_inner - tr.j0, ri = g.m_outer - tr.i0;
          const int nj = int(rj < bi ? rj : bi), ni = int(ri < g.bo ? ri : g.bo);
          const uint32_t blk = uint32_t(nj) * ROW_BYTES;
          mbar_arrive_expect_tx(&full[s], blk * uint32_t(ni));
          for (int ob = 0; ob < ni; ++ob)
            bulk_g2s(smem + s * TILE_BYTES + ob * bi * ROW_BYTES, g.rows_in + (tr.i0 + ob) * g.in_so + tr.j0 * N, blk,
                     &full[s], pol);
        } else {
          mbar_arrive_expect_tx(&full[s], TILE_BYTES);  // full box; rows outside the grid are zero-filled
          tma_load_3d(smem + s * TILE_BYTES, &tm_in, 0, int(tr.j0), int(tr.i0), &full[s], pol);
        }
        if constexpr (kClc) {
          tile = clc_result(ctl, clc_phase);
        } else {
          tile += gridDim.x;
        }
      }
    }
    return;
  }

  // ---------------- consumers
  int it = 0;
  // fused quantization fast path, in the accumulator domain (y = d * s_res):
  // scale = max|d| |s_res| / Q, code multiplier = sign(s_res) Q / max|d|
  const float q_qs = copysignf(qmax_of<QT == QT_NONE ? QT_E4M3 : QT>(), s_res);
  const float q_ss = fabsf(s_res) / qmax_of<QT == QT_NONE ? QT_E4M3 : QT>();
  (void)q_qs;
  (void)q_ss;
  if constexpr (N == 128) {
    uint32_t A1[4], A2[4];
    make_const_a<DT>(0xFu, A1);  // H_16 over element bits {0,1,2,3}
    make_const_a<DT>(0x7u, A2);  // H_8 over bits {4,5,6} (x) I_2 (bit 1, same row)
    constexpr int FR = TILE_ROWS / 2;  // fragments (row pairs) per tile
    static_assert(FR % (NT * U) == 0, "n=128 work split");
    for (;; ++it) {
      const int s = it % STAGES;
      mbar_wait(&full[s], (it / STAGES) & 1);
      const int64_t tile = ctl->stage_tile[s];
      if (tile < 0) break;
      const TileRows tr(g, tile);
      const TileRowsFast trf(g, tile);
      (void)trf;
      const int64_t left = g.m_outer - tr.i0;
      const int rows_left = left < TILE_ROWS ? int(left) : TILE_ROWS;  // FLAT only
      const uint8_t* tb = smem + s * TILE_BYTES;
      const int lin_rows = trf.ni << trf.lbi;  // linear_rows: valid rows of the box
      // the epilogue's row addressing, specialised per tile on the box shape (LINR: linear rows)
      auto tile_body = [&](auto linr) {
      constexpr bool LINR = decltype(linr)::value;
      (void)LINR;
      for (int f0 = warp; f0 < FR; f0 += NT * U) {
        uint32_t x[U][4], y[U][4], z[U][4];
        (void)z;
        float d[U][8];
#pragma unroll
        for (int u = 0; u < U; ++u) {
          const uint8_t* ra = tb + (2 * (f0 + u * NT)) * ROW_BYTES + lane * 8;
          lds64(ra, x[u][0], x[u][2]);              // row A elements 4l..4l+3
          lds64(ra + ROW_BYTES, x[u][1], x[u][3]);  // row B
        }
#pragma unroll
        for (int u = 0; u < U; ++u) {
#ifdef HC_SIMT
          if constexpr (QT >= 0) {
            stage_ca<DT>(A1, x[u][0], x[u][2], x[u][1], x[u][3], y[u]);
            stage_ca_f32<DT>(A2, y[u][0], y[u][1], y[u][2], y[u][3], d[u]);
            continue;
          }
          simt_fwht_pack<DT>(x[u], 0x7Fu, ldexpf(s_res, -total_shift<N>()), z[u]);  // all bits but the row bit b7
          const uint32_t t1 = z[u][1];  // natural slots: row A in (z0, z2), row B in (z1, z3)
          z[u][1] = z[u][2];
          z[u][2] = t1;
#else
          stage_ca<DT>(A1, x[u][0], x[u][2], x[u][1], x[u][3], y[u]);
          stage_ca_f32<DT>(A2, y[u][0], y[u][1], y[u][2], y[u][3], d[u]);
          if constexpr (QT < 0) scale_pack<DT>(d[u], s_res, z[u]);
#endif
        }
#pragma unroll
        for (int u = 0; u < U; ++u) {
          const int f = f0 + u * NT;
          if constexpr (QT >= 0) {  // rows A (d[0..3] = elements 4l..4l+3) and B (d[4..7])
            float am[2];
#pragma unroll
            for (int h = 0; h < 2; ++h) {
              float a = 0.f;
#pragma unroll
              for (int e = 0; e < 4; ++e) a = absmax_nan(a, d[u][4 * h + e]);
              am[h] = warp_absmax(a);  // max |d| of the row; |y| = |d| |s_res|
            }
#pragma unroll
            for (int h = 0; h < 2; ++h) {
              const float* v = &d[u][4 * h];
              float sc;
              uint32_t code;
              if (quant_fast_range(am[h], 0x1p100f)) {
                sc = am[h] * q_ss;
                code = quant4_fast<QT>(v[0], v[1], v[2], v[3], q_qs * rcp_ftz(am[h]));
              } else {
                float inv;
                row_scale_of<QT>(am[h] * fabsf(s_res), sc, inv);
                const float mul = s_res * inv;
                code = quant4<QT>(v[0] * mul, v[1] * mul, v[2] * mul, v[3] * mul);
              }
              const bool ok = FLAT ? 2 * f + h < rows_left : (LINR ? 2 * f + h < lin_rows : trf.valid(2 * f + h));
              const int64_t row = FLAT ? tr.i0 + 2 * f + h
                                       : (LINR ? trf.lin0 + 2 * f + h : trf.lin(g, 2 * f + h));  // codes/scales: [rows, n]
              if constexpr (QT == QT_INT4) {
                stg16_if(out_q + row * (N / 2) + lane * 2, code, ok);
              } else {
                stg32_if(out_q + row * N + lane * 4, code, ok);
              }
              stf32_if(row_scale + row, sc, ok && lane == 0);
            }
          } else {
            if constexpr (FLAT) {
              uint16_t* o = out + (tr.i0 + 2 * f) * N + lane * 4;
              if (2 * f < rows_left) stg64(o, z[u][0], z[u][1]);
              if (2 * f + 1 < rows_left) stg64(o + N, z[u][2], z[u][3]);
            } else {
              if (LINR ? 2 * f < lin_rows : trf.valid(2 * f)) stg64(out + trf.off(g, 2 * f) + lane * 4, z[u][0], z[u][1]);
              if (LINR ? 2 * f + 1 < lin_rows : trf.valid(2 * f + 1))
                stg64(out + trf.off(g, 2 * f + 1) + lane * 4, z[u][2], z[u][3]);
            }
          }
        }
      }
      };
      if (QT >= 0 && !FLAT && trf.linear_rows(g)) {  // (the transform measured 3-5 % slower specialised)
        tile_body(std::true_type{});
      } else {
        tile_body(std::false_type{});
      }
      fence_proxy_async_smem();
      __syncwarp();
      if (lane == 0) mbar_arrive(&empty[s]);
    }
  } else if constexpr (N == 256) {
    uint32_t A1[4];
    make_const_a<DT>(0xFu, A1);
    static_assert(TILE_ROWS % (NT * U) == 0, "n=256 work split");
    for (;; ++it) {
      const int s = it % STAGES;
      mbar_wait(&full[s], (it / STAGES) & 1);
      const int64_t tile = ctl->stage_tile[s];
      if (tile < 0) break;
      const TileRows tr(g, tile);
      const TileRowsFast trf(g, tile);
      (void)trf;
      const int64_t left = g.m_outer - tr.i0;
      const int rows_left = left < TILE_ROWS ? int(left) : TILE_ROWS;  // FLAT only
      const uint8_t* tb = smem + s * TILE_BYTES;
      const int lin_rows = trf.ni << trf.lbi;  // linear_rows: valid rows of the box
      auto tile_body = [&](auto linr) {
      constexpr bool LINR = decltype(linr)::value;
      (void)LINR;
      for (int r0 = warp; r0 < TILE_ROWS; r0 += NT * U) {
        uint32_t x[U][4], y[U][4], z[U][4];
        (void)z;
        float d[U][8];
#pragma unroll
        for (int u = 0; u < U; ++u) lds128(tb + (r0 + u * NT) * ROW_BYTES + lane * 16, x[u][0], x[u][1], x[u][2], x[u][3]);
#pragma unroll
        for (int u = 0; u < U; ++u) {
#ifdef HC_SIMT
          if constexpr (QT < 0) {
            simt_fwht_pack<DT>(x[u], 0xFFu, ldexpf(s_res, -total_shift<N>()), z[u]);
            continue;
          }
#endif
          stage_ca<DT>(A1, x[u][0], x[u][2], x[u][1], x[u][3], y[u]);
          stage_ca_f32<DT>(A1, y[u][0], y[u][2], y[u][1], y[u][3], d[u]);
          if constexpr (QT < 0) scale_pack<DT>(d[u], s_res, z[u]);
        }
#pragma unroll
        for (int u = 0; u < U; ++u) {
          const int r = r0 + u * NT;
          if constexpr (QT >= 0) {  // d[0..7] = elements 8l..8l+7 of row r
            float a = 0.f;
#pragma unroll
            for (int e = 0; e < 8; ++e) a = absmax_nan(a, d[u][e]);
            const float am = warp_absmax(a);  // max |d| of the row; |y| = |d| |s_res|
            const float* v = d[u];
            float sc;
            uint32_t c0, c1;
            if (quant_fast_range(am, 0x1p100f)) {
              sc = am * q_ss;
              const float mul = q_qs * rcp_ftz(am);
              c0 = quant4_fast<QT>(v[0], v[1], v[2], v[3], mul);
              c1 = quant4_fast<QT>(v[4], v[5], v[6], v[7], mul);
            } else {
              float inv;
              row_scale_of<QT>(am * fabsf(s_res), sc, inv);
              const float mul = s_res * inv;
              c0 = quant4<QT>(v[0] * mul, v[1] * mul, v[2] * mul, v[3] * mul);
              c1 = quant4<QT>(v[4] * mul, v[5] * mul, v[6] * mul, v[7] * mul);
            }
            const bool ok = FLAT ? r < rows_left : (LINR ? r < lin_rows : trf.valid(r));
            const int64_t row = FLAT ? tr.i0 + r : (LINR ? trf.lin0 + r : trf.lin(g, r));
            if constexpr (QT == QT_INT4) {
              stg32_if(out_q + row * (N / 2) + lane * 4, __byte_perm(c0, c1, 0x5410), ok);
            } else {
              stg64_if(out_q + row * N + lane * 8, c0, c1, ok);
            }
            stf32_if(row_scale + row, sc, ok && lane == 0);
          } else {
            if constexpr (FLAT) {
              if (r < rows_left) stg128(out + (tr.i0 + r) * N + lane * 8, z[u][0], z[u][1], z[u][2], z[u][3]);
            } else {
              if (LINR ? r < lin_rows : trf.valid(r)) stg128(out + trf.off(g, r) + lane * 8, z[u][0], z[u][1], z[u][2], z[u][3]);
            }
          }
        }
      }
      };
      if (QT >= 0 && !FLAT && trf.linear_rows(g)) {  // (the transform measured 3-5 % slower specialised)
        tile_body(std::true_type{});
      } else {
        tile_body(std::false_type{});
      }
      fence_proxy_async_smem();
      __syncwarp();
      if (lane == 0) mbar_arrive(&empty[s]);
    }
  } else {
    static_assert(N <= 256, "rows longer than 256 use fwht_rows_kernel");
    (void)out_q;
    (void)row_scale;
  }
}

// Byte offset, inside a row's shared-memory image, of granule g (8 elements) of
// 256-chunk c.  The 4-D TMA box (64 el, C chunks, 4 segments, rows) with
// SWIZZLE_128B lays a row out as 128-byte lines L = s*C + c (s = g >> 3) and XORs
// the 16-byte granule index inside a line with L & 7 (tools/fragment_model.py gaddrT).
template <int C>
__device__ __forceinline__ uint32_t gofs(uint32_t c, uint32_t g) {
  const uint32_t L = (g >> 3) * C + c;
  return L * 128u + 16u * ((g & 7u) ^ (L & 7u));
}

// Build switches (tools/tune.py diagnostics): HC_STG_OUT = copy-out with LDS.128 +
// STG.128 by the consumers instead of TMA tensor stores; HC_SEG = per-segment boxes.
#ifdef HC_STG_OUT
constexpr bool kStgOut = true;
#else
constexpr bool kStgOut = false;
#endif
// SEG mode of fwht_rows_kernel (n >= 8192, tiles of <= 4 rows): every (row, 128-byte-
// line segment) of a tile is its own TMA box, stored as soon as its 8 phase-2 items
// are final and refilled as soon as that store has read it.  Shared with the host so
// the tensor-map box always matches what the kernel expects.
__host__ __device__ constexpr bool seg_mode(int n, int tile_rows) {
#ifdef HC_SEG  // opt-in: measured slower than whole-tile boxes (profiles/r01_tune_sweep11_paired.txt)
  return !kStgOut && tile_rows <= 4 && n >= 8192;
#else
  return false;
#endif
}

// Loads boxes K..NB-1 of a SEG tile (box k = row k/4, segment k%4); with WAIT, box k
// first waits until the store that read the same bytes (issued k-th of NB) is done.
template <int K, int NB, int ROW_BYTES, bool WAIT, typename TR>
__device__ __forceinline__ void seg_loads(uint8_t* stage, const void* tmap, const TR& tr, uint64_t* bar,
                                          uint64_t pol) {
  if constexpr (K < NB) {
    if constexpr (WAIT) bulk_wait_read<NB - 1 - K>();
    constexpr int r = K / 4;
    tma_load_5d(stage + r * ROW_BYTES + (K % 4) * (ROW_BYTES / 4), tmap, 0, 0, K % 4,
                int(tr.j0 + (r & ((1 << tr.lbi) - 1))), int(tr.i0 + (r >> tr.lbi)), bar, pol);
    seg_loads<K + 1, NB, ROW_BYTES, WAIT>(stage, tmap, tr, bar, pol);
  }
}

// ------------------------------------------------------------------ rows > 256
// Rows of n = 256 * 2^Q elements (P:120-129 [Sec. 3.2]).  The producer warp moves
// whole row tiles with 4-D TMA tensor copies in both directions; the hardware 128B
// swizzle is exactly the per-chunk XOR swizzle phase 2 needs, so there is no
// copy-out pass.  Consumers: phase 1 = H_256 per chunk in place (LDS/STS.128),
// team barrier, phase 2 = H_{n/256} across chunks via ldmatrix/stmatrix.trans,
// then signal the producer, which stores the tile and refills the stage.
template <int N, int DT, int TILE_ROWS, int STAGES, int NT, int P, int U, int CTAS, int QT>
__global__ void __launch_bounds__((NT + 1) * 32, CTAS)
    fwht_rows_kernel(const __grid_constant__ CUtensorMap tm_in, const __grid_constant__ CUtensorMap tm_out,
                     uint16_t* __restrict__ out, uint8_t* __restrict__ out_q, float* __restrict__ row_scale,
                     const RowGrid g, float s_res) {
  constexpr int ROW_BYTES = 2 * N;
  constexpr int TILE_BYTES = TILE_ROWS * ROW_BYTES;
  constexpr int Q = log2_n<N>() - 8;
  constexpr int C = N / 256;  // 256-chunks per row
  using PL = PlanL<Q>;
  constexpr int NLOOP = 1 << PL::nloop_bits;            // phase-2 items per row
  static_assert(NLOOP << PL::nx == C, "phase-2 fragment count");
  constexpr int NTEAMS = NT / P;
  static_assert(NT % P == 0 && TILE_ROWS % NTEAMS == 0, "team layout");
  constexpr int RPT = TILE_ROWS / NTEAMS;                // rows per team
  constexpr int ITEMS1 = RPT * C, ITEMS2 = RPT * NLOOP;  // phase-1 and phase-2 items per team
  constexpr int U1 = (ITEMS1 / P) >= U ? U : 1;
  constexpr int U2 = (ITEMS2 / P) >= U ? U : 1;
  static_assert(ITEMS1 % (P * U1) == 0 && ITEMS2 % (P * U2) == 0, "work split");

  // SEG: phase-2 items are the rows' 32 granule columns; each (row, segment) box is
  // stored (and refilled) as soon as its 8 items are done (seg_mode above).
  constexpr bool STG_OUT = kStgOut || QT >= 0;  // quantized output is written by the consumers
  constexpr bool SEG = QT < 0 && seg_mode(N, TILE_ROWS);
  constexpr int NSEG = SEG ? 4 * TILE_ROWS : 1;  // boxes (and done barriers) per tile
  constexpr int SEG_BYTES = ROW_BYTES / 4;

  extern __shared__ __align__(1024) uint8_t smem[];
  SchedCtl* ctl = reinterpret_cast<SchedCtl*>(smem + STAGES * TILE_BYTES);
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + STAGES * TILE_BYTES + sizeof(SchedCtl));
  uint64_t* done = full + STAGES;  // [STAGES][NSEG] consumers -> producer: ready to store
  float* red = reinterpret_cast<float*>(smem + STAGES * TILE_BYTES + sizeof(SchedCtl) + 17 * STAGES * 8);
  static_assert(STAGES <= 16, "SchedCtl holds 16 stages");
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t num_tiles = g.num_tiles;

  if (threadIdx.x == 0) {
    mbar_init(&ctl->clc_bar, 1);
#pragma unroll
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(&full[s], 1);
#pragma unroll
      for (int g = 0; g < NSEG; ++g) mbar_init(&done[s * NSEG + g], SEG ? NLOOP / 4 : NT);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    fence_proxy_async_smem();
  }
  __syncthreads();

  pdl_launch_dependents();
  if (warp == NT) {
    // ---------------- producer: TMA tensor loads and stores of whole row tiles
    if (lane == 0) {
      tma_prefetch(&tm_in);
      tma_prefetch(&tm_out);
      pdl_wait();  // the previous kernel on the stream has completed; all our global traffic follows this
#ifdef HC_TRACE
      g_span[blockIdx.x][0] = gtime();
#endif
      const uint64_t pol = policy_evict_first();
      auto load_tile = [&](int st, int64_t tile, auto wait_store_read) {
        mbar_arrive_expect_tx(&full[st], TILE_BYTES);  // full box, OOB rows zero-filled
        const TileRows tr(g, tile);
        if constexpr (SEG) {
          if constexpr (decltype(wait_store_read(0))::value) {
            seg_loads<0, NSEG, ROW_BYTES, true>(smem + st * TILE_BYTES, &tm_in, tr, &full[st], pol);
          } else {
            seg_loads<0, NSEG, ROW_BYTES, false>(smem + st * TILE_BYTES, &tm_in, tr, &full[st], pol);
          }
        } else {
          if constexpr (decltype(wait_store_read(0))::value) bulk_wait_read<0>();
          tma_load_5d(smem + st * TILE_BYTES, &tm_in, 0, 0, 0, int(tr.j0), int(tr.i0), &full[st], pol);
        }
      };
      // the tag says whether a refill must first wait for the previous occupant's
      // stores to have read the stage
      auto no_wait = [](int) { return std::false_type{}; };
      auto wait_reads = [](int) { return std::true_type{}; };
      uint32_t clc_phase = 0;
      int64_t tile = blockIdx.x;  // the next tile to load
      auto advance = [&](int64_t t) -> int64_t {
        if constexpr (kClc) {
          return clc_result(ctl, clc_phase);
        } else {
          return t + gridDim.x;
        }
      };
      bool ended = false;
      for (int k = 0; k < STAGES && !ended; ++k) {  // fill the ring
        if (tile < 0 || tile >= num_tiles) {
          ctl->stage_tile[k] = -1;
          mbar_arrive(&full[k]);
          ended = true;
          break;
        }
        ctl->stage_tile[k] = int(tile);
        if constexpr (kClc) clc_request(ctl);
        trace(k, 0);
        load_tile(k, tile, no_wait);
        tile = advance(tile);
      }
      for (int it = 0;; ++it) {
        const int s = it % STAGES;
        const uint32_t ph = (it / STAGES) & 1;
        const int64_t t = ctl->stage_tile[s];
        if (t < 0) break;
#pragma unroll
        for (int gs = 0; gs < NSEG; ++gs) {
          mbar_wait(&done[s * NSEG + gs], ph);
          if (gs == 0) trace(it, 1);
          if constexpr (STG_OUT) continue;
          const TileRows tr(g, t);
          if constexpr (SEG) {
            const int r = gs / 4;
            tma_store_5d(&tm_out, 0, 0, gs % 4, int(tr.j0 + (r & ((1 << tr.lbi) - 1))), int(tr.i0 + (r >> tr.lbi)),
                         smem + s * TILE_BYTES + r * ROW_BYTES + (gs % 4) * SEG_BYTES);
          } else {  // rows outside the grid are clipped by the TMA unit
            tma_store_5d(&tm_out, 0, 0, 0, int(tr.j0), int(tr.i0), smem + s * TILE_BYTES);
          }
          bulk_commit();
        }
        trace(it, 2);
        if (ended) continue;
        if (tile < 0 || tile >= num_tiles) {  // no more tiles: tell the consumers
          ctl->stage_tile[s] = -1;
          mbar_arrive(&full[s]);
          ended = true;
          continue;
        }
        ctl->stage_tile[s] = int(tile);
        if constexpr (kClc) clc_request(ctl);
        if constexpr (STG_OUT) {
          load_tile(s, tile, no_wait);
        } else {
          load_tile(s, tile, wait_reads);
        }
        trace(it + STAGES, 0);
        tile = advance(tile);
      }
      bulk_wait_all();
    }
    return;
  }

  // ---------------- consumers
  const int team = warp / P, wt = warp % P;
  uint32_t A256[4];
  make_const_a<DT>(0xFu, A256);
  uint32_t Pa[4], Pb[4], Bc0[2], Bc1[2];
  if constexpr (PL::two_stage && kJ0Mma) {
    make_const_a<DT>(0xFu, Pa);  // H_16 over (r0, r1, r2, j1)
    make_const_a<DT>(0x8u, Pb);  // H_2 over j0 (x) I_8
  } else {
    make_const_b<DT>(PL::mask_a, 0, Bc0);  // two-stage (n >= 8192): j0 then by fp32 butterflies
    make_const_b<DT>(PL::mask_a, 1, Bc1);
  }
  (void)Pa;
  (void)Pb;
  // phase-2 slot bits of this lane (ldmatrix row address provider: lane = 8*j + r)
  const uint32_t r0 = lane & 1, r1 = (lane >> 1) & 1, r2 = (lane >> 2) & 1, j0 = (lane >> 3) & 1,
                 j1 = (lane >> 4) & 1;
  uint32_t c_l = 0, g_l = 0;  // chunk / granule bits supplied by the lane
  if constexpr (Q == 1) { c_l = r0;                                g_l = j0 | (r1 << 1) | (r2 << 2) | (j1 << 3); }
  if constexpr (Q == 2) { c_l = r0 | (r1 << 1);                    g_l = j0 | (j1 << 1) | (r2 << 2); }
  if constexpr (Q == 3) { c_l = r0 | (r1 << 1) | (r2 << 2);        g_l = j0 | (j1 << 1); }
  if constexpr (Q == 4) { c_l = r0 | (r1 << 1) | (r2 << 2) | (j1 << 3); g_l = j0; }
  if constexpr (Q >= 5) { c_l = r0 | (r1 << 1) | (r2 << 2) | (j1 << 3) | (j0 << 4); g_l = 0; }
  constexpr int LOOP_SHIFT = 5 - PL::nloop_bits;  // loop index = top granule bits
  const uint32_t sm_base = smem_addr(smem);

  auto team_sync = [&]() {
    if constexpr (P == 1) {
      __syncwarp();
    } else {
      named_bar_sync(1 + team, P * 32);
    }
  };

  int it = 0;
  if constexpr (QT >= 0) {
    // ---------------- fused quantization (NEXT-1): the two factors in the other order.
    // H_n = H_{n/256} (x) H_256 and the factors commute (they act on different index
    // bits), so the cross-chunk factor runs first, on the raw rows (phase A, the
    // same ldmatrix/stmatrix exchange as phase 2 below, written back as a 16-bit
    // intermediate), and the per-chunk H_256 last (phase B): its fp32 results stay in
    // registers, in natural order (lane l holds elements 8l..8l+7 of its chunk), until
    // the team has the row maximum; the codes are then computed and stored straight
    // from registers (coalesced STG.64 / STG.32) -- no 16-bit image, no second pass over
    // shared memory, and the stage is released to the producer right after phase B.
    constexpr int IW = ITEMS1 / P;  // phase-B chunks per warp per tile
    // PK: keep the phase-B results as packed 16-bit y (RNE16(d * s_res), half the registers) so
    // that more CTAs fit per SM (HC_QPACK_N = the n that uses it); codes then come from y16
    constexpr bool PK = (N == HC_QPACK_N);
    static_assert(ITEMS1 % P == 0, "phase-B split");
    const float q_qs = copysignf(qmax_of<QT>(), s_res);  // code multiplier numerator (sign folded)
    const float q_ss = fabsf(s_res) / qmax_of<QT>();     // row scale per unit of max |d|
    for (;; ++it) {
      const int s = it % STAGES;
      mbar_wait(&full[s], (it / STAGES) & 1);
      const int64_t tile = ctl->stage_tile[s];
      if (tile < 0) break;
      uint8_t* const tb = smem + s * TILE_BYTES;

      // ---- phase A: H_{n/256} across chunks of the raw rows (residual factor P:146)
      for (int i0 = wt; i0 < ITEMS2; i0 += P * U2) {
        uint32_t x[U2][1 << PL::nx][4];
        uint32_t addr[U2][1 << PL::nx];
#pragma unroll
        for (int u = 0; u < U2; ++u) {
          const int item = i0 + u * P, r = team + NTEAMS * (item / NLOOP), lp = item % NLOOP;
          const uint32_t gg = g_l | (uint32_t(lp) << LOOP_SHIFT);
#pragma unroll
          for (int xi = 0; xi < (1 << PL::nx); ++xi) {
            addr[u][xi] = sm_base + s * TILE_BYTES + r * ROW_BYTES + gofs<C>(c_l | (uint32_t(xi) << 5), gg);
            ldsm_x4_t(addr[u][xi], x[u][xi]);
          }
        }
#pragma unroll
        for (int u = 0; u < U2; ++u) {
          float dd[1 << PL::nx][8];
#pragma unroll
          for (int xi = 0; xi < (1 << PL::nx); ++xi) {
            if constexpr (PL::two_stage && kJ0Mma) {
              uint32_t y[4];
              stage_ca<DT>(Pa, x[u][xi][0], x[u][xi][2], x[u][xi][1], x[u][xi][3], y);
              stage_ca_f32<DT>(Pb, y[0], y[2], y[1], y[3], dd[xi]);
            } else if constexpr (PL::two_stage) {
              stage_da_j0_f32<DT>(x[u][xi], Bc0, Bc1, dd[xi]);
            } else {
              stage_da_f32<DT>(x[u][xi], Bc0, Bc1, dd[xi]);
            }
          }
#pragma unroll
          for (int b = 0; b < PL::nx; ++b)
#pragma unroll
            for (int xi = 0; xi < (1 << PL::nx); ++xi)
              if (!((xi >> b) & 1)) bfly8(dd[xi], dd[xi | (1 << b)]);
#pragma unroll
          for (int xi = 0; xi < (1 << PL::nx); ++xi) {
            uint32_t z[4];
#pragma unroll
            for (int q = 0; q < 4; ++q) z[q] = pack2<DT>(dd[xi][2 * q], dd[xi][2 * q + 1]);  // exact 2^-k scaling is in the constants
            stsm_x4_t(addr[u][xi], z);
          }
        }
      }
      team_sync();  // P:126 "Sync across the threadblock"

      // ---- phase B: H_256 per chunk, results kept in registers
      float d[PK ? 1 : IW][8];
      uint32_t dp[PK ? IW : 1][4];
      float am[RPT];
#pragma unroll
      for (int k = 0; k < RPT; ++k) am[k] = 0.f;
#pragma unroll
      for (int k = 0; k < IW; ++k) {
        const int item = wt + k * P, rl = item / C, r = team + NTEAMS * rl, c = item % C;
        uint32_t x[4], y[4];
        float* dk = d[PK ? 0 : k];
        lds128(tb + r * ROW_BYTES + gofs<C>(uint32_t(c), uint32_t(lane)), x[0], x[1], x[2], x[3]);
        stage_ca<DT>(A256, x[0], x[2], x[1], x[3], y);
        stage_ca_f32<DT>(A256, y[0], y[2], y[1], y[3], dk);
        float a = 0.f;
#pragma unroll
        for (int e = 0; e < 8; ++e) a = absmax_nan(a, dk[e]);
        if constexpr (PK) scale_pack<DT>(dk, s_res, dp[k]);
#pragma unroll
        for (int kk = 0; kk < RPT; ++kk)
          if (kk == rl) am[kk] = absmax_nan(am[kk], a);
      }
      // the stage's shared memory is no longer read: release it to the producer now
      fence_proxy_async_smem();
      __syncwarp();
      if (lane == 0) mbar_arrive(&done[s]);

      // ---- row max over the team (max |d|; |y| = |d| |s_res|), then codes from registers
#pragma unroll
      for (int k = 0; k < RPT; ++k) {
        const float a = warp_absmax(am[k]);
        if (lane == 0) red[(team * RPT + k) * P + wt] = a;
      }
      team_sync();
      float mul_r[RPT];
      uint32_t fast_r = 0, ok_r = 0;
      uint8_t* q_r[RPT];
      const TileRows tr(g, tile);
#pragma unroll
      for (int k = 0; k < RPT; ++k) {
        float a = 0.f;
        for (int w = 0; w < P; ++w) a = absmax_nan(a, red[(team * RPT + k) * P + w]);
        float sc;
        if (quant_fast_range(a, 0x1p100f)) {
          sc = a * q_ss;
          mul_r[k] = PK ? qmax_of<QT>() * rcp_ftz(a * fabsf(s_res)) : q_qs * rcp_ftz(a);  // PK: per unit of y
          fast_r |= 1u << k;
        } else {
          float inv;
          row_scale_of<QT>(a * fabsf(s_res), sc, inv);
          mul_r[k] = PK ? inv : s_res * inv;
        }
        int64_t i = 0, j = 0;
        const bool ok = tr.at(g, team + NTEAMS * k, i, j);
        ok_r |= uint32_t(ok) << k;
        q_r[k] = out_q + (i * g.m_inner + j) * (QT == QT_INT4 ? N / 2 : N) + lane * (QT == QT_INT4 ? 4 : 8);
        stf32_if(row_scale + (i * g.m_inner + j), sc, ok && wt == 0 && lane == 0);
      }
#pragma unroll
      for (int k = 0; k < IW; ++k) {
        const int item = wt + k * P, rl = item / C, c = item % C;
        float mul = 0.f;
        uint8_t* qp = nullptr;
#pragma unroll
        for (int kk = 0; kk < RPT; ++kk)
          if (kk == rl) {
            mul = mul_r[kk];
            qp = q_r[kk];
          }
        float vv[8];
        if constexpr (PK) unpack8<DT>(dp[k], vv);  // y16 (an overflowed fp16 y is +-Inf: codes saturate to +-Q)
        const float* v = PK ? vv : d[PK ? 0 : k];
        uint32_t c0, c1;
        if ((fast_r >> rl) & 1u) {
          c0 = quant4_fast<QT>(v[0], v[1], v[2], v[3], mul);
          c1 = quant4_fast<QT>(v[4], v[5], v[6], v[7], mul);
        } else {
          c0 = quant4<QT>(v[0] * mul, v[1] * mul, v[2] * mul, v[3] * mul);
          c1 = quant4<QT>(v[4] * mul, v[5] * mul, v[6] * mul, v[7] * mul);
        }
        if constexpr (QT == QT_INT4) {
          stg32_if(qp + c * 128, __byte_perm(c0, c1, 0x5410), (ok_r >> rl) & 1u);
        } else {
          stg64_if(qp + c * 256, c0, c1, (ok_r >> rl) & 1u);
        }
      }
      // (red[] is rewritten only after the next tile's phase-A barrier: no race)
    }
  } else
  for (;; ++it) {
    const int s = it % STAGES;
    mbar_wait(&full[s], (it / STAGES) & 1);
    const int64_t tile = ctl->stage_tile[s];
    if (tile < 0) break;
    if (warp == 0 && lane == 0) trace(it, 4);
    uint8_t* const tb = smem + s * TILE_BYTES;

    // ---- phase 1: H_256 on every 256-chunk, in place
    for (int i0 = wt; i0 < ITEMS1; i0 += P * U1) {
      uint32_t x[U1][4], y[U1][4], z[U1][4];
      uint8_t* p[U1];
#pragma unroll
      for (int u = 0; u < U1; ++u) {
        const int item = i0 + u * P, r = team + NTEAMS * (item / C), c = item % C;
        p[u] = tb + r * ROW_BYTES + gofs<C>(uint32_t(c), uint32_t(lane));
        lds128(p[u], x[u][0], x[u][1], x[u][2], x[u][3]);
      }
#pragma unroll
      for (int u = 0; u < U1; ++u) {
#ifdef HC_SIMT
        simt_fwht_pack<DT>(x[u], 0xFFu, 0.0625f, z[u]);
#else
        stage_ca<DT>(A256, x[u][0], x[u][2], x[u][1], x[u][3], y[u]);
        stage_ca<DT>(A256, y[u][0], y[u][2], y[u][1], y[u][3], z[u]);
#endif
      }
#pragma unroll
      for (int u = 0; u < U1; ++u) stg_sh128(p[u], z[u]);
    }
    team_sync();  // P:126 "Sync across the threadblock"
    if (warp == 0 && lane == 0) trace(it, 5);

    // ---- phase 2: H_{n/256} across chunks (residual 2^a factor)
    for (int i0 = wt; i0 < ITEMS2; i0 += P * U2) {
      uint32_t x[U2][1 << PL::nx][4];
      uint32_t addr[U2][1 << PL::nx];
#pragma unroll
      for (int u = 0; u < U2; ++u) {
        const int item = i0 + u * P, r = team + NTEAMS * (item / NLOOP), lp = item % NLOOP;
        const uint32_t g = g_l | (uint32_t(lp) << LOOP_SHIFT);
#pragma unroll
        for (int xi = 0; xi < (1 << PL::nx); ++xi) {
          addr[u][xi] = sm_base + s * TILE_BYTES + r * ROW_BYTES + gofs<C>(c_l | (uint32_t(xi) << 5), g);
          ldsm_x4_t(addr[u][xi], x[u][xi]);
        }
      }
#pragma unroll
      for (int u = 0; u < U2; ++u) {
        float d[1 << PL::nx][8];
#pragma unroll
        for (int xi = 0; xi < (1 << PL::nx); ++xi) {
#ifdef HC_SIMT
          unpack8<DT>(x[u][xi], d[xi]);
          simt_butterflies(d[xi], PL::mask_a | (PL::two_stage ? 0x80u : 0u));
#pragma unroll
          for (int e = 0; e < 8; ++e) d[xi][e] *= ldexpf(1.f, -stage_shift(PL::mask_a));
#else
          if constexpr (PL::two_stage && kJ0Mma) {
            uint32_t y[4];
            stage_ca<DT>(Pa, x[u][xi][0], x[u][xi][2], x[u][xi][1], x[u][xi][3], y);
            stage_ca_f32<DT>(Pb, y[0], y[2], y[1], y[3], d[xi]);
          } else if constexpr (PL::two_stage) {
            stage_da_j0_f32<DT>(x[u][xi], Bc0, Bc1, d[xi]);
          } else {
            stage_da_f32<DT>(x[u][xi], Bc0, Bc1, d[xi]);
          }
#endif
        }
        // chunk bits 5, 6 live in per-lane fragments: fp32 butterflies (P:50-64 listing)
#pragma unroll
        for (int b = 0; b < PL::nx; ++b)
#pragma unroll
          for (int xi = 0; xi < (1 << PL::nx); ++xi)
            if (!((xi >> b) & 1)) bfly8(d[xi], d[xi | (1 << b)]);
#pragma unroll
        for (int xi = 0; xi < (1 << PL::nx); ++xi) {
          uint32_t z[4];
          scale_pack<DT>(d[xi], s_res, z);
          stsm_x4_t(addr[u][xi], z);
        }
        if constexpr (SEG) {  // this item's granule column is final: count it for its (row, segment)
          const int item = i0 + u * P, r = team + NTEAMS * (item / NLOOP), lp = item % NLOOP;
          fence_proxy_async_smem();
          __syncwarp();
          if (lane == 0) mbar_arrive(&done[s * NSEG + 4 * r + (lp >> 3)]);
        }
      }
    }
    if constexpr (STG_OUT) {
      team_sync();
      const TileRows tr(g, tile);
      for (int i0 = wt; i0 < ITEMS1; i0 += P * U1) {
        uint32_t z[U1][4];
#pragma unroll
        for (int u = 0; u < U1; ++u) {
          const int item = i0 + u * P, r = team + NTEAMS * (item / C), c = item % C;
          lds128(tb + r * ROW_BYTES + gofs<C>(uint32_t(c), uint32_t(lane)), z[u][0], z[u][1], z[u][2], z[u][3]);
        }
#pragma unroll
        for (int u = 0; u < U1; ++u) {
          const int item = i0 + u * P, r = team + NTEAMS * (item / C), c = item % C;
          int64_t i, j;
          if (tr.at(g, r, i, j))
            stg128(out + i * g.out_so + j * g.out_si + c * 256 + lane * 8, z[u][0], z[u][1], z[u][2], z[u][3]);
        }
      }
    }
    if constexpr (!SEG) {
      fence_proxy_async_smem();  // make this warp's smem writes visible to the TMA store
      __syncwarp();
      if (lane == 0) mbar_arrive(&done[s]);
    }
    if (warp == 0 && lane == 0) trace(it, 6);
  }
#ifdef HC_TRACE
  if (warp == 0 && lane == 0) {
    g_span[blockIdx.x][1] = gtime();
    g_span[blockIdx.x][2] = it;
  }
#endif
}

// ------------------------------------------------------------------ fp32 debug path
// HADACORE_F32 (north_star's "fp32 debug path", tolerance 1e-5): the P:50-64
// butterflies in fp32 on a shared-memory copy of ROWS rows, one __syncthreads per
// butterfly stage, scale applied once at the end (R3).  Correctness
// reference for the 16-bit paths on the GPU, not a performance path.
template <int N, int ROWS>
__global__ void __launch_bounds__(512) fwht_f32_kernel(const float* __restrict__ in, float* __restrict__ out,
                                                        int64_t m, float scale) {
  extern __shared__ __align__(16) float srow[];
  pdl_launch_dependents();
  pdl_wait();
  for (int64_t r0 = int64_t(blockIdx.x) * ROWS; r0 < m; r0 += int64_t(gridDim.x) * ROWS) {
    const int rows = (m - r0) < ROWS ? int(m - r0) : ROWS;
    const int cnt = rows * N;  // a multiple of 4 unless n < 4 (then copied by element)
    if (cnt % 4 == 0) {
      for (int i = threadIdx.x; i < cnt / 4; i += blockDim.x)
        reinterpret_cast<float4*>(srow)[i] = reinterpret_cast<const float4*>(in + r0 * N)[i];
    } else {
      for (int i = threadIdx.x; i < cnt; i += blockDim.x) srow[i] = in[r0 * N + i];
    }
    __syncthreads();
    for (int h = 1; h < N; h *= 2) {
      for (int idx = threadIdx.x; idx < rows * (N / 2); idx += blockDim.x) {
        const int r = idx / (N / 2), p = idx % (N / 2);
        const int j = r * N + (p / h) * (2 * h) + (p % h);
        const float a = srow[j], b = srow[j + h];
        srow[j] = a + b;
        srow[j + h] = a - b;
      }
      __syncthreads();
    }
    if (cnt % 4 == 0) {
      for (int i = threadIdx.x; i < cnt / 4; i += blockDim.x) {
        float4 v = reinterpret_cast<float4*>(srow)[i];
        v.x *= scale;
        v.y *= scale;
        v.z *= scale;
        v.w *= scale;
        reinterpret_cast<float4*>(out + r0 * N)[i] = v;
      }
    } else {
      for (int i = threadIdx.x; i < cnt; i += blockDim.x) out[r0 * N + i] = srow[i] * scale;
    }
    __syncthreads();
  }
}

}  // namespace hadacore
