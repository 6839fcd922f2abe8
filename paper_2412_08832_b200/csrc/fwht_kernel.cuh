// fwht_kernel.cuh -- sm_100a kernel for the batched normalized Walsh-Hadamard
// transform (HadaCore, arXiv 2412.08832).  "P:NN" = /root/reference/PAPER.md line.
//
// Design:
//  * Persistent CTAs; one producer warp streams row tiles HBM -> shared memory with
//    cp.async.bulk (TMA bulk copy, SASS UBLKCP) into a STAGES-deep mbarrier ring, so
//    tens of KB per SM are always in flight.  Every element is read once and written
//    once (P:264 in-place allowed: tiles are disjoint and read before written).
//  * The Kronecker factors H_16 (x) ... (P:150 [Sec. 3.4]) are contractions on the
//    tensor cores with register operands (mma.sync m16n8k16, SASS HMMA), as in the
//    paper's Sec. 3: a 256-element fragment lives in one warp, 8 elements per
//    lane.  Unlike the paper we never transpose with shuffles/movmatrix: putting the
//    CONSTANT in the A operand and the data in the B operand makes each stage return
//    D = K * X^T, i.e. the transpose comes free, and two such stages give
//    K_b * X * K_a in natural orientation (P:109's "transpose, H16, transpose back").
//  * Rows longer than 256 (P:120-129 [Sec. 3.2]): phase 1 applies H_256 to every
//    256-chunk, writes it back to shared memory with a per-chunk XOR swizzle of the
//    32-bit word index, phase 2 gathers fragments across chunks (bank-conflict free
//    because of the swizzle) and applies H_{n/256} (residual 2^a factors as
//    H_2^a (x) I blocks, P:146 [Sec. 3.3]), phase 3 un-swizzles and stores.
//  * Normalization: every stage multiplies by an exact power of two
//    (+-2^-floor(h/2) entries); the last stage accumulates in fp32 and multiplies by
//    s_res = scale * 2^E before the single round-to-nearest-even to 16 bits.
//  * bf16 (P:294 [App. C]): fp32 accumulate, cvt.rn.bf16x2 between stages.
//    fp16: fp16 accumulate between stages, fp32 in the last stage.
//
// The lane/register slot algebra is modelled and checked in tools/fragment_model.py.
#pragma once
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

__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n\t.reg .pred p;\n"
      "WAIT_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
      "@!p bra WAIT_%=;\n}" ::"r"(smem_addr(bar)),
      "r"(parity)
      : "memory");
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
__device__ __forceinline__ void stg32(uint16_t* p, uint32_t v) { *reinterpret_cast<uint32_t*>(p) = v; }
__device__ __forceinline__ void stg64(uint16_t* p, uint32_t a, uint32_t b) {
  *reinterpret_cast<uint2*>(p) = make_uint2(a, b);
}
__device__ __forceinline__ void stg128(uint16_t* p, uint32_t a, uint32_t b, uint32_t c, uint32_t d) {
  *reinterpret_cast<uint4*>(p) = make_uint4(a, b, c, d);
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

// A-operand (row-major 16x16) registers of 2^-shift * K(hmask) for this lane.
template <int DT>
__device__ __forceinline__ void make_const_a(uint32_t hmask, uint32_t a[4]) {
  const int lane = threadIdx.x & 31, g = lane >> 2, t = lane & 3;
  const float s = ldexpf(1.f, -stage_shift(hmask));
  a[0] = pack2<DT>(s * kron_entry(hmask, g, 2 * t), s * kron_entry(hmask, g, 2 * t + 1));
  a[1] = pack2<DT>(s * kron_entry(hmask, g + 8, 2 * t), s * kron_entry(hmask, g + 8, 2 * t + 1));
  a[2] = pack2<DT>(s * kron_entry(hmask, g, 2 * t + 8), s * kron_entry(hmask, g, 2 * t + 9));
  a[3] = pack2<DT>(s * kron_entry(hmask, g + 8, 2 * t + 8), s * kron_entry(hmask, g + 8, 2 * t + 9));
}

// B-operand (16x8, "col") registers of columns [8T, 8T+8) of 2^-shift * K(hmask).
template <int DT>
__device__ __forceinline__ void make_const_b(uint32_t hmask, int T, uint32_t b[2]) {
  const int lane = threadIdx.x & 31, g = lane >> 2, t = lane & 3;
  const float s = ldexpf(1.f, -stage_shift(hmask));
  const int n = 8 * T + g;
  b[0] = pack2<DT>(s * kron_entry(hmask, 2 * t, n), s * kron_entry(hmask, 2 * t + 1, n));
  b[1] = pack2<DT>(s * kron_entry(hmask, 2 * t + 8, n), s * kron_entry(hmask, 2 * t + 9, n));
}

// ------------------------------------------------------------------ stages
// "const-A" stage: tile T uses B = (x[rT0], x[rT1]); outputs
//   y0 = D_0 rows 0..7, y1 = D_0 rows 8..15, y2 = D_1 rows 0..7, y3 = D_1 rows 8..15.
template <int DT>
__device__ __forceinline__ void stage_ca(const uint32_t a[4], uint32_t b00, uint32_t b01, uint32_t b10,
                                         uint32_t b11, uint32_t y[4]) {
  mma_pk<DT>(a, b00, b01, y[0], y[1]);
  mma_pk<DT>(a, b10, b11, y[2], y[3]);
}
// Same, final stage: fp32 accumulate, * s_res, RNE pack.
template <int DT>
__device__ __forceinline__ void stage_ca_final(const uint32_t a[4], uint32_t b00, uint32_t b01,
                                               uint32_t b10, uint32_t b11, float s_res, uint32_t y[4]) {
  float d0[4], d1[4];
  mma_f32<DT>(a, b00, b01, d0);
  mma_f32<DT>(a, b10, b11, d1);
  y[0] = pack2<DT>(d0[0] * s_res, d0[1] * s_res);
  y[1] = pack2<DT>(d0[2] * s_res, d0[3] * s_res);
  y[2] = pack2<DT>(d1[0] * s_res, d1[1] * s_res);
  y[3] = pack2<DT>(d1[2] * s_res, d1[3] * s_res);
}
// "data-as-A" final stage: D = X * Bc (X in A layout, 4 regs); output layout == input.
template <int DT>
__device__ __forceinline__ void stage_da_final(const uint32_t x[4], const uint32_t bc0[2],
                                               const uint32_t bc1[2], float s_res, uint32_t y[4]) {
  float d0[4], d1[4];
  mma_f32<DT>(x, bc0[0], bc0[1], d0);  // output columns 0..7  -> A-layout regs R0 (rows g), R1 (g+8)
  mma_f32<DT>(x, bc1[0], bc1[1], d1);  // output columns 8..15 -> R2, R3
  y[0] = pack2<DT>(d0[0] * s_res, d0[1] * s_res);
  y[1] = pack2<DT>(d0[2] * s_res, d0[3] * s_res);
  y[2] = pack2<DT>(d1[0] * s_res, d1[1] * s_res);
  y[3] = pack2<DT>(d1[2] * s_res, d1[3] * s_res);
}

// ------------------------------------------------------------------ per-n plans
// Phase-2 slot ids: 0..4 = lane bits (t0, t1, g0, g1, g2), 5 = r1 (X1/X0), 6 = r2 (X2/X0).
// See tools/fragment_model.py::phase2_plan and DESIGN.md "Phase 2".
template <int Q>
struct Phase2Plan;
#define HC_PLAN(Q, SINGLE, MASK_A, MASK_B, NCH, C0, C1, C2, C3, C4, C5, C6, NW, W0, W1, W2, W3, W4, W5, NLC, \
                L0, L1, L2, L3, L4, A)                                                                       \
  template <>                                                                                                \
  struct Phase2Plan<Q> {                                                                                     \
    static constexpr bool single = SINGLE;                                                                   \
    static constexpr uint32_t mask_a = MASK_A, mask_b = MASK_B;                                              \
    static constexpr int nch = NCH, nw = NW, nlc = NLC, a = A;                                               \
    __host__ __device__ static constexpr int ch(int i) {                                                     \
      return i == 0 ? C0 : i == 1 ? C1 : i == 2 ? C2 : i == 3 ? C3 : i == 4 ? C4 : i == 5 ? C5 : C6;          \
    }                                                                                                        \
    __host__ __device__ static constexpr int w(int i) {                                                      \
      return i == 0 ? W0 : i == 1 ? W1 : i == 2 ? W2 : i == 3 ? W3 : i == 4 ? W4 : W5;                        \
    }                                                                                                        \
    __host__ __device__ static constexpr int lc(int i) {                                                     \
      return i == 0 ? L0 : i == 1 ? L1 : i == 2 ? L2 : i == 3 ? L3 : L4;                                      \
    }                                                                                                        \
  };
//     Q  single mask_a mask_b nch chunk slots            nw word slots           nlc lane-chunk slots  a
HC_PLAN(1, true, 0x8u, 0x0u, 1, 6, 0, 0, 0, 0, 0, 0, 6, 0, 1, 2, 3, 4, 5, 0, 0, 0, 0, 0, 0, 5)
HC_PLAN(2, true, 0xAu, 0x0u, 2, 6, 0, 0, 0, 0, 0, 0, 5, 1, 2, 3, 4, 5, 0, 1, 0, 0, 0, 0, 0, 4)
HC_PLAN(3, true, 0xEu, 0x0u, 3, 6, 0, 1, 0, 0, 0, 0, 4, 2, 3, 4, 5, 0, 0, 2, 0, 1, 0, 0, 0, 3)
HC_PLAN(4, false, 0x8u, 0xBu, 4, 5, 6, 2, 3, 0, 0, 0, 3, 0, 1, 4, 0, 0, 0, 2, 2, 3, 0, 0, 0, 3)
HC_PLAN(5, false, 0x8u, 0xFu, 5, 5, 6, 2, 3, 4, 0, 0, 2, 0, 1, 0, 0, 0, 0, 3, 2, 3, 4, 0, 0, 2)
HC_PLAN(6, false, 0xAu, 0xFu, 6, 5, 6, 2, 3, 4, 0, 0, 1, 1, 0, 0, 0, 0, 0, 4, 0, 2, 3, 4, 0, 1)
HC_PLAN(7, false, 0xEu, 0xFu, 7, 5, 6, 2, 3, 4, 0, 1, 0, 0, 0, 0, 0, 0, 0, 5, 0, 1, 2, 3, 4, 0)
#undef HC_PLAN

__device__ __forceinline__ int slot_bit(int slot, int lane, int j) {
  return slot < 5 ? (lane >> slot) & 1 : (j >> (slot - 5)) & 1;
}

// Per-chunk XOR swizzle of the 32-bit word index inside a 512-byte chunk: the chunk
// bits that sit in lanes during phase 2 go to bank bits [a, 5) (bank-conflict free).
template <int Q>
__device__ __forceinline__ uint32_t swz(uint32_t c) {
  using P = Phase2Plan<Q>;
  uint32_t f = 0;
#pragma unroll
  for (int r = 0; r < P::nlc; ++r) {
    int idx = 0;
#pragma unroll
    for (int i = 0; i < P::nch; ++i)
      if (P::ch(i) == P::lc(r)) idx = i;
    f |= ((c >> idx) & 1u) << (P::a + r);
  }
  return f;
}

// Total power-of-two exponent E applied by the per-stage constants for this n.
template <int N>
__host__ __device__ constexpr int total_shift() {
  if constexpr (N == 128) return stage_shift(0xFu) + stage_shift(0x7u);
  else if constexpr (N == 256) return 2 * stage_shift(0xFu);
  else {
    constexpr int q = (N == 512) ? 1 : (N == 1024) ? 2 : (N == 2048) ? 3 : (N == 4096) ? 4
                      : (N == 8192) ? 5 : (N == 16384) ? 6 : 7;
    return 2 * stage_shift(0xFu) + stage_shift(Phase2Plan<q>::mask_a) + stage_shift(Phase2Plan<q>::mask_b);
  }
}

template <int N>
__host__ __device__ constexpr int log2_n() {
  int k = 0;
  while ((1 << k) < N) ++k;
  return k;
}

// ------------------------------------------------------------------ kernel
// Template parameters: N (row length), DT (dtype), TILE_ROWS (rows per pipeline
// stage), STAGES (ring depth), NT (compute warps), P (warps per row team, n>256).
template <int N, int DT, int TILE_ROWS, int STAGES, int NT, int P>
__global__ void __launch_bounds__((NT + 1) * 32, 1)
    fwht_kernel(const uint16_t* __restrict__ in, uint16_t* __restrict__ out, int64_t m, float s_res) {
  constexpr int ROW_BYTES = 2 * N;
  constexpr int TILE_BYTES = TILE_ROWS * ROW_BYTES;
  static_assert(TILE_BYTES % 16 == 0, "bulk copy granularity");
  extern __shared__ __align__(1024) uint8_t smem[];
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + STAGES * TILE_BYTES);
  uint64_t* empty = full + STAGES;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t num_tiles = (m + TILE_ROWS - 1) / TILE_ROWS;

  if (threadIdx.x == 0) {
#pragma unroll
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], NT);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    fence_proxy_async_smem();
  }
  __syncthreads();

  if (warp == NT) {
    // ---------------- producer: TMA bulk loads of row tiles into the ring
    if (lane == 0) {
      const uint64_t pol = policy_evict_first();
      int it = 0;
      for (int64_t tile = blockIdx.x; tile < num_tiles; tile += gridDim.x, ++it) {
        const int s = it % STAGES;
        const uint32_t ph = (it / STAGES) & 1;
        mbar_wait(&empty[s], ph ^ 1);
        const int64_t row0 = tile * TILE_ROWS;
        const int64_t rem = m - row0;
        const int rows = rem < TILE_ROWS ? int(rem) : TILE_ROWS;
        const uint32_t bytes = uint32_t(rows) * ROW_BYTES;
        mbar_arrive_expect_tx(&full[s], bytes);
        bulk_g2s(smem + s * TILE_BYTES, in + row0 * N, bytes, &full[s], pol);
      }
    }
    return;
  }

  // ---------------- consumers
  
  int it = 0;
  if constexpr (N == 128) {
    uint32_t A1[4], A2[4];
    make_const_a<DT>(0xFu, A1);  // H_16 over element bits {0,1,2,3}
    make_const_a<DT>(0x7u, A2);  // H_8 over bits {4,5,6} (x) I_2 (bit 1, same row)
    constexpr int FR = TILE_ROWS / 2;  // fragments (row pairs) per tile
    for (int64_t tile = blockIdx.x; tile < num_tiles; tile += gridDim.x, ++it) {
      const int s = it % STAGES;
      mbar_wait(&full[s], (it / STAGES) & 1);
      const int64_t row0 = tile * TILE_ROWS;
      const int rows = (m - row0) < TILE_ROWS ? int(m - row0) : TILE_ROWS;
      uint8_t* const tb = smem + s * TILE_BYTES;
#pragma unroll 2
      for (int f = warp; f < FR; f += NT) {
        const uint8_t* ra = tb + (2 * f) * ROW_BYTES + lane * 8;
        const uint8_t* rb = ra + ROW_BYTES;
        uint32_t x[4], y[4], z[4];
        lds64(ra, x[0], x[2]);  // row A elements 4l..4l+3
        lds64(rb, x[1], x[3]);  // row B
        stage_ca<DT>(A1, x[0], x[2], x[1], x[3], y);
        stage_ca_final<DT>(A2, y[0], y[1], y[2], y[3], s_res, z);
        uint16_t* o = out + (row0 + 2 * f) * N + lane * 4;
        if (2 * f < rows) stg64(o, z[0], z[1]);
        if (2 * f + 1 < rows) stg64(o + N, z[2], z[3]);
      }
      fence_proxy_async_smem();
      __syncwarp();
      if (lane == 0) mbar_arrive(&empty[s]);
    }
  } else if constexpr (N == 256) {
    uint32_t A1[4];
    make_const_a<DT>(0xFu, A1);
    for (int64_t tile = blockIdx.x; tile < num_tiles; tile += gridDim.x, ++it) {
      const int s = it % STAGES;
      mbar_wait(&full[s], (it / STAGES) & 1);
      const int64_t row0 = tile * TILE_ROWS;
      const int rows = (m - row0) < TILE_ROWS ? int(m - row0) : TILE_ROWS;
      uint8_t* const tb = smem + s * TILE_BYTES;
#pragma unroll 2
      for (int r = warp; r < TILE_ROWS; r += NT) {
        uint32_t x[4], y[4], z[4];
        lds128(tb + r * ROW_BYTES + lane * 16, x[0], x[1], x[2], x[3]);
        stage_ca<DT>(A1, x[0], x[2], x[1], x[3], y);
        stage_ca_final<DT>(A1, y[0], y[2], y[1], y[3], s_res, z);
        if (r < rows) stg128(out + (row0 + r) * N + lane * 8, z[0], z[1], z[2], z[3]);
      }
      fence_proxy_async_smem();
      __syncwarp();
      if (lane == 0) mbar_arrive(&empty[s]);
    }
  } else {
    constexpr int Q = log2_n<N>() - 8;
    constexpr int C = N / 256;  // chunks per row
    using PL = Phase2Plan<Q>;
    constexpr int NFRAG = 1 << (7 - PL::nw);  // phase-2 fragments per row (== C)
    static_assert(NFRAG == C, "phase-2 fragment count");
    constexpr int NTEAMS = NT / P;
    static_assert(NT % P == 0 && TILE_ROWS % NTEAMS == 0, "team layout");
    constexpr int ROWS_PER_TEAM = TILE_ROWS / NTEAMS;
    const int team = warp / P, wt = warp % P;

    uint32_t A256[4];
    make_const_a<DT>(0xFu, A256);
    uint32_t Pa[4], Pb[4], Bc0[2], Bc1[2];
    if constexpr (PL::single) {
      make_const_b<DT>(PL::mask_a, 0, Bc0);
      make_const_b<DT>(PL::mask_a, 1, Bc1);
    } else {
      make_const_a<DT>(PL::mask_a, Pa);
      make_const_a<DT>(PL::mask_b, Pb);
    }
    // per-lane phase-2 word offsets (within a row, in 32-bit words) for the 4 regs
    uint32_t off2[4];
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      uint32_t c = 0, w = 0;
#pragma unroll
      for (int i = 0; i < PL::nch; ++i) c |= uint32_t(slot_bit(PL::ch(i), lane, j)) << i;
#pragma unroll
      for (int i = 0; i < PL::nw; ++i) w |= uint32_t(slot_bit(PL::w(i), lane, j)) << i;
      off2[j] = c * 128u + (w ^ swz<Q>(c));
    }

    auto team_sync = [&]() {
      if constexpr (P == 1) {
        __syncwarp();
      } else {
        named_bar_sync(1 + team, P * 32);
      }
    };

    for (int64_t tile = blockIdx.x; tile < num_tiles; tile += gridDim.x, ++it) {
      const int s = it % STAGES;
      mbar_wait(&full[s], (it / STAGES) & 1);
      const int64_t row0 = tile * TILE_ROWS;
      const int rows = (m - row0) < TILE_ROWS ? int(m - row0) : TILE_ROWS;
      uint8_t* const tb = smem + s * TILE_BYTES;

      // ---- phase 1: H_256 on every 256-chunk of the team's rows
#pragma unroll 2
      for (int item = wt; item < ROWS_PER_TEAM * C; item += P) {
        const int r = team + NTEAMS * (item / C), c = item % C;
        uint8_t* const cb = tb + r * ROW_BYTES + c * 512;
        uint32_t x[4], y[4], z[4];
#pragma unroll
        for (int j = 0; j < 4; ++j) x[j] = lds32(cb + 4 * (lane + 32 * j));
        stage_ca<DT>(A256, x[0], x[2], x[1], x[3], y);
        stage_ca<DT>(A256, y[0], y[2], y[1], y[3], z);
        const uint32_t f = swz<Q>(uint32_t(c));
#pragma unroll
        for (int j = 0; j < 4; ++j) sts32(cb + 4 * ((lane + 32 * j) ^ f), z[j]);
      }
      team_sync();  // P:126 "Sync across the threadblock"

      // ---- phase 2: H_{n/256} across chunks, residual 2^a block
#pragma unroll 2
      for (int item = wt; item < ROWS_PER_TEAM * NFRAG; item += P) {
        const int r = team + NTEAMS * (item / NFRAG), fr = item % NFRAG;
        uint8_t* const rb = tb + r * ROW_BYTES;
        const uint32_t fx = uint32_t(fr) << PL::nw;
        uint32_t x[4], y[4], z[4];
#pragma unroll
        for (int j = 0; j < 4; ++j) x[j] = lds32(rb + 4 * (off2[j] ^ fx));
        if constexpr (PL::single) {
          stage_da_final<DT>(x, Bc0, Bc1, s_res, z);
        } else {
          stage_ca<DT>(Pa, x[0], x[2], x[1], x[3], y);
          stage_ca_final<DT>(Pb, y[0], y[2], y[1], y[3], s_res, z);
        }
#pragma unroll
        for (int j = 0; j < 4; ++j) sts32(rb + 4 * (off2[j] ^ fx), z[j]);
      }
      team_sync();

      // ---- phase 3: un-swizzle and store (coalesced 128 B per warp instruction)
#pragma unroll 2
      for (int item = wt; item < ROWS_PER_TEAM * C; item += P) {
        const int r = team + NTEAMS * (item / C), c = item % C;
        uint8_t* const cb = tb + r * ROW_BYTES + c * 512;
        const uint32_t f = swz<Q>(uint32_t(c));
        uint32_t z[4];
#pragma unroll
        for (int j = 0; j < 4; ++j) z[j] = lds32(cb + 4 * ((lane + 32 * j) ^ f));
        if (r < rows) {
          uint16_t* o = out + (row0 + r) * N + c * 256;
#pragma unroll
          for (int j = 0; j < 4; ++j) stg32(o + 2 * (lane + 32 * j), z[j]);
        }
      }
      fence_proxy_async_smem();
      __syncwarp();
      if (lane == 0) mbar_arrive(&empty[s]);
    }
  }
}

}  // namespace hadacore
