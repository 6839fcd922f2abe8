// Fused FWHT + per-row quantization on the 5th-generation tensor cores (tcgen05 + TMEM)
// for rows of n = 4096 .. 32768 (NEXT-1, round 2; DESIGN.md §5 "Fused quantization,
// tcgen05").  Included by hadacore.cu after fwht_kernel.cuh (whose PTX helpers, phase-2
// plans and quantization epilogues it reuses).
//
// The contract is hadacore_fwht_quant's (include/hadacore.h): y = scale * H_n * x per row
// (P:41), then per-row symmetric codes with s = max|y| / Q (R21, R22).
// H_n = H_{n/256} (x) H_256 and the two factors act on different index bits, so they
// commute (P:150 [Sec. 3.4]):
//
//   phase A (cross-chunk factor H_{n/256}, residual factor P:146): the
//     ldmatrix/stmatrix exchange of fwht_rows_kernel on the raw rows, legacy mma.sync,
//     written back in place as a 16-bit intermediate -- NA dedicated warps;
//   phase B (per-chunk factor H_256): tcgen05.mma from shared memory into
//     tensor memory.  A = the tile's 128 chunks as rows of 128 elements (the lower / upper
//     halves of every 256-chunk; K-major, 128-byte swizzled -- the layout the TMA load
//     already produced), B = H_128 (+-1, K-major, built once per CTA), D = fp32 in TMEM:
//     P = H_128 x_lo and R = H_128 x_hi per chunk (8 K-steps each, 16 MMAs per tile); in
//     Sylvester order H_256 = [[H_128, H_128], [H_128, -H_128]], so the last H_2 is
//     the epilogue's packed butterfly y_lo = P + R, y_hi = P - R -- one elected thread
//     issues the MMAs;
//   epilogue (NE warps): TMEM -> registers twice -- once for the row maximum of |y|
//     (FADD2/FSUB2 butterflies, FMNMX3), once for the codes (FFMA2 + cvt, the quant4_fast epilogues of
//     fwht_kernel.cuh).  The codes are staged, 128-byte swizzled, in the epilogue group's own
//     code buffer and one elected thread of the group writes them with one TMA tensor store
//     per tile (a thread's 32 contiguous codes sit 256 B from its neighbours': direct 16-byte
//     stores touched 32 lines per instruction and cost 35 %); HC_QTC_CB=0 stages them in the
//     tile's own (consumed) stage instead, stored by the producer before it refills it.
//
// Nothing is held in registers across the row-maximum barrier (the fp32 results live in
// tensor memory: 2 x 256 columns, two tiles in flight), so the phase-A warps, the MMA
// and the epilogue warps work on different tiles at the same time.
//
// Tile = 128 chunks (64 KiB of 16-bit input) = R = 128 / C rows of C = n / 256 chunks,
// a bo x bi rectangle of a row grid (contiguous m x n is bi = 1).
// It arrives as two TMA boxes (64 elements, C chunks, bi, bo, 2 segments): segment-major,
// so the 128 chunk lines of one 64-element segment are consecutive 128-byte lines -- an MMA
// operand with rows m = r * C + c at 128-byte pitch, 8-row groups 1024 B apart (SBO), and
// the SWIZZLE_128B granule XOR (line & 7) that both the TMA unit and the tensor core apply.
// Shared memory: 2 stages x 64 KiB, refilled as soon as the MMAs have read them, + EG code
// buffers (32 / 16 KiB) + H_128 32 KiB.  (HC_QTC_CB=0: 3 stages; the upper half of a stage is
// refilled once the MMAs have read it, the lower half first receives the tile's codes.)
#pragma once

namespace hadacore {

// ------------------------------------------------------------------ tcgen05 helpers
// Shared-memory matrix descriptor (sm_100 UMMA): K-major, SWIZZLE_128B, 8-row groups
// 1024 B apart; start address in 16-byte units.  K steps of 16 elements inside a
// 64-element swizzle atom advance the start address by 32 B.
__device__ __forceinline__ uint64_t umma_desc_sw128(uint32_t saddr) {
  return uint64_t((saddr >> 4) & 0x3FFFu) | (uint64_t(1) << 16) | (uint64_t(1024 >> 4) << 32) |
         (uint64_t(1) << 46) | (uint64_t(2) << 61);
}
// Instruction descriptor of kind::f16: fp32 accumulate, A/B fp16 or bf16, both K-major.
template <int DT>
__host__ __device__ constexpr uint32_t umma_idesc(int M, int N) {
  return (1u << 4) | (uint32_t(DT == DT_BF16) << 7) | (uint32_t(DT == DT_BF16) << 10) |
         (uint32_t(N >> 3) << 17) | (uint32_t(M >> 4) << 24);
}
__device__ __forceinline__ void umma_f16(uint32_t tmem_d, uint64_t a, uint64_t b, uint32_t idesc, uint32_t acc) {
  asm volatile(
      "{.reg .pred p;\n setp.ne.b32 p, %4, 0;\n"
      " tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;}" ::"r"(tmem_d),
      "l"(a), "l"(b), "r"(idesc), "r"(acc)
      : "memory");
}
// arrives on `bar` when every tcgen05.mma this thread issued so far has completed
__device__ __forceinline__ void umma_commit(uint64_t* bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_addr(bar))
               : "memory");
}
__device__ __forceinline__ void tc_fence_before() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void tc_fence_after() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void tmem_wait_ld() { asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory"); }
// 32 lanes x 32 columns of fp32: thread t gets lane (base lane + t), columns col..col+31
__device__ __forceinline__ void tmem_ld32(uint32_t taddr, float (&v)[32]) {
  uint32_t* u = reinterpret_cast<uint32_t*>(v);
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
      "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
      : "=r"(u[0]), "=r"(u[1]), "=r"(u[2]), "=r"(u[3]), "=r"(u[4]), "=r"(u[5]), "=r"(u[6]), "=r"(u[7]),
        "=r"(u[8]), "=r"(u[9]), "=r"(u[10]), "=r"(u[11]), "=r"(u[12]), "=r"(u[13]), "=r"(u[14]), "=r"(u[15]),
        "=r"(u[16]), "=r"(u[17]), "=r"(u[18]), "=r"(u[19]), "=r"(u[20]), "=r"(u[21]), "=r"(u[22]), "=r"(u[23]),
        "=r"(u[24]), "=r"(u[25]), "=r"(u[26]), "=r"(u[27]), "=r"(u[28]), "=r"(u[29]), "=r"(u[30]), "=r"(u[31])
      : "r"(taddr)
      : "memory");
}
// running max of |a|, |b| (NaN-propagating, one FMNMX3)
__device__ __forceinline__ float absmax3(float acc, float a, float b) {
  float r;
  asm("max.NaN.f32 %0, %1, %2, %3;" : "=f"(r) : "f"(acc), "f"(fabsf(a)), "f"(fabsf(b)));
  return r;
}
__device__ __forceinline__ void stg128_cs(void* p, uint32_t a, uint32_t b, uint32_t c, uint32_t d) {
  asm volatile("st.global.cs.v4.b32 [%0], {%1, %2, %3, %4};" ::"l"(p), "r"(a), "r"(b), "r"(c), "r"(d) : "memory");
}

// Byte offset of granule g (8 elements) of chunk c of tile row r in the segment-major
// 128-byte-swizzled tile image: line L = segment * 128 + r * C + c.
template <int C>
__device__ __forceinline__ uint32_t goff_tc(uint32_t r, uint32_t c, uint32_t g) {
  const uint32_t L = (g >> 3) * 128u + r * uint32_t(C) + c;
  return L * 128u + 16u * ((g & 7u) ^ (L & 7u));
}

// HC_TC_DIAG (diagnostic builds, wrong output): bit 0 skips phase A's arithmetic, bit 1 the
// epilogue's, bit 2 the MMAs, bit 3 the code stores, bit 4 the epilogue's second pass (the
// pipeline and its barriers still run)
#ifndef HC_TC_DIAG
#define HC_TC_DIAG 0
#endif
// HC_TC_NEGB: the MMAs produce y directly (32 per tile; the negate-B bit for y_hi) instead of
// H_128 x_lo, H_128 x_hi (16 per tile) + the epilogue's butterfly -- twice the operand reads
#ifdef HC_TC_NEGB
constexpr bool kTcNegB = true;
#else
constexpr bool kTcNegB = false;
#endif
#ifndef HC_QTC_UA
#define HC_QTC_UA 2
#endif
// HC_QTC_CB = 1: each epilogue group stages its tile's codes in a buffer of its own and
// stores them itself, so a stage is free for the next tile as soon as the MMAs have read
// it (2 stages); 0: codes staged in the stage's lower half, stored by the producer before
// it refills that half (3 stages)
#ifndef HC_QTC_CB
#define HC_QTC_CB 1
#endif
constexpr bool kTcCodeBuf = HC_QTC_CB != 0;
// HC_QTC_SPLIT = 1 (with HC_QTC_CB): the two half-tile boxes complete on their own mbarriers
// (lower half first) and phase A takes the items of the lower half first, so it starts
// while the upper half is still in flight
#ifndef HC_QTC_SPLIT
#define HC_QTC_SPLIT 0  // measured slower: E4M3 -4 %, INT4 -5..-13 % (profiles/r02_quant_tc_cb_ab.txt)
#endif
constexpr bool kTcSplit = kTcCodeBuf && HC_QTC_SPLIT != 0;
constexpr int kTcTile = 65536;   // 128 chunks of 256 16-bit elements
constexpr int kTcHBytes = 32768; // H_128, 16-bit, K-major SW128 (two 64-column atoms)
// HC_QTC_H64 (INT4 with code buffers): B = H_64 only (8 KiB) and N = 64 MMAs, H_128 = H_2 (x) H_64
// being [[H_64, H_64], [H_64, -H_64]]: output columns 0..63 of a half-chunk accumulate the two
// K-halves against H_64, columns 64..127 the second K-half with the negate-B bit.  Twice the
// A-operand reads, but 24 KiB of shared memory freed: 3 stages + one code buffer shared by the
// two epilogue groups (each waits for the other's store to have read it).
#ifndef HC_QTC_H64
#define HC_QTC_H64 0  // measured 7-9 % slower for INT4 (profiles/r02_quant_tc_small_c_ab.txt): off
#endif
template <int QT>
__host__ __device__ constexpr bool tc_h64() {
  return HC_QTC_H64 != 0 && kTcCodeBuf && QT == QT_INT4;
}
template <int QT>
__host__ __device__ constexpr int tc_hbytes() {
  return tc_h64<QT>() ? 8192 : kTcHBytes;
}
template <int QT, int EG>
__host__ __device__ constexpr int tc_ncb() {  // code buffers
  return kTcCodeBuf ? (tc_h64<QT>() ? 1 : EG) : 0;
}
constexpr int kTcCols = 512;     // TMEM columns: two tiles x (y_lo 128 + y_hi 128)

template <int QT>
__host__ __device__ constexpr int tc_code_bytes() {  // a tile's codes
  return QT == QT_INT4 ? kTcTile / 4 : kTcTile / 2;
}
template <int STAGES, int NE, int QT, int EG>
__host__ __device__ constexpr int tc_smem_bytes() {
  return STAGES * kTcTile + tc_ncb<QT, EG>() * tc_code_bytes<QT>() + tc_hbytes<QT>() + int(sizeof(SchedCtl)) +
         (5 * STAGES + 5) * 8 + 32 + 2 * NE * 2 * 4;
}

// Template parameters: N row length (4096..32768), DT dtype, QT code type, STAGES ring
// depth (64 KiB stages), NA phase-A warps, NE epilogue warps (4 or 8).  Warps [0, NE)
// are the epilogue (warp % 4 = its TMEM lane quadrant), [NE, NE + NA) phase A, then the
// TMA producer warp and the MMA warp.
template <int N, int DT, int QT, int STAGES, int NA, int NE, int EG>
__global__ void __launch_bounds__((EG * NE + NA + 2) * 32, 1)
    fwht_quant_tc_kernel(const __grid_constant__ CUtensorMap tm_in, const __grid_constant__ CUtensorMap tm_q,
                         float* __restrict__ row_scale, const RowGrid g, float s_res) {
  constexpr int C = N / 256, R = 128 / C, Q = log2_n<N>() - 8;
  static_assert(C >= 2 && C <= 128, "n = 512 .. 32768");
  static_assert(C >= 16 || NE == 4, "rows of < 16 chunks: a thread holds its whole chunk (row max in-warp)");
  static_assert(NE == 4 || NE == 8, "epilogue warps");
  using PL = PlanL<Q>;
  constexpr int NLOOP = 1 << PL::nloop_bits;
  constexpr int ITEMS = R * NLOOP;  // phase-A items per tile
  constexpr int UA = (HC_QTC_UA >> PL::nx) > 0 ? (HC_QTC_UA >> PL::nx) : 1;  // phase-A items in flight per warp
  constexpr uint32_t IDESC = umma_idesc<DT>(128, 128);
  constexpr uint32_t IDESC_NEG = IDESC | (1u << 14);  // B negated: the -H_128 blocks of H_256
  constexpr bool H64 = tc_h64<QT>();
  constexpr int NCB = tc_ncb<QT, EG>();
  constexpr uint32_t IDESC64 = umma_idesc<DT>(128, 64);
  constexpr uint32_t IDESC64_NEG = IDESC64 | (1u << 14);
  const int64_t num_tiles = g.num_tiles;

  extern __shared__ __align__(1024) uint8_t smem[];
  uint8_t* const codebuf = smem + STAGES * kTcTile;  // kTcCodeBuf: NCB code buffers (1024-aligned)
  uint8_t* const Hs = codebuf + NCB * tc_code_bytes<QT>();
  SchedCtl* ctl = reinterpret_cast<SchedCtl*>(Hs + tc_hbytes<QT>());
  uint64_t* full = reinterpret_cast<uint64_t*>(ctl + 1);  // TMA -> phase A
  uint64_t* adone = full + STAGES;                         // phase A -> MMA (NA arrivals)
  uint64_t* cready = adone + STAGES;                       // epilogue -> producer: codes staged (NE)
  uint64_t* ufree = cready + STAGES;                       // MMA commit -> producer: stage read
  uint64_t* tfull = ufree + STAGES;                        // [2] MMA -> epilogue (commit + arrive)
  uint64_t* tempty = tfull + 2;                            // [2] epilogue -> MMA (NE arrivals)
  uint64_t* full_hi = tempty + 2;                          // kTcSplit: TMA -> phase A, upper half
  uint64_t* cbuf_free = full_hi + STAGES;                  // NCB == 1: the shared code buffer was read
  int* buf_tile = reinterpret_cast<int*>(cbuf_free + 1);   // [2] tile id of each TMEM buffer
  int* buf_stage = buf_tile + 2;                           // [2] ... and the stage it came from
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(buf_stage + 2);
  float* red = reinterpret_cast<float*>(tmem_slot + 2);    // [2][NE * 2] row-max partials

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int WP = EG * NE + NA, WM = EG * NE + NA + 1;  // producer and MMA warps

  if (threadIdx.x == 0) {
    mbar_init(&ctl->clc_bar, 1);
#pragma unroll
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&adone[s], NA);
      mbar_init(&cready[s], NE);
      mbar_init(&ufree[s], 1);
      mbar_init(&full_hi[s], 1);
    }
#pragma unroll
    for (int b = 0; b < 2; ++b) {
      mbar_init(&tfull[b], 2);
      mbar_init(&tempty[b], NE);
    }
    mbar_init(cbuf_free, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  // B operand: H_128 (unnormalized +-1, Sylvester order), row n (output element),
  // column k (input element), K-major SW128: atom k >> 6, line n, granule (k & 63) >> 3
  // (H64: H_64 only, one atom of 64 lines)
  for (int i = threadIdx.x; i < (H64 ? 64 * 8 : 128 * 16); i += blockDim.x) {
    const int nrow = H64 ? (i >> 3) : (i >> 4), g = H64 ? (i & 7) : (i & 15);
    uint32_t w[4];
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const int k0 = 8 * g + 2 * q;
      const float a = (__popc(nrow & k0) & 1) ? -1.f : 1.f, b = (__popc(nrow & (k0 + 1)) & 1) ? -1.f : 1.f;
#ifdef HC_NEGCTL
      w[q] = pack2<DT>((nrow == 3 && k0 == 4) ? -a : a, b);  // negative control: one sign flipped
#else
      w[q] = pack2<DT>(a, b);
#endif
    }
    const int atom = g >> 3, gs = g & 7;
    *reinterpret_cast<uint4*>(Hs + atom * 16384 + nrow * 128 + ((gs ^ (nrow & 7)) << 4)) =
        make_uint4(w[0], w[1], w[2], w[3]);
  }
  fence_proxy_async_smem();  // the tensor core reads Hs through the async proxy
  if (warp == WM) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_addr(tmem_slot)),
                 "n"(kTcCols)
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  pdl_launch_dependents();

  if (warp == WP) {
    // ---------------- producer.  A tile arrives as two 32 KiB TMA boxes (segments 0-1 = the
    // lower half of the stage, segments 2-3 = the upper half; rows outside the grid zero-
    // filled).  Once the MMAs have read a stage, the next tile's upper half is loaded into it
    // at once; the lower half receives the finished tile's codes (epilogue), which one TMA
    // tensor store writes out (rows outside the grid clipped) before the next tile's lower
    // half is loaded there.
    if (lane == 0) {
      tma_prefetch(&tm_in);
      tma_prefetch(&tm_q);
      pdl_wait();
      const uint64_t pol = policy_evict_first();
      uint32_t clc_phase = 0;
      int64_t tile = blockIdx.x;
      auto next_tile = [&](int64_t t) {
        if constexpr (kClc) {
          tile = clc_result(ctl, clc_phase);
        } else {
          tile = t + gridDim.x;
        }
      };
      auto load_half = [&](int st, int64_t t, int half, uint64_t* bar = nullptr) {
        const TileRows tr(g, t);
        tma_load_5d(smem + st * kTcTile + half * (kTcTile / 2), &tm_in, 0, 0, int(tr.j0), int(tr.i0), 2 * half,
                    bar ? bar : &full[st], pol);
      };
      bool ended = false;
      for (int k = 0; k < STAGES; ++k) {  // fill the ring
        if (ended || tile < 0 || tile >= num_tiles) {
          ctl->stage_tile[k] = -1;
          mbar_arrive(&full[k]);
          ended = true;
          break;
        }
        const int64_t t = tile;
        ctl->stage_tile[k] = int(t);
        if constexpr (kClc) clc_request(ctl);
        trace(k, 0);
        if constexpr (kTcSplit) {
          mbar_arrive_expect_tx(&full[k], kTcTile / 2);
          load_half(k, t, 0);
          mbar_arrive_expect_tx(&full_hi[k], kTcTile / 2);
          load_half(k, t, 1, &full_hi[k]);
        } else {
          mbar_arrive_expect_tx(&full[k], kTcTile);
          load_half(k, t, 1);
          load_half(k, t, 0);
        }
        next_tile(t);
      }
      for (int it = 0;; ++it) {
        const int s = it % STAGES;
        const uint32_t ph = (it / STAGES) & 1;
        const int t = ctl->stage_tile[s];
        if (t < 0) break;
        mbar_wait(&ufree[s], ph);  // the MMAs have read the stage: its upper half is free
        jitter(10, it);
        int64_t nt = -1;
        if (!ended) {
          if (tile < 0 || tile >= num_tiles) {
            ctl->stage_tile[s] = -1;  // no more tiles: the consumers stop at this stage
            mbar_arrive(&full[s]);
            ended = true;
          } else {
            nt = tile;
            ctl->stage_tile[s] = int(nt);
            if constexpr (kClc) clc_request(ctl);
            trace(it + STAGES, 0);
            if constexpr (kTcSplit) {  // the codes live elsewhere: the whole stage is free
              mbar_arrive_expect_tx(&full[s], kTcTile / 2);
              load_half(s, nt, 0);
              mbar_arrive_expect_tx(&full_hi[s], kTcTile / 2);
              load_half(s, nt, 1, &full_hi[s]);
            } else {
              mbar_arrive_expect_tx(&full[s], kTcTile);
              load_half(s, nt, 1);
              if constexpr (kTcCodeBuf) load_half(s, nt, 0);  // the codes live elsewhere: the whole stage is free
            }
            next_tile(nt);
          }
        }
        if constexpr (kTcCodeBuf) continue;
        mbar_wait(&cready[s], ph);  // the codes of tile t are staged in the lower half
        jitter(11, it);
        const TileRows tr(g, t);
        tma_store_4d(&tm_q, 0, 0, int(tr.j0), int(tr.i0), smem + s * kTcTile);
        bulk_commit();
        if (nt >= 0) {
          bulk_wait_read<0>();  // the store has read the lower half
          load_half(s, nt, 0);
        }
      }
      bulk_wait_all();
    }
  } else if (warp == WM) {
    // ---------------- MMA issuer: phase B of a tile = 2 halves x 8 K-steps of 128x128x16
    if (lane == 0) {
      const uint32_t sm0 = smem_addr(smem), hs0 = smem_addr(Hs);
      for (int it = 0;; ++it) {
        const int s = it % STAGES, b = it & 1;
        mbar_wait(&adone[s], (it / STAGES) & 1);
        trace(it, 7);
        const int tile = ctl->stage_tile[s];
        mbar_wait(&tempty[b], ((it >> 1) & 1) ^ 1);  // the epilogue has drained buffer b
        jitter(12, it);
        trace(it, 3);
        if (tile < 0) {  // end: every epilogue group sees a -1 tile (group e drains iteration it + e)
#pragma unroll
          for (int e = 0; e < EG; ++e) {
            const int ie = it + e, be = ie & 1;
            if (e > 0) mbar_wait(&tempty[be], ((ie >> 1) & 1) ^ 1);
            buf_tile[be] = -1;
            mbar_arrive(&tfull[be]);
            mbar_arrive(&tfull[be]);
          }
          break;
        }
        tc_fence_after();
        if (H64 && !(HC_TC_DIAG & 4)) {
          // D_h = H_128 x_h as two 64-column halves: q = 0: x_h,lo H_64 + x_h,hi H_64; q = 1: x_h,lo H_64 - x_h,hi H_64
#pragma unroll
          for (int h = 0; h < 2; ++h)
#pragma unroll
            for (int q = 0; q < 2; ++q)
#pragma unroll
              for (int kk = 0; kk < 8; ++kk) {
                const uint32_t a = sm0 + s * kTcTile + (2 * h + (kk >> 2)) * 16384 + (kk & 3) * 32;
                const uint32_t bh = hs0 + (kk & 3) * 32;
                umma_f16(tmem + b * 256 + h * 128 + q * 64, umma_desc_sw128(a), umma_desc_sw128(bh),
                         (q == 1 && kk >= 4) ? IDESC64_NEG : IDESC64, kk > 0 ? 1u : 0u);
              }
        } else if (!(HC_TC_DIAG & 4))
#pragma unroll
        for (int h = 0; h < 2; ++h)
#pragma unroll
          for (int kk = 0; kk < (kTcNegB ? 16 : 8); ++kk) {
            // kTcNegB: D_h = y_lo / y_hi directly (K = 256: the chunk's 4 segments, B = H_128
            // twice, negated for y_hi's upper half); else D_h = H_128 x_h (K = 128, segments
            // 2h, 2h + 1) and the epilogue's butterfly gives y
            const int seg = kTcNegB ? (kk >> 2) : 2 * h + (kk >> 2);
            const uint32_t a = sm0 + s * kTcTile + seg * 16384 + (kk & 3) * 32;
            const uint32_t bh = hs0 + ((kk >> 2) & 1) * 16384 + (kk & 3) * 32;
            umma_f16(tmem + b * 256 + h * 128, umma_desc_sw128(a), umma_desc_sw128(bh),
                     (kTcNegB && h == 1 && kk >= 8) ? IDESC_NEG : IDESC, kk > 0 ? 1u : 0u);
          }
        umma_commit(&ufree[s]);
        buf_tile[b] = tile;
        buf_stage[b] = s;
        umma_commit(&tfull[b]);
        mbar_arrive(&tfull[b]);
      }
    }
  } else if (warp >= EG * NE) {
    // ---------------- phase A: H_{n/256} across the chunks of the raw rows, in place
    const int wa = warp - EG * NE;
    uint32_t Bc0[2], Bc1[2];
    make_const_b<DT>(PL::mask_a, 0, Bc0);
    make_const_b<DT>(PL::mask_a, 1, Bc1);
    const uint32_t r0 = lane & 1, r1 = (lane >> 1) & 1, r2 = (lane >> 2) & 1, j0 = (lane >> 3) & 1,
                   j1 = (lane >> 4) & 1;
    uint32_t c_l = 0, g_l = 0;  // chunk / granule bits supplied by the lane (as fwht_rows_kernel)
    if constexpr (Q == 1) { c_l = r0; g_l = j0 | (r1 << 1) | (r2 << 2) | (j1 << 3); }
    if constexpr (Q == 2) { c_l = r0 | (r1 << 1); g_l = j0 | (j1 << 1) | (r2 << 2); }
    if constexpr (Q == 3) { c_l = r0 | (r1 << 1) | (r2 << 2); g_l = j0 | (j1 << 1); }
    if constexpr (Q == 4) { c_l = r0 | (r1 << 1) | (r2 << 2) | (j1 << 3); g_l = j0; }
    if constexpr (Q >= 5) { c_l = r0 | (r1 << 1) | (r2 << 2) | (j1 << 3) | (j0 << 4); g_l = 0; }
    constexpr int LOOP_SHIFT = 5 - PL::nloop_bits;
    const uint32_t sm0 = smem_addr(smem);
    for (int it = 0;; ++it) {
      const int s = it % STAGES;
      mbar_wait(&full[s], (it / STAGES) & 1);
      if (wa == 0 && lane == 0) trace(it, 1);
      const int tile = ctl->stage_tile[s];
      if (tile >= 0 && !(HC_TC_DIAG & 1)) {
        // UA items in flight per warp (ILP: the ldmatrix -> mma -> stmatrix chain of one
        // item is latency-bound)
        constexpr int F = 1 << PL::nx;  // fragments per item
        for (int item0 = wa; item0 < ITEMS; item0 += NA * UA) {
          uint32_t x[UA][F][4], addr[UA][F];
#pragma unroll
          for (int u = 0; u < UA; ++u) {
            const int item = item0 + u * NA < ITEMS ? item0 + u * NA : item0;  // (tail: redo item0)
            uint32_t r, lp;
            if constexpr (kTcSplit) {  // lower-half items (top loop bit clear = segments 0-1) first
              constexpr int HALF = ITEMS / 2, HL = NLOOP / 2;
              const int hi = item >= HALF, rest = item - hi * HALF;
              r = uint32_t(rest / HL);
              lp = uint32_t(hi * HL + rest % HL);
              if (hi) mbar_wait(&full_hi[s], uint32_t((it / STAGES) & 1));
            } else {
              r = uint32_t(item / NLOOP);
              lp = uint32_t(item % NLOOP);
            }
            const uint32_t gg = g_l | (lp << LOOP_SHIFT);
#pragma unroll
            for (int xi = 0; xi < F; ++xi) {
              addr[u][xi] = sm0 + s * kTcTile + goff_tc<C>(r, c_l | (uint32_t(xi) << 5), gg);
              ldsm_x4_t(addr[u][xi], x[u][xi]);
            }
          }
#pragma unroll
          for (int u = 0; u < UA; ++u) {
            float dd[F][8];
#pragma unroll
            for (int xi = 0; xi < F; ++xi) {
              if constexpr (PL::two_stage) {
                stage_da_j0_f32<DT>(x[u][xi], Bc0, Bc1, dd[xi]);
              } else {
                stage_da_f32<DT>(x[u][xi], Bc0, Bc1, dd[xi]);
              }
            }
#pragma unroll
            for (int bb = 0; bb < PL::nx; ++bb)
#pragma unroll
              for (int xi = 0; xi < F; ++xi)
                if (!((xi >> bb) & 1)) bfly8(dd[xi], dd[xi | (1 << bb)]);
            if (u > 0 && item0 + u * NA >= ITEMS) continue;  // the tail's duplicate: no store
#pragma unroll
            for (int xi = 0; xi < F; ++xi) {
              uint32_t z[4];
#pragma unroll
              for (int q = 0; q < 4; ++q) z[q] = pack2<DT>(dd[xi][2 * q], dd[xi][2 * q + 1]);
              stsm_x4_t(addr[u][xi], z);
            }
          }
        }
      }
      fence_proxy_async_smem();  // our 16-bit image is read next by the tensor core (async proxy)
      jitter(13, it);
      __syncwarp();
      if (lane == 0) mbar_arrive(&adone[s]);
      if (wa == 0 && lane == 0) trace(it, 2);
      if (tile < 0) break;
    }
  } else {
    // ---------------- epilogue: TMEM lane quadrant warp % 4 = chunks 32q .. 32q + 31 of the tile
    // EG groups of NE warps take alternate tiles (EG = 2: group g always drains TMEM buffer g)
    const int eg = warp / NE, ew = warp % NE;
    const int quad = ew & 3, ch = ew >> 2;  // ch: column half (NE = 8)
    const int mrow = 32 * quad + lane;           // chunk row of the tile = TMEM lane
    const int r = mrow / C, c = mrow % C;
    constexpr int NJ = NE == 4 ? 4 : 2;          // 32-column groups per thread and pass
    const int j0 = NE == 4 ? 0 : 2 * ch;
    const float q_qs = copysignf(qmax_of<QT>(), s_res), q_ss = fabsf(s_res) / qmax_of<QT>();
    for (int it = eg;; it += EG) {
      const int b = it & 1;
      mbar_wait(&tfull[b], (it >> 1) & 1);
      if (warp == 0 && lane == 0) trace(it, 4);
      tc_fence_after();
      const int tile = buf_tile[b], s = buf_stage[b];
      const bool elect = ew == 0 && lane == 0;  // issues this group's code stores (kTcCodeBuf)
      if (tile < 0) {
        if (kTcCodeBuf && elect) bulk_wait_all();
        break;
      }
      if (HC_TC_DIAG & 2) {
        __syncwarp();
        if (lane == 0) mbar_arrive(&tempty[b]);
        continue;
      }
      const uint32_t tb = tmem + (uint32_t(32 * quad) << 16) + uint32_t(b * 256);
      // pass 1: max |y| over this thread's outputs (columns 32 j.. of y_lo and of y_hi)
      float a = 0.f;
#pragma unroll 1
      for (int j = j0; j < j0 + NJ; ++j) {
        float P[32], Rr[32];
        tmem_ld32(tb + 32 * j, P);
        tmem_ld32(tb + 128 + 32 * j, Rr);
        tmem_wait_ld();
#pragma unroll
        for (int e = 0; e < 32; e += 2) {
          if constexpr (!kTcNegB) bfly2(P[e], P[e + 1], Rr[e], Rr[e + 1]);  // y_lo, y_hi
          a = absmax3(a, P[e], P[e + 1]);
          a = absmax3(a, Rr[e], Rr[e + 1]);
        }
      }
      // the row's maximum: 16-lane groups (C >= 16 chunks per row), then across warps; rows of
      // C < 16 chunks are C consecutive lanes of one warp
      uint32_t au = __float_as_uint(a);
#pragma unroll
      for (int o = (C < 16 ? C : 16) / 2; o >= 1; o >>= 1) au = max(au, __shfl_xor_sync(0xffffffffu, au, o));
      if (C >= 16 && (lane & 15) == 0) red[b * NE * 2 + ew * 2 + (lane >> 4)] = __uint_as_float(au);
      jitter(14, it);
      if (kTcCodeBuf && elect) bulk_wait_read<0>();  // this group's previous code store has read its buffer
      if (NCB == 1 && elect && it > 0) mbar_wait(cbuf_free, uint32_t((it - 1) & 1));  // ... and the other group's
      named_bar_sync(1 + eg, NE * 32);
      if (warp == 0 && lane == 0) trace(it, 5);
      float am = C < 16 ? __uint_as_float(au) : 0.f;
      if constexpr (C >= 16) {
        constexpr int G = C / 16;  // 16-lane groups per row
#pragma unroll
        for (int gi = 0; gi < G; ++gi) {
          const int g16 = r * G + gi;  // covers chunks 16 g16 .. 16 g16 + 15 -> warp quadrant g16 / 2
#pragma unroll
          for (int hh = 0; hh < NE / 4; ++hh) am = absmax_nan(am, red[b * NE * 2 + ((g16 >> 1) + 4 * hh) * 2 + (g16 & 1)]);
        }
      }
      int64_t ri, rj;
      const bool valid = TileRows(g, tile).at(g, r, ri, rj);
      const int64_t row = ri * g.m_inner + rj;  // codes and scales in (i, j) row order
      float mul, sc;
      const bool fast = quant_fast_range(am, 0x1p100f);
      if (fast) {
        sc = am * q_ss;
        mul = q_qs * rcp_ftz(am);
      } else {
        float inv;
        row_scale_of<QT>(am * fabsf(s_res), sc, inv);
        mul = s_res * inv;
      }
      stf32_if(row_scale + row, sc, valid && c == 0 && ch == 0);
      // pass 2: codes, staged in the tile's (consumed) stage as the 128-byte-swizzled image of
      // its contiguous code block: 128-byte lines L (E4M3 / INT8: L = 2 m + h, the half-chunk
      // h of chunk row m; INT4: L = m), 16-byte granule q at (q ^ (L & 7))
      uint8_t* const qs = kTcCodeBuf ? codebuf + (NCB == 1 ? 0 : eg) * tc_code_bytes<QT>() : smem + s * kTcTile;
#pragma unroll 1
      for (int j = j0; j < j0 + ((HC_TC_DIAG & 16) ? 0 : NJ); ++j) {
        float P[32], Rr[32];
        tmem_ld32(tb + 32 * j, P);
        tmem_ld32(tb + 128 + 32 * j, Rr);
        tmem_wait_ld();
        if constexpr (!kTcNegB) {
#pragma unroll
          for (int e = 0; e < 32; e += 2) bfly2(P[e], P[e + 1], Rr[e], Rr[e + 1]);  // y_lo, y_hi
        }
        uint32_t w[2][8];
        if (fast) {  // a real branch: both epilogues inline would be computed and selected
#pragma unroll
          for (int hf = 0; hf < 2; ++hf)
#pragma unroll
            for (int q = 0; q < 8; ++q) {
              const float* v = hf ? Rr : P;
              w[hf][q] = quant4_fast<QT>(v[4 * q], v[4 * q + 1], v[4 * q + 2], v[4 * q + 3], mul);
            }
        } else {
#pragma unroll
          for (int hf = 0; hf < 2; ++hf)
#pragma unroll
            for (int q = 0; q < 8; ++q) {
              const float* v = hf ? Rr : P;
              w[hf][q] = quant4<QT>(v[4 * q] * mul, v[4 * q + 1] * mul, v[4 * q + 2] * mul, v[4 * q + 3] * mul);
            }
        }
        if (!(HC_TC_DIAG & 8)) {
#pragma unroll
          for (int hf = 0; hf < 2; ++hf) {
            if constexpr (QT == QT_INT4) {  // 32 codes = 16 bytes: granule 4 hf + j of line m
              const uint32_t L = uint32_t(mrow), gq = uint32_t(4 * hf + j);
              *reinterpret_cast<uint4*>(qs + L * 128 + ((gq ^ (L & 7u)) << 4)) =
                  make_uint4(__byte_perm(w[hf][0], w[hf][1], 0x5410), __byte_perm(w[hf][2], w[hf][3], 0x5410),
                             __byte_perm(w[hf][4], w[hf][5], 0x5410), __byte_perm(w[hf][6], w[hf][7], 0x5410));
            } else {  // 32 codes = granules 2 j, 2 j + 1 of line 2 m + hf
              const uint32_t L = uint32_t(2 * mrow + hf), gq = uint32_t(2 * j);
              *reinterpret_cast<uint4*>(qs + L * 128 + ((gq ^ (L & 7u)) << 4)) =
                  make_uint4(w[hf][0], w[hf][1], w[hf][2], w[hf][3]);
              *reinterpret_cast<uint4*>(qs + L * 128 + (((gq + 1) ^ (L & 7u)) << 4)) =
                  make_uint4(w[hf][4], w[hf][5], w[hf][6], w[hf][7]);
            }
          }
        }
      }
      tc_fence_before();
      fence_proxy_async_smem();  // the staged codes are read next by the TMA store (async proxy)
      jitter(15, it);
      __syncwarp();
      if (lane == 0) {
        mbar_arrive(&tempty[b]);
        if constexpr (!kTcCodeBuf) mbar_arrive(&cready[s]);
      }
      if constexpr (kTcCodeBuf) {  // the group's codes are staged: one TMA tensor store of them
        named_bar_sync(1 + eg, NE * 32);
        if (elect) {
          jitter(16, it);
          const TileRows tr(g, tile);
          tma_store_4d(&tm_q, 0, 0, int(tr.j0), int(tr.i0), qs);
          bulk_commit();
          if constexpr (NCB == 1) {  // the next tile (the other group) may write the buffer once this store read it
            bulk_wait_read<0>();
            mbar_arrive(cbuf_free);
          }
        }
      }
      if (warp == 0 && lane == 0) trace(it, 6);
    }
  }
  // teardown: every role is done with tensor memory
  tc_fence_before();
  __syncthreads();
  if (warp == WM) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "n"(kTcCols) : "memory");
  }
}

}  // namespace hadacore
