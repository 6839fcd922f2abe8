// fwht_small.cuh -- sm_100a kernel for rows shorter than 128 elements (n = 2..64),
// SURVEY.md 8(f) NEXT-2 ("size breadth: n = 2..64", SPEC S:49's domain 2 <= d).
// "P:NN" = /root/reference/PAPER.md line NN.
//
// Why not the tensor cores here: a 256-element mma fragment would hold 256/n rows,
// and with two m16n8k16 stages every fragment bit but one is contracted by one of
// them, so a row bit would be contracted with a
// structural-zero I_2 factor -- 0 * Inf = NaN would leak a non-finite row into its
// neighbours (reading R13).  With k = log2 n <= 6 butterfly stages the work is
// ~k + 3 fp32 instructions per element, far below the issue rate that the HBM
// stream needs, so the P:50-64 listing runs as fp32 register
// butterflies.
//
// Layout of the work: the producer warp streams contiguous 1-D byte ranges
// HBM -> shared memory (cp.async.bulk, UBLKCP) into a STAGES-deep ring and writes
// finished stages back with 1-D bulk stores (shared -> global), like
// fwht_rows_kernel.  A consumer lane owns one ITEM: for n <= 8 one 16-byte granule
// (8 elements = 8/n whole rows), for n >= 16 one whole row of G = n/8 granules.
// Bank conflicts of the per-lane row reads (row stride 2n bytes) are avoided by
// reading granule j ^ c (c a lane constant, so 8 consecutive lanes touch 8
// different 16-byte bank groups); the granule-bit butterflies then use the sign
// trick of DESIGN.md (a butterfly with its second operand negated is the butterfly
// followed by a swap across that bit), so the result for granule j ^ c lands in
// register slot j up to a known sign, which is folded into the final scale; slot
// j is written back to the address it was read from.
#pragma once
#include "fwht_kernel.cuh"

#ifndef HC_SMALL_STAGE_CODES
#define HC_SMALL_STAGE_CODES 1
#endif

namespace hadacore {

#ifndef HC_SMALL_SPLIT
#define HC_SMALL_SPLIT 0  // bit 0: n = 32, bit 1: n = 64 fused quantization with half rows per lane (SPLIT): measured 15-25 % slower, off
#endif
#ifndef HC_SMALL_PACKED
#define HC_SMALL_PACKED 0  // 1: packed f32x2 butterflies in fwht_small_kernel -- measured mixed (quant n = 32, 64 -2..-6 %, Q/K quant n = 8..64 +3 %), off
#endif
#ifndef HC_SMALL_PACKED_GRID
#define HC_SMALL_PACKED_GRID 1  // ... but on for the row-grid (Q/K head) instantiations: Q/K quant n = 8..64 +3 %
#endif
constexpr bool kSmallPacked = HC_SMALL_PACKED != 0;
// packed butterfly with the second operand times s: (a0, a1) <- b * s + a, (b0, b1) <- b * ns + a (ns = -s)
// (fma.rn.f32x2, SASS FFMA2: IEEE-identical to the two scalar fmaf of each half)
__device__ __forceinline__ void bfly2_sgn(float& a0, float& a1, float& b0, float& b1, float s, float ns) {
  asm("{.reg .b64 a, b, p, q, r, t;\n mov.b64 a, {%0,%1};\n mov.b64 b, {%2,%3};\n mov.b64 p, {%4,%4};\n"
      " mov.b64 q, {%5,%5};\n fma.rn.f32x2 r, b, p, a;\n fma.rn.f32x2 t, b, q, a;\n"
      " mov.b64 {%0,%1}, r;\n mov.b64 {%2,%3}, t;}"
      : "+f"(a0), "+f"(a1), "+f"(b0), "+f"(b1)
      : "f"(s), "f"(ns));
}

__device__ __forceinline__ void bulk_s2g(void* dst, const void* src, uint32_t bytes) {
#if HC_STORE_HINT  // evict-first in L2, as the TMA tensor stores (fwht_kernel.cuh)
  asm volatile("cp.async.bulk.global.shared::cta.bulk_group.L2::cache_hint [%0], [%1], %2, %3;" ::"l"(dst),
               "r"(smem_addr(src)), "r"(bytes), "l"(policy_evict_first())
               : "memory");
#else
  asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(dst), "r"(smem_addr(src)),
               "r"(bytes)
               : "memory");
#endif
}

// Fused quantization with rows of >= 16 elements: the codes of a tile are staged in a
// per-stage shared-memory buffer and written by the producer with one 1-D bulk store,
// instead of per-lane 4/8-byte global stores at a row stride (which touch 32 sectors per
// warp instruction).  Bytes of that buffer per stage (0: codes from registers).  A row-grid
// tile uses it when its codes are one contiguous range of a multiple of 16 bytes (whole
// inner rows per box, bi == m_inner); otherwise its codes go from registers
// (profiles/r01_ab_small_stage_codes.txt).
template <int N, int QT, bool GRID, int TILE_BYTES>
__host__ __device__ constexpr int small_code_stage_bytes() {
  // (contiguous rows: only with >= 16 code bytes per row -- INT4 n = 16 measured faster from registers)
  return (QT >= 0 && N >= 16 && (GRID || N * (QT == QT_INT4 ? 1 : 2) / 2 % 16 == 0) && HC_SMALL_STAGE_CODES)
             ? TILE_BYTES / 2 * (QT == QT_INT4 ? 1 : 2) / 2
             : 0;
}

template <int DT>
__device__ __forceinline__ void unpack2(uint32_t w, float& lo, float& hi) {
  if constexpr (DT == DT_F16) {
    const float2 f = __half22float2(*reinterpret_cast<const __half2*>(&w));
    lo = f.x;
    hi = f.y;
  } else {
    lo = __uint_as_float(w << 16);
    hi = __uint_as_float(w & 0xffff0000u);
  }
}

// Rows of N = 2..64 elements; TILE_BYTES per ring stage, NT consumer warps, U items
// per lane in flight.
// QT >= 0: fused per-row quantization (NEXT-1 for n < 128): a lane holds whole rows, so
// the row max is in-lane; codes go straight from registers to out_q, scales to row_scale.
// GRID: rows on a 2-level grid (NEXT-3 row grids, n >= 8): a tile is a
// bo x bi box of rows moved by 3-D TMA tensor copies (rows outside the grid are zero-filled
// on load and clipped on store), instead of a contiguous byte range.
template <int N, int DT, int TILE_BYTES, int STAGES, int NT, int U, int QT = QT_NONE, bool GRID = false>
__global__ void __launch_bounds__((NT + 1) * 32, 1)
    fwht_small_kernel(const uint16_t* __restrict__ in, uint16_t* __restrict__ out, int64_t total_bytes,
                      int64_t num_tiles, float scale, uint8_t* __restrict__ out_q = nullptr,
                      float* __restrict__ row_scale = nullptr, const __grid_constant__ CUtensorMap tm_in = {},
                      const __grid_constant__ CUtensorMap tm_out = {}, const RowGrid g = {}) {
  constexpr int K = log2_n<N>();
  // SPLIT (fused quantization of contiguous rows, n = 32, 64): an item is HALF a row, held by
  // lanes 2r, 2r + 1; the top index bit is a butterfly across the lane pair (shuffles), the
  // row maximum one more shuffle -- half the registers of a whole row per lane
  constexpr bool SPLIT = QT >= 0 && !GRID && (N == 64 || N == 32) && (HC_SMALL_SPLIT & (N / 32)) != 0;
  constexpr int G = N >= 8 ? N / 8 / (SPLIT ? 2 : 1) : 1;  // granules per item
  constexpr int ITEM_BYTES = 16 * G;
  constexpr int KG = N >= 16 ? K - 3 - (SPLIT ? 1 : 0) : 0;  // granule bits of an item
  constexpr int KE = K < 3 ? K : 3;                // element bits inside a granule
  static_assert(TILE_BYTES % ITEM_BYTES == 0 && STAGES <= 16, "tile layout");
  static_assert(!GRID || N >= 8, "row grids: n >= 8 (16-byte TMA rows)");

  constexpr int CODE_STAGE = small_code_stage_bytes<N, QT, GRID, TILE_BYTES>();
  constexpr bool PACKED = kSmallPacked || (GRID && HC_SMALL_PACKED_GRID != 0);  // f32x2 butterflies
  extern __shared__ __align__(1024) uint8_t smem[];
  uint8_t* const codes = smem + STAGES * TILE_BYTES;  // CODE_STAGE bytes per stage (may be 0)
  SchedCtl* ctl = reinterpret_cast<SchedCtl*>(smem + STAGES * (TILE_BYTES + CODE_STAGE));
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + STAGES * (TILE_BYTES + CODE_STAGE) + sizeof(SchedCtl));
  uint64_t* done = full + STAGES;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;

  if (threadIdx.x == 0) {
    mbar_init(&ctl->clc_bar, 1);
#pragma unroll
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&done[s], NT);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    fence_proxy_async_smem();
  }
  __syncthreads();

  // bytes of tile t, and its 16-byte-multiple prefix moved by the bulk engine (the
  // rest, < 16 bytes, exists only for n <= 4 and is handled by one consumer lane)
  auto tile_bytes = [&](int64_t t) -> int {
    if constexpr (GRID) return int(total_bytes);  // GRID: total_bytes carries the (full) box size
    const int64_t left = total_bytes - t * TILE_BYTES;
    return int(left < TILE_BYTES ? left : TILE_BYTES);
  };

  // codes of tile t staged in shared memory (CODE_STAGE > 0): the destination byte offset
  // in out_q and the byte count, or a count of 0 (codes from registers)
  constexpr int CR = N * (QT == QT_INT4 ? 1 : 2) / 2;  // code bytes per row
  // contiguous rows with >= 16 code bytes each: every tile's codes are staged
  constexpr bool STAGE_ALWAYS = CODE_STAGE > 0 && !GRID;
  auto staged_codes = [&](int64_t t, int64_t& dst) -> uint32_t {
    if constexpr (CODE_STAGE == 0) {
      return 0u;
    } else if constexpr (GRID) {
      if (g.nib != 1 || g.m_inner != (int64_t(1) << g.lbi) || ((CR << (g.lbi + g.lp)) & 15) != 0) return 0u;
      const TileRowsFast tr(g, t);
      dst = (tr.lin0 << g.lp) * CR;
      return uint32_t(tr.ni << (g.lbi + g.lp)) * CR;
    } else {
      const uint32_t cb = uint32_t(tile_bytes(t)) / (2 * N) * CR;
      dst = t * CODE_STAGE;
      return (cb & 15u) ? 0u : cb;
    }
  };

  pdl_launch_dependents();
  if (warp == NT) {
    // ---------------- producer: 1-D bulk loads into the ring, 1-D bulk stores out of it
    if (lane == 0) {
      pdl_wait();  // the previous kernel on the stream has completed
      const uint64_t pol = policy_evict_first();
      uint32_t clc_phase = 0;
      int64_t tile = blockIdx.x;
      auto advance = [&](int64_t t) -> int64_t {
        if constexpr (kClc) {
          return clc_result(ctl, clc_phase);
        } else {
          return t + gridDim.x;
        }
      };
      if constexpr (GRID) {
        tma_prefetch(&tm_in);
        tma_prefetch(&tm_out);
      }
      auto load = [&](int st, int64_t t) {
        const uint32_t b16 = uint32_t(tile_bytes(t)) & ~15u;
        mbar_arrive_expect_tx(&full[st], b16);
        if constexpr (GRID) {
          const TileRows tr(g, t);
          tma_load_3d(smem + st * TILE_BYTES, &tm_in, 0, int(tr.j0), int(tr.i0), &full[st], pol);
        } else {
          if (b16) bulk_g2s(smem + st * TILE_BYTES, reinterpret_cast<const uint8_t*>(in) + t * TILE_BYTES, b16, &full[st], pol);
        }
      };
      bool ended = false;
      for (int k = 0; k < STAGES; ++k) {  // fill the ring
        if (tile < 0 || tile >= num_tiles) {
          ctl->stage_tile[k] = -1;
          mbar_arrive(&full[k]);
          ended = true;
          break;
        }
        ctl->stage_tile[k] = int(tile);
        if constexpr (kClc) clc_request(ctl);
        load(k, tile);
        tile = advance(tile);
      }
      for (int it = 0;; ++it) {
        const int s = it % STAGES;
        const int64_t t = ctl->stage_tile[s];
        if (t < 0) break;
        mbar_wait(&done[s], (it / STAGES) & 1);
        const uint32_t b16 = uint32_t(tile_bytes(t)) & ~15u;
        if constexpr (QT < 0) {
          if constexpr (GRID) {
            const TileRows tr(g, t);  // rows outside the grid are clipped by the TMA unit
            tma_store_3d(&tm_out, 0, int(tr.j0), int(tr.i0), smem + s * TILE_BYTES);
          } else {
            if (b16) bulk_s2g(reinterpret_cast<uint8_t*>(out) + t * TILE_BYTES, smem + s * TILE_BYTES, b16);
          }
        } else {  // quantizing: the stage itself is not written back; the staged codes are
          int64_t dst = 0;
          const uint32_t cb = staged_codes(t, dst);
          if (cb) bulk_s2g(out_q + dst, codes + s * CODE_STAGE, cb);
        }
        bulk_commit();
        if (ended) continue;
        if (tile < 0 || tile >= num_tiles) {
          ctl->stage_tile[s] = -1;
          mbar_arrive(&full[s]);
          ended = true;
          continue;
        }
        ctl->stage_tile[s] = int(tile);
        if constexpr (kClc) clc_request(ctl);
        bulk_wait_read<0>();  // the store just issued (and older ones) has read the stage
        load(s, tile);
        tile = advance(tile);
      }
      bulk_wait_all();
    }
    return;
  }

  // ---------------- consumers
  // granule XOR of this lane: 8 consecutive lanes read 8 distinct bank groups
  constexpr int LG = KG;  // log2 G
  const uint32_t c = G > 1 ? (uint32_t(lane) >> (3 - LG)) & uint32_t(G - 1) : 0u;
  // per-slot scale: scale * (-1)^popcount((j ^ c) & c) (sign left by the swapped butterflies)
  float sc[G];
#pragma unroll
  for (int j = 0; j < G; ++j) sc[j] = (__popc((uint32_t(j) ^ c) & c) & 1) ? -scale : scale;
  // fused quantization, fast path: scale = max|v| |scale| / Q, multiplier sign(scale) Q / max|v|
  const float q_qs = copysignf(qmax_of<QT == QT_NONE ? QT_E4M3 : QT>(), scale);
  const float q_ss = fabsf(scale) / qmax_of<QT == QT_NONE ? QT_E4M3 : QT>();
  (void)q_qs;
  (void)q_ss;
  float sg[KG > 0 ? KG : 1];  // sign of the second operand of the granule-bit butterflies
#pragma unroll
  for (int b = 0; b < KG; ++b) sg[b] = ((c >> b) & 1u) ? -1.f : 1.f;

  for (int it = 0;; ++it) {
    const int s = it % STAGES;
    mbar_wait(&full[s], (it / STAGES) & 1);
    const int64_t tile = ctl->stage_tile[s];
    if (tile < 0) break;
    uint8_t* const tb = smem + s * TILE_BYTES;
    const int bytes = tile_bytes(tile);
    const int b16 = bytes & ~15;
    const int items = (bytes + ITEM_BYTES - 1) / ITEM_BYTES;
    int64_t qdst_unused = 0;
    const bool stage_q = STAGE_ALWAYS || staged_codes(tile, qdst_unused) != 0u;
    (void)stage_q;
    for (int i0 = warp * 32 + lane; i0 < items; i0 += NT * 32 * U) {
      float v[U][8 * G];
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const int item = i0 + u * NT * 32;
        if (item >= items) continue;
        const uint8_t* p = tb + item * ITEM_BYTES;
#pragma unroll
        for (int j = 0; j < G; ++j) {
          uint32_t w[4];
          if (N <= 4 && item * 16 + 16 > b16) {
            // partial last granule (n <= 4, total bytes not a multiple of 16): whole rows
            // of 4 or 8 bytes straight from global memory (after the producer's pdl_wait
            // via the full barrier), zero-filled
            const uint32_t* gsrc =
                reinterpret_cast<const uint32_t*>(reinterpret_cast<const uint8_t*>(in) + tile * TILE_BYTES + item * 16);
            const int nw = (bytes - item * 16) / 4;
#pragma unroll
            for (int q = 0; q < 4; ++q) w[q] = q < nw ? gsrc[q] : 0u;
          } else {
            lds128(p + 16 * (uint32_t(j) ^ c), w[0], w[1], w[2], w[3]);
          }
#pragma unroll
          for (int q = 0; q < 4; ++q) unpack2<DT>(w[q], v[u][8 * j + 2 * q], v[u][8 * j + 2 * q + 1]);
        }
      }
#pragma unroll
      for (int u = 0; u < U; ++u) {
        // element bits (inside a granule; for n <= 8 each row of n elements is
        // contiguous in the granule, so bits 0..k-1 never cross rows): P:50-64 butterflies
        // (bits >= 1 as packed FADD2 / FFMA2 pairs of elements e, e + 1: the same IEEE
        // operations as the scalar form, half the issue slots; bit 0 pairs e with e + 1 itself)
#pragma unroll
        for (int b = 0; b < KE; ++b)
#pragma unroll
          for (int e = 0; e < 8 * G; ++e)
            if (!(e & (1 << b))) {
              if (b == 0 || !PACKED) {
                const float p0 = v[u][e], p1 = v[u][e | (1 << b)];
                v[u][e] = p0 + p1;
                v[u][e | (1 << b)] = p0 - p1;
              } else if (!(e & 1)) {
                bfly2(v[u][e], v[u][e + 1], v[u][e | (1 << b)], v[u][(e | (1 << b)) + 1]);
              }
            }
        // granule bits: butterflies with the second operand times sg[b] (= the plain
        // butterfly followed by a swap across bit b when c has bit b set)
#pragma unroll
        for (int b = 0; b < KG; ++b)
#pragma unroll
          for (int e = 0; e < 8 * G; ++e)
            if (!(e & (8 << b))) {
              if (!PACKED) {
                const float p0 = v[u][e], p1 = v[u][e | (8 << b)];
                v[u][e] = fmaf(p1, sg[b], p0);
                v[u][e | (8 << b)] = fmaf(p1, -sg[b], p0);
              } else if (!(e & 1)) {
                bfly2_sgn(v[u][e], v[u][e + 1], v[u][e | (8 << b)], v[u][(e | (8 << b)) + 1], sg[b], -sg[b]);
              }
            }
      }
      if constexpr (SPLIT) {
        // the top index bit across the lane pair (same slot -> granule map and slot signs in
        // both lanes: c depends on lane >> 1): lane 2r keeps a + b, lane 2r + 1 a - b, the
        // P:50-64 butterfly in the same order and fp32 rounding as the in-lane version
        const unsigned pair = __activemask();  // partners are active together (whole rows)
        const bool hi = lane & 1;
#pragma unroll
        for (int u = 0; u < U; ++u)
#pragma unroll
          for (int e = 0; e < 8 * G; ++e) {
            const float p = __shfl_xor_sync(pair, v[u][e], 1);
            v[u][e] = hi ? p - v[u][e] : v[u][e] + p;
          }
      }
      if constexpr (QT >= 0) {
        // ---- fused quantization: rows are in-lane (n >= 16: the item; n <= 8: 8/n rows of
        // the granule, contiguous in v); y = v * sc[j], so |y| = |v| |scale|
        constexpr int RI = N >= 8 ? 1 : 8 / N;  // rows per item
        constexpr int CB2 = QT == QT_INT4 ? 1 : 2;  // code bytes per 2 elements
#pragma unroll
        for (int u = 0; u < U; ++u) {
          const int item = i0 + u * NT * 32;
          if (item >= items) continue;
          int64_t el0 = (tile * TILE_BYTES + int64_t(item) * ITEM_BYTES) / 2;  // first element of the item
          if constexpr (GRID) {  // n >= 8: one row per item, at (i, j) of the grid; codes/scales in row order
            int64_t gi = 0, gj = 0;
            if (!TileRows(g, tile).at(g, item >> g.lp, gi, gj)) continue;  // (pseudo-)row of the grid
            el0 = (((gi * g.m_inner + gj) << g.lp) + (item & ((1 << g.lp) - 1))) * N;
          }
          float mul[RI], scr[RI];
          bool fast = true;
#pragma unroll
          for (int rr = 0; rr < RI; ++rr) {
            float a = 0.f;
#pragma unroll
            for (int e = 0; e < (N >= 8 ? 8 * G : N); ++e) a = absmax_nan(a, v[u][rr * N + e]);
            if constexpr (SPLIT) a = absmax_nan(a, __shfl_xor_sync(__activemask(), a, 1));  // |.| of a max is itself
            if (quant_fast_range(a, 0x1p100f)) {
              scr[rr] = a * q_ss;                 // max |y| / Q
              mul[rr] = q_qs * rcp_ftz(a);        // Q / max |v|, times sign(scale)
            } else {
              float inv;
              row_scale_of<QT>(a * fabsf(scale), scr[rr], inv);
              mul[rr] = inv * scale;              // per unit of v (y = v * scale * sign_j)
              fast = false;
            }
          }
          // row scales: the item's RI rows are consecutive -> one vector store when whole
          const int64_t row0 = el0 / N;
          // (row_scale need only be 4-byte aligned: vector stores when it is 8/16-byte aligned)
          const bool whole = (N >= 8 || item * 16 + 16 <= b16) &&
                             (reinterpret_cast<uintptr_t>(row_scale) & (RI == 4 ? 15u : (RI == 2 ? 7u : 3u))) == 0;
          if constexpr (RI == 4) {
            if (whole) *reinterpret_cast<float4*>(row_scale + row0) = make_float4(scr[0], scr[1], scr[2], scr[3]);
          } else if constexpr (RI == 2) {
            if (whole) *reinterpret_cast<float2*>(row_scale + row0) = make_float2(scr[0], scr[1]);
          } else {
            if (!SPLIT || !(lane & 1)) row_scale[row0] = scr[0];
          }
          if (!whole)  // partial granule (n <= 4): the valid rows only
            for (int rr = 0; rr < RI; ++rr)
              if (item * 16 + rr * 2 * N < bytes) row_scale[row0 + rr] = scr[rr];
#pragma unroll
          for (int j = 0; j < G; ++j) {
            // slot sign (sc[j] = +-scale): the multipliers above already carry sign(scale)
            const float sj = (sc[j] < 0.f) != (scale < 0.f) ? -1.f : 1.f;
            uint32_t c0, c1;
            const float* vv = &v[u][8 * j];
            if (fast && N >= 4) {  // one multiplier per group of 4 (a row has >= 4 elements)
              c0 = quant4_fast<QT>(vv[0], vv[1], vv[2], vv[3], sj * mul[N >= 8 ? 0 : 0]);
              c1 = quant4_fast<QT>(vv[4], vv[5], vv[6], vv[7], sj * mul[N >= 8 ? 0 : (4 / N < RI ? 4 / N : 0)]);
            } else {
              float t[8];
#pragma unroll
              for (int e = 0; e < 8; ++e)  // + 0: a zero stays +0 (code 0x00) whatever the slot's sign
                t[e] = fmaf(vv[e] * sj, mul[N >= 8 ? 0 : (e / N)], 0.f);
              c0 = quant4<QT>(t[0], t[1], t[2], t[3]);
              c1 = quant4<QT>(t[4], t[5], t[6], t[7]);
            }
            const int64_t cbyte = ((el0 + 8 * int64_t(uint32_t(j) ^ c)) * CB2) / 2;  // slot j holds granule j ^ c
            if (N <= 4 && item * 16 + 16 > b16) {  // partial last granule: only the valid rows' codes
              const int valid = (bytes - item * 16) / 2 * CB2 / 2;  // code bytes
              const uint32_t cw[2] = {QT == QT_INT4 ? __byte_perm(c0, c1, 0x5410) : c0, c1};
              for (int bq = 0; bq < valid; ++bq) out_q[cbyte + bq] = uint8_t(cw[bq >> 2] >> (8 * (bq & 3)));
            } else if (STAGE_ALWAYS || (CODE_STAGE > 0 && stage_q)) {  // into the stage's code buffer (row `item`)
              uint8_t* dst = codes + s * CODE_STAGE + ((int64_t(item) * (8 * G) + 8 * int64_t(uint32_t(j) ^ c)) * CB2) / 2;
              if constexpr (QT == QT_INT4) {
                asm volatile("st.shared.u32 [%0], %1;" ::"r"(smem_addr(dst)), "r"(__byte_perm(c0, c1, 0x5410)) : "memory");
              } else {
                asm volatile("st.shared.v2.u32 [%0], {%1, %2};" ::"r"(smem_addr(dst)), "r"(c0), "r"(c1) : "memory");
              }
            } else if constexpr (QT == QT_INT4) {
              *reinterpret_cast<uint32_t*>(out_q + cbyte) = __byte_perm(c0, c1, 0x5410);
            } else {
              *reinterpret_cast<uint2*>(out_q + cbyte) = make_uint2(c0, c1);
            }
          }
        }
      } else {
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const int item = i0 + u * NT * 32;
        if (item >= items) continue;
        uint8_t* p = tb + item * ITEM_BYTES;
#pragma unroll
        for (int j = 0; j < G; ++j) {
          uint32_t w[4];
#pragma unroll
          for (int q = 0; q < 4; ++q)  // fma with +0: an exact zero is +0 whatever the slot's sign (so the
            w[q] = pack2<DT>(fmaf(v[u][8 * j + 2 * q], sc[j], 0.f),   // bits do not depend on the lane a row lands on)
                             fmaf(v[u][8 * j + 2 * q + 1], sc[j], 0.f));
          if (N <= 4 && item * 16 + 16 > b16) {
            uint32_t* gdst = reinterpret_cast<uint32_t*>(reinterpret_cast<uint8_t*>(out) + tile * TILE_BYTES + item * 16);
            const int nw = (bytes - item * 16) / 4;
#pragma unroll
            for (int q = 0; q < 4; ++q)
              if (q < nw) gdst[q] = w[q];
          } else {
            stg_sh128(p + 16 * (uint32_t(j) ^ c), w);
          }
        }
      }
      }
    }
    fence_proxy_async_smem();  // this warp's smem writes -> visible to the bulk store
    __syncwarp();
    if (lane == 0) mbar_arrive(&done[s]);
  }
}

}  // namespace hadacore
