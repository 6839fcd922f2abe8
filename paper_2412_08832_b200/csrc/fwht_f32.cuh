// fwht_f32.cuh -- full-speed fp32 path (SURVEY.md 8(f) NEXT-2 "a full-speed fp32
// path"; north_star's fp32 path, tolerance 1e-5).  "P:NN" = /root/reference/PAPER.md.
//
// fp32 has no tensor-core shortcut that keeps 1e-5 (tf32 rounds operands to 10
// mantissa bits), so the P:50-64 listing runs as fp32 register butterflies.  The row
// tile sits in shared memory (1-D bulk copies in and out by a producer warp, CLC tile
// scheduling, as fwht_small_kernel) and the k = log2 n index bits are processed in
// phases of up to 5 bits, one register-resident column of <= 32 elements per lane:
//   phase 0   bits 0..4: a lane owns 32 contiguous floats (8 granules of 16 B); lane
//             l reads granule j ^ (l & 7) into slot j (8 consecutive lanes -> 8 bank
//             groups) and the granule-bit butterflies are the sign-folded variant
//             (out_p = alpha u + v, out_q = u - alpha v, alpha = -1 where the lane's
//             XOR has the bit) so slot j ends holding exactly the result for
//             granule j ^ c -- written back to where it was read, with no extra op;
//   phase p   bits 5p..5p+4: a lane owns a column of 2^w elements at stride 2^5p;
//             consecutive lanes take consecutive columns, so every LDS.32/STS.32 of
//             a warp touches 32 consecutive words (conflict-free).
// A named barrier over the consumer warps separates phases; the last phase applies
// `scale`.  Rows of n = 2^15 (128 KiB of fp32) do not fit a double-buffered ring of
// whole rows in one CTA: fwht_f32_stream_kernel (the default, below) streams them in
// 64 KiB chunks and gathers the cross-chunk phase into registers; fwht_f32_ring_kernel
// (HC_F32_STREAM=0), fwht_f32_pair_kernel (HC_F32_PAIR, 2-CTA clusters), fwht_f32_mc_kernel
// (HC_F32_MC) and the two-pass variant (HC_F32_TWO_PASS) are kept for A/B.
#pragma once
#include "fwht_small.cuh"

namespace hadacore {

// Bit plan of the fp32 kernel (k = log2 n): phase 0 takes B0 bits on 2^max(B0, 5)
// contiguous floats per lane; later phases take W bits starting at LO.  Widths
// are balanced so that no phase spends a full shared-memory round trip on a
// single bit (k = 11: 6 + 5, k = 12: 6 + 6 instead of 5 + 5 + 1, 5 + 5 + 2).
#ifndef HC_F32_WIDE
#define HC_F32_WIDE 0  // 1: k = 13, 14 in two 7-bit phases (128 floats per lane): measured 6.7 -> 5.4 TB/s, off
#endif
template <int K>
struct F32Plan {
  static constexpr bool WIDE = HC_F32_WIDE && K >= 13;
  static constexpr int B0 = WIDE ? 7 : ((K == 11 || K == 12) ? 6 : (K < 5 ? K : 5));
  static constexpr int NPH = K <= 5 ? 1 : ((K <= 12 || WIDE) ? 2 : 3);
  static constexpr int W1 = NPH == 1 ? 0 : (WIDE ? K - 7 : (K == 13 ? 4 : (K - B0 < 5 ? K - B0 : (K == 12 ? 6 : 5))));
  static constexpr int LO2 = B0 + W1;
  static constexpr int W2 = NPH == 3 ? K - LO2 : 0;
};

// Phase of the fp32 kernel on a tile of `rows` whole rows in shared memory: bits
// LO .. LO+W-1 over columns of CW = 2^W floats at stride 2^LO; a lane takes
// CPL = max(1, 32 / CW) columns per iteration (NT*32 apart, so a warp's accesses are
// 32 consecutive words); LAST multiplies by `scale`.
template <int N, int LO, int W, bool LAST, int NT>
__device__ __forceinline__ void f32_phase(float* tb, int rows, int tid, float scale) {
  constexpr int K = log2_n<N>();
  constexpr int CW = 1 << W, CPL = CW >= 32 ? 1 : 32 / CW, LPR = K - W, VL = CW * CPL;
  const int cols = rows << LPR;
  for (int q0 = tid; q0 < cols; q0 += NT * 32 * CPL) {
    float v[VL];
    int base[CPL];
#pragma unroll
    for (int k2 = 0; k2 < CPL; ++k2) {
      const int q = q0 + k2 * NT * 32;
      const int r = q >> LPR, cc = q & ((1 << LPR) - 1);
      base[k2] = q < cols ? r * N + ((cc >> LO) << (LO + W)) + (cc & ((1 << LO) - 1)) : -1;
#pragma unroll
      for (int t = 0; t < CW; ++t) v[k2 * CW + t] = base[k2] >= 0 ? tb[base[k2] + (t << LO)] : 0.f;
    }
#pragma unroll
    for (int b = 0; b < W; ++b)
#pragma unroll
      for (int e = 0; e < VL; ++e)
        if (!(e & (1 << b))) {
          const float p0 = v[e], p1 = v[e | (1 << b)];
          v[e] = p0 + p1;
          v[e | (1 << b)] = p0 - p1;
        }
    if constexpr (LAST) {
#pragma unroll
      for (int e = 0; e < VL; ++e) v[e] *= scale;
    }
#pragma unroll
    for (int k2 = 0; k2 < CPL; ++k2)
#pragma unroll
      for (int t = 0; t < CW; ++t)
        if (base[k2] >= 0) tb[base[k2] + (t << LO)] = v[k2 * CW + t];
  }
}

template <int N, int TILE_BYTES, int STAGES, int NT>
__global__ void __launch_bounds__((NT + 1) * 32, 1)
    fwht_f32_fast_kernel(const float* __restrict__ in, float* __restrict__ out, int64_t total_bytes,
                         int64_t num_tiles, float scale) {
  constexpr int K = log2_n<N>();
  using PL = F32Plan<K>;
  constexpr int NPH = PL::NPH;
  constexpr int K0 = PL::B0;                    // bits of phase 0
  constexpr int V0 = K0 > 5 ? (1 << K0) : 32;   // floats per lane in phase 0
  constexpr int G0 = V0 / 4;                    // granules per lane in phase 0 (XOR on the low 3 bits)
  constexpr uint32_t M0 = K0 > 2 ? ((1u << (K0 - 2)) - 1u) & 7u : 0u;  // transformed XOR-ed granule bits
  static_assert(TILE_BYTES % (4 * V0) == 0 && (N < 32 || TILE_BYTES % (4 * N) == 0), "tile layout");

  extern __shared__ __align__(1024) uint8_t smem[];
  SchedCtl* ctl = reinterpret_cast<SchedCtl*>(smem + STAGES * TILE_BYTES);
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + STAGES * TILE_BYTES + sizeof(SchedCtl));
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

  auto tile_bytes = [&](int64_t t) -> int {
    const int64_t left = total_bytes - t * TILE_BYTES;
    return int(left < TILE_BYTES ? left : TILE_BYTES);
  };

  pdl_launch_dependents();
  if (warp == NT) {
    // ---------------- producer (as fwht_small_kernel): 1-D bulk loads / stores
    if (lane == 0) {
      pdl_wait();
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
      auto load = [&](int st, int64_t t) {
        const uint32_t b16 = uint32_t(tile_bytes(t)) & ~15u;
        mbar_arrive_expect_tx(&full[st], b16);
        if (b16) bulk_g2s(smem + st * TILE_BYTES, reinterpret_cast<const uint8_t*>(in) + t * TILE_BYTES, b16, &full[st], pol);
      };
      bool ended = false;
      for (int k = 0; k < STAGES; ++k) {
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
        if (b16) bulk_s2g(reinterpret_cast<uint8_t*>(out) + t * TILE_BYTES, smem + s * TILE_BYTES, b16);
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
        bulk_wait_read<0>();
        load(s, tile);
        tile = advance(tile);
      }
      bulk_wait_all();
    }
    return;
  }

  // ---------------- consumers
  const int tid = threadIdx.x;  // 0 .. NT*32-1
  const uint32_t c = uint32_t(lane) & 7u;
  float al[3];  // phase-0 granule-bit butterfly signs (alpha), only transformed bits flip
#pragma unroll
  for (int b = 0; b < 3; ++b) al[b] = (((c & M0) >> b) & 1u) ? -1.f : 1.f;

  for (int it = 0;; ++it) {
    const int s = it % STAGES;
    mbar_wait(&full[s], (it / STAGES) & 1);
    const int64_t tile = ctl->stage_tile[s];
    if (tile < 0) break;
    float* const tb = reinterpret_cast<float*>(smem + s * TILE_BYTES);
    const int bytes = tile_bytes(tile);
    const int b16 = bytes & ~15;

    // ---- phase 0: bits 0 .. K0-1 on V0 contiguous floats per lane
    const int items = (bytes + 4 * V0 - 1) / (4 * V0);
    for (int item = tid; item < items; item += NT * 32) {
      float v[V0];
#pragma unroll
      for (int j = 0; j < G0; ++j) {
        const int gi = item * G0 + int(uint32_t(j) ^ c);
        float4 w;
        if (N >= 32 || 16 * gi + 16 <= b16) {
          w = *reinterpret_cast<const float4*>(tb + 4 * gi);
        } else if (16 * gi < bytes) {  // partial granule (n = 2, odd m): the valid 8 bytes from global
          const float* g = reinterpret_cast<const float*>(reinterpret_cast<const uint8_t*>(in) + tile * TILE_BYTES) + 4 * gi;
          w = make_float4(g[0], g[1], 0.f, 0.f);
        } else {
          w = make_float4(0.f, 0.f, 0.f, 0.f);
        }
        v[4 * j] = w.x;
        v[4 * j + 1] = w.y;
        v[4 * j + 2] = w.z;
        v[4 * j + 3] = w.w;
      }
#pragma unroll
      for (int b = 0; b < (K0 < 2 ? K0 : 2); ++b)  // element bits inside a granule
#pragma unroll
        for (int e = 0; e < V0; ++e)
          if (!(e & (1 << b))) {
            const float p0 = v[e], p1 = v[e | (1 << b)];
            v[e] = p0 + p1;
            v[e | (1 << b)] = p0 - p1;
          }
#pragma unroll
      for (int b = 0; b < K0 - 2; ++b)  // granule bits, sign-folded where XOR-ed (see header)
#pragma unroll
        for (int e = 0; e < V0; ++e)
          if (!(e & (4 << b))) {
            const float p0 = v[e], p1 = v[e | (4 << b)];
            const float a = b < 3 ? al[b < 3 ? b : 0] : 1.f;
            v[e] = fmaf(p0, a, p1);
            v[e | (4 << b)] = fmaf(p1, -a, p0);
          }
      if constexpr (NPH == 1) {
#pragma unroll
        for (int e = 0; e < V0; ++e) v[e] *= scale;
      }
#pragma unroll
      for (int j = 0; j < G0; ++j) {
        const int gi = item * G0 + int(uint32_t(j) ^ c);
        const float4 w = make_float4(v[4 * j], v[4 * j + 1], v[4 * j + 2], v[4 * j + 3]);
        if (N >= 32 || 16 * gi + 16 <= b16) {
          *reinterpret_cast<float4*>(tb + 4 * gi) = w;
        } else if (16 * gi < bytes) {
          float* g = reinterpret_cast<float*>(reinterpret_cast<uint8_t*>(out) + tile * TILE_BYTES) + 4 * gi;
          g[0] = w.x;
          g[1] = w.y;
        }
      }
    }

    // ---- phases 1..NPH-1: bits LO .. LO+W-1 (F32Plan), columns of 2^W floats at stride 2^LO
    if constexpr (NPH > 1) {
      const int rows = bytes / (4 * N);
      named_bar_sync(1, NT * 32);
      f32_phase<N, PL::B0, PL::W1, NPH == 2, NT>(tb, rows, tid, scale);
      if constexpr (NPH > 2) {
        named_bar_sync(1, NT * 32);
        f32_phase<N, PL::LO2, PL::W2, true, NT>(tb, rows, tid, scale);
      }
    }
    fence_proxy_async_smem();
    __syncwarp();
    if (lane == 0) mbar_arrive(&done[s]);
  }
}

// ---------------------------------------------------------------- n = 2^15, 2-CTA clusters
// A 128 KiB fp32 row does not fit a double-buffered ring in one CTA, so a CLUSTER of two
// CTAs owns a row: CTA rank h holds half h (64 KiB) in its own ring and applies
// H_2^14 to it (phases 0-2 of fwht_f32_fast_kernel); the last factor, H_2 over the top
// index bit, needs both halves: every consumer thread reads the partner's elements
// at half of the positions through distributed shared memory (mapa +
// ld.shared::cluster; 32 KiB per CTA and tile) and computes both scale * (a + b) and
// scale * (a - b) there; each CTA stores its two 32 KiB output pieces.  Two mbarriers
// per stage order the exchange: ready[s] (the partner's half is final) and
// consumed[s] (the partner has read this CTA's half, so it may be overwritten), each
// armed by ONE remote mbarrier.arrive.release.cluster from the partner's group after
// a group barrier.  Rows are scheduled
// statically (row = cluster id + k * clusters), identically in both CTAs.  The
// consumer warps form G groups that take alternate tiles, so one group's exchange
// (two cross-SM handshakes and the DSMEM reads) overlaps the other's butterflies.
__device__ __forceinline__ uint32_t mapa_shared(uint32_t addr, uint32_t rank) {
  uint32_t r;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(addr), "r"(rank));
  return r;
}
__device__ __forceinline__ uint32_t cluster_ctarank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}
__device__ __forceinline__ void cluster_sync_all() {  // non-.aligned: callable from diverged warps
  asm volatile("barrier.cluster.arrive.release;\n\tbarrier.cluster.wait.acquire;" ::: "memory");
}
__device__ __forceinline__ void mbar_arrive_remote(uint32_t cluster_addr) {
  asm volatile("mbarrier.arrive.release.cluster.shared::cluster.b64 _, [%0];" ::"r"(cluster_addr) : "memory");
}
__device__ __forceinline__ void mbar_wait_cluster(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n\t.reg .pred p;\n"
      "WAITCL_%=:\n\t"
      "mbarrier.try_wait.parity.acquire.cluster.shared::cta.b64 p, [%0], %1;\n\t"
      "@!p bra WAITCL_%=;\n}" ::"r"(smem_addr(bar)),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ float4 ld_cluster_f4(uint32_t cluster_addr) {
  float4 v;
  asm volatile("ld.shared::cluster.v4.f32 {%0, %1, %2, %3}, [%4];"
               : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w)
               : "r"(cluster_addr)
               : "memory");
  return v;
}

template <int STAGES, int NT, int G>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__((NT + 1) * 32, 1)
    fwht_f32_pair_kernel(const float* __restrict__ in, float* __restrict__ out, int64_t m, float scale) {
  constexpr int NH = 16384;                 // elements per half row (per CTA)
  constexpr int TILE_BYTES = NH * 4;        // 64 KiB
  constexpr int K = 14;
  constexpr int NTG = NT / G;               // consumer warps per group; group g takes tiles it = g mod G
  constexpr int PER_THREAD = NH / 8 / (NTG * 32);  // float4 positions of the final factor per consumer thread
  // G <= STAGES: a group never waits on a stage barrier two phases ahead of its
  // current phase (parity waits cannot tell those apart)
  static_assert(NT % G == 0 && G <= STAGES, "groups");
  static_assert(PER_THREAD * NTG * 32 * 8 == NH, "the final factor's positions split evenly over a group");
  extern __shared__ __align__(1024) uint8_t smem[];
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + STAGES * TILE_BYTES);
  uint64_t* done = full + STAGES;
  uint64_t* ready = done + STAGES;
  uint64_t* consumed = ready + STAGES;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint32_t rank = cluster_ctarank(), peer = rank ^ 1u;
  const int64_t cid = blockIdx.x >> 1, nclusters = gridDim.x >> 1;

  if (threadIdx.x == 0) {
#pragma unroll
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&done[s], NTG);
      mbar_init(&ready[s], 1);
      mbar_init(&consumed[s], 1);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    fence_proxy_async_smem();
  }
  cluster_sync_all();  // both CTAs' barriers exist before any remote arrival
  pdl_launch_dependents();

  if (warp == NT) {
    if (lane == 0) {
      pdl_wait();
      const uint64_t pol = policy_evict_first();
      auto src = [&](int64_t r) { return reinterpret_cast<const uint8_t*>(in + r * 2 * NH + rank * NH); };
      int64_t r_load = cid;
      for (int k = 0; k < STAGES && r_load < m; ++k, r_load += nclusters) {
        mbar_arrive_expect_tx(&full[k], TILE_BYTES);
        bulk_g2s(smem + k * TILE_BYTES, src(r_load), TILE_BYTES, &full[k], pol);
      }
      int it = 0;
      for (int64_t r = cid; r < m; r += nclusters, ++it) {
        const int s = it % STAGES;
        mbar_wait(&done[s], (it / STAGES) & 1);
        jitter(1, it);
        // smem [0, NH/2) = y_lo at this CTA's positions, [NH/2, NH) = y_hi at them
        bulk_s2g(out + r * 2 * NH + rank * (NH / 2), smem + s * TILE_BYTES, TILE_BYTES / 2);
        bulk_s2g(out + r * 2 * NH + NH + rank * (NH / 2), smem + s * TILE_BYTES + TILE_BYTES / 2, TILE_BYTES / 2);
        bulk_commit();
        if (r_load < m) {
          bulk_wait_read<0>();
          jitter(2, it);
          mbar_arrive_expect_tx(&full[s], TILE_BYTES);
          bulk_g2s(smem + s * TILE_BYTES, src(r_load), TILE_BYTES, &full[s], pol);
          r_load += nclusters;
        }
      }
      bulk_wait_all();
    }
  } else {
    const int grp = warp / NTG, tid = threadIdx.x - grp * NTG * 32;
    const uint32_t c = uint32_t(lane) & 7u;
    float al[3];
#pragma unroll
    for (int b = 0; b < 3; ++b) al[b] = ((c >> b) & 1u) ? -1.f : 1.f;
    for (int it = grp;; it += G) {
      const int64_t r = cid + int64_t(it) * nclusters;
      if (r >= m) break;
      const int s = it % STAGES;
      const uint32_t ph = (it / STAGES) & 1;
      mbar_wait(&full[s], ph);
      float* const tb = reinterpret_cast<float*>(smem + s * TILE_BYTES);
      // phase 0: bits 0..4, 32 contiguous floats per lane (sign-folded granule butterflies)
      for (int item = tid; item < NH / 32; item += NTG * 32) {
        float v[32];
#pragma unroll
        for (int j = 0; j < 8; ++j) {
          const float4 w = *reinterpret_cast<const float4*>(tb + 4 * (item * 8 + int(uint32_t(j) ^ c)));
          v[4 * j] = w.x;
          v[4 * j + 1] = w.y;
          v[4 * j + 2] = w.z;
          v[4 * j + 3] = w.w;
        }
#pragma unroll
        for (int b = 0; b < 2; ++b)
#pragma unroll
          for (int e = 0; e < 32; ++e)
            if (!(e & (1 << b))) {
              const float p0 = v[e], p1 = v[e | (1 << b)];
              v[e] = p0 + p1;
              v[e | (1 << b)] = p0 - p1;
            }
#pragma unroll
        for (int b = 0; b < 3; ++b)
#pragma unroll
          for (int e = 0; e < 32; ++e)
            if (!(e & (4 << b))) {
              const float p0 = v[e], p1 = v[e | (4 << b)];
              v[e] = fmaf(p0, al[b], p1);
              v[e | (4 << b)] = fmaf(p1, -al[b], p0);
            }
#pragma unroll
        for (int j = 0; j < 8; ++j)
          *reinterpret_cast<float4*>(tb + 4 * (item * 8 + int(uint32_t(j) ^ c))) =
              make_float4(v[4 * j], v[4 * j + 1], v[4 * j + 2], v[4 * j + 3]);
      }
      named_bar_sync(1 + grp, NTG * 32);
      f32_phase<NH, 5, 5, false, NTG>(tb, 1, tid, 1.f);
      named_bar_sync(1 + grp, NTG * 32);
      f32_phase<NH, 10, 4, false, NTG>(tb, 1, tid, 1.f);  // the last in-CTA phase (scale applied below)
      static_assert(K == 14, "half rows of 2^14");
      // this group's half is final (group barrier); one thread tells the partner with a
      // release at cluster scope, cumulative over the group's writes it synchronized with
      const uint32_t tb_addr = smem_addr(tb);
      named_bar_sync(1 + grp, NTG * 32);
      if (tid == 0) {
        jitter(3, it);
        mbar_arrive_remote(mapa_shared(smem_addr(&ready[s]), peer));
      }
      mbar_wait_cluster(&ready[s], ph);  // the partner's half is final
      jitter(4, it);
      // positions [rank * NH/2, (rank+1) * NH/2) of both halves are this CTA's: it reads
      // the partner's half only there (32 KiB over DSMEM), and produces both outputs
      // y_lo = a + b and y_hi = a - b for them
      float4 own[PER_THREAD], pb[PER_THREAD];
      const uint32_t peer_tb = mapa_shared(tb_addr, peer);
      const int q0 = int(rank) * (NH / 8);  // first float4 of this CTA's positions
#pragma unroll
      for (int k2 = 0; k2 < PER_THREAD; ++k2)
#ifdef HC_PAIR_NODSMEM  // diagnostic (wrong results): local reads instead of the partner's
        pb[k2] = *reinterpret_cast<const float4*>(tb + 4 * (q0 + tid + k2 * NTG * 32) + 1);
#else
        pb[k2] = ld_cluster_f4(peer_tb + 16u * uint32_t(q0 + tid + k2 * NTG * 32));
#endif
#pragma unroll
      for (int k2 = 0; k2 < PER_THREAD; ++k2) own[k2] = *reinterpret_cast<const float4*>(tb + 4 * (q0 + tid + k2 * NTG * 32));
      named_bar_sync(1 + grp, NTG * 32);  // the whole group has read the partner's half
      if (tid == 0) {
        jitter(5, it);
        mbar_arrive_remote(mapa_shared(smem_addr(&consumed[s]), peer));
      }
      mbar_wait_cluster(&consumed[s], ph);  // the partner is done reading ours
#pragma unroll
      for (int k2 = 0; k2 < PER_THREAD; ++k2) {
        // rank 0 holds the low half (own = a, partner = b); rank 1 the high half (own = b)
        const float4 a = rank == 0 ? own[k2] : pb[k2];
        const float4 b = rank == 0 ? pb[k2] : own[k2];
        const int e4 = tid + k2 * NTG * 32;
        *reinterpret_cast<float4*>(tb + 4 * e4) =
            make_float4((a.x + b.x) * scale, (a.y + b.y) * scale, (a.z + b.z) * scale, (a.w + b.w) * scale);
        *reinterpret_cast<float4*>(tb + 4 * (NH / 8 + e4)) =
            make_float4((a.x - b.x) * scale, (a.y - b.y) * scale, (a.z - b.z) * scale, (a.w - b.w) * scale);
      }
      fence_proxy_async_smem();
      __syncwarp();
      if (lane == 0) mbar_arrive(&done[s]);
    }
  }
  __syncwarp();
  cluster_sync_all();  // no CTA leaves while its partner may still touch its shared memory
}

// ---------------------------------------------------------------- n = 2^15, top bit first
// (round 2; VERDICT r1 "fp32 at n = 2^15": the pair kernel above exchanges the halves AFTER
// they are transformed, a synchronous cross-SM handshake per row that left 23 % of its stall
// samples waiting on the partner).  The factors of H_2^15 = (H_2 (x) I) (I (x) H_2^14)
// commute, so the top-bit butterfly can come FIRST: CTA h of a 2-CTA cluster
// computes u_h = x_lo + (1 - 2h) x_hi and then y_h = scale * H_2^14 u_h, the output half h.
// Each CTA needs both input halves: CTA h loads 16 KiB pieces of half h with a MULTICAST bulk
// copy that lands in both CTAs' shared memory (HBM and L2 read each byte once), so the only
// cross-CTA traffic is the input itself, pipelined through an S-slot ring; a slot is refilled
// when the consumers of BOTH CTAs have released it (an empty mbarrier with one local and one
// remote arrival per use) -- an asynchronous, ring-deep dependency instead of a per-row
// handshake.  The combine u = x_lo +- x_hi is fused into phase 0 (bits 0..4); phases 1, 2
// (bits 5..9, 10..13, scale applied in the last) run on the CTA's 64 KiB row buffer as in
// fwht_f32_fast_kernel; then one bulk store of y_h.  One consumer group consumes the pieces
// strictly in sequence (two groups sharing the slots could wait on a slot two fills ahead,
// which a parity wait cannot tell apart -- the first version hung); rows alternate two 64 KiB
// row buffers so a row's store overlaps the next row's combine.  Smem: NRB x 64 KiB + S x 32 KiB.
// MEASURED SLOWER than the pair kernel (HC_F32_MC builds: 3.57 TB/s with 3 slots and two row
// buffers, 3.2 with 4-5 slots and one, vs 4.78; profiles/r02_f32_mc_ab.txt): the shared-memory
// budget leaves less than one row of input in flight (3 x 16 KiB of a CTA's own half), so each
// row's last piece is loaded only once the combine has started, and the two CTAs advance in
// lockstep through the shared slots.  Kept as a build option for the record.
__device__ __forceinline__ void bulk_g2s_mc2(void* dst, const void* src, uint32_t bytes, uint64_t* bar,
                                             uint64_t policy) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.multicast::cluster.L2::cache_hint"
      " [%0], [%1], %2, [%3], %4, %5;" ::"r"(smem_addr(dst)),
      "l"(src), "r"(bytes), "r"(smem_addr(bar)), "h"(uint16_t(3)), "l"(policy)
      : "memory");
}

template <int S, int NT, int NRB>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__((NT + 1) * 32, 1)
    fwht_f32_mc_kernel(const float* __restrict__ in, float* __restrict__ out, int64_t m, float scale) {
  constexpr int NH = 16384;                 // elements per half row (per CTA)
  constexpr int PIECE = 4096;               // floats per multicast piece (16 KiB)
  constexpr int NPIECE = NH / PIECE;        // pieces per half row
  constexpr int ROWBUF = NH * 4;            // 64 KiB
  constexpr int SLOT = 2 * PIECE * 4;       // lo piece + hi piece, 32 KiB
  constexpr int PAR = NT * 32 / (PIECE / 32);  // pieces combined at once (one 32-float item per thread)
  static_assert(PAR >= 1 && NPIECE % PAR == 0 && PAR * (PIECE / 32) == NT * 32, "item split");
  static_assert(S >= PAR, "slots");
  extern __shared__ __align__(1024) uint8_t smem[];
  uint8_t* const slots = smem + NRB * ROWBUF;
  uint64_t* full = reinterpret_cast<uint64_t*>(slots + S * SLOT);
  uint64_t* empty = full + S;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint32_t rank = cluster_ctarank(), peer = rank ^ 1u;
  const int64_t cid = blockIdx.x >> 1, nclusters = gridDim.x >> 1;

  if (threadIdx.x == 0) {
#pragma unroll
    for (int k = 0; k < S; ++k) {
      mbar_init(&full[k], 1);
      mbar_init(&empty[k], 2);  // this CTA's consumers + the partner's
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    fence_proxy_async_smem();
  }
  cluster_sync_all();  // both CTAs' barriers exist before any multicast or remote arrival
  pdl_launch_dependents();

  if (warp == NT) {
    // ---------------- producer: this CTA's half of every piece, multicast to both CTAs
    if (lane == 0) {
      pdl_wait();
      const uint64_t pol = policy_evict_first();
      int u = 0;  // piece sequence number (both CTAs walk the same sequence)
      for (int64_t r = cid; r < m; r += nclusters) {
#pragma unroll 1
        for (int p = 0; p < NPIECE; ++p, ++u) {
          const int k = u % S;
          mbar_wait_cluster(&empty[k], ((u / S) & 1) ^ 1);  // both CTAs have released slot k
          jitter(6, u);
          mbar_arrive_expect_tx(&full[k], SLOT);            // own half + the partner's
          bulk_g2s_mc2(slots + k * SLOT + rank * (SLOT / 2), in + r * 2 * NH + int64_t(rank) * NH + p * PIECE,
                       SLOT / 2, &full[k], pol);
        }
      }
    }
  } else {
    // ---------------- consumers (one group, pieces consumed strictly in sequence, so a
    // parity wait is never two phases ahead of its slot); rows alternate two row buffers
    const int tid = threadIdx.x, half = tid / (PIECE / 32), item = tid % (PIECE / 32);
    const uint32_t c = uint32_t(lane) & 7u;
    float al[3];
#pragma unroll
    for (int b = 0; b < 3; ++b) al[b] = ((c >> b) & 1u) ? -1.f : 1.f;
    const float hs = rank == 0 ? 1.f : -1.f;  // u_h = x_lo + hs * x_hi
    int rows = 0;
    for (int64_t r = cid; r < m; r += nclusters, ++rows) {
      float* const rb = reinterpret_cast<float*>(smem + (rows % NRB) * ROWBUF);
      if (rows >= NRB) {  // the store of NRB rows ago (same buffer) has read it
        if (tid == 0) bulk_wait_read<NRB - 1>();
        named_bar_sync(1, NT * 32);
      }
      // combine (top bit) + phase 0 (bits 0..4): PAR pieces at once, 32 floats per thread
#pragma unroll 1
      for (int p0 = 0; p0 < NPIECE; p0 += PAR) {
        const int p = p0 + half, u = rows * NPIECE + p, ks = u % S;
        mbar_wait(&full[ks], (u / S) & 1);
        const float* lo = reinterpret_cast<const float*>(slots + ks * SLOT);
        const float* hi = lo + PIECE;
        float v[32];
#pragma unroll
        for (int j = 0; j < 8; ++j) {
          const int o = 4 * (item * 8 + int(uint32_t(j) ^ c));
          const float4 a = *reinterpret_cast<const float4*>(lo + o);
          const float4 b = *reinterpret_cast<const float4*>(hi + o);
          v[4 * j] = fmaf(b.x, hs, a.x);
          v[4 * j + 1] = fmaf(b.y, hs, a.y);
          v[4 * j + 2] = fmaf(b.z, hs, a.z);
          v[4 * j + 3] = fmaf(b.w, hs, a.w);
        }
        // the slots are read: release them to both producers
        named_bar_sync(1, NT * 32);
        if (item == 0) {
          jitter(7, u);
          mbar_arrive(&empty[ks]);
          mbar_arrive_remote(mapa_shared(smem_addr(&empty[ks]), peer));
        }
#pragma unroll
        for (int b = 0; b < 2; ++b)
#pragma unroll
          for (int e = 0; e < 32; ++e)
            if (!(e & (1 << b))) {
              const float q0 = v[e], q1 = v[e | (1 << b)];
              v[e] = q0 + q1;
              v[e | (1 << b)] = q0 - q1;
            }
#pragma unroll
        for (int b = 0; b < 3; ++b)
#pragma unroll
          for (int e = 0; e < 32; ++e)
            if (!(e & (4 << b))) {
              const float q0 = v[e], q1 = v[e | (4 << b)];
              v[e] = fmaf(q0, al[b], q1);
              v[e | (4 << b)] = fmaf(q1, -al[b], q0);
            }
        float* const dst = rb + p * PIECE;
#pragma unroll
        for (int j = 0; j < 8; ++j)
          *reinterpret_cast<float4*>(dst + 4 * (item * 8 + int(uint32_t(j) ^ c))) =
              make_float4(v[4 * j], v[4 * j + 1], v[4 * j + 2], v[4 * j + 3]);
      }
      named_bar_sync(1, NT * 32);
      f32_phase<NH, 5, 5, false, NT>(rb, 1, tid, 1.f);
      named_bar_sync(1, NT * 32);
      f32_phase<NH, 10, 4, true, NT>(rb, 1, tid, scale);
      fence_proxy_async_smem();  // the bulk store reads rb through the async proxy
      named_bar_sync(1, NT * 32);
      if (tid == 0) {
        bulk_s2g(out + r * 2 * NH + int64_t(rank) * NH, rb, ROWBUF);
        bulk_commit();
      }
    }
    if (threadIdx.x == 0) bulk_wait_all();
  }
  __syncwarp();
  cluster_sync_all();  // no CTA leaves while its partner may still multicast into it or arrive remotely
}

// ---------------------------------------------------------------- n = 2^15, one CTA, chunk ring
// (round 2; VERDICT r1 "fp32 at n = 2^15", third design).  A row (128 KiB) streams into a
// ring of S chunk slots of CH floats (14 x 16 KiB = 224 KiB), so one row is resident while
// most of the next one is already in flight.  The bits of the index split by where their
// butterflies can run:
//   bits 0..9  lie inside a chunk: consumer group g (GT = CH/32 threads) takes the row's
//              chunks c = g mod NG as they land -- phase 0 (bits 0..4, 32 contiguous floats
//              per lane, sign-folded granule butterflies as fwht_f32_fast_kernel) and phase
//              1 (bits 5..9, 32-float columns at stride 32) -- with only a group barrier;
//   bits 10..14 span the chunks: after a barrier over all consumers, phase 2 takes
//              32-float columns at stride 1024 (value t of column col is element
//              t * 1024 + col, in chunk t * 1024 / CH) straight from the chunk slots,
//              applies `scale` and writes back in place.
// Every element makes the same shared-memory trips as in the n <= 2^14 kernel (TMA in,
// three phases, TMA out).  The producer warp (one thread) loads chunk u (the CTA's u-th,
// rows in order) into slot u mod S and, once the consumers have signalled a row done
// (row_done, NT arrivals), stores its chunks -- one bulk group per chunk, so a slot is
// refilled as soon as ITS store has been read, not the whole row's.  S <= 2 CPR - 1 keeps
// the row_done parity unambiguous: row k+1 cannot finish before row k's store was issued.
// Rows are static (row = blockIdx.x + k * gridDim.x), one CTA per SM.
#ifndef HC_RING_STCS
#define HC_RING_STCS 0
#endif
__device__ __forceinline__ void bulk_wait_read_upto(int pending) {  // wait until <= pending groups read
  switch (pending < 0 ? 0 : pending) {
    case 0: bulk_wait_read<0>(); break;
    case 1: bulk_wait_read<1>(); break;
    case 2: bulk_wait_read<2>(); break;
    case 3: bulk_wait_read<3>(); break;
    case 4: bulk_wait_read<4>(); break;
    case 5: bulk_wait_read<5>(); break;
    case 6: bulk_wait_read<6>(); break;
    default: bulk_wait_read<7>(); break;  // stricter than asked: safe
  }
}

template <int CH, int S, int NT, bool DIRECT>
__global__ void __launch_bounds__((NT + 1) * 32, 1)
    fwht_f32_ring_kernel(const float* __restrict__ in, float* __restrict__ out, int64_t m, float scale) {
  constexpr int N = 32768, CPR = N / CH, CB = CH * 4;
  constexpr int GT = CH / 32;         // threads of a group: one 32-float item / column each
  constexpr int NG = NT * 32 / GT;    // consumer groups
  static_assert(CH >= 1024 && CH % 1024 == 0 && CPR >= 2, "chunks hold whole 1024-float blocks");
  static_assert(NG * GT == NT * 32 && NG >= 1 && CPR % NG == 0 && NG + 1 < 16, "groups");
  static_assert(S >= CPR && S <= 2 * CPR - 1, "ring: one row resident, row_done parity unambiguous");
  constexpr int CPT = 1024 / (NT * 32);  // DIRECT: adjacent columns per thread in the cross-chunk phase
  static_assert(!DIRECT || CPT == 2 || CPT == 4, "DIRECT holds the row in registers: 8 or 16 consumer warps");
  extern __shared__ __align__(1024) uint8_t smem[];
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + S * CB);
  uint64_t* row_done = full + S;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t rows = m > int64_t(blockIdx.x) ? (m - 1 - int64_t(blockIdx.x)) / gridDim.x + 1 : 0;

  if (threadIdx.x == 0) {
#pragma unroll
    for (int s = 0; s < S; ++s) mbar_init(&full[s], 1);
    mbar_init(row_done, NT);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    fence_proxy_async_smem();
  }
  __syncthreads();
  pdl_launch_dependents();

  if (warp == NT) {
    if (lane == 0) {
      pdl_wait();
      const uint64_t pol = policy_evict_first();
      const int64_t total = rows * CPR;
      int64_t stored = 0;  // chunks whose store has been issued (in chunk order) / released (DIRECT)
      auto store_row = [&](int64_t k) {
        mbar_wait(row_done, uint32_t(k & 1));
        jitter(8, uint32_t(k));
        if constexpr (!DIRECT) {
          const int64_t r = int64_t(blockIdx.x) + k * gridDim.x;
#pragma unroll 1
          for (int c = 0; c < CPR; ++c) {
            bulk_s2g(out + r * N + c * CH, smem + int((k * CPR + c) % S) * CB, CB);
            bulk_commit();
          }
        }
        stored += CPR;
      };
      for (int64_t u = 0; u < total; ++u) {
        const int s = int(u % S);
        if (u >= S) {  // slot s held chunk u - S: its row must be done and its store read
          while (stored <= u - S) store_row(stored / CPR);
          if constexpr (!DIRECT) bulk_wait_read_upto(int(stored - (u - S) - 1));
          jitter(9, uint32_t(u));
        }
        const int64_t r = int64_t(blockIdx.x) + (u / CPR) * gridDim.x;
        mbar_arrive_expect_tx(&full[s], CB);
        bulk_g2s(smem + s * CB, in + r * N + (u % CPR) * CH, CB, &full[s], pol);
      }
      if constexpr (!DIRECT) {
        while (stored < total) store_row(stored / CPR);
      }
      bulk_wait_all();
    }
    return;
  }

  // ---------------- consumers
  const int grp = threadIdx.x / GT, gtid = threadIdx.x - grp * GT, tid = threadIdx.x;
  const uint32_t c = uint32_t(lane) & 7u;
  float al[3];
#pragma unroll
  for (int b = 0; b < 3; ++b) al[b] = ((c >> b) & 1u) ? -1.f : 1.f;
  for (int64_t k = 0; k < rows; ++k) {
    // ---- bits 0..9, chunk by chunk as they land
#pragma unroll 1
    for (int cc = grp; cc < CPR; cc += NG) {
      const int64_t u = k * CPR + cc;
      const int s = int(u % S);
      mbar_wait(&full[s], uint32_t((u / S) & 1));
      float* const tb = reinterpret_cast<float*>(smem + s * CB);
      float v[32];
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        const float4 w = *reinterpret_cast<const float4*>(tb + 4 * (gtid * 8 + int(uint32_t(j) ^ c)));
        v[4 * j] = w.x;
        v[4 * j + 1] = w.y;
        v[4 * j + 2] = w.z;
        v[4 * j + 3] = w.w;
      }
#pragma unroll
      for (int b = 0; b < 2; ++b)
#pragma unroll
        for (int e = 0; e < 32; ++e)
          if (!(e & (1 << b))) {
            const float p0 = v[e], p1 = v[e | (1 << b)];
            v[e] = p0 + p1;
            v[e | (1 << b)] = p0 - p1;
          }
#pragma unroll
      for (int b = 0; b < 3; ++b)
#pragma unroll
        for (int e = 0; e < 32; ++e)
          if (!(e & (4 << b))) {
            const float p0 = v[e], p1 = v[e | (4 << b)];
            v[e] = fmaf(p0, al[b], p1);
            v[e | (4 << b)] = fmaf(p1, -al[b], p0);
          }
#pragma unroll
      for (int j = 0; j < 8; ++j)
        *reinterpret_cast<float4*>(tb + 4 * (gtid * 8 + int(uint32_t(j) ^ c))) =
            make_float4(v[4 * j], v[4 * j + 1], v[4 * j + 2], v[4 * j + 3]);
      named_bar_sync(1 + grp, GT);
      f32_phase<CH, 5, 5, false, GT / 32>(tb, 1, gtid, 1.f);
    }
    // ---- bits 10..14 across the row's chunks
    named_bar_sync(1 + NG, NT * 32);
    jitter(10, uint32_t(k));
    uint32_t base[CPR];  // shared address of chunk j's slot
    {
      const int s0 = int((k * CPR) % S);
#pragma unroll
      for (int j = 0; j < CPR; ++j) base[j] = smem_addr(smem + (s0 + j < S ? s0 + j : s0 + j - S) * CB);
    }
    if constexpr (DIRECT) {
      // the whole row into registers (CPT adjacent columns per thread), release the slots
      // at once, then butterflies and vector stores straight to global memory
      float v[32][CPT];
#pragma unroll
      for (int t = 0; t < 32; ++t) {
        const uint32_t a = base[(t * 1024) / CH] + 4u * uint32_t(((t * 1024) % CH) + CPT * tid);
        if constexpr (CPT == 4) {
          asm volatile("ld.shared.v4.f32 {%0, %1, %2, %3}, [%4];"
                       : "=f"(v[t][0]), "=f"(v[t][1]), "=f"(v[t][2]), "=f"(v[t][3])
                       : "r"(a)
                       : "memory");
        } else {
          asm volatile("ld.shared.v2.f32 {%0, %1}, [%2];" : "=f"(v[t][0]), "=f"(v[t][1]) : "r"(a) : "memory");
        }
      }
      __syncwarp();
      if (lane == 0) {
        jitter(11, uint32_t(k));
        mbar_arrive(row_done);  // this warp has read the row: the producer may refill its slots
      }
#pragma unroll
      for (int b = 0; b < 5; ++b)
#pragma unroll
        for (int e = 0; e < 32; ++e)
          if (!(e & (1 << b)))
#pragma unroll
            for (int q = 0; q < CPT; ++q) {
              const float p0 = v[e][q], p1 = v[e | (1 << b)][q];
              v[e][q] = p0 + p1;
              v[e | (1 << b)][q] = p0 - p1;
            }
      float* const orow = out + (int64_t(blockIdx.x) + k * gridDim.x) * N + CPT * tid;
#pragma unroll
      for (int t = 0; t < 32; ++t) {
        if constexpr (CPT == 4) {
          *reinterpret_cast<float4*>(orow + t * 1024) =
              make_float4(v[t][0] * scale, v[t][1] * scale, v[t][2] * scale, v[t][3] * scale);
        } else {
#if HC_RING_STCS
          __stcs(reinterpret_cast<float2*>(orow + t * 1024), make_float2(v[t][0] * scale, v[t][1] * scale));
#else
          *reinterpret_cast<float2*>(orow + t * 1024) = make_float2(v[t][0] * scale, v[t][1] * scale);
#endif
        }
      }
    } else {
#pragma unroll 1
      for (int col = tid; col < 1024; col += NT * 32) {
        float v[32];
#pragma unroll
        for (int t = 0; t < 32; ++t) {
          const uint32_t a = base[(t * 1024) / CH] + 4u * uint32_t(((t * 1024) % CH) + col);
          asm volatile("ld.shared.f32 %0, [%1];" : "=f"(v[t]) : "r"(a) : "memory");
        }
#pragma unroll
        for (int b = 0; b < 5; ++b)
#pragma unroll
          for (int e = 0; e < 32; ++e)
            if (!(e & (1 << b))) {
              const float p0 = v[e], p1 = v[e | (1 << b)];
              v[e] = p0 + p1;
              v[e | (1 << b)] = p0 - p1;
            }
#pragma unroll
        for (int t = 0; t < 32; ++t) {
          const uint32_t a = base[(t * 1024) / CH] + 4u * uint32_t(((t * 1024) % CH) + col);
          asm volatile("st.shared.f32 [%0], %1;" ::"r"(a), "f"(v[t] * scale) : "memory");
        }
      }
      fence_proxy_async_smem();
      __syncwarp();
      if (lane == 0) {
        jitter(11, uint32_t(k));
        mbar_arrive(row_done);
      }
    }
  }
}

// ---------------------------------------------------------------- n = 2^15, one CTA, chunks released early
// (round 2, after fwht_f32_ring_kernel: there a row's slots stay occupied until its last
// chunk has landed and been transformed, so only S - CPR slots of loads are in flight at the
// row boundary).  Here every consumer thread takes part in every chunk: phase 0 and phase 1
// (bits 0..9) on the chunk with CTA-wide barriers, then each thread reads ITS values of the
// cross-chunk phase out of the chunk -- columns 2 tid, 2 tid + 1 at every 1024-block the
// chunk holds -- into registers and the warp releases the slot at once (empty[s], NT
// arrivals).  After the row's last chunk a thread holds 2 complete columns of 32 values:
// bits 10..14 as register butterflies, `scale`, 8-byte stores straight to global memory.
// A slot is thus occupied for one chunk's transform only, and S - 1 chunks of loads stay
// in flight all the time.
#ifndef HC_STREAM_ST128
#define HC_STREAM_ST128 0  // 1: lane-pair swap + 16-byte stores of the results -- measured 6.43 -> 5.90 TB/s, off
#endif
#ifndef HC_F32_STREAM_CLC
#define HC_F32_STREAM_CLC 1  // 0: static round-robin rows over a persistent grid (A/B)
#endif
constexpr bool kStreamClc = kClc && HC_F32_STREAM_CLC != 0;
template <int CH, int S, int NT>
__global__ void __launch_bounds__((NT + 1) * 32, 1)
    fwht_f32_stream_kernel(const float* __restrict__ in, float* __restrict__ out, int64_t m, float scale) {
  constexpr int N = 32768, CPR = N / CH, CB = CH * 4;
  constexpr int TPC = CH / 1024;  // 1024-blocks (values of a cross-chunk column) per chunk
  constexpr int CPT = 1024 / (NT * 32);  // adjacent columns of the cross-chunk phase per thread
  static_assert(CPT == 2 || CPT == 4, "8 or 16 consumer warps");
  static_assert(CH >= 1024 && CH % 1024 == 0 && CPR >= 2 && S >= 2, "chunks");
  extern __shared__ __align__(1024) uint8_t smem[];
  SchedCtl* ctl = reinterpret_cast<SchedCtl*>(smem + S * CB);  // stage_tile[s] = the row of slot s (-1: end)
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + S * CB + sizeof(SchedCtl));
  uint64_t* empty = full + S;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  static_assert(S <= 16, "SchedCtl::stage_tile");

  if (threadIdx.x == 0) {
    mbar_init(&ctl->clc_bar, 1);
#pragma unroll
    for (int s = 0; s < S; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], NT);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    fence_proxy_async_smem();
  }
  __syncthreads();
  pdl_launch_dependents();

  if (warp == NT) {
    // rows: this CTA's own (blockIdx.x), then rows of not-yet-launched CTAs taken over with
    // cluster launch control (kClc; as fwht_f32_fast_kernel), or static round-robin
    if (lane == 0) {
      pdl_wait();
      const uint64_t pol = policy_evict_first();
      uint32_t clc_phase = 0;
      int64_t u = 0;  // chunk sequence number of this CTA
      auto slot = [&](int64_t uu) {
        const int s = int(uu % S);
        if (uu >= S) mbar_wait(&empty[s], uint32_t(((uu / S) - 1) & 1));  // chunk uu - S released
        jitter(12, uint32_t(uu));
        return s;
      };
      for (int64_t row = blockIdx.x;;) {
        if (row < 0 || row >= m) {  // end: the consumers stop at the next slot
          const int s = slot(u);
          ctl->stage_tile[s] = -1;
          mbar_arrive(&full[s]);
          break;
        }
        if constexpr (kStreamClc) clc_request(ctl);
#pragma unroll 1
        for (int c = 0; c < CPR; ++c, ++u) {
          const int s = slot(u);
          ctl->stage_tile[s] = int(row);
          mbar_arrive_expect_tx(&full[s], CB);
          bulk_g2s(smem + s * CB, in + row * N + c * CH, CB, &full[s], pol);
        }
        if constexpr (kStreamClc) {
          row = clc_result(ctl, clc_phase);
        } else {
          row += gridDim.x;
        }
      }
    }
    return;
  }

  const int tid = threadIdx.x;
  const uint32_t c = uint32_t(lane) & 7u;
  float al[3];
#pragma unroll
  for (int b = 0; b < 3; ++b) al[b] = ((c >> b) & 1u) ? -1.f : 1.f;
  for (int k = 0;; ++k) {  // (32-bit chunk counters: at most 2 m chunks per CTA)
    {
      const int u0 = k * CPR;
      mbar_wait(&full[u0 % S], uint32_t((u0 / S) & 1));
    }
    const int row = ctl->stage_tile[(k * CPR) % S];
    if (row < 0) break;
    float v[32][CPT];  // value t of columns CPT tid .. CPT tid + CPT - 1 (element t * 1024 + col)
#pragma unroll
    for (int cc = 0; cc < CPR; ++cc) {
      const int u = k * CPR + cc;
      const int s = u % S;
      if (cc > 0) mbar_wait(&full[s], uint32_t((u / S) & 1));
      float* const tb = reinterpret_cast<float*>(smem + s * CB);
      // phase 0: bits 0..4, 32 contiguous floats per item
#pragma unroll 1
      for (int item = tid; item < CH / 32; item += NT * 32) {
        float w[32];
#pragma unroll
        for (int j = 0; j < 8; ++j) {
          const float4 g = *reinterpret_cast<const float4*>(tb + 4 * (item * 8 + int(uint32_t(j) ^ c)));
          w[4 * j] = g.x;
          w[4 * j + 1] = g.y;
          w[4 * j + 2] = g.z;
          w[4 * j + 3] = g.w;
        }
#pragma unroll
        for (int b = 0; b < 2; ++b)
#pragma unroll
          for (int e = 0; e < 32; ++e)
            if (!(e & (1 << b))) {
              const float p0 = w[e], p1 = w[e | (1 << b)];
              w[e] = p0 + p1;
              w[e | (1 << b)] = p0 - p1;
            }
#pragma unroll
        for (int b = 0; b < 3; ++b)
#pragma unroll
          for (int e = 0; e < 32; ++e)
            if (!(e & (4 << b))) {
              const float p0 = w[e], p1 = w[e | (4 << b)];
              w[e] = fmaf(p0, al[b], p1);
              w[e | (4 << b)] = fmaf(p1, -al[b], p0);
            }
#pragma unroll
        for (int j = 0; j < 8; ++j)
          *reinterpret_cast<float4*>(tb + 4 * (item * 8 + int(uint32_t(j) ^ c))) =
              make_float4(w[4 * j], w[4 * j + 1], w[4 * j + 2], w[4 * j + 3]);
      }
      named_bar_sync(1, NT * 32);
      f32_phase<CH, 5, 5, false, NT>(tb, 1, tid, 1.f);  // phase 1: bits 5..9
      named_bar_sync(1, NT * 32);
      // this thread's values of the cross-chunk phase, then release the slot
#pragma unroll
      for (int j = 0; j < TPC; ++j) {
        if constexpr (CPT == 4) {
          const float4 g = *reinterpret_cast<const float4*>(tb + j * 1024 + 4 * tid);
          v[cc * TPC + j][0] = g.x;
          v[cc * TPC + j][1] = g.y;
          v[cc * TPC + j][2] = g.z;
          v[cc * TPC + j][3] = g.w;
        } else {
          const float2 g = *reinterpret_cast<const float2*>(tb + j * 1024 + 2 * tid);
          v[cc * TPC + j][0] = g.x;
          v[cc * TPC + j][1] = g.y;
        }
      }
      __syncwarp();
      if (lane == 0) {
        jitter(13, uint32_t(u));
        mbar_arrive(&empty[s]);
      }
    }
    // bits 10..14 in registers, scale, stores
#pragma unroll
    for (int b = 0; b < 5; ++b)
#pragma unroll
      for (int e = 0; e < 32; ++e)
        if (!(e & (1 << b)))
#pragma unroll
          for (int q = 0; q < CPT; ++q) {
            const float p0 = v[e][q], p1 = v[e | (1 << b)][q];
            v[e][q] = p0 + p1;
            v[e | (1 << b)][q] = p0 - p1;
          }
    float* const orow = out + int64_t(row) * N + CPT * tid;
    if constexpr (CPT == 2 && HC_STREAM_ST128) {
      // lane pairs swap halves so that each lane stores 4 adjacent columns of every other
      // block: 16 STG.128 per lane instead of 32 STG.64 (fewer entries in the store queue)
      const bool odd = lane & 1;
      float* const orow4 = out + int64_t(row) * N + 4 * (tid >> 1);
#pragma unroll
      for (int t2 = 0; t2 < 16; ++t2) {
        const float s0 = odd ? v[2 * t2][0] : v[2 * t2 + 1][0], s1 = odd ? v[2 * t2][1] : v[2 * t2 + 1][1];
        const float m0 = odd ? v[2 * t2 + 1][0] : v[2 * t2][0], m1 = odd ? v[2 * t2 + 1][1] : v[2 * t2][1];
        const float r0 = __shfl_xor_sync(0xffffffffu, s0, 1), r1 = __shfl_xor_sync(0xffffffffu, s1, 1);
        const float4 o = odd ? make_float4(r0 * scale, r1 * scale, m0 * scale, m1 * scale)
                             : make_float4(m0 * scale, m1 * scale, r0 * scale, r1 * scale);
        *reinterpret_cast<float4*>(orow4 + (2 * t2 + (odd ? 1 : 0)) * 1024) = o;
      }
    } else
#pragma unroll
    for (int t = 0; t < 32; ++t)
      if constexpr (CPT == 4) {
        *reinterpret_cast<float4*>(orow + t * 1024) =
            make_float4(v[t][0] * scale, v[t][1] * scale, v[t][2] * scale, v[t][3] * scale);
      } else {
        *reinterpret_cast<float2*>(orow + t * 1024) = make_float2(v[t][0] * scale, v[t][1] * scale);
      }
  }
}

// n = 2^15 in fp32, second pass: rows are [a | b] with a, b = H_2^14-transformed halves;
// out = scale * [a + b | a - b] (the remaining H_2 factor over the top index bit).
__global__ void f32_half_butterfly_kernel(const float* __restrict__ in, float* __restrict__ out, int64_t m,
                                          float scale) {
  constexpr int64_t H = 16384 / 4;  // float4 per half row
  const int64_t total = m * H;
  const int64_t stride = int64_t(gridDim.x) * blockDim.x;
  pdl_launch_dependents();
  pdl_wait();
  for (int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < total; i += stride) {
    const int64_t r = i / H, j = i - r * H;
    const float4 a = reinterpret_cast<const float4*>(in)[r * 2 * H + j];
    const float4 b = reinterpret_cast<const float4*>(in)[r * 2 * H + H + j];
    reinterpret_cast<float4*>(out)[r * 2 * H + j] =
        make_float4((a.x + b.x) * scale, (a.y + b.y) * scale, (a.z + b.z) * scale, (a.w + b.w) * scale);
    reinterpret_cast<float4*>(out)[r * 2 * H + H + j] =
        make_float4((a.x - b.x) * scale, (a.y - b.y) * scale, (a.z - b.z) * scale, (a.w - b.w) * scale);
  }
}

}  // namespace hadacore
