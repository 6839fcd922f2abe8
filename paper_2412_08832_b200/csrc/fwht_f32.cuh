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
// `scale`.  Rows of n = 2^15 (128 KiB of fp32) do not fit a double-buffered ring:
// they are transformed as two rows of 2^14 by this kernel and finished by
// f32_half_butterfly_kernel (H_2 (x) I across the halves).
#pragma once
#include "fwht_small.cuh"

namespace hadacore {

// Phase P >= 1 of the fp32 kernel on a tile of `rows` whole rows in shared memory:
// bits 5P .. 5P+w-1 (w <= 5) over columns of CW = 2^w floats at stride 2^(5P); a lane
// takes CPL = 32 / CW columns per iteration (NT*32 apart, so a warp's accesses are
// 32 consecutive words); the last phase multiplies by `scale`.
template <int N, int P, int NT>
__device__ __forceinline__ void f32_phase(float* tb, int rows, int tid, float scale) {
  constexpr int K = log2_n<N>();
  constexpr int NPH = (K + 4) / 5;
  constexpr int LO = 5 * P;
  constexpr int W = (K - LO) < 5 ? (K - LO) : 5;
  constexpr int CW = 1 << W, CPL = 32 / CW, LPR = K - W;
  const int cols = rows << LPR;
  for (int q0 = tid; q0 < cols; q0 += NT * 32 * CPL) {
    float v[32];
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
      for (int e = 0; e < 32; ++e)
        if (!(e & (1 << b))) {
          const float p0 = v[e], p1 = v[e | (1 << b)];
          v[e] = p0 + p1;
          v[e | (1 << b)] = p0 - p1;
        }
    if constexpr (P == NPH - 1) {
#pragma unroll
      for (int e = 0; e < 32; ++e) v[e] *= scale;
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
  constexpr int NPH = (K + 4) / 5;              // phases of <= 5 bits
  constexpr int K0 = K < 5 ? K : 5;             // bits of phase 0
  constexpr uint32_t M0 = K0 > 2 ? ((1u << (K0 - 2)) - 1u) : 0u;  // transformed granule bits of phase 0
  static_assert(TILE_BYTES % 128 == 0 && (N < 32 || TILE_BYTES % (4 * N) == 0), "tile layout");

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

    // ---- phase 0: bits 0 .. K0-1 on 32 contiguous floats per lane
    const int items = (bytes + 127) / 128;
    for (int item = tid; item < items; item += NT * 32) {
      float v[32];
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        const int gi = item * 8 + int(uint32_t(j) ^ c);
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
        for (int e = 0; e < 32; ++e)
          if (!(e & (1 << b))) {
            const float p0 = v[e], p1 = v[e | (1 << b)];
            v[e] = p0 + p1;
            v[e | (1 << b)] = p0 - p1;
          }
#pragma unroll
      for (int b = 0; b < K0 - 2; ++b)  // granule bits, sign-folded (see header)
#pragma unroll
        for (int e = 0; e < 32; ++e)
          if (!(e & (4 << b))) {
            const float p0 = v[e], p1 = v[e | (4 << b)];
            v[e] = fmaf(p0, al[b], p1);
            v[e | (4 << b)] = fmaf(p1, -al[b], p0);
          }
      if constexpr (NPH == 1) {
#pragma unroll
        for (int e = 0; e < 32; ++e) v[e] *= scale;
      }
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        const int gi = item * 8 + int(uint32_t(j) ^ c);
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

    // ---- phases 1..NPH-1: bits 5p .. 5p+w-1, columns of 2^w floats at stride 2^(5p)
    if constexpr (NPH > 1) {
      const int rows = bytes / (4 * N);
      named_bar_sync(1, NT * 32);
      f32_phase<N, 1, NT>(tb, rows, tid, scale);
      if constexpr (NPH > 2) {
        named_bar_sync(1, NT * 32);
        f32_phase<N, 2, NT>(tb, rows, tid, scale);
      }
    }
    fence_proxy_async_smem();
    __syncwarp();
    if (lane == 0) mbar_arrive(&done[s]);
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
