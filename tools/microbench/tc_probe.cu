// tcgen05 probe (round 2): validates the smem-descriptor / instruction-descriptor / TMEM
// conventions the fused-quantization kernel relies on, on one 128 x 128 x 128 problem:
//   D[m][n] = sum_k X[m][k] * H[n][k]      (A = X, B = H, both K-major, 128B-swizzled)
// with X random fp16/bf16 and H = the 128 x 128 Sylvester matrix (+-1), D fp32 in TMEM,
// read back with tcgen05.ld.32x32b.x32 (thread = TMEM lane = row m).  Also times
// back-to-back MMAs of the shape the kernel issues (M = 128, N = 128, K = 16).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tc_probe tc_probe.cu && ./tc_probe
#include <cuda_bf16.h>
#include <cuda_fp16.h>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cmath>
#include <vector>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("CUDA %s at %d\n", cudaGetErrorString(e), __LINE__); exit(1); } } while (0)

__device__ __forceinline__ uint32_t sa(const void* p) { return uint32_t(__cvta_generic_to_shared(p)); }

// byte offset of element (row, k) of a K-major SW128 operand with K = 128 (two 64-element atoms)
__host__ __device__ inline uint32_t sw_off(int row, int k) {
  const int atom = k >> 6, g = (k & 63) >> 3;
  return atom * 16384 + row * 128 + ((g ^ (row & 7)) << 4) + (k & 7) * 2;
}

__device__ __forceinline__ uint64_t sdesc(uint32_t addr) {
  uint64_t d = 0;
  d |= uint64_t((addr >> 4) & 0x3FFF);
  d |= uint64_t(1) << 16;            // LBO (ignored for swizzled K-major)
  d |= uint64_t(1024 >> 4) << 32;    // SBO: 8 rows x 128 B
  d |= uint64_t(1) << 46;            // version (sm_100)
  d |= uint64_t(2) << 61;            // SWIZZLE_128B
  return d;
}

template <bool BF>
__host__ __device__ constexpr uint32_t idesc(int M, int N) {
  return (1u << 4) | ((BF ? 1u : 0u) << 7) | ((BF ? 1u : 0u) << 10) | (uint32_t(N >> 3) << 17) |
         (uint32_t(M >> 4) << 24);
}

template <bool BF, int MM = 128, int LANE_OFF = 0>
__global__ void __launch_bounds__(128) probe(const uint16_t* X, const uint16_t* H, float* D, int reps,
                                             long long* cycles) {
  extern __shared__ __align__(1024) uint8_t smem[];
  uint8_t* As = smem;
  uint8_t* Bs = smem + 32768;
  __shared__ uint64_t bar;
  __shared__ uint32_t tbase;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  for (int i = tid; i < 128 * 128; i += 128) {
    const int r = i >> 7, k = i & 127;
    *reinterpret_cast<uint16_t*>(As + sw_off(r, k)) = X[i];
    *reinterpret_cast<uint16_t*>(Bs + sw_off(r, k)) = H[i];
  }
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  if (tid == 0) {
    asm volatile("mbarrier.init.shared.b64 [%0], 1;" ::"r"(sa(&bar)));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 128;" ::"r"(sa(&tbase)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tmem = tbase;
  constexpr uint32_t ID = idesc<BF>(MM, 128);
  long long t0 = 0, t1 = 0;
  if (tid == 0) {
    t0 = clock64();
    for (int rep = 0; rep < reps; ++rep) {
#pragma unroll
      for (int kk = 0; kk < 8; ++kk) {
        const uint32_t off = (kk >> 2) * 16384 + (kk & 3) * 32;
        const uint64_t ad = sdesc(sa(As) + off), bd = sdesc(sa(Bs) + off);
        const uint32_t acc = kk > 0 ? 1u : 0u;
        asm volatile(
            "{.reg .pred p; setp.ne.b32 p, %4, 0;\n"
            "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;}" ::"r"(tmem + (uint32_t(LANE_OFF) << 16)),
            "l"(ad), "l"(bd), "r"(ID), "r"(acc));
      }
    }
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(sa(&bar))
                 : "memory");
  }
  // wait for the MMAs
  asm volatile(
      "{.reg .pred P1; LAB_WAIT: mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], 0; @P1 bra DONE; bra LAB_WAIT; "
      "DONE: }" ::"r"(sa(&bar)));
  if (tid == 0) {
    t1 = clock64();
    cycles[0] = t1 - t0;
  }
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  // warp w reads TMEM lanes 32w..32w+31 (rows m), 32 columns at a time
  for (int c0 = 0; c0 < 128; c0 += 32) {
    uint32_t v[32];
    const uint32_t addr = tmem + (uint32_t(32 * warp) << 16) + c0;
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
        "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
        : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]),
          "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]),
          "=r"(v[15]), "=r"(v[16]), "=r"(v[17]), "=r"(v[18]), "=r"(v[19]), "=r"(v[20]), "=r"(v[21]),
          "=r"(v[22]), "=r"(v[23]), "=r"(v[24]), "=r"(v[25]), "=r"(v[26]), "=r"(v[27]), "=r"(v[28]),
          "=r"(v[29]), "=r"(v[30]), "=r"(v[31])
        : "r"(addr));
    asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
    for (int j = 0; j < 32; ++j) D[(32 * warp + lane) * 128 + c0 + j] = __uint_as_float(v[j]);
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 128;" ::"r"(tmem));
}

template <bool BF>
int run() {
  const int M = 128, K = 128;
  std::vector<uint16_t> X(M * K), H(M * K);
  std::vector<float> Xf(M * K), Hf(M * K);
  srand(1234);
  for (int i = 0; i < M * K; ++i) {
    float v = float(rand() % 2001 - 1000) / 256.f;
    if (BF) {
      __nv_bfloat16 b = __float2bfloat16(v);
      X[i] = *reinterpret_cast<uint16_t*>(&b);
      Xf[i] = __bfloat162float(b);
    } else {
      __half h = __float2half(v);
      X[i] = *reinterpret_cast<uint16_t*>(&h);
      Xf[i] = __half2float(h);
    }
    const int n = i / K, k = i % K;
    const float s = (__builtin_popcount(n & k) & 1) ? -1.f : 1.f;
    Hf[i] = s;
    if (BF) {
      __nv_bfloat16 b = __float2bfloat16(s);
      H[i] = *reinterpret_cast<uint16_t*>(&b);
    } else {
      __half h = __float2half(s);
      H[i] = *reinterpret_cast<uint16_t*>(&h);
    }
  }
  uint16_t *dX, *dH;
  float* dD;
  long long* dc;
  CK(cudaMalloc(&dX, M * K * 2));
  CK(cudaMalloc(&dH, M * K * 2));
  CK(cudaMalloc(&dD, M * 128 * 4));
  CK(cudaMalloc(&dc, 8));
  CK(cudaMemcpy(dX, X.data(), M * K * 2, cudaMemcpyHostToDevice));
  CK(cudaMemcpy(dH, H.data(), M * K * 2, cudaMemcpyHostToDevice));
  CK(cudaFuncSetAttribute(probe<BF>, cudaFuncAttributeMaxDynamicSharedMemorySize, 65536 + 1024));
  probe<BF><<<1, 128, 65536 + 1024>>>(dX, dH, dD, 1, dc);
  CK(cudaDeviceSynchronize());
  std::vector<float> D(M * 128);
  CK(cudaMemcpy(D.data(), dD, M * 128 * 4, cudaMemcpyDeviceToHost));
  double maxerr = 0;
  for (int m = 0; m < M; ++m)
    for (int n = 0; n < 128; ++n) {
      double ref = 0;
      for (int k = 0; k < K; ++k) ref += double(Xf[m * K + k]) * Hf[n * K + k];
      maxerr = fmax(maxerr, fabs(ref - D[m * 128 + n]));
    }
  printf("%s: max |D - ref| = %.3e  (D[0][0..3] = %g %g %g %g)\n", BF ? "bf16" : "fp16", maxerr, D[0], D[1], D[2],
         D[3]);
  for (int reps : {1, 16, 256}) {
    probe<BF><<<1, 128, 65536 + 1024>>>(dX, dH, dD, reps, dc);
    CK(cudaDeviceSynchronize());
    long long cyc;
    CK(cudaMemcpy(&cyc, dc, 8, cudaMemcpyDeviceToHost));
    printf("  %d x 8 MMA (128x128x16): %lld cycles, %.1f cycles per MMA\n", reps, cyc, double(cyc) / (8.0 * reps));
  }
  return maxerr < 1e-3 ? 0 : 1;
}


// TMEM read throughput: W warps each load 32 lanes x 32 columns (4 KiB) `reps` times,
// waiting after every `batch` loads; returns cycles (max over warps)
template <int W>
__global__ void __launch_bounds__(W * 32) tmem_rd(int reps, long long* cycles, float* sink) {
  __shared__ uint32_t tbase;
  const int warp = threadIdx.x >> 5;
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(sa(&tbase)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tmem = tbase + (uint32_t(32 * (warp & 3)) << 16) + 64 * (warp >> 2);
  float acc = 0.f;
  __syncthreads();
  const long long t0 = clock64();
  for (int r = 0; r < reps; ++r) {
    uint32_t v[32];
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
        "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
        : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]),
          "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]),
          "=r"(v[15]), "=r"(v[16]), "=r"(v[17]), "=r"(v[18]), "=r"(v[19]), "=r"(v[20]), "=r"(v[21]),
          "=r"(v[22]), "=r"(v[23]), "=r"(v[24]), "=r"(v[25]), "=r"(v[26]), "=r"(v[27]), "=r"(v[28]),
          "=r"(v[29]), "=r"(v[30]), "=r"(v[31])
        : "r"(tmem + (r & 1) * 32));
    asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
    acc += __uint_as_float(v[r & 31]);
  }
  __syncthreads();
  const long long t1 = clock64();
  if (threadIdx.x == 0) cycles[0] = t1 - t0;
  sink[threadIdx.x] = acc;
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tbase));
}

template <int W>
void tmem_bw() {
  long long* dc;
  float* sink;
  CK(cudaMalloc(&dc, 8));
  CK(cudaMalloc(&sink, 4096));
  const int reps = 4096;
  tmem_rd<W><<<1, W * 32>>>(reps, dc, sink);
  CK(cudaDeviceSynchronize());
  long long cyc;
  CK(cudaMemcpy(&cyc, dc, 8, cudaMemcpyDeviceToHost));
  printf("TMEM read, %2d warps x %d loads of 4 KiB (wait after each): %lld cycles, %.1f B/cycle per SM\n", W, reps,
         cyc, double(W) * reps * 4096 / cyc);
}

// M = 64: which TMEM lanes hold which rows of D (A = rows 0..63 of X)
void probe_m64() {
  const int M = 128, K = 128;
  std::vector<uint16_t> X(M * K), H(M * K);
  std::vector<float> Xf(M * K), Hf(M * K);
  srand(99);
  for (int i = 0; i < M * K; ++i) {
    float v = float(rand() % 2001 - 1000) / 256.f;
    __half h = __float2half(v);
    X[i] = *reinterpret_cast<uint16_t*>(&h);
    Xf[i] = __half2float(h);
    const int n = i / K, k = i % K;
    const float s = (__builtin_popcount(n & k) & 1) ? -1.f : 1.f;
    Hf[i] = s;
    __half hh = __float2half(s);
    H[i] = *reinterpret_cast<uint16_t*>(&hh);
  }
  uint16_t *dX, *dH;
  float* dD;
  long long* dc;
  CK(cudaMalloc(&dX, M * K * 2));
  CK(cudaMalloc(&dH, M * K * 2));
  CK(cudaMalloc(&dD, M * 128 * 4));
  CK(cudaMalloc(&dc, 8));
  CK(cudaMemcpy(dX, X.data(), M * K * 2, cudaMemcpyHostToDevice));
  CK(cudaMemcpy(dH, H.data(), M * K * 2, cudaMemcpyHostToDevice));
  CK(cudaMemset(dD, 0, M * 128 * 4));
  CK(cudaFuncSetAttribute(probe<false, 64, 16>, cudaFuncAttributeMaxDynamicSharedMemorySize, 65536 + 1024));
  probe<false, 64, 16><<<1, 128, 65536 + 1024>>>(dX, dH, dD, 1, dc);
  CK(cudaDeviceSynchronize());
  std::vector<float> D(M * 128);
  CK(cudaMemcpy(D.data(), dD, M * 128 * 4, cudaMemcpyDeviceToHost));
  printf("M=64 with D lane offset 16, lane map (lane: row matched over cols 0..127, or -1):\n");
  for (int lane = 0; lane < 128; ++lane) {
    int found = -1, cols = 0;
    for (int row = 0; row < 64 && found < 0; ++row) {
      int ok = 0;
      for (int n = 0; n < 128; ++n) {
        double ref = 0;
        for (int k = 0; k < K; ++k) ref += double(Xf[row * K + k]) * Hf[n * K + k];
        ok += fabs(ref - D[lane * 128 + n]) < 1e-3;
      }
      if (ok == 128) found = row;
      if (ok > cols) cols = ok;
    }
    // partial matches: a row might be split over column halves
    printf("%d:%d%s ", lane, found, found < 0 && cols > 0 ? "*" : "");
    if (lane % 16 == 15) printf("\n");
  }
}

// TMEM read throughput by shape: 4 warps, each load = 4 KiB per warp (32 x 32 b x 32 / 16 x 256 b x 8 /
// 16 x 128 b x 16 / 32 x 32 b x 128 = 16 KiB), no wait between loads of a batch of 4
template <int SHAPE>
__global__ void __launch_bounds__(128) tmem_rd_shape(int reps, long long* cycles, float* sink) {
  __shared__ uint32_t tbase;
  const int warp = threadIdx.x >> 5;
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(sa(&tbase)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tmem = tbase + (uint32_t(32 * (warp & 3)) << 16);
  uint32_t acc = 0;
  __syncthreads();
  const long long t0 = clock64();
  for (int r = 0; r < reps; ++r) {
    uint32_t v[32];
    const uint32_t a = tmem + (r & 3) * 64;
    if constexpr (SHAPE == 0) {
      asm volatile(
          "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
          "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
          : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]),
            "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]),
            "=r"(v[15]), "=r"(v[16]), "=r"(v[17]), "=r"(v[18]), "=r"(v[19]), "=r"(v[20]), "=r"(v[21]),
            "=r"(v[22]), "=r"(v[23]), "=r"(v[24]), "=r"(v[25]), "=r"(v[26]), "=r"(v[27]), "=r"(v[28]),
            "=r"(v[29]), "=r"(v[30]), "=r"(v[31])
          : "r"(a));
    } else if constexpr (SHAPE == 1) {
      asm volatile(
          "tcgen05.ld.sync.aligned.16x256b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
          "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
          : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]),
            "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]),
            "=r"(v[15]), "=r"(v[16]), "=r"(v[17]), "=r"(v[18]), "=r"(v[19]), "=r"(v[20]), "=r"(v[21]),
            "=r"(v[22]), "=r"(v[23]), "=r"(v[24]), "=r"(v[25]), "=r"(v[26]), "=r"(v[27]), "=r"(v[28]),
            "=r"(v[29]), "=r"(v[30]), "=r"(v[31])
          : "r"(a));
    } else {
      asm volatile(
          "tcgen05.ld.sync.aligned.16x128b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
          "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
          : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]),
            "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]),
            "=r"(v[15]), "=r"(v[16]), "=r"(v[17]), "=r"(v[18]), "=r"(v[19]), "=r"(v[20]), "=r"(v[21]),
            "=r"(v[22]), "=r"(v[23]), "=r"(v[24]), "=r"(v[25]), "=r"(v[26]), "=r"(v[27]), "=r"(v[28]),
            "=r"(v[29]), "=r"(v[30]), "=r"(v[31])
          : "r"(a));
    }
    if ((r & 1) == 1) asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
    for (int j = 0; j < 32; ++j) acc += v[j];
  }
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
  __syncthreads();
  const long long t1 = clock64();
  if (threadIdx.x == 0) cycles[0] = t1 - t0;
  sink[threadIdx.x] = float(acc);
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tbase));
}
template <int SHAPE>
void tmem_shape() {
  long long* dc;
  float* sink;
  CK(cudaMalloc(&dc, 8));
  CK(cudaMalloc(&sink, 4096));
  const int reps = 4096;
  tmem_rd_shape<SHAPE><<<1, 128>>>(reps, dc, sink);
  CK(cudaDeviceSynchronize());
  long long cyc;
  CK(cudaMemcpy(&cyc, dc, 8, cudaMemcpyDeviceToHost));
  const char* nm[3] = {"32x32b.x32", "16x256b.x8", "16x128b.x16"};
  printf("TMEM read %s, 4 warps x %d loads of 4 KiB (wait every 2nd): %.1f B/cycle per SM\n", nm[SHAPE], reps,
         4.0 * reps * 4096 / cyc);
}

int main() {
  tmem_shape<0>();
  tmem_shape<1>();
  tmem_shape<2>();
  probe_m64();
  tmem_bw<4>();
  tmem_bw<8>();
  tmem_bw<16>();
  int bad = run<false>() + run<true>();
  printf(bad ? "PROBE FAILED\n" : "PROBE OK\n");
  return bad;
}
