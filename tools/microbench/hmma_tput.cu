// Microbenchmark: legacy mma.sync (HMMA) throughput on sm_100a, f16 and bf16->f32.
// Dev tool only (not part of the product path).
#include <cstdio>
#include <cuda_runtime.h>
#include <cstdint>

template <int CHAINS>
__global__ void hmma_f16(uint32_t* out, int iters) {
  uint32_t a0 = threadIdx.x, a1 = a0 * 3, a2 = a0 * 5, a3 = a0 * 7;
  uint32_t b0 = a0 ^ 0x3c003c00u, b1 = a1 ^ 0x3c003c00u;
  uint32_t d[CHAINS][2];
#pragma unroll
  for (int c = 0; c < CHAINS; ++c) { d[c][0] = c; d[c][1] = c + 1; }
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int c = 0; c < CHAINS; ++c) {
      asm volatile("mma.sync.aligned.m16n8k16.row.col.f16.f16.f16.f16 {%0,%1}, {%2,%3,%4,%5}, {%6,%7}, {%0,%1};\n"
                   : "+r"(d[c][0]), "+r"(d[c][1]) : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1));
    }
  }
  uint32_t s = 0;
#pragma unroll
  for (int c = 0; c < CHAINS; ++c) s ^= d[c][0] ^ d[c][1];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

template <int CHAINS>
__global__ void hmma_bf16(uint32_t* out, int iters) {
  uint32_t a0 = threadIdx.x, a1 = a0 * 3, a2 = a0 * 5, a3 = a0 * 7;
  uint32_t b0 = a0 ^ 0x3f803f80u, b1 = a1 ^ 0x3f803f80u;
  float d[CHAINS][4];
#pragma unroll
  for (int c = 0; c < CHAINS; ++c) { d[c][0] = c; d[c][1] = c; d[c][2] = c; d[c][3] = c; }
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int c = 0; c < CHAINS; ++c) {
      asm volatile("mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};\n"
                   : "+f"(d[c][0]), "+f"(d[c][1]), "+f"(d[c][2]), "+f"(d[c][3])
                   : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1));
    }
  }
  float s = 0;
#pragma unroll
  for (int c = 0; c < CHAINS; ++c) s += d[c][0] + d[c][1] + d[c][2] + d[c][3];
  out[blockIdx.x * blockDim.x + threadIdx.x] = __float_as_uint(s);
}

template <typename K>
void run(const char* name, K kern, int blocks, int threads, int iters, int chains) {
  uint32_t* out; cudaMalloc(&out, blocks * threads * 4);
  kern<<<blocks, threads>>>(out, 10);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  cudaEventRecord(e0);
  kern<<<blocks, threads>>>(out, iters);
  cudaEventRecord(e1); cudaEventSynchronize(e1);
  float ms; cudaEventElapsedTime(&ms, e0, e1);
  double mmas = (double)blocks * (threads / 32) * iters * chains;
  double flops = mmas * 2.0 * 16 * 8 * 16;
  int dev; cudaGetDevice(&dev); int clk; cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, dev);
  printf("%s blocks=%d threads=%d chains=%d: %.3f ms, %.1f TFLOP/s, %.1f flop/clk/SM @%.0fMHz(attr), HMMA/clk/SM=%.3f\n", name, blocks, threads, chains,
         ms, flops / ms / 1e9, flops / (ms * 1e-3) / 148 / (clk * 1e3), clk / 1e3, mmas / (ms * 1e-3) / 148 / (clk * 1e3));
  cudaFree(out);
}

int main() {
  for (int t : {128, 256, 512, 1024}) {
    run("f16 ", hmma_f16<4>, 148 * 2, t, 20000, 4);
    run("bf16", hmma_bf16<4>, 148 * 2, t, 20000, 4);
  }
  run("f16 c8", hmma_f16<8>, 148 * 2, 512, 10000, 8);
  run("bf16 c8", hmma_bf16<8>, 148 * 2, 512, 10000, 8);
  run("f16 c1", hmma_f16<1>, 148, 32, 100000, 1);
  run("bf16 c1", hmma_bf16<1>, 148, 32, 100000, 1);
  return 0;
}
