// Microbenchmark: achievable HBM copy bandwidth on B200 (dev tool only).
#include <cstdio>
#include <cuda_runtime.h>
#include <cstdint>

__global__ void copy_v4(const int4* __restrict__ in, int4* __restrict__ out, size_t n16) {
  size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x;
  size_t stride = (size_t)gridDim.x * blockDim.x;
  for (; i + 3 * stride < n16; i += 4 * stride) {
    int4 a = in[i], b = in[i + stride], c = in[i + 2 * stride], d = in[i + 3 * stride];
    out[i] = a; out[i + stride] = b; out[i + 2 * stride] = c; out[i + 3 * stride] = d;
  }
  for (; i < n16; i += stride) out[i] = in[i];
}

int main() {
  size_t bytes = 1ull << 30;
  void *a, *b; cudaMalloc(&a, bytes); cudaMalloc(&b, bytes);
  cudaMemset(a, 1, bytes); cudaMemset(b, 0, bytes);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  float ms;
  for (int r = 0; r < 3; ++r) {
    cudaEventRecord(e0); cudaMemcpyAsync(b, a, bytes, cudaMemcpyDeviceToDevice); cudaEventRecord(e1);
    cudaEventSynchronize(e1); cudaEventElapsedTime(&ms, e0, e1);
    printf("memcpy D2D 1GiB: %.3f ms  %.1f GB/s (r+w)\n", ms, 2.0 * bytes / ms / 1e6);
  }
  for (int bpsm : {1, 2, 4, 8}) for (int t : {256, 512, 1024}) {
    int blocks = 148 * bpsm;
    copy_v4<<<blocks, t>>>((int4*)a, (int4*)b, bytes / 16);
    cudaEventRecord(e0); copy_v4<<<blocks, t>>>((int4*)a, (int4*)b, bytes / 16); cudaEventRecord(e1);
    cudaEventSynchronize(e1); cudaEventElapsedTime(&ms, e0, e1);
    printf("copy_v4 blocks=%d threads=%d: %.3f ms %.1f GB/s\n", blocks, t, ms, 2.0 * bytes / ms / 1e6);
  }
  // in-place read-modify-write
  copy_v4<<<148*4, 512>>>((int4*)a, (int4*)a, bytes / 16);
  cudaEventRecord(e0); copy_v4<<<148*4, 512>>>((int4*)a, (int4*)a, bytes / 16); cudaEventRecord(e1);
  cudaEventSynchronize(e1); cudaEventElapsedTime(&ms, e0, e1);
  printf("copy_v4 in-place: %.3f ms %.1f GB/s\n", ms, 2.0 * bytes / ms / 1e6);
  return 0;
}
