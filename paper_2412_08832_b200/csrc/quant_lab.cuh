// quant_lab.cuh -- GPU kernels of the rotation / quantization-error experiment
// (SPEC quant_lab S:397-440; the paper's motivation P:24
// [Sec. 1] "Hadamard rotations ... reduce the magnitude of outliers" and P:180
// [Sec. 4.2] "comparable quantization error reduction").  The rotations themselves
// are hadacore_fwht calls (fp32 path); these kernels are the experiment's harness:
//   * row_amax_kernel      max |x| of every row (warp per row)
//   * tensor_amax_kernel   max over the rows' maxima, broadcast back (one CTA)
//   * fake_quant_kernel    symmetric quantize -> dequantize with scale = amax / Q
//   * row_sq_error_kernel  sum_j (a_ij - b_ij)^2 per row, fp64 accumulation
// All fp32 in, fp32 out (fp64 error sums); rows contiguous, n a power of two.
#pragma once
#include <cuda_fp16.h>
#include <stdint.h>

namespace hadacore {
namespace lab {

enum : int { LQ_E4M3 = 0, LQ_INT8 = 1, LQ_INT4 = 2 };

template <int Q>
__host__ __device__ constexpr float qmax() {
  return Q == LQ_E4M3 ? 448.f : (Q == LQ_INT8 ? 127.f : 7.f);
}

__device__ __forceinline__ float warp_max(float v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = fmaxf(v, __shfl_xor_sync(0xffffffffu, v, o));
  return v;
}

__global__ void row_amax_kernel(const float* __restrict__ x, float* __restrict__ amax, int64_t m, int64_t n) {
  const int lane = threadIdx.x & 31;
  const int64_t warps = int64_t(gridDim.x) * (blockDim.x >> 5);
  for (int64_t r = int64_t(blockIdx.x) * (blockDim.x >> 5) + (threadIdx.x >> 5); r < m; r += warps) {
    const float* row = x + r * n;
    float a = 0.f;
    if (n % 128 == 0) {
      for (int64_t j = 4 * lane; j < n; j += 128) {
        const float4 v = *reinterpret_cast<const float4*>(row + j);
        a = fmaxf(a, fmaxf(fmaxf(fabsf(v.x), fabsf(v.y)), fmaxf(fabsf(v.z), fabsf(v.w))));
      }
    } else {
      for (int64_t j = lane; j < n; j += 32) a = fmaxf(a, fabsf(row[j]));
    }
    a = warp_max(a);
    if (lane == 0) amax[r] = a;
  }
}

// one CTA: amax[i] <- max_k amax[k] for every i (PerTensor: one scale for the matrix)
__global__ void tensor_amax_kernel(float* __restrict__ amax, int64_t m) {
  __shared__ float part[32];
  float a = 0.f;
  for (int64_t i = threadIdx.x; i < m; i += blockDim.x) a = fmaxf(a, amax[i]);
  a = warp_max(a);
  if ((threadIdx.x & 31) == 0) part[threadIdx.x >> 5] = a;
  __syncthreads();
  if (threadIdx.x < 32) {
    float b = threadIdx.x < (blockDim.x >> 5) ? part[threadIdx.x] : 0.f;
    b = warp_max(b);
    if (threadIdx.x == 0) part[0] = b;
  }
  __syncthreads();
  const float t = part[0];
  for (int64_t i = threadIdx.x; i < m; i += blockDim.x) amax[i] = t;
}

// code of v = x / s: E4M3 by the hardware RNE satfinite conversion, integers by
// rint (ties to even) clamped to +-Q; returns the dequantized code value
template <int Q>
__device__ __forceinline__ float code_value(float v) {
  if constexpr (Q == LQ_E4M3) {
    uint16_t c;
    asm("cvt.rn.satfinite.e4m3x2.f32 %0, %1, %2;" : "=h"(c) : "f"(0.f), "f"(v));
    uint32_t h2;
    asm("cvt.rn.f16x2.e4m3x2 %0, %1;" : "=r"(h2) : "h"(c));
    return __half2float(__ushort_as_half(uint16_t(h2 & 0xffffu)));
  } else {
    return fminf(fmaxf(rintf(v), -qmax<Q>()), qmax<Q>());
  }
}

template <int Q>
__global__ void fake_quant_kernel(const float* __restrict__ x, float* __restrict__ out,
                                  const float* __restrict__ amax, int64_t total, int log2n) {
  const int64_t stride = int64_t(gridDim.x) * blockDim.x;
  for (int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < total; i += stride) {
    const float a = amax[i >> log2n];
    const float s = a > 0.f ? a / qmax<Q>() : 1.f;  // S:421 scale = max_abs / Q; all-zero -> 1
    out[i] = a > 0.f ? code_value<Q>(x[i] / s) * s : 0.f;
  }
}

__global__ void row_sq_error_kernel(const float* __restrict__ a, const float* __restrict__ b,
                                    double* __restrict__ out, int64_t m, int64_t n) {
  const int lane = threadIdx.x & 31;
  const int64_t warps = int64_t(gridDim.x) * (blockDim.x >> 5);
  for (int64_t r = int64_t(blockIdx.x) * (blockDim.x >> 5) + (threadIdx.x >> 5); r < m; r += warps) {
    double acc = 0.0;
    for (int64_t j = lane; j < n; j += 32) {
      const double d = double(a[r * n + j]) - double(b[r * n + j]);
      acc = fma(d, d, acc);
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
    if (lane == 0) out[r] = acc;
  }
}

}  // namespace lab
}  // namespace hadacore
