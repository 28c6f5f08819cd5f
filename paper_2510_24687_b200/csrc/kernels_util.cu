// Small vector kernels of the iterative driver's setup (tat_power_norm): a counter-based random
// start vector and fixed-order partial dot products (deterministic; summed in float64 on the
// host).  Not on the per-iteration path.
#include "tat_internal.h"

namespace tat {

// splitmix64 of (seed, i) -> uniform in [-1, 1)
__device__ __forceinline__ float hash_uniform(unsigned long long seed, unsigned long long i) {
  unsigned long long z = seed * 0x9E3779B97F4A7C15ull + i + 0x632BE59BD9B4E019ull;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  z ^= z >> 31;
  return (float)((z >> 40) * (1.0 / 16777216.0)) * 2.f - 1.f;
}

__global__ void k_fill_random(float* v, size_t count, unsigned long long seed) {
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < count; i += (size_t)gridDim.x * blockDim.x)
    v[i] = hash_uniform(seed, i);
}

__global__ void k_scale(float* v, size_t count, float s) {
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < count; i += (size_t)gridDim.x * blockDim.x)
    v[i] *= s;
}

// partial[blockIdx.x] = sum over this block's grid-stride elements of a[i] * b[i]
__global__ void __launch_bounds__(256) k_dot_partial(const float* a, const float* b, size_t count, float* partial) {
  __shared__ float red[256];
  float s = 0.f;
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < count; i += (size_t)gridDim.x * blockDim.x)
    s = fmaf(a[i], b[i], s);
  red[threadIdx.x] = s;
  __syncthreads();
  for (int w = 128; w > 0; w >>= 1) {
    if ((int)threadIdx.x < w) red[threadIdx.x] += red[threadIdx.x + w];
    __syncthreads();
  }
  if (threadIdx.x == 0) partial[blockIdx.x] = red[0];
}

cudaError_t launch_fill_random(float* v, size_t count, unsigned long long seed, cudaStream_t s) {
  k_fill_random<<<kUtilBlocks, 256, 0, s>>>(v, count, seed);
  return cudaGetLastError();
}
cudaError_t launch_scale(float* v, size_t count, float f, cudaStream_t s) {
  k_scale<<<kUtilBlocks, 256, 0, s>>>(v, count, f);
  return cudaGetLastError();
}
cudaError_t launch_dot_partial(const float* a, const float* b, size_t count, float* partial, cudaStream_t s) {
  k_dot_partial<<<kUtilBlocks, 256, 0, s>>>(a, b, count, partial);
  return cudaGetLastError();
}

}  // namespace tat
