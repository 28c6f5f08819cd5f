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

// Per-image squared norms of the NNLS update f - fp and of the iterate f (the 0.3 % stopping
// rule, §4.3): block (k, b) sums a fixed contiguous range of image b with a
// fixed per-thread order and a fixed float64 tree, so the result is bitwise reproducible.
__global__ void __launch_bounds__(256) k_diff_norms(const float* __restrict__ f, const float* __restrict__ fp,
                                                    size_t per, double* part) {
  __shared__ double red[2][256];
  const int b = blockIdx.y, k = blockIdx.x;
  const size_t chunk = (per + kNormParts - 1) / kNormParts;
  const size_t i0 = (size_t)k * chunk, i1 = i0 + chunk < per ? i0 + chunk : per;
  const float* x = f + (size_t)b * per;
  const float* y = fp + (size_t)b * per;
  float sd = 0.f, sf = 0.f;
  for (size_t i = i0 + threadIdx.x; i < i1; i += blockDim.x) {
    const float a = __ldg(&x[i]), d = a - __ldg(&y[i]);
    sd = fmaf(d, d, sd);
    sf = fmaf(a, a, sf);
  }
  red[0][threadIdx.x] = sd;
  red[1][threadIdx.x] = sf;
  __syncthreads();
  for (int w = 128; w > 0; w >>= 1) {
    if ((int)threadIdx.x < w) {
      red[0][threadIdx.x] += red[0][threadIdx.x + w];
      red[1][threadIdx.x] += red[1][threadIdx.x + w];
    }
    __syncthreads();
  }
  if (threadIdx.x == 0) {
    part[((size_t)b * kNormParts + k) * 2] = red[0][0];
    part[((size_t)b * kNormParts + k) * 2 + 1] = red[1][0];
  }
}

cudaError_t launch_diff_norms(const float* f, const float* fp, int batch, size_t per_image, double* part,
                              cudaStream_t s) {
  k_diff_norms<<<dim3(kNormParts, batch), 256, 0, s>>>(f, fp, per_image, part);
  return cudaGetLastError();
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

// Reading G25 (low-harmonic quadrature variant): out[b] = coef * sum of image b (times the G26
// factors d[ix] d[iy] when dw != nullptr), as kLowkParts fixed-range partial sums per image in
// float64; the CTA that finishes last (per-image counter) adds the partials in a fixed order and
// resets the counter, so the result is deterministic.
constexpr int kLowkParts = 32;
__global__ void __launch_bounds__(256) k_lowk_sum(const float* __restrict__ x, size_t per, int b0, double coef,
                                                  const float* __restrict__ dw, int n, float* __restrict__ out,
                                                  double* __restrict__ part, unsigned int* __restrict__ cnt) {
  __shared__ double red[8];
  __shared__ bool last;
  pdl_trigger();
  const int b = b0 + blockIdx.y, q = blockIdx.x;
  const float* p = x + (size_t)b * per;
  double acc = 0.0;
  if (dw) {   // rows [n q / P, n (q + 1) / P) of D f
    const int y0 = n * q / kLowkParts, y1 = n * (q + 1) / kLowkParts;
    for (int iy = y0 + (threadIdx.x >> 5); iy < y1; iy += blockDim.x >> 5) {
      double row = 0.0;
      for (int ix = threadIdx.x & 31; ix < n; ix += 32) row += (double)__ldg(p + (size_t)iy * n + ix) * dw[ix];
      acc += row * dw[iy];
    }
  } else {
    const size_t i0 = per * q / kLowkParts, i1 = per * (q + 1) / kLowkParts;
    for (size_t i = i0 + threadIdx.x; i < i1; i += blockDim.x) acc += (double)__ldg(p + i);
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = acc;
  __syncthreads();
  if (threadIdx.x == 0) {
    double s = 0.0;
    for (int w = 0; w < 8; ++w) s += red[w];
    part[(size_t)b * kLowkParts + q] = s;
    __threadfence();
    last = atomicAdd(&cnt[b], 1u) == kLowkParts - 1;
  }
  __syncthreads();
  if (last && threadIdx.x == 0) {
    __threadfence();
    double s = 0.0;
    for (int k = 0; k < kLowkParts; ++k) s += *((volatile double*)&part[(size_t)b * kLowkParts + k]);
    out[b] = (float)(coef * s);
    cnt[b] = 0;
  }
}

cudaError_t launch_lowk_sum(const DevPlan& P, const float* x, size_t per_image, double coef, bool image,
                            cudaStream_t s) {
  k_lowk_sum<<<dim3(kLowkParts, P.C.batch), 256, 0, s>>>(x, per_image, P.C.b0, coef, image ? P.deapod : nullptr,
                                                         P.C.n, P.lowk_add, P.lowk_part, P.lowk_cnt);
  return cudaGetLastError();
}

}  // namespace tat
