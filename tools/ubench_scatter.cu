// Microbenchmark for the K2Ta access pattern: CTA per (column, image) writing a contiguous
// ~520-entry float2 range of a 136 MB buffer, optionally reading a ~384-entry window first.
#include <cstdio>
#include <cuda_runtime.h>

__global__ void k_write(float2* out, int per, int ncols) {
  const int p = blockIdx.x, b = blockIdx.y;
  float2* o = out + ((size_t)b * ncols + p) * per;
  for (int i = threadIdx.x; i < per; i += blockDim.x) o[i] = make_float2(i, p);
}
__global__ void k_rw(const float2* __restrict__ in, float2* out, int per, int win, int ncols) {
  extern __shared__ float2 w[];
  const int p = blockIdx.x, b = blockIdx.y;
  const float2* s = in + ((size_t)b * ncols + p) * (win / 2);
  for (int i = threadIdx.x; i < win; i += blockDim.x) w[i] = s[i];
  __syncthreads();
  float2* o = out + ((size_t)b * ncols + p) * per;
  for (int i = threadIdx.x; i < per; i += blockDim.x) { float2 v = w[(i * 7) % win]; o[i] = v; }
}
int main() {
  const int ncols = 2049, B = 16, per = 520, win = 384;
  float2 *out, *in;
  cudaMalloc(&out, (size_t)B * ncols * per * 8);
  cudaMalloc(&in, (size_t)B * ncols * win * 8);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  float ms;
  for (int th : {128, 256}) {
    k_write<<<dim3(ncols, B), th>>>(out, per, ncols);
    cudaEventRecord(e0);
    for (int r = 0; r < 5; ++r) k_write<<<dim3(ncols, B), th>>>(out, per, ncols);
    cudaEventRecord(e1); cudaEventSynchronize(e1); cudaEventElapsedTime(&ms, e0, e1);
    printf("write-only   %d thr: %.1f us  (%.2f TB/s)\n", th, ms / 5 * 1000, (double)B * ncols * per * 8 / (ms / 5 * 1e-3) / 1e12);
    k_rw<<<dim3(ncols, B), th, win * 8>>>(in, out, per, win, ncols);
    cudaEventRecord(e0);
    for (int r = 0; r < 5; ++r) k_rw<<<dim3(ncols, B), th, win * 8>>>(in, out, per, win, ncols);
    cudaEventRecord(e1); cudaEventSynchronize(e1); cudaEventElapsedTime(&ms, e0, e1);
    printf("window+write %d thr: %.1f us\n", th, ms / 5 * 1000);
  }
  // one big CTA count alternative: persistent grid-stride write
  return 0;
}
