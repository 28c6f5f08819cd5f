// Microbenchmark: shared-memory LDS.64 / STS.64 and SHFL throughput per SM on sm_100a
// (calibrates the exchange cost model of the FFT passes).
#include <cstdio>
#include <cuda_runtime.h>
#define ITERS 2048

__global__ void k_lds64(float* out, int stride) {
  __shared__ float2 s[4096];
  for (int i = threadIdx.x; i < 4096; i += blockDim.x) s[i] = make_float2(i, i);
  __syncthreads();
  float2 acc = make_float2(0, 0);
  int idx = threadIdx.x;
  for (int it = 0; it < ITERS; ++it) {
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      float2 v = s[(idx + u * 256) & 4095];
      acc.x += v.x; acc.y += v.y;
    }
    idx += 1;
  }
  if (acc.x == 1.234f) out[0] = acc.y;
}
__global__ void k_sts64(float* out, int stride) {
  __shared__ float2 s[4096];
  int idx = threadIdx.x;
  float2 v = make_float2(threadIdx.x, 1);
  for (int it = 0; it < ITERS; ++it) {
#pragma unroll
    for (int u = 0; u < 8; ++u) s[(idx + u * 256) & 4095] = v;
    idx += 1; v.x += 1.f;
  }
  __syncthreads();
  if (s[threadIdx.x].x == 1.234f) out[0] = 1;
}
__global__ void k_shfl(float* out, int stride) {
  float a[8];
  for (int u = 0; u < 8; ++u) a[u] = threadIdx.x + u;
  for (int it = 0; it < ITERS; ++it) {
#pragma unroll
    for (int u = 0; u < 8; ++u) a[u] = __shfl_xor_sync(0xffffffff, a[u], 1 + (u & 3));
  }
  float s = 0; for (int u = 0; u < 8; ++u) s += a[u];
  if (s == 1.234f) out[0] = s;
}
// LDS.64 and SHFL interleaved: if both reach their solo rate the datapaths are separate
__global__ void k_mixed(float* out, int stride) {
  __shared__ float2 s[4096];
  for (int i = threadIdx.x; i < 4096; i += blockDim.x) s[i] = make_float2(i, i);
  __syncthreads();
  float2 acc = make_float2(0, 0);
  float a[4];
  for (int u = 0; u < 4; ++u) a[u] = threadIdx.x + u;
  int idx = threadIdx.x;
  for (int it = 0; it < ITERS; ++it) {
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      float2 v = s[(idx + u * 256) & 4095];
      acc.x += v.x; acc.y += v.y;
      a[u] = __shfl_xor_sync(0xffffffff, a[u], 1 + u);
      a[u] = __shfl_xor_sync(0xffffffff, a[u], 2 + u);
    }
    idx += 1;
  }
  float t = a[0] + a[1] + a[2] + a[3];
  if (acc.x == 1.234f || t == 1.234f) out[0] = acc.y + t;
}
template <class K>
void run(const char* name, K k, int inst_per_iter) {
  float* out; cudaMalloc(&out, 4);
  int sms = 0; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  int blocks = sms * 4, threads = 256;
  k<<<blocks, threads>>>(out, 1);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  cudaEventRecord(e0);
  for (int r = 0; r < 5; ++r) k<<<blocks, threads>>>(out, 1);
  cudaEventRecord(e1); cudaEventSynchronize(e1);
  float ms; cudaEventElapsedTime(&ms, e0, e1);
  double warp_inst = 5.0 * blocks * (threads / 32) * (double)ITERS * inst_per_iter;
  double cyc = ms * 1e-3 * 1.965e9;
  printf("%-6s %8.3f ms  warp-inst per SM-cycle %.3f\n", name, ms, warp_inst / sms / cyc);
}
int main() {
  run("LDS64", k_lds64, 8);
  run("STS64", k_sts64, 8);
  run("SHFL", k_shfl, 8);
  run("MIXED(4 LDS.64 + 8 SHFL)", k_mixed, 12);
  return 0;
}
