// Microbenchmark: FP32 pipe throughput on sm_100a for FFMA / FFMA2 / FADD / FADD2 / FMUL2,
// to calibrate the instruction-floor model of the FFT kernels.
#include <cstdio>
#include <cuda_runtime.h>

#define ITERS 4096
#define ACC 8

__global__ void k_ffma(float* out, float a, float b) {
  float x[ACC];
  for (int i = 0; i < ACC; ++i) x[i] = threadIdx.x * 1e-3f + i;
  float c = b * 0.5f, d = a * 0.25f;
  for (int it = 0; it < ITERS; ++it) {
#pragma unroll
    for (int i = 0; i < ACC; ++i) x[i] = fmaf(x[i], c, d);
  }
  float s = 0; for (int i = 0; i < ACC; ++i) s += x[i];
  if (s == 1.2345f) out[0] = s;
}
__global__ void k_ffma2(float* out, float a, float b) {
  float2 x[ACC];
  for (int i = 0; i < ACC; ++i) x[i] = make_float2(threadIdx.x * 1e-3f + i, i);
  float2 c = make_float2(b * 0.5f, b * 0.7f), d = make_float2(a * 0.25f, a);
  for (int it = 0; it < ITERS; ++it) {
#pragma unroll
    for (int i = 0; i < ACC; ++i) x[i] = __ffma2_rn(x[i], c, d);
  }
  float s = 0; for (int i = 0; i < ACC; ++i) s += x[i].x + x[i].y;
  if (s == 1.2345f) out[0] = s;
}
__global__ void k_fadd(float* out, float a, float b) {
  float x[ACC];
  for (int i = 0; i < ACC; ++i) x[i] = threadIdx.x * 1e-3f + i;
  float c = b * 0.5f;
  for (int it = 0; it < ITERS; ++it) {
#pragma unroll
    for (int i = 0; i < ACC; ++i) x[i] = x[i] + c;
  }
  float s = 0; for (int i = 0; i < ACC; ++i) s += x[i];
  if (s == 1.2345f) out[0] = s;
}
__global__ void k_fadd2(float* out, float a, float b) {
  float2 x[ACC];
  for (int i = 0; i < ACC; ++i) x[i] = make_float2(threadIdx.x * 1e-3f + i, i);
  float2 c = make_float2(b * 0.5f, b);
  for (int it = 0; it < ITERS; ++it) {
#pragma unroll
    for (int i = 0; i < ACC; ++i) x[i] = __fadd2_rn(x[i], c);
  }
  float s = 0; for (int i = 0; i < ACC; ++i) s += x[i].x + x[i].y;
  if (s == 1.2345f) out[0] = s;
}
__global__ void k_fmul2(float* out, float a, float b) {
  float2 x[ACC];
  for (int i = 0; i < ACC; ++i) x[i] = make_float2(threadIdx.x * 1e-3f + i, i);
  float2 c = make_float2(b * 0.5f, b);
  for (int it = 0; it < ITERS; ++it) {
#pragma unroll
    for (int i = 0; i < ACC; ++i) x[i] = __fmul2_rn(x[i], c);
  }
  float s = 0; for (int i = 0; i < ACC; ++i) s += x[i].x + x[i].y;
  if (s == 1.2345f) out[0] = s;
}
// mixed: 1 FFMA2 + 1 FADD2 alternating (FFT-like mix)
__global__ void k_mix(float* out, float a, float b) {
  float2 x[ACC], y[ACC];
  for (int i = 0; i < ACC; ++i) { x[i] = make_float2(threadIdx.x * 1e-3f + i, i); y[i] = x[i]; }
  float2 c = make_float2(b * 0.5f, b * 0.7f), d = make_float2(a * 0.25f, a);
  for (int it = 0; it < ITERS; ++it) {
#pragma unroll
    for (int i = 0; i < ACC; ++i) { x[i] = __ffma2_rn(x[i], c, d); y[i] = __fadd2_rn(y[i], c); }
  }
  float s = 0; for (int i = 0; i < ACC; ++i) s += x[i].x + x[i].y + y[i].x;
  if (s == 1.2345f) out[0] = s;
}

template <class K>
void run(const char* name, K k, int ops_per_inst_lane, int inst_per_iter) {
  float* out; cudaMalloc(&out, 4);
  int sms = 0; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  int blocks = sms * 8, threads = 256;
  k<<<blocks, threads>>>(out, 1.f, 2.f);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  cudaEventRecord(e0);
  for (int r = 0; r < 5; ++r) k<<<blocks, threads>>>(out, 1.f, 2.f);
  cudaEventRecord(e1); cudaEventSynchronize(e1);
  float ms; cudaEventElapsedTime(&ms, e0, e1);
  double warp_inst = 5.0 * blocks * (threads / 32) * (double)ITERS * ACC * inst_per_iter;
  int clk; cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  double secs = ms * 1e-3;
  double inst_per_s_per_sm = warp_inst / secs / sms;
  printf("%-6s %8.3f ms  warp-inst/s/SM %.3e  lane-ops/s (chip) %.3e  [clockRate attr %d kHz]\n", name, ms,
         inst_per_s_per_sm, warp_inst * 32 * ops_per_inst_lane / secs, clk);
}

int main() {
  run("FFMA", k_ffma, 1, 1);
  run("FFMA2", k_ffma2, 2, 1);
  run("FADD", k_fadd, 1, 1);
  run("FADD2", k_fadd2, 2, 1);
  run("FMUL2", k_fmul2, 2, 1);
  run("MIX", k_mix, 2, 2);
  return 0;
}
