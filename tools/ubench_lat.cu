// Microbenchmark: FADD2 dependent latency, and throughput vs (warps per SM, independent chains),
// plus LDS.64 + FADD2 overlap.  Answers whether the FFT kernels are latency- or pipe-bound.
#include <cstdio>
#include <cuda_runtime.h>

#define ITERS 2048

template <int ILP>
__global__ void k_chain(float* out, float b, long long* cyc) {
  float2 x[ILP];
  for (int i = 0; i < ILP; ++i) x[i] = make_float2(threadIdx.x * 1e-3f + i, i);
  const float2 c = make_float2(b * 0.5f, b);
  long long t0 = clock64();
  for (int it = 0; it < ITERS; ++it) {
#pragma unroll
    for (int i = 0; i < ILP; ++i) x[i] = __fadd2_rn(x[i], c);
  }
  long long t1 = clock64();
  float s = 0;
  for (int i = 0; i < ILP; ++i) s += x[i].x + x[i].y;
  if (s == 1.2345f) out[0] = s;
  if (threadIdx.x == 0 && blockIdx.x == 0) cyc[0] = t1 - t0;
}

// LDS.64 stream + FADD2 chains: per iteration NL loads and NF adds (independent)
template <int NL, int NF>
__global__ void k_mixls(float* out, float b) {
  __shared__ float2 sm[4096];
  for (int i = threadIdx.x; i < 4096; i += blockDim.x) sm[i] = make_float2(i, b);
  __syncthreads();
  float2 acc[8];
  for (int i = 0; i < 8; ++i) acc[i] = make_float2(0.f, 0.f);
  const float2 c = make_float2(b * 0.5f, b);
  int base = threadIdx.x & 31;
  for (int it = 0; it < ITERS; ++it) {
#pragma unroll
    for (int l = 0; l < NL; ++l) {
      float2 v = sm[(base + 32 * l + it * 7) & 4095];
      acc[l & 7] = __fadd2_rn(acc[l & 7], v);
    }
#pragma unroll
    for (int f = 0; f < NF; ++f) acc[f & 7] = __fadd2_rn(acc[f & 7], c);
  }
  float s = 0;
  for (int i = 0; i < 8; ++i) s += acc[i].x + acc[i].y;
  if (s == 1.2345f) out[0] = s;
}

template <class K>
float timeit(K k, int blocks, int threads, float* out) {
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0); cudaEventCreate(&e1);
  k<<<blocks, threads>>>(out, 2.f);
  cudaEventRecord(e0);
  for (int r = 0; r < 3; ++r) k<<<blocks, threads>>>(out, 2.f);
  cudaEventRecord(e1); cudaEventSynchronize(e1);
  float ms; cudaEventElapsedTime(&ms, e0, e1);
  return ms / 3;
}

int main() {
  float* out; cudaMalloc(&out, 4);
  long long* cyc; cudaMalloc(&cyc, 8);
  int sms = 0; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  long long h;
  k_chain<1><<<1, 32>>>(out, 2.f, cyc); cudaMemcpy(&h, cyc, 8, cudaMemcpyDeviceToHost);
  printf("FADD2 dependent latency: %.2f cycles\n", (double)h / ITERS);
  k_chain<4><<<1, 32>>>(out, 2.f, cyc); cudaMemcpy(&h, cyc, 8, cudaMemcpyDeviceToHost);
  printf("FADD2 4 chains, 1 warp: %.2f cycles per instr\n", (double)h / ITERS / 4);
  // throughput: warps per SM w (4 SMSPs), ILP
  int ws[] = {4, 8, 12, 16, 32};
  for (int w : ws) {
    auto run = [&](auto kern, int ilp) {
      float ms = timeit([&](float* o, float bb) { kern<<<sms, w * 32>>>(o, bb, cyc); }, 0, 0, out);
      (void)ms;
    };
    (void)run;
    float t1, t2, t4, t8;
    {
      cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
      auto T = [&](auto kk) { kk<<<sms, w * 32>>>(out, 2.f, cyc); cudaEventRecord(e0);
        for (int r = 0; r < 3; ++r) kk<<<sms, w * 32>>>(out, 2.f, cyc);
        cudaEventRecord(e1); cudaEventSynchronize(e1); float ms; cudaEventElapsedTime(&ms, e0, e1); return ms / 3; };
      t1 = T(k_chain<1>); t2 = T(k_chain<2>); t4 = T(k_chain<4>); t8 = T(k_chain<8>);
    }
    // warp-instr per SM per ns -> per cycle at ~1.9 GHz reported separately
    auto rate = [&](float ms, int ilp) { return (double)w * ITERS * ilp / (ms * 1e6); };  // warp-inst / ns / SM
    printf("warps/SM %2d: FADD2 warp-inst/ns/SM  ILP1 %.3f  ILP2 %.3f  ILP4 %.3f  ILP8 %.3f\n", w,
           rate(t1, 1), rate(t2, 2), rate(t4, 4), rate(t8, 8));
  }
  // LDS + FADD2 overlap (12 warps/SM)
  {
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    auto T = [&](auto kk, int w) { kk<<<sms, w * 32>>>(out, 2.f); cudaEventRecord(e0);
      for (int r = 0; r < 3; ++r) kk<<<sms, w * 32>>>(out, 2.f);
      cudaEventRecord(e1); cudaEventSynchronize(e1); float ms; cudaEventElapsedTime(&ms, e0, e1); return ms / 3; };
    for (int w : {12, 16, 32}) {
      float a = T(k_mixls<8, 0>, w), bq = T(k_mixls<0, 16>, w), cq = T(k_mixls<8, 16>, w);
      printf("warps/SM %2d: 8 LDS.64 only %.3f ms | 16 FADD2 only %.3f ms | both %.3f ms\n", w, a, bq, cq);
    }
  }
  return 0;
}
