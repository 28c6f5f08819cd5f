// tcgen05.mma issue-rate microbenchmark: one CTA per SM, one thread issues `iters` MMAs on
// static shared-memory operands (no-swizzle K-major), commits, waits; reports cycles per MMA
// and TFLOP/s for kind::tf32 (K = 8) and kind::f16 (bf16, K = 16) at N = 128 / 256.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t su32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ uint64_t desc(uint32_t a, uint32_t lbo, uint32_t sbo) {
  return (uint64_t)((a >> 4) & 0x3FFF) | ((uint64_t)((lbo >> 4) & 0x3FFF) << 16) |
         ((uint64_t)((sbo >> 4) & 0x3FFF) << 32) | ((uint64_t)1 << 46);
}

template <int KIND, int N>   // KIND 0: tf32, 1: bf16
__global__ void bench(int iters, long long* cyc) {
  extern __shared__ __align__(1024) unsigned char sm[];
  __shared__ uint32_t tslot;
  __shared__ __align__(8) uint64_t bar;
  const int t = threadIdx.x;
  for (int i = t; i < 65536 / 4; i += blockDim.x) reinterpret_cast<float*>(sm)[i] = 0.f;
  if (t < 32) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(su32(&tslot)), "r"(256));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  if (t == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(&bar)));
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  asm volatile("fence.proxy.async.shared::cta;");
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t tmem = tslot;
  if (t == 0) {
    const uint32_t fa = KIND == 0 ? 2u : 1u;   // tf32 : bf16
    const uint32_t cf = KIND == 0 ? 0u : 0u;
    (void)cf;
    const uint32_t idesc = (1u << 4) | (fa << 7) | (fa << 10) | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(128 >> 4) << 24);
    const uint64_t da = desc(su32(sm), 128, 1024), db = desc(su32(sm + 16384), 128, 1024);
    long long c0 = clock64();
    for (int i = 0; i < iters; ++i) {
      if (KIND == 0)
        asm volatile("{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\ntcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n}\n" ::"r"(tmem), "l"(da), "l"(db), "r"(idesc), "r"(1));
      else
        asm volatile("{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\ntcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n}\n" ::"r"(tmem), "l"(da), "l"(db), "r"(idesc), "r"(1));
    }
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(su32(&bar)));
    asm volatile("{\n.reg .pred P1;\nW:\nmbarrier.try_wait.parity.shared::cta.b64 P1, [%0], 0;\n@!P1 bra W;\n}\n" ::"r"(su32(&bar)));
    long long c1 = clock64();
    cyc[blockIdx.x] = c1 - c0;
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (t < 32) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(256));
}

template <int KIND, int N>
void run(const char* name) {
  const int iters = 4096, grid = 148;
  long long* d;
  cudaMalloc(&d, grid * sizeof(long long));
  cudaFuncSetAttribute(bench<KIND, N>, cudaFuncAttributeMaxDynamicSharedMemorySize, 65536);
  bench<KIND, N><<<grid, 128, 65536>>>(16, d);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0); cudaEventCreate(&e1);
  cudaEventRecord(e0);
  bench<KIND, N><<<grid, 128, 65536>>>(iters, d);
  cudaEventRecord(e1);
  cudaError_t e = cudaDeviceSynchronize();
  float ms; cudaEventElapsedTime(&ms, e0, e1);
  long long h[148]; cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
  const double K = KIND == 0 ? 8 : 16;
  const double fl = 2.0 * 128 * N * K * iters * grid;
  printf("%-10s N=%3d  %s  cycles/MMA %.1f  %.1f TFLOP/s\n", name, N, cudaGetErrorString(e),
         (double)h[0] / iters, fl / (ms * 1e-3) / 1e12);
  cudaFree(d);
}

int main() {
  run<0, 128>("tf32");
  run<0, 256>("tf32");
  run<1, 128>("bf16");
  run<1, 256>("bf16");
  return 0;
}
