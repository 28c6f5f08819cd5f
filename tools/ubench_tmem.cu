// TMEM load / store throughput per SM (B200): W warps per CTA (4 per lane quarter pattern), each
// issuing tcgen05.ld / tcgen05.st 32x32b.x32 (32 lanes x 32 columns x 4 B = 4 KB per warp-op) in a
// loop; one CTA per SM.  Prints bytes per SM-cycle.  Measured on B200: ld 53-55 B/clk/SM for 4-16
// warps (the 16x256b shape the same), st 500-750 B/clk/SM.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t su32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

template <bool LD>
__global__ void k(int iters, long long* cyc, float* sink) {
  __shared__ uint32_t tslot;
  const int t = threadIdx.x, warp = t >> 5, quarter = warp & 3;
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(su32(&tslot)), "r"(512));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t tm = tslot + ((uint32_t)(32 * quarter) << 16);
  const uint32_t c0w = 32 * (warp >> 2);
  uint32_t v[32];
  for (int i = 0; i < 32; ++i) v[i] = t + i;
  __syncthreads();
  long long c0 = clock64();
  float acc = 0.f;
  for (int it = 0; it < iters; ++it) {
    const uint32_t a = tm + ((c0w + it * 64) & 480);   // a 32-column block inside the 512 allocated
    if (LD) {
      asm volatile("tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
                   "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
                   : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]),
                     "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15]),
                     "=r"(v[16]), "=r"(v[17]), "=r"(v[18]), "=r"(v[19]), "=r"(v[20]), "=r"(v[21]), "=r"(v[22]), "=r"(v[23]),
                     "=r"(v[24]), "=r"(v[25]), "=r"(v[26]), "=r"(v[27]), "=r"(v[28]), "=r"(v[29]), "=r"(v[30]), "=r"(v[31])
                   : "r"(a));
      asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
      acc += __uint_as_float(v[it & 31]);
    } else {
      asm volatile("tcgen05.st.sync.aligned.32x32b.x32.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,"
                   "%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31,%32};"
                   ::"r"(a), "r"(v[0]), "r"(v[1]), "r"(v[2]), "r"(v[3]), "r"(v[4]), "r"(v[5]), "r"(v[6]), "r"(v[7]),
                     "r"(v[8]), "r"(v[9]), "r"(v[10]), "r"(v[11]), "r"(v[12]), "r"(v[13]), "r"(v[14]), "r"(v[15]),
                     "r"(v[16]), "r"(v[17]), "r"(v[18]), "r"(v[19]), "r"(v[20]), "r"(v[21]), "r"(v[22]), "r"(v[23]),
                     "r"(v[24]), "r"(v[25]), "r"(v[26]), "r"(v[27]), "r"(v[28]), "r"(v[29]), "r"(v[30]), "r"(v[31]));
      asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
    }
  }
  __syncthreads();
  long long c1 = clock64();
  if (t == 0) cyc[blockIdx.x] = c1 - c0;
  if (acc == 12345.f) sink[t] = acc;
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tslot), "r"(512));
}

template <bool LD>
void run(int warps) {
  const int iters = 4096;
  long long* d;
  float* s;
  cudaMalloc(&d, 148 * 8);
  cudaMalloc(&s, 1024 * 4);
  k<LD><<<148, 32 * warps>>>(16, d, s);
  k<LD><<<148, 32 * warps>>>(iters, d, s);
  cudaError_t e = cudaDeviceSynchronize();
  long long h;
  cudaMemcpy(&h, d, 8, cudaMemcpyDeviceToHost);
  const double bytes = (double)iters * warps * 4096;
  printf("%s  %2d warps: %.1f B/clk/SM (%s)\n", LD ? "tcgen05.ld" : "tcgen05.st", warps, bytes / h, cudaGetErrorString(e));
  cudaFree(d);
  cudaFree(s);
}

int main() {
  for (int w : {4, 8, 16}) run<true>(w);
  for (int w : {4, 8, 16}) run<false>(w);
  return 0;
}
