// Prototype (not on the product path): the K2 column transform F[q] = sum_{y<n} x[y] W_N^{q (y - n/2)},
// n = 512, N = 4096, as two tensor-core GEMM stages with an error-free two-part fp16 split
// (hi*hi + hi*lo + lo*hi, fp32 accumulation in TMEM), to measure accuracy and speed of the
// "tensor-core column DFT" lever before building it into k2c_fwd.
//   y = j + 32 r, q = q0 + 128 q1, q0 = s + 8 k1:
//   stage A  D[(col,j)][q0] = sum_r x[j + 32 r] W_N^{32 s r} W_16^{k1 r}   (M 128 = 4 cols x 32 j,
//            K 32 real, N 256 real), then Y = D * W_N^{s (j - n/2)} W_n^{k1 (j - n/2)}
//   stage B  F[q0 + 128 q1] = sum_j W_32^{q1 j} Y[j][q0]                      (per column: M 128 q0,
//            K 64 real, N 64 real)
// usage: proto_tcfft [columns]   (prints max / rel-L2 error vs an fp64 DFT and the time per launch)
#include <cstdio>
#include <cstdint>
#include <cstdlib>
#include <cmath>
#include <vector>
#include <cuda_runtime.h>
#include <cuda_fp16.h>

constexpr int n = 512, N = 4096, J = 32, R = 16, Q0 = 128, NCOL = 4;   // 4 columns per group
constexpr int WPQ = 4, NTHR = 128 * WPQ;   // warps per TMEM lane quarter
// stage A operand tiles: A_A [128 rows][32 K] fp16, B_A [256 rows][32 K]; stage B: A_B per column
// [128 rows][64 K], B_B [64 rows][64 K].  No-swizzle K-major cores (8 rows x 16 B); K-adjacent
// cores LBO apart, row groups SBO apart.  LBO = 144 B (not a multiple of 128 B) so the transposed
// stage-B operand writes (lane = j -> K chunk j/4) land in distinct banks.
constexpr uint32_t LBO = 144;
constexpr uint32_t KA = 32, KB = 64;
constexpr uint32_t SBO_A = (KA / 8) * LBO, SBO_B = (KB / 8) * LBO;        // 576, 1152
constexpr uint32_t SZ_AA = 128 / 8 * SBO_A, SZ_BA = 256 / 8 * SBO_A;       // bytes per part
constexpr uint32_t SZ_AB = 128 / 8 * SBO_B, SZ_BB = 64 / 8 * SBO_B;

__host__ __device__ inline uint32_t off_k(uint32_t row, uint32_t k, uint32_t sbo) {
  return (row / 8) * sbo + (k / 8) * LBO + (row % 8) * 16 + (k % 8) * 2;
}
__device__ __forceinline__ uint32_t su32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ uint64_t desc(uint32_t a, uint32_t sbo) {
  return (uint64_t)((a >> 4) & 0x3FFF) | ((uint64_t)((LBO >> 4) & 0x3FFF) << 16) |
         ((uint64_t)((sbo >> 4) & 0x3FFF) << 32) | ((uint64_t)1 << 46);
}
__host__ __device__ constexpr uint32_t idesc_f16(int M, int Nn) {   // D f32, A/B f16, K-major
  return (1u << 4) | (0u << 7) | (0u << 10) | ((uint32_t)(Nn >> 3) << 17) | ((uint32_t)(M >> 4) << 24);
}
__device__ __forceinline__ void mma(uint32_t d, uint64_t a, uint64_t b, uint32_t idesc, bool acc) {
  asm volatile("{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\ntcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n}\n"
               ::"r"(d), "l"(a), "l"(b), "r"(idesc), "r"((uint32_t)acc));
}
__device__ __forceinline__ void commit_wait(uint64_t* bar, uint32_t& ph) {
  if (threadIdx.x == 0)
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(su32(bar)));
  asm volatile("{\n.reg .pred P1;\nW_%=:\nmbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n@!P1 bra W_%=;\n}\n"
               ::"r"(su32(bar)), "r"(ph) : "memory");
  ph ^= 1;
}
__device__ __forceinline__ void ld32(uint32_t ta, float* v) {
  uint32_t* u = reinterpret_cast<uint32_t*>(v);
  asm volatile("tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
               "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
               : "=r"(u[0]), "=r"(u[1]), "=r"(u[2]), "=r"(u[3]), "=r"(u[4]), "=r"(u[5]), "=r"(u[6]), "=r"(u[7]),
                 "=r"(u[8]), "=r"(u[9]), "=r"(u[10]), "=r"(u[11]), "=r"(u[12]), "=r"(u[13]), "=r"(u[14]), "=r"(u[15]),
                 "=r"(u[16]), "=r"(u[17]), "=r"(u[18]), "=r"(u[19]), "=r"(u[20]), "=r"(u[21]), "=r"(u[22]), "=r"(u[23]),
                 "=r"(u[24]), "=r"(u[25]), "=r"(u[26]), "=r"(u[27]), "=r"(u[28]), "=r"(u[29]), "=r"(u[30]), "=r"(u[31])
               : "r"(ta));
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
}
// x = hi + lo, both fp16 (x pre-scaled into fp16's normal range)
__device__ __forceinline__ void split(float x, __half& hi, __half& lo) {
  hi = __float2half_rn(x);
  lo = __float2half_rn(x - __half2float(hi));
}
// the same for a complex value with packed conversions (cvt.rn.f16x2.f32)
__device__ __forceinline__ void split2(float re, float im, __half2& hi, __half2& lo) {
  hi = __floats2half2_rn(re, im);
  const float2 b = __half22float2(hi);
  lo = __floats2half2_rn(re - b.x, im - b.y);
}

__global__ void __launch_bounds__(NTHR, 1) tcfft(const float2* __restrict__ x, float2* __restrict__ F, int ncols,
                                               const unsigned char* __restrict__ gB, const float2* __restrict__ tw,
                                               int write_out, float* __restrict__ chk) {
  extern __shared__ __align__(1024) unsigned char sm[];
  unsigned char* BA = sm;                              // hi, lo
  unsigned char* BB = BA + 2 * SZ_BA;                  // hi, lo
  unsigned char* AA = BB + 2 * SZ_BB;                  // hi, lo
  unsigned char* AB = AA + 2 * SZ_AA;                  // [4 cols][hi, lo]
  const float2* wtab = tw;   // W_N^m, m < N (32 KB, L1-resident)
  uint64_t* bar = reinterpret_cast<uint64_t*>(AB + NCOL * 2 * SZ_AB);
  uint32_t* tslot = reinterpret_cast<uint32_t*>(bar + 1);
  const int t = threadIdx.x, warp = t >> 5, lane = t & 31, quarter = warp & 3, sub = warp >> 2;
  for (uint32_t i = t * 16; i < 2 * SZ_BA + 2 * SZ_BB; i += NTHR * 16)
    *reinterpret_cast<uint4*>(sm + i) = *reinterpret_cast<const uint4*>(gB + i);
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(su32(tslot)), "r"(512));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  if (t == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(bar)));
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t tmem = *tslot, tq = tmem + ((uint32_t)(32 * quarter) << 16);
  uint32_t ph = 0;
  float csum = 0.f;
  // per-thread twiddle factors (lane = j; this warp's q0 = 16 a + b with a in {2 sub, 2 sub + 1}):
  // W_N^{q0 (j - n/2)} = P[b] Q[a - 2 sub], P[b] = W_N^{b (j - n/2)}, Q = W_N^{16 a (j - n/2)}
  float2 Pw[16], Qw[2];
  {
    const int jm = lane - n / 2;
#pragma unroll
    for (int b = 0; b < 16; ++b) Pw[b] = __ldg(&wtab[(b * jm + 64 * N) & (N - 1)]);
#pragma unroll
    for (int c = 0; c < 2; ++c) Qw[c] = __ldg(&wtab[(16 * (2 * sub + c) * jm + 64 * N) & (N - 1)]);
  }
  constexpr uint32_t IA = idesc_f16(128, 256), IB = idesc_f16(128, 64);
  // software pipeline: MMA B(g) and MMA A(g+1) run back to back while the threads prefetch
  // x(g+2) and then read out F(g); the twiddle phase of g+1 finds A(g+1) done
  uint64_t* barA = bar;                                   // stage-A MMAs retired
  uint64_t* barB = bar + 16;                              // stage-B MMAs retired (byte 128)
  float* red = reinterpret_cast<float*>(bar + 2) + 8;     // [16] per-warp maxima
  float* isBv = reinterpret_cast<float*>(bar + 2);        // [4] 1 / sB per column
  uint32_t phA = 0, phB = 0;
  const int G = ncols / NCOL;
  auto load_x = [&](int gg, float2 (&v)[4]) {
    if (gg < G) {
      const float2* xc = x + (size_t)(gg * NCOL + quarter) * n;
#pragma unroll
      for (int r = 0; r < 4; ++r) v[r] = __ldg(&xc[lane + J * (4 * sub + r)]);
    }
  };
  // column scale (reduced over the 4 warps of the quarter) and the stage-A operand of group gg
  auto put_a = [&](const float2 (&v)[4]) -> float {
    float mx = 0.f;
#pragma unroll
    for (int r = 0; r < 4; ++r) mx = fmaxf(mx, fmaxf(fabsf(v[r].x), fabsf(v[r].y)));
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) mx = fmaxf(mx, __shfl_xor_sync(~0u, mx, o));
    if (lane == 0) red[warp] = mx;
    asm volatile("bar.sync 1, %0;" ::"n"(NTHR) : "memory");
    mx = fmaxf(fmaxf(red[quarter], red[quarter + 4]), fmaxf(red[quarter + 8], red[quarter + 12]));
    int ea;
    frexpf(mx > 0.f ? mx : 1.f, &ea);
    const float sA = ldexpf(1.f, 14 - ea);
    __half2 h[4], l[4];
#pragma unroll
    for (int r = 0; r < 4; ++r) split2(v[r].x * sA, v[r].y * sA, h[r], l[r]);
    const int row = 32 * quarter + lane;
    *reinterpret_cast<uint4*>(AA + off_k(row, 8 * sub, SBO_A)) = *reinterpret_cast<uint4*>(h);
    *reinterpret_cast<uint4*>(AA + SZ_AA + off_k(row, 8 * sub, SBO_A)) = *reinterpret_cast<uint4*>(l);
    return ldexpf(1.f, ea - 14);   // 1 / sA
  };
  auto mma_a = [&]() {
    asm volatile("tcgen05.fence::after_thread_sync;");
    const uint32_t ah = su32(AA), al = ah + SZ_AA, bh = su32(BA), bl = bh + SZ_BA;
#pragma unroll
    for (int k = 0; k < 2; ++k) {
      const uint32_t o = k * 2 * LBO;
      mma(tmem, desc(ah + o, SBO_A), desc(bh + o, SBO_A), IA, k > 0);
      mma(tmem, desc(ah + o, SBO_A), desc(bl + o, SBO_A), IA, true);
      mma(tmem, desc(al + o, SBO_A), desc(bh + o, SBO_A), IA, true);
    }
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(su32(barA)));
  };
  auto wait = [&](uint64_t* b, uint32_t& ph) {
    asm volatile("{\n.reg .pred P1;\nW_%=:\nmbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n@!P1 bra W_%=;\n}\n"
                 ::"r"(su32(b)), "r"(ph) : "memory");
    ph ^= 1;
  };
  if (t == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(barB)));
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  __syncthreads();
  int g = blockIdx.x;
  float2 vn[4];
  float isA = 1.f;
  if (g < G) {
    load_x(g, vn);
    isA = put_a(vn);
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    __syncthreads();
    if (t == 0) mma_a();
    load_x(g + gridDim.x, vn);
  }
  for (; g < G; g += gridDim.x) {
    wait(barA, phA);
    asm volatile("tcgen05.fence::after_thread_sync;");
    // ---- twiddle, rescale, transpose into the stage-B operand of column `quarter`
    {
      const int j = lane;
      const float sBr = 1.f / 16.f;   // D is in units of sA: x sA / 16 keeps |Y| in fp16's range
      unsigned char* ab = AB + quarter * 2 * SZ_AB;
#pragma unroll
      for (int cb = 0; cb < 2; ++cb) {
        float d[32];
        ld32(tq + (2 * sub + cb) * 32, d);
#pragma unroll
        for (int e = 0; e < 16; ++e) {
          const int q0 = (2 * sub + cb) * 16 + e;
          const float2 w = make_float2(Pw[e].x * Qw[cb].x - Pw[e].y * Qw[cb].y, Pw[e].x * Qw[cb].y + Pw[e].y * Qw[cb].x);
          const float re = d[2 * e] * sBr, im = d[2 * e + 1] * sBr;
          __half2 hi, lo;
          split2(re * w.x - im * w.y, re * w.y + im * w.x, hi, lo);
          const uint32_t o = off_k(q0, 2 * j, SBO_B);
          *reinterpret_cast<__half2*>(ab + o) = hi;
          *reinterpret_cast<__half2*>(ab + SZ_AB + o) = lo;
        }
      }
      if (lane == 0 && sub == 0) isBv[quarter] = 16.f * isA;   // 1 / sB
    }
    // ---- stage-A operand of the next group (AA is free: A(g) retired)
    const bool more = g + (int)gridDim.x < G;
    float isA_next = 1.f;
    if (more) isA_next = put_a(vn);
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    if (t == 0) {
      asm volatile("tcgen05.fence::after_thread_sync;");
      const uint32_t bh = su32(BB), bl = bh + SZ_BB;
      for (int c = 0; c < NCOL; ++c) {
        const uint32_t ah = su32(AB + c * 2 * SZ_AB), al = ah + SZ_AB, dd = tmem + 256 + 64 * c;
#pragma unroll
        for (int k = 0; k < 4; ++k) {
          const uint32_t o = k * 2 * LBO;
          mma(dd, desc(ah + o, SBO_B), desc(bh + o, SBO_B), IB, k > 0);
          mma(dd, desc(ah + o, SBO_B), desc(bl + o, SBO_B), IB, true);
          mma(dd, desc(al + o, SBO_B), desc(bh + o, SBO_B), IB, true);
        }
      }
      asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(su32(barB)));
      if (more) mma_a();   // A(g+1): its TMEM columns were read out above
    }
    if (more) load_x(g + 2 * (int)gridDim.x, vn);
    wait(barB, phB);
    asm volatile("tcgen05.fence::after_thread_sync;");
    // ---- output: lane q0 = 32 quarter + lane; warp `sub` reads column sub, q1 = 0..31
    {
      const int c = sub;
      const float isB = isBv[c];
      const int q0 = 32 * quarter + lane, colc = g * NCOL + c;
#pragma unroll
      for (int cb = 0; cb < 2; ++cb) {
        float d[32];
        ld32(tq + 256 + 64 * c + 32 * cb, d);
#pragma unroll
        for (int e = 0; e < 16; ++e) {
          const int q1 = cb * 16 + e;
          const float2 f = make_float2(d[2 * e] * isB, d[2 * e + 1] * isB);
          if (write_out) F[(size_t)colc * N + q0 + Q0 * q1] = f;
          else csum += f.x + f.y;
        }
      }
    }
    isA = isA_next;
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();   // AB / TMEM-B / isBv reused by the next group
  }
  if (chk) chk[blockIdx.x * NTHR + t] = csum;
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(512));
}

int main(int argc, char** argv) {
  setvbuf(stdout, nullptr, _IONBF, 0);
  const int ncols = argc > 1 ? atoi(argv[1]) : 32768;
  const double PI = 3.14159265358979323846;
  // ---- tables
  std::vector<unsigned char> hB(2 * SZ_BA + 2 * SZ_BB, 0);
  auto put = [&](unsigned char* base, uint32_t sz, uint32_t sbo, int row, int k, double val) {
    const __half h = __float2half_rn((float)val);
    const __half l = __float2half_rn((float)(val - (double)__half2float(h)));
    *reinterpret_cast<__half*>(base + off_k(row, k, sbo)) = h;
    *reinterpret_cast<__half*>(base + sz + off_k(row, k, sbo)) = l;
  };
  // B_A: row n = 2 q0 + d (d: re / im of output), K k = 2 r + c (c: re / im of input)
  for (int q0 = 0; q0 < Q0; ++q0) {
    const int s = q0 % 8, k1 = q0 / 8;
    for (int r = 0; r < R; ++r) {
      const double a = -2 * PI * ((double)(32 * s * r) / N + (double)(k1 * r) / R);
      const double cr = cos(a), ci = sin(a);
      put(hB.data(), SZ_BA, SBO_A, 2 * q0, 2 * r, cr);       // re out <- re in
      put(hB.data(), SZ_BA, SBO_A, 2 * q0, 2 * r + 1, -ci);  // re out <- im in
      put(hB.data(), SZ_BA, SBO_A, 2 * q0 + 1, 2 * r, ci);   // im out <- re in
      put(hB.data(), SZ_BA, SBO_A, 2 * q0 + 1, 2 * r + 1, cr);
    }
  }
  unsigned char* hBB = hB.data() + 2 * SZ_BA;
  for (int q1 = 0; q1 < 32; ++q1)
    for (int j = 0; j < J; ++j) {
      const double a = -2 * PI * (double)(q1 * j) / 32;
      const double cr = cos(a), ci = sin(a);
      put(hBB, SZ_BB, SBO_B, 2 * q1, 2 * j, cr);
      put(hBB, SZ_BB, SBO_B, 2 * q1, 2 * j + 1, -ci);
      put(hBB, SZ_BB, SBO_B, 2 * q1 + 1, 2 * j, ci);
      put(hBB, SZ_BB, SBO_B, 2 * q1 + 1, 2 * j + 1, cr);
    }
  std::vector<float2> htw(N);   // W_N^m: the stage-A twiddle W_N^{s (j - n/2)} W_n^{k1 (j - n/2)} = W_N^{q0 (j - n/2)}
  for (int m = 0; m < N; ++m) htw[m] = make_float2((float)cos(-2 * PI * m / N), (float)sin(-2 * PI * m / N));
  // ---- input: smooth-ish spectra with dynamic range (decay along y, random phases)
  std::vector<float2> hx((size_t)ncols * n);
  srand(1);
  for (int c = 0; c < ncols; ++c) {
    const double amp = pow(10.0, -3.0 * (c % 7) / 6.0);
    for (int y = 0; y < n; ++y) {
      const double env = exp(-fabs(y - n / 2) / 90.0);
      hx[(size_t)c * n + y] = make_float2((float)(amp * env * (rand() / (double)RAND_MAX - 0.5)),
                                          (float)(amp * env * (rand() / (double)RAND_MAX - 0.5)));
    }
  }
  float2 *dx, *dF, *dtw;
  unsigned char* dB;
  float* dchk;
  cudaMalloc(&dx, hx.size() * 8);
  cudaMalloc(&dF, (size_t)ncols * N * 8);
  cudaMalloc(&dtw, htw.size() * 8);
  cudaMalloc(&dB, hB.size());
  cudaMalloc(&dchk, 148 * NTHR * 4);
  cudaMemcpy(dx, hx.data(), hx.size() * 8, cudaMemcpyHostToDevice);
  cudaMemcpy(dtw, htw.data(), htw.size() * 8, cudaMemcpyHostToDevice);
  cudaMemcpy(dB, hB.data(), hB.size(), cudaMemcpyHostToDevice);
  const size_t smem = 2 * SZ_BA + 2 * SZ_BB + 2 * SZ_AA + NCOL * 2 * SZ_AB + 512;
  cudaFuncSetAttribute(tcfft, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  printf("smem %zu B\n", smem);
  tcfft<<<148, NTHR, smem>>>(dx, dF, ncols, dB, dtw, 1, nullptr);
  cudaError_t e = cudaDeviceSynchronize();
  printf("run: %s\n", cudaGetErrorString(e));
  if (e != cudaSuccess) return 1;
  // ---- accuracy on sampled columns vs fp64
  std::vector<float2> hF(N);
  double emax = 0, num = 0, den = 0, gmax = 0;
  for (int c : {0, 1, 5, 6, 123, ncols / 2 + 3, ncols - 1}) {
    cudaMemcpy(hF.data(), dF + (size_t)c * N, N * 8, cudaMemcpyDeviceToHost);
    for (int q = 0; q < N; ++q) {
      double sr = 0, si = 0;
      for (int y = 0; y < n; ++y) {
        const long ph = ((long)q * (y - n / 2)) % N;
        const double a = -2 * PI * (double)ph / N;
        const float2 xv = hx[(size_t)c * n + y];
        sr += xv.x * cos(a) - xv.y * sin(a);
        si += xv.x * sin(a) + xv.y * cos(a);
      }
      const double dr = hF[q].x - sr, di = hF[q].y - si;
      num += dr * dr + di * di;
      den += sr * sr + si * si;
      emax = fmax(emax, fmax(fabs(dr), fabs(di)));
      gmax = fmax(gmax, fmax(fabs(sr), fabs(si)));
    }
  }
  printf("sampled columns: rel-L2 %.3e, max|err|/max|F| %.3e\n", sqrt(num / den), emax / gmax);
  // ---- timing (no output write)
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  for (int i = 0; i < 3; ++i) tcfft<<<148, NTHR, smem>>>(dx, dF, ncols, dB, dtw, 0, dchk);
  cudaEventRecord(e0);
  const int reps = 10;
  for (int i = 0; i < reps; ++i) tcfft<<<148, NTHR, smem>>>(dx, dF, ncols, dB, dtw, 0, dchk);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms;
  cudaEventElapsedTime(&ms, e0, e1);
  printf("%d columns: %.1f us per launch (%s)\n", ncols, 1000.0 * ms / reps, cudaGetErrorString(cudaGetLastError()));
  return 0;
}
