// The four oversampled-DFT kernels (the O(n^2 log n) "2D FFT" of Alg. 1 steps 1-3 and
// Alg. 2 steps 5-7), built on the residue FFT engine:
//
//   K1   f [B][n][n]        -> S1 [B][N/2+1][n]   row DFT (pairs of real rows packed)
//   K2   S1                 -> S2 [B][n_phi/2][NL] column DFT + bilinear gather to polar nodes
//   K2T  S2                 -> S1                  transposed gather (CSR) + inverse column DFT
//   K1T  S1                 -> f                   inverse row DFT (Hermitian completion)
//
// S1 is column-major ([p][y]) so K2/K2T read and write whole columns contiguously.
#include "fft_engine.cuh"
#include "tat_internal.h"

namespace tat {

using namespace fe;

constexpr int kStrip = 16;   // K2: columns per CTA (sliding window, one halo column recomputed)

// ------------------------------------------------------------------ helpers
// Per-residue-group barrier: a group is the n/8 threads of one residue transform.
template <int n>
__device__ __forceinline__ void gsync(int g, int L) {
  if constexpr (n / 8 <= 32) {
    __syncwarp();
  } else {
    if (L <= 15) named_bar(1 + g, n / 8);
    else __syncthreads();
  }
}

// Passes 1..P-1 of one residue transform (pass-0 output in b0), twiddles generated on the fly.
// WLAST: write the last pass (natural order) to smem; returns 0 if it lands in b0, 1 if in b1.
template <int n, int S, bool WLAST>
__device__ __forceinline__ int passes_g(float2 (&v)[8], float2* b0, float2* b1, int j, int g, int L,
                                        const float2* __restrict__ tw_n) {
  constexpr int P = Plan<n>::P;
  gsync<n>(g, L);
  pass_g<n, 1, S, true, (P > 2) || WLAST>(v, b0, b1, j, tw_n);
  if constexpr (P > 2) {
    gsync<n>(g, L);
    pass_g<n, 2, S, true, (P > 3) || WLAST>(v, b1, b0, j, tw_n);
  }
  if constexpr (P > 3) {
    gsync<n>(g, L);
    pass_g<n, 3, S, true, WLAST>(v, b0, b1, j, tw_n);
  }
  return (P - 1) & 1;
}

// ================================================================== K2 forward
// One thread = one radix-8 butterfly of one residue (blockDim = L n / 8).  Strip of kStrip
// columns with a sliding window of two column spectra; S2 is written in node order (contiguous).
template <int n>
__global__ void __launch_bounds__(1024) k2_fwd(DevPlan P) {
  extern __shared__ float2 sm[];
  const Consts& C = P.C;
  constexpr int pn = padded(n);
  const int L = C.Lres, ln = L * pn, N = C.N;
  const int b = blockIdx.y;
  const int P0 = blockIdx.x * kStrip;
  const int Pend = min(P0 + kStrip, C.ncols);
  const int plast = min(Pend, C.ncols - 1);
  const int g = threadIdx.x / (n / 8), j = threadIdx.x % (n / 8);
  const int so = g * pn;
  float2 pre[8];
#pragma unroll
  for (int r = 0; r < 8; ++r) pre[r] = __ldg(&P.tw_pre[g * n + j + r * (n / 8)]);
  const float2* S1 = P.S1 + (size_t)b * C.ncols * n;
  float2* S2 = P.S2 + (size_t)b * C.half * C.NL;
  int prev = 2;
  for (int p = P0; p <= plast; ++p) {
    const float2* col = S1 + (size_t)p * n;
    float2 v[8];
    // FFT slot y' = j + r n/8 holds sample y = (y' + n/2) mod n
#pragma unroll
    for (int r = 0; r < 8; ++r)
      v[r] = cmul(__ldg(&col[j + (r < 4 ? n / 2 + r * (n / 8) : (r - 4) * (n / 8))]), pre[r]);
    const int i0 = prev == 0 ? 1 : 0, i1 = prev == 2 ? 1 : 2;
    float2* X = sm + i0 * ln;
    float2* Y = sm + i1 * ln;
    pass_g<n, 0, -1, false, true>(v, nullptr, X + so, j, P.tw_n);
    const int cur = passes_g<n, -1, true>(v, X + so, Y + so, j, g, L, P.tw_n) ? i1 : i0;
    __syncthreads();
    if (p > P0) {
      const float2* Xa = sm + prev * ln;
      const float2* Xb = sm + cur * ln;
      const int e1 = P.k2_colptr[p];
      for (int e = P.k2_colptr[p - 1] + threadIdx.x; e < e1; e += blockDim.x) {
        const int4 nd = __ldg(&P.k2_nodes[e]);
        const float a = __int_as_float(nd.z), bb = __int_as_float(nd.w);
        const int q0 = nd.y & (N - 1), q1 = (nd.y + 1) & (N - 1);
        const int i00 = (q0 & (L - 1)) * pn + phys(q0 / L);
        const int i01 = (q1 & (L - 1)) * pn + phys(q1 / L);
        const float2 f00 = Xa[i00], f01 = Xa[i01], f10 = Xb[i00], f11 = Xb[i01];
        const float2 c0 = __ffma2_rn(make_float2(a, a), csub(f10, f00), f00);
        const float2 c1 = __ffma2_rn(make_float2(a, a), csub(f11, f01), f01);
        S2[e] = __ffma2_rn(make_float2(bb, bb), csub(c1, c0), c0);
      }
      __syncthreads();
    }
    prev = cur;
  }
  if (Pend == C.ncols) {   // p0 = N/2: alpha == 0, only F[N/2] is used
    const float2* Xa = sm + prev * ln;
    for (int e = P.k2_colptr[C.ncols - 1] + threadIdx.x; e < P.k2_colptr[C.ncols]; e += blockDim.x) {
      const int4 nd = __ldg(&P.k2_nodes[e]);
      const float bb = __int_as_float(nd.w);
      const int q0 = nd.y & (N - 1), q1 = (nd.y + 1) & (N - 1);
      const float2 f00 = Xa[(q0 & (L - 1)) * pn + phys(q0 / L)];
      const float2 f01 = Xa[(q1 & (L - 1)) * pn + phys(q1 / L)];
      S2[e] = __ffma2_rn(make_float2(bb, bb), csub(f01, f00), f00);
    }
  }
}

// ================================================================== K1 forward (row pairs)
// z = f_y + i f_{y+1}; Z[p] = sum_x z e^{-2 pi i p (x-n/2)/N}; two row pairs per CTA so that
// each p writes one full 32-byte sector S1[p][y0..y0+3].
template <int n>
__global__ void __launch_bounds__(1024) k1_fwd(DevPlan P, const float* __restrict__ f) {
  extern __shared__ float2 sm[];
  const Consts& C = P.C;
  constexpr int pn = padded(n);
  const int L = C.Lres, ln = L * pn, N = C.N;
  const int b = blockIdx.y, y0 = 4 * blockIdx.x;
  const int g = threadIdx.x / (n / 8), j = threadIdx.x % (n / 8);
  const int so = g * pn;
  float2 pre[8];
#pragma unroll
  for (int r = 0; r < 8; ++r) pre[r] = __ldg(&P.tw_pre[g * n + j + r * (n / 8)]);
  float2* ZA = nullptr;
  float2* ZB = nullptr;
#pragma unroll 1
  for (int pr = 0; pr < 2; ++pr) {
    const float* r0 = f + ((size_t)b * n + y0 + 2 * pr) * n;
    float2 v[8];
#pragma unroll
    for (int r = 0; r < 8; ++r) {
      const int xi = j + (r < 4 ? n / 2 + r * (n / 8) : (r - 4) * (n / 8));
      v[r] = cmul(make_float2(__ldg(&r0[xi]), __ldg(&r0[n + xi])), pre[r]);
    }
    float2* b0 = pr == 0 ? sm : sm + 2 * ln;
    float2* b1 = pr == 0 ? sm + ln : (ZA == sm ? sm + ln : sm);
    pass_g<n, 0, -1, false, true>(v, nullptr, b0 + so, j, P.tw_n);
    const int fin = passes_g<n, -1, true>(v, b0 + so, b1 + so, j, g, L, P.tw_n);
    if (pr == 0) ZA = fin ? b1 : b0;
    else ZB = fin ? b1 : b0;
  }
  __syncthreads();
  float4* out = reinterpret_cast<float4*>(P.S1 + (size_t)b * C.ncols * n);
  for (int p = threadIdx.x; p < C.ncols; p += blockDim.x) {
    const int pm = (N - p) & (N - 1);
    const int ip = (p & (L - 1)) * pn + phys(p / L);
    const int im = (pm & (L - 1)) * pn + phys(pm / L);
    const float2 za = ZA[ip], zam = ZA[im], zb = ZB[ip], zbm = ZB[im];
    // row y: (Z[p] + conj Z[-p]) / 2 ; row y+1: (Z[p] - conj Z[-p]) / (2 i)
    float4 o0, o1;
    o0.x = 0.5f * (za.x + zam.x); o0.y = 0.5f * (za.y - zam.y);
    o0.z = 0.5f * (za.y + zam.y); o0.w = -0.5f * (za.x - zam.x);
    o1.x = 0.5f * (zb.x + zbm.x); o1.y = 0.5f * (zb.y - zbm.y);
    o1.z = 0.5f * (zb.y + zbm.y); o1.w = -0.5f * (zb.x - zbm.x);
    float4* dst = out + (((size_t)p * n + y0) >> 1);
    dst[0] = o0;
    dst[1] = o1;
  }
}

// ================================================================== K2T (transpose of K2)
// Column p: R[q] = sum_{CSR} w P~ (fixed order), L inverse residue FFTs, then
// S~1[p][y] = sum_s X_s[y'] conj(W_N^{s y''}), the residue sum reduced through smem.
template <int n>
__global__ void __launch_bounds__(1024) k2t_adj(DevPlan P) {
  extern __shared__ float2 sm[];
  const Consts& C = P.C;
  constexpr int pn = padded(n);
  const int L = C.Lres, ln = L * pn;
  const int b = blockIdx.y;
  const int P0 = blockIdx.x * kStrip;
  const int Pend = min(P0 + kStrip, C.ncols);
  const int g = threadIdx.x / (n / 8), j = threadIdx.x % (n / 8);
  const int so = g * pn;
  float2 post[8];
#pragma unroll
  for (int e = 0; e < 8; ++e) post[e] = __ldg(&P.tw_pre[g * n + last_pos<n>(j, e)]);
  const float2* S2 = P.S2 + (size_t)b * C.half * C.NL;
  float2* out = P.S1 + (size_t)b * C.ncols * n;
  float2* R = sm;            // gather target (kept zero outside the CSR targets)
  float2* Xb = sm + ln;      // ping-pong
  float2* red = sm + 2 * ln; // ping-pong partner, then residue-sum staging [L][n]
  for (int i = threadIdx.x; i < ln; i += blockDim.x) R[i] = make_float2(0.f, 0.f);
  __syncthreads();
  for (int p = P0; p < Pend; ++p) {
    for (int t = P.k2t_colptr[p] + threadIdx.x; t < P.k2t_colptr[p + 1]; t += blockDim.x) {
      const int qm = __ldg(&P.k2t_tq[t]);
      float2 acc = make_float2(0.f, 0.f);
      const int e1 = __ldg(&P.k2t_tstart[t + 1]);
      for (int e = __ldg(&P.k2t_tstart[t]); e < e1; ++e) {
        const int2 en = __ldg(&P.k2t_ent[e]);
        acc = __ffma2_rn(make_float2(__int_as_float(en.y), __int_as_float(en.y)), __ldg(&S2[en.x]), acc);
      }
      R[(qm & (L - 1)) * pn + phys(qm / L)] = acc;
    }
    __syncthreads();
    float2 v[8];
    // pass 0 reads R and re-zeroes what it read (each element is read by exactly one thread)
    {
      float2* a = R + so + phys(j);
#pragma unroll
      for (int r = 0; r < 8; ++r) {
        v[r] = a[r * (n / 8) + ((r * (n / 8)) >> 4)];
        a[r * (n / 8) + ((r * (n / 8)) >> 4)] = make_float2(0.f, 0.f);
      }
    }
    pass_g<n, 0, 1, false, true>(v, nullptr, Xb + so, j, P.tw_n);
    passes_g<n, 1, false>(v, Xb + so, red + so, j, g, L, P.tw_n);   // result in registers
    __syncthreads();   // every group is done with `red` as scratch
#pragma unroll
    for (int e = 0; e < 8; ++e) red[so + last_pos<n>(j, e)] = cmulc(v[e], post[e]);
    __syncthreads();
    for (int yp = threadIdx.x; yp < n; yp += blockDim.x) {
      float2 acc = red[yp];
      for (int gg = 1; gg < L; ++gg) acc = cadd(acc, red[gg * pn + yp]);
      out[(size_t)p * n + ((yp + n / 2) & (n - 1))] = acc;
    }
    __syncthreads();
  }
}

// ================================================================== K1T (transpose of K1)
// Two row pairs per CTA: Z[p] = C_y[p] + i C_{y+1}[p] (Hermitian completion of the half
// spectra, C[0], C[N/2] = 2 Re), inverse residue FFTs, residue sum -> f~ rows.
template <int n>
__global__ void __launch_bounds__(1024) k1t_adj(DevPlan P, float* __restrict__ fout) {
  extern __shared__ float2 sm[];
  const Consts& C = P.C;
  constexpr int pn = padded(n);
  const int L = C.Lres, ln = L * pn, N = C.N;
  const int b = blockIdx.y, y0 = 4 * blockIdx.x;
  const int g = threadIdx.x / (n / 8), j = threadIdx.x % (n / 8);
  const int so = g * pn;
  float2 post[8];
#pragma unroll
  for (int e = 0; e < 8; ++e) post[e] = __ldg(&P.tw_pre[g * n + last_pos<n>(j, e)]);
  float2* ZA = sm;
  float2* ZB = sm + ln;
  float2* X = sm + 2 * ln;
  const float4* in = reinterpret_cast<const float4*>(P.S1 + (size_t)b * C.ncols * n);
  for (int p = threadIdx.x; p < C.ncols; p += blockDim.x) {
    const float4* src = in + (((size_t)p * n + y0) >> 1);
    const float4 v0 = src[0], v1 = src[1];   // rows y0, y0+1 | y0+2, y0+3
    const int ip = (p & (L - 1)) * pn + phys(p / L);
    if (p == 0 || p == N / 2) {
      ZA[ip] = make_float2(2.f * v0.x, 2.f * v0.z);
      ZB[ip] = make_float2(2.f * v1.x, 2.f * v1.z);
    } else {
      const int pm = N - p;
      const int im = (pm & (L - 1)) * pn + phys(pm / L);
      ZA[ip] = make_float2(v0.x - v0.w, v0.y + v0.z);
      ZA[im] = make_float2(v0.x + v0.w, -v0.y + v0.z);
      ZB[ip] = make_float2(v1.x - v1.w, v1.y + v1.z);
      ZB[im] = make_float2(v1.x + v1.w, -v1.y + v1.z);
    }
  }
  __syncthreads();
#pragma unroll 1
  for (int pr = 0; pr < 2; ++pr) {
    float2* Zs = pr ? ZB : ZA;
    float2 v[8];
    pass_g<n, 0, 1, true, true>(v, Zs + so, X + so, j, P.tw_n);
    passes_g<n, 1, false>(v, X + so, Zs + so, j, g, L, P.tw_n);
    __syncthreads();
    float2* red = Zs;   // free now (results are in registers)
#pragma unroll
    for (int e = 0; e < 8; ++e) red[so + last_pos<n>(j, e)] = cmulc(v[e], post[e]);
    __syncthreads();
    float* o = fout + ((size_t)b * n + y0 + 2 * pr) * n;
    for (int xp = threadIdx.x; xp < n; xp += blockDim.x) {
      float2 acc = red[xp];
      for (int gg = 1; gg < L; ++gg) acc = cadd(acc, red[gg * pn + xp]);
      const int x = (xp + n / 2) & (n - 1);
      o[x] = acc.x;
      o[n + x] = acc.y;
    }
    __syncthreads();
  }
}

// ================================================================== dispatch
size_t smem_fft4(const Consts& C) { return (size_t)3 * C.Lres * (C.n + C.n / 16) * sizeof(float2); }
int fft_threads(const Consts& C) { return C.Lres * (C.n / 8); }

template <int n>
static cudaError_t cfg_one() {
  cudaError_t e = cudaSuccess;
  const int big = 3 * 16 * padded(n) * (int)sizeof(float2);
  const int lim = big > 227 * 1024 ? 227 * 1024 : big;
  if (e == cudaSuccess) e = cudaFuncSetAttribute(k2_fwd<n>, cudaFuncAttributeMaxDynamicSharedMemorySize, lim);
  if (e == cudaSuccess) e = cudaFuncSetAttribute(k1_fwd<n>, cudaFuncAttributeMaxDynamicSharedMemorySize, lim);
  if (e == cudaSuccess) e = cudaFuncSetAttribute(k2t_adj<n>, cudaFuncAttributeMaxDynamicSharedMemorySize, lim);
  if (e == cudaSuccess) e = cudaFuncSetAttribute(k1t_adj<n>, cudaFuncAttributeMaxDynamicSharedMemorySize, lim);
  return e;
}

#define TAT_DISPATCH_N(...)                                    \
  switch (C.n) {                                               \
    case 32: { constexpr int NN = 32; __VA_ARGS__; } break;    \
    case 64: { constexpr int NN = 64; __VA_ARGS__; } break;    \
    case 128: { constexpr int NN = 128; __VA_ARGS__; } break;  \
    case 256: { constexpr int NN = 256; __VA_ARGS__; } break;  \
    case 512: { constexpr int NN = 512; __VA_ARGS__; } break;  \
    case 1024: { constexpr int NN = 1024; __VA_ARGS__; } break; \
    default: return cudaErrorInvalidValue;                     \
  }

cudaError_t configure_fft_kernels(const Consts& C) {
  TAT_DISPATCH_N(return cfg_one<NN>());
  return cudaSuccess;
}

cudaError_t launch_k1(const DevPlan& P, const float* f, cudaStream_t s) {
  const Consts& C = P.C;
  const dim3 grid(C.n / 4, C.batch);
  TAT_DISPATCH_N(k1_fwd<NN><<<grid, fft_threads(C), smem_fft4(C), s>>>(P, f));
  return cudaGetLastError();
}
cudaError_t launch_k2(const DevPlan& P, cudaStream_t s) {
  const Consts& C = P.C;
  const dim3 grid((C.ncols + kStrip - 1) / kStrip, C.batch);
  TAT_DISPATCH_N(k2_fwd<NN><<<grid, fft_threads(C), smem_fft4(C), s>>>(P));
  return cudaGetLastError();
}
cudaError_t launch_k2t(const DevPlan& P, cudaStream_t s) {
  const Consts& C = P.C;
  const dim3 grid((C.ncols + kStrip - 1) / kStrip, C.batch);
  TAT_DISPATCH_N(k2t_adj<NN><<<grid, fft_threads(C), smem_fft4(C), s>>>(P));
  return cudaGetLastError();
}
cudaError_t launch_k1t(const DevPlan& P, float* f, cudaStream_t s) {
  const Consts& C = P.C;
  const dim3 grid(C.n / 4, C.batch);
  TAT_DISPATCH_N(k1t_adj<NN><<<grid, fft_threads(C), smem_fft4(C), s>>>(P, f));
  return cudaGetLastError();
}

}  // namespace tat
