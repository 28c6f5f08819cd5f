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

template <int n>
struct Geo {
  static constexpr int T8 = n / 8;   // threads per residue FFT
};

// ------------------------------------------------------------------ helpers
// Run passes 1..P-1 of the thread's residues, ping-ponging between b0 (holding the pass-0
// output) and b1.  WLAST: write the last pass to smem (forward); otherwise the result stays in
// registers at positions last_pos<n>(j, e).  Returns 0 if a written result ends in b0, 1 if in
// b1.  Starts and ends with __syncthreads().
template <int n, int S, int RPT, bool WLAST>
__device__ __forceinline__ int passes_rest(float2 (&v)[RPT][8], float2* b0, float2* b1,
                                           const int (&soff)[RPT], int j, const PassTw<n, S>& T) {
  constexpr int P = Plan<n>::P;
  __syncthreads();
#pragma unroll
  for (int i = 0; i < RPT; ++i)
    pass<n, 1, S, true, (P > 2) || WLAST>(v[i], b0 + soff[i], b1 + soff[i], j, T.tw[0]);
  __syncthreads();
  if constexpr (P > 2) {
#pragma unroll
    for (int i = 0; i < RPT; ++i)
      pass<n, 2, S, true, (P > 3) || WLAST>(v[i], b1 + soff[i], b0 + soff[i], j, T.tw[1]);
    __syncthreads();
  }
  if constexpr (P > 3) {
#pragma unroll
    for (int i = 0; i < RPT; ++i) pass<n, 3, S, true, WLAST>(v[i], b0 + soff[i], b1 + soff[i], j, T.tw[2]);
    __syncthreads();
  }
  return (P - 1) & 1;   // pass p writes b1 for odd p, b0 for even p
}

// ================================================================== K2 forward
template <int n, int RPT>
__global__ void __launch_bounds__(512) k2_fwd(DevPlan P) {
  extern __shared__ float2 sm[];
  const Consts& C = P.C;
  const int L = C.Lres, ln = L * n, N = C.N;
  const int b = blockIdx.y;
  const int P0 = blockIdx.x * kStrip;
  const int Pend = min(P0 + kStrip, C.ncols);
  const int plast = min(Pend, C.ncols - 1);
  const int g = threadIdx.x / (n / 8), j = threadIdx.x % (n / 8);
  int soff[RPT];
  float2 pre[RPT][8];
#pragma unroll
  for (int i = 0; i < RPT; ++i) {
    soff[i] = (g * RPT + i) * n;
#pragma unroll
    for (int r = 0; r < 8; ++r) pre[i][r] = __ldg(&P.tw_pre[soff[i] + j + r * (n / 8)]);
  }
  PassTw<n, -1> T;
  T.load(j, P.tw_n);
  const float2* S1 = P.S1 + (size_t)b * C.ncols * n;
  float2* S2 = P.S2 + (size_t)b * C.half * C.NL;
  float2* buf[3] = {sm, sm + ln, sm + 2 * ln};
  int prev = 2;
  for (int p = P0; p <= plast; ++p) {
    const float2* col = S1 + (size_t)p * n;
    float2 v[RPT][8];
    {
      float2 x[8];
#pragma unroll
      for (int r = 0; r < 8; ++r) x[r] = __ldg(&col[(j + r * (n / 8) + n / 2) & (n - 1)]);
#pragma unroll
      for (int i = 0; i < RPT; ++i)
#pragma unroll
        for (int r = 0; r < 8; ++r) v[i][r] = cmul(x[r], pre[i][r]);
    }
    const int i0 = (prev + 1) % 3, i1 = (prev + 2) % 3;
#pragma unroll
    for (int i = 0; i < RPT; ++i) pass<n, 0, -1, false, true>(v[i], nullptr, buf[i0] + soff[i], j, nullptr);
    const int fin = passes_rest<n, -1, RPT, true>(v, buf[i0], buf[i1], soff, j, T);
    const int cur = fin ? i1 : i0;
    if (p > P0) {
      const float2* Xa = buf[prev];
      const float2* Xb = buf[cur];
      const int e1 = P.k2_colptr[p];
      for (int e = P.k2_colptr[p - 1] + threadIdx.x; e < e1; e += blockDim.x) {
        const int4 nd = __ldg(&P.k2_nodes[e]);
        const float a = __int_as_float(nd.z), bb = __int_as_float(nd.w);
        const int q0 = nd.y & (N - 1), q1 = (nd.y + 1) & (N - 1);
        const int i00 = (q0 & (L - 1)) * n + swz(q0 / L);
        const int i01 = (q1 & (L - 1)) * n + swz(q1 / L);
        const float2 f00 = Xa[i00], f01 = Xa[i01], f10 = Xb[i00], f11 = Xb[i01];
        const float2 c0 = __ffma2_rn(make_float2(a, a), csub(f10, f00), f00);
        const float2 c1 = __ffma2_rn(make_float2(a, a), csub(f11, f01), f01);
        S2[nd.x] = __ffma2_rn(make_float2(bb, bb), csub(c1, c0), c0);
      }
      __syncthreads();
    }
    prev = cur;
  }
  if (Pend == C.ncols) {   // p0 = N/2: alpha == 0, only F[N/2] is used
    const float2* Xa = buf[prev];
    for (int e = P.k2_colptr[C.ncols - 1] + threadIdx.x; e < P.k2_colptr[C.ncols]; e += blockDim.x) {
      const int4 nd = __ldg(&P.k2_nodes[e]);
      const float bb = __int_as_float(nd.w);
      const int q0 = nd.y & (N - 1), q1 = (nd.y + 1) & (N - 1);
      const float2 f00 = Xa[(q0 & (L - 1)) * n + swz(q0 / L)];
      const float2 f01 = Xa[(q1 & (L - 1)) * n + swz(q1 / L)];
      S2[nd.x] = __ffma2_rn(make_float2(bb, bb), csub(f01, f00), f00);
    }
  }
}

// ================================================================== K1 forward (row pairs)
// z = f_y + i f_{y+1}; Z[p] = sum_x z e^{-2 pi i p (x-n/2)/N}; two row pairs per CTA so that
// each p writes one full 32-byte sector S1[p][y0..y0+3].
template <int n, int RPT>
__global__ void __launch_bounds__(512) k1_fwd(DevPlan P, const float* __restrict__ f) {
  extern __shared__ float2 sm[];
  const Consts& C = P.C;
  const int L = C.Lres, ln = L * n, N = C.N;
  const int b = blockIdx.y, y0 = 4 * blockIdx.x;
  const int g = threadIdx.x / (n / 8), j = threadIdx.x % (n / 8);
  int soff[RPT];
  float2 pre[RPT][8];
#pragma unroll
  for (int i = 0; i < RPT; ++i) {
    soff[i] = (g * RPT + i) * n;
#pragma unroll
    for (int r = 0; r < 8; ++r) pre[i][r] = __ldg(&P.tw_pre[soff[i] + j + r * (n / 8)]);
  }
  PassTw<n, -1> T;
  T.load(j, P.tw_n);
  float2* buf[3] = {sm, sm + ln, sm + 2 * ln};
  const float2* ZA = nullptr;
  const float2* ZB = nullptr;
  // pair A (rows y0, y0+1) in buffers 0/1; pair B (rows y0+2, y0+3) in buffer 2 and the free one
#pragma unroll 1
  for (int pr = 0; pr < 2; ++pr) {
    const float* r0 = f + ((size_t)b * n + y0 + 2 * pr) * n;
    float2 v[RPT][8];
    {
      float2 x[8];
#pragma unroll
      for (int r = 0; r < 8; ++r) {
        const int xi = (j + r * (n / 8) + n / 2) & (n - 1);
        x[r] = make_float2(__ldg(&r0[xi]), __ldg(&r0[n + xi]));
      }
#pragma unroll
      for (int i = 0; i < RPT; ++i)
#pragma unroll
        for (int r = 0; r < 8; ++r) v[i][r] = cmul(x[r], pre[i][r]);
    }
    float2* b0 = pr == 0 ? buf[0] : buf[2];
    float2* b1 = pr == 0 ? buf[1] : (ZA == buf[0] ? buf[1] : buf[0]);
#pragma unroll
    for (int i = 0; i < RPT; ++i) pass<n, 0, -1, false, true>(v[i], nullptr, b0 + soff[i], j, nullptr);
    const int fin = passes_rest<n, -1, RPT, true>(v, b0, b1, soff, j, T);
    if (pr == 0) ZA = fin ? b1 : b0;
    else ZB = fin ? b1 : b0;
  }
  float4* out = reinterpret_cast<float4*>(P.S1 + (size_t)b * C.ncols * n);
  for (int p = threadIdx.x; p < C.ncols; p += blockDim.x) {
    const int pm = (N - p) & (N - 1);
    const int ip = (p & (L - 1)) * n + swz(p / L);
    const int im = (pm & (L - 1)) * n + swz(pm / L);
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
// S~1[p][y] = sum_s X_s[y'] conj(W_N^{s y''}); the residue sum is reduced through smem.
template <int n, int RPT>
__global__ void __launch_bounds__(512) k2t_adj(DevPlan P) {
  extern __shared__ float2 sm[];
  const Consts& C = P.C;
  const int L = C.Lres, ln = L * n;
  const int b = blockIdx.y;
  const int P0 = blockIdx.x * kStrip;
  const int Pend = min(P0 + kStrip, C.ncols);
  const int g = threadIdx.x / (n / 8), j = threadIdx.x % (n / 8);
  const int G = L / RPT;   // residue groups
  int soff[RPT];
  float2 post[RPT][8];
#pragma unroll
  for (int i = 0; i < RPT; ++i) {
    soff[i] = (g * RPT + i) * n;
#pragma unroll
    for (int e = 0; e < 8; ++e) post[i][e] = __ldg(&P.tw_pre[soff[i] + last_pos<n>(j, e)]);
  }
  PassTw<n, 1> T;
  T.load(j, P.tw_n);
  const float2* S2 = P.S2 + (size_t)b * C.half * C.NL;
  float2* out = P.S1 + (size_t)b * C.ncols * n;
  float2* R = sm;            // gather target (zeroed)
  float2* Xb = sm + ln;      // ping-pong
  float2* red = sm + 2 * ln; // residue-sum staging [G][n]
  for (int i = threadIdx.x; i < ln; i += blockDim.x) R[i] = make_float2(0.f, 0.f);
  __syncthreads();
  for (int p = P0; p < Pend; ++p) {
    // scatter column p from the CSR (each target written once)
    for (int t = P.k2t_colptr[p] + threadIdx.x; t < P.k2t_colptr[p + 1]; t += blockDim.x) {
      const int qm = __ldg(&P.k2t_tq[t]);
      float2 acc = make_float2(0.f, 0.f);
      const int e1 = __ldg(&P.k2t_tstart[t + 1]);
      for (int e = __ldg(&P.k2t_tstart[t]); e < e1; ++e) {
        const int2 en = __ldg(&P.k2t_ent[e]);
        acc = __ffma2_rn(make_float2(__int_as_float(en.y), __int_as_float(en.y)), S2[en.x], acc);
      }
      R[(qm & (L - 1)) * n + swz(qm / L)] = acc;
    }
    __syncthreads();
    float2 v[RPT][8];
    // pass 0 reads R and re-zeroes what it read (every element is read exactly once)
#pragma unroll
    for (int i = 0; i < RPT; ++i) {
#pragma unroll
      for (int r = 0; r < 8; ++r) {
        float2* a = R + soff[i] + swz(j + r * (n / 8));
        v[i][r] = *a;
        *a = make_float2(0.f, 0.f);
      }
      dft8<1>(v[i]);
    }
    // pass-0 results go to Xb (Stockham Ns = 1 positions)
#pragma unroll
    for (int i = 0; i < RPT; ++i)
#pragma unroll
      for (int r = 0; r < 8; ++r) Xb[soff[i] + swz(j * 8 + r)] = v[i][r];
    passes_rest<n, 1, RPT, false>(v, Xb, red, soff, j, T);   // result in registers
    float2 part[8];
#pragma unroll
    for (int e = 0; e < 8; ++e) {
      part[e] = cmulc(v[0][e], post[0][e]);
#pragma unroll
      for (int i = 1; i < RPT; ++i) part[e] = cadd(part[e], cmulc(v[i][e], post[i][e]));
    }
    // residue-group reduction through smem: red[g][pos] (natural position)
#pragma unroll
    for (int e = 0; e < 8; ++e) red[g * n + last_pos<n>(j, e)] = part[e];
    __syncthreads();
    for (int yp = threadIdx.x; yp < n; yp += blockDim.x) {
      float2 acc = red[yp];
      for (int gg = 1; gg < G; ++gg) acc = cadd(acc, red[gg * n + yp]);
      out[(size_t)p * n + ((yp + n / 2) & (n - 1))] = acc;
    }
    __syncthreads();
  }
}

// ================================================================== K1T (transpose of K1)
// Two row pairs per CTA: Z[p] = C_y[p] + i C_{y+1}[p] (Hermitian completion of the half
// spectra, C[0], C[N/2] = 2 Re), inverse residue FFTs, residue sum -> f~ rows.
template <int n, int RPT>
__global__ void __launch_bounds__(512) k1t_adj(DevPlan P, float* __restrict__ fout) {
  extern __shared__ float2 sm[];
  const Consts& C = P.C;
  const int L = C.Lres, ln = L * n, N = C.N;
  const int b = blockIdx.y, y0 = 4 * blockIdx.x;
  const int g = threadIdx.x / (n / 8), j = threadIdx.x % (n / 8);
  const int G = L / RPT;
  int soff[RPT];
  float2 post[RPT][8];
#pragma unroll
  for (int i = 0; i < RPT; ++i) {
    soff[i] = (g * RPT + i) * n;
#pragma unroll
    for (int e = 0; e < 8; ++e) post[i][e] = __ldg(&P.tw_pre[soff[i] + last_pos<n>(j, e)]);
  }
  PassTw<n, 1> T;
  T.load(j, P.tw_n);
  float2* ZA = sm;
  float2* ZB = sm + ln;
  float2* X = sm + 2 * ln;
  const float4* in = reinterpret_cast<const float4*>(P.S1 + (size_t)b * C.ncols * n);
  for (int p = threadIdx.x; p < C.ncols; p += blockDim.x) {
    const float4* src = in + (((size_t)p * n + y0) >> 1);
    const float4 v0 = src[0], v1 = src[1];   // rows y0, y0+1 | y0+2, y0+3
    const int ip = (p & (L - 1)) * n + swz(p / L);
    if (p == 0 || p == N / 2) {
      ZA[ip] = make_float2(2.f * v0.x, 2.f * v0.z);
      ZB[ip] = make_float2(2.f * v1.x, 2.f * v1.z);
    } else {
      const int pm = N - p;
      const int im = (pm & (L - 1)) * n + swz(pm / L);
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
    float2 v[RPT][8];
#pragma unroll
    for (int i = 0; i < RPT; ++i) {
#pragma unroll
      for (int r = 0; r < 8; ++r) v[i][r] = Zs[soff[i] + swz(j + r * (n / 8))];
      dft8<1>(v[i]);
    }
    __syncthreads();   // everyone has read Zs before it is reused as scratch
#pragma unroll
    for (int i = 0; i < RPT; ++i)
#pragma unroll
      for (int r = 0; r < 8; ++r) X[soff[i] + swz(j * 8 + r)] = v[i][r];
    passes_rest<n, 1, RPT, false>(v, X, Zs, soff, j, T);
    float2 part[8];
#pragma unroll
    for (int e = 0; e < 8; ++e) {
      part[e] = cmulc(v[0][e], post[0][e]);
#pragma unroll
      for (int i = 1; i < RPT; ++i) part[e] = cadd(part[e], cmulc(v[i][e], post[i][e]));
    }
    float2* red = Zs;   // Zs is free now (passes are finished, results in registers)
#pragma unroll
    for (int e = 0; e < 8; ++e) red[g * n + last_pos<n>(j, e)] = part[e];
    __syncthreads();
    float* o = fout + ((size_t)b * n + y0 + 2 * pr) * n;
    for (int xp = threadIdx.x; xp < n; xp += blockDim.x) {
      float2 acc = red[xp];
      for (int gg = 1; gg < G; ++gg) acc = cadd(acc, red[gg * n + xp]);
      const int x = (xp + n / 2) & (n - 1);
      o[x] = acc.x;
      o[n + x] = acc.y;
    }
    __syncthreads();
  }
}

// ================================================================== dispatch
size_t smem_fft4(const Consts& C) { return (size_t)3 * C.Lres * C.n * sizeof(float2); }

template <int n, int RPT>
static cudaError_t cfg_one() {
  cudaError_t e = cudaSuccess;
  const int big = 3 * 16 * n * (int)sizeof(float2);
  const int lim = big > 227 * 1024 ? 227 * 1024 : big;
  if (e == cudaSuccess) e = cudaFuncSetAttribute(k2_fwd<n, RPT>, cudaFuncAttributeMaxDynamicSharedMemorySize, lim);
  if (e == cudaSuccess) e = cudaFuncSetAttribute(k1_fwd<n, RPT>, cudaFuncAttributeMaxDynamicSharedMemorySize, lim);
  if (e == cudaSuccess) e = cudaFuncSetAttribute(k2t_adj<n, RPT>, cudaFuncAttributeMaxDynamicSharedMemorySize, lim);
  if (e == cudaSuccess) e = cudaFuncSetAttribute(k1t_adj<n, RPT>, cudaFuncAttributeMaxDynamicSharedMemorySize, lim);
  return e;
}

cudaError_t configure_fft_kernels(const Consts& C) {
  const int R = (C.Lres * C.n >= 1024) ? 2 : 1;
  switch (C.n) {
    case 32: return R == 2 ? cfg_one<32, 2>() : cfg_one<32, 1>();
    case 64: return R == 2 ? cfg_one<64, 2>() : cfg_one<64, 1>();
    case 128: return cfg_one<128, 2>();
    case 256: return cfg_one<256, 2>();
    case 512: return cfg_one<512, 2>();
    case 1024: return cfg_one<1024, 2>();
  }
  return cudaErrorInvalidValue;
}

int fft_threads(const Consts& C) {
  const int R = (C.Lres * C.n >= 1024) ? 2 : 1;
  return (C.Lres / R) * (C.n / 8);
}

#define TAT_DISPATCH_N(NN, CALL)                                          \
  switch (C.n) {                                                           \
    case 32: { constexpr int NN = 32; if (R == 2) { constexpr int RP = 2; CALL; } else { constexpr int RP = 1; CALL; } } break; \
    case 64: { constexpr int NN = 64; if (R == 2) { constexpr int RP = 2; CALL; } else { constexpr int RP = 1; CALL; } } break; \
    case 128: { constexpr int NN = 128; constexpr int RP = 2; CALL; } break; \
    case 256: { constexpr int NN = 256; constexpr int RP = 2; CALL; } break; \
    case 512: { constexpr int NN = 512; constexpr int RP = 2; CALL; } break; \
    case 1024: { constexpr int NN = 1024; constexpr int RP = 2; CALL; } break; \
    default: return cudaErrorInvalidValue;                                 \
  }

cudaError_t launch_k1(const DevPlan& P, const float* f, cudaStream_t s) {
  const Consts& C = P.C;
  const int R = (C.Lres * C.n >= 1024) ? 2 : 1;
  dim3 grid(C.n / 4, C.batch);
  const int th = fft_threads(C);
  const size_t sm = smem_fft4(C);
  TAT_DISPATCH_N(NN, (k1_fwd<NN, RP><<<grid, th, sm, s>>>(P, f)));
  return cudaGetLastError();
}
cudaError_t launch_k2(const DevPlan& P, cudaStream_t s) {
  const Consts& C = P.C;
  const int R = (C.Lres * C.n >= 1024) ? 2 : 1;
  dim3 grid((C.ncols + kStrip - 1) / kStrip, C.batch);
  const int th = fft_threads(C);
  const size_t sm = smem_fft4(C);
  TAT_DISPATCH_N(NN, (k2_fwd<NN, RP><<<grid, th, sm, s>>>(P)));
  return cudaGetLastError();
}
cudaError_t launch_k2t(const DevPlan& P, cudaStream_t s) {
  const Consts& C = P.C;
  const int R = (C.Lres * C.n >= 1024) ? 2 : 1;
  dim3 grid((C.ncols + kStrip - 1) / kStrip, C.batch);
  const int th = fft_threads(C);
  const size_t sm = smem_fft4(C);
  TAT_DISPATCH_N(NN, (k2t_adj<NN, RP><<<grid, th, sm, s>>>(P)));
  return cudaGetLastError();
}
cudaError_t launch_k1t(const DevPlan& P, float* f, cudaStream_t s) {
  const Consts& C = P.C;
  const int R = (C.Lres * C.n >= 1024) ? 2 : 1;
  dim3 grid(C.n / 4, C.batch);
  const int th = fft_threads(C);
  const size_t sm = smem_fft4(C);
  TAT_DISPATCH_N(NN, (k1t_adj<NN, RP><<<grid, th, sm, s>>>(P, f)));
  return cudaGetLastError();
}

}  // namespace tat
