// sm_100a kernels of the fast forward operator A (Alg. 1) and its exact
// transpose A* (Alg. 2 order, L666-692).  Stage names follow DESIGN.md / SURVEY §8(a):
//
//   K1  zero-extend + row DFT          f  [B][n][n]        -> S1 [B][N/2+1][n]   (Alg.1 st.1-2)
//   K2  column DFT + bilinear to polar S1                  -> S2 [B][n_phi/2][NL] (st.2-3)
//   K3  angular DFT + Bessel multiply  S2                  -> S3 [B][K+1][NL]     (st.4, E:eq2)
//   K4  lambda -> t cosine transform   S3                  -> S4 [B][K+1][n_t]    (st.5)
//   K5  angular synthesis + restrict   S4                  -> g  [B][n_t][n_det]  (st.6-7)
//   and K5T..K1T, the transposed chain, for A*.
//
// All FFTs are exact DFTs of the stated sums with fp64-built fp32 twiddle tables (index
// reduction in integers); the zero-padded 2-D DFT of size N = L n is split into L residue
// classes q = L a + s, each an n-point FFT of the pre-twiddled column (no cuFFT).
#include "tat_internal.h"

#include <cstdio>

namespace tat {

// ------------------------------------------------------------------ complex helpers
__device__ __forceinline__ float2 cmul(float2 a, float2 b) {
  return make_float2(fmaf(a.x, b.x, -a.y * b.y), fmaf(a.x, b.y, a.y * b.x));
}
__device__ __forceinline__ float2 cmulc(float2 a, float2 b) {   // a * conj(b)
  return make_float2(fmaf(a.x, b.x, a.y * b.y), fmaf(a.y, b.x, -a.x * b.y));
}
__device__ __forceinline__ float2 cadd(float2 a, float2 b) { return make_float2(a.x + b.x, a.y + b.y); }
__device__ __forceinline__ float2 csub(float2 a, float2 b) { return make_float2(a.x - b.x, a.y - b.y); }
__device__ __forceinline__ float2 conjf2(float2 a) { return make_float2(a.x, -a.y); }
__device__ __forceinline__ float2 cscale(float2 a, float s) { return make_float2(a.x * s, a.y * s); }
// multiply by i^e (e mod 4), exact
__device__ __forceinline__ float2 mul_ipow(float2 a, int e) {
  switch (e & 3) {
    case 0: return a;
    case 1: return make_float2(-a.y, a.x);
    case 2: return make_float2(-a.x, -a.y);
    default: return make_float2(a.y, -a.x);
  }
}

// ------------------------------------------------------------------ shared-memory FFT
// Stockham autosort, mixed radix 4/2/3, `count` transforms of length `len` stored
// contiguously ([count][len]) in A; B is scratch of the same size.  tw[k] = exp(-2 pi i k/len).
// SIGN = -1: X[k] = sum x[j] e^{-2 pi i jk/len};  SIGN = +1: conjugate kernel (no 1/len).
// Returns the buffer holding the result.  Must be called by all threads of the block.
template <int SIGN>
__device__ float2* smem_fft(float2* A, float2* B, int len, int count,
                            const float2* __restrict__ tw) {
  int Ns = 1, rem = len;
  while (Ns < len) {
    const int R = (rem % 4 == 0) ? 4 : ((rem % 2 == 0) ? 2 : 3);
    const int stride = len / R;
    const int twstep = len / (Ns * R);
    const int total = count * stride;
    for (int idx = threadIdx.x; idx < total; idx += blockDim.x) {
      const int t = idx / stride, j = idx - t * stride;
      const float2* a = A + (size_t)t * len;
      float2* b = B + (size_t)t * len;
      const int k = j % Ns;
      float2 v[4];
      for (int r = 0; r < R; ++r) {
        float2 x = a[j + r * stride];
        if (r > 0 && k > 0) {
          float2 w = __ldg(&tw[(k * r * twstep) % len]);
          x = (SIGN < 0) ? cmul(x, w) : cmulc(x, w);
        }
        v[r] = x;
      }
      if (R == 2) {
        float2 t0 = cadd(v[0], v[1]), t1 = csub(v[0], v[1]);
        v[0] = t0; v[1] = t1;
      } else if (R == 4) {
        float2 s02 = cadd(v[0], v[2]), d02 = csub(v[0], v[2]);
        float2 s13 = cadd(v[1], v[3]), d13 = csub(v[1], v[3]);
        // SIGN=-1: X1 = d02 - i d13, X3 = d02 + i d13
        float2 jd13 = (SIGN < 0) ? make_float2(d13.y, -d13.x) : make_float2(-d13.y, d13.x);
        v[0] = cadd(s02, s13);
        v[2] = csub(s02, s13);
        v[1] = cadd(d02, jd13);
        v[3] = csub(d02, jd13);
      } else {  // R == 3
        const float c3 = -0.5f, s3 = (SIGN < 0 ? -1.f : 1.f) * 0.86602540378443864676f;
        float2 s12 = cadd(v[1], v[2]), d12 = csub(v[1], v[2]);
        float2 m = make_float2(v[0].x + c3 * s12.x, v[0].y + c3 * s12.y);
        float2 rot = make_float2(-s3 * d12.y, s3 * d12.x);   // i s3 d12
        v[0] = cadd(v[0], s12);
        v[1] = cadd(m, rot);
        v[2] = csub(m, rot);
      }
      const int base = (j / Ns) * Ns * R + k;
      for (int r = 0; r < R; ++r) b[base + r * Ns] = v[r];
    }
    __syncthreads();
    float2* tmp = A; A = B; B = tmp;
    Ns *= R;
    rem /= R;
  }
  return A;
}

// ------------------------------------------------------------------ tile sizes
__host__ __device__ inline int tile_ring(int n_ring) { int t = 4096 / n_ring; return t < 1 ? 1 : (t > 16 ? 16 : t); }
constexpr int kK2Strip = 16;
constexpr int kThreads = 256;

size_t max_smem_needed(const Consts& C) {
  size_t ln = (size_t)C.Lres * C.n * sizeof(float2);
  size_t s = 3 * ln;                                               // K2
  if (dct_fast_r(C)) s = std::max(s, smem_dct_fast(C));            // K4 / K4T
  else s = std::max(s, (size_t)2 * 2 * C.M * sizeof(float2));
  if (ring_fast_ok(C)) s = std::max(s, smem_ring_fast(C));           // K3/K5
  else s = std::max(s, (size_t)2 * tile_ring(C.n_ring) * C.n_ring * sizeof(float2));
  return s;
}

// ================================================================== forward kernels
// K1: row pair (y, y+1) packed as z = f_y + i f_{y+1}; Z[p] = sum_x z[x] e^{-2 pi i p (x-n/2)/N}
// for all p, as L residue FFTs; split into the two rows' half spectra p in [0, N/2].
__global__ void k1_row_dft(DevPlan P, const float* __restrict__ f) {
  extern __shared__ float2 sm[];
  const Consts& C = P.C;
  const int n = C.n, L = C.Lres, N = C.N;
  const int b = blockIdx.y, y = 2 * blockIdx.x;
  float2* A = sm;
  float2* Bf = sm + (size_t)L * n;
  const float* f0 = f + ((size_t)b * n + y) * n;
  for (int idx = threadIdx.x; idx < L * n; idx += blockDim.x) {
    int s = idx / n, yp = idx - s * n;
    int x = (yp + n / 2) & (n - 1);
    float2 z = make_float2(__ldg(&f0[x]), __ldg(&f0[n + x]));
    A[idx] = cmul(z, __ldg(&P.tw_pre[idx]));
  }
  __syncthreads();
  float2* X = smem_fft<-1>(A, Bf, n, L, P.tw_n);
  float4* out = reinterpret_cast<float4*>(P.S1 + (size_t)b * C.ncols * n);
  for (int p = threadIdx.x; p < C.ncols; p += blockDim.x) {
    int pm = (N - p) & (N - 1);
    float2 zp = X[(p % L) * n + p / L];
    float2 zm = conjf2(X[(pm % L) * n + pm / L]);
    float2 s = cadd(zp, zm), d = csub(zp, zm);
    // row y: (zp + conj zm)/2 ; row y+1: (zp - conj zm)/(2i) = -i d / 2
    out[((size_t)p * n + y) >> 1] = make_float4(0.5f * s.x, 0.5f * s.y, 0.5f * d.y, -0.5f * d.x);
  }
}

// column DFT of S1 column p into smem: X[s*n + a] = F[p][q], q mod N = L a + s (unscaled)
__device__ float2* column_dft(const DevPlan& P, const float2* __restrict__ col, float2* A,
                              float2* Bf) {
  const int n = P.C.n, L = P.C.Lres;
  for (int idx = threadIdx.x; idx < L * n; idx += blockDim.x) {
    int s = idx / n, yp = idx - s * n;
    int y = (yp + n / 2) & (n - 1);
    A[idx] = cmul(__ldg(&col[y]), __ldg(&P.tw_pre[idx]));
  }
  __syncthreads();
  return smem_fft<-1>(A, Bf, n, L, P.tw_n);
}

__device__ __forceinline__ float2 fq(const float2* X, int q, int n, int L, int N) {
  int qm = q & (N - 1);
  return X[(qm % L) * n + qm / L];
}

// K2: strip of kK2Strip columns, sliding window of two column spectra (one halo recompute).
__global__ void k2_col_dft_gather(DevPlan P) {
  extern __shared__ float2 sm[];
  const Consts& C = P.C;
  const int n = C.n, L = C.Lres, N = C.N, ln = L * n;
  const int b = blockIdx.y;
  const int P0 = blockIdx.x * kK2Strip;
  const int Pend = min(P0 + kK2Strip, C.ncols);           // owned p0 in [P0, Pend)
  const float2* S1 = P.S1 + (size_t)b * C.ncols * n;
  float2* S2 = P.S2 + (size_t)b * C.half * C.NL;
  float2* buf[3] = {sm, sm + ln, sm + 2 * ln};
  int prev = -1;
  const int plast = min(Pend, C.ncols - 1);                // last column to compute
  for (int p = P0; p <= plast; ++p) {
    int i0 = (prev + 1) % 3, i1 = (prev + 2) % 3;
    float2* X = column_dft(P, S1 + (size_t)p * n, buf[i0], buf[i1]);
    int cur = (X == buf[i0]) ? i0 : i1;
    if (p > P0) {
      const float2* Xa = buf[prev];
      const float2* Xb = buf[cur];
      for (int e = P.k2_colptr[p - 1] + threadIdx.x; e < P.k2_colptr[p]; e += blockDim.x) {
        int4 nd = __ldg(&P.k2_nodes[e]);
        float a = __int_as_float(nd.z), bb = __int_as_float(nd.w);
        float2 f00 = fq(Xa, nd.y, n, L, N), f01 = fq(Xa, nd.y + 1, n, L, N);
        float2 f10 = fq(Xb, nd.y, n, L, N), f11 = fq(Xb, nd.y + 1, n, L, N);
        float2 c0 = make_float2((1.f - a) * f00.x + a * f10.x, (1.f - a) * f00.y + a * f10.y);
        float2 c1 = make_float2((1.f - a) * f01.x + a * f11.x, (1.f - a) * f01.y + a * f11.y);
        S2[nd.x] = make_float2((1.f - bb) * c0.x + bb * c1.x, (1.f - bb) * c0.y + bb * c1.y);
      }
    }
    __syncthreads();
    prev = cur;
  }
  if (Pend == C.ncols) {   // last column p0 = N/2: alpha == 0, only F[N/2] is used
    const float2* Xa = buf[prev];
    for (int e = P.k2_colptr[C.ncols - 1] + threadIdx.x; e < P.k2_colptr[C.ncols]; e += blockDim.x) {
      int4 nd = __ldg(&P.k2_nodes[e]);
      float bb = __int_as_float(nd.w);
      float2 f00 = fq(Xa, nd.y, n, L, N), f01 = fq(Xa, nd.y + 1, n, L, N);
      S2[nd.x] = make_float2((1.f - bb) * f00.x + bb * f01.x, (1.f - bb) * f00.y + bb * f01.y);
    }
  }
}

// K3: angular DFT over the full ring (half plane + conjugate mirror), times i^k m'[k][j].
__global__ void k3_angular_mult(DevPlan P) {
  extern __shared__ float2 sm[];
  const Consts& C = P.C;
  const int nphi = C.n_ring, half = C.half, NL = C.NL, JT = tile_ring(nphi);
  const int b = blockIdx.y, j0 = blockIdx.x * JT;
  const int jt = min(JT, NL - j0);
  float2* A = sm;
  float2* Bf = sm + (size_t)JT * nphi;
  const float2* S2 = P.S2 + (size_t)b * half * NL;
  for (int idx = threadIdx.x; idx < half * JT; idx += blockDim.x) {
    int lp = idx / JT, jj = idx - lp * JT;
    float2 v = (jj < jt) ? S2[(size_t)lp * NL + j0 + jj] : make_float2(0.f, 0.f);
    int l = (lp - nphi / 4) & (nphi - 1);
    A[jj * nphi + l] = v;
    A[jj * nphi + ((l + half) & (nphi - 1))] = conjf2(v);
  }
  __syncthreads();
  float2* X = smem_fft<-1>(A, Bf, nphi, JT, P.tw_ring);
  float2* S3 = P.S3 + (size_t)b * C.Kp * NL;
  for (int idx = threadIdx.x; idx < C.Kp * JT; idx += blockDim.x) {
    int k = idx / JT, jj = idx - k * JT;
    if (jj >= jt) continue;
    int j = j0 + jj;
    float m = __ldg(&P.mult[(size_t)k * NL + j]);
    S3[(size_t)k * NL + j] = mul_ipow(cscale(X[jj * nphi + k], m), k);
  }
}

// K4: G[m] = sum_j H[j] cos(pi j (m+1)/M) = (X[m+1] + X[2M-m-1]) / 2, X = 2M-point DFT of H.
__global__ void k4_dct(DevPlan P) {
  extern __shared__ float2 sm[];
  const Consts& C = P.C;
  const int M2 = 2 * C.M, NL = C.NL;
  const int b = blockIdx.y, k = blockIdx.x;
  float2* A = sm;
  float2* Bf = sm + M2;
  const float2* H = P.S3 + ((size_t)b * C.Kp + k) * NL;
  for (int j = threadIdx.x; j < M2; j += blockDim.x) A[j] = (j < NL) ? H[j] : make_float2(0.f, 0.f);
  __syncthreads();
  float2* X = smem_fft<-1>(A, Bf, M2, 1, P.tw_dct);
  float2* G = P.S4 + ((size_t)b * C.Kp + k) * C.n_t;
  for (int m = threadIdx.x; m < C.n_t; m += blockDim.x)
    G[m] = cscale(cadd(X[m + 1], X[M2 - m - 1]), 0.5f);
}

// K5: C2R angular synthesis g(t, phi_l) = sum_k G_k e^{i k phi_l} (Hermitian), gather ring.
__global__ void k5_synth_restrict(DevPlan P, float* __restrict__ g) {
  extern __shared__ float2 sm[];
  const Consts& C = P.C;
  const int nphi = C.n_ring, K = C.K, TT = tile_ring(nphi);
  const int b = blockIdx.y, t0 = blockIdx.x * TT, tt_n = min(TT, C.n_t - t0);
  float2* A = sm;
  float2* Bf = sm + (size_t)TT * nphi;
  const float2* S4 = P.S4 + (size_t)b * C.Kp * C.n_t;
  for (int idx = threadIdx.x; idx < C.Kp * TT; idx += blockDim.x) {
    int k = idx / TT, tt = idx - k * TT;
    float2 v = (tt < tt_n) ? S4[(size_t)k * C.n_t + t0 + tt] : make_float2(0.f, 0.f);
    A[tt * nphi + k] = v;
    if (k >= 1 && k < K) A[tt * nphi + nphi - k] = conjf2(v);
  }
  __syncthreads();
  float2* X = smem_fft<1>(A, Bf, nphi, TT, P.tw_ring);
  for (int idx = threadIdx.x; idx < tt_n * C.n_det; idx += blockDim.x) {
    int tt = idx / C.n_det, d = idx - tt * C.n_det;
    g[((size_t)b * C.n_t + t0 + tt) * C.n_det + d] = X[tt * nphi + __ldg(&P.ring[d])].x;
  }
}

// ================================================================== adjoint kernels
// K5T: zero-extend to the ring, R2C analysis G~[k] = sum_l g_l e^{-i k phi_l}, k in [0, K].
__global__ void k5t_analysis(DevPlan P, const float* __restrict__ g) {
  extern __shared__ float2 sm[];
  const Consts& C = P.C;
  const int nphi = C.n_ring, TT = tile_ring(nphi);
  const int b = blockIdx.y, t0 = blockIdx.x * TT, tt_n = min(TT, C.n_t - t0);
  float2* A = sm;
  float2* Bf = sm + (size_t)TT * nphi;
  for (int idx = threadIdx.x; idx < TT * nphi; idx += blockDim.x) A[idx] = make_float2(0.f, 0.f);
  __syncthreads();
  for (int idx = threadIdx.x; idx < tt_n * C.n_det; idx += blockDim.x) {
    int tt = idx / C.n_det, d = idx - tt * C.n_det;
    A[tt * nphi + __ldg(&P.ring[d])].x = g[((size_t)b * C.n_t + t0 + tt) * C.n_det + d];
  }
  __syncthreads();
  float2* X = smem_fft<-1>(A, Bf, nphi, TT, P.tw_ring);
  float2* S4 = P.S4 + (size_t)b * C.Kp * C.n_t;
  for (int idx = threadIdx.x; idx < C.Kp * TT; idx += blockDim.x) {
    int k = idx / TT, tt = idx - k * TT;
    if (tt < tt_n) S4[(size_t)k * C.n_t + t0 + tt] = X[tt * nphi + k];
  }
}

// K4T: Hc[j] = sum_m G~[m] cos(pi j (m+1)/M) = (Y[j] + Y[2M-j])/2; H~ = (-i)^k omega m' Hc.
__global__ void k4t_dct(DevPlan P) {
  extern __shared__ float2 sm[];
  const Consts& C = P.C;
  const int M2 = 2 * C.M, NL = C.NL;
  const int b = blockIdx.y, k = blockIdx.x;
  float2* A = sm;
  float2* Bf = sm + M2;
  const float2* G = P.S4 + ((size_t)b * C.Kp + k) * C.n_t;
  for (int i = threadIdx.x; i < M2; i += blockDim.x)
    A[i] = (i >= 1 && i <= C.n_t) ? G[i - 1] : make_float2(0.f, 0.f);
  __syncthreads();
  float2* X = smem_fft<-1>(A, Bf, M2, 1, P.tw_dct);
  float2* H = P.S3 + ((size_t)b * C.Kp + k) * NL;
  const float om = (float)C.omega;
  for (int j = threadIdx.x; j < NL; j += blockDim.x) {
    float2 y = cscale(cadd(X[j], X[(M2 - j) % M2]), 0.5f);
    float m = om * __ldg(&P.mult[(size_t)k * NL + j]);
    H[j] = mul_ipow(cscale(y, m), -k);
  }
}

// K3T: P~[l] = sum_{k=-K}^{K-1} H~_k e^{i k phi_l} on the half plane l' in [0, n_phi/2),
// with H~_{-k} = (-1)^k conj(H~_k) (1 <= k < K) and H~_{-K} = H~_K.
__global__ void k3t_angular(DevPlan P) {
  extern __shared__ float2 sm[];
  const Consts& C = P.C;
  const int nphi = C.n_ring, half = C.half, NL = C.NL, K = C.K, JT = tile_ring(nphi);
  const int b = blockIdx.y, j0 = blockIdx.x * JT, jt = min(JT, NL - j0);
  float2* A = sm;
  float2* Bf = sm + (size_t)JT * nphi;
  const float2* S3 = P.S3 + (size_t)b * C.Kp * NL;
  for (int idx = threadIdx.x; idx < C.Kp * JT; idx += blockDim.x) {
    int k = idx / JT, jj = idx - k * JT;
    float2 v = (jj < jt) ? S3[(size_t)k * NL + j0 + jj] : make_float2(0.f, 0.f);
    A[jj * nphi + k] = v;                                   // k in [0, K]; index K is k = -K
    if (k >= 1 && k < K) {
      float2 w = conjf2(v);
      if (k & 1) w = make_float2(-w.x, -w.y);
      A[jj * nphi + nphi - k] = w;
    }
  }
  __syncthreads();
  float2* X = smem_fft<1>(A, Bf, nphi, JT, P.tw_ring);
  float2* S2 = P.S2 + (size_t)b * half * NL;
  for (int idx = threadIdx.x; idx < half * JT; idx += blockDim.x) {
    int lp = idx / JT, jj = idx - lp * JT;
    if (jj >= jt) continue;
    int l = (lp - nphi / 4) & (nphi - 1);
    S2[(size_t)lp * NL + j0 + jj] = X[jj * nphi + l];
  }
}

// K2T: per column p: R[q] = sum of w * P~ over the CSR (deterministic order), then
// S~1[y][p] = sum_q R[q] e^{+2 pi i q (y-n/2)/N} via L inverse residue FFTs.
__global__ void k2t_gather_col_idft(DevPlan P) {
  extern __shared__ float2 sm[];
  const Consts& C = P.C;
  const int n = C.n, L = C.Lres, ln = L * n;
  const int b = blockIdx.y, p = blockIdx.x;
  float2* A = sm;
  float2* Bf = sm + ln;
  const float2* S2 = P.S2 + (size_t)b * C.half * C.NL;
  for (int i = threadIdx.x; i < ln; i += blockDim.x) A[i] = make_float2(0.f, 0.f);
  __syncthreads();
  for (int t = P.k2t_colptr[p] + threadIdx.x; t < P.k2t_colptr[p + 1]; t += blockDim.x) {
    int qm = __ldg(&P.k2t_tq[t]);
    float2 acc = make_float2(0.f, 0.f);
    for (int e = __ldg(&P.k2t_tstart[t]); e < __ldg(&P.k2t_tstart[t + 1]); ++e) {
      int2 en = __ldg(&P.k2t_ent[e]);
      float w = __int_as_float(en.y);
      float2 v = S2[en.x];
      acc.x = fmaf(w, v.x, acc.x);
      acc.y = fmaf(w, v.y, acc.y);
    }
    A[(qm % L) * n + qm / L] = acc;
  }
  __syncthreads();
  float2* X = smem_fft<1>(A, Bf, n, L, P.tw_n);
  float2* out = P.S1 + ((size_t)b * C.ncols + p) * n;
  for (int y = threadIdx.x; y < n; y += blockDim.x) {
    int yp = (y + n / 2) & (n - 1);
    float2 acc = make_float2(0.f, 0.f);
    for (int s = 0; s < L; ++s)
      acc = cadd(acc, cmulc(X[s * n + yp], __ldg(&P.tw_pre[s * n + yp])));
    out[y] = acc;
  }
}

// K1T: rows (y, y+1) from their half spectra (Hermitian completion, C[0] and C[N/2] = 2 Re),
// packed Z = C_y + i C_{y+1}; f~_y + i f~_{y+1} = sum_p Z[p] e^{+2 pi i p (x-n/2)/N}.
__global__ void k1t_row_idft(DevPlan P, float* __restrict__ fout) {
  extern __shared__ float2 sm[];
  const Consts& C = P.C;
  const int n = C.n, L = C.Lres, N = C.N, ln = L * n;
  const int b = blockIdx.y, y = 2 * blockIdx.x;
  float2* A = sm;
  float2* Bf = sm + ln;
  const float4* in = reinterpret_cast<const float4*>(P.S1 + (size_t)b * C.ncols * n);
  for (int p = threadIdx.x; p < C.ncols; p += blockDim.x) {
    float4 v = in[((size_t)p * n + y) >> 1];        // (S~1[y][p], S~1[y+1][p])
    float2 cy = make_float2(v.x, v.y), cy1 = make_float2(v.z, v.w);
    if (p == 0 || p == N / 2) {
      float2 z = make_float2(2.f * cy.x, 2.f * cy1.x);    // 2Re + i 2Re
      A[(p % L) * n + p / L] = z;
    } else {
      // Z[p] = cy + i cy1 ; Z[N-p] = conj(cy) + i conj(cy1)
      A[(p % L) * n + p / L] = make_float2(cy.x - cy1.y, cy.y + cy1.x);
      int pm = N - p;
      A[(pm % L) * n + pm / L] = make_float2(cy.x + cy1.y, -cy.y + cy1.x);
    }
  }
  __syncthreads();
  float2* X = smem_fft<1>(A, Bf, n, L, P.tw_n);
  float* o0 = fout + ((size_t)b * n + y) * n;
  for (int x = threadIdx.x; x < n; x += blockDim.x) {
    int xp = (x + n / 2) & (n - 1);
    float2 acc = make_float2(0.f, 0.f);
    for (int s = 0; s < L; ++s)
      acc = cadd(acc, cmulc(X[s * n + xp], __ldg(&P.tw_pre[s * n + xp])));
    o0[x] = acc.x;
    o0[n + x] = acc.y;
  }
}

// ================================================================== launchers
static size_t smem_ring(const Consts& C) { return (size_t)2 * tile_ring(C.n_ring) * C.n_ring * sizeof(float2); }
static size_t smem_ln2(const Consts& C) { return (size_t)2 * C.Lres * C.n * sizeof(float2); }
static size_t smem_k2(const Consts& C) { return (size_t)3 * C.Lres * C.n * sizeof(float2); }
static size_t smem_dct(const Consts& C) { return (size_t)2 * 2 * C.M * sizeof(float2); }

cudaError_t configure_kernels(const DevPlan& P) {
  const Consts& C = P.C;
  cudaError_t e = cudaSuccess;
#define SETSM(kern, bytes)                                                                   \
  if (e == cudaSuccess)                                                                      \
    e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)(bytes));
  if (e == cudaSuccess) e = configure_fft_kernels(C);
  if (e == cudaSuccess) e = configure_ring_kernels(C);
  if (e == cudaSuccess) e = configure_dct_kernels(C);
  SETSM(k3_angular_mult, smem_ring(C));
  SETSM(k4_dct, smem_dct(C));
  SETSM(k5_synth_restrict, smem_ring(C));
  SETSM(k5t_analysis, smem_ring(C));
  SETSM(k4t_dct, smem_dct(C));
  SETSM(k3t_angular, smem_ring(C));

#undef SETSM
  return e;
}

cudaError_t launch_forward(const DevPlan& P, const float* f, float* g, cudaStream_t s,
                           cudaEvent_t* ev) {
  const Consts& C = P.C;
  const int B = C.batch;
  const int JT = tile_ring(C.n_ring);
  if (ev) cudaEventRecord(ev[0], s);
  cudaError_t e = launch_k1(P, f, s);
  if (e != cudaSuccess) return e;
  if (ev) cudaEventRecord(ev[1], s);
  e = launch_k2(P, s);
  if (e != cudaSuccess) return e;
  if (ev) cudaEventRecord(ev[2], s);
  if (ring_fast_ok(C)) e = launch_k3(P, s);
  else k3_angular_mult<<<dim3((C.NL + JT - 1) / JT, B), kThreads, smem_ring(C), s>>>(P);
  if (e != cudaSuccess) return e;
  if (ev) cudaEventRecord(ev[3], s);
  if (dct_fast_r(C)) e = launch_k4_fast(P, false, s);
  else k4_dct<<<dim3(C.Kp, B), kThreads, smem_dct(C), s>>>(P);
  if (e != cudaSuccess) return e;
  if (ev) cudaEventRecord(ev[4], s);
  if (ring_fast_ok(C)) e = launch_k5(P, g, s);
  else k5_synth_restrict<<<dim3((C.n_t + JT - 1) / JT, B), kThreads, smem_ring(C), s>>>(P, g);
  if (e != cudaSuccess) return e;
  if (ev) cudaEventRecord(ev[5], s);
  return cudaGetLastError();
}

cudaError_t launch_adjoint(const DevPlan& P, const float* g, float* f, cudaStream_t s,
                           cudaEvent_t* ev) {
  const Consts& C = P.C;
  const int B = C.batch;
  const int JT = tile_ring(C.n_ring);
  if (ev) cudaEventRecord(ev[0], s);
  cudaError_t e = cudaSuccess;
  if (ring_fast_ok(C)) e = launch_k5t(P, g, s);
  else k5t_analysis<<<dim3((C.n_t + JT - 1) / JT, B), kThreads, smem_ring(C), s>>>(P, g);
  if (e != cudaSuccess) return e;
  if (ev) cudaEventRecord(ev[1], s);
  if (dct_fast_r(C)) e = launch_k4_fast(P, true, s);
  else k4t_dct<<<dim3(C.Kp, B), kThreads, smem_dct(C), s>>>(P);
  if (e != cudaSuccess) return e;
  if (ev) cudaEventRecord(ev[2], s);
  if (ring_fast_ok(C)) e = launch_k3t(P, s);
  else k3t_angular<<<dim3((C.NL + JT - 1) / JT, B), kThreads, smem_ring(C), s>>>(P);
  if (e != cudaSuccess) return e;
  if (ev) cudaEventRecord(ev[3], s);
  e = launch_k2t(P, s);
  if (e != cudaSuccess) return e;
  if (ev) cudaEventRecord(ev[4], s);
  e = launch_k1t(P, f, s);
  if (e != cudaSuccess) return e;
  if (ev) cudaEventRecord(ev[5], s);
  return cudaGetLastError();
}

}  // namespace tat
