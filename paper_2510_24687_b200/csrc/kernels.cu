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
constexpr int kThreads = 256;

size_t max_smem_needed(const Consts& C) {
  size_t s = smem_fft4(C);                                         // K1/K2/K2T/K1T
  if (col_ok(C)) s = std::max(s, smem_k2c_fwd(C));                 // K2 two-stage
  if (dct4_ok(C)) s = std::max(s, smem_k4c(C));
  if (dct_fast_r(C)) s = std::max(s, smem_dct_fast(C));            // K4 / K4T
  else s = std::max(s, (size_t)2 * 2 * C.M * sizeof(float2));
  if (ring_fast_ok(C)) s = std::max(s, smem_ring_fast(C));           // K3/K5
  else s = std::max(s, (size_t)2 * tile_ring(C.n_ring) * C.n_ring * sizeof(float2));
  return s;
}


// K3: angular DFT over the full ring (half plane + conjugate mirror), times i^k m'[k][j].
__global__ void k3_angular_mult(DevPlan P) {
  extern __shared__ float2 sm[];
  const Consts& C = P.C;
  const int nphi = C.n_ring, half = C.half, NL = C.NL, JT = tile_ring(nphi);
  const int b = C.b0 + blockIdx.y, j0 = blockIdx.x * JT;
  const int jt = min(JT, NL - j0);
  float2* A = sm;
  float2* Bf = sm + (size_t)JT * nphi;
  const float2* S2 = P.S2 + (size_t)b * half * NL;
  for (int idx = threadIdx.x; idx < half * JT; idx += blockDim.x) {
    int lp = idx / JT, jj = idx - lp * JT;
    float2 v = (jj < jt) ? S2[(size_t)(j0 + jj) * half + lp] : make_float2(0.f, 0.f);
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
  const int b = C.b0 + blockIdx.y, k = blockIdx.x;
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
  const int b = C.b0 + blockIdx.y, t0 = blockIdx.x * TT, tt_n = min(TT, C.n_t - t0);
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
    const size_t i = ((size_t)b * C.n_t + t0 + tt) * C.n_det + d;
    g[i] = epi_fwd(P, i, X[tt * nphi + __ldg(&P.ring[d])].x);
  }
}

// ================================================================== adjoint kernels
// K5T: zero-extend to the ring, R2C analysis G~[k] = sum_l g_l e^{-i k phi_l}, k in [0, K].
__global__ void k5t_analysis(DevPlan P, const float* __restrict__ g) {
  extern __shared__ float2 sm[];
  const Consts& C = P.C;
  const int nphi = C.n_ring, TT = tile_ring(nphi);
  const int b = C.b0 + blockIdx.y, t0 = blockIdx.x * TT, tt_n = min(TT, C.n_t - t0);
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
  const int b = C.b0 + blockIdx.y, k = blockIdx.x;
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
  const int b = C.b0 + blockIdx.y, j0 = blockIdx.x * JT, jt = min(JT, NL - j0);
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
    S2[P.node_perm[(size_t)(j0 + jj) * half + lp]] = X[jj * nphi + l];
  }
}

// ================================================================== launchers
static size_t smem_ring(const Consts& C) { return (size_t)2 * tile_ring(C.n_ring) * C.n_ring * sizeof(float2); }
static size_t smem_dct(const Consts& C) { return (size_t)2 * 2 * C.M * sizeof(float2); }

cudaError_t configure_kernels(const DevPlan& P) {
  const Consts& C = P.C;
  cudaError_t e = cudaSuccess;
#define SETSM(kern, bytes)                                                                   \
  if (e == cudaSuccess)                                                                      \
    e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)(bytes));
  if (e == cudaSuccess) e = configure_fft_kernels(C);
  if (e == cudaSuccess) e = configure_col_kernels(C);
  if (e == cudaSuccess) e = configure_ring_kernels(C);
  if (e == cudaSuccess) e = configure_dct_kernels(C);
  if (e == cudaSuccess) e = configure_dense_kernels(C);
  if (smem_ring(C) > (size_t)kSmemLimit || smem_dct(C) > (size_t)kSmemLimit) return cudaErrorInvalidConfiguration;
  SETSM(k3_angular_mult, kSmemLimit);
  SETSM(k4_dct, kSmemLimit);
  SETSM(k5_synth_restrict, kSmemLimit);
  SETSM(k5t_analysis, kSmemLimit);
  SETSM(k4t_dct, kSmemLimit);
  SETSM(k3t_angular, kSmemLimit);

#undef SETSM
  return e;
}

cudaError_t launch_forward(const DevPlan& P, const CUtensorMap& tm, const float* f, float* g,
                           cudaStream_t s, cudaEvent_t* ev) {
  const Consts& C = P.C;
  const int B = C.batch;
  const int JT = tile_ring(C.n_ring);
  if (ev) cudaEventRecord(ev[0], s);
  cudaError_t e = cudaSuccess;
  if (P.lowk_add)   // reading G25: c sum(f) per image, added in the last kernel's epilogue
    e = launch_lowk_sum(P, f, (size_t)C.n * C.n, C.lowk_c, true, s);
  if (e != cudaSuccess) return e;
  e = launch_k1(P, tm, f, s);
  if (e != cudaSuccess) return e;
  if (ev) cudaEventRecord(ev[1], s);
  e = launch_k2(P, tm, s);
  if (e != cudaSuccess) return e;
  if (ev) cudaEventRecord(ev[2], s);
  if (ring_fast_ok(C)) e = launch_k3(P, s);
  else k3_angular_mult<<<dim3((C.NL + JT - 1) / JT, B), kThreads, smem_ring(C), s>>>(P);
  if (e != cudaSuccess) return e;
  if (ev) cudaEventRecord(ev[3], s);
  if (dct4_ok(C)) e = launch_k4c(P, false, s);
  else if (dct_fast_r(C)) e = launch_k4_fast(P, false, s);
  else k4_dct<<<dim3(C.Kp, B), kThreads, smem_dct(C), s>>>(P);
  if (e != cudaSuccess) return e;
  if (ev) cudaEventRecord(ev[4], s);
  if (C.dense) e = C.k5tc_kp > 0 ? launch_k5d_tc(P, g, s) : launch_k5d(P, g, s);
  else if (ring_fast_ok(C)) e = launch_k5(P, g, s);
  else k5_synth_restrict<<<dim3((C.n_t + JT - 1) / JT, B), kThreads, smem_ring(C), s>>>(P, g);
  if (e != cudaSuccess) return e;
  if (ev) cudaEventRecord(ev[5], s);
  return cudaGetLastError();
}

cudaError_t launch_adjoint(const DevPlan& P, const CUtensorMap& tm, const float* g, float* f,
                           cudaStream_t s, cudaEvent_t* ev) {
  const Consts& C = P.C;
  const int B = C.batch;
  const int JT = tile_ring(C.n_ring);
  if (ev) cudaEventRecord(ev[0], s);
  cudaError_t e = cudaSuccess;
  if (P.lowk_add)   // reading G25: omega c sum(g) per image, added in K1T's epilogue
    e = launch_lowk_sum(P, g, (size_t)C.n_t * C.n_det, C.omega * C.lowk_c, false, s);
  if (e != cudaSuccess) return e;
  if (C.dense) e = C.k5ttc_kp > 0 ? launch_k5dt_tc(P, g, s) : launch_k5dt(P, g, s);
  else if (ring_fast_ok(C)) e = launch_k5t(P, g, s);
  else k5t_analysis<<<dim3((C.n_t + JT - 1) / JT, B), kThreads, smem_ring(C), s>>>(P, g);
  if (e != cudaSuccess) return e;
  if (ev) cudaEventRecord(ev[1], s);
  if (dct4_ok(C)) e = launch_k4c(P, true, s);
  else if (dct_fast_r(C)) e = launch_k4_fast(P, true, s);
  else k4t_dct<<<dim3(C.Kp, B), kThreads, smem_dct(C), s>>>(P);
  if (e != cudaSuccess) return e;
  if (ev) cudaEventRecord(ev[2], s);
  if (ring_fast_ok(C)) e = launch_k3t(P, s);
  else k3t_angular<<<dim3((C.NL + JT - 1) / JT, B), kThreads, smem_ring(C), s>>>(P);
  if (e != cudaSuccess) return e;
  if (ev) cudaEventRecord(ev[3], s);
  e = launch_k2t(P, s, ev ? ev[6] : nullptr);
  if (e != cudaSuccess) return e;
  if (ev) cudaEventRecord(ev[4], s);
  e = launch_k1t(P, tm, f, s);
  if (e != cudaSuccess) return e;
  if (ev) cudaEventRecord(ev[5], s);
  return cudaGetLastError();
}

// Algorithm 3 through step 6: the adjoint chain with the sine transform and the
// J' multiplier (P has dct_sine = 1, omega = 1, the inverse tables), the polar -> Cartesian
// interpolation in place of K2Ta.  Steps 7-8 (constant, projection) are launched by the caller.
cudaError_t launch_inverse(const DevPlan& P, const CUtensorMap& tm, const float* g, float* f,
                           cudaStream_t s) {
  const Consts& C = P.C;
  cudaError_t e = cudaSuccess;
  if (ring_fast_ok(C)) e = launch_k5t(P, g, s);
  else k5t_analysis<<<dim3((C.n_t + tile_ring(C.n_ring) - 1) / tile_ring(C.n_ring), C.batch), kThreads,
                      smem_ring(C), s>>>(P, g);
  if (e != cudaSuccess) return e;
  if (dct4_ok(C)) e = launch_k4c(P, true, s);
  else if (dct_fast_r(C)) e = launch_k4_fast(P, true, s);
  else return cudaErrorNotSupported;
  if (e != cudaSuccess) return e;
  if (ring_fast_ok(C)) e = launch_k3t(P, s);
  else k3t_angular<<<dim3((C.NL + tile_ring(C.n_ring) - 1) / tile_ring(C.n_ring), C.batch), kThreads,
                     smem_ring(C), s>>>(P);
  if (e != cudaSuccess) return e;
  e = launch_k2i_interp(P, s);
  if (e != cudaSuccess) return e;
  e = launch_k2tb(P, s);
  if (e != cudaSuccess) return e;
  e = launch_k1t(P, tm, f, s);
  if (e != cudaSuccess) return e;
  return cudaGetLastError();
}

}  // namespace tat
