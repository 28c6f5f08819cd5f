// Angular-harmonic kernels on the register FFT engine (n_phi-point transforms):
//
//   K3   S2 [B][n_phi/2][NL] -> S3 [B][K+1][NL]  angular DFT (E:eq3) of the polar
//        samples, completed from the half plane by P(phi + pi) = conj P(phi) (reading G12), times
//        i^k m'[k][j] (E:eq2; 1/n_phi and h^2/2pi folded into m').
//   K3T  S3 -> S2  transpose: P~[l] = sum_{k=-K}^{K-1} H~_k e^{i k phi_l} on the half plane, with
//        H~_{-k} = (-1)^k conj(H~_k) and H~_{-K} = H~_K.
//   K5   S4 [B][K+1][n_t] -> g [B][n_t][n_det]  C2R angular synthesis (E:FourSerForg)
//        restricted to the detectors (Alg.1 steps 6-7); two time samples per complex FFT.
//   K5T  g -> S4  zero-extension to the ring + R2C analysis (Alg.2 steps 1-2).
//
// Each CTA stages its tile through shared memory so that every global access is a contiguous
// run along the fastest axis, then runs G transforms with cta_fft (G = blockDim.x / (n_phi/8)).
#include "fft_engine.cuh"
#include "tat_internal.h"

namespace tat {
#ifdef TAT_RING_NOFFT   // timing experiment only: skip the transform (wrong results)
#define TAT_RING_FFT(nf, S) (__syncthreads(), A)
#else
#define TAT_RING_FFT(nf, S) cta_fft_g<nf, S>(A, B, P.tw_ring)
#endif

using namespace fe;

template <int nf>
__host__ __device__ constexpr int ring_G() {
  return (4096 / nf) < 16 ? (4096 / nf) : 16;   // transforms per CTA (<= 512 threads)
}

__device__ __forceinline__ float2 mul_ipow_(float2 a, int e) {
  switch (e & 3) {
    case 0: return a;
    case 1: return make_float2(-a.y, a.x);
    case 2: return make_float2(-a.x, -a.y);
    default: return make_float2(a.y, -a.x);
  }
}

// Global loads of each phase are issued together (unrolled item loops, registers) before any
// dependent work, so a CTA pays one memory latency per phase.

// ------------------------------------------------------------------ K3
// Two rings per complex FFT: Z = P_1 + i P_2 (each ring completed from the half plane by
// P(l + n/2) = conj P(l)); since F(-k) = (-1)^k conj F(k) for each ring,
//   F_1[k] = (Z[k] + (-1)^k conj Z[-k]) / 2,  F_2[k] = (Z[k] - (-1)^k conj Z[-k]) / (2i).
template <int nf>
__global__ void __launch_bounds__(512) k3_ring(DevPlan P) {
  extern __shared__ float2 sm[];
  constexpr int G = ring_G<nf>();   // transforms per CTA (2G rings)
  constexpr int rs = rstride(nf);
  constexpr int T = G * nf / 8, Kp = nf / 2 + 1, half = nf / 2;
  constexpr int NIN = half * G / T;                      // = 4
  constexpr int NOUT = (Kp * G + T - 1) / T;             // <= 5 items (k, ring pair)
  const Consts& C = P.C;
  const int NL = C.NL;
  const int b = C.b0 + blockIdx.y, j0 = blockIdx.x * (2 * G);
  float2* A = sm;
  float2* B = sm + G * rs;
  const float2* S2 = P.S2 + (size_t)b * half * NL;
  // output item (k, gg): both rings of transform gg at harmonic k (one pair of reads of the
  // spectrum for the two outputs); multiplier values loaded early
  float2 mo[NOUT];
#pragma unroll
  for (int u = 0; u < NOUT; ++u) {
    const int idx = threadIdx.x + u * T;
    const int k = idx / G, ja = j0 + 2 * (idx - k * G);
    const bool ok = idx < Kp * G;
    mo[u] = make_float2((ok && ja < NL) ? __ldg(&P.mult[(size_t)k * NL + ja]) : 0.f,
                        (ok && ja + 1 < NL) ? __ldg(&P.mult[(size_t)k * NL + ja + 1]) : 0.f);
  }
  pdl_wait();
  pdl_trigger();
  float2 va[NIN], vb[NIN];
#pragma unroll
  for (int u = 0; u < NIN; ++u) {
    const int idx = threadIdx.x + u * T;
    const int gg = idx / half, lp = idx - gg * half;
    const int ja = j0 + 2 * gg;
    va[u] = ja < NL ? S2[(size_t)ja * half + lp] : make_float2(0.f, 0.f);
    vb[u] = ja + 1 < NL ? S2[(size_t)(ja + 1) * half + lp] : make_float2(0.f, 0.f);
  }
#pragma unroll
  for (int u = 0; u < NIN; ++u) {
    const int idx = threadIdx.x + u * T;
    const int gg = idx / half, lp = idx - gg * half;
    const int l = (lp - nf / 4) & (nf - 1);
    A[gg * rs + phys(l)] = make_float2(va[u].x - vb[u].y, va[u].y + vb[u].x);   // va + i vb
    A[gg * rs + phys((l + half) & (nf - 1))] = make_float2(va[u].x + vb[u].y, -va[u].y + vb[u].x);
  }
  const float2* X = TAT_RING_FFT(nf, -1);
  float2* S3 = P.S3 + (size_t)b * C.Kp * NL;
#pragma unroll
  for (int u = 0; u < NOUT; ++u) {
    const int idx = threadIdx.x + u * T;
    const int k = idx / G, gg = idx - k * G, ja = j0 + 2 * gg;
    if (idx < Kp * G && ja < NL) {
      const float2 zk = X[gg * rs + phys(k)];
      float2 zm = X[gg * rs + phys((nf - k) & (nf - 1))];
      if (k & 1) zm = make_float2(-zm.x, -zm.y);
      // F1 = (zk + conj zm)/2 ; F2 = (zk - conj zm)/(2i)
      const float2 F1 = make_float2(0.5f * (zk.x + zm.x), 0.5f * (zk.y - zm.y));
      const float2 F2 = make_float2(0.5f * (zk.y + zm.y), -0.5f * (zk.x - zm.x));
      float2* o = S3 + (size_t)k * NL + ja;
      o[0] = mul_ipow_(cscale(F1, mo[u].x), k);   // (measured: ipow_scale here 37.3 -> 39.1 us at C4)
      if (ja + 1 < NL) o[1] = mul_ipow_(cscale(F2, mo[u].y), k);
    }
  }
}

// ------------------------------------------------------------------ K3T
// Two rings per complex inverse FFT: spectra completed by H~_{-k} = (-1)^k conj H~_k, packed
// Z = E_1 + i E_2; the outputs satisfy P~(l + n/2) = conj P~(l), so
//   P~_1[l] = (z[l] + conj z[l + n/2]) / 2,  P~_2[l] = (z[l] - conj z[l + n/2]) / (2i).
template <int nf>
__global__ void __launch_bounds__(512) k3t_ring(DevPlan P) {
  extern __shared__ float2 sm[];
  constexpr int G = ring_G<nf>();
  constexpr int rs = rstride(nf);
  constexpr int T = G * nf / 8, Kp = nf / 2 + 1, half = nf / 2, K = nf / 2;
  constexpr int NIN = (Kp * G + T - 1) / T;   // <= 5
  constexpr int NOUT = half * 2 * G / T;      // = 8
  const Consts& C = P.C;
  const int NL = C.NL;
  const int b = C.b0 + blockIdx.y, j0 = blockIdx.x * (2 * G);
  float2* A = sm;
  float2* B = sm + G * rs;
  const float2* S3 = P.S3 + (size_t)b * C.Kp * NL;
  pdl_wait();
  pdl_trigger();
  float2 e1[NIN], e2[NIN];
#pragma unroll
  for (int u = 0; u < NIN; ++u) {
    const int idx = threadIdx.x + u * T;
    const int k = idx / G, gg = idx - k * G;
    const int ja = j0 + 2 * gg;
    const bool ok = idx < Kp * G;
    e1[u] = (ok && ja < NL) ? S3[(size_t)k * NL + ja] : make_float2(0.f, 0.f);
    e2[u] = (ok && ja + 1 < NL) ? S3[(size_t)k * NL + ja + 1] : make_float2(0.f, 0.f);
  }
#pragma unroll
  for (int u = 0; u < NIN; ++u) {
    const int idx = threadIdx.x + u * T;
    if (idx < Kp * G) {
      const int k = idx / G, gg = idx - k * G;
      A[gg * rs + phys(k)] = make_float2(e1[u].x - e2[u].y, e1[u].y + e2[u].x);   // slot K is -K
      if (k >= 1 && k < K) {
        const float sg = (k & 1) ? -1.f : 1.f;   // E(-k) = (-1)^k conj E(k)
        A[gg * rs + phys(nf - k)] = make_float2(sg * (e1[u].x + e2[u].y), sg * (-e1[u].y + e2[u].x));
      }
    }
  }
  // outputs in adjoint-S2 order (k3t_dst: this ring group's nodes sorted by position, ring-major
  // runs inside each column), so that consecutive threads store to consecutive positions;
  // the (position, source) pairs are loaded before the transform
  const int nout = min(2 * G, NL - j0) * half;
  const int2* dst = P.k3t_dst + (size_t)j0 * half;
  int2 dd[NOUT];
#pragma unroll
  for (int u = 0; u < NOUT; ++u) {
    const int idx = threadIdx.x + u * T;
    dd[u] = idx < nout ? __ldg(&dst[idx]) : make_int2(0, 0);
  }
  const float2* X = TAT_RING_FFT(nf, 1);
  float2* S2 = P.S2 + (size_t)b * half * NL;
#pragma unroll
  for (int u = 0; u < NOUT; ++u) {
    const int idx = threadIdx.x + u * T;
    if (idx < nout) {
      const int jj = dd[u].y >> 11, lp = dd[u].y & 2047, gg = jj >> 1;
      const int l = (lp - nf / 4) & (nf - 1);
      const float2 z = X[gg * rs + phys(l)];
      const float2 zh = X[gg * rs + phys((l + half) & (nf - 1))];
      S2[dd[u].x] = (jj & 1) ? make_float2(0.5f * (z.y + zh.y), -0.5f * (z.x - zh.x))
                             : make_float2(0.5f * (z.x + zh.x), 0.5f * (z.y - zh.y));
    }
  }
}

// ------------------------------------------------------------------ K5
// transform g carries time samples t0 + 2g (real part) and t0 + 2g + 1 (imaginary part)
template <int nf, bool VAR, bool SUB>
__global__ void __launch_bounds__(512) k5_ring(DevPlan P, float* __restrict__ gout) {
  extern __shared__ float2 sm[];
  constexpr int G = ring_G<nf>();
  constexpr int rs = rstride(nf);
  constexpr int T = G * nf / 8, Kp = nf / 2 + 1, K = nf / 2;
  constexpr int NIN = (Kp * G + T - 1) / T;   // <= 5
  const Consts& C = P.C;
  const int n_t = C.n_t, n_det = C.n_det;
  const int b = C.b0 + blockIdx.y, t0 = blockIdx.x * (2 * G);
  float2* A = sm;
  float2* B = sm + G * rs;
  const float2* S4 = P.S4 + (size_t)b * C.Kp * n_t;
  const int tt_n = min(2 * G, n_t - t0);
  // fused residual (A x - g_obs): this thread's first detector's g_obs samples, loaded before
  // the dependency wait (g_obs is an input of the whole chain)
  const bool pre = SUB && (int)threadIdx.x < n_det;   // SUB: launched for plans with epi_sub
  float es[2 * G];
  if (pre) {
    const float* sb = P.epi_sub + ((size_t)b * n_t + t0) * n_det + threadIdx.x;
#pragma unroll
    for (int tt = 0; tt < 2 * G; ++tt) es[tt] = tt < tt_n ? __ldg(&sb[(size_t)tt * n_det]) : 0.f;
  }
  pdl_wait();
  pdl_trigger();
  float2 w0[NIN], w1[NIN];
#pragma unroll
  for (int u = 0; u < NIN; ++u) {
    const int idx = threadIdx.x + u * T;
    const int k = idx / G, gg = idx - k * G;
    const int t = t0 + 2 * gg;
    const bool ok = idx < Kp * G;
    w0[u] = (ok && t < n_t) ? S4[(size_t)k * n_t + t] : make_float2(0.f, 0.f);
    w1[u] = (ok && t + 1 < n_t) ? S4[(size_t)k * n_t + t + 1] : make_float2(0.f, 0.f);
  }
#pragma unroll
  for (int u = 0; u < NIN; ++u) {
    const int idx = threadIdx.x + u * T;
    if (idx < Kp * G) {
      const int k = idx / G, gg = idx - k * G;
      const float2 v0 = w0[u], v1 = w1[u];
      if (k >= 1 && k < K) {
        A[gg * rs + phys(k)] = make_float2(v0.x - v1.y, v0.y + v1.x);          // v0 + i v1
        A[gg * rs + phys(nf - k)] = make_float2(v0.x + v1.y, -v0.y + v1.x);   // conj v0 + i conj v1
      } else {   // k = 0 and the Nyquist k = K enter through their real parts (C2R convention)
        A[gg * rs + phys(k)] = make_float2(v0.x, v1.x);
      }
    }
  }
  const float2* X = TAT_RING_FFT(nf, 1);
  // detector-major loop (no integer division): thread d restricts all 2G samples of detector d
  for (int d = threadIdx.x; d < n_det; d += blockDim.x) {
    const int pos = phys(__ldg(&P.ring[d]));
    const size_t i0 = ((size_t)b * n_t + t0) * n_det + d;
    if (pre && d == (int)threadIdx.x) {
#pragma unroll
      for (int gg = 0; gg < G; ++gg) {
        if (2 * gg < tt_n) {
          const float2 z = X[gg * rs + pos];
          const size_t i = i0 + (size_t)(2 * gg) * n_det;
          gout[i] = epi_fwd_pre<VAR>(P, i, z.x, es[2 * gg]);
          if (2 * gg + 1 < tt_n) gout[i + n_det] = epi_fwd_pre<VAR>(P, i + n_det, z.y, es[2 * gg + 1]);
        }
      }
      continue;
    }
#pragma unroll
    for (int gg = 0; gg < G; ++gg) {   // transform gg: samples 2 gg (real part), 2 gg + 1 (imag)
      if (2 * gg < tt_n) {
        const float2 z = X[gg * rs + pos];
        const size_t i = i0 + (size_t)(2 * gg) * n_det;
        gout[i] = epi_fwd<VAR>(P, i, z.x);
        if (2 * gg + 1 < tt_n) gout[i + n_det] = epi_fwd<VAR>(P, i + n_det, z.y);
      }
    }
  }
}

// ------------------------------------------------------------------ K5T
template <int nf>
__global__ void __launch_bounds__(512) k5t_ring(DevPlan P, const float* __restrict__ gin) {
  extern __shared__ float2 sm[];
  constexpr int G = ring_G<nf>();
  constexpr int rs = rstride(nf);
  constexpr int T = G * nf / 8, Kp = nf / 2 + 1;
  constexpr int NOUT = (Kp * G + T - 1) / T;  // <= 5
  const Consts& C = P.C;
  const int n_t = C.n_t, n_det = C.n_det;
  const int b = C.b0 + blockIdx.y, t0 = blockIdx.x * (2 * G);
  float2* A = sm;
  float2* B = sm + G * rs;
  const int tt_n = min(2 * G, n_t - t0);
  for (int i = threadIdx.x; i < G * rs; i += blockDim.x) A[i] = make_float2(0.f, 0.f);
  pdl_wait();
  pdl_trigger();
  __syncthreads();
  // detector-major (no integer division): thread d places the 2G samples of detector d, the
  // pair (2 gg, 2 gg + 1) as transform gg's (real, imag) at ring position r_d
  for (int d = threadIdx.x; d < n_det; d += blockDim.x) {
    const int pos = phys(__ldg(&P.ring[d]));
    const float* gi = gin + ((size_t)b * n_t + t0) * n_det + d;
    float gv[2 * G];
#pragma unroll
    for (int tt = 0; tt < 2 * G; ++tt) gv[tt] = tt < tt_n ? gi[(size_t)tt * n_det] : 0.f;
#pragma unroll
    for (int gg = 0; gg < G; ++gg) A[gg * rs + pos] = make_float2(gv[2 * gg], gv[2 * gg + 1]);
  }
  const float2* X = TAT_RING_FFT(nf, -1);
  float2* S4 = P.S4 + (size_t)b * C.Kp * n_t;
#pragma unroll
  for (int u = 0; u < NOUT; ++u) {
    const int idx = threadIdx.x + u * T;
    if (idx < Kp * G) {
      const int k = idx / G, gg = idx - k * G;
      const int t = t0 + 2 * gg;
      const float2 zk = X[gg * rs + phys(k)];
      const float2 zm = X[gg * rs + phys((nf - k) & (nf - 1))];
      // even sample: (Z[k] + conj Z[-k]) / 2 ; odd sample: (Z[k] - conj Z[-k]) / (2i)
      const float2 ge = make_float2(0.5f * (zk.x + zm.x), 0.5f * (zk.y - zm.y));
      const float2 go = make_float2(0.5f * (zk.y + zm.y), -0.5f * (zk.x - zm.x));
      if (t < n_t) S4[(size_t)k * n_t + t] = ge;
      if (t + 1 < n_t) S4[(size_t)k * n_t + t + 1] = go;
    }
  }
}

// ------------------------------------------------------------------ dispatch
bool ring_fast_ok(const Consts& C) { return C.n_ring >= 32 && C.n_ring <= 2048; }

size_t smem_ring_fast(const Consts& C) {
  const int nf = C.n_ring;
  const int G = (4096 / nf) < 16 ? (4096 / nf) : 16;
  return (size_t)2 * G * rstride(nf) * sizeof(float2);
}

#define TAT_RING_SWITCH(...)                      \
  switch (C.n_ring) {                              \
    case 32: { constexpr int NF = 32; __VA_ARGS__; } break;     \
    case 64: { constexpr int NF = 64; __VA_ARGS__; } break;     \
    case 128: { constexpr int NF = 128; __VA_ARGS__; } break;   \
    case 256: { constexpr int NF = 256; __VA_ARGS__; } break;   \
    case 512: { constexpr int NF = 512; __VA_ARGS__; } break;   \
    case 1024: { constexpr int NF = 1024; __VA_ARGS__; } break; \
    case 2048: { constexpr int NF = 2048; __VA_ARGS__; } break; \
    default: return cudaErrorInvalidValue;          \
  }

cudaError_t configure_ring_kernels(const Consts& C) {
  if (!ring_fast_ok(C)) return cudaSuccess;
  if (smem_ring_fast(C) > (size_t)kSmemLimit) return cudaErrorInvalidConfiguration;
  const int sm = kSmemLimit;
  cudaError_t e = cudaSuccess;
  TAT_RING_SWITCH({
    if (e == cudaSuccess) e = cudaFuncSetAttribute(k3_ring<NF>, cudaFuncAttributeMaxDynamicSharedMemorySize, sm);
    if (e == cudaSuccess) e = cudaFuncSetAttribute(k3t_ring<NF>, cudaFuncAttributeMaxDynamicSharedMemorySize, sm);
    if (e == cudaSuccess) e = cudaFuncSetAttribute(k5_ring<NF, false, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, sm);
    if (e == cudaSuccess) e = cudaFuncSetAttribute(k5_ring<NF, true, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, sm);
    if (e == cudaSuccess) e = cudaFuncSetAttribute(k5_ring<NF, false, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, sm);
    if (e == cudaSuccess) e = cudaFuncSetAttribute(k5_ring<NF, true, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, sm);
    if (e == cudaSuccess) e = cudaFuncSetAttribute(k5t_ring<NF>, cudaFuncAttributeMaxDynamicSharedMemorySize, sm);
  });
  if (e == cudaSuccess) e = configure_ring2_kernels(C);
  return e;
}

cudaError_t launch_k3(const DevPlan& P, cudaStream_t s) {
  const Consts& C = P.C;
  cudaError_t e = cudaSuccess;
  if (ring2_on(C, 1)) return launch_ring2(P, 1, nullptr, nullptr, s);
  const size_t sm = smem_ring_fast(C);
  TAT_RING_SWITCH({
    constexpr int G = ring_G<NF>();
    e = launch_pdl(C.pdl, k3_ring<NF>, dim3((C.NL + 2 * G - 1) / (2 * G), C.batch), dim3(G * NF / 8), sm, s, P);
  });
  return e != cudaSuccess ? e : cudaGetLastError();
}
cudaError_t launch_k3t(const DevPlan& P, cudaStream_t s) {
  const Consts& C = P.C;
  cudaError_t e = cudaSuccess;
  if (ring2_on(C, 2)) return launch_ring2(P, 2, nullptr, nullptr, s);
  const size_t sm = smem_ring_fast(C);
  TAT_RING_SWITCH({
    constexpr int G = ring_G<NF>();
    e = launch_pdl(C.pdl, k3t_ring<NF>, dim3((C.NL + 2 * G - 1) / (2 * G), C.batch), dim3(G * NF / 8), sm, s, P);
  });
  return e != cudaSuccess ? e : cudaGetLastError();
}
cudaError_t launch_k5(const DevPlan& P, float* g, cudaStream_t s) {
  const Consts& C = P.C;
  cudaError_t e = cudaSuccess;
  if (ring2_on(C, 4)) return launch_ring2(P, 4, nullptr, g, s);
  const size_t sm = smem_ring_fast(C);
  TAT_RING_SWITCH({
    constexpr int G = ring_G<NF>();
    const dim3 grid((C.n_t + 2 * G - 1) / (2 * G), C.batch), blk(G * NF / 8);
    if (P.lowk_add)
      e = P.epi_sub ? launch_pdl(C.pdl, k5_ring<NF, true, true>, grid, blk, sm, s, P, g)
                    : launch_pdl(C.pdl, k5_ring<NF, true, false>, grid, blk, sm, s, P, g);
    else
      e = P.epi_sub ? launch_pdl(C.pdl, k5_ring<NF, false, true>, grid, blk, sm, s, P, g)
                    : launch_pdl(C.pdl, k5_ring<NF, false, false>, grid, blk, sm, s, P, g);
  });
  return e != cudaSuccess ? e : cudaGetLastError();
}
cudaError_t launch_k5t(const DevPlan& P, const float* g, cudaStream_t s) {
  const Consts& C = P.C;
  cudaError_t e = cudaSuccess;
  if (ring2_on(C, 8)) return launch_ring2(P, 8, g, nullptr, s);
  const size_t sm = smem_ring_fast(C);
  TAT_RING_SWITCH({
    constexpr int G = ring_G<NF>();
    e = launch_pdl(C.pdl, k5t_ring<NF>, dim3((C.n_t + 2 * G - 1) / (2 * G), C.batch), dim3(G * NF / 8), sm, s, P, g);
  });
  return e != cudaSuccess ? e : cudaGetLastError();
}

}  // namespace tat
