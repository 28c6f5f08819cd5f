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
#include "col_engine.cuh"
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
// i^e m a without branches (e varies across the lanes of a warp): the sign of i^e folded into m
__device__ __forceinline__ float2 ipow_scale(float2 a, float m, int e) {
  const float2 r = (e & 1) ? make_float2(-a.y, a.x) : a;
  return cscale(r, (e & 2) ? -m : m);
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

// ------------------------------------------------------------------ K3, two-stage (n_phi = 512)
// The same transform as k3_ring with one shared-memory crossing per point instead of a Stockham
// pass per radix-8 level: l = j + 16 r, k = k1 + 32 k2,
//   Z[k1 + 32 k2] = sum_j W_16^{j k2} W_512^{j k1} sum_r z[j + 16 r] W_32^{r k1}.
// Stage A (thread (j, gg)): the 16 half-plane samples j + 16 m of both rings of ring pair gg are
// loaded straight from S2 into registers (coalesced: consecutive j, consecutive l'); each gives
// two points of the completed ring (l and l + 256, the second conjugated); 32-point DFT over r,
// twiddle W_512^{j k1}, one store per point.  Stage B (thread (kp, gg)): the two 16-point DFTs over
// j of k1 = kp and k1 = 32 - kp (kp = 0: k1 = 0 and 16), so that Z[k] and Z[-k] -- both needed
// to separate the two rings -- are in the same thread; outputs stored straight to S3 (the
// threads of one kp cover 2G consecutive rings: contiguous runs of S3 row k).
namespace {
constexpr int kR2G = kRing2G;                       // ring pairs per CTA (32 rings)
constexpr int kR2P = 33;                            // Y row stride (j): odd
constexpr int kR2S = 16 * kR2P + 16 / kR2G;         // Y stride per ring pair: odd for G = 16
}  // namespace
#ifndef TAT_R2_MINB
#define TAT_R2_MINB 2   // CTAs per SM the two-stage ring kernels are compiled for
#endif
#ifndef TAT_R2_MINB_K3
#define TAT_R2_MINB_K3 TAT_R2_MINB
#endif
#ifndef TAT_R2_MINB_K3T
#define TAT_R2_MINB_K3T TAT_R2_MINB
#endif
#ifndef TAT_R2_MINB_K5
#define TAT_R2_MINB_K5 TAT_R2_MINB
#endif
#ifndef TAT_R2_MINB_K5T
#define TAT_R2_MINB_K5T 3
#endif
#ifndef TAT_R2_TWLD
#define TAT_R2_TWLD 0   // stage-A twiddles W^{j k1}: 1 = table loads (L1), 0 = powers in registers
#endif
// y[k1] = x[k1] W_512^{+-j k1} (CONJ: the conjugate twiddles), k1 < 32
template <bool CONJ>
__device__ __forceinline__ void r2_twiddle_store(float2* y, const float2 (&x)[32], const float2* __restrict__ tw,
                                                 int j) {
  y[0] = x[0];
#if TAT_R2_TWLD
#pragma unroll
  for (int k1 = 1; k1 < 32; ++k1) {
    const float2 w = __ldg(&tw[(j * k1) & 511]);
    y[k1] = CONJ ? cmulc(x[k1], w) : cmul(x[k1], w);
  }
#else
  float2 pw[32];
  const float2 w = __ldg(&tw[j]);
  ce::pow_tree<32>(CONJ ? make_float2(w.x, -w.y) : w, pw);
#pragma unroll
  for (int k1 = 1; k1 < 32; ++k1) y[k1] = cmul(x[k1], pw[k1]);
#endif
}
__global__ void __launch_bounds__(16 * kR2G, TAT_R2_MINB_K3) k3_ring2(DevPlan P) {
  constexpr int half = 256, G = kR2G;   // n_phi = 512
  extern __shared__ float2 sm[];
  const Consts& C = P.C;
  const int NL = C.NL;
  const int b = C.b0 + blockIdx.y, j0 = blockIdx.x * (2 * G);
  const float2* S2 = P.S2 + (size_t)b * half * NL;
  float2* Y = sm;
  pdl_wait();
  pdl_trigger();
  {   // stage A
    const int j = threadIdx.x & 15, gg = threadIdx.x >> 4, ja = j0 + 2 * gg;
    const float2* ra = S2 + (size_t)ja * half + j;
    float2 va[16], vb[16];
#pragma unroll
    for (int m = 0; m < 16; ++m) {
      va[m] = ja < NL ? ra[16 * m] : make_float2(0.f, 0.f);
      vb[m] = ja + 1 < NL ? ra[half + 16 * m] : make_float2(0.f, 0.f);
    }
    float2 x[32];
#pragma unroll
    for (int m = 0; m < 16; ++m) {
      const float2 d = make_float2(va[m].x - vb[m].y, va[m].y + vb[m].x);    // va + i vb
      const float2 c = make_float2(va[m].x + vb[m].y, -va[m].y + vb[m].x);   // conj va + i conj vb
      x[m < 8 ? m + 24 : m - 8] = d;   // l' = j + 16 m -> l = l' - 128 (mod 512)
      x[m + 8] = c;                    // l + 256
    }
    ce::dftr<32, -1>(x);
    r2_twiddle_store<false>(Y + gg * kR2S + j * kR2P, x, P.tw_ring, j);   // x W_512^{j k1}
  }
  // multiplier values of this thread's 16 (kp = 0: 17) outputs, loaded before the barrier so
  // that their latency overlaps stage B (output slot s: k = kout(s), see below)
  const int gg = threadIdx.x % G, kp = threadIdx.x / G, ja = j0 + 2 * gg;
  const int ka = kp == 0 ? 0 : kp, kb = kp == 0 ? 16 : 32 - kp;
  auto kout = [&](int s) { return kp == 0 ? (s <= 8 ? 32 * s : 16 + 32 * (s - 9)) : (s < 8 ? ka + 32 * s : kb + 32 * (s - 8)); };
  const bool ok0 = ja < NL, ok1 = ja + 1 < NL;
  float2 mo[17];
#pragma unroll
  for (int s = 0; s < 17; ++s) {
    const int k = kout(s);
    const bool v = s < 16 || kp == 0;
    mo[s] = make_float2(v && ok0 ? __ldg(&P.mult[(size_t)k * NL + ja]) : 0.f,
                        v && ok1 ? __ldg(&P.mult[(size_t)k * NL + ja + 1]) : 0.f);
  }
  __syncthreads();
  {   // stage B + output
    const float2* y = Y + gg * kR2S;
    float2 za[16], zb[16];
#pragma unroll
    for (int j = 0; j < 16; ++j) {
      za[j] = y[j * kR2P + ka];
      zb[j] = y[j * kR2P + kb];
    }
    ce::dftr<16, -1>(za);   // Z[ka + 32 k2]
    ce::dftr<16, -1>(zb);   // Z[kb + 32 k2]
    float2* S3 = P.S3 + (size_t)b * C.Kp * NL;
    // output k from Z[k] and Z[-k]; (k1, k2) -> -k = (32 - k1) + 32 (15 - k2) for k1 > 0,
    // (0, k2) -> (0, 16 - k2) (mod 16)
    auto out = [&](int s, float2 zk, float2 zm) {
      const int k = kout(s);
      if (k & 1) zm = make_float2(-zm.x, -zm.y);
      const float2 F1 = make_float2(0.5f * (zk.x + zm.x), 0.5f * (zk.y - zm.y));
      const float2 F2 = make_float2(0.5f * (zk.y + zm.y), -0.5f * (zk.x - zm.x));
      float2* o = S3 + (size_t)k * NL + ja;
      if (ok0) o[0] = ipow_scale(F1, mo[s].x, k);
      if (ok1) o[1] = ipow_scale(F2, mo[s].y, k);
    };
    if (kp == 0) {
#pragma unroll
      for (int k2 = 0; k2 <= 8; ++k2) out(k2, za[k2 & 15], za[(16 - k2) & 15]);
#pragma unroll
      for (int k2 = 0; k2 < 8; ++k2) out(9 + k2, zb[k2], zb[15 - k2]);
    } else {
#pragma unroll
      for (int k2 = 0; k2 < 8; ++k2) out(k2, za[k2], zb[15 - k2]);
#pragma unroll
      for (int k2 = 0; k2 < 8; ++k2) out(8 + k2, zb[k2], za[15 - k2]);
    }
  }
}

// ------------------------------------------------------------------ K3T, two-stage (n_phi = 512)
// The transpose of k3_ring2, as k3t_ring computes it (below), with k = a + 16 r, l = k1 + 32 k2:
//   z[k1 + 32 k2] = sum_a W_16^{-a k2} W_512^{-a k1} sum_r Z[a + 16 r] W_32^{-r k1}.
// Stage A (thread (a, gg); lanes = ring pairs, so each S3 row k is read as one contiguous run of
// 2G rings): Z[k] for k <= 256 from S3 row k, for k > 256 from row 512 - k by the completion
// (read twice, from L1/L2, instead of a shared-memory pass); 32-point DFT, twiddle.  Stage B
// (thread (kp, gg)): 16-point DFTs of k1 = kp and kp + 16, in place.  Output as in k3t_ring: the
// group's nodes in destination order (k3t_dst, groups of 2G rings).
__global__ void __launch_bounds__(16 * kR2G, TAT_R2_MINB_K3T) k3t_ring2(DevPlan P) {
  constexpr int nf = 512, half = 256, G = kR2G;
  extern __shared__ float2 sm[];
  const Consts& C = P.C;
  const int NL = C.NL;
  const int b = C.b0 + blockIdx.y, j0 = blockIdx.x * (2 * G);
  float2* Y = sm;
  const int gg0 = threadIdx.x % G, i0 = threadIdx.x / G;   // (a or kp, gg) of both stages
  const int ja = j0 + 2 * gg0;
  const bool ok0 = ja < NL, ok1 = ja + 1 < NL;
  pdl_wait();
  pdl_trigger();
  {   // stage A
    const int a = i0;
    const float2* S3 = P.S3 + (size_t)b * C.Kp * NL + ja;
    float2 x[32];
#pragma unroll
    for (int r = 0; r < 32; ++r) {
      const int k = a + 16 * r;
      const bool dir = k <= half;
      const int kk = dir ? k : nf - k;
      const float2 e1 = ok0 ? S3[(size_t)kk * NL] : make_float2(0.f, 0.f);
      const float2 e2 = ok1 ? S3[(size_t)kk * NL + 1] : make_float2(0.f, 0.f);
      if (dir) {
        x[r] = make_float2(e1.x - e2.y, e1.y + e2.x);   // E1 + i E2 (slot 256 is -K)
      } else {
        const float sg = (kk & 1) ? -1.f : 1.f;         // E(-k) = (-1)^k conj E(k)
        x[r] = make_float2(sg * (e1.x + e2.y), sg * (-e1.y + e2.x));
      }
    }
    ce::dftr<32, 1>(x);
    r2_twiddle_store<true>(Y + gg0 * kR2S + a * kR2P, x, P.tw_ring, a);   // x W_512^{-a k1}
  }
  __syncthreads();
  // the output records (position, source) of the first chunk, loaded during stage B
  const int nout = min(2 * G, NL - j0) * half;
  const int2* dst = P.k3t_dst + (size_t)j0 * half;
  constexpr int T = 16 * G, U = 8;
  int2 dd[U];
#pragma unroll
  for (int u = 0; u < U; ++u) {
    const int i = threadIdx.x + u * T;
    dd[u] = i < nout ? __ldg(&dst[i]) : make_int2(0, 0);
  }
  {   // stage B, in place: Y[gg][k2][k1] = z[k1 + 32 k2]
    float2* y = Y + gg0 * kR2S;
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      const int k1 = i0 + 16 * h;
      float2 z[16];
#pragma unroll
      for (int a = 0; a < 16; ++a) z[a] = y[a * kR2P + k1];
      ce::dftr<16, 1>(z);
#pragma unroll
      for (int k2 = 0; k2 < 16; ++k2) y[k2 * kR2P + k1] = z[k2];
    }
  }
  __syncthreads();
  float2* S2 = P.S2 + (size_t)b * half * NL;
  for (int i = threadIdx.x; i < nout; i += U * T) {
    int2 dn[U];   // next chunk's records, in flight while this chunk is stored
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int in = i + (U + u) * T;
      dn[u] = in < nout ? __ldg(&dst[in]) : make_int2(0, 0);
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
      if (i + u * T < nout) {
        const int jj = dd[u].y >> 11, lp = dd[u].y & 2047, gg = jj >> 1;
        const int l = (lp - nf / 4) & (nf - 1), lh = (l + half) & (nf - 1);
        const float2 z = Y[gg * kR2S + (l >> 5) * kR2P + (l & 31)];
        const float2 zh = Y[gg * kR2S + (lh >> 5) * kR2P + (lh & 31)];
        S2[dd[u].x] = (jj & 1) ? make_float2(0.5f * (z.y + zh.y), -0.5f * (z.x - zh.x))
                               : make_float2(0.5f * (z.x + zh.x), 0.5f * (z.y - zh.y));
      }
    }
#pragma unroll
    for (int u = 0; u < U; ++u) dd[u] = dn[u];
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
template <int nf, bool VAR>
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
  const int tt_n = min(2 * G, n_t - t0);
  // detector-major loop (no integer division): thread d restricts all 2G samples of detector d
  for (int d = threadIdx.x; d < n_det; d += blockDim.x) {
    const int pos = phys(__ldg(&P.ring[d]));
    const size_t i0 = ((size_t)b * n_t + t0) * n_det + d;
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

// ------------------------------------------------------------------ K5 / K5T, two-stage (n_phi = 512)
// K5: the C2R synthesis of k5_ring with k = a + 16 r, l = k1 + 32 k2 (as k3t_ring2): stage A reads
// S4 rows straight into registers (lanes = transforms: contiguous runs of 2G time samples of row
// k; k > 256 from row 512 - k by the completion), stage B in place, then the detector restriction
// from shared memory as in k5_ring.
template <bool VAR>
__global__ void __launch_bounds__(16 * kR2G, TAT_R2_MINB_K5) k5_ring2(DevPlan P, float* __restrict__ gout) {
  constexpr int nf = 512, half = 256, G = kR2G;
  extern __shared__ float2 sm[];
  const Consts& C = P.C;
  const int n_t = C.n_t, n_det = C.n_det;
  const int b = C.b0 + blockIdx.y, t0 = blockIdx.x * (2 * G);
  float2* Y = sm;
  const int gg0 = threadIdx.x % G, i0 = threadIdx.x / G;
  const int t = t0 + 2 * gg0;
  const bool ok0 = t < n_t, ok1 = t + 1 < n_t;
  pdl_wait();
  pdl_trigger();
  {   // stage A
    const int a = i0;
    const float2* S4 = P.S4 + (size_t)b * C.Kp * n_t + t;
    float2 x[32];
#pragma unroll
    for (int r = 0; r < 32; ++r) {
      const int k = a + 16 * r;
      const bool dir = k <= half;
      const int kk = dir ? k : nf - k;
      const float2 v0 = ok0 ? S4[(size_t)kk * n_t] : make_float2(0.f, 0.f);
      const float2 v1 = ok1 ? S4[(size_t)kk * n_t + 1] : make_float2(0.f, 0.f);
      if (k == 0 || k == half) x[r] = make_float2(v0.x, v1.x);   // real parts (C2R convention)
      else if (dir) x[r] = make_float2(v0.x - v1.y, v0.y + v1.x);  // v0 + i v1
      else x[r] = make_float2(v0.x + v1.y, -v0.y + v1.x);         // conj v0 + i conj v1
    }
    ce::dftr<32, 1>(x);
    r2_twiddle_store<true>(Y + gg0 * kR2S + a * kR2P, x, P.tw_ring, a);   // x W_512^{-a k1}
  }
  __syncthreads();
  {   // stage B, in place: Y[gg][k2][k1] = X[k1 + 32 k2]
    float2* y = Y + gg0 * kR2S;
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      const int k1 = i0 + 16 * h;
      float2 z[16];
#pragma unroll
      for (int a = 0; a < 16; ++a) z[a] = y[a * kR2P + k1];
      ce::dftr<16, 1>(z);
#pragma unroll
      for (int k2 = 0; k2 < 16; ++k2) y[k2 * kR2P + k1] = z[k2];
    }
  }
  __syncthreads();
  const int tt_n = min(2 * G, n_t - t0);
  for (int d = threadIdx.x; d < n_det; d += blockDim.x) {
    const int l = __ldg(&P.ring[d]);
    const int pos = (l >> 5) * kR2P + (l & 31);
    const size_t i0g = ((size_t)b * n_t + t0) * n_det + d;
#pragma unroll
    for (int gg = 0; gg < G; ++gg) {   // transform gg: samples 2 gg (real part), 2 gg + 1 (imag)
      if (2 * gg < tt_n) {
        const float2 z = Y[gg * kR2S + pos];
        const size_t i = i0g + (size_t)(2 * gg) * n_det;
        gout[i] = epi_fwd<VAR>(P, i, z.x);
        if (2 * gg + 1 < tt_n) gout[i + n_det] = epi_fwd<VAR>(P, i + n_det, z.y);
      }
    }
  }
}

// K5T: detectors placed at their ring positions in shared memory (zeros elsewhere unless every
// position has a detector), then the two stages of k3_ring2 (stage A reading shared memory) with
// the outputs of each (k, -k) pair formed in one thread and stored straight to S4 (contiguous runs
// of 2G time samples of row k).
__global__ void __launch_bounds__(16 * kR2G, TAT_R2_MINB_K5T) k5t_ring2(DevPlan P, const float* __restrict__ gin) {
  constexpr int nf = 512, G = kR2G;
  constexpr int XS = nf + nf / 32 + 1;   // input row stride: l + (l >> 5), odd
  extern __shared__ float2 sm[];
  const Consts& C = P.C;
  const int n_t = C.n_t, n_det = C.n_det;
  const int b = C.b0 + blockIdx.y, t0 = blockIdx.x * (2 * G);
  float2* X0 = sm;                  // [G][XS] detector samples on the ring
  float2* Y = sm;                   // [G][kR2S] after stage A's reads (aliases X0)
  const int tt_n = min(2 * G, n_t - t0);
  if (n_det < nf)
    for (int i = threadIdx.x; i < G * XS; i += blockDim.x) X0[i] = make_float2(0.f, 0.f);
  pdl_wait();
  pdl_trigger();
  if (n_det < nf) __syncthreads();
  for (int d = threadIdx.x; d < n_det; d += blockDim.x) {
    const int l = __ldg(&P.ring[d]);
    const float* gi = gin + ((size_t)b * n_t + t0) * n_det + d;
    float gv[2 * G];
#pragma unroll
    for (int tt = 0; tt < 2 * G; ++tt) gv[tt] = tt < tt_n ? gi[(size_t)tt * n_det] : 0.f;
#pragma unroll
    for (int gg = 0; gg < G; ++gg) X0[gg * XS + l + (l >> 5)] = make_float2(gv[2 * gg], gv[2 * gg + 1]);
  }
  __syncthreads();
  {   // stage A (thread (j, gg)): x[r] = X0[gg][j + 16 r]
    const int j = threadIdx.x & 15, gg = threadIdx.x >> 4;
    float2 x[32];
#pragma unroll
    for (int r = 0; r < 32; ++r) {
      const int l = j + 16 * r;
      x[r] = X0[gg * XS + l + (l >> 5)];
    }
    __syncthreads();   // Y aliases X0
    ce::dftr<32, -1>(x);
    r2_twiddle_store<false>(Y + gg * kR2S + j * kR2P, x, P.tw_ring, j);   // x W_512^{j k1}
  }
  __syncthreads();
  {   // stage B + output
    const int gg = threadIdx.x % G, kp = threadIdx.x / G, t = t0 + 2 * gg;
    const int ka = kp == 0 ? 0 : kp, kb = kp == 0 ? 16 : 32 - kp;
    const float2* y = Y + gg * kR2S;
    float2 za[16], zb[16];
#pragma unroll
    for (int j = 0; j < 16; ++j) {
      za[j] = y[j * kR2P + ka];
      zb[j] = y[j * kR2P + kb];
    }
    ce::dftr<16, -1>(za);
    ce::dftr<16, -1>(zb);
    float2* S4 = P.S4 + (size_t)b * C.Kp * n_t;
    const bool ok0 = t < n_t, ok1 = t + 1 < n_t;
    // even sample: (Z[k] + conj Z[-k]) / 2 ; odd sample: (Z[k] - conj Z[-k]) / (2i)
    auto out = [&](int k, float2 zk, float2 zm) {
      float2* o = S4 + (size_t)k * n_t + t;
      if (ok0) o[0] = make_float2(0.5f * (zk.x + zm.x), 0.5f * (zk.y - zm.y));
      if (ok1) o[1] = make_float2(0.5f * (zk.y + zm.y), -0.5f * (zk.x - zm.x));
    };
    if (kp == 0) {
#pragma unroll
      for (int k2 = 0; k2 <= 8; ++k2) out(32 * k2, za[k2 & 15], za[(16 - k2) & 15]);
#pragma unroll
      for (int k2 = 0; k2 < 8; ++k2) out(16 + 32 * k2, zb[k2], zb[15 - k2]);
    } else {
#pragma unroll
      for (int k2 = 0; k2 < 8; ++k2) out(ka + 32 * k2, za[k2], zb[15 - k2]);
#pragma unroll
      for (int k2 = 0; k2 < 8; ++k2) out(kb + 32 * k2, zb[k2], za[15 - k2]);
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
    if (e == cudaSuccess) e = cudaFuncSetAttribute(k5_ring<NF, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, sm);
    if (e == cudaSuccess) e = cudaFuncSetAttribute(k5_ring<NF, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, sm);
    if (e == cudaSuccess) e = cudaFuncSetAttribute(k5t_ring<NF>, cudaFuncAttributeMaxDynamicSharedMemorySize, sm);
  });
  if (e == cudaSuccess) e = cudaFuncSetAttribute(k3_ring2, cudaFuncAttributeMaxDynamicSharedMemorySize, sm);
  if (e == cudaSuccess) e = cudaFuncSetAttribute(k3t_ring2, cudaFuncAttributeMaxDynamicSharedMemorySize, sm);
  if (e == cudaSuccess) e = cudaFuncSetAttribute(k5_ring2<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, sm);
  if (e == cudaSuccess) e = cudaFuncSetAttribute(k5_ring2<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, sm);
  if (e == cudaSuccess) e = cudaFuncSetAttribute(k5t_ring2, cudaFuncAttributeMaxDynamicSharedMemorySize, sm);
  return e;
}

cudaError_t launch_k3(const DevPlan& P, cudaStream_t s) {
  const Consts& C = P.C;
  cudaError_t e = cudaSuccess;
  if (ring2_on(C, 1)) {
    e = launch_pdl(C.pdl, k3_ring2, dim3((C.NL + 2 * kR2G - 1) / (2 * kR2G), C.batch), dim3(16 * kR2G),
                   (size_t)kR2G * kR2S * sizeof(float2), s, P);
    return e != cudaSuccess ? e : cudaGetLastError();
  }
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
  if (ring2_on(C, 2)) {
    e = launch_pdl(C.pdl, k3t_ring2, dim3((C.NL + 2 * kR2G - 1) / (2 * kR2G), C.batch), dim3(16 * kR2G),
                   (size_t)kR2G * kR2S * sizeof(float2), s, P);
    return e != cudaSuccess ? e : cudaGetLastError();
  }
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
  if (ring2_on(C, 4)) {
    const dim3 grid((C.n_t + 2 * kR2G - 1) / (2 * kR2G), C.batch), blk(16 * kR2G);
    const size_t sm2 = (size_t)kR2G * kR2S * sizeof(float2);
    e = P.lowk_add ? launch_pdl(C.pdl, k5_ring2<true>, grid, blk, sm2, s, P, g)
                   : launch_pdl(C.pdl, k5_ring2<false>, grid, blk, sm2, s, P, g);
    return e != cudaSuccess ? e : cudaGetLastError();
  }
  const size_t sm = smem_ring_fast(C);
  TAT_RING_SWITCH({
    constexpr int G = ring_G<NF>();
    if (P.lowk_add)
      e = launch_pdl(C.pdl, k5_ring<NF, true>, dim3((C.n_t + 2 * G - 1) / (2 * G), C.batch), dim3(G * NF / 8), sm, s, P, g);
    else
      e = launch_pdl(C.pdl, k5_ring<NF, false>, dim3((C.n_t + 2 * G - 1) / (2 * G), C.batch), dim3(G * NF / 8), sm, s, P, g);
  });
  return e != cudaSuccess ? e : cudaGetLastError();
}
cudaError_t launch_k5t(const DevPlan& P, const float* g, cudaStream_t s) {
  const Consts& C = P.C;
  cudaError_t e = cudaSuccess;
  if (ring2_on(C, 8)) {
    e = launch_pdl(C.pdl, k5t_ring2, dim3((C.n_t + 2 * kR2G - 1) / (2 * kR2G), C.batch), dim3(16 * kR2G),
                   (size_t)kR2G * kR2S * sizeof(float2), s, P, g);
    return e != cudaSuccess ? e : cudaGetLastError();
  }
  const size_t sm = smem_ring_fast(C);
  TAT_RING_SWITCH({
    constexpr int G = ring_G<NF>();
    e = launch_pdl(C.pdl, k5t_ring<NF>, dim3((C.n_t + 2 * G - 1) / (2 * G), C.batch), dim3(G * NF / 8), sm, s, P, g);
  });
  return e != cudaSuccess ? e : cudaGetLastError();
}

}  // namespace tat
