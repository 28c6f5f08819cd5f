// Angular transforms K3 / K3T / K5 / K5T as two-stage register FFTs (n_phi = 256, 512): the same
// operators as kernels_ring.cu (the radix-8 Stockham kernels, kept for the other ring sizes and
// as TAT_RING2=0), with one shared-memory crossing per point instead of one per radix-8 pass.
//
// With n_phi = R J (R = 32 at n_phi = 512, R = 16 at 256; J = 16), index l = j + J r on the
// input side and k = k1 + R k2 on the output side:
//   Z[k1 + R k2] = sum_j W_J^{j k2} W_nphi^{j k1} sum_r z[j + J r] W_R^{r k1}     (sign S)
//   stage A (thread (j, gg)): the R-point DFT over r in registers, twiddle W_nphi^{j k1}, one
//                             shared-memory store per point;
//   stage B (thread (kp, gg)): the J-point DFTs over j of two k1 columns in registers.
// A CTA holds G = 16 transforms (32 rings of K3 / K3T, 32 time samples of K5 / K5T; two real
// sequences per complex transform, as in kernels_ring.cu), 16 J threads.
//
//   K3  (forward): the half-plane samples are loaded straight from S2 into the stage-A registers
//       (each gives the points l and l + n_phi/2 of the completed ring); stage B takes the column
//       pair k1 = kp, R - kp (kp = 0: 0 and R/2) so that Z[k] and Z[-k] -- both needed to
//       separate the two rings -- are in one thread; outputs x i^k m' stored straight to S3
//       (the lanes of one kp are consecutive rings: contiguous runs of a row of S3).
//   K3T (adjoint): stage A reads S3 rows straight into registers (k > n_phi/2 from row n_phi - k
//       by H~_{-k} = (-1)^k conj H~_k); stage B in place; outputs through k3t_dst (destination
//       order, as k3t_ring).
//   K5  (forward): as K3T with the C2R completion of S4, then the detector restriction.
//   K5T (adjoint): detectors placed on the ring in shared memory, then as K3 with the outputs
//       (Z[k] +- conj Z[-k]) / 2 of the two time samples stored to S4.
// References: E:eq3 / E:eq2, E:FourSerForg, Alg. 2 steps 1-2
// (P:L671-675); readings G12 (half plane), DESIGN.md §6.2.
#include "col_engine.cuh"
#include "fft_engine.cuh"
#include "tat_internal.h"

namespace tat {

using namespace fe;

#ifndef TAT_R2_MINB
#define TAT_R2_MINB 2   // CTAs per SM the two-stage ring kernels are compiled for
#endif
#ifndef TAT_R2_MINB_K5
#define TAT_R2_MINB_K5 3    // (measured at C4: K5 22.2 -> 20.5 us at 3; used at n_phi = 256 only)
#endif
#ifndef TAT_R2_MINB_K5T
#define TAT_R2_MINB_K5T 3   // (measured at C3: K5T 22.4 -> 20.8 us at 3; K3 spills at 3)
#endif

namespace {

template <int nf>
struct R2 {
  static constexpr int R = nf >= 512 ? 32 : 16;   // stage-A DFT length (over r)
  static constexpr int J = nf / R;                  // stage-B DFT length (over j): 16, or 32 at 1024
  static constexpr int G = ring2_G(nf);             // transforms per CTA (16, or 8 at 1024)
  static constexpr int T = G * J;                   // threads (stage A: one per (j, gg)) = 256
  static constexpr int CPT = J == 32 ? 1 : 2;       // stage-B columns k1 per thread
  static constexpr int NB = G * R / CPT;            // stage-B jobs (kp, gg)
  static constexpr int P = R + 1;                   // Y row stride (j): odd
  // Y stride per transform: odd for G = 16 (lanes = 16 transforms in a half-warp), 2 mod 16 for
  // G = 8 (lanes = 8 transforms x 2 rows / columns)
  static constexpr int S = J * P + (G == 16 ? 1 : 2);
  static constexpr int half = nf / 2, quarter = nf / 4;
  static constexpr int XS = nf + nf / 32 + 1;       // K5T input row stride (l + l / 32): odd
  static_assert(T == 256 && (J == 16 || nf == 1024), "ring2 layout");
  // element l = k1 + R k2 of transform gg after stage B
  __device__ static __forceinline__ int yidx(int gg, int l) {
    return gg * S + (int)((unsigned)l / R) * P + (int)((unsigned)l % R);
  }
};

// y[k1] = x[k1] W_nphi^{+-j k1} (CONJ: the conjugate twiddles), k1 < R
template <int R, bool CONJ>
__device__ __forceinline__ void r2_twiddle_store(float2* y, const float2 (&x)[R], const float2* __restrict__ tw,
                                                 int j) {
  float2 pw[R];
  const float2 w = __ldg(&tw[j]);
  ce::pow_tree<R>(CONJ ? make_float2(w.x, -w.y) : w, pw);
  y[0] = x[0];
#pragma unroll
  for (int k1 = 1; k1 < R; ++k1) y[k1] = cmul(x[k1], pw[k1]);
}

// i^e m a without branches (e varies across the lanes of a warp): the sign of i^e folded into m
__device__ __forceinline__ float2 ipow_scale(float2 a, float m, int e) {
  const float2 r = (e & 1) ? make_float2(-a.y, a.x) : a;
  return cscale(r, (e & 2) ? -m : m);
}

// Stage A of the forward-sign transforms (K3, K5T): x[r] = z[j + J r] -> Y[gg][j][k1]
template <int nf>
__device__ __forceinline__ void r2_stage_a_fwd(float2 (&x)[R2<nf>::R], float2* Y, const float2* tw, int j, int gg) {
  using Q = R2<nf>;
  ce::dftr<Q::R, -1>(x);
  r2_twiddle_store<Q::R, false>(Y + gg * Q::S + j * Q::P, x, tw, j);
}

// Stage B with the (k, -k) pairing of the forward-sign transforms: thread (kp, gg) returns
// za = Z[ka + R k2], zb = Z[kb + R k2] (k2 < J), ka = kp, kb = R - kp (kp = 0: 0 and R/2)
template <int nf>
__device__ __forceinline__ void r2_stage_b_pair(const float2* Y, int gg, int ka, int kb, float2 (&za)[16],
                                                float2 (&zb)[16]) {
  using Q = R2<nf>;
  const float2* y = Y + gg * Q::S;
#pragma unroll
  for (int j = 0; j < Q::J; ++j) {
    za[j] = y[j * Q::P + ka];
    zb[j] = y[j * Q::P + kb];
  }
  ce::dftr<Q::J, -1>(za);
  ce::dftr<Q::J, -1>(zb);
}

// Calls f(s, k, Z[k], Z[-k]) for the outputs k <= nf/2 of thread kp (slot s < J + 1):
// kp > 0: k = ka + R k2, then kb + R k2 (k2 < J/2); kp = 0: k = R k2 (k2 <= J/2), then R/2 + R k2
template <int nf, class F>
__device__ __forceinline__ void r2_pairs(int kp, int ka, int kb, const float2 (&za)[16], const float2 (&zb)[16],
                                         F&& f) {
  using Q = R2<nf>;
  constexpr int J = Q::J, R = Q::R, H = J / 2;
  if (kp == 0) {
#pragma unroll
    for (int k2 = 0; k2 <= H; ++k2) f(k2, R * k2, za[k2 % J], za[(J - k2) % J]);
#pragma unroll
    for (int k2 = 0; k2 < H; ++k2) f(H + 1 + k2, R / 2 + R * k2, zb[k2], zb[J - 1 - k2]);
  } else {
#pragma unroll
    for (int k2 = 0; k2 < H; ++k2) f(k2, ka + R * k2, za[k2], zb[J - 1 - k2]);
#pragma unroll
    for (int k2 = 0; k2 < H; ++k2) f(H + k2, kb + R * k2, zb[k2], za[J - 1 - k2]);
  }
}
template <int nf>
__device__ __forceinline__ int r2_kout(int kp, int ka, int kb, int s) {
  using Q = R2<nf>;
  constexpr int R = Q::R, H = Q::J / 2;
  return kp == 0 ? (s <= H ? R * s : R / 2 + R * (s - H - 1)) : (s < H ? ka + R * s : kb + R * (s - H));
}

// Stage B in place (sign S): Y[gg][k2][k1] = sum_j W_J^{S j k2} Y[gg][j][k1] for the CPT
// columns k1 = kp + (R / CPT) h of thread (kp, gg)
template <int nf, int S>
__device__ __forceinline__ void r2_stage_b_inplace(float2* Y, int gg, int kp) {
  using Q = R2<nf>;
  float2* y = Y + gg * Q::S;
#pragma unroll
  for (int h = 0; h < Q::CPT; ++h) {
    const int k1 = kp + (Q::R / Q::CPT) * h;
    float2 z[Q::J];
#pragma unroll
    for (int a = 0; a < Q::J; ++a) z[a] = y[a * Q::P + k1];
    ce::dftr<Q::J, S>(z);
#pragma unroll
    for (int k2 = 0; k2 < Q::J; ++k2) y[k2 * Q::P + k1] = z[k2];
  }
}
template <int nf>
__device__ __forceinline__ void r2_stage_b_inv(float2* Y, int gg, int kp) { r2_stage_b_inplace<nf, 1>(Y, gg, kp); }

}  // namespace

// ------------------------------------------------------------------ K3
template <int nf>
__global__ void __launch_bounds__(R2<nf>::T, TAT_R2_MINB) k3_ring2(DevPlan P) {
  using Q = R2<nf>;
  constexpr int R = Q::R, J = Q::J, G = Q::G, half = Q::half, M = R / 2;   // M loads per ring
  extern __shared__ float2 sm[];
  const Consts& C = P.C;
  const int NL = C.NL;
  const int b = C.b0 + blockIdx.y, j0 = blockIdx.x * (2 * G);
  const float2* S2 = P.S2 + (size_t)b * half * NL;
  float2* Y = sm;
  pdl_wait();
  pdl_trigger();
  {   // stage A: samples l' = j + J m of both rings of pair gg (l = l' - nf/4 mod nf) and their
      // conjugate partners l + nf/2
    const int j = threadIdx.x % J, gg = threadIdx.x / J, ja = j0 + 2 * gg;
    const float2* ra = S2 + (size_t)ja * half + j;
    float2 va[M], vb[M];
#pragma unroll
    for (int m = 0; m < M; ++m) {
      va[m] = ja < NL ? ra[J * m] : make_float2(0.f, 0.f);
      vb[m] = ja + 1 < NL ? ra[half + J * m] : make_float2(0.f, 0.f);
    }
    float2 x[R];
#pragma unroll
    for (int m = 0; m < M; ++m) {
      const float2 d = make_float2(va[m].x - vb[m].y, va[m].y + vb[m].x);    // va + i vb
      const float2 c = make_float2(va[m].x + vb[m].y, -va[m].y + vb[m].x);   // conj va + i conj vb
      const int r = m < R / 4 ? m + 3 * R / 4 : m - R / 4;
      x[r] = d;
      x[(r + R / 2) % R] = c;
    }
    r2_stage_a_fwd<nf>(x, Y, P.tw_ring, j, gg);
  }
  if constexpr (J == 32) {   // n_phi = 1024: stage B in place, then the (k, -k) pairs from smem
    const int gg = threadIdx.x % G, kk = threadIdx.x / G, ja = j0 + 2 * gg;   // item (k, gg)
    const bool ok0 = ja < NL, ok1 = ja + 1 < NL;
    constexpr int NI = (half + 1 + Q::T / G - 1) / (Q::T / G);                   // items per thread
    float2 mo[NI];
#pragma unroll
    for (int u = 0; u < NI; ++u) {
      const int k = kk + (Q::T / G) * u;
      mo[u] = make_float2(k <= half && ok0 ? __ldg(&P.mult[(size_t)k * NL + ja]) : 0.f,
                          k <= half && ok1 ? __ldg(&P.mult[(size_t)k * NL + ja + 1]) : 0.f);
    }
    __syncthreads();
    r2_stage_b_inplace<nf, -1>(Y, gg, kk);
    __syncthreads();
    float2* S3 = P.S3 + (size_t)b * C.Kp * NL;
#pragma unroll
    for (int u = 0; u < NI; ++u) {
      const int k = kk + (Q::T / G) * u;
      if (k <= half) {
        const float2 zk = Y[Q::yidx(gg, k)];
        float2 zm = Y[Q::yidx(gg, (nf - k) & (nf - 1))];
        if (k & 1) zm = make_float2(-zm.x, -zm.y);
        const float2 F1 = make_float2(0.5f * (zk.x + zm.x), 0.5f * (zk.y - zm.y));
        const float2 F2 = make_float2(0.5f * (zk.y + zm.y), -0.5f * (zk.x - zm.x));
        float2* o = S3 + (size_t)k * NL + ja;
        if (ok0) o[0] = ipow_scale(F1, mo[u].x, k);
        if (ok1) o[1] = ipow_scale(F2, mo[u].y, k);
      }
    }
  } else {
  // multiplier values of this thread's outputs, loaded before the barrier (latency under stage B)
  const int gg = threadIdx.x % G, kp = threadIdx.x / G, ja = j0 + 2 * gg;
  const bool act = threadIdx.x < Q::NB;
  const int ka = kp == 0 ? 0 : kp, kb = kp == 0 ? R / 2 : R - kp;
  const bool ok0 = act && ja < NL, ok1 = act && ja + 1 < NL;
  float2 mo[J + 1];
#pragma unroll
  for (int s = 0; s <= J; ++s) {
    const int k = r2_kout<nf>(kp, ka, kb, s);
    const bool v = s < J || kp == 0;
    mo[s] = make_float2(v && ok0 ? __ldg(&P.mult[(size_t)k * NL + ja]) : 0.f,
                        v && ok1 ? __ldg(&P.mult[(size_t)k * NL + ja + 1]) : 0.f);
  }
  __syncthreads();
  if (act) {   // stage B + output: F1 = (Z[k] + conj Z'[-k]) / 2, F2 = (Z[k] - conj Z'[-k]) / 2i
    float2 za[16], zb[16];
    r2_stage_b_pair<nf>(Y, gg, ka, kb, za, zb);
    float2* S3 = P.S3 + (size_t)b * C.Kp * NL;
    r2_pairs<nf>(kp, ka, kb, za, zb, [&](int s, int k, float2 zk, float2 zm) {
      if (k & 1) zm = make_float2(-zm.x, -zm.y);   // Z'[-k] = (-1)^k Z[-k]
      const float2 F1 = make_float2(0.5f * (zk.x + zm.x), 0.5f * (zk.y - zm.y));
      const float2 F2 = make_float2(0.5f * (zk.y + zm.y), -0.5f * (zk.x - zm.x));
      float2* o = S3 + (size_t)k * NL + ja;
      if (ok0) o[0] = ipow_scale(F1, mo[s].x, k);
      if (ok1) o[1] = ipow_scale(F2, mo[s].y, k);
    });
  }
  }
}

// ------------------------------------------------------------------ K3T
template <int nf>
__global__ void __launch_bounds__(R2<nf>::T, TAT_R2_MINB) k3t_ring2(DevPlan P) {
  using Q = R2<nf>;
  constexpr int R = Q::R, J = Q::J, G = Q::G, half = Q::half;
  extern __shared__ float2 sm[];
  const Consts& C = P.C;
  const int NL = C.NL;
  const int b = C.b0 + blockIdx.y, j0 = blockIdx.x * (2 * G);
  float2* Y = sm;
  const int gg = threadIdx.x % G, a = threadIdx.x / G, ja = j0 + 2 * gg;
  const bool ok0 = ja < NL, ok1 = ja + 1 < NL;
  const float2* S3 = P.S3 + (size_t)b * C.Kp * NL + ja;
  pdl_wait();
  pdl_trigger();
  {   // stage A (thread (a, gg), lanes = ring pairs): Z[a + J r], r < R
    float2 x[R];
#pragma unroll
    for (int r = 0; r < R; ++r) {
      const int k = a + J * r;
      const bool dir = k <= half;
      const int kk = dir ? k : nf - k;
      const float2 e1 = ok0 ? S3[(size_t)kk * NL] : make_float2(0.f, 0.f);
      const float2 e2 = ok1 ? S3[(size_t)kk * NL + 1] : make_float2(0.f, 0.f);
      if (dir) {
        x[r] = make_float2(e1.x - e2.y, e1.y + e2.x);   // E1 + i E2 (slot nf/2 is -K)
      } else {
        const float sg = (kk & 1) ? -1.f : 1.f;         // E(-k) = (-1)^k conj E(k)
        x[r] = make_float2(sg * (e1.x + e2.y), sg * (-e1.y + e2.x));
      }
    }
    ce::dftr<R, 1>(x);
    r2_twiddle_store<R, true>(Y + gg * Q::S + a * Q::P, x, P.tw_ring, a);   // x W^{-a k1}
  }
  __syncthreads();
  // the output records (position, source) of the first chunk, loaded during stage B (measured:
  // issued before the barrier instead, K3T 37.0 -> 39.1 us at C3)
  const int nout = min(2 * G, NL - j0) * half;
  const int2* dst = P.k3t_dst + (size_t)j0 * half;
  constexpr int T = Q::T, U = 8;
  int2 dd[U];
#pragma unroll
  for (int u = 0; u < U; ++u) {
    const int i = threadIdx.x + u * T;
    dd[u] = i < nout ? __ldg(&dst[i]) : make_int2(0, 0);
  }
  if (threadIdx.x < Q::NB) r2_stage_b_inv<nf>(Y, gg, a);
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
      if (i + u * T < nout) {   // P~_1 = (z + conj z[l + nf/2]) / 2, P~_2 = (z - conj z[..]) / 2i
        const int jj = dd[u].y >> 11, lp = dd[u].y & 2047, gg = jj >> 1;
        const int l = (lp - Q::quarter) & (nf - 1), lh = (l + half) & (nf - 1);
        const float2 z = Y[Q::yidx(gg, l)];
        const float2 zh = Y[Q::yidx(gg, lh)];
        S2[dd[u].x] = (jj & 1) ? make_float2(0.5f * (z.y + zh.y), -0.5f * (z.x - zh.x))
                               : make_float2(0.5f * (z.x + zh.x), 0.5f * (z.y - zh.y));
      }
    }
#pragma unroll
    for (int u = 0; u < U; ++u) dd[u] = dn[u];
  }
}

// ------------------------------------------------------------------ K5
// transform gg carries time samples t0 + 2 gg (real part) and t0 + 2 gg + 1 (imaginary part)
template <int nf, bool VAR>
__global__ void __launch_bounds__(R2<nf>::T, TAT_R2_MINB_K5) k5_ring2(DevPlan P, float* __restrict__ gout) {
  using Q = R2<nf>;
  constexpr int R = Q::R, J = Q::J, G = Q::G, half = Q::half;
  extern __shared__ float2 sm[];
  const Consts& C = P.C;
  const int n_t = C.n_t, n_det = C.n_det;
  const int b = C.b0 + blockIdx.y, t0 = blockIdx.x * (2 * G);
  float2* Y = sm;
  const int gg = threadIdx.x % G, a = threadIdx.x / G, t = t0 + 2 * gg;
  const bool ok0 = t < n_t, ok1 = t + 1 < n_t;
  const float2* S4 = P.S4 + (size_t)b * C.Kp * n_t + t;
  pdl_wait();
  pdl_trigger();
  {   // stage A (thread (a, gg), lanes = transforms): C2R completion of S4 rows a + J r
    float2 x[R];
#pragma unroll
    for (int r = 0; r < R; ++r) {
      const int k = a + J * r;
      const bool dir = k <= half;
      const int kk = dir ? k : nf - k;
      const float2 v0 = ok0 ? S4[(size_t)kk * n_t] : make_float2(0.f, 0.f);
      const float2 v1 = ok1 ? S4[(size_t)kk * n_t + 1] : make_float2(0.f, 0.f);
      if (k == 0 || k == half) x[r] = make_float2(v0.x, v1.x);   // real parts (C2R convention)
      else if (dir) x[r] = make_float2(v0.x - v1.y, v0.y + v1.x);  // v0 + i v1
      else x[r] = make_float2(v0.x + v1.y, -v0.y + v1.x);         // conj v0 + i conj v1
    }
    ce::dftr<R, 1>(x);
    r2_twiddle_store<R, true>(Y + gg * Q::S + a * Q::P, x, P.tw_ring, a);
  }
  __syncthreads();
  if (threadIdx.x < Q::NB) r2_stage_b_inv<nf>(Y, gg, a);
  __syncthreads();
  const int tt_n = min(2 * G, n_t - t0);
  for (int d = threadIdx.x; d < n_det; d += blockDim.x) {
    const int pos = Q::yidx(0, __ldg(&P.ring[d]));
    const size_t i0g = ((size_t)b * n_t + t0) * n_det + d;
#pragma unroll
    for (int tg = 0; tg < G; ++tg) {   // transform tg: samples 2 tg (real part), 2 tg + 1 (imag)
      if (2 * tg < tt_n) {
        const float2 z = Y[tg * Q::S + pos];
        const size_t i = i0g + (size_t)(2 * tg) * n_det;
        gout[i] = epi_fwd<VAR>(P, i, z.x);
        if (2 * tg + 1 < tt_n) gout[i + n_det] = epi_fwd<VAR>(P, i + n_det, z.y);
      }
    }
  }
}

// ------------------------------------------------------------------ K5T
template <int nf>
__global__ void __launch_bounds__(R2<nf>::T, TAT_R2_MINB_K5T) k5t_ring2(DevPlan P, const float* __restrict__ gin) {
  using Q = R2<nf>;
  constexpr int R = Q::R, J = Q::J, G = Q::G, XS = Q::XS;
  extern __shared__ float2 sm[];
  const Consts& C = P.C;
  const int n_t = C.n_t, n_det = C.n_det;
  const int b = C.b0 + blockIdx.y, t0 = blockIdx.x * (2 * G);
  float2* X0 = sm;                  // [G][XS] detector samples on the ring
  float2* Y = sm;                   // [G][S] after stage A's reads (aliases X0)
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
  {   // stage A (thread (j, gg)): x[r] = X0[gg][j + J r]
    const int j = threadIdx.x % J, gg = threadIdx.x / J;
    float2 x[R];
#pragma unroll
    for (int r = 0; r < R; ++r) {
      const int l = j + J * r;
      x[r] = X0[gg * XS + l + (l >> 5)];
    }
    __syncthreads();   // Y aliases X0
    r2_stage_a_fwd<nf>(x, Y, P.tw_ring, j, gg);
  }
  __syncthreads();
  if constexpr (J == 32) {   // n_phi = 1024: stage B in place, then the (k, -k) pairs from smem
    const int gg = threadIdx.x % G, kk = threadIdx.x / G, t = t0 + 2 * gg;
    r2_stage_b_inplace<nf, -1>(Y, gg, kk);
    __syncthreads();
    float2* S4 = P.S4 + (size_t)b * C.Kp * n_t;
    const bool ok0 = t < n_t, ok1 = t + 1 < n_t;
    for (int k = kk; k <= Q::half; k += Q::T / G) {
      const float2 zk = Y[Q::yidx(gg, k)];
      const float2 zm = Y[Q::yidx(gg, (nf - k) & (nf - 1))];
      float2* o = S4 + (size_t)k * n_t + t;
      if (ok0) o[0] = make_float2(0.5f * (zk.x + zm.x), 0.5f * (zk.y - zm.y));
      if (ok1) o[1] = make_float2(0.5f * (zk.y + zm.y), -0.5f * (zk.x - zm.x));
    }
  } else if (threadIdx.x < Q::NB) {   // stage B + output: (Z[k] + conj Z[-k]) / 2 (even
                                      // sample), (Z[k] - conj Z[-k]) / 2i (odd sample)
    const int gg = threadIdx.x % G, kp = threadIdx.x / G, t = t0 + 2 * gg;
    const int ka = kp == 0 ? 0 : kp, kb = kp == 0 ? R / 2 : R - kp;
    float2 za[16], zb[16];
    r2_stage_b_pair<nf>(Y, gg, ka, kb, za, zb);
    float2* S4 = P.S4 + (size_t)b * C.Kp * n_t;
    const bool ok0 = t < n_t, ok1 = t + 1 < n_t;
    r2_pairs<nf>(kp, ka, kb, za, zb, [&](int, int k, float2 zk, float2 zm) {
      float2* o = S4 + (size_t)k * n_t + t;
      if (ok0) o[0] = make_float2(0.5f * (zk.x + zm.x), 0.5f * (zk.y - zm.y));
      if (ok1) o[1] = make_float2(0.5f * (zk.y + zm.y), -0.5f * (zk.x - zm.x));
    });
  }
}

// ------------------------------------------------------------------ dispatch
template <int nf>
static size_t r2_smem() {
  using Q = R2<nf>;
  const size_t y = (size_t)Q::G * Q::S, x0 = (size_t)Q::G * Q::XS;
  return (y > x0 ? y : x0) * sizeof(float2);
}

#define TAT_RING2_SWITCH(...)                                   \
  switch (C.n_ring) {                                           \
    case 256: { constexpr int NF = 256; __VA_ARGS__; } break;   \
    case 512: { constexpr int NF = 512; __VA_ARGS__; } break;   \
    case 1024: { constexpr int NF = 1024; __VA_ARGS__; } break; \
    default: return cudaErrorInvalidValue;                      \
  }

cudaError_t configure_ring2_kernels(const Consts& C) {
  if (!ring2_size_ok(C.n_ring)) return cudaSuccess;
  cudaError_t e = cudaSuccess;
  const int sm = kSmemLimit;
#define SET2(k) if (e == cudaSuccess) e = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, sm);
  TAT_RING2_SWITCH({
    SET2(k3_ring2<NF>);
    SET2(k3t_ring2<NF>);
    SET2((k5_ring2<NF, false>));
    SET2((k5_ring2<NF, true>));
    SET2(k5t_ring2<NF>);
  });
#undef SET2
  return e;
}

cudaError_t launch_ring2(const DevPlan& P, int which, const float* gin, float* gout, cudaStream_t s) {
  const Consts& C = P.C;
  cudaError_t e = cudaSuccess;
  const int G = ring2_G(C.n_ring);
  const dim3 gj((C.NL + 2 * G - 1) / (2 * G), C.batch), gt((C.n_t + 2 * G - 1) / (2 * G), C.batch);
  TAT_RING2_SWITCH({
    const dim3 blk(R2<NF>::T);
    const size_t sm = r2_smem<NF>();
    switch (which) {
      case 1: e = launch_pdl(C.pdl, k3_ring2<NF>, gj, blk, sm, s, P); break;
      case 2: e = launch_pdl(C.pdl, k3t_ring2<NF>, gj, blk, sm, s, P); break;
      case 4:
        e = P.lowk_add ? launch_pdl(C.pdl, k5_ring2<NF, true>, gt, blk, sm, s, P, gout)
                       : launch_pdl(C.pdl, k5_ring2<NF, false>, gt, blk, sm, s, P, gout);
        break;
      default: e = launch_pdl(C.pdl, k5t_ring2<NF>, gt, blk, sm, s, P, gin); break;
    }
  });
  return e != cudaSuccess ? e : cudaGetLastError();
}

}  // namespace tat
