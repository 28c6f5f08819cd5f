// The oversampled-DFT kernels (the O(n^2 log n) "2D FFT" of Alg. 1 steps 1-3 and Alg. 2
// steps 5-7), built on the residue FFT engine:
//
//   K1    f [B][n][n]   -> S1 [B][N/2+1][n]   row DFT (pairs of real rows packed)
//   K2    S1            -> S2 [B][nodes]      column DFT + bilinear gather to the polar nodes
//   K2Ta  S2            -> Rc [B][targets]    transposed bilinear: per Cartesian target the
//                                             fixed-order sum of w * P~ (deterministic CSR)
//   K2Tb  Rc            -> S1                  scatter targets into the column + inverse DFT
//   K1T   S1            -> f                   inverse row DFT (Hermitian completion)
//
// S1 is column-major ([p][y]); S2 is ring-major ([j][l'], half plane).
// One thread = one radix-8 butterfly of one residue transform; L residues x n/8 threads.
#include "async_copy.cuh"
#include "fft_engine.cuh"
#include "tat_internal.h"

#include <cudaTypedefs.h>

namespace tat {

using namespace fe;

// K2 / K2T columns per CTA: C.col_strip / C.col_strip_adj (K2: sliding window, one halo column)

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

// Passes 1..P-1 of one residue transform (pass-0 output in b0), twiddles generated on the fly;
// the last pass is written (natural order) to smem; returns 0 if it lands in b0, 1 if in b1.
template <int n, int S>
__device__ __forceinline__ int passes_fwd(float2 (&v)[8], float2* b0, float2* b1, int j, int g, int L,
                                          const float2* __restrict__ tw_n) {
  constexpr int P = Plan<n>::P;
  gsync<n>(g, L);
  pass_g<n, 1, S, true, true>(v, b0, b1, j, tw_n);
  if constexpr (P > 2) {
    gsync<n>(g, L);
    pass_g<n, 2, S, true, true>(v, b1, b0, j, tw_n);
  }
  if constexpr (P > 3) {
    gsync<n>(g, L);
    pass_g<n, 3, S, true, true>(v, b0, b1, j, tw_n);
  }
  return (P - 1) & 1;
}

// Inverse transform of a residue stored in A (natural order): pass 0 reads A, passes ping-pong
// A <-> B, the last pass leaves the result in registers (positions last_pos).  ZA: the last pass
// that reads A also re-zeroes what it read (A must stay zero for the next scatter).
template <int n, bool ZA>
__device__ __forceinline__ void passes_inv(float2 (&v)[8], float2* A, float2* B, int j, int g, int L,
                                           const float2* __restrict__ tw_n) {
  constexpr int P = Plan<n>::P;
  pass_g<n, 0, 1, true, true, ZA && (P == 2)>(v, A, B, j, tw_n);
  gsync<n>(g, L);
  if constexpr (P == 2) {
    pass_g<n, 1, 1, true, false>(v, B, A, j, tw_n);
  } else if constexpr (P == 3) {
    pass_g<n, 1, 1, true, true>(v, B, A, j, tw_n);
    gsync<n>(g, L);
    pass_g<n, 2, 1, true, false, ZA>(v, A, B, j, tw_n);
  } else {
    pass_g<n, 1, 1, true, true>(v, B, A, j, tw_n);
    gsync<n>(g, L);
    pass_g<n, 2, 1, true, true, ZA>(v, A, B, j, tw_n);
    gsync<n>(g, L);
    pass_g<n, 3, 1, true, false>(v, B, A, j, tw_n);
  }
}

__device__ __forceinline__ int fidx(int q, int L1, int lg, int rs) {   // F[q] in residue layout
  return (q & L1) * rs + phys(q >> lg);
}

// ================================================================== K2 forward
// Strip of C.col_strip columns with a sliding window of two column spectra.  The next column is
// fetched with a 1-D TMA bulk copy into a double buffer while the current one is transformed;
// the first node record of each gather is prefetched into registers before the transform.
template <int n>
__global__ void __launch_bounds__(1024) k2_fwd(DevPlan P) {
  extern __shared__ __align__(128) float2 sm[];
  constexpr int rs = rstride(n);
  const Consts& C = P.C;
  const int L = C.Lres, L1 = L - 1, lg = C.log2L, ln = L * rs, N1 = C.N - 1;
  const int b = C.b0 + blockIdx.y;
  const int P0 = blockIdx.x * C.col_strip;
  const int Pend = min(P0 + C.col_strip, C.ncols);
  const int plast = min(Pend, C.ncols - 1);
  const int g = threadIdx.x / (n / 8), j = threadIdx.x & (n / 8 - 1);
  const int so = g * rs;
  float2* xbuf = sm + 3 * ln;                                   // 2 x n, TMA destination
  uint64_t* bar = reinterpret_cast<uint64_t*>(xbuf + 2 * n);    // 2 mbarriers
  float2 pre[8];
#pragma unroll
  for (int r = 0; r < 8; ++r) pre[r] = __ldg(&P.tw_pre[g * n + j + r * (n / 8)]);
  const float2* S1 = P.S1 + (size_t)b * C.ncols * n;
  float2* S2 = P.S2 + (size_t)b * C.half * C.NL;
  if (threadIdx.x == 0) {
    ac::mbar_init(&bar[0], 1);
    ac::mbar_init(&bar[1], 1);
    ac::fence_mbar_init();
    ac::mbar_expect_tx(&bar[0], n * 8);
    ac::bulk_g2s(xbuf, S1 + (size_t)P0 * n, n * 8, &bar[0]);
  }
  __syncthreads();
  int prev = 2;
  for (int p = P0; p <= plast; ++p) {
    const int it = p - P0, slot = it & 1;
    if (threadIdx.x == 0 && p < plast) {   // prefetch column p + 1 (its buffer was released)
      ac::fence_proxy_async();
      ac::mbar_expect_tx(&bar[slot ^ 1], n * 8);
      ac::bulk_g2s(xbuf + (slot ^ 1) * n, S1 + (size_t)(p + 1) * n, n * 8, &bar[slot ^ 1]);
    }
    // gather of this iteration (p0 = p - 1): prefetch its first node record
    const int e0 = (p > P0) ? __ldg(&P.k2_colptr[p - 1]) : 0;
    const int e1 = (p > P0) ? __ldg(&P.k2_colptr[p]) : 0;
    int4 nd0 = make_int4(0, 0, 0, 0);
    if (e0 + (int)threadIdx.x < e1) nd0 = __ldg(&P.k2_nodes[e0 + threadIdx.x]);
    ac::mbar_wait(&bar[slot], (it >> 1) & 1);
    const float2* xs = xbuf + slot * n;
    float2 v[8];
    // FFT slot y' = j + r n/8 holds sample y = (y' + n/2) mod n
#pragma unroll
    for (int r = 0; r < 8; ++r) v[r] = cmul(xs[j + (r < 4 ? n / 2 + r * (n / 8) : (r - 4) * (n / 8))], pre[r]);
    const int i0 = prev == 0 ? 1 : 0, i1 = prev == 2 ? 1 : 2;
    float2* X = sm + i0 * ln;
    float2* Y = sm + i1 * ln;
    pass_g<n, 0, -1, false, true>(v, nullptr, X + so, j, P.tw_n);
    const int cur = passes_fwd<n, -1>(v, X + so, Y + so, j, g, L, P.tw_n) ? i1 : i0;
    __syncthreads();
    if (p > P0) {
      const float2* Xa = sm + prev * ln;
      const float2* Xb = sm + cur * ln;
      int e = e0 + threadIdx.x;
      int4 nd = nd0;
      while (e < e1) {
        const float a = __int_as_float(nd.z), bb = __int_as_float(nd.w);
        const int i00 = fidx(nd.y & N1, L1, lg, rs), i01 = fidx((nd.y + 1) & N1, L1, lg, rs);
        const float2 f00 = Xa[i00], f01 = Xa[i01], f10 = Xb[i00], f11 = Xb[i01];
        const float2 c0 = __ffma2_rn(make_float2(a, a), csub(f10, f00), f00);
        const float2 c1 = __ffma2_rn(make_float2(a, a), csub(f11, f01), f01);
        S2[nd.x] = __ffma2_rn(make_float2(bb, bb), csub(c1, c0), c0);
        e += blockDim.x;
        if (e < e1) nd = __ldg(&P.k2_nodes[e]);
      }
    }
    __syncthreads();
    prev = cur;
  }
  if (Pend == C.ncols) {   // p0 = N/2: alpha == 0, only F[N/2] is used
    const float2* Xa = sm + prev * ln;
    for (int e = P.k2_colptr[C.ncols - 1] + threadIdx.x; e < P.k2_colptr[C.ncols]; e += blockDim.x) {
      const int4 nd = __ldg(&P.k2_nodes[e]);
      const float bb = __int_as_float(nd.w);
      const float2 f00 = Xa[fidx(nd.y & N1, L1, lg, rs)];
      const float2 f01 = Xa[fidx((nd.y + 1) & N1, L1, lg, rs)];
      S2[nd.x] = __ffma2_rn(make_float2(bb, bb), csub(f01, f00), f00);
    }
  }
}

// ================================================================== K1 forward (row pairs)
// z = f_y + i f_{y+1}; Z[p] = sum_x z e^{-2 pi i p (x-n/2)/N}; two row pairs per CTA so that
// each p writes one full 32-byte sector S1[p][y0..y0+3].
template <int n>
__global__ void __launch_bounds__(1024) k1_fwd(DevPlan P, const __grid_constant__ CUtensorMap tm,
                                                const float* __restrict__ f) {
  extern __shared__ __align__(128) float2 sm[];
  constexpr int rs = rstride(n);
  const Consts& C = P.C;
  const int L = C.Lres, L1 = L - 1, lg = C.log2L, ln = L * rs, N = C.N;
  const int b = C.b0 + blockIdx.y, y0 = 4 * blockIdx.x;
  const int g = threadIdx.x / (n / 8), j = threadIdx.x & (n / 8 - 1);
  const int so = g * rs;
  float2 pre[8];
#pragma unroll
  for (int r = 0; r < 8; ++r) pre[r] = __ldg(&P.tw_pre[g * n + j + r * (n / 8)]);
  // both row pairs' samples are loaded up front (independent loads, one latency)
  float2 xa[8], xb[8];
  {
    const float* r0 = f + ((size_t)b * n + y0) * n;
#pragma unroll
    for (int r = 0; r < 8; ++r) {
      const int xi = j + (r < 4 ? n / 2 + r * (n / 8) : (r - 4) * (n / 8));
      xa[r] = make_float2(__ldg(&r0[xi]), __ldg(&r0[n + xi]));
      xb[r] = make_float2(__ldg(&r0[2 * n + xi]), __ldg(&r0[3 * n + xi]));
    }
    if (P.deapod) {   // reading G26: f / K on the nodes, K separable
      const float w0 = P.deapod[y0], w1 = P.deapod[y0 + 1], w2 = P.deapod[y0 + 2], w3 = P.deapod[y0 + 3];
#pragma unroll
      for (int r = 0; r < 8; ++r) {
        const float cw = P.deapod[j + (r < 4 ? n / 2 + r * (n / 8) : (r - 4) * (n / 8))];
        xa[r].x *= cw * w0;
        xa[r].y *= cw * w1;
        xb[r].x *= cw * w2;
        xb[r].y *= cw * w3;
      }
    }
  }
  int iA, iB;
  {
    float2 v[8];
#pragma unroll
    for (int r = 0; r < 8; ++r) v[r] = cmul(xa[r], pre[r]);
    pass_g<n, 0, -1, false, true>(v, nullptr, sm + so, j, P.tw_n);
    iA = passes_fwd<n, -1>(v, sm + so, sm + ln + so, j, g, L, P.tw_n) ? 1 : 0;
  }
  {
    const int i1 = iA == 0 ? 1 : 0;
    float2 v[8];
#pragma unroll
    for (int r = 0; r < 8; ++r) v[r] = cmul(xb[r], pre[r]);
    pass_g<n, 0, -1, false, true>(v, nullptr, sm + 2 * ln + so, j, P.tw_n);
    iB = passes_fwd<n, -1>(v, sm + 2 * ln + so, sm + i1 * ln + so, j, g, L, P.tw_n) ? i1 : 2;
  }
  __syncthreads();
  const float2* ZA = sm + iA * ln;
  const float2* ZB = sm + iB * ln;
  // output: S1[p][y0..y0+3] staged as [256 p][4 y] tiles in the free buffer, stored by TMA
  float2* stg = sm + (3 - iA - iB) * ln;
  const int BP = C.s1boxP, CH = BP * kS1BoxY;      // complex values per tile
  const int nslot = (ln / CH) < 4 ? (ln / CH) : 4;  // >= 2 by construction of s1boxP
  const int nch = (C.ncols + BP - 1) / BP;
  for (int c = 0; c < nch; ++c) {
    const int slot = c % nslot;
    if (c >= nslot) {   // the store that used this slot must have finished reading it
      if (threadIdx.x == 0) ac::bulk_wait_read<0>();
      __syncthreads();
    }
    float2* t = stg + slot * CH;
    for (int u = threadIdx.x; u < 2 * BP; u += blockDim.x) {
      const int pl = u >> 1, pr = u & 1, p = c * BP + pl;
      if (p < C.ncols) {
        const float2* Z = pr ? ZB : ZA;
        const int pm = (N - p) & (N - 1);
        const float2 za = Z[fidx(p, L1, lg, rs)], zm = Z[fidx(pm, L1, lg, rs)];
        // row y: (Z[p] + conj Z[-p]) / 2 ; row y+1: (Z[p] - conj Z[-p]) / (2 i)
        t[pl * 4 + 2 * pr] = make_float2(0.5f * (za.x + zm.x), 0.5f * (za.y - zm.y));
        t[pl * 4 + 2 * pr + 1] = make_float2(0.5f * (za.y + zm.y), -0.5f * (za.x - zm.x));
      }
    }
    ac::fence_proxy_async();
    __syncthreads();
    if (threadIdx.x == 0) {
      ac::tma_store_3d(&tm, t, y0, c * BP, b);
      ac::bulk_commit();
    }
  }
  if (threadIdx.x == 0) ac::bulk_wait_all();
}

// ================================================================== K2Ta: target sums
// Transposed bilinear (D2^T, reading G12): every Cartesian target (p, q) of the half plane
// gets the fixed-order sum of its entries w * P~[node] (deterministic, no atomics).
// One CTA per (column p, image): the targets of column p only reference nodes with
// p0 in {p-1, p}, a contiguous range of the (p0-sorted) adjoint S2 that is staged in shared
// memory (coalesced loads, issued together with the coalesced 16-byte target records).
constexpr int kSumKT = 4;   // target records per thread loaded before the window barrier
constexpr int kSumThreads = 128;

__device__ __forceinline__ float2 k2t_target(const int4 rc, const float2* w, const int2* __restrict__ ov) {
  const float w0 = __int_as_float(rc.y);
  float2 acc = __fmul2_rn(make_float2(w0, w0), w[rc.x]);
  if (rc.z >= 0) {
    const float w1 = __int_as_float(rc.w);
    acc = __ffma2_rn(make_float2(w1, w1), w[rc.z], acc);
  } else {
    const int k0 = -rc.z - 1, cnt = rc.w;
    for (int e = 0; e < cnt - 1; ++e) {
      const int2 en = __ldg(&ov[k0 + e]);
      const float ww = __int_as_float(en.y);
      acc = __ffma2_rn(make_float2(ww, ww), w[en.x], acc);
    }
  }
  return acc;
}

__global__ void __launch_bounds__(kSumThreads) k2t_sum(DevPlan P) {
  extern __shared__ __align__(16) float2 win[];
  const Consts& C = P.C;
  const int p = blockIdx.x, b = C.b0 + blockIdx.y, tid = threadIdx.x;
  const int n0 = __ldg(&P.k2_colptr[p > 0 ? p - 1 : 0]), nw = __ldg(&P.k2_colptr[p + 1]) - n0;
  const int ta = __ldg(&P.k2t_colptr[p]), tb = __ldg(&P.k2t_colptr[p + 1]);
  int4 rec[kSumKT];
#pragma unroll
  for (int k = 0; k < kSumKT; ++k) {
    const int t = ta + tid + kSumThreads * k;
    rec[k] = (t < tb) ? __ldg(&P.k2t_rec[t]) : make_int4(0, 0, 0, 0);
  }
  const float2* S2 = P.S2 + (size_t)b * C.half * C.NL + n0;
  pdl_wait();
  pdl_trigger();
  for (int i = tid; i < nw; i += kSumThreads) win[i] = __ldg(&S2[i]);
  __syncthreads();
  float2* Rc = P.Rc + (size_t)b * C.ntpad;
  const float2* w = win - n0;
#pragma unroll
  for (int k = 0; k < kSumKT; ++k) {
    const int t = ta + tid + kSumThreads * k;
    if (t < tb) Rc[t] = k2t_target(rec[k], w, P.k2t_ov);
  }
  for (int t = ta + tid + kSumThreads * kSumKT; t < tb; t += kSumThreads) Rc[t] = k2t_target(__ldg(&P.k2t_rec[t]), w, P.k2t_ov);
}

static cudaError_t launch_k2t_sum(const DevPlan& P, cudaStream_t s) {
  const Consts& C = P.C;
  const cudaError_t e = launch_pdl(C.pdl, k2t_sum, dim3(C.ncols, C.batch), dim3(kSumThreads),
                                   (size_t)C.k2t_win * sizeof(float2), s, P);
  return e != cudaSuccess ? e : cudaGetLastError();
}

// ================================================================== K2Tb (transpose of K2)
// Column p: scatter its targets into R (kept zero elsewhere), L inverse residue FFTs, then
// S~1[p][y] = sum_s X_s[y'] conj(W_N^{s y''}), the residue sum reduced through smem.
template <int n>
__global__ void __launch_bounds__(1024) k2t_adj(DevPlan P) {
  extern __shared__ __align__(128) float2 sm[];
  constexpr int rs = rstride(n);
  const Consts& C = P.C;
  const int L = C.Lres, L1 = L - 1, lg = C.log2L, ln = L * rs;
  const int b = C.b0 + blockIdx.y;
  const int P0 = blockIdx.x * C.col_strip_adj;
  const int Pend = min(P0 + C.col_strip_adj, C.ncols);
  const int g = threadIdx.x / (n / 8), j = threadIdx.x & (n / 8 - 1);
  const int so = g * rs;
  float2 post[8];
#pragma unroll
  for (int e = 0; e < 8; ++e) post[e] = __ldg(&P.tw_pre[g * n + last_pos<n>(j, e)]);
  const float2* Rc = P.Rc + (size_t)b * C.ntpad;
  float2* out = P.S1 + (size_t)b * C.ncols * n;
  float2* R = sm;        // scatter target, zero outside the targets
  float2* Xb = sm + ln;  // ping-pong, then residue-sum staging
  for (int i = threadIdx.x; i < ln; i += blockDim.x) R[i] = make_float2(0.f, 0.f);
  // prefetch the first target of column P0
  int t0 = __ldg(&P.k2t_colptr[P0]), t1 = __ldg(&P.k2t_colptr[P0 + 1]);
  float2 rv = make_float2(0.f, 0.f);
  int rq = 0;
  if (t0 + (int)threadIdx.x < t1) {
    rv = __ldg(&Rc[t0 + threadIdx.x]);
    rq = __ldg(&P.k2t_tq[t0 + threadIdx.x]);
  }
  __syncthreads();
  for (int p = P0; p < Pend; ++p) {
    {   // scatter column p
      int t = t0 + threadIdx.x;
      if (t < t1) R[fidx(rq, L1, lg, rs)] = rv;
      for (t += blockDim.x; t < t1; t += blockDim.x)
        R[fidx(__ldg(&P.k2t_tq[t]), L1, lg, rs)] = __ldg(&Rc[t]);
    }
    // prefetch the next column's first targets (consumed after this column's transform)
    if (p + 1 < Pend) {
      t0 = t1;
      t1 = __ldg(&P.k2t_colptr[p + 2]);
      if (t0 + (int)threadIdx.x < t1) {
        rv = __ldg(&Rc[t0 + threadIdx.x]);
        rq = __ldg(&P.k2t_tq[t0 + threadIdx.x]);
      }
    }
    __syncthreads();
    float2 v[8];
    passes_inv<n, true>(v, R + so, Xb + so, j, g, L, P.tw_n);
    __syncthreads();   // all groups are done with Xb as scratch
#pragma unroll
    for (int e = 0; e < 8; ++e) Xb[so + last_pos<n>(j, e)] = cmulc(v[e], post[e]);
    __syncthreads();
    for (int yp = threadIdx.x; yp < n; yp += blockDim.x) {
      float2 acc = Xb[yp];
      for (int gg = 1; gg < L; ++gg) acc = cadd(acc, Xb[gg * rs + yp]);
      out[(size_t)p * n + ((yp + n / 2) & (n - 1))] = acc;
    }
    __syncthreads();
  }
}

// ================================================================== K1T (transpose of K1)
// Two row pairs per CTA: Z[p] = C_y[p] + i C_{y+1}[p] (Hermitian completion of the half
// spectra, C[0], C[N/2] = 2 Re), inverse residue FFTs, residue sum -> f~ rows.
template <int n>
__global__ void __launch_bounds__(1024) k1t_adj(DevPlan P, const __grid_constant__ CUtensorMap tm,
                                                 float* __restrict__ fout) {
  extern __shared__ __align__(128) float2 sm[];
  constexpr int rs = rstride(n);
  const Consts& C = P.C;
  const int L = C.Lres, L1 = L - 1, lg = C.log2L, ln = L * rs, N = C.N;
  const int b = C.b0 + blockIdx.y, y0 = 4 * blockIdx.x;
  const int g = threadIdx.x / (n / 8), j = threadIdx.x & (n / 8 - 1);
  const int so = g * rs;
  float2 post[8];
#pragma unroll
  for (int e = 0; e < 8; ++e) post[e] = __ldg(&P.tw_pre[g * n + last_pos<n>(j, e)]);
  float2* ZA = sm;
  float2* ZB = sm + ln;
  float2* X = sm + 2 * ln;
  uint64_t* bar = reinterpret_cast<uint64_t*>(sm + 3 * ln + 2 * n);
  // input: S~1[p][y0..y0+3] as [256 p][4 y] tiles loaded by TMA into X (free before the FFTs)
  const int BP = C.s1boxP, CH = BP * kS1BoxY;
  const int nslot = (ln / CH) < 4 ? (ln / CH) : 4;
  const int nch = (C.ncols + BP - 1) / BP;
  if (threadIdx.x == 0) {
    for (int q = 0; q < nslot; ++q) ac::mbar_init(&bar[q], 1);
    ac::fence_mbar_init();
    for (int c = 0; c < nch && c < nslot; ++c) {
      ac::mbar_expect_tx(&bar[c], CH * 8);
      ac::tma_load_3d(X + c * CH, &tm, y0, c * BP, b, &bar[c]);
    }
  }
  __syncthreads();
  for (int c = 0; c < nch; ++c) {
    const int slot = c % nslot;
    ac::mbar_wait(&bar[slot], (c / nslot) & 1);
    const float2* t = X + slot * CH;
    for (int pl = threadIdx.x; pl < BP; pl += blockDim.x) {
      const int p = c * BP + pl;
      if (p >= C.ncols) break;
      const float2 a0 = t[pl * 4], a1 = t[pl * 4 + 1], b0 = t[pl * 4 + 2], b1 = t[pl * 4 + 3];
      const int ip = fidx(p, L1, lg, rs);
      if (p == 0 || p == N / 2) {
        ZA[ip] = make_float2(2.f * a0.x, 2.f * a1.x);
        ZB[ip] = make_float2(2.f * b0.x, 2.f * b1.x);
      } else {
        const int im = fidx(N - p, L1, lg, rs);
        ZA[ip] = make_float2(a0.x - a1.y, a0.y + a1.x);    // C_y + i C_{y+1}
        ZA[im] = make_float2(a0.x + a1.y, -a0.y + a1.x);   // conj C_y + i conj C_{y+1}
        ZB[ip] = make_float2(b0.x - b1.y, b0.y + b1.x);
        ZB[im] = make_float2(b0.x + b1.y, -b0.y + b1.x);
      }
    }
    __syncthreads();   // slot consumed
    if (threadIdx.x == 0 && c + nslot < nch) {
      ac::fence_proxy_async();
      ac::mbar_expect_tx(&bar[slot], CH * 8);
      ac::tma_load_3d(X + slot * CH, &tm, y0, (c + nslot) * BP, b, &bar[slot]);
    }
  }
#pragma unroll 1
  for (int pr = 0; pr < 2; ++pr) {
    float2* Zs = pr ? ZB : ZA;
    float2 v[8];
    passes_inv<n, false>(v, Zs + so, X + so, j, g, L, P.tw_n);
    __syncthreads();
    float2* red = X;   // free now (results are in registers)
#pragma unroll
    for (int e = 0; e < 8; ++e) red[so + last_pos<n>(j, e)] = cmulc(v[e], post[e]);
    __syncthreads();
    const size_t o = ((size_t)b * n + y0 + 2 * pr) * n;
    const int oxy = (y0 + 2 * pr) * n;
    for (int xp = threadIdx.x; xp < n; xp += blockDim.x) {
      float2 acc = red[xp];
      for (int gg = 1; gg < L; ++gg) acc = cadd(acc, red[gg * rs + xp]);
      const int x = (xp + n / 2) & (n - 1);
      epi_adj_store(P, fout, o + x, oxy + x, acc.x);
      epi_adj_store(P, fout, o + n + x, oxy + n + x, acc.y);
    }
    __syncthreads();
  }
}

// ================================================================== dispatch
static size_t rstride_h(int n) { return (size_t)rstride(n); }
size_t smem_fft4(const Consts& C) {
  return (size_t)3 * C.Lres * rstride_h(C.n) * sizeof(float2) + 2 * C.n * sizeof(float2) + 64;
}
static size_t smem_k2t(const Consts& C) { return (size_t)2 * C.Lres * rstride_h(C.n) * sizeof(float2); }
int fft_threads(const Consts& C) { return C.Lres * (C.n / 8); }

template <int n>
static cudaError_t cfg_one() {
  cudaError_t e = cudaSuccess;
  const int lim = 227 * 1024;
  if (e == cudaSuccess) e = cudaFuncSetAttribute(k2_fwd<n>, cudaFuncAttributeMaxDynamicSharedMemorySize, lim);
  if (e == cudaSuccess) e = cudaFuncSetAttribute(k1_fwd<n>, cudaFuncAttributeMaxDynamicSharedMemorySize, lim);
  if (e == cudaSuccess) e = cudaFuncSetAttribute(k2t_adj<n>, cudaFuncAttributeMaxDynamicSharedMemorySize, lim);
  if (e == cudaSuccess) e = cudaFuncSetAttribute(k1t_adj<n>, cudaFuncAttributeMaxDynamicSharedMemorySize, lim);
  if (e == cudaSuccess) e = cudaFuncSetAttribute(k2t_sum, cudaFuncAttributeMaxDynamicSharedMemorySize, lim);
  return e;
}

#define TAT_DISPATCH_N(...)                                     \
  switch (C.n) {                                                \
    case 32: { constexpr int NN = 32; __VA_ARGS__; } break;     \
    case 64: { constexpr int NN = 64; __VA_ARGS__; } break;     \
    case 128: { constexpr int NN = 128; __VA_ARGS__; } break;   \
    case 256: { constexpr int NN = 256; __VA_ARGS__; } break;   \
    case 512: { constexpr int NN = 512; __VA_ARGS__; } break;   \
    case 1024: { constexpr int NN = 1024; __VA_ARGS__; } break; \
    default: return cudaErrorInvalidValue;                      \
  }

cudaError_t configure_fft_kernels(const Consts& C) {
  TAT_DISPATCH_N(return cfg_one<NN>());
  return cudaSuccess;
}

cudaError_t make_s1_tensor_map(const DevPlan& P, CUtensorMap* out, bool blocked) {
  static PFN_cuTensorMapEncodeTiled_v12000 encode = nullptr;
  if (!encode) {
    void* fn = nullptr;
    cudaDriverEntryPointQueryResult q;
    cudaError_t e = cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q);
    if (e != cudaSuccess || !fn) return e != cudaSuccess ? e : cudaErrorNotSupported;
    encode = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(fn);
  }
  const Consts& C = P.C;
  if (blocked) {   // the two-stage engine's forward S1 [B][n/4][ncols][4 y]: boxes of one column
    cuuint64_t d4[4] = {4, (cuuint64_t)C.ncols, (cuuint64_t)C.n / 4, (cuuint64_t)C.batch};
    cuuint64_t s4[3] = {32, (cuuint64_t)C.ncols * 32, (cuuint64_t)C.ncols * 32 * (C.n / 4)};
    cuuint32_t b4[4] = {4, 1, (cuuint32_t)C.n / 4, 1};
    cuuint32_t e4[4] = {1, 1, 1, 1};
    CUresult r4 = encode(out, CU_TENSOR_MAP_DATA_TYPE_UINT64, 4, P.S1, d4, s4, b4, e4,
                         CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                         CU_TENSOR_MAP_L2_PROMOTION_L2_128B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    return r4 == CUDA_SUCCESS ? cudaSuccess : cudaErrorInvalidValue;
  }
  cuuint64_t dims[3] = {(cuuint64_t)C.n, (cuuint64_t)C.ncols, (cuuint64_t)C.batch};
  cuuint64_t strides[2] = {(cuuint64_t)C.n * 8, (cuuint64_t)C.ncols * C.n * 8};
  cuuint32_t box[3] = {kS1BoxY, (cuuint32_t)C.s1boxP, 1};
  cuuint32_t estr[3] = {1, 1, 1};
  CUresult r = encode(out, CU_TENSOR_MAP_DATA_TYPE_UINT64, 3, P.S1, dims, strides, box, estr,
                      CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                      CU_TENSOR_MAP_L2_PROMOTION_L2_128B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS ? cudaSuccess : cudaErrorInvalidValue;
}

cudaError_t launch_k1(const DevPlan& P, const CUtensorMap& tm, const float* f, cudaStream_t s) {
  const Consts& C = P.C;
  if (col_ok(C)) return launch_k1c_fwd(P, tm, f, s);
  const dim3 grid(C.n / 4, C.batch);
  TAT_DISPATCH_N(k1_fwd<NN><<<grid, fft_threads(C), smem_fft4(C), s>>>(P, tm, f));
  return cudaGetLastError();
}
cudaError_t launch_k2(const DevPlan& P, const CUtensorMap& tm, cudaStream_t s) {
  const Consts& C = P.C;
  if (col_ok(C)) return launch_k2c_fwd(P, tm, s);
  const dim3 grid((C.ncols + C.col_strip - 1) / C.col_strip, C.batch);
  TAT_DISPATCH_N(k2_fwd<NN><<<grid, fft_threads(C), smem_fft4(C), s>>>(P));
  return cudaGetLastError();
}
cudaError_t launch_k2tb(const DevPlan& P, cudaStream_t s) {   // K2Tb only (targets in Rc)
  const Consts& C = P.C;
  if (col_ok(C)) return launch_k2c_adj(P, s);
  const dim3 grid((C.ncols + C.col_strip_adj - 1) / C.col_strip_adj, C.batch);
  TAT_DISPATCH_N(k2t_adj<NN><<<grid, fft_threads(C), smem_k2t(C), s>>>(P));
  return cudaGetLastError();
}

cudaError_t launch_k2t(const DevPlan& P, cudaStream_t s, cudaEvent_t mid) {
  const Consts& C = P.C;
  if (C.k2f == 1) {   // fused: target sums inside the column kernel (no Rc round trip)
    if (mid) cudaEventRecord(mid, s);
    return launch_k2c_adjf(P, s);
  }
  cudaError_t e = C.k2f == 3 ? launch_k2t_strip(P, s)
                  : C.k2f == 2 ? launch_k2t_sumf(P, s) : launch_k2t_sum(P, s);
  if (e != cudaSuccess) return e;
  if (mid) cudaEventRecord(mid, s);
  if (col_ok(C)) return launch_k2c_adj(P, s);
  const dim3 grid((C.ncols + C.col_strip_adj - 1) / C.col_strip_adj, C.batch);
  TAT_DISPATCH_N(k2t_adj<NN><<<grid, fft_threads(C), smem_k2t(C), s>>>(P));
  return cudaGetLastError();
}
cudaError_t launch_k1t(const DevPlan& P, const CUtensorMap& tm, float* f, cudaStream_t s) {
  const Consts& C = P.C;
  if (col_ok(C)) return launch_k1c_adj(P, tm, f, s);
  const dim3 grid(C.n / 4, C.batch);
  TAT_DISPATCH_N(k1t_adj<NN><<<grid, fft_threads(C), smem_fft4(C), s>>>(P, tm, f));
  return cudaGetLastError();
}

}  // namespace tat
