// Column stage of the oversampled 2-D DFT (Alg. 1 steps 2-3 and Alg. 2 steps 5-6, PAPER.md
// L547-551, L684-687) as a two-stage split with R = 16 points per thread in registers:
//
//   F[q] = sum_{y<n} x[y] W_N^{q (y - n/2)},  N = L n,  y = j + J r  (J = n/R),
//   q = q0 + Q0 q1  (Q0 = R L, q0 = s + L k1):
//   F[q0 + Q0 q1] = sum_j W_J^{q1 j} * W_n^{k1 (j - n/2)} *
//                   sum_r x[j + J r] W_N^{s (j + J r - n/2)} W_R^{k1 r}
//
//   stage A (thread (j, s)): pre-twiddle, R-point DFT over r, post-twiddle b^k1 (b = W_n^{j-n/2})
//   stage B (thread q0)    : J-point DFT over j (pure, in place in shared memory)
//
// Each point crosses shared memory once between the stages (vs. P-1 exchanges of a radix-8
// Stockham), and a thread reads its column samples once for all of its residues s.
// The transposed kernel runs the conjugate stages in reverse order (exact adjoint).
//
//   k2c_fwd : S1 [B][ncols][n] -> S2 [B][nodes]   column DFT + bilinear gather (as k2_fwd)
//   k2c_adj : Rc [B][targets]  -> S1              target values -> inverse column DFT
//                                                 (targets per column ordered by (q0, q1))
#include "async_copy.cuh"
#include "col_engine.cuh"
#include "tat_internal.h"

#include <algorithm>

namespace tat {

namespace {

#ifndef TAT_FACT_POW
#define TAT_FACT_POW 0
#endif
// post-twiddle powers of the stage-A jobs (PowR): all R - 1 powers in registers (0; one complex
// multiply per point) or factored b^(k mod 4) (b^4)^(k div 4) (1; ~1.9 multiplies per point,
// 16 fewer registers).  Measured at C3 (round 2): full powers K2 236 -> 231 us, K2Tb 218 -> 212,
// K4 66 -> 65, K4T 75 -> 73; C5 K2 344 -> 324, K2Tb 314 -> 296.  K1 keeps the factored powers
// (the full ones spill there: 4 bytes at 168 registers, and K1 measured 52 -> 54 us).
constexpr bool kFactPow = TAT_FACT_POW;
constexpr bool kFactPowK1 = true;

__host__ __device__ constexpr int ilog2c(int v) { return v <= 1 ? 0 : 1 + ilog2c(v / 2); }

// R points per thread in stage A: 16 for n <= 512, 32 for n = 1024 (keeps J = n / R <= 32)
template <int n_, int L_ = 8, int PAD_ = 1>
struct ColGeo {
  static constexpr int n = n_, L = L_, R = (n_ >= 1024) ? 32 : 16, J = n / R, Q0 = R * L, T = Q0;
  static constexpr int NG = T / J;        // residue groups (threads sharing j)
  static constexpr int NRES = J * L / T;  // residues per thread in stage A
  static constexpr int LGQ0 = ilog2c(Q0); // log2 Q0
  static_assert(J >= R && J <= 32 && (L == 8 || L == 4), "n in {256, 512, 1024}, L in {4, 8}");
  // element (q0, c) of a column buffer [Q0][J]: a padded row stride J + 1 (PAD_ = 1) or an XOR
  // swizzle (PAD_ = 0); both are conflict-free for the 8-byte accesses of both stages.  The
  // padding saves the per-access XOR (measured: K2 258 -> 237 us, K4 75 -> 68, K2Tb 229 -> 219 at
  // C3); K1T keeps the swizzle (67 vs 72 us padded).
  static constexpr int WP = J + PAD_, WS = Q0 * WP;   // row stride, buffer size (float2)
  __device__ static __forceinline__ int widx(int q0, int c) {
    return PAD_ ? q0 * WP + c : q0 * J + (c ^ (q0 & (J - 1)));
  }
  __device__ static __forceinline__ int fq(int q) { return widx(q & (Q0 - 1), q >> LGQ0); }
};

}  // namespace

using ce::cmul;
using ce::cmulc;
using ce::csub;

// ------------------------------------------------------------------ post-twiddle powers b^k
// FULL: b^1..b^(R-1) in registers (binary splitting).  FACT: b^k = b^(k mod 4) (b^4)^(k div 4)
// from 3 + R/4 - 1 registers (one extra multiply for most k; lower register pressure).
template <int R, bool FACT>
struct PowR {
  float2 p[R];
  __device__ __forceinline__ void init(float2 b) { ce::pow_tree<R>(b, p); }
  __device__ __forceinline__ float2 mul(float2 v, int k) const { return cmul(v, p[k]); }
  __device__ __forceinline__ float2 mulc(float2 v, int k) const { return cmulc(v, p[k]); }
};
template <int R>
struct PowR<R, true> {
  float2 lo[4], hi[R / 4];
  __device__ __forceinline__ void init(float2 b) {
    lo[1] = b;
    lo[2] = cmul(b, b);
    lo[3] = cmul(lo[2], b);
    hi[1] = cmul(lo[2], lo[2]);
#pragma unroll
    for (int i = 2; i < R / 4; ++i) hi[i] = cmul(hi[i / 2], hi[i - i / 2]);
  }
  __device__ __forceinline__ float2 mul(float2 v, int k) const {
    if (k & 3) v = cmul(v, lo[k & 3]);
    if (k >> 2) v = cmul(v, hi[k >> 2]);
    return v;
  }
  __device__ __forceinline__ float2 mulc(float2 v, int k) const {
    if (k & 3) v = cmulc(v, lo[k & 3]);
    if (k >> 2) v = cmulc(v, hi[k >> 2]);
    return v;
  }
};

// ------------------------------------------------------------------ shared stage code
// Per-thread twiddles: A[i][r] = tab[s_i][j + J r] (s_i = sg + NG i; for the column transform
// tab = tw_col, W_N^{s (y - n/2)}), pw[k] = b^k with b = W_n^{j - shift}.
template <class G, class PW>
__device__ __forceinline__ void col_twiddles(const float2* __restrict__ tab, const float2* __restrict__ tw_n,
                                             int shift, int j, int sg, float2 (&A)[G::NRES][G::R], PW& pw) {
  constexpr int n = G::n;
#pragma unroll
  for (int i = 0; i < G::NRES; ++i)
#pragma unroll
    for (int r = 0; r < G::R; ++r) A[i][r] = __ldg(&tab[(sg + G::NG * i) * n + j + G::J * r]);
  pw.init(__ldg(&tw_n[(j - shift) & (n - 1)]));
}

// stage A: samples x[r] = x[j + J r] -> W[(s + L k1, j)] for the thread's residues s
template <class G, class PW>
__device__ __forceinline__ void stage_a_fwd(const float2 (&x)[G::R], const float2 (&A)[G::NRES][G::R],
                                            const PW& pw, float2* W, int j, int sg) {
#pragma unroll
  for (int i = 0; i < G::NRES; ++i) {
    const int s = sg + G::NG * i;
    float2 v[G::R];
#pragma unroll
    for (int r = 0; r < G::R; ++r) v[r] = cmul(x[r], A[i][r]);
    ce::dftr<G::R, -1>(v);
#pragma unroll
    for (int k1 = 1; k1 < G::R; ++k1) v[k1] = pw.mul(v[k1], k1);
#pragma unroll
    for (int k1 = 0; k1 < G::R; ++k1) W[G::widx(s + G::L * k1, j)] = v[k1];
  }
}

// stage B: J-point DFT (sign S) of row q0 of W, in place
template <class G, int S>
__device__ __forceinline__ void stage_b(float2* W, int q0) {
  float2 u[G::J];
#pragma unroll
  for (int c = 0; c < G::J; ++c) u[c] = W[G::widx(q0, c)];
  ce::dftr<G::J, S>(u);
#pragma unroll
  for (int c = 0; c < G::J; ++c) W[G::widx(q0, c)] = u[c];
}

// stage A^H: W -> acc[r] = sum over the thread's residues of the conjugate chain at j + J r
template <class G, class PW>
__device__ __forceinline__ void stage_a_adj(const float2* W, const float2 (&A)[G::NRES][G::R],
                                            const PW& pw, int j, int sg, float2 (&acc)[G::R]) {
#pragma unroll
  for (int i = 0; i < G::NRES; ++i) {
    const int s = sg + G::NG * i;
    float2 v[G::R];
#pragma unroll
    for (int k1 = 0; k1 < G::R; ++k1) v[k1] = W[G::widx(s + G::L * k1, j)];
#pragma unroll
    for (int k1 = 1; k1 < G::R; ++k1) v[k1] = pw.mulc(v[k1], k1);
    ce::dftr<G::R, 1>(v);
#pragma unroll
    for (int r = 0; r < G::R; ++r) {
      const float2 w = cmulc(v[r], A[i][r]);
      acc[r] = (i == 0) ? w : ce::cadd(acc[r], w);
    }
  }
}

// residue-group partial sums -> W[0..n) (fixed order); starts with the barrier that ends the
// stage-A^H reads of W, ends with a barrier (W[y] = sum, y in [0, n))
template <class G>
__device__ __forceinline__ void residue_reduce(float2* W, const float2 (&acc)[G::R], int j, int sg) {
  constexpr int n = G::n;
  __syncthreads();
#pragma unroll
  for (int r = 0; r < G::R; ++r) W[sg * n + j + G::J * r] = acc[r];
  __syncthreads();
}
template <class G>
__device__ __forceinline__ float2 residue_sum(const float2* W, int y) {
  float2 s = W[y];
#pragma unroll
  for (int g = 1; g < G::NG; ++g) s = ce::cadd(s, W[g * G::n + y]);
  return s;
}

// The forward's S1 in the two-stage engine is blocked [B][n/4][ncols][4 y]: the 4 rows y of one
// quad at one p are 32 contiguous bytes, so K1's output for a quad of rows is one contiguous
// range, while a column p (K2's input) is one TMA box of n/4 pieces of 32 bytes.  The adjoint's
// S~1 (K2Tb -> K1T) stays column-major [B][ncols][n].
__device__ __forceinline__ size_t s1b(const Consts& C, int b, int y, int p) {
  return (((size_t)b * (C.n / 4) + (y >> 2)) * C.ncols + p) * 4 + (y & 3);
}
// ================================================================== forward
#ifndef TAT_K2_3BUF
#define TAT_K2_3BUF 0   // three column buffers at every n (default: only where occupancy is 1 anyway)
#endif
// Three column buffers drop the barrier between a column's gather and the next stage A.  At
// n >= 1024 one CTA fits per SM either way and the third buffer is free (C5 K2 300 -> 290 us); at
// n = 512 it costs the third resident CTA (C3 K2 229 -> 252 us), so two buffers there.
__host__ __device__ constexpr int k2_bufs(int n) { return (TAT_K2_3BUF || n >= 1024) ? 3 : 2; }
template <int n>
__global__ void __launch_bounds__(ColGeo<n>::T, n >= 1024 ? 1 : (TAT_K2_3BUF ? 2 : 3))
    k2c_fwd(DevPlan P, const __grid_constant__ CUtensorMap tm) {
  constexpr int kK2Bufs = k2_bufs(n);
  using G = ColGeo<n>;
  constexpr int R = G::R, J = G::J, NRES = G::NRES;
  extern __shared__ __align__(128) float2 sm[];
  const Consts& C = P.C;
  const int N1 = C.N - 1;
  const int t = threadIdx.x, j = t % J, sg = t / J;
  const int b = C.b0 + blockIdx.y;
  const int P0 = blockIdx.x * C.col_strip;
  const int Pend = min(P0 + C.col_strip, C.ncols);
  const int plast = min(Pend, C.ncols - 1);
  float2* Fa = sm;
  float2* Fb = sm + G::WS;
  float2* xbuf = sm + kK2Bufs * G::WS;                    // 2 x n, TMA destination
  uint64_t* bar = reinterpret_cast<uint64_t*>(xbuf + 2 * n);
  float2 A[NRES][R];
  PowR<G::R, kFactPow> pw;
  col_twiddles<G>(P.tw_col, P.tw_n, n / 2, j, sg, A, pw);
  float2* S2 = P.S2 + (size_t)b * C.half * C.NL;
  pdl_wait();
  pdl_trigger();
  // column p of the blocked S1 (s1b): one TMA box of n/4 pieces of 32 bytes, in y order
  if (t == 0) {
    ac::mbar_init(&bar[0], 1);
    ac::mbar_init(&bar[1], 1);
    ac::fence_mbar_init();
    ac::mbar_expect_tx(&bar[0], n * 8);
    ac::tma_load_4d(xbuf, &tm, 0, P0, 0, b, &bar[0]);
  }
  __syncthreads();
  float2* Fprev = Fb;
  float2* Fcur = Fa;
  for (int p = P0; p <= plast; ++p) {
    const int it = p - P0, slot = it & 1;
    if (t == 0 && p < plast) {
      ac::fence_proxy_async();
      ac::mbar_expect_tx(&bar[slot ^ 1], n * 8);
      ac::tma_load_4d(xbuf + (slot ^ 1) * n, &tm, 0, p + 1, 0, b, &bar[slot ^ 1]);
    }
    ac::mbar_wait(&bar[slot], (it >> 1) & 1);
    {   // stage A
      const float2* xs = xbuf + slot * n;
      float2 x[R];
#pragma unroll
      for (int r = 0; r < R; ++r) x[r] = xs[j + J * r];
      stage_a_fwd<G>(x, A, pw, Fcur, j, sg);
    }
    // first node record of this column's gather, loaded while stage B runs (after stage A, whose
    // registers are dead by then).  (Measured: all records by cp.async into the consumed input
    // slot instead: K2 229 -> 239 us at C3; the gather is not record-latency bound.)
    const int e0 = (p > P0) ? __ldg(&P.k2_colptr[p - 1]) : 0;
    const int e1 = (p > P0) ? __ldg(&P.k2_colptr[p]) : 0;
    int4 nd0 = make_int4(0, 0, 0, 0), nd1 = make_int4(0, 0, 0, 0);   // (the second for columns
    if (e0 + t < e1) nd0 = __ldg(&P.k2_nodes[e0 + t]);                // with more than T nodes)
    if (e0 + t + G::T < e1) nd1 = __ldg(&P.k2_nodes[e0 + t + G::T]);
    __syncthreads();
    stage_b<G, -1>(Fcur, t);   // stage B (in place)
    __syncthreads();
    if (p > P0) {   // bilinear gather of the nodes with p0 = p - 1 (Alg. 1 step 3)
      int e = e0 + t;
      int4 nd = nd0, nn = nd1;
      while (e < e1) {
        const float a = __int_as_float(nd.z), bb = __int_as_float(nd.w);
        const int i00 = G::fq(nd.y & N1), i01 = G::fq((nd.y + 1) & N1);
        const float2 f00 = Fprev[i00], f01 = Fprev[i01], f10 = Fcur[i00], f11 = Fcur[i01];
        const float2 c0 = __ffma2_rn(make_float2(a, a), csub(f10, f00), f00);
        const float2 c1 = __ffma2_rn(make_float2(a, a), csub(f11, f01), f01);
#ifndef TAT_K2_NOSTORE
        S2[nd.x] = __ffma2_rn(make_float2(bb, bb), csub(c1, c0), c0);
#else   // timing experiment only (wrong results): the stores skipped unless impossible
        const float2 vv = __ffma2_rn(make_float2(bb, bb), csub(c1, c0), c0);
        if (vv.x == 1.2345e-38f) S2[nd.x] = vv;
#endif
        e += G::T;
        nd = nn;
        if (e + G::T < e1) nn = __ldg(&P.k2_nodes[e + G::T]);
      }
    }
    if (kK2Bufs == 2) {
      __syncthreads();   // the next stage A overwrites Fprev
      float2* tmp = Fprev;
      Fprev = Fcur;
      Fcur = tmp;
    } else {             // three buffers: the next stage A writes the third one
      float2* nxt = (Fcur == Fa) ? Fb : (Fcur == Fb ? sm + 2 * G::WS : Fa);
      Fprev = Fcur;
      Fcur = nxt;
    }
  }
  if (Pend == C.ncols) {   // p0 = N/2: alpha == 0, only F[N/2] is used
    for (int e = P.k2_colptr[C.ncols - 1] + t; e < P.k2_colptr[C.ncols]; e += G::T) {
      const int4 nd = __ldg(&P.k2_nodes[e]);
      const float bb = __int_as_float(nd.w);
      const float2 f00 = Fprev[G::fq(nd.y & N1)];
      const float2 f01 = Fprev[G::fq((nd.y + 1) & N1)];
      S2[nd.x] = __ffma2_rn(make_float2(bb, bb), csub(f01, f00), f00);
    }
  }
}

// ================================================================== adjoint (transpose)
// Column p: the target values of column p (Rc, ordered by (q0, q1), moved by one bulk copy per
// column into a double buffer) -> stage B^H (thread q0, only the present q1 are read) ->
// stage A^H (thread (j, s)) -> residue-group partial sums -> S~1[b][p][y].
template <int n, bool CHORD>
__global__ void __launch_bounds__(ColGeo<n>::T, n >= 1024 ? 1 : 3) k2c_adj(DevPlan P) {
  using G = ColGeo<n>;
  constexpr int R = G::R, J = G::J, NRES = G::NRES, Q0 = G::Q0;
  extern __shared__ __align__(128) float2 sm[];
  const Consts& C = P.C;
  const int t = threadIdx.x, j = t % J, sg = t / J;
  const int b = C.b0 + blockIdx.y;
  const int P0 = blockIdx.x * C.col_strip_adj;
  const int Pend = min(P0 + C.col_strip_adj, C.ncols);
  const int RB = C.k2c_rbuf;                                  // entries per target buffer
  float2* Wb = sm;
  float2* rbuf = sm + G::WS;
  uint64_t* bar = reinterpret_cast<uint64_t*>(rbuf + 2 * RB);
  float2 A[NRES][R];
  PowR<G::R, kFactPow> pw;
  col_twiddles<G>(P.tw_col, P.tw_n, n / 2, j, sg, A, pw);
  const float2* Rc = P.Rc + (size_t)b * C.ntpad;
  auto issue = [&](int p, int slot) {   // thread 0: bulk copy of column p's targets
    const int s0 = __ldg(&P.k2t_colptr[p]) & ~1;
    const int s1 = (__ldg(&P.k2t_colptr[p + 1]) + 1) & ~1;
    if (s1 > s0) {
      ac::mbar_expect_tx(&bar[slot], (s1 - s0) * 8);
      ac::bulk_g2s(rbuf + slot * RB, Rc + s0, (s1 - s0) * 8, &bar[slot]);
    } else {
      asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(ac::smem_u32(&bar[slot])) : "memory");
    }
  };
  pdl_wait();
  pdl_trigger();
  if (t == 0) {
    ac::mbar_init(&bar[0], 1);
    ac::mbar_init(&bar[1], 1);
    ac::fence_mbar_init();
    issue(P0, 0);
  }
  __syncthreads();
  uint32_t m = 0;
  int base = 0;
  if (!CHORD) {
    m = __ldg(&P.k2c_mask[(size_t)P0 * Q0 + t]);
    base = __ldg(&P.k2c_base[(size_t)P0 * Q0 + t]) - (__ldg(&P.k2t_colptr[P0]) & ~1);
  }
  for (int p = P0; p < Pend; ++p) {
    const int it = p - P0, slot = it & 1;
    if (t == 0 && p + 1 < Pend) {
      ac::fence_proxy_async();
      issue(p + 1, slot ^ 1);
    }
    uint32_t m_next = 0;
    int base_next = 0;
    if (!CHORD && p + 1 < Pend) {
      m_next = __ldg(&P.k2c_mask[(size_t)(p + 1) * Q0 + t]);
      base_next = __ldg(&P.k2c_base[(size_t)(p + 1) * Q0 + t]) - (__ldg(&P.k2t_colptr[p + 1]) & ~1);
    }
    ac::mbar_wait(&bar[slot], (it >> 1) & 1);
    {   // stage B^H: A~[q0][j] = sum_q1 W_J^{-q1 j} F~[q0 + Q0 q1]
      float2 u[J];
      if (CHORD) {   // targets q = -Qp .. Qp at offset q + Qp of the column
        const int Qp = __ldg(&P.k2c_chord[p]);
        const float2* rb = rbuf + slot * RB + (__ldg(&P.k2t_colptr[p]) & 1) + Qp;
#pragma unroll
        for (int c = 0; c < J; ++c) {
          const int qm = t + Q0 * c, q = qm < C.N / 2 ? qm : qm - C.N;
          u[c] = (q >= -Qp && q <= Qp) ? rb[q] : make_float2(0.f, 0.f);
        }
      } else {
        const float2* rb = rbuf + slot * RB + base;
#pragma unroll
        for (int c = 0; c < J; ++c) {
          const uint32_t below = m & ((1u << c) - 1u);
          u[c] = ((m >> c) & 1u) ? rb[__popc(below)] : make_float2(0.f, 0.f);
        }
      }
      ce::dftr<J, 1>(u);
#pragma unroll
      for (int c = 0; c < J; ++c) Wb[G::widx(t, c)] = u[c];
    }
    __syncthreads();
    float2 acc[R];
    stage_a_adj<G>(Wb, A, pw, j, sg, acc);
    residue_reduce<G>(Wb, acc, j, sg);
    // the adjoint's S~1 is column-major (coalesced column stores; K1T reads [128 p][4 y] TMA tiles).
    // (Measured with the forward's blocked layout here: K2Tb 211.5 -> 218 us at C3, 8 pieces of
    // 32 bytes per warp store; staged and stored as one TMA box: 219.)
    float2* out = P.S1 + ((size_t)b * C.ncols + p) * n;
    for (int y = t; y < n; y += G::T) out[y] = residue_sum<G>(Wb, y);
    __syncthreads();   // Wb free; rbuf[slot] consumed
    m = m_next;
    base = base_next;
  }
}

// ================================================================== adjoint, fused (K2T)
// The whole adjoint column stage A*-4 in one kernel (Alg. 2 steps 5-6, with
// step 5's interpolation replaced by the exact transpose of A-2's bilinear gather, reading G4):
// one CTA per (column p, group of images).  The column's target records (which nodes of the
// window, with which bilinear weights, sum into each Cartesian target (p, q); 12 bytes each)
// are staged in shared memory once and reused for every image; per image, the node window
// (the nodes with p0 in {p-1, p}: one contiguous range of the adjoint S2) arrives by a bulk
// copy double-buffered one image ahead.  Phase 1 forms the target sums in a fixed order
// (deterministic, no atomics) into a compact array that aliases the column buffer; then stage
// B^H (only the present q1 are read), stage A^H and the residue sums as in k2c_adj.  Columns
// whose records or window exceed the shared-memory caps (the origin columns) read them from
// global memory instead.
template <int n>
__global__ void __launch_bounds__(ColGeo<n>::T, n >= 1024 ? 1 : 3) k2c_adjf(DevPlan P) {
  using G = ColGeo<n>;
  constexpr int R = G::R, J = G::J, NRES = G::NRES, Q0 = G::Q0, T = G::T, NW = T / 32;
  extern __shared__ __align__(128) float2 sm[];
  const Consts& C = P.C;
  const int t = threadIdx.x, j = t % J, sg = t / J, lane = t & 31, warp = t >> 5;
  // CTA -> work item: the slow columns (origin region: over the shared-memory caps) first, one
  // image per CTA, so they run concurrently with everything else and are not the kernel's tail;
  // then the other columns, k2f_ipc images per CTA
  const int ngrp = (C.batch + C.k2f_ipc - 1) / C.k2f_ipc;
  const int nsl = C.k2f_nslow * C.batch;
  const bool slow = (int)blockIdx.x < nsl;
  int p, bA, bB;
  if (slow) {
    p = __ldg(&P.k2f_cols[blockIdx.x / C.batch]);
    bA = C.b0 + blockIdx.x % C.batch;
    bB = bA + 1;
  } else {
    const int id = blockIdx.x - nsl;
    p = __ldg(&P.k2f_cols[C.k2f_nslow + id / ngrp]);
    bA = C.b0 + (id % ngrp) * C.k2f_ipc;
    bB = min(bA + C.k2f_ipc, C.b0 + C.batch);
  }
  float2* Wb = sm;                                                     // column buffer / targets
  uint32_t* recs = reinterpret_cast<uint32_t*>(sm + G::WS);            // [rcap][3]
  float2* win = sm + G::WS + (3 * C.k2f_rcap + 1) / 2;                 // 2 x [wcap]
  uint64_t* bar = reinterpret_cast<uint64_t*>(win + 2 * C.k2f_wcap);
  float2 A[NRES][R];
  PowR<G::R, kFactPow> pw;
  col_twiddles<G>(P.tw_col, P.tw_n, n / 2, j, sg, A, pw);
  const int r0 = __ldg(&P.k2f_recptr[p]), nrec = __ldg(&P.k2f_recptr[p + 1]) - r0;
  const int t0 = __ldg(&P.k2t_colptr[p]), ntg = __ldg(&P.k2t_colptr[p + 1]) - t0;
  const int w0 = __ldg(&P.k2_colptr[p > 0 ? p - 1 : 0]), nwin = __ldg(&P.k2_colptr[p + 1]) - w0;
  const uint32_t m = __ldg(&P.k2c_mask[(size_t)p * Q0 + t]);
  const int base = __ldg(&P.k2c_base[(size_t)p * Q0 + t]) - t0;
  const size_t img = (size_t)C.half * C.NL;
  const uint32_t* rp = slow ? P.k2f_rec + (size_t)3 * r0 : recs;
  // targets with more than two entries: their descriptors (index in column, first entry, count)
  // and entry lists are column constants, staged after the records once per CTA (fast columns)
  const int o0 = __ldg(&P.k2f_ovptr[p]), nov = __ldg(&P.k2f_ovptr[p + 1]) - o0;
  const int e0 = nov > 0 ? __ldg(&P.k2f_ovt[o0]).y : 0;
  const int ne = nov > 0 ? __ldg(&P.k2f_ovt[o0 + nov - 1]).y + __ldg(&P.k2f_ovt[o0 + nov - 1]).z - e0 : 0;
  int4* ovt_s = reinterpret_cast<int4*>(recs + 3 * nrec);                // nrec: multiple of 4
  int2* ove_s = reinterpret_cast<int2*>(ovt_s + nov);
  const int4* ovt = slow ? P.k2f_ovt + o0 : ovt_s;
  const int2* ove = slow ? P.k2f_ov + e0 : ove_s;
  if (!slow) {
    for (int i = t; i < nov; i += T) ovt_s[i] = __ldg(&P.k2f_ovt[o0 + i]);
    for (int i = t; i < ne; i += T) ove_s[i] = __ldg(&P.k2f_ov[e0 + i]);
  }
  auto issue = [&](int b, int slot) {   // thread 0: node window of image b -> win[slot]
    const size_t s0 = ((size_t)b * img + w0) & ~(size_t)1;
    const size_t s1 = ((size_t)b * img + w0 + nwin + 1) & ~(size_t)1;
    ac::mbar_expect_tx(&bar[slot], (uint32_t)(s1 - s0) * 8);
    ac::bulk_g2s(win + slot * C.k2f_wcap, P.S2 + s0, (uint32_t)(s1 - s0) * 8, &bar[slot]);
  };
  if (t == 0) {   // the records are plan tables: staged before the predecessor has finished
    ac::mbar_init(&bar[0], 1);
    ac::mbar_init(&bar[1], 1);
    ac::mbar_init(&bar[2], 1);
    ac::fence_mbar_init();
    if (!slow && nrec > 0) {
      ac::mbar_expect_tx(&bar[2], (uint32_t)nrec * 12);
      ac::bulk_g2s(recs, P.k2f_rec + (size_t)3 * r0, (uint32_t)nrec * 12, &bar[2]);
    }
  }
  pdl_wait();
  pdl_trigger();
  if (t == 0 && !slow) issue(bA, 0);
  __syncthreads();
  if (!slow && nrec > 0) ac::mbar_wait(&bar[2], 0);
  for (int b = bA; b < bB; ++b) {
    const int it = b - bA, slot = it & 1;
    if (t == 0 && !slow && b + 1 < bB) {
      ac::fence_proxy_async();
      issue(b + 1, slot ^ 1);
    }
    const float2* wv;
    if (!slow) {
      ac::mbar_wait(&bar[slot], (it >> 1) & 1);
      wv = win + slot * C.k2f_wcap + (int)(((size_t)b * img + w0) & 1);
    } else {
      wv = P.S2 + (size_t)b * img + w0;
    }
    // phase 1: target sums (fixed order: entry 0, then entry 1), KU targets per thread per
    // pass with every load issued before the arithmetic (the slow columns read global memory)
    constexpr int KU = 4;
    for (int q = t; q < ntg; q += KU * T) {
      uint32_t i01[KU], wa[KU], wb[KU];
#pragma unroll
      for (int k = 0; k < KU; ++k) {
        const int qq = q + k * T;
        const bool ok = qq < ntg;
        i01[k] = ok ? rp[3 * qq] : 0u;
        wa[k] = ok ? rp[3 * qq + 1] : 0u;
        wb[k] = ok ? rp[3 * qq + 2] : 0u;
      }
      float2 v0[KU], v1[KU];
#pragma unroll
      for (int k = 0; k < KU; ++k) {
        const bool ov = (i01[k] >> 16) == 0xFFFFu;
        v0[k] = ov ? make_float2(0.f, 0.f) : wv[i01[k] & 0xFFFFu];
        v1[k] = ov ? make_float2(0.f, 0.f) : wv[i01[k] >> 16];
      }
#pragma unroll
      for (int k = 0; k < KU; ++k) {
        const int qq = q + k * T;
        if (qq >= ntg) break;
        if ((i01[k] >> 16) == 0xFFFFu) continue;   // more than two entries: second pass
        const float w0f = __uint_as_float(wa[k]), w1f = __uint_as_float(wb[k]);
        float2 acc = __fmul2_rn(make_float2(w0f, w0f), v0[k]);
        Wb[qq] = __ffma2_rn(make_float2(w1f, w1f), v1[k], acc);
      }
    }
    // second pass: targets with more than two entries (1.5 % at C3; up to ~280 entries near the
    // origin), one warp each: lane l sums the entries e = l (mod 32) in order, then a fixed
    // xor-butterfly combines the lanes (deterministic)
    auto butterfly_store = [&](float2 acc, int dst) {
#pragma unroll
      for (int off = 16; off > 0; off >>= 1) {
        acc.x += __shfl_xor_sync(0xffffffffu, acc.x, off);
        acc.y += __shfl_xor_sync(0xffffffffu, acc.y, off);
      }
      if (lane == 0) Wb[dst] = acc;
    };
    for (int o = warp; o < nov; o += NW) {
      const int4 d = ovt[o];
      float2 acc = make_float2(0.f, 0.f);
      for (int e = lane; e < d.z; e += 32) {
        const int2 en = ove[d.y - e0 + e];
        const float w = __int_as_float(en.y);
        acc = __ffma2_rn(make_float2(w, w), wv[en.x], acc);
      }
      butterfly_store(acc, d.x);
    }
    __syncthreads();
    {   // stage B^H: A~[q0][j] = sum_q1 W_J^{-q1 j} F~[q0 + Q0 q1]
      float2 u[J];
      const float2* rb = Wb + base;
#pragma unroll
      for (int c = 0; c < J; ++c) {
        const uint32_t below = m & ((1u << c) - 1u);
        u[c] = ((m >> c) & 1u) ? rb[__popc(below)] : make_float2(0.f, 0.f);
      }
      __syncthreads();   // the target sums alias the column buffer
      ce::dftr<J, 1>(u);
#pragma unroll
      for (int c = 0; c < J; ++c) Wb[G::widx(t, c)] = u[c];
    }
    __syncthreads();
    float2 acc[R];
    stage_a_adj<G>(Wb, A, pw, j, sg, acc);
    residue_reduce<G>(Wb, acc, j, sg);
    float2* out = P.S1 + ((size_t)b * C.ncols + p) * n;   // column-major (see k2c_adj)
    for (int y = t; y < n; y += T) out[y] = residue_sum<G>(Wb, y);
    __syncthreads();   // Wb free; win[slot] consumed
  }
}

// ================================================================== K2Ta, multi-image
// The transposed bilinear alone (target sums -> Rc, read by k2c_adj), with k2c_adjf's tables and
// work split: one CTA per (column, group of images), the column's records and overflow lists
// staged in shared memory once, one node window per image double-buffered by bulk copies; the
// slow (origin) columns run one image per CTA at the head of the grid from global memory.
// Fixed-order sums, the > 2-entry targets by one warp each (lane-strided, xor butterfly).
constexpr int kSumfT = 256;
__global__ void __launch_bounds__(kSumfT) k2t_sumf(DevPlan P) {
  constexpr int T = kSumfT, NW = T / 32;
  extern __shared__ __align__(128) float2 sm[];
  const Consts& C = P.C;
  const int t = threadIdx.x, lane = t & 31, warp = t >> 5;
  const int ngrp = (C.batch + C.k2f_ipc - 1) / C.k2f_ipc;
  const int nsl = C.k2f_nslow * C.batch;
  const bool slow = (int)blockIdx.x < nsl;
  int p, bA, bB;
  if (slow) {
    p = __ldg(&P.k2f_cols[blockIdx.x / C.batch]);
    bA = C.b0 + blockIdx.x % C.batch;
    bB = bA + 1;
  } else {
    const int id = blockIdx.x - nsl;
    p = __ldg(&P.k2f_cols[C.k2f_nslow + id / ngrp]);
    bA = C.b0 + (id % ngrp) * C.k2f_ipc;
    bB = min(bA + C.k2f_ipc, C.b0 + C.batch);
  }
  uint32_t* recs = reinterpret_cast<uint32_t*>(sm);                    // [rcap][3]
  float2* win = sm + (3 * C.k2f_rcap + 1) / 2;                         // 2 x [wcap]
  uint64_t* bar = reinterpret_cast<uint64_t*>(win + 2 * C.k2f_wcap);
  const int r0 = __ldg(&P.k2f_recptr[p]), nrec = __ldg(&P.k2f_recptr[p + 1]) - r0;
  const int t0 = __ldg(&P.k2t_colptr[p]), ntg = __ldg(&P.k2t_colptr[p + 1]) - t0;
  const int w0 = __ldg(&P.k2_colptr[p > 0 ? p - 1 : 0]), nwin = __ldg(&P.k2_colptr[p + 1]) - w0;
  const size_t img = (size_t)C.half * C.NL;
  const uint32_t* rp = slow ? P.k2f_rec + (size_t)3 * r0 : recs;
  const int o0 = __ldg(&P.k2f_ovptr[p]), nov = __ldg(&P.k2f_ovptr[p + 1]) - o0;
  const int e0 = nov > 0 ? __ldg(&P.k2f_ovt[o0]).y : 0;
  const int ne = nov > 0 ? __ldg(&P.k2f_ovt[o0 + nov - 1]).y + __ldg(&P.k2f_ovt[o0 + nov - 1]).z - e0 : 0;
  int4* ovt_s = reinterpret_cast<int4*>(recs + 3 * nrec);
  int2* ove_s = reinterpret_cast<int2*>(ovt_s + nov);
  const int4* ovt = slow ? P.k2f_ovt + o0 : ovt_s;
  const int2* ove = slow ? P.k2f_ov + e0 : ove_s;
  if (!slow) {
    for (int i = t; i < nov; i += T) ovt_s[i] = __ldg(&P.k2f_ovt[o0 + i]);
    for (int i = t; i < ne; i += T) ove_s[i] = __ldg(&P.k2f_ov[e0 + i]);
  }
  auto issue = [&](int b, int slot) {
    const size_t s0 = ((size_t)b * img + w0) & ~(size_t)1;
    const size_t s1 = ((size_t)b * img + w0 + nwin + 1) & ~(size_t)1;
    ac::mbar_expect_tx(&bar[slot], (uint32_t)(s1 - s0) * 8);
    ac::bulk_g2s(win + slot * C.k2f_wcap, P.S2 + s0, (uint32_t)(s1 - s0) * 8, &bar[slot]);
  };
  if (t == 0) {
    ac::mbar_init(&bar[0], 1);
    ac::mbar_init(&bar[1], 1);
    ac::mbar_init(&bar[2], 1);
    ac::fence_mbar_init();
    if (!slow && nrec > 0) {
      ac::mbar_expect_tx(&bar[2], (uint32_t)nrec * 12);
      ac::bulk_g2s(recs, P.k2f_rec + (size_t)3 * r0, (uint32_t)nrec * 12, &bar[2]);
    }
  }
  pdl_wait();
  pdl_trigger();
  if (t == 0 && !slow) issue(bA, 0);
  __syncthreads();
  if (!slow && nrec > 0) ac::mbar_wait(&bar[2], 0);
  for (int b = bA; b < bB; ++b) {
    const int it = b - bA, slot = it & 1;
    if (t == 0 && !slow && b + 1 < bB) {
      ac::fence_proxy_async();
      issue(b + 1, slot ^ 1);
    }
    const float2* wv;
    if (!slow) {
      ac::mbar_wait(&bar[slot], (it >> 1) & 1);
      wv = win + slot * C.k2f_wcap + (int)(((size_t)b * img + w0) & 1);
    } else {
      wv = P.S2 + (size_t)b * img + w0;
    }
    float2* Rc = P.Rc + (size_t)b * C.ntpad + t0;
    constexpr int KU = 4;
    for (int q = t; q < ntg; q += KU * T) {
      uint32_t i01[KU], wa[KU], wb[KU];
#pragma unroll
      for (int k = 0; k < KU; ++k) {
        const int qq = q + k * T;
        const bool ok = qq < ntg;
        i01[k] = ok ? rp[3 * qq] : 0u;
        wa[k] = ok ? rp[3 * qq + 1] : 0u;
        wb[k] = ok ? rp[3 * qq + 2] : 0u;
      }
      float2 v0[KU], v1[KU];
#pragma unroll
      for (int k = 0; k < KU; ++k) {
        const bool ov = (i01[k] >> 16) == 0xFFFFu;
        v0[k] = ov ? make_float2(0.f, 0.f) : wv[i01[k] & 0xFFFFu];
        v1[k] = ov ? make_float2(0.f, 0.f) : wv[i01[k] >> 16];
      }
#pragma unroll
      for (int k = 0; k < KU; ++k) {
        const int qq = q + k * T;
        if (qq >= ntg) break;
        if ((i01[k] >> 16) == 0xFFFFu) continue;
        const float w0f = __uint_as_float(wa[k]), w1f = __uint_as_float(wb[k]);
        const float2 acc = __fmul2_rn(make_float2(w0f, w0f), v0[k]);
        Rc[qq] = __ffma2_rn(make_float2(w1f, w1f), v1[k], acc);
      }
    }
    for (int o = warp; o < nov; o += NW) {
      const int4 d = ovt[o];
      float2 acc = make_float2(0.f, 0.f);
      for (int e = lane; e < d.z; e += 32) {
        const int2 en = ove[d.y - e0 + e];
        const float w = __int_as_float(en.y);
        acc = __ffma2_rn(make_float2(w, w), wv[en.x], acc);
      }
#pragma unroll
      for (int off = 16; off > 0; off >>= 1) {
        acc.x += __shfl_xor_sync(0xffffffffu, acc.x, off);
        acc.y += __shfl_xor_sync(0xffffffffu, acc.y, off);
      }
      if (lane == 0) Rc[d.x] = acc;
    }
    __syncthreads();   // win[slot] consumed
  }
}

// ================================================================== K2Ta, streaming strips
// The transposed bilinear (D2^T, reading G12) as a streaming kernel: one CTA per (strip of
// columns, image).  The strip's union node window (one contiguous range of the adjoint S2)
// arrives by ONE bulk copy while every thread's target records (12 bytes, coalesced, L2-
// resident across images) are loaded into registers, so each CTA has ~60 KB in flight; then the
// fixed-order sums are stored contiguously to Rc.  Targets with more than two entries are
// summed by one warp each (lane-strided, fixed xor butterfly).  Deterministic, no atomics.
// One CTA per (strip, group of k2s_ipc images): the strip's records (KR per thread) and its
// first overflow targets (KO per warp, one entry per lane) are image-independent and loaded into
// registers ONCE; per image only the window arrives (bulk copy, double-buffered one image ahead)
// and the sums are stored, so the per-image critical path is one bulk copy.
#ifndef TAT_STRIP_SLOTS
#define TAT_STRIP_SLOTS 2   // measured at C3: 2 -> K2Ta 54.7 us, 3 -> 57.8, 4 -> 65.7
#endif
constexpr int kStripT = 256, kStripKR = (kStripTargets + kStripT - 1) / kStripT;   // 10
constexpr int kStripSlots = TAT_STRIP_SLOTS;   // node-window buffers (windows in flight + 1)
#ifndef TAT_STRIP_MINB
#define TAT_STRIP_MINB 3   // (4 CTAs per SM: 64 registers with spills, K2Ta 53.7 -> 67 us at C3)
#endif
__global__ void __launch_bounds__(kStripT, TAT_STRIP_MINB) k2t_strip(DevPlan P) {
  constexpr int T = kStripT, KR = kStripKR, NW = T / 32;
  extern __shared__ __align__(128) float2 win[];
  const Consts& C = P.C;
  const int t = threadIdx.x, lane = t & 31, warp = t >> 5;
  // heavy strips (origin region: long overflow lists read from global memory) first, one image
  // per CTA; then the others, k2s_ipc images per CTA
  const int ngrp = (C.batch + C.k2s_ipc - 1) / C.k2s_ipc;
  const int nhv = C.k2s_nheavy * C.batch;
  int s, bA, bB;
  if ((int)blockIdx.x < nhv) {
    s = blockIdx.x / C.batch;
    bA = C.b0 + blockIdx.x % C.batch;
    bB = bA + 1;
  } else {
    const int id = blockIdx.x - nhv;
    s = C.k2s_nheavy + id / ngrp;
    bA = C.b0 + (id % ngrp) * C.k2s_ipc;
    bB = min(bA + C.k2s_ipc, C.b0 + C.batch);
  }
  const int4 st = __ldg(&P.k2s_strip[s]);   // (window start, nodes, first target, targets)
  const int ntg = st.w;
  uint64_t* bar = reinterpret_cast<uint64_t*>(win + kStripSlots * C.k2s_wcap + C.k2s_ovcap / 8);
  const size_t img = (size_t)C.half * C.NL;
  const uint32_t* rp = P.k2s_rec + (size_t)3 * st.z;
  uint32_t i01[KR], wa[KR], wb[KR];
#pragma unroll
  for (int k = 0; k < KR; ++k) {
    const int qq = t + k * T;
    const bool ok = qq < ntg;
    i01[k] = ok ? __ldg(&rp[3 * qq]) : 0xFFFF0000u;   // (an absent record reads as "overflow")
    wa[k] = ok ? __ldg(&rp[3 * qq + 1]) : 0u;
    wb[k] = ok ? __ldg(&rp[3 * qq + 2]) : 0u;
  }
  // overflow lists (targets with > 2 entries): light strips stage descriptors and entries in
  // shared memory once (image-independent); heavy strips (origin region) read global memory
  const int2 ovr = __ldg(&P.k2s_ovr[s]);
  const int nov = ovr.y - ovr.x;
  const int e0 = nov > 0 ? __ldg(&P.k2s_ovt[ovr.x]).y : 0;
  const int ne = nov > 0 ? __ldg(&P.k2s_ovt[ovr.y - 1]).y + __ldg(&P.k2s_ovt[ovr.y - 1]).z - e0 : 0;
  if (s < C.k2s_nheavy) {
    // heavy strip (origin region: node window or overflow lists over the smem budgets), one
    // image: everything from global memory (L2); the long lists one warp per target, lane l
    // summing the entries l (mod 32) in order, a fixed xor butterfly combining the lanes
    pdl_wait();
    pdl_trigger();
    const float2* __restrict__ gw = P.S2 + (size_t)bA * img + st.x;
    float2* Rc = P.Rc + (size_t)bA * C.ntpad + st.z;
    for (int q = t; q < ntg; q += T) {
      const uint32_t a = __ldg(&rp[3 * q]);
      if ((a >> 16) == 0xFFFFu) continue;
      const float w0f = __uint_as_float(__ldg(&rp[3 * q + 1])), w1f = __uint_as_float(__ldg(&rp[3 * q + 2]));
      const float2 acc = __fmul2_rn(make_float2(w0f, w0f), gw[a & 0xFFFFu]);
      Rc[q] = __ffma2_rn(make_float2(w1f, w1f), gw[a >> 16], acc);
    }
    for (int o = ovr.x + warp; o < ovr.y; o += NW) {
      const int4 d = __ldg(&P.k2s_ovt[o]);
      float2 acc = make_float2(0.f, 0.f);
      for (int e = lane; e < d.z; e += 32) {
        const int2 en = __ldg(&P.k2s_ov[d.y + e]);
        const float w = __int_as_float(en.y);
        acc = __ffma2_rn(make_float2(w, w), gw[en.x], acc);
      }
#pragma unroll
      for (int off = 16; off > 0; off >>= 1) {
        acc.x += __shfl_xor_sync(0xffffffffu, acc.x, off);
        acc.y += __shfl_xor_sync(0xffffffffu, acc.y, off);
      }
      if (lane == 0) Rc[d.x] = acc;
    }
    return;
  }
  // light strip: overflow descriptors and entries staged in shared memory once
  int4* ovt_s = reinterpret_cast<int4*>(win + kStripSlots * C.k2s_wcap);
  int2* ove_s = reinterpret_cast<int2*>(ovt_s + nov);
  for (int i = t; i < nov; i += T) ovt_s[i] = __ldg(&P.k2s_ovt[ovr.x + i]);
  for (int i = t; i < ne; i += T) ove_s[i] = __ldg(&P.k2s_ov[e0 + i]);
  auto issue = [&](int b, int slot) {
    const size_t src = (size_t)b * img + st.x;
    const size_t s0 = src & ~(size_t)1, s1 = (src + st.y + 1) & ~(size_t)1;
    ac::mbar_expect_tx(&bar[slot], (uint32_t)(s1 - s0) * 8);
    ac::bulk_g2s(win + slot * C.k2s_wcap, P.S2 + s0, (uint32_t)(s1 - s0) * 8, &bar[slot]);
  };
  if (t == 0) {
    for (int q = 0; q < kStripSlots; ++q) ac::mbar_init(&bar[q], 1);
    ac::fence_mbar_init();
  }
  pdl_wait();
  pdl_trigger();
  if (t == 0)   // windows kStripSlots - 1 images ahead
    for (int q = 0; q < kStripSlots - 1 && bA + q < bB; ++q) issue(bA + q, q);
  __syncthreads();
  for (int b = bA; b < bB; ++b) {
    const int it = b - bA, slot = it % kStripSlots;
    if (t == 0 && b + kStripSlots - 1 < bB) {   // the slot consumed in the previous iteration
      ac::fence_proxy_async();
      issue(b + kStripSlots - 1, (it + kStripSlots - 1) % kStripSlots);
    }
    ac::mbar_wait(&bar[slot], (it / kStripSlots) & 1);
    const float2* wv = win + slot * C.k2s_wcap + (int)(((size_t)b * img + st.x) & 1);
    float2* Rc = P.Rc + (size_t)b * C.ntpad + st.z;
#pragma unroll
    for (int k = 0; k < KR; ++k) {
      if ((i01[k] >> 16) == 0xFFFFu) continue;    // absent, or more than two entries
      const float w0f = __uint_as_float(wa[k]), w1f = __uint_as_float(wb[k]);
      const float2 acc = __fmul2_rn(make_float2(w0f, w0f), wv[i01[k] & 0xFFFFu]);
      Rc[t + k * T] = __ffma2_rn(make_float2(w1f, w1f), wv[i01[k] >> 16], acc);
    }
    for (int q = t + KR * T; q < ntg; q += T) {   // strips with more than KR T targets
      const uint32_t a = __ldg(&rp[3 * q]);
      if ((a >> 16) == 0xFFFFu) continue;
      const float w0f = __uint_as_float(__ldg(&rp[3 * q + 1])), w1f = __uint_as_float(__ldg(&rp[3 * q + 2]));
      const float2 acc = __fmul2_rn(make_float2(w0f, w0f), wv[a & 0xFFFFu]);
      Rc[q] = __ffma2_rn(make_float2(w1f, w1f), wv[a >> 16], acc);
    }
    // targets with more than two entries (deterministic fixed-order sums): one thread per
    // target, its entries in order, all in smem
    for (int o = t; o < nov; o += T) {
      const int4 d = ovt_s[o];
      const int2* en = ove_s + (d.y - e0);
      float w = __int_as_float(en[0].y);
      float2 acc = __fmul2_rn(make_float2(w, w), wv[en[0].x]);
      for (int e = 1; e < d.z; ++e) {
        w = __int_as_float(en[e].y);
        acc = __ffma2_rn(make_float2(w, w), wv[en[e].x], acc);
      }
      Rc[d.x] = acc;
    }
    __syncthreads();   // win[slot] consumed
  }
}

size_t smem_k2t_strip(const Consts& C) {
  return (size_t)kStripSlots * C.k2s_wcap * 8 + C.k2s_ovcap + 8 * kStripSlots;
}

cudaError_t launch_k2t_strip(const DevPlan& P, cudaStream_t s) {
  const Consts& C = P.C;
  const dim3 grid(C.k2s_nheavy * C.batch + (C.k2s_n - C.k2s_nheavy) * ((C.batch + C.k2s_ipc - 1) / C.k2s_ipc));
  const cudaError_t e = launch_pdl(C.pdl, k2t_strip, grid, dim3(kStripT), smem_k2t_strip(C), s, P);
  return e != cudaSuccess ? e : cudaGetLastError();
}

size_t smem_k2t_sumf(const Consts& C) {
  return (size_t)C.k2f_rcap * 12 + (size_t)2 * C.k2f_wcap * 8 + 64;
}

cudaError_t launch_k2t_sumf(const DevPlan& P, cudaStream_t s) {
  const Consts& C = P.C;
  const dim3 grid(C.k2f_nslow * C.batch + (C.ncols - C.k2f_nslow) * ((C.batch + C.k2f_ipc - 1) / C.k2f_ipc));
  const cudaError_t e = launch_pdl(C.pdl, k2t_sumf, grid, dim3(kSumfT), smem_k2t_sumf(C), s, P);
  return e != cudaSuccess ? e : cudaGetLastError();
}

// ================================================================== K1 forward (row pairs)
// z = f_y + i f_{y+1}; Z[p] = sum_x z[x] W_N^{p (x - n/2)} (Alg. 1 steps 1-2, the zero-extended
// row DFT); S1[b][p][y] = (Z[p] + conj Z[-p]) / 2, S1[b][p][y+1] = (Z[p] - conj Z[-p]) / (2i)
// for p in [0, N/2].  One CTA (128 threads) per two row pairs (rows y0..y0+3), whose outputs
// are one contiguous range of the blocked S1 (s1b: 32 bytes per p), stored by the threads.
constexpr int kK1BoxP = 128;   // p extent of one K1T input chunk
#ifndef TAT_K1_PAD
#define TAT_K1_PAD 1           // K1 column buffers: padded rows (1) or XOR swizzle (0)
#endif
#ifndef TAT_K1T_SLOTS
#define TAT_K1T_SLOTS 8
#endif
constexpr int kK1TSlots = TAT_K1T_SLOTS;   // K1T: S~1 tiles in flight (TMA loads issued ahead)
constexpr int kK1TEpiBars = 2 * kK1TSlots + 2;   // K1T mbarriers (tiles, consumed, epilogue), 16-B multiple
#ifndef TAT_K1T_EMPTY
#define TAT_K1T_EMPTY 0        // K1T: per-slot consumed barriers instead of a CTA barrier per tile
                               // (measured: K1T 69.7 -> 70.3 us at C3, 93 -> 100 at C5)
#endif

template <int n, bool VAR>
__global__ void __launch_bounds__(ColGeo<n>::T, n >= 1024 ? 1 : 3) k1c_fwd(DevPlan P, const __grid_constant__ CUtensorMap tm,
                                                  const float* __restrict__ f) {
  using G = ColGeo<n, 8, TAT_K1_PAD>;
  extern __shared__ __align__(128) float2 sm[];
  const Consts& C = P.C;
  const int t = threadIdx.x, j = t % G::J, sg = t / G::J;
  const int b = C.b0 + blockIdx.y, y0 = 4 * blockIdx.x, N = C.N;
  float2* W0 = sm;
  float2* W1 = sm + G::WS;
  // the 4 input rows (2n float2)
  float2* stg = sm + 2 * G::WS;
  constexpr int STG = 2 * n;
  uint64_t* bar = reinterpret_cast<uint64_t*>(stg + STG);
  const float* rows = reinterpret_cast<const float*>(stg);
  float2 A[G::NRES][G::R];
  PowR<G::R, kFactPowK1> pw;
  col_twiddles<G>(P.tw_col, P.tw_n, n / 2, j, sg, A, pw);
  pdl_wait();
  pdl_trigger();
  if (t == 0) {   // the 4 rows y0..y0+3 are one contiguous 16n-byte range of f
    ac::mbar_init(bar, 1);
    ac::fence_mbar_init();
    ac::mbar_expect_tx(bar, 16 * n);
    ac::bulk_g2s(stg, f + ((size_t)b * n + y0) * n, 16 * n, bar);
  }
  __syncthreads();
  ac::mbar_wait(bar, 0);
#pragma unroll 1
  for (int pr = 0; pr < 2; ++pr) {
    float2 x[G::R];
#pragma unroll
    for (int r = 0; r < G::R; ++r)
      x[r] = make_float2(rows[(2 * pr) * n + j + G::J * r], rows[(2 * pr + 1) * n + j + G::J * r]);
    if (VAR && P.deapod) {   // reading G26: f / K on the nodes, K separable
      const float w0 = P.deapod[y0 + 2 * pr], w1 = P.deapod[y0 + 2 * pr + 1];
#pragma unroll
      for (int r = 0; r < G::R; ++r) {
        const float cw = P.deapod[j + G::J * r];
        x[r].x *= cw * w0;
        x[r].y *= cw * w1;
      }
    }
    stage_a_fwd<G>(x, A, pw, pr ? W1 : W0, j, sg);
  }
  __syncthreads();   // (also: every thread is done with the rows before stg is reused)
  stage_b<G, -1>(W0, t);
  stage_b<G, -1>(W1, t);
  __syncthreads();
  // S1 blocked (s1b): the quad of rows y0..y0+3 is one contiguous run of ncols x 32 bytes, stored
  // by consecutive threads (consecutive p) with 16-byte stores.  (Measured at C3: K1 52 -> 43.5 us
  // against the column-major S1 written by TMA tile stores through a 2-slot staging ring.)
  float4* dst = reinterpret_cast<float4*>(P.S1 + s1b(C, b, y0, 0));
  for (int p = t; p < C.ncols; p += G::T) {
    const int ia = G::fq(p), im = G::fq((N - p) & (N - 1));
    const float2 za = W0[ia], zm = W0[im], zb = W1[ia], zn = W1[im];
    dst[2 * p] = make_float4(0.5f * (za.x + zm.x), 0.5f * (za.y - zm.y), 0.5f * (za.y + zm.y),
                             -0.5f * (za.x - zm.x));
    dst[2 * p + 1] = make_float4(0.5f * (zb.x + zn.x), 0.5f * (zb.y - zn.y), 0.5f * (zb.y + zn.y),
                                 -0.5f * (zb.x - zn.x));
  }
}

// ================================================================== K1T (transpose of K1)
// Z[p] = C_y[p] + i C_{y+1}[p] and Z[-p] = conj C_y[p] + i conj C_{y+1}[p] (Hermitian
// completion; C[0], C[N/2] -> 2 Re), conjugate transform, f~_y = Re z~, f~_{y+1} = Im z~.
// Two row pairs per CTA; the [128 p][4 y] tiles of S~1 (column-major) arrive by TMA tensor loads,
// kK1TSlots in flight.
template <int n, bool VAR>
__global__ void __launch_bounds__(ColGeo<n>::T, n >= 1024 ? 1 : 3) k1c_adj(DevPlan P, const __grid_constant__ CUtensorMap tm,
                                                  float* __restrict__ fout) {
  using G = ColGeo<n, 8, 0>;
  extern __shared__ __align__(128) float2 sm[];
  const Consts& C = P.C;
  const int t = threadIdx.x, j = t % G::J, sg = t / G::J;
  const int b = C.b0 + blockIdx.y, y0 = 4 * blockIdx.x, N = C.N;
  float2* W0 = sm;
  float2* W1 = sm + G::WS;
  float2* stg = sm + 2 * G::WS;
  uint64_t* bar = reinterpret_cast<uint64_t*>(stg + kK1TSlots * kK1BoxP * 4);
  float2 A[G::NRES][G::R];
  PowR<G::R, kFactPow> pw;
  col_twiddles<G>(P.tw_col, P.tw_n, n / 2, j, sg, A, pw);
  pdl_wait();
  pdl_trigger();
  const int nch = (C.ncols + kK1BoxP - 1) / kK1BoxP;
  uint64_t* ebar = bar + kK1TSlots;   // per-slot "consumed" barriers (arrival count T)
  uint64_t* pbar = bar + 2 * kK1TSlots;   // the staged epilogue inputs
  // fused update epilogue (tat_adjoint_step): the CTA's 4 rows of f (and of the roi mask) are
  // brought in by bulk copies at the start instead of being loaded at the store
  // (measured at C3: K1T with the update 111 -> 65 us; the NNLS loop 44.6 -> 41.1 ms)
  float* epf = reinterpret_cast<float*>(bar + kK1TEpiBars);
  float* epr = epf + 4 * n;
  const bool stage_epi = P.epi_update != 0;
  // S~1 is column-major [B][ncols][n] (written by K2Tb with coalesced column stores): chunk c is the
  // [128 p][4 y] TMA tile at (y0, 128 c, b), rows beyond ncols zero-filled
  auto chunk = [&](int c, int slot) {   // thread 0
    ac::mbar_expect_tx(&bar[slot], kK1BoxP * 32);
    ac::tma_load_3d(stg + slot * kK1BoxP * 4, &tm, y0, c * kK1BoxP, b, &bar[slot]);
  };
  if (t == 0) {
    for (int q = 0; q < kK1TSlots; ++q) ac::mbar_init(&bar[q], 1);
    if (TAT_K1T_EMPTY)
      for (int q = 0; q < kK1TSlots; ++q) ac::mbar_init(&ebar[q], G::T);
    ac::mbar_init(pbar, 1);
    ac::fence_mbar_init();
    if (stage_epi) {
      ac::mbar_expect_tx(pbar, (P.epi_roi ? 32 : 16) * n);
      ac::bulk_g2s(epf, fout + ((size_t)b * n + y0) * n, 16 * n, pbar);
      if (P.epi_roi) ac::bulk_g2s(epr, P.epi_roi + (size_t)y0 * n, 16 * n, pbar);
    }
    for (int c = 0; c < kK1TSlots && c < nch; ++c) chunk(c, c);
  }
  __syncthreads();
  for (int c = 0; c < nch; ++c) {
    const int slot = c % kK1TSlots;
    ac::mbar_wait(&bar[slot], (c / kK1TSlots) & 1);
    const float4* tile = reinterpret_cast<const float4*>(stg + slot * kK1BoxP * 4);
    const int p = c * kK1BoxP + t;
    if (t < kK1BoxP && p < C.ncols) {
      const float4 a = tile[2 * t], cc = tile[2 * t + 1];   // (C_y, C_{y+1}), (C_{y+2}, C_{y+3})
      const int ia = G::fq(p);
      if (p == 0 || p == N / 2) {
        W0[ia] = make_float2(2.f * a.x, 2.f * a.z);
        W1[ia] = make_float2(2.f * cc.x, 2.f * cc.z);
      } else {
        const int im = G::fq(N - p);
        W0[ia] = make_float2(a.x - a.w, a.y + a.z);
        W0[im] = make_float2(a.x + a.w, -a.y + a.z);
        W1[ia] = make_float2(cc.x - cc.w, cc.y + cc.z);
        W1[im] = make_float2(cc.x + cc.w, -cc.y + cc.z);
      }
    }
#if TAT_K1T_EMPTY
    // no CTA barrier per tile: each thread marks the slot consumed; thread 0 refills it once
    // every thread has (the other warps run ahead on the tiles already in flight)
    ac::mbar_arrive(&ebar[slot]);
    if (t == 0 && c + kK1TSlots < nch) {
      ac::mbar_wait(&ebar[slot], (c / kK1TSlots) & 1);
      ac::fence_proxy_async();
      chunk(c + kK1TSlots, slot);
    }
  }
  __syncthreads();   // W0 / W1 complete
#else
    __syncthreads();   // tile consumed
    if (t == 0 && c + kK1TSlots < nch) {
      ac::fence_proxy_async();
      chunk(c + kK1TSlots, slot);
    }
  }
#endif
  stage_b<G, 1>(W0, t);
  stage_b<G, 1>(W1, t);
  __syncthreads();
  const bool active = !P.epi_active || __ldg(&P.epi_active[b]);
  if (stage_epi) ac::mbar_wait(pbar, 0);
#pragma unroll 1
  for (int pr = 0; pr < 2; ++pr) {
    float2* W = pr ? W1 : W0;
    float2 acc[G::R];
    stage_a_adj<G>(W, A, pw, j, sg, acc);
    residue_reduce<G>(W, acc, j, sg);
    const size_t o = ((size_t)b * n + y0 + 2 * pr) * n;
    const int oxy = (y0 + 2 * pr) * n;
    for (int xx = t; xx < n; xx += G::T) {
      const float2 z = residue_sum<G>(W, xx);
      if (stage_epi) {
        const int r0 = 2 * pr * n + xx, r1 = r0 + n;
        epi_adj_store_pre<VAR>(P, fout, o + xx, oxy + xx, z.x, epf[r0], P.epi_roi ? epr[r0] : 1.f, active);
        epi_adj_store_pre<VAR>(P, fout, o + n + xx, oxy + n + xx, z.y, epf[r1], P.epi_roi ? epr[r1] : 1.f, active);
      } else {
        epi_adj_store<VAR>(P, fout, o + xx, oxy + xx, z.x);
        epi_adj_store<VAR>(P, fout, o + n + xx, oxy + n + xx, z.y);
      }
    }
  }
}

// ================================================================== K4 / K4T (DCT-I)
// lambda <-> t cosine transforms (Alg. 1 step 5, E:inverse_cos_tr P:L475-478; Alg. 2 step 3):
//   out[u] = (X(u) + X(-u)) / 2,  X(u) = sum_i c_i W_2M^{i u},  2M = 12 n,
// with the inputs decimated by 3 (i = 3 i' + e, i' < n): X(u) = sum_e W_2M^{e u} Y_e(u mod 4n),
// Y_e = the 4n-point DFT of c_{3 i' + e} -- three two-stage transforms (L = 4) per row, one
// per 64-thread group.  The single input i = 3n (j = J, forward only) adds h_J cos(pi u / 2).
//   K4  (ADJ = false): c_j = H[k][j] (S3 row, j <= J), out for u = m + 1, m < n_t -> S4 row
//   K4T (ADJ = true) : c_i = G~[k][i - 1] (S4 row, 1 <= i <= n_t), out for u = j <= J, then
//                      x (-i)^k omega m'[k][j] -> S3 row
// Persistent CTAs loop over the rows (b, k); the next row is prefetched into shared memory by a
// 1-D bulk copy while the current one is transformed, and the per-thread twiddles are loaded once.
template <int n, bool ADJ>
#ifndef TAT_K4_MINB
#define TAT_K4_MINB 2
#endif
#ifndef TAT_K4_TWS
#define TAT_K4_TWS 0   // output twiddles staged in smem per CTA (1) or read from L1 per output
                       // (0; measured at C3: K4 68.3 -> 66.2 us, K4T 77.9 -> 74.8 us)
#endif
#ifndef TAT_K4_U
#define TAT_K4_U 0     // K4/K4T outputs per thread per pass (twiddle loads issued together);
                       // 0: 4 for K4, 8 for K4T (measured with W1REC: K4T 69.7 -> 68.0 us)
#endif
#ifndef TAT_K4_W2SQ
#define TAT_K4_W2SQ 1  // W^{2u} as the square of W^u instead of a table load (measured at C3:
                       // K4 61.7 -> 59.7 us, K4T 72.0 -> 69.7)
#endif
#ifndef TAT_K4_W1REC
#define TAT_K4_W1REC -1 // W^u of a thread's later outputs by multiplication with W^{blockDim}
                        // (-1: K4T only; for K4 it measured 59.7 -> 62.0 us)
#endif
#ifndef TAT_K4_ALDG
#define TAT_K4_ALDG 0  // stage-A pre-twiddles from L1 at each use (1) or in registers (0)
#endif
__global__ void __launch_bounds__(3 * ColGeo<n, 4>::T, n >= 1024 ? 1 : TAT_K4_MINB) k4c_dct(DevPlan P) {
  using G = ColGeo<n, 4>;
  constexpr int N4 = 4 * n;
  extern __shared__ __align__(128) float2 sm[];
  const Consts& C = P.C;
  const int t = threadIdx.x, e = t / G::T, tl = t % G::T, j = tl % G::J, sg = tl / G::J;
  const int M2 = 2 * C.M, NL = C.NL, n_t = C.n_t;
  const int cnt = ADJ ? n_t : NL;                 // input entries per row
  const int IB = (cnt + 3) & ~1;                  // slot size (entries; alignment slack)
  const int rows = C.Kp * C.batch;
  const float2* in_all = ADJ ? P.S4 : P.S3;
  float2* W = sm + e * G::WS;
  float2* ibuf = sm + 3 * G::WS;
  const int U = ADJ ? NL : n_t + 1;               // output twiddle index range u in [0, U)
  float4* tws = reinterpret_cast<float4*>(ibuf + 2 * IB);   // (W^u, W^{2u}), W = W_2M
  uint64_t* bar = reinterpret_cast<uint64_t*>(tws + (TAT_K4_TWS ? U : 0));
  const long rbase = (long)C.b0 * C.Kp;   // global row of local row 0
  auto issue = [&](int r, int slot) {   // thread 0: row r -> ibuf[slot] (16-B aligned range)
    const long s0 = ((rbase + r) * cnt) & ~1L, s1 = ((rbase + r) * cnt + cnt + 1) & ~1L;
    ac::mbar_expect_tx(&bar[slot], (uint32_t)(s1 - s0) * 8);
    ac::bulk_g2s(ibuf + slot * IB, in_all + s0, (uint32_t)(s1 - s0) * 8, &bar[slot]);
  };
#if TAT_K4_ALDG
  // pre-twiddles read from the (L1-resident, 16 KB) table at each use instead of 2 NRES R
  // registers per thread: the register budget of 3 CTAs per SM
  PowR<G::R, kFactPow> pw;
  pw.init(__ldg(&P.tw_n[j & (n - 1)]));
#else
  float2 A[G::NRES][G::R];
  PowR<G::R, kFactPow || n >= 1024> pw;   // (full powers spill at n = 1024)
  col_twiddles<G>(P.tw_dct4, P.tw_n, 0, j, sg, A, pw);
#endif
  if (TAT_K4_TWS)
    for (int u = t; u < U; u += blockDim.x) {   // output twiddles, once per CTA
      const int u2 = 2 * u >= M2 ? 2 * u - M2 : 2 * u;
      const float2 a = __ldg(&P.tw_dct[u]), c = __ldg(&P.tw_dct[u2]);
      tws[u] = make_float4(a.x, a.y, c.x, c.y);
    }
  pdl_wait();
  pdl_trigger();
  if (t == 0) {
    ac::mbar_init(&bar[0], 1);
    ac::mbar_init(&bar[1], 1);
    ac::fence_mbar_init();
    if ((int)blockIdx.x < rows) issue(blockIdx.x, 0);
  }
  __syncthreads();
  int it = 0;
  for (int row = blockIdx.x; row < rows; row += gridDim.x, ++it) {
    const int slot = it & 1;
    if (t == 0 && row + (int)gridDim.x < rows) {
      ac::fence_proxy_async();
      issue(row + gridDim.x, slot ^ 1);
    }
    const int k = row % C.Kp;
    ac::mbar_wait(&bar[slot], (it >> 1) & 1);
    const float2* in = ibuf + slot * IB + (int)(((rbase + row) * cnt) & 1L);
    float2 x[G::R];
#pragma unroll
    for (int r = 0; r < G::R; ++r) {
      const int i = 3 * (j + G::J * r) + e, src = ADJ ? i - 1 : i;
      x[r] = (src >= 0 && src < cnt) ? in[src] : make_float2(0.f, 0.f);
    }
#if TAT_K4_ALDG
#pragma unroll
    for (int i = 0; i < G::NRES; ++i) {
      const int s = sg + G::NG * i;
      float2 v[G::R];
#pragma unroll
      for (int r = 0; r < G::R; ++r) v[r] = cmul(x[r], __ldg(&P.tw_dct4[s * n + j + G::J * r]));
      ce::dftr<G::R, -1>(v);
#pragma unroll
      for (int k1 = 1; k1 < G::R; ++k1) v[k1] = pw.mul(v[k1], k1);
#pragma unroll
      for (int k1 = 0; k1 < G::R; ++k1) W[G::widx(s + G::L * k1, j)] = v[k1];
    }
#else
    stage_a_fwd<G>(x, A, pw, W, j, sg);
#endif
    // stage B of group e reads only group e's buffer: a named barrier of its G::T threads
    asm volatile("bar.sync %0, %1;" ::"r"(1 + e), "r"(G::T) : "memory");
    stage_b<G, -1>(W, tl);
    __syncthreads();
    // S(u) = X(u) + X(-u) = sum_e [W^{eu} Y_e(u) + conj(W^{eu}) Y_e(-u)], W = W_2M, 0 <= u < 4n;
    // outputs in groups of 4 per thread with all twiddle loads issued first
    // D(u) = X(u) - X(-u) for the sine transform of the inverse (C.dct_sine, ADJ only):
    // sum_i c_i sin(theta i u) = i D(u) / 2
    const bool sine = ADJ && C.dct_sine;
    auto Ssum = [&](int u, float2 w1, float2 w2) -> float2 {
      const int vp = G::fq(u & (N4 - 1)), vm = G::fq((N4 - u) & (N4 - 1));
      if (sine) {
        const float2 a = csub(sm[vp], sm[vm]);
        const float2 c1 = csub(cmul(sm[G::WS + vp], w1), cmulc(sm[G::WS + vm], w1));
        const float2 c2 = csub(cmul(sm[2 * G::WS + vp], w2), cmulc(sm[2 * G::WS + vm], w2));
        const float2 dd = ce::cadd(a, ce::cadd(c1, c2));
        return make_float2(-dd.y, dd.x);   // i D
      }
      const float2 a = ce::cadd(sm[vp], sm[vm]);
      const float2 c1 = ce::cadd(cmul(sm[G::WS + vp], w1), cmulc(sm[G::WS + vm], w1));
      const float2 c2 = ce::cadd(cmul(sm[2 * G::WS + vp], w2), cmulc(sm[2 * G::WS + vm], w2));
      return ce::cadd(a, ce::cadd(c1, c2));
    };
    constexpr int U4 = TAT_K4_U > 0 ? TAT_K4_U : (ADJ ? 8 : 4);
    constexpr bool W1REC = TAT_K4_W1REC < 0 ? ADJ : (TAT_K4_W1REC != 0);
    const int nout = ADJ ? NL : n_t;
    const float2 hJ = (!ADJ && NL == 3 * n + 1) ? in[3 * n] : make_float2(0.f, 0.f);
    const float om = (float)C.omega;
    float2* out = ADJ ? P.S3 + (size_t)(rbase + row) * NL : P.S4 + (size_t)(rbase + row) * n_t;
    const float2 wstep = W1REC ? __ldg(&P.tw_dct[blockDim.x]) : make_float2(1.f, 0.f);
    for (int o0 = t; o0 < nout; o0 += U4 * (int)blockDim.x) {
      float2 w1[U4], w2[U4];
      float ml[U4];
#pragma unroll
      for (int q = 0; q < U4; ++q) {
        const int o = o0 + q * blockDim.x;
        const int u = ADJ ? o : o + 1;
        if (TAT_K4_TWS) {
          const float4 tw = o < nout ? tws[u] : make_float4(0.f, 0.f, 0.f, 0.f);
          w1[q] = make_float2(tw.x, tw.y);
          w2[q] = make_float2(tw.z, tw.w);
        } else {
          const int uu = o < nout ? u : 0, u2 = 2 * uu >= M2 ? 2 * uu - M2 : 2 * uu;
          if (W1REC && q > 0) w1[q] = cmul(w1[q - 1], wstep);   // W^{u + q T}
          else w1[q] = __ldg(&P.tw_dct[uu]);
          if (TAT_K4_W2SQ) w2[q] = cmul(w1[q], w1[q]);   // W^{2u} = (W^u)^2 (one rounding more)
          else w2[q] = __ldg(&P.tw_dct[u2]);
        }
        ml[q] = (ADJ && o < nout) ? __ldg(&P.mult[(size_t)k * NL + o]) : 0.f;
      }
#pragma unroll
      for (int q = 0; q < U4; ++q) {
        const int o = o0 + q * blockDim.x;
        if (o >= nout) break;
        const int u = ADJ ? o : o + 1;
        const float2 y = fe::cscale(Ssum(u, w1[q], w2[q]), 0.5f);
        if (!ADJ) {
          float2 g = y;
          if ((u & 3) == 0) g = ce::cadd(g, hJ);
          else if ((u & 3) == 2) g = csub(g, hJ);
          out[o] = g;
        } else {
          const float2 z = fe::cscale(y, om * ml[q]);
          float2 r;
          switch ((-k) & 3) {   // (-i)^k
            case 0: r = z; break;
            case 1: r = make_float2(-z.y, z.x); break;
            case 2: r = make_float2(-z.x, -z.y); break;
            default: r = make_float2(z.y, -z.x); break;
          }
          out[o] = r;
        }
      }
    }
    __syncthreads();   // W and ibuf[slot] free
  }
}

// ================================================================== dispatch
int col_R(int n) { return n >= 1024 ? 32 : 16; }
static int col_T(int n, int L) { return col_R(n) * L; }

bool dct4_ok(const Consts& C) {
  return (C.n == 256 || C.n == 512 || C.n == 1024) && 2L * C.M == 12L * C.n && C.J <= 3 * C.n &&
         C.n_t <= 3 * C.n - 1;
}
size_t smem_k4c(const Consts& C) {
  const int cnt = std::max(C.NL, C.n_t);
  const int R4 = col_R(C.n), J4 = C.n / R4;
  return (size_t)3 * (R4 * 4) * (J4 + 1) * 8 + (size_t)2 * ((cnt + 3) & ~1) * 8 +
         (size_t)std::max(C.NL, C.n_t + 1) * 16 * TAT_K4_TWS + 64;
}

cudaError_t launch_k4c(const DevPlan& P, bool adj, cudaStream_t s) {
  const Consts& C = P.C;
  cudaError_t e = cudaSuccess;
  const int rows = C.Kp * C.batch;
  const dim3 grid(std::min(rows, (C.n >= 1024 ? 1 : TAT_K4_MINB) * 148));
  const dim3 blk(3 * col_T(C.n, 4));
  const size_t sm = smem_k4c(C);
  if (C.n == 1024) {
    if (adj) e = launch_pdl(C.pdl, k4c_dct<1024, true>, grid, blk, sm, s, P);
    else e = launch_pdl(C.pdl, k4c_dct<1024, false>, grid, blk, sm, s, P);
  } else if (C.n == 512) {
    if (adj) e = launch_pdl(C.pdl, k4c_dct<512, true>, grid, blk, sm, s, P);
    else e = launch_pdl(C.pdl, k4c_dct<512, false>, grid, blk, sm, s, P);
  } else {
    if (adj) e = launch_pdl(C.pdl, k4c_dct<256, true>, grid, blk, sm, s, P);
    else e = launch_pdl(C.pdl, k4c_dct<256, false>, grid, blk, sm, s, P);
  }
  return e != cudaSuccess ? e : cudaGetLastError();
}

bool col_ok(const Consts& C) { return C.Lres == 8 && (C.n == 256 || C.n == 512 || C.n == 1024); }

size_t smem_k2c_fwd(const Consts& C) {
  const int Q0 = col_R(C.n) * 8, J = C.n / col_R(C.n);
  return (size_t)k2_bufs(C.n) * Q0 * (J + 1) * 8 + (size_t)2 * C.n * 8 + 64;
}
size_t smem_k2c_adj(const Consts& C) {
  const int Q0 = col_R(C.n) * 8, J = C.n / col_R(C.n);
  return (size_t)Q0 * (J + 1) * 8 + (size_t)2 * C.k2c_rbuf * 8 + 64;
}

size_t smem_k2c_adjf(const Consts& C) {
  const int Q0 = col_R(C.n) * 8, J = C.n / col_R(C.n);
  return (size_t)Q0 * (J + 1) * 8 + (size_t)C.k2f_rcap * 12 + (size_t)2 * C.k2f_wcap * 8 + 64;
}

size_t smem_k1c(const Consts& C) {
  return (size_t)2 * (col_R(C.n) * 8) * (C.n / col_R(C.n) + TAT_K1_PAD) * 8 + (size_t)2 * C.n * 8 + 64;
}
size_t smem_k1c_adj(const Consts& C, bool epi) {
  return (size_t)2 * 8 * C.n * 8 + (size_t)kK1TSlots * kK1BoxP * 32 + 8 * kK1TEpiBars + (epi ? (size_t)32 * C.n : 0);
}

template <int n>
static cudaError_t cfg_col() {
  cudaError_t e = cudaSuccess;
  const int lim = 227 * 1024;
#define SETC(k) if (e == cudaSuccess) e = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, lim);
  SETC((k2c_fwd<n>));
  SETC((k2c_adj<n, false>));
  SETC((k2c_adj<n, true>));
  SETC((k2c_adjf<n>));
  SETC(k2t_sumf);
  SETC(k2t_strip);
  SETC((k1c_fwd<n, false>));
  SETC((k1c_adj<n, false>));
  SETC((k1c_fwd<n, true>));
  SETC((k1c_adj<n, true>));
  SETC((k4c_dct<n, false>));
  SETC((k4c_dct<n, true>));
#undef SETC
  return e;
}

cudaError_t configure_col_kernels(const Consts& C) {
  if (!col_ok(C) && !dct4_ok(C)) return cudaSuccess;
  return C.n == 1024 ? cfg_col<1024>() : (C.n == 512 ? cfg_col<512>() : cfg_col<256>());
}

cudaError_t launch_k2c_fwd(const DevPlan& P, const CUtensorMap& tm, cudaStream_t s) {
  const Consts& C = P.C;
  cudaError_t e = cudaSuccess;
  const dim3 grid((C.ncols + C.col_strip - 1) / C.col_strip, C.batch);
  const dim3 blk(col_T(C.n, 8));
  if (C.n == 1024) e = launch_pdl(C.pdl, k2c_fwd<1024>, grid, blk, smem_k2c_fwd(C), s, P, tm);
  else if (C.n == 512) e = launch_pdl(C.pdl, k2c_fwd<512>, grid, blk, smem_k2c_fwd(C), s, P, tm);
  else e = launch_pdl(C.pdl, k2c_fwd<256>, grid, blk, smem_k2c_fwd(C), s, P, tm);
  return e != cudaSuccess ? e : cudaGetLastError();
}

cudaError_t launch_k2c_adj(const DevPlan& P, cudaStream_t s) {
  const Consts& C = P.C;
  cudaError_t e = cudaSuccess;
  const dim3 grid((C.ncols + C.col_strip_adj - 1) / C.col_strip_adj, C.batch);
  const dim3 blk(col_T(C.n, 8));
  const bool ch = P.k2c_chord != nullptr;
  if (C.n == 1024) e = ch ? launch_pdl(C.pdl, k2c_adj<1024, true>, grid, blk, smem_k2c_adj(C), s, P)
                          : launch_pdl(C.pdl, k2c_adj<1024, false>, grid, blk, smem_k2c_adj(C), s, P);
  else if (C.n == 512) e = ch ? launch_pdl(C.pdl, k2c_adj<512, true>, grid, blk, smem_k2c_adj(C), s, P)
                              : launch_pdl(C.pdl, k2c_adj<512, false>, grid, blk, smem_k2c_adj(C), s, P);
  else e = ch ? launch_pdl(C.pdl, k2c_adj<256, true>, grid, blk, smem_k2c_adj(C), s, P)
              : launch_pdl(C.pdl, k2c_adj<256, false>, grid, blk, smem_k2c_adj(C), s, P);
  return e != cudaSuccess ? e : cudaGetLastError();
}

cudaError_t launch_k2c_adjf(const DevPlan& P, cudaStream_t s) {
  const Consts& C = P.C;
  cudaError_t e = cudaSuccess;
  const dim3 grid(C.k2f_nslow * C.batch + (C.ncols - C.k2f_nslow) * ((C.batch + C.k2f_ipc - 1) / C.k2f_ipc));
  const dim3 blk(col_T(C.n, 8));
  const size_t sm = smem_k2c_adjf(C);
  if (C.n == 1024) e = launch_pdl(C.pdl, k2c_adjf<1024>, grid, blk, sm, s, P);
  else if (C.n == 512) e = launch_pdl(C.pdl, k2c_adjf<512>, grid, blk, sm, s, P);
  else e = launch_pdl(C.pdl, k2c_adjf<256>, grid, blk, sm, s, P);
  return e != cudaSuccess ? e : cudaGetLastError();
}

template <int n>
static cudaError_t launch_k1c_n(const DevPlan& P, const CUtensorMap& tm, const float* f, float* fo, cudaStream_t s) {
  const Consts& C = P.C;
  const dim3 grid(C.n / 4, C.batch);
  const dim3 blk(col_T(C.n, 8));
  if (f) {   // forward: only the G26 input scaling is a K1 variant
    if (P.deapod) return launch_pdl(C.pdl, k1c_fwd<n, true>, grid, blk, smem_k1c(C), s, P, tm, f);
    return launch_pdl(C.pdl, k1c_fwd<n, false>, grid, blk, smem_k1c(C), s, P, tm, f);
  }
  if (P.deapod || P.lowk_add) return launch_pdl(C.pdl, k1c_adj<n, true>, grid, blk, smem_k1c_adj(C, P.epi_update != 0), s, P, tm, fo);
  return launch_pdl(C.pdl, k1c_adj<n, false>, grid, blk, smem_k1c_adj(C, P.epi_update != 0), s, P, tm, fo);
}

cudaError_t launch_k1c_fwd(const DevPlan& P, const CUtensorMap& tm, const float* f, cudaStream_t s) {
  const int n = P.C.n;
  const cudaError_t e = n == 1024 ? launch_k1c_n<1024>(P, tm, f, nullptr, s)
                        : n == 512 ? launch_k1c_n<512>(P, tm, f, nullptr, s)
                                   : launch_k1c_n<256>(P, tm, f, nullptr, s);
  return e != cudaSuccess ? e : cudaGetLastError();
}

cudaError_t launch_k1c_adj(const DevPlan& P, const CUtensorMap& tm, float* f, cudaStream_t s) {
  const int n = P.C.n;
  const cudaError_t e = n == 1024 ? launch_k1c_n<1024>(P, tm, nullptr, f, s)
                        : n == 512 ? launch_k1c_n<512>(P, tm, nullptr, f, s)
                                   : launch_k1c_n<256>(P, tm, nullptr, f, s);
  return e != cudaSuccess ? e : cudaGetLastError();
}

}  // namespace tat
