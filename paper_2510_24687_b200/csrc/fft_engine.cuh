// Register/shared-memory FFT engine for the L residue transforms of the zero-padded 2-D DFT.
//
// The N = L n point DFT of a column with n non-zero samples (Alg. 1 step 2, the zero-extended
// 2-D FFT of PAPER.md L545-548) is split into L residue classes q = L a + s:
//   F[L a + s] = sum_{y''} (x[y''] W_N^{s y''}) W_n^{a y''},  y'' in [-n/2, n/2),
// i.e. a pre-twiddle and an n-point FFT per residue.  Each thread owns one radix-8 butterfly
// (8 complex points) of RPT residues; passes are Stockham (natural-order output) with radix
// 8, 8, ..., and a final radix 2 or 4 (n = 8^a * {1, 2, 4}).  Data moves between passes
// through shared memory with an XOR swizzle that makes every pass's 8-byte accesses
// bank-conflict free.  Complex arithmetic maps to FADD2 / FMUL2 / FFMA2 (two fp32 lanes
// per instruction: {re, im}).
#pragma once
#include <cuda_runtime.h>

namespace tat {
namespace fe {

// ------------------------------------------------------------------ packed complex ops
__device__ __forceinline__ float2 cadd(float2 a, float2 b) { return __fadd2_rn(a, b); }
__device__ __forceinline__ float2 csub(float2 a, float2 b) {
  return __fadd2_rn(a, make_float2(-b.x, -b.y));
}
// a * w  (FMUL2 + FFMA2)
__device__ __forceinline__ float2 cmul(float2 a, float2 w) {
  float2 t = __fmul2_rn(w, make_float2(a.x, a.x));
  return __ffma2_rn(make_float2(-w.y, w.x), make_float2(a.y, a.y), t);
}
// a * conj(w)
__device__ __forceinline__ float2 cmulc(float2 a, float2 w) {
  float2 t = __fmul2_rn(make_float2(w.x, -w.y), make_float2(a.x, a.x));
  return __ffma2_rn(make_float2(w.y, w.x), make_float2(a.y, a.y), t);
}
__device__ __forceinline__ float2 cscale(float2 a, float s) { return __fmul2_rn(a, make_float2(s, s)); }
// a + S i b  (S = +1 or -1)
template <int S>
__device__ __forceinline__ float2 add_ib(float2 a, float2 b) {
  return (S > 0) ? __fadd2_rn(a, make_float2(-b.y, b.x)) : __fadd2_rn(a, make_float2(b.y, -b.x));
}

// ------------------------------------------------------------------ small DFTs (in place)
// X[k] = sum_r a[r] e^{S 2 pi i r k / R}, natural order.
template <int S>
__device__ __forceinline__ void dft2(float2* a) {
  float2 t = cadd(a[0], a[1]);
  a[1] = csub(a[0], a[1]);
  a[0] = t;
}
template <int S>
__device__ __forceinline__ void dft4(float2* a) {
  float2 s02 = cadd(a[0], a[2]), d02 = csub(a[0], a[2]);
  float2 s13 = cadd(a[1], a[3]), d13 = csub(a[1], a[3]);
  a[0] = cadd(s02, s13);
  a[2] = csub(s02, s13);
  a[1] = add_ib<S>(d02, d13);
  a[3] = add_ib<-S>(d02, d13);
}
template <int S>
__device__ __forceinline__ void dft8(float2* a) {
  const float h = 0.70710678118654752440f;
  float2 t0 = cadd(a[0], a[4]), u0 = csub(a[0], a[4]);
  float2 t1 = cadd(a[1], a[5]), u1 = csub(a[1], a[5]);
  float2 t2 = cadd(a[2], a[6]), u2 = csub(a[2], a[6]);
  float2 t3 = cadd(a[3], a[7]), u3 = csub(a[3], a[7]);
  // odd half twiddles: u1 (1 + S i)/sqrt2, u2 (S i), u3 (-1 + S i)/sqrt2 = S i (1 + S i)/sqrt2 u3
  float2 v1 = cscale(add_ib<S>(u1, u1), h);
  float2 v3 = cscale(add_ib<S>(u3, u3), h);
  // even: DFT4(t0, t1, t2, t3)
  float2 s02 = cadd(t0, t2), d02 = csub(t0, t2);
  float2 s13 = cadd(t1, t3), d13 = csub(t1, t3);
  a[0] = cadd(s02, s13);
  a[4] = csub(s02, s13);
  a[2] = add_ib<S>(d02, d13);
  a[6] = add_ib<-S>(d02, d13);
  // odd: DFT4(u0, v1, S i u2, S i v3)
  float2 os02 = add_ib<S>(u0, u2), od02 = add_ib<-S>(u0, u2);
  float2 os13 = add_ib<S>(v1, v3), od13 = add_ib<-S>(v1, v3);
  a[1] = cadd(os02, os13);
  a[5] = csub(os02, os13);
  a[3] = add_ib<S>(od02, od13);
  a[7] = add_ib<-S>(od02, od13);
}
template <int R, int S>
__device__ __forceinline__ void dft(float2* a) {
  if constexpr (R == 8) dft8<S>(a);
  else if constexpr (R == 4) dft4<S>(a);
  else dft2<S>(a);
}

// ------------------------------------------------------------------ pass plan for size n
template <int n>
struct Plan {
  static constexpr int P = (n == 32 || n == 64) ? 2 : ((n >= 1024) ? 4 : 3);
  static constexpr int Rlast =
      (n == 32) ? 4 : (n == 128 ? 2 : (n == 256 ? 4 : (n == 1024 ? 2 : (n == 2048 ? 4 : 8))));
  template <int p> __host__ __device__ static constexpr int R() { return p == P - 1 ? Rlast : 8; }
  template <int p> __host__ __device__ static constexpr int Ns() { return p == 0 ? 1 : (p == 1 ? 8 : (p == 2 ? 64 : 512)); }
  static constexpr int NTW = 7;   // twiddles per thread per pass (nb * (R - 1) <= 7)
  static_assert(n == 32 || n == 64 || n == 128 || n == 256 || n == 512 || n == 1024 ||
                    n == 2048 || n == 4096,
                "n");
};

// conflict-free swizzle of an element index inside one residue region (bijection on [0, n))
__device__ __forceinline__ int swz(int e) { return e ^ ((e >> 4) & 15) ^ (((e >> 6) & 1) << 3); }

// Twiddles of pass p for butterfly index j (S = -1: e^{-2pi i ...}, S = +1: conjugate).
// tw_n[stride * k] = exp(-2 pi i k / n) (stride > 1 when the table holds a multiple of n roots).
template <int n, int p, int S>
__device__ __forceinline__ void load_tw(float2* tw, int j, const float2* __restrict__ tw_n,
                                        int stride = 1) {
  constexpr int R = Plan<n>::template R<p>();
  constexpr int Ns = Plan<n>::template Ns<p>();
  constexpr int nb = 8 / R;
#pragma unroll
  for (int u = 0; u < nb; ++u) {
    const int jb = j * nb + u;
    const int k = jb % Ns;
#pragma unroll
    for (int r = 1; r < R; ++r) {
      float2 w = __ldg(&tw_n[((k * r * (n / (Ns * R))) & (n - 1)) * stride]);
      if (S > 0) w.y = -w.y;
      tw[u * (R - 1) + r - 1] = w;
    }
  }
}

// One Stockham pass on registers v[8] of one residue: optional read from src (smem region),
// twiddle (p > 0), DFT_R, optional write to dst (smem region).
template <int n, int p, int S, bool READ, bool WRITE>
__device__ __forceinline__ void pass(float2 (&v)[8], const float2* src, float2* dst, int j,
                                     const float2* tw) {
  constexpr int R = Plan<n>::template R<p>();
  constexpr int Ns = Plan<n>::template Ns<p>();
  constexpr int nb = 8 / R;
  constexpr int stride = n / R;
  if constexpr (READ) {
#pragma unroll
    for (int u = 0; u < nb; ++u)
#pragma unroll
      for (int r = 0; r < R; ++r) v[u * R + r] = src[swz(j * nb + u + r * stride)];
  }
  if constexpr (p > 0) {
#pragma unroll
    for (int u = 0; u < nb; ++u)
#pragma unroll
      for (int r = 1; r < R; ++r) v[u * R + r] = cmul(v[u * R + r], tw[u * (R - 1) + r - 1]);
  }
#pragma unroll
  for (int u = 0; u < nb; ++u) dft<R, S>(&v[u * R]);
  if constexpr (WRITE) {
#pragma unroll
    for (int u = 0; u < nb; ++u) {
      const int jb = j * nb + u;
      const int base = (jb / Ns) * Ns * R + (jb % Ns);
#pragma unroll
      for (int r = 0; r < R; ++r) dst[swz(base + r * Ns)] = v[u * R + r];
    }
  }
}

// Per-thread twiddles of passes 1..P-1 (depend only on the butterfly index j).
template <int n, int S>
struct PassTw {
  float2 tw[3][7];
  __device__ __forceinline__ void load(int j, const float2* __restrict__ tw_n, int stride = 1) {
    constexpr int P = Plan<n>::P;
    if constexpr (P > 1) load_tw<n, 1, S>(tw[0], j, tw_n, stride);
    if constexpr (P > 2) load_tw<n, 2, S>(tw[1], j, tw_n, stride);
    if constexpr (P > 3) load_tw<n, 3, S>(tw[2], j, tw_n, stride);
  }
};

// CTA-cooperative FFT of G = blockDim.x / (n/8) transforms stored in smem buffer A
// ([G][n], element e of transform g at A[g*n + swz(e)], natural order), scratch B.
// Output natural order; returns the buffer holding it.  Starts and ends with __syncthreads().
template <int n, int S>
__device__ __forceinline__ float2* cta_fft(float2* A, float2* B, const PassTw<n, S>& T) {
  constexpr int P = Plan<n>::P;
  const int g = threadIdx.x / (n / 8), j = threadIdx.x % (n / 8);
  float2 v[8];
  __syncthreads();
  pass<n, 0, S, true, true>(v, A + g * n, B + g * n, j, nullptr);
  __syncthreads();
  pass<n, 1, S, true, true>(v, B + g * n, A + g * n, j, T.tw[0]);
  __syncthreads();
  if constexpr (P > 2) {
    pass<n, 2, S, true, true>(v, A + g * n, B + g * n, j, T.tw[1]);
    __syncthreads();
  }
  if constexpr (P > 3) {
    pass<n, 3, S, true, true>(v, B + g * n, A + g * n, j, T.tw[2]);
    __syncthreads();
  }
  return (P & 1) ? B : A;
}

// ---- low-register variant: twiddles generated from one table value per butterfly
// w^r for r = 1..7 from w by repeated multiplication (error ~3 ulp at r = 7).
__device__ __forceinline__ void tw_powers(float2 w, float2* t) {   // t[0..6] = w^1..w^7
  t[0] = w;
  t[1] = cmul(w, w);
  t[2] = cmul(t[1], w);
  t[3] = cmul(t[1], t[1]);
  t[4] = cmul(t[3], w);
  t[5] = cmul(t[2], t[2]);
  t[6] = cmul(t[3], t[2]);
}

// ---- padded layout: element e of a region lives at e + (e >> 4) (one pad slot per 16).
// Every access pattern of a pass is phys(base) + compile-time offset (no carries out of the
// low 4 bits), so a pass needs one address computation per butterfly.
__host__ __device__ constexpr int padded(int n) { return n + n / 16; }
// stride between residue regions: padded(n) rounded up to 2 mod 16 (8-byte words), so that
// accesses running across residues (consecutive q = L a + s) hit distinct bank pairs
__host__ __device__ constexpr int rstride(int n) { return padded(n) + ((18 - padded(n) % 16) % 16); }
__device__ __forceinline__ int phys(int e) { return e + (e >> 4); }
template <int c>
__device__ __forceinline__ constexpr int poff() { return c + (c >> 4); }

// Stockham pass p of one n-point transform (8 points per thread, padded smem layout);
// twiddles of p > 0 generated from one table value per butterfly.
template <int n, int p, int S, bool READ, bool WRITE, bool ZERO = false>
__device__ __forceinline__ void pass_g(float2 (&v)[8], float2* src, float2* dst, int j,
                                       const float2* __restrict__ tw_n, int stride = 1) {
  constexpr int R = Plan<n>::template R<p>();
  constexpr int Ns = Plan<n>::template Ns<p>();
  constexpr int nb = 8 / R;
  constexpr int strd = n / R;
  float2 wb[nb];
  if constexpr (p > 0) {
#pragma unroll
    for (int u = 0; u < nb; ++u) {
      const int k = (j * nb + u) % Ns;
      float2 w = __ldg(&tw_n[((k * (n / (Ns * R))) & (n - 1)) * stride]);
      if (S > 0) w.y = -w.y;
      wb[u] = w;
    }
  }
  if constexpr (READ) {
#pragma unroll
    for (int u = 0; u < nb; ++u) {
      float2* sb = src + phys(j * nb + u);
#pragma unroll
      for (int r = 0; r < R; ++r) {
        v[u * R + r] = sb[r * strd + ((r * strd) >> 4)];
        if constexpr (ZERO) sb[r * strd + ((r * strd) >> 4)] = make_float2(0.f, 0.f);
      }
    }
  }
  if constexpr (p > 0) {
#pragma unroll
    for (int u = 0; u < nb; ++u) {
      if constexpr (R == 8) {
        float2 t[7];
        tw_powers(wb[u], t);
#pragma unroll
        for (int r = 1; r < 8; ++r) v[r] = cmul(v[r], t[r - 1]);
      } else if constexpr (R == 4) {
        const float2 w2 = cmul(wb[u], wb[u]);
        v[u * 4 + 1] = cmul(v[u * 4 + 1], wb[u]);
        v[u * 4 + 2] = cmul(v[u * 4 + 2], w2);
        v[u * 4 + 3] = cmul(v[u * 4 + 3], cmul(w2, wb[u]));
      } else {
        v[u * 2 + 1] = cmul(v[u * 2 + 1], wb[u]);
      }
    }
  }
#pragma unroll
  for (int u = 0; u < nb; ++u) dft<R, S>(&v[u * R]);
  if constexpr (WRITE) {
#pragma unroll
    for (int u = 0; u < nb; ++u) {
      const int jb = j * nb + u;
      float2* db = dst + phys((jb / Ns) * Ns * R + (jb % Ns));
#pragma unroll
      for (int r = 0; r < R; ++r) db[r * Ns + ((r * Ns) >> 4)] = v[u * R + r];
    }
  }
}

// Named barrier over `count` threads (id 1..15; id 0 is __syncthreads).
__device__ __forceinline__ void named_bar(int id, int count) {
  asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(count) : "memory");
}

// Barrier of the n/8 threads of transform group g (G groups in the CTA).
template <int n>
__device__ __forceinline__ void group_sync(int g, int G) {
  if constexpr (n / 8 <= 32) {
    __syncwarp();
  } else {
    if (G <= 15) named_bar(1 + g, n / 8);
    else __syncthreads();
  }
}

// CTA-cooperative transforms, padded layout: G = blockDim.x / (n/8) transforms, transform g in
// A + g * rstride(n) (natural order, element e at phys(e)), scratch B of the same shape.  The
// output (natural order, padded) is returned; starts and ends with __syncthreads().
template <int n, int S>
__device__ __forceinline__ float2* cta_fft_g(float2* A, float2* B, const float2* __restrict__ tw_n,
                                             int stride = 1) {
  constexpr int P = Plan<n>::P;
  constexpr int rs = rstride(n);
  const int g = threadIdx.x / (n / 8), j = threadIdx.x & (n / 8 - 1);
  const int G = blockDim.x / (n / 8);
  float2 v[8];
  __syncthreads();
  pass_g<n, 0, S, true, true>(v, A + g * rs, B + g * rs, j, tw_n, stride);
  group_sync<n>(g, G);
  pass_g<n, 1, S, true, true>(v, B + g * rs, A + g * rs, j, tw_n, stride);
  if constexpr (P > 2) {
    group_sync<n>(g, G);
    pass_g<n, 2, S, true, true>(v, A + g * rs, B + g * rs, j, tw_n, stride);
  }
  if constexpr (P > 3) {
    group_sync<n>(g, G);
    pass_g<n, 3, S, true, true>(v, B + g * rs, A + g * rs, j, tw_n, stride);
  }
  __syncthreads();
  return (P & 1) ? B : A;
}

// Output position (natural order) of register element e after the LAST pass.
template <int n>
__device__ __forceinline__ int last_pos(int j, int e) {
  constexpr int R = Plan<n>::Rlast;
  constexpr int nb = 8 / R;
  return j * nb + e / R + (e % R) * (n / R);
}

}  // namespace fe
}  // namespace tat
