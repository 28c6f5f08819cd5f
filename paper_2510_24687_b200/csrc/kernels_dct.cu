// lambda <-> t cosine transforms (Alg. 1 step 5, E:inverse_cos_tr P:L475-478; Alg. 2 step 3,
// E:Four_coef_u P:L649-651) on the register FFT engine.
//
//   K4   G[m]  = sum_{j=0}^{J} H[j] cos(pi j (m+1)/M)          (S3 row k -> S4 row k)
//   K4T  Hc[j] = sum_{m=0}^{n_t-1} G~[m] cos(pi j (m+1)/M),  H~ = (-i)^k omega m'[k][j] Hc
//
// Both are "X[u] = sum_i c[i] W_2M^{i u}, out = (X[u] + X[-u]) / 2" with the 2M-point DFT split
// into r output residues u = r a + v (r in {1, 3}): X[r a + v] = FFT_nf(c[i] W_2M^{i v})[a],
// nf = 2M / r, valid when every input index i < nf (no folding).  One CTA per (image, k); the r
// residue transforms run one after another on nf/8 threads and stay in shared memory.
#include "fft_engine.cuh"
#include "tat_internal.h"

namespace tat {

using namespace fe;

__device__ __forceinline__ float2 mul_ipow_d(float2 a, int e) {
  switch (e & 3) {
    case 0: return a;
    case 1: return make_float2(-a.y, a.x);
    case 2: return make_float2(-a.x, -a.y);
    default: return make_float2(a.y, -a.x);
  }
}

// ADJ = false: K4 (input S3 row, J+1 values at i = j; outputs m' = m + 1, m < n_t)
// ADJ = true : K4T (input S4 row, n_t values at i = m + 1; outputs j in [0, J])
template <int nf, bool ADJ>
__global__ void __launch_bounds__(512) k4_dct_fast(DevPlan P, int r) {
  extern __shared__ float2 sm[];
  constexpr int rs = rstride(nf);
  constexpr int PP = Plan<nf>::P;
  const Consts& C = P.C;
  const int M2 = 2 * C.M, NL = C.NL, n_t = C.n_t;
  const int b = C.b0 + blockIdx.y, k = blockIdx.x;
  const int j = threadIdx.x;                 // butterfly index, blockDim.x == nf / 8
  const float2* in = ADJ ? P.S4 + ((size_t)b * C.Kp + k) * n_t : P.S3 + ((size_t)b * C.Kp + k) * NL;
  const int lo = ADJ ? 1 : 0;                // input index of in[0]
  const int cnt = ADJ ? n_t : NL;
  float mloc[8];   // K4T multiplier row, loaded before the transforms
#pragma unroll
  for (int u = 0; u < 8; ++u) {
    const int jj = threadIdx.x + u * (nf / 8);
    mloc[u] = (ADJ && jj < NL) ? __ldg(&P.mult[(size_t)k * NL + jj]) : 0.f;
  }
  // buffer pool: r results + one scratch; pass p writes A for even p, B for odd p
  constexpr bool finB = (PP % 2) == 0;
  int res_slot[3] = {0, 0, 0};
  int fa = 0, fb = 1, fresh = 2;
  // inputs (shared by all residues) and the residue twiddles W_2M^{i v}, v = 1, 2, loaded at once
  float2 xin[8], tw1[8], tw2[8];
#pragma unroll
  for (int e = 0; e < 8; ++e) {
    const int i = j + e * (nf / 8);
    const int src = i - lo;
    xin[e] = (src >= 0 && src < cnt) ? __ldg(&in[src]) : make_float2(0.f, 0.f);
    tw1[e] = r > 1 ? __ldg(&P.tw_dct[(int)((long long)i % M2)]) : make_float2(1.f, 0.f);
    tw2[e] = r > 2 ? __ldg(&P.tw_dct[(int)(((long long)i * 2) % M2)]) : make_float2(1.f, 0.f);
  }
  for (int v = 0; v < r; ++v) {
    float2* A = sm + fa * rs;
    float2* B = sm + fb * rs;
    float2 x[8];
#pragma unroll
    for (int e = 0; e < 8; ++e) x[e] = v == 0 ? xin[e] : cmul(xin[e], v == 1 ? tw1[e] : tw2[e]);
    pass_g<nf, 0, -1, false, true>(x, nullptr, A, j, P.tw_dct, r);
    __syncthreads();
    pass_g<nf, 1, -1, true, true>(x, A, B, j, P.tw_dct, r);
    __syncthreads();
    if constexpr (PP > 2) {
      pass_g<nf, 2, -1, true, true>(x, B, A, j, P.tw_dct, r);
      __syncthreads();
    }
    if constexpr (PP > 3) {
      pass_g<nf, 3, -1, true, true>(x, A, B, j, P.tw_dct, r);
      __syncthreads();
    }
    if (finB) { res_slot[v] = fb; fb = fresh++; }
    else { res_slot[v] = fa; fa = fresh++; }
  }
  // gather X[u] and X[-u] from the residue results
  auto X = [&](int u) -> float2 {
    const int vv = u % r, a = u / r;
    return sm[res_slot[vv] * rs + phys(a)];
  };
  if (!ADJ) {
    float2* out = P.S4 + ((size_t)b * C.Kp + k) * n_t;
    for (int m = threadIdx.x; m < n_t; m += blockDim.x) {
      const int u = m + 1;
      out[m] = cscale(cadd(X(u), X(M2 - u)), 0.5f);
    }
  } else {
    float2* out = P.S3 + ((size_t)b * C.Kp + k) * NL;
    const float om = (float)C.omega;
#pragma unroll
    for (int u = 0; u < 8; ++u) {   // NL <= nf = 8 * blockDim.x
      const int jj = threadIdx.x + u * (nf / 8);
      if (jj < NL) {
        // cosine: (X(u) + X(-u)) / 2;  sine (C.dct_sine): i (X(u) - X(-u)) / 2
        const float2 xp = X(jj), xm = X(jj == 0 ? 0 : M2 - jj);
        const float2 y = C.dct_sine ? cscale(make_float2(xm.y - xp.y, xp.x - xm.x), 0.5f)
                                    : cscale(cadd(xp, xm), 0.5f);
        out[jj] = mul_ipow_d(cscale(y, om * mloc[u]), -k);
      }
    }
  }
}

// fast path applicability: 2M = r nf, r in {1, 3}, nf a supported power of two, inputs fit
int dct_fast_r(const Consts& C) {
  const long M2 = 2L * C.M;
  for (int r : {1, 3}) {
    if (M2 % r) continue;
    const long nf = M2 / r;
    if (nf < 32 || nf > 4096 || (nf & (nf - 1))) continue;
    if (C.NL > nf || C.n_t + 1 > nf) continue;
    return r;
  }
  return 0;
}
int dct_fast_nf(const Consts& C) { const int r = dct_fast_r(C); return r ? (2 * C.M) / r : 0; }
size_t smem_dct_fast(const Consts& C) { return (size_t)4 * rstride(dct_fast_nf(C)) * sizeof(float2); }

#define TAT_DCT_SWITCH(NFV, ...)                        \
  switch (NFV) {                                         \
    case 32: { constexpr int NF = 32; __VA_ARGS__; } break;     \
    case 64: { constexpr int NF = 64; __VA_ARGS__; } break;     \
    case 128: { constexpr int NF = 128; __VA_ARGS__; } break;   \
    case 256: { constexpr int NF = 256; __VA_ARGS__; } break;   \
    case 512: { constexpr int NF = 512; __VA_ARGS__; } break;   \
    case 1024: { constexpr int NF = 1024; __VA_ARGS__; } break; \
    case 2048: { constexpr int NF = 2048; __VA_ARGS__; } break; \
    case 4096: { constexpr int NF = 4096; __VA_ARGS__; } break; \
    default: return cudaErrorInvalidValue;               \
  }

cudaError_t configure_dct_kernels(const Consts& C) {
  const int nf = dct_fast_nf(C);
  if (!nf) return cudaSuccess;
  if (smem_dct_fast(C) > (size_t)kSmemLimit) return cudaErrorInvalidConfiguration;
  const int sm = kSmemLimit;
  cudaError_t e = cudaSuccess;
  TAT_DCT_SWITCH(nf, {
    if (e == cudaSuccess) e = cudaFuncSetAttribute(k4_dct_fast<NF, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, sm);
    if (e == cudaSuccess) e = cudaFuncSetAttribute(k4_dct_fast<NF, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, sm);
  });
  return e;
}

cudaError_t launch_k4_fast(const DevPlan& P, bool adj, cudaStream_t s) {
  const Consts& C = P.C;
  const int nf = dct_fast_nf(C), r = dct_fast_r(C);
  const size_t sm = smem_dct_fast(C);
  TAT_DCT_SWITCH(nf, {
    if (adj) k4_dct_fast<NF, true><<<dim3(C.Kp, C.batch), NF / 8, sm, s>>>(P, r);
    else k4_dct_fast<NF, false><<<dim3(C.Kp, C.batch), NF / 8, sm, s>>>(P, r);
  });
  return cudaGetLastError();
}

}  // namespace tat
