// In-register DFTs with compile-time twiddles for the two-stage column transforms
// (kernels_col.cu).  An R-point DFT (R = 16, 32, 64) is done entirely in one thread's
// registers as R1 x R2 (radix-4/8 butterflies of fft_engine.cuh + constant inter-twiddles),
// so a thread's R points never touch shared memory between the two radix levels.
#pragma once
#include "fft_engine.cuh"

namespace tat {
namespace ce {

using fe::cadd;
using fe::cmul;
using fe::cmulc;
using fe::csub;

// cos(2 pi k / 64), double literals (constant-folded after unrolling)
__host__ __device__ constexpr double cos64(int k) {
  switch (k & 63) {
    case 0: return 1.0;
    case 1: return 0.9951847266721969;
    case 2: return 0.9807852804032304;
    case 3: return 0.9569403357322088;
    case 4: return 0.9238795325112867;
    case 5: return 0.881921264348355;
    case 6: return 0.8314696123025452;
    case 7: return 0.773010453362737;
    case 8: return 0.7071067811865476;
    case 9: return 0.6343932841636455;
    case 10: return 0.5555702330196023;
    case 11: return 0.4713967368259978;
    case 12: return 0.38268343236508984;
    case 13: return 0.29028467725446233;
    case 14: return 0.19509032201612833;
    case 15: return 0.09801714032956077;
    case 16: return 6.123233995736766e-17;
    case 17: return -0.09801714032956065;
    case 18: return -0.1950903220161282;
    case 19: return -0.29028467725446216;
    case 20: return -0.3826834323650897;
    case 21: return -0.4713967368259977;
    case 22: return -0.555570233019602;
    case 23: return -0.6343932841636454;
    case 24: return -0.7071067811865475;
    case 25: return -0.773010453362737;
    case 26: return -0.8314696123025453;
    case 27: return -0.8819212643483549;
    case 28: return -0.9238795325112867;
    case 29: return -0.9569403357322088;
    case 30: return -0.9807852804032304;
    case 31: return -0.9951847266721968;
    case 32: return -1.0;
    case 33: return -0.9951847266721969;
    case 34: return -0.9807852804032304;
    case 35: return -0.9569403357322089;
    case 36: return -0.9238795325112868;
    case 37: return -0.881921264348355;
    case 38: return -0.8314696123025455;
    case 39: return -0.7730104533627371;
    case 40: return -0.7071067811865477;
    case 41: return -0.6343932841636459;
    case 42: return -0.5555702330196022;
    case 43: return -0.47139673682599786;
    case 44: return -0.38268343236509034;
    case 45: return -0.29028467725446244;
    case 46: return -0.19509032201612866;
    case 47: return -0.09801714032956045;
    case 48: return -1.8369701987210297e-16;
    case 49: return 0.09801714032956009;
    case 50: return 0.1950903220161283;
    case 51: return 0.29028467725446205;
    case 52: return 0.38268343236509;
    case 53: return 0.4713967368259976;
    case 54: return 0.5555702330196018;
    case 55: return 0.6343932841636456;
    case 56: return 0.7071067811865474;
    case 57: return 0.7730104533627367;
    case 58: return 0.8314696123025452;
    case 59: return 0.8819212643483548;
    case 60: return 0.9238795325112865;
    case 61: return 0.9569403357322088;
    case 62: return 0.9807852804032303;
    case 63: return 0.9951847266721969;
  }
  return 0.0;
}

// a * exp(S 2 pi i e / R) for a compile-time-foldable e (after unrolling); R divides 64.
template <int R, int S>
__device__ __forceinline__ float2 twk(float2 a, int e) {
  const int E = ((e % R) + R) % R;            // exp(S 2 pi i E / R)
  if (E == 0) return a;
  const int Es = (S > 0) ? E : (R - E) % R;   // as exp(+2 pi i Es / R)
  if (4 * Es == R) return make_float2(-a.y, a.x);          // * i
  if (2 * Es == R) return make_float2(-a.x, -a.y);         // * -1
  if (4 * Es == 3 * R) return make_float2(a.y, -a.x);      // * -i
  const int k = Es * (64 / R);
  const float c = (float)cos64(k), s = (float)cos64(k - 16);
  return cmul(a, make_float2(c, s));
}

// Natural-order in-place DFT of R = R1 * R2 points in registers:
//   X[k] = sum_m a[m] exp(S 2 pi i m k / R).
template <int R1, int R2, int S>
__device__ __forceinline__ void dft_2l(float2* a) {
  constexpr int R = R1 * R2;
  float2 b[R];
#pragma unroll
  for (int m2 = 0; m2 < R2; ++m2) {
    float2 t[R1];
#pragma unroll
    for (int m1 = 0; m1 < R1; ++m1) t[m1] = a[m2 + R2 * m1];
    fe::dft<R1, S>(t);
#pragma unroll
    for (int k1 = 0; k1 < R1; ++k1) b[m2 * R1 + k1] = twk<R, S>(t[k1], m2 * k1);
  }
#pragma unroll
  for (int k1 = 0; k1 < R1; ++k1) {
    float2 t[R2];
#pragma unroll
    for (int m2 = 0; m2 < R2; ++m2) t[m2] = b[m2 * R1 + k1];
    fe::dft<R2, S>(t);
#pragma unroll
    for (int k2 = 0; k2 < R2; ++k2) a[k1 + R1 * k2] = t[k2];
  }
}

template <int R, int S>
__device__ __forceinline__ void dftr(float2* a) {
  if constexpr (R == 8) fe::dft<8, S>(a);
  else if constexpr (R == 16) dft_2l<4, 4, S>(a);
  else if constexpr (R == 32) dft_2l<8, 4, S>(a);
  else {
    static_assert(R == 64, "R");
    dft_2l<8, 8, S>(a);
  }
}

// pw[k] = b^k for k = 1 .. R-1 by binary splitting (depth log2 R; error ~ log2 R ulp).
template <int R>
__device__ __forceinline__ void pow_tree(float2 b, float2* pw) {
  pw[0] = make_float2(1.f, 0.f);
  pw[1] = b;
#pragma unroll
  for (int k = 2; k < R; ++k) pw[k] = cmul(pw[k / 2], pw[k - k / 2]);
}

}  // namespace ce
}  // namespace tat
