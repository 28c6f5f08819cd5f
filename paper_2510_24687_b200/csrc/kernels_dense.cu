// Dense angular synthesis / analysis for detectors off any canonical ring (reading G24; SURVEY
// §8(f) f4 (ii)).  Steps 6-7 of Algorithm 1 (E:FourSerForg P:L407-411, restriction P:L562) and
// steps 1-2 of Algorithm 2 evaluated at the exact detector angles theta_d:
//
//   K5d : g[b][m][d] = sum_{k=0}^{K} Re( S4[b][k][m] E5[k][d] ),  E5 = c_k e^{i s_k k theta_d}
//   K5dT: S4[b][k][m] = sum_d g[b][m][d] conj(E5T[k][d]),        E5T = e^{i s_k k theta_d}
//
// (c_0 = c_K = 1, c_k = 2 otherwise; s_K = -1: row K holds the harmonic -K; its row is real,
// reading G24).  Both are real GEMMs of shape [n_t x 2(K+1)] x [2(K+1) x n_det] per image, tiled
// through shared memory with 8 x 8 (K5d, register-staged next chunk) / 4 x 4 register blocks
// (exact fp32: single-pass TF32 tensor cores would miss the 1e-4 bar).
#include "tat_internal.h"

namespace tat {

// ---- K5d: out[m][d] over a 128 x 128 (m, d) tile, reduction over k; 256 threads, 8 x 8 per
// thread (rows ty + 16 i, columns tx + 16 j: conflict-free shared-memory reads)
constexpr int kST = 128, kSK = 8;
__global__ void __launch_bounds__(256) k5d_synth(DevPlan P, float* __restrict__ gout) {
  __shared__ float2 As[kSK][kST];   // S4 rows k, columns m
  __shared__ float2 Bs[kSK][kST];   // E5 rows k, columns d
  const Consts& C = P.C;
  const int b = C.b0 + blockIdx.z;
  const int m0 = blockIdx.y * kST, d0 = blockIdx.x * kST;
  const int tx = threadIdx.x & 15, ty = threadIdx.x >> 4;
  const float2* S4 = P.S4 + (size_t)b * C.Kp * C.n_t;
  float acc[8][8] = {};
  pdl_wait();
  pdl_trigger();
  float2 ra[4], rb[4];   // next chunk, 4 elements of each operand per thread
  auto fetch = [&](int k0) {
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const int i = threadIdx.x + 256 * q, kk = i / kST, c = i - kk * kST, k = k0 + kk;
      ra[q] = (k < C.Kp && m0 + c < C.n_t) ? S4[(size_t)k * C.n_t + m0 + c] : make_float2(0.f, 0.f);
      rb[q] = (k < C.Kp && d0 + c < C.n_det) ? __ldg(&P.dense_e5[(size_t)k * C.n_det + d0 + c])
                                             : make_float2(0.f, 0.f);
    }
  };
  fetch(0);
  for (int k0 = 0; k0 < C.Kp; k0 += kSK) {
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const int i = threadIdx.x + 256 * q, kk = i / kST, c = i - kk * kST;
      As[kk][c] = ra[q];
      Bs[kk][c] = rb[q];
    }
    __syncthreads();
    if (k0 + kSK < C.Kp) fetch(k0 + kSK);
#pragma unroll
    for (int kk = 0; kk < kSK; ++kk) {
      float2 a[8], e[8];
#pragma unroll
      for (int i = 0; i < 8; ++i) a[i] = As[kk][ty + 16 * i];
#pragma unroll
      for (int j = 0; j < 8; ++j) e[j] = Bs[kk][tx + 16 * j];
#pragma unroll
      for (int i = 0; i < 8; ++i)
#pragma unroll
        for (int j = 0; j < 8; ++j) acc[i][j] = fmaf(a[i].x, e[j].x, fmaf(-a[i].y, e[j].y, acc[i][j]));
    }
    __syncthreads();
  }
#pragma unroll
  for (int i = 0; i < 8; ++i) {
    const int m = m0 + ty + 16 * i;
    if (m >= C.n_t) continue;
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      const int d = d0 + tx + 16 * j;
      if (d < C.n_det) {
        const size_t o = ((size_t)b * C.n_t + m) * C.n_det + d;
        gout[o] = epi_fwd(P, o, acc[i][j]);
      }
    }
  }
}

constexpr int kDT = 64;   // K5dT output tile (both dims)
constexpr int kDK = 16;   // K5dT reduction chunk

// ---- K5dT: out[k][m] (complex) over k-tile x m-tile, reduction over d
__global__ void __launch_bounds__(256) k5d_anal(DevPlan P, const float* __restrict__ gin) {
  __shared__ float2 Es[kDK][kDT + 1];   // E5T rows d (chunk), columns k
  __shared__ float Gs[kDK][kDT + 1];    // g rows d (chunk), columns m
  const Consts& C = P.C;
  const int b = C.b0 + blockIdx.z;
  const int k0 = blockIdx.y * kDT, m0 = blockIdx.x * kDT;
  const int tx = threadIdx.x & 15, ty = threadIdx.x >> 4;
  const float* g = gin + (size_t)b * C.n_t * C.n_det;
  float2 acc[4][4];
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j) acc[i][j] = make_float2(0.f, 0.f);
  pdl_wait();
  pdl_trigger();
  for (int dd0 = 0; dd0 < C.n_det; dd0 += kDK) {
    for (int i = threadIdx.x; i < kDK * kDT; i += 256) {
      const int r = i / kDK, c = i - r * kDK;    // r: k or m within the tile, c: d within the chunk
      const int d = dd0 + c;
      Es[c][r] = (k0 + r < C.Kp && d < C.n_det) ? __ldg(&P.dense_e5t[(size_t)(k0 + r) * C.n_det + d])
                                                : make_float2(0.f, 0.f);
      Gs[c][r] = (m0 + r < C.n_t && d < C.n_det) ? g[(size_t)(m0 + r) * C.n_det + d] : 0.f;
    }
    __syncthreads();
#pragma unroll
    for (int c = 0; c < kDK; ++c) {
      float2 e[4];
      float gv[4];
#pragma unroll
      for (int i = 0; i < 4; ++i) e[i] = Es[c][ty * 4 + i];
#pragma unroll
      for (int j = 0; j < 4; ++j) gv[j] = Gs[c][tx * 4 + j];
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          acc[i][j].x = fmaf(e[i].x, gv[j], acc[i][j].x);
          acc[i][j].y = fmaf(-e[i].y, gv[j], acc[i][j].y);
        }
    }
    __syncthreads();
  }
  float2* S4 = P.S4 + (size_t)b * C.Kp * C.n_t;
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const int k = k0 + ty * 4 + i;
    if (k >= C.Kp) continue;
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const int m = m0 + tx * 4 + j;
      if (m < C.n_t) S4[(size_t)k * C.n_t + m] = acc[i][j];
    }
  }
}

cudaError_t launch_k5d(const DevPlan& P, float* g, cudaStream_t s) {
  const Consts& C = P.C;
  const dim3 grid((C.n_det + kST - 1) / kST, (C.n_t + kST - 1) / kST, C.batch);
  const cudaError_t e = launch_pdl(C.pdl, k5d_synth, grid, dim3(256), 0, s, P, g);
  return e != cudaSuccess ? e : cudaGetLastError();
}

cudaError_t launch_k5dt(const DevPlan& P, const float* g, cudaStream_t s) {
  const Consts& C = P.C;
  const dim3 grid((C.n_t + kDT - 1) / kDT, (C.Kp + kDT - 1) / kDT, C.batch);
  const cudaError_t e = launch_pdl(C.pdl, k5d_anal, grid, dim3(256), 0, s, P, g);
  return e != cudaSuccess ? e : cudaGetLastError();
}

}  // namespace tat
