// Kernels specific to the inverse A^{-1} (Algorithm 3); every other stage
// of the inverse reuses the adjoint chain (K5T, the sine variant of K4T, K3T, K2Tb, K1T).
//
//   k2i_interp : Alg. 3 step 5 -- bilinear interpolation in (lambda, phi) from the half-plane
//                polar values (adjoint S2 node order; the other half by conjugate symmetry) to
//                every Cartesian node of the half spectrum inside the disk |xi| < lambda_max
//                (reading G22).  One thread per target for all images: its 32-byte record
//                (4 node codes, 4 weights) is read once and reused across the batch.
//   k2i_const  : step 7 -- per image, the sum of v over the annulus r0 < |x| < R as kInvParts
//                fixed-order partial sums (one CTA each; deterministic).
//   k2i_project: step 8 -- f = (v + C) on |x| <= r0, 0 elsewhere, C = -sum / count (the
//                partials summed in a fixed order once per CTA).
#include "tat_internal.h"

namespace tat {


__device__ __forceinline__ float2 inv_node(const float2* __restrict__ S2, int code) {
  // code >= 0: node value; code < 0: conj of node (-code - 1) (the mirror angle phi + pi)
  if (code >= 0) return __ldg(&S2[code]);
  const float2 v = __ldg(&S2[-code - 1]);
  return make_float2(v.x, -v.y);
}

__global__ void __launch_bounds__(256) k2i_interp(DevPlan P) {
  const Consts& C = P.C;
  const int t = blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= C.ntargets) return;
  const int4 nd = __ldg(&P.inv_nodes[t]);
  const float4 w = __ldg(&P.inv_w[t]);
  const size_t img = (size_t)C.half * C.NL;
  const float2* S2 = P.S2 + C.b0 * img;
  float2* Rc = P.Rc + (size_t)C.b0 * C.ntpad + t;
#pragma unroll 1   // one image at a time: deeper unrolling measured slower (L2 working set)
  for (int b = 0; b < C.batch; ++b, S2 += img, Rc += C.ntpad) {
    float2 acc = __fmul2_rn(make_float2(w.x, w.x), inv_node(S2, nd.x));
    acc = __ffma2_rn(make_float2(w.y, w.y), inv_node(S2, nd.y), acc);
    acc = __ffma2_rn(make_float2(w.z, w.z), inv_node(S2, nd.z), acc);
    acc = __ffma2_rn(make_float2(w.w, w.w), inv_node(S2, nd.w), acc);
    *Rc = acc;
  }
}

// region[iy * n + ix]: 1 in Omega_0 (|x| <= r0), 2 in the annulus r0 < |x| < R, 0 elsewhere
__global__ void __launch_bounds__(256) k2i_const(DevPlan P, const float* __restrict__ v,
                                                 const unsigned char* __restrict__ region,
                                                 float* __restrict__ csum) {
  __shared__ float red[256];
  const Consts& C = P.C;
  const int b = C.b0 + blockIdx.y, nn = C.n * C.n;
  const int i0 = (int)(((long)nn * blockIdx.x) / kInvParts), i1 = (int)(((long)nn * (blockIdx.x + 1)) / kInvParts);
  const float* vb = v + (size_t)b * nn;
  float s = 0.f;
  for (int i = i0 + threadIdx.x; i < i1; i += blockDim.x)
    if (__ldg(&region[i]) == 2) s += vb[i];
  red[threadIdx.x] = s;
  __syncthreads();
  for (int w = 128; w > 0; w >>= 1) {
    if ((int)threadIdx.x < w) red[threadIdx.x] += red[threadIdx.x + w];
    __syncthreads();
  }
  if (threadIdx.x == 0) csum[(size_t)b * kInvParts + blockIdx.x] = red[0];
}

__global__ void __launch_bounds__(256) k2i_project(DevPlan P, float* __restrict__ f,
                                                   const unsigned char* __restrict__ region,
                                                   const float* __restrict__ csum, float inv_count) {
  const Consts& C = P.C;
  const int nn = C.n * C.n;
  const int b = C.b0 + blockIdx.y;
  __shared__ float cst_s;
  if (threadIdx.x == 0) {   // the partials in a fixed order, once per CTA
    float sum = 0.f;
    for (int q = 0; q < kInvParts; ++q) sum += __ldg(&csum[(size_t)b * kInvParts + q]);
    cst_s = -sum * inv_count;
  }
  __syncthreads();
  const float cst = cst_s;
  float* fb = f + (size_t)b * nn;
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < nn; i += gridDim.x * blockDim.x)
    fb[i] = (__ldg(&region[i]) == 1) ? fb[i] + cst : 0.f;
}

cudaError_t launch_k2i_interp(const DevPlan& P, cudaStream_t s) {
  const Consts& C = P.C;
  k2i_interp<<<(C.ntargets + 255) / 256, 256, 0, s>>>(P);
  return cudaGetLastError();
}

cudaError_t launch_k2i_finish(const DevPlan& P, float* f, const unsigned char* region, float* csum,
                              int annulus_count, cudaStream_t s) {
  const Consts& C = P.C;
  k2i_const<<<dim3(kInvParts, C.batch), 256, 0, s>>>(P, f, region, csum);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return e;
  const float inv = annulus_count > 0 ? 1.f / (float)annulus_count : 0.f;
  k2i_project<<<dim3((C.n * C.n + 255) / 256, C.batch), 256, 0, s>>>(P, f, region, csum, inv);
  return cudaGetLastError();
}

}  // namespace tat
