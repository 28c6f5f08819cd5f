// Dense angular synthesis / analysis for detectors off any canonical ring (reading G24; SURVEY
// §8(f) f4 (ii)).  Steps 6-7 of Algorithm 1 (E:FourSerForg P:L407-411, restriction P:L562) and
// steps 1-2 of Algorithm 2 evaluated at the exact detector angles theta_d:
//
//   K5d : g[b][m][d] = sum_{k=0}^{K} Re( S4[b][k][m] E5[k][d] ),  E5 = c_k e^{i s_k k theta_d}
//   K5dT: S4[b][k][m] = sum_d g[b][m][d] conj(E5T[k][d]),        E5T = e^{i s_k k theta_d}
//
// (c_0 = c_K = 1, c_k = 2 otherwise; s_K = -1: row K holds the harmonic -K; its row is real,
// reading G24).  Both are real GEMMs of shape [n_t x 2(K+1)] x [2(K+1) x n_det] per image.  They
// run on the tensor cores as 3xTF32 GEMMs (k5d_tc / k5dt_tc below; single-pass TF32 would miss
// the 1e-4 bar); k5d_synth / k5d_anal are exact-fp32 SIMT versions (shared-memory tiles, 8 x 8 /
// 4 x 4 register blocks) kept behind TAT_DENSE_TC=0.
#include "tat_internal.h"
#include "async_copy.cuh"

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


// ================================================================== K5d on tcgen05 (3xTF32)
// The same synthesis as k5d_synth as a real GEMM D[m][d] = sum_k' A[m][k'] B[k'][d] on the 5th-
// generation tensor cores: A[m][2k] = Re S4[k][m], A[m][2k+1] = Im S4[k][m]; B[2k][d] = Re E5,
// B[2k+1][d] = -Im E5 (pre-split on the host into TF32 hi / lo parts, packed in the operand
// layout).  fp32-level accuracy from three TF32 products per step, A_hi B_hi + A_hi B_lo +
// A_lo B_hi, accumulated in fp32 in TMEM.  Tile 128 (m = time) x 128 (d = detector), K chunks of
// 8 complex (16 real) values.
//
// A tf32 M128 N128 K8 MMA with both operands in shared memory reads 8 KB per 64 cycles, the
// whole 128 B/clk of the SM's shared-memory port, so every other shared-memory byte (the staged
// copies, the hi / lo split) stalls the tensor pipe.  A therefore goes to TMEM: 6 warps,
//   warp 0 (one thread)  streams each chunk's packed B tiles (2 x 8 KB) into a kSlots-deep
//                        shared-memory ring.  One SM's bulk-copy engine sustains only ~25 B/clk
//                        plus ~100 cycles per copy, so B, the same for every time tile, is
//                        multicast: the cs CTAs of a cluster (consecutive time tiles, same
//                        detector tile) each fetch 1/cs of it into all cs CTAs' slots;
//   warps 2..5           one time row m per thread (TMEM lane = warp % 4 quarter): the row's
//                        8 complex values per chunk arrive by cp.async (LSU path, kRawD chunks
//                        ahead, each thread reading back only its own bytes), are split hi / lo
//                        and tcgen05.st to one of kABufs TMEM A buffers (16 hi + 16 lo columns);
//   warp 1 (one thread)  issues the chunk's 6 tcgen05.mma (A from TMEM, B from shared memory in
//                        the canonical no-swizzle K-major layout: 8-row x 16-byte core matrices,
//                        K-adjacent cores 128 B apart, row groups 32 KC bytes apart) and commits
//                        them to the slot's mbarrier in every CTA of the cluster: a slot is
//                        refilled once all cs CTAs' MMAs on it retired (count cs).
// Epilogue (warps 2..5): tcgen05.ld of the accumulator (lanes = rows m), fused epi_fwd, 16-B stores.
namespace tc {
constexpr int MT = 128, NT = 128, KC = kK5tcKC, kSlots = 8, kABufs = 4, kRawD = 8;
constexpr uint32_t kLBO = 128, kSBO = (KC / 4) * 128;   // bytes
constexpr uint32_t kTile = NT * KC * 4;                  // one 128 x KC fp32 B tile (8 KB)
constexpr uint32_t kRawA = (KC / 2) * MT * 8;            // KC / 2 S4 rows of 128 complex (8 KB)
constexpr uint32_t kSlot = 2 * kTile;                    // B hi + B lo
constexpr uint32_t kTmemCols = 256;                      // accumulator 128 + kABufs x 2 KC
static_assert(NT + kABufs * 2 * KC <= (int)kTmemCols, "TMEM budget");

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ uint64_t desc_kmajor(uint32_t saddr) {
  uint64_t d = 0;
  d |= (uint64_t)((saddr >> 4) & 0x3FFF);
  d |= (uint64_t)((kLBO >> 4) & 0x3FFF) << 16;
  d |= (uint64_t)((kSBO >> 4) & 0x3FFF) << 32;
  d |= (uint64_t)1 << 46;   // version 1 (sm_100); base offset 0, lbo mode 0, no swizzle
  return d;
}
// kind::tf32, D f32, A/B tf32, both K-major, M = 128, N = 128
constexpr uint32_t kIdesc = (1u << 4) | (2u << 7) | (2u << 10) | ((uint32_t)(NT >> 3) << 17) |
                            ((uint32_t)(MT >> 4) << 24);

// TF32 high part by truncation (a LOP3; cvt.rna.tf32 issues on the slow XU pipe).  x - hi is
// exact in fp32 and the MMA reads the low part's top 19 bits, so the split keeps ~21 significant
// bits of every operand: fp32-level products.
__device__ __forceinline__ float tf32_hi(float x) { return __uint_as_float(__float_as_uint(x) & 0xFFFFE000u); }
// instruction descriptor of kind::tf32 with f32 accumulation, K-major A and B, M x N
__device__ __forceinline__ uint32_t idesc_tf32(int M, int N) {
  return (1u << 4) | (2u << 7) | (2u << 10) | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(M >> 4) << 24);
}
// D[tmem d] (+)= A[tmem a] B[smem desc b]
__device__ __forceinline__ void mma_tf32_ts(uint32_t d, uint32_t a, uint64_t b, uint32_t idesc, bool acc) {
  asm volatile(
      "{\n\t.reg .pred pa;\n\tsetp.ne.b32 pa, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::tf32 [%0], [%1], %2, %3, pa;\n\t}\n" ::"r"(d),
      "r"(a), "l"(b), "r"(idesc), "r"((uint32_t)acc));
}
// arrive on the mbarrier at this offset in every CTA of cmask once all prior MMAs retired
__device__ __forceinline__ void commit_mc(uint64_t* bar, uint16_t cmask) {
  asm volatile(
      "tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 "
      "[%0], %1;" ::"r"(smem_u32(bar)), "h"(cmask));
}
// 1-D bulk copy global -> the same shared offset in every CTA of cmask (complete_tx on each bar)
__device__ __forceinline__ void bulk_mc(void* dst, const void* src, uint32_t bytes, uint64_t* bar, uint16_t cmask) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.multicast::cluster "
      "[%0], [%1], %2, [%3], %4;" ::"r"(smem_u32(dst)), "l"(src), "r"(bytes), "r"(smem_u32(bar)), "h"(cmask)
      : "memory");
}
__device__ __forceinline__ void cluster_sync() {
  asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}
__device__ __forceinline__ void tmem_st32(uint32_t taddr, const uint32_t (&v)[32]) {
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x32.b32 [%0], {%1, %2, %3, %4, %5, %6, %7, %8, %9, %10, "
      "%11, %12, %13, %14, %15, %16, %17, %18, %19, %20, %21, %22, %23, %24, %25, %26, %27, "
      "%28, %29, %30, %31, %32};" ::"r"(taddr),
      "r"(v[0]), "r"(v[1]), "r"(v[2]), "r"(v[3]), "r"(v[4]), "r"(v[5]), "r"(v[6]), "r"(v[7]),
      "r"(v[8]), "r"(v[9]), "r"(v[10]), "r"(v[11]), "r"(v[12]), "r"(v[13]), "r"(v[14]),
      "r"(v[15]), "r"(v[16]), "r"(v[17]), "r"(v[18]), "r"(v[19]), "r"(v[20]), "r"(v[21]),
      "r"(v[22]), "r"(v[23]), "r"(v[24]), "r"(v[25]), "r"(v[26]), "r"(v[27]), "r"(v[28]),
      "r"(v[29]), "r"(v[30]), "r"(v[31]));
}
__device__ __forceinline__ void tmem_ld16(uint32_t taddr, uint32_t (&v)[16]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0, %1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, "
      "%12, %13, %14, %15}, [%16];"
      : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]),
        "=r"(v[7]), "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]),
        "=r"(v[14]), "=r"(v[15])
      : "r"(taddr));
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
}
}  // namespace tc

__global__ void __launch_bounds__(192, 1) k5d_tc(DevPlan P, float* __restrict__ gout) {
  using namespace tc;
  extern __shared__ __align__(1024) unsigned char smraw[];
  unsigned char* ring = smraw;                                   // kSlots x (B hi, B lo)
  unsigned char* rawr = smraw + kSlots * kSlot;                  // kRawD x raw A (cp.async)
  uint64_t* full = reinterpret_cast<uint64_t*>(rawr + kRawD * kRawA);   // slot landed (TMA)
  uint64_t* done = full + kSlots;                                // slot's MMAs retired (commit)
  uint64_t* conv = done + kSlots;                                // A buffer written (128 arrivals)
  uint32_t* tslot = reinterpret_cast<uint32_t*>(conv + kABufs);
  const Consts& C = P.C;
  const int t = threadIdx.x, warp = t >> 5;
  const int b = C.b0 + blockIdx.z;
  const int m0 = blockIdx.y * MT, d0 = blockIdx.x * NT;
  const int KP = C.k5tc_kp, nch = KP / KC;
  const int mrows = min(MT, C.n_t - m0);
  const float2* S4 = P.S4 + (size_t)b * C.Kp * C.n_t + m0;
  const unsigned char* Bsrc = reinterpret_cast<const unsigned char*>(P.k5tc_b) + (size_t)blockIdx.x * nch * 2 * kTile;
  uint32_t cs, crank;   // cluster size (along time tiles) and this CTA's rank in it
  asm("mov.u32 %0, %%cluster_nctarank;" : "=r"(cs));
  asm("mov.u32 %0, %%cluster_ctarank;" : "=r"(crank));
  const uint16_t cmask = (uint16_t)((1u << cs) - 1);
  const uint32_t bpiece = 2 * kTile / cs;   // this CTA's share of a chunk's B (multiple of 16 B)
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tslot)), "r"(kTmemCols));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  if (t == 0) {
    for (int i = 0; i < kSlots; ++i) ac::mbar_init(full + i, 1);
    for (int i = 0; i < kSlots; ++i) ac::mbar_init(done + i, cs);
    for (int i = 0; i < kABufs; ++i) ac::mbar_init(conv + i, 128);
    ac::fence_mbar_init();
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  // peers multicast into this CTA's slots and barriers: all barriers initialised cluster-wide first
  cluster_sync();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t tmem = *tslot;
  pdl_wait();
  pdl_trigger();
  if (warp == 0) {
    // ---- producer: chunk ch -> slot ch % kSlots once the MMAs of chunk ch - kSlots retired
    if (t == 0)
      for (int ch = 0; ch < nch; ++ch) {
        const int sl = ch % kSlots;
        if (ch >= kSlots) ac::mbar_wait(done + sl, ((ch - kSlots) / kSlots) & 1);
        unsigned char* dst = ring + sl * kSlot;
        ac::mbar_expect_tx(full + sl, 2 * kTile);
        bulk_mc(dst + crank * bpiece, Bsrc + (size_t)ch * 2 * kTile + crank * bpiece, bpiece, full + sl, cmask);
      }
  } else if (warp == 1) {
    // ---- MMA issuer: 3 TF32 products per K-step of 8, all chunks into one TMEM accumulator
    if (t == 32)
      for (int ch = 0; ch < nch; ++ch) {
        const int sl = ch % kSlots, ab = ch % kABufs;
        ac::mbar_wait(full + sl, (ch / kSlots) & 1);
        ac::mbar_wait(conv + ab, (ch / kABufs) & 1);
        asm volatile("tcgen05.fence::after_thread_sync;");
        const uint32_t ta = tmem + NT + ab * 2 * KC, b0 = smem_u32(ring + sl * kSlot);
#pragma unroll
        for (int k8 = 0; k8 < KC / 8; ++k8) {
          const uint32_t off = k8 * 2 * kLBO;
          const uint32_t ah = ta + k8 * 8, al = ta + KC + k8 * 8;
          const uint64_t bh = desc_kmajor(b0 + off), bl = desc_kmajor(b0 + kTile + off);
          const bool first = ch == 0 && k8 == 0;
          mma_tf32_ts(tmem, ah, bh, kIdesc, !first);
          mma_tf32_ts(tmem, ah, bl, kIdesc, true);
          mma_tf32_ts(tmem, al, bh, kIdesc, true);
        }
        commit_mc(done + sl, cmask);
      }
  } else {
    // ---- converters (warps 2..5): row m = TMEM lane; raw S4 -> TF32 hi / lo columns of TMEM
    const int quarter = warp & 3, r = 32 * quarter + (t & 31);
    const bool mok = r < mrows;
    const uint32_t tl = tmem + ((uint32_t)(32 * quarter) << 16);
    float2* rawme = reinterpret_cast<float2*>(rawr) + r;   // this row's values: [slot][kl * MT]
    auto issue = [&](int ch) {   // chunk ch's 8 values of row r -> raw slot ch % kRawD
      if (ch < nch && mok) {
        const int k0 = ch * (KC / 2);
        float2* d = rawme + (ch % kRawD) * (KC / 2) * MT;
#pragma unroll
        for (int kl = 0; kl < KC / 2; ++kl)
          if (k0 + kl < C.Kp)
            asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(smem_u32(d + kl * MT)),
                         "l"(S4 + (size_t)(k0 + kl) * C.n_t + r) : "memory");
      }
      asm volatile("cp.async.commit_group;" ::: "memory");
    };
#pragma unroll 1
    for (int c = 0; c < kRawD; ++c) issue(c);
    for (int ch = 0; ch < nch; ++ch) {
      const int ab = ch % kABufs;
      asm volatile("cp.async.wait_group %0;" ::"n"(kRawD - 1) : "memory");
      // A buffer ab was last read by the MMAs of chunk ch - kABufs (committed to its slot)
      if (ch >= kABufs) ac::mbar_wait(done + (ch - kABufs) % kSlots, ((ch - kABufs) / kSlots) & 1);
      const float2* raw = rawme + (ch % kRawD) * (KC / 2) * MT;
      const int k0 = ch * (KC / 2);
      uint32_t v[2 * KC];   // [0, KC): hi, [KC, 2 KC): lo; column j = k' = 2 (k - k0) + re/im
#pragma unroll
      for (int kl = 0; kl < KC / 2; ++kl) {
        const float2 x = (mok && k0 + kl < C.Kp) ? raw[kl * MT] : make_float2(0.f, 0.f);
        const float hx = tf32_hi(x.x), hy = tf32_hi(x.y);
        v[2 * kl] = __float_as_uint(hx);
        v[2 * kl + 1] = __float_as_uint(hy);
        v[KC + 2 * kl] = __float_as_uint(x.x - hx);
        v[KC + 2 * kl + 1] = __float_as_uint(x.y - hy);
      }
      tmem_st32(tl + NT + ab * 2 * KC, v);
      asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
      asm volatile("tcgen05.fence::before_thread_sync;");
      asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(conv + ab)) : "memory");
      issue(ch + kRawD);   // this thread has consumed its values of raw slot ch % kRawD
    }
  }
  if (warp < 2) {   // the producer / issuer warps only hold the TMEM allocation
    __syncwarp();
    asm volatile("tcgen05.fence::before_thread_sync;");
    // no CTA leaves while a peer may still multicast into its shared memory / barriers
    cluster_sync();
    if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(kTmemCols));
    return;
  }
  ac::mbar_wait(done + (nch - 1) % kSlots, ((nch - 1) / kSlots) & 1);
  asm volatile("tcgen05.fence::after_thread_sync;");
  // epilogue: warp w may read TMEM lanes 32 (w % 4) .. + 31 (rows m); 128 columns (d) in 4 x 32
  const int quarter = warp & 3, row = 32 * quarter + (t & 31), m = m0 + row;
#pragma unroll 1
  for (int cb = 0; cb < NT / 32; ++cb) {
    uint32_t v[32];
    const uint32_t ta = tmem + ((uint32_t)(32 * quarter) << 16) + cb * 32;
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0, %1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, "
        "%12, %13, %14, %15, %16, %17, %18, %19, %20, %21, %22, %23, %24, %25, %26, %27, %28, %29, "
        "%30, %31}, [%32];"
        : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]),
          "=r"(v[7]), "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]),
          "=r"(v[14]), "=r"(v[15]), "=r"(v[16]), "=r"(v[17]), "=r"(v[18]), "=r"(v[19]), "=r"(v[20]),
          "=r"(v[21]), "=r"(v[22]), "=r"(v[23]), "=r"(v[24]), "=r"(v[25]), "=r"(v[26]), "=r"(v[27]),
          "=r"(v[28]), "=r"(v[29]), "=r"(v[30]), "=r"(v[31])
        : "r"(ta));
    asm volatile("tcgen05.wait::ld.sync.aligned;");
    if (m < C.n_t) {
      const int dc = d0 + cb * 32;
      const size_t o = ((size_t)b * C.n_t + m) * C.n_det + dc;
      if (dc + 32 <= C.n_det && (C.n_det & 3) == 0) {
#pragma unroll
        for (int i = 0; i < 32; i += 4) {
          float4 w;
          w.x = epi_fwd(P, o + i, __uint_as_float(v[i]));
          w.y = epi_fwd(P, o + i + 1, __uint_as_float(v[i + 1]));
          w.z = epi_fwd(P, o + i + 2, __uint_as_float(v[i + 2]));
          w.w = epi_fwd(P, o + i + 3, __uint_as_float(v[i + 3]));
          *reinterpret_cast<float4*>(gout + o + i) = w;
        }
      } else {
#pragma unroll
        for (int i = 0; i < 32; ++i)
          if (dc + i < C.n_det) gout[o + i] = epi_fwd(P, o + i, __uint_as_float(v[i]));
      }
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  cluster_sync();
}

size_t smem_k5d_tc() {
  return (size_t)tc::kSlots * tc::kSlot + tc::kRawD * tc::kRawA + 16 * tc::kSlots + 8 * tc::kABufs + 16;
}

// ================================================================== K5dT on tcgen05 (3xTF32)
// The analysis as a GEMM D[m][j] = sum_d A[m][d] B[d][j]: A = g (the traces, K-major: detectors
// contiguous), B[d][2k] = Re E5T[k][d], B[d][2k+1] = -Im E5T[k][d] (host-packed TF32 hi / lo,
// N tile nt = 2 (K+1) split into C.k5ttc_nb blocks of C.k5ttc_nt <= 256 columns), D[m][2k + c]
// = (Re, Im) S4[k][m].  The same 6-warp pipeline as k5d_tc: warp 0 multicasts B chunks (16
// detectors) across the cluster, warps 2..5 cp.async their row's 16 trace values (kRawD
// chunks ahead), split them hi / lo into TMEM, warp 1 issues the 6 MMAs per chunk (M 128, N nt,
// K 8; A from TMEM).  Epilogue: (Re, Im) column pairs of lane m -> S4[k][m] (coalesced in m).
namespace tct {
constexpr int MT = 128, KC = kK5tcKC, kSlots = 4, kABufs = 4, kRawD = 8, kNTMax = 256;
constexpr uint32_t kRawA = MT * KC * 4;            // 16 trace values of 128 rows (8 KB)
constexpr uint32_t kSlotMax = 2 * kNTMax * KC * 4; // B hi + lo at the widest tile (32 KB)
constexpr uint32_t kTmemCols = 512;                // accumulator [0, 256) + A buffers [256, 384)
}  // namespace tct

__global__ void __launch_bounds__(192, 1) k5dt_tc(DevPlan P, const float* __restrict__ gin) {
  using namespace tct;
  extern __shared__ __align__(1024) unsigned char smraw[];
  const Consts& C = P.C;
  const int NTa = C.k5ttc_nt;                                   // columns of this N tile
  const uint32_t slotb = (uint32_t)NTa * KC * 4 * 2;            // B hi + lo bytes per chunk
  unsigned char* ring = smraw;                                   // kSlots x (B hi, B lo)
  unsigned char* rawr = smraw + kSlots * kSlotMax;               // kRawD x raw A (cp.async)
  uint64_t* full = reinterpret_cast<uint64_t*>(rawr + kRawD * kRawA);
  uint64_t* done = full + kSlots;
  uint64_t* conv = done + kSlots;
  uint32_t* tslot = reinterpret_cast<uint32_t*>(conv + kABufs);
  const int t = threadIdx.x, warp = t >> 5;
  const int b = C.b0 + blockIdx.z;
  const int m0 = blockIdx.y * MT, n0 = blockIdx.x * NTa;
  const int nch = C.k5ttc_kp / KC;
  const int mrows = min(MT, C.n_t - m0);
  const unsigned char* Bsrc = reinterpret_cast<const unsigned char*>(P.k5ttc_b) + (size_t)blockIdx.x * nch * slotb;
  uint32_t cs, crank;
  asm("mov.u32 %0, %%cluster_nctarank;" : "=r"(cs));
  asm("mov.u32 %0, %%cluster_ctarank;" : "=r"(crank));
  const uint16_t cmask = (uint16_t)((1u << cs) - 1);
  const uint32_t bpiece = slotb / cs;
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(tc::smem_u32(tslot)), "r"(kTmemCols));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  if (t == 0) {
    for (int i = 0; i < kSlots; ++i) ac::mbar_init(full + i, 1);
    for (int i = 0; i < kSlots; ++i) ac::mbar_init(done + i, cs);
    for (int i = 0; i < kABufs; ++i) ac::mbar_init(conv + i, 128);
    ac::fence_mbar_init();
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  tc::cluster_sync();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t tmem = *tslot;
  pdl_wait();
  pdl_trigger();
  if (warp == 0) {
    if (t == 0)
      for (int ch = 0; ch < nch; ++ch) {
        const int sl = ch % kSlots;
        if (ch >= kSlots) ac::mbar_wait(done + sl, ((ch - kSlots) / kSlots) & 1);
        ac::mbar_expect_tx(full + sl, slotb);
        tc::bulk_mc(ring + sl * kSlotMax + crank * bpiece, Bsrc + (size_t)ch * slotb + crank * bpiece, bpiece,
                    full + sl, cmask);
      }
  } else if (warp == 1) {
    if (t == 32) {
      const uint32_t idesc = tc::idesc_tf32(MT, NTa);
      for (int ch = 0; ch < nch; ++ch) {
        const int sl = ch % kSlots, ab = ch % kABufs;
        ac::mbar_wait(full + sl, (ch / kSlots) & 1);
        ac::mbar_wait(conv + ab, (ch / kABufs) & 1);
        asm volatile("tcgen05.fence::after_thread_sync;");
        const uint32_t ta = tmem + kNTMax + ab * 2 * KC, b0 = tc::smem_u32(ring + sl * kSlotMax);
        const uint32_t btile = (uint32_t)NTa * KC * 4;
#pragma unroll
        for (int k8 = 0; k8 < KC / 8; ++k8) {
          const uint32_t off = k8 * 2 * tc::kLBO;
          const uint64_t bh = tc::desc_kmajor(b0 + off), bl = tc::desc_kmajor(b0 + btile + off);
          const bool first = ch == 0 && k8 == 0;
          tc::mma_tf32_ts(tmem, ta + k8 * 8, bh, idesc, !first);
          tc::mma_tf32_ts(tmem, ta + k8 * 8, bl, idesc, true);
          tc::mma_tf32_ts(tmem, ta + KC + k8 * 8, bh, idesc, true);
        }
        tc::commit_mc(done + sl, cmask);
      }
    }
  } else {
    const int quarter = warp & 3, r = 32 * quarter + (t & 31);
    const bool mok = r < mrows;
    const uint32_t tl = tmem + ((uint32_t)(32 * quarter) << 16);
    const float* grow = gin + ((size_t)b * C.n_t + m0 + r) * C.n_det;
    const bool vec = (C.n_det & 3) == 0;
    const int sw = (r >> 1) & 3;   // 16-B group swizzle: conflict-free LDS.128 read-back
    unsigned char* rawme = rawr + r * KC * 4;
    auto issue = [&](int ch) {
      if (ch < nch && mok) {
        unsigned char* d = rawme + (ch % kRawD) * kRawA;
        const int d0 = ch * KC;
        if (vec) {
#pragma unroll
          for (int q = 0; q < KC / 4; ++q)
            if (d0 + 4 * q < C.n_det)
              asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(tc::smem_u32(d + 16 * (q ^ sw))),
                           "l"(grow + d0 + 4 * q) : "memory");
        } else {
#pragma unroll
          for (int i = 0; i < KC; ++i)
            if (d0 + i < C.n_det)
              asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" ::"r"(tc::smem_u32(d + 16 * ((i >> 2) ^ sw) + 4 * (i & 3))),
                           "l"(grow + d0 + i) : "memory");
        }
      }
      asm volatile("cp.async.commit_group;" ::: "memory");
    };
#pragma unroll 1
    for (int c = 0; c < kRawD; ++c) issue(c);
    for (int ch = 0; ch < nch; ++ch) {
      const int ab = ch % kABufs;
      asm volatile("cp.async.wait_group %0;" ::"n"(kRawD - 1) : "memory");
      if (ch >= kABufs) ac::mbar_wait(done + (ch - kABufs) % kSlots, ((ch - kABufs) / kSlots) & 1);
      const unsigned char* raw = rawme + (ch % kRawD) * kRawA;
      const int d0 = ch * KC;
      uint32_t v[2 * KC];
#pragma unroll
      for (int q = 0; q < KC / 4; ++q) {
        float4 x = *reinterpret_cast<const float4*>(raw + 16 * (q ^ sw));
        const float xs[4] = {x.x, x.y, x.z, x.w};
#pragma unroll
        for (int e = 0; e < 4; ++e) {
          const float xv = (mok && d0 + 4 * q + e < C.n_det) ? xs[e] : 0.f;
          const float h = tc::tf32_hi(xv);
          v[4 * q + e] = __float_as_uint(h);
          v[KC + 4 * q + e] = __float_as_uint(xv - h);
        }
      }
      tc::tmem_st32(tl + kNTMax + ab * 2 * KC, v);
      asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
      asm volatile("tcgen05.fence::before_thread_sync;");
      asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(tc::smem_u32(conv + ab)) : "memory");
      issue(ch + kRawD);
    }
  }
  if (warp < 2) {
    __syncwarp();
    asm volatile("tcgen05.fence::before_thread_sync;");
    tc::cluster_sync();
    if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(kTmemCols));
    return;
  }
  ac::mbar_wait(done + (nch - 1) % kSlots, ((nch - 1) / kSlots) & 1);
  asm volatile("tcgen05.fence::after_thread_sync;");
  const int quarter = warp & 3, row = 32 * quarter + (t & 31), m = m0 + row;
  float2* S4 = P.S4 + (size_t)b * C.Kp * C.n_t;
#pragma unroll 1
  for (int cb = 0; cb < NTa / 16; ++cb) {
    uint32_t v[16];
    tc::tmem_ld16(tmem + ((uint32_t)(32 * quarter) << 16) + cb * 16, v);
    if (m < C.n_t) {
#pragma unroll
      for (int q = 0; q < 8; ++q) {
        const int k = (n0 + cb * 16) / 2 + q;
        if (k < C.Kp) S4[(size_t)k * C.n_t + m] = make_float2(__uint_as_float(v[2 * q]), __uint_as_float(v[2 * q + 1]));
      }
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  tc::cluster_sync();
}

size_t smem_k5dt_tc() {
  return (size_t)tct::kSlots * tct::kSlotMax + tct::kRawD * tct::kRawA + 16 * tct::kSlots + 8 * tct::kABufs + 16;
}

// launch with a (1, cs, 1) cluster along the time tiles (B multicast) and optional PDL
template <typename Kern, typename Arg>
static cudaError_t launch_cluster(const Consts& C, Kern kern, dim3 grid, size_t smem, cudaStream_t s,
                                  const DevPlan& P, Arg a) {
  const int cs = grid.y % 4 == 0 ? 4 : grid.y % 2 == 0 ? 2 : 1;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = dim3(192);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute at[2];
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = 1;
  at[0].val.clusterDim.y = cs;
  at[0].val.clusterDim.z = 1;
  at[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[1].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = at;
  cfg.numAttrs = C.pdl ? 2 : 1;
  const cudaError_t e = cudaLaunchKernelEx(&cfg, kern, P, a);
  return e != cudaSuccess ? e : cudaGetLastError();
}

cudaError_t launch_k5d_tc(const DevPlan& P, float* g, cudaStream_t s) {
  const Consts& C = P.C;
  const dim3 grid((C.n_det + tc::NT - 1) / tc::NT, (C.n_t + tc::MT - 1) / tc::MT, C.batch);
  return launch_cluster(C, k5d_tc, grid, smem_k5d_tc(), s, P, g);
}

cudaError_t launch_k5dt_tc(const DevPlan& P, const float* g, cudaStream_t s) {
  const Consts& C = P.C;
  const dim3 grid(C.k5ttc_nb, (C.n_t + tct::MT - 1) / tct::MT, C.batch);
  return launch_cluster(C, k5dt_tc, grid, smem_k5dt_tc(), s, P, g);
}

cudaError_t configure_dense_kernels(const Consts& C) {
  if (!C.dense) return cudaSuccess;
  cudaError_t e = cudaFuncSetAttribute(k5d_tc, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem_k5d_tc());
  if (e == cudaSuccess)
    e = cudaFuncSetAttribute(k5dt_tc, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem_k5dt_tc());
  return e;
}

}  // namespace tat
