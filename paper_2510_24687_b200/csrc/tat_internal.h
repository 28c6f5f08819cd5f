// Internal declarations shared by the host plan builder and the sm_100a kernels.
// Nothing here is part of the public ABI (see include/tat.h).
#pragma once
#include <algorithm>
#include <cstddef>
#include <cstdint>
#include <string>
#include <vector>
#include <cuda.h>
#include <cuda_runtime.h>

namespace tat {

// Derived constants of the discretisation (D0).
struct Consts {
  int n = 0, n_det = 0, n_t = 0, batch = 0;
  int b0 = 0;       // first image of a launch (sub-batch pipelining); batch = images in it
  int dct_sine = 0; // K4T computes sum_m G~ sin(c lambda_j t_m) (the inverse, Alg. 3 step 3)
  int pdl = 1;      // launch the chain kernels with programmatic dependent launch
  int dense = 0;    // detectors off any canonical ring: K5 / K5T as dense sums (reading G24)
  int k5tc_kp = 0;  // dense K5 on tcgen05: padded K' = 2 (K+1) rounded up to kK5tcKC (0: SIMT path)
  int k5ttc_kp = 0; // dense K5T on tcgen05: n_det rounded up to kK5tcKC (0: SIMT path)
  int k5ttc_nt = 0; // its N tile (<= 256, multiple of 16) and number of N tiles over 2 (K+1)
  int k5ttc_nb = 0;
  int col_strip = 16; // K2: columns per CTA (k2c_fwd recomputes one halo column;
                      // 12-16 measured best at C3, 20-32 slower)
  int col_strip_adj = 16; // K2Tb (k2c_adj): columns per CTA
  int ring2 = -1;   // two-stage ring kernels (n_ring 256 / 512) instead of the Stockham ones: bit
                    // mask (ring2_on), -1 = auto (all; K5 at n_ring = 512 stays Stockham: 21.8 vs
                    // 22.0 us at C3, while at 256 the two-stage K5 wins: 24.1 -> 22.3 at C4)
  double R = 1, c = 1, T = 1;
  double h = 0, T_new0 = 0, T_new = 0, Lbox = 0, dxi = 0, dt = 0, dlam = 0, lam_max = 0;
  double wJ = 1, omega = 0;
  double lowk_c = 0;   // reading G25: (dlam^2 / 12) (h^2 / 2 pi)
  int N = 0;        // Cartesian FFT size
  int Lres = 0;     // residues N / n (oversampling factor, power of two)
  int log2L = 0;
  int M = 0;        // DCT-I length; 2M-point FFT
  int J = 0, NL = 0;
  int n_ring = 0, K = 0, Kp = 0, half = 0;
  int ncols = 0;    // N/2 + 1 Cartesian columns kept (p in [0, N/2])
  int ntargets = 0; // K2T: distinct Cartesian targets (p, q) of the transposed bilinear
  int s1boxP = 0;   // TMA box extent along p for S1 tiles (box = {4 y, s1boxP p, 1})
  int ntpad = 0;    // per-image stride of Rc (ntargets rounded up to even: 16-B bulk copies)
  int k2c_rbuf = 0; // k2c_adj: entries per column target buffer (max targets per column + 2)
  int k2t_win = 0;  // k2t_sum: max nodes with p0 in {p-1, p} over columns p
  int k2f = 0;      // adjoint column stage: 0 k2t_sum + k2c_adj; 1 fused k2c_adjf;
                    // 2 k2t_sumf (multi-image target sums on k2c_adjf's tables) + k2c_adj
  int k2f_rcap = 0; // k2c_adjf: shared-memory capacity for a column's records (multiple of 4)
  int k2f_wcap = 0; // ... and for one image's node window (even); larger columns read global
  int k2f_ipc = 0;  // ... images per CTA (the records of a column are staged once per CTA)
  int k2f_nslow = 0; // ... columns run from global memory, one image per CTA (k2f_cols head)
  int k2s_n = 0;     // k2t_strip: number of strips; k2s_wcap: largest strip window (nodes, even)
  int k2s_wcap = 0;
  int k2s_ipc = 0;   // k2t_strip: images per CTA (the strip's records stay in registers)
  int k2s_ovcap = 0; // k2t_strip: smem bytes for a light strip's overflow lists
  int k2s_nheavy = 0; // k2t_strip: leading heavy strips, one image per CTA
};


// Host-side tables (float64 built, float32/int stored), uploaded by tat_plan_create.
struct HostTables {
  std::vector<float> mult;          // [Kp][NL]: (h^2/2pi)(1/n_phi) w_j dlam lam_j J_k(R lam_j)
  std::vector<float2> tw_n;         // n roots exp(-2 pi i k / n)
  std::vector<float2> tw_pre;       // [Lres][n]: exp(-2 pi i s y'' / N) at FFT slot y' = y'' mod n
  std::vector<float2> tw_ring;      // n_ring roots
  std::vector<float2> tw_dct;       // 2M roots
  std::vector<float2> tw_col;       // [Lres][n]: exp(-2 pi i s (y - n/2) / N) (kernels_col.cu)
  std::vector<float2> tw_dct4;      // [4][n]: exp(-2 pi i s i' / 4n) (kernels_col.cu K4/K4T)
  // K2 forward gather: half-plane nodes sorted by p0
  std::vector<int> k2_colptr;       // [ncols + 1]
  std::vector<int4> k2_nodes;       // (l'*NL + j, q0, alpha bits, beta bits), sorted by p0
  std::vector<int> node_perm;       // [NL][n_ring/2]: (j, l') -> adjoint S2 position
  std::vector<int2> k3t_dst;        // K3T: per ring group, (adjoint position, jj << 11 | l') sorted
  // K2T transposed gather: per column p, targets (q mod N) with entry ranges
  std::vector<int> k2t_colptr;      // [ncols + 1] into targets
  std::vector<int> k2t_tq;          // [T] q mod N
  std::vector<int> k2t_tstart;      // [T + 1] into entries (host only: builds k2t_rec)
  std::vector<int2> k2t_ent;        // [E] (src sorted node position, weight bits) (host only)
  // per target: (src0, w0 bits, src1, w1 bits); one entry: src1 = src0, w1 = 0; more than
  // two: (src0, w0 bits, -(k+1), count) with entries 1..count-1 at k2t_ov[k ..]
  std::vector<int4> k2t_rec;        // [T]
  std::vector<int2> k2t_ov;         // overflow entries (src, w bits)
  std::vector<int> ring;            // [n_det] (-1 in dense mode)
  // dense mode: E5[k][d] = c_k (cos, sin)(s_k k theta_d), E5T without c_k (s_K = -1, c = 1, 2, 1)
  std::vector<float2> dense_e5, dense_e5t;   // [Kp][n_det]
  std::vector<float> k5ttc_b;                // tcgen05 K5dT operand B (hi / lo TF32 parts, packed)
  std::vector<float> k5tc_b;                 // tcgen05 K5d operand B (hi / lo TF32 parts, packed)
  // k2c_adj: per (column p, q0 = q mod 16L): bit q1 set if target (p, q0 + 16L q1) exists,
  // and the index of the first such target (targets of a column are ordered by (q0, q1))
  std::vector<uint32_t> k2c_mask;   // [ncols][16L] (only when col_ok)
  std::vector<int> k2c_base;        // [ncols][16L]
  // k2c_adjf (fused adjoint column stage): window-relative target records, 3 words each
  std::vector<uint32_t> k2f_rec;    // {i0 | i1 << 16, w0 bits, w1 bits}, column blocks padded to 4
  std::vector<int> k2f_recptr;      // [ncols + 1] first record of each column (empty: not fused)
  std::vector<int2> k2f_ov;         // overflow entries (window offset, w bits)
  std::vector<int4> k2f_ovt;        // targets with > 2 entries: (index in column, first entry, count, 0)
  std::vector<int> k2f_ovptr;       // [ncols + 1] into k2f_ovt
  // k2t_strip (streaming transposed bilinear): column strips (window start, window nodes,
  // first target, targets), strip-relative records as k2f_rec, overflow lists per strip
  std::vector<int4> k2s_strip;      // empty: not available
  std::vector<uint32_t> k2s_rec;
  std::vector<int4> k2s_ovt;        // (target in strip, first entry, count, 0)
  std::vector<int2> k2s_ov;
  std::vector<int> k2s_ovptr;       // [strips + 1] into k2s_ovt (host only, in build order)
  std::vector<int2> k2s_ovr;        // [strips] overflow range of each strip (device order)
  int k2s_nheavy = 0;               // heavy strips, placed first (one image per CTA)
  int k2s_ovcap = 0;                // smem budget for a light strip's overflow lists (bytes)
};
#ifndef TAT_STRIP_NODES
#define TAT_STRIP_NODES 4096
#endif
#ifndef TAT_STRIP_TARGETS
#define TAT_STRIP_TARGETS 2560
#endif
constexpr int kStripNodes = TAT_STRIP_NODES;     // k2t_strip: node-window budget of a strip
constexpr int kStripTargets = TAT_STRIP_TARGETS; // ... and its target budget (<= 256 KR)
// ... and for its overflow lists (descriptors + entries, staged in smem); measured at C3 / C5:
// 8 KB -> K2Ta 93 / 142 us, 16 KB -> 65.5 / 93, 24 KB -> 68.6 / 81 (fewer heavy strips vs
// occupancy)
inline int strip_ov_bytes(int n) { return n >= 1024 ? 24576 : 16384; }
// two-stage ring kernels (kernels_ring2.cu, n_ring in {256, 512, 1024}): transforms (ring pairs)
// per CTA (ring2_G), hence rings per K3T CTA (k3t_dst groups)
__host__ __device__ constexpr int ring2_G(int n_ring) { return n_ring >= 1024 ? 8 : 16; }
// C.ring2 bits: 1 K3, 2 K3T, 4 K5, 8 K5T
inline bool ring2_size_ok(int n_ring) { return n_ring == 256 || n_ring == 512 || n_ring == 1024; }
inline bool ring2_on(const Consts& C, int bit) {
  const int m = C.ring2 >= 0 ? C.ring2 : (C.n_ring == 512 ? 11 : 15);
  return (m & bit) && ring2_size_ok(C.n_ring);
}
inline int k3t_group_rings(const Consts& C) {
  return ring2_on(C, 2) ? 2 * ring2_G(C.n_ring) : 2 * std::min(4096 / C.n_ring, 16);
}

// returns "" on success, else an error message; code receives 1 (invalid) or 2 (unsupported)
std::string derive_consts(int n, int n_det, int n_t, double R, double c, double T, int batch,
                          const double* angles, Consts& out, std::vector<int>& ring, int& code);
std::string gpu_support(const Consts& C);    // "" if the sm_100a kernels implement C
void build_tables(const Consts& C, const std::vector<int>& ring, const double* angles,
                  HostTables& H);
void bessel_row(double x, int kmax, double* out);   // J_0..J_kmax(x), Miller recurrence

// Device-side view of a plan (pointers into device memory).
struct DevPlan {
  Consts C;
  // tables
  const float* mult = nullptr;
  const float2* tw_n = nullptr;
  const float2* tw_pre = nullptr;
  const float2* tw_ring = nullptr;
  const float2* tw_dct = nullptr;
  const float2* tw_col = nullptr;
  const float2* tw_dct4 = nullptr;
  const int* k2_colptr = nullptr;
  const int4* k2_nodes = nullptr;
  const int* node_perm = nullptr;
  const int2* k3t_dst = nullptr;
  const int* k2t_colptr = nullptr;
  const int* k2t_tq = nullptr;
  const int4* k2t_rec = nullptr;
  const int2* k2t_ov = nullptr;
  const int* ring = nullptr;
  const uint32_t* k2c_mask = nullptr;
  const int* k2c_base = nullptr;
  const uint32_t* k2f_rec = nullptr;  // fused adjoint column stage tables (HostTables)
  const int* k2f_recptr = nullptr;
  const int2* k2f_ov = nullptr;
  const int4* k2f_ovt = nullptr;
  const int* k2f_ovptr = nullptr;
  const int* k2f_cols = nullptr;      // [ncols] column order of the grid: slow columns first
  const int4* k2s_strip = nullptr;    // k2t_strip tables (HostTables)
  const uint32_t* k2s_rec = nullptr;
  const int4* k2s_ovt = nullptr;
  const int2* k2s_ov = nullptr;
  const int2* k2s_ovr = nullptr;
  // inverse (Alg. 3 step 5): per Cartesian target 4 polar corners (sorted node index, or
  // -(index + 1) for the conjugate mirror node) and bilinear weights
  const float2* dense_e5 = nullptr;
  const float2* dense_e5t = nullptr;
  const float* k5ttc_b = nullptr;  // tcgen05 K5dT operand B: [n block][chunk][hi, lo][nt x 16 core layout]
  const float* k5tc_b = nullptr;   // tcgen05 K5d operand B: [d block][chunk][hi, lo][128 x 32 core layout]
  const int4* inv_nodes = nullptr;
  const float4* inv_w = nullptr;
  // workspace
  float2* S1 = nullptr;   // [B][ncols][n]
  float2* S2 = nullptr;   // [B][half * NL]: forward ring-major [j][l'], adjoint K2 node order
  float2* S3 = nullptr;   // [B][Kp][NL]
  float2* S4 = nullptr;   // [B][Kp][n_t]
  float2* Rc = nullptr;   // [B][ntpad]: K2T target sums (transposed bilinear), column order
  // epilogue of the last stage of a launch (fused iterative-driver steps, tat_residual /
  // tat_adjoint_step): forward stores A f - epi_sub when epi_sub != nullptr; adjoint with
  // epi_update != 0 stores f <- f - epi_tau (A* g) in place, then max(0, .) if epi_update == 2,
  // then times epi_roi[iy][ix] if epi_roi != nullptr.
  const float* epi_sub = nullptr;
  const float* epi_roi = nullptr;
  float epi_scale = 1.f;   // forward: stores epi_scale * (A f) (- epi_sub)
  float epi_tau = 0.f;
  int epi_update = 0;
  // tat_nnls_converge: per-image flags [batch]; an image whose flag is 0 keeps its iterate (the
  // update epilogue stores nothing for it).  nullptr: every image is updated.
  const int* epi_active = nullptr;
  // low-harmonic quadrature variant (reading G25; tat_plan_set_quadrature): when set, [batch]
  // per-image constants (coef * sum of the call's input image / data), written by k_lowk_sum
  // at the start of each forward / adjoint call and added to every output in the epilogues
  float* lowk_add = nullptr;
  double* lowk_part = nullptr;        // [batch][32] partial sums (k_lowk_sum)
  unsigned int* lowk_cnt = nullptr;   // [batch] finished-part counters (kept at 0 between calls)
  // inverse (tat_inverse): the Cartesian targets of column p are the whole chord |q| <= Q_p of
  // the disk, stored in natural q order; k2c_adj then reads them by index (no mask / base)
  const int* k2c_chord = nullptr;
  // de-apodised bilinear variant (reading G26; tat_plan_set_interpolation): [n] factors
  // 1 / sinc^2(x_i / 2L); K1 scales f[iy][ix] by d[ix] d[iy], K1T's epilogue its output likewise
  const float* deapod = nullptr;
};

#ifdef __CUDACC__
// Programmatic dependent launch (sm_90+): a kernel launched with the PDL attribute may start
// while its predecessor in the stream drains; everything before pdl_wait() (plan-table loads,
// shared-memory and barrier setup) overlaps the predecessor's tail, and pdl_wait() blocks until
// the predecessor has completed and its memory is visible.  Both are no-ops without PDL.
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void pdl_trigger() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }

template <class... KArgs, class... Args>
cudaError_t launch_pdl(bool pdl, void (*kern)(KArgs...), dim3 grid, dim3 block, size_t smem,
                       cudaStream_t s, Args... args) {
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = at;
  cfg.numAttrs = pdl ? 1 : 0;
  return cudaLaunchKernelEx(&cfg, kern, args...);
}

// forward epilogue: value at flat output index i of g
// VAR = false: the kernel was instantiated for plans without the G25 / G26 variants
// as epi_fwd with epi_sub[i] already loaded (sub; 0 when there is no subtraction)
template <bool VAR = true>
__device__ __forceinline__ float epi_fwd_pre(const DevPlan& P, size_t i, float v, float sub) {
  if (VAR && P.lowk_add) v += P.lowk_add[i / ((size_t)P.C.n_t * P.C.n_det)];
  return v * P.epi_scale - sub;
}
template <bool VAR = true>
__device__ __forceinline__ float epi_fwd(const DevPlan& P, size_t i, float v) {
  if (VAR && P.lowk_add) v += P.lowk_add[i / ((size_t)P.C.n_t * P.C.n_det)];
  v *= P.epi_scale;
  return P.epi_sub ? v - __ldg(&P.epi_sub[i]) : v;
}
// adjoint epilogue: store value v of A* g at flat index i of f (pixel ixy = i mod n^2)
// as epi_adj_store with the update's inputs already at hand: fold = f[i], roi = epi_roi[ixy]
// (staged in shared memory by the caller); `active` = epi_active of the image
template <bool VAR = true>
__device__ __forceinline__ void epi_adj_store_pre(const DevPlan& P, float* f, size_t i, int ixy, float v,
                                                  float fold, float roi, bool active) {
  if (VAR && P.lowk_add) v += P.lowk_add[i / ((size_t)P.C.n * P.C.n)];
  if (VAR && P.deapod) v *= P.deapod[ixy % P.C.n] * P.deapod[ixy / P.C.n];
  if (!active) return;
  float o = fold - P.epi_tau * v;
  if (P.epi_update == 2) o = fmaxf(o, 0.f);
  f[i] = o * roi;
}
template <bool VAR = true>
__device__ __forceinline__ void epi_adj_store(const DevPlan& P, float* f, size_t i, int ixy, float v) {
  if (VAR && P.lowk_add) v += P.lowk_add[i / ((size_t)P.C.n * P.C.n)];
  if (VAR && P.deapod) v *= P.deapod[ixy % P.C.n] * P.deapod[ixy / P.C.n];
  if (P.epi_update) {
    if (P.epi_active && !__ldg(&P.epi_active[i / ((size_t)P.C.n * P.C.n)])) return;
    float o = f[i] - P.epi_tau * v;
    if (P.epi_update == 2) o = fmaxf(o, 0.f);
    if (P.epi_roi) o *= __ldg(&P.epi_roi[ixy]);
    f[i] = o;
  } else {
    f[i] = v;
  }
}
#endif

// Launchers (kernels.cu).  ev != nullptr: record ev[i] before stage i and ev[5] at the end
// (adjoint: ev[6] between the two K2T kernels).
constexpr int kProfEv = 7;
// Every kernel's dynamic shared-memory attribute is set to this device-wide limit (never to a
// per-plan size): the attribute is process-global, so a later plan with smaller tables must not
// lower the limit an earlier plan's launches rely on.  Launch sizes are checked against it.
constexpr int kSmemLimit = 227 * 1024;
cudaError_t launch_forward(const DevPlan& P, const CUtensorMap& tm, const float* f, float* g,
                           cudaStream_t s, cudaEvent_t* ev);
cudaError_t launch_adjoint(const DevPlan& P, const CUtensorMap& tm, const float* g, float* f,
                           cudaStream_t s, cudaEvent_t* ev);
cudaError_t configure_kernels(const DevPlan& P);   // smem attributes
// kernels_fft.cu: residue-FFT kernels K1, K2, K2T, K1T
cudaError_t configure_fft_kernels(const Consts& C);
size_t smem_fft4(const Consts& C);
// S1 viewed as a 3-D tensor {n (y), ncols (p), batch} of 8-byte elements; TMA box {4, 256, 1}
constexpr int kS1BoxY = 4;
cudaError_t make_s1_tensor_map(const DevPlan& P, CUtensorMap* out, bool blocked);   // forward (blocked) / column-major
cudaError_t launch_k1(const DevPlan& P, const CUtensorMap& tm, const float* f, cudaStream_t s);
cudaError_t launch_k2(const DevPlan& P, const CUtensorMap& tm, cudaStream_t s);
cudaError_t launch_k2t(const DevPlan& P, cudaStream_t s, cudaEvent_t mid = nullptr);   // target sums + column IDFT
cudaError_t launch_k2tb(const DevPlan& P, cudaStream_t s);  // column IDFT of the targets in Rc
cudaError_t launch_k1t(const DevPlan& P, const CUtensorMap& tm, float* f, cudaStream_t s);
// kernels_ring.cu: K3, K3T, K5, K5T on n_phi-point register FFTs
bool ring_fast_ok(const Consts& C);
size_t smem_ring_fast(const Consts& C);
cudaError_t configure_ring_kernels(const Consts& C);
cudaError_t configure_ring2_kernels(const Consts& C);
// two-stage ring kernels: which = 1 K3, 2 K3T, 4 K5 (g out), 8 K5T (g in)
cudaError_t launch_ring2(const DevPlan& P, int which, const float* gin, float* gout, cudaStream_t s);
cudaError_t launch_k3(const DevPlan& P, cudaStream_t s);
cudaError_t launch_k3t(const DevPlan& P, cudaStream_t s);
cudaError_t launch_k5(const DevPlan& P, float* g, cudaStream_t s);
cudaError_t launch_k5t(const DevPlan& P, const float* g, cudaStream_t s);
// kernels_dct.cu: K4, K4T as r residue FFTs of size 2M / r
int dct_fast_r(const Consts& C);
size_t smem_dct_fast(const Consts& C);
cudaError_t configure_dct_kernels(const Consts& C);
cudaError_t launch_k4_fast(const DevPlan& P, bool adj, cudaStream_t s);
size_t max_smem_needed(const Consts& C);
// kernels_col.cu: two-stage column transforms (L = 8, n in {256, 512})
bool col_ok(const Consts& C);
int col_R(int n);   // stage-A points per thread of the two-stage engine (Q0 = col_R(n) * L)
size_t smem_k2c_fwd(const Consts& C);
size_t smem_k2c_adj(const Consts& C);
cudaError_t configure_col_kernels(const Consts& C);
cudaError_t launch_k2c_fwd(const DevPlan& P, const CUtensorMap& tm, cudaStream_t s);
cudaError_t launch_k2c_adj(const DevPlan& P, cudaStream_t s);
size_t smem_k2c_adjf(const Consts& C);
cudaError_t launch_k2c_adjf(const DevPlan& P, cudaStream_t s);
size_t smem_k2t_sumf(const Consts& C);
cudaError_t launch_k2t_sumf(const DevPlan& P, cudaStream_t s);
size_t smem_k2t_strip(const Consts& C);
cudaError_t launch_k2t_strip(const DevPlan& P, cudaStream_t s);
bool dct4_ok(const Consts& C);
size_t smem_k4c(const Consts& C);
cudaError_t launch_k4c(const DevPlan& P, bool adj, cudaStream_t s);
cudaError_t launch_k1c_fwd(const DevPlan& P, const CUtensorMap& tm, const float* f, cudaStream_t s);
cudaError_t launch_k1c_adj(const DevPlan& P, const CUtensorMap& tm, float* f, cudaStream_t s);

// kernels_dense.cu: dense angular synthesis / analysis (reading G24)
cudaError_t launch_k5d(const DevPlan& P, float* g, cudaStream_t s);
cudaError_t launch_k5dt(const DevPlan& P, const float* g, cudaStream_t s);
constexpr int kK5tcKC = 16;   // tcgen05 K5d: K' chunk (real values) per pipeline slot
cudaError_t launch_k5d_tc(const DevPlan& P, float* g, cudaStream_t s);
cudaError_t launch_k5dt_tc(const DevPlan& P, const float* g, cudaStream_t s);
cudaError_t configure_dense_kernels(const Consts& C);
// kernels_inv.cu: inverse-specific stages (Alg. 3 steps 5, 7, 8)
constexpr int kInvParts = 64;   // k2i_const partial sums per image (fixed order)
cudaError_t launch_k2i_interp(const DevPlan& P, cudaStream_t s);
cudaError_t launch_k2i_finish(const DevPlan& P, float* f, const unsigned char* region, float* csum,
                              int annulus_count, cudaStream_t s);
// host tables of the inverse (built on first use)
struct InvTables {
  std::vector<float> mult;          // [Kp][NL]: (dxi^2/2pi)(1/n_phi) dt (-2 J'_k(lambda_j))
  std::vector<int4> nodes;          // [T] corner codes
  std::vector<float4> w;            // [T] corner weights (x 1/2 on column p = 0)
  std::vector<int> colptr;          // [ncols + 1]
  std::vector<int> tq;              // [T] q mod N
  std::vector<uint32_t> mask;       // [ncols][16L] (col_ok only)
  std::vector<int> base;            // [ncols][16L]
  std::vector<int> chord;           // [ncols] Q_p: column p's targets are q = -Q_p .. Q_p, in order
  int max_per_col = 0;
};
void build_inverse_tables(const Consts& C, const std::vector<int>& node_perm, InvTables& I);
cudaError_t launch_inverse(const DevPlan& P, const CUtensorMap& tm, const float* g, float* f,
                           cudaStream_t s);

// kernels_util.cu: setup vector kernels (power iteration)
constexpr int kUtilBlocks = 296;
cudaError_t launch_fill_random(float* v, size_t count, unsigned long long seed, cudaStream_t s);
cudaError_t launch_scale(float* v, size_t count, float f, cudaStream_t s);
cudaError_t launch_dot_partial(const float* a, const float* b, size_t count, float* partial, cudaStream_t s);
// tat_nnls_converge: per image b, kNormParts fixed-range partials of (sum (f - fp)^2, sum f^2)
// in float64 at part[(b * kNormParts + k) * 2 + {0, 1}] (summed on the host in a fixed order)
constexpr int kNormParts = 32;
cudaError_t launch_diff_norms(const float* f, const float* fp, int batch, size_t per_image, double* part,
                              cudaStream_t s);
// G25: P.lowk_add[b] = coef * sum of image b of x (per_image floats each), b = b0 .. b0 + batch - 1
// (forward: weighted by the G26 factors when P.deapod is set)
cudaError_t launch_lowk_sum(const DevPlan& P, const float* x, size_t per_image, double coef, bool image,
                            cudaStream_t s);

constexpr int kLaunchesForward = 5;
constexpr int kLaunchesAdjoint = 6;   // K5T K4T K3T K2Ta K2Tb K1T

}  // namespace tat
