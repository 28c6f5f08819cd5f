// C ABI of libtat (include/tat.h): plan lifetime, argument validation, dispatch.
#include "tat.h"
#include "tat_internal.h"

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <new>
#include <string>
#include <utility>
#include <vector>

using namespace tat;

// The operator entry points take `const tat_plan*` (tat.h): the operator a plan applies is fixed
// between tat_plan_set_* calls.  State those calls create lazily (host-variant staging, power-
// iteration and inverse buffers, profiling slots) is not part of the operator and is `mutable`.
struct tat_plan {
  DevPlan P;
  CUtensorMap tm_s1;    // forward S1 (blocked for the two-stage engine, else column-major)
  CUtensorMap tm_s1a;   // adjoint S~1 (column-major)
  std::vector<int> ring;
  mutable std::vector<void*> allocs;
  mutable size_t workspace_bytes = 0, table_bytes = 0;
  unsigned generation = 0;      // bumped by every tat_plan_set_* call that changes the operator
  mutable float* stage_in = nullptr;    // host-variant staging: [B][n][n]
  mutable float* stage_out = nullptr;   // [B][n_t][n_det]
  mutable float* pw_img = nullptr;      // power iteration: second image buffer [B][n][n]
  mutable float* pw_part = nullptr;     // kUtilBlocks partial dot products
  // tat_nnls_converge (stopping rule): previous iterate, per-image norm partials, active flags
  mutable float* nn_prev = nullptr;
  mutable double* nn_part = nullptr;
  mutable int* nn_active = nullptr;
  // tat_pair_host pipeline: two staging sets, copy streams, per-set events
  mutable bool hp_ready = false, hp_joined = true;
  mutable unsigned long long hp_calls = 0;
  mutable cudaStream_t hp_in = nullptr, hp_out = nullptr;
  mutable cudaEvent_t hp_entry = nullptr, hp_in_done[2] = {}, hp_cmp_done[2] = {}, hp_out_done[2] = {};
  mutable float *hp_f[2] = {}, *hp_g[2] = {}, *hp_u[2] = {};
  float* lowk_buf = nullptr;    // [B] G25 per-image constants (tat_plan_set_quadrature)
  double* lowk_part = nullptr;  // [B][32] their partial sums
  unsigned int* lowk_cnt = nullptr;
  const float* deapod_buf = nullptr;   // [n] G26 factors (tat_plan_set_interpolation)
  // inverse (built on first use)
  std::vector<int> node_perm;   // host copy: (j, l') -> adjoint S2 position
  mutable bool inv_ready = false;
  mutable DevPlan Pinv;                 // P with the inverse tables swapped in
  mutable double inv_r0 = -1.0;
  mutable unsigned char* inv_region = nullptr;
  mutable float* inv_csum = nullptr;
  mutable int inv_annulus = 0;
  // profiling
  mutable int prof_max = 0, prof_fwd = 0, prof_adj = 0;
  mutable std::vector<cudaEvent_t> prof_ev;   // (prof_max) sets of kProfEv events
  mutable std::vector<char> prof_kind;        // 1 = forward, 0 = adjoint, per used slot
};

// Device buffers handed to the kernels must be 16-byte aligned (bulk copies, TMA, float4 and
// 16-byte cp.async accesses); an unaligned view is rejected before any launch.
static bool al16(const void* p) { return ((uintptr_t)p & 15u) == 0; }

static thread_local std::string g_last_error;

static tat_status fail(tat_status s, const std::string& msg) {
  g_last_error = msg;
  return s;
}
static tat_status cuda_fail(cudaError_t e, const char* where) {
  g_last_error = std::string(where) + ": " + cudaGetErrorString(e);
  return e == cudaErrorMemoryAllocation ? TAT_ERR_OUT_OF_MEMORY : TAT_ERR_CUDA;
}

template <class T>
static cudaError_t upload(const tat_plan* p, const std::vector<T>& h, const T** dst, size_t& bytes) {
  void* d = nullptr;
  size_t nb = h.size() * sizeof(T);
  if (nb == 0) nb = sizeof(T);
  cudaError_t e = cudaMalloc(&d, nb);
  if (e != cudaSuccess) return e;
  p->allocs.push_back(d);
  bytes += nb;
  if (!h.empty()) e = cudaMemcpy(d, h.data(), h.size() * sizeof(T), cudaMemcpyHostToDevice);
  *dst = static_cast<const T*>(d);
  return e;
}

static cudaError_t alloc_ws(const tat_plan* p, size_t nb, void** dst) {
  cudaError_t e = cudaMalloc(dst, nb);
  if (e == cudaSuccess) { p->allocs.push_back(*dst); p->workspace_bytes += nb; }
  return e;
}

static void free_all(const tat_plan* p) {
  if (p->hp_ready) {
    cudaStreamSynchronize(p->hp_in);
    cudaStreamSynchronize(p->hp_out);
    for (int k = 0; k < 2; ++k) {
      cudaEventDestroy(p->hp_in_done[k]);
      cudaEventDestroy(p->hp_cmp_done[k]);
      cudaEventDestroy(p->hp_out_done[k]);
    }
    cudaEventDestroy(p->hp_entry);
    cudaStreamDestroy(p->hp_in);
    cudaStreamDestroy(p->hp_out);
    p->hp_ready = false;
  }
  for (void* a : p->allocs) cudaFree(a);
  p->allocs.clear();
  for (cudaEvent_t e : p->prof_ev) cudaEventDestroy(e);
  p->prof_ev.clear();
}

extern "C" {

const char* tat_status_string(tat_status s) {
  switch (s) {
    case TAT_OK: return "TAT_OK";
    case TAT_ERR_INVALID_ARGUMENT: return "TAT_ERR_INVALID_ARGUMENT";
    case TAT_ERR_UNSUPPORTED_GEOMETRY: return "TAT_ERR_UNSUPPORTED_GEOMETRY";
    case TAT_ERR_OUT_OF_MEMORY: return "TAT_ERR_OUT_OF_MEMORY";
    case TAT_ERR_CUDA: return "TAT_ERR_CUDA";
  }
  return "TAT_ERR_UNKNOWN";
}

const char* tat_last_error(void) { return g_last_error.c_str(); }

static void fill_info(const Consts& C, tat_plan_info_t* o) {
  std::memset(o, 0, sizeof *o);
  o->n = C.n; o->n_det = C.n_det; o->n_t = C.n_t; o->batch = C.batch;
  o->N = C.N; o->J = C.J; o->M = C.M; o->n_ring = C.n_ring; o->K = C.K;
  o->n_nodes_half = C.half * C.NL;
  o->L = C.Lbox; o->T_new = C.T_new; o->dxi = C.dxi; o->dlam = C.dlam; o->omega = C.omega;
  o->dt = C.dt; o->h = C.h; o->wJ = C.wJ;
  o->launches_forward = kLaunchesForward;
  o->launches_adjoint = kLaunchesAdjoint - (C.k2f == 1 ? 1 : 0);   // fused K2T: one kernel
  o->n_targets = C.ntargets;
}

// Host-only: derive the plan constants without touching the device (used by CPU tests).
tat_status tat_plan_derive(int n, int n_det, int n_t, double R, double c, double T, int batch,
                           const double* detector_angles, tat_plan_info_t* out, int* ring_index) {
  if (!out) return fail(TAT_ERR_INVALID_ARGUMENT, "out is NULL");
  Consts C;
  std::vector<int> ring;
  int code = 0;
  std::string err = derive_consts(n, n_det, n_t, R, c, T, batch, detector_angles, C, ring, code);
  if (!err.empty()) return fail(code == 2 ? TAT_ERR_UNSUPPORTED_GEOMETRY : TAT_ERR_INVALID_ARGUMENT, err);
  std::string sup = gpu_support(C);
  fill_info(C, out);
  if (ring_index) for (int d = 0; d < C.n_det; ++d) ring_index[d] = ring[d];
  if (!sup.empty()) return fail(TAT_ERR_UNSUPPORTED_GEOMETRY, sup);
  return TAT_OK;
}

// Host-only: the multiplier table m'[k][j] (float32, [K+1][J+1]) the plan would upload.
tat_status tat_plan_host_multiplier(int n, int n_det, int n_t, double R, double c, double T,
                                    const double* detector_angles, float* out, size_t out_len) {
  Consts C;
  std::vector<int> ring;
  int code = 0;
  std::string err = derive_consts(n, n_det, n_t, R, c, T, 1, detector_angles, C, ring, code);
  if (!err.empty()) return fail(code == 2 ? TAT_ERR_UNSUPPORTED_GEOMETRY : TAT_ERR_INVALID_ARGUMENT, err);
  if (!out || out_len < (size_t)C.Kp * C.NL) return fail(TAT_ERR_INVALID_ARGUMENT, "out too small");
  HostTables H;
  build_tables(C, ring, detector_angles, H);
  std::memcpy(out, H.mult.data(), H.mult.size() * sizeof(float));
  return TAT_OK;
}

tat_status tat_plan_create(tat_plan** plan, int n, int n_det, int n_t, double R, double c,
                           double T, int batch, const double* detector_angles) {
  if (!plan) return fail(TAT_ERR_INVALID_ARGUMENT, "plan is NULL");
  Consts C;
  std::vector<int> ring;
  int code = 0;
  std::string err = derive_consts(n, n_det, n_t, R, c, T, batch, detector_angles, C, ring, code);
  if (!err.empty()) return fail(code == 2 ? TAT_ERR_UNSUPPORTED_GEOMETRY : TAT_ERR_INVALID_ARGUMENT, err);
  std::string sup = gpu_support(C);
  if (!sup.empty()) return fail(TAT_ERR_UNSUPPORTED_GEOMETRY, sup);

  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return cuda_fail(e, "cudaGetDevice");

  HostTables H;
  build_tables(C, ring, detector_angles, H);

  tat_plan* p = new (std::nothrow) tat_plan();
  if (!p) return fail(TAT_ERR_OUT_OF_MEMORY, "host allocation");
  DevPlan& P = p->P;
  P.C = C;
  p->ring = ring;
  size_t tb = 0;
  do {
    if ((e = upload(p, H.mult, &P.mult, tb)) != cudaSuccess) break;
    if ((e = upload(p, H.tw_n, &P.tw_n, tb)) != cudaSuccess) break;
    if ((e = upload(p, H.tw_pre, &P.tw_pre, tb)) != cudaSuccess) break;
    if ((e = upload(p, H.tw_ring, &P.tw_ring, tb)) != cudaSuccess) break;
    if ((e = upload(p, H.tw_dct, &P.tw_dct, tb)) != cudaSuccess) break;
    if ((e = upload(p, H.k2_colptr, &P.k2_colptr, tb)) != cudaSuccess) break;
    if ((e = upload(p, H.k2_nodes, &P.k2_nodes, tb)) != cudaSuccess) break;
    if ((e = upload(p, H.node_perm, &P.node_perm, tb)) != cudaSuccess) break;
    if ((e = upload(p, H.k3t_dst, &P.k3t_dst, tb)) != cudaSuccess) break;
    p->node_perm = H.node_perm;
    if ((e = upload(p, H.k2t_colptr, &P.k2t_colptr, tb)) != cudaSuccess) break;
    if ((e = upload(p, H.k2t_tq, &P.k2t_tq, tb)) != cudaSuccess) break;
    if ((e = upload(p, H.k2t_rec, &P.k2t_rec, tb)) != cudaSuccess) break;
    if ((e = upload(p, H.k2t_ov, &P.k2t_ov, tb)) != cudaSuccess) break;
    if ((e = upload(p, H.ring, &P.ring, tb)) != cudaSuccess) break;
    if ((e = upload(p, H.dense_e5, &P.dense_e5, tb)) != cudaSuccess) break;
    if ((e = upload(p, H.dense_e5t, &P.dense_e5t, tb)) != cudaSuccess) break;
    if ((e = upload(p, H.k5tc_b, &P.k5tc_b, tb)) != cudaSuccess) break;
    if ((e = upload(p, H.k5ttc_b, &P.k5ttc_b, tb)) != cudaSuccess) break;
    if ((e = upload(p, H.tw_col, &P.tw_col, tb)) != cudaSuccess) break;
    if ((e = upload(p, H.tw_dct4, &P.tw_dct4, tb)) != cudaSuccess) break;
    if ((e = upload(p, H.k2c_mask, &P.k2c_mask, tb)) != cudaSuccess) break;
    if ((e = upload(p, H.k2c_base, &P.k2c_base, tb)) != cudaSuccess) break;
    const size_t B = (size_t)C.batch;
    void* d;
    if ((e = alloc_ws(p, B * C.ncols * C.n * sizeof(float2), &d)) != cudaSuccess) break;
    P.S1 = (float2*)d;
    if ((e = alloc_ws(p, B * C.half * C.NL * sizeof(float2), &d)) != cudaSuccess) break;
    P.S2 = (float2*)d;
    if ((e = alloc_ws(p, B * C.Kp * C.NL * sizeof(float2) + 16, &d)) != cudaSuccess) break;
    P.S3 = (float2*)d;
    if ((e = alloc_ws(p, B * C.Kp * C.n_t * sizeof(float2) + 16, &d)) != cudaSuccess) break;
    P.S4 = (float2*)d;
    P.C.ntargets = (int)H.k2t_tq.size();
    P.C.ntpad = (P.C.ntargets + 1) & ~1;
    {
      int mx = 0;
      for (int q = 0; q < C.ncols; ++q) mx = std::max(mx, H.k2t_colptr[q + 1] - H.k2t_colptr[q]);
      P.C.k2c_rbuf = (mx + 3) & ~1;   // even: 16-B aligned bulk-copy destinations
      int mw = 0;
      for (int q = 0; q < C.ncols; ++q)
        mw = std::max(mw, H.k2_colptr[q + 1] - H.k2_colptr[q > 0 ? q - 1 : 0]);
      P.C.k2t_win = std::max(mw, 1);
      const char* pdl = getenv("TAT_PDL");   // debugging switch: TAT_PDL=0 disables PDL
      P.C.pdl = pdl ? atoi(pdl) : 1;
      const char* sf = getenv("TAT_STRIP_FWD");   // tuning switches: columns per CTA of K2 / K2Tb
      const char* sa = getenv("TAT_STRIP_ADJ");
      // small problems (few columns x images): narrower strips so that the column kernels still
      // have ~4 CTAs per SM (measured at C2, n = 256, batch 1: strips 16 -> 2 take the step from
      // 98 to 59 us); large ones keep 16 (the halo column of K2 costs 1/strip)
      const int auto_strip = std::max(2, std::min(16, (int)((long)C.ncols * C.batch / (4 * 148))));
      P.C.col_strip = sf ? std::max(2, atoi(sf)) : auto_strip;
      P.C.col_strip_adj = sa ? std::max(1, atoi(sa)) : auto_strip;
    }
    if ((size_t)P.C.k2t_win * 8 > 227 * 1024) {
      e = cudaErrorInvalidConfiguration;
      break;
    }
    if (col_ok(P.C) && smem_k2c_adj(P.C) > 227 * 1024) {
      e = cudaErrorInvalidConfiguration;
      break;
    }
    if ((e = alloc_ws(p, B * (size_t)P.C.ntpad * sizeof(float2) + 16, &d)) != cudaSuccess) break;
    P.Rc = (float2*)d;
    // fused adjoint column stage (k2c_adjf): shared-memory caps for a column's records and one
    // image's node window, the largest over the columns p >= 2 (the origin columns 0 and 1 are
    // 2-3x larger and read global memory), shrunk until 3 CTAs fit per SM (n <= 512)
    // adjoint column stage variant (Consts::k2f); TAT_K2F=0/1/2 overrides (debugging, tuning)
    const char* k2f_env = getenv("TAT_K2F");
    const int k2f_mode = k2f_env ? atoi(k2f_env) : 3;
    if (col_ok(P.C) && !H.k2s_strip.empty() && k2f_mode == 3) {   // k2t_strip + k2c_adj
      int wmax = 2;   // the light strips' windows are staged in smem (heavy ones read global)
      for (size_t s = H.k2s_nheavy; s < H.k2s_strip.size(); ++s) wmax = std::max(wmax, H.k2s_strip[s].y + 2);
      P.C.k2s_n = (int)H.k2s_strip.size();
      P.C.k2s_ovcap = H.k2s_ovcap;
      P.C.k2s_wcap = (wmax + 1) & ~1;
      const char* sipc = getenv("TAT_K2S_IPC");   // tuning switch: images per CTA
      // images per CTA: about 4.5 waves of (3 CTAs x 148 SMs) over the light strips (measured at
      // C3: 4 -> 54.5 us, 8 -> 66, 16 -> 110; at C4 8 -> 45, 4 -> 48)
      const int ipc_auto = (int)std::lround((double)(P.C.k2s_n - H.k2s_nheavy) * C.batch / 2000.0);
      P.C.k2s_ipc = std::max(1, std::min(C.batch, sipc ? atoi(sipc) : ipc_auto));
      if (getenv("TAT_VERBOSE"))
        fprintf(stderr, "tat: K2T mode 3 strips %d (heavy %d) window cap %d smem %zu\n", P.C.k2s_n,
                H.k2s_nheavy, P.C.k2s_wcap, smem_k2t_strip(P.C));
      if (smem_k2t_strip(P.C) <= (size_t)kSmemLimit) {
        if ((e = upload(p, H.k2s_strip, &P.k2s_strip, tb)) != cudaSuccess) break;
        if ((e = upload(p, H.k2s_rec, &P.k2s_rec, tb)) != cudaSuccess) break;
        if ((e = upload(p, H.k2s_ovt, &P.k2s_ovt, tb)) != cudaSuccess) break;
        if ((e = upload(p, H.k2s_ov, &P.k2s_ov, tb)) != cudaSuccess) break;
        if ((e = upload(p, H.k2s_ovr, &P.k2s_ovr, tb)) != cudaSuccess) break;
        P.C.k2s_nheavy = H.k2s_nheavy;
        P.C.k2f = 3;
      }
    }
    if (col_ok(P.C) && !H.k2f_recptr.empty() && (k2f_mode == 1 || k2f_mode == 2)) {
      const int Q0 = col_R(C.n) * 8, Jc = C.n / col_R(C.n);
      int rcap = 4, wcap = 2, tmax = 0;
      for (int q = 0; q < C.ncols; ++q) {
        tmax = std::max(tmax, H.k2t_colptr[q + 1] - H.k2t_colptr[q]);
        if (q < 2) continue;
        int nb = 12 * (H.k2f_recptr[q + 1] - H.k2f_recptr[q]);   // records + overflow lists
        for (int o = H.k2f_ovptr[q]; o < H.k2f_ovptr[q + 1]; ++o) nb += 16 + 8 * H.k2f_ovt[o].z;
        rcap = std::max(rcap, (nb + 11) / 12);
        wcap = std::max(wcap, H.k2_colptr[q + 1] - H.k2_colptr[q - 1] + 2);
      }
      if (k2f_mode == 2 || tmax <= Q0 * (Jc + 1)) {   // fused: the target sums alias the column buffer
        P.C.k2f_rcap = (rcap + 3) & ~3;
        P.C.k2f_wcap = (wcap + 1) & ~1;
        // fused: 3 CTAs of 128 threads per SM (n <= 512); k2t_sumf: 4 CTAs of 256 threads
        const size_t budget = k2f_mode == 2 ? (size_t)55 * 1024
                              : C.n >= 1024 ? (size_t)kSmemLimit : (size_t)74 * 1024;
        auto need = [&]() { return k2f_mode == 2 ? smem_k2t_sumf(P.C) : smem_k2c_adjf(P.C); };
        while (need() > budget && P.C.k2f_rcap > 4) {
          P.C.k2f_rcap = std::max(4, (P.C.k2f_rcap * 15 / 16) & ~3);
          P.C.k2f_wcap = std::max(2, (P.C.k2f_wcap * 15 / 16) & ~1);
        }
        const char* ipc = getenv("TAT_K2F_IPC");   // tuning switch: images per CTA
        P.C.k2f_ipc = std::max(1, std::min(C.batch, ipc ? atoi(ipc) : 8));
        // slow columns (records + overflow lists over the record cap, or the window over its
        // cap: the origin region) run one image per CTA at the head of the grid, reading global
        // memory; the others k2f_ipc images per CTA with the column constants staged once
        std::vector<int> cols, slow;
        for (int q = 0; q < C.ncols; ++q) {
          size_t bytes = (size_t)12 * (H.k2f_recptr[q + 1] - H.k2f_recptr[q]);
          for (int o = H.k2f_ovptr[q]; o < H.k2f_ovptr[q + 1]; ++o) bytes += 16 + 8 * (size_t)H.k2f_ovt[o].z;
          const bool sl = bytes > (size_t)12 * P.C.k2f_rcap ||
                          H.k2_colptr[q + 1] - H.k2_colptr[q > 0 ? q - 1 : 0] + 2 > P.C.k2f_wcap;
          (sl ? slow : cols).push_back(q);
        }
        P.C.k2f_nslow = (int)slow.size();
        if (getenv("TAT_VERBOSE"))
          fprintf(stderr, "tat: K2T mode %d rcap %d wcap %d smem %zu ipc %d slow columns %d of %d\n",
                  k2f_mode, P.C.k2f_rcap, P.C.k2f_wcap, need(), P.C.k2f_ipc, P.C.k2f_nslow, C.ncols);
        cols.insert(cols.begin(), slow.begin(), slow.end());
        if (need() <= (size_t)kSmemLimit) {
          if ((e = upload(p, cols, &P.k2f_cols, tb)) != cudaSuccess) break;
          if ((e = upload(p, H.k2f_rec, &P.k2f_rec, tb)) != cudaSuccess) break;
          if ((e = upload(p, H.k2f_recptr, &P.k2f_recptr, tb)) != cudaSuccess) break;
          if ((e = upload(p, H.k2f_ov, &P.k2f_ov, tb)) != cudaSuccess) break;
          if ((e = upload(p, H.k2f_ovt, &P.k2f_ovt, tb)) != cudaSuccess) break;
          if ((e = upload(p, H.k2f_ovptr, &P.k2f_ovptr, tb)) != cudaSuccess) break;
          P.C.k2f = k2f_mode == 1 ? 1 : 2;
        }
      }
    }
    e = configure_kernels(P);
    if (e == cudaSuccess) e = make_s1_tensor_map(P, &p->tm_s1, col_ok(P.C));
    if (e == cudaSuccess) e = make_s1_tensor_map(P, &p->tm_s1a, false);
  } while (false);
  p->table_bytes = tb;
  if (e != cudaSuccess) {
    tat_status st = cuda_fail(e, "tat_plan_create");
    free_all(p);
    delete p;
    return st;
  }
  *plan = p;
  return TAT_OK;
}

void tat_plan_destroy(tat_plan* plan) {
  if (!plan) return;
  free_all(plan);
  delete plan;
}

tat_status tat_plan_info(const tat_plan* plan, tat_plan_info_t* out, int* ring_index) {
  if (!plan || !out) return fail(TAT_ERR_INVALID_ARGUMENT, "plan or out is NULL");
  fill_info(plan->P.C, out);
  out->workspace_bytes = plan->workspace_bytes;
  out->generation = plan->generation;
  out->table_bytes = plan->table_bytes;
  if (ring_index)
    for (int d = 0; d < plan->P.C.n_det; ++d) ring_index[d] = plan->ring[d];
  return TAT_OK;
}

static cudaEvent_t* prof_slot(const tat_plan* p, bool fwd) {
  if (p->prof_max <= 0) return nullptr;
  int used = p->prof_fwd + p->prof_adj;
  if (used >= p->prof_max) return nullptr;
  (fwd ? p->prof_fwd : p->prof_adj)++;
  p->prof_kind.push_back(fwd ? 1 : 0);
  return &p->prof_ev[(size_t)used * kProfEv];
}

tat_status tat_forward(const tat_plan* plan, const float* f, float* g, cudaStream_t stream) {
  if (!plan || !f || !g) return fail(TAT_ERR_INVALID_ARGUMENT, "NULL plan or buffer");
  if (!al16(f) || !al16(g)) return fail(TAT_ERR_INVALID_ARGUMENT, "f and g must be 16-byte aligned");
  cudaEvent_t* ev = prof_slot(plan, true);
  cudaError_t e = launch_forward(plan->P, plan->tm_s1, f, g, stream, ev);
  if (e != cudaSuccess) return cuda_fail(e, "tat_forward launch");
  return TAT_OK;
}

tat_status tat_adjoint(const tat_plan* plan, const float* g, float* f, cudaStream_t stream) {
  if (!plan || !f || !g) return fail(TAT_ERR_INVALID_ARGUMENT, "NULL plan or buffer");
  if (!al16(f) || !al16(g)) return fail(TAT_ERR_INVALID_ARGUMENT, "f and g must be 16-byte aligned");
  cudaEvent_t* ev = prof_slot(plan, false);
  cudaError_t e = launch_adjoint(plan->P, plan->tm_s1a, g, f, stream, ev);
  if (e != cudaSuccess) return cuda_fail(e, "tat_adjoint launch");
  return TAT_OK;
}

static tat_status ensure_staging(const tat_plan* p) {
  if (p->stage_in) return TAT_OK;
  const Consts& C = p->P.C;
  void *a = nullptr, *b = nullptr;
  cudaError_t e = cudaMalloc(&a, (size_t)C.batch * C.n * C.n * sizeof(float));
  if (e == cudaSuccess) e = cudaMalloc(&b, (size_t)C.batch * C.n_t * C.n_det * sizeof(float));
  if (e != cudaSuccess) {
    if (a) cudaFree(a);
    return cuda_fail(e, "staging allocation");
  }
  p->allocs.push_back(a);
  p->allocs.push_back(b);
  p->stage_in = (float*)a;
  p->stage_out = (float*)b;
  return TAT_OK;
}

tat_status tat_forward_host(const tat_plan* plan, const float* f_host, float* g_host,
                            cudaStream_t stream) {
  if (!plan || !f_host || !g_host) return fail(TAT_ERR_INVALID_ARGUMENT, "NULL plan or buffer");
  const tat_plan* p = plan;
  tat_status st = ensure_staging(p);
  if (st != TAT_OK) return st;
  const Consts& C = p->P.C;
  size_t nin = (size_t)C.batch * C.n * C.n * sizeof(float);
  size_t nout = (size_t)C.batch * C.n_t * C.n_det * sizeof(float);
  cudaError_t e = cudaMemcpyAsync(p->stage_in, f_host, nin, cudaMemcpyHostToDevice, stream);
  if (e != cudaSuccess) return cuda_fail(e, "H2D");
  st = tat_forward(plan, p->stage_in, p->stage_out, stream);
  if (st != TAT_OK) return st;
  e = cudaMemcpyAsync(g_host, p->stage_out, nout, cudaMemcpyDeviceToHost, stream);
  if (e != cudaSuccess) return cuda_fail(e, "D2H");
  return TAT_OK;
}

tat_status tat_adjoint_host(const tat_plan* plan, const float* g_host, float* f_host,
                            cudaStream_t stream) {
  if (!plan || !f_host || !g_host) return fail(TAT_ERR_INVALID_ARGUMENT, "NULL plan or buffer");
  const tat_plan* p = plan;
  tat_status st = ensure_staging(p);
  if (st != TAT_OK) return st;
  const Consts& C = p->P.C;
  size_t nimg = (size_t)C.batch * C.n * C.n * sizeof(float);
  size_t ndat = (size_t)C.batch * C.n_t * C.n_det * sizeof(float);
  cudaError_t e = cudaMemcpyAsync(p->stage_out, g_host, ndat, cudaMemcpyHostToDevice, stream);
  if (e != cudaSuccess) return cuda_fail(e, "H2D");
  st = tat_adjoint(plan, p->stage_out, p->stage_in, stream);
  if (st != TAT_OK) return st;
  e = cudaMemcpyAsync(f_host, p->stage_in, nimg, cudaMemcpyDeviceToHost, stream);
  if (e != cudaSuccess) return cuda_fail(e, "D2H");
  return TAT_OK;
}

// ------------------------------------------------------------------ pipelined host-buffer pair
static tat_status ensure_pair(const tat_plan* p) {
  if (p->hp_ready) return TAT_OK;
  const Consts& C = p->P.C;
  const size_t nimg = (size_t)C.batch * C.n * C.n * sizeof(float);
  const size_t ndat = (size_t)C.batch * C.n_t * C.n_det * sizeof(float);
  cudaError_t e = cudaSuccess;
  void* d = nullptr;
  for (int k = 0; k < 2 && e == cudaSuccess; ++k) {
    if ((e = alloc_ws(p, nimg, &d)) == cudaSuccess) p->hp_f[k] = (float*)d; else break;
    if ((e = alloc_ws(p, ndat, &d)) == cudaSuccess) p->hp_g[k] = (float*)d; else break;
    if ((e = alloc_ws(p, nimg, &d)) == cudaSuccess) p->hp_u[k] = (float*)d; else break;
  }
  if (e == cudaSuccess) e = cudaStreamCreateWithFlags(&p->hp_in, cudaStreamNonBlocking);
  if (e == cudaSuccess) e = cudaStreamCreateWithFlags(&p->hp_out, cudaStreamNonBlocking);
  if (e == cudaSuccess) e = cudaEventCreateWithFlags(&p->hp_entry, cudaEventDisableTiming);
  for (int k = 0; k < 2 && e == cudaSuccess; ++k) {
    e = cudaEventCreateWithFlags(&p->hp_in_done[k], cudaEventDisableTiming);
    if (e == cudaSuccess) e = cudaEventCreateWithFlags(&p->hp_cmp_done[k], cudaEventDisableTiming);
    if (e == cudaSuccess) e = cudaEventCreateWithFlags(&p->hp_out_done[k], cudaEventDisableTiming);
  }
  if (e != cudaSuccess) return cuda_fail(e, "tat_pair_host setup");
  p->hp_ready = true;
  return TAT_OK;
}

tat_status tat_pair_host(const tat_plan* plan, const float* f_host, float* g_host, float* u_host,
                         cudaStream_t stream) {
  if (!plan || !f_host || !u_host) return fail(TAT_ERR_INVALID_ARGUMENT, "NULL plan or buffer");
  tat_status st = ensure_pair(plan);
  if (st != TAT_OK) return st;
  const tat_plan* p = plan;
  const Consts& C = p->P.C;
  const size_t nimg = (size_t)C.batch * C.n * C.n * sizeof(float);
  const size_t ndat = (size_t)C.batch * C.n_t * C.n_det * sizeof(float);
  const int k = (int)(p->hp_calls & 1);
  cudaError_t e = cudaSuccess;
  if (p->hp_joined) {   // first call after a join: ordered after the work already on `stream`
    e = cudaEventRecord(p->hp_entry, stream);
    if (e == cudaSuccess) e = cudaStreamWaitEvent(p->hp_in, p->hp_entry, 0);
  }
  // set k is free once the compute of call i-2 has read hp_f[k] (and its D2H, below, is done)
  if (e == cudaSuccess) e = cudaStreamWaitEvent(p->hp_in, p->hp_cmp_done[k], 0);
  if (e == cudaSuccess) e = cudaMemcpyAsync(p->hp_f[k], f_host, nimg, cudaMemcpyHostToDevice, p->hp_in);
  if (e == cudaSuccess) e = cudaEventRecord(p->hp_in_done[k], p->hp_in);
  if (e == cudaSuccess) e = cudaStreamWaitEvent(stream, p->hp_in_done[k], 0);
  if (e == cudaSuccess) e = cudaStreamWaitEvent(stream, p->hp_out_done[k], 0);
  if (e != cudaSuccess) return cuda_fail(e, "tat_pair_host H2D");
  st = tat_forward(plan, p->hp_f[k], p->hp_g[k], stream);
  if (st != TAT_OK) return st;
  st = tat_adjoint(plan, p->hp_g[k], p->hp_u[k], stream);
  if (st != TAT_OK) return st;
  e = cudaEventRecord(p->hp_cmp_done[k], stream);
  if (e == cudaSuccess) e = cudaStreamWaitEvent(p->hp_out, p->hp_cmp_done[k], 0);
  if (e == cudaSuccess) e = cudaMemcpyAsync(u_host, p->hp_u[k], nimg, cudaMemcpyDeviceToHost, p->hp_out);
  if (e == cudaSuccess && g_host) e = cudaMemcpyAsync(g_host, p->hp_g[k], ndat, cudaMemcpyDeviceToHost, p->hp_out);
  if (e == cudaSuccess) e = cudaEventRecord(p->hp_out_done[k], p->hp_out);
  if (e != cudaSuccess) return cuda_fail(e, "tat_pair_host D2H");
  p->hp_calls++;
  p->hp_joined = false;
  return TAT_OK;
}

tat_status tat_host_join(const tat_plan* plan, cudaStream_t stream) {
  if (!plan) return fail(TAT_ERR_INVALID_ARGUMENT, "NULL plan");
  if (!plan->hp_ready || plan->hp_calls == 0) return TAT_OK;
  const int k = (int)((plan->hp_calls - 1) & 1);   // the copy-out stream is in order
  cudaError_t e = cudaStreamWaitEvent(stream, plan->hp_out_done[k], 0);
  if (e != cudaSuccess) return cuda_fail(e, "tat_host_join");
  plan->hp_joined = true;
  return TAT_OK;
}

// ------------------------------------------------------------------ autograd support
tat_status tat_transpose(const tat_plan* plan, const float* g, float* f, cudaStream_t stream) {
  if (!plan || !f || !g) return fail(TAT_ERR_INVALID_ARGUMENT, "NULL plan or buffer");
  if (!al16(f) || !al16(g)) return fail(TAT_ERR_INVALID_ARGUMENT, "f and g must be 16-byte aligned");
  DevPlan Q = plan->P;
  Q.C.omega = 1.0;   // omega enters only through the K4T multiplier: A^T = A* / omega
  cudaError_t e = launch_adjoint(Q, plan->tm_s1a, g, f, stream, nullptr);
  if (e != cudaSuccess) return cuda_fail(e, "tat_transpose launch");
  return TAT_OK;
}

tat_status tat_plan_set_quadrature(tat_plan* plan, int rule) {
  if (!plan) return fail(TAT_ERR_INVALID_ARGUMENT, "NULL plan");
  if (rule != TAT_QUAD_TRAPEZOID && rule != TAT_QUAD_LOWK)
    return fail(TAT_ERR_INVALID_ARGUMENT, "unknown quadrature rule");
  if (rule == TAT_QUAD_TRAPEZOID) {
    if (plan->P.lowk_add) plan->generation++;
    plan->P.lowk_add = nullptr;
    return TAT_OK;
  }
  if (!plan->P.lowk_add) plan->generation++;
  if (!plan->lowk_buf) {
    const size_t B = (size_t)plan->P.C.batch;
    void* d = nullptr;
    cudaError_t e = alloc_ws(plan, B * (32 * sizeof(double) + sizeof(float) + sizeof(unsigned int)) + 64, &d);
    if (e == cudaSuccess) e = cudaMemset(d, 0, B * (32 * sizeof(double) + sizeof(float) + sizeof(unsigned int)) + 64);
    if (e != cudaSuccess) return cuda_fail(e, "tat_plan_set_quadrature alloc");
    plan->lowk_part = (double*)d;
    plan->lowk_buf = (float*)(plan->lowk_part + 32 * B);
    plan->lowk_cnt = (unsigned int*)(plan->lowk_buf + B);
  }
  plan->P.lowk_add = plan->lowk_buf;
  plan->P.lowk_part = plan->lowk_part;
  plan->P.lowk_cnt = plan->lowk_cnt;
  return TAT_OK;
}

tat_status tat_plan_set_interpolation(tat_plan* plan, int rule) {
  if (!plan) return fail(TAT_ERR_INVALID_ARGUMENT, "NULL plan");
  if (rule != TAT_INTERP_BILINEAR && rule != TAT_INTERP_DEAPOD)
    return fail(TAT_ERR_INVALID_ARGUMENT, "unknown interpolation rule");
  if (rule == TAT_INTERP_BILINEAR) {
    if (plan->P.deapod) plan->generation++;
    plan->P.deapod = nullptr;
    return TAT_OK;
  }
  if (!plan->P.deapod) plan->generation++;
  if (!plan->deapod_buf) {
    const Consts& C = plan->P.C;
    std::vector<float> w(C.n);
    for (int i = 0; i < C.n; ++i) {   // 1 / sinc^2(x / 2L), x = (i - n/2) h, sinc(u) = sin(pi u)/(pi u)
      const double u = 3.14159265358979323846 * (i - C.n / 2) * C.h / (2.0 * C.Lbox);
      const double s = (u == 0.0) ? 1.0 : std::sin(u) / u;
      w[i] = (float)(1.0 / (s * s));
    }
    size_t tb = 0;
    const float* d = nullptr;
    cudaError_t e = upload(plan, w, &d, tb);
    if (e != cudaSuccess) return cuda_fail(e, "tat_plan_set_interpolation upload");
    plan->deapod_buf = d;
  }
  plan->P.deapod = plan->deapod_buf;
  return TAT_OK;
}

tat_status tat_forward_scaled(const tat_plan* plan, const float* f, float* g, float alpha,
                              cudaStream_t stream) {
  if (!plan || !f || !g) return fail(TAT_ERR_INVALID_ARGUMENT, "NULL plan or buffer");
  if (!al16(f) || !al16(g)) return fail(TAT_ERR_INVALID_ARGUMENT, "f and g must be 16-byte aligned");
  if (!std::isfinite(alpha)) return fail(TAT_ERR_INVALID_ARGUMENT, "alpha is not finite");
  DevPlan Q = plan->P;
  Q.epi_scale = alpha;
  cudaError_t e = launch_forward(Q, plan->tm_s1, f, g, stream, nullptr);
  if (e != cudaSuccess) return cuda_fail(e, "tat_forward_scaled launch");
  return TAT_OK;
}

// ------------------------------------------------------------------ inverse (Algorithm 3)
static tat_status inverse_setup(const tat_plan* p) {
  if (p->inv_ready) return TAT_OK;
  const Consts& C = p->P.C;
  InvTables I;
  build_inverse_tables(C, p->node_perm, I);
  DevPlan Q = p->P;
  size_t tb = 0;
  cudaError_t e = cudaSuccess;
  do {
    if ((e = upload(p, I.mult, &Q.mult, tb)) != cudaSuccess) break;
    if ((e = upload(p, I.nodes, &Q.inv_nodes, tb)) != cudaSuccess) break;
    if ((e = upload(p, I.w, &Q.inv_w, tb)) != cudaSuccess) break;
    if ((e = upload(p, I.colptr, &Q.k2t_colptr, tb)) != cudaSuccess) break;
    if ((e = upload(p, I.tq, &Q.k2t_tq, tb)) != cudaSuccess) break;
    if ((e = upload(p, I.mask, &Q.k2c_mask, tb)) != cudaSuccess) break;
    if ((e = upload(p, I.base, &Q.k2c_base, tb)) != cudaSuccess) break;
    if (col_ok(C) && !I.chord.empty()) {
      if ((e = upload(p, I.chord, &Q.k2c_chord, tb)) != cudaSuccess) break;
    } else {
      Q.k2c_chord = nullptr;
    }
    Q.C.ntargets = (int)I.tq.size();
    Q.C.ntpad = (Q.C.ntargets + 1) & ~1;
    Q.C.k2c_rbuf = (I.max_per_col + 3) & ~1;
    Q.C.omega = 1.0;
    Q.C.dct_sine = 1;
    void* d = nullptr;
    if ((e = alloc_ws(p, (size_t)C.batch * Q.C.ntpad * sizeof(float2) + 16, &d)) != cudaSuccess) break;
    Q.Rc = (float2*)d;
    if ((e = alloc_ws(p, (size_t)C.n * C.n, &d)) != cudaSuccess) break;
    p->inv_region = (unsigned char*)d;
    if ((e = alloc_ws(p, (size_t)C.batch * kInvParts * sizeof(float), &d)) != cudaSuccess) break;
    p->inv_csum = (float*)d;
  } while (false);
  p->table_bytes += tb;
  if (e != cudaSuccess) return cuda_fail(e, "inverse tables");
  if (col_ok(Q.C) && smem_k2c_adj(Q.C) > 227 * 1024)
    return fail(TAT_ERR_UNSUPPORTED_GEOMETRY, "inverse: column target buffer exceeds shared memory");
  Q.lowk_add = nullptr;   // A^{-1} (Algorithm 3) has no quadrature / interpolation variant
  Q.deapod = nullptr;
  p->Pinv = Q;
  p->inv_ready = true;
  return TAT_OK;
}

tat_status tat_inverse(const tat_plan* plan, const float* g, float* f, double r0,
                       cudaStream_t stream) {
  if (!plan || !f || !g) return fail(TAT_ERR_INVALID_ARGUMENT, "NULL plan or buffer");
  if (!al16(f) || !al16(g)) return fail(TAT_ERR_INVALID_ARGUMENT, "f and g must be 16-byte aligned");
  const Consts& C = plan->P.C;
  if (!(r0 > 0.0 && r0 < C.R)) return fail(TAT_ERR_INVALID_ARGUMENT, "r0 must lie in (0, R)");
  if (C.R != 1.0 || C.c != 1.0)
    return fail(TAT_ERR_UNSUPPORTED_GEOMETRY, "inverse: the paper derives A^-1 for R = c = 1");
  if (C.dense)
    return fail(TAT_ERR_UNSUPPORTED_GEOMETRY, "inverse: needs detectors on a canonical ring");
  if (!dct4_ok(C) && !dct_fast_r(C))
    return fail(TAT_ERR_UNSUPPORTED_GEOMETRY, "inverse: no sine-transform kernel for this 2M");
  const tat_plan* p = plan;
  tat_status st = inverse_setup(p);
  if (st != TAT_OK) return st;
  cudaError_t e = cudaSuccess;
  if (r0 != p->inv_r0) {   // region mask of Pi_Omega0 and the annulus (float64 decisions)
    std::vector<unsigned char> reg((size_t)C.n * C.n);
    int cnt = 0;
    for (int iy = 0; iy < C.n; ++iy)
      for (int ix = 0; ix < C.n; ++ix) {
        const double r = std::hypot((ix - C.n / 2) * C.h, (iy - C.n / 2) * C.h);
        unsigned char v = 0;
        if (r <= r0) v = 1;
        else if (r < C.R) { v = 2; ++cnt; }
        reg[(size_t)iy * C.n + ix] = v;
      }
    // ordered on `stream`: earlier inverse calls still reading the old mask finish first; the
    // synchronisation keeps the host vector alive until the (pageable) copy has been staged
    e = cudaMemcpyAsync(p->inv_region, reg.data(), reg.size(), cudaMemcpyHostToDevice, stream);
    if (e == cudaSuccess) e = cudaStreamSynchronize(stream);
    if (e != cudaSuccess) return cuda_fail(e, "inverse region upload");
    p->inv_r0 = r0;
    p->inv_annulus = cnt;
  }
  e = launch_inverse(p->Pinv, p->tm_s1a, g, f, stream);
  if (e == cudaSuccess) e = launch_k2i_finish(p->Pinv, f, p->inv_region, p->inv_csum, p->inv_annulus, stream);
  if (e != cudaSuccess) return cuda_fail(e, "tat_inverse launch");
  return TAT_OK;
}

// ------------------------------------------------------------------ iterative driver
// NNLS / projected Landweber (§4.2): r = A f - g (fused into the last forward
// stage), f <- Pi max(0, f - lambda A* r) (fused into the last adjoint stage).
tat_status tat_residual(const tat_plan* plan, const float* f, const float* g_obs, float* r,
                        cudaStream_t stream) {
  if (!plan || !f || !g_obs || !r) return fail(TAT_ERR_INVALID_ARGUMENT, "NULL plan or buffer");
  if (!al16(f) || !al16(g_obs) || !al16(r)) return fail(TAT_ERR_INVALID_ARGUMENT, "buffers must be 16-byte aligned");
  DevPlan Q = plan->P;
  Q.epi_sub = g_obs;
  cudaError_t e = launch_forward(Q, plan->tm_s1, f, r, stream, nullptr);
  if (e != cudaSuccess) return cuda_fail(e, "tat_residual launch");
  return TAT_OK;
}

tat_status tat_adjoint_step(const tat_plan* plan, const float* r, float* f, float lambda,
                            int nonneg, const float* roi, cudaStream_t stream) {
  if (!plan || !f || !r) return fail(TAT_ERR_INVALID_ARGUMENT, "NULL plan or buffer");
  if (!al16(f) || !al16(r) || !al16(roi)) return fail(TAT_ERR_INVALID_ARGUMENT, "buffers must be 16-byte aligned");
  if (!std::isfinite(lambda)) return fail(TAT_ERR_INVALID_ARGUMENT, "lambda is not finite");
  DevPlan Q = plan->P;
  Q.epi_update = nonneg ? 2 : 1;
  Q.epi_tau = lambda;
  Q.epi_roi = roi;
  cudaError_t e = launch_adjoint(Q, plan->tm_s1a, r, f, stream, nullptr);
  if (e != cudaSuccess) return cuda_fail(e, "tat_adjoint_step launch");
  return TAT_OK;
}

tat_status tat_nnls(const tat_plan* plan, const float* g_obs, float* f, float* r_work,
                    float lambda, int iters, int nonneg, const float* roi, cudaStream_t stream) {
  if (!plan || !g_obs || !f || !r_work) return fail(TAT_ERR_INVALID_ARGUMENT, "NULL plan or buffer");
  if (iters < 0) return fail(TAT_ERR_INVALID_ARGUMENT, "iters < 0");
  if (!std::isfinite(lambda)) return fail(TAT_ERR_INVALID_ARGUMENT, "lambda is not finite");
  for (int k = 0; k < iters; ++k) {
    tat_status st = tat_residual(plan, f, g_obs, r_work, stream);
    if (st != TAT_OK) return st;
    st = tat_adjoint_step(plan, r_work, f, lambda, nonneg, roi, stream);
    if (st != TAT_OK) return st;
  }
  return TAT_OK;
}

tat_status tat_nnls_converge(const tat_plan* plan, const float* g_obs, float* f, float* r_work,
                             float lambda, int max_iters, int check_every, double rel_tol, int nonneg,
                             const float* roi, int* iters_out, cudaStream_t stream) {
  if (!plan || !g_obs || !f || !r_work || !iters_out)
    return fail(TAT_ERR_INVALID_ARGUMENT, "NULL plan or buffer");
  if (!al16(f) || !al16(g_obs) || !al16(r_work) || !al16(roi))
    return fail(TAT_ERR_INVALID_ARGUMENT, "buffers must be 16-byte aligned");
  if (max_iters < 1 || check_every < 1 || !(rel_tol > 0.0) || !std::isfinite(lambda))
    return fail(TAT_ERR_INVALID_ARGUMENT, "max_iters, check_every must be >= 1, rel_tol > 0, lambda finite");
  const tat_plan* p = plan;
  const Consts& C = p->P.C;
  const int B = C.batch;
  const size_t per = (size_t)C.n * C.n;
  cudaError_t e = cudaSuccess;
  void* d = nullptr;
  if (!p->nn_prev) {
    if ((e = alloc_ws(p, (size_t)B * per * sizeof(float), &d)) == cudaSuccess) p->nn_prev = (float*)d;
    if (e == cudaSuccess && (e = alloc_ws(p, (size_t)B * kNormParts * 2 * sizeof(double), &d)) == cudaSuccess)
      p->nn_part = (double*)d;
    if (e == cudaSuccess && (e = alloc_ws(p, (size_t)B * sizeof(int), &d)) == cudaSuccess) p->nn_active = (int*)d;
    if (e != cudaSuccess) {
      p->nn_prev = nullptr;
      return cuda_fail(e, "tat_nnls_converge buffers");
    }
  }
  std::vector<int> active(B, 1), iters(B, -max_iters);
  std::vector<double> first(B, 0.0), part((size_t)B * kNormParts * 2);
  e = cudaMemcpyAsync(p->nn_active, active.data(), B * sizeof(int), cudaMemcpyHostToDevice, stream);
  if (e == cudaSuccess) e = cudaStreamSynchronize(stream);
  DevPlan R = p->P;          // r = A f - g_obs
  R.epi_sub = g_obs;
  DevPlan U = p->P;          // f <- P(f - lambda A* r) for the active images
  U.epi_update = nonneg ? 2 : 1;
  U.epi_tau = lambda;
  U.epi_roi = roi;
  U.epi_active = p->nn_active;
  int live = B;
  for (int k = 1; k <= max_iters && live > 0 && e == cudaSuccess; ++k) {
    bool unset = false;
    for (int b = 0; b < B; ++b) unset |= active[b] && first[b] == 0.0;
    const bool chk = unset || k % check_every == 0;
    if (chk) e = cudaMemcpyAsync(p->nn_prev, f, (size_t)B * per * sizeof(float), cudaMemcpyDeviceToDevice, stream);
    if (e == cudaSuccess) e = launch_forward(R, p->tm_s1, f, r_work, stream, nullptr);
    if (e == cudaSuccess) e = launch_adjoint(U, p->tm_s1a, r_work, f, stream, nullptr);
    if (e != cudaSuccess || !chk) continue;
    e = launch_diff_norms(f, p->nn_prev, B, per, p->nn_part, stream);
    if (e == cudaSuccess) e = cudaMemcpyAsync(part.data(), p->nn_part, part.size() * sizeof(double),
                                              cudaMemcpyDeviceToHost, stream);
    if (e == cudaSuccess) e = cudaStreamSynchronize(stream);
    if (e != cudaSuccess) break;
    bool changed = false;
    for (int b = 0; b < B; ++b) {
      if (!active[b]) continue;
      double dd = 0.0, ff = 0.0;
      for (int q = 0; q < kNormParts; ++q) {   // fixed order
        dd += part[((size_t)b * kNormParts + q) * 2];
        ff += part[((size_t)b * kNormParts + q) * 2 + 1];
      }
      if (first[b] == 0.0) {   // the first non-zero approximation sets the scale (no test on it)
        if (ff > 0.0) first[b] = std::sqrt(ff);
      } else if (std::sqrt(dd) < rel_tol * first[b]) {
        active[b] = 0;
        iters[b] = k;
        --live;
        changed = true;
      }
    }
    if (changed && live > 0) {
      e = cudaMemcpyAsync(p->nn_active, active.data(), B * sizeof(int), cudaMemcpyHostToDevice, stream);
      if (e == cudaSuccess) e = cudaStreamSynchronize(stream);
    }
  }
  if (e == cudaSuccess) e = cudaStreamSynchronize(stream);
  if (e != cudaSuccess) return cuda_fail(e, "tat_nnls_converge");
  for (int b = 0; b < B; ++b) iters_out[b] = iters[b];
  return TAT_OK;
}

static cudaError_t dot_host(const tat_plan* p, const float* a, const float* b, size_t count,
                            cudaStream_t s, double* out) {
  cudaError_t e = launch_dot_partial(a, b, count, p->pw_part, s);
  float part[kUtilBlocks];
  if (e == cudaSuccess) e = cudaMemcpyAsync(part, p->pw_part, sizeof part, cudaMemcpyDeviceToHost, s);
  if (e == cudaSuccess) e = cudaStreamSynchronize(s);
  double acc = 0.0;
  for (int i = 0; i < kUtilBlocks; ++i) acc += part[i];   // fixed order
  *out = acc;
  return e;
}

tat_status tat_power_norm(const tat_plan* plan, int iters, unsigned long long seed,
                          double* lambda_max, cudaStream_t stream) {
  if (!plan || !lambda_max || iters < 1) return fail(TAT_ERR_INVALID_ARGUMENT, "bad arguments");
  const tat_plan* p = plan;
  tat_status st = ensure_staging(p);
  if (st != TAT_OK) return st;
  const Consts& C = p->P.C;
  const size_t nimg = (size_t)C.batch * C.n * C.n;
  cudaError_t e = cudaSuccess;
  if (!p->pw_img) {
    void* a = nullptr;
    void* b = nullptr;
    e = cudaMalloc(&a, nimg * sizeof(float));
    if (e == cudaSuccess) e = cudaMalloc(&b, kUtilBlocks * sizeof(float));
    if (e != cudaSuccess) {
      if (a) cudaFree(a);
      return cuda_fail(e, "power-iteration buffers");
    }
    p->allocs.push_back(a);
    p->allocs.push_back(b);
    p->pw_img = (float*)a;
    p->pw_part = (float*)b;
  }
  float* v = p->stage_in;    // current vector
  float* u = p->pw_img;      // A* A v
  float* w = p->stage_out;   // A v
  e = launch_fill_random(v, nimg, seed, stream);
  double lam = 0.0;
  for (int it = 0; it < iters && e == cudaSuccess; ++it) {
    double vv = 0.0;
    e = dot_host(p, v, v, nimg, stream, &vv);
    if (e != cudaSuccess) break;
    if (!(vv > 0.0)) return fail(TAT_ERR_CUDA, "power iteration collapsed to zero");
    e = launch_scale(v, nimg, (float)(1.0 / std::sqrt(vv)), stream);
    if (e == cudaSuccess) e = launch_forward(p->P, p->tm_s1, v, w, stream, nullptr);
    if (e == cudaSuccess) e = launch_adjoint(p->P, p->tm_s1a, w, u, stream, nullptr);
    if (e == cudaSuccess) e = dot_host(p, v, u, nimg, stream, &lam);   // Rayleigh quotient
    std::swap(v, u);
  }
  if (e != cudaSuccess) return cuda_fail(e, "tat_power_norm");
  *lambda_max = lam;
  return TAT_OK;
}

tat_status tat_profile_begin(tat_plan* plan, int max_calls) {
  if (!plan || max_calls < 0) return fail(TAT_ERR_INVALID_ARGUMENT, "bad arguments");
  for (cudaEvent_t e : plan->prof_ev) cudaEventDestroy(e);
  plan->prof_ev.assign((size_t)max_calls * kProfEv, nullptr);
  plan->prof_kind.clear();
  for (auto& e : plan->prof_ev) {
    cudaError_t r = cudaEventCreate(&e);
    if (r != cudaSuccess) return cuda_fail(r, "cudaEventCreate");
  }
  plan->prof_max = max_calls;
  plan->prof_fwd = plan->prof_adj = 0;
  return TAT_OK;
}

tat_status tat_profile_end(tat_plan* plan, float* stage_ms, int* n_forward, int* n_adjoint) {
  if (!plan || !stage_ms) return fail(TAT_ERR_INVALID_ARGUMENT, "bad arguments");
  for (int i = 0; i < 11; ++i) stage_ms[i] = 0.f;
  int used = plan->prof_fwd + plan->prof_adj;
  for (int u = 0; u < used; ++u) {
    cudaEvent_t* ev = &plan->prof_ev[(size_t)u * kProfEv];
    cudaError_t r = cudaEventSynchronize(ev[5]);
    if (r != cudaSuccess) return cuda_fail(r, "cudaEventSynchronize");
    const bool fwd = plan->prof_kind[u] != 0;
    // forward: ev[0..5] bound K1..K5; adjoint: ev[0..3] K5T..K3T, ev[3] -> ev[6] K2Ta,
    // ev[6] -> ev[4] K2Tb, ev[4] -> ev[5] K1T
    static const int fa[5] = {0, 1, 2, 3, 4}, fb[5] = {1, 2, 3, 4, 5};
    static const int aa[6] = {0, 1, 2, 3, 6, 4}, ab[6] = {1, 2, 3, 6, 4, 5};
    for (int s = 0; s < (fwd ? 5 : 6); ++s) {
      float ms = 0.f;
      r = cudaEventElapsedTime(&ms, ev[fwd ? fa[s] : aa[s]], ev[fwd ? fb[s] : ab[s]]);
      if (r != cudaSuccess) return cuda_fail(r, "cudaEventElapsedTime");
      stage_ms[(fwd ? 0 : 5) + s] += ms;
    }
  }
  if (n_forward) *n_forward = plan->prof_fwd;
  if (n_adjoint) *n_adjoint = plan->prof_adj;
  for (cudaEvent_t e : plan->prof_ev) cudaEventDestroy(e);
  plan->prof_ev.clear();
  plan->prof_kind.clear();
  plan->prof_max = 0;
  plan->prof_fwd = plan->prof_adj = 0;
  return TAT_OK;
}

}  // extern "C"
