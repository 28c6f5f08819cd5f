// Host plan builder (float64): constants, Bessel multiplier, resampling tables.
//
// PAPER.md L571-574 / L698-701: "additional time saving is achieved by pre-computing and
// storing the values of the Bessel functions J_|k|(lambda) for the values of k from 0 to half
// the number of discretization points in theta, and for all values of lambda".  This file
// builds those tables (and the bilinear cells of Alg. 1 step 3) once per
// geometry.  It shares no code with oracle/ (which uses scipy for J and dense DFTs).
#include "tat_internal.h"

#include <algorithm>
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <numeric>

namespace tat {

static const double kPi = 3.14159265358979323846264338327950288;

static bool is_pow2(long v) { return v > 0 && (v & (v - 1)) == 0; }

static std::string fmt(const char* f, double a = 0, double b = 0) {
  char buf[256];
  snprintf(buf, sizeof buf, f, a, b);
  return buf;
}

// D0: every constant in float64, mirroring the paper's grid rules.
std::string derive_consts(int n, int n_det, int n_t, double R, double c, double T, int batch,
                          const double* angles, Consts& C, std::vector<int>& ring_out,
                          int& code) {
  code = 1;
  if (!angles) return "detector_angles is NULL";
  if (n < 8 || (n & 1) || !is_pow2(n)) return fmt("n=%g must be an even power of two >= 8", n);
  if (n_det < 1) return "n_det must be >= 1";
  if (n_t < 1) return "n_t must be >= 1";
  if (batch < 1) return "batch must be >= 1";
  if (!(std::isfinite(R) && R > 0)) return "R must be finite and > 0";
  if (!(std::isfinite(c) && c > 0)) return "c must be finite and > 0";
  if (!(std::isfinite(T) && T > 0)) return "T must be finite and > 0";
  for (int d = 0; d < n_det; ++d)
    if (!std::isfinite(angles[d])) return fmt("detector angle %g is not finite", d);

  C = Consts();
  C.n = n; C.n_det = n_det; C.n_t = n_t; C.batch = batch; C.R = R; C.c = c; C.T = T;
  if (const char* r2 = std::getenv("TAT_RING2")) C.ring2 = std::atoi(r2);   // tuning switch: 0 = Stockham ring kernels
  C.h = 2.0 / n;
  C.T_new0 = std::max(2.0 * c * T, 6.0);
  C.Lbox = std::pow(2.0, std::ceil(std::log2(C.T_new0 + 2.0) - 1e-12));
  C.N = (int)std::lround(2.0 * C.Lbox / C.h);
  C.Lres = C.N / n;
  C.log2L = 0;
  while ((1 << C.log2L) < C.Lres) ++C.log2L;
  C.dxi = kPi / C.Lbox;
  C.dt = T / n_t;
  double Mf = std::ceil(C.T_new0 / (c * C.dt) - 1e-9);
  if (Mf > 1e8) { code = 2; return "T_new / (c dt) too large"; }
  C.M = (int)Mf;
  C.T_new = C.M * c * C.dt;
  C.dlam = kPi / C.T_new;
  C.lowk_c = (C.dlam * C.dlam / 12.0) * (C.h * C.h / (2.0 * kPi));
  C.lam_max = kPi / C.h;
  C.J = (int)std::floor(C.lam_max / C.dlam + 1e-9);
  C.NL = C.J + 1;
  C.wJ = (std::fabs(C.J * C.dlam - C.lam_max) <= 1e-9 * C.lam_max) ? 0.5 : 1.0;

  // canonical ring (reading G3): smallest multiple of 4 >= n_det holding every angle
  code = 2;
  int start = std::max(4, 4 * ((n_det + 3) / 4));
  std::vector<int> ring(n_det);
  int n_ring = 0;
  for (int cand = start; cand <= 65536 && !n_ring; cand += 4) {
    bool ok = true;
    for (int d = 0; d < n_det && ok; ++d) {
      double x = angles[d] * cand / (2.0 * kPi);
      double r = std::nearbyint(x);
      if (std::fabs(x - r) * (2.0 * kPi / cand) >= 1e-9) ok = false;
      else {
        long ri = (long)r % cand;
        if (ri < 0) ri += cand;
        ring[d] = (int)ri;
      }
    }
    if (ok) n_ring = cand;
  }
  if (!n_ring) {
    // reading G24: detectors off every canonical ring -> dense mode, polar grid n_phi = the
    // smallest power of two >= max(n_det, 8); synthesis/analysis at the exact angles
    n_ring = 8;
    while (n_ring < n_det) n_ring *= 2;
    C.dense = 1;
    {
      const char* ev = std::getenv("TAT_DENSE_TC");   // debug switch: 0 = SIMT K5d / K5dT, 2 = SIMT K5dT
      const bool tc = !(ev && ev[0] == '0');
      const int nt2 = 2 * (n_ring / 2 + 1);   // real columns of the complex harmonics 0..K
      C.k5tc_kp = tc ? (nt2 + kK5tcKC - 1) / kK5tcKC * kK5tcKC : 0;
      C.k5ttc_kp = (tc && !(ev && ev[0] == '2')) ? (n_det + kK5tcKC - 1) / kK5tcKC * kK5tcKC : 0;
      C.k5ttc_nb = (nt2 + 255) / 256;
      C.k5ttc_nt = ((nt2 + C.k5ttc_nb - 1) / C.k5ttc_nb + 15) / 16 * 16;
    }
    std::fill(ring.begin(), ring.end(), -1);
  } else {
    std::vector<int> s(ring);
    std::sort(s.begin(), s.end());
    if (std::adjacent_find(s.begin(), s.end()) != s.end())
      return "two detectors share one ring position";
  }
  C.n_ring = n_ring;
  ring_out = ring;
  C.K = n_ring / 2;
  C.Kp = C.K + 1;
  C.half = n_ring / 2;
  C.ncols = C.N / 2 + 1;
  C.omega = C.dt * 2.0 * kPi * R / (n_ring * C.h * C.h);
  {   // S1 TMA tile: largest power of two <= min(256, L * rstride(n) / 8)
    const int pn = n + n / 16, rs = pn + ((18 - pn % 16) % 16);
    const int lim = std::min(256, C.Lres * rs / 8);
    C.s1boxP = 1;
    while (C.s1boxP * 2 <= lim) C.s1boxP *= 2;
    if (col_ok(C)) C.s1boxP = 128;   // kernels_col.cu K1/K1T tiles
  }
  code = 0;
  return "";
}

static bool smooth23(long v) {   // v = 2^a 3^b (radix-4/2/3 Stockham passes)
  while (v % 3 == 0) v /= 3;
  return is_pow2(v);
}

std::string gpu_support(const Consts& C) {
  if (C.n < 32 || C.n > 1024) return fmt("n=%g outside the implemented range [32, 1024]", C.n);
  if (!is_pow2(C.Lres) || C.Lres < 2 || C.Lres > 16)
    return fmt("oversampling N/n=%g unsupported", C.Lres);
  if (!is_pow2(C.n_ring) || C.n_ring < 8 || C.n_ring > 2048)
    return fmt("n_ring=%g: kernels implement powers of two in [8, 2048]", C.n_ring);
  if (!smooth23(2L * C.M)) return fmt("2M=%g is not of the form 2^a 3^b", 2.0 * C.M);
  if (C.NL > 2 * C.M) return "J+1 > 2M (time step coarser than twice the pixel pitch)";
  if (C.n_t > 2 * C.M - 1) return "n_t too large for the DCT length";
  if ((long)C.Lres * C.n > 8192) return fmt("L n = %g > 8192 (threads per CTA)", (double)C.Lres * C.n);
  if (max_smem_needed(C) > 227 * 1024) return fmt("shared memory need %g KB > 227 KB",
                                                  max_smem_needed(C) / 1024.0);
  return "";
}

// Miller's downward recurrence for J_0..J_kmax(x), normalised by J_0 + 2 sum J_2m = 1.
// Start index kmax + max(20, 1.5 x) + 20 (made even); rescales to avoid overflow.
void bessel_row(double x, int kmax, double* out) {
  if (x == 0.0) {
    out[0] = 1.0;
    for (int k = 1; k <= kmax; ++k) out[k] = 0.0;
    return;
  }
  int start = kmax + std::max(20, (int)(1.5 * x)) + 20;
  if (start & 1) ++start;
  for (int k = 0; k <= kmax; ++k) out[k] = 0.0;
  double bjp = 0.0, bj = 1e-30, sum = 0.0;
  for (int k = start; k > 0; --k) {
    double bjm = (2.0 * k / x) * bj - bjp;     // J_{k-1}
    bjp = bj;
    bj = bjm;
    int km1 = k - 1;
    if (std::fabs(bj) > 1e250) {
      bj *= 1e-250; bjp *= 1e-250; sum *= 1e-250;
      for (int i = km1 + 1; i <= kmax; ++i) out[i] *= 1e-250;
    }
    if (km1 <= kmax) out[km1] = bj;
    if (km1 == 0) sum += bj;
    else if ((km1 & 1) == 0) sum += 2.0 * bj;
  }
  double inv = 1.0 / sum;
  for (int k = 0; k <= kmax; ++k) out[k] *= inv;
}

static float2 root(long r, long Nr, int sign) {   // exp(sign 2 pi i r / Nr), r reduced
  r %= Nr;
  if (r < 0) r += Nr;
  double a = 2.0 * kPi * (double)r / (double)Nr;
  return make_float2((float)std::cos(a), (float)(sign * std::sin(a)));
}

static void unit_circle(int l, int n_phi, double& cs, double& sn) {
  // quadrant-reduced (cos, sin)(2 pi l / n_phi): multiples of pi/2 are exact
  int Q = n_phi / 4;
  int qd = l / Q, rem = l % Q;
  double b = 2.0 * kPi * rem / n_phi;
  double c0 = std::cos(b), s0 = std::sin(b);
  switch (qd) {
    case 0: cs = c0; sn = s0; break;
    case 1: cs = -s0; sn = c0; break;
    case 2: cs = -c0; sn = -s0; break;
    default: cs = s0; sn = -c0; break;
  }
}

static inline int fbits(float f) { int i; std::memcpy(&i, &f, 4); return i; }

// TF32 split operand for the tcgen05 GEMMs (kernels_dense.cu): B[row][k] for nb tiles of nt rows
// and KP (a multiple of kK5tcKC) reduction indices, packed [tile][chunk][hi, lo][nt x KC] in the
// no-swizzle K-major core layout: element (r, k) of a tile at float offset (r / 8) * 8 KC +
// (k / 4) * 32 + (r % 8) * 4 + k % 4.  hi = round-to-nearest TF32 (10 mantissa bits), lo = its
// residual, rounded the same way.
template <typename F>
static void pack_kmajor(std::vector<float>& out, int nb, int nt, int KP, F val) {
  constexpr int KC = kK5tcKC;
  auto tf32 = [](float x) {
    uint32_t u;
    std::memcpy(&u, &x, 4);
    u = (u + 0x1000u) & 0xFFFFE000u;
    float r;
    std::memcpy(&r, &u, 4);
    return r;
  };
  const int nch = KP / KC;
  out.assign((size_t)nb * nt * KP * 2, 0.f);
  for (int tb = 0; tb < nb; ++tb)
    for (int r = 0; r < nt; ++r)
      for (int k = 0; k < KP; ++k) {
        const float v = val(tb * nt + r, k);
        const size_t tile = ((size_t)tb * nch + k / KC) * 2;
        const int kk = k % KC;
        const size_t off = (size_t)(r / 8) * 8 * KC + (kk / 4) * 32 + (r % 8) * 4 + kk % 4;
        const float hi = tf32(v);
        out[tile * nt * KC + off] = hi;
        out[(tile + 1) * nt * KC + off] = tf32(v - hi);
      }
}

void build_tables(const Consts& C, const std::vector<int>& ring, const double* angles,
                  HostTables& H) {
  const int n = C.n, N = C.N, L = C.Lres, NL = C.NL, Kp = C.Kp, nphi = C.n_ring;
  // ---- multiplier m'[k][j] (E:eq2 P:L463-466 + trapezoid in lambda; scale of D1 and D3)
  H.mult.assign((size_t)Kp * NL, 0.f);
  {
    std::vector<double> row(Kp);
    const double scale = (C.h * C.h / (2.0 * kPi)) / nphi;
    for (int j = 0; j < NL; ++j) {
      double lam = j * C.dlam;
      double w = (j == 0) ? 0.5 : (j == C.J ? C.wJ : 1.0);
      bessel_row(C.R * lam, C.K, row.data());
      double wl = scale * w * C.dlam * lam;
      for (int k = 0; k < Kp; ++k) H.mult[(size_t)k * NL + j] = (float)(wl * row[k]);
    }
  }
  // ---- twiddles
  H.tw_n.resize(n);
  for (int k = 0; k < n; ++k) H.tw_n[k] = root(k, n, -1);
  H.tw_pre.resize((size_t)L * n);
  for (int s = 0; s < L; ++s)
    for (int yp = 0; yp < n; ++yp) {
      long ypp = (yp < n / 2) ? yp : yp - n;        // y'' in [-n/2, n/2)
      H.tw_pre[(size_t)s * n + yp] = root((long)s * ypp, N, -1);
    }
  H.tw_ring.resize(nphi);
  for (int k = 0; k < nphi; ++k) H.tw_ring[k] = root(k, nphi, -1);
  H.tw_col.resize((size_t)L * n);
  for (int s = 0; s < L; ++s)
    for (int y = 0; y < n; ++y) H.tw_col[(size_t)s * n + y] = root((long)s * (y - n / 2), N, -1);
  H.tw_dct4.resize((size_t)4 * n);
  for (int s = 0; s < 4; ++s)
    for (int i = 0; i < n; ++i) H.tw_dct4[(size_t)s * n + i] = root((long)s * i, 4L * n, -1);
  H.tw_dct.resize(2 * (size_t)C.M);
  for (int k = 0; k < 2 * C.M; ++k) H.tw_dct[k] = root(k, 2L * C.M, -1);
  H.ring = ring;
  if (C.dense) {   // dense synthesis / analysis tables (reading G24), angles reduced in float64
    H.dense_e5.resize((size_t)C.Kp * C.n_det);
    H.dense_e5t.resize((size_t)C.Kp * C.n_det);
    for (int k = 0; k < C.Kp; ++k) {
      const double sk = (k == C.K) ? -1.0 : 1.0;            // row K holds the harmonic -K
      const double ck = (k == 0 || k == C.K) ? 1.0 : 2.0;   // C2R weights
      for (int d = 0; d < C.n_det; ++d) {
        const double a = std::fmod(sk * k * angles[d], 2.0 * kPi);
        // the harmonic -K enters through its real part only (G_{-K} is real for real f and
        // even K = n_phi / 2; Re keeps G_{-K} cos(K theta), reading G24), so its row is real
        const double cs = std::cos(a), sn = (k == C.K) ? 0.0 : std::sin(a);
        H.dense_e5[(size_t)k * C.n_det + d] = make_float2((float)(ck * cs), (float)(ck * sn));
        H.dense_e5t[(size_t)k * C.n_det + d] = make_float2((float)cs, (float)sn);
      }
    }
    if (C.k5tc_kp > 0) {   // tcgen05 synthesis operand B[2k][d] = Re E5, B[2k+1][d] = -Im E5
      const int KP = C.k5tc_kp, D = (C.n_det + 127) / 128 * 128;
      pack_kmajor(H.k5tc_b, D / 128, 128, KP, [&](int d, int kp) -> float {
        if (d >= C.n_det || kp >= 2 * C.Kp) return 0.f;
        const float2 e = H.dense_e5[(size_t)(kp / 2) * C.n_det + d];
        return (kp & 1) ? -e.y : e.x;
      });
    }
    if (C.k5ttc_kp > 0)   // tcgen05 analysis operand B[d][2k] = Re E5T, B[d][2k+1] = -Im E5T
      pack_kmajor(H.k5ttc_b, C.k5ttc_nb, C.k5ttc_nt, C.k5ttc_kp, [&](int j, int d) -> float {
        if (d >= C.n_det || j >= 2 * C.Kp) return 0.f;
        const float2 e = H.dense_e5t[(size_t)(j / 2) * C.n_det + d];
        return (j & 1) ? -e.y : e.x;
      });
  }

  // ---- half-plane polar nodes (Alg. 1 step 3; readings G12, G13)
  const int half = C.half;
  const long nodes = (long)half * NL;
  std::vector<int> p0v(nodes), q0v(nodes);
  std::vector<double> av(nodes), bv(nodes);
  for (int lp = 0; lp < half; ++lp) {
    int l = ((lp - nphi / 4) % nphi + nphi) % nphi;
    double cs, sn;
    unit_circle(l, nphi, cs, sn);
    for (int j = 0; j < NL; ++j) {
      double rho = (j * C.Lbox) / C.T_new;        // lambda_j / dxi
      double u = rho * cs, v = rho * sn;
      double fu = std::floor(u), fv = std::floor(v);
      long i = (long)lp * NL + j;
      int p0 = (int)fu;
      double a = u - fu;
      if (p0 >= N / 2) { p0 = N / 2; a = 0.0; }   // edge: the p0+1 column does not exist
      if (p0 < 0) { p0 = 0; a = 0.0; }            // u >= 0 on the half plane (cos >= 0)
      p0v[i] = p0; av[i] = a;
      q0v[i] = (int)fv; bv[i] = v - fv;
    }
  }
  // Node order: column blocks by p0 (k2_colptr), ring-major (j, then l') inside each column.
  // Forward S2 is ring-major [j][l'] (K2 gathers the nodes of a column in this order, so that
  // the nodes of one ring arc are stored to neighbouring slots; K3 reads whole rings).  The
  // adjoint S2 is in the node order itself (node_perm: (j, l') -> position): K3T stores a ring
  // group's nodes in destination order (k3t_dst, contiguous runs per column) and the K2T
  // target sums read one contiguous window per column / strip.  (Measured: the forward in node
  // order too, K3 reading through k3t_dst, was K2 -3.6 us but K3 +17.5 us at C3.)
  H.k2_colptr.assign(C.ncols + 1, 0);
  for (long i = 0; i < nodes; ++i) H.k2_colptr[p0v[i] + 1]++;
  for (int p = 0; p < C.ncols; ++p) H.k2_colptr[p + 1] += H.k2_colptr[p];
  H.k2_nodes.resize(nodes);
  H.node_perm.assign(nodes, 0);
  std::vector<int> sorted_pos(nodes);
  {
    std::vector<int> pos(H.k2_colptr.begin(), H.k2_colptr.end() - 1);
    for (int j = 0; j < NL; ++j)
      for (int lp = 0; lp < half; ++lp) {
        const long i = (long)lp * NL + j;
        const int sp = pos[p0v[i]]++;
        sorted_pos[i] = sp;
        H.node_perm[(size_t)j * half + lp] = sp;
        int4 e;
        e.x = j * half + lp;   // forward S2 slot, ring-major [j][l']
        e.y = q0v[i];
        e.z = fbits((float)av[i]);
        e.w = fbits((float)bv[i]);
        H.k2_nodes[sp] = e;
      }
  }
  // K3T output order: per ring group of 2G rings (one K3T CTA; G = min(4096 / n_phi, 16)), its
  // nodes sorted by adjoint position: (position, (ring in group) << 11 | l')
  {
    const int G2 = k3t_group_rings(C);
    H.k3t_dst.clear();
    H.k3t_dst.reserve(nodes);
    for (int j0 = 0; j0 < NL; j0 += G2) {
      const size_t base = H.k3t_dst.size();
      for (int jj = 0; jj < G2 && j0 + jj < NL; ++jj)
        for (int lp = 0; lp < half; ++lp)
          H.k3t_dst.push_back(make_int2(H.node_perm[(size_t)(j0 + jj) * half + lp], (jj << 11) | lp));
      std::sort(H.k3t_dst.begin() + base, H.k3t_dst.end(),
                [](const int2& a, const int2& b) { return a.x < b.x; });
    }
  }
  // K2T: entries (p, q mod N, src, w) for corners with non-zero weight; group by (p, q)
  struct Ent { int p, q, src; float w; };
  std::vector<Ent> ent;
  ent.reserve(nodes * 4);
  for (long i = 0; i < nodes; ++i) {
    double a = av[i], b = bv[i];
    int p0 = p0v[i], q0 = q0v[i];
    const double w[4] = {(1 - a) * (1 - b), a * (1 - b), (1 - a) * b, a * b};
    const int pp[4] = {p0, p0 + 1, p0, p0 + 1};
    const int qq[4] = {q0, q0, q0 + 1, q0 + 1};
    for (int c4 = 0; c4 < 4; ++c4) {
      if (w[c4] == 0.0) continue;
      int qm = ((qq[c4] % N) + N) % N;
      ent.push_back({pp[c4], qm, sorted_pos[i], (float)w[c4]});
    }
  }
  // two-pass stable counting sort: by key(q), then by p.  key(q) = (q mod Q0, q / Q0) with
  // Q0 = col_R(n) L orders a column's targets by the (q0, q1) split of kernels_col.cu
  const int Q0 = col_R(n) * L;
  auto qkey = [&](int q) { return (q % Q0) * (N / Q0) + q / Q0; };
  {
    std::vector<int> cnt(N + 1, 0);
    for (auto& e : ent) cnt[qkey(e.q) + 1]++;
    for (int q = 0; q < N; ++q) cnt[q + 1] += cnt[q];
    std::vector<Ent> tmp(ent.size());
    for (auto& e : ent) tmp[cnt[qkey(e.q)]++] = e;
    std::vector<int> cp(C.ncols + 1, 0);
    for (auto& e : tmp) cp[e.p + 1]++;
    for (int p = 0; p < C.ncols; ++p) cp[p + 1] += cp[p];
    for (auto& e : tmp) ent[cp[e.p]++] = e;
  }
  H.k2t_colptr.assign(C.ncols + 1, 0);
  H.k2t_tq.clear();
  H.k2t_tstart.clear();
  H.k2t_ent.resize(ent.size());
  for (size_t e = 0; e < ent.size(); ++e) {
    if (e == 0 || ent[e].p != ent[e - 1].p || ent[e].q != ent[e - 1].q) {
      H.k2t_tq.push_back(ent[e].q);
      H.k2t_tstart.push_back((int)e);
      H.k2t_colptr[ent[e].p + 1]++;
    }
    H.k2t_ent[e] = make_int2(ent[e].src, fbits(ent[e].w));
  }
  H.k2t_tstart.push_back((int)ent.size());
  for (int p = 0; p < C.ncols; ++p) H.k2t_colptr[p + 1] += H.k2t_colptr[p];
  // fixed-size target records (98.8 % of the C3 targets have one or two entries)
  {
    const size_t T = H.k2t_tq.size();
    H.k2t_rec.resize(T);
    H.k2t_ov.clear();
    for (size_t t = 0; t < T; ++t) {
      const int e0 = H.k2t_tstart[t], e1 = H.k2t_tstart[t + 1], cnt = e1 - e0;
      const int2 a = H.k2t_ent[e0];
      if (cnt == 1) {
        H.k2t_rec[t] = make_int4(a.x, a.y, a.x, 0);
      } else if (cnt == 2) {
        const int2 c2 = H.k2t_ent[e0 + 1];
        H.k2t_rec[t] = make_int4(a.x, a.y, c2.x, c2.y);
      } else {
        H.k2t_rec[t] = make_int4(a.x, a.y, -((int)H.k2t_ov.size() + 1), cnt);
        for (int e = e0 + 1; e < e1; ++e) H.k2t_ov.push_back(H.k2t_ent[e]);
      }
    }
  }
  // k2c_adj: per (p, q0) presence mask over q1 and first target index
  if (col_ok(C)) {
    H.k2c_mask.assign((size_t)C.ncols * Q0, 0u);
    H.k2c_base.assign((size_t)C.ncols * Q0, 0);
    for (int p = 0; p < C.ncols; ++p) {
      for (int t = H.k2t_colptr[p + 1] - 1; t >= H.k2t_colptr[p]; --t) {
        const int q = H.k2t_tq[t], q0 = q % Q0, q1 = q / Q0;
        H.k2c_mask[(size_t)p * Q0 + q0] |= 1u << q1;
        H.k2c_base[(size_t)p * Q0 + q0] = t;
      }
    }
    // fused adjoint column stage (k2c_adjf): the same target records with node references
    // relative to the column's node window (nodes with p0 in {p-1, p}, one contiguous range of
    // the adjoint S2), 12 bytes each {i0 | i1 << 16, w0, w1}; a target with more than two
    // entries has i1 = 0xFFFF, w0 = first index into k2f_ov, w1 = entry count (bit patterns).
    // Each column's block starts at a multiple of 4 records (48 bytes: 16-B bulk copies).
    H.k2f_recptr.assign(C.ncols + 1, 0);
    H.k2f_rec.clear();
    H.k2f_ov.clear();
    H.k2f_ovt.clear();
    H.k2f_ovptr.assign(1, 0);
    bool fits = true;
    for (int p = 0; p < C.ncols; ++p) {
      const int wlo = H.k2_colptr[p > 0 ? p - 1 : 0], whi = H.k2_colptr[p + 1];
      if (whi - wlo >= 0xFFFF) fits = false;
      H.k2f_recptr[p] = (int)(H.k2f_rec.size() / 3);
      for (int t = H.k2t_colptr[p]; t < H.k2t_colptr[p + 1]; ++t) {
        const int e0 = H.k2t_tstart[t], e1 = H.k2t_tstart[t + 1];
        auto rel = [&](int src) {
          if (src < wlo || src >= whi) fits = false;
          return (uint32_t)(src - wlo);
        };
        if (e1 - e0 <= 2) {
          const int2 a = H.k2t_ent[e0];
          const int2 c = (e1 - e0 == 2) ? H.k2t_ent[e0 + 1] : make_int2(a.x, 0);
          H.k2f_rec.push_back(rel(a.x) | (rel(c.x) << 16));
          H.k2f_rec.push_back((uint32_t)a.y);
          H.k2f_rec.push_back((uint32_t)c.y);
        } else {   // summed by one warp in the kernel's second pass (k2f_ovt)
          H.k2f_ovt.push_back(make_int4(t - H.k2t_colptr[p], (int)H.k2f_ov.size(), e1 - e0, 0));
          H.k2f_rec.push_back(0xFFFF0000u);
          H.k2f_rec.push_back((uint32_t)H.k2f_ov.size());
          H.k2f_rec.push_back((uint32_t)(e1 - e0));
          for (int e = e0; e < e1; ++e) H.k2f_ov.push_back(make_int2((int)rel(H.k2t_ent[e].x), H.k2t_ent[e].y));
        }
      }
      H.k2f_ovptr.push_back((int)H.k2f_ovt.size());
      while ((H.k2f_rec.size() / 3) % 4) {   // pad the column block to 4 records
        H.k2f_rec.push_back(0u);
        H.k2f_rec.push_back(0u);
        H.k2f_rec.push_back(0u);
      }
    }
    H.k2f_recptr[C.ncols] = (int)(H.k2f_rec.size() / 3);
    if (!fits) H.k2f_recptr.clear();   // window too large for 16-bit offsets: no fused stage

    // k2t_strip (the transposed bilinear as a streaming kernel): columns grouped into strips
    // whose union node window (p0 in [P0-1, P1-1]) and target count stay under kStripNodes /
    // kStripTargets; records {i0 | i1 << 16, w0, w1} relative to the strip's window; targets with
    // more than two entries: i1 = 0xFFFF, w0 = index into k2s_ovt (summed by one warp each)
    H.k2s_strip.clear();
    H.k2s_rec.clear();
    H.k2s_ovt.clear();
    H.k2s_ov.clear();
    H.k2s_ovptr.assign(1, 0);
    const long kStripOvBytes = strip_ov_bytes(C.n);
    H.k2s_ovcap = (int)kStripOvBytes;
    bool sfits = true;
    std::vector<long> ovb(C.ncols, 0);   // overflow-list bytes of each column (targets with > 2 entries)
    for (int p = 0; p < C.ncols; ++p)
      for (int t = H.k2t_colptr[p]; t < H.k2t_colptr[p + 1]; ++t) {
        const int cnt = H.k2t_tstart[t + 1] - H.k2t_tstart[t];
        if (cnt > 2) ovb[p] += 16 + 8L * cnt;
      }
    for (int P0 = 0; P0 < C.ncols;) {
      const int wlo = H.k2_colptr[P0 > 0 ? P0 - 1 : 0];
      int P1 = P0 + 1;
      long ob = ovb[P0];
      while (P1 < C.ncols && H.k2_colptr[P1 + 1] - wlo <= kStripNodes &&
             H.k2t_colptr[P1 + 1] - H.k2t_colptr[P0] <= kStripTargets && ob + ovb[P1] <= kStripOvBytes)
        ob += ovb[P1++];
      const int whi = H.k2_colptr[P1];
      if (whi - wlo >= 0xFFFF) sfits = false;   // 16-bit window offsets
      const int ta = H.k2t_colptr[P0], tb2 = H.k2t_colptr[P1];
      H.k2s_strip.push_back(make_int4(wlo, whi - wlo, ta, tb2 - ta));
      for (int t = ta; t < tb2; ++t) {
        const int e0 = H.k2t_tstart[t], e1 = H.k2t_tstart[t + 1];
        auto rel = [&](int src) { return (uint32_t)(src - wlo); };
        if (e1 - e0 <= 2) {
          const int2 a = H.k2t_ent[e0];
          const int2 c = (e1 - e0 == 2) ? H.k2t_ent[e0 + 1] : make_int2(a.x, 0);
          H.k2s_rec.push_back(rel(a.x) | (rel(c.x) << 16));
          H.k2s_rec.push_back((uint32_t)a.y);
          H.k2s_rec.push_back((uint32_t)c.y);
        } else {
          H.k2s_rec.push_back(0xFFFF0000u);
          H.k2s_rec.push_back((uint32_t)H.k2s_ovt.size());
          H.k2s_rec.push_back((uint32_t)(e1 - e0));
          H.k2s_ovt.push_back(make_int4(t - ta, (int)H.k2s_ov.size(), e1 - e0, 0));
          for (int e = e0; e < e1; ++e) H.k2s_ov.push_back(make_int2((int)rel(H.k2t_ent[e].x), H.k2t_ent[e].y));
        }
      }
      H.k2s_ovptr.push_back((int)H.k2s_ovt.size());
      P0 = P1;
    }
    if (!sfits) H.k2s_strip.clear();
    // heavy strips (single origin-region columns whose overflow lists or node window exceed the
    // shared-memory budgets) first, so that they run one image per CTA at the head of the grid
    // and read global memory; every strip carries its own overflow range (k2s_ovr)
    {
      std::vector<int> heavy, light;
      const int ns = (int)H.k2s_strip.size();
      for (int s = 0; s < ns; ++s) {
        size_t bytes = 0;   // overflow descriptors + entries, staged in shared memory
        for (int o = H.k2s_ovptr[s]; o < H.k2s_ovptr[s + 1]; ++o) bytes += 16 + 8 * (size_t)H.k2s_ovt[o].z;
        const bool hv = bytes > (size_t)kStripOvBytes || H.k2s_strip[s].y > kStripNodes;
        (hv ? heavy : light).push_back(s);
      }
      std::vector<int4> st;
      H.k2s_ovr.clear();
      for (int pass = 0; pass < 2; ++pass)
        for (int s : pass ? light : heavy) {
          st.push_back(H.k2s_strip[s]);
          H.k2s_ovr.push_back(make_int2(H.k2s_ovptr[s], H.k2s_ovptr[s + 1]));
        }
      H.k2s_strip.swap(st);
      H.k2s_nheavy = (int)heavy.size();
    }
  }
}

}  // namespace tat

namespace tat {

// Inverse tables (Algorithm 3; readings G21-G23, see oracle/tat_oracle.py "Inverse").
void build_inverse_tables(const Consts& C, const std::vector<int>& node_perm, InvTables& I) {
  const int N = C.N, nphi = C.n_ring, half = C.half, NL = C.NL, Kp = C.Kp;
  // ---- step 3 multiplier (with step 2's 1/n_phi and step 6's dxi^2 / 2pi folded in)
  I.mult.assign((size_t)Kp * NL, 0.f);
  {
    std::vector<double> row(Kp + 1);
    const double scale = (C.dxi * C.dxi / (2.0 * kPi)) / nphi * C.dt;
    for (int j = 0; j < NL; ++j) {
      bessel_row(j * C.dlam, C.K + 1, row.data());
      for (int k = 0; k < Kp; ++k) {
        const double jp = (k == 0) ? -row[1] : 0.5 * (row[k - 1] - row[k + 1]);   // J'_k
        I.mult[(size_t)k * NL + j] = (float)(scale * (-2.0 * jp));
      }
    }
  }
  // ---- step 5 targets: Cartesian (p, q), p in [0, N/2], |xi| < lambda_max
  const int Q0 = col_R(C.n) * C.Lres;
  auto code = [&](int j, long l) {
    const long lp = ((l + nphi / 4) % nphi + nphi) % nphi;
    if (lp < half) return node_perm[(size_t)j * half + lp];
    return -(node_perm[(size_t)j * half + (lp - half)] + 1);
  };
  struct Tg { int key, q; int4 nd; float4 w; };
  std::vector<Tg> col;
  const double rscale = C.dxi / C.dlam, tscale = nphi / (2.0 * kPi);
  // pass 0: natural q order (every column is a chord of the disk, |q| <= Q_p: the condition is
  // symmetric and monotone in |q|); pass 1 (only if some column were not): the (q0, q1) order
  // of the mask / base path
  for (int pass = 0; pass < 2; ++pass) {
  I.colptr.assign(C.ncols + 1, 0);
  I.nodes.clear();
  I.w.clear();
  I.tq.clear();
  I.chord.clear();
  I.max_per_col = 0;
  bool chords = true;
  for (int p = 0; p < C.ncols; ++p) {
    col.clear();
    for (int q = -N / 2; q < N / 2; ++q) {
      const double rho = std::hypot((double)p, (double)q) * rscale;
      if (!(rho < C.J - 1e-9)) continue;
      double th = std::fmod(std::atan2((double)q, (double)p), 2.0 * kPi);
      if (th < 0) th += 2.0 * kPi;
      th *= tscale;
      const int j0 = std::min((int)std::floor(rho), C.J - 1);
      const double a = rho - j0;
      const double l0f = std::floor(th), bb = th - l0f;
      const long l0 = (((long)l0f) % nphi + nphi) % nphi, l1 = (l0 + 1) % nphi;
      const double hw = (p == 0) ? 0.5 : 1.0;   // Hermitian half spectrum (K1T doubles p = 0)
      Tg t;
      t.q = ((q % N) + N) % N;
      t.key = pass == 0 ? q : (t.q % Q0) * (N / Q0) + t.q / Q0;   // pass 0: along the chord
      t.nd = make_int4(code(j0, l0), code(j0 + 1, l0), code(j0, l1), code(j0 + 1, l1));
      t.w = make_float4((float)(hw * (1 - a) * (1 - bb)), (float)(hw * a * (1 - bb)),
                        (float)(hw * (1 - a) * bb), (float)(hw * a * bb));
      col.push_back(t);
    }
    std::sort(col.begin(), col.end(), [](const Tg& x, const Tg& y) { return x.key < y.key; });
    for (const Tg& t : col) {
      I.nodes.push_back(t.nd);
      I.w.push_back(t.w);
      I.tq.push_back(t.q);
    }
    I.colptr[p + 1] = I.colptr[p] + (int)col.size();
    I.max_per_col = std::max(I.max_per_col, (int)col.size());
    I.chord.push_back(col.empty() ? -1 : -col.front().key);
    if (!col.empty() && (col.back().key != -col.front().key || (int)col.size() != 2 * col.back().key + 1))
      chords = false;
  }
  if (pass == 0 && chords) break;
  I.chord.clear();   // pass 1: no chord table (k2c_adj uses mask / base)
  }
  I.mask.clear();
  I.base.clear();
  if (col_ok(C)) {
    I.mask.assign((size_t)C.ncols * Q0, 0u);
    I.base.assign((size_t)C.ncols * Q0, 0);
    for (int p = 0; p < C.ncols; ++p)
      for (int t = I.colptr[p + 1] - 1; t >= I.colptr[p]; --t) {
        const int q = I.tq[t], q0 = q % Q0, q1 = q / Q0;
        I.mask[(size_t)p * Q0 + q0] |= 1u << q1;
        I.base[(size_t)p * Q0 + q0] = t;
      }
  }
}

}  // namespace tat
