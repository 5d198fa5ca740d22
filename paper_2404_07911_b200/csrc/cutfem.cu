// cutfem.cu — C ABI (include/cutfem.h): setup, stream-ordered apply, CSR path.
//
// setup (host, once; SURVEY §3 call stack 2): validate the arrays, build the
// 1-D tables (tables.h), the per-cell descriptors (face neighbours, face types,
// ghost-penalty faces), sort cut cells by decreasing point count (heaviest
// first: "cut cells are batched by quadrature-point count", north_star), and
// upload everything.  apply: the structured kernel on the caller's stream and
// the unstructured kernel on a forked side stream (they write disjoint v
// blocks), joined by an event — no host synchronisation.
#include <cuda_runtime.h>
#include <cusparse.h>
#include <nccl.h>

#include <algorithm>
#include <array>
#include <type_traits>
#include <map>
#include <unordered_map>
#include <queue>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>
#include <unordered_map>
#include <map>
#include <vector>

#include "../../include/cutfem.h"
#ifndef CUTFEM_CUT1_MAXN
#define CUTFEM_CUT1_MAXN 3  // n <= this: a few threads per cut cell (k_cut1) instead of a warp (k_cutp)
#endif
#ifndef CUT1_TPC2
#define CUT1_TPC2 1  // k_cut1 threads per cut cell at n = 2 (2: kernel alone 69.7 -> 57.3 us, apply 119.9 -> 121.9)
#endif
#ifndef CUT1_TPC3
#define CUT1_TPC3 2  // ... at n = 3 (C3 p=2 apply: 1 thread 246, 2: 213, 4: 236, 8: 282 us; k_cutp<3> 238)
#endif
#include "kernels.cuh"
#include "tables.h"
#ifndef CUT_ORDER
#define CUT_ORDER 2  // measured: C5 apply 5566 -> 5457 us, C3 p=6 -1 %, p=8 neutral (pure spatial: p=8 +30 %)
#endif
#ifndef CUT_HEAVY_PCT
#define CUT_HEAVY_PCT 5
#endif

namespace {

thread_local std::string g_err;

int fail(int code, const std::string &msg) {
  g_err = msg;
  return code;
}

#define CU(call)                                                                         \
  do {                                                                                   \
    cudaError_t e_ = (call);                                                             \
    if (e_ != cudaSuccess)                                                               \
      return fail(CUTFEM_ECUDA, std::string(#call) + ": " + cudaGetErrorString(e_));     \
  } while (0)

}  // namespace

struct cutfem_cg_work;                    // cg.inl
void cg_free(cutfem_cg_work *w);

struct cutfem_handle {
  int device = 0;
  int degree = 1;
  int n = 2;
  double h = 1;
  int64_t n_active = 0, n_uncut = 0, n_cut = 0;
  int64_t n_plain = 0;     // uncut cells whose six neighbours are active and uncut (first in d_udesc)
  int64_t n_own = 0;       // computed blocks (= n_active unless distributed; ghosts follow)
  // descriptor ranges per part (0 all, 1 interior, 2 slab boundary): plain, general, cut
  int64_t r_off[3][3] = {{0}}, r_cnt[3][3] = {{0}};
  // distributed (x-slab) state
  int rank = 0, nranks = 1;
  bool dist = false;
  int64_t ghost_lo = 0, ghost_hi = 0;      // ghost blocks after the owned ones
  int64_t plane_lo = 0, plane_hi = 0;      // owned blocks of the first / last owned plane
  void *comm = nullptr;                    // ncclComm_t
  // test-only NCCL loopback (cutfem_debug_loopback): a 1-rank communicator whose
  // halo exchange sends these caller buffers to itself into the ghost slots
  bool loopback = false;
  const double *lb_lo = nullptr, *lb_hi = nullptr;
  cudaStream_t comm_stream = nullptr;
  cudaEvent_t ev_comm = nullptr, ev_comm_fork = nullptr;
  int sm_count = 148;
  uint32_t mask = CUTFEM_TERM_ALL;
  KParams kp;
  FaceTab ft;
  // thread-per-cell structured kernel (N <= 4): warp-tiles per part (0 all, 1 interior, 2 boundary)
  // tile sets: [0] uncut cells, volume + SIPG (v = ...); [1] cells with ghost-
  // penalty faces (cut cells and their uncut neighbours) + the cut cells'
  // full-face SIPG
  void *d_tiles = nullptr;
  int64_t t_off[3][3] = {{0}}, t_cnt[3][3] = {{0}};
  int occ_tile[3] = {1, 1, 1};
  std::vector<char> ttab;  // TileTab<N> bytes
  CDesc2 *d_cdesc2 = nullptr;  // k_cutp: cut cells grouped per warp (LPT), their cut-face points
  double *d_fac = nullptr;
  int *d_wstart = nullptr;      // per part: warp -> first cell (grid_cutp[part] * WARPS + 1 entries)
  int *d_kstart = nullptr;      // per part: warp -> first packet
  CPacket *d_chunks = nullptr;  // packets of the point-chunk stream, per warp in consumption order
  char *d_stream = nullptr;     // the packed stream (chunk headers + point rows)
  int64_t w_off[3] = {0};
  int grid_cutp[3] = {0};
  int occ_cutp = 1;
  UDesc *d_udesc = nullptr;
  CDesc *d_cdesc = nullptr;
  double *d_vol = nullptr, *d_srf = nullptr, *d_sfp = nullptr;
  int64_t *d_volptr = nullptr, *d_srfptr = nullptr, *d_sfptr = nullptr;
  double *d_line_srf = nullptr;  // k_cut line cells: per volume line its interface point [t, W, n_ax, n_B1, n_B2, 0]
                                 // (W = 0: none), staged with the line's points
  cudaStream_t side = nullptr;
  cudaEvent_t ev_fork = nullptr, ev_join = nullptr;
  cudaEvent_t ev_started = nullptr;  // k_cutp launch completion (all CTAs begun)
  // host path buffers (the batched path: two pairs, copy streams, events)
  double *d_u = nullptr, *d_v = nullptr;
  double *d_ub[2] = {nullptr, nullptr}, *d_vb[2] = {nullptr, nullptr};
  cudaStream_t s_h2d = nullptr, s_d2h = nullptr;
  cudaEvent_t ev_in[2] = {nullptr, nullptr}, ev_done[2] = {nullptr, nullptr}, ev_out[2] = {nullptr, nullptr};
  // CSR
  int64_t csr_nnz = 0;
  bool csr_i64 = false;
  void *d_rowptr = nullptr, *d_col = nullptr;
  double *d_val = nullptr;
  void *d_spbuf = nullptr;
  size_t spbuf_size = 0;
  cusparseHandle_t sp = nullptr;
  cusparseSpMatDescr_t spA = nullptr;
  std::vector<uint8_t> color;  // (i + 2j + 3k) mod 7, distance-2 colouring for CSR probing
  cutfem_stats_t stats;
  int64_t dev_bytes = 0;
  cutfem_cg_work *cg = nullptr;  // CG work vectors (lazy)
  std::vector<int32_t> blk_ijk;  // cell of every block (owned, then ghosts): probe colouring
  std::vector<uint8_t> blk_cut;  // is_cut of every block (owned, then ghosts): multigrid block classes
  int32_t n_cells[3] = {0, 0, 0};
  double lower[3] = {0, 0, 0};
};

namespace {

template <class T>
int upload(cutfem_handle *hd, T **dst, const T *src, size_t count) {
  size_t bytes = sizeof(T) * std::max<size_t>(count, 1);
  cudaError_t e = cudaMalloc((void **)dst, bytes);
  if (e != cudaSuccess) return fail(CUTFEM_ENOMEM, std::string("cudaMalloc: ") + cudaGetErrorString(e));
  hd->dev_bytes += (int64_t)bytes;
  if (count) CU(cudaMemcpy(*dst, src, sizeof(T) * count, cudaMemcpyHostToDevice));
  return 0;
}

void make_eo(int n, const std::vector<long double> &Mx, EO &out) {
  std::memset(&out, 0, sizeof(out));
  const int H = n / 2, HC = (n + 1) / 2;
  for (int i = 0; i < HC; ++i) {
    for (int j = 0; j < H; ++j)
      out.E[i * HC + j] = (double)((Mx[i * n + j] + Mx[i * n + (n - 1 - j)]) / 2);
    if (n & 1) out.E[i * HC + H] = (double)Mx[i * n + H];
  }
  for (int i = 0; i < H; ++i)
    for (int j = 0; j < H; ++j) out.O[i * H + j] = (double)((Mx[i * n + j] - Mx[i * n + (n - 1 - j)]) / 2);
}

int upload_tables(int p) {
  cutfem_tables::Ref r = cutfem_tables::build(p);
  const int n = p + 1;
  RefTab t;
  std::memset(&t, 0, sizeof(t));
  std::vector<long double> St(n * n);
  for (int a = 0; a < n; ++a)
    for (int b = 0; b < n; ++b) St[a * n + b] = r.S[b * n + a];
  make_eo(n, r.S, t.S);
  make_eo(n, St, t.St);
  make_eo(n, r.Kc, t.Kc);
  make_eo(n, r.M, t.M);
  for (int a = 0; a < n; ++a) {
    t.x[a] = (double)r.x[a];
    t.cinv[a] = (double)r.cinv[a];
    t.gw[a] = (double)r.w[a];
    t.d0[a] = (double)r.tr[(1 * 2 + 0) * n + a];
    t.d1[a] = (double)r.tr[(1 * 2 + 1) * n + a];
  }
  // monomial coefficients of l_a in t = 2x - 1 (product expansion in long double)
  for (int a = 0; a < n; ++a) {
    std::vector<long double> c(1, 1.0L);
    for (int m = 0; m < n; ++m) {
      if (m == a) continue;
      const long double tm = 2 * r.x[m] - 1, den = (2 * r.x[a] - 1) - tm;
      std::vector<long double> d(c.size() + 1, 0.0L);
      for (size_t k = 0; k < c.size(); ++k) {
        d[k + 1] += c[k] / den;
        d[k] -= c[k] * tm / den;
      }
      c.swap(d);
    }
    for (int k = 0; k < n; ++k) {
      t.mc[a][k] = (double)c[k];
      t.md[a][k] = (double)(2 * k * c[k]);
    }
  }
  CU(cudaMemcpyToSymbol(c_ref, &t, sizeof(RefTab), sizeof(RefTab) * (n - 2)));
  return 0;
}

// The 1-D ghost-penalty coupling of a face, own cell on the PLUS side (its lo face):
// the face's stabilisation matrix is  (this 2n x 2n own/neighbour coupling) (x) in-face
// mass M (x) M  for both kinds, so both run through the same line-operator code.
//   face GP (BASELINE configs[0]): own-own  h sum_j g_j l_m^(j)(0) l_a^(j)(0),
//     own-nb  -h sum_j g_j l_m^(j)(0) l_a^(j)(1)   (jump [.] = (.)^- - (.)^+, physical
//     derivatives: g_j h^(2j-1) h^-2j h^2 = g_j h)
//   volume GP: the patch E1 u E2 in the own cell's coordinates is
//     [-1, 1] (the neighbour E1 at [-1, 0]); tau_v / h^2 int_P (u1 - u2)(v1 - v2) with
//     the polynomials extended over the patch = tau_v h [G (x) M (x) M],
//     own-own  tau_v h int_{-1}^{1} l_m l_a,  own-nb  -tau_v h int_{-1}^{1} l_m(y) l_a(y+1)
//     ((p+1)-point Gauss on [-1,0] and [0,1]: exact for the degree-2p products).
// The own-MINUS blocks are the centro-symmetric mirrors (GLL symmetry).
void gp_blocks(int p, double h, const double *gpg, int kind, double tau_v, std::vector<long double> &oo,
               std::vector<long double> &on) {
  typedef long double ld;
  const int n = p + 1;
  cutfem_tables::Ref r = cutfem_tables::build(p);
  oo.assign(n * n, 0);
  on.assign(n * n, 0);
  auto tr = [&](int j, int s, int a) { return r.tr[(j * 2 + s) * n + a]; };
  for (int m = 0; m < n; ++m)
    for (int a = 0; a < n; ++a) {
      if (kind == CUTFEM_GP_FACE) {
        for (int j = 0; j <= p; ++j) {
          oo[m * n + a] += (ld)h * gpg[j] * tr(j, 0, m) * tr(j, 0, a);
          on[m * n + a] -= (ld)h * gpg[j] * tr(j, 0, m) * tr(j, 1, a);
        }
      } else {
        ld so = 0, sn = 0;
        for (int q = 0; q < n; ++q)
          for (int half = 0; half < 2; ++half) {
            const ld y = r.g[q] - (half ? 0 : 1);  // [-1,0] then [0,1]
            const ld lm = cutfem_tables::lag(r.x, m, y);
            so += r.w[q] * lm * cutfem_tables::lag(r.x, a, y);
            sn += r.w[q] * lm * cutfem_tables::lag(r.x, a, y + 1);
          }
        oo[m * n + a] = (ld)tau_v * h * so;
        on[m * n + a] = -(ld)tau_v * h * sn;
      }
    }
}

void build_facetab(int p, double h, const double *gpg, int kind, double tau_v, FaceTab &ft) {
  const int n = p + 1;
  std::vector<long double> oo, on;
  gp_blocks(p, h, gpg, kind, tau_v, oo, on);
  std::memset(&ft, 0, sizeof(ft));
  // ft[s]: s = 0 own minus (mirror), s = 1 own plus; the kernels compute Goo uo - Gon un
  for (int m = 0; m < n; ++m)
    for (int a = 0; a < n; ++a) {
      const int k = m * n + a, km = (n - 1 - m) * n + (n - 1 - a);
      ft.Goo[1][k] = (double)oo[k];
      ft.Gon[1][k] = (double)(-on[k]);
      ft.Goo[0][k] = (double)oo[km];
      ft.Gon[0][k] = (double)(-on[km]);
    }
}

// ---- k_tile: per-handle line operators (long double, then rounded)
template <int N>
void build_tiletab(double h, double sipg_gamma, const double *gpg, int gp_kind, double tau_v, uint32_t mask,
                   TileTab<N> &tt) {
  typedef long double ld;
  const int p = N - 1, n = N;
  cutfem_tables::Ref r = cutfem_tables::build(p);
  std::vector<ld> K1(n * n, 0), Mi(n * n, 0), A(n * n);
  for (int a = 0; a < n; ++a)
    for (int b = 0; b < n; ++b) {
      ld k = 0;
      for (int q = 0; q < n; ++q)
        k += r.w[q] * cutfem_tables::dlag(r.x, a, r.g[q]) * cutfem_tables::dlag(r.x, b, r.g[q]);
      K1[a * n + b] = k;
    }
  // M^{-1} by Gauss-Jordan (M is SPD, well conditioned for n <= 9)
  for (int i = 0; i < n * n; ++i) A[i] = r.M[i];
  for (int i = 0; i < n; ++i) Mi[i * n + i] = 1;
  for (int c = 0; c < n; ++c) {
    int piv = c;
    for (int i = c + 1; i < n; ++i)
      if (std::fabs((double)A[i * n + c]) > std::fabs((double)A[piv * n + c])) piv = i;
    for (int j = 0; j < n; ++j) {
      std::swap(A[c * n + j], A[piv * n + j]);
      std::swap(Mi[c * n + j], Mi[piv * n + j]);
    }
    const ld d = A[c * n + c];
    for (int j = 0; j < n; ++j) {
      A[c * n + j] /= d;
      Mi[c * n + j] /= d;
    }
    for (int i = 0; i < n; ++i) {
      if (i == c) continue;
      const ld f = A[i * n + c];
      for (int j = 0; j < n; ++j) {
        A[i * n + j] -= f * A[c * n + j];
        Mi[i * n + j] -= f * Mi[c * n + j];
      }
    }
  }
  auto tr = [&](int j, int s, int a) { return r.tr[(j * 2 + s) * n + a]; };  // l_a^(j)(s)
  std::memset(&tt, 0, sizeof(tt));
  for (int i = 0; i < n; ++i)
    for (int j = 0; j < n; ++j) {
      ld x = 0;
      for (int k = 0; k < n; ++k) x += Mi[i * n + k] * K1[k * n + j];
      tt.L[i * n + j] = (double)(h * x);
      tt.M[i * n + j] = (double)r.M[i * n + j];
    }
  // lo face (own cell is the plus side, own face node 0); the hi face uses the
  // mirrored entries (see TileTab)
  const ld h2sig = (ld)h * sipg_gamma, hs = (ld)h / 2;
  for (int m = 0; m < n; ++m) {
    ld be = 0;
    for (int k = 0; k < n; ++k) be += Mi[m * n + k] * tr(1, 0, k);
    const ld al = Mi[m * n + 0];
    tt.cJ[m] = (double)(al * h2sig + be * hs);
    tt.cA[m] = (double)(al * hs);
    tt.d0[m] = (double)tr(1, 0, m);
  }
  // ghost penalty (lo face, own cell the plus side; gp_blocks): M^{-1}-premultiplied
  std::vector<ld> Goo, Gon;
  gp_blocks(p, h, gpg, gp_kind, tau_v, Goo, Gon);
  for (int m = 0; m < n; ++m)
    for (int a = 0; a < n; ++a) {
      ld go = 0, gn = 0;
      for (int k = 0; k < n; ++k) {
        go += Mi[m * n + k] * Goo[k * n + a];
        gn += Mi[m * n + k] * Gon[k * n + a];
      }
      tt.Goo[m * n + a] = (double)go;
      tt.Gon[m * n + a] = (double)gn;
    }
  // folded operator for cells with six faces (k_tile2): Lf = L (cell term) + the own
  // parts of both SIPG faces, lo face F[m][k] = cJ[m] delta_k0 + cA[m] d0[k], hi face its
  // mirror; neighbour coefficients nJ = -cJ, nA = -cA (0 without the SIPG term)
  const bool con = (mask & CUTFEM_TERM_CELL) != 0, son = (mask & CUTFEM_TERM_SIPG) != 0;
  for (int m = 0; m < n; ++m) {
    for (int k = 0; k < n; ++k) {
      ld x = con ? (ld)tt.L[m * n + k] : 0;
      if (son) {
        const int mm = n - 1 - m, km = n - 1 - k;
        x += (k == 0 ? (ld)tt.cJ[m] : 0) + (ld)tt.cA[m] * tt.d0[k];
        x += (km == 0 ? (ld)tt.cJ[mm] : 0) + (ld)tt.cA[mm] * tt.d0[km];
      }
      tt.Lf[m * n + k] = (double)x;
    }
    tt.nJ[m] = son ? -tt.cJ[m] : 0.0;
    tt.nA[m] = son ? -tt.cA[m] : 0.0;
  }
  {
    std::vector<ld> Ll(n * n), Ml(n * n);
    for (int k = 0; k < n * n; ++k) {
      Ll[k] = tt.L[k];
      Ml[k] = r.M[k];
    }
    make_eo(n, Ll, tt.Leo);
    make_eo(n, Ml, tt.Meo);
  }
}

template <int N>
int build_ttab(cutfem_handle *hd, const cutfem_problem *pb) {
  hd->ttab.resize(sizeof(TileTab<N>));
  build_tiletab<N>(pb->h, pb->sipg_gamma, pb->gp_gamma, pb->gp_kind, pb->tau_v, hd->mask,
                   *reinterpret_cast<TileTab<N> *>(hd->ttab.data()));
  return 0;
}

// ---- k_tile*: one cell of a tile set: block, face neighbours, face masks
struct TCell {
  int32_t blk;
  int32_t nb[6];
  uint32_t gp, sipg;  // faces (bits 0..5) with ghost penalty / SIPG in this pass
  bool vol;
};

// Group cells into warp-tiles of <= 32 cells (bricks of the background grid,
// partial bricks merged in brick order) and number the slots: own cells first
// (slot = cell index), then the face-neighbour halo of the faces with work, face
// by face (so that the lanes of one face read consecutive slots).
template <class C>
void build_tiles(const std::vector<TCell> &cells, const cutfem_problem *pb, std::vector<char> &out) {
  using R = TileRec<C::SMAX>;
  auto used = [&](const TCell &c, int f) { return c.nb[f] >= 0 && (((c.gp | c.sipg) >> f) & 1u); };
  std::vector<std::pair<int64_t, int64_t>> key(cells.size());
  for (size_t c = 0; c < cells.size(); ++c) {
    const int32_t *q = pb->active_ijk + 3 * (size_t)cells[c].blk;
    const int64_t bk = ((int64_t)(q[0] / C::BX) << 42) | ((int64_t)(q[1] / C::BY) << 21) | (int64_t)(q[2] / C::BZ);
    const int64_t in = ((int64_t)q[0] << 42) | ((int64_t)q[1] << 21) | (int64_t)q[2];
    key[c] = {bk, in};
  }
  std::vector<size_t> ord(cells.size());
  for (size_t c = 0; c < ord.size(); ++c) ord[c] = c;
  std::sort(ord.begin(), ord.end(), [&](size_t a, size_t b) { return key[a] < key[b]; });
  std::vector<R> tiles;
  std::vector<size_t> cur;
  std::unordered_map<int32_t, int> set;
  auto blocks_of = [&](const std::vector<size_t> &cs, std::unordered_map<int32_t, int> &m) {
    for (size_t c : cs) {
      m.emplace(cells[c].blk, 0);
      for (int f = 0; f < 6; ++f)
        if (used(cells[c], f)) m.emplace(cells[c].nb[f], 0);
    }
  };
  auto flush = [&]() {
    if (cur.empty()) return;
    R t;
    std::memset(&t, 0, sizeof(t));
    std::unordered_map<int32_t, int> slot;
    int ns = 0;
    for (size_t c : cur) {
      slot[cells[c].blk] = ns;
      t.blk[ns++] = cells[c].blk;
    }
    for (int f = 0; f < 6; ++f)
      for (size_t c : cur) {
        if (!used(cells[c], f)) continue;
        const int32_t nb = cells[c].nb[f];
        if (!slot.count(nb)) {
          slot[nb] = ns;
          t.blk[ns++] = nb;
        }
      }
    t.nslot = ns;
    t.ncell = (int32_t)cur.size();
    for (size_t l = 0; l < cur.size(); ++l) {
      const TCell &d = cells[cur[l]];
      uint32_t sl[6];
      for (int f = 0; f < 6; ++f) sl[f] = used(d, f) ? (uint32_t)slot[d.nb[f]] : 0xffu;
      const uint32_t gp = d.gp & 0x3fu, sp = d.sipg & 0x3fu;
      t.lane_nb[l][0] = sl[0] | (sl[1] << 8) | (sl[2] << 16) | (sl[3] << 24);
      t.lane_nb[l][1] = sl[4] | (sl[5] << 8) | (gp << 16) | (sp << 24) | ((d.vol ? 1u : 0u) << 30);
    }
    for (int l = (int)cur.size(); l < 32; ++l) {
      t.lane_nb[l][0] = 0xffffffffu;
      t.lane_nb[l][1] = 0x0000ffffu;
    }
    tiles.push_back(t);
    cur.clear();
    set.clear();
  };
  size_t i = 0;
  while (i < ord.size()) {
    size_t j = i;
    while (j < ord.size() && key[ord[j]].first == key[ord[i]].first) ++j;
    std::vector<size_t> g(ord.begin() + i, ord.begin() + j);
    std::unordered_map<int32_t, int> trial = set;
    blocks_of(g, trial);
    if ((int)(cur.size() + g.size()) > C::TC || (int)trial.size() > C::SMAX) {
      flush();
      trial.clear();
      blocks_of(g, trial);
    }
    cur.insert(cur.end(), g.begin(), g.end());
    set.swap(trial);
    i = j;
  }
  flush();
  out.resize(tiles.size() * sizeof(R));
  if (!tiles.empty()) std::memcpy(out.data(), tiles.data(), out.size());
}

// A cut cell's volume points in LINES: consecutive groups of n points that share
// two reference coordinates exactly (dimension-reduction quadrature), all along one
// axis.  Returns the axis (0..2) or -1 (the cell then streams single points).
static int vol_line_axis(const double *vp, int64_t nv, int n) {
  if (nv <= 0 || nv % n != 0 || n < 2) return -1;
  int ax = -1;
  for (int64_t g = 0; g < nv; g += n) {
    const double *a = vp + 4 * g;
    for (int t = 1; t < n; ++t) {
      const double *b = vp + 4 * (g + t);
      int diff = -1, nd = 0;
      for (int d = 0; d < 3; ++d)
        if (a[d] != b[d]) {
          diff = d;
          ++nd;
        }
      if (nd != 1) return -1;
      if (ax < 0) ax = diff;
      if (diff != ax) return -1;
    }
  }
  return ax;
}

// The interface points of a line cell that lie on its volume lines (same two base
// coordinates, at most one per line): line index per interface point, or empty if
// any point is off the lines (the cell then streams its interface points singly).
static std::vector<int> srf_on_lines(const double *vp, int64_t nv, const double *sp, int64_t ns, int n, int ax) {
  std::vector<int> li;
  if (ns <= 0) return li;
  const int b1 = ax == 0 ? 1 : 0, b2 = ax == 2 ? 1 : 2;
  std::map<std::pair<double, double>, int> key;
  for (int64_t l = 0; l < nv / n; ++l) key[{vp[4 * l * n + b1], vp[4 * l * n + b2]}] = (int)l;
  std::vector<char> used(nv / n, 0);
  li.resize(ns);
  for (int64_t q = 0; q < ns; ++q) {
    auto it = key.find({sp[7 * q + b1], sp[7 * q + b2]});
    if (it == key.end() || used[it->second]) return {};
    used[it->second] = 1;
    li[q] = it->second;
  }
  return li;
}

template <int N>
int setup_tiles(cutfem_handle *hd, const cutfem_problem *pb, const std::vector<UDesc> &ud,
                const std::vector<CDesc> &cd) {
  using C = TileCfg<N>;
  // per part (1 interior, 2 slab boundary): K1 = uncut cells, K2 = GP cells
  std::vector<TCell> set[3][2];
  for (int pt = 1; pt <= 2; ++pt) {
    for (int k = 0; k < 2; ++k)
      for (int64_t i = hd->r_off[pt][k]; i < hd->r_off[pt][k] + hd->r_cnt[pt][k]; ++i) {
        const UDesc &d = ud[i];
        TCell c;
        c.blk = d.blk;
        uint32_t nbm = 0;
        for (int f = 0; f < 6; ++f) {
          c.nb[f] = d.nb[f];
          if (d.nb[f] >= 0) nbm |= 1u << f;
        }
        // set 0 (k_tile2): cells without ghost-penalty faces; set 1 (k_uncw<4>): the
        // cells next to cut cells, every structured term (volume, SIPG, GP).  The two
        // sets and k_cutp's cut cells are disjoint: no kernel reads another's v.
        c.gp = d.flags & nbm & 0x3fu;
        c.sipg = nbm;  // faces of an uncut cell are inside the domain: full SIPG
        c.vol = true;
        // k_tile2 (folded operators) takes the cells with all six faces and no ghost
        // penalty; the rest (next to cut cells, on the box boundary) go to k_uncw<4>
        set[(c.gp || nbm != 0x3fu) ? 1 : 0][pt - 1].push_back(c);
      }

  }
  // set 0: k_tile2 tiles (Tile2Cfg<4>::T); set 1: k_uncw<4> tiles (TileCfg<4>).
  // Offsets are in BYTES.
  using CG = typename std::conditional<N == 4, TileCfgX<N, UNCW4_TC>, C>::type;
  using CK = typename std::conditional<N == 4, typename Tile2Cfg<4>::T, C>::type;
  std::vector<char> all;
  // (n <= 3: the uncut cells run k_cell from their descriptors; no tiles)
  for (int k = 0; k < (N == 4 ? 2 : 0); ++k) {
    const int64_t rs = k == 0 ? (int64_t)sizeof(TileRec<CK::SMAX>) : (int64_t)sizeof(TileRec<CG::SMAX>);
    std::vector<char> b0, b1;
    if (k == 0) {
      build_tiles<CK>(set[k][0], pb, b0);
      build_tiles<CK>(set[k][1], pb, b1);
    } else {
      build_tiles<CG>(set[k][0], pb, b0);
      build_tiles<CG>(set[k][1], pb, b1);
    }
    hd->t_off[k][0] = hd->t_off[k][1] = (int64_t)all.size();
    hd->t_cnt[k][1] = (int64_t)b0.size() / rs;
    hd->t_off[k][2] = hd->t_off[k][1] + (int64_t)b0.size();
    hd->t_cnt[k][2] = (int64_t)b1.size() / rs;
    hd->t_cnt[k][0] = hd->t_cnt[k][1] + hd->t_cnt[k][2];
    all.insert(all.end(), b0.begin(), b0.end());
    all.insert(all.end(), b1.begin(), b1.end());
  }
  int rc = upload(hd, reinterpret_cast<char **>(&hd->d_tiles), all.data(), all.size());
  if (rc) return rc;
  if constexpr (N > CUTFEM_CUT1_MAXN) {  // (n <= CUTFEM_CUT1_MAXN: k_cut1 reads the descriptors directly)
    // k_cutp: per cut cell its own list of cut-face points in its reference
    // coordinates [xi, eta, zeta, W] (normal coordinate exactly 0 or 1)
    std::vector<CDesc2> c2(cd.size());
    std::vector<double> fac;
    std::vector<std::array<int, 6>> fcn(cd.size());  // cut-face points per face of the cell
    for (size_t i = 0; i < cd.size(); ++i) {
      const CDesc &d = cd[i];
      CDesc2 &e = c2[i];
      std::memset(&e, 0, sizeof(e));
      e.blk = d.blk;
      e.vb = d.vb;
      e.sb = d.sb;
      e.nv = d.nv;
      e.ns = d.ns;
      e.fb = (int64_t)fac.size() / 4;
      for (int f = 0; f < 6; ++f) {
        e.nb[f] = d.nb[f] >= 0 ? d.nb[f] : -1;
        if (d.nb[f] >= 0) {
          if (d.flags & (1u << f)) e.smask |= 1u << f;               // ghost penalty (the cell is cut)
          if (d.flags & (1u << (6 + f))) e.smask |= 1u << (8 + f);   // full face inside Omega: SIPG
        }
        if (!((d.flags >> (12 + f)) & 1u) || d.nb[f] < 0) continue;
        e.fmask |= 1u << f;
        const int dd = f >> 1, e1 = dd == 0 ? 1 : 0, e2 = dd == 2 ? 1 : 2;
        for (int64_t q = pb->sf_ptr[d.sf[f]]; q < pb->sf_ptr[d.sf[f] + 1]; ++q) {
          double x[4];
          x[dd] = (f & 1) ? 1.0 : 0.0;
          x[e1] = pb->sf_pts[3 * q];
          x[e2] = pb->sf_pts[3 * q + 1];
          x[3] = pb->sf_pts[3 * q + 2];
          fac.insert(fac.end(), x, x + 4);
        }
        fcn[i][f] = (int)(pb->sf_ptr[d.sf[f] + 1] - pb->sf_ptr[d.sf[f]]);
      }
      e.nf = (int32_t)((int64_t)fac.size() / 4 - e.fb);
    }
    // cut-face points in LINES (k_cutp<4>, face_line_rt): per cell, line records
    // [xg, f + 8 la, (x_t, W_t) x N] into flrec (fl0[i] = the cell's first record, -1 if
    // some face's points are not all in lines: the cell then streams single points)
    std::vector<double> flrec;
    std::vector<int64_t> fl0(cd.size(), -1);
    std::vector<int> fln(cd.size(), 0);
    if constexpr (CutPCfg<N>::FLINES) {
      for (size_t i = 0; i < cd.size(); ++i) {
        const CDesc2 &e = c2[i];
        if (e.nf <= 0) continue;
        std::vector<double> rec;
        bool ok = true;
        int64_t row = e.fb;
        for (int f = 0; f < 6 && ok; ++f) {
          const int cnt = fcn[i][f];
          if (cnt % N != 0) ok = false;
          const int dd = f >> 1, e1 = dd == 0 ? 1 : 0, e2 = dd == 2 ? 1 : 2;
          for (int g = 0; g < cnt && ok; g += N) {
            const double *a = &fac[4 * (row + g)];
            int la = -1;
            for (int t = 1; t < N && ok; ++t) {
              const double *b = &fac[4 * (row + g + t)];
              const bool s1 = a[e1] == b[e1], s2 = a[e2] == b[e2];
              const int v = (s1 && !s2) ? e2 : ((s2 && !s1) ? e1 : -1);
              if (v < 0 || (la >= 0 && v != la)) ok = false;
              la = v;
            }
            if (!ok) break;
            const int ga = 3 - dd - la;
            rec.push_back(a[ga]);
            rec.push_back((double)(f + 8 * la));
            for (int t = 0; t < N; ++t) {
              rec.push_back(fac[4 * (row + g + t) + la]);
              rec.push_back(fac[4 * (row + g + t) + 3]);
            }
          }
          row += cnt;
        }
        if (!ok) continue;
        fl0[i] = (int64_t)flrec.size() / (2 + 2 * N);
        fln[i] = (int)(rec.size() / (2 + 2 * N));
        flrec.insert(flrec.end(), rec.begin(), rec.end());
      }
    }
    CU(cudaFuncSetAttribute(k_cutp<N>, cudaFuncAttributeMaxDynamicSharedMemorySize, CutPCfg<N>::SMEM));
    CU(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&hd->occ_cutp, k_cutp<N>, 32 * CutPCfg<N>::WARPS,
                                                     CutPCfg<N>::SMEM));
    hd->occ_cutp = std::max(1, hd->occ_cutp);
    // per part: longest-processing-time assignment of the cells to the warps of
    // the launch (cost ~ point chunks + a fixed per-cell part), cells of a warp
    // stored contiguously, heaviest first
    constexpr int WP = CutPCfg<N>::WARPS;
    std::vector<int> ws, ks;
    std::vector<CChunk> chunk;
    std::vector<CDesc2> c2o(c2.size());
    for (int pt = 1; pt <= 2; ++pt) {
      const int64_t o = hd->r_off[pt][2], n = hd->r_cnt[pt][2];
      const int grid = (int)std::max<int64_t>(1, std::min<int64_t>((n + WP - 1) / WP, (int64_t)hd->occ_cutp * hd->sm_count));
      hd->grid_cutp[pt] = n > 0 ? grid : 0;
      hd->w_off[pt] = (int64_t)ws.size();
      const int W = grid * WP;
      std::vector<int64_t> idx(n);
      // cost of a cell in point-chunk units: its chunks + a fixed per-cell part; volume
      // points in lines cost ~2.8 point chunks per 32 lines (128 points) at n = 4
      std::vector<char> isline(c2.size(), 0);
      for (int64_t i = 0; i < n; ++i) {
        const CDesc2 &e = c2[o + i];
        isline[o + i] = N >= 3 && e.nv > 0 && vol_line_axis(pb->vol_pts + 4 * e.vb, e.nv, N) >= 0;
      }
#ifndef CUTP_C_LINE
#define CUTP_C_LINE 2.8
#endif
#ifndef CUTP_C_FLINE
#define CUTP_C_FLINE 1.2
#endif
#ifndef CUTP_C_CELL
#define CUTP_C_CELL 1.5
#endif
#ifndef CUTP_C_SAX
#define CUTP_C_SAX 0.0
#endif
#ifndef CUTP_C_TRACE
#define CUTP_C_TRACE 0.0
#endif
      auto cost = [&](const CDesc2 &e) {
        const int64_t i = &e - c2.data();
        // a chunk of 32 cut-face lines costs about CUTP_C_FLINE point chunks
        const double fl = fl0[i] >= 0 ? CUTP_C_FLINE * ((fln[i] + 31) / 32) : 0.0;
        const int nf = fl0[i] >= 0 ? 0 : e.nf;
        // per cell: a fixed part, the axes with structured (GP / full-face SIPG) faces, the
        // cut faces' traces
        const uint32_t st = (e.smask & 0x3fu) | ((e.smask >> 8) & 0x3fu);
        const int sax = ((st & 3u) != 0) + ((st & 12u) != 0) + ((st & 48u) != 0);
        const double cell = CUTP_C_CELL + CUTP_C_SAX * sax + CUTP_C_TRACE * __builtin_popcount(e.fmask);
        if (isline[i]) return CUTP_C_LINE * ((e.nv / N + 31) / 32) + (double)((e.ns + nf + 31) / 32) + fl + cell;
        return (double)((e.nv + e.ns + nf + 31) / 32) + fl + cell;
      };
      for (int64_t i = 0; i < n; ++i) idx[i] = o + i;
      std::stable_sort(idx.begin(), idx.end(), [&](int64_t a, int64_t b) { return cost(c2[a]) > cost(c2[b]); });
      std::vector<std::vector<int64_t>> lists(W);
      std::priority_queue<std::pair<double, int>, std::vector<std::pair<double, int>>, std::greater<>> heap;
      for (int w = 0; w < W; ++w) heap.push({0.0, w});
      for (int64_t i : idx) {
        auto top = heap.top();
        heap.pop();
        lists[top.second].push_back(i);
        heap.push({top.first + cost(c2[i]), top.second});
      }
      int64_t pos = o;
      for (int w = 0; w < W; ++w) {
        ws.push_back((int)(pos - o));
        ks.push_back((int)chunk.size());
        for (int64_t i : lists[w]) {
          const CDesc2 &e = c2[i];
          c2o[pos++] = e;
          // the chunks of this cell (a chunk never mixes a cut-face point with another kind:
          // one code path per chunk, which pays at n = 4 where registers are tight)
          int nv = (hd->mask & CUTFEM_TERM_CELL) ? e.nv : 0;
          int ns = (hd->mask & CUTFEM_TERM_NITSCHE) ? e.ns : 0;
          const bool fon = (hd->mask & CUTFEM_TERM_SIPG) != 0;
          const size_t k0 = chunk.size();
          // volume points in lines: chunks of <= 32 lines (sign bit, axis << 24), then the
          // cell's other points as below with no volume points left
          const int lax = (N >= 3 && nv > 0) ? vol_line_axis(pb->vol_pts + 4 * e.vb, nv, N) : -1;
          int nlc = 0;  // line chunks of the cell (packed into nchunk's high half)
          if (lax >= 0) {
            const int nl = nv / N;
            // the interface points ride on the lines when they all sit on distinct lines
            // (needs both the cell and the Nitsche term: a record carries both)
            const bool son = ns > 0 && nv > 0 &&
                             !srf_on_lines(pb->vol_pts + 4 * e.vb, nv, pb->srf_pts + 7 * e.sb, ns, N, lax).empty();
            for (int l0 = 0; l0 < nl; l0 += 32) {
              CChunk r;
              r.vo = (int32_t)(e.vb + (int64_t)l0 * N);
              r.so = (int32_t)e.sb;
              r.fo = (int32_t)e.fb;
              r.cnt = (int32_t)(0x80000000u | (son ? 1u << 29 : 0u) | ((uint32_t)lax << 24) |
                                (uint32_t)std::min(32, nl - l0));
              chunk.push_back(r);
              ++nlc;
            }
            nv = 0;
            if (son) ns = 0;
          }
          // cut-face lines of every face in chunks of <= 32 (bit 30, first record in vo)
          int nfc = 0;
          const bool fdone = fon && fl0[i] >= 0;
          if (fdone) {
            for (int l0 = 0; l0 < fln[i]; l0 += 32) {
              CChunk r;
              r.vo = (int32_t)(fl0[i] + l0);
              r.so = (int32_t)e.sb;
              r.fo = (int32_t)e.fb;
              r.cnt = (int32_t)((1u << 30) | (uint32_t)std::min(32, fln[i] - l0));
              chunk.push_back(r);
              ++nfc;
            }
          }
          // [volume | interface] points in chunks of 32, then the cut-face points (one
          // stream over every face axis: runtime-axis update)
          for (int q0 = 0; q0 < nv + ns; q0 += 32) {
            const int cv = std::max(0, std::min(32, nv - q0));
            const int qs = std::max(0, q0 - nv), cs = std::max(0, std::min(32 - cv, ns - qs));
            CChunk r;
            r.vo = (int32_t)(e.vb + q0);
            r.so = (int32_t)(e.sb + qs);
            r.fo = (int32_t)e.fb;
            r.cnt = cv | (cs << 8);
            chunk.push_back(r);
          }
          if (fon && !fdone) {  // every face axis in one stream (runtime-axis update)
            for (int q0 = 0; q0 < e.nf; q0 += 32) {
              CChunk r;
              r.vo = (int32_t)e.vb;
              r.so = (int32_t)e.sb;
              r.fo = (int32_t)(e.fb + q0);
              r.cnt = std::min(32, e.nf - q0) << 16;
              chunk.push_back(r);
            }
          }
          if (chunk.size() - k0 > 0xffff || nlc > 0xff || nfc > 0xff)
            return fail(CUTFEM_EUNSUPPORTED, "k_cutp: too many point chunks in a cell");
          c2o[pos - 1].nchunk =
              (int32_t)((uint32_t)(chunk.size() - k0) | ((uint32_t)nlc << 16) | ((uint32_t)nfc << 24));
        }
      }
      ws.push_back((int)(pos - o));
      ks.push_back((int)chunk.size());
    }
    // pack every warp's chunks, in consumption order, into a contiguous stream
    // (16-byte chunk header {cnt} + volume rows [xi,eta,zeta,W] + interface rows
    // [xi,eta,zeta,nx,ny,nz,W,0] + cut-face rows [xi,eta,zeta,W]) and cut it into
    // packets of <= CUTP_PK bytes, one bulk copy each
    std::vector<double> strm;
    std::vector<CPacket> pk;
    std::map<int64_t, size_t> cell_of_vb;  // first volume point -> cut cell (line chunks)
    for (size_t i = 0; i < c2.size(); ++i)
      if (c2[i].nv > 0) cell_of_vb[c2[i].vb] = i;
    std::vector<int> ps;
    ps.reserve(ks.size());
    for (size_t w = 0; w + 1 < ks.size(); ++w) {
      ps.push_back((int)pk.size());
      if (ks[w + 1] < ks[w]) continue;  // part boundary entry (no chunks)
      CPacket cur = {(int64_t)strm.size() * 8, 0, 0};
      for (int k = ks[w]; k < ks[w + 1]; ++k) {
        const CChunk &r = chunk[k];
        const bool line = r.cnt < 0, lsrf = line && ((r.cnt >> 29) & 1);
        const bool fline = !line && ((r.cnt >> 30) & 1);
        const int cv = r.cnt & 0xff, cs = (line || fline) ? 0 : (r.cnt >> 8) & 0xff,
                  cf = (line || fline) ? 0 : (r.cnt >> 16) & 0xff;
        const int bytes = line    ? 16 + (16 + 16 * N + (lsrf ? 48 : 0)) * cv
                          : fline ? 16 + (16 + 16 * N) * cv
                                  : 16 + 32 * cv + 64 * cs + 32 * cf;
        if (cur.nch > 0 && cur.bytes + bytes > CutPCfg<N>::PK) {
          pk.push_back(cur);
          cur = {(int64_t)strm.size() * 8, 0, 0};
        }
        double hdr[2] = {0.0, 0.0};
        std::memcpy(hdr, &r.cnt, sizeof(int32_t));
        strm.insert(strm.end(), hdr, hdr + 2);
        if (fline) {
          strm.insert(strm.end(), flrec.begin() + (2 + 2 * N) * (size_t)r.vo,
                      flrec.begin() + (2 + 2 * N) * ((size_t)r.vo + cv));
          cur.bytes += bytes;
          ++cur.nch;
          continue;
        }
        if (line) {
          // per line: the two base coordinates (ascending axes), then (coordinate, W) per point
          const int ax = (r.cnt >> 24) & 3, b1 = ax == 0 ? 1 : 0, b2 = ax == 2 ? 1 : 2;
          // the cell's lines and (lsrf) which interface point sits on each
          std::vector<int> on;  // interface point per line of this chunk, -1 none
          if (lsrf) {
            // the cut cell of this chunk: its first line chunk starts at the cell's vb
            auto it = cell_of_vb.upper_bound(r.vo);
            --it;
            const CDesc2 &e = c2[it->second];
            const std::vector<int> li = srf_on_lines(pb->vol_pts + 4 * e.vb, e.nv, pb->srf_pts + 7 * e.sb, e.ns, N, ax);
            const int l0 = (int)((r.vo - e.vb) / N);
            on.assign(cv, -1);
            for (size_t q = 0; q < li.size(); ++q)
              if (li[q] >= l0 && li[q] < l0 + cv) on[li[q] - l0] = (int)(e.sb + (int64_t)q);
          }
          for (int l = 0; l < cv; ++l) {
            const double *x = pb->vol_pts + 4 * ((size_t)r.vo + (size_t)l * N);
            strm.push_back(x[b1]);
            strm.push_back(x[b2]);
            for (int t = 0; t < N; ++t) {
              strm.push_back(x[4 * t + ax]);
              strm.push_back(x[4 * t + 3]);
            }
            if (lsrf) {
              double rs6[6] = {0, 0, 0, 0, 0, 0};
              if (on[l] >= 0) {
                const double *y = pb->srf_pts + 7 * (size_t)on[l];  // xi eta zeta nx ny nz W
                rs6[0] = y[ax];
                rs6[1] = y[6];
                rs6[2] = y[3 + ax];
                rs6[3] = y[3 + b1];
                rs6[4] = y[3 + b2];
              }
              strm.insert(strm.end(), rs6, rs6 + 6);
            }
          }
          cur.bytes += bytes;
          ++cur.nch;
          continue;
        }
        strm.insert(strm.end(), pb->vol_pts + 4 * (size_t)r.vo, pb->vol_pts + 4 * ((size_t)r.vo + cv));
        for (int q = 0; q < cs; ++q) {
          const double *x = pb->srf_pts + 7 * ((size_t)r.so + q);
          strm.insert(strm.end(), x, x + 7);
          strm.push_back(0.0);
        }
        strm.insert(strm.end(), fac.begin() + 4 * (size_t)r.fo, fac.begin() + 4 * ((size_t)r.fo + cf));
        cur.bytes += bytes;
        ++cur.nch;
      }
      if (cur.nch > 0) pk.push_back(cur);
    }
    ps.push_back((int)pk.size());
    hd->w_off[0] = hd->w_off[1];
    hd->grid_cutp[0] = -1;  // part 0 launches parts 1 and 2 (see launch_tiles)
    if ((rc = upload(hd, &hd->d_cdesc2, c2o.data(), c2o.size()))) return rc;
    if ((rc = upload(hd, &hd->d_fac, fac.data(), fac.size()))) return rc;
    if ((rc = upload(hd, &hd->d_wstart, ws.data(), ws.size()))) return rc;
    if ((rc = upload(hd, &hd->d_kstart, ps.data(), ps.size()))) return rc;
    if ((rc = upload(hd, &hd->d_chunks, pk.data(), pk.size()))) return rc;
    if ((rc = upload(hd, &hd->d_stream, reinterpret_cast<const char *>(strm.data()), strm.size() * 8))) return rc;
    {
      int64_t mx = (int64_t)fac.size() / 4;
      for (const CDesc2 &e : c2) mx = std::max(mx, std::max(e.vb + e.nv, e.sb + e.ns));
      if (mx > INT32_MAX) return fail(CUTFEM_EUNSUPPORTED, "k_cutp point offsets need int32");
    }
  }
  hd->ttab.resize(sizeof(TileTab<N>));
  build_tiletab<N>(pb->h, pb->sipg_gamma, pb->gp_gamma, pb->gp_kind, pb->tau_v, hd->mask,
                   *reinterpret_cast<TileTab<N> *>(hd->ttab.data()));
  if constexpr (N == 4) {
    using C2 = Tile2Cfg<N>;
    CU(cudaFuncSetAttribute(k_tile2<N, 0>, cudaFuncAttributeMaxDynamicSharedMemorySize, C2::SMEM));
    CU(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&hd->occ_tile[0], k_tile2<N, 0>, C2::THREADS, C2::SMEM));
    using CU4 = UncwCfg<N, UNCW4_TC>;
    CU(cudaFuncSetAttribute(k_uncw<N, UNCW4_TC>, cudaFuncAttributeMaxDynamicSharedMemorySize, CU4::SMEM));
    CU(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&hd->occ_tile[1], k_uncw<N, UNCW4_TC>, CU4::THREADS, CU4::SMEM));
  }
  for (int k = 0; k < 3; ++k) hd->occ_tile[k] = std::max(1, hd->occ_tile[k]);
  return 0;
}

// N = 5..9: uncut cells through k_uncw (every structured term, GP included); cut
// cells stay on k_cut.
template <int N>
int setup_uncw(cutfem_handle *hd, const cutfem_problem *pb, const std::vector<UDesc> &ud) {
  using C = TileCfg<N>;
  std::vector<TCell> part[2];
  for (int pt = 1; pt <= 2; ++pt)
    for (int k = 0; k < 2; ++k)
      for (int64_t i = hd->r_off[pt][k]; i < hd->r_off[pt][k] + hd->r_cnt[pt][k]; ++i) {
        const UDesc &d = ud[i];
        TCell c;
        c.blk = d.blk;
        uint32_t nbm = 0;
        for (int f = 0; f < 6; ++f) {
          c.nb[f] = d.nb[f];
          if (d.nb[f] >= 0) nbm |= 1u << f;
        }
        c.gp = d.flags & nbm & 0x3fu;
        c.sipg = nbm;
        c.vol = true;
        part[pt - 1].push_back(c);
      }
  const int64_t rs = (int64_t)sizeof(TileRec<C::SMAX>);
  std::vector<char> b0, b1;
  build_tiles<TileCfg<N>>(part[0], pb, b0);
  build_tiles<TileCfg<N>>(part[1], pb, b1);
  hd->t_off[0][0] = hd->t_off[0][1] = 0;
  hd->t_cnt[0][1] = (int64_t)b0.size() / rs;
  hd->t_off[0][2] = hd->t_cnt[0][1];
  hd->t_cnt[0][2] = (int64_t)b1.size() / rs;
  hd->t_cnt[0][0] = hd->t_cnt[0][1] + hd->t_cnt[0][2];
  b0.insert(b0.end(), b1.begin(), b1.end());
  int rc = upload(hd, reinterpret_cast<char **>(&hd->d_tiles), b0.data(), b0.size());
  if (rc) return rc;
  hd->ttab.resize(sizeof(TileTab<N>));
  build_tiletab<N>(pb->h, pb->sipg_gamma, pb->gp_gamma, pb->gp_kind, pb->tau_v, hd->mask,
                   *reinterpret_cast<TileTab<N> *>(hd->ttab.data()));
  CU(cudaFuncSetAttribute(k_uncw<N>, cudaFuncAttributeMaxDynamicSharedMemorySize, UncwCfg<N>::SMEM));
  CU(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&hd->occ_tile[0], k_uncw<N>, UncwCfg<N>::THREADS,
                                                   UncwCfg<N>::SMEM));
  hd->occ_tile[0] = std::max(1, hd->occ_tile[0]);
  return 0;
}

int dispatch_tiles(cutfem_handle *hd, const cutfem_problem *pb, const std::vector<UDesc> &ud,
                   const std::vector<CDesc> &cd) {
  switch (hd->n) {
    case 2: return setup_tiles<2>(hd, pb, ud, cd);
    case 3: return setup_tiles<3>(hd, pb, ud, cd);
    case 4: return setup_tiles<4>(hd, pb, ud, cd);
    case 5: return setup_uncw<5>(hd, pb, ud);
    case 6: return setup_uncw<6>(hd, pb, ud);
    // n = 5..9: k_uncw (pipelined tiles; odd n by 8-byte cp.async: C3 p=6 structured
    // 323 -> 139 us, p=8 376 -> 195 us against round 1's warp-per-line k_uncut)
    case 7: return setup_uncw<7>(hd, pb, ud);
    case 8: return setup_uncw<8>(hd, pb, ud);
    case 9: return setup_uncw<9>(hd, pb, ud);
  }
  return 0;
}

// Launch on `st`; pdl: with the programmatic-serialization attribute (the kernel may
// start once every CTA of the previous kernel in the stream has begun; see pdl_trigger).
template <typename... KArgs, typename... Args>
int launch_k(void (*kern)(KArgs...), unsigned grid, unsigned block, size_t smem, cudaStream_t st, bool pdl,
             Args... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(block);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = pdl ? at : nullptr;
  cfg.numAttrs = pdl ? 1 : 0;
  CU(cudaLaunchKernelEx(&cfg, kern, static_cast<KArgs>(args)...));
  return 0;
}

// N <= 4, one stream: k_cutp (cut cells, every term, v = ...; normal launch), then
// the uncut cells -- k_cell (n <= 3), or k_tile2 (cells without ghost-penalty faces,
// volume + SIPG) and k_uncw<4> (the cells next to cut cells, every term) -- each
// v = ... on disjoint blocks, launched as programmatic dependents (kernels.cuh
// pdl_trigger): they start only once all of k_cutp's CTAs have begun (k_cutp, the long
// pole, holds its SM slots first; two free-running streams let the uncut kernels take
// the SMs first in some applies: the r1 slow steps) and fill the slots its warps free.
template <int N>
int launch_tiles(cutfem_handle *hd, const double *u, double *v, cudaStream_t st, int which, int part) {
  constexpr int NT = (N <= 4 ? N : 4);
  const int64_t nc = (which & 2) ? hd->r_cnt[part][2] : 0;
  const int64_t n0 = (which & 1) ? hd->t_cnt[0][part] : 0;
  const int64_t n1 = (which & 1) ? hd->t_cnt[1][part] : 0;
  const int64_t ncell = (which & 1) ? hd->r_cnt[part][0] + hd->r_cnt[part][1] : 0;
  bool pdl = false;  // the first kernel of the apply is a normal launch
  int rc;
  if constexpr (NT <= CUTFEM_CUT1_MAXN) {
    if (nc > 0) {
      constexpr int TPC = NT == 2 ? CUT1_TPC2 : CUT1_TPC3;
      if ((rc = launch_k(k_cut1<NT, TPC>, (unsigned)((nc * TPC + 127) / 128), 128, 0, st, pdl, u, v,
                         hd->d_cdesc + hd->r_off[part][2], (int)nc, hd->d_vol, hd->d_srf, hd->d_sfp, hd->d_sfptr,
                         hd->kp, *reinterpret_cast<const TileTab<NT> *>(hd->ttab.data()))))
        return rc;
      pdl = true;
    }
  } else if (nc > 0) {
    using CP = CutPCfg<NT>;
    // part 0 = the interior list then the slab-boundary list (each with its own warp schedule)
    for (int pt = 1; pt <= 2; ++pt) {
      if (part != 0 && part != pt) continue;
      if (hd->grid_cutp[pt] <= 0) continue;
      if ((rc = launch_k(k_cutp<NT>, (unsigned)hd->grid_cutp[pt], 32 * CP::WARPS, CP::SMEM, st, pdl, u, v,
                         hd->d_cdesc2 + hd->r_off[pt][2], hd->d_chunks, hd->d_stream, hd->d_wstart + hd->w_off[pt],
                         hd->d_kstart + hd->w_off[pt], hd->kp, *reinterpret_cast<const TileTab<NT> *>(hd->ttab.data()))))
        return rc;
      pdl = true;
    }
  }
  const TileTab<NT> &tt = *reinterpret_cast<const TileTab<NT> *>(hd->ttab.data());
  const char *tb = reinterpret_cast<const char *>(hd->d_tiles);  // byte offsets per set
  if constexpr (NT <= 3) {
    // p = 1, 2: one thread per uncut cell (plain cells, then the cells next to cut cells)
    const int64_t np = hd->r_cnt[part][0], ng = hd->r_cnt[part][1];
    if (ncell > 0 && (rc = launch_k(k_cell<NT>, (unsigned)(((np + ng) * CELL_TPC + 127) / 128), 128, 0, st, pdl, u, v,
                                    hd->d_udesc + hd->r_off[part][0], (int)np, hd->d_udesc + hd->r_off[part][1],
                                    (int)ng, tt, hd->kp.mask)))
      return rc;
  } else {
    if (n0 > 0) {  // cells without ghost-penalty faces: volume + SIPG
      const unsigned grid = (unsigned)std::min<int64_t>(n0, (int64_t)hd->occ_tile[0] * hd->sm_count);
      const auto *t0 = reinterpret_cast<const TileRec<Tile2Cfg<NT>::SMAX> *>(tb + hd->t_off[0][part]);
      if ((rc = launch_k(k_tile2<NT, 0>, grid, Tile2Cfg<NT>::THREADS, Tile2Cfg<NT>::SMEM, st, pdl, u, v, t0, (int)n0,
                         tt, hd->kp.mask)))
        return rc;
      pdl = true;
    }
    if (n1 > 0) {  // cells next to cut cells: volume + SIPG + ghost penalty
      const unsigned grid = (unsigned)std::min<int64_t>(n1, (int64_t)hd->occ_tile[1] * hd->sm_count);
      const auto *t1 = reinterpret_cast<const TileRec<TileCfgX<NT, UNCW4_TC>::SMAX> *>(tb + hd->t_off[1][part]);
      if ((rc = launch_k(k_uncw<NT, UNCW4_TC>, grid, UncwCfg<NT, UNCW4_TC>::THREADS, UncwCfg<NT, UNCW4_TC>::SMEM, st,
                         pdl, u, v, t1, (int)n1, tt, hd->kp.mask)))
        return rc;
    }
  }
  return 0;
}

// which: bit0 structured (uncut) kernels, bit1 unstructured (cut) kernel; part:
// 0 all owned cells, 1 slab-interior cells, 2 slab-boundary cells.  With both
// kinds, the cut kernel runs on the forked side stream, concurrently.
template <int N>
int launch(cutfem_handle *hd, const double *u, double *v, cudaStream_t st, int which = 3, int part = 0) {
  if constexpr (N <= 4) return launch_tiles<N>(hd, u, v, st, which, part);
  else {
  const int64_t np = (which & 1) ? hd->r_cnt[part][0] : 0, ng = (which & 1) ? hd->r_cnt[part][1] : 0;
  const int64_t nc = (which & 2) ? hd->r_cnt[part][2] : 0;
  const CDesc *dc = hd->d_cdesc + hd->r_off[part][2];
  const int64_t nu = np + ng;
  const bool fork = nc > 0 && nu > 0;
  cudaStream_t cs = fork ? hd->side : st;
  // n = 5, 6, 8: the persistent uncut kernel (k_uncw), after the cut-cell kernel
  auto launch_uncw = [&]() -> int {
    if (!(nu > 0 && N >= 5 && hd->d_tiles)) return 0;
    constexpr int NU = N >= 5 ? N : 5;
    const int64_t nt = hd->t_cnt[0][part];
    if (nt > 0) {
      const int occ = hd->occ_tile[0];
      const unsigned grid = (unsigned)std::min<int64_t>(nt, (int64_t)occ * hd->sm_count);
      k_uncw<NU><<<grid, UncwCfg<NU>::THREADS, UncwCfg<NU>::SMEM, st>>>(
          u, v, reinterpret_cast<const TileRec<TileCfg<NU>::SMAX> *>(hd->d_tiles) + hd->t_off[0][part], (int)nt,
          *reinterpret_cast<const TileTab<NU> *>(hd->ttab.data()), hd->kp.mask);
      CU(cudaGetLastError());
    }
    return 0;
  };
  if (fork) {
    CU(cudaEventRecord(hd->ev_fork, st));
    CU(cudaStreamWaitEvent(hd->side, hd->ev_fork, 0));
  }
  if (nc > 0) {
    {
      k_cut<N><<<(unsigned)nc, CutCfg<N>::THREADS, CutCfg<N>::SMEM, cs>>>(
          u, v, dc, (int)nc, hd->d_vol, hd->d_volptr, hd->d_srf, hd->d_srfptr, hd->d_sfp, hd->d_sfptr, hd->kp,
          hd->ft, *reinterpret_cast<const TileTab<N> *>(hd->ttab.data()), hd->d_line_srf);
    }
    CU(cudaGetLastError());
  }
  if (nu > 0) {
    if (!hd->d_tiles) return fail(CUTFEM_ECUDA, "uncut-cell tiles missing");
    launch_uncw();  // n = 5..9
  }
  if (fork) {
    CU(cudaEventRecord(hd->ev_join, hd->side));
    CU(cudaStreamWaitEvent(st, hd->ev_join, 0));
  }
  return 0;
  }
}

template <int N>
int set_attrs() {
  if constexpr (N >= 5) {
    CU(cudaFuncSetAttribute(k_cut<N>, cudaFuncAttributeMaxDynamicSharedMemorySize, CutCfg<N>::SMEM));
  }
  return 0;
}

int dispatch_part(cutfem_handle *hd, const double *u, double *v, cudaStream_t st, int which, int part) {
  switch (hd->n) {
    case 2: return launch<2>(hd, u, v, st, which, part);
    case 3: return launch<3>(hd, u, v, st, which, part);
    case 4: return launch<4>(hd, u, v, st, which, part);
    case 5: return launch<5>(hd, u, v, st, which, part);
    case 6: return launch<6>(hd, u, v, st, which, part);
    case 7: return launch<7>(hd, u, v, st, which, part);
    case 8: return launch<8>(hd, u, v, st, which, part);
    case 9: return launch<9>(hd, u, v, st, which, part);
  }
  return fail(CUTFEM_EUNSUPPORTED, "degree");
}

int halo_exchange(cutfem_handle *hd, const double *u_ext, cudaStream_t st);  // dist.inl

int dispatch_apply(cutfem_handle *hd, const double *u, double *v, cudaStream_t st, int which = 3) {
  if (!hd->dist) return dispatch_part(hd, u, v, st, which, 0);
  // x-slab: the halo exchange runs on the comm stream while the slab-interior
  // cells compute; the boundary cells follow once the ghost blocks have landed
  int rc = halo_exchange(hd, u, st);
  if (rc) return rc;
  if ((rc = dispatch_part(hd, u, v, st, which, 1))) return rc;
  if (hd->ev_comm) CU(cudaStreamWaitEvent(st, hd->ev_comm, 0));
  return dispatch_part(hd, u, v, st, which, 2);
}

int dispatch_attrs(int n) {
  switch (n) {
    case 2: return set_attrs<2>();
    case 3: return set_attrs<3>();
    case 4: return set_attrs<4>();
    case 5: return set_attrs<5>();
    case 6: return set_attrs<6>();
    case 7: return set_attrs<7>();
    case 8: return set_attrs<8>();
    case 9: return set_attrs<9>();
  }
  return fail(CUTFEM_EUNSUPPORTED, "degree");
}

void free_handle(cutfem_handle *hd) {
  if (!hd) return;
  cudaFree(hd->d_udesc);
  cudaFree(hd->d_tiles);
  cg_free(hd->cg);
  cudaFree(hd->d_cdesc2);
  cudaFree(hd->d_wstart);
  cudaFree(hd->d_kstart);
  cudaFree(hd->d_chunks);
  cudaFree(hd->d_stream);
  cudaFree(hd->d_fac);
  cudaFree(hd->d_cdesc);
  cudaFree(hd->d_vol);
  cudaFree(hd->d_srf);
  cudaFree(hd->d_sfp);
  cudaFree(hd->d_volptr);
  cudaFree(hd->d_line_srf);
  cudaFree(hd->d_srfptr);
  cudaFree(hd->d_sfptr);
  cudaFree(hd->d_u);
  cudaFree(hd->d_v);
  for (int b = 0; b < 2; ++b) {
    cudaFree(hd->d_ub[b]);
    cudaFree(hd->d_vb[b]);
    if (hd->ev_in[b]) cudaEventDestroy(hd->ev_in[b]);
    if (hd->ev_done[b]) cudaEventDestroy(hd->ev_done[b]);
    if (hd->ev_out[b]) cudaEventDestroy(hd->ev_out[b]);
  }
  if (hd->s_h2d) cudaStreamDestroy(hd->s_h2d);
  if (hd->s_d2h) cudaStreamDestroy(hd->s_d2h);
  cudaFree(hd->d_rowptr);
  cudaFree(hd->d_col);
  cudaFree(hd->d_val);
  cudaFree(hd->d_spbuf);
  if (hd->spA) cusparseDestroySpMat(hd->spA);
  if (hd->sp) cusparseDestroy(hd->sp);
  if (hd->side) cudaStreamDestroy(hd->side);
  if (hd->comm) ncclCommDestroy((ncclComm_t)hd->comm);
  if (hd->comm_stream) cudaStreamDestroy(hd->comm_stream);
  if (hd->ev_comm) cudaEventDestroy(hd->ev_comm);
  if (hd->ev_comm_fork) cudaEventDestroy(hd->ev_comm_fork);
  if (hd->ev_fork) cudaEventDestroy(hd->ev_fork);
  if (hd->ev_join) cudaEventDestroy(hd->ev_join);
  if (hd->ev_started) cudaEventDestroy(hd->ev_started);
  delete hd;
}

int setup_impl(const cutfem_problem *pb, int device, cutfem_handle *hd, int64_t n_compute = -1) {
  if (!pb) return fail(CUTFEM_EINVAL, "null problem");
  const int p = pb->degree;
  if (p < 1 || p > 8) return fail(CUTFEM_EINVAL, "degree must be in 1..8");
  if (!(pb->h > 0)) return fail(CUTFEM_EINVAL, "h must be > 0");
  for (int i = 0; i < 3; ++i)
    if (pb->n_cells[i] < 1) return fail(CUTFEM_EINVAL, "n_cells must be >= 1");
  if (pb->n_active < 0 || (pb->n_active > 0 && (!pb->active_ijk || !pb->is_cut)))
    return fail(CUTFEM_EINVAL, "active arrays");
  if (!pb->gp_gamma) return fail(CUTFEM_EINVAL, "gp_gamma is NULL");
  const int n = p + 1;
  const int64_t na = pb->n_active;
  const int64_t nx = pb->n_cells[0], ny = pb->n_cells[1], nz = pb->n_cells[2];
  if ((double)na * n * n * n > 9.0e18) return fail(CUTFEM_EINVAL, "too many DoFs");
  hd->device = device;
  hd->degree = p;
  hd->n = n;
  hd->h = pb->h;
  hd->n_active = na;
  hd->mask = pb->term_mask ? pb->term_mask : CUTFEM_TERM_ALL;
  if (na > 0) hd->blk_ijk.assign(pb->active_ijk, pb->active_ijk + 3 * na);
  if (na > 0) hd->blk_cut.assign(pb->is_cut, pb->is_cut + na);
  for (int i = 0; i < 3; ++i) {
    hd->n_cells[i] = pb->n_cells[i];
    hd->lower[i] = pb->lower[i];
  }
  CU(cudaSetDevice(device));
  // grid -> block map
  std::vector<int32_t> grid((size_t)(nx * ny * nz), -1);
  std::vector<int64_t> cut_ord(na, -1);
  int64_t nc = 0;
  for (int64_t b = 0; b < na; ++b) {
    const int32_t i = pb->active_ijk[3 * b], j = pb->active_ijk[3 * b + 1], k = pb->active_ijk[3 * b + 2];
    if (i < 0 || j < 0 || k < 0 || i >= nx || j >= ny || k >= nz)
      return fail(CUTFEM_EINVAL, "active_ijk out of range");
    int32_t &g = grid[(size_t)((i * ny + j) * nz + k)];
    if (g >= 0) return fail(CUTFEM_EINVAL, "duplicate active cell");
    g = (int32_t)b;
    if (pb->is_cut[b]) cut_ord[b] = nc++;
  }
  hd->color.resize(na);
  for (int64_t b = 0; b < na; ++b)
    hd->color[b] = (uint8_t)((pb->active_ijk[3 * b] + 2 * pb->active_ijk[3 * b + 1] + 3 * pb->active_ijk[3 * b + 2]) % 7);
  hd->n_cut = nc;
  hd->n_uncut = na - nc;
  if (nc > 0 && (!pb->vol_ptr || !pb->srf_ptr)) return fail(CUTFEM_EINVAL, "vol_ptr/srf_ptr NULL");
  const int64_t nvol = nc ? pb->vol_ptr[nc] : 0, nsrf = nc ? pb->srf_ptr[nc] : 0;
  if (nc && (pb->vol_ptr[0] != 0 || pb->srf_ptr[0] != 0)) return fail(CUTFEM_EINVAL, "ptr[0] != 0");
  for (int64_t c = 0; c < nc; ++c)
    if (pb->vol_ptr[c + 1] < pb->vol_ptr[c] || pb->srf_ptr[c + 1] < pb->srf_ptr[c])
      return fail(CUTFEM_EINVAL, "ptr not monotone");
  if ((nvol && !pb->vol_pts) || (nsrf && !pb->srf_pts)) return fail(CUTFEM_EINVAL, "points NULL");
  const double tol = 1e-12;
  for (int64_t q = 0; q < nvol; ++q) {
    const double *x = pb->vol_pts + 4 * q;
    for (int d = 0; d < 3; ++d)
      if (!(x[d] >= -tol && x[d] <= 1 + tol)) return fail(CUTFEM_EINVAL, "volume point outside [0,1]^3");
    if (!(x[3] >= 0)) return fail(CUTFEM_EINVAL, "negative volume weight");
  }
  for (int64_t q = 0; q < nsrf; ++q) {
    const double *x = pb->srf_pts + 7 * q;
    for (int d = 0; d < 3; ++d)
      if (!(x[d] >= -tol && x[d] <= 1 + tol)) return fail(CUTFEM_EINVAL, "surface point outside [0,1]^3");
    const double nn = std::sqrt(x[3] * x[3] + x[4] * x[4] + x[5] * x[5]);
    if (!(std::fabs(nn - 1) <= 1e-10)) return fail(CUTFEM_EINVAL, "surface normal not unit");
    if (!(x[6] >= 0)) return fail(CUTFEM_EINVAL, "negative surface weight");
  }
  // listed faces
  const int64_t nsf = pb->n_sfaces;
  if (nsf < 0 || (nsf > 0 && (!pb->sf_cells || !pb->sf_axis || !pb->sf_ptr)))
    return fail(CUTFEM_EINVAL, "sf arrays");
  const int64_t nfp = nsf ? pb->sf_ptr[nsf] : 0;
  if (nsf && pb->sf_ptr[0] != 0) return fail(CUTFEM_EINVAL, "sf_ptr[0] != 0");
  if (nfp && !pb->sf_pts) return fail(CUTFEM_EINVAL, "sf_pts NULL");
  for (int64_t q = 0; q < nfp; ++q) {
    const double *x = pb->sf_pts + 3 * q;
    if (!(x[0] >= -tol && x[0] <= 1 + tol && x[1] >= -tol && x[1] <= 1 + tol))
      return fail(CUTFEM_EINVAL, "face point outside [0,1]^2");
    if (!(x[2] >= 0)) return fail(CUTFEM_EINVAL, "negative face weight");
  }
  // sf index per (cell, face)
  std::vector<int32_t> sfid((size_t)na * 6, -1);
  int64_t n_fcut = 0, n_fempty = 0;
  for (int64_t f = 0; f < nsf; ++f) {
    const int32_t m = pb->sf_cells[2 * f], pl = pb->sf_cells[2 * f + 1];
    const int d = pb->sf_axis[f];
    if (d > 2 || m < 0 || pl < 0 || m >= na || pl >= na) return fail(CUTFEM_EINVAL, "bad listed face");
    if (pb->sf_ptr[f + 1] < pb->sf_ptr[f]) return fail(CUTFEM_EINVAL, "sf_ptr not monotone");
    for (int t = 0; t < 3; ++t) {
      const int32_t want = pb->active_ijk[3 * m + t] + (t == d ? 1 : 0);
      if (pb->active_ijk[3 * pl + t] != want) return fail(CUTFEM_EINVAL, "listed face cells not adjacent");
    }
    if (!pb->is_cut[m] || !pb->is_cut[pl])
      return fail(CUTFEM_EINVAL, "listed face touches an uncut cell (its faces are inside Ω)");
    if (sfid[m * 6 + 2 * d + 1] >= 0) return fail(CUTFEM_EINVAL, "duplicate listed face");
    sfid[m * 6 + 2 * d + 1] = (int32_t)f;
    sfid[pl * 6 + 2 * d] = (int32_t)f;
    if (pb->sf_ptr[f + 1] > pb->sf_ptr[f]) ++n_fcut; else ++n_fempty;
  }
  // ghost-penalty faces per (block, face): face GP on every face with a cut side;
  // volume GP on the stable-neighbour patches (include/cutfem.h CUTFEM_GP_VOLUME)
  if (pb->gp_kind != CUTFEM_GP_FACE && pb->gp_kind != CUTFEM_GP_VOLUME) return fail(CUTFEM_EINVAL, "gp_kind");
  if (pb->gp_kind == CUTFEM_GP_VOLUME && !(pb->tau_v >= 0)) return fail(CUTFEM_EINVAL, "tau_v < 0");
  if (pb->gp_kind == CUTFEM_GP_VOLUME && n_compute >= 0 && n_compute != na)
    return fail(CUTFEM_EUNSUPPORTED, "volume ghost penalty on a distributed handle");
  auto nb_of = [&](int64_t b, int f) -> int32_t {
    int32_t q[3] = {pb->active_ijk[3 * b], pb->active_ijk[3 * b + 1], pb->active_ijk[3 * b + 2]};
    const int d = f >> 1;
    q[d] += (f & 1) ? 1 : -1;
    if (q[d] < 0 || q[d] >= pb->n_cells[d]) return -1;
    return grid[(size_t)((q[0] * ny + q[1]) * nz + q[2])];
  };
  std::vector<uint8_t> gpf((size_t)na * 6, 0);
  if (pb->gp_kind == CUTFEM_GP_FACE) {
    for (int64_t b = 0; b < na; ++b)
      for (int f = 0; f < 6; ++f) {
        const int32_t q = nb_of(b, f);
        if (q >= 0 && (pb->is_cut[b] || pb->is_cut[q])) gpf[b * 6 + f] = 1;
      }
  } else {
    std::vector<double> frac(na, 1.0);  // |E cap Omega| / |E|: 1 for uncut cells
    const double h3 = pb->h * pb->h * pb->h;
    for (int64_t b = 0; b < na; ++b)
      if (pb->is_cut[b]) {
        const int64_t c = cut_ord[b];
        double s = 0;
        for (int64_t q = pb->vol_ptr[c]; q < pb->vol_ptr[c + 1]; ++q) s += pb->vol_pts[4 * q + 3];
        frac[b] = s / h3;
      }
    for (int64_t b = 0; b < na; ++b) {
      if (!pb->is_cut[b]) continue;
      int best = -1;
      for (int f = 0; f < 6; ++f) {
        const int32_t q = nb_of(b, f);
        if (q >= 0 && (best < 0 || frac[q] > frac[nb_of(b, best)])) best = f;
      }
      if (best < 0) continue;  // an isolated cut cell: nothing to stabilise against
      gpf[b * 6 + best] = 1;
      gpf[(size_t)nb_of(b, best) * 6 + (best ^ 1)] = 1;
    }
  }
  // descriptors
  std::vector<UDesc> ud;
  std::vector<CDesc> cd;
  std::vector<double> line_srf;  // k_cut: interface record per volume line of the line cells (6 doubles)
  std::vector<int64_t> ccost;
  if (n_compute < 0) n_compute = na;
  hd->n_own = n_compute;
  ud.reserve(na - nc);
  cd.reserve(nc);
  std::vector<uint8_t> ubnd, cbnd;  // slab-boundary flag (a neighbour is a ghost block)
  int64_t n_struct = 0, n_gp = 0;
  for (int64_t b = 0; b < n_compute; ++b) {
    const int32_t ijk[3] = {pb->active_ijk[3 * b], pb->active_ijk[3 * b + 1], pb->active_ijk[3 * b + 2]};
    int32_t nb[6];
    for (int f = 0; f < 6; ++f) {
      int32_t q[3] = {ijk[0], ijk[1], ijk[2]};
      const int d = f >> 1;
      q[d] += (f & 1) ? 1 : -1;
      const int64_t lim = pb->n_cells[d];
      nb[f] = (q[d] < 0 || q[d] >= lim) ? -1 : grid[(size_t)((q[0] * ny + q[1]) * nz + q[2])];
    }
    const bool cut = pb->is_cut[b] != 0;
    bool bnd = false;
    for (int f = 0; f < 6; ++f)
      if (nb[f] >= n_compute) bnd = true;
    if (!cut) {
      ubnd.push_back(bnd ? 1 : 0);
      UDesc u;
      std::memset(&u, 0, sizeof(u));
      u.blk = (int32_t)b;
      for (int f = 0; f < 6; ++f) {
        u.nb[f] = nb[f];
        if (nb[f] >= 0 && gpf[b * 6 + f]) u.flags |= 1u << f;  // ghost-penalty face
      }
      ud.push_back(u);
    } else {
      CDesc c;
      std::memset(&c, 0, sizeof(c));
      c.blk = (int32_t)b;
      c.cut = (int32_t)cut_ord[b];
      c.vb = pb->vol_ptr[c.cut];
      c.sb = pb->srf_ptr[c.cut];
      c.nv = (int32_t)(pb->vol_ptr[c.cut + 1] - pb->vol_ptr[c.cut]);
      c.ns = (int32_t)(pb->srf_ptr[c.cut + 1] - pb->srf_ptr[c.cut]);
      int64_t cost = (pb->vol_ptr[c.cut + 1] - pb->vol_ptr[c.cut]) + (pb->srf_ptr[c.cut + 1] - pb->srf_ptr[c.cut]);
      for (int f = 0; f < 6; ++f) {
        c.nb[f] = nb[f];
        c.sf[f] = -1;
        if (nb[f] < 0) continue;
        if (gpf[b * 6 + f]) c.flags |= 1u << f;  // ghost-penalty face
        const int32_t s = sfid[b * 6 + f];
        if (s < 0) {
          c.flags |= 1u << (6 + f);
        } else if (pb->sf_ptr[s + 1] > pb->sf_ptr[s]) {
          c.flags |= 1u << (12 + f);
          c.sf[f] = s;
          cost += (pb->sf_ptr[s + 1] - pb->sf_ptr[s]) / 2;
        }
      }
      // k_cut (n >= 5): volume points in lines -> flag bit 26, axis in bits 24-25; the
      // interface points on the lines -> bit 27, per-line index list from c.pad
      if (n >= 5) {
        const int lax = vol_line_axis(pb->vol_pts + 4 * c.vb, c.nv, n);
        if (lax >= 0) {
          c.flags |= (1u << 26) | ((uint32_t)lax << 24);
          const std::vector<int> li = srf_on_lines(pb->vol_pts + 4 * c.vb, c.nv, pb->srf_pts + 7 * c.sb, c.ns, n, lax);
          if (!li.empty()) {
            c.flags |= 1u << 27;
            c.pad = (int32_t)(line_srf.size() / 6);
            const size_t l0 = line_srf.size() / 6;
            line_srf.resize(6 * (l0 + c.nv / n), 0.0);
            const int b1 = lax == 0 ? 1 : 0, b2 = lax == 2 ? 1 : 2;
            for (size_t q = 0; q < li.size(); ++q) {
              const double *y = pb->srf_pts + 7 * (c.sb + (int64_t)q);  // xi eta zeta nx ny nz W
              double *r = &line_srf[6 * (l0 + li[q])];
              r[0] = y[lax];
              r[1] = y[6];
              r[2] = y[3 + lax];
              r[3] = y[3 + b1];
              r[4] = y[3 + b2];
            }
          }
        }
      }
      cd.push_back(c);
      ccost.push_back(cost + (bnd ? (int64_t)1 << 40 : 0));  // boundary cells sort last (key), heavy first
      cbnd.push_back(bnd ? 1 : 0);
    }
    // count every interior face once, from its minus side (hi face f = 2d+1)
    for (int d = 0; d < 3; ++d) {
      const int32_t q = nb[2 * d + 1];
      if (q < 0) continue;
      if (gpf[b * 6 + 2 * d + 1]) ++n_gp;
      if (sfid[b * 6 + 2 * d + 1] < 0) ++n_struct;
    }
  }
  // uncut order: [plain interior | plain boundary | general interior | general boundary];
  // plain = six active uncut neighbours
  {
    std::vector<UDesc> cls[2][2];
    for (size_t i = 0; i < ud.size(); ++i) {
      const UDesc &x = ud[i];
      bool pl = true;
      for (int f = 0; f < 6; ++f)
        if (x.nb[f] < 0 || pb->is_cut[x.nb[f]]) pl = false;
      cls[pl ? 0 : 1][ubnd[i]].push_back(x);
    }
    ud.clear();
    int64_t off = 0;
    for (int k = 0; k < 2; ++k) {
      hd->r_off[1][k] = off;
      hd->r_cnt[1][k] = (int64_t)cls[k][0].size();
      hd->r_off[2][k] = off + (int64_t)cls[k][0].size();
      hd->r_cnt[2][k] = (int64_t)cls[k][1].size();
      hd->r_off[0][k] = off;
      hd->r_cnt[0][k] = (int64_t)(cls[k][0].size() + cls[k][1].size());
      for (int bd = 0; bd < 2; ++bd) ud.insert(ud.end(), cls[k][bd].begin(), cls[k][bd].end());
      off += hd->r_cnt[0][k];
    }
    hd->n_plain = hd->r_cnt[0][0];
  }
  // cut order: [interior | boundary], each heaviest first (LPT order for the block scheduler)
  {
    std::vector<int64_t> order(cd.size());
    for (size_t i = 0; i < order.size(); ++i) order[i] = (int64_t)i;
    // n >= 5 (k_cut: one CTA per cut cell, in this order): CUT_ORDER 0 heaviest first;
    // 1 spatial (block order: neighbour blocks shared by consecutive CTAs stay in L2);
    // 2 the heaviest CUT_HEAVY_PCT % first, the rest spatial
    const int corder = n >= 5 ? CUT_ORDER : 0;
    std::vector<uint8_t> heavy(cd.size(), 0);
    if (corder == 2 && !cd.empty()) {
      std::vector<int64_t> cs(ccost.begin(), ccost.end());
      const size_t k = std::min(cs.size() - 1, (size_t)(cs.size() * (100 - CUT_HEAVY_PCT) / 100));
      std::nth_element(cs.begin(), cs.begin() + k, cs.end());
      for (size_t i = 0; i < cd.size(); ++i) heavy[i] = ccost[i] > cs[k];
    }
    std::stable_sort(order.begin(), order.end(), [&](int64_t a, int64_t b) {
      if (cbnd[a] != cbnd[b]) return cbnd[a] < cbnd[b];
      if (corder == 1) return cd[a].blk < cd[b].blk;
      if (corder == 2) {
        if (heavy[a] != heavy[b]) return heavy[a] > heavy[b];
        if (heavy[a]) return ccost[a] > ccost[b];
        return cd[a].blk < cd[b].blk;
      }
      return ccost[a] > ccost[b];
    });
    std::vector<CDesc> s(cd.size());
    int64_t nci = 0;
    for (size_t i = 0; i < order.size(); ++i) {
      s[i] = cd[order[i]];
      if (!cbnd[order[i]]) ++nci;
    }
    cd.swap(s);
    hd->r_off[0][2] = 0;
    hd->r_cnt[0][2] = (int64_t)cd.size();
    hd->r_off[1][2] = 0;
    hd->r_cnt[1][2] = nci;
    hd->r_off[2][2] = nci;
    hd->r_cnt[2][2] = (int64_t)cd.size() - nci;
  }
  hd->n_uncut = (int64_t)ud.size();
  hd->n_cut = (int64_t)cd.size();
  int rc;
  if ((rc = upload(hd, &hd->d_udesc, ud.data(), ud.size()))) return rc;
  if ((rc = upload(hd, &hd->d_cdesc, cd.data(), cd.size()))) return rc;
  if ((rc = upload(hd, &hd->d_vol, pb->vol_pts, (size_t)(4 * nvol)))) return rc;
  {
    // repack interface points to 64-byte rows and face points to 32-byte rows so
    // that every point list is a 16-byte aligned contiguous bulk-copy source
    std::vector<double> s8((size_t)8 * nsrf, 0.0), f4((size_t)4 * nfp, 0.0);
    for (int64_t q = 0; q < nsrf; ++q)
      for (int k = 0; k < 7; ++k) s8[8 * q + k] = pb->srf_pts[7 * q + k];
    for (int64_t q = 0; q < nfp; ++q)
      for (int k = 0; k < 3; ++k) f4[4 * q + k] = pb->sf_pts[3 * q + k];
    if ((rc = upload(hd, &hd->d_srf, s8.data(), s8.size()))) return rc;
    if ((rc = upload(hd, &hd->d_sfp, f4.data(), f4.size()))) return rc;
  }
  if ((rc = upload(hd, &hd->d_volptr, pb->vol_ptr, (size_t)(nc ? nc + 1 : 0)))) return rc;
  if (!line_srf.empty() && (rc = upload(hd, &hd->d_line_srf, line_srf.data(), line_srf.size()))) return rc;
  if ((rc = upload(hd, &hd->d_srfptr, pb->srf_ptr, (size_t)(nc ? nc + 1 : 0)))) return rc;
  if ((rc = upload(hd, &hd->d_sfptr, pb->sf_ptr, (size_t)(nsf ? nsf + 1 : 0)))) return rc;
  if ((rc = dispatch_tiles(hd, pb, ud, cd))) return rc;
  if ((rc = upload_tables(p))) return rc;
  if (hd->ttab.empty()) {  // line operators for k_cut's structured faces (any degree)
    switch (p + 1) {
      case 2: rc = build_ttab<2>(hd, pb); break;
      case 3: rc = build_ttab<3>(hd, pb); break;
      case 4: rc = build_ttab<4>(hd, pb); break;
      case 5: rc = build_ttab<5>(hd, pb); break;
      case 6: rc = build_ttab<6>(hd, pb); break;
      case 7: rc = build_ttab<7>(hd, pb); break;
      case 8: rc = build_ttab<8>(hd, pb); break;
      case 9: rc = build_ttab<9>(hd, pb); break;
      default: break;
    }
    if (rc) return rc;
  }
  if ((rc = dispatch_attrs(n))) return rc;
  {
    int dev = device, smc = 148;
    cudaDeviceGetAttribute(&smc, cudaDevAttrMultiProcessorCount, dev);
    hd->sm_count = smc;
  }
  build_facetab(p, pb->h, pb->gp_gamma, pb->gp_kind, pb->tau_v, hd->ft);
  hd->kp.h = pb->h;
  hd->kp.sigma = pb->sipg_gamma / pb->h;
  hd->kp.tau = pb->nitsche_tau / pb->h;
  hd->kp.ih = 1.0 / pb->h;
  hd->kp.ih2 = 1.0 / (pb->h * pb->h);
  hd->kp.i2h = 0.5 / pb->h;
  hd->kp.h2sig = pb->h * pb->h * hd->kp.sigma;
  hd->kp.hh = 0.5 * pb->h;
  hd->kp.mask = hd->mask;
  hd->kp.n_cells = 0;
  CU(cudaStreamCreateWithFlags(&hd->side, cudaStreamNonBlocking));
  CU(cudaEventCreateWithFlags(&hd->ev_fork, cudaEventDisableTiming));
  CU(cudaEventCreateWithFlags(&hd->ev_join, cudaEventDisableTiming));
  CU(cudaEventCreateWithFlags(&hd->ev_started, cudaEventDisableTiming));
  cutfem_stats_t &s = hd->stats;
  std::memset(&s, 0, sizeof(s));
  s.n_active = hd->n_own;
  s.n_uncut = hd->n_uncut;
  s.n_cut = hd->n_cut;
  s.n_vol_pts = nvol;
  s.n_srf_pts = nsrf;
  s.n_face_pts = nfp;
  s.n_faces_struct = n_struct;
  s.n_faces_cut = n_fcut;
  s.n_faces_empty = n_fempty;
  s.n_faces_gp = n_gp;
  s.n_dofs = hd->n_own * n * n * n;
  s.n_ext_dofs = na * n * n * n;
  s.degree = p;
  s.device = device;
  // kernels per apply (single-GPU handle): the cut-cell kernel, then n <= 3 one k_cell
  // launch, n = 4 k_tile2 and / or k_uncw<4,8>, n >= 5 one k_uncw launch
  s.launches_per_apply = (hd->n_cut > 0) + (hd->n <= 3 ? (hd->n_uncut > 0)
                                            : hd->n == 4 ? (hd->t_cnt[0][0] > 0) + (hd->t_cnt[1][0] > 0)
                                                         : (hd->n_uncut > 0));
  return 0;
}

}  // namespace

extern "C" {

const char *cutfem_last_error(void) { return g_err.c_str(); }

int cutfem_setup(const cutfem_problem *pb, int device, cutfem_handle **out) {
  if (!out) return fail(CUTFEM_EINVAL, "out is NULL");
  *out = nullptr;
  cutfem_handle *hd = new (std::nothrow) cutfem_handle();
  if (!hd) return fail(CUTFEM_ENOMEM, "host allocation");
  int rc = setup_impl(pb, device, hd);
  if (rc) {
    free_handle(hd);
    return rc;
  }
  hd->stats.dev_bytes = hd->dev_bytes;
  *out = hd;
  return 0;
}

int cutfem_apply(cutfem_handle *hd, const double *u_dev, double *v_dev, void *cuda_stream) {
  if (!hd) return fail(CUTFEM_EINVAL, "null handle");
  if (hd->n_active > 0 && (!u_dev || !v_dev)) return fail(CUTFEM_EINVAL, "null vector");
  if (u_dev == v_dev && hd->n_active > 0) return fail(CUTFEM_EINVAL, "u and v must not alias");
  // 16 bytes: blocks are moved by bulk copies / 16-byte vector accesses (even n)
  if (((uintptr_t)u_dev | (uintptr_t)v_dev) & 15) return fail(CUTFEM_EINVAL, "vectors must be 16-byte aligned");
  CU(cudaSetDevice(hd->device));
  return dispatch_apply(hd, u_dev, v_dev, (cudaStream_t)cuda_stream);
}

int cutfem_apply_kernel(cutfem_handle *hd, int which, const double *u_dev, double *v_dev, void *cuda_stream) {
  if (!hd) return fail(CUTFEM_EINVAL, "null handle");
  if (which != 0 && which != 1) return fail(CUTFEM_EINVAL, "which must be 0 (structured) or 1 (unstructured)");
  if (u_dev == v_dev && hd->n_active > 0) return fail(CUTFEM_EINVAL, "u and v must not alias");
  if (hd->n_active > 0 && (!u_dev || !v_dev)) return fail(CUTFEM_EINVAL, "null vector");
  if (((uintptr_t)u_dev | (uintptr_t)v_dev) & 15) return fail(CUTFEM_EINVAL, "vectors must be 16-byte aligned");
  CU(cudaSetDevice(hd->device));
  return dispatch_apply(hd, u_dev, v_dev, (cudaStream_t)cuda_stream, which == 0 ? 1 : 2);
}

int cutfem_apply_host(cutfem_handle *hd, const double *u_host, double *v_host, void *cuda_stream) {
  if (!hd) return fail(CUTFEM_EINVAL, "null handle");
  if (hd->stats.n_dofs > 0 && (!u_host || !v_host)) return fail(CUTFEM_EINVAL, "null vector");
  CU(cudaSetDevice(hd->device));
  const size_t bytes = sizeof(double) * (size_t)hd->stats.n_dofs;
  // u holds the ghost blocks behind the owned ones on a distributed handle
  // (the halo exchange receives into them): size it with n_ext_dofs
  const size_t ubytes = sizeof(double) * (size_t)std::max<int64_t>(hd->stats.n_ext_dofs, hd->stats.n_dofs);
  if (!hd->d_u) {
    CU(cudaMalloc(&hd->d_u, std::max<size_t>(ubytes, 16)));
    CU(cudaMalloc(&hd->d_v, std::max<size_t>(bytes, 16)));
    hd->dev_bytes += (int64_t)(ubytes + bytes);
  }
  cudaStream_t st = (cudaStream_t)cuda_stream;
  CU(cudaMemcpyAsync(hd->d_u, u_host, bytes, cudaMemcpyHostToDevice, st));
  int rc = dispatch_apply(hd, hd->d_u, hd->d_v, st);
  if (rc) return rc;
  CU(cudaMemcpyAsync(v_host, hd->d_v, bytes, cudaMemcpyDeviceToHost, st));
  CU(cudaStreamSynchronize(st));
  return 0;
}

int cutfem_apply_host_batch(cutfem_handle *hd, const double *const *u_host, double *const *v_host, int64_t nbatch,
                            void *cuda_stream) {
  if (!hd) return fail(CUTFEM_EINVAL, "null handle");
  if (hd->dist) return fail(CUTFEM_EUNSUPPORTED, "batched host applies on a distributed handle");
  if (nbatch < 0 || (nbatch > 0 && (!u_host || !v_host))) return fail(CUTFEM_EINVAL, "batch arrays");
  for (int64_t k = 0; k < nbatch; ++k)
    if (hd->stats.n_dofs > 0 && (!u_host[k] || !v_host[k])) return fail(CUTFEM_EINVAL, "null vector in the batch");
  CU(cudaSetDevice(hd->device));
  const size_t bytes = sizeof(double) * (size_t)hd->stats.n_dofs;
  if (!hd->d_ub[0]) {
    for (int b = 0; b < 2; ++b) {
      CU(cudaMalloc(&hd->d_ub[b], std::max<size_t>(bytes, 16)));
      CU(cudaMalloc(&hd->d_vb[b], std::max<size_t>(bytes, 16)));
      CU(cudaEventCreateWithFlags(&hd->ev_in[b], cudaEventDisableTiming));
      CU(cudaEventCreateWithFlags(&hd->ev_done[b], cudaEventDisableTiming));
      CU(cudaEventCreateWithFlags(&hd->ev_out[b], cudaEventDisableTiming));
    }
    CU(cudaStreamCreateWithFlags(&hd->s_h2d, cudaStreamNonBlocking));
    CU(cudaStreamCreateWithFlags(&hd->s_d2h, cudaStreamNonBlocking));
    hd->dev_bytes += (int64_t)(4 * bytes);
  }
  cudaStream_t st = (cudaStream_t)cuda_stream;
  // the copy streams start after the caller's prior work on st
  CU(cudaEventRecord(hd->ev_done[0], st));
  CU(cudaStreamWaitEvent(hd->s_h2d, hd->ev_done[0], 0));
  CU(cudaStreamWaitEvent(hd->s_d2h, hd->ev_done[0], 0));
  for (int64_t k = 0; k < nbatch; ++k) {
    const int b = (int)(k & 1);
    // u_k into buffer b once apply k-2 (the last reader of d_ub[b]) is done
    if (k >= 2) CU(cudaStreamWaitEvent(hd->s_h2d, hd->ev_done[b], 0));
    CU(cudaMemcpyAsync(hd->d_ub[b], u_host[k], bytes, cudaMemcpyHostToDevice, hd->s_h2d));
    CU(cudaEventRecord(hd->ev_in[b], hd->s_h2d));
    // apply k once u_k has landed and v_{k-2} has left d_vb[b]
    CU(cudaStreamWaitEvent(st, hd->ev_in[b], 0));
    if (k >= 2) CU(cudaStreamWaitEvent(st, hd->ev_out[b], 0));
    int rc = dispatch_apply(hd, hd->d_ub[b], hd->d_vb[b], st);
    if (rc) return rc;
    CU(cudaEventRecord(hd->ev_done[b], st));
    // v_k out once apply k is done
    CU(cudaStreamWaitEvent(hd->s_d2h, hd->ev_done[b], 0));
    CU(cudaMemcpyAsync(v_host[k], hd->d_vb[b], bytes, cudaMemcpyDeviceToHost, hd->s_d2h));
    CU(cudaEventRecord(hd->ev_out[b], hd->s_d2h));
  }
  CU(cudaStreamSynchronize(hd->s_d2h));
  CU(cudaStreamSynchronize(st));
  return 0;
}

// debug: kernel timeline of the last applies (build with -DCUTFEM_TIMELINE; not in the
// public header).  reset != 0 clears it; out[2k], out[2k+1] = first start / last end (ns)
int cutfem_debug_timeline(int reset, unsigned long long *out) {
#ifdef CUTFEM_TIMELINE
  unsigned long long h[8][2];
  if (reset) {
    for (int k = 0; k < 8; ++k) {
      h[k][0] = ~0ull;
      h[k][1] = 0;
    }
    CU(cudaMemcpyToSymbol(g_tl, h, sizeof(h)));
    std::vector<unsigned long long> z(3 * 8192, 0);
    CU(cudaMemcpyToSymbol(g_tlw, z.data(), sizeof(unsigned long long) * 3 * 8192));
  } else {
    CU(cudaMemcpyFromSymbol(h, g_tl, sizeof(h)));
    for (int k = 0; k < 8; ++k) {
      out[2 * k] = h[k][0];
      out[2 * k + 1] = h[k][1];
    }
    CU(cudaMemcpyFromSymbol(out + 16, g_tlw, sizeof(unsigned long long) * 3 * 8192));
  }
  return 0;
#else
  (void)reset;
  (void)out;
  return fail(CUTFEM_EUNSUPPORTED, "built without CUTFEM_TIMELINE");
#endif
}

int cutfem_stats(const cutfem_handle *hd, cutfem_stats_t *out) {
  if (!hd || !out) return fail(CUTFEM_EINVAL, "null");
  *out = hd->stats;
  out->dev_bytes = hd->dev_bytes;
  return 0;
}

int cutfem_destroy(cutfem_handle *hd) {
  if (!hd) return 0;
  cudaSetDevice(hd->device);
  cudaDeviceSynchronize();
  free_handle(hd);
  return 0;
}

}  // extern "C"

#include "csr.inl"
#include "dist.inl"
#include "cg.inl"
#include "h1.inl"
#include "mg.inl"
