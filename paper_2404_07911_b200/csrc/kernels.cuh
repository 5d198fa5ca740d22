// sm_100a FP64 kernels of the DG-CutFEM operator apply (included by cutfem.cu).
//
// Two element-centric kernels; every v block is written exactly once by the
// kernel that owns its cell, so no atomics are needed (BASELINE north_star:
// "Face contributions use warp-level primitives or element-centric loops so
// that no atomics land on the hot path").  Each cell also evaluates its own
// side of the six faces (SIPG, ghost penalty, cut-face SIPG), reading the
// neighbour blocks from L2.
//
//   structured cells (Alg. 1 "inside" branch): kernels_tile.cuh
//     (k_tile2, k_uncw, k_cell);
//   k_cut<N>:   unstructured cells (Alg. 1 "intersected" branch):
//     one CTA per cut cell, one thread per quadrature point for the per-point
//     tensor evaluation (eq:unstructured_cell), then a DoF-parallel
//     reduction over points for the integration; faces with the face-normal
//     reduction + in-face per-point evaluation (eq:unstructured_face P:491-496).
#pragma once
#include <cstdint>
#include <type_traits>

#define CUTFEM_NMAX 9

// Opt-in timeline probe (build with -DCUTFEM_TIMELINE; tools/timeline.py): first CTA
// start and last CTA end of each kernel family, from %globaltimer (ns).  Not in the
// default build (it uses atomics).
#ifdef CUTFEM_TIMELINE
__device__ unsigned long long g_tl[8][2];
__device__ __forceinline__ unsigned long long gtimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}
__device__ unsigned long long g_tlw[3][8192];  // k_cutp: per-warp end time, start time, SM id
#define TL_WARP_END(gw) \
  if ((threadIdx.x & 31) == 0 && (gw) < 8192) g_tlw[0][gw] = gtimer();
#define TL_WARP_BEGIN(gw)                                 \
  if ((threadIdx.x & 31) == 0 && (gw) < 8192) {           \
    unsigned sm;                                          \
    asm volatile("mov.u32 %0, %%smid;" : "=r"(sm));       \
    g_tlw[1][gw] = gtimer();                              \
    g_tlw[2][gw] = sm;                                    \
  }
#define TL_BEGIN(k) \
  if (threadIdx.x == 0) atomicMin(&g_tl[k][0], gtimer());
#define TL_END(k) \
  if (threadIdx.x == 0) atomicMax(&g_tl[k][1], gtimer());
#else
#define TL_BEGIN(k)
#define TL_END(k)
#define TL_WARP_END(gw)
#define TL_WARP_BEGIN(gw)
#endif
#ifndef CUTFEM_USE_BULK
#define CUTFEM_USE_BULK 1
#endif

// Even-odd factors of a centro-symmetric n x n matrix M (M[i][j] = M[n-1-i][n-1-j]):
//   E[i][j] = (M[i][j] + M[i][n-1-j]) / 2 (j < H), E[i][H] = M[i][H] (n odd), i < HC
//   O[i][j] = (M[i][j] - M[i][n-1-j]) / 2, i, j < H
// out_i = E_i + O_i, out_{n-1-i} = E_i - O_i: n^2/2 + 2n flops instead of n^2 FMAs.
struct EO {
  double E[25];
  double O[16];
};

struct RefTab {
  EO S;   // GLL values -> Gauss values
  EO St;  // transpose (integration back to GLL)
  EO Kc;  // D_g^T W D_g on the Gauss collocation points
  EO M;   // GLL mass
  double x[CUTFEM_NMAX];     // GLL nodes
  double cinv[CUTFEM_NMAX];  // 1 / prod_{m != a} (x_a - x_m)
  double gw[CUTFEM_NMAX];    // Gauss weights
  double d0[CUTFEM_NMAX];    // l_a'(0)
  double d1[CUTFEM_NMAX];    // l_a'(1)
  double mc[CUTFEM_NMAX][CUTFEM_NMAX];  // l_a(x) = sum_k mc[a][k] t^k, t = 2x - 1 (k_cutp basis)
  double md[CUTFEM_NMAX][CUTFEM_NMAX];  // 2 k mc[a][k]: d/dx = 2 d/dt
};

__constant__ RefTab c_ref[8];  // index N - 2

// Handle-specific ghost-penalty line operators (h and gp_gamma folded in):
//   Goo[s][m][a] = h sum_j g_j e_j[m] e_j[a], Gon[s][m][a] = h sum_j g_j e_j[m] o_j[a]
// with e_j = l^(j)(own face), o_j = l^(j)(neighbour face); s = 0 own cell is the
// minus side (face at xi_d = 1), s = 1 own cell is the plus side.
// Per-handle line operators (h, penalties folded), all warp-uniform.  Only the
// lo-face (s = 0) variants are stored: every 1-D operator here is
// centro-symmetric (GLL nodes and Gauss points are symmetric about 1/2), so the
// hi face uses the reversed entries:  l'_a(1) = -l'_{n-1-a}(0),
// cJ_hi[m] = cJ_lo[n-1-m], cA_hi[m] = -cA_lo[n-1-m], G_hi[m][a] = G_lo[n-1-m][n-1-a],
// and L, M satisfy X[i][j] = X[n-1-i][n-1-j].  Reading only the canonical half
// keeps ~20 distinct constants live next to the 64-double accumulator.
template <int N>
struct TileTab {
  double L[N * N];    // M^{-1} h K1: volume term along one axis
  double M[N * N];    // GLL mass M1
  double d0[N];       // l'_a(0)
  double cJ[N];       // SIPG (lo face): w_line += cJ [u] + cA (d u_own + d u_nb)
  double cA[N];
  double Goo[N * N];  // ghost penalty (lo face), own line:        M^{-1} G_oo
  double Gon[N * N];  // ghost penalty (lo face), neighbour line: -M^{-1} G_on
  // k_tile2 (cells with all six faces, no ghost penalty): the volume line operator and
  // the OWN-side SIPG parts of both faces folded into one operator (centro-symmetric),
  // the neighbour parts as a rank-2 update (lo face: w += nJ u_nb(N-1) + nA sum_k
  // d0[N-1-k] u_nb(k); the hi face mirrored); the handle's term mask is built in
  double Lf[N * N];
  double nJ[N], nA[N];
  EO Leo, Meo;  // even-odd factors of L and M (k_uncw, n >= 5; north_star "even-odd decomposition")
};

// canonical index of a centro-symmetric n x n matrix entry
template <int N>
__device__ __forceinline__ constexpr int csym(int k) {
  return k < N * N - 1 - k ? k : N * N - 1 - k;
}


struct FaceTab {
  double Goo[2][CUTFEM_NMAX * CUTFEM_NMAX];
  double Gon[2][CUTFEM_NMAX * CUTFEM_NMAX];
};

struct KParams {
  double h;      // cell edge
  double sigma;  // SIPG penalty gamma / h
  double tau;    // Nitsche penalty tau_D / h
  double ih;     // 1 / h
  double ih2;    // 1 / h^2
  double i2h;    // 1 / (2 h)
  double h2sig;  // h^2 sigma
  double hh;     // h / 2
  uint32_t mask; // CUTFEM_TERM_* bits
  int32_t n_cells;
};

// per uncut cell: block id, 6 face neighbours (-1: none / inactive), GP bits
struct __align__(16) UDesc {
  int32_t blk;
  int32_t nb[6];
  uint32_t flags;  // bit f: ghost penalty on face f (neighbour cut)
};

// per cut cell
struct __align__(16) CDesc {
  int32_t blk;
  int32_t nb[6];
  uint32_t flags;  // bit f: GP; bit 6+f: structured SIPG; bit 12+f: cut-face SIPG (points)
  int32_t sf[6];   // face-point list index for cut faces, else -1
  int32_t cut;     // ordinal in vol_ptr / srf_ptr
  int32_t pad;
  int64_t vb, sb;  // first volume / interface point
  int32_t nv, ns;  // volume / interface point counts
};

#define TERM_CELL 1u
#define TERM_SIPG 2u
#define TERM_NITSCHE 4u
#define TERM_GP 8u

template <int N>
__device__ __forceinline__ void eo_mv(const EO &m, const double (&in)[N], double (&out)[N]) {
  constexpr int H = N / 2, HC = (N + 1) / 2;
  double e[HC], o[H];
#pragma unroll
  for (int j = 0; j < H; ++j) {
    e[j] = in[j] + in[N - 1 - j];
    o[j] = in[j] - in[N - 1 - j];
  }
  if (N & 1) e[H] = in[H];
#pragma unroll
  for (int i = 0; i < H; ++i) {
    double E = 0.0, O = 0.0;
#pragma unroll
    for (int j = 0; j < HC; ++j) E = fma(m.E[i * HC + j], e[j], E);
#pragma unroll
    for (int j = 0; j < H; ++j) O = fma(m.O[i * H + j], o[j], O);
    out[i] = E + O;
    out[N - 1 - i] = E - O;
  }
  if (N & 1) {
    double E = 0.0;
#pragma unroll
    for (int j = 0; j < HC; ++j) E = fma(m.E[H * HC + j], e[j], E);
    out[H] = E;
  }
}

// Padded cell block in shared memory: index c*PS + b*P + a.  (P, PS) per N
// minimise 64-bit bank conflicts of the 1-D lines in all three directions
// (searched offline: worst case 2-way for N >= 4, conflict-free for N <= 3).
template <int N>
struct BlkPad {
  static constexpr int P = (N == 2 || N == 3 || N == 5 || N == 7) ? N : N + 1;
  static constexpr int PS = N == 2 ? 4 : (N == 3 ? 12 : (N == 5 ? 25 : (N == 7 ? 52 : N * (N + 1))));
};
template <int N>
struct Blk {
  static constexpr int P = BlkPad<N>::P;
  static constexpr int PS = BlkPad<N>::PS;
  static constexpr int NN = N * N;
  static constexpr int N3 = N * N * N;
  static constexpr int SZ = N * PS;
  __device__ static __forceinline__ int pad(int l) { return (l / NN) * PS + ((l / N) % N) * P + (l % N); }
  __device__ static __forceinline__ int at(int a, int b, int c) { return c * PS + b * P + a; }
  template <int D>
  __host__ __device__ static constexpr int lstride() { return D == 0 ? 1 : (D == 1 ? P : PS); }
  template <int D>
  __device__ static __forceinline__ int lbase(int t) {
    const int t0 = t % N, t1 = t / N;
    return D == 0 ? t1 * PS + t0 * P : (D == 1 ? t1 * PS + t0 : t1 * P + t0);
  }
  // line t (t = t0 + N*t1, t0 along the lower in-face axis) in direction d
  __device__ static __forceinline__ void line(int d, int t, int &base, int &stride) {
    const int t0 = t % N, t1 = t / N;
    if (d == 0) {
      base = t1 * PS + t0 * P;
      stride = 1;
    } else if (d == 1) {
      base = t1 * PS + t0;
      stride = P;
    } else {
      base = t1 * P + t0;
      stride = PS;
    }
  }
};

// Unpadded block (the global layout): destination of bulk (TMA) copies.
template <int N>
struct BlkU {
  static constexpr int P = N, PS = N * N, NN = N * N, N3 = N * N * N, SZ = N3;
  __device__ static __forceinline__ int at(int a, int b, int c) { return c * PS + b * P + a; }
  template <int D>
  __host__ __device__ static constexpr int lstride() { return D == 0 ? 1 : (D == 1 ? P : PS); }
  template <int D>
  __device__ static __forceinline__ int lbase(int t) {
    const int t0 = t % N, t1 = t / N;
    return D == 0 ? t1 * PS + t0 * P : (D == 1 ? t1 * PS + t0 : t1 * P + t0);
  }
};

// ---- programmatic dependent launch (griddepcontrol, sm_90+).  An apply at p <= 3 is
// ONE stream: k_cutp (normal launch) -> uncut-cell kernel(s) launched with the
// programmatic-serialization attribute.  Every CTA triggers its dependents at its
// start, so a dependent grid is released only once ALL k_cutp CTAs have begun (k_cutp,
// the long pole, holds its SM slots first) and then fills the slots k_cutp's warps
// free.  The dependents never read what their primary writes (disjoint v blocks), so
// they do not wait up front; one CTA of each dependent waits at its END, which makes
// the dependent grid complete only after its primary has completed (transitively the
// whole apply), so stream order after the apply holds.
__device__ __forceinline__ void pdl_trigger() { asm volatile("griddepcontrol.launch_dependents;\n" ::: "memory"); }
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;\n" ::: "memory"); }

// ---- mbarrier + cp.async.bulk (TMA bulk copy, SASS UBLKCP) helpers
__device__ __forceinline__ uint32_t smem_u32(const void *p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(uint64_t *bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_fence_init() {
  asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t *bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(smem_u32(bar)), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void bulk_g2s(void *dst, const void *src, uint32_t bytes, uint64_t *bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n" ::"r"(
                   smem_u32(dst)),
               "l"(src), "r"(bytes), "r"(smem_u32(bar))
               : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t *bar, uint32_t parity) {
  asm volatile(
      "{\n .reg .pred p;\n WAIT_%=:\n mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n @!p bra WAIT_%=;\n}\n" ::"r"(
          smem_u32(bar)),
      "r"(parity)
      : "memory");
}
// generic-proxy accesses before this fence are ordered before later async-proxy (bulk) writes
__device__ __forceinline__ void fence_proxy_async() { asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory"); }

// MODE 0: dst = M src; MODE 1: dst += s * M src; MODE 2: dst = s * M src
template <int N, int MODE>
__device__ __forceinline__ void sweep_line(const double *src, double *dst, int base, int stride,
                                           const EO &m, double s) {
  double in[N], out[N];
#pragma unroll
  for (int k = 0; k < N; ++k) in[k] = src[base + k * stride];
  eo_mv<N>(m, in, out);
#pragma unroll
  for (int k = 0; k < N; ++k) {
    if (MODE == 0) dst[base + k * stride] = out[k];
    else if (MODE == 1) dst[base + k * stride] = fma(s, out[k], dst[base + k * stride]);
    else dst[base + k * stride] = s * out[k];
  }
}

// 1-D Lagrange basis values and derivatives at t (product form with prefix /
// suffix products; "evaluate the actual polynomial basis by 1D evaluations").
template <int N>
__device__ __forceinline__ void basis_vd(const RefTab &R, double t, double (&v)[N], double (&dv)[N]) {
  double d[N], pre[N], dpre[N];
#pragma unroll
  for (int m = 0; m < N; ++m) d[m] = t - R.x[m];
  double p = 1.0, dp = 0.0;
#pragma unroll
  for (int a = 0; a < N; ++a) {
    pre[a] = p;
    dpre[a] = dp;
    dp = fma(dp, d[a], p);
    p *= d[a];
  }
  double s = 1.0, ds = 0.0;
#pragma unroll
  for (int a = N - 1; a >= 0; --a) {
    v[a] = R.cinv[a] * pre[a] * s;
    dv[a] = R.cinv[a] * fma(dpre[a], s, pre[a] * ds);
    ds = fma(ds, d[a], s);
    s *= d[a];
  }
}

// The thread's half of a line's basis for the line_chunks thread pairs: entries
// i0 + ii (ii < H = ceil(n/2), i0 = part H; an index >= n is a zero dummy) of l_a(x),
// l_a'(x).  The GLL nodes are symmetric, l_{n-1-a}(x) = l_a(1 - x), so the upper half
// is the lower half at 1 - x in reverse order with the derivative's sign flipped
// (odd n: shifted by one, the middle function belongs to the lower half): H
// functions and H selects instead of n functions and H n selects.
template <int N, int H>
__device__ __forceinline__ void basis_vd_half(const RefTab &R, double x, int part, double (&vh)[H], double (&dh)[H]) {
  static_assert(H == (N + 1) / 2, "H = ceil(n / 2)");
  constexpr int SH = N % 2;  // odd n: part 1's entry ii is l_{H-2-ii}(1 - x), the last a dummy
  const double t = part ? 1.0 - x : x;
  double d[N], pre[H], dpre[H], lv[H], ld[H];
#pragma unroll
  for (int m = 0; m < N; ++m) d[m] = t - R.x[m];
  double p = 1.0, dp = 0.0;
#pragma unroll
  for (int a = 0; a < H; ++a) {
    pre[a] = p;
    dpre[a] = dp;
    dp = fma(dp, d[a], p);
    p *= d[a];
  }
  double s = 1.0, ds = 0.0;
#pragma unroll
  for (int a = N - 1; a >= 0; --a) {
    if (a < H) {
      lv[a] = R.cinv[a] * pre[a] * s;
      ld[a] = R.cinv[a] * fma(dpre[a], s, pre[a] * ds);
    }
    if (a > 0) {
      ds = fma(ds, d[a], s);
      s *= d[a];
    }
  }
#pragma unroll
  for (int ii = 0; ii < H; ++ii) {
    const int m = H - 1 - SH - ii;  // mirrored index (< 0: the odd-n dummy)
    vh[ii] = part ? (m >= 0 ? lv[m >= 0 ? m : 0] : 0.0) : lv[ii];
    dh[ii] = part ? (m >= 0 ? -ld[m >= 0 ? m : 0] : 0.0) : ld[ii];
  }
}

template <int N>
__device__ __forceinline__ void basis_v(const RefTab &R, double t, double (&v)[N]) {
  double d[N], pre[N];
#pragma unroll
  for (int m = 0; m < N; ++m) d[m] = t - R.x[m];
  double p = 1.0;
#pragma unroll
  for (int a = 0; a < N; ++a) {
    pre[a] = p;
    p *= d[a];
  }
  double s = 1.0;
#pragma unroll
  for (int a = N - 1; a >= 0; --a) {
    v[a] = R.cinv[a] * pre[a] * s;
    s *= d[a];
  }
}

__device__ __forceinline__ void cp_async8(void *smem, const void *gmem) {
  const unsigned s = (unsigned)__cvta_generic_to_shared(smem);
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"(s), "l"(gmem));
}
__device__ __forceinline__ void cp_async16(void *smem, const void *gmem) {
  const unsigned s = (unsigned)__cvta_generic_to_shared(smem);
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(s), "l"(gmem));
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::); }
template <int K>
__device__ __forceinline__ void cp_async_wait() { asm volatile("cp.async.wait_group %0;\n" ::"n"(K)); }

// ============================================================== cut cells
#ifndef CUT_PREF_MAXN
#define CUT_PREF_MAXN 9  // neighbour blocks by cp.async at entry up to this n (round 2: 7 -> 9,
                         // with the w-space faces: C3 p=7 apply 1139 -> 998 us, p=8 2225 -> 2024 us)
#endif
// CTAs per SM the register allocation of k_cut<n> must allow (ptxas's own choice
// without a bound gave these at n = 5..9; an explicit 1 lets it take up to 255
// registers and was measured 15 % slower at n = 5, 7)
#ifndef CUT_MINB5
#define CUT_MINB5 6
#endif
#ifndef CUT_MINB6
#define CUT_MINB6 3
#endif
#ifndef CUT_MINB7
#define CUT_MINB7 3
#endif
#ifndef CUT_LB_UNROLL
#define CUT_LB_UNROLL 0  // unroll factor of the line base contraction's outer loop (0: per degree,
                         // full up to n = 7, none above: measured)
#endif
#ifndef CUT_WFACE_MASK
#define CUT_WFACE_MASK 0x3e0  // bit n: structured faces in w-space (n = 5..9)
#endif
#ifndef CUT_BFACE_MASK
#define CUT_BFACE_MASK 0x1c0  // bit n: the cut faces batched (n = 6, 7, 8)
#endif
#ifndef CUT_PPF_MASK
#define CUT_PPF_MASK 0x300  // bit n: prefetch the point rows (n = 8, 9: measured faster; 6, 7 slower)
#endif
#ifndef CUT_ROWINT_MINN
#define CUT_ROWINT_MINN 5
#endif
#ifndef CUT_RPT
#define CUT_RPT 3  // x-rows per thread in the row integration, n = 5, 6
#endif
#ifndef CUT_RPT7
#define CUT_RPT7 3  // n >= 7
#endif
#ifndef CUT_SPLIT_MASK
#define CUT_SPLIT_MASK 0x2ff  // bit n: split the point phase over THREADS / CHUNK threads (not n = 8: measured slower)
#endif
#ifndef CUT_TH5
#define CUT_TH5 64  // threads per k_cut<5> CTA (one cut cell per CTA; 128 -> 64 with 6 CTAs / SM: C3 p=4 k_cut 426 -> 397 us)
#endif
#ifndef CUT_CH5
#define CUT_CH5 32  // points per chunk at n = 5 (THREADS / CHUNK = SPL threads per point)
#endif
#ifndef CUT_TH6
#define CUT_TH6 128
#endif
#ifndef CUT_CH6
#define CUT_CH6 64
#endif
template <int N>
struct CutCfg {
  static constexpr int THREADS = N == 5 ? CUT_TH5 : (N == 6 ? CUT_TH6 : 128);
  static constexpr int MINB = N <= 4 ? 1 : (N == 5 ? CUT_MINB5 : (N == 6 ? CUT_MINB6 : (N == 7 ? CUT_MINB7 : 2)));
  static constexpr int NN = N * N, N3 = N * N * N;
  static constexpr int ROW0 = 2 * NN + 2 * N;
  static constexpr int ROW = (ROW0 % 2 == 0) ? ROW0 + 1 : ROW0;  // odd stride: no bank conflicts
  static constexpr int CHUNK = N <= 4 ? 128 : (N == 5 ? CUT_CH5 : (N == 6 ? CUT_CH6 : 32));
  static constexpr int FROW = 2 * N + 3;  // cut-face point row: l(s), l(t), c1, c2 (+pad)
  static constexpr int KPT = (N3 + THREADS - 1) / THREADS;
  // integration phase: each thread owns RPT x-rows (b, c) of the block (sharing the
  // x-basis loads), TG threads cover the N^2 rows, G groups split the chunk's points
  // (N >= 7; below, one thread per DoF looping over the points is faster)
  static constexpr bool ROWINT = N >= CUT_ROWINT_MINN;
  static constexpr int RPT = ROWINT ? (N >= 7 ? CUT_RPT7 : CUT_RPT) : 1;
  static constexpr int TG = ROWINT ? (NN + RPT - 1) / RPT : THREADS;
  static constexpr int G = ROWINT ? THREADS / TG : 1;
  // per-point phase: SPL threads per point, each evaluating CPS of the N z-planes
  static constexpr int SPL = ((CUT_SPLIT_MASK >> N) & 1) ? THREADS / CHUNK : 1, CPS = (N + SPL - 1) / SPL;
  // neighbour blocks prefetched (cp.async at entry, overlapping the point work) up
  // to n = CUT_PREF_MAXN; above, loaded face by face
  static constexpr bool PREF = N <= CUT_PREF_MAXN;
  static constexpr int NBN = PREF ? 6 : 1;
  // structured faces in w-space (one parallel pass + one M (x) M (x) M sweep) instead
  // of face by face; needs the prefetched neighbours (measured faster at n = 5, 6, 7)
  static constexpr bool WFACE = PREF && ((CUT_WFACE_MASK >> N) & 1);
  // (w-space degrees) every cut face of the cell in one batched pass instead of face by
  // face with its barriers (C3 p=5 cut kernel 444 -> 401 us, p=6 767 -> 750, p=7 888 -> 866;
  // p=4 398 -> 403, p=8 1861 -> 1895: off there)
  static constexpr bool BFACE = WFACE && ((CUT_BFACE_MASK >> N) & 1);
  // U, T, R, NB[NBN] (padded blocks) + JA, JB, FC1, FC2 (NN each) + point rows
  // point rows of the next chunk prefetched (cp.async, double buffer of 8 doubles a
  // point) while the current one is processed
  static constexpr bool PPF = N >= 5 && ((CUT_PPF_MASK >> N) & 1);
  static constexpr int PBUF = PPF ? 2 * CHUNK * 8 : 0;
  static constexpr int OFF_PS = (3 + NBN) * Blk<N>::SZ + 4 * NN;
  static constexpr int OFF_PB = (OFF_PS + CHUNK * ROW + 1) & ~1;  // 16-byte aligned
  // volume lines (ROWINT degrees): rows of 3 NN + 3 N doubles, CL lines per chunk, whose
  // points [xi, eta, zeta, W] are staged in shared memory (LB) once per chunk
  static constexpr int LRL0 = 3 * NN + 3 * N, LRL = (LRL0 % 2 == 0) ? LRL0 + 1 : LRL0;
  static constexpr int LCL0 = (CHUNK * ROW) / LRL, LCL = LCL0 < THREADS / 2 ? LCL0 : THREADS / 2;
  static constexpr int LBUF = ROWINT ? LCL * N * 4 : 0;
  static constexpr int LSBUF = ROWINT ? LCL * 6 : 0;  // the lines' interface records
  static constexpr int OFF_LB = OFF_PB + PBUF;  // even: 16-byte aligned
  static constexpr int SMEM_D = OFF_LB + LBUF + LSBUF;
  static constexpr int SMEM = SMEM_D * 8;
};

// E-phase for one point: returns (value, reference gradient)
template <int N>
__device__ __forceinline__ void eval_point(const double *U, const double (&vx)[N], const double (&dvx)[N],
                                           const double (&vy)[N], const double (&dvy)[N],
                                           const double (&vz)[N], const double (&dvz)[N], double &u0,
                                           double &ux, double &uy, double &uz) {
  constexpr int P = Blk<N>::P, PS = Blk<N>::PS;
  u0 = ux = uy = uz = 0.0;
#pragma unroll
  for (int c = 0; c < N; ++c) {
    double t00 = 0.0, t10 = 0.0, t01 = 0.0;
#pragma unroll
    for (int b = 0; b < N; ++b) {
      double s0 = 0.0, s1 = 0.0;
      const double *row = U + c * PS + b * P;
#pragma unroll
      for (int a = 0; a < N; ++a) {
        const double uu = row[a];
        s0 = fma(vx[a], uu, s0);
        s1 = fma(dvx[a], uu, s1);
      }
      t00 = fma(vy[b], s0, t00);
      t10 = fma(dvy[b], s0, t10);
      t01 = fma(vy[b], s1, t01);
    }
    u0 = fma(vz[c], t00, u0);
    uz = fma(dvz[c], t00, uz);
    uy = fma(vz[c], t10, uy);
    ux = fma(vz[c], t01, ux);
  }
}

// same, with the block in layout L (padded or unpadded)
template <int N, class L>
__device__ __forceinline__ void eval_point_l(const double *U, const double (&vx)[N], const double (&dvx)[N],
                                             const double (&vy)[N], const double (&dvy)[N],
                                             const double (&vz)[N], const double (&dvz)[N], double &u0,
                                             double &ux, double &uy, double &uz) {
  u0 = ux = uy = uz = 0.0;
#pragma unroll
  for (int c = 0; c < N; ++c) {
    double t00 = 0.0, t10 = 0.0, t01 = 0.0;
#pragma unroll
    for (int b = 0; b < N; ++b) {
      double s0 = 0.0, s1 = 0.0;
      const double *row = U + c * L::PS + b * L::P;
#pragma unroll
      for (int a = 0; a < N; ++a) {
        const double uu = row[a];
        s0 = fma(vx[a], uu, s0);
        s1 = fma(dvx[a], uu, s1);
      }
      t00 = fma(vy[b], s0, t00);
      t10 = fma(dvy[b], s0, t10);
      t01 = fma(vy[b], s1, t01);
    }
    u0 = fma(vz[c], t00, u0);
    uz = fma(dvz[c], t00, uz);
    uy = fma(vz[c], t10, uy);
    ux = fma(vz[c], t01, ux);
  }
}

template <int N, bool SURF>
__device__ __forceinline__ void point_chunks(const double *__restrict__ pts, int64_t pb, int64_t pe,
                                             const double *U, double *PS, double (&acc)[CutCfg<N>::RPT][N],
                                             const KParams &kp, const RefTab &R) {
  using C = CutCfg<N>;
  constexpr int NN = C::NN, ROW = C::ROW, RPT = C::RPT, TG = C::TG, G = C::G;
  const int tid = threadIdx.x;
  const int grp = tid / TG, rl = tid % TG;
  constexpr int SPL = C::SPL, CPS = C::CPS;
  const int pq = tid / SPL, part = tid % SPL;  // point of the chunk, z-plane share
  const double ih = kp.ih, ih2 = kp.ih2;  // (no divisions in the kernels)
  constexpr int RL = SURF ? 8 : 4;  // doubles per point row
  double *PB = PS - C::OFF_PS + C::OFF_PB;  // [2][CHUNK * 8] prefetch buffers (16-byte aligned)
  // rows [c, min(c + CHUNK, pe)) into buffer b: 16-byte pieces over the CTA
  auto prefetch = [&](int64_t c, int b) {
    if constexpr (C::PPF) {
      const int cnt = (int)((pe - c) < C::CHUNK ? (pe - c) : C::CHUNK);
      for (int e = tid; e < cnt * (RL / 2); e += C::THREADS)
        cp_async16(PB + b * C::CHUNK * 8 + 2 * e, pts + RL * c + 2 * e);
      cp_async_commit();
    }
  };
  if (pb < pe) prefetch(pb, 0);
  int it = 0;
  for (int64_t c0 = pb; c0 < pe; c0 += C::CHUNK, ++it) {
    if constexpr (C::PPF) {
      // the next chunk goes to the other buffer (last read before the previous
      // chunk's integration barrier); wait for this one
      if (c0 + C::CHUNK < pe) {
        prefetch(c0 + C::CHUNK, (it + 1) & 1);
        cp_async_wait<1>();
      } else {
        cp_async_wait<0>();
      }
      __syncthreads();
    }
    if (pq < C::CHUNK) {
      const int64_t q = c0 + pq;
      double xi = 0.5, eta = 0.5, zeta = 0.5, W = 0.0, nx = 0.0, ny = 0.0, nz = 0.0;
      if (C::PPF && q < pe) {
        const double *p = PB + (it & 1) * C::CHUNK * 8 + RL * pq;
        const double2 a = *reinterpret_cast<const double2 *>(p);
        const double2 b = *reinterpret_cast<const double2 *>(p + 2);
        xi = a.x;
        eta = a.y;
        zeta = b.x;
        if (SURF) {
          const double2 c = *reinterpret_cast<const double2 *>(p + 4);
          const double2 d = *reinterpret_cast<const double2 *>(p + 6);
          nx = b.y;
          ny = c.x;
          nz = c.y;
          W = d.x;
        } else {
          W = b.y;
        }
      } else if (q < pe) {
        if (SURF) {
          const double *p = pts + 8 * q;
          xi = __ldg(p);
          eta = __ldg(p + 1);
          zeta = __ldg(p + 2);
          nx = __ldg(p + 3);
          ny = __ldg(p + 4);
          nz = __ldg(p + 5);
          W = __ldg(p + 6);
        } else {
          const double2 a = __ldg(reinterpret_cast<const double2 *>(pts + 4 * q));
          const double2 b = __ldg(reinterpret_cast<const double2 *>(pts + 4 * q) + 1);
          xi = a.x;
          eta = a.y;
          zeta = b.x;
          W = b.y;
        }
      }
      double vx[N], dvx[N], vy[N], dvy[N], vz[N], dvz[N];
      basis_vd<N>(R, xi, vx, dvx);
      basis_vd<N>(R, eta, vy, dvy);
      basis_vd<N>(R, zeta, vz, dvz);
      // this thread's z-planes c = part * CPS + cc (cc < CPS, c < N)
      double vzl[CPS], dvzl[CPS];
#pragma unroll
      for (int cc = 0; cc < CPS; ++cc) {
        double a = 0.0, b = 0.0;
#pragma unroll
        for (int k = 0; k < SPL; ++k)
          if (k * CPS + cc < N && part == k) {
            a = vz[k * CPS + cc];
            b = dvz[k * CPS + cc];
          }
        vzl[cc] = a;
        dvzl[cc] = b;
      }
      double u0 = 0.0, ux = 0.0, uy = 0.0, uz = 0.0;
#pragma unroll
      for (int cc = 0; cc < CPS; ++cc) {
        const int c = part * CPS + cc;
        if ((N % SPL) != 0 && c >= N) break;
        double t00 = 0.0, t10 = 0.0, t01 = 0.0;
#pragma unroll
        for (int b = 0; b < N; ++b) {
          double s0 = 0.0, s1 = 0.0;
          const double *row = U + c * Blk<N>::PS + b * Blk<N>::P;
#pragma unroll
          for (int a = 0; a < N; ++a) {
            const double uu = row[a];
            s0 = fma(vx[a], uu, s0);
            s1 = fma(dvx[a], uu, s1);
          }
          t00 = fma(vy[b], s0, t00);
          t10 = fma(dvy[b], s0, t10);
          t01 = fma(vy[b], s1, t01);
        }
        u0 = fma(vzl[cc], t00, u0);
        uz = fma(dvzl[cc], t00, uz);
        uy = fma(vzl[cc], t10, uy);
        ux = fma(vzl[cc], t01, ux);
      }
      // sum the SPL partial evaluations (xor butterfly: every thread of the point
      // gets the same bits)
#pragma unroll
      for (int o = 1; o < SPL; o <<= 1) {
        u0 += __shfl_xor_sync(0xffffffffu, u0, o);
        ux += __shfl_xor_sync(0xffffffffu, ux, o);
        uy += __shfl_xor_sync(0xffffffffu, uy, o);
        uz += __shfl_xor_sync(0xffffffffu, uz, o);
      }
      // B: quadrature-point operation
      double c0v, c1, c2, c3;
      if (SURF) {
        const double un = (nx * ux + ny * uy + nz * uz) * ih;  // physical normal derivative
        c0v = W * (kp.tau * u0 - un);
        const double g = -W * u0 * ih;
        c1 = g * nx;
        c2 = g * ny;
        c3 = g * nz;
      } else {
        c0v = 0.0;
        const double sw = W * ih2;
        c1 = sw * ux;
        c2 = sw * uy;
        c3 = sw * uz;
      }
      // I (z and y stages per point, this thread's z-planes); the x stage is the
      // row integration below
      double *row = PS + pq * ROW;
#pragma unroll
      for (int cc = 0; cc < CPS; ++cc) {
        const int c = part * CPS + cc;
        if ((N % SPL) != 0 && c >= N) break;
        const double T0 = fma(c0v, vzl[cc], c3 * dvzl[cc]), T1 = c2 * vzl[cc], T2 = c1 * vzl[cc];
#pragma unroll
        for (int b = 0; b < N; ++b) {
          row[b + N * c] = fma(vy[b], T0, dvy[b] * T1);
          row[NN + b + N * c] = vy[b] * T2;
        }
      }
      if (part == 0) {
#pragma unroll
        for (int a = 0; a < N; ++a) {
          row[2 * NN + a] = vx[a];
          row[2 * NN + N + a] = dvx[a];
        }
      }
    }
    __syncthreads();
    const int cnt = (int)((pe - c0) < C::CHUNK ? (pe - c0) : C::CHUNK);
    if constexpr (!C::ROWINT) {
      // one thread per DoF (a, bc): acc[k][0] over all the chunk's points
#pragma unroll
      for (int k = 0; k < C::KPT; ++k) {
        const int l = tid + k * C::THREADS;
        if (l < N * NN) {
          const int a = l % N, bc = l / N;
          double sacc = acc[0][k];
          for (int qq = 0; qq < cnt; ++qq) {
            const double *row = PS + qq * ROW;
            sacc = fma(row[2 * NN + a], row[bc], sacc);
            sacc = fma(row[2 * NN + N + a], row[NN + bc], sacc);
          }
          acc[0][k] = sacc;
        }
      }
    } else if (grp < G) {
      // x stage: acc[r][a] += vx[a] S0[bc_r] + dvx[a] S1[bc_r] over this group's points
      for (int qq = grp; qq < cnt; qq += G) {
        const double *row = PS + qq * ROW;
        double xv[N], xd[N];
#pragma unroll
        for (int a = 0; a < N; ++a) {
          xv[a] = row[2 * NN + a];
          xd[a] = row[2 * NN + N + a];
        }
#pragma unroll
        for (int r = 0; r < RPT; ++r) {
          const int bc = rl * RPT + r;
          if (bc < NN) {
            const double s0 = row[bc], s1 = row[NN + bc];
#pragma unroll
            for (int a = 0; a < N; ++a) acc[r][a] = fma(xv[a], s0, fma(xd[a], s1, acc[r][a]));
          }
        }
      }
    }
    __syncthreads();
  }
}

// Volume points in LINES (dimension-reduction quadrature: the n Gauss points of a
// line of the height axis ax share the two base coordinates; the cell's points are
// stored line by line).  Per line (one thread): the base-plane contraction
//   P_i = sum_jk u l1_j l2_k,  Q1_i = sum u l1'_j l2_k,  Q2_i = sum u l1_j l2'_k
// once, then per point only n-term sums for u, grad u and the test coefficients
//   R0_i += c_ax la'_i,  R1_i += c_B1 la_i,  R2_i += c_B2 la_i
// (i along ax, j along B1 < B2, k along B2; the paper's partial-sum reuse, P:874-878,
// extended across the points of a line).  The line's contribution
//   R0_i l1_j l2_k + R1_i l1'_j l2_k + R2_i l1_j l2'_k
// is written as rows in the x-stage form  X0[a] S0[bc] + X1[a] S1[bc] (+ X2[a] S2[bc]
// when the lines run along x), so the row-blocked integration runs once per LINE.
template <int N, int AX, int H>
__device__ __forceinline__ void line_base(const double *U, int i0, const double (&v1)[N], const double (&d1)[N],
                                          const double (&v2)[N], const double (&d2)[N], double (&Pp)[H],
                                          double (&Q1)[H], double (&Q2)[H]) {
  using B = Blk<N>;
  constexpr int LBU = CUT_LB_UNROLL > 0 ? CUT_LB_UNROLL : (N <= 7 ? H : 1);
#pragma unroll LBU
  for (int ii = 0; ii < H; ++ii) {
    const int i = i0 + ii < N ? i0 + ii : N - 1;  // (odd n: the upper half's last slot is a dummy)
    double p = 0.0, q1 = 0.0, q2 = 0.0;
#pragma unroll
    for (int k = 0; k < N; ++k) {
      double s0 = 0.0, s1 = 0.0;
#pragma unroll
      for (int j = 0; j < N; ++j) {
        const double uu = AX == 0 ? U[B::at(i, j, k)] : (AX == 1 ? U[B::at(j, i, k)] : U[B::at(j, k, i)]);
        s0 = fma(v1[j], uu, s0);
        s1 = fma(d1[j], uu, s1);
      }
      p = fma(v2[k], s0, p);
      q1 = fma(v2[k], s1, q1);
      q2 = fma(d2[k], s0, q2);
    }
    Pp[ii] = p;
    Q1[ii] = q1;
    Q2[ii] = q2;
  }
}

// Lines are split over a thread pair along i (the line axis): each thread holds
// the base sums and test coefficients of its half of the i range; the n-term sums
// over i of a point are combined by one __shfl_xor (same bits on both threads).
template <int N>
__device__ __forceinline__ void line_chunks(const double *__restrict__ pts, int64_t pb, int64_t pe, int ax,
                                            const double *U, double *PS, double (&acc)[CutCfg<N>::RPT][N],
                                            const KParams &kp, const RefTab &R, const double *__restrict__ lsrf) {
  using C = CutCfg<N>;
  constexpr int NN = C::NN, RPT = C::RPT, TG = C::TG, G = C::G;
  constexpr int RL = C::LRL, CL = C::LCL;  // row: S0 S1 S2 X0 X1 X2; lines per chunk
  constexpr int H = (N + 1) / 2;  // i values per thread
  double *LB = PS - C::OFF_PS + C::OFF_LB;  // the chunk's line points (CL N rows of 4 doubles)
  double *LS = LB + C::LBUF;                 // the chunk's line interface records (CL rows of 6)
  const int tid = threadIdx.x, grp = tid / TG, rl = tid % TG;
  const int lq = tid >> 1, part = tid & 1, i0 = part * H;
  const double ih = kp.ih, ih2 = kp.ih2;
  const int64_t nl = (pe - pb) / N;
  for (int64_t l0 = 0; l0 < nl; l0 += CL) {
    const int cnt = (int)((nl - l0) < CL ? (nl - l0) : CL);
    {  // stage the chunk's points (16-byte pieces; the previous chunk is done with LB)
      const double *src = pts + 4 * (pb + l0 * N);
      for (int e = tid; e < cnt * N * 2; e += C::THREADS) cp_async16(LB + 2 * e, src + 2 * e);
      if (lsrf)  // the lines' interface records [t, W, n_ax, n_B1, n_B2, 0] (LS: CL rows of 6)
        for (int e = tid; e < cnt * 3; e += C::THREADS) cp_async16(LS + 2 * e, lsrf + 6 * l0 + 2 * e);
      cp_async_commit();
      cp_async_wait<0>();
      __syncthreads();
    }
    {  // every thread takes part in the shuffles (idle pairs work on a dummy line)
      const bool live = lq < cnt;
      const double *p = LB + 4 * ((live ? lq : 0) * N);
      const double b1 = ax == 0 ? p[1] : p[0], b2 = ax == 2 ? p[1] : p[2];
      double Pp[H], Q1[H], Q2[H];
      {  // the base bases are recomputed for the rows below (not kept live over the points)
        double v1[N], d1[N], v2[N], d2[N];
        basis_vd<N>(R, b1, v1, d1);
        basis_vd<N>(R, b2, v2, d2);
        if (ax == 0) line_base<N, 0, H>(U, i0, v1, d1, v2, d2, Pp, Q1, Q2);
        else if (ax == 1) line_base<N, 1, H>(U, i0, v1, d1, v2, d2, Pp, Q1, Q2);
        else line_base<N, 2, H>(U, i0, v1, d1, v2, d2, Pp, Q1, Q2);
      }
      double R0[H], R1[H], R2[H];
#pragma unroll
      for (int ii = 0; ii < H; ++ii) R0[ii] = R1[ii] = R2[ii] = 0.0;
#pragma unroll 1
      for (int t = 0; t < N; ++t) {
        const double tc = p[4 * t + ax], W = live ? p[4 * t + 3] : 0.0;
        double vh[H], dh[H];  // this thread's half (i0 + ii), dummy slot zero
        basis_vd_half<N, H>(R, tc, part, vh, dh);
        double uA = 0.0, uB1 = 0.0, uB2 = 0.0;
#pragma unroll
        for (int ii = 0; ii < H; ++ii) {
          uA = fma(dh[ii], Pp[ii], uA);
          uB1 = fma(vh[ii], Q1[ii], uB1);
          uB2 = fma(vh[ii], Q2[ii], uB2);
        }
        uA += __shfl_xor_sync(0xffffffffu, uA, 1);
        uB1 += __shfl_xor_sync(0xffffffffu, uB1, 1);
        uB2 += __shfl_xor_sync(0xffffffffu, uB2, 1);
        const double sw = W * ih2;
        const double cA = sw * uA, cB1 = sw * uB1, cB2 = sw * uB2;
#pragma unroll
        for (int ii = 0; ii < H; ++ii) {
          R0[ii] = fma(cA, dh[ii], R0[ii]);
          R1[ii] = fma(cB1, vh[ii], R1[ii]);
          R2[ii] = fma(cB2, vh[ii], R2[ii]);
        }
      }
      if (lsrf) {
        // the line's interface (Nitsche) point, if any; every pair runs this (W = 0 when
        // absent) so the shuffles stay convergent; value term folded into R0
        const double *y = LS + 6 * (live ? lq : 0);
        const double tc = y[0], W = live ? y[1] : 0.0;
        const double nA = y[2], nB1 = y[3], nB2 = y[4];
        double vh[H], dh[H];
        basis_vd_half<N, H>(R, tc, part, vh, dh);
        double u0 = 0.0, uA = 0.0, uB1 = 0.0, uB2 = 0.0;
#pragma unroll
        for (int ii = 0; ii < H; ++ii) {
          u0 = fma(vh[ii], Pp[ii], u0);
          uA = fma(dh[ii], Pp[ii], uA);
          uB1 = fma(vh[ii], Q1[ii], uB1);
          uB2 = fma(vh[ii], Q2[ii], uB2);
        }
        u0 += __shfl_xor_sync(0xffffffffu, u0, 1);
        uA += __shfl_xor_sync(0xffffffffu, uA, 1);
        uB1 += __shfl_xor_sync(0xffffffffu, uB1, 1);
        uB2 += __shfl_xor_sync(0xffffffffu, uB2, 1);
        const double un = (nA * uA + nB1 * uB1 + nB2 * uB2) * ih;  // physical normal derivative
        const double c0 = W * (kp.tau * u0 - un), g = -W * u0 * ih;
        const double cA = g * nA, cB1 = g * nB1, cB2 = g * nB2;
#pragma unroll
        for (int ii = 0; ii < H; ++ii) {
          R0[ii] = fma(cA, dh[ii], fma(c0, vh[ii], R0[ii]));
          R1[ii] = fma(cB1, vh[ii], R1[ii]);
          R2[ii] = fma(cB2, vh[ii], R2[ii]);
        }
      }
      if (live) {
        double v1[N], d1[N], v2[N], d2[N];
        basis_vd<N>(R, b1, v1, d1);
        basis_vd<N>(R, b2, v2, d2);
        double *row = PS + lq * RL;
        if (ax == 0) {  // i = a: X = R (own a), S[b + N c] = l1_b l2_c, l1'_b l2_c, l1_b l2'_c (c parity)
#pragma unroll
          for (int c = 0; c < N; ++c) {
            if ((c & 1) != part) continue;
#pragma unroll
            for (int b = 0; b < N; ++b) {
              row[b + N * c] = v1[b] * v2[c];
              row[NN + b + N * c] = d1[b] * v2[c];
              row[2 * NN + b + N * c] = v1[b] * d2[c];
            }
          }
#pragma unroll
          for (int ii = 0; ii < H; ++ii) {
            const int a = i0 + ii;
            if (a < N) {
              row[3 * NN + a] = R0[ii];
              row[3 * NN + N + a] = R1[ii];
              row[3 * NN + 2 * N + a] = R2[ii];
            }
          }
        } else {  // j = a: X0 = l1, X1 = l1'; own i = b (ax = y) or c (ax = z)
#pragma unroll
          for (int ii = 0; ii < H; ++ii) {
            const int i = i0 + ii;
            if (i >= N) continue;
#pragma unroll
            for (int k = 0; k < N; ++k) {
              const int bc = ax == 1 ? i + N * k : k + N * i;
              row[bc] = fma(R0[ii], v2[k], R2[ii] * d2[k]);
              row[NN + bc] = R1[ii] * v2[k];
            }
          }
          if (part == 0) {
#pragma unroll
            for (int a = 0; a < N; ++a) {
              row[3 * NN + a] = v1[a];
              row[3 * NN + N + a] = d1[a];
            }
          }
        }
      }
    }
    __syncthreads();
    if (grp < G) {
      for (int qq = grp; qq < cnt; qq += G) {
        const double *row = PS + qq * RL;
        double x0[N], x1[N];
#pragma unroll
        for (int a = 0; a < N; ++a) {
          x0[a] = row[3 * NN + a];
          x1[a] = row[3 * NN + N + a];
        }
        if (ax == 0) {
          double x2[N];
#pragma unroll
          for (int a = 0; a < N; ++a) x2[a] = row[3 * NN + 2 * N + a];
#pragma unroll
          for (int r = 0; r < RPT; ++r) {
            const int bc = rl * RPT + r;
            if (bc < NN) {
              const double s0 = row[bc], s1 = row[NN + bc], s2 = row[2 * NN + bc];
#pragma unroll
              for (int a = 0; a < N; ++a) acc[r][a] = fma(x0[a], s0, fma(x1[a], s1, fma(x2[a], s2, acc[r][a])));
            }
          }
        } else {
#pragma unroll
          for (int r = 0; r < RPT; ++r) {
            const int bc = rl * RPT + r;
            if (bc < NN) {
              const double s0 = row[bc], s1 = row[NN + bc];
#pragma unroll
              for (int a = 0; a < N; ++a) acc[r][a] = fma(x0[a], s0, fma(x1[a], s1, acc[r][a]));
            }
          }
        }
      }
    }
    __syncthreads();
  }
}

template <int N>
__global__ void __launch_bounds__(CutCfg<N>::THREADS, CutCfg<N>::MINB) k_cut(const double *__restrict__ u, double *__restrict__ v,
                                             const CDesc *__restrict__ desc, int ncut,
                                             const double *__restrict__ vol_pts,
                                             const int64_t *__restrict__ vol_ptr,
                                             const double *__restrict__ srf_pts,
                                             const int64_t *__restrict__ srf_ptr,
                                             const double *__restrict__ sf_pts,
                                             const int64_t *__restrict__ sf_ptr, KParams kp, FaceTab ft,
                                             TileTab<N> tt, const double *__restrict__ line_srf) {
  using B = Blk<N>;
  using C = CutCfg<N>;
  constexpr int NN = B::NN, N3 = B::N3, SZ = B::SZ, TH = C::THREADS;
  const RefTab &R = c_ref[N - 2];
  extern __shared__ double smem[];
  double *U = smem, *T = smem + SZ, *Rb = smem + 2 * SZ, *NBs = smem + 3 * SZ;
  double *JA = smem + (3 + C::NBN) * SZ, *JB = JA + NN, *FC1 = JB + NN, *FC2 = FC1 + NN;
  double *PS = FC2 + NN;
  const int tid = threadIdx.x;
  const CDesc dsc = desc[blockIdx.x];
  auto face_on = [&](int f, bool &gp, bool &ss, bool &sc) {
    gp = ((dsc.flags >> f) & 1u) && (kp.mask & TERM_GP);
    ss = ((dsc.flags >> (6 + f)) & 1u) && (kp.mask & TERM_SIPG);
    sc = ((dsc.flags >> (12 + f)) & 1u) && (kp.mask & TERM_SIPG);
    return dsc.nb[f] >= 0 && (gp || ss || sc);
  };
  if constexpr (C::PREF) {
    // the neighbour blocks of every face with work, in flight during the point phases
    for (int f = 0; f < 6; ++f) {
      bool gp, ss, sc;
      if (!face_on(f, gp, ss, sc)) continue;
      const double *nbp = u + (size_t)dsc.nb[f] * N3;
      for (int l = tid; l < N3; l += TH) cp_async8(NBs + f * SZ + B::pad(l), nbp + l);
    }
    cp_async_commit();
  }
  {
    const double *ub = u + (size_t)dsc.blk * N3;
    for (int l = tid; l < N3; l += TH) U[B::pad(l)] = __ldg(ub + l);
  }
  __syncthreads();
  double acc[C::RPT][N];
#pragma unroll
  for (int r = 0; r < C::RPT; ++r)
#pragma unroll
    for (int a = 0; a < N; ++a) acc[r][a] = 0.0;
  if (kp.mask & TERM_CELL)
  {
    if constexpr (C::ROWINT) {
      if ((dsc.flags >> 26) & 1u)  // volume points in lines along axis (flags >> 24) & 3
        line_chunks<N>(vol_pts, vol_ptr[dsc.cut], vol_ptr[dsc.cut + 1], (int)((dsc.flags >> 24) & 3u), U, PS, acc,
                       kp, R, ((dsc.flags >> 27) & 1u) && (kp.mask & TERM_NITSCHE) ? line_srf + 6 * (int64_t)dsc.pad : nullptr);
      else
        point_chunks<N, false>(vol_pts, vol_ptr[dsc.cut], vol_ptr[dsc.cut + 1], U, PS, acc, kp, R);
    } else {
      point_chunks<N, false>(vol_pts, vol_ptr[dsc.cut], vol_ptr[dsc.cut + 1], U, PS, acc, kp, R);
    }
  }
  if ((kp.mask & TERM_NITSCHE) && !(C::ROWINT && ((dsc.flags >> 27) & 1u) && (kp.mask & TERM_CELL)))
    point_chunks<N, true>(srf_pts, srf_ptr[dsc.cut], srf_ptr[dsc.cut + 1], U, PS, acc, kp, R);
  if constexpr (!C::ROWINT) {
    static_assert(C::KPT <= N, "acc[0] holds the thread's DoFs");
#pragma unroll
    for (int k = 0; k < C::KPT; ++k) {
      const int l = tid + k * TH;
      if (l < N3) Rb[B::pad(l)] = acc[0][k];
    }
  } else {
    // sum the groups' partial rows (the chunk buffer is free now) into Rb
    static_assert(C::G * N3 <= C::CHUNK * C::ROW, "reduction buffer");
    const int grp = tid / C::TG, rl = tid % C::TG;
    if (grp < C::G) {
#pragma unroll
      for (int r = 0; r < C::RPT; ++r) {
        const int bc = rl * C::RPT + r;
        if (bc < NN)
#pragma unroll
          for (int a = 0; a < N; ++a) PS[grp * N3 + a + N * bc] = acc[r][a];
      }
    }
    __syncthreads();
    for (int l = tid; l < N3; l += TH) {
      double s = 0.0;
      for (int g = 0; g < C::G; ++g) s += PS[g * N3 + l];
      Rb[B::pad(l)] = s;
    }
  }
  __syncthreads();

  const double h = kp.h, h2 = h * h;
  if constexpr (C::PREF) {
    cp_async_wait<0>();
    __syncthreads();
    // structured faces (ghost penalty, full-face SIPG) in w-space (as k_cutp): per
    // (axis, line) item both faces of the axis through M^{-1}-premultiplied line
    // operators (the hi face in the line-reversed frame with the lo-face
    // coefficients), one buffer per axis; then v += (M (x) M (x) M) sum_axes w
    uint32_t gmk = 0, smk = 0;
#pragma unroll
    for (int f = 0; f < 6 && C::WFACE; ++f) {
      bool gp, ss, sc;
      if (!face_on(f, gp, ss, sc)) continue;
      gmk |= (uint32_t)gp << f;
      smk |= (uint32_t)ss << f;
    }
    if (gmk | smk) {
      double *WS = PS;  // [3][SZ] (the point rows are consumed)
      for (int it = tid; it < 3 * NN; it += TH) {
        const int D = it / NN, t = it - D * NN;
        int b0, st;
        B::line(D, t, b0, st);
        double uo[N], w[N];
#pragma unroll
        for (int m = 0; m < N; ++m) {
          uo[m] = U[b0 + m * st];
          w[m] = 0.0;
        }
#pragma unroll
        for (int sd = 0; sd < 2; ++sd) {
          const int f = 2 * D + sd;
          const bool g = (gmk >> f) & 1u, sp = (smk >> f) & 1u;
          if (!(g || sp)) continue;
          const double *NBf = NBs + f * SZ;
          double uu[N], un[N], out[N];
#pragma unroll
          for (int m = 0; m < N; ++m) {
            const int pm = sd ? N - 1 - m : m;
            uu[m] = uo[pm];
            un[m] = NBf[b0 + pm * st];
            out[m] = 0.0;
          }
          if (g) {
#pragma unroll
            for (int m = 0; m < N; ++m) {
              double x = 0.0;
#pragma unroll
              for (int a = 0; a < N; ++a) x = fma(tt.Goo[m * N + a], uu[a], fma(tt.Gon[m * N + a], un[a], x));
              out[m] = x;
            }
          }
          if (sp) {
            double A0 = 0.0, A1 = 0.0;
#pragma unroll
            for (int m = 0; m < N; ++m) {
              A0 = fma(tt.d0[m], uu[m], A0);
              A1 = fma(-tt.d0[N - 1 - m], un[m], A1);
            }
            const double J = uu[0] - un[N - 1], A = A0 + A1;
#pragma unroll
            for (int m = 0; m < N; ++m) out[m] = fma(tt.cJ[m], J, fma(tt.cA[m], A, out[m]));
          }
#pragma unroll
          for (int m = 0; m < N; ++m) w[sd ? N - 1 - m : m] += out[m];
        }
#pragma unroll
        for (int m = 0; m < N; ++m) WS[D * SZ + b0 + m * st] = w[m];
      }
      __syncthreads();
#pragma unroll
      for (int D = 0; D < 3; ++D) {
        for (int t = tid; t < NN; t += TH) {
          int b0, st;
          B::line(D, t, b0, st);
          double x[N];
#pragma unroll
          for (int m = 0; m < N; ++m) {
            const int l = b0 + m * st;
            x[m] = D == 0 ? (WS[l] + WS[SZ + l]) + WS[2 * SZ + l] : WS[l];
          }
#pragma unroll
          for (int i = 0; i < N; ++i) {
            double y = 0.0;
#pragma unroll
            for (int j = 0; j < N; ++j) y = fma(tt.M[csym<N>(i * N + j)], x[j], y);
            if (D < 2) WS[b0 + i * st] = y;
            else Rb[b0 + i * st] += y;
          }
        }
        __syncthreads();
      }
    }
  }
  if constexpr (C::BFACE) {
    // cut faces (eq:unstructured_face P:491-496), all of the cell's faces in one pass:
    // traces of every cut face, then the faces' points as one concatenated stream in
    // chunks, each (face, in-face node) item summed by one thread, then one pass over
    // the DoFs adds every face's line coefficients and writes v (no per-face barriers)
    uint32_t scm = 0;
#pragma unroll
    for (int f = 0; f < 6; ++f) {
      bool gp, ss, sc;
      if (face_on(f, gp, ss, sc) && sc) scm |= 1u << f;
    }
    double *vb = v + (size_t)dsc.blk * N3;
    if (!scm) {
      for (int l = tid; l < N3; l += TH) vb[l] = Rb[B::pad(l)];
      return;
    }
    constexpr int FR = C::FROW, FCH = TH;
    double *JAa = PS, *JBa = PS + 6 * NN, *F1a = PS + 12 * NN, *F2a = PS + 18 * NN, *RW = PS + 24 * NN;
    long long *PBs = reinterpret_cast<long long *>(RW + FCH * FR);  // [6] first point, [7] prefix offsets
    static_assert(24 * NN + FCH * FR + 13 <= C::CHUNK * C::ROW, "cut-face buffers fit the point rows");
    const int nsc = __popc(scm);
    auto kth = [&](int k) {  // the k-th cut face (k < nsc)
      uint32_t m = scm;
      for (int i = 0; i < k; ++i) m &= m - 1;
      return __ffs(m) - 1;
    };
    if (tid == 0) {  // the faces' first points and prefix offsets in the concatenation
      long long cu = 0;
#pragma unroll
      for (int f = 0; f < 6; ++f) {
        long long b = 0, c = 0;
        if ((scm >> f) & 1u) {
          b = __ldg(sf_ptr + dsc.sf[f]);
          c = __ldg(sf_ptr + dsc.sf[f] + 1) - b;
        }
        PBs[f] = b;
        PBs[6 + f] = cu;
        cu += c;
      }
      PBs[12] = cu;
    }
    for (int it = tid; it < nsc * NN; it += TH) {
      const int k = it / NN, t = it - k * NN, f = kth(k);
      const int dd = f >> 1, side = f & 1;
      const double *NBf = NBs + f * SZ;
      const double *dow = side ? R.d1 : R.d0, *dnb = side ? R.d0 : R.d1;
      int b0, st;
      B::line(dd, t, b0, st);
      double A = 0.0;
#pragma unroll
      for (int m = 0; m < N; ++m) A = fma(dow[m], U[b0 + m * st], fma(dnb[m], NBf[b0 + m * st], A));
      JAa[f * NN + t] = side ? U[b0 + (N - 1) * st] - NBf[b0] : U[b0] - NBf[b0 + (N - 1) * st];
      JBa[f * NN + t] = A;
      F1a[f * NN + t] = 0.0;
      F2a[f * NN + t] = 0.0;
    }
    __syncthreads();
    const long long *cum = PBs + 6;
    const long long Q = cum[6];
    for (long long c0 = 0; c0 < Q; c0 += FCH) {
      {
        const long long g = c0 + tid;
        if (g < Q) {
          int f = 0;
#pragma unroll
          for (int i = 1; i < 6; ++i) f += g >= cum[i];
          const long long q = PBs[f] + (g - cum[f]);
          const double s = __ldg(sf_pts + 4 * q), tq = __ldg(sf_pts + 4 * q + 1), W = __ldg(sf_pts + 4 * q + 2);
          const double sg = (f & 1) ? 1.0 : -1.0;
          double ls[N], lt[N];
          basis_v<N>(R, s, ls);
          basis_v<N>(R, tq, lt);
          const double *JA = JAa + f * NN, *JB = JBa + f * NN;
          double J0 = 0.0, A = 0.0;
#pragma unroll
          for (int j = 0; j < N; ++j) {
            double r0 = 0.0, r1 = 0.0;
#pragma unroll
            for (int i = 0; i < N; ++i) {
              r0 = fma(ls[i], JA[i + N * j], r0);
              r1 = fma(ls[i], JB[i + N * j], r1);
            }
            J0 = fma(lt[j], r0, J0);
            A = fma(lt[j], r1, A);
          }
          double *row = RW + tid * FR;
#pragma unroll
          for (int i = 0; i < N; ++i) {
            row[i] = ls[i];
            row[N + i] = lt[i];
          }
          row[2 * N] = W * (kp.sigma * J0 - sg * A * kp.i2h);
          row[2 * N + 1] = -W * sg * J0 * kp.i2h;
        }
      }
      __syncthreads();
      for (int it = tid; it < nsc * NN; it += TH) {
        const int k = it / NN, ij = it - k * NN, f = kth(k);
        const int i = ij % N, j = ij / N;
        const long long lo = cum[f] > c0 ? cum[f] : c0, hi = cum[f + 1] < c0 + FCH ? cum[f + 1] : c0 + FCH;
        double f1 = F1a[f * NN + ij], f2 = F2a[f * NN + ij];
        for (int r = (int)(lo - c0); r < (int)(hi - c0); ++r) {
          const double *row = RW + r * FR;
          const double psi = row[i] * row[N + j];
          f1 = fma(psi, row[2 * N], f1);
          f2 = fma(psi, row[2 * N + 1], f2);
        }
        F1a[f * NN + ij] = f1;
        F2a[f * NN + ij] = f2;
      }
      __syncthreads();
    }
    // v = Rb + every cut face's line coefficients: DoF (a, b, c) lies on line t of
    // axis dd at position m (B::line's numbering: t = (b, c), (a, c), (a, b))
    for (int l = tid; l < N3; l += TH) {
      const int a = l % N, bb = (l / N) % N, c = l / NN;
      double r = Rb[B::pad(l)];
#pragma unroll
      for (int f = 0; f < 6; ++f) {
        if (!((scm >> f) & 1u)) continue;
        const int dd = f >> 1, side = f & 1;
        const int m = dd == 0 ? a : (dd == 1 ? bb : c);
        const int t = dd == 0 ? bb + N * c : (dd == 1 ? a + N * c : a + N * bb);
        const double dw = side ? R.d1[m] : R.d0[m];
        r = fma(dw, F2a[f * NN + t], r);
        if (m == (side ? N - 1 : 0)) r += F1a[f * NN + t];
      }
      vb[l] = r;
    }
    return;
  }
  if constexpr (!C::BFACE)  // face by face (structured and cut faces, or cut faces only)
  for (int f = 0; f < 6; ++f) {
    bool gp, ss, sc;
    if (!face_on(f, gp, ss, sc)) continue;
    if (C::WFACE && !sc) continue;  // structured parts done above
    double *NB = C::PREF ? NBs + f * SZ : NBs;
    if constexpr (!C::PREF) {
      const double *nbp = u + (size_t)dsc.nb[f] * N3;
      for (int l = tid; l < N3; l += TH) NB[B::pad(l)] = __ldg(nbp + l);
      __syncthreads();
    }
    const int dd = f >> 1, side = f & 1;
    const int fo = side ? N - 1 : 0, fn = side ? 0 : N - 1;
    const double sg = side ? 1.0 : -1.0;
    const double *dow = side ? R.d1 : R.d0;
    const double *dnb = side ? R.d0 : R.d1;
    const double *Goo = ft.Goo[side ? 0 : 1];
    const double *Gon = ft.Gon[side ? 0 : 1];
    const bool structured = !C::WFACE && (gp || ss);
    for (int t = tid; t < NN; t += TH) {
      int b0, st;
      B::line(dd, t, b0, st);
      double uo[N], un[N];
#pragma unroll
      for (int m = 0; m < N; ++m) {
        uo[m] = U[b0 + m * st];
        un[m] = NB[b0 + m * st];
      }
      const double J0 = uo[fo] - un[fn];
      double A = 0.0;
#pragma unroll
      for (int m = 0; m < N; ++m) A = fma(dow[m], uo[m], fma(dnb[m], un[m], A));
      JA[t] = J0;
      JB[t] = A;
      FC1[t] = 0.0;
      FC2[t] = 0.0;
      if (structured) {
        const double F1 = ss ? h2 * (kp.sigma * J0 - sg * A * kp.i2h) : 0.0;
        const double F2 = ss ? -0.5 * h * sg * J0 : 0.0;
#pragma unroll
        for (int m = 0; m < N; ++m) {
          double F = 0.0;
          if (gp) {
#pragma unroll
            for (int a = 0; a < N; ++a) F = fma(Goo[m * N + a], uo[a], fma(-Gon[m * N + a], un[a], F));
          }
          F = fma(dow[m], F2, F);
          if (m == fo) F += F1;
          T[b0 + m * st] = F;
        }
      }
    }
    __syncthreads();
    if (structured) {
      const int e1 = (dd == 0) ? 1 : 0, e2 = (dd == 2) ? 1 : 2;
      for (int t = tid; t < NN; t += TH) {
        int b0, st;
        B::line(e1, t, b0, st);
        sweep_line<N, 0>(T, T, b0, st, R.M, 1.0);
      }
      __syncthreads();
      for (int t = tid; t < NN; t += TH) {
        int b0, st;
        B::line(e2, t, b0, st);
        sweep_line<N, 0>(T, T, b0, st, R.M, 1.0);
      }
      __syncthreads();
    }
    if (sc) {
      // unstructured in-face quadrature (eq:unstructured_face P:491-496)
      const int64_t pb = sf_ptr[dsc.sf[f]], pe = sf_ptr[dsc.sf[f] + 1];
      constexpr int FR = C::FROW;
      constexpr int FCH = (C::CHUNK * C::ROW) / FR < TH ? (C::CHUNK * C::ROW) / FR : TH;
      constexpr int FG = TH / NN >= 1 ? TH / NN : 1;  // thread groups over the points
      static_assert(2 * FG * NN <= C::CHUNK * C::ROW, "partial sums fit the point rows");
      double f1 = 0.0, f2 = 0.0;
      for (int64_t c0 = pb; c0 < pe; c0 += FCH) {
        if (tid < FCH) {
          const int64_t q = c0 + tid;
          double s = 0.5, tt = 0.5, W = 0.0;
          if (q < pe) {
            s = __ldg(sf_pts + 4 * q);
            tt = __ldg(sf_pts + 4 * q + 1);
            W = __ldg(sf_pts + 4 * q + 2);
          }
          double ls[N], lt[N];
          basis_v<N>(R, s, ls);
          basis_v<N>(R, tt, lt);
          double J0 = 0.0, A = 0.0;
#pragma unroll
          for (int j = 0; j < N; ++j) {
            double r0 = 0.0, r1 = 0.0;
#pragma unroll
            for (int i = 0; i < N; ++i) {
              r0 = fma(ls[i], JA[i + N * j], r0);
              r1 = fma(ls[i], JB[i + N * j], r1);
            }
            J0 = fma(lt[j], r0, J0);
            A = fma(lt[j], r1, A);
          }
          double *row = PS + tid * FR;
#pragma unroll
          for (int i = 0; i < N; ++i) {
            row[i] = ls[i];
            row[N + i] = lt[i];
          }
          row[2 * N] = W * (kp.sigma * J0 - sg * A * kp.i2h);
          row[2 * N + 1] = -W * sg * J0 * kp.i2h;
        }
        __syncthreads();
        const int cnt = (int)((pe - c0) < FCH ? (pe - c0) : FCH);
        // FG groups of NN threads split the chunk's points (in-face node (i, j) per thread)
        if (tid < FG * NN) {
          const int fg = tid / NN, i = (tid % NN) % N, j = (tid % NN) / N;
          for (int qq = fg; qq < cnt; qq += FG) {
            const double *row = PS + qq * FR;
            const double psi = row[i] * row[N + j];
            f1 = fma(psi, row[2 * N], f1);
            f2 = fma(psi, row[2 * N + 1], f2);
          }
        }
        __syncthreads();
      }
      if constexpr (FG > 1) {  // the groups' partial sums, added in group order
        if (tid < FG * NN) {
          PS[2 * tid] = f1;
          PS[2 * tid + 1] = f2;
        }
        __syncthreads();
        if (tid < NN) {
#pragma unroll
          for (int g = 1; g < FG; ++g) {
            f1 += PS[2 * (g * NN + tid)];
            f2 += PS[2 * (g * NN + tid) + 1];
          }
        }
        __syncthreads();  // PS is the next face's point rows
      }
      if constexpr (C::WFACE) {
        // thread t accumulated line t's coefficients itself (NN <= THREADS): apply them
        // directly (no FC round trip; lines of one axis are disjoint)
        if (tid < NN) {
          int b0, st;
          B::line(dd, tid, b0, st);
#pragma unroll
          for (int m = 0; m < N; ++m) Rb[b0 + m * st] = fma(dow[m], f2, Rb[b0 + m * st]);
          Rb[b0 + fo * st] += f1;
        }
      } else {
        if (tid < NN) {
          FC1[tid] = f1;
          FC2[tid] = f2;
        }
        __syncthreads();
      }
    }
    if constexpr (!C::WFACE) {
      for (int t = tid; t < NN; t += TH) {
        int b0, st;
        B::line(dd, t, b0, st);
        if (structured) {
#pragma unroll
          for (int m = 0; m < N; ++m) Rb[b0 + m * st] += T[b0 + m * st];
        }
        if (sc) {
          const double fa = FC1[t], fb = FC2[t];
#pragma unroll
          for (int m = 0; m < N; ++m) Rb[b0 + m * st] = fma(dow[m], fb, Rb[b0 + m * st]);
          Rb[b0 + fo * st] += fa;
        }
      }
    }
    // (w-space path: the next face's Rb updates come after its own trace barrier)
    if constexpr (!C::WFACE) __syncthreads();
  }
  if constexpr (C::WFACE) __syncthreads();  // every Rb update done
  double *vb = v + (size_t)dsc.blk * N3;
  for (int l = tid; l < N3; l += TH) vb[l] = Rb[B::pad(l)];
}

// ------------------------------------------------------------ helpers
template <int V>
struct IC {
  static constexpr int value = V;
};
template <int I, int E, class Fn>
__device__ __forceinline__ void static_for(Fn &&fn) {
  if constexpr (I < E) {
    fn(IC<I>{});
    static_for<I + 1, E>(fn);
  }
}

#include "kernels_tile.cuh"
#include "kernels_cut.cuh"
