// Structured (uncut) cells in registers (included by kernels.cuh): k_tile2 (n = 4),
// k_uncw (n = 4: the cells next to cut cells; n = 5, 6, 8: all), k_cell (n = 2, 3).
//
// Why: the line-per-lane kernels sweep every 1-D line through shared memory,
// i.e. one shared-memory access per FMA; the FP64 pipe needs ~4 FMAs per
// 8-byte shared access to stay busy (64 DFMA vs 16 doubles per clock per SM),
// so they saturate shared memory at ~25% of the FP64 peak.  Here the sum
// factorisation runs entirely on registers; shared memory only supplies the
// own block once and each neighbour block once per face.
//
// Arithmetic (exactly the structured terms of Alg. 1, on a
// Cartesian cell; the (p+1)-point Gauss rule integrates every product below
// exactly, so this is algebraically identical to quadrature):
//   volume     h K1 (x) M (x) M + M (x) h K1 (x) M + M (x) M (x) h K1
//   SIPG face  h^2 (M (x) M)_in-face  (x)  rank-2 1-D trace operator
//   face GP    h^2 (M (x) M)_in-face  (x)  G_oo / G_on line operators   (BASELINE configs[0])
// Every term is (M (x) M (x) M) applied to a sum of 1-D line operators along
// one axis each, premultiplied by M^{-1} on that axis:
//   v = (M (x) M (x) M) w,  w = sum_d [ (M^{-1} h K1)_d u + face terms_d ],
// so a cell costs 3 "line-operator" sweeps + the face traces + 3 mass sweeps
// (6 n^4 FMAs + O(n^3) per face), all with warp-uniform coefficients from the
// kernel parameter block (constant-bank operands).
//
// Data movement: a warp owns a tile of <= 32 uncut cells (a 2x4x4 brick of the
// background grid, partial bricks merged; built on the host).  All blocks the
// tile touches (its cells, then the face-neighbour halo) are copied by TMA bulk
// copies (cp.async.bulk + mbarrier complete_tx, SASS UBLKCP) into padded
// shared-memory slots (stride chosen so 16-byte per-lane reads of 32 different
// slots are bank-conflict free), the result is written back into the cell's
// own slot and stored by a bulk shared->global copy.  Each v block is written
// once, no atomics.  Odd n (blocks not 16-byte multiples) uses coalesced
// LDG/STS staging instead of bulk copies.
#pragma once
#ifndef T2MINB
#define T2MINB 1
#endif
#ifndef T1MINB
#define T1MINB 1
#endif
#ifndef TILE8_SMAX
#define TILE8_SMAX 36  // slots of an 8-cell tile (a full 2x2x2 brick needs 32; merged partial bricks
                       // more; 32 measured: k_uncw<6> 3 CTAs/SM instead of 2, same time)
#endif
#ifndef UNCW4_TC
#define UNCW4_TC 8  // cells per k_uncw<4> tile (the cells next to cut cells at n = 4)
#endif
#ifndef UNCW_EO
#define UNCW_EO 1  // k_uncw (n >= 5): even-odd decomposition of the centro-symmetric L and M sweeps
#endif
#ifndef K2_FOLD
#define K2_FOLD 1  // k_tile2: folded volume + own-side SIPG operator (cells with six faces)
#endif
#ifndef K1_TC
#define K1_TC 32  // cells per k_tile2 tile (16 measured: structured 40 -> 42 us, apply 109 -> 150 us at C2)
#endif

// Tiles of TCELLS cells (a brick of the background grid) + their face-neighbour halo.
template <int N, int TCELLS>
struct TileCfgX {
  static constexpr int N3 = N * N * N;
  static constexpr bool BULK = CUTFEM_USE_BULK && (N3 * 8) % 16 == 0;  // 16-byte multiple blocks
  // slot stride (doubles): consecutive slots on different banks for 8- / 16-byte reads
  static constexpr int ST = N == 2 ? 10 : (N == 3 ? 27 : (N == 4 ? 66 : (BULK ? N3 + 2 : N3)));
  static constexpr int TC = TCELLS;  // cells per tile
  // slots per tile: the brick + its face halo (2x4x4: 32 + 64, 2x2x4: 16 + 40,
  // 2x2x2: 8 + 24, 1x2x2: 4 + 16)
  static constexpr int SMAX = TC == 32 ? (N <= 3 ? 128 : 100) : (TC == 16 ? 60 : (TC == 8 ? TILE8_SMAX : 20));
  static constexpr int SMEM = 16 + SMAX * ST * 8;
  static constexpr int BX = TC == 4 ? 1 : 2, BY = TC == 32 ? 4 : 2, BZ = (TC == 8 || TC == 4) ? 2 : 4;
};
template <int N>
struct TileCfg : TileCfgX<N, (N <= 4 ? 32 : (N == 5 ? 16 : (N == 6 ? 8 : 4)))> {};

// One warp-tile.  lane_nb[l] = {slot of faces 0..3 (bytes), slot of faces 4,5
// (bytes 0,1) | ghost-penalty face bits << 16}; slot 255 = no neighbour.  Lane l
// computes the cell in slot l (l < ncell).
template <int SMAX>
struct __align__(16) TileRec {
  int32_t nslot, ncell, pad0, pad1;
  uint32_t lane_nb[32][2];
  int32_t blk[SMAX];
};

// TileTab<N> (the per-handle line operators) and csym live in kernels.cuh.

// position m along axis D of line t (t = t0 + N t1 over the two other axes, ascending)
template <int N, int D>
__device__ __forceinline__ constexpr int lix(int t, int m) {
  return D == 0 ? (m + N * (t % N) + N * N * (t / N))
                : (D == 1 ? ((t % N) + N * m + N * N * (t / N)) : ((t % N) + N * (t / N) + N * N * m));
}

__device__ __forceinline__ void bulk_s2g(void *dst, const void *src, uint32_t bytes) {
  asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;\n" ::"l"(dst), "r"(smem_u32(src)),
               "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void bulk_commit() { asm volatile("cp.async.bulk.commit_group;\n" ::: "memory"); }
__device__ __forceinline__ void bulk_wait_read0() { asm volatile("cp.async.bulk.wait_group.read 0;\n" ::: "memory"); }
__device__ __forceinline__ void bulk_wait0() { asm volatile("cp.async.bulk.wait_group 0;\n" ::: "memory"); }

// SIPG contribution of face (D, S) to line t from the own line uo[] and the
// neighbour's line un[]; en = 1 (face present) or 0 (no face: un is a dummy).
template <int N, int D, int S, int W>
__device__ __forceinline__ void sipg_line(double (&w)[W], int t, const double (&uo)[N], const double (&un)[N],
                                          double en, const TileTab<N> &tt) {
  double A0 = 0.0, A1 = 0.0;
#pragma unroll
  for (int m = 0; m < N; ++m) {
    if (S == 0) {  // own l'(0), neighbour l'(1) = -l'_{n-1-m}(0)
      A0 = fma(tt.d0[m], uo[m], A0);
      A1 = fma(-tt.d0[N - 1 - m], un[m], A1);
    } else {       // own l'(1), neighbour l'(0)
      A0 = fma(-tt.d0[N - 1 - m], uo[m], A0);
      A1 = fma(tt.d0[m], un[m], A1);
    }
  }
  const double J = en * (S ? (uo[N - 1] - un[0]) : (uo[0] - un[N - 1]));
  const double A = en * (A0 + A1);
#pragma unroll
  for (int m = 0; m < N; ++m) {
    double &r = w[lix<N, D>(t, m)];
    if (S == 0) r = fma(tt.cJ[m], J, fma(tt.cA[m], A, r));
    else r = fma(tt.cJ[N - 1 - m], J, fma(-tt.cA[N - 1 - m], A, r));
  }
}

// ghost penalty of face S on a line: rows [R0, R1) of the line operator, output
// row m written to w[wi(m)]
template <int N, int S, int R0, int R1, class WI, int W>
__device__ __forceinline__ void gp_rows(double (&w)[W], WI wi, const double (&uo)[N], const double (&un)[N],
                                        double eg, const TileTab<N> &tt) {
#pragma unroll
  for (int m = R0; m < R1; ++m) {
    double r = 0.0;
#pragma unroll
    for (int a = 0; a < N; ++a) {
      const int k = S ? (N - 1 - m) * N + (N - 1 - a) : m * N + a;
      r = fma(tt.Goo[k], uo[a], fma(tt.Gon[k], un[a], r));
    }
    w[wi(m)] = fma(eg, r, w[wi(m)]);
  }
}

// Load line t along D of the block at B (shared memory), 16-byte words where
// the line is contiguous (D = 0, even N).
template <int N, int D>
__device__ __forceinline__ void ld_line(const double *B, int t, double (&a)[N]) {
  if constexpr ((N % 2) == 0 && D == 0) {
#pragma unroll
    for (int k = 0; k < N / 2; ++k) {
      const double2 x = *reinterpret_cast<const double2 *>(B + lix<N, 0>(t, 2 * k));
      a[2 * k] = x.x;
      a[2 * k + 1] = x.y;
    }
  } else {
#pragma unroll
    for (int m = 0; m < N; ++m) a[m] = B[lix<N, D>(t, m)];
  }
}
// Lines t and t+1 (t0 even, D != 0, even N) share 16-byte words.
template <int N, int D>
__device__ __forceinline__ void ld_pair(const double *B, int t, double (&a)[N], double (&b)[N]) {
#pragma unroll
  for (int m = 0; m < N; ++m) {
    const double2 x = *reinterpret_cast<const double2 *>(B + lix<N, D>(t, m));
    a[m] = x.x;
    b[m] = x.y;
  }
}

template <int N, int D, int W>
__device__ __forceinline__ void vol_line(double (&w)[W], int t, const double (&uo)[N], double ev,
                                         const TileTab<N> &tt) {
#pragma unroll
  for (int i = 0; i < N; ++i) {
    double r = 0.0;
#pragma unroll
    for (int j = 0; j < N; ++j) r = fma(tt.L[csym<N>(i * N + j)], uo[j], r);
    w[lix<N, D>(t, i)] = fma(ev, r, w[lix<N, D>(t, i)]);
  }
}

// ===================================================================== k_tile2
// k_tile2<N> (N = 4): the same arithmetic with TWO threads per cell, because a
// 64-double accumulator plus in-flight lines does not fit 255 registers.
// Thread (cell, h) owns the P = N/2 z-planes of its half, and works in the
// z-MIRRORED frame when h = 1 (z -> N-1-z): every operator is invariant under
// the reflection (GLL/Gauss symmetric, SIPG/GP reflection-invariant), so both
// halves run the same instructions with the same warp-uniform coefficients
// (rows 0..P-1 of the z-line operators), only the shared-memory addresses
// differ.  x/y terms are plane-local.  z terms: each thread evaluates its own
// (mirrored-lo) z face's traces [u], {d_z u} and swaps them with its partner
// (__shfl_xor 16; the partner's A changes sign with the frame), and the final
// z mass sweep swaps the partner's planes the same way.  Lanes l and l^16 are
// the two halves of cell 16*warp + (l & 15), so every 8-lane quarter of a warp
// reads 8 different slots (16-byte reads, slot stride 33 x 16 B: conflict free).
template <int N>
struct Tile2Cfg {
  // K1_TC cells per tile (32: a 2x4x4 brick, 2 warps; 16: 2x2x4, one warp), 2 threads per cell
  using T = TileCfgX<N, K1_TC>;
  static constexpr int P = N / 2, NN = N * N, N3 = N * NN, NP = NN * P;
  static constexpr int ST = T::ST, SMAX = T::SMAX;
  static constexpr int SMEM = T::SMEM;
  static constexpr int THREADS = 2 * K1_TC;
};

// x or y (D = 0, 1) terms of plane cc (pointers already at the plane)
template <int N, int D, int W>
__device__ __forceinline__ void axis_plane(double (&w)[W], const double *Up, const double *Lp, const double *Hp,
                                           int cc, double ev, double el, double eh, const TileTab<N> &tt) {
  if constexpr (D == 1 && (N % 2) == 0) {
#pragma unroll
    for (int q = 0; q < N; q += 2) {
      double u0[N], u1[N], a0[N], a1[N];
      ld_pair<N, D>(Up, q, u0, u1);
      vol_line<N, D>(w, q + N * cc, u0, ev, tt);
      vol_line<N, D>(w, q + 1 + N * cc, u1, ev, tt);
      ld_pair<N, D>(Lp, q, a0, a1);
      sipg_line<N, D, 0>(w, q + N * cc, u0, a0, el, tt);
      sipg_line<N, D, 0>(w, q + 1 + N * cc, u1, a1, el, tt);
      ld_pair<N, D>(Hp, q, a0, a1);
      sipg_line<N, D, 1>(w, q + N * cc, u0, a0, eh, tt);
      sipg_line<N, D, 1>(w, q + 1 + N * cc, u1, a1, eh, tt);
    }
  } else {
#pragma unroll
    for (int q = 0; q < N; ++q) {
      double u0[N], a0[N];
      ld_line<N, D>(Up, q, u0);
      vol_line<N, D>(w, q + N * cc, u0, ev, tt);
      ld_line<N, D>(Lp, q, a0);
      sipg_line<N, D, 0>(w, q + N * cc, u0, a0, el, tt);
      ld_line<N, D>(Hp, q, a0);
      sipg_line<N, D, 1>(w, q + N * cc, u0, a0, eh, tt);
    }
  }
}

// ---- folded forms (K2_FOLD): cells with all six faces; tt.Lf holds the volume
// operator plus the own-side SIPG parts of both faces, so a line costs one n x n
// product plus the neighbours' rank-2 parts (J_nb = a neighbour trace value, A_nb =
// its normal derivative: n FMAs per face) -- 12 instead of 20 operations per line and
// face.
template <int N, int D, int W>
__device__ __forceinline__ void lineop_f(double (&w)[W], int t, const double (&uo)[N], const double (&ul)[N],
                                         const double (&uh)[N], const TileTab<N> &tt) {
  double Al = 0.0, Ah = 0.0;
#pragma unroll
  for (int k = 0; k < N; ++k) {
    Al = fma(tt.d0[N - 1 - k], ul[k], Al);  // lo neighbour (minus side): its l'(1) = -d0 mirrored
    Ah = fma(tt.d0[k], uh[k], Ah);          // hi neighbour (plus side): its l'(0)
  }
  const double Jl = ul[N - 1], Jh = uh[0];
#pragma unroll
  for (int i = 0; i < N; ++i) {
    double r = w[lix<N, D>(t, i)];
#pragma unroll
    for (int j = 0; j < N; ++j) r = fma(tt.Lf[csym<N>(i * N + j)], uo[j], r);
    r = fma(tt.nJ[i], Jl, fma(tt.nA[i], Al, r));
    r = fma(tt.nJ[N - 1 - i], Jh, fma(tt.nA[N - 1 - i], Ah, r));
    w[lix<N, D>(t, i)] = r;
  }
}

template <int N, int D, int W>
__device__ __forceinline__ void axis_plane_f(double (&w)[W], const double *Up, const double *Lp, const double *Hp,
                                             int cc, const TileTab<N> &tt) {
  if constexpr (D == 1 && (N % 2) == 0) {
#pragma unroll
    for (int q = 0; q < N; q += 2) {
      double u0[N], u1[N], l0[N], l1[N], h0[N], h1[N];
      ld_pair<N, D>(Up, q, u0, u1);
      ld_pair<N, D>(Lp, q, l0, l1);
      ld_pair<N, D>(Hp, q, h0, h1);
      lineop_f<N, D>(w, q + N * cc, u0, l0, h0, tt);
      lineop_f<N, D>(w, q + 1 + N * cc, u1, l1, h1, tt);
    }
  } else {
#pragma unroll
    for (int q = 0; q < N; ++q) {
      double u0[N], l0[N], h0[N];
      ld_line<N, D>(Up, q, u0);
      ld_line<N, D>(Lp, q, l0);
      ld_line<N, D>(Hp, q, h0);
      lineop_f<N, D>(w, q + N * cc, u0, l0, h0, tt);
    }
  }
}

// z-line t = a + N b read in the thread's frame: position m at zb + zs*m
template <int N>
__device__ __forceinline__ void ld_zpair(const double *B, int t, int zb, int zs, double (&a)[N], double (&b)[N]) {
#pragma unroll
  for (int m = 0; m < N; ++m) {
    const double2 x = *reinterpret_cast<const double2 *>(B + t + zb + zs * m);
    a[m] = x.x;
    b[m] = x.y;
  }
}

// z terms of line t for the P own planes: volume rows 0..P-1, the own
// (mirrored-lo) face traces, their exchange with the partner, the SIPG spread
// of both faces; ghost penalty of either face if flagged.
template <int N, int W>
__device__ __forceinline__ void z_line(double (&w)[W], int t, const double (&uo)[N], const double (&ul)[N],
                                       double ev, double el, unsigned act, const TileTab<N> &tt) {
  constexpr int P = N / 2, NN = N * N;
#pragma unroll
  for (int c = 0; c < P; ++c) {
    double r = 0.0;
#pragma unroll
    for (int j = 0; j < N; ++j) r = fma(tt.L[csym<N>(c * N + j)], uo[j], r);
    w[t + NN * c] = fma(ev, r, w[t + NN * c]);
  }
  double A0 = 0.0, A1 = 0.0;
#pragma unroll
  for (int m = 0; m < N; ++m) {
    A0 = fma(tt.d0[m], uo[m], A0);
    A1 = fma(-tt.d0[N - 1 - m], ul[m], A1);
  }
  const double Jl = el * (uo[0] - ul[N - 1]);
  const double Al = el * (A0 + A1);
  const double Jh = __shfl_xor_sync(act, Jl, 16);
  const double Ah = -__shfl_xor_sync(act, Al, 16);
#pragma unroll
  for (int c = 0; c < P; ++c) {
    double &r = w[t + NN * c];
    r = fma(tt.cJ[c], Jl, fma(tt.cA[c], Al, r));
    r = fma(tt.cJ[N - 1 - c], Jh, fma(-tt.cA[N - 1 - c], Ah, r));
  }
}

// folded z line: rows 0..P-1 of Lf on the own line, the lo neighbour's parts, and the
// hi neighbour's parts from the partner (its lo neighbour in its mirrored frame:
// J' = u_hi(0), A' = sum_k d0[k] u_hi(k) -- no sign change)
template <int N, int W>
__device__ __forceinline__ void z_line_f(double (&w)[W], int t, const double (&uo)[N], const double (&ul)[N],
                                         unsigned act, const TileTab<N> &tt) {
  constexpr int P = N / 2, NN = N * N;
  double An = 0.0;
#pragma unroll
  for (int k = 0; k < N; ++k) An = fma(tt.d0[N - 1 - k], ul[k], An);
  const double Jn = ul[N - 1];
  const double Jp = __shfl_xor_sync(act, Jn, 16), Ap = __shfl_xor_sync(act, An, 16);
#pragma unroll
  for (int c = 0; c < P; ++c) {
    double r = w[t + NN * c];
#pragma unroll
    for (int j = 0; j < N; ++j) r = fma(tt.Lf[csym<N>(c * N + j)], uo[j], r);
    r = fma(tt.nJ[c], Jn, fma(tt.nA[c], An, r));
    r = fma(tt.nJ[N - 1 - c], Jp, fma(tt.nA[N - 1 - c], Ap, r));
    w[t + NN * c] = r;
  }
}

// z SIPG of face S (own frame) on line t, rows 0..P-1 only (both faces known)
template <int N, int S, int W>
__device__ __forceinline__ void zsipg_line(double (&w)[W], int t, const double (&uo)[N], const double (&un)[N],
                                           double en, const TileTab<N> &tt) {
  constexpr int P = N / 2, NN = N * N;
  double A0 = 0.0, A1 = 0.0;
#pragma unroll
  for (int m = 0; m < N; ++m) {
    if (S == 0) {
      A0 = fma(tt.d0[m], uo[m], A0);
      A1 = fma(-tt.d0[N - 1 - m], un[m], A1);
    } else {
      A0 = fma(-tt.d0[N - 1 - m], uo[m], A0);
      A1 = fma(tt.d0[m], un[m], A1);
    }
  }
  const double J = en * (S ? (uo[N - 1] - un[0]) : (uo[0] - un[N - 1]));
  const double A = en * (A0 + A1);
#pragma unroll
  for (int c = 0; c < P; ++c) {
    double &r = w[t + NN * c];
    if (S == 0) r = fma(tt.cJ[c], J, fma(tt.cA[c], A, r));
    else r = fma(tt.cJ[N - 1 - c], J, fma(-tt.cA[N - 1 - c], A, r));
  }
}

// Per-lane tile record fields (prefetched one tile ahead)
struct TileLane {
  int nslot, ncell, myblk, b0, b1;
  uint2 ln;
};
template <int SMAX>
__device__ __forceinline__ TileLane tile_lane(const TileRec<SMAX> *T, int cell, int tid, int nthr) {
  TileLane r;
  r.nslot = T->nslot;
  r.ncell = T->ncell;
  r.ln = *reinterpret_cast<const uint2 *>(&T->lane_nb[cell][0]);
  r.myblk = cell < r.ncell ? T->blk[cell] : 0;
  r.b0 = tid < r.nslot ? T->blk[tid] : 0;
  r.b1 = tid + nthr < r.nslot ? T->blk[tid + nthr] : 0;
  return r;
}

// MODE 0 (the only one): volume (per-lane bit) + SIPG (per-face bits) of uncut cells
// without ghost-penalty faces, v = result.
// Lane flags: lane_nb[l][1] byte 2 = GP faces, byte 3 = SIPG faces | volume << 6.
template <int N, int MODE>
__global__ void __launch_bounds__(64, T2MINB) k_tile2(const double *__restrict__ u, double *__restrict__ v,
                                                      const TileRec<Tile2Cfg<N>::SMAX> *__restrict__ tiles,
                                                      int ntiles, TileTab<N> tt, uint32_t mask) {
  static_assert(N % 2 == 0, "k_tile2 needs even N");
  using C = Tile2Cfg<N>;
  constexpr int P = C::P, NN = C::NN, N3 = C::N3, NP = C::NP, ST = C::ST;
  static_assert(C::SMAX <= 2 * C::THREADS, "two slot copies per thread");
  extern __shared__ __align__(16) double smem[];
  uint64_t *bar = reinterpret_cast<uint64_t *>(smem);  // [0] tile blocks
  double *S = smem + 2;
  const int tid = threadIdx.x, lane = tid & 31;
  const int cell = 16 * (tid >> 5) + (lane & 15), h = lane >> 4;
  const bool cell_on = (mask & TERM_CELL) != 0, sipg_on = (mask & TERM_SIPG) != 0, gp_on = (mask & TERM_GP) != 0;
  // the thread's frame: plane cc of the half is physical plane zb + zs cc; z position m at zb + zs m
  const int zb = h ? NN * (N - 1) : 0, zs = h ? -NN : NN;
  TL_BEGIN(1);
  pdl_trigger();
  if (tid == 0) {
    mbar_init(bar, 1);
    mbar_fence_init();
  }
  __syncthreads();
  uint32_t it = 0;
  TileLane nx;
  if ((int)blockIdx.x < ntiles) nx = tile_lane(tiles + blockIdx.x, cell, tid, C::THREADS);
  for (int tile = blockIdx.x; tile < ntiles; tile += gridDim.x, ++it) {
    const TileLane cu = nx;
    const bool on = cell < cu.ncell;
    fence_proxy_async();  // this thread's generic accesses to the slots precede the next bulk writes
    __syncthreads();
    if (tid == 0) mbar_expect_tx(bar, (uint32_t)(cu.nslot * N3 * 8));
    __syncthreads();
    if (tid < cu.nslot) bulk_g2s(S + tid * ST, u + (size_t)cu.b0 * N3, N3 * 8, bar);
    if (tid + C::THREADS < cu.nslot) bulk_g2s(S + (tid + C::THREADS) * ST, u + (size_t)cu.b1 * N3, N3 * 8, bar);
    if (tile + (int)gridDim.x < ntiles) nx = tile_lane(tiles + tile + gridDim.x, cell, tid, C::THREADS);
    mbar_wait(bar, it & 1);
    const unsigned act = __ballot_sync(0xffffffffu, on);
    double w[NP];
#pragma unroll
    for (int l = 0; l < NP; ++l) w[l] = 0.0;
    int nbs[6];
    uint32_t gpb = (cu.ln.y >> 16) & 0x3fu, spb = (cu.ln.y >> 24) & 0x3fu;
    const bool vol = ((cu.ln.y >> 30) & 1u) && cell_on;
    if (!gp_on) gpb = 0;
    if (!sipg_on) spb = 0;
#pragma unroll
    for (int f = 0; f < 4; ++f) nbs[f] = (cu.ln.x >> (8 * f)) & 0xff;
    nbs[4] = cu.ln.y & 0xff;
    nbs[5] = (cu.ln.y >> 8) & 0xff;
    if (h) {  // mirrored frame: the z faces swap
      const int x = nbs[4];
      nbs[4] = nbs[5];
      nbs[5] = x;
      gpb = (gpb & 0xfu) | (((gpb >> 4) & 1u) << 5) | (((gpb >> 5) & 1u) << 4);
      spb = (spb & 0xfu) | (((spb >> 4) & 1u) << 5) | (((spb >> 5) & 1u) << 4);
    }
    if (!on) gpb = spb = 0;
    const double *Us = S + cell * ST;
    const double *Nb[6];
#pragma unroll
    for (int f = 0; f < 6; ++f) Nb[f] = nbs[f] != 0xff ? S + nbs[f] * ST : Us;  // dummy source when absent
    static_assert(MODE == 0, "k_tile2: volume + SIPG only");
    if (on && K2_FOLD) {
      // every k_tile2 cell has six faces and no ghost penalty (host routing): folded operators
      static_for<0, 2>([&](auto dc) {
        constexpr int D = decltype(dc)::value;
#pragma unroll
        for (int cc = 0; cc < P; ++cc) {
          const int pz = zb + zs * cc;
          axis_plane_f<N, D>(w, Us + pz, Nb[2 * D] + pz, Nb[2 * D + 1] + pz, cc, tt);
        }
      });
#pragma unroll
      for (int t = 0; t < NN; t += 2) {
        double u0[N], u1[N], a0[N], a1[N];
        ld_zpair<N>(Us, t, zb, zs, u0, u1);
        ld_zpair<N>(Nb[4], t, zb, zs, a0, a1);
        z_line_f<N>(w, t, u0, a0, act, tt);
        z_line_f<N>(w, t + 1, u1, a1, act, tt);
      }
    } else if (on) {
      {
        const double ev = vol ? 1.0 : 0.0;
        // x and y: plane-local
        static_for<0, 2>([&](auto dc) {
          constexpr int D = decltype(dc)::value;
          const double el = ((spb >> (2 * D)) & 1u) ? 1.0 : 0.0, eh = ((spb >> (2 * D + 1)) & 1u) ? 1.0 : 0.0;
#pragma unroll
          for (int cc = 0; cc < P; ++cc) {
            const int pz = zb + zs * cc;
            axis_plane<N, D>(w, Us + pz, Nb[2 * D] + pz, Nb[2 * D + 1] + pz, cc, ev, el, eh, tt);
          }
        });
        // z: the own (mirrored-lo) face; the other face's traces come from the partner
        const double el = ((spb >> 4) & 1u) ? 1.0 : 0.0;
#pragma unroll
        for (int t = 0; t < NN; t += 2) {
          double u0[N], u1[N], a0[N], a1[N];
          ld_zpair<N>(Us, t, zb, zs, u0, u1);
          ld_zpair<N>(Nb[4], t, zb, zs, a0, a1);
          z_line<N>(w, t, u0, a0, ev, el, act, tt);
          z_line<N>(w, t + 1, u1, a1, ev, el, act, tt);
        }
      }
    }
    __syncthreads();  // every thread is done reading the tile's blocks
    if (on) {
      // v = (M (x) M (x) M) w: x and y sweeps on the own planes ...
      static_for<0, 2>([&](auto dc) {
        constexpr int D = decltype(dc)::value;
#pragma unroll
        for (int t = 0; t < N * P; ++t) {
          double x[N];
#pragma unroll
          for (int i = 0; i < N; ++i) {
            double r = 0.0;
#pragma unroll
            for (int j = 0; j < N; ++j) r = fma(tt.M[csym<N>(i * N + j)], w[lix<N, D>(t, j)], r);
            x[i] = r;
          }
#pragma unroll
          for (int i = 0; i < N; ++i) w[lix<N, D>(t, i)] = x[i];
        }
      });
      // ... and z with the partner's planes (its plane c sits at position N-1-c of our frame)
#pragma unroll
      for (int t = 0; t < NN; ++t) {
        double yp[P], x[P];
#pragma unroll
        for (int c = 0; c < P; ++c) yp[c] = __shfl_xor_sync(act, w[t + NN * c], 16);
#pragma unroll
        for (int i = 0; i < P; ++i) {
          double r = 0.0;
#pragma unroll
          for (int c = 0; c < P; ++c) {
            r = fma(tt.M[csym<N>(i * N + c)], w[t + NN * c], r);
            r = fma(tt.M[csym<N>(i * N + N - 1 - c)], yp[c], r);
          }
          x[i] = r;
        }
#pragma unroll
        for (int i = 0; i < P; ++i) w[t + NN * i] = x[i];
      }
      double *Uw = S + cell * ST;
#pragma unroll
      for (int c = 0; c < P; ++c)
#pragma unroll
        for (int t = 0; t < NN; t += 2)
          *reinterpret_cast<double2 *>(Uw + zb + zs * c + t) = make_double2(w[t + NN * c], w[t + 1 + NN * c]);
    }
    __syncwarp();  // both halves of the warp's 16 cells are in their slots
    // ---- coalesced write-back: one 512-byte row (a cell block) per instruction
    {
      static_assert(N3 == 64, "one double2 per lane per block");
      const int c0 = 16 * (tid >> 5);
      const int ncw = min(16, cu.ncell - c0);
#pragma unroll
      for (int g = 0; g < 16; g += 8) {
        double2 x[8];
        int ob[8];
#pragma unroll
        for (int c = 0; c < 8; ++c) {
          ob[c] = __shfl_sync(0xffffffffu, cu.myblk, g + c);
          if (g + c < ncw) {
            x[c] = *reinterpret_cast<const double2 *>(S + (c0 + g + c) * ST + 2 * lane);
          }
        }
#pragma unroll
        for (int c = 0; c < 8; ++c)
          if (g + c < ncw) *reinterpret_cast<double2 *>(v + (size_t)ob[c] * N3 + 2 * lane) = x[c];
      }
    }
  }

  TL_END(1);
  if (blockIdx.x == 0) pdl_wait();  // complete only after the primary (k_cutp) has
}

// ===================================================================== k_uncw
// k_uncw<N> (N = 5..9): uncut cells at high degree, every structured term (volume,
// SIPG on all faces, ghost penalty on faces to cut cells), v = result.  The same
// w-space arithmetic as k_tile2, organised for small code (runtime line loops, w in
// shared memory, small code): TPC threads per cell take every TPC-th line; the
// volume line operator and both faces of an axis touch the same lines, so only a
// __syncwarp separates the axes.
template <int N, int TCN = TileCfg<N>::TC>
struct UncwCfg {
  using T = TileCfgX<N, TCN>;
  static constexpr int N3 = N * N * N, NN = N * N;
  static constexpr int TC = TCN, TPC = 128 / TC;
  static constexpr int WST = N3 + ((N3 & 1) ? 0 : 1);  // odd: consecutive cells on different banks
  static constexpr int THREADS = 128;
  static constexpr int SMEM = T::SMEM + TC * WST * 8;
};

template <int N, int TCN = TileCfg<N>::TC>
__global__ void __launch_bounds__(128) k_uncw(const double *__restrict__ u, double *__restrict__ v,
                                              const TileRec<TileCfgX<N, TCN>::SMAX> *__restrict__ tiles, int ntiles,
                                              TileTab<N> tt, uint32_t mask) {
  using TC_ = TileCfgX<N, TCN>;
  using C = UncwCfg<N, TCN>;
  constexpr int NN = C::NN, N3 = C::N3, ST = TC_::ST, WST = C::WST, TPC = C::TPC;
  static_assert(32 % TPC == 0, "a cell's threads in one warp");
  extern __shared__ __align__(16) double smem[];
  uint64_t *bar = reinterpret_cast<uint64_t *>(smem);
  double *S = smem + 2;
  double *Wb = S + TC_::SMAX * ST;
  const int tid = threadIdx.x, cell = tid / TPC, r = tid % TPC;
  const bool cell_on = (mask & TERM_CELL) != 0, sipg_on = (mask & TERM_SIPG) != 0, gp_on = (mask & TERM_GP) != 0;
  pdl_trigger();
  TL_BEGIN(2);
  if (TC_::BULK && tid == 0) {
    mbar_init(bar, 1);
    mbar_fence_init();
  }
  __syncthreads();
  uint32_t it = 0;
  // bulk path: software pipeline -- the next tile's blocks are copied while this tile's
  // mass sweeps and write-back run (the slots are free once the axis terms are done)
  auto issue = [&](int tl) {
    const TileRec<TC_::SMAX> *Tn = tiles + tl;
    const int ns = Tn->nslot;
    fence_proxy_async();  // this thread's generic reads of the slots precede the bulk writes
    __syncthreads();
    if (tid == 0) mbar_expect_tx(bar, (uint32_t)(ns * N3 * 8));
    __syncthreads();
    for (int sl = tid; sl < ns; sl += C::THREADS) bulk_g2s(S + sl * ST, u + (size_t)Tn->blk[sl] * N3, N3 * 8, bar);
  };
  // odd n (blocks not a 16-byte multiple): the same pipeline with 8-byte cp.async
  // (every slot entry in flight at once, one wait_group per tile)
  auto issue_async = [&](int tl) {
    const TileRec<TC_::SMAX> *Tn = tiles + tl;
    const int ns = Tn->nslot;
    __syncthreads();  // every thread is done reading the slots
    for (int e = tid; e < ns * N3; e += C::THREADS) {
      const int sl = e / N3, l = e - sl * N3;
      cp_async8(S + sl * ST + l, u + (size_t)Tn->blk[sl] * N3 + l);
    }
    cp_async_commit();
  };
  if constexpr (TC_::BULK) {
    if ((int)blockIdx.x < ntiles) issue(blockIdx.x);
  } else {
    if ((int)blockIdx.x < ntiles) issue_async(blockIdx.x);
  }
  for (int tile = blockIdx.x; tile < ntiles; tile += gridDim.x, ++it) {
    const TileRec<TC_::SMAX> *T = tiles + tile;
    const int ncell = T->ncell;
    const bool on = cell < ncell;
    const uint2 ln = *reinterpret_cast<const uint2 *>(&T->lane_nb[on ? cell : 0][0]);
    // ---- the tile's blocks (issued during the previous tile)
    double *W = Wb + (on ? cell : 0) * WST;  // (axis 0 stores, the other axes accumulate)
    if constexpr (TC_::BULK) mbar_wait(bar, it & 1);
    else cp_async_wait<0>();
    __syncthreads();
    int nbs[6];
#pragma unroll
    for (int f = 0; f < 4; ++f) nbs[f] = (ln.x >> (8 * f)) & 0xff;
    nbs[4] = ln.y & 0xff;
    nbs[5] = (ln.y >> 8) & 0xff;
    const uint32_t gpb = (on && gp_on) ? (ln.y >> 16) & 0x3fu : 0u;
    const uint32_t spb = (on && sipg_on) ? (ln.y >> 24) & 0x3fu : 0u;
    const bool vol = on && cell_on && ((ln.y >> 30) & 1u);
    const double *Us = S + (on ? cell : 0) * ST;
    static_for<0, 3>([&](auto dc) {
      constexpr int D = decltype(dc)::value;
      constexpr int str = D == 0 ? 1 : (D == 1 ? N : NN);
      const bool gl = (gpb >> (2 * D)) & 1u, gh = (gpb >> (2 * D + 1)) & 1u;
      const bool sl = (spb >> (2 * D)) & 1u, sh = (spb >> (2 * D + 1)) & 1u;
      const double *Nl = (gl || sl) ? S + nbs[2 * D] * ST : Us;
      const double *Nh = (gh || sh) ? S + nbs[2 * D + 1] * ST : Us;
      if (on) {
#pragma unroll 1
        for (int t = r; t < NN; t += TPC) {
          const int t0 = t % N, t1 = t / N;
          const int b0 = D == 0 ? N * t0 + NN * t1 : (D == 1 ? t0 + NN * t1 : t0 + N * t1);
          double uo[N], out[N];
#pragma unroll
          for (int m = 0; m < N; ++m) uo[m] = Us[b0 + m * str];
          if constexpr (UNCW_EO && N >= 5) {  // even-odd: n^2/2 + 2n operations instead of n^2
            if (vol) eo_mv<N>(tt.Leo, uo, out);
            else {
#pragma unroll
              for (int i = 0; i < N; ++i) out[i] = 0.0;
            }
          } else {
#pragma unroll
            for (int i = 0; i < N; ++i) {
              double x = 0.0;
              if (vol) {
#pragma unroll
                for (int j = 0; j < N; ++j) x = fma(tt.L[csym<N>(i * N + j)], uo[j], x);
              }
              out[i] = x;
            }
          }
          static_for<0, 2>([&](auto sc) {
            constexpr int SS = decltype(sc)::value;
            const bool g = SS ? gh : gl, sp = SS ? sh : sl;
            if (!(g || sp)) return;
            const double *Nf = SS ? Nh : Nl;
            double un[N];
#pragma unroll
            for (int m = 0; m < N; ++m) un[m] = Nf[b0 + m * str];
            if (g) {
#pragma unroll
              for (int m = 0; m < N; ++m) {
                double x = out[m];
#pragma unroll
                for (int a = 0; a < N; ++a) {
                  const int k = SS ? (N - 1 - m) * N + (N - 1 - a) : m * N + a;
                  x = fma(tt.Goo[k], uo[a], fma(tt.Gon[k], un[a], x));
                }
                out[m] = x;
              }
            }
            if (sp) {
              double A0 = 0.0, A1 = 0.0;
#pragma unroll
              for (int m = 0; m < N; ++m) {
                if (SS == 0) {
                  A0 = fma(tt.d0[m], uo[m], A0);
                  A1 = fma(-tt.d0[N - 1 - m], un[m], A1);
                } else {
                  A0 = fma(-tt.d0[N - 1 - m], uo[m], A0);
                  A1 = fma(tt.d0[m], un[m], A1);
                }
              }
              const double J = SS ? (uo[N - 1] - un[0]) : (uo[0] - un[N - 1]);
              const double A = A0 + A1;
#pragma unroll
              for (int m = 0; m < N; ++m) {
                if (SS == 0) out[m] = fma(tt.cJ[m], J, fma(tt.cA[m], A, out[m]));
                else out[m] = fma(tt.cJ[N - 1 - m], J, fma(-tt.cA[N - 1 - m], A, out[m]));
              }
            }
          });
#pragma unroll
          for (int m = 0; m < N; ++m) {
            if (D == 0) W[b0 + m * str] = out[m];  // axis 0's lines cover every position once
            else W[b0 + m * str] += out[m];
          }
        }
      }
      __syncwarp();  // the next axis updates other threads' positions
    });
    if (tile + (int)gridDim.x < ntiles) {
      if constexpr (TC_::BULK) issue(tile + (int)gridDim.x);
      else issue_async(tile + (int)gridDim.x);
    }
    // ---- v = (M (x) M (x) M) w, sweeps in shared memory
    static_for<0, 3>([&](auto dc) {
      constexpr int D = decltype(dc)::value;
      constexpr int str = D == 0 ? 1 : (D == 1 ? N : NN);
      if (on) {
#pragma unroll 1
        for (int t = r; t < NN; t += TPC) {
          const int t0 = t % N, t1 = t / N;
          const int b0 = D == 0 ? N * t0 + NN * t1 : (D == 1 ? t0 + NN * t1 : t0 + N * t1);
          double x[N], y[N];
#pragma unroll
          for (int m = 0; m < N; ++m) x[m] = W[b0 + m * str];
          if constexpr (UNCW_EO && N >= 5) {
            eo_mv<N>(tt.Meo, x, y);
          } else {
#pragma unroll
            for (int i = 0; i < N; ++i) {
              double sacc = 0.0;
#pragma unroll
              for (int j = 0; j < N; ++j) sacc = fma(tt.M[csym<N>(i * N + j)], x[j], sacc);
              y[i] = sacc;
            }
          }
#pragma unroll
          for (int m = 0; m < N; ++m) W[b0 + m * str] = y[m];
        }
      }
      __syncwarp();
    });
    __syncthreads();  // all w final
    for (int e = tid; e < ncell * N3; e += C::THREADS) {
      const int c = e / N3, l = e - c * N3;
      v[(size_t)T->blk[c] * N3 + l] = Wb[c * WST + l];
    }
  }
  TL_END(2);
  if (blockIdx.x == 0) pdl_wait();  // complete only after the primary grid has
}

// ===================================================================== k_cell
// k_cell<N> (N = 2, 3): every structured term of the uncut cells (volume, SIPG on
// all faces, ghost penalty on the faces to cut cells), v = result.  At these
// degrees a block is 64 / 216 bytes: staging tiles with halos through TMA issues
// many tiny copies and amplifies the reads ~4x, so here ONE THREAD owns one cell,
// reads its block and each face neighbour's block straight from global memory
// (neighbours are shared by nearby threads: L1/L2 hits), keeps u, w and the
// neighbour block in registers and applies the same w-space operators as
// k_tile / k_uncw (M^{-1}-premultiplied line operators, then M (x) M (x) M).
// Cells: desc0[0, n0) then desc1[0, n1) (plain cells, cells next to cut cells).
#ifndef CELL_TPC
#define CELL_TPC 1  // threads per uncut cell in k_cell (1 or 2; 2 measured slower: p=1 80 -> 90 us)
#endif
#ifndef CELL_G2
#define CELL_G2 1  // measured: grouping the neighbour loads costs more occupancy than it hides
#endif
#ifndef CELL_G3
#define CELL_G3 1
#endif
#ifndef CELL_LD128
#define CELL_LD128 1  // k_cell<3>: 128-bit loads / stores on the 16-byte aligned part of the 216-byte blocks
#endif
#ifndef CELL_LD256
#define CELL_LD256 1  // n = 2: the 64-byte blocks through 256-bit loads / stores when 32-byte aligned
#endif
// sm_100: 256-bit global accesses (LDG.E.ENL2.256 / STG.E.ENL2.256), 32-byte aligned
__device__ __forceinline__ void ldg256(const double *p, double &a, double &b, double &c, double &d) {
  asm("ld.global.nc.v4.f64 {%0, %1, %2, %3}, [%4];" : "=d"(a), "=d"(b), "=d"(c), "=d"(d) : "l"(p));
}
__device__ __forceinline__ void stg256(double *p, double a, double b, double c, double d) {
  asm volatile("st.global.v4.f64 [%0], {%1, %2, %3, %4};" ::"l"(p), "d"(a), "d"(b), "d"(c), "d"(d) : "memory");
}

template <int N>
__device__ __forceinline__ void load_block(const double *__restrict__ p, double (&x)[N * N * N]) {
  constexpr int N3 = N * N * N;
  if constexpr (CELL_LD256 && (N3 % 4) == 0) {
    if ((reinterpret_cast<uintptr_t>(p) & 31) == 0) {  // (uniform: blocks are 32-byte multiples)
#pragma unroll
      for (int k = 0; k < N3; k += 4) ldg256(p + k, x[k], x[k + 1], x[k + 2], x[k + 3]);
      return;
    }
  }
  if constexpr ((N3 % 2) == 0) {
#pragma unroll
    for (int k = 0; k < N3; k += 2) {
      const double2 t = __ldg(reinterpret_cast<const double2 *>(p + k));
      x[k] = t.x;
      x[k + 1] = t.y;
    }
  } else if constexpr (CELL_LD128) {
    // odd N3 (n = 3): a block is only 8-byte aligned.  Its 16-byte aligned part (N3 - 1
    // values from p + par, par = the parity of the block's address in doubles) goes through
    // 128-bit loads, the one remaining value (the first or the last) through a 64-bit load:
    // 14 load instructions instead of 27 (the LSU queue was the top stall, lg_throttle)
    constexpr int H = N3 / 2;
    const bool par = ((reinterpret_cast<uintptr_t>(p) >> 3) & 1u) != 0;
    const double2 *q = reinterpret_cast<const double2 *>(p + (par ? 1 : 0));
    double V[2 * H];
#pragma unroll
    for (int i = 0; i < H; ++i) {
      const double2 t = __ldg(q + i);
      V[2 * i] = t.x;
      V[2 * i + 1] = t.y;
    }
    const double e = __ldg(p + (par ? 0 : N3 - 1));
#pragma unroll
    for (int k = 0; k < N3; ++k) x[k] = par ? (k == 0 ? e : V[k > 0 ? k - 1 : 0]) : (k == N3 - 1 ? e : V[k < N3 - 1 ? k : 0]);
  } else {
#pragma unroll
    for (int k = 0; k < N3; ++k) x[k] = __ldg(p + k);
  }
}

// the same split for the store of an odd-length block
template <int N>
__device__ __forceinline__ void store_block(double *__restrict__ p, const double (&w)[N * N * N]) {
  constexpr int N3 = N * N * N, H = N3 / 2;
  static_assert(N3 % 2 == 1, "odd blocks only");
  const bool par = ((reinterpret_cast<uintptr_t>(p) >> 3) & 1u) != 0;
  double2 *q = reinterpret_cast<double2 *>(p + (par ? 1 : 0));
#pragma unroll
  for (int i = 0; i < H; ++i) q[i] = par ? make_double2(w[2 * i + 1], w[2 * i + 2]) : make_double2(w[2 * i], w[2 * i + 1]);
  p[par ? 0 : N3 - 1] = par ? w[0] : w[N3 - 1];
}

template <int N>
__global__ void __launch_bounds__(128) k_cell(const double *__restrict__ u, double *__restrict__ v,
                                              const UDesc *__restrict__ desc0, int n0,
                                              const UDesc *__restrict__ desc1, int n1, TileTab<N> tt,
                                              uint32_t mask) {
  constexpr int NN = N * N, N3 = NN * N, TPC = CELL_TPC;
  // CELL_TPC = 2: a cell on a thread pair, faces 0-2 / 3-5 (halving each thread's chain of
  // dependent neighbour loads), w summed by one __shfl_xor per value
  const int gt = blockIdx.x * blockDim.x + threadIdx.x, i = gt / TPC, part = gt % TPC;
  // CTA 0 completes only after the primary (k_cutp) has: the apply's end in stream order
  if (blockIdx.x == 0 && threadIdx.x == 0) pdl_wait();
  if (TPC == 1 && i >= n0 + n1) return;
  const bool valid = i < n0 + n1;  // (TPC = 2: every thread stays for the shuffles)
  const int ic = valid ? i : 0;
  const UDesc d = ic < n0 ? desc0[ic] : desc1[ic - n0];
  const bool cell_on = (mask & TERM_CELL) != 0, sipg_on = (mask & TERM_SIPG) != 0, gp_on = (mask & TERM_GP) != 0;
  double uo[N3], w[N3];
  load_block<N>(u + (size_t)d.blk * N3, uo);
#pragma unroll
  for (int l = 0; l < N3; ++l) w[l] = 0.0;
  // volume: w += (M^{-1} h K1)_D along every axis
  if (cell_on) {
    static_for<0, 3>([&](auto dc) {
      constexpr int D = decltype(dc)::value;
      if (TPC == 2 && (D == 2) != (part == 1)) return;  // pair: axes 0, 1 / axis 2
#pragma unroll
      for (int t = 0; t < NN; ++t)
#pragma unroll
        for (int a = 0; a < N; ++a) {
          double x = w[lix<N, D>(t, a)];
#pragma unroll
          for (int b = 0; b < N; ++b) x = fma(tt.L[csym<N>(a * N + b)], uo[lix<N, D>(t, b)], x);
          w[lix<N, D>(t, a)] = x;
        }
    });
  }
  // faces: SIPG (every face with an active neighbour) and ghost penalty (faces to cut
  // cells).  The neighbour blocks of a group of faces (all six at n = 2, the two of an
  // axis at n = 3) are loaded together so their latencies overlap.
  constexpr int G = N == 2 ? CELL_G2 : CELL_G3;  // 1, 2, 3 or 6
  double nbv[G][N3];
  auto face_need = [&](int F, bool &sp, bool &g) {
    const int nbk = d.nb[F];
    sp = sipg_on && nbk >= 0;
    g = gp_on && nbk >= 0 && ((d.flags >> F) & 1u);
    return sp || g;
  };
  auto load_group = [&](int F0) {
#pragma unroll
    for (int k = 0; k < G; ++k) {
      bool sp, g;
      if (face_need(F0 + k, sp, g)) load_block<N>(u + (size_t)d.nb[F0 + k] * N3, nbv[k]);
    }
  };
  static_for<0, 6>([&](auto fc) {
    constexpr int F = decltype(fc)::value, D = F / 2, SS = F % 2;
    if (TPC == 2 && (F >= 3) != (part == 1)) return;  // pair: faces 0-2 / 3-5
    if constexpr (F % G == 0) load_group(F);
    bool sp, g;
    if (!face_need(F, sp, g)) return;
    const double(&un)[N3] = nbv[F % G];
#pragma unroll
    for (int t = 0; t < NN; ++t) {
      double o[N], n_[N], out[N];
#pragma unroll
      for (int m = 0; m < N; ++m) {
        o[m] = uo[lix<N, D>(t, m)];
        n_[m] = un[lix<N, D>(t, m)];
        out[m] = 0.0;
      }
      if (g) {
#pragma unroll
        for (int m = 0; m < N; ++m) {
          double x = 0.0;
#pragma unroll
          for (int a = 0; a < N; ++a) {
            const int k = SS ? (N - 1 - m) * N + (N - 1 - a) : m * N + a;
            x = fma(tt.Goo[k], o[a], fma(tt.Gon[k], n_[a], x));
          }
          out[m] = x;
        }
      }
      if (sp) {
        double A0 = 0.0, A1 = 0.0;
#pragma unroll
        for (int m = 0; m < N; ++m) {
          if (SS == 0) {
            A0 = fma(tt.d0[m], o[m], A0);
            A1 = fma(-tt.d0[N - 1 - m], n_[m], A1);
          } else {
            A0 = fma(-tt.d0[N - 1 - m], o[m], A0);
            A1 = fma(tt.d0[m], n_[m], A1);
          }
        }
        const double J = SS ? (o[N - 1] - n_[0]) : (o[0] - n_[N - 1]);
        const double A = A0 + A1;
#pragma unroll
        for (int m = 0; m < N; ++m) {
          if (SS == 0) out[m] = fma(tt.cJ[m], J, fma(tt.cA[m], A, out[m]));
          else out[m] = fma(tt.cJ[N - 1 - m], J, fma(-tt.cA[N - 1 - m], A, out[m]));
        }
      }
#pragma unroll
      for (int m = 0; m < N; ++m) w[lix<N, D>(t, m)] += out[m];
    }
  });
  if constexpr (TPC == 2) {
#pragma unroll
    for (int l = 0; l < N3; ++l) w[l] += __shfl_xor_sync(0xffffffffu, w[l], 1);
  }
  // v = (M (x) M (x) M) w
  static_for<0, 3>([&](auto dc) {
    constexpr int D = decltype(dc)::value;
#pragma unroll
    for (int t = 0; t < NN; ++t) {
      double x[N];
#pragma unroll
      for (int m = 0; m < N; ++m) x[m] = w[lix<N, D>(t, m)];
#pragma unroll
      for (int a = 0; a < N; ++a) {
        double y = 0.0;
#pragma unroll
        for (int b = 0; b < N; ++b) y = fma(tt.M[csym<N>(a * N + b)], x[b], y);
        w[lix<N, D>(t, a)] = y;
      }
    }
  });
  if (!valid) return;
  double *vb = v + (size_t)d.blk * N3;
  constexpr int H = TPC == 2 ? ((N3 / 2 + 1) & ~1) : N3;  // the pair splits the store (even cut)
  if constexpr (CELL_LD256 && TPC == 1 && (N3 % 4) == 0) {
    if ((reinterpret_cast<uintptr_t>(vb) & 31) == 0) {
#pragma unroll
      for (int k = 0; k < N3; k += 4) stg256(vb + k, w[k], w[k + 1], w[k + 2], w[k + 3]);
      return;
    }
  }
  if constexpr ((N3 % 2) == 0) {
#pragma unroll
    for (int k = 0; k < N3; k += 2)
      if (TPC == 1 || (k < H) == (part == 0)) *reinterpret_cast<double2 *>(vb + k) = make_double2(w[k], w[k + 1]);
  } else if constexpr (CELL_LD128 && TPC == 1) {
    store_block<N>(vb, w);
  } else {
#pragma unroll
    for (int k = 0; k < N3; ++k)
      if (TPC == 1 || (k < H) == (part == 0)) vb[k] = w[k];
  }
}
