// k_cutp<N> (N = p+1 = 4) and k_cut1<N, TPC> (N = 2, 3, at the end of this file): the
// unstructured terms of the cut cells (Alg. 1 "intersected" branch),
// included by kernels.cuh.
//
// One warp per cut cell, lanes = quadrature points (the paper's vectorisation
// over points), persistent: every warp walks its own list of cells, the
// lists balanced on the host by longest-processing-time assignment.  Three kinds of points form ONE stream per cell:
//   volume points     (xi, W):        W grad u . grad phi                    (eq:unstructured_cell)
//   interface points  (xi, n, W):     Nitsche  W [-(d_n phi) u - phi d_n u + tau/h phi u]
//   cut-face points   (xi on a face): SIPG over F cap Omega                  (eq:unstructured_face P:489-496)
// A cut-face point lies on a face of the cell, so its own-side test functions
// are the cell's tensor basis at that point (value l_m(face) = delta, normal
// derivative l'_m(face)): its flux  W [(sigma [u] - {d_n u}) [phi] - {d_n phi} [u]]
// is an ordinary point update with coefficients on phi and d_d phi.  [u] and
// {d_n u} at the point come from the face traces J_t = u_own - u_nb and
// A_t = d u_own + d u_nb on the n x n in-face nodes, evaluated by 2-D tensor
// interpolation (normal reduction first, then in-face evaluation).
// Every point is integrated into per-lane register accumulators for all n^3
// DoFs by the factored contraction; one butterfly reduction over the
// warp per cell, one coalesced write of the block.  The structured faces of the
// cut cell (full-face SIPG, ghost penalty) are computed here too, in w-space.
//
// Latency: the next cell's block + cut-face neighbour blocks are fetched (TMA
// bulk copies, or cp.async for odd n) into the second buffer set while the
// current cell's points run; point chunks of 32 are double-buffered across cell
// boundaries, so the stream never waits on a cold start.
#pragma once
#ifndef CUTP_MINB
#define CUTP_MINB 1
#endif
#ifdef CUTP_MAXNREG  // register cap (experiments: more warps per SM)
#define CUTP_BOUNDS __maxnreg__(CUTP_MAXNREG)
#else
#define CUTP_BOUNDS __launch_bounds__(32 * CUTP_WARPS, CUTP_MINB)
#endif
#ifndef CUTP_WARPS
#define CUTP_WARPS 1  // warps (cut cells in flight) per CTA: 1 lets other kernels share SMs
#endif

struct __align__(16) CDesc2 {
  int32_t blk;
  int32_t nb[6];     // neighbour block of each face with work, else -1
  uint32_t fmask;    // bit f: cut face f with points
  int64_t vb, sb, fb;  // first volume / interface / cut-face point of the cell
  int32_t nv, ns, nf;
  uint32_t smask;    // bits 0-5: ghost-penalty faces, bits 8-13: full-face SIPG faces
  int32_t nchunk;    // chunks of the cell in the plan, | (volume-line chunks, the first ones) << 16
                     // (a new point chunk starts at the
                     // volume/interface -> face boundary and at every face-axis boundary)
};

// value + reference gradient at a point from the unpadded block U (16-byte
// loads of the x rows when n is even)
template <int N>
__device__ __forceinline__ void eval_u(const double *U, const double (&vx)[N], const double (&dvx)[N],
                                       const double (&vy)[N], const double (&dvy)[N], const double (&vz)[N],
                                       const double (&dvz)[N], double &u0, double &ux, double &uy, double &uz) {
  u0 = ux = uy = uz = 0.0;
#pragma unroll
  for (int c = 0; c < N; ++c) {
    double t00 = 0.0, t10 = 0.0, t01 = 0.0;
#pragma unroll
    for (int b = 0; b < N; ++b) {
      double row[N];
      const double *rp = U + c * N * N + b * N;
      if constexpr ((N % 2) == 0) {
#pragma unroll
        for (int k = 0; k < N; k += 2) {
          const double2 x = *reinterpret_cast<const double2 *>(rp + k);
          row[k] = x.x;
          row[k + 1] = x.y;
        }
      } else {
#pragma unroll
        for (int k = 0; k < N; ++k) row[k] = rp[k];
      }
      double s0 = 0.0, s1 = 0.0;
#pragma unroll
      for (int a = 0; a < N; ++a) {
        s0 = fma(vx[a], row[a], s0);
        s1 = fma(dvx[a], row[a], s1);
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

// l_a(x), l_a'(x) from the monomial form in t = 2x - 1 and the symmetry
// l_{n-1-a}(t) = l_a(-t): even/odd parts in t^2 by Horner.
template <int N>
__device__ __forceinline__ void basis_vd_sym(const RefTab &R, double x, double (&v)[N], double (&dv)[N]) {
  const double t = fma(2.0, x, -1.0), t2 = t * t;
#pragma unroll
  for (int a = 0; a < (N + 1) / 2; ++a) {
    // E = sum_{k even} c_k t^k, O = sum_{k odd} c_k t^k; E' / O' of d/dx = 2 d/dt
    double E = 0.0, O = 0.0, Ed = 0.0, Od = 0.0;
#pragma unroll
    for (int k = N - 1; k >= 0; --k) {
      if (k % 2 == 0) E = fma(E, t2, R.mc[a][k]);
      else O = fma(O, t2, R.mc[a][k]);
    }
    O *= t;
#pragma unroll
    for (int k = N - 1; k >= 1; --k) {  // R.md[a][k] = 2 k mc[a][k]
      if (k % 2 == 1) Ed = fma(Ed, t2, R.md[a][k]);  // k odd: t^{k-1} even
      else Od = fma(Od, t2, R.md[a][k]);             // k even: t^{k-1} odd
    }
    Od *= t;
    if (a == N - 1 - a) {
      v[a] = E + O;
      dv[a] = Ed + Od;
    } else {
      v[a] = E + O;
      v[N - 1 - a] = E - O;
      dv[a] = Ed + Od;
      dv[N - 1 - a] = Od - Ed;
    }
  }
}

// A chunk of <= 32 stream points of one cell: vol rows [vo, vo+cv), interface
// rows [so, so+cs), cut-face rows [fo, fo+cf).  Built on the host per warp, in the
// order the warp consumes them.
struct __align__(16) CChunk {
  int32_t vo, so, fo;
  int32_t cnt;  // cv | cs << 8 | cf << 16
};

// A packet: consecutive chunks of one warp's stream, stored contiguously (each
// chunk = a 16-byte header {cnt} followed by its rows), fetched by ONE bulk copy.
struct __align__(16) CPacket {
  int64_t off;    // byte offset in the stream buffer
  int32_t bytes;  // multiple of 16
  int32_t nch;    // chunks in the packet
};
#ifndef CUTP_PK
#define CUTP_PK 4608  // packet capacity (bytes)
#endif
#ifndef CUTP_NB
#define CUTP_NB 3  // packet ring depth
#endif
#ifndef CUTP_FLINES
#define CUTP_FLINES 1  // n = 4: cut-face points in lines (face_line_rt)
#endif

// values only (cut-face points need no in-face derivatives)
template <int N>
__device__ __forceinline__ void basis_v_sym(const RefTab &R, double x, double (&v)[N]) {
  const double t = fma(2.0, x, -1.0), t2 = t * t;
#pragma unroll
  for (int a = 0; a < (N + 1) / 2; ++a) {
    double E = 0.0, O = 0.0;
#pragma unroll
    for (int k = N - 1; k >= 0; --k) {
      if (k % 2 == 0) E = fma(E, t2, R.mc[a][k]);
      else O = fma(O, t2, R.mc[a][k]);
    }
    O *= t;
    v[a] = E + O;
    if (a != N - 1 - a) v[N - 1 - a] = E - O;
  }
}

// One cut-face point (own-side reference coordinates; the normal coordinate is
// exactly 0 or 1, which selects the face axis d at run time, so chunks mix axes).
// Own-side test functions at the point: l_m(face) = delta_{m,fo} along d,
// l'_m(face) = dw[m], in-face values ls (lower in-face axis), lt (upper).  [u] = J
// and d u_own + d u_nb = A are interpolated from the face traces; the
// flux  W [(sigma J - s A/(2h)) phi - (s J/(2h)) d_d phi]  (s = +-1: own side) is
// the rank-1 update acc[c][b][a] += X_a Y_b Z_c with the normal factor T on axis d
// and the in-face bases on the others (selected, not branched).
template <int N, int ACC>
__device__ __forceinline__ void face_point_rt(double (&acc)[ACC], const RefTab &R, const double *JAB, double xi,
                                              double eta, double zeta, double W, const KParams &kp) {
  constexpr int NN = N * N;
  const int d = (xi == 0.0 || xi == 1.0) ? 0 : ((eta == 0.0 || eta == 1.0) ? 1 : 2);
  const double xd = d == 0 ? xi : (d == 1 ? eta : zeta);
  const int sd = xd == 1.0 ? 1 : 0;
  double ls[N], lt[N];
  basis_v_sym<N>(R, d == 0 ? eta : xi, ls);
  basis_v_sym<N>(R, d == 2 ? eta : zeta, lt);
  const double *JA = JAB + (2 * d + sd) * 2 * NN, *JB = JA + NN;
  double J = 0.0, A = 0.0;
#pragma unroll
  for (int j = 0; j < N; ++j) {
    double r0 = 0.0, r1 = 0.0;
#pragma unroll
    for (int i = 0; i < N; ++i) {
      r0 = fma(ls[i], JA[i + N * j], r0);
      r1 = fma(ls[i], JB[i + N * j], r1);
    }
    J = fma(lt[j], r0, J);
    A = fma(lt[j], r1, A);
  }
  const double sg = sd ? kp.i2h : -kp.i2h;
  const double k1 = W * fma(kp.sigma, J, -sg * A), k2 = -W * sg * J;
  double T[N];
#pragma unroll
  for (int m = 0; m < N; ++m) T[m] = k2 * (sd ? R.d1[m] : R.d0[m]);
  if (sd) T[N - 1] += k1;
  else T[0] += k1;
  double X[N], Y[N], Z[N];
#pragma unroll
  for (int m = 0; m < N; ++m) {
    X[m] = d == 0 ? T[m] : ls[m];
    Y[m] = d == 0 ? ls[m] : (d == 1 ? T[m] : lt[m]);
    Z[m] = d == 2 ? T[m] : lt[m];
  }
#pragma unroll
  for (int c = 0; c < N; ++c)
#pragma unroll
    for (int b = 0; b < N; ++b) {
      const double yz = Y[b] * Z[c];
#pragma unroll
      for (int a = 0; a < N; ++a) {
        double &r = acc[(c * N + b) * N + a];
        r = fma(X[a], yz, r);
      }
    }
}

// Cut-face points in LINES (the 2-D dimension reduction on the face plane, P:45-48:
// the q = n Gauss points of a line share the normal and one in-face coordinate).
// Record [xg, f + 8 la, (x_t, W_t) x n]: face f = 2 d + sd, points along axis la, the
// fixed in-face coordinate xg on the third axis g.  As for a cut-face point, the flux
// W [(sigma J - s A/(2h)) phi - (s J/(2h)) d_d phi] (eq:unstructured_face P:489-496)
// needs [u] = J and A = d u_own + d u_nb from the face traces: the fixed-axis sum is
// done once per line, then n-term sums per point.  Summed over the line's points the
// update is rank 2 on the axes (d, la, g):
//   acc += Dv (x) R2 (x) lg  +  e_fo (x) R1 (x) lg,
//   R2 = sum_t k2_t le(x_t),  R1 = sum_t k1_t le(x_t),  Dv = l'(face),  e_fo = l(face),
// the axes assigned at run time through a per-lane shared-memory slot (every face of
// a cell shares one chunk; the slot replaces ~100 selects).
template <int N, int ACC>
__device__ __forceinline__ void face_line_rt(double (&acc)[ACC], const RefTab &R, const double *JAB,
                                             const double *rec, const KParams &kp, double *slot) {
  constexpr int NN = N * N;
  const int meta = (int)rec[1], f = meta & 7, la = meta >> 3, d = f >> 1, sd = f & 1;
  const int g = 3 - d - la;
  // trace index i + N j: i along the lower in-face axis, j along the upper
  const bool lo = la < g;
  const int sl = lo ? 1 : N, sf = lo ? N : 1;  // strides of the line index, the fixed index
  double lg[N];
  basis_v_sym<N>(R, rec[0], lg);
  const double *JA = JAB + f * 2 * NN, *JB = JA + NN;
  double rJ[N], rA[N];
#pragma unroll
  for (int k = 0; k < N; ++k) {
    double x = 0.0, y = 0.0;
#pragma unroll
    for (int m = 0; m < N; ++m) {
      x = fma(lg[m], JA[k * sl + m * sf], x);
      y = fma(lg[m], JB[k * sl + m * sf], y);
    }
    rJ[k] = x;
    rA[k] = y;
  }
  const double sgn = sd ? kp.i2h : -kp.i2h;
  double R1[N], R2[N];
#pragma unroll
  for (int k = 0; k < N; ++k) R1[k] = R2[k] = 0.0;
#pragma unroll
  for (int t = 0; t < N; ++t) {
    const double2 tw = *reinterpret_cast<const double2 *>(rec + 2 + 2 * t);
    double le[N];
    basis_v_sym<N>(R, tw.x, le);
    double J = 0.0, A = 0.0;
#pragma unroll
    for (int k = 0; k < N; ++k) {
      J = fma(le[k], rJ[k], J);
      A = fma(le[k], rA[k], A);
    }
    const double k1 = tw.y * fma(kp.sigma, J, -sgn * A), k2 = -tw.y * sgn * J;
#pragma unroll
    for (int k = 0; k < N; ++k) {
      R1[k] = fma(k1, le[k], R1[k]);
      R2[k] = fma(k2, le[k], R2[k]);
    }
  }
  // slot[a N + m]: the factor on axis a; term 1 (Dv, R2, lg), then term 2 (e_fo, R1, lg)
#pragma unroll
  for (int m = 0; m < N; ++m) {
    slot[g * N + m] = lg[m];
    slot[la * N + m] = R2[m];
    slot[d * N + m] = sd ? R.d1[m] : R.d0[m];
  }
#pragma unroll
  for (int term = 0; term < 2; ++term) {
    if (term == 1) {
#pragma unroll
      for (int m = 0; m < N; ++m) {
        slot[la * N + m] = R1[m];
        slot[d * N + m] = m == (sd ? N - 1 : 0) ? 1.0 : 0.0;
      }
    }
    double X[N], Y[N], Z[N];
#pragma unroll
    for (int m = 0; m < N; ++m) {
      X[m] = slot[m];
      Y[m] = slot[N + m];
      Z[m] = slot[2 * N + m];
    }
#pragma unroll
    for (int c = 0; c < N; ++c)
#pragma unroll
      for (int b = 0; b < N; ++b) {
        const double yz = Y[b] * Z[c];
#pragma unroll
        for (int a = 0; a < N; ++a) {
          double &r = acc[(c * N + b) * N + a];
          r = fma(X[a], yz, r);
        }
      }
  }
}

// Volume points that come in LINES (dimension-reduction quadrature: along
// each line of the height axis AX the q = n Gauss points share the two base
// coordinates).  The base-plane part of the contraction is then done once per
// line instead of once per point (the paper's partial-sum reuse, P:874-878,
// extended across the points of a line):
//   P_i = sum_jk u(i,j,k) l1_j l2_k,  Q1_i = sum u l1'_j l2_k,  Q2_i = sum u l1_j l2'_k
//   per point t: u, d_AX u, d_B1 u, d_B2 u from 4 n-term sums over i, and the test
//   coefficients accumulated into R0_i = sum_t c_AX la'_i, R1_i = sum_t c_B1 la_i,
//   R2_i = sum_t c_B2 la_i
//   acc(i,j,k) += R0_i l1_j l2_k + R1_i l1'_j l2_k + R2_i l1_j l2'_k
// (i along AX, j along the lower base axis B1, k along the upper B2).  Record:
// [b1, b2, (t, W) x n].  About a third of the per-point FP64 work at n = 4.
template <int N, int AX>
__device__ __forceinline__ constexpr int lpos(int i, int j, int k) {
  // i along AX, j along B1 < B2, k along B2 -> l = x + N y + N^2 z
  return AX == 0 ? (i + N * j + N * N * k) : (AX == 1 ? (j + N * i + N * N * k) : (j + N * k + N * N * i));
}
// P_i, Q1_i, Q2_i of one volume line and its test coefficients R0, R1, R2 (every
// point of the line, and the line's interface point when srf and its W != 0).  U is
// the cell block in the LINE frame (i along the line, j, k along the base axes
// B1 < B2: UL[i + N j + N^2 k]), so one instance serves the three line axes and
// only the accumulation (vol_line_int) depends on the axis (smaller hot code).
template <int N>
__device__ __forceinline__ void vol_line_eval(const RefTab &R, const double *U, const double *rec, const KParams &kp,
                                              bool srf, double (&v1)[N], double (&d1)[N], double (&v2)[N],
                                              double (&d2)[N], double (&R0)[N], double (&R1)[N], double (&R2)[N]) {
  const double ih2 = kp.ih2;
  basis_vd_sym<N>(R, rec[0], v1, d1);
  basis_vd_sym<N>(R, rec[1], v2, d2);
  double Pp[N], Q1[N], Q2[N];
#pragma unroll
  for (int i = 0; i < N; ++i) Pp[i] = Q1[i] = Q2[i] = 0.0;
#pragma unroll
  for (int k = 0; k < N; ++k) {
    double s0[N], s1[N];
#pragma unroll
    for (int i = 0; i < N; ++i) s0[i] = s1[i] = 0.0;
#pragma unroll
    for (int j = 0; j < N; ++j) {
      double row[N];
      const double *rp = U + N * j + N * N * k;
      if constexpr ((N % 2) == 0) {
#pragma unroll
        for (int i = 0; i < N; i += 2) {
          const double2 x = *reinterpret_cast<const double2 *>(rp + i);
          row[i] = x.x;
          row[i + 1] = x.y;
        }
      } else {
#pragma unroll
        for (int i = 0; i < N; ++i) row[i] = rp[i];
      }
#pragma unroll
      for (int i = 0; i < N; ++i) {
        s0[i] = fma(v1[j], row[i], s0[i]);
        s1[i] = fma(d1[j], row[i], s1[i]);
      }
    }
#pragma unroll
    for (int i = 0; i < N; ++i) {
      Pp[i] = fma(v2[k], s0[i], Pp[i]);
      Q1[i] = fma(v2[k], s1[i], Q1[i]);
      Q2[i] = fma(d2[k], s0[i], Q2[i]);
    }
  }
#pragma unroll
  for (int i = 0; i < N; ++i) R0[i] = R1[i] = R2[i] = 0.0;
#pragma unroll
  for (int t = 0; t < N; ++t) {
    const double2 tw = *reinterpret_cast<const double2 *>(rec + 2 + 2 * t);
    double va[N], da[N];
    basis_vd_sym<N>(R, tw.x, va, da);
    double uA = 0.0, uB1 = 0.0, uB2 = 0.0;
#pragma unroll
    for (int i = 0; i < N; ++i) {
      uA = fma(da[i], Pp[i], uA);
      uB1 = fma(va[i], Q1[i], uB1);
      uB2 = fma(va[i], Q2[i], uB2);
    }
    const double sw = tw.y * ih2;
    const double cA = sw * uA, cB1 = sw * uB1, cB2 = sw * uB2;
#pragma unroll
    for (int i = 0; i < N; ++i) {
      R0[i] = fma(cA, da[i], R0[i]);
      R1[i] = fma(cB1, va[i], R1[i]);
      R2[i] = fma(cB2, va[i], R2[i]);
    }
  }
  if (srf) {
    // the line's interface (Nitsche) point, if any (W = 0 otherwise): rec[2 + 2N ..] =
    // t, W, n_ax, n_B1, n_B2 (the unit normal in the line's axes); value term folded into R0
    const double2 tw = *reinterpret_cast<const double2 *>(rec + 2 + 2 * N);
    const double2 nn = *reinterpret_cast<const double2 *>(rec + 4 + 2 * N);
    const double n2 = rec[6 + 2 * N];
    if (tw.y != 0.0) {
      double va[N], da[N];
      basis_vd_sym<N>(R, tw.x, va, da);
      double u0 = 0.0, uA = 0.0, uB1 = 0.0, uB2 = 0.0;
#pragma unroll
      for (int i = 0; i < N; ++i) {
        u0 = fma(va[i], Pp[i], u0);
        uA = fma(da[i], Pp[i], uA);
        uB1 = fma(va[i], Q1[i], uB1);
        uB2 = fma(va[i], Q2[i], uB2);
      }
      const double un = (nn.x * uA + nn.y * uB1 + n2 * uB2) * kp.ih;  // physical normal derivative
      const double c0 = tw.y * (kp.tau * u0 - un), g = -tw.y * u0 * kp.ih;
      const double cA = g * nn.x, cB1 = g * nn.y, cB2 = g * n2;
#pragma unroll
      for (int i = 0; i < N; ++i) {
        R0[i] = fma(cA, da[i], fma(c0, va[i], R0[i]));
        R1[i] = fma(cB1, va[i], R1[i]);
        R2[i] = fma(cB2, va[i], R2[i]);
      }
    }
  }
}

// acc(i,j,k) += R0_i l1_j l2_k + R1_i l1'_j l2_k + R2_i l1_j l2'_k in the cell frame
template <int N, int AX, int ACC>
__device__ __forceinline__ void vol_line_int(double (&acc)[ACC], const double (&v1)[N], const double (&d1)[N],
                                             const double (&v2)[N], const double (&d2)[N], const double (&R0)[N],
                                             const double (&R1)[N], const double (&R2)[N]) {
#pragma unroll
  for (int i = 0; i < N; ++i)
#pragma unroll
    for (int k = 0; k < N; ++k) {
      const double T0 = fma(R0[i], v2[k], R2[i] * d2[k]), T1 = R1[i] * v2[k];
#pragma unroll
      for (int j = 0; j < N; ++j) {
        double &r = acc[lpos<N, AX>(i, j, k)];
        r = fma(v1[j], T0, fma(d1[j], T1, r));
      }
    }
}

template <int N>
struct CutPCfg {
  static constexpr bool BULK = CUTFEM_USE_BULK && (N % 2) == 0;
  static constexpr int WARPS = CUTP_WARPS;
  static constexpr int NB = CUTP_NB;  // packet ring depth (NB-1 packets in flight while one is consumed)
  static constexpr int PK = CUTP_PK;  // packet capacity in bytes (>= the largest chunk)
  // largest chunks: 32 interface rows (64 B), 32 volume lines with their interface point
  static_assert(PK >= 16 + 32 * 64 && PK >= 16 + 32 * 8 * (2 + 2 * N + 6), "CUTP_PK below the largest chunk");
  static_assert(N == 4, "k_cutp serves n = 4 (n = 2, 3: k_cut1; n >= 5: k_cut)");
  static constexpr int NN = N * N, N3 = N * N * N, N3P = (N3 + 1) & ~1;
  static constexpr int ACC = 64;  // n^3 accumulators per lane
  // the reduction: one butterfly level (xor 16) + a 16-lane shared-memory transpose
  // cut-face points in lines (face_line_rt; its per-lane axis slots live in the
  // reduction buffer, which is free until the cell's reduction)
  static constexpr bool FLINES = CUTP_FLINES;
  static_assert(!FLINES || 32 * (3 * N + 1) <= 32 * 17, "face-line slots exceed the reduction buffer");
  // bars(2 + NB) | UB[2][7][N3P] | JAB[6][2][NN] | ring[NB][2 + PK/8] (nch + packet)
  static constexpr int OFF_UB = (2 + NB + 1) & ~1;
  static constexpr int OFF_JAB = OFF_UB + 2 * 7 * N3P;
  static constexpr int OFF_RING = OFF_JAB + ((6 * 2 * NN + 1) & ~1);
  static constexpr int RSLOT = 2 + PK / 8;
  static constexpr int OFF_WS = OFF_RING + NB * RSLOT;  // w of the structured faces (n^3)
  static constexpr int OFF_RED = OFF_WS + ((N3 + 1) & ~1);  // reduction transpose [32][17]
  // the warp's next <= DG cell descriptors, staged by one coalesced load per group
  // (8: 640 B, what is left of the SM's shared memory at 8 warps per SM)
  static constexpr int DG = 8;
  static constexpr int RED_SZ = 32 * 17;
  static constexpr int OFF_DSC = OFF_RED + RED_SZ;
  // the cell block in the line frame (vol_line_eval): inside the reduction buffer after
  // the face-line slots when it fits (both are free until the reduction), else its own
  static constexpr int SLOTS = FLINES ? 32 * (3 * N + 1) : 0;
  static constexpr bool UL_IN_RED = SLOTS + N3P <= RED_SZ;
  static constexpr int OFF_UL = UL_IN_RED ? OFF_RED + SLOTS : OFF_DSC + DG * (int)(sizeof(CDesc2) / 8);
  static constexpr int WSLOT = OFF_DSC + DG * (int)(sizeof(CDesc2) / 8) + (UL_IN_RED ? 0 : N3P);
  static constexpr int SMEM = WARPS * WSLOT * 8;
};

template <int N>
__global__ void CUTP_BOUNDS k_cutp(const double *__restrict__ u, double *__restrict__ v,
                                              const CDesc2 *__restrict__ desc, const CPacket *__restrict__ packets,
                                              const char *__restrict__ stream, const int *__restrict__ wstart,
                                              const int *__restrict__ pstart, KParams kp, TileTab<N> tt) {
  using C = CutPCfg<N>;
  using LN = BlkU<N>;
  constexpr int NN = C::NN, N3 = C::N3, N3P = C::N3P, NB = C::NB;
  const RefTab &R = c_ref[N - 2];
  extern __shared__ __align__(16) double smem[];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  // warp gw owns cells [wstart[gw], wstart[gw+1]) and their packets [pstart[gw], pstart[gw+1])
  // (longest-processing-time assignment computed at setup, heaviest first)
  pdl_trigger();  // every CTA of k_cutp has begun -> the uncut-cell kernels may start
  // a k_cutp launched behind another one (interior + boundary lists) completes only
  // after it (no-op for the apply's first, normally launched kernel)
  if (blockIdx.x == 0 && threadIdx.x == 0) pdl_wait();
  const int gw = blockIdx.x * C::WARPS + warp;
  const int c0w = wstart[gw], c1w = wstart[gw + 1];
  if (c0w >= c1w) return;
  TL_BEGIN(0);
  TL_WARP_BEGIN(gw);
  const int p0w = pstart[gw], p1w = pstart[gw + 1];
  double *base = smem + warp * C::WSLOT;
  uint64_t *bar = reinterpret_cast<uint64_t *>(base);  // 0,1: block sets; 2..2+NB: chunk ring
  double *UB = base + C::OFF_UB, *JAB = base + C::OFF_JAB, *RING = base + C::OFF_RING, *WS = base + C::OFF_WS;
  const bool gp_on = (kp.mask & TERM_GP) != 0;
  const bool cell_on = (kp.mask & TERM_CELL) != 0, nit_on = (kp.mask & TERM_NITSCHE) != 0,
             sipg_on = (kp.mask & TERM_SIPG) != 0;
  auto counts = [&](const CDesc2 &d, int &nv, int &ns, int &nf) {
    nv = cell_on ? d.nv : 0;
    ns = nit_on ? d.ns : 0;
    nf = sipg_on ? d.nf : 0;
  };
  auto fmask_of = [&](const CDesc2 &d) { return sipg_on ? d.fmask : 0u; };
  auto gmask_of = [&](const CDesc2 &d) { return gp_on ? (d.smask & 0x3fu) : 0u; };
  auto smask_of = [&](const CDesc2 &d) { return sipg_on ? ((d.smask >> 8) & 0x3fu) : 0u; };
  // blocks of a cell (own + cut-face neighbours) into set s
  auto issue_blocks = [&](const CDesc2 &d, int s) {
    double *U = UB + s * 7 * N3P;
    const uint32_t fm = fmask_of(d) | gmask_of(d) | smask_of(d);  // neighbour blocks needed
    if constexpr (C::BULK) {
      if (lane == 0) {
        mbar_expect_tx(bar + s, (uint32_t)((1 + __popc(fm)) * N3 * 8));
        bulk_g2s(U, u + (size_t)d.blk * N3, N3 * 8, bar + s);
#pragma unroll
        for (int f = 0; f < 6; ++f)
          if ((fm >> f) & 1u) bulk_g2s(U + (1 + f) * N3P, u + (size_t)d.nb[f] * N3, N3 * 8, bar + s);
      }
    } else {
      if (lane < N3) {
        cp_async8(U + lane, u + (size_t)d.blk * N3 + lane);
#pragma unroll
        for (int f = 0; f < 6; ++f)
          if ((fm >> f) & 1u) cp_async8(U + (1 + f) * N3P + lane, u + (size_t)d.nb[f] * N3 + lane);
      }
      cp_async_commit();
    }
  };
  // packet j of the warp's list (record r) into ring slot (j - p0w) % NB (lane 0)
  auto issue_packet = [&](int j, const CPacket &r) {
    if (lane != 0 || j >= p1w) return;
    const int b = (j - p0w) % NB;
    double *S = RING + b * C::RSLOT;
    reinterpret_cast<int *>(S)[0] = r.nch;
    mbar_expect_tx(bar + 2 + b, (uint32_t)r.bytes);
    bulk_g2s(S + 2, stream + r.off, (uint32_t)r.bytes, bar + 2 + b);
  };
  if (lane == 0) {
#pragma unroll
    for (int i = 0; i < 2 + NB; ++i) mbar_init(bar + i, 1);
    mbar_fence_init();
  }
  __syncwarp();
  // descriptors: groups of DG staged in shared memory (5 lanes per 80-byte descriptor,
  // one 16-byte word each; a global descriptor load per cell was exposed latency: ~4 %
  // of the stall samples)
  CDesc2 *DS = reinterpret_cast<CDesc2 *>(base + C::OFF_DSC);
  auto stage_desc = [&](int g0) {
    constexpr int W16 = (int)(sizeof(CDesc2) / 16);
    __syncwarp();
    for (int k = lane; k < C::DG * W16; k += 32) {
      const int c = g0 + k / W16;
      if (c < c1w)
        reinterpret_cast<uint4 *>(DS)[k] = reinterpret_cast<const uint4 *>(desc + c)[k % W16];
    }
    __syncwarp();
  };
  stage_desc(c0w);
  CDesc2 cd = DS[0];
  issue_blocks(cd, 0);
  // prologue: NB-1 packets in flight, the record of the next one prefetched into a register
  CPacket rn = {0, 0, 0};
  if (lane == 0) {
#pragma unroll
    for (int j = 0; j < NB - 1; ++j)
      if (p0w + j < p1w) issue_packet(p0w + j, packets[p0w + j]);
    if (p0w + NB - 1 < p1w) rn = packets[p0w + NB - 1];
  }
  int pj = p0w - 1, left = 0, pos = 0;  // packet being consumed, its chunks left, read position
  const double *S = RING;
  const double ih = kp.ih, ih2 = kp.ih2;
  int it = 0;
  for (int c = c0w; c < c1w; ++c, ++it) {
    const int set = it & 1;
    const bool has_next = c + 1 < c1w;
    CDesc2 nd;
    if (has_next) {
      if (((c + 1 - c0w) % C::DG) == 0) stage_desc(c + 1);  // cd (this cell) is in registers
      nd = DS[(c + 1 - c0w) % C::DG];
    }
    int nv, ns, nf;
    counts(cd, nv, ns, nf);
    // chunks of the cell: the first KL are volume lines
    // (lines never occur at n = 2: the host plans none, and the loop is compiled out)
    const int K = (int)((uint32_t)cd.nchunk & 0xffffu), KL = (int)(((uint32_t)cd.nchunk >> 16) & 0xffu);
    const int KF = C::FLINES ? (int)(((uint32_t)cd.nchunk >> 24) & 0xffu) : 0;  // cut-face line chunks
    const uint32_t fm = fmask_of(cd);
    // ---- this cell's blocks
    if constexpr (C::BULK) {
      mbar_wait(bar + set, (it >> 1) & 1);
    } else {
      cp_async_wait<0>();
      __syncwarp();
    }
    const double *U = UB + set * 7 * N3P;
    // ---- cut-face traces J_t = u_own - u_nb, A_t = d u_own + d u_nb (lanes: two faces per pass)
    if (fm) {
      const int side = lane >= NN ? 1 : 0, t = lane - side * NN;
      static_for<0, 3>([&](auto dc) {
        constexpr int D = decltype(dc)::value;
        const int f = 2 * D + side;
        if (lane < 2 * NN && ((fm >> f) & 1u)) {
          const double *NBf = U + (1 + f) * N3P;
          constexpr int st = LN::template lstride<D>();
          const int b0 = LN::template lbase<D>(t);
          const double *dow = side ? R.d1 : R.d0;
          const double *dnb = side ? R.d0 : R.d1;
          double A = 0.0;
#pragma unroll
          for (int m = 0; m < N; ++m) A = fma(dow[m], U[b0 + m * st], fma(dnb[m], NBf[b0 + m * st], A));
          const double J = side ? (U[b0 + (N - 1) * st] - NBf[b0]) : (U[b0] - NBf[b0 + (N - 1) * st]);
          JAB[f * 2 * NN + t] = J;
          JAB[f * 2 * NN + NN + t] = A;
        }
      });
      __syncwarp();
    }
    // ---- structured faces of the cut cell (ghost penalty, full-face SIPG) in w-space:
    //      w += M^-1-premultiplied line operators along each face normal, then
    //      w <- (M (x) M (x) M) w; added to the point sums at the end (lanes 0..15 = lines)
    const uint32_t gm = gmask_of(cd), sm = smask_of(cd);
    if (gm | sm) {
      // per axis: lanes 0..15 the lo face in the own frame, lanes 16..31 the hi face in
      // the line-reversed frame (same lo-face coefficients: all operators are
      // centro-symmetric); the hi half's rows are folded into the lo half by a shuffle.
      // The three axes are computed first (independent chains), then accumulated into w.
      const int hs = lane >> 4, t = lane & 15;
      double oa[3][N];
      static_for<0, 3>([&](auto dc) {
        constexpr int D = dc.value;
        constexpr int str = D == 0 ? 1 : (D == 1 ? N : NN);
        const int f = 2 * D + hs;
        const bool g = ((gm >> f) & 1u) != 0, sp = ((sm >> f) & 1u) != 0;
        const bool anyg = __any_sync(0xffffffffu, g), anys = __any_sync(0xffffffffu, sp);
        if (anyg || anys) {
          const double *NBf = U + (1 + (g || sp ? f : 2 * D)) * N3P;
          const int tt0 = (t < NN ? t : 0) % N, tt1 = (t < NN ? t : 0) / N;
          const int b0 = D == 0 ? N * tt0 + NN * tt1 : (D == 1 ? tt0 + NN * tt1 : tt0 + N * tt1);
          double uo[N], un[N], out[N];
#pragma unroll
          for (int m = 0; m < N; ++m) {
            const int pm = hs ? N - 1 - m : m;
            uo[m] = U[b0 + pm * str];
            un[m] = (g || sp) ? NBf[b0 + pm * str] : 0.0;
            out[m] = 0.0;
          }
          if (anyg) {
            const double eg = g ? 1.0 : 0.0;
#pragma unroll
            for (int m = 0; m < N; ++m) {
              double x = 0.0;
#pragma unroll
              for (int a2 = 0; a2 < N; ++a2) x = fma(tt.Goo[m * N + a2], uo[a2], fma(tt.Gon[m * N + a2], un[a2], x));
              out[m] = eg * x;
            }
          }
          if (anys) {
            double A0 = 0.0, A1 = 0.0;
#pragma unroll
            for (int m = 0; m < N; ++m) {
              A0 = fma(tt.d0[m], uo[m], A0);
              A1 = fma(-tt.d0[N - 1 - m], un[m], A1);
            }
            const double es = sp ? 1.0 : 0.0;
            const double J = es * (uo[0] - un[N - 1]);
            const double A = es * (A0 + A1);
#pragma unroll
            for (int m = 0; m < N; ++m) out[m] = fma(tt.cJ[m], J, fma(tt.cA[m], A, out[m]));
          }
          double o2[N];
#pragma unroll
          for (int m = 0; m < N; ++m) o2[m] = __shfl_xor_sync(0xffffffffu, out[m], 16);
#pragma unroll
          for (int m = 0; m < N; ++m) oa[D][m] = out[m] + o2[N - 1 - m];
        } else {
#pragma unroll
          for (int m = 0; m < N; ++m) oa[D][m] = 0.0;
        }
      });
      // w = sum over the axes (axis 0's lines cover every position once: plain store first)
      static_for<0, 3>([&](auto dc) {
        constexpr int D = dc.value;
        constexpr int str = D == 0 ? 1 : (D == 1 ? N : NN);
        if (hs == 0 && t < NN) {
          const int tt0 = t % N, tt1 = t / N;
          const int b0 = D == 0 ? N * tt0 + NN * tt1 : (D == 1 ? tt0 + NN * tt1 : tt0 + N * tt1);
#pragma unroll
          for (int m = 0; m < N; ++m) {
            if (D == 0) WS[b0 + m * str] = oa[D][m];
            else WS[b0 + m * str] += oa[D][m];
          }
        }
        __syncwarp();
      });
      // w <- (M (x) M (x) M) w: line t, rows split between the halves (the hi half in the
      // reversed frame computes rows n-1, n-2, ... with the same coefficients)
      static_for<0, 3>([&](auto dc) {
        constexpr int D = dc.value;
        constexpr int str = D == 0 ? 1 : (D == 1 ? N : NN);
        constexpr int R = (N % 2 == 0) ? N / 2 : N;  // rows per half (odd n: the lo half does all)
        const bool act = t < NN && ((N % 2 == 0) || hs == 0);
        double x[N], y[R];
        const int tt0 = (t < NN ? t : 0) % N, tt1 = (t < NN ? t : 0) / N;
        const int b0 = D == 0 ? N * tt0 + NN * tt1 : (D == 1 ? tt0 + NN * tt1 : tt0 + N * tt1);
        if (act) {
#pragma unroll
          for (int m = 0; m < N; ++m) x[m] = WS[b0 + (hs ? N - 1 - m : m) * str];
#pragma unroll
          for (int i = 0; i < R; ++i) {
            double sacc = 0.0;
#pragma unroll
            for (int j = 0; j < N; ++j) sacc = fma(tt.M[csym<N>(i * N + j)], x[j], sacc);
            y[i] = sacc;
          }
        }
        __syncwarp();
        if (act) {
#pragma unroll
          for (int i = 0; i < R; ++i) WS[b0 + (hs ? N - 1 - i : i) * str] = y[i];
        }
        __syncwarp();
      });
    }
    // ---- next cell's blocks into the other set (its previous user, cell it-1, is done)
    if (has_next) issue_blocks(nd, set ^ 1);
    // ---- the point stream
    double acc[C::ACC];
#pragma unroll
    for (int i = 0; i < C::ACC; ++i) acc[i] = 0.0;
    auto next_packet = [&]() {  // wait for the next packet, refill the slot of the previous one
      ++pj;
      const int b = (pj - p0w) % NB;
      mbar_wait(bar + 2 + b, ((pj - p0w) / NB) & 1);
      if (lane == 0) {
        issue_packet(pj + NB - 1, rn);
        if (pj + NB < p1w) rn = packets[pj + NB];
      }
      S = RING + b * C::RSLOT;
      left = reinterpret_cast<const int *>(S)[0];
      pos = 2;
    };
    // volume LINES first (their own loop: the point loop below keeps its code
    // generation): chunks of cv lines along axis (cnt >> 24) & 3, records of 2 + 2N doubles
    const double *UL = U;  // the block in the line frame (a copy when the lines are not along x)
    for (int k = 0; k < KL; ++k) {
      if (left == 0) next_packet();
      const int cnt = reinterpret_cast<const int *>(S + pos)[0];
      const int cv = cnt & 0xff, ax = (cnt >> 24) & 3;
      const bool srf = (cnt >> 29) & 1;  // records carry the line's interface point
      const int rs = 2 + 2 * N + (srf ? 6 : 0);
      const double *P = S + pos + 2;
      --left;
      pos += 2 + rs * cv;
      if (k == 0 && ax != 0) {
        // UL[i + N j + N^2 k] = U[lpos<AX>(i, j, k)] (every line of a cell has one axis)
        double *Ut = base + C::OFF_UL;
        for (int l = lane; l < N3; l += 32) {
          const int i = l % N, j = (l / N) % N, kk = l / NN;
          Ut[l] = U[ax == 1 ? (j + N * i + NN * kk) : (j + N * kk + NN * i)];
        }
        __syncwarp();
        UL = Ut;
      }
      if (lane < cv) {
        const double *rec = P + rs * lane;
        double v1[N], d1[N], v2[N], d2[N], R0[N], R1[N], R2[N];
        vol_line_eval<N>(R, UL, rec, kp, srf, v1, d1, v2, d2, R0, R1, R2);
        if (ax == 0) vol_line_int<N, 0>(acc, v1, d1, v2, d2, R0, R1, R2);
        else if (ax == 1) vol_line_int<N, 1>(acc, v1, d1, v2, d2, R0, R1, R2);
        else vol_line_int<N, 2>(acc, v1, d1, v2, d2, R0, R1, R2);
      }
      __syncwarp();
      if (lane == 0 && left == 0) fence_proxy_async();
    }
    // cut-face LINES (n = 4): chunks of <= 32 line records of any face, 2 + 2N doubles each
    for (int k = KL; k < (C::FLINES ? KL + KF : KL); ++k) {
      if (left == 0) next_packet();
      const int cl = reinterpret_cast<const int *>(S + pos)[0] & 0xff;
      const double *P = S + pos + 2;
      --left;
      pos += 2 + (2 + 2 * N) * cl;
      if (lane < cl) face_line_rt<N>(acc, R, JAB, P + (2 + 2 * N) * lane, kp, base + C::OFF_RED + lane * (3 * N + 1));
      __syncwarp();
      if (lane == 0 && left == 0) fence_proxy_async();
    }
    for (int k = KL + KF; k < K; ++k) {
      if (left == 0) next_packet();
      const int cnt = reinterpret_cast<const int *>(S + pos)[0];
      const int cv = cnt & 0xff, cs = (cnt >> 8) & 0xff, cf = (cnt >> 16) & 0xff;
      const double *P = S + pos + 2;  // the chunk's rows
      --left;
      pos += 2 + 4 * cv + 8 * cs + 4 * cf;
      // kind: 0 volume, 1 interface, 2 cut face, 3 idle lane
      const int kind = lane < cv ? 0 : (lane < cv + cs ? 1 : (lane < cv + cs + cf ? 2 : 3));
      double xi = 0.5, eta = 0.5, zeta = 0.5, W = 0.0, nx = 0.0, ny = 0.0, nz = 0.0;
      if (kind == 0 || kind == 2) {
        const double *pp = P + (kind == 0 ? 4 * lane : 4 * cv + 8 * cs + 4 * (lane - cv - cs));
        const double2 p0 = *reinterpret_cast<const double2 *>(pp);
        const double2 p1 = *reinterpret_cast<const double2 *>(pp + 2);
        xi = p0.x;
        eta = p0.y;
        zeta = p1.x;
        W = p1.y;
      } else if (kind == 1) {
        const double *pp = P + 4 * cv + 8 * (lane - cv);
        const double2 p0 = *reinterpret_cast<const double2 *>(pp);
        const double2 p1 = *reinterpret_cast<const double2 *>(pp + 2);
        const double2 p2 = *reinterpret_cast<const double2 *>(pp + 4);
        const double2 p3 = *reinterpret_cast<const double2 *>(pp + 6);
        xi = p0.x;
        eta = p0.y;
        zeta = p1.x;
        nx = p1.y;
        ny = p2.x;
        nz = p2.y;
        W = p3.x;
      }
      if (kind < 2) {
        double vx[N], dvx[N], vy[N], dvy[N], vz[N], dvz[N];
        basis_vd_sym<N>(R, xi, vx, dvx);
        basis_vd_sym<N>(R, eta, vy, dvy);
        basis_vd_sym<N>(R, zeta, vz, dvz);
        double c0 = 0.0, c1, c2, c3;
        double u0, ux, uy, uz;
        eval_u<N>(U, vx, dvx, vy, dvy, vz, dvz, u0, ux, uy, uz);
        if (kind == 1) {
          const double un = (nx * ux + ny * uy + nz * uz) * ih;  // physical normal derivative
          c0 = W * (kp.tau * u0 - un);
          const double g = -W * u0 * ih;
          c1 = g * nx;
          c2 = g * ny;
          c3 = g * nz;
        } else {
          const double sw = W * ih2;
          c1 = sw * ux;
          c2 = sw * uy;
          c3 = sw * uz;
        }
#pragma unroll
        for (int cz = 0; cz < N; ++cz) {
          const double T0 = fma(c0, vz[cz], c3 * dvz[cz]);
          const double T1 = c2 * vz[cz];
          const double T2 = c1 * vz[cz];
#pragma unroll
          for (int by = 0; by < N; ++by) {
            const double S0 = fma(vy[by], T0, dvy[by] * T1);
            const double S1 = vy[by] * T2;
#pragma unroll
            for (int ax = 0; ax < N; ++ax) {
              double &r = acc[(cz * N + by) * N + ax];
              r = fma(vx[ax], S0, fma(dvx[ax], S1, r));
            }
          }
        }
      } else if (kind == 2) {
        // cut-face point: the face is the coordinate that is exactly 0 or 1
        face_point_rt<N>(acc, R, JAB, xi, eta, zeta, W, kp);
      }
      __syncwarp();  // every lane is done with the ring slot before it is refilled
      if (lane == 0 && left == 0) fence_proxy_async();
    }
    // ---- reduce over the warp and write the block (every cut cell block written once):
    // lanes l, l^16 exchange halves (xor 16): half h = lane >> 4 then holds entries
    // 32 h + i summed over the pair; two passes transpose 16 of them over the 16 lanes
    // of each half through shared memory, lane l summing entry 32 (l >> 4) + 16 ps + (l & 15)
    // over the 16 lanes in a fixed order
    double *RED = base + C::OFF_RED;
    double *vb = v + (size_t)cd.blk * N3;
    const bool st_on = (gm | sm) != 0;
    {
      const bool up = (lane & 16) != 0;
      double a32[32];
#pragma unroll
      for (int i = 0; i < 32; ++i) {
        const double send = up ? acc[i] : acc[i + 32];
        const double keep = up ? acc[i + 32] : acc[i];
        a32[i] = keep + __shfl_xor_sync(0xffffffffu, send, 16);
      }
      const int h = lane >> 4, l16 = lane & 15;
#pragma unroll
      for (int ps = 0; ps < 2; ++ps) {
#pragma unroll
        for (int i = 0; i < 16; ++i) RED[(h * 16 + i) * 17 + l16] = a32[ps * 16 + i];
        __syncwarp();
        double s0 = 0.0, s1 = 0.0, s2 = 0.0, s3 = 0.0;
#pragma unroll
        for (int k = 0; k < 16; k += 4) {
          s0 += RED[lane * 17 + k];
          s1 += RED[lane * 17 + k + 1];
          s2 += RED[lane * 17 + k + 2];
          s3 += RED[lane * 17 + k + 3];
        }
        const int e = 32 * h + 16 * ps + l16;
        vb[e] = ((s0 + s1) + (s2 + s3)) + (st_on ? WS[e] : 0.0);
        __syncwarp();
      }
    }
    if constexpr (!C::BULK) __syncwarp();
    if (has_next) cd = nd;
  }
  TL_WARP_END(gw);
  TL_END(0);
}


// ======================================================= cut cells, p = 1, 2 (k_cut1)
#ifndef CUT1_LD128
#define CUT1_LD128 1  // own block and result through 128-bit loads / stores
#endif
#ifndef CUT1_PT256
#define CUT1_PT256 1  // point rows through 256-bit loads
#endif
#ifndef CUT1_NBREG
#define CUT1_NBREG 1  // structured faces: the neighbour block in registers (128-bit loads) instead of per-line loads
#endif
// One THREAD (p = 1) or a thread PAIR (p = 2) per cut cell (k_cell's layout for the
// uncut cells): at p = 1, 2 a cut cell has ~30 / ~85 points and 8 / 27 DoFs, so a warp
// per cell (k_cutp) spends most of its time in per-cell work done by a few lanes
// (traces, structured faces, the cross-lane reduction); here 32 / 16 cells run side by
// side in SIMT and every accumulator is the thread's own.  Cells come heavy-first in the descriptor list, so a warp's cells
// have similar point counts.  Per cell (all FP64, same formulas as k_cutp):
//   1. structured faces (ghost penalty, full-face SIPG) in w-space with the
//      M^-1-premultiplied line operators (k_cell), then w <- (M (x) M (x) M) w; acc = w
//   2. volume points   acc += W/h^2 grad u . grad phi               (eq:unstructured_cell)
//   3. interface points acc += Nitsche W [-(d_n phi) u - phi d_n u + tau phi u]
//   4. cut faces: traces [u], d u_own + d u_nb on the n^2 in-face nodes, per point
//      the 2-D interpolation and the flux coefficients summed per in-face node, then
//      applied along the face normal (eq:unstructured_face P:489-496)
// Neighbour values are read straight from global memory (L1 / L2 hits).
// TPC > 1: a cell on TPC consecutive lanes (k = lane % TPC): face F's structured part on
// lane F % TPC, every TPC-th point of each kind on each lane, the cut faces' traces on
// all of them; each lane applies M (x) M (x) M to its own structured part (linear), and
// the TPC partial accumulators are summed by an xor butterfly (commutative: every lane
// of the group gets the same bits); lane k writes the entries l = k mod TPC.
template <int N, int TPC>
__global__ void __launch_bounds__(128) k_cut1(const double *__restrict__ u, double *__restrict__ v,
                                              const CDesc *__restrict__ desc, int ncut,
                                              const double *__restrict__ vol_pts, const double *__restrict__ srf_pts,
                                              const double *__restrict__ sf_pts, const int64_t *__restrict__ sf_ptr,
                                              KParams kp, TileTab<N> tt) {
  constexpr int NN = N * N, N3 = NN * N;
  static_assert(TPC >= 1 && TPC <= 32 && (32 % TPC) == 0, "TPC divides the warp");
  const RefTab &R = c_ref[N - 2];
  pdl_trigger();  // every CTA has begun -> the uncut-cell kernels may start
  if (blockIdx.x == 0 && threadIdx.x == 0) pdl_wait();
  const int gi = blockIdx.x * blockDim.x + threadIdx.x, kk = gi % TPC;
  const int i0 = gi / TPC;
  if constexpr (TPC == 1) {
    if (i0 >= ncut) return;
  } else {
    if (__all_sync(0xffffffffu, i0 >= ncut)) return;  // (the butterfly needs whole warps)
  }
  const bool valid = i0 < ncut;
  const int i = valid ? i0 : ncut - 1;
  const CDesc d = desc[i];
  const bool cell_on = (kp.mask & TERM_CELL) != 0, sipg_on = (kp.mask & TERM_SIPG) != 0,
             nit_on = (kp.mask & TERM_NITSCHE) != 0, gp_on = (kp.mask & TERM_GP) != 0;
  double uo[N3], acc[N3];
  {
    const double *ub = u + (size_t)d.blk * N3;
    if constexpr (CUT1_LD128) load_block<N>(ub, uo);  // 128-bit loads (kernels_tile.cuh)
    else {
#pragma unroll
      for (int k = 0; k < N3; ++k) uo[k] = __ldg(ub + k);
    }
  }
  // n = 3: the cut faces' point ranges requested now (consumed in step 4, so the dependent
  // loads stay off that step's critical path; C3 p=2 apply 213 -> 210 us).  n = 2: at the
  // face (the 24 extra registers cost k_cell's co-running warps more: 120 -> 124 us)
  constexpr bool HOIST = N >= 3;
  int64_t fpb[6], fpe[6];
#pragma unroll
  for (int F = 0; F < 6; ++F) {
    const bool cf = HOIST && sipg_on && d.nb[F] >= 0 && ((d.flags >> (12 + F)) & 1u);
    fpb[F] = cf ? __ldg(sf_ptr + d.sf[F]) : 0;
    fpe[F] = cf ? __ldg(sf_ptr + d.sf[F] + 1) : 0;
  }
  // ---- 1. structured faces in w-space
#pragma unroll
  for (int l = 0; l < N3; ++l) acc[l] = 0.0;
  bool any_st = false;
  static_for<0, 6>([&](auto fc) {
    constexpr int F = decltype(fc)::value, D = F / 2, SS = F % 2;
    const bool g = gp_on && d.nb[F] >= 0 && ((d.flags >> F) & 1u);
    const bool sp = sipg_on && d.nb[F] >= 0 && ((d.flags >> (6 + F)) & 1u);
    if (!(g || sp) || (F % TPC) != kk) return;
    any_st = true;
    const double *nbp = u + (size_t)d.nb[F] * N3;
    double nbv[CUT1_NBREG ? N3 : 1];
    if constexpr (CUT1_NBREG) load_block<N>(nbp, nbv);  // the neighbour block by 128-bit loads
#pragma unroll
    for (int t = 0; t < NN; ++t) {
      double o[N], n_[N], out[N];
#pragma unroll
      for (int m = 0; m < N; ++m) {
        o[m] = uo[lix<N, D>(t, m)];
        if constexpr (CUT1_NBREG) n_[m] = nbv[lix<N, D>(t, m)];
        else n_[m] = __ldg(nbp + lix<N, D>(t, m));
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
      for (int m = 0; m < N; ++m) acc[lix<N, D>(t, m)] += out[m];
    }
  });
  if (any_st) {  // acc <- (M (x) M (x) M) acc
    static_for<0, 3>([&](auto dc) {
      constexpr int D = decltype(dc)::value;
#pragma unroll
      for (int t = 0; t < NN; ++t) {
        double x[N];
#pragma unroll
        for (int m = 0; m < N; ++m) x[m] = acc[lix<N, D>(t, m)];
#pragma unroll
        for (int a = 0; a < N; ++a) {
          double y = 0.0;
#pragma unroll
          for (int b = 0; b < N; ++b) y = fma(tt.M[csym<N>(a * N + b)], x[b], y);
          acc[lix<N, D>(t, a)] = y;
        }
      }
    });
  }
  // ---- 2./3. volume and interface points: value + reference gradient, the point
  //      coefficients, the rank-update of acc (c0 on phi, c1..c3 on d_x, d_y, d_z phi)
  auto point = [&](double xi, double eta, double zeta, double W, bool nit, double nx, double ny, double nz) {
    double vx[N], dvx[N], vy[N], dvy[N], vz[N], dvz[N];
    basis_vd_sym<N>(R, xi, vx, dvx);
    basis_vd_sym<N>(R, eta, vy, dvy);
    basis_vd_sym<N>(R, zeta, vz, dvz);
    double u0 = 0.0, ux = 0.0, uy = 0.0, uz = 0.0;
#pragma unroll
    for (int c = 0; c < N; ++c) {
      double t00 = 0.0, t10 = 0.0, t01 = 0.0;
#pragma unroll
      for (int b = 0; b < N; ++b) {
        double s0 = 0.0, s1 = 0.0;
#pragma unroll
        for (int a = 0; a < N; ++a) {
          s0 = fma(vx[a], uo[(c * N + b) * N + a], s0);
          s1 = fma(dvx[a], uo[(c * N + b) * N + a], s1);
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
    double c0 = 0.0, c1, c2, c3;
    if (nit) {
      const double un = (nx * ux + ny * uy + nz * uz) * kp.ih;  // physical normal derivative
      c0 = W * (kp.tau * u0 - un);
      const double g = -W * u0 * kp.ih;
      c1 = g * nx;
      c2 = g * ny;
      c3 = g * nz;
    } else {
      const double sw = W * kp.ih2;
      c1 = sw * ux;
      c2 = sw * uy;
      c3 = sw * uz;
    }
#pragma unroll
    for (int cz = 0; cz < N; ++cz) {
      const double T0 = fma(c0, vz[cz], c3 * dvz[cz]);
      const double T1 = c2 * vz[cz];
      const double T2 = c1 * vz[cz];
#pragma unroll
      for (int by = 0; by < N; ++by) {
        const double S0 = fma(vy[by], T0, dvy[by] * T1);
        const double S1 = vy[by] * T2;
#pragma unroll
        for (int ax = 0; ax < N; ++ax) {
          double &r = acc[(cz * N + by) * N + ax];
          r = fma(vx[ax], S0, fma(dvx[ax], S1, r));
        }
      }
    }
  };
  // point rows are 32 (volume, cut face) / 64 bytes (interface) in cudaMalloc'ed arrays:
  // one / two 256-bit loads per point (CUT1_PT256; the kernel is bound by the number of
  // load instructions in flight)
  auto ld_row = [](const double *r, double2 &a, double2 &b) {
    if constexpr (CUT1_PT256) ldg256(r, a.x, a.y, b.x, b.y);
    else {
      a = __ldg(reinterpret_cast<const double2 *>(r));
      b = __ldg(reinterpret_cast<const double2 *>(r) + 1);
    }
  };
  if (cell_on && kk < d.nv) {
    const double *p = vol_pts + 4 * d.vb;
    double2 a, b;
    ld_row(p + 4 * kk, a, b);
    for (int q = kk; q < d.nv; q += TPC) {
      const double2 ca = a, cb = b;
      if (q + TPC < d.nv) ld_row(p + 4 * (q + TPC), a, b);  // the next point's row in flight while this one is evaluated
      point(ca.x, ca.y, cb.x, cb.y, false, 0.0, 0.0, 0.0);
    }
  }
  if (nit_on && kk < d.ns) {
    const double *p = srf_pts + 8 * d.sb;
    double2 a, b, c, e;
    ld_row(p + 8 * kk, a, b);
    ld_row(p + 8 * kk + 4, c, e);
    for (int q = kk; q < d.ns; q += TPC) {
      const double2 ca = a, cb = b, cc = c, ce = e;
      if (q + TPC < d.ns) {
        ld_row(p + 8 * (q + TPC), a, b);
        ld_row(p + 8 * (q + TPC) + 4, c, e);
      }
      point(ca.x, ca.y, cb.x, ce.x, true, cb.y, cc.x, cc.y);
    }
  }
  // ---- 4. cut faces
  if (sipg_on) {
    static_for<0, 6>([&](auto fc) {
      constexpr int F = decltype(fc)::value, D = F / 2, SS = F % 2;
      if (!(d.nb[F] >= 0 && ((d.flags >> (12 + F)) & 1u))) return;
      const double *nbp = u + (size_t)d.nb[F] * N3;
      constexpr int fo = SS ? N - 1 : 0, fn = SS ? 0 : N - 1;
      const double *dow = SS ? R.d1 : R.d0;
      const double *dnb = SS ? R.d0 : R.d1;
      double JA[NN], JB[NN], F1[NN], F2[NN];
#pragma unroll
      for (int t = 0; t < NN; ++t) {
        double A = 0.0;
#pragma unroll
        for (int m = 0; m < N; ++m) A = fma(dow[m], uo[lix<N, D>(t, m)], fma(dnb[m], __ldg(nbp + lix<N, D>(t, m)), A));
        JA[t] = uo[lix<N, D>(t, fo)] - __ldg(nbp + lix<N, D>(t, fn));
        JB[t] = A;
        F1[t] = F2[t] = 0.0;
      }
      const double sg = SS ? 1.0 : -1.0;
      const int64_t pb = HOIST ? fpb[F] : sf_ptr[d.sf[F]], pe = HOIST ? fpe[F] : sf_ptr[d.sf[F] + 1];
      double2 nst = make_double2(0.5, 0.5), nw = make_double2(0.0, 0.0);
      if (pb + kk < pe) ld_row(sf_pts + 4 * (pb + kk), nst, nw);
      for (int64_t q = pb + kk; q < pe; q += TPC) {
        const double2 st = nst;
        const double W = nw.x;
        if (q + TPC < pe) ld_row(sf_pts + 4 * (q + TPC), nst, nw);  // the next point's row in flight
        double ls[N], lt[N];
        basis_v_sym<N>(R, st.x, ls);
        basis_v_sym<N>(R, st.y, lt);
        double J0 = 0.0, A = 0.0;
#pragma unroll
        for (int j = 0; j < N; ++j) {
          double r0 = 0.0, r1 = 0.0;
#pragma unroll
          for (int a = 0; a < N; ++a) {
            r0 = fma(ls[a], JA[a + N * j], r0);
            r1 = fma(ls[a], JB[a + N * j], r1);
          }
          J0 = fma(lt[j], r0, J0);
          A = fma(lt[j], r1, A);
        }
        const double k1 = W * (kp.sigma * J0 - sg * A * kp.i2h), k2 = -W * sg * J0 * kp.i2h;
#pragma unroll
        for (int j = 0; j < N; ++j)
#pragma unroll
          for (int a = 0; a < N; ++a) {
            const double psi = ls[a] * lt[j];
            F1[a + N * j] = fma(psi, k1, F1[a + N * j]);
            F2[a + N * j] = fma(psi, k2, F2[a + N * j]);
          }
      }
#pragma unroll
      for (int t = 0; t < NN; ++t) {
#pragma unroll
        for (int m = 0; m < N; ++m) acc[lix<N, D>(t, m)] = fma(dow[m], F2[t], acc[lix<N, D>(t, m)]);
        acc[lix<N, D>(t, fo)] += F1[t];
      }
    });
  }
  if constexpr (TPC > 1) {
#pragma unroll
    for (int o = 1; o < TPC; o <<= 1)
#pragma unroll
      for (int k = 0; k < N3; ++k) acc[k] += __shfl_xor_sync(0xffffffffu, acc[k], o);
  }
  if (!valid) return;
  double *vb = v + (size_t)d.blk * N3;
  if constexpr (CUT1_LD128 && CELL_LD256 && TPC == 1 && (N3 % 4) == 0) {
    if ((reinterpret_cast<uintptr_t>(vb) & 31) == 0) {
#pragma unroll
      for (int k = 0; k < N3; k += 4) stg256(vb + k, acc[k], acc[k + 1], acc[k + 2], acc[k + 3]);
      return;
    }
  }
  if constexpr (CUT1_LD128) {
    // 128-bit stores on the 16-byte aligned part of the block (all of it at even n^3), the
    // pairs dealt round-robin to the cell's lanes (every lane holds the full sum)
    constexpr int H = N3 / 2;
    const bool par = (N3 % 2) && ((reinterpret_cast<uintptr_t>(vb) >> 3) & 1u) != 0;
    double2 *q = reinterpret_cast<double2 *>(vb + (par ? 1 : 0));
#pragma unroll
    for (int i = 0; i < H; ++i)
      if (TPC == 1 || i % TPC == kk)
        q[i] = par ? make_double2(acc[2 * i + 1], acc[(2 * i + 2) % N3]) : make_double2(acc[2 * i], acc[2 * i + 1]);
    if constexpr (N3 % 2 == 1) {
      if (kk == 0) vb[par ? 0 : N3 - 1] = par ? acc[0] : acc[N3 - 1];
    }
  } else {
#pragma unroll
    for (int k = 0; k < N3; ++k)
      if (TPC == 1 || k % TPC == kk) vb[k] = acc[k];
  }
}
