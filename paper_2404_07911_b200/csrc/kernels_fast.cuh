// Latency-hiding variants of the two element-centric kernels (included by
// kernels.cuh).  Both fetch the cell block and its six neighbour blocks with
// cp.async, so the neighbour traffic (L2) overlaps the volume / point work, and
// evaluate the six faces in joint phases (traces of all faces, in-face mass of
// all faces, then one gather of every face contribution into the cell's own
// block).  Face directions are compile-time constants (static_for), so the
// line addressing of every face costs no integer work at run time.
//
// k_uncut2<N> (N <= 5): structured cells, lanes = 1-D lines, 32/N^2 cells/warp.
// k_cutw<N>   (N <= 4): cut cells, one warp per cell, lanes = quadrature points,
//   per-lane register accumulators for all n^3 DoFs and a warp butterfly at the
//   end; point data (cell and cut faces) is staged through shared memory with
//   cp.async one round ahead.

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

template <int N>
__device__ __forceinline__ double pick(const double *tab, int m) {
  double r = tab[0];
#pragma unroll
  for (int k = 1; k < N; ++k)
    if (m == k) r = tab[k];
  return r;
}

// Own-side data of face (DD, side) for in-face node t, written in place into the
// neighbour's line t (the calling lane owns that line):
//   full: F[m] = GP line (G_oo u_own - G_on u_nb)[m] + SIPG spread terms
//   else: the two SIPG in-face fields F1 (line position 0) and F2 (position 1).
// JA/JB (optional) receive the jump [u]-trace and the summed normal derivatives.
template <int N, int DD>
__device__ __forceinline__ void face_trace(const double *U, double *NBf, int side, int t, bool gp, bool sipg,
                                           bool full, const KParams &kp, const FaceTab &ft,
                                           const RefTab &R, double *JA, double *JB) {
  using B = Blk<N>;
  constexpr int st = B::template lstride<DD>();
  const int b0 = B::template lbase<DD>(t);
  const double sg = side ? 1.0 : -1.0;
  const double *dow = side ? R.d1 : R.d0;
  const double *dnb = side ? R.d0 : R.d1;
  double uo[N], un[N];
#pragma unroll
  for (int m = 0; m < N; ++m) {
    uo[m] = U[b0 + m * st];
    un[m] = NBf[b0 + m * st];
  }
  const double J0 = side ? (uo[N - 1] - un[0]) : (uo[0] - un[N - 1]);
  double A0 = 0.0, A1 = 0.0;
#pragma unroll
  for (int m = 0; m < N; ++m) {
    A0 = fma(dow[m], uo[m], A0);
    A1 = fma(dnb[m], un[m], A1);
  }
  const double A = A0 + A1;
  if (JA) {
    JA[t] = J0;
    JB[t] = A;
  }
  const double h = kp.h;
  const double F1 = sipg ? h * h * (kp.sigma * J0 - sg * A / (2.0 * h)) : 0.0;
  const double F2 = sipg ? -0.5 * h * sg * J0 : 0.0;
  if (full) {
    const double *Goo = ft.Goo[side ? 0 : 1];
    const double *Gon = ft.Gon[side ? 0 : 1];
    double F[N];
#pragma unroll
    for (int m = 0; m < N; ++m) {
      double p0 = 0.0, p1 = 0.0;
      if (gp) {
#pragma unroll
        for (int a = 0; a < N; ++a) {
          p0 = fma(Goo[m * N + a], uo[a], p0);
          p1 = fma(Gon[m * N + a], un[a], p1);
        }
      }
      F[m] = fma(dow[m], F2, p0 - p1);
    }
    if (side) F[N - 1] += F1;
    else F[0] += F1;
#pragma unroll
    for (int m = 0; m < N; ++m) NBf[b0 + m * st] = F[m];
  } else {
    NBf[b0] = F1;
    NBf[b0 + st] = F2;
  }
}

// In-face mass sweep WHICH (0: along the lower in-face axis e1, 1: along e2) of
// a face with normal DD, task t.  full: line t of the whole n-layer block;
// else one line of the embedded 2-field (F1 at position 0, F2 at 1) array.
template <int N, int DD, int WHICH>
__device__ __forceinline__ void face_mass(double *NBf, int t, bool full, const RefTab &R) {
  using B = Blk<N>;
  constexpr int E1 = (DD == 0) ? 1 : 0, E2 = (DD == 2) ? 1 : 2;
  constexpr int ED = WHICH ? E2 : E1;
  if (full) {
    sweep_line<N, 0>(NBf, NBf, B::template lbase<ED>(t), B::template lstride<ED>(), R.M, 1.0);
  } else {
    if (t >= 2 * N) return;
    constexpr int st = B::template lstride<DD>();
    const int field = t / N, j = t % N;
    int base[N];
#pragma unroll
    for (int i = 0; i < N; ++i) base[i] = B::template lbase<DD>(WHICH ? (j + N * i) : (i + N * j)) + field * st;
    double in[N], out[N];
#pragma unroll
    for (int i = 0; i < N; ++i) in[i] = NBf[base[i]];
    eo_mv<N>(R.M, in, out);
#pragma unroll
    for (int i = 0; i < N; ++i) NBf[base[i]] = out[i];
  }
}

// ======================================================= structured cells
template <int N>
struct Uncut2Cfg {
  static constexpr int NN = N * N;
  static constexpr int LPS = NN;          // N <= 5: one lane per line
  static constexpr int CPW = 32 / NN;
  static constexpr int WARPS = 4;
  static constexpr int SLOT = 9 * Blk<N>::SZ;  // U, NB[6], Q, R
  static constexpr int SMEM = WARPS * CPW * SLOT * 8;
};

template <int N>
__global__ void __launch_bounds__(128) k_uncut2(const double *__restrict__ u, double *__restrict__ v,
                                                const UDesc *__restrict__ desc, int ncell, KParams kp,
                                                FaceTab ft) {
  static_assert(N * N <= 32, "k_uncut2 needs N <= 5");
  using B = Blk<N>;
  using C = Uncut2Cfg<N>;
  constexpr int NN = B::NN, N3 = B::N3, SZ = B::SZ, LPS = C::LPS;
  const RefTab &R = c_ref[N - 2];
  extern __shared__ double smem[];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int slot = lane / LPS, t = lane % LPS;
  const int cell = (blockIdx.x * C::WARPS + warp) * C::CPW + slot;
  const bool valid = slot < C::CPW && cell < ncell;
  double *base = smem + (warp * C::CPW + (slot < C::CPW ? slot : 0)) * C::SLOT;
  double *U = base, *NB = base + SZ, *Q = base + 7 * SZ, *Rb = base + 8 * SZ;

  int blk = 0;
  uint32_t act = 0, gpm = 0;  // faces with work / ghost-penalty faces
  const bool sipg = (kp.mask & TERM_SIPG) != 0;
  if (valid) {
    const UDesc d = desc[cell];
    blk = d.blk;
    const double *ub = u + (size_t)blk * N3;
    for (int l = t; l < N3; l += LPS) cp_async8(U + B::pad(l), ub + l);
    cp_async_commit();
#pragma unroll
    for (int f = 0; f < 6; ++f) {
      if (d.nb[f] < 0) continue;
      const bool g = ((d.flags >> f) & 1u) && (kp.mask & TERM_GP);
      if (!(g || sipg)) continue;
      act |= 1u << f;
      if (g) gpm |= 1u << f;
      const double *nbp = u + (size_t)d.nb[f] * N3;
      for (int l = t; l < N3; l += LPS) cp_async8(NB + f * SZ + B::pad(l), nbp + l);
    }
    cp_async_commit();
    cp_async_wait<1>();
  }
  __syncwarp();
  const double h = kp.h;
  if (kp.mask & TERM_CELL) {
    // E: GLL -> Gauss values along x, y, z
    static_for<0, 3>([&](auto dc) {
      constexpr int D = decltype(dc)::value;
      if (valid)
        sweep_line<N, 0>(D == 0 ? U : Q, Q, B::template lbase<D>(t), B::template lstride<D>(), R.S, 1.0);
      __syncwarp();
    });
    // B: collocation derivative, weight h w w w and its transpose, per direction
    static_for<0, 3>([&](auto dc) {
      constexpr int D = decltype(dc)::value;
      if (valid) {
        const double s = h * R.gw[t % N] * R.gw[t / N];
        if (D == 0) sweep_line<N, 2>(Q, Rb, B::template lbase<D>(t), B::template lstride<D>(), R.Kc, s);
        else sweep_line<N, 1>(Q, Rb, B::template lbase<D>(t), B::template lstride<D>(), R.Kc, s);
      }
      __syncwarp();
    });
    // I: Gauss -> GLL
    static_for<0, 3>([&](auto dc) {
      constexpr int D = decltype(dc)::value;
      if (valid) sweep_line<N, 0>(Rb, Rb, B::template lbase<D>(t), B::template lstride<D>(), R.St, 1.0);
      __syncwarp();
    });
  } else {
    if (valid)
      for (int l = t; l < SZ; l += LPS) Rb[l] = 0.0;
  }
  if (valid) cp_async_wait<0>();
  __syncwarp();
  // ---- faces, all six at once
  if (valid)
    static_for<0, 6>([&](auto fc) {
      constexpr int F = decltype(fc)::value;
      if ((act >> F) & 1u) {
        const bool g = (gpm >> F) & 1u;
        face_trace<N, F / 2>(U, NB + F * SZ, F & 1, t, g, sipg, g, kp, ft, R, nullptr, nullptr);
      }
    });
  __syncwarp();
  static_for<0, 2>([&](auto wc) {
    constexpr int W = decltype(wc)::value;
    if (valid)
      static_for<0, 6>([&](auto fc) {
        constexpr int F = decltype(fc)::value;
        if ((act >> F) & 1u) face_mass<N, F / 2, W>(NB + F * SZ, t, (gpm >> F) & 1u, R);
      });
    __syncwarp();
  });
  if (valid) {
    double *vb = v + (size_t)blk * N3;
    for (int l = t; l < N3; l += LPS) {
      const int a = l % N, b = (l / N) % N, c = l / NN;
      const int pl = B::at(a, b, c);
      double acc = Rb[pl];
      static_for<0, 6>([&](auto fc) {
        constexpr int F = decltype(fc)::value, DD = F / 2, SIDE = F & 1;
        if ((act >> F) & 1u) {
          const double *NBf = NB + F * SZ;
          if ((gpm >> F) & 1u) {
            acc += NBf[pl];
          } else {
            const int m = DD == 0 ? a : (DD == 1 ? b : c);
            const int tt = DD == 0 ? (b + N * c) : (DD == 1 ? (a + N * c) : (a + N * b));
            const int b0 = B::template lbase<DD>(tt);
            acc = fma(pick<N>(SIDE ? R.d1 : R.d0, m), NBf[b0 + B::template lstride<DD>()], acc);
            if (m == (SIDE ? N - 1 : 0)) acc += NBf[b0];
          }
        }
      });
      vb[l] = acc;
    }
  }
}

// ============================================================ cut cells
template <int N>
struct CutWCfg {
  static constexpr int WARPS = 4;
  static constexpr int NN = N * N, N3 = N * N * N;
  static constexpr int ACC = N == 4 ? 64 : (N == 3 ? 32 : 8);
  static constexpr int ACC2 = N == 4 ? 32 : (N == 3 ? 32 : 8);
  static constexpr int PROW = 8;          // doubles per staged cell point
  static constexpr int FROW = 4;          // doubles per staged face point
  static constexpr int FARR = 4 * NN;     // JA, JB, FC1, FC2 per face
  static constexpr int WSLOT = 8 * Blk<N>::SZ + 6 * FARR + 2 * 32 * PROW + 6 * 32 * FROW;
  static constexpr int SMEM = WARPS * WSLOT * 8;
};

template <int N>
__global__ void __launch_bounds__(128) k_cutw(const double *__restrict__ u, double *__restrict__ v,
                                              const CDesc *__restrict__ desc, int ncut,
                                              const double *__restrict__ vol_pts,
                                              const int64_t *__restrict__ vol_ptr,
                                              const double *__restrict__ srf_pts,
                                              const int64_t *__restrict__ srf_ptr,
                                              const double *__restrict__ sf_pts,
                                              const int64_t *__restrict__ sf_ptr, KParams kp, FaceTab ft) {
  static_assert(2 * N * N <= 32, "k_cutw needs N <= 4");
  using B = Blk<N>;
  using C = CutWCfg<N>;
  constexpr int NN = B::NN, N3 = B::N3, SZ = B::SZ;
  const RefTab &R = c_ref[N - 2];
  extern __shared__ double smem[];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int cell = blockIdx.x * C::WARPS + warp;
  if (cell >= ncut) return;
  double *base = smem + warp * C::WSLOT;
  double *U = base, *NB = base + SZ, *Rb = base + 7 * SZ, *FAR = base + 8 * SZ;
  double *PB = FAR + 6 * C::FARR;   // [2][32][PROW] cell points
  double *FPB = PB + 2 * 32 * C::PROW;  // [6][32][FROW] first face points
  const CDesc dsc = desc[cell];
  const bool sipg_on = (kp.mask & TERM_SIPG) != 0, gp_on = (kp.mask & TERM_GP) != 0;
  uint32_t nbm = 0;
#pragma unroll
  for (int f = 0; f < 6; ++f)
    if (dsc.nb[f] >= 0) nbm |= 1u << f;
  const uint32_t gpm = gp_on ? (dsc.flags & 0x3fu & nbm) : 0u;
  const uint32_t ssm = sipg_on ? ((dsc.flags >> 6) & 0x3fu & nbm) : 0u;
  const uint32_t scm = sipg_on ? ((dsc.flags >> 12) & 0x3fu & nbm) : 0u;
  const uint32_t act = gpm | ssm | scm, stm = gpm | ssm;

  const int64_t vb = dsc.vb, sb = dsc.sb;
  const int nv = (kp.mask & TERM_CELL) ? dsc.nv : 0;
  const int ns = (kp.mask & TERM_NITSCHE) ? dsc.ns : 0;
  const int total = nv + ns;
  auto stage = [&](int q0, int buf) {  // lane-private copy of its point's data
    const int q = q0 + lane;
    double *dst = PB + (buf * 32 + lane) * C::PROW;
    if (q < nv) {
      const double *src = vol_pts + 4 * (vb + q);
#pragma unroll
      for (int k = 0; k < 4; ++k) cp_async8(dst + k, src + k);
    } else if (q < total) {
      const double *src = srf_pts + 7 * (sb + q - nv);
#pragma unroll
      for (int k = 0; k < 7; ++k) cp_async8(dst + k, src + k);
    }
  };
  auto issue_neighbours = [&]() {
#pragma unroll
    for (int f = 0; f < 6; ++f) {
      if (!((act >> f) & 1u)) continue;
      const double *nbp = u + (size_t)dsc.nb[f] * N3;
      for (int l = lane; l < N3; l += 32) cp_async8(NB + f * SZ + B::pad(l), nbp + l);
      if ((scm >> f) & 1u) {  // first 32 points of the cut face
        const int64_t pb = sf_ptr[dsc.sf[f]], pe = sf_ptr[dsc.sf[f] + 1];
        if (pb + lane < pe) {
          const double *src = sf_pts + 3 * (pb + lane);
          double *dst = FPB + (f * 32 + lane) * C::FROW;
#pragma unroll
          for (int k = 0; k < 3; ++k) cp_async8(dst + k, src + k);
        }
      }
    }
  };
  {
    const double *ub = u + (size_t)dsc.blk * N3;
    for (int l = lane; l < N3; l += 32) cp_async8(U + B::pad(l), ub + l);
    if (total > 0) stage(0, 0);
    cp_async_commit();  // group: U + first point chunk
  }
  const double h = kp.h, ih = 1.0 / h, ih2 = ih * ih;
  bool nb_issued = false;
  {
    double acc[C::ACC];
#pragma unroll
    for (int i = 0; i < C::ACC; ++i) acc[i] = 0.0;
    cp_async_wait<0>();
    __syncwarp();
    int buf = 0;
    for (int q0 = 0; q0 < total; q0 += 32, buf ^= 1) {
      // the neighbour blocks travel with the last staged chunk, so they land
      // while the last round(s) of point work run
      if (!nb_issued && q0 + 64 >= total) {
        issue_neighbours();
        nb_issued = true;
      }
      if (q0 + 32 < total) stage(q0 + 32, buf ^ 1);
      cp_async_commit();
      cp_async_wait<1>();  // the current chunk has landed (own lane's copies)
      const int q = q0 + lane;
      const double *pp = PB + (buf * 32 + lane) * C::PROW;
      double xi = 0.5, eta = 0.5, zeta = 0.5, W = 0.0, nx = 0.0, ny = 0.0, nz = 0.0;
      const bool srf = q >= nv && q < total;
      if (q < nv) {
        xi = pp[0];
        eta = pp[1];
        zeta = pp[2];
        W = pp[3];
      } else if (srf) {
        xi = pp[0];
        eta = pp[1];
        zeta = pp[2];
        nx = pp[3];
        ny = pp[4];
        nz = pp[5];
        W = pp[6];
      }
      double vx[N], dvx[N], vy[N], dvy[N], vz[N], dvz[N];
      basis_vd<N>(R, xi, vx, dvx);
      basis_vd<N>(R, eta, vy, dvy);
      basis_vd<N>(R, zeta, vz, dvz);
      double u0, ux, uy, uz;
      eval_point<N>(U, vx, dvx, vy, dvy, vz, dvz, u0, ux, uy, uz);
      double c0v, c1, c2, c3;
      if (srf) {
        const double un = (nx * ux + ny * uy + nz * uz) * ih;
        c0v = W * (kp.tau * u0 - un);
        const double g = -W * u0 * ih;
        c1 = g * nx;
        c2 = g * ny;
        c3 = g * nz;
      } else {
        c0v = 0.0;
        const double s = W * ih2;
        c1 = s * ux;
        c2 = s * uy;
        c3 = s * uz;
      }
#pragma unroll
      for (int c = 0; c < N; ++c) {
        const double T0 = fma(c0v, vz[c], c3 * dvz[c]);
        const double T1 = c2 * vz[c];
        const double T2 = c1 * vz[c];
#pragma unroll
        for (int b = 0; b < N; ++b) {
          const double S0 = fma(vy[b], T0, dvy[b] * T1);
          const double S1 = vy[b] * T2;
#pragma unroll
          for (int a = 0; a < N; ++a) {
            double &r = acc[(c * N + b) * N + a];
            r = fma(vx[a], S0, fma(dvx[a], S1, r));
          }
        }
      }
    }
    butterfly<C::ACC>(acc, lane);
    if (BF<C::ACC>::writer(lane)) {
#pragma unroll
      for (int j = 0; j < BF<C::ACC>::LF; ++j) {
        const int l = BF<C::ACC>::idx(lane, j);
        if (l < N3) Rb[B::pad(l)] = acc[j];
      }
    }
  }
  if (!nb_issued) {
    issue_neighbours();
    cp_async_commit();
  }
  cp_async_wait<0>();
  __syncwarp();
  // ---------------- faces: traces, 2 faces (lo, hi) of one axis per pass
  const int fside = lane >= NN ? 1 : 0, ft_t = lane - fside * NN;
  static_for<0, 3>([&](auto dc) {
    constexpr int DD = decltype(dc)::value;
    const int f = 2 * DD + fside;
    if (lane < 2 * NN && ((act >> f) & 1u)) {
      double *fa = FAR + f * C::FARR;
      face_trace<N, DD>(U, NB + f * SZ, fside, ft_t, (gpm >> f) & 1u, (ssm >> f) & 1u, (stm >> f) & 1u, kp,
                        ft, R, fa, fa + NN);
    }
  });
  __syncwarp();
  static_for<0, 2>([&](auto wc) {
    constexpr int W = decltype(wc)::value;
    static_for<0, 3>([&](auto dc) {
      constexpr int DD = decltype(dc)::value;
      const int f = 2 * DD + fside;
      if (lane < 2 * NN && ((stm >> f) & 1u)) face_mass<N, DD, W>(NB + f * SZ, ft_t, true, R);
    });
    __syncwarp();
  });
  // ---------------- cut faces: in-face unstructured quadrature
  for (int f = 0; f < 6; ++f) {
    if (!((scm >> f) & 1u)) continue;
    double *JA = FAR + f * C::FARR, *JB = JA + NN, *FC1 = JB + NN, *FC2 = FC1 + NN;
    const double sg = (f & 1) ? 1.0 : -1.0;
    const int sfi = __ldg(&desc[cell].sf[f]);
    const int64_t pb = __ldg(sf_ptr + sfi), pe = __ldg(sf_ptr + sfi + 1);
    double fa[C::ACC2];
#pragma unroll
    for (int i = 0; i < C::ACC2; ++i) fa[i] = 0.0;
    for (int64_t q0 = pb; q0 < pe; q0 += 32) {
      const int64_t q = q0 + lane;
      double s = 0.5, tt = 0.5, W = 0.0;
      if (q < pe) {
        if (q0 == pb) {
          const double *pp = FPB + (f * 32 + lane) * C::FROW;
          s = pp[0];
          tt = pp[1];
          W = pp[2];
        } else {
          s = __ldg(sf_pts + 3 * q);
          tt = __ldg(sf_pts + 3 * q + 1);
          W = __ldg(sf_pts + 3 * q + 2);
        }
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
      const double k1 = W * (kp.sigma * J0 - sg * A / (2.0 * h));
      const double k2 = -W * sg * J0 / (2.0 * h);
#pragma unroll
      for (int j = 0; j < N; ++j) {
        const double a1 = lt[j] * k1, a2 = lt[j] * k2;
#pragma unroll
        for (int i = 0; i < N; ++i) {
          fa[i + N * j] = fma(ls[i], a1, fa[i + N * j]);
          fa[NN + i + N * j] = fma(ls[i], a2, fa[NN + i + N * j]);
        }
      }
    }
    butterfly<C::ACC2>(fa, lane);
    if (BF<C::ACC2>::writer(lane)) {
#pragma unroll
      for (int j = 0; j < BF<C::ACC2>::LF; ++j) {
        const int l = BF<C::ACC2>::idx(lane, j);
        if (l < NN) FC1[l] = fa[j];
        else if (l < 2 * NN) FC2[l - NN] = fa[j];
      }
    }
  }
  __syncwarp();
  // ---------------- gather every face contribution into the cell block
  double *vbk = v + (size_t)dsc.blk * N3;
  for (int l = lane; l < N3; l += 32) {
    const int a = l % N, b = (l / N) % N, c = l / NN;
    const int pl = B::at(a, b, c);
    double accv = Rb[pl];
    static_for<0, 6>([&](auto fc) {
      constexpr int F = decltype(fc)::value, DD = F / 2, SIDE = F & 1;
      if ((stm >> F) & 1u) accv += NB[F * SZ + pl];
      if ((scm >> F) & 1u) {
        const int m = DD == 0 ? a : (DD == 1 ? b : c);
        const int tt = DD == 0 ? (b + N * c) : (DD == 1 ? (a + N * c) : (a + N * b));
        const double *FC1 = FAR + F * C::FARR + 2 * NN, *FC2 = FC1 + NN;
        accv = fma(pick<N>(SIDE ? R.d1 : R.d0, m), FC2[tt], accv);
        if (m == (SIDE ? N - 1 : 0)) accv += FC1[tt];
      }
    });
    vbk[l] = accv;
  }
}
