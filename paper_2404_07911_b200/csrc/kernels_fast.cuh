// Latency-hiding variants of the two element-centric kernels (included by
// kernels.cuh).
//
//  - Data movement: the cell block and its six neighbour blocks (and, in the
//    unstructured kernel, the quadrature-point lists) are brought into shared
//    memory by TMA bulk copies (cp.async.bulk ... mbarrier::complete_tx, SASS
//    UBLKCP) issued by one lane, completion tracked by mbarriers, so the L2
//    traffic overlaps the volume / point work and costs no per-element load
//    instructions.  (Odd n: blocks are not 16-byte multiples, so those fall back
//    to 8-byte cp.async.)
//  - Faces: the six faces are evaluated in joint phases (traces of all faces,
//    in-face mass of all faces, then the contributions are added into the
//    cell's own block line by line).  Face directions are compile-time
//    constants (static_for), so face addressing costs no run-time integer work.
//
// k_uncut2<N> (N <= 5): structured cells, lanes = 1-D lines, 32/N^2 cells/warp.
// k_cutw<N>   (N <= 4): cut cells, one warp per cell, lanes = quadrature points,
//   per-lane register accumulators for all n^3 DoFs, reduced over the warp by a
//   padded shared-memory transpose at the end.

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

// Own-side data of face (DD, side) for in-face node t, written in place into the
// neighbour's line t (the calling lane owns that line):
//   full: F[m] = GP line (G_oo u_own - G_on u_nb)[m] + SIPG spread terms
//   else: the two SIPG in-face fields F1 (line position 0) and F2 (position 1).
// JA/JB (optional) receive the jump [u]-trace and the summed normal derivatives.
template <int N, int DD, class LU, class LN>
__device__ __forceinline__ void face_trace(const double *U, double *NBf, int side, int t, bool gp, bool sipg,
                                           bool full, const KParams &kp, const FaceTab &ft,
                                           const RefTab &R, double *JA, double *JB) {
  constexpr int su = LU::template lstride<DD>(), sn = LN::template lstride<DD>();
  const int bu = LU::template lbase<DD>(t), bn = LN::template lbase<DD>(t);
  const double sg = side ? 1.0 : -1.0;
  const double *dow = side ? R.d1 : R.d0;
  const double *dnb = side ? R.d0 : R.d1;
  double uo[N], un[N];
#pragma unroll
  for (int m = 0; m < N; ++m) {
    uo[m] = U[bu + m * su];
    un[m] = NBf[bn + m * sn];
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
  // F1 = h^2 (sigma [u] - {d_n u}), F2 = -(h/2) [v]-sign * [u]
  const double F1 = sipg ? fma(kp.h2sig, J0, -sg * kp.hh * A) : 0.0;
  const double F2 = sipg ? -sg * kp.hh * J0 : 0.0;
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
    for (int m = 0; m < N; ++m) NBf[bn + m * sn] = F[m];
  } else {
    NBf[bn] = F1;
    NBf[bn + sn] = F2;
  }
}

// In-face mass sweep WHICH (0: along the lower in-face axis e1, 1: along e2) of
// a face with normal DD, task t.  full: line t of the whole n-layer block;
// else one line of the embedded 2-field (F1 at position 0, F2 at 1) array.
template <int N, int DD, int WHICH, class LN>
__device__ __forceinline__ void face_mass(double *NBf, int t, bool full, const RefTab &R) {
  constexpr int E1 = (DD == 0) ? 1 : 0, E2 = (DD == 2) ? 1 : 2;
  constexpr int ED = WHICH ? E2 : E1;
  if (full) {
    sweep_line<N, 0>(NBf, NBf, LN::template lbase<ED>(t), LN::template lstride<ED>(), R.M, 1.0);
  } else {
    if (t >= 2 * N) return;
    constexpr int st = LN::template lstride<DD>();
    const int field = t / N, j = t % N;
    int base[N];
#pragma unroll
    for (int i = 0; i < N; ++i) base[i] = LN::template lbase<DD>(WHICH ? (j + N * i) : (i + N * j)) + field * st;
    double in[N], out[N];
#pragma unroll
    for (int i = 0; i < N; ++i) in[i] = NBf[base[i]];
    eo_mv<N>(R.M, in, out);
#pragma unroll
    for (int i = 0; i < N; ++i) NBf[base[i]] = out[i];
  }
}

// Add the own-side contributions of the two faces of axis DD to line t (along
// DD) of the padded accumulator block: full faces add the whole mass-applied
// line, SIPG-only faces add F1 at the face node and l'_m(face) F2 along the line.
template <int N, int DD, class LN>
__device__ __forceinline__ void face_accumulate(double *Rb, const double *NB, int t, uint32_t act, uint32_t full,
                                                const RefTab &R) {
  using B = Blk<N>;
  constexpr int sr = B::template lstride<DD>(), sn = LN::template lstride<DD>();
  constexpr int SZN = LN::SZ;
  const int br = B::template lbase<DD>(t), bn = LN::template lbase<DD>(t);
  double r[N];
#pragma unroll
  for (int m = 0; m < N; ++m) r[m] = Rb[br + m * sr];
#pragma unroll
  for (int side = 0; side < 2; ++side) {
    const int f = 2 * DD + side;
    if (!((act >> f) & 1u)) continue;
    const double *NBf = NB + f * SZN;
    if ((full >> f) & 1u) {
#pragma unroll
      for (int m = 0; m < N; ++m) r[m] += NBf[bn + m * sn];
    } else {
      const double F1 = NBf[bn], F2 = NBf[bn + sn];
      const double *dw = side ? R.d1 : R.d0;
#pragma unroll
      for (int m = 0; m < N; ++m) r[m] = fma(dw[m], F2, r[m]);
      r[side ? N - 1 : 0] += F1;
    }
  }
#pragma unroll
  for (int m = 0; m < N; ++m) Rb[br + m * sr] = r[m];
}

// ======================================================= structured cells
template <int N>
struct Uncut2Cfg {
  static constexpr bool BULK = CUTFEM_USE_BULK && (N % 2) == 0;   // blocks are 16-byte multiples
  using LN = typename std::conditional<BULK, BlkU<N>, Blk<N>>::type;  // U / NB layout
  static constexpr int NN = N * N, N3 = N * N * N;
  static constexpr int LPS = NN;               // N <= 5: one lane per line
  static constexpr int CPW = 32 / NN;
  static constexpr int WARPS = 4;
  static constexpr int SLOT0 = 2 + 7 * LN::SZ + 2 * Blk<N>::SZ;  // bars, U, NB[6], Q, R
  static constexpr int SLOT = (SLOT0 + 1) & ~1;                 // 16-byte multiple
  static constexpr int SMEM = WARPS * CPW * SLOT * 8;
};

template <int N>
__global__ void __launch_bounds__(128) k_uncut2(const double *__restrict__ u, double *__restrict__ v,
                                                const UDesc *__restrict__ desc, int ncell, KParams kp,
                                                FaceTab ft) {
  static_assert(N * N <= 32, "k_uncut2 needs N <= 5");
  using B = Blk<N>;
  using C = Uncut2Cfg<N>;
  using LN = typename C::LN;
  constexpr int NN = B::NN, N3 = B::N3, SZ = B::SZ, SZN = LN::SZ, LPS = C::LPS;
  const RefTab &R = c_ref[N - 2];
  extern __shared__ __align__(16) double smem[];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int slot = lane / LPS, t = lane % LPS;
  const int cell = (blockIdx.x * C::WARPS + warp) * C::CPW + slot;
  const bool valid = slot < C::CPW && cell < ncell;
  double *base = smem + (warp * C::CPW + (slot < C::CPW ? slot : 0)) * C::SLOT;
  uint64_t *bar = reinterpret_cast<uint64_t *>(base);
  double *U = base + 2, *NB = U + SZN, *Q = NB + 6 * SZN, *Rb = Q + SZ;

  int blk = 0;
  uint32_t act = 0, gpm = 0;  // faces with work / ghost-penalty faces
  const bool sipg = (kp.mask & TERM_SIPG) != 0;
  int nbk[6];
  if (valid) {
    const UDesc d = desc[cell];
    blk = d.blk;
#pragma unroll
    for (int f = 0; f < 6; ++f) {
      nbk[f] = d.nb[f];
      if (d.nb[f] < 0) continue;
      const bool g = ((d.flags >> f) & 1u) && (kp.mask & TERM_GP);
      if (!(g || sipg)) continue;
      act |= 1u << f;
      if (g) gpm |= 1u << f;
    }
  }
  if constexpr (C::BULK) {
    if (valid && t == 0) {
      mbar_init(bar, 1);
      mbar_init(bar + 1, 1);
      mbar_fence_init();
    }
    __syncwarp();
    if (valid && t == 0) {
      mbar_expect_tx(bar, N3 * 8);
      bulk_g2s(U, u + (size_t)blk * N3, N3 * 8, bar);
      mbar_expect_tx(bar + 1, __popc(act) * N3 * 8);
#pragma unroll
      for (int f = 0; f < 6; ++f)
        if ((act >> f) & 1u) bulk_g2s(NB + f * SZN, u + (size_t)nbk[f] * N3, N3 * 8, bar + 1);
    }
    if (valid) mbar_wait(bar, 0);
  } else {
    if (valid) {
      const double *ub = u + (size_t)blk * N3;
      for (int l = t; l < N3; l += LPS) cp_async8(U + LN::at(l % N, (l / N) % N, l / NN), ub + l);
      cp_async_commit();
#pragma unroll
      for (int f = 0; f < 6; ++f) {
        if (!((act >> f) & 1u)) continue;
        const double *nbp = u + (size_t)nbk[f] * N3;
        for (int l = t; l < N3; l += LPS) cp_async8(NB + f * SZN + LN::at(l % N, (l / N) % N, l / NN), nbp + l);
      }
      cp_async_commit();
      cp_async_wait<1>();
    }
  }
  __syncwarp();
  const double h = kp.h;
  if (kp.mask & TERM_CELL) {
    // E: GLL -> Gauss values along x (U -> Q), y, z
    if (valid) {
      double in[N], out[N];
      const int bu = LN::template lbase<0>(t);
#pragma unroll
      for (int k = 0; k < N; ++k) in[k] = U[bu + k];
      eo_mv<N>(R.S, in, out);
      const int bq = B::template lbase<0>(t);
#pragma unroll
      for (int k = 0; k < N; ++k) Q[bq + k] = out[k];
    }
    __syncwarp();
    static_for<1, 3>([&](auto dc) {
      constexpr int D = decltype(dc)::value;
      if (valid) sweep_line<N, 0>(Q, Q, B::template lbase<D>(t), B::template lstride<D>(), R.S, 1.0);
      __syncwarp();
    });
    // B: collocation derivative, weight h w w w and its transpose, per direction
    const double s = h * R.gw[t % N] * R.gw[t / N];
    static_for<0, 3>([&](auto dc) {
      constexpr int D = decltype(dc)::value;
      if (valid) {
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
  if constexpr (C::BULK) {
    if (valid) mbar_wait(bar + 1, 0);
  } else {
    if (valid) cp_async_wait<0>();
  }
  __syncwarp();
  // ---- faces, all six at once
  if (valid)
    static_for<0, 6>([&](auto fc) {
      constexpr int F = decltype(fc)::value;
      if ((act >> F) & 1u) {
        const bool g = (gpm >> F) & 1u;
        face_trace<N, F / 2, LN, LN>(U, NB + F * SZN, F & 1, t, g, sipg, g, kp, ft, R, nullptr, nullptr);
      }
    });
  __syncwarp();
  static_for<0, 2>([&](auto wc) {
    constexpr int W = decltype(wc)::value;
    if (valid)
      static_for<0, 6>([&](auto fc) {
        constexpr int F = decltype(fc)::value;
        if ((act >> F) & 1u) face_mass<N, F / 2, W, LN>(NB + F * SZN, t, (gpm >> F) & 1u, R);
      });
    __syncwarp();
  });
  static_for<0, 3>([&](auto dc) {
    constexpr int DD = decltype(dc)::value;
    if (valid) face_accumulate<N, DD, LN>(Rb, NB, t, act, gpm, R);
    __syncwarp();
  });
  if (valid) {
    double *vb = v + (size_t)blk * N3;
    for (int l = t; l < N3; l += LPS) vb[l] = Rb[B::pad(l)];
  }
}

// ============================================================ cut cells
template <int N>
struct CutWCfg {
  static constexpr bool BULK = CUTFEM_USE_BULK && (N % 2) == 0;
  using LN = typename std::conditional<BULK, BlkU<N>, Blk<N>>::type;
  static constexpr int WARPS = 4;
  static constexpr int NN = N * N, N3 = N * N * N;
  static constexpr int ACC = N == 4 ? 64 : (N == 3 ? 32 : 8);   // padded n^3
  static constexpr int ACC2 = N == 4 ? 32 : (N == 3 ? 32 : 8);  // padded 2 n^2
  static constexpr int RROWS = ACC < 32 ? ACC : 32;             // reduction rows per pass
  static constexpr int FARR = 4 * NN;                           // JA, JB, FC1, FC2 per face
  // bars(4) | U | NB[6] | R(padded) | FAR[6] | face points [6][32][4]
  // | { vol chunk [2][32][4], srf chunk [2][32][8] } aliased with reduction [RROWS][33]
  static constexpr int OFF_U = 4;
  static constexpr int OFF_NB = OFF_U + LN::SZ + (LN::SZ & 1);
  static constexpr int OFF_R = OFF_NB + 6 * LN::SZ + ((6 * LN::SZ) & 1);
  static constexpr int OFF_FAR = OFF_R + Blk<N>::SZ + (Blk<N>::SZ & 1);
  static constexpr int OFF_FP = OFF_FAR + 6 * FARR;
  static constexpr int OFF_PV = OFF_FP + 6 * 32 * 4;
  static constexpr int OFF_PS = OFF_PV + 2 * 32 * 4;
  static constexpr int OFF_RB = OFF_PV;
  static constexpr int END0 = (OFF_PS + 2 * 32 * 8) > (OFF_RB + RROWS * 33) ? (OFF_PS + 2 * 32 * 8)
                                                                              : (OFF_RB + RROWS * 33);
  static constexpr int WSLOT = (END0 + 1) & ~1;
  static constexpr int SMEM = WARPS * WSLOT * 8;
};

// Warp sum of L per-lane partial sums through a padded shared-memory transpose:
// lane l ends with the total of entry (pass*32 + l).  Writes `out[l]` for l < LIM.
template <int L, int ROWS, class OutF>
__device__ __forceinline__ void warp_reduce_smem(const double (&a)[L], double *RB, int lane, OutF &&out) {
#pragma unroll
  for (int p = 0; p < L / ROWS; ++p) {
#pragma unroll
    for (int i = 0; i < ROWS; ++i) RB[i * 33 + lane] = a[p * ROWS + i];
    __syncwarp();
    if (lane < ROWS) {
      double s0 = 0.0, s1 = 0.0, s2 = 0.0, s3 = 0.0;
#pragma unroll
      for (int k = 0; k < 32; k += 4) {
        s0 += RB[lane * 33 + k];
        s1 += RB[lane * 33 + k + 1];
        s2 += RB[lane * 33 + k + 2];
        s3 += RB[lane * 33 + k + 3];
      }
      out(p * ROWS + lane, (s0 + s1) + (s2 + s3));
    }
    __syncwarp();
  }
}

// STRUCT = false: the structured faces of the cut cell (full-face SIPG next to
// uncut cells, ghost penalty) are left to k_tile*<MODE 1>, which adds them
// afterwards; this kernel then does the points and the cut faces only.
template <int N, bool STRUCT = true>
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
  using LN = typename C::LN;
  constexpr int NN = B::NN, N3 = B::N3, SZN = LN::SZ;
  const RefTab &R = c_ref[N - 2];
  extern __shared__ __align__(16) double smem[];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int cell = blockIdx.x * C::WARPS + warp;
  if (cell >= ncut) return;
  double *base = smem + warp * C::WSLOT;
  uint64_t *bar = reinterpret_cast<uint64_t *>(base);  // 0: U, 1: neighbours, 2/3: point chunks
  double *U = base + C::OFF_U, *NB = base + C::OFF_NB, *Rb = base + C::OFF_R, *FAR = base + C::OFF_FAR;
  double *PV = base + C::OFF_PV, *PS = base + C::OFF_PS, *FP = base + C::OFF_FP, *RB = base + C::OFF_RB;
  const CDesc dsc = desc[cell];
  const bool sipg_on = (kp.mask & TERM_SIPG) != 0, gp_on = (kp.mask & TERM_GP) != 0;
  uint32_t nbm = 0;
#pragma unroll
  for (int f = 0; f < 6; ++f)
    if (dsc.nb[f] >= 0) nbm |= 1u << f;
  const uint32_t gpm = (STRUCT && gp_on) ? (dsc.flags & 0x3fu & nbm) : 0u;
  const uint32_t ssm = (STRUCT && sipg_on) ? ((dsc.flags >> 6) & 0x3fu & nbm) : 0u;
  const uint32_t scm = sipg_on ? ((dsc.flags >> 12) & 0x3fu & nbm) : 0u;
  const uint32_t act = gpm | ssm | scm, stm = gpm | ssm;

  const int64_t vb = dsc.vb, sb = dsc.sb;
  const int nv = (kp.mask & TERM_CELL) ? dsc.nv : 0;
  const int ns = (kp.mask & TERM_NITSCHE) ? dsc.ns : 0;
  const int total = nv + ns;
  // chunk k covers stream points [32k, 32k+32): volume rows then interface rows
  auto issue_chunk = [&](int q0, int b) {  // lane 0 only
    const int cv = max(0, min(32, nv - q0));
    const int qs = max(0, q0 - nv);
    const int cs = max(0, min(32 - cv, ns - qs));
    mbar_expect_tx(bar + 2 + b, (uint32_t)(cv * 32 + cs * 64));
    if (cv) bulk_g2s(PV + b * 128, vol_pts + 4 * (vb + q0), (uint32_t)(cv * 32), bar + 2 + b);
    if (cs) bulk_g2s(PS + b * 256, srf_pts + 8 * (sb + qs), (uint32_t)(cs * 64), bar + 2 + b);
  };
  if (lane == 0) {
#pragma unroll
    for (int i = 0; i < 4; ++i) mbar_init(bar + i, 1);
    mbar_fence_init();
  }
  __syncwarp();
  if (lane == 0) {
    if constexpr (C::BULK) {
      mbar_expect_tx(bar, N3 * 8);
      bulk_g2s(U, u + (size_t)dsc.blk * N3, N3 * 8, bar);
    }
    if (total > 0) issue_chunk(0, 0);
    // neighbours + first points of each cut face (overlap with the point work)
    uint32_t bytes = C::BULK ? __popc(act) * N3 * 8 : 0;
    int64_t fpb[6];
    int fcnt[6];
#pragma unroll
    for (int f = 0; f < 6; ++f) {
      fcnt[f] = 0;
      fpb[f] = 0;
      if ((scm >> f) & 1u) {
        fpb[f] = sf_ptr[dsc.sf[f]];
        fcnt[f] = (int)min((int64_t)32, sf_ptr[dsc.sf[f] + 1] - fpb[f]);
        bytes += fcnt[f] * 32;
      }
    }
    mbar_expect_tx(bar + 1, bytes);
#pragma unroll
    for (int f = 0; f < 6; ++f) {
      if (C::BULK && ((act >> f) & 1u)) bulk_g2s(NB + f * SZN, u + (size_t)dsc.nb[f] * N3, N3 * 8, bar + 1);
      if (fcnt[f]) bulk_g2s(FP + f * 128, sf_pts + 4 * fpb[f], (uint32_t)(fcnt[f] * 32), bar + 1);
    }
  }
  if constexpr (!C::BULK) {
    const double *ub = u + (size_t)dsc.blk * N3;
    for (int l = lane; l < N3; l += 32) cp_async8(U + LN::at(l % N, (l / N) % N, l / NN), ub + l);
    cp_async_commit();
#pragma unroll
    for (int f = 0; f < 6; ++f) {
      if (!((act >> f) & 1u)) continue;
      const double *nbp = u + (size_t)dsc.nb[f] * N3;
      for (int l = lane; l < N3; l += 32) cp_async8(NB + f * SZN + LN::at(l % N, (l / N) % N, l / NN), nbp + l);
    }
    cp_async_commit();
    cp_async_wait<1>();
    __syncwarp();
  } else {
    mbar_wait(bar, 0);
  }
  const double ih = kp.ih, ih2 = kp.ih2;
  {
    double acc[C::ACC];
#pragma unroll
    for (int i = 0; i < C::ACC; ++i) acc[i] = 0.0;
    int k = 0;
    for (int q0 = 0; q0 < total; q0 += 32, ++k) {
      const int b = k & 1;
      if (lane == 0 && q0 + 32 < total) issue_chunk(q0 + 32, b ^ 1);
      mbar_wait(bar + 2 + b, (k >> 1) & 1);
      const int q = q0 + lane;
      const int cv = max(0, min(32, nv - q0));
      double xi = 0.5, eta = 0.5, zeta = 0.5, W = 0.0, nx = 0.0, ny = 0.0, nz = 0.0;
      const bool srf = q >= nv && q < total;
      if (q < nv) {
        const double2 p0 = *reinterpret_cast<const double2 *>(PV + b * 128 + 4 * lane);
        const double2 p1 = *reinterpret_cast<const double2 *>(PV + b * 128 + 4 * lane + 2);
        xi = p0.x;
        eta = p0.y;
        zeta = p1.x;
        W = p1.y;
      } else if (srf) {
        const double *pp = PS + b * 256 + 8 * (lane - cv);
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
      double vx[N], dvx[N], vy[N], dvy[N], vz[N], dvz[N];
      basis_vd<N>(R, xi, vx, dvx);
      basis_vd<N>(R, eta, vy, dvy);
      basis_vd<N>(R, zeta, vz, dvz);
      double u0, ux, uy, uz;
      eval_point_l<N, LN>(U, vx, dvx, vy, dvy, vz, dvz, u0, ux, uy, uz);
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
        for (int bb = 0; bb < N; ++bb) {
          const double S0 = fma(vy[bb], T0, dvy[bb] * T1);
          const double S1 = vy[bb] * T2;
#pragma unroll
          for (int a = 0; a < N; ++a) {
            double &r = acc[(c * N + bb) * N + a];
            r = fma(vx[a], S0, fma(dvx[a], S1, r));
          }
        }
      }
      __syncwarp();  // all lanes are done with buffer b before it is refilled
      if (lane == 0) fence_proxy_async();
    }
    warp_reduce_smem<C::ACC, C::RROWS>(acc, RB, lane, [&](int l, double val) {
      if (l < N3) Rb[B::pad(l)] = val;
    });
  }
  if constexpr (!C::BULK) cp_async_wait<0>();
  mbar_wait(bar + 1, 0);
  __syncwarp();
  // ---------------- faces: traces, the 2 faces (lo, hi) of one axis per pass
  const int fside = lane >= NN ? 1 : 0, ft_t = lane - fside * NN;
  static_for<0, 3>([&](auto dc) {
    constexpr int DD = decltype(dc)::value;
    const int f = 2 * DD + fside;
    if (lane < 2 * NN && ((act >> f) & 1u)) {
      double *fa = FAR + f * C::FARR;
      face_trace<N, DD, LN, LN>(U, NB + f * SZN, fside, ft_t, (gpm >> f) & 1u, (ssm >> f) & 1u, (stm >> f) & 1u,
                                kp, ft, R, fa, fa + NN);
    }
  });
  __syncwarp();
  static_for<0, 2>([&](auto wc) {
    constexpr int W = decltype(wc)::value;
    static_for<0, 3>([&](auto dc) {
      constexpr int DD = decltype(dc)::value;
      const int f = 2 * DD + fside;
      if (lane < 2 * NN && ((stm >> f) & 1u)) face_mass<N, DD, W, LN>(NB + f * SZN, ft_t, true, R);
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
        const double *pp = (q0 == pb) ? (FP + f * 128 + 4 * lane) : (sf_pts + 4 * q);
        const double2 p0 = *reinterpret_cast<const double2 *>(pp);
        s = p0.x;
        tt = p0.y;
        W = pp[2];
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
      const double k1 = W * fma(kp.sigma, J0, -sg * kp.i2h * A);
      const double k2 = -W * sg * kp.i2h * J0;
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
    warp_reduce_smem<C::ACC2, (C::ACC2 < 32 ? C::ACC2 : 32)>(fa, RB, lane, [&](int l, double val) {
      if (l < NN) FC1[l] = val;
      else if (l < 2 * NN) FC2[l - NN] = val;
    });
  }
  __syncwarp();
  // ---------------- add every face contribution into the cell block, line by line
  static_for<0, 3>([&](auto dc) {
    constexpr int DD = decltype(dc)::value;
    for (int t = lane; t < NN; t += 32) {
      face_accumulate<N, DD, LN>(Rb, NB, t, stm, stm, R);
      // cut-face SIPG (already integrated): F1 at the face node, l'_m F2 along the line
      constexpr int sr = B::template lstride<DD>();
      const int br = B::template lbase<DD>(t);
#pragma unroll
      for (int side = 0; side < 2; ++side) {
        const int f = 2 * DD + side;
        if (!((scm >> f) & 1u)) continue;
        const double *FC1 = FAR + f * C::FARR + 2 * NN, *FC2 = FC1 + NN;
        const double F1 = FC1[t], F2 = FC2[t];
        const double *dw = side ? R.d1 : R.d0;
#pragma unroll
        for (int m = 0; m < N; ++m) Rb[br + m * sr] = fma(dw[m], F2, Rb[br + m * sr]);
        Rb[br + (side ? N - 1 : 0) * sr] += F1;
      }
    }
    __syncwarp();
  });
  double *vbk = v + (size_t)dsc.blk * N3;
  for (int l = lane; l < N3; l += 32) vbk[l] = Rb[B::pad(l)];
}
#include "kernels_uncut3.cuh"
