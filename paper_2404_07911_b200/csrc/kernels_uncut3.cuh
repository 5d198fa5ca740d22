// k_uncut3<N, PLAIN>: persistent structured-cell kernel (N <= 5).
//
// Each cell slot (N^2 lanes = one lane per 1-D line; 32/N^2 slots per warp)
// walks through the cells s, s + S, s + 2S, ... (S = all slots of the grid).
// The block and the six neighbour blocks of the NEXT-but-one cell are fetched by
// TMA bulk copies into a second buffer set while the current cell is computed
// (double buffering, one mbarrier per buffer and phase), so DRAM/L2 latency is
// off the critical path.  PLAIN = every face of the cell is an interior SIPG
// face between uncut cells (no ghost penalty, all six neighbours active): the
// face work then needs no per-face branches.  Faces are processed axis by axis:
// the lo and hi face of one axis share the trace, in-face mass and accumulation
// phases, with all lanes busy.

template <int N>
struct Uncut3Cfg {
  static constexpr bool BULK = CUTFEM_USE_BULK && (N % 2) == 0;
  using LN = typename std::conditional<BULK, BlkU<N>, Blk<N>>::type;  // U / NB layout
  static constexpr int NN = N * N, N3 = N * N * N;
  static constexpr int LPS = NN;
  static constexpr int CPW = 32 / NN;
  static constexpr int WARPS = 4;
  static constexpr int SET = 7 * LN::SZ + ((7 * LN::SZ) & 1);  // U + NB[6]
  // bars[4] | desc[2] (4 doubles each) | set0 | set1 | Q | R | FB[2 sides][2 fields][NN]
  static constexpr int OFF_D = 4;
  static constexpr int OFF_S0 = 12;
  static constexpr int OFF_Q = OFF_S0 + 2 * SET;
  static constexpr int OFF_R = OFF_Q + Blk<N>::SZ + (Blk<N>::SZ & 1);
  static constexpr int OFF_FB = OFF_R + Blk<N>::SZ + (Blk<N>::SZ & 1);
  static constexpr int SLOT = OFF_FB + 4 * NN + ((4 * NN) & 1);
  static constexpr int SMEM = WARPS * CPW * SLOT * 8;
};

// SIPG traces of face (DD, side): writes the two in-face fields F1 (FB[t]) and
// F2 (FB[NN + t]) of the own side.
template <int N, int DD, class LU, class LN>
__device__ __forceinline__ void sipg_fields(const double *U, const double *NBf, int side, int t,
                                            const KParams &kp, const RefTab &R, double *FB) {
  constexpr int su = LU::template lstride<DD>(), sn = LN::template lstride<DD>();
  const int bu = LU::template lbase<DD>(t), bn = LN::template lbase<DD>(t);
  const double sg = side ? 1.0 : -1.0;
  const double *dow = side ? R.d1 : R.d0;
  const double *dnb = side ? R.d0 : R.d1;
  double A0 = 0.0, A1 = 0.0, uof = 0.0, unf = 0.0;
#pragma unroll
  for (int m = 0; m < N; ++m) {
    const double a = U[bu + m * su], b = NBf[bn + m * sn];
    A0 = fma(dow[m], a, A0);
    A1 = fma(dnb[m], b, A1);
    if (m == (side ? N - 1 : 0)) uof = a;
    if (m == (side ? 0 : N - 1)) unf = b;
  }
  const double J0 = uof - unf, A = A0 + A1;
  FB[t] = fma(kp.h2sig, J0, -sg * kp.hh * A);
  FB[N * N + t] = -sg * kp.hh * J0;
}

// ACC: v += result (the ghost-penalty pass after k_tile / k_tile2, mask = GP)
template <int N, bool PLAIN, bool ACC = false>
__global__ void __launch_bounds__(128) k_uncut3(const double *__restrict__ u, double *__restrict__ v,
                                                const UDesc *__restrict__ desc, int ncell, KParams kp,
                                                FaceTab ft) {
  static_assert(N * N <= 32, "k_uncut3 needs N <= 5");
  using B = Blk<N>;
  using C = Uncut3Cfg<N>;
  using LN = typename C::LN;
  constexpr int NN = B::NN, N3 = B::N3, SZ = B::SZ, SZN = LN::SZ, LPS = C::LPS;
  const RefTab &R = c_ref[N - 2];
  extern __shared__ __align__(16) double smem[];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int slot = lane / LPS, t = lane % LPS;
  if (slot >= C::CPW) return;  // lanes beyond the last full slot
  const unsigned mask = ((LPS == 32) ? 0xffffffffu : ((1u << LPS) - 1u)) << (slot * LPS);
  const int s0 = (blockIdx.x * C::WARPS + warp) * C::CPW + slot;
  const int S = gridDim.x * C::WARPS * C::CPW;
  double *base = smem + (warp * C::CPW + slot) * C::SLOT;
  uint64_t *bar = reinterpret_cast<uint64_t *>(base);  // [set][U, NB]
  double *Q = base + C::OFF_Q, *Rb = base + C::OFF_R, *FB = base + C::OFF_FB;
  const bool sipg = (kp.mask & TERM_SIPG) != 0, gp_on = (kp.mask & TERM_GP) != 0;

  auto masks = [&](const UDesc &d, uint32_t &act, uint32_t &gpm) {
    act = 0;
    gpm = 0;
#pragma unroll
    for (int f = 0; f < 6; ++f) {
      if (d.nb[f] < 0) continue;
      const bool g = ((d.flags >> f) & 1u) && gp_on;
      if (!(g || sipg)) continue;
      act |= 1u << f;
      if (g) gpm |= 1u << f;
    }
  };
  // issue the loads of `cell` into buffer set `st` (lane t == 0 of the slot)
  auto issue = [&](const UDesc &d, int st) {
    *reinterpret_cast<UDesc *>(base + C::OFF_D + 4 * st) = d;
    uint32_t act, gpm;
    masks(d, act, gpm);
    double *Us = base + C::OFF_S0 + st * C::SET, *NBs = Us + SZN;
    if constexpr (C::BULK) {
      mbar_expect_tx(bar + 2 * st, N3 * 8);
      bulk_g2s(Us, u + (size_t)d.blk * N3, N3 * 8, bar + 2 * st);
      mbar_expect_tx(bar + 2 * st + 1, __popc(act) * N3 * 8);
#pragma unroll
      for (int f = 0; f < 6; ++f)
        if ((act >> f) & 1u) bulk_g2s(NBs + f * SZN, u + (size_t)d.nb[f] * N3, N3 * 8, bar + 2 * st + 1);
    }
  };
  // odd N: every lane copies its share with 8-byte cp.async (no bulk copy)
  auto issue_lanes = [&](int cell, int st) {
    const UDesc d = desc[cell];
    if (t == 0) *reinterpret_cast<UDesc *>(base + C::OFF_D + 4 * st) = d;
    uint32_t act, gpm;
    masks(d, act, gpm);
    double *Us = base + C::OFF_S0 + st * C::SET, *NBs = Us + SZN;
    const double *ub = u + (size_t)d.blk * N3;
    for (int l = t; l < N3; l += LPS) cp_async8(Us + LN::at(l % N, (l / N) % N, l / NN), ub + l);
#pragma unroll
    for (int f = 0; f < 6; ++f) {
      if (!((act >> f) & 1u)) continue;
      const double *nbp = u + (size_t)d.nb[f] * N3;
      for (int l = t; l < N3; l += LPS) cp_async8(NBs + f * SZN + LN::at(l % N, (l / N) % N, l / NN), nbp + l);
    }
    cp_async_commit();
  };
  if (s0 >= ncell) return;
  if constexpr (C::BULK) {
    if (t == 0) {
#pragma unroll
      for (int i = 0; i < 4; ++i) mbar_init(bar + i, 1);
      mbar_fence_init();
    }
    __syncwarp(mask);
    if (t == 0) {
      issue(desc[s0], 0);
      if (s0 + S < ncell) issue(desc[s0 + S], 1);
    }
    __syncwarp(mask);  // the staged descriptors are visible to the slot
  } else {
    issue_lanes(s0, 0);
    if (s0 + S < ncell) issue_lanes(s0 + S, 1);
    else cp_async_commit();  // keep one group per set in flight
  }
  const double h = kp.h;
  const double sK = h * R.gw[t % N] * R.gw[t / N];
  int k = 0;
  for (int cell = s0; cell < ncell; cell += S, ++k) {
    const int st = k & 1;
    const uint32_t par = (k >> 1) & 1;
    double *U = base + C::OFF_S0 + st * C::SET, *NB = U + SZN;
    uint32_t act, gpm;
    act = 0x3fu;
    gpm = 0u;
    UDesc dn;  // descriptor of cell + 2S (lane 0), prefetched a full iteration ahead
    if (C::BULK && t == 0 && cell + 2 * S < ncell) dn = desc[cell + 2 * S];
    if constexpr (C::BULK) {
      mbar_wait(bar + 2 * st, par);
    } else {
      cp_async_wait<1>();
      __syncwarp(mask);
    }
    const UDesc d = *reinterpret_cast<const UDesc *>(base + C::OFF_D + 4 * st);
    if (!PLAIN) masks(d, act, gpm);
    // ---------------- volume: E (S x, y, z), B (K_c per direction), I (S^T)
    if (kp.mask & TERM_CELL) {
      {
        double in[N], out[N];
        const int bu = LN::template lbase<0>(t);
#pragma unroll
        for (int q = 0; q < N; ++q) in[q] = U[bu + q];
        eo_mv<N>(R.S, in, out);
        const int bq = B::template lbase<0>(t);
#pragma unroll
        for (int q = 0; q < N; ++q) Q[bq + q] = out[q];
      }
      __syncwarp(mask);
      static_for<1, 3>([&](auto dc) {
        constexpr int D = decltype(dc)::value;
        sweep_line<N, 0>(Q, Q, B::template lbase<D>(t), B::template lstride<D>(), R.S, 1.0);
        __syncwarp(mask);
      });
      static_for<0, 3>([&](auto dc) {
        constexpr int D = decltype(dc)::value;
        if (D == 0) sweep_line<N, 2>(Q, Rb, B::template lbase<D>(t), B::template lstride<D>(), R.Kc, sK);
        else sweep_line<N, 1>(Q, Rb, B::template lbase<D>(t), B::template lstride<D>(), R.Kc, sK);
        __syncwarp(mask);
      });
      static_for<0, 3>([&](auto dc) {
        constexpr int D = decltype(dc)::value;
        sweep_line<N, 0>(Rb, Rb, B::template lbase<D>(t), B::template lstride<D>(), R.St, 1.0);
        __syncwarp(mask);
      });
    } else {
      for (int l = t; l < SZ; l += LPS) Rb[l] = 0.0;
      __syncwarp(mask);
    }
    if constexpr (C::BULK) {
      mbar_wait(bar + 2 * st + 1, par);
    }
    // ---------------- faces, axis by axis (lo and hi face together)
    if constexpr (PLAIN) {
      // spread the SIPG fields of both faces along the normal line first, then
      // apply the in-face mass once to the spread (n-layer) block: 3 phases/axis
      double *T = Q;
      static_for<0, 3>([&](auto dc) {
        constexpr int DD = decltype(dc)::value;
        constexpr int E1 = (DD == 0) ? 1 : 0, E2 = (DD == 2) ? 1 : 2;
        constexpr int su = LN::template lstride<DD>();
        {
          const int bu = LN::template lbase<DD>(t);
          const double *NLo = NB + (2 * DD) * SZN, *NHi = NB + (2 * DD + 1) * SZN;
          double uo[N], ul[N], uh[N];
#pragma unroll
          for (int m = 0; m < N; ++m) {
            uo[m] = U[bu + m * su];
            ul[m] = NLo[bu + m * su];
            uh[m] = NHi[bu + m * su];
          }
          double Alo = 0.0, Ahi = 0.0;
#pragma unroll
          for (int m = 0; m < N; ++m) {
            Alo = fma(R.d0[m], uo[m], fma(R.d1[m], ul[m], Alo));
            Ahi = fma(R.d1[m], uo[m], fma(R.d0[m], uh[m], Ahi));
          }
          const double Jlo = uo[0] - ul[N - 1], Jhi = uo[N - 1] - uh[0];
          const double F1lo = fma(kp.h2sig, Jlo, kp.hh * Alo), F2lo = kp.hh * Jlo;
          const double F1hi = fma(kp.h2sig, Jhi, -kp.hh * Ahi), F2hi = -kp.hh * Jhi;
          constexpr int sr = B::template lstride<DD>();
          const int br = B::template lbase<DD>(t);
#pragma unroll
          for (int m = 0; m < N; ++m) {
            double x = fma(R.d0[m], F2lo, R.d1[m] * F2hi);
            if (m == 0) x += F1lo;
            if (m == N - 1) x += F1hi;
            T[br + m * sr] = x;
          }
        }
        __syncwarp(mask);
        sweep_line<N, 0>(T, T, B::template lbase<E1>(t), B::template lstride<E1>(), R.M, 1.0);
        __syncwarp(mask);
        sweep_line<N, 1>(T, Rb, B::template lbase<E2>(t), B::template lstride<E2>(), R.M, 1.0);
        __syncwarp(mask);
      });
    } else {
    static_for<0, 3>([&](auto dc) {
      constexpr int DD = decltype(dc)::value;
      constexpr int E1 = (DD == 0) ? 1 : 0, E2 = (DD == 2) ? 1 : 2;
      // A: traces -> SIPG fields (FB) or full GP lines (in place in NB_f)
#pragma unroll
      for (int side = 0; side < 2; ++side) {
        const int f = 2 * DD + side;
        if (!PLAIN && !((act >> f) & 1u)) continue;
        if (!PLAIN && ((gpm >> f) & 1u))
          face_trace<N, DD, LN, LN>(U, NB + f * SZN, side, t, true, sipg, true, kp, ft, R, nullptr, nullptr);
        else if (PLAIN || sipg)
          sipg_fields<N, DD, LN, LN>(U, NB + f * SZN, side, t, kp, R, FB + side * 2 * NN);
      }
      __syncwarp(mask);
      // B, C: in-face mass (e1 then e2)
      static_for<0, 2>([&](auto wc) {
        constexpr int W = decltype(wc)::value;
        constexpr int ED = W ? E2 : E1;
        // SIPG field lines: task k in [0, 4N): side = k / 2N, field = (k / N) % 2, line j = k % N
        for (int kk = t; kk < 4 * N; kk += LPS) {
          const int side = kk / (2 * N), j = kk % N;
          const int f = 2 * DD + side;
          if (!PLAIN && (!((act >> f) & 1u) || ((gpm >> f) & 1u) || !sipg)) continue;
          double *F = FB + (kk / N) * NN;  // [side][field] blocks of NN
          double in[N], out[N];
#pragma unroll
          for (int i = 0; i < N; ++i) in[i] = F[W ? (j + N * i) : (i + N * j)];
          eo_mv<N>(R.M, in, out);
#pragma unroll
          for (int i = 0; i < N; ++i) F[W ? (j + N * i) : (i + N * j)] = out[i];
        }
        if (!PLAIN) {
#pragma unroll
          for (int side = 0; side < 2; ++side) {
            const int f = 2 * DD + side;
            if (((act & gpm) >> f) & 1u)
              sweep_line<N, 0>(NB + f * SZN, NB + f * SZN, LN::template lbase<ED>(t), LN::template lstride<ED>(),
                               R.M, 1.0);
          }
        }
        __syncwarp(mask);
      });
      // D: add both faces' contributions into line t (along DD) of the cell block
      {
        constexpr int sr = B::template lstride<DD>(), sn = LN::template lstride<DD>();
        const int br = B::template lbase<DD>(t), bn = LN::template lbase<DD>(t);
        double r[N];
#pragma unroll
        for (int m = 0; m < N; ++m) r[m] = Rb[br + m * sr];
#pragma unroll
        for (int side = 0; side < 2; ++side) {
          const int f = 2 * DD + side;
          if (!PLAIN && !((act >> f) & 1u)) continue;
          if (!PLAIN && ((gpm >> f) & 1u)) {
            const double *NBf = NB + f * SZN;
#pragma unroll
            for (int m = 0; m < N; ++m) r[m] += NBf[bn + m * sn];
          } else if (PLAIN || sipg) {
            const double F1 = FB[side * 2 * NN + t], F2 = FB[side * 2 * NN + NN + t];
            const double *dw = side ? R.d1 : R.d0;
#pragma unroll
            for (int m = 0; m < N; ++m) r[m] = fma(dw[m], F2, r[m]);
            r[side ? N - 1 : 0] += F1;
          }
        }
#pragma unroll
        for (int m = 0; m < N; ++m) Rb[br + m * sr] = r[m];
      }
      __syncwarp(mask);
    });
    }
    // ---------------- write the block, then reuse this buffer set for cell + 2S
    {
      double *vb = v + (size_t)d.blk * N3;
      if (ACC)
        for (int l = t; l < N3; l += LPS) vb[l] += Rb[B::pad(l)];
      else
        for (int l = t; l < N3; l += LPS) vb[l] = Rb[B::pad(l)];
    }
    __syncwarp(mask);
    if (cell + 2 * S < ncell) {
      if constexpr (C::BULK) {
        if (t == 0) {
          fence_proxy_async();
          issue(dn, st);
        }
      } else {
        issue_lanes(cell + 2 * S, st);
      }
    } else if constexpr (!C::BULK) {
      cp_async_commit();
    }
  }
}
