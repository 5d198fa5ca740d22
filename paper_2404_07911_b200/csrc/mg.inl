// mg.inl — Chebyshev smoothing and polynomial multigrid around the operator (included
// by cutfem.cu after cg.inl, whose dot kernels it uses; C ABI in include/cutfem.h).
//
// PAPER §3.5 "Iterative solution": preconditioned CG; for DG a p-multigrid
// preconditioner (p-transfer between polynomial degrees) with Chebyshev smoothers whose
// inner preconditioner is additive Schwarz on the cells (the inverse diagonal blocks).
// SURVEY §8(f) f4.  Every step runs in the kernels below or in the operator's own
// kernels (dispatch_apply); the host only sequences launches and holds the scalar
// Chebyshev coefficients.  Oracle: oracle/solver.py (chebyshev, prolongate / restrict,
// vcycle, pcg); DESIGN.md §5.12 and readings A26-A29.

namespace {

constexpr int MG_THREADS = 256;

struct MGTab {
  double I[CUTFEM_NMAX * CUTFEM_NMAX];  // I[a * nc + b] = l^c_b(x^f_a)
};

__device__ __forceinline__ int64_t mg_grid_stride() { return (int64_t)gridDim.x * blockDim.x; }
__device__ __forceinline__ int64_t mg_tid() { return (int64_t)blockIdx.x * blockDim.x + threadIdx.x; }

// u = 1 on local index l of every block of colour c, else 0
__global__ void k_mg_probe_set(double *__restrict__ u, const uint8_t *__restrict__ col, int64_t n, int n3, int c,
                               int l) {
  for (int64_t i = mg_tid(); i < n; i += mg_grid_stride()) {
    const int64_t K = i / n3;
    u[i] = (col[K] == c && (int)(i - K * n3) == l) ? 1.0 : 0.0;
  }
}

// column l of A_KK for every probed block that owns a slot (slot 0, the shared block
// of the plain uncut cells, is written by its representative block `rep` only)
__global__ void k_mg_probe_take(double *__restrict__ blocks, const double *__restrict__ v,
                                const uint8_t *__restrict__ col, const int32_t *__restrict__ slot, int64_t rep,
                                int64_t n, int n3, int c, int l) {
  for (int64_t i = mg_tid(); i < n; i += mg_grid_stride()) {
    const int64_t K = i / n3;
    if (col[K] != c) continue;
    const int s = slot[K];
    if (s == 0 && K != rep) continue;
    const int a = (int)(i - K * n3);
    blocks[((int64_t)s * n3 + a) * n3 + l] = v[i];
  }
}

// the diagonal entries (K, l) of the probed colour
__global__ void k_probe_take_diag(double *__restrict__ dd, const double *__restrict__ v,
                                  const uint8_t *__restrict__ col, int64_t n, int n3, int c, int l) {
  for (int64_t i = mg_tid(); i < n; i += mg_grid_stride()) {
    const int64_t K = i / n3;
    if (col[K] == c && (int)(i - K * n3) == l) dd[i] = v[i];
  }
}

// in-place inverse of one SPD m x m block per CTA (Gauss-Jordan sweep, no pivoting:
// for each k, a_ij -= a_ik a_kj / a_kk (i, j != k); a_kj /= a_kk; a_ik *= -1/a_kk; a_kk = 1/a_kk)
__global__ void __launch_bounds__(MG_THREADS) k_mg_invert(double *__restrict__ blocks, int m) {
  double *M = blocks + (int64_t)blockIdx.x * m * m;
  for (int k = 0; k < m; ++k) {
    const double ip = 1.0 / M[k * m + k];
    for (int e = threadIdx.x; e < m * m; e += blockDim.x) {
      const int i = e / m, j = e - i * m;
      if (i != k && j != k) M[e] -= M[i * m + k] * M[k * m + j] * ip;
    }
    __syncthreads();
    for (int e = threadIdx.x; e < 2 * m; e += blockDim.x) {
      if (e < m) {
        if (e != k) M[k * m + e] *= ip;
      } else if (e - m != k) {
        M[(e - m) * m + k] *= -ip;
      }
    }
    __syncthreads();
    if (threadIdx.x == 0) M[k * m + k] = ip;
    __syncthreads();
  }
}

// One Chebyshev step, thread per entry (K, a):
//   t = D^-1 (r - q)    (q == null: r;  BLOCK: sum_j Binv[slot K][j][a] (r - q)[K, j]
//                        (the blocks are symmetric: column reads are coalesced);  else dinv (r - q))
//   d = c1 d + c2 t     (c1 == 0: d = c2 t, d may hold garbage)
//   x = x + d  (xadd)   or   x = d
// x and d are written by the thread that reads them; r, q are only read.
template <bool BLOCK>
__global__ void __launch_bounds__(MG_THREADS)
    k_mg_cheb(double *x, double *d, const double *__restrict__ r, const double *__restrict__ q,
              const double *__restrict__ dinv, const double *__restrict__ blocks, const int32_t *__restrict__ slot,
              int64_t n, int n3, double c1, double c2, int xadd) {
  for (int64_t i = mg_tid(); i < n; i += mg_grid_stride()) {
    double t;
    if constexpr (BLOCK) {
      const int64_t K = i / n3;
      const int a = (int)(i - K * n3);
      const double *B = blocks + (int64_t)slot[K] * n3 * n3 + a;
      const double *rK = r + K * n3, *qK = q ? q + K * n3 : nullptr;
      double s0 = 0.0, s1 = 0.0;
      int j = 0;
      for (; j + 1 < n3; j += 2) {
        s0 = fma(B[(int64_t)j * n3], qK ? rK[j] - qK[j] : rK[j], s0);
        s1 = fma(B[(int64_t)(j + 1) * n3], qK ? rK[j + 1] - qK[j + 1] : rK[j + 1], s1);
      }
      if (j < n3) s0 = fma(B[(int64_t)j * n3], qK ? rK[j] - qK[j] : rK[j], s0);
      t = s0 + s1;
    } else {
      t = dinv[i] * (q ? r[i] - q[i] : r[i]);
    }
    const double di = c1 == 0.0 ? c2 * t : fma(c1, d[i], c2 * t);
    d[i] = di;
    x[i] = xadd ? x[i] + di : di;
  }
}

// The cell-block step for a compile-time block size N3 = n^3: a CTA takes groups of
// CPB = max(1, 256 / N3) cells, stages e = r - q of the group in shared memory, and each
// thread forms rows a of t = Binv[slot K] e_K (8-way unrolled column sweep, four
// independent sums: the block reads are the only HBM traffic, each entry read once),
// then d = c1 d + c2 t, x (+)= d as k_mg_cheb.
template <int N3>
__global__ void __launch_bounds__(MG_THREADS)
    k_mg_chebb(double *x, double *d, const double *__restrict__ r, const double *__restrict__ q,
               const double *__restrict__ blocks, const int32_t *__restrict__ slot, int64_t nblk, double c1,
               double c2, int xadd) {
  constexpr int CPB = N3 >= MG_THREADS ? 1 : MG_THREADS / N3;
  __shared__ double e[CPB * N3];
  for (int64_t g0 = (int64_t)blockIdx.x * CPB; g0 < nblk; g0 += (int64_t)gridDim.x * CPB) {
    const int nc = (int)(nblk - g0 < CPB ? nblk - g0 : CPB);
    const int64_t base = g0 * N3;
    for (int i = threadIdx.x; i < nc * N3; i += MG_THREADS) e[i] = q ? r[base + i] - q[base + i] : r[base + i];
    __syncthreads();
    for (int i = threadIdx.x; i < nc * N3; i += MG_THREADS) {
      const int c = i / N3, a = i - c * N3;
      const double *B = blocks + (int64_t)slot[g0 + c] * N3 * N3 + a;
      const double *ec = e + c * N3;
      double s0 = 0.0, s1 = 0.0, s2 = 0.0, s3 = 0.0;
      int j = 0;
#pragma unroll 2
      for (; j + 8 <= N3; j += 8) {
        double b[8];
#pragma unroll
        for (int k = 0; k < 8; ++k) b[k] = B[(int64_t)(j + k) * N3];
        s0 = fma(b[0], ec[j], s0);
        s1 = fma(b[1], ec[j + 1], s1);
        s2 = fma(b[2], ec[j + 2], s2);
        s3 = fma(b[3], ec[j + 3], s3);
        s0 = fma(b[4], ec[j + 4], s0);
        s1 = fma(b[5], ec[j + 5], s1);
        s2 = fma(b[6], ec[j + 6], s2);
        s3 = fma(b[7], ec[j + 7], s3);
      }
      for (; j < N3; ++j) s0 = fma(B[(int64_t)j * N3], ec[j], s0);
      const double t = (s0 + s1) + (s2 + s3);
      const int64_t gi = base + i;
      const double di = c1 == 0.0 ? c2 * t : fma(c1, d[gi], c2 * t);
      d[gi] = di;
      x[gi] = xadd ? x[gi] + di : di;
    }
    __syncthreads();
  }
}

// x_f (+)= P x_c: thread per fine entry (K, a = ax + nf ay + nf^2 az):
//   sum_b I[ax][bx] I[ay][by] I[az][bz] x_c[cmap K][b]   (0 when cmap K < 0)
__global__ void __launch_bounds__(MG_THREADS)
    k_mg_prolong(double *__restrict__ xf, const double *__restrict__ xc, const int32_t *__restrict__ cmap, MGTab t,
                 int64_t nblk_f, int nf, int nc, int add) {
  const int nf3 = nf * nf * nf, nc3 = nc * nc * nc;
  for (int64_t i = mg_tid(); i < nblk_f * nf3; i += mg_grid_stride()) {
    const int64_t K = i / nf3;
    const int a = (int)(i - K * nf3), ax = a % nf, ay = (a / nf) % nf, az = a / (nf * nf);
    const int c = cmap[K];
    double s = 0.0;
    if (c >= 0) {
      const double *X = xc + (int64_t)c * nc3;
      for (int bz = 0; bz < nc; ++bz) {
        double sy = 0.0;
        for (int by = 0; by < nc; ++by) {
          double sx = 0.0;
          for (int bx = 0; bx < nc; ++bx) sx = fma(t.I[ax * nc + bx], X[(bz * nc + by) * nc + bx], sx);
          sy = fma(t.I[ay * nc + by], sx, sy);
        }
        s = fma(t.I[az * nc + bz], sy, s);
      }
    }
    xf[i] = add ? xf[i] + s : s;
  }
}

// r_c = P^T (r_f - q_f): thread per coarse entry (Kc, b): sum_a I[ax][bx] I[ay][by] I[az][bz]
// (r_f - q_f)[fmap Kc][a]   (0 when fmap Kc < 0; q_f == null: r_f)
__global__ void __launch_bounds__(MG_THREADS)
    k_mg_restrict(double *__restrict__ rc, const double *__restrict__ rf, const double *__restrict__ qf,
                  const int32_t *__restrict__ fmap, MGTab t, int64_t nblk_c, int nf, int nc) {
  const int nf3 = nf * nf * nf, nc3 = nc * nc * nc;
  for (int64_t i = mg_tid(); i < nblk_c * nc3; i += mg_grid_stride()) {
    const int64_t Kc = i / nc3;
    const int b = (int)(i - Kc * nc3), bx = b % nc, by = (b / nc) % nc, bz = b / (nc * nc);
    const int K = fmap[Kc];
    double s = 0.0;
    if (K >= 0) {
      const double *R = rf + (int64_t)K * nf3, *Q = qf ? qf + (int64_t)K * nf3 : nullptr;
      for (int az = 0; az < nf; ++az) {
        double sy = 0.0;
        for (int ay = 0; ay < nf; ++ay) {
          double sx = 0.0;
          for (int ax = 0; ax < nf; ++ax) {
            const int a = (az * nf + ay) * nf + ax;
            sx = fma(t.I[ax * nc + bx], Q ? R[a] - Q[a] : R[a], sx);
          }
          sy = fma(t.I[ay * nc + by], sx, sy);
        }
        s = fma(t.I[az * nc + bz], sy, s);
      }
    }
    rc[i] = s;
  }
}

// the Lanczos start vector: U(-1, 1) from a counter-based hash (splitmix64) of the index
__global__ void k_mg_random(double *__restrict__ x, int64_t n, uint64_t seed) {
  for (int64_t i = mg_tid(); i < n; i += mg_grid_stride()) {
    uint64_t z = seed + 0x9e3779b97f4a7c15ull * (uint64_t)(i + 1);
    z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ull;
    z = (z ^ (z >> 27)) * 0x94d049bb133111ebull;
    z ^= z >> 31;
    x[i] = 2.0 * ((double)(z >> 11) * (1.0 / 9007199254740992.0)) - 1.0;
  }
}

// r = b - q, p = r (q == null: r = b); partial sums of |r|^2
__global__ void __launch_bounds__(CG_THREADS) k_mg_res(double *__restrict__ r, const double *__restrict__ b,
                                                       const double *__restrict__ q, int64_t n,
                                                       double *__restrict__ part_rr) {
  __shared__ double sh[CG_THREADS];
  double s = 0.0;
  for (int64_t i = blockIdx.x * (int64_t)CG_THREADS + threadIdx.x; i < n; i += (int64_t)gridDim.x * CG_THREADS) {
    const double ri = q ? b[i] - q[i] : b[i];
    r[i] = ri;
    s = fma(ri, ri, s);
  }
  s = block_sum(s, sh);
  if (threadIdx.x == 0) part_rr[blockIdx.x] = s;
}

// the largest eigenvalue of a symmetric tridiagonal matrix (diagonal a, off-diagonal b)
// by bisection on the Sturm sequence count
double tridiag_max_eig(const std::vector<double> &a, const std::vector<double> &b) {
  const int m = (int)a.size();
  double lo = 1e300, hi = -1e300;
  for (int i = 0; i < m; ++i) {
    const double r = (i > 0 ? std::fabs(b[i - 1]) : 0.0) + (i + 1 < m ? std::fabs(b[i]) : 0.0);
    lo = std::min(lo, a[i] - r);
    hi = std::max(hi, a[i] + r);
  }
  auto count_below = [&](double x) {  // eigenvalues < x
    int c = 0;
    double dd = 1.0;
    for (int i = 0; i < m; ++i) {
      dd = a[i] - x - (i > 0 ? b[i - 1] * b[i - 1] / dd : 0.0);
      if (dd == 0.0) dd = -1e-300;
      if (dd < 0) ++c;
    }
    return c;
  };
  for (int it = 0; it < 200 && hi - lo > 1e-14 * std::max(std::fabs(hi), 1e-300); ++it) {
    const double mid = 0.5 * (lo + hi);
    if (count_below(mid) >= m) hi = mid;
    else lo = mid;
  }
  return hi;
}

}  // namespace

struct cutfem_mg_level {
  cutfem_handle *hd = nullptr;
  int degree = 1, n = 2, n3 = 8;
  int64_t nblk = 0, ndof = 0;
  double lam = 1.0;
  // inner preconditioner
  double *dinv = nullptr;                               // JACOBI
  double *blocks = nullptr;                             // BLOCK: [nslot][n3][n3] inverses
  int32_t *slot = nullptr;                              // BLOCK: slot of every block (0: the shared plain block)
  int64_t nslot = 0;
  // to the next coarser level (unused on level 0)
  int32_t *cmap = nullptr;                              // fine block -> coarse block or -1
  int32_t *fmap = nullptr;                              // coarse block -> fine block or -1
  MGTab tab;
  // work vectors (r, x: this level's right-hand side / correction inside a V-cycle)
  double *r = nullptr, *x = nullptr, *q = nullptr, *d = nullptr;
};

struct cutfem_mg {
  std::vector<cutfem_mg_level> lv;
  cutfem_mg_params prm;
  int device = 0;
  // PCG on the finest level (and the Lanczos runs)
  double *r = nullptr, *z = nullptr, *p = nullptr, *q = nullptr, *xs = nullptr, *bs = nullptr;
  double *partial = nullptr, *partial2 = nullptr, *rz = nullptr, *pq = nullptr, *rr = nullptr;
  int cap = 0;
};

namespace {

unsigned mg_grid(const cutfem_handle *hd, int64_t n) {
  return (unsigned)std::max<int64_t>(1, std::min<int64_t>((n + MG_THREADS - 1) / MG_THREADS, 16 * hd->sm_count));
}

void mg_free(cutfem_mg *mg) {
  if (!mg) return;
  for (auto &L : mg->lv) {
    for (double *x : {L.dinv, L.blocks, L.r, L.x, L.q, L.d}) cudaFree(x);
    cudaFree(L.slot);
    cudaFree(L.cmap);
    cudaFree(L.fmap);
  }
  for (double *x : {mg->r, mg->z, mg->p, mg->q, mg->xs, mg->bs, mg->partial, mg->partial2, mg->rz, mg->pq, mg->rr})
    cudaFree(x);
  delete mg;
}

int mg_alloc(double **p, int64_t n) {
  cudaError_t e = cudaMalloc((void **)p, sizeof(double) * (size_t)std::max<int64_t>(n, 2));
  if (e != cudaSuccess) return fail(CUTFEM_ENOMEM, std::string("cudaMalloc: ") + cudaGetErrorString(e));
  return 0;
}

template <class T>
int mg_upload(T **dst, const std::vector<T> &src) {
  cudaError_t e = cudaMalloc((void **)dst, sizeof(T) * std::max<size_t>(src.size(), 1));
  if (e != cudaSuccess) return fail(CUTFEM_ENOMEM, std::string("cudaMalloc: ") + cudaGetErrorString(e));
  if (!src.empty()) CU(cudaMemcpy(*dst, src.data(), sizeof(T) * src.size(), cudaMemcpyHostToDevice));
  return 0;
}

int mg_pcg_cap(cutfem_mg *mg, int iters) {
  if (mg->cap >= iters + 1) return 0;
  for (double *x : {mg->rz, mg->pq, mg->rr}) cudaFree(x);
  mg->cap = iters + 1;
  int rc;
  if ((rc = mg_alloc(&mg->rz, mg->cap + 1)) || (rc = mg_alloc(&mg->pq, mg->cap + 1)) ||
      (rc = mg_alloc(&mg->rr, mg->cap + 1)))
    return rc;
  return 0;
}

// one Chebyshev step kernel on level L (see k_mg_cheb)
int mg_cheb_kernel(cutfem_mg *mg, cutfem_mg_level &L, double *x, double *d, const double *r, const double *q,
                   double c1, double c2, int xadd, cudaStream_t st) {
  const unsigned g = mg_grid(L.hd, L.ndof);
  if (mg->prm.inner == CUTFEM_INNER_BLOCK) {
    const unsigned gb = (unsigned)std::max<int64_t>(1, std::min<int64_t>(L.nblk, 16 * L.hd->sm_count));
#define MG_CHEBB(NN)                                                                                         \
  case NN:                                                                                                   \
    k_mg_chebb<NN * NN * NN><<<gb, MG_THREADS, 0, st>>>(x, d, r, q, L.blocks, L.slot, L.nblk, c1, c2, xadd); \
    break;
    switch (L.n) {
      MG_CHEBB(2)
      MG_CHEBB(3)
      MG_CHEBB(4)
      MG_CHEBB(5)
      MG_CHEBB(6)
      MG_CHEBB(7)
      MG_CHEBB(8)
      MG_CHEBB(9)
      default:
        k_mg_cheb<true><<<g, MG_THREADS, 0, st>>>(x, d, r, q, nullptr, L.blocks, L.slot, L.ndof, L.n3, c1, c2, xadd);
    }
#undef MG_CHEBB
  } else
    k_mg_cheb<false><<<g, MG_THREADS, 0, st>>>(x, d, r, q, L.dinv, nullptr, nullptr, L.ndof, L.n3, c1, c2, xadd);
  CU(cudaGetLastError());
  return 0;
}

// x <- `degree` Chebyshev steps for A x = r on [lmin, lmax] (oracle/solver.py chebyshev)
int mg_chebyshev(cutfem_mg *mg, cutfem_mg_level &L, const double *r, double *x, int degree, double lmax, double lmin,
                 bool x0, cudaStream_t st) {
  const double theta = 0.5 * (lmax + lmin), delta = 0.5 * (lmax - lmin), sigma = theta / delta;
  int rc;
  if (x0) {
    if ((rc = dispatch_apply(L.hd, x, L.q, st))) return rc;
    if ((rc = mg_cheb_kernel(mg, L, x, L.d, r, L.q, 0.0, 1.0 / theta, 1, st))) return rc;
  } else {
    if ((rc = mg_cheb_kernel(mg, L, x, L.d, r, nullptr, 0.0, 1.0 / theta, 0, st))) return rc;
  }
  double rho = 1.0 / sigma;
  for (int j = 1; j < degree; ++j) {
    const double rho_new = 1.0 / (2.0 * sigma - rho);
    if ((rc = dispatch_apply(L.hd, x, L.q, st))) return rc;
    if ((rc = mg_cheb_kernel(mg, L, x, L.d, r, L.q, rho_new * rho, 2.0 * rho_new / delta, 1, st))) return rc;
    rho = rho_new;
  }
  return 0;
}

// x_f (+)= P x_c (fine level li, coarse li - 1)
int mg_prolong(cutfem_mg *mg, int li, const double *xc, double *xf, int add, cudaStream_t st) {
  cutfem_mg_level &F = mg->lv[li], &C = mg->lv[li - 1];
  k_mg_prolong<<<mg_grid(F.hd, F.ndof), MG_THREADS, 0, st>>>(xf, xc, F.cmap, F.tab, F.nblk, F.n, C.n, add);
  CU(cudaGetLastError());
  return 0;
}

// r_c = P^T (r_f - q_f)
int mg_restrict(cutfem_mg *mg, int li, const double *rf, const double *qf, double *rc, cudaStream_t st) {
  cutfem_mg_level &F = mg->lv[li], &C = mg->lv[li - 1];
  k_mg_restrict<<<mg_grid(C.hd, C.ndof), MG_THREADS, 0, st>>>(rc, rf, qf, F.fmap, F.tab, C.nblk, F.n, C.n);
  CU(cudaGetLastError());
  return 0;
}

// x = B_li r (oracle/solver.py vcycle)
int mg_cycle(cutfem_mg *mg, int li, const double *r, double *x, cudaStream_t st) {
  cutfem_mg_level &L = mg->lv[li];
  const cutfem_mg_params &P = mg->prm;
  if (li == 0) return mg_chebyshev(mg, L, r, x, P.coarse_degree, L.lam, L.lam / P.coarse_range, false, st);
  const double lmin = L.lam / P.smooth_range;
  int rc;
  if ((rc = mg_chebyshev(mg, L, r, x, P.smooth_degree, L.lam, lmin, false, st))) return rc;
  if ((rc = dispatch_apply(L.hd, x, L.q, st))) return rc;
  cutfem_mg_level &C = mg->lv[li - 1];
  if ((rc = mg_restrict(mg, li, r, L.q, C.r, st))) return rc;
  if ((rc = mg_cycle(mg, li - 1, C.r, C.x, st))) return rc;
  if ((rc = mg_prolong(mg, li, C.x, x, 1, st))) return rc;
  return mg_chebyshev(mg, L, r, x, P.smooth_degree, L.lam, lmin, true, st);
}

// PCG on level L with z = prec(r) (device-resident scalars, fixed-order dots):
// rr[k] = |r_k|^2, rz[k] = r_k.z_k, pq[k] = p_k.A p_k
template <class Prec>
int mg_pcg_run(cutfem_mg *mg, cutfem_mg_level &L, Prec prec, const double *b, double *x, int iters, double tol,
               int *iters_done, cudaStream_t st) {
  const int64_t n = L.ndof;
  int rc;
  if ((rc = mg_pcg_cap(mg, iters))) return rc;
  if ((rc = dispatch_apply(L.hd, x, mg->q, st))) return rc;
  k_mg_res<<<CG_BLOCKS, CG_THREADS, 0, st>>>(mg->r, b, mg->q, n, mg->partial);
  CU(cudaGetLastError());
  if ((rc = cg_reduce(nullptr, mg->partial, mg->rr, st))) return rc;
  if ((rc = prec(mg->r, mg->z))) return rc;
  k_dot<<<CG_BLOCKS, CG_THREADS, 0, st>>>(mg->r, mg->z, n, mg->partial);
  if ((rc = cg_reduce(nullptr, mg->partial, mg->rz, st))) return rc;
  CU(cudaMemcpyAsync(mg->p, mg->z, sizeof(double) * n, cudaMemcpyDeviceToDevice, st));
  double bb = 0.0;
  if (tol > 0) {
    k_dot<<<CG_BLOCKS, CG_THREADS, 0, st>>>(b, b, n, mg->partial);
    if ((rc = cg_reduce(nullptr, mg->partial, mg->pq + mg->cap, st))) return rc;
    CU(cudaMemcpyAsync(&bb, mg->pq + mg->cap, sizeof(double), cudaMemcpyDeviceToHost, st));
    CU(cudaStreamSynchronize(st));
  }
  int k = 0;
  for (; k < iters; ++k) {
    if ((rc = dispatch_apply(L.hd, mg->p, mg->q, st))) return rc;
    k_dot<<<CG_BLOCKS, CG_THREADS, 0, st>>>(mg->p, mg->q, n, mg->partial);
    if ((rc = cg_reduce(nullptr, mg->partial, mg->pq + k, st))) return rc;
    // x += alpha p, r -= alpha q, |r|^2 partials (no inner preconditioner here)
    k_cg_xr<<<CG_BLOCKS, CG_THREADS, 0, st>>>(x, mg->r, nullptr, nullptr, mg->p, mg->q, n, mg->rz, mg->pq, k,
                                              mg->partial, mg->partial2);
    CU(cudaGetLastError());
    if ((rc = cg_reduce(nullptr, mg->partial, mg->rr + k + 1, st))) return rc;
    if ((rc = prec(mg->r, mg->z))) return rc;
    k_dot<<<CG_BLOCKS, CG_THREADS, 0, st>>>(mg->r, mg->z, n, mg->partial);
    if ((rc = cg_reduce(nullptr, mg->partial, mg->rz + k + 1, st))) return rc;
    k_cg_p<<<CG_BLOCKS, CG_THREADS, 0, st>>>(mg->p, mg->z, n, mg->rz, k);
    CU(cudaGetLastError());
    if (tol > 0) {
      double rk = 0.0;
      CU(cudaMemcpyAsync(&rk, mg->rr + k + 1, sizeof(double), cudaMemcpyDeviceToHost, st));
      CU(cudaStreamSynchronize(st));
      if (std::sqrt(rk) <= tol * std::sqrt(bb)) {
        ++k;
        break;
      }
    }
  }
  if (iters_done) *iters_done = k;
  return 0;
}

// lam_max of D^-1 A on level L: the largest Ritz value of the Lanczos matrix of
// eig_iters D^-1-preconditioned CG steps from a fixed pseudo-random start (x = 0)
int mg_estimate(cutfem_mg *mg, cutfem_mg_level &L, cudaStream_t st) {
  const int m = mg->prm.eig_iters;
  k_mg_random<<<mg_grid(L.hd, L.ndof), MG_THREADS, 0, st>>>(mg->bs, L.ndof, 0x5eedull + (uint64_t)L.degree);
  CU(cudaGetLastError());
  CU(cudaMemsetAsync(mg->xs, 0, sizeof(double) * L.ndof, st));
  auto inner = [&](const double *r, double *z) { return mg_cheb_kernel(mg, L, z, z, r, nullptr, 0.0, 1.0, 0, st); };
  int done = 0, rc;
  if ((rc = mg_pcg_run(mg, L, inner, mg->bs, mg->xs, m, 0.0, &done, st))) return rc;
  std::vector<double> rz(m + 1), pq(m);
  CU(cudaMemcpyAsync(rz.data(), mg->rz, sizeof(double) * (m + 1), cudaMemcpyDeviceToHost, st));
  CU(cudaMemcpyAsync(pq.data(), mg->pq, sizeof(double) * m, cudaMemcpyDeviceToHost, st));
  CU(cudaStreamSynchronize(st));
  std::vector<double> a, b;
  for (int j = 0; j < m; ++j) {
    if (!(pq[j] > 0) || !(rz[j] > 0)) break;
    const double alpha = rz[j] / pq[j];
    double dj = 1.0 / alpha;
    if (j > 0) {
      const double alpha_p = rz[j - 1] / pq[j - 1], beta_p = rz[j] / rz[j - 1];
      dj += beta_p / alpha_p;
    }
    a.push_back(dj);
    if (j + 1 < m && rz[j + 1] > 0) b.push_back(std::sqrt(rz[j + 1] / rz[j]) / alpha);
  }
  if (a.empty()) return fail(CUTFEM_EINVAL, "eigenvalue estimate: no Lanczos step");
  b.resize(a.size() - 1);
  L.lam = mg->prm.eig_safety * tridiag_max_eig(a, b);
  return 0;
}

// the inner preconditioner of level L
int mg_inner_setup(cutfem_mg *mg, cutfem_mg_level &L, cudaStream_t st) {
  cutfem_handle *hd = L.hd;
  const int n3 = L.n3;
  const int64_t nb = L.nblk;
  int rc;
  std::vector<uint8_t> col(nb);
  for (int64_t K = 0; K < nb; ++K)
    col[K] = (uint8_t)((hd->blk_ijk[3 * K] + hd->blk_ijk[3 * K + 1] + hd->blk_ijk[3 * K + 2]) & 1);
  uint8_t *d_col = nullptr;
  if ((rc = mg_upload(&d_col, col))) return rc;
  std::vector<int32_t> slot(nb, 0);
  int64_t rep = -1;
  if (mg->prm.inner == CUTFEM_INNER_BLOCK) {
    // plain cells: uncut with six active uncut face neighbours -> all share one block
    std::unordered_map<int64_t, int64_t> where;
    auto key = [&](int64_t i, int64_t j, int64_t k) { return (i * (hd->n_cells[1] + 2) + j) * (hd->n_cells[2] + 2) + k; };
    for (int64_t K = 0; K < nb; ++K) where[key(hd->blk_ijk[3 * K], hd->blk_ijk[3 * K + 1], hd->blk_ijk[3 * K + 2])] = K;
    int64_t ns = 1;
    for (int64_t K = 0; K < nb; ++K) {
      bool plain = !hd->blk_cut[K];
      for (int f = 0; f < 6 && plain; ++f) {
        int64_t c[3] = {hd->blk_ijk[3 * K], hd->blk_ijk[3 * K + 1], hd->blk_ijk[3 * K + 2]};
        c[f >> 1] += (f & 1) ? 1 : -1;
        auto it = where.find(key(c[0], c[1], c[2]));
        plain = it != where.end() && !hd->blk_cut[it->second];
      }
      if (plain) {
        slot[K] = 0;
        if (rep < 0) rep = K;
      } else {
        slot[K] = (int32_t)ns++;
      }
    }
    L.nslot = ns;
    if ((rc = mg_upload(&L.slot, slot))) return rc;
    cudaError_t e = cudaMalloc((void **)&L.blocks, sizeof(double) * (size_t)ns * n3 * n3);
    if (e != cudaSuccess) {
      cudaFree(d_col);
      return fail(CUTFEM_ENOMEM, std::string("multigrid blocks: ") + cudaGetErrorString(e));
    }
    CU(cudaMemsetAsync(L.blocks, 0, sizeof(double) * (size_t)ns * n3 * n3, st));
  } else {
    if ((rc = mg_alloc(&L.dinv, L.ndof))) return rc;
  }
  // probing: u = e_l on the cells of one colour -> v = A u holds column l of every A_KK there
  const unsigned g = mg_grid(hd, L.ndof);
  for (int c = 0; c < 2; ++c)
    for (int l = 0; l < n3; ++l) {
      k_mg_probe_set<<<g, MG_THREADS, 0, st>>>(L.x, d_col, L.ndof, n3, c, l);
      CU(cudaGetLastError());
      if ((rc = dispatch_apply(hd, L.x, L.q, st))) return rc;
      if (mg->prm.inner == CUTFEM_INNER_BLOCK) {
        k_mg_probe_take<<<g, MG_THREADS, 0, st>>>(L.blocks, L.q, d_col, L.slot, rep, L.ndof, n3, c, l);
      } else {
        k_probe_take_diag<<<g, MG_THREADS, 0, st>>>(L.dinv, L.q, d_col, L.ndof, n3, c, l);
      }
      CU(cudaGetLastError());
    }
  if (mg->prm.inner == CUTFEM_INNER_BLOCK) {
    if (L.nslot > 0) {
      k_mg_invert<<<(unsigned)L.nslot, MG_THREADS, 0, st>>>(L.blocks, n3);
      CU(cudaGetLastError());
    }
  } else {
    k_recip<<<g, 256, 0, st>>>(L.dinv, L.ndof);
    CU(cudaGetLastError());
  }
  CU(cudaStreamSynchronize(st));
  cudaFree(d_col);
  return 0;
}

}  // namespace

extern "C" {

int cutfem_mg_setup(cutfem_handle *const *levels, int32_t n_levels, const cutfem_mg_params *prm, void *cuda_stream,
                    cutfem_mg **out) {
  if (!out) return fail(CUTFEM_EINVAL, "null out");
  *out = nullptr;
  if (!levels || n_levels < 1 || !prm) return fail(CUTFEM_EINVAL, "levels / params");
  if (prm->inner != CUTFEM_INNER_JACOBI && prm->inner != CUTFEM_INNER_BLOCK) return fail(CUTFEM_EINVAL, "inner");
  if (prm->smooth_degree < 1 || prm->coarse_degree < 1 || !(prm->smooth_range > 1) || !(prm->coarse_range > 1) ||
      prm->eig_iters < 0 || !(prm->eig_safety >= 1))
    return fail(CUTFEM_EINVAL, "multigrid parameters");
  for (int i = 0; i < n_levels; ++i) {
    const cutfem_handle *a = levels[i];
    if (!a) return fail(CUTFEM_EINVAL, "null level handle");
    if (a->dist) return fail(CUTFEM_EUNSUPPORTED, "multigrid on a distributed handle");
    if (i > 0) {
      const cutfem_handle *b = levels[i - 1];
      if (a->degree <= b->degree) return fail(CUTFEM_EINVAL, "level degrees must increase");
      if (a->device != b->device || a->h != b->h)
        return fail(CUTFEM_EINVAL, "levels must share the device and the mesh");
      for (int d = 0; d < 3; ++d)
        if (a->n_cells[d] != b->n_cells[d] || a->lower[d] != b->lower[d])
          return fail(CUTFEM_EINVAL, "levels must share the mesh");
    }
  }
  CU(cudaSetDevice(levels[0]->device));
  cudaStream_t st = (cudaStream_t)cuda_stream;
  cutfem_mg *mg = new cutfem_mg();
  mg->prm = *prm;
  mg->device = levels[0]->device;
  mg->lv.resize(n_levels);
  int rc = 0;
  for (int i = 0; i < n_levels && !rc; ++i) {
    cutfem_mg_level &L = mg->lv[i];
    L.hd = levels[i];
    L.degree = L.hd->degree;
    L.n = L.hd->n;
    L.n3 = L.n * L.n * L.n;
    L.nblk = L.hd->n_active;
    L.ndof = L.nblk * L.n3;
    if ((rc = mg_alloc(&L.r, L.ndof)) || (rc = mg_alloc(&L.x, L.ndof)) || (rc = mg_alloc(&L.q, L.ndof)) ||
        (rc = mg_alloc(&L.d, L.ndof)))
      break;
    if (i > 0) {
      // block maps by cell index, the 1-D interpolation matrix (tables.h GLL nodes)
      const cutfem_mg_level &C = mg->lv[i - 1];
      std::unordered_map<int64_t, int32_t> wc;
      auto key = [&](const std::vector<int32_t> &ijk, int64_t K) {
        return ((int64_t)ijk[3 * K] * L.hd->n_cells[1] + ijk[3 * K + 1]) * L.hd->n_cells[2] + ijk[3 * K + 2];
      };
      for (int64_t K = 0; K < C.nblk; ++K) wc[key(C.hd->blk_ijk, K)] = (int32_t)K;
      std::vector<int32_t> cmap(L.nblk, -1), fmap(C.nblk, -1);
      for (int64_t K = 0; K < L.nblk; ++K) {
        auto it = wc.find(key(L.hd->blk_ijk, K));
        if (it != wc.end()) {
          cmap[K] = it->second;
          fmap[it->second] = (int32_t)K;
        }
      }
      if ((rc = mg_upload(&L.cmap, cmap)) || (rc = mg_upload(&L.fmap, fmap))) break;
      cutfem_tables::Ref rf = cutfem_tables::build(L.degree), rcx = cutfem_tables::build(C.degree);
      std::memset(&L.tab, 0, sizeof(L.tab));
      for (int a = 0; a < L.n; ++a)
        for (int b = 0; b < C.n; ++b) L.tab.I[a * C.n + b] = (double)cutfem_tables::lag(rcx.x, b, rf.x[a]);
    }
  }
  const cutfem_mg_level &F = mg->lv.back();
  if (!rc) {
    for (double **p : {&mg->r, &mg->z, &mg->p, &mg->q, &mg->xs, &mg->bs})
      if ((rc = mg_alloc(p, F.ndof))) break;
  }
  if (!rc && ((rc = mg_alloc(&mg->partial, CG_BLOCKS)) || (rc = mg_alloc(&mg->partial2, CG_BLOCKS)) ||
              (rc = mg_pcg_cap(mg, std::max(prm->eig_iters, 1))))) {
  }
  for (int i = 0; i < n_levels && !rc; ++i) {
    if ((rc = mg_inner_setup(mg, mg->lv[i], st))) break;
    if (prm->eig_iters > 0 && (rc = mg_estimate(mg, mg->lv[i], st))) break;
  }
  if (!rc) {
    cudaError_t e = cudaStreamSynchronize(st);
    if (e != cudaSuccess) rc = fail(CUTFEM_ECUDA, cudaGetErrorString(e));
  }
  if (rc) {
    mg_free(mg);
    return rc;
  }
  *out = mg;
  return 0;
}

int cutfem_mg_lambda(const cutfem_mg *mg, double *lam_max) {
  if (!mg || !lam_max) return fail(CUTFEM_EINVAL, "null argument");
  for (size_t i = 0; i < mg->lv.size(); ++i) lam_max[i] = mg->lv[i].lam;
  return 0;
}

int cutfem_mg_set_lambda(cutfem_mg *mg, const double *lam_max) {
  if (!mg || !lam_max) return fail(CUTFEM_EINVAL, "null argument");
  for (size_t i = 0; i < mg->lv.size(); ++i)
    if (!(lam_max[i] > 0)) return fail(CUTFEM_EINVAL, "lam_max must be > 0");
  for (size_t i = 0; i < mg->lv.size(); ++i) mg->lv[i].lam = lam_max[i];
  return 0;
}

static int mg_check_vec(const cutfem_mg *mg, const void *a, const void *b) {
  if (!mg) return fail(CUTFEM_EINVAL, "null multigrid");
  if (!a || !b) return fail(CUTFEM_EINVAL, "null vector");
  if (((uintptr_t)a | (uintptr_t)b) & 15) return fail(CUTFEM_EINVAL, "vectors must be 16-byte aligned");
  if (a == b) return fail(CUTFEM_EINVAL, "vectors must not alias");
  return 0;
}

int cutfem_mg_vcycle(cutfem_mg *mg, const double *r_dev, double *z_dev, void *cuda_stream) {
  int rc;
  if ((rc = mg_check_vec(mg, r_dev, z_dev))) return rc;
  CU(cudaSetDevice(mg->device));
  return mg_cycle(mg, (int)mg->lv.size() - 1, r_dev, z_dev, (cudaStream_t)cuda_stream);
}

int cutfem_mg_pcg(cutfem_mg *mg, const double *b_dev, double *x_dev, int iters, double tol, double *res_hist,
                  int *iters_done, void *cuda_stream) {
  int rc;
  if ((rc = mg_check_vec(mg, b_dev, x_dev))) return rc;
  if (iters < 0) return fail(CUTFEM_EINVAL, "iters < 0");
  CU(cudaSetDevice(mg->device));
  cudaStream_t st = (cudaStream_t)cuda_stream;
  const int top = (int)mg->lv.size() - 1;
  auto prec = [&](const double *r, double *z) { return mg_cycle(mg, top, r, z, st); };
  int done = 0;
  if ((rc = mg_pcg_run(mg, mg->lv[top], prec, b_dev, x_dev, iters, tol, &done, st))) return rc;
  if (res_hist) {
    std::vector<double> h2(done + 1);
    CU(cudaMemcpyAsync(h2.data(), mg->rr, sizeof(double) * (done + 1), cudaMemcpyDeviceToHost, st));
    CU(cudaStreamSynchronize(st));
    for (int i = 0; i <= done; ++i) res_hist[i] = std::sqrt(h2[i]);
  } else {
    CU(cudaStreamSynchronize(st));
  }
  if (iters_done) *iters_done = done;
  return 0;
}

int cutfem_mg_smooth(cutfem_mg *mg, int32_t level, const double *r_dev, double *x_dev, int32_t degree,
                     double lam_max, double lam_min, int32_t x0_given, void *cuda_stream) {
  int rc;
  if ((rc = mg_check_vec(mg, r_dev, x_dev))) return rc;
  if (level < 0 || level >= (int)mg->lv.size() || degree < 1 || !(lam_max > lam_min) || !(lam_min > 0))
    return fail(CUTFEM_EINVAL, "level / degree / interval");
  CU(cudaSetDevice(mg->device));
  return mg_chebyshev(mg, mg->lv[level], r_dev, x_dev, degree, lam_max, lam_min, x0_given != 0,
                      (cudaStream_t)cuda_stream);
}

int cutfem_mg_transfer(cutfem_mg *mg, int32_t level, int32_t dir, const double *src_dev, double *dst_dev,
                       void *cuda_stream) {
  int rc;
  if ((rc = mg_check_vec(mg, src_dev, dst_dev))) return rc;
  if (level < 1 || level >= (int)mg->lv.size() || (dir != 0 && dir != 1))
    return fail(CUTFEM_EINVAL, "level / direction");
  CU(cudaSetDevice(mg->device));
  cudaStream_t st = (cudaStream_t)cuda_stream;
  return dir == 0 ? mg_prolong(mg, level, src_dev, dst_dev, 0, st) : mg_restrict(mg, level, src_dev, nullptr, dst_dev, st);
}

int cutfem_mg_destroy(cutfem_mg *mg) {
  if (!mg) return 0;
  cudaSetDevice(mg->device);
  cudaDeviceSynchronize();
  mg_free(mg);
  return 0;
}

}  // extern "C"
