// cg.inl — right-hand side and the CG loop around the operator (included by
// cutfem.cu; C ABI in include/cutfem.h).  BASELINE.json configs[4]: 50
// unpreconditioned CG iterations on f = 1 with Dirichlet zero via Nitsche.
//
// All vector work runs in these kernels; the CG scalars stay on the device
// (rr[k] = ||r_k||^2, pq[k] = p_k . A p_k), so an iteration needs no host sync.
// Dot products: fixed grid, per-block tree sums, one final block summing the
// partials in order -> bitwise reproducible; on a distributed handle each dot is
// then summed over ranks with ncclAllReduce (two per iteration).

namespace {

constexpr int CG_BLOCKS = 1184;  // 8 per SM: fixed, so reductions are reproducible
constexpr int CG_THREADS = 256;

__device__ __forceinline__ double block_sum(double x, double *sh) {
  const int t = threadIdx.x;
  sh[t] = x;
  __syncthreads();
  for (int s = blockDim.x / 2; s > 0; s >>= 1) {
    if (t < s) sh[t] += sh[t + s];
    __syncthreads();
  }
  return sh[0];
}

// partial[b] = sum over this block's grid-stride range of a_i * b_i (16-byte
// accesses over the pairs; an odd n -- odd p with an odd cell count -- leaves one
// tail entry, added by thread 0 of block 0)
__global__ void __launch_bounds__(CG_THREADS) k_dot(const double *__restrict__ a, const double *__restrict__ b,
                                                    int64_t n, double *__restrict__ partial) {
  __shared__ double sh[CG_THREADS];
  double s = 0.0;
  const double2 *a2 = reinterpret_cast<const double2 *>(a), *b2 = reinterpret_cast<const double2 *>(b);
  for (int64_t i = blockIdx.x * (int64_t)CG_THREADS + threadIdx.x; i < n / 2; i += (int64_t)gridDim.x * CG_THREADS) {
    const double2 x = a2[i], y = b2[i];
    s = fma(x.x, y.x, fma(x.y, y.y, s));
  }
  if ((n & 1) && blockIdx.x == 0 && threadIdx.x == 0) s = fma(a[n - 1], b[n - 1], s);
  s = block_sum(s, sh);
  if (threadIdx.x == 0) partial[blockIdx.x] = s;
}

__global__ void __launch_bounds__(CG_THREADS) k_dot_final(const double *__restrict__ partial, int np,
                                                          double *__restrict__ out) {
  __shared__ double sh[CG_THREADS];
  double s = 0.0;
  for (int i = threadIdx.x; i < np; i += CG_THREADS) s += partial[i];
  s = block_sum(s, sh);
  if (threadIdx.x == 0) *out = s;
}

// x += alpha p, r -= alpha q (alpha = rz[k] / pq[k]); with a Jacobi preconditioner
// (dinv != null) z = dinv r; partial sums of r.z (part_rz) and |r|^2 (part_rr; only
// when preconditioned -- else r.z = |r|^2)
__global__ void __launch_bounds__(CG_THREADS) k_cg_xr(double *__restrict__ x, double *__restrict__ r,
                                                      double *__restrict__ z, const double *__restrict__ dinv,
                                                      const double *__restrict__ p, const double *__restrict__ q,
                                                      int64_t n, const double *__restrict__ rz,
                                                      const double *__restrict__ pq, int k,
                                                      double *__restrict__ part_rz, double *__restrict__ part_rr) {
  __shared__ double sh[CG_THREADS];
  const double alpha = rz[k] / pq[k];
  double s = 0.0, s2 = 0.0;
  double2 *x2 = reinterpret_cast<double2 *>(x), *r2 = reinterpret_cast<double2 *>(r);
  const double2 *p2 = reinterpret_cast<const double2 *>(p), *q2 = reinterpret_cast<const double2 *>(q);
  for (int64_t i = blockIdx.x * (int64_t)CG_THREADS + threadIdx.x; i < n / 2; i += (int64_t)gridDim.x * CG_THREADS) {
    const double2 xi = x2[i], pi = p2[i], qi = q2[i], ri0 = r2[i];
    x2[i] = make_double2(fma(alpha, pi.x, xi.x), fma(alpha, pi.y, xi.y));
    const double2 ri = make_double2(fma(-alpha, qi.x, ri0.x), fma(-alpha, qi.y, ri0.y));
    r2[i] = ri;
    if (dinv) {
      const double2 di = reinterpret_cast<const double2 *>(dinv)[i];
      const double2 zi = make_double2(di.x * ri.x, di.y * ri.y);
      reinterpret_cast<double2 *>(z)[i] = zi;
      s = fma(ri.x, zi.x, fma(ri.y, zi.y, s));
      s2 = fma(ri.x, ri.x, fma(ri.y, ri.y, s2));
    } else {
      s = fma(ri.x, ri.x, fma(ri.y, ri.y, s));
    }
  }
  if ((n & 1) && blockIdx.x == 0 && threadIdx.x == 0) {  // odd n: the tail entry
    x[n - 1] = fma(alpha, p[n - 1], x[n - 1]);
    const double rt = fma(-alpha, q[n - 1], r[n - 1]);
    r[n - 1] = rt;
    if (dinv) {
      const double zt = dinv[n - 1] * rt;
      z[n - 1] = zt;
      s = fma(rt, zt, s);
      s2 = fma(rt, rt, s2);
    } else {
      s = fma(rt, rt, s);
    }
  }
  s = block_sum(s, sh);
  if (threadIdx.x == 0) part_rz[blockIdx.x] = s;
  if (dinv) {
    __syncthreads();
    s2 = block_sum(s2, sh);
    if (threadIdx.x == 0) part_rr[blockIdx.x] = s2;
  }
}

// p = z + beta p, beta = rz[k+1] / rz[k]
__global__ void __launch_bounds__(CG_THREADS) k_cg_p(double *__restrict__ p, const double *__restrict__ z, int64_t n,
                                                     const double *__restrict__ rz, int k) {
  const double beta = rz[k + 1] / rz[k];
  double2 *p2 = reinterpret_cast<double2 *>(p);
  const double2 *z2 = reinterpret_cast<const double2 *>(z);
  for (int64_t i = blockIdx.x * (int64_t)CG_THREADS + threadIdx.x; i < n / 2; i += (int64_t)gridDim.x * CG_THREADS) {
    const double2 pi = p2[i], zi = z2[i];
    p2[i] = make_double2(fma(beta, pi.x, zi.x), fma(beta, pi.y, zi.y));
  }
  if ((n & 1) && blockIdx.x == 0 && threadIdx.x == 0) p[n - 1] = fma(beta, p[n - 1], z[n - 1]);
}

// r = b - q, z = dinv r (or r), p = z, partial sums of r.z and |r|^2
__global__ void __launch_bounds__(CG_THREADS) k_cg_init(double *__restrict__ r, double *__restrict__ z,
                                                        double *__restrict__ p, const double *__restrict__ dinv,
                                                        const double *__restrict__ b, const double *__restrict__ q,
                                                        int64_t n, double *__restrict__ part_rz,
                                                        double *__restrict__ part_rr) {
  __shared__ double sh[CG_THREADS];
  double s = 0.0, s2 = 0.0;
  for (int64_t i = blockIdx.x * (int64_t)CG_THREADS + threadIdx.x; i < n; i += (int64_t)gridDim.x * CG_THREADS) {
    const double ri = b[i] - q[i];
    const double zi = dinv ? dinv[i] * ri : ri;
    r[i] = ri;
    if (dinv) z[i] = zi;
    p[i] = zi;
    s = fma(ri, zi, s);
    s2 = fma(ri, ri, s2);
  }
  s = block_sum(s, sh);
  if (threadIdx.x == 0) part_rz[blockIdx.x] = s;
  __syncthreads();
  s2 = block_sum(s2, sh);
  if (threadIdx.x == 0) part_rr[blockIdx.x] = s2;
}

// dinv = 1 / d (the Jacobi preconditioner from the probed diagonal)
__global__ void k_recip(double *__restrict__ d, int64_t n) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    d[i] = 1.0 / d[i];
}

// diagonal probing: u[e] = 1 on the entries of probe (colour, local index), else 0
__global__ void k_probe_unit(double *__restrict__ u, const int32_t *__restrict__ probe_of, int32_t probe, int64_t n) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    u[i] = probe_of[i] == probe ? 1.0 : 0.0;
}
// d[e] = v[e] on the entries of the probe
__global__ void k_probe_take(double *__restrict__ d, const double *__restrict__ v, const int32_t *__restrict__ probe_of,
                             int32_t probe, int64_t n) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    if (probe_of[i] == probe) d[i] = v[i];
}

// ---- right-hand side b = f int_Ω phi_i
struct RhsTab {
  double m[CUTFEM_NMAX];  // int_0^1 l_a = sum_q w_q l_a(g_q)
  double x[CUTFEM_NMAX];  // GLL nodes
  double cinv[CUTFEM_NMAX];
};

// uncut cells: b = f h^3 m_a m_b m_c (tensor Gauss, exact)
__global__ void k_rhs_uncut(double *__restrict__ b, const UDesc *__restrict__ desc, int64_t ncell, int n, double fh3,
                            RhsTab t) {
  const int n3 = n * n * n;
  const int64_t total = ncell * n3;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total; e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t c = e / n3;
    const int l = (int)(e - c * n3);
    const int a = l % n, bb = (l / n) % n, cc = l / (n * n);
    b[(size_t)desc[c].blk * n3 + l] = fh3 * t.m[a] * t.m[bb] * t.m[cc];
  }
}

// cut cells (one CTA per cell): b_l = f sum_q W_q phi_l(x_q) over the volume rule;
// 1-D bases of a point chunk staged in shared memory
__global__ void __launch_bounds__(128) k_rhs_cut(double *__restrict__ b, const CDesc *__restrict__ desc,
                                                 const double *__restrict__ vol, int n, double f, RhsTab t) {
  __shared__ double bas[128][3][CUTFEM_NMAX];
  __shared__ double wq[128];
  const CDesc d = desc[blockIdx.x];
  const int n3 = n * n * n;
  double acc[6] = {0, 0, 0, 0, 0, 0};  // n^3 <= 729 -> <= 6 per thread
  for (int64_t q0 = 0; q0 < d.nv; q0 += 128) {
    const int cnt = (int)min((int64_t)128, (int64_t)d.nv - q0);
    if (threadIdx.x < cnt) {
      const double *pq = vol + 4 * (d.vb + q0 + threadIdx.x);
      for (int dim = 0; dim < 3; ++dim) {
        const double xv = pq[dim];
        for (int a = 0; a < n; ++a) {
          double prod = t.cinv[a];
          for (int m = 0; m < n; ++m)
            if (m != a) prod *= xv - t.x[m];
          bas[threadIdx.x][dim][a] = prod;
        }
      }
      wq[threadIdx.x] = pq[3];
    }
    __syncthreads();
    for (int k = 0; k < 6; ++k) {
      const int l = threadIdx.x + 128 * k;
      if (l >= n3) break;
      const int a = l % n, bb = (l / n) % n, cc = l / (n * n);
      double s = acc[k];
      for (int q = 0; q < cnt; ++q) s = fma(wq[q] * bas[q][0][a], bas[q][1][bb] * bas[q][2][cc], s);
      acc[k] = s;
    }
    __syncthreads();
  }
  for (int k = 0; k < 6; ++k) {
    const int l = threadIdx.x + 128 * k;
    if (l < n3) b[(size_t)d.blk * n3 + l] = f * acc[k];
  }
}

}  // namespace

struct cutfem_cg_work {
  double *r = nullptr, *p = nullptr, *q = nullptr, *z = nullptr, *partial = nullptr, *partial2 = nullptr;
  double *rr = nullptr, *rz = nullptr, *pq = nullptr, *bb = nullptr;
  double *dinv = nullptr;         // Jacobi: 1 / diag(A) (probed, lazily)
  int32_t *probe_of = nullptr;    // probe index of every entry (diagonal probing)
  int64_t n = 0, n_p = 0;         // vector length; p length (ghost room for a distributed apply)
  int cap = 0;                    // iterations the scalar arrays hold
};

void cg_free(cutfem_cg_work *w) {
  if (!w) return;
  for (double *x : {w->r, w->p, w->q, w->z, w->partial, w->partial2, w->rr, w->rz, w->pq, w->bb, w->dinv}) cudaFree(x);
  cudaFree(w->probe_of);
  delete w;
}

namespace {

int cg_alloc(cutfem_cg_work &w, int64_t n, int64_t n_p, int iters, int64_t &dev_bytes) {
  if (!w.r) {
    w.n = n;
    w.n_p = n_p;
    CU(cudaMalloc(&w.r, sizeof(double) * std::max<int64_t>(n, 2)));
    CU(cudaMalloc(&w.z, sizeof(double) * std::max<int64_t>(n, 2)));
    CU(cudaMalloc(&w.p, sizeof(double) * std::max<int64_t>(n_p, 2)));  // ghost room for the apply
    CU(cudaMalloc(&w.q, sizeof(double) * std::max<int64_t>(n, 2)));
    CU(cudaMalloc(&w.partial, sizeof(double) * CG_BLOCKS));
    CU(cudaMalloc(&w.partial2, sizeof(double) * CG_BLOCKS));
    CU(cudaMalloc(&w.bb, sizeof(double) * 2));
    dev_bytes += (int64_t)sizeof(double) * (3 * n + n_p + 2 * CG_BLOCKS);
  }
  if (w.cap < iters + 1) {
    cudaFree(w.rr);
    cudaFree(w.rz);
    cudaFree(w.pq);
    w.cap = iters + 1;
    CU(cudaMalloc(&w.rr, sizeof(double) * (w.cap + 1)));
    CU(cudaMalloc(&w.rz, sizeof(double) * (w.cap + 1)));
    CU(cudaMalloc(&w.pq, sizeof(double) * (w.cap + 1)));
  }
  return 0;
}

// Jacobi diagonal by probing (P:228's "column by column through unit vectors"): for
// every probe index k, u = 1 on the entries of probe k, v = A u, diag = v there.  The
// probe classes are chosen so that no two entries of one class couple (the caller's
// colouring), so v on a probed entry is exactly its diagonal entry.  dinv = 1 / diag.
template <class Apply>
int cg_probe_diag(cutfem_cg_work &w, int nprobe, Apply apply, cudaStream_t st, int sms, int64_t &dev_bytes) {
  const unsigned g = (unsigned)std::min<int64_t>((w.n_p + 255) / 256, 16 * sms);
  if (!w.dinv) {
    CU(cudaMalloc(&w.dinv, sizeof(double) * std::max<int64_t>(w.n, 2)));
    dev_bytes += (int64_t)sizeof(double) * w.n;
  }
  for (int k = 0; k < nprobe; ++k) {
    k_probe_unit<<<g, 256, 0, st>>>(w.p, w.probe_of, k, w.n_p);
    CU(cudaGetLastError());
    int rc = apply(w.p, w.q);
    if (rc) return rc;
    k_probe_take<<<g, 256, 0, st>>>(w.dinv, w.q, w.probe_of, k, w.n);
    CU(cudaGetLastError());
  }
  k_recip<<<g, 256, 0, st>>>(w.dinv, w.n);
  CU(cudaGetLastError());
  return 0;
}

// (Preconditioned) conjugate gradients, every vector operation in the kernels above,
// the scalars on the device (no host sync per iteration unless tol > 0).
template <class Apply, class Reduce>
int cg_run(cutfem_cg_work &w, Apply apply, Reduce reduce, const double *b, double *x, int iters, double tol,
           bool jacobi, double *res_hist, int *iters_done, cudaStream_t st) {
  const int64_t n = w.n;
  const double *dinv = jacobi ? w.dinv : nullptr;
  double *z = jacobi ? w.z : w.r;
  int rc;
  // r0 = b - A x0, z0 = M^-1 r0, p0 = z0
  if ((rc = apply(x, w.q))) return rc;
  k_cg_init<<<CG_BLOCKS, CG_THREADS, 0, st>>>(w.r, z, w.p, dinv, b, w.q, n, w.partial, w.partial2);
  CU(cudaGetLastError());
  if ((rc = reduce(w.partial, w.rz))) return rc;
  if ((rc = reduce(w.partial2, w.rr))) return rc;
  double bb = 0.0;
  if (tol > 0) {
    k_dot<<<CG_BLOCKS, CG_THREADS, 0, st>>>(b, b, n, w.partial);
    if ((rc = reduce(w.partial, w.bb))) return rc;
    CU(cudaMemcpyAsync(&bb, w.bb, sizeof(double), cudaMemcpyDeviceToHost, st));
    CU(cudaStreamSynchronize(st));
  }
  int k = 0;
  for (; k < iters; ++k) {
    if ((rc = apply(w.p, w.q))) return rc;  // q = A p
    k_dot<<<CG_BLOCKS, CG_THREADS, 0, st>>>(w.p, w.q, n, w.partial);
    if ((rc = reduce(w.partial, w.pq + k))) return rc;
    k_cg_xr<<<CG_BLOCKS, CG_THREADS, 0, st>>>(x, w.r, z, dinv, w.p, w.q, n, w.rz, w.pq, k, w.partial, w.partial2);
    CU(cudaGetLastError());
    if ((rc = reduce(w.partial, w.rz + k + 1))) return rc;
    if (jacobi && (rc = reduce(w.partial2, w.rr + k + 1))) return rc;
    k_cg_p<<<CG_BLOCKS, CG_THREADS, 0, st>>>(w.p, z, n, w.rz, k);
    CU(cudaGetLastError());
    if (tol > 0) {
      double rk = 0.0;
      CU(cudaMemcpyAsync(&rk, (jacobi ? w.rr : w.rz) + k + 1, sizeof(double), cudaMemcpyDeviceToHost, st));
      CU(cudaStreamSynchronize(st));
      if (std::sqrt(rk) <= tol * std::sqrt(bb)) {
        ++k;
        break;
      }
    }
  }
  if (res_hist) {
    std::vector<double> h2(k + 1);
    if (jacobi) {
      CU(cudaMemcpyAsync(h2.data(), w.rr, sizeof(double) * (k + 1), cudaMemcpyDeviceToHost, st));
    } else {  // |r_0|^2 from the init, |r_k|^2 = r.z for k >= 1
      CU(cudaMemcpyAsync(h2.data(), w.rz, sizeof(double) * (k + 1), cudaMemcpyDeviceToHost, st));
    }
    CU(cudaStreamSynchronize(st));
    for (int i = 0; i <= k; ++i) res_hist[i] = std::sqrt(h2[i]);
  } else {
    CU(cudaStreamSynchronize(st));
  }
  if (iters_done) *iters_done = k;
  return 0;
}

int cg_reduce(cutfem_handle *hd, double *partial, double *out, cudaStream_t st) {
  k_dot_final<<<1, CG_THREADS, 0, st>>>(partial, CG_BLOCKS, out);
  CU(cudaGetLastError());
  if (hd && hd->dist && hd->comm && (hd->nranks > 1 || hd->loopback)) {
    ncclResult_t r = ncclAllReduce(out, out, 1, ncclDouble, ncclSum, (ncclComm_t)hd->comm, st);
    if (r != ncclSuccess) return fail(CUTFEM_ENCCL, std::string("ncclAllReduce: ") + ncclGetErrorString(r));
  }
  return 0;
}

// DG probe classes: block colour (i + j + k) mod 2 (face neighbours differ) x local index
int dg_probes(cutfem_handle *hd, cutfem_cg_work &w) {
  if (w.probe_of) return 0;
  const int n3 = hd->n * hd->n * hd->n;
  std::vector<int32_t> pr((size_t)w.n_p, -1);
  for (int64_t K = 0; K < (int64_t)hd->blk_ijk.size() / 3; ++K) {
    const int c = (int)((hd->blk_ijk[3 * K] + hd->blk_ijk[3 * K + 1] + hd->blk_ijk[3 * K + 2]) & 1);
    for (int l = 0; l < n3; ++l) pr[(size_t)K * n3 + l] = c * n3 + l;
  }
  return upload(hd, &w.probe_of, pr.data(), pr.size());
}

}  // namespace

extern "C" {

int cutfem_rhs_const(cutfem_handle *hd, double f, double *b_dev, void *cuda_stream) {
  if (!hd) return fail(CUTFEM_EINVAL, "null handle");
  if (hd->stats.n_dofs > 0 && !b_dev) return fail(CUTFEM_EINVAL, "null vector");
  CU(cudaSetDevice(hd->device));
  cudaStream_t st = (cudaStream_t)cuda_stream;
  const int n = hd->n, p = hd->degree;
  cutfem_tables::Ref r = cutfem_tables::build(p);
  RhsTab t;
  std::memset(&t, 0, sizeof(t));
  for (int a = 0; a < n; ++a) {
    long double m = 0;
    for (int q = 0; q < n; ++q) m += r.w[q] * cutfem_tables::lag(r.x, a, r.g[q]);
    t.m[a] = (double)m;
    t.x[a] = (double)r.x[a];
    t.cinv[a] = (double)r.cinv[a];
  }
  const double h = hd->h;
  if (hd->n_uncut > 0) {
    const int64_t total = hd->n_uncut * (int64_t)n * n * n;
    const unsigned grid = (unsigned)std::min<int64_t>((total + 255) / 256, 8 * hd->sm_count);
    k_rhs_uncut<<<grid, 256, 0, st>>>(b_dev, hd->d_udesc, hd->n_uncut, n, f * h * h * h, t);
    CU(cudaGetLastError());
  }
  if (hd->n_cut > 0) {
    k_rhs_cut<<<(unsigned)hd->n_cut, 128, 0, st>>>(b_dev, hd->d_cdesc, hd->d_vol, n, f, t);
    CU(cudaGetLastError());
  }
  return 0;
}

int cutfem_pcg(cutfem_handle *hd, const double *b_dev, double *x_dev, int iters, double tol, int precond,
               double *res_hist, int *iters_done, void *cuda_stream) {
  if (!hd) return fail(CUTFEM_EINVAL, "null handle");
  if (iters < 0) return fail(CUTFEM_EINVAL, "iters < 0");
  if (precond != CUTFEM_PRECOND_NONE && precond != CUTFEM_PRECOND_JACOBI) return fail(CUTFEM_EINVAL, "precond");
  if (hd->stats.n_dofs > 0 && (!b_dev || !x_dev)) return fail(CUTFEM_EINVAL, "null vector");
  if (((uintptr_t)b_dev | (uintptr_t)x_dev) & 15) return fail(CUTFEM_EINVAL, "vectors must be 16-byte aligned");
  if (b_dev == x_dev && hd->stats.n_dofs > 0) return fail(CUTFEM_EINVAL, "b and x must not alias");
  CU(cudaSetDevice(hd->device));
  cudaStream_t st = (cudaStream_t)cuda_stream;
  if (!hd->cg) hd->cg = new cutfem_cg_work();
  cutfem_cg_work &w = *hd->cg;
  int rc;
  if ((rc = cg_alloc(w, hd->stats.n_dofs, hd->stats.n_ext_dofs, iters, hd->dev_bytes))) return rc;
  auto apply = [&](const double *u, double *v) { return dispatch_apply(hd, u, v, st); };
  auto reduce = [&](double *part, double *out) { return cg_reduce(hd, part, out, st); };
  const bool jac = precond == CUTFEM_PRECOND_JACOBI;
  if (jac && !w.dinv) {
    if ((rc = dg_probes(hd, w))) return rc;
    if ((rc = cg_probe_diag(w, 2 * hd->n * hd->n * hd->n, apply, st, hd->sm_count, hd->dev_bytes))) return rc;
  }
  return cg_run(w, apply, reduce, b_dev, x_dev, iters, tol, jac, res_hist, iters_done, st);
}

int cutfem_cg(cutfem_handle *hd, const double *b_dev, double *x_dev, int iters, double tol, double *res_hist,
              int *iters_done, void *cuda_stream) {
  return cutfem_pcg(hd, b_dev, x_dev, iters, tol, CUTFEM_PRECOND_NONE, res_hist, iters_done, cuda_stream);
}

int cutfem_diag(cutfem_handle *hd, double *d_dev, void *cuda_stream) {
  if (!hd) return fail(CUTFEM_EINVAL, "null handle");
  if (hd->stats.n_dofs > 0 && !d_dev) return fail(CUTFEM_EINVAL, "null vector");
  CU(cudaSetDevice(hd->device));
  cudaStream_t st = (cudaStream_t)cuda_stream;
  if (!hd->cg) hd->cg = new cutfem_cg_work();
  cutfem_cg_work &w = *hd->cg;
  int rc;
  if ((rc = cg_alloc(w, hd->stats.n_dofs, hd->stats.n_ext_dofs, 1, hd->dev_bytes))) return rc;
  auto apply = [&](const double *u, double *v) { return dispatch_apply(hd, u, v, st); };
  if (!w.dinv) {
    if ((rc = dg_probes(hd, w))) return rc;
    if ((rc = cg_probe_diag(w, 2 * hd->n * hd->n * hd->n, apply, st, hd->sm_count, hd->dev_bytes))) return rc;
  }
  const unsigned g = (unsigned)std::min<int64_t>((w.n + 255) / 256, 16 * hd->sm_count);
  CU(cudaMemcpyAsync(d_dev, w.dinv, sizeof(double) * w.n, cudaMemcpyDeviceToDevice, st));
  k_recip<<<g, 256, 0, st>>>(d_dev, w.n);
  CU(cudaGetLastError());
  return 0;
}

}  // extern "C"
