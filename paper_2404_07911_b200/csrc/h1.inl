// h1.inl — the H^1-conforming (continuous Galerkin) CutFEM operator (SURVEY §8(f)
// f2; PAPER eq:bilinear_cg P:68-76 with the face ghost penalty), included by
// cutfem.cu.  C ABI in include/cutfem.h (cutfem_h1_*).
//
// The continuous Q_p space of the active cells (GLL nodes, shared on faces, edges
// and vertices) has the global basis  phi_g = sum over the cell basis functions on
// lattice node g,  so  A_CG = P^T A P  with P the 0/1 gather from the global vector
// to the cell blocks and A the block operator WITHOUT the SIPG terms (volume,
// Nitsche, ghost penalty: the same integrals; the j = 0 ghost-penalty jump of a
// continuous field is 0).  The apply is therefore three stream-ordered steps:
//   1. gather  ub[K, l] = u[map[K, l]]                  (k_h1_gather, coalesced writes)
//   2. vb = A ub  with the DG kernels (k_cutp / k_tile2 / k_uncw / k_cut / k_cell),
//      SIPG masked off at setup
//   3. scatter v[g] = sum of vb over the (<= 8) block entries of node g, in a fixed
//      order, one thread per node -- conflict free, no atomics (k_h1_scatter)
// Global numbering: lattice node (p i + a, p j + b, p k + c) of cell (i, j, k), local
// l = a + n b + n^2 c; the nodes of active cells in lexicographic order (x slowest).

struct cutfem_h1 {
  cutfem_handle *dg = nullptr;  // block operator, SIPG masked off
  int device = 0;
  int64_t n_h1 = 0, n_blk = 0;  // global nodes; block entries n_active * n^3
  int32_t *d_map = nullptr;     // [n_blk] global node of each block entry
  int64_t *d_rp = nullptr;      // [n_h1 + 1] inverse map row pointers
  int32_t *d_ent = nullptr;     // [n_blk] block entries of each node, ascending
  double *d_ub = nullptr, *d_vb = nullptr;
  std::vector<int32_t> map;     // host copy (cutfem_h1_map)
  std::vector<int64_t> lat;     // lattice coordinates of every node (3 per node): probe colouring
  cutfem_cg_work *cg = nullptr;
};

int cutfem_h1_apply_impl(cutfem_h1 *h, const double *u_dev, double *v_dev, cudaStream_t st);

namespace {

__global__ void k_h1_gather(double *__restrict__ ub, const double *__restrict__ u, const int32_t *__restrict__ map,
                            int64_t n) {
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < n; e += (int64_t)gridDim.x * blockDim.x)
    ub[e] = __ldg(u + map[e]);
}

__global__ void k_h1_scatter(double *__restrict__ v, const double *__restrict__ vb, const int64_t *__restrict__ rp,
                             const int32_t *__restrict__ ent, int64_t n) {
  for (int64_t g = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; g < n; g += (int64_t)gridDim.x * blockDim.x) {
    double s = 0.0;
    for (int64_t k = rp[g]; k < rp[g + 1]; ++k) s += vb[ent[k]];
    v[g] = s;
  }
}

void h1_free(cutfem_h1 *h) {
  if (!h) return;
  cg_free(h->cg);
  if (h->dg) free_handle(h->dg);
  cudaFree(h->d_map);
  cudaFree(h->d_rp);
  cudaFree(h->d_ent);
  cudaFree(h->d_ub);
  cudaFree(h->d_vb);
  delete h;
}

// lattice colouring (I, J, K) mod (2p+1): nodes of one class share no cell and no
// ghost-penalty face pair (a GP face couples nodes <= 2p lattice steps apart)
int h1_probe_diag(cutfem_h1 *h, cudaStream_t st) {
  cutfem_cg_work &w = *h->cg;
  const int m = 2 * h->dg->degree + 1;
  if (!w.probe_of) {
    std::vector<int32_t> pr((size_t)h->n_h1);
    for (int64_t g = 0; g < h->n_h1; ++g)
      pr[g] = (int32_t)(((h->lat[3 * g] % m) * m + h->lat[3 * g + 1] % m) * m + h->lat[3 * g + 2] % m);
    int rc = upload(h->dg, &w.probe_of, pr.data(), pr.size());
    if (rc) return rc;
  }
  auto apply = [&](const double *u, double *v) { return cutfem_h1_apply_impl(h, u, v, st); };
  return cg_probe_diag(w, m * m * m, apply, st, h->dg->sm_count, h->dg->dev_bytes);
}

}  // namespace

extern "C" {

int cutfem_h1_setup(const cutfem_problem *pb, int device, cutfem_h1 **out) {
  if (!out) return fail(CUTFEM_EINVAL, "out is NULL");
  *out = nullptr;
  if (!pb) return fail(CUTFEM_EINVAL, "null problem");
  cutfem_problem q = *pb;
  const uint32_t m = pb->term_mask ? pb->term_mask : CUTFEM_TERM_ALL;
  q.term_mask = m & (CUTFEM_TERM_CELL | CUTFEM_TERM_NITSCHE | CUTFEM_TERM_GP);
  if (!q.term_mask) q.term_mask = CUTFEM_TERM_CELL;  // (a mask of SIPG alone: the H1 operator has no SIPG)
  cutfem_h1 *h = new (std::nothrow) cutfem_h1();
  if (!h) return fail(CUTFEM_ENOMEM, "host allocation");
  h->device = device;
  h->dg = new (std::nothrow) cutfem_handle();
  if (!h->dg) {
    delete h;
    return fail(CUTFEM_ENOMEM, "host allocation");
  }
  int rc = setup_impl(&q, device, h->dg);
  if (rc) {
    h1_free(h);
    return rc;
  }
  if (pb->term_mask && !(pb->term_mask & (CUTFEM_TERM_CELL | CUTFEM_TERM_NITSCHE | CUTFEM_TERM_GP)))
    h->dg->kp.mask = 0;  // SIPG only requested: the H1 operator is zero
  h->dg->stats.dev_bytes = h->dg->dev_bytes;
  // ---- numbering (host): lattice keys of every block entry, sorted unique
  const int p = pb->degree, n = p + 1, n3 = n * n * n;
  const int64_t na = pb->n_active;
  h->n_blk = na * n3;
  if (h->n_blk > INT32_MAX) {
    h1_free(h);
    return fail(CUTFEM_EUNSUPPORTED, "H1 operator: block entries need int32");
  }
  const int64_t LX = (int64_t)pb->n_cells[0] * p + 1, LY = (int64_t)pb->n_cells[1] * p + 1,
                LZ = (int64_t)pb->n_cells[2] * p + 1;
  std::vector<int64_t> key(h->n_blk);
  for (int64_t K = 0; K < na; ++K) {
    const int64_t i = pb->active_ijk[3 * K], j = pb->active_ijk[3 * K + 1], k = pb->active_ijk[3 * K + 2];
    for (int c = 0; c < n; ++c)
      for (int b = 0; b < n; ++b)
        for (int a = 0; a < n; ++a)
          key[K * n3 + a + n * b + n * n * c] = ((p * i + a) * LY + (p * j + b)) * LZ + (p * k + c);
  }
  (void)LX;
  std::vector<int64_t> uk(key);
  std::sort(uk.begin(), uk.end());
  uk.erase(std::unique(uk.begin(), uk.end()), uk.end());
  h->n_h1 = (int64_t)uk.size();
  if (h->n_h1 > INT32_MAX) {
    h1_free(h);
    return fail(CUTFEM_EUNSUPPORTED, "H1 operator: nodes need int32");
  }
  h->lat.resize(3 * h->n_h1);
  for (int64_t g = 0; g < h->n_h1; ++g) {
    h->lat[3 * g] = uk[g] / (LY * LZ);
    h->lat[3 * g + 1] = (uk[g] / LZ) % LY;
    h->lat[3 * g + 2] = uk[g] % LZ;
  }
  h->map.resize(h->n_blk);
  std::vector<int64_t> rp(h->n_h1 + 1, 0);
  for (int64_t e = 0; e < h->n_blk; ++e) {
    const int32_t g = (int32_t)(std::lower_bound(uk.begin(), uk.end(), key[e]) - uk.begin());
    h->map[e] = g;
    ++rp[g + 1];
  }
  for (int64_t g = 0; g < h->n_h1; ++g) rp[g + 1] += rp[g];
  std::vector<int32_t> ent(h->n_blk);
  {
    std::vector<int64_t> pos(rp.begin(), rp.end() - 1);
    for (int64_t e = 0; e < h->n_blk; ++e) ent[pos[h->map[e]]++] = (int32_t)e;  // ascending e per node
  }
  cutfem_handle *dg = h->dg;
  if ((rc = upload(dg, &h->d_map, h->map.data(), h->map.size())) || (rc = upload(dg, &h->d_rp, rp.data(), rp.size())) ||
      (rc = upload(dg, &h->d_ent, ent.data(), ent.size()))) {
    h1_free(h);
    return rc;
  }
  if (cudaMalloc(&h->d_ub, sizeof(double) * std::max<int64_t>(h->n_blk, 2)) != cudaSuccess ||
      cudaMalloc(&h->d_vb, sizeof(double) * std::max<int64_t>(h->n_blk, 2)) != cudaSuccess) {
    h1_free(h);
    return fail(CUTFEM_ENOMEM, "H1 block scratch");
  }
  dg->dev_bytes += 2 * (int64_t)sizeof(double) * h->n_blk;
  *out = h;
  return 0;
}

int cutfem_h1_ndofs(const cutfem_h1 *h, int64_t *n_h1) {
  if (!h || !n_h1) return fail(CUTFEM_EINVAL, "null");
  *n_h1 = h->n_h1;
  return 0;
}

int cutfem_h1_map(const cutfem_h1 *h, int32_t *map_host) {
  if (!h || (!map_host && h->n_blk)) return fail(CUTFEM_EINVAL, "null");
  std::memcpy(map_host, h->map.data(), sizeof(int32_t) * h->map.size());
  return 0;
}

int cutfem_h1_apply(cutfem_h1 *h, const double *u_dev, double *v_dev, void *cuda_stream) {
  if (!h) return fail(CUTFEM_EINVAL, "null handle");
  if (h->n_h1 > 0 && (!u_dev || !v_dev)) return fail(CUTFEM_EINVAL, "null vector");
  if (u_dev == v_dev && h->n_h1 > 0) return fail(CUTFEM_EINVAL, "u and v must not alias");
  if (((uintptr_t)u_dev | (uintptr_t)v_dev) & 7) return fail(CUTFEM_EINVAL, "vectors must be 8-byte aligned");
  if (h->n_h1 == 0) return 0;
  CU(cudaSetDevice(h->device));
  return cutfem_h1_apply_impl(h, u_dev, v_dev, (cudaStream_t)cuda_stream);
}

}  // extern "C"

int cutfem_h1_apply_impl(cutfem_h1 *h, const double *u_dev, double *v_dev, cudaStream_t st) {
  const int sms = h->dg->sm_count;
  const unsigned gb = (unsigned)std::min<int64_t>((h->n_blk + 255) / 256, 16 * sms);
  k_h1_gather<<<gb, 256, 0, st>>>(h->d_ub, u_dev, h->d_map, h->n_blk);
  CU(cudaGetLastError());
  int rc = dispatch_apply(h->dg, h->d_ub, h->d_vb, st);
  if (rc) return rc;
  const unsigned gs = (unsigned)std::min<int64_t>((h->n_h1 + 255) / 256, 16 * sms);
  k_h1_scatter<<<gs, 256, 0, st>>>(v_dev, h->d_vb, h->d_rp, h->d_ent, h->n_h1);
  CU(cudaGetLastError());
  return 0;
}

extern "C" {

int cutfem_h1_rhs_const(cutfem_h1 *h, double f, double *b_dev, void *cuda_stream) {
  if (!h) return fail(CUTFEM_EINVAL, "null handle");
  if (h->n_h1 > 0 && !b_dev) return fail(CUTFEM_EINVAL, "null vector");
  if (h->n_h1 == 0) return 0;
  CU(cudaSetDevice(h->device));
  cudaStream_t st = (cudaStream_t)cuda_stream;
  int rc = cutfem_rhs_const(h->dg, f, h->d_vb, st);
  if (rc) return rc;
  const unsigned gs = (unsigned)std::min<int64_t>((h->n_h1 + 255) / 256, 16 * h->dg->sm_count);
  k_h1_scatter<<<gs, 256, 0, st>>>(b_dev, h->d_vb, h->d_rp, h->d_ent, h->n_h1);
  CU(cudaGetLastError());
  return 0;
}

int cutfem_h1_pcg(cutfem_h1 *h, const double *b_dev, double *x_dev, int iters, double tol, int precond,
                  double *res_hist, int *iters_done, void *cuda_stream) {
  if (!h) return fail(CUTFEM_EINVAL, "null handle");
  if (iters < 0) return fail(CUTFEM_EINVAL, "iters < 0");
  if (precond != CUTFEM_PRECOND_NONE && precond != CUTFEM_PRECOND_JACOBI) return fail(CUTFEM_EINVAL, "precond");
  if (h->n_h1 > 0 && (!b_dev || !x_dev)) return fail(CUTFEM_EINVAL, "null vector");
  if (((uintptr_t)b_dev | (uintptr_t)x_dev) & 15) return fail(CUTFEM_EINVAL, "vectors must be 16-byte aligned");
  if (b_dev == x_dev && h->n_h1 > 0) return fail(CUTFEM_EINVAL, "b and x must not alias");
  CU(cudaSetDevice(h->device));
  cudaStream_t st = (cudaStream_t)cuda_stream;
  if (!h->cg) h->cg = new cutfem_cg_work();
  cutfem_cg_work &w = *h->cg;
  int rc;
  if ((rc = cg_alloc(w, h->n_h1, h->n_h1, iters, h->dg->dev_bytes))) return rc;
  auto apply = [&](const double *u, double *v) { return cutfem_h1_apply(h, u, v, st); };
  auto reduce = [&](double *part, double *out) { return cg_reduce(nullptr, part, out, st); };
  const bool jac = precond == CUTFEM_PRECOND_JACOBI;
  if (jac && !w.dinv && (rc = h1_probe_diag(h, st))) return rc;
  return cg_run(w, apply, reduce, b_dev, x_dev, iters, tol, jac, res_hist, iters_done, st);
}

int cutfem_h1_diag(cutfem_h1 *h, double *d_dev, void *cuda_stream) {
  if (!h) return fail(CUTFEM_EINVAL, "null handle");
  if (h->n_h1 > 0 && !d_dev) return fail(CUTFEM_EINVAL, "null vector");
  CU(cudaSetDevice(h->device));
  cudaStream_t st = (cudaStream_t)cuda_stream;
  if (!h->cg) h->cg = new cutfem_cg_work();
  cutfem_cg_work &w = *h->cg;
  int rc;
  if ((rc = cg_alloc(w, h->n_h1, h->n_h1, 1, h->dg->dev_bytes))) return rc;
  if (!w.dinv && (rc = h1_probe_diag(h, st))) return rc;
  const unsigned g = (unsigned)std::min<int64_t>((w.n + 255) / 256, 16 * h->dg->sm_count);
  CU(cudaMemcpyAsync(d_dev, w.dinv, sizeof(double) * w.n, cudaMemcpyDeviceToDevice, st));
  k_recip<<<g, 256, 0, st>>>(d_dev, w.n);
  CU(cudaGetLastError());
  return 0;
}

int cutfem_h1_stats(const cutfem_h1 *h, cutfem_stats_t *out) {
  if (!h || !out) return fail(CUTFEM_EINVAL, "null");
  *out = h->dg->stats;
  out->dev_bytes = h->dg->dev_bytes;
  return 0;
}

int cutfem_h1_destroy(cutfem_h1 *h) {
  if (!h) return 0;
  cudaSetDevice(h->device);
  cudaDeviceSynchronize();
  h1_free(h);
  return 0;
}

}  // extern "C"
