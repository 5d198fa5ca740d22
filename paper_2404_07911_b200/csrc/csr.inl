// csr.inl — the sparse-matrix comparison path (included by cutfem.cu).
//
// PAPER.md §3.1: the operator is equivalent to y = A u with the
// assembled matrix A; "the local matrices A_e can also be computed
// column-by-column by applying I_e B_e E_e on element-wise unit vectors".
// cutfem_csr_assemble does exactly that on the device, batched: DG couples
// only face neighbours, and the colour c(K) = (i + 2j + 3k) mod 7 gives any two
// cells of one colour an L1 distance >= 3, so their closed neighbourhoods are
// disjoint.  For each colour and local DoF l, one matrix-free apply on the
// probe u = sum_{K of colour c} e_{K,l} yields column (K,l) of A in the
// neighbourhood of every K of that colour at once: 7 (p+1)^3 applies in total.
// The SpMV itself is cuSPARSE (the library baseline named by north_star).

namespace {

__global__ void k_csr_cols32(const int32_t *__restrict__ nbl, const int32_t *__restrict__ nbc,
                             const int64_t *__restrict__ rowptr64, int32_t *__restrict__ col, int64_t nrows,
                             int n3) {
  const int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (r >= nrows) return;
  const int64_t B = r / n3;
  int64_t pos = rowptr64[r];
  const int cnt = nbc[B];
  for (int k = 0; k < cnt; ++k) {
    const int32_t K = nbl[B * 7 + k];
    for (int l = 0; l < n3; ++l) col[pos++] = (int32_t)((int64_t)K * n3 + l);
  }
}

__global__ void k_csr_cols64(const int32_t *__restrict__ nbl, const int32_t *__restrict__ nbc,
                             const int64_t *__restrict__ rowptr64, int64_t *__restrict__ col, int64_t nrows,
                             int n3) {
  const int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (r >= nrows) return;
  const int64_t B = r / n3;
  int64_t pos = rowptr64[r];
  const int cnt = nbc[B];
  for (int k = 0; k < cnt; ++k) {
    const int64_t K = nbl[B * 7 + k];
    for (int l = 0; l < n3; ++l) col[pos++] = K * n3 + l;
  }
}

__global__ void k_probe_set(double *__restrict__ u, const uint8_t *__restrict__ color, int64_t nblk, int n3,
                            int c, int l) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= nblk * n3) return;
  const int64_t B = i / n3;
  u[i] = (color[B] == c && (i % n3) == l) ? 1.0 : 0.0;
}

__global__ void k_probe_scatter(const double *__restrict__ v, const uint8_t *__restrict__ color,
                                const int32_t *__restrict__ nbl, const int32_t *__restrict__ nbc,
                                const int64_t *__restrict__ rowptr64, double *__restrict__ val, int64_t nrows,
                                int n3, int c, int l) {
  const int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (r >= nrows) return;
  const int64_t B = r / n3;
  const int cnt = nbc[B];
  for (int k = 0; k < cnt; ++k) {
    const int32_t K = nbl[B * 7 + k];
    if (color[K] == c) {
      val[rowptr64[r] + (int64_t)k * n3 + l] = v[r];
      return;
    }
  }
}

int csr_free(cutfem_handle *hd) {
  if (hd->spA) cusparseDestroySpMat(hd->spA);
  hd->spA = nullptr;
  cudaFree(hd->d_rowptr);
  cudaFree(hd->d_col);
  cudaFree(hd->d_val);
  cudaFree(hd->d_spbuf);
  hd->d_rowptr = hd->d_col = nullptr;
  hd->d_val = nullptr;
  hd->d_spbuf = nullptr;
  hd->spbuf_size = 0;
  hd->csr_nnz = 0;
  return 0;
}

int csr_make_descr(cutfem_handle *hd) {
  if (!hd->sp && cusparseCreate(&hd->sp) != CUSPARSE_STATUS_SUCCESS)
    return fail(CUTFEM_ECUDA, "cusparseCreate failed");
  const int64_t nrows = hd->stats.n_dofs;
  const cusparseIndexType_t it = hd->csr_i64 ? CUSPARSE_INDEX_64I : CUSPARSE_INDEX_32I;
  if (cusparseCreateCsr(&hd->spA, nrows, nrows, hd->csr_nnz, hd->d_rowptr, hd->d_col, hd->d_val, it, it,
                        CUSPARSE_INDEX_BASE_ZERO, CUDA_R_64F) != CUSPARSE_STATUS_SUCCESS)
    return fail(CUTFEM_ECUDA, "cusparseCreateCsr failed");
  // workspace for SpMV
  double *x = nullptr, *y = nullptr;
  CU(cudaMalloc(&x, sizeof(double) * std::max<int64_t>(nrows, 1)));
  CU(cudaMalloc(&y, sizeof(double) * std::max<int64_t>(nrows, 1)));
  cusparseDnVecDescr_t vx, vy;
  cusparseCreateDnVec(&vx, nrows, x, CUDA_R_64F);
  cusparseCreateDnVec(&vy, nrows, y, CUDA_R_64F);
  const double one = 1.0, zero = 0.0;
  size_t sz = 0;
  cusparseStatus_t s = cusparseSpMV_bufferSize(hd->sp, CUSPARSE_OPERATION_NON_TRANSPOSE, &one, hd->spA, vx,
                                               &zero, vy, CUDA_R_64F, CUSPARSE_SPMV_CSR_ALG1, &sz);
  cusparseDestroyDnVec(vx);
  cusparseDestroyDnVec(vy);
  cudaFree(x);
  cudaFree(y);
  if (s != CUSPARSE_STATUS_SUCCESS) return fail(CUTFEM_ECUDA, "cusparseSpMV_bufferSize failed");
  hd->spbuf_size = sz;
  if (sz) CU(cudaMalloc(&hd->d_spbuf, sz));
  return 0;
}

}  // namespace

extern "C" {

int cutfem_csr_setup(cutfem_handle *hd, int64_t n_rows, const int64_t *row_ptr, const int32_t *col,
                     const double *val) {
  if (!hd || !row_ptr || (n_rows > 0 && (!col || !val))) return fail(CUTFEM_EINVAL, "null");
  if (n_rows != hd->stats.n_dofs) return fail(CUTFEM_EINVAL, "n_rows != n_dofs");
  CU(cudaSetDevice(hd->device));
  csr_free(hd);
  const int64_t nnz = row_ptr[n_rows];
  hd->csr_nnz = nnz;
  hd->csr_i64 = nnz >= (int64_t)INT32_MAX;
  if (hd->csr_i64) {
    CU(cudaMalloc(&hd->d_rowptr, sizeof(int64_t) * (n_rows + 1)));
    CU(cudaMemcpy(hd->d_rowptr, row_ptr, sizeof(int64_t) * (n_rows + 1), cudaMemcpyHostToDevice));
    std::vector<int64_t> c64(col, col + nnz);
    CU(cudaMalloc(&hd->d_col, sizeof(int64_t) * std::max<int64_t>(nnz, 1)));
    CU(cudaMemcpy(hd->d_col, c64.data(), sizeof(int64_t) * nnz, cudaMemcpyHostToDevice));
  } else {
    std::vector<int32_t> r32(row_ptr, row_ptr + n_rows + 1);
    CU(cudaMalloc(&hd->d_rowptr, sizeof(int32_t) * (n_rows + 1)));
    CU(cudaMemcpy(hd->d_rowptr, r32.data(), sizeof(int32_t) * (n_rows + 1), cudaMemcpyHostToDevice));
    CU(cudaMalloc(&hd->d_col, sizeof(int32_t) * std::max<int64_t>(nnz, 1)));
    CU(cudaMemcpy(hd->d_col, col, sizeof(int32_t) * nnz, cudaMemcpyHostToDevice));
  }
  CU(cudaMalloc(&hd->d_val, sizeof(double) * std::max<int64_t>(nnz, 1)));
  CU(cudaMemcpy(hd->d_val, val, sizeof(double) * nnz, cudaMemcpyHostToDevice));
  return csr_make_descr(hd);
}

int cutfem_csr_assemble(cutfem_handle *hd, int64_t *nnz_out) {
  if (!hd) return fail(CUTFEM_EINVAL, "null handle");
  if (hd->dist || hd->n_own != hd->n_active) return fail(CUTFEM_EUNSUPPORTED, "CSR assembly needs a single-GPU handle");
  CU(cudaSetDevice(hd->device));
  csr_free(hd);
  // The handle's descriptors live on the device; rebuild the block graph from them.
  const int64_t na = hd->n_active;
  const int n = hd->n, n3 = n * n * n;
  std::vector<UDesc> ud(hd->n_uncut);
  std::vector<CDesc> cd(hd->n_cut);
  if (hd->n_uncut) CU(cudaMemcpy(ud.data(), hd->d_udesc, sizeof(UDesc) * ud.size(), cudaMemcpyDeviceToHost));
  if (hd->n_cut) CU(cudaMemcpy(cd.data(), hd->d_cdesc, sizeof(CDesc) * cd.size(), cudaMemcpyDeviceToHost));
  std::vector<int32_t> nbl((size_t)na * 7, -1), nbc(na, 0);
  std::vector<uint8_t> color(na, 0);
  auto put = [&](int32_t blk, const int32_t *nb) {
    int32_t lst[7];
    int c = 0;
    lst[c++] = blk;
    for (int f = 0; f < 6; ++f)
      if (nb[f] >= 0) lst[c++] = nb[f];
    std::sort(lst, lst + c);
    for (int k = 0; k < c; ++k) nbl[(size_t)blk * 7 + k] = lst[k];
    nbc[blk] = c;
  };
  for (auto &u : ud) put(u.blk, u.nb);
  for (auto &c : cd) put(c.blk, c.nb);
  if ((int64_t)hd->color.size() != na) return fail(CUTFEM_EINVAL, "colour table missing");
  color = hd->color;
  std::vector<int64_t> rowptr((size_t)na * n3 + 1, 0);
  for (int64_t B = 0; B < na; ++B)
    for (int i = 0; i < n3; ++i) rowptr[B * n3 + i + 1] = rowptr[B * n3 + i] + (int64_t)nbc[B] * n3;
  const int64_t nrows = na * n3, nnz = rowptr[nrows];
  hd->csr_nnz = nnz;
  hd->csr_i64 = nnz >= (int64_t)INT32_MAX;
  int32_t *d_nbl = nullptr, *d_nbc = nullptr;
  uint8_t *d_color = nullptr;
  int64_t *d_rp64 = nullptr;
  double *d_pu = nullptr, *d_pv = nullptr;
  CU(cudaMalloc(&d_nbl, sizeof(int32_t) * nbl.size()));
  CU(cudaMalloc(&d_nbc, sizeof(int32_t) * std::max<int64_t>(na, 1)));
  CU(cudaMalloc(&d_color, std::max<int64_t>(na, 1)));
  CU(cudaMalloc(&d_rp64, sizeof(int64_t) * rowptr.size()));
  CU(cudaMemcpy(d_nbl, nbl.data(), sizeof(int32_t) * nbl.size(), cudaMemcpyHostToDevice));
  CU(cudaMemcpy(d_nbc, nbc.data(), sizeof(int32_t) * na, cudaMemcpyHostToDevice));
  CU(cudaMemcpy(d_color, color.data(), na, cudaMemcpyHostToDevice));
  CU(cudaMemcpy(d_rp64, rowptr.data(), sizeof(int64_t) * rowptr.size(), cudaMemcpyHostToDevice));
  const int TB = 256;
  const unsigned gr = (unsigned)((nrows + TB - 1) / TB);
  if (hd->csr_i64) {
    CU(cudaMalloc(&hd->d_rowptr, sizeof(int64_t) * rowptr.size()));
    CU(cudaMemcpy(hd->d_rowptr, d_rp64, sizeof(int64_t) * rowptr.size(), cudaMemcpyDeviceToDevice));
    CU(cudaMalloc(&hd->d_col, sizeof(int64_t) * std::max<int64_t>(nnz, 1)));
    if (nrows) k_csr_cols64<<<gr, TB>>>(d_nbl, d_nbc, d_rp64, (int64_t *)hd->d_col, nrows, n3);
  } else {
    std::vector<int32_t> r32(rowptr.begin(), rowptr.end());
    CU(cudaMalloc(&hd->d_rowptr, sizeof(int32_t) * r32.size()));
    CU(cudaMemcpy(hd->d_rowptr, r32.data(), sizeof(int32_t) * r32.size(), cudaMemcpyHostToDevice));
    CU(cudaMalloc(&hd->d_col, sizeof(int32_t) * std::max<int64_t>(nnz, 1)));
    if (nrows) k_csr_cols32<<<gr, TB>>>(d_nbl, d_nbc, d_rp64, (int32_t *)hd->d_col, nrows, n3);
  }
  CU(cudaGetLastError());
  CU(cudaMalloc(&hd->d_val, sizeof(double) * std::max<int64_t>(nnz, 1)));
  CU(cudaMalloc(&d_pu, sizeof(double) * std::max<int64_t>(nrows, 1)));
  CU(cudaMalloc(&d_pv, sizeof(double) * std::max<int64_t>(nrows, 1)));
  for (int c = 0; c < 7 && nrows; ++c)
    for (int l = 0; l < n3; ++l) {
      k_probe_set<<<gr, TB>>>(d_pu, d_color, na, n3, c, l);
      int rc = dispatch_apply(hd, d_pu, d_pv, 0);
      if (rc) return rc;
      k_probe_scatter<<<gr, TB>>>(d_pv, d_color, d_nbl, d_nbc, d_rp64, hd->d_val, nrows, n3, c, l);
    }
  CU(cudaGetLastError());
  CU(cudaDeviceSynchronize());
  cudaFree(d_nbl);
  cudaFree(d_nbc);
  cudaFree(d_color);
  cudaFree(d_rp64);
  cudaFree(d_pu);
  cudaFree(d_pv);
  if (nnz_out) *nnz_out = nnz;
  return csr_make_descr(hd);
}

int cutfem_csr_apply(cutfem_handle *hd, const double *u_dev, double *v_dev, void *cuda_stream) {
  if (!hd || !hd->spA) return fail(CUTFEM_EINVAL, "no CSR matrix (call cutfem_csr_setup/assemble)");
  CU(cudaSetDevice(hd->device));
  const int64_t nrows = hd->stats.n_dofs;
  cusparseSetStream(hd->sp, (cudaStream_t)cuda_stream);
  cusparseDnVecDescr_t vx, vy;
  cusparseCreateDnVec(&vx, nrows, (void *)u_dev, CUDA_R_64F);
  cusparseCreateDnVec(&vy, nrows, v_dev, CUDA_R_64F);
  const double one = 1.0, zero = 0.0;
  cusparseStatus_t s = cusparseSpMV(hd->sp, CUSPARSE_OPERATION_NON_TRANSPOSE, &one, hd->spA, vx, &zero, vy,
                                    CUDA_R_64F, CUSPARSE_SPMV_CSR_ALG1, hd->d_spbuf);
  cusparseDestroyDnVec(vx);
  cusparseDestroyDnVec(vy);
  if (s != CUSPARSE_STATUS_SUCCESS) return fail(CUTFEM_ECUDA, "cusparseSpMV failed");
  return 0;
}

int64_t cutfem_csr_nnz(const cutfem_handle *hd) { return hd ? hd->csr_nnz : -1; }

int cutfem_csr_download(const cutfem_handle *hd, int64_t *row_ptr, int32_t *col, double *val) {
  if (!hd || !hd->spA) return fail(CUTFEM_EINVAL, "no CSR matrix");
  CU(cudaSetDevice(hd->device));
  const int64_t nrows = hd->stats.n_dofs, nnz = hd->csr_nnz;
  if (hd->csr_i64) {
    CU(cudaMemcpy(row_ptr, hd->d_rowptr, sizeof(int64_t) * (nrows + 1), cudaMemcpyDeviceToHost));
    std::vector<int64_t> c64(nnz);
    CU(cudaMemcpy(c64.data(), hd->d_col, sizeof(int64_t) * nnz, cudaMemcpyDeviceToHost));
    for (int64_t i = 0; i < nnz; ++i) col[i] = (int32_t)c64[i];
  } else {
    std::vector<int32_t> r32(nrows + 1);
    CU(cudaMemcpy(r32.data(), hd->d_rowptr, sizeof(int32_t) * (nrows + 1), cudaMemcpyDeviceToHost));
    for (int64_t i = 0; i <= nrows; ++i) row_ptr[i] = r32[i];
    CU(cudaMemcpy(col, hd->d_col, sizeof(int32_t) * nnz, cudaMemcpyDeviceToHost));
  }
  CU(cudaMemcpy(val, hd->d_val, sizeof(double) * nnz, cudaMemcpyDeviceToHost));
  return 0;
}

}  // extern "C"
