// dist.inl — x-slab partition, local problems with ghost planes, NCCL halo
// exchange (included by cutfem.cu).
//
// DG couples only face neighbours (SIPG, ghost penalty and the
// cut-face terms are face terms; volume and Nitsche terms are
// cell-local), so the background mesh is cut into contiguous x-slabs of cell
// planes, balanced by weighted work (PAPER §3.5: weights 1 / w_cut / 0
// for inside / intersected / outside cells).  Blocks are ordered x-slowest, so a
// slab's owned blocks, its first and last planes and each neighbour's boundary
// plane are contiguous ranges: the halo is two ncclSend/ncclRecv pairs of whole
// blocks straight from / into the vector, no packing.  The slab-interior cells
// compute while the exchange is in flight; the slab-boundary cells follow.
#include <nccl.h>

namespace {

struct LocalStore {
  std::vector<int32_t> ijk;
  std::vector<uint8_t> cut;
  std::vector<int64_t> vptr, sptr, fptr;
  std::vector<double> vpts, spts, fpts;
  std::vector<int32_t> fcells;
  std::vector<uint8_t> faxis;
  std::vector<double> gp;
};

// [start, end) block range of every x-plane; requires x-slowest block order
int plane_ranges(const cutfem_problem *pb, std::vector<int64_t> &start) {
  const int nx = pb->n_cells[0];
  start.assign(nx + 1, 0);
  int prev_i = -1;
  for (int64_t b = 0; b < pb->n_active; ++b) {
    const int i = pb->active_ijk[3 * b];
    if (i < prev_i) return fail(CUTFEM_EUNSUPPORTED, "distributed setup needs x-slowest block order");
    prev_i = i;
  }
  int64_t b = 0;
  for (int i = 0; i <= nx; ++i) {
    while (b < pb->n_active && pb->active_ijk[3 * b] < i) ++b;
    start[i] = b;
  }
  return 0;
}

int local_build(const cutfem_problem *g, int32_t x_begin, int32_t x_end, cutfem_local *out) {
  std::memset(out, 0, sizeof(*out));
  const int nx = g->n_cells[0];
  if (x_begin < 0 || x_end > nx || x_begin >= x_end) return fail(CUTFEM_EINVAL, "bad slab range");
  std::vector<int64_t> ps;
  int rc = plane_ranges(g, ps);
  if (rc) return rc;
  const int64_t o0 = ps[x_begin], o1 = ps[x_end];
  const int64_t l0 = x_begin > 0 ? ps[x_begin - 1] : o0, l1 = o0;
  const int64_t h0 = o1, h1 = x_end < nx ? ps[x_end + 1] : o1;
  const int64_t n_own = o1 - o0, n_lo = l1 - l0, n_hi = h1 - h0;
  auto local_of = [&](int64_t gb) -> int64_t {
    if (gb >= o0 && gb < o1) return gb - o0;
    if (gb >= l0 && gb < l1) return n_own + (gb - l0);
    if (gb >= h0 && gb < h1) return n_own + n_lo + (gb - h0);
    return -1;
  };
  // global cut ordinal of every block
  std::vector<int64_t> cord(g->n_active, -1);
  int64_t nc = 0;
  for (int64_t b = 0; b < g->n_active; ++b)
    if (g->is_cut[b]) cord[b] = nc++;
  LocalStore *S = new LocalStore();
  const int64_t nl = n_own + n_lo + n_hi;
  std::vector<int64_t> glob(nl);
  for (int64_t b = o0; b < o1; ++b) glob[b - o0] = b;
  for (int64_t b = l0; b < l1; ++b) glob[n_own + b - l0] = b;
  for (int64_t b = h0; b < h1; ++b) glob[n_own + n_lo + b - h0] = b;
  S->ijk.resize(3 * nl);
  S->cut.resize(nl);
  S->vptr.push_back(0);
  S->sptr.push_back(0);
  for (int64_t lb = 0; lb < nl; ++lb) {
    const int64_t b = glob[lb];
    for (int t = 0; t < 3; ++t) S->ijk[3 * lb + t] = g->active_ijk[3 * b + t];
    S->cut[lb] = g->is_cut[b];
    if (g->is_cut[b]) {
      const int64_t c = cord[b];
      S->vpts.insert(S->vpts.end(), g->vol_pts + 4 * g->vol_ptr[c], g->vol_pts + 4 * g->vol_ptr[c + 1]);
      S->spts.insert(S->spts.end(), g->srf_pts + 7 * g->srf_ptr[c], g->srf_pts + 7 * g->srf_ptr[c + 1]);
      S->vptr.push_back((int64_t)S->vpts.size() / 4);
      S->sptr.push_back((int64_t)S->spts.size() / 7);
    }
  }
  S->fptr.push_back(0);
  for (int64_t f = 0; f < g->n_sfaces; ++f) {
    const int64_t m = local_of(g->sf_cells[2 * f]), p = local_of(g->sf_cells[2 * f + 1]);
    if (m < 0 || p < 0 || (m >= n_own && p >= n_own)) continue;
    S->fcells.push_back((int32_t)m);
    S->fcells.push_back((int32_t)p);
    S->faxis.push_back(g->sf_axis[f]);
    S->fpts.insert(S->fpts.end(), g->sf_pts + 3 * g->sf_ptr[f], g->sf_pts + 3 * g->sf_ptr[f + 1]);
    S->fptr.push_back((int64_t)S->fpts.size() / 3);
  }
  S->gp.assign(g->gp_gamma, g->gp_gamma + g->degree + 1);
  cutfem_problem &pb = out->pb;
  pb = *g;
  pb.n_active = nl;
  pb.active_ijk = S->ijk.data();
  pb.is_cut = S->cut.data();
  pb.vol_ptr = S->vptr.data();
  pb.vol_pts = S->vpts.data();
  pb.srf_ptr = S->sptr.data();
  pb.srf_pts = S->spts.data();
  pb.n_sfaces = (int64_t)S->faxis.size();
  pb.sf_cells = S->fcells.data();
  pb.sf_axis = S->faxis.data();
  pb.sf_ptr = S->fptr.data();
  pb.sf_pts = S->fpts.data();
  pb.gp_gamma = S->gp.data();
  out->n_own = n_own;
  out->n_ghost_lo = n_lo;
  out->n_ghost_hi = n_hi;
  out->global_begin = o0;
  out->plane_lo = ps[x_begin + 1] - o0;
  out->plane_hi = o1 - ps[x_end - 1];
  out->storage = S;
  return 0;
}

int halo_exchange(cutfem_handle *hd, const double *u_ext, cudaStream_t st) {
  if ((hd->nranks <= 1 && !hd->loopback) || !hd->comm) return 0;
  const int64_t n3 = (int64_t)hd->n * hd->n * hd->n;
  ncclComm_t comm = (ncclComm_t)hd->comm;
  CU(cudaEventRecord(hd->ev_comm_fork, st));
  CU(cudaStreamWaitEvent(hd->comm_stream, hd->ev_comm_fork, 0));
  double *ue = const_cast<double *>(u_ext);
  ncclResult_t r = ncclGroupStart();
  if (hd->loopback) {
    // test-only: rank 0 plays both neighbours; sends and receives to the same peer
    // match in issue order (lo first, then hi)
    if (r == ncclSuccess && hd->ghost_lo)
      r = ncclSend(hd->lb_lo, (size_t)(hd->ghost_lo * n3), ncclDouble, 0, comm, hd->comm_stream);
    if (r == ncclSuccess && hd->ghost_hi)
      r = ncclSend(hd->lb_hi, (size_t)(hd->ghost_hi * n3), ncclDouble, 0, comm, hd->comm_stream);
    if (r == ncclSuccess && hd->ghost_lo)
      r = ncclRecv(ue + hd->n_own * n3, (size_t)(hd->ghost_lo * n3), ncclDouble, 0, comm, hd->comm_stream);
    if (r == ncclSuccess && hd->ghost_hi)
      r = ncclRecv(ue + (hd->n_own + hd->ghost_lo) * n3, (size_t)(hd->ghost_hi * n3), ncclDouble, 0, comm,
                   hd->comm_stream);
  } else if (hd->rank > 0) {
    if (r == ncclSuccess && hd->plane_lo)
      r = ncclSend(ue, (size_t)(hd->plane_lo * n3), ncclDouble, hd->rank - 1, comm, hd->comm_stream);
    if (r == ncclSuccess && hd->ghost_lo)
      r = ncclRecv(ue + hd->n_own * n3, (size_t)(hd->ghost_lo * n3), ncclDouble, hd->rank - 1, comm,
                   hd->comm_stream);
  }
  if (!hd->loopback && hd->rank < hd->nranks - 1) {
    if (r == ncclSuccess && hd->plane_hi)
      r = ncclSend(ue + (hd->n_own - hd->plane_hi) * n3, (size_t)(hd->plane_hi * n3), ncclDouble, hd->rank + 1,
                   comm, hd->comm_stream);
    if (r == ncclSuccess && hd->ghost_hi)
      r = ncclRecv(ue + (hd->n_own + hd->ghost_lo) * n3, (size_t)(hd->ghost_hi * n3), ncclDouble, hd->rank + 1,
                   comm, hd->comm_stream);
  }
  const ncclResult_t r2 = ncclGroupEnd();
  if (r != ncclSuccess || r2 != ncclSuccess)
    return fail(CUTFEM_ENCCL, std::string("NCCL halo exchange: ") + ncclGetErrorString(r != ncclSuccess ? r : r2));
  CU(cudaEventRecord(hd->ev_comm, hd->comm_stream));
  return 0;
}

}  // namespace

extern "C" {

int cutfem_local_build(const cutfem_problem *global_pb, int32_t x_begin, int32_t x_end, cutfem_local *out) {
  if (!global_pb || !out) return fail(CUTFEM_EINVAL, "null");
  return local_build(global_pb, x_begin, x_end, out);
}

void cutfem_local_free(cutfem_local *loc) {
  if (!loc) return;
  delete static_cast<LocalStore *>(loc->storage);
  std::memset(loc, 0, sizeof(*loc));
}

int cutfem_partition_x(const cutfem_problem *pb, int nparts, double w_cut, int32_t *x_split) {
  if (!pb || !x_split || nparts < 1) return fail(CUTFEM_EINVAL, "bad arguments");
  const int nx = pb->n_cells[0];
  if (nparts > nx) return fail(CUTFEM_EINVAL, "more slabs than x-planes");
  std::vector<double> w(nx, 0.0);
  for (int64_t b = 0; b < pb->n_active; ++b) {
    const int i = pb->active_ijk[3 * b];
    if (i < 0 || i >= nx) return fail(CUTFEM_EINVAL, "active_ijk out of range");
    w[i] += pb->is_cut[b] ? w_cut : 1.0;
  }
  double total = 0;
  for (double x : w) total += x;
  // greedy prefix split at the plane boundary nearest to each k/nparts of the weight
  x_split[0] = 0;
  double acc = 0;
  int i = 0;
  for (int k = 1; k < nparts; ++k) {
    const double target = total * k / nparts;
    while (i < nx && acc + w[i] <= target) acc += w[i++];
    if (i < nx && (target - acc) > (acc + w[i] - target)) acc += w[i++];
    const int lo = x_split[k - 1] + 1, hi = nx - (nparts - k);
    i = std::max(lo, std::min(i, hi));
    acc = 0;
    for (int t = 0; t < i; ++t) acc += w[t];
    x_split[k] = i;
  }
  x_split[nparts] = nx;
  return 0;
}

int cutfem_nccl_unique_id(void *out, int64_t size) {
  if (!out || size < (int64_t)sizeof(ncclUniqueId)) return fail(CUTFEM_EINVAL, "buffer too small");
  ncclUniqueId id;
  const ncclResult_t r = ncclGetUniqueId(&id);
  if (r != ncclSuccess) return fail(CUTFEM_ENCCL, std::string("ncclGetUniqueId: ") + ncclGetErrorString(r));
  std::memcpy(out, &id, sizeof(id));
  return 0;
}

int cutfem_setup_dist(const cutfem_problem *global_pb, int32_t x_begin, int32_t x_end, int rank, int nranks,
                      const void *nccl_id, int device, cutfem_handle **out) {
  if (!out) return fail(CUTFEM_EINVAL, "out is NULL");
  *out = nullptr;
  if (nranks < 1 || rank < 0 || rank >= nranks) return fail(CUTFEM_EINVAL, "bad rank / nranks");
  if (nranks > 1 && !nccl_id) return fail(CUTFEM_EINVAL, "nccl_id is NULL");
  cutfem_local loc;
  int rc = local_build(global_pb, x_begin, x_end, &loc);
  if (rc) return rc;
  cutfem_handle *hd = new (std::nothrow) cutfem_handle();
  if (!hd) {
    cutfem_local_free(&loc);
    return fail(CUTFEM_ENOMEM, "host allocation");
  }
  rc = setup_impl(&loc.pb, device, hd, loc.n_own);
  if (!rc) {
    hd->dist = true;
    hd->rank = rank;
    hd->nranks = nranks;
    hd->ghost_lo = loc.n_ghost_lo;
    hd->ghost_hi = loc.n_ghost_hi;
    hd->plane_lo = loc.plane_lo;
    hd->plane_hi = loc.plane_hi;
    hd->stats.dev_bytes = hd->dev_bytes;
    if (nranks > 1) {
      ncclUniqueId id;
      std::memcpy(&id, nccl_id, sizeof(id));
      ncclComm_t comm;
      const ncclResult_t r = ncclCommInitRank(&comm, nranks, id, rank);
      if (r != ncclSuccess) rc = fail(CUTFEM_ENCCL, std::string("ncclCommInitRank: ") + ncclGetErrorString(r));
      else hd->comm = comm;
      if (!rc && cudaStreamCreateWithFlags(&hd->comm_stream, cudaStreamNonBlocking) != cudaSuccess)
        rc = fail(CUTFEM_ECUDA, "comm stream");
      if (!rc && (cudaEventCreateWithFlags(&hd->ev_comm, cudaEventDisableTiming) != cudaSuccess ||
                  cudaEventCreateWithFlags(&hd->ev_comm_fork, cudaEventDisableTiming) != cudaSuccess))
        rc = fail(CUTFEM_ECUDA, "comm events");
    }
  }
  cutfem_local_free(&loc);
  if (rc) {
    free_handle(hd);
    return rc;
  }
  *out = hd;
  return 0;
}

// Test-only (not in the public header): turn a 1-rank distributed handle into an
// NCCL loopback -- a real 1-rank communicator, the halo exchange sending src_lo /
// src_hi (device, ghost_lo / ghost_hi blocks: what the neighbours would send) to
// itself into the ghost slots, and cutfem_cg's dots going through ncclAllReduce --
// so the NCCL data plane, the comm stream and its events run on one GPU.
int cutfem_debug_loopback(cutfem_handle *hd, const double *src_lo, const double *src_hi) {
  if (!hd || !hd->dist || hd->nranks != 1) return fail(CUTFEM_EINVAL, "loopback needs a 1-rank distributed handle");
  if ((hd->ghost_lo && !src_lo) || (hd->ghost_hi && !src_hi)) return fail(CUTFEM_EINVAL, "null source");
  CU(cudaSetDevice(hd->device));
  if (!hd->comm) {
    ncclUniqueId id;
    ncclResult_t r = ncclGetUniqueId(&id);
    ncclComm_t comm;
    if (r == ncclSuccess) r = ncclCommInitRank(&comm, 1, id, 0);
    if (r != ncclSuccess) return fail(CUTFEM_ENCCL, std::string("loopback comm: ") + ncclGetErrorString(r));
    hd->comm = comm;
    if (cudaStreamCreateWithFlags(&hd->comm_stream, cudaStreamNonBlocking) != cudaSuccess ||
        cudaEventCreateWithFlags(&hd->ev_comm, cudaEventDisableTiming) != cudaSuccess ||
        cudaEventCreateWithFlags(&hd->ev_comm_fork, cudaEventDisableTiming) != cudaSuccess)
      return fail(CUTFEM_ECUDA, "comm stream / events");
  }
  hd->loopback = true;
  hd->lb_lo = src_lo;
  hd->lb_hi = src_hi;
  return 0;
}

int cutfem_dist_info(const cutfem_handle *hd, int64_t *n_own_blocks, int64_t *n_ghost_lo, int64_t *n_ghost_hi) {
  if (!hd) return fail(CUTFEM_EINVAL, "null handle");
  if (n_own_blocks) *n_own_blocks = hd->n_own;
  if (n_ghost_lo) *n_ghost_lo = hd->ghost_lo;
  if (n_ghost_hi) *n_ghost_hi = hd->ghost_hi;
  return 0;
}

}  // extern "C"
