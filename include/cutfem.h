/*
 * cutfem.h — C ABI of the B200-native matrix-free DG-CutFEM operator apply.
 *
 * The operator (§2.1 eq:bilinear_dg P:83-92 with the Nitsche terms of
 * eq:bilinear_cg P:68-76, plus the face ghost penalty fixed by BASELINE.json
 * configs[0]; SURVEY.md §8(c) "Definition"):
 *
 *   a(v,u) = sum_K int_{K∩Ω} ∇v·∇u
 *          + sum_{K cut} int_{Γ∩K} [ -(∂_n v) u - v ∂_n u + (τ/h) v u ]
 *          + sum_F int_{F∩Ω} [ -{∂_n v}[u] - [v]{∂_n u} + (γ/h)[v][u] ]
 *          + sum_{F touching a cut cell} sum_{j=0..p} g_j h^(2j-1) int_F [∂_n^j v][∂_n^j u]
 *
 * evaluated matrix-free as v = A·u (eq:matrixfreeopcompact P:209-212):
 * structured (tensor Gauss, sum factorisation) on uncut cells and faces,
 * unstructured per-point tensor evaluation on cut cells / interface / cut faces
 * (§3.2, Alg. 1-2).  All arithmetic is FP64.
 *
 * Conventions
 *  - Background mesh: n_cells[0..2] cubic cells of edge h, lower corner `lower`.
 *    Cell (i,j,k) has reference coords xi = (x - lower)/h - (i,j,k) in [0,1]^3.
 *  - Basis: Lagrange polynomials of degree p on the p+1 Gauss-Lobatto nodes of
 *    [0,1] per direction; local DoF l = a + n*b + n^2*c, n = p+1, x
 *    fastest.  Global DoF = block*n^3 + l, block = row of active_ijk.
 *  - Ω = {phi < 0}; [·] = (·)^- - (·)^+, {·} = mean; minus = the cell with
 *    the lower coordinate on the face axis, n = +e_d.
 *  - Faces between two active cells that are NOT listed in sf_* are full faces
 *    fully inside Ω (structured SIPG).  A listed face uses its points (s,t = the
 *    two in-face axes in ascending order, W physical); an empty point range
 *    means face∩Ω = ∅ (no SIPG).  Faces of the background box carry no term.
 *  - Ghost-penalty faces (both cells active, >= 1 is_cut) are derived here.
 *
 * Return codes: 0 OK, -1 EINVAL, -2 ENOMEM, -3 ECUDA, -4 ENCCL, -5 EUNSUPPORTED.
 * On error cutfem_last_error() returns a thread-local message.
 */
#ifndef CUTFEM_H
#define CUTFEM_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define CUTFEM_OK 0
#define CUTFEM_EINVAL (-1)
#define CUTFEM_ENOMEM (-2)
#define CUTFEM_ECUDA (-3)
#define CUTFEM_ENCCL (-4)
#define CUTFEM_EUNSUPPORTED (-5)

/* term_mask bits (per-term parity) */
#define CUTFEM_TERM_CELL 1u    /* volume ∫∇v·∇u (uncut + cut cells)            */
#define CUTFEM_TERM_SIPG 2u    /* interior-face SIPG (structured + cut faces)   */
#define CUTFEM_TERM_NITSCHE 4u /* interface Nitsche terms on Γ                  */
#define CUTFEM_TERM_GP 8u      /* face ghost penalty, orders 0..p              */
#define CUTFEM_TERM_ALL 15u

typedef struct cutfem_handle cutfem_handle; /* opaque */

/* Problem description.  All pointers are HOST pointers; cutfem_setup deep-copies
 * them, so the caller may free them as soon as it returns. */
typedef struct {
  int32_t n_cells[3];
  double lower[3];
  double h;                  /* cell edge (cubic cells)                           */
  int32_t degree;            /* p in 1..8 (BASELINE "k")                          */
  int64_t n_active;
  const int32_t *active_ijk; /* [n_active][3]: defines the u/v block order         */
  const uint8_t *is_cut;     /* [n_active]: 0 uncut (structured), 1 cut            */
  const int64_t *vol_ptr;    /* [n_cut+1], cut cells in block order               */
  const double *vol_pts;     /* [n_vol][4]: xi,eta,zeta in [0,1], W = physical JxW */
  const int64_t *srf_ptr;    /* [n_cut+1]                                          */
  const double *srf_pts;     /* [n_srf][7]: xi,eta,zeta, nx,ny,nz (unit, out of Ω), W */
  int64_t n_sfaces;          /* faces between two active cells not fully inside Ω */
  const int32_t *sf_cells;   /* [n_sfaces][2] (minus, plus) block ids              */
  const uint8_t *sf_axis;    /* [n_sfaces] 0..2                                     */
  const int64_t *sf_ptr;     /* [n_sfaces+1]                                        */
  const double *sf_pts;      /* [n_fp][3]: s,t in [0,1], W physical                 */
  double sipg_gamma;         /* sigma = sipg_gamma / h (BASELINE: 10 p^2)           */
  double nitsche_tau;        /* tau   = nitsche_tau / h (BASELINE: 10 p^2)          */
  const double *gp_gamma;    /* [degree+1]: weight gp_gamma[j] * h^(2j-1) (BASELINE 0.1) */
  uint32_t term_mask;        /* CUTFEM_TERM_* bits; 0 means ALL                      */
  int32_t gp_kind;           /* stabilisation: CUTFEM_GP_FACE (default, BASELINE configs[0])
                                or CUTFEM_GP_VOLUME (PAPER eq:volume_based_gp P:96-108)  */
  double tau_v;              /* volume GP: tau_v (P:595 uses 1); unused for face GP */
} cutfem_problem;

/* Ghost-penalty kinds.
 * CUTFEM_GP_FACE: on every face between two active cells with >= 1 cut cell,
 *   sum_{j=0..p} gp_gamma[j] h^(2j-1) int_F [d_n^j v][d_n^j u] (full-face Gauss).
 * CUTFEM_GP_VOLUME: the paper's volume-based ghost penalty with the stable-neighbour
 *   strategy: every cut cell forms ONE patch P = E1 u E2 with its most
 *   stable face neighbour -- largest volume fraction |E cap Omega| / |E| (uncut = 1,
 *   cut = sum of its volume weights / h^3), ties to the lowest face index 2d + s (s = 0
 *   lower, 1 upper) (reading A23) -- duplicates merged, and
 *   g_v = tau_v / h^2 int_P (v1 - v2)(u1 - u2) with v1, v2 the two cells' polynomials
 *   extended to the whole patch (the extrapolation operator E), by the
 *   (p+1)-point tensor Gauss rule on each cell (exact).  Not supported on distributed
 *   handles (CUTFEM_EUNSUPPORTED: a ghost cell's choice needs a second ghost plane). */
#define CUTFEM_GP_FACE 0
#define CUTFEM_GP_VOLUME 1

typedef struct {
  int64_t n_active, n_uncut, n_cut;
  int64_t n_vol_pts, n_srf_pts, n_face_pts;
  int64_t n_faces_struct;    /* interior faces with structured SIPG              */
  int64_t n_faces_cut;       /* listed faces with >= 1 point                     */
  int64_t n_faces_empty;     /* listed faces with no point                       */
  int64_t n_faces_gp;        /* ghost-penalty faces                              */
  int64_t n_dofs;
  int32_t degree;
  int32_t device;
  int64_t dev_bytes;         /* device memory held by the handle                  */
  int32_t launches_per_apply;
  int32_t reserved;
  int64_t n_ext_dofs;        /* u length incl. ghost blocks (distributed handles) */
} cutfem_stats_t;

/* Build device tables for `pb` on CUDA device `device`.  Validation failures
 * (degree outside 1..8, points outside [0,1] by > 1e-12, |n|-1 > 1e-10, W < 0,
 * inconsistent sizes, listed faces that are not between adjacent active cells
 * or that touch an uncut cell) return CUTFEM_EINVAL and leave *out NULL. */
int cutfem_setup(const cutfem_problem *pb, int device, cutfem_handle **out);

/* v = A u.  u_dev, v_dev: DEVICE pointers to n_active*(p+1)^3 doubles
 * (caller-owned, 16-byte aligned -- blocks move by bulk copies and 16-byte
 * vector accesses; a misaligned pointer returns CUTFEM_EINVAL -- and must not
 * alias).  v is fully overwritten.
 * Stream-ordered on `cuda_stream` (a cudaStream_t, NULL = legacy default);
 * no host synchronisation.  One apply in flight per handle. */
int cutfem_apply(cutfem_handle *hd, const double *u_dev, double *v_dev, void *cuda_stream);

/* Launch only one of the two kernels of cutfem_apply on `cuda_stream`:
 * which = 0 the structured kernel (uncut cells and their faces), which = 1 the
 * unstructured kernel (cut cells, interface, cut faces).  Only the v blocks
 * owned by that kernel are written.  For per-kernel timing / roofline
 * attribution; cutfem_apply = both, concurrently. */
int cutfem_apply_kernel(cutfem_handle *hd, int which, const double *u_dev, double *v_dev, void *cuda_stream);

/* Same operator with HOST buffers: copies u host->device, applies, copies
 * v device->host, synchronises the stream (the end-to-end path).  u_host: the
 * n_dofs owned values; the library's device copy of u has room for the ghost
 * blocks of a distributed handle (n_ext_dofs), which the halo exchange fills. */
int cutfem_apply_host(cutfem_handle *hd, const double *u_host, double *v_host, void *cuda_stream);

/* Batch of independent applies with HOST buffers, pipelined: v_k = A u_k for
 * k = 0..nbatch-1, u_host[k] / v_host[k] host pointers to n_dofs doubles each
 * (page-locked memory lets the copies run asynchronously; the same pointer may repeat).
 * Two device buffer pairs: the host->device copy of u_{k+1} (copy stream) and the
 * device->host copy of v_{k-1} (second copy stream) overlap the apply of u_k (cuda_stream);
 * every u_k is copied in and every v_k copied out.  Returns when all v_k are in host
 * memory.  Single-GPU handles only (CUTFEM_EUNSUPPORTED on distributed ones). */
int cutfem_apply_host_batch(cutfem_handle *hd, const double *const *u_host, double *const *v_host, int64_t nbatch,
                            void *cuda_stream);

/* Sparse-matrix comparison path (P:224-227 eq:matrixbasedop).
 * cutfem_csr_assemble builds the global CSR matrix ON THE DEVICE from the same
 * operator by probing (local matrices column by column through unit vectors,
 * P:228), using a distance-2 colouring of the face-neighbour graph.
 * cutfem_csr_setup instead uploads a host CSR (int32 columns).  Both replace
 * any previously held matrix.  cutfem_csr_apply computes v = A_csr u
 * (cuSPARSE SpMV, FP64).  *nnz_out (may be NULL) receives the nnz. */
int cutfem_csr_assemble(cutfem_handle *hd, int64_t *nnz_out);
int cutfem_csr_setup(cutfem_handle *hd, int64_t n_rows, const int64_t *row_ptr,
                     const int32_t *col, const double *val);
int cutfem_csr_apply(cutfem_handle *hd, const double *u_dev, double *v_dev, void *cuda_stream);
/* Copy the device CSR to host arrays sized by cutfem_csr_nnz (for tests). */
int64_t cutfem_csr_nnz(const cutfem_handle *hd);
int cutfem_csr_download(const cutfem_handle *hd, int64_t *row_ptr, int32_t *col, double *val);

/* ---------------------------------------------------------------- x-slabs
 * the mesh is split into contiguous x-slabs of cell planes
 * (requires x-slowest block order, as cutgen emits); each rank owns the active
 * cells of its planes [x_begin, x_end) and reads one ghost plane from each
 * neighbour.  Work balance follows PAPER §3.5 with weight 1 for uncut
 * and w_cut for cut cells. */
typedef struct {
  cutfem_problem pb;       /* local problem: owned blocks (global order), then the
                              ghost blocks of plane x_begin-1, then of plane x_end */
  int64_t n_own;           /* owned blocks = global blocks [global_begin, +n_own) */
  int64_t n_ghost_lo, n_ghost_hi;
  int64_t global_begin;
  int64_t plane_lo, plane_hi; /* owned blocks in the first / last owned plane (halo sends) */
  void *storage;           /* library-owned; release with cutfem_local_free */
} cutfem_local;

/* Host only (no GPU): split planes 0..n_cells[0] into nparts weighted slabs;
 * x_split has nparts+1 entries (x_split[0] = 0, x_split[nparts] = n_cells[0]). */
int cutfem_partition_x(const cutfem_problem *pb, int nparts, double w_cut, int32_t *x_split);
/* Host only: the local problem of slab [x_begin, x_end) (for tests / inspection). */
int cutfem_local_build(const cutfem_problem *global_pb, int32_t x_begin, int32_t x_end, cutfem_local *out);
void cutfem_local_free(cutfem_local *loc);
/* NCCL unique id (ncclUniqueId, 128 bytes) for cutfem_setup_dist; created on one
 * rank and broadcast by the caller (torch.distributed). */
int cutfem_nccl_unique_id(void *out, int64_t size);
/* Distributed handle for slab [x_begin, x_end) of the GLOBAL problem pb.  Its
 * cutfem_apply takes u_dev with room for n_own + n_ghost_lo + n_ghost_hi blocks
 * (owned values first; the ghost tail is filled by the NCCL halo exchange inside
 * the apply) and writes the n_own owned blocks of v_dev.  nranks == 1 needs no
 * id.  The exchange runs on an internal stream, overlapped with the slab-interior
 * cells; the slab-boundary cells run after it. */
int cutfem_setup_dist(const cutfem_problem *global_pb, int32_t x_begin, int32_t x_end, int rank, int nranks,
                      const void *nccl_id, int device, cutfem_handle **out);
int cutfem_dist_info(const cutfem_handle *hd, int64_t *n_own_blocks, int64_t *n_ghost_lo, int64_t *n_ghost_hi);

/* ---- Solver loop around the operator (C5: BASELINE.json configs[4]).
 *
 * cutfem_rhs_const: b_i = f * int_Ω phi_i (PAPER §2.1 P:78 right-hand side for a
 * constant source; with g = 0 on Γ the Nitsche data terms vanish): the tensor
 * (p+1)-point Gauss rule on uncut cells, the cell's volume rule on cut cells.
 * b_dev: device, n_dofs doubles (owned blocks), overwritten.  Stream ordered.
 *
 * cutfem_cg: unpreconditioned conjugate gradients on A x = b (the iterative
 * solver the operator evaluation serves), x0 = x_dev (in/out, the
 * owned blocks; a distributed handle needs room for the ghost blocks too).
 * b_dev and x_dev must be 16-byte aligned and must not alias (CUTFEM_EINVAL).
 * Runs exactly `iters` iterations, or stops early once ||r|| <= tol ||b|| when
 * tol > 0.  All vector work (dots, axpys) runs in the library's kernels with the
 * CG scalars kept on the device; dot products are reduced deterministically
 * (fixed-order two-level sum) and, on distributed handles, summed across ranks
 * by ncclAllReduce (two per iteration).  res_hist (host, may be NULL): >= iters+1
 * entries, receives ||r_k||_2, k = 0..done.  iters_done (may be NULL) receives
 * the number of iterations run.  Work vectors are owned by the handle.  The call
 * synchronises the stream once at the end. */
int cutfem_rhs_const(cutfem_handle *hd, double f, double *b_dev, void *cuda_stream);
int cutfem_cg(cutfem_handle *hd, const double *b_dev, double *x_dev, int iters, double tol, double *res_hist,
              int *iters_done, void *cuda_stream);

/* ---- Preconditioned solve (PAPER P:573-578 uses a preconditioned CG).
 * cutfem_pcg: cutfem_cg with a preconditioner M^-1: CUTFEM_PRECOND_NONE (= cutfem_cg)
 *   or CUTFEM_PRECOND_JACOBI (M = diag(A)).  res_hist receives ||r_k||_2 (the true
 *   residual, not r.z).  The diagonal is probed once per handle on first use
 *   (2 (p+1)^3 applies: unit vectors on each local index of the cells of one colour
 *   of the checkerboard (i+j+k) mod 2 -- face neighbours differ in colour, so each
 *   probe returns exact diagonal entries).
 * cutfem_diag: d_dev (n_dofs doubles, device) <- diag(A) (the same probing). */
#define CUTFEM_PRECOND_NONE 0
#define CUTFEM_PRECOND_JACOBI 1
int cutfem_pcg(cutfem_handle *hd, const double *b_dev, double *x_dev, int iters, double tol, int precond,
               double *res_hist, int *iters_done, void *cuda_stream);
int cutfem_diag(cutfem_handle *hd, double *d_dev, void *cuda_stream);

/* ---- H^1-conforming (continuous Galerkin) operator.
 * PAPER eq:bilinear_cg: a_CG(v,u) = (grad v, grad u)_Omega + Nitsche on
 * Gamma, plus the face ghost penalty of the problem (BASELINE configs[0]), on the
 * CONTINUOUS Q_p space of the active cells (GLL nodes, shared on faces, edges and
 * vertices).  v = A_CG u with A_CG = P^T A P: P gathers the global vector into the
 * cell blocks, A is the block operator of cutfem_apply without the SIPG terms (the
 * same integrals; the j = 0 ghost-penalty jump of a continuous field is zero).
 * Global numbering: lattice node (p i + a, p j + b, p k + c) of active cell (i,j,k),
 * local l = a + n b + n^2 c, nodes of active cells in lexicographic order (x slowest).
 * cutfem_h1_setup: as cutfem_setup (host arrays deep-copied; pb->term_mask's SIPG
 *   bit is ignored); *out receives an opaque handle, NULL on error.
 * cutfem_h1_ndofs: number of global nodes n_h1.
 * cutfem_h1_map: host array [n_active * n^3] <- global node of each block entry.
 * cutfem_h1_apply: u_dev, v_dev DEVICE pointers to n_h1 doubles (8-byte aligned, no
 *   alias); v is overwritten; stream ordered, no host sync; every node summed by one
 *   thread in a fixed order (deterministic, no atomics).
 * cutfem_h1_rhs_const: b_i = f int_Omega phi_i, b_dev: n_h1 doubles.
 * Errors as cutfem_setup / cutfem_apply. */
typedef struct cutfem_h1 cutfem_h1;
int cutfem_h1_setup(const cutfem_problem *pb, int device, cutfem_h1 **out);
int cutfem_h1_ndofs(const cutfem_h1 *h, int64_t *n_h1);
int cutfem_h1_map(const cutfem_h1 *h, int32_t *map_host);
int cutfem_h1_apply(cutfem_h1 *h, const double *u_dev, double *v_dev, void *cuda_stream);
int cutfem_h1_rhs_const(cutfem_h1 *h, double f, double *b_dev, void *cuda_stream);
int cutfem_h1_stats(const cutfem_h1 *h, cutfem_stats_t *out);
/* PCG / diagonal of the H1 operator (as cutfem_pcg / cutfem_diag; vectors of n_h1
 * doubles, 16-byte aligned).  The diagonal is probed with the lattice colouring
 * (I, J, K) mod (2p+1) per axis ((2p+1)^3 applies): two nodes of one colour never
 * share a cell or a ghost-penalty face pair, so each probe returns exact diagonal
 * entries. */
int cutfem_h1_pcg(cutfem_h1 *h, const double *b_dev, double *x_dev, int iters, double tol, int precond,
                  double *res_hist, int *iters_done, void *cuda_stream);
int cutfem_h1_diag(cutfem_h1 *h, double *d_dev, void *cuda_stream);
int cutfem_h1_destroy(cutfem_h1 *h);

/* ---- Chebyshev smoothing and polynomial multigrid (PAPER §3.5
 * "a preconditioned conjugate gradient iteration ... polynomial multigrid
 * (p-transfer) ... a Chebyshev smoother with an additive Schwarz inner
 * preconditioner ... inverses of the diagonal blocks").  Oracle: oracle/solver.py.
 *
 * A cutfem_mg holds n_levels DG handles of ONE mesh (same n_cells, lower, h; not
 * distributed), levels[0] the coarsest, degrees strictly increasing.  Each level
 * smooths with the Chebyshev iteration (degree smooth_degree, interval
 * [lam_max / smooth_range, lam_max] of D^-1 A) around an inner preconditioner D^-1:
 *   CUTFEM_INNER_JACOBI  D = diag(A) (probed, as cutfem_diag);
 *   CUTFEM_INNER_BLOCK   D = the (p+1)^3 x (p+1)^3 diagonal cell blocks A_KK (additive
 *     Schwarz on the cells): probed with the (i+j+k) mod 2 checkerboard (2 (p+1)^3
 *     applies), inverted on the device (in-place Gauss-Jordan sweep; the blocks are
 *     SPD); every uncut cell whose six neighbours are active and uncut has the SAME
 *     block (translation invariance), stored once; the other cells one each
 *     ((p+1)^6 doubles per cell: memory grows with the number of cut cells and their
 *     neighbours).
 * Transfers (p-transfer): prolongation interpolates a cell's degree-p_c
 * polynomial at the degree-p_f GLL nodes (cells matched by (i,j,k); a fine cell
 * without a coarse counterpart gets 0), restriction is its transpose.  The
 * coarsest level runs coarse_degree Chebyshev steps on [lam_max / coarse_range,
 * lam_max] (a fixed polynomial: the V-cycle stays linear and symmetric).
 * lam_max per level: eig_safety x the largest Ritz value of eig_iters Lanczos steps
 * (the D^-1-preconditioned CG coefficients from a fixed pseudo-random start), or set
 * by the caller (cutfem_mg_set_lambda).
 *
 * cutfem_mg_setup: probes / inverts, estimates lam_max (if eig_iters > 0); stream
 *   ordered, synchronises once.  The handles must outlive the cutfem_mg.
 * cutfem_mg_vcycle: z = B r on the finest level (device vectors, n_dofs of
 *   levels[n_levels-1], 16-byte aligned, no alias).  One level: B is the coarse
 *   Chebyshev iteration (Chebyshev-preconditioned CG).
 * cutfem_mg_pcg: CG on A x = b (finest handle) preconditioned by the V-cycle; x_dev
 *   in/out; res_hist (host, may be NULL) >= iters+1 entries: ||r_k||_2; stops once
 *   ||r|| <= tol ||b|| when tol > 0.
 * cutfem_mg_smooth: `degree` Chebyshev steps on level `level` for A x = r on
 *   [lam_min, lam_max] (x_dev in/out; x0_given = 0: the start is 0).  For tests.
 * cutfem_mg_transfer: dir 0: dst (level) = P src (level-1); dir 1: dst (level-1) =
 *   P^T src (level).  For tests.
 * Errors: CUTFEM_EINVAL (arguments, mismatched meshes / degrees, alignment),
 * CUTFEM_ENOMEM, CUTFEM_EUNSUPPORTED (distributed handles), CUTFEM_ECUDA. */
#define CUTFEM_INNER_JACOBI 0
#define CUTFEM_INNER_BLOCK 1
typedef struct {
  int32_t inner;          /* CUTFEM_INNER_JACOBI | CUTFEM_INNER_BLOCK */
  int32_t smooth_degree;  /* Chebyshev steps per pre- and post-smoothing (>= 1) */
  double smooth_range;    /* > 1 */
  int32_t coarse_degree;  /* Chebyshev steps on the coarsest level (>= 1) */
  double coarse_range;    /* > 1 */
  int32_t eig_iters;      /* Lanczos steps for lam_max (0: the caller sets them) */
  double eig_safety;      /* lam_max = eig_safety x largest Ritz value (>= 1) */
} cutfem_mg_params;
typedef struct cutfem_mg cutfem_mg;
int cutfem_mg_setup(cutfem_handle *const *levels, int32_t n_levels, const cutfem_mg_params *prm, void *cuda_stream,
                    cutfem_mg **out);
int cutfem_mg_lambda(const cutfem_mg *mg, double *lam_max);      /* host [n_levels] out */
int cutfem_mg_set_lambda(cutfem_mg *mg, const double *lam_max);  /* host [n_levels] in */
int cutfem_mg_vcycle(cutfem_mg *mg, const double *r_dev, double *z_dev, void *cuda_stream);
int cutfem_mg_pcg(cutfem_mg *mg, const double *b_dev, double *x_dev, int iters, double tol, double *res_hist,
                  int *iters_done, void *cuda_stream);
int cutfem_mg_smooth(cutfem_mg *mg, int32_t level, const double *r_dev, double *x_dev, int32_t degree,
                     double lam_max, double lam_min, int32_t x0_given, void *cuda_stream);
int cutfem_mg_transfer(cutfem_mg *mg, int32_t level, int32_t dir, const double *src_dev, double *dst_dev,
                       void *cuda_stream);
int cutfem_mg_destroy(cutfem_mg *mg);

int cutfem_stats(const cutfem_handle *hd, cutfem_stats_t *out);
const char *cutfem_last_error(void);
int cutfem_destroy(cutfem_handle *hd);

#ifdef __cplusplus
}
#endif
#endif /* CUTFEM_H */
