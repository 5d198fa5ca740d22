"""Oracle operator: element / face / interface matrices by direct basis evaluation.

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).  Follows SURVEY.md §8(c)
"Algorithm, step by step", which restates PAPER.md:

  a(v,u) = sum_K int_{K∩Ω} ∇v·∇u                         (Poisson, eq:bilinear_cg P:71)
         + sum_K int_{Γ∩K} [-(∂_n v) u - v ∂_n u + τ_D/h v u]  (Nitsche)
         + sum_F int_{F∩Ω} [-{∂_n v}[u] - [v]{∂_n u} + γ/h [v][u]]  (SIPG, eq:bilinear_dg P:85-90)
         + sum_{F touching a cut cell} sum_{j=0..p} g_j h^(2j-1) int_F [∂_n^j v][∂_n^j u]
                                                         (face ghost penalty, BASELINE configs[0])
     or  + sum_{P} tau_v/h^2 int_P [v]_P [u]_P          (volume ghost penalty, eq:volume_based_gp
                                                         P:96-108, stable-neighbour patches, prob.gp_kind = 1)

with [·] = (·)^- - (·)^+, {·} = ((·)^- + (·)^+)/2, minus = lower cell,
n = +e_d.  Uncut cells/faces and all GP faces use the tensor
Gauss rule with p+1 points per direction; cut cells/faces use
the generator's arrays.  Each local matrix is A = B^T diag(W) B with B the
directly evaluated basis values/derivatives at the points (K1).
The operator apply is v = sum_K A_K u_K + sum_F A_F [u^-; u^+]
(eq:matrixfreeopcompact); the CSR assembly scatters the same blocks
(eq:matrixbasedop).

Term mask bits: 1 volume, 2 SIPG, 4 Nitsche, 8 ghost penalty (include/cutfem.h).
"""
from __future__ import annotations

import numpy as np
import scipy.sparse as sp

from .basis import Basis1D

TERM_CELL, TERM_SIPG, TERM_NITSCHE, TERM_GP = 1, 2, 4, 8
TERM_ALL = 15


class Oracle:
    def __init__(self, prob, term_mask: int = TERM_ALL):
        self.P = prob
        self.mask = term_mask
        self.p = prob.degree
        self.n = prob.degree + 1
        self.nd = self.n ** 3
        self.h = float(prob.h)
        self.b = Basis1D(self.p)
        ijk = np.asarray(prob.active_ijk, dtype=np.int64)
        self.ijk = ijk
        self.lookup = {tuple(int(v) for v in r): k for k, r in enumerate(ijk)}
        self.is_cut = np.asarray(prob.is_cut, dtype=bool)
        self.cut_index = np.full(len(ijk), -1, dtype=np.int64)
        self.cut_index[self.is_cut] = np.arange(int(self.is_cut.sum()))
        self.sface = {}
        for f in range(prob.sf_cells.shape[0]):
            m, pl = (int(v) for v in prob.sf_cells[f])
            self.sface[(m, int(prob.sf_axis[f]))] = f
        # tensor Gauss rules (reference) for uncut cells and full faces
        gx, gw = self.b.gauss_x, self.b.gauss_w
        Z, Y, X = np.meshgrid(gx, gx, gx, indexing="ij")
        WZ, WY, WX = np.meshgrid(gw, gw, gw, indexing="ij")
        self.cell_rule = np.stack([X.ravel(), Y.ravel(), Z.ravel(), (WX * WY * WZ).ravel()], 1)
        T, S = np.meshgrid(gx, gx, indexing="ij")
        WT, WS = np.meshgrid(gw, gw, indexing="ij")
        self.face_rule = np.stack([S.ravel(), T.ravel(), (WS * WT).ravel()], 1)
        self.faces = self._enumerate_faces()
        self.gp_kind = int(getattr(prob, "gp_kind", 0))
        self.tau_v = float(getattr(prob, "tau_v", 1.0))
        self.patches = self._stable_neighbour_patches() if self.gp_kind == 1 else set()

    # ------------------------------------------------------------ basis
    def _phi(self, xi):
        """Direct evaluation: Phi[q, l] = l_a(xi_q) l_b(eta_q) l_c(zeta_q), l = a + n b + n^2 c."""
        b = self.b
        va = [b.values(xi[:, d]) for d in range(3)]
        return np.einsum("qc,qb,qa->qcba", va[2], va[1], va[0]).reshape(len(xi), -1)

    def _grad(self, xi):
        """Reference gradient [d/dxi, d/deta, d/dzeta] of every basis function: (3, q, n^3)."""
        b = self.b
        va = [b.values(xi[:, d]) for d in range(3)]
        da = [b.derivs(xi[:, d]) for d in range(3)]
        gx = np.einsum("qc,qb,qa->qcba", va[2], va[1], da[0]).reshape(len(xi), -1)
        gy = np.einsum("qc,qb,qa->qcba", va[2], da[1], va[0]).reshape(len(xi), -1)
        gz = np.einsum("qc,qb,qa->qcba", da[2], va[1], va[0]).reshape(len(xi), -1)
        return np.stack([gx, gy, gz])

    def _normal_deriv_on_face(self, j, side, d, st):
        """∂^j/∂xi_d^j phi_l at the points of face xi_d = side, in-face coords st (q,2)."""
        b = self.b
        other = [a for a in range(3) if a != d]
        tr = b.trace(j, side)  # l_a^(j)(side)
        v = [None, None, None]
        v[d] = np.broadcast_to(tr, (st.shape[0], self.n))
        v[other[0]] = b.values(st[:, 0])
        v[other[1]] = b.values(st[:, 1])
        return np.einsum("qc,qb,qa->qcba", v[2], v[1], v[0]).reshape(st.shape[0], -1)

    def _face_points_3d(self, d, side, st):
        xi = np.zeros((st.shape[0], 3))
        other = [a for a in range(3) if a != d]
        xi[:, d] = side
        xi[:, other[0]] = st[:, 0]
        xi[:, other[1]] = st[:, 1]
        return xi

    # -------------------------------------------------------- local matrices
    def cell_matrix(self, K: int, mask: int | None = None):
        """A_K (n^3 x n^3): volume (+ Nitsche if cut), SURVEY §8(c) step 2."""
        mask = self.mask if mask is None else mask
        P, h = self.P, self.h
        A = np.zeros((self.nd, self.nd))
        if self.is_cut[K]:
            c = self.cut_index[K]
            vol = P.vol_pts[P.vol_ptr[c]:P.vol_ptr[c + 1]]
            srf = P.srf_pts[P.srf_ptr[c]:P.srf_ptr[c + 1]]
        else:
            vol = self.cell_rule.copy()
            vol[:, 3] *= h ** 3
            srf = np.zeros((0, 7))
        if mask & TERM_CELL and len(vol):
            G = self._grad(vol[:, :3]) / h  # physical gradients
            W = vol[:, 3]
            for d in range(3):
                A += G[d].T @ (W[:, None] * G[d])
        if mask & TERM_NITSCHE and len(srf):
            Phi = self._phi(srf[:, :3])
            G = self._grad(srf[:, :3]) / h
            nrm = srf[:, 3:6]
            N = G[0] * nrm[:, 0:1] + G[1] * nrm[:, 1:2] + G[2] * nrm[:, 2:3]
            W = srf[:, 6]
            tau = P.nitsche_tau / h
            A += tau * Phi.T @ (W[:, None] * Phi) - Phi.T @ (W[:, None] * N) - N.T @ (W[:, None] * Phi)
        return A

    def _enumerate_faces(self):
        """Faces between two active cells: (minus, plus, axis, sf index or -1)."""
        out = []
        for K, (i, j, k) in enumerate(self.ijk):
            for d in range(3):
                nb = [int(i), int(j), int(k)]
                nb[d] += 1
                L = self.lookup.get(tuple(nb))
                if L is None:
                    continue
                out.append((K, L, d, self.sface.get((K, d), -1)))
        return out

    def _stable_neighbour_patches(self):
        """P:108 stable-neighbour strategy: every cut cell forms one patch with the face
        neighbour of largest volume fraction |E cap Omega| / |E| (uncut cells: 1; cut cells:
        sum of the volume weights / h^3), ties to the lowest face index 2d + s (s = 0 the
        lower neighbour) -- DESIGN reading A23.  Returns {(minus, plus, d)}."""
        P, h = self.P, self.h
        frac = np.ones(len(self.ijk))
        for K in np.where(self.is_cut)[0]:
            c = self.cut_index[K]
            acc = 0.0  # sequential fp64 sum in point order: the argmax below is a floating-point
            for w in P.vol_pts[P.vol_ptr[c]:P.vol_ptr[c + 1], 3].tolist():  # decision, taken in
                acc += w  # the same arithmetic as the library's setup (DESIGN reading A23)
            frac[K] = acc / (h * h * h)
        out = set()
        for K in np.where(self.is_cut)[0]:
            best = None
            for f in range(6):
                d, s = f // 2, f % 2
                nb = [int(v) for v in self.ijk[K]]
                nb[d] += 1 if s else -1
                L = self.lookup.get(tuple(nb))
                if L is not None and (best is None or frac[L] > frac[best[0]]):
                    best = (L, d, s)
            if best is not None:
                L, d, s = best
                out.add((int(K), L, d) if s else (L, int(K), d))
        return out

    def face_matrix(self, minus: int, plus: int, d: int, sf: int, mask: int | None = None):
        """A_F (2n^3 x 2n^3) on [u^-; u^+]: SIPG + ghost penalty."""
        mask = self.mask if mask is None else mask
        P, h = self.P, self.h
        A = np.zeros((2 * self.nd, 2 * self.nd))
        full = self.face_rule.copy()
        full[:, 2] *= h * h
        if mask & TERM_SIPG:
            pts = full if sf < 0 else P.sf_pts[P.sf_ptr[sf]:P.sf_ptr[sf + 1]]
            if len(pts):
                st, W = pts[:, :2], pts[:, 2]
                Pm = self._phi(self._face_points_3d(d, 1.0, st))
                Pp = self._phi(self._face_points_3d(d, 0.0, st))
                Dm = self._grad(self._face_points_3d(d, 1.0, st))[d] / h
                Dp = self._grad(self._face_points_3d(d, 0.0, st))[d] / h
                J = np.hstack([Pm, -Pp])           # [v] rows
                Av = 0.5 * np.hstack([Dm, Dp])     # {∂_n v} rows
                sigma = P.sipg_gamma / h
                A += sigma * J.T @ (W[:, None] * J) - Av.T @ (W[:, None] * J) - J.T @ (W[:, None] * Av)
        if mask & TERM_GP and self.gp_kind == 1 and (minus, plus, d) in self.patches:
            # volume GP on the patch E1 (minus) u E2 (plus): tau_v / h^2 int_P [v]_P [u]_P with
            # [u]_E1 = u1 - E u2, [u]_E2 = E u1 - u2, E the polynomial extension into the
            # neighbour; tensor Gauss with p+1 points per direction on each cell
            cell = self.cell_rule.copy()
            shift = np.zeros(3)
            shift[d] = 1.0
            for pts, off1, off2 in ((cell[:, :3], 0.0, -1.0), (cell[:, :3], 1.0, 0.0)):
                Jm = self._phi(pts + off1 * shift)   # minus-cell basis at the points (its coordinates)
                Jp = self._phi(pts + off2 * shift)   # plus-cell basis at the same points
                J = np.hstack([Jm, -Jp])
                W = cell[:, 3] * h ** 3
                A += self.tau_v / h ** 2 * J.T @ (W[:, None] * J)
        if mask & TERM_GP and self.gp_kind == 0 and (self.is_cut[minus] or self.is_cut[plus]):
            st, W = full[:, :2], full[:, 2]
            for j in range(self.p + 1):
                Dm = self._normal_deriv_on_face(j, 1, d, st) * h ** (-j)
                Dp = self._normal_deriv_on_face(j, 0, d, st) * h ** (-j)
                D = np.hstack([Dm, -Dp])
                A += P.gp_gamma[j] * h ** (2 * j - 1) * D.T @ (W[:, None] * D)
        return A

    # --------------------------------------------------------------- apply
    def apply(self, u, blocks=None, absolute: bool = False):
        """v = A u (blockwise).  ``blocks``: optional iterable of block ids; then only
        those output blocks are formed (returned as dict block -> v_K).  With
        ``absolute`` the result is |A| |u| (the per-block tolerance scale)."""
        nd = self.nd
        u = np.asarray(u, dtype=np.float64).reshape(-1, nd)
        if absolute:
            u = np.abs(u)
        want = None if blocks is None else set(int(b) for b in blocks)
        v = np.zeros_like(u) if want is None else {b: np.zeros(nd) for b in want}
        f = np.abs if absolute else (lambda x: x)
        cells = range(u.shape[0]) if want is None else sorted(want)
        for K in cells:
            v[K] += f(self.cell_matrix(K)) @ u[K]
        for (m, pl, d, sf) in self.faces:
            if want is not None and m not in want and pl not in want:
                continue
            A = f(self.face_matrix(m, pl, d, sf))
            r = A @ np.concatenate([u[m], u[pl]])
            if want is None or m in want:
                v[m] += r[:nd]
            if want is None or pl in want:
                v[pl] += r[nd:]
        return v.reshape(-1) if want is None else v

    def assemble_csr(self):
        """Global CSR (int32 columns when nnz < 2^31) from the same local blocks."""
        nd = self.nd
        rows, cols, vals = [], [], []
        loc = np.arange(nd)
        RR, CC = np.meshgrid(loc, loc, indexing="ij")

        def put(bi, bj, blk):
            rows.append((bi * nd + RR).ravel())
            cols.append((bj * nd + CC).ravel())
            vals.append(blk.ravel())

        for K in range(self.ijk.shape[0]):
            put(K, K, self.cell_matrix(K))
        for (m, pl, d, sf) in self.faces:
            A = self.face_matrix(m, pl, d, sf)
            put(m, m, A[:nd, :nd])
            put(m, pl, A[:nd, nd:])
            put(pl, m, A[nd:, :nd])
            put(pl, pl, A[nd:, nd:])
        N = self.ijk.shape[0] * nd
        M = sp.coo_matrix((np.concatenate(vals), (np.concatenate(rows), np.concatenate(cols))),
                          shape=(N, N)).tocsr()
        M.sum_duplicates()
        M.sort_indices()
        return M

    # ------------------------------------------------------- solve helpers
    def rhs(self, f):
        """b_i = int_Ω f φ_i (Nitsche data terms vanish for g = 0)."""
        P, h = self.P, self.h
        b = np.zeros((self.ijk.shape[0], self.nd))
        lower = np.asarray(P.lower)
        for K in range(self.ijk.shape[0]):
            if self.is_cut[K]:
                c = self.cut_index[K]
                vol = P.vol_pts[P.vol_ptr[c]:P.vol_ptr[c + 1]]
            else:
                vol = self.cell_rule.copy()
                vol[:, 3] *= h ** 3
            if not len(vol):
                continue
            x = lower + h * (self.ijk[K] + vol[:, :3])
            b[K] = self._phi(vol[:, :3]).T @ (vol[:, 3] * f(x))
        return b.reshape(-1)

    def l2_error(self, uh, uex, extra: int = 2):
        """||u_h - u||_{L2(Ω)} / ||u||_{L2(Ω)} using the vol rules (cut cells) and a
        (p+1+extra)-point tensor rule on uncut cells."""
        P, h = self.P, self.h
        from .basis import gauss_mp
        gx, gw = (np.array([float(v) for v in a]) for a in gauss_mp(self.n + extra))
        Z, Y, X = np.meshgrid(gx, gx, gx, indexing="ij")
        WZ, WY, WX = np.meshgrid(gw, gw, gw, indexing="ij")
        rule = np.stack([X.ravel(), Y.ravel(), Z.ravel(), (WX * WY * WZ).ravel() * h ** 3], 1)
        uh = uh.reshape(-1, self.nd)
        lower = np.asarray(P.lower)
        e2 = n2 = 0.0
        for K in range(self.ijk.shape[0]):
            if self.is_cut[K]:
                c = self.cut_index[K]
                vol = P.vol_pts[P.vol_ptr[c]:P.vol_ptr[c + 1]]
            else:
                vol = rule
            x = lower + h * (self.ijk[K] + vol[:, :3])
            val = self._phi(vol[:, :3]) @ uh[K]
            ex = uex(x)
            e2 += np.sum(vol[:, 3] * (val - ex) ** 2)
            n2 += np.sum(vol[:, 3] * ex ** 2)
        return float(np.sqrt(e2 / n2))


def cg(apply, b, x0=None, tol=1e-12, maxiter=10000, M=None):
    """Plain (optionally Jacobi-preconditioned) conjugate gradients."""
    x = np.zeros_like(b) if x0 is None else x0.copy()
    r = b - apply(x)
    z = r if M is None else M * r
    pvec = z.copy()
    rz = r @ z
    nb = np.linalg.norm(b)
    for it in range(maxiter):
        Ap = apply(pvec)
        alpha = rz / (pvec @ Ap)
        x += alpha * pvec
        r -= alpha * Ap
        if np.linalg.norm(r) <= tol * nb:
            return x, it + 1
        z = r if M is None else M * r
        rz_new = r @ z
        pvec = z + (rz_new / rz) * pvec
        rz = rz_new
    return x, maxiter
