"""CPU ORACLE for the DG-CutFEM operator apply v = A u — TEST INFRASTRUCTURE ONLY.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s ``cpu_baseline`` /
``--impl reference`` legs may import this package.  The product path
(``paper_2404_07911_b200``) never imports it, and this package never imports the
product path; the two share only the seeded input generator ``cutgen``.

What it computes (PAPER.md eq:bilinear_dg P:83-92, eq:bilinear_cg P:68-76, the
face ghost penalty of BASELINE.json configs[0]; SURVEY.md §8(c) "Definition"):
the plain definition — every element, face and interface matrix is formed by
direct basis evaluation phi_l(x_q) = l_a(xi) l_b(eta) l_c(zeta) at every
quadrature point (naive interpolation S_ql), with no sum
factorisation, then applied blockwise (eq:matrixfreeopcompact P:209-212) or
assembled into CSR (eq:matrixbasedop P:224-227).

Pins (tests/test_oracle_pins.py, tests/test_oracle_plane.py): Q1 Kronecker
cell matrix, Q2 face closed form, Q3 GP closed form order by order, Q4 "level
set misses the mesh" = standard SIPG, Q5 axis-aligned plane = sum of Kronecker
products (every term, cut faces included), Q6 exact identities, Q7 symmetry,
Q8 SPD, Q9 quadrature moments, Q10 tensor rule as cut rule, Q11 convergence
order, Q12 CSR = blockwise, Q13 the sphere's cut-cell volume + Nitsche terms
against the Gamma-function closed form of a(q, r) for global polynomials
(DESIGN.md §4 maps every function to its pin).
Q14 the cut-face SIPG next to the sphere against 1-D polynomial integrals (broken
polynomials across a mesh plane: the faces in it tile a disk).  No function of this
package is left "parity unpinned".
"""
from .basis import Basis1D  # noqa: F401
from .operator import Oracle  # noqa: F401
