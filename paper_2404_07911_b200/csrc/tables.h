// Reference 1-D tables of the CUDA path (host side, long double), built in
// cutfem_setup.  Independent of oracle/ (which uses mpmath).
//
//   x[a]     GLL nodes on [0,1] (P:391 nodal Lagrange basis on Gauss-Lobatto points)
//   g[q],w   (p+1)-point Gauss-Legendre rule on [0,1]
//   S[q][a]  = l_a(g_q): GLL values -> Gauss-point values (P:291-295 S_{x,ri})
//   Kc       = D_g^T diag(w) D_g, D_g the collocation derivative on the Gauss
//              points ("collocation derivative"); folds E-B-I of the
//              Cartesian Laplacian along one direction
//   M        = S^T diag(w) S, the GLL mass matrix (in-face mass on full faces)
//   dj[j][s][a] = l_a^(j)(s), s in {0,1}: face traces and the ghost
//              penalty's normal-derivative traces (BASELINE configs[0])
#pragma once
#include <cmath>
#include <vector>

namespace cutfem_tables {

typedef long double ld;

inline void legendre(int n, ld z, ld &pn, ld &dpn) {
  ld p0 = 1, p1 = 0;
  for (int j = 1; j <= n; ++j) {
    ld p2 = p1;
    p1 = p0;
    p0 = ((2 * j - 1) * z * p1 - (j - 1) * p2) / j;
  }
  pn = p0;
  dpn = n * (z * p0 - p1) / (z * z - 1);
}

inline void gauss(int n, std::vector<ld> &x, std::vector<ld> &w) {
  x.assign(n, 0);
  w.assign(n, 0);
  const ld pi = 3.141592653589793238462643383279502884L;
  for (int i = 0; i < n; ++i) {
    ld z = std::cos(pi * (i + 0.75L) / (n + 0.5L));
    for (int it = 0; it < 100; ++it) {
      ld pn, dp;
      legendre(n, z, pn, dp);
      ld dz = pn / dp;
      z -= dz;
      if (std::fabs(dz) < 1e-21L) break;
    }
    ld pn, dp;
    legendre(n, z, pn, dp);
    x[n - 1 - i] = (z + 1) / 2;
    w[n - 1 - i] = 1 / ((1 - z * z) * dp * dp);
  }
}

inline void gll(int p, std::vector<ld> &x) {
  x.assign(p + 1, 0);
  x[0] = 0;
  x[p] = 1;
  const ld pi = 3.141592653589793238462643383279502884L;
  for (int i = 1; i < p; ++i) {
    ld z = -std::cos(pi * i / p);
    for (int it = 0; it < 100; ++it) {
      ld pn, dp;
      legendre(p, z, pn, dp);
      ld d2p = (2 * z * dp - p * (p + 1) * pn) / (1 - z * z);
      ld dz = dp / d2p;
      z -= dz;
      if (std::fabs(dz) < 1e-21L) break;
    }
    x[i] = (z + 1) / 2;
  }
}

// Lagrange basis on nodes xn: value and first derivative of l_a at t.
inline ld lag(const std::vector<ld> &xn, int a, ld t) {
  ld v = 1;
  for (size_t m = 0; m < xn.size(); ++m)
    if ((int)m != a) v *= (t - xn[m]) / (xn[a] - xn[m]);
  return v;
}
inline ld dlag(const std::vector<ld> &xn, int a, ld t) {
  ld s = 0;
  for (size_t k = 0; k < xn.size(); ++k) {
    if ((int)k == a) continue;
    ld term = 1 / (xn[a] - xn[k]);
    for (size_t m = 0; m < xn.size(); ++m)
      if ((int)m != a && m != k) term *= (t - xn[m]) / (xn[a] - xn[m]);
    s += term;
  }
  return s;
}

struct Ref {
  int n;
  std::vector<ld> x, g, w, cinv;
  std::vector<ld> S, Kc, M;           // n*n row-major
  std::vector<ld> tr;                 // [(j*2 + s)*n + a] = l_a^(j)(s)
};

inline Ref build(int p) {
  Ref r;
  int n = p + 1;
  r.n = n;
  gll(p, r.x);
  gauss(n, r.g, r.w);
  r.cinv.assign(n, 0);
  for (int a = 0; a < n; ++a) {
    ld d = 1;
    for (int m = 0; m < n; ++m)
      if (m != a) d *= r.x[a] - r.x[m];
    r.cinv[a] = 1 / d;
  }
  r.S.assign(n * n, 0);
  for (int q = 0; q < n; ++q)
    for (int a = 0; a < n; ++a) r.S[q * n + a] = lag(r.x, a, r.g[q]);
  std::vector<ld> Dg(n * n);
  for (int q = 0; q < n; ++q)
    for (int s = 0; s < n; ++s) Dg[q * n + s] = dlag(r.g, s, r.g[q]);
  r.Kc.assign(n * n, 0);
  r.M.assign(n * n, 0);
  for (int a = 0; a < n; ++a)
    for (int b = 0; b < n; ++b) {
      ld k = 0, m = 0;
      for (int q = 0; q < n; ++q) {
        k += r.w[q] * Dg[q * n + a] * Dg[q * n + b];
        m += r.w[q] * r.S[q * n + a] * r.S[q * n + b];
      }
      r.Kc[a * n + b] = k;
      r.M[a * n + b] = m;
    }
  // derivative traces via powers of the nodal differentiation matrix (endpoints
  // are GLL nodes, so rows 0 and p of D^j are exact traces of l^(j))
  std::vector<ld> D(n * n), Dj(n * n), tmp(n * n);
  for (int i = 0; i < n; ++i)
    for (int a = 0; a < n; ++a) D[i * n + a] = dlag(r.x, a, r.x[i]);
  for (int i = 0; i < n * n; ++i) Dj[i] = (i / n == i % n) ? 1 : 0;
  r.tr.assign((p + 1) * 2 * n, 0);
  for (int j = 0; j <= p; ++j) {
    for (int a = 0; a < n; ++a) {
      r.tr[(j * 2 + 0) * n + a] = Dj[0 * n + a];
      r.tr[(j * 2 + 1) * n + a] = Dj[p * n + a];
    }
    for (int i = 0; i < n; ++i)
      for (int a = 0; a < n; ++a) {
        ld s = 0;
        for (int k = 0; k < n; ++k) s += D[i * n + k] * Dj[k * n + a];
        tmp[i * n + a] = s;
      }
    Dj = tmp;
  }
  return r;
}

}  // namespace cutfem_tables
