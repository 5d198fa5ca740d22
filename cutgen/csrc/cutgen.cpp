// cutgen: the shared, seeded INPUT generator for the DG-CutFEM operator.
//
// It builds the Cartesian background mesh, classifies cells and faces against a
// level set phi (Omega = {phi < 0}), and produces the unstructured cut-cell
// volume, interface (surface) and cut-face quadrature rules by dimension
// reduction (§1 P:45-48 "dimension reduction of integrals" [Saye 2015];
// refinement of cut cells raises the point count by 2^(d*n_ref)).
// BASELINE.json north_star: "The cut-cell quadrature is generated once on the
// host by the shared input generator (dimension-reduction style) and consumed
// as arrays."
//
// This module holds NONE of the operator's arithmetic (no basis functions, no
// penalties, no element matrices): it only produces geometry and quadrature
// arrays. Both the CPU oracle (oracle/) and the CUDA library consume them.
//
// Algorithm (per cut cell, reference box [0,1]^3, x = x_K + h*xi):
//   1. height direction k3 = argmax |d phi/d x_k| at the box centre; phi must be
//      monotone in k3 over the box (sampled check), else the box is split into
//      2^3 children (up to max_depth levels).
//   2. the base (the two other dims) is integrated recursively: the base
//      integrand is smooth except where phi = 0 crosses the bottom/top faces in
//      k3, so the base is partitioned at the zeros of psi_0 = phi|x_k3=lo and
//      psi_1 = phi|x_k3=hi: height k2 for the psi (monotone check as above),
//      outer direction k1 broken at the zeros of psi_i on the base's edges.
//   3. innermost: along each k3 line, the roots of phi split [lo,hi]; a q-point
//      Gauss rule is placed on every sub-interval with phi < 0 (volume points),
//      and each root is a surface point with weight w_base*|grad phi|/|d_k3 phi|
//      and unit normal grad phi/|grad phi| (outward from Omega).
// Cut faces use the 2-D instance of the same construction on the face plane.
#include <algorithm>
#include <atomic>
#include <cmath>
#include <cstdint>
#include <cstdlib>
#include <cstring>
#include <thread>
#include <vector>

namespace {

// ---------------------------------------------------------------- level sets
struct LevelSet {
  int type = 0;  // 0 sphere |x-c|-r ; 1 gyroid sum sin cos - c ; 2 plane n.x - off
  double c[3] = {0, 0, 0};
  double r = 1;
  double n[3] = {1, 0, 0};
  double off = 0;
  double gc = 0;  // gyroid offset

  double phi(const double x[3]) const {
    if (type == 0) {
      double dx = x[0] - c[0], dy = x[1] - c[1], dz = x[2] - c[2];
      return std::sqrt(dx * dx + dy * dy + dz * dz) - r;
    } else if (type == 1) {
      const double tp = 2.0 * M_PI;
      double sx = std::sin(tp * x[0]), cx = std::cos(tp * x[0]);
      double sy = std::sin(tp * x[1]), cy = std::cos(tp * x[1]);
      double sz = std::sin(tp * x[2]), cz = std::cos(tp * x[2]);
      return sx * cy + sy * cz + sz * cx - gc;
    } else {
      return n[0] * x[0] + n[1] * x[1] + n[2] * x[2] - off;
    }
  }
  void grad(const double x[3], double g[3]) const {
    if (type == 0) {
      double d[3] = {x[0] - c[0], x[1] - c[1], x[2] - c[2]};
      double nr = std::sqrt(d[0] * d[0] + d[1] * d[1] + d[2] * d[2]);
      if (nr == 0) nr = 1e-300;
      for (int i = 0; i < 3; ++i) g[i] = d[i] / nr;
    } else if (type == 1) {
      const double tp = 2.0 * M_PI;
      double sx = std::sin(tp * x[0]), cx = std::cos(tp * x[0]);
      double sy = std::sin(tp * x[1]), cy = std::cos(tp * x[1]);
      double sz = std::sin(tp * x[2]), cz = std::cos(tp * x[2]);
      g[0] = tp * (cx * cy - sz * sx);
      g[1] = tp * (-sx * sy + cy * cz);
      g[2] = tp * (-sy * sz + cz * cx);
    } else {
      for (int i = 0; i < 3; ++i) g[i] = n[i];
    }
  }
  // Conservative [min,max] of phi over the axis-aligned box [lo,hi] (physical).
  void bounds(const double lo[3], const double hi[3], double &mn, double &mx) const {
    if (type == 0) {
      double dmin2 = 0, dmax2 = 0;
      for (int i = 0; i < 3; ++i) {
        double a = lo[i] - c[i], b = hi[i] - c[i];
        double near = (a > 0) ? a : (b < 0 ? b : 0.0);
        double far = std::max(std::fabs(a), std::fabs(b));
        dmin2 += near * near;
        dmax2 += far * far;
      }
      mn = std::sqrt(dmin2) - r;
      mx = std::sqrt(dmax2) - r;
    } else if (type == 2) {
      mn = mx = -off;
      for (int i = 0; i < 3; ++i) {
        double a = n[i] * lo[i], b = n[i] * hi[i];
        mn += std::min(a, b);
        mx += std::max(a, b);
      }
    } else {
      // sampled extrema widened by a Lipschitz margin; |grad phi| <= 2*pi*sqrt(6)
      const int m = 4;
      const double L = 2.0 * M_PI * std::sqrt(6.0);
      mn = 1e300;
      mx = -1e300;
      double diag2 = 0;
      for (int i = 0; i < 3; ++i) {
        double d = (hi[i] - lo[i]) / m;
        diag2 += d * d;
      }
      for (int a = 0; a <= m; ++a)
        for (int b = 0; b <= m; ++b)
          for (int cc = 0; cc <= m; ++cc) {
            double x[3] = {lo[0] + (hi[0] - lo[0]) * a / m, lo[1] + (hi[1] - lo[1]) * b / m,
                           lo[2] + (hi[2] - lo[2]) * cc / m};
            double v = phi(x);
            mn = std::min(mn, v);
            mx = std::max(mx, v);
          }
      double margin = 0.5 * L * std::sqrt(diag2);
      mn -= margin;
      mx += margin;
    }
  }
};

// ------------------------------------------------------------- Gauss rules
struct Gauss1D {
  std::vector<double> x, w;  // on [0,1]
  explicit Gauss1D(int n) : x(n), w(n) {
    for (int i = 0; i < n; ++i) {
      long double z = std::cos(M_PI * (i + 0.75L) / (n + 0.5L));
      for (int it = 0; it < 100; ++it) {
        long double p0 = 1, p1 = 0;
        for (int j = 1; j <= n; ++j) {
          long double p2 = p1;
          p1 = p0;
          p0 = ((2 * j - 1) * z * p1 - (j - 1) * p2) / j;
        }
        long double dp = n * (z * p0 - p1) / (z * z - 1);
        long double dz = p0 / dp;
        z -= dz;
        if (std::fabs((double)dz) < 1e-19) break;
      }
      long double p0 = 1, p1 = 0;
      for (int j = 1; j <= n; ++j) {
        long double p2 = p1;
        p1 = p0;
        p0 = ((2 * j - 1) * z * p1 - (j - 1) * p2) / j;
      }
      long double dp = n * (z * p0 - p1) / (z * z - 1);
      long double ww = 2 / ((1 - z * z) * dp * dp);
      x[n - 1 - i] = (double)((z + 1) / 2);  // roots come out descending in z
      w[n - 1 - i] = (double)(ww / 2);
    }
  }
};

// ------------------------------------------------------------ root finding
// Roots of f(t) = phi(p + t*e) for t in (a,b); f(t) < 0 counts as "inside".
struct LineFn {
  const LevelSet *ls;
  double p[3];
  int dim;  // the line runs along axis `dim` (physical coordinate)
  double at(double t) const {
    double x[3] = {p[0], p[1], p[2]};
    x[dim] = t;
    return ls->phi(x);
  }
  double d(double t) const {
    double x[3] = {p[0], p[1], p[2]};
    x[dim] = t;
    double g[3];
    ls->grad(x, g);
    return g[dim];
  }
};

void line_roots(const LineFn &f, double a, double b, int nsamp, std::vector<double> &out) {
  double ta = a, fa = f.at(a);
  for (int s = 1; s <= nsamp; ++s) {
    double tb = a + (b - a) * s / nsamp;
    if (s == nsamp) tb = b;
    double fb = f.at(tb);
    bool ina = fa < 0, inb = fb < 0;
    if (ina != inb) {
      double lo = ta, hi = tb, flo = fa;
      // bisection to a small bracket, then safeguarded Newton
      for (int it = 0; it < 200 && (hi - lo) > 1e-6 * (b - a); ++it) {
        double mid = 0.5 * (lo + hi);
        double fm = f.at(mid);
        if ((fm < 0) == (flo < 0)) {
          lo = mid;
          flo = fm;
        } else {
          hi = mid;
        }
      }
      double t = 0.5 * (lo + hi);
      for (int it = 0; it < 50; ++it) {
        double ft = f.at(t), dt = f.d(t);
        if (ft == 0) break;
        if ((ft < 0) == (flo < 0)) lo = t; else hi = t;
        double tn = (dt != 0) ? t - ft / dt : 0.5 * (lo + hi);
        if (!(tn > lo && tn < hi)) tn = 0.5 * (lo + hi);
        if (std::fabs(tn - t) <= 1e-16 * std::max(1.0, std::fabs(t))) {
          t = tn;
          break;
        }
        t = tn;
        if (hi - lo < 1e-16 * std::max(1.0, std::fabs(t))) break;
      }
      if (t > a && t < b) out.push_back(t);
    }
    ta = tb;
    fa = fb;
  }
}

struct Emit {
  std::vector<double> vol;  // xi, eta, zeta, W
  std::vector<double> srf;  // xi, eta, zeta, nx, ny, nz, W
};

struct Ctx {
  const LevelSet *ls;
  const Gauss1D *g;
  double xK[3];  // physical lower corner of the cell
  double h;
  int max_depth;
  int nsamp;
  long n_subdiv = 0;
  long n_nonmono = 0;
};

inline void to_phys(const Ctx &c, const double xi[3], double x[3]) {
  for (int i = 0; i < 3; ++i) x[i] = c.xK[i] + c.h * xi[i];
}

// sampled check that d phi / d x_k keeps one strict sign on a box (reference
// coords); `fixdim`>=0 restricts to the face xi_fixdim = fixval.
bool monotone(const Ctx &c, const double lo[3], const double hi[3], int k, int fixdim, double fixval) {
  const int m = 4;
  int sgn = 0;
  for (int a = 0; a <= m; ++a)
    for (int b = 0; b <= m; ++b)
      for (int d = 0; d <= m; ++d) {
        double xi[3] = {lo[0] + (hi[0] - lo[0]) * a / m, lo[1] + (hi[1] - lo[1]) * b / m,
                        lo[2] + (hi[2] - lo[2]) * d / m};
        if (fixdim >= 0) {
          xi[fixdim] = fixval;
          int idx = fixdim == 0 ? a : (fixdim == 1 ? b : d);
          if (idx != 0) continue;
        }
        double x[3], gr[3];
        to_phys(c, xi, x);
        c.ls->grad(x, gr);
        double v = gr[k];
        int s = v > 0 ? 1 : (v < 0 ? -1 : 0);
        if (s == 0) return false;
        if (sgn == 0) sgn = s;
        else if (s != sgn) return false;
      }
  return true;
}

bool box_has_zero(const Ctx &c, const double lo[3], const double hi[3]) {
  double plo[3], phi_[3];
  to_phys(c, lo, plo);
  to_phys(c, hi, phi_);
  double mn, mx;
  c.ls->bounds(plo, phi_, mn, mx);
  return mn < 0 && mx > 0;
}

void tensor_fill(const Ctx &c, const double lo[3], const double hi[3], Emit &e) {
  const Gauss1D &g = *c.g;
  int q = (int)g.x.size();
  double vol = (hi[0] - lo[0]) * (hi[1] - lo[1]) * (hi[2] - lo[2]);
  for (int k = 0; k < q; ++k)
    for (int j = 0; j < q; ++j)
      for (int i = 0; i < q; ++i) {
        e.vol.push_back(lo[0] + (hi[0] - lo[0]) * g.x[i]);
        e.vol.push_back(lo[1] + (hi[1] - lo[1]) * g.x[j]);
        e.vol.push_back(lo[2] + (hi[2] - lo[2]) * g.x[k]);
        e.vol.push_back(c.h * c.h * c.h * vol * g.w[i] * g.w[j] * g.w[k]);
      }
}

// 3-D cut-cell rule on the reference sub-box [lo,hi]
void cell_box(Ctx &c, const double lo[3], const double hi[3], int depth, Emit &e) {
  double plo[3], phi_[3];
  to_phys(c, lo, plo);
  to_phys(c, hi, phi_);
  double mn, mx;
  c.ls->bounds(plo, phi_, mn, mx);
  if (mn >= 0) return;  // sub-box outside Omega
  if (mx < 0) {         // sub-box inside Omega
    tensor_fill(c, lo, hi, e);
    return;
  }
  double ctr[3] = {0.5 * (lo[0] + hi[0]), 0.5 * (lo[1] + hi[1]), 0.5 * (lo[2] + hi[2])};
  double pc[3], gc[3];
  to_phys(c, ctr, pc);
  c.ls->grad(pc, gc);
  int k3 = 0;
  for (int i = 1; i < 3; ++i)
    if (std::fabs(gc[i]) > std::fabs(gc[k3])) k3 = i;
  int a = (k3 == 0) ? 1 : 0, b = (k3 == 2) ? 1 : 2;
  int k2 = std::fabs(gc[a]) >= std::fabs(gc[b]) ? a : b;
  int k1 = (k2 == a) ? b : a;
  bool ok = monotone(c, lo, hi, k3, -1, 0);
  if (ok) {
    // base functions psi_0, psi_1 must be monotone in k2 where they vanish
    for (int side = 0; side < 2 && ok; ++side) {
      double flo[3] = {lo[0], lo[1], lo[2]}, fhi[3] = {hi[0], hi[1], hi[2]};
      double v = side ? hi[k3] : lo[k3];
      flo[k3] = fhi[k3] = v;
      if (box_has_zero(c, flo, fhi) && !monotone(c, lo, hi, k2, k3, v)) ok = false;
    }
  }
  if (!ok) {
    if (depth < c.max_depth) {
      ++c.n_subdiv;
      for (int ch = 0; ch < 8; ++ch) {
        double clo[3], chi[3];
        for (int i = 0; i < 3; ++i) {
          double m = 0.5 * (lo[i] + hi[i]);
          bool up = (ch >> i) & 1;
          clo[i] = up ? m : lo[i];
          chi[i] = up ? hi[i] : m;
        }
        cell_box(c, clo, chi, depth + 1, e);
      }
      return;
    }
    ++c.n_nonmono;
  }
  const Gauss1D &g = *c.g;
  const int q = (int)g.x.size();
  const double h = c.h;
  // physical coordinates of the box edges
  auto P = [&](int dim, double xi) { return c.xK[dim] + h * xi; };
  // --- outer direction k1: breakpoints at zeros of psi_i on the base edges
  std::vector<double> sb = {lo[k1], hi[k1]};
  {
    std::vector<double> rts;
    for (int s3 = 0; s3 < 2; ++s3)
      for (int s2 = 0; s2 < 2; ++s2) {
        LineFn f;
        f.ls = c.ls;
        f.dim = k1;
        f.p[k3] = P(k3, s3 ? hi[k3] : lo[k3]);
        f.p[k2] = P(k2, s2 ? hi[k2] : lo[k2]);
        f.p[k1] = 0;
        line_roots(f, P(k1, lo[k1]), P(k1, hi[k1]), c.nsamp, rts);
      }
    for (double t : rts) sb.push_back((t - c.xK[k1]) / h);
    std::sort(sb.begin(), sb.end());
  }
  std::vector<double> tb, rts2, r3;
  for (size_t is = 0; is + 1 < sb.size(); ++is) {
    double s0 = sb[is], s1 = sb[is + 1];
    if (s1 - s0 <= 1e-15) continue;
    for (int i = 0; i < q; ++i) {
      double s = s0 + (s1 - s0) * g.x[i];
      double ws = (s1 - s0) * g.w[i];
      // --- middle direction k2: breakpoints at zeros of psi_0, psi_1 along k2
      tb.assign({lo[k2], hi[k2]});
      rts2.clear();
      for (int s3 = 0; s3 < 2; ++s3) {
        LineFn f;
        f.ls = c.ls;
        f.dim = k2;
        f.p[k3] = P(k3, s3 ? hi[k3] : lo[k3]);
        f.p[k1] = P(k1, s);
        f.p[k2] = 0;
        line_roots(f, P(k2, lo[k2]), P(k2, hi[k2]), c.nsamp, rts2);
      }
      for (double t : rts2) tb.push_back((t - c.xK[k2]) / h);
      std::sort(tb.begin(), tb.end());
      for (size_t it = 0; it + 1 < tb.size(); ++it) {
        double t0 = tb[it], t1 = tb[it + 1];
        if (t1 - t0 <= 1e-15) continue;
        for (int j = 0; j < q; ++j) {
          double t = t0 + (t1 - t0) * g.x[j];
          double wt = (t1 - t0) * g.w[j];
          // --- height direction k3: roots of phi along the line
          LineFn f;
          f.ls = c.ls;
          f.dim = k3;
          f.p[k1] = P(k1, s);
          f.p[k2] = P(k2, t);
          f.p[k3] = 0;
          r3.clear();
          line_roots(f, P(k3, lo[k3]), P(k3, hi[k3]), c.nsamp, r3);
          std::vector<double> hb = {lo[k3]};
          for (double r : r3) {
            double xr = (r - c.xK[k3]) / h;
            hb.push_back(xr);
            // surface point
            double x[3];
            x[k1] = P(k1, s);
            x[k2] = P(k2, t);
            x[k3] = r;
            double gr[3];
            c.ls->grad(x, gr);
            double gn = std::sqrt(gr[0] * gr[0] + gr[1] * gr[1] + gr[2] * gr[2]);
            double xi[3];
            xi[k1] = s;
            xi[k2] = t;
            xi[k3] = xr;
            e.srf.push_back(xi[0]);
            e.srf.push_back(xi[1]);
            e.srf.push_back(xi[2]);
            e.srf.push_back(gr[0] / gn);
            e.srf.push_back(gr[1] / gn);
            e.srf.push_back(gr[2] / gn);
            e.srf.push_back(h * h * ws * wt * gn / std::fabs(gr[k3]));
          }
          hb.push_back(hi[k3]);
          for (size_t ih = 0; ih + 1 < hb.size(); ++ih) {
            double z0 = hb[ih], z1 = hb[ih + 1];
            if (z1 - z0 <= 0) continue;
            double xm[3];
            xm[k1] = P(k1, s);
            xm[k2] = P(k2, t);
            xm[k3] = P(k3, 0.5 * (z0 + z1));
            if (!(c.ls->phi(xm) < 0)) continue;
            for (int kk = 0; kk < q; ++kk) {
              double z = z0 + (z1 - z0) * g.x[kk];
              double xi[3];
              xi[k1] = s;
              xi[k2] = t;
              xi[k3] = z;
              e.vol.push_back(xi[0]);
              e.vol.push_back(xi[1]);
              e.vol.push_back(xi[2]);
              e.vol.push_back(h * h * h * ws * wt * (z1 - z0) * g.w[kk]);
            }
          }
        }
      }
    }
  }
}

// 2-D rule on the face plane x_d = xK[d] + h (the upper face of cell K),
// in-face reference coords over dims (fa, fb) ascending; box [lo,hi] in the
// two in-face coords (index 0 -> fa, 1 -> fb).
void face_box(Ctx &c, int d, const double lo2[2], const double hi2[2], int depth, std::vector<double> &out) {
  int fa = (d == 0) ? 1 : 0, fb = (d == 2) ? 1 : 2;
  int dims[2] = {fa, fb};
  const double h = c.h;
  double lo[3], hi[3];
  lo[d] = hi[d] = 1.0;
  lo[fa] = lo2[0];
  hi[fa] = hi2[0];
  lo[fb] = lo2[1];
  hi[fb] = hi2[1];
  double plo[3], phi_[3];
  to_phys(c, lo, plo);
  to_phys(c, hi, phi_);
  double mn, mx;
  c.ls->bounds(plo, phi_, mn, mx);
  const Gauss1D &g = *c.g;
  const int q = (int)g.x.size();
  if (mn >= 0) return;
  if (mx < 0) {
    double area = (hi2[0] - lo2[0]) * (hi2[1] - lo2[1]);
    for (int j = 0; j < q; ++j)
      for (int i = 0; i < q; ++i) {
        out.push_back(lo2[0] + (hi2[0] - lo2[0]) * g.x[i]);
        out.push_back(lo2[1] + (hi2[1] - lo2[1]) * g.x[j]);
        out.push_back(h * h * area * g.w[i] * g.w[j]);
      }
    return;
  }
  double ctr[3];
  for (int i = 0; i < 3; ++i) ctr[i] = 0.5 * (lo[i] + hi[i]);
  double pc[3], gc[3];
  to_phys(c, ctr, pc);
  c.ls->grad(pc, gc);
  int ih = std::fabs(gc[fa]) >= std::fabs(gc[fb]) ? 0 : 1;  // height index within dims
  int k2 = dims[ih], k1 = dims[1 - ih];
  bool ok = monotone(c, lo, hi, k2, d, 1.0);
  if (!ok) {
    if (depth < c.max_depth) {
      ++c.n_subdiv;
      for (int ch = 0; ch < 4; ++ch) {
        double clo[2], chi[2];
        for (int i = 0; i < 2; ++i) {
          double m = 0.5 * (lo2[i] + hi2[i]);
          bool up = (ch >> i) & 1;
          clo[i] = up ? m : lo2[i];
          chi[i] = up ? hi2[i] : m;
        }
        face_box(c, d, clo, chi, depth + 1, out);
      }
      return;
    }
    ++c.n_nonmono;
  }
  auto P = [&](int dim, double xi) { return c.xK[dim] + h * xi; };
  std::vector<double> sb = {lo[k1], hi[k1]}, rts, r2;
  for (int s2 = 0; s2 < 2; ++s2) {
    LineFn f;
    f.ls = c.ls;
    f.dim = k1;
    f.p[d] = P(d, 1.0);
    f.p[k2] = P(k2, s2 ? hi[k2] : lo[k2]);
    f.p[k1] = 0;
    line_roots(f, P(k1, lo[k1]), P(k1, hi[k1]), c.nsamp, rts);
  }
  for (double t : rts) sb.push_back((t - c.xK[k1]) / h);
  std::sort(sb.begin(), sb.end());
  for (size_t is = 0; is + 1 < sb.size(); ++is) {
    double s0 = sb[is], s1 = sb[is + 1];
    if (s1 - s0 <= 1e-15) continue;
    for (int i = 0; i < q; ++i) {
      double s = s0 + (s1 - s0) * g.x[i];
      double ws = (s1 - s0) * g.w[i];
      LineFn f;
      f.ls = c.ls;
      f.dim = k2;
      f.p[d] = P(d, 1.0);
      f.p[k1] = P(k1, s);
      f.p[k2] = 0;
      r2.clear();
      line_roots(f, P(k2, lo[k2]), P(k2, hi[k2]), c.nsamp, r2);
      std::vector<double> hb = {lo[k2]};
      for (double r : r2) hb.push_back((r - c.xK[k2]) / h);
      hb.push_back(hi[k2]);
      for (size_t j = 0; j + 1 < hb.size(); ++j) {
        double z0 = hb[j], z1 = hb[j + 1];
        if (z1 - z0 <= 0) continue;
        double xm[3];
        xm[d] = P(d, 1.0);
        xm[k1] = P(k1, s);
        xm[k2] = P(k2, 0.5 * (z0 + z1));
        if (!(c.ls->phi(xm) < 0)) continue;
        for (int kk = 0; kk < q; ++kk) {
          double z = z0 + (z1 - z0) * g.x[kk];
          double xi[3];
          xi[k1] = s;
          xi[k2] = z;
          out.push_back(xi[fa]);
          out.push_back(xi[fb]);
          out.push_back(h * h * ws * (z1 - z0) * g.w[kk]);
        }
      }
    }
  }
}

template <class F>
void parallel_for(int64_t n, int nthreads, F fn) {
  if (nthreads <= 1 || n < 64) {
    for (int64_t i = 0; i < n; ++i) fn(i, 0);
    return;
  }
  std::atomic<int64_t> next(0);
  std::vector<std::thread> th;
  for (int t = 0; t < nthreads; ++t)
    th.emplace_back([&, t]() {
      for (;;) {
        int64_t s = next.fetch_add(256);
        if (s >= n) break;
        int64_t e = std::min<int64_t>(n, s + 256);
        for (int64_t i = s; i < e; ++i) fn(i, t);
      }
    });
  for (auto &x : th) x.join();
}

}  // namespace

extern "C" {

typedef struct {
  int32_t ls_type;        // 0 sphere, 1 gyroid, 2 plane
  double ls_params[8];    // sphere: cx,cy,cz,r ; gyroid: c ; plane: nx,ny,nz,off
  int32_t n_cells[3];
  double lower[3];
  double h;
  int32_t q;              // Gauss points per direction per sub-interval
  int32_t max_depth;      // cut-cell subdivision levels
  int32_t force_cut_cells;  // 1: every active cell through the unstructured path (tensor rule)
  int32_t force_cut_faces;  // 1: every face between two cut cells carries explicit points
  int32_t nthreads;
} cutgen_params;

typedef struct {
  int64_t n_active;
  int32_t *active_ijk;  // [n_active][3], x slowest, z fastest
  uint8_t *is_cut;      // [n_active]
  int64_t n_cut;
  int64_t *vol_ptr;     // [n_cut+1]
  double *vol_pts;      // [n_vol][4]
  int64_t *srf_ptr;     // [n_cut+1]
  double *srf_pts;      // [n_srf][7]
  int64_t n_sfaces;
  int32_t *sf_cells;    // [n_sfaces][2]
  uint8_t *sf_axis;     // [n_sfaces]
  int64_t *sf_ptr;      // [n_sfaces+1]
  double *sf_pts;       // [n_fp][3]
  int64_t n_subdivided;
  int64_t n_nonmonotone;
} cutgen_result;

int cutgen_generate(const cutgen_params *pp, cutgen_result *res) {
  std::memset(res, 0, sizeof(*res));
  const cutgen_params &p = *pp;
  if (p.q < 1 || p.q > 32 || p.h <= 0) return -1;
  for (int i = 0; i < 3; ++i)
    if (p.n_cells[i] < 1) return -1;
  LevelSet ls;
  ls.type = p.ls_type;
  if (ls.type == 0) {
    for (int i = 0; i < 3; ++i) ls.c[i] = p.ls_params[i];
    ls.r = p.ls_params[3];
  } else if (ls.type == 1) {
    ls.gc = p.ls_params[0];
  } else if (ls.type == 2) {
    for (int i = 0; i < 3; ++i) ls.n[i] = p.ls_params[i];
    ls.off = p.ls_params[3];
  } else {
    return -1;
  }
  Gauss1D g(p.q);
  const int nx = p.n_cells[0], ny = p.n_cells[1], nz = p.n_cells[2];
  const int64_t ncell = (int64_t)nx * ny * nz;
  const double h = p.h;
  int nth = p.nthreads > 0 ? p.nthreads : (int)std::max(1u, std::thread::hardware_concurrency());
  // 1. classify: 0 outside, 1 inside, 2 candidate cut
  std::vector<uint8_t> cls(ncell);
  parallel_for(ncell, nth, [&](int64_t id, int) {
    int i = (int)(id / ((int64_t)ny * nz)), j = (int)((id / nz) % ny), k = (int)(id % nz);
    double lo[3] = {p.lower[0] + h * i, p.lower[1] + h * j, p.lower[2] + h * k};
    double hi[3] = {lo[0] + h, lo[1] + h, lo[2] + h};
    double mn, mx;
    ls.bounds(lo, hi, mn, mx);
    cls[id] = (mn >= 0) ? 0 : (mx < 0 ? 1 : 2);
  });
  // 2. cut-cell rules for candidates
  std::vector<int64_t> cand;
  for (int64_t id = 0; id < ncell; ++id)
    if (cls[id] == 2) cand.push_back(id);
  std::vector<Emit> rules(cand.size());
  std::vector<long> nsub(nth, 0), nnm(nth, 0);
  parallel_for((int64_t)cand.size(), nth, [&](int64_t ci, int t) {
    int64_t id = cand[ci];
    int i = (int)(id / ((int64_t)ny * nz)), j = (int)((id / nz) % ny), k = (int)(id % nz);
    Ctx c;
    c.ls = &ls;
    c.g = &g;
    c.xK[0] = p.lower[0] + h * i;
    c.xK[1] = p.lower[1] + h * j;
    c.xK[2] = p.lower[2] + h * k;
    c.h = h;
    c.max_depth = p.max_depth;
    c.nsamp = 16;
    double lo[3] = {0, 0, 0}, hi[3] = {1, 1, 1};
    cell_box(c, lo, hi, 0, rules[ci]);
    nsub[t] += c.n_subdiv;
    nnm[t] += c.n_nonmono;
  });
  // finalize activity: candidates with no volume points are inactive; those
  // with a full volume and no interface points are inside.
  std::vector<int64_t> cand_of(ncell, -1);
  for (size_t ci = 0; ci < cand.size(); ++ci) {
    int64_t id = cand[ci];
    Emit &e = rules[ci];
    if (e.vol.empty()) {
      cls[id] = 0;
    } else if (e.srf.empty()) {
      double vs = 0;
      for (size_t t = 3; t < e.vol.size(); t += 4) vs += e.vol[t];
      if (std::fabs(vs - h * h * h) <= 1e-12 * h * h * h) cls[id] = 1;
      else cand_of[id] = (int64_t)ci;
    } else {
      cand_of[id] = (int64_t)ci;
    }
  }
  // block ids (x slowest, z fastest)
  std::vector<int32_t> blk(ncell, -1);
  int64_t na = 0, nc = 0;
  for (int64_t id = 0; id < ncell; ++id)
    if (cls[id] != 0) blk[id] = (int32_t)na++;
  res->n_active = na;
  res->active_ijk = (int32_t *)std::malloc(sizeof(int32_t) * 3 * std::max<int64_t>(na, 1));
  res->is_cut = (uint8_t *)std::malloc(std::max<int64_t>(na, 1));
  Emit tensor_rule;
  {
    Ctx c;
    c.ls = &ls;
    c.g = &g;
    c.h = h;
    double lo[3] = {0, 0, 0}, hi[3] = {1, 1, 1};
    tensor_fill(c, lo, hi, tensor_rule);
  }
  std::vector<const Emit *> cut_rules;
  for (int64_t id = 0; id < ncell; ++id) {
    if (cls[id] == 0) continue;
    int64_t b = blk[id];
    int i = (int)(id / ((int64_t)ny * nz)), j = (int)((id / nz) % ny), k = (int)(id % nz);
    res->active_ijk[3 * b] = i;
    res->active_ijk[3 * b + 1] = j;
    res->active_ijk[3 * b + 2] = k;
    bool cut = (cls[id] == 2 && cand_of[id] >= 0) || p.force_cut_cells;
    res->is_cut[b] = cut ? 1 : 0;
    if (cut) {
      cut_rules.push_back((cls[id] == 2 && cand_of[id] >= 0) ? &rules[cand_of[id]] : &tensor_rule);
      ++nc;
    }
  }
  res->n_cut = nc;
  res->vol_ptr = (int64_t *)std::malloc(sizeof(int64_t) * (nc + 1));
  res->srf_ptr = (int64_t *)std::malloc(sizeof(int64_t) * (nc + 1));
  int64_t nv = 0, ns = 0;
  res->vol_ptr[0] = res->srf_ptr[0] = 0;
  for (int64_t ci = 0; ci < nc; ++ci) {
    nv += cut_rules[ci]->vol.size() / 4;
    ns += cut_rules[ci]->srf.size() / 7;
    res->vol_ptr[ci + 1] = nv;
    res->srf_ptr[ci + 1] = ns;
  }
  res->vol_pts = (double *)std::malloc(sizeof(double) * 4 * std::max<int64_t>(nv, 1));
  res->srf_pts = (double *)std::malloc(sizeof(double) * 7 * std::max<int64_t>(ns, 1));
  for (int64_t ci = 0; ci < nc; ++ci) {
    std::memcpy(res->vol_pts + 4 * res->vol_ptr[ci], cut_rules[ci]->vol.data(),
                sizeof(double) * cut_rules[ci]->vol.size());
    std::memcpy(res->srf_pts + 7 * res->srf_ptr[ci], cut_rules[ci]->srf.data(),
                sizeof(double) * cut_rules[ci]->srf.size());
  }
  // 3. faces between two active cells that are not fully inside Omega
  struct FaceRec {
    int32_t m, pl;
    uint8_t axis;
    std::vector<double> pts;
  };
  std::vector<std::vector<FaceRec>> per_cell(na);
  std::vector<int64_t> act_ids;
  act_ids.reserve(na);
  for (int64_t id = 0; id < ncell; ++id)
    if (cls[id] != 0) act_ids.push_back(id);
  parallel_for(na, nth, [&](int64_t b, int) {
    int64_t id = act_ids[b];
    int i = (int)(id / ((int64_t)ny * nz)), j = (int)((id / nz) % ny), k = (int)(id % nz);
    int ijk[3] = {i, j, k};
    for (int d = 0; d < 3; ++d) {
      int nijk[3] = {i, j, k};
      nijk[d] += 1;
      if (nijk[d] >= p.n_cells[d]) continue;
      int64_t nid = ((int64_t)nijk[0] * ny + nijk[1]) * nz + nijk[2];
      if (cls[nid] == 0) continue;
      bool mcut = res->is_cut[b], pcut = res->is_cut[blk[nid]];
      bool m_real = cls[id] == 2 && cand_of[id] >= 0, p_real = cls[nid] == 2 && cand_of[nid] >= 0;
      // face fully inside Omega unless both neighbours are genuinely cut
      bool maybe_cut = m_real && p_real;
      FaceRec fr;
      fr.m = (int32_t)b;
      fr.pl = blk[nid];
      fr.axis = (uint8_t)d;
      Ctx c;
      c.ls = &ls;
      c.g = &g;
      for (int t = 0; t < 3; ++t) c.xK[t] = p.lower[t] + h * ijk[t];
      c.h = h;
      c.max_depth = p.max_depth;
      c.nsamp = 16;
      double lo2[2] = {0, 0}, hi2[2] = {1, 1};
      if (maybe_cut) {
        double lo[3], hi[3];
        for (int t = 0; t < 3; ++t) {
          lo[t] = c.xK[t];
          hi[t] = c.xK[t] + h;
        }
        lo[d] = hi[d] = c.xK[d] + h;
        double mn, mx;
        ls.bounds(lo, hi, mn, mx);
        if (mx < 0) {
          maybe_cut = false;  // fully inside
        } else {
          if (mn < 0) face_box(c, d, lo2, hi2, 0, fr.pts);
          per_cell[b].push_back(std::move(fr));  // cut (possibly empty)
          continue;
        }
      }
      if (p.force_cut_faces && mcut && pcut) {
        face_box(c, d, lo2, hi2, 0, fr.pts);  // fully inside: tensor rule
        per_cell[b].push_back(std::move(fr));
      }
    }
  });
  int64_t nf = 0, nfp = 0;
  for (auto &v : per_cell)
    for (auto &f : v) {
      ++nf;
      nfp += f.pts.size() / 3;
    }
  res->n_sfaces = nf;
  res->sf_cells = (int32_t *)std::malloc(sizeof(int32_t) * 2 * std::max<int64_t>(nf, 1));
  res->sf_axis = (uint8_t *)std::malloc(std::max<int64_t>(nf, 1));
  res->sf_ptr = (int64_t *)std::malloc(sizeof(int64_t) * (nf + 1));
  res->sf_pts = (double *)std::malloc(sizeof(double) * 3 * std::max<int64_t>(nfp, 1));
  int64_t fi = 0, pi = 0;
  res->sf_ptr[0] = 0;
  for (auto &v : per_cell)
    for (auto &f : v) {
      res->sf_cells[2 * fi] = f.m;
      res->sf_cells[2 * fi + 1] = f.pl;
      res->sf_axis[fi] = f.axis;
      std::memcpy(res->sf_pts + 3 * pi, f.pts.data(), sizeof(double) * f.pts.size());
      pi += f.pts.size() / 3;
      ++fi;
      res->sf_ptr[fi] = pi;
    }
  long s1 = 0, s2 = 0;
  for (int t = 0; t < nth; ++t) {
    s1 += nsub[t];
    s2 += nnm[t];
  }
  res->n_subdivided = s1;
  res->n_nonmonotone = s2;
  return 0;
}

void cutgen_free(cutgen_result *r) {
  std::free(r->active_ijk);
  std::free(r->is_cut);
  std::free(r->vol_ptr);
  std::free(r->vol_pts);
  std::free(r->srf_ptr);
  std::free(r->srf_pts);
  std::free(r->sf_cells);
  std::free(r->sf_axis);
  std::free(r->sf_ptr);
  std::free(r->sf_pts);
  std::memset(r, 0, sizeof(*r));
}

}  // extern "C"
