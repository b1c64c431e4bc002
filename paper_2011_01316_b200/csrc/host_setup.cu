// Host-side setup of the B200 library: LGL basis (device constants) and the
// seeded synthetic inputs of BASELINE.json's configs C1-C5.
// Setup only — never on the timed path.  Same arithmetic as the reference's
// proj/src/basis.cpp:11-85 and proj/src/mesh.cpp:315-386 so that the device
// constants and initial states match the oracle's bit for bit.
#include <algorithm>
#include <cmath>
#include <cstdint>
#include <cstring>
#include <stdexcept>
#include <vector>

#include "krylov.cuh"

namespace expdg {

namespace {

std::pair<double, double> legendre(int k, double x) {
  double p0 = 1.0, p1 = x;
  if (k == 0) return {p0, 0.0};
  double dp0 = 0.0, dp1 = 1.0;
  for (int n = 1; n < k; ++n) {
    const double p2 = ((2 * n + 1) * x * p1 - n * p0) / (n + 1);
    const double dp2 = dp0 + (2 * n + 1) * p1;
    p0 = p1; p1 = p2;
    dp0 = dp1; dp1 = dp2;
  }
  return {p1, dp1};
}

std::vector<double> bary(const std::vector<double>& x) {
  const int n = (int)x.size();
  std::vector<double> w(n, 1.0);
  for (int i = 0; i < n; ++i)
    for (int j = 0; j < n; ++j)
      if (j != i) w[i] /= (x[i] - x[j]);
  return w;
}

struct Rule {
  std::vector<double> p, w;
};

Rule gauss(int np) {
  Rule r;
  r.p.assign(np, 0.0);
  r.w.assign(np, 0.0);
  for (int i = 0; i < np; ++i) {
    double x = -std::cos(M_PI * (i + 0.75) / (np + 0.5));
    double dp = 1.0;
    for (int it = 0; it < 100; ++it) {
      auto [p, d] = legendre(np, x);
      dp = d;
      const double dx = p / dp;
      x -= dx;
      if (std::abs(dx) < 1e-15) break;
    }
    r.p[i] = x;
    r.w[i] = 2.0 / ((1.0 - x * x) * dp * dp);
  }
  for (int i = 0; i < np / 2; ++i) {
    const double s = 0.5 * (r.p[np - 1 - i] - r.p[i]);
    r.p[i] = -s;
    r.p[np - 1 - i] = s;
    const double w = 0.5 * (r.w[i] + r.w[np - 1 - i]);
    r.w[i] = r.w[np - 1 - i] = w;
  }
  if (np % 2 == 1) r.p[np / 2] = 0.0;
  return r;
}

std::vector<double> lagrange(const HostBasis& b, double x) {
  const int n = b.order + 1;
  std::vector<double> v(n, 0.0);
  for (int i = 0; i < n; ++i)
    if (x == b.nodes[i]) { v[i] = 1.0; return v; }
  const std::vector<double> bw = bary(b.nodes);
  double den = 0.0;
  for (int i = 0; i < n; ++i) { v[i] = bw[i] / (x - b.nodes[i]); den += v[i]; }
  for (int i = 0; i < n; ++i) v[i] /= den;
  return v;
}

// Symmetric LDLT with diagonal pivoting (Eigen::LDLT semantics).
struct Ldlt {
  int n = 0;
  std::vector<double> l, d;
  std::vector<int> perm;
  void compute(std::vector<double> a, int nn) {
    n = nn;
    perm.resize(n);
    for (int i = 0; i < n; ++i) perm[i] = i;
    auto A = [&](int i, int j) -> double& { return a[(size_t)i * n + j]; };
    for (int k = 0; k < n; ++k) {
      int piv = k;
      double best = std::abs(A(k, k));
      for (int i = k + 1; i < n; ++i)
        if (std::abs(A(i, i)) > best) { best = std::abs(A(i, i)); piv = i; }
      if (piv != k) {
        for (int j = 0; j < n; ++j) std::swap(A(k, j), A(piv, j));
        for (int i = 0; i < n; ++i) std::swap(A(i, k), A(i, piv));
        std::swap(perm[k], perm[piv]);
      }
      const double dk = A(k, k);
      for (int i = k + 1; i < n; ++i) A(i, k) /= dk;
      for (int i = k + 1; i < n; ++i)
        for (int j = k + 1; j <= i; ++j) {
          A(i, j) -= A(i, k) * dk * A(j, k);
          A(j, i) = A(i, j);
        }
    }
    l.assign((size_t)n * n, 0.0);
    d.assign(n, 0.0);
    for (int i = 0; i < n; ++i) {
      d[i] = A(i, i);
      l[(size_t)i * n + i] = 1.0;
      for (int j = 0; j < i; ++j) l[(size_t)i * n + j] = A(i, j);
    }
  }
  std::vector<double> solve(const std::vector<double>& b) const {
    std::vector<double> y(n), x(n);
    for (int i = 0; i < n; ++i) y[i] = b[perm[i]];
    for (int i = 0; i < n; ++i)
      for (int j = 0; j < i; ++j) y[i] -= l[(size_t)i * n + j] * y[j];
    for (int i = 0; i < n; ++i) y[i] /= d[i];
    for (int i = n - 1; i >= 0; --i)
      for (int j = i + 1; j < n; ++j) y[i] -= l[(size_t)j * n + i] * y[j];
    for (int i = 0; i < n; ++i) x[perm[i]] = y[i];
    return x;
  }
};

struct SplitMix64 {
  uint64_t state;
  bool has_spare = false;
  double spare = 0.0;
  uint64_t next() {
    uint64_t z = (state += 0x9E3779B97F4A7C15ULL);
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
    return z ^ (z >> 31);
  }
  double uniform() { return double(next() >> 11) * 0x1.0p-53; }
  double normal() {
    if (has_spare) { has_spare = false; return spare; }
    const double u1 = 1.0 - uniform();
    const double u2 = uniform();
    const double r = std::sqrt(-2.0 * std::log(u1));
    const double th = 2.0 * M_PI * u2;
    spare = r * std::sin(th);
    has_spare = true;
    return r * std::cos(th);
  }
};

double ubreak(double a, double b, int i, int n) { return i == n ? b : a + (b - a) * i / n; }

// Isentropic vortex (proj/src/euler.cpp:160-184) with the C4 parameters.
void vortex_c4(double x, double y, double* q) {
  const double gamma = 1.4, alpha = 1.0, lambda = 5.0, uinf = 1.0, vinf = 1.0;
  const double cp = gamma / (gamma - 1.0);
  double xt = x - 5.0 - uinf * 0.0;
  double yt = y - 5.0 - vinf * 0.0;
  xt -= 10.0 * std::round(xt / 10.0);
  yt -= 10.0 * std::round(yt / 10.0);
  const double r2 = xt * xt + yt * yt;
  const double s = lambda / (2.0 * M_PI);
  const double e1 = std::exp(0.5 * alpha * (1.0 - r2));
  const double u = uinf - s * yt * e1;
  const double v = vinf + s * xt * e1;
  const double T = 1.0 - s * s / (2.0 * alpha * cp) * std::exp(alpha * (1.0 - r2));
  const double rho = 1.0 * std::pow(T / 1.0, 1.0 / (gamma - 1.0));
  const double p = 1.0 * std::pow(T / 1.0, gamma / (gamma - 1.0));
  q[0] = rho;
  q[1] = rho * u;
  q[2] = rho * v;
  q[3] = p / (gamma - 1.0) + 0.5 * rho * (u * u + v * v);
}

}  // namespace

HostBasis host_lgl_basis(int order) {
  if (order < 1 || order > 20) throw std::invalid_argument("lgl_basis: order must be in [1, 20]");
  const int n = order + 1;
  HostBasis b;
  b.order = order;
  b.nodes.assign(n, 0.0);
  b.weights.assign(n, 0.0);
  b.nodes[0] = -1.0;
  b.nodes[order] = 1.0;
  for (int i = 1; i < order; ++i) {
    double x = -std::cos(M_PI * i / order);
    for (int it = 0; it < 100; ++it) {
      auto [p, dp] = legendre(order, x);
      const double d2p = (2.0 * x * dp - order * (order + 1) * p) / (1.0 - x * x);
      const double dx = dp / d2p;
      x -= dx;
      if (std::abs(dx) < 1e-15) break;
    }
    b.nodes[i] = x;
  }
  for (int i = 0; i < n / 2; ++i) {
    const double s = 0.5 * (b.nodes[n - 1 - i] - b.nodes[i]);
    b.nodes[i] = -s;
    b.nodes[n - 1 - i] = s;
  }
  if (n % 2 == 1) b.nodes[n / 2] = 0.0;
  for (int i = 0; i < n; ++i) {
    auto [p, dp] = legendre(order, b.nodes[i]);
    (void)dp;
    b.weights[i] = 2.0 / (order * (order + 1) * p * p);
  }
  const std::vector<double> bw = bary(b.nodes);
  b.D.assign((size_t)n * n, 0.0);
  for (int i = 0; i < n; ++i) {
    double row = 0.0;
    for (int j = 0; j < n; ++j) {
      if (j == i) continue;
      b.D[(size_t)i * n + j] = (bw[j] / bw[i]) / (b.nodes[i] - b.nodes[j]);
      row += b.D[(size_t)i * n + j];
    }
    b.D[(size_t)i * n + i] = -row;
  }
  return b;
}

// Over-integration matrices of BurgersOperator (proj/src/burgers.cpp:39-51), built
// with the same products as the reference; M^-1 by LDLT solves of the unit vectors.
HostOI host_burgers_oi(int order) {
  const HostBasis b = host_lgl_basis(order);
  const int np = order + 1;
  const Rule quad = gauss((3 * order + 2 + 1) / 2);
  const int nq = (int)quad.p.size();
  HostOI o;
  o.nq = nq;
  o.I.assign((size_t)nq * np, 0.0);
  for (int q = 0; q < nq; ++q) {
    const std::vector<double> v = lagrange(b, quad.p[q]);
    for (int j = 0; j < np; ++j) o.I[(size_t)q * np + j] = v[j];
  }
  std::vector<double> dI((size_t)nq * np, 0.0);  // dinterp = I D
  for (int q = 0; q < nq; ++q)
    for (int k = 0; k < np; ++k)
      for (int j = 0; j < np; ++j) dI[(size_t)q * np + j] += o.I[(size_t)q * np + k] * b.D[(size_t)k * np + j];
  o.G.assign((size_t)np * np, 0.0);  // (I^T W) dI
  for (int i = 0; i < np; ++i)
    for (int q = 0; q < nq; ++q) {
      const double a = o.I[(size_t)q * np + i] * quad.w[q];
      for (int j = 0; j < np; ++j) o.G[(size_t)i * np + j] += a * dI[(size_t)q * np + j];
    }
  o.Lv.assign((size_t)np * nq, 0.0);  // dI^T W
  for (int i = 0; i < np; ++i)
    for (int q = 0; q < nq; ++q) o.Lv[(size_t)i * nq + q] = dI[(size_t)q * np + i] * quad.w[q];
  std::vector<double> M((size_t)np * np, 0.0);  // (I^T W) I
  for (int i = 0; i < np; ++i)
    for (int q = 0; q < nq; ++q) {
      const double a = o.I[(size_t)q * np + i] * quad.w[q];
      for (int j = 0; j < np; ++j) M[(size_t)i * np + j] += a * o.I[(size_t)q * np + j];
    }
  Ldlt l;
  l.compute(M, np);
  o.Mi.assign((size_t)np * np, 0.0);
  for (int j = 0; j < np; ++j) {
    std::vector<double> e(np, 0.0);
    e[j] = 1.0;
    const std::vector<double> c = l.solve(e);
    for (int i = 0; i < np; ++i) o.Mi[(size_t)i * np + j] = c[i];
  }
  return o;
}

// Weak load of BurgersConfig::source (proj/src/burgers.cpp:80-92): per element
// 0.5 h_e I^T (W s(x_q)) on the operator's quadrature (Gauss (3k+3)/2 points when
// over-integrated, the LGL nodes otherwise).
void host_burgers_source(int order, int ne, double a, double b, bool over_integrate,
                         double (*fn)(double, void*), void* user, double* out) {
  const HostBasis basis = host_lgl_basis(order);
  const int np = order + 1;
  std::vector<double> pts, wts, I;
  if (over_integrate) {
    const Rule quad = gauss((3 * order + 2 + 1) / 2);
    pts = quad.p;
    wts = quad.w;
    I.assign(pts.size() * np, 0.0);
    for (size_t q = 0; q < pts.size(); ++q) {
      const std::vector<double> v = lagrange(basis, pts[q]);
      for (int j = 0; j < np; ++j) I[q * np + j] = v[j];
    }
  } else {
    pts = basis.nodes;
    wts = basis.weights;
    I.assign((size_t)np * np, 0.0);
    for (int j = 0; j < np; ++j) I[(size_t)j * np + j] = 1.0;
  }
  const int nq = (int)pts.size();
  std::vector<double> ws(nq);
  for (int e = 0; e < ne; ++e) {
    const double x0 = ubreak(a, b, e, ne), hx = ubreak(a, b, e + 1, ne) - x0;
    for (int q = 0; q < nq; ++q) ws[q] = wts[q] * fn(x0 + 0.5 * (pts[q] + 1.0) * hx, user);
    for (int i = 0; i < np; ++i) {
      double acc = 0.0;
      for (int q = 0; q < nq; ++q) acc += I[(size_t)q * np + i] * ws[q];
      out[(size_t)e * np + i] = 0.5 * hx * acc;
    }
  }
}

// Per-element {h_e, 2 / h_e} of uniform breakpoints (proj/src/mesh.cpp:11-16), for the
// Burgers element kernels (no divisions on the device).
// Axis breakpoints: the grading list when given (checked like proj/src/mesh.cpp:18-24), else the
// uniform breakpoints of proj/src/mesh.cpp:11-16
std::vector<double> host_axis_breaks(double a, double b, int n, const double* grade) {
  std::vector<double> xs(n + 1);
  if (!grade) {
    for (int i = 0; i <= n; ++i) xs[i] = i == n ? b : a + (b - a) * i / n;
    return xs;
  }
  for (int i = 0; i <= n; ++i) xs[i] = grade[i];
  if (xs.front() != a || xs.back() != b) throw std::invalid_argument("grading list must span the domain");
  for (int i = 1; i <= n; ++i)
    if (xs[i] <= xs[i - 1]) throw std::invalid_argument("grading list must be strictly increasing");
  return xs;
}

// {h_e, 2 / h_e} per element of an axis with the given breakpoints
std::vector<double> host_h_table(const std::vector<double>& xs) {
  const int ne = (int)xs.size() - 1;
  std::vector<double> t(2 * (size_t)ne);
  for (int e = 0; e < ne; ++e) {
    t[2 * e] = xs[e + 1] - xs[e];
    t[2 * e + 1] = 2.0 / (xs[e + 1] - xs[e]);
  }
  return t;
}

std::vector<double> host_h_table(double a, double b, int ne) {
  std::vector<double> t(2 * (size_t)ne);
  for (int e = 0; e < ne; ++e) {
    const double x0 = e == ne ? b : a + (b - a) * e / ne;
    const double x1 = e + 1 == ne ? b : a + (b - a) * (e + 1) / ne;
    t[2 * e] = x1 - x0;
    t[2 * e + 1] = 2.0 / (x1 - x0);
  }
  return t;
}

// Seeded inputs (identical generator and formulas to the oracle's inputs.cpp).
void host_initial_condition(int cfg, int nx, int order, uint64_t seed, double noise, double* out) {
  const HostBasis b = host_lgl_basis(order);
  const int np1 = order + 1;
  SplitMix64 rng{seed};
  if (cfg == 1 || cfg == 2) {
    const double a = 0.0, bb = 2.0 * M_PI;
    double amp[16], ph[16];
    if (cfg == 2)
      for (int k = 0; k < 16; ++k) {
        amp[k] = -0.1 + 0.2 * rng.uniform();
        ph[k] = 2.0 * M_PI * rng.uniform();
      }
    for (int e = 0; e < nx; ++e) {
      const double x0 = ubreak(a, bb, e, nx), hx = ubreak(a, bb, e + 1, nx) - x0;
      for (int i = 0; i < np1; ++i) {
        const double x = x0 + 0.5 * (b.nodes[i] + 1.0) * hx;
        double v;
        if (cfg == 2) {
          v = 0.5;
          for (int k = 0; k < 16; ++k) v += amp[k] * std::sin((k + 1) * x + ph[k]);
        } else {
          v = 0.5 + std::sin(x) + 0.01 * rng.normal();
        }
        out[(size_t)e * np1 + i] = v;
      }
    }
    return;
  }
  if (cfg == 3) {
    const int np = np1 * np1;
    for (int je = 0; je < nx; ++je)
      for (int ie = 0; ie < nx; ++ie) {
        const size_t e = (size_t)je * nx + ie;
        const double x0 = ubreak(0.0, 1.0, ie, nx), hx = ubreak(0.0, 1.0, ie + 1, nx) - x0;
        const double y0 = ubreak(0.0, 1.0, je, nx), hy = ubreak(0.0, 1.0, je + 1, nx) - y0;
        for (int j = 0; j < np1; ++j)
          for (int i = 0; i < np1; ++i) {
            const double x = x0 + 0.5 * (b.nodes[i] + 1.0) * hx;
            const double y = y0 + 0.5 * (b.nodes[j] + 1.0) * hy;
            out[e * np + j * np1 + i] =
                std::sin(2.0 * M_PI * x) * std::sin(2.0 * M_PI * y) + 0.01 * rng.normal();
          }
      }
    return;
  }
  if (cfg == 4) {
    // l2_project_system with gauss_quadrature(k+2) (proj/src/harness.cpp:51,71-75)
    const int np = np1 * np1;
    const Rule quad = gauss(order + 2);
    const int nq = (int)quad.p.size();
    std::vector<double> iq((size_t)nq * np1);
    for (int q = 0; q < nq; ++q) {
      const std::vector<double> v = lagrange(b, quad.p[q]);
      for (int j = 0; j < np1; ++j) iq[(size_t)q * np1 + j] = v[j];
    }
    std::vector<double> mass((size_t)np1 * np1);
    for (int i = 0; i < np1; ++i)
      for (int j = 0; j < np1; ++j) {
        double s = 0.0;
        for (int q = 0; q < nq; ++q) s += iq[(size_t)q * np1 + i] * quad.w[q] * iq[(size_t)q * np1 + j];
        mass[(size_t)i * np1 + j] = s;
      }
    Ldlt ldlt;
    ldlt.compute(mass, np1);
    std::vector<double> fq((size_t)nq * nq * 4), rhs(np1), cx((size_t)np1 * nq);
    for (int je = 0; je < nx; ++je)
      for (int ie = 0; ie < nx; ++ie) {
        const size_t e = (size_t)je * nx + ie;
        const double x0 = ubreak(0.0, 10.0, ie, nx), hx = ubreak(0.0, 10.0, ie + 1, nx) - x0;
        const double y0 = ubreak(0.0, 10.0, je, nx), hy = ubreak(0.0, 10.0, je + 1, nx) - y0;
        for (int qy = 0; qy < nq; ++qy) {
          const double y = y0 + 0.5 * (quad.p[qy] + 1.0) * hy;
          for (int qx = 0; qx < nq; ++qx) {
            const double x = x0 + 0.5 * (quad.p[qx] + 1.0) * hx;
            vortex_c4(x, y, &fq[((size_t)qx * nq + qy) * 4]);
          }
        }
        for (int c = 0; c < 4; ++c) {
          for (int qy = 0; qy < nq; ++qy) {
            for (int i = 0; i < np1; ++i) {
              double s = 0.0;
              for (int qx = 0; qx < nq; ++qx)
                s += iq[(size_t)qx * np1 + i] * (quad.w[qx] * fq[((size_t)qx * nq + qy) * 4 + c]);
              rhs[i] = s;
            }
            const std::vector<double> sol = ldlt.solve(rhs);
            for (int i = 0; i < np1; ++i) cx[(size_t)i * nq + qy] = sol[i];
          }
          double* block = out + (e * 4 + c) * np;
          for (int i = 0; i < np1; ++i) {
            for (int j = 0; j < np1; ++j) {
              double s = 0.0;
              for (int qy = 0; qy < nq; ++qy) s += iq[(size_t)qy * np1 + j] * (quad.w[qy] * cx[(size_t)i * nq + qy]);
              rhs[j] = s;
            }
            const std::vector<double> cy = ldlt.solve(rhs);
            for (int j = 0; j < np1; ++j) block[j * np1 + i] = cy[j];
          }
        }
      }
    for (size_t e = 0; e < (size_t)nx * nx; ++e)
      for (int nd = 0; nd < np; ++nd) out[(e * 4 + 0) * np + nd] += noise * rng.normal();
    return;
  }
  if (cfg == 5) {
    const double box[6] = {0.0, 2.0 * M_PI, 0.0, 2.0 * M_PI, 0.0, 2.0 * M_PI};
    host_tgv_slab(nx, nx, nx, order, box, 0, nx, out);
    return;
  }
  throw std::invalid_argument("initial_condition: config must be 1..5");
}

// C5's Taylor-Green state (Mach 0.1, rho0 = 1) on an nx x ny x nz hex mesh of `box`, z-planes
// [k0, k1) only (element-major, z slowest: the owned slab of a z-partitioned rank, so no rank
// builds the global array); the cubic 2 pi-periodic case is bit-identical to the oracle's
// inputs.cpp generator.
void host_tgv_slab(int nx, int ny, int nz, int order, const double* box, int k0, int k1, double* out) {
  if (nx < 1 || ny < 1 || nz < 1 || k0 < 0 || k1 > nz || k0 >= k1) throw std::invalid_argument("tgv slab: bad mesh");
  const HostBasis b = host_lgl_basis(order);
  const int np1 = order + 1;
  {
    const double gamma = 1.4, rho0 = 1.0, p0 = 1.0 / (gamma * 0.01);
    const int np = np1 * np1 * np1;
    const double hx = (box[1] - box[0]) / nx, hy = (box[3] - box[2]) / ny, hz = (box[5] - box[4]) / nz;
    for (int k = k0; k < k1; ++k)
      for (int j = 0; j < ny; ++j)
        for (int i = 0; i < nx; ++i) {
          const size_t e = ((size_t)(k - k0) * ny + j) * nx + i;
          for (int c2 = 0; c2 < np1; ++c2)
            for (int c1 = 0; c1 < np1; ++c1)
              for (int c0 = 0; c0 < np1; ++c0) {
                const double x = box[0] + i * hx + 0.5 * (b.nodes[c0] + 1.0) * hx;
                const double y = box[2] + j * hy + 0.5 * (b.nodes[c1] + 1.0) * hy;
                const double z = box[4] + k * hz + 0.5 * (b.nodes[c2] + 1.0) * hz;
                const double u = std::sin(x) * std::cos(y) * std::cos(z);
                const double v = -std::cos(x) * std::sin(y) * std::cos(z);
                const double w = 0.0;
                const double p =
                    p0 + (rho0 / 16.0) * (std::cos(2.0 * x) + std::cos(2.0 * y)) * (std::cos(2.0 * z) + 2.0);
                const int node = (c2 * np1 + c1) * np1 + c0;
                const double E = p / (gamma - 1.0) + 0.5 * rho0 * (u * u + v * v + w * w);
                out[(e * 5 + 0) * np + node] = rho0;
                out[(e * 5 + 1) * np + node] = rho0 * u;
                out[(e * 5 + 2) * np + node] = rho0 * v;
                out[(e * 5 + 3) * np + node] = rho0 * w;
                out[(e * 5 + 4) * np + node] = E;
              }
        }
  }
}

}  // namespace expdg
