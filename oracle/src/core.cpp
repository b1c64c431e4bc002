// ORACLE (test infrastructure): dense linear algebra, LGL basis and meshes.
// Restates proj/src/basis.cpp and proj/src/mesh.cpp without Eigen.
#include <algorithm>
#include <cmath>
#include <limits>

#include "oracle.hpp"

namespace oracle {

// ---------------------------------------------------------------- linalg
Mat matmul(const Mat& a, const Mat& b) {
  if (a.c != b.r) throw std::invalid_argument("matmul: shape mismatch");
  Mat out(a.r, b.c);
  for (int i = 0; i < a.r; ++i)
    for (int k = 0; k < a.c; ++k) {
      const double aik = a(i, k);
      for (int j = 0; j < b.c; ++j) out(i, j) += aik * b(k, j);
    }
  return out;
}

Vec matvec(const Mat& a, const Vec& x) {
  Vec y(a.r, 0.0);
  for (int i = 0; i < a.r; ++i) {
    double s = 0.0;
    for (int j = 0; j < a.c; ++j) s += a(i, j) * x[j];
    y[i] = s;
  }
  return y;
}

double dot(const Vec& a, const Vec& b) {
  double s = 0.0;
  for (size_t i = 0; i < a.size(); ++i) s += a[i] * b[i];
  return s;
}

double norm(const Vec& a) { return std::sqrt(dot(a, a)); }

Vec axpby(double a, const Vec& x, double b, const Vec& y) {
  Vec z(x.size());
  for (size_t i = 0; i < x.size(); ++i) z[i] = a * x[i] + b * y[i];
  return z;
}

Vec add(const Vec& x, const Vec& y) {
  Vec z(x.size());
  for (size_t i = 0; i < x.size(); ++i) z[i] = x[i] + y[i];
  return z;
}

Vec scale(double a, const Vec& x) {
  Vec z(x.size());
  for (size_t i = 0; i < x.size(); ++i) z[i] = a * x[i];
  return z;
}

double max_abs(const Vec& x) {
  double m = 0.0;
  for (double v : x) m = std::max(m, std::abs(v));
  return m;
}

bool all_finite(const Vec& x) {
  for (double v : x)
    if (!std::isfinite(v)) return false;
  return true;
}

// Eigen::LDLT: symmetric pivoting on the largest remaining diagonal entry.
void LDLT::compute(const Mat& a0) {
  n = a0.r;
  Mat a = a0;
  perm.resize(n);
  for (int i = 0; i < n; ++i) perm[i] = i;
  for (int k = 0; k < n; ++k) {
    int piv = k;
    double best = std::abs(a(k, k));
    for (int i = k + 1; i < n; ++i)
      if (std::abs(a(i, i)) > best) { best = std::abs(a(i, i)); piv = i; }
    if (piv != k) {
      for (int j = 0; j < n; ++j) std::swap(a(k, j), a(piv, j));
      for (int i = 0; i < n; ++i) std::swap(a(i, k), a(i, piv));
      std::swap(perm[k], perm[piv]);
    }
    const double dk = a(k, k);
    for (int i = k + 1; i < n; ++i) a(i, k) /= dk;
    for (int i = k + 1; i < n; ++i)
      for (int j = k + 1; j <= i; ++j) {
        a(i, j) -= a(i, k) * dk * a(j, k);
        a(j, i) = a(i, j);
      }
  }
  l = Mat(n, n);
  d.assign(n, 0.0);
  for (int i = 0; i < n; ++i) {
    d[i] = a(i, i);
    l(i, i) = 1.0;
    for (int j = 0; j < i; ++j) l(i, j) = a(i, j);
  }
}

Vec LDLT::solve(const Vec& b) const {
  Vec y(n);
  for (int i = 0; i < n; ++i) y[i] = b[perm[i]];
  for (int i = 0; i < n; ++i)
    for (int j = 0; j < i; ++j) y[i] -= l(i, j) * y[j];
  for (int i = 0; i < n; ++i) y[i] /= d[i];
  for (int i = n - 1; i >= 0; --i)
    for (int j = i + 1; j < n; ++j) y[i] -= l(j, i) * y[j];
  Vec x(n);
  for (int i = 0; i < n; ++i) x[perm[i]] = y[i];
  return x;
}

// ---------------------------------------------------------------- basis
namespace {

// proj/src/basis.cpp:11-22 — Legendre P_k and derivative, three-term recurrence.
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

// proj/src/basis.cpp:24-31
Vec barycentric_weights(const Vec& nodes) {
  const int n = int(nodes.size());
  Vec w(n, 1.0);
  for (int i = 0; i < n; ++i)
    for (int j = 0; j < n; ++j)
      if (j != i) w[i] /= (nodes[i] - nodes[j]);
  return w;
}

}  // namespace

// proj/src/basis.cpp:35-85
NodalBasis lgl_basis(int order) {
  if (order < 1 || order > 20) throw std::invalid_argument("lgl_basis: order must be in [1, 20]");
  const int n = order + 1;
  NodalBasis b;
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
  const Vec bw = barycentric_weights(b.nodes);
  b.diff = Mat(n, n);
  for (int i = 0; i < n; ++i) {
    double row_sum = 0.0;
    for (int j = 0; j < n; ++j) {
      if (j == i) continue;
      b.diff(i, j) = (bw[j] / bw[i]) / (b.nodes[i] - b.nodes[j]);
      row_sum += b.diff(i, j);
    }
    b.diff(i, i) = -row_sum;
  }
  return b;
}

// proj/src/basis.cpp:87-119
QuadratureRule gauss_quadrature(int num_points) {
  if (num_points < 1) throw std::invalid_argument("gauss_quadrature: need at least one point");
  QuadratureRule r;
  r.points.assign(num_points, 0.0);
  r.weights.assign(num_points, 0.0);
  r.exact_degree = 2 * num_points - 1;
  for (int i = 0; i < num_points; ++i) {
    double x = -std::cos(M_PI * (i + 0.75) / (num_points + 0.5));
    double dp = 1.0;
    for (int it = 0; it < 100; ++it) {
      auto [p, d] = legendre(num_points, x);
      dp = d;
      const double dx = p / dp;
      x -= dx;
      if (std::abs(dx) < 1e-15) break;
    }
    r.points[i] = x;
    r.weights[i] = 2.0 / ((1.0 - x * x) * dp * dp);
  }
  const int n = num_points;
  for (int i = 0; i < n / 2; ++i) {
    const double s = 0.5 * (r.points[n - 1 - i] - r.points[i]);
    r.points[i] = -s;
    r.points[n - 1 - i] = s;
    const double w = 0.5 * (r.weights[i] + r.weights[n - 1 - i]);
    r.weights[i] = r.weights[n - 1 - i] = w;
  }
  if (n % 2 == 1) r.points[n / 2] = 0.0;
  return r;
}

// proj/src/basis.cpp:121-127
QuadratureRule lgl_quadrature(const NodalBasis& b) {
  QuadratureRule r;
  r.points = b.nodes;
  r.weights = b.weights;
  r.exact_degree = 2 * b.order - 1;
  return r;
}

// proj/src/basis.cpp:129-147
Vec lagrange_values(const NodalBasis& b, double x) {
  const int n = b.num_nodes();
  Vec v(n, 0.0);
  for (int i = 0; i < n; ++i)
    if (x == b.nodes[i]) { v[i] = 1.0; return v; }
  const Vec bw = barycentric_weights(b.nodes);
  double denom = 0.0;
  for (int i = 0; i < n; ++i) {
    v[i] = bw[i] / (x - b.nodes[i]);
    denom += v[i];
  }
  for (int i = 0; i < n; ++i) v[i] /= denom;
  return v;
}

// proj/src/basis.cpp:149-155
Mat interpolation_matrix(const NodalBasis& b, const Vec& points) {
  Mat m(int(points.size()), b.num_nodes());
  for (size_t q = 0; q < points.size(); ++q) {
    const Vec v = lagrange_values(b, points[q]);
    for (int j = 0; j < b.num_nodes(); ++j) m(int(q), j) = v[j];
  }
  return m;
}

// ---------------------------------------------------------------- mesh
namespace {
// proj/src/mesh.cpp:11-16
Vec uniform_breaks(double a, double b, int n) {
  Vec xs(n + 1);
  for (int i = 0; i <= n; ++i) xs[i] = a + (b - a) * i / n;
  xs[n] = b;
  return xs;
}
// proj/src/mesh.cpp:18-24
void check_grading(const Vec& g, double lo, double hi) {
  if (g.front() != lo || g.back() != hi) throw std::invalid_argument("grading list must span the domain");
  for (size_t i = 1; i < g.size(); ++i)
    if (g[i] <= g[i - 1]) throw std::invalid_argument("grading list must be strictly increasing");
}
// the grading list when given (its size fixes the element count, proj/src/mesh.cpp:105-118), else uniform
Vec axis_breaks(const Vec& grade, double lo, double hi, int& n) {
  if (grade.empty()) return uniform_breaks(lo, hi, n);
  check_grading(grade, lo, hi);
  n = int(grade.size()) - 1;
  return grade;
}
int locate(const Vec& breaks, double x) {
  const int n = int(breaks.size()) - 1;
  int i = int(std::upper_bound(breaks.begin(), breaks.end(), x) - breaks.begin()) - 1;
  return std::clamp(i, 0, n - 1);
}
}  // namespace

// proj/src/mesh.cpp:41-94
Mesh build_interval_mesh(double a, double b, int ne, BoundaryKind bc) {
  if (!(a < b)) throw std::invalid_argument("degenerate interval");
  if (ne < 1) throw std::invalid_argument("need at least one element");
  Mesh mesh;
  mesh.dim = 1;
  mesh.nx = ne;
  mesh.bc = bc;
  mesh.xs = uniform_breaks(a, b, ne);
  mesh.elements.resize(ne);
  for (int i = 0; i < ne; ++i) {
    Element& e = mesh.elements[i];
    e.x0 = mesh.xs[i];
    e.x1 = mesh.xs[i + 1];
    e.hx = e.x1 - e.x0;
    e.measure = e.hx;
  }
  for (int i = 1; i < ne; ++i) {
    Face f;
    f.owner = i - 1; f.neighbor = i; f.owner_side = 1; f.neighbor_side = 0;
    f.normal = 1.0; f.h_owner = mesh.elements[i - 1].hx;
    mesh.faces.push_back(f);
  }
  if (bc == BoundaryKind::periodic) {
    Face f;
    f.owner = ne - 1; f.neighbor = 0; f.owner_side = 1; f.neighbor_side = 0;
    f.normal = 1.0; f.h_owner = mesh.elements[ne - 1].hx;
    mesh.faces.push_back(f);
  } else {
    Face left;
    left.owner = 0; left.neighbor = -1; left.owner_side = 0; left.normal = -1.0;
    left.h_owner = mesh.elements[0].hx;
    mesh.faces.push_back(left);
    Face right;
    right.owner = ne - 1; right.neighbor = -1; right.owner_side = 1; right.normal = 1.0;
    right.h_owner = mesh.elements[ne - 1].hx;
    mesh.faces.push_back(right);
  }
  return mesh;
}

// proj/src/mesh.cpp:96-227 (optional grading lists replace the uniform axis breakpoints)
Mesh build_quad_mesh(double x0, double x1, double y0, double y1, int nx, int ny,
                     BoundaryKind bc, const Vec& grade_x, const Vec& grade_y) {
  if (!(x0 < x1) || !(y0 < y1)) throw std::invalid_argument("degenerate box");
  if (nx < 1 || ny < 1) throw std::invalid_argument("need at least one element per axis");
  Mesh mesh;
  mesh.dim = 2;
  mesh.bc = bc;
  mesh.xs = axis_breaks(grade_x, x0, x1, nx);
  mesh.ys = axis_breaks(grade_y, y0, y1, ny);
  mesh.nx = nx;
  mesh.ny = ny;
  mesh.elements.resize(size_t(nx) * ny);
  for (int j = 0; j < ny; ++j)
    for (int i = 0; i < nx; ++i) {
      Element& e = mesh.elements[size_t(j) * nx + i];
      e.x0 = mesh.xs[i]; e.x1 = mesh.xs[i + 1];
      e.y0 = mesh.ys[j]; e.y1 = mesh.ys[j + 1];
      e.hx = e.x1 - e.x0; e.hy = e.y1 - e.y0;
      e.measure = e.hx * e.hy;
    }
  auto elem = [nx](int i, int j) { return j * nx + i; };
  auto make = [&](int axis, int owner, int nbr, int os, int ns, double normal) {
    Face f;
    f.axis = axis; f.owner = owner; f.neighbor = nbr;
    f.owner_side = os; f.neighbor_side = ns; f.normal = normal;
    f.h_owner = axis == 0 ? mesh.elements[owner].hx : mesh.elements[owner].hy;
    f.measure = axis == 0 ? mesh.elements[owner].hy : mesh.elements[owner].hx;
    return f;
  };
  for (int j = 0; j < ny; ++j) {
    for (int i = 1; i < nx; ++i) mesh.faces.push_back(make(0, elem(i - 1, j), elem(i, j), 1, 0, 1.0));
    if (bc == BoundaryKind::periodic) {
      mesh.faces.push_back(make(0, elem(nx - 1, j), elem(0, j), 1, 0, 1.0));
    } else {
      mesh.faces.push_back(make(0, elem(0, j), -1, 0, 0, -1.0));
      mesh.faces.push_back(make(0, elem(nx - 1, j), -1, 1, 0, 1.0));
    }
  }
  for (int i = 0; i < nx; ++i) {
    for (int j = 1; j < ny; ++j) mesh.faces.push_back(make(1, elem(i, j - 1), elem(i, j), 1, 0, 1.0));
    if (bc == BoundaryKind::periodic) {
      mesh.faces.push_back(make(1, elem(i, ny - 1), elem(i, 0), 1, 0, 1.0));
    } else {
      mesh.faces.push_back(make(1, elem(i, 0), -1, 0, 0, -1.0));
      mesh.faces.push_back(make(1, elem(i, ny - 1), -1, 1, 0, 1.0));
    }
  }
  return mesh;
}

Mesh build_hex_mesh(double x0, double x1, double y0, double y1, double z0, double z1,
                    int nx, int ny, int nz, const Vec& grade_x, const Vec& grade_y, const Vec& grade_z) {
  Mesh mesh;
  mesh.dim = 3;
  mesh.bc = BoundaryKind::periodic;
  mesh.xs = axis_breaks(grade_x, x0, x1, nx);
  mesh.ys = axis_breaks(grade_y, y0, y1, ny);
  mesh.zs = axis_breaks(grade_z, z0, z1, nz);
  mesh.nx = nx; mesh.ny = ny; mesh.nz = nz;
  mesh.elements.resize(size_t(nx) * ny * nz);
  for (int k = 0; k < nz; ++k)
    for (int j = 0; j < ny; ++j)
      for (int i = 0; i < nx; ++i) {
        Element& e = mesh.elements[(size_t(k) * ny + j) * nx + i];
        e.x0 = mesh.xs[i]; e.x1 = mesh.xs[i + 1];
        e.y0 = mesh.ys[j]; e.y1 = mesh.ys[j + 1];
        e.z0 = mesh.zs[k]; e.z1 = mesh.zs[k + 1];
        e.hx = e.x1 - e.x0; e.hy = e.y1 - e.y0; e.hz = e.z1 - e.z0;
        e.measure = e.hx * e.hy * e.hz;
      }
  auto elem = [nx, ny](int i, int j, int k) { return (k * ny + j) * nx + i; };
  auto make = [&](int axis, int owner, int nbr) {
    Face f;
    f.axis = axis; f.owner = owner; f.neighbor = nbr;
    f.owner_side = 1; f.neighbor_side = 0; f.normal = 1.0;
    const Element& e = mesh.elements[owner];
    f.h_owner = axis == 0 ? e.hx : axis == 1 ? e.hy : e.hz;
    f.measure = axis == 0 ? e.hy * e.hz : axis == 1 ? e.hx * e.hz : e.hx * e.hy;
    return f;
  };
  for (int k = 0; k < nz; ++k)
    for (int j = 0; j < ny; ++j)
      for (int i = 0; i < nx; ++i)
        mesh.faces.push_back(make(0, elem(i, j, k), elem((i + 1) % nx, j, k)));
  for (int k = 0; k < nz; ++k)
    for (int j = 0; j < ny; ++j)
      for (int i = 0; i < nx; ++i)
        mesh.faces.push_back(make(1, elem(i, j, k), elem(i, (j + 1) % ny, k)));
  for (int k = 0; k < nz; ++k)
    for (int j = 0; j < ny; ++j)
      for (int i = 0; i < nx; ++i)
        mesh.faces.push_back(make(2, elem(i, j, k), elem(i, j, (k + 1) % nz)));
  return mesh;
}

// proj/src/mesh.cpp:229-239
double min_node_spacing(const Mesh& mesh, const NodalBasis& b) {
  double min_gap = 2.0;
  for (int i = 0; i < b.order; ++i) min_gap = std::min(min_gap, b.nodes[i + 1] - b.nodes[i]);
  double dx = std::numeric_limits<double>::infinity();
  for (const auto& e : mesh.elements) {
    dx = std::min(dx, e.hx * min_gap / 2.0);
    if (mesh.dim >= 2) dx = std::min(dx, e.hy * min_gap / 2.0);
    if (mesh.dim >= 3) dx = std::min(dx, e.hz * min_gap / 2.0);
  }
  return dx;
}

int nodes_per_element(const Mesh& mesh, const NodalBasis& b) {
  int np = b.num_nodes();
  return mesh.dim == 1 ? np : mesh.dim == 2 ? np * np : np * np * np;
}

// proj/src/mesh.cpp:253-271 (+ z-faces for the 3D extension)
std::vector<int> face_node_indices(const Mesh& mesh, const NodalBasis& b, const Face& face,
                                   bool owner_side) {
  const int np1 = b.num_nodes();
  const int side = owner_side ? face.owner_side : face.neighbor_side;
  const int fixed = side == 0 ? 0 : b.order;
  std::vector<int> idx;
  if (mesh.dim == 1) { idx.push_back(fixed); return idx; }
  if (mesh.dim == 2) {
    for (int t = 0; t < np1; ++t)
      idx.push_back(face.axis == 0 ? t * np1 + fixed : fixed * np1 + t);
    return idx;
  }
  for (int t2 = 0; t2 < np1; ++t2)
    for (int t1 = 0; t1 < np1; ++t1) {
      int i, j, k;
      if (face.axis == 0) { i = fixed; j = t1; k = t2; }
      else if (face.axis == 1) { i = t1; j = fixed; k = t2; }
      else { i = t1; j = t2; k = fixed; }
      idx.push_back((k * np1 + j) * np1 + i);
    }
  return idx;
}

// proj/src/mesh.cpp:315-340 (1D branch)
Vec l2_project_1d(const std::function<double(double)>& f, const Mesh& mesh, const NodalBasis& b,
                  const QuadratureRule& quad) {
  if (quad.exact_degree < 2 * b.order)
    throw std::invalid_argument("l2_project: quadrature must integrate degree 2k exactly");
  const int np = b.num_nodes();
  const Mat iq = interpolation_matrix(b, quad.points);
  Mat mass(np, np);
  for (int i = 0; i < np; ++i)
    for (int j = 0; j < np; ++j) {
      double s = 0.0;
      for (int q = 0; q < iq.r; ++q) s += iq(q, i) * quad.weights[q] * iq(q, j);
      mass(i, j) = s;
    }
  LDLT ldlt;
  ldlt.compute(mass);
  const int nq = int(quad.points.size());
  Vec out(size_t(mesh.num_elements()) * np);
  Vec fq(nq), rhs(np);
  for (int e = 0; e < mesh.num_elements(); ++e) {
    const Element& el = mesh.elements[e];
    for (int q = 0; q < nq; ++q) fq[q] = f(el.x0 + 0.5 * (quad.points[q] + 1.0) * el.hx);
    for (int i = 0; i < np; ++i) {
      double s = 0.0;
      for (int q = 0; q < nq; ++q) s += iq(q, i) * (quad.weights[q] * fq[q]);
      rhs[i] = s;
    }
    const Vec c = ldlt.solve(rhs);
    for (int i = 0; i < np; ++i) out[size_t(e) * np + i] = c[i];
  }
  return out;
}

// proj/src/mesh.cpp:342-386 (2D tensor branch of l2_project, per component)
Vec l2_project_system_2d(const std::function<void(double, double, double*)>& f, int components,
                         const Mesh& mesh, const NodalBasis& b, const QuadratureRule& quad) {
  if (quad.exact_degree < 2 * b.order)
    throw std::invalid_argument("l2_project: quadrature must integrate degree 2k exactly");
  const int np1 = b.num_nodes(), np = np1 * np1;
  const Mat iq = interpolation_matrix(b, quad.points);
  Mat mass(np1, np1);
  for (int i = 0; i < np1; ++i)
    for (int j = 0; j < np1; ++j) {
      double s = 0.0;
      for (int q = 0; q < iq.r; ++q) s += iq(q, i) * quad.weights[q] * iq(q, j);
      mass(i, j) = s;
    }
  LDLT ldlt;
  ldlt.compute(mass);
  const int nq = int(quad.points.size());
  Vec out(size_t(mesh.num_elements()) * np * components, 0.0);
  std::vector<double> fq(size_t(nq) * nq * components);
  Vec col(nq), rhs(np1);
  Mat cx(np1, nq);
  for (int e = 0; e < mesh.num_elements(); ++e) {
    const Element& el = mesh.elements[e];
    for (int qy = 0; qy < nq; ++qy) {
      const double y = el.y0 + 0.5 * (quad.points[qy] + 1.0) * el.hy;
      for (int qx = 0; qx < nq; ++qx) {
        const double x = el.x0 + 0.5 * (quad.points[qx] + 1.0) * el.hx;
        f(x, y, &fq[(size_t(qx) * nq + qy) * components]);
      }
    }
    for (int c = 0; c < components; ++c) {
      for (int qy = 0; qy < nq; ++qy) {
        for (int i = 0; i < np1; ++i) {
          double s = 0.0;
          for (int qx = 0; qx < nq; ++qx)
            s += iq(qx, i) * (quad.weights[qx] * fq[(size_t(qx) * nq + qy) * components + c]);
          rhs[i] = s;
        }
        const Vec sol = ldlt.solve(rhs);
        for (int i = 0; i < np1; ++i) cx(i, qy) = sol[i];
      }
      double* block = &out[(size_t(e) * components + c) * np];
      for (int i = 0; i < np1; ++i) {
        for (int j = 0; j < np1; ++j) {
          double s = 0.0;
          for (int qy = 0; qy < nq; ++qy) s += iq(qy, j) * (quad.weights[qy] * cx(i, qy));
          rhs[j] = s;
        }
        const Vec cy = ldlt.solve(rhs);
        for (int j = 0; j < np1; ++j) block[j * np1 + i] = cy[j];
      }
    }
  }
  return out;
}

// proj/src/mesh.cpp:388-411
double evaluate_1d(const Vec& u, const Mesh& mesh, const NodalBasis& b, double x) {
  const int e = locate(mesh.xs, x);
  const Element& el = mesh.elements[e];
  const double r = 2.0 * (x - el.x0) / el.hx - 1.0;
  const Vec l = lagrange_values(b, r);
  double v = 0.0;
  for (int i = 0; i < b.num_nodes(); ++i) v += l[i] * u[size_t(e) * b.num_nodes() + i];
  return v;
}

double evaluate_2d(const Vec& u, int components, const Mesh& mesh, const NodalBasis& b, double x,
                   double y, int comp) {
  const int np1 = b.num_nodes(), np = np1 * np1;
  const int i = locate(mesh.xs, x), j = locate(mesh.ys, y);
  const int e = j * mesh.nx + i;
  const Element& el = mesh.elements[e];
  const Vec lx = lagrange_values(b, 2.0 * (x - el.x0) / el.hx - 1.0);
  const Vec ly = lagrange_values(b, 2.0 * (y - el.y0) / el.hy - 1.0);
  const double* block = &u[(size_t(e) * components + comp) * np];
  double v = 0.0;
  for (int jj = 0; jj < np1; ++jj)
    for (int ii = 0; ii < np1; ++ii) v += ly[jj] * lx[ii] * block[jj * np1 + ii];
  return v;
}

}  // namespace oracle
