// ORACLE (test infrastructure): viscous Burgers operators.
// Restates proj/src/burgers.cpp (1D, all branches) and adds the 2D
// tensor-product extension used for config C3.
#include <algorithm>
#include <cmath>

#include "oracle.hpp"

namespace oracle {

// proj/src/burgers.cpp:8-13
double entropy_flux(double um, double up, double jump, double sigma, double h) {
  const double avg_half_sq = 0.25 * (um * um + up * up);
  const double avg = 0.5 * (um + up);
  return (avg_half_sq + avg * avg) / 3.0 + (sigma / h) * jump;
}

// proj/src/burgers.cpp:15-18
double lax_friedrichs_flux(double um, double up, double jump) {
  const double avg_half_sq = 0.25 * (um * um + up * up);
  return avg_half_sq + 0.5 * std::max(std::abs(um), std::abs(up)) * jump;
}

namespace {
Mat transpose(const Mat& m) {
  Mat t(m.c, m.r);
  for (int i = 0; i < m.r; ++i)
    for (int j = 0; j < m.c; ++j) t(j, i) = m(i, j);
  return t;
}
Mat diag_right(const Mat& m, const Vec& w) {  // m * diag(w)
  Mat o = m;
  for (int i = 0; i < m.r; ++i)
    for (int j = 0; j < m.c; ++j) o(i, j) = m(i, j) * w[j];
  return o;
}
}  // namespace

// proj/src/burgers.cpp:20-93
BurgersOperator::BurgersOperator(const Mesh& mesh, const NodalBasis& basis, BurgersConfig cfg,
                                 Vec utilde)
    : mesh_(&mesh), basis_(&basis), cfg_(std::move(cfg)), utilde_(std::move(utilde)) {
  if (mesh.dim != 1) throw std::invalid_argument("BurgersOperator: 1d meshes only");
  if (!(cfg_.kappa > 0.0)) throw std::invalid_argument("BurgersOperator: kappa must be positive");
  if (cfg_.sigma < 0.0) throw std::invalid_argument("BurgersOperator: sigma must be nonnegative");
  np_ = basis.num_nodes();
  dim_ = long(mesh.num_elements()) * np_;
  if (long(utilde_.size()) != dim_)
    throw std::invalid_argument("BurgersOperator: reference state size mismatch");
  if (!all_finite(utilde_))
    throw std::invalid_argument("BurgersOperator: reference state not finite");

  const int k = basis.order;
  QuadratureRule quad;
  if (cfg_.over_integrate) {
    quad = gauss_quadrature((3 * k + 2 + 1) / 2);
    interp_ = interpolation_matrix(basis, quad.points);
  } else {
    quad = lgl_quadrature(basis);
    interp_ = Mat::identity(np_);
  }
  wq_ = quad.weights;
  dinterp_ = matmul(interp_, basis.diff);
  grad_vol_ = matmul(diag_right(transpose(interp_), wq_), dinterp_);
  lift_vol_ = diag_right(transpose(dinterp_), wq_);
  mass_.compute(matmul(diag_right(transpose(interp_), wq_), interp_));
  mass_diagonal_ = !cfg_.over_integrate;

  const int ne = mesh.num_elements();
  const int nq = int(wq_.size());
  utilde_q_ = Mat(nq, ne);
  for (int e = 0; e < ne; ++e) {
    const Vec uq = seg_matvec(interp_, utilde_, e);
    for (int q = 0; q < nq; ++q) utilde_q_(q, e) = uq[q];
  }
  faces_.resize(mesh.faces.size());
  for (size_t f = 0; f < mesh.faces.size(); ++f) {
    const Face& face = mesh.faces[f];
    FaceFrozen& fd = faces_[f];
    const int own_node = face.owner_side == 0 ? 0 : k;
    fd.ut_minus = utilde_[size_t(face.owner) * np_ + own_node];
    if (face.neighbor >= 0) {
      const int nb_node = face.neighbor_side == 0 ? 0 : k;
      fd.ut_plus = utilde_[size_t(face.neighbor) * np_ + nb_node];
    } else {
      fd.ut_plus = 0.0;
    }
    fd.diss = 0.5 * std::max(std::abs(fd.ut_minus), std::abs(fd.ut_plus));
    fd.inv_h = 1.0 / face.h_owner;
    const double sigma = cfg_.sigma_adaptive
                             ? cfg_.kappa / 100.0 +
                                   face.h_owner * std::max(std::abs(fd.ut_minus), std::abs(fd.ut_plus))
                             : cfg_.sigma;
    fd.sigma_over_h = sigma * fd.inv_h;
  }
  if (cfg_.source) {
    source_weak_.assign(dim_, 0.0);
    Vec sq(nq);
    for (int e = 0; e < ne; ++e) {
      const Element& el = mesh.elements[e];
      for (int q = 0; q < nq; ++q) sq[q] = cfg_.source(el.x0 + 0.5 * (quad.points[q] + 1.0) * el.hx);
      const double s = 0.5 * el.hx;
      for (int i = 0; i < np_; ++i) {
        double acc = 0.0;
        for (int q = 0; q < nq; ++q) acc += (s * interp_(q, i)) * (wq_[q] * sq[q]);
        source_weak_[size_t(e) * np_ + i] = acc;
      }
    }
  }
}

Vec BurgersOperator::seg_matvec(const Mat& m, const Vec& u, int e) const {
  Vec out(m.r);
  for (int i = 0; i < m.r; ++i) {
    double s = 0.0;
    for (int j = 0; j < m.c; ++j) s += m(i, j) * u[size_t(e) * np_ + j];
    out[i] = s;
  }
  return out;
}

// (2/h_e) * M^-1 r_e per element (proj/src/burgers.cpp:125-129, :175-178)
Vec BurgersOperator::mass_solve_scaled(const Vec& r) const {
  Vec out(dim_);
  Vec seg(np_);
  for (int e = 0; e < mesh_->num_elements(); ++e) {
    const double c = 2.0 / mesh_->elements[e].hx;
    for (int i = 0; i < np_; ++i) seg[i] = r[size_t(e) * np_ + i];
    const Vec s = mass_.solve(seg);
    for (int i = 0; i < np_; ++i) out[size_t(e) * np_ + i] = c * s[i];
  }
  return out;
}

// proj/src/burgers.cpp:95-103
void BurgersOperator::trace_values(const Vec& u, int fi, double& um, double& up) const {
  const Face& face = mesh_->faces[fi];
  const int k = basis_->order;
  um = u[size_t(face.owner) * np_ + (face.owner_side == 0 ? 0 : k)];
  up = face.neighbor >= 0 ? u[size_t(face.neighbor) * np_ + (face.neighbor_side == 0 ? 0 : k)] : 0.0;
}

// proj/src/burgers.cpp:105-130
Vec BurgersOperator::gradient(const Vec& u) const {
  const int ne = mesh_->num_elements();
  const int k = basis_->order;
  Vec r(dim_);
  for (int e = 0; e < ne; ++e) {
    const Vec s = seg_matvec(grad_vol_, u, e);
    for (int i = 0; i < np_; ++i) r[size_t(e) * np_ + i] = s[i];
  }
  for (size_t f = 0; f < mesh_->faces.size(); ++f) {
    const Face& face = mesh_->faces[f];
    double um, up;
    trace_values(u, int(f), um, up);
    const double ustar = face.neighbor >= 0 ? 0.5 * (um + up) : 0.0;
    r[size_t(face.owner) * np_ + (face.owner_side == 0 ? 0 : k)] += face.normal * (ustar - um);
    if (face.neighbor >= 0)
      r[size_t(face.neighbor) * np_ + (face.neighbor_side == 0 ? 0 : k)] -= face.normal * (ustar - up);
  }
  return mass_solve_scaled(r);
}

// proj/src/burgers.cpp:132-135
double BurgersOperator::face_linear_flux(const FaceFrozen& fd, double um, double up,
                                         double jump) const {
  return 0.5 * (fd.ut_minus * um + fd.ut_plus * up) + fd.diss * jump;
}

// proj/src/burgers.cpp:137-144
double BurgersOperator::face_nonlinear_flux(const FaceFrozen& fd, double um, double up,
                                            double jump) const {
  if (cfg_.flux == FluxKind::lax_friedrichs) return lax_friedrichs_flux(um, up, jump);
  const double avg_half_sq = 0.25 * (um * um + up * up);
  const double avg = 0.5 * (um + up);
  return (avg_half_sq + avg * avg) / 3.0 + fd.sigma_over_h * jump;
}

// proj/src/burgers.cpp:146-180 — the JVP L x
Vec BurgersOperator::apply_linear(const Vec& u) const {
  const Vec q = gradient(u);
  const int ne = mesh_->num_elements();
  const int k = basis_->order;
  const int nq = int(wq_.size());
  Vec r(dim_);
  Vec gq(nq);
  for (int e = 0; e < ne; ++e) {
    const Vec iq = seg_matvec(interp_, q, e);
    const Vec iu = seg_matvec(interp_, u, e);
    for (int p = 0; p < nq; ++p) {
      gq[p] = cfg_.kappa * iq[p];
      gq[p] -= utilde_q_(p, e) * iu[p];
    }
    for (int i = 0; i < np_; ++i) {
      double s = 0.0;
      for (int p = 0; p < nq; ++p) s += lift_vol_(i, p) * gq[p];
      r[size_t(e) * np_ + i] = -s;
    }
  }
  for (size_t f = 0; f < mesh_->faces.size(); ++f) {
    const Face& face = mesh_->faces[f];
    const FaceFrozen& fd = faces_[f];
    double um, up, qm, qp;
    trace_values(u, int(f), um, up);
    trace_values(q, int(f), qm, qp);
    const double jump = face.normal * (um - up);
    const double qstar = face.neighbor >= 0 ? 0.5 * (qm + qp) : qm;
    const double flux = cfg_.kappa * qstar - face_linear_flux(fd, um, up, jump);
    r[size_t(face.owner) * np_ + (face.owner_side == 0 ? 0 : k)] += face.normal * flux;
    if (face.neighbor >= 0)
      r[size_t(face.neighbor) * np_ + (face.neighbor_side == 0 ? 0 : k)] -= face.normal * flux;
  }
  return mass_solve_scaled(r);
}

// proj/src/burgers.cpp:182-215
Vec BurgersOperator::apply_nonlinear(const Vec& u) const {
  const int ne = mesh_->num_elements();
  const int k = basis_->order;
  const int nq = int(wq_.size());
  Vec r(dim_);
  Vec gq(nq);
  for (int e = 0; e < ne; ++e) {
    const Vec uq = seg_matvec(interp_, u, e);
    for (int p = 0; p < nq; ++p) gq[p] = utilde_q_(p, e) * uq[p] - 0.5 * (uq[p] * uq[p]);
    for (int i = 0; i < np_; ++i) {
      double s = 0.0;
      for (int p = 0; p < nq; ++p) s += lift_vol_(i, p) * gq[p];
      r[size_t(e) * np_ + i] = -s;
    }
  }
  if (!source_weak_.empty())
    for (long i = 0; i < dim_; ++i) r[i] += source_weak_[i];
  for (size_t f = 0; f < mesh_->faces.size(); ++f) {
    const Face& face = mesh_->faces[f];
    const FaceFrozen& fd = faces_[f];
    double um, up;
    trace_values(u, int(f), um, up);
    const double jump = face.normal * (um - up);
    const double flux = face_linear_flux(fd, um, up, jump) - face_nonlinear_flux(fd, um, up, jump);
    r[size_t(face.owner) * np_ + (face.owner_side == 0 ? 0 : k)] += face.normal * flux;
    if (face.neighbor >= 0)
      r[size_t(face.neighbor) * np_ + (face.neighbor_side == 0 ? 0 : k)] -= face.normal * flux;
  }
  return mass_solve_scaled(r);
}

// proj/src/burgers.cpp:217-265
Vec BurgersOperator::full_rhs(const Vec& u) const {
  const Vec q = gradient(u);
  const int ne = mesh_->num_elements();
  const int k = basis_->order;
  const int nq = int(wq_.size());
  Vec r(dim_);
  Vec gq(nq);
  for (int e = 0; e < ne; ++e) {
    const Vec uq = seg_matvec(interp_, u, e);
    const Vec iq = seg_matvec(interp_, q, e);
    for (int p = 0; p < nq; ++p) gq[p] = cfg_.kappa * iq[p] - 0.5 * (uq[p] * uq[p]);
    for (int i = 0; i < np_; ++i) {
      double s = 0.0;
      for (int p = 0; p < nq; ++p) s += lift_vol_(i, p) * gq[p];
      r[size_t(e) * np_ + i] = -s;
    }
  }
  if (!source_weak_.empty())
    for (long i = 0; i < dim_; ++i) r[i] += source_weak_[i];
  for (size_t f = 0; f < mesh_->faces.size(); ++f) {
    const Face& face = mesh_->faces[f];
    double um, up, qm, qp;
    trace_values(u, int(f), um, up);
    trace_values(q, int(f), qm, qp);
    const double jump = face.normal * (um - up);
    const double qstar = face.neighbor >= 0 ? 0.5 * (qm + qp) : qm;
    double fstar;
    if (cfg_.flux == FluxKind::lax_friedrichs) {
      fstar = lax_friedrichs_flux(um, up, jump);
    } else {
      const double sigma_over_h =
          cfg_.sigma_adaptive ? cfg_.kappa / (100.0 * face.h_owner) + std::max(std::abs(um), std::abs(up))
                              : cfg_.sigma / face.h_owner;
      const double avg_half_sq = 0.25 * (um * um + up * up);
      const double avg = 0.5 * (um + up);
      fstar = (avg_half_sq + avg * avg) / 3.0 + sigma_over_h * jump;
    }
    const double flux = cfg_.kappa * qstar - fstar;
    r[size_t(face.owner) * np_ + (face.owner_side == 0 ? 0 : k)] += face.normal * flux;
    if (face.neighbor >= 0)
      r[size_t(face.neighbor) * np_ + (face.neighbor_side == 0 ? 0 : k)] -= face.normal * flux;
  }
  return mass_solve_scaled(r);
}

// proj/src/burgers.cpp:267-277
double BurgersOperator::inner_product(const Vec& a, const Vec& b) const {
  double sum = 0.0;
  for (int e = 0; e < mesh_->num_elements(); ++e) {
    const Vec aq = seg_matvec(interp_, a, e);
    const Vec bq = seg_matvec(interp_, b, e);
    double s = 0.0;
    for (size_t q = 0; q < wq_.size(); ++q) s += wq_[q] * aq[q] * bq[q];
    sum += 0.5 * mesh_->elements[e].hx * s;
  }
  return sum;
}

// proj/src/burgers.cpp:279-289
double BurgersOperator::penalty_seminorm_sq(const Vec& u) const {
  double sum = 0.0;
  for (size_t f = 0; f < mesh_->faces.size(); ++f) {
    double um, up;
    trace_values(u, int(f), um, up);
    const double jump = mesh_->faces[f].normal * (um - up);
    sum += faces_[f].sigma_over_h * jump * jump;
  }
  return sum;
}

// proj/src/burgers.cpp:291-307
double BurgersOperator::dg_norm_sq(const Vec& u) const {
  double sum = 0.0;
  for (int e = 0; e < mesh_->num_elements(); ++e) {
    const double jac = 2.0 / mesh_->elements[e].hx;
    const Vec d = seg_matvec(dinterp_, u, e);
    double s = 0.0;
    for (size_t q = 0; q < wq_.size(); ++q) s += wq_[q] * (jac * d[q]) * (jac * d[q]);
    sum += 0.5 * mesh_->elements[e].hx * s;
  }
  for (size_t f = 0; f < mesh_->faces.size(); ++f) {
    double um, up;
    trace_values(u, int(f), um, up);
    const double jump = mesh_->faces[f].normal * (um - up);
    sum += faces_[f].inv_h * jump * jump;
  }
  return sum;
}

// ================================================================ 2D extension
namespace {

// One line of the collocated 1D LDG operator (the restated 1D algorithm with
// interp = I): `nel` elements of `np` nodes, values gathered with a stride.
struct Line {
  int nel, np;
  const double* h;    // element sizes along the line
  bool periodic;
  // accessor: value index of (element, node) in the flat field
  std::function<size_t(int, int)> idx;
};

void line_apply(int mode, const Line& L, const Vec& u, const Vec& ut, const Mat& G, const Mat& Lv,
                const Vec& w, const BurgersConfig& cfg, Vec& out_add, bool first) {
  const int np = L.np, ne = L.nel, k = np - 1;
  std::vector<double> r(size_t(ne) * np), q(size_t(ne) * np);
  auto U = [&](int e, int i) { return u[L.idx(e, i)]; };
  auto UT = [&](int e, int i) { return ut[L.idx(e, i)]; };
  // face list: interior (e-1|e) for e=1..ne-1, then wrap (periodic) or two dirichlet faces
  struct F { int own, nb; double normal; int own_node, nb_node; double h; };
  std::vector<F> faces;
  for (int e = 1; e < ne; ++e) faces.push_back({e - 1, e, 1.0, k, 0, L.h[e - 1]});
  if (L.periodic) faces.push_back({ne - 1, 0, 1.0, k, 0, L.h[ne - 1]});
  else {
    faces.push_back({0, -1, -1.0, 0, 0, L.h[0]});
    faces.push_back({ne - 1, -1, 1.0, k, 0, L.h[ne - 1]});
  }
  auto trace = [&](auto&& V, const F& f, double& m, double& p) {
    m = V(f.own, f.own_node);
    p = f.nb >= 0 ? V(f.nb, f.nb_node) : 0.0;
  };
  const bool need_q = mode != 1;
  if (need_q) {
    for (int e = 0; e < ne; ++e)
      for (int i = 0; i < np; ++i) {
        double s = 0.0;
        for (int j = 0; j < np; ++j) s += G(i, j) * U(e, j);
        r[size_t(e) * np + i] = s;
      }
    for (const F& f : faces) {
      double um, up;
      trace(U, f, um, up);
      const double ustar = f.nb >= 0 ? 0.5 * (um + up) : 0.0;
      r[size_t(f.own) * np + f.own_node] += f.normal * (ustar - um);
      if (f.nb >= 0) r[size_t(f.nb) * np + f.nb_node] -= f.normal * (ustar - up);
    }
    for (int e = 0; e < ne; ++e) {
      const double c = 2.0 / L.h[e];
      for (int i = 0; i < np; ++i) q[size_t(e) * np + i] = c * (r[size_t(e) * np + i] / w[i]);
    }
  }
  auto Q = [&](int e, int i) { return q[size_t(e) * np + i]; };
  std::vector<double> gq(np);
  for (int e = 0; e < ne; ++e) {
    for (int p = 0; p < np; ++p) {
      const double x = U(e, p);
      if (mode == 0) { gq[p] = cfg.kappa * Q(e, p); gq[p] -= UT(e, p) * x; }
      else if (mode == 1) gq[p] = UT(e, p) * x - 0.5 * (x * x);
      else gq[p] = cfg.kappa * Q(e, p) - 0.5 * (x * x);
    }
    for (int i = 0; i < np; ++i) {
      double s = 0.0;
      for (int p = 0; p < np; ++p) s += Lv(i, p) * gq[p];
      r[size_t(e) * np + i] = -s;
    }
  }
  for (const F& f : faces) {
    double um, up;
    trace(U, f, um, up);
    const double jump = f.normal * (um - up);
    double flux;
    double ut_m = 0, ut_p = 0;
    if (mode != 2) trace(UT, f, ut_m, ut_p);
    const double diss = 0.5 * std::max(std::abs(ut_m), std::abs(ut_p));
    const double lin = 0.5 * (ut_m * um + ut_p * up) + diss * jump;
    auto nonlin = [&](bool use_frozen_sigma) {
      if (cfg.flux == FluxKind::lax_friedrichs) return lax_friedrichs_flux(um, up, jump);
      double soh;
      if (use_frozen_sigma) {
        const double sigma = cfg.sigma_adaptive ? cfg.kappa / 100.0 + f.h * std::max(std::abs(ut_m), std::abs(ut_p))
                                                : cfg.sigma;
        soh = sigma * (1.0 / f.h);
      } else {
        soh = cfg.sigma_adaptive ? cfg.kappa / (100.0 * f.h) + std::max(std::abs(um), std::abs(up))
                                 : cfg.sigma / f.h;
      }
      const double ahs = 0.25 * (um * um + up * up);
      const double avg = 0.5 * (um + up);
      return (ahs + avg * avg) / 3.0 + soh * jump;
    };
    if (mode == 0) {
      double qm, qp;
      trace(Q, f, qm, qp);
      const double qstar = f.nb >= 0 ? 0.5 * (qm + qp) : qm;
      flux = cfg.kappa * qstar - lin;
    } else if (mode == 1) {
      flux = lin - nonlin(true);
    } else {
      double qm, qp;
      trace(Q, f, qm, qp);
      const double qstar = f.nb >= 0 ? 0.5 * (qm + qp) : qm;
      flux = cfg.kappa * qstar - nonlin(false);
    }
    r[size_t(f.own) * np + f.own_node] += f.normal * flux;
    if (f.nb >= 0) r[size_t(f.nb) * np + f.nb_node] -= f.normal * flux;
  }
  for (int e = 0; e < ne; ++e) {
    const double c = 2.0 / L.h[e];
    for (int i = 0; i < np; ++i) {
      const double v = c * (r[size_t(e) * np + i] / w[i]);
      double& o = out_add[L.idx(e, i)];
      o = first ? v : o + v;
    }
  }
}

}  // namespace

Burgers2DOperator::Burgers2DOperator(const Mesh& mesh, const NodalBasis& basis, BurgersConfig cfg,
                                     Vec utilde)
    : mesh_(&mesh), basis_(&basis), cfg_(std::move(cfg)), utilde_(std::move(utilde)) {
  if (mesh.dim != 2) throw std::invalid_argument("Burgers2DOperator: 2d meshes only");
  if (!(cfg_.kappa > 0.0)) throw std::invalid_argument("Burgers2DOperator: kappa must be positive");
  if (cfg_.over_integrate) throw std::invalid_argument("Burgers2DOperator: collocation only");
  np1_ = basis.num_nodes();
  np_ = np1_ * np1_;
  dim_ = long(mesh.num_elements()) * np_;
  if (long(utilde_.size()) != dim_) throw std::invalid_argument("Burgers2DOperator: size mismatch");
  grad_vol_ = Mat(np1_, np1_);
  lift_vol_ = Mat(np1_, np1_);
  for (int i = 0; i < np1_; ++i)
    for (int j = 0; j < np1_; ++j) {
      grad_vol_(i, j) = basis.weights[i] * basis.diff(i, j);
      lift_vol_(i, j) = basis.diff(j, i) * basis.weights[j];
    }
}

Vec Burgers2DOperator::apply(const Vec& u, Mode mode) const {
  const int nx = mesh_->nx, ny = mesh_->ny, np1 = np1_, np = np_;
  Vec out(dim_, 0.0);
  std::vector<double> hx(nx), hy(ny);
  for (int i = 0; i < nx; ++i) hx[i] = mesh_->xs[i + 1] - mesh_->xs[i];
  for (int j = 0; j < ny; ++j) hy[j] = mesh_->ys[j + 1] - mesh_->ys[j];
  const bool periodic = mesh_->bc == BoundaryKind::periodic;
  // x-lines: element row je, node row jj
  for (int je = 0; je < ny; ++je)
    for (int jj = 0; jj < np1; ++jj) {
      Line L{nx, np1, hx.data(), periodic,
             [=](int e, int i) { return (size_t(je) * nx + e) * np + size_t(jj) * np1 + i; }};
      line_apply(int(mode), L, u, utilde_, grad_vol_, lift_vol_, basis_->weights, cfg_, out, true);
    }
  for (int ie = 0; ie < nx; ++ie)
    for (int ii = 0; ii < np1; ++ii) {
      Line L{ny, np1, hy.data(), periodic,
             [=](int e, int j) { return (size_t(e) * nx + ie) * np + size_t(j) * np1 + ii; }};
      line_apply(int(mode), L, u, utilde_, grad_vol_, lift_vol_, basis_->weights, cfg_, out, false);
    }
  return out;
}

Vec Burgers2DOperator::apply_linear(const Vec& u) const { return apply(u, kLinear); }
Vec Burgers2DOperator::apply_nonlinear(const Vec& u) const { return apply(u, kNonlinear); }
Vec Burgers2DOperator::full_rhs(const Vec& u) const { return apply(u, kFull); }

}  // namespace oracle
