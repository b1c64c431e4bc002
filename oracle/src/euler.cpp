// ORACLE (test infrastructure): compressible Euler operators.
// Restates proj/src/euler.cpp (2D, Roe and Lax-Friedrichs) and adds the 3D
// Lax-Friedrichs extension used for config C5.
#include <algorithm>
#include <cmath>

#include "oracle.hpp"

namespace oracle {

namespace {
inline State4 mat4_vec(const Mat4& a, const State4& q) {
  State4 r;
  for (int i = 0; i < 4; ++i)
    r[i] = a[i * 4 + 0] * q[0] + a[i * 4 + 1] * q[1] + a[i * 4 + 2] * q[2] + a[i * 4 + 3] * q[3];
  return r;
}
}  // namespace

// proj/src/euler.cpp:8-13
bool admissible(const State4& q, double gamma) {
  if (!(q[0] > 0.0)) return false;
  const double p = (gamma - 1.0) * (q[3] - 0.5 * (q[1] * q[1] + q[2] * q[2]) / q[0]);
  return p > 0.0;
}

// proj/src/euler.cpp:15-24
EulerPrimitives primitives(const State4& q, double gamma) {
  EulerPrimitives pr;
  pr.rho = q[0];
  pr.u = q[1] / q[0];
  pr.v = q[2] / q[0];
  pr.p = (gamma - 1.0) * (q[3] - 0.5 * pr.rho * (pr.u * pr.u + pr.v * pr.v));
  pr.a = std::sqrt(gamma * pr.p / pr.rho);
  pr.H = (q[3] + pr.p) / pr.rho;
  return pr;
}

// proj/src/euler.cpp:26-40
void euler_flux(const State4& q, double gamma, double f[4][2]) {
  if (!admissible(q, gamma)) throw std::domain_error("euler_flux: inadmissible state");
  const EulerPrimitives pr = primitives(q, gamma);
  f[0][0] = q[1];
  f[1][0] = q[1] * pr.u + pr.p;
  f[2][0] = q[2] * pr.u;
  f[3][0] = q[0] * pr.u * pr.H;
  f[0][1] = q[2];
  f[1][1] = q[1] * pr.v;
  f[2][1] = q[2] * pr.v + pr.p;
  f[3][1] = q[0] * pr.v * pr.H;
}

namespace {
// proj/src/euler.cpp:44-73
Mat4 jacobian_from_primitives(const EulerPrimitives& pr, double nx, double ny, double gamma) {
  const double gm1 = gamma - 1.0;
  const double u = pr.u, v = pr.v;
  const double un = u * nx + v * ny;
  const double phi = 0.5 * gm1 * (u * u + v * v);
  const double H = pr.H;
  Mat4 a;
  a[0] = 0.0; a[1] = nx; a[2] = ny; a[3] = 0.0;
  a[4] = phi * nx - u * un;
  a[5] = u * nx - gm1 * nx * u + un;
  a[6] = u * ny - gm1 * nx * v;
  a[7] = gm1 * nx;
  a[8] = phi * ny - v * un;
  a[9] = v * nx - gm1 * ny * u;
  a[10] = v * ny - gm1 * ny * v + un;
  a[11] = gm1 * ny;
  a[12] = (phi - H) * un;
  a[13] = H * nx - gm1 * u * un;
  a[14] = H * ny - gm1 * v * un;
  a[15] = gamma * un;
  return a;
}

// proj/src/euler.cpp:75-103 — |A| = R |Lambda| R^-1 at a Roe state
Mat4 abs_jacobian_from(double rho, double u, double v, double H, double a, double nx, double ny,
                       double gamma) {
  const double gm1 = gamma - 1.0;
  const double un = u * nx + v * ny;
  const double ut = -u * ny + v * nx;
  const double phi = 0.5 * gm1 * (u * u + v * v);
  const double a2 = a * a;
  double r[4][4];  // r[row][col]
  const double c0[4] = {1.0, u - a * nx, v - a * ny, H - a * un};
  const double c1[4] = {1.0, u, v, 0.5 * (u * u + v * v)};
  const double c2[4] = {0.0, -ny, nx, ut};
  const double c3[4] = {1.0, u + a * nx, v + a * ny, H + a * un};
  for (int i = 0; i < 4; ++i) { r[i][0] = c0[i]; r[i][1] = c1[i]; r[i][2] = c2[i]; r[i][3] = c3[i]; }
  const double dp[4] = {phi, -gm1 * u, -gm1 * v, gm1};
  const double dun[4] = {-un / rho, nx / rho, ny / rho, 0.0};
  const double dut[4] = {-ut / rho, -ny / rho, nx / rho, 0.0};
  double rinv[4][4];
  const double e0[4] = {1, 0, 0, 0};
  for (int j = 0; j < 4; ++j) {
    rinv[0][j] = (dp[j] - rho * a * dun[j]) / (2.0 * a2);
    rinv[1][j] = e0[j] - dp[j] / a2;
    rinv[2][j] = rho * dut[j];
    rinv[3][j] = (dp[j] + rho * a * dun[j]) / (2.0 * a2);
  }
  const double lam[4] = {std::abs(un - a), std::abs(un), std::abs(un), std::abs(un + a)};
  double rl[4][4];
  for (int i = 0; i < 4; ++i)
    for (int j = 0; j < 4; ++j) rl[i][j] = r[i][j] * lam[j];
  Mat4 out;
  for (int i = 0; i < 4; ++i)
    for (int j = 0; j < 4; ++j)
      out[i * 4 + j] = rl[i][0] * rinv[0][j] + rl[i][1] * rinv[1][j] + rl[i][2] * rinv[2][j] +
                       rl[i][3] * rinv[3][j];
  return out;
}
}  // namespace

// proj/src/euler.cpp:107-112
Mat4 flux_jacobian(const State4& q, double nx, double ny, double gamma) {
  if (!admissible(q, gamma)) throw std::domain_error("flux_jacobian: inadmissible state");
  return jacobian_from_primitives(primitives(q, gamma), nx, ny, gamma);
}

// proj/src/euler.cpp:114-131
RoeAverage roe_average(const State4& qm, const State4& qp, double gamma) {
  if (!admissible(qm, gamma) || !admissible(qp, gamma))
    throw std::domain_error("roe_average: inadmissible state");
  const EulerPrimitives pm = primitives(qm, gamma), pp = primitives(qp, gamma);
  const double sm = std::sqrt(pm.rho), sp = std::sqrt(pp.rho);
  RoeAverage avg;
  avg.rho = sm * sp;
  avg.u = (sm * pm.u + sp * pp.u) / (sm + sp);
  avg.v = (sm * pm.v + sp * pp.v) / (sm + sp);
  avg.H = (sm * pm.H + sp * pp.H) / (sm + sp);
  const double a2 = (gamma - 1.0) * (avg.H - 0.5 * (avg.u * avg.u + avg.v * avg.v));
  if (!(a2 > 0.0)) throw std::domain_error("roe_average: inadmissible pair");
  avg.a = std::sqrt(a2);
  return avg;
}

// proj/src/euler.cpp:133-136
Mat4 abs_flux_jacobian(const RoeAverage& avg, double nx, double ny, double gamma) {
  return abs_jacobian_from(avg.rho, avg.u, avg.v, avg.H, avg.a, nx, ny, gamma);
}

// proj/src/euler.cpp:138-145
State4 roe_flux(const State4& qm, const State4& qp, double nx, double ny, double gamma) {
  const RoeAverage avg = roe_average(qm, qp, gamma);
  double fm[4][2], fp[4][2];
  euler_flux(qm, gamma, fm);
  euler_flux(qp, gamma, fp);
  const Mat4 aa = abs_flux_jacobian(avg, nx, ny, gamma);
  State4 dq{qm[0] - qp[0], qm[1] - qp[1], qm[2] - qp[2], qm[3] - qp[3]};
  const State4 ad = mat4_vec(aa, dq);
  State4 out;
  for (int i = 0; i < 4; ++i)
    out[i] = 0.5 * ((fm[i][0] + fp[i][0]) * nx + (fm[i][1] + fp[i][1]) * ny) + 0.5 * ad[i];
  return out;
}

// proj/src/euler.cpp:147-158
State4 euler_lax_friedrichs_flux(const State4& qm, const State4& qp, double nx, double ny,
                                 double gamma) {
  const EulerPrimitives pm = primitives(qm, gamma), pp = primitives(qp, gamma);
  const double cm = std::abs(pm.u * nx + pm.v * ny) + pm.a;
  const double cp = std::abs(pp.u * nx + pp.v * ny) + pp.a;
  double fm[4][2], fp[4][2];
  euler_flux(qm, gamma, fm);
  euler_flux(qp, gamma, fp);
  const double s = 0.5 * std::max(cm, cp);
  State4 out;
  for (int i = 0; i < 4; ++i)
    out[i] = 0.5 * ((fm[i][0] + fp[i][0]) * nx + (fm[i][1] + fp[i][1]) * ny) + s * (qm[i] - qp[i]);
  return out;
}

// proj/src/euler.cpp:160-184
State4 isentropic_vortex(double x, double y, double t, const EulerConfig& cfg) {
  const VortexParams& vp = cfg.vortex;
  const double gamma = cfg.gamma;
  const double cp = gamma / (gamma - 1.0);
  double xt = x - vp.xc - vp.u_inf * t;
  double yt = y - vp.yc - vp.v_inf * t;
  if (vp.wrap_lx > 0.0) xt -= vp.wrap_lx * std::round(xt / vp.wrap_lx);
  if (vp.wrap_ly > 0.0) yt -= vp.wrap_ly * std::round(yt / vp.wrap_ly);
  const double r2 = xt * xt + yt * yt;
  const double s = vp.lambda / (2.0 * M_PI);
  const double e1 = std::exp(0.5 * vp.alpha * (1.0 - r2));
  const double u = vp.u_inf - s * yt * e1;
  const double v = vp.v_inf + s * xt * e1;
  const double T = vp.T_inf - s * s / (2.0 * vp.alpha * cp) * std::exp(vp.alpha * (1.0 - r2));
  const double rho = vp.rho_inf * std::pow(T / vp.T_inf, 1.0 / (gamma - 1.0));
  const double p = vp.p_inf * std::pow(T / vp.T_inf, gamma / (gamma - 1.0));
  State4 q;
  q[0] = rho;
  q[1] = rho * u;
  q[2] = rho * v;
  q[3] = p / (gamma - 1.0) + 0.5 * rho * (u * u + v * v);
  return q;
}

// proj/src/euler.cpp:186-244
EulerOperator::EulerOperator(const Mesh& mesh, const NodalBasis& basis, EulerConfig cfg,
                             const Vec& qtilde)
    : mesh_(&mesh), basis_(&basis), cfg_(cfg) {
  if (mesh.dim != 2) throw std::invalid_argument("EulerOperator: 2d meshes only");
  if (mesh.bc != BoundaryKind::periodic) throw std::invalid_argument("EulerOperator: periodic boundaries only");
  np1_ = basis.num_nodes();
  np_ = np1_ * np1_;
  dim_ = long(mesh.num_elements()) * np_ * 4;
  if (long(qtilde.size()) != dim_) throw std::invalid_argument("EulerOperator: reference state size mismatch");
  const int ne = mesh.num_elements();
  jac_x_.resize(size_t(ne) * np_);
  jac_y_.resize(size_t(ne) * np_);
  auto node_state = [&](int e, int node) {
    State4 q;
    for (int c = 0; c < 4; ++c) q[c] = qtilde[(size_t(e) * 4 + c) * np_ + node];
    return q;
  };
  for (int e = 0; e < ne; ++e)
    for (int node = 0; node < np_; ++node) {
      const State4 q = node_state(e, node);
      if (!admissible(q, cfg.gamma)) throw std::domain_error("EulerOperator: inadmissible reference state");
      const EulerPrimitives pr = primitives(q, cfg.gamma);
      jac_x_[size_t(e) * np_ + node] = jacobian_from_primitives(pr, 1.0, 0.0, cfg.gamma);
      jac_y_[size_t(e) * np_ + node] = jacobian_from_primitives(pr, 0.0, 1.0, cfg.gamma);
    }
  face_frozen_.resize(mesh.faces.size() * np1_);
  for (size_t f = 0; f < mesh.faces.size(); ++f) {
    const Face& face = mesh.faces[f];
    const double nx = face.axis == 0 ? face.normal : 0.0;
    const double ny = face.axis == 0 ? 0.0 : face.normal;
    const auto own = face_node_indices(mesh, basis, face, true);
    const auto nbr = face_node_indices(mesh, basis, face, false);
    for (int fn = 0; fn < np1_; ++fn) {
      const State4 qm = node_state(face.owner, own[fn]);
      const State4 qp = node_state(face.neighbor, nbr[fn]);
      FaceFrozen& fd = face_frozen_[f * np1_ + fn];
      const EulerPrimitives pm = primitives(qm, cfg.gamma), pp = primitives(qp, cfg.gamma);
      fd.a_minus = jacobian_from_primitives(pm, nx, ny, cfg.gamma);
      fd.a_plus = jacobian_from_primitives(pp, nx, ny, cfg.gamma);
      if (cfg.flux == EulerFluxKind::roe) {
        fd.a_abs = abs_flux_jacobian(roe_average(qm, qp, cfg.gamma), nx, ny, cfg.gamma);
      } else {
        const double cm = std::abs(pm.u * nx + pm.v * ny) + pm.a;
        const double cp = std::abs(pp.u * nx + pp.v * ny) + pp.a;
        fd.a_abs.fill(0.0);
        const double lam = std::max(cm, cp);
        for (int i = 0; i < 4; ++i) fd.a_abs[i * 5] = lam;
      }
    }
  }
}

// proj/src/euler.cpp:246-258
void EulerOperator::apply_inverse_mass(Vec& r) const {
  const Vec& w = basis_->weights;
  for (int e = 0; e < mesh_->num_elements(); ++e) {
    const Element& el = mesh_->elements[e];
    const double scale = 4.0 / (el.hx * el.hy);
    for (int c = 0; c < 4; ++c) {
      double* block = r.data() + (size_t(e) * 4 + c) * np_;
      for (int j = 0; j < np1_; ++j)
        for (int i = 0; i < np1_; ++i) block[j * np1_ + i] *= scale / (w[i] * w[j]);
    }
  }
}

// proj/src/euler.cpp:260-297
void EulerOperator::rhs_faces(const Vec& q, bool linear_part, Vec& r) const {
  const Vec& w = basis_->weights;
  for (size_t f = 0; f < mesh_->faces.size(); ++f) {
    const Face& face = mesh_->faces[f];
    const double nx = face.axis == 0 ? face.normal : 0.0;
    const double ny = face.axis == 0 ? 0.0 : face.normal;
    const auto own = face_node_indices(*mesh_, *basis_, face, true);
    const auto nbr = face_node_indices(*mesh_, *basis_, face, false);
    const double half_edge = 0.5 * face.measure;
    for (int fn = 0; fn < np1_; ++fn) {
      State4 qm, qp;
      for (int c = 0; c < 4; ++c) {
        qm[c] = q[(size_t(face.owner) * 4 + c) * np_ + own[fn]];
        qp[c] = q[(size_t(face.neighbor) * 4 + c) * np_ + nbr[fn]];
      }
      const FaceFrozen& fd = face_frozen_[f * np1_ + fn];
      const State4 am = mat4_vec(fd.a_minus, qm), ap = mat4_vec(fd.a_plus, qp);
      State4 dq{qm[0] - qp[0], qm[1] - qp[1], qm[2] - qp[2], qm[3] - qp[3]};
      const State4 ad = mat4_vec(fd.a_abs, dq);
      State4 flux;
      for (int c = 0; c < 4; ++c) flux[c] = 0.5 * (am[c] + ap[c]) + 0.5 * ad[c];
      if (!linear_part) {
        const State4 full = cfg_.flux == EulerFluxKind::roe
                                ? roe_flux(qm, qp, nx, ny, cfg_.gamma)
                                : euler_lax_friedrichs_flux(qm, qp, nx, ny, cfg_.gamma);
        for (int c = 0; c < 4; ++c) flux[c] = full[c] - flux[c];
      }
      const double fw = half_edge * w[fn];
      for (int c = 0; c < 4; ++c) {
        r[(size_t(face.owner) * 4 + c) * np_ + own[fn]] -= fw * flux[c];
        r[(size_t(face.neighbor) * 4 + c) * np_ + nbr[fn]] += fw * flux[c];
      }
    }
  }
}

// proj/src/euler.cpp:299-336 / :343-383 (volume integrals of both parts)
void EulerOperator::volume(const Vec& q, bool linear_part, Vec& r) const {
  const Mat& d = basis_->diff;
  const Vec& w = basis_->weights;
  std::vector<State4> fx(np_), fy(np_);
  for (int e = 0; e < mesh_->num_elements(); ++e) {
    const Element& el = mesh_->elements[e];
    for (int node = 0; node < np_; ++node) {
      State4 qn;
      for (int c = 0; c < 4; ++c) qn[c] = q[(size_t(e) * 4 + c) * np_ + node];
      const State4 ax = mat4_vec(jac_x_[size_t(e) * np_ + node], qn);
      const State4 ay = mat4_vec(jac_y_[size_t(e) * np_ + node], qn);
      if (linear_part) {
        fx[node] = ax;
        fy[node] = ay;
      } else {
        const EulerPrimitives pr = primitives(qn, cfg_.gamma);
        const State4 fxc{qn[1], qn[1] * pr.u + pr.p, qn[2] * pr.u, qn[0] * pr.u * pr.H};
        const State4 fyc{qn[2], qn[1] * pr.v, qn[2] * pr.v + pr.p, qn[0] * pr.v * pr.H};
        for (int c = 0; c < 4; ++c) {
          fx[node][c] = fxc[c] - ax[c];
          fy[node][c] = fyc[c] - ay[c];
        }
      }
    }
    for (int c = 0; c < 4; ++c) {
      double* rb = r.data() + (size_t(e) * 4 + c) * np_;
      for (int j = 0; j < np1_; ++j) {
        const double sy = 0.5 * el.hy * w[j];
        for (int m = 0; m < np1_; ++m) {
          double acc = 0.0;
          for (int i = 0; i < np1_; ++i) acc += w[i] * d(i, m) * fx[j * np1_ + i][c];
          rb[j * np1_ + m] += sy * acc;
        }
      }
      for (int i = 0; i < np1_; ++i) {
        const double sx = 0.5 * el.hx * w[i];
        for (int m = 0; m < np1_; ++m) {
          double acc = 0.0;
          for (int j = 0; j < np1_; ++j) acc += w[j] * d(j, m) * fy[j * np1_ + i][c];
          rb[m * np1_ + i] += sx * acc;
        }
      }
    }
  }
}

// proj/src/euler.cpp:299-341 — the Euler JVP
Vec EulerOperator::apply_linear(const Vec& q) const {
  Vec r(dim_, 0.0);
  volume(q, true, r);
  rhs_faces(q, true, r);
  apply_inverse_mass(r);
  return r;
}

// proj/src/euler.cpp:343-388
Vec EulerOperator::apply_nonlinear(const Vec& q) const {
  Vec r(dim_, 0.0);
  volume(q, false, r);
  rhs_faces(q, false, r);
  apply_inverse_mass(r);
  return r;
}

// proj/src/euler.cpp:403-408
Vec euler_full_rhs(const Mesh& mesh, const NodalBasis& basis, const EulerConfig& cfg, const Vec& q) {
  const EulerOperator op(mesh, basis, cfg, q);
  return add(op.apply_linear(q), op.apply_nonlinear(q));
}

// ================================================================ 3D extension
bool admissible3(const State5& q, double gamma) {
  if (!(q[0] > 0.0)) return false;
  const double p = (gamma - 1.0) * (q[4] - 0.5 * (q[1] * q[1] + q[2] * q[2] + q[3] * q[3]) / q[0]);
  return p > 0.0;
}

namespace {
struct Prim3 { double rho, u, v, w, p, a, H; };
Prim3 primitives3(const State5& q, double gamma) {
  Prim3 pr;
  pr.rho = q[0];
  pr.u = q[1] / q[0];
  pr.v = q[2] / q[0];
  pr.w = q[3] / q[0];
  pr.p = (gamma - 1.0) * (q[4] - 0.5 * pr.rho * (pr.u * pr.u + pr.v * pr.v + pr.w * pr.w));
  pr.a = std::sqrt(gamma * pr.p / pr.rho);
  pr.H = (q[4] + pr.p) / pr.rho;
  return pr;
}
Mat5 jac3(const Prim3& pr, const double n[3], double gamma) {
  const double gm1 = gamma - 1.0;
  const double u = pr.u, v = pr.v, w = pr.w;
  const double un = u * n[0] + v * n[1] + w * n[2];
  const double phi = 0.5 * gm1 * (u * u + v * v + w * w);
  const double H = pr.H;
  const double vel[3] = {u, v, w};
  Mat5 a;
  a[0] = 0.0; a[1] = n[0]; a[2] = n[1]; a[3] = n[2]; a[4] = 0.0;
  for (int r = 0; r < 3; ++r) {
    double* row = &a[(r + 1) * 5];
    row[0] = phi * n[r] - vel[r] * un;
    for (int c = 0; c < 3; ++c) {
      row[c + 1] = vel[r] * n[c] - gm1 * n[r] * vel[c];
      if (c == r) row[c + 1] += un;
    }
    row[4] = gm1 * n[r];
  }
  a[20] = (phi - H) * un;
  a[21] = H * n[0] - gm1 * u * un;
  a[22] = H * n[1] - gm1 * v * un;
  a[23] = H * n[2] - gm1 * w * un;
  a[24] = gamma * un;
  return a;
}
inline State5 mat5_vec(const Mat5& a, const State5& q) {
  State5 r;
  for (int i = 0; i < 5; ++i)
    r[i] = a[i * 5 + 0] * q[0] + a[i * 5 + 1] * q[1] + a[i * 5 + 2] * q[2] + a[i * 5 + 3] * q[3] +
           a[i * 5 + 4] * q[4];
  return r;
}
void flux3(const State5& q, const Prim3& pr, int dir, State5& f) {
  const double vn = dir == 0 ? pr.u : dir == 1 ? pr.v : pr.w;
  f[0] = q[dir + 1];
  f[1] = q[1] * vn;
  f[2] = q[2] * vn;
  f[3] = q[3] * vn;
  f[dir + 1] += pr.p;
  f[4] = q[0] * vn * pr.H;
}
}  // namespace

Mat5 flux_jacobian3(const State5& q, const double n[3], double gamma) {
  if (!admissible3(q, gamma)) throw std::domain_error("flux_jacobian3: inadmissible state");
  return jac3(primitives3(q, gamma), n, gamma);
}

Euler3DOperator::Euler3DOperator(const Mesh& mesh, const NodalBasis& basis, double gamma,
                                 const Vec& qtilde)
    : mesh_(&mesh), basis_(&basis), gamma_(gamma), qtilde_(qtilde) {
  if (mesh.dim != 3) throw std::invalid_argument("Euler3DOperator: 3d meshes only");
  np1_ = basis.num_nodes();
  np_ = np1_ * np1_ * np1_;
  dim_ = long(mesh.num_elements()) * np_ * 5;
  if (long(qtilde.size()) != dim_) throw std::invalid_argument("Euler3DOperator: size mismatch");
  for (int e = 0; e < mesh.num_elements(); ++e)
    for (int node = 0; node < np_; ++node) {
      State5 q;
      for (int c = 0; c < 5; ++c) q[c] = qtilde[(size_t(e) * 5 + c) * np_ + node];
      if (!admissible3(q, gamma)) throw std::domain_error("Euler3DOperator: inadmissible reference state");
    }
}

Vec Euler3DOperator::apply(const Vec& q, bool linear_part) const {
  const Mat& d = basis_->diff;
  const Vec& w = basis_->weights;
  const int np1 = np1_, np = np_;
  Vec r(dim_, 0.0);
  auto load = [&](const Vec& v, int e, int node) {
    State5 s;
    for (int c = 0; c < 5; ++c) s[c] = v[(size_t(e) * 5 + c) * np + node];
    return s;
  };
  std::vector<State5> fl[3];
  for (auto& f : fl) f.resize(np);
  for (int e = 0; e < mesh_->num_elements(); ++e) {
    const Element& el = mesh_->elements[e];
    for (int node = 0; node < np; ++node) {
      const State5 qn = load(q, e, node);
      const Prim3 pt = primitives3(load(qtilde_, e, node), gamma_);
      for (int dir = 0; dir < 3; ++dir) {
        const double n[3] = {dir == 0 ? 1.0 : 0.0, dir == 1 ? 1.0 : 0.0, dir == 2 ? 1.0 : 0.0};
        const State5 aq = mat5_vec(jac3(pt, n, gamma_), qn);
        if (linear_part) {
          fl[dir][node] = aq;
        } else {
          State5 f;
          flux3(qn, primitives3(qn, gamma_), dir, f);
          for (int c = 0; c < 5; ++c) fl[dir][node][c] = f[c] - aq[c];
        }
      }
    }
    const double hs[3] = {el.hx, el.hy, el.hz};
    for (int c = 0; c < 5; ++c) {
      double* rb = r.data() + (size_t(e) * 5 + c) * np;
      for (int dir = 0; dir < 3; ++dir) {
        // transverse area factor (1/4) h_a h_b
        const double area = 0.25 * hs[(dir + 1) % 3] * hs[(dir + 2) % 3];
        for (int t2 = 0; t2 < np1; ++t2)
          for (int t1 = 0; t1 < np1; ++t1) {
            auto node_of = [&](int along) {
              int ii, jj, kk;
              if (dir == 0) { ii = along; jj = t1; kk = t2; }
              else if (dir == 1) { ii = t1; jj = along; kk = t2; }
              else { ii = t1; jj = t2; kk = along; }
              return (kk * np1 + jj) * np1 + ii;
            };
            const double s = area * w[t1] * w[t2];
            for (int m = 0; m < np1; ++m) {
              double acc = 0.0;
              for (int i = 0; i < np1; ++i) acc += w[i] * d(i, m) * fl[dir][node_of(i)][c];
              rb[node_of(m)] += s * acc;
            }
          }
      }
    }
  }
  // faces: x, then y, then z (mesh face order)
  for (const Face& face : mesh_->faces) {
    double n[3] = {0, 0, 0};
    n[face.axis] = face.normal;
    const auto own = face_node_indices(*mesh_, *basis_, face, true);
    const auto nbr = face_node_indices(*mesh_, *basis_, face, false);
    const double quarter = 0.25 * face.measure;
    for (int fn = 0; fn < np1 * np1; ++fn) {
      const State5 qm = load(q, face.owner, own[fn]), qp = load(q, face.neighbor, nbr[fn]);
      const Prim3 tm = primitives3(load(qtilde_, face.owner, own[fn]), gamma_);
      const Prim3 tp = primitives3(load(qtilde_, face.neighbor, nbr[fn]), gamma_);
      const State5 am = mat5_vec(jac3(tm, n, gamma_), qm), ap = mat5_vec(jac3(tp, n, gamma_), qp);
      const double cm = std::abs(tm.u * n[0] + tm.v * n[1] + tm.w * n[2]) + tm.a;
      const double cp = std::abs(tp.u * n[0] + tp.v * n[1] + tp.w * n[2]) + tp.a;
      const double lam = std::max(cm, cp);
      State5 flux;
      for (int c = 0; c < 5; ++c) flux[c] = 0.5 * (am[c] + ap[c]) + 0.5 * (lam * (qm[c] - qp[c]));
      if (!linear_part) {
        if (!admissible3(qm, gamma_) || !admissible3(qp, gamma_))
          throw std::domain_error("euler3d flux: inadmissible state");
        const Prim3 pm = primitives3(qm, gamma_), pp = primitives3(qp, gamma_);
        const double sm = std::abs(pm.u * n[0] + pm.v * n[1] + pm.w * n[2]) + pm.a;
        const double sp = std::abs(pp.u * n[0] + pp.v * n[1] + pp.w * n[2]) + pp.a;
        State5 fm, fp;
        flux3(qm, pm, face.axis, fm);
        flux3(qp, pp, face.axis, fp);
        const double s = 0.5 * std::max(sm, sp);
        for (int c = 0; c < 5; ++c) {
          const double full = 0.5 * ((fm[c] + fp[c]) * face.normal) + s * (qm[c] - qp[c]);
          flux[c] = full - flux[c];
        }
      }
      const int t1 = fn % np1, t2 = fn / np1;
      const double fw = quarter * w[t1] * w[t2];
      for (int c = 0; c < 5; ++c) {
        r[(size_t(face.owner) * 5 + c) * np + own[fn]] -= fw * flux[c];
        r[(size_t(face.neighbor) * 5 + c) * np + nbr[fn]] += fw * flux[c];
      }
    }
  }
  for (int e = 0; e < mesh_->num_elements(); ++e) {
    const Element& el = mesh_->elements[e];
    const double scale = 8.0 / (el.hx * el.hy * el.hz);
    for (int c = 0; c < 5; ++c) {
      double* block = r.data() + (size_t(e) * 5 + c) * np;
      for (int k = 0; k < np1; ++k)
        for (int j = 0; j < np1; ++j)
          for (int i = 0; i < np1; ++i) block[(k * np1 + j) * np1 + i] *= scale / (w[i] * w[j] * w[k]);
    }
  }
  return r;
}

Vec Euler3DOperator::apply_linear(const Vec& q) const { return apply(q, true); }
Vec Euler3DOperator::apply_nonlinear(const Vec& q) const { return apply(q, false); }

}  // namespace oracle
