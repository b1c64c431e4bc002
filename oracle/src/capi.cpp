// ORACLE (test infrastructure): flat C entry points for tests/ (ctypes) and
// bench.py's cpu_baseline leg.  Never linked by the product library.
#include <chrono>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <memory>
#include <random>

#include "oracle.hpp"
#include "oracle_inputs.hpp"

using namespace oracle;

extern "C" {

typedef struct {
  int kind;  // 1 burgers1d, 2 burgers2d, 3 euler2d, 4 euler3d
  int order;
  int nx, ny, nz;
  double x0, x1, y0, y1, z0, z1;
  int bc;  // 0 periodic, 1 dirichlet_zero
  double kappa;
  int flux;  // burgers: 0 lax_friedrichs, 1 entropy
  double sigma;
  int sigma_adaptive;
  int over_integrate;
  double gamma;
  int euler_flux;  // 0 roe, 1 lax_friedrichs
  // optional grading lists (build_quad_mesh grade_x / grade_y, proj/src/mesh.cpp:96-120; 3D: + grade_z),
  // nx+1 / ny+1 / nz+1 breakpoints, NULL: uniform
  const double* grade_x;
  const double* grade_y;
  const double* grade_z;
} oracle_problem_desc;

}

namespace {

thread_local char g_err[512];

void set_err(const char* what) {
  std::snprintf(g_err, sizeof(g_err), "%s", what);
}

struct Problem {
  oracle_problem_desc d;
  Mesh mesh;
  NodalBasis basis;
  BurgersConfig bcfg;
  EulerConfig ecfg;
  long dim = 0;
};

SplitOperator make_split(const Problem& P, const Vec& ref) {
  SplitOperator s;
  s.dim = P.dim;
  switch (P.d.kind) {
    case 1: {
      auto op = std::make_shared<BurgersOperator>(P.mesh, P.basis, P.bcfg, ref);
      s.linear = [op](const Vec& u) { return op->apply_linear(u); };
      s.nonlinear = [op](const Vec& u) { return op->apply_nonlinear(u); };
      break;
    }
    case 2: {
      auto op = std::make_shared<Burgers2DOperator>(P.mesh, P.basis, P.bcfg, ref);
      s.linear = [op](const Vec& u) { return op->apply_linear(u); };
      s.nonlinear = [op](const Vec& u) { return op->apply_nonlinear(u); };
      break;
    }
    case 3: {
      auto op = std::make_shared<EulerOperator>(P.mesh, P.basis, P.ecfg, ref);
      s.linear = [op](const Vec& u) { return op->apply_linear(u); };
      s.nonlinear = [op](const Vec& u) { return op->apply_nonlinear(u); };
      break;
    }
    case 4: {
      auto op = std::make_shared<Euler3DOperator>(P.mesh, P.basis, P.ecfg.gamma, ref);
      s.linear = [op](const Vec& u) { return op->apply_linear(u); };
      s.nonlinear = [op](const Vec& u) { return op->apply_nonlinear(u); };
      break;
    }
    default:
      throw std::invalid_argument("unknown problem kind");
  }
  return s;
}

Vec full_rhs(const Problem& P, const Vec& u) {
  switch (P.d.kind) {
    case 1: return BurgersOperator(P.mesh, P.basis, P.bcfg, Vec(P.dim, 0.0)).full_rhs(u);
    case 2: return Burgers2DOperator(P.mesh, P.basis, P.bcfg, Vec(P.dim, 0.0)).full_rhs(u);
    case 3: return euler_full_rhs(P.mesh, P.basis, P.ecfg, u);
    case 4: {
      Euler3DOperator op(P.mesh, P.basis, P.ecfg.gamma, u);
      return add(op.apply_linear(u), op.apply_nonlinear(u));
    }
  }
  throw std::invalid_argument("unknown problem kind");
}

}  // namespace

extern "C" {

const char* oracle_last_error() { return g_err; }

void* oracle_problem_create(const oracle_problem_desc* d) {
  try {
    auto P = std::make_unique<Problem>();
    P->d = *d;
    P->basis = lgl_basis(d->order);
    const BoundaryKind bc = d->bc == 0 ? BoundaryKind::periodic : BoundaryKind::dirichlet_zero;
    switch (d->kind) {
      case 1: P->mesh = build_interval_mesh(d->x0, d->x1, d->nx, bc); break;
      case 2:
      case 3: {
        const Vec gx = d->grade_x ? Vec(d->grade_x, d->grade_x + d->nx + 1) : Vec();
        const Vec gy = d->grade_y ? Vec(d->grade_y, d->grade_y + d->ny + 1) : Vec();
        P->mesh = build_quad_mesh(d->x0, d->x1, d->y0, d->y1, d->nx, d->ny, bc, gx, gy);
        break;
      }
      case 4: {
        const Vec gx = d->grade_x ? Vec(d->grade_x, d->grade_x + d->nx + 1) : Vec();
        const Vec gy = d->grade_y ? Vec(d->grade_y, d->grade_y + d->ny + 1) : Vec();
        const Vec gz = d->grade_z ? Vec(d->grade_z, d->grade_z + d->nz + 1) : Vec();
        P->mesh = build_hex_mesh(d->x0, d->x1, d->y0, d->y1, d->z0, d->z1, d->nx, d->ny, d->nz, gx, gy, gz);
        break;
      }
      default: throw std::invalid_argument("unknown problem kind");
    }
    P->bcfg.kappa = d->kappa;
    P->bcfg.flux = d->flux == 1 ? FluxKind::entropy : FluxKind::lax_friedrichs;
    P->bcfg.sigma = d->sigma;
    P->bcfg.sigma_adaptive = d->sigma_adaptive != 0;
    P->bcfg.over_integrate = d->over_integrate != 0;
    P->ecfg.gamma = d->gamma;
    P->ecfg.flux = d->euler_flux == 0 ? EulerFluxKind::roe : EulerFluxKind::lax_friedrichs;
    const int comps = d->kind == 3 ? 4 : d->kind == 4 ? 5 : 1;
    P->dim = long(P->mesh.num_elements()) * nodes_per_element(P->mesh, P->basis) * comps;
    return P.release();
  } catch (const std::exception& e) {
    set_err(e.what());
    return nullptr;
  }
}

void oracle_problem_destroy(void* h) { delete static_cast<Problem*>(h); }
long oracle_problem_dim(void* h) { return static_cast<Problem*>(h)->dim; }

// which: 0 = L (apply_linear at ref), 1 = N (apply_nonlinear at ref), 2 = full rhs
// returns 0 ok, 1 invalid_argument, 2 domain_error, 3 other
int oracle_apply(void* h, int which, const double* ref, const double* x, double* y) {
  try {
    const Problem& P = *static_cast<Problem*>(h);
    const Vec xv(x, x + P.dim);
    Vec out;
    if (which == 2) {
      out = full_rhs(P, xv);
    } else {
      const SplitOperator s = make_split(P, Vec(ref, ref + P.dim));
      out = which == 0 ? s.linear(xv) : s.nonlinear(xv);
    }
    std::memcpy(y, out.data(), sizeof(double) * P.dim);
    return 0;
  } catch (const std::invalid_argument& e) { set_err(e.what()); return 1; }
  catch (const std::domain_error& e) { set_err(e.what()); return 2; }
  catch (const std::exception& e) { set_err(e.what()); return 3; }
}

// Burgers 1D diagnostics used by the energy-identity pins.
int oracle_burgers_diag(void* h, const double* ref, const double* u, double* q_out, double* ip_u_rhs,
                        double* ip_q_q, double* pen, double* ip_u_u) {
  try {
    const Problem& P = *static_cast<Problem*>(h);
    const Vec uv(u, u + P.dim);
    BurgersOperator op(P.mesh, P.basis, P.bcfg, Vec(ref, ref + P.dim));
    const Vec rhs = add(op.apply_linear(uv), op.apply_nonlinear(uv));
    const Vec q = op.gradient(uv);
    if (q_out) std::memcpy(q_out, q.data(), sizeof(double) * P.dim);
    *ip_u_rhs = op.inner_product(uv, rhs);
    *ip_q_q = op.inner_product(q, q);
    *pen = op.penalty_seminorm_sq(uv);
    *ip_u_u = op.inner_product(uv, uv);
    return 0;
  } catch (const std::exception& e) { set_err(e.what()); return 3; }
}

// Mass inner product <a, b> of the Burgers operator's quadrature (BurgersOperator::inner_product):
// the checker for device right-hand sides in the energy / conservation identities.
int oracle_burgers_inner(void* h, const double* a, const double* b, double* out) {
  try {
    const Problem& P = *static_cast<Problem*>(h);
    BurgersOperator op(P.mesh, P.basis, P.bcfg, Vec(a, a + P.dim));
    *out = op.inner_product(Vec(a, a + P.dim), Vec(b, b + P.dim));
    return 0;
  } catch (const std::exception& e) { set_err(e.what()); return 3; }
}

// integrator: 0 exp_euler 1 epi2 2 exprb32 3 exprb42 4 rk2 5 rk3 6 rk4
// Per-step outputs (nullable, capacity max_steps): cumulative Krylov iterations, max|u|.
int oracle_integrate(void* h, int integrator, double* u, double dt, double t_final, double tol,
                     int max_basis, int orth_length, int max_steps, long* iters_per_step,
                     double* amax_per_step, int* steps_out, int* status_out, int* blow_up_step_out,
                     double* max_abs_out, long* total_iters_out, double* seconds_out, int snapshot_every,
                     double* snaps, double* snap_t, int snap_cap, int* n_snaps) {
  try {
    const Problem& P = *static_cast<Problem*>(h);
    SplitProblem sp;
    sp.dim = P.dim;
    sp.linearize = [&P](const Vec& ref) { return make_split(P, ref); };
    std::shared_ptr<BurgersOperator> b1;
    std::shared_ptr<Burgers2DOperator> b2;
    if (P.d.kind == 1) b1 = std::make_shared<BurgersOperator>(P.mesh, P.basis, P.bcfg, Vec(P.dim, 0.0));
    if (P.d.kind == 2) b2 = std::make_shared<Burgers2DOperator>(P.mesh, P.basis, P.bcfg, Vec(P.dim, 0.0));
    sp.rhs = [&P, b1, b2](const Vec& v) {
      if (b1) return b1->full_rhs(v);
      if (b2) return b2->full_rhs(v);
      return full_rhs(P, v);
    };
    TimeLoopConfig tl;
    tl.dt = dt;
    tl.t_final = t_final;
    tl.krylov.tol = tol;
    tl.krylov.max_basis = max_basis;
    tl.krylov.orth_length = orth_length;
    tl.snapshot_every = snapshot_every;
    tl.on_step = [&](int step, double, double amax, long iters) {
      if (step - 1 < max_steps) {
        if (iters_per_step) iters_per_step[step - 1] = iters;
        if (amax_per_step) amax_per_step[step - 1] = amax;
      }
    };
    const IntegratorKind kinds[] = {IntegratorKind::exp_euler, IntegratorKind::epi2, IntegratorKind::exprb32,
                                    IntegratorKind::exprb42,   IntegratorKind::rk2,  IntegratorKind::rk3,
                                    IntegratorKind::rk4};
    const auto t0 = std::chrono::steady_clock::now();
    IntegrationResult r = integrate(sp, kinds[integrator], Vec(u, u + P.dim), tl);
    const auto t1 = std::chrono::steady_clock::now();
    if (seconds_out) *seconds_out = std::chrono::duration<double>(t1 - t0).count();
    std::memcpy(u, r.u.data(), sizeof(double) * P.dim);
    *steps_out = r.steps;
    *status_out = r.status == RunStatus::completed ? 0 : 1;
    *blow_up_step_out = r.blow_up_step;
    *max_abs_out = r.max_abs;
    *total_iters_out = r.krylov_iterations;
    int k = 0;
    for (const auto& sn : r.snapshots) {
      if (k >= snap_cap) break;
      if (snap_t) snap_t[k] = sn.first;
      if (snaps) std::memcpy(snaps + size_t(k) * P.dim, sn.second.data(), sizeof(double) * P.dim);
      ++k;
    }
    if (n_snaps) *n_snaps = (int)r.snapshots.size();
    return 0;
  } catch (const std::invalid_argument& e) { set_err(e.what()); return 1; }
  catch (const std::exception& e) { set_err(e.what()); return 3; }
}

// ------------------------------------------------------------ phi engine on dense operators
int oracle_phi_dense_op(int n, const double* A, int p, const double* b, double dt, double tol,
                        int max_basis, int orth_length, double* out, long* iters, int* substeps,
                        double* last_estimate) {
  try {
    Mat M(n, n);
    std::memcpy(M.a.data(), A, sizeof(double) * n * n);
    PhiCombinationProblem prob;
    prob.op = [&M](const Vec& v) { return matvec(M, v); };
    for (int i = 0; i <= p; ++i) prob.b.emplace_back(b + size_t(i) * n, b + size_t(i + 1) * n);
    prob.dt = dt;
    prob.tol = tol;
    prob.max_basis = max_basis;
    prob.orth_length = orth_length;
    const PhiCombinationResult r = phi_combination(prob);
    std::memcpy(out, r.value.data(), sizeof(double) * n);
    *iters = r.stats.iterations;
    *substeps = r.stats.substeps;
    return 0;
  } catch (const KrylovError& e) {
    set_err(e.what());
    if (last_estimate) *last_estimate = e.last_estimate;
    return 4;
  } catch (const std::invalid_argument& e) { set_err(e.what()); return 1; }
  catch (const std::exception& e) { set_err(e.what()); return 3; }
}

// ------------------------------------------------------------ user LinearAction / SplitProblem
// (host callbacks on host vectors: the reference's std::function plug-ins,
// proj/include/expdg/phi.hpp:11 and proj/include/expdg/integrators.hpp:48-52)
typedef int (*UserApply)(const double* x, double* y, void* user);
typedef int (*UserLinearize)(const double* ref, void* user);

static void user_status(int rc, const char* what) {
  if (rc == 0) return;
  if (rc == 2) throw std::domain_error(std::string("user operator: ") + what);
  if (rc == 1) throw std::invalid_argument(std::string("user operator: ") + what);
  throw std::runtime_error(std::string("user operator: ") + what);
}

static LinearAction user_action(long n, UserApply f, void* user, const char* what) {
  return [n, f, user, what](const Vec& v) {
    Vec y(n, 0.0);
    if (f) user_status(f(v.data(), y.data(), user), what);
    return y;
  };
}

int oracle_phi_user(int n, UserApply apply, void* user, int p, const double* b, double dt, double tol,
                    int max_basis, int orth_length, double* out, long* iters, int* substeps,
                    double* last_estimate) {
  try {
    PhiCombinationProblem prob;
    prob.op = user_action(n, apply, user, "apply_linear");
    for (int i = 0; i <= p; ++i) prob.b.emplace_back(b + size_t(i) * n, b + size_t(i + 1) * n);
    prob.dt = dt;
    prob.tol = tol;
    prob.max_basis = max_basis;
    prob.orth_length = orth_length;
    const PhiCombinationResult r = phi_combination(prob);
    std::memcpy(out, r.value.data(), sizeof(double) * n);
    *iters = r.stats.iterations;
    *substeps = r.stats.substeps;
    return 0;
  } catch (const KrylovError& e) {
    set_err(e.what());
    if (last_estimate) *last_estimate = e.last_estimate;
    return 4;
  } catch (const std::invalid_argument& e) { set_err(e.what()); return 1; }
  catch (const std::domain_error& e) { set_err(e.what()); return 2; }
  catch (const std::exception& e) { set_err(e.what()); return 3; }
}

int oracle_integrate_user(long n, UserApply lin, UserApply nonlin, UserLinearize linearize, void* user,
                          int integrator, double* u, double dt, double t_final, double tol, int max_basis,
                          int orth_length, int max_steps, long* iters_per_step, double* amax_per_step,
                          int* steps_out, int* status_out, int* blow_up_step_out, double* max_abs_out,
                          long* total_iters_out, int snapshot_every, double* snaps, double* snap_t, int snap_cap,
                          int* n_snaps) {
  try {
    SplitProblem sp;
    sp.dim = n;
    sp.linearize = [=](const Vec& ref) {
      if (linearize) user_status(linearize(ref.data(), user), "linearize");
      SplitOperator op;
      op.dim = n;
      op.linear = user_action(n, lin, user, "apply_linear");
      op.nonlinear = user_action(n, nonlin, user, "apply_nonlinear");
      return op;
    };
    TimeLoopConfig tl;
    tl.dt = dt;
    tl.t_final = t_final;
    tl.krylov.tol = tol;
    tl.krylov.max_basis = max_basis;
    tl.krylov.orth_length = orth_length;
    tl.snapshot_every = snapshot_every;
    tl.on_step = [&](int step, double, double amax, long it) {
      if (step - 1 < max_steps) {
        if (iters_per_step) iters_per_step[step - 1] = it;
        if (amax_per_step) amax_per_step[step - 1] = amax;
      }
    };
    const IntegratorKind kinds[] = {IntegratorKind::exp_euler, IntegratorKind::epi2, IntegratorKind::exprb32,
                                    IntegratorKind::exprb42};
    if (integrator < 0 || integrator > 3) throw std::invalid_argument("integrate_user: exponential integrators only");
    IntegrationResult r = integrate(sp, kinds[integrator], Vec(u, u + n), tl);
    std::memcpy(u, r.u.data(), sizeof(double) * n);
    *steps_out = r.steps;
    *status_out = r.status == RunStatus::completed ? 0 : 1;
    *blow_up_step_out = r.blow_up_step;
    *max_abs_out = r.max_abs;
    *total_iters_out = r.krylov_iterations;
    int k = 0;
    for (const auto& sn : r.snapshots) {
      if (k >= snap_cap) break;
      if (snap_t) snap_t[k] = sn.first;
      if (snaps) std::memcpy(snaps + size_t(k) * n, sn.second.data(), sizeof(double) * n);
      ++k;
    }
    if (n_snaps) *n_snaps = (int)r.snapshots.size();
    return 0;
  } catch (const std::invalid_argument& e) { set_err(e.what()); return 1; }
  catch (const std::domain_error& e) { set_err(e.what()); return 2; }
  catch (const std::exception& e) { set_err(e.what()); return 3; }
}

int oracle_expm(int n, const double* a, double* out) {
  Mat M(n, n);
  std::memcpy(M.a.data(), a, sizeof(double) * n * n);
  const Mat E = expm(M);
  std::memcpy(out, E.a.data(), sizeof(double) * n * n);
  return 0;
}

int oracle_phi_dense_family(int p, int n, const double* a, double* out /*(p+1) n n*/) {
  Mat M(n, n);
  std::memcpy(M.a.data(), a, sizeof(double) * n * n);
  const auto fam = phi_dense_family(p, M);
  for (int i = 0; i <= p; ++i) std::memcpy(out + size_t(i) * n * n, fam[i].a.data(), sizeof(double) * n * n);
  return 0;
}

double oracle_phi_scalar(int i, double tau) { return phi_scalar(i, tau); }

int oracle_krylov_build(int n, const double* A, const double* seed, int m, int orth_length,
                        double* basis /* n x (m+1) row-major */, double* hess /* (m+1) x m */,
                        int* m_out, int* invariant, double* seed_norm) {
  try {
    Mat M(n, n);
    std::memcpy(M.a.data(), A, sizeof(double) * n * n);
    const KrylovFactorization f =
        krylov_build([&M](const Vec& v) { return matvec(M, v); }, Vec(seed, seed + n), m, orth_length);
    *m_out = f.m;
    *invariant = f.invariant_subspace ? 1 : 0;
    *seed_norm = f.seed_norm;
    for (int i = 0; i < n; ++i)
      for (int j = 0; j < f.basis.c; ++j) basis[size_t(i) * (m + 1) + j] = f.basis(i, j);
    for (int i = 0; i < f.hessenberg.r; ++i)
      for (int j = 0; j < f.hessenberg.c; ++j) hess[size_t(i) * m + j] = f.hessenberg(i, j);
    return 0;
  } catch (const std::invalid_argument& e) { set_err(e.what()); return 1; }
}

// ------------------------------------------------------------ basis / mesh helpers
int oracle_lgl(int order, double* nodes, double* weights, double* D) {
  try {
    const NodalBasis b = lgl_basis(order);
    const int n = b.num_nodes();
    std::memcpy(nodes, b.nodes.data(), sizeof(double) * n);
    std::memcpy(weights, b.weights.data(), sizeof(double) * n);
    std::memcpy(D, b.diff.a.data(), sizeof(double) * n * n);
    return 0;
  } catch (const std::invalid_argument& e) { set_err(e.what()); return 1; }
}

int oracle_gauss(int npts, double* pts, double* w) {
  try {
    const QuadratureRule r = gauss_quadrature(npts);
    std::memcpy(pts, r.points.data(), sizeof(double) * npts);
    std::memcpy(w, r.weights.data(), sizeof(double) * npts);
    return 0;
  } catch (const std::invalid_argument& e) { set_err(e.what()); return 1; }
}

int oracle_euler_pointwise(int what, const double* qm, const double* qp, double nx, double ny,
                           double gamma, double* out) {
  // what: 0 flux(qm) 4x2, 1 jacobian(qm,n) 4x4, 2 roe flux, 3 LF flux, 4 |A|(roe avg), 5 roe avg
  try {
    State4 a{qm[0], qm[1], qm[2], qm[3]}, b{qp[0], qp[1], qp[2], qp[3]};
    switch (what) {
      case 0: { double f[4][2]; euler_flux(a, gamma, f); for (int i = 0; i < 4; ++i) { out[2 * i] = f[i][0]; out[2 * i + 1] = f[i][1]; } break; }
      case 1: { const Mat4 m = flux_jacobian(a, nx, ny, gamma); std::memcpy(out, m.data(), 16 * 8); break; }
      case 2: { const State4 f = roe_flux(a, b, nx, ny, gamma); std::memcpy(out, f.data(), 32); break; }
      case 3: { const State4 f = euler_lax_friedrichs_flux(a, b, nx, ny, gamma); std::memcpy(out, f.data(), 32); break; }
      case 4: { const Mat4 m = abs_flux_jacobian(roe_average(a, b, gamma), nx, ny, gamma); std::memcpy(out, m.data(), 128); break; }
      case 5: { const RoeAverage r = roe_average(a, b, gamma); out[0] = r.rho; out[1] = r.u; out[2] = r.v; out[3] = r.H; out[4] = r.a; break; }
      default: return 1;
    }
    return 0;
  } catch (const std::domain_error& e) { set_err(e.what()); return 2; }
}

double oracle_burgers_flux(int kind, double um, double up, double jump, double sigma, double h) {
  return kind == 1 ? entropy_flux(um, up, jump, sigma, h) : lax_friedrichs_flux(um, up, jump);
}

int oracle_vortex(double x, double y, double t, const double* vp /*11 params*/, double gamma, double* out) {
  EulerConfig c;
  c.gamma = gamma;
  c.vortex = VortexParams{vp[0], vp[1], vp[2], vp[3], vp[4], vp[5], vp[6], vp[7], vp[8], vp[9], vp[10]};
  const State4 q = isentropic_vortex(x, y, t, c);
  std::memcpy(out, q.data(), 32);
  return 0;
}

// ------------------------------------------------------------ inputs
// cfg: 1 (C1), 2 (C2), 3 (C3), 4 (C4), 5 (C5)
int oracle_ic(int cfg, int nx, int order, uint64_t seed, double noise, double* out) {
  try {
    Vec v;
    switch (cfg) {
      case 1: case 2: v = ic_burgers1d(cfg, nx, order, seed); break;
      case 3: v = ic_burgers2d(nx, nx, order, seed); break;
      case 4: v = ic_euler2d_vortex(nx, order, seed, noise); break;
      case 5: v = ic_euler3d_tgv(nx, order, 1.4); break;
      default: throw std::invalid_argument("unknown config");
    }
    std::memcpy(out, v.data(), sizeof(double) * v.size());
    return 0;
  } catch (const std::exception& e) { set_err(e.what()); return 1; }
}

double oracle_splitmix_normal(uint64_t seed, int count, double* out) {
  SplitMix64 r{seed};
  for (int i = 0; i < count; ++i) out[i] = r.normal();
  return 0.0;
}

// Courant numbers of a state (proj/src/harness.cpp:216-238)
int oracle_courant(void* h, const double* u, double dt, double* cr_a, double* cr_d) {
  const Problem& P = *static_cast<Problem*>(h);
  const int comps = P.d.kind == 3 ? 4 : 1;
  const CourantNumbers c = courant_numbers(Vec(u, u + P.dim), P.mesh, P.basis, comps, dt, P.d.kappa,
                                           P.d.kind == 3, P.d.gamma);
  *cr_a = c.cr_a;
  *cr_d = c.cr_d;
  return 0;
}

}  // extern "C"
