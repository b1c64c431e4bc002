// ORACLE (test infrastructure): restatement of the reference acceptance
// criteria that print digits (proj/tests/acceptance.cpp:110-527), used to pin
// this oracle against proj/test_output.txt:18-28.
#include <algorithm>
#include <cmath>
#include <cstring>

#include "oracle.hpp"

using namespace oracle;

namespace {

struct RunRow {
  double scale, error, cr_a, cr_d;
  long iters;
  bool ok;
};

Vec discrete_error(const ProblemContext& ctx, const Vec& u, const ProblemContext& ref, const Vec& uref) {
  if (ctx.mesh->dim == 1)
    return l2_error(u, 1, *ctx.mesh, *ctx.basis, [&](double x, double, int) {
      return evaluate_1d(uref, *ref.mesh, *ref.basis, x);
    });
  return l2_error(u, ctx.components, *ctx.mesh, *ctx.basis, [&](double x, double y, int c) {
    return evaluate_2d(uref, ref.components, *ref.mesh, *ref.basis, x, y, c);
  });
}

// proj/src/harness.cpp:388-479 restricted to the pieces the criteria read.
// ref_mode: 0 exact, 1 generate (rk4 ref with ref_k / ref_dt on the same ne)
RunRow run_point(const ExperimentConfig& cfg, const std::string& integ, int k, int ne, double dt,
                 double t_final, int ref_mode, int ref_k, double ref_dt, int comp = 0) {
  ProblemContext ctx = make_problem(cfg, ne, k);
  TimeLoopConfig tl;
  tl.dt = dt;
  tl.t_final = t_final;
  tl.krylov.tol = 1e-12;
  tl.krylov.max_basis = 128;
  tl.krylov.orth_length = 128;
  const CourantNumbers cr = courant_numbers(ctx.u0, *ctx.mesh, *ctx.basis, ctx.components, dt,
                                            ctx.is_euler ? 0.0 : ctx.burgers.kappa, ctx.is_euler,
                                            ctx.euler.gamma);
  const IntegrationResult run = integrate(ctx.split, integrator_from_name(integ), ctx.u0, tl);
  RunRow row{0, NAN, cr.cr_a, cr.cr_d, run.krylov_iterations, run.status == RunStatus::completed};
  row.scale = ctx.mesh->elements.front().hx;
  if (!row.ok) return row;
  if (ref_mode == 0) {
    auto exact = ctx.exact;
    row.error = l2_error(run.u, ctx.components, *ctx.mesh, *ctx.basis, [&](double x, double y, int c) {
                  return exact(x, y, t_final, c);
                })[comp];
  } else {
    ExperimentConfig rc = cfg;
    rc.over_integrate = ctx.burgers.over_integrate ? 1 : 0;
    rc.sigma_adaptive = ctx.burgers.sigma_adaptive;
    ProblemContext rctx = make_problem(rc, ne, ref_k);
    TimeLoopConfig rtl;
    rtl.dt = ref_dt;
    rtl.t_final = t_final;
    const IntegrationResult rr = integrate(rctx.split, IntegratorKind::rk4, rctx.u0, rtl);
    row.error = discrete_error(ctx, run.u, rctx, rr.u)[comp];
  }
  return row;
}

}  // namespace

extern "C" {

// Criterion 2/3 (proj/tests/acceptance.cpp:112-155): burgers-mms, exprb32,
// ne = {20,40,80,160}, dt = 5e-5, t = 0.01; errors[4] vs the exact solution.
int oracle_acc_mms(int k, int entropy_flux, double sigma, double* errors) {
  ExperimentConfig cfg;
  cfg.problem = "burgers-mms";
  cfg.flux = entropy_flux ? "ef" : "lf";
  cfg.sigma = sigma;
  const int nes[4] = {20, 40, 80, 160};
  for (int i = 0; i < 4; ++i) errors[i] = run_point(cfg, "exprb32", k, nes[i], 5e-5, 0.01, 0, 0, 0).error;
  return 0;
}

// Criterion 4 (acceptance.cpp:159-195): burgers-smooth k=4 ne=40 lf, dt sweep
// {0.5,0.25,0.1,0.05,0.01}, reference rk4 k=4 dt=1e-5 on the same mesh.
int oracle_acc_temporal(int integrator /*1 epi2, 2 exprb32*/, double* errors /*5*/) {
  ExperimentConfig cfg;
  cfg.problem = "burgers-smooth";
  cfg.flux = "lf";
  const double dts[5] = {0.5, 0.25, 0.1, 0.05, 0.01};
  // the reference solution is shared across the sweep
  ProblemContext rctx = make_problem(cfg, 40, 4);
  TimeLoopConfig rtl;
  rtl.dt = 1e-5;
  rtl.t_final = 1.0;
  const IntegrationResult rr = integrate(rctx.split, IntegratorKind::rk4, rctx.u0, rtl);
  for (int i = 0; i < 5; ++i) {
    ProblemContext ctx = make_problem(cfg, 40, 4);
    TimeLoopConfig tl;
    tl.dt = dts[i];
    tl.t_final = 1.0;
    tl.krylov.tol = 1e-12;
    const IntegrationResult run =
        integrate(ctx.split, integrator == 1 ? IntegratorKind::epi2 : IntegratorKind::exprb32, ctx.u0, tl);
    errors[i] = run.status == RunStatus::completed ? discrete_error(ctx, run.u, rctx, rr.u)[0] : NAN;
  }
  return 0;
}

// Criterion 5 (acceptance.cpp:199-237): burgers-smooth k=4 ne=40, EF sigma=3e-4.
// out: [cr_d, epi2 completed, epi2 max_abs / initial max, rk2 blew up, rk2 blow_up_step]
int oracle_acc_large_courant(double* out) {
  ExperimentConfig cfg;
  cfg.problem = "burgers-smooth";
  cfg.flux = "ef";
  cfg.sigma = 3e-4;
  ProblemContext ctx = make_problem(cfg, 40, 4);
  TimeLoopConfig tl;
  tl.dt = 0.1;
  tl.t_final = 1.0;
  const double initial_max = max_abs(ctx.u0);
  const IntegrationResult epi2 = integrate(ctx.split, IntegratorKind::epi2, ctx.u0, tl);
  const CourantNumbers cr = courant_numbers(ctx.u0, *ctx.mesh, *ctx.basis, 1, 0.1, ctx.burgers.kappa, false);
  tl.dt = 2e-4;
  const IntegrationResult rk2 = integrate(ctx.split, IntegratorKind::rk2, ctx.u0, tl);
  out[0] = cr.cr_d;
  out[1] = epi2.status == RunStatus::completed ? 1.0 : 0.0;
  out[2] = epi2.max_abs / initial_max;
  out[3] = rk2.status == RunStatus::blew_up ? 1.0 : 0.0;
  out[4] = rk2.blow_up_step;
  return 0;
}

// Criterion 8 (acceptance.cpp:333-355): euler-vortex exprb42 (Roe), ne {256, 1024},
// dt 0.01, t 1; out: rho errors at both resolutions.
int oracle_acc_vortex(int k, double* errors) {
  ExperimentConfig cfg;
  cfg.problem = "euler-vortex";
  errors[0] = run_point(cfg, "exprb42", k, 256, 0.01, 1.0, 0, 0, 0).error;
  errors[1] = run_point(cfg, "exprb42", k, 1024, 0.01, 1.0, 0, 0, 0).error;
  return 0;
}

// Criterion 9 Burgers part (acceptance.cpp:392-416): smooth k=3 ne=20 lf,
// dt {0.4,0.2,0.1,0.05}, rk4 ref k=3 dt 1e-5; returns the last order.
double oracle_acc_burgers_order(int integrator /*0..3*/) {
  static const char* names[] = {"exp_euler", "epi2", "exprb32", "exprb42"};
  ExperimentConfig cfg;
  cfg.problem = "burgers-smooth";
  cfg.flux = "lf";
  ProblemContext rctx = make_problem(cfg, 20, 3);
  TimeLoopConfig rtl;
  rtl.dt = 1e-5;
  rtl.t_final = 1.0;
  const IntegrationResult rr = integrate(rctx.split, IntegratorKind::rk4, rctx.u0, rtl);
  double e[2];
  const double dts[2] = {0.1, 0.05};
  for (int i = 0; i < 2; ++i) {
    ProblemContext ctx = make_problem(cfg, 20, 3);
    TimeLoopConfig tl;
    tl.dt = dts[i];
    tl.t_final = 1.0;
    tl.krylov.tol = 1e-12;
    const IntegrationResult run = integrate(ctx.split, integrator_from_name(names[integrator]), ctx.u0, tl);
    e[i] = discrete_error(ctx, run.u, rctx, rr.u)[0];
  }
  return std::log(e[0] / e[1]) / std::log(2.0);
}

// Criterion 9 ODE part (acceptance.cpp:364-390, proj/tests/test_util.hpp:11-52).
double oracle_acc_ode_order(int integrator /*0..3*/) {
  const double lambda = -10.0, y0 = 0.2, t_final = 1.0;
  SplitProblem prob;
  prob.dim = 1;
  prob.linearize = [lambda](const Vec& ref) {
    const double yt = ref[0];
    SplitOperator op;
    op.dim = 1;
    op.linear = [lambda, yt](const Vec& y) { return Vec{(lambda + 2.0 * yt) * y[0]}; };
    op.nonlinear = [yt](const Vec& y) { return Vec{y[0] * y[0] - 2.0 * yt * y[0]}; };
    return op;
  };
  prob.rhs = [lambda](const Vec& y) { return Vec{lambda * y[0] + y[0] * y[0]}; };
  auto f = [lambda](double y) { return lambda * y + y * y; };
  double y = y0, t = 0.0;
  while (t < t_final - 1e-12) {
    const double h = std::min(1e-6, t_final - t);
    const double k1 = f(y), k2 = f(y + 0.5 * h * k1), k3 = f(y + 0.5 * h * k2), k4 = f(y + h * k3);
    y += h / 6.0 * (k1 + 2 * k2 + 2 * k3 + k4);
    t += h;
  }
  const IntegratorKind kinds[] = {IntegratorKind::exp_euler, IntegratorKind::epi2, IntegratorKind::exprb32,
                                  IntegratorKind::exprb42};
  double e[3];
  const double dts[3] = {0.1, 0.05, 0.025};
  for (int i = 0; i < 3; ++i) {
    TimeLoopConfig cfg;
    cfg.dt = dts[i];
    cfg.t_final = t_final;
    const IntegrationResult r = integrate(prob, kinds[integrator], Vec{y0}, cfg);
    e[i] = std::abs(r.u[0] - y);
  }
  return std::log2(e[1] / e[2]);
}

// Criterion 10 (acceptance.cpp:420-454): exp_euler, dt ~ h, vs rk4 k=6 ne=80 ref.
int oracle_acc_exp_euler_joint(double* errors /*3*/) {
  ExperimentConfig rc;
  rc.problem = "burgers-smooth";
  rc.flux = "lf";
  rc.over_integrate = 1;
  rc.kappa = 0.03;
  ProblemContext rctx = make_problem(rc, 80, 6);
  TimeLoopConfig rtl;
  rtl.dt = 5e-6;
  rtl.t_final = 1.0;
  const IntegrationResult rr = integrate(rctx.split, IntegratorKind::rk4, rctx.u0, rtl);
  const int nes[3] = {10, 20, 40};
  const double dts[3] = {0.2, 0.1, 0.05};
  ExperimentConfig cfg;
  cfg.problem = "burgers-smooth";
  cfg.flux = "lf";
  for (int i = 0; i < 3; ++i) {
    ProblemContext ctx = make_problem(cfg, nes[i], 2);
    TimeLoopConfig tl;
    tl.dt = dts[i];
    tl.t_final = 1.0;
    const IntegrationResult run = integrate(ctx.split, IntegratorKind::exp_euler, ctx.u0, tl);
    errors[i] = discrete_error(ctx, run.u, rctx, rr.u)[0];
  }
  return 0;
}

}  // extern "C"

// ---------------------------------------------------------------- checker helpers for the
// device replays of the acceptance criteria (tests/test_gpu_acceptance.py)
extern "C" {

// make_problem (proj/src/harness.cpp:48-142) for the Burgers problems: u0, the weak
// source load vector (zeros when none) and the effective BurgersConfig.
// out_cfg = {kappa, flux(0 lf/1 ef), sigma, sigma_adaptive, over_integrate}
int oracle_harness_burgers(const char* problem, int ne, int k, const char* flux, double sigma, int sigma_adaptive,
                           int over_integrate, double kappa, double* u0, double* src_weak, double* out_cfg) {
  try {
    ExperimentConfig cfg;
    cfg.problem = problem;
    cfg.flux = flux;
    cfg.sigma = sigma;
    cfg.sigma_adaptive = sigma_adaptive != 0;
    cfg.over_integrate = over_integrate;
    cfg.kappa = kappa;
    ProblemContext ctx = make_problem(cfg, ne, k);
    std::memcpy(u0, ctx.u0.data(), sizeof(double) * ctx.u0.size());
    const BurgersConfig& bc = ctx.burgers;
    const int np = k + 1;
    std::fill(src_weak, src_weak + (size_t)ne * np, 0.0);
    if (bc.source) {
      // proj/src/burgers.cpp:80-92
      const QuadratureRule quad = bc.over_integrate ? gauss_quadrature((3 * k + 2 + 1) / 2) : lgl_quadrature(*ctx.basis);
      const Mat interp = bc.over_integrate ? interpolation_matrix(*ctx.basis, quad.points) : Mat::identity(np);
      const int nq = int(quad.points.size());
      for (int e = 0; e < ne; ++e) {
        const Element& el = ctx.mesh->elements[e];
        const double s = 0.5 * el.hx;
        for (int i = 0; i < np; ++i) {
          double acc = 0.0;
          for (int q = 0; q < nq; ++q)
            acc += (s * interp(q, i)) * (quad.weights[q] * bc.source(el.x0 + 0.5 * (quad.points[q] + 1.0) * el.hx));
          src_weak[(size_t)e * np + i] = acc;
        }
      }
    }
    out_cfg[0] = bc.kappa;
    out_cfg[1] = bc.flux == FluxKind::entropy ? 1.0 : 0.0;
    out_cfg[2] = bc.sigma;
    out_cfg[3] = bc.sigma_adaptive ? 1.0 : 0.0;
    out_cfg[4] = bc.over_integrate ? 1.0 : 0.0;
    return 0;
  } catch (const std::exception&) {
    return 1;
  }
}

// L2 error (component comp) of a harness state against the problem's exact solution at
// time t (burgers-mms, euler-vortex; proj/src/harness.cpp:418-440)
double oracle_l2_error_exact(const char* problem, int ne, int k, const double* u, double t, int comp) {
  ExperimentConfig cfg;
  cfg.problem = problem;
  ProblemContext ctx = make_problem(cfg, ne, k);
  auto exact = ctx.exact;
  return l2_error(Vec(u, u + ctx.u0.size()), ctx.components, *ctx.mesh, *ctx.basis,
                  [&](double x, double y, int c) { return exact(x, y, t, c); })[comp];
}

// u0 of any harness problem (make_problem, proj/src/harness.cpp:48-142); returns the
// dimension, writes u0 when out is non-null
long oracle_harness_u0(const char* problem, int ne, int k, double* out) {
  try {
    ExperimentConfig cfg;
    cfg.problem = problem;
    ProblemContext ctx = make_problem(cfg, ne, k);
    if (out) std::memcpy(out, ctx.u0.data(), sizeof(double) * ctx.u0.size());
    return (long)ctx.u0.size();
  } catch (const std::exception&) {
    return -1;
  }
}

// rk4 reference of a Burgers harness problem (generate_reference, proj/src/harness.cpp:364-386)
int oracle_rk4_reference(const char* problem, int ne, int k, const char* flux, int over_integrate, double dt,
                         double t_final, double* u_out) {
  ExperimentConfig cfg;
  cfg.problem = problem;
  cfg.flux = flux;
  cfg.over_integrate = over_integrate;
  ProblemContext ctx = make_problem(cfg, ne, k);
  TimeLoopConfig tl;
  tl.dt = dt;
  tl.t_final = t_final;
  const IntegrationResult r = integrate(ctx.split, IntegratorKind::rk4, ctx.u0, tl);
  std::memcpy(u_out, r.u.data(), sizeof(double) * r.u.size());
  return r.status == RunStatus::completed ? 0 : 1;
}

// discrete L2 error (proj/src/harness.cpp:190-199) of u (ne, k) against uref (ref_ne, ref_k)
// on the harness mesh of `problem`
double oracle_l2_error_discrete(const char* problem, int ne, int k, const double* u, int ref_ne, int ref_k,
                                const double* uref) {
  ExperimentConfig cfg;
  cfg.problem = problem;
  ProblemContext a = make_problem(cfg, ne, k);
  ProblemContext b = make_problem(cfg, ref_ne, ref_k);
  const Vec ur(uref, uref + b.u0.size());
  return l2_error(Vec(u, u + a.u0.size()), 1, *a.mesh, *a.basis,
                  [&](double x, double, int) { return evaluate_1d(ur, *b.mesh, *b.basis, x); })[0];
}

}  // extern "C"

namespace oracle {
double mms_source(double x, double kappa);
}  // namespace oracle

// the burgers-mms forcing s(x) = u u_x - kappa u_xx (proj/src/harness.cpp:97-104)
extern "C" double oracle_mms_source(double x, double kappa) { return oracle::mms_source(x, kappa); }
