// ORACLE (test infrastructure): time integrators and the harness subset.
// Restates proj/src/integrators.cpp and proj/src/harness.cpp:15-238.
#include <algorithm>
#include <cmath>
#include <limits>

#include "oracle.hpp"

namespace oracle {

// proj/src/integrators.cpp:20-30
IntegratorKind integrator_from_name(const std::string& name) {
  if (name == "exp_euler") return IntegratorKind::exp_euler;
  if (name == "epi2") return IntegratorKind::epi2;
  if (name == "exprb32") return IntegratorKind::exprb32;
  if (name == "exprb42") return IntegratorKind::exprb42;
  if (name == "rk2") return IntegratorKind::rk2;
  if (name == "rk3") return IntegratorKind::rk3;
  if (name == "rk4") return IntegratorKind::rk4;
  throw std::invalid_argument("unknown integrator '" + name + "'");
}

namespace {
// proj/src/integrators.cpp:46-57
PhiCombinationResult combine(const SplitOperator& op, std::vector<Vec> b, double dt,
                             const KrylovSettings& ks) {
  PhiCombinationProblem prob;
  prob.op = op.linear;
  prob.b = std::move(b);
  prob.dt = dt;
  prob.tol = ks.tol;
  prob.max_basis = ks.max_basis;
  prob.orth_length = ks.orth_length;
  return phi_combination(prob);
}
void add_stats(KrylovStats* s, const KrylovStats& r) {
  if (!s) return;
  s->iterations += r.iterations;
  s->substeps += r.substeps;
}
}  // namespace

// proj/src/integrators.cpp:67-74
Vec step_exp_euler(const SplitOperator& op, const Vec& u, double dt, const KrylovSettings& ks,
                   KrylovStats* stats) {
  auto res = combine(op, {u, op.nonlinear(u)}, dt, ks);
  add_stats(stats, res.stats);
  return res.value;
}

// proj/src/integrators.cpp:76-83
Vec step_epi2(const SplitOperator& op, const Vec& u, double dt, const KrylovSettings& ks,
              KrylovStats* stats) {
  const Vec r = add(op.linear(u), op.nonlinear(u));
  auto res = combine(op, {Vec(u.size(), 0.0), r}, dt, ks);
  add_stats(stats, res.stats);
  return add(u, res.value);
}

// proj/src/integrators.cpp:85-98
Vec step_exprb32(const SplitOperator& op, const Vec& u, double dt, const KrylovSettings& ks,
                 KrylovStats* stats) {
  const Vec zero(u.size(), 0.0);
  const Vec nu = op.nonlinear(u);
  const Vec r = add(op.linear(u), nu);
  auto stage = combine(op, {zero, r}, dt, ks);
  add_stats(stats, stage.stats);
  const Vec d2 = axpby(1.0, op.nonlinear(add(u, stage.value)), -1.0, nu);
  auto full = combine(op, {zero, r, zero, scale(2.0 / (dt * dt), d2)}, dt, ks);
  add_stats(stats, full.stats);
  return add(u, full.value);
}

// proj/src/integrators.cpp:100-113
Vec step_exprb42(const SplitOperator& op, const Vec& u, double dt, const KrylovSettings& ks,
                 KrylovStats* stats) {
  const Vec zero(u.size(), 0.0);
  const Vec nu = op.nonlinear(u);
  const Vec r = add(op.linear(u), nu);
  auto stage = combine(op, {zero, r}, 0.75 * dt, ks);
  add_stats(stats, stage.stats);
  const Vec d2 = axpby(1.0, op.nonlinear(add(u, stage.value)), -1.0, nu);
  auto full = combine(op, {zero, r, zero, scale(32.0 / 9.0 / (dt * dt), d2)}, dt, ks);
  add_stats(stats, full.stats);
  return add(u, full.value);
}

// proj/src/integrators.cpp:115-138
Vec step_rk(IntegratorKind kind, const RhsAction& rhs, const Vec& u, double dt) {
  switch (kind) {
    case IntegratorKind::rk2: {
      const Vec k1 = rhs(u);
      const Vec k2 = rhs(axpby(1.0, u, dt, k1));
      Vec out(u.size());
      for (size_t i = 0; i < u.size(); ++i) out[i] = u[i] + 0.5 * dt * (k1[i] + k2[i]);
      return out;
    }
    case IntegratorKind::rk3: {
      const Vec u1 = axpby(1.0, u, dt, rhs(u));
      const Vec r1 = rhs(u1);
      Vec u2(u.size());
      for (size_t i = 0; i < u.size(); ++i) u2[i] = 0.75 * u[i] + 0.25 * (u1[i] + dt * r1[i]);
      const Vec r2 = rhs(u2);
      Vec out(u.size());
      for (size_t i = 0; i < u.size(); ++i)
        out[i] = (1.0 / 3.0) * u[i] + (2.0 / 3.0) * (u2[i] + dt * r2[i]);
      return out;
    }
    case IntegratorKind::rk4: {
      const Vec k1 = rhs(u);
      const Vec k2 = rhs(axpby(1.0, u, 0.5 * dt, k1));
      const Vec k3 = rhs(axpby(1.0, u, 0.5 * dt, k2));
      const Vec k4 = rhs(axpby(1.0, u, dt, k3));
      Vec out(u.size());
      for (size_t i = 0; i < u.size(); ++i)
        out[i] = u[i] + (dt / 6.0) * (k1[i] + 2.0 * k2[i] + 2.0 * k3[i] + k4[i]);
      return out;
    }
    default:
      throw std::invalid_argument("step_rk: not an RK kind");
  }
}

// proj/src/integrators.cpp:140-201
IntegrationResult integrate(const SplitProblem& problem, IntegratorKind kind, Vec u0,
                            const TimeLoopConfig& cfg) {
  if (!(cfg.dt > 0.0)) throw std::invalid_argument("integrate: dt must be positive");
  if (cfg.t_final < cfg.dt) throw std::invalid_argument("integrate: t_final must be at least dt");
  IntegrationResult res;
  res.u = std::move(u0);
  res.max_abs = res.u.empty() ? 0.0 : max_abs(res.u);
  const double blow_up_scale = 1e10 * (1.0 + res.max_abs);
  SplitOperator frozen;
  if (kind == IntegratorKind::exp_euler) frozen = problem.linearize(res.u);
  KrylovStats stats;
  const double t_end = cfg.t_final * (1.0 - 1e-14);
  while (res.t < t_end) {
    const double dt = std::min(cfg.dt, cfg.t_final - res.t);
    bool failed = false;
    try {
      switch (kind) {
        case IntegratorKind::exp_euler:
          res.u = step_exp_euler(frozen, res.u, dt, cfg.krylov, &stats);
          break;
        case IntegratorKind::epi2:
          res.u = step_epi2(problem.linearize(res.u), res.u, dt, cfg.krylov, &stats);
          break;
        case IntegratorKind::exprb32:
          res.u = step_exprb32(problem.linearize(res.u), res.u, dt, cfg.krylov, &stats);
          break;
        case IntegratorKind::exprb42:
          res.u = step_exprb42(problem.linearize(res.u), res.u, dt, cfg.krylov, &stats);
          break;
        default:
          res.u = step_rk(kind, problem.rhs, res.u, dt);
      }
    } catch (const KrylovError&) {
      failed = true;
    } catch (const std::domain_error&) {
      failed = true;
    }
    res.t += dt;
    ++res.steps;
    const double amax = all_finite(res.u) ? max_abs(res.u) : std::numeric_limits<double>::infinity();
    if (failed || !std::isfinite(amax) || amax > blow_up_scale) {
      res.status = RunStatus::blew_up;
      res.blow_up_step = res.steps;
      break;
    }
    res.max_abs = std::max(res.max_abs, amax);
    // proj/src/integrators.cpp:195-196
    if (cfg.snapshot_every > 0 && res.steps % cfg.snapshot_every == 0) res.snapshots.emplace_back(res.t, res.u);
    if (cfg.on_step) cfg.on_step(res.steps, res.t, amax, stats.iterations);
  }
  res.krylov_iterations = stats.iterations;
  return res;
}

// ---------------------------------------------------------------- harness subset
namespace {
// proj/src/harness.cpp:16-32
double mms_solution(double x) { return std::sin(x * x) * x * (x - 1.0); }
double mms_solution_dx(double x) {
  return 2.0 * x * std::cos(x * x) * (x * x - x) + std::sin(x * x) * (2.0 * x - 1.0);
}
double mms_solution_dxx(double x) {
  const double s = std::sin(x * x), c = std::cos(x * x);
  return 2.0 * c * (x * x - x) - 4.0 * x * x * s * (x * x - x) + 4.0 * x * c * (2.0 * x - 1.0) + 2.0 * s;
}
}  // namespace
double mms_source(double x, double kappa) { return mms_solution(x) * mms_solution_dx(x) - kappa * mms_solution_dxx(x); }
namespace {
double smooth_initial(double x) {
  const double s = std::sin(2.0 * M_PI * x);
  return s * s * s * std::pow(1.0 - x, 1.5);
}
FluxKind flux_from_name(const std::string& n) {
  if (n == "lf") return FluxKind::lax_friedrichs;
  if (n == "ef") return FluxKind::entropy;
  throw std::invalid_argument("unknown flux '" + n + "' (use lf or ef)");
}
}  // namespace

// proj/src/harness.cpp:48-142
ProblemContext make_problem(const ExperimentConfig& cfg, int ne, int k) {
  ProblemContext ctx;
  ctx.basis = std::make_shared<NodalBasis>(lgl_basis(k));
  const QuadratureRule proj_quad = gauss_quadrature(k + 2);
  if (cfg.problem == "euler-vortex") {
    const int nx = int(std::lround(std::sqrt(double(ne))));
    if (nx * nx != ne) throw std::invalid_argument("euler-vortex: ne must be a perfect square");
    ctx.mesh = std::make_shared<Mesh>(build_quad_mesh(0, 10, -5, 5, nx, nx, BoundaryKind::periodic));
    ctx.is_euler = true;
    ctx.components = 4;
    ctx.euler = EulerConfig{};
    if (cfg.flux == "lf") ctx.euler.flux = EulerFluxKind::lax_friedrichs;
    else if (!cfg.flux.empty() && cfg.flux != "roe")
      throw std::invalid_argument("euler-vortex flux must be roe or lf");
    const EulerConfig ecfg = ctx.euler;
    ctx.exact = [ecfg](double x, double y, double t, int c) { return isentropic_vortex(x, y, t, ecfg)[c]; };
    ctx.u0 = l2_project_system_2d(
        [&ecfg](double x, double y, double* out) {
          const State4 q = isentropic_vortex(x, y, 0.0, ecfg);
          for (int c = 0; c < 4; ++c) out[c] = q[c];
        },
        4, *ctx.mesh, *ctx.basis, proj_quad);
    auto mesh = ctx.mesh;
    auto basis = ctx.basis;
    ctx.split.dim = long(ctx.u0.size());
    ctx.split.linearize = [mesh, basis, ecfg](const Vec& ref) {
      auto op = std::make_shared<EulerOperator>(*mesh, *basis, ecfg, ref);
      SplitOperator s;
      s.dim = op->dim();
      s.linear = [op](const Vec& q) { return op->apply_linear(q); };
      s.nonlinear = [op](const Vec& q) { return op->apply_nonlinear(q); };
      return s;
    };
    ctx.split.rhs = [mesh, basis, ecfg](const Vec& q) { return euler_full_rhs(*mesh, *basis, ecfg, q); };
    return ctx;
  }
  BurgersConfig bc;
  bc.flux = flux_from_name(cfg.flux.empty() ? "lf" : cfg.flux);
  bc.sigma = cfg.sigma;
  bc.sigma_adaptive = cfg.sigma_adaptive;
  bc.over_integrate = cfg.over_integrate < 0 ? true : cfg.over_integrate != 0;
  std::function<double(double)> initial;
  if (cfg.problem == "burgers-mms") {
    bc.kappa = cfg.kappa >= 0.0 ? cfg.kappa : 0.03;
    const double kap = bc.kappa;
    bc.source = [kap](double x) {
      return mms_solution(x) * mms_solution_dx(x) - kap * mms_solution_dxx(x);
    };
    initial = mms_solution;
    ctx.exact = [](double x, double, double, int) { return mms_solution(x); };
  } else if (cfg.problem == "burgers-smooth") {
    bc.kappa = cfg.kappa >= 0.0 ? cfg.kappa : 0.03;
    initial = smooth_initial;
  } else if (cfg.problem == "burgers-shock") {
    bc.kappa = cfg.kappa >= 0.0 ? cfg.kappa : 0.002;
    if (ne % 2 != 0) throw std::invalid_argument("burgers-shock: ne must be even");
    if (bc.flux == FluxKind::entropy && bc.sigma == 0.0 && !bc.sigma_adaptive) bc.sigma_adaptive = true;
    initial = [](double x) { return std::sin(2.0 * M_PI * x); };
  } else {
    throw std::invalid_argument("unknown problem '" + cfg.problem + "'");
  }
  ctx.mesh = std::make_shared<Mesh>(build_interval_mesh(0.0, 1.0, ne, BoundaryKind::dirichlet_zero));
  ctx.components = 1;
  ctx.burgers = bc;
  ctx.u0 = l2_project_1d(initial, *ctx.mesh, *ctx.basis, proj_quad);
  auto mesh = ctx.mesh;
  auto basis = ctx.basis;
  ctx.split.dim = long(ctx.u0.size());
  ctx.split.linearize = [mesh, basis, bc](const Vec& ref) {
    auto op = std::make_shared<BurgersOperator>(*mesh, *basis, bc, ref);
    SplitOperator s;
    s.dim = op->dim();
    s.linear = [op](const Vec& u) { return op->apply_linear(u); };
    s.nonlinear = [op](const Vec& u) { return op->apply_nonlinear(u); };
    return s;
  };
  auto full_op = std::make_shared<BurgersOperator>(*mesh, *basis, bc, Vec(ctx.u0.size(), 0.0));
  ctx.split.rhs = [mesh, basis, full_op](const Vec& u) { return full_op->full_rhs(u); };
  return ctx;
}

// proj/src/harness.cpp:144-188
Vec l2_error(const Vec& u, int components, const Mesh& mesh, const NodalBasis& b,
             const std::function<double(double, double, int)>& ref) {
  const QuadratureRule quad = gauss_quadrature(b.order + 2);
  const Mat iq = interpolation_matrix(b, quad.points);
  const int nq = int(quad.points.size());
  const int np1 = b.num_nodes();
  Vec err2(components, 0.0);
  if (mesh.dim == 1) {
    for (int e = 0; e < mesh.num_elements(); ++e) {
      const Element& el = mesh.elements[e];
      for (int c = 0; c < components; ++c) {
        const double* blk = &u[(size_t(e) * components + c) * np1];
        for (int q = 0; q < nq; ++q) {
          double uq = 0.0;
          for (int j = 0; j < np1; ++j) uq += iq(q, j) * blk[j];
          const double x = el.x0 + 0.5 * (quad.points[q] + 1.0) * el.hx;
          const double d = uq - ref(x, 0.0, c);
          err2[c] += 0.5 * el.hx * quad.weights[q] * d * d;
        }
      }
    }
  } else {
    const int np = np1 * np1;
    for (int e = 0; e < mesh.num_elements(); ++e) {
      const Element& el = mesh.elements[e];
      for (int c = 0; c < components; ++c) {
        const double* blk = &u[(size_t(e) * components + c) * np];
        // uq = iq * nodal * iq^T with nodal(i,j) = blk[j*np1+i]
        Mat t(nq, np1);
        for (int qx = 0; qx < nq; ++qx)
          for (int j = 0; j < np1; ++j) {
            double s = 0.0;
            for (int i = 0; i < np1; ++i) s += iq(qx, i) * blk[j * np1 + i];
            t(qx, j) = s;
          }
        for (int qy = 0; qy < nq; ++qy) {
          const double y = el.y0 + 0.5 * (quad.points[qy] + 1.0) * el.hy;
          for (int qx = 0; qx < nq; ++qx) {
            double uq = 0.0;
            for (int j = 0; j < np1; ++j) uq += t(qx, j) * iq(qy, j);
            const double x = el.x0 + 0.5 * (quad.points[qx] + 1.0) * el.hx;
            const double d = uq - ref(x, y, c);
            err2[c] += 0.25 * el.hx * el.hy * quad.weights[qx] * quad.weights[qy] * d * d;
          }
        }
      }
    }
  }
  for (auto& v : err2) v = std::sqrt(v);
  return err2;
}

// proj/src/harness.cpp:216-238
CourantNumbers courant_numbers(const Vec& u, const Mesh& mesh, const NodalBasis& b, int components,
                               double dt, double kappa, bool euler, double gamma) {
  const double dx = min_node_spacing(mesh, b);
  double c = 0.0;
  const int np = nodes_per_element(mesh, b);
  for (int e = 0; e < mesh.num_elements(); ++e)
    for (int n = 0; n < np; ++n) {
      if (euler) {
        State4 q;
        for (int comp = 0; comp < 4; ++comp) q[comp] = u[(size_t(e) * components + comp) * np + n];
        const EulerPrimitives pr = primitives(q, gamma);
        c = std::max(c, std::max(std::abs(pr.u), std::abs(pr.v)) + pr.a);
      } else {
        c = std::max(c, std::abs(u[size_t(e) * np + n]));
      }
    }
  CourantNumbers cr;
  cr.cr_a = c * dt / dx;
  cr.cr_d = kappa * dt / (dx * dx);
  return cr;
}

}  // namespace oracle
