// Minimal C++ user of the drop-in API (include/expdg_b200.hpp): the reference's
// harness flow make_problem -> integrate (proj/src/harness.cpp:400-419) for the
// C4 physics on a small mesh.  `--host-only` exercises the host setup entry
// points only (no GPU needed).
#include <cmath>
#include <cstdio>
#include <cstring>
#include <vector>

#include "expdg_b200.hpp"

int main(int argc, char** argv) {
  using namespace expdg::b200;
  const int order = 4, nx = 16;
  const NodalBasis b = lgl_basis(order);
  std::vector<double> u0((size_t)nx * nx * (order + 1) * (order + 1) * 4);
  check(expdg_initial_condition(4, nx, order, 20201106ULL, 1e-6, u0.data()));
  std::printf("lgl nodes[1] = %.17g, u0[0] = %.17g\n", b.nodes[1], u0[0]);
  if (argc > 1 && std::strcmp(argv[1], "--host-only") == 0) return 0;

  Context ctx(0);
  expdg_op_desc d{};
  d.kind = EXPDG_EULER2D;
  d.order = order;
  d.nx = d.ny = nx;
  d.nz = 1;
  d.x0 = 0; d.x1 = 10; d.y0 = 0; d.y1 = 10; d.z0 = 0; d.z1 = 1;
  d.periodic = 1;
  d.gamma = 1.4;
  d.euler_flux = 1;
  SplitOperator op(ctx, d);
  TimeLoopConfig cfg;
  cfg.dt = 0.05;
  cfg.t_final = 0.15;
  cfg.krylov.tol = 1e-10;
  cfg.krylov.max_basis = 40;
  cfg.krylov.orth_length = 40;
  cfg.snapshot_every = 2;
  cfg.on_step = [](int s, double t, double amax, long it) {
    std::printf("step %d t=%.3f max|u|=%.6f krylov=%ld\n", s, t, amax, it);
  };
  const IntegrationResult r = integrate(ctx, op, IntegratorKind::epi2, u0, cfg);
  std::printf("status=%s steps=%d t=%.3f krylov=%ld max_abs=%.6f snapshots=%zu\n",
              r.status == RunStatus::completed ? "completed" : "blew_up", r.steps, r.t, r.krylov_iterations,
              r.max_abs, r.snapshots.size());
  return r.status == RunStatus::completed ? 0 : 1;
}
