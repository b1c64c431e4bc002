// expdg_b200.hpp — header-only C++ mirror of the reference `expdg` hot-path API
// (/root/reference/proj/include/expdg/{split_operator,phi,integrators}.hpp) on
// top of the C ABI in expdg_b200.h.  Same names, argument meaning and
// exception types as the reference; vectors are std::vector<double> on the
// host (the reference uses Eigen::VectorXd, absent in this image) or raw device
// pointers.
//
//   reference                                         here
//   ------------------------------------------------  -----------------------------------------
//   burgers_split_operator(mesh, basis, cfg, u~)      SplitOperator(ctx, desc).linearize(u~)
//   euler_split_operator(...)   (proj/src/euler.cpp:390-401)
//   SplitOperator::linear / nonlinear                 SplitOperator::linear / nonlinear
//   phi_combination(PhiCombinationProblem)            phi_combination(ctx, op, b, dt, settings)
//   step_epi2(op, u, dt, ks, stats)                   step_epi2(ctx, op, u, dt, ks, stats)
//   integrate(problem, kind, u0, TimeLoopConfig)      integrate(ctx, op, kind, u0, TimeLoopConfig)
//   user LinearAction / SplitProblem                  SplitOperator(ctx, n, DeviceSplitProblem{...})
//   krylov_build(op, seed, m, orth_length)            krylov_build(ctx, op, seed_dev, m, orth_length)
//   KrylovError{last_estimate}                        KrylovError{last_estimate}
//   std::invalid_argument / std::domain_error         same types
#pragma once

#include <cstddef>
#include <stdexcept>
#include <string>
#include <array>
#include <functional>
#include <utility>
#include <vector>

#include "expdg_b200.h"

namespace expdg {
namespace b200 {

// proj/include/expdg/phi.hpp:61-66
class KrylovError : public std::runtime_error {
 public:
  KrylovError(const std::string& what, double estimate) : std::runtime_error(what), last_estimate(estimate) {}
  double last_estimate;
};

class DeviceError : public std::runtime_error {
 public:
  using std::runtime_error::runtime_error;
};

inline void check(int rc, double estimate = 0.0) {
  if (rc == EXPDG_OK) return;
  const std::string msg = expdg_last_error();
  switch (rc) {
    case EXPDG_E_INVALID: throw std::invalid_argument(msg);
    case EXPDG_E_DOMAIN: throw std::domain_error(msg);
    case EXPDG_E_KRYLOV: throw KrylovError(msg, estimate);
    case EXPDG_E_UNSUPPORTED: throw std::invalid_argument("unsupported on the device path: " + msg);
    case EXPDG_E_COMM: throw DeviceError("communicator: " + msg);
    default: throw DeviceError(msg);
  }
}

// proj/include/expdg/phi.hpp:25-28
struct KrylovStats {
  long iterations = 0;
  int substeps = 0;
};

// proj/include/expdg/integrators.hpp:20-24
struct KrylovSettings {
  double tol = 1e-12;
  int max_basis = 128;
  int orth_length = 128;
};

enum class IntegratorKind { exp_euler, epi2, exprb32, exprb42 };
enum class RunStatus { completed, blew_up };

// proj/include/expdg/integrators.hpp:58-63.  on_step runs per completed step, in step order,
// as each step finishes on the device (a stream-ordered host function: no CUDA calls in it)
struct TimeLoopConfig {
  double dt = 0.1;
  double t_final = 1.0;
  KrylovSettings krylov;
  int snapshot_every = 0;  // 0: keep no intermediate states
  std::function<void(int, double, double, long)> on_step;
  bool device_control = true;  // CUDA-graph WHILE-node controller (no host round-trip)
};

// proj/include/expdg/integrators.hpp:66-74
struct IntegrationResult {
  std::vector<double> u;
  double t = 0.0;
  RunStatus status = RunStatus::completed;
  int steps = 0;
  long krylov_iterations = 0;
  int blow_up_step = -1;
  double max_abs = 0.0;
  std::vector<std::pair<double, std::vector<double>>> snapshots;
};

// proj/include/expdg/phi.hpp:30-36 (basis on the host, n x (m+1) column-major)
struct KrylovFactorization {
  std::vector<double> basis;
  std::vector<double> hessenberg;  // (m+1) x m row-major
  double seed_norm = 0;
  int m = 0;
  bool invariant_subspace = false;
};

// A user LinearAction / SplitProblem on device vectors (proj/include/expdg/phi.hpp:11,
// proj/include/expdg/integrators.hpp:48-52): linear / nonlinear act on the operator frozen by
// the last linearize(ref).  Callables may throw std::domain_error / std::invalid_argument like the
// reference's operators.  graph_safe: they only enqueue work on `stream` (see expdg_user_op_fns).
struct DeviceSplitProblem {
  std::function<void(const double* x_dev, double* y_dev, void* stream)> linear;
  std::function<void(const double* x_dev, double* y_dev, void* stream)> nonlinear;  // empty: N = 0
  std::function<void(const double* ref_dev, void* stream)> linearize;                // empty: L fixed
  bool graph_safe = false;
};

namespace detail {
template <class F>
inline int guarded(F&& f) {
  try {
    f();
    return EXPDG_OK;
  } catch (const std::domain_error&) {
    return EXPDG_E_DOMAIN;
  } catch (const std::invalid_argument&) {
    return EXPDG_E_INVALID;
  } catch (...) {
    return EXPDG_E_CUDA;
  }
}
inline int user_linear(const double* x, double* y, void* s, void* u) {
  return guarded([&] { static_cast<DeviceSplitProblem*>(u)->linear(x, y, s); });
}
inline int user_nonlinear(const double* x, double* y, void* s, void* u) {
  return guarded([&] { static_cast<DeviceSplitProblem*>(u)->nonlinear(x, y, s); });
}
inline int user_linearize(const double* r, void* s, void* u) {
  return guarded([&] { static_cast<DeviceSplitProblem*>(u)->linearize(r, s); });
}
}  // namespace detail

class Context {
 public:
  explicit Context(int device = 0) { check(expdg_ctx_create(device, &h_)); }
  ~Context() { expdg_ctx_destroy(h_); }
  Context(const Context&) = delete;
  Context& operator=(const Context&) = delete;
  expdg_ctx* get() const { return h_; }
  void synchronize() { check(expdg_ctx_synchronize(h_)); }
  // multi-GPU slab partition (one process per GPU): collective over `size` ranks
  Context& attach_nccl(const std::array<unsigned char, 128>& id, int rank, int size) {
    check(expdg_ctx_attach_nccl(h_, id.data(), rank, size));
    return *this;
  }
  std::pair<int, int> comm() const {
    int r = 0, n = 1;
    check(expdg_ctx_comm(h_, &r, &n));
    return {r, n};
  }

 private:
  expdg_ctx* h_ = nullptr;
};

// rank 0 creates the id and broadcasts it (MPI, sockets, torch.distributed ...)
inline std::array<unsigned char, 128> nccl_unique_id() {
  std::array<unsigned char, 128> id{};
  check(expdg_nccl_unique_id(id.data()));
  return id;
}

// The split operator (proj/include/expdg/split_operator.hpp:12-20), frozen at
// the state passed to linearize (device pointer).  linear/nonlinear act on
// device pointers; the host-vector overloads copy in and out.
class SplitOperator {
 public:
  SplitOperator(Context& ctx, const expdg_op_desc& desc) : ctx_(&ctx) { check(expdg_op_create(ctx.get(), &desc, &h_)); }
  SplitOperator(Context& ctx, int n, const double* dense_rowmajor) : ctx_(&ctx) {
    check(expdg_dense_op_create(ctx.get(), n, dense_rowmajor, &h_));
  }
  // a user LinearAction / SplitProblem (kept alive by this object)
  SplitOperator(Context& ctx, long long n, DeviceSplitProblem problem)
      : ctx_(&ctx), user_(new DeviceSplitProblem(std::move(problem))) {
    expdg_user_op_fns f{};
    f.apply_linear = detail::user_linear;
    f.apply_nonlinear = user_->nonlinear ? detail::user_nonlinear : nullptr;
    f.linearize = user_->linearize ? detail::user_linearize : nullptr;
    f.graph_safe = user_->graph_safe ? 1 : 0;
    check(expdg_user_op_create(ctx.get(), n, &f, user_, &h_));
  }
  ~SplitOperator() {
    expdg_op_destroy(h_);
    delete user_;
  }
  SplitOperator(const SplitOperator&) = delete;
  SplitOperator& operator=(const SplitOperator&) = delete;

  long long dim() const { return expdg_op_dim(h_); }
  expdg_op* get() const { return h_; }
  Context& context() const { return *ctx_; }
  SplitOperator& linearize(const double* ref_dev) {
    check(expdg_op_linearize(h_, ref_dev));
    return *this;
  }
  // BurgersConfig::source (proj/include/expdg/burgers.hpp:22), as a weak load already on the
  // device or as the function itself (evaluated on the operator's quadrature).
  SplitOperator& set_source(const double* weak_source_dev) {
    check(expdg_op_set_source(h_, weak_source_dev));
    return *this;
  }
  SplitOperator& set_source(const std::function<double(double)>& s) {
    auto tramp = [](double x, void* u) { return (*static_cast<const std::function<double(double)>*>(u))(x); };
    check(expdg_op_set_source_fn(h_, tramp, const_cast<std::function<double(double)>*>(&s)));
    return *this;
  }
  void linear(const double* x_dev, double* y_dev, void* stream = nullptr) const {
    check(expdg_op_apply_linear(h_, x_dev, y_dev, stream));
  }
  void nonlinear(const double* x_dev, double* y_dev, void* stream = nullptr) const {
    check(expdg_op_apply_nonlinear(h_, x_dev, y_dev, stream));
  }
  void full_rhs(const double* x_dev, double* y_dev, void* stream = nullptr) const {
    check(expdg_op_full_rhs(h_, x_dev, y_dev, stream));
  }


 private:
  Context* ctx_;
  expdg_op* h_ = nullptr;
  DeviceSplitProblem* user_ = nullptr;
};

// proj/src/phi.cpp:115-130 on the device engine
inline KrylovFactorization krylov_build(Context& ctx, SplitOperator& op, const double* seed_dev, int m,
                                        int orth_length, double* basis_dev = nullptr) {
  KrylovFactorization f;
  std::vector<double> h((size_t)(m + 1) * m);
  int mo = 0, inv = 0;
  check(expdg_krylov_build(ctx.get(), op.get(), seed_dev, m, orth_length, basis_dev, h.data(), &f.seed_norm, &mo,
                           &inv));
  f.m = mo;
  f.invariant_subspace = inv != 0;
  h.resize((size_t)(mo + 1) * mo);
  f.hessenberg = std::move(h);
  return f;
}

// proj/src/phi.cpp:133-260: out = sum_i dt^i phi_i(dt L) b_i (device pointers, b[i] may be null)
inline KrylovStats phi_combination(Context& ctx, SplitOperator& op, const std::vector<const double*>& b_dev,
                                   double dt, const KrylovSettings& ks, double* out_dev, int initial_basis = 16,
                                   int max_substeps = 40) {
  if (b_dev.empty()) throw std::invalid_argument("phi_combination: empty b list");
  expdg_krylov_cfg c{ks.tol, ks.max_basis, ks.orth_length, initial_basis, max_substeps};
  expdg_krylov_stats s{};
  const int rc = expdg_phi_combination(ctx.get(), op.get(), b_dev.data(), (int)b_dev.size() - 1, dt, &c, out_dev, &s);
  check(rc, s.last_estimate);
  return KrylovStats{(long)s.iterations, s.substeps};
}

// proj/src/integrators.cpp:76-83 (u updated in place on the device)
inline void step_epi2(Context& ctx, SplitOperator& op, double* u_dev, double dt, const KrylovSettings& ks,
                      KrylovStats* stats = nullptr) {
  expdg_krylov_cfg c{ks.tol, ks.max_basis, ks.orth_length, 0, 0};
  expdg_krylov_stats s{};
  const int rc = expdg_step_epi2(ctx.get(), op.get(), u_dev, dt, &c, &s);
  check(rc, s.last_estimate);
  if (stats) {
    stats->iterations += (long)s.iterations;
    stats->substeps += s.substeps;
  }
}

// proj/src/integrators.cpp:140-201 from a HOST initial state (copied in/out).
inline IntegrationResult integrate(Context& ctx, SplitOperator& op, IntegratorKind kind, std::vector<double> u0,
                                   const TimeLoopConfig& cfg) {
  expdg_time_cfg t{};
  t.integrator = kind == IntegratorKind::epi2      ? EXPDG_EPI2
                 : kind == IntegratorKind::exprb32 ? EXPDG_EXPRB32
                 : kind == IntegratorKind::exprb42 ? EXPDG_EXPRB42
                                                   : EXPDG_EXP_EULER;
  t.dt = cfg.dt;
  t.t_final = cfg.t_final;
  t.krylov = expdg_krylov_cfg{cfg.krylov.tol, cfg.krylov.max_basis, cfg.krylov.orth_length, 0, 0};
  t.use_graph = cfg.device_control ? 1 : 0;
  const int cap = (int)(cfg.t_final / cfg.dt + 2.5);
  std::vector<long long> iters(cap > 0 ? cap : 1);
  std::vector<double> amax(cap > 0 ? cap : 1);
  const size_t n = u0.size();
  const int scap = cfg.snapshot_every > 0 ? cap / cfg.snapshot_every : 0;
  std::vector<double> snaps((size_t)scap * n), snap_t(scap);
  t.snapshot_every = cfg.snapshot_every;
  t.snapshot_cap = scap;
  t.snapshots = scap ? snaps.data() : nullptr;
  t.snapshot_times = scap ? snap_t.data() : nullptr;
  if (cfg.on_step) {
    t.on_step = [](int s, double tt, double a, long long it, void* u) {
      (*static_cast<const std::function<void(int, double, double, long)>*>(u))(s, tt, a, (long)it);
    };
    t.on_step_user = const_cast<std::function<void(int, double, double, long)>*>(&cfg.on_step);
  }
  expdg_integration_result r{};
  check(expdg_integrate_host(ctx.get(), op.get(), u0.data(), &t, &r, iters.data(), amax.data(), cap));
  IntegrationResult out;
  out.u = std::move(u0);
  out.t = r.t;
  out.status = r.status == 0 ? RunStatus::completed : RunStatus::blew_up;
  out.steps = r.steps;
  out.krylov_iterations = (long)r.krylov_iterations;
  out.blow_up_step = r.blow_up_step;
  out.max_abs = r.max_abs;
  for (int k = 0; k < r.snapshots && k < scap; ++k)
    out.snapshots.emplace_back(snap_t[k], std::vector<double>(snaps.begin() + (size_t)k * n,
                                                              snaps.begin() + (size_t)(k + 1) * n));
  return out;
}

// proj/src/basis.cpp:35-85
struct NodalBasis {
  int order = 0;
  std::vector<double> nodes, weights, diff_matrix;  // diff row-major
};
inline NodalBasis lgl_basis(int order) {
  NodalBasis b;
  b.order = order;
  b.nodes.resize(order + 1);
  b.weights.resize(order + 1);
  b.diff_matrix.resize((size_t)(order + 1) * (order + 1));
  check(expdg_lgl_basis(order, b.nodes.data(), b.weights.data(), b.diff_matrix.data()));
  return b;
}

}  // namespace b200
}  // namespace expdg
