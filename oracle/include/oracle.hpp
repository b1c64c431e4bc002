// ORACLE — test infrastructure only.
//
// Eigen-free CPU restatement of the reference exponential-DG library
// (/root/reference/proj, "expdg", arXiv 2011.01316).  It is the parity
// checker for the B200 product path and the `cpu_baseline` leg of bench.py.
// Only tests/, __graft_entry__.smoke() and bench.py's CPU legs may load it;
// the product library (paper_2011_01316_b200) never links or calls it.
//
// Parity pinning: the reference cannot be compiled in this image (it needs
// Eigen3, doctest and CLI11, none of which are present).  This
// restatement is pinned against the reference's own known-answer tests
// (proj/tests/*.cpp) and the digits recorded by the reference's acceptance run
// (proj/test_output.txt:18-28) — see tests/test_oracle_pins.py.
//
// Every function cites the reference file:line it restates.  The only
// third-party arithmetic on the path is Eigen's MatrixFunctions `exp()`
// (proj/src/phi.cpp:5,40; Eigen >= 3.3, version unpinned), restated here as
// Higham (2005) Pade scaling-and-squaring; and Eigen's LDLT (diagonal
// pivoting) for the over-integrated Burgers mass matrix.
//
// Extensions (not in the reference): a 2D tensor-product
// LDG Burgers operator and a 3D Lax-Friedrichs Euler operator, built so that a
// y-invariant (resp. z-invariant, w = 0) field reproduces the 1D Burgers
// (resp. 2D Euler) operator of the reference.
#pragma once

#include <array>
#include <cmath>
#include <functional>
#include <memory>
#include <stdexcept>
#include <string>
#include <vector>

namespace oracle {

using Vec = std::vector<double>;

// Row-major dense matrix (replaces Eigen::MatrixXd on the few call sites).
struct Mat {
  int r = 0, c = 0;
  std::vector<double> a;
  Mat() = default;
  Mat(int rows, int cols, double v = 0.0) : r(rows), c(cols), a(size_t(rows) * cols, v) {}
  double& operator()(int i, int j) { return a[size_t(i) * c + j]; }
  double operator()(int i, int j) const { return a[size_t(i) * c + j]; }
  static Mat identity(int n) {
    Mat m(n, n);
    for (int i = 0; i < n; ++i) m(i, i) = 1.0;
    return m;
  }
};

Mat matmul(const Mat& a, const Mat& b);
Vec matvec(const Mat& a, const Vec& x);
double dot(const Vec& a, const Vec& b);
double norm(const Vec& a);
Vec axpby(double a, const Vec& x, double b, const Vec& y);  // a x + b y
Vec add(const Vec& x, const Vec& y);
Vec scale(double a, const Vec& x);
double max_abs(const Vec& x);
bool all_finite(const Vec& x);

// ---------------------------------------------------------------- basis
// proj/include/expdg/basis.hpp:9-38, proj/src/basis.cpp
struct NodalBasis {
  int order = 0;
  Vec nodes, weights;
  Mat diff;  // D(i,j) = dl_j/dx at node i
  int num_nodes() const { return order + 1; }
};
struct QuadratureRule {
  Vec points, weights;
  int exact_degree = 0;
};
NodalBasis lgl_basis(int order);
QuadratureRule gauss_quadrature(int num_points);
QuadratureRule lgl_quadrature(const NodalBasis& b);
Vec lagrange_values(const NodalBasis& b, double x);
Mat interpolation_matrix(const NodalBasis& b, const Vec& points);

// ---------------------------------------------------------------- mesh
// proj/include/expdg/mesh.hpp, proj/src/mesh.cpp
enum class BoundaryKind { periodic, dirichlet_zero };
struct Element {
  double x0 = 0, x1 = 0, y0 = 0, y1 = 0, z0 = 0, z1 = 0;
  double hx = 0, hy = 0, hz = 0, measure = 0;
};
struct Face {
  int owner = -1, neighbor = -1, axis = 0;
  double normal = 1.0;
  int owner_side = 1, neighbor_side = 0;
  double h_owner = 0, measure = 1.0;
};
struct Mesh {
  int dim = 1, nx = 0, ny = 1, nz = 1;
  Vec xs, ys, zs;
  std::vector<Element> elements;
  std::vector<Face> faces;
  BoundaryKind bc = BoundaryKind::periodic;
  int num_elements() const { return int(elements.size()); }
};
Mesh build_interval_mesh(double a, double b, int ne, BoundaryKind bc);
Mesh build_quad_mesh(double x0, double x1, double y0, double y1, int nx, int ny,
                     BoundaryKind bc, const Vec& grade_x = {}, const Vec& grade_y = {});
// Extension (C5): periodic hex mesh, x-faces then y-faces then z-faces.
Mesh build_hex_mesh(double x0, double x1, double y0, double y1, double z0,
                    double z1, int nx, int ny, int nz, const Vec& grade_x = {},
                    const Vec& grade_y = {}, const Vec& grade_z = {});
double min_node_spacing(const Mesh& mesh, const NodalBasis& b);
std::vector<int> face_node_indices(const Mesh& mesh, const NodalBasis& b,
                                   const Face& f, bool owner_side);
int nodes_per_element(const Mesh& mesh, const NodalBasis& b);

// L2 projection onto the broken space (proj/src/mesh.cpp:315-386).
Vec l2_project_1d(const std::function<double(double)>& f, const Mesh& mesh,
                  const NodalBasis& b, const QuadratureRule& quad);
// 2D, `components` interleaved per element as [e][c][node]; f returns all comps.
Vec l2_project_system_2d(const std::function<void(double, double, double*)>& f,
                         int components, const Mesh& mesh, const NodalBasis& b,
                         const QuadratureRule& quad);
double evaluate_1d(const Vec& u, const Mesh& mesh, const NodalBasis& b, double x);
double evaluate_2d(const Vec& u, int components, const Mesh& mesh,
                   const NodalBasis& b, double x, double y, int comp);

// Dense symmetric LDLT with diagonal pivoting (Eigen::LDLT semantics).
struct LDLT {
  int n = 0;
  Mat l;                  // unit lower factor (in permuted order)
  Vec d;
  std::vector<int> perm;  // row i of the factor is original row perm[i]
  void compute(const Mat& a);
  Vec solve(const Vec& b) const;
};

// ---------------------------------------------------------------- burgers
// proj/include/expdg/burgers.hpp, proj/src/burgers.cpp
enum class FluxKind { lax_friedrichs, entropy };
struct BurgersConfig {
  double kappa = 0.03;
  FluxKind flux = FluxKind::lax_friedrichs;
  double sigma = 0.0;
  bool sigma_adaptive = false;
  bool over_integrate = false;
  std::function<double(double)> source;
};
double entropy_flux(double um, double up, double jump, double sigma, double h);
double lax_friedrichs_flux(double um, double up, double jump);

class BurgersOperator {
 public:
  BurgersOperator(const Mesh& mesh, const NodalBasis& basis, BurgersConfig cfg, Vec utilde);
  Vec apply_linear(const Vec& u) const;
  Vec apply_nonlinear(const Vec& u) const;
  Vec full_rhs(const Vec& u) const;
  Vec gradient(const Vec& u) const;
  double inner_product(const Vec& a, const Vec& b) const;
  double penalty_seminorm_sq(const Vec& u) const;
  double dg_norm_sq(const Vec& u) const;
  long dim() const { return dim_; }

 private:
  struct FaceFrozen {
    double ut_minus = 0, ut_plus = 0, diss = 0, sigma_over_h = 0, inv_h = 0;
  };
  double face_linear_flux(const FaceFrozen& fd, double um, double up, double jump) const;
  double face_nonlinear_flux(const FaceFrozen& fd, double um, double up, double jump) const;
  void trace_values(const Vec& u, int f, double& um, double& up) const;
  Vec seg_matvec(const Mat& m, const Vec& u, int e) const;
  Vec mass_solve_scaled(const Vec& r) const;

  const Mesh* mesh_;
  const NodalBasis* basis_;
  BurgersConfig cfg_;
  Vec utilde_;
  long dim_ = 0;
  int np_ = 0;
  Mat interp_, dinterp_, grad_vol_, lift_vol_;
  Vec wq_;
  LDLT mass_;
  bool mass_diagonal_ = false;
  Mat utilde_q_;  // (nq x ne)
  std::vector<FaceFrozen> faces_;
  Vec source_weak_;
};

// Extension (C3): 2D tensor-product LDG Burgers, flux (u^2/2, u^2/2),
// collocated LGL, periodic or dirichlet_zero quads.  The operator is the sum of
// the reference 1D LDG operator applied along every element row (x) and every
// element column (y), which is exactly the collocated 2D weak form on a
// Cartesian mesh; a y-invariant field therefore reproduces the 1D operator.
class Burgers2DOperator {
 public:
  Burgers2DOperator(const Mesh& mesh, const NodalBasis& basis, BurgersConfig cfg, Vec utilde);
  Vec apply_linear(const Vec& u) const;
  Vec apply_nonlinear(const Vec& u) const;
  Vec full_rhs(const Vec& u) const;
  long dim() const { return dim_; }

 private:
  enum Mode { kLinear, kNonlinear, kFull };
  Vec apply(const Vec& u, Mode mode) const;
  const Mesh* mesh_;
  const NodalBasis* basis_;
  BurgersConfig cfg_;
  Vec utilde_;
  long dim_ = 0;
  int np1_ = 0, np_ = 0;
  Mat grad_vol_, lift_vol_;
};

// ---------------------------------------------------------------- euler 2D
// proj/include/expdg/euler.hpp, proj/src/euler.cpp
struct EulerPrimitives { double rho, u, v, p, a, H; };
struct VortexParams {
  double alpha = 2.0, lambda = 0.05, u_inf = 0.2, v_inf = 0.0;
  double rho_inf = 1.0, T_inf = 1.0, p_inf = 1.0, xc = 5.0, yc = 0.0;
  double wrap_lx = 10.0, wrap_ly = 10.0;
};
enum class EulerFluxKind { roe, lax_friedrichs };
struct EulerConfig {
  double gamma = 1.4;
  EulerFluxKind flux = EulerFluxKind::roe;
  VortexParams vortex;
};
using State4 = std::array<double, 4>;
using Mat4 = std::array<double, 16>;  // row-major
bool admissible(const State4& q, double gamma);
EulerPrimitives primitives(const State4& q, double gamma);
void euler_flux(const State4& q, double gamma, double f[4][2]);
Mat4 flux_jacobian(const State4& q, double nx, double ny, double gamma);
struct RoeAverage { double rho, u, v, H, a; };
RoeAverage roe_average(const State4& qm, const State4& qp, double gamma);
Mat4 abs_flux_jacobian(const RoeAverage& avg, double nx, double ny, double gamma);
State4 roe_flux(const State4& qm, const State4& qp, double nx, double ny, double gamma);
State4 euler_lax_friedrichs_flux(const State4& qm, const State4& qp, double nx, double ny,
                                 double gamma);
State4 isentropic_vortex(double x, double y, double t, const EulerConfig& cfg);

class EulerOperator {
 public:
  EulerOperator(const Mesh& mesh, const NodalBasis& basis, EulerConfig cfg, const Vec& qtilde);
  Vec apply_linear(const Vec& q) const;
  Vec apply_nonlinear(const Vec& q) const;
  long dim() const { return dim_; }

 private:
  void rhs_faces(const Vec& q, bool linear_part, Vec& r) const;
  void apply_inverse_mass(Vec& r) const;
  void volume(const Vec& q, bool linear_part, Vec& r) const;
  const Mesh* mesh_;
  const NodalBasis* basis_;
  EulerConfig cfg_;
  long dim_ = 0;
  int np1_ = 0, np_ = 0;
  std::vector<Mat4> jac_x_, jac_y_;
  struct FaceFrozen { Mat4 a_minus, a_plus, a_abs; };
  std::vector<FaceFrozen> face_frozen_;
};
Vec euler_full_rhs(const Mesh& mesh, const NodalBasis& basis, const EulerConfig& cfg,
                   const Vec& q);

// ---------------------------------------------------------------- euler 3D
// Extension (C5): 5 conserved variables (rho, rho u, rho v, rho w, rho E),
// Lax-Friedrichs flux, periodic hex mesh, same split as the 2D operator
// (L = frozen Jacobians + LF dissipation frozen at the reference traces).
using State5 = std::array<double, 5>;
using Mat5 = std::array<double, 25>;
Mat5 flux_jacobian3(const State5& q, const double n[3], double gamma);
bool admissible3(const State5& q, double gamma);
class Euler3DOperator {
 public:
  Euler3DOperator(const Mesh& mesh, const NodalBasis& basis, double gamma, const Vec& qtilde);
  Vec apply_linear(const Vec& q) const;
  Vec apply_nonlinear(const Vec& q) const;
  long dim() const { return dim_; }

 private:
  Vec apply(const Vec& q, bool linear_part) const;
  const Mesh* mesh_;
  const NodalBasis* basis_;
  double gamma_;
  Vec qtilde_;
  long dim_ = 0;
  int np1_ = 0, np_ = 0;
};

// ---------------------------------------------------------------- phi
// proj/include/expdg/phi.hpp, proj/src/phi.cpp
using LinearAction = std::function<Vec(const Vec&)>;
double phi_scalar(int i, double tau);
Mat expm(const Mat& m);
std::vector<Mat> phi_dense_family(int p, const Mat& m);
Mat phi_dense(int i, const Mat& m);

struct KrylovStats {
  long iterations = 0;
  int substeps = 0;
};
struct KrylovFactorization {
  Mat basis;       // n x (m+1) (stored column-major as Mat(rows=m+1? no: n x cols))
  Mat hessenberg;  // (m+1) x m
  double seed_norm = 0;
  int m = 0;
  bool invariant_subspace = false;
};
KrylovFactorization krylov_build(const LinearAction& op, const Vec& seed, int m, int orth_length);

struct PhiCombinationProblem {
  LinearAction op;
  std::vector<Vec> b;
  double dt = 1.0, tol = 1e-12;
  int max_basis = 128, orth_length = 128, max_substeps = 40, initial_basis = 16;
};
struct PhiCombinationResult {
  Vec value;
  KrylovStats stats;
};
class KrylovError : public std::runtime_error {
 public:
  KrylovError(const std::string& w, double e) : std::runtime_error(w), last_estimate(e) {}
  double last_estimate;
};
PhiCombinationResult phi_combination(const PhiCombinationProblem& prob);

// ---------------------------------------------------------------- integrators
// proj/include/expdg/integrators.hpp, proj/src/integrators.cpp
enum class IntegratorKind { exp_euler, epi2, exprb32, exprb42, rk2, rk3, rk4 };
IntegratorKind integrator_from_name(const std::string& name);
struct KrylovSettings {
  double tol = 1e-12;
  int max_basis = 128, orth_length = 128;
};
struct SplitOperator {
  long dim = 0;
  LinearAction linear, nonlinear;
};
Vec step_exp_euler(const SplitOperator& op, const Vec& u, double dt, const KrylovSettings& ks,
                   KrylovStats* stats = nullptr);
Vec step_epi2(const SplitOperator& op, const Vec& u, double dt, const KrylovSettings& ks,
              KrylovStats* stats = nullptr);
Vec step_exprb32(const SplitOperator& op, const Vec& u, double dt, const KrylovSettings& ks,
                 KrylovStats* stats = nullptr);
Vec step_exprb42(const SplitOperator& op, const Vec& u, double dt, const KrylovSettings& ks,
                 KrylovStats* stats = nullptr);
using RhsAction = std::function<Vec(const Vec&)>;
Vec step_rk(IntegratorKind kind, const RhsAction& rhs, const Vec& u, double dt);

struct SplitProblem {
  long dim = 0;
  std::function<SplitOperator(const Vec& ref)> linearize;
  RhsAction rhs;
};
enum class RunStatus { completed, blew_up };
struct TimeLoopConfig {
  double dt = 0.1, t_final = 1.0;
  KrylovSettings krylov;
  int snapshot_every = 0;  // 0: keep no intermediate states
  std::function<void(int, double, double, long)> on_step;
};
struct IntegrationResult {
  Vec u;
  double t = 0.0;
  RunStatus status = RunStatus::completed;
  int steps = 0;
  long krylov_iterations = 0;
  int blow_up_step = -1;
  double max_abs = 0.0;
  std::vector<std::pair<double, Vec>> snapshots;
};
IntegrationResult integrate(const SplitProblem& problem, IntegratorKind kind, Vec u0,
                            const TimeLoopConfig& cfg);

// ---------------------------------------------------------------- harness subset
// proj/src/harness.cpp:48-238
struct CourantNumbers { double cr_a = 0, cr_d = 0; };
CourantNumbers courant_numbers(const Vec& u, const Mesh& mesh, const NodalBasis& b, int components,
                               double dt, double kappa, bool euler, double gamma = 1.4);
struct ProblemContext {
  std::shared_ptr<Mesh> mesh;
  std::shared_ptr<NodalBasis> basis;
  int components = 1;
  SplitProblem split;
  Vec u0;
  std::function<double(double, double, double, int)> exact;
  bool is_euler = false;
  BurgersConfig burgers;
  EulerConfig euler;
};
struct ExperimentConfig {
  std::string problem = "burgers-smooth";
  std::string flux;
  double sigma = 0.0;
  bool sigma_adaptive = false;
  int over_integrate = -1;  // -1: problem default
  double kappa = -1.0;
};
ProblemContext make_problem(const ExperimentConfig& cfg, int ne, int k);
Vec l2_error(const Vec& u, int components, const Mesh& mesh, const NodalBasis& b,
             const std::function<double(double, double, int)>& ref);

}  // namespace oracle
