/* expdg_b200 — C ABI of the B200-native exponential-DG hot path.
 *
 * Drop-in boundary for the reference library `expdg` (/root/reference/proj,
 * arXiv 2011.01316).  The reference is a C++20/Eigen library whose plugin
 * boundary is the split operator
 *     SplitOperator{dim, LinearAction linear, nonlinear}      proj/include/expdg/split_operator.hpp:12-20
 *     LinearAction = std::function<VectorXd(const VectorXd&)> proj/include/expdg/phi.hpp:11
 * produced by burgers_split_operator / euler_split_operator
 * (proj/include/expdg/burgers.hpp:94-96, proj/include/expdg/euler.hpp:105-107),
 * consumed by phi_combination (proj/include/expdg/phi.hpp:44-71), step_epi2
 * (proj/include/expdg/integrators.hpp:29-31) and integrate (:81-82).
 * Each entry point below replaces one of those; the C++ mirror of the
 * reference signatures lives in include/expdg_b200.hpp.
 *
 * Conventions: plain pointers and sizes; *_dev pointers are CUDA device
 * pointers (fp64), *_host pointers are host memory; `stream` is a cudaStream_t:
 * a non-NULL stream makes the call asynchronous on it; NULL runs on the
 * context's stream and returns when the work is complete.  Every call returns a status code; the
 * message of the last failure on the calling thread is expdg_last_error().
 * A context is not internally synchronised: one host thread per context.
 */
#ifndef EXPDG_B200_H
#define EXPDG_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* Status codes: the reference's exception types (SURVEY.md §8b "Errors"). */
#define EXPDG_OK 0
#define EXPDG_E_INVALID 1     /* std::invalid_argument  (e.g. proj/src/burgers.cpp:24-35)      */
#define EXPDG_E_DOMAIN 2      /* std::domain_error      (proj/src/euler.cpp:27-28, :210-211)    */
#define EXPDG_E_KRYLOV 3      /* KrylovError            (proj/include/expdg/phi.hpp:61-66)      */
#define EXPDG_E_CUDA 4        /* device / runtime failure (no reference analogue)             */
#define EXPDG_E_UNSUPPORTED 5 /* valid for the reference, not on the device path (e.g. 3D Roe)       */
#define EXPDG_E_COMM 6        /* communicator (NCCL / local group) failure of the multi-GPU path  */

/* Operator kinds. */
#define EXPDG_BURGERS1D 1 /* BurgersOperator (proj/src/burgers.cpp)                         */
#define EXPDG_BURGERS2D 2 /* extension: tensor-product LDG Burgers (config C3)               */
#define EXPDG_EULER2D 3   /* EulerOperator (proj/src/euler.cpp), Lax-Friedrichs split        */
#define EXPDG_EULER3D 4   /* extension: 3D Lax-Friedrichs Euler (config C5)                  */
#define EXPDG_DENSE 5     /* dense matrix LinearAction (the test fakes of proj/tests/test_phi.cpp) */
#define EXPDG_USER 6      /* user-supplied LinearAction / SplitProblem (expdg_user_op_create)     */

/* Integrator kinds: IntegratorKind (proj/include/expdg/integrators.hpp:15). */
#define EXPDG_EXP_EULER 0
#define EXPDG_EPI2 1
#define EXPDG_EXPRB32 2 /* step_exprb32 (proj/src/integrators.cpp:85-98): two phi calls (p = 1, p = 3) */
#define EXPDG_EXPRB42 3 /* step_exprb42 (proj/src/integrators.cpp:100-113) */

typedef struct expdg_ctx expdg_ctx;
typedef struct expdg_op expdg_op;

/* Mesh + physics of one operator.  Mirrors build_interval_mesh / build_quad_mesh
 * (proj/include/expdg/mesh.hpp:47-54, uniform breakpoints), BurgersConfig
 * (proj/include/expdg/burgers.hpp:16-23) and EulerConfig (proj/include/expdg/euler.hpp:33-37). */
typedef struct {
  int kind;            /* EXPDG_BURGERS1D .. EXPDG_EULER3D */
  int order;           /* LGL degree k (device: 1..8; 3D Euler 1..5) */
  int nx, ny, nz;      /* elements per axis */
  double x0, x1, y0, y1, z0, z1;
  int periodic;        /* 1 periodic, 0 zero-Dirichlet (Burgers 1D/2D only) */
  double kappa;        /* BurgersConfig::kappa */
  int flux;            /* Burgers: 0 lax_friedrichs, 1 entropy */
  double sigma;        /* entropy-flux jump penalty */
  int sigma_adaptive;
  int over_integrate;  /* 1D Burgers: Gauss rule of (3k+3)/2 points + consistent mass (proj/src/burgers.cpp:39-51) */
  double gamma;        /* Euler */
  int euler_flux;      /* 0 roe (2D only, proj/src/euler.cpp:114-145), 1 lax_friedrichs */
  /* Slab partition (0, 0 = the whole mesh): this rank owns the element
   * layers [part_begin, part_end) along the slowest axis — elements of a 1D Burgers mesh,
   * element rows of a 2D mesh (Burgers, Euler), z-planes of a 3D Euler mesh.  The global mesh stays nx x ny (x nz); the operator's state holds
   * only the owned layers and exchanges one halo layer with its periodic neighbours
   * (rank -+ 1) through the context's communicator. */
  int part_begin, part_end;
  /* Optional grading lists of build_quad_mesh (proj/src/mesh.cpp:96-120; grade_z: the 3D extension):
   * host arrays of nx+1 / ny+1 / nz+1 strictly increasing breakpoints spanning [x0, x1] / [y0, y1] /
   * [z0, z1] exactly ("grading list must span the domain" / "... strictly increasing" otherwise);
   * NULL: uniform breakpoints.  2D / 3D kinds only (the interval mesh has no grading).  Copied at
   * operator creation. */
  const double* grade_x;
  const double* grade_y;
  const double* grade_z;
} expdg_op_desc;

/* KrylovSettings (proj/include/expdg/integrators.hpp:20-24) + the two
 * PhiCombinationProblem knobs it does not expose (proj/include/expdg/phi.hpp:52-53);
 * 0 selects the reference default for initial_basis (16) / max_substeps (40). */
typedef struct {
  double tol;
  int max_basis;
  int orth_length;
  int initial_basis;
  int max_substeps;
} expdg_krylov_cfg;

/* KrylovStats (proj/include/expdg/phi.hpp:25-28) + KrylovError::last_estimate. */
typedef struct {
  long long iterations;
  int substeps;
  double last_estimate;
} expdg_krylov_stats;

/* TimeLoopConfig (proj/include/expdg/integrators.hpp:58-63). */
typedef struct {
  int integrator; /* EXPDG_EXP_EULER, EXPDG_EPI2, EXPDG_EXPRB32, EXPDG_EXPRB42 */
  double dt;
  double t_final;
  expdg_krylov_cfg krylov;
  int use_graph;  /* 1: device-resident control in CUDA-graph WHILE nodes; 0: host-stepped control */
  /* TimeLoopConfig::snapshot_every / IntegrationResult::snapshots (proj/include/expdg/integrators.hpp:60,
   * :73; proj/src/integrators.cpp:195-196): after every snapshot_every-th completed step (0: none), u is
   * copied into the next of snapshot_cap rows of `snapshots` (snapshot_cap x n doubles: device memory for
   * expdg_integrate, host memory for expdg_integrate_host) and its time into snapshot_times (host). */
  int snapshot_every;
  int snapshot_cap;
  double* snapshots;
  double* snapshot_times;
  /* TimeLoopConfig::on_step (proj/include/expdg/integrators.hpp:62): (step, t, max-norm of u, Krylov
   * iterations so far) for every completed step, in order, as soon as that step finishes on the device
   * (a stream-ordered host function: it must not call CUDA).  Not called for the step that blows up. */
  void (*on_step)(int step, double t, double max_abs, long long krylov_iterations, void* user);
  void* on_step_user;
} expdg_time_cfg;

/* IntegrationResult (proj/include/expdg/integrators.hpp:66-74), minus u (in place). */
typedef struct {
  double t;
  int status; /* 0 completed, 1 blew_up (RunStatus) */
  int steps;
  long long krylov_iterations;
  int blow_up_step;
  double max_abs;
  int snapshots;  /* snapshots taken (IntegrationResult::snapshots.size(); rows past snapshot_cap not stored) */
} expdg_integration_result;

const char* expdg_last_error(void);

/* Context: one device, one stream, the phi-engine workspace. */
int expdg_ctx_create(int device, expdg_ctx** out);
int expdg_ctx_destroy(expdg_ctx* ctx);
void* expdg_ctx_stream(expdg_ctx* ctx);
int expdg_ctx_synchronize(expdg_ctx* ctx);

/* Multi-GPU (slab partition, one process per GPU): the reference is single-threaded
 * and has no distributed layer; these add the two collectives the partitioned path
 * needs (sum/max allreduce of the reduced Gram-Schmidt dots and norms, neighbour
 * halo exchange).  Attach the communicator before creating partitioned operators;
 * with NCCL or the host-staged local group the control runs host-stepped, with the
 * peer-memory communicator (below) it stays in the CUDA graphs.
 *   NCCL: rank 0 calls expdg_nccl_unique_id, broadcasts the 128 bytes, every rank
 *         calls expdg_ctx_attach_nccl (collective, like ncclCommInitRank).
 *   Local group: several ranks driven by threads of one process (host-staged
 *         exchange; single-GPU tests of the partitioned algorithm). */
typedef struct expdg_local_group expdg_local_group;
int expdg_nccl_unique_id(unsigned char out[128]);
int expdg_ctx_attach_nccl(expdg_ctx* ctx, const unsigned char unique_id[128], int rank, int size);
int expdg_local_group_create(int size, expdg_local_group** out);
int expdg_local_group_destroy(expdg_local_group* g);
int expdg_ctx_attach_local(expdg_ctx* ctx, expdg_local_group* g, int rank);
int expdg_ctx_comm(const expdg_ctx* ctx, int* rank, int* size); /* 0, 1 without a communicator */
/* Device-resident peer-memory communicator: the allreduce and the halo exchange as plain kernels
 * over peer memory (P2P stores over NVLink + release/acquire epoch flags, fixed rank-order sums),
 * so a partitioned run keeps the CUDA-graph WHILE-node control (no host round-trip per Krylov
 * cycle).  halo_doubles: the largest element layer any operator of the context exchanges.
 *   One process per GPU: every rank calls expdg_ctx_peer_export (allocates its region, returns a
 *         64-byte CUDA IPC handle), the handles are all-gathered (rank order), every rank calls
 *         expdg_ctx_attach_peer.
 *   Threads of one process, one device (tests): expdg_peer_group_create + expdg_ctx_attach_peer_local.
 * Every device-side wait for a peer is bounded (EXPDG_PEER_TIMEOUT_MS, default 60000; 0 = unbounded): a peer that
 * never arrives ends expdg_phi_combination / expdg_integrate with EXPDG_E_COMM instead of hanging
 * the GPU; the results of that call are invalid. */
typedef struct expdg_peer_group expdg_peer_group;
int expdg_peer_group_create(int size, long long halo_doubles, expdg_peer_group** out);
int expdg_peer_group_destroy(expdg_peer_group* g);
int expdg_ctx_attach_peer_local(expdg_ctx* ctx, expdg_peer_group* g, int rank);
int expdg_ctx_peer_export(expdg_ctx* ctx, int size, long long halo_doubles, unsigned char handle_out[64]);
int expdg_ctx_attach_peer(expdg_ctx* ctx, const unsigned char* handles, int rank, int size);

/* Orthogonalisation of fully orthogonalised phi calls (orth_length >= max_basis):
 * EXPDG_ORTH_DCGS2 classical Gram-Schmidt with the reorthogonalisation of
 * column j-1 lagged into the two streaming passes of column j; EXPDG_ORTH_CGS2
 * classical Gram-Schmidt twice (three passes).  Both are the reference's two-pass
 * projector (proj/src/phi.cpp:94-100) up to rounding.  IOP windows always use one
 * classical pass over the window. */
#define EXPDG_ORTH_CGS2 0
#define EXPDG_ORTH_DCGS2 1
#define EXPDG_ORTH_AUTO 2 /* default: DCGS2 from 2^18 DOF up, CGS2 below (launch-latency bound) */
int expdg_ctx_set_orthogonalization(expdg_ctx* ctx, int mode);
/* Pipelined DCGS2 (default 1): each DCGS2 column applies the operator to the previous column's
 * image (a lookahead) and forms the new candidate's image by the Arnoldi relation, so the update
 * of column j, that image and the pass-1 dots of column j+1 share ONE stream of the basis
 * (8 n (j + 6) bytes + one operator application per column instead of two basis streams).
 * Same projector; 0 selects the two-pass DCGS2. */
int expdg_ctx_set_pipelined(expdg_ctx* ctx, int enable);
/* Small problems (1D Burgers, <= 2^15 DOF, one rank, CGS2) run each phi call as one
 * single-CTA kernel with the controller state in shared memory (default 1); 0 forces
 * the multi-kernel engine.  Same algorithm either way. */
int expdg_ctx_set_fused(expdg_ctx* ctx, int enable);

/* Operator factory: replaces BurgersOperator / EulerOperator construction
 * (proj/src/burgers.cpp:20-93, proj/src/euler.cpp:186-244) minus the frozen
 * state, which expdg_op_linearize supplies. */
int expdg_op_create(expdg_ctx* ctx, const expdg_op_desc* desc, expdg_op** out);
/* Dense LinearAction y = A x (row-major n x n, host memory): the dense fakes of
 * proj/tests/test_phi.cpp:16-29 and proj/tests/test_integrators.cpp:15-23. */
int expdg_dense_op_create(expdg_ctx* ctx, int n, const double* a_host, expdg_op** out);
/* User operator: any reference LinearAction (proj/include/expdg/phi.hpp:11) or SplitProblem
 * (proj/include/expdg/integrators.hpp:48-52) drives the device phi engine and time loop.
 * The callbacks receive DEVICE pointers of n doubles and the stream to enqueue on, and return
 * EXPDG_OK or a status code (EXPDG_E_DOMAIN plays the reference's std::domain_error — inside
 * integrate it fails the step, which then reports blew_up like proj/src/integrators.cpp:179-193;
 * EXPDG_E_INVALID plays std::invalid_argument and propagates).
 *   apply_linear     y = L x at the frozen state (SplitOperator::linear).  Required.
 *   apply_nonlinear  y = N x (SplitOperator::nonlinear).  NULL: N = 0 (a plain LinearAction).
 *   linearize        freeze the user's operator at ref (SplitProblem::linearize(ref)); called by
 *                    expdg_op_linearize and by integrate at u^n every step (at u0 once for
 *                    exp_euler).  NULL: L does not depend on the state.  ref stays valid until
 *                    the next linearize call.
 *   graph_safe       1: the callbacks only enqueue stream-ordered work on `stream` (no host sync,
 *                    no allocation), so the library may record them once into its CUDA graphs and
 *                    replay them (device-resident control, no host round-trip per Krylov cycle);
 *                    their host-side code then runs only while recording.  0: host-stepped
 *                    control, every callback invoked for real each time.
 * The engine hands the callbacks fixed scratch vectors (the same x / y pointers every cycle).
 * Not slab-partitioned: refused on a context whose communicator spans several ranks. */
typedef struct {
  int (*apply_linear)(const double* x_dev, double* y_dev, void* stream, void* user);
  int (*apply_nonlinear)(const double* x_dev, double* y_dev, void* stream, void* user);
  int (*linearize)(const double* ref_dev, void* stream, void* user);
  int graph_safe;
} expdg_user_op_fns;
int expdg_user_op_create(expdg_ctx* ctx, long long n, const expdg_user_op_fns* fns, void* user, expdg_op** out);
int expdg_op_destroy(expdg_op* op);
long long expdg_op_dim(const expdg_op* op);

/* Freeze the reference state u~ (copied): burgers_split_operator / euler_split_operator
 * (proj/src/burgers.cpp:309-320, proj/src/euler.cpp:390-401).  EXPDG_E_DOMAIN on an
 * inadmissible Euler state (proj/src/euler.cpp:210-211). */
int expdg_op_linearize(expdg_op* op, const double* ref_dev);
/* Steady weak source of BurgersConfig::source (proj/src/burgers.cpp:80-92): the per-element
 * load vector 0.5 h_e I^T (W s) in state layout (n doubles, device, copied), added to N and
 * the full RHS.  1D Burgers only. */
int expdg_op_set_source(expdg_op* op, const double* weak_source_dev);
/* Same, from the source function itself (BurgersConfig::source, proj/include/expdg/burgers.hpp:22):
 * the library evaluates source(x, user) at the operator's quadrature points and builds the
 * weak load exactly as proj/src/burgers.cpp:80-92. */
int expdg_op_set_source_fn(expdg_op* op, double (*source)(double x, void* user), void* user);
/* SplitOperator::linear — the JVP (proj/src/burgers.cpp:146-180, proj/src/euler.cpp:299-341). */
int expdg_op_apply_linear(expdg_op* op, const double* x_dev, double* y_dev, void* stream);
/* SplitOperator::nonlinear (proj/src/burgers.cpp:182-215, proj/src/euler.cpp:343-388). */
int expdg_op_apply_nonlinear(expdg_op* op, const double* x_dev, double* y_dev, void* stream);
/* burgers_full_rhs / euler_full_rhs (proj/include/expdg/burgers.hpp:99-101, euler.hpp:110-111). */
int expdg_op_full_rhs(expdg_op* op, const double* x_dev, double* y_dev, void* stream);

/* phi_combination (proj/src/phi.cpp:133-260): out = sum_i dt^i phi_i(dt L) b_i with
 * L the op's linear action at its frozen state; b_dev[0..p], NULL entries are zero
 * vectors.  Synchronous; EXPDG_E_KRYLOV maps KrylovError (stats->last_estimate set). */
int expdg_phi_combination(expdg_ctx* ctx, expdg_op* op, const double* const* b_dev, int p, double dt,
                          const expdg_krylov_cfg* cfg, double* out_dev, expdg_krylov_stats* stats);

/* krylov_build (proj/include/expdg/phi.hpp:40-42, proj/src/phi.cpp:115-130): Arnoldi
 * (orth_length >= m) or incomplete-orthogonalisation factorisation of span{seed, L seed, ...}
 * on the device engine (classical Gram-Schmidt with one reorthogonalisation pass; the
 * reference's two MGS passes up to rounding; its breakdown test).  seed_dev: n doubles.
 * Outputs (any may be NULL): basis_dev n x (m+1) column-major device matrix (columns past the
 * returned m + (invariant ? 0 : 1) are left untouched), hessenberg_host (m+1) x m row-major,
 * seed_norm, m_out (columns built), invariant (happy breakdown before m).  EXPDG_E_INVALID on a
 * zero seed ("krylov_build: zero seed"); m <= 128. */
int expdg_krylov_build(expdg_ctx* ctx, expdg_op* op, const double* seed_dev, int m, int orth_length,
                       double* basis_dev, double* hessenberg_host, double* seed_norm, int* m_out,
                       int* invariant);

/* step_epi2 (proj/src/integrators.cpp:76-83) with the op linearised at u:
 * u <- u + phi_combination({0, L u + N u}).  Synchronous. */
int expdg_step_epi2(expdg_ctx* ctx, expdg_op* op, double* u_dev, double dt, const expdg_krylov_cfg* cfg,
                    expdg_krylov_stats* stats);

/* integrate (proj/src/integrators.cpp:140-201) for EPI2 / EXPRB32 / EXPRB42 (relinearised
 * each step) and exp_euler (frozen at u0).  u_dev updated in place.  Optional per-step outputs
 * (capacity `cap`): cumulative Krylov iterations and max|u| (the on_step payload,
 * proj/include/expdg/integrators.hpp:62).  Blow-up is reported, not returned as an error. */
int expdg_integrate(expdg_ctx* ctx, expdg_op* op, double* u_dev, const expdg_time_cfg* cfg,
                    expdg_integration_result* res, long long* iters_per_step, double* amax_per_step, int cap);
/* Same from/to HOST memory (the H2D / D2H copies are part of the call). */
int expdg_integrate_host(expdg_ctx* ctx, expdg_op* op, double* u_host, const expdg_time_cfg* cfg,
                         expdg_integration_result* res, long long* iters_per_step, double* amax_per_step,
                         int cap);

/* Device matrix exponential (the controller's Higham 2005 expm, one CTA),
 * n <= 130, row-major host in/out: the Eigen MatrixFunctions exp() call site
 * proj/src/phi.cpp:40. */
int expdg_expm(expdg_ctx* ctx, int n, const double* a_host, double* out_host);
/* Engine path of the last phi_combination / integrate call (instrumentation, so tests can
 * assert they ran the path bench.py times): out4 = {DCGS2 orthogonalisation (0: CGS2 / IOP,
 * 1: DCGS2, 2: pipelined DCGS2 -- one V stream per column),
 * the operator sweep took the DCGS2 pass-1 dots of every column, device-resident control in
 * CUDA-graph WHILE nodes, small-problem fused / cluster engine}. */
int expdg_ctx_last_path(expdg_ctx* ctx, int* out4);
/* Controller state of the last phi call (16 doubles, for diagnostics). */
int expdg_debug_state(expdg_ctx* ctx, double* out16);
/* Micro-benchmark of one CGS2 streaming pass (mode 0 dots, 1 update+dots,
 * 2 update+norm, 3 combine) against k basis vectors of length n; avg ms. */
int expdg_bench_ts(expdg_ctx* ctx, long long n, int k, int mode, int reps, double* ms);
/* Micro-benchmark of one phi-cycle operator application at column j (mode 0; the
 * operator kernel also takes the DCGS2 pass-1 dots where it does so in the engine), of the
 * separate DCGS2 dots pass at column j (mode 1), or of the pipelined DCGS2 lookahead application
 * (mode 2: slot j+1 -> slot j+2, the plain kernel) on the current Krylov slots;
 * the operator must be linearized; avg ms (diagnostics). */
int expdg_bench_apply(expdg_ctx* ctx, expdg_op* op, int j, int mode, int reps, double* ms);
/* Hessenberg matrix of the last phi call, (129 x 128) row-major (diagnostics). */
int expdg_debug_hessenberg(expdg_ctx* ctx, double* out);

/* Setup helpers. */
int expdg_lgl_basis(int order, double* nodes, double* weights, double* diff_rowmajor);
/* Seeded synthetic inputs of BASELINE.json configs 1..5. */
int expdg_initial_condition(int config, int nx, int order, uint64_t seed, double noise, double* out_host);
/* Config 5's Taylor-Green state on an nx x ny x nz mesh of box6 = {x0,x1,y0,y1,z0,z1}, z-planes
 * [layer_begin, layer_end) only: each rank of a z-partitioned run (C5 at 128^3 over N GPUs) builds
 * just its slab.  The cubic [0, 2 pi]^3 case equals expdg_initial_condition(5, ...) bit for bit. */
int expdg_initial_condition_slab(int config, int nx, int ny, int nz, int order, const double* box6,
                                 int layer_begin, int layer_end, double* out_host);
/* Number of device kernels launched by this context since creation (instrumentation). */
long long expdg_ctx_kernel_launches(expdg_ctx* ctx);
/* Device-event time (ms) of the last expdg_integrate call's step loop. */
double expdg_ctx_last_loop_ms(expdg_ctx* ctx);
/* Canonical algorithmic HBM bytes of the last integrate / phi call's
 * realised trajectory, and its counts of Arnoldi columns, avnorm applications and
 * accepted substeps: out4 = {bytes, columns, avnorms, combines}. */
/* Roofline of the dominant kernel (the DCGS2 update pass): with enable = 1 the next
 * host-stepped runs (expdg_time_cfg.use_graph = 0) record CUDA events around every
 * DCGS2 update-pass launch (enable 1) or every phi-cycle operator application
 * (enable 2) on the context stream.  out3 = {summed launch ms, summed algorithmic bytes
 * (update pass 8 n (j + 4); Euler 2D strip sweep 32 n + 8 n j with fused dots),
 * launches that extended a column}. */
int expdg_ctx_time_dominant(expdg_ctx* ctx, int enable /* 0 off, 1 DCGS2 update pass, 2 operator sweep */);
int expdg_ctx_dominant_stats(expdg_ctx* ctx, double* out3);
/* Fused small-problem engine: SM clock cycles spent per phase in the last run
 * (apply, dots, updates, combine, controller; 0 for the multi-kernel engine). */
int expdg_debug_profile(expdg_ctx* ctx, long long* out8);
/* SM clock cycles of the controller's expm sub-phases summed over its calls: norm + scaling,
 * Pade powers / U / V, LU elimination, back substitution, squarings; then calls, squarings taken. */
int expdg_debug_expm_profile(expdg_ctx* ctx, long long* out8);
int expdg_ctx_traffic(expdg_ctx* ctx, double* out4);

#ifdef __cplusplus
}
#endif

#endif /* EXPDG_B200_H */
