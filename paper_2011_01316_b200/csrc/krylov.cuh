// Host-side interface of the device-resident phi engine (krylov.cu) and of the
// operator kernels (ops_*.cu).
#pragma once

#include <memory>
#include <vector>

#include "comm.cuh"
#include "expdg_internal.cuh"

namespace expdg {

// Vectors b_1..b_p that the augmented operator adds (proj/src/phi.cpp:151-158).
struct BArgs {
  const double* b[kMaxP + 1];  // b[0] .. b[p]; nullptr = zero vector
  int p;
};

#ifdef __CUDACC__
// v + sum_{k<p} xt[k] b_{p-k}[g] (the augmented columns of proj/src/phi.cpp:151-158), in the
// reference's order; compile-time indices into b so the kernel parameter stays out of local memory
__device__ __forceinline__ double aug_tail(const BArgs& b, const double* xt, size_t g, double v) {
#pragma unroll
  for (int m = kMaxP; m >= 1; --m)
    if (m <= b.p && b.b[m]) v = fma(xt[b.p - m], b.b[m][g], v);
  return v;
}
#endif

class Engine;

// Device operator: one DG operator frozen at a reference state (ũ pointer).
class OpDevice {
 public:
  virtual ~OpDevice() = default;
  expdg_op_desc desc{};
  long long n = 0;        // local DOF count
  int comps = 1;
  const double* ref = nullptr;  // ũ (device), not owned
  // Slab-partitioned operators (desc.part_end > desc.part_begin) hold only their
  // element rows and exchange one halo row per application through `comm`.
  Comm* comm = nullptr;
  bool partitioned() const { return desc.part_end > desc.part_begin; }
  // Cycle apply: y = dt * aug(s_j V_j) into slot j+1 plus ||y||^2 (action EXTEND/AVNORM).
  // stage 2 (pipelined DCGS2 lookahead): the engine passes base + ld, so the kernels apply the
  // operator to s_j slot_{j+1} and write slot j+2; operators then pick their plain (no fused
  // dots) kernel variant.  The kernels gate themselves on apply_go().
  virtual void launch_phi_apply(cudaStream_t s, PhiState* st, double* base, double* partials,
                                const BArgs& b, int stage = 1) = 0;
  // Standalone: which 0 = L x (at ref), 1 = N x (at ref), 2 = full rhs (no ref).
  virtual void launch_apply(cudaStream_t s, int which, const double* x, double* y) = 0;
  // Step residual R = L u + N u at ref = u, with ||R||^2 -> st->red.bnorm2[1] and the
  // inadmissibility flag -> st->domain_flag.  Skipped when st->stopped.
  virtual void launch_residual(cudaStream_t s, const double* u, double* r, PhiState* st,
                               double* partials) = 0;
  // Whether the apply kernel also writes pass-A dots (else the generic kernel runs).
  virtual bool fused_dots() const { return false; }
  // DCGS2: the apply kernel also takes the pass-1 dots (k_ts2<TS2_DOTS>) of columns
  // j <= this bound (-1: never); k_ts2<TS2_DOTS> no-ops for those columns.
  virtual int fused_dcgs_dots_jmax() const { return -1; }
  // Whether launch_phi_apply / launch_apply / launch_residual only enqueue stream work that
  // may be recorded once into a CUDA graph and replayed (user operators may not).
  virtual bool graph_capturable() const { return true; }
  // Small problems: the whole phi call as one single-CTA kernel (fused.cuh)
  virtual bool fused_capable() const { return false; }
  virtual void launch_fused(cudaStream_t, Engine&, const BArgs&) {}
  // Freeze the reference state (proj/src/burgers.cpp:53-78, proj/src/euler.cpp:198-243):
  // operators that keep derived frozen data compute it here.
  virtual void freeze(cudaStream_t s, const double* r) { ref = r; }
  // Weak steady source added to N and the full RHS (BurgersConfig::source,
  // proj/src/burgers.cpp:80-92): per element (s, l_j) values, state layout.
  virtual void set_source(cudaStream_t, const double*) {
    throw std::invalid_argument("this operator has no source term");
  }
};

std::unique_ptr<OpDevice> make_burgers1d(const expdg_op_desc& d);
std::unique_ptr<OpDevice> make_burgers2d(const expdg_op_desc& d);
std::unique_ptr<OpDevice> make_euler2d(const expdg_op_desc& d);
std::unique_ptr<OpDevice> make_euler3d(const expdg_op_desc& d);
std::unique_ptr<OpDevice> make_dense(int n, const double* a_host);
std::unique_ptr<OpDevice> make_user(long long n, const expdg_user_op_fns& fns, void* user, int num_sms);

// Host-side LGL basis (same arithmetic as proj/src/basis.cpp:35-85).
struct HostBasis {
  int order = 0;
  std::vector<double> nodes, weights, D;  // D row-major
};
HostBasis host_lgl_basis(int order);
struct HostOI {
  int nq = 0;
  std::vector<double> I, G, Lv, Mi;  // interp (nq x np), grad_vol, lift_vol (np x nq), M^-1
};
HostOI host_burgers_oi(int order);
std::vector<double> host_h_table(double a, double b, int ne);
std::vector<double> host_h_table(const std::vector<double>& breaks);
std::vector<double> host_axis_breaks(double a, double b, int n, const double* grade);
void host_tgv_slab(int nx, int ny, int nz, int order, const double* box, int k0, int k1, double* out);
void host_burgers_source(int order, int ne, double a, double b, bool over_integrate,
                         double (*fn)(double, void*), void* user, double* out);

// Device workspace + launch helpers of the phi engine.
struct TsTuning {
  // dynamic smem per CTA of the tall-skinny passes (216 KB; 192 KB: C4 same box 198.7 vs 195.3 ms
  // per step, k_ts3 3.79 vs 3.68 ms per launch)
  int budget = 221184;
  int stages = 2;       // pipeline depth cap
  int min_T = 64;       // smallest tile (doubles) before giving up stages
};

class Engine {
 public:
  TsTuning ts_tuning;
  int ld_odd = 1;
  int use_dcgs = 1;  // 0 CGS2, 1 auto (DCGS2 from 2^18 DOF), 2 DCGS2 (EXPDG_ORTH=cgs2|dcgs2)
  int use_fused = 1;  // small problems run each phi call as one fused kernel (EXPDG_FUSED=0: off)
  int use_pipe = 1;   // pipelined DCGS2: one V stream per Krylov column (EXPDG_PIPE=0: off)
  int pipe_restart = 0;  // diagnostics: direct application every n-th column (EXPDG_PIPE_RESTART)
  // merged-pass stage cap after the tile choice (EXPDG_TS3_STAGES): 4 stages where they fit
  // (C4 same box: 3.78 vs 3.89 ms per k_ts3 launch, 198.8 vs 201.1 ms per step)
  int ts3_stages = 4;
  int ts3_tstages = 0;  // stages the merged pass's tile choice assumes (EXPDG_TS3_TSTAGES; 0: 2)
  int ts3_pow2 = 0;     // power-of-two merged-pass tiles only (EXPDG_TS3_POW2=1: the round-2 rule, for A/B runs)
  // host-stepped runs: CUDA events around every DCGS2 update pass (time_kind 1) or every
  // phi-cycle operator application (2), so bench.py can report the live per-launch
  // bandwidth of the dominant kernel
  int time_kind = 0;
  std::vector<cudaEvent_t> upd_events;
  size_t upd_used = 0;
  double upd_ms() const;
  bool fused_ok(const OpDevice& op) const;
  void fetch_control(cudaStream_t s);  // host-stepped loops: action, phase, j and stopped to st_host
  // Set when the context belongs to a slab-partitioned group: every reducing
  // kernel is followed by a sum-allreduce of PhiState::loc -> PhiState::red; the
  // control stays in the CUDA graphs when the communicator's collectives are kernels
  // (peer memory), else runs host-stepped (NCCL, host-staged group).
  Comm* comm = nullptr;
  void reduce(cudaStream_t s);
  explicit Engine(int device);
  ~Engine();
  int device = 0;
  int num_sms = 148;
  cudaStream_t stream = nullptr;

  // workspace
  long long ld = 0;
  int slots = 0;
  long long cur_len = -1;
  double* base = nullptr;      // slots * ld
  PhiState* st = nullptr;
  PhiState* st_host = nullptr;  // pinned mirror
  double* partials = nullptr;
  double* ework = nullptr;     // expm workspace
  size_t ework_doubles = 0;
  double* scratch = nullptr;   // 2 vectors of ld: R and a spare
  long long scratch_ld = 0;
  int scratch_count = 0;

  void ensure(long long len, int mmax);
  void ensure_scratch(long long len, int count);
  double* slot(int i) const { return base + (size_t)i * ld; }

  // Host-computed configuration for a phi call (proj/src/phi.cpp:133-183).
  PhiState config(long long n, int p, double dt, const expdg_krylov_cfg& kc) const;
  void upload_config(const PhiState& cfg, cudaStream_t s);

  // Kernel sequences.
  void launch_phi_init(cudaStream_t s, const BArgs& b);
  void launch_ts(cudaStream_t s, int mode);
  double bench_ts(long long n, int k, int mode, int reps);
  // mmax: the phi call's basis bound (decides whether the DCGS2 dots pass can be left
  // out entirely because the operator kernel takes the dots of every column)
  // hact / hj: the action and column of this cycle when the host knows them (host-stepped
  // loops read them back after every cycle, fetch_control): kernels that would no-op are
  // not launched, and neither are their allreduces (slab-partitioned runs); -1: unknown
  void launch_body(cudaStream_t s, OpDevice& op, const BArgs& b, cudaGraphConditionalHandle h,
                   int use_graph, bool dcgs, int mmax, int hact = -1, int hj = -1);
  long long body_launches = 0;  // kernels launch_body enqueued (host-stepped launch accounting)
  // kernels one launch_body enqueues
  static int body_kernels(const OpDevice& op, bool dcgs, int mmax, bool pipe = false);
  // Runs one phi call to completion; host-stepped or graph-driven control.
  void run_phi(OpDevice& op, const BArgs& b, int use_graph);
  // Builds a while-node graph around launch_body; caller owns the exec.
  cudaGraphExec_t build_phi_graph(OpDevice& op, const BArgs& b);
};

// DCGS2 kernels (dcgs.cu): which 0 dots pass (no-op for columns j <= fused_jmax), 1 coefficients,
// 2 update pass.
void launch_dcgs(cudaStream_t s, Engine& e, int which, int fused_jmax = -1);

// Halo send buffers <- first / last element layer of the slot the next phi-cycle apply
// reads (slab-partitioned operators).
void launch_pack_slot(cudaStream_t s, const PhiState* st, const double* base, long long layer, long long last,
                      double* lo, double* hi);

// Small utility kernels.
void launch_axpy_into(cudaStream_t s, double* u, const double* w, long long n);  // u += w
void launch_copy(cudaStream_t s, double* dst, const double* src, long long n);

}  // namespace expdg
