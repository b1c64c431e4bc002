// C ABI of the B200 exponential-DG hot path (include/expdg_b200.h).
// Maps the reference's exception types onto status codes.
#include <chrono>
#include <algorithm>
#include <cmath>
#include <cstring>
#include <memory>
#include <string>
#include <vector>

#include "krylov.cuh"

namespace expdg {
void host_initial_condition(int cfg, int nx, int order, uint64_t seed, double noise, double* out);
void launch_step_begin(cudaStream_t s, PhiState* st, const double* dt_seq);
void launch_step_finish(cudaStream_t s, PhiState* st, double* u, const double* w, int mode, StepRecord* rec,
                        double* partials, int grid);
void launch_absmax(cudaStream_t s, const double* u, long long n, double* out2, int grid);
void launch_step_decide(cudaStream_t s, PhiState* st, StepRecord* rec);
void launch_phi_config(cudaStream_t s, PhiState* st, const double* dt_seq, int p, double mult, int mmax,
                       int full_orth, int window, int grow_cap, int dcgs);
void launch_vec_add(cudaStream_t s, const PhiState* st, double* out, const double* u, const double* w, long long n);
void launch_exprb_d2(cudaStream_t s, const PhiState* st, const double* dt_seq, double* d, const double* a,
                     const double* b, double c, long long n);
int op_check_ref(OpDevice& op, cudaStream_t s, const double* ref);  // 0 ok, 1 not finite, 2 inadmissible
void device_expm(cudaStream_t s, double* work, int N, double* out);

struct Unsupported : std::invalid_argument {
  using std::invalid_argument::invalid_argument;
};
struct KrylovFailure : std::runtime_error {
  double estimate;
  KrylovFailure(const std::string& w, double e) : std::runtime_error(w), estimate(e) {}
};
}  // namespace expdg

using namespace expdg;

struct expdg_local_group {
  std::shared_ptr<LocalGroup> g;
};

struct expdg_peer_group {
  std::shared_ptr<PeerGroup> g;
};

struct expdg_ctx {
  std::unique_ptr<Comm> comm;  // declared before eng: destroyed after it
  std::unique_ptr<Engine> eng;
  long long launches = 0;
  double last_loop_ms = 0.0;
  double* udev = nullptr;  // staging for expdg_integrate_host
  long long udev_len = 0;
  double* work2 = nullptr;  // small reduction buffer
  cudaEvent_t ev0 = nullptr, ev1 = nullptr;
  // integrate's per-call buffers, kept across calls: a pinned allocation per call cost
  // ~40 ms of host time (the e2e path calls integrate once per step)
  int* stop_host = nullptr;   // pinned: the lagged early-exit flag
  cudaEvent_t chunk_ev = nullptr;
  double* dts_dev = nullptr;  // dt sequence
  StepRecord* rec_dev = nullptr;
  long long steps_cap = 0;
  std::shared_ptr<PeerExport> peer_export;  // this rank's exported peer region, until attach
  // engine path of the last phi / integrate call (expdg_ctx_last_path)
  int last_path[4] = {0, 0, 0, 0};
};

struct expdg_op {
  expdg_ctx* ctx = nullptr;
  std::unique_ptr<OpDevice> dev;
  double* ref_owned = nullptr;
};

namespace {

thread_local std::string g_err;

template <class F>
int guard(F&& f) {
  try {
    f();
    return EXPDG_OK;
  } catch (const Unsupported& e) {
    g_err = e.what();
    return EXPDG_E_UNSUPPORTED;
  } catch (const std::invalid_argument& e) {
    g_err = e.what();
    return EXPDG_E_INVALID;
  } catch (const std::domain_error& e) {
    g_err = e.what();
    return EXPDG_E_DOMAIN;
  } catch (const KrylovFailure& e) {
    g_err = e.what();
    return EXPDG_E_KRYLOV;
  } catch (const CommError& e) {
    g_err = e.what();
    return EXPDG_E_COMM;
  } catch (const CudaError& e) {
    g_err = e.what();
    return EXPDG_E_CUDA;
  } catch (const std::exception& e) {
    g_err = e.what();
    return EXPDG_E_CUDA;
  }
}

cudaStream_t pick(expdg_op* op, void* stream) {
  return stream ? static_cast<cudaStream_t>(stream) : op->ctx->eng->stream;
}

bool use_graph_default() {
  const char* e = std::getenv("EXPDG_HOST_CONTROL");
  return !(e && e[0] == '1');
}

void validate_desc(const expdg_op_desc& d) {
  if (d.kind < EXPDG_BURGERS1D || d.kind > EXPDG_EULER3D) throw std::invalid_argument("unknown operator kind");
  if (d.order < 1 || d.order > 20) throw std::invalid_argument("lgl_basis: order must be in [1, 20]");
  if (d.order > 8) throw Unsupported("device operators support orders 1..8");
  if (d.nx < 1 || ((d.kind == EXPDG_BURGERS2D || d.kind == EXPDG_EULER2D) && d.ny < 1) ||
      (d.kind == EXPDG_EULER3D && (d.ny < 1 || d.nz < 1)))
    throw std::invalid_argument("need at least one element per axis");
  if (!(d.x0 < d.x1)) throw std::invalid_argument("degenerate interval");
  // build_quad_mesh: "degenerate box" (proj/src/mesh.cpp:99)
  if (d.kind != EXPDG_BURGERS1D && !(d.y0 < d.y1)) throw std::invalid_argument("degenerate box");
  if (d.kind == EXPDG_EULER3D && !(d.z0 < d.z1)) throw std::invalid_argument("degenerate box");
  if (d.kind == EXPDG_BURGERS1D || d.kind == EXPDG_BURGERS2D) {
    if (!(d.kappa > 0.0)) throw std::invalid_argument("BurgersOperator: kappa must be positive");
    if (d.sigma < 0.0) throw std::invalid_argument("BurgersOperator: sigma must be nonnegative");
    if (d.over_integrate && d.kind == EXPDG_BURGERS2D)
      throw Unsupported("over-integrated 2D Burgers is not on the device path");
  } else {
    if (!d.periodic) throw std::invalid_argument("EulerOperator: periodic boundaries only");
    if (d.euler_flux != 1 && d.kind == EXPDG_EULER3D)
      throw Unsupported("3D Euler: Lax-Friedrichs flux only (the Roe flux is 2D, proj/src/euler.cpp:114-145)");
  }
  if (d.kind == EXPDG_BURGERS1D && d.grade_x)
    throw Unsupported("1D Burgers: the interval mesh has uniform breakpoints (proj/src/mesh.cpp:41-94)");
  if ((d.kind == EXPDG_BURGERS1D || d.kind == EXPDG_BURGERS2D || d.kind == EXPDG_EULER2D) && d.grade_z)
    throw std::invalid_argument("grade_z: 3D meshes only");
  host_axis_breaks(d.x0, d.x1, d.nx, d.grade_x);  // throws on a bad grading list
  if (d.kind != EXPDG_BURGERS1D) host_axis_breaks(d.y0, d.y1, d.ny, d.grade_y);
  if (d.kind == EXPDG_EULER3D) host_axis_breaks(d.z0, d.z1, d.nz, d.grade_z);
  if (d.part_end > d.part_begin) {
    const int layers = d.kind == EXPDG_BURGERS1D ? d.nx : (d.kind == EXPDG_EULER3D ? d.nz : d.ny);
    if (d.part_begin < 0 || d.part_end > layers) throw std::invalid_argument("slab partition: layers out of range");
    if (d.kind == EXPDG_BURGERS1D && d.part_end - d.part_begin < (d.over_integrate ? 2 : 1))
      throw std::invalid_argument("slab partition: over-integrated Burgers needs two elements per rank");
  } else if (d.part_begin != 0 || d.part_end != 0) {
    throw std::invalid_argument("slab partition: empty row range");
  }
}

void map_phi_status(const PhiState& s) {
  switch (s.status) {
    case PHI_OK: return;
    case PHI_ERR_BUDGET: throw KrylovFailure("phi_combination: no convergence within substep budget", s.last_estimate);
    case PHI_ERR_NONFINITE: throw KrylovFailure("phi_combination: non-finite input", s.last_estimate);
    case PHI_ERR_UNDERFLOW: throw KrylovFailure("phi_combination: substep underflow", s.last_estimate);
    case PHI_ERR_DOMAIN: throw std::domain_error("EulerOperator: inadmissible reference state");
    default: throw CudaError("phi engine: controller did not finish (status " + std::to_string(s.status) + ")");
  }
}

// The engine takes "distributed" from the context's communicator: a whole-mesh or dense
// operator on a context whose communicator spans several ranks would have its
// Gram-Schmidt sums allreduced over replicated data (and its phi tail dropped on ranks
// > 0).  Refuse the combination instead of computing a wrong phi.
void check_pair(const expdg_ctx* ctx, const expdg_op* op) {
  if (op->ctx != ctx) throw std::invalid_argument("operator belongs to another context");
  const bool multi = ctx->comm && ctx->comm->size > 1;
  if (multi && !op->dev->partitioned())
    throw std::invalid_argument("context communicator spans " + std::to_string(ctx->comm->size) +
                                " ranks: the operator must be slab-partitioned (desc.part_begin / part_end)");
  if (op->dev->partitioned() && !ctx->comm)
    throw std::invalid_argument("partitioned operator: attach a communicator to the context first");
}

}  // namespace

extern "C" {

const char* expdg_last_error(void) { return g_err.c_str(); }

int expdg_ctx_create(int device, expdg_ctx** out) {
  return guard([&] {
    auto c = std::make_unique<expdg_ctx>();
    c->eng = std::make_unique<Engine>(device);
    EXPDG_CUDA(cudaMalloc(&c->work2, sizeof(double) * 2 * 4096));
    EXPDG_CUDA(cudaEventCreate(&c->ev0));
    EXPDG_CUDA(cudaEventCreate(&c->ev1));
    *out = c.release();
  });
}

int expdg_ctx_destroy(expdg_ctx* ctx) {
  return guard([&] {
    if (!ctx) return;
    cudaStreamSynchronize(ctx->eng->stream);
    cudaFree(ctx->udev);
    cudaFree(ctx->work2);
    cudaEventDestroy(ctx->ev0);
    cudaEventDestroy(ctx->ev1);
    if (ctx->stop_host) cudaFreeHost(ctx->stop_host);
    if (ctx->chunk_ev) cudaEventDestroy(ctx->chunk_ev);
    cudaFree(ctx->dts_dev);
    cudaFree(ctx->rec_dev);
    delete ctx;
  });
}

void* expdg_ctx_stream(expdg_ctx* ctx) { return ctx ? (void*)ctx->eng->stream : nullptr; }

int expdg_ctx_synchronize(expdg_ctx* ctx) {
  return guard([&] { EXPDG_CUDA(cudaStreamSynchronize(ctx->eng->stream)); });
}

long long expdg_ctx_kernel_launches(expdg_ctx* ctx) { return ctx ? ctx->launches : 0; }
double expdg_ctx_last_loop_ms(expdg_ctx* ctx) { return ctx ? ctx->last_loop_ms : 0.0; }

int expdg_nccl_unique_id(unsigned char out[128]) {
  return guard([&] {
    if (!out) throw std::invalid_argument("null argument");
    nccl_unique_id(out);
  });
}

int expdg_ctx_attach_nccl(expdg_ctx* ctx, const unsigned char unique_id[128], int rank, int size) {
  return guard([&] {
    if (!ctx || !unique_id) throw std::invalid_argument("null argument");
    if (ctx->comm) throw std::invalid_argument("context already has a communicator");
    EXPDG_CUDA(cudaSetDevice(ctx->eng->device));
    ctx->comm = make_nccl_comm(unique_id, rank, size);
    ctx->eng->comm = ctx->comm.get();
  });
}

int expdg_local_group_create(int size, expdg_local_group** out) {
  return guard([&] {
    if (!out) throw std::invalid_argument("null argument");
    auto g = std::make_unique<expdg_local_group>();
    g->g = make_local_group(size);
    *out = g.release();
  });
}

int expdg_local_group_destroy(expdg_local_group* g) {
  return guard([&] { delete g; });
}

int expdg_ctx_attach_local(expdg_ctx* ctx, expdg_local_group* g, int rank) {
  return guard([&] {
    if (!ctx || !g) throw std::invalid_argument("null argument");
    if (ctx->comm) throw std::invalid_argument("context already has a communicator");
    ctx->comm = make_local_comm(g->g, rank);
    ctx->eng->comm = ctx->comm.get();
  });
}

int expdg_peer_group_create(int size, long long halo_doubles, expdg_peer_group** out) {
  return guard([&] {
    if (!out) throw std::invalid_argument("null argument");
    auto g = std::make_unique<expdg_peer_group>();
    g->g = make_peer_group(size, halo_doubles);
    *out = g.release();
  });
}

int expdg_peer_group_destroy(expdg_peer_group* g) {
  return guard([&] { delete g; });
}

int expdg_ctx_attach_peer_local(expdg_ctx* ctx, expdg_peer_group* g, int rank) {
  return guard([&] {
    if (!ctx || !g) throw std::invalid_argument("null argument");
    if (ctx->comm) throw std::invalid_argument("context already has a communicator");
    EXPDG_CUDA(cudaSetDevice(ctx->eng->device));
    ctx->comm = make_peer_comm_local(g->g, rank);
    ctx->eng->comm = ctx->comm.get();
  });
}

int expdg_ctx_peer_export(expdg_ctx* ctx, int size, long long halo_doubles, unsigned char handle_out[64]) {
  return guard([&] {
    if (!ctx || !handle_out) throw std::invalid_argument("null argument");
    if (ctx->comm) throw std::invalid_argument("context already has a communicator");
    EXPDG_CUDA(cudaSetDevice(ctx->eng->device));
    ctx->peer_export = make_peer_export(size, halo_doubles, handle_out);
  });
}

int expdg_ctx_attach_peer(expdg_ctx* ctx, const unsigned char* handles, int rank, int size) {
  return guard([&] {
    if (!ctx || !handles) throw std::invalid_argument("null argument");
    if (ctx->comm) throw std::invalid_argument("context already has a communicator");
    if (!ctx->peer_export) throw std::invalid_argument("call expdg_ctx_peer_export first");
    EXPDG_CUDA(cudaSetDevice(ctx->eng->device));
    ctx->comm = make_peer_comm_ipc(ctx->peer_export, handles, rank, size);
    ctx->eng->comm = ctx->comm.get();
    ctx->peer_export.reset();  // owned by the communicator now
  });
}

int expdg_ctx_set_orthogonalization(expdg_ctx* ctx, int mode) {
  return guard([&] {
    if (!ctx) throw std::invalid_argument("null argument");
    if (mode != EXPDG_ORTH_CGS2 && mode != EXPDG_ORTH_DCGS2 && mode != EXPDG_ORTH_AUTO)
      throw std::invalid_argument("unknown orthogonalization");
    ctx->eng->use_dcgs = mode == EXPDG_ORTH_AUTO ? 1 : (mode == EXPDG_ORTH_DCGS2 ? 2 : 0);
  });
}

int expdg_ctx_set_pipelined(expdg_ctx* ctx, int enable) {
  return guard([&] {
    if (!ctx) throw std::invalid_argument("null argument");
    ctx->eng->use_pipe = enable != 0;
  });
}

int expdg_ctx_set_fused(expdg_ctx* ctx, int enable) {
  return guard([&] {
    if (!ctx) throw std::invalid_argument("null argument");
    ctx->eng->use_fused = enable != 0;
  });
}

int expdg_ctx_comm(const expdg_ctx* ctx, int* rank, int* size) {
  return guard([&] {
    if (!ctx) throw std::invalid_argument("null argument");
    if (rank) *rank = ctx->comm ? ctx->comm->rank : 0;
    if (size) *size = ctx->comm ? ctx->comm->size : 1;
  });
}

int expdg_op_create(expdg_ctx* ctx, const expdg_op_desc* desc, expdg_op** out) {
  return guard([&] {
    if (!ctx || !desc) throw std::invalid_argument("null argument");
    validate_desc(*desc);
    if (desc->part_end > desc->part_begin && !ctx->comm)
      throw std::invalid_argument("partitioned operator: attach a communicator to the context first");
    if (desc->part_end <= desc->part_begin && ctx->comm && ctx->comm->size > 1)
      throw std::invalid_argument("context communicator spans several ranks: the operator must be slab-partitioned");
    EXPDG_CUDA(cudaSetDevice(ctx->eng->device));
    auto op = std::make_unique<expdg_op>();
    op->ctx = ctx;
    switch (desc->kind) {
      case EXPDG_BURGERS1D: op->dev = make_burgers1d(*desc); break;
      case EXPDG_BURGERS2D: op->dev = make_burgers2d(*desc); break;
      case EXPDG_EULER2D: op->dev = make_euler2d(*desc); break;
      case EXPDG_EULER3D: op->dev = make_euler3d(*desc); break;
    }
    op->dev->comm = ctx->comm.get();
    // the grading lists were copied into the operator's width tables
    op->dev->desc.grade_x = op->dev->desc.grade_y = op->dev->desc.grade_z = nullptr;
    *out = op.release();
  });
}

int expdg_dense_op_create(expdg_ctx* ctx, int n, const double* a_host, expdg_op** out) {
  return guard([&] {
    if (!ctx || !a_host || n < 1) throw std::invalid_argument("dense op: bad arguments");
    if (ctx->comm && ctx->comm->size > 1)
      throw std::invalid_argument("dense op: not on a context whose communicator spans several ranks");
    auto op = std::make_unique<expdg_op>();
    op->ctx = ctx;
    op->dev = make_dense(n, a_host);
    *out = op.release();
  });
}

int expdg_user_op_create(expdg_ctx* ctx, long long n, const expdg_user_op_fns* fns, void* user, expdg_op** out) {
  return guard([&] {
    if (!ctx || !fns || !out || n < 1) throw std::invalid_argument("user op: bad arguments");
    if (!fns->apply_linear) throw std::invalid_argument("user op: apply_linear is required");
    if (ctx->comm && ctx->comm->size > 1)
      throw std::invalid_argument("user op: not on a context whose communicator spans several ranks");
    EXPDG_CUDA(cudaSetDevice(ctx->eng->device));
    auto op = std::make_unique<expdg_op>();
    op->ctx = ctx;
    op->dev = make_user(n, *fns, user, ctx->eng->num_sms);
    *out = op.release();
  });
}

int expdg_op_destroy(expdg_op* op) {
  return guard([&] {
    if (!op) return;
    cudaFree(op->ref_owned);
    delete op;
  });
}

long long expdg_op_dim(const expdg_op* op) { return op ? op->dev->n : 0; }

// op_check_ref, max-reduced over the ranks of a partitioned operator (every rank
// then throws or proceeds to the collective freeze together)
static int check_ref(expdg_op* op, cudaStream_t s, const double* ref) {
  int chk = op_check_ref(*op->dev, s, ref);
  if (op->dev->partitioned()) {
    op->ctx->comm->host_barrier();
    int* d = reinterpret_cast<int*>(op->ctx->work2);
    EXPDG_CUDA(cudaMemcpyAsync(d, &chk, sizeof(int), cudaMemcpyHostToDevice, s));
    op->ctx->comm->allreduce(d, d, 1, COMM_I32, COMM_MAX, s);
    EXPDG_CUDA(cudaMemcpyAsync(&chk, d, sizeof(int), cudaMemcpyDeviceToHost, s));
    EXPDG_CUDA(cudaStreamSynchronize(s));
  }
  return chk;
}

int expdg_op_linearize(expdg_op* op, const double* ref_dev) {
  return guard([&] {
    if (!op || !ref_dev) throw std::invalid_argument("null argument");
    cudaStream_t s = op->ctx->eng->stream;
    const int chk = check_ref(op, s, ref_dev);
    if (chk == 1) throw std::invalid_argument("reference state not finite");
    if (chk == 2) throw std::domain_error("EulerOperator: inadmissible reference state");
    if (!op->ref_owned) EXPDG_CUDA(cudaMalloc(&op->ref_owned, sizeof(double) * op->dev->n));
    if (op->dev->partitioned()) op->ctx->comm->host_barrier();
    EXPDG_CUDA(cudaMemcpyAsync(op->ref_owned, ref_dev, sizeof(double) * op->dev->n, cudaMemcpyDeviceToDevice, s));
    op->dev->freeze(s, op->ref_owned);
    // the caller may release ref_dev on return: finish reading it
    EXPDG_CUDA(cudaStreamSynchronize(s));
  });
}

int expdg_op_set_source(expdg_op* op, const double* weak_source_dev) {
  return guard([&] {
    if (!op || !weak_source_dev) throw std::invalid_argument("null argument");
    op->dev->set_source(op->ctx->eng->stream, weak_source_dev);
    EXPDG_CUDA(cudaStreamSynchronize(op->ctx->eng->stream));
  });
}

int expdg_op_set_source_fn(expdg_op* op, double (*source)(double x, void* user), void* user) {
  return guard([&] {
    if (!op || !source) throw std::invalid_argument("null argument");
    const expdg_op_desc& d = op->dev->desc;
    if (d.kind != EXPDG_BURGERS1D) throw std::invalid_argument("source terms are 1D Burgers only");
    std::vector<double> wg((size_t)d.nx * (d.order + 1));
    host_burgers_source(d.order, d.nx, d.x0, d.x1, d.over_integrate != 0, source, user, wg.data());
    const size_t off = (size_t)(d.part_end > d.part_begin ? d.part_begin : 0) * (d.order + 1);
    std::vector<double> w(wg.begin() + off, wg.begin() + off + (size_t)op->dev->n);  // owned elements
    cudaStream_t s = op->ctx->eng->stream;
    double* tmp = nullptr;
    EXPDG_CUDA(cudaMallocAsync(&tmp, sizeof(double) * w.size(), s));
    EXPDG_CUDA(cudaMemcpyAsync(tmp, w.data(), sizeof(double) * w.size(), cudaMemcpyHostToDevice, s));
    op->dev->set_source(s, tmp);
    EXPDG_CUDA(cudaFreeAsync(tmp, s));
    EXPDG_CUDA(cudaStreamSynchronize(s));
  });
}

static int apply_common(expdg_op* op, int which, const double* x, double* y, void* stream) {
  return guard([&] {
    if (!op || !x || !y) throw std::invalid_argument("null argument");
    if (which != 2 && !op->dev->ref && op->dev->desc.kind != EXPDG_DENSE)
      throw std::invalid_argument("operator not linearized (call expdg_op_linearize)");
    cudaStream_t s = pick(op, stream);
    // work queued on the context stream (linearize) precedes the caller's stream
    if (stream) EXPDG_CUDA(cudaStreamSynchronize(op->ctx->eng->stream));
    op->dev->launch_apply(s, which, x, y);
    op->ctx->launches++;
    EXPDG_CUDA(cudaGetLastError());
    // NULL stream: the context stream, completed before return (no ordering with
    // the caller's streams is implied otherwise)
    if (!stream) EXPDG_CUDA(cudaStreamSynchronize(s));
  });
}

int expdg_op_apply_linear(expdg_op* op, const double* x_dev, double* y_dev, void* stream) {
  return apply_common(op, 0, x_dev, y_dev, stream);
}
int expdg_op_apply_nonlinear(expdg_op* op, const double* x_dev, double* y_dev, void* stream) {
  return apply_common(op, 1, x_dev, y_dev, stream);
}
int expdg_op_full_rhs(expdg_op* op, const double* x_dev, double* y_dev, void* stream) {
  return apply_common(op, 2, x_dev, y_dev, stream);
}

int expdg_phi_combination(expdg_ctx* ctx, expdg_op* op, const double* const* b_dev, int p, double dt,
                          const expdg_krylov_cfg* cfg, double* out_dev, expdg_krylov_stats* stats) {
  return guard([&] {
    if (!ctx || !op || !b_dev || !cfg || !out_dev) throw std::invalid_argument("null argument");
    if (p < 0) throw std::invalid_argument("phi_combination: empty b list");
    if (p > kMaxP) throw Unsupported("phi_combination: p > 4");
    if (!(dt > 0.0)) throw std::invalid_argument("phi_combination: dt must be positive");
    if (cfg->max_basis > kMaxBasis) throw Unsupported("phi_combination: max_basis > 128");
    if (cfg->max_basis < 1) throw std::invalid_argument("phi_combination: max_basis must be positive");
    check_pair(ctx, op);
    if (!op->dev->ref && op->dev->desc.kind != EXPDG_DENSE)
      throw std::invalid_argument("operator not linearized (call expdg_op_linearize)");
    Engine& e = *ctx->eng;
    const long long n = op->dev->n;
    PhiState c = e.config(n, p, dt, *cfg);
    e.ensure(n + p, c.mmax);
    c = e.config(n, p, dt, *cfg);
    c.max_steps = 1;
    e.upload_config(c, e.stream);
    BArgs b{};
    b.p = p;
    for (int i = 0; i <= p; ++i) b.b[i] = b_dev[i];
    const long long bl0 = e.body_launches;
    ctx->last_path[0] = c.dcgs ? (e.use_pipe ? 2 : 1) : 0;
    ctx->last_path[1] = c.dcgs && op->dev->fused_dcgs_dots_jmax() >= c.mmax;
    ctx->last_path[2] = use_graph_default() && (!e.comm || e.comm->graph_capturable()) && !e.fused_ok(*op->dev) &&
                        op->dev->graph_capturable();
    ctx->last_path[3] = e.fused_ok(*op->dev) ? 1 : 0;
    if (e.comm) e.comm->host_barrier();
    e.run_phi(*op->dev, b, use_graph_default() ? 1 : 0);
    EXPDG_CUDA(cudaMemcpy(e.st_host, e.st, sizeof(PhiState), cudaMemcpyDeviceToHost));
    const PhiState& s = *e.st_host;
    const long long hosted = e.body_launches - bl0;  // host-stepped cycles count their launches
    ctx->launches += 2 + (hosted > 0 ? hosted
                                     : s.body_runs * Engine::body_kernels(*op->dev, s.dcgs != 0, s.mmax,
                                                                          s.dcgs && e.use_pipe));
    if (stats) {
      stats->iterations = s.iterations;
      stats->substeps = s.substeps;
      stats->last_estimate = s.last_estimate;
    }
    map_phi_status(s);
    EXPDG_CUDA(cudaMemcpyAsync(out_dev, e.slot(0), sizeof(double) * n, cudaMemcpyDeviceToDevice, e.stream));
    EXPDG_CUDA(cudaStreamSynchronize(e.stream));
    if (e.comm) e.comm->check();
  });
}

__global__ void k_scale_columns(const PhiState* st, const double* base, long long ld, long long n, int cols,
                                double* out) {
  const long long stride = (long long)gridDim.x * blockDim.x;
  for (int c = 0; c < cols; ++c) {
    const double sc = st->scale[c];
    const double* src = base + (size_t)c * ld;
    double* dst = out + (size_t)c * n;
    for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride) dst[i] = sc * src[i];
  }
}

int expdg_krylov_build(expdg_ctx* ctx, expdg_op* op, const double* seed_dev, int m, int orth_length,
                       double* basis_dev, double* hessenberg_host, double* seed_norm, int* m_out,
                       int* invariant) {
  return guard([&] {
    if (!ctx || !op || !seed_dev) throw std::invalid_argument("null argument");
    if (m < 1) throw std::invalid_argument("krylov_build: m must be positive");
    if (m > kMaxBasis) throw Unsupported("krylov_build: m > 128");
    check_pair(ctx, op);
    if (!op->dev->ref && op->dev->desc.kind != EXPDG_DENSE)
      throw std::invalid_argument("operator not linearized (call expdg_op_linearize)");
    Engine& e = *ctx->eng;
    const long long n = op->dev->n;
    // the plain operator (p = 0: no augmentation, dt = 1), m columns from the seed, then stop
    // (proj/src/phi.cpp:115-130); CGS2 so every column is final in its own cycle
    const expdg_krylov_cfg kc{1e-12, m, orth_length, m, 1};
    e.ensure(n, m);
    PhiState c = e.config(n, 0, 1.0, kc);
    c.mmax = m;
    c.initial_basis = m;
    c.full_orth = orth_length >= m ? 1 : 0;
    c.window = c.full_orth ? m : std::max(1, orth_length);
    c.grow_cap = m;
    c.dcgs = 0;
    c.build_only = 1;
    c.max_steps = 1;
    e.upload_config(c, e.stream);
    BArgs b{};
    b.p = 0;
    b.b[0] = seed_dev;
    const int fused_saved = e.use_fused;
    e.use_fused = 0;
    const long long bl0 = e.body_launches;
    try {
      e.run_phi(*op->dev, b, use_graph_default() ? 1 : 0);
    } catch (...) {
      e.use_fused = fused_saved;
      throw;
    }
    e.use_fused = fused_saved;
    EXPDG_CUDA(cudaMemcpy(e.st_host, e.st, sizeof(PhiState), cudaMemcpyDeviceToHost));
    const PhiState& st = *e.st_host;
    const long long hosted = e.body_launches - bl0;
    ctx->launches += 2 + (hosted > 0 ? hosted : st.body_runs * Engine::body_kernels(*op->dev, false, st.mmax));
    if (!(st.red.bnorm2[0] > 0.0)) throw std::invalid_argument("krylov_build: zero seed");
    map_phi_status(st);
    const int built = st.mc;
    if (m_out) *m_out = built;
    if (invariant) *invariant = st.breakdown;
    if (seed_norm) *seed_norm = st.beta;
    if (hessenberg_host)
      for (int i = 0; i <= built; ++i)
        for (int j = 0; j < built; ++j) hessenberg_host[(size_t)i * built + j] = st.H[(size_t)i * kMaxBasis + j];
    if (basis_dev) {
      const int cols = built + (st.breakdown ? 0 : 1);
      k_scale_columns<<<std::min<long long>(1184, (n + 255) / 256), 256, 0, e.stream>>>(e.st, e.base, e.ld, n, cols,
                                                                                      basis_dev);
      ctx->launches++;
      EXPDG_CUDA(cudaGetLastError());
    }
    EXPDG_CUDA(cudaStreamSynchronize(e.stream));
  });
}

int expdg_step_epi2(expdg_ctx* ctx, expdg_op* op, double* u_dev, double dt, const expdg_krylov_cfg* cfg,
                    expdg_krylov_stats* stats) {
  return guard([&] {
    if (!ctx || !op || !u_dev || !cfg) throw std::invalid_argument("null argument");
    check_pair(ctx, op);
    Engine& e = *ctx->eng;
    const long long n = op->dev->n;
    if (!op->dev->ref && op->dev->desc.kind != EXPDG_DENSE) {
      if (expdg_op_linearize(op, u_dev) != EXPDG_OK) {
        const std::string m = g_err;
        if (m.find("inadmissible") != std::string::npos) throw std::domain_error(m);
        throw std::invalid_argument(m);
      }
    }
    e.ensure_scratch(n, 2);
    double* r = e.scratch;
    double* t = e.scratch + e.scratch_ld;
    // r = L u + N u (proj/src/integrators.cpp:79)
    op->dev->launch_apply(e.stream, 0, u_dev, r);
    if (op->dev->desc.kind != EXPDG_DENSE) {
      op->dev->launch_apply(e.stream, 1, u_dev, t);
      launch_axpy_into(e.stream, r, t, n);
    }
    ctx->launches += 3;
    const double* b[2] = {nullptr, r};
    expdg_krylov_stats st{};
    const int rc = expdg_phi_combination(ctx, op, b, 1, dt, cfg, t, &st);
    if (stats) *stats = st;
    if (rc == EXPDG_E_KRYLOV) throw KrylovFailure(g_err, st.last_estimate);
    if (rc != EXPDG_OK) throw CudaError(g_err);
    launch_axpy_into(e.stream, u_dev, t, n);
    ctx->launches++;
    EXPDG_CUDA(cudaStreamSynchronize(e.stream));
  });
}

// TimeLoopConfig::on_step from the stream: the step's record is copied to pinned memory
// behind the step's kernels, then a host function hands it to the callback in step order
struct OnStepFeed {
  void (*fn)(int, double, double, long long, void*) = nullptr;
  void* user = nullptr;
  StepRecord* rec = nullptr;  // pinned, one per step
  const double* tcum = nullptr;
  bool blown = false;
};
struct OnStepItem {
  OnStepFeed* feed;
  int idx;
};
static void CUDART_CB on_step_host(void* p) {
  const OnStepItem& it = *static_cast<OnStepItem*>(p);
  OnStepFeed& f = *it.feed;
  if (f.blown) return;
  const StepRecord& r = f.rec[it.idx];
  if (r.status) {  // the failing step: no callback (proj/src/integrators.cpp:186-197)
    f.blown = true;
    return;
  }
  f.fn(it.idx + 1, f.tcum[it.idx], r.amax, r.iterations_cum, f.user);
}

static void restore_ref(OpDevice& dev, cudaStream_t s, const double* saved) {
  if (saved) dev.freeze(s, saved);
  else dev.ref = nullptr;
}

static void integrate_impl(expdg_ctx* ctx, expdg_op* op, double* u, const expdg_time_cfg* cfg,
                           expdg_integration_result* res, long long* iters, double* amaxs, int cap) {
  // EXPDG_TIMING=1: host wall-clock phases of the call on stderr (diagnostics)
  static const bool timing = std::getenv("EXPDG_TIMING") && std::getenv("EXPDG_TIMING")[0] == '1';
  auto tclk = std::chrono::steady_clock::now();
  auto tmark = [&](const char* what) {
    if (!timing) return;
    const auto now = std::chrono::steady_clock::now();
    std::fprintf(stderr, "[integrate] %-24s %8.3f ms\n", what,
                 std::chrono::duration<double, std::milli>(now - tclk).count());
    tclk = now;
  };
  if (!ctx || !op || !u || !cfg || !res) throw std::invalid_argument("null argument");
  if (!(cfg->dt > 0.0)) throw std::invalid_argument("integrate: dt must be positive");
  if (cfg->t_final < cfg->dt) throw std::invalid_argument("integrate: t_final must be at least dt");
  const int kind = cfg->integrator;
  if (kind < EXPDG_EXP_EULER || kind > EXPDG_EXPRB42) throw Unsupported("integrate: device integrators are "
                                                                        "exp_euler, epi2, exprb32, exprb42");
  if (cfg->krylov.max_basis > kMaxBasis) throw Unsupported("max_basis > 128");
  check_pair(ctx, op);
  Engine& e = *ctx->eng;
  OpDevice& dev = *op->dev;
  const long long n = dev.n;
  const bool exprb = kind == EXPDG_EXPRB32 || kind == EXPDG_EXPRB42;
  // dt sequence of proj/src/integrators.cpp:155-157
  std::vector<double> dts;
  {
    double t = 0.0;
    const double t_end = cfg->t_final * (1.0 - 1e-14);
    while (t < t_end) {
      const double dt = std::min(cfg->dt, cfg->t_final - t);
      dts.push_back(dt);
      t += dt;
    }
  }
  const int S = (int)dts.size();
  const int pmax = exprb ? 3 : 1;
  e.ensure(n + pmax, std::max(e.config(n, 1, cfg->dt, cfg->krylov).mmax, e.config(n, pmax, cfg->dt, cfg->krylov).mmax));
  const PhiState c1 = e.config(n, 1, cfg->dt, cfg->krylov);  // after ensure: carries the slot stride
  e.ensure_scratch(n, 6);
  double* sb[6];
  for (int i = 0; i < 6; ++i) sb[i] = e.scratch + (size_t)i * e.scratch_ld;
  double* rbuf = sb[0];    // R (EPI2 / EXPRB) or N(u) (exp_euler)
  double* refbuf = sb[1];  // exp_euler: frozen u0
  double* nu = sb[2];      // EXPRB: N(u)
  double* stage = sb[3];   // EXPRB: u + w1
  double* ns = sb[4];      // EXPRB: N(u + w1)
  double* d2 = sb[5];      // EXPRB: c/dt^2 (N(u + w1) - N(u))
  // max|u0| -> blow-up scale (proj/src/integrators.cpp:148-149)
  const int rgrid = std::min(4096, std::max(1, (int)std::min<long long>(e.num_sms * 4, (n + 255) / 256)));
  launch_absmax(e.stream, u, n, ctx->work2, rgrid);
  std::vector<double> h2(2 * rgrid);
  EXPDG_CUDA(cudaMemcpyAsync(h2.data(), ctx->work2, sizeof(double) * 2 * rgrid, cudaMemcpyDeviceToHost, e.stream));
  EXPDG_CUDA(cudaStreamSynchronize(e.stream));
  double max0 = 0.0;
  for (int i = 0; i < rgrid; ++i) max0 = std::max(max0, h2[2 * i]);
  if (e.comm) e.comm->host_barrier();  // every rank past its allocations before the first collective
  // partitioned: max over ranks (host value staged through a device double)
  auto global_max = [&](double v) {
    if (!e.comm) return v;
    EXPDG_CUDA(cudaMemcpyAsync(ctx->work2, &v, sizeof(double), cudaMemcpyHostToDevice, e.stream));
    e.comm->allreduce(ctx->work2, ctx->work2, 1, COMM_F64, COMM_MAX, e.stream);
    EXPDG_CUDA(cudaMemcpyAsync(&v, ctx->work2, sizeof(double), cudaMemcpyDeviceToHost, e.stream));
    EXPDG_CUDA(cudaStreamSynchronize(e.stream));
    return v;
  };
  max0 = global_max(max0);
  // the first linearisation of a non-finite Burgers state throws invalid_argument out of
  // integrate (proj/src/burgers.cpp:34-35; integrate only converts KrylovError /
  // domain_error, proj/src/integrators.cpp:179-183); Euler reports it as a domain error
  // (blew_up at step 1) through the residual's admissibility test
  {
    double nonfinite = 0.0;
    for (int i = 0; i < rgrid; ++i) nonfinite = std::max(nonfinite, h2[2 * i + 1]);
    nonfinite = global_max(nonfinite);
    const int k = dev.desc.kind;
    if (nonfinite > 0.0 && (k == EXPDG_BURGERS1D || k == EXPDG_BURGERS2D))
      throw std::invalid_argument("BurgersOperator: reference state not finite");
  }
  if (kind == EXPDG_EXP_EULER) {
    const int chk = (int)global_max((double)op_check_ref(dev, e.stream, u));
    if (chk == 2) throw std::domain_error("EulerOperator: inadmissible reference state");
    EXPDG_CUDA(cudaMemcpyAsync(refbuf, u, sizeof(double) * n, cudaMemcpyDeviceToDevice, e.stream));
  }
  tmark("setup + absmax check");
  PhiState c = c1;
  c.max_steps = S;
  c.blow_up_scale = 1e10 * (1.0 + max0);
  e.upload_config(c, e.stream);
  if (ctx->steps_cap < S) {
    cudaFree(ctx->dts_dev);
    cudaFree(ctx->rec_dev);
    ctx->dts_dev = nullptr;
    ctx->rec_dev = nullptr;
    ctx->steps_cap = 0;
    const long long cap2 = std::max<long long>(S, 64);
    EXPDG_CUDA(cudaMalloc(&ctx->dts_dev, sizeof(double) * cap2));
    EXPDG_CUDA(cudaMalloc(&ctx->rec_dev, sizeof(StepRecord) * cap2));
    ctx->steps_cap = cap2;
  }
  if (!ctx->stop_host) EXPDG_CUDA(cudaMallocHost(&ctx->stop_host, sizeof(int) * 2));
  if (!ctx->chunk_ev) EXPDG_CUDA(cudaEventCreateWithFlags(&ctx->chunk_ev, cudaEventDisableTiming));
  double* dts_dev = ctx->dts_dev;
  StepRecord* rec_dev = ctx->rec_dev;
  EXPDG_CUDA(cudaMemcpyAsync(dts_dev, dts.data(), sizeof(double) * S, cudaMemcpyHostToDevice, e.stream));
  const double* saved_ref = dev.ref;
  if (kind == EXPDG_EXP_EULER) dev.freeze(e.stream, refbuf);
  else dev.ref = u;  // re-frozen at u^n by the residual kernel every step

  // ---- the step as segments: pre, {phi, mid}..., post
  BArgs b1{}, b2{};
  b1.p = 1;
  b1.b[0] = kind == EXPDG_EXP_EULER ? u : nullptr;
  b1.b[1] = rbuf;
  b2.p = 3;
  b2.b[1] = rbuf;
  b2.b[3] = d2;
  const PhiState c3 = e.config(n, 3, cfg->dt, cfg->krylov);
  const double mult1 = kind == EXPDG_EXPRB42 ? 0.75 : 1.0;         // proj/src/integrators.cpp:106
  const double dcoef = kind == EXPDG_EXPRB42 ? 32.0 / 9.0 : 2.0;  // :97 / :111
  const int vgrid = 1184;
  auto pre = [&](cudaStream_t s) {
    launch_step_begin(s, e.st, dts_dev);
    if (kind == EXPDG_EXP_EULER) {
      dev.launch_apply(s, 1, u, rbuf);  // N(u) at the frozen u0 (proj/src/integrators.cpp:71)
    } else {
      dev.launch_residual(s, u, rbuf, e.st, e.partials);  // R = L u + N u at u~ = u
      if (e.comm) e.comm->allreduce(&e.st->domain_flag, &e.st->domain_flag, 1, COMM_I32, COMM_MAX, s);
      if (exprb) {
        dev.launch_apply(s, 1, u, nu);
        launch_phi_config(s, e.st, dts_dev, 1, mult1, c1.mmax, c1.full_orth, c1.window, c1.grow_cap, c1.dcgs);
      }
    }
    e.launch_phi_init(s, b1);
  };
  auto mid = [&](cudaStream_t s) {
    launch_vec_add(s, e.st, stage, u, e.slot(0), n);
    dev.launch_apply(s, 1, stage, ns);
    launch_exprb_d2(s, e.st, dts_dev, d2, ns, nu, dcoef, n);
    launch_phi_config(s, e.st, dts_dev, 3, 1.0, c3.mmax, c3.full_orth, c3.window, c3.grow_cap, c3.dcgs);
    e.launch_phi_init(s, b2);
  };
  const int fgrid = std::min(2048, std::max(1, (int)std::min<long long>(e.num_sms * 4, (n + 255) / 256)));
  auto post = [&](cudaStream_t s) {
    launch_step_finish(s, e.st, u, e.slot(0), kind == EXPDG_EXP_EULER ? 1 : 0, rec_dev, e.partials, fgrid);
    if (e.comm) {  // blow-up test on the max over ranks
      e.comm->allreduce(e.st->mx, e.st->mx, 2, COMM_F64, COMM_MAX, s);
      launch_step_decide(s, e.st, rec_dev);
    }
  };
  (void)vgrid;
  const bool fused = e.fused_ok(dev);
  const int per_step = (exprb ? 13 : 5) + (e.comm ? 1 : 0) + (fused ? (exprb ? 2 : 1) : 0);
  const bool pipe = c1.dcgs && e.use_pipe;
  const int body_k = Engine::body_kernels(dev, c1.dcgs != 0, exprb ? std::max(c1.mmax, c3.mmax) : c1.mmax, pipe) +
                     (dev.partitioned() ? (pipe ? 2 : 1) : 0);  // + halo pack kernel(s)
  cudaGraphExec_t ex = nullptr;
  // partitioned runs keep the graphs with the peer-memory communicator (kernel collectives), run
  // host-stepped over NCCL / the host-staged group; user operators only when graph-safe
  const bool graph = cfg->use_graph != 0 && (!e.comm || e.comm->graph_capturable()) && dev.graph_capturable();
  // host callbacks must not see the states after a blow-up: look at `stopped` after every step
  const bool check_each_step = !dev.graph_capturable();
  ctx->last_path[0] = c1.dcgs ? (e.use_pipe ? 2 : 1) : 0;
  ctx->last_path[1] = c1.dcgs && dev.fused_dcgs_dots_jmax() >= (exprb ? std::max(c1.mmax, c3.mmax) : c1.mmax);
  ctx->last_path[2] = graph ? 1 : 0;
  ctx->last_path[3] = fused ? 1 : 0;
  int launched = 0;

  // Adds a WHILE node after the current capture position; returns its body graph.
  auto add_while = [&](cudaStream_t cs, cudaGraph_t g, cudaGraphConditionalHandle* h) {
    EXPDG_CUDA(cudaGraphConditionalHandleCreate(h, g, 1, cudaGraphCondAssignDefault));
    cudaStreamCaptureStatus cst;
    const cudaGraphNode_t* deps = nullptr;
    size_t ndeps = 0;
    cudaGraph_t cg;
    EXPDG_CUDA(cudaStreamGetCaptureInfo(cs, &cst, nullptr, &cg, &deps, &ndeps));
    cudaGraphNodeParams cp = {};
    cp.type = cudaGraphNodeTypeConditional;
    cp.conditional.handle = *h;
    cp.conditional.type = cudaGraphCondTypeWhile;
    cp.conditional.size = 1;
    cudaGraphNode_t cnode;
    EXPDG_CUDA(cudaGraphAddNode(&cnode, g, deps, ndeps, &cp));
    EXPDG_CUDA(cudaStreamUpdateCaptureDependencies(cs, &cnode, 1, cudaStreamSetCaptureDependencies));
    return cp.conditional.phGraph_out[0];
  };
  const long long bl0 = e.body_launches;
  auto host_loop = [&](const BArgs& b, bool dcgs, int mmax) {
    int hact = -1, hj = -1;  // the first cycle after phi init: unknown, launch every kernel
    for (long long cyc = 0;; ++cyc) {
      e.launch_body(e.stream, dev, b, cudaGraphConditionalHandle{}, 0, dcgs, mmax, hact, hj);
      e.fetch_control(e.stream);  // action, phase, j + stopped only (not the whole PhiState)
      if (e.st_host->action == ACT_DONE || e.st_host->action == ACT_NONE || e.st_host->stopped) break;
      hact = e.st_host->action;
      hj = e.st_host->j;
      if (cyc > 10000000) throw CudaError("host-stepped phi did not terminate");
    }
  };
  try {
    if (graph) {
      cudaGraph_t g;
      EXPDG_CUDA(cudaGraphCreate(&g, 0));
      cudaStream_t cs;
      EXPDG_CUDA(cudaStreamCreateWithFlags(&cs, cudaStreamNonBlocking));
      EXPDG_CUDA(cudaStreamBeginCaptureToGraph(cs, g, nullptr, nullptr, 0, cudaStreamCaptureModeRelaxed));
      pre(cs);
      if (fused) {  // small problem: each phi call is one fused kernel node
        dev.launch_fused(cs, e, b1);
        if (exprb) {
          mid(cs);
          dev.launch_fused(cs, e, b2);
        }
        post(cs);
        EXPDG_CUDA(cudaStreamEndCapture(cs, &g));
      } else {
        cudaGraphConditionalHandle h1, h2;
        cudaGraph_t body1 = add_while(cs, g, &h1), body2 = nullptr;
        if (exprb) {
          mid(cs);
          body2 = add_while(cs, g, &h2);
        }
        post(cs);
        EXPDG_CUDA(cudaStreamEndCapture(cs, &g));
        EXPDG_CUDA(cudaStreamBeginCaptureToGraph(cs, body1, nullptr, nullptr, 0, cudaStreamCaptureModeRelaxed));
        e.launch_body(cs, dev, b1, h1, 1, c1.dcgs != 0, c1.mmax);
        EXPDG_CUDA(cudaStreamEndCapture(cs, &body1));
        if (exprb) {
          EXPDG_CUDA(cudaStreamBeginCaptureToGraph(cs, body2, nullptr, nullptr, 0, cudaStreamCaptureModeRelaxed));
          e.launch_body(cs, dev, b2, h2, 1, c3.dcgs != 0, c3.mmax);
          EXPDG_CUDA(cudaStreamEndCapture(cs, &body2));
        }
      }
      EXPDG_CUDA(cudaGraphInstantiate(&ex, g, 0));
      tmark("graph capture + instantiate");
      cudaGraphDestroy(g);
      cudaStreamDestroy(cs);
    }
    // snapshots and on_step, enqueued behind each step
    const int snap_every = cfg->snapshot_every > 0 ? cfg->snapshot_every : 0;
    int snaps_taken = 0;
    std::vector<double> tcum(S);
    for (int i = 0; i < S; ++i) tcum[i] = (i ? tcum[i - 1] : 0.0) + dts[i];
    OnStepFeed feed;
    std::vector<OnStepItem> items;
    StepRecord* rec_pinned = nullptr;
    if (cfg->on_step) {
      EXPDG_CUDA(cudaMallocHost(&rec_pinned, sizeof(StepRecord) * S));
      feed.fn = cfg->on_step;
      feed.user = cfg->on_step_user;
      feed.rec = rec_pinned;
      feed.tcum = tcum.data();
      items.resize(S);
      for (int i = 0; i < S; ++i) items[i] = OnStepItem{&feed, i};
    }
    // pending host functions read feed / items / rec_pinned: drain the stream before they go
    // (also when an exception unwinds this scope)
    struct PinnedFree {
      StepRecord*& p;
      cudaStream_t s;
      ~PinnedFree() {
        if (p) {
          cudaStreamSynchronize(s);
          cudaFreeHost(p);
        }
      }
    } pinned_free{rec_pinned, e.stream};
    auto after_step = [&](int idx) {
      if (snap_every && (idx + 1) % snap_every == 0) {
        if (snaps_taken < cfg->snapshot_cap && cfg->snapshots)
          EXPDG_CUDA(cudaMemcpyAsync(cfg->snapshots + (size_t)snaps_taken * n, u, sizeof(double) * n,
                                     cudaMemcpyDefault, e.stream));
        ++snaps_taken;
      }
      if (cfg->on_step) {
        EXPDG_CUDA(cudaMemcpyAsync(rec_pinned + idx, rec_dev + idx, sizeof(StepRecord), cudaMemcpyDeviceToHost,
                                   e.stream));
        EXPDG_CUDA(cudaLaunchHostFunc(e.stream, on_step_host, &items[idx]));
      }
    };
    if (e.comm) e.comm->host_barrier();  // every rank's graph and buffers ready before the loop
    // lagged early-exit check: launch in chunks, look at `stopped` of the chunk before
    int* stop_host = ctx->stop_host;
    stop_host[0] = stop_host[1] = 0;
    cudaEvent_t chunk_ev = ctx->chunk_ev;
    EXPDG_CUDA(cudaEventRecord(ctx->ev0, e.stream));
    const int chunk = 32;
    bool pending = false;
    while (launched < S) {
      const int cnt = std::min(chunk, S - launched);
      for (int i = 0; i < cnt; ++i) {
        if (graph) {
          EXPDG_CUDA(cudaGraphLaunch(ex, e.stream));
          after_step(launched + i);
        } else {
          pre(e.stream);
          if (fused) dev.launch_fused(e.stream, e, b1);
          else host_loop(b1, c1.dcgs != 0, c1.mmax);
          if (exprb) {
            mid(e.stream);
            if (fused) dev.launch_fused(e.stream, e, b2);
            else host_loop(b2, c3.dcgs != 0, c3.mmax);
          }
          post(e.stream);
          after_step(launched + i);
          if (check_each_step) {
            EXPDG_CUDA(cudaMemcpyAsync(stop_host, &e.st->stopped, sizeof(int), cudaMemcpyDeviceToHost, e.stream));
            EXPDG_CUDA(cudaStreamSynchronize(e.stream));
            if (stop_host[0]) {
              launched += i + 1;
              goto steps_done;
            }
          }
        }
      }
      launched += cnt;
      if (pending) {
        EXPDG_CUDA(cudaEventSynchronize(chunk_ev));
        if (stop_host[0]) break;
      }
      EXPDG_CUDA(cudaMemcpyAsync(stop_host, &e.st->stopped, sizeof(int), cudaMemcpyDeviceToHost, e.stream));
      EXPDG_CUDA(cudaEventRecord(chunk_ev, e.stream));
      pending = true;
    }
  steps_done:
    EXPDG_CUDA(cudaEventRecord(ctx->ev1, e.stream));
    EXPDG_CUDA(cudaStreamSynchronize(e.stream));
    if (e.comm) e.comm->check();
    float ms = 0.f;
    EXPDG_CUDA(cudaEventElapsedTime(&ms, ctx->ev0, ctx->ev1));
    ctx->last_loop_ms = ms;
    tmark("step loop");
  } catch (...) {
    if (ex) cudaGraphExecDestroy(ex);
    restore_ref(dev, e.stream, saved_ref);
    throw;
  }
  if (ex) cudaGraphExecDestroy(ex);
  restore_ref(dev, e.stream, saved_ref);
  EXPDG_CUDA(cudaMemcpy(e.st_host, e.st, sizeof(PhiState), cudaMemcpyDeviceToHost));
  const PhiState st = *e.st_host;
  ctx->launches += (long long)launched * per_step +
                   (fused ? 0 : (graph ? st.body_runs * body_k : e.body_launches - bl0));
  std::vector<StepRecord> rec(std::max(1, st.step));
  if (st.step > 0)
    EXPDG_CUDA(cudaMemcpy(rec.data(), rec_dev, sizeof(StepRecord) * st.step, cudaMemcpyDeviceToHost));
  tmark("teardown + readback");
  res->steps = st.step;
  res->status = 0;
  res->blow_up_step = -1;
  res->max_abs = max0;
  res->t = 0.0;
  for (int i = 0; i < st.step; ++i) res->t += dts[i];
  for (int i = 0; i < st.step; ++i) {
    if (rec[i].status) {
      res->status = 1;
      res->blow_up_step = i + 1;
      break;
    }
    res->max_abs = std::max(res->max_abs, rec[i].amax);
    if (i < cap) {
      if (iters) iters[i] = rec[i].iterations_cum;
      if (amaxs) amaxs[i] = rec[i].amax;
    }
  }
  res->krylov_iterations = st.iterations_total;
  // snapshots of completed, non-failing steps only (the reference stops before pushing one)
  const int ok_steps = res->status ? res->blow_up_step - 1 : res->steps;
  res->snapshots = cfg->snapshot_every > 0 ? ok_steps / cfg->snapshot_every : 0;
  if (cfg->snapshot_times)
    for (int k = 0; k < std::min(res->snapshots, cfg->snapshot_cap); ++k)
      cfg->snapshot_times[k] = k < S ? [&] {
        double t = 0.0;
        for (int i = 0; i < (k + 1) * cfg->snapshot_every; ++i) t += dts[i];
        return t;
      }() : 0.0;
}

int expdg_integrate(expdg_ctx* ctx, expdg_op* op, double* u_dev, const expdg_time_cfg* cfg,
                    expdg_integration_result* res, long long* iters_per_step, double* amax_per_step, int cap) {
  return guard([&] { integrate_impl(ctx, op, u_dev, cfg, res, iters_per_step, amax_per_step, cap); });
}

int expdg_integrate_host(expdg_ctx* ctx, expdg_op* op, double* u_host, const expdg_time_cfg* cfg,
                         expdg_integration_result* res, long long* iters_per_step, double* amax_per_step,
                         int cap) {
  return guard([&] {
    if (!ctx || !op || !u_host) throw std::invalid_argument("null argument");
    Engine& e = *ctx->eng;
    const long long n = op->dev->n;
    if (ctx->udev_len < n) {
      cudaFree(ctx->udev);
      ctx->udev = nullptr;
      EXPDG_CUDA(cudaMalloc(&ctx->udev, sizeof(double) * n));
      ctx->udev_len = n;
    }
    EXPDG_CUDA(cudaMemcpyAsync(ctx->udev, u_host, sizeof(double) * n, cudaMemcpyHostToDevice, e.stream));
    integrate_impl(ctx, op, ctx->udev, cfg, res, iters_per_step, amax_per_step, cap);
    EXPDG_CUDA(cudaMemcpyAsync(u_host, ctx->udev, sizeof(double) * n, cudaMemcpyDeviceToHost, e.stream));
    EXPDG_CUDA(cudaStreamSynchronize(e.stream));
  });
}

int expdg_expm(expdg_ctx* ctx, int n, const double* a_host, double* out_host) {
  return guard([&] {
    if (!ctx || n < 1 || n > kMaxBasis + 2) throw std::invalid_argument("expm: 1 <= n <= 130");
    Engine& e = *ctx->eng;
    double* out = nullptr;
    EXPDG_CUDA(cudaMalloc(&out, sizeof(double) * n * n));
    EXPDG_CUDA(cudaMemcpyAsync(e.ework, a_host, sizeof(double) * n * n, cudaMemcpyHostToDevice, e.stream));
    device_expm(e.stream, e.ework, n, out);
    ctx->launches++;
    EXPDG_CUDA(cudaMemcpyAsync(out_host, out, sizeof(double) * n * n, cudaMemcpyDeviceToHost, e.stream));
    EXPDG_CUDA(cudaStreamSynchronize(e.stream));
    cudaFree(out);
  });
}

int expdg_ctx_last_path(expdg_ctx* ctx, int* out4) {
  return guard([&] {
    if (!ctx || !out4) throw std::invalid_argument("null argument");
    std::memcpy(out4, ctx->last_path, sizeof(ctx->last_path));
  });
}

int expdg_debug_state(expdg_ctx* ctx, double* out16) {
  return guard([&] {
    Engine& e = *ctx->eng;
    EXPDG_CUDA(cudaMemcpy(e.st_host, e.st, sizeof(PhiState), cudaMemcpyDeviceToHost));
    const PhiState& s = *e.st_host;
    const double v[16] = {(double)s.mc, s.h, s.t, s.beta, s.avnorm, s.last_estimate, (double)s.substeps,
                          (double)s.iterations, (double)s.breakdown, (double)s.status, (double)s.mmax,
                          (double)s.grow_cap, (double)s.full_orth, (double)s.cycles, s.pre_norm, (double)s.m};
    std::memcpy(out16, v, sizeof(v));
  });
}

int expdg_ctx_time_dominant(expdg_ctx* ctx, int enable) {
  return guard([&] {
    if (!ctx) throw std::invalid_argument("null argument");
    if (enable < 0 || enable > 2) throw std::invalid_argument("time_dominant: 0 off, 1 update pass, 2 apply");
    ctx->eng->time_kind = enable;
    ctx->eng->upd_used = 0;
    EXPDG_CUDA(cudaMemsetAsync(reinterpret_cast<char*>(ctx->eng->st) + offsetof(PhiState, upd_bytes), 0,
                               2 * (sizeof(double) + sizeof(long long)), ctx->eng->stream));
    EXPDG_CUDA(cudaStreamSynchronize(ctx->eng->stream));
  });
}

int expdg_ctx_dominant_stats(expdg_ctx* ctx, double* out3) {
  return guard([&] {
    if (!ctx || !out3) throw std::invalid_argument("null argument");
    Engine& e = *ctx->eng;
    EXPDG_CUDA(cudaMemcpy(e.st_host, e.st, sizeof(PhiState), cudaMemcpyDeviceToHost));
    out3[0] = e.upd_ms();
    const bool app = e.time_kind == 2;
    out3[1] = app ? e.st_host->app_bytes : e.st_host->upd_bytes;
    out3[2] = (double)(app ? e.st_host->app_launches : e.st_host->upd_launches);
  });
}

int expdg_debug_profile(expdg_ctx* ctx, long long* out8) {
  return guard([&] {
    if (!ctx || !out8) throw std::invalid_argument("null argument");
    EXPDG_CUDA(cudaMemcpy(ctx->eng->st_host, ctx->eng->st, sizeof(PhiState), cudaMemcpyDeviceToHost));
    for (int i = 0; i < 8; ++i) out8[i] = ctx->eng->st_host->prof[i];
  });
}

int expdg_debug_expm_profile(expdg_ctx* ctx, long long* out8) {
  return guard([&] {
    if (!ctx || !out8) throw std::invalid_argument("null argument");
    EXPDG_CUDA(cudaMemcpy(ctx->eng->st_host, ctx->eng->st, sizeof(PhiState), cudaMemcpyDeviceToHost));
    for (int i = 0; i < 8; ++i) out8[i] = ctx->eng->st_host->xprof[i];
  });
}

int expdg_ctx_traffic(expdg_ctx* ctx, double* out4) {
  return guard([&] {
    Engine& e = *ctx->eng;
    EXPDG_CUDA(cudaMemcpy(e.st_host, e.st, sizeof(PhiState), cudaMemcpyDeviceToHost));
    const PhiState& s = *e.st_host;
    out4[0] = s.alg_bytes;
    out4[1] = (double)s.extend_cols;
    out4[2] = (double)s.avnorms;
    out4[3] = (double)s.combines;
  });
}

int expdg_bench_ts(expdg_ctx* ctx, long long n, int k, int mode, int reps, double* ms) {
  return guard([&] {
    if (k < 1 || k > kMaxBasis) throw std::invalid_argument("bench_ts: 1 <= k <= 128");
    *ms = ctx->eng->bench_ts(n, k, mode, reps);
  });
}

// Times one phi-cycle operator application at column j (mode 0; with the DCGS2 dots
// when the operator takes them) or the separate DCGS2 dots pass at column j (mode 1),
// on the current slots; diagnostics for the fused sweep.  The operator must be linearized.
int expdg_bench_apply(expdg_ctx* ctx, expdg_op* op, int j, int mode, int reps, double* ms) {
  return guard([&] {
    if (j < 0 || j >= kMaxBasis) throw std::invalid_argument("bench_apply: 0 <= j < 128");
    if (!op->dev->ref) throw std::invalid_argument("operator not linearized (call expdg_op_linearize)");
    Engine& e = *ctx->eng;
    const long long n = op->dev->n;
    e.ensure(n + 1, j + 3);
    e.ensure_scratch(n + 1, 1);
    EXPDG_CUDA(cudaMemsetAsync(e.scratch, 0, sizeof(double) * (n + 1), e.stream));
    PhiState c = e.config(n, 1, 1e-3, expdg_krylov_cfg{1e-10, std::max(j + 1, 1), std::max(j + 1, 1), 0, 0});
    c.dcgs = 1;
    c.pl_look = mode == 2 ? 1 : 0;  // mode 2: the pipelined DCGS2 lookahead application (stage 2)
    c.action = ACT_EXTEND;
    c.j = j;
    c.mc = j + 1;
    for (int i = 0; i < kMaxSlots; ++i) c.scale[i] = 1.0;
    e.upload_config(c, e.stream);
    BArgs b{};
    b.p = 1;
    b.b[1] = e.scratch;
    auto one = [&] {
      if (mode == 0) op->dev->launch_phi_apply(e.stream, e.st, e.base, e.partials, b);
      else if (mode == 2) op->dev->launch_phi_apply(e.stream, e.st, e.base + e.ld, e.partials, b, 2);
      else launch_dcgs(e.stream, e, 0, -1);
    };
    one();  // warm-up
    cudaEvent_t a, z;
    EXPDG_CUDA(cudaEventCreate(&a));
    EXPDG_CUDA(cudaEventCreate(&z));
    EXPDG_CUDA(cudaEventRecord(a, e.stream));
    for (int r = 0; r < reps; ++r) one();
    EXPDG_CUDA(cudaEventRecord(z, e.stream));
    EXPDG_CUDA(cudaEventSynchronize(z));
    float t = 0.f;
    EXPDG_CUDA(cudaEventElapsedTime(&t, a, z));
    cudaEventDestroy(a);
    cudaEventDestroy(z);
    EXPDG_CUDA(cudaGetLastError());
    *ms = t / reps;
  });
}

int expdg_debug_hessenberg(expdg_ctx* ctx, double* out /* (kMaxBasis+1) x kMaxBasis */) {
  return guard([&] {
    Engine& e = *ctx->eng;
    EXPDG_CUDA(cudaMemcpy(e.st_host, e.st, sizeof(PhiState), cudaMemcpyDeviceToHost));
    std::memcpy(out, e.st_host->H, sizeof(e.st_host->H));
  });
}

int expdg_lgl_basis(int order, double* nodes, double* weights, double* diff) {
  return guard([&] {
    const HostBasis b = host_lgl_basis(order);
    const int n = order + 1;
    std::memcpy(nodes, b.nodes.data(), sizeof(double) * n);
    std::memcpy(weights, b.weights.data(), sizeof(double) * n);
    std::memcpy(diff, b.D.data(), sizeof(double) * n * n);
  });
}

int expdg_initial_condition_slab(int config, int nx, int ny, int nz, int order, const double* box6,
                                 int layer_begin, int layer_end, double* out_host) {
  return guard([&] {
    if (!out_host || !box6) throw std::invalid_argument("initial_condition_slab: null argument");
    if (config != 5) throw Unsupported("initial_condition_slab: config 5 (the z-partitioned Taylor-Green) only");
    if (order < 1 || order > 20) throw std::invalid_argument("lgl_basis: order must be in [1, 20]");
    host_tgv_slab(nx, ny, nz, order, box6, layer_begin, layer_end, out_host);
  });
}

int expdg_initial_condition(int config, int nx, int order, uint64_t seed, double noise, double* out_host) {
  return guard([&] {
    if (nx < 1 || !out_host) throw std::invalid_argument("initial_condition: bad arguments");
    host_initial_condition(config, nx, order, seed, noise, out_host);
  });
}

}  // extern "C"
