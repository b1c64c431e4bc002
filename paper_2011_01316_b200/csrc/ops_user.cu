// User operators: any LinearAction (proj/include/expdg/phi.hpp:11) or SplitProblem
// (proj/include/expdg/integrators.hpp:48-52) supplied as C callbacks on device vectors
// drives the device phi engine and time loop (expdg_user_op_create).
//
// The phi-cycle apply is split around the user's action:
//   k_user_gather   x = s_j V_j (head of Krylov slot j) into a fixed scratch vector
//   user callback   y = L x (the user's kernels, on the engine stream)
//   k_user_scatter  slot j+1 = dt (y + sum_i x_tail[i] b_{p-i}) plus the tail, and ||.||^2
// so the callback always sees the same two pointers (a CUDA graph can record it once when
// the user declares it graph-safe).  Both kernels no-op unless the controller's action of
// this cycle applies the operator, exactly like the built-in operator kernels.
#include <algorithm>

#include "krylov.cuh"

namespace expdg {

namespace {

constexpr int kUThreads = 256;

__global__ void __launch_bounds__(kUThreads) k_user_gather(const PhiState* st, const double* base,
                                                           double* __restrict__ x, long long n) {
  if (st->stopped) return;
  if (!apply_go(st, base)) return;
  const double xs = st->scale[st->j];
  const double* src = base + (size_t)st->j * st->ld;
  const long long stride = (long long)gridDim.x * blockDim.x;
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride) x[i] = xs * src[i];
}

// proj/src/phi.cpp:151-158: y = dt (L x + sum_i x_tail[i] b_{p-i}), tail shifted up by one
__global__ void __launch_bounds__(kUThreads) k_user_scatter(PhiState* st, double* base,
                                                            const double* __restrict__ ly, BArgs b,
                                                            double* partials, long long n) {
  __shared__ int s_go, s_j;
  __shared__ double s_dt, s_xt[kMaxP];
  __shared__ long long s_ld;
  __shared__ double s_buf[kUThreads / 32];
  __shared__ double s_red[1];
  if (threadIdx.x == 0) {
    s_go = apply_go(st, base);
    if (s_go) {
      s_j = st->j;
      s_dt = st->dt;
      s_ld = st->ld;
      const double xs = st->scale[s_j];
      const double* xslot = base + (size_t)s_j * st->ld;
      for (int i = 0; i < kMaxP; ++i) s_xt[i] = (i < b.p) ? xslot[n + i] * xs : 0.0;
    }
  }
  __syncthreads();
  if (!s_go) return;
  double* y = base + (size_t)(s_j + 1) * s_ld;
  const double dt = s_dt;
  double nacc = 0.0;
  const long long stride = (long long)gridDim.x * blockDim.x;
  for (long long g = (long long)blockIdx.x * blockDim.x + threadIdx.x; g < n; g += stride) {
    const double v = dt * aug_tail(b, s_xt, (size_t)g, ly[g]);
    y[g] = v;
    nacc = fma(v, v, nacc);
  }
  if (blockIdx.x == 0 && threadIdx.x < kTailPad) {
    const int i = threadIdx.x;
    const double v = (i + 1 < b.p) ? dt * s_xt[i + 1] : 0.0;
    y[n + i] = v;
    nacc = fma(v, v, nacc);
  }
  const double tot = block_sum(nacc, s_buf);
  if (threadIdx.x == 0) s_red[0] = tot;
  __syncthreads();
  grid_reduce_last(s_red, 1, partials, kMaxSlots, &st->ticket[4], [&](int, double v) { st->rs().nrmA = v; });
}

__global__ void k_user_add(double* __restrict__ r, const double* __restrict__ t, long long n) {
  const long long stride = (long long)gridDim.x * blockDim.x;
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride) r[i] += t[i];
}

__global__ void k_user_flag_domain(PhiState* st) {
  if (!st->stopped) st->domain_flag = 1;
}

class UserOp : public OpDevice {
 public:
  expdg_user_op_fns f{};
  void* user = nullptr;
  double* xbuf = nullptr;  // fixed scratch: the callbacks' x
  double* ybuf = nullptr;  // fixed scratch: the callbacks' y
  double* tbuf = nullptr;  // N x of the residual
  int grid = 296;

  UserOp(long long nn, const expdg_user_op_fns& fns, void* u, int num_sms) : f(fns), user(u) {
    desc.kind = EXPDG_USER;
    n = nn;
    comps = 1;
    grid = (int)std::max<long long>(1, std::min<long long>(2LL * num_sms, (n + kUThreads - 1) / kUThreads));
    const size_t bytes = sizeof(double) * (size_t)(n + kTailPad);
    EXPDG_CUDA(cudaMalloc(&xbuf, bytes));
    EXPDG_CUDA(cudaMalloc(&ybuf, bytes));
    EXPDG_CUDA(cudaMalloc(&tbuf, bytes));
    EXPDG_CUDA(cudaMemset(xbuf, 0, bytes));
    EXPDG_CUDA(cudaMemset(ybuf, 0, bytes));
    EXPDG_CUDA(cudaMemset(tbuf, 0, bytes));
    if (!f.linearize) ref = xbuf;  // a plain LinearAction is always "linearised"
  }
  ~UserOp() override {
    cudaFree(xbuf);
    cudaFree(ybuf);
    cudaFree(tbuf);
  }
  bool graph_capturable() const override { return f.graph_safe != 0; }

  // the reference's exceptions from a callback's status code
  static void check(int rc, const char* what) {
    if (rc == EXPDG_OK) return;
    const std::string w = std::string("user operator: ") + what + " returned status " + std::to_string(rc);
    if (rc == EXPDG_E_DOMAIN) throw std::domain_error(w);
    if (rc == EXPDG_E_INVALID) throw std::invalid_argument(w);
    throw CudaError(w);
  }
  void linear(cudaStream_t s, const double* x, double* y) { check(f.apply_linear(x, y, s, user), "apply_linear"); }
  void nonlinear(cudaStream_t s, const double* x, double* y) {
    if (f.apply_nonlinear) check(f.apply_nonlinear(x, y, s, user), "apply_nonlinear");
    else EXPDG_CUDA(cudaMemsetAsync(y, 0, sizeof(double) * (size_t)n, s));
  }

  void freeze(cudaStream_t s, const double* r) override {
    ref = r;
    if (f.linearize) check(f.linearize(r, s, user), "linearize");
  }
  void launch_phi_apply(cudaStream_t s, PhiState* st, double* base, double* partials, const BArgs& b, int stage = 1) override {
    k_user_gather<<<grid, kUThreads, 0, s>>>(st, base, xbuf, n);
    linear(s, xbuf, ybuf);
    k_user_scatter<<<grid, kUThreads, 0, s>>>(st, base, ybuf, b, partials, n);
  }
  void launch_apply(cudaStream_t s, int which, const double* x, double* y) override {
    if (which == 0) {
      linear(s, x, y);
    } else if (which == 1) {
      nonlinear(s, x, y);
    } else {  // full rhs: L(x) x + N(x) x with the split rebuilt at x
      freeze(s, x);
      linear(s, x, y);
      nonlinear(s, x, tbuf);
      k_user_add<<<grid, kUThreads, 0, s>>>(y, tbuf, n);
    }
  }
  // R = L u + N u with the split rebuilt at u^n (proj/src/integrators.cpp:79, :164-170); a
  // domain error of linearize fails the step (blew_up), like the reference's catch
  void launch_residual(cudaStream_t s, const double* u, double* r, PhiState* st, double*) override {
    if (f.linearize) {
      const int rc = f.linearize(u, s, user);
      if (rc == EXPDG_E_DOMAIN) {
        k_user_flag_domain<<<1, 1, 0, s>>>(st);
        return;
      }
      check(rc, "linearize");
    }
    ref = u;
    linear(s, u, r);
    nonlinear(s, u, tbuf);
    k_user_add<<<grid, kUThreads, 0, s>>>(r, tbuf, n);
  }
};

}  // namespace

std::unique_ptr<OpDevice> make_user(long long n, const expdg_user_op_fns& fns, void* user, int num_sms) {
  return std::make_unique<UserOp>(n, fns, user, num_sms);
}

}  // namespace expdg
