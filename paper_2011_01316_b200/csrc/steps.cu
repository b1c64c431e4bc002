// Time-loop kernels of the device integrate() (proj/src/integrators.cpp:140-201):
// per-step dt, the blow-up test and the per-step record ring, so a whole run is
// a sequence of graph launches with no host round-trip.
#include "krylov.cuh"

namespace expdg {

__global__ void k_step_begin(PhiState* st, const double* dt_seq) {
  if (st->stopped) return;
  st->dt = dt_seq[st->step];
  st->domain_flag = 0;
  st->step_failed = 0;
}

// Per-call configuration of the phi calls of an EXPRB step (p and the dt factor
// differ between the two calls, proj/src/integrators.cpp:85-113).
__global__ void k_phi_config(PhiState* st, const double* dt_seq, int p, double mult, int mmax, int full_orth,
                             int window, int grow_cap, int dcgs) {
  if (st->stopped) return;
  st->p = p;
  st->len = st->n + p;
  st->dt = dt_seq[st->step] * mult;
  st->mmax = mmax;
  st->full_orth = full_orth;
  st->window = window;
  st->grow_cap = grow_cap;
  st->dcgs = dcgs;
}

// S = u + w (the EXPRB internal stage, proj/src/integrators.cpp:93 / :108)
__global__ void k_vec_add(const PhiState* st, double* s, const double* u, const double* w, long long n) {
  if (st->stopped || st->step_failed) return;
  const long long stride = (long long)gridDim.x * blockDim.x;
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride) s[i] = u[i] + w[i];
}

// d = (c / (dt*dt)) * (a - b) with dt the step's dt (2/dt^2 for EXPRB32, 32/9/dt^2 for EXPRB42)
__global__ void k_exprb_d2(const PhiState* st, const double* dt_seq, double* d, const double* a, const double* b,
                           double c, long long n) {
  if (st->stopped || st->step_failed) return;
  const double dt = dt_seq[st->step];
  const double f = c / (dt * dt);
  const long long stride = (long long)gridDim.x * blockDim.x;
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride) d[i] = f * (a[i] - b[i]);
}

__device__ void step_decide(PhiState* st, StepRecord* rec, double mx, double bad) {
  const int step = st->step;
  const bool failed = st->step_failed || st->status != PHI_OK;
  const double am = bad > 0.0 ? INFINITY : mx;
  st->alg_bytes += 40.0 * (double)st->n;
  StepRecord r;
  r.dt = st->dt;
  r.t = 0.0;
  r.amax = am;
  r.iterations_cum = st->iterations_total;
  r.substeps = st->substeps;
  r.phi_status = st->status;
  r.pad = 0;
  if (failed || !isfinite(am) || am > st->blow_up_scale) {
    r.status = 1;
    st->stopped = 1;
  } else {
    r.status = 0;
  }
  rec[step] = r;
  st->step = step + 1;
  if (st->step >= st->max_steps) st->stopped = 1;
}

// mode 0 (EPI2): u <- u + w ; mode 1 (exp_euler): u <- w.  Then max|u|, finiteness,
// blow-up test against 1e10 (1 + max|u0|) (proj/src/integrators.cpp:149, :186-193).
__global__ void __launch_bounds__(256) k_step_finish(PhiState* st, double* u, const double* w, int mode,
                                                     StepRecord* rec, double* partials) {
  __shared__ double s_buf[8];
  __shared__ double s_red[2];
  __shared__ int s_ok;
  if (st->stopped) return;
  if (threadIdx.x == 0) s_ok = st->status == PHI_OK && !st->step_failed;
  __syncthreads();
  const bool ok = s_ok;
  const long long n = st->n;
  double amax = 0.0, nonfinite = 0.0;
  const long long stride = (long long)gridDim.x * blockDim.x;
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride) {
    double v = u[i];
    if (ok) {
      v = mode == 0 ? v + w[i] : w[i];
      u[i] = v;
    }
    if (!isfinite(v)) nonfinite = 1.0;
    else amax = fmax(amax, fabs(v));
  }
  const double m = block_max(amax, s_buf);
  const double nf = block_max(nonfinite, s_buf);
  if (threadIdx.x == 0) { s_red[0] = m; s_red[1] = nf; }
  __syncthreads();
  // max-reduction through the sum machinery: encode as partials and take max in the sink
  __shared__ bool s_last;
  for (int i = threadIdx.x; i < 2; i += blockDim.x) partials[(size_t)blockIdx.x * kMaxSlots + i] = s_red[i];
  __threadfence();
  __syncthreads();
  if (threadIdx.x == 0) s_last = atomicAdd(&st->ticket[7], 1u) == gridDim.x - 1;
  __syncthreads();
  if (!s_last) return;
  __threadfence();
  if (threadIdx.x == 0) {
    double mx = 0.0, bad = 0.0;
    for (unsigned int b = 0; b < gridDim.x; ++b) {
      mx = fmax(mx, __ldcg(&partials[(size_t)b * kMaxSlots]));
      bad = fmax(bad, __ldcg(&partials[(size_t)b * kMaxSlots + 1]));
    }
    st->ticket[7] = 0u;
    if (st->multi) {  // partitioned: max-allreduce of st->mx, then k_step_decide
      st->mx[0] = mx;
      st->mx[1] = bad;
    } else {
      step_decide(st, rec, mx, bad);
    }
  }
}

// The blow-up decision on the (rank-reduced) max|u| and non-finite flag.
__global__ void k_step_decide(PhiState* st, StepRecord* rec) {
  if (st->stopped) return;
  step_decide(st, rec, st->mx[0], st->mx[1]);
}

// max|u| (and finiteness) of the initial state.
__global__ void __launch_bounds__(256) k_absmax(const double* u, long long n, double* out2 /* [grid][2] */) {
  __shared__ double s_buf[8];
  double amax = 0.0, nf = 0.0;
  const long long stride = (long long)gridDim.x * blockDim.x;
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride) {
    const double v = u[i];
    if (!isfinite(v)) nf = 1.0;
    else amax = fmax(amax, fabs(v));
  }
  const double m = block_max(amax, s_buf);
  const double f = block_max(nf, s_buf);
  if (threadIdx.x == 0) { out2[2 * blockIdx.x] = m; out2[2 * blockIdx.x + 1] = f; }
}

void launch_step_begin(cudaStream_t s, PhiState* st, const double* dt_seq) { k_step_begin<<<1, 1, 0, s>>>(st, dt_seq); }
void launch_step_finish(cudaStream_t s, PhiState* st, double* u, const double* w, int mode, StepRecord* rec,
                        double* partials, int grid) {
  k_step_finish<<<grid, 256, 0, s>>>(st, u, w, mode, rec, partials);
}
void launch_phi_config(cudaStream_t s, PhiState* st, const double* dt_seq, int p, double mult, int mmax,
                       int full_orth, int window, int grow_cap, int dcgs) {
  k_phi_config<<<1, 1, 0, s>>>(st, dt_seq, p, mult, mmax, full_orth, window, grow_cap, dcgs);
}
void launch_vec_add(cudaStream_t s, const PhiState* st, double* out, const double* u, const double* w, long long n) {
  k_vec_add<<<1184, 256, 0, s>>>(st, out, u, w, n);
}
void launch_exprb_d2(cudaStream_t s, const PhiState* st, const double* dt_seq, double* d, const double* a,
                     const double* b, double c, long long n) {
  k_exprb_d2<<<1184, 256, 0, s>>>(st, dt_seq, d, a, b, c, n);
}
void launch_step_decide(cudaStream_t s, PhiState* st, StepRecord* rec) { k_step_decide<<<1, 1, 0, s>>>(st, rec); }
void launch_absmax(cudaStream_t s, const double* u, long long n, double* out2, int grid) {
  k_absmax<<<grid, 256, 0, s>>>(u, n, out2);
}

}  // namespace expdg
