// Internal device/host definitions of the B200 exponential-DG engine.
//
// Layout in HBM:
//   * fields: element-major, then component, then node (x fastest), exactly the
//     reference FieldState layout (proj/include/expdg/mesh.hpp:61-80);
//   * Krylov basis: (mmax + 2) slots of `ld` doubles, slot 0 doubles as the
//     running phi vector w (proj/src/phi.cpp:160-165, :227-237), slot i >= 1 holds
//     V_i UNNORMALISED with a per-slot scale s_i (V_i = s_i * slot_i), so no
//     normalisation pass is ever streamed; `ld` is padded to a multiple of
//     kLdAlign with zeros so every tall-skinny tile is a full TMA bulk copy;
//   * the p augmentation scalars of the phi vector sit at [n, n+p) of every slot.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include <cmath>
#include <cstdio>
#include <stdexcept>
#include <string>

#include "expdg_b200.h"

namespace expdg {

constexpr int kMaxBasis = 128;            // proj/include/expdg/phi.hpp:47 default
constexpr int kMaxSlots = kMaxBasis + 2;  // V_0..V_mmax plus one scratch slot
constexpr int kMaxP = 4;                  // b_0..b_4 (integrators use p <= 3)
constexpr int kTailPad = 8;               // [n, n+8) is the tail region of a slot
constexpr long long kLdAlign = 2048;      // largest tall-skinny tile (doubles)
constexpr int kTsThreads = 256;
constexpr int kMaxPartials = 2048;        // max CTAs contributing partial sums

enum Action : int {
  ACT_NONE = 0,
  ACT_START = 1,    // phi vector initialised: controller computes beta and resets
  ACT_EXTEND = 2,   // Arnoldi column j: y = A V_j, orthogonalise (CGS2 / IOP)
  ACT_AVNORM = 3,   // ||A V_mc|| (proj/src/phi.cpp:195-199)
  ACT_COMBINE = 4,  // w = V_{0:mc} (beta f(0:mc, 0))  (proj/src/phi.cpp:227)
  ACT_DONE = 5,
};

enum Phase : int { PH_SUBSTEP = 0, PH_POST = 1, PH_DECIDE = 2, PH_DONE = 3, PH_EXTEND = 4 };

enum PhiStatus : int {
  PHI_RUNNING = 0,
  PHI_OK = 1,
  PHI_ERR_BUDGET = 2,     // proj/src/phi.cpp:186-188
  PHI_ERR_NONFINITE = 3,  // proj/src/phi.cpp:191-192
  PHI_ERR_UNDERFLOW = 4,  // proj/src/phi.cpp:252-253
  PHI_ERR_DOMAIN = 5,     // inadmissible Euler state (proj/src/euler.cpp:210-211)
  PHI_ERR_CYCLES = 6,     // safety valve: controller cycle budget exhausted
};

// Device-resident state of one phi_combination call (and of the step around it).
struct PhiState {
  // ---- configuration (host-written at call setup)
  long long n;       // local head length
  long long len;     // n + p (the p-scalar tail is replicated on every rank)
  long long ld;      // slot stride
  int p;
  int tail_here;     // this rank counts the tail in reductions (rank 0)
  double dt;
  double tol;
  int mmax, window, grow_cap, max_substeps, full_orth, initial_basis;
  int max_cycles;
  int build_only;    // krylov_build: stop after the Arnoldi columns (no avnorm / expm / combine)
  int pipe_cfg;      // pipelined DCGS2 allowed (see pl_direct / pl_look)
  int pipe_restart;  // diagnostics: apply the operator directly to every pipe_restart-th candidate
  int ts3_stages;    // merged pass: stage cap after the tile choice (0: the tile rule's cap)
  int ts3_tstages;   // merged pass: stages the tile choice assumes (0: the tall-skinny rule's)
  int ts3_pow2;      // merged pass: power-of-two tiles only (EXPDG_TS3_POW2=1, diagnostics)
  double* base;      // slot 0 of the Krylov workspace (stage-1 operator applications)
  // ---- dynamic control (action, phase, j, pl_direct, pl_look: read back together by
  // host-stepped loops, Engine::fetch_control)
  int action, phase, j;
  // Pipelined DCGS2 (dcgs.cu k_ts3): the merged pass of column j also builds the next
  // candidate's operator image by the Arnoldi relation from a lookahead application
  // dt A (slot j+1) written to slot j+2, plus the next column's pass-1 dots, so V is
  // streamed once per column.  Per cycle:
  //   pl_direct  stage-1 application dt A (s_j slot_j) -> slot j+1 and the pass-1 dots run
  //              (substep start, after a grow, CGS2 / IOP); 0: slot j+1 and the dots come
  //              from the previous cycle's merged pass
  //   pl_look    stage-2 (lookahead) application dt A (s_j slot_{j+1}) -> slot j+2 and the
  //              merged pass instead of the plain update pass
  int pl_direct, pl_look;
  int pl_ready;      // column whose W (slot j+1) and pass-1 dots the last merged pass left (-1: none)
  int j0, k;
  int target, m, mc, breakdown, status;
  long long iterations;  // this call
  int substeps;          // this call
  int cycles;
  double beta, avnorm, t, h, last_estimate, pre_norm;
  // ---- reduced results of the last kernels.  Single rank: the kernels' grid
  // reductions land in `red` directly.  Slab-partitioned (multi = 1): they land
  // in `loc` (this rank's partial sums) and the host enqueues a sum-allreduce
  // loc -> red after every reducing kernel (idempotent when a kernel no-ops).
  struct Red {
    double nrmA;  // ||y||^2 after the operator
    double nrmC;  // ||y||^2 after pass C
    double w2;    // ||w_head||^2 after combine / init
    double dotA[kMaxSlots];
    double dotB[kMaxSlots];
    double bnorm2[kMaxP + 1];
    double nrmU;  // DCGS2: ||reorthogonalised candidate||^2 after the update pass
    double nrmW;  // DCGS2: ||next candidate||^2 after the update pass
  };
  Red red;
  Red loc;
  int multi;
  int pad_multi;
  double mx[2];  // per-step max reductions (max|u|, non-finite flag), allreduced in place
#ifdef __CUDACC__
  __device__ __forceinline__ Red& rs() { return multi ? loc : red; }
#endif
  // ---- per-slot scale and combine coefficients
  double scale[kMaxSlots];
  double comb[kMaxSlots];
  double tailw[kMaxP];
  // ---- DCGS2: classical Gram-Schmidt with the reorthogonalisation of column j-1
  // lagged into the pass that first projects column j (one dots pass + one update
  // pass per column instead of CGS2's three).  Slot j holds the candidate u_j
  // (projected once, scale[j] provisional); the JVP runs on it and the second
  // projection of u_j rides in the same two passes as the first projection of A u_j.
  int dcgs;        // 1: DCGS2 (full orthogonalisation only), 0: CGS2 / IOP passes
  int dots_fused;  // the operator kernel of this cycle also took the DCGS2 pass-1 dots
  int dc_pending;  // the AVNORM cycle already extended column mc provisionally
  double dc_gam;   // slot-space coefficient of the old candidate in the w update
  double dc_c, dc_d, dc_ab;  // <u,u>, <u,w>, a.b (true, scaled)
  double dc_gp;              // gamma used by the update pass (Pythagorean beta)
  double pre_prev;           // ||dt A V_{j-1}|| (the lagged breakdown test, proj/src/phi.cpp:104-108)
  long long dc_fixups;       // Pythagorean vs exact reorthogonalised norm disagreed (diagnostic)
  double dc_wsc;             // W_true = dc_wsc * slot_{j+1} (1 after a stage-1 application, s_j after a merged pass)
  double pl_zy, pl_zw, pl_kj; // merged pass: znew = zy Y - zw W - sum_l kappa_l slot_l - kj unew
  double pl_kappa[kMaxSlots];
  double dc_a[kMaxSlots];      // a_i = <V_i, u>
  double dc_b[kMaxSlots];      // b_i = <V_i, w>
  double dc_g[kMaxSlots];      // (H a)_l with column j-1 corrected, l < j
  double dc_alpha[kMaxSlots];  // slot-space update coefficients of u
  double dc_mu[kMaxSlots];     // slot-space update coefficients of w
  // ---- last-block reduction tickets, one per reducing kernel kind
  unsigned int ticket[16];
  // ---- step-level bookkeeping (integrate)
  int stopped;        // a previous step blew up / finished: every kernel no-ops
  int step;           // steps completed
  int max_steps;
  int domain_flag;    // set by operator kernels on inadmissible states
  int step_failed;    // a phi call of this step failed (KrylovError / domain): skip the rest
  int any_b;          // some b_i nonzero
  long long iterations_total;
  long long body_runs;  // controller invocations (one per engine cycle)
  // canonical algorithmic HBM bytes of the realised trajectory:
  // JVP 32 n per operator application, CGS2 8 n (3k + 6) per column against k
  // vectors, combine 8 n (m + 1) per accepted substep, 40 n per step.
  double alg_bytes;
  long long extend_cols, avnorms, combines;
  double blow_up_scale;
  double amax_step;
  long long prof[8];  // fused engine: SM clock cycles per phase (apply, dots, update, combine, ctl)
  long long xprof[8]; // expm sub-phases (ctl.cuh, EXPM_PROBE)
  double upd_bytes;   // algorithmic bytes of the DCGS2 update passes that ran (8 n (j + 4) each)
  long long upd_launches;
  double app_bytes;   // the same for the Euler 2D strip sweep: 32 n (JVP) + 8 n j (fused dots)
  long long app_launches;
  // ---- Hessenberg (mmax+1) x mmax, row stride kMaxBasis; last, so the controller
  // copies the scalar state plus only the rows in use
  alignas(16) double H[(kMaxBasis + 1) * kMaxBasis];
};

#ifdef __CUDACC__
// Stage of a phi-cycle operator application: 1 = the candidate s_j slot_j -> slot j+1 (base is
// the workspace), 2 = pipelined DCGS2 lookahead s_j slot_{j+1} -> slot j+2 (the engine passes
// base + ld, so every operator kernel's "slot j" / "slot j+1" address the next slots).
__device__ __forceinline__ int apply_stage(const PhiState* st, const double* base) {
  return base == st->base ? 1 : 2;
}
__device__ __forceinline__ bool apply_go(const PhiState* st, const double* base) {
  if (st->stopped) return false;
  if (apply_stage(st, base) == 2) return st->pl_look != 0 && (st->action == ACT_EXTEND || st->action == ACT_AVNORM);
  const int a = st->action;
  return (a == ACT_EXTEND || a == ACT_AVNORM) && st->pl_direct;
}
#endif

// One record per integrate step, read back by the host at the end.
struct StepRecord {
  double t, dt, amax;
  long long iterations_cum;
  int status;  // 0 ok, 1 blew up (KrylovError / domain / non-finite / > scale)
  int substeps;
  int phi_status;
  int pad;
};

// ---------------------------------------------------------------- errors
struct CudaError : std::runtime_error {
  using std::runtime_error::runtime_error;
};
// a communicator (NCCL / local group) call failed
struct CommError : CudaError {
  using CudaError::CudaError;
};

#define EXPDG_CUDA(call)                                                                  \
  do {                                                                                    \
    cudaError_t e_ = (call);                                                              \
    if (e_ != cudaSuccess)                                                                \
      throw ::expdg::CudaError(std::string(#call) + ": " + cudaGetErrorString(e_));      \
  } while (0)

// ---------------------------------------------------------------- device helpers
__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}
__device__ __forceinline__ double warp_max(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = fmax(v, __shfl_xor_sync(0xffffffffu, v, o));
  return v;
}

// Deterministic block sum (fixed tree order).  `buf` needs blockDim/32 doubles.
__device__ __forceinline__ double block_sum(double v, double* buf) {
  v = warp_sum(v);
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  __syncthreads();
  if (lane == 0) buf[wid] = v;
  __syncthreads();
  double s = 0.0;
  if (wid == 0) {
    const int nw = blockDim.x >> 5;
    s = lane < nw ? buf[lane] : 0.0;
    s = warp_sum(s);
  }
  return s;  // valid in thread 0
}

__device__ __forceinline__ double block_max(double v, double* buf) {
  v = warp_max(v);
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  __syncthreads();
  if (lane == 0) buf[wid] = v;
  __syncthreads();
  double s = 0.0;
  if (wid == 0) {
    const int nw = blockDim.x >> 5;
    s = lane < nw ? buf[lane] : 0.0;
    s = warp_max(s);
  }
  return s;
}

// Last-block deterministic grid reduction: every CTA stores `cnt` partial sums
// at partials[blockIdx.x * stride + i]; the CTA that arrives last sums them in
// block order and calls `sink(i, total)`.  Returns true in the last CTA.
template <class Sink>
__device__ __forceinline__ bool grid_reduce_last(const double* mine, int cnt, double* partials,
                                                 int stride, unsigned int* ticket, Sink sink) {
  __shared__ bool s_last;
  for (int i = threadIdx.x; i < cnt; i += blockDim.x) partials[(size_t)blockIdx.x * stride + i] = mine[i];
  __threadfence();
  __syncthreads();
  if (threadIdx.x == 0) {
    const unsigned int prev = atomicAdd(ticket, 1u);
    s_last = (prev == gridDim.x - 1);
  }
  __syncthreads();
  if (!s_last) return false;
  __threadfence();
  for (int i = threadIdx.x; i < cnt; i += blockDim.x) {
    double s = 0.0;
    for (unsigned int b = 0; b < gridDim.x; ++b) s += __ldcg(&partials[(size_t)b * stride + i]);
    sink(i, s);
  }
  __syncthreads();
  if (threadIdx.x == 0) *ticket = 0u;
  return true;
}

// ---------------------------------------------------------------- TMA bulk copy (1D)
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}
__device__ __forceinline__ void fence_mbar_init() {
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void fence_proxy_async() {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}
__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n\t.reg .pred P;\n"
      "WAIT_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 P, [%0], %1;\n\t"
      "@!P bra WAIT_%=;\n}" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ void bulk_g2s(void* dst_smem, const void* src_gmem, uint32_t bytes, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
          smem_u32(dst_smem)),
      "l"(src_gmem), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}

// 8-byte asynchronous copies (for data whose rows are not 16-byte aligned, which 1D TMA
// bulk copies require); cp_async_arrive makes the barrier count one arrival of the
// executing thread once all its prior cp.async copies have landed
__device__ __forceinline__ void cp_async8(void* dst_smem, const void* src_gmem) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(smem_u32(dst_smem)), "l"(src_gmem) : "memory");
}
__device__ __forceinline__ void cp_async_arrive(uint64_t* bar) {
  asm volatile("cp.async.mbarrier.arrive.noinc.shared::cta.b64 [%0];" ::"r"(smem_u32(bar)) : "memory");
}

// named barrier over the 256 consumer threads of a warp-specialised CTA
__device__ __forceinline__ void consumer_sync() { asm volatile("bar.sync 1, 256;" ::: "memory"); }
// named barrier over the CONS consumer threads of a strip kernel (producer warp excluded)
// L2 prefetch of a global range (bytes a multiple of 16, 16-byte aligned)
__device__ __forceinline__ void bulk_prefetch_l2(const void* src_gmem, uint32_t bytes) {
  asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(src_gmem), "r"(bytes) : "memory");
}
template <int CONS>
__device__ __forceinline__ void strip_sync() { asm volatile("bar.sync 1, %0;" ::"n"(CONS) : "memory"); }
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void mbar_arrive_cnt(uint64_t* bar, uint32_t cnt) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(cnt) : "memory");
}

__host__ __device__ inline long long round_up(long long a, long long b) { return (a + b - 1) / b * b; }

}  // namespace expdg
