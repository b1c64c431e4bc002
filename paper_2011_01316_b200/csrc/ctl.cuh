// Device code shared by the multi-kernel engine (krylov.cu) and the fused small-problem
// engines (fused_*.cu): block dense linear algebra and Higham expm, the controller
// (ctl_body), and the fused single-CTA / cluster phi kernels with their launchers.
// Split out so the fused engines' operator instantiations compile in parallel TUs.
#pragma once

#include <cooperative_groups.h>

#include <algorithm>
#include <cstddef>
#include <cstdlib>

#include "fused.cuh"
#include "krylov.cuh"

namespace expdg {

// ------------------------------------------------------------------ block dense linear algebra
// diagnostics (expdg_debug_expm_profile): SM cycles of the expm sub-phases, summed over calls:
// 0 norm + scaling, 1 Pade powers / U / V, 2 LU elimination, 3 back substitution + un-permute,
// 4 squarings, 5 calls, 6 squarings taken
// (PhiState::xprof; xp may be null)
#define EXPM_PROBE(slot, t)                                     \
  if (threadIdx.x == 0 && xp) {                                 \
    const long long now_ = clock64();                           \
    xp[slot] += now_ - (t);                                     \
    (t) = now_;                                                 \
  }
// C = A B out of shared memory: a 2 x 2 register tile per thread (4 loads per 4 FMAs; one
// output per thread is 2 loads per FMA and was load-bound: 2.6k SM cycles at N = 18), four k
// steps of loads in flight, every output summed in k order.
// (an integer division by a run-time divisor is ~200 cycles of dependent latency here: the
// callers pass this thread's first-round indices, formed once per expm)
struct BlkIdx {
  int ti, tj;   // 2 x 2 tile of idx = tid in a row of (N + 1) / 2 tiles
  bool diag;    // idx = tid is a diagonal entry of the N x N matrix
};
static __device__ BlkIdx blk_idx(int N) {
  const int H = (N + 1) / 2, t = threadIdx.x;
  BlkIdx b;
  b.ti = t / H;
  b.tj = t - b.ti * H;
  b.diag = t % (N + 1) == 0;
  return b;
}
static __device__ void blk_matmul(double* C, const double* A, const double* B, int N, const BlkIdx& bx) {
  const int T = blockDim.x, H = (N + 1) / 2, tiles = H * H;
  for (int t = threadIdx.x; t < tiles; t += T) {
    const int ti = t < T ? bx.ti : t / H, tj = t < T ? bx.tj : t - ti * H;
    const int i0 = 2 * ti, j0 = 2 * tj;
    const int i1 = i0 + 1 < N ? i0 + 1 : i0, j1 = j0 + 1 < N ? j0 + 1 : j0;
    const double* a0 = A + i0 * N;
    const double* a1 = A + i1 * N;
    const double* b0 = B + j0;
    const double* b1 = B + j1;
    double c00 = 0.0, c01 = 0.0, c10 = 0.0, c11 = 0.0;
    int k = 0;
    for (; k + 4 <= N; k += 4) {
      double x0[4], x1[4], y0[4], y1[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        x0[u] = a0[k + u];
        x1[u] = a1[k + u];
        y0[u] = b0[(k + u) * N];
        y1[u] = b1[(k + u) * N];
      }
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        c00 = fma(x0[u], y0[u], c00);
        c01 = fma(x0[u], y1[u], c01);
        c10 = fma(x1[u], y0[u], c10);
        c11 = fma(x1[u], y1[u], c11);
      }
    }
    for (; k < N; ++k) {
      const double x0 = a0[k], x1 = a1[k], y0 = b0[k * N], y1 = b1[k * N];
      c00 = fma(x0, y0, c00);
      c01 = fma(x0, y1, c01);
      c10 = fma(x1, y0, c10);
      c11 = fma(x1, y1, c11);
    }
    C[i0 * N + j0] = c00;
    if (j1 != j0) C[i0 * N + j1] = c01;
    if (i1 != i0) {
      C[i1 * N + j0] = c10;
      if (j1 != j0) C[i1 * N + j1] = c11;
    }
  }
  __syncthreads();
}

// out = sum c_m M_m + ident * I
static __device__ void blk_lincomb(double* out, int N, int cnt, const double* c, const double* const* M, double ident,
                                   const BlkIdx& bx) {
  for (int idx = threadIdx.x; idx < N * N; idx += blockDim.x) {
    double s = 0.0;
    for (int m = 0; m < cnt; ++m) s += c[m] * M[m][idx];
    if (idx < (int)blockDim.x ? bx.diag : idx % (N + 1) == 0) s += ident;
    out[idx] = s;
  }
  __syncthreads();
}

// v = sum c_m M_m + ident * I;  num = U + v, den = v - U  (the Pade numerator and denominator)
static __device__ void blk_numden(double* num, double* den, const double* U, int N, int cnt, const double* c,
                                  const double* const* M, double ident, const BlkIdx& bx) {
  for (int idx = threadIdx.x; idx < N * N; idx += blockDim.x) {
    double s = 0.0;
    for (int m = 0; m < cnt; ++m) s += c[m] * M[m][idx];
    if (idx < (int)blockDim.x ? bx.diag : idx % (N + 1) == 0) s += ident;
    const double u = U[idx];
    num[idx] = u + s;
    den[idx] = s - u;
  }
  __syncthreads();
}

// Solves A X = B by LU with partial pivoting (first maximal pivot); A and B are destroyed, X is
// a third N x N array.  One CTA barrier per column in each phase: every warp finds the pivot
// of column k itself (three warp reductions on the bit pattern of |a|), rows are pivoted
// through a double-buffered permutation (no row swaps), the multipliers are applied to B as
// they are formed (never stored) with the pivot reciprocal; the back substitution is
// column-oriented over all threads (x_i = b_i / u_ii, then b_r -= u_ri x_i for r < i) and
// writes X in natural row order.  (History at N = 18, C1: swaps + stored multipliers + four
// barriers per column 53k SM cycles; permutation + two barriers + one thread per column of B
// in the back substitution 36k; this version: tools/c1_profile.py.)
static __device__ void blk_lu_solve(double* __restrict__ A, double* __restrict__ B, double* __restrict__ X, int N,
                                    long long& tp, long long* xp) {
  __shared__ int s_perm[2][kMaxBasis + 2];
  __shared__ double s_inv[kMaxBasis + 2];
  const int tid = threadIdx.x, lane = tid & 31, T = blockDim.x;
  for (int i = tid; i < N; i += T) s_perm[0][i] = i;
  __syncthreads();
  // (row offset, column) of idx = tid and the step to idx + T, without a division per element
  const int q0 = tid / N, j0 = tid - q0 * N, dq = T / N, dj = T - dq * N;
  for (int k = 0; k < N; ++k) {
    const int* perm = s_perm[k & 1];
    int* pnew = s_perm[(k + 1) & 1];
    // pivot of column k among rows i >= k: max |a|, first index on ties
    unsigned long long bits = 0ull;
    int bi = 0x7fffffff;
    for (int i = k + lane; i < N; i += 32) {
      const unsigned long long v = (unsigned long long)__double_as_longlong(fabs(A[perm[i] * N + k]));
      if (bi == 0x7fffffff || v > bits) { bits = v; bi = i; }
    }
    const bool valid = bi != 0x7fffffff;
    const unsigned hi = valid ? (unsigned)(bits >> 32) : 0u;
    const unsigned m1 = __reduce_max_sync(0xffffffffu, hi);
    const bool c1 = valid && hi == m1;
    const unsigned m2 = __reduce_max_sync(0xffffffffu, c1 ? (unsigned)bits : 0u);
    const bool c2 = c1 && (unsigned)bits == m2;
    bi = (int)__reduce_min_sync(0xffffffffu, c2 ? (unsigned)bi : 0x7fffffffu);
    const int pk = perm[k], rk = perm[bi];
    const double inv = 1.0 / A[rk * N + k];
    if (tid == 0) s_inv[k] = inv;
    for (int i = tid; i < N; i += T) pnew[i] = i == k ? rk : (i == bi ? pk : perm[i]);
    // rows below k: l = A[r][k] / A[rk][k]; A[r][j] -= l A[rk][j] (j > k), B[r][j] -= l B[rk][j]
    const int cnt = (N - k - 1) * N;
    int q = q0, j = j0;
    for (int idx = tid; idx < cnt; idx += T) {
      const int ii = k + 1 + q;
      const int r = ii == bi ? pk : perm[ii];
      const double l = A[r * N + k] * inv;
      if (j > k) A[r * N + j] -= l * A[rk * N + j];
      B[r * N + j] -= l * B[rk * N + j];
      q += dq;
      j += dj;
      if (j >= N) { j -= N; ++q; }
    }
    __syncthreads();
  }
  EXPM_PROBE(2, tp);
  const int* perm = s_perm[N & 1];
  for (int i = N - 1; i >= 0; --i) {
    const int ri = perm[i];
    const double inv = s_inv[i];
    const int cnt = (i + 1) * N;
    int q = q0, j = j0;
    for (int idx = tid; idx < cnt; idx += T) {
      const double x = B[ri * N + j] * inv;
      if (q == i) {
        X[i * N + j] = x;
      } else {
        const int r = perm[q];
        B[r * N + j] -= A[r * N + i] * x;
      }
      q += dq;
      j += dj;
      if (j >= N) { j -= N; ++q; }
    }
    __syncthreads();
  }
  EXPM_PROBE(3, tp);
}

// Higham (2005) scaling and squaring, the algorithm of Eigen's MatrixFunctions
// exp() (proj/src/phi.cpp:40).  A (N x N) in W[0]; result in *out (one of W's).
static __device__ double* blk_expm(double* W, int N, long long* xp = nullptr) {
  __shared__ double s_l1;
  __shared__ int s_sq;
  __shared__ double s_buf[32];
  const size_t NN = (size_t)N * N;
  double* A = W;
  double* A2 = W + NN;
  double* A4 = W + 2 * NN;
  double* A6 = W + 3 * NN;
  double* A8 = W + 4 * NN;
  double* U = W + 5 * NN;
  double* V = W + 6 * NN;
  double* T1 = W + 7 * NN;
  double* T2 = W + 8 * NN;
  long long tp = clock64();
  const BlkIdx bx = blk_idx(N);
  // 1-norm
  double colmax = 0.0;
  for (int j = threadIdx.x; j < N; j += blockDim.x) {
    double s = 0.0;
    for (int i = 0; i < N; ++i) s += fabs(A[i * N + j]);
    colmax = fmax(colmax, s);
  }
  const double l1 = block_max(colmax, s_buf);
  if (threadIdx.x == 0) s_l1 = l1;
  __syncthreads();
  const double nrm = s_l1;
  int deg;
  if (nrm < 1.495585217958292e-002) deg = 3;
  else if (nrm < 2.539398330063230e-001) deg = 5;
  else if (nrm < 9.504178996162932e-001) deg = 7;
  else if (nrm < 2.097847961257068e+000) deg = 9;
  else deg = 13;
  if (deg == 13) {
    if (threadIdx.x == 0) {
      int e;
      frexp(nrm / 5.371920351148152, &e);
      s_sq = e < 0 ? 0 : e;
    }
    __syncthreads();
    const int sq = s_sq;
    for (size_t idx = threadIdx.x; idx < NN; idx += blockDim.x) A[idx] = ldexp(A[idx], -sq);
    __syncthreads();
  } else if (threadIdx.x == 0) {
    s_sq = 0;
  }
  __syncthreads();
  EXPM_PROBE(0, tp);
  blk_matmul(A2, A, A, N, bx);
  if (deg == 3) {
    const double b[] = {120.0, 60.0, 12.0, 1.0};
    { const double c[] = {b[3]}; const double* M[] = {A2}; blk_lincomb(T1, N, 1, c, M, b[1], bx); }
    blk_matmul(U, A, T1, N, bx);
    { const double c[] = {b[2]}; const double* M[] = {A2}; blk_numden(T1, T2, U, N, 1, c, M, b[0], bx); }
  } else if (deg == 5) {
    const double b[] = {30240.0, 15120.0, 3360.0, 420.0, 30.0, 1.0};
    blk_matmul(A4, A2, A2, N, bx);
    { const double c[] = {b[5], b[3]}; const double* M[] = {A4, A2}; blk_lincomb(T1, N, 2, c, M, b[1], bx); }
    blk_matmul(U, A, T1, N, bx);
    { const double c[] = {b[4], b[2]}; const double* M[] = {A4, A2}; blk_numden(T1, T2, U, N, 2, c, M, b[0], bx); }
  } else if (deg == 7) {
    const double b[] = {17297280.0, 8648640.0, 1995840.0, 277200.0, 25200.0, 1512.0, 56.0, 1.0};
    blk_matmul(A4, A2, A2, N, bx);
    blk_matmul(A6, A4, A2, N, bx);
    { const double c[] = {b[7], b[5], b[3]}; const double* M[] = {A6, A4, A2}; blk_lincomb(T1, N, 3, c, M, b[1], bx); }
    blk_matmul(U, A, T1, N, bx);
    { const double c[] = {b[6], b[4], b[2]}; const double* M[] = {A6, A4, A2}; blk_numden(T1, T2, U, N, 3, c, M, b[0], bx); }
  } else if (deg == 9) {
    const double b[] = {17643225600.0, 8821612800.0, 2075673600.0, 302702400.0, 30270240.0,
                        2162160.0,     110880.0,     3960.0,       90.0,        1.0};
    blk_matmul(A4, A2, A2, N, bx);
    blk_matmul(A6, A4, A2, N, bx);
    blk_matmul(A8, A6, A2, N, bx);
    { const double c[] = {b[9], b[7], b[5], b[3]}; const double* M[] = {A8, A6, A4, A2}; blk_lincomb(T1, N, 4, c, M, b[1], bx); }
    blk_matmul(U, A, T1, N, bx);
    { const double c[] = {b[8], b[6], b[4], b[2]}; const double* M[] = {A8, A6, A4, A2}; blk_numden(T1, T2, U, N, 4, c, M, b[0], bx); }
  } else {
    const double b[] = {64764752532480000.0, 32382376266240000.0, 7771770303897600.0,
                        1187353796428800.0,  129060195264000.0,   10559470521600.0,
                        670442572800.0,      33522128640.0,       1323241920.0,
                        40840800.0,          960960.0,            16380.0,
                        182.0,               1.0};
    blk_matmul(A4, A2, A2, N, bx);
    blk_matmul(A6, A4, A2, N, bx);
    { const double c[] = {b[13], b[11], b[9]}; const double* M[] = {A6, A4, A2}; blk_lincomb(T1, N, 3, c, M, 0.0, bx); }
    blk_matmul(T2, A6, T1, N, bx);
    { const double c[] = {1.0, b[7], b[5], b[3]}; const double* M[] = {T2, A6, A4, A2}; blk_lincomb(T1, N, 4, c, M, b[1], bx); }
    blk_matmul(U, A, T1, N, bx);
    { const double c[] = {b[12], b[10], b[8]}; const double* M[] = {A6, A4, A2}; blk_lincomb(T1, N, 3, c, M, 0.0, bx); }
    blk_matmul(V, A6, T1, N, bx);
    { const double c[] = {1.0, b[6], b[4], b[2]}; const double* M[] = {V, A6, A4, A2}; blk_numden(T1, T2, U, N, 4, c, M, b[0], bx); }
  }
  // numer = U + V -> T1, denom = V - U -> T2 (blk_numden above); solve denom X = numer into U
  EXPM_PROBE(1, tp);
  blk_lu_solve(T2, T1, U, N, tp, xp);
  double* cur = U;
  double* oth = A2;
  for (int i = 0; i < s_sq; ++i) {
    blk_matmul(oth, cur, cur, N, bx);
    double* t = cur; cur = oth; oth = t;
  }
  EXPM_PROBE(4, tp);
  if (threadIdx.x == 0 && xp) {
    xp[5] += 1;
    xp[6] += s_sq;
  }
  return cur;
}

// Standalone device expm (one CTA) of an N x N matrix in W[0..N*N); result copied to out.
// ------------------------------------------------------------------ controller
__device__ __forceinline__ void set_window(PhiState* st, int j) {
  st->j = j;
  st->j0 = st->full_orth ? 0 : max(0, j + 1 - st->window);
  st->k = j - st->j0 + 1;
}

// DCGS2 (dcgs.cu): after the update pass of the cycle for column j, finish
// column j-1 (reorthogonalisation correction H(:, j-1) += a, exact H(j, j-1) =
// ||u - V a||, breakdown test of proj/src/phi.cpp:104-108 one cycle late) and write
// column j provisionally from a, b, <u,w> and H.  Thread 0 of k_ctl.
// Returns 1 on breakdown (mc = j), else 0.
static __device__ int dcgs_finish(PhiState* st, double* Hst) {
  const int j = st->j;
  const double nd = (double)st->n;
  // stage-1 JVP 32n + dots pass 8n(j + 2) (with the dots in the JVP sweep, dots_fused: u and w
  // are not re-read, 8n j); then the update pass 8n(j + 4), or with the lookahead (pipelined
  // DCGS2) the stage-2 JVP 32n + the merged pass 8n(j + 6)
  if (st->pl_direct) st->alg_bytes += 32.0 * nd + 8.0 * nd * (st->dots_fused ? (double)j : j + 2.0);
  st->alg_bytes += st->pl_look ? 32.0 * nd + 8.0 * nd * (j + 6.0) : 8.0 * nd * (j + 4.0);
  // the merged pass left the next column's image (slot j+2) and pass-1 dots
  st->pl_ready = st->pl_look ? j + 1 : -1;
  double beta = 1.0;
  // distinct PhiState arrays: restrict lets the loads of the loops below be issued ahead
  double* __restrict__ Hm = Hst;
  const double* __restrict__ da = st->dc_a;
  const double* __restrict__ db = st->dc_b;
  const double* __restrict__ dg = st->dc_g;
  if (j >= 1) {
    beta = st->scale[j] * sqrt(st->red.nrmU);
#pragma unroll 4
    for (int l = 0; l < j; ++l) Hm[l * kMaxBasis + (j - 1)] += da[l];
    if (beta <= 1e-14 * fmax(st->pre_prev, 1e-300)) {
      Hst[j * kMaxBasis + (j - 1)] = 0.0;
      st->mc = j;
      st->breakdown = 1;
      st->pl_ready = -1;
      return 1;
    }
    Hst[j * kMaxBasis + (j - 1)] = beta;
    st->scale[j] = 1.0 / sqrt(st->red.nrmU);  // V_j = slot_j / ||slot_j||
  }
  const double ib = 1.0 / beta;
  // column j = kMaxBasis (the avnorm cycle at mc = mmax = 128) has no storage and no
  // use: the space cannot grow past mmax
  const bool store = j < kMaxBasis;
  double hh = 0.0;
#pragma unroll 4
  for (int l = 0; l < j; ++l) {
    const double h = (db[l] - dg[l]) * ib;
    if (store) Hm[l * kMaxBasis + j] = h;
    hh = fma(h, h, hh);
  }
  // the V_j coefficient the update pass actually removed (gamma from the Pythagorean
  // beta); the next cycle's reorthogonalisation adds the remainder
  const double gj = j >= 1 ? beta * st->dc_a[j - 1] : 0.0;
  const double hj = st->dc_gp - gj * ib;
  if (store) Hst[j * kMaxBasis + j] = hj;
  hh = fma(hj, hj, hh);
  st->scale[j + 1] = ib;                                   // u_{j+1} = slot_{j+1} / beta
  st->pre_prev = sqrt(st->red.nrmW * ib * ib + hh);        // ||dt A V_j|| (incl. the augmentation)
  return 0;
}

// Pipelined DCGS2 flags of the next cycle (see PhiState::pl_direct / pl_look): look ahead on every
// extension; apply the operator to the candidate directly unless the last merged pass already
// left this column's image and dots
__device__ __forceinline__ void set_pipe(PhiState* st) {
  const int a = st->action;
  const bool pipe = st->dcgs && st->pipe_cfg;
  // the avnorm cycle looks ahead too when the space may still grow: a direct application in the
  // middle of a pipelined basis injects the recurrence's accumulated rounding into H at once
  // (on the stiff criterion-5 operator, ||dt A|| ~ 2e3, direct re-applications after grows or
  // periodic restarts cost 4-6 digits of H at m = 128; one uninterrupted recurrence keeps it at
  // the two-pass DCGS2 level, tools/pipe_hess.py); slot j+2 exists for j < mmax
  st->pl_look = pipe && (a == ACT_EXTEND || (a == ACT_AVNORM && st->j < st->grow_cap));
  const bool restart = st->j > 0 && st->pipe_restart > 0 && st->j % st->pipe_restart == 0;
  st->pl_direct = !(pipe && (a == ACT_EXTEND || a == ACT_AVNORM) && st->pl_ready == st->j && !restart);
}

// Hg: the Hessenberg storage when `st` is a copy of the state's header only (k_ctl: the header in
// shared memory, H left in global memory); null: st->H.
__device__ __forceinline__ void ctl_body(PhiState* st, double* slot0, double* W, double* Wsm, int ws_cap,
                                         cudaGraphConditionalHandle cond, int use_graph, double* Hg = nullptr) {
  double* const Hst = Hg ? Hg : st->H;
  __shared__ int s_phase, s_exit, s_zeroH, s_done;
  const int tid = threadIdx.x;
  // CGS2 / IOP column j of H from the two passes' sums (proj/src/phi.cpp:96-104), one entry per
  // thread: thread 0's serial loop over the column cost ~100 cycles per entry (every access
  // goes through the state pointer, nothing can be hoisted)
  if (st->action == ACT_EXTEND && !st->dcgs && !st->stopped) {
    const int j = st->j, full = st->full_orth;
    for (int i = st->j0 + tid; i <= j; i += blockDim.x) {
      const double sci = st->scale[i];
      const double h1 = sci * st->red.dotA[i];
      Hst[i * kMaxBasis + j] = full ? h1 + sci * st->red.dotB[i] : h1;
    }
  }
  if (tid == 0) {
    st->body_runs++;
    s_exit = 0; s_zeroH = 0; s_done = 0;
    if (st->stopped || st->action == ACT_DONE || st->action == ACT_NONE) {
      s_done = 1;
    } else {
      st->cycles++;
      int phase = st->phase;
      switch (st->action) {
        case ACT_START:
          phase = PH_SUBSTEP;
          break;
        case ACT_EXTEND: {
          if (st->dcgs) {
            if (dcgs_finish(st, Hst)) {
              phase = PH_POST;  // breakdown in column j-1: no avnorm
            } else {
              st->iterations++;
              st->extend_cols++;
              const int mc = st->j + 1;
              st->mc = mc;
              if (mc < st->target) {
                set_window(st, mc);
                st->action = ACT_EXTEND;
                s_exit = 1;
              } else {
                phase = PH_POST;
              }
            }
            break;
          }
          const int j = st->j;  // H(j0..j, j): filled by all threads above
          {
            const double nd = (double)st->n, kk = (double)(j - st->j0 + 1);
            st->alg_bytes += 32.0 * nd + 8.0 * nd * (st->full_orth ? 3.0 * kk + 6.0 : 2.0 * kk + 4.0);
            st->extend_cols++;
          }
          const double pre_norm = sqrt(st->red.nrmA);
          const double hnext = sqrt(st->red.nrmC);
          st->pre_norm = pre_norm;
          Hst[(j + 1) * kMaxBasis + j] = hnext;
          const int mc = j + 1;
          st->mc = mc;
          st->iterations++;
          if (hnext <= 1e-14 * fmax(pre_norm, 1e-300)) {
            Hst[mc * kMaxBasis + (mc - 1)] = 0.0;
            st->breakdown = 1;
            phase = PH_POST;
          } else {
            st->scale[mc] = 1.0 / hnext;
            if (mc < st->target) {
              set_window(st, mc);
              st->action = ACT_EXTEND;
              s_exit = 1;
            } else {
              phase = PH_POST;
            }
          }
          break;
        }
        case ACT_AVNORM:
          if (st->dcgs) {  // the avnorm cycle extends column mc provisionally as well
            if (dcgs_finish(st, Hst)) {
              st->avnorm = 0.0;  // breakdown in column mc-1 (the reference computes no avnorm)
            } else {
              st->iterations++;
              st->avnorms++;
              st->avnorm = st->pre_prev;  // ||dt A V_mc|| (proj/src/phi.cpp:195-199)
              st->dc_pending = 1;
            }
            phase = PH_DECIDE;
            break;
          }
          st->alg_bytes += 32.0 * (double)st->n;
          st->avnorms++;
          st->avnorm = sqrt(st->red.nrmA);
          phase = PH_DECIDE;
          break;
        case ACT_COMBINE: {
          st->alg_bytes += 8.0 * (double)st->n * (double)(st->mc + 1);
          st->combines++;
          double w2 = st->red.w2;
          for (int j = 0; j < st->p; ++j) slot0[st->n + j] = st->tailw[j];  // replicated tail
          for (int j = 0; j < st->p; ++j) w2 += st->tailw[j] * st->tailw[j];
          st->red.w2 = w2;
          phase = st->t < 1.0 - 1e-14 ? PH_SUBSTEP : PH_DONE;
          break;
        }
        default:
          break;
      }
      if (st->cycles > st->max_cycles) {
        st->status = PHI_ERR_CYCLES;
        phase = PH_DONE;
        s_exit = 0;
      }
      s_phase = phase;
    }
  }
  __syncthreads();
  if (s_done) {
    if (tid == 0 && use_graph) cudaGraphSetConditional(cond, 0u);
    return;
  }
  while (!s_exit) {
    const int phase = s_phase;
    if (phase == PH_DECIDE) {
      // hbar (mc+2)^2 = [H(0:mc, 0:mc-1) 0; 0 .. 1 0], scaled by h (proj/src/phi.cpp:208-211)
      const int mc = st->mc, N = mc + 2;
      const double h = st->h;
      double* Wx = 9 * N * N <= ws_cap ? Wsm : W;
      for (int idx = tid; idx < N * N; idx += blockDim.x) {
        const int i = idx / N, j = idx % N;
        double v = 0.0;
        if (i <= mc && j < mc) v = Hst[i * kMaxBasis + j];
        if (i == mc + 1 && j == mc) v = 1.0;
        Wx[idx] = h * v;
      }
      __syncthreads();
      const long long te0 = clock64();
      const double* F = blk_expm(9 * N * N <= ws_cap ? Wsm : W, N, st->xprof);
      if (tid == 0) {  // diagnostics (expdg_debug_profile slots 5, 6): SM cycles in the expm, calls
        st->prof[5] += clock64() - te0;
        st->prof[6] += 1;
      }
      if (tid == 0) {
        const double beta = st->beta;
        double err = 0.0;
        if (!st->breakdown) {
          const double p1 = fabs(beta * F[mc * N]);
          const double p2 = fabs(beta * F[(mc + 1) * N]) * st->avnorm;
          if (p1 > 10.0 * p2) err = p2;
          else if (p1 > p2) err = p1 * p2 / (p1 - p2);
          else err = p1;
        }
        st->last_estimate = err;
        const double tol = st->tol;
        if (st->breakdown || err <= 0.5 * tol * beta * h) {
          for (int i = 0; i < mc; ++i) st->comb[i] = beta * F[i * N];
          const double t = st->t + h;
          st->t = t;
          st->substeps++;
          for (int j = 0; j < st->p; ++j) {
            double v = 1.0;
            for (int q = 1; q <= st->p - 1 - j; ++q) v *= st->dt * t / q;
            st->tailw[j] = v;
          }
          double hn = h;
          if (err < 1e-3 * tol * beta * h) hn *= 2.0;
          st->h = fmin(hn, 1.0 - t);
          st->action = ACT_COMBINE;
          s_exit = 1;
        } else if (mc < st->grow_cap) {
          const int m = min(st->grow_cap, max(mc + 1, (3 * mc) / 2));
          st->m = m;
          st->target = m;
          if (st->dcgs && st->dc_pending) {
            // column mc was extended by the avnorm cycle; the reference re-applies A to
            // V_mc here, which counts as an iteration (proj/src/phi.cpp:84-112)
            st->dc_pending = 0;
            st->iterations++;
            st->extend_cols++;
            st->mc = mc + 1;
            if (mc + 1 < m) {
              set_window(st, mc + 1);
              st->action = ACT_EXTEND;
            } else {
              st->j = mc + 1;
              st->action = ACT_AVNORM;
            }
          } else {
            set_window(st, mc);
            st->action = ACT_EXTEND;
          }
          s_exit = 1;
        } else {
          st->h = h * 0.5;
          if (st->h < 1e-12) {
            st->status = PHI_ERR_UNDERFLOW;
            s_phase = PH_DONE;
          }
        }
      }
      __syncthreads();
      continue;
    }
    if (tid == 0) {
      if (phase == PH_SUBSTEP) {
        if (st->substeps >= st->max_substeps) {
          st->status = PHI_ERR_BUDGET;
          s_phase = PH_DONE;
        } else {
          const double beta = sqrt(st->red.w2);
          if (beta == 0.0) {
            s_phase = PH_DONE;
          } else if (!isfinite(beta)) {
            st->status = PHI_ERR_NONFINITE;
            st->last_estimate = beta;
            s_phase = PH_DONE;
          } else {
            st->beta = beta;
            st->mc = 0;
            st->breakdown = 0;
            st->pl_ready = -1;  // slot 0 holds a new phi vector
            st->scale[0] = 1.0 / beta;
            st->dc_pending = 0;
            st->target = st->m;
            set_window(st, 0);
            st->action = ACT_EXTEND;
            s_zeroH = 1;
            s_exit = 1;
          }
        }
      } else if (phase == PH_POST) {
        if (st->build_only) {  // krylov_build (proj/src/phi.cpp:115-130): the factorisation only
          s_phase = PH_DONE;
        } else if (!st->breakdown) {
          st->j = st->mc;
          st->action = ACT_AVNORM;
          if (!st->dcgs) st->iterations++;  // DCGS2 counts it when the cycle finds no breakdown
          s_exit = 1;
        } else {
          st->avnorm = 0.0;
          s_phase = PH_DECIDE;
        }
      } else if (phase == PH_DONE) {
        if (st->status == PHI_RUNNING) st->status = PHI_OK;
        // stats of a call that returned are kept (add_stats, proj/src/integrators.cpp:59-65);
        // a KrylovError drops them and fails the step
        if (st->status == PHI_OK) st->iterations_total += st->iterations;
        else st->step_failed = 1;
        st->action = ACT_DONE;
        s_done = 1;
        s_exit = 1;
      }
    }
    __syncthreads();
  }
  if (s_zeroH) {
    const int rows = st->mmax + 1;
    for (int idx = tid; idx < rows * kMaxBasis; idx += blockDim.x) Hst[idx] = 0.0;
  }
  if (tid == 0) {
    st->phase = s_phase;
    set_pipe(st);
  }
  if (tid == 0 && s_done && use_graph) cudaGraphSetConditional(cond, 0u);
}

// ------------------------------------------------------------------ fused small-problem engine
// (fused.cuh).  PhiState is copied into shared memory up to the Hessenberg rows in use.
constexpr size_t kPhiHOff = offsetof(PhiState, H);
static_assert(kPhiHOff % 8 == 0 && offsetof(PhiState, H) + sizeof(double) * (kMaxBasis + 1) * kMaxBasis ==
                  sizeof(PhiState), "H must be the last PhiState member");

// [0, HOff + hbytes) in 8-byte words, 16 independent loads in flight per thread
__device__ __forceinline__ void state_copy(unsigned char* dst, const unsigned char* src, size_t hbytes) {
  const size_t nw = (kPhiHOff + hbytes) / 8;
  const unsigned long long* s = reinterpret_cast<const unsigned long long*>(src);
  unsigned long long* d = reinterpret_cast<unsigned long long*>(dst);
  const size_t t = threadIdx.x, nt = blockDim.x;
  for (size_t b0 = 0; b0 < nw; b0 += 16 * nt) {
    unsigned long long v[16];
#pragma unroll
    for (int u = 0; u < 16; ++u) {
      const size_t i = b0 + u * nt + t;
      v[u] = i < nw ? s[i] : 0ull;
    }
#pragma unroll
    for (int u = 0; u < 16; ++u) {
      const size_t i = b0 + u * nt + t;
      if (i < nw) d[i] = v[u];
    }
  }
}

// The fused passes run over [0, Lp), Lp = L rounded up to the block size (<= ld): the
// slot padding is zero and stays zero, so no per-element predicates; 32-bit indices.
//
// dst[i] = <slot_{i0+i}, y> for i < k: one warp per vector, four lane accumulators,
// fixed-order warp reductions.
__device__ __forceinline__ void fused_dots(const double* base, int ld, int i0, int k, const double* y, int Lp,
                                           double* dst) {
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = blockDim.x >> 5;
  for (int i = wid; i < k; i += nw) {
    const double* v = base + (i0 + i) * ld;
    double p0 = 0.0, p1 = 0.0, p2 = 0.0, p3 = 0.0;
    int d = lane;
    for (; d + 96 < Lp; d += 128) {
      p0 = fma(v[d], y[d], p0);
      p1 = fma(v[d + 32], y[d + 32], p1);
      p2 = fma(v[d + 64], y[d + 64], p2);
      p3 = fma(v[d + 96], y[d + 96], p3);
    }
    for (; d < Lp; d += 32) p0 = fma(v[d], y[d], p0);
    const double p = warp_sum((p0 + p1) + (p2 + p3));
    if (lane == 0) dst[i] = p;
  }
  __syncthreads();
}

// y -= sum_i c_i slot_{i0+i}; a thread updates up to 8 of its elements together,
// two basis vectors per step (16 independent loads in flight); returns its ||y||^2 share
__device__ __forceinline__ double fused_update(double* base, int ld, int i0, int k, const double* c, double* y,
                                               int Lp) {
  const int T = blockDim.x, nq = Lp / T;
  const double* v0 = base + i0 * ld + threadIdx.x;
  double* yt = y + threadIdx.x;
  double nacc = 0.0;
  for (int q0 = 0; q0 < nq; q0 += 8) {
    const int qn = min(8, nq - q0);
    double a[8], b2[8];
#pragma unroll
    for (int q = 0; q < 8; ++q) {
      a[q] = q < qn ? yt[(q0 + q) * T] : 0.0;
      b2[q] = 0.0;
    }
    int i = 0;
    for (; i + 1 < k; i += 2) {
      const double c0 = c[i], c1 = c[i + 1];
      const double* p0 = v0 + i * ld + q0 * T;
      const double* p1 = p0 + ld;
#pragma unroll
      for (int q = 0; q < 8; ++q)
        if (q < qn) {
          a[q] = fma(-c0, p0[q * T], a[q]);
          b2[q] = fma(-c1, p1[q * T], b2[q]);
        }
    }
    if (i < k) {
      const double c0 = c[i];
      const double* p0 = v0 + i * ld + q0 * T;
#pragma unroll
      for (int q = 0; q < 8; ++q)
        if (q < qn) a[q] = fma(-c0, p0[q * T], a[q]);
    }
#pragma unroll
    for (int q = 0; q < 8; ++q)
      if (q < qn) {
        const double yv = a[q] + b2[q];
        yt[(q0 + q) * T] = yv;
        nacc = fma(yv, yv, nacc);
      }
  }
  return nacc;
}

// dynamic shared memory of the fused kernel: PhiState up to the Hessenberg rows in use,
// then the controller's expm workspace when the augmented Hessenberg is small
__host__ __device__ constexpr size_t fused_state_bytes(int mmax) {
  return ((kPhiHOff + sizeof(double) * (size_t)(mmax + 2 < kMaxBasis + 1 ? mmax + 2 : kMaxBasis + 1) * kMaxBasis +
           15) / 16) * 16;
}
constexpr int kFusedWsN = 48;  // expm workspace in shared memory for N <= 48 (9 N^2 doubles)

template <class EL>
__global__ void __launch_bounds__(kFusedThreads, 1) k_phi_fused(PhiState* gst, double* base, double* W, BArgs b,
                                                               EL el, int ws_cap) {
  extern __shared__ __align__(16) unsigned char fsm[];
  PhiState* st = reinterpret_cast<PhiState*>(fsm);
  __shared__ size_t s_hb;
  __shared__ int s_act;
  __shared__ double s_buf[kFusedThreads / 32];
  __shared__ double s_c[kMaxSlots];
  __shared__ double s_xt[kMaxP];
  const int tid = threadIdx.x;
  if (tid == 0) s_hb = sizeof(double) * (size_t)min(gst->mmax + 2, kMaxBasis + 1) * kMaxBasis;
  __syncthreads();
  const size_t hb = s_hb;
  double* Wsm = reinterpret_cast<double*>(fsm + ((kPhiHOff + hb + 15) / 16) * 16);
  state_copy(fsm, reinterpret_cast<const unsigned char*>(gst), hb);
  __syncthreads();
  const long long n = st->n, L = n + kTailPad, ld = st->ld;
  const int ld32 = (int)ld;
  const long long Lr = ((L + kFusedThreads - 1) / kFusedThreads) * kFusedThreads;
  const int Lp = (int)(Lr < ld ? Lr : ld);
  constexpr int NP = EL::kNP;
  long long t0 = clock64();
  auto mark = [&](int slot) {  // thread 0 after a barrier: cycles of the phase just finished
    if (tid == 0) {
      const long long t1 = clock64();
      st->prof[slot] += t1 - t0;
      t0 = t1;
    }
  };
  for (;;) {
    if (tid == 0) s_act = st->stopped ? ACT_DONE : st->action;
    __syncthreads();
    const int act = s_act;
    if (act == ACT_DONE || act == ACT_NONE) break;
    if (act == ACT_EXTEND || act == ACT_AVNORM) {
      // y = dt (L s_j V_j + sum x_tail b) into slot j+1 (proj/src/phi.cpp:151-158)
      const int j = st->j;
      const double xs = st->scale[j], dt = st->dt;
      const double* x = base + (size_t)j * ld;
      double* y = base + (size_t)(j + 1) * ld;
      if (tid < kMaxP) s_xt[tid] = tid < b.p ? x[n + tid] * xs : 0.0;
      __syncthreads();
      double nacc = 0.0;
      const int ne = el.elements();
      for (int e = tid; e < ne; e += kFusedThreads) {
        double out[NP];
        el.apply(e, x, xs, out);
#pragma unroll
        for (int i = 0; i < NP; ++i) {
          const size_t g = (size_t)e * NP + i;
          const double v = dt * aug_tail(b, s_xt, g, out[i]);
          y[g] = v;
          nacc = fma(v, v, nacc);
        }
      }
      if (tid < kTailPad) {
        const double v = (tid + 1 < b.p) ? dt * s_xt[tid + 1] : 0.0;
        y[n + tid] = v;
        nacc = fma(v, v, nacc);
      }
      const double tot = block_sum(nacc, s_buf);
      if (tid == 0) st->red.nrmA = tot;
      __syncthreads();
      mark(0);
      if (act == ACT_EXTEND) {  // CGS2 passes of krylov.cu (same coefficients), or one IOP pass
        const int i0 = st->j0, k = j - i0 + 1;
        fused_dots(base, ld32, i0, k, y, Lp, st->red.dotA + i0);
        mark(1);
        if (st->full_orth) {
          for (int i = tid; i < k; i += blockDim.x) {
            const double sc = st->scale[i0 + i];
            s_c[i] = sc * sc * st->red.dotA[i0 + i];
          }
          __syncthreads();
          fused_update(base, ld32, i0, k, s_c, y, Lp);
          __syncthreads();
          mark(2);
          fused_dots(base, ld32, i0, k, y, Lp, st->red.dotB + i0);
          mark(1);
        }
        for (int i = tid; i < k; i += blockDim.x) {
          const double sc = st->scale[i0 + i];
          s_c[i] = sc * sc * (st->full_orth ? st->red.dotB[i0 + i] : st->red.dotA[i0 + i]);
        }
        __syncthreads();
        const double nn = block_sum(fused_update(base, ld32, i0, k, s_c, y, Lp), s_buf);
        if (tid == 0) st->red.nrmC = nn;
        __syncthreads();
        mark(2);
      }
    } else if (act == ACT_COMBINE) {
      // w = V_{0:mc} (beta f(0:mc, 0)) in place in slot 0 (proj/src/phi.cpp:227)
      const int k = st->mc;
      for (int i = tid; i < k; i += blockDim.x) s_c[i] = st->scale[i] * st->comb[i];
      __syncthreads();
      double nacc = 0.0;
      for (long long d = tid; d < L; d += blockDim.x) {
        double a = 0.0;
        for (int i = 0; i < k; ++i) a = fma(s_c[i], base[(size_t)i * ld + d], a);
        base[d] = a;
        if (d < n) nacc = fma(a, a, nacc);
      }
      const double tot = block_sum(nacc, s_buf);
      if (tid == 0) st->red.w2 = tot;
      __syncthreads();
      mark(3);
    }
    ctl_body(st, base, W, Wsm, ws_cap, cudaGraphConditionalHandle{}, 0);
    __syncthreads();
    mark(4);
  }
  __syncthreads();
  state_copy(reinterpret_cast<unsigned char*>(gst), fsm, hb);
}

// ------------------------------------------------------------------ cluster engine (small problems)
// The fused engine spread over a thread-block cluster: CTA r of an 8-CTA cluster owns
// elements [r epc, (r+1) epc) and keeps its slice of EVERY Krylov vector in its own
// shared memory; neighbour elements of the operator and the partial sums of every
// reduction are read from the other CTAs' shared memory (DSMEM).  Each reduction is
// one cluster barrier: every CTA writes its partials to its own (double-buffered)
// buffer, then every CTA sums all of them in rank order (identical totals).  Every CTA
// holds its own copy of PhiState in shared memory and runs the controller (ctl_body) on the
// identical totals, so all CTAs take identical decisions with no broadcast and no cluster
// barrier after the controller (a cluster barrier costs ~1.6k SM cycles, as much as a
// column's arithmetic at C1); CTA 0's copy goes back to global memory at the end.  No basis
// traffic leaves the SMs.
namespace cg = cooperative_groups;
constexpr int kClusterCTAs = 8;
constexpr int kClusterThreads = 256;

template <class EL>
__global__ void __launch_bounds__(kClusterThreads, 1)
    k_phi_cluster(PhiState* gst, double* base, double* W, BArgs b, EL el, int epc, int lds, int nslots,
                  int ws_cap, int state_off, int ws_off, int redund) {
  cg::cluster_group cl = cg::this_cluster();
  const int rank = (int)cl.block_rank(), CS = (int)cl.num_blocks();
  extern __shared__ __align__(16) unsigned char csm[];
  double* V = reinterpret_cast<double*>(csm);
  double* part = V + (size_t)nslots * lds;  // 2 x (2 kMaxSlots + 2)
  double* ul = part + 2 * (2 * kMaxSlots + 2);  // u~ of elements [e_lo - 1, e_hi + 1), frozen for the call
  double* bl = ul + (size_t)(epc + 2) * EL::kNP;  // b_1..b_p slices: p x (epc NP)
  PhiState* st0 = reinterpret_cast<PhiState*>(csm + state_off);
  double* Wsm = reinterpret_cast<double*>(csm + ws_off);
  __shared__ int s_act, s_j, s_j0, s_full, s_mc, s_p, s_tailhere;
  __shared__ double s_dt;
  __shared__ double s_scale[kMaxSlots], s_c[kMaxSlots], s_mine[2 * kMaxSlots + 2], s_tot[2 * kMaxSlots + 2];
  __shared__ double s_xt[kMaxP], s_buf[kClusterThreads / 32];
  __shared__ size_t s_hb;
  constexpr int NP = EL::kNP;
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5, T = blockDim.x;
  const int nel = el.elements();
  const int e_lo = min(rank * epc, nel), e_hi = min(e_lo + epc, nel);
  const int nloc = (e_hi - e_lo) * NP, tail_at = epc * NP;
  const long long n = gst->n;
  // ---- init: this CTA's slice of slot 0 (the phi vector of k_phi_init); CTA 0: PhiState
  for (int i = tid; i < nloc; i += T) V[i] = base[(size_t)e_lo * NP + i];
  for (int i = tid; i < kTailPad; i += T) V[tail_at + i] = base[n + i];
  for (int i = tid; i < (e_hi - e_lo + 2) * NP; i += T) {  // u~ with one element either side
    double o[NP];
    el.gather([&](int w, double* oo) {
#pragma unroll
      for (int q = 0; q < NP; ++q) oo[q] = el.P.ut[(size_t)w * NP + q];
    }, e_lo - 1 + i / NP, o);
    ul[i] = o[i % NP];
  }
  for (int m = 1; m <= b.p && m <= kMaxP; ++m)
    for (int i = tid; i < nloc; i += T) bl[(size_t)(m - 1) * epc * NP + i] = b.b[m] ? b.b[m][(size_t)e_lo * NP + i] : 0.0;
  // redund (every CTA runs the controller): each CTA has its own state copy and expm
  // workspace; else CTA 0 alone (EXPDG_CLUSTER_CTL=0, diagnostics)
  const bool ctl_here = redund || rank == 0;
  if (redund) W += (size_t)rank * 9 * (kMaxBasis + 2) * (kMaxBasis + 2);
  if (ctl_here) {
    if (tid == 0) s_hb = sizeof(double) * (size_t)min(gst->mmax + 2, kMaxBasis + 1) * kMaxBasis;
    __syncthreads();
    state_copy(reinterpret_cast<unsigned char*>(st0), reinterpret_cast<const unsigned char*>(gst), s_hb);
  }
  const PhiState* S = redund ? st0 : cl.map_shared_rank(st0, 0);
  const int nsc = nslots < kMaxSlots ? nslots : kMaxSlots;
  // the controller's decision (action, column, scales) into shared scalars: from this CTA's own
  // state (redund), or pushed by CTA 0 into every CTA's shared memory
  auto push = [&]() {
    __syncthreads();
    if (redund) {
      if (tid == 0) {
        s_act = st0->stopped ? ACT_DONE : st0->action;
        s_j = st0->j;
        s_j0 = st0->j0;
        s_full = st0->full_orth;
        s_mc = st0->mc;
        s_dt = st0->dt;
      }
      for (int i = tid; i < nsc; i += T) s_scale[i] = st0->scale[i];
      return;
    }
    for (int r = tid; r < CS; r += T) {
      *cl.map_shared_rank(&s_act, r) = st0->stopped ? ACT_DONE : st0->action;
      *cl.map_shared_rank(&s_j, r) = st0->j;
      *cl.map_shared_rank(&s_j0, r) = st0->j0;
      *cl.map_shared_rank(&s_full, r) = st0->full_orth;
      *cl.map_shared_rank(&s_mc, r) = st0->mc;
      *cl.map_shared_rank(&s_dt, r) = st0->dt;
    }
    for (int idx = tid; idx < CS * nsc; idx += T) {
      const int r = idx / nsc, i = idx - r * nsc;
      cl.map_shared_rank(s_scale, r)[i] = st0->scale[i];
    }
  };
  if (ctl_here) push();
  cl.sync();
  int round = 0;
  // cluster totals of cnt partial sums in s_mine -> s_tot (every CTA, rank order)
  auto reduce = [&](int cnt) {
    double* buf = part + (round & 1) * (2 * kMaxSlots + 2);
    for (int i = tid; i < cnt; i += T) buf[i] = s_mine[i];
    cl.sync();
    for (int i = tid; i < cnt; i += T) {
      // all CS remote loads in flight at once (one DSMEM round trip, not CS), summed in rank order
      double v[kClusterCTAs];
#pragma unroll
      for (int r = 0; r < kClusterCTAs; ++r) v[r] = r < CS ? cl.map_shared_rank(buf, r)[i] : 0.0;
      double sum = 0.0;
#pragma unroll
      for (int r = 0; r < kClusterCTAs; ++r)
        if (r < CS) sum += v[r];
      s_tot[i] = sum;
    }
    __syncthreads();
    ++round;
  };
  // this CTA's <V_{i0+i}, y> for i < k, one warp per vector (the tail counts on rank 0)
  // (two vectors per warp and pass: their FMA chains and shuffle reductions interleave; each
  // vector's sum keeps its order, so the totals are bit-identical to one vector per pass)
  auto local_dots = [&](int i0, int k, const double* y) {
    constexpr int NW = kClusterThreads / 32;
    for (int i = wid; i < k; i += 2 * NW) {
      const bool two = i + NW < k;
      const double* v = V + (size_t)(i0 + i) * lds;
      const double* w = V + (size_t)(i0 + (two ? i + NW : i)) * lds;
      double p0 = 0.0, p1 = 0.0, q0 = 0.0, q1 = 0.0;
      for (int d = lane; d < nloc; d += 64) {
        const double y0 = y[d];
        p0 = fma(v[d], y0, p0);
        q0 = fma(w[d], y0, q0);
        if (d + 32 < nloc) {
          const double y1 = y[d + 32];
          p1 = fma(v[d + 32], y1, p1);
          q1 = fma(w[d + 32], y1, q1);
        }
      }
      if (s_tailhere && lane < kTailPad) {
        p0 = fma(v[tail_at + lane], y[tail_at + lane], p0);
        q0 = fma(w[tail_at + lane], y[tail_at + lane], q0);
      }
      double p = p0 + p1, q = q0 + q1;
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) {
        p += __shfl_xor_sync(0xffffffffu, p, o);
        q += __shfl_xor_sync(0xffffffffu, q, o);
      }
      if (lane == 0) {
        s_mine[i] = p;
        if (two) s_mine[i + NW] = q;
      }
    }
    __syncthreads();
  };
  // y -= sum_i c_i V_{i0+i} on the local head and the replicated tail; returns this thread's ||y||^2
  auto local_update = [&](int i0, int k, double* y) {
    double nacc = 0.0;
    for (int d = tid; d < nloc + kTailPad; d += T) {
      const int dd = d < nloc ? d : tail_at + (d - nloc);
      double a = y[dd], a2 = 0.0;
      int i = 0;
      for (; i + 1 < k; i += 2) {
        a = fma(-s_c[i], V[(size_t)(i0 + i) * lds + dd], a);
        a2 = fma(-s_c[i + 1], V[(size_t)(i0 + i + 1) * lds + dd], a2);
      }
      if (i < k) a = fma(-s_c[i], V[(size_t)(i0 + i) * lds + dd], a);
      const double yv = a + a2;
      y[dd] = yv;
      if (d < nloc || s_tailhere) nacc = fma(yv, yv, nacc);
    }
    return nacc;
  };
  bool cl_pending = false;  // a cluster barrier arrived at, not yet waited for
  long long t0 = clock64();
  auto mark = [&](int slot) {  // CTA 0, thread 0: SM cycles of the phase just finished
    if (rank == 0 && tid == 0) {
      const long long t1 = clock64();
      st0->prof[slot] += t1 - t0;
      t0 = t1;
    }
  };
  for (;;) {
    if (tid == 0) {
      s_p = b.p;
      s_tailhere = rank == 0;
    }
    __syncthreads();
    const int act = s_act;
    if (act == ACT_DONE || act == ACT_NONE) break;
    if (act == ACT_EXTEND || act == ACT_AVNORM) {
      const int j = s_j;
      const double xs = s_scale[j], dt = s_dt;
      const double* x = V + (size_t)j * lds;
      double* y = V + (size_t)(j + 1) * lds;
      if (tid < kMaxP) s_xt[tid] = tid < s_p ? x[tail_at + tid] * xs : 0.0;
      __syncthreads();
      double nacc = 0.0;
      for (int e = e_lo + tid; e < e_hi; e += T) {
        double out[NP];
        el.apply_with(
            e,
            [&](int w, double* o) {
              const int r = w / epc, li = w - r * epc;
              const double* src = (r == rank ? V : cl.map_shared_rank(V, r)) + (size_t)j * lds + (size_t)li * NP;
#pragma unroll
              for (int i = 0; i < NP; ++i) o[i] = src[i] * xs;
            },
            [&](int w, double* o) {  // u~ of a neighbour element (w is already wrapped)
              int li = w - (e_lo - 1);
              if (li < 0) li += nel;
              if (li >= e_hi - e_lo + 2) li -= nel;
#pragma unroll
              for (int i = 0; i < NP; ++i) o[i] = ul[(size_t)li * NP + i];
            },
            out);
        const int le = e - e_lo;
#pragma unroll
        for (int i = 0; i < NP; ++i) {
          double v = out[i];
          for (int m = kMaxP; m >= 1; --m)  // aug_tail order (proj/src/phi.cpp:151-158)
            if (m <= s_p && b.b[m]) v = fma(s_xt[s_p - m], bl[(size_t)(m - 1) * epc * NP + le * NP + i], v);
          v = dt * v;
          y[le * NP + i] = v;
          nacc = fma(v, v, nacc);
        }
      }
      if (tid < kTailPad) {
        const double v = (tid + 1 < s_p) ? dt * s_xt[tid + 1] : 0.0;
        y[tail_at + tid] = v;
        if (s_tailhere) nacc = fma(v, v, nacc);
      }
      const double tot = block_sum(nacc, s_buf);
      if (act != ACT_EXTEND) {
        if (tid == 0) s_mine[0] = tot;
        __syncthreads();
        reduce(1);
        if (ctl_here && tid == 0) st0->red.nrmA = s_tot[0];
      }
      mark(0);
      if (act == ACT_EXTEND) {  // CGS2 passes (krylov.cu coefficients) or one IOP pass
        const int i0 = s_j0, k = j - i0 + 1;
        // ||y||^2 rides in the first dots reduction (one cluster barrier fewer per column)
        if (tid == 0) s_mine[k] = tot;
        local_dots(i0, k, y);
        reduce(k + 1);
        if (ctl_here) {
          for (int i = tid; i < k; i += T) st0->red.dotA[i0 + i] = s_tot[i];
          if (tid == 0) st0->red.nrmA = s_tot[k];
        }
        mark(1);
        if (s_full && redund) {
          // Two cluster reductions per column instead of three: ||y'||^2 (y' = y after the first
          // update) rides in the second dots reduction and the norm of the twice-orthogonalised
          // vector follows from it, ||y''||^2 = ||y'||^2 - sum_i (s_i d_i)^2 with d_i = <V_i, y'>
          // (the second-pass corrections are O(eps) ||y'||, so the identity holds to O(eps^2));
          // the cluster barrier that orders the last update before the neighbours' next reads is
          // split around the controller (arrive here, wait after ctl_body).
          for (int i = tid; i < k; i += T) s_c[i] = s_scale[i0 + i] * s_scale[i0 + i] * s_tot[i];
          __syncthreads();
          const double n1 = block_sum(local_update(i0, k, y), s_buf);
          if (tid == 0) s_mine[k] = n1;
          __syncthreads();
          mark(2);
          local_dots(i0, k, y);
          reduce(k + 1);
          mark(1);
          for (int i = tid; i < k; i += T) {
            st0->red.dotB[i0 + i] = s_tot[i];
            s_c[i] = s_scale[i0 + i] * s_scale[i0 + i] * s_tot[i];
          }
          if (tid == 0) {
            double corr = 0.0;
            for (int i = 0; i < k; ++i) {
              const double sd = s_scale[i0 + i] * s_tot[i];
              corr = fma(sd, sd, corr);
            }
            st0->red.nrmC = fmax(s_tot[k] - corr, 0.0);
          }
          __syncthreads();
          local_update(i0, k, y);
          asm volatile("barrier.cluster.arrive.release.aligned;" ::: "memory");
          cl_pending = true;
          mark(2);
        } else {
          if (s_full) {
            for (int i = tid; i < k; i += T) s_c[i] = s_scale[i0 + i] * s_scale[i0 + i] * s_tot[i];
            __syncthreads();
            local_update(i0, k, y);
            __syncthreads();
            mark(2);
            local_dots(i0, k, y);
            reduce(k);
            mark(1);
            if (ctl_here)
              for (int i = tid; i < k; i += T) st0->red.dotB[i0 + i] = s_tot[i];
          }
          for (int i = tid; i < k; i += T) s_c[i] = s_scale[i0 + i] * s_scale[i0 + i] * s_tot[i];
          __syncthreads();
          const double nn = block_sum(local_update(i0, k, y), s_buf);
          if (tid == 0) s_mine[0] = nn;
          __syncthreads();
          reduce(1);
          if (ctl_here && tid == 0) st0->red.nrmC = s_tot[0];
          mark(2);
        }
      }
    } else if (act == ACT_COMBINE) {
      const int k = s_mc;
      for (int i = tid; i < k; i += T) s_c[i] = s_scale[i] * S->comb[i];
      __syncthreads();
      double nacc = 0.0;
      for (int d = tid; d < nloc + kTailPad; d += T) {
        const int dd = d < nloc ? d : tail_at + (d - nloc);
        double a = 0.0;
        for (int i = 0; i < k; ++i) a = fma(s_c[i], V[(size_t)i * lds + dd], a);
        V[dd] = a;
        if (d < nloc) nacc = fma(a, a, nacc);
      }
      const double tot = block_sum(nacc, s_buf);
      if (tid == 0) s_mine[0] = tot;
      __syncthreads();
      reduce(1);
      if (ctl_here && tid == 0) st0->red.w2 = s_tot[0];
      mark(3);
    }
    if (ctl_here) {
      __syncthreads();
      // the controller writes the phi tail into this CTA's slot-0 tail (slot0[n + j])
      ctl_body(st0, V + tail_at - n, W, Wsm, ws_cap, cudaGraphConditionalHandle{}, 0);
      push();
    }
    // redund: the last reduction's cluster barrier already ordered every basis write this
    // cycle before any CTA's next read of a neighbour's slice
    if (cl_pending) {  // the column's last update is visible cluster-wide from here
      asm volatile("barrier.cluster.wait.acquire.aligned;" ::: "memory");
      cl_pending = false;
    }
    if (!redund) {
      cl.sync();
      if (act == ACT_COMBINE && rank != 0 && tid < kTailPad)  // replicate the reset tail
        V[tail_at + tid] = cl.map_shared_rank(V, 0)[tail_at + tid];
    }
    __syncthreads();
    mark(4);
  }
  // ---- the phi vector back to global slot 0; CTA 0: PhiState
  for (int i = tid; i < nloc; i += T) base[(size_t)e_lo * NP + i] = V[i];
  if (rank == 0) {
    for (int i = tid; i < kTailPad; i += T) base[n + i] = V[tail_at + i];
    __syncthreads();
    state_copy(reinterpret_cast<unsigned char*>(gst), reinterpret_cast<const unsigned char*>(st0), s_hb);
  }
  cl.sync();  // no CTA leaves while others may still read its shared memory
}

template <class EL>
bool launch_phi_cluster(cudaStream_t s, Engine& e, const EL& el, const BArgs& b) {
  static int max_dyn = -1;
  if (max_dyn < 0) {
    cudaFuncAttributes fa;
    EXPDG_CUDA(cudaFuncGetAttributes(&fa, k_phi_cluster<EL>));
    max_dyn = 232448 - (int)fa.sharedSizeBytes;
    EXPDG_CUDA(cudaFuncSetAttribute(k_phi_cluster<EL>, cudaFuncAttributeMaxDynamicSharedMemorySize, max_dyn));
  }
  const PhiState& c = *e.st_host;
  const int nel = (int)(c.n / EL::kNP);
  if (nel < 2 * kClusterCTAs) return false;
  const int epc = (nel + kClusterCTAs - 1) / kClusterCTAs;
  const int lds = ((epc * EL::kNP + kTailPad + 1) / 2) * 2;
  const int nslots = std::min(c.mmax + 2, kMaxSlots);
  const size_t vbytes = sizeof(double) * ((size_t)nslots * lds + 2 * (2 * kMaxSlots + 2) +
                                          (size_t)(epc + 2) * EL::kNP + (size_t)b.p * epc * EL::kNP);
  const size_t state_off = ((vbytes + 15) / 16) * 16;
  const size_t state = fused_state_bytes(c.mmax);
  if (state_off + state > (size_t)max_dyn) return false;
  int nws = std::min(c.mmax + 2, kFusedWsN);
  while (nws > 0 && state_off + state + sizeof(double) * 9 * nws * nws > (size_t)max_dyn) --nws;
  const size_t smem = state_off + state + sizeof(double) * 9 * nws * nws;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(kClusterCTAs);
  cfg.blockDim = dim3(kClusterThreads);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = kClusterCTAs;
  at[0].val.clusterDim.y = 1;
  at[0].val.clusterDim.z = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  static const int redund = [] {
    const char* v = std::getenv("EXPDG_CLUSTER_CTL");
    return v && v[0] == '0' ? 0 : 1;
  }();
  EXPDG_CUDA(cudaLaunchKernelEx(&cfg, k_phi_cluster<EL>, e.st, e.base, e.ework, b, el, epc, lds, nslots,
                                9 * nws * nws, (int)state_off, (int)(state_off + state), redund));
  return true;
}

template <class EL>
void launch_phi_fused(cudaStream_t s, Engine& e, const EL& el, const BArgs& b) {
  if (e.use_fused != 2 && launch_phi_cluster(s, e, el, b)) return;  // EXPDG_FUSED=2: single CTA
  static int max_dyn = -1;
  if (max_dyn < 0) {
    cudaFuncAttributes fa;
    EXPDG_CUDA(cudaFuncGetAttributes(&fa, k_phi_fused<EL>));
    max_dyn = 232448 - (int)fa.sharedSizeBytes;
    EXPDG_CUDA(cudaFuncSetAttribute(k_phi_fused<EL>, cudaFuncAttributeMaxDynamicSharedMemorySize, max_dyn));
  }
  const int mmax = e.st_host->mmax;
  const size_t state = fused_state_bytes(mmax);
  int nws = std::min(mmax + 2, kFusedWsN);
  while (nws > 0 && state + sizeof(double) * 9 * nws * nws > (size_t)max_dyn) --nws;
  const size_t smem = state + sizeof(double) * 9 * nws * nws;
  k_phi_fused<EL><<<1, kFusedThreads, smem, s>>>(e.st, e.base, e.ework, b, el, 9 * nws * nws);
}


}  // namespace expdg
