// Device-resident adaptive Krylov phi engine (the B200 replacement of
// proj/src/phi.cpp:133-260 and the Arnoldi loop of proj/src/phi.cpp:84-112).
//
// One "cycle" of the engine is a fixed sequence of six kernels:
//   [operator apply] -> [pass A dots] -> [pass B update+dots] -> [pass C update+norm]
//   -> [combine] -> [controller]
// Each kernel reads the action chosen by the previous controller from device
// memory and no-ops when it is not its turn, so the sequence is captured once
// into the body of a CUDA-graph WHILE node; the controller (one CTA) runs the
// Higham expm of the small augmented Hessenberg matrix, the reference error
// estimator and the accept / grow / halve rules, and clears the WHILE
// condition when the call is done.  No host round-trip per step.
//
// Orthogonalisation is classical Gram-Schmidt with one reorthogonalisation
// (CGS2) instead of the reference's two-pass MGS (proj/src/phi.cpp:94-100): the
// same projector in exact arithmetic, three streaming passes over V per column
// instead of 2(k+1) sequential ones.  IOP windows use one pass (reference: one
// MGS pass over the window).
#include <algorithm>
#include <cstddef>
#include <cstdlib>
#include <cstring>

#include <cooperative_groups.h>

#include "fused.cuh"
#include "krylov.cuh"

namespace expdg {

void launch_dcgs(cudaStream_t s, Engine& e, int which);
void dcgs_init_attrs(int maxsm);

enum TsMode { TS_DOTS = 0, TS_UPD_DOTS = 1, TS_UPD_NORM = 2, TS_COMBINE = 3 };
enum Ticket { TK_DOTS = 0, TK_UPD_DOTS = 1, TK_UPD_NORM = 2, TK_COMBINE = 3, TK_APPLY = 4, TK_INIT = 5,
              TK_RES = 6, TK_FINISH = 7, TK_MAX = 8 };

constexpr int kTsMaxStages = 8;
constexpr int kAccPerLane = (kMaxSlots + 7) / 8;

// ------------------------------------------------------------------ tall-skinny passes
// One CGS2 streaming pass over the k active basis vectors (and y).  Warp
// specialised: warp 8 is the TMA producer (1D bulk copies of T-double tiles of
// every stream into an S-stage smem ring, full/empty mbarriers), warps 0-7
// consume.  Dots keep the y tile in registers (lane owns d = lane + 32 m), the
// update runs one DOF per thread with two independent FMA chains.  T and S
// adapt to k so one stage is ~budget/S bytes in flight.
constexpr int kTsConsumers = 256;
constexpr int kTsBlock = kTsConsumers + 32;
constexpr int kTsMaxT = 2048;
constexpr int kTsChunk = 256;  // doubles of y held in registers per dot chunk (128 pairs)


// Consumer side of one tall-skinny pass (warps 0-7).  NV = most basis vectors
// any warp owns in the dots (ceil(k/8)), a compile-time bound so the per-vector
// accumulators stay in registers without per-chunk checks of all 17 slots.
template <int MODE, int NV>
__device__ __forceinline__ void ts_consume(const PhiState* st, double* base, double* smem, uint64_t* full,
                                           uint64_t* empty, const double* s_coef, int k, int T, int S,
                                           long long ntiles, long long n, long long ndot, int nst,
                                           double* ybase, double (&acc)[kAccPerLane], double& nacc) {
  const int tid = threadIdx.x;
  const int lane = tid & 31, wid = tid >> 5;
  int s = 0, use = 0;
  for (long long tl = blockIdx.x; tl < ntiles; tl += gridDim.x) {
    mbar_wait(&full[s], use & 1);
    double* V = smem + (size_t)s * nst * T;
    double* Y = V + (size_t)k * T;
    const long long g0 = tl * T;
    // element pairs: one LDS.128 per stream and coefficient pair feeds 4 FMAs
    const double2* V2 = reinterpret_cast<const double2*>(V);
    const double2* C2 = reinterpret_cast<const double2*>(s_coef);
    const int T2 = T >> 1;
    if (MODE == TS_UPD_DOTS || MODE == TS_UPD_NORM) {
      for (int p = tid; p < T2; p += kTsConsumers) {
        const double2 y = reinterpret_cast<const double2*>(Y)[p];
        double a0 = y.x, a1 = y.y, b0 = 0.0, b1 = 0.0;
        int i = 0;
        for (; i + 1 < k; i += 2) {
          const double2 c = C2[i >> 1];
          const double2 v0 = V2[(size_t)i * T2 + p];
          const double2 v1 = V2[(size_t)(i + 1) * T2 + p];
          a0 = fma(-c.x, v0.x, a0);
          a1 = fma(-c.x, v0.y, a1);
          b0 = fma(-c.y, v1.x, b0);
          b1 = fma(-c.y, v1.y, b1);
        }
        if (i < k) {
          const double c = s_coef[i];
          const double2 v0 = V2[(size_t)i * T2 + p];
          a0 = fma(-c, v0.x, a0);
          a1 = fma(-c, v0.y, a1);
        }
        const double2 yv = make_double2(a0 + b0, a1 + b1);
        reinterpret_cast<double2*>(Y)[p] = yv;
        reinterpret_cast<double2*>(ybase + g0)[p] = yv;
        if (MODE == TS_UPD_NORM) {
          if (g0 + 2 * p < ndot) nacc = fma(yv.x, yv.x, nacc);
          if (g0 + 2 * p + 1 < ndot) nacc = fma(yv.y, yv.y, nacc);
        }
      }
      if (MODE == TS_UPD_DOTS) consumer_sync();
    } else if (MODE == TS_COMBINE) {
      for (int p = tid; p < T2; p += kTsConsumers) {
        double a0 = 0.0, a1 = 0.0, b0 = 0.0, b1 = 0.0;
        int i = 0;
        for (; i + 1 < k; i += 2) {
          const double2 c = C2[i >> 1];
          const double2 v0 = V2[(size_t)i * T2 + p];
          const double2 v1 = V2[(size_t)(i + 1) * T2 + p];
          a0 = fma(c.x, v0.x, a0);
          a1 = fma(c.x, v0.y, a1);
          b0 = fma(c.y, v1.x, b0);
          b1 = fma(c.y, v1.y, b1);
        }
        if (i < k) {
          const double c = s_coef[i];
          const double2 v0 = V2[(size_t)i * T2 + p];
          a0 = fma(c, v0.x, a0);
          a1 = fma(c, v0.y, a1);
        }
        const double2 wv = make_double2(a0 + b0, a1 + b1);
        reinterpret_cast<double2*>(base + g0)[p] = wv;  // slot 0, in place (this tile already staged)
        if (g0 + 2 * p < n) nacc = fma(wv.x, wv.x, nacc);
        if (g0 + 2 * p + 1 < n) nacc = fma(wv.y, wv.y, nacc);
      }
    }
    if ((MODE == TS_DOTS || MODE == TS_UPD_DOTS) && g0 + T > ndot) {
      // a non-zero rank's tile holding the replicated phi tail: keep it out of the dots
      consumer_sync();
      for (int d = tid; d < T; d += kTsConsumers)
        if (g0 + d >= ndot) Y[d] = 0.0;
      consumer_sync();
    }
    if (MODE == TS_DOTS || MODE == TS_UPD_DOTS) {
      // y chunk of 256 doubles in registers (lane owns pairs c0/2 + lane + 32 m)
      const double2* Y2 = reinterpret_cast<const double2*>(Y);
      for (int c0 = 0; c0 < T; c0 += kTsChunk) {
        const int per = min(T - c0, kTsChunk) >> 6;  // pairs per lane (T >= 64)
        double2 yr[kTsChunk / 64];
#pragma unroll
        for (int m = 0; m < kTsChunk / 64; ++m)
          yr[m] = m < per ? Y2[(c0 >> 1) + lane + 32 * m] : make_double2(0.0, 0.0);
#pragma unroll
        for (int v = 0; v < NV; ++v) {
          const int i = wid + 8 * v;
          if (i < k) {
            const double2* Vi = V2 + (size_t)i * T2 + (c0 >> 1) + lane;
            double a0 = 0.0, a1 = 0.0;
#pragma unroll
            for (int m = 0; m < kTsChunk / 64; ++m) {
              if (m < per) {
                const double2 x = Vi[32 * m];
                a0 = fma(x.x, yr[m].x, a0);
                a1 = fma(x.y, yr[m].y, a1);
              }
            }
            acc[v] += a0 + a1;
          }
        }
      }
    }
    __syncwarp();
    if (lane == 0) mbar_arrive(&empty[s]);
    if (++s == S) { s = 0; ++use; }
  }
}

template <int MODE>
__global__ void __launch_bounds__(kTsBlock, 1) k_ts(PhiState* st, double* base, double* partials, int budget,
                                                    int max_stages, int min_T) {
  extern __shared__ __align__(128) double smem[];
  __shared__ uint64_t full[kTsMaxStages], empty[kTsMaxStages];
  __shared__ int s_active, s_i0, s_k, s_y, s_T, s_S;
  __shared__ long long s_ld, s_n, s_ndot;
  __shared__ __align__(16) double s_coef[kMaxSlots + 2];
  __shared__ double s_red[kMaxSlots + 1];
  __shared__ double s_buf[kTsBlock / 32];

  const int tid = threadIdx.x;
  const int lane = tid & 31, wid = tid >> 5;
  if (tid == 0) {
    int active = 0, i0 = 0, k = 0, y = 0;
    if (!st->stopped) {
      const int a = st->action;
      if (MODE == TS_DOTS) active = a == ACT_EXTEND;
      else if (MODE == TS_UPD_DOTS) active = a == ACT_EXTEND && st->full_orth;
      else if (MODE == TS_UPD_NORM) active = a == ACT_EXTEND;
      else active = a == ACT_COMBINE;
    }
    if (active) {
      if (MODE == TS_COMBINE) { i0 = 0; k = st->mc; y = 0; }
      else { i0 = st->j0; k = st->j - st->j0 + 1; y = st->j + 1; }
    }
    const int nst = k + (MODE == TS_COMBINE ? 0 : 1);
    int T = kTsMaxT;
    while (T > min_T && max_stages * nst * T * 8 > budget) T >>= 1;
    int S = budget / (nst * T * 8);
    while (S < 2 && T > 64) {  // T >= 64: whole 32-lane pair rows
      T >>= 1;
      S = budget / (nst * T * 8);
    }
    S = S > max_stages ? max_stages : S;
    s_active = active; s_i0 = i0; s_k = k; s_y = y; s_T = T; s_S = S;
    s_ld = st->ld; s_n = st->n;
    s_ndot = st->tail_here ? st->ld : st->n;  // the replicated tail counts on rank 0 only
    if (active) {
      for (int q = 0; q < S; ++q) {
        mbar_init(&full[q], 1);
        mbar_init(&empty[q], kTsConsumers / 32);
      }
      fence_mbar_init();
    }
  }
  __syncthreads();
  if (!s_active) return;
  const int i0 = s_i0, k = s_k, T = s_T, S = s_S;
  const long long ld = s_ld, n = s_n, ndot = s_ndot;
  for (int i = tid; i < k; i += blockDim.x) {
    const int slot = i0 + i;
    const double sc = st->scale[slot];
    double c;
    if (MODE == TS_DOTS) c = 0.0;
    else if (MODE == TS_UPD_DOTS) c = sc * sc * st->red.dotA[slot];
    else if (MODE == TS_UPD_NORM) c = sc * sc * (st->full_orth ? st->red.dotB[slot] : st->red.dotA[slot]);
    else c = sc * st->comb[slot];
    s_coef[i] = c;
  }
  __syncthreads();
  const bool hasY = MODE != TS_COMBINE;
  const int nst = k + (hasY ? 1 : 0);
  double* ybase = base + (size_t)s_y * ld;
  const long long ntiles = ld / T;
  const uint32_t tile_bytes = (uint32_t)T * 8u;

  double acc[kAccPerLane];
#pragma unroll
  for (int v = 0; v < kAccPerLane; ++v) acc[v] = 0.0;
  double nacc = 0.0;

  if (wid == kTsConsumers / 32) {
    // ---------------- producer warp
    if (lane == 0) {
      int s = 0, use = 0;
      for (long long tl = blockIdx.x; tl < ntiles; tl += gridDim.x) {
        mbar_wait(&empty[s], (use & 1) ^ 1);
        double* dst = smem + (size_t)s * nst * T;
        mbar_arrive_expect_tx(&full[s], tile_bytes * (uint32_t)nst);
        for (int q = 0; q < k; ++q)
          bulk_g2s(dst + (size_t)q * T, base + (size_t)(i0 + q) * ld + tl * T, tile_bytes, &full[s]);
        if (hasY) bulk_g2s(dst + (size_t)k * T, ybase + tl * T, tile_bytes, &full[s]);
        if (++s == S) { s = 0; ++use; }
      }
    }
  } else {
    // ---------------- consumer warps
    const int nvw = (k + 7) / 8;
    if (MODE == TS_UPD_NORM || MODE == TS_COMBINE || nvw <= 1) ts_consume<MODE, 1>(st, base, smem, full, empty, s_coef, k, T, S, ntiles, n, ndot, nst, ybase, acc, nacc);
    else if (nvw <= 2) ts_consume<MODE, 2>(st, base, smem, full, empty, s_coef, k, T, S, ntiles, n, ndot, nst, ybase, acc, nacc);
    else if (nvw <= 3) ts_consume<MODE, 3>(st, base, smem, full, empty, s_coef, k, T, S, ntiles, n, ndot, nst, ybase, acc, nacc);
    else if (nvw <= 5) ts_consume<MODE, 5>(st, base, smem, full, empty, s_coef, k, T, S, ntiles, n, ndot, nst, ybase, acc, nacc);
    else if (nvw <= 8) ts_consume<MODE, 8>(st, base, smem, full, empty, s_coef, k, T, S, ntiles, n, ndot, nst, ybase, acc, nacc);
    else ts_consume<MODE, kAccPerLane>(st, base, smem, full, empty, s_coef, k, T, S, ntiles, n, ndot, nst, ybase, acc, nacc);
  }
  __syncthreads();

  // ---- deterministic reductions (all warps; the producer contributes zeros)
  if (MODE == TS_DOTS || MODE == TS_UPD_DOTS) {
#pragma unroll
    for (int v = 0; v < kAccPerLane; ++v) {
      const int i = wid + 8 * v;
      const double r = warp_sum(acc[v]);
      if (wid < kTsConsumers / 32 && i < k && lane == 0) s_red[i] = r;
    }
    __syncthreads();
    double* dst = MODE == TS_DOTS ? st->rs().dotA : st->rs().dotB;
    grid_reduce_last(s_red, k, partials, kMaxSlots, &st->ticket[MODE == TS_DOTS ? TK_DOTS : TK_UPD_DOTS],
                     [&](int i, double v) { dst[i0 + i] = v; });
  } else {
    const double tot = block_sum(nacc, s_buf);
    if (tid == 0) s_red[0] = tot;
    __syncthreads();
    grid_reduce_last(s_red, 1, partials, kMaxSlots, &st->ticket[MODE == TS_COMBINE ? TK_COMBINE : TK_UPD_NORM],
                     [&](int, double v) {
                       if (MODE == TS_COMBINE) st->rs().w2 = v;
                       else st->rs().nrmC = v;
                     });
  }
}

// ------------------------------------------------------------------ phi init
// w = [b_0; 0 ... 0, 1] (proj/src/phi.cpp:160-165); ||b_i||^2 for the all-zero
// early exit (proj/src/phi.cpp:141-145) and ||w_head||^2 for beta.
__global__ void __launch_bounds__(256) k_phi_init(PhiState* st, double* slot0, BArgs b, double* partials) {
  __shared__ double s_buf[8];
  __shared__ double s_red[kMaxP + 2];
  if (st->stopped) return;
  const long long n = st->n;
  double acc[kMaxP + 1];
#pragma unroll
  for (int i = 0; i <= kMaxP; ++i) acc[i] = 0.0;
  const long long stride = (long long)gridDim.x * blockDim.x;
  for (long long d = (long long)blockIdx.x * blockDim.x + threadIdx.x; d < n; d += stride) {
    const double w0 = b.b[0] ? b.b[0][d] : 0.0;
    slot0[d] = w0;
#pragma unroll
    for (int i = 0; i <= kMaxP; ++i)
      if (i <= b.p && b.b[i]) {
        const double v = b.b[i][d];
        acc[i] = fma(v, v, acc[i]);
      }
  }
  if (blockIdx.x == 0 && threadIdx.x < kTailPad)
    slot0[n + threadIdx.x] = (b.p > 0 && (int)threadIdx.x == b.p - 1) ? 1.0 : 0.0;
#pragma unroll
  for (int i = 0; i <= kMaxP; ++i) {
    const double t = block_sum(acc[i], s_buf);
    if (threadIdx.x == 0) s_red[i] = t;
  }
  __syncthreads();
  grid_reduce_last(s_red, kMaxP + 1, partials, kMaxSlots, &st->ticket[TK_INIT], [&](int i, double v) {
    st->rs().bnorm2[i] = v;
  });
}

// ------------------------------------------------------------------ block dense linear algebra
__device__ void blk_matmul(double* C, const double* A, const double* B, int N) {
  for (int idx = threadIdx.x; idx < N * N; idx += blockDim.x) {
    const int i = idx / N, j = idx - i * N;
    double s = 0.0;
    for (int k = 0; k < N; ++k) s = fma(A[i * N + k], B[k * N + j], s);
    C[idx] = s;
  }
  __syncthreads();
}

// out = sum c_m M_m + ident * I
__device__ void blk_lincomb(double* out, int N, int cnt, const double* c, const double* const* M, double ident) {
  for (int idx = threadIdx.x; idx < N * N; idx += blockDim.x) {
    double s = 0.0;
    for (int m = 0; m < cnt; ++m) s += c[m] * M[m][idx];
    if (idx / N == idx % N) s += ident;
    out[idx] = s;
  }
  __syncthreads();
}

// Solves A X = B (partial pivoting, first maximal pivot), B overwritten.
__device__ void blk_lu_solve(double* A, double* B, int N) {
  __shared__ int s_piv;
  const int tid = threadIdx.x;
  for (int k = 0; k < N; ++k) {
    if (tid < 32) {
      double best = -1.0;
      int bi = k;
      for (int i = k + tid; i < N; i += 32) {
        const double v = fabs(A[i * N + k]);
        if (v > best) { best = v; bi = i; }
      }
      for (int o = 16; o > 0; o >>= 1) {
        const double ov = __shfl_xor_sync(0xffffffffu, best, o);
        const int oi = __shfl_xor_sync(0xffffffffu, bi, o);
        if (ov > best || (ov == best && oi < bi)) { best = ov; bi = oi; }
      }
      if (tid == 0) s_piv = bi;
    }
    __syncthreads();
    const int p = s_piv;
    if (p != k) {
      for (int j = tid; j < N; j += blockDim.x) {
        double t = A[k * N + j]; A[k * N + j] = A[p * N + j]; A[p * N + j] = t;
        t = B[k * N + j]; B[k * N + j] = B[p * N + j]; B[p * N + j] = t;
      }
      __syncthreads();
    }
    const double d = A[k * N + k];
    for (int i = k + 1 + tid; i < N; i += blockDim.x) A[i * N + k] = A[i * N + k] / d;
    __syncthreads();
    const int rows = N - k - 1;
    for (int idx = tid; idx < rows * N; idx += blockDim.x) {
      const int i = k + 1 + idx / N, j = idx % N;
      const double l = A[i * N + k];
      if (j > k) A[i * N + j] -= l * A[k * N + j];
      B[i * N + j] -= l * B[k * N + j];
    }
    __syncthreads();
  }
  for (int j = tid; j < N; j += blockDim.x) {
    for (int i = N - 1; i >= 0; --i) {
      double s = B[i * N + j];
      for (int kk = i + 1; kk < N; ++kk) s -= A[i * N + kk] * B[kk * N + j];
      B[i * N + j] = s / A[i * N + i];
    }
  }
  __syncthreads();
}

// Higham (2005) scaling and squaring, the algorithm of Eigen's MatrixFunctions
// exp() (proj/src/phi.cpp:40).  A (N x N) in W[0]; result in *out (one of W's).
__device__ double* blk_expm(double* W, int N) {
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
  blk_matmul(A2, A, A, N);
  if (deg == 3) {
    const double b[] = {120.0, 60.0, 12.0, 1.0};
    { const double c[] = {b[3]}; const double* M[] = {A2}; blk_lincomb(T1, N, 1, c, M, b[1]); }
    blk_matmul(U, A, T1, N);
    { const double c[] = {b[2]}; const double* M[] = {A2}; blk_lincomb(V, N, 1, c, M, b[0]); }
  } else if (deg == 5) {
    const double b[] = {30240.0, 15120.0, 3360.0, 420.0, 30.0, 1.0};
    blk_matmul(A4, A2, A2, N);
    { const double c[] = {b[5], b[3]}; const double* M[] = {A4, A2}; blk_lincomb(T1, N, 2, c, M, b[1]); }
    blk_matmul(U, A, T1, N);
    { const double c[] = {b[4], b[2]}; const double* M[] = {A4, A2}; blk_lincomb(V, N, 2, c, M, b[0]); }
  } else if (deg == 7) {
    const double b[] = {17297280.0, 8648640.0, 1995840.0, 277200.0, 25200.0, 1512.0, 56.0, 1.0};
    blk_matmul(A4, A2, A2, N);
    blk_matmul(A6, A4, A2, N);
    { const double c[] = {b[7], b[5], b[3]}; const double* M[] = {A6, A4, A2}; blk_lincomb(T1, N, 3, c, M, b[1]); }
    blk_matmul(U, A, T1, N);
    { const double c[] = {b[6], b[4], b[2]}; const double* M[] = {A6, A4, A2}; blk_lincomb(V, N, 3, c, M, b[0]); }
  } else if (deg == 9) {
    const double b[] = {17643225600.0, 8821612800.0, 2075673600.0, 302702400.0, 30270240.0,
                        2162160.0,     110880.0,     3960.0,       90.0,        1.0};
    blk_matmul(A4, A2, A2, N);
    blk_matmul(A6, A4, A2, N);
    blk_matmul(A8, A6, A2, N);
    { const double c[] = {b[9], b[7], b[5], b[3]}; const double* M[] = {A8, A6, A4, A2}; blk_lincomb(T1, N, 4, c, M, b[1]); }
    blk_matmul(U, A, T1, N);
    { const double c[] = {b[8], b[6], b[4], b[2]}; const double* M[] = {A8, A6, A4, A2}; blk_lincomb(V, N, 4, c, M, b[0]); }
  } else {
    const double b[] = {64764752532480000.0, 32382376266240000.0, 7771770303897600.0,
                        1187353796428800.0,  129060195264000.0,   10559470521600.0,
                        670442572800.0,      33522128640.0,       1323241920.0,
                        40840800.0,          960960.0,            16380.0,
                        182.0,               1.0};
    blk_matmul(A4, A2, A2, N);
    blk_matmul(A6, A4, A2, N);
    { const double c[] = {b[13], b[11], b[9]}; const double* M[] = {A6, A4, A2}; blk_lincomb(T1, N, 3, c, M, 0.0); }
    blk_matmul(T2, A6, T1, N);
    { const double c[] = {1.0, b[7], b[5], b[3]}; const double* M[] = {T2, A6, A4, A2}; blk_lincomb(T1, N, 4, c, M, b[1]); }
    blk_matmul(U, A, T1, N);
    { const double c[] = {b[12], b[10], b[8]}; const double* M[] = {A6, A4, A2}; blk_lincomb(T1, N, 3, c, M, 0.0); }
    blk_matmul(T2, A6, T1, N);
    { const double c[] = {1.0, b[6], b[4], b[2]}; const double* M[] = {T2, A6, A4, A2}; blk_lincomb(V, N, 4, c, M, b[0]); }
  }
  // numer = U + V -> T1 ; denom = V - U -> T2 ; solve denom X = numer
  { const double c[] = {1.0, 1.0}; const double* M[] = {U, V}; blk_lincomb(T1, N, 2, c, M, 0.0); }
  { const double c[] = {-1.0, 1.0}; const double* M[] = {U, V}; blk_lincomb(T2, N, 2, c, M, 0.0); }
  blk_lu_solve(T2, T1, N);
  double* cur = T1;
  double* oth = A2;
  for (int i = 0; i < s_sq; ++i) {
    blk_matmul(oth, cur, cur, N);
    double* t = cur; cur = oth; oth = t;
  }
  return cur;
}

// Standalone device expm (one CTA) of an N x N matrix in W[0..N*N); result copied to out.
__global__ void __launch_bounds__(256) k_expm(double* W, int N, double* out) {
  const double* F = blk_expm(W, N);
  for (int i = threadIdx.x; i < N * N; i += blockDim.x) out[i] = F[i];
}

void device_expm(cudaStream_t s, double* work, int N, double* out) { k_expm<<<1, 256, 0, s>>>(work, N, out); }

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
__device__ int dcgs_finish(PhiState* st) {
  const int j = st->j;
  const double nd = (double)st->n;
  st->alg_bytes += 32.0 * nd + 8.0 * nd * (2.0 * j + 6.0);
  double beta = 1.0;
  if (j >= 1) {
    beta = st->scale[j] * sqrt(st->red.nrmU);
    for (int l = 0; l < j; ++l) st->H[l * kMaxBasis + (j - 1)] += st->dc_a[l];
    if (beta <= 1e-14 * fmax(st->pre_prev, 1e-300)) {
      st->H[j * kMaxBasis + (j - 1)] = 0.0;
      st->mc = j;
      st->breakdown = 1;
      return 1;
    }
    st->H[j * kMaxBasis + (j - 1)] = beta;
    st->scale[j] = 1.0 / sqrt(st->red.nrmU);  // V_j = slot_j / ||slot_j||
  }
  const double ib = 1.0 / beta;
  // column j = kMaxBasis (the avnorm cycle at mc = mmax = 128) has no storage and no
  // use: the space cannot grow past mmax
  const bool store = j < kMaxBasis;
  double hh = 0.0;
  for (int l = 0; l < j; ++l) {
    const double h = (st->dc_b[l] - st->dc_g[l]) * ib;
    if (store) st->H[l * kMaxBasis + j] = h;
    hh = fma(h, h, hh);
  }
  // the V_j coefficient the update pass actually removed (gamma from the Pythagorean
  // beta); the next cycle's reorthogonalisation adds the remainder
  const double gj = j >= 1 ? beta * st->dc_a[j - 1] : 0.0;
  const double hj = st->dc_gp - gj * ib;
  if (store) st->H[j * kMaxBasis + j] = hj;
  hh = fma(hj, hj, hh);
  st->scale[j + 1] = ib;                                   // u_{j+1} = slot_{j+1} / beta
  st->pre_prev = sqrt(st->red.nrmW * ib * ib + hh);        // ||dt A V_j|| (incl. the augmentation)
  return 0;
}

__device__ __forceinline__ void ctl_body(PhiState* st, double* slot0, double* W, double* Wsm, int ws_cap,
                                         cudaGraphConditionalHandle cond, int use_graph) {
  __shared__ int s_phase, s_exit, s_zeroH, s_done;
  const int tid = threadIdx.x;
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
            if (dcgs_finish(st)) {
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
          const int j = st->j;
          const double* sc = st->scale;
          for (int i = st->j0; i <= j; ++i) {
            const double h1 = sc[i] * st->red.dotA[i];
            const double h2 = st->full_orth ? sc[i] * st->red.dotB[i] : 0.0;
            st->H[i * kMaxBasis + j] = st->full_orth ? (h1 + h2) : h1;
          }
          {
            const double nd = (double)st->n, kk = (double)(j - st->j0 + 1);
            st->alg_bytes += 32.0 * nd + 8.0 * nd * (st->full_orth ? 3.0 * kk + 6.0 : 2.0 * kk + 4.0);
            st->extend_cols++;
          }
          const double pre_norm = sqrt(st->red.nrmA);
          const double hnext = sqrt(st->red.nrmC);
          st->pre_norm = pre_norm;
          st->H[(j + 1) * kMaxBasis + j] = hnext;
          const int mc = j + 1;
          st->mc = mc;
          st->iterations++;
          if (hnext <= 1e-14 * fmax(pre_norm, 1e-300)) {
            st->H[mc * kMaxBasis + (mc - 1)] = 0.0;
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
            if (dcgs_finish(st)) {
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
        if (i <= mc && j < mc) v = st->H[i * kMaxBasis + j];
        if (i == mc + 1 && j == mc) v = 1.0;
        Wx[idx] = h * v;
      }
      __syncthreads();
      const double* F = blk_expm(9 * N * N <= ws_cap ? Wsm : W, N);
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
        if (!st->breakdown) {
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
    for (int idx = tid; idx < rows * kMaxBasis; idx += blockDim.x) st->H[idx] = 0.0;
  }
  if (tid == 0) st->phase = s_phase;
  if (tid == 0 && s_done && use_graph) cudaGraphSetConditional(cond, 0u);
}

__global__ void __launch_bounds__(256) k_ctl(PhiState* st, double* slot0, double* W,
                                             cudaGraphConditionalHandle cond, int use_graph) {
  ctl_body(st, slot0, W, nullptr, 0, cond, use_graph);
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
// buffer, then every CTA sums all of them in rank order (identical totals).  CTA 0
// holds PhiState in shared memory and runs the controller (ctl_body); the others read
// its decisions through DSMEM.  No basis traffic leaves the SMs.
namespace cg = cooperative_groups;
constexpr int kClusterCTAs = 8;
constexpr int kClusterThreads = 256;

template <class EL>
__global__ void __launch_bounds__(kClusterThreads, 1)
    k_phi_cluster(PhiState* gst, double* base, double* W, BArgs b, EL el, int epc, int lds, int nslots,
                  int ws_cap, int state_off, int ws_off) {
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
  if (rank == 0) {
    if (tid == 0) s_hb = sizeof(double) * (size_t)min(gst->mmax + 2, kMaxBasis + 1) * kMaxBasis;
    __syncthreads();
    state_copy(reinterpret_cast<unsigned char*>(st0), reinterpret_cast<const unsigned char*>(gst), s_hb);
  }
  const PhiState* S = cl.map_shared_rank(st0, 0);
  const int nsc = nslots < kMaxSlots ? nslots : kMaxSlots;
  // CTA 0 pushes the controller's decision (action, column, scales) into every CTA's
  // shared memory, so the other CTAs never chase scalars through DSMEM
  auto push = [&]() {
    __syncthreads();
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
  if (rank == 0) push();
  cl.sync();
  int round = 0;
  // cluster totals of cnt partial sums in s_mine -> s_tot (every CTA, rank order)
  auto reduce = [&](int cnt) {
    double* buf = part + (round & 1) * (2 * kMaxSlots + 2);
    for (int i = tid; i < cnt; i += T) buf[i] = s_mine[i];
    cl.sync();
    for (int i = tid; i < cnt; i += T) {
      double sum = 0.0;
      for (int r = 0; r < CS; ++r) sum += cl.map_shared_rank(buf, r)[i];
      s_tot[i] = sum;
    }
    __syncthreads();
    ++round;
  };
  // this CTA's <V_{i0+i}, y> for i < k, one warp per vector (the tail counts on rank 0)
  auto local_dots = [&](int i0, int k, const double* y) {
    for (int i = wid; i < k; i += T / 32) {
      const double* v = V + (size_t)(i0 + i) * lds;
      double p0 = 0.0, p1 = 0.0;
      for (int d = lane; d < nloc; d += 64) {
        p0 = fma(v[d], y[d], p0);
        if (d + 32 < nloc) p1 = fma(v[d + 32], y[d + 32], p1);
      }
      if (s_tailhere && lane < kTailPad) p0 = fma(v[tail_at + lane], y[tail_at + lane], p0);
      const double p = warp_sum(p0 + p1);
      if (lane == 0) s_mine[i] = p;
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
      if (tid == 0) s_mine[0] = tot;
      __syncthreads();
      reduce(1);
      if (rank == 0 && tid == 0) st0->red.nrmA = s_tot[0];
      mark(0);
      if (act == ACT_EXTEND) {  // CGS2 passes (krylov.cu coefficients) or one IOP pass
        const int i0 = s_j0, k = j - i0 + 1;
        local_dots(i0, k, y);
        reduce(k);
        if (rank == 0)
          for (int i = tid; i < k; i += T) st0->red.dotA[i0 + i] = s_tot[i];
        mark(1);
        if (s_full) {
          for (int i = tid; i < k; i += T) s_c[i] = s_scale[i0 + i] * s_scale[i0 + i] * s_tot[i];
          __syncthreads();
          local_update(i0, k, y);
          __syncthreads();
          mark(2);
          local_dots(i0, k, y);
          reduce(k);
          mark(1);
          if (rank == 0)
            for (int i = tid; i < k; i += T) st0->red.dotB[i0 + i] = s_tot[i];
        }
        for (int i = tid; i < k; i += T) s_c[i] = s_scale[i0 + i] * s_scale[i0 + i] * s_tot[i];
        __syncthreads();
        const double nn = block_sum(local_update(i0, k, y), s_buf);
        if (tid == 0) s_mine[0] = nn;
        __syncthreads();
        reduce(1);
        if (rank == 0 && tid == 0) st0->red.nrmC = s_tot[0];
        mark(2);
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
      if (rank == 0 && tid == 0) st0->red.w2 = s_tot[0];
      mark(3);
    }
    if (rank == 0) {
      __syncthreads();
      // the controller writes the phi tail into CTA 0's slot-0 tail (slot0[n + j])
      ctl_body(st0, V + tail_at - n, W, Wsm, ws_cap, cudaGraphConditionalHandle{}, 0);
      push();
    }
    cl.sync();
    if (act == ACT_COMBINE && rank != 0 && tid < kTailPad)  // replicate the reset tail
      V[tail_at + tid] = cl.map_shared_rank(V, 0)[tail_at + tid];
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
  EXPDG_CUDA(cudaLaunchKernelEx(&cfg, k_phi_cluster<EL>, e.st, e.base, e.ework, b, el, epc, lds, nslots,
                                9 * nws * nws, (int)state_off, (int)(state_off + state)));
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

template void launch_phi_fused<B1FusedElem<2>>(cudaStream_t, Engine&, const B1FusedElem<2>&, const BArgs&);
template void launch_phi_fused<B1FusedElem<3>>(cudaStream_t, Engine&, const B1FusedElem<3>&, const BArgs&);
template void launch_phi_fused<B1FusedElem<4>>(cudaStream_t, Engine&, const B1FusedElem<4>&, const BArgs&);
template void launch_phi_fused<B1FusedElem<5>>(cudaStream_t, Engine&, const B1FusedElem<5>&, const BArgs&);
template void launch_phi_fused<B1FusedElem<6>>(cudaStream_t, Engine&, const B1FusedElem<6>&, const BArgs&);
template void launch_phi_fused<B1FusedElem<7>>(cudaStream_t, Engine&, const B1FusedElem<7>&, const BArgs&);
template void launch_phi_fused<B1FusedElem<8>>(cudaStream_t, Engine&, const B1FusedElem<8>&, const BArgs&);
template void launch_phi_fused<B1FusedElem<9>>(cudaStream_t, Engine&, const B1FusedElem<9>&, const BArgs&);
#define FUSED_OI(NP, NQ) \
  template void launch_phi_fused<B1OIFusedElem<NP, NQ>>(cudaStream_t, Engine&, const B1OIFusedElem<NP, NQ>&, const BArgs&);
FUSED_OI(2, 3)
FUSED_OI(3, 4)
FUSED_OI(4, 6)
FUSED_OI(5, 7)
FUSED_OI(6, 9)
FUSED_OI(7, 10)
FUSED_OI(8, 12)
FUSED_OI(9, 13)
#undef FUSED_OI

// Sets action = START / DONE after the init reduction (separate tiny kernel so the
// decision sees the fully reduced norms).
__global__ void k_phi_start(PhiState* st) {
  if (st->stopped) return;
  if (st->step_failed) {  // an earlier phi call of this step failed: skip this one
    st->action = ACT_DONE;
    return;
  }
  int any = 0;
  for (int i = 0; i <= st->p; ++i) any |= st->red.bnorm2[i] > 0.0;
  st->any_b = any;
  st->iterations = 0;
  st->substeps = 0;
  st->cycles = 0;
  st->t = 0.0;
  st->h = 1.0;
  st->m = min(st->initial_basis, st->mmax);
  st->mc = 0;
  st->breakdown = 0;
  st->last_estimate = 0.0;
  st->red.w2 = st->red.bnorm2[0] + (st->p > 0 ? 1.0 : 0.0);
  // partitioned: the body's allreduces rebuild red from loc before the controller reads it
  if (st->multi) st->loc.w2 = st->loc.bnorm2[0] + ((st->p > 0 && st->tail_here) ? 1.0 : 0.0);
  for (int j = 0; j < kMaxP; ++j) st->tailw[j] = (j == st->p - 1) ? 1.0 : 0.0;
  if (st->domain_flag) {
    st->status = PHI_ERR_DOMAIN;
    st->step_failed = 1;
    st->action = ACT_DONE;
  } else if (!any) {
    st->status = PHI_OK;
    st->action = ACT_DONE;
  } else {
    st->status = PHI_RUNNING;
    st->action = ACT_START;
  }
  st->phase = PH_SUBSTEP;
}

// ------------------------------------------------------------------ host side
Engine::Engine(int dev) : device(dev) {
  EXPDG_CUDA(cudaSetDevice(dev));
  EXPDG_CUDA(cudaDeviceGetAttribute(&num_sms, cudaDevAttrMultiProcessorCount, dev));
  EXPDG_CUDA(cudaStreamCreateWithFlags(&stream, cudaStreamNonBlocking));
  EXPDG_CUDA(cudaMalloc(&st, sizeof(PhiState)));
  EXPDG_CUDA(cudaMemset(st, 0, sizeof(PhiState)));
  EXPDG_CUDA(cudaMallocHost(&st_host, sizeof(PhiState)));
  EXPDG_CUDA(cudaMalloc(&partials, sizeof(double) * kMaxPartials * kMaxSlots));
  ework_doubles = size_t(9) * (kMaxBasis + 2) * (kMaxBasis + 2);
  EXPDG_CUDA(cudaMalloc(&ework, sizeof(double) * ework_doubles));
  const int maxsm = 200 * 1024;
  EXPDG_CUDA(cudaFuncSetAttribute(k_ts<TS_DOTS>, cudaFuncAttributeMaxDynamicSharedMemorySize, maxsm));
  EXPDG_CUDA(cudaFuncSetAttribute(k_ts<TS_UPD_DOTS>, cudaFuncAttributeMaxDynamicSharedMemorySize, maxsm));
  EXPDG_CUDA(cudaFuncSetAttribute(k_ts<TS_UPD_NORM>, cudaFuncAttributeMaxDynamicSharedMemorySize, maxsm));
  EXPDG_CUDA(cudaFuncSetAttribute(k_ts<TS_COMBINE>, cudaFuncAttributeMaxDynamicSharedMemorySize, maxsm));
  if (const char* v = std::getenv("EXPDG_TS_BUDGET")) ts_tuning.budget = std::atoi(v);
  if (const char* v = std::getenv("EXPDG_TS_STAGES")) ts_tuning.stages = std::atoi(v);
  if (const char* v = std::getenv("EXPDG_TS_MIN_T")) ts_tuning.min_T = std::atoi(v);
  if (const char* v = std::getenv("EXPDG_LD_ODD")) ld_odd = std::atoi(v);
  if (const char* v = std::getenv("EXPDG_FUSED")) use_fused = std::atoi(v);
  if (const char* v = std::getenv("EXPDG_ORTH"))
    use_dcgs = std::strcmp(v, "cgs2") == 0 ? 0 : (std::strcmp(v, "dcgs2") == 0 ? 2 : 1);
  dcgs_init_attrs(maxsm);
}

Engine::~Engine() {
  cudaFree(base);
  cudaFree(st);
  cudaFreeHost(st_host);
  cudaFree(partials);
  cudaFree(ework);
  cudaFree(scratch);
  if (stream) cudaStreamDestroy(stream);
}

// Slot stride: a multiple of kLdAlign doubles, and for vectors past 2 MB an odd
// number of 2 MB pages so the k concurrent basis streams spread over all TLB
// sets (8-set x 16-way, 2 MB pages) instead of aliasing into one.
static long long slot_stride(long long len, int odd) {
  long long ld = round_up(len + kTailPad, kLdAlign);
  const long long page = (2LL << 20) / 8;  // doubles per 2 MB page
  if (odd && ld > page) {
    ld = round_up(ld, page);
    if ((ld / page) % 2 == 0) ld += page;
  }
  return ld;
}

void Engine::ensure(long long len, int mmax) {
  const long long need_ld = slot_stride(len, ld_odd);
  const int need_slots = mmax + 2;
  if (base && need_ld == ld && need_slots <= slots) {
    // the zero padding beyond [0, len) must hold for every slot: clear stale
    // data from a previous call with a longer vector
    if (len != cur_len) EXPDG_CUDA(cudaMemsetAsync(base, 0, sizeof(double) * (size_t)ld * slots, stream));
    cur_len = len;
    return;
  }
  cur_len = len;
  if (base) EXPDG_CUDA(cudaFree(base));
  base = nullptr;
  ld = need_ld;
  slots = need_slots;
  EXPDG_CUDA(cudaMalloc(&base, sizeof(double) * (size_t)ld * slots));
  EXPDG_CUDA(cudaMemset(base, 0, sizeof(double) * (size_t)ld * slots));
}

void Engine::ensure_scratch(long long len, int count) {
  const long long need = round_up(len + kTailPad, kLdAlign);
  if (scratch && scratch_ld >= need && scratch_count >= count) return;
  if (scratch) EXPDG_CUDA(cudaFree(scratch));
  scratch_ld = need;
  scratch_count = count;
  EXPDG_CUDA(cudaMalloc(&scratch, sizeof(double) * (size_t)need * count));
  EXPDG_CUDA(cudaMemset(scratch, 0, sizeof(double) * (size_t)need * count));
}

PhiState Engine::config(long long n, int p, double dt, const expdg_krylov_cfg& kc) const {
  PhiState c;
  std::memset(&c, 0, sizeof(c));
  c.n = n;
  c.p = p;
  c.tail_here = comm ? (comm->rank == 0 ? 1 : 0) : 1;
  c.multi = comm ? 1 : 0;
  c.len = n + p;
  c.ld = ld;
  c.dt = dt;
  c.tol = std::max(kc.tol, 5e-15);  // proj/src/phi.cpp:167
  const long long dim = n + p;
  c.mmax = (int)std::min<long long>(kc.max_basis, dim);  // :168
  c.initial_basis = kc.initial_basis > 0 ? kc.initial_basis : 16;
  c.max_substeps = kc.max_substeps > 0 ? kc.max_substeps : 40;
  const int orth = kc.orth_length;
  c.full_orth = (orth >= c.mmax || dim <= std::max(c.initial_basis, 16)) ? 1 : 0;  // :171-173
  c.window = c.full_orth ? c.mmax : orth;
  // DCGS2 saves a streaming pass per column; below ~2^18 DOF the passes are launch-
  // latency bound and CGS2's lighter kernels win (C1: 789 vs 904 us/step)
  c.dcgs = (c.full_orth && use_dcgs && (use_dcgs == 2 || n >= (1LL << 18))) ? 1 : 0;
  c.grow_cap = c.full_orth ? c.mmax : std::min(c.mmax, 32);  // :177
  c.max_cycles = 200000;
  c.action = ACT_NONE;
  return c;
}

// Uploads only the configuration prefix of PhiState (dynamic fields are reset on device).
void Engine::upload_config(const PhiState& c, cudaStream_t s) {
  std::memcpy(st_host, &c, sizeof(PhiState));
  EXPDG_CUDA(cudaMemcpyAsync(st, st_host, sizeof(PhiState), cudaMemcpyHostToDevice, s));
}

void Engine::reduce(cudaStream_t s) {
  if (!comm) return;
  constexpr long long cnt = sizeof(PhiState::Red) / sizeof(double);
  const char* p = reinterpret_cast<const char*>(st);
  comm->allreduce(p + offsetof(PhiState, loc), const_cast<char*>(p) + offsetof(PhiState, red), cnt, COMM_F64,
                  COMM_SUM, s);
}

void Engine::launch_phi_init(cudaStream_t s, const BArgs& b) {
  const int grid = num_sms * 2;
  k_phi_init<<<grid, 256, 0, s>>>(st, slot(0), b, partials);
  reduce(s);
  k_phi_start<<<1, 1, 0, s>>>(st);
}

static int ts_grid(const Engine& e) {
  const long long tiles = e.ld / 128;
  const int per_sm = e.ts_tuning.budget > 113 * 1024 ? 1 : 2;
  return (int)std::max<long long>(1, std::min<long long>((long long)per_sm * e.num_sms, tiles));
}

void Engine::launch_ts(cudaStream_t s, int mode) {
  const int g = ts_grid(*this);
  const TsTuning& t = ts_tuning;
  switch (mode) {
    case TS_DOTS: k_ts<TS_DOTS><<<g, kTsBlock, t.budget, s>>>(st, base, partials, t.budget, t.stages, t.min_T); break;
    case TS_UPD_DOTS: k_ts<TS_UPD_DOTS><<<g, kTsBlock, t.budget, s>>>(st, base, partials, t.budget, t.stages, t.min_T); break;
    case TS_UPD_NORM: k_ts<TS_UPD_NORM><<<g, kTsBlock, t.budget, s>>>(st, base, partials, t.budget, t.stages, t.min_T); break;
    default: k_ts<TS_COMBINE><<<g, kTsBlock, t.budget, s>>>(st, base, partials, t.budget, t.stages, t.min_T); break;
  }
}

void Engine::launch_body(cudaStream_t s, OpDevice& op, const BArgs& b, cudaGraphConditionalHandle h,
                         int use_graph, bool dcgs) {
  op.launch_phi_apply(s, st, base, partials, b);
  reduce(s);
  if (dcgs) {  // one dots pass + coefficients + one update pass (dcgs.cu)
    launch_dcgs(s, *this, 0);
    reduce(s);
    launch_dcgs(s, *this, 1);
    launch_dcgs(s, *this, 2);
    reduce(s);
    launch_ts(s, TS_COMBINE);
    reduce(s);
    k_ctl<<<1, 256, 0, s>>>(st, slot(0), ework, h, use_graph);
    return;
  }
  if (!op.fused_dots()) {
    launch_ts(s, TS_DOTS);
    reduce(s);
  }
  launch_ts(s, TS_UPD_DOTS);
  reduce(s);
  launch_ts(s, TS_UPD_NORM);
  reduce(s);
  launch_ts(s, TS_COMBINE);
  reduce(s);
  k_ctl<<<1, 256, 0, s>>>(st, slot(0), ework, h, use_graph);
}

// Micro-benchmark of one tall-skinny pass at column k-1 (diagnostics / tuning).
double Engine::bench_ts(long long n, int k, int mode, int reps) {
  ensure(n + 1, k + 1);
  PhiState c;
  std::memset(&c, 0, sizeof(c));
  c.n = n;
  c.len = n + 1;
  c.ld = ld;
  c.p = 1;
  c.tail_here = 1;
  c.full_orth = 1;
  c.mmax = k + 1;
  c.action = mode == TS_COMBINE ? ACT_COMBINE : ACT_EXTEND;
  c.j0 = 0;
  c.j = k - 1;
  c.mc = k;
  for (int i = 0; i < kMaxSlots; ++i) {
    c.scale[i] = 1.0;
    c.red.dotA[i] = 1e-3;
    c.red.dotB[i] = 1e-3;
    c.comb[i] = 1e-3;
  }
  upload_config(c, stream);
  cudaEvent_t a, b;
  EXPDG_CUDA(cudaEventCreate(&a));
  EXPDG_CUDA(cudaEventCreate(&b));
  launch_ts(stream, mode);  // warm-up
  EXPDG_CUDA(cudaEventRecord(a, stream));
  for (int r = 0; r < reps; ++r) launch_ts(stream, mode);
  EXPDG_CUDA(cudaEventRecord(b, stream));
  EXPDG_CUDA(cudaEventSynchronize(b));
  float ms = 0.f;
  EXPDG_CUDA(cudaEventElapsedTime(&ms, a, b));
  cudaEventDestroy(a);
  cudaEventDestroy(b);
  EXPDG_CUDA(cudaGetLastError());
  return ms / reps;
}

bool Engine::fused_ok(const OpDevice& op) const {
  return use_fused && !comm && !st_host->dcgs && op.fused_capable();
}

void Engine::run_phi(OpDevice& op, const BArgs& b, int use_graph) {
  if (fused_ok(op)) {  // small problem: the whole call in one single-CTA kernel
    launch_phi_init(stream, b);
    op.launch_fused(stream, *this, b);
    EXPDG_CUDA(cudaStreamSynchronize(stream));
    return;
  }
  if (use_graph && !comm) {
    cudaGraphExec_t ex = build_phi_graph(op, b);
    EXPDG_CUDA(cudaGraphLaunch(ex, stream));
    EXPDG_CUDA(cudaStreamSynchronize(stream));
    cudaGraphExecDestroy(ex);
    return;
  }
  launch_phi_init(stream, b);
  for (int cyc = 0; cyc < 1000000; ++cyc) {
    launch_body(stream, op, b, cudaGraphConditionalHandle{}, 0, st_host->dcgs != 0);
    EXPDG_CUDA(cudaMemcpyAsync(st_host, st, sizeof(PhiState), cudaMemcpyDeviceToHost, stream));
    EXPDG_CUDA(cudaStreamSynchronize(stream));
    if (st_host->action == ACT_DONE || st_host->action == ACT_NONE || st_host->stopped) return;
  }
  throw std::runtime_error("phi host loop did not terminate");
}

cudaGraphExec_t Engine::build_phi_graph(OpDevice& op, const BArgs& b) {
  cudaGraph_t g;
  EXPDG_CUDA(cudaGraphCreate(&g, 0));
  cudaStream_t cs;
  EXPDG_CUDA(cudaStreamCreateWithFlags(&cs, cudaStreamNonBlocking));
  // init part
  EXPDG_CUDA(cudaStreamBeginCaptureToGraph(cs, g, nullptr, nullptr, 0, cudaStreamCaptureModeRelaxed));
  launch_phi_init(cs, b);
  cudaGraphConditionalHandle h;
  EXPDG_CUDA(cudaGraphConditionalHandleCreate(&h, g, 1, cudaGraphCondAssignDefault));
  cudaStreamCaptureStatus cst;
  const cudaGraphNode_t* deps = nullptr;
  size_t ndeps = 0;
  cudaGraph_t cg;
  EXPDG_CUDA(cudaStreamGetCaptureInfo(cs, &cst, nullptr, &cg, &deps, &ndeps));
  cudaGraphNodeParams cp = {};
  cp.type = cudaGraphNodeTypeConditional;
  cp.conditional.handle = h;
  cp.conditional.type = cudaGraphCondTypeWhile;
  cp.conditional.size = 1;
  cudaGraphNode_t cnode;
  EXPDG_CUDA(cudaGraphAddNode(&cnode, g, deps, ndeps, &cp));
  EXPDG_CUDA(cudaStreamUpdateCaptureDependencies(cs, &cnode, 1, cudaStreamSetCaptureDependencies));
  EXPDG_CUDA(cudaStreamEndCapture(cs, &g));
  cudaGraph_t body = cp.conditional.phGraph_out[0];
  EXPDG_CUDA(cudaStreamBeginCaptureToGraph(cs, body, nullptr, nullptr, 0, cudaStreamCaptureModeRelaxed));
  launch_body(cs, op, b, h, 1, st_host->dcgs != 0);
  EXPDG_CUDA(cudaStreamEndCapture(cs, &body));
  cudaGraphExec_t ex;
  EXPDG_CUDA(cudaGraphInstantiate(&ex, g, 0));
  cudaGraphDestroy(g);
  cudaStreamDestroy(cs);
  return ex;
}

// ------------------------------------------------------------------ utilities
__global__ void k_axpy_into(double* u, const double* w, long long n) {
  const long long stride = (long long)gridDim.x * blockDim.x;
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride) u[i] += w[i];
}
__global__ void k_copy(double* d, const double* s, long long n) {
  const long long stride = (long long)gridDim.x * blockDim.x;
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride) d[i] = s[i];
}
void launch_axpy_into(cudaStream_t s, double* u, const double* w, long long n) {
  k_axpy_into<<<592, 256, 0, s>>>(u, w, n);
}
void launch_copy(cudaStream_t s, double* dst, const double* src, long long n) {
  k_copy<<<592, 256, 0, s>>>(dst, src, n);
}

}  // namespace expdg
