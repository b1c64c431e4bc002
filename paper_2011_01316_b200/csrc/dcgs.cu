// DCGS2 Arnoldi passes: classical Gram-Schmidt with delayed reorthogonalisation
// (one dots pass + one update pass per Krylov column; CGS2 needs three).
//
// The reference orthogonalises every new column twice with modified Gram-Schmidt
// (proj/src/phi.cpp:94-100).  Here the second projection of column j-1 is lagged
// into the passes of column j: slot j holds the once-projected candidate u_j, the
// operator is applied to it (w = dt A u_j, the JVP kernel), and
//   pass 1 (k_ts2<TS2_DOTS>):  a = V^T u, b = V^T w, <u,u>, <u,w>   over V_0..V_{j-1}, u, w
//   coefficients (k_dcgs_coef): reorthogonalisation of u, projection of w
//   pass 2 (k_ts2<TS2_UPD>):   u <- u - V a (= beta V_j), w <- w - gamma u - V mu (= beta u_{j+1}),
//                              exact ||u||^2, ||w||^2
// Because A V_i = V H(:, i) for the finished columns, the projections of A V_j
// follow from a, b and H without another pass; the controller finishes column
// j-1 (H += a, H(j, j-1) = exact ||u - V a||) and writes column j provisionally.
// The projector is the same as CGS2 / MGS2 in exact arithmetic; the only
// Pythagorean quantity is the coefficient gamma of the candidate direction, whose
// rounding error the next column's reorthogonalisation removes.
#include "krylov.cuh"

namespace expdg {

enum Ts2Mode { TS2_DOTS = 0, TS2_UPD = 1 };
constexpr int kT2Consumers = 256;
constexpr int kT2Block = kT2Consumers + 32;
constexpr int kT2MaxT = 2048;
constexpr int kT2Chunk = 256;
constexpr int kT2Acc = (kMaxSlots + 7) / 8;

// Pass-1 dots of one staged tile: acc1[v] += <V_i, U>, acc2[v] += <V_i, W> for the vectors
// i = wid + 8 v <= j (i = j: U itself).  Streams of the tile: V_0..V_{j-1}, U, W consecutive.
template <int NV, int NA>
__device__ __forceinline__ void ts2_tile_dots(const double* V, int j, int T, int lane, int wid,
                                              double (&acc1)[NA], double (&acc2)[NA], int len = -1) {
  const int T2 = T >> 1;  // stream stride in the tile; len (a multiple of 64) <= T doubles are valid
  if (len < 0) len = T;
  const double2* V2 = reinterpret_cast<const double2*>(V);
  const double2* U2 = reinterpret_cast<const double2*>(V + (size_t)j * T);
  const double2* W2 = U2 + T2;
  for (int c0 = 0; c0 < len; c0 += kT2Chunk) {
    const int per = min(len - c0, kT2Chunk) >> 6;
    double2 yu[kT2Chunk / 64], yw[kT2Chunk / 64];
#pragma unroll
    for (int m = 0; m < kT2Chunk / 64; ++m) {
      yu[m] = m < per ? U2[(c0 >> 1) + lane + 32 * m] : make_double2(0.0, 0.0);
      yw[m] = m < per ? W2[(c0 >> 1) + lane + 32 * m] : make_double2(0.0, 0.0);
    }
#pragma unroll
    for (int v = 0; v < NV; ++v) {
      const int i = wid + 8 * v;  // vectors 0..j (j = the candidate itself)
      if (i <= j) {
        const double2* Vi = V2 + (size_t)i * T2 + (c0 >> 1) + lane;
        double a0 = 0.0, a1 = 0.0, b0 = 0.0, b1 = 0.0;
#pragma unroll
        for (int m = 0; m < kT2Chunk / 64; ++m) {
          if (m < per) {
            const double2 x = Vi[32 * m];
            a0 = fma(x.x, yu[m].x, a0);
            a1 = fma(x.y, yu[m].y, a1);
            b0 = fma(x.x, yw[m].x, b0);
            b1 = fma(x.y, yw[m].y, b1);
          }
        }
        acc1[v] += a0 + a1;
        acc2[v] += b0 + b1;
      }
    }
  }
}

// A non-zero rank's tile holding the replicated phi tail: U, W (streams j, j+1) beyond ndot
// are kept out of the dots.  Consumer-wide.
__device__ __forceinline__ void ts2_mask_tail(double* V, int j, int T, long long g0, long long ndot, int tid,
                                              int len = -1) {
  if (len < 0) len = T;
  if (g0 + len <= ndot) return;
  double* U = V + (size_t)j * T;
  double* W = U + T;
  consumer_sync();
  for (int d = tid; d < len; d += kT2Consumers)
    if (g0 + d >= ndot) {
      U[d] = 0.0;
      W[d] = 0.0;
    }
  consumer_sync();
}

// Consumer warps.  Streams of a tile: V_0..V_{j-1}, U (= slot j), W (= slot j+1).
template <int MODE, int NV>
__device__ __forceinline__ void ts2_consume(double* base, double* smem, uint64_t* full, uint64_t* empty,
                                            const double* s_al, const double* s_mu, double gam, double wsc, int j,
                                            int T, int S, long long ntiles, long long ld, long long ndot, int nst,
                                            double (&acc1)[kT2Acc], double (&acc2)[kT2Acc], double& nu, double& nw) {
  const int tid = threadIdx.x;
  const int lane = tid & 31, wid = tid >> 5;
  const int T2 = T >> 1;
  const double2* AL2 = reinterpret_cast<const double2*>(s_al);
  const double2* MU2 = reinterpret_cast<const double2*>(s_mu);
  double2* ug = reinterpret_cast<double2*>(base + (size_t)j * ld);
  double2* wg = reinterpret_cast<double2*>(base + (size_t)(j + 1) * ld);
  int s = 0, use = 0;
  for (long long tl = blockIdx.x; tl < ntiles; tl += gridDim.x) {
    mbar_wait(&full[s], use & 1);
    double* V = smem + (size_t)s * nst * T;
    double* U = V + (size_t)j * T;
    double* W = U + T;
    const double2* V2 = reinterpret_cast<const double2*>(V);
    const long long g0 = tl * T;
    if (MODE == TS2_DOTS) {
      ts2_mask_tail(V, j, T, g0, ndot, tid);
      ts2_tile_dots<NV>(V, j, T, lane, wid, acc1, acc2);
    } else {
      const double2* U2 = reinterpret_cast<const double2*>(U);
      const double2* W2 = reinterpret_cast<const double2*>(W);
      for (int p = tid; p < T2; p += kT2Consumers) {
        const double2 u = U2[p];
        const double2 w = W2[p];
        double ua0 = u.x, ua1 = u.y, ub0 = 0.0, ub1 = 0.0;
        // W_true = wsc * slot_{j+1} (wsc = 1 after a stage-1 application: bit-identical to w)
        double wa0 = fma(-gam, u.x, wsc * w.x), wa1 = fma(-gam, u.y, wsc * w.y), wb0 = 0.0, wb1 = 0.0;
        int i = 0;
        for (; i + 1 < j; i += 2) {
          const double2 al = AL2[i >> 1], mu = MU2[i >> 1];
          const double2 v0 = V2[(size_t)i * T2 + p];
          const double2 v1 = V2[(size_t)(i + 1) * T2 + p];
          ua0 = fma(-al.x, v0.x, ua0);
          ua1 = fma(-al.x, v0.y, ua1);
          wa0 = fma(-mu.x, v0.x, wa0);
          wa1 = fma(-mu.x, v0.y, wa1);
          ub0 = fma(-al.y, v1.x, ub0);
          ub1 = fma(-al.y, v1.y, ub1);
          wb0 = fma(-mu.y, v1.x, wb0);
          wb1 = fma(-mu.y, v1.y, wb1);
        }
        if (i < j) {
          const double al = s_al[i], mu = s_mu[i];
          const double2 v0 = V2[(size_t)i * T2 + p];
          ua0 = fma(-al, v0.x, ua0);
          ua1 = fma(-al, v0.y, ua1);
          wa0 = fma(-mu, v0.x, wa0);
          wa1 = fma(-mu, v0.y, wa1);
        }
        const double2 un = make_double2(ua0 + ub0, ua1 + ub1);
        const double2 wn = make_double2(wa0 + wb0, wa1 + wb1);
        ug[(g0 >> 1) + p] = un;
        wg[(g0 >> 1) + p] = wn;
        if (g0 + 2 * p < ndot) {
          nu = fma(un.x, un.x, nu);
          nw = fma(wn.x, wn.x, nw);
        }
        if (g0 + 2 * p + 1 < ndot) {
          nu = fma(un.y, un.y, nu);
          nw = fma(wn.y, wn.y, nw);
        }
      }
    }
    __syncwarp();
    if (lane == 0) mbar_arrive(&empty[s]);
    if (++s == S) {
      s = 0;
      ++use;
    }
  }
}

template <int MODE>
__global__ void __launch_bounds__(kT2Block, 1) k_ts2(PhiState* st, double* base, double* partials, int budget,
                                                     int max_stages, int min_T, int fused_jmax) {
  extern __shared__ __align__(128) double smem[];
  __shared__ uint64_t full[8], empty[8];
  __shared__ int s_active, s_j, s_T, s_S;
  __shared__ long long s_ld, s_ndot;
  __shared__ double s_gam, s_wsc;
  __shared__ __align__(16) double s_al[kMaxSlots + 2];
  __shared__ __align__(16) double s_mu[kMaxSlots + 2];
  __shared__ double s_red[2 * kMaxSlots + 2];
  __shared__ double s_buf[kT2Block / 32];
  const int tid = threadIdx.x;
  const int lane = tid & 31, wid = tid >> 5;
  if (tid == 0) {
    const int a = st->action;
    int active = !st->stopped && st->dcgs && (a == ACT_EXTEND || a == ACT_AVNORM);
    // the operator kernel already took the dots of this column (fused_dcgs_dots_jmax); with
    // pipelined DCGS2 they come from the last merged pass unless this cycle applied the
    // operator to the candidate directly (pl_direct)
    if (MODE == TS2_DOTS && active && (st->j <= fused_jmax || !st->pl_direct)) active = 0;
    // the merged pass (k_ts3) updates instead when this cycle looks ahead
    if (MODE == TS2_UPD && active && st->pl_look) active = 0;
    const int j = active ? st->j : 0;
    const int nst = j + 2;
    int T = kT2MaxT;
    while (T > min_T && max_stages * nst * T * 8 > budget) T >>= 1;
    int S = budget / (nst * T * 8);
    while (S < 2 && T > 64) {
      T >>= 1;
      S = budget / (nst * T * 8);
    }
    S = S > max_stages ? max_stages : (S > 8 ? 8 : S);
    s_active = active;
    s_j = j;
    s_T = T;
    s_S = S;
    s_ld = st->ld;
    s_ndot = st->tail_here ? st->ld : st->n;
    s_gam = st->dc_gam;
    s_wsc = st->dc_wsc;
    if (active)
      for (int q = 0; q < S; ++q) {
        mbar_init(&full[q], 1);
        mbar_init(&empty[q], kT2Consumers / 32);
      }
    fence_mbar_init();
  }
  __syncthreads();
  if (!s_active) return;
  const int j = s_j, T = s_T, S = s_S, nst = j + 2;
  const long long ld = s_ld, ndot = s_ndot;
  if (MODE == TS2_UPD)
    for (int i = tid; i < j; i += blockDim.x) {
      s_al[i] = st->dc_alpha[i];
      s_mu[i] = st->dc_mu[i];
    }
  __syncthreads();
  const long long ntiles = ld / T;
  const uint32_t tile_bytes = (uint32_t)T * 8u;
  double acc1[kT2Acc], acc2[kT2Acc];
#pragma unroll
  for (int v = 0; v < kT2Acc; ++v) acc1[v] = acc2[v] = 0.0;
  double nu = 0.0, nw = 0.0;
  if (wid == kT2Consumers / 32) {
    if (lane == 0) {  // producer: slots 0..j+1 are consecutive
      int s = 0, use = 0;
      for (long long tl = blockIdx.x; tl < ntiles; tl += gridDim.x) {
        mbar_wait(&empty[s], (use & 1) ^ 1);
        double* dst = smem + (size_t)s * nst * T;
        mbar_arrive_expect_tx(&full[s], tile_bytes * (uint32_t)nst);
        for (int q = 0; q < nst; ++q) bulk_g2s(dst + (size_t)q * T, base + (size_t)q * ld + tl * T, tile_bytes, &full[s]);
        if (++s == S) {
          s = 0;
          ++use;
        }
      }
    }
  } else {
    const int nvw = (j + 1 + 7) / 8;
    const double g = s_gam, wsc = s_wsc;
#define T2C(NVV) \
  ts2_consume<MODE, NVV>(base, smem, full, empty, s_al, s_mu, g, wsc, j, T, S, ntiles, ld, ndot, nst, acc1, acc2, nu, nw)
    if (MODE == TS2_UPD || nvw <= 1) T2C(1);
    else if (nvw <= 2) T2C(2);
    else if (nvw <= 3) T2C(3);
    else if (nvw <= 5) T2C(5);
    else if (nvw <= 8) T2C(8);
    else T2C(kT2Acc);
#undef T2C
  }
  __syncthreads();
  if (MODE == TS2_DOTS) {
    const int cnt = j + 1;
#pragma unroll
    for (int v = 0; v < kT2Acc; ++v) {
      const int i = wid + 8 * v;
      const double r1 = warp_sum(acc1[v]);
      const double r2 = warp_sum(acc2[v]);
      if (wid < kT2Consumers / 32 && i < cnt && lane == 0) {
        s_red[i] = r1;
        s_red[cnt + i] = r2;
      }
    }
    __syncthreads();
    grid_reduce_last(s_red, 2 * cnt, partials, 2 * kMaxSlots + 2, &st->ticket[8], [&](int i, double v) {
      if (i < cnt) st->rs().dotA[i] = v;
      else st->rs().dotB[i - cnt] = v;
    });
  } else {
    const double tu = block_sum(nu, s_buf);
    const double tw = block_sum(nw, s_buf);
    if (tid == 0) {
      s_red[0] = tu;
      s_red[1] = tw;
    }
    __syncthreads();
    grid_reduce_last(s_red, 2, partials, 2 * kMaxSlots + 2, &st->ticket[9], [&](int i, double v) {
      if (i == 0) st->rs().nrmU = v;
      else st->rs().nrmW = v;
    });
    if (blockIdx.x == 0 && tid == 0) {  // per-launch algorithmic bytes (the dominant kernel's roofline)
      st->upd_bytes += 8.0 * (double)st->n * (double)(j + 4);
      st->upd_launches++;
    }
  }
}

// Coefficients of the update pass from the reduced dots (one CTA).  True
// quantities: a_i = <V_i,u>, b_i = <V_i,w>, c = <u,u>, d = <u,w> with V_i = s_i
// slot_i, u = sigma slot_j; beta_p^2 = c - |a|^2; gamma = (d - a.b) / beta_p^2.
__global__ void __launch_bounds__(128) k_dcgs_coef(PhiState* st) {
  __shared__ double s_buf[4];
  __shared__ int s_go;
  if (threadIdx.x == 0) {
    const int a = st->action;
    s_go = !st->stopped && st->dcgs && (a == ACT_EXTEND || a == ACT_AVNORM);
  }
  __syncthreads();
  if (!s_go) return;
  const int j = st->j;
  const double sig = st->scale[j];
  // W_true = wsc * slot_{j+1}: the stage-1 application wrote dt A (s_j slot_j) itself; a merged
  // pass wrote dt A (slot_j), whose scale s_j is the candidate's (set by the controller)
  const double wsc = st->pl_direct ? 1.0 : sig;
  double sa2 = 0.0, sab = 0.0;
  for (int i = threadIdx.x; i < j; i += blockDim.x) {
    const double si = st->scale[i];
    const double ai = si * sig * st->red.dotA[i];
    const double bi = si * wsc * st->red.dotB[i];
    st->dc_a[i] = ai;
    st->dc_b[i] = bi;
    st->dc_alpha[i] = si * si * st->red.dotA[i];
    sa2 = fma(ai, ai, sa2);
    sab = fma(ai, bi, sab);
  }
  sa2 = block_sum(sa2, s_buf);
  __syncthreads();
  sab = block_sum(sab, s_buf);
  __shared__ double s_gamma;
  if (threadIdx.x == 0) {
    const double c = sig * sig * st->red.dotA[j];
    const double d = sig * wsc * st->red.dotB[j];
    st->dc_wsc = wsc;
    const double beta2 = j == 0 ? 1.0 : c - sa2;
    const double gamma = beta2 > 0.0 ? (d - sab) / beta2 : 0.0;
    st->dc_c = c;
    st->dc_d = d;
    st->dc_ab = sab;
    st->dc_gam = gamma * sig;
    st->dc_gp = gamma;
    s_gamma = gamma;
  }
  __syncthreads();
  const double gamma = s_gamma;
  for (int l = threadIdx.x; l < j; l += blockDim.x) {
    const double al = st->dc_a[l];
    st->dc_mu[l] = (st->dc_b[l] - gamma * al) * st->scale[l];
    // (H a)_l over the finished columns 0..j-2 plus column j-1 corrected by a_l
    double g = 0.0;
    for (int i = 0; i < j; ++i) g = fma(st->H[l * kMaxBasis + i], st->dc_a[i], g);
    st->dc_g[l] = fma(al, st->dc_a[j - 1], g);
  }
  if (!st->pl_look) return;
  // Pipelined DCGS2: the merged pass also forms znew = dt A wnew (the next candidate's image)
  // from the lookahead Y = dt A (s_j slot_{j+1}) by the Arnoldi relation
  //   dt A wnew = wsc dt A slot_{j+1} - dc_gam dt A slot_j - sum_i mu_i dt A slot_i,
  //   dt A slot_j = W_true / s_j,  dt A V_i = sum_{l <= i+1} H(l, i) V_l  (V_l = s_l slot_l),
  // column j-1 with its reorthogonalisation correction a and H(j, j-1) V_j = s_j unew:
  //   znew = (wsc / s_j) Y - gamma wsc W - sum_{l<j} kappa_l slot_l - kappa_j unew,
  //   kappa_l = s_l sum_{i >= l-1} t_i Hf(l, i),  kappa_j = t_{j-1} s_j,  t_i = b_i - gamma a_i.
  __syncthreads();
  for (int l = threadIdx.x; l < j; l += blockDim.x) {
    double k = 0.0;
    for (int i = l > 0 ? l - 1 : 0; i < j; ++i) {
      const double t = st->dc_mu[i] / st->scale[i];  // b_i - gamma a_i
      const double h = st->H[l * kMaxBasis + i] + (i == j - 1 ? st->dc_a[l] : 0.0);
      k = fma(t, h, k);
    }
    st->pl_kappa[l] = st->scale[l] * k;
  }
  if (threadIdx.x == 0) {
    st->pl_zy = wsc / sig;
    st->pl_zw = s_gamma * wsc;
    st->pl_kj = j >= 1 ? st->dc_mu[j - 1] / st->scale[j - 1] * sig : 0.0;
  }
}

// ------------------------------------------------------------------ merged pass (pipelined DCGS2)
// One streaming pass per Krylov column: the update of column j (k_ts2<TS2_UPD>) plus the
// image of the next candidate by the Arnoldi relation plus the next column's pass-1 dots
// (k_ts2<TS2_DOTS>), every tile staged once:
//   phase 1  unew = u - V alpha (slot j), wnew = wsc W - gam u - V mu (slot j+1),
//            znew = zy Y - zw W - V kappa - kj unew (slot j+2, over the lookahead Y)
//   phase 2  the dots of [V_0..V_{j-1}, unew, wnew] against wnew and znew from the same
//            shared-memory tile (the DCGS2 pass-1 dots of column j+1)
// Streams of a tile: slots 0..j+2 (V, u, W, Y), consecutive in HBM: 8 n (j + 6) bytes.
template <int NV, int NA>
__device__ __forceinline__ void ts3_consume(double* base, double* smem, uint64_t* full, uint64_t* empty,
                                            const double* s_al, const double* s_mu, const double* s_ka,
                                            double gam, double wsc, double zy, double zw, double kj, int j, int T,
                                            int S, long long ntiles, long long ld, long long ndot, int nst,
                                            double (&acc1)[NA], double (&acc2)[NA], double& nu) {
  const int tid = threadIdx.x;
  const int lane = tid & 31, wid = tid >> 5;
  const int T2 = T >> 1;
  double2* ug = reinterpret_cast<double2*>(base + (size_t)j * ld);
  double2* wg = reinterpret_cast<double2*>(base + (size_t)(j + 1) * ld);
  double2* zg = reinterpret_cast<double2*>(base + (size_t)(j + 2) * ld);
  int s = 0, use = 0;
  for (long long tl = blockIdx.x; tl < ntiles; tl += gridDim.x) {
    mbar_wait(&full[s], use & 1);
    double* V = smem + (size_t)s * nst * T;
    double2* U2 = reinterpret_cast<double2*>(V + (size_t)j * T);
    double2* W2 = U2 + T2;
    double2* Y2 = W2 + T2;
    const double2* V2 = reinterpret_cast<const double2*>(V);
    const long long g0 = tl * T;
    const int len = (int)min((long long)T, ld - g0);  // the last tile may be short (T need not divide ld)
    const int L2 = len >> 1;
    for (int p = tid; p < L2; p += kT2Consumers) {
      const double2 u = U2[p], w = W2[p], y = Y2[p];
      double ux = u.x, uy = u.y;
      double wx = fma(-gam, u.x, wsc * w.x), wy = fma(-gam, u.y, wsc * w.y);
      double zx = fma(-zw, w.x, zy * y.x), zz = fma(-zw, w.y, zy * y.y);
      for (int i = 0; i < j; ++i) {
        const double al = s_al[i], mu = s_mu[i], ka = s_ka[i];
        const double2 v = V2[(size_t)i * T2 + p];
        ux = fma(-al, v.x, ux);
        uy = fma(-al, v.y, uy);
        wx = fma(-mu, v.x, wx);
        wy = fma(-mu, v.y, wy);
        zx = fma(-ka, v.x, zx);
        zz = fma(-ka, v.y, zz);
      }
      zx = fma(-kj, ux, zx);
      zz = fma(-kj, uy, zz);
      const double2 un = make_double2(ux, uy), wn = make_double2(wx, wy), zn = make_double2(zx, zz);
      U2[p] = un;
      W2[p] = wn;
      Y2[p] = zn;
      ug[(g0 >> 1) + p] = un;
      wg[(g0 >> 1) + p] = wn;
      zg[(g0 >> 1) + p] = zn;
      if (g0 + 2 * p < ndot) nu = fma(un.x, un.x, nu);
      if (g0 + 2 * p + 1 < ndot) nu = fma(un.y, un.y, nu);
    }
    consumer_sync();  // the tile now holds [V_0..V_{j-1}, unew, wnew, znew]
    ts2_mask_tail(V, j + 1, T, g0, ndot, tid, len);
    ts2_tile_dots<NV>(V, j + 1, T, lane, wid, acc1, acc2, len);
    __syncwarp();
    if (lane == 0) mbar_arrive(&empty[s]);
    if (++s == S) {
      s = 0;
      ++use;
    }
  }
}

// (tried: a second instantiation at two CTAs per SM for columns j + 2 <= 64 -- 96 registers,
// spills, half the staging: 4.59 vs 3.55 ms per launch at C4)
__global__ void __launch_bounds__(kT2Block, 1) k_ts3(PhiState* st, double* base, double* partials, int budget,
                                                     int max_stages, int min_T) {
  extern __shared__ __align__(128) double smem[];
  __shared__ uint64_t full[8], empty[8];
  __shared__ int s_active, s_j, s_T, s_S;
  __shared__ long long s_ld, s_ndot;
  __shared__ double s_sc[6];
  __shared__ __align__(16) double s_al[kMaxSlots + 2];
  __shared__ __align__(16) double s_mu[kMaxSlots + 2];
  __shared__ __align__(16) double s_ka[kMaxSlots + 2];
  __shared__ double s_red[2 * kMaxSlots + 2];
  __shared__ double s_buf[kT2Block / 32];
  const int tid = threadIdx.x;
  const int lane = tid & 31, wid = tid >> 5;
  if (tid == 0) {
    const int active =
        !st->stopped && st->dcgs && st->pl_look && (st->action == ACT_EXTEND || st->action == ACT_AVNORM);
    const int j = active ? st->j : 0;
    const int nst = j + 3;
    const int tile_stages = st->ts3_tstages > 0 ? st->ts3_tstages : max_stages;  // stages the tile choice assumes
    // the largest tile (a multiple of 64 doubles, not only a power of two: halving at
    // j = 25 cost C4's large columns ~13 % of their bandwidth) two stages of which fit
    int T = min(kT2MaxT, budget / (tile_stages * nst * 8) / 64 * 64);
    if (st->ts3_pow2) {  // diagnostics: the power-of-two choice
      T = kT2MaxT;
      while (T > min_T && tile_stages * nst * T * 8 > budget) T >>= 1;
    }
    T = max(T, min(min_T, 64));
    int S = budget / (nst * T * 8);
    while (S < 2 && T > 64) {
      T = max(64, (T >> 1) / 64 * 64);
      S = budget / (nst * T * 8);
    }
    // the stages then fill the budget (up to st->ts3_stages), so small columns keep more
    // bytes in flight
    const int cap = st->ts3_stages > 0 ? st->ts3_stages : max_stages;
    S = S > cap ? cap : (S > 8 ? 8 : S);
    s_active = active;
    s_j = j;
    s_T = T;
    s_S = S;
    s_ld = st->ld;
    s_ndot = st->tail_here ? st->ld : st->n;
    s_sc[0] = st->dc_gam;
    s_sc[1] = st->dc_wsc;
    s_sc[2] = st->pl_zy;
    s_sc[3] = st->pl_zw;
    s_sc[4] = st->pl_kj;
    if (active)
      for (int q = 0; q < S; ++q) {
        mbar_init(&full[q], 1);
        mbar_init(&empty[q], kT2Consumers / 32);
      }
    fence_mbar_init();
  }
  __syncthreads();
  if (!s_active) return;
  const int j = s_j, T = s_T, S = s_S, nst = j + 3;
  const long long ld = s_ld, ndot = s_ndot;
  for (int i = tid; i < j; i += blockDim.x) {
    s_al[i] = st->dc_alpha[i];
    s_mu[i] = st->dc_mu[i];
    s_ka[i] = st->pl_kappa[i];
  }
  __syncthreads();
  const long long ntiles = (ld + T - 1) / T;
  double acc1[kT2Acc], acc2[kT2Acc];
#pragma unroll
  for (int v = 0; v < kT2Acc; ++v) acc1[v] = acc2[v] = 0.0;
  double nu = 0.0;
  if (wid == kT2Consumers / 32) {
    if (lane == 0) {  // producer: slots 0..j+2 are consecutive
      int s = 0, use = 0;
      for (long long tl = blockIdx.x; tl < ntiles; tl += gridDim.x) {
        mbar_wait(&empty[s], (use & 1) ^ 1);
        double* dst = smem + (size_t)s * nst * T;
        const uint32_t tile_bytes = (uint32_t)min((long long)T, ld - tl * T) * 8u;
        mbar_arrive_expect_tx(&full[s], tile_bytes * (uint32_t)nst);
        for (int q = 0; q < nst; ++q) bulk_g2s(dst + (size_t)q * T, base + (size_t)q * ld + tl * T, tile_bytes, &full[s]);
        if (++s == S) {
          s = 0;
          ++use;
        }
      }
    }
  } else {
    const int nvw = (j + 2 + 7) / 8;  // dots over vectors 0..j+1
#define T3C(NVV)                                                                                             \
  ts3_consume<NVV, kT2Acc>(base, smem, full, empty, s_al, s_mu, s_ka, s_sc[0], s_sc[1], \
                                                  s_sc[2], s_sc[3], s_sc[4], j, T, S, ntiles, ld, ndot, nst, acc1, \
                                                  acc2, nu)
    if (nvw <= 1) T3C(1);
    else if (nvw <= 2) T3C(2);
    else if (nvw <= 3) T3C(3);
    else if (nvw <= 5) T3C(5);
    else if (nvw <= 8) T3C(8);
    else T3C(kT2Acc);
#undef T3C
  }
  __syncthreads();
  const int cnt = j + 2;
#pragma unroll
  for (int v = 0; v < kT2Acc; ++v) {
    const int i = wid + 8 * v;
    const double r1 = warp_sum(acc1[v]);
    const double r2 = warp_sum(acc2[v]);
    if (wid < kT2Consumers / 32 && i < cnt && lane == 0) {
      s_red[i] = r1;
      s_red[cnt + i] = r2;
    }
  }
  const double tu = block_sum(nu, s_buf);
  if (tid == 0) s_red[2 * cnt] = tu;
  __syncthreads();
  grid_reduce_last(s_red, 2 * cnt + 1, partials, 2 * kMaxSlots + 2, &st->ticket[10], [&](int i, double v) {
    if (i < cnt) st->rs().dotA[i] = v;
    else if (i < 2 * cnt) st->rs().dotB[i - cnt] = v;
    else st->rs().nrmU = v;
    if (i == cnt - 1) st->rs().nrmW = v;  // <wnew, wnew>
  });
  if (blockIdx.x == 0 && tid == 0) {  // the dominant kernel's per-launch algorithmic bytes
    st->upd_bytes += 8.0 * (double)st->n * (double)(j + 6);
    st->upd_launches++;
  }
}

void launch_dcgs(cudaStream_t s, Engine& e, int which, int fused_jmax) {
  const int g = std::max(1, e.num_sms);
  const TsTuning& t = e.ts_tuning;
  if (which == 0)
    k_ts2<TS2_DOTS><<<g, kT2Block, t.budget, s>>>(e.st, e.base, e.partials, t.budget, t.stages, t.min_T, fused_jmax);
  else if (which == 1) k_dcgs_coef<<<1, 128, 0, s>>>(e.st);
  else if (which == 2) k_ts2<TS2_UPD><<<g, kT2Block, t.budget, s>>>(e.st, e.base, e.partials, t.budget, t.stages, t.min_T, -1);
  else k_ts3<<<g, kT2Block, t.budget, s>>>(e.st, e.base, e.partials, t.budget, t.stages, t.min_T);
}

void dcgs_init_attrs(int maxsm) {
  EXPDG_CUDA(cudaFuncSetAttribute(k_ts2<TS2_DOTS>, cudaFuncAttributeMaxDynamicSharedMemorySize, maxsm));
  EXPDG_CUDA(cudaFuncSetAttribute(k_ts2<TS2_UPD>, cudaFuncAttributeMaxDynamicSharedMemorySize, maxsm));
  EXPDG_CUDA(cudaFuncSetAttribute(k_ts3, cudaFuncAttributeMaxDynamicSharedMemorySize, maxsm));
}

}  // namespace expdg
