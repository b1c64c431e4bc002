// 2D compressible Euler DG operators on sm_100a, Lax-Friedrichs or Roe split:
// the JVP L q = frozen-Jacobian volume + linearised LF faces
// (proj/src/euler.cpp:299-341, rhs_faces :260-297, inverse mass :246-258),
// N q (:343-388) and the full RHS (:403-408).
//
// No frozen arrays: the reference stores 2 x 16 doubles of A(q~) per node and
// 3 x 16 per face node (proj/src/euler.cpp:207-243); here A(q~) is recomputed
// from q~ (32 B/node) in registers, so the JVP streams x, q~, b_1 and y only.
// One thread per LGL node, a CTA tile of floor(256 / NP^2) consecutive elements
// staged in shared memory; face neighbours come from the tile when present,
// else from L2.
#include <algorithm>
#include <cstdlib>
#include <vector>

#include "dots.cuh"
#include "krylov.cuh"

namespace expdg {

namespace {


template <int NP>
struct E2P {
  int nx, ny;
  double gamma;
  double w[NP];
  double WD[NP * NP];  // WD(a, b) = w_a D(a, b)
  const double* ut;    // frozen primitives (u, v, H, a) of q~ per node, state layout
  const double* hx;    // element widths per column (uniform breakpoints, proj/src/mesh.cpp:11-16)
  const double* hy;    // element heights per row
  const double* ihx;   // 1 / hx, 1 / hy
  const double* ihy;
  long long n;
  // slab partition: rows -1 and ny are the neighbours' halo rows (raw values of the
  // applied vector / the frozen primitives), exchanged before the kernel runs
  int part;
  const double* gx_lo;
  const double* gx_hi;
  const double* gt_lo;
  const double* gt_hi;
  int dbg;  // EXPDG_E2_DBG (diagnostics): bit 0 = the DOT sweep's dot warps skip their arithmetic, bit 1 = pairs only
};

struct Prim {
  double rho, u, v, p, a, H;
};

// proj/src/euler.cpp:15-24
__device__ __forceinline__ Prim prim_of(const double q[4], double gamma) {
  Prim pr;
  pr.rho = q[0];
  pr.u = q[1] / q[0];
  pr.v = q[2] / q[0];
  pr.p = (gamma - 1.0) * (q[3] - 0.5 * pr.rho * (pr.u * pr.u + pr.v * pr.v));
  pr.a = sqrt(gamma * pr.p / pr.rho);
  pr.H = (q[3] + pr.p) / pr.rho;
  return pr;
}

// frozen (u, v, H, a) -> the primitives the linearised flux reads (rho, p unused)
__device__ __forceinline__ Prim prim_frozen(const double t[4]) {
  Prim pr;
  pr.rho = 0.0;
  pr.p = 0.0;
  pr.u = t[0];
  pr.v = t[1];
  pr.H = t[2];
  pr.a = t[3];
  return pr;
}

__device__ __forceinline__ bool admissible4(const double q[4], double gamma) {
  if (!(q[0] > 0.0)) return false;
  const double p = (gamma - 1.0) * (q[3] - 0.5 * (q[1] * q[1] + q[2] * q[2]) / q[0]);
  return p > 0.0;
}

// out = A(pr, n) x for n = e_x (dir 0) or e_y (dir 1): jacobian_from_primitives
// (proj/src/euler.cpp:44-73) with n substituted, factored so both directions share the
// x-dependent scalars:  with u.m = u x_1 + v x_2,
//   P = phi x_0 - (g-1) u.m + (g-1) x_3,   Q = (phi - H) x_0 - (g-1) u.m + g x_3,
//   s = x_{1+d} - u_d x_0:   out_0 = x_{1+d},  out_{1+r} = u_r s + u_d x_{1+r} + delta_rd P,
//   out_3 = u_d Q + H x_{1+d}.
__device__ __forceinline__ void jac_pre(const Prim& pr, double gamma, const double x[4], double& P, double& Q) {
  const double gm1 = gamma - 1.0;
  const double phi = 0.5 * gm1 * fma(pr.u, pr.u, pr.v * pr.v);
  const double um = fma(pr.u, x[1], pr.v * x[2]);
  P = fma(gm1, x[3] - um, phi * x[0]);
  Q = fma(gamma, x[3], fma(-gm1, um, (phi - pr.H) * x[0]));
}

template <int D>
__device__ __forceinline__ void jac_dir(const Prim& pr, double P, double Q, const double x[4], double out[4]) {
  const double un = D == 0 ? pr.u : pr.v;
  const double sd = fma(-un, x[0], x[1 + D]);
  out[0] = x[1 + D];
  const double v1 = fma(pr.u, sd, un * x[1]);
  const double v2 = fma(pr.v, sd, un * x[2]);
  out[1] = D == 0 ? v1 + P : v1;
  out[2] = D == 1 ? v2 + P : v2;
  out[3] = fma(un, Q, pr.H * x[1 + D]);
}

__device__ __forceinline__ void jac_apply(const Prim& pr, int dir, double gamma, const double x[4], double out[4]) {
  double P, Q;
  jac_pre(pr, gamma, x, P, Q);
  if (dir == 0) jac_dir<0>(pr, P, Q, x, out);
  else jac_dir<1>(pr, P, Q, x, out);
}

// both directions of one node (the volume fluxes)
__device__ __forceinline__ void jac_apply_xy(const Prim& pr, double gamma, const double x[4], double fx[4],
                                             double fy[4]) {
  double P, Q;
  jac_pre(pr, gamma, x, P, Q);
  jac_dir<0>(pr, P, Q, x, fx);
  jac_dir<1>(pr, P, Q, x, fy);
}

// physical flux F(q) . e_dir (proj/src/euler.cpp:26-40)
__device__ __forceinline__ void flux_dir(const double q[4], const Prim& pr, int dir, double f[4]) {
  if (dir == 0) {
    f[0] = q[1];
    f[1] = q[1] * pr.u + pr.p;
    f[2] = q[2] * pr.u;
    f[3] = q[0] * pr.u * pr.H;
  } else {
    f[0] = q[2];
    f[1] = q[1] * pr.v;
    f[2] = q[2] * pr.v + pr.p;
    f[3] = q[0] * pr.v * pr.H;
  }
}

// |A(avg, e_dir)| dq = R |Lambda| R^-1 dq at a Roe state (abs_jacobian_from,
// proj/src/euler.cpp:75-103), applied to the vector without forming the matrix.
__device__ __forceinline__ void roe_abs_apply(int dir, double gamma, double rho, double u, double v, double H,
                                              double a, const double dq[4], double out[4]) {
  const double gm1 = gamma - 1.0;
  const double n0 = dir == 0 ? 1.0 : 0.0, n1 = dir == 0 ? 0.0 : 1.0;
  const double un = dir == 0 ? u : v;
  const double ut = dir == 0 ? v : -u;
  const double phi = 0.5 * gm1 * (u * u + v * v);
  const double a2 = a * a;
  const double dp = phi * dq[0] - gm1 * u * dq[1] - gm1 * v * dq[2] + gm1 * dq[3];
  const double dun = (-un * dq[0] + n0 * dq[1] + n1 * dq[2]) / rho;
  const double dut = (-ut * dq[0] - n1 * dq[1] + n0 * dq[2]) / rho;
  const double w0 = fabs(un - a) * ((dp - rho * a * dun) / (2.0 * a2));
  const double w1 = fabs(un) * (dq[0] - dp / a2);
  const double w2 = fabs(un) * (rho * dut);
  const double w3 = fabs(un + a) * ((dp + rho * a * dun) / (2.0 * a2));
  out[0] = w0 + w1 + w3;
  out[1] = (u - a * n0) * w0 + u * w1 - n1 * w2 + (u + a * n0) * w3;
  out[2] = (v - a * n1) * w0 + v * w1 + n0 * w2 + (v + a * n1) * w3;
  out[3] = (H - a * un) * w0 + 0.5 * (u * u + v * v) * w1 + ut * w2 + (H + a * un) * w3;
}

// roe_average (proj/src/euler.cpp:114-131) from (u, v, H) and sqrt(rho) of both sides;
// false when the averaged sound speed is not real.
__device__ __forceinline__ bool roe_avg(double sm, double um, double vm, double Hm, double sp, double up, double vp,
                                        double Hp, double gamma, double& rho, double& u, double& v, double& H,
                                        double& a) {
  rho = sm * sp;
  u = (sm * um + sp * up) / (sm + sp);
  v = (sm * vm + sp * vp) / (sm + sp);
  H = (sm * Hm + sp * Hp) / (sm + sp);
  const double a2 = (gamma - 1.0) * (H - 0.5 * (u * u + v * v));
  a = sqrt(a2);
  return a2 > 0.0;
}

// Numerical normal flux on a face with n = +e_dir between owner (qm, utm) and
// neighbour (qp, utp):  mode 0 linearised, 1 full - linearised, 2 full.
// ROE: Roe flux (frozen |A| at the Roe average of q~, proj/src/euler.cpp:232-236,
// roe_flux :138-145); else Lax-Friedrichs (:237-241, :147-158).  The frozen
// slot 3 holds sqrt(rho~) for Roe, a~ for LF.
template <bool ROE>
__device__ __forceinline__ void face_flux(int mode, int dir, double gamma, const double qm[4], const double qp[4],
                                          const double utm[4], const double utp[4], double f[4], bool& bad) {
  double lin[4] = {0, 0, 0, 0};
  if (mode != 2) {
    const Prim tm = prim_frozen(utm), tp = prim_frozen(utp);
    double am[4], ap[4], dq[4], dis[4];
    jac_apply(tm, dir, gamma, qm, am);
    jac_apply(tp, dir, gamma, qp, ap);
#pragma unroll
    for (int c = 0; c < 4; ++c) dq[c] = qm[c] - qp[c];
    if (ROE) {
      double rho, u, v, H, a;
      roe_avg(utm[3], tm.u, tm.v, tm.H, utp[3], tp.u, tp.v, tp.H, gamma, rho, u, v, H, a);
      roe_abs_apply(dir, gamma, rho, u, v, H, a, dq, dis);
    } else {
      const double cm = fabs(dir == 0 ? tm.u : tm.v) + tm.a;
      const double cp = fabs(dir == 0 ? tp.u : tp.v) + tp.a;
      const double lam = fmax(cm, cp);
#pragma unroll
      for (int c = 0; c < 4; ++c) dis[c] = lam * dq[c];
    }
#pragma unroll
    for (int c = 0; c < 4; ++c) lin[c] = 0.5 * (am[c] + ap[c]) + 0.5 * dis[c];
  }
  if (mode == 0) {
#pragma unroll
    for (int c = 0; c < 4; ++c) f[c] = lin[c];
    return;
  }
  if (!admissible4(qm, gamma) || !admissible4(qp, gamma)) bad = true;
  const Prim pm = prim_of(qm, gamma), pp = prim_of(qp, gamma);
  double fm[4], fp[4], dis[4];
  flux_dir(qm, pm, dir, fm);
  flux_dir(qp, pp, dir, fp);
  if (ROE) {
    double dq[4], rho, u, v, H, a;
#pragma unroll
    for (int c = 0; c < 4; ++c) dq[c] = qm[c] - qp[c];
    if (!roe_avg(sqrt(pm.rho), pm.u, pm.v, pm.H, sqrt(pp.rho), pp.u, pp.v, pp.H, gamma, rho, u, v, H, a)) bad = true;
    roe_abs_apply(dir, gamma, rho, u, v, H, a, dq, dis);
#pragma unroll
    for (int c = 0; c < 4; ++c) dis[c] *= 0.5;
  } else {
    const double cm = fabs(dir == 0 ? pm.u : pm.v) + pm.a;
    const double cp = fabs(dir == 0 ? pp.u : pp.v) + pp.a;
    const double sc = 0.5 * fmax(cm, cp);
#pragma unroll
    for (int c = 0; c < 4; ++c) dis[c] = sc * (qm[c] - qp[c]);
  }
#pragma unroll
  for (int c = 0; c < 4; ++c) {
    const double full = 0.5 * (fm[c] + fp[c]) + dis[c];
    f[c] = mode == 1 ? full - lin[c] : full;
  }
}

// frozen data per node: (u, v, H, a) for LF, (u, v, H, sqrt(rho)) for Roe
template <bool ROE>
__device__ __forceinline__ void frozen_of(const double q[4], double gamma, double fv[4]) {
  const Prim pr = prim_of(q, gamma);
  fv[0] = pr.u;
  fv[1] = pr.v;
  fv[2] = pr.H;
  fv[3] = ROE ? sqrt(pr.rho) : pr.a;
}


template <int NP>
struct E2Tile {
  static constexpr int NN = NP * NP;
  static constexpr int TE = 256 / NN;  // elements per CTA tile
  static constexpr int VALS = TE * 4 * NN;
};

// Loads node `node` of element `e` (4 comps) of x (scaled) / ut, from the staged
// tile when e is in it, else from global memory.
template <int NP>
__device__ __forceinline__ void load_node(const double* sx, const double* su, int e0, int te, int e, int node,
                                          const double* x, double xs, const double* ut, double q[4], double t[4],
                                          bool need_ut) {
  constexpr int NN = NP * NP;
  const int le = e - e0;
  if (le >= 0 && le < te) {
#pragma unroll
    for (int c = 0; c < 4; ++c) {
      q[c] = sx[(le * 4 + c) * NN + node];
      t[c] = need_ut ? su[(le * 4 + c) * NN + node] : 0.0;
    }
  } else {
#pragma unroll
    for (int c = 0; c < 4; ++c) {
      const size_t g = ((size_t)e * 4 + c) * NN + node;
      q[c] = x[g] * xs;
      t[c] = need_ut ? ut[g] : 0.0;
    }
  }
}

// Computes the operator for every node of a tile; result per thread in out[4]
// (valid when the thread maps to a node of the tile).
template <int NP, bool ROE>
__device__ __forceinline__ void e2_tile(const E2P<NP>& P, int mode, int e0, int te, const double* x, double xs,
                                        double* sx, double* su, double* sf, double out[4], bool& bad) {
  constexpr int NN = NP * NP;
  constexpr int N = NP - 1;
  const int t = threadIdx.x;
  const int le = t / NN, node = t % NN;
  const int i = node % NP, j = node / NP;
  const bool active = le < te;
  const bool need_ut = mode != 2;
  // stage x, ut of the tile (coalesced: the tile is contiguous)
  const int cnt = te * 4 * NN;
  const size_t gbase = (size_t)e0 * 4 * NN;
  for (int idx = t; idx < cnt; idx += blockDim.x) {
    sx[idx] = x[gbase + idx] * xs;
    if (need_ut) su[idx] = P.ut[gbase + idx];
  }
  __syncthreads();
  double q[4], ut[4];
  const int e = e0 + le;
  int ie = 0, je = 0;
  if (active) {
    je = e / P.nx;
    ie = e - je * P.nx;
#pragma unroll
    for (int c = 0; c < 4; ++c) {
      q[c] = sx[(le * 4 + c) * NN + node];
      ut[c] = need_ut ? su[(le * 4 + c) * NN + node] : 0.0;
    }
    // volume fluxes: fx, fy (linear: A(ut) q; nonlinear: F(q) - A(ut) q; full: F(q))
    double fx[4], fy[4];
    if (mode != 2) {
      const Prim tp = prim_frozen(ut);
      jac_apply_xy(tp, P.gamma, q, fx, fy);
    }
    if (mode != 0) {
      if (!admissible4(q, P.gamma)) bad = true;
      const Prim pq = prim_of(q, P.gamma);
      double Fx[4], Fy[4];
      flux_dir(q, pq, 0, Fx);
      flux_dir(q, pq, 1, Fy);
#pragma unroll
      for (int c = 0; c < 4; ++c) {
        fx[c] = mode == 1 ? Fx[c] - fx[c] : Fx[c];
        fy[c] = mode == 1 ? Fy[c] - fy[c] : Fy[c];
      }
    }
#pragma unroll
    for (int c = 0; c < 4; ++c) {
      sf[((le * 2 + 0) * 4 + c) * NN + node] = fx[c];
      sf[((le * 2 + 1) * 4 + c) * NN + node] = fy[c];
    }
  }
  __syncthreads();
  if (!active) return;
  const double hx = __ldg(P.hx + ie);
  const double hy = __ldg(P.hy + je);
  const double sy = 0.5 * hy * P.w[j];
  const double sxs = 0.5 * hx * P.w[i];
  double r[4];
#pragma unroll
  for (int c = 0; c < 4; ++c) {
    const double* fxr = sf + ((le * 2 + 0) * 4 + c) * NN + j * NP;  // row j
    const double* fyc = sf + ((le * 2 + 1) * 4 + c) * NN + i;       // column i
    double ax = 0.0, ay = 0.0;
#pragma unroll
    for (int k = 0; k < NP; ++k) {
      ax = fma(P.WD[k * NP + i], fxr[k], ax);
      ay = fma(P.WD[k * NP + j], fyc[k * NP], ay);
    }
    r[c] = sy * ax;
    r[c] += sxs * ay;
  }
  // x-faces (owner on the low side, normal +e_x, periodic)
  if (i == N || i == 0) {
    const bool owner = i == N;
    const int ie2 = owner ? (ie + 1 == P.nx ? 0 : ie + 1) : (ie == 0 ? P.nx - 1 : ie - 1);
    const int e2 = je * P.nx + ie2;
    const int node2 = j * NP + (owner ? 0 : N);
    double q2[4], u2[4], f[4];
    load_node<NP>(sx, su, e0, te, e2, node2, x, xs, P.ut, q2, u2, need_ut);
    if (owner) face_flux<ROE>(mode, 0, P.gamma, q, q2, ut, u2, f, bad);
    else face_flux<ROE>(mode, 0, P.gamma, q2, q, u2, ut, f, bad);
    // half edge length of the owner element (uniform breaks along y)
    const double fw = 0.5 * hy * P.w[j];
#pragma unroll
    for (int c = 0; c < 4; ++c) r[c] = owner ? r[c] - fw * f[c] : r[c] + fw * f[c];
  }
  if (j == N || j == 0) {
    const bool owner = j == N;
    const int jn = owner ? je + 1 : je - 1;
    const int node2 = (owner ? 0 : N) * NP + i;
    double q2[4], u2[4], f[4];
    if (P.part && (jn < 0 || jn >= P.ny)) {  // halo row of the neighbouring rank
      const double* gx = jn < 0 ? P.gx_lo : P.gx_hi;
      const double* gt = jn < 0 ? P.gt_lo : P.gt_hi;
#pragma unroll
      for (int c = 0; c < 4; ++c) {
        const size_t g = ((size_t)ie * 4 + c) * NN + node2;
        q2[c] = gx[g] * xs;
        u2[c] = need_ut ? gt[g] : 0.0;
      }
    } else {
      const int je2 = jn < 0 ? P.ny - 1 : (jn >= P.ny ? 0 : jn);
      load_node<NP>(sx, su, e0, te, je2 * P.nx + ie, node2, x, xs, P.ut, q2, u2, need_ut);
    }
    if (owner) face_flux<ROE>(mode, 1, P.gamma, q, q2, ut, u2, f, bad);
    else face_flux<ROE>(mode, 1, P.gamma, q2, q, u2, ut, f, bad);
    const double fw = 0.5 * hx * P.w[i];
#pragma unroll
    for (int c = 0; c < 4; ++c) r[c] = owner ? r[c] - fw * f[c] : r[c] + fw * f[c];
  }
  const double scale = 4.0 / (hx * hy);
  const double im = scale / (P.w[i] * P.w[j]);
#pragma unroll
  for (int c = 0; c < 4; ++c) out[c] = r[c] * im;
}

template <int NP, bool ROE>
__global__ void __launch_bounds__(256) k_e2_apply(E2P<NP> P, int mode, const double* __restrict__ x,
                                                  double* __restrict__ y, PhiState* st, double* frozen) {
  constexpr int NN = NP * NP, TE = E2Tile<NP>::TE;
  __shared__ double sx[E2Tile<NP>::VALS], su[E2Tile<NP>::VALS], sf[2 * E2Tile<NP>::VALS];
  if (st && st->stopped) return;
  const int ne = P.nx * P.ny;
  const int ntiles = (ne + TE - 1) / TE;
  bool bad = false;
  for (int tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
    const int e0 = tile * TE;
    const int te = ne - e0 < TE ? ne - e0 : TE;
    __syncthreads();
    double out[4];
    e2_tile<NP, ROE>(P, mode, e0, te, x, 1.0, sx, su, sf, out, bad);
    const int t = threadIdx.x, le = t / NN, node = t % NN;
    if (le < te) {
      const int e = e0 + le;
#pragma unroll
      for (int c = 0; c < 4; ++c) y[((size_t)e * 4 + c) * NN + node] = out[c];
      if (frozen && mode == 2) {
        // freeze (u, v, H, a) of the state for the JVPs of this step (ref = x)
        double qn[4];
#pragma unroll
        for (int c = 0; c < 4; ++c) qn[c] = x[((size_t)e * 4 + c) * NN + node];
        double fv[4];
        frozen_of<ROE>(qn, P.gamma, fv);
#pragma unroll
        for (int c = 0; c < 4; ++c) frozen[((size_t)e * 4 + c) * NN + node] = fv[c];
      }
    }
  }
  if (bad && st) st->domain_flag = 1;
}

// phi-cycle apply: y = dt (L s_j V_j + aug) into slot j+1, ||y||^2 -> red.nrmA
template <int NP, bool ROE>
__global__ void __launch_bounds__(256) k_e2_phi(E2P<NP> P, PhiState* st, double* base, double* partials, BArgs b) {
  constexpr int NN = NP * NP, TE = E2Tile<NP>::TE;
  __shared__ double sx[E2Tile<NP>::VALS], su[E2Tile<NP>::VALS], sf[2 * E2Tile<NP>::VALS];
  __shared__ int s_go, s_j;
  __shared__ double s_xs, s_dt, s_xt[kMaxP];
  __shared__ long long s_ld;
  __shared__ double s_buf[8];
  __shared__ double s_red[1];
  if (threadIdx.x == 0) {
    s_go = apply_go(st, base);
    if (s_go) {
      s_j = st->j;
      s_xs = st->scale[s_j];
      s_dt = st->dt;
      s_ld = st->ld;
      const double* xslot = base + (size_t)s_j * st->ld;
      for (int i = 0; i < kMaxP; ++i) s_xt[i] = (i < b.p) ? xslot[P.n + i] * s_xs : 0.0;
    }
  }
  __syncthreads();
  if (!s_go) return;
  const double* x = base + (size_t)s_j * s_ld;
  double* y = base + (size_t)(s_j + 1) * s_ld;
  const double xs = s_xs, dt = s_dt;
  const int ne = P.nx * P.ny;
  const int ntiles = (ne + TE - 1) / TE;
  double nacc = 0.0;
  bool bad = false;
  for (int tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
    const int e0 = tile * TE;
    const int te = ne - e0 < TE ? ne - e0 : TE;
    __syncthreads();
    double out[4];
    e2_tile<NP, ROE>(P, 0, e0, te, x, xs, sx, su, sf, out, bad);
    const int t = threadIdx.x, le = t / NN, node = t % NN;
    __syncthreads();
    if (le < te) {
#pragma unroll
      for (int c = 0; c < 4; ++c) sx[(le * 4 + c) * NN + node] = out[c];
    }
    __syncthreads();
    for (int idx = t; idx < te * 4 * NN; idx += blockDim.x) {
      const size_t g = (size_t)e0 * 4 * NN + idx;
      double v = sx[idx];
      v = aug_tail(b, s_xt, g, v);
      v = dt * v;
      y[g] = v;
      nacc = fma(v, v, nacc);
    }
  }
  // the p-scalar tail is replicated on every rank; rank 0 counts it
  if (blockIdx.x == 0 && threadIdx.x < kTailPad) {
    const int i = threadIdx.x;
    const double v = (i + 1 < b.p) ? dt * s_xt[i + 1] : 0.0;
    y[P.n + i] = v;
    if (st->tail_here) nacc = fma(v, v, nacc);
  }
  const double tot = block_sum(nacc, s_buf);
  if (threadIdx.x == 0) s_red[0] = tot;
  __syncthreads();
  grid_reduce_last(s_red, 1, partials, kMaxSlots, &st->ticket[4], [&](int, double v) { st->rs().nrmA = v; });
}

// ---------------------------------------------------------------- 2.5D strip JVP (phi cycle)
// A CTA owns a strip of W element columns and marches up a chunk of element
// rows.  Warp CW streams whole element rows (x = slot j and the frozen
// primitives, each with its E/W halo element) by 1D TMA bulk copies into a
// 4-row smem ring (full/empty mbarriers); warps 0..CW-1 compute row r from the
// ring rows r-1, r, r+1, so every byte of x and q~ comes from HBM once per JVP.
//
// DOT = true also takes the DCGS2 pass-1 dots of the cycle (dcgs.cu,
// k_ts2<TS2_DOTS>: a_i = <V_i,u>, b_i = <V_i,w>, <u,u>, <u,w> with u = slot j,
// w = the JVP result) in the same sweep: warp CW+1 streams the row tiles of
// V_0..V_{j-1} into a VS-stage ring and two dot warps (one per tile half) consume
// them against u (the centre of the x ring row) and w (the row just computed,
// handed over through a double-buffered smem row).  u and w are never re-read
// from HBM, and the JVP arithmetic runs under the V stream instead of before it.
// The V ring takes what shared memory the JVP leaves (single-buffered volume
// fluxes in this variant, one more CTA barrier per row).
// the sweep takes the dots of columns j < 44 (C4's basis bound is 40: the separate dots
// pass is then not launched); with b_1 read in place and up to 16 V stages the sweep beats
// the separate passes at every j <= 40 (tools/fusedbench.py: 5.84 vs 6.09 ms at j = 40)
constexpr int kE2DotJ = 44;

template <int NP, int CW, bool DOT>
struct E2Strip {
  static constexpr int NN = NP * NP;
  static constexpr int CONS = 32 * CW;        // consumer threads (CW warps) + one producer warp
  static constexpr int W = CONS / NN > 0 ? CONS / NN : 1;  // elements per strip
  static constexpr int BLK = 4 * NN;          // doubles per element
  static constexpr int ROWD = (W + 2) * BLK;  // doubles per array per row (with halo)
  static constexpr int BUFD = 2 * ROWD;  // x + frozen primitives, with halo (b_1 is read in place)
  static constexpr int NBUF = 4;
  static constexpr int FX = (W + 1) * NP * 4;   // x-face fluxes of a row
  static constexpr int FY = W * NP * 4;         // y-face fluxes of one face row
  static constexpr int TILE = W * BLK;          // doubles of one row of one vector
  static constexpr int ND = DOT ? 2 : 0;        // dot warps, one per tile half (12 warps: <= 168 registers)
  static constexpr int JMAX = DOT ? kE2DotJ - 1 : -1;
  static constexpr int SFB = DOT ? 1 : 2;       // volume-flux buffers (DOT: single, one more barrier per row)
  static constexpr int THREADS = CONS + 32 + (DOT ? 32 + 32 * ND : 0);
  // ring + volume fluxes (double-buffered without DOT) and double-buffered x-face fluxes +
  // a 3-deep ring of y-face rows, so consecutive rows need one CTA barrier between them
  static constexpr int BASE = NBUF * BUFD + SFB * (2 * W * BLK) + 2 * FX + 3 * FY;
  // DOT: two w rows + a V ring of as many row tiles (<= 12) as the 227 KB opt-in
  // shared memory leaves next to ~3 KB of static shared memory
  static constexpr int SMAX = 232448 / 8 - 384;
  static constexpr int VSF = (SMAX - BASE - 2 * TILE) / TILE;
  static constexpr int VS = DOT ? (VSF > 16 ? 16 : (VSF < 1 ? 1 : VSF)) : 1;
  static constexpr bool FITS = !DOT || VSF >= 4;
  static constexpr int SMEM = (BASE + (DOT ? 2 * TILE + VS * TILE : 0)) * 8;
};


// The (strip, row) row-steps of a CTA: one contiguous range [k0, k1) of the
// strip-major row-step order, walked as units of consecutive rows of one strip.
struct StripUnit {
  int ie0, w, r0, r1;
};
template <int W>
__device__ __forceinline__ StripUnit strip_unit(long long& k, long long k1, int nx, int ny) {
  StripUnit u;
  const int strip = (int)(k / ny);
  u.r0 = (int)(k - (long long)strip * ny);
  u.r1 = (int)min((long long)ny, u.r0 + (k1 - k));
  k += u.r1 - u.r0;
  u.ie0 = strip * W;
  u.w = min(W, nx - u.ie0);
  return u;
}

template <class S>
__device__ __forceinline__ void strip_dots(const double* ring, const double* swr, const double* vring,
                                           uint64_t* full, uint64_t* empty, uint64_t* wfull, uint64_t* wempty,
                                           uint64_t* vfull, uint64_t* vempty, long long k0, long long k1, int nx,
                                           int ny, int j, double* s_acc, int skip) {
  const int lane = threadIdx.x & 31;
  const int h = (threadIdx.x >> 5) - (S::CONS / 32 + 2);
  double* acc = s_acc + h * 2 * (S::JMAX + 1);
  RingPos vp, wp;  // V ring; the w-row double buffer
  long long seq = 0;
  for (long long k = k0; k < k1;) {
    const StripUnit su = strip_unit<S::W>(k, k1, nx, ny);
    const int cnt2 = su.w * S::BLK / 2;  // double2 per row tile
    for (int r = su.r0; r < su.r1; ++r) {
      const long long q = r - su.r0 + 1;  // ring index of row r
      const int bsel = wp.s;
      mbar_wait(&wfull[bsel], wp.ph);
      wp.next<2>();
      const int sl = (int)((seq + q) % S::NBUF);
      mbar_wait(&full[sl], (int)(((seq + q) / S::NBUF) & 1));  // completed phase: returns at once
      const double2* U2 = reinterpret_cast<const double2*>(ring + (size_t)sl * S::BUFD + S::BLK);
      const double2* W2 = reinterpret_cast<const double2*>(swr + bsel * S::TILE);
      if (su.w == S::W) dots_row<S, true>(U2, W2, vring, vfull, vempty, vp, j, cnt2, lane, h, acc, skip);
      else dots_row<S, false>(U2, W2, vring, vfull, vempty, vp, j, cnt2, lane, h, acc, skip);
      __syncwarp();
      if (lane == 0) {  // u (the x ring row) and the w row are free
        mbar_arrive(&wempty[bsel]);
        mbar_arrive(&empty[sl]);
      }
    }
    seq += su.r1 - su.r0 + 2;
  }
}

template <int NP, bool ROE, int CW, bool DOT>
__global__ void __launch_bounds__(E2Strip<NP, CW, DOT>::THREADS, CW <= 4 ? 3 : 1)
    k_e2_phi_strip(E2P<NP> P, PhiState* st, double* base, double* partials, BArgs b) {
  using S = E2Strip<NP, CW, DOT>;
  constexpr int NN = S::NN, W = S::W, BLK = S::BLK, NBUF = S::NBUF, N = NP - 1;
  constexpr int NWARP = S::THREADS / 32;
  extern __shared__ __align__(128) double smem[];
  double* ring = smem;
  double* sf0 = smem + NBUF * S::BUFD;
  double* sfx0 = sf0 + S::SFB * (2 * W * BLK);
  double* sfy = sfx0 + 2 * S::FX;
  double* swr = smem + S::BASE;       // DOT: w rows handed to the dot warps
  double* vring = swr + 2 * S::TILE;  // DOT: V row tiles
  __shared__ uint64_t full[NBUF], empty[NBUF];
  __shared__ uint64_t wfull[2], wempty[2], vfull[S::VS], vempty[S::VS];
  __shared__ double s_wd[NP * NP], s_wq[NP];
  __shared__ int s_go, s_j, s_dots;
  __shared__ double s_xs, s_dt, s_xt[kMaxP];
  __shared__ long long s_ld;
  __shared__ double s_buf[NWARP];
  // DOT: per tile half, the dot sums 2 i + {0: <V_i,u>, 1: <V_i,w>}; then (reused in place)
  // the grid-reduction inputs [dotA_0..j, dotB_0..j, ||y||^2]
  __shared__ double s_red[DOT ? 4 * (S::JMAX + 1) : 1];
  const int tid = threadIdx.x, wid = tid >> 5, lane = tid & 31;
  if (tid == 0) {
    s_go = apply_go(st, base);
    if (s_go) {
      s_j = st->j;
      s_dots = DOT && st->dcgs && s_j <= S::JMAX && apply_stage(st, base) == 1;
      if (blockIdx.x == 0) {
        if (apply_stage(st, base) == 1) st->dots_fused = s_dots;  // stage 2 never takes the dots
        // algorithmic bytes of this sweep (bench.py's dominant-kernel roofline): x, q~, b_1, y
        // plus, with the dots, V_0..V_{j-1}
        st->app_bytes += 8.0 * (double)P.n * (4.0 + (s_dots ? (double)s_j : 0.0));
        st->app_launches++;
      }
      s_xs = st->scale[s_j];
      s_dt = st->dt;
      s_ld = st->ld;
      const double* xslot = base + (size_t)s_j * st->ld;
      for (int i = 0; i < kMaxP; ++i) s_xt[i] = (i < b.p) ? xslot[P.n + i] * s_xs : 0.0;
      for (int q = 0; q < NBUF; ++q) {
        mbar_init(&full[q], 1);
        mbar_init(&empty[q], 1 + S::ND);  // the JVP warps + (DOT) every dot warp
      }
      if (DOT) {
        for (int q = 0; q < 2; ++q) {
          mbar_init(&wfull[q], CW);
          mbar_init(&wempty[q], S::ND);
        }
        for (int q = 0; q < S::VS; ++q) {
          mbar_init(&vfull[q], 1);
          mbar_init(&vempty[q], S::ND);  // both tile-half dot warps
        }
      }
      fence_mbar_init();
    }
  }
  for (int q = tid; q < NP * NP; q += blockDim.x) s_wd[q] = P.WD[q];
  for (int q = tid; q < NP; q += blockDim.x) s_wq[q] = P.w[q];
  if (DOT)
    for (int q = tid; q < 4 * (S::JMAX + 1); q += blockDim.x) s_red[q] = 0.0;
  __syncthreads();
  if (!s_go) return;
  const double* x = base + (size_t)s_j * s_ld;
  double* y = base + (size_t)(s_j + 1) * s_ld;
  const double xs = s_xs, dt = s_dt;
  const int nx = P.nx, ny = P.ny;
  const bool dots = DOT && s_dots;
  // ring rows the dot warps also read (u) are released by them too; halo rows and,
  // without dots, every row are released by the JVP warps for all 1 + ND arrivals
  const uint32_t rel_row = dots ? 1u : 1u + S::ND, rel_halo = 1u + S::ND;
  const int nstrips = (nx + W - 1) / W;
  // each CTA owns one contiguous range of the (strip, row) row-steps: equal work per CTA,
  // one or two segments (a new segment restarts the ring with its lower halo row)
  const long long rsteps = (long long)nstrips * ny;
  const long long k0 = rsteps * blockIdx.x / gridDim.x, k1 = rsteps * (blockIdx.x + 1) / gridDim.x;
  // p == 1 (EPI2, exp_euler): the single aug vector b_1 rides in the TMA ring too
  const double* b1 = (b.p == 1) ? b.b[1] : nullptr;
  double nacc = 0.0;

  if (wid == CW) {
    // ---------------- producer: x / frozen / b_1 rows
    if (lane == 0) {
      long long seq = 0;
      for (long long k = k0; k < k1;) {
        const StripUnit su = strip_unit<W>(k, k1, nx, ny);
        const int ie0 = su.ie0, w = su.w, r0 = su.r0, r1 = su.r1;
        for (int q = 0; q < r1 - r0 + 2; ++q) {
          int row = r0 - 1 + q;
          const double* srcx = x;
          const double* srct = P.ut;
          if (P.part && (row < 0 || row >= ny)) {  // halo row of the neighbouring rank
            srcx = row < 0 ? P.gx_lo : P.gx_hi;
            srct = row < 0 ? P.gt_lo : P.gt_hi;
            row = 0;
          } else {
            row = row < 0 ? row + ny : (row >= ny ? row - ny : row);
          }
          const int sl = (int)(seq % NBUF);
          const int use = (int)(seq / NBUF);
          mbar_wait(&empty[sl], (use & 1) ^ 1);
          double* dst = ring + (size_t)sl * S::BUFD;
          const uint32_t eb = BLK * 8;
          mbar_arrive_expect_tx(&full[sl], 2u * (uint32_t)(w + 2) * eb);
          const size_t rbase = (size_t)row * nx;
          const int left = ie0 == 0 ? nx - 1 : ie0 - 1;
          const int right = ie0 + w == nx ? 0 : ie0 + w;
          for (int arr = 0; arr < 2; ++arr) {
            const double* src = arr == 0 ? srcx : srct;
            double* d = dst + arr * S::ROWD;
            if (ie0 >= 1 && ie0 + w < nx) {
              bulk_g2s(d, src + (rbase + left) * BLK, (uint32_t)(w + 2) * eb, &full[sl]);
            } else {
              bulk_g2s(d, src + (rbase + left) * BLK, eb, &full[sl]);
              bulk_g2s(d + BLK, src + (rbase + ie0) * BLK, (uint32_t)w * eb, &full[sl]);
              bulk_g2s(d + (size_t)(w + 1) * BLK, src + (rbase + right) * BLK, eb, &full[sl]);
            }
          }
          ++seq;
        }
      }
    }
  } else if (DOT && wid == CW + 1) {
    // ---------------- producer: row tiles of V_0..V_{j-1} for the dot warps
    if (dots && lane == 0) {
      const int j = s_j;
      const long long ld = s_ld;
      RingPos vp;
      for (long long k = k0; k < k1;) {
        const StripUnit su = strip_unit<W>(k, k1, nx, ny);
        const uint32_t bytes = (uint32_t)(su.w * BLK * 8);
        for (int r = su.r0; r < su.r1; ++r) {
          const double* src = base + ((size_t)r * nx + su.ie0) * BLK;
          for (int i = 0; i < j; ++i) {
            const int stg = vp.s;
            mbar_wait(&vempty[stg], vp.ph ^ 1u);
            mbar_arrive_expect_tx(&vfull[stg], bytes);
            bulk_g2s(vring + (size_t)stg * S::TILE, src + (size_t)i * ld, bytes, &vfull[stg]);
            vp.next<S::VS>();
          }
        }
      }
    }
  } else if (DOT && wid > CW + 1) {
    // ---------------- dot warps
    if (dots) {
      strip_dots<S>(ring, swr, vring, full, empty, wfull, wempty, vfull, vempty, k0, k1, nx, ny, s_j, s_red,
                    P.dbg);
    }
  } else {
    // ---------------- consumers: one thread per node of the strip row
    const int le = tid / NN, node = tid % NN;
    const int i = node % NP, j = node / NP;
    // per-thread basis constants in registers (a runtime index into the kernel
    // parameter arrays would spill them to local memory)
    double wdi[NP], wdj[NP];
#pragma unroll
    for (int q = 0; q < NP; ++q) {
      wdi[q] = s_wd[q * NP + i];
      wdj[q] = s_wd[q * NP + j];
    }
    const double wi = s_wq[i], wj = s_wq[j];
    const double iwij = 1.0 / (wi * wj);
    long long seq = 0;
    int rowc = 0;
    for (long long k = k0; k < k1;) {
      const StripUnit su = strip_unit<W>(k, k1, nx, ny);
      const int ie0 = su.ie0, w = su.w, r0 = su.r0, r1 = su.r1;
      const bool active = le < w;
      const int ie = ie0 + le;
      const double hx = active ? __ldg(P.hx + ie) : 1.0;
      const double ihx = active ? __ldg(P.ihx + ie) : 1.0;
      const double sxs = 0.5 * hx * wi;
      auto slot = [&](long long q) { return ring + (size_t)((seq + q) % NBUF) * S::BUFD; };
      auto wait_row = [&](long long q) { mbar_wait(&full[(seq + q) % NBUF], (int)(((seq + q) / NBUF) & 1)); };
      wait_row(0);
      wait_row(1);
      for (int r = r0; r < r1; ++r) {
        const long long q = r - r0 + 1;  // ring index of row r
        // b_1 of this node (p == 1), read in place: issued now, used in phase C
        double bv[4] = {0.0, 0.0, 0.0, 0.0};
        if (b1 && active) {
          const size_t e = (size_t)r * nx + ie;
#pragma unroll
          for (int c = 0; c < 4; ++c) bv[c] = __ldg(b1 + (e * 4 + c) * NN + node);
        }
        wait_row(q + 1);
        const double* cur = slot(q);
        const double* lo = slot(q - 1);
        const double* hi = slot(q + 1);
        double* sf = sf0 + (S::SFB == 2 ? (q & 1) : 0) * (2 * W * BLK);
        if (S::SFB == 1 && r > r0) strip_sync<S::CONS>();  // C of row r-1 has read sf
        double* sfx = sfx0 + (q & 1) * S::FX;
        const double hy = __ldg(P.hy + r);
        const double ihy = __ldg(P.ihy + r);
        double qv[4], tv[4];
        if (active) {
#pragma unroll
          for (int c = 0; c < 4; ++c) {
            qv[c] = cur[(le + 1) * BLK + c * NN + node] * xs;
            tv[c] = cur[S::ROWD + (le + 1) * BLK + c * NN + node];
          }
          const Prim tp = prim_frozen(tv);
          double fx[4], fy[4];
          jac_apply_xy(tp, P.gamma, qv, fx, fy);
#pragma unroll
          for (int c = 0; c < 4; ++c) {
            sf[((le * 2 + 0) * 4 + c) * NN + node] = fx[c];
            sf[((le * 2 + 1) * 4 + c) * NN + node] = fy[c];
          }
        }
        // ---- numerical fluxes, once per face node (the reference's rhs_faces loop,
        // proj/src/euler.cpp:260-297): x-faces of row r, the y-faces above it and, on the
        // first row of a unit, the y-faces below it; the y-face row above is the next
        // row's lower face row (2-deep ring)
        {
          double* ytop = sfy + ((r - r0 + 1) % 3) * S::FY;
          double* ybot = sfy + ((r - r0) % 3) * S::FY;
          const int nxf = (w + 1) * NP, nyf = w * NP;
          // diagnostics (EXPDG_E2_DBG bit 2): skip the face fluxes (wrong results; timing only)
          const int total = (P.dbg & 4) ? 0 : nxf + nyf + (r == r0 ? nyf : 0);
          for (int t = tid; t < total; t += S::CONS) {  // the consumer warps
            double qa[4], ta[4], qb[4], tb[4], f[4];
            const double* ra;
            const double* rb;
            int pa, pb, na, nb, dir;
            double* dst;
            if (t < nxf) {  // between ring elements fi (W side) and fi + 1 (E side)
              const int fi = t / NP, jn = t - fi * NP;
              ra = cur; rb = cur; pa = fi; pb = fi + 1; na = jn * NP + N; nb = jn * NP; dir = 0;
              dst = sfx + (fi * NP + jn) * 4;
            } else if (t < nxf + nyf) {  // top face of element le: (le, j = N) | row above (le, j = 0)
              const int tt = t - nxf, le2 = tt / NP, in = tt - le2 * NP;
              ra = cur; rb = hi; pa = pb = le2 + 1; na = N * NP + in; nb = in; dir = 1;
              dst = ytop + (le2 * NP + in) * 4;
            } else {  // bottom face of element le (first row of the unit)
              const int tt = t - nxf - nyf, le2 = tt / NP, in = tt - le2 * NP;
              ra = lo; rb = cur; pa = pb = le2 + 1; na = N * NP + in; nb = in; dir = 1;
              dst = ybot + (le2 * NP + in) * 4;
            }
#pragma unroll
            for (int c = 0; c < 4; ++c) {
              qa[c] = ra[pa * BLK + c * NN + na] * xs;
              ta[c] = ra[S::ROWD + pa * BLK + c * NN + na];
              qb[c] = rb[pb * BLK + c * NN + nb] * xs;
              tb[c] = rb[S::ROWD + pb * BLK + c * NN + nb];
            }
            bool bad = false;
            face_flux<ROE>(0, dir, P.gamma, qa, qb, ta, tb, f, bad);
#pragma unroll
            for (int c = 0; c < 4; ++c) dst[c] = f[c];
          }
        }
        strip_sync<S::CONS>();  // A/B of row r done; every thread has also finished C of row r-1
        if (tid == 0) mbar_arrive_cnt(&empty[(seq + q - 1) % NBUF], q == 1 ? rel_halo : rel_row);  // row r-1 free
        const int bsel = rowc & 1;
        double* wrow = swr + bsel * S::TILE;
        if (dots) mbar_wait(&wempty[bsel], ((rowc >> 1) & 1) ^ 1);  // the dot warps took row r-2
        if (active) {
          const double sy = 0.5 * hy * wj;
          double rr[4];
#pragma unroll
          for (int c = 0; c < 4; ++c) {
            const double* fxr = sf + ((le * 2 + 0) * 4 + c) * NN + j * NP;
            const double* fyc = sf + ((le * 2 + 1) * 4 + c) * NN + i;
            double ax = 0.0, ay = 0.0;
#pragma unroll
            for (int k = 0; k < NP; ++k) {
              ax = fma(wdi[k], fxr[k], ax);
              ay = fma(wdj[k], fyc[k * NP], ay);
            }
            rr[c] = sy * ax;
            rr[c] += sxs * ay;
          }
          // scatter of the face fluxes: owner side (normal +e) subtracts, neighbour adds
          if (i == N || i == 0) {
            const double* f = sfx + (((i == N ? le + 1 : le) * NP) + j) * 4;
            const double fw = (i == N ? -0.5 : 0.5) * hy * wj;
#pragma unroll
            for (int c = 0; c < 4; ++c) rr[c] = fma(fw, f[c], rr[c]);
          }
          if (j == N || j == 0) {
            const double* f = sfy + (((r - r0 + (j == N ? 1 : 0)) % 3) * S::FY) + (le * NP + i) * 4;
            const double fw = (j == N ? -0.5 : 0.5) * hx * wi;
#pragma unroll
            for (int c = 0; c < 4; ++c) rr[c] = fma(fw, f[c], rr[c]);
          }
          const double im = (4.0 * ihx * ihy) * iwij;  // 4 / (hx hy w_i w_j)
          const size_t e = (size_t)r * nx + ie;
#pragma unroll
          for (int c = 0; c < 4; ++c) {
            const size_t g = (e * 4 + c) * NN + node;
            double v = rr[c] * im;
            if (b1) {
              v = fma(s_xt[0], bv[c], v);
            } else {
              v = aug_tail(b, s_xt, g, v);
            }
            v = dt * v;
            y[g] = v;
            if (dots) wrow[le * BLK + c * NN + node] = v;
            nacc = fma(v, v, nacc);
          }
        }
        if (dots) {
          __syncwarp();
          if (lane == 0) mbar_arrive(&wfull[bsel]);
        }
        ++rowc;
      }
      strip_sync<S::CONS>();  // C of the unit's last row done
      if (tid == 0) {
        mbar_arrive_cnt(&empty[(seq + (r1 - r0)) % NBUF], r1 - r0 == 0 ? rel_halo : rel_row);  // row r1 - 1
        mbar_arrive_cnt(&empty[(seq + (r1 - r0) + 1) % NBUF], rel_halo);                        // row r1 (upper halo)
      }
      seq += r1 - r0 + 2;
    }
  }
  __syncthreads();
  const int cnt = dots ? s_j + 1 : 0;
  if (blockIdx.x == 0 && tid < kTailPad) {  // replicated tail, counted on rank 0
    const double v = (tid + 1 < b.p) ? dt * s_xt[tid + 1] : 0.0;
    y[P.n + tid] = v;
    if (st->tail_here) nacc = fma(v, v, nacc);
  }
  const double tot = block_sum(nacc, s_buf);
  // dots: the two tile halves, plus (rank 0) the tail region [n, n + kTailPad) of every
  // slot, which k_ts2 streams with the head; cnt <= JMAX + 1 <= blockDim.x
  double ca = 0.0, cb = 0.0;
  if (tid < cnt) {
    constexpr int JS = 2 * (S::JMAX + 1);
    ca = s_red[2 * tid] + s_red[JS + 2 * tid];
    cb = s_red[2 * tid + 1] + s_red[JS + 2 * tid + 1];
    if (blockIdx.x == 0 && st->tail_here) {
      const double* ut = base + (size_t)s_j * s_ld + P.n;
      const double* vt = base + (size_t)tid * s_ld + P.n;
      for (int t = 0; t < kTailPad; ++t) {
        const double yt = (t + 1 < b.p) ? dt * s_xt[t + 1] : 0.0;
        ca = fma(vt[t], ut[t], ca);
        cb = fma(vt[t], yt, cb);
      }
    }
  }
  __syncthreads();
  if (tid < cnt) {
    s_red[tid] = ca;
    s_red[cnt + tid] = cb;
  }
  if (tid == 0) s_red[2 * cnt] = tot;
  __syncthreads();
  grid_reduce_last(s_red, 2 * cnt + 1, partials, 2 * kMaxSlots + 2, &st->ticket[4], [&](int i, double v) {
    if (i < cnt) st->rs().dotA[i] = v;
    else if (i < 2 * cnt) st->rs().dotB[i - cnt] = v;
    else st->rs().nrmA = v;
  });
}

// ---------------------------------------------------------------- strip JVP with face warps
// The plain (no dots) strip JVP, role-split like the 3D z-march (ops_euler3d.cu,
// k_e3_phi_march_fw): the node warps compute the volume fluxes of row r into a double-buffered
// flux array, pass one barrier, then differentiate / scatter / store row r; FWARPS face warps
// compute every numerical flux of the row (the reference's rhs_faces loop,
// proj/src/euler.cpp:260-297) one row ahead into double-buffered x-face arrays and a 4-deep ring
// of y-face rows, handed over by full/empty mbarriers.  The face arithmetic leaves the node
// warps' critical path (volume -> barrier -> differentiate).
#ifndef EXPDG_E2_FWARPS
#define EXPDG_E2_FWARPS 1
#endif
#ifndef EXPDG_E2_FW_NBUF
#define EXPDG_E2_FW_NBUF 4
#endif
#ifndef EXPDG_E2_FW_PER_SM
#define EXPDG_E2_FW_PER_SM 3
#endif
template <int NP, int CW>
struct E2StripFW {
  using B = E2Strip<NP, CW, false>;
  static constexpr int NN = B::NN, CONS = B::CONS, W = B::W, BLK = B::BLK, ROWD = B::ROWD, BUFD = B::BUFD;
  static constexpr int NBUF = EXPDG_E2_FW_NBUF, FX = B::FX, FY = B::FY;
  static constexpr int FWARPS = EXPDG_E2_FWARPS, FTH = 32 * FWARPS;
  static constexpr int THREADS = CONS + 32 + FTH;
  static constexpr int SF = 2 * W * BLK;  // volume fluxes of a row, two buffers
  static constexpr int NYL = 4;           // y-face rows in flight
  static constexpr int SMEM = (NBUF * BUFD + 2 * SF + 2 * FX + NYL * FY) * 8;
  static constexpr int PER_SM = CW <= 4 ? EXPDG_E2_FW_PER_SM : 1;
  // rows r (node warps), r + 1, r + 2 (face warps, up to two rows ahead) and one row in flight;
  // measured at C4 (-DEXPDG_E2_FW_NBUF / _PER_SM): 5, 6 or 8 rows at two CTAs per SM 0.904 /
  // 0.904 / 0.895 ms per launch against 0.860 ms for 4 rows at three CTAs per SM -- the kernel
  // follows the resident warps, not the bytes in flight; 3 rows deadlock
  static_assert(NBUF >= 4, "the face warps run up to two rows ahead of the node warps");
};

// MODE 0: the linear operator (the phi cycle's JVP).  Standalone only: MODE 2, the full right-hand
// side R(x) (proj/src/euler.cpp:249-297: nonlinear volume fluxes, full LF / Roe face fluxes, no
// frozen state), which also writes the frozen primitives of x for the step's JVPs (`frozen`) and
// raises fst->domain_flag on an inadmissible state -- the residual of every step
// (expdg_op_full_rhs, launch_residual); MODE 1, the nonlinear remainder N(x) = R(x) - L x of the
// split (expdg_op_apply_nonlinear, the EXPRB stages).
template <int NP, bool ROE, int CW, int MODE, bool SOLO>
__global__ void __launch_bounds__(E2StripFW<NP, CW>::THREADS, E2StripFW<NP, CW>::PER_SM)
    k_e2_phi_strip_fw(E2P<NP> P, PhiState* st, double* base, double* partials, BArgs b, const double* xin,
                      double* yout, PhiState* fst, double* frozen) {
  // SOLO: the standalone operator application y = L x / N(x) / R(x) (expdg_op_apply_linear, ..),
  // x / y the caller's vectors, no augmentation tail, no reductions (st is null).  A compile-time
  // switch: the phi-cycle instantiation runs at 96 registers and a run-time one cost it spills
  // (0.860 -> 0.935 ms per launch at C4).
  static_assert(SOLO || MODE == 0, "the phi cycle applies the linear operator");
  constexpr int NARR = MODE == 2 ? 1 : 2;  // ring arrays in use: x (+ the frozen primitives)
  if (MODE != 0 && fst && fst->stopped) return;
  bool bad = false;
  using S = E2StripFW<NP, CW>;
  constexpr int NN = S::NN, W = S::W, BLK = S::BLK, NBUF = S::NBUF, N = NP - 1;
  extern __shared__ __align__(128) double smem[];
  double* ring = smem;
  double* sf0 = smem + NBUF * S::BUFD;
  double* sfx0 = sf0 + 2 * S::SF;
  double* sfy0 = sfx0 + 2 * S::FX;
  __shared__ uint64_t full[NBUF], empty[NBUF], ffull[2], fempty[2];
  __shared__ double s_wd[NP * NP], s_wq[NP];
  __shared__ int s_go, s_j;
  __shared__ double s_xs, s_dt, s_xt[kMaxP];
  __shared__ long long s_ld;
  __shared__ double s_buf[S::THREADS / 32];
  __shared__ double s_red[1];
  const int tid = threadIdx.x, wid = tid >> 5, lane = tid & 31;
  if (tid == 0) {
    s_go = SOLO ? 1 : apply_go(st, base);
    if (s_go) {
      if constexpr (!SOLO) {
        s_j = st->j;
        if (blockIdx.x == 0) {
          if (apply_stage(st, base) == 1) st->dots_fused = 0;
          st->app_bytes += 8.0 * (double)P.n * 4.0;
          st->app_launches++;
        }
        s_xs = st->scale[s_j];
        s_dt = st->dt;
        s_ld = st->ld;
        const double* xslot = base + (size_t)s_j * st->ld;
        for (int i = 0; i < kMaxP; ++i) s_xt[i] = (i < b.p) ? xslot[P.n + i] * s_xs : 0.0;
      } else {
        s_j = 0;
        s_xs = 1.0;
        s_dt = 1.0;
        s_ld = 0;
        for (int i = 0; i < kMaxP; ++i) s_xt[i] = 0.0;
      }
      for (int q = 0; q < NBUF; ++q) {
        mbar_init(&full[q], 1);
        mbar_init(&empty[q], 1 + S::FWARPS);  // the node warps + every face warp
      }
      for (int q = 0; q < 2; ++q) {
        mbar_init(&ffull[q], S::FWARPS);
        mbar_init(&fempty[q], 1);
      }
      fence_mbar_init();
    }
  }
  for (int q = tid; q < NP * NP; q += blockDim.x) s_wd[q] = P.WD[q];
  for (int q = tid; q < NP; q += blockDim.x) s_wq[q] = P.w[q];
  __syncthreads();
  if (!s_go) return;
  const double* x = SOLO ? xin : base + (size_t)s_j * s_ld;
  double* y = SOLO ? yout : base + (size_t)(s_j + 1) * s_ld;
  const double xs = s_xs, dt = s_dt;
  const int nx = P.nx, ny = P.ny;
  const int nstrips = (nx + W - 1) / W;
  const long long rsteps = (long long)nstrips * ny;
  const long long k0 = rsteps * blockIdx.x / gridDim.x, k1 = rsteps * (blockIdx.x + 1) / gridDim.x;
  const double* b1 = (b.p == 1) ? b.b[1] : nullptr;
  double nacc = 0.0;

  if (wid == CW) {
    // ---------------- producer: x / frozen rows with their E/W halo elements
    if (lane == 0) {
      long long seq = 0;
      for (long long k = k0; k < k1;) {
        const StripUnit su = strip_unit<W>(k, k1, nx, ny);
        const int ie0 = su.ie0, w = su.w, r0 = su.r0, r1 = su.r1;
        for (int q = 0; q < r1 - r0 + 2; ++q) {
          int row = r0 - 1 + q;
          const double* srcx = x;
          const double* srct = P.ut;
          if (P.part && (row < 0 || row >= ny)) {  // halo row of the neighbouring rank
            srcx = row < 0 ? P.gx_lo : P.gx_hi;
            srct = row < 0 ? P.gt_lo : P.gt_hi;
            row = 0;
          } else {
            row = row < 0 ? row + ny : (row >= ny ? row - ny : row);
          }
          const int sl = (int)(seq % NBUF);
          mbar_wait(&empty[sl], (int)(((seq / NBUF) & 1) ^ 1));
          double* dst = ring + (size_t)sl * S::BUFD;
          const uint32_t eb = BLK * 8;
          mbar_arrive_expect_tx(&full[sl], (uint32_t)NARR * (uint32_t)(w + 2) * eb);
          const size_t rbase = (size_t)row * nx;
          const int left = ie0 == 0 ? nx - 1 : ie0 - 1;
          const int right = ie0 + w == nx ? 0 : ie0 + w;
          for (int arr = 0; arr < NARR; ++arr) {
            const double* src = arr == 0 ? srcx : srct;
            double* d = dst + arr * S::ROWD;
            if (ie0 >= 1 && ie0 + w < nx) {
              bulk_g2s(d, src + (rbase + left) * BLK, (uint32_t)(w + 2) * eb, &full[sl]);
            } else {
              bulk_g2s(d, src + (rbase + left) * BLK, eb, &full[sl]);
              bulk_g2s(d + BLK, src + (rbase + ie0) * BLK, (uint32_t)w * eb, &full[sl]);
              bulk_g2s(d + (size_t)(w + 1) * BLK, src + (rbase + right) * BLK, eb, &full[sl]);
            }
          }
          ++seq;
        }
      }
    }
  } else if (wid > CW) {
    // ---------------- face warps: x-faces of row r, the y-faces above it and, on a unit's first
    // row, the y-faces below it
    const int ft = tid - (S::CONS + 32), fw = wid - (CW + 1);
    long long seq = 0;
    unsigned it = 0, lc = 0;
    for (long long k = k0; k < k1;) {
      const StripUnit su = strip_unit<W>(k, k1, nx, ny);
      const int w = su.w, r0 = su.r0, r1 = su.r1;
      auto slot = [&](long long q) { return ring + (size_t)((seq + q) % NBUF) * S::BUFD; };
      auto wait_row = [&](long long q) { mbar_wait(&full[(seq + q) % NBUF], (int)(((seq + q) / NBUF) & 1)); };
      wait_row(0);
      wait_row(1);
      unsigned lb = lc++ % S::NYL;
      const int nxf = (w + 1) * NP, nyf = w * NP;
      for (int r = r0; r < r1; ++r, ++it) {
        const long long q = r - r0 + 1;
        const unsigned lt = lc++ % S::NYL;
        wait_row(q + 1);
        const int set = it & 1;
        mbar_wait(&fempty[set], ((it >> 1) & 1) ^ 1);  // the node warps consumed this set two rows ago
        const double* cur = slot(q);
        const double* lo = slot(q - 1);
        const double* hi = slot(q + 1);
        double* sfx = sfx0 + set * S::FX;
        double* ytop = sfy0 + lt * S::FY;
        double* ybot = sfy0 + lb * S::FY;
        const int total = nxf + nyf + (r == r0 ? nyf : 0);
        for (int t = ft; t < total; t += S::FTH) {
          double qa[4], ta[4], qb[4], tb[4], f[4];
          const double* ra;
          const double* rb;
          int pa, pb, na, nb, dir;
          double* dst;
          if (t < nxf) {  // between ring elements fi (W side) and fi + 1 (E side)
            const int fi = t / NP, jn = t - fi * NP;
            ra = cur; rb = cur; pa = fi; pb = fi + 1; na = jn * NP + N; nb = jn * NP; dir = 0;
            dst = sfx + (fi * NP + jn) * 4;
          } else if (t < nxf + nyf) {  // top face of element le: (le, j = N) | row above (le, j = 0)
            const int tt = t - nxf, le2 = tt / NP, in = tt - le2 * NP;
            ra = cur; rb = hi; pa = pb = le2 + 1; na = N * NP + in; nb = in; dir = 1;
            dst = ytop + (le2 * NP + in) * 4;
          } else {  // bottom face of element le (first row of the unit)
            const int tt = t - nxf - nyf, le2 = tt / NP, in = tt - le2 * NP;
            ra = lo; rb = cur; pa = pb = le2 + 1; na = N * NP + in; nb = in; dir = 1;
            dst = ybot + (le2 * NP + in) * 4;
          }
#pragma unroll
          for (int c = 0; c < 4; ++c) {
            qa[c] = ra[pa * BLK + c * NN + na] * xs;
            ta[c] = MODE == 2 ? 0.0 : ra[S::ROWD + pa * BLK + c * NN + na];
            qb[c] = rb[pb * BLK + c * NN + nb] * xs;
            tb[c] = MODE == 2 ? 0.0 : rb[S::ROWD + pb * BLK + c * NN + nb];
          }
          face_flux<ROE>(MODE, dir, P.gamma, qa, qb, ta, tb, f, bad);
#pragma unroll
          for (int c = 0; c < 4; ++c) dst[c] = f[c];
        }
        __syncwarp();
        if (lane == 0) {
          mbar_arrive(&ffull[set]);
          // row r is no longer needed here; the halo rows are read by the face warps only, so
          // warp 0 also arrives for the node warps
          mbar_arrive(&empty[(seq + q) % NBUF]);
          if (r == r0) mbar_arrive_cnt(&empty[seq % NBUF], fw == 0 ? 2u : 1u);
          if (r == r1 - 1) mbar_arrive_cnt(&empty[(seq + q + 1) % NBUF], fw == 0 ? 2u : 1u);
        }
        lb = lt;
      }
      seq += r1 - r0 + 2;
    }
  } else {
    // ---------------- node warps: one thread per node of the strip row
    const int le = tid / NN, node = tid % NN;
    const int i = node % NP, j = node / NP;
    double wdi[NP], wdj[NP];
#pragma unroll
    for (int q = 0; q < NP; ++q) {
      wdi[q] = s_wd[q * NP + i];
      wdj[q] = s_wd[q * NP + j];
    }
    const double wi = s_wq[i], wj = s_wq[j];
    const double iwij = 1.0 / (wi * wj);
    long long seq = 0;
    unsigned it = 0, lc = 0;
    int prev_slot = -1;
    for (long long k = k0; k < k1;) {
      const StripUnit su = strip_unit<W>(k, k1, nx, ny);
      const int ie0 = su.ie0, w = su.w, r0 = su.r0, r1 = su.r1;
      const bool active = le < w;
      const int ie = ie0 + le;
      const double hx = active ? __ldg(P.hx + ie) : 1.0;
      const double ihx = active ? __ldg(P.ihx + ie) : 1.0;
      const double sxs = 0.5 * hx * wi;
      unsigned lb = lc++ % S::NYL;
      for (int r = r0; r < r1; ++r, ++it) {
        const long long q = r - r0 + 1;  // ring index of row r
        const unsigned lt = lc++ % S::NYL;
        // b_1 of this node (p == 1), read in place: issued now, used after the barrier
        double bv[4] = {0.0, 0.0, 0.0, 0.0};
        if (b1 && active) {
          const size_t e = (size_t)r * nx + ie;
#pragma unroll
          for (int c = 0; c < 4; ++c) bv[c] = __ldg(b1 + (e * 4 + c) * NN + node);
        }
        const double hy = __ldg(P.hy + r);
        const double ihy = __ldg(P.ihy + r);
        const int sl = (int)((seq + q) % NBUF);
        mbar_wait(&full[sl], (int)(((seq + q) / NBUF) & 1));
        const double* cur = ring + (size_t)sl * S::BUFD;
        double* sf = sf0 + (it & 1) * S::SF;
        if (active) {
          double qv[4], fx[4], fy[4];
#pragma unroll
          for (int c = 0; c < 4; ++c) qv[c] = cur[(le + 1) * BLK + c * NN + node] * xs;
          if constexpr (MODE != 2) {
            double tv[4];
#pragma unroll
            for (int c = 0; c < 4; ++c) tv[c] = cur[S::ROWD + (le + 1) * BLK + c * NN + node];
            const Prim tp = prim_frozen(tv);
            jac_apply_xy(tp, P.gamma, qv, fx, fy);
          }
          if constexpr (MODE != 0) {  // F(q) (MODE 2), F(q) - A(q~) q (MODE 1), as the tile kernel (e2_tile)
            if (!admissible4(qv, P.gamma)) bad = true;
            const Prim pq = prim_of(qv, P.gamma);
            double Fx[4], Fy[4];
            flux_dir(qv, pq, 0, Fx);
            flux_dir(qv, pq, 1, Fy);
#pragma unroll
            for (int c = 0; c < 4; ++c) {
              fx[c] = MODE == 1 ? Fx[c] - fx[c] : Fx[c];
              fy[c] = MODE == 1 ? Fy[c] - fy[c] : Fy[c];
            }
            if (MODE == 2 && frozen) {  // (u, v, H, a | sqrt(rho)) of the state for this step's JVPs
              double fv[4];
              frozen_of<ROE>(qv, P.gamma, fv);
              const size_t e = (size_t)r * nx + ie;
#pragma unroll
              for (int c = 0; c < 4; ++c) frozen[(e * 4 + c) * NN + node] = fv[c];
            }
          }
#pragma unroll
          for (int c = 0; c < 4; ++c) {
            sf[((le * 2 + 0) * 4 + c) * NN + node] = fx[c];
            sf[((le * 2 + 1) * 4 + c) * NN + node] = fy[c];
          }
        }
        strip_sync<S::CONS>();  // volume fluxes of row r complete; every thread is past row r - 1
        if (tid == 0 && prev_slot >= 0) {
          mbar_arrive(&empty[prev_slot]);
          mbar_arrive(&fempty[(it - 1) & 1]);
        }
        prev_slot = sl;
        mbar_wait(&ffull[it & 1], (it >> 1) & 1);  // the face fluxes of row r
        if (active) {
          const double* sfx = sfx0 + (it & 1) * S::FX;
          const double sy = 0.5 * hy * wj;
          double rr[4];
#pragma unroll
          for (int c = 0; c < 4; ++c) {
            const double* fxr = sf + ((le * 2 + 0) * 4 + c) * NN + j * NP;
            const double* fyc = sf + ((le * 2 + 1) * 4 + c) * NN + i;
            double ax = 0.0, ay = 0.0;
#pragma unroll
            for (int m = 0; m < NP; ++m) {
              ax = fma(wdi[m], fxr[m], ax);
              ay = fma(wdj[m], fyc[m * NP], ay);
            }
            rr[c] = sy * ax;
            rr[c] += sxs * ay;
          }
          // scatter of the face fluxes: owner side (normal +e) subtracts, neighbour adds
          if (i == N || i == 0) {
            const double* f = sfx + (((i == N ? le + 1 : le) * NP) + j) * 4;
            const double fw = (i == N ? -0.5 : 0.5) * hy * wj;
#pragma unroll
            for (int c = 0; c < 4; ++c) rr[c] = fma(fw, f[c], rr[c]);
          }
          if (j == N || j == 0) {
            const double* f = sfy0 + (j == N ? lt : lb) * S::FY + (le * NP + i) * 4;
            const double fw = (j == N ? -0.5 : 0.5) * hx * wi;
#pragma unroll
            for (int c = 0; c < 4; ++c) rr[c] = fma(fw, f[c], rr[c]);
          }
          const double im = (4.0 * ihx * ihy) * iwij;  // 4 / (hx hy w_i w_j)
          const size_t e = (size_t)r * nx + ie;
#pragma unroll
          for (int c = 0; c < 4; ++c) {
            const size_t g = (e * 4 + c) * NN + node;
            double v = rr[c] * im;
            if (b1) v = fma(s_xt[0], bv[c], v);
            else v = aug_tail(b, s_xt, g, v);
            v = dt * v;
            y[g] = v;
            nacc = fma(v, v, nacc);
          }
        }
        lb = lt;
      }
      seq += r1 - r0 + 2;
    }
    strip_sync<S::CONS>();
    if (tid == 0 && prev_slot >= 0) {
      mbar_arrive(&empty[prev_slot]);
      mbar_arrive(&fempty[(it - 1) & 1]);
    }
  }
  if (MODE != 0 && bad && fst) fst->domain_flag = 1;
  if constexpr (!SOLO) {
    __syncthreads();
    if (blockIdx.x == 0 && tid < kTailPad) {  // replicated tail, counted on rank 0
      const double v = (tid + 1 < b.p) ? dt * s_xt[tid + 1] : 0.0;
      y[P.n + tid] = v;
      if (st->tail_here) nacc = fma(v, v, nacc);
    }
    const double tot = block_sum(nacc, s_buf);
    if (tid == 0) s_red[0] = tot;
    __syncthreads();
    grid_reduce_last(s_red, 1, partials, 2 * kMaxSlots + 2, &st->ticket[4], [&](int, double v) { st->rs().nrmA = v; });
  }
}

// (u, v, H, a | sqrt(rho)) of q~ per node (proj/src/euler.cpp:15-24): the frozen
// data of the linearised operator, 32 B/node like q~ itself.
template <bool ROE>
__global__ void k_e2_freeze(const double* __restrict__ q, long long nelem, int nn, double gamma,
                            double* __restrict__ frozen) {
  const long long nodes = nelem * nn;
  const long long stride = (long long)gridDim.x * blockDim.x;
  for (long long g = (long long)blockIdx.x * blockDim.x + threadIdx.x; g < nodes; g += stride) {
    const long long e = g / nn;
    const int node = (int)(g - e * nn);
    double qn[4];
    for (int c = 0; c < 4; ++c) qn[c] = q[(e * 4 + c) * nn + node];
    double fv[4];
    frozen_of<ROE>(qn, gamma, fv);
    for (int c = 0; c < 4; ++c) frozen[(e * 4 + c) * nn + node] = fv[c];
  }
}


template <int NP>
class Euler2D : public OpDevice {
 public:
  E2P<NP> P{};
  int grid = 1;
  double* frozen = nullptr;
  double* hbuf = nullptr;
  bool use_strip = true;
  bool roe = false;
  int strip_cw = 8;  // consumer warps per strip CTA (EXPDG_E2_CW=4: half-width strips, 2 CTAs / SM)
  // the same for the pipelined lookahead application (EXPDG_E2_CW2): half-width strips at three
  // CTAs per SM (128 registers) run it in 1.01 vs 1.12 ms at C4 (same box)
  int strip_cw2 = 4;
  // the plain half-width strip with face warps (EXPDG_E2_FW=0: the single-role strip)
  bool use_fw = true;
  bool fw_align = false;  // EXPDG_E2_ALIGN=1: whole CTAs per strip (see launch_strip_fw)
  bool rhs_strip = true;  // EXPDG_E2_RHS_TILE=1: the element-tile kernel for R(x) (residual, full_rhs)
  int fw_per_sm = 1, fw2_per_sm = 1;
  void launch_strip_fw(cudaStream_t s, const E2P<NP>& p, PhiState* st, double* base, double* partials,
                       const BArgs& b, const double* xin = nullptr, double* yout = nullptr) {
    using SS = E2StripFW<NP, 4>;
    const long long nstrips = (P.nx + SS::W - 1) / SS::W;
    const long long rows = nstrips * P.ny;
    int g = (int)std::max<long long>(1, std::min<long long>(rows, 148LL * fw_per_sm));
    // EXPDG_E2_ALIGN=1 (diagnostics): whole CTAs per strip, every strip cut at the same rows, so
    // the CTAs of neighbouring strips march the same rows at the same time and the E/W halo
    // elements (2 of every W + 2 staged: 40 % more x / q~ reads at W = 5 when they miss) come
    // from L2.  Measured slower at C4 (410 instead of 444 CTAs: 0.918 vs 0.860 ms per launch):
    // the kernel is latency-bound, not DRAM-bound, and the lost CTAs cost more than the misses.
    const long long q = g / nstrips;
    if (fw_align && q >= 1 && P.ny % q == 0 && nstrips * q * 10 >= (long long)g * 8) g = (int)(nstrips * q);
    if (st) {
      if (roe)
        k_e2_phi_strip_fw<NP, true, 4, 0, false><<<g, SS::THREADS, SS::SMEM, s>>>(p, st, base, partials, b, nullptr,
                                                                                  nullptr, nullptr, nullptr);
      else
        k_e2_phi_strip_fw<NP, false, 4, 0, false><<<g, SS::THREADS, SS::SMEM, s>>>(p, st, base, partials, b, nullptr,
                                                                                   nullptr, nullptr, nullptr);
    } else {
      if (roe)
        k_e2_phi_strip_fw<NP, true, 4, 0, true><<<g, SS::THREADS, SS::SMEM, s>>>(p, nullptr, nullptr, nullptr, b, xin,
                                                                                 yout, nullptr, nullptr);
      else
        k_e2_phi_strip_fw<NP, false, 4, 0, true><<<g, SS::THREADS, SS::SMEM, s>>>(p, nullptr, nullptr, nullptr, b, xin,
                                                                                  yout, nullptr, nullptr);
    }
  }
  // N(x) -> y through the strip kernel (MODE 1)
  void launch_strip_nonlinear(cudaStream_t s, const E2P<NP>& p, const double* x, double* y) {
    using SS = E2StripFW<NP, 4>;
    const long long rows = (long long)((P.nx + SS::W - 1) / SS::W) * P.ny;
    const int g = (int)std::max<long long>(1, std::min<long long>(rows, 148LL * fw2_per_sm));
    if (roe)
      k_e2_phi_strip_fw<NP, true, 4, 1, true><<<g, SS::THREADS, SS::SMEM, s>>>(p, nullptr, nullptr, nullptr, BArgs{}, x, y,
                                                                         nullptr, nullptr);
    else
      k_e2_phi_strip_fw<NP, false, 4, 1, true><<<g, SS::THREADS, SS::SMEM, s>>>(p, nullptr, nullptr, nullptr, BArgs{}, x, y,
                                                                          nullptr, nullptr);
  }
  // R(x) -> y through the strip kernel (MODE 2); frozen_out / fst may be null (expdg_op_full_rhs)
  void launch_strip_rhs(cudaStream_t s, const E2P<NP>& p, const double* x, double* y, PhiState* fst,
                        double* frozen_out) {
    using SS = E2StripFW<NP, 4>;
    const long long rows = (long long)((P.nx + SS::W - 1) / SS::W) * P.ny;
    const int g = (int)std::max<long long>(1, std::min<long long>(rows, 148LL * fw2_per_sm));
    if (roe)
      k_e2_phi_strip_fw<NP, true, 4, 2, true><<<g, SS::THREADS, SS::SMEM, s>>>(p, nullptr, nullptr, nullptr, BArgs{}, x, y,
                                                                         fst, frozen_out);
    else
      k_e2_phi_strip_fw<NP, false, 4, 2, true><<<g, SS::THREADS, SS::SMEM, s>>>(p, nullptr, nullptr, nullptr, BArgs{}, x, y,
                                                                          fst, frozen_out);
  }
  template <int CW, bool DOT>
  void launch_strip(cudaStream_t s, const E2P<NP>& p, PhiState* st, double* base, double* partials,
                    const BArgs& b) {
    using SS = E2Strip<NP, CW, DOT>;
    int per_sm = 1;
    EXPDG_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_e2_phi_strip<NP, false, CW, DOT>,
                                                             SS::THREADS, SS::SMEM));
    const long long rows = (long long)((P.nx + SS::W - 1) / SS::W) * P.ny;
    const int g = (int)std::max<long long>(1, std::min<long long>(rows, 148LL * std::max(1, per_sm)));
    if (roe) k_e2_phi_strip<NP, true, CW, DOT><<<g, SS::THREADS, SS::SMEM, s>>>(p, st, base, partials, b);
    else k_e2_phi_strip<NP, false, CW, DOT><<<g, SS::THREADS, SS::SMEM, s>>>(p, st, base, partials, b);
  }
  // The strip JVP also takes the DCGS2 pass-1 dots of columns j <= JMAX (EXPDG_E2_DOTS=0:
  // off).  Same-box A/B at C4 (bench.py, 5 steps): 257.7 vs 263.3 ms per step.
  static constexpr bool kDotFits = E2Strip<NP, 8, true>::FITS;
  bool use_dots = true;
  bool dots_on() const { return kDotFits && use_dots && use_strip && strip_cw == 8; }
  int fused_dcgs_dots_jmax() const override { return dots_on() ? E2Strip<NP, 8, true>::JMAX : -1; }
  template <int CW, bool DOT>
  static void set_strip_attrs() {
    using SS = E2Strip<NP, CW, DOT>;
    EXPDG_CUDA(cudaFuncSetAttribute(k_e2_phi_strip<NP, false, CW, DOT>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                    SS::SMEM));
    EXPDG_CUDA(cudaFuncSetAttribute(k_e2_phi_strip<NP, true, CW, DOT>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                    SS::SMEM));
  }
  // slab partition: halo rows (x lo/hi, frozen lo/hi) and send staging (lo/hi)
  double* halo = nullptr;
  long long rowd = 0;  // doubles per element row
  ~Euler2D() override {
    cudaFree(frozen);
    cudaFree(hbuf);
    cudaFree(halo);
  }
  double* hx_lo() const { return halo; }
  double* hx_hi() const { return halo + rowd; }
  double* ht_lo() const { return halo + 2 * rowd; }
  double* ht_hi() const { return halo + 3 * rowd; }
  double* sb_lo() const { return halo + 4 * rowd; }
  double* sb_hi() const { return halo + 5 * rowd; }
  // neighbour rows of a state-layout vector v -> (lo, hi) halo buffers
  void exchange(cudaStream_t s, const double* v, double* lo, double* hi) {
    comm->halo(v, v + (size_t)(P.ny - 1) * rowd, lo, hi, rowd, s);
  }
  E2P<NP> params(const double* ut) const {
    E2P<NP> p = P;
    p.ut = ut;
    if (p.part) {
      p.gx_lo = hx_lo();
      p.gx_hi = hx_hi();
      p.gt_lo = ht_lo();
      p.gt_hi = ht_hi();
    }
    return p;
  }
  void freeze(cudaStream_t s, const double* r) override {
    ref = r;
    if (roe) k_e2_freeze<true><<<1184, 256, 0, s>>>(r, (long long)P.nx * P.ny, NP * NP, P.gamma, frozen);
    else k_e2_freeze<false><<<1184, 256, 0, s>>>(r, (long long)P.nx * P.ny, NP * NP, P.gamma, frozen);
    if (P.part) exchange(s, frozen, ht_lo(), ht_hi());
  }
  explicit Euler2D(const expdg_op_desc& d) {
    desc = d;
    const HostBasis hb = host_lgl_basis(d.order);
    const bool part = d.part_end > d.part_begin;
    const int row0 = part ? d.part_begin : 0;
    const int nyl = part ? d.part_end - d.part_begin : d.ny;
    P.nx = d.nx;
    P.ny = nyl;
    P.part = part ? 1 : 0;
    P.gamma = d.gamma;
    std::vector<double> hs(2 * (d.nx + nyl));
    // element widths from the axis breakpoints: uniform or the grading lists (proj/src/mesh.cpp:96-120)
    const std::vector<double> xs = host_axis_breaks(d.x0, d.x1, d.nx, d.grade_x);
    const std::vector<double> ys = host_axis_breaks(d.y0, d.y1, d.ny, d.grade_y);
    for (int i = 0; i < d.nx; ++i) hs[i] = xs[i + 1] - xs[i];
    for (int j = 0; j < nyl; ++j) hs[d.nx + j] = ys[row0 + j + 1] - ys[row0 + j];
    for (int q = 0; q < d.nx + nyl; ++q) hs[d.nx + nyl + q] = 1.0 / hs[q];
    EXPDG_CUDA(cudaMalloc(&hbuf, sizeof(double) * hs.size()));
    EXPDG_CUDA(cudaMemcpy(hbuf, hs.data(), sizeof(double) * hs.size(), cudaMemcpyHostToDevice));
    P.hx = hbuf;
    P.hy = hbuf + d.nx;
    P.ihx = hbuf + d.nx + nyl;
    P.ihy = hbuf + 2 * d.nx + nyl;
    for (int a = 0; a < NP; ++a) {
      P.w[a] = hb.weights[a];
      for (int b2 = 0; b2 < NP; ++b2) P.WD[a * NP + b2] = hb.weights[a] * hb.D[a * NP + b2];
    }
    n = (long long)d.nx * nyl * NP * NP * 4;
    P.n = n;
    comps = 4;
    rowd = (long long)d.nx * NP * NP * 4;
    EXPDG_CUDA(cudaMalloc(&frozen, sizeof(double) * n));
    if (part) {
      EXPDG_CUDA(cudaMalloc(&halo, sizeof(double) * 6 * rowd));
      EXPDG_CUDA(cudaMemset(halo, 0, sizeof(double) * 6 * rowd));
    }
    use_strip = !(std::getenv("EXPDG_E2_TILE") && std::getenv("EXPDG_E2_TILE")[0] == '1');
    roe = d.euler_flux == 0;
    if (const char* v = std::getenv("EXPDG_E2_CW")) strip_cw = std::atoi(v) == 4 ? 4 : 8;
    if (const char* v = std::getenv("EXPDG_E2_CW2")) strip_cw2 = std::atoi(v) == 8 ? 8 : 4;
    if (const char* v = std::getenv("EXPDG_E2_DOTS")) use_dots = v[0] != '0';
    if (const char* v = std::getenv("EXPDG_E2_DBG")) P.dbg = std::atoi(v);
    if (const char* v = std::getenv("EXPDG_E2_FW")) use_fw = v[0] != '0';
    if (const char* v = std::getenv("EXPDG_E2_ALIGN")) fw_align = v[0] == '1';
    if (const char* v = std::getenv("EXPDG_E2_RHS_TILE")) rhs_strip = v[0] != '1';
    set_strip_attrs<8, false>();
    set_strip_attrs<4, false>();
    {  // the face-warp strip: attributes and occupancy here, never on the launch path (a runtime
       // call that synchronises the device must not run while another rank's collective spins)
      using SF = E2StripFW<NP, 4>;
      EXPDG_CUDA(cudaFuncSetAttribute(k_e2_phi_strip_fw<NP, false, 4, 0, false>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                      SF::SMEM));
      EXPDG_CUDA(cudaFuncSetAttribute(k_e2_phi_strip_fw<NP, true, 4, 0, false>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                      SF::SMEM));
      EXPDG_CUDA(cudaFuncSetAttribute(k_e2_phi_strip_fw<NP, false, 4, 2, true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                      SF::SMEM));
      EXPDG_CUDA(cudaFuncSetAttribute(k_e2_phi_strip_fw<NP, true, 4, 2, true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                      SF::SMEM));
      EXPDG_CUDA(cudaFuncSetAttribute(k_e2_phi_strip_fw<NP, false, 4, 1, true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                      SF::SMEM));
      EXPDG_CUDA(cudaFuncSetAttribute(k_e2_phi_strip_fw<NP, true, 4, 1, true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                      SF::SMEM));
      EXPDG_CUDA(cudaFuncSetAttribute(k_e2_phi_strip_fw<NP, false, 4, 0, true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                      SF::SMEM));
      EXPDG_CUDA(cudaFuncSetAttribute(k_e2_phi_strip_fw<NP, true, 4, 0, true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                      SF::SMEM));
      EXPDG_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&fw_per_sm, k_e2_phi_strip_fw<NP, false, 4, 0, false>,
                                                               SF::THREADS, SF::SMEM));
      fw_per_sm = std::max(1, fw_per_sm);
      EXPDG_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&fw2_per_sm, k_e2_phi_strip_fw<NP, false, 4, 2, true>,
                                                               SF::THREADS, SF::SMEM));
      fw2_per_sm = std::max(1, fw2_per_sm);
    }
    if constexpr (kDotFits) set_strip_attrs<8, true>();
    const long long ntiles = ((long long)d.nx * nyl + E2Tile<NP>::TE - 1) / E2Tile<NP>::TE;
    grid = (int)std::max<long long>(1, std::min<long long>(ntiles, 148LL * 8));
  }
  void launch_phi_apply(cudaStream_t s, PhiState* st, double* base, double* partials, const BArgs& b, int stage = 1) override {
    if (P.part) {  // halo rows of the slot this cycle applies the operator to
      launch_pack_slot(s, st, base, rowd, (long long)(P.ny - 1) * rowd, sb_lo(), sb_hi());
      comm->halo(sb_lo(), sb_hi(), hx_lo(), hx_hi(), rowd, s);
    }
    const E2P<NP> p = params(frozen);
    if (use_strip) {
      if (strip_cw == 4 || (stage == 2 && strip_cw2 == 4)) {
        if (use_fw) launch_strip_fw(s, p, st, base, partials, b);
        else launch_strip<4, false>(s, p, st, base, partials, b);
      } else if (dots_on() && stage == 1) {
        if constexpr (kDotFits) launch_strip<8, true>(s, p, st, base, partials, b);
      } else {
        launch_strip<8, false>(s, p, st, base, partials, b);
      }
    } else {
      if (roe) k_e2_phi<NP, true><<<grid, 256, 0, s>>>(p, st, base, partials, b);
      else k_e2_phi<NP, false><<<grid, 256, 0, s>>>(p, st, base, partials, b);
    }
  }
  void launch_apply(cudaStream_t s, int which, const double* x, double* y) override {
    if (P.part) exchange(s, x, hx_lo(), hx_hi());
    const E2P<NP> p = params(frozen);
    if (which == 0 && use_strip && use_fw && x != y) {  // y = L x through the strip JVP (the same kernel as the phi cycle)
      launch_strip_fw(s, p, nullptr, nullptr, nullptr, BArgs{}, x, y);
      return;
    }
    if (which == 2 && use_strip && use_fw && rhs_strip && x != y) {  // y = R(x)
      launch_strip_rhs(s, p, x, y, nullptr, nullptr);
      return;
    }
    if (which == 1 && use_strip && use_fw && rhs_strip && x != y) {  // y = N(x) = R(x) - L x
      launch_strip_nonlinear(s, p, x, y);
      return;
    }
    if (roe) k_e2_apply<NP, true><<<grid, 256, 0, s>>>(p, which, x, y, nullptr, nullptr);
    else k_e2_apply<NP, false><<<grid, 256, 0, s>>>(p, which, x, y, nullptr, nullptr);
  }
  // R = full rhs(u) and, as a side product, the frozen primitives of u (ref = u)
  void launch_residual(cudaStream_t s, const double* u, double* r, PhiState* st, double*) override {
    if (P.part) exchange(s, u, hx_lo(), hx_hi());
    const E2P<NP> p = params(nullptr);
    if (use_strip && use_fw && rhs_strip && u != r) launch_strip_rhs(s, p, u, r, st, frozen);
    else if (roe) k_e2_apply<NP, true><<<grid, 256, 0, s>>>(p, 2, u, r, st, frozen);
    else k_e2_apply<NP, false><<<grid, 256, 0, s>>>(p, 2, u, r, st, frozen);
    if (P.part) exchange(s, frozen, ht_lo(), ht_hi());  // frozen halo for this step's JVPs
  }
};

}  // namespace

std::unique_ptr<OpDevice> make_euler2d(const expdg_op_desc& d) {
  switch (d.order + 1) {
    case 2: return std::make_unique<Euler2D<2>>(d);
    case 3: return std::make_unique<Euler2D<3>>(d);
    case 4: return std::make_unique<Euler2D<4>>(d);
    case 5: return std::make_unique<Euler2D<5>>(d);
    case 6: return std::make_unique<Euler2D<6>>(d);
    case 7: return std::make_unique<Euler2D<7>>(d);
    case 8: return std::make_unique<Euler2D<8>>(d);
    case 9: return std::make_unique<Euler2D<9>>(d);
  }
  throw std::invalid_argument("euler2d: device orders are 1..8");
}

}  // namespace expdg
