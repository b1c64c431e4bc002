// 3D compressible Euler, Lax-Friedrichs split (config C5, an extension of the
// reference's 2D EulerOperator, proj/src/euler.cpp:186-388, to hexahedra and
// five conserved variables; the CPU definition is oracle/src/euler.cpp,
// Euler3DOperator).  A z-invariant state with w = 0 reproduces the 2D operator.
//
// Residual / standalone applies: one thread per LGL node, CTA tile of
// floor(256 / NP^3) elements.  Phi-cycle JVP: the z-march kernel below.  The frozen
// data are the per-node primitives (u, v, w, H, a) of q~ (40 B/node, the size of q~
// itself) written once per step by the residual kernel.
#include <algorithm>
#include <cstdlib>
#include <vector>

#include "dots.cuh"
#include "krylov.cuh"

namespace expdg {

namespace {

template <int NP>
struct E3P {
  int nx, ny, nz;
  double gamma;
  double w[NP];
  double WD[NP * NP];
  const double* ut;  // frozen (u, v, w, H, a) per node
  const double* hx;
  const double* hy;
  const double* hz;
  const double* ihx;  // 1 / h tables (the z-march kernel multiplies instead of dividing)
  const double* ihy;
  const double* ihz;
  long long n;
  // z-slab partition: planes -1 and nz are the neighbours' halo planes (raw values of the
  // applied vector / the frozen primitives), exchanged before the kernel runs
  int part;
  int dbg;  // EXPDG_E3_DBG (diagnostics)
  const double* gx_lo;
  const double* gx_hi;
  const double* gt_lo;
  const double* gt_hi;
};

struct Prim3 {
  double u[3], H, a, p;
};

__device__ __forceinline__ Prim3 prim3_of(const double q[5], double gamma) {
  Prim3 pr;
  const double rho = q[0];
  pr.u[0] = q[1] / rho;
  pr.u[1] = q[2] / rho;
  pr.u[2] = q[3] / rho;
  pr.p = (gamma - 1.0) * (q[4] - 0.5 * rho * (pr.u[0] * pr.u[0] + pr.u[1] * pr.u[1] + pr.u[2] * pr.u[2]));
  pr.a = sqrt(gamma * pr.p / rho);
  pr.H = (q[4] + pr.p) / rho;
  return pr;
}

__device__ __forceinline__ Prim3 prim3_frozen(const double t[5]) {
  Prim3 pr;
  pr.u[0] = t[0];
  pr.u[1] = t[1];
  pr.u[2] = t[2];
  pr.H = t[3];
  pr.a = t[4];
  pr.p = 0.0;
  return pr;
}

__device__ __forceinline__ bool admissible5(const double q[5], double gamma) {
  if (!(q[0] > 0.0)) return false;
  const double p = (gamma - 1.0) * (q[4] - 0.5 * (q[1] * q[1] + q[2] * q[2] + q[3] * q[3]) / q[0]);
  return p > 0.0;
}

// out = A(pr, e_dir) x  (rows of the 3D flux Jacobian, oracle jac3), factored so the three
// directions share the x-dependent scalars:  with u.m = sum_c u_c x_{1+c},
//   P = phi x_0 - (g-1) u.m + (g-1) x_4,   Q = (phi - H) x_0 - (g-1) u.m + g x_4,
//   s = x_{1+d} - u_d x_0:   out_0 = x_{1+d},  out_{1+r} = u_r s + u_d x_{1+r} + delta_rd P,
//   out_4 = u_d Q + H x_{1+d}.
// (The entry-by-entry form multiplied by the zero entries: IEEE x * 0 cannot be folded away,
// and the JVP kernels are fp64-bound.)
__device__ __forceinline__ void jac3_pre(const Prim3& pr, double gamma, const double x[5], double& P, double& Q) {
  const double gm1 = gamma - 1.0;
  const double phi = 0.5 * gm1 * fma(pr.u[0], pr.u[0], fma(pr.u[1], pr.u[1], pr.u[2] * pr.u[2]));
  const double um = fma(pr.u[0], x[1], fma(pr.u[1], x[2], pr.u[2] * x[3]));
  P = fma(gm1, x[4] - um, phi * x[0]);
  Q = fma(gamma, x[4], fma(-gm1, um, (phi - pr.H) * x[0]));
}

template <int D>
__device__ __forceinline__ void jac3_dir(const Prim3& pr, double P, double Q, const double x[5], double out[5]) {
  const double un = pr.u[D];
  const double sd = fma(-un, x[0], x[1 + D]);
  out[0] = x[1 + D];
#pragma unroll
  for (int r = 0; r < 3; ++r) {
    const double v = fma(pr.u[r], sd, un * x[1 + r]);
    out[1 + r] = r == D ? v + P : v;
  }
  out[4] = fma(un, Q, pr.H * x[1 + D]);
}

__device__ __forceinline__ void jac3_apply(const Prim3& pr, int dir, double gamma, const double x[5],
                                           double out[5]) {
  double P, Q;
  jac3_pre(pr, gamma, x, P, Q);
  if (dir == 0) jac3_dir<0>(pr, P, Q, x, out);
  else if (dir == 1) jac3_dir<1>(pr, P, Q, x, out);
  else jac3_dir<2>(pr, P, Q, x, out);
}

__device__ __forceinline__ void flux3_dir(const double q[5], const Prim3& pr, int dir, double f[5]) {
  const double vn = pr.u[dir];
  f[0] = q[dir + 1];
  f[1] = q[1] * vn;
  f[2] = q[2] * vn;
  f[3] = q[3] * vn;
  f[dir + 1] += pr.p;
  f[4] = q[0] * vn * pr.H;
}

// face normal +e_dir between owner (m) and neighbour (p): 0 linear LF, 1 full - linear, 2 full
__device__ __forceinline__ void face3(int mode, int dir, double gamma, const double qm[5], const double qp[5],
                                      const double tm_[5], const double tp_[5], double f[5], bool& bad) {
  double lin[5] = {0, 0, 0, 0, 0};
  if (mode != 2) {
    const Prim3 tm = prim3_frozen(tm_), tp = prim3_frozen(tp_);
    double am[5], ap[5];
    jac3_apply(tm, dir, gamma, qm, am);
    jac3_apply(tp, dir, gamma, qp, ap);
    const double lam = fmax(fabs(tm.u[dir]) + tm.a, fabs(tp.u[dir]) + tp.a);
#pragma unroll
    for (int c = 0; c < 5; ++c) lin[c] = 0.5 * (am[c] + ap[c]) + 0.5 * (lam * (qm[c] - qp[c]));
  }
  if (mode == 0) {
#pragma unroll
    for (int c = 0; c < 5; ++c) f[c] = lin[c];
    return;
  }
  if (!admissible5(qm, gamma) || !admissible5(qp, gamma)) bad = true;
  const Prim3 pm = prim3_of(qm, gamma), pp = prim3_of(qp, gamma);
  double fm[5], fp[5];
  flux3_dir(qm, pm, dir, fm);
  flux3_dir(qp, pp, dir, fp);
  const double s = 0.5 * fmax(fabs(pm.u[dir]) + pm.a, fabs(pp.u[dir]) + pp.a);
#pragma unroll
  for (int c = 0; c < 5; ++c) {
    const double full = 0.5 * (fm[c] + fp[c]) + s * (qm[c] - qp[c]);
    f[c] = mode == 1 ? full - lin[c] : full;
  }
}

template <int NP>
struct E3Tile {
  static constexpr int NN = NP * NP * NP;
  static constexpr int TE = 256 / NN > 0 ? 256 / NN : 1;
  static constexpr int VALS = TE * 5 * NN;
};

template <int NP>
__device__ __forceinline__ void load5(const double* sx, const double* su, long long e0, int te, long long e, int node,
                                      const double* x, double xs, const double* ut, double q[5], double t[5],
                                      bool need_ut) {
  constexpr int NN = NP * NP * NP;
  const long long le = e - e0;
  if (le >= 0 && le < te) {
#pragma unroll
    for (int c = 0; c < 5; ++c) {
      q[c] = sx[(le * 5 + c) * NN + node];
      t[c] = need_ut ? ut[((size_t)e * 5 + c) * NN + node] : 0.0;
    }
  } else {
#pragma unroll
    for (int c = 0; c < 5; ++c) {
      const size_t g = ((size_t)e * 5 + c) * NN + node;
      q[c] = x[g] * xs;
      t[c] = need_ut ? ut[g] : 0.0;
    }
  }
}

template <int NP>
__device__ __forceinline__ void e3_tile(const E3P<NP>& P, int mode, long long e0, int te, const double* x, double xs,
                                        double* sx, double* su, double* sf, double out[5], bool& bad) {
  constexpr int NN = NP * NP * NP;
  constexpr int N = NP - 1;
  const int t = threadIdx.x;
  const int le = t / NN, node = t % NN;
  const int i = node % NP, j = (node / NP) % NP, k = node / (NP * NP);
  const bool active = le < te;
  const bool need_ut = mode != 2;
  const int cnt = te * 5 * NN;
  const size_t gbase = (size_t)e0 * 5 * NN;
  for (int idx = t; idx < cnt; idx += blockDim.x) sx[idx] = x[gbase + idx] * xs;
  __syncthreads();
  double q[5], ut[5];
  const long long e = e0 + le;
  int ix = 0, iy = 0, iz = 0;
  if (active) {
    const long long exy = (long long)P.nx * P.ny;
    iz = (int)(e / exy);
    const long long r = e - (long long)iz * exy;
    iy = (int)(r / P.nx);
    ix = (int)(r - (long long)iy * P.nx);
#pragma unroll
    for (int c = 0; c < 5; ++c) {
      q[c] = sx[(le * 5 + c) * NN + node];
      ut[c] = need_ut ? P.ut[gbase + (le * 5 + c) * NN + node] : 0.0;
    }
    double fl[3][5];
    if (mode != 2) {
      const Prim3 tp = prim3_frozen(ut);
#pragma unroll
      for (int d = 0; d < 3; ++d) jac3_apply(tp, d, P.gamma, q, fl[d]);
    }
    if (mode != 0) {
      if (!admissible5(q, P.gamma)) bad = true;
      const Prim3 pq = prim3_of(q, P.gamma);
#pragma unroll
      for (int d = 0; d < 3; ++d) {
        double F[5];
        flux3_dir(q, pq, d, F);
#pragma unroll
        for (int c = 0; c < 5; ++c) fl[d][c] = mode == 1 ? F[c] - fl[d][c] : F[c];
      }
    }
#pragma unroll
    for (int d = 0; d < 3; ++d)
#pragma unroll
      for (int c = 0; c < 5; ++c) sf[((le * 3 + d) * 5 + c) * NN + node] = fl[d][c];
  }
  __syncthreads();
  if (!active) return;
  const double hx = __ldg(P.hx + ix), hy = __ldg(P.hy + iy), hz = __ldg(P.hz + iz);
  const double sxv = (0.25 * hy * hz) * P.w[j] * P.w[k];
  const double syv = (0.25 * hz * hx) * P.w[i] * P.w[k];
  const double szv = (0.25 * hx * hy) * P.w[i] * P.w[j];
  double r[5];
#pragma unroll
  for (int c = 0; c < 5; ++c) {
    const double* fx = sf + ((le * 3 + 0) * 5 + c) * NN + (k * NP + j) * NP;
    const double* fy = sf + ((le * 3 + 1) * 5 + c) * NN + k * NP * NP + i;
    const double* fz = sf + ((le * 3 + 2) * 5 + c) * NN + j * NP + i;
    double ax = 0.0, ay = 0.0, az = 0.0;
#pragma unroll
    for (int m = 0; m < NP; ++m) {
      ax = fma(P.WD[m * NP + i], fx[m], ax);
      ay = fma(P.WD[m * NP + j], fy[m * NP], ay);
      az = fma(P.WD[m * NP + k], fz[m * NP * NP], az);
    }
    r[c] = sxv * ax;
    r[c] += syv * ay;
    r[c] += szv * az;
  }
  // faces: x, y, z (oracle face order), owner on the low side, periodic
  const int idx3[3] = {i, j, k};
  const int nel[3] = {P.nx, P.ny, P.nz};
  const int pos[3] = {ix, iy, iz};
  const double area[3] = {0.25 * (hy * hz), 0.25 * (hx * hz), 0.25 * (hx * hy)};
#pragma unroll
  for (int d = 0; d < 3; ++d) {
    const int a = idx3[d];
    if (a != 0 && a != N) continue;
    const bool owner = a == N;
    int p2[3] = {pos[0], pos[1], pos[2]};
    const int nb = owner ? pos[d] + 1 : pos[d] - 1;
    p2[d] = nb < 0 ? nel[d] - 1 : (nb >= nel[d] ? 0 : nb);
    int n2[3] = {i, j, k};
    n2[d] = owner ? 0 : N;
    const int node2 = (n2[2] * NP + n2[1]) * NP + n2[0];
    double q2[5], u2[5], f[5];
    if (P.part && d == 2 && (nb < 0 || nb >= nel[2])) {  // halo plane of the neighbouring rank
      const double* gx = nb < 0 ? P.gx_lo : P.gx_hi;
      const double* gt = nb < 0 ? P.gt_lo : P.gt_hi;
      const size_t ge = (size_t)p2[1] * P.nx + p2[0];
#pragma unroll
      for (int c = 0; c < 5; ++c) {
        q2[c] = gx[(ge * 5 + c) * NN + node2] * xs;
        u2[c] = need_ut ? gt[(ge * 5 + c) * NN + node2] : 0.0;
      }
    } else {
      const long long e2 = ((long long)p2[2] * P.ny + p2[1]) * P.nx + p2[0];
      load5<NP>(sx, su, e0, te, e2, node2, x, xs, P.ut, q2, u2, need_ut);
    }
    if (owner) face3(mode, d, P.gamma, q, q2, ut, u2, f, bad);
    else face3(mode, d, P.gamma, q2, q, u2, ut, f, bad);
    // face quadrature weight (1/4 area) w_t1 w_t2 with (t1, t2) the two tangential node indices
    const int t1 = d == 0 ? j : i;
    const int t2 = d == 2 ? j : k;
    const double fw = area[d] * P.w[t1] * P.w[t2];
#pragma unroll
    for (int c = 0; c < 5; ++c) r[c] = owner ? r[c] - fw * f[c] : r[c] + fw * f[c];
  }
  const double scale = 8.0 / (hx * hy * hz);
  const double im = scale / (P.w[i] * P.w[j] * P.w[k]);
#pragma unroll
  for (int c = 0; c < 5; ++c) out[c] = r[c] * im;
}

template <int NP>
__global__ void __launch_bounds__(256) k_e3_apply(E3P<NP> P, int mode, const double* __restrict__ x,
                                                  double* __restrict__ y, PhiState* st, double* frozen) {
  constexpr int NN = NP * NP * NP, TE = E3Tile<NP>::TE;
  __shared__ double sx[E3Tile<NP>::VALS], sf[3 * E3Tile<NP>::VALS];
  double* su = nullptr;
  if (st && st->stopped) return;
  const long long ne = (long long)P.nx * P.ny * P.nz;
  const long long ntiles = (ne + TE - 1) / TE;
  bool bad = false;
  for (long long tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
    const long long e0 = tile * TE;
    const int te = (int)(ne - e0 < TE ? ne - e0 : TE);
    __syncthreads();
    double out[5];
    e3_tile<NP>(P, mode, e0, te, x, 1.0, sx, su, sf, out, bad);
    const int t = threadIdx.x, le = t / NN, node = t % NN;
    if (le < te) {
      const long long e = e0 + le;
#pragma unroll
      for (int c = 0; c < 5; ++c) y[((size_t)e * 5 + c) * NN + node] = out[c];
      if (frozen && mode == 2) {
        double qn[5];
#pragma unroll
        for (int c = 0; c < 5; ++c) qn[c] = x[((size_t)e * 5 + c) * NN + node];
        const Prim3 pr = prim3_of(qn, P.gamma);
        const double fv[5] = {pr.u[0], pr.u[1], pr.u[2], pr.H, pr.a};
#pragma unroll
        for (int c = 0; c < 5; ++c) frozen[((size_t)e * 5 + c) * NN + node] = fv[c];
      }
    }
  }
  if (bad && st) st->domain_flag = 1;
}

template <int NP>
__global__ void __launch_bounds__(256) k_e3_phi(E3P<NP> P, PhiState* st, double* base, double* partials, BArgs b) {
  constexpr int NN = NP * NP * NP, TE = E3Tile<NP>::TE;
  __shared__ double sx[E3Tile<NP>::VALS], sf[3 * E3Tile<NP>::VALS];
  double* su = nullptr;
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
  const long long ne = (long long)P.nx * P.ny * P.nz;
  const long long ntiles = (ne + TE - 1) / TE;
  double nacc = 0.0;
  bool bad = false;
  for (long long tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
    const long long e0 = tile * TE;
    const int te = (int)(ne - e0 < TE ? ne - e0 : TE);
    __syncthreads();
    double out[5];
    e3_tile<NP>(P, 0, e0, te, x, xs, sx, su, sf, out, bad);
    const int t = threadIdx.x, le = t / NN, node = t % NN;
    __syncthreads();
    if (le < te) {
#pragma unroll
      for (int c = 0; c < 5; ++c) sx[(le * 5 + c) * NN + node] = out[c];
    }
    __syncthreads();
    for (int idx = t; idx < te * 5 * NN; idx += blockDim.x) {
      const size_t g = (size_t)e0 * 5 * NN + idx;
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

// ---------------------------------------------------------------- z-march JVP (phi cycle)
// A CTA owns a TX x TY tile of element columns at a time and marches up all its
// z-planes.  Warp CW streams the tile's elements of every plane (x = slot j, the frozen
// primitives, b_1) by 1D TMA bulk copies into a 4-plane shared-memory ring, so every
// byte of x and q~ leaves HBM once per JVP; only the face nodes of the x/y neighbour
// elements outside the tile are gathered from L2.  Per plane: phase A computes the
// volume fluxes A(q~) x of every node and every face flux of the plane ONCE (the
// reference's rhs_faces loop, proj/src/euler.cpp:260-297, extended to 3D as in
// oracle/src/euler.cpp): the x- and y-faces of the tile and the z-faces above it (and,
// on a unit's first plane, below it); phase C differentiates and scatters the face
// fluxes into each node.  Orders whose element block (5 NP^3 doubles) is a multiple of
// 16 bytes (NP = 2, 4) use it; NP = 3 keeps the element-tile kernel.
constexpr int kE3DotJ = 44;  // DOT: the sweep takes the DCGS2 dots of columns j < 44

template <int NP, bool DOT = false>
struct E3March {
  static constexpr int NN = NP * NP * NP, NF = NP * NP, BLK = 5 * NN;
  static constexpr int TX = NP == 4 ? 2 : 4, TY = NP == 4 ? 2 : 8;  // TX * TY * NN = 256 (1x2 tiles at two CTAs per SM measured slower)
  static constexpr int TE = TX * TY;
  static constexpr int CONS = TE * NN;
  static constexpr int CW = CONS / 32;
  static constexpr int PL = TE * BLK;           // doubles per array per ring plane
  // x, q~ primitives (+ b_1 without DOT; with DOT b_1 is read in place to leave room for V)
  static constexpr int BUFD = (DOT ? 2 : 3) * PL;
  static constexpr int NBUF = 4;
  static constexpr int FXD = (TX + 1) * TY * NF * 5;  // x-face fluxes of a plane
  static constexpr int FYD = TX * (TY + 1) * NF * 5;  // y-face fluxes
  static constexpr int FZD = TE * NF * 5;              // one layer of z-face fluxes
  static constexpr int BASE = NBUF * BUFD + 3 * 5 * CONS + FXD + FYD + 2 * FZD;
  // DOT (the fused DCGS2 dots, as in the 2D strip sweep, dots.cuh): a V producer warp, two
  // dot warps, the double-buffered w tile handed over by the JVP warps, a V ring
  static constexpr int TILE = TE * BLK;
  static constexpr int ND = DOT ? 2 : 0;
  static constexpr int JMAX = DOT ? kE3DotJ - 1 : -1;
  static constexpr int THREADS = CONS + 32 + (DOT ? 32 + 32 * ND : 0);
  static constexpr int SMAX = 232448 / 8 - 384;
  static constexpr int VSF = (SMAX - BASE - 2 * TILE) / TILE;
  static constexpr int VS = DOT ? (VSF > 16 ? 16 : (VSF < 1 ? 1 : VSF)) : 1;
  static constexpr bool FITS = !DOT || VSF >= 4;
  static constexpr int SMEM = (BASE + (DOT ? 2 * TILE + VS * TILE : 0)) * 8;
  static constexpr bool OK = (BLK * 8) % 16 == 0 && CONS <= 256;  // NP = 2, 4; the other orders keep the tile kernel
};

// Dot warps of the fused z-march: the march's (tile, plane) sequence, u = the tile's x in the
// plane's ring slot, w = the tile handed over by the JVP warps (full tiles only).
template <class S>
__device__ __forceinline__ void march_dots(const double* ring, const double* swr, const double* vring, uint64_t* full,
                                           uint64_t* empty, uint64_t* wfull, uint64_t* wempty, uint64_t* vfull,
                                           uint64_t* vempty, long long ntiles, int nz, int j, double* s_acc) {
  const int lane = threadIdx.x & 31;
  const int h = (threadIdx.x >> 5) - (S::CONS / 32 + 2);
  double* acc = s_acc + h * 2 * (S::JMAX + 1);
  RingPos vp, wp;
  long long seq = 0;
  constexpr int cnt2 = S::TILE / 2;
  for (long long tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
    for (int z = 0; z < nz; ++z) {
      const long long q = z + 1;  // ring index of plane z
      const int bsel = wp.s;
      mbar_wait(&wfull[bsel], wp.ph);
      wp.next<2>();
      const int sl = (int)((seq + q) % S::NBUF);
      mbar_wait(&full[sl], (int)(((seq + q) / S::NBUF) & 1));  // completed phase: returns at once
      const double2* U2 = reinterpret_cast<const double2*>(ring + (size_t)sl * S::BUFD);
      const double2* W2 = reinterpret_cast<const double2*>(swr + bsel * S::TILE);
      dots_row<S, true>(U2, W2, vring, vfull, vempty, vp, j, cnt2, lane, h, acc, 0);
      __syncwarp();
      if (lane == 0) {  // u (the ring plane) and the w tile are free
        mbar_arrive(&wempty[bsel]);
        mbar_arrive(&empty[sl]);
      }
    }
    seq += nz + 2;
  }
}

template <int NP, bool DOT>
__global__ void __launch_bounds__(E3March<NP, DOT>::THREADS, 1)
    k_e3_phi_march(E3P<NP> P, PhiState* st, double* base, double* partials, BArgs b) {
  using S = E3March<NP, DOT>;
  constexpr int NN = S::NN, NF = S::NF, BLK = S::BLK, TX = S::TX, TY = S::TY, NBUF = S::NBUF, N = NP - 1;
  constexpr int CWN = S::CW;  // JVP warps
  extern __shared__ __align__(128) double smem[];
  double* ring = smem;
  double* sf = ring + NBUF * S::BUFD;  // [dir][c][thread]
  double* fxf = sf + 3 * 5 * S::CONS;
  double* fyf = fxf + S::FXD;
  double* fzf = fyf + S::FYD;          // two layers
  double* swr = smem + S::BASE;        // DOT: w tiles handed to the dot warps
  double* vring = swr + 2 * S::TILE;   // DOT: V tiles
  __shared__ uint64_t full[NBUF], empty[NBUF];
  __shared__ uint64_t wfull[2], wempty[2], vfull[S::VS], vempty[S::VS];
  __shared__ int s_go, s_j, s_dots;
  __shared__ double s_xs, s_dt, s_xt[kMaxP];
  __shared__ long long s_ld;
  __shared__ double s_buf[S::THREADS / 32];
  __shared__ double s_red[DOT ? 2 * S::ND * (S::JMAX + 1) : 1];
  const int tid = threadIdx.x, wid = tid >> 5, lane = tid & 31;
  if (tid == 0) {
    s_go = apply_go(st, base);
    if (s_go) {
      s_j = st->j;
      s_dots = DOT && st->dcgs && s_j <= S::JMAX && apply_stage(st, base) == 1;
      if (blockIdx.x == 0) {
        if (DOT && apply_stage(st, base) == 1) st->dots_fused = s_dots;
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
          mbar_init(&wfull[q], CWN);
          mbar_init(&wempty[q], S::ND);
        }
        for (int q = 0; q < S::VS; ++q) {
          mbar_init(&vfull[q], 1);
          mbar_init(&vempty[q], S::ND);
        }
      }
      fence_mbar_init();
    }
  }
  if (DOT)
    for (int q = tid; q < 2 * S::ND * (S::JMAX + 1); q += blockDim.x) s_red[q] = 0.0;
  __syncthreads();
  if (!s_go) return;
  const bool dots = DOT && s_dots;
  const uint32_t rel_row = dots ? 1u : 1u + S::ND, rel_halo = 1u + S::ND;
  const double* x = base + (size_t)s_j * s_ld;
  double* y = base + (size_t)(s_j + 1) * s_ld;
  const double xs = s_xs, dt = s_dt;
  const int nx = P.nx, ny = P.ny, nz = P.nz;
  const int ntx = (nx + TX - 1) / TX, nty = (ny + TY - 1) / TY;
  // CTA c marches tiles c, c + G, c + 2G, ... over the whole z range: at any time the G
  // CTAs work on G consecutive tiles at similar z, so the x/y neighbour faces they gather
  // were staged by a neighbouring CTA moments before and come from L2
  const long long ntiles = (long long)ntx * nty;
  const double* b1 = (b.p == 1) ? b.b[1] : nullptr;
  double nacc = 0.0;
  auto unit = [&](long long tile, int& ix0, int& iy0, int& tx, int& ty, int& z0, int& z1) {
    z0 = 0;
    z1 = nz;
    ix0 = (int)(tile % ntx) * TX;
    iy0 = (int)(tile / ntx) * TY;
    tx = min(TX, nx - ix0);
    ty = min(TY, ny - iy0);
  };

  if (wid == S::CW) {
    // ---------------- producer: the tile's elements of planes z0 - 1 .. z1
    if (lane == 0) {
      long long seq = 0;
      for (long long tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
        int ix0, iy0, tx, ty, z0, z1;
        unit(tile, ix0, iy0, tx, ty, z0, z1);
        for (int q = 0; q < z1 - z0 + 2; ++q, ++seq) {
          int z = z0 - 1 + q;
          const double* srcx = x;
          const double* srct = P.ut;
          size_t pbase;
          if (P.part && (z < 0 || z >= nz)) {  // halo plane of the neighbouring rank
            srcx = z < 0 ? P.gx_lo : P.gx_hi;
            srct = z < 0 ? P.gt_lo : P.gt_hi;
            pbase = 0;
          } else {
            z = z < 0 ? z + nz : (z >= nz ? z - nz : z);
            pbase = (size_t)z * ny * nx;
          }
          const int sl = (int)(seq % NBUF);
          mbar_wait(&empty[sl], (int)(((seq / NBUF) & 1) ^ 1));
          double* dst = ring + (size_t)sl * S::BUFD;
          const bool with_b = !DOT && b1 && q >= 1 && q <= z1 - z0;
          const uint32_t rowb = (uint32_t)tx * BLK * 8;
          mbar_arrive_expect_tx(&full[sl], (2u + (with_b ? 1u : 0u)) * (uint32_t)ty * rowb);
          for (int ly = 0; ly < ty; ++ly) {
            const size_t e = pbase + (size_t)(iy0 + ly) * nx + ix0;
            bulk_g2s(dst + (size_t)ly * TX * BLK, srcx + e * BLK, rowb, &full[sl]);
            bulk_g2s(dst + S::PL + (size_t)ly * TX * BLK, srct + e * BLK, rowb, &full[sl]);
            if (with_b) {
              const size_t eb = ((size_t)(z0 - 1 + q) * ny + iy0 + ly) * nx + ix0;
              bulk_g2s(dst + 2 * S::PL + (size_t)ly * TX * BLK, b1 + eb * BLK, rowb, &full[sl]);
            }
          }
        }
      }
    }
  } else if (wid == S::CW + 1) {
    // ---------------- producer: the tile's elements of V_0..V_{j-1} for every plane (DOT)
    if constexpr (DOT) {
      if (dots && lane == 0) {
        const int jj = s_j;
        const long long ld = s_ld;
        RingPos vp;
        for (long long tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
          int ix0, iy0, tx, ty, z0, z1;
          unit(tile, ix0, iy0, tx, ty, z0, z1);
          const uint32_t rowb = (uint32_t)tx * BLK * 8;
          for (int z = z0; z < z1; ++z) {
            for (int i = 0; i < jj; ++i) {
              const int stg = vp.s;
              mbar_wait(&vempty[stg], vp.ph ^ 1u);
              mbar_arrive_expect_tx(&vfull[stg], (uint32_t)ty * rowb);
              for (int ly = 0; ly < ty; ++ly) {
                const size_t e = ((size_t)z * ny + iy0 + ly) * nx + ix0;
                bulk_g2s(vring + (size_t)stg * S::TILE + (size_t)ly * TX * BLK, base + (size_t)i * ld + e * BLK, rowb,
                         &vfull[stg]);
              }
              vp.next<S::VS>();
            }
          }
        }
      }
    }
  } else if (wid > S::CW + 1) {
    // ---------------- dot warps (DOT)
    if constexpr (DOT) {
      if (dots) march_dots<S>(ring, swr, vring, full, empty, wfull, wempty, vfull, vempty, ntiles, nz, s_j, s_red);
    }
  } else {
    // ---------------- consumers: one thread per node of the tile
    const int le = tid / NN, node = tid % NN;
    const int lx = le % TX, ly = le / TX;
    const int i = node % NP, j = (node / NP) % NP, kk = node / NF;
    // per-thread basis constants in registers (runtime indices into the kernel parameter
    // arrays would be indexed constant-bank loads in the inner loops)
    double wdi[NP], wdj[NP], wdk[NP];
#pragma unroll
    for (int m = 0; m < NP; ++m) {
      wdi[m] = P.WD[m * NP + i];
      wdj[m] = P.WD[m * NP + j];
      wdk[m] = P.WD[m * NP + kk];
    }
    const double wi = P.w[i], wj = P.w[j], wk = P.w[kk];
    const double iw3 = 1.0 / (wi * wj * wk);
    long long seq = 0;
    for (long long tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
      int ix0, iy0, tx, ty, z0, z1;
      unit(tile, ix0, iy0, tx, ty, z0, z1);
      const bool active = lx < tx && ly < ty;
      const int ix = ix0 + lx, iy = iy0 + ly;
      const double hx = active ? __ldg(P.hx + ix) : 1.0, hy = active ? __ldg(P.hy + iy) : 1.0;
      const double ihxy = active ? __ldg(P.ihx + ix) * __ldg(P.ihy + iy) : 1.0;
      auto slot = [&](long long q) { return ring + (size_t)((seq + q) % NBUF) * S::BUFD; };
      auto wait_plane = [&](long long q) { mbar_wait(&full[(seq + q) % NBUF], (int)(((seq + q) / NBUF) & 1)); };
      // faces are enumerated over the full TX x TY tile (compile-time divisors); the ones
      // outside a partial tile are skipped
      constexpr int NFX = (TX + 1) * TY * NF, NFY = TX * (TY + 1) * NF, NFZ = TX * TY * NF;
      wait_plane(0);
      wait_plane(1);
      int wrc = 0;  // DOT: planes handed to the dot warps
      for (int z = z0; z < z1; ++z) {
        const long long q = z - z0 + 1;
        // b_1 of this node (p == 1), read in place: issued now, used in phase C
        double bv[5] = {0.0, 0.0, 0.0, 0.0, 0.0};
        if (DOT && b1 && active) {
          const size_t e = ((size_t)z * ny + iy) * nx + ix;
#pragma unroll
          for (int c = 0; c < 5; ++c) bv[c] = __ldg(b1 + (e * 5 + c) * NN + node);
        }
        wait_plane(q + 1);
        const double* cur = slot(q);
        const double* lo = slot(q - 1);
        const double* hi = slot(q + 1);
        double* fz_bot = fzf + ((z - z0) & 1) * S::FZD;
        double* fz_top = fzf + ((z - z0 + 1) & 1) * S::FZD;
        // ---- phase A.  The operands of this thread's first face flux are gathered first, so
        // the L2 latency of the x/y neighbour faces overlaps the volume arithmetic.
        const int total = NFX + NFY + NFZ + (z == z0 ? NFZ : 0);
        auto from_ring = [&](const double* pl, int e, int nd, double(&qq)[5], double(&tt)[5]) {
#pragma unroll
          for (int c = 0; c < 5; ++c) {
            qq[c] = pl[e * BLK + c * NN + nd] * xs;
            tt[c] = pl[S::PL + e * BLK + c * NN + nd];
          }
        };
        auto from_gmem = [&](int gx, int gy, int nd, double(&qq)[5], double(&tt)[5]) {
          const size_t e = ((size_t)z * ny + gy) * nx + gx;
#pragma unroll
          for (int c = 0; c < 5; ++c) {
            qq[c] = x[(e * 5 + c) * NN + nd] * xs;
            tt[c] = __ldg(P.ut + (e * 5 + c) * NN + nd);
          }
        };
        // operands of face f (false: outside a partial tile)
        auto load_face = [&](int f, double(&qa)[5], double(&ta)[5], double(&qb)[5], double(&tb)[5], int& dir,
                             double*& dst) {
          if (f < NFX) {  // x-face column fc between tile columns fc - 1 (low) and fc (high)
            const int fc = f / (TY * NF), rem = f - fc * TY * NF, fy = rem / NF, fn = rem - fy * NF;
            if (fc > tx || fy >= ty) return false;
            const int nlo = fn * NP + N, nhi = fn * NP;  // fn = k NP + j
            if (fc == 0) from_gmem(ix0 == 0 ? nx - 1 : ix0 - 1, iy0 + fy, nlo, qa, ta);
            else from_ring(cur, fy * TX + fc - 1, nlo, qa, ta);
            if (fc == tx) from_gmem(ix0 + tx == nx ? 0 : ix0 + tx, iy0 + fy, nhi, qb, tb);
            else from_ring(cur, fy * TX + fc, nhi, qb, tb);
            dir = 0;
            dst = fxf + ((fc * TY + fy) * NF + fn) * 5;
          } else if (f < NFX + NFY) {  // y-face row fc between tile rows fc - 1 and fc
            const int g = f - NFX, fc = g / (TX * NF), rem = g - fc * TX * NF, fxl = rem / NF, fn = rem - fxl * NF;
            if (fc > ty || fxl >= tx) return false;
            const int fi = fn % NP, fk = fn / NP;
            const int nlo = (fk * NP + N) * NP + fi, nhi = (fk * NP) * NP + fi;
            if (fc == 0) from_gmem(ix0 + fxl, iy0 == 0 ? ny - 1 : iy0 - 1, nlo, qa, ta);
            else from_ring(cur, (fc - 1) * TX + fxl, nlo, qa, ta);
            if (fc == ty) from_gmem(ix0 + fxl, iy0 + ty == ny ? 0 : iy0 + ty, nhi, qb, tb);
            else from_ring(cur, fc * TX + fxl, nhi, qb, tb);
            dir = 1;
            dst = fyf + ((fc * TX + fxl) * NF + fn) * 5;
          } else {  // z-faces: above this plane (ring planes z | z + 1), or below it on the unit's first plane
            const int g = f - NFX - NFY;
            const bool top = g < NFZ;
            const int gg = top ? g : g - NFZ;
            const int el = gg / NF, fn = gg - el * NF;  // ring element index
            if (el % TX >= tx || el / TX >= ty) return false;
            const int nlo = (N * NP) * NP + fn, nhi = fn;
            from_ring(top ? cur : lo, el, nlo, qa, ta);
            from_ring(top ? hi : cur, el, nhi, qb, tb);
            dir = 2;
            dst = (top ? fz_top : fz_bot) + (el * NF + fn) * 5;
          }
          return true;
        };
        auto face_out = [&](int dir, const double(&qa)[5], const double(&ta)[5], const double(&qb)[5],
                            const double(&tb)[5], double* dst) {
          double fl[5];
          bool bad = false;
          // a compile-time direction keeps the state arrays in registers (jac3_apply indexes them by dir)
          if (dir == 0) face3(0, 0, P.gamma, qa, qb, ta, tb, fl, bad);
          else if (dir == 1) face3(0, 1, P.gamma, qa, qb, ta, tb, fl, bad);
          else face3(0, 2, P.gamma, qa, qb, ta, tb, fl, bad);
#pragma unroll
          for (int c = 0; c < 5; ++c) dst[c] = fl[c];
        };
        double qa[5], ta[5], qb[5], tb[5];
        int dir0 = 0;
        double* dst0 = nullptr;
        const bool has0 = tid < total && load_face(tid, qa, ta, qb, tb, dir0, dst0);
        // volume fluxes of this node
        if (active) {
          double qv[5], tv[5];
#pragma unroll
          for (int c = 0; c < 5; ++c) {
            qv[c] = cur[le * BLK + c * NN + node] * xs;
            tv[c] = cur[S::PL + le * BLK + c * NN + node];
          }
          const Prim3 tp = prim3_frozen(tv);
          double Pv, Qv, fl[5];
          jac3_pre(tp, P.gamma, qv, Pv, Qv);
          jac3_dir<0>(tp, Pv, Qv, qv, fl);
#pragma unroll
          for (int c = 0; c < 5; ++c) sf[(0 * 5 + c) * S::CONS + tid] = fl[c];
          jac3_dir<1>(tp, Pv, Qv, qv, fl);
#pragma unroll
          for (int c = 0; c < 5; ++c) sf[(1 * 5 + c) * S::CONS + tid] = fl[c];
          jac3_dir<2>(tp, Pv, Qv, qv, fl);
#pragma unroll
          for (int c = 0; c < 5; ++c) sf[(2 * 5 + c) * S::CONS + tid] = fl[c];
        }
        // every face flux of the plane, once
        if (has0) face_out(dir0, qa, ta, qb, tb, dst0);
        for (int f = tid + S::CONS; f < total; f += S::CONS) {
          int dir;
          double* dst;
          if (load_face(f, qa, ta, qb, tb, dir, dst)) face_out(dir, qa, ta, qb, tb, dst);
        }
        strip_sync<S::CONS>();  // phase A of plane z complete
        if (tid == 0) mbar_arrive_cnt(&empty[(seq + q - 1) % NBUF], q == 1 ? rel_halo : rel_row);  // plane z - 1
        const int bsel = wrc & 1;
        double* wt = swr + bsel * S::TILE;
        if (dots) mbar_wait(&wempty[bsel], ((wrc >> 1) & 1) ^ 1);  // the dot warps took plane z - 2
        // ---- phase C: differentiate, scatter the face fluxes, scale
        if (active) {
          const double hz = __ldg(P.hz + z);
          const double sxv = (0.25 * hy * hz) * wj * wk;
          const double syv = (0.25 * hz * hx) * wi * wk;
          const double szv = (0.25 * hx * hy) * wi * wj;
          const int t0 = tid - node;  // this element's first thread
          double r[5];
#pragma unroll
          for (int c = 0; c < 5; ++c) {
            const double* fx = sf + (0 * 5 + c) * S::CONS + t0 + (kk * NP + j) * NP;
            const double* fy = sf + (1 * 5 + c) * S::CONS + t0 + kk * NF + i;
            const double* fzz = sf + (2 * 5 + c) * S::CONS + t0 + j * NP + i;
            double ax = 0.0, ay = 0.0, az = 0.0;
#pragma unroll
            for (int m = 0; m < NP; ++m) {
              ax = fma(wdi[m], fx[m], ax);
              ay = fma(wdj[m], fy[m * NP], ay);
              az = fma(wdk[m], fzz[m * NF], az);
            }
            r[c] = sxv * ax;
            r[c] += syv * ay;
            r[c] += szv * az;
          }
          // faces x, y, z (oracle order); owner (low side, node a = N) subtracts
          if (i == 0 || i == N) {
            const double* f = fxf + (((lx + (i == N ? 1 : 0)) * TY + ly) * NF + kk * NP + j) * 5;
            const double fw = (0.25 * (hy * hz)) * wj * wk;
#pragma unroll
            for (int c = 0; c < 5; ++c) r[c] = i == N ? r[c] - fw * f[c] : r[c] + fw * f[c];
          }
          if (j == 0 || j == N) {
            const double* f = fyf + (((ly + (j == N ? 1 : 0)) * TX + lx) * NF + kk * NP + i) * 5;
            const double fw = (0.25 * (hx * hz)) * wi * wk;
#pragma unroll
            for (int c = 0; c < 5; ++c) r[c] = j == N ? r[c] - fw * f[c] : r[c] + fw * f[c];
          }
          if (kk == 0 || kk == N) {
            const double* f = (kk == N ? fz_top : fz_bot) + (le * NF + j * NP + i) * 5;
            const double fw = (0.25 * (hx * hy)) * wi * wj;
#pragma unroll
            for (int c = 0; c < 5; ++c) r[c] = kk == N ? r[c] - fw * f[c] : r[c] + fw * f[c];
          }
          const double im = (8.0 * ihxy * __ldg(P.ihz + z)) * iw3;  // 8 / (hx hy hz w_i w_j w_k)
          const size_t e = ((size_t)z * ny + iy) * nx + ix;
#pragma unroll
          for (int c = 0; c < 5; ++c) {
            const size_t g = (e * 5 + c) * NN + node;
            double v = r[c] * im;
            if (b1) v = fma(s_xt[0], DOT ? bv[c] : cur[(DOT ? 0 : 2) * S::PL + le * BLK + c * NN + node], v);
            else v = aug_tail(b, s_xt, g, v);
            v = dt * v;
            y[g] = v;
            if (dots) wt[le * BLK + c * NN + node] = v;
            nacc = fma(v, v, nacc);
          }
        }
        if (dots) {
          __syncwarp();
          if (lane == 0) mbar_arrive(&wfull[bsel]);
        }
        ++wrc;
        strip_sync<S::CONS>();  // phase C of plane z complete (sf, face arrays reusable)
      }
      if (tid == 0) {
        mbar_arrive_cnt(&empty[(seq + (z1 - z0)) % NBUF], rel_row);       // plane z1 - 1
        mbar_arrive_cnt(&empty[(seq + (z1 - z0) + 1) % NBUF], rel_halo);  // plane z1 (upper halo)
      }
      seq += z1 - z0 + 2;
    }
  }
  __syncthreads();
  if (blockIdx.x == 0 && tid < kTailPad) {  // replicated tail, counted on rank 0
    const double v = (tid + 1 < b.p) ? dt * s_xt[tid + 1] : 0.0;
    y[P.n + tid] = v;
    if (st->tail_here) nacc = fma(v, v, nacc);
  }
  const double tot = block_sum(nacc, s_buf);
  // dots (DOT): the dot warps' sums in warp order, plus (rank 0) the tail region
  // [n, n + kTailPad) of every slot; cnt <= JMAX + 1 <= blockDim.x
  const int cnt = dots ? s_j + 1 : 0;
  double ca = 0.0, cb = 0.0;
  if (DOT && tid < cnt) {
    constexpr int JS = 2 * (S::JMAX + 1);
#pragma unroll
    for (int q = 0; q < (DOT ? S::ND : 1); ++q) {
      ca += s_red[q * JS + 2 * tid];
      cb += s_red[q * JS + 2 * tid + 1];
    }
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
  if (DOT && tid < cnt) {
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

#ifndef EXPDG_E3_FWARPS
#define EXPDG_E3_FWARPS 6
#endif
// ---------------------------------------------------------------- z-march with face warps
// The plain (no dots) march of the phi cycle, role-split: eight node warps (one thread per node:
// volume fluxes of plane z into a double-buffered flux array, one CTA-group barrier, then the
// differentiation / face scatter / store of plane z), four face warps computing every face flux
// of the plane ONE PLANE AHEAD of the node warps (double-buffered x/y face arrays, a 4-layer ring
// of z-face layers, full/empty mbarriers), and the TMA producer warp.  The face warps' L2
// gathers of the x/y neighbour faces and their flux arithmetic run under the node warps'
// phases instead of between their barriers, and the node warps need one barrier per plane.
template <int NP>
struct E3MarchFW {
  using B = E3March<NP, false>;
  static constexpr int NN = B::NN, NF = B::NF, BLK = B::BLK, TX = B::TX, TY = B::TY, TE = B::TE;
  static constexpr int CONS = B::CONS, CW = B::CW, PL = B::PL;
  static constexpr int FWARPS = EXPDG_E3_FWARPS, FTH = 32 * FWARPS;
  static constexpr int THREADS = CONS + 32 + FTH;
  static constexpr int BUFD = 3 * PL;  // x, q~ primitives, b_1
  static constexpr int NBUF = 4;
  // x-face columns / y-face rows padded by two doubles: the low- and high-side nodes of an
  // element then read their faces from different banks in the scatter
  static constexpr int FXC = TY * NF * 5 + 2, FYR = TX * NF * 5 + 2;
  static constexpr int FXD = (TX + 1) * FXC, FYD = (TY + 1) * FYR, FZD = B::FZD;
  static constexpr int SF = 3 * 5 * CONS;  // [dir][c][thread], two buffers
  static constexpr int NZL = 4;            // z-face layers in flight
  static constexpr int SMEM = (NBUF * BUFD + 2 * SF + 2 * (FXD + FYD) + NZL * FZD) * 8;
  static constexpr bool OK = B::OK && SMEM <= 232448 - 3072;
};

// MODE 0: the linear operator (the phi cycle's JVP).  Standalone only: MODE 2, the full right-hand
// side R(x) (oracle/src/euler.cpp, Euler3DOperator: nonlinear volume fluxes, full LF face fluxes),
// which also writes the frozen primitives of x for the step's JVPs and raises fst->domain_flag on
// an inadmissible state -- the residual of every step (expdg_op_full_rhs, launch_residual);
// MODE 1, the nonlinear remainder N(x) = R(x) - L x (expdg_op_apply_nonlinear, the EXPRB stages).
template <int NP, int MODE, bool SOLO>
__global__ void __launch_bounds__(E3MarchFW<NP>::THREADS, 1)
    k_e3_phi_march_fw(E3P<NP> P, PhiState* st, double* base, double* partials, BArgs b, const double* xin,
                      double* yout, PhiState* fst, double* frozen) {
  // SOLO: the standalone operator application y = L x / N(x) / R(x) (expdg_op_apply_linear, ..),
  // x / y the caller's vectors, no augmentation tail, no reductions (st is null); a compile-time
  // switch so that the phi-cycle instantiation keeps its registers
  static_assert(SOLO || MODE == 0, "the phi cycle applies the linear operator");
  if (MODE != 0 && fst && fst->stopped) return;
  bool bad = false;
  using S = E3MarchFW<NP>;
  constexpr int NN = S::NN, NF = S::NF, BLK = S::BLK, TX = S::TX, TY = S::TY, NBUF = S::NBUF, N = NP - 1;
  extern __shared__ __align__(128) double smem[];
  double* ring = smem;
  double* sf0 = ring + NBUF * S::BUFD;
  double* fxy0 = sf0 + 2 * S::SF;                  // two sets of [x faces | y faces]
  double* fzl = fxy0 + 2 * (S::FXD + S::FYD);      // NZL layers
  __shared__ uint64_t full[NBUF], empty[NBUF], ffull[2], fempty[2];
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
  __syncthreads();
  if (!s_go) return;
  const double* x = SOLO ? xin : base + (size_t)s_j * s_ld;
  double* y = SOLO ? yout : base + (size_t)(s_j + 1) * s_ld;
  const double xs = s_xs, dt = s_dt;
  const int nx = P.nx, ny = P.ny, nz = P.nz;
  const int ntx = (nx + TX - 1) / TX, nty = (ny + TY - 1) / TY;
  const long long ntiles = (long long)ntx * nty;  // CTA c marches tiles c, c + G, ... (see k_e3_phi_march)
  const double* b1 = (b.p == 1) ? b.b[1] : nullptr;
  const bool l2pf = (P.dbg & 8) == 0;  // EXPDG_E3_DBG bit 3: no neighbour prefetch
  double nacc = 0.0;
  auto unit = [&](long long tile, int& ix0, int& iy0, int& tx, int& ty) {
    ix0 = (int)(tile % ntx) * TX;
    iy0 = (int)(tile / ntx) * TY;
    tx = min(TX, nx - ix0);
    ty = min(TY, ny - iy0);
  };

  if (wid == S::CW) {
    // ---------------- producer: the tile's elements of planes -1 .. nz
    if (lane == 0) {
      long long seq = 0;
      for (long long tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
        int ix0, iy0, tx, ty;
        unit(tile, ix0, iy0, tx, ty);
        for (int q = 0; q < nz + 2; ++q, ++seq) {
          int z = q - 1;
          const double* srcx = x;
          const double* srct = P.ut;
          size_t pbase;
          if (P.part && (z < 0 || z >= nz)) {  // halo plane of the neighbouring rank
            srcx = z < 0 ? P.gx_lo : P.gx_hi;
            srct = z < 0 ? P.gt_lo : P.gt_hi;
            pbase = 0;
          } else {
            z = z < 0 ? z + nz : (z >= nz ? z - nz : z);
            pbase = (size_t)z * ny * nx;
          }
          const int sl = (int)(seq % NBUF);
          mbar_wait(&empty[sl], (int)(((seq / NBUF) & 1) ^ 1));
          double* dst = ring + (size_t)sl * S::BUFD;
          const bool with_b = b1 && q >= 1 && q <= nz;
          const uint32_t rowb = (uint32_t)tx * BLK * 8;
          mbar_arrive_expect_tx(&full[sl], ((MODE == 2 ? 1u : 2u) + (with_b ? 1u : 0u)) * (uint32_t)ty * rowb);
          for (int ly = 0; ly < ty; ++ly) {
            const size_t e = pbase + (size_t)(iy0 + ly) * nx + ix0;
            bulk_g2s(dst + (size_t)ly * TX * BLK, srcx + e * BLK, rowb, &full[sl]);
            if (MODE != 2) bulk_g2s(dst + S::PL + (size_t)ly * TX * BLK, srct + e * BLK, rowb, &full[sl]);
            if (with_b) {
              const size_t eb = ((size_t)(q - 1) * ny + iy0 + ly) * nx + ix0;
              bulk_g2s(dst + 2 * S::PL + (size_t)ly * TX * BLK, b1 + eb * BLK, rowb, &full[sl]);
            }
          }
          // The x/y neighbour elements of this plane into L2 ahead of the face warps' gathers of
          // their face nodes (L2 hit rate of the launch 29 -> 45 %, 0.912 -> 0.906 ms at C5).  The
          // DRAM bytes do not move (2.36 GB read for 2.01 algorithmic): the excess is the y-neighbour
          // rows across round boundaries (CTA c marches tiles c, c + G, ...: a round is 4.6 tile
          // rows, so ~22 % of the tiles meet their N or S neighbour a whole round, ~280 MB of
          // traffic, later), which no prefetch distance covers.
          if (l2pf && q >= 1 && q <= nz) {
            const uint32_t eb = BLK * 8;
            const int gw = ix0 == 0 ? nx - 1 : ix0 - 1, ge = ix0 + tx == nx ? 0 : ix0 + tx;
            const int gs = iy0 == 0 ? ny - 1 : iy0 - 1, gn = iy0 + ty == ny ? 0 : iy0 + ty;
            for (int ly = 0; ly < ty; ++ly) {
              const size_t row = pbase + (size_t)(iy0 + ly) * nx;
              bulk_prefetch_l2(x + (row + gw) * BLK, eb);
              bulk_prefetch_l2(x + (row + ge) * BLK, eb);
              if (MODE != 2) {
                bulk_prefetch_l2(P.ut + (row + gw) * BLK, eb);
                bulk_prefetch_l2(P.ut + (row + ge) * BLK, eb);
              }
            }
            bulk_prefetch_l2(x + (pbase + (size_t)gs * nx + ix0) * BLK, rowb);
            bulk_prefetch_l2(x + (pbase + (size_t)gn * nx + ix0) * BLK, rowb);
            if (MODE != 2) {
              bulk_prefetch_l2(P.ut + (pbase + (size_t)gs * nx + ix0) * BLK, rowb);
              bulk_prefetch_l2(P.ut + (pbase + (size_t)gn * nx + ix0) * BLK, rowb);
            }
          }
        }
      }
    }
  } else if (wid > S::CW) {
    // ---------------- face warps: every face flux of plane z, once (the reference's rhs_faces
    // loop, proj/src/euler.cpp:260-297, extended to 3D as in oracle/src/euler.cpp)
    const int ft = tid - (S::CONS + 32), fw = wid - (S::CW + 1);
    constexpr int NFX = (TX + 1) * TY * NF, NFY = TX * (TY + 1) * NF, NFZ = TX * TY * NF;
    long long seq = 0;
    unsigned it = 0, lc = 0;
    for (long long tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
      int ix0, iy0, tx, ty;
      unit(tile, ix0, iy0, tx, ty);
      auto wait_plane = [&](long long q) { mbar_wait(&full[(seq + q) % NBUF], (int)(((seq + q) / NBUF) & 1)); };
      auto slot = [&](long long q) { return ring + (size_t)((seq + q) % NBUF) * S::BUFD; };
      wait_plane(0);
      wait_plane(1);
      unsigned lb = lc++ % S::NZL;
      for (int z = 0; z < nz; ++z, ++it) {
        const long long q = z + 1;
        const unsigned lt = lc++ % S::NZL;
        wait_plane(q + 1);
        const int set = it & 1;
        mbar_wait(&fempty[set], ((it >> 1) & 1) ^ 1);  // the node warps consumed this set two planes ago
        const double* cur = slot(q);
        const double* lo = slot(q - 1);
        const double* hi = slot(q + 1);
        double* fxf = fxy0 + set * (S::FXD + S::FYD);
        double* fyf = fxf + S::FXD;
        double* fz_bot = fzl + lb * S::FZD;
        double* fz_top = fzl + lt * S::FZD;
        const int total = NFX + NFY + NFZ + (z == 0 ? NFZ : 0);
        auto from_ring = [&](const double* pl, int e, int nd, double(&qq)[5], double(&tt)[5]) {
#pragma unroll
          for (int c = 0; c < 5; ++c) {
            qq[c] = pl[e * BLK + c * NN + nd] * xs;
            tt[c] = MODE == 2 ? 0.0 : pl[S::PL + e * BLK + c * NN + nd];
          }
        };
        auto from_gmem = [&](int gx, int gy, int nd, double(&qq)[5], double(&tt)[5]) {
          const size_t e = ((size_t)z * ny + gy) * nx + gx;
#pragma unroll
          for (int c = 0; c < 5; ++c) {
            qq[c] = x[(e * 5 + c) * NN + nd] * xs;
            tt[c] = MODE == 2 ? 0.0 : __ldg(P.ut + (e * 5 + c) * NN + nd);
          }
        };
        for (int f = ft; f < total; f += S::FTH) {
          double qa[5], ta[5], qb[5], tb[5], fl[5];
          double* dst;
          if (f < NFX) {  // x-face column fc between tile columns fc - 1 (low) and fc (high)
            const int fc = f / (TY * NF), rem = f - fc * TY * NF, fy = rem / NF, fn = rem - fy * NF;
            if (fc > tx || fy >= ty) continue;
            const int nlo = fn * NP + N, nhi = fn * NP;  // fn = k NP + j
            if (fc == 0) from_gmem(ix0 == 0 ? nx - 1 : ix0 - 1, iy0 + fy, nlo, qa, ta);
            else from_ring(cur, fy * TX + fc - 1, nlo, qa, ta);
            if (fc == tx) from_gmem(ix0 + tx == nx ? 0 : ix0 + tx, iy0 + fy, nhi, qb, tb);
            else from_ring(cur, fy * TX + fc, nhi, qb, tb);
            face3(MODE, 0, P.gamma, qa, qb, ta, tb, fl, bad);
            dst = fxf + fc * S::FXC + (fy * NF + fn) * 5;
          } else if (f < NFX + NFY) {  // y-face row fc between tile rows fc - 1 and fc
            const int g = f - NFX, fc = g / (TX * NF), rem = g - fc * TX * NF, fxl = rem / NF, fn = rem - fxl * NF;
            if (fc > ty || fxl >= tx) continue;
            const int fi = fn % NP, fk = fn / NP;
            const int nlo = (fk * NP + N) * NP + fi, nhi = (fk * NP) * NP + fi;
            if (fc == 0) from_gmem(ix0 + fxl, iy0 == 0 ? ny - 1 : iy0 - 1, nlo, qa, ta);
            else from_ring(cur, (fc - 1) * TX + fxl, nlo, qa, ta);
            if (fc == ty) from_gmem(ix0 + fxl, iy0 + ty == ny ? 0 : iy0 + ty, nhi, qb, tb);
            else from_ring(cur, fc * TX + fxl, nhi, qb, tb);
            face3(MODE, 1, P.gamma, qa, qb, ta, tb, fl, bad);
            dst = fyf + fc * S::FYR + (fxl * NF + fn) * 5;
          } else {  // z-faces: above this plane, or below it on the tile's first plane
            const int g = f - NFX - NFY;
            const bool top = g < NFZ;
            const int gg = top ? g : g - NFZ;
            const int el = gg / NF, fn = gg - el * NF;
            if (el % TX >= tx || el / TX >= ty) continue;
            from_ring(top ? cur : lo, el, (N * NP) * NP + fn, qa, ta);
            from_ring(top ? hi : cur, el, fn, qb, tb);
            face3(MODE, 2, P.gamma, qa, qb, ta, tb, fl, bad);
            dst = (top ? fz_top : fz_bot) + (el * NF + fn) * 5;
          }
#pragma unroll
          for (int c = 0; c < 5; ++c) dst[c] = fl[c];
        }
        __syncwarp();
        if (lane == 0) {
          mbar_arrive(&ffull[set]);
          // plane z is no longer needed here (the next iteration reads z + 1, z + 2); the halo
          // planes are read by the face warps only, so warp 0 also arrives for the node warps
          mbar_arrive(&empty[(seq + q) % NBUF]);
          if (z == 0) mbar_arrive_cnt(&empty[seq % NBUF], fw == 0 ? 2u : 1u);
          if (z == nz - 1) mbar_arrive_cnt(&empty[(seq + q + 1) % NBUF], fw == 0 ? 2u : 1u);
        }
        lb = lt;
      }
      seq += nz + 2;
    }
  } else {
    // ---------------- node warps: one thread per node of the tile
    const int le = tid / NN, node = tid % NN;
    const int lx = le % TX, ly = le / TX;
    const int i = node % NP, j = (node / NP) % NP, kk = node / NF;
    double wdi[NP], wdj[NP], wdk[NP];
#pragma unroll
    for (int m = 0; m < NP; ++m) {
      wdi[m] = P.WD[m * NP + i];
      wdj[m] = P.WD[m * NP + j];
      wdk[m] = P.WD[m * NP + kk];
    }
    const double wi = P.w[i], wj = P.w[j], wk = P.w[kk];
    const double iw3 = 1.0 / (wi * wj * wk);
    long long seq = 0;
    unsigned it = 0, lc = 0;
    int prev_slot = -1;  // ring slot of the plane differentiated in the previous iteration
    for (long long tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
      int ix0, iy0, tx, ty;
      unit(tile, ix0, iy0, tx, ty);
      const bool active = lx < tx && ly < ty;
      const int ix = ix0 + lx, iy = iy0 + ly;
      const double hx = active ? __ldg(P.hx + ix) : 1.0, hy = active ? __ldg(P.hy + iy) : 1.0;
      const double ihxy = active ? __ldg(P.ihx + ix) * __ldg(P.ihy + iy) : 1.0;
      unsigned lb = lc++ % S::NZL;
      for (int z = 0; z < nz; ++z, ++it) {
        const long long q = z + 1;
        const unsigned lt = lc++ % S::NZL;
        const int sl = (int)((seq + q) % NBUF);
        const double hz = __ldg(P.hz + z), ihz = __ldg(P.ihz + z);  // issued before the waits, used after them
        mbar_wait(&full[sl], (int)(((seq + q) / NBUF) & 1));
        const double* cur = ring + (size_t)sl * S::BUFD;
        double* sf = sf0 + (it & 1) * S::SF;
        // ---- volume fluxes of this node
        if (active) {
          double qv[5], fl[5];
#pragma unroll
          for (int c = 0; c < 5; ++c) qv[c] = cur[le * BLK + c * NN + node] * xs;
          if constexpr (MODE == 0) {  // one direction at a time: 5 live flux values, not 15
            double tv[5];
#pragma unroll
            for (int c = 0; c < 5; ++c) tv[c] = cur[S::PL + le * BLK + c * NN + node];
            const Prim3 tp = prim3_frozen(tv);
            double Pv, Qv;
            jac3_pre(tp, P.gamma, qv, Pv, Qv);
            jac3_dir<0>(tp, Pv, Qv, qv, fl);
#pragma unroll
            for (int c = 0; c < 5; ++c) sf[(0 * 5 + c) * S::CONS + tid] = fl[c];
            jac3_dir<1>(tp, Pv, Qv, qv, fl);
#pragma unroll
            for (int c = 0; c < 5; ++c) sf[(1 * 5 + c) * S::CONS + tid] = fl[c];
            jac3_dir<2>(tp, Pv, Qv, qv, fl);
#pragma unroll
            for (int c = 0; c < 5; ++c) sf[(2 * 5 + c) * S::CONS + tid] = fl[c];
          } else {  // F(q) (MODE 2), F(q) - A(q~) q (MODE 1), as the tile kernel (e3_tile)
            double lin[3][5];
            if constexpr (MODE == 1) {
              double tv[5];
#pragma unroll
              for (int c = 0; c < 5; ++c) tv[c] = cur[S::PL + le * BLK + c * NN + node];
              const Prim3 tp = prim3_frozen(tv);
              double Pv, Qv;
              jac3_pre(tp, P.gamma, qv, Pv, Qv);
              jac3_dir<0>(tp, Pv, Qv, qv, lin[0]);
              jac3_dir<1>(tp, Pv, Qv, qv, lin[1]);
              jac3_dir<2>(tp, Pv, Qv, qv, lin[2]);
            }
            if (!admissible5(qv, P.gamma)) bad = true;
            const Prim3 pq = prim3_of(qv, P.gamma);
#pragma unroll
            for (int d = 0; d < 3; ++d) {
              flux3_dir(qv, pq, d, fl);
#pragma unroll
              for (int c = 0; c < 5; ++c) sf[(d * 5 + c) * S::CONS + tid] = MODE == 1 ? fl[c] - lin[d][c] : fl[c];
            }
            if (MODE == 2 && frozen) {  // (u, v, w, H, a) of the state for this step's JVPs
              const double fv[5] = {pq.u[0], pq.u[1], pq.u[2], pq.H, pq.a};
              const size_t e = ((size_t)z * ny + iy) * nx + ix;
#pragma unroll
              for (int c = 0; c < 5; ++c) frozen[(e * 5 + c) * NN + node] = fv[c];
            }
          }
        }
        strip_sync<S::CONS>();  // volume fluxes of plane z complete; every thread is past plane z - 1
        if (tid == 0 && prev_slot >= 0) {
          mbar_arrive(&empty[prev_slot]);
          mbar_arrive(&fempty[(it - 1) & 1]);
        }
        prev_slot = sl;
        mbar_wait(&ffull[it & 1], (it >> 1) & 1);  // the face fluxes of plane z
        // ---- differentiate, scatter the face fluxes, scale
        if (active) {
          const double* fxf = fxy0 + (it & 1) * (S::FXD + S::FYD);
          const double* fyf = fxf + S::FXD;
          const double* fz_bot = fzl + lb * S::FZD;
          const double* fz_top = fzl + lt * S::FZD;
          const double sxv = (0.25 * hy * hz) * wj * wk;
          const double syv = (0.25 * hz * hx) * wi * wk;
          const double szv = (0.25 * hx * hy) * wi * wj;
          const int t0 = tid - node;  // this element's first thread
          double r[5];
#pragma unroll
          for (int c = 0; c < 5; ++c) {
            const double* fx = sf + (0 * 5 + c) * S::CONS + t0 + (kk * NP + j) * NP;
            const double* fy = sf + (1 * 5 + c) * S::CONS + t0 + kk * NF + i;
            const double* fzz = sf + (2 * 5 + c) * S::CONS + t0 + j * NP + i;
            double ax = 0.0, ay = 0.0, az = 0.0;
#pragma unroll
            for (int m = 0; m < NP; ++m) {
              ax = fma(wdi[m], fx[m], ax);
              ay = fma(wdj[m], fy[m * NP], ay);
              az = fma(wdk[m], fzz[m * NF], az);
            }
            r[c] = sxv * ax;
            r[c] += syv * ay;
            r[c] += szv * az;
          }
          // faces x, y, z (oracle order); owner (low side, node a = N) subtracts
          if (i == 0 || i == N) {
            const double* f = fxf + (lx + (i == N ? 1 : 0)) * S::FXC + (ly * NF + kk * NP + j) * 5;
            const double fw = (0.25 * (hy * hz)) * wj * wk;
#pragma unroll
            for (int c = 0; c < 5; ++c) r[c] = i == N ? r[c] - fw * f[c] : r[c] + fw * f[c];
          }
          if (j == 0 || j == N) {
            const double* f = fyf + (ly + (j == N ? 1 : 0)) * S::FYR + (lx * NF + kk * NP + i) * 5;
            const double fw = (0.25 * (hx * hz)) * wi * wk;
#pragma unroll
            for (int c = 0; c < 5; ++c) r[c] = j == N ? r[c] - fw * f[c] : r[c] + fw * f[c];
          }
          if (kk == 0 || kk == N) {
            const double* f = (kk == N ? fz_top : fz_bot) + (le * NF + j * NP + i) * 5;
            const double fw = (0.25 * (hx * hy)) * wi * wj;
#pragma unroll
            for (int c = 0; c < 5; ++c) r[c] = kk == N ? r[c] - fw * f[c] : r[c] + fw * f[c];
          }
          const double im = (8.0 * ihxy * ihz) * iw3;  // 8 / (hx hy hz w_i w_j w_k)
          const size_t e = ((size_t)z * ny + iy) * nx + ix;
#pragma unroll
          for (int c = 0; c < 5; ++c) {
            const size_t g = (e * 5 + c) * NN + node;
            double v = r[c] * im;
            if (b1) v = fma(s_xt[0], cur[2 * S::PL + le * BLK + c * NN + node], v);
            else v = aug_tail(b, s_xt, g, v);
            v = dt * v;
            y[g] = v;
            nacc = fma(v, v, nacc);
          }
        }
        lb = lt;
      }
      seq += nz + 2;
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

__global__ void k_e3_freeze(const double* __restrict__ q, long long nelem, int nn, double gamma,
                            double* __restrict__ frozen) {
  const long long nodes = nelem * nn;
  const long long stride = (long long)gridDim.x * blockDim.x;
  for (long long g = (long long)blockIdx.x * blockDim.x + threadIdx.x; g < nodes; g += stride) {
    const long long e = g / nn;
    const int node = (int)(g - e * nn);
    double qn[5];
    for (int c = 0; c < 5; ++c) qn[c] = q[(e * 5 + c) * nn + node];
    const Prim3 pr = prim3_of(qn, gamma);
    const double fv[5] = {pr.u[0], pr.u[1], pr.u[2], pr.H, pr.a};
    for (int c = 0; c < 5; ++c) frozen[(e * 5 + c) * nn + node] = fv[c];
  }
}


template <int NP>
class Euler3D : public OpDevice {
 public:
  E3P<NP> P{};
  int grid = 1;
  double* frozen = nullptr;
  double* hbuf = nullptr;
  double* halo = nullptr;  // slab partition: x lo/hi, frozen lo/hi, send lo/hi planes
  long long plane = 0;     // doubles per element plane
  bool use_march = E3March<NP>::OK;  // EXPDG_E3_TILE=1: the element-tile JVP
  int march_grid = 1;
  // the plain march with face warps (EXPDG_E3_FW=0: the single-role march)
  static constexpr bool kFwOk = E3March<NP>::OK && E3MarchFW<NP>::OK;
  bool use_fw = kFwOk;
  bool rhs_march = true;  // EXPDG_E3_RHS_TILE=1: the element-tile kernel for R(x) (residual, full_rhs)
  // the z-march also takes the DCGS2 pass-1 dots (EXPDG_E3_DOTS=0: off) on meshes of whole
  // tiles (the dot warps read the tile's elements as one contiguous block)
  static constexpr bool kDotFits = E3March<NP>::OK && E3March<NP, true>::FITS;
  bool use_dots = true;
  bool whole_tiles = false;
  int dots_grid = 1;
  bool dots_on() const { return kDotFits && use_march && use_dots && whole_tiles; }
  int fused_dcgs_dots_jmax() const override { return dots_on() ? E3March<NP, true>::JMAX : -1; }
  ~Euler3D() override {
    cudaFree(frozen);
    cudaFree(hbuf);
    cudaFree(halo);
  }
  double* hb_(int q) const { return halo + (size_t)q * plane; }
  void exchange(cudaStream_t s, const double* v, double* lo, double* hi) {
    comm->halo(v, v + (size_t)(P.nz - 1) * plane, lo, hi, plane, s);
  }
  E3P<NP> params(const double* ut) const {
    E3P<NP> p = P;
    p.ut = ut;
    if (p.part) {
      p.gx_lo = hb_(0);
      p.gx_hi = hb_(1);
      p.gt_lo = hb_(2);
      p.gt_hi = hb_(3);
    }
    return p;
  }
  explicit Euler3D(const expdg_op_desc& d) {
    desc = d;
    const HostBasis hb = host_lgl_basis(d.order);
    const bool part = d.part_end > d.part_begin;
    const int z0 = part ? d.part_begin : 0;
    const int nzl = part ? d.part_end - d.part_begin : d.nz;
    P.nx = d.nx;
    P.ny = d.ny;
    P.nz = nzl;
    P.part = part ? 1 : 0;
    P.gamma = d.gamma;
    std::vector<double> hs(2 * (d.nx + d.ny + nzl));
    const std::vector<double> xs = host_axis_breaks(d.x0, d.x1, d.nx, d.grade_x);
    const std::vector<double> ys = host_axis_breaks(d.y0, d.y1, d.ny, d.grade_y);
    const std::vector<double> zs = host_axis_breaks(d.z0, d.z1, d.nz, d.grade_z);
    for (int i = 0; i < d.nx; ++i) hs[i] = xs[i + 1] - xs[i];
    for (int j = 0; j < d.ny; ++j) hs[d.nx + j] = ys[j + 1] - ys[j];
    for (int k = 0; k < nzl; ++k) hs[d.nx + d.ny + k] = zs[z0 + k + 1] - zs[z0 + k];
    EXPDG_CUDA(cudaMalloc(&hbuf, sizeof(double) * hs.size()));
    EXPDG_CUDA(cudaMemcpy(hbuf, hs.data(), sizeof(double) * hs.size(), cudaMemcpyHostToDevice));
    const int nh = d.nx + d.ny + nzl;
    for (int q = 0; q < nh; ++q) hs[nh + q] = 1.0 / hs[q];
    EXPDG_CUDA(cudaMemcpy(hbuf, hs.data(), sizeof(double) * hs.size(), cudaMemcpyHostToDevice));
    P.hx = hbuf;
    P.hy = hbuf + d.nx;
    P.hz = hbuf + d.nx + d.ny;
    P.ihx = hbuf + nh;
    P.ihy = hbuf + nh + d.nx;
    P.ihz = hbuf + nh + d.nx + d.ny;
    for (int a = 0; a < NP; ++a) {
      P.w[a] = hb.weights[a];
      for (int b2 = 0; b2 < NP; ++b2) P.WD[a * NP + b2] = hb.weights[a] * hb.D[a * NP + b2];
    }
    n = (long long)d.nx * d.ny * nzl * NP * NP * NP * 5;
    P.n = n;
    comps = 5;
    plane = (long long)d.nx * d.ny * NP * NP * NP * 5;
    EXPDG_CUDA(cudaMalloc(&frozen, sizeof(double) * n));
    if (part) {
      EXPDG_CUDA(cudaMalloc(&halo, sizeof(double) * 6 * plane));
      EXPDG_CUDA(cudaMemset(halo, 0, sizeof(double) * 6 * plane));
    }
    const long long ntiles = ((long long)d.nx * d.ny * nzl + E3Tile<NP>::TE - 1) / E3Tile<NP>::TE;
    grid = (int)std::max<long long>(1, std::min<long long>(ntiles, 148LL * 8));
    if (const char* v = std::getenv("EXPDG_E3_TILE")) use_march = use_march && v[0] != '1';
    if (const char* v = std::getenv("EXPDG_E3_DOTS")) use_dots = v[0] != '0';
    if constexpr (E3March<NP>::OK) {
      using SM = E3March<NP>;
      EXPDG_CUDA(cudaFuncSetAttribute(k_e3_phi_march<NP, false>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                      SM::SMEM));
      int per_sm = 1;
      EXPDG_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_e3_phi_march<NP, false>, SM::THREADS,
                                                               SM::SMEM));
      const long long tiles = (long long)((d.nx + SM::TX - 1) / SM::TX) * ((d.ny + SM::TY - 1) / SM::TY);
      march_grid = (int)std::max<long long>(1, std::min<long long>(tiles, 148LL * std::max(1, per_sm)));
      whole_tiles = d.nx % SM::TX == 0 && d.ny % SM::TY == 0;
      if (const char* v = std::getenv("EXPDG_E3_FW")) use_fw = use_fw && v[0] != '0';
    if (const char* v = std::getenv("EXPDG_E3_DBG")) P.dbg = std::atoi(v);
    if (const char* v = std::getenv("EXPDG_E3_RHS_TILE")) rhs_march = v[0] != '1';
      if constexpr (kFwOk)
      {
        EXPDG_CUDA(cudaFuncSetAttribute(k_e3_phi_march_fw<NP, 0, false>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                        E3MarchFW<NP>::SMEM));
        EXPDG_CUDA(cudaFuncSetAttribute(k_e3_phi_march_fw<NP, 0, true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                        E3MarchFW<NP>::SMEM));
        EXPDG_CUDA(cudaFuncSetAttribute(k_e3_phi_march_fw<NP, 2, true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                        E3MarchFW<NP>::SMEM));
        EXPDG_CUDA(cudaFuncSetAttribute(k_e3_phi_march_fw<NP, 1, true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                        E3MarchFW<NP>::SMEM));
      }
      if constexpr (kDotFits) {
        using SD = E3March<NP, true>;
        EXPDG_CUDA(cudaFuncSetAttribute(k_e3_phi_march<NP, true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                        SD::SMEM));
        int pd = 1;
        EXPDG_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&pd, k_e3_phi_march<NP, true>, SD::THREADS, SD::SMEM));
        dots_grid = (int)std::max<long long>(1, std::min<long long>(tiles, 148LL * std::max(1, pd)));
      }
    }
  }
  void freeze(cudaStream_t s, const double* r) override {
    ref = r;
    k_e3_freeze<<<1184, 256, 0, s>>>(r, (long long)P.nx * P.ny * P.nz, NP * NP * NP, P.gamma, frozen);
    if (P.part) exchange(s, frozen, hb_(2), hb_(3));
  }
  void launch_phi_apply(cudaStream_t s, PhiState* st, double* base, double* partials, const BArgs& b, int stage = 1) override {
    if (P.part) {  // halo planes of the slot this cycle applies the operator to
      launch_pack_slot(s, st, base, plane, (long long)(P.nz - 1) * plane, hb_(4), hb_(5));
      comm->halo(hb_(4), hb_(5), hb_(0), hb_(1), plane, s);
    }
    if constexpr (E3March<NP>::OK) {
      if (use_march) {
        if constexpr (kDotFits) {
          if (dots_on() && stage == 1) {
            using SD = E3March<NP, true>;
            k_e3_phi_march<NP, true><<<dots_grid, SD::THREADS, SD::SMEM, s>>>(params(frozen), st, base, partials, b);
            return;
          }
        }
        if constexpr (kFwOk) {
          if (use_fw) {
            k_e3_phi_march_fw<NP, 0, false><<<march_grid, E3MarchFW<NP>::THREADS, E3MarchFW<NP>::SMEM, s>>>(
                params(frozen), st, base, partials, b, nullptr, nullptr, nullptr, nullptr);
            return;
          }
        }
        k_e3_phi_march<NP, false><<<march_grid, E3March<NP>::THREADS, E3March<NP>::SMEM, s>>>(params(frozen), st,
                                                                                             base, partials, b);
        return;
      }
    }
    k_e3_phi<NP><<<grid, 256, 0, s>>>(params(frozen), st, base, partials, b);
  }
  void launch_apply(cudaStream_t s, int which, const double* x, double* y) override {
    if (P.part) exchange(s, x, hb_(0), hb_(1));
    if constexpr (kFwOk) {
      if (which == 0 && use_march && use_fw && x != y) {  // y = L x through the z-march JVP (the phi cycle's kernel)
        k_e3_phi_march_fw<NP, 0, true><<<march_grid, E3MarchFW<NP>::THREADS, E3MarchFW<NP>::SMEM, s>>>(
            params(frozen), nullptr, nullptr, nullptr, BArgs{}, x, y, nullptr, nullptr);
        return;
      }
      if (which == 2 && use_march && use_fw && rhs_march && x != y) {  // y = R(x)
        k_e3_phi_march_fw<NP, 2, true><<<march_grid, E3MarchFW<NP>::THREADS, E3MarchFW<NP>::SMEM, s>>>(
            params(frozen), nullptr, nullptr, nullptr, BArgs{}, x, y, nullptr, nullptr);
        return;
      }
      if (which == 1 && use_march && use_fw && rhs_march && x != y) {  // y = N(x) = R(x) - L x
        k_e3_phi_march_fw<NP, 1, true><<<march_grid, E3MarchFW<NP>::THREADS, E3MarchFW<NP>::SMEM, s>>>(
            params(frozen), nullptr, nullptr, nullptr, BArgs{}, x, y, nullptr, nullptr);
        return;
      }
    }
    k_e3_apply<NP><<<grid, 256, 0, s>>>(params(frozen), which, x, y, nullptr, nullptr);
  }
  void launch_residual(cudaStream_t s, const double* u, double* r, PhiState* st, double*) override {
    if (P.part) exchange(s, u, hb_(0), hb_(1));
    bool done = false;
    if constexpr (kFwOk) {
      if (use_march && use_fw && rhs_march && u != r) {
        k_e3_phi_march_fw<NP, 2, true><<<march_grid, E3MarchFW<NP>::THREADS, E3MarchFW<NP>::SMEM, s>>>(
            params(nullptr), nullptr, nullptr, nullptr, BArgs{}, u, r, st, frozen);
        done = true;
      }
    }
    if (!done) k_e3_apply<NP><<<grid, 256, 0, s>>>(params(nullptr), 2, u, r, st, frozen);
    if (P.part) exchange(s, frozen, hb_(2), hb_(3));  // frozen halo for this step's JVPs
  }
};

}  // namespace

std::unique_ptr<OpDevice> make_euler3d(const expdg_op_desc& d) {
  switch (d.order + 1) {
    case 2: return std::make_unique<Euler3D<2>>(d);
    case 3: return std::make_unique<Euler3D<3>>(d);
    case 4: return std::make_unique<Euler3D<4>>(d);
    case 5: return std::make_unique<Euler3D<5>>(d);  // element-tile kernels (2 / 1 elements per CTA)
    case 6: return std::make_unique<Euler3D<6>>(d);
  }
  throw std::invalid_argument("euler3d: device orders are 1..5");
}

}  // namespace expdg
