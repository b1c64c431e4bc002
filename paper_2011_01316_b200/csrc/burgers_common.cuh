// Shared device code of the LDG Burgers operators: the 1D element kernel of
// proj/src/burgers.cpp (gradient :105-130, linear :146-180, nonlinear :182-215,
// full rhs :217-265) for one element line, used by the 1D operator and, along
// every x- and y-line, by the 2D tensor-product extension.
#pragma once

#include "krylov.cuh"

namespace expdg {
namespace burgers {

template <int NP>
struct B1P {
  int ne;
  int periodic;
  double a, b;
  double kappa, sigma;
  int entropy, sigma_adaptive;
  double w[NP];
  double G[NP * NP];   // grad_vol(i,j) = w_i D(i,j)      (proj/src/burgers.cpp:49)
  double Lv[NP * NP];  // lift_vol(i,j) = D(j,i) w_j      (proj/src/burgers.cpp:50)
  const double* ut;
  const double* src;   // weak source (proj/src/burgers.cpp:80-92), may be null
  const double* hh;    // per global element: h_e, 2 / h_e (host-computed from the breakpoints)
  double iw[NP];       // 1 / w_i
  long long n;  // slab partition: this rank owns elements [eoff, eoff + nel) of the
  // ne-element mesh; the H elements either side come from the halo buffers
  int nel;
  long long eoff;
  int part;
  const double* gx_lo;
  const double* gx_hi;
  const double* gt_lo;
  const double* gt_hi;
};

// Stages local elements [e0 - H, e0 + E + H) of x (scaled by xs) and u~ into shared
// memory: zero-Dirichlet ghosts outside the global mesh, periodic wrap when the mesh is
// whole, the neighbouring rank's halo elements when it is slab-partitioned.
template <int NP, int H, class PP>
__device__ __forceinline__ void stage_elements(const PP& P, long long e0, int E, const double* x, double xs,
                                               bool want_ut, double* sx, double* su) {
  const int cnt = (E + 2 * H) * NP;
  for (int idx = threadIdx.x; idx < cnt; idx += blockDim.x) {
    const long long le = e0 - H + idx / NP;
    const int node = idx % NP;
    const long long gg = P.eoff + le;
    double xv = 0.0, uv = 0.0;
    if ((gg < 0 || gg >= P.ne) && !P.periodic) {
      // outside the interval: zero Dirichlet data
    } else if (le < 0 || le >= P.nel) {
      if (P.part) {
        const size_t hi = le < 0 ? (size_t)((le + H) * NP + node) : (size_t)((le - P.nel) * NP + node);
        xv = (le < 0 ? P.gx_lo : P.gx_hi)[hi] * xs;
        if (want_ut) uv = (le < 0 ? P.gt_lo : P.gt_hi)[hi];
      } else {
        const long long w = ((le % P.nel) + P.nel) % P.nel;
        xv = x[w * NP + node] * xs;
        if (want_ut) uv = P.ut[w * NP + node];
      }
    } else {
      xv = x[le * NP + node] * xs;
      if (want_ut) uv = P.ut[le * NP + node];
    }
    sx[idx] = xv;
    su[idx] = uv;
  }
}

// x_e of the uniform breakpoints (proj/src/mesh.cpp:11-16)
__device__ __forceinline__ double b1_break(double a, double b, int i, int ne) {
  return i == ne ? b : a + (b - a) * i / ne;
}

template <int NP>
__device__ __forceinline__ double b1_face_flux(const B1P<NP>& P, int mode, double um, double up, double utm,
                                               double utp, double qstar, double h) {
  const double jump = um - up;  // normal = +1 on every face this helper sees
  double lin = 0.0;
  if (mode != 2) {
    const double diss = 0.5 * fmax(fabs(utm), fabs(utp));
    lin = 0.5 * (utm * um + utp * up) + diss * jump;
  }
  if (mode == 0) return P.kappa * qstar - lin;
  double nl;
  if (!P.entropy) {
    const double ahs = 0.25 * (um * um + up * up);
    nl = ahs + 0.5 * fmax(fabs(um), fabs(up)) * jump;
  } else {
    double soh;
    if (mode == 1) {
      const double sig = P.sigma_adaptive ? P.kappa / 100.0 + h * fmax(fabs(utm), fabs(utp)) : P.sigma;
      soh = sig * (1.0 / h);
    } else {
      soh = P.sigma_adaptive ? P.kappa / (100.0 * h) + fmax(fabs(um), fabs(up)) : P.sigma / h;
    }
    const double ahs = 0.25 * (um * um + up * up);
    const double avg = 0.5 * (um + up);
    nl = (ahs + avg * avg) / 3.0 + soh * jump;
  }
  if (mode == 1) return lin - nl;
  return P.kappa * qstar - nl;
}

// Element e of the operator; x*/u* point at NP values of the left / centre /
// right elements (left/right ignored when the face is a Dirichlet boundary).
template <int NP>
__device__ __forceinline__ void b1_element(const B1P<NP>& P, int mode, int e, const double* xL,
                                           const double* xC, const double* xR, const double* uL,
                                           const double* uC, const double* uR, double* out) {
  constexpr int N = NP - 1;
  const bool hasL = P.periodic || e > 0;
  const bool hasR = P.periodic || e < P.ne - 1;
  const int eL = e == 0 ? P.ne - 1 : e - 1;
  const int eR = e == P.ne - 1 ? 0 : e + 1;
  // element widths of the breakpoints (proj/src/mesh.cpp:11-16) and 2 / h from the host table
  const double hC = P.hh[2 * e], hL = P.hh[2 * eL], hR = P.hh[2 * eR];
  const double cC = P.hh[2 * e + 1];
  double q[NP], qLN = 0.0, qR0 = 0.0;
  if (mode != 1) {
    // LDG gradient (proj/src/burgers.cpp:105-130)
    double r[NP];
#pragma unroll
    for (int i = 0; i < NP; ++i) {
      double s = 0.0;
#pragma unroll
      for (int j = 0; j < NP; ++j) s = fma(P.G[i * NP + j], xC[j], s);
      r[i] = s;
    }
    if (hasL) {
      const double us = 0.5 * (xL[N] + xC[0]);
      r[0] -= (us - xC[0]);
      double s = 0.0;
#pragma unroll
      for (int j = 0; j < NP; ++j) s = fma(P.G[N * NP + j], xL[j], s);
      s += (us - xL[N]);
      qLN = P.hh[2 * eL + 1] * (s * P.iw[N]);
    } else {
      r[0] += -1.0 * (0.0 - xC[0]);
    }
    if (hasR) {
      const double us = 0.5 * (xC[N] + xR[0]);
      r[N] += (us - xC[N]);
      double s = 0.0;
#pragma unroll
      for (int j = 0; j < NP; ++j) s = fma(P.G[j], xR[j], s);
      s -= (us - xR[0]);
      qR0 = P.hh[2 * eR + 1] * (s * P.iw[0]);
    } else {
      r[N] += (0.0 - xC[N]);
    }
#pragma unroll
    for (int i = 0; i < NP; ++i) q[i] = cC * (r[i] * P.iw[i]);
  }
  // volume: gq = kappa q - u~ x | u~ x - x^2/2 | kappa q - x^2/2 ; r = -lift gq
  double gq[NP];
#pragma unroll
  for (int p = 0; p < NP; ++p) {
    const double x = xC[p];
    if (mode == 0) gq[p] = fma(-uC[p], x, P.kappa * q[p]);
    else if (mode == 1) gq[p] = uC[p] * x - 0.5 * (x * x);
    else gq[p] = P.kappa * q[p] - 0.5 * (x * x);
  }
  double r[NP];
#pragma unroll
  for (int i = 0; i < NP; ++i) {
    double s = 0.0;
#pragma unroll
    for (int p = 0; p < NP; ++p) s = fma(P.Lv[i * NP + p], gq[p], s);
    r[i] = -s;
  }
  if (mode != 0 && P.src) {
#pragma unroll
    for (int i = 0; i < NP; ++i) r[i] += P.src[(long long)(e - P.eoff) * NP + i];
  }
  // faces (proj/src/burgers.cpp:159-173)
  if (hasL) {
    const double f = b1_face_flux(P, mode, xL[N], xC[0], mode == 2 ? 0.0 : uL[N], mode == 2 ? 0.0 : uC[0],
                                  0.5 * (qLN + q[0]), hL);
    r[0] -= f;
  } else {
    // boundary face: owner e, node 0, normal -1, ghost 0; q** one-sided
    const double um = xC[0];
    const double jump = -um;
    double f;
    const double utm = mode == 2 ? 0.0 : uC[0];
    const double lin = 0.5 * (utm * um + 0.0) + 0.5 * fmax(fabs(utm), 0.0) * jump;
    if (mode == 0) {
      f = P.kappa * q[0] - lin;
    } else {
      double nl;
      if (!P.entropy) {
        nl = 0.25 * (um * um) + 0.5 * fabs(um) * jump;
      } else {
        double soh;
        if (mode == 1) soh = (P.sigma_adaptive ? P.kappa / 100.0 + hC * fabs(utm) : P.sigma) * (1.0 / hC);
        else soh = P.sigma_adaptive ? P.kappa / (100.0 * hC) + fabs(um) : P.sigma / hC;
        const double avg = 0.5 * um;
        nl = (0.25 * (um * um) + avg * avg) / 3.0 + soh * jump;
      }
      f = mode == 1 ? lin - nl : P.kappa * q[0] - nl;
    }
    r[0] += -1.0 * f;
  }
  if (hasR) {
    const double f = b1_face_flux(P, mode, xC[N], xR[0], mode == 2 ? 0.0 : uC[N], mode == 2 ? 0.0 : uR[0],
                                  0.5 * (q[N] + qR0), hC);
    r[N] += f;
  } else {
    const double um = xC[N];
    const double jump = um;
    const double utm = mode == 2 ? 0.0 : uC[N];
    const double lin = 0.5 * (utm * um + 0.0) + 0.5 * fmax(fabs(utm), 0.0) * jump;
    double f;
    if (mode == 0) {
      f = P.kappa * q[N] - lin;
    } else {
      double nl;
      if (!P.entropy) {
        nl = 0.25 * (um * um) + 0.5 * fabs(um) * jump;
      } else {
        double soh;
        if (mode == 1) soh = (P.sigma_adaptive ? P.kappa / 100.0 + hC * fabs(utm) : P.sigma) * (1.0 / hC);
        else soh = P.sigma_adaptive ? P.kappa / (100.0 * hC) + fabs(um) : P.sigma / hC;
        const double avg = 0.5 * um;
        nl = (0.25 * (um * um) + avg * avg) / 3.0 + soh * jump;
      }
      f = mode == 1 ? lin - nl : P.kappa * q[N] - nl;
    }
    r[N] += f;
  }
#pragma unroll
  for (int i = 0; i < NP; ++i) out[i] = cC * (r[i] * P.iw[i]);
}

}  // namespace burgers
}  // namespace expdg

namespace expdg {
namespace burgers {

// Over-integrated variant (BurgersConfig::over_integrate, proj/src/burgers.cpp:39-51):
// Gauss rule of NQ = (3k+3)/2 points, interp I (NQ x NP), consistent mass M (dense,
// applied as M^-1, the reference's LDLT solve), grad_vol = I^T W I D, lift_vol = (I D)^T W.
template <int NP, int NQ>
struct B1OP {
  int ne;
  int periodic;
  double a, b;
  double kappa, sigma;
  int entropy, sigma_adaptive;
  double G[NP * NP];    // grad_vol
  double Lv[NP * NQ];   // lift_vol (NP x NQ)
  double I[NQ * NP];    // interp
  double Mi[NP * NP];   // M^-1
  const double* ut;
  const double* src;    // weak source (proj/src/burgers.cpp:80-92), may be null
  const double* hh;     // per global element: h_e, 2 / h_e
  long long n;
  // slab partition: this rank owns elements [eoff, eoff + nel) of the
  // ne-element mesh; the H elements either side come from the halo buffers
  int nel;
  long long eoff;
  int part;
  const double* gx_lo;
  const double* gx_hi;
  const double* gt_lo;
  const double* gt_hi;
};

// r of one element's LDG gradient system before the mass solve (proj/src/burgers.cpp:105-123):
// xL2/xR2 are the end values of the elements two away (needed for the face terms of the
// neighbours), has* flags as in b1_element.
template <int NP, int NQ>
__device__ __forceinline__ void b1oi_grad_r(const B1OP<NP, NQ>& P, const double* xm, const double* xc,
                                            const double* xp, bool hasL, bool hasR, double* r) {
  constexpr int N = NP - 1;
#pragma unroll
  for (int i = 0; i < NP; ++i) {
    double s = 0.0;
#pragma unroll
    for (int j = 0; j < NP; ++j) s = fma(P.G[i * NP + j], xc[j], s);
    r[i] = s;
  }
  if (hasL) r[0] -= (0.5 * (xm[N] + xc[0]) - xc[0]);
  else r[0] += -1.0 * (0.0 - xc[0]);
  if (hasR) r[N] += (0.5 * (xc[N] + xp[0]) - xc[N]);
  else r[N] += (0.0 - xc[N]);
}

template <int NP, int NQ>
__device__ __forceinline__ void b1oi_minv(const B1OP<NP, NQ>& P, double c, const double* r, double* q) {
#pragma unroll
  for (int i = 0; i < NP; ++i) {
    double s = 0.0;
#pragma unroll
    for (int j = 0; j < NP; ++j) s = fma(P.Mi[i * NP + j], r[j], s);
    q[i] = c * s;
  }
}

// Element e; x*/u* point at NP values of elements e-2 .. e+2 (only the end values of
// the outer two are used).
template <int NP, int NQ>
__device__ __forceinline__ void b1oi_element(const B1OP<NP, NQ>& P, int mode, int e, const double* xLL,
                                             const double* xL, const double* xC, const double* xR,
                                             const double* xRR, const double* uL, const double* uC,
                                             const double* uR, double* out) {
  constexpr int N = NP - 1;
  const int ne = P.ne;
  const bool hasL = P.periodic || e > 0;
  const bool hasR = P.periodic || e < ne - 1;
  const int eL = e == 0 ? ne - 1 : e - 1;
  const int eR = e == ne - 1 ? 0 : e + 1;
  const double hC = P.hh[2 * e], hL = P.hh[2 * eL], hR = P.hh[2 * eR];
  double q[NP], qLN = 0.0, qR0 = 0.0;
  if (mode != 1) {
    double r[NP], t[NP];
    b1oi_grad_r(P, xL, xC, xR, hasL, hasR, r);
    b1oi_minv(P, P.hh[2 * e + 1], r, q);
    if (hasL) {
      const bool hLL = P.periodic || eL > 0;
      b1oi_grad_r(P, xLL, xL, xC, hLL, true, r);
      b1oi_minv(P, P.hh[2 * eL + 1], r, t);
      qLN = t[N];
    }
    if (hasR) {
      const bool hRR = P.periodic || eR < ne - 1;
      b1oi_grad_r(P, xC, xR, xRR, true, hRR, r);
      b1oi_minv(P, P.hh[2 * eR + 1], r, t);
      qR0 = t[0];
    }
  }
  // volume at the Gauss points (proj/src/burgers.cpp:152-157, :187-193, :223-230)
  double r[NP];
#pragma unroll
  for (int i = 0; i < NP; ++i) r[i] = 0.0;
#pragma unroll
  for (int p = 0; p < NQ; ++p) {
    double xq = 0.0, uq = 0.0, qq = 0.0;
#pragma unroll
    for (int j = 0; j < NP; ++j) {
      xq = fma(P.I[p * NP + j], xC[j], xq);
      if (mode != 2) uq = fma(P.I[p * NP + j], uC[j], uq);
      if (mode != 1) qq = fma(P.I[p * NP + j], q[j], qq);
    }
    double g;
    if (mode == 0) g = fma(-uq, xq, P.kappa * qq);
    else if (mode == 1) g = uq * xq - 0.5 * (xq * xq);
    else g = P.kappa * qq - 0.5 * (xq * xq);
#pragma unroll
    for (int i = 0; i < NP; ++i) r[i] = fma(P.Lv[i * NQ + p], g, r[i]);
  }
#pragma unroll
  for (int i = 0; i < NP; ++i) r[i] = -r[i];
  if (mode != 0 && P.src) {
#pragma unroll
    for (int i = 0; i < NP; ++i) r[i] += P.src[(long long)(e - P.eoff) * NP + i];
  }
  // faces: identical to the collocated operator (traces are nodal end values)
  B1P<NP> F{};
  F.kappa = P.kappa;
  F.sigma = P.sigma;
  F.entropy = P.entropy;
  F.sigma_adaptive = P.sigma_adaptive;
  if (hasL) {
    r[0] -= b1_face_flux(F, mode, xL[N], xC[0], mode == 2 ? 0.0 : uL[N], mode == 2 ? 0.0 : uC[0],
                         0.5 * (qLN + q[0]), hL);
  } else {
    const double um = xC[0], jump = -um;
    const double utm = mode == 2 ? 0.0 : uC[0];
    const double lin = 0.5 * (utm * um + 0.0) + 0.5 * fmax(fabs(utm), 0.0) * jump;
    double f;
    if (mode == 0) {
      f = P.kappa * q[0] - lin;
    } else {
      double nl;
      if (!P.entropy) {
        nl = 0.25 * (um * um) + 0.5 * fabs(um) * jump;
      } else {
        double soh;
        if (mode == 1) soh = (P.sigma_adaptive ? P.kappa / 100.0 + hC * fabs(utm) : P.sigma) * (1.0 / hC);
        else soh = P.sigma_adaptive ? P.kappa / (100.0 * hC) + fabs(um) : P.sigma / hC;
        const double avg = 0.5 * um;
        nl = (0.25 * (um * um) + avg * avg) / 3.0 + soh * jump;
      }
      f = mode == 1 ? lin - nl : P.kappa * q[0] - nl;
    }
    r[0] += -1.0 * f;
  }
  if (hasR) {
    r[N] += b1_face_flux(F, mode, xC[N], xR[0], mode == 2 ? 0.0 : uC[N], mode == 2 ? 0.0 : uR[0],
                         0.5 * (q[N] + qR0), hC);
  } else {
    const double um = xC[N], jump = um;
    const double utm = mode == 2 ? 0.0 : uC[N];
    const double lin = 0.5 * (utm * um + 0.0) + 0.5 * fmax(fabs(utm), 0.0) * jump;
    double f;
    if (mode == 0) {
      f = P.kappa * q[N] - lin;
    } else {
      double nl;
      if (!P.entropy) {
        nl = 0.25 * (um * um) + 0.5 * fabs(um) * jump;
      } else {
        double soh;
        if (mode == 1) soh = (P.sigma_adaptive ? P.kappa / 100.0 + hC * fabs(utm) : P.sigma) * (1.0 / hC);
        else soh = P.sigma_adaptive ? P.kappa / (100.0 * hC) + fabs(um) : P.sigma / hC;
        const double avg = 0.5 * um;
        nl = (0.25 * (um * um) + avg * avg) / 3.0 + soh * jump;
      }
      f = mode == 1 ? lin - nl : P.kappa * q[N] - nl;
    }
    r[N] += f;
  }
  b1oi_minv(P, P.hh[2 * e + 1], r, out);
}

}  // namespace burgers
}  // namespace expdg
