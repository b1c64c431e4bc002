// Fused single-CTA phi engine for small problems (C1: n = 2560 DOF).
//
// At small n every engine cycle of the multi-kernel engine (operator apply, three
// CGS2 passes, combine, controller) is launch- and latency-bound: ~6 kernels and
// their grid reductions per Krylov column for a few KB of data.  This engine runs
// a whole phi_combination call inside ONE kernel of one 1024-thread CTA: the
// controller state (PhiState incl. the Hessenberg rows in use) lives in shared
// memory for the whole call, the Krylov basis stays in L2, reductions are block
// reductions in a fixed order, and the controller is the same device code as the
// multi-kernel engine (ctl_body).  Same algorithm (CGS2 / IOP windows, the
// reference's accept / grow / halve rules), so the parity bar is unchanged.
#pragma once

#include "burgers_common.cuh"

namespace expdg {

constexpr int kFusedThreads = 512;
constexpr long long kFusedMaxN = 1LL << 15;  // larger problems: the multi-CTA engine is faster

// Element-local operator applies for the fused engine (x = slot j scaled by xs).
template <int NP>
struct B1FusedElem {
  static constexpr int kNP = NP;
  burgers::B1P<NP> P;
  __device__ __forceinline__ void load(const double* v, double s, long long le, double* out) const {
    // single rank (eoff = 0, nel = ne): zero Dirichlet data or periodic wrap
    int w = (int)le;
    if (w < 0 || w >= P.nel) {
      if (!P.periodic) {
#pragma unroll
        for (int i = 0; i < NP; ++i) out[i] = 0.0;
        return;
      }
      w = w < 0 ? w + P.nel : w - P.nel;
    }
#pragma unroll
    for (int i = 0; i < NP; ++i) out[i] = v[w * NP + i] * s;
  }
  __device__ __forceinline__ void apply(int e, const double* x, double xs, double* out) const {
    double xl[NP], xc[NP], xr[NP], ul[NP], uc[NP], ur[NP];
    load(x, xs, e - 1, xl);
    load(x, xs, e, xc);
    load(x, xs, e + 1, xr);
    load(P.ut, 1.0, e - 1, ul);
    load(P.ut, 1.0, e, uc);
    load(P.ut, 1.0, e + 1, ur);
    burgers::b1_element<NP>(P, 0, e, xl, xc, xr, ul, uc, ur, out);
  }
  // same with the applied vector and u~ gathered by fx / fu(element, out[NP]) (cluster
  // engine: shared-memory slices, possibly another CTA's); boundary handling as load()
  template <class FX, class FU>
  __device__ __forceinline__ void apply_with(int e, FX&& fx, FU&& fu, double* out) const {
    double xl[NP], xc[NP], xr[NP], ul[NP], uc[NP], ur[NP];
    gather(fx, e - 1, xl);
    gather(fx, e, xc);
    gather(fx, e + 1, xr);
    gather(fu, e - 1, ul);
    gather(fu, e, uc);
    gather(fu, e + 1, ur);
    burgers::b1_element<NP>(P, 0, e, xl, xc, xr, ul, uc, ur, out);
  }
  template <class FX>
  __device__ __forceinline__ void gather(FX&& fx, int le, double* out) const {
    int w = le;
    if (w < 0 || w >= P.nel) {
      if (!P.periodic) {
#pragma unroll
        for (int i = 0; i < NP; ++i) out[i] = 0.0;
        return;
      }
      w = w < 0 ? w + P.nel : w - P.nel;
    }
    fx(w, out);
  }
  __device__ __forceinline__ int elements() const { return P.nel; }
};

template <int NP, int NQ>
struct B1OIFusedElem {
  static constexpr int kNP = NP;
  burgers::B1OP<NP, NQ> P;
  __device__ __forceinline__ void load(const double* v, double s, long long le, double* out) const {
    // single rank (eoff = 0, nel = ne): zero Dirichlet data or periodic wrap
    int w = (int)le;
    if (w < 0 || w >= P.nel) {
      if (!P.periodic) {
#pragma unroll
        for (int i = 0; i < NP; ++i) out[i] = 0.0;
        return;
      }
      w = w < 0 ? w + P.nel : w - P.nel;
    }
#pragma unroll
    for (int i = 0; i < NP; ++i) out[i] = v[w * NP + i] * s;
  }
  __device__ __forceinline__ void apply(int e, const double* x, double xs, double* out) const {
    double xll[NP], xl[NP], xc[NP], xr[NP], xrr[NP], ul[NP], uc[NP], ur[NP];
    load(x, xs, e - 2, xll);
    load(x, xs, e - 1, xl);
    load(x, xs, e, xc);
    load(x, xs, e + 1, xr);
    load(x, xs, e + 2, xrr);
    load(P.ut, 1.0, e - 1, ul);
    load(P.ut, 1.0, e, uc);
    load(P.ut, 1.0, e + 1, ur);
    burgers::b1oi_element<NP, NQ>(P, 0, e, xll, xl, xc, xr, xrr, ul, uc, ur, out);
  }
  template <class FX, class FU>
  __device__ __forceinline__ void apply_with(int e, FX&& fx, FU&& fu, double* out) const {
    double xll[NP], xl[NP], xc[NP], xr[NP], xrr[NP], ul[NP], uc[NP], ur[NP];
    gather(fx, e - 2, xll);
    gather(fx, e - 1, xl);
    gather(fx, e, xc);
    gather(fx, e + 1, xr);
    gather(fx, e + 2, xrr);
    gather(fu, e - 1, ul);
    gather(fu, e, uc);
    gather(fu, e + 1, ur);
    burgers::b1oi_element<NP, NQ>(P, 0, e, xll, xl, xc, xr, xrr, ul, uc, ur, out);
  }
  template <class FX>
  __device__ __forceinline__ void gather(FX&& fx, int le, double* out) const {
    int w = le;
    if (w < 0 || w >= P.nel) {
      if (!P.periodic) {
#pragma unroll
        for (int i = 0; i < NP; ++i) out[i] = 0.0;
        return;
      }
      w = w < 0 ? w + P.nel : w - P.nel;
    }
    fx(w, out);
  }
  __device__ __forceinline__ int elements() const { return P.nel; }
};

template <class EL>
void launch_phi_fused(cudaStream_t s, Engine& e, const EL& el, const BArgs& b);

}  // namespace expdg
