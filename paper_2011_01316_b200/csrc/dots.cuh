// Dot warps of the fused JVP + DCGS2-dots sweeps (ops_euler2d.cu strip, ops_euler3d.cu
// z-march): the pass-1 dots of k_ts2<TS2_DOTS> (dcgs.cu) taken against row / plane tiles of
// V_0..V_{j-1} streamed through a shared-memory ring.  S provides TILE (doubles per
// tile), ND (dot warps) and VS (ring stages).
#pragma once

#include "krylov.cuh"

namespace expdg {

// Dot warps of the DOT sweep.  The two dot warps split every row tile by 32-double2
// blocks (warp h takes the double2 elements 64 m + 32 h + lane, conflict-free and
// with immediate smem offsets).  The V_i tiles are consumed in quads (then a pair, a single), the
// four per-lane sums of a pair reduced across the warp by one butterfly (6 64-bit
// shuffles) and accumulated in shared memory, s_acc[h][2 i + {0: <V_i,u>, 1: <V_i,w>}]
// (i = j: the candidate u itself).
__device__ __forceinline__ void dots_bfly_add(double* acc, int lane, int ia, int ib, double xa, double ya,
                                              double xb, double yb) {
  // lanes [0,8) <V_ia,u>, [8,16) <V_ia,w>, [16,24) <V_ib,u>, [24,32) <V_ib,w>
  const bool b4 = lane & 16, b3 = lane & 8;
  const double a0 = (b4 ? xb : xa) + __shfl_xor_sync(0xffffffffu, b4 ? xa : xb, 16);
  const double a1 = (b4 ? yb : ya) + __shfl_xor_sync(0xffffffffu, b4 ? ya : yb, 16);
  double t = (b3 ? a1 : a0) + __shfl_xor_sync(0xffffffffu, b3 ? a0 : a1, 8);
  t += __shfl_xor_sync(0xffffffffu, t, 4);
  t += __shfl_xor_sync(0xffffffffu, t, 2);
  t += __shfl_xor_sync(0xffffffffu, t, 1);
  if ((lane & 7) == 0) {
    const int which = lane >> 3;
    const int i = which < 2 ? ia : ib;
    if (i >= 0) acc[2 * i + (which & 1)] += t;
  }
}

// Position in an mbarrier ring: stage index and the parity of its current phase.
struct RingPos {
  int s = 0;
  uint32_t ph = 0;
  template <int N>
  __device__ __forceinline__ void next() {
    if (++s == N) {
      s = 0;
      ph ^= 1u;
    }
  }
};

// One row of dots.  FULL: a full-width strip (every element in range except the
// tail of the last block, whose index is clamped); else every index is clamped.
// u and w are read from shared memory next to each V tile (no register cache:
// 16 accumulator chains per quad stay in flight); a clamped lane re-reads a valid
// element against zero u, w.
template <class S, bool FULL>
__device__ __forceinline__ void dots_row(const double2* U2, const double2* W2, const double* vring, uint64_t* vfull,
                                         uint64_t* vempty, RingPos& vp, int j, int cnt2, int lane, int h,
                                         double* acc, int mode) {
  constexpr int T2 = S::TILE / 2;          // double2 per row tile
  constexpr int PER = (T2 + 63) / 64;      // blocks of 64 double2 (32 per dot warp)
  const int e0 = 32 * h + lane;
  auto eidx = [&](int m) {
    const bool in_range = FULL && 64 * m + 64 <= T2;  // compile-time per unrolled m
    return in_range ? e0 + 64 * m : min(e0 + 64 * m, cnt2 - 1);
  };
  auto valid = [&](int m) { return (FULL && 64 * m + 64 <= T2) || e0 + 64 * m < cnt2; };
  auto ld_uw = [&](int m, double2& u, double2& w) {
    const bool v = valid(m);
    const int e = eidx(m);
    u = v ? U2[e] : make_double2(0.0, 0.0);
    w = v ? W2[e] : make_double2(0.0, 0.0);
  };
  auto take = [&]() {
    const int s = vp.s;
    mbar_wait(&vfull[s], vp.ph);
    vp.next<S::VS>();
    return s;
  };
  auto tile = [&](int s) { return reinterpret_cast<const double2*>(vring + (size_t)s * S::TILE); };
  if (mode & 1) {  // diagnostics: the V stream without the arithmetic
    for (int i = 0; i < j; ++i) {
      const int s = take();
      __syncwarp();
      if (lane == 0) mbar_arrive(&vempty[s]);
    }
    return;
  }
  int i0 = 0;
  for (; !(mode & 2) && i0 + 3 < j; i0 += 4) {  // quads: 16 independent FMA chains, two butterflies
    const int sa = take(), sb = take(), sc = take(), sd = take();
    const double2 *A = tile(sa), *B = tile(sb), *C = tile(sc), *D = tile(sd);
    double xa0 = 0.0, xa1 = 0.0, ya0 = 0.0, ya1 = 0.0, xb0 = 0.0, xb1 = 0.0, yb0 = 0.0, yb1 = 0.0;
    double xc0 = 0.0, xc1 = 0.0, yc0 = 0.0, yc1 = 0.0, xd0 = 0.0, xd1 = 0.0, yd0 = 0.0, yd1 = 0.0;
#pragma unroll
    for (int m = 0; m < PER; ++m) {
      const int e = eidx(m);
      double2 u, w;
      ld_uw(m, u, w);
      const double2 ta = A[e], tb = B[e], tc = C[e], td = D[e];
      xa0 = fma(ta.x, u.x, xa0);
      xb0 = fma(tb.x, u.x, xb0);
      xc0 = fma(tc.x, u.x, xc0);
      xd0 = fma(td.x, u.x, xd0);
      ya0 = fma(ta.x, w.x, ya0);
      yb0 = fma(tb.x, w.x, yb0);
      yc0 = fma(tc.x, w.x, yc0);
      yd0 = fma(td.x, w.x, yd0);
      xa1 = fma(ta.y, u.y, xa1);
      xb1 = fma(tb.y, u.y, xb1);
      xc1 = fma(tc.y, u.y, xc1);
      xd1 = fma(td.y, u.y, xd1);
      ya1 = fma(ta.y, w.y, ya1);
      yb1 = fma(tb.y, w.y, yb1);
      yc1 = fma(tc.y, w.y, yc1);
      yd1 = fma(td.y, w.y, yd1);
    }
    __syncwarp();
    if (lane == 0) {
      mbar_arrive(&vempty[sa]);
      mbar_arrive(&vempty[sb]);
      mbar_arrive(&vempty[sc]);
      mbar_arrive(&vempty[sd]);
    }
    dots_bfly_add(acc, lane, i0, i0 + 1, xa0 + xa1, ya0 + ya1, xb0 + xb1, yb0 + yb1);
    dots_bfly_add(acc, lane, i0 + 2, i0 + 3, xc0 + xc1, yc0 + yc1, xd0 + xd1, yd0 + yd1);
  }
  // the remaining 0..3 V tiles, then the candidate u itself (i = j), two per butterfly
  for (; i0 <= j; i0 += 2) {
    const int sa = i0 < j ? take() : -1, sb = i0 + 1 < j ? take() : -1;
    const double2* A = tile(max(sa, 0));
    const double2* B = tile(max(sb, 0));
    double xa0 = 0.0, xa1 = 0.0, ya0 = 0.0, ya1 = 0.0, xb0 = 0.0, xb1 = 0.0, yb0 = 0.0, yb1 = 0.0;
#pragma unroll
    for (int m = 0; m < PER; ++m) {
      const int e = eidx(m);
      double2 u, w;
      ld_uw(m, u, w);
      const double2 ta = sa >= 0 ? A[e] : u;  // i0 == j: the candidate
      const double2 tb = sb >= 0 ? B[e] : (i0 + 1 == j ? u : make_double2(0.0, 0.0));
      xa0 = fma(ta.x, u.x, xa0);
      xb0 = fma(tb.x, u.x, xb0);
      ya0 = fma(ta.x, w.x, ya0);
      yb0 = fma(tb.x, w.x, yb0);
      xa1 = fma(ta.y, u.y, xa1);
      xb1 = fma(tb.y, u.y, xb1);
      ya1 = fma(ta.y, w.y, ya1);
      yb1 = fma(tb.y, w.y, yb1);
    }
    __syncwarp();
    if (lane == 0) {
      if (sa >= 0) mbar_arrive(&vempty[sa]);
      if (sb >= 0) mbar_arrive(&vempty[sb]);
    }
    dots_bfly_add(acc, lane, i0, i0 + 1 <= j ? i0 + 1 : -1, xa0 + xa1, ya0 + ya1, xb0 + xb1, yb0 + yb1);
  }
}

}  // namespace expdg
