// 2D viscous Burgers (config C3, an extension: BurgersOperator is 1D only,
// proj/src/burgers.cpp:24-25).  Collocated tensor-product LDG on a Cartesian
// quad mesh = the reference 1D LDG operator applied along every element x-line
// plus along every y-line (see oracle/src/burgers.cpp, Burgers2DOperator), so a
// y-invariant field reproduces the 1D operator exactly.
//
// CTA tile of floor(256 / NP) elements; phase 1: one thread per (element, row)
// runs the 1D element kernel along x; phase 2: one thread per (element, column)
// along y and adds.  Line neighbours come from L2.
#include <algorithm>
#include <cstdlib>

#include "burgers_common.cuh"
#include "dots.cuh"

namespace expdg {

namespace {

using namespace burgers;

template <int NP>
struct B2Tile {
  static constexpr int TE = 256 / NP;
};

// line of NP values: x-line (row j) or y-line (column i) of element e
__device__ __forceinline__ void gather(const double* v, double s, long long e, int NP_, int line, bool xdir,
                                       double* out) {
  const int NN = NP_ * NP_;
  for (int t = 0; t < NP_; ++t) out[t] = v[e * NN + (xdir ? line * NP_ + t : t * NP_ + line)] * s;
}

template <int NP>
__device__ __forceinline__ void b2_tile(const B1P<NP>& Px, const B1P<NP>& Py, int nx, int ny, int mode, long long e0,
                                        int te, const double* x, double xs, double* sout) {
  constexpr int NN = NP * NP;
  const int t = threadIdx.x;
  const int le = t / NP, line = t % NP;
  const bool active = le < te;
  const bool need_ut = mode != 2;
  double xL[NP], xC[NP], xR[NP], uL[NP], uC[NP], uR[NP], out[NP];
  long long e = 0;
  int ie = 0, je = 0;
  if (active) {
    e = e0 + le;
    je = (int)(e / nx);
    ie = (int)(e - (long long)je * nx);
    // x-line (row `line`)
    const long long eW = (long long)je * nx + (ie == 0 ? nx - 1 : ie - 1);
    const long long eE = (long long)je * nx + (ie == nx - 1 ? 0 : ie + 1);
    gather(x, xs, eW, NP, line, true, xL);
    gather(x, xs, e, NP, line, true, xC);
    gather(x, xs, eE, NP, line, true, xR);
    if (need_ut) {
      gather(Px.ut, 1.0, eW, NP, line, true, uL);
      gather(Px.ut, 1.0, e, NP, line, true, uC);
      gather(Px.ut, 1.0, eE, NP, line, true, uR);
    }
    b1_element<NP>(Px, mode, ie, xL, xC, xR, uL, uC, uR, out);
#pragma unroll
    for (int i = 0; i < NP; ++i) sout[le * NN + line * NP + i] = out[i];
  }
  __syncthreads();
  if (active) {
    // y-line (column `line`); a row slab takes rows -1 / ny from the halo rows
    const bool gS = Py.part && je == 0, gN = Py.part && je == ny - 1;
    const long long eS = (long long)(je == 0 ? ny - 1 : je - 1) * nx + ie;
    const long long eN = (long long)(je == ny - 1 ? 0 : je + 1) * nx + ie;
    gather(gS ? Py.gx_lo : x, xs, gS ? ie : eS, NP, line, false, xL);
    gather(x, xs, e, NP, line, false, xC);
    gather(gN ? Py.gx_hi : x, xs, gN ? ie : eN, NP, line, false, xR);
    if (need_ut) {
      gather(gS ? Py.gt_lo : Py.ut, 1.0, gS ? ie : eS, NP, line, false, uL);
      gather(Py.ut, 1.0, e, NP, line, false, uC);
      gather(gN ? Py.gt_hi : Py.ut, 1.0, gN ? ie : eN, NP, line, false, uR);
    }
    b1_element<NP>(Py, mode, (int)Py.eoff + je, xL, xC, xR, uL, uC, uR, out);
#pragma unroll
    for (int j = 0; j < NP; ++j) sout[le * NN + j * NP + line] += out[j];
  }
  __syncthreads();
}

template <int NP>
__global__ void __launch_bounds__(256) k_b2_apply(B1P<NP> Px, B1P<NP> Py, int nx, int ny, int mode,
                                                  const double* __restrict__ x, double* __restrict__ y,
                                                  const PhiState* st) {
  constexpr int NN = NP * NP, TE = B2Tile<NP>::TE;
  __shared__ double sout[TE * NN];
  if (st && st->stopped) return;
  const long long ne = (long long)nx * ny;
  const long long ntiles = (ne + TE - 1) / TE;
  for (long long tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
    const long long e0 = tile * TE;
    const int te = (int)(ne - e0 < TE ? ne - e0 : TE);
    b2_tile<NP>(Px, Py, nx, ny, mode, e0, te, x, 1.0, sout);
    for (int idx = threadIdx.x; idx < te * NN; idx += blockDim.x) y[e0 * NN + idx] = sout[idx];
    __syncthreads();
  }
}

template <int NP>
__global__ void __launch_bounds__(256) k_b2_phi(B1P<NP> Px, B1P<NP> Py, int nx, int ny, PhiState* st, double* base,
                                                double* partials, BArgs b) {
  constexpr int NN = NP * NP, TE = B2Tile<NP>::TE;
  __shared__ double sout[TE * NN];
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
      for (int i = 0; i < kMaxP; ++i) s_xt[i] = (i < b.p) ? xslot[Px.n + i] * s_xs : 0.0;
    }
  }
  __syncthreads();
  if (!s_go) return;
  const double* x = base + (size_t)s_j * s_ld;
  double* y = base + (size_t)(s_j + 1) * s_ld;
  const double xs = s_xs, dt = s_dt;
  const long long ne = (long long)nx * ny;
  const long long ntiles = (ne + TE - 1) / TE;
  double nacc = 0.0;
  for (long long tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
    const long long e0 = tile * TE;
    const int te = (int)(ne - e0 < TE ? ne - e0 : TE);
    b2_tile<NP>(Px, Py, nx, ny, 0, e0, te, x, xs, sout);
    for (int idx = threadIdx.x; idx < te * NN; idx += blockDim.x) {
      const long long g = e0 * NN + idx;
      double v = sout[idx];
      v = aug_tail(b, s_xt, g, v);
      v = dt * v;
      y[g] = v;
      nacc = fma(v, v, nacc);
    }
    __syncthreads();
  }
  // the p-scalar tail is replicated on every rank; rank 0 counts it
  if (blockIdx.x == 0 && threadIdx.x < kTailPad) {
    const int i = threadIdx.x;
    const double v = (i + 1 < b.p) ? dt * s_xt[i + 1] : 0.0;
    y[Px.n + i] = v;
    if (st->tail_here) nacc = fma(v, v, nacc);
  }
  const double tot = block_sum(nacc, s_buf);
  if (threadIdx.x == 0) s_red[0] = tot;
  __syncthreads();
  grid_reduce_last(s_red, 1, partials, kMaxSlots, &st->ticket[4], [&](int, double v) { st->rs().nrmA = v; });
}

// ---------------------------------------------------------------- strip JVP (phi cycle)
// A CTA owns a strip of W = 32 (16 for orders 7, 8) element columns and marches up a contiguous range of
// element rows (the Euler strip kernel's scheme, ops_euler2d.cu): warp CW streams whole
// element rows of x (slot j) and u~ with their E/W halo elements, plus b_1, by
// asynchronous copies into a 4-row shared-memory ring; the consumer threads take row r's
// x-lines (thread per element row-line, neighbours from the ring row's halo elements)
// and y-lines (thread per element column-line, neighbours from ring rows r -+ 1), so
// every byte of x and u~ leaves HBM once per JVP instead of being gathered from L2 by
// three elements in two directions.
// DOT (as the 2D Euler strip sweep, ops_euler2d.cu): the sweep also takes the DCGS2 pass-1
// dots of column j (a = V^T u, b = V^T w with u = slot j, w = the JVP output) — a TMA producer
// warp streams the row tiles of V_0..V_{j-1} into a ring and two dot warps consume them
// (dots.cuh).  Needs full-width strips whose rows are 16-byte aligned (nx % W == 0).
constexpr int kB2DotJ = 44;
#ifndef EXPDG_B2_SPLIT
#define EXPDG_B2_SPLIT 1
#endif

template <int NP, bool DOT = false>
struct B2Strip {
  static constexpr int NN = NP * NP;
  static constexpr int W = NP <= 7 ? 32 : 16;        // elements per strip
  static constexpr int LN = (W * NP + 31) / 32 * 32;  // threads of one line set (one per element line)
  // the plain strip runs the x-lines and the y-lines of a row on separate warps at the same time
  // (two line sets); with the dots, one set does both in turn (the dot warps take the threads)
  static constexpr bool SPLIT = !DOT && EXPDG_B2_SPLIT;
  static constexpr int CONS = (SPLIT ? 2 : 1) * LN;  // consumer threads
  static constexpr int CW = CONS / 32;       // consumer warps
  static constexpr int ROWD = (W + 2) * NN;  // doubles per array per ring row (with halo)
  // DOT: the x row starts one double into its slot when NN is odd, so that its interior
  // (the dots' u) is 16-byte aligned
  static constexpr int XOFF = DOT && (NN & 1) ? 1 : 0;
  static constexpr int BUFD = (XOFF + 2 * ROWD + W * NN + 1) / 2 * 2;  // x + u~ (with halo) + b_1
  static constexpr int NBUF = 4;
  static constexpr int OUT = W * NN;         // one row of x-line or y-line results
  static constexpr int TILE = W * NN;        // doubles of one row of one vector
  static constexpr int ND = DOT ? 2 : 0;     // dot warps (one per tile half)
  static constexpr int JMAX = DOT ? kB2DotJ - 1 : -1;
  static constexpr int THREADS = CONS + 32 + (DOT ? 32 + 32 * ND : 0);
  static constexpr int BASE = NBUF * BUFD + 2 * 2 * OUT;  // ring + double-buffered sX, sY
  static constexpr int SMAX = 232448 / 8 - 384;
  static constexpr int VSF = (SMAX - BASE - 2 * TILE) / TILE;
  static constexpr int VS = DOT ? (VSF > 16 ? 16 : (VSF < 1 ? 1 : VSF)) : 1;
  static constexpr bool FITS = !DOT || (VSF >= 4 && TILE % 2 == 0);
  static constexpr int SMEM = (BASE + (DOT ? 2 * TILE + VS * TILE : 0)) * 8;
};

template <int NP, bool DOT>
__global__ void __launch_bounds__(B2Strip<NP, DOT>::THREADS)
    k_b2_phi_strip(B1P<NP> Px, B1P<NP> Py, int nx, int ny, PhiState* st, double* base, double* partials, BArgs b) {
  using S = B2Strip<NP, DOT>;
  constexpr int NN = S::NN, W = S::W, NBUF = S::NBUF, CW = S::CW;
  extern __shared__ __align__(128) double smem[];
  double* ring = smem;
  double* sout = smem + NBUF * S::BUFD;  // [parity][X | Y][W * NN]
  double* swr = smem + S::BASE;          // DOT: w rows handed to the dot warps
  double* vring = swr + 2 * S::TILE;     // DOT: V row tiles
  __shared__ uint64_t full[NBUF], empty[NBUF];
  __shared__ uint64_t wfull[2], wempty[2], vfull[S::VS], vempty[S::VS];
  __shared__ int s_go, s_j, s_dots;
  __shared__ double s_xs, s_dt, s_xt[kMaxP];
  __shared__ long long s_ld;
  __shared__ double s_buf[S::THREADS / 32];
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
        // algorithmic bytes of this sweep: x, u~, b_1, y plus, with the dots, V_0..V_{j-1}
        st->app_bytes += 8.0 * (double)Px.n * (4.0 + (s_dots ? (double)s_j : 0.0));
        st->app_launches++;
      }
      s_xs = st->scale[s_j];
      s_dt = st->dt;
      s_ld = st->ld;
      const double* xslot = base + (size_t)s_j * st->ld;
      for (int i = 0; i < kMaxP; ++i) s_xt[i] = (i < b.p) ? xslot[Px.n + i] * s_xs : 0.0;
      for (int q = 0; q < NBUF; ++q) {
        mbar_init(&full[q], 32);  // every producer lane's cp.async arrival
        mbar_init(&empty[q], 1 + S::ND);  // the JVP warps + (DOT) every dot warp
      }
      if (DOT) {
        for (int q = 0; q < 2; ++q) {
          mbar_init(&wfull[q], CW);
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
    for (int q = tid; q < 4 * (S::JMAX + 1); q += blockDim.x) s_red[q] = 0.0;
  __syncthreads();
  if (!s_go) return;
  const double* x = base + (size_t)s_j * s_ld;
  double* y = base + (size_t)(s_j + 1) * s_ld;
  const double xs = s_xs, dt = s_dt;
  const bool dots = DOT && s_dots;
  // ring rows the dot warps also read (u) are released by them too; halo rows and,
  // without dots, every row are released by the JVP warps for all 1 + ND arrivals
  const uint32_t rel_row = dots ? 1u : 1u + S::ND, rel_halo = 1u + S::ND;
  const int nstrips = (nx + W - 1) / W;
  const long long rsteps = (long long)nstrips * ny;
  const long long k0 = rsteps * blockIdx.x / gridDim.x, k1 = rsteps * (blockIdx.x + 1) / gridDim.x;
  const double* b1 = (b.p == 1) ? b.b[1] : nullptr;
  double nacc = 0.0;
  auto unit = [&](long long& k, int& ie0, int& w, int& r0, int& r1) {
    const int strip = (int)(k / ny);
    r0 = (int)(k - (long long)strip * ny);
    r1 = (int)min((long long)ny, r0 + (k1 - k));
    k += r1 - r0;
    ie0 = strip * W;
    w = min(W, nx - ie0);
  };

  if (wid == CW) {
    // ---------------- producer warp: x / u~ rows with their E/W halo elements, b_1 rows.
    // Element rows of NP^2 doubles are 8- but not 16-byte aligned, so the rows move by
    // coalesced 8-byte cp.async (one warp) rather than TMA bulk copies; every lane's
    // copies complete an arrival on the row's full barrier.
    long long seq = 0;
    auto copy = [&](double* d, const double* src, int cnt) {
      for (int t = lane; t < cnt; t += 32) cp_async8(d + t, src + t);
    };
    for (long long k = k0; k < k1;) {
      int ie0, w, r0, r1;
      unit(k, ie0, w, r0, r1);
      for (int q = 0; q < r1 - r0 + 2; ++q, ++seq) {
        int row = r0 - 1 + q;
        const double* srcx = x;
        const double* srct = Py.ut;
        if (Py.part && (row < 0 || row >= ny)) {  // halo row of the neighbouring rank
          srcx = row < 0 ? Py.gx_lo : Py.gx_hi;
          srct = row < 0 ? Py.gt_lo : Py.gt_hi;
          row = 0;
        } else {
          row = row < 0 ? row + ny : (row >= ny ? row - ny : row);
        }
        const int sl = (int)(seq % NBUF);
        if (lane == 0) mbar_wait(&empty[sl], (int)(((seq / NBUF) & 1) ^ 1));
        __syncwarp();
        double* dst = ring + (size_t)sl * S::BUFD + S::XOFF;
        const bool with_b = b1 && q >= 1 && q <= r1 - r0;
        const size_t rbase = (size_t)row * nx;
        const int left = ie0 == 0 ? nx - 1 : ie0 - 1;
        const int right = ie0 + w == nx ? 0 : ie0 + w;
        for (int arr = 0; arr < 2; ++arr) {
          const double* src = arr == 0 ? srcx : srct;
          double* d = dst + arr * S::ROWD;
          if (ie0 >= 1 && ie0 + w < nx) {
            copy(d, src + (rbase + left) * NN, (w + 2) * NN);
          } else {
            copy(d, src + (rbase + left) * NN, NN);
            copy(d + NN, src + (rbase + ie0) * NN, w * NN);
            copy(d + (size_t)(w + 1) * NN, src + (rbase + right) * NN, NN);
          }
        }
        if (with_b) copy(dst + 2 * S::ROWD, b1 + ((size_t)(r0 - 1 + q) * nx + ie0) * NN, w * NN);
        cp_async_arrive(&full[sl]);
      }
    }
  } else if (DOT && wid == CW + 1) {
    // ---------------- producer: row tiles of V_0..V_{j-1} for the dot warps (TMA)
    if (dots && lane == 0) {
      const int j = s_j;
      const long long ld = s_ld;
      RingPos vp;
      for (long long k = k0; k < k1;) {
        int ie0, w, r0, r1;
        unit(k, ie0, w, r0, r1);
        const uint32_t bytes = (uint32_t)(w * NN * 8);
        for (int r = r0; r < r1; ++r) {
          const double* src = base + ((size_t)r * nx + ie0) * NN;
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
    // ---------------- dot warps: u = the x row in the ring, w = the row handed over
    if (dots) {
      const int h = wid - (CW + 2);
      double* acc = s_red + h * 2 * (S::JMAX + 1);
      RingPos vp, wp;
      long long seq = 0;
      for (long long k = k0; k < k1;) {
        int ie0, w, r0, r1;
        unit(k, ie0, w, r0, r1);
        const int cnt2 = w * NN / 2;
        for (int r = r0; r < r1; ++r) {
          const long long q = r - r0 + 1;
          const int bsel = wp.s;
          mbar_wait(&wfull[bsel], wp.ph);
          wp.next<2>();
          const int sl = (int)((seq + q) % NBUF);
          mbar_wait(&full[sl], (int)(((seq + q) / NBUF) & 1));  // completed phase: returns at once
          const double2* U2 = reinterpret_cast<const double2*>(ring + (size_t)sl * S::BUFD + S::XOFF + NN);
          const double2* W2 = reinterpret_cast<const double2*>(swr + bsel * S::TILE);
          dots_row<S, true>(U2, W2, vring, vfull, vempty, vp, s_j, cnt2, lane, h, acc, 0);
          __syncwarp();
          if (lane == 0) {  // u (the x ring row) and the w row are free
            mbar_arrive(&wempty[bsel]);
            mbar_arrive(&empty[sl]);
          }
        }
        seq += r1 - r0 + 2;
      }
    }
  } else {
    // ---------------- consumers: thread (element le, line l)
    const int half = S::SPLIT ? tid / S::LN : 0, lt = S::SPLIT ? tid - half * S::LN : tid;
    const int le = lt / NP, l = lt % NP;
    const bool do_x = !S::SPLIT || half == 0, do_y = !S::SPLIT || half == 1;
    long long seq = 0;
    int rowc = 0;
    for (long long k = k0; k < k1;) {
      int ie0, w, r0, r1;
      unit(k, ie0, w, r0, r1);
      const bool active = le < w;
      auto slot = [&](long long q) { return ring + (size_t)((seq + q) % NBUF) * S::BUFD + S::XOFF; };
      auto wait_row = [&](long long q) { mbar_wait(&full[(seq + q) % NBUF], (int)(((seq + q) / NBUF) & 1)); };
      wait_row(0);
      wait_row(1);
      for (int r = r0; r < r1; ++r, ++rowc) {
        const long long q = r - r0 + 1;
        wait_row(q + 1);
        const double* cur = slot(q);
        const double* lo = slot(q - 1);
        const double* hi = slot(q + 1);
        double* sX = sout + (rowc & 1) * 2 * S::OUT;
        double* sY = sX + S::OUT;
        if (active) {
          double xL[NP], xC[NP], xR[NP], uL[NP], uC[NP], uR[NP], out[NP];
          if (do_x) {
            // x-line l (element row l): ring elements le, le + 1, le + 2 of row r
#pragma unroll
            for (int t = 0; t < NP; ++t) {
              xL[t] = cur[le * NN + l * NP + t] * xs;
              xC[t] = cur[(le + 1) * NN + l * NP + t] * xs;
              xR[t] = cur[(le + 2) * NN + l * NP + t] * xs;
              uL[t] = cur[S::ROWD + le * NN + l * NP + t];
              uC[t] = cur[S::ROWD + (le + 1) * NN + l * NP + t];
              uR[t] = cur[S::ROWD + (le + 2) * NN + l * NP + t];
            }
            b1_element<NP>(Px, 0, ie0 + le, xL, xC, xR, uL, uC, uR, out);
#pragma unroll
            for (int t = 0; t < NP; ++t) sX[le * NN + l * NP + t] = out[t];
          }
          if (do_y) {
            // y-line l (element column l): element le + 1 of ring rows r - 1, r, r + 1
#pragma unroll
            for (int t = 0; t < NP; ++t) {
              xL[t] = lo[(le + 1) * NN + t * NP + l] * xs;
              xC[t] = cur[(le + 1) * NN + t * NP + l] * xs;
              xR[t] = hi[(le + 1) * NN + t * NP + l] * xs;
              uL[t] = lo[S::ROWD + (le + 1) * NN + t * NP + l];
              uC[t] = cur[S::ROWD + (le + 1) * NN + t * NP + l];
              uR[t] = hi[S::ROWD + (le + 1) * NN + t * NP + l];
            }
            b1_element<NP>(Py, 0, (int)Py.eoff + r, xL, xC, xR, uL, uC, uR, out);
#pragma unroll
            for (int t = 0; t < NP; ++t) sY[le * NN + t * NP + l] = out[t];
          }
        }
        strip_sync<S::CONS>();  // sX, sY of row r complete; row r-1 is no longer read
        if (tid == 0) mbar_arrive_cnt(&empty[(seq + q - 1) % NBUF], q == 1 ? rel_halo : rel_row);  // row r-1 free
        const int bsel = rowc & 1;
        double* wrow = swr + bsel * S::TILE;
        if (dots) mbar_wait(&wempty[bsel], ((rowc >> 1) & 1) ^ 1);  // the dot warps took row r-2
        const size_t g0 = ((size_t)r * nx + ie0) * NN;
        for (int idx = tid; idx < w * NN; idx += S::CONS) {
          double v = sX[idx] + sY[idx];
          if (b1) v = fma(s_xt[0], cur[2 * S::ROWD + idx], v);
          else v = aug_tail(b, s_xt, g0 + idx, v);
          v = dt * v;
          y[g0 + idx] = v;
          if (dots) wrow[idx] = v;
          nacc = fma(v, v, nacc);
        }
        if (dots) {
          __syncwarp();
          if (lane == 0) mbar_arrive(&wfull[bsel]);
        }
      }
      strip_sync<S::CONS>();  // the unit's last row is done
      if (tid == 0) {
        mbar_arrive_cnt(&empty[(seq + (r1 - r0)) % NBUF], r1 - r0 == 0 ? rel_halo : rel_row);  // row r1 - 1
        mbar_arrive_cnt(&empty[(seq + (r1 - r0) + 1) % NBUF], rel_halo);                        // row r1 (upper halo)
      }
      seq += r1 - r0 + 2;
    }
  }
  __syncthreads();
  if (blockIdx.x == 0 && tid < kTailPad) {  // replicated tail, counted on rank 0
    const double v = (tid + 1 < b.p) ? dt * s_xt[tid + 1] : 0.0;
    y[Px.n + tid] = v;
    if (st->tail_here) nacc = fma(v, v, nacc);
  }
  const double tot = block_sum(nacc, s_buf);
  if constexpr (DOT) {
    // dots: the two tile halves, plus (rank 0) the tail region [n, n + kTailPad) of every
    // slot, which k_ts2 streams with the head; cnt <= JMAX + 1 <= blockDim.x
    const int cnt = dots ? s_j + 1 : 0;
    double ca = 0.0, cb = 0.0;
    if (tid < cnt) {
      constexpr int JS = 2 * (S::JMAX + 1);
      ca = s_red[2 * tid] + s_red[JS + 2 * tid];
      cb = s_red[2 * tid + 1] + s_red[JS + 2 * tid + 1];
      if (blockIdx.x == 0 && st->tail_here) {
        const double* ut = base + (size_t)s_j * s_ld + Px.n;
        const double* vt = base + (size_t)tid * s_ld + Px.n;
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
  } else {
    if (tid == 0) s_red[0] = tot;
    __syncthreads();
    grid_reduce_last(s_red, 1, partials, kMaxSlots, &st->ticket[4], [&](int, double v) { st->rs().nrmA = v; });
  }
}

template <int NP>
class Burgers2D : public OpDevice {
 public:
  B1P<NP> Px{}, Py{};
  int nx = 0, ny = 0, grid = 1;  // ny: owned element rows
  double* halo = nullptr;        // row slab: x lo/hi, u~ lo/hi, send lo/hi (one element row each)
  double* htab = nullptr;        // {h, 2 / h} per element column, then per element row
  long long rowd = 0;
  bool use_strip = true;         // EXPDG_B2_TILE=1: the element-tile kernel (neighbours from L2)
  int strip_grid = 1;
  ~Burgers2D() override {
    cudaFree(halo);
    cudaFree(htab);
  }
  double* hq(int i) const { return halo + (size_t)i * rowd; }
  explicit Burgers2D(const expdg_op_desc& d) {
    desc = d;
    const HostBasis hb = host_lgl_basis(d.order);
    const bool part = d.part_end > d.part_begin;
    nx = d.nx;
    ny = part ? d.part_end - d.part_begin : d.ny;
    for (B1P<NP>* P : {&Px, &Py}) {
      P->periodic = d.periodic;
      P->kappa = d.kappa;
      P->sigma = d.sigma;
      P->entropy = d.flux == 1;
      P->sigma_adaptive = d.sigma_adaptive;
      for (int i = 0; i < NP; ++i) {
        P->w[i] = hb.weights[i];
        P->iw[i] = 1.0 / hb.weights[i];
        for (int j = 0; j < NP; ++j) {
          P->G[i * NP + j] = hb.weights[i] * hb.D[i * NP + j];
          P->Lv[i * NP + j] = hb.D[j * NP + i] * hb.weights[j];
        }
      }
    }
    Px.ne = d.nx;
    Px.nel = d.nx;
    Px.a = d.x0;
    Px.b = d.x1;
    Py.ne = d.ny;  // global rows: boundary faces and h come from the global index
    Py.nel = ny;
    Py.eoff = part ? d.part_begin : 0;
    Py.part = part ? 1 : 0;
    Py.a = d.y0;
    Py.b = d.y1;
    n = (long long)d.nx * ny * NP * NP;
    Px.n = Py.n = n;
    comps = 1;
    rowd = (long long)d.nx * NP * NP;
    {
      std::vector<double> ht = host_h_table(host_axis_breaks(d.x0, d.x1, d.nx, d.grade_x));
      const std::vector<double> hy = host_h_table(host_axis_breaks(d.y0, d.y1, d.ny, d.grade_y));
      ht.insert(ht.end(), hy.begin(), hy.end());
      EXPDG_CUDA(cudaMalloc(&htab, sizeof(double) * ht.size()));
      EXPDG_CUDA(cudaMemcpy(htab, ht.data(), sizeof(double) * ht.size(), cudaMemcpyHostToDevice));
      Px.hh = htab;
      Py.hh = htab + 2 * (size_t)d.nx;
    }
    if (part) {
      EXPDG_CUDA(cudaMalloc(&halo, sizeof(double) * 6 * rowd));
      EXPDG_CUDA(cudaMemset(halo, 0, sizeof(double) * 6 * rowd));
    }
    const long long ntiles = ((long long)d.nx * ny + B2Tile<NP>::TE - 1) / B2Tile<NP>::TE;
    grid = (int)std::max<long long>(1, std::min<long long>(ntiles, 148LL * 8));
    use_strip = !(std::getenv("EXPDG_B2_TILE") && std::getenv("EXPDG_B2_TILE")[0] == '1');
    using SS = B2Strip<NP>;
    EXPDG_CUDA(cudaFuncSetAttribute(k_b2_phi_strip<NP, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, SS::SMEM));
    int per_sm = 1;
    EXPDG_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_b2_phi_strip<NP, false>, SS::THREADS, SS::SMEM));
    const long long rsteps = (long long)((d.nx + SS::W - 1) / SS::W) * ny;
    strip_grid = (int)std::max<long long>(1, std::min<long long>(rsteps, 148LL * std::max(1, per_sm)));
    if (const char* v = std::getenv("EXPDG_B2_DOTS")) use_dots = v[0] != '0';
    // the fused dots stream whole strip rows of V by TMA: full-width strips (then every
    // row tile starts on a 16-byte boundary)
    dots_ok = d.nx % SS::W == 0;
    if constexpr (kDotFits) {
      using SD = B2Strip<NP, true>;
      EXPDG_CUDA(cudaFuncSetAttribute(k_b2_phi_strip<NP, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, SD::SMEM));
      int per_sm_d = 1;
      EXPDG_CUDA(
          cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm_d, k_b2_phi_strip<NP, true>, SD::THREADS, SD::SMEM));
      dots_grid = (int)std::max<long long>(1, std::min<long long>(rsteps, 148LL * std::max(1, per_sm_d)));
    }
  }
  // The strip JVP also takes the DCGS2 pass-1 dots of columns j <= JMAX (EXPDG_B2_DOTS=0: off).
  static constexpr bool kDotFits = B2Strip<NP, true>::FITS;
  bool use_dots = true, dots_ok = false;
  int dots_grid = 1;
  bool dots_on() const { return kDotFits && use_dots && use_strip && dots_ok; }
  int fused_dcgs_dots_jmax() const override { return dots_on() ? B2Strip<NP, true>::JMAX : -1; }
  void exchange(cudaStream_t s, const double* v, double* lo, double* hi) {
    comm->halo(v, v + (size_t)(ny - 1) * rowd, lo, hi, rowd, s);
  }
  void with_halo(B1P<NP>& py, bool x_is_ut) const {
    if (!Py.part) return;
    py.gt_lo = hq(2);
    py.gt_hi = hq(3);
    py.gx_lo = x_is_ut ? hq(2) : hq(0);
    py.gx_hi = x_is_ut ? hq(3) : hq(1);
  }
  void freeze(cudaStream_t s, const double* r) override {
    ref = r;
    if (Py.part) exchange(s, r, hq(2), hq(3));
  }
  void launch_phi_apply(cudaStream_t s, PhiState* st, double* base, double* partials, const BArgs& b, int stage = 1) override {
    if (Py.part) {
      launch_pack_slot(s, st, base, rowd, (long long)(ny - 1) * rowd, hq(4), hq(5));
      comm->halo(hq(4), hq(5), hq(0), hq(1), rowd, s);
    }
    B1P<NP> px = Px, py = Py;
    px.ut = py.ut = ref;
    with_halo(py, false);
    if (dots_on() && stage == 1) {
      if constexpr (kDotFits)
        k_b2_phi_strip<NP, true><<<dots_grid, B2Strip<NP, true>::THREADS, B2Strip<NP, true>::SMEM, s>>>(
            px, py, nx, ny, st, base, partials, b);
    } else if (use_strip)
      k_b2_phi_strip<NP, false><<<strip_grid, B2Strip<NP>::THREADS, B2Strip<NP>::SMEM, s>>>(px, py, nx, ny, st, base,
                                                                                            partials, b);
    else
      k_b2_phi<NP><<<grid, 256, 0, s>>>(px, py, nx, ny, st, base, partials, b);
  }
  void launch_apply(cudaStream_t s, int which, const double* x, double* y) override {
    if (Py.part) exchange(s, x, hq(0), hq(1));
    B1P<NP> px = Px, py = Py;
    px.ut = py.ut = ref;
    with_halo(py, false);
    k_b2_apply<NP><<<grid, 256, 0, s>>>(px, py, nx, ny, which, x, y, nullptr);
  }
  void launch_residual(cudaStream_t s, const double* u, double* r, PhiState* st, double*) override {
    if (Py.part) exchange(s, u, hq(2), hq(3));  // u~ = u for this step's residual and JVPs
    B1P<NP> px = Px, py = Py;
    px.ut = py.ut = u;
    with_halo(py, true);
    k_b2_apply<NP><<<grid, 256, 0, s>>>(px, py, nx, ny, 2, u, r, st);
  }
};

}  // namespace

std::unique_ptr<OpDevice> make_burgers2d(const expdg_op_desc& d) {
  switch (d.order + 1) {
    case 2: return std::make_unique<Burgers2D<2>>(d);
    case 3: return std::make_unique<Burgers2D<3>>(d);
    case 4: return std::make_unique<Burgers2D<4>>(d);
    case 5: return std::make_unique<Burgers2D<5>>(d);
    case 6: return std::make_unique<Burgers2D<6>>(d);
    case 7: return std::make_unique<Burgers2D<7>>(d);
    case 8: return std::make_unique<Burgers2D<8>>(d);
    case 9: return std::make_unique<Burgers2D<9>>(d);
  }
  throw std::invalid_argument("burgers2d: device orders are 1..8");
}

}  // namespace expdg
