// 1D viscous Burgers LDG operators on sm_100a: the JVP L x
// (proj/src/burgers.cpp:146-180), N x (:182-215) and the full RHS (:217-265),
// collocated LGL (over_integrate = false), periodic or zero-Dirichlet.
//
// One thread per element over a CTA tile of 128 elements staged (with a
// one-element halo each side) in shared memory by coalesced loads; the LDG
// gradient of the two neighbours is recomputed at the shared face node instead
// of being written to HBM, so L x streams x, u~ and (in the phi cycle) b_1 once
// and writes y once: 32 B/DOF (SURVEY.md §8d canonical JVP bytes).
#include <algorithm>

#include "fused.cuh"

namespace expdg {

namespace {

using namespace burgers;
constexpr int kB1Threads = 128;

// Standalone apply: y = L x | N x | rhs(x).
template <int NP>
__global__ void __launch_bounds__(kB1Threads) k_b1_apply(B1P<NP> P, int mode, const double* __restrict__ x,
                                                         double* __restrict__ y, const PhiState* st) {
  __shared__ double sx[(kB1Threads + 2) * NP], su[(kB1Threads + 2) * NP], sy[kB1Threads * NP];
  if (st && st->stopped) return;
  const int ntiles = (P.nel + kB1Threads - 1) / kB1Threads;
  for (int tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
    const long long e0 = (long long)tile * kB1Threads;
    const int E = (int)(P.nel - e0 < kB1Threads ? P.nel - e0 : kB1Threads);
    __syncthreads();
    stage_elements<NP, 1>(P, e0, E, x, 1.0, mode != 2, sx, su);
    __syncthreads();
    const int t = threadIdx.x;
    if (t < E) {
      double out[NP];
      b1_element<NP>(P, mode, (int)(P.eoff + e0 + t), sx + t * NP, sx + (t + 1) * NP, sx + (t + 2) * NP, su + t * NP,
                     su + (t + 1) * NP, su + (t + 2) * NP, out);
#pragma unroll
      for (int i = 0; i < NP; ++i) sy[t * NP + i] = out[i];
    }
    __syncthreads();
    for (int idx = threadIdx.x; idx < E * NP; idx += blockDim.x) y[e0 * NP + idx] = sy[idx];
  }
}

// Phi-cycle apply: y = dt (L s_j V_j + sum_i x_tail[i] b_{p-i}) into slot j+1
// (proj/src/phi.cpp:151-158) and ||y||^2 (pre_norm / avnorm).
template <int NP>
__global__ void __launch_bounds__(kB1Threads) k_b1_phi(B1P<NP> P, PhiState* st, double* base, double* partials,
                                                       BArgs b) {
  __shared__ double sx[(kB1Threads + 2) * NP], su[(kB1Threads + 2) * NP], sy[kB1Threads * NP];
  __shared__ int s_go, s_j;
  __shared__ double s_xs, s_dt, s_xt[kMaxP];
  __shared__ long long s_ld;
  __shared__ double s_buf[kB1Threads / 32];
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
  double nacc = 0.0;
  const int ntiles = (P.nel + kB1Threads - 1) / kB1Threads;
  for (int tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
    const long long e0 = (long long)tile * kB1Threads;
    const int E = (int)(P.nel - e0 < kB1Threads ? P.nel - e0 : kB1Threads);
    __syncthreads();
    stage_elements<NP, 1>(P, e0, E, x, xs, true, sx, su);
    __syncthreads();
    const int t = threadIdx.x;
    if (t < E) {
      double out[NP];
      b1_element<NP>(P, 0, (int)(P.eoff + e0 + t), sx + t * NP, sx + (t + 1) * NP, sx + (t + 2) * NP, su + t * NP,
                     su + (t + 1) * NP, su + (t + 2) * NP, out);
#pragma unroll
      for (int i = 0; i < NP; ++i) sy[t * NP + i] = out[i];
    }
    __syncthreads();
    for (int idx = threadIdx.x; idx < E * NP; idx += blockDim.x) {
      const long long g = e0 * NP + idx;
      double v = sy[idx];
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

// Mesh / slab-partition plumbing shared by the 1D Burgers operators (halo depth H
// elements: 1 collocated, 2 over-integrated).  Partitioned operators own elements
// [part_begin, part_end) and exchange H elements with each periodic neighbour
// before every application (the reference mesh is one interval).
template <class PP, int NP, int H>
class B1Base : public OpDevice {
 public:
  PP P{};
  int grid = 1;
  double* src = nullptr;
  double* halo = nullptr;  // x lo/hi, u~ lo/hi, send lo/hi: H NP doubles each
  double* htab = nullptr;  // {h_e, 2 / h_e} per global element
  long long layer = 0;
  ~B1Base() override {
    cudaFree(src);
    cudaFree(halo);
    cudaFree(htab);
  }
  double* hq(int i) const { return halo + (size_t)i * layer; }
  void init_mesh(const expdg_op_desc& d) {
    desc = d;
    const bool part = d.part_end > d.part_begin;
    P.ne = d.nx;
    P.periodic = d.periodic;
    P.a = d.x0;
    P.b = d.x1;
    P.kappa = d.kappa;
    P.sigma = d.sigma;
    P.entropy = d.flux == 1;
    P.sigma_adaptive = d.sigma_adaptive;
    P.eoff = part ? d.part_begin : 0;
    P.nel = part ? d.part_end - d.part_begin : d.nx;
    P.part = part ? 1 : 0;
    n = (long long)P.nel * NP;
    P.n = n;
    comps = 1;
    layer = (long long)H * NP;
    if (part) {
      EXPDG_CUDA(cudaMalloc(&halo, sizeof(double) * 6 * layer));
      EXPDG_CUDA(cudaMemset(halo, 0, sizeof(double) * 6 * layer));
    }
    const int ntiles = (P.nel + kB1Threads - 1) / kB1Threads;
    grid = std::max(1, std::min(ntiles, 148 * 8));
    const std::vector<double> ht = host_h_table(d.x0, d.x1, d.nx);
    EXPDG_CUDA(cudaMalloc(&htab, sizeof(double) * ht.size()));
    EXPDG_CUDA(cudaMemcpy(htab, ht.data(), sizeof(double) * ht.size(), cudaMemcpyHostToDevice));
    P.hh = htab;
  }
  void exchange(cudaStream_t s, const double* v, double* lo, double* hi) {
    comm->halo(v, v + (size_t)(P.nel - H) * NP, lo, hi, layer, s);
  }
  PP params(const double* ut) const {
    PP p = P;
    p.ut = ut;
    if (p.part) {
      p.gx_lo = hq(0);
      p.gx_hi = hq(1);
      p.gt_lo = hq(2);
      p.gt_hi = hq(3);
    }
    return p;
  }
  virtual void run_phi(cudaStream_t s, const PP& p, PhiState* st, double* base, double* partials,
                       const BArgs& b) = 0;
  virtual void run_apply(cudaStream_t s, const PP& p, int mode, const double* x, double* y, const PhiState* st) = 0;

  void set_source(cudaStream_t s, const double* weak) override {
    if (!src) EXPDG_CUDA(cudaMalloc(&src, sizeof(double) * n));
    EXPDG_CUDA(cudaMemcpyAsync(src, weak, sizeof(double) * n, cudaMemcpyDeviceToDevice, s));
    P.src = src;
  }
  void freeze(cudaStream_t s, const double* r) override {
    ref = r;
    if (P.part) exchange(s, r, hq(2), hq(3));
  }
  void launch_phi_apply(cudaStream_t s, PhiState* st, double* base, double* partials, const BArgs& b, int stage = 1) override {
    if (P.part) {  // halo elements of the slot this cycle applies the operator to
      launch_pack_slot(s, st, base, layer, (long long)(P.nel - H) * NP, hq(4), hq(5));
      comm->halo(hq(4), hq(5), hq(0), hq(1), layer, s);
    }
    run_phi(s, params(ref), st, base, partials, b);
  }
  void launch_apply(cudaStream_t s, int which, const double* x, double* y) override {
    if (P.part) exchange(s, x, hq(0), hq(1));
    run_apply(s, params(ref), which, x, y, nullptr);
  }
  // R at u~ = u; u's halo serves both the applied vector and u~ (and this step's JVPs)
  void launch_residual(cudaStream_t s, const double* u, double* r, PhiState* st, double*) override {
    PP p = params(u);
    if (P.part) {
      exchange(s, u, hq(2), hq(3));
      p.gx_lo = hq(2);
      p.gx_hi = hq(3);
    }
    run_apply(s, p, 2, u, r, st);
  }
};

template <int NP>
class Burgers1D : public B1Base<B1P<NP>, NP, 1> {
 public:
  using B = B1Base<B1P<NP>, NP, 1>;
  explicit Burgers1D(const expdg_op_desc& d) {
    const HostBasis hb = host_lgl_basis(d.order);
    this->init_mesh(d);
    for (int i = 0; i < NP; ++i) {
      this->P.w[i] = hb.weights[i];
      this->P.iw[i] = 1.0 / hb.weights[i];
      for (int j = 0; j < NP; ++j) {
        this->P.G[i * NP + j] = hb.weights[i] * hb.D[i * NP + j];
        this->P.Lv[i * NP + j] = hb.D[j * NP + i] * hb.weights[j];
      }
    }
  }
  void run_phi(cudaStream_t s, const B1P<NP>& p, PhiState* st, double* base, double* partials,
               const BArgs& b) override {
    k_b1_phi<NP><<<this->grid, kB1Threads, 0, s>>>(p, st, base, partials, b);
  }
  bool fused_capable() const override { return !this->P.part && this->n <= kFusedMaxN; }
  void launch_fused(cudaStream_t s, Engine& e, const BArgs& b) override {
    B1FusedElem<NP> el{this->params(this->ref)};
    launch_phi_fused(s, e, el, b);
  }
  void run_apply(cudaStream_t s, const B1P<NP>& p, int mode, const double* x, double* y,
                 const PhiState* st) override {
    k_b1_apply<NP><<<this->grid, kB1Threads, 0, s>>>(p, mode, x, y, st);
  }
};

// ---------------------------------------------------------------- over-integrated 1D Burgers
// Over-integrated kernels stage a two-element halo: the dense consistent-mass solve
// makes a neighbour's face q depend on its other face.
template <int NP, int NQ>
__global__ void __launch_bounds__(kB1Threads) k_b1oi_apply(B1OP<NP, NQ> P, int mode, const double* __restrict__ x,
                                                           double* __restrict__ y, const PhiState* st) {
  __shared__ double sx[(kB1Threads + 4) * NP], su[(kB1Threads + 4) * NP], sy[kB1Threads * NP];
  if (st && st->stopped) return;
  const int ntiles = (P.nel + kB1Threads - 1) / kB1Threads;
  for (int tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
    const long long e0 = (long long)tile * kB1Threads;
    const int E = (int)(P.nel - e0 < kB1Threads ? P.nel - e0 : kB1Threads);
    __syncthreads();
    stage_elements<NP, 2>(P, e0, E, x, 1.0, mode != 2, sx, su);
    __syncthreads();
    const int t = threadIdx.x;
    if (t < E) {
      double out[NP];
      const double* b = sx + (t + 2) * NP;
      const double* ub = su + (t + 2) * NP;
      b1oi_element<NP, NQ>(P, mode, (int)(P.eoff + e0 + t), b - 2 * NP, b - NP, b, b + NP, b + 2 * NP, ub - NP, ub, ub + NP,
                           out);
#pragma unroll
      for (int i = 0; i < NP; ++i) sy[t * NP + i] = out[i];
    }
    __syncthreads();
    for (int idx = threadIdx.x; idx < E * NP; idx += blockDim.x) y[e0 * NP + idx] = sy[idx];
  }
}

template <int NP, int NQ>
__global__ void __launch_bounds__(kB1Threads) k_b1oi_phi(B1OP<NP, NQ> P, PhiState* st, double* base,
                                                         double* partials, BArgs b) {
  __shared__ double sx[(kB1Threads + 4) * NP], su[(kB1Threads + 4) * NP], sy[kB1Threads * NP];
  __shared__ int s_go, s_j;
  __shared__ double s_xs, s_dt, s_xt[kMaxP];
  __shared__ long long s_ld;
  __shared__ double s_buf[kB1Threads / 32];
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
  double nacc = 0.0;
  const int ntiles = (P.nel + kB1Threads - 1) / kB1Threads;
  for (int tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
    const long long e0 = (long long)tile * kB1Threads;
    const int E = (int)(P.nel - e0 < kB1Threads ? P.nel - e0 : kB1Threads);
    __syncthreads();
    stage_elements<NP, 2>(P, e0, E, x, xs, true, sx, su);
    __syncthreads();
    const int t = threadIdx.x;
    if (t < E) {
      double out[NP];
      const double* bb = sx + (t + 2) * NP;
      const double* ub = su + (t + 2) * NP;
      b1oi_element<NP, NQ>(P, 0, (int)(P.eoff + e0 + t), bb - 2 * NP, bb - NP, bb, bb + NP, bb + 2 * NP, ub - NP, ub,
                           ub + NP, out);
#pragma unroll
      for (int i = 0; i < NP; ++i) sy[t * NP + i] = out[i];
    }
    __syncthreads();
    for (int idx = threadIdx.x; idx < E * NP; idx += blockDim.x) {
      const long long g = e0 * NP + idx;
      double v = sy[idx];
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

template <int NP, int NQ>
class Burgers1DOI : public B1Base<B1OP<NP, NQ>, NP, 2> {
 public:
  explicit Burgers1DOI(const expdg_op_desc& d) {
    const HostOI o = host_burgers_oi(d.order);
    if (o.nq != NQ) throw std::invalid_argument("burgers1d: over-integration rule mismatch");
    this->init_mesh(d);
    for (int i = 0; i < NP * NP; ++i) {
      this->P.G[i] = o.G[i];
      this->P.Mi[i] = o.Mi[i];
    }
    for (int i = 0; i < NP * NQ; ++i) {
      this->P.Lv[i] = o.Lv[i];
      this->P.I[i] = o.I[i];
    }
  }
  void run_phi(cudaStream_t s, const B1OP<NP, NQ>& p, PhiState* st, double* base, double* partials,
               const BArgs& b) override {
    k_b1oi_phi<NP, NQ><<<this->grid, kB1Threads, 0, s>>>(p, st, base, partials, b);
  }
  bool fused_capable() const override { return !this->P.part && this->n <= kFusedMaxN; }
  void launch_fused(cudaStream_t s, Engine& e, const BArgs& b) override {
    B1OIFusedElem<NP, NQ> el{this->params(this->ref)};
    launch_phi_fused(s, e, el, b);
  }
  void run_apply(cudaStream_t s, const B1OP<NP, NQ>& p, int mode, const double* x, double* y,
                 const PhiState* st) override {
    k_b1oi_apply<NP, NQ><<<this->grid, kB1Threads, 0, s>>>(p, mode, x, y, st);
  }
};

// ---------------------------------------------------------------- dense (test operator)
__global__ void k_dense_apply(int n, const double* __restrict__ A, const double* __restrict__ x, double xs,
                              double* __restrict__ y) {
  const int row = blockIdx.x * (blockDim.x / 32) + (threadIdx.x >> 5);
  const int lane = threadIdx.x & 31;
  if (row >= n) return;
  double s = 0.0;
  for (int c = lane; c < n; c += 32) s = fma(A[(size_t)row * n + c], x[c] * xs, s);
  s = warp_sum(s);
  if (lane == 0) y[row] = s;
}

// y = dt (A s_j V_j + aug) into slot j+1, ||y||^2 -> red.nrmA (single CTA, test sizes)
__global__ void k_dense_phi(int n, const double* __restrict__ A, PhiState* st, double* base, BArgs b) {
  __shared__ double s_buf[32];
  __shared__ double s_xt[kMaxP];
  if (st->stopped) return;
  if (!apply_go(st, base)) return;
  const int j = st->j;
  const double xs = st->scale[j], dt = st->dt;
  const long long ld = st->ld;
  const double* x = base + (size_t)j * ld;
  double* y = base + (size_t)(j + 1) * ld;
  if (threadIdx.x < kMaxP) s_xt[threadIdx.x] = (threadIdx.x < b.p) ? x[n + threadIdx.x] * xs : 0.0;
  __syncthreads();
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = blockDim.x >> 5;
  double nacc = 0.0;
  for (int row = wid; row < n; row += nw) {
    double s = 0.0;
    for (int c = lane; c < n; c += 32) s = fma(A[(size_t)row * n + c], x[c] * xs, s);
    s = warp_sum(s);
    if (lane == 0) {
      double v = s;
      for (int i = 0; i < b.p; ++i)
        if (b.b[b.p - i]) v = fma(s_xt[i], b.b[b.p - i][row], v);
      v = dt * v;
      y[row] = v;
      nacc = fma(v, v, nacc);
    }
  }
  if (threadIdx.x < kTailPad) {
    const int i = threadIdx.x;
    const double v = (i + 1 < b.p) ? dt * s_xt[i + 1] : 0.0;
    y[n + i] = v;
    nacc = fma(v, v, nacc);
  }
  const double tot = block_sum(nacc, s_buf);
  if (threadIdx.x == 0) st->rs().nrmA = tot;
}

class DenseOp : public OpDevice {
 public:
  double* A = nullptr;
  DenseOp(int nn, const double* a_host) {
    n = nn;
    desc.kind = EXPDG_DENSE;
    EXPDG_CUDA(cudaMalloc(&A, sizeof(double) * (size_t)nn * nn));
    EXPDG_CUDA(cudaMemcpy(A, a_host, sizeof(double) * (size_t)nn * nn, cudaMemcpyHostToDevice));
  }
  ~DenseOp() override { cudaFree(A); }
  void launch_phi_apply(cudaStream_t s, PhiState* st, double* base, double*, const BArgs& b, int = 1) override {
    k_dense_phi<<<1, 1024, 0, s>>>((int)n, A, st, base, b);
  }
  void launch_apply(cudaStream_t s, int which, const double* x, double* y) override {
    if (which != 0) throw std::invalid_argument("dense operator: only the linear action exists");
    k_dense_apply<<<(unsigned)((n + 7) / 8), 256, 0, s>>>((int)n, A, x, 1.0, y);
  }
  void launch_residual(cudaStream_t s, const double* u, double* r, PhiState*, double*) override {
    k_dense_apply<<<(unsigned)((n + 7) / 8), 256, 0, s>>>((int)n, A, u, 1.0, r);
  }
};

}  // namespace

std::unique_ptr<OpDevice> make_burgers1d(const expdg_op_desc& d) {
  if (d.over_integrate) {
    switch (d.order) {  // NQ = (3k + 3) / 2 Gauss points (proj/src/burgers.cpp:41)
      case 1: return std::make_unique<Burgers1DOI<2, 3>>(d);
      case 2: return std::make_unique<Burgers1DOI<3, 4>>(d);
      case 3: return std::make_unique<Burgers1DOI<4, 6>>(d);
      case 4: return std::make_unique<Burgers1DOI<5, 7>>(d);
      case 5: return std::make_unique<Burgers1DOI<6, 9>>(d);
      case 6: return std::make_unique<Burgers1DOI<7, 10>>(d);
      case 7: return std::make_unique<Burgers1DOI<8, 12>>(d);
      case 8: return std::make_unique<Burgers1DOI<9, 13>>(d);
    }
    throw std::invalid_argument("burgers1d: device orders are 1..8");
  }
  switch (d.order + 1) {
    case 2: return std::make_unique<Burgers1D<2>>(d);
    case 3: return std::make_unique<Burgers1D<3>>(d);
    case 4: return std::make_unique<Burgers1D<4>>(d);
    case 5: return std::make_unique<Burgers1D<5>>(d);
    case 6: return std::make_unique<Burgers1D<6>>(d);
    case 7: return std::make_unique<Burgers1D<7>>(d);
    case 8: return std::make_unique<Burgers1D<8>>(d);
    case 9: return std::make_unique<Burgers1D<9>>(d);
  }
  throw std::invalid_argument("burgers1d: device orders are 1..8");
}

std::unique_ptr<OpDevice> make_dense(int n, const double* a_host) { return std::make_unique<DenseOp>(n, a_host); }

}  // namespace expdg
