// Reference-state checks shared by the operators: finiteness (Burgers,
// proj/src/burgers.cpp:34-35) and Euler admissibility (proj/src/euler.cpp:8-13,
// :210-211).
#include <algorithm>

#include "krylov.cuh"

namespace expdg {

__global__ void k_check_ref(const double* __restrict__ q, long long nelem, int comps, int np, int euler_dim,
                            double gm1, int* flag) {
  const long long nodes = nelem * np;
  const long long stride = (long long)gridDim.x * blockDim.x;
  for (long long g = (long long)blockIdx.x * blockDim.x + threadIdx.x; g < nodes; g += stride) {
    const long long e = g / np;
    const int node = (int)(g % np);
    const double* b = q + e * comps * np + node;
    if (euler_dim == 0) {
      if (!isfinite(b[0])) atomicOr(flag, 1);
      continue;
    }
    const double rho = b[0];
    double m2 = 0.0;
    for (int d = 0; d < euler_dim; ++d) m2 += b[(1 + d) * np] * b[(1 + d) * np];
    const double E = b[(1 + euler_dim) * np];
    bool ok = rho > 0.0;
    if (ok) {
      const double p = gm1 * (E - 0.5 * m2 / rho);  // admissible(q, cfg.gamma), proj/src/euler.cpp:8-13
      ok = p > 0.0;
    }
    if (!ok) atomicOr(flag, 2);
  }
}

// First / last owned element layer of Krylov slot j (the vector the next phi-cycle
// apply reads) into the halo send buffers; no-op unless this cycle applies the operator.
__global__ void k_pack_slot(const PhiState* st, const double* base, long long layer, long long last,
                            double* __restrict__ lo, double* __restrict__ hi) {
  if (!apply_go(st, base)) return;
  const double* x = base + (size_t)st->j * st->ld;
  const long long stride = (long long)gridDim.x * blockDim.x;
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < layer; i += stride) {
    lo[i] = x[i];
    hi[i] = x[last + i];
  }
}

void launch_pack_slot(cudaStream_t s, const PhiState* st, const double* base, long long layer, long long last,
                      double* lo, double* hi) {
  const long long blocks = std::min<long long>(592, (layer + 255) / 256);
  k_pack_slot<<<(unsigned)std::max<long long>(1, blocks), 256, 0, s>>>(st, base, layer, last, lo, hi);
}

int op_check_ref(OpDevice& op, cudaStream_t s, const double* ref) {
  const expdg_op_desc& d = op.desc;
  if (d.kind == EXPDG_DENSE || d.kind == EXPDG_USER) return 0;  // no reference-state check of their own
  int* flag = nullptr;
  EXPDG_CUDA(cudaMallocAsync(&flag, sizeof(int), s));
  EXPDG_CUDA(cudaMemsetAsync(flag, 0, sizeof(int), s));
  const int np1 = d.order + 1;
  int np = np1, comps = 1, edim = 0;
  long long ne = d.nx;
  if (d.kind == EXPDG_BURGERS2D) { np = np1 * np1; ne = (long long)d.nx * d.ny; }
  if (d.kind == EXPDG_EULER2D) { np = np1 * np1; ne = (long long)d.nx * d.ny; comps = 4; edim = 2; }
  if (d.kind == EXPDG_EULER3D) { np = np1 * np1 * np1; ne = (long long)d.nx * d.ny * d.nz; comps = 5; edim = 3; }
  ne = op.n / ((long long)comps * np);  // the owned elements (slab-partitioned operators)
  k_check_ref<<<592, 256, 0, s>>>(ref, ne, comps, np, edim, d.gamma - 1.0, flag);
  int h = 0;
  EXPDG_CUDA(cudaMemcpyAsync(&h, flag, sizeof(int), cudaMemcpyDeviceToHost, s));
  EXPDG_CUDA(cudaFreeAsync(flag, s));
  EXPDG_CUDA(cudaStreamSynchronize(s));
  if (h & 2) return 2;
  if (h & 1) return 1;
  return 0;
}

}  // namespace expdg
