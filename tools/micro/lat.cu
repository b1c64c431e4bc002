// Micro-benchmarks behind the controller work: dependent DFMA latency, shared-memory
// load latency (generic / shared addressing), CTA barrier cost at 256 threads, fp64 division.
#include <cstdio>
#include <cuda_runtime.h>
__global__ void k(long long* out, double* gbuf) {
  __shared__ double sm[1024];
  __shared__ int idxs[1024];
  const int tid = threadIdx.x;
  for (int i = tid; i < 1024; i += blockDim.x) { sm[i] = 1.0 + 1e-9 * i; idxs[i] = (i * 7 + 1) & 1023; }
  __syncthreads();
  double a = 1.0 + tid * 1e-12, b = 0.999999, c = 1e-7;
  long long t0 = clock64();
#pragma unroll 1
  for (int i = 0; i < 256; ++i) {
    a = fma(a, b, c); a = fma(a, b, c); a = fma(a, b, c); a = fma(a, b, c);
  }
  long long t1 = clock64();
  if (tid == 0) out[0] = (t1 - t0) / 1024;  // dependent DFMA
  // pointer-chasing LDS (shared addressing)
  int p = tid & 1023;
  t0 = clock64();
#pragma unroll 1
  for (int i = 0; i < 256; ++i) { p = idxs[p]; p = idxs[p]; p = idxs[p]; p = idxs[p]; }
  t1 = clock64();
  if (tid == 0) out[1] = (t1 - t0) / 1024;
  // generic addressing
  const int* gi = idxs;
  asm volatile("" : "+l"(gi));
  t0 = clock64();
#pragma unroll 1
  for (int i = 0; i < 256; ++i) { p = gi[p]; p = gi[p]; p = gi[p]; p = gi[p]; }
  t1 = clock64();
  if (tid == 0) out[2] = (t1 - t0) / 1024;
  // barrier
  t0 = clock64();
#pragma unroll 1
  for (int i = 0; i < 256; ++i) { __syncthreads(); __syncthreads(); __syncthreads(); __syncthreads(); }
  t1 = clock64();
  if (tid == 0) out[3] = (t1 - t0) / 1024;
  // division chain
  t0 = clock64();
#pragma unroll 1
  for (int i = 0; i < 256; ++i) { a = 1.0 / a; a = 1.0 / a; a = 1.0 / a; a = 1.0 / a; }
  t1 = clock64();
  if (tid == 0) out[4] = (t1 - t0) / 1024;
  // sqrt chain
  t0 = clock64();
#pragma unroll 1
  for (int i = 0; i < 256; ++i) { a = sqrt(a); a = sqrt(a); a = sqrt(a); a = sqrt(a); }
  t1 = clock64();
  if (tid == 0) out[5] = (t1 - t0) / 1024;
  // redux
  unsigned r = tid;
  t0 = clock64();
#pragma unroll 1
  for (int i = 0; i < 256; ++i) { r = __reduce_max_sync(0xffffffffu, r + 1); r = __reduce_max_sync(0xffffffffu, r + 1); r = __reduce_max_sync(0xffffffffu, r + 1); r = __reduce_max_sync(0xffffffffu, r + 1); }
  t1 = clock64();
  if (tid == 0) out[6] = (t1 - t0) / 1024;
  // dependent double load + fma (smem)
  t0 = clock64();
#pragma unroll 1
  for (int i = 0; i < 256; ++i) { a = fma(a, sm[(i * 4) & 1023], c); a = fma(a, sm[(i * 4 + 1) & 1023], c); a = fma(a, sm[(i * 4 + 2) & 1023], c); a = fma(a, sm[(i * 4 + 3) & 1023], c); }
  t1 = clock64();
  if (tid == 0) out[7] = (t1 - t0) / 1024;
  gbuf[tid] = a + p + r;
}
int main() {
  long long* out; double* g;
  cudaMalloc(&out, 64); cudaMalloc(&g, 8 * 1024);
  for (int th : {32, 256}) {
    k<<<1, th>>>(out, g);
    long long h[8];
    cudaMemcpy(h, out, 64, cudaMemcpyDeviceToHost);
    printf("threads %d: dfma %lld, lds(shared) %lld, lds(generic) %lld, barrier %lld, ddiv %lld, dsqrt %lld, redux %lld, fma+lds stream %lld cycles\n",
           th, h[0], h[1], h[2], h[3], h[4], h[5], h[6], h[7]);
  }
  return 0;
}
