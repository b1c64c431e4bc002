// Micro-benchmark: fp64 FMA pipe (DFMA) vs fp64 tensor-core MMA (mma.sync m8n8k4 f64)
// throughput on one B200, to decide whether the DG operators' small contractions belong
// on tensor cores (BASELINE.json north star (1)).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o fp64_pipes tools/fp64_pipes.cu && ./fp64_pipes
#include <cstdio>
#include <cuda_runtime.h>

constexpr int ITERS = 4096;

__global__ void k_dfma(double* out, double a, double b) {
  double x[8];
#pragma unroll
  for (int i = 0; i < 8; ++i) x[i] = threadIdx.x * 1e-3 + i;
  for (int it = 0; it < ITERS; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i) x[i] = fma(x[i], a, b);
  }
  double s = 0.0;
#pragma unroll
  for (int i = 0; i < 8; ++i) s += x[i];
  if (s == 1.2345) out[threadIdx.x] = s;
}

__global__ void k_dmma(double* out, double a, double b) {
  double c[4][2];
#pragma unroll
  for (int i = 0; i < 4; ++i) c[i][0] = c[i][1] = threadIdx.x * 1e-3 + i;
  const double av = a + threadIdx.x * 1e-9, bv = b - threadIdx.x * 1e-9;
  for (int it = 0; it < ITERS; ++it) {
#pragma unroll
    for (int i = 0; i < 4; ++i)
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0, %1}, {%2}, {%3}, {%0, %1};"
                   : "+d"(c[i][0]), "+d"(c[i][1])
                   : "d"(av), "d"(bv));
  }
  double s = 0.0;
#pragma unroll
  for (int i = 0; i < 4; ++i) s += c[i][0] + c[i][1];
  if (s == 1.2345) out[threadIdx.x] = s;
}

int main() {
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  double* out;
  cudaMalloc(&out, 1024 * sizeof(double));
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  for (int warps = 4; warps <= 32; warps *= 2) {
    const int blocks = sms * 2, threads = warps * 32 / 2;
    float ms;
    k_dfma<<<blocks, threads>>>(out, 1.0000001, 1e-7);
    cudaEventRecord(e0);
    k_dfma<<<blocks, threads>>>(out, 1.0000001, 1e-7);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    cudaEventElapsedTime(&ms, e0, e1);
    const double fl_fma = 2.0 * blocks * threads * 8.0 * ITERS;
    k_dmma<<<blocks, threads>>>(out, 1.0000001, 1e-7);
    cudaEventRecord(e0);
    k_dmma<<<blocks, threads>>>(out, 1.0000001, 1e-7);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms2;
    cudaEventElapsedTime(&ms2, e0, e1);
    // m8n8k4: 8 x 8 x 4 = 256 FMA per warp-level MMA
    const double fl_mma = 2.0 * 256.0 * (blocks * threads / 32.0) * 4.0 * ITERS;
    printf("{\"warps_per_sm\": %d, \"dfma_tflops\": %.2f, \"dmma_tflops\": %.2f}\n", warps,
           fl_fma / (ms * 1e-3) / 1e12, fl_mma / (ms2 * 1e-3) / 1e12);
  }
  printf("err: %s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
