// FP64 peak microbenchmarks on B200 (sm_100a): the roofline denominators for the FP64
// path (MEASURED_PEAKS.json has no FP64 entry).
//   dfma : FFMA.F64 chains on the CUDA cores (8 independent accumulators per thread)
//   dmma : mma.sync.aligned.m8n8k4.row.col.f64 (SASS DMMA) chains, 4 accumulators per warp
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/fp64_peak tools/fp64_peak.cu
#include <cstdio>
#include <cuda_runtime.h>

__global__ void k_dfma(double* out, int iters, double a, double b) {
  double x[8];
#pragma unroll
  for (int i = 0; i < 8; ++i) x[i] = threadIdx.x * 1e-9 + i;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i) x[i] = fma(x[i], a, b);
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < 8; ++i) s += x[i];
  if (s == 12345.678) out[0] = s;
}

__global__ void k_dmma(double* out, int iters) {
  double a = 1.0 + threadIdx.x * 1e-9, b = 0.999;
  double c[4][2];
#pragma unroll
  for (int i = 0; i < 4; ++i) c[i][0] = c[i][1] = 0.0;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 4; ++i)
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                   : "+d"(c[i][0]), "+d"(c[i][1])
                   : "d"(a), "d"(b));
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < 4; ++i) s += c[i][0] + c[i][1];
  if (s == 12345.678) out[0] = s;
}

int main() {
  double* d;
  cudaMalloc(&d, 8);
  cudaDeviceProp prop;
  cudaGetDeviceProperties(&prop, 0);
  const int sms = prop.multiProcessorCount;
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  float ms;
  // DFMA
  double best_dfma = 0;
  for (int rep = 0; rep < 5; ++rep) {
    const int blocks = sms * 8, threads = 256, iters = 20000;
    cudaEventRecord(e0);
    k_dfma<<<blocks, threads>>>(d, iters, 0.9999999, 1e-7);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    cudaEventElapsedTime(&ms, e0, e1);
    const double fl = 2.0 * 8 * iters * (double)blocks * threads;
    if (rep > 0 && fl / (ms * 1e-3) > best_dfma) best_dfma = fl / (ms * 1e-3);
  }
  double best_dmma = 0;
  for (int rep = 0; rep < 5; ++rep) {
    const int blocks = sms * 8, threads = 256, iters = 20000;
    cudaEventRecord(e0);
    k_dmma<<<blocks, threads>>>(d, iters);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    cudaEventElapsedTime(&ms, e0, e1);
    const double warps = (double)blocks * threads / 32;
    const double fl = 2.0 * 8 * 8 * 4 * 4 * (double)iters * warps;
    if (rep > 0 && fl / (ms * 1e-3) > best_dmma) best_dmma = fl / (ms * 1e-3);
  }
  cudaError_t err = cudaGetLastError();
  printf("{\"sms\": %d, \"dfma_tflops\": %.3f, \"dmma_tflops\": %.3f, \"cuda\": \"%s\"}\n", sms, best_dfma * 1e-12,
         best_dmma * 1e-12, cudaGetErrorString(err));
  return 0;
}
