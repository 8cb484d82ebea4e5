// FP64 FMA throughput of this GPU (the denominator for FP64-pipe fractions):
// every thread runs 8 independent DFMA chains in registers; grid = SMs x 8
// blocks of 256.  Prints {"fp64_tflops": ...}.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o dfma_peak dfma_peak.cu
#include <cstdio>
#include <cuda_runtime.h>

__global__ void k_dfma(double* out, int iters, double a, double b) {
  double x[8];
  for (int i = 0; i < 8; ++i) x[i] = threadIdx.x * 1e-3 + i;
  for (int it = 0; it < iters; ++it)
#pragma unroll
    for (int i = 0; i < 8; ++i) x[i] = fma(x[i], a, b);
  double s = 0;
  for (int i = 0; i < 8; ++i) s += x[i];
  if (s == 12345.678) out[threadIdx.x] = s;  // keep the chains live
}

int main() {
  int dev = 0, sms = 0, clk = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, dev);
  double* out;
  cudaMalloc(&out, 1024 * sizeof(double));
  const int blocks = sms * 8, threads = 256, iters = 1 << 16;
  k_dfma<<<blocks, threads>>>(out, 1024, 0.999999, 1e-7);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  double best = 0;
  for (int rep = 0; rep < 5; ++rep) {
    cudaEventRecord(e0);
    k_dfma<<<blocks, threads>>>(out, iters, 0.999999, 1e-7);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms = 0;
    cudaEventElapsedTime(&ms, e0, e1);
    const double flops = 2.0 * 8.0 * iters * double(blocks) * threads;
    const double tf = flops / (ms * 1e-3) / 1e12;
    if (tf > best) best = tf;
  }
  printf("{\"fp64_tflops\": %.3f, \"sms\": %d, \"clock_mhz_attr\": %d, \"kernel\": \"8 independent DFMA chains/thread, %d x %d\"}\n",
         best, sms, clk / 1000, blocks, threads);
  return 0;
}
