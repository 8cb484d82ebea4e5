// Times the tiny control kernels of the PD loop in isolation.
#include <cstdio>
#include <cuda_runtime.h>
#include "../../include/hdk.h"
__global__ void k_empty() {}
int main() {
  hdk_ctl* ctl; double* part;
  cudaMalloc(&ctl, sizeof(hdk_ctl)); cudaMalloc(&part, HDK_RED_BLOCKS * HDK_RED_Q * 8);
  cudaMemset(part, 0, HDK_RED_BLOCKS * HDK_RED_Q * 8);
  cudaStream_t st; cudaStreamCreate(&st);
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  float ms;
  for (int rep = 0; rep < 2; ++rep) {
    cudaEventRecord(a, st);
    for (int i = 0; i < 1000; ++i) k_empty<<<1, 256, 0, st>>>();
    cudaEventRecord(b, st); cudaEventSynchronize(b); cudaEventElapsedTime(&ms, a, b);
    printf("empty kernel: %.2f us\n", ms);
    cudaEventRecord(a, st);
    for (int i = 0; i < 1000; ++i) hdk_ctl_init(ctl, 8, 1e8, 500, 0, 0, 1e-10, 0.1, 1, st);
    cudaEventRecord(b, st); cudaEventSynchronize(b); cudaEventElapsedTime(&ms, a, b);
    printf("ctl_init: %.2f us\n", ms);
    for (int mode = 0; mode < 2; ++mode) {
      hdk_ctl_init(ctl, 8, 1e8, 100000, 0, 0, 1e-30, 0.1, 1, st);
      cudaEventRecord(a, st);
      for (int i = 0; i < 1000; ++i) hdk_aa_solve(ctl, part, mode, st);
      cudaEventRecord(b, st); cudaEventSynchronize(b); cudaEventElapsedTime(&ms, a, b);
      printf("aa_solve mode %d: %.2f us  err=%s\n", mode, ms, cudaGetErrorString(cudaGetLastError()));
    }
    // graph of 1000 aa_solve
    cudaGraph_t g; cudaGraphExec_t ge;
    cudaStreamBeginCapture(st, cudaStreamCaptureModeThreadLocal);
    for (int i = 0; i < 100; ++i) hdk_aa_solve(ctl, part, 1, st);
    cudaStreamEndCapture(st, &g); cudaGraphInstantiate(&ge, g, 0);
    cudaEventRecord(a, st);
    for (int i = 0; i < 10; ++i) cudaGraphLaunch(ge, st);
    cudaEventRecord(b, st); cudaEventSynchronize(b); cudaEventElapsedTime(&ms, a, b);
    printf("aa_solve in graph: %.2f us each\n", ms);
  }
  return 0;
}
