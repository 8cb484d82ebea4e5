// Batch reductions of the system-ID evaluation (C5): per-sample trajectory
// loss 1/2|q_T - q_target|^2 and the fixed-order sum over a GPU's samples of
// [loss, dL/dE] that enters the NCCL all-reduce.  Both are
// deterministic: one block, fixed strided partials, fixed tree.
#include "../../include/hdk.h"
#include "launch.cuh"

namespace {

constexpr int kT = 1024;

__device__ double block_sum(double v, double* sh) {
  for (int o = 16; o > 0; o >>= 1) v += __shfl_down_sync(0xffffffffu, v, o);
  const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
  if (l == 0) sh[w] = v;
  __syncthreads();
  v = threadIdx.x < (blockDim.x >> 5) ? sh[threadIdx.x] : 0.0;
  if (w == 0)
    for (int o = 16; o > 0; o >>= 1) v += __shfl_down_sync(0xffffffffu, v, o);
  return v;
}

__global__ void __launch_bounds__(kT) k_half_sqdist(int n, const double* __restrict__ q,
                                                    const double* __restrict__ ref, double* out) {
  __shared__ double sh[32];
  hdk::pdl_wait();
  double s = 0;
  for (int i = threadIdx.x; i < n; i += kT) {
    const double d = q[i] - ref[i];
    s += d * d;
  }
  s = block_sum(s, sh);
  if (threadIdx.x == 0) *out = 0.5 * s;
  hdk::pdl_trigger();
}

// out[0] = sum_s loss[s]; out[1 + i] = sum_s vec[s][i], summed in sample order.
__global__ void k_batch_sum(int samples, int n, const double* const* __restrict__ vec,
                            const double* __restrict__ loss, double* __restrict__ out) {
  hdk::pdl_wait();
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i == 0) {
    double l = 0;
    for (int s = 0; s < samples; ++s) l += loss[s];
    out[0] = l;
  }
  if (i < n) {
    double a = 0;
    for (int s = 0; s < samples; ++s) a += vec[s][i];
    out[1 + i] = a;
  }
  hdk::pdl_trigger();
}

cudaStream_t S(void* s) { return static_cast<cudaStream_t>(s); }
int last() { return static_cast<int>(cudaGetLastError()); }

}  // namespace

HDK_API int hdk_half_sqdist(int n, const double* q, const double* ref, double* out, void* stream) {
  hdk::launch(k_half_sqdist, dim3(1), dim3(kT), 0, S(stream), n, q, ref, out);
  return last();
}

HDK_API int hdk_batch_sum(int samples, int n, const double* const* vec, const double* loss, double* out,
                          void* stream) {
  hdk::launch(k_batch_sum, dim3((n + 255) / 256 > 0 ? (n + 255) / 256 : 1), dim3(256), 0, S(stream), samples, n, vec,
              loss, out);
  return last();
}
