// Values of the explicit inverse factor S' = D^{-1/2} L^{-1} on the device
// (the host build's step 5, factor.cpp; reference SparseFactor::factorize
// builds S column by column, factor.cpp:11-104).  Column c of L^{-1} lives on
// c's path to the root of the elimination tree; walking up that path, the
// value at node v is final when v is reached and is then scattered, through
// L(:, v), into v's ancestors further up the same path.  One warp per column
// with the path's values in shared memory (indexed by distance from c, so
// L's entries carry their depth distance instead of a row index); the walk
// and every subtraction run in the host loop's order, so the values are
// bitwise the host's.  Each value lands directly at its place in the
// tile-major stream the solve passes read.
#include <cuda_runtime.h>

#include "../../include/hdk.h"
#include "launch.cuh"

namespace {

__global__ void k_inverse_values(hdk_inverse_build b, int per_block, double* __restrict__ stream) {
  extern __shared__ double smem[];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int c = blockIdx.x * per_block + warp;
  if (c >= b.n) return;
  const int slot = b.max_depth + 1;
  double* work = smem + (size_t)warp * slot;
  const int len = b.depth[c] + 1;
  for (int k = lane; k < len; k += 32) work[k] = 0.0;
  __syncwarp();
  if (lane == 0) work[0] = 1.0;
  __syncwarp();
  const int tile_c = c / b.tile_w;
  int v = c;
  for (int k = 0; k < len; ++k) {
    const double xv = work[k];
    const int vnext = b.parent[v];
    if (lane == 0) {
      const int pslot = b.row_pslot[v] + (tile_c - b.row_first[v] / b.tile_w);
      stream[b.seg_off[pslot] + (c - b.seg_clo[pslot])] = __dmul_rn(xv, b.dis[v]);
    }
    if (xv != 0.0) {
      const long long p1 = b.lp[v + 1];
      for (long long p = b.lp[v] + lane; p < p1; p += 32)  // no FMA contraction: the host loop rounds twice
        work[k + b.ldist[p]] = __dsub_rn(work[k + b.ldist[p]], __dmul_rn(b.lx[p], xv));
    }
    __syncwarp();
    v = vnext;
  }
}

}  // namespace

extern "C" {

HDK_API int hdk_inverse_values(const hdk_inverse_build* b, double* stream, void* stream_handle) {
  if (b->n <= 0) return 0;
  const size_t slot = sizeof(double) * static_cast<size_t>(b->max_depth + 1);
  int per_block = 8;
  while (per_block > 1 && per_block * slot > 200 * 1024) per_block /= 2;
  if (per_block * slot > 220 * 1024) return static_cast<int>(cudaErrorInvalidValue);  // elimination tree too deep
  const size_t smem = per_block * slot;
  cudaFuncSetAttribute(k_inverse_values, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem));
  const int blocks = (b->n + per_block - 1) / per_block;
  k_inverse_values<<<blocks, 32 * per_block, smem, static_cast<cudaStream_t>(stream_handle)>>>(*b, per_block, stream);
  return static_cast<int>(cudaGetLastError());
}

}  // extern "C"
