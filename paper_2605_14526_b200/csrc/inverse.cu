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

#include <algorithm>

#include "../../include/hdk.h"
#include "launch.cuh"

namespace {

// Per step the walk's latency chain is parent -> lp -> (lx, ldist) -> the
// shared update, plus row_pslot -> seg_off for the value's place.  None of
// those loads depends on the work values, so they run ahead of the walk:
// node k+1's first 64 entries and destination, and node k+2's column range,
// are issued while node k is updated.  Within a step every entry of L(:, v)
// hits a distinct work slot, so the entries may be applied in any order; the
// walk itself stays in the host loop's order (bitwise the host values).
constexpr int kPre = 2;  // prefetched 32-entry chunks per node
constexpr int kBatch = 4;  // chunks per batch of loads beyond the prefetch

struct Chunk {
  double x[kPre];
  int d[kPre];
};

__device__ __forceinline__ void load_chunk(const hdk_inverse_build& b, long long pb, long long pe, int lane,
                                           Chunk& ch) {
#pragma unroll
  for (int u = 0; u < kPre; ++u) {
    const long long p = pb + 32 * u + lane;
    const bool in = p < pe;
    ch.x[u] = in ? __ldg(b.lx + p) : 0.0;
    ch.d[u] = in ? __ldg(b.ldist + p) : 0;
  }
}

__global__ void k_inverse_values(hdk_inverse_build b, int per_block, double* __restrict__ stream) {
  extern __shared__ double smem[];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int c = blockIdx.x * per_block + warp;
  if (c >= b.n) return;
  const int slot = b.max_depth + 1;
  double* work = smem + (size_t)warp * slot;
  const int len = __ldg(b.depth + c) + 1;
  for (int k = lane; k < len; k += 32) work[k] = 0.0;
  __syncwarp();
  if (lane == 0) work[0] = 1.0;
  const int tile_c = c / b.tile_w;
  const auto pslot_of = [&](int v) {
    return __ldg(b.row_pslot + v) + (tile_c - __ldg(b.row_first + v) / b.tile_w);
  };
  // node k (= c): range, first chunks, destination, D^{-1/2}
  long long pb0 = __ldg(b.lp + c), pe0 = __ldg(b.lp + c + 1);
  Chunk ch0;
  load_chunk(b, pb0, pe0, lane, ch0);
  int ps = pslot_of(c);
  long long so0 = __ldg(b.seg_off + ps);
  int sc0 = __ldg(b.seg_clo + ps);
  double dis0 = __ldg(b.dis + c);
  // node k+1: id, range, destination row data; node k+2: id
  int v1 = __ldg(b.parent + c);
  long long pb1 = 0, pe1 = 0;
  int rp1 = 0;
  double dis1 = 0.0;
  int v2 = -1;
  if (v1 >= 0) {
    pb1 = __ldg(b.lp + v1);
    pe1 = __ldg(b.lp + v1 + 1);
    rp1 = pslot_of(v1);
    dis1 = __ldg(b.dis + v1);
    v2 = __ldg(b.parent + v1);
  }
  __syncwarp();
  for (int k = 0; k < len; ++k) {
    // run ahead: node k+1's chunks and destination, node k+2's range and row data
    Chunk ch1;
    load_chunk(b, pb1, pe1, lane, ch1);
    long long so1 = 0;
    int sc1 = 0;
    if (v1 >= 0) {
      so1 = __ldg(b.seg_off + rp1);
      sc1 = __ldg(b.seg_clo + rp1);
    }
    long long pb2 = 0, pe2 = 0;
    int rp2 = 0, v3 = -1;
    double dis2 = 0.0;
    if (v2 >= 0) {
      pb2 = __ldg(b.lp + v2);
      pe2 = __ldg(b.lp + v2 + 1);
      rp2 = pslot_of(v2);
      dis2 = __ldg(b.dis + v2);
      v3 = __ldg(b.parent + v2);
    }
    // node k
    const double xv = work[k];
    if (xv != 0.0) {  // no FMA contraction: the host loop rounds twice
#pragma unroll
      for (int u = 0; u < kPre; ++u)
        if (pb0 + 32 * u + lane < pe0) work[k + ch0.d[u]] = __dsub_rn(work[k + ch0.d[u]], __dmul_rn(ch0.x[u], xv));
      for (long long p = pb0 + 32 * kPre + lane; p < pe0; p += 32 * kBatch) {
        double x[kBatch];
        int d[kBatch];
#pragma unroll
        for (int u = 0; u < kBatch; ++u) {
          const bool in = p + 32 * u < pe0;
          x[u] = in ? __ldg(b.lx + p + 32 * u) : 0.0;
          d[u] = in ? __ldg(b.ldist + p + 32 * u) : 0;
        }
#pragma unroll
        for (int u = 0; u < kBatch; ++u)
          if (p + 32 * u < pe0) work[k + d[u]] = __dsub_rn(work[k + d[u]], __dmul_rn(x[u], xv));
      }
    }
    if (lane == 0) stream[so0 + (c - sc0)] = __dmul_rn(xv, dis0);
    __syncwarp();
    pb0 = pb1;
    pe0 = pe1;
    ch0 = ch1;
    so0 = so1;
    sc0 = sc1;
    dis0 = dis1;
    v1 = v2;
    pb1 = pb2;
    pe1 = pe2;
    rp1 = rp2;
    dis1 = dis2;
    v2 = v3;
  }
}

// The plain walk (loads issued when the step needs them): fewer instructions
// per step, the better form when many warps share an SM (short paths, C2 /
// the lockstep batch); the run-ahead form wins when shared memory limits
// the SM to a few columns (C3: 13.6 vs 18.8 ms; C5 64 x C2: 49 vs 45 ms).
__global__ void k_inverse_values_plain(hdk_inverse_build b, int per_block, double* __restrict__ stream) {
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
  if (slot > 220 * 1024) return static_cast<int>(cudaErrorInvalidValue);  // elimination tree too deep
  // columns per block: the most resident columns per SM (shared memory
  // bound, at most 32 blocks per SM), ties to the larger block
  constexpr size_t kSmem = 227 * 1024;
  int per_block = 1, per_sm = 0;
  for (int pb = 8; pb >= 1; pb /= 2) {
    if (pb * slot > 200 * 1024) continue;
    const int blocks_sm = static_cast<int>(std::min<size_t>(32, kSmem / (pb * slot)));
    if (pb * blocks_sm > per_sm) {
      per_sm = pb * blocks_sm;
      per_block = pb;
    }
  }
  const size_t smem = per_block * slot;
  const int blocks = (b->n + per_block - 1) / per_block;
  // few resident columns per SM -> run-ahead walk
  const auto kern = per_sm < 24 ? k_inverse_values : k_inverse_values_plain;
  cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem));
  kern<<<blocks, 32 * per_block, smem, static_cast<cudaStream_t>(stream_handle)>>>(*b, per_block, stream);
  return static_cast<int>(cudaGetLastError());
}

}  // extern "C"
