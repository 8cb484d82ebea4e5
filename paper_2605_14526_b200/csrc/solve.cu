// Global solve x = A^{-1} b = S'^T (S' b) on three right-hand sides (x, y, z)
// — the B200 replacement of SparseFactor::apply_inverse / solve_free
// (reference factor.cpp:106-109, 196-208; csr.cpp:40-47 does each of the six
// serial CSR passes there).
//
// Layout (see hdk.h): S' = D^{-1/2} L^{-1} in a postordered elimination order,
// so row r is dense over its etree subtree [r-len_r+1, r] and needs no column
// indices: 8 B per nonzero instead of the reference's 12 B, and both passes
// stream the same value array once, coalesced, for all three axes.
//
// Work decomposition: columns are cut into tiles of 256; a segment is one
// row's part inside one tile; a work unit (one CTA) is a run of segments of one
// tile with ~nnz/592 values.  Inside a CTA, lane j of every warp owns the tile
// columns j + 32 m (m = 0..7), so the right-hand side (pass 1) or the
// accumulators (pass 2) of a whole tile live in 24 registers per lane, every
// segment read is a coalesced 256-byte row slice, and the segment descriptors
// are staged once in shared memory.
//
//   pass 1  k_rowdot   partial z_{r,t} = S'(r, tile t) . b_t   (warp per segment)
//   reduce  k_zreduce  z_r = sum_t z_{r,t}                     (warp per row, fixed order)
//   pass 2  k_coltile  x_t += S'(r, tile t)^T z_r               (warp-private accumulators,
//                                                               fixed-order CTA fold)
//   reduce  k_xreduce  x_c = sum over the tile's units; scatter to xyz-interleaved
// Every sum has a fixed order, so results are bitwise reproducible.
#include <cuda_runtime.h>

#include "../../include/hdk.h"

namespace {

constexpr int kW = 256;        // tile width (columns)
constexpr int kM = kW / 32;    // columns per lane
constexpr int kWarps = 8;      // warps per CTA
constexpr int kThreads = 32 * kWarps;
constexpr int kSegSmem = 512;  // descriptors staged per chunk

struct SegS {
  long long off;
  int row, clo, len, pslot;
};

__device__ __forceinline__ void stage_segments(const hdk_seg* __restrict__ g, int s0, int n, SegS* sm) {
  for (int i = threadIdx.x; i < n; i += blockDim.x) {
    const hdk_seg s = g[s0 + i];
    sm[i].off = s.off;
    sm[i].row = s.row;
    sm[i].clo = s.clo;
    sm[i].len = s.len;
    sm[i].pslot = s.pslot;
  }
}

__global__ void __launch_bounds__(kThreads) k_rowdot(hdk_factor f, const double* __restrict__ rhs) {
  __shared__ SegS ss[kSegSmem];
  const int u = blockIdx.x;
  const int c0 = f.unit_tile[u] * kW;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  // right-hand side of the tile in registers: lane owns columns c0 + lane + 32 m
  double b0[kM], b1[kM], b2[kM];
#pragma unroll
  for (int m = 0; m < kM; ++m) {
    const int c = c0 + lane + 32 * m;
    const bool ok = c < f.n;
    b0[m] = ok ? __ldg(rhs + 3 * (size_t)c) : 0.0;
    b1[m] = ok ? __ldg(rhs + 3 * (size_t)c + 1) : 0.0;
    b2[m] = ok ? __ldg(rhs + 3 * (size_t)c + 2) : 0.0;
  }
  const int s_beg = f.unit_seg[u], s_end = f.unit_seg[u + 1];
  for (int base = s_beg; base < s_end; base += kSegSmem) {
    const int cnt = min(kSegSmem, s_end - base);
    __syncthreads();
    stage_segments(f.seg, base, cnt, ss);
    __syncthreads();
    for (int i = warp; i < cnt; i += kWarps) {
      const SegS sg = ss[i];
      const double* __restrict__ val = f.sval + sg.off - (sg.clo - c0);  // val[c - c0] = S'(row, c)
      const int lo = sg.clo - c0, hi = lo + sg.len;
      double a0 = 0.0, a1 = 0.0, a2 = 0.0;
#pragma unroll
      for (int m = 0; m < kM; ++m) {
        const int cl = lane + 32 * m;
        if (cl >= lo && cl < hi) {
          const double w = __ldg(val + cl);
          a0 += w * b0[m];
          a1 += w * b1[m];
          a2 += w * b2[m];
        }
      }
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) {
        a0 += __shfl_xor_sync(0xffffffffu, a0, o);
        a1 += __shfl_xor_sync(0xffffffffu, a1, o);
        a2 += __shfl_xor_sync(0xffffffffu, a2, o);
      }
      if (lane == 0) {
        double* p = f.part1 + 3 * (size_t)sg.pslot;
        p[0] = a0;
        p[1] = a1;
        p[2] = a2;
      }
    }
  }
}

// z_r = sum of the row's tile partials in tile order; one warp per row.
__global__ void __launch_bounds__(256) k_zreduce(hdk_factor f) {
  const int r = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (r >= f.n) return;
  const int s0 = f.row_pslot[r], s1 = f.row_pslot[r + 1];
  double a0 = 0.0, a1 = 0.0, a2 = 0.0;
  for (int s = s0 + lane; s < s1; s += 32) {
    const double* p = f.part1 + 3 * (size_t)s;
    a0 += p[0];
    a1 += p[1];
    a2 += p[2];
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    a0 += __shfl_xor_sync(0xffffffffu, a0, o);
    a1 += __shfl_xor_sync(0xffffffffu, a1, o);
    a2 += __shfl_xor_sync(0xffffffffu, a2, o);
  }
  if (lane == 0) {
    double* z = f.z + 3 * (size_t)r;
    z[0] = a0;
    z[1] = a1;
    z[2] = a2;
  }
}

__global__ void __launch_bounds__(kThreads) k_coltile(hdk_factor f) {
  __shared__ SegS ss[kSegSmem];
  __shared__ double fold[kWarps / 2][3][kW];  // cross-warp fold, two rounds
  const int u = blockIdx.x;
  const int c0 = f.unit_tile[u] * kW;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  double x0[kM], x1[kM], x2[kM];
#pragma unroll
  for (int m = 0; m < kM; ++m) x0[m] = x1[m] = x2[m] = 0.0;
  const int s_beg = f.unit_seg[u], s_end = f.unit_seg[u + 1];
  for (int base = s_beg; base < s_end; base += kSegSmem) {
    const int cnt = min(kSegSmem, s_end - base);
    __syncthreads();
    stage_segments(f.seg, base, cnt, ss);
    __syncthreads();
    int i = warp;
    // two segments per iteration for memory-level parallelism
    for (; i + kWarps < cnt; i += 2 * kWarps) {
      const SegS sa = ss[i], sb = ss[i + kWarps];
      const double* __restrict__ va = f.sval + sa.off - (sa.clo - c0);
      const double* __restrict__ vb = f.sval + sb.off - (sb.clo - c0);
      const int la = sa.clo - c0, ha = la + sa.len, lb = sb.clo - c0, hb = lb + sb.len;
      const double* za = f.z + 3 * (size_t)sa.row;
      const double* zb = f.z + 3 * (size_t)sb.row;
      double wa[kM], wb[kM];
#pragma unroll
      for (int m = 0; m < kM; ++m) {
        const int cl = lane + 32 * m;
        wa[m] = (cl >= la && cl < ha) ? __ldg(va + cl) : 0.0;
        wb[m] = (cl >= lb && cl < hb) ? __ldg(vb + cl) : 0.0;
      }
      const double za0 = __ldg(za), za1 = __ldg(za + 1), za2 = __ldg(za + 2);
      const double zb0 = __ldg(zb), zb1 = __ldg(zb + 1), zb2 = __ldg(zb + 2);
#pragma unroll
      for (int m = 0; m < kM; ++m) {
        x0[m] += wa[m] * za0;
        x1[m] += wa[m] * za1;
        x2[m] += wa[m] * za2;
        x0[m] += wb[m] * zb0;
        x1[m] += wb[m] * zb1;
        x2[m] += wb[m] * zb2;
      }
    }
    for (; i < cnt; i += kWarps) {
      const SegS sa = ss[i];
      const double* __restrict__ va = f.sval + sa.off - (sa.clo - c0);
      const int la = sa.clo - c0, ha = la + sa.len;
      const double* za = f.z + 3 * (size_t)sa.row;
      const double za0 = __ldg(za), za1 = __ldg(za + 1), za2 = __ldg(za + 2);
#pragma unroll
      for (int m = 0; m < kM; ++m) {
        const int cl = lane + 32 * m;
        const double w = (cl >= la && cl < ha) ? __ldg(va + cl) : 0.0;
        x0[m] += w * za0;
        x1[m] += w * za1;
        x2[m] += w * za2;
      }
    }
  }
  // fixed-order fold of the 8 warp-private accumulators: warps 4..7 park,
  // 0..3 add; then 2..3 park, 0..1 add; then 1 parks, 0 adds and writes.
  __syncthreads();
#pragma unroll
  for (int half = kWarps / 2; half >= 1; half >>= 1) {
    if (warp >= half && warp < 2 * half) {
#pragma unroll
      for (int m = 0; m < kM; ++m) {
        const int cl = lane + 32 * m;
        fold[warp - half][0][cl] = x0[m];
        fold[warp - half][1][cl] = x1[m];
        fold[warp - half][2][cl] = x2[m];
      }
    }
    __syncthreads();
    if (warp < half) {
#pragma unroll
      for (int m = 0; m < kM; ++m) {
        const int cl = lane + 32 * m;
        x0[m] += fold[warp][0][cl];
        x1[m] += fold[warp][1][cl];
        x2[m] += fold[warp][2][cl];
      }
    }
    __syncthreads();
  }
  if (warp == 0) {
#pragma unroll
    for (int m = 0; m < kM; ++m) {
      double* p = f.part2 + 3 * ((size_t)u * kW + lane + 32 * m);
      p[0] = x0[m];
      p[1] = x1[m];
      p[2] = x2[m];
    }
  }
}

template <bool kScatter>
__global__ void k_xreduce(hdk_factor f, double* __restrict__ out) {
  const int c = blockIdx.x * blockDim.x + threadIdx.x;
  if (c >= f.n) return;
  const int t = c / kW, cl = c - t * kW;
  double a0 = 0.0, a1 = 0.0, a2 = 0.0;
  const int ue = f.tile_unit[t + 1];
  for (int u = f.tile_unit[t]; u < ue; ++u) {
    const double* p = f.part2 + 3 * ((size_t)u * kW + cl);
    a0 += p[0];
    a1 += p[1];
    a2 += p[2];
  }
  double* o = kScatter ? out + 3 * (size_t)f.p2v[c] : out + 3 * (size_t)c;
  o[0] = a0;
  o[1] = a1;
  o[2] = a2;
}

int launch(const hdk_factor* f, const double* rhs_perm, double* out, bool scatter, cudaStream_t st) {
  if (f->n <= 0) return 0;
  if (f->tile_w != kW) return static_cast<int>(cudaErrorInvalidValue);
  k_rowdot<<<f->n_units, kThreads, 0, st>>>(*f, rhs_perm);
  k_zreduce<<<(f->n * 32 + 255) / 256, 256, 0, st>>>(*f);
  k_coltile<<<f->n_units, kThreads, 0, st>>>(*f);
  if (scatter)
    k_xreduce<true><<<(f->n + 255) / 256, 256, 0, st>>>(*f, out);
  else
    k_xreduce<false><<<(f->n + 255) / 256, 256, 0, st>>>(*f, out);
  return static_cast<int>(cudaGetLastError());
}

}  // namespace

extern "C" {

HDK_API int hdk_apply_inverse3(const hdk_factor* f, const double* rhs_perm, double* out_full, void* stream) {
  return launch(f, rhs_perm, out_full, true, static_cast<cudaStream_t>(stream));
}

HDK_API int hdk_apply_inverse3_perm(const hdk_factor* f, const double* rhs_perm, double* out_perm, void* stream) {
  return launch(f, rhs_perm, out_perm, false, static_cast<cudaStream_t>(stream));
}

}  // extern "C"
