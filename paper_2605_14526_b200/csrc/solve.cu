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
//   pass 1 (row dots):  z_r = S'(r,:) . b     warp per segment, b tile in smem
//   reduce 1:           z_r = sum over the row's tile segments (fixed order)
//   pass 2 (col tiles): x_c = sum_r S'(r,c) z_r   thread per column, z broadcast
//   reduce 2:           x_c = sum over the tile's work units (fixed order),
//                        scattered to the full xyz-interleaved vector
// Every sum has a fixed order, so results are bitwise reproducible.
#include <cuda_runtime.h>

#include "../../include/hdk.h"

namespace {

constexpr int kP1Threads = 256;

__global__ void __launch_bounds__(kP1Threads) k_rowdot(hdk_factor f, const double* __restrict__ rhs) {
  extern __shared__ double vs[];  // [3][tile_w]
  const int u = blockIdx.x;
  const int t = f.unit_tile[u];
  const int W = f.tile_w;
  const int c0 = t * W;
  const int cw = min(W, f.n - c0);
  for (int i = threadIdx.x; i < cw; i += blockDim.x) {
    const double* src = rhs + 3 * (size_t)(c0 + i);
    vs[i] = src[0];
    vs[W + i] = src[1];
    vs[2 * W + i] = src[2];
  }
  __syncthreads();
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int s_end = f.unit_seg[u + 1];
  for (int s = f.unit_seg[u] + warp; s < s_end; s += kP1Threads / 32) {
    const hdk_seg sg = f.seg[s];
    const double* __restrict__ val = f.sval + sg.off;
    const int lo = sg.clo - c0;
    double a0 = 0.0, a1 = 0.0, a2 = 0.0;
    int i = lane;
    for (; i + 96 < sg.len; i += 128) {
      const double w0 = __ldg(val + i), w1 = __ldg(val + i + 32), w2 = __ldg(val + i + 64), w3 = __ldg(val + i + 96);
      const int c = lo + i;
      a0 += w0 * vs[c] + w1 * vs[c + 32] + w2 * vs[c + 64] + w3 * vs[c + 96];
      a1 += w0 * vs[W + c] + w1 * vs[W + c + 32] + w2 * vs[W + c + 64] + w3 * vs[W + c + 96];
      a2 += w0 * vs[2 * W + c] + w1 * vs[2 * W + c + 32] + w2 * vs[2 * W + c + 64] + w3 * vs[2 * W + c + 96];
    }
    for (; i < sg.len; i += 32) {
      const double w0 = __ldg(val + i);
      const int c = lo + i;
      a0 += w0 * vs[c];
      a1 += w0 * vs[W + c];
      a2 += w0 * vs[2 * W + c];
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      a0 += __shfl_down_sync(0xffffffffu, a0, o);
      a1 += __shfl_down_sync(0xffffffffu, a1, o);
      a2 += __shfl_down_sync(0xffffffffu, a2, o);
    }
    if (lane == 0) {
      double* p = f.part1 + 3 * (size_t)sg.pslot;
      p[0] = a0;
      p[1] = a1;
      p[2] = a2;
    }
  }
}

__global__ void k_zreduce(hdk_factor f) {
  const int r = blockIdx.x * blockDim.x + threadIdx.x;
  if (r >= f.n) return;
  double a0 = 0.0, a1 = 0.0, a2 = 0.0;
  const int e = f.row_pslot[r + 1];
  for (int s = f.row_pslot[r]; s < e; ++s) {
    const double* p = f.part1 + 3 * (size_t)s;
    a0 += p[0];
    a1 += p[1];
    a2 += p[2];
  }
  double* z = f.z + 3 * (size_t)r;
  z[0] = a0;
  z[1] = a1;
  z[2] = a2;
}

constexpr int kUnroll = 4;

__global__ void __launch_bounds__(256) k_coltile(hdk_factor f) {
  const int u = blockIdx.x;
  const int t = f.unit_tile[u];
  const int W = f.tile_w;
  const int c = t * W + threadIdx.x;  // global column owned by this thread
  double a0 = 0.0, a1 = 0.0, a2 = 0.0;
  const int s_beg = f.unit_seg[u], s_end = f.unit_seg[u + 1];
  int s = s_beg;
  for (; s + kUnroll <= s_end; s += kUnroll) {
    double w[kUnroll];
    int row[kUnroll];
#pragma unroll
    for (int k = 0; k < kUnroll; ++k) {
      const hdk_seg sg = f.seg[s + k];
      const int d = c - sg.clo;
      row[k] = sg.row;
      w[k] = (d >= 0 && d < sg.len) ? __ldg(f.sval + sg.off + d) : 0.0;
    }
#pragma unroll
    for (int k = 0; k < kUnroll; ++k) {
      const double* z = f.z + 3 * (size_t)row[k];
      a0 += w[k] * z[0];
      a1 += w[k] * z[1];
      a2 += w[k] * z[2];
    }
  }
  for (; s < s_end; ++s) {
    const hdk_seg sg = f.seg[s];
    const int d = c - sg.clo;
    if (d >= 0 && d < sg.len) {
      const double w = __ldg(f.sval + sg.off + d);
      const double* z = f.z + 3 * (size_t)sg.row;
      a0 += w * z[0];
      a1 += w * z[1];
      a2 += w * z[2];
    }
  }
  double* p = f.part2 + 3 * ((size_t)u * W + threadIdx.x);
  p[0] = a0;
  p[1] = a1;
  p[2] = a2;
}

template <bool kScatter>
__global__ void k_xreduce(hdk_factor f, double* __restrict__ out) {
  const int c = blockIdx.x * blockDim.x + threadIdx.x;
  if (c >= f.n) return;
  const int W = f.tile_w;
  const int t = c / W, cl = c - t * W;
  double a0 = 0.0, a1 = 0.0, a2 = 0.0;
  const int ue = f.tile_unit[t + 1];
  for (int u = f.tile_unit[t]; u < ue; ++u) {
    const double* p = f.part2 + 3 * ((size_t)u * W + cl);
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
  const size_t smem = 3 * sizeof(double) * (size_t)f->tile_w;
  k_rowdot<<<f->n_units, kP1Threads, smem, st>>>(*f, rhs_perm);
  k_zreduce<<<(f->n + 255) / 256, 256, 0, st>>>(*f);
  k_coltile<<<f->n_units, f->tile_w, 0, st>>>(*f);
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
