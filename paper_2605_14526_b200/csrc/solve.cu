// Global solve x = A^{-1} b = S'^T (S' b) on three right-hand sides (x, y, z)
// — the B200 replacement of SparseFactor::apply_inverse / solve_free
// (reference factor.cpp:106-109, 196-208; csr.cpp:40-47 does each of the six
// serial CSR passes there).
//
// Layout (hdk.h): S' = D^{-1/2} L^{-1} in a postordered elimination order, so
// row r is dense over its etree subtree and needs no column indices (8 B per
// nonzero instead of the reference's 12 B).  Values are stored tile-major as
// one stream of 16-byte aligned chunks (whole row segments of one 256-column
// tile), so each pass is a pure stream: persistent CTA b owns the contiguous
// chunk range [b C / G, (b+1) C / G) and a single elected thread keeps a ring
// of kStages chunks in flight with
// bulk asynchronous copies (cp.async.bulk, the TMA engine's 1-D mode) that
// complete on mbarriers, while 8 warps consume the chunk in shared memory.
// Lane j owns the tile columns j + 32 m (m = 0..7): the right-hand side
// (pass 1) or the accumulators (pass 2) of a tile live in 24 registers.
//
//   pass 1  k_rowdot   partial z_{r,t} = S'(r, tile t) . b_t   (warp per segment)
//   reduce  k_zreduce  z_r = sum_t z_{r,t}                     (warp per row, fixed order)
//   pass 2  k_coltile  x_t += S'(r, tile t)^T z_r               (warp-private accumulators,
//                                                               fixed-order CTA fold per tile)
//   reduce  k_xreduce  x_c = sum over the CTAs that touched the tile; scatter
// Work assignment and every sum are fixed, so results are bitwise reproducible.
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdlib>

#include "../../include/hdk.h"
#include "launch.cuh"

HDK_TRACE_TU(solve)

namespace {

constexpr int kW = 256;       // tile width (columns)
constexpr int kM = kW / 32;   // columns per lane
constexpr int kWarps = 8;     // consumer warps
constexpr int kThreads = 32 * (kWarps + 1);  // + one producer warp
constexpr int kVals = HDK_CHUNK_VALS;
constexpr int kSegs = HDK_CHUNK_SEGS;
#ifndef HDK_STAGES1
#define HDK_STAGES1 3
#endif
#ifndef HDK_STAGES2
#define HDK_STAGES2 5
#endif
constexpr int kStages1 = HDK_STAGES1;   // pass 1 ring depth (2 CTAs / SM)
// Pass 1 with W consumer warps: W = 8 runs 2 CTAs per SM with a 3-stage ring;
// W = 16 (multi-column passes, which are compute-bound) 1 CTA per SM, 6 stages.
template <int W>
struct Pass1 {
  static constexpr int threads = 32 * (W + 1), min_blocks = W == 8 ? 2 : 1, stages = W == 8 ? kStages1 : 6;
};
constexpr int kStages2 = HDK_STAGES2;   // pass 2 ring depth (1 CTA / SM)
constexpr int kThreads2 = 32 * (kWarps + 2);  // pass 2: + copy warp + z-gather warp

static_assert(kW == 256, "tile width is fixed by the factor layout");

// ---- bulk-copy / mbarrier primitives (PTX) ----------------------------------
__device__ __forceinline__ uint32_t smem_addr(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_addr(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_fence_init() { asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory"); }
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_addr(bar)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_addr(bar)) : "memory");
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(smem_addr(dst)),
      "l"(src), "r"(bytes), "r"(smem_addr(bar))
      : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "WAIT_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      "@!p bra WAIT_%=;\n"
      "}\n" ::"r"(smem_addr(bar)),
      "r"(parity)
      : "memory");
}
// Same, with an L2 eviction-priority policy (createpolicy): the factor stream
// is marked evict_first so the once-per-pass values do not push the vectors,
// partials and the adjoint's element differentials out of L2.
__device__ __forceinline__ uint64_t policy_evict_first() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
  return p;
}
__device__ __forceinline__ void bulk_g2s_hint(void* dst, const void* src, uint32_t bytes, uint64_t* bar, uint64_t pol) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], %4;" ::"r"(
          smem_addr(dst)),
      "l"(src), "r"(bytes), "r"(smem_addr(bar)), "l"(pol)
      : "memory");
}
// 8-byte asynchronous global->shared copy (LDGSTS); completion is tracked by
// cp_async_arrive on an mbarrier.
__device__ __forceinline__ void cp_async8(void* dst, const void* src) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(smem_addr(dst)), "l"(src) : "memory");
}
// The mbarrier receives one arrival once all of this thread's prior cp.async
// copies have landed (pending count not incremented: count them at init).
__device__ __forceinline__ void cp_async_arrive(uint64_t* bar) {
  asm volatile("cp.async.mbarrier.arrive.noinc.shared::cta.b64 [%0];" ::"r"(smem_addr(bar)) : "memory");
}
__device__ __forceinline__ void fence_proxy_async() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }
__device__ __forceinline__ void consumers_sync() { asm volatile("bar.sync 1, %0;" ::"n"(32 * kWarps) : "memory"); }

// Per-chunk ring trace of the multi-column passes (profiling; set by
// hdk_set_chunk_trace, null otherwise): for chunk c, [4c] the producer's
// clock when it could issue (before its empty wait), [4c + 1] when it
// issued, [4c + 2] when the consumers saw it land, [4c + 3] when its last
// worker finished (SM-local clock64).
__device__ long long* g_chunk_trace = nullptr;
__device__ __forceinline__ long long sm_clock() { return clock64(); }

// Per-CTA timing trace, compiled only into microbenchmarks that define
// HDK_SOLVE_TRACE: [2 b] = start, [2 b + 1] = end (globaltimer, ns) of CTA b.
#ifdef HDK_SOLVE_TRACE
__device__ unsigned long long* g_cta_trace = nullptr;
#define HDK_TRACE_PTR g_cta_trace
#else
#define HDK_TRACE_PTR static_cast<unsigned long long*>(nullptr)
#endif
__device__ __forceinline__ unsigned long long globaltimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}

// z-fold by warp tasks (host-built, hdk_factor::ztask): a task is either one
// long row (more than 8 tile partials: the separator rows at the top of the
// elimination tree, up to n/256 partials) folded by a whole warp, or up to
// four consecutive short rows folded by eight lanes each.  Every lane issues
// all of its loads before adding, so a task costs one L2 round trip, and
// tasks are equal-cost, so warps stay balanced (a row-per-8-lanes split left
// the few long rows as a 4x longer tail).  Fixed lane split and shuffle
// tree: bitwise reproducible.
constexpr int kZLong = 3;  // partials per lane held in flight (long rows up to 96 partials per round)
// A z-fold warp task's rows and partial-slot ranges: static (the factor's
// layout), so k_zreduce reads them before its PDL wait.
struct ZRows {
  int r, stride, s0, s1;
  bool writer;
};
__device__ __forceinline__ ZRows zfold_rows(const hdk_factor& f, int2 task) {
  const int lane = threadIdx.x & 31;
  ZRows z;
  if (task.y < 0) {  // long row: 32 lanes
    z.r = task.x;
    z.stride = 32;
    z.writer = lane == 0;
  } else {  // short rows: 8 lanes per row
    z.r = task.x + (lane >> 3);
    z.stride = 8;
    z.writer = (lane & 7) == 0 && (lane >> 3) < task.y;
  }
  const bool live = task.y < 0 || (lane >> 3) < task.y;
  z.s0 = live ? __ldg(f.row_pslot + z.r) : 0;
  z.s1 = live ? __ldg(f.row_pslot + z.r + 1) : 0;
  return z;
}

__device__ __forceinline__ void zfold_task(const hdk_factor& f, const ZRows& zr, int column) {
  const int lane = threadIdx.x & 31;
  const double* part1 = f.part1 + (size_t)column * 3 * (size_t)f.n_pslot;
  double* zc = f.z + (size_t)column * 3 * (size_t)f.n;
  double a0 = 0.0, a1 = 0.0, a2 = 0.0;
  const int r = zr.r, stride = zr.stride, s0 = zr.s0, s1 = zr.s1;
  const bool writer = zr.writer;
  const int sub = lane & (stride - 1);
  for (int s = s0 + sub; s < s1; s += kZLong * stride) {
    double v[kZLong][3];
#pragma unroll
    for (int k = 0; k < kZLong; ++k) {
      const int sk = s + k * stride;
      const double* p = part1 + 3 * (size_t)sk;
      v[k][0] = sk < s1 ? __ldg(p) : 0.0;
      v[k][1] = sk < s1 ? __ldg(p + 1) : 0.0;
      v[k][2] = sk < s1 ? __ldg(p + 2) : 0.0;
    }
#pragma unroll
    for (int k = 0; k < kZLong; ++k) {
      a0 += v[k][0];
      a1 += v[k][1];
      a2 += v[k][2];
    }
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    if (o >= stride) continue;
    a0 += __shfl_xor_sync(0xffffffffu, a0, o);
    a1 += __shfl_xor_sync(0xffffffffu, a1, o);
    a2 += __shfl_xor_sync(0xffffffffu, a2, o);
  }
  if (writer) {
    double* z = zc + 3 * (size_t)r;
    z[0] = a0;
    z[1] = a1;
    z[2] = a2;
  }
}

// Multi-column solves (hdk_apply_inverse3_multi): R independent 3-vector
// right-hand sides share one stream of the factor.  Column c's rhs / z live at
// +c * 3n, its row partials at +c * 3 * n_pslot, its tile partials at
// +c * part2_stride(f).
__host__ __device__ __forceinline__ size_t part2_stride(const hdk_factor& f) {
  return 3 * (size_t)f.tile_w * (size_t)(f.n_tiles + f.max_ctas);
}

// Balanced contiguous chunk ranges: CTA b of G owns [first(b), first(b+1)).
__device__ __forceinline__ int range_first(long long b, int G, int C) { return static_cast<int>(b * C / G); }
// The CTA owning chunk c (G <= C, so no range is empty).
__device__ __forceinline__ int cta_of(long long c, int G, int C) {
  return static_cast<int>(((c + 1) * G + C - 1) / C) - 1;
}

struct ChunkInfo {
  int nseg, tile, seg0, pad;
};

template <int S, typename V = double>
struct Ring {
  V vals[S][kVals];
  hdk_seg segs[S][kSegs];
  ChunkInfo info[S];  // written by the producer before its arrive (release)
  uint64_t full[S];
  uint64_t empty[S];
};

template <int S, typename V>
__device__ __forceinline__ void ring_init(Ring<S, V>& r, int consumers = kWarps) {
  if (threadIdx.x == 0) {
    for (int s = 0; s < S; ++s) {
      mbar_init(&r.full[s], 1);
      mbar_init(&r.empty[s], consumers);
    }
    mbar_fence_init();
  }
  __syncthreads();
}

// Producer warp (one elected lane): keeps S chunks in flight; a stage is
// refilled once all consumer warps have released it.
// The first min(S, n) chunks are requested before the kernel's PDL wait: the
// factor stream does not depend on the previous kernel, so the ring fills
// while that kernel drains.  After the wait the producer honours the run
// flag; an iteration that is skipped drains the requested stages first (no
// bulk copy may be outstanding when the CTA exits).  Returns false if skipped.
template <int S, class FullBars>
__device__ __forceinline__ bool after_prefill(const hdk_factor& f, FullBars& full, int issued) {
  hdk::pdl_wait();
  if (f.run_flag && *f.run_flag == 0) {
    for (int k = 0; k < issued; ++k) mbar_wait(&full[k % S], 0);
    return false;
  }
  return true;
}

// The value stream a pass reads: fp64 (exact solves) or the fp32 copy
// (preconditioner-only solves, hdk_factor::use32), with its chunk table.
template <typename V>
__device__ __forceinline__ const V* value_stream(const hdk_factor& f);
template <>
__device__ __forceinline__ const double* value_stream<double>(const hdk_factor& f) { return f.sval; }
template <>
__device__ __forceinline__ const float* value_stream<float>(const hdk_factor& f) { return f.sval32; }
template <typename V>
__device__ __forceinline__ const hdk_chunk* chunk_table(const hdk_factor& f) {
  return sizeof(V) == 8 ? f.chunk : f.chunk32;
}

template <int S, typename V>
__device__ __forceinline__ void produce(const hdk_factor& f, Ring<S, V>& r, int c_beg, int c_end, bool reverse) {
  if ((threadIdx.x & 31) != 0) return;
  const int n = c_end - c_beg;
  auto chunk_at = [&](int k) { return reverse ? c_end - 1 - k : c_beg + k; };
  const hdk_chunk* ctab = chunk_table<V>(f);
  const V* vsrc = value_stream<V>(f);
  hdk_chunk nxt = n > 0 ? ctab[chunk_at(0)] : hdk_chunk{};
  const uint64_t pol = policy_evict_first();
  const int pre = n < S ? n : S;
  if (pre == 0 && !after_prefill<S>(f, r.full, 0)) return;
  for (int k = 0; k < n; ++k) {
    if (k == pre && !after_prefill<S>(f, r.full, pre)) return;
    const int st = k % S;
    const hdk_chunk ch = nxt;
    if (k + 1 < n) nxt = ctab[chunk_at(k + 1)];  // descriptor prefetch, off the critical path
    long long* tr = g_chunk_trace;
    const long long t_ready = tr ? sm_clock() : 0;
    if (k >= S) mbar_wait(&r.empty[st], ((k / S) - 1) & 1);
    if (tr && k >= S) {  // (the prefilled chunks are not traced: they are issued before the run flag is read)
      tr[4 * (size_t)chunk_at(k)] = t_ready;
      tr[4 * (size_t)chunk_at(k) + 1] = sm_clock();
    }
    fence_proxy_async();
    r.info[st] = ChunkInfo{ch.nseg, ch.tile, ch.seg0, 0};
    const uint32_t vb = static_cast<uint32_t>(ch.len) * static_cast<uint32_t>(sizeof(V)), sb = static_cast<uint32_t>(ch.nseg) * 16u;
    mbar_expect_tx(&r.full[st], vb + sb);
    if (vb) {
      if (f.l2_hint) bulk_g2s_hint(r.vals[st], vsrc + ch.off, vb, &r.full[st], pol);
      else bulk_g2s(r.vals[st], vsrc + ch.off, vb, &r.full[st]);
    }
    bulk_g2s(r.segs[st], f.seg + ch.seg0, sb, &r.full[st]);
  }
  if (pre == n && n > 0) after_prefill<S>(f, r.full, n);
}

// Pass 2 ring: as Ring, plus the z rows of each staged chunk's segments,
// gathered into shared memory by the producer warp (zfull) so the consumers
// never wait on a global load.
template <int S, int R, typename V = double>
struct Ring2 {
  V vals[S][kVals];
  hdk_seg segs[S][kSegs];
  double zs[S][kSegs][3 * R];
  ChunkInfo info[S];
  uint64_t full[S];
  uint64_t zfull[S];
  uint64_t empty[S];
};

template <int S, int R, typename V>
__device__ __forceinline__ void ring2_init(Ring2<S, R, V>& r) {
  if (threadIdx.x == 0) {
    for (int s = 0; s < S; ++s) {
      mbar_init(&r.full[s], 1);
      mbar_init(&r.zfull[s], 32);  // one cp.async arrival per producer lane
      mbar_init(&r.empty[s], kWarps);
    }
    mbar_fence_init();
  }
  __syncthreads();
}

// Pass 2 producer warps.  Warp kWarps (lane 0) streams chunks in reverse
// order exactly as produce(); warp kWarps + 1 waits for each chunk to land and
// gathers the z rows of its segments into zs with asynchronous 8-byte copies
// that complete on zfull, so neither the stream nor the consumers wait on a
// dependent global load.
template <int S, int R, typename V>
__device__ __forceinline__ void gather_z(const hdk_factor& f, Ring2<S, R, V>& r, int n) {
  const int lane = threadIdx.x & 31;
  for (int j = 0; j < n; ++j) {
    const int st = j % S;
    mbar_wait(&r.full[st], (j / S) & 1);
    const int nseg = r.info[st].nseg;
    for (int i = lane; i < nseg; i += 32) {
      const size_t row = 3 * (size_t)r.segs[st][i].row;
#pragma unroll
      for (int c = 0; c < R; ++c) {
        const double* z = f.z + (size_t)c * 3 * (size_t)f.n + row;
        cp_async8(&r.zs[st][i][3 * c], z);
        cp_async8(&r.zs[st][i][3 * c + 1], z + 1);
        cp_async8(&r.zs[st][i][3 * c + 2], z + 2);
      }
    }
    cp_async_arrive(&r.zfull[st]);
  }
}

template <int S, int R, typename V>
__device__ __forceinline__ void stream2(const hdk_factor& f, Ring2<S, R, V>& r, int c_beg, int c_end) {
  if ((threadIdx.x & 31) != 0) return;
  const int n = c_end - c_beg;
  const hdk_chunk* ctab = chunk_table<V>(f);
  const V* vsrc = value_stream<V>(f);
  hdk_chunk nxt = n > 0 ? ctab[c_end - 1] : hdk_chunk{};
  const uint64_t pol = policy_evict_first();
  const int pre = n < S ? n : S;
  if (pre == 0 && !after_prefill<S>(f, r.full, 0)) return;
  for (int k = 0; k < n; ++k) {
    if (k == pre && !after_prefill<S>(f, r.full, pre)) return;
    const int st = k % S;
    const hdk_chunk ch = nxt;
    if (k + 1 < n) nxt = ctab[c_end - 2 - k];
    if (k >= S) mbar_wait(&r.empty[st], ((k / S) - 1) & 1);
    fence_proxy_async();
    r.info[st] = ChunkInfo{ch.nseg, ch.tile, ch.seg0, 0};
    const uint32_t vb = static_cast<uint32_t>(ch.len) * static_cast<uint32_t>(sizeof(V)), sb = static_cast<uint32_t>(ch.nseg) * 16u;
    mbar_expect_tx(&r.full[st], vb + sb);
    if (vb) {
      if (f.l2_hint) bulk_g2s_hint(r.vals[st], vsrc + ch.off, vb, &r.full[st], pol);
      else bulk_g2s(r.vals[st], vsrc + ch.off, vb, &r.full[st]);
    }
    bulk_g2s(r.segs[st], f.seg + ch.seg0, sb, &r.full[st]);
  }
  if (pre == n && n > 0) after_prefill<S>(f, r.full, n);
}

// ---- pass 1 ------------------------------------------------------------------
template <bool kDry, int R, int W, typename V>
__device__ __forceinline__ void rowdot_consume(const hdk_factor& f, Ring<Pass1<W>::stages, V>& ring,
                                               const double* __restrict__ rhs, int c_beg, int c_end);

// R columns: consumer warp w serves column w / (W / R) and every (W / R)-th
// segment pair of each staged chunk, so the chunk is streamed once for all R
// columns and a warp still holds one column's right-hand side tile.
template <bool kDry = false, int R = 1, int W = kWarps, typename V = double>  // kDry: stream only (microbenchmarks)
__global__ void __launch_bounds__(Pass1<W>::threads, Pass1<W>::min_blocks) k_rowdot(hdk_factor f,
                                                                                   const double* __restrict__ rhs) {
  constexpr int S = Pass1<W>::stages;
  hdk::pdl_trigger();  // the producer prefills before the PDL wait; consumers wait below
  extern __shared__ __align__(128) unsigned char smem_raw[];
  Ring<S, V>& ring = *reinterpret_cast<Ring<S, V>*>(smem_raw);
  const int warp = threadIdx.x >> 5;
  unsigned long long* trace = HDK_TRACE_PTR;
  if (trace && threadIdx.x == 0) trace[2 * blockIdx.x] = globaltimer();
  ring_init(ring, W);
  const int c_beg = f.first1 ? f.first1[blockIdx.x] : range_first(blockIdx.x, gridDim.x, f.n_chunks);
  const int c_end = f.first1 ? f.first1[blockIdx.x + 1] : range_first(blockIdx.x + 1LL, gridDim.x, f.n_chunks);
  if (warp == W) {
    produce(f, ring, c_beg, c_end, false);
    return;
  }
  HDK_TRACED_WAIT(hdk::kTrRowdot);
  if (f.run_flag && *f.run_flag == 0) return;
  rowdot_consume<kDry, R, W, V>(f, ring, rhs, c_beg, c_end);
  if (trace) {
    asm volatile("bar.sync 1, %0;" ::"r"(32 * W) : "memory");
    if (threadIdx.x == 0) trace[2 * blockIdx.x + 1] = globaltimer();
  }
}

template <bool kDry, int R, int W, typename V>
__device__ __forceinline__ void rowdot_consume(const hdk_factor& f, Ring<Pass1<W>::stages, V>& ring,
                                               const double* __restrict__ rhs, int c_beg, int c_end) {
  constexpr int S = Pass1<W>::stages;
  constexpr int WPC = W / R;  // consumer warps per column
  static_assert(WPC * R == W, "columns must divide the consumer warps");
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int colr = warp / WPC, sub = warp % WPC;
  rhs += (size_t)colr * 3 * (size_t)f.n;
  double* const part1 = f.part1 + (size_t)colr * 3 * (size_t)f.n_pslot;
  double b0[kM], b1[kM], b2[kM];
  int tile = -1;
  for (int c = c_beg, k = 0; c < c_end; ++c, ++k) {
    const int st = k % S;
    mbar_wait(&ring.full[st], (k / S) & 1);
    const ChunkInfo ch = ring.info[st];
    if (ch.tile != tile) {  // right-hand side of the tile into registers
      tile = ch.tile;
#pragma unroll
      for (int m = 0; m < kM; ++m) {
        const int col = tile * kW + lane + 32 * m;
        const bool ok = col < f.n;
        b0[m] = ok ? __ldg(rhs + 3 * (size_t)col) : 0.0;
        b1[m] = ok ? __ldg(rhs + 3 * (size_t)col + 1) : 0.0;
        b2[m] = ok ? __ldg(rhs + 3 * (size_t)col + 2) : 0.0;
      }
    }
    const V* vals = ring.vals[st];
    // segment pair p = {2p, 2p+1} of the chunk goes to warp (seg0/2 + p) mod 8
    // (balanced over chunks); the two dot products share one shuffle tree.
    // The stage is released as soon as the warp's last pair sits in
    // registers, so the producer refills it while the arithmetic runs.
    const int npair = (ch.nseg + 1) >> 1;
    bool released = false;
    for (int pi = (sub - (ch.seg0 >> 1)) & (WPC - 1); pi < (kDry ? 0 : npair); pi += WPC) {
      const int ia = 2 * pi, ib = ia + 1;
      const bool hasb = ib < ch.nseg;
      const hdk_seg sa = ring.segs[st][ia];
      const hdk_seg sb = hasb ? ring.segs[st][ib] : sa;
      const int la = sa.clo_len & 0xffff, ha = la + (sa.clo_len >> 16);
      const int lb = sb.clo_len & 0xffff, hb = hasb ? lb + (sb.clo_len >> 16) : lb;
      const V* va = vals + sa.coff - la;
      const V* vb = vals + sb.coff - lb;
      double wa[kM], wb[kM];
#pragma unroll
      for (int m = 0; m < kM; ++m) {
        const int cl = lane + 32 * m;
        wa[m] = (cl >= la && cl < ha) ? static_cast<double>(va[cl]) : 0.0;
        wb[m] = (cl >= lb && cl < hb) ? static_cast<double>(vb[cl]) : 0.0;
      }
      if (pi + WPC >= npair) {
        __syncwarp();
        if (lane == 0) mbar_arrive(&ring.empty[st]);
        released = true;
      }
      double a0 = 0.0, a1 = 0.0, a2 = 0.0, c0 = 0.0, c1 = 0.0, c2 = 0.0;
#pragma unroll
      for (int m = 0; m < kM; ++m) {
        a0 += wa[m] * b0[m];
        a1 += wa[m] * b1[m];
        a2 += wa[m] * b2[m];
        c0 += wb[m] * b0[m];
        c1 += wb[m] * b1[m];
        c2 += wb[m] * b2[m];
      }
      // reduce-scatter: lanes 0-15 keep segment a, lanes 16-31 segment b
      // after the first exchange, so the pair costs 15 shuffles, not 30
      // (a full butterfly over the six sums, 8 shuffles, measured slower:
      // more live registers, spills)
      const bool lo = lane < 16;
      double k0 = lo ? a0 : c0, k1 = lo ? a1 : c1, k2 = lo ? a2 : c2;
      k0 += __shfl_xor_sync(0xffffffffu, lo ? c0 : a0, 16);
      k1 += __shfl_xor_sync(0xffffffffu, lo ? c1 : a1, 16);
      k2 += __shfl_xor_sync(0xffffffffu, lo ? c2 : a2, 16);
#pragma unroll
      for (int o = 8; o > 0; o >>= 1) {
        k0 += __shfl_xor_sync(0xffffffffu, k0, o);
        k1 += __shfl_xor_sync(0xffffffffu, k1, o);
        k2 += __shfl_xor_sync(0xffffffffu, k2, o);
      }
      if (lane == 0 || (lane == 16 && hasb)) {
        double* p = part1 + 3 * (size_t)(lane == 0 ? sa.pslot : sb.pslot);
        p[0] = k0;
        p[1] = k1;
        p[2] = k2;
      }
    }
    if (!released) {
      __syncwarp();
      if (lane == 0) mbar_arrive(&ring.empty[st]);
    }
  }
}

// Multi-column pass 1 with two columns per warp (R = 2 or 4): each staged
// value is loaded from shared memory once per column pair, and the twelve
// sums of a segment pair (2 segments x 2 columns x 3 axes) share one
// reduce-scatter tree (18 shuffles instead of 30).  8 consumer warps, 1 CTA
// per SM (~170 registers per thread), 6-stage ring.
constexpr int kStagesC2 = 6;
template <int R>
__device__ __forceinline__ void rowdot_consume_c2(const hdk_factor& f, Ring<kStagesC2>& ring,
                                                  const double* __restrict__ rhs, int c_beg, int c_end) {
  constexpr int S = kStagesC2, W = kWarps, G = R / 2;
  constexpr int WPC = W / G;  // consumer warps per column pair
  static_assert(G * 2 == R && WPC * G == W, "column pairs must divide the consumer warps");
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int pair = warp / WPC, sub = warp % WPC;
  const double* r0 = rhs + (size_t)(2 * pair) * 3 * (size_t)f.n;
  const double* r1 = r0 + 3 * (size_t)f.n;
  double* const pa = f.part1 + (size_t)(2 * pair) * 3 * (size_t)f.n_pslot;
  double* const pb = pa + 3 * (size_t)f.n_pslot;
  double b[2][3][kM];
  int tile = -1;
  for (int c = c_beg, k = 0; c < c_end; ++c, ++k) {
    const int st = k % S;
    mbar_wait(&ring.full[st], (k / S) & 1);
    const ChunkInfo ch = ring.info[st];
    if (ch.tile != tile) {
      tile = ch.tile;
#pragma unroll
      for (int m = 0; m < kM; ++m) {
        const int col = tile * kW + lane + 32 * m;
        const bool ok = col < f.n;
#pragma unroll
        for (int a = 0; a < 3; ++a) {
          b[0][a][m] = ok ? __ldg(r0 + 3 * (size_t)col + a) : 0.0;
          b[1][a][m] = ok ? __ldg(r1 + 3 * (size_t)col + a) : 0.0;
        }
      }
    }
    const double* vals = ring.vals[st];
    const int npair = (ch.nseg + 1) >> 1;
    bool released = false;
    for (int pi = (sub - (ch.seg0 >> 1)) & (WPC - 1); pi < npair; pi += WPC) {
      const int ia = 2 * pi, ib = ia + 1;
      const bool hasb = ib < ch.nseg;
      const hdk_seg sa = ring.segs[st][ia];
      const hdk_seg sb = hasb ? ring.segs[st][ib] : sa;
      const int la = sa.clo_len & 0xffff, ha = la + (sa.clo_len >> 16);
      const int lb = sb.clo_len & 0xffff, hb = hasb ? lb + (sb.clo_len >> 16) : lb;
      const double* va = vals + sa.coff - la;
      const double* vb = vals + sb.coff - lb;
      double wa[kM], wb[kM];
#pragma unroll
      for (int m = 0; m < kM; ++m) {
        const int cl = lane + 32 * m;
        wa[m] = (cl >= la && cl < ha) ? va[cl] : 0.0;
        wb[m] = (cl >= lb && cl < hb) ? vb[cl] : 0.0;
      }
      if (pi + WPC >= npair) {
        __syncwarp();
        if (lane == 0) mbar_arrive(&ring.empty[st]);
        released = true;
      }
      double acc[2][2][3];  // [segment][column][axis]
#pragma unroll
      for (int q = 0; q < 2; ++q)
#pragma unroll
        for (int a = 0; a < 3; ++a) acc[0][q][a] = acc[1][q][a] = 0.0;
#pragma unroll
      for (int m = 0; m < kM; ++m)
#pragma unroll
        for (int q = 0; q < 2; ++q)
#pragma unroll
          for (int a = 0; a < 3; ++a) {
            acc[0][q][a] += wa[m] * b[q][a][m];
            acc[1][q][a] += wb[m] * b[q][a][m];
          }
      // reduce-scatter: offset 16 splits the segments, offset 8 the columns,
      // then a butterfly over the remaining 8 lanes
      const bool lo = lane < 16, c0 = (lane & 8) == 0;
      double kq[2][3];
#pragma unroll
      for (int q = 0; q < 2; ++q)
#pragma unroll
        for (int a = 0; a < 3; ++a)
          kq[q][a] = (lo ? acc[0][q][a] : acc[1][q][a]) +
                     __shfl_xor_sync(0xffffffffu, lo ? acc[1][q][a] : acc[0][q][a], 16);
      double h[3];
#pragma unroll
      for (int a = 0; a < 3; ++a)
        h[a] = (c0 ? kq[0][a] : kq[1][a]) + __shfl_xor_sync(0xffffffffu, c0 ? kq[1][a] : kq[0][a], 8);
#pragma unroll
      for (int o = 4; o > 0; o >>= 1)
#pragma unroll
        for (int a = 0; a < 3; ++a) h[a] += __shfl_xor_sync(0xffffffffu, h[a], o);
      if ((lane & 7) == 0 && (lo || hasb)) {
        double* p = (c0 ? pa : pb) + 3 * (size_t)(lo ? sa.pslot : sb.pslot);
        p[0] = h[0];
        p[1] = h[1];
        p[2] = h[2];
      }
    }
    if (!released) {
      __syncwarp();
      if (lane == 0) mbar_arrive(&ring.empty[st]);
    }
  }
}

template <int R>
__global__ void __launch_bounds__(kThreads, 1) k_rowdot_c2(hdk_factor f, const double* __restrict__ rhs) {
  hdk::pdl_trigger();
  extern __shared__ __align__(128) unsigned char smem_raw[];
  Ring<kStagesC2>& ring = *reinterpret_cast<Ring<kStagesC2>*>(smem_raw);
  const int warp = threadIdx.x >> 5;
  unsigned long long* trace = HDK_TRACE_PTR;
  if (trace && threadIdx.x == 0) trace[2 * blockIdx.x] = globaltimer();
  ring_init(ring, kWarps);
  const int c_beg = f.first1 ? f.first1[blockIdx.x] : range_first(blockIdx.x, gridDim.x, f.n_chunks);
  const int c_end = f.first1 ? f.first1[blockIdx.x + 1] : range_first(blockIdx.x + 1LL, gridDim.x, f.n_chunks);
  if (warp == kWarps) {
    produce(f, ring, c_beg, c_end, false);
    return;
  }
  HDK_TRACED_WAIT(hdk::kTrRowdot);
  if (f.run_flag && *f.run_flag == 0) return;
  rowdot_consume_c2<R>(f, ring, rhs, c_beg, c_end);
  if (trace) {
    asm volatile("bar.sync 1, %0;" ::"r"(32 * kWarps) : "memory");
    if (threadIdx.x == 0) trace[2 * blockIdx.x + 1] = globaltimer();
  }
}

// ---- pass 1 of the multi-column solve on the FP64 tensor cores ---------------
// With R columns every staged value of S' meets 3R right-hand sides.  Eight
// segments of a chunk form the rows of an m8n8k4 DMMA tile: A = their values
// over four tile columns (zero outside each row's range), B = those columns'
// right-hand sides staged per tile in shared memory, D accumulates the eight
// row dots of up to eight right-hand sides in registers over the group's
// column range — no per-lane predicated FMA sweep over all 256 columns and no
// shuffle reduction per segment, and the small register footprint lets 16
// consumer warps hide the shared-memory latency.  Fragment layout
// (mma.m8n8k4.row.col.f64): A(g, t), B(t, g), D(g, 2t + i) with
// g = lane / 4, t = lane % 4.  The sums run in k order inside the tensor core:
// same values as the FMA passes up to rounding.
constexpr int kWarpsMma = 16;
template <int R>
struct MmaPass1Smem {
  static constexpr int S = 6;  // ring depth (229.6 KB with the R = 8 B tile)
  // row pitch 8 NB + 4: the 16 lanes of a half-warp (4 t x 4 g) hit 16 distinct 8-byte banks
  static constexpr int NQ = 3 * R, NB = (NQ + 7) / 8, LD = 8 * NB + 4;
  Ring<S> ring;
  double bt[kW * LD];  // the tile's right-hand sides: bt[col * LD + q], q = 3 column + axis
};

__device__ __forceinline__ void dmma_m8n8k4(double (&d)[2], double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0, %1}, {%2}, {%3}, {%0, %1};"
               : "+d"(d[0]), "+d"(d[1])
               : "d"(a), "d"(b));
}
__device__ __forceinline__ void mma_consumers_sync() {
  asm volatile("bar.sync 1, %0;" ::"n"(32 * kWarpsMma) : "memory");
}

template <int R>
__global__ void __launch_bounds__(32 * (kWarpsMma + 1), 1) k_rowdot_mma(hdk_factor f, const double* __restrict__ rhs) {
  using Sm = MmaPass1Smem<R>;
  constexpr int NQ = Sm::NQ, NB = Sm::NB, LD = Sm::LD, S = Sm::S, W = kWarpsMma;
  hdk::pdl_trigger();
  extern __shared__ __align__(128) unsigned char smem_raw[];
  Sm& sm = *reinterpret_cast<Sm*>(smem_raw);
  Ring<S>& ring = sm.ring;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  ring_init(ring, W);
  const int c_beg = f.first1 ? f.first1[blockIdx.x] : range_first(blockIdx.x, gridDim.x, f.n_chunks);
  const int c_end = f.first1 ? f.first1[blockIdx.x + 1] : range_first(blockIdx.x + 1LL, gridDim.x, f.n_chunks);
  if (warp == W) {
    produce(f, ring, c_beg, c_end, false);
    return;
  }
  HDK_TRACED_WAIT(hdk::kTrRowdot);
  if (f.run_flag && *f.run_flag == 0) return;
  const int g = lane >> 2, t = lane & 3;
  const size_t ps = 3 * (size_t)f.n_pslot;
  int tile = -1;
  for (int c = c_beg, k = 0; c < c_end; ++c, ++k) {
    const int st = k % S;
    mbar_wait(&ring.full[st], (k / S) & 1);
    long long* tr = g_chunk_trace;
    if (tr && warp == 0 && lane == 0) {
      tr[4 * (size_t)c + 2] = sm_clock();
      tr[4 * (size_t)c + 3] = ((ring.info[st].nseg + 7) >> 3);  // groups
    }
    const ChunkInfo ch = ring.info[st];
    if (ch.tile != tile) {  // every consumer warp reaches the new tile at this chunk
      mma_consumers_sync();
      tile = ch.tile;
      for (int e = threadIdx.x; e < kW * 8 * NB; e += 32 * W) {
        const int col = e / (8 * NB), q = e - col * (8 * NB);
        const int gc = tile * kW + col;
        double v = 0.0;
        if (q < NQ && gc < f.n) v = __ldg(rhs + (size_t)(q / 3) * 3 * (size_t)f.n + 3 * (size_t)gc + (q % 3));
        sm.bt[col * LD + q] = v;
      }
      mma_consumers_sync();
    }
    const double* vals = ring.vals[st];
    const int ngroups = (ch.nseg + 7) >> 3;
    for (int grp = (warp - (ch.seg0 >> 3)) & (W - 1); grp < ngroups; grp += W) {
      const int i = 8 * grp + g;
      const bool live = i < ch.nseg;
      const hdk_seg sg = ring.segs[st][live ? i : 0];
      const int lo = live ? (sg.clo_len & 0xffff) : kW;
      const int hi = live ? lo + (sg.clo_len >> 16) : 0;
      int ulo = lo, uhi = hi;
#pragma unroll
      for (int o = 4; o < 32; o <<= 1) {
        ulo = min(ulo, __shfl_xor_sync(0xffffffffu, ulo, o));
        uhi = max(uhi, __shfl_xor_sync(0xffffffffu, uhi, o));
      }
      const double* v = vals + sg.coff - lo;
      // four accumulator sets over consecutive k-steps: four independent DMMA
      // chains per n-block instead of one (the tensor core's latency, not its
      // rate, bounded the single chain)
      constexpr int kAcc = NB >= 3 ? 2 : 4;  // register budget of 16 consumer warps
      double d[kAcc][NB][2];
#pragma unroll
      for (int u = 0; u < kAcc; ++u)
#pragma unroll
        for (int nb = 0; nb < NB; ++nb) d[u][nb][0] = d[u][nb][1] = 0.0;
      int kc = ulo & ~3;
      for (; kc + 4 * (kAcc - 1) < uhi; kc += 4 * kAcc) {
#pragma unroll
        for (int u = 0; u < kAcc; ++u) {
          const int col = kc + 4 * u + t;
          const double a = (col >= lo && col < hi) ? v[col] : 0.0;
#pragma unroll
          for (int nb = 0; nb < NB; ++nb) dmma_m8n8k4(d[u][nb], a, sm.bt[col * LD + 8 * nb + g]);
        }
      }
#pragma unroll
      for (int u = 0; u < kAcc - 1; ++u) {  // remainder: at most kAcc - 1 k-steps (warp-uniform bound)
        if (kc + 4 * u >= uhi) break;
        const int col = kc + 4 * u + t;
        const double a = (col >= lo && col < hi) ? v[col] : 0.0;
#pragma unroll
        for (int nb = 0; nb < NB; ++nb) dmma_m8n8k4(d[u][nb], a, sm.bt[col * LD + 8 * nb + g]);
      }
      if (live) {
#pragma unroll
        for (int nb = 0; nb < NB; ++nb)
#pragma unroll
          for (int j = 0; j < 2; ++j) {
            const int q = 8 * nb + 2 * t + j;
            if (q < NQ) {
              double sum = d[0][nb][j];
#pragma unroll
              for (int u = 1; u < kAcc; ++u) sum = sum + d[u][nb][j];  // fixed order
              f.part1[(size_t)(q / 3) * ps + 3 * (size_t)sg.pslot + (q % 3)] = sum;
            }
          }
      }
    }
    __syncwarp();
    if (lane == 0) mbar_arrive(&ring.empty[st]);
  }
}

// The same pass with the work of a staged chunk split finer: an item is one
// group of eight segments x one n-block of eight right-hand sides, so a chunk
// of g groups gives g NB items for the consumer warps (not g).  A stage is
// released only when every consumer warp has finished it, so with ~2 groups
// per chunk the group-per-warp form kept most warps waiting behind the few
// long groups; here each warp's share of a chunk is a third as long and the
// ring turns over faster.  Each item runs kAccN independent DMMA chains.
template <int R>
__global__ void __launch_bounds__(32 * (kWarpsMma + 1), 1) k_rowdot_mma_nb(hdk_factor f, const double* __restrict__ rhs) {
  using Sm = MmaPass1Smem<R>;
  constexpr int NQ = Sm::NQ, NB = Sm::NB, LD = Sm::LD, S = Sm::S, W = kWarpsMma;
  constexpr int kAccN = 4;
  hdk::pdl_trigger();
  extern __shared__ __align__(128) unsigned char smem_raw[];
  Sm& sm = *reinterpret_cast<Sm*>(smem_raw);
  Ring<S>& ring = sm.ring;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  ring_init(ring, W);
  const int c_beg = f.first1 ? f.first1[blockIdx.x] : range_first(blockIdx.x, gridDim.x, f.n_chunks);
  const int c_end = f.first1 ? f.first1[blockIdx.x + 1] : range_first(blockIdx.x + 1LL, gridDim.x, f.n_chunks);
  if (warp == W) {
    produce(f, ring, c_beg, c_end, false);
    return;
  }
  HDK_TRACED_WAIT(hdk::kTrRowdot);
  if (f.run_flag && *f.run_flag == 0) return;
  const int g = lane >> 2, t = lane & 3;
  const size_t ps = 3 * (size_t)f.n_pslot;
  int tile = -1;
  for (int c = c_beg, k = 0; c < c_end; ++c, ++k) {
    const int st = k % S;
    mbar_wait(&ring.full[st], (k / S) & 1);
    const ChunkInfo ch = ring.info[st];
    if (ch.tile != tile) {  // every consumer warp reaches the new tile at this chunk
      mma_consumers_sync();
      tile = ch.tile;
      for (int e = threadIdx.x; e < kW * 8 * NB; e += 32 * W) {
        const int col = e / (8 * NB), q = e - col * (8 * NB);
        const int gc = tile * kW + col;
        double v = 0.0;
        if (q < NQ && gc < f.n) v = __ldg(rhs + (size_t)(q / 3) * 3 * (size_t)f.n + 3 * (size_t)gc + (q % 3));
        sm.bt[col * LD + q] = v;
      }
      mma_consumers_sync();
    }
    const double* vals = ring.vals[st];
    const int items = ((ch.nseg + 7) >> 3) * NB;
    for (int it = (warp - (ch.seg0 >> 3) * NB) & (W - 1); it < items; it += W) {
      const int grp = it / NB, nb = it - grp * NB;
      const int i = 8 * grp + g;
      const bool live = i < ch.nseg;
      const hdk_seg sg = ring.segs[st][live ? i : 0];
      const int lo = live ? (sg.clo_len & 0xffff) : kW;
      const int hi = live ? lo + (sg.clo_len >> 16) : 0;
      int ulo = lo, uhi = hi;
#pragma unroll
      for (int o = 4; o < 32; o <<= 1) {
        ulo = min(ulo, __shfl_xor_sync(0xffffffffu, ulo, o));
        uhi = max(uhi, __shfl_xor_sync(0xffffffffu, uhi, o));
      }
      const double* v = vals + sg.coff - lo;
      const double* bcol = sm.bt + 8 * nb + g;
      double d[kAccN][2];
#pragma unroll
      for (int u = 0; u < kAccN; ++u) d[u][0] = d[u][1] = 0.0;
      int kc = ulo & ~3;
      for (; kc + 4 * (kAccN - 1) < uhi; kc += 4 * kAccN) {
        double a[kAccN], b[kAccN];
#pragma unroll
        for (int u = 0; u < kAccN; ++u) {
          const int col = kc + 4 * u + t;
          a[u] = (col >= lo && col < hi) ? v[col] : 0.0;
          b[u] = bcol[col * LD];
        }
#pragma unroll
        for (int u = 0; u < kAccN; ++u) dmma_m8n8k4(d[u], a[u], b[u]);
      }
#pragma unroll
      for (int u = 0; u < kAccN - 1; ++u) {  // remainder: at most kAccN - 1 k-steps (warp-uniform bound)
        if (kc + 4 * u >= uhi) break;
        const int col = kc + 4 * u + t;
        const double a = (col >= lo && col < hi) ? v[col] : 0.0;
        dmma_m8n8k4(d[u], a, bcol[col * LD]);
      }
      if (live) {
#pragma unroll
        for (int j = 0; j < 2; ++j) {
          const int q = 8 * nb + 2 * t + j;
          if (q < NQ) {
            double sum = d[0][j];
#pragma unroll
            for (int u = 1; u < kAccN; ++u) sum = sum + d[u][j];  // fixed order
            f.part1[(size_t)(q / 3) * ps + 3 * (size_t)sg.pslot + (q % 3)] = sum;
          }
        }
      }
    }
    __syncwarp();
    if (lane == 0) mbar_arrive(&ring.empty[st]);
  }
}

// fp32 copy of the value stream, chunk by chunk (one block per chunk).
__global__ void k_to_fp32(const double* __restrict__ sval, const hdk_chunk* __restrict__ chunk,
                          float* __restrict__ sval32, const hdk_chunk* __restrict__ chunk32) {
  const hdk_chunk c = chunk[blockIdx.x], c32 = chunk32[blockIdx.x];
  for (int i = threadIdx.x; i < c32.len; i += blockDim.x)
    sval32[c32.off + i] = i < c.len ? static_cast<float>(sval[c.off + i]) : 0.0f;
}

// z-fold: one warp per task.  (Folding z in the row-dot kernel's epilogue
// behind a grid barrier measured 1-2 us slower than this separate launch.)
__global__ void __launch_bounds__(256) k_zreduce(hdk_factor f) {
  const int t = blockIdx.x * 8 + (threadIdx.x >> 5);  // one task per warp
  const bool has = t < f.n_ztask;
  const ZRows zr = zfold_rows(f, has ? __ldg(f.ztask + t) : make_int2(0, 0));
  HDK_TRACED_WAIT(hdk::kTrZfold);
  hdk::pdl_trigger();
  if (f.run_flag && *f.run_flag == 0) return;
  if (has) zfold_task(f, zr, blockIdx.y);
}

// ---- pass 2 ------------------------------------------------------------------
// Ring depth of pass 2 for R columns (the z rows of every column are staged
// with each chunk; 227 KB of shared memory per CTA).
template <int R>
struct Stages2 {
  static constexpr int value = R == 1 ? kStages2 : R == 2 ? 6 : R == 4 ? 6 : 5;
};

template <int R, typename V = double>
struct Pass2Smem {
  Ring2<Stages2<R>::value, R, V> ring;
  double fold[kWarps / 2][3][kW];
};

// Fixed-order fold of the consumer warps' accumulators (4..7 into 0..3, 2..3
// into 0..1, 1 into 0; with R columns within each column's 8 / R warps) and
// write of the tile partial; consumer warps only.
template <int R, typename V>
__device__ __forceinline__ void fold_and_write(const hdk_factor& f, Pass2Smem<R, V>& sm, int slot, double (&x0)[kM],
                                               double (&x1)[kM], double (&x2)[kM]) {
  constexpr int WPC = kWarps / R;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int colr = warp / WPC, sub = warp % WPC;
#pragma unroll
  for (int half = WPC / 2; half >= 1; half >>= 1) {
    consumers_sync();
    if (sub >= half && sub < 2 * half) {
      const int fb = colr * (WPC / 2) + sub - half;
#pragma unroll
      for (int m = 0; m < kM; ++m) {
        const int cl = lane + 32 * m;
        sm.fold[fb][0][cl] = x0[m];
        sm.fold[fb][1][cl] = x1[m];
        sm.fold[fb][2][cl] = x2[m];
      }
    }
    consumers_sync();
    if (sub < half) {
      const int fb = colr * (WPC / 2) + sub;
#pragma unroll
      for (int m = 0; m < kM; ++m) {
        const int cl = lane + 32 * m;
        x0[m] += sm.fold[fb][0][cl];
        x1[m] += sm.fold[fb][1][cl];
        x2[m] += sm.fold[fb][2][cl];
      }
    }
  }
  if (sub == 0) {
    double* const part2 = f.part2 + (size_t)colr * part2_stride(f);
#pragma unroll
    for (int m = 0; m < kM; ++m) {
      double* p = part2 + 3 * ((size_t)slot * kW + lane + 32 * m);
      p[0] = x0[m];
      p[1] = x1[m];
      p[2] = x2[m];
    }
  }
#pragma unroll
  for (int m = 0; m < kM; ++m) x0[m] = x1[m] = x2[m] = 0.0;
}

template <bool kDry = false, int R = 1, typename V = double>
__global__ void __launch_bounds__(kThreads2) k_coltile(hdk_factor f) {
  constexpr int S = Stages2<R>::value, WPC = kWarps / R;
  hdk::pdl_trigger();  // the producer prefills before the PDL wait; the others wait below
  extern __shared__ __align__(128) unsigned char smem_raw[];
  Pass2Smem<R, V>& sm = *reinterpret_cast<Pass2Smem<R, V>*>(smem_raw);
  Ring2<S, R, V>& ring = sm.ring;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  unsigned long long* trace = HDK_TRACE_PTR;
  if (trace && threadIdx.x == 0) trace[2 * blockIdx.x] = globaltimer();
  ring2_init(ring);
  const int c_beg = f.first2 ? f.first2[blockIdx.x] : range_first(blockIdx.x, gridDim.x, f.n_chunks);
  const int c_end = f.first2 ? f.first2[blockIdx.x + 1] : range_first(blockIdx.x + 1LL, gridDim.x, f.n_chunks);
  // Pass 2 walks its range backwards: the tail pass 1 just streamed is still
  // in L2, and pass 2 ends where the next pass 1 begins.
  if (warp == kWarps) {
    stream2(f, ring, c_beg, c_end);
    return;
  }
  HDK_TRACED_WAIT(hdk::kTrColtile);
  if (f.run_flag && *f.run_flag == 0) return;
  if (warp == kWarps + 1) {
    gather_z(f, ring, c_end - c_beg);
    return;
  }
  double x0[kM], x1[kM], x2[kM];
#pragma unroll
  for (int m = 0; m < kM; ++m) x0[m] = x1[m] = x2[m] = 0.0;
  int tile = -1;
  for (int k = 0; k < c_end - c_beg; ++k) {
    const int st = k % S;
    mbar_wait(&ring.zfull[st], (k / S) & 1);
    const ChunkInfo ch = ring.info[st];
    if (ch.tile != tile) {  // partial of the previous tile: slot tile + b is unique
      if (tile >= 0) fold_and_write(f, sm, tile + blockIdx.x, x0, x1, x2);
      tile = ch.tile;
    }
    const V* vals = ring.vals[st];
    const int i0 = (warp % WPC - ch.seg0) & (WPC - 1);
    const int zc = 3 * (warp / WPC);
    for (int i = i0; i < (kDry ? 0 : ch.nseg); i += WPC) {
      const hdk_seg sg = ring.segs[st][i];
      const int lo = sg.clo_len & 0xffff, hi = lo + (sg.clo_len >> 16);
      const V* v = vals + sg.coff - lo;
      const double z0 = ring.zs[st][i][zc], z1 = ring.zs[st][i][zc + 1], z2 = ring.zs[st][i][zc + 2];
#pragma unroll
      for (int m = 0; m < kM; ++m) {
        const int cl = lane + 32 * m;
        if (cl >= lo && cl < hi) {
          const double w = static_cast<double>(v[cl]);
          x0[m] += w * z0;
          x1[m] += w * z1;
          x2[m] += w * z2;
        }
      }
    }
    __syncwarp();
    if (lane == 0) mbar_arrive(&ring.empty[st]);
  }
  if (tile >= 0) fold_and_write(f, sm, tile + blockIdx.x, x0, x1, x2);
  if (trace) {
    consumers_sync();
    if (threadIdx.x == 0) trace[2 * blockIdx.x + 1] = globaltimer();
  }
}

// Multi-column pass 2 with two columns per warp (R = 2 or 4): each staged
// value is loaded once per column pair and feeds six accumulator rows; the
// 8 / (R / 2) warps of a pair fold each column in turn through the same
// shared buffer as fold_and_write.
template <int WPC>
__device__ __forceinline__ void fold_write_col(const hdk_factor& f, double (*fold)[3][kW], int slot, int col,
                                               int pair, int sub, double (&x0)[kM], double (&x1)[kM],
                                               double (&x2)[kM]) {
  const int lane = threadIdx.x & 31;
#pragma unroll
  for (int half = WPC / 2; half >= 1; half >>= 1) {
    consumers_sync();
    if (sub >= half && sub < 2 * half) {
      const int fb = pair * (WPC / 2) + sub - half;
#pragma unroll
      for (int m = 0; m < kM; ++m) {
        const int cl = lane + 32 * m;
        fold[fb][0][cl] = x0[m];
        fold[fb][1][cl] = x1[m];
        fold[fb][2][cl] = x2[m];
      }
    }
    consumers_sync();
    if (sub < half) {
      const int fb = pair * (WPC / 2) + sub;
#pragma unroll
      for (int m = 0; m < kM; ++m) {
        const int cl = lane + 32 * m;
        x0[m] += fold[fb][0][cl];
        x1[m] += fold[fb][1][cl];
        x2[m] += fold[fb][2][cl];
      }
    }
  }
  if (sub == 0) {
    double* const part2 = f.part2 + (size_t)col * part2_stride(f);
#pragma unroll
    for (int m = 0; m < kM; ++m) {
      double* p = part2 + 3 * ((size_t)slot * kW + lane + 32 * m);
      p[0] = x0[m];
      p[1] = x1[m];
      p[2] = x2[m];
    }
  }
#pragma unroll
  for (int m = 0; m < kM; ++m) x0[m] = x1[m] = x2[m] = 0.0;
}

template <int R>
__global__ void __launch_bounds__(kThreads2, 1) k_coltile_c2(hdk_factor f) {
  constexpr int S = Stages2<R>::value, G = R / 2, WPC = kWarps / G;
  static_assert(G * 2 == R && WPC * G == kWarps && WPC / 2 * G <= kWarps / 2, "column pairs");
  hdk::pdl_trigger();
  extern __shared__ __align__(128) unsigned char smem_raw[];
  Pass2Smem<R>& sm = *reinterpret_cast<Pass2Smem<R>*>(smem_raw);
  Ring2<S, R>& ring = sm.ring;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  unsigned long long* trace = HDK_TRACE_PTR;
  if (trace && threadIdx.x == 0) trace[2 * blockIdx.x] = globaltimer();
  ring2_init(ring);
  const int c_beg = f.first2 ? f.first2[blockIdx.x] : range_first(blockIdx.x, gridDim.x, f.n_chunks);
  const int c_end = f.first2 ? f.first2[blockIdx.x + 1] : range_first(blockIdx.x + 1LL, gridDim.x, f.n_chunks);
  if (warp == kWarps) {
    stream2(f, ring, c_beg, c_end);
    return;
  }
  HDK_TRACED_WAIT(hdk::kTrColtile);
  if (f.run_flag && *f.run_flag == 0) return;
  if (warp == kWarps + 1) {
    gather_z(f, ring, c_end - c_beg);
    return;
  }
  const int pair = warp / WPC, sub = warp % WPC;
  double x0[kM], x1[kM], x2[kM], y0[kM], y1[kM], y2[kM];
#pragma unroll
  for (int m = 0; m < kM; ++m) x0[m] = x1[m] = x2[m] = y0[m] = y1[m] = y2[m] = 0.0;
  int tile = -1;
  for (int k = 0; k < c_end - c_beg; ++k) {
    const int st = k % S;
    mbar_wait(&ring.zfull[st], (k / S) & 1);
    const ChunkInfo ch = ring.info[st];
    if (ch.tile != tile) {
      if (tile >= 0) {
        fold_write_col<WPC>(f, sm.fold, tile + blockIdx.x, 2 * pair, pair, sub, x0, x1, x2);
        fold_write_col<WPC>(f, sm.fold, tile + blockIdx.x, 2 * pair + 1, pair, sub, y0, y1, y2);
      }
      tile = ch.tile;
    }
    const double* vals = ring.vals[st];
    const int i0 = (sub - ch.seg0) & (WPC - 1);
    const int zc = 6 * pair;
    for (int i = i0; i < ch.nseg; i += WPC) {
      const hdk_seg sg = ring.segs[st][i];
      const int lo = sg.clo_len & 0xffff, hi = lo + (sg.clo_len >> 16);
      const double* v = vals + sg.coff - lo;
      const double* z = ring.zs[st][i] + zc;
      const double z0 = z[0], z1 = z[1], z2 = z[2], z3 = z[3], z4 = z[4], z5 = z[5];
#pragma unroll
      for (int m = 0; m < kM; ++m) {
        const int cl = lane + 32 * m;
        if (cl >= lo && cl < hi) {
          const double w = v[cl];
          x0[m] += w * z0;
          x1[m] += w * z1;
          x2[m] += w * z2;
          y0[m] += w * z3;
          y1[m] += w * z4;
          y2[m] += w * z5;
        }
      }
    }
    __syncwarp();
    if (lane == 0) mbar_arrive(&ring.empty[st]);
  }
  if (tile >= 0) {
    fold_write_col<WPC>(f, sm.fold, tile + blockIdx.x, 2 * pair, pair, sub, x0, x1, x2);
    fold_write_col<WPC>(f, sm.fold, tile + blockIdx.x, 2 * pair + 1, pair, sub, y0, y1, y2);
  }
  if (trace) {
    consumers_sync();
    if (threadIdx.x == 0) trace[2 * blockIdx.x + 1] = globaltimer();
  }
}

// ---- pass 2 of the multi-column solve on the FP64 tensor cores ---------------
// x_tile (256 columns x 3R) += S'(segments, tile)^T z(segments): an m8n8k4
// DMMA takes eight tile columns (M), four segments (K) and eight right-hand
// sides (N).  Consumer warp w owns tile columns [16 w, 16 w + 16) for the
// whole tile, so its accumulators stay in registers (no cross-warp fold) and
// are written as the CTA's tile partial when the tile ends; a group of four
// segments that misses the warp's columns is skipped.  z rows are staged by
// the gather warp exactly as for the FMA pass.
constexpr int kWarpsMma2 = 16;
template <int R>
struct MmaPass2Smem {
  Ring2<Stages2<R>::value, R> ring;
};

template <int R>
__device__ __forceinline__ void coltile_mma_write(const hdk_factor& f, int slot, int warp, double (&d)[2][(3 * R + 7) / 8][2]) {
  constexpr int NQ = 3 * R, NB = (NQ + 7) / 8;
  const int lane = threadIdx.x & 31, g = lane >> 2, t = lane & 3;
#pragma unroll
  for (int mb = 0; mb < 2; ++mb) {
    const int col = 16 * warp + 8 * mb + g;
#pragma unroll
    for (int nb = 0; nb < NB; ++nb)
#pragma unroll
      for (int j = 0; j < 2; ++j) {
        const int q = 8 * nb + 2 * t + j;
        if (q < NQ) f.part2[(size_t)(q / 3) * part2_stride(f) + 3 * ((size_t)slot * kW + col) + (q % 3)] = d[mb][nb][j];
        d[mb][nb][j] = 0.0;
      }
  }
}

template <int R>
__global__ void __launch_bounds__(32 * (kWarpsMma2 + 2), 1) k_coltile_mma(hdk_factor f) {
  constexpr int S = Stages2<R>::value, NQ = 3 * R, NB = (NQ + 7) / 8, W = kWarpsMma2;
  static_assert(W * 16 == kW, "16 columns per consumer warp");
  hdk::pdl_trigger();
  extern __shared__ __align__(128) unsigned char smem_raw[];
  MmaPass2Smem<R>& sm = *reinterpret_cast<MmaPass2Smem<R>*>(smem_raw);
  Ring2<S, R>& ring = sm.ring;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  if (threadIdx.x == 0) {
    for (int st = 0; st < S; ++st) {
      mbar_init(&ring.full[st], 1);
      mbar_init(&ring.zfull[st], 32);
      mbar_init(&ring.empty[st], W);
    }
    mbar_fence_init();
  }
  __syncthreads();
  const int c_beg = f.first2 ? f.first2[blockIdx.x] : range_first(blockIdx.x, gridDim.x, f.n_chunks);
  const int c_end = f.first2 ? f.first2[blockIdx.x + 1] : range_first(blockIdx.x + 1LL, gridDim.x, f.n_chunks);
  if (warp == W) {
    stream2(f, ring, c_beg, c_end);
    return;
  }
  HDK_TRACED_WAIT(hdk::kTrColtile);
  if (f.run_flag && *f.run_flag == 0) return;
  if (warp == W + 1) {
    gather_z(f, ring, c_end - c_beg);
    return;
  }
  const int g = lane >> 2, t = lane & 3;
  const int wlo = 16 * warp, whi = wlo + 16;
  double d[2][NB][2];
#pragma unroll
  for (int mb = 0; mb < 2; ++mb)
#pragma unroll
    for (int nb = 0; nb < NB; ++nb) d[mb][nb][0] = d[mb][nb][1] = 0.0;
  int tile = -1;
  for (int k = 0; k < c_end - c_beg; ++k) {
    const int st = k % S;
    mbar_wait(&ring.zfull[st], (k / S) & 1);
    const ChunkInfo ch = ring.info[st];
    if (ch.tile != tile) {
      if (tile >= 0) coltile_mma_write<R>(f, tile + blockIdx.x, warp, d);
      tile = ch.tile;
    }
    const double* vals = ring.vals[st];
    for (int kg = 0; 4 * kg < ch.nseg; ++kg) {
      const int i = 4 * kg + t;
      const bool live = i < ch.nseg;
      const hdk_seg sg = ring.segs[st][live ? i : 0];
      const int lo = live ? (sg.clo_len & 0xffff) : kW;
      const int hi = live ? lo + (sg.clo_len >> 16) : 0;
      int ulo = lo, uhi = hi;
      ulo = min(ulo, __shfl_xor_sync(0xffffffffu, ulo, 1));
      uhi = max(uhi, __shfl_xor_sync(0xffffffffu, uhi, 1));
      ulo = min(ulo, __shfl_xor_sync(0xffffffffu, ulo, 2));
      uhi = max(uhi, __shfl_xor_sync(0xffffffffu, uhi, 2));
      if (uhi <= wlo || ulo >= whi) continue;  // no column of this warp (uniform over the warp)
      double b[NB];
#pragma unroll
      for (int nb = 0; nb < NB; ++nb) {
        const int q = 8 * nb + g;
        b[nb] = (live && q < NQ) ? ring.zs[st][i][q] : 0.0;
      }
      const double* v = vals + sg.coff - lo;
#pragma unroll
      for (int mb = 0; mb < 2; ++mb) {
        const int c0 = wlo + 8 * mb;
        if (uhi <= c0 || ulo >= c0 + 8) continue;
        const int col = c0 + g;
        // A(m = g, k = t) = S'(segment t, column c0 + g): each lane needs its
        // segment t's value at column col (lanes of one t share a segment)
        const double a = (col >= lo && col < hi) ? v[col] : 0.0;
#pragma unroll
        for (int nb = 0; nb < NB; ++nb) dmma_m8n8k4(d[mb][nb], a, b[nb]);
      }
    }
    __syncwarp();
    if (lane == 0) mbar_arrive(&ring.empty[st]);
  }
  if (tile >= 0) coltile_mma_write<R>(f, tile + blockIdx.x, warp, d);
}

// x_c = sum of the tile partials of the CTAs whose chunk ranges touch the
// column's tile (CTA order), scattered to the full vector.
template <bool kScatter>
__global__ void k_xreduce(hdk_factor f, int G, double* __restrict__ out) {
  // the tile's CTA range and the output slot are static: read before the wait
  hdk::pdl_trigger();
  const int c = blockIdx.x * blockDim.x + threadIdx.x;
  const bool live = c < f.n;
  const int cc = live ? c : 0;
  const int t = cc / kW, cl = cc - t * kW;
  const int b0 = f.tile_cta2 ? __ldg(f.tile_cta2 + 2 * t) : cta_of(__ldg(f.tile_chunk + t), G, f.n_chunks);
  const int b1 = f.tile_cta2 ? __ldg(f.tile_cta2 + 2 * t + 1) : cta_of(__ldg(f.tile_chunk + t + 1) - 1, G, f.n_chunks);
  const int slot = kScatter ? __ldg(f.p2v + cc) : cc;
  hdk::pdl_wait();
  if (!live) return;
  double a0 = 0.0, a1 = 0.0, a2 = 0.0;
  for (int b = b0; b <= b1; ++b) {
    const double* p = f.part2 + 3 * ((size_t)(t + b) * kW + cl);
    a0 += p[0];
    a1 += p[1];
    a2 += p[2];
  }
  double* o = out + 3 * (size_t)slot;
  o[0] = a0;
  o[1] = a1;
  o[2] = a2;
}

struct Grids {
  int g1, g2;
};

// One resident wave per pass, computed once per process (thread-safe static).
const Grids& grids() {
  static const Grids g = [] {
    const size_t s1 = sizeof(Ring<kStages1>), s2 = sizeof(Pass2Smem<1>);
    cudaFuncSetAttribute(k_rowdot<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(s1));
    cudaFuncSetAttribute(k_coltile<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(s2));
    cudaFuncSetAttribute(k_rowdot<false, 1, kWarps, float>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         static_cast<int>(sizeof(Ring<kStages1, float>)));
    cudaFuncSetAttribute(k_coltile<false, 1, float>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         static_cast<int>(sizeof(Pass2Smem<1, float>)));
    const int s16 = static_cast<int>(sizeof(Ring<Pass1<16>::stages>));
    cudaFuncSetAttribute(k_rowdot<false, 2, 16>, cudaFuncAttributeMaxDynamicSharedMemorySize, s16);
    cudaFuncSetAttribute(k_rowdot<false, 4, 16>, cudaFuncAttributeMaxDynamicSharedMemorySize, s16);
    const int sc2 = static_cast<int>(sizeof(Ring<kStagesC2>));
    cudaFuncSetAttribute(k_rowdot_c2<2>, cudaFuncAttributeMaxDynamicSharedMemorySize, sc2);
    cudaFuncSetAttribute(k_rowdot_c2<4>, cudaFuncAttributeMaxDynamicSharedMemorySize, sc2);
    cudaFuncSetAttribute(k_coltile_mma<2>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         static_cast<int>(sizeof(MmaPass2Smem<2>)));
    cudaFuncSetAttribute(k_coltile_mma<4>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         static_cast<int>(sizeof(MmaPass2Smem<4>)));
    cudaFuncSetAttribute(k_rowdot_mma<2>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         static_cast<int>(sizeof(MmaPass1Smem<2>)));
    cudaFuncSetAttribute(k_rowdot_mma<4>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         static_cast<int>(sizeof(MmaPass1Smem<4>)));
    cudaFuncSetAttribute(k_rowdot_mma<8>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         static_cast<int>(sizeof(MmaPass1Smem<8>)));
    cudaFuncSetAttribute(k_rowdot_mma_nb<2>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         static_cast<int>(sizeof(MmaPass1Smem<2>)));
    cudaFuncSetAttribute(k_rowdot_mma_nb<4>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         static_cast<int>(sizeof(MmaPass1Smem<4>)));
    cudaFuncSetAttribute(k_rowdot_mma_nb<8>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         static_cast<int>(sizeof(MmaPass1Smem<8>)));
    cudaFuncSetAttribute(k_coltile_c2<8>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         static_cast<int>(sizeof(Pass2Smem<8>)));
    cudaFuncSetAttribute(k_rowdot_c2<8>, cudaFuncAttributeMaxDynamicSharedMemorySize, sc2);
    cudaFuncSetAttribute(k_rowdot<false, 8, 16>, cudaFuncAttributeMaxDynamicSharedMemorySize, s16);
    cudaFuncSetAttribute(k_coltile<false, 8>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         static_cast<int>(sizeof(Pass2Smem<8>)));
    cudaFuncSetAttribute(k_coltile_mma<8>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         static_cast<int>(sizeof(MmaPass2Smem<8>)));
    cudaFuncSetAttribute(k_coltile<false, 2>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         static_cast<int>(sizeof(Pass2Smem<2>)));
    cudaFuncSetAttribute(k_coltile<false, 4>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         static_cast<int>(sizeof(Pass2Smem<4>)));
    cudaFuncSetAttribute(k_coltile_c2<2>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         static_cast<int>(sizeof(Pass2Smem<2>)));
    cudaFuncSetAttribute(k_coltile_c2<4>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         static_cast<int>(sizeof(Pass2Smem<4>)));
    int dev = 0, sms = 148, b1 = 1, b2 = 1;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&b1, k_rowdot<false>, kThreads, s1);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&b2, k_coltile<false>, kThreads2, s2);
    return Grids{sms * (b1 > 0 ? b1 : 1), sms * (b2 > 0 ? b2 : 1)};
  }();
  return g;
}

void pick_grids(const hdk_factor* f, int& g1, int& g2) {
  g1 = grids().g1 < f->n_chunks ? grids().g1 : f->n_chunks;
  g2 = grids().g2 < f->n_chunks ? grids().g2 : f->n_chunks;
  if (f->grid_cap > 0 && g1 > f->grid_cap) g1 = f->grid_cap;
  if (f->grid_cap > 0 && g2 > f->grid_cap) g2 = f->grid_cap;
  if (g2 > f->max_ctas) g2 = f->max_ctas;
}

// R-column passes only (tile partials left in part2 for the callers' folds).
template <int R>
int launch_multi(const hdk_factor* f, const double* rhs, cudaStream_t st) {
  if (f->n <= 0) return 0;
  if (f->tile_w != kW) return static_cast<int>(cudaErrorInvalidValue);
  int g1, g2;
  pick_grids(f, g1, g2);
  if (g1 != f->grid1 || g2 != f->grid2) return static_cast<int>(cudaErrorInvalidValue);
  // pass 1 is compute-bound with R columns: 16 consumer warps, 1 CTA per SM,
  // on pass 2's grid and chunk ranges
  hdk_factor f1 = *f;
  f1.first1 = f->first2;
  static const int mode1 = [] {  // pass 1: 2 = FP64 tensor cores (default), 1 = two columns per warp, 0 = one
    const char* e = std::getenv("HETERODYN_ROWDOT");
    if (e) return std::atoi(e);
    const char* c = std::getenv("HETERODYN_ROWDOT_C2");
    return (c && c[0] == '0') ? 0 : 2;
  }();
  if (mode1 == 3)
    hdk::launch(k_rowdot_mma_nb<R>, dim3(g2), dim3(32 * (kWarpsMma + 1)), sizeof(MmaPass1Smem<R>), st, f1, rhs);
  else if (mode1 == 2)
    hdk::launch(k_rowdot_mma<R>, dim3(g2), dim3(32 * (kWarpsMma + 1)), sizeof(MmaPass1Smem<R>), st, f1, rhs);
  else if (mode1 == 1) hdk::launch(k_rowdot_c2<R>, dim3(g2), dim3(kThreads), sizeof(Ring<kStagesC2>), st, f1, rhs);
  else hdk::launch(k_rowdot<false, R, 16>, dim3(g2), dim3(Pass1<16>::threads), sizeof(Ring<Pass1<16>::stages>), st, f1, rhs);
  hdk::launch(k_zreduce, dim3((f->n_ztask + 7) / 8, R), dim3(256), 0, st, *f);
  // pass 2: 2 = FP64 tensor cores (default at R = 8: 67.8 vs 85.9 us at C4),
  // 1 = two columns per warp (default at R <= 4: 50.8 vs 59.5 us), 0 = one
  static const int mode2_env = [] {
    const char* e = std::getenv("HETERODYN_COLTILE");
    if (e) return std::atoi(e);
    const char* c = std::getenv("HETERODYN_COLTILE_C2");
    return (c && c[0] == '0') ? 0 : -1;
  }();
  const int mode2 = mode2_env >= 0 ? mode2_env : (R >= 8 ? 2 : 1);
  if (mode2 == 2)
    hdk::launch(k_coltile_mma<R>, dim3(g2), dim3(32 * (kWarpsMma2 + 2)), sizeof(MmaPass2Smem<R>), st, *f);
  else if (mode2 == 1) hdk::launch(k_coltile_c2<R>, dim3(g2), dim3(kThreads2), sizeof(Pass2Smem<R>), st, *f);
  else hdk::launch(k_coltile<false, R>, dim3(g2), dim3(kThreads2), sizeof(Pass2Smem<R>), st, *f);
  return static_cast<int>(cudaGetLastError());
}

int launch(const hdk_factor* f, const double* rhs_perm, double* out, bool scatter, cudaStream_t st,
           bool fold = true, unsigned skip = 0u) {
  if (f->n <= 0) return 0;
  if (f->tile_w != kW) return static_cast<int>(cudaErrorInvalidValue);
  const size_t s1 = sizeof(Ring<kStages1>), s2 = sizeof(Pass2Smem<1>);
  int g1, g2;
  pick_grids(f, g1, g2);
  hdk_factor fl = *f;  // balanced ranges only if they were built for these grids
  if (g1 != f->grid1) fl.first1 = nullptr;
  if (g2 != f->grid2) {
    fl.first2 = nullptr;
    fl.tile_cta2 = nullptr;
  }
  const bool fp32 = f->use32 && f->sval32 && f->chunk32;  // preconditioner-only solve
  if (!(skip & 1u)) {
    if (fp32)
      hdk::launch(k_rowdot<false, 1, kWarps, float>, dim3(g1), dim3(kThreads), sizeof(Ring<kStages1, float>), st, fl,
                  rhs_perm);
    else
      hdk::launch(k_rowdot<false>, dim3(g1), dim3(kThreads), s1, st, fl, rhs_perm);
  }
  if (!(skip & 2u)) hdk::launch(k_zreduce, dim3((f->n_ztask + 7) / 8), dim3(256), 0, st, fl);
  if (!(skip & 4u)) {
    if (fp32)
      hdk::launch(k_coltile<false, 1, float>, dim3(g2), dim3(kThreads2), sizeof(Pass2Smem<1, float>), st, fl);
    else
      hdk::launch(k_coltile<false>, dim3(g2), dim3(kThreads2), s2, st, fl);
  }
  if (!fold) return static_cast<int>(cudaGetLastError());
  if (scatter)
    hdk::launch(k_xreduce<true>, dim3((f->n + 255) / 256), dim3(256), 0, st, fl, g2, out);
  else
    hdk::launch(k_xreduce<false>, dim3((f->n + 255) / 256), dim3(256), 0, st, fl, g2, out);
  return static_cast<int>(cudaGetLastError());
}

}  // namespace

extern "C" {

HDK_API int hdk_apply_inverse3(const hdk_factor* f, const double* rhs_perm, double* out_full, void* stream) {
  return launch(f, rhs_perm, out_full, true, static_cast<cudaStream_t>(stream));
}

HDK_API int hdk_solve_grids(const hdk_factor* f, int* grid1, int* grid2) {
  int g1 = 0, g2 = 0;
  pick_grids(f, g1, g2);
  if (grid1) *grid1 = g1;
  if (grid2) *grid2 = g2;
  return static_cast<int>(cudaGetLastError());
}

HDK_API int hdk_apply_inverse3_partial(const hdk_factor* f, const double* rhs_perm, void* stream) {
  return launch(f, rhs_perm, nullptr, true, static_cast<cudaStream_t>(stream), false);
}

HDK_API int hdk_apply_inverse3_ablate(const hdk_factor* f, const double* rhs_perm, unsigned skip, void* stream) {
  return launch(f, rhs_perm, nullptr, true, static_cast<cudaStream_t>(stream), false, skip);
}

HDK_API int hdk_apply_inverse3_multi(const hdk_factor* f, const double* rhs_perm, int columns, void* stream) {
  const cudaStream_t st = static_cast<cudaStream_t>(stream);
  switch (columns) {
    case 1: return launch(f, rhs_perm, nullptr, true, st, false);
    case 2: return launch_multi<2>(f, rhs_perm, st);
    case 4: return launch_multi<4>(f, rhs_perm, st);
    case 8: return launch_multi<8>(f, rhs_perm, st);
    default: return static_cast<int>(cudaErrorInvalidValue);
  }
}

HDK_API size_t hdk_factor_part2_stride(const hdk_factor* f) { return part2_stride(*f); }

HDK_API int hdk_factor_to_fp32(const hdk_factor* f, float* sval32, const hdk_chunk* chunk32, void* stream) {
  if (f->n_chunks <= 0) return 0;
  k_to_fp32<<<f->n_chunks, 256, 0, static_cast<cudaStream_t>(stream)>>>(f->sval, f->chunk, sval32, chunk32);
  return static_cast<int>(cudaGetLastError());
}

HDK_API int hdk_set_chunk_trace(long long* const* trace, void* stream) {  // trace: pinned host cell
  return static_cast<int>(cudaMemcpyToSymbolAsync(g_chunk_trace, trace, sizeof(long long*), 0,
                                                  cudaMemcpyHostToDevice, static_cast<cudaStream_t>(stream)));
}

HDK_API int hdk_apply_inverse3_perm(const hdk_factor* f, const double* rhs_perm, double* out_perm, void* stream) {
  return launch(f, rhs_perm, out_perm, false, static_cast<cudaStream_t>(stream));
}

}  // extern "C"
