// Microbenchmark: streaming read bandwidth on B200 — cp.async.bulk rings vs LDG.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t sa(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(uint64_t* b, uint32_t c) { asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(sa(b)), "r"(c) : "memory"); }
__device__ __forceinline__ void expect_tx(uint64_t* b, uint32_t n) { asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(sa(b)), "r"(n) : "memory"); }
__device__ __forceinline__ void bulk(void* d, const void* s, uint32_t n, uint64_t* b) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(sa(d)), "l"(s), "r"(n), "r"(sa(b)) : "memory"); }
__device__ __forceinline__ void wait(uint64_t* b, uint32_t ph) {
  asm volatile("{\n.reg .pred p;\nW_%=:\nmbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n@!p bra W_%=;\n}\n" ::"r"(sa(b)), "r"(ph) : "memory"); }

template <int CH, int ST, bool RANGE>
__global__ void k_bulk(const double* __restrict__ src, size_t n, double* out) {
  extern __shared__ __align__(128) unsigned char sm[];
  double* buf = (double*)sm;
  uint64_t* full = (uint64_t*)(sm + (size_t)ST * CH * 8);
  const size_t nch = n / CH;
  if (threadIdx.x == 0) { for (int s = 0; s < ST; ++s) mbar_init(&full[s], 1); asm volatile("fence.mbarrier_init.release.cluster;"); }
  __syncthreads();
  const size_t step = RANGE ? 1 : gridDim.x;
  const size_t cb = RANGE ? blockIdx.x * nch / gridDim.x : blockIdx.x;
  const size_t ce = RANGE ? (blockIdx.x + 1) * nch / gridDim.x : nch;
  size_t c = cb, cp = cb;
  if (threadIdx.x == 0) for (int s = 0; s < ST && cp < ce; ++s, cp += step) { expect_tx(&full[s], CH * 8); bulk(buf + (size_t)s * CH, src + cp * CH, CH * 8, &full[s]); }
  double acc = 0;
  for (int k = 0; c < ce; ++k, c += step) {
    const int st = k % ST;
    wait(&full[st], (k / ST) & 1);
    for (int i = threadIdx.x; i < CH; i += blockDim.x) acc += buf[(size_t)st * CH + i];
    __syncthreads();
    if (threadIdx.x == 0 && cp < ce) { asm volatile("fence.proxy.async.shared::cta;"); expect_tx(&full[st], CH * 8); bulk(buf + (size_t)st * CH, src + cp * CH, CH * 8, &full[st]); cp += step; }
  }
  if (acc == 12345.678) out[0] = acc;
}

__global__ void k_ldg(const double2* __restrict__ src, size_t n2, double* out) {
  double acc = 0;
  size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x, stride = (size_t)gridDim.x * blockDim.x;
  for (; i + 3 * stride < n2; i += 4 * stride) {
    double2 a = __ldg(src + i), b = __ldg(src + i + stride), c = __ldg(src + i + 2 * stride), d = __ldg(src + i + 3 * stride);
    acc += a.x + a.y + b.x + b.y + c.x + c.y + d.x + d.y;
  }
  for (; i < n2; i += stride) { double2 a = __ldg(src + i); acc += a.x + a.y; }
  if (acc == 12345.678) out[0] = acc;
}

template <int CH, int ST, bool RANGE = false>
float run_bulk(const double* d, size_t n, double* out, int blocks_per_sm, int threads) {
  size_t smem = (size_t)ST * CH * 8 + ST * 8;
  cudaFuncSetAttribute(k_bulk<CH, ST, RANGE>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  int occ = 0; cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k_bulk<CH, ST, RANGE>, threads, smem);
  int bps = blocks_per_sm < occ ? blocks_per_sm : occ;
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  k_bulk<CH, ST, RANGE><<<148 * bps, threads, smem>>>(d, n, out);
  cudaEventRecord(a);
  for (int r = 0; r < 5; ++r) k_bulk<CH, ST, RANGE><<<148 * bps, threads, smem>>>(d, n, out);
  cudaEventRecord(b); cudaEventSynchronize(b);
  float ms; cudaEventElapsedTime(&ms, a, b);
  double gbs = 5.0 * n * 8 / (ms / 1e3) / 1e9;
  printf("bulk %s CH=%5d ST=%d smem=%6zu bps=%d(occ %d) thr=%d : %8.1f GB/s  err=%s\n", RANGE ? "range" : "inter", CH, ST, smem, bps, occ, threads, gbs, cudaGetErrorString(cudaGetLastError()));
  return (float)gbs;
}

int main() {
  size_t n = (size_t)1 << 27;  // 1 GiB of doubles
  double *d, *out; cudaMalloc(&d, n * 8); cudaMalloc(&out, 8); cudaMemset(d, 0, n * 8);
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  for (int bl : {1, 2, 4, 8}) {
    k_ldg<<<148 * bl, 256>>>((const double2*)d, n / 2, out);
    cudaEventRecord(a);
    for (int r = 0; r < 5; ++r) k_ldg<<<148 * bl, 256>>>((const double2*)d, n / 2, out);
    cudaEventRecord(b); cudaEventSynchronize(b);
    float ms; cudaEventElapsedTime(&ms, a, b);
    printf("ldg128 blocks/SM=%d : %8.1f GB/s\n", bl, 5.0 * n * 8 / (ms / 1e3) / 1e9);
  }
  run_bulk<3072, 3>(d, n, out, 2, 256);
  run_bulk<3072, 3, true>(d, n, out, 2, 256);
  run_bulk<3072, 2, true>(d, n, out, 2, 256);
  run_bulk<3072, 3, true>(d, n / 6, out, 2, 256);
  run_bulk<3072, 3, false>(d, n / 6, out, 2, 256);
  run_bulk<3072, 4, true>(d, n / 6, out, 1, 288);
  return 0;
}
