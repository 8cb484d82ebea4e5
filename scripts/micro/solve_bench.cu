// Times the two streaming passes of the global solve on the real C3 factor
// layout (dumped by the host library) — wet (real consumers) vs dry (stream only).
#define HDK_SOLVE_TRACE 1
#include "../../paper_2605_14526_b200/csrc/solve.cu"
#include <cstdio>
#include <algorithm>
#include <vector>
#include <fstream>
#include "../../paper_2605_14526_b200/csrc/host.hpp"
#include <sstream>

template <class K>
float time_kernel(K k, int grid, size_t smem, const hdk_factor& f, const double* rhs, int reps) {
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  cudaEventRecord(a);
  for (int i = 0; i < reps; ++i) k(grid, smem, f, rhs);
  cudaEventRecord(b); cudaEventSynchronize(b);
  float ms; cudaEventElapsedTime(&ms, a, b);
  return ms * 1000.f / reps;
}

int main(int argc, char** argv) {
  std::ifstream in(argv[1]); std::stringstream ss; ss << in.rdbuf();
  hdb::Scene s = hdb::parse_scene(ss.str());
  hdb::HostFactor F = hdb::build_factor(s.mesh, s.material, s.solver.h, s.fixed, s.ordering);
  printf("n %d nnz %lld chunks %zu stream %zu\n", F.n, F.row_off.back(), F.chunks.size(), F.stream.size());
  hdk_factor f{};
  f.n = F.n; f.tile_w = F.tile_w; f.n_tiles = (int)F.tile_chunk.size() - 1; f.n_chunks = (int)F.chunks.size(); f.max_ctas = 148 * 8; f.grid_cap = 0;
  auto up = [](const void* h, size_t bytes) { void* d; cudaMalloc(&d, bytes); cudaMemcpy(d, h, bytes, cudaMemcpyHostToDevice); return d; };
  f.sval = (const double*)up(F.stream.data(), F.stream.size() * 8);
  f.seg = (const hdk_seg*)up(F.sdesc.data(), F.sdesc.size() * 16);
  f.chunk = (const hdk_chunk*)up(F.chunks.data(), F.chunks.size() * 24);
  f.tile_chunk = (const int*)up(F.tile_chunk.data(), F.tile_chunk.size() * 4);
  f.row_pslot = (const int*)up(F.row_pslot.data(), F.row_pslot.size() * 4);
  f.p2v = (const int*)up(F.p2v.data(), F.p2v.size() * 4);
  cudaMalloc(&f.part1, 3 * 8 * (size_t)F.row_pslot.back());
  cudaMalloc(&f.part2, 3 * 8 * (size_t)F.tile_w * (f.n_tiles + f.max_ctas));
  cudaMalloc(&f.z, 3 * 8 * (size_t)F.n);
  cudaMemset(f.z, 0, 3 * 8 * (size_t)F.n);
  std::vector<double> rhs(3 * F.n, 1.0);
  double* drhs = (double*)up(rhs.data(), rhs.size() * 8);
  double* out; cudaMalloc(&out, 3 * 8 * (size_t)F.n);
  const size_t s1 = sizeof(Ring<kStages1>), s2 = sizeof(Pass2Smem);
  cudaFuncSetAttribute(k_rowdot<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)s1);
  cudaFuncSetAttribute(k_rowdot<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)s1);
  cudaFuncSetAttribute(k_coltile<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)s2);
  cudaFuncSetAttribute(k_coltile<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)s2);
  int o1, o2; cudaOccupancyMaxActiveBlocksPerMultiprocessor(&o1, k_rowdot<false>, kThreads, s1);
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&o2, k_coltile<false>, kThreads2, s2);
  printf("smem1 %zu occ %d | smem2 %zu occ %d\n", s1, o1, s2, o2);
  const double gb = F.stream.size() * 8.0 / 1e9;
  for (int rep = 0; rep < 2; ++rep) {
    float t;
    t = time_kernel([](int g, size_t sm, const hdk_factor& f, const double* r) { k_rowdot<false><<<g, kThreads, sm>>>(f, r); }, 148 * o1, s1, f, drhs, 50);
    printf("rowdot wet  %7.2f us  %7.1f GB/s\n", t, gb / (t * 1e-6));
    t = time_kernel([](int g, size_t sm, const hdk_factor& f, const double* r) { k_rowdot<true><<<g, kThreads, sm>>>(f, r); }, 148 * o1, s1, f, drhs, 50);
    printf("rowdot dry  %7.2f us  %7.1f GB/s\n", t, gb / (t * 1e-6));
    t = time_kernel([](int g, size_t sm, const hdk_factor& f, const double* r) { k_coltile<false><<<g, kThreads2, sm>>>(f); }, 148 * o2, s2, f, drhs, 50);
    printf("coltile wet %7.2f us  %7.1f GB/s\n", t, gb / (t * 1e-6));
    t = time_kernel([](int g, size_t sm, const hdk_factor& f, const double* r) { k_coltile<true><<<g, kThreads2, sm>>>(f); }, 148 * o2, s2, f, drhs, 50);
    printf("coltile dry %7.2f us  %7.1f GB/s\n", t, gb / (t * 1e-6));
    t = time_kernel([](int g, size_t sm, const hdk_factor& f, const double* r) { k_zreduce<<<(f.n * 8 + 255) / 256, 256>>>(f); }, 0, 0, f, drhs, 50);
    printf("zreduce     %7.2f us\n", t);
    // full solve (alternating pass directions keep L2 warm)
    t = time_kernel([out](int g, size_t sm, const hdk_factor& f, const double* r) { hdk_apply_inverse3_perm(&f, r, out, 0); }, 0, 0, f, drhs, 50);
    printf("full solve  %7.2f us  (alg %7.1f GB/s)\n", t, 2 * gb / (t * 1e-6));
  }
  // cost-balanced CTA ranges: sweep the per-segment cost of both passes
  {
    const int G1 = 148 * o1, G2 = 148 * o2;
    unsigned long long* tr; cudaMalloc(&tr, 16 * (size_t)std::max(G1, G2));
    std::vector<unsigned long long> h(2 * std::max(G1, G2));
    auto spread = [&](int G, const char* what) {
      cudaMemcpy(h.data(), tr, 16 * (size_t)G, cudaMemcpyDeviceToHost);
      unsigned long long t0 = ~0ull;
      for (int b = 0; b < G; ++b) t0 = std::min(t0, h[2 * b]);
      std::vector<double> d(G);
      for (int b = 0; b < G; ++b) d[b] = (h[2 * b + 1] - t0) * 1e-3;
      std::sort(d.begin(), d.end());
      printf("    %s CTA ends: min %.2f p50 %.2f p90 %.2f max %.2f us\n", what, d[0], d[G / 2], d[G * 9 / 10], d[G - 1]);
    };
    for (double a : {0.0, 200.0, 300.0, 400.0, 600.0}) {
      std::vector<int> f1 = hdb::balanced_ranges(F.chunks, G1, a), f2 = hdb::balanced_ranges(F.chunks, G2, a);
      std::vector<int> tc = hdb::tile_cta_ranges(F.tile_chunk, f2);
      hdk_factor fb = f;
      fb.grid1 = G1; fb.grid2 = G2;
      fb.first1 = (const int*)up(f1.data(), f1.size() * 4);
      fb.first2 = (const int*)up(f2.data(), f2.size() * 4);
      fb.tile_cta2 = (const int*)up(tc.data(), tc.size() * 4);
      float t1 = time_kernel([](int g, size_t sm, const hdk_factor& f, const double* r) { k_rowdot<false><<<g, kThreads, sm>>>(f, r); }, G1, s1, fb, drhs, 50);
      float t2 = time_kernel([](int g, size_t sm, const hdk_factor& f, const double* r) { k_coltile<false><<<g, kThreads2, sm>>>(f); }, G2, s2, fb, drhs, 50);
      float t3 = time_kernel([out](int g, size_t sm, const hdk_factor& f, const double* r) { hdk_apply_inverse3_perm(&f, r, out, 0); }, 0, 0, fb, drhs, 50);
      printf("seg cost %5.0f: rowdot %.2f us  coltile %.2f us  full %.2f us (alg %.1f GB/s)\n", a, t1, t2, t3, 2 * gb / (t3 * 1e-6));
      cudaMemcpyToSymbol(g_cta_trace, &tr, sizeof(tr));
      k_rowdot<false><<<G1, kThreads, s1>>>(fb, drhs); cudaDeviceSynchronize(); spread(G1, "rowdot ");
      k_coltile<false><<<G2, kThreads2, s2>>>(fb); cudaDeviceSynchronize(); spread(G2, "coltile");
      unsigned long long* nul = nullptr;
      cudaMemcpyToSymbol(g_cta_trace, &nul, sizeof(nul));
    }
  }
  printf("err %s\n", cudaGetErrorString(cudaGetLastError()));
}
