// heterodyn-b200 host library: scene/mesh/material setup, the explicit inverse
// factor build, and the device-resident forward/backward engine.  This is the
// product's C++ solver API (the reference's is in /root/reference/proj/src
// mesh.hpp, material.hpp, factor.hpp, forward.hpp, backward.hpp); the hot
// path runs on sm_100a through the hdk_* launchers (include/hdk.h).
#pragma once

#include <algorithm>
#include <array>
#include <cstdint>
#include <exception>
#include <stdexcept>
#include <string>
#include <thread>
#include <vector>

namespace hdb {

// common.hpp:19-45 numbering (identical to hd_status).
enum class Code : int {
  Ok = 0, Parse = 1, Validation = 2, DegenerateElement = 3, InvalidPoisson = 4, NonPositiveJacobian = 5,
  ProxDiverged = 6, SingularFilteredHessian = 7, NotPositiveDefinite = 8, SingularContactSystem = 9,
  AdjointDiverged = 10, LineSearchFailed = 11, Io = 12, InvalidArgument = 13,
};
struct Error : std::runtime_error {
  Code code;
  Error(Code c, const std::string& m) : std::runtime_error(m), code(c) {}
};
[[noreturn]] inline void raise(Code c, const std::string& m) { throw Error(c, m); }

using Vec = std::vector<double>;

// fn(lo, hi) over [0, n) split into contiguous ranges on up to `workers`
// host threads (0 = hardware threads); the first exception is rethrown.
template <class F>
void parallel_ranges(long long n, F&& fn, int workers = 0, long long grain = 4096) {
  int w = workers > 0 ? workers : static_cast<int>(std::thread::hardware_concurrency());
  w = static_cast<int>(std::max<long long>(1, std::min<long long>({static_cast<long long>(w), 64LL, n / grain})));
  if (w <= 1) {
    fn(0LL, n);
    return;
  }
  std::vector<std::thread> pool;
  std::vector<std::exception_ptr> errs(w);
  for (int t = 0; t < w; ++t)
    pool.emplace_back([&, t] {
      try {
        fn(n * t / w, n * (t + 1) / w);
      } catch (...) {
        errs[t] = std::current_exception();
      }
    });
  for (auto& th : pool) th.join();
  for (auto& e : errs)
    if (e) std::rethrow_exception(e);
}
struct P3 { double x = 0, y = 0, z = 0; };

// Tetrahedral mesh (mesh.hpp:16-60).  bm holds Dm^{-1} row-major per element.
struct Mesh {
  int nv = 0, ne = 0;
  Vec rest;                             // 3 nv
  std::vector<std::array<int, 4>> el;   // ne
  Vec bm;                               // 9 ne
  Vec vol;                              // ne
  Vec mass;                             // nv (per vertex; every axis equal)
  std::vector<int> boundary;
  std::uint64_t topology = 0;
  double total_volume = 0;
};
Mesh make_mesh(const Vec& rest, const std::vector<std::array<int, 4>>& el, double density);
Mesh hex_grid(int nx, int ny, int nz, double spacing, double density);

enum class Kind { Corotated = 0, NeoHookean = 1 };
// Heterogeneous material field (material.hpp:60-90).
struct Material {
  Kind kind = Kind::NeoHookean;
  bool barrier = false;
  double poisson = 0, alpha = 0, beta0 = 0;
  Vec young, mu, lambda, beta;
  double mu_bar = 0, lambda_bar = 0, k_bar = 0;
  bool frozen = false;
  std::uint64_t version = 0;
  Vec seg_means;  // lockstep batch: (mu, lambda, k) prox means per sample (empty otherwise)
  double weight(int e) const { return 2.0 * mu[e] + lambda[e]; }
  double contrast() const;
  void set_young(const Vec& y, const Vec& vol);
  void freeze();
};
Material make_material(const Mesh& m, const Vec& young, double poisson, Kind kind, bool barrier, double alpha,
                       double beta0);

struct Obstacle {  // contact.hpp:18-26
  int kind = 0;    // 0 half-space, 1 sphere
  P3 normal{0, 1, 0};
  double offset = 0;
  P3 center;
  double radius = 1, friction = 0;
};

struct Solver {  // forward.hpp:19-27
  double h = 0.01, eps_rel = 1e-4, eps_abs = 1e-9;
  int k_max = 500;
  double eps_tr = 0.1;
  int aa_window = 0;
  double contact_margin = 1e-4;
};

struct Scene {  // scene.hpp:14-34
  std::string name;
  Mesh mesh;
  Material material;
  std::vector<int> fixed;
  std::vector<Obstacle> obstacles;
  P3 gravity;
  Vec f_extra;
  bool hook = false;
  int hook_vertex = -1;
  P3 hook_anchor;
  double hook_k = 0, hook_d = 0;
  Solver solver;
  int frames = 1;
  Vec q0, v0;
  std::vector<int> region;
  int region_count = 0;
  std::string ordering = "nd-mvc";  // B200 extension: fill-reducing ordering of the factor
};
Scene parse_scene(const std::string& text);
Scene builtin_scene(const std::string& name);
Vec external_force(const Scene& s);  // gravity lumped + point forces (scene.cpp:530-540)
// A lockstep batch of `samples` copies of `s` (contact-free, no Dirichlet
// vertices, no state hook): vertex / element index spaces concatenated, each
// copy's material built from its own moduli (young: samples x ne, NULL = the
// scene's), per-copy prox means kept in material.seg_means (engine.cpp
// segments > 1).
Scene make_segmented_scene(const Scene& s, int samples, const double* young);
void segmented_set_young(Material& mat, const Vec& young, const Vec& vol, int samples);

// Scalar CSR (rows in elimination order).
struct Csr {
  int rows = 0, cols = 0;
  std::vector<int> off, col;
  Vec val;
};

// Explicit inverse factor A_ff^{-1} = S'^T S' (see hdk.h for the layout).
struct Segment { long long off; int row, clo, len, pslot; };  // off: row-major sval
struct SegDesc { int row, pslot, clo_len, coff; };              // device descriptor (hdk_seg)
struct ChunkDesc { long long off; int len, seg0, nseg, tile; };  // device chunk (hdk_chunk)
// Inputs of the device-side S' value build (inverse.cu): the postordered
// elimination tree, L by columns with each entry's depth distance, D^{-1/2},
// and where every (row, tile) segment sits in the value stream.
struct DeviceBuild {
  std::vector<int> parent, depth, ldist, row_first, seg_clo;
  std::vector<long long> lp, seg_off;
  std::vector<int> li;  // L row indices by column (the device refactorization's symbolic input)
  Vec lx, dis;
  int max_depth = 0;
};
struct HostFactor {
  int n = 0, nv = 0;
  std::vector<int> p2v, v2p, fixed;
  std::vector<long long> row_off;
  std::vector<int> row_len;
  Vec sval;
  int tile_w = 256;
  std::vector<Segment> seg;
  std::vector<int> row_pslot;
  // tile-major stream for the device passes
  Vec stream;
  std::vector<SegDesc> sdesc;
  std::vector<ChunkDesc> chunks;
  std::vector<int> tile_chunk;
  Csr a_ff;  // free x free, elimination order
  Csr a_fd;  // free rows (elimination order) x fixed columns (index into fixed)
  long long l_nnz = 0;
  long long stream_len = 0;  // values in the tile-major stream (F.stream holds them unless built on the device)
  DeviceBuild build;         // filled when build_factor(..., device_values = true)
  double millis = 0;
  double ms_phase[5] = {};  // cumulative ms after assembly, ordering, etree, LDL^T, S' values
  std::string ordering;
  double weight_contrast = 1;
};
// Cost-balanced contiguous chunk ranges for G persistent CTAs: chunk cost =
// values + seg_cost * segments; G + 1 boundaries, every range non-empty when
// chunks >= G.
std::vector<int> balanced_ranges(const std::vector<ChunkDesc>& chunks, int G, double seg_cost);
// For each tile, the first and last CTA (of the ranges `first`) owning one of
// its chunks (2 * n_tiles entries).
std::vector<int> tile_cta_ranges(const std::vector<int>& tile_chunk, const std::vector<int>& first);
// Setup-time self-check of a built factor on the host: max over three axes of
// |A_ff S'^T S' b - b| / |b| for a deterministic b (no solve path runs here).
double factor_inverse_residual(const HostFactor& F);
// order_cache: when it holds an ordering of the same size it is used as is
// (the ordering depends only on the graph of the free vertices); otherwise
// the computed ordering is stored into it.  prev: the factor being replaced;
// its stream layout is reused when the new elimination order and row lengths
// match (device-built values only).
HostFactor build_factor(const Mesh& mesh, const Material& mat, double h, const std::vector<int>& fixed,
                        const std::string& ordering, bool device_values = false,
                        std::vector<int>* order_cache = nullptr, const HostFactor* prev = nullptr);

}  // namespace hdb
