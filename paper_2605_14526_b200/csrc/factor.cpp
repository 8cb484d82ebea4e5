// Explicit inverse factor for the B200 global solve (host build, once per
// material/topology/Dirichlet change — reference GlobalSystem::refresh and
// SparseFactor::factorize, factor.cpp:11-104, 121-184).
//
//   A = (1 + alpha h) M / h^2 + sum_e (w_e + beta_e / h) V_e g g^T  (scalar, per axis)
//   P A_ff P^T = L D L^T,  S' = D^{-1/2} L^{-1},  A_ff^{-1} = P^T S'^T S' P.
//
// B200-first choices (same operator, different layout):
//  * ordering "nd-mvc" (default): nested dissection whose separators are
//    minimum vertex covers between adjacent BFS levels, chosen by a model of
//    nnz(S') (the sum of elimination-tree depths); "nd-bfs" is the
//    reference's BFS-level scheme (ordering.cpp:73-144) with natural order in
//    leaves and separators; "nd-geometric" coordinate bisection; "metis"
//    cuSOLVER's METIS.  Measured nnz(S') at C3: nd-mvc 19.82 M, nd-bfs
//    21.17 M, metis 22.13 M, nd-geometric 24.95 M;
//  * the elimination order is postordered, so every row of S' is dense over a
//    contiguous column range (its etree subtree) and is stored without column
//    indices;
//  * rows are cut into 256-column tile segments, packed tile-major into
//    16-byte aligned chunks that the two streaming passes (solve.cu) split
//    evenly over persistent CTAs.
#include <algorithm>
#include <atomic>
#include <condition_variable>
#include <mutex>
#include <exception>
#include <chrono>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <functional>
#include <numeric>
#include <set>
#include <thread>

#include <cusolverSp.h>

#include "host.hpp"

namespace hdb {

namespace {
constexpr int HDK_VALS = 3072;  // == HDK_CHUNK_VALS (include/hdk.h)
constexpr int HDK_SEGS = 64;    // == HDK_CHUNK_SEGS

int hw_threads() {
  int n = static_cast<int>(std::thread::hardware_concurrency());
  return std::max(1, std::min(n, 64));
}

template <class F>
void parallel_chunks(int n, F&& fn) {
  const int w = std::min(hw_threads(), std::max(1, n / 64));
  if (w <= 1) {
    fn(0, n, 0);
    return;
  }
  std::vector<std::thread> pool;
  for (int t = 0; t < w; ++t) {
    const int lo = static_cast<int>(static_cast<long long>(n) * t / w), hi = static_cast<int>(static_cast<long long>(n) * (t + 1) / w);
    pool.emplace_back([&fn, lo, hi, t] { fn(lo, hi, t); });
  }
  for (auto& th : pool) th.join();
}

// Scalar operator over all vertices; duplicates summed in sorted order and
// exact zeros dropped (csr.cpp:7-32), so the graph matches the reference's.
// Row-parallel assembly: each vertex row gathers its incident elements'
// contributions (vertex -> element incidence), sums equal columns in a fixed
// order (inertia first, then elements ascending) and drops exact zeros like
// csr.cpp:24.  Same operator as the triplet sort of csr.cpp:9-31; the
// summation order within an entry is fixed here instead of sort-dependent.
Csr assemble(const Mesh& m, const Material& mat, double h) {
  if (!(h > 0)) raise(Code::Validation, "step size must be positive");
  const int nv = m.nv, ne = m.ne;
  std::vector<int> inc_off(nv + 1, 0), inc(4 * static_cast<size_t>(ne));
  for (int e = 0; e < ne; ++e)
    for (int i = 0; i < 4; ++i) ++inc_off[m.el[e][i] + 1];
  for (int v = 0; v < nv; ++v) inc_off[v + 1] += inc_off[v];
  {
    std::vector<int> cur(inc_off.begin(), inc_off.end() - 1);
    for (int e = 0; e < ne; ++e)
      for (int i = 0; i < 4; ++i) inc[cur[m.el[e][i]]++] = 4 * e + i;  // ascending e per vertex
  }
  // per element: w_e V_e and the four shape gradients
  std::vector<double> G(12 * static_cast<size_t>(ne)), W(ne);
  parallel_chunks(ne, [&](int lo, int hi, int) {
    for (int e = lo; e < hi; ++e) {
      W[e] = (mat.weight(e) + mat.beta[e] / h) * m.vol[e];
      const double* b = &m.bm[9 * static_cast<size_t>(e)];
      double* g = &G[12 * static_cast<size_t>(e)];
      for (int c = 0; c < 3; ++c) {
        g[3 + c] = b[0 * 3 + c];
        g[6 + c] = b[1 * 3 + c];
        g[9 + c] = b[2 * 3 + c];
        g[c] = -(g[3 + c] + g[6 + c] + g[9 + c]);
      }
    }
  });
  const double inertia = (1.0 + mat.alpha * h) / (h * h);
  std::vector<std::vector<std::pair<int, double>>> rows(nv);
  parallel_chunks(nv, [&](int lo, int hi, int) {
    std::vector<std::pair<int, double>> t;
    for (int v = lo; v < hi; ++v) {
      t.clear();
      t.push_back({v, inertia * m.mass[v]});
      for (int k = inc_off[v]; k < inc_off[v + 1]; ++k) {
        const int e = inc[k] >> 2, i = inc[k] & 3;
        const double* g = &G[12 * static_cast<size_t>(e)];
        for (int j = 0; j < 4; ++j)
          t.push_back({m.el[e][j], W[e] * (g[3 * i] * g[3 * j] + g[3 * i + 1] * g[3 * j + 1] + g[3 * i + 2] * g[3 * j + 2])});
      }
      std::stable_sort(t.begin(), t.end(), [](const auto& a, const auto& b) { return a.first < b.first; });
      auto& r = rows[v];
      for (size_t q = 0; q < t.size();) {
        const int c = t[q].first;
        double sum = 0;
        while (q < t.size() && t[q].first == c) sum += t[q++].second;
        if (sum != 0.0) r.push_back({c, sum});
      }
    }
  });
  Csr a;
  a.rows = a.cols = nv;
  a.off.assign(nv + 1, 0);
  for (int v = 0; v < nv; ++v) a.off[v + 1] = a.off[v] + static_cast<int>(rows[v].size());
  a.col.resize(a.off[nv]);
  a.val.resize(a.off[nv]);
  parallel_chunks(nv, [&](int lo, int hi, int) {
    for (int v = lo; v < hi; ++v)
      for (size_t q = 0; q < rows[v].size(); ++q) {
        a.col[a.off[v] + q] = rows[v][q].first;
        a.val[a.off[v] + q] = rows[v][q].second;
      }
  });
  return a;
}

// ---- orderings ---------------------------------------------------------------
using Graph = std::vector<std::vector<int>>;

// Nested dissection by recursive coordinate bisection.  The separator is the
// set of upper-half vertices adjacent to the lower half, which is a grid
// plane when the median falls on one.
void nd_geometric(const Graph& g, const std::vector<P3>& x, std::vector<int> blk, std::vector<int>& out,
                  std::vector<char>& side) {
  if (blk.size() <= 64) {
    std::sort(blk.begin(), blk.end());
    out.insert(out.end(), blk.begin(), blk.end());
    return;
  }
  double lo[3] = {1e300, 1e300, 1e300}, hi[3] = {-1e300, -1e300, -1e300};
  for (int v : blk) {
    const double c[3] = {x[v].x, x[v].y, x[v].z};
    for (int a = 0; a < 3; ++a) {
      lo[a] = std::min(lo[a], c[a]);
      hi[a] = std::max(hi[a], c[a]);
    }
  }
  int axes[3] = {0, 1, 2};
  std::sort(axes, axes + 3, [&](int a, int b) { return hi[a] - lo[a] > hi[b] - lo[b]; });
  auto coord = [&](int v, int a) { return a == 0 ? x[v].x : a == 1 ? x[v].y : x[v].z; };
  for (int ai = 0; ai < 3; ++ai) {
    const int a = axes[ai];
    if (!(hi[a] > lo[a])) break;
    std::vector<double> cs(blk.size());
    for (size_t i = 0; i < blk.size(); ++i) cs[i] = coord(blk[i], a);
    std::nth_element(cs.begin(), cs.begin() + cs.size() / 2, cs.end());
    double med = cs[cs.size() / 2];
    if (med <= lo[a]) {  // keep both sides nonempty
      double next = 1e300;
      for (double c : cs)
        if (c > lo[a]) next = std::min(next, c);
      med = next;
    }
    std::vector<int> left, right, sep;
    for (int v : blk) side[v] = coord(v, a) < med ? 1 : 2;
    for (int v : blk) {
      if (side[v] == 1) {
        left.push_back(v);
        continue;
      }
      bool touches = false;
      for (int w : g[v])
        if (side[w] == 1) { touches = true; break; }
      (touches ? sep : right).push_back(v);
    }
    for (int v : blk) side[v] = 0;
    if (left.empty() || (right.empty() && sep.size() == blk.size())) continue;
    nd_geometric(g, x, std::move(left), out, side);
    nd_geometric(g, x, std::move(right), out, side);
    std::sort(sep.begin(), sep.end());
    out.insert(out.end(), sep.begin(), sep.end());
    return;
  }
  std::sort(blk.begin(), blk.end());
  out.insert(out.end(), blk.begin(), blk.end());
}

// Nested dissection by BFS level bisection (the reference's scheme,
// ordering.cpp:73-156) with natural order on leaves and separators.
void nd_bfs(const Graph& g, std::vector<int> blk, std::vector<int>& out, std::vector<int>& level,
            std::vector<char>& mark) {
  if (blk.size() <= 48) {
    std::sort(blk.begin(), blk.end());
    out.insert(out.end(), blk.begin(), blk.end());
    return;
  }
  for (int v : blk) mark[v] = 1;
  auto bfs = [&](int root, std::vector<int>& order) {
    for (int v : blk) level[v] = -1;
    order.clear();
    order.push_back(root);
    level[root] = 0;
    for (size_t h = 0; h < order.size(); ++h)
      for (int w : g[order[h]])
        if (mark[w] && level[w] < 0) {
          level[w] = level[order[h]] + 1;
          order.push_back(w);
        }
  };
  std::vector<int> order;
  bfs(blk.front(), order);
  if (order.size() < blk.size()) {
    std::vector<int> rest;
    for (int v : blk)
      if (level[v] < 0) rest.push_back(v);
    for (int v : blk) mark[v] = 0;
    nd_bfs(g, order, out, level, mark);
    nd_bfs(g, rest, out, level, mark);
    return;
  }
  int root = blk.front();
  for (int s = 0; s < 2; ++s) {
    bfs(root, order);
    root = order.back();
  }
  bfs(root, order);
  int maxl = 0;
  for (int v : blk) maxl = std::max(maxl, level[v]);
  for (int v : blk) mark[v] = 0;
  if (maxl < 2) {
    std::sort(blk.begin(), blk.end());
    out.insert(out.end(), blk.begin(), blk.end());
    return;
  }
  std::vector<int> cnt(maxl + 1, 0);
  for (int v : blk) ++cnt[level[v]];
  int split = 0, cum = 0;
  while (split < maxl && cum + cnt[split] < static_cast<int>(blk.size()) / 2) cum += cnt[split++];
  split = std::min(std::max(split, 1), maxl - 1);
  std::vector<int> l, r, s;
  for (int v : blk) (level[v] < split ? l : level[v] > split ? r : s).push_back(v);
  nd_bfs(g, std::move(l), out, level, mark);
  nd_bfs(g, std::move(r), out, level, mark);
  std::sort(s.begin(), s.end());
  out.insert(out.end(), s.begin(), s.end());
}

// Nested dissection tuned for the explicit-inverse factor, whose size is
// nnz(S') = sum over vertices of their elimination-tree depth: a separator S
// of a block B adds about |S| |B| to it.  Per block: BFS level structures from
// a few pseudo-peripheral roots; for every split level k in the balanced
// window the separator is a minimum vertex cover of the edges between levels
// k and k+1 (Koenig, by bipartite matching), and the candidate with the least
// estimated cost |S| |B| + c (|A|^(5/3) + |B'|^(5/3)) wins.
struct MvcScratch {
  std::vector<int> level, idx;
  std::vector<char> mark;
};

// Minimum vertex cover of the bipartite graph between vertex sets X (level k)
// and Y (level k+1) restricted to the block; returns the cover.
std::vector<int> min_cover(const Graph& g, const std::vector<int>& X, const std::vector<int>& Y, MvcScratch& w) {
  // local indices
  for (size_t i = 0; i < X.size(); ++i) w.idx[X[i]] = static_cast<int>(i);
  for (size_t j = 0; j < Y.size(); ++j) w.idx[Y[j]] = static_cast<int>(j);
  const int nx = static_cast<int>(X.size()), ny = static_cast<int>(Y.size());
  std::vector<std::vector<int>> adj(nx);
  const int ly = w.level[Y.empty() ? X[0] : Y[0]];
  for (int i = 0; i < nx; ++i)
    for (int u : g[X[i]])
      if (w.mark[u] && w.level[u] == ly) adj[i].push_back(w.idx[u]);
  std::vector<int> mx(nx, -1), my(ny, -1), vis(ny, -1);
  std::function<bool(int, int)> aug = [&](int i, int st) -> bool {
    for (int j : adj[i]) {
      if (vis[j] == st) continue;
      vis[j] = st;
      if (my[j] < 0 || aug(my[j], st)) {
        mx[i] = j;
        my[j] = i;
        return true;
      }
    }
    return false;
  };
  for (int i = 0; i < nx; ++i) aug(i, i);
  // Koenig: Z = vertices reachable from unmatched X by alternating paths;
  // cover = (X \ Z) u (Y n Z)
  std::vector<char> zx(nx, 0), zy(ny, 0);
  std::vector<int> stack;
  for (int i = 0; i < nx; ++i)
    if (mx[i] < 0) {
      zx[i] = 1;
      stack.push_back(i);
    }
  while (!stack.empty()) {
    const int i = stack.back();
    stack.pop_back();
    for (int j : adj[i])
      if (!zy[j]) {
        zy[j] = 1;
        const int i2 = my[j];
        if (i2 >= 0 && !zx[i2]) {
          zx[i2] = 1;
          stack.push_back(i2);
        }
      }
  }
  std::vector<int> cover;
  for (int i = 0; i < nx; ++i)
    if (!zx[i]) cover.push_back(X[i]);
  for (int j = 0; j < ny; ++j)
    if (zy[j]) cover.push_back(Y[j]);
  return cover;
}

// Returns the model cost of the ordering it appends: separators as chains,
// cost(B) = cost(pieces) + |S| (|B| - |S|) + |S| (|S| + 1) / 2 (the sum of
// elimination-tree depths within B).  `look` > 0: the best `look` candidate
// separators (by the estimate) are each ordered in full and the cheapest by
// the model is kept.  (On C3 a 12-candidate look-ahead at the top of the tree
// and grid-plane candidates both matched the greedy choice, so the default
// is greedy.)
double nd_mvc(const Graph& g, std::vector<int> blk, std::vector<int>& out, MvcScratch& w, int look = 0) {
  const double nb = static_cast<double>(blk.size());
  if (blk.size() <= 48) {
    std::sort(blk.begin(), blk.end());
    out.insert(out.end(), blk.begin(), blk.end());
    return nb * (nb + 1) / 2;  // dense leaf: a chain
  }
  for (int v : blk) w.mark[v] = 1;
  auto bfs = [&](int root, std::vector<int>& order) {
    for (int v : blk) w.level[v] = -1;
    order.clear();
    order.push_back(root);
    w.level[root] = 0;
    for (size_t h = 0; h < order.size(); ++h)
      for (int u : g[order[h]])
        if (w.mark[u] && w.level[u] < 0) {
          w.level[u] = w.level[order[h]] + 1;
          order.push_back(u);
        }
  };
  std::vector<int> order;
  bfs(blk.front(), order);
  if (order.size() < blk.size()) {  // disconnected: components one after another
    std::vector<int> rest;
    for (int v : blk)
      if (w.level[v] < 0) rest.push_back(v);
    for (int v : blk) w.mark[v] = 0;
    double c = nd_mvc(g, order, out, w, look);
    c += nd_mvc(g, rest, out, w, look);
    return c;
  }
  // estimate constants fitted on C3 (nnz(S') 21.17 M nd-bfs -> 19.82 M)
  constexpr double kC = 2.0, kLo = 0.3;
  auto est = [](double m) { return kC * std::pow(m, 5.0 / 3.0); };
  struct Cand {
    double cost;
    std::vector<int> sep;
  };
  std::vector<Cand> cands;
  std::vector<int> roots;
  {  // pseudo-peripheral roots: the classic double sweep, then the far ends of two more sweeps
    int r = blk.front();
    for (int s2 = 0; s2 < 2; ++s2) {
      bfs(r, order);
      r = order.back();
    }
    roots.push_back(r);
    bfs(r, order);
    roots.push_back(order.back());
    bfs(order.back(), order);
    roots.push_back(order[order.size() / 2]);
  }
  for (int root : roots) {
    bfs(root, order);
    int maxl = 0;
    for (int v : blk) maxl = std::max(maxl, w.level[v]);
    if (maxl < 2) continue;
    std::vector<std::vector<int>> lv(maxl + 1);
    for (int v : order) lv[w.level[v]].push_back(v);
    int cum = 0;
    for (int k = 0; k < maxl; ++k) {
      cum += static_cast<int>(lv[k].size());  // levels <= k
      const double f = cum / nb;
      if (f < kLo || f > 1.0 - kLo) continue;
      std::vector<int> sep = min_cover(g, lv[k], lv[k + 1], w);
      const double cost = static_cast<double>(sep.size()) * nb + est(cum) + est(nb - cum);
      cands.push_back({cost, std::move(sep)});
    }
  }
  for (int v : blk) w.mark[v] = 0;
  if (cands.empty()) {
    std::sort(blk.begin(), blk.end());
    out.insert(out.end(), blk.begin(), blk.end());
    return nb * (nb + 1) / 2;
  }
  std::sort(cands.begin(), cands.end(), [](const Cand& a, const Cand& b) { return a.cost < b.cost; });
  const int tries = look > 0 ? std::min<int>(look, static_cast<int>(cands.size())) : 1;
  double best = 1e300;
  std::vector<int> best_order;
  for (int c = 0; c < tries; ++c) {
    std::vector<int>& sep = cands[c].sep;
    for (int v : blk) w.mark[v] = 1;
    for (int v : sep) w.mark[v] = 0;
    std::vector<int> restv;
    for (int v : blk)
      if (w.mark[v]) restv.push_back(v);
    for (int v : blk) w.mark[v] = 0;
    std::vector<int> sub;
    const double ns = static_cast<double>(sep.size());
    const double cost = nd_mvc(g, restv, sub, w, 0) + ns * (nb - ns) + ns * (ns + 1) / 2;
    if (cost < best) {
      best = cost;
      std::sort(sep.begin(), sep.end());
      sub.insert(sub.end(), sep.begin(), sep.end());
      best_order = std::move(sub);
    }
  }
  out.insert(out.end(), best_order.begin(), best_order.end());
  return best;
}

// METIS nested dissection through cuSOLVER's host entry point
// (cusolverSpXcsrmetisndHost); the etree postorder below is applied on top.
void metis_nd(const Graph& g, std::vector<int>& out) {
  const int n = static_cast<int>(g.size());
  std::vector<int> rp(n + 1, 0), ci;
  for (int i = 0; i < n; ++i) {
    std::vector<int> row = g[i];
    row.push_back(i);
    std::sort(row.begin(), row.end());
    ci.insert(ci.end(), row.begin(), row.end());
    rp[i + 1] = static_cast<int>(ci.size());
  }
  cusolverSpHandle_t h = nullptr;
  if (cusolverSpCreate(&h) != CUSOLVER_STATUS_SUCCESS) raise(Code::InvalidArgument, "factor: cusolverSpCreate failed");
  cusparseMatDescr_t d = nullptr;
  cusparseCreateMatDescr(&d);
  cusparseSetMatType(d, CUSPARSE_MATRIX_TYPE_GENERAL);
  cusparseSetMatIndexBase(d, CUSPARSE_INDEX_BASE_ZERO);
  out.assign(n, 0);
  const cusolverStatus_t st = cusolverSpXcsrmetisndHost(h, n, rp[n], d, rp.data(), ci.data(), nullptr, out.data());
  cusparseDestroyMatDescr(d);
  cusolverSpDestroy(h);
  if (st != CUSOLVER_STATUS_SUCCESS) raise(Code::InvalidArgument, "factor: METIS ordering failed");
}

}  // namespace

HostFactor build_factor(const Mesh& mesh, const Material& mat, double h, const std::vector<int>& fixed,
                        const std::string& ordering, bool device_values, std::vector<int>* order_cache,
                        const HostFactor* prev) {
  const auto t0 = std::chrono::steady_clock::now();
  HostFactor F;
  F.nv = mesh.nv;
  F.fixed = fixed;
  F.ordering = ordering;
  F.weight_contrast = mat.contrast();
  std::vector<char> is_fixed(mesh.nv, 0);
  for (int v : fixed) is_fixed[v] = 1;
  std::vector<int> freev;
  for (int v = 0; v < mesh.nv; ++v)
    if (!is_fixed[v]) freev.push_back(v);
  const int n = static_cast<int>(freev.size());
  if (n == 0) raise(Code::Validation, "all vertices are constrained");
  F.n = n;
  std::vector<int> v2f(mesh.nv, -1), fixed_idx(mesh.nv, -1);
  for (int i = 0; i < n; ++i) v2f[freev[i]] = i;
  for (size_t i = 0; i < fixed.size(); ++i) fixed_idx[fixed[i]] = static_cast<int>(i);

  const Csr A = assemble(mesh, mat, h);
  // Free-free graph (free index space).
  Graph g(n);
  for (int i = 0; i < n; ++i) {
    const int v = freev[i];
    for (int k = A.off[v]; k < A.off[v + 1]; ++k) {
      const int w = v2f[A.col[k]];
      if (w >= 0 && w != i) g[i].push_back(w);
    }
  }
  const auto lap = [&t0](double& acc) {
    const auto now = std::chrono::steady_clock::now();
    acc = std::chrono::duration<double, std::milli>(now - t0).count();
  };
  lap(F.ms_phase[0]);  // assembly
  // 1. fill-reducing order (free index space)
  std::vector<int> order;
  order.reserve(n);
  if (order_cache && static_cast<int>(order_cache->size()) == n) {
    order = *order_cache;  // the ordering depends only on the free-vertex graph: reuse it on refactorization
  } else {
    std::vector<int> all(n);
    std::iota(all.begin(), all.end(), 0);
    if (ordering == "nd-bfs") {
      std::vector<int> level(n, -1);
      std::vector<char> mark(n, 0);
      nd_bfs(g, all, order, level, mark);
    } else if (ordering == "metis") {
      metis_nd(g, order);
    } else if (ordering == "nd-mvc") {
      MvcScratch w;
      w.level.assign(n, -1);
      w.idx.assign(n, -1);
      w.mark.assign(n, 0);
      nd_mvc(g, all, order, w);
    } else {
      std::vector<P3> x(n);
      for (int i = 0; i < n; ++i) x[i] = {mesh.rest[3 * freev[i]], mesh.rest[3 * freev[i] + 1], mesh.rest[3 * freev[i] + 2]};
      std::vector<char> side(n, 0);
      nd_geometric(g, x, all, order, side);
    }
    if (order_cache) *order_cache = order;
  }
  std::vector<int> pos(n);
  for (int p = 0; p < n; ++p) pos[order[p]] = p;
  lap(F.ms_phase[1]);  // ordering
  // 2. elimination tree of the ordered matrix (Liu, with path compression)
  auto etree = [&](const std::vector<int>& ps, std::vector<int>& parent) {
    std::vector<int> anc(n, -1);
    parent.assign(n, -1);
    std::vector<std::vector<int>> lower(n);  // row k: columns j < k
    for (int i = 0; i < n; ++i)
      for (int w : g[i]) {
        const int r = ps[i], c = ps[w];
        if (c < r) lower[r].push_back(c);
      }
    for (int k = 0; k < n; ++k)
      for (int j : lower[k]) {
        int i = j;
        while (i != -1 && i < k) {
          const int nxt = anc[i];
          anc[i] = k;
          if (nxt == -1) { parent[i] = k; break; }
          i = nxt;
        }
      }
  };
  std::vector<int> parent;
  etree(pos, parent);
  // 3. postorder (children in ascending order), composed into the ordering
  {
    std::vector<int> head(n, -1), next(n, -1);
    for (int j = n - 1; j >= 0; --j)
      if (parent[j] >= 0) {
        next[j] = head[parent[j]];
        head[parent[j]] = j;
      }
    std::vector<int> post(n), stack;
    int k = 0;
    for (int r = 0; r < n; ++r) {
      if (parent[r] != -1) continue;
      stack.push_back(r);
      while (!stack.empty()) {
        const int p = stack.back();
        const int c = head[p];
        if (c == -1) {
          stack.pop_back();
          post[k++] = p;
        } else {
          head[p] = next[c];
          stack.push_back(c);
        }
      }
    }
    std::vector<int> newpos(n);  // old position -> postorder position
    for (int i = 0; i < n; ++i) newpos[post[i]] = i;
    for (int i = 0; i < n; ++i) pos[i] = newpos[pos[i]];
  }
  etree(pos, parent);
  // subtree sizes -> row ranges of S'
  std::vector<int> sz(n, 1);
  for (int j = 0; j < n; ++j)
    if (parent[j] >= 0) sz[parent[j]] += sz[j];
  for (int j = 0; j < n; ++j)
    if (j - sz[j] + 1 < 0) raise(Code::NotPositiveDefinite, "factor: elimination order is not a postorder");
  F.p2v.assign(n, -1);
  F.v2p.assign(mesh.nv, -1);
  for (int i = 0; i < n; ++i) {
    F.p2v[pos[i]] = freev[i];
    F.v2p[freev[i]] = pos[i];
  }
  lap(F.ms_phase[2]);  // etree, postorder
  // 4. permuted matrix rows (lower triangle incl. diagonal) and LDL^T (up-looking)
  std::vector<std::vector<std::pair<int, double>>> rowl(n);
  for (int i = 0; i < n; ++i) {
    const int v = freev[i], r = pos[i];
    for (int k = A.off[v]; k < A.off[v + 1]; ++k) {
      const int w = v2f[A.col[k]];
      if (w < 0) continue;
      const int c = pos[w];
      if (c <= r) rowl[r].push_back({c, A.val[k]});
    }
    std::sort(rowl[r].begin(), rowl[r].end());
  }
  std::vector<int> cnt(n, 0), flag(n, -1);
  for (int k = 0; k < n; ++k) {
    flag[k] = k;
    for (const auto& [j0, val] : rowl[k])
      for (int i = j0; i < k && flag[i] != k; i = parent[i]) {
        ++cnt[i];
        flag[i] = k;
      }
  }
  std::vector<long long> lp(n + 1, 0);
  for (int j = 0; j < n; ++j) lp[j + 1] = lp[j] + cnt[j];
  F.l_nnz = lp[n];
  std::vector<int> li(static_cast<size_t>(lp[n]));
  Vec lx(static_cast<size_t>(lp[n])), d(n), y(n, 0.0);
  std::vector<int> fill(n, 0);
  // Up-looking row k touches only its own elimination subtree (its pattern,
  // the columns it appends to and the y entries it scatters into are all
  // descendants of k), so disjoint subtrees factor concurrently; the rows
  // above them (the top separators) follow serially in elimination order.
  const auto up_rows = [&](int r0, int r1, std::vector<int>& pattern) {
    for (int k = r0; k <= r1; ++k) {
      int top = n;
      flag[k] = k;
      y[k] = 0.0;
      for (const auto& [j0, val] : rowl[k]) {
        y[j0] += val;
        int len = 0;
        for (int i = j0; flag[i] != k; i = parent[i]) {
          pattern[len++] = i;
          flag[i] = k;
        }
        while (len > 0) pattern[--top] = pattern[--len];
      }
      double dk = y[k];
      y[k] = 0.0;
      for (; top < n; ++top) {
        const int i = pattern[top];
        const double yi = y[i];
        y[i] = 0.0;
        const long long end = lp[i] + fill[i];
        for (long long p = lp[i]; p < end; ++p) y[li[p]] -= lx[p] * yi;
        const double l = yi / d[i];
        dk -= l * yi;
        li[end] = k;
        lx[end] = l;
        ++fill[i];
      }
      if (!(dk > 0.0))
        raise(Code::NotPositiveDefinite, "non-positive pivot " + std::to_string(dk) + " at position " + std::to_string(k));
      d[k] = dk;
    }
  };
  {
    // Dependency-driven schedule over the elimination tree (subtree cost
    // proxy: sum of cnt^2; the scatter work of a column is actually spent by
    // the rows above it, so the separator rows weigh more than this says):
    // a subtree cheaper than `thresh` is one unit
    // (its rows in order); every costlier node is a unit of its own, ready
    // once all its children's units are done.  Sibling separators and their
    // subtrees factor concurrently; only the chain above the first branching
    // point stays serial.  A worker that completes a node's last child
    // continues with that node directly.
    std::vector<double> cost(n);
    std::vector<int> nkids(n, 0);
    for (int j = 0; j < n; ++j) cost[j] = 1.0 + static_cast<double>(cnt[j]) * cnt[j];
    for (int j = 0; j < n; ++j)
      if (parent[j] >= 0) {
        cost[parent[j]] += cost[j];
        ++nkids[parent[j]];
      }
    double total = 0;
    for (int j = 0; j < n; ++j)
      if (parent[j] < 0) total += cost[j];
    const int T = hw_threads();
    const double thresh = total / (16.0 * T);
    std::vector<int> pending(n, 0), ready;
    int units = 0;
    for (int j = 0; j < n; ++j) {
      if (cost[j] >= thresh) {
        ++units;
        pending[j] = nkids[j];
        if (nkids[j] == 0) ready.push_back(j);
      } else if (parent[j] < 0 || cost[parent[j]] >= thresh) {
        ++units;
        ready.push_back(j);
      }
    }
    std::sort(ready.begin(), ready.end(), [&](int x, int y) { return cost[x] < cost[y]; });  // costliest popped first
    std::mutex mu;
    std::condition_variable cv;
    int done = 0;
    bool abort = false;
    std::exception_ptr err;
    const auto worker = [&] {
      std::vector<int> pattern(n);
      int j = -1;
      for (;;) {
        if (j < 0) {
          std::unique_lock<std::mutex> lk(mu);
          cv.wait(lk, [&] { return abort || done == units || !ready.empty(); });
          if (abort || ready.empty()) return;
          j = ready.back();
          ready.pop_back();
        }
        try {
          if (cost[j] < thresh) up_rows(j - sz[j] + 1, j, pattern);
          else up_rows(j, j, pattern);
        } catch (...) {
          std::lock_guard<std::mutex> lk(mu);
          if (!err) err = std::current_exception();
          abort = true;
          cv.notify_all();
          return;
        }
        const int p = parent[j];
        std::lock_guard<std::mutex> lk(mu);
        ++done;
        j = -1;
        if (p >= 0 && --pending[p] == 0) j = p;  // continue with the parent
        if (done == units) cv.notify_all();
      }
    };
    std::vector<std::thread> pool;
    for (int t = 1; t < T; ++t) pool.emplace_back(worker);
    worker();
    {
      std::lock_guard<std::mutex> lk(mu);
      cv.notify_all();
    }
    for (auto& th : pool) th.join();
    if (err) std::rethrow_exception(err);
  }
  lap(F.ms_phase[3]);  // LDL^T
  // 5. S' rows: column c of L^{-1} lives on c's ancestor path; every entry of
  //    L(:, v) for v on that path is also on it, so a dense scratch suffices.
  F.row_len = sz;
  F.row_off.assign(n + 1, 0);
  for (int r = 0; r < n; ++r) F.row_off[r + 1] = F.row_off[r] + sz[r];
  Vec dis(n);
  for (int i = 0; i < n; ++i) dis[i] = 1.0 / std::sqrt(d[i]);
  if (device_values) {  // the values are computed on the device (inverse.cu): hand over the builder inputs
    DeviceBuild& B = F.build;
    B.parent = parent;
    B.depth.assign(n, 0);
    for (int v = n - 1; v >= 0; --v) B.depth[v] = parent[v] < 0 ? 0 : B.depth[parent[v]] + 1;  // parent > v
    B.max_depth = n ? *std::max_element(B.depth.begin(), B.depth.end()) : 0;
    B.lp = lp;
    B.li = li;
    B.ldist.resize(li.size());
    for (int v = 0; v < n; ++v)
      for (long long p = lp[v]; p < lp[v + 1]; ++p) B.ldist[p] = B.depth[v] - B.depth[li[p]];
    B.lx = lx;
    B.dis = dis;
    B.row_first.resize(n);
    for (int r = 0; r < n; ++r) B.row_first[r] = r - sz[r] + 1;
  } else {
  F.sval.assign(static_cast<size_t>(F.row_off[n]), 0.0);
  parallel_chunks(n, [&](int lo, int hi, int) {
    Vec work(n, 0.0);
    for (int c = lo; c < hi; ++c) {
      work[c] = 1.0;
      for (int v = c; v >= 0; v = parent[v]) {
        const double xv = work[v];
        work[v] = 0.0;
        if (xv != 0.0)
          for (long long p = lp[v]; p < lp[v + 1]; ++p) work[li[p]] -= lx[p] * xv;
        F.sval[static_cast<size_t>(F.row_off[v] + (c - (v - sz[v] + 1)))] = xv * dis[v];
      }
    }
  });
  }
  lap(F.ms_phase[4]);  // S' values
  // 6. segments (row parts inside 256-column tiles).  The layout depends only
  //    on the elimination order and the row lengths, so a refactorization
  //    whose structure is unchanged takes it from the previous factor.
  const bool reuse = device_values && prev && prev->n == n && prev->tile_w == F.tile_w && prev->p2v == F.p2v &&
                     prev->row_len == F.row_len && !prev->row_pslot.empty() &&
                     prev->build.seg_off.size() == static_cast<size_t>(prev->row_pslot.back());
  if (reuse) {
    F.row_pslot = prev->row_pslot;
    F.seg = prev->seg;
    F.sdesc = prev->sdesc;
    F.chunks = prev->chunks;
    F.tile_chunk = prev->tile_chunk;
    F.stream_len = prev->stream_len;
    F.build.seg_off = prev->build.seg_off;
    F.build.seg_clo = prev->build.seg_clo;
  } else {
    const int W = F.tile_w;
    const int ntiles = (n + W - 1) / W;
    F.row_pslot.assign(n + 1, 0);
    std::vector<std::vector<Segment>> per_tile(ntiles);
    for (int r = 0; r < n; ++r) {
      const int first = r - sz[r] + 1;
      const int t0 = first / W, t1 = r / W;
      F.row_pslot[r + 1] = F.row_pslot[r] + (t1 - t0 + 1);
      for (int t = t0; t <= t1; ++t) {
        const int clo = std::max(first, t * W), chi = std::min(r, t * W + W - 1);
        per_tile[t].push_back({F.row_off[r] + (clo - first), r, clo, chi - clo + 1, F.row_pslot[r] + (t - t0)});
      }
    }
    for (int t = 0; t < ntiles; ++t) F.seg.insert(F.seg.end(), per_tile[t].begin(), per_tile[t].end());
    // 6b. tile-major value stream: per tile, chunks of whole segments, every
    //     chunk 16-byte aligned, descriptors contiguous per chunk
    {
      F.tile_chunk.assign(ntiles + 1, 0);
      if (!device_values) F.stream.reserve(static_cast<size_t>(F.row_off[n] * 1.02) + 16);
      else {
        F.build.seg_off.assign(F.row_pslot[n], 0);
        F.build.seg_clo.assign(F.row_pslot[n], 0);
      }
      long long slen = 0;
      for (int t = 0; t < ntiles; ++t) {
        const auto& list = per_tile[t];
        size_t s = 0;
        while (s < list.size()) {
          ChunkDesc c{slen, 0, static_cast<int>(F.sdesc.size()), 0, t};
          int vals = 0;
          while (s < list.size() && c.nseg < HDK_SEGS && vals + list[s].len <= HDK_VALS) {
            const Segment& g = list[s];
            F.sdesc.push_back({g.row, g.pslot, (g.clo - t * W) | (g.len << 16), vals});
            if (device_values) {
              F.build.seg_off[g.pslot] = slen + vals;
              F.build.seg_clo[g.pslot] = g.clo;
            } else {
              F.stream.insert(F.stream.end(), F.sval.begin() + g.off, F.sval.begin() + g.off + g.len);
            }
            vals += g.len;
            ++c.nseg;
            ++s;
          }
          if (vals & 1) {
            if (!device_values) F.stream.push_back(0.0);
            ++vals;
          }
          c.len = vals;
          slen += vals;
          F.chunks.push_back(c);
        }
        F.tile_chunk[t + 1] = static_cast<int>(F.chunks.size());
      }
      F.stream_len = slen;
    }
  }
  // 7. A_ff and A_fd in elimination order (apply_a_free / fixed coupling):
  //    row sizes first, then rows filled in parallel
  F.a_ff.rows = F.a_ff.cols = n;
  F.a_ff.off.assign(n + 1, 0);
  F.a_fd.rows = n;
  F.a_fd.cols = static_cast<int>(fixed.size());
  F.a_fd.off.assign(n + 1, 0);
  for (int p = 0; p < n; ++p) {
    const int v = F.p2v[p];
    int ff = 0, fd = 0;
    for (int k = A.off[v]; k < A.off[v + 1]; ++k) (F.v2p[A.col[k]] >= 0 ? ff : fd) += 1;
    F.a_ff.off[p + 1] = F.a_ff.off[p] + ff;
    F.a_fd.off[p + 1] = F.a_fd.off[p] + fd;
  }
  F.a_ff.col.resize(F.a_ff.off[n]);
  F.a_ff.val.resize(F.a_ff.off[n]);
  F.a_fd.col.resize(F.a_fd.off[n]);
  F.a_fd.val.resize(F.a_fd.off[n]);
  parallel_chunks(n, [&](int lo, int hi, int) {
    std::vector<std::pair<int, double>> ff;
    for (int p = lo; p < hi; ++p) {
      const int v = F.p2v[p];
      ff.clear();
      int q = F.a_fd.off[p];
      for (int k = A.off[v]; k < A.off[v + 1]; ++k) {
        const int w = A.col[k];
        if (F.v2p[w] >= 0) ff.push_back({F.v2p[w], A.val[k]});
        else {
          F.a_fd.col[q] = fixed_idx[w];
          F.a_fd.val[q++] = A.val[k];
        }
      }
      std::sort(ff.begin(), ff.end());
      for (size_t i = 0; i < ff.size(); ++i) {
        F.a_ff.col[F.a_ff.off[p] + i] = ff[i].first;
        F.a_ff.val[F.a_ff.off[p] + i] = ff[i].second;
      }
    }
  });
  F.millis = std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
  return F;
}

double factor_inverse_residual(const HostFactor& F) {
  const int n = F.n;
  double worst = 0;
  for (int axis = 0; axis < 3; ++axis) {
    Vec b(n), z(n, 0.0), x(n, 0.0);
    for (int i = 0; i < n; ++i) b[i] = std::sin(0.7 * i + axis) + 0.1 * axis;
    for (int row = 0; row < n; ++row) {
      const int first = row - F.row_len[row] + 1;
      double s = 0;
      for (int c = first; c <= row; ++c) s += F.sval[F.row_off[row] + (c - first)] * b[c];
      z[row] = s;
    }
    for (int row = 0; row < n; ++row) {
      const int first = row - F.row_len[row] + 1;
      for (int c = first; c <= row; ++c) x[c] += F.sval[F.row_off[row] + (c - first)] * z[row];
    }
    double rn = 0, bn = 0;
    for (int p = 0; p < n; ++p) {
      double s = 0;
      for (int k = F.a_ff.off[p]; k < F.a_ff.off[p + 1]; ++k) s += F.a_ff.val[k] * x[F.a_ff.col[k]];
      rn += (s - b[p]) * (s - b[p]);
      bn += b[p] * b[p];
    }
    worst = std::max(worst, std::sqrt(rn / bn));
  }
  return worst;
}

std::vector<int> balanced_ranges(const std::vector<ChunkDesc>& chunks, int G, double seg_cost) {
  const int C = static_cast<int>(chunks.size());
  std::vector<double> pre(C + 1, 0.0);
  for (int c = 0; c < C; ++c) pre[c + 1] = pre[c] + chunks[c].len + seg_cost * chunks[c].nseg;
  std::vector<int> first(G + 1, C);
  first[0] = 0;
  for (int b = 1; b < G; ++b) {
    const double target = pre[C] * b / G;
    int c = static_cast<int>(std::lower_bound(pre.begin(), pre.end(), target) - pre.begin());
    // the chunk straddling the target goes to whichever side it mostly covers
    if (c > 0 && c <= C && target - pre[c - 1] < pre[c] - target) --c;
    if (C >= G) {  // keep every range non-empty
      c = std::max(c, first[b - 1] + 1);
      c = std::min(c, C - (G - b));
    }
    first[b] = std::max(c, first[b - 1]);
  }
  first[G] = C;
  return first;
}

std::vector<int> tile_cta_ranges(const std::vector<int>& tile_chunk, const std::vector<int>& first) {
  const int T = static_cast<int>(tile_chunk.size()) - 1;
  const auto owner = [&](int c) {
    return static_cast<int>(std::upper_bound(first.begin(), first.end() - 1, c) - first.begin()) - 1;
  };
  std::vector<int> out(2 * static_cast<size_t>(T));
  for (int t = 0; t < T; ++t) {
    out[2 * t] = owner(tile_chunk[t]);
    out[2 * t + 1] = owner(tile_chunk[t + 1] - 1);
  }
  return out;
}

}  // namespace hdb
