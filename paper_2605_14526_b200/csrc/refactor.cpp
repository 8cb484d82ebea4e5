// Symbolic multifrontal plan and assembly plan of the device refactorization
// (refactor.hpp), and the CPU reference of the numeric kernels (refactor.cu).
#include "refactor.hpp"

#include <cuda_runtime.h>

#include "../../include/hdk.h"

#include <algorithm>
#include <string>

namespace hdb {

MfPlan mf_plan(const HostFactor& F) {
  const DeviceBuild& B = F.build;
  const int n = F.n;
  if (B.parent.size() != static_cast<size_t>(n) || B.li.size() != B.lx.size())
    raise(Code::InvalidArgument, "mf_plan: the factor was built without its device-build data");
  MfPlan P;
  P.n = n;
  P.lp = B.lp;
  const auto cnt = [&](int j) { return static_cast<int>(B.lp[j + 1] - B.lp[j]); };
  std::vector<int> nkids(n, 0);
  for (int j = 0; j < n; ++j)
    if (B.parent[j] >= 0) ++nkids[B.parent[j]];
  // fundamental supernodes: j joins j-1's when j is j-1's parent, its only
  // child, and column j-1's structure is {j} + column j's
  P.sfirst.push_back(0);
  for (int j = 1; j < n; ++j)
    if (!(B.parent[j - 1] == j && nkids[j] == 1 && cnt(j - 1) == cnt(j) + 1)) P.sfirst.push_back(j);
  P.sfirst.push_back(n);
  P.nsuper = static_cast<int>(P.sfirst.size()) - 1;
  std::vector<int> super_of(n);
  for (int s = 0; s < P.nsuper; ++s)
    for (int j = P.sfirst[s]; j < P.sfirst[s + 1]; ++j) super_of[j] = s;
  // front rows = own columns + the last column's structure
  P.frow_off.assign(P.nsuper + 1, 0);
  P.fm.resize(P.nsuper);
  P.foff.resize(P.nsuper);
  std::vector<int> sparent(P.nsuper, -1);
  for (int s = 0; s < P.nsuper; ++s) {
    const int f = P.sfirst[s], l = P.sfirst[s + 1] - 1;
    for (int j = f; j <= l; ++j) P.frow.push_back(j);
    for (long long q = B.lp[l]; q < B.lp[l + 1]; ++q) P.frow.push_back(B.li[q]);
    P.frow_off[s + 1] = static_cast<int>(P.frow.size());
    P.fm[s] = P.frow_off[s + 1] - P.frow_off[s];
    P.max_front = std::max(P.max_front, P.fm[s]);
    for (int j = f; j <= l; ++j)  // the column structures nest (fundamental supernode)
      if (cnt(j) != P.fm[s] - 1 - (j - f)) raise(Code::InvalidArgument, "mf_plan: supernode structure mismatch");
    if (B.parent[l] >= 0) sparent[s] = super_of[B.parent[l]];
  }
  long long off = 0;
  for (int s = 0; s < P.nsuper; ++s) {
    P.foff[s] = off;
    off += static_cast<long long>(P.fm[s]) * P.fm[s];
  }
  P.pool = off;
  // children (ascending) and levels (leaves first)
  std::vector<std::vector<int>> kids(P.nsuper);
  for (int s = 0; s < P.nsuper; ++s)
    if (sparent[s] >= 0) kids[sparent[s]].push_back(s);
  P.child_off.assign(P.nsuper + 1, 0);
  std::vector<int> level(P.nsuper, 0);
  for (int s = 0; s < P.nsuper; ++s) {  // children precede parents (postorder)
    for (int c : kids[s]) level[s] = std::max(level[s], level[c] + 1);
    P.child.insert(P.child.end(), kids[s].begin(), kids[s].end());
    P.child_off[s + 1] = static_cast<int>(P.child.size());
  }
  P.nlevels = P.nsuper ? 1 + *std::max_element(level.begin(), level.end()) : 0;
  P.level_off.assign(P.nlevels + 1, 0);
  for (int s = 0; s < P.nsuper; ++s) ++P.level_off[level[s] + 1];
  for (int L = 0; L < P.nlevels; ++L) P.level_off[L + 1] += P.level_off[L];
  P.level_node.resize(P.nsuper);
  {
    std::vector<int> cur(P.level_off.begin(), P.level_off.end() - 1);
    for (int s = 0; s < P.nsuper; ++s) P.level_node[cur[level[s]]++] = s;
  }
  // extend-add maps: each update row's position in the parent's front
  P.emap_off.assign(P.nsuper + 1, 0);
  for (int s = 0; s < P.nsuper; ++s) {
    const int p = sparent[s];
    const int piv = P.sfirst[s + 1] - P.sfirst[s];
    if (p >= 0) {
      const int* pr = P.frow.data() + P.frow_off[p];
      const int pm = P.fm[p];
      for (int k = P.frow_off[s] + piv; k < P.frow_off[s + 1]; ++k) {
        const int* it = std::lower_bound(pr, pr + pm, P.frow[k]);
        if (it == pr + pm || *it != P.frow[k]) raise(Code::InvalidArgument, "mf_plan: update row outside the parent front");
        P.emap.push_back(static_cast<int>(it - pr));
      }
    } else if (P.fm[s] != piv) {
      raise(Code::InvalidArgument, "mf_plan: a root front with update rows");
    }
    P.emap_off[s + 1] = static_cast<int>(P.emap.size());
  }
  // A entries (lower triangle, column j) -> front offsets of j's supernode
  std::vector<std::vector<std::pair<int, int>>> ae(P.nsuper);
  const Csr& A = F.a_ff;
  for (int i = 0; i < n; ++i)
    for (int k = A.off[i]; k < A.off[i + 1]; ++k) {
      const int j = A.col[k];
      if (j > i) continue;
      const int s = super_of[j];
      const int* fr = P.frow.data() + P.frow_off[s];
      const int* it = std::lower_bound(fr, fr + P.fm[s], i);
      if (it == fr + P.fm[s] || *it != i) raise(Code::InvalidArgument, "mf_plan: A entry outside the front");
      ae[s].push_back({k, static_cast<int>(it - fr) + (j - P.sfirst[s]) * P.fm[s]});
    }
  P.aent_off.assign(P.nsuper + 1, 0);
  for (int s = 0; s < P.nsuper; ++s) {
    for (const auto& [src, dst] : ae[s]) {
      P.aent_src.push_back(src);
      P.aent_dst.push_back(dst);
    }
    P.aent_off[s + 1] = static_cast<int>(P.aent_src.size());
  }
  return P;
}

// The panel width and the operation order are shared with refactor.cu
// (k_mf_level): every product and sum is one IEEE-rounded operation there
// (__dmul_rn / __dadd_rn / __dsub_rn / __ddiv_rn), so CPU and GPU fronts agree
// bit for bit.
static constexpr int kPanel = HDK_MF_PANEL;

void mf_factor_host(const MfPlan& P, const Vec& aval, Vec& lx, Vec& d) {
  Vec pool(static_cast<size_t>(P.pool), 0.0);
  lx.assign(static_cast<size_t>(P.lp[P.n]), 0.0);
  d.assign(P.n, 0.0);
  for (int L = 0; L < P.nlevels; ++L)
    for (int q = P.level_off[L]; q < P.level_off[L + 1]; ++q) {
      const int s = P.level_node[q];
      const int m = P.fm[s], f = P.sfirst[s], piv = P.sfirst[s + 1] - f;
      double* Fm = pool.data() + P.foff[s];
      std::fill(Fm, Fm + static_cast<size_t>(m) * m, 0.0);
      for (int k = P.aent_off[s]; k < P.aent_off[s + 1]; ++k) Fm[P.aent_dst[k]] = aval[P.aent_src[k]];
      for (int ci = P.child_off[s]; ci < P.child_off[s + 1]; ++ci) {
        const int c = P.child[ci];
        const int mc = P.fm[c], pc = P.sfirst[c + 1] - P.sfirst[c], r = mc - pc;
        const double* U = pool.data() + P.foff[c];
        const int* map = P.emap.data() + P.emap_off[c];
        for (int j = 0; j < r; ++j)
          for (int i = j; i < r; ++i)
            Fm[map[i] + static_cast<size_t>(map[j]) * m] += U[(pc + i) + static_cast<size_t>(pc + j) * mc];
      }
      for (int c0 = 0; c0 < piv; c0 += kPanel) {
        const int cb = std::min(kPanel, piv - c0);
        for (int c = c0; c < c0 + cb; ++c) {
          const double dc = Fm[c + static_cast<size_t>(c) * m];
          if (!(dc > 0.0))
            raise(Code::NotPositiveDefinite, "non-positive pivot " + std::to_string(dc) + " at position " +
                                                 std::to_string(f + c));
          for (int i = c + 1; i < m; ++i) Fm[i + static_cast<size_t>(c) * m] = Fm[i + static_cast<size_t>(c) * m] / dc;
          for (int j = c + 1; j < c0 + cb; ++j) {  // the rest of the panel: A_ij -= L_ic (L_jc d_c)
            const double w = Fm[j + static_cast<size_t>(c) * m] * dc;
            for (int i = j; i < m; ++i)
              Fm[i + static_cast<size_t>(j) * m] = Fm[i + static_cast<size_t>(j) * m] - Fm[i + static_cast<size_t>(c) * m] * w;
          }
        }
        for (int j = c0 + cb; j < m; ++j) {  // trailing update by the whole panel
          double w[kPanel];
          for (int c = c0; c < c0 + cb; ++c) w[c - c0] = Fm[j + static_cast<size_t>(c) * m] * Fm[c + static_cast<size_t>(c) * m];
          for (int i = j; i < m; ++i) {
            double acc = 0.0;
            for (int c = c0; c < c0 + cb; ++c) acc = acc + Fm[i + static_cast<size_t>(c) * m] * w[c - c0];
            Fm[i + static_cast<size_t>(j) * m] = Fm[i + static_cast<size_t>(j) * m] - acc;
          }
        }
      }
      for (int c = 0; c < piv; ++c) {
        d[f + c] = Fm[c + static_cast<size_t>(c) * m];
        const long long base = P.lp[f + c];
        for (int i = c + 1; i < m; ++i) lx[base + (i - c - 1)] = Fm[i + static_cast<size_t>(c) * m];
      }
    }
}

AssemblyPlan assembly_plan(const Mesh& mesh, const HostFactor& F) {
  AssemblyPlan P;
  const int nv = mesh.nv, ne = mesh.ne;
  std::vector<int> inc_off(nv + 1, 0), inc(4 * static_cast<size_t>(ne));
  for (int e = 0; e < ne; ++e)
    for (int i = 0; i < 4; ++i) ++inc_off[mesh.el[e][i] + 1];
  for (int v = 0; v < nv; ++v) inc_off[v + 1] += inc_off[v];
  {
    std::vector<int> cur(inc_off.begin(), inc_off.end() - 1);
    for (int e = 0; e < ne; ++e)
      for (int i = 0; i < 4; ++i) inc[cur[mesh.el[e][i]]++] = 4 * e + i;  // ascending e (factor.cpp assemble)
  }
  // contributions of (v, w): the incident elements of v in order, the corner of w in each
  const auto pairs = [&](int v, int w, std::vector<int>& out) {
    for (int k = inc_off[v]; k < inc_off[v + 1]; ++k) {
      const int e = inc[k] >> 2, i = inc[k] & 3;
      for (int j = 0; j < 4; ++j)
        if (mesh.el[e][j] == w) out.push_back(((4 * e + i) << 2) | j);
    }
  };
  std::vector<int> fixed_of(F.fixed.size());
  for (size_t k = 0; k < F.fixed.size(); ++k) fixed_of[k] = F.fixed[k];
  P.ff_off.assign(1, 0);
  P.fd_off.assign(1, 0);
  for (int p = 0; p < F.n; ++p) {
    const int v = F.p2v[p];
    for (int k = F.a_ff.off[p]; k < F.a_ff.off[p + 1]; ++k) {
      const int w = F.p2v[F.a_ff.col[k]];
      pairs(v, w, P.ff_pair);
      P.ff_off.push_back(static_cast<int>(P.ff_pair.size()));
      P.ff_diag.push_back(v == w ? v : -1);
    }
    for (int k = F.a_fd.off[p]; k < F.a_fd.off[p + 1]; ++k) {
      pairs(v, fixed_of[F.a_fd.col[k]], P.fd_pair);
      P.fd_off.push_back(static_cast<int>(P.fd_pair.size()));
    }
  }
  // A_df = A_fd^T in the engine's transpose order (engine.cpp build_factor_device)
  const Csr& fd = F.a_fd;
  std::vector<int> cur(fd.cols + 1, 0);
  for (int c : fd.col) ++cur[c + 1];
  for (int r = 0; r < fd.cols; ++r) cur[r + 1] += cur[r];
  P.df_from_fd.assign(fd.col.size(), 0);
  for (int p = 0; p < fd.rows; ++p)
    for (int k = fd.off[p]; k < fd.off[p + 1]; ++k) P.df_from_fd[cur[fd.col[k]]++] = k;
  return P;
}

}  // namespace hdb
