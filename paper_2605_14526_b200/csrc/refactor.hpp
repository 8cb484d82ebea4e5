// Device refactorization (reference factor.cpp:11-136
// SparseFactor::factorize + assemble_global_scalar): when only the values of
// the global operator change (a system-ID parameter update keeps the mesh,
// the fixed set and the step), the whole numeric part runs on the GPU:
//   1. A's values for the fixed pattern, each entry summed from its element
//      contributions in the host assembly's order (factor.cpp assemble),
//   2. LDL^T by a multifrontal method over the supernodal elimination tree:
//      one CTA per front, fronts of one tree level per launch, dense blocked
//      partial factorization of each front, children's Schur complements
//      extended-added into the parent, L and D written in the host factor's
//      column layout,
//   3. D^{-1/2} and the S' values (inverse.cu, unchanged).
// The symbolic part (supernodes, front row lists, extend-add and assembly
// maps) is built once on the host from the first factorization.  mf_factor_host
// is the same numeric algorithm on the CPU (explicit rounding order shared
// with the kernels), used by the tests as the bitwise reference of the
// device fronts.
#pragma once

#include <vector>

#include "host.hpp"

namespace hdb {

struct MfPlan {
  int n = 0, nsuper = 0, nlevels = 0;
  std::vector<int> sfirst;       // nsuper + 1: supernode s = columns [sfirst[s], sfirst[s + 1])
  std::vector<int> fm;           // front order (pivots + update rows)
  std::vector<long long> foff;   // front offset in the pool (m x m, column-major)
  long long pool = 0;            // doubles
  std::vector<int> frow_off, frow;      // front rows (elimination positions, ascending)
  std::vector<int> level_off, level_node;
  std::vector<int> child_off, child;    // children (ascending)
  std::vector<int> emap_off, emap;      // per supernode: its update rows' positions in the parent's front
  std::vector<int> aent_off, aent_src, aent_dst;  // per supernode: a_ff value index -> front offset
  std::vector<long long> lp;     // L by columns (the host factor's layout)
  int max_front = 0;
};

// Symbolic multifrontal plan of a built factor (needs F.build.parent/lp/li and F.a_ff).
MfPlan mf_plan(const HostFactor& F);
// CPU reference of the device numeric factorization: L values (host layout) and D.
void mf_factor_host(const MfPlan& P, const Vec& a_ff_val, Vec& lx, Vec& d);

// Element contributions of every A_ff / A_fd entry, in the host assembly's
// summation order (factor.cpp assemble): entry k sums corner pairs
// cpair[coff[k] .. coff[k + 1]) = (4 e + i) << 2 | j, plus inertia * m_v on
// the diagonal first.
struct AssemblyPlan {
  std::vector<int> ff_off, fd_off;  // per a_ff / a_fd value
  std::vector<int> ff_pair, fd_pair;
  std::vector<int> ff_diag;         // vertex of a diagonal a_ff entry, else -1
  std::vector<int> df_from_fd;      // a_df value j = a_fd value df_from_fd[j]
};
AssemblyPlan assembly_plan(const Mesh& mesh, const HostFactor& F);

}  // namespace hdb
