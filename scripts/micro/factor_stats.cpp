// Prints the chunk / segment shape of the C3 factor stream (host only).
#include <algorithm>
#include <cstdio>
#include <fstream>
#include <sstream>
#include <vector>
#include "../../paper_2605_14526_b200/csrc/host.hpp"
int main(int argc, char** argv) {
  std::ifstream in(argv[1]); std::stringstream ss; ss << in.rdbuf();
  hdb::Scene s = hdb::parse_scene(ss.str());
  hdb::HostFactor F = hdb::build_factor(s.mesh, s.material, s.solver.h, s.fixed, s.ordering);
  std::vector<int> hist_nseg(9, 0), hist_len(10, 0);
  long long segs_in_heavy = 0, vals_in_heavy = 0, m_iters = 0, m_needed = 0;
  for (const auto& c : F.chunks) {
    int b = 0; while ((1 << (b + 1)) <= c.nseg && b < 8) ++b;
    hist_nseg[b]++;
    if (c.nseg >= 64) { segs_in_heavy += c.nseg; vals_in_heavy += c.len; }
    for (int i = 0; i < c.nseg; ++i) {
      const auto& sg = F.sdesc[c.seg0 + i];
      const int lo = sg.clo_len & 0xffff, len = sg.clo_len >> 16;
      int lb = 0; while ((1 << (lb + 1)) <= len && lb < 9) ++lb;
      hist_len[lb]++;
      m_iters += 8;
      m_needed += (lo + len - 1) / 32 - lo / 32 + 1;
    }
  }
  printf("chunks %zu segs %zu\n", F.chunks.size(), F.sdesc.size());
  for (int b = 0; b < 9; ++b) printf("nseg in [%d,%d): %d chunks\n", 1 << b, 1 << (b + 1), hist_nseg[b]);
  for (int b = 0; b < 10; ++b) printf("len in [%d,%d): %d segs\n", 1 << b, 1 << (b + 1), hist_len[b]);
  printf("heavy chunks (>=64 segs): %lld segs, %lld vals\n", segs_in_heavy, vals_in_heavy);
  printf("lane-column iterations: issued %lld, needed %lld (%.1f%%)\n", m_iters, m_needed, 100.0 * m_needed / m_iters);
}
