// Per-element Anderson step of the adjoint backbone (backward.cpp:170-204)
// used by the dots kernel (vec.cu k_bb_dots): given t_i (folded from the
// solve's tile partials), write t by elimination order and by vertex, push
// the history entry (s = dq + dg and dg) and accumulate the 18 dot products
// DG^T dg_new, DG^T g, |g|^2, |t|^2.  (Running it per finished tile inside the
// column pass, instead of as a kernel, stalled the pass: 25 -> 59 us.)
#pragma once

#include <cuda_runtime.h>

#include "../../include/hdk.h"
#include "launch.cuh"

namespace hdk {

struct BbArgs {
  hdk_ctl* ctl;
  double* tp;        // t, elimination order [n][3]
  double* tv;        // t by vertex (input of B t)
  const double* xp;  // x, elimination order
  double *last_q, *last_g, *dq, *dg;
};

struct BbState {
  int m, c, ns, c2, push;
  int ph[HDK_AA_MAX];
};

__device__ __forceinline__ BbState bb_state(const hdk_ctl* ctl) {
  BbState s;
  s.m = ctl->window;
  s.c = ctl->count;
  const int h = ctl->head;
  s.push = ctl->has_last != 0;
  s.ns = 0;
  s.c2 = s.c;
  int h2 = h;
  if (s.push) {
    s.ns = s.c < s.m ? (h + s.c) % s.m : h;
    s.c2 = s.c < s.m ? s.c + 1 : s.m;
    h2 = s.c < s.m ? h : (h + 1) % s.m;
  }
#pragma unroll
  for (int j = 0; j < HDK_AA_MAX; ++j) s.ph[j] = (h2 + j) % s.m;
  return s;
}

// Loads of one element that do not depend on t (issued before t is folded).
struct BbIn {
  double qc, lq, lg;
  double dgh[HDK_AA_MAX];
};

__device__ __forceinline__ BbIn bb_prefetch(const BbArgs& a, const BbState& s, size_t n3, size_t i,
                                            unsigned long long pol) {
  BbIn v;
  v.qc = ld_keep(a.xp + i, pol);
  v.lq = s.push ? ld_keep(a.last_q + i, pol) : 0.0;
  v.lg = s.push ? ld_keep(a.last_g + i, pol) : 0.0;
#pragma unroll
  for (int j = 0; j < HDK_AA_MAX; ++j)
    v.dgh[j] = (s.push && j < s.c2 && s.ph[j] != s.ns) ? ld_keep(a.dg + s.ph[j] * n3 + i, pol) : 0.0;
  return v;
}

__device__ __forceinline__ void bb_dots_elem(const BbArgs& a, const BbState& s, const BbIn& v,
                                             const int* __restrict__ p2v, size_t n3, size_t i, double th,
                                             double (&acc)[2 * HDK_AA_MAX + 2], unsigned long long pol) {
  const int col = static_cast<int>(i / 3), ax = static_cast<int>(i - 3 * (size_t)col);
  st_keep(a.tp + i, th, pol);
  a.tv[3 * (size_t)__ldg(p2v + col) + ax] = th;
  const double qc = v.qc;
  const double g = th - qc;
  acc[2 * HDK_AA_MAX] += g * g;
  acc[2 * HDK_AA_MAX + 1] += th * th;
  if (s.push) {
    const double dqn = qc - v.lq;
    const double dgn = g - v.lg;
    st_keep(a.dq + s.ns * n3 + i, dqn + dgn, pol);  // the mix only ever uses dq_j + dg_j
    st_keep(a.dg + s.ns * n3 + i, dgn, pol);
#pragma unroll
    for (int j = 0; j < HDK_AA_MAX; ++j) {
      if (j < s.c2) {
        const double dgj = s.ph[j] == s.ns ? dgn : v.dgh[j];
        acc[j] += dgn * dgj;
        acc[HDK_AA_MAX + j] += dgj * g;
      }
    }
  }
  st_keep(a.last_q + i, qc, pol);
  st_keep(a.last_g + i, g, pol);
}

// One level of a reduce-scatter butterfly over N per-lane values (fixed
// order, bitwise reproducible): lanes with bit O set keep the upper half.
template <int N, int O>
__device__ __forceinline__ void rs_level(const double (&v)[N], double (&w)[(N + 1) / 2], int lane, int& q0,
                                         int& len) {
  constexpr int H = (N + 1) / 2;
  const bool up = (lane & O) != 0;
#pragma unroll
  for (int i = 0; i < H; ++i) {
    const double lo = v[i];
    const double hi = (i + H < N) ? v[i + H] : 0.0;
    const double r = __shfl_xor_sync(0xffffffffu, up ? lo : hi, O);
    w[i] = (up ? hi : lo) + r;
  }
  if (up) {
    q0 += H;
    len -= H;
  } else if (len > H) {
    len = H;
  }
}

// Warp sums of the 18 quantities: lane l holds quantity q0 (valid if len >= 1).
__device__ __forceinline__ double warp_rs_18(const double (&v)[18], int lane, int& q0, int& len) {
  q0 = 0;
  len = 18;
  double a9[9], a5[5], a3[3], a2[2], a1[1];
  rs_level<18, 16>(v, a9, lane, q0, len);
  rs_level<9, 8>(a9, a5, lane, q0, len);
  rs_level<5, 4>(a5, a3, lane, q0, len);
  rs_level<3, 2>(a3, a2, lane, q0, len);
  rs_level<2, 1>(a2, a1, lane, q0, len);
  return a1[0];
}

}  // namespace hdk
