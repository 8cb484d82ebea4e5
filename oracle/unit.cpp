// ORACLE — test infrastructure only.  Unit-level C entry points (ho_*) over
// the CPU restatement, used by tests/ to pin the oracle against the known
// answers of the reference's own unit tests (test_material.cpp,
// test_localstep.cpp, test_contact.cpp).
#include <cstring>

#include "oracle.hpp"

using namespace hdo;

namespace {
Mat3 m3(const double* a) {
  Mat3 m;
  std::memcpy(m.m, a, sizeof(m.m));
  return m;
}
template <class F>
int guard(F&& f) {
  try {
    f();
    return 0;
  } catch (const Error& e) {
    return static_cast<int>(e.code());
  } catch (...) {
    return 13;
  }
}
}  // namespace

extern "C" {
__attribute__((visibility("default"))) int ho_lame(double young, double poisson, double* mu, double* lambda) {
  return guard([&] {
    const Lame l = lame_from_young_poisson(young, poisson);
    *mu = l.mu;
    *lambda = l.lambda;
  });
}
__attribute__((visibility("default"))) int ho_nh_energy(const double* f, double mu, double lambda, double* out) {
  return guard([&] { *out = nh_energy(m3(f), mu, lambda); });
}
__attribute__((visibility("default"))) int ho_stretch_hessian_eigs(const double* s, double mu, double lambda, double* out) {
  return guard([&] {
    Vec3 val;
    Mat3 vec;
    sym_eig3(stretch_hessian(Vec3(s[0], s[1], s[2]), mu, lambda), val, vec);
    for (int i = 0; i < 3; ++i) out[i] = val[i];
  });
}
__attribute__((visibility("default"))) int ho_signed_svd(const double* f, double* u, double* s, double* v) {
  return guard([&] {
    const SvdResult r = signed_svd(m3(f));
    std::memcpy(u, r.u.m, sizeof(r.u.m));
    std::memcpy(v, r.v.m, sizeof(r.v.m));
    for (int i = 0; i < 3; ++i) s[i] = r.sigma[i];
  });
}
// kind: 0 nh_prox(mu,lambda,k) 1 volume_project 2 log_barrier_prox(mu,lambda) 3 corotated_project
__attribute__((visibility("default"))) int ho_project(int kind, const double* f, double mu, double lambda, double k,
                                                      double* p, double* sigma_star, double* sigma_f) {
  return guard([&] {
    ProxResult r;
    if (kind == 0) r = nh_prox(m3(f), mu, lambda, k);
    else if (kind == 1) r = volume_project(m3(f));
    else if (kind == 2) r = log_barrier_prox(m3(f), mu, lambda);
    else r = corotated_project(m3(f));
    std::memcpy(p, r.p_star.m, sizeof(r.p_star.m));
    for (int i = 0; i < 3; ++i) {
      sigma_star[i] = r.sigma_star[i];
      sigma_f[i] = r.sigma_f[i];
    }
  });
}
// Dense 9x9 (column-major) differential of the projection at f; for NH the
// filtered Hessian uses tau.
__attribute__((visibility("default"))) int ho_prox_differential(int kind, const double* f, double mu, double lambda,
                                                                double k, double tau, double* d9) {
  return guard([&] {
    ProxDifferential d;
    if (kind == 0) {
      const ProxResult r = nh_prox(m3(f), mu, lambda, k);
      d = nh_prox_differential(r, tr_blend(prox_hessian(r.sigma_star, mu, lambda, k), tau), k);
    } else if (kind == 1) {
      d = volume_differential(volume_project(m3(f)));
    } else if (kind == 2) {
      d = barrier_differential(log_barrier_prox(m3(f), mu, lambda), mu, lambda);
    } else {
      d = polar_differential(corotated_project(m3(f)));
    }
    d.dense(d9);
  });
}
__attribute__((visibility("default"))) int ho_tr_blend(const double* s, double mu, double lambda, double k, double tau,
                                                       double* h_filtered) {
  return guard([&] {
    const ProxHessian h = tr_blend(prox_hessian(Vec3(s[0], s[1], s[2]), mu, lambda, k), tau);
    std::memcpy(h_filtered, h.h_filtered.m, sizeof(h.h_filtered.m));
  });
}
// Single-row (frictionless) contact_iteration (contact.cpp:237-256).
__attribute__((visibility("default"))) int ho_contact_scalar(double w, double omega, double e_diag, double h_vec,
                                                             double jq_mid, double lambda, double* out) {
  return guard([&] {
    ContactSet set;
    ContactPoint c;
    c.vertex = 0;
    c.normal = Vec3(0, 0, 1);
    c.friction = 0.0;
    set.contacts = {c};
    MatX W(1, 1);
    W(0, 0) = w;
    WeightSet ws;
    ws.omega = {omega};
    ws.e_diag = {e_diag};
    *out = contact_iteration(set, W, ws, {h_vec}, {jq_mid}, {lambda})[0];
  });
}
// One frictional contact: project (lambda_n, lambda_t1, lambda_t2).
__attribute__((visibility("default"))) int ho_cone_project(double mu, const double* lam_in, double* lam_out) {
  return guard([&] {
    ContactSet set;
    ContactPoint c;
    c.vertex = 0;
    c.friction = mu;
    set.contacts = {c};
    const VecX r = project_multipliers(set, {lam_in[0], lam_in[1], lam_in[2]});
    for (int i = 0; i < 3; ++i) lam_out[i] = r[i];
  });
}
__attribute__((visibility("default"))) int ho_prox_means(const char* scene_json, double* out) {
  return guard([&] {
    const SceneSpec s = parse_scene_json(scene_json);
    const ProxMeans& m = s.material.prox_means();
    out[0] = m.mu;
    out[1] = m.lambda;
    out[2] = m.stiffness;
  });
}
}
