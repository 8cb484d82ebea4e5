// hd_* C ABI of include/heterodyn.h over the B200 engine.  Reference half:
// capi.cpp:94-322 (opaque handles, status codes, thread-local errors,
// exceptions never cross the boundary); B200 extensions: recorded frames,
// backward chain, state control and counters.
#include <cstdlib>
#include <chrono>
#include <cmath>
#include <cstring>
#include <cstdio>
#include <memory>

#include <nlohmann/json.hpp>

#include "../../include/heterodyn.h"
#include "batch.hpp"
#include "engine.hpp"
#include "drivers.hpp"
#include "refactor.hpp"

using namespace hdb;

struct hd_scene {
  Scene spec;
};

struct hd_sim {
  const hd_scene* scene = nullptr;
  std::unique_ptr<Engine> eng;
  GradOut last_grad;
};

struct hd_batch {
  const hd_scene* scene = nullptr;
  std::unique_ptr<Batch> b;
};

namespace {
thread_local int t_code = 0;
thread_local std::string t_msg;

void set_error(int c, const std::string& m) {
  t_code = c;
  t_msg = m;
}

template <class F>
hd_status guarded(F&& f) {
  try {
    f();
    return HD_OK;
  } catch (const Error& e) {
    set_error(static_cast<int>(e.code), e.what());
    return static_cast<hd_status>(e.code);
  } catch (const std::exception& e) {
    set_error(HD_ERR_INVALID_ARGUMENT, std::string("unexpected error: ") + e.what());
    return HD_ERR_INVALID_ARGUMENT;
  }
}

hd_status bad_arg(const std::string& m) {
  set_error(HD_ERR_INVALID_ARGUMENT, m);
  return HD_ERR_INVALID_ARGUMENT;
}

char* dup(const std::string& s) {
  char* p = static_cast<char*>(std::malloc(s.size() + 1));
  if (p) std::memcpy(p, s.c_str(), s.size() + 1);
  return p;
}


template <class Make>
hd_scene* make_scene(const char* who, const void* arg, Make&& make) {
  if (!arg) {
    bad_arg(std::string(who) + ": NULL argument");
    return nullptr;
  }
  auto s = std::make_unique<hd_scene>();
  if (guarded([&] { s->spec = make(); }) != HD_OK) return nullptr;
  return s.release();
}

// stdio, not iostreams: the library links its own libstdc++, whose stream
// locale state is not set up when it is dlopen'ed next to another one.
std::string read_file(const char* path) {
  FILE* f = std::fopen(path, "rb");
  if (!f) raise(Code::Io, std::string("cannot open scene file: ") + path);
  std::string text;
  char buf[65536];
  for (size_t n; (n = std::fread(buf, 1, sizeof buf, f)) > 0;) text.append(buf, n);
  std::fclose(f);
  return text;
}
}  // namespace

extern "C" {

const char* hd_last_error(void) { return t_msg.c_str(); }
int hd_last_error_code(void) { return t_code; }
void hd_string_free(char* s) { std::free(s); }

hd_scene* hd_scene_load(const char* path) {
  return make_scene("hd_scene_load", path, [&] { return parse_scene(read_file(path)); });
}
hd_scene* hd_scene_parse(const char* text) {
  return make_scene("hd_scene_parse", text, [&] { return parse_scene(text); });
}
hd_scene* hd_scene_builtin(const char* name) {
  return make_scene("hd_scene_builtin", name, [&] { return builtin_scene(name); });
}
void hd_scene_free(hd_scene* s) { delete s; }
int hd_scene_vertex_count(const hd_scene* s) { return s ? s->spec.mesh.nv : 0; }
int hd_scene_element_count(const hd_scene* s) { return s ? s->spec.mesh.ne : 0; }
int hd_scene_frame_count(const hd_scene* s) { return s ? s->spec.frames : 0; }
const char* hd_scene_name(const hd_scene* s) { return s ? s->spec.name.c_str() : ""; }

int hd_scene_region_count(const hd_scene* s) { return s ? s->spec.region_count : 0; }
hd_status hd_scene_regions(const hd_scene* s, int* out, size_t cap) {
  if (!s) return bad_arg("hd_scene_regions: scene is NULL");
  const size_t ne = static_cast<size_t>(s->spec.mesh.ne);
  if (!out || cap < ne) return bad_arg("hd_scene_regions: output buffer too small");
  for (size_t e = 0; e < ne; ++e) out[e] = e < s->spec.region.size() ? s->spec.region[e] : 0;
  return HD_OK;
}
hd_status hd_scene_rest_positions(const hd_scene* s, double* out, size_t cap) {
  if (!s) return bad_arg("hd_scene_rest_positions: scene is NULL");
  const Vec& r = s->spec.mesh.rest;
  if (!out || cap < r.size()) return bad_arg("hd_scene_rest_positions: output buffer too small");
  std::copy(r.begin(), r.end(), out);
  return HD_OK;
}
hd_status hd_scene_vertex_masses(const hd_scene* s, double* out, size_t cap) {
  if (!s) return bad_arg("hd_scene_vertex_masses: scene is NULL");
  const Vec& m = s->spec.mesh.mass;
  if (!out || cap < m.size()) return bad_arg("hd_scene_vertex_masses: output buffer too small");
  std::copy(m.begin(), m.end(), out);
  return HD_OK;
}

hd_status hd_scene_elements(const hd_scene* s, int* out, size_t cap) {
  if (!s) return bad_arg("hd_scene_elements: scene is NULL");
  const auto& el = s->spec.mesh.el;
  if (!out || cap < 4 * el.size()) return bad_arg("hd_scene_elements: output buffer too small");
  for (size_t e = 0; e < el.size(); ++e)
    for (int k = 0; k < 4; ++k) out[4 * e + k] = el[e][k];
  return HD_OK;
}
hd_status hd_scene_young_moduli(const hd_scene* s, double* out, size_t cap) {
  if (!s) return bad_arg("hd_scene_young_moduli: scene is NULL");
  const Vec& y = s->spec.material.young;
  if (!out || cap < y.size()) return bad_arg("hd_scene_young_moduli: output buffer too small");
  std::copy(y.begin(), y.end(), out);
  return HD_OK;
}

hd_sim* hd_sim_create(const hd_scene* scene) {
  if (!scene) {
    bad_arg("hd_sim_create: scene is NULL");
    return nullptr;
  }
  auto sim = std::make_unique<hd_sim>();
  sim->scene = scene;
  if (guarded([&] { sim->eng = std::make_unique<Engine>(scene->spec); }) != HD_OK) return nullptr;
  return sim.release();
}
void hd_sim_free(hd_sim* sim) { delete sim; }

hd_status hd_sim_step(hd_sim* sim) {
  if (!sim) return bad_arg("hd_sim_step: sim is NULL");
  return guarded([&] { sim->eng->step(); });
}
double hd_sim_time(const hd_sim* sim) { return sim ? sim->eng->time() : 0.0; }
int hd_sim_dof_count(const hd_sim* sim) { return sim ? sim->eng->dofs() : 0; }
// capacity check first (capi.cpp:63-72 of the reference), then one copy
// straight into the caller's buffer
hd_status hd_sim_positions(const hd_sim* sim, double* out, size_t cap) {
  if (!sim) return bad_arg("hd_sim_positions: sim is NULL");
  if (!out || cap < sim->eng->dof_count()) return bad_arg("hd_sim_positions: output buffer too small");
  return guarded([&] { sim->eng->positions_into(out); });
}
hd_status hd_sim_velocities(const hd_sim* sim, double* out, size_t cap) {
  if (!sim) return bad_arg("hd_sim_velocities: sim is NULL");
  if (!out || cap < sim->eng->dof_count()) return bad_arg("hd_sim_velocities: output buffer too small");
  return guarded([&] { sim->eng->velocities_into(out); });
}
int hd_sim_last_iterations(const hd_sim* sim) { return sim ? sim->eng->last_iterations : 0; }
int hd_sim_last_converged(const hd_sim* sim) { return sim && sim->eng->last_converged ? 1 : 0; }
int hd_sim_last_contact_count(const hd_sim* sim) { return sim ? sim->eng->last_contacts : 0; }
hd_status hd_sim_contact_trace(const hd_sim* sim, int* vertex, int* obstacle, size_t row_capacity,
                               double* clamp, size_t clamp_capacity, double* cone, size_t cone_capacity,
                               int* counts) {
  if (!sim) return bad_arg("hd_sim_contact_trace: sim is NULL");
  return guarded([&] {
    std::vector<int> v, o;
    std::vector<double> cl, co;
    int nc = 0, nf = 0, iters = 0;
    sim->eng->contact_trace(v, o, cl, co, nc, nf, iters);
    if (counts) {
      counts[0] = nc;
      counts[1] = nf;
      counts[2] = iters;
    }
    if ((vertex || obstacle) && row_capacity < v.size())
      hdb::raise(hdb::Code::InvalidArgument, "hd_sim_contact_trace: row capacity too small");
    if ((clamp && clamp_capacity < cl.size()) || (cone && cone_capacity < co.size()))
      hdb::raise(hdb::Code::InvalidArgument, "hd_sim_contact_trace: pattern capacity too small");
    if (vertex) std::copy(v.begin(), v.end(), vertex);
    if (obstacle) std::copy(o.begin(), o.end(), obstacle);
    if (clamp) std::copy(cl.begin(), cl.end(), clamp);
    if (cone) std::copy(co.begin(), co.end(), cone);
  });
}
double hd_sim_last_fb_residual(const hd_sim* sim) {
  double r = 0.0;
  if (sim) guarded([&] { r = sim->eng->last_fb_residual(); });
  return r;
}
double hd_sim_penetration(const hd_sim* sim) {
  double r = 0.0;
  if (sim) guarded([&] { r = sim->eng->penetration(); });
  return r;
}

// The simulate driver (drivers.cpp; reference drivers.cpp:238-365): summary
// JSON, and trajectory.jsonl / metrics.csv / summary.json under out_dir.
hd_status hd_run_simulate(const hd_scene* scene, const char* out_dir, char** summary_json) {
  if (!scene) return bad_arg("hd_run_simulate: scene is NULL");
  std::string out, err;
  const int code = heterodyn_driver::run_simulate(scene, out_dir, &out, &err);
  if (code != HD_OK) {
    set_error(code, err);
    return static_cast<hd_status>(code);
  }
  if (summary_json) *summary_json = dup(out);
  return HD_OK;
}

hd_status hd_run_gradcheck(const hd_scene* scene, const char* vars_csv, const char* out_path, char** report_json,
                           int* pass) {
  if (!scene) return bad_arg("hd_run_gradcheck: scene is NULL");
  std::string out, err;
  bool ok = false;
  const int code = heterodyn_driver::run_gradcheck(scene, vars_csv, out_path, &out, &ok, &err);
  if (code != HD_OK) {
    set_error(code, err);
    return static_cast<hd_status>(code);
  }
  if (report_json) *report_json = dup(out);
  if (pass) *pass = ok ? 1 : 0;
  return HD_OK;
}
// System identification: the L-BFGS driver over this library's own ABI
// (drivers.cpp; reference capi.cpp:279-308).
static hd_status identify_finish(int code, const std::string& out, bool st, const std::string& err, char** result_json,
                          int* stalled) {
  if (code != HD_OK) {
    set_error(code, err);
    return static_cast<hd_status>(code);
  }
  if (result_json) *result_json = dup(out);
  if (stalled) *stalled = st ? 1 : 0;
  return HD_OK;
}
hd_status hd_run_identify(const char* problem_json, const char* out_dir, char** result_json, int* stalled) {
  if (!problem_json) return bad_arg("hd_run_identify: problem is NULL");
  std::string out, err;
  bool st = false;
  const int code = heterodyn_driver::run_identify(problem_json, out_dir ? out_dir : "", &out, &st, &err);
  return identify_finish(code, out, st, err, result_json, stalled);
}
hd_status hd_run_identify_file(const char* problem_path, const char* out_dir, char** result_json, int* stalled) {
  if (!problem_path) return bad_arg("hd_run_identify_file: path is NULL");
  std::string out, err;
  bool st = false;
  const int code = heterodyn_driver::run_identify_file(problem_path, out_dir ? out_dir : "", &out, &st, &err);
  return identify_finish(code, out, st, err, result_json, stalled);
}

// Host-only: builds the factor without touching the GPU (drivers.cpp:990-1006).
hd_status hd_factor_stats(const hd_scene* scene, char** stats_json) {
  if (!scene) return bad_arg("hd_factor_stats: scene is NULL");
  return guarded([&] {
    const Scene& s = scene->spec;
    const HostFactor F = build_factor(s.mesh, s.material, s.solver.h, s.fixed, s.ordering);
    nlohmann::json j;
    j["vertices"] = s.mesh.nv;
    j["elements"] = s.mesh.ne;
    j["dofs"] = 3 * s.mesh.nv;
    j["free_vertices"] = F.n;
    j["fixed_vertices"] = static_cast<int>(s.fixed.size());
    j["ordering"] = F.ordering;
    j["factor_nnz"] = F.row_off.back();
    j["factor_fill_ratio"] = static_cast<double>(F.row_off.back()) / (static_cast<double>(F.n) * F.n);
    j["l_nnz"] = F.l_nnz;
    j["factor_millis"] = F.millis;
    {  // host build phases (ms): assembly, ordering, elimination tree, LDL^T, S' values, packing
      const double* c = F.ms_phase;
      j["factor_phase_millis"] = {{"assembly", c[0]}, {"ordering", c[1] - c[0]}, {"etree", c[2] - c[1]},
                                  {"ldlt", c[3] - c[2]}, {"inverse_values", c[4] - c[3]},
                                  {"stream_packing", F.millis - c[4]}};
    }
    j["segments"] = F.seg.size();
    j["chunks"] = F.chunks.size();
    j["stream_values"] = F.stream.size();
    j["weight_contrast"] = s.material.contrast();
    j["refactorizations"] = 1;
    j["inverse_residual"] = factor_inverse_residual(F);
    if (const char* mc = std::getenv("HETERODYN_MF_CHECK"); mc && std::atoi(mc) != 0) {
      // the device refactorization's plan and its CPU reference against the host LDL^T
      const HostFactor G = build_factor(s.mesh, s.material, s.solver.h, s.fixed, s.ordering, true);
      const auto t0 = std::chrono::steady_clock::now();
      const MfPlan P = mf_plan(G);
      Vec lx, d;
      mf_factor_host(P, G.a_ff.val, lx, d);
      const double ms = std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
      double lmax = 0, dmax = 0, lnorm = 0;
      for (size_t k = 0; k < lx.size(); ++k) {
        lmax = std::max(lmax, std::fabs(lx[k] - G.build.lx[k]));
        lnorm = std::max(lnorm, std::fabs(G.build.lx[k]));
      }
      for (int i = 0; i < G.n; ++i) {
        const double di = 1.0 / std::sqrt(d[i]);
        dmax = std::max(dmax, std::fabs(di - G.build.dis[i]) / G.build.dis[i]);
      }
      long long flops = 0;
      for (int q = 0; q < P.nsuper; ++q) {
        const long long m = P.fm[q], p = P.sfirst[q + 1] - P.sfirst[q];
        for (long long c = 0; c < p; ++c) flops += (m - c) * (m - c);
      }
      j["mf_check"] = {{"supernodes", P.nsuper}, {"levels", P.nlevels}, {"pool_doubles", P.pool},
                       {"max_front", P.max_front}, {"lx_max_abs_diff_rel", lnorm > 0 ? lmax / lnorm : 0.0},
                       {"dis_max_rel_diff", dmax}, {"host_ms", ms}, {"front_update_flops", flops}};
    }
    if (stats_json) *stats_json = dup(j.dump(2));
  });
}

hd_status hd_sim_record(hd_sim* sim, int enable) {
  if (!sim) return bad_arg("hd_sim_record: sim is NULL");
  sim->eng->record(enable != 0);
  return HD_OK;
}
int hd_sim_recorded_frames(const hd_sim* sim) { return sim ? sim->eng->recorded() : 0; }

hd_status hd_sim_set_state(hd_sim* sim, const double* q, const double* v, double time) {
  if (!sim) return bad_arg("hd_sim_set_state: sim is NULL");
  return guarded([&] { sim->eng->set_state(q, v, time); });
}

hd_status hd_sim_external_force(const hd_sim* sim, double* out, size_t cap) {
  if (!sim) return bad_arg("hd_sim_external_force: sim is NULL");
  if (!out || cap < sim->eng->dof_count()) return bad_arg("hd_sim_external_force: output buffer too small");
  return guarded([&] { sim->eng->external_force_into(out); });
}
hd_status hd_sim_set_external_force(hd_sim* sim, const double* f, size_t count) {
  if (!sim) return bad_arg("hd_sim_set_external_force: sim is NULL");
  if (!f || count != sim->eng->dof_count()) return bad_arg("hd_sim_set_external_force: expected dof doubles");
  return guarded([&] { sim->eng->set_external_force(f); });
}

hd_status hd_sim_backward(hd_sim* sim, const double* direct, const double* dq_final, const double* dv_final,
                          double* dl_dq0, double* dl_dv0, double* dl_df_ext, double* dl_de, double* dl_dw,
                          size_t dl_dw_capacity) {
  if (!sim) return bad_arg("hd_sim_backward: sim is NULL");
  return guarded([&] {
    if (dl_dw && dl_dw_capacity < sim->eng->dw_count())
      raise(Code::InvalidArgument, "hd_sim_backward: dl_dw buffer too small");
    Engine::GradSinks sinks;
    sinks.dq0 = dl_dq0;
    sinks.dv0 = dl_dv0;
    sinks.df_ext = dl_df_ext;
    sinks.de = dl_de;
    sinks.dw = dl_dw;
    sim->last_grad = sim->eng->backward(direct, dq_final, dv_final, false, true, nullptr, &sinks);
  });
}

hd_status hd_sim_backward_tau(const hd_sim* sim, double* tau, double* rho, size_t cap) {
  if (!sim) return bad_arg("hd_sim_backward_tau: sim is NULL");
  const auto& g = sim->last_grad;
  if (cap < g.tau.size()) return bad_arg("hd_sim_backward_tau: output buffer too small");
  if (tau) std::memcpy(tau, g.tau.data(), g.tau.size() * sizeof(double));
  if (rho) std::memcpy(rho, g.rho.data(), g.rho.size() * sizeof(double));
  return HD_OK;
}
int hd_sim_backward_iterations(const hd_sim* sim) { return sim ? sim->last_grad.adjoint_iterations : 0; }

hd_status hd_sim_solve_free(hd_sim* sim, const double* rhs, const double* fixed_q, double* out) {
  if (!sim || !rhs || !out) return bad_arg("hd_sim_solve_free: NULL argument");
  return guarded([&] {
    const Vec x = sim->eng->solve_free(rhs, fixed_q);
    // fixed entries of the result are the prescribed positions (factor.cpp:197)
    std::memcpy(out, x.data(), x.size() * sizeof(double));
    for (int v : sim->scene->spec.fixed)
      for (int a = 0; a < 3; ++a) out[3 * v + a] = fixed_q ? fixed_q[3 * v + a] : 0.0;
  });
}

hd_status hd_sim_set_young(hd_sim* sim, const double* young, size_t count, int freeze) {
  if (!sim || !young) return bad_arg("hd_sim_set_young: NULL argument");
  return guarded([&] { sim->eng->set_young(Vec(young, young + count), freeze != 0); });
}

hd_status hd_sim_set_deflation(hd_sim* sim, int on) {
  if (!sim) return bad_arg("hd_sim_set_deflation: sim is NULL");
  return guarded([&] { sim->eng->set_deflation(on != 0); });
}

hd_status hd_sim_backward_canonical(hd_sim* sim, double* dl_dq0, double* dl_dv0, double* dl_df_ext, double* dl_de,
                                    double* dl_dw, size_t dl_dw_capacity) {
  if (!sim) return bad_arg("hd_sim_backward_canonical: sim is NULL");
  return guarded([&] {
    const bool any = dl_dq0 || dl_dv0 || dl_df_ext || dl_de || dl_dw;
    if (dl_dw && dl_dw_capacity < sim->eng->dw_count()) raise(Code::InvalidArgument, "dl_dw buffer too small");
    Engine::GradSinks sinks;
    sinks.dq0 = dl_dq0;
    sinks.dv0 = dl_dv0;
    sinks.df_ext = dl_df_ext;
    sinks.de = dl_de;
    sinks.dw = dl_dw;
    sim->last_grad = sim->eng->backward(nullptr, nullptr, nullptr, true, false, nullptr, any ? &sinks : nullptr);
  });
}

void* hd_sim_stream(const hd_sim* sim) { return sim ? static_cast<void*>(sim->eng->stream()) : nullptr; }
long long hd_sim_kernel_launches(const hd_sim* sim) { return sim ? sim->eng->kernel_launches : 0; }

hd_status hd_sim_time_solve(hd_sim* sim, int reps, double* ms, double* bytes) {
  if (!sim || !ms || reps < 1) return bad_arg("hd_sim_time_solve: bad argument");
  return guarded([&] { *ms = sim->eng->time_solve(reps, bytes); });
}

hd_status hd_sim_time_backbone(hd_sim* sim, int reps, unsigned skip_mask, double* ms) {
  if (!sim || !ms || reps < 1) return bad_arg("hd_sim_time_backbone: bad argument");
  return guarded([&] {
    // bit 16: the multi-column contact-adjoint iteration instead (bits 17-18: skip solve / column kernels)
    *ms = (skip_mask & 0x10000u) ? sim->eng->time_columns(reps, (skip_mask >> 17) & 3u)
                                 : sim->eng->time_backbone(reps, skip_mask);
  });
}

hd_status hd_sim_trace_backbone(hd_sim* sim, int reps, double* out, size_t capacity) {
  if (!sim || !out || reps < 1) return bad_arg("hd_sim_trace_backbone: bad argument");
  return guarded([&] {
    std::vector<double> v;
    sim->eng->trace_backbone(reps, v);
    if (v.size() > capacity) raise(Code::InvalidArgument, "hd_sim_trace_backbone: capacity too small");
    std::copy(v.begin(), v.end(), out);
  });
}

hd_status hd_sim_trace_loop(hd_sim* sim, double* out, size_t capacity, int* iterations) {
  if (!sim || !out) return bad_arg("hd_sim_trace_loop: bad argument");
  return guarded([&] {
    std::vector<double> v;
    sim->eng->trace_loop(v);
    if (v.size() > capacity) raise(Code::InvalidArgument, "hd_sim_trace_loop: capacity too small");
    std::copy(v.begin(), v.end(), out);
    if (iterations) *iterations = static_cast<int>(v.size() / 42);
  });
}

long long hd_sim_factor_nnz(const hd_sim* sim) { return sim ? sim->eng->factor().row_off.back() : 0; }
int hd_sim_free_count(const hd_sim* sim) { return sim ? sim->eng->factor().n : 0; }
long long hd_sim_solve_count(const hd_sim* sim) { return sim ? sim->eng->solve_count : 0; }
long long hd_sim_factor_streams(const hd_sim* sim) { return sim ? sim->eng->factor_streams() : 0; }
long long hd_sim_a_spmv_count(const hd_sim* sim) { return sim ? sim->eng->a_spmv_count : 0; }
long long hd_sim_refactor_count(const hd_sim* sim) { return sim ? sim->eng->refactor_count : 0; }

}  // extern "C"

hd_batch* hd_batch_create(const hd_scene* scene, int samples, const double* young, size_t young_count, int threads) {
  if (!scene) {
    bad_arg("hd_batch_create: scene is NULL");
    return nullptr;
  }
  auto b = std::make_unique<hd_batch>();
  b->scene = scene;
  const hd_status st = guarded([&] {
    if (young && young_count != static_cast<size_t>(samples) * scene->spec.mesh.ne)
      raise(Code::InvalidArgument, "hd_batch_create: young must hold samples x element_count values");
    b->b = std::make_unique<Batch>(scene->spec, samples, young, threads);
  });
  return st == HD_OK ? b.release() : nullptr;
}

void hd_batch_free(hd_batch* batch) { delete batch; }
int hd_batch_sample_count(const hd_batch* batch) { return batch ? batch->b->samples() : 0; }

hd_status hd_batch_set_target(hd_batch* batch, const double* q, size_t count) {
  if (!batch || !q) return bad_arg("hd_batch_set_target: NULL argument");
  if (count != 3 * static_cast<size_t>(batch->scene->spec.mesh.nv)) return bad_arg("hd_batch_set_target: count != dof");
  return guarded([&] { batch->b->set_target(q); });
}

hd_status hd_batch_set_young(hd_batch* batch, const double* young, size_t count, int freeze_means) {
  if (!batch || !young) return bad_arg("hd_batch_set_young: NULL argument");
  if (count != static_cast<size_t>(batch->b->samples()) * batch->scene->spec.mesh.ne)
    return bad_arg("hd_batch_set_young: young must hold samples x element_count values");
  return guarded([&] { batch->b->set_young(young, freeze_means != 0); });
}

hd_status hd_batch_evaluate(hd_batch* batch, int frames, double* loss, size_t loss_cap, double* grad, size_t grad_cap,
                            void* device_out) {
  if (!batch) return bad_arg("hd_batch_evaluate: batch is NULL");
  if (loss && loss_cap < static_cast<size_t>(batch->b->samples()))
    return bad_arg("hd_batch_evaluate: loss buffer too small");
  if (grad && grad_cap < static_cast<size_t>(batch->scene->spec.mesh.ne))
    return bad_arg("hd_batch_evaluate: gradient buffer too small");
  return guarded([&] { batch->b->evaluate(frames, loss, grad, static_cast<double*>(device_out)); });
}

double hd_batch_last_ms(const hd_batch* batch) { return batch ? batch->b->last_ms : 0.0; }
long long hd_batch_kernel_launches(const hd_batch* batch) { return batch ? batch->b->kernel_launches() : 0; }
long long hd_batch_solve_count(const hd_batch* batch) { return batch ? batch->b->solve_count() : 0; }
hd_status hd_batch_time_solve(hd_batch* batch, int reps, double* ms, double* bytes) {
  if (!batch || !ms || reps < 1) return bad_arg("hd_batch_time_solve: bad argument");
  return guarded([&] { *ms = batch->b->time_solve(reps, bytes); });
}
int hd_batch_lockstep(const hd_batch* batch) { return batch && batch->b->lockstep() ? 1 : 0; }
double hd_batch_solve_bytes(const hd_batch* batch) { return batch ? batch->b->solve_bytes() : 0.0; }
