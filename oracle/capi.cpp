// ORACLE — test infrastructure only.  The hd_* C ABI of include/heterodyn.h
// over the CPU restatement (reference capi.cpp:94-322 for the reference half;
// the B200-extension half routes to roll/chain_backward, drivers.cpp:31-99).
#include <chrono>
#include <cstdlib>
#include <cstring>
#include <fstream>


#include <nlohmann/json.hpp>

#include "../paper_2605_14526_b200/csrc/drivers.hpp"

#include "../include/heterodyn.h"
#include "oracle.hpp"

using namespace hdo;

struct hd_scene {
  SceneSpec spec;
};

struct hd_sim {
  const hd_scene* scene = nullptr;
  MaterialField material;  // per-sim copy so set_young does not touch the scene
  GlobalSystem system;
  StateForce hook_storage;
  const StateForce* hook = nullptr;
  VecX f_ext;
  SimState state;
  int last_iterations = 0;
  bool last_converged = false;
  int last_contact_count = 0;
  double last_fb_residual = 0;
  std::vector<int> trace_vertex, trace_obstacle;
  std::vector<double> trace_clamp, trace_cone;
  int trace_nf = 0;
  bool record = false;
  std::vector<ForwardCache> caches;
  std::vector<double> tau, rho;
  int backward_iterations = 0;
  long long solve_count_base = 0;
};

namespace {
thread_local int g_code = 0;
thread_local std::string g_msg;
void set_error(int code, const std::string& m) {
  g_code = code;
  g_msg = m;
}
template <typename Fn>
hd_status guarded(Fn&& fn) {
  try {
    fn();
    return HD_OK;
  } catch (const Error& e) {
    set_error(static_cast<int>(e.code()), e.what());
    return static_cast<hd_status>(e.code());
  } catch (const std::exception& e) {
    set_error(HD_ERR_INVALID_ARGUMENT, std::string("unexpected error: ") + e.what());
    return HD_ERR_INVALID_ARGUMENT;
  }
}
char* copy_string(const std::string& s) {
  char* out = static_cast<char*>(std::malloc(s.size() + 1));
  if (out) std::memcpy(out, s.c_str(), s.size() + 1);
  return out;
}
hd_status copy_vector(const VecX& v, double* out, size_t cap, const char* who) {
  if (out == nullptr || cap < v.size()) {
    set_error(HD_ERR_INVALID_ARGUMENT, std::string(who) + ": output buffer too small");
    return HD_ERR_INVALID_ARGUMENT;
  }
  std::memcpy(out, v.data(), sizeof(double) * v.size());
  return HD_OK;
}
hd_status null_arg(const char* who) {
  set_error(HD_ERR_INVALID_ARGUMENT, std::string(who) + ": NULL argument");
  return HD_ERR_INVALID_ARGUMENT;
}
}  // namespace

extern "C" {

const char* hd_last_error(void) { return g_msg.c_str(); }
int hd_last_error_code(void) { return g_code; }
void hd_string_free(char* s) { std::free(s); }

hd_scene* hd_scene_load(const char* path) {
  if (!path) { null_arg("hd_scene_load"); return nullptr; }
  hd_scene* s = new hd_scene;
  if (guarded([&] { s->spec = load_scene_file(path); }) != HD_OK) { delete s; return nullptr; }
  return s;
}
hd_scene* hd_scene_parse(const char* text) {
  if (!text) { null_arg("hd_scene_parse"); return nullptr; }
  hd_scene* s = new hd_scene;
  if (guarded([&] { s->spec = parse_scene_json(text); }) != HD_OK) { delete s; return nullptr; }
  return s;
}
hd_scene* hd_scene_builtin(const char* name) {
  if (!name) { null_arg("hd_scene_builtin"); return nullptr; }
  hd_scene* s = new hd_scene;
  if (guarded([&] { s->spec = builtin_scene(name); }) != HD_OK) { delete s; return nullptr; }
  return s;
}
void hd_scene_free(hd_scene* s) { delete s; }
int hd_scene_vertex_count(const hd_scene* s) { return s ? s->spec.mesh.vertex_count() : 0; }
int hd_scene_element_count(const hd_scene* s) { return s ? s->spec.mesh.element_count() : 0; }
int hd_scene_frame_count(const hd_scene* s) { return s ? s->spec.frames : 0; }
const char* hd_scene_name(const hd_scene* s) { return s ? s->spec.name.c_str() : ""; }

int hd_scene_region_count(const hd_scene* s) { return s ? s->spec.region_count : 0; }
hd_status hd_scene_regions(const hd_scene* s, int* out, size_t cap) {
  if (!s) return null_arg("hd_scene_regions");
  const size_t ne = static_cast<size_t>(s->spec.mesh.element_count());
  if (!out || cap < ne) {
    set_error(HD_ERR_INVALID_ARGUMENT, "hd_scene_regions: output buffer too small");
    return HD_ERR_INVALID_ARGUMENT;
  }
  const auto& r = s->spec.region_of_element;
  for (size_t e = 0; e < ne; ++e) out[e] = e < r.size() ? r[e] : 0;
  return HD_OK;
}
hd_status hd_scene_rest_positions(const hd_scene* s, double* out, size_t cap) {
  if (!s) return null_arg("hd_scene_rest_positions");
  return copy_vector(s->spec.mesh.rest_vector(), out, cap, "hd_scene_rest_positions");
}
hd_status hd_scene_vertex_masses(const hd_scene* s, double* out, size_t cap) {
  if (!s) return null_arg("hd_scene_vertex_masses");
  const int nv = s->spec.mesh.vertex_count();
  if (!out || cap < static_cast<size_t>(nv)) {
    set_error(HD_ERR_INVALID_ARGUMENT, "hd_scene_vertex_masses: output buffer too small");
    return HD_ERR_INVALID_ARGUMENT;
  }
  for (int v = 0; v < nv; ++v) out[v] = s->spec.mesh.vertex_mass(v);
  return HD_OK;
}

hd_status hd_scene_elements(const hd_scene* s, int* out, size_t cap) {
  if (!s) return null_arg("hd_scene_elements");
  const auto& el = s->spec.mesh.elements();
  if (!out || cap < 4 * el.size()) {
    set_error(HD_ERR_INVALID_ARGUMENT, "hd_scene_elements: output buffer too small");
    return HD_ERR_INVALID_ARGUMENT;
  }
  for (size_t e = 0; e < el.size(); ++e)
    for (int k = 0; k < 4; ++k) out[4 * e + k] = el[e][k];
  return HD_OK;
}
hd_status hd_scene_young_moduli(const hd_scene* s, double* out, size_t cap) {
  if (!s) return null_arg("hd_scene_young_moduli");
  const int ne = s->spec.material.element_count();
  if (!out || cap < static_cast<size_t>(ne)) {
    set_error(HD_ERR_INVALID_ARGUMENT, "hd_scene_young_moduli: output buffer too small");
    return HD_ERR_INVALID_ARGUMENT;
  }
  for (int e = 0; e < ne; ++e) out[e] = s->spec.material.young(e);
  return HD_OK;
}

hd_sim* hd_sim_create(const hd_scene* scene) {
  if (!scene) { null_arg("hd_sim_create"); return nullptr; }
  hd_sim* sim = new hd_sim;
  const hd_status st = guarded([&] {
    sim->scene = scene;
    const SceneSpec& s = scene->spec;
    sim->material = s.material;
    sim->system.refresh(s.mesh, sim->material, s.solver.h, s.fixed_vertices);
    if (s.has_hook) {
      sim->hook_storage = make_hook(s);
      sim->hook = &sim->hook_storage;
    }
    sim->f_ext = scene_external_force(s);
    sim->state.q = s.q0;
    sim->state.v = s.v0;
    sim->state.time = 0.0;
  });
  if (st != HD_OK) { delete sim; return nullptr; }
  return sim;
}
void hd_sim_free(hd_sim* sim) { delete sim; }

hd_status hd_sim_step(hd_sim* sim) {
  if (!sim) return null_arg("hd_sim_step");
  return guarded([&] {
    const SceneSpec& s = sim->scene->spec;
    SimState st = sim->state;
    ForwardCache cache = forward_step(s.mesh, sim->material, sim->system, s.solver, s.obstacles, s.fixed_vertices,
                                      st, sim->f_ext, sim->hook);
    sim->state = st;
    sim->last_iterations = cache.iteration_count;
    sim->last_converged = cache.converged;
    sim->last_contact_count = cache.contacts.normal_count();
    double fb = 0;  // max_normal_fb_residual (drivers.cpp:147-159)
    for (int c = 0; c < cache.contacts.normal_count(); ++c) {
      const ContactPoint& cp = cache.contacts.contacts[c];
      const double delta = cp.normal.dot(seg3(cache.q_star, cp.vertex)) - cp.gap_offset;
      fb = std::max(fb, std::abs(fb_residual(delta, cp.r_n, cache.lambda_star[c])));
    }
    sim->last_fb_residual = fb;
    sim->trace_vertex.clear();
    sim->trace_obstacle.clear();
    for (const ContactPoint& cp : cache.contacts.contacts) {
      sim->trace_vertex.push_back(cp.vertex);
      sim->trace_obstacle.push_back(cp.obstacle_id);
    }
    sim->trace_nf = cache.contacts.friction_pair_count();
    sim->trace_clamp = cache.trace_clamp;
    sim->trace_cone = cache.trace_cone;
    if (sim->record) sim->caches.push_back(std::move(cache));
  });
}
double hd_sim_time(const hd_sim* sim) { return sim ? sim->state.time : 0.0; }
int hd_sim_dof_count(const hd_sim* sim) { return sim ? static_cast<int>(sim->state.q.size()) : 0; }
hd_status hd_sim_positions(const hd_sim* sim, double* out, size_t cap) {
  if (!sim) return null_arg("hd_sim_positions");
  return copy_vector(sim->state.q, out, cap, "hd_sim_positions");
}
hd_status hd_sim_velocities(const hd_sim* sim, double* out, size_t cap) {
  if (!sim) return null_arg("hd_sim_velocities");
  return copy_vector(sim->state.v, out, cap, "hd_sim_velocities");
}
int hd_sim_last_iterations(const hd_sim* sim) { return sim ? sim->last_iterations : 0; }
int hd_sim_last_converged(const hd_sim* sim) { return sim && sim->last_converged ? 1 : 0; }
int hd_sim_last_contact_count(const hd_sim* sim) { return sim ? sim->last_contact_count : 0; }
hd_status hd_sim_contact_trace(const hd_sim* sim, int* vertex, int* obstacle, size_t row_capacity,
                               double* clamp, size_t clamp_capacity, double* cone, size_t cone_capacity,
                               int* counts) {
  if (!sim) return null_arg("hd_sim_contact_trace");
  const int nc = static_cast<int>(sim->trace_vertex.size()), nf = sim->trace_nf;
  const int iters = nc > 0 ? static_cast<int>(sim->trace_clamp.size() / nc) : 0;
  if (counts) {
    counts[0] = nc;
    counts[1] = nf;
    counts[2] = iters;
  }
  if ((vertex || obstacle) && row_capacity < static_cast<size_t>(nc)) {
    set_error(HD_ERR_INVALID_ARGUMENT, "hd_sim_contact_trace: row capacity too small");
    return HD_ERR_INVALID_ARGUMENT;
  }
  if ((clamp && clamp_capacity < sim->trace_clamp.size()) || (cone && cone_capacity < sim->trace_cone.size())) {
    set_error(HD_ERR_INVALID_ARGUMENT, "hd_sim_contact_trace: pattern capacity too small");
    return HD_ERR_INVALID_ARGUMENT;
  }
  if (vertex) std::copy(sim->trace_vertex.begin(), sim->trace_vertex.end(), vertex);
  if (obstacle) std::copy(sim->trace_obstacle.begin(), sim->trace_obstacle.end(), obstacle);
  if (clamp) std::copy(sim->trace_clamp.begin(), sim->trace_clamp.end(), clamp);
  if (cone) std::copy(sim->trace_cone.begin(), sim->trace_cone.end(), cone);
  return HD_OK;
}
double hd_sim_last_fb_residual(const hd_sim* sim) { return sim ? sim->last_fb_residual : 0.0; }
double hd_sim_penetration(const hd_sim* sim) {  // max_penetration_at (drivers.cpp:101-111)
  if (!sim) return 0.0;
  double pen = 0;
  for (const auto& ob : sim->scene->spec.obstacles)
    for (int v = 0; v < sim->scene->spec.mesh.vertex_count(); ++v)
      pen = std::max(pen, -obstacle_signed_distance(ob, seg3(sim->state.q, v)));
  return pen;
}

// ---- drivers: simulate, gradcheck, identify (the shared drivers.cpp) ----
hd_status hd_run_simulate(const hd_scene* scene, const char* out_dir, char** summary_json) {
  if (!scene) return null_arg("hd_run_simulate");
  std::string out, err;
  const int code = heterodyn_driver::run_simulate(scene, out_dir, &out, &err);
  if (code != HD_OK) {
    set_error(code, err);
    return static_cast<hd_status>(code);
  }
  if (summary_json) *summary_json = copy_string(out);
  return HD_OK;
}
hd_status hd_run_gradcheck(const hd_scene* scene, const char* vars_csv, const char* out_path, char** report_json,
                           int* pass) {
  if (!scene) return null_arg("hd_run_gradcheck");
  std::string out, err;
  bool ok = false;
  const int code = heterodyn_driver::run_gradcheck(scene, vars_csv, out_path, &out, &ok, &err);
  if (code != HD_OK) {
    set_error(code, err);
    return static_cast<hd_status>(code);
  }
  if (report_json) *report_json = copy_string(out);
  if (pass) *pass = ok ? 1 : 0;
  return HD_OK;
}
// System identification: the product's L-BFGS driver (drivers.cpp, written
// against the public ABI only) linked over this library's CPU restatement, so
// the parity tests compare the solvers underneath one optimizer.
static hd_status identify_finish(int code, const std::string& out, bool st, const std::string& err, char** result_json,
                          int* stalled) {
  if (code != HD_OK) {
    set_error(code, err);
    return static_cast<hd_status>(code);
  }
  if (result_json) *result_json = copy_string(out);
  if (stalled) *stalled = st ? 1 : 0;
  return HD_OK;
}
hd_status hd_run_identify(const char* problem_json, const char* out_dir, char** result_json, int* stalled) {
  if (!problem_json) return null_arg("hd_run_identify");
  std::string out, err;
  bool st = false;
  const int code = heterodyn_driver::run_identify(problem_json, out_dir ? out_dir : "", &out, &st, &err);
  return identify_finish(code, out, st, err, result_json, stalled);
}
hd_status hd_run_identify_file(const char* problem_path, const char* out_dir, char** result_json, int* stalled) {
  if (!problem_path) return null_arg("hd_run_identify_file");
  std::string out, err;
  bool st = false;
  const int code = heterodyn_driver::run_identify_file(problem_path, out_dir ? out_dir : "", &out, &st, &err);
  return identify_finish(code, out, st, err, result_json, stalled);
}
hd_status hd_factor_stats(const hd_scene* scene, char** stats_json) {
  if (!scene) return null_arg("hd_factor_stats");
  return guarded([&] {
    const SceneSpec& s = scene->spec;
    GlobalSystem sys;
    sys.refresh(s.mesh, s.material, s.solver.h, s.fixed_vertices);
    nlohmann::json j;
    j["vertices"] = s.mesh.vertex_count();
    j["elements"] = s.mesh.element_count();
    j["dofs"] = s.mesh.dof_count();
    j["free_vertices"] = sys.free_count();
    j["fixed_vertices"] = static_cast<int>(sys.fixed_vertices().size());
    j["ordering"] = sys.factor().ordering_name();
    j["factor_nnz"] = sys.factor().s_nnz();
    j["factor_fill_ratio"] = sys.factor().s_fill_ratio();
    j["l_nnz"] = sys.factor().l_nnz();
    j["factor_millis"] = sys.factor().factor_millis();
    j["weight_contrast"] = s.material.weight_contrast();
    j["refactorizations"] = sys.refactor_count();
    if (stats_json) *stats_json = copy_string(j.dump(2));
  });
}

// ---- B200 extensions -------------------------------------------------------
hd_status hd_sim_record(hd_sim* sim, int enable) {
  if (!sim) return null_arg("hd_sim_record");
  sim->record = enable != 0;
  if (!enable) sim->caches.clear();
  return HD_OK;
}
int hd_sim_recorded_frames(const hd_sim* sim) { return sim ? static_cast<int>(sim->caches.size()) : 0; }

hd_status hd_sim_set_state(hd_sim* sim, const double* q, const double* v, double time) {
  if (!sim) return null_arg("hd_sim_set_state");
  const size_t n = sim->state.q.size();
  if (q) sim->state.q.assign(q, q + n);
  if (v) sim->state.v.assign(v, v + n);
  sim->state.time = time;
  sim->caches.clear();
  return HD_OK;
}

hd_status hd_sim_external_force(const hd_sim* sim, double* out, size_t cap) {
  if (!sim) return null_arg("hd_sim_external_force");
  return copy_vector(sim->f_ext, out, cap, "hd_sim_external_force");
}
hd_status hd_sim_set_external_force(hd_sim* sim, const double* f, size_t count) {
  if (!sim) return null_arg("hd_sim_set_external_force");
  if (!f || count != static_cast<size_t>(sim->f_ext.size())) {
    set_error(HD_ERR_INVALID_ARGUMENT, "hd_sim_set_external_force: expected dof doubles");
    return HD_ERR_INVALID_ARGUMENT;
  }
  sim->f_ext.assign(f, f + count);
  return HD_OK;
}

hd_status hd_sim_backward(hd_sim* sim, const double* dl_dq_direct, const double* dl_dq_final,
                          const double* dl_dv_final, double* dl_dq0, double* dl_dv0, double* dl_df_ext,
                          double* dl_de, double* dl_dw, size_t dl_dw_capacity) {
  if (!sim) return null_arg("hd_sim_backward");
  return guarded([&] {
    const SceneSpec& s = sim->scene->spec;
    const int frames = static_cast<int>(sim->caches.size());
    if (frames == 0) fail(ErrorCode::InvalidArgument, "hd_sim_backward: no recorded frames");
    const int n = s.mesh.dof_count();
    std::vector<VecX> direct(frames + 1, zeros(n));
    if (dl_dq_direct) {
      for (int t = 0; t <= frames; ++t) direct[t].assign(dl_dq_direct + static_cast<size_t>(t) * n, dl_dq_direct + static_cast<size_t>(t + 1) * n);
    } else if (dl_dq_final) {
      direct[frames].assign(dl_dq_final, dl_dq_final + n);
    }
    const VecX vfin = dl_dv_final ? VecX(dl_dv_final, dl_dv_final + n) : zeros(n);
    const ChainResult r = chain_backward(s.mesh, sim->material, sim->system, sim->caches, direct, vfin, sim->hook,
                                         s.solver.eps_tr);
    if (dl_dw && dl_dw_capacity < r.dl_dw.size()) fail(ErrorCode::InvalidArgument, "hd_sim_backward: dl_dw buffer too small");
    if (dl_dq0) std::memcpy(dl_dq0, r.dl_dq0.data(), sizeof(double) * n);
    if (dl_dv0) std::memcpy(dl_dv0, r.dl_dv0.data(), sizeof(double) * n);
    if (dl_df_ext) std::memcpy(dl_df_ext, r.dl_df_ext.data(), sizeof(double) * n);
    if (dl_de) std::memcpy(dl_de, r.dl_de.data(), sizeof(double) * r.dl_de.size());
    if (dl_dw) std::memcpy(dl_dw, r.dl_dw.data(), sizeof(double) * r.dl_dw.size());
    sim->tau = r.tau;
    sim->rho = r.rho;
    sim->backward_iterations = r.adjoint_iterations;
  });
}

hd_status hd_sim_backward_tau(const hd_sim* sim, double* tau, double* rho, size_t cap) {
  if (!sim) return null_arg("hd_sim_backward_tau");
  if (cap < sim->tau.size()) {
    set_error(HD_ERR_INVALID_ARGUMENT, "hd_sim_backward_tau: output buffer too small");
    return HD_ERR_INVALID_ARGUMENT;
  }
  if (tau) std::memcpy(tau, sim->tau.data(), sizeof(double) * sim->tau.size());
  if (rho) std::memcpy(rho, sim->rho.data(), sizeof(double) * sim->rho.size());
  return HD_OK;
}
int hd_sim_backward_iterations(const hd_sim* sim) { return sim ? sim->backward_iterations : 0; }

hd_status hd_sim_solve_free(hd_sim* sim, const double* rhs, const double* fixed_q, double* out) {
  if (!sim || !rhs || !out) return null_arg("hd_sim_solve_free");
  return guarded([&] {
    const size_t n = sim->state.q.size();
    const VecX r(rhs, rhs + n);
    const VecX fq = fixed_q ? VecX(fixed_q, fixed_q + n) : zeros(static_cast<int>(n));
    const VecX x = sim->system.solve_free(r, fq);
    std::memcpy(out, x.data(), sizeof(double) * n);
  });
}

hd_status hd_sim_set_deflation(hd_sim* sim, int) {  // the CPU restatement has no recycled subspace
  if (!sim) return null_arg("hd_sim_set_deflation");
  return HD_OK;
}

hd_status hd_sim_set_young(hd_sim* sim, const double* young, size_t count, int freeze) {
  if (!sim || !young) return null_arg("hd_sim_set_young");
  return guarded([&] {
    if (freeze) sim->material.freeze_means(sim->material.prox_means());
    sim->material.set_young(std::vector<double>(young, young + count));
    const SceneSpec& s = sim->scene->spec;
    sim->system.refresh(s.mesh, sim->material, s.solver.h, s.fixed_vertices);
    sim->caches.clear();
  });
}

hd_status hd_sim_backward_canonical(hd_sim* sim, double* dl_dq0, double* dl_dv0, double* dl_df_ext, double* dl_de,
                                    double* dl_dw, size_t dl_dw_capacity) {
  if (!sim) return null_arg("hd_sim_backward_canonical");
  const SceneSpec& s = sim->scene->spec;
  VecX dq = sim->state.q;
  for (size_t i = 0; i < dq.size(); ++i) dq[i] -= s.mesh.rest_vector()[i];
  return hd_sim_backward(sim, nullptr, dq.data(), sim->state.v.data(), dl_dq0, dl_dv0, dl_df_ext, dl_de, dl_dw,
                         dl_dw_capacity);
}
void* hd_sim_stream(const hd_sim*) { return nullptr; }
long long hd_sim_kernel_launches(const hd_sim*) { return 0; }
hd_status hd_sim_trace_loop(hd_sim*, double*, size_t, int*) {
  return null_arg("hd_sim_trace_loop: GPU profiling only");
}
hd_status hd_sim_trace_backbone(hd_sim*, int, double*, size_t) {
  return null_arg("hd_sim_trace_backbone: GPU profiling only");
}
hd_status hd_sim_time_backbone(hd_sim*, int, unsigned, double*) {
  return null_arg("hd_sim_time_backbone: GPU profiling only");
}
hd_status hd_sim_time_solve(hd_sim* sim, int reps, double* ms, double* bytes) {
  if (!sim || !ms || reps < 1) return null_arg("hd_sim_time_solve");
  return guarded([&] {
    const size_t n = sim->state.q.size();
    VecX rhs(n, 1.0), fq(n, 0.0);
    const auto t0 = std::chrono::steady_clock::now();
    for (int i = 0; i < reps; ++i) sim->system.solve_free(rhs, fq);
    *ms = std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count() / reps;
    if (bytes) *bytes = 24.0 * static_cast<double>(sim->system.factor().s_nnz());
  });
}

long long hd_sim_factor_nnz(const hd_sim* sim) { return sim ? sim->system.factor().s_nnz() : 0; }
int hd_sim_free_count(const hd_sim* sim) { return sim ? sim->system.free_count() : 0; }
long long hd_sim_solve_count(const hd_sim* sim) {
  return sim ? static_cast<long long>(sim->system.factor().apply_inverse_count / 3) : 0;
}
long long hd_sim_factor_streams(const hd_sim* sim) { return hd_sim_solve_count(sim); }
long long hd_sim_a_spmv_count(const hd_sim* sim) { return sim ? static_cast<long long>(sim->system.a_spmv_count) : 0; }
long long hd_sim_refactor_count(const hd_sim* sim) { return sim ? static_cast<long long>(sim->system.refactor_count()) : 0; }


// ---- batched system-ID (config C5): the checker runs the samples in order
// with the single-trajectory API above (roll + chain_backward per sample,
// drivers.cpp:31-99; objective of run_identify, drivers.cpp:848-851).
struct hd_batch {
  const hd_scene* scene = nullptr;
  int samples = 0;
  std::vector<double> young;  // samples x ne, empty = scene's
  std::vector<double> target;
  int freeze = 0;             // freeze_means of the last hd_batch_set_young
};

hd_batch* hd_batch_create(const hd_scene* scene, int samples, const double* young, size_t young_count, int) {
  if (!scene) { null_arg("hd_batch_create"); return nullptr; }
  const size_t ne = scene->spec.mesh.element_count();
  if (samples < 1 || (young && young_count != ne * static_cast<size_t>(samples))) {
    set_error(HD_ERR_INVALID_ARGUMENT, "hd_batch_create: bad sample count or young size");
    return nullptr;
  }
  hd_batch* b = new hd_batch;
  b->scene = scene;
  b->samples = samples;
  if (young) b->young.assign(young, young + young_count);
  b->target = scene->spec.q0;
  return b;
}
void hd_batch_free(hd_batch* b) { delete b; }
int hd_batch_sample_count(const hd_batch* b) { return b ? b->samples : 0; }
hd_status hd_batch_set_target(hd_batch* b, const double* q, size_t count) {
  if (!b || !q) return null_arg("hd_batch_set_target");
  if (count != b->target.size()) {
    set_error(HD_ERR_INVALID_ARGUMENT, "hd_batch_set_target: count != dof");
    return HD_ERR_INVALID_ARGUMENT;
  }
  b->target.assign(q, q + count);
  return HD_OK;
}
hd_status hd_batch_set_young(hd_batch* b, const double* young, size_t count, int freeze_means) {
  if (!b || !young) return null_arg("hd_batch_set_young");
  if (count != b->scene->spec.mesh.element_count() * static_cast<size_t>(b->samples)) {
    set_error(HD_ERR_INVALID_ARGUMENT, "hd_batch_set_young: young must hold samples x element_count values");
    return HD_ERR_INVALID_ARGUMENT;
  }
  b->young.assign(young, young + count);
  b->freeze = freeze_means != 0;
  return HD_OK;
}
hd_status hd_batch_evaluate(hd_batch* b, int frames, double* loss, size_t loss_cap, double* grad, size_t grad_cap,
                            void* device_out) {
  if (!b) return null_arg("hd_batch_evaluate");
  const size_t ne = b->scene->spec.mesh.element_count(), n = b->target.size();
  if (device_out || frames < 1 || (loss && loss_cap < static_cast<size_t>(b->samples)) || (grad && grad_cap < ne)) {
    set_error(HD_ERR_INVALID_ARGUMENT, "hd_batch_evaluate: bad argument (the CPU oracle has no device output)");
    return HD_ERR_INVALID_ARGUMENT;
  }
  std::vector<double> sum(ne, 0.0), dle(ne), q(n), dq(n);
  for (int s = 0; s < b->samples; ++s) {
    hd_sim* sim = hd_sim_create(b->scene);
    if (!sim) return static_cast<hd_status>(hd_last_error_code());
    hd_status st = HD_OK;
    if (!b->young.empty()) st = hd_sim_set_young(sim, b->young.data() + s * ne, ne, b->freeze);
    if (st == HD_OK) st = hd_sim_record(sim, 1);
    for (int f = 0; f < frames && st == HD_OK; ++f) st = hd_sim_step(sim);
    if (st == HD_OK) st = hd_sim_positions(sim, q.data(), n);
    double l = 0;
    for (size_t i = 0; i < n; ++i) {
      dq[i] = q[i] - b->target[i];
      l += dq[i] * dq[i];
    }
    if (st == HD_OK) st = hd_sim_backward(sim, nullptr, dq.data(), nullptr, nullptr, nullptr, nullptr, dle.data(), nullptr, 0);
    hd_sim_free(sim);
    if (st != HD_OK) return st;
    if (loss) loss[s] = 0.5 * l;
    for (size_t e = 0; e < ne; ++e) sum[e] += dle[e];
  }
  if (grad) std::memcpy(grad, sum.data(), ne * sizeof(double));
  return HD_OK;
}
double hd_batch_last_ms(const hd_batch*) { return 0.0; }
long long hd_batch_kernel_launches(const hd_batch*) { return 0; }
long long hd_batch_solve_count(const hd_batch*) { return 0; }
double hd_batch_solve_bytes(const hd_batch*) { return 0.0; }
// profiling hooks of the device batch: nothing to time on the CPU checker
hd_status hd_batch_time_solve(hd_batch* batch, int reps, double* ms, double* bytes) {
  if (!batch || !ms || reps < 1) return null_arg("hd_batch_time_solve");
  *ms = 0.0;
  if (bytes) *bytes = 0.0;
  return HD_OK;
}
int hd_batch_lockstep(const hd_batch*) { return 0; }

}  // extern "C"
