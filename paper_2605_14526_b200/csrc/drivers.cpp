// Host drivers of the reference ABI: system identification (run_identify,
// drivers.cpp:570-979, with lbfgs_minimize, lbfgs.cpp:40-143), the
// finite-difference gradient check (run_gradcheck, drivers.cpp:367-531) and
// the simulate driver's outputs (run_simulate, drivers.cpp:238-365).
//
// Written against the public C ABI only (heterodyn.h: scenes, hd_sim_step,
// hd_sim_set_young, hd_sim_set_state, hd_sim_record, hd_sim_backward), so the
// optimizer, the design-variable chain rules and the losses are host control
// logic around the hot path: every forward frame and every adjoint frame runs
// through whichever library this file is linked into (the device engine in
// libheterodyn_b200.so; the CPU restatement in the oracle library, which links
// the same driver so the tests compare the solvers underneath it).
#include "drivers.hpp"

#include <algorithm>
#include <array>
#include <cmath>
#include <deque>
#include <cstdio>
#include <functional>
#include <limits>
#include <memory>
#include <vector>

#include <nlohmann/json.hpp>
#include <sys/stat.h>

#include "../../include/heterodyn.h"

namespace heterodyn_driver {
namespace {

using nlohmann::json;
using V = std::vector<double>;

struct Failure {
  int code;
  std::string msg;
};
[[noreturn]] void fail(int code, std::string msg) { throw Failure{code, std::move(msg)}; }
// Rethrows the library's own failure (thread-local code + message).
void check(hd_status s) {
  if (s != HD_OK) fail(s, hd_last_error());
}

double dot(const V& a, const V& b) {
  double s = 0;
  for (size_t i = 0; i < a.size(); ++i) s += a[i] * b[i];
  return s;
}

// ---- L-BFGS (lbfgs.cpp:40-143): two-loop recursion with gamma = s.y / y.y,
//      strong-Wolfe line search by bracketing and bisection -------------------
struct LbfgsConfig {
  int memory = 10;
  int max_evals = 100;
  double grad_tol = 1e-6;
};
struct LbfgsResult {
  V x;
  double loss = 0;
  int evaluations = 0;
  bool converged = false, stalled = false;
};
using Objective = std::function<double(const V&, V&)>;

struct Pair {
  V s, y;
  double rho;
};

V two_loop(const std::deque<Pair>& pairs, const V& g) {  // lbfgs.cpp:18-34
  V q = g;
  std::vector<double> a(pairs.size());
  for (int i = static_cast<int>(pairs.size()) - 1; i >= 0; --i) {
    a[i] = pairs[i].rho * dot(pairs[i].s, q);
    for (size_t k = 0; k < q.size(); ++k) q[k] -= a[i] * pairs[i].y[k];
  }
  if (!pairs.empty()) {
    const Pair& p = pairs.back();
    const double scale = dot(p.s, p.y) / dot(p.y, p.y);
    for (double& v : q) v *= scale;
  }
  for (size_t i = 0; i < pairs.size(); ++i) {
    const double b = pairs[i].rho * dot(pairs[i].y, q);
    for (size_t k = 0; k < q.size(); ++k) q[k] += (a[i] - b) * pairs[i].s[k];
  }
  return q;
}

LbfgsResult lbfgs(const Objective& f, const V& x0, const LbfgsConfig& cfg) {
  constexpr double c1 = 1e-4, c2 = 0.9;  // lbfgs.cpp:42-43
  LbfgsResult r;
  r.x = x0;
  const size_t n = x0.size();
  auto eval = [&](const V& x, V& g) {
    ++r.evaluations;
    return f(x, g);
  };
  V g(n);
  double loss = eval(r.x, g);
  r.loss = loss;
  if (!std::isfinite(loss)) {
    r.stalled = true;
    return r;
  }
  std::deque<Pair> pairs;
  for (;;) {
    double gmax = 0;
    for (double v : g) gmax = std::max(gmax, std::abs(v));
    if (gmax <= cfg.grad_tol) {
      r.converged = true;
      break;
    }
    if (r.evaluations >= cfg.max_evals) {
      r.stalled = true;
      break;
    }
    V d = two_loop(pairs, g);
    for (double& v : d) v = -v;
    double slope = dot(g, d);
    if (!(slope < 0)) {  // ascent from the history: restart with steepest descent
      pairs.clear();
      for (size_t k = 0; k < n; ++k) d[k] = -g[k];
      slope = dot(g, d);
    }
    double t = 1.0, lo = 0.0, hi = 0.0;
    bool bracketed = false, accepted = false;
    V xt(n), gt(n);
    double ft = loss;
    for (int ls = 0; ls < 30 && r.evaluations < cfg.max_evals; ++ls) {
      for (size_t k = 0; k < n; ++k) xt[k] = r.x[k] + t * d[k];
      ft = eval(xt, gt);
      const bool armijo = std::isfinite(ft) && ft <= loss + c1 * t * slope;
      const double dslope = dot(gt, d);
      if (!armijo) {
        hi = t;
        bracketed = true;
      } else if (std::abs(dslope) <= -c2 * slope) {
        accepted = true;
        break;
      } else if (dslope >= 0) {
        hi = t;
        lo = std::max(lo, 0.0);
        bracketed = true;
      } else {
        lo = t;
        if (!bracketed) {
          t *= 2;
          continue;
        }
      }
      if (bracketed && hi > lo) {
        t = 0.5 * (lo + hi);
        if (hi - lo < 1e-12) {
          accepted = armijo && ft < loss;
          break;
        }
      } else {
        t *= 2;
      }
    }
    if (!accepted && std::isfinite(ft) && ft < loss) accepted = true;
    if (!accepted) {
      r.stalled = true;
      break;
    }
    V s(n), y(n);
    for (size_t k = 0; k < n; ++k) {
      s[k] = xt[k] - r.x[k];
      y[k] = gt[k] - g[k];
    }
    const double sy = dot(s, y);
    if (sy > 1e-12 * std::sqrt(dot(s, s)) * std::sqrt(dot(y, y))) {
      pairs.push_back({s, y, 1.0 / sy});
      if (static_cast<int>(pairs.size()) > cfg.memory) pairs.pop_front();
    }
    r.x = xt;
    loss = ft;
    g = gt;
    r.loss = loss;
  }
  return r;
}

// ---- problem document (drivers.cpp:570-708) --------------------------------
enum class Design { Young, YoungRegions, V0, Orientation };
enum class Loss { Trajectory, FinalPose, TargetCom };

struct SceneDeleter {
  void operator()(hd_scene* s) const { hd_scene_free(s); }
};
struct SimDeleter {
  void operator()(hd_sim* s) const { hd_sim_free(s); }
};
using ScenePtr = std::unique_ptr<hd_scene, SceneDeleter>;
using SimPtr = std::unique_ptr<hd_sim, SimDeleter>;

struct Problem {
  ScenePtr scene;
  int nv = 0, ne = 0, frames = 0, region_count = 0;
  std::vector<int> region;
  V rest, mass;
  Design design = Design::Young;
  V initial;  // optimizer space (log-moduli for the Young designs)
  V truth;    // natural space; empty when absent
  Loss loss = Loss::Trajectory;
  double target[3] = {0, 0, 0};
  int loss_frame = 0;  // 1-based; 0 = last frame
  LbfgsConfig opt;
};

V number_or_array(const json& j, const std::string& field, std::vector<std::string>& errs) {
  if (j.is_number()) return V{j.get<double>()};
  if (j.is_array() && !j.empty()) {
    V v;
    for (const auto& e : j) {
      if (!e.is_number()) {
        errs.push_back(field + ": expected numbers");
        return V();
      }
      v.push_back(e.get<double>());
    }
    return v;
  }
  errs.push_back(field + ": expected a number or a non-empty numeric array");
  return V();
}

Problem parse_problem(const std::string& text) {
  json j;
  try {
    j = json::parse(text);
  } catch (const json::parse_error& e) {
    fail(HD_ERR_PARSE, std::string("problem JSON: ") + e.what());
  }
  Problem p;
  if (j.contains("scene_file") && j["scene_file"].is_string()) {
    p.scene.reset(hd_scene_load(j["scene_file"].get<std::string>().c_str()));
  } else if (j.contains("scene") && j["scene"].is_object()) {
    p.scene.reset(hd_scene_parse(j["scene"].dump().c_str()));
  } else {
    fail(HD_ERR_VALIDATION, "problem: expected \"scene\" object or \"scene_file\" path");
  }
  if (!p.scene) fail(hd_last_error_code(), hd_last_error());
  hd_scene* sc = p.scene.get();
  p.nv = hd_scene_vertex_count(sc);
  p.ne = hd_scene_element_count(sc);
  p.frames = hd_scene_frame_count(sc);
  p.region_count = hd_scene_region_count(sc);
  p.region.resize(p.ne);
  p.rest.resize(3 * static_cast<size_t>(p.nv));
  p.mass.resize(p.nv);
  check(hd_scene_regions(sc, p.region.data(), p.region.size()));
  check(hd_scene_rest_positions(sc, p.rest.data(), p.rest.size()));
  check(hd_scene_vertex_masses(sc, p.mass.data(), p.mass.size()));

  std::vector<std::string> errs;
  if (!j.contains("design") || !j["design"].is_object() || !j["design"].contains("variable")) {
    errs.push_back("design.variable: required");
  } else {
    const json& d = j["design"];
    const std::string var = d["variable"].is_string() ? d["variable"].get<std::string>() : std::string();
    V init;
    if (d.contains("initial")) init = number_or_array(d["initial"], "design.initial", errs);
    else errs.push_back("design.initial: required");
    const auto logs = [](const V& v) {
      V o(v.size());
      for (size_t i = 0; i < v.size(); ++i) o[i] = std::log(v[i]);
      return o;
    };
    if (var == "young") {
      p.design = Design::Young;
      if (init.size() == 1 && init[0] > 0) p.initial = logs(init);
      else if (!init.empty()) errs.push_back("design.initial: young expects one positive modulus");
    } else if (var == "young_regions") {
      p.design = Design::YoungRegions;
      bool positive = true;
      for (double v : init) positive = positive && v > 0;
      if (p.region_count < 1) errs.push_back("design.variable: scene has no element regions");
      else if (static_cast<int>(init.size()) != p.region_count)
        errs.push_back("design.initial: expected one modulus per region (" + std::to_string(p.region_count) + ")");
      else if (!positive) errs.push_back("design.initial: moduli must be positive");
      else p.initial = logs(init);
    } else if (var == "v0") {
      p.design = Design::V0;
      if (init.size() != 3) errs.push_back("design.initial: v0 expects a 3-vector");
      else p.initial = init;
    } else if (var == "orientation") {
      p.design = Design::Orientation;
      if (init.size() != 3) errs.push_back("design.initial: orientation expects 3 Euler angles");
      else p.initial = init;
    } else {
      errs.push_back("design.variable: expected young, young_regions, v0, or orientation");
    }
  }
  if (j.contains("true")) {
    p.truth = number_or_array(j["true"], "true", errs);
    if (!p.initial.empty() && !p.truth.empty() && p.truth.size() != p.initial.size() &&
        !(p.design == Design::Young && p.truth.size() == 1))
      errs.push_back("true: size must match design.initial");
  }
  std::string kind = "trajectory";
  if (j.contains("loss") && j["loss"].is_object()) {
    const json& l = j["loss"];
    if (l.contains("kind") && l["kind"].is_string()) kind = l["kind"].get<std::string>();
    if (l.contains("target")) {
      std::vector<std::string> ignored;
      const V t = number_or_array(l["target"], "loss.target", ignored);
      if (t.size() != 3) errs.push_back("loss.target: expected a 3-vector");
      else for (int k = 0; k < 3; ++k) p.target[k] = t[k];
    }
    if (l.contains("frame")) p.loss_frame = l["frame"].get<int>();
  }
  if (kind == "trajectory") p.loss = Loss::Trajectory;
  else if (kind == "final_pose") p.loss = Loss::FinalPose;
  else if (kind == "target_com") {
    p.loss = Loss::TargetCom;
    if (!j.contains("loss") || !j["loss"].contains("target")) errs.push_back("loss.target: required for target_com");
  } else {
    errs.push_back("loss.kind: expected trajectory, final_pose, or target_com");
  }
  if (p.loss != Loss::TargetCom && p.truth.empty())
    errs.push_back("true: required to synthesize the reference trajectory");
  if (p.loss_frame < 0 || p.loss_frame > p.frames) errs.push_back("loss.frame: out of range");
  if (p.loss_frame == 0) p.loss_frame = p.frames;
  if (j.contains("optimizer") && j["optimizer"].is_object()) {
    const json& o = j["optimizer"];
    p.opt.memory = o.value("memory", p.opt.memory);
    p.opt.max_evals = o.value("max_evals", p.opt.max_evals);
    p.opt.grad_tol = o.value("grad_tol", p.opt.grad_tol);
  }
  if (!errs.empty()) {
    std::string msg = "problem validation failed:";
    for (const auto& e : errs) msg += "\n  - " + e;
    fail(HD_ERR_VALIDATION, msg);
  }
  return p;
}

// ---- design variables (drivers.cpp:186-234, 710-803) ------------------------
using M3 = std::array<double, 9>;  // row-major
M3 mul(const M3& a, const M3& b) {
  M3 c{};
  for (int i = 0; i < 3; ++i)
    for (int j = 0; j < 3; ++j)
      for (int k = 0; k < 3; ++k) c[3 * i + j] += a[3 * i + k] * b[3 * k + j];
  return c;
}
// R = Rz(c) Ry(b) Rx(a) and its partials (drivers.cpp:176-224)
M3 rot(int axis, double t, bool deriv) {
  const double c = std::cos(t), s = std::sin(t);
  if (axis == 0) return deriv ? M3{0, 0, 0, 0, -s, -c, 0, c, -s} : M3{1, 0, 0, 0, c, -s, 0, s, c};
  if (axis == 1) return deriv ? M3{-s, 0, c, 0, 0, 0, -c, 0, -s} : M3{c, 0, s, 0, 1, 0, -s, 0, c};
  return deriv ? M3{-s, -c, 0, c, -s, 0, 0, 0, 0} : M3{c, -s, 0, s, c, 0, 0, 0, 1};
}
M3 euler(const V& a, int deriv_axis) {
  return mul(rot(2, a[2], deriv_axis == 2), mul(rot(1, a[1], deriv_axis == 1), rot(0, a[0], deriv_axis == 0)));
}
std::array<double, 3> mass_center(const Problem& p, const double* q) {
  std::array<double, 3> c{0, 0, 0};
  double total = 0;
  for (int v = 0; v < p.nv; ++v) {
    for (int k = 0; k < 3; ++k) c[k] += p.mass[v] * q[3 * v + k];
    total += p.mass[v];
  }
  for (double& x : c) x /= total;
  return c;
}

struct DesignState {
  V q0, v0, young;
  bool material = false;
};

DesignState apply_design(const Problem& p, const V& q0, const V& v0, const V& x) {
  DesignState s{q0, v0, {}, false};
  switch (p.design) {
    case Design::Young:
      s.young.assign(p.ne, std::exp(x[0]));
      s.material = true;
      break;
    case Design::YoungRegions:
      s.young.resize(p.ne);
      for (int e = 0; e < p.ne; ++e) s.young[e] = std::exp(x[p.region[e]]);
      s.material = true;
      break;
    case Design::V0:
      for (int v = 0; v < p.nv; ++v)
        for (int k = 0; k < 3; ++k) s.v0[3 * v + k] = x[k];
      break;
    case Design::Orientation: {
      const M3 r = euler(x, -1);
      const auto com = mass_center(p, p.rest.data());
      for (int v = 0; v < p.nv; ++v) {
        const double d[3] = {p.rest[3 * v] - com[0], p.rest[3 * v + 1] - com[1], p.rest[3 * v + 2] - com[2]};
        for (int i = 0; i < 3; ++i) s.q0[3 * v + i] = com[i] + r[3 * i] * d[0] + r[3 * i + 1] * d[1] + r[3 * i + 2] * d[2];
      }
      break;
    }
  }
  return s;
}

struct Grads {
  V dq0, dv0, de;
};

V design_gradient(const Problem& p, const V& x, const Grads& g) {
  V out(x.size(), 0.0);
  switch (p.design) {
    case Design::Young: {
      double s = 0;
      for (double v : g.de) s += v;
      out[0] = s * std::exp(x[0]);
      break;
    }
    case Design::YoungRegions:
      for (int e = 0; e < p.ne; ++e) out[p.region[e]] += g.de[e] * std::exp(x[p.region[e]]);
      break;
    case Design::V0:
      for (int v = 0; v < p.nv; ++v)
        for (int k = 0; k < 3; ++k) out[k] += g.dv0[3 * v + k];
      break;
    case Design::Orientation: {
      const auto com = mass_center(p, p.rest.data());
      for (int axis = 0; axis < 3; ++axis) {
        const M3 dr = euler(x, axis);
        double acc = 0;
        for (int v = 0; v < p.nv; ++v) {
          const double d[3] = {p.rest[3 * v] - com[0], p.rest[3 * v + 1] - com[1], p.rest[3 * v + 2] - com[2]};
          for (int i = 0; i < 3; ++i)
            acc += g.dq0[3 * v + i] * (dr[3 * i] * d[0] + dr[3 * i + 1] * d[1] + dr[3 * i + 2] * d[2]);
        }
        out[axis] = acc;
      }
      break;
    }
  }
  return out;
}

const char* design_name(Design d) {
  switch (d) {
    case Design::Young: return "young";
    case Design::YoungRegions: return "young_regions";
    case Design::V0: return "v0";
    default: return "orientation";
  }
}

// Rolls the scene's frames from (q0, v0) at time 0 (drivers.cpp:31-54); the
// state after frame t goes to traj[t] when traj is given.
void roll(hd_sim* sim, const DesignState& ds, int frames, bool record, std::vector<V>* traj, V* final_q) {
  const size_t dof = ds.q0.size();
  check(hd_sim_set_state(sim, ds.q0.data(), ds.v0.data(), 0.0));
  check(hd_sim_record(sim, 0));
  if (record) check(hd_sim_record(sim, 1));
  if (traj) traj->assign(frames, V(dof));
  for (int t = 0; t < frames; ++t) {
    check(hd_sim_step(sim));
    if (traj) check(hd_sim_positions(sim, (*traj)[t].data(), dof));
  }
  if (final_q) {
    final_q->resize(dof);
    check(hd_sim_positions(sim, final_q->data(), dof));
  }
}

std::string result_json(const Problem& p, const LbfgsResult& opt, long long factorizations,
                        long long material_updates) {
  json r;
  r["variable"] = design_name(p.design);
  V rec = opt.x;
  if (p.design == Design::Young || p.design == Design::YoungRegions)
    for (double& v : rec) v = std::exp(v);
  r["recovered"] = rec;
  if (!p.truth.empty()) {
    r["true"] = p.truth;
    if (p.truth.size() == rec.size()) {
      V rel;
      for (size_t i = 0; i < rec.size(); ++i)
        rel.push_back(std::abs(rec[i] - p.truth[i]) / std::max(std::abs(p.truth[i]), 1e-30));
      r["rel_errors"] = rel;
    }
    r["reference"] = "synthetic (inverse crime)";
  }
  r["loss"] = opt.loss;
  r["evaluations"] = opt.evaluations;
  r["factorizations"] = factorizations;
  r["material_updates"] = material_updates;
  r["converged"] = opt.converged;
  r["stalled"] = opt.stalled;
  return r.dump(2);
}

std::string identify(const std::string& text, const std::string& out_dir, bool* stalled) {
  const Problem p = parse_problem(text);
  hd_scene* sc = p.scene.get();
  const size_t dof = 3 * static_cast<size_t>(p.nv);

  SimPtr sim(hd_sim_create(sc));
  if (!sim) fail(hd_last_error_code(), hd_last_error());
  V q0(dof), v0(dof);  // the scene's initial state
  check(hd_sim_positions(sim.get(), q0.data(), dof));
  check(hd_sim_velocities(sim.get(), v0.data(), dof));

  // Reference trajectory from the true parameters on its own sim
  // (drivers.cpp:822-834).
  std::vector<V> ref;
  if (!p.truth.empty()) {
    V xt = p.truth;
    if (p.design == Design::Young || p.design == Design::YoungRegions)
      for (double& v : xt) v = std::log(v);
    const DesignState ds = apply_design(p, q0, v0, xt);
    SimPtr rs(hd_sim_create(sc));
    if (!rs) fail(hd_last_error_code(), hd_last_error());
    if (ds.material) check(hd_sim_set_young(rs.get(), ds.young.data(), ds.young.size(), 0));
    roll(rs.get(), ds, p.frames, false, &ref, nullptr);
  }

  const long long refactor_base = hd_sim_refactor_count(sim.get());
  long long material_updates = 0;
  std::vector<std::pair<double, double>> log;  // (loss, best so far)
  const bool need_traj = p.loss == Loss::Trajectory || (p.loss == Loss::TargetCom && p.loss_frame != p.frames);

  auto evaluate = [&](const V& x, V& grad) -> double {  // drivers.cpp:848-920
    const DesignState ds = apply_design(p, q0, v0, x);
    if (ds.material) check(hd_sim_set_young(sim.get(), ds.young.data(), ds.young.size(), 0));
    if (ds.material || material_updates == 0) ++material_updates;
    std::vector<V> traj;
    V qf;
    roll(sim.get(), ds, p.frames, true, need_traj ? &traj : nullptr, &qf);
    double loss = 0;
    V direct((static_cast<size_t>(p.frames) + 1) * dof, 0.0);
    switch (p.loss) {
      case Loss::Trajectory:
        for (int t = 0; t < p.frames; ++t) {
          double* d = direct.data() + (t + 1) * dof;
          for (size_t k = 0; k < dof; ++k) {
            d[k] = traj[t][k] - ref[t][k];
            loss += 0.5 * d[k] * d[k];
          }
        }
        break;
      case Loss::FinalPose: {
        double* d = direct.data() + p.frames * dof;
        for (size_t k = 0; k < dof; ++k) {
          d[k] = qf[k] - ref.back()[k];
          loss += 0.5 * d[k] * d[k];
        }
        break;
      }
      case Loss::TargetCom: {
        const V& qt = p.loss_frame == p.frames ? qf : traj[p.loss_frame - 1];
        const auto com = mass_center(p, qt.data());
        double diff[3], total = 0;
        for (int k = 0; k < 3; ++k) {
          diff[k] = com[k] - p.target[k];
          loss += 0.5 * diff[k] * diff[k];
        }
        for (int v = 0; v < p.nv; ++v) total += p.mass[v];
        double* d = direct.data() + p.loss_frame * dof;
        for (int v = 0; v < p.nv; ++v)
          for (int k = 0; k < 3; ++k) d[3 * v + k] = (p.mass[v] / total) * diff[k];
        break;
      }
    }
    Grads g{V(dof), V(dof), V(p.ne)};
    check(hd_sim_backward(sim.get(), direct.data(), nullptr, nullptr, g.dq0.data(), g.dv0.data(), nullptr,
                          g.de.data(), nullptr, 0));
    grad = design_gradient(p, x, g);
    log.push_back({loss, log.empty() ? loss : std::min(loss, log.back().second)});
    return loss;
  };
  // An unsimulatable probe reports an infinite loss so the line search backs
  // off (drivers.cpp:924-936).
  auto objective = [&](const V& x, V& grad) -> double {
    try {
      return evaluate(x, grad);
    } catch (const Failure&) {
      grad.assign(x.size(), 0.0);
      const double inf = std::numeric_limits<double>::infinity();
      log.push_back({inf, log.empty() ? inf : log.back().second});
      return inf;
    }
  };
  const LbfgsResult opt = lbfgs(objective, p.initial, p.opt);
  // The factor built at sim creation serves the first evaluation when the
  // design leaves the material alone (the reference counts that build).
  const bool material_design = p.design == Design::Young || p.design == Design::YoungRegions;
  const long long factorizations = hd_sim_refactor_count(sim.get()) - refactor_base + (material_design ? 0 : 1);
  const std::string out = result_json(p, opt, factorizations, material_updates);
  if (!out_dir.empty()) {  // stdio, not iostreams: the library may carry its own libstdc++
    FILE* curve = std::fopen((out_dir + "/loss_curve.csv").c_str(), "w");
    FILE* res = std::fopen((out_dir + "/result.json").c_str(), "w");
    const bool ok = curve && res;
    if (ok) {
      std::fprintf(curve, "evaluation,loss,best_so_far\n");
      for (size_t i = 0; i < log.size(); ++i)
        std::fprintf(curve, "%zu,%.17g,%.17g\n", i + 1, log[i].first, log[i].second);
      std::fprintf(res, "%s\n", out.c_str());
    }
    if (curve) std::fclose(curve);
    if (res) std::fclose(res);
    if (!ok) fail(HD_ERR_IO, "cannot write to output directory: " + out_dir);
  }
  if (stalled) *stalled = opt.stalled;
  return out;
}

}  // namespace

int run_identify(const std::string& problem_text, const std::string& out_dir, std::string* result, bool* stalled,
                 std::string* error) {
  try {
    if (!out_dir.empty()) {  // create_directories (drivers.cpp:955)
      for (size_t pos = out_dir.find('/', 1); pos != std::string::npos; pos = out_dir.find('/', pos + 1))
        ::mkdir(out_dir.substr(0, pos).c_str(), 0755);
      ::mkdir(out_dir.c_str(), 0755);
    }
    *result = identify(problem_text, out_dir, stalled);
    return HD_OK;
  } catch (const Failure& f) {
    *error = f.msg;
    return f.code;
  } catch (const std::exception& e) {
    *error = e.what();
    return HD_ERR_INVALID_ARGUMENT;
  }
}

int run_identify_file(const std::string& path, const std::string& out_dir, std::string* result, bool* stalled,
                      std::string* error) {
  FILE* f = std::fopen(path.c_str(), "rb");
  if (!f) {
    *error = "cannot open problem file: " + path;
    return HD_ERR_IO;
  }
  std::string text;
  char buf[65536];
  for (size_t n; (n = std::fread(buf, 1, sizeof buf, f)) > 0;) text.append(buf, n);
  std::fclose(f);
  return run_identify(text, out_dir, result, stalled, error);
}

namespace {

// ---- gradient check (drivers.cpp:367-531) ----------------------------------
// sample_indices (drivers.cpp:174-181): at most `cap` evenly spaced indices
std::vector<int> sample_indices(int n, int cap) {
  const int m = std::min(n, cap);
  std::vector<int> idx(m);
  for (int k = 0; k < m; ++k) idx[k] = static_cast<int>((static_cast<long long>(k) * n) / m);
  return idx;
}

double norm(const V& a) { return std::sqrt(dot(a, a)); }

std::vector<std::string> split_csv(const char* csv) {  // capi.cpp:74-90
  std::vector<std::string> out;
  if (!csv) return out;
  const std::string text(csv);
  for (size_t start = 0; start <= text.size();) {
    size_t comma = text.find(',', start);
    if (comma == std::string::npos) comma = text.size();
    const std::string item = text.substr(start, comma - start);
    const size_t a = item.find_first_not_of(" \t"), b = item.find_last_not_of(" \t");
    if (a != std::string::npos) out.push_back(item.substr(a, b - a + 1));
    start = comma + 1;
  }
  return out;
}

std::string gradcheck(const hd_scene* sc, std::vector<std::string> vars, const std::string& out_path, bool* pass) {
  if (vars.empty()) vars = {"q0", "v0", "f_ext", "E"};  // capi.cpp:269
  for (const auto& v : vars)
    if (v != "q0" && v != "v0" && v != "f_ext" && v != "E" && v != "w")
      fail(HD_ERR_INVALID_ARGUMENT, "gradcheck: unknown variable \"" + v + "\" (expected q0, v0, f_ext, E, w)");
  const int nv = hd_scene_vertex_count(sc), ne = hd_scene_element_count(sc), frames = hd_scene_frame_count(sc);
  const size_t n = 3 * static_cast<size_t>(nv);
  SimPtr sim(hd_sim_create(sc));
  if (!sim) fail(hd_last_error_code(), hd_last_error());
  hd_sim* s = sim.get();
  V q0(n), v0(n), f0(n), rest(n), young(ne);
  check(hd_sim_positions(s, q0.data(), n));
  check(hd_sim_velocities(s, v0.data(), n));
  check(hd_sim_external_force(s, f0.data(), n));
  check(hd_scene_rest_positions(sc, rest.data(), n));
  check(hd_scene_young_moduli(sc, young.data(), young.size()));
  // FD convention: the mesh-wide prox means stay at the scene's values while
  // single moduli move (drivers.cpp:384-387)
  check(hd_sim_set_young(s, young.data(), young.size(), 1));

  // L = 1/2 |q_T - rest|^2 + 1/2 |v_T|^2 of a rollout (drivers.cpp:400-406)
  V qf(n), vf(n);
  std::vector<int> iterations;
  const auto rollout = [&](const V& q, const V& v, const V& f, bool record) {
    check(hd_sim_set_external_force(s, f.data(), n));
    check(hd_sim_set_state(s, q.data(), v.data(), 0.0));
    check(hd_sim_record(s, 0));
    if (record) check(hd_sim_record(s, 1));
    for (int t = 0; t < frames; ++t) {
      check(hd_sim_step(s));
      if (record) iterations.push_back(hd_sim_last_iterations(s));
    }
    check(hd_sim_positions(s, qf.data(), n));
    check(hd_sim_velocities(s, vf.data(), n));
    double l = 0;
    for (size_t k = 0; k < n; ++k) l += 0.5 * (qf[k] - rest[k]) * (qf[k] - rest[k]) + 0.5 * vf[k] * vf[k];
    return l;
  };
  const auto loss_of = [&](const V& q, const V& v, const V& f) { return rollout(q, v, f, false); };

  // analytic pass: recorded rollout + chained adjoint (drivers.cpp:408-415)
  rollout(q0, v0, f0, true);
  V seed_q(n);
  for (size_t k = 0; k < n; ++k) seed_q[k] = qf[k] - rest[k];
  V g_q0(n), g_v0(n), g_f(n), g_e(ne), g_w(2 * static_cast<size_t>(ne), 0.0);
  check(hd_sim_backward(s, nullptr, seed_q.data(), vf.data(), g_q0.data(), g_v0.data(), g_f.data(), g_e.data(),
                        g_w.data(), g_w.size()));
  V tau(frames), rho(frames);
  check(hd_sim_backward_tau(s, tau.data(), rho.data(), frames));

  json grad_norms = json::object(), per_var = json::object();
  double max_rel = 0;
  std::string worst_param;
  const auto check_var = [&](const std::string& var, const V& analytic, int count, auto&& eval_at) {
    grad_norms[var] = norm(analytic);
    double scale = 0;
    for (double a : analytic) scale = std::max(scale, std::abs(a));
    scale = std::max(scale, 1e-30);
    double worst = 0;
    int worst_i = -1;
    for (int i : sample_indices(count, 24)) {
      const auto [fd, g] = eval_at(i, analytic);
      const double denom = std::max({std::abs(fd), std::abs(g), 1e-4 * scale, 1e-12});
      const double rel = std::abs(fd - g) / denom;
      if (rel > worst) {
        worst = rel;
        worst_i = i;
      }
    }
    per_var[var] = worst;
    if (worst > max_rel) {
      max_rel = worst;
      worst_param = var + "[" + std::to_string(worst_i) + "]";
    }
  };
  for (const auto& var : vars) {
    if (var == "q0" || var == "v0" || var == "f_ext") {
      const V& analytic = var == "q0" ? g_q0 : var == "v0" ? g_v0 : g_f;
      const V& center = var == "q0" ? q0 : var == "v0" ? v0 : f0;
      double cscale = 0;  // step floor tied to the variable's magnitude (drivers.cpp:462-466)
      for (double c : center) cscale = std::max(cscale, std::abs(c));
      check_var(var, analytic, static_cast<int>(n), [&](int i, const V& g) {
        const double step = std::max({1e-6 * std::abs(center[i]), 1e-4 * cscale, 1e-7});
        V plus = center, minus = center;
        plus[i] += step;
        minus[i] -= step;
        double lp, lm;
        if (var == "q0") {
          lp = loss_of(plus, v0, f0);
          lm = loss_of(minus, v0, f0);
        } else if (var == "v0") {
          lp = loss_of(q0, plus, f0);
          lm = loss_of(q0, minus, f0);
        } else {
          lp = loss_of(q0, v0, plus);
          lm = loss_of(q0, v0, minus);
        }
        return std::pair<double, double>{(lp - lm) / (2 * step), g[i]};
      });
    } else if (var == "E") {
      check_var("E", g_e, ne, [&](int e, const V& g) {
        const double step = 1e-4 * young[e];
        V y = young;
        y[e] = young[e] + step;
        check(hd_sim_set_young(s, y.data(), y.size(), 1));
        const double lp = loss_of(q0, v0, f0);
        y[e] = young[e] - step;
        check(hd_sim_set_young(s, y.data(), y.size(), 1));
        const double lm = loss_of(q0, v0, f0);
        check(hd_sim_set_young(s, young.data(), young.size(), 1));
        return std::pair<double, double>{(lp - lm) / (2 * step), g[e]};
      });
    } else {  // "w": norm only (the weights are linear images of the moduli)
      grad_norms["w"] = norm(g_w);
    }
  }
  json j;  // report_to_json (drivers.cpp:517-531)
  j["vars"] = vars;
  j["tau"] = tau;
  j["rho"] = rho;
  j["iterations"] = iterations;
  j["grad_norms"] = grad_norms;
  json fd;
  fd["max_rel_err"] = max_rel;
  fd["worst_param"] = worst_param;
  fd["per_var_max_rel_err"] = per_var;
  j["fd_check"] = fd;
  j["pass"] = max_rel <= 2e-3;
  *pass = max_rel <= 2e-3;
  const std::string out = j.dump(2);
  if (!out_path.empty()) {
    const size_t slash = out_path.rfind('/');
    if (slash != std::string::npos && slash > 0) {  // create the parent directories
      const std::string dir = out_path.substr(0, slash);
      for (size_t pos = dir.find('/', 1); pos != std::string::npos; pos = dir.find('/', pos + 1))
        ::mkdir(dir.substr(0, pos).c_str(), 0755);
      ::mkdir(dir.c_str(), 0755);
    }
    FILE* f = std::fopen(out_path.c_str(), "w");
    if (!f) fail(HD_ERR_IO, "cannot open output file: " + out_path);
    std::fprintf(f, "%s\n", out.c_str());
    std::fclose(f);
  }
  return out;
}

}  // namespace

int run_gradcheck(const hd_scene* scene, const char* vars_csv, const char* out_path, std::string* report,
                  bool* pass, std::string* error) {
  try {
    *report = gradcheck(scene, split_csv(vars_csv), out_path ? out_path : "", pass);
    return HD_OK;
  } catch (const Failure& f) {
    *error = f.msg;
    return f.code;
  } catch (const std::exception& e) {
    *error = e.what();
    return HD_ERR_INVALID_ARGUMENT;
  }
}

namespace {

// ---- simulate (drivers.cpp:238-365) -----------------------------------------
// Worst vertex distance to the group's best rigid fit from rest (Kabsch,
// drivers.cpp:115-145): one-sided Jacobi SVD of the 3x3 cross-covariance.
double rigid_fit_residual(const std::vector<int>& verts, const V& rest, const V& q) {
  if (verts.empty()) return 0.0;
  double rc[3] = {0, 0, 0}, qc[3] = {0, 0, 0};
  for (int v : verts)
    for (int k = 0; k < 3; ++k) {
      rc[k] += rest[3 * v + k];
      qc[k] += q[3 * v + k];
    }
  for (int k = 0; k < 3; ++k) {
    rc[k] /= verts.size();
    qc[k] /= verts.size();
  }
  double a[3][3] = {}, vm[3][3] = {{1, 0, 0}, {0, 1, 0}, {0, 0, 1}};  // a = H = sum (r - rc)(q - qc)^T
  for (int v : verts)
    for (int i = 0; i < 3; ++i)
      for (int j = 0; j < 3; ++j) a[i][j] += (rest[3 * v + i] - rc[i]) * (q[3 * v + j] - qc[j]);
  for (int sweep = 0; sweep < 60; ++sweep) {  // rotate column pairs of a until orthogonal: a = U S, H = U S V^T
    double off = 0;
    for (int p = 0; p < 2; ++p)
      for (int r = p + 1; r < 3; ++r) {
        double al = 0, be = 0, ga = 0;
        for (int i = 0; i < 3; ++i) {
          al += a[i][p] * a[i][p];
          be += a[i][r] * a[i][r];
          ga += a[i][p] * a[i][r];
        }
        if (std::abs(ga) <= 1e-15 * std::sqrt(al * be) || ga == 0.0) continue;
        off = std::max(off, std::abs(ga) / std::sqrt(al * be));
        const double z = (be - al) / (2 * ga);
        const double t = (z >= 0 ? 1.0 : -1.0) / (std::abs(z) + std::sqrt(1 + z * z));
        const double c = 1 / std::sqrt(1 + t * t), s = c * t;
        for (int i = 0; i < 3; ++i) {
          const double x = a[i][p], y = a[i][r];
          a[i][p] = c * x - s * y;
          a[i][r] = s * x + c * y;
          const double vx = vm[i][p], vy = vm[i][r];
          vm[i][p] = c * vx - s * vy;
          vm[i][r] = s * vx + c * vy;
        }
      }
    if (off <= 1e-15) break;
  }
  double sig[3];
  int ord[3] = {0, 1, 2};
  for (int k = 0; k < 3; ++k) sig[k] = std::sqrt(a[0][k] * a[0][k] + a[1][k] * a[1][k] + a[2][k] * a[2][k]);
  std::sort(ord, ord + 3, [&](int x, int y) { return sig[x] > sig[y]; });
  double u[3][3], w[3][3];  // sorted U, V columns
  for (int k = 0; k < 3; ++k)
    for (int i = 0; i < 3; ++i) {
      u[i][k] = sig[ord[k]] > 0 ? a[i][ord[k]] / sig[ord[k]] : 0.0;
      w[i][k] = vm[i][ord[k]];
    }
  const double tiny = 1e-12 * std::max(sig[ord[0]], 1e-300);
  if (sig[ord[1]] <= tiny) {  // rank <= 1: complete U from its first column (or e_x)
    double u0[3] = {u[0][0], u[1][0], u[2][0]};
    if (sig[ord[0]] <= 0) u0[0] = 1, u0[1] = 0, u0[2] = 0;
    const double e[3] = {std::abs(u0[0]) < 0.9 ? 1.0 : 0.0, std::abs(u0[0]) < 0.9 ? 0.0 : 1.0, 0.0};
    const double c1[3] = {u0[1] * e[2] - u0[2] * e[1], u0[2] * e[0] - u0[0] * e[2], u0[0] * e[1] - u0[1] * e[0]};
    const double nn = std::sqrt(c1[0] * c1[0] + c1[1] * c1[1] + c1[2] * c1[2]);
    for (int i = 0; i < 3; ++i) {
      u[i][0] = u0[i];
      u[i][1] = c1[i] / nn;
    }
  }
  if (sig[ord[2]] <= tiny) {  // rank <= 2: third column of U = first x second
    u[0][2] = u[1][0] * u[2][1] - u[2][0] * u[1][1];
    u[1][2] = u[2][0] * u[0][1] - u[0][0] * u[2][1];
    u[2][2] = u[0][0] * u[1][1] - u[1][0] * u[0][1];
  }
  double rot[3][3];  // V U^T, reflected on the smallest singular direction if det < 0
  const auto build = [&](double sgn) {
    for (int i = 0; i < 3; ++i)
      for (int j = 0; j < 3; ++j) rot[i][j] = w[i][0] * u[j][0] + w[i][1] * u[j][1] + sgn * w[i][2] * u[j][2];
  };
  build(1.0);
  const double det = rot[0][0] * (rot[1][1] * rot[2][2] - rot[1][2] * rot[2][1]) -
                     rot[0][1] * (rot[1][0] * rot[2][2] - rot[1][2] * rot[2][0]) +
                     rot[0][2] * (rot[1][0] * rot[2][1] - rot[1][1] * rot[2][0]);
  if (det < 0) build(-1.0);
  double worst = 0;
  for (int v : verts) {
    const double d[3] = {rest[3 * v] - rc[0], rest[3 * v + 1] - rc[1], rest[3 * v + 2] - rc[2]};
    double e2 = 0;
    for (int i = 0; i < 3; ++i) {
      const double fit = rot[i][0] * d[0] + rot[i][1] * d[1] + rot[i][2] * d[2] + qc[i];
      e2 += (q[3 * v + i] - fit) * (q[3 * v + i] - fit);
    }
    worst = std::max(worst, std::sqrt(e2));
  }
  return worst;
}

std::string simulate(const hd_scene* sc, const std::string& out_dir) {
  const int nv = hd_scene_vertex_count(sc), ne = hd_scene_element_count(sc), frames = hd_scene_frame_count(sc);
  const int nreg = hd_scene_region_count(sc);
  const size_t n = 3 * static_cast<size_t>(nv);
  V rest(n), young(ne);
  std::vector<int> region(ne), el(4 * static_cast<size_t>(ne));
  check(hd_scene_rest_positions(sc, rest.data(), n));
  check(hd_scene_young_moduli(sc, young.data(), young.size()));
  check(hd_scene_regions(sc, region.data(), region.size()));
  check(hd_scene_elements(sc, el.data(), el.size()));
  // region deformation tracking: softest and stiffest regions by mean modulus
  std::vector<std::vector<int>> rverts;
  std::vector<char> soft, stiff;
  bool track = false;
  if (nreg >= 2) {
    V mean(nreg, 0.0);
    std::vector<int> count(nreg, 0);
    rverts.assign(nreg, {});
    std::vector<std::vector<char>> seen(nreg, std::vector<char>(nv, 0));
    for (int e = 0; e < ne; ++e) {
      const int r = region[e];
      mean[r] += young[e];
      ++count[r];
      for (int k = 0; k < 4; ++k) {
        const int v = el[4 * e + k];
        if (!seen[r][v]) {
          seen[r][v] = 1;
          rverts[r].push_back(v);
        }
      }
    }
    for (int r = 0; r < nreg; ++r)
      if (count[r] > 0) mean[r] /= count[r];
    const double lo = *std::min_element(mean.begin(), mean.end()), hi = *std::max_element(mean.begin(), mean.end());
    soft.assign(nreg, 0);
    stiff.assign(nreg, 0);
    for (int r = 0; r < nreg; ++r) {
      if (count[r] == 0) continue;
      if (mean[r] <= lo * (1 + 1e-9)) soft[r] = 1;
      if (mean[r] >= hi * (1 - 1e-9)) stiff[r] = 1;
    }
    track = hi > lo * (1 + 1e-9);
  }
  SimPtr sim(hd_sim_create(sc));
  if (!sim) fail(hd_last_error_code(), hd_last_error());
  hd_sim* s = sim.get();
  FILE* traj = nullptr;
  FILE* metrics = nullptr;
  const bool emit = !out_dir.empty();
  struct Closer {
    FILE*& f;
    ~Closer() {
      if (f) std::fclose(f);
    }
  } c1{traj}, c2{metrics};
  if (emit) {
    for (size_t pos = out_dir.find('/', 1); pos != std::string::npos; pos = out_dir.find('/', pos + 1))
      ::mkdir(out_dir.substr(0, pos).c_str(), 0755);
    ::mkdir(out_dir.c_str(), 0755);
    traj = std::fopen((out_dir + "/trajectory.jsonl").c_str(), "w");
    metrics = std::fopen((out_dir + "/metrics.csv").c_str(), "w");
    if (!traj || !metrics) fail(HD_ERR_IO, "cannot open output file in: " + out_dir);
    std::fprintf(metrics, "frame,time,iterations,converged,contact_count,max_fb_residual,max_penetration\n");
  }
  std::vector<int> iterations;
  bool all = true;
  double max_pen = 0, soft_d = 0, stiff_d = 0;
  V q(n), v(n);
  for (int t = 0; t < frames; ++t) {
    check(hd_sim_step(s));
    const int it = hd_sim_last_iterations(s);
    const bool conv = hd_sim_last_converged(s) != 0;
    iterations.push_back(it);
    all = all && conv;
    const double pen = hd_sim_penetration(s);
    max_pen = std::max(max_pen, pen);
    if (track || emit) check(hd_sim_positions(s, q.data(), n));
    if (track)
      for (int r = 0; r < nreg; ++r) {
        if (!soft[r] && !stiff[r]) continue;
        const double d = rigid_fit_residual(rverts[r], rest, q);
        if (soft[r]) soft_d = std::max(soft_d, d);
        if (stiff[r]) stiff_d = std::max(stiff_d, d);
      }
    if (emit) {
      check(hd_sim_velocities(s, v.data(), n));
      json rec;
      rec["time"] = hd_sim_time(s);
      rec["q"] = q;
      rec["v"] = v;
      rec["iterations"] = it;
      rec["converged"] = conv;
      rec["contact_count"] = hd_sim_last_contact_count(s);
      std::fprintf(traj, "%s\n", rec.dump().c_str());
      std::fprintf(metrics, "%d,%g,%d,%d,%d,%g,%g\n", t + 1, hd_sim_time(s), it, conv ? 1 : 0,
                   hd_sim_last_contact_count(s), hd_sim_last_fb_residual(s), pen);
    }
  }
  json sum;  // summary_to_json (drivers.cpp:352-365)
  sum["frames"] = frames;
  sum["iterations"] = iterations;
  sum["refactorizations"] = hd_sim_refactor_count(s);
  sum["all_converged"] = all;
  sum["max_penetration"] = max_pen;
  if (track && stiff_d > 0) sum["displacement_ratio"] = soft_d / stiff_d;
  const std::string out = sum.dump(2);
  if (emit) {
    FILE* f = std::fopen((out_dir + "/summary.json").c_str(), "w");
    if (!f) fail(HD_ERR_IO, "cannot open output file: " + out_dir + "/summary.json");
    std::fprintf(f, "%s\n", out.c_str());
    std::fclose(f);
  }
  return out;
}

}  // namespace

int run_simulate(const hd_scene* scene, const char* out_dir, std::string* summary, std::string* error) {
  try {
    *summary = simulate(scene, out_dir ? out_dir : "");
    return HD_OK;
  } catch (const Failure& f) {
    *error = f.msg;
    return f.code;
  } catch (const std::exception& e) {
    *error = e.what();
    return HD_ERR_INVALID_ARGUMENT;
  }
}

}  // namespace heterodyn_driver
