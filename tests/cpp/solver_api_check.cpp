// C++ solver API checks (include/heterodyn/solver.hpp), written the way the
// reference's own doctest cases call forward_step / backward_step
// (/root/reference/proj/tests/test_forward.cpp, test_backward.cpp,
// test_material.cpp, test_mesh.cpp, drivers.cpp:31-99 roll / chain_backward).
// Built with the reference's include names (-I include/heterodyn/compat).
//
//   solver_api_check host               mesh / material known answers (no GPU)
//   solver_api_check device             step-level properties on the device engine
//   solver_api_check roll <scene.json>  roll + chained backward_step, results as JSON
//                                       (tests/test_cpp_api.py compares them with the oracle)
#include <algorithm>
#include <cmath>
#include <cstdio>
#include <fstream>
#include <sstream>
#include <string>
#include <vector>

#include "backward.hpp"
#include "forward.hpp"
#include "scene.hpp"

using namespace heterodyn;

static int g_fail = 0, g_checks = 0;
#define CHECK(c)                                                              \
  do {                                                                        \
    ++g_checks;                                                               \
    if (!(c)) {                                                               \
      ++g_fail;                                                               \
      std::fprintf(stderr, "%s:%d: CHECK failed: %s\n", __FILE__, __LINE__, #c); \
    }                                                                         \
  } while (0)

static bool close(double a, double b, double rel) { return std::fabs(a - b) <= rel * std::max(1.0, std::fabs(b)); }

// ---- host known answers ------------------------------------------------------------------------

static void host_checks() {
  // test_material.cpp:13-14
  const Lame l = lame_from_young_poisson(1e6, 0.4);
  CHECK(close(l.mu, 357142.85714285716, 1e-13));
  CHECK(close(l.lambda, 1428571.4285714286, 1e-13));
  bool threw = false;
  try {
    lame_from_young_poisson(1e6, 0.5);
  } catch (const Error& e) {
    threw = e.code() == ErrorCode::InvalidPoisson;
  }
  CHECK(threw);
  // unit tetrahedron: rest volume 1/6, quarter-volume lumped masses
  MatX rest(4, 3);
  rest << 0, 0, 0, 1, 0, 0, 0, 1, 0, 0, 0, 1;
  const TetMesh tet = build_tet_mesh(rest, {{0, 1, 2, 3}}, 1000.0);
  CHECK(tet.vertex_count() == 4 && tet.element_count() == 1 && tet.dof_count() == 12);
  CHECK(close(tet.volume(0), 1.0 / 6.0, 1e-15));
  CHECK(close(tet.vertex_mass(2), 1000.0 / 24.0, 1e-14));
  CHECK(tet.boundary_vertices().size() == 4);
  // F at rest is the identity; a stretched configuration is recovered exactly
  VecX q = tet.rest_vector();
  Mat3 f = deformation_gradient(tet, 0, q);
  CHECK(std::fabs(f(0, 0) - 1) < 1e-15 && std::fabs(f(1, 0)) < 1e-15 && std::fabs(f.determinant() - 1) < 1e-15);
  q[3] = 2.0;  // vertex 1 moves to x = 2
  f = deformation_gradient(tet, 0, q);
  CHECK(std::fabs(f(0, 0) - 2.0) < 1e-15);
  // an inverted tetrahedron is rejected (mesh.cpp: DegenerateElement)
  threw = false;
  try {
    build_tet_mesh(rest, {{0, 2, 1, 3}}, 1000.0);
  } catch (const Error& e) {
    threw = e.code() == ErrorCode::DegenerateElement;
  }
  CHECK(threw);
  // hex grid: 6 tets per cell, (n+1)^3 vertices, total volume = box volume
  const TetMesh grid = ingest_hex_grid({2, 2, 2}, 0.1, 1000.0);
  CHECK(grid.element_count() == 48 && grid.vertex_count() == 27);
  CHECK(close(grid.total_volume(), 0.008, 1e-14));
  // test_material.cpp:108-113: volume-weighted prox means; set_young bumps the
  // version and refreshes the means unless frozen
  MaterialField m = build_material(grid, std::vector<Scalar>(48, 2e5), 0.25, EnergyKind::NeoHookean, false, 0.0, 0.0);
  const std::uint64_t v0 = m.version();
  CHECK(close(m.prox_means().mu, lame_from_young_poisson(2e5, 0.25).mu, 1e-14));
  m.set_young(std::vector<Scalar>(48, 4e5));
  CHECK(m.version() != v0);
  CHECK(close(m.prox_means().mu, lame_from_young_poisson(4e5, 0.25).mu, 1e-14));
  const ProxMeans frozen = m.prox_means();
  m.freeze_means(frozen);
  m.set_young(std::vector<Scalar>(48, 8e5));
  CHECK(m.means_frozen() && m.prox_means().mu == frozen.mu);
  CHECK(close(m.mu(0), lame_from_young_poisson(8e5, 0.25).mu, 1e-14));
  // a copied field is independent (value semantics)
  MaterialField c = m;
  c.set_young(std::vector<Scalar>(48, 1e5));
  CHECK(m.young(0) == 8e5 && c.young(0) == 1e5);
  // obstacles (contact.cpp:8-37): normalised half-space, validation
  const Obstacle hs = make_halfspace(Vec3(0, 0, 2), 1.0, 0.3);
  CHECK(hs.normal[2] == 1.0 && hs.offset == 0.5);
  CHECK(obstacle_signed_distance(hs, Vec3(0, 0, 2)) == 1.5);
  threw = false;
  try {
    make_sphere(Vec3(0, 0, 0), -1.0, 0.0);
  } catch (const Error& e) {
    threw = e.code() == ErrorCode::Validation;
  }
  CHECK(threw);
  // scenes: builtin shape table (test_scene.cpp:40-47) and JSON errors
  const SceneSpec two = builtin_scene("two-tet");
  CHECK(two.mesh.element_count() == 2);
  threw = false;
  try {
    parse_scene_json("{not json");
  } catch (const Error& e) {
    threw = e.code() == ErrorCode::Parse;
  }
  CHECK(threw);
}

// ---- device properties ---------------------------------------------------------------------------

struct Block {  // test_util.hpp:80-145 block_scene
  SceneSpec s;
  Block(std::array<int, 3> dims, Scalar gz, bool fix_x0, bool floor, bool hook, Scalar v0_amp) {
    s.mesh = ingest_hex_grid(dims, 0.1, 1000.0);
    const int ne = s.mesh.element_count(), nv = s.mesh.vertex_count();
    const MatX rest = s.mesh.rest_positions();
    const Scalar zmid = 0.5 * (rest.col(2).minCoeff() + rest.col(2).maxCoeff());
    std::vector<Scalar> young(ne, 5e4);
    for (int e = 0; e < ne; ++e) {
      Scalar cz = 0;
      for (int k = 0; k < 4; ++k) cz += rest(s.mesh.elements()[e][k], 2) / 4.0;
      if (cz > zmid) young[e] = 20 * 5e4;
    }
    s.material = build_material(s.mesh, young, 0.4, EnergyKind::NeoHookean, false, 0.01, 0.0);
    s.gravity = Vec3(0, 0, gz);
    if (floor) s.obstacles.push_back(make_halfspace(Vec3(0, 0, 1), 0.0, 0.4));
    if (fix_x0) {
      for (int v = 0; v < nv; ++v)
        if (rest(v, 0) <= 1e-12) s.fixed_vertices.push_back(v);
    }
    s.solver.h = 0.01;
    s.solver.eps_rel = 1e-12;
    s.solver.eps_abs = 1e-14;
    s.q0 = s.mesh.rest_vector();
    s.v0 = VecX::Zero(s.mesh.dof_count());
    for (int i = 0; i < s.v0.size(); ++i) s.v0[i] = v0_amp * std::sin(0.7 * i);
    for (int v : s.fixed_vertices) s.v0.segment<3>(3 * v).setZero();
    if (hook) {
      s.has_hook = true;
      s.hook_vertex = nv - 1;
      s.hook_anchor = Vec3(rest(nv - 1, 0) + 0.02, rest(nv - 1, 1) - 0.01, rest(nv - 1, 2) + 0.05);
      s.hook_stiffness = 2e3;
      s.hook_damping = 5.0;
    }
  }
};


static void device_checks() {
  {  // test_forward.cpp:284-332 ballistic translation, symplectic Euler
    Block b({2, 2, 2}, -2.0, false, false, false, 0.0);
    b.s.material = build_material(b.s.mesh, std::vector<Scalar>(b.s.mesh.element_count(), 5e4), 0.4,
                                  EnergyKind::NeoHookean, false, 0.0, 0.0);
    b.s.solver.eps_rel = 1e-4;
    b.s.solver.eps_abs = 1e-9;
    GlobalSystem sys;
    SimState st{b.s.q0, b.s.v0, 0.0};
    const VecX q0 = st.q, f = scene_external_force(b.s);
    const Scalar h = b.s.solver.h, g = -2.0;
    ForwardCache last;
    for (int k = 0; k < 3; ++k)
      last = forward_step(b.s.mesh, b.s.material, sys, b.s.solver, b.s.obstacles, b.s.fixed_vertices, st, f, nullptr);
    bool ok = true;
    for (int v = 0; v < b.s.mesh.vertex_count(); ++v) {
      ok = ok && close(st.q[3 * v], q0[3 * v], 1e-12) && close(st.q[3 * v + 1], q0[3 * v + 1], 1e-12);
      ok = ok && std::fabs(st.q[3 * v + 2] - (q0[3 * v + 2] + g * h * h * 6.0)) <= 1e-10 * std::fabs(q0[3 * v + 2] + 1);
      ok = ok && std::fabs(st.v[3 * v + 2] - 3 * h * g) <= 1e-10 * 3 * h * std::fabs(g);
    }
    CHECK(ok);
    CHECK(last.converged && last.iteration_count <= 3 && last.contacts.empty() && last.h == h);
    CHECK(std::fabs(st.time - 3 * h) < 1e-15);
    CHECK((last.v_star - (last.q_star - last.q_t) / h).norm() == 0.0);
    SimState probe{last.q_t, last.v_t, 0.0};
    CHECK((free_fall_target(b.s.mesh, probe, last.f_ext, nullptr, h) - last.q_tilde()).norm() <=
          1e-15 * last.q_tilde().norm());
    CHECK(sys.refactor_count() == 1);
  }
  {  // test_forward.cpp:175-190: damped rest configurations are fixed points of the global solve
    const TetMesh mesh = ingest_hex_grid({2, 2, 2}, 0.1, 1000.0);
    const VecX rest = mesh.rest_vector();
    const MaterialField mat = build_material(mesh, std::vector<Scalar>(mesh.element_count(), 5e4), 0.4,
                                             EnergyKind::NeoHookean, false, 0.05, 0.2);
    GlobalSystem sys;
    CHECK(sys.refresh(mesh, mat, 0.01, {}));
    CHECK(!sys.refresh(mesh, mat, 0.01, {}));  // same signature: no refactorization
    SimState st{rest, VecX::Zero(mesh.dof_count()), 0.0};
    SolverConfig cfg;
    cfg.eps_rel = 1e-12;
    cfg.eps_abs = 1e-14;
    forward_step(mesh, mat, sys, cfg, {}, {}, st, VecX::Zero(mesh.dof_count()), nullptr);
    CHECK((st.q - rest).cwiseAbs().maxCoeff() <= 1e-10);
  }
  {  // test_forward.cpp:334-359: pinned vertices remain bitwise fixed
    Block b({3, 2, 2}, -2.0, true, false, false, 0.05);
    GlobalSystem sys;
    SimState st{b.s.q0, b.s.v0, 0.0};
    const VecX f = scene_external_force(b.s);
    for (int k = 0; k < 3; ++k)
      forward_step(b.s.mesh, b.s.material, sys, b.s.solver, b.s.obstacles, b.s.fixed_vertices, st, f, nullptr);
    bool ok = !b.s.fixed_vertices.empty();
    for (int v : b.s.fixed_vertices)
      for (int k = 0; k < 3; ++k) ok = ok && st.q[3 * v + k] == b.s.q0[3 * v + k];
    CHECK(ok);
    CHECK(sys.free_count() + static_cast<int>(sys.fixed_vertices().size()) == b.s.mesh.vertex_count());
  }
  {  // test_backward.cpp:245-300: one-step gradients match central differences (1e-4), contact-free
    MatX rest(5, 3);
    rest << 0, 0, 0, 1, 0, 0, 0, 1, 0, 0, 0, 1, 0, 0, -2;
    const TetMesh mesh = build_tet_mesh(rest, {{0, 1, 2, 3}, {0, 2, 1, 4}}, 1000.0);
    const MaterialField mat = build_material(mesh, {4e4, 9e4}, 0.35, EnergyKind::NeoHookean, false, 0.01, 0.05);
    SolverConfig cfg;
    cfg.eps_rel = 1e-12;
    cfg.eps_abs = 1e-14;
    const int n = mesh.dof_count();
    const VecX r0 = mesh.rest_vector();
    VecX q_t = r0, v_t = VecX::Zero(n), f = VecX::Zero(n);
    for (int i = 0; i < n; ++i) {  // test_util.hpp:51-55 wiggle
      q_t[i] += 0.01 * std::sin(0.7 * i + 0.2);
      v_t[i] += 0.2 * std::sin(0.7 * i + 1.0);
    }
    for (int v = 0; v < mesh.vertex_count(); ++v) f[3 * v + 2] = -2.0 * mesh.vertex_mass(v);
    GlobalSystem sys;
    SimState st{q_t, v_t, 0.0};
    const ForwardCache c = forward_step(mesh, mat, sys, cfg, {}, {}, st, f, nullptr);
    CHECK(c.converged);
    const GradientBundle g = backward_step(mesh, mat, sys, c, AdjointSeed{c.q_star - r0, c.v_star}, nullptr, cfg.eps_tr);
    CHECK(!g.contact_path && g.adjoint_iterations > 0 && (g.tau_used == 0.5 || g.tau_used == 1.0));
    auto loss_at = [&](const VecX& q0, const VecX& v0, const VecX& fe) {
      GlobalSystem s2;
      SimState x{q0, v0, 0.0};
      forward_step(mesh, mat, s2, cfg, {}, {}, x, fe, nullptr);
      return 0.5 * (x.q - r0).squaredNorm() + 0.5 * x.v.squaredNorm();
    };
    bool ok = true;
    for (int i : {0, 5, 3 * 4 + 2}) {
      const double eps = 1e-6;
      VecX qp = q_t, qm = q_t, vp = v_t, vm = v_t, fp = f, fm = f;
      qp[i] += eps;
      qm[i] -= eps;
      vp[i] += eps;
      vm[i] -= eps;
      // forces: a step of 1e-3 of the ~80 N gravity load; at 1e-6 the loss change
      // (~1e-11) is at the level of the converged iterate's own round-off in v
      const double epf = 1e-1;
      fp[i] += epf;
      fm[i] -= epf;
      const double fd[3] = {(loss_at(qp, v_t, f) - loss_at(qm, v_t, f)) / (2 * eps),
                            (loss_at(q_t, vp, f) - loss_at(q_t, vm, f)) / (2 * eps),
                            (loss_at(q_t, v_t, fp) - loss_at(q_t, v_t, fm)) / (2 * epf)};
      const double an[3] = {g.dl_dq_t[i], g.dl_dv_t[i], g.dl_df_ext[i]};
      for (int k = 0; k < 3; ++k) {
        const bool good = std::fabs(fd[k] - an[k]) <= 1e-4 * std::max({std::fabs(fd[k]), std::fabs(an[k]), 1e-6});
        if (!good) std::fprintf(stderr, "FD mismatch var %d index %d: fd %.10e adjoint %.10e\n", k, i, fd[k], an[k]);
        ok = ok && good;
      }
    }
    CHECK(ok);
  }
  {  // caches keep their frame (and factor) across a moduli refresh; slots are reused
    Block b({3, 2, 2}, -2.0, true, false, false, 0.05);
    const VecX f = scene_external_force(b.s);
    GlobalSystem sys;
    SimState st{b.s.q0, b.s.v0, 0.0};
    ForwardCache c0 =
        forward_step(b.s.mesh, b.s.material, sys, b.s.solver, b.s.obstacles, b.s.fixed_vertices, st, f, nullptr);
    const GradientBundle g0 = backward_step(b.s.mesh, b.s.material, sys, c0, AdjointSeed{st.q, st.v}, nullptr, 0.1);
    MaterialField m2 = b.s.material;
    std::vector<Scalar> y(m2.element_count(), 7e4);
    m2.set_young(y);
    SimState st2{b.s.q0, b.s.v0, 0.0};
    forward_step(b.s.mesh, m2, sys, b.s.solver, b.s.obstacles, b.s.fixed_vertices, st2, f, nullptr);
    CHECK(sys.refactor_count() == 2);
    const GradientBundle g1 = backward_step(b.s.mesh, b.s.material, sys, c0, AdjointSeed{c0.q_star, c0.v_star},
                                            nullptr, 0.1);
    // the same frame's adjoint again: equal to the CG stopping tolerance (the
    // second solve is deflated with the first one's recycled Ritz vectors;
    // HETERODYN_DEFLATION=0 makes repeated solves bitwise equal)
    CHECK((g1.dl_dq_t - g0.dl_dq_t).norm() <= 1e-8 * g0.dl_dq_t.norm() &&
          (g1.dl_de - g0.dl_de).norm() <= 1e-8 * g0.dl_de.norm());
  }
  {  // errors cross as heterodyn::Error with the reference's codes
    Block b({2, 2, 2}, -2.0, false, false, false, 0.0);
    GlobalSystem sys;
    SimState bad{VecX::Zero(5), VecX::Zero(5), 0.0};
    bool threw = false;
    try {
      forward_step(b.s.mesh, b.s.material, sys, b.s.solver, {}, {}, bad, VecX(), nullptr);
    } catch (const Error& e) {
      threw = e.code() == ErrorCode::InvalidArgument;
    }
    CHECK(threw);
  }
}

// ---- roll + chain (drivers.cpp:31-99) over a scene file, printed for the oracle comparison --------

static void put(std::FILE* o, const char* k, const VecX& v, bool last = false) {
  std::fprintf(o, "\"%s\": [", k);
  for (Index i = 0; i < v.size(); ++i) std::fprintf(o, "%s%.17g", i ? "," : "", v[i]);
  std::fprintf(o, "]%s\n", last ? "" : ",");
}

static void roll(const std::string& path, int frames) {
  const SceneSpec s = load_scene_file(path);
  const StateForce hook = make_hook(s);
  const StateForce* hp = s.has_hook ? &hook : nullptr;
  const VecX f = scene_external_force(s);
  GlobalSystem sys;
  SimState st{s.q0, s.v0, 0.0};
  std::vector<ForwardCache> caches;
  std::vector<int> iters, contacts;
  for (int t = 0; t < frames; ++t) {
    caches.push_back(forward_step(s.mesh, s.material, sys, s.solver, s.obstacles, s.fixed_vertices, st, f, hp));
    iters.push_back(caches.back().iteration_count);
    contacts.push_back(caches.back().contacts.normal_count());
  }
  // L = 1/2 |q_T|^2 + 1/2 |v_T|^2: seeds q_T, v_T
  AdjointSeed seed{st.q, st.v};
  VecX dfe = VecX::Zero(s.mesh.dof_count()), dw, de;
  std::vector<double> tau(frames);
  int adj = 0;
  for (int t = frames - 1; t >= 0; --t) {
    const GradientBundle g = backward_step(s.mesh, s.material, sys, caches[t], seed, hp, s.solver.eps_tr);
    dfe += g.dl_df_ext;
    dw = dw.size() ? dw + g.dl_dw : g.dl_dw;
    de = de.size() ? de + g.dl_de : g.dl_de;
    tau[t] = g.tau_used;
    adj += g.adjoint_iterations;
    seed = AdjointSeed{g.dl_dq_t, g.dl_dv_t};
  }
  std::FILE* o = stdout;
  std::fprintf(o, "{\n");
  put(o, "q", st.q);
  put(o, "v", st.v);
  put(o, "dl_dq0", seed.dl_dq_next);
  put(o, "dl_dv0", seed.dl_dv_next);
  put(o, "dl_df_ext", dfe);
  put(o, "dl_dw", dw);
  put(o, "dl_de", de);
  put(o, "tau", VecX(tau));
  std::vector<double> it(iters.begin(), iters.end()), cc(contacts.begin(), contacts.end());
  put(o, "iterations", VecX(it));
  put(o, "contacts", VecX(cc));
  std::fprintf(o, "\"adjoint_iterations\": %d, \"refactor_count\": %llu\n}\n", adj,
               static_cast<unsigned long long>(sys.refactor_count()));
}

int main(int argc, char** argv) {
  const std::string mode = argc > 1 ? argv[1] : "host";
  try {
    if (mode == "host") host_checks();
    else if (mode == "device") device_checks();
    else if (mode == "roll" && argc > 3) {
      roll(argv[2], std::atoi(argv[3]));
      return 0;
    } else {
      std::fprintf(stderr, "usage: %s host | device | roll <scene.json> <frames>\n", argv[0]);
      return 2;
    }
  } catch (const Error& e) {
    std::fprintf(stderr, "uncaught heterodyn::Error %d: %s\n", static_cast<int>(e.code()), e.what());
    return 1;
  }
  std::printf("%s: %d checks, %d failed\n", mode.c_str(), g_checks, g_fail);
  return g_fail ? 1 : 0;
}
