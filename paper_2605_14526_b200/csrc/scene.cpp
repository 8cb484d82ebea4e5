// Scene setup for the B200 engine: mesh (reference mesh.cpp:27-140), material
// field (material.cpp:13-107) and the scene JSON schema with its built-in
// generators (scene.cpp:100-680).  Host-only, runs once per scene.
#include <algorithm>
#include <atomic>
#include <cmath>
#include <fstream>
#include <limits>
#include <map>
#include <set>


#include <nlohmann/json.hpp>

#include "host.hpp"

namespace hdb {

namespace {
std::atomic<std::uint64_t> g_topo{1}, g_version{1};

inline double det_cols(const double a[3], const double b[3], const double c[3]) {
  // det [a b c] (columns), first-column cofactor expansion
  return a[0] * (b[1] * c[2] - c[1] * b[2]) - a[1] * (b[0] * c[2] - c[0] * b[2]) + a[2] * (b[0] * c[1] - c[0] * b[1]);
}
}  // namespace

// ---- mesh ------------------------------------------------------------------
Mesh make_mesh(const Vec& rest, const std::vector<std::array<int, 4>>& el, double density) {
  if (rest.size() % 3) raise(Code::Validation, "rest positions must be n x 3");
  if (!(density > 0)) raise(Code::Validation, "density must be positive");
  Mesh m;
  m.nv = static_cast<int>(rest.size() / 3);
  if (m.nv < 4) raise(Code::Validation, "mesh needs at least 4 vertices");
  m.ne = static_cast<int>(el.size());
  m.rest = rest;
  m.el = el;
  m.topology = g_topo.fetch_add(1);
  double lo[3], hi[3];
  for (int a = 0; a < 3; ++a) lo[a] = hi[a] = rest[a];
  for (int v = 0; v < m.nv; ++v)
    for (int a = 0; a < 3; ++a) {
      lo[a] = std::min(lo[a], rest[3 * v + a]);
      hi[a] = std::max(hi[a], rest[3 * v + a]);
    }
  const double diag = std::max(std::sqrt((hi[0] - lo[0]) * (hi[0] - lo[0]) + (hi[1] - lo[1]) * (hi[1] - lo[1]) +
                                         (hi[2] - lo[2]) * (hi[2] - lo[2])), 1e-12);
  const double floor_v = 1e-12 * diag * diag * diag;
  m.bm.assign(9 * static_cast<size_t>(m.ne), 0.0);
  m.vol.assign(m.ne, 0.0);
  m.mass.assign(m.nv, 0.0);
  for (int e = 0; e < m.ne; ++e) {
    const auto& t = el[e];
    for (int i = 0; i < 4; ++i) {
      if (t[i] < 0 || t[i] >= m.nv) raise(Code::Validation, "element vertex out of range");
      for (int j = 0; j < i; ++j)
        if (t[i] == t[j]) raise(Code::DegenerateElement, "repeated vertex in element");
    }
    double d[3][3];  // columns x_{k+1} - x_0
    for (int k = 0; k < 3; ++k)
      for (int a = 0; a < 3; ++a) d[k][a] = rest[3 * t[k + 1] + a] - rest[3 * t[0] + a];
    const double det = det_cols(d[0], d[1], d[2]);
    const double v6 = det / 6.0;
    if (v6 <= floor_v)
      raise(Code::DegenerateElement, "element " + std::to_string(e) + " has non-positive or degenerate rest volume");
    m.vol[e] = v6;
    m.total_volume += v6;
    // Dm^{-1} by cofactors; Dm(a, k) = d[k][a]
    auto D = [&](int r, int c) { return d[c][r]; };
    const double inv = 1.0 / det;
    double* b = &m.bm[9 * static_cast<size_t>(e)];
    b[0] = (D(1, 1) * D(2, 2) - D(1, 2) * D(2, 1)) * inv;
    b[1] = (D(0, 2) * D(2, 1) - D(0, 1) * D(2, 2)) * inv;
    b[2] = (D(0, 1) * D(1, 2) - D(0, 2) * D(1, 1)) * inv;
    b[3] = (D(1, 2) * D(2, 0) - D(1, 0) * D(2, 2)) * inv;
    b[4] = (D(0, 0) * D(2, 2) - D(0, 2) * D(2, 0)) * inv;
    b[5] = (D(0, 2) * D(1, 0) - D(0, 0) * D(1, 2)) * inv;
    b[6] = (D(1, 0) * D(2, 1) - D(1, 1) * D(2, 0)) * inv;
    b[7] = (D(0, 1) * D(2, 0) - D(0, 0) * D(2, 1)) * inv;
    b[8] = (D(0, 0) * D(1, 1) - D(0, 1) * D(1, 0)) * inv;
    for (int i = 0; i < 4; ++i) m.mass[t[i]] += density * v6 / 4.0;
  }
  std::map<std::array<int, 3>, int> faces;
  static const int fidx[4][3] = {{1, 2, 3}, {0, 3, 2}, {0, 1, 3}, {0, 2, 1}};
  for (const auto& t : el)
    for (const auto& f : fidx) {
      std::array<int, 3> k{t[f[0]], t[f[1]], t[f[2]]};
      std::sort(k.begin(), k.end());
      ++faces[k];
    }
  std::vector<char> on(m.nv, 0);
  for (const auto& [k, c] : faces)
    if (c == 1) on[k[0]] = on[k[1]] = on[k[2]] = 1;
  for (int v = 0; v < m.nv; ++v)
    if (on[v]) m.boundary.push_back(v);
  return m;
}

// Kuhn split of an axis-aligned hex grid, mirrored in x on odd cells
// (mesh.cpp:100-140) — the element order and orientation fix are the
// reference's so that meshes (and JSON per-element fields) line up.
Mesh hex_grid(int nx, int ny, int nz, double spacing, double density) {
  if (nx < 1 || ny < 1 || nz < 1) raise(Code::Validation, "grid dims must be >= 1");
  if (!(spacing > 0)) raise(Code::Validation, "grid spacing must be positive");
  const int sx = nx + 1, sy = ny + 1, sz = nz + 1;
  Vec rest(3 * static_cast<size_t>(sx) * sy * sz);
  for (int k = 0; k < sz; ++k)
    for (int j = 0; j < sy; ++j)
      for (int i = 0; i < sx; ++i) {
        const size_t v = i + static_cast<size_t>(sx) * (j + static_cast<size_t>(sy) * k);
        rest[3 * v] = i * spacing;
        rest[3 * v + 1] = j * spacing;
        rest[3 * v + 2] = k * spacing;
      }
  static const int tets[6][4] = {{0, 1, 3, 7}, {0, 3, 2, 7}, {0, 2, 6, 7}, {0, 6, 4, 7}, {0, 4, 5, 7}, {0, 5, 1, 7}};
  std::vector<std::array<int, 4>> el;
  el.reserve(6 * static_cast<size_t>(nx) * ny * nz);
  for (int k = 0; k < nz; ++k)
    for (int j = 0; j < ny; ++j)
      for (int i = 0; i < nx; ++i) {
        const bool odd = (i + j + k) & 1;
        int corner[8];
        for (int c = 0; c < 8; ++c) {
          const int bx = odd ? 1 - (c & 1) : (c & 1);
          corner[c] = (i + bx) + sx * ((j + ((c >> 1) & 1)) + sy * (k + ((c >> 2) & 1)));
        }
        for (const auto& t : tets) {
          std::array<int, 4> e{corner[t[0]], corner[t[1]], corner[t[2]], corner[t[3]]};
          double d[3][3];
          for (int c = 0; c < 3; ++c)
            for (int a = 0; a < 3; ++a) d[c][a] = rest[3 * e[c + 1] + a] - rest[3 * e[0] + a];
          if (det_cols(d[0], d[1], d[2]) < 0.0) std::swap(e[2], e[3]);
          el.push_back(e);
        }
      }
  return make_mesh(rest, el, density);
}

// ---- material ----------------------------------------------------------------
namespace {
void lame(double E, double nu, double& mu, double& la) {
  if (E <= 0) raise(Code::Validation, "Young's modulus must be positive");
  if (!(nu > -1.0 && nu < 0.5)) raise(Code::InvalidPoisson, "Poisson ratio must lie in (-1, 0.5), got " + std::to_string(nu));
  mu = E / (2.0 * (1.0 + nu));
  la = E * nu / ((1.0 + nu) * (1.0 - 2.0 * nu));
}
void refresh(Material& m, const Vec& vol) {
  const size_t ne = m.young.size();
  m.mu.resize(ne);
  m.lambda.resize(ne);
  m.beta.resize(ne);
  double mu_max = 0;
  for (size_t e = 0; e < ne; ++e) {
    lame(m.young[e], m.poisson, m.mu[e], m.lambda[e]);
    mu_max = std::max(mu_max, m.mu[e]);
  }
  for (size_t e = 0; e < ne; ++e) m.beta[e] = m.beta0 * m.mu[e] / mu_max;
  if (!m.frozen) {
    double V = 0, M = 0, L = 0;
    for (size_t e = 0; e < ne; ++e) {
      V += vol[e];
      M += vol[e] * m.mu[e];
      L += vol[e] * m.lambda[e];
    }
    m.mu_bar = M / V;
    m.lambda_bar = L / V;
    m.k_bar = 2.0 * m.mu_bar + m.lambda_bar;
  }
  m.version = g_version.fetch_add(1);
}
}  // namespace

double Material::contrast() const {
  double lo = weight(0), hi = lo;
  for (size_t e = 1; e < young.size(); ++e) {
    lo = std::min(lo, weight(static_cast<int>(e)));
    hi = std::max(hi, weight(static_cast<int>(e)));
  }
  return hi / lo;
}
void Material::set_young(const Vec& y, const Vec& vol) {
  if (y.size() != young.size()) raise(Code::Validation, "set_young: element count mismatch");
  young = y;
  refresh(*this, vol);
}
void Material::freeze() {
  frozen = true;
  version = g_version.fetch_add(1);
}

Material make_material(const Mesh& m, const Vec& young, double poisson, Kind kind, bool barrier, double alpha,
                       double beta0) {
  if (static_cast<int>(young.size()) != m.ne)
    raise(Code::Validation, "build_material: one Young's modulus per element required");
  if (alpha < 0 || beta0 < 0) raise(Code::Validation, "damping coefficients must be >= 0");
  if (barrier && kind != Kind::Corotated)
    raise(Code::Validation, "log volume barrier composes with the corotated rotation step");
  Material mat;
  mat.kind = kind;
  mat.barrier = barrier;
  mat.poisson = poisson;
  mat.alpha = alpha;
  mat.beta0 = beta0;
  mat.young = young;
  refresh(mat, m.vol);
  return mat;
}

// ---- scenes ------------------------------------------------------------------
namespace {
using nlohmann::json;
using Errs = std::vector<std::string>;

P3 vec3(const json& j, const std::string& what, Errs& errs) {
  if (!j.is_array() || j.size() != 3 || !j[0].is_number() || !j[1].is_number() || !j[2].is_number()) {
    errs.push_back(what + ": expected an array of 3 numbers");
    return {};
  }
  return {j[0].get<double>(), j[1].get<double>(), j[2].get<double>()};
}

Obstacle halfspace(P3 n, double offset, double mu) {
  const double len = std::sqrt(n.x * n.x + n.y * n.y + n.z * n.z);
  if (!(len > 0)) raise(Code::Validation, "half-space normal must be nonzero");
  if (mu < 0) raise(Code::Validation, "friction coefficient must be nonnegative");
  Obstacle o;
  o.kind = 0;
  o.normal = {n.x / len, n.y / len, n.z / len};
  o.offset = offset / len;
  o.friction = mu;
  return o;
}
Obstacle sphere(P3 c, double r, double mu) {
  if (!(r > 0)) raise(Code::Validation, "sphere radius must be positive");
  if (mu < 0) raise(Code::Validation, "friction coefficient must be nonnegative");
  Obstacle o;
  o.kind = 1;
  o.center = c;
  o.radius = r;
  o.friction = mu;
  return o;
}

std::vector<int> in_box(const Mesh& m, P3 lo, P3 hi) {
  std::vector<int> out;
  for (int v = 0; v < m.nv; ++v) {
    const double* p = &m.rest[3 * static_cast<size_t>(v)];
    if (p[0] >= lo.x && p[1] >= lo.y && p[2] >= lo.z && p[0] <= hi.x && p[1] <= hi.y && p[2] <= hi.z) out.push_back(v);
  }
  return out;
}

std::vector<int> thirds(const Mesh& m, int axis) {
  Vec c(m.ne);
  double lo = std::numeric_limits<double>::max(), hi = std::numeric_limits<double>::lowest();
  for (int e = 0; e < m.ne; ++e) {
    double s = 0;
    for (int k = 0; k < 4; ++k) s += m.rest[3 * static_cast<size_t>(m.el[e][k]) + axis];
    c[e] = s / 4;
    lo = std::min(lo, c[e]);
    hi = std::max(hi, c[e]);
  }
  const double span = std::max(hi - lo, 1e-12);
  std::vector<int> r(m.ne);
  for (int e = 0; e < m.ne; ++e) r[e] = std::min(2, static_cast<int>(3 * (c[e] - lo) / span));
  return r;
}

Vec per_region(const std::vector<int>& r, std::initializer_list<double> vals) {
  const std::vector<double> v(vals);
  Vec y(r.size());
  for (size_t e = 0; e < r.size(); ++e) y[e] = v[r[e]];
  return y;
}

void defaults(Scene& s) {
  if (s.q0.empty()) s.q0 = s.mesh.rest;
  if (s.v0.empty()) s.v0.assign(s.mesh.rest.size(), 0.0);
  if (s.f_extra.empty()) s.f_extra.assign(s.mesh.rest.size(), 0.0);
}

Mesh ico_ball(double radius, double density, P3 c) {
  const double phi = (1.0 + std::sqrt(5.0)) / 2.0;
  const double pts[12][3] = {{-1, phi, 0}, {1, phi, 0}, {-1, -phi, 0}, {1, -phi, 0}, {0, -1, phi}, {0, 1, phi},
                             {0, -1, -phi}, {0, 1, -phi}, {phi, 0, -1}, {phi, 0, 1}, {-phi, 0, -1}, {-phi, 0, 1}};
  static const int tri[20][3] = {{0, 11, 5}, {0, 5, 1}, {0, 1, 7}, {0, 7, 10}, {0, 10, 11}, {1, 5, 9}, {5, 11, 4},
                                 {11, 10, 2}, {10, 7, 6}, {7, 1, 8}, {3, 9, 4}, {3, 4, 2}, {3, 2, 6}, {3, 6, 8},
                                 {3, 8, 9}, {4, 9, 5}, {2, 4, 11}, {6, 2, 10}, {8, 6, 7}, {9, 8, 1}};
  const double sc = radius / std::sqrt(1.0 + phi * phi);
  Vec rest(39);
  for (int i = 0; i < 12; ++i) {
    rest[3 * i] = c.x + sc * pts[i][0];
    rest[3 * i + 1] = c.y + sc * pts[i][1];
    rest[3 * i + 2] = c.z + sc * pts[i][2];
  }
  rest[36] = c.x;
  rest[37] = c.y;
  rest[38] = c.z;
  std::vector<std::array<int, 4>> el;
  for (const auto& f : tri) {
    std::array<int, 4> e{12, f[0], f[1], f[2]};
    double d[3][3];
    for (int k = 0; k < 3; ++k)
      for (int a = 0; a < 3; ++a) d[k][a] = rest[3 * e[k + 1] + a] - rest[3 * e[0] + a];
    if (det_cols(d[0], d[1], d[2]) < 0) std::swap(e[2], e[3]);
    el.push_back(e);
  }
  return make_mesh(rest, el, density);
}

// Built-in scenes (scene.cpp:115-251).
Scene generator(const std::string& name, const json& p, Errs& errs) {
  Scene s;
  const double contrast = p.contains("contrast") ? p["contrast"].get<double>() : 10.0;
  if (name == "two-tet") {
    s.name = name;
    s.mesh = make_mesh({0, 0, 0, 1, 0, 0, 0, 1, 0, 0, 0, 1, 1, 1, 1}, {{0, 1, 2, 3}, {1, 2, 3, 4}}, 1000.0);
    s.material = make_material(s.mesh, {5e4, 8e4}, 0.35, Kind::NeoHookean, false, 0.01, 0.0);
    s.region = {0, 1};
    s.region_count = 2;
    s.gravity = {0, 0, -2.0};
    s.frames = 3;
    s.solver.eps_rel = 1e-12;
    s.solver.eps_abs = 1e-14;
    defaults(s);
    for (size_t i = 0; i < s.v0.size(); ++i) s.v0[i] = 0.05 * std::sin(0.7 * static_cast<double>(i));
    return s;
  }
  if (name == "cantilever3" || name == "twist-bar") {
    const bool twist_bar = name == "twist-bar";
    const double twist = twist_bar ? (p.contains("twist") ? p["twist"].get<double>() : 1.2) : 0.0;
    const double h = 0.05, e0 = 5e4;
    s.name = name;
    s.mesh = hex_grid(12, 3, 3, h, 1000.0);
    s.region = thirds(s.mesh, 0);
    s.region_count = 3;
    s.material = make_material(s.mesh, per_region(s.region, {e0, contrast * e0, e0}), 0.35,
                               twist_bar ? Kind::NeoHookean : Kind::Corotated, false, 0.02, 0.01);
    s.fixed = in_box(s.mesh, {-1e-9, -1, -1}, {0.5 * h, 1, 1});
    defaults(s);
    if (twist != 0) {
      const double L = 12 * h, cy = 1.5 * h, cz = 1.5 * h;
      for (int v = 0; v < s.mesh.nv; ++v) {
        const double* r = &s.mesh.rest[3 * static_cast<size_t>(v)];
        const double a = twist * r[0] / L, dy = r[1] - cy, dz = r[2] - cz;
        s.q0[3 * v + 1] = cy + std::cos(a) * dy - std::sin(a) * dz;
        s.q0[3 * v + 2] = cz + std::sin(a) * dy + std::cos(a) * dz;
      }
    } else {
      s.gravity = {0, 0, -9.81};
    }
    s.frames = twist != 0 ? 40 : 60;
    return s;
  }
  if (name == "ball-drop") {
    const int regions = p.contains("regions") ? p["regions"].get<int>() : 1;
    s.name = name;
    s.mesh = ico_ball(0.25, 800.0, {0, 0, 0.5});
    if (regions != 1 && regions != 3) errs.push_back("mesh.regions: ball-drop supports 1 or 3 regions");
    if (regions == 3) {
      s.region = thirds(s.mesh, 2);
      s.region_count = 3;
      s.material = make_material(s.mesh, per_region(s.region, {2e5, 1e6, 2e6}), 0.3, Kind::NeoHookean, false, 0.02, 0.0);
    } else {
      s.region.assign(s.mesh.ne, 0);
      s.region_count = 1;
      s.material = make_material(s.mesh, Vec(s.mesh.ne, 1e6), 0.3, Kind::NeoHookean, false, 0.02, 0.0);
    }
    s.obstacles.push_back(halfspace({0, 0, 1}, 0.0, 0.4));
    s.gravity = {0, 0, -9.81};
    s.frames = 50;
    defaults(s);
    for (int v = 0; v < s.mesh.nv; ++v) s.v0[3 * v + 2] = -1.0;
    return s;
  }
  if (name == "slab-on-sphere") {
    s.name = name;
    s.mesh = hex_grid(8, 8, 1, 0.05, 900.0);
    s.material = make_material(s.mesh, Vec(s.mesh.ne, 3e4), 0.45, Kind::Corotated, false, 0.03, 0.01);
    s.obstacles.push_back(sphere({0.2, 0.2, -0.13}, 0.12, 0.3));
    s.gravity = {0, 0, -9.81};
    s.frames = 60;
    defaults(s);
    return s;
  }
  if (name == "resting-box") {
    s.name = name;
    s.mesh = hex_grid(2, 2, 2, 0.1, 1000.0);
    s.material = make_material(s.mesh, Vec(s.mesh.ne, 1e5), 0.35, Kind::Corotated, false, 0.05, 0.01);
    s.obstacles.push_back(halfspace({0, 0, 1}, 0.0, 0.5));
    s.gravity = {0, 0, -9.81};
    s.frames = 30;
    defaults(s);
    return s;
  }
  errs.push_back("mesh.generator: unknown generator \"" + name + "\"");
  return generator("two-tet", json::object(), errs);
}

std::string joined(const Errs& errs) {
  std::string m = "scene validation failed:";
  for (const auto& e : errs) m += "\n  - " + e;
  return m;
}

// Document overrides on top of a generator or a bare mesh (scene.cpp:255-528).
void overrides(Scene& s, const json& j, bool gen, Errs& errs) {
  if (j.contains("name") && j["name"].is_string()) s.name = j["name"].get<std::string>();
  if (j.contains("material")) {
    const json& m = j["material"];
    if (!m.is_object()) {
      errs.push_back("material: expected an object");
    } else {
      Material& mat = s.material;
      double nu = mat.poisson, alpha = mat.alpha, beta0 = mat.beta0;
      Kind kind = mat.kind;
      bool barrier = mat.barrier;
      Vec young = mat.young;
      if (m.contains("poisson")) {
        if (m["poisson"].is_number()) nu = m["poisson"].get<double>();
        else errs.push_back("material.poisson: expected a number");
      } else if (!gen) {
        errs.push_back("material.poisson: required");
      }
      if (m.contains("energy")) {
        const std::string en = m["energy"].is_string() ? m["energy"].get<std::string>() : "";
        if (en == "neo-hookean") kind = Kind::NeoHookean;
        else if (en == "corotated") kind = Kind::Corotated;
        else errs.push_back("material.energy: expected \"neo-hookean\" or \"corotated\"");
      }
      if (m.contains("log_barrier")) {
        if (m["log_barrier"].is_boolean()) barrier = m["log_barrier"].get<bool>();
        else errs.push_back("material.log_barrier: expected a boolean");
      }
      if (m.contains("alpha")) alpha = m["alpha"].get<double>();
      if (m.contains("beta0")) beta0 = m["beta0"].get<double>();
      if (m.contains("young")) {
        const json& y = m["young"];
        if (y.is_number()) {
          std::fill(young.begin(), young.end(), y.get<double>());
        } else if (y.is_array() && static_cast<int>(y.size()) == s.mesh.ne) {
          for (int e = 0; e < s.mesh.ne; ++e) young[e] = y[e].get<double>();
        } else if (y.is_object() && y.contains("per_region")) {
          const json& pr = y["per_region"];
          if (s.region_count == 0 || static_cast<int>(pr.size()) != s.region_count)
            errs.push_back("material.young.per_region: size must match the scene's region count");
          else
            for (int e = 0; e < s.mesh.ne; ++e) young[e] = pr[s.region[e]].get<double>();
        } else {
          errs.push_back("material.young: expected a number, a per-element array, or {\"per_region\": [...]}");
        }
      }
      if (std::any_of(young.begin(), young.end(), [](double y) { return !(y > 0); }))
        errs.push_back("material.young: moduli must be positive");
      if (errs.empty()) {
        try {
          mat = make_material(s.mesh, young, nu, kind, barrier, alpha, beta0);
        } catch (const Error& e) {
          errs.push_back(std::string("material: ") + e.what());
        }
      }
    }
  } else if (!gen) {
    errs.push_back("material: required (with poisson) for non-generator scenes");
  }
  if (j.contains("gravity")) s.gravity = vec3(j["gravity"], "gravity", errs);
  if (j.contains("obstacles")) {
    if (!j["obstacles"].is_array()) {
      errs.push_back("obstacles: expected an array");
    } else {
      s.obstacles.clear();
      int i = 0;
      for (const json& o : j["obstacles"]) {
        const std::string tag = "obstacles[" + std::to_string(i++) + "]";
        const std::string type = o.contains("type") && o["type"].is_string() ? o["type"].get<std::string>() : "";
        const double mu = o.contains("friction") ? o["friction"].get<double>() : 0.0;
        try {
          if (type == "halfspace") s.obstacles.push_back(halfspace(vec3(o["normal"], tag + ".normal", errs), o.value("offset", 0.0), mu));
          else if (type == "sphere") s.obstacles.push_back(sphere(vec3(o["center"], tag + ".center", errs), o.value("radius", 1.0), mu));
          else errs.push_back(tag + ".type: expected \"halfspace\" or \"sphere\"");
        } catch (const Error& e) {
          errs.push_back(tag + ": " + e.what());
        }
      }
    }
  }
  std::set<int> fixed(s.fixed.begin(), s.fixed.end());
  if (j.contains("dirichlet")) {
    if (!j["dirichlet"].is_array()) {
      errs.push_back("dirichlet: expected an array");
    } else {
      int i = 0;
      for (const json& d : j["dirichlet"]) {
        const std::string tag = "dirichlet[" + std::to_string(i++) + "]";
        if (!d.contains("vertex") || !d["vertex"].is_number_integer()) { errs.push_back(tag + ".vertex: expected an integer"); continue; }
        const int v = d["vertex"].get<int>();
        if (v < 0 || v >= s.mesh.nv) { errs.push_back(tag + ".vertex: index out of range"); continue; }
        fixed.insert(v);
        if (d.contains("position")) {
          const P3 p = vec3(d["position"], tag + ".position", errs);
          s.q0[3 * v] = p.x;
          s.q0[3 * v + 1] = p.y;
          s.q0[3 * v + 2] = p.z;
        }
      }
    }
  }
  if (j.contains("fix_region")) {
    const json& fr = j["fix_region"];
    if (!fr.is_object() || !fr.contains("min") || !fr.contains("max")) {
      errs.push_back("fix_region: expected {\"min\": [...], \"max\": [...]}");
    } else {
      const P3 lo = vec3(fr["min"], "fix_region.min", errs), hi = vec3(fr["max"], "fix_region.max", errs);
      for (int v : in_box(s.mesh, lo, hi)) fixed.insert(v);
    }
  }
  s.fixed.assign(fixed.begin(), fixed.end());
  if (j.contains("f_ext")) {
    if (!j["f_ext"].is_array()) {
      errs.push_back("f_ext: expected an array of {vertex, force}");
    } else {
      s.f_extra.assign(s.mesh.rest.size(), 0.0);
      int i = 0;
      for (const json& f : j["f_ext"]) {
        const std::string tag = "f_ext[" + std::to_string(i++) + "]";
        if (!f.contains("vertex") || !f["vertex"].is_number_integer()) { errs.push_back(tag + ".vertex: expected an integer"); continue; }
        const int v = f["vertex"].get<int>();
        if (v < 0 || v >= s.mesh.nv) { errs.push_back(tag + ".vertex: index out of range"); continue; }
        const P3 p = vec3(f["force"], tag + ".force", errs);
        s.f_extra[3 * v] += p.x;
        s.f_extra[3 * v + 1] += p.y;
        s.f_extra[3 * v + 2] += p.z;
      }
    }
  }
  if (j.contains("f_state")) {
    const json& fs = j["f_state"];
    if (!fs.is_object() || !fs.contains("point_spring")) {
      errs.push_back("f_state: expected {\"point_spring\": {...}}");
    } else {
      const json& ps = fs["point_spring"];
      if (!ps.contains("vertex") || !ps["vertex"].is_number_integer()) {
        errs.push_back("f_state.point_spring.vertex: expected an integer");
      } else {
        s.hook = true;
        s.hook_vertex = ps["vertex"].get<int>();
        if (s.hook_vertex < 0 || s.hook_vertex >= s.mesh.nv) errs.push_back("f_state.point_spring.vertex: index out of range");
        s.hook_anchor = ps.contains("anchor") ? vec3(ps["anchor"], "f_state.point_spring.anchor", errs) : P3{};
        s.hook_k = ps.value("stiffness", 0.0);
        s.hook_d = ps.value("damping", 0.0);
      }
    }
  }
  if (j.contains("solver")) {
    const json& so = j["solver"];
    if (!so.is_object()) {
      errs.push_back("solver: expected an object");
    } else {
      Solver& c = s.solver;
      c.h = so.value("h", c.h);
      c.eps_rel = so.value("eps_rel", c.eps_rel);
      c.eps_abs = so.value("eps_abs", c.eps_abs);
      c.k_max = so.value("k_max", c.k_max);
      c.eps_tr = so.value("eps_tr", c.eps_tr);
      c.aa_window = so.value("aa_window", c.aa_window);
      c.contact_margin = so.value("contact_margin", c.contact_margin);
      if (!(c.h > 0)) errs.push_back("solver.h: must be positive");
    }
  }
  if (j.contains("frames")) {
    if (!j["frames"].is_number_integer() || j["frames"].get<int>() < 1) errs.push_back("frames: expected an integer >= 1");
    else s.frames = j["frames"].get<int>();
  }
  if (j.contains("initial")) {
    const json& in = j["initial"];
    if (in.contains("velocity")) {
      const json& vel = in["velocity"];
      if (vel.is_array() && vel.size() == 3) {
        const P3 u = vec3(vel, "initial.velocity", errs);
        for (int v = 0; v < s.mesh.nv; ++v) {
          s.v0[3 * v] = u.x;
          s.v0[3 * v + 1] = u.y;
          s.v0[3 * v + 2] = u.z;
        }
      } else if (vel.is_array() && vel.size() == s.mesh.rest.size()) {
        for (size_t i = 0; i < vel.size(); ++i) s.v0[i] = vel[i].get<double>();
      } else {
        errs.push_back("initial.velocity: expected a 3-vector or a full DoF array");
      }
    }
    if (in.contains("position_offset")) {
      const P3 u = vec3(in["position_offset"], "initial.position_offset", errs);
      for (int v = 0; v < s.mesh.nv; ++v) {
        s.q0[3 * v] += u.x;
        s.q0[3 * v + 1] += u.y;
        s.q0[3 * v + 2] += u.z;
      }
    }
  }
  // B200 extension: {"factor": {"ordering": "nd-geometric" | "nd-bfs" | "metis"}}
  if (j.contains("factor") && j["factor"].is_object()) {
    const std::string o = j["factor"].value("ordering", s.ordering);
    if (o != "nd-geometric" && o != "nd-bfs" && o != "metis" && o != "nd-mvc")
      errs.push_back("factor.ordering: expected \"nd-geometric\", \"nd-bfs\", \"nd-mvc\" or \"metis\"");
    else s.ordering = o;
  }
}
}  // namespace

Vec external_force(const Scene& s) {
  Vec f = s.f_extra.size() == s.mesh.rest.size() ? s.f_extra : Vec(s.mesh.rest.size(), 0.0);
  for (int v = 0; v < s.mesh.nv; ++v) {
    f[3 * v] += s.mesh.mass[v] * s.gravity.x;
    f[3 * v + 1] += s.mesh.mass[v] * s.gravity.y;
    f[3 * v + 2] += s.mesh.mass[v] * s.gravity.z;
  }
  return f;
}

Scene builtin_scene(const std::string& name) {
  Errs errs;
  Scene s = generator(name, json::object(), errs);
  if (!errs.empty()) raise(Code::Validation, errs.front());
  return s;
}

Scene parse_scene(const std::string& text) {
  json j;
  try {
    j = json::parse(text);
  } catch (const json::parse_error& e) {
    raise(Code::Parse, std::string("scene JSON: ") + e.what());
  }
  if (!j.is_object()) raise(Code::Validation, "scene: expected a JSON object");
  Errs errs;
  Scene s;
  bool have = false;
  const bool has_mesh = j.contains("mesh") && j["mesh"].is_object();
  if (!has_mesh) {
    errs.push_back("mesh: required object");
  } else {
    const json& m = j["mesh"];
    try {
      if (m.contains("generator")) {
        if (!m["generator"].is_string()) {
          errs.push_back("mesh.generator: expected a string");
        } else {
          s = generator(m["generator"].get<std::string>(), m, errs);
          have = true;
        }
      } else if (m.contains("grid")) {
        const json& g = m["grid"];
        int d[3] = {1, 1, 1};
        if (g.contains("dims") && g["dims"].is_array() && g["dims"].size() == 3)
          for (int i = 0; i < 3; ++i) d[i] = g["dims"][i].get<int>();
        else
          errs.push_back("mesh.grid.dims: expected an array of 3 integers");
        s.mesh = hex_grid(d[0], d[1], d[2], g.value("spacing", 0.1), g.value("density", 1000.0));
        have = true;
      } else if (m.contains("vertices") && m.contains("elements")) {
        const json& vs = m["vertices"];
        const json& es = m["elements"];
        if (!vs.is_array() || vs.empty()) {
          errs.push_back("mesh.vertices: expected a non-empty array");
        } else if (!es.is_array() || es.empty()) {
          errs.push_back("mesh.elements: expected a non-empty array");
        } else {
          Vec rest(3 * vs.size());
          for (size_t i = 0; i < vs.size(); ++i) {
            const P3 p = vec3(vs[i], "mesh.vertices[" + std::to_string(i) + "]", errs);
            rest[3 * i] = p.x;
            rest[3 * i + 1] = p.y;
            rest[3 * i + 2] = p.z;
          }
          std::vector<std::array<int, 4>> el;
          for (size_t i = 0; i < es.size(); ++i) {
            if (!es[i].is_array() || es[i].size() != 4) {
              errs.push_back("mesh.elements[" + std::to_string(i) + "]: expected 4 vertex indices");
              continue;
            }
            el.push_back({es[i][0].get<int>(), es[i][1].get<int>(), es[i][2].get<int>(), es[i][3].get<int>()});
          }
          if (errs.empty()) {
            s.mesh = make_mesh(rest, el, m.value("density", 1000.0));
            have = true;
          }
        }
      } else {
        errs.push_back("mesh: expected \"generator\", \"grid\", or \"vertices\"+\"elements\"");
      }
    } catch (const Error& e) {
      errs.push_back(std::string("mesh: ") + e.what());
    }
  }
  if (!have) raise(Code::Validation, joined(errs));
  if (s.material.young.empty()) s.material = make_material(s.mesh, Vec(s.mesh.ne, 1e5), 0.3, Kind::NeoHookean, false, 0, 0);
  defaults(s);
  try {
    overrides(s, j, j["mesh"].contains("generator"), errs);
  } catch (const json::exception& e) {
    errs.push_back(std::string("scene: ") + e.what());
  }
  if (!errs.empty()) raise(Code::Validation, joined(errs));
  return s;
}

}  // namespace hdb
