// The reference's C++ solver API (include/heterodyn/solver.hpp) over the
// device engine.  Reference: mesh.cpp / material.cpp (host setup, restated in
// scene.cpp), factor.cpp:147-208 (GlobalSystem::refresh / solve_free),
// forward.cpp:59-68,148-272 (free_fall_target, forward_step),
// backward.cpp:286-315,396-414 (route_gradients' hook terms, backward_step),
// scene.cpp:542-566 (make_hook).
//
// One GlobalSystem owns an EngineBox: a resolved hdb::Scene (mesh, material,
// fixed set, solver settings, obstacles) and the hdb::Engine built on it (the
// factor in HBM, the forward/adjoint CUDA graphs).  Every forward_step records
// its frame into a free slot of the box's engine; the ForwardCache's
// FrameLease returns the slot when the last copy of the cache goes away, and
// keeps the box (hence the factor the step ran on) alive until then.  A
// refresh that changes anything but Young's moduli — or changes the moduli
// while caches are still alive — builds a new box; a moduli-only change with
// no live caches refactors in place (Engine::set_young, the device-built S'
// values written into the existing stream).
#include "../../include/heterodyn/solver.hpp"

#include <algorithm>
#include <cstring>
#include <fstream>
#include <sstream>

#include "engine.hpp"
#include "host.hpp"

namespace heterodyn {

namespace detail {

struct MeshData {
  hdb::Mesh m;
};

struct MaterialData {
  hdb::Material m;
  hdb::Vec vol;               // rest volumes (the prox means weight by them)
  std::uint64_t lineage = 0;  // build_material call this field descends from
};

struct EngineBox {
  hdb::Scene scene;
  std::unique_ptr<hdb::Engine> eng;
  std::vector<int> free_slots;
  int next_slot = 0;
  int live = 0;
  std::vector<double> last_q, last_v, last_f;  // host copies of the device state / f_ext
  int acquire() {
    ++live;
    if (!free_slots.empty()) {
      const int s = free_slots.back();
      free_slots.pop_back();
      return s;
    }
    return next_slot++;
  }
  void release(int s) {
    --live;
    free_slots.push_back(s);
  }
};

struct FrameLease {
  std::shared_ptr<EngineBox> box;
  int slot = -1;
  bool has_contacts = false;
  FrameLease(std::shared_ptr<EngineBox> b, int s) : box(std::move(b)), slot(s) {}
  ~FrameLease() {
    if (box) box->release(slot);
  }
};

struct Signature {  // factor.hpp:62-73 plus what else the engine bakes
  std::uint64_t topology = 0, material = 0, lineage = 0;
  std::vector<int> fixed;
  double alpha = 0, beta0 = 0, h = 0;
};

struct SystemImpl {
  std::shared_ptr<EngineBox> box;
  Signature sig;
  bool has_sig = false;
  std::uint64_t refactors = 0;
  std::vector<int> free_, fixed_, v2f_;
};

}  // namespace detail

namespace {

using detail::EngineBox;

[[noreturn]] void rethrow_native(const hdb::Error& e) { throw Error(static_cast<ErrorCode>(e.code), e.what()); }

template <class F>
auto guarded(F&& f) -> decltype(f()) {
  try {
    return f();
  } catch (const hdb::Error& e) {
    rethrow_native(e);
  }
}

const hdb::Mesh& nm(const TetMesh& m) {
  if (!m.data_) fail(ErrorCode::InvalidArgument, "TetMesh: empty mesh");
  return m.data_->m;
}
const hdb::Material& nmat(const MaterialField& f) {
  if (!f.data_) fail(ErrorCode::InvalidArgument, "MaterialField: empty material");
  return f.data_->m;
}

hdb::Obstacle to_native(const Obstacle& o) {
  hdb::Obstacle n;
  n.kind = o.kind == Obstacle::Kind::Sphere ? 1 : 0;
  n.normal = {o.normal[0], o.normal[1], o.normal[2]};
  n.offset = o.offset;
  n.center = {o.center[0], o.center[1], o.center[2]};
  n.radius = o.radius;
  n.friction = o.friction;
  return n;
}
Obstacle from_native(const hdb::Obstacle& n) {
  Obstacle o;
  o.kind = n.kind == 1 ? Obstacle::Kind::Sphere : Obstacle::Kind::HalfSpace;
  o.normal = Vec3(n.normal.x, n.normal.y, n.normal.z);
  o.offset = n.offset;
  o.center = Vec3(n.center.x, n.center.y, n.center.z);
  o.radius = n.radius;
  o.friction = n.friction;
  return o;
}
bool same_obstacles(const std::vector<hdb::Obstacle>& a, const std::vector<hdb::Obstacle>& b) {
  if (a.size() != b.size()) return false;
  for (size_t i = 0; i < a.size(); ++i) {
    const hdb::Obstacle& x = a[i];
    const hdb::Obstacle& y = b[i];
    if (x.kind != y.kind || x.normal.x != y.normal.x || x.normal.y != y.normal.y || x.normal.z != y.normal.z ||
        x.offset != y.offset || x.center.x != y.center.x || x.center.y != y.center.y || x.center.z != y.center.z ||
        x.radius != y.radius || x.friction != y.friction)
      return false;
  }
  return true;
}
// what the engine's graphs bake besides the factor inputs (eps_tr: Engine::set_eps_tr)
bool same_loop_settings(const hdb::Solver& a, const hdb::Solver& b) {
  return a.h == b.h && a.eps_rel == b.eps_rel && a.eps_abs == b.eps_abs && a.k_max == b.k_max &&
         a.aa_window == b.aa_window && a.contact_margin == b.contact_margin;
}
hdb::Solver to_native(const SolverConfig& c) {
  hdb::Solver s;
  s.h = c.h;
  s.eps_rel = c.eps_rel;
  s.eps_abs = c.eps_abs;
  s.k_max = c.k_max;
  s.eps_tr = c.eps_tr;
  s.aa_window = c.aa_window;
  s.contact_margin = c.contact_margin;
  return s;
}

std::vector<int> sorted_unique(const std::vector<int>& v, int nv) {
  std::vector<int> s(v);
  std::sort(s.begin(), s.end());
  s.erase(std::unique(s.begin(), s.end()), s.end());
  for (int x : s)
    if (x < 0 || x >= nv) fail(ErrorCode::InvalidArgument, "fixed vertex index out of range");
  return s;
}

bool same_material_but_young(const hdb::Material& a, const hdb::Material& b) {
  return a.kind == b.kind && a.barrier == b.barrier && a.poisson == b.poisson && a.alpha == b.alpha &&
         a.beta0 == b.beta0 && a.frozen == b.frozen &&
         (!a.frozen || (a.mu_bar == b.mu_bar && a.lambda_bar == b.lambda_bar && a.k_bar == b.k_bar));
}

std::shared_ptr<EngineBox> make_box(const TetMesh& mesh, const MaterialField& mat, const std::vector<int>& fixed,
                                    const hdb::Solver& solver, const std::vector<hdb::Obstacle>& obstacles) {
  auto box = std::make_shared<EngineBox>();
  hdb::Scene& s = box->scene;
  s.name = "cpp-api";
  s.mesh = nm(mesh);
  s.material = nmat(mat);
  s.fixed = fixed;
  s.obstacles = obstacles;
  s.solver = solver;
  s.q0 = s.mesh.rest;
  s.v0.assign(s.mesh.rest.size(), 0.0);
  s.f_extra.assign(s.mesh.rest.size(), 0.0);
  box->eng = std::make_unique<hdb::Engine>(s);
  box->last_f.assign(s.mesh.rest.size(), 0.0);  // the scene above has no gravity and no point forces
  return box;
}

void set_free_lists(detail::SystemImpl& S, int nv, const std::vector<int>& fixed) {
  S.fixed_ = fixed;
  S.free_.clear();
  S.v2f_.assign(nv, -1);
  size_t k = 0;
  for (int v = 0; v < nv; ++v) {
    if (k < fixed.size() && fixed[k] == v) {
      ++k;
      continue;
    }
    S.v2f_[v] = static_cast<int>(S.free_.size());
    S.free_.push_back(v);
  }
}

// refresh + engine match for a step: returns true when the factor was rebuilt
bool prepare(GlobalSystem& system, const TetMesh& mesh, const MaterialField& material, const hdb::Solver& solver,
             const std::vector<hdb::Obstacle>* obstacles, const std::vector<int>& fixed_in) {
  if (!system.impl_) system.impl_ = std::make_shared<detail::SystemImpl>();
  detail::SystemImpl& S = *system.impl_;
  const hdb::Mesh& m = nm(mesh);
  const hdb::Material& mat = nmat(material);
  if (static_cast<int>(mat.young.size()) != m.ne)
    fail(ErrorCode::InvalidArgument, "material element count does not match the mesh");
  const std::vector<int> fixed = sorted_unique(fixed_in, m.nv);
  detail::Signature sig;
  sig.topology = m.topology;
  sig.material = mat.version;
  sig.lineage = material.data_->lineage;
  sig.fixed = fixed;
  sig.alpha = mat.alpha;
  sig.beta0 = mat.beta0;
  sig.h = solver.h;
  const bool sig_same = S.has_sig && S.sig.topology == sig.topology && S.sig.material == sig.material &&
                        S.sig.lineage == sig.lineage && S.sig.fixed == sig.fixed && S.sig.alpha == sig.alpha &&
                        S.sig.beta0 == sig.beta0 && S.sig.h == sig.h;
  const std::vector<hdb::Obstacle> obs = obstacles ? *obstacles : (S.box ? S.box->scene.obstacles : std::vector<hdb::Obstacle>{});
  if (sig_same && S.box) {
    if (!same_loop_settings(S.box->scene.solver, solver) || !same_obstacles(S.box->scene.obstacles, obs))
      S.box = make_box(mesh, material, fixed, solver, obs);  // same factor inputs: no refactorization counted
    return false;
  }
  // moduli-only change, no live frames on the current engine: refactor in place
  if (S.box && S.has_sig && S.box->live == 0 && S.sig.topology == sig.topology && S.sig.lineage == sig.lineage &&
      S.sig.fixed == sig.fixed && S.sig.h == sig.h && same_material_but_young(S.box->scene.material, mat) &&
      same_loop_settings(S.box->scene.solver, solver) && same_obstacles(S.box->scene.obstacles, obs)) {
    EngineBox& B = *S.box;
    B.eng->set_young(mat.young, false);
    B.scene.material = mat;
    B.free_slots.clear();  // set_young drops the recorded frames (none are live)
    B.next_slot = 0;
    S.sig = sig;
    ++S.refactors;
    return true;
  }
  S.box = make_box(mesh, material, fixed, solver, obs);
  S.sig = sig;
  S.has_sig = true;
  set_free_lists(S, m.nv, fixed);
  ++S.refactors;
  return true;
}

EngineBox& box_of(const GlobalSystem& s) {
  if (!s.impl_ || !s.impl_->box) fail(ErrorCode::InvalidArgument, "GlobalSystem: not refreshed yet");
  return *s.impl_->box;
}

bool bits_equal(const std::vector<double>& a, const double* b, size_t n) {
  return a.size() == n && std::memcmp(a.data(), b, n * sizeof(double)) == 0;
}

}  // namespace

// ---- TetMesh -------------------------------------------------------------------------

TetMesh::TetMesh() = default;
int TetMesh::vertex_count() const { return data_ ? data_->m.nv : 0; }
int TetMesh::element_count() const { return data_ ? data_->m.ne : 0; }
MatX TetMesh::rest_positions() const {
  MatX r(vertex_count(), 3);
  for (int v = 0; v < vertex_count(); ++v)
    for (int k = 0; k < 3; ++k) r(v, k) = data_->m.rest[3 * v + k];
  return r;
}
const std::vector<std::array<int, 4>>& TetMesh::elements() const { return nm(*this).el; }
Scalar TetMesh::volume(int e) const { return nm(*this).vol.at(e); }
Scalar TetMesh::total_volume() const { return nm(*this).total_volume; }
Mat3 TetMesh::inv_reference(int e) const {
  Mat3 b;
  const double* p = nm(*this).bm.data() + 9 * static_cast<size_t>(e);
  for (int r = 0; r < 3; ++r)
    for (int c = 0; c < 3; ++c) b(r, c) = p[3 * r + c];
  return b;
}
VecX TetMesh::lumped_mass() const {
  VecX m(dof_count());
  for (int v = 0; v < vertex_count(); ++v)
    for (int k = 0; k < 3; ++k) m[3 * v + k] = data_->m.mass[v];
  return m;
}
Scalar TetMesh::vertex_mass(int v) const { return nm(*this).mass.at(v); }
std::array<int, 12> TetMesh::element_dofs(int e) const {
  std::array<int, 12> d{};
  const auto& el = nm(*this).el.at(e);
  for (int i = 0; i < 4; ++i)
    for (int k = 0; k < 3; ++k) d[3 * i + k] = 3 * el[i] + k;
  return d;
}
VecX TetMesh::rest_vector() const { return VecX(nm(*this).rest); }
const std::vector<int>& TetMesh::boundary_vertices() const { return nm(*this).boundary; }
std::uint64_t TetMesh::topology_id() const { return data_ ? data_->m.topology : 0; }
const Scalar* TetMesh::rest_data() const { return nm(*this).rest.data(); }
const Scalar* TetMesh::vertex_mass_data() const { return nm(*this).mass.data(); }
const void* TetMesh::native() const { return data_ ? &data_->m : nullptr; }

TetMesh build_tet_mesh(const MatX& rest, const std::vector<std::array<int, 4>>& elements, Scalar density) {
  if (rest.cols() != 3) fail(ErrorCode::Validation, "build_tet_mesh: rest positions must be n x 3");
  hdb::Vec r(3 * static_cast<size_t>(rest.rows()));
  for (Index v = 0; v < rest.rows(); ++v)
    for (int k = 0; k < 3; ++k) r[3 * v + k] = rest(v, k);
  TetMesh m;
  auto d = std::make_shared<detail::MeshData>();
  d->m = guarded([&] { return hdb::make_mesh(r, elements, density); });
  m.data_ = std::move(d);
  return m;
}

TetMesh ingest_hex_grid(const std::array<int, 3>& dims, Scalar spacing, Scalar density) {
  TetMesh m;
  auto d = std::make_shared<detail::MeshData>();
  d->m = guarded([&] { return hdb::hex_grid(dims[0], dims[1], dims[2], spacing, density); });
  m.data_ = std::move(d);
  return m;
}

Mat3 deformation_gradient(const TetMesh& mesh, int e, const VecX& q) {  // mesh.cpp:142-151: F = Ds Dm^{-1}
  const auto& el = mesh.elements().at(e);
  const Mat3 bm = mesh.inv_reference(e);
  Mat3 ds;
  for (int c = 0; c < 3; ++c)
    for (int r = 0; r < 3; ++r) ds(r, c) = q[3 * el[c + 1] + r] - q[3 * el[0] + r];
  return ds * bm;
}

// ---- MaterialField -------------------------------------------------------------------

MaterialField::MaterialField() = default;
MaterialField::~MaterialField() = default;
MaterialField::MaterialField(MaterialField&&) noexcept = default;
MaterialField& MaterialField::operator=(MaterialField&&) noexcept = default;
MaterialField::MaterialField(const MaterialField& o)
    : data_(o.data_ ? std::make_unique<detail::MaterialData>(*o.data_) : nullptr) {}
MaterialField& MaterialField::operator=(const MaterialField& o) {
  if (this != &o) data_ = o.data_ ? std::make_unique<detail::MaterialData>(*o.data_) : nullptr;
  return *this;
}
EnergyKind MaterialField::kind() const {
  return nmat(*this).kind == hdb::Kind::Corotated ? EnergyKind::Corotated : EnergyKind::NeoHookean;
}
bool MaterialField::log_volume_barrier() const { return nmat(*this).barrier; }
Scalar MaterialField::poisson() const { return nmat(*this).poisson; }
Scalar MaterialField::alpha() const { return nmat(*this).alpha; }
Scalar MaterialField::beta0() const { return nmat(*this).beta0; }
Scalar MaterialField::young(int e) const { return nmat(*this).young.at(e); }
Scalar MaterialField::mu(int e) const { return nmat(*this).mu.at(e); }
Scalar MaterialField::lambda(int e) const { return nmat(*this).lambda.at(e); }
Scalar MaterialField::beta(int e) const { return nmat(*this).beta.at(e); }
int MaterialField::element_count() const { return data_ ? static_cast<int>(data_->m.young.size()) : 0; }
ProxMeans MaterialField::prox_means() const {
  const hdb::Material& m = nmat(*this);
  return ProxMeans{m.mu_bar, m.lambda_bar, m.k_bar};
}
Scalar MaterialField::weight_contrast() const { return nmat(*this).contrast(); }
void MaterialField::set_young(const std::vector<Scalar>& young) {
  nmat(*this);
  guarded([&] {
    data_->m.set_young(young, data_->vol);
    return 0;
  });
}
void MaterialField::freeze_means(const ProxMeans& means) {  // material.cpp: pins the prox means
  nmat(*this);
  data_->m.mu_bar = means.mu;
  data_->m.lambda_bar = means.lambda;
  data_->m.k_bar = means.stiffness;
  data_->m.freeze();
}
bool MaterialField::means_frozen() const { return nmat(*this).frozen; }
std::uint64_t MaterialField::version() const { return nmat(*this).version; }
const void* MaterialField::native() const { return data_ ? &data_->m : nullptr; }

MaterialField build_material(const TetMesh& mesh, std::vector<Scalar> young, Scalar poisson, EnergyKind kind,
                             bool log_volume_barrier, Scalar alpha, Scalar beta0) {
  MaterialField f;
  auto d = std::make_unique<detail::MaterialData>();
  d->m = guarded([&] {
    return hdb::make_material(nm(mesh), young, poisson,
                              kind == EnergyKind::Corotated ? hdb::Kind::Corotated : hdb::Kind::NeoHookean,
                              log_volume_barrier, alpha, beta0);
  });
  d->vol = nm(mesh).vol;
  d->lineage = d->m.version;
  f.data_ = std::move(d);
  return f;
}

Lame lame_from_young_poisson(Scalar young, Scalar poisson) {  // material.cpp:13-22
  if (young <= 0.0) fail(ErrorCode::Validation, "Young's modulus must be positive");
  if (!(poisson > -1.0 && poisson < 0.5))
    fail(ErrorCode::InvalidPoisson, "Poisson ratio must lie in (-1, 0.5), got " + std::to_string(poisson));
  return Lame{young / (2.0 * (1.0 + poisson)), young * poisson / ((1.0 + poisson) * (1.0 - 2.0 * poisson))};
}

// ---- obstacles (contact.cpp:8-52) ------------------------------------------------------

Obstacle make_halfspace(const Vec3& normal, Scalar offset, Scalar friction) {
  const Scalar len = normal.norm();
  if (!(len > 0)) fail(ErrorCode::Validation, "half-space normal must be nonzero");
  if (friction < 0) fail(ErrorCode::Validation, "friction coefficient must be nonnegative");
  Obstacle ob;
  ob.kind = Obstacle::Kind::HalfSpace;
  ob.normal = normal / len;
  ob.offset = offset / len;
  ob.friction = friction;
  return ob;
}
Obstacle make_sphere(const Vec3& center, Scalar radius, Scalar friction) {
  if (!(radius > 0)) fail(ErrorCode::Validation, "sphere radius must be positive");
  if (friction < 0) fail(ErrorCode::Validation, "friction coefficient must be nonnegative");
  Obstacle ob;
  ob.kind = Obstacle::Kind::Sphere;
  ob.center = center;
  ob.radius = radius;
  ob.friction = friction;
  return ob;
}
Scalar obstacle_signed_distance(const Obstacle& ob, const Vec3& x) {
  if (ob.kind == Obstacle::Kind::HalfSpace) return ob.normal.dot(x) - ob.offset;
  return (x - ob.center).norm() - ob.radius;
}

// ---- GlobalSystem ------------------------------------------------------------------------

GlobalSystem::GlobalSystem() = default;
GlobalSystem::~GlobalSystem() = default;
GlobalSystem::GlobalSystem(GlobalSystem&&) noexcept = default;
GlobalSystem& GlobalSystem::operator=(GlobalSystem&&) noexcept = default;

bool GlobalSystem::refresh(const TetMesh& mesh, const MaterialField& material, Scalar h,
                           const std::vector<int>& fixed_vertices) {
  return guarded([&] {
    hdb::Solver so = impl_ && impl_->box ? impl_->box->scene.solver : hdb::Solver{};
    so.h = h;
    return prepare(*this, mesh, material, so, nullptr, fixed_vertices);
  });
}
bool GlobalSystem::ready() const { return impl_ && impl_->box; }
int GlobalSystem::free_count() const { return impl_ ? static_cast<int>(impl_->free_.size()) : 0; }
const std::vector<int>& GlobalSystem::free_vertices() const {
  box_of(*this);
  return impl_->free_;
}
const std::vector<int>& GlobalSystem::fixed_vertices() const {
  box_of(*this);
  return impl_->fixed_;
}
int GlobalSystem::free_index(int vertex) const {
  box_of(*this);
  return impl_->v2f_.at(vertex);
}
VecX GlobalSystem::gather_free(const VecX& full, int axis) const {
  const auto& fr = free_vertices();
  VecX out(static_cast<Index>(fr.size()));
  for (size_t i = 0; i < fr.size(); ++i) out[i] = full[3 * fr[i] + axis];
  return out;
}
void GlobalSystem::scatter_free(const VecX& scalar, int axis, VecX& full) const {
  const auto& fr = free_vertices();
  for (size_t i = 0; i < fr.size(); ++i) full[3 * fr[i] + axis] = scalar[i];
}
VecX GlobalSystem::restrict_free(const VecX& full) const {
  const auto& fr = free_vertices();
  VecX out(3 * static_cast<Index>(fr.size()));
  for (size_t i = 0; i < fr.size(); ++i)
    for (int k = 0; k < 3; ++k) out[3 * i + k] = full[3 * fr[i] + k];
  return out;
}
void GlobalSystem::expand_free(const VecX& free_vec, VecX& full) const {
  const auto& fr = free_vertices();
  for (size_t i = 0; i < fr.size(); ++i)
    for (int k = 0; k < 3; ++k) full[3 * fr[i] + k] = free_vec[3 * i + k];
}
VecX GlobalSystem::solve_free(const VecX& rhs_full, const VecX& fixed_q) const {
  EngineBox& B = box_of(*this);
  const size_t n3 = B.scene.mesh.rest.size();
  if (static_cast<size_t>(rhs_full.size()) != n3) fail(ErrorCode::InvalidArgument, "solve_free: rhs size");
  const bool fq = static_cast<size_t>(fixed_q.size()) == n3;
  return VecX(guarded([&] { return B.eng->solve_free(rhs_full.data(), fq ? fixed_q.data() : nullptr); }));
}
std::uint64_t GlobalSystem::refactor_count() const { return impl_ ? impl_->refactors : 0; }
std::uint64_t GlobalSystem::factor_nnz() const {
  return impl_ && impl_->box ? static_cast<std::uint64_t>(impl_->box->eng->factor().stream_len) : 0;
}
std::uint64_t GlobalSystem::apply_inverse_count() const {
  return impl_ && impl_->box ? static_cast<std::uint64_t>(impl_->box->eng->solve_count) : 0;
}

// ---- forward / backward ---------------------------------------------------------------------

VecX free_fall_target(const TetMesh& mesh, const SimState& state, const VecX& f_ext, const StateForce* hook,
                      Scalar h) {  // forward.cpp:59-68 (host: it is O(n) and not on the device path)
  VecX force = f_ext;
  if (hook && hook->force) force += hook->force(state.q, state.v);
  const hdb::Mesh& m = nm(mesh);
  VecX out(state.q.size());
  for (Index i = 0; i < state.q.size(); ++i)
    out[i] = state.q[i] + h * state.v[i] + h * h * force[i] / m.mass[i / 3];
  return out;
}

ForwardCache forward_step(const TetMesh& mesh, const MaterialField& material, GlobalSystem& system,
                          const SolverConfig& config, const std::vector<Obstacle>& obstacles,
                          const std::vector<int>& fixed_vertices, SimState& state, const VecX& f_ext,
                          const StateForce* hook) {
  return guarded([&] {
    const int n3 = mesh.dof_count();
    if (state.q.size() != n3 || state.v.size() != n3) fail(ErrorCode::InvalidArgument, "forward_step: state size");
    std::vector<hdb::Obstacle> obs;
    for (const Obstacle& o : obstacles) obs.push_back(to_native(o));
    prepare(system, mesh, material, to_native(config), &obs, fixed_vertices);
    std::shared_ptr<EngineBox> boxp = system.impl_->box;
    EngineBox& B = *boxp;
    B.eng->set_eps_tr(config.eps_tr);
    // f_ext + hook force at the step's input state (forward.cpp:59-68)
    VecX f = f_ext.size() == n3 ? f_ext : VecX::Zero(n3);
    if (hook && hook->force) f += hook->force(state.q, state.v);
    if (!bits_equal(B.last_f, f.data(), n3)) {
      B.eng->set_external_force(f.data());
      B.last_f = f.std_vector();
    }
    // the device state is the previous step's output unless the caller changed it
    const bool same_q = bits_equal(B.last_q, state.q.data(), n3), same_v = bits_equal(B.last_v, state.v.data(), n3);
    B.eng->set_state(same_q ? nullptr : state.q.data(), same_v ? nullptr : state.v.data(), state.time, true);
    const int slot = B.acquire();
    try {
      B.eng->step_into(slot);
    } catch (...) {
      B.release(slot);
      B.last_q.clear();  // resynchronise on the next call
      B.last_v.clear();
      throw;
    }
    ForwardCache c;
    c.frame = std::make_shared<detail::FrameLease>(boxp, slot);
    c.h = config.h;
    c.q_t = state.q;
    c.v_t = state.v;
    c.f_ext = f;
    B.eng->positions_into(state.q.data());
    B.eng->velocities_into(state.v.data());
    state.time += config.h;
    B.last_q = state.q.std_vector();
    B.last_v = state.v.std_vector();
    c.q_star = state.q;
    c.v_star = state.v;
    c.iteration_count = B.eng->last_iterations;
    c.converged = B.eng->last_converged != 0;
    if (B.eng->last_contacts > 0) {
      std::vector<int> vx, ob;
      std::vector<double> cl, co;
      int nc = 0, nf = 0, it = 0;
      B.eng->contact_trace(vx, ob, cl, co, nc, nf, it);
      for (int i = 0; i < nc; ++i) c.contacts.contacts.push_back(ContactPoint{vx[i], ob[i], obstacles.at(ob[i]).friction});
      c.frame->has_contacts = true;
    }
    return c;
  });
}

VecX ForwardCache::q_tilde() const {
  if (!frame) fail(ErrorCode::InvalidArgument, "ForwardCache: no recorded frame");
  return VecX(guarded([&] { return frame->box->eng->frame_vector(frame->slot, 0); }));
}
VecX ForwardCache::q_prev_iterate() const {
  if (!frame) fail(ErrorCode::InvalidArgument, "ForwardCache: no recorded frame");
  return VecX(guarded([&] { return frame->box->eng->frame_vector(frame->slot, 1); }));
}

GradientBundle backward_step(const TetMesh& mesh, const MaterialField& material, const GlobalSystem& system,
                             const ForwardCache& cache, const AdjointSeed& seed, const StateForce* hook,
                             Scalar eps_tr) {
  (void)material;
  (void)system;  // the cache's own engine (the factor its step ran on) runs the adjoint
  return guarded([&] {
    if (!cache.frame) fail(ErrorCode::InvalidArgument, "backward_step: the cache has no recorded frame");
    const int n3 = mesh.dof_count();
    EngineBox& B = *cache.frame->box;
    B.eng->set_eps_tr(eps_tr);
    const double* dq = seed.dl_dq_next.size() == n3 ? seed.dl_dq_next.data() : nullptr;
    const double* dv = seed.dl_dv_next.size() == n3 ? seed.dl_dv_next.data() : nullptr;
    hdb::GradOut g = B.eng->backward_slot(cache.frame->slot, dq, dv);
    GradientBundle out;
    out.dl_dq_t = VecX(std::move(g.dl_dq0));
    out.dl_dv_t = VecX(std::move(g.dl_dv0));
    out.dl_df_ext = VecX(std::move(g.dl_df_ext));
    out.dl_dw = VecX(std::move(g.dl_dw));
    out.dl_de = VecX(std::move(g.dl_de));
    out.tau_used = g.tau.at(0);
    out.tr_ratio = g.rho.at(0);
    out.adjoint_iterations = g.adjoint_iterations;
    out.contact_path = cache.frame->has_contacts;
    // backward.cpp:306-315: the hook's transposed Jacobians against mu = dL/df_ext
    if (hook && hook->dv_transpose_apply) out.dl_dv_t += hook->dv_transpose_apply(cache.q_t, cache.v_t, out.dl_df_ext);
    if (hook && hook->dq_transpose_apply) out.dl_dq_t += hook->dq_transpose_apply(cache.q_t, cache.v_t, out.dl_df_ext);
    return out;
  });
}

// ---- scenes ---------------------------------------------------------------------------------------

namespace {
SceneSpec from_native(const hdb::Scene& s) {
  SceneSpec o;
  o.name = s.name;
  auto md = std::make_shared<detail::MeshData>();
  md->m = s.mesh;
  o.mesh.data_ = md;
  auto mt = std::make_unique<detail::MaterialData>();
  mt->m = s.material;
  mt->vol = s.mesh.vol;
  mt->lineage = s.material.version;
  o.material.data_ = std::move(mt);
  o.fixed_vertices = s.fixed;
  for (const hdb::Obstacle& ob : s.obstacles) o.obstacles.push_back(from_native(ob));
  o.gravity = Vec3(s.gravity.x, s.gravity.y, s.gravity.z);
  o.f_ext_extra = s.f_extra.empty() ? VecX::Zero(3 * s.mesh.nv) : VecX(s.f_extra);
  o.has_hook = s.hook;
  o.hook_vertex = s.hook_vertex;
  o.hook_anchor = Vec3(s.hook_anchor.x, s.hook_anchor.y, s.hook_anchor.z);
  o.hook_stiffness = s.hook_k;
  o.hook_damping = s.hook_d;
  o.solver = SolverConfig{s.solver.h, s.solver.eps_rel, s.solver.eps_abs, s.solver.k_max,
                          s.solver.eps_tr, s.solver.aa_window, s.solver.contact_margin};
  o.frames = s.frames;
  o.q0 = VecX(s.q0);
  o.v0 = VecX(s.v0);
  if (s.region.size() == static_cast<size_t>(s.mesh.ne)) o.region_of_element = s.region;
  o.region_count = s.region_count;
  return o;
}
}  // namespace

VecX scene_external_force(const SceneSpec& scene) {  // scene.cpp:530-540: lumped gravity + point forces
  const hdb::Mesh& m = nm(scene.mesh);
  VecX f = scene.f_ext_extra.size() == 3 * m.nv ? scene.f_ext_extra : VecX::Zero(3 * m.nv);
  for (int v = 0; v < m.nv; ++v)
    for (int k = 0; k < 3; ++k) f[3 * v + k] += m.mass[v] * scene.gravity[k];
  return f;
}

StateForce make_hook(const SceneSpec& scene) {  // scene.cpp:542-566
  StateForce hook;
  if (!scene.has_hook) return hook;
  const int v = scene.hook_vertex;
  const Vec3 a = scene.hook_anchor;
  const Scalar k = scene.hook_stiffness, d = scene.hook_damping;
  hook.force = [v, a, k, d](const VecX& q, const VecX& vel) {
    VecX f = VecX::Zero(q.size());
    for (int i = 0; i < 3; ++i) f[3 * v + i] = -k * (q[3 * v + i] - a[i]) - d * vel[3 * v + i];
    return f;
  };
  hook.dq_transpose_apply = [v, k](const VecX&, const VecX&, const VecX& mu) {
    VecX out = VecX::Zero(mu.size());
    for (int i = 0; i < 3; ++i) out[3 * v + i] = -k * mu[3 * v + i];
    return out;
  };
  hook.dv_transpose_apply = [v, d](const VecX&, const VecX&, const VecX& mu) {
    VecX out = VecX::Zero(mu.size());
    for (int i = 0; i < 3; ++i) out[3 * v + i] = -d * mu[3 * v + i];
    return out;
  };
  return hook;
}

SceneSpec builtin_scene(const std::string& name) {
  return guarded([&] { return from_native(hdb::builtin_scene(name)); });
}
SceneSpec parse_scene_json(const std::string& text) {
  return guarded([&] { return from_native(hdb::parse_scene(text)); });
}
SceneSpec load_scene_file(const std::string& path) {
  std::ifstream in(path);
  if (!in) fail(ErrorCode::Io, "cannot read scene file: " + path);
  std::stringstream ss;
  ss << in.rdbuf();
  return parse_scene_json(ss.str());
}

}  // namespace heterodyn
