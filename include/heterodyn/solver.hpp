// heterodyn-b200 C++ solver API: the reference's C++ entry points for the
// forward/backward Projective Dynamics step, with a device-resident
// GlobalSystem and ForwardCache behind them.
//
// Reference interface this header replaces (paths under /root/reference/proj/src):
//   common.hpp:11-45     Scalar/VecX/Vec3/Mat3/MatX, ErrorCode, Error
//   mesh.hpp:16-70       TetMesh, build_tet_mesh, ingest_hex_grid, deformation_gradient
//   material.hpp:10-90   EnergyKind, Lame, lame_from_young_poisson, ProxMeans,
//                        MaterialField (set_young, freeze_means), build_material
//   contact.hpp:18-92    Obstacle, make_halfspace, make_sphere, ContactPoint, ContactSet
//   factor.hpp:85-130    GlobalSystem (refresh, solve_free, gather/scatter, counters)
//   forward.hpp:19-139   SolverConfig, SimState, StateForce, ForwardCache, forward_step
//   backward.hpp:11-97   AdjointSeed, GradientBundle, backward_step
//   scene.hpp:14-66      SceneSpec, scene_external_force, make_hook, builtin_scene,
//                        parse_scene_json, load_scene_file
//
// Differences a caller sees:
//  * Eigen is not a dependency: VecX / MatX / Vec3 / Mat3 are this header's
//    own dense types with the Eigen subset the reference's callers use
//    (Zero/Constant/Ones, size, (i)/[i], data, norm/dot, +-*/ , comma
//    initialisation, segment).
//  * GlobalSystem owns a device engine (factor S' = D^{-1/2} L^{-1} streamed
//    from HBM, CUDA-graph PD and adjoint loops); ForwardCache holds one
//    device-resident recorded frame of that engine plus host copies of the
//    step's inputs and outputs.  The rest of the reference cache (q_tilde,
//    q_prev_iterate, contacts) is mirrored to the host only on request.
//  * backward_step runs on the engine that produced the cache (its factor),
//    so a cache stays valid after the system is refreshed for new material.
//  * StateForce callbacks run on the host: force(q_t, v_t) is folded into the
//    step's external force, the transposed applies into dL/dq_t and dL/dv_t
//    (forward.cpp:59-68, backward.cpp:306-315) — exactly where the reference
//    uses them.
#pragma once

#include <array>
#include <cmath>
#include <cstdint>
#include <functional>
#include <initializer_list>
#include <memory>
#include <stdexcept>
#include <string>
#include <vector>

namespace heterodyn {

using Scalar = double;
using Index = long;

// ---- dense types (the Eigen subset the reference's callers use) -------------

class VecX;

// Comma initialiser: `v << 1, 2, 3;` fills in order (row-major for matrices).
template <class T>
class CommaInit {
 public:
  CommaInit(T& t, Scalar first) : t_(t), i_(0) { push(first); }
  CommaInit& operator,(Scalar x) {
    push(x);
    return *this;
  }

 private:
  void push(Scalar x) {
    if (i_ >= t_.size()) throw std::out_of_range("comma initialiser: too many coefficients");
    t_.set_rowmajor(i_++, x);
  }
  T& t_;
  Index i_;
};

// A contiguous view of n coefficients of a VecX (`v.segment(i, n)`, `v.segment<3>(i)`).
class VecSegment {
 public:
  VecSegment(Scalar* p, Index n) : p_(p), n_(n) {}
  Index size() const { return n_; }
  Scalar& operator[](Index i) const { return p_[i]; }
  Scalar& operator()(Index i) const { return p_[i]; }
  inline VecSegment& operator=(const VecX& x);
  inline VecSegment& operator+=(const VecX& x);
  inline VecSegment& operator-=(const VecX& x);
  VecSegment& operator*=(Scalar s) {
    for (Index i = 0; i < n_; ++i) p_[i] *= s;
    return *this;
  }
  VecSegment& setZero() {
    for (Index i = 0; i < n_; ++i) p_[i] = 0.0;
    return *this;
  }
  inline operator VecX() const;

 private:
  Scalar* p_;
  Index n_;
};

class VecX {
 public:
  VecX() = default;
  explicit VecX(Index n) : d_(static_cast<size_t>(n), 0.0) {}
  VecX(std::initializer_list<Scalar> l) : d_(l) {}
  explicit VecX(std::vector<Scalar> v) : d_(std::move(v)) {}
  static VecX Zero(Index n) { return VecX(n); }
  static VecX Constant(Index n, Scalar c) {
    VecX v(n);
    v.setConstant(c);
    return v;
  }
  static VecX Ones(Index n) { return Constant(n, 1.0); }
  Index size() const { return static_cast<Index>(d_.size()); }
  Index rows() const { return size(); }
  Scalar* data() { return d_.data(); }
  const Scalar* data() const { return d_.data(); }
  Scalar& operator[](Index i) { return d_[static_cast<size_t>(i)]; }
  Scalar operator[](Index i) const { return d_[static_cast<size_t>(i)]; }
  Scalar& operator()(Index i) { return d_[static_cast<size_t>(i)]; }
  Scalar operator()(Index i) const { return d_[static_cast<size_t>(i)]; }
  void resize(Index n) { d_.assign(static_cast<size_t>(n), 0.0); }
  VecX& setZero() { return setConstant(0.0); }
  VecX& setConstant(Scalar c) {
    for (Scalar& x : d_) x = c;
    return *this;
  }
  Scalar squaredNorm() const { return dot(*this); }
  Scalar norm() const { return std::sqrt(squaredNorm()); }
  Scalar sum() const {
    Scalar s = 0;
    for (Scalar x : d_) s += x;
    return s;
  }
  Scalar dot(const VecX& o) const {
    Scalar s = 0;
    for (size_t i = 0; i < d_.size(); ++i) s += d_[i] * o.d_[i];
    return s;
  }
  Scalar maxCoeff() const {
    Scalar m = d_.empty() ? 0 : d_[0];
    for (Scalar x : d_) m = x > m ? x : m;
    return m;
  }
  Scalar minCoeff() const {
    Scalar m = d_.empty() ? 0 : d_[0];
    for (Scalar x : d_) m = x < m ? x : m;
    return m;
  }
  VecX cwiseAbs() const {
    VecX r(*this);
    for (Scalar& x : r.d_) x = std::fabs(x);
    return r;
  }
  VecX cwiseProduct(const VecX& o) const {
    VecX r(*this);
    for (size_t i = 0; i < d_.size(); ++i) r.d_[i] *= o.d_[i];
    return r;
  }
  VecSegment segment(Index start, Index n) { return VecSegment(data() + start, n); }
  VecX segment(Index start, Index n) const {
    return VecX(std::vector<Scalar>(d_.begin() + start, d_.begin() + start + n));
  }
  template <int N>
  VecSegment segment(Index start) { return segment(start, N); }
  template <int N>
  VecX segment(Index start) const { return segment(start, N); }
  VecX& operator+=(const VecX& o) {
    for (size_t i = 0; i < d_.size(); ++i) d_[i] += o.d_[i];
    return *this;
  }
  VecX& operator-=(const VecX& o) {
    for (size_t i = 0; i < d_.size(); ++i) d_[i] -= o.d_[i];
    return *this;
  }
  VecX& operator*=(Scalar s) {
    for (Scalar& x : d_) x *= s;
    return *this;
  }
  VecX& operator/=(Scalar s) {
    for (Scalar& x : d_) x /= s;
    return *this;
  }
  CommaInit<VecX> operator<<(Scalar x) { return CommaInit<VecX>(*this, x); }
  void set_rowmajor(Index i, Scalar x) { (*this)[i] = x; }
  const std::vector<Scalar>& std_vector() const { return d_; }

 private:
  std::vector<Scalar> d_;
};

inline VecX operator+(VecX a, const VecX& b) { return a += b; }
inline VecX operator-(VecX a, const VecX& b) { return a -= b; }
inline VecX operator-(VecX a) { return a *= -1.0; }
inline VecX operator*(VecX a, Scalar s) { return a *= s; }
inline VecX operator*(Scalar s, VecX a) { return a *= s; }
inline VecX operator/(VecX a, Scalar s) { return a /= s; }

inline VecSegment& VecSegment::operator=(const VecX& x) {
  for (Index i = 0; i < n_; ++i) p_[i] = x[i];
  return *this;
}
inline VecSegment& VecSegment::operator+=(const VecX& x) {
  for (Index i = 0; i < n_; ++i) p_[i] += x[i];
  return *this;
}
inline VecSegment& VecSegment::operator-=(const VecX& x) {
  for (Index i = 0; i < n_; ++i) p_[i] -= x[i];
  return *this;
}
inline VecSegment::operator VecX() const { return VecX(std::vector<Scalar>(p_, p_ + n_)); }

// Column-major dense matrix (Eigen's default storage).
class MatX {
 public:
  MatX() = default;
  MatX(Index r, Index c) : r_(r), c_(c), d_(static_cast<size_t>(r * c), 0.0) {}
  static MatX Zero(Index r, Index c) { return MatX(r, c); }
  static MatX Identity(Index r, Index c) {
    MatX m(r, c);
    for (Index i = 0; i < r && i < c; ++i) m(i, i) = 1.0;
    return m;
  }
  Index rows() const { return r_; }
  Index cols() const { return c_; }
  Index size() const { return r_ * c_; }
  Scalar* data() { return d_.data(); }
  const Scalar* data() const { return d_.data(); }
  Scalar& operator()(Index i, Index j) { return d_[static_cast<size_t>(j * r_ + i)]; }
  Scalar operator()(Index i, Index j) const { return d_[static_cast<size_t>(j * r_ + i)]; }
  void resize(Index r, Index c) {
    r_ = r;
    c_ = c;
    d_.assign(static_cast<size_t>(r * c), 0.0);
  }
  VecX col(Index j) const { return VecX(std::vector<Scalar>(d_.begin() + j * r_, d_.begin() + (j + 1) * r_)); }
  CommaInit<MatX> operator<<(Scalar x) { return CommaInit<MatX>(*this, x); }
  void set_rowmajor(Index k, Scalar x) { (*this)(k / c_, k % c_) = x; }

 private:
  Index r_ = 0, c_ = 0;
  std::vector<Scalar> d_;
};

class Vec3 {
 public:
  Vec3() = default;
  Vec3(Scalar x, Scalar y, Scalar z) : v_{x, y, z} {}
  static Vec3 Zero() { return Vec3(); }
  static Vec3 UnitX() { return Vec3(1, 0, 0); }
  static Vec3 UnitY() { return Vec3(0, 1, 0); }
  static Vec3 UnitZ() { return Vec3(0, 0, 1); }
  Index size() const { return 3; }
  Scalar* data() { return v_; }
  const Scalar* data() const { return v_; }
  Scalar& operator[](Index i) { return v_[i]; }
  Scalar operator[](Index i) const { return v_[i]; }
  Scalar& operator()(Index i) { return v_[i]; }
  Scalar operator()(Index i) const { return v_[i]; }
  Scalar x() const { return v_[0]; }
  Scalar y() const { return v_[1]; }
  Scalar z() const { return v_[2]; }
  Scalar dot(const Vec3& o) const { return v_[0] * o.v_[0] + v_[1] * o.v_[1] + v_[2] * o.v_[2]; }
  Vec3 cross(const Vec3& o) const {
    return Vec3(v_[1] * o.v_[2] - v_[2] * o.v_[1], v_[2] * o.v_[0] - v_[0] * o.v_[2], v_[0] * o.v_[1] - v_[1] * o.v_[0]);
  }
  Scalar squaredNorm() const { return dot(*this); }
  Scalar norm() const { return std::sqrt(squaredNorm()); }
  Vec3 normalized() const {
    const Scalar n = norm();
    return Vec3(v_[0] / n, v_[1] / n, v_[2] / n);
  }
  Vec3& operator+=(const Vec3& o) {
    for (int i = 0; i < 3; ++i) v_[i] += o.v_[i];
    return *this;
  }
  Vec3& operator-=(const Vec3& o) {
    for (int i = 0; i < 3; ++i) v_[i] -= o.v_[i];
    return *this;
  }
  Vec3& operator*=(Scalar s) {
    for (Scalar& x : v_) x *= s;
    return *this;
  }
  Vec3& operator/=(Scalar s) {
    for (Scalar& x : v_) x /= s;
    return *this;
  }
  CommaInit<Vec3> operator<<(Scalar x) { return CommaInit<Vec3>(*this, x); }
  void set_rowmajor(Index i, Scalar x) { v_[i] = x; }

 private:
  Scalar v_[3] = {0, 0, 0};
};
inline Vec3 operator+(Vec3 a, const Vec3& b) { return a += b; }
inline Vec3 operator-(Vec3 a, const Vec3& b) { return a -= b; }
inline Vec3 operator-(Vec3 a) { return a *= -1.0; }
inline Vec3 operator*(Vec3 a, Scalar s) { return a *= s; }
inline Vec3 operator*(Scalar s, Vec3 a) { return a *= s; }
inline Vec3 operator/(Vec3 a, Scalar s) { return a /= s; }

class Mat3 {
 public:
  Mat3() = default;
  static Mat3 Zero() { return Mat3(); }
  static Mat3 Identity() {
    Mat3 m;
    m(0, 0) = m(1, 1) = m(2, 2) = 1.0;
    return m;
  }
  Index rows() const { return 3; }
  Index cols() const { return 3; }
  Index size() const { return 9; }
  Scalar& operator()(Index i, Index j) { return a_[j * 3 + i]; }
  Scalar operator()(Index i, Index j) const { return a_[j * 3 + i]; }
  Scalar* data() { return a_; }
  const Scalar* data() const { return a_; }
  Scalar determinant() const {
    const Mat3& m = *this;
    return m(0, 0) * (m(1, 1) * m(2, 2) - m(1, 2) * m(2, 1)) - m(0, 1) * (m(1, 0) * m(2, 2) - m(1, 2) * m(2, 0)) +
           m(0, 2) * (m(1, 0) * m(2, 1) - m(1, 1) * m(2, 0));
  }
  Mat3 transpose() const {
    Mat3 t;
    for (int i = 0; i < 3; ++i)
      for (int j = 0; j < 3; ++j) t(i, j) = (*this)(j, i);
    return t;
  }
  Scalar squaredNorm() const {
    Scalar s = 0;
    for (Scalar x : a_) s += x * x;
    return s;
  }
  Scalar norm() const { return std::sqrt(squaredNorm()); }
  CommaInit<Mat3> operator<<(Scalar x) { return CommaInit<Mat3>(*this, x); }
  void set_rowmajor(Index k, Scalar x) { (*this)(k / 3, k % 3) = x; }

 private:
  Scalar a_[9] = {0, 0, 0, 0, 0, 0, 0, 0, 0};
};
inline Mat3 operator*(const Mat3& a, const Mat3& b) {
  Mat3 c;
  for (int i = 0; i < 3; ++i)
    for (int j = 0; j < 3; ++j) c(i, j) = a(i, 0) * b(0, j) + a(i, 1) * b(1, j) + a(i, 2) * b(2, j);
  return c;
}
inline Vec3 operator*(const Mat3& a, const Vec3& v) {
  return Vec3(a(0, 0) * v[0] + a(0, 1) * v[1] + a(0, 2) * v[2], a(1, 0) * v[0] + a(1, 1) * v[1] + a(1, 2) * v[2],
              a(2, 0) * v[0] + a(2, 1) * v[1] + a(2, 2) * v[2]);
}

// ---- errors (common.hpp:19-45, the hd_status numbering) ---------------------

enum class ErrorCode : int {
  Ok = 0,
  Parse = 1,
  Validation = 2,
  DegenerateElement = 3,
  InvalidPoisson = 4,
  NonPositiveJacobian = 5,
  ProxDiverged = 6,
  SingularFilteredHessian = 7,
  NotPositiveDefinite = 8,
  SingularContactSystem = 9,
  AdjointDiverged = 10,
  LineSearchFailed = 11,
  Io = 12,
  InvalidArgument = 13,
};

class Error : public std::runtime_error {
 public:
  Error(ErrorCode code, const std::string& what) : std::runtime_error(what), code_(code) {}
  ErrorCode code() const { return code_; }

 private:
  ErrorCode code_;
};
[[noreturn]] inline void fail(ErrorCode code, const std::string& msg) { throw Error(code, msg); }

namespace detail {
struct MeshData;
struct MaterialData;
struct SystemImpl;
struct FrameLease;
}  // namespace detail

// ---- mesh (mesh.hpp:16-70) ---------------------------------------------------

class TetMesh {
 public:
  TetMesh();
  int vertex_count() const;
  int element_count() const;
  int dof_count() const { return 3 * vertex_count(); }
  MatX rest_positions() const;  // n_v x 3
  const std::vector<std::array<int, 4>>& elements() const;
  Scalar volume(int e) const;
  Scalar total_volume() const;
  Mat3 inv_reference(int e) const;  // Dm^{-1}
  VecX lumped_mass() const;         // one entry per DoF
  Scalar vertex_mass(int v) const;
  std::array<int, 12> element_dofs(int e) const;
  VecX rest_vector() const;
  const std::vector<int>& boundary_vertices() const;
  std::uint64_t topology_id() const;
  // B200 extensions: the host mirror's raw arrays (xyz interleaved rest
  // positions, per-vertex masses) and the engine-side mesh.
  const Scalar* rest_data() const;
  const Scalar* vertex_mass_data() const;
  const void* native() const;

  std::shared_ptr<const detail::MeshData> data_;
};

TetMesh build_tet_mesh(const MatX& rest, const std::vector<std::array<int, 4>>& elements, Scalar density);
TetMesh ingest_hex_grid(const std::array<int, 3>& dims, Scalar spacing, Scalar density);
Mat3 deformation_gradient(const TetMesh& mesh, int e, const VecX& q);

// ---- material (material.hpp:10-90) ---------------------------------------------

enum class EnergyKind { Corotated, NeoHookean };

struct Lame {
  Scalar mu = 0.0;
  Scalar lambda = 0.0;
};
Lame lame_from_young_poisson(Scalar young, Scalar poisson);

struct ProxMeans {
  Scalar mu = 0.0;
  Scalar lambda = 0.0;
  Scalar stiffness = 0.0;  // 2*mu + lambda
};

class MaterialField {
 public:
  MaterialField();
  MaterialField(const MaterialField& o);
  MaterialField& operator=(const MaterialField& o);
  MaterialField(MaterialField&&) noexcept;
  MaterialField& operator=(MaterialField&&) noexcept;
  ~MaterialField();
  EnergyKind kind() const;
  bool log_volume_barrier() const;
  Scalar poisson() const;
  Scalar alpha() const;
  Scalar beta0() const;
  Scalar young(int e) const;
  Scalar mu(int e) const;
  Scalar lambda(int e) const;
  Scalar beta(int e) const;
  Scalar total_weight(int e) const { return 2.0 * mu(e) + lambda(e); }
  Scalar rotation_weight(int e) const { return 2.0 * mu(e); }
  Scalar volume_weight(int e) const { return lambda(e); }
  int element_count() const;
  ProxMeans prox_means() const;
  Scalar weight_contrast() const;
  void set_young(const std::vector<Scalar>& young);
  void freeze_means(const ProxMeans& means);
  bool means_frozen() const;
  std::uint64_t version() const;
  const void* native() const;

  std::unique_ptr<detail::MaterialData> data_;
};

MaterialField build_material(const TetMesh& mesh, std::vector<Scalar> young, Scalar poisson, EnergyKind kind,
                             bool log_volume_barrier, Scalar alpha, Scalar beta0);

// ---- contact (contact.hpp:18-92) -------------------------------------------------

struct Obstacle {
  enum class Kind { HalfSpace, Sphere };
  Kind kind = Kind::HalfSpace;
  Vec3 normal = Vec3::UnitY();
  Scalar offset = 0;
  Vec3 center = Vec3::Zero();
  Scalar radius = 1;
  Scalar friction = 0;
};
Obstacle make_halfspace(const Vec3& normal, Scalar offset, Scalar friction);
Obstacle make_sphere(const Vec3& center, Scalar radius, Scalar friction);
Scalar obstacle_signed_distance(const Obstacle& ob, const Vec3& x);

struct ContactPoint {
  int vertex = -1;
  int obstacle_id = -1;
  Scalar friction = 0;
};

// Host mirror of a step's contact rows: normal rows in detection order
// (vertex-major, obstacle-minor, contact.cpp:126-141), then two tangent rows
// per frictional contact.  The engine has no bilateral rows (none of the
// reference's generators or detect_contacts produce them).
class ContactSet {
 public:
  std::vector<ContactPoint> contacts;
  int normal_count() const { return static_cast<int>(contacts.size()); }
  int bilateral_count() const { return 0; }
  int friction_pair_count() const {
    int n = 0;
    for (const ContactPoint& c : contacts) n += c.friction > 0;
    return n;
  }
  int row_count() const { return normal_count() + 2 * friction_pair_count(); }
  bool empty() const { return row_count() == 0; }
};

// ---- forward step (forward.hpp:19-139) -----------------------------------------------

struct SolverConfig {
  Scalar h = 0.01;
  Scalar eps_rel = 1e-4;
  Scalar eps_abs = 1e-9;
  int k_max = 500;
  Scalar eps_tr = 0.1;
  int aa_window = 0;
  Scalar contact_margin = 1e-4;
};

struct SimState {
  VecX q;
  VecX v;
  Scalar time = 0;
};

struct StateForce {
  std::function<VecX(const VecX& q, const VecX& v)> force;
  std::function<VecX(const VecX& q, const VecX& v, const VecX& mu)> dq_transpose_apply;
  std::function<VecX(const VecX& q, const VecX& v, const VecX& mu)> dv_transpose_apply;
};

// One converged step, device-resident: `frame` pins a recorded frame of the
// engine that ran it (q_t, v_t, q~, q*^-1, q*, the per-element projection
// cache, the contact set with its multipliers and inverse columns) until the
// last copy of the cache is destroyed.  The host fields are copies the step
// produced anyway (the caller's state goes in and comes out on the host).
struct ForwardCache {
  Scalar h = 0;
  VecX q_t, v_t;
  VecX f_ext;  // external force of the step, the hook's force(q_t, v_t) included
  VecX q_star, v_star;
  ContactSet contacts;
  int iteration_count = 0;
  bool converged = false;
  std::shared_ptr<detail::FrameLease> frame;
  // host mirrors on request (device -> host copies)
  VecX q_tilde() const;
  VecX q_prev_iterate() const;
};

class GlobalSystem {
 public:
  GlobalSystem();
  ~GlobalSystem();
  GlobalSystem(GlobalSystem&&) noexcept;
  GlobalSystem& operator=(GlobalSystem&&) noexcept;
  GlobalSystem(const GlobalSystem&) = delete;
  GlobalSystem& operator=(const GlobalSystem&) = delete;

  // Staleness check (factor.hpp:89-90): refactorizes when the mesh topology,
  // material version, fixed set, damping or step size changed; returns true
  // when it did.
  bool refresh(const TetMesh& mesh, const MaterialField& material, Scalar h, const std::vector<int>& fixed_vertices);
  bool ready() const;
  int free_count() const;
  const std::vector<int>& free_vertices() const;
  const std::vector<int>& fixed_vertices() const;
  int free_index(int vertex) const;
  VecX gather_free(const VecX& full, int axis) const;
  void scatter_free(const VecX& scalar, int axis, VecX& full) const;
  VecX restrict_free(const VecX& full) const;
  void expand_free(const VecX& free_vec, VecX& full) const;
  // A x = rhs on the free DoFs of all three axes on the device (fixed entries
  // of the result copied from fixed_q).
  VecX solve_free(const VecX& rhs_full, const VecX& fixed_q) const;
  std::uint64_t refactor_count() const;
  std::uint64_t factor_nnz() const;  // nnz of S' (the streamed inverse factor)
  std::uint64_t apply_inverse_count() const;  // 3-axis device solves so far

  std::shared_ptr<detail::SystemImpl> impl_;
};

VecX free_fall_target(const TetMesh& mesh, const SimState& state, const VecX& f_ext, const StateForce* hook, Scalar h);

ForwardCache forward_step(const TetMesh& mesh, const MaterialField& material, GlobalSystem& system,
                          const SolverConfig& config, const std::vector<Obstacle>& obstacles,
                          const std::vector<int>& fixed_vertices, SimState& state, const VecX& f_ext,
                          const StateForce* hook);

// ---- backward step (backward.hpp:11-97) -----------------------------------------------

struct AdjointSeed {
  VecX dl_dq_next;
  VecX dl_dv_next;
};

struct GradientBundle {
  VecX dl_dq_t;
  VecX dl_dv_t;
  VecX dl_df_ext;
  VecX dl_dw;
  VecX dl_de;
  Scalar tau_used = 1;
  Scalar tr_ratio = 1;
  int adjoint_iterations = 0;
  bool contact_path = false;
};

GradientBundle backward_step(const TetMesh& mesh, const MaterialField& material, const GlobalSystem& system,
                             const ForwardCache& cache, const AdjointSeed& seed, const StateForce* hook,
                             Scalar eps_tr);

// ---- scenes (scene.hpp:14-66) ----------------------------------------------------------

struct SceneSpec {
  std::string name;
  TetMesh mesh;
  MaterialField material;
  std::vector<int> fixed_vertices;
  std::vector<Obstacle> obstacles;
  Vec3 gravity = Vec3::Zero();
  VecX f_ext_extra;
  bool has_hook = false;
  int hook_vertex = -1;
  Vec3 hook_anchor = Vec3::Zero();
  Scalar hook_stiffness = 0;
  Scalar hook_damping = 0;
  SolverConfig solver;
  int frames = 1;
  VecX q0, v0;
  std::vector<int> region_of_element;
  int region_count = 0;
};

VecX scene_external_force(const SceneSpec& scene);
StateForce make_hook(const SceneSpec& scene);
SceneSpec builtin_scene(const std::string& name);
SceneSpec parse_scene_json(const std::string& text);
SceneSpec load_scene_file(const std::string& path);

}  // namespace heterodyn
