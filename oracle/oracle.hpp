// ORACLE — test infrastructure only (parity checker + CPU baseline).
// CPU restatement of the reference heterodyn forward/backward PD step.  Every
// declaration cites the reference file:line it follows (paths relative to
// /root/reference/proj/src).  Only tests/, __graft_entry__.smoke() and
// bench.py's cpu_baseline leg may load the library built from this directory.
#pragma once

#include <atomic>

#include <array>
#include <cstdint>
#include <functional>
#include <stdexcept>
#include <string>
#include <utility>
#include <vector>

#include "la.hpp"

namespace hdo {

using VecX = std::vector<double>;

// common.hpp:19-45
enum class ErrorCode : int {
  Ok = 0, Parse = 1, Validation = 2, DegenerateElement = 3, InvalidPoisson = 4,
  NonPositiveJacobian = 5, ProxDiverged = 6, SingularFilteredHessian = 7,
  NotPositiveDefinite = 8, SingularContactSystem = 9, AdjointDiverged = 10,
  LineSearchFailed = 11, Io = 12, InvalidArgument = 13,
};
class Error : public std::runtime_error {
 public:
  Error(ErrorCode c, const std::string& w) : std::runtime_error(w), code_(c) {}
  ErrorCode code() const { return code_; }
 private:
  ErrorCode code_;
};
[[noreturn]] inline void fail(ErrorCode c, const std::string& m) { throw Error(c, m); }

// common.cpp:9-41 — deterministic fork/join over contiguous chunks.
int worker_count();
void parallel_for(int n, const std::function<void(int)>& fn);
void parallel_tasks(int n, const std::function<void(int)>& fn);

// ---- vector helpers ------------------------------------------------------
inline VecX zeros(int n) { return VecX(static_cast<size_t>(n), 0.0); }
double dot(const VecX& a, const VecX& b);
double norm(const VecX& a);
inline Vec3 seg3(const VecX& x, int v) { return Vec3(x[3 * v], x[3 * v + 1], x[3 * v + 2]); }
inline void set3(VecX& x, int v, const Vec3& a) { x[3 * v] = a[0]; x[3 * v + 1] = a[1]; x[3 * v + 2] = a[2]; }
inline void add3(VecX& x, int v, const Vec3& a) { x[3 * v] += a[0]; x[3 * v + 1] += a[1]; x[3 * v + 2] += a[2]; }

// ---- csr.hpp:14-57 -------------------------------------------------------
struct Triplet { int row = 0, col = 0; double value = 0; };
class CsrMatrix {
 public:
  CsrMatrix() = default;
  CsrMatrix(int r, int c) : rows_(r), cols_(c), off_(r + 1, 0) {}
  static CsrMatrix from_triplets(int rows, int cols, std::vector<Triplet> t);  // csr.cpp:7-32
  int rows() const { return rows_; }
  int cols() const { return cols_; }
  int nnz() const { return static_cast<int>(val_.size()); }
  const std::vector<int>& row_offsets() const { return off_; }
  const std::vector<int>& col_indices() const { return col_; }
  const std::vector<double>& values() const { return val_; }
  VecX multiply(const VecX& x) const;                                         // csr.cpp:34-38
  void multiply_add(const VecX& x, double alpha, VecX& y) const;              // csr.cpp:40-47
  VecX multiply_transpose(const VecX& x) const;                               // csr.cpp:49-58
  CsrMatrix transposed() const;                                               // csr.cpp:60-76
  CsrMatrix submatrix(const std::vector<int>& rm, int nr, const std::vector<int>& cm, int nc) const;
  double coeff(int r, int c) const;
 private:
  int rows_ = 0, cols_ = 0;
  std::vector<int> off_, col_;
  std::vector<double> val_;
};

// ---- mesh.hpp:16-76 ------------------------------------------------------
struct Shape { double g[4][3]; };  // g[i][c]: F(r,c) = sum_i g[i][c] x_i[r]
class TetMesh {
 public:
  int vertex_count() const { return static_cast<int>(rest_.size() / 3); }
  int element_count() const { return static_cast<int>(elements_.size()); }
  int dof_count() const { return static_cast<int>(rest_.size()); }
  const VecX& rest_vector() const { return rest_; }
  Vec3 rest(int v) const { return seg3(rest_, v); }
  const std::vector<std::array<int, 4>>& elements() const { return elements_; }
  double volume(int e) const { return volumes_[e]; }
  double total_volume() const { return total_volume_; }
  const VecX& lumped_mass() const { return mass_; }
  double vertex_mass(int v) const { return mass_[3 * v]; }
  const Shape& shape_gradient(int e) const { return shape_[e]; }
  const Mat3& inv_reference(int e) const { return inv_ref_[e]; }
  const std::vector<int>& boundary_vertices() const { return boundary_; }
  std::uint64_t topology_id() const { return topology_id_; }
  friend TetMesh build_tet_mesh(const VecX& rest, const std::vector<std::array<int, 4>>& el, double density);
 private:
  VecX rest_;
  std::vector<std::array<int, 4>> elements_;
  std::vector<Mat3> inv_ref_;
  std::vector<Shape> shape_;
  std::vector<double> volumes_;
  double total_volume_ = 0;
  VecX mass_;
  std::vector<int> boundary_;
  std::uint64_t topology_id_ = 0;
};
TetMesh build_tet_mesh(const VecX& rest, const std::vector<std::array<int, 4>>& el, double density);  // mesh.cpp:27-98
TetMesh ingest_hex_grid(const std::array<int, 3>& dims, double spacing, double density);          // mesh.cpp:100-140
Mat3 deformation_gradient(const TetMesh& mesh, int e, const VecX& q);                              // mesh.cpp:142-151
// V * G^T vec(P): the 12-vector scattered by pd_rhs (forward.cpp:113-114 with
// element_operator mesh.cpp:153-160): local[3i + r] = sum_c P(r,c) g[i][c].
void element_force(const Shape& s, const Mat3& p, double scale, double out[12]);

// ---- material.hpp:18-90 --------------------------------------------------
enum class EnergyKind { Corotated, NeoHookean };
struct Lame { double mu = 0, lambda = 0; };
Lame lame_from_young_poisson(double young, double poisson);  // material.cpp:13-22
double nh_energy(const Mat3& f, double mu, double lambda);   // material.cpp:24-29
struct ProxMeans { double mu = 0, lambda = 0, stiffness = 0; };
class MaterialField {
 public:
  EnergyKind kind() const { return kind_; }
  bool log_volume_barrier() const { return barrier_; }
  double poisson() const { return poisson_; }
  double alpha() const { return alpha_; }
  double beta0() const { return beta0_; }
  double young(int e) const { return young_[e]; }
  double mu(int e) const { return mu_[e]; }
  double lambda(int e) const { return lambda_[e]; }
  double beta(int e) const { return beta_[e]; }
  double total_weight(int e) const { return 2.0 * mu_[e] + lambda_[e]; }
  double rotation_weight(int e) const { return 2.0 * mu_[e]; }
  double volume_weight(int e) const { return lambda_[e]; }
  int element_count() const { return static_cast<int>(young_.size()); }
  const ProxMeans& prox_means() const { return means_; }
  double weight_contrast() const;                  // material.cpp:38-45
  void set_young(const std::vector<double>& y);    // material.cpp:75-80
  void freeze_means(const ProxMeans& m);           // material.cpp:82-86
  std::uint64_t version() const { return version_; }
  friend MaterialField build_material(const TetMesh&, std::vector<double>, double, EnergyKind, bool, double, double);
 private:
  void recompute(bool refresh_means);              // material.cpp:47-73
  std::vector<double> volume_;
  EnergyKind kind_ = EnergyKind::NeoHookean;
  bool barrier_ = false;
  double poisson_ = 0, alpha_ = 0, beta0_ = 0;
  std::vector<double> young_, mu_, lambda_, beta_;
  ProxMeans means_;
  bool frozen_ = false;
  std::uint64_t version_ = 0;
};
MaterialField build_material(const TetMesh& mesh, std::vector<double> young, double poisson,
                             EnergyKind kind, bool barrier, double alpha, double beta0);  // material.cpp:88-107

// ---- ordering.hpp / factor.hpp ------------------------------------------
struct OrderingResult { std::vector<int> order; bool used_fallback = false; };
OrderingResult nested_dissection_order(const std::vector<std::vector<int>>& adj);       // ordering.cpp:148-156
std::vector<int> min_degree_order(const std::vector<std::vector<int>>& adj, const std::vector<int>& block);  // ordering.cpp:9-47

class SparseFactor {  // factor.hpp:13-50
 public:
  void factorize(const CsrMatrix& a);  // factor.cpp:11-104
  int size() const { return n_; }
  bool ready() const { return n_ > 0; }
  VecX apply_inverse(const VecX& v) const;  // factor.cpp:106-109
  const std::vector<std::pair<int, double>>& s_column(int j) const { return cols_[j]; }
  VecX inverse_column(int v) const;         // factor.cpp:111-119
  const CsrMatrix& s_factor() const { return s_; }
  const CsrMatrix& s_transpose() const { return st_; }
  long long s_nnz() const { return s_.nnz(); }
  double s_fill_ratio() const { return n_ ? double(s_.nnz()) / (double(n_) * n_) : 0.0; }
  const std::string& ordering_name() const { return ordering_name_; }
  double factor_millis() const { return factor_ms_; }
  long long l_nnz() const { return l_nnz_; }
  const std::vector<int>& perm() const { return perm_; }
  mutable std::atomic<std::uint64_t> apply_inverse_count{0};  // atomic: the oracle solves contact columns in parallel
 private:
  int n_ = 0;
  std::vector<int> perm_;
  CsrMatrix s_, st_;
  std::vector<std::vector<std::pair<int, double>>> cols_;
  std::string ordering_name_ = "none";
  double factor_ms_ = 0;
  long long l_nnz_ = 0;
};

struct SpikeRow { int free_vertex = 0; Vec3 direction; };  // factor.hpp:53-57
struct DelassusResult { MatX w; std::vector<VecX> columns; std::vector<VecX> scalar_cols; };
struct FactorSignature {  // factor.hpp:64-75
  std::uint64_t topology = 0, material = 0, dirichlet = 0;
  double alpha = 0, beta0 = 0, h = 0;
  bool matches(const FactorSignature& o) const {
    return topology == o.topology && material == o.material && dirichlet == o.dirichlet &&
           alpha == o.alpha && beta0 == o.beta0 && h == o.h;
  }
};
CsrMatrix assemble_global_scalar(const TetMesh& mesh, const MaterialField& mat, double h);  // factor.cpp:121-136
std::uint64_t hash_fixed_set(const std::vector<int>& fixed);                                  // factor.cpp:138-145

class GlobalSystem {  // factor.hpp:85-130
 public:
  bool refresh(const TetMesh& mesh, const MaterialField& mat, double h, const std::vector<int>& fixed);  // factor.cpp:147-184
  bool ready() const { return factor_.ready(); }
  const SparseFactor& factor() const { return factor_; }
  const CsrMatrix& a_free() const { return a_ff_; }
  const CsrMatrix& a_free_fixed() const { return a_fd_; }
  int free_count() const { return static_cast<int>(free_.size()); }
  const std::vector<int>& free_vertices() const { return free_; }
  const std::vector<int>& fixed_vertices() const { return fixed_; }
  int free_index(int v) const { return v2f_[v]; }
  VecX gather_free(const VecX& full, int axis) const;
  void scatter_free(const VecX& s, int axis, VecX& full) const;
  VecX solve_free(const VecX& rhs_full, const VecX& fixed_q) const;  // factor.cpp:196-208
  VecX apply_a_free(const VecX& x_free) const;                        // factor.cpp:210-221
  VecX restrict_free(const VecX& full) const;
  void expand_free(const VecX& free_vec, VecX& full) const;
  DelassusResult delassus(const std::vector<SpikeRow>& rows) const;  // factor.cpp:237-289
  std::uint64_t refactor_count() const { return refactor_count_; }
  mutable std::uint64_t a_spmv_count = 0;
 private:
  FactorSignature sig_;
  bool has_sig_ = false;
  std::vector<int> free_, fixed_, v2f_;
  CsrMatrix a_full_, a_ff_, a_fd_;
  SparseFactor factor_;
  std::uint64_t refactor_count_ = 0;
};

// ---- localstep.hpp:20-151 ------------------------------------------------
struct SvdResult { Mat3 u, v; Vec3 sigma; };
SvdResult signed_svd(const Mat3& f);                                   // localstep.cpp:99-114
double stretch_energy(const Vec3& s, double mu, double lambda);        // :116-120
Vec3 stretch_gradient(const Vec3& s, double mu, double lambda);        // :122-129
Mat3 stretch_hessian(const Vec3& s, double mu, double lambda);         // :131-145
double barrier_energy(const Vec3& s, double mu, double lambda);        // :147-150
Vec3 barrier_gradient(const Vec3& s, double mu, double lambda);        // :152-159
Mat3 barrier_hessian(const Vec3& s, double mu, double lambda);         // :161-174
struct ProxResult {
  Mat3 p_star = Mat3::identity();
  Vec3 sigma_star = Vec3::ones();
  Mat3 u_rot = Mat3::identity(), v_rot = Mat3::identity();
  Vec3 sigma_f = Vec3::ones();
  int newton_iters = 0;
};
ProxResult corotated_project(const Mat3& f);                                    // :176-179
ProxResult volume_project(const Mat3& f);                                       // :181-237
ProxResult nh_prox(const Mat3& f, double mu, double lambda, double k);          // :239-249
ProxResult log_barrier_prox(const Mat3& f, double mu_e, double lambda_e);       // :251-261
inline double log_barrier_penalty(double mu, double lambda) { return 2.0 * mu + lambda; }
double nh_envelope_value(const ProxResult& pr, double mu, double lambda, double k);  // :263-267
double barrier_envelope_value(const ProxResult& pr, double mu, double lambda);       // :269-274
struct ProxHessian { Mat3 h_prox = Mat3::identity(); double tau = 0; Mat3 h_filtered = Mat3::identity(); };
ProxHessian prox_hessian(const Vec3& s, double mu, double lambda, double k);    // :276-284
ProxHessian tr_blend(const ProxHessian& h, double tau);                        // :286-303
class ProxDifferential {                                                        // :305-357
 public:
  ProxDifferential() = default;
  ProxDifferential(const Mat3& u, const Mat3& v, const Vec3& sigma_f, const Vec3& mapped, const Mat3& jac);
  Mat3 apply(const Mat3& df) const;
  void dense(double out[81]) const;  // column-major 9x9
  Mat3 u_, v_, jac_;
  double pair_a_[3] = {0, 0, 0}, pair_b_[3] = {0, 0, 0};
};
ProxDifferential nh_prox_differential(const ProxResult& pr, const ProxHessian& h, double k);  // :359-371
ProxDifferential polar_differential(const ProxResult& pr);                                   // :373-376
ProxDifferential volume_differential(const ProxResult& pr);                                  // :378-406
ProxDifferential barrier_differential(const ProxResult& pr, double mu, double lambda);       // :408-423

// ---- contact.hpp:18-134 ---------------------------------------------------
struct Obstacle {
  enum class Kind { HalfSpace, Sphere };
  Kind kind = Kind::HalfSpace;
  Vec3 normal = Vec3(0, 1, 0);
  double offset = 0;
  Vec3 center;
  double radius = 1;
  double friction = 0;
};
Obstacle make_halfspace(const Vec3& n, double offset, double friction);  // contact.cpp:8-22
Obstacle make_sphere(const Vec3& c, double r, double friction);          // contact.cpp:24-37
double obstacle_signed_distance(const Obstacle& ob, const Vec3& x);      // contact.cpp:39-44
Vec3 obstacle_normal(const Obstacle& ob, const Vec3& x);                 // contact.cpp:46-52
std::pair<Vec3, Vec3> tangent_basis(const Vec3& n);                      // contact.cpp:54-66
struct ContactPoint {
  int vertex = -1;
  Vec3 normal = Vec3(0, 1, 0);
  double gap_offset = 0;
  Vec3 t1 = Vec3(1, 0, 0), t2 = Vec3(0, 0, 1);
  int obstacle_id = -1;
  double friction = 0, r_n = 0, r_f = 0;
};
struct BilateralRow { int vertex = -1; Vec3 direction = Vec3(1, 0, 0); double target = 0; };
class ContactSet {
 public:
  std::vector<ContactPoint> contacts;
  std::vector<BilateralRow> bilateral;
  int normal_count() const { return static_cast<int>(contacts.size()); }
  int bilateral_count() const { return static_cast<int>(bilateral.size()); }
  int friction_pair_count() const;
  int row_count() const { return normal_count() + bilateral_count() + 2 * friction_pair_count(); }
  bool empty() const { return row_count() == 0; }
  int normal_row(int c) const { return c; }
  int bilateral_row(int i) const { return normal_count() + i; }
  int friction_row(int f) const { return normal_count() + bilateral_count() + 2 * f; }
  std::vector<int> friction_contacts() const;
  std::vector<SpikeRow> rows() const;
  VecX zero_multipliers() const { return zeros(row_count()); }
  VecX constraint_values(const VecX& q) const;
};
ContactSet detect_contacts(const TetMesh& mesh, const VecX& q, const std::vector<Obstacle>& obs,
                           double margin, const std::vector<char>& vertex_free);  // contact.cpp:117-144
double fb_residual(double delta, double r, double lambda);                        // contact.cpp:146-149
std::pair<double, double> ncp_weights(double delta, double r, double lambda);    // contact.cpp:151-158
struct WeightSet { VecX omega, e_diag; };
WeightSet contact_weights(const ContactSet& s, const VecX& q, const VecX& q_t, const VecX& lambda);  // :160-196
VecX offset_vector(const ContactSet& s, const WeightSet& w, const VecX& q_t);                       // :198-216
VecX project_multipliers(const ContactSet& s, VecX lambda);                                         // :218-235
VecX contact_iteration(const ContactSet& s, const MatX& w, const WeightSet& wt, const VecX& h_vec,
                       const VecX& jq_mid, const VecX& lambda, VecX* unprojected = nullptr);        // :237-256

// ---- forward.hpp:19-139 ----------------------------------------------------
struct SolverConfig {
  double h = 0.01, eps_rel = 1e-4, eps_abs = 1e-9;
  int k_max = 500;
  double eps_tr = 0.1;
  int aa_window = 0;
  double contact_margin = 1e-4;
};
struct SimState { VecX q, v; double time = 0; };
struct StateForce {
  std::function<VecX(const VecX&, const VecX&)> force;
  std::function<VecX(const VecX&, const VecX&, const VecX&)> dq_transpose_apply;
  std::function<VecX(const VecX&, const VecX&, const VecX&)> dv_transpose_apply;
};
struct ElementProjection { ProxResult primary, secondary; bool has_secondary = false; };
class AaHistory {  // forward.hpp:56-83, forward.cpp:17-57
 public:
  explicit AaHistory(int window, double guard = 10) : window_(window < 1 ? 1 : window), guard_(guard) {}
  int window() const { return window_; }
  int stored() const { return static_cast<int>(dq_.size()); }
  bool guard_tripped() const { return tripped_; }
  VecX mix(const VecX& q_prev, const VecX& g);
  void clear();
 private:
  int window_ = 1;
  double guard_ = 10;
  std::vector<VecX> dq_, dg_;
  bool has_last_ = false, tripped_ = false;
  VecX last_q_, last_g_;
};
struct ForwardCache {  // forward.hpp:86-102
  double h = 0;
  VecX q_t, v_t, f_ext, q_tilde, q_prev_iterate, q_star, v_star, b_star;
  std::vector<ElementProjection> projections;
  ContactSet contacts;
  VecX lambda_star;
  WeightSet weights_star;
  MatX delassus;
  std::vector<VecX> cached_columns;
  int iteration_count = 0;
  bool converged = false;
  // Parity observability (not in the reference cache): per iteration, the
  // decision values of project_multipliers (contact.cpp:218-235), see
  // hd_sim_contact_trace.
  std::vector<double> trace_clamp, trace_cone;
};
VecX free_fall_target(const TetMesh& mesh, const SimState& st, const VecX& f_ext, const StateForce* hook, double h);  // forward.cpp:59-68
std::vector<ElementProjection> local_solve(const TetMesh& mesh, const MaterialField& mat, const VecX& q);           // :70-94
VecX pd_rhs(const TetMesh& mesh, const MaterialField& mat, const VecX& q_tilde,
            const std::vector<ElementProjection>& proj, double h);                                                // :96-117
VecX damping_rhs(const TetMesh& mesh, const MaterialField& mat, const VecX& q_t, double h);                        // :119-138
bool dual_gate(const VecX& qk, const VecX& qk1, const VecX& bk, const VecX& bk1, double er, double ea, int k);    // :140-146
ForwardCache forward_step(const TetMesh& mesh, const MaterialField& mat, GlobalSystem& sys, const SolverConfig& cfg,
                          const std::vector<Obstacle>& obs, const std::vector<int>& fixed, SimState& st,
                          const VecX& f_ext, const StateForce* hook);                                              // :148-272

// ---- backward.hpp:9-97 -----------------------------------------------------
struct AdjointSeed { VecX dl_dq_next, dl_dv_next; };
struct GradientBundle {
  VecX dl_dq_t, dl_dv_t, dl_df_ext, dl_dw, dl_de;
  double tau_used = 1, tr_ratio = 1;
  int adjoint_iterations = 0;
  bool contact_path = false;
};
double primal_energy(const TetMesh& mesh, const MaterialField& mat, const GlobalSystem& sys, const VecX& q,
                     const VecX& q_tilde, double h);                                   // backward.cpp:49-73
struct TrSelection { double tau = 1, rho = 1; };
TrSelection tr_select_tau(const TetMesh& mesh, const MaterialField& mat, const GlobalSystem& sys,
                          const ForwardCache& cache, double eps_tr);                   // backward.cpp:75-108
struct DbDqOperator {
  CsrMatrix matrix;
  VecX apply(const VecX& dq) const { return matrix.multiply(dq); }
};
DbDqOperator assemble_db_dq(const TetMesh& mesh, const MaterialField& mat, const ForwardCache& cache, double tau);  // :117-163
struct AdjointResult { VecX mu, y_q, y_lambda, b_mu; int iterations = 0; bool contact_path = false; };
AdjointResult adjoint_solve(const GlobalSystem& sys, const DbDqOperator& b, const ForwardCache& cache, const VecX& seed);  // :208-284
GradientBundle route_gradients(const TetMesh& mesh, const MaterialField& mat, const GlobalSystem& sys,
                               const ForwardCache& cache, const AdjointResult& adj, const AdjointSeed& seed,
                               const StateForce* hook);                                 // :286-394
GradientBundle backward_step(const TetMesh& mesh, const MaterialField& mat, const GlobalSystem& sys,
                             const ForwardCache& cache, const AdjointSeed& seed, const StateForce* hook,
                             double eps_tr);                                            // :396-414

// ---- scene.hpp:14-55 -------------------------------------------------------
struct SceneSpec {
  std::string name;
  TetMesh mesh;
  MaterialField material;
  std::vector<int> fixed_vertices;
  std::vector<Obstacle> obstacles;
  Vec3 gravity;
  VecX f_ext_extra;
  bool has_hook = false;
  int hook_vertex = -1;
  Vec3 hook_anchor;
  double hook_stiffness = 0, hook_damping = 0;
  SolverConfig solver;
  int frames = 1;
  VecX q0, v0;
  std::vector<int> region_of_element;
  int region_count = 0;
};
VecX scene_external_force(const SceneSpec& s);          // scene.cpp:530-540
StateForce make_hook(const SceneSpec& s);                // scene.cpp:542-566
SceneSpec builtin_scene(const std::string& name);        // scene.cpp:568-573
SceneSpec parse_scene_json(const std::string& text);     // scene.cpp:575-680
SceneSpec load_scene_file(const std::string& path);      // scene.cpp:682-688

// ---- drivers.cpp:31-99 -----------------------------------------------------
struct ChainResult {
  VecX dl_dq0, dl_dv0, dl_df_ext, dl_dw, dl_de;
  std::vector<double> tau, rho;
  int adjoint_iterations = 0;
};
ChainResult chain_backward(const TetMesh& mesh, const MaterialField& mat, const GlobalSystem& sys,
                           const std::vector<ForwardCache>& caches, const std::vector<VecX>& dl_dq_direct,
                           const VecX& dl_dv_final, const StateForce* hook, double eps_tr);

}  // namespace hdo
