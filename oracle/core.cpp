// ORACLE — test infrastructure only.  Restates common.cpp, csr.cpp, mesh.cpp
// and material.cpp of /root/reference/proj/src.
#include <algorithm>
#include <atomic>
#include <cstdlib>
#include <map>
#include <thread>

#include "oracle.hpp"

namespace hdo {

// common.cpp:9-21
int worker_count() {
  static const int cached = [] {
    int hw = static_cast<int>(std::thread::hardware_concurrency());
    if (hw < 1) hw = 1;
    if (const char* env = std::getenv("HETERODYN_THREADS")) {
      char* end = nullptr;
      long v = std::strtol(env, &end, 10);
      if (end != env && v >= 1) hw = static_cast<int>(std::min<long>(v, 256));
    }
    return hw;
  }();
  return cached;
}

// common.cpp:23-41 — one std::thread per chunk on every call, like the
// reference (its spawn cost is part of the baseline being timed).
namespace {
thread_local bool t_in_worker = false;  // nested parallel_for runs serially inside a worker
}
void parallel_for(int n, const std::function<void(int)>& fn) {
  const int workers = std::min(worker_count(), n);
  if (workers <= 1 || n < 64 || t_in_worker) {
    for (int i = 0; i < n; ++i) fn(i);
    return;
  }
  std::vector<std::thread> pool;
  const int chunk = (n + workers - 1) / workers;
  for (int w = 0; w < workers; ++w) {
    const int lo = w * chunk, hi = std::min(n, lo + chunk);
    if (lo >= hi) break;
    pool.emplace_back([lo, hi, &fn] {
      t_in_worker = true;
      for (int i = lo; i < hi; ++i) fn(i);
    });
  }
  for (auto& t : pool) t.join();
}

// One task per index on up to worker_count() threads (dynamic assignment);
// used for independent work items larger than an element (contact columns).
void parallel_tasks(int n, const std::function<void(int)>& fn) {
  const int workers = std::min(worker_count(), n);
  if (workers <= 1 || t_in_worker) {
    for (int i = 0; i < n; ++i) fn(i);
    return;
  }
  std::atomic<int> next{0};
  std::vector<std::thread> pool;
  for (int w = 0; w < workers; ++w)
    pool.emplace_back([&] {
      t_in_worker = true;
      for (int i = next++; i < n; i = next++) fn(i);
    });
  for (auto& t : pool) t.join();
}

double dot(const VecX& a, const VecX& b) {
  double s = 0;
  for (size_t i = 0; i < a.size(); ++i) s += a[i] * b[i];
  return s;
}
double norm(const VecX& a) { return std::sqrt(dot(a, a)); }

// ---- csr.cpp ---------------------------------------------------------------
// csr.cpp:7-32: sort (row, col), sum duplicates in sorted order, drop exact 0.
CsrMatrix CsrMatrix::from_triplets(int rows, int cols, std::vector<Triplet> t) {
  CsrMatrix m(rows, cols);
  std::sort(t.begin(), t.end(), [](const Triplet& a, const Triplet& b) {
    return a.row != b.row ? a.row < b.row : a.col < b.col;
  });
  std::vector<int> counts(rows, 0);
  m.col_.reserve(t.size());
  m.val_.reserve(t.size());
  size_t i = 0;
  while (i < t.size()) {
    const int r = t[i].row, c = t[i].col;
    if (r < 0 || r >= rows || c < 0 || c >= cols) fail(ErrorCode::InvalidArgument, "triplet index out of range");
    double sum = 0.0;
    while (i < t.size() && t[i].row == r && t[i].col == c) sum += t[i++].value;
    if (sum != 0.0) {
      m.col_.push_back(c);
      m.val_.push_back(sum);
      ++counts[r];
    }
  }
  for (int r = 0; r < rows; ++r) m.off_[r + 1] = m.off_[r] + counts[r];
  return m;
}

VecX CsrMatrix::multiply(const VecX& x) const {
  VecX y = zeros(rows_);
  multiply_add(x, 1.0, y);
  return y;
}

// csr.cpp:40-47 (serial, as in the reference)
void CsrMatrix::multiply_add(const VecX& x, double alpha, VecX& y) const {
  for (int r = 0; r < rows_; ++r) {
    double acc = 0.0;
    for (int k = off_[r]; k < off_[r + 1]; ++k) acc += val_[k] * x[col_[k]];
    y[r] += alpha * acc;
  }
}

// csr.cpp:49-58
VecX CsrMatrix::multiply_transpose(const VecX& x) const {
  VecX y = zeros(cols_);
  for (int r = 0; r < rows_; ++r) {
    const double xr = x[r];
    if (xr == 0.0) continue;
    for (int k = off_[r]; k < off_[r + 1]; ++k) y[col_[k]] += val_[k] * xr;
  }
  return y;
}

// csr.cpp:60-76
CsrMatrix CsrMatrix::transposed() const {
  CsrMatrix t(cols_, rows_);
  std::vector<int> counts(cols_, 0);
  for (int c : col_) ++counts[c];
  for (int c = 0; c < cols_; ++c) t.off_[c + 1] = t.off_[c] + counts[c];
  t.col_.resize(val_.size());
  t.val_.resize(val_.size());
  std::vector<int> cursor(t.off_.begin(), t.off_.end() - 1);
  for (int r = 0; r < rows_; ++r)
    for (int k = off_[r]; k < off_[r + 1]; ++k) {
      const int pos = cursor[col_[k]]++;
      t.col_[pos] = r;
      t.val_[pos] = val_[k];
    }
  return t;
}

// csr.cpp:78-90
CsrMatrix CsrMatrix::submatrix(const std::vector<int>& rm, int nr, const std::vector<int>& cm, int nc) const {
  std::vector<Triplet> trips;
  for (int r = 0; r < rows_; ++r) {
    if (rm[r] < 0) continue;
    for (int k = off_[r]; k < off_[r + 1]; ++k) {
      const int c = cm[col_[k]];
      if (c < 0) continue;
      trips.push_back({rm[r], c, val_[k]});
    }
  }
  return from_triplets(nr, nc, std::move(trips));
}

double CsrMatrix::coeff(int r, int c) const {
  for (int k = off_[r]; k < off_[r + 1]; ++k)
    if (col_[k] == c) return val_[k];
  return 0.0;
}

// ---- mesh.cpp ----------------------------------------------------------------
namespace {
std::atomic<std::uint64_t> g_topology{1};
std::atomic<std::uint64_t> g_material{1};
}  // namespace

// mesh.cpp:27-98
TetMesh build_tet_mesh(const VecX& rest, const std::vector<std::array<int, 4>>& elements, double density) {
  if (rest.size() % 3 != 0) fail(ErrorCode::Validation, "rest positions must be n x 3");
  if (density <= 0.0) fail(ErrorCode::Validation, "density must be positive");
  const int nv = static_cast<int>(rest.size() / 3);
  if (nv < 4) fail(ErrorCode::Validation, "mesh needs at least 4 vertices");
  TetMesh m;
  m.rest_ = rest;
  m.elements_ = elements;
  m.topology_id_ = g_topology.fetch_add(1);
  Vec3 lo = seg3(rest, 0), hi = lo;
  for (int v = 1; v < nv; ++v)
    for (int a = 0; a < 3; ++a) {
      lo[a] = std::min(lo[a], rest[3 * v + a]);
      hi[a] = std::max(hi[a], rest[3 * v + a]);
    }
  const double char_len = std::max((hi - lo).norm(), 1e-12);
  const double vol_floor = 1e-12 * char_len * char_len * char_len;
  const int ne = static_cast<int>(elements.size());
  m.inv_ref_.resize(ne);
  m.shape_.resize(ne);
  m.volumes_.resize(ne);
  m.mass_ = zeros(3 * nv);
  for (int e = 0; e < ne; ++e) {
    const auto& el = elements[e];
    for (int i = 0; i < 4; ++i) {
      if (el[i] < 0 || el[i] >= nv) fail(ErrorCode::Validation, "element vertex out of range");
      for (int j = i + 1; j < 4; ++j)
        if (el[i] == el[j]) fail(ErrorCode::DegenerateElement, "repeated vertex in element");
    }
    Mat3 dm;
    for (int k = 0; k < 3; ++k) dm.set_col(k, seg3(rest, el[k + 1]) - seg3(rest, el[0]));
    const double vol = dm.determinant() / 6.0;
    if (vol <= vol_floor)
      fail(ErrorCode::DegenerateElement, "element " + std::to_string(e) + " has non-positive or degenerate rest volume");
    m.volumes_[e] = vol;
    m.total_volume_ += vol;
    m.inv_ref_[e] = dm.inverse();
    const Mat3& bm = m.inv_ref_[e];
    Shape& g = m.shape_[e];
    for (int c = 0; c < 3; ++c) g.g[0][c] = 0.0;
    for (int k = 0; k < 3; ++k)
      for (int c = 0; c < 3; ++c) {
        g.g[k + 1][c] = bm(k, c);
        g.g[0][c] -= bm(k, c);
      }
    const double quarter = density * vol / 4.0;
    for (int i = 0; i < 4; ++i)
      for (int a = 0; a < 3; ++a) m.mass_[3 * el[i] + a] += quarter;
  }
  std::map<std::array<int, 3>, int> face_count;
  static const int faces[4][3] = {{1, 2, 3}, {0, 3, 2}, {0, 1, 3}, {0, 2, 1}};
  for (const auto& el : elements)
    for (const auto& f : faces) {
      std::array<int, 3> key{el[f[0]], el[f[1]], el[f[2]]};
      std::sort(key.begin(), key.end());
      ++face_count[key];
    }
  std::vector<char> on(nv, 0);
  for (const auto& kv : face_count)
    if (kv.second == 1)
      for (int v : kv.first) on[v] = 1;
  for (int v = 0; v < nv; ++v)
    if (on[v]) m.boundary_.push_back(v);
  return m;
}

// mesh.cpp:100-140 — Kuhn 6-tet split, x-mirrored on odd cells.
TetMesh ingest_hex_grid(const std::array<int, 3>& dims, double spacing, double density) {
  const int nx = dims[0], ny = dims[1], nz = dims[2];
  if (nx < 1 || ny < 1 || nz < 1) fail(ErrorCode::Validation, "grid dims must be >= 1");
  if (spacing <= 0.0) fail(ErrorCode::Validation, "grid spacing must be positive");
  const int vx = nx + 1, vy = ny + 1, vz = nz + 1;
  VecX rest(3 * static_cast<size_t>(vx) * vy * vz);
  auto vid = [&](int i, int j, int k) { return i + vx * (j + vy * k); };
  for (int k = 0; k < vz; ++k)
    for (int j = 0; j < vy; ++j)
      for (int i = 0; i < vx; ++i) set3(rest, vid(i, j, k), Vec3(i * spacing, j * spacing, k * spacing));
  static const int kuhn[6][4] = {{0, 1, 3, 7}, {0, 3, 2, 7}, {0, 2, 6, 7}, {0, 6, 4, 7}, {0, 4, 5, 7}, {0, 5, 1, 7}};
  std::vector<std::array<int, 4>> elements;
  elements.reserve(static_cast<size_t>(nx) * ny * nz * 6);
  for (int k = 0; k < nz; ++k)
    for (int j = 0; j < ny; ++j)
      for (int i = 0; i < nx; ++i) {
        const bool mirror = ((i + j + k) & 1) != 0;
        int corner[8];
        for (int c = 0; c < 8; ++c) {
          int bx = c & 1, by = (c >> 1) & 1, bz = (c >> 2) & 1;
          if (mirror) bx = 1 - bx;
          corner[c] = vid(i + bx, j + by, k + bz);
        }
        for (const auto& t : kuhn) {
          std::array<int, 4> el{corner[t[0]], corner[t[1]], corner[t[2]], corner[t[3]]};
          Mat3 dm;
          for (int c = 0; c < 3; ++c) dm.set_col(c, seg3(rest, el[c + 1]) - seg3(rest, el[0]));
          if (dm.determinant() < 0.0) std::swap(el[2], el[3]);
          elements.push_back(el);
        }
      }
  return build_tet_mesh(rest, elements, density);
}

// mesh.cpp:142-151
Mat3 deformation_gradient(const TetMesh& mesh, int e, const VecX& q) {
  const auto& el = mesh.elements()[e];
  const Shape& g = mesh.shape_gradient(e);
  Mat3 f;
  for (int i = 0; i < 4; ++i) {
    const Vec3 x = seg3(q, el[i]);
    for (int r = 0; r < 3; ++r)
      for (int c = 0; c < 3; ++c) f(r, c) += x[r] * g.g[i][c];
  }
  return f;
}

// op^T * vec(P) scaled, op = element_operator (mesh.cpp:153-160):
// op(3c + r, 3i + r) = g(i, c)  =>  (op^T p)[3i + r] = sum_c g(i,c) P(r,c).
void element_force(const Shape& s, const Mat3& p, double scale, double out[12]) {
  for (int i = 0; i < 4; ++i)
    for (int r = 0; r < 3; ++r) {
      double acc = 0;
      for (int c = 0; c < 3; ++c) acc += s.g[i][c] * p(r, c);
      out[3 * i + r] = scale * acc;
    }
}

// ---- material.cpp ------------------------------------------------------------
// material.cpp:13-22
Lame lame_from_young_poisson(double young, double poisson) {
  if (young <= 0.0) fail(ErrorCode::Validation, "Young's modulus must be positive");
  if (!(poisson > -1.0 && poisson < 0.5))
    fail(ErrorCode::InvalidPoisson, "Poisson ratio must lie in (-1, 0.5), got " + std::to_string(poisson));
  Lame l;
  l.mu = young / (2.0 * (1.0 + poisson));
  l.lambda = young * poisson / ((1.0 + poisson) * (1.0 - 2.0 * poisson));
  return l;
}

// material.cpp:24-29
double nh_energy(const Mat3& f, double mu, double lambda) {
  const double j = f.determinant();
  if (j <= 0.0) fail(ErrorCode::NonPositiveJacobian, "nh_energy: det(F) <= 0");
  const double logj = std::log(j);
  return 0.5 * mu * (f.squaredNorm() - 3.0) - mu * logj + 0.5 * lambda * logj * logj;
}

double MaterialField::weight_contrast() const {
  double lo = total_weight(0), hi = lo;
  for (int e = 1; e < element_count(); ++e) {
    lo = std::min(lo, total_weight(e));
    hi = std::max(hi, total_weight(e));
  }
  return hi / lo;
}

void MaterialField::recompute(bool refresh_means) {
  const int ne = element_count();
  mu_.resize(ne);
  lambda_.resize(ne);
  beta_.resize(ne);
  double mu_ref = 0.0;
  for (int e = 0; e < ne; ++e) {
    const Lame l = lame_from_young_poisson(young_[e], poisson_);
    mu_[e] = l.mu;
    lambda_[e] = l.lambda;
    mu_ref = std::max(mu_ref, l.mu);
  }
  for (int e = 0; e < ne; ++e) beta_[e] = beta0_ * mu_[e] / mu_ref;
  if (refresh_means && !frozen_) {
    double vol = 0, ms = 0, ls = 0;
    for (int e = 0; e < ne; ++e) {
      vol += volume_[e];
      ms += volume_[e] * mu_[e];
      ls += volume_[e] * lambda_[e];
    }
    means_.mu = ms / vol;
    means_.lambda = ls / vol;
    means_.stiffness = 2.0 * means_.mu + means_.lambda;
  }
  version_ = g_material.fetch_add(1);
}

void MaterialField::set_young(const std::vector<double>& y) {
  if (static_cast<int>(y.size()) != element_count()) fail(ErrorCode::Validation, "set_young: element count mismatch");
  young_ = y;
  recompute(true);
}

void MaterialField::freeze_means(const ProxMeans& m) {
  means_ = m;
  frozen_ = true;
  version_ = g_material.fetch_add(1);
}

MaterialField build_material(const TetMesh& mesh, std::vector<double> young, double poisson, EnergyKind kind,
                             bool barrier, double alpha, double beta0) {
  if (static_cast<int>(young.size()) != mesh.element_count())
    fail(ErrorCode::Validation, "build_material: one Young's modulus per element required");
  if (alpha < 0.0 || beta0 < 0.0) fail(ErrorCode::Validation, "damping coefficients must be >= 0");
  if (barrier && kind != EnergyKind::Corotated)
    fail(ErrorCode::Validation, "log volume barrier composes with the corotated rotation step");
  MaterialField m;
  m.volume_.resize(mesh.element_count());
  for (int e = 0; e < mesh.element_count(); ++e) m.volume_[e] = mesh.volume(e);
  m.kind_ = kind;
  m.barrier_ = barrier;
  m.poisson_ = poisson;
  m.alpha_ = alpha;
  m.beta0_ = beta0;
  m.young_ = std::move(young);
  m.recompute(true);
  return m;
}

}  // namespace hdo
