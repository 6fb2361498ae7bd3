// phmat_b200.hpp — header-only C++ drop-in for the reference's public API
// (proj/include/phmat/phmatrix.hpp, kernels.hpp:47-62) over the C ABI
// (phmat_b200.h). Code written against the reference switches by changing
// the include and the namespace:
//
//   reference (phmatrix.hpp)                         here (namespace phmat_b200)
//   ------------------------                         --------------------------
//   PHConfig, KernelSpec, NearMode (:18-35)          same names and defaults (+ Snapshot mode,
//                                                    per-dim p_theta, amplitude, sharding)
//   StageCounters / KernelEvalCounter (kernels.hpp)  same (offline / online / audit tallies)
//   offline_h / offline_h2(points, cfg, counters)    same signatures (:82-91); GPU resident
//   LinearOperator { rows(); apply(x) } (:95-100)    same interface
//   InstantiatedHMatrix / InstantiatedH2Matrix       LinearOperators with parent, theta,
//     (:102-128)                                     far_h[i] / near_d[i] (device -> host on
//                                                    access), to_dense(guard), online_entries_*
//   instantiate(shared_ptr<const PM>, span theta,    same (:133-138); the counter receives the
//               KernelEvalCounter*)                  online kernel evaluations (0 in TT /
//                                                    snapshot mode, as the reference)
//   metrics / StructureMetrics (:141-156)            same
//   save_parametric / load_parametric_h / _h2 /      same (:158-164), HMAT v1
//     artifact_is_h2
//   std::domain_error / invalid_argument /           same types, thrown from the status codes
//     logic_error / runtime_error
//
// Vectors and matrices: Eigen::VectorXd / Eigen::MatrixXd when Eigen is
// included first (EIGEN_WORLD_VERSION defined), exactly as the reference;
// otherwise the minimal column-major phmat_b200::Vector / Matrix below.
// Points are n x d (row i = point i) in both cases.
#pragma once

#include <cmath>
#include <cstdint>
#include <cstring>
#include <memory>
#include <span>
#include <stdexcept>
#include <string>
#include <vector>

#include "phmat_b200.h"

namespace phmat_b200 {

using Index = std::int64_t;

inline void check(int code) {
  if (code == PHM_OK) return;
  const std::string msg = phm_last_error();
  switch (code) {
    case PHM_ERR_DOMAIN: throw std::domain_error(msg);
    case PHM_ERR_INVALID: throw std::invalid_argument(msg);
    case PHM_ERR_RANGE: throw std::out_of_range(msg);
    case PHM_ERR_LOGIC: throw std::logic_error(msg);
    default: throw std::runtime_error(msg);
  }
}

// ------------------------------------------------------------ vector types
#ifdef EIGEN_WORLD_VERSION
using Vector = Eigen::VectorXd;
using Matrix = Eigen::MatrixXd;
inline Matrix make_matrix(Index r, Index c) { return Matrix::Zero(r, c); }
#else
// Column-major dense storage with the Eigen calls the reference's callers use.
class Matrix {
 public:
  Matrix() = default;
  Matrix(Index r, Index c) : r_(r), c_(c), a_(static_cast<size_t>(r * c), 0.0) {}
  Index rows() const { return r_; }
  Index cols() const { return c_; }
  Index size() const { return r_ * c_; }
  double* data() { return a_.data(); }
  const double* data() const { return a_.data(); }
  double& operator()(Index i, Index j) { return a_[static_cast<size_t>(i + j * r_)]; }
  double operator()(Index i, Index j) const { return a_[static_cast<size_t>(i + j * r_)]; }

 private:
  Index r_ = 0, c_ = 0;
  std::vector<double> a_;
};
class Vector {
 public:
  Vector() = default;
  explicit Vector(Index n) : a_(static_cast<size_t>(n), 0.0) {}
  Index size() const { return static_cast<Index>(a_.size()); }
  double* data() { return a_.data(); }
  const double* data() const { return a_.data(); }
  double& operator[](Index i) { return a_[static_cast<size_t>(i)]; }
  double operator[](Index i) const { return a_[static_cast<size_t>(i)]; }
  double& operator()(Index i) { return a_[static_cast<size_t>(i)]; }
  double operator()(Index i) const { return a_[static_cast<size_t>(i)]; }

 private:
  std::vector<double> a_;
};
inline Matrix make_matrix(Index r, Index c) { return Matrix(r, c); }
#endif

// ------------------------------------------------------------------ config
// KernelFamily (kernels.hpp:21) + the single-parameter families of SURVEY.md
// Appendix A.
enum class KernelFamily {
  Exponential = PHM_KERNEL_E,
  ThinPlateSpline = PHM_KERNEL_TPS,
  SquaredExponential = PHM_KERNEL_SE,
  Multiquadric = PHM_KERNEL_MC,
  Matern = PHM_KERNEL_MN,
  Gaussian = PHM_KERNEL_GAUSS,
  Matern32 = PHM_KERNEL_MATERN32,
  Matern52 = PHM_KERNEL_MATERN52
};

struct Interval {
  double lo = 0.0;
  double hi = 0.0;
  double width() const { return hi - lo; }
  bool contains(double x) const { return x >= lo && x <= hi; }
};

// KernelSpec (kernels.hpp:31-38); amplitude: trailing sigma^2 parameter.
struct KernelSpec {
  KernelFamily family = KernelFamily::SquaredExponential;
  std::vector<Interval> theta_box;
  bool amplitude = false;
  int d_theta() const { return static_cast<int>(theta_box.size()); }
};

// default_kernel_spec (kernels.cpp:41-47).
inline KernelSpec default_kernel_spec(KernelFamily family) {
  KernelSpec s;
  s.family = family;
  s.theta_box = {{0.25, 1.0}};
  if (family == KernelFamily::Matern) s.theta_box.push_back({0.5, 3.0});
  return s;
}

enum class NearMode { TT = PHM_NEAR_TT, Direct = PHM_NEAR_DIRECT, Snapshot = PHM_NEAR_SNAPSHOT };

// PHConfig (phmatrix.hpp:20-35), reference defaults, plus the B200 fields.
struct PHConfig {
  KernelSpec spec;
  int l_max = 2;
  int p_s = 15;
  int p_theta = 27;
  std::vector<int> p_theta_per_dim;  // optional: one p_theta per theta dimension
  double eps = 1e-5;
  double eta = 0.0;
  Index r_max_far = 120;
  Index r_max_near = 150;
  std::uint64_t seed = 0;
  NearMode near_mode = NearMode::TT;
  bool translation_cache = true;
  int threads = 0;
  // B200 extensions
  int shard_rank = 0, shard_count = 1;
  bool symmetric_near = true;

  double resolved_eta(int d) const;

  phm_config to_c(int format) const {
    phm_config c;
    phm_config_default(&c);
    c.family = static_cast<int32_t>(spec.family);
    c.amplitude = spec.amplitude ? 1 : 0;
    c.d_theta = spec.d_theta();
    for (int k = 0; k < c.d_theta && k < 3; ++k) {
      c.theta_lo[k] = spec.theta_box[k].lo;
      c.theta_hi[k] = spec.theta_box[k].hi;
      c.p_theta[k] = p_theta_per_dim.empty() ? p_theta : p_theta_per_dim[k];
    }
    c.format = format;
    c.l_max = l_max;
    c.p_s = p_s;
    c.near_mode = static_cast<int32_t>(near_mode);
    c.eps = eps;
    c.eta = eta;
    c.r_max_far = r_max_far;
    c.r_max_near = r_max_near;
    c.seed = seed;
    c.translation_cache = translation_cache ? 1 : 0;
    c.threads = threads;
    c.shard_rank = shard_rank;
    c.shard_count = shard_count;
    c.symmetric_near = symmetric_near ? 1 : 0;
    return c;
  }
  static PHConfig from_c(const phm_config& c) {
    PHConfig p;
    p.spec.family = static_cast<KernelFamily>(c.family);
    p.spec.amplitude = c.amplitude != 0;
    for (int k = 0; k < c.d_theta; ++k) p.spec.theta_box.push_back({c.theta_lo[k], c.theta_hi[k]});
    p.p_theta = c.p_theta[0];
    for (int k = 0; k < c.d_theta; ++k) p.p_theta_per_dim.push_back(c.p_theta[k]);
    p.l_max = c.l_max;
    p.p_s = c.p_s;
    p.near_mode = static_cast<NearMode>(c.near_mode);
    p.eps = c.eps;
    p.eta = c.eta;
    p.r_max_far = c.r_max_far;
    p.r_max_near = c.r_max_near;
    p.seed = c.seed;
    p.translation_cache = c.translation_cache != 0;
    p.threads = c.threads;
    p.shard_rank = c.shard_rank;
    p.shard_count = c.shard_count;
    p.symmetric_near = c.symmetric_near != 0;
    return p;
  }
};

inline double PHConfig::resolved_eta(int d) const { return eta > 0.0 ? eta : std::sqrt(double(d)); }

// KernelEvalCounter / StageCounters (kernels.hpp:47-62).
class KernelEvalCounter {
 public:
  void add(std::uint64_t k = 1) noexcept { n_ += k; }
  std::uint64_t value() const noexcept { return n_; }
  void reset() noexcept { n_ = 0; }

 private:
  std::uint64_t n_ = 0;
};
struct StageCounters {
  KernelEvalCounter offline;
  KernelEvalCounter online;
  KernelEvalCounter baseline;
  KernelEvalCounter audit;
};

// StructureMetrics (phmatrix.hpp:141-153).
struct StructureMetrics {
  Index n = 0;
  Index storage_entries = 0;
  double storage_gb = 0.0;
  double nf_ratio = 0.0;
  double ff_ratio = 0.0;
  double coupling_ratio = 0.0;
  double rank = 0.0;
  Index c_sp = 0;
  Index m_a = 0;
  Index n_far = 0;
  Index n_near = 0;
};

// generate_points (harness.hpp:77-78, harness.cpp:174-181): the reference's
// seeded U[0,1)^d stream, n x d.
inline Matrix generate_points(Index n, int d, std::uint64_t seed) {
  std::vector<double> p(static_cast<size_t>(n * d));
  check(phm_generate_points(n, d, seed, p.data()));
  Matrix out = make_matrix(n, d);
  for (Index i = 0; i < n; ++i)
    for (int k = 0; k < d; ++k) out(i, k) = p[static_cast<size_t>(i * d + k)];
  return out;
}

// ----------------------------------------------------------------- context
// One CUDA device + stream; shared by every matrix built on it.
class Context {
 public:
  explicit Context(int device = 0) {
    phm_context h = nullptr;
    check(phm_context_create(device, &h));
    h_.reset(h, [](phm_context p) { phm_context_destroy(p); });
  }
  phm_context get() const { return h_.get(); }
  // the process-wide default context on device 0
  static Context& default_context() {
    static Context ctx(0);
    return ctx;
  }

 private:
  std::shared_ptr<phm_context_s> h_;
};

// ------------------------------------------------------- parametric matrix
// Common part of ParametricHMatrix / ParametricH2Matrix (phmatrix.hpp:38-80):
// the offline data lives on the GPU; structure views copy to the host.
class ParametricMatrix {
 public:
  ParametricMatrix(phm_matrix h, Context ctx) : ctx_(std::move(ctx)) {
    h_.reset(h, [](phm_matrix p) { phm_matrix_destroy(p); });
    phm_config c;
    check(phm_matrix_config(h_.get(), &c));
    config = PHConfig::from_c(c);
  }
  virtual ~ParametricMatrix() = default;
  PHConfig config;

  phm_matrix get() const { return h_.get(); }
  const Context& context() const { return ctx_; }
  phm_info info() const {
    phm_info i;
    check(phm_matrix_info(h_.get(), &i));
    return i;
  }
  Index n() const { return info().n; }
  int d() const { return static_cast<int>(info().d); }
  bool is_h2() const { return config_format() == PHM_FORMAT_H2; }
  // the tree-order permutation (leaf index sets in leaf-id order)
  std::vector<std::int32_t> perm() const {
    std::vector<std::int32_t> p(static_cast<size_t>(n()));
    check(phm_matrix_perm(h_.get(), p.data()));
    return p;
  }

 protected:
  int config_format() const {
    phm_config c;
    check(phm_matrix_config(h_.get(), &c));
    return c.format;
  }

 private:
  Context ctx_;
  std::shared_ptr<phm_matrix_s> h_;
};

struct ParametricHMatrix : ParametricMatrix {
  using ParametricMatrix::ParametricMatrix;
};
struct ParametricH2Matrix : ParametricMatrix {
  using ParametricMatrix::ParametricMatrix;
};

namespace detail {
template <typename M>
inline std::vector<double> points_row_major(const M& points, Index& n, int& d) {
  n = static_cast<Index>(points.rows());
  d = static_cast<int>(points.cols());
  std::vector<double> p(static_cast<size_t>(n * d));
  for (Index i = 0; i < n; ++i)
    for (int k = 0; k < d; ++k) p[static_cast<size_t>(i * d + k)] = points(i, k);
  return p;
}
template <typename PM>
inline PM build(const double* pts, Index n, int d, const PHConfig& cfg, int format, StageCounters& counters,
                const Context& ctx) {
  const phm_config c = cfg.to_c(format);
  phm_matrix h = nullptr;
  check(phm_matrix_build(ctx.get(), pts, n, d, &c, &h));
  PM pm(h, ctx);
  counters.offline.add(pm.info().evals_offline);
  return pm;
}
}  // namespace detail

// offline_h / offline_h2 (phmatrix.hpp:82-91): tree over the unit box; the
// offline kernel evaluations are added to counters.offline.
template <typename Points>
inline ParametricHMatrix offline_h(const Points& points, const PHConfig& config, StageCounters& counters,
                                   const Context& ctx = Context::default_context()) {
  Index n;
  int d;
  const auto p = detail::points_row_major(points, n, d);
  return detail::build<ParametricHMatrix>(p.data(), n, d, config, PHM_FORMAT_H, counters, ctx);
}
template <typename Points>
inline ParametricH2Matrix offline_h2(const Points& points, const PHConfig& config, StageCounters& counters,
                                     const Context& ctx = Context::default_context()) {
  Index n;
  int d;
  const auto p = detail::points_row_major(points, n, d);
  return detail::build<ParametricH2Matrix>(p.data(), n, d, config, PHM_FORMAT_H2, counters, ctx);
}

// ---------------------------------------------------------- linear operator
// LinearOperator (phmatrix.hpp:95-100).
class LinearOperator {
 public:
  virtual ~LinearOperator() = default;
  virtual Index rows() const = 0;
  virtual Vector apply(const Vector& x) const = 0;
};

class InstantiatedMatrix;

// far_h[i] / near_d[i] of the reference (public vector<MatrixXd> members,
// phmatrix.hpp:105-106, 119-120): views that copy one block device -> host.
class FarHView {
 public:
  explicit FarHView(const InstantiatedMatrix* m) : m_(m) {}
  Matrix operator[](Index i) const;
  Index size() const;

 private:
  const InstantiatedMatrix* m_;
};
class NearDView {
 public:
  explicit NearDView(const InstantiatedMatrix* m) : m_(m) {}
  Matrix operator[](Index b) const;
  Index size() const;

 private:
  const InstantiatedMatrix* m_;
};

// Instantiated{H,H2}Matrix (phmatrix.hpp:102-128).
class InstantiatedMatrix : public LinearOperator {
 public:
  InstantiatedMatrix(std::shared_ptr<const ParametricMatrix> p, phm_instance h, std::vector<double> th)
      : parent(std::move(p)), theta(std::move(th)), far_h(this), near_d(this) {
    h_.reset(h, [](phm_instance q) { phm_instance_destroy(q); });
  }
  InstantiatedMatrix(const InstantiatedMatrix& o)
      : LinearOperator(o), parent(o.parent), theta(o.theta), far_h(this), near_d(this), h_(o.h_) {}
  InstantiatedMatrix& operator=(const InstantiatedMatrix& o) {
    parent = o.parent;
    theta = o.theta;
    h_ = o.h_;
    return *this;
  }

  std::shared_ptr<const ParametricMatrix> parent;
  std::vector<double> theta;
  FarHView far_h;
  NearDView near_d;

  Index rows() const override { return parent->n(); }
  // y = K(theta) x (phmatrix.cpp:227-269), original point order
  Vector apply(const Vector& x) const override {
    Vector y(rows());
    check(phm_apply(h_.get(), x.data(), static_cast<Index>(x.size()), y.data(), 1));
    return y;
  }
  // block right-hand sides (n x m, column-major): the DMMA near field
  Matrix apply_block(const Matrix& X) const {
    Matrix Y = make_matrix(rows(), X.cols());
    check(phm_apply(h_.get(), X.data(), static_cast<Index>(X.rows()), Y.data(), static_cast<Index>(X.cols())));
    return Y;
  }
  // instantiate(theta') + apply(x) as one overlapped GPU step (the HPO step)
  Vector instantiate_apply(std::span<const double> th, const Vector& x) {
    Vector y(rows());
    check(phm_instantiate_apply(h_.get(), th.data(), static_cast<int>(th.size()), x.data(),
                                static_cast<Index>(x.size()), y.data(), 1));
    theta.assign(th.begin(), th.end());
    return y;
  }
  Matrix to_dense(Index guard = 8192) const {
    const Index n = rows();
    if (n > guard) throw std::runtime_error("to_dense: matrix exceeds the size guard");
    Matrix out = make_matrix(n, n);
    check(phm_to_dense(h_.get(), out.data(), guard));
    return out;
  }
  // online_entries_far / _near (phmatrix.cpp:319-340): stored online entries
  Index online_entries_near() const { return parent->info().near_entries; }
  Index online_entries_far() const {
    Index s = 0;
    const Index nf = parent->info().n_far;
    for (Index i = 0; i < nf; ++i) {
      Index r = 0, c = 0;
      check(phm_instance_far_h(h_.get(), i, nullptr, &r, &c));
      s += r * c;
    }
    return s;
  }
  phm_instance get() const { return h_.get(); }

 private:
  std::shared_ptr<phm_instance_s> h_;
};

struct InstantiatedHMatrix : InstantiatedMatrix {
  using InstantiatedMatrix::InstantiatedMatrix;
};
struct InstantiatedH2Matrix : InstantiatedMatrix {
  using InstantiatedMatrix::InstantiatedMatrix;
};

inline Matrix FarHView::operator[](Index i) const {
  Index r = 0, c = 0;
  check(phm_instance_far_h(m_->get(), i, nullptr, &r, &c));
  Matrix out = make_matrix(r, c);
  check(phm_instance_far_h(m_->get(), i, out.data(), nullptr, nullptr));
  return out;
}
inline Index FarHView::size() const { return m_->parent->info().n_far; }

inline Matrix NearDView::operator[](Index b) const {
  const phm_info inf = m_->parent->info();
  std::vector<std::int32_t> near(static_cast<size_t>(2 * inf.n_near)), far(static_cast<size_t>(2 * inf.n_far)),
      key(static_cast<size_t>(inf.n_far));
  check(phm_matrix_blocks(m_->parent->get(), near.data(), far.data(), key.data()));
  std::vector<std::int32_t> ints(static_cast<size_t>(7 * inf.nodes));
  std::vector<double> boxes(static_cast<size_t>(6 * inf.nodes));
  check(phm_matrix_nodes(m_->parent->get(), ints.data(), boxes.data()));
  const Index ns = ints[static_cast<size_t>(7 * near[2 * b] + 3)], nt = ints[static_cast<size_t>(7 * near[2 * b + 1] + 3)];
  Matrix out = make_matrix(ns, nt);
  check(phm_instance_near_d(m_->get(), b, out.data()));
  return out;
}
inline Index NearDView::size() const { return m_->parent->info().n_near; }

namespace detail {
template <typename Inst>
inline Inst instantiate(std::shared_ptr<const ParametricMatrix> pm, std::span<const double> theta,
                        KernelEvalCounter* counter) {
  const std::uint64_t before = pm->info().evals_online;
  phm_instance h = nullptr;
  check(phm_instantiate(pm->get(), theta.data(), static_cast<int>(theta.size()), &h));
  if (counter) counter->add(pm->info().evals_online - before);
  return Inst(std::move(pm), h, std::vector<double>(theta.begin(), theta.end()));
}
}  // namespace detail

// instantiate (phmatrix.hpp:133-138): zero kernel evaluations in TT and
// snapshot near mode; Direct mode charges one per near entry to `counter`.
inline InstantiatedHMatrix instantiate(std::shared_ptr<const ParametricHMatrix> pm, std::span<const double> theta,
                                       KernelEvalCounter* counter = nullptr) {
  return detail::instantiate<InstantiatedHMatrix>(std::move(pm), theta, counter);
}
inline InstantiatedH2Matrix instantiate(std::shared_ptr<const ParametricH2Matrix> pm, std::span<const double> theta,
                                        KernelEvalCounter* counter = nullptr) {
  return detail::instantiate<InstantiatedH2Matrix>(std::move(pm), theta, counter);
}

// metrics (phmatrix.hpp:155-156).
inline StructureMetrics metrics(const ParametricMatrix& pm) {
  const phm_info i = pm.info();
  StructureMetrics m;
  m.n = i.n;
  m.storage_entries = i.storage_entries;
  m.storage_gb = i.storage_gb;
  m.nf_ratio = i.nf_ratio;
  m.ff_ratio = i.ff_ratio;
  m.coupling_ratio = i.coupling_ratio;
  m.rank = i.rank;
  m.c_sp = i.c_sp;
  m.m_a = i.n_classes;
  m.n_far = i.n_far;
  m.n_near = i.n_near;
  return m;
}

// save_parametric / load_parametric_h / _h2 / artifact_is_h2
// (phmatrix.hpp:158-164): HMAT v1, byte-compatible with the reference.
inline void save_parametric(const ParametricMatrix& pm, const std::string& path) {
  check(phm_matrix_save(pm.get(), path.c_str()));
}
inline bool artifact_is_h2(const std::string& path) {
  int v = 0;
  check(phm_artifact_is_h2(path.c_str(), &v));
  return v != 0;
}
inline ParametricHMatrix load_parametric_h(const std::string& path,
                                           const Context& ctx = Context::default_context()) {
  if (artifact_is_h2(path)) throw std::runtime_error("artifact holds the other matrix format");
  phm_matrix h = nullptr;
  check(phm_matrix_load(ctx.get(), path.c_str(), 0, &h));
  return ParametricHMatrix(h, ctx);
}
inline ParametricH2Matrix load_parametric_h2(const std::string& path,
                                             const Context& ctx = Context::default_context()) {
  if (!artifact_is_h2(path)) throw std::runtime_error("artifact holds the other matrix format");
  phm_matrix h = nullptr;
  check(phm_matrix_load(ctx.get(), path.c_str(), 0, &h));
  return ParametricH2Matrix(h, ctx);
}

}  // namespace phmat_b200
