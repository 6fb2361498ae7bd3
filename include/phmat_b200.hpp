// phmat_b200.hpp — header-only C++ facade over the C ABI (phmat_b200.h) with
// the reference's names and exception types, so code written against
// proj/include/phmat/phmatrix.hpp switches by changing the include and
// namespace:
//
//   reference (phmatrix.hpp)                      here
//   ------------------------                      ----
//   phmat::PHConfig                               phmat_b200::PHConfig
//   phmat::offline_h2(points, cfg, counters)      phmat_b200::offline_h2(points, n, d, cfg)
//   phmat::instantiate(pm, theta)                 phmat_b200::instantiate(pm, theta)
//   LinearOperator::apply(x)                      InstantiatedMatrix::apply(x)
//   far_h[i] / near_d[i] / to_dense()             far_h(i) / near_d(i) / to_dense()
//   std::domain_error / invalid_argument / ...    same types, thrown from status codes
//
// Vectors are std::vector<double> (the reference uses Eigen::VectorXd; an
// Eigen user passes v.data() / v.size()). Point sets are n x d row-major.
#pragma once

#include <cstdint>
#include <memory>
#include <stdexcept>
#include <string>
#include <vector>

#include "phmat_b200.h"

namespace phmat_b200 {

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

// PHConfig (phmatrix.hpp:20-35) with the reference defaults.
struct PHConfig {
  phm_config c;
  PHConfig() { phm_config_default(&c); }
};

class Context {
 public:
  explicit Context(int device = 0) {
    phm_context h = nullptr;
    check(phm_context_create(device, &h));
    h_.reset(h, [](phm_context p) { phm_context_destroy(p); });
  }
  phm_context get() const { return h_.get(); }

 private:
  std::shared_ptr<phm_context_s> h_;
};

class ParametricMatrix {
 public:
  ParametricMatrix(phm_matrix h, Context ctx) : ctx_(std::move(ctx)) {
    h_.reset(h, [](phm_matrix p) { phm_matrix_destroy(p); });
  }
  phm_matrix get() const { return h_.get(); }
  phm_info info() const {
    phm_info i;
    check(phm_matrix_info(h_.get(), &i));
    return i;
  }
  std::int64_t n() const { return info().n; }

 private:
  Context ctx_;
  std::shared_ptr<phm_matrix_s> h_;
};

// offline_h / offline_h2 (phmatrix.hpp:82-91): tree over the unit box.
inline ParametricMatrix offline(const double* points, std::int64_t n, int d, PHConfig cfg, int format,
                                Context ctx = Context()) {
  cfg.c.format = format;
  phm_matrix h = nullptr;
  check(phm_matrix_build(ctx.get(), points, n, d, &cfg.c, &h));
  return ParametricMatrix(h, ctx);
}
inline ParametricMatrix offline_h(const double* p, std::int64_t n, int d, const PHConfig& cfg,
                                  Context ctx = Context()) {
  return offline(p, n, d, cfg, PHM_FORMAT_H, ctx);
}
inline ParametricMatrix offline_h2(const double* p, std::int64_t n, int d, const PHConfig& cfg,
                                   Context ctx = Context()) {
  return offline(p, n, d, cfg, PHM_FORMAT_H2, ctx);
}

// Instantiated{H,H2}Matrix (phmatrix.hpp:102-128): a LinearOperator.
class InstantiatedMatrix {
 public:
  InstantiatedMatrix(ParametricMatrix parent, phm_instance h) : parent_(std::move(parent)) {
    h_.reset(h, [](phm_instance p) { phm_instance_destroy(p); });
  }
  std::int64_t rows() const { return parent_.n(); }
  std::vector<double> apply(const std::vector<double>& x) const {
    std::vector<double> y(static_cast<size_t>(rows()));
    check(phm_apply(h_.get(), x.data(), static_cast<std::int64_t>(x.size()), y.data(), 1));
    return y;
  }
  std::vector<double> far_h(std::int64_t i, std::int64_t* r = nullptr, std::int64_t* c = nullptr) const {
    std::int64_t rr = 0, cc = 0;
    check(phm_instance_far_h(h_.get(), i, nullptr, &rr, &cc));
    std::vector<double> out(static_cast<size_t>(rr * cc));
    check(phm_instance_far_h(h_.get(), i, out.data(), nullptr, nullptr));
    if (r) *r = rr;
    if (c) *c = cc;
    return out;
  }
  std::vector<double> to_dense(std::int64_t guard = 8192) const {
    std::vector<double> out(static_cast<size_t>(rows() * rows()));
    check(phm_to_dense(h_.get(), out.data(), guard));
    return out;
  }
  phm_instance get() const { return h_.get(); }

 private:
  ParametricMatrix parent_;
  std::shared_ptr<phm_instance_s> h_;
};

// instantiate(pm, theta) (phmatrix.hpp:133-138).
inline InstantiatedMatrix instantiate(const ParametricMatrix& pm, const std::vector<double>& theta) {
  phm_instance h = nullptr;
  check(phm_instantiate(pm.get(), theta.data(), static_cast<int>(theta.size()), &h));
  return InstantiatedMatrix(pm, h);
}

}  // namespace phmat_b200
