// Drop-in check (TEST INFRASTRUCTURE): the same program text written twice,
// once against the reference's API (namespace phmat, /root/reference/proj,
// linked as oracle/_ref/libphmat_ref.so) and once against the product's C++
// facade (namespace phmat_b200, include/phmat_b200.hpp over
// libphmat_b200.so, GPU), with Eigen types on both sides (the Eigen API shim).
//
//  1. the reference builds a parametric H^2 (and H) matrix with its own
//     TT-cross and saves it (`phmat build --artifact`);
//  2. the facade loads that file onto the GPU (load_parametric_h2);
//  3. both instantiate at the same thetas through their LinearOperator and
//     apply to the same x; far_h[i], near_d[b], y, to_dense compared;
//  4. the facade's own offline_h2 on the same points: structure metrics equal
//     the reference's, and y agrees to the offline tolerance;
//  5. a theta outside the box throws std::domain_error on both sides.
// Prints one JSON line; exit status 0 iff every check holds.
#include <Eigen/Dense>

#include <cmath>
#include <cstdio>
#include <memory>
#include <string>
#include <vector>

#include "phmat/harness.hpp"
#include "phmat/phmatrix.hpp"
#include "phmat_b200.hpp"

namespace {

double rel(const Eigen::MatrixXd& a, const Eigen::MatrixXd& b) {
  const double nb = b.norm();
  return (a - b).norm() / (nb > 0 ? nb : 1.0);
}

template <typename PM_ref, typename PM_gpu>
bool compare(const std::shared_ptr<const PM_ref>& rpm, const std::shared_ptr<const PM_gpu>& gpm,
             const std::vector<double>& thetas, double& worst_block, double& worst_y, phmat_b200::StageCounters& gc) {
  bool ok = true;
  phmat::Rng rng(7);
  Eigen::VectorXd x(rpm->n());
  for (phmat::Index i = 0; i < x.size(); ++i) x[i] = rng.uniform(-1.0, 1.0);
  for (double th : thetas) {
    const std::vector<double> theta{th};
    const auto ri = phmat::instantiate(rpm, theta);
    const auto gi = phmat_b200::instantiate(gpm, theta, &gc.online);
    const phmat::LinearOperator& rop = ri;
    const phmat_b200::LinearOperator& gop = gi;
    ok = ok && rop.rows() == gop.rows();
    const double ey = rel(gop.apply(x), rop.apply(x));
    worst_y = std::max(worst_y, ey);
    for (std::size_t i = 0; i < ri.far_h.size(); i += 7)
      worst_block = std::max(worst_block, rel(gi.far_h[static_cast<phmat_b200::Index>(i)], ri.far_h[i]));
    for (std::size_t b = 0; b < ri.near_d.size(); b += 5)
      worst_block = std::max(worst_block, rel(gi.near_d[static_cast<phmat_b200::Index>(b)], ri.near_d[b]));
    worst_y = std::max(worst_y, rel(gi.to_dense(), ri.to_dense()));
  }
  return ok && worst_block <= 1e-12 && worst_y <= 1e-11;
}

}  // namespace

int main(int argc, char** argv) {
  const std::string dir = argc > 1 ? argv[1] : "/tmp";
  const Eigen::MatrixXd points = phmat::generate_points(1500, 3, 11);
  phmat::PHConfig rc;
  rc.spec = phmat::default_kernel_spec(phmat::KernelFamily::SquaredExponential);
  rc.l_max = 2;
  rc.p_s = 4;
  rc.p_theta = 6;
  rc.eps = 1e-6;
  rc.eta = 1.0;
  rc.near_mode = phmat::NearMode::TT;
  phmat::StageCounters rcnt;
  auto rpm2 = std::make_shared<phmat::ParametricH2Matrix>(phmat::offline_h2(points, rc, rcnt));
  auto rpm1 = std::make_shared<phmat::ParametricHMatrix>(phmat::offline_h(points, rc, rcnt));
  const std::string p2 = dir + "/dropin_h2.hmat", p1 = dir + "/dropin_h.hmat";
  phmat::save_parametric(*rpm2, p2);
  phmat::save_parametric(*rpm1, p1);

  phmat_b200::StageCounters gc;
  auto gpm2 = std::make_shared<phmat_b200::ParametricH2Matrix>(phmat_b200::load_parametric_h2(p2));
  auto gpm1 = std::make_shared<phmat_b200::ParametricHMatrix>(phmat_b200::load_parametric_h(p1));
  const std::vector<double> thetas{0.25, 0.5314, 1.0};
  double wb2 = 0, wy2 = 0, wb1 = 0, wy1 = 0;
  const bool ok2 = compare(std::shared_ptr<const phmat::ParametricH2Matrix>(rpm2),
                           std::shared_ptr<const phmat_b200::ParametricH2Matrix>(gpm2), thetas, wb2, wy2, gc);
  const bool ok1 = compare(std::shared_ptr<const phmat::ParametricHMatrix>(rpm1),
                           std::shared_ptr<const phmat_b200::ParametricHMatrix>(gpm1), thetas, wb1, wy1, gc);

  // the facade's own offline build (snapshot near field) on the same points
  phmat_b200::PHConfig gcfg;
  gcfg.spec = phmat_b200::default_kernel_spec(phmat_b200::KernelFamily::SquaredExponential);
  gcfg.l_max = rc.l_max;
  gcfg.p_s = rc.p_s;
  gcfg.p_theta = rc.p_theta;
  gcfg.eps = rc.eps;
  gcfg.eta = rc.eta;
  gcfg.near_mode = phmat_b200::NearMode::Snapshot;
  auto own = std::make_shared<phmat_b200::ParametricH2Matrix>(phmat_b200::offline_h2(points, gcfg, gc));
  const auto gm = phmat_b200::metrics(*own);
  const auto rm = phmat::metrics(*rpm2);
  const bool struct_ok = gm.n_near == rm.n_near && gm.n_far == rm.n_far && gm.m_a == rm.m_a && gm.c_sp == rm.c_sp;
  const std::vector<double> th{0.5314};
  Eigen::VectorXd x = Eigen::VectorXd::Constant(1500, 1.0);
  const double e_own = rel(phmat_b200::instantiate(std::shared_ptr<const phmat_b200::ParametricH2Matrix>(own), th)
                               .apply(x),
                           phmat::instantiate(std::shared_ptr<const phmat::ParametricH2Matrix>(rpm2), th).apply(x));

  bool dom_ref = false, dom_gpu = false;
  try {
    phmat::instantiate(std::shared_ptr<const phmat::ParametricH2Matrix>(rpm2), std::vector<double>{2.0});
  } catch (const std::domain_error&) {
    dom_ref = true;
  }
  try {
    phmat_b200::instantiate(std::shared_ptr<const phmat_b200::ParametricH2Matrix>(gpm2), std::vector<double>{2.0});
  } catch (const std::domain_error&) {
    dom_gpu = true;
  }
  bool len_gpu = false;
  try {
    phmat_b200::instantiate(std::shared_ptr<const phmat_b200::ParametricH2Matrix>(gpm2), th).apply(Eigen::VectorXd(7));
  } catch (const std::invalid_argument&) {
    len_gpu = true;
  }
  const bool ok = ok1 && ok2 && struct_ok && e_own <= 1e-4 && dom_ref && dom_gpu && len_gpu &&
                  gc.online.value() == 0 && gc.offline.value() > 0;
  std::printf(
      "{\"ok\": %s, \"h2_block\": %.3e, \"h2_y\": %.3e, \"h_block\": %.3e, \"h_y\": %.3e, \"own_build_y\": %.3e, "
      "\"structure_equal\": %s, \"domain_error\": [%s, %s], \"length_error\": %s, \"online_evals\": %llu}\n",
      ok ? "true" : "false", wb2, wy2, wb1, wy1, e_own, struct_ok ? "true" : "false", dom_ref ? "true" : "false",
      dom_gpu ? "true" : "false", len_gpu ? "true" : "false", static_cast<unsigned long long>(gc.online.value()));
  return ok ? 0 : 1;
}
