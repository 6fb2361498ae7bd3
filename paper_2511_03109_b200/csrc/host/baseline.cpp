// Non-parametric baselines of the reference (proj/src/baselines.cpp): an
// H-matrix with ACA far blocks (H-ACA) and an H^2-matrix whose couplings are
// ACA factorisations of the Chebyshev node-interaction matrices (H^2-HCA),
// both built at one fixed theta. The host side restates their construction;
// the device side reuses the parametric engine's apply unchanged (H form:
// S_b = V_b, H_b = I, T_b = Y_b; H^2 form: C_k = V_k Y_k^T, shared basis),
// with the dense near blocks evaluated on the GPU (Direct near mode).
#include <chrono>
#include <cmath>
#include <map>

#include "phm.hpp"

namespace phm {

namespace {
constexpr double kPi = 3.141592653589793238462643383279502884;  // std::numbers::pi
double now_s() {
  return std::chrono::duration<double>(std::chrono::steady_clock::now().time_since_epoch()).count();
}
}  // namespace

std::unique_ptr<HostMatrix> build_baseline_host(const double* points, Index n, int d, const Config& cfg_in,
                                                Baseline method, const double* theta, int n_theta, double eps,
                                                Index r_max) {
  PHM_CHECK(method == Baseline::HAca || method == Baseline::H2Hca, "unknown baseline");
  PHM_CHECK(eps > 0.0, "baseline: eps must be positive");
  cfg_in.spec.validate();
  PHM_CHECK(n_theta == cfg_in.spec.d_theta(), "baseline: theta length must match the kernel's parameters");
  auto hm = std::make_unique<HostMatrix>();
  HostMatrix& M = *hm;
  M.cfg = cfg_in;
  M.cfg.format = method == Baseline::HAca ? Format::H : Format::H2;
  M.cfg.near_mode = NearMode::Direct;
  M.cfg.shard_rank = 0;
  M.cfg.shard_count = 1;
  M.cfg.symmetric_near = false;
  const Config& cfg = M.cfg;
  const double t0 = now_s();
  Box root;
  root.d = d;
  for (int k = 0; k < d; ++k) {
    root.lo[k] = 0.0;
    root.hi[k] = 1.0;
  }
  M.tree = std::make_unique<Tree>(points, n, d, root, cfg.l_max);
  const Tree& T = *M.tree;
  M.blocks = build_blocks(T, cfg.resolved_eta(d));
  M.grids = make_theta_grids(cfg.spec, cfg.p_theta);
  M.stats.tree_s = now_s() - t0;
  M.row_begin = 0;
  M.row_end = T.n;
  M.node_local.assign(T.nodes.size(), 1);
  M.near_local.assign(M.blocks.near.size(), 1);
  M.far_local.assign(M.blocks.far.size(), 1);

  BaselineData& B = M.baseline;
  B.method = method;
  B.theta.assign(theta, theta + n_theta);
  const std::vector<double> th = B.theta;
  const double t1 = now_s();
  EvalCounter far_evals;
  if (method == Baseline::HAca) {
    // one ACA per far block on kernel entries (baselines.cpp:63-87)
    const Index nf = static_cast<Index>(M.blocks.far.size());
    M.far_s.resize(nf);
    M.far_t.resize(nf);
    std::vector<char> capped(nf, 0);
    parallel_for(
        nf,
        [&](Index i) {
          const Block b = M.blocks.far[i];
          const TreeNode& sn = T.nodes[b.sigma];
          const TreeNode& tn = T.nodes[b.tau];
          auto entry = [&](Index r, Index c) {
            const Index oi = T.perm[sn.begin + r], oj = T.perm[tn.begin + c];
            double r2 = 0.0;
            for (int k = 0; k < d; ++k) {
              const double delta = T.coord(oi, k) - T.coord(oj, k);
              r2 += delta * delta;
            }
            far_evals.add();
            return kernel_value(cfg.spec, std::sqrt(r2), th.data());
          };
          Rng rng(mix_seed(0x61636121ULL, static_cast<std::uint64_t>(i)));
          LowRank f = aca_partial_rng(entry, sn.count, tn.count, eps, r_max, rng);
          capped[i] = f.capped;
          M.far_s[i] = std::move(f.v);
          M.far_t[i] = std::move(f.y);
        },
        cfg.threads);
    // every far block is its own class with H_b = I_t
    M.far_key.resize(nf);
    M.class_rep.resize(nf);
    M.class_keys.resize(nf);
    double sum_rank = 0.0;
    for (Index i = 0; i < nf; ++i) {
      M.far_key[i] = static_cast<int>(i);
      M.class_rep[i] = static_cast<int>(i);
      const Index t = M.far_s[i].cols;
      B.rank.push_back(static_cast<int>(t));
      sum_rank += static_cast<double>(t);
      B.any_capped = B.any_capped || capped[i];
    }
    B.mean_far_rank = nf ? sum_rank / static_cast<double>(nf) : 0.0;
  } else {
    // translation classes share one node-interaction factorisation
    // (baselines.cpp:151-189), first-seen order like the parametric build
    std::map<std::array<std::int64_t, 4>, int> seen;
    M.far_key.resize(M.blocks.far.size());
    for (size_t i = 0; i < M.blocks.far.size(); ++i) {
      const TreeNode& s = T.nodes[M.blocks.far[i].sigma];
      const TreeNode& u = T.nodes[M.blocks.far[i].tau];
      std::array<std::int64_t, 4> key{s.level, 0, 0, 0};
      for (int k = 0; k < d; ++k) key[1 + k] = u.coords[k] - s.coords[k];
      auto it = seen.find(key);
      if (it == seen.end()) {
        it = seen.emplace(key, static_cast<int>(M.class_rep.size())).first;
        M.class_rep.push_back(static_cast<int>(i));
        M.class_keys.push_back(key);
      }
      M.far_key[i] = it->second;
    }
    const Index ncls = static_cast<Index>(M.class_rep.size());
    const int p_s = cfg.p_s;
    Index P = 1;
    for (int k = 0; k < d; ++k) P *= p_s;
    std::vector<LowRank> built(ncls);
    parallel_for(
        ncls,
        [&](Index c) {
          const Block b = M.blocks.far[M.class_rep[c]];
          const TreeNode& sn = T.nodes[b.sigma];
          const TreeNode& tn = T.nodes[b.tau];
          std::array<double, kMaxDim> box_delta{};
          std::vector<std::vector<double>> offsets;
          for (int k = 0; k < d; ++k) {
            const double side = T.level_side(sn.level, k);
            box_delta[k] = static_cast<double>(sn.coords[k] - tn.coords[k]) * side;
            std::vector<double> u(p_s);
            for (int j = 0; j < p_s; ++j) {
              const double cs = std::cos((2.0 * j + 1.0) * kPi / (2.0 * p_s));
              u[p_s - 1 - j] = 0.5 * (cs + 1.0) * side;
            }
            offsets.push_back(std::move(u));
          }
          auto entry = [&](Index r, Index cidx) {
            double r2 = 0.0;
            Index ri = r, ci = cidx;
            for (int k = 0; k < d; ++k) {
              const double delta = box_delta[k] + offsets[k][ri % p_s] - offsets[k][ci % p_s];
              r2 += delta * delta;
              ri /= p_s;
              ci /= p_s;
            }
            far_evals.add();
            return kernel_value(cfg.spec, std::sqrt(r2), th.data());
          };
          const auto& key = M.class_keys[c];
          std::uint64_t s = mix_seed(0x68636121ULL, static_cast<std::uint64_t>(key[0]));
          for (int k = 0; k < kMaxDim; ++k) s = mix_seed(s, static_cast<std::uint64_t>(key[1 + k]));
          Rng rng(s);
          built[c] = aca_partial_rng(entry, P, P, eps, r_max, rng);
        },
        cfg.threads);
    B.fixed_c.assign(static_cast<size_t>(ncls * P * P), 0.0);
    for (Index c = 0; c < ncls; ++c) {
      const LowRank& f = built[c];
      const Index t = f.rank();
      B.rank.push_back(static_cast<int>(t));
      B.any_capped = B.any_capped || f.capped;
      double* C = &B.fixed_c[static_cast<size_t>(c * P * P)];
      for (Index j = 0; j < P; ++j)
        for (Index i = 0; i < P; ++i) {
          double acc = 0.0;
          for (Index l = 0; l < t; ++l) acc += f.v(i, l) * f.y(j, l);
          C[i + j * P] = acc;
        }
    }
    // mean over far blocks (shared factors counted per block) and the
    // coupling ratio (2/n^2) sum_b p_s^d t_b (baselines.cpp:264-280)
    double sum_rank = 0.0;
    for (size_t i = 0; i < M.blocks.far.size(); ++i) sum_rank += B.rank[M.far_key[i]];
    const double nf = static_cast<double>(M.blocks.far.size());
    B.mean_far_rank = nf > 0 ? sum_rank / nf : 0.0;
    B.coupling_ratio = 2.0 * static_cast<double>(P) * sum_rank / (static_cast<double>(n) * static_cast<double>(n));
  }
  // H_b = I_t per class (the H form applies S (H (T^T x)) with H = I; the
  // H^2 form keeps them for far_h only)
  std::int64_t off = 0;
  for (int t : B.rank) {
    B.h_off.push_back(off);
    for (int j = 0; j < t; ++j)
      for (int i = 0; i < t; ++i) B.fixed_h.push_back(i == j ? 1.0 : 0.0);
    off += static_cast<std::int64_t>(t) * t;
  }
  B.far_s = now_s() - t1;
  B.far_evals = far_evals.value();
  for (const Block& b : M.blocks.near)
    B.near_evals += static_cast<std::uint64_t>(T.nodes[b.sigma].count) * static_cast<std::uint64_t>(T.nodes[b.tau].count);
  return hm;
}

}  // namespace phm
