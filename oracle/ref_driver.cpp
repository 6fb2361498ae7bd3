// C driver around the COMPILED REFERENCE: TEST INFRASTRUCTURE ONLY.
//
// Linked with the unmodified /root/reference/proj/src/*.cpp (built against
// oracle/eigen_shim by oracle/ref_build.sh) into oracle/_ref/libphmat_ref.so.
// Only tests/, __graft_entry__.smoke() and bench.py's reference / CPU-baseline
// legs load it, as the checker or as the timed reference arm; the product
// (paper_2511_03109_b200/) never does.
//
// Every computation below is a call into the reference's own public API:
//   generate_points            harness.cpp:174-181
//   ClusterTree / blocks       geometry.cpp:46-157
//   translation classes        phmatrix.cpp:29-41 (restated: anonymous there;
//                              built on the public translation_key,
//                              farfield.cpp:31-39)
//   make_theta_grids           farfield.cpp:9-14
//   NestedClusterBasis         chebyshev.cpp:195-298
//   near_oracle (snapshots)    nearfield.cpp:7-48
//   nearfield_online           nearfield.cpp:71-80
//   pttk_offline / pttk_online farfield.cpp:126-155
//   assemble_L_R               farfield.cpp:157-184
//   coupling_apply             farfield.cpp:186-212
//   offline_h2 / instantiate   phmatrix.cpp:51-225
//   Instantiated*::apply       phmatrix.cpp:227-269
//   to_dense                   phmatrix.cpp:273-317
// The driver only moves data in and out (plain pointers, status codes) and
// assembles the reference's structs from offline data handed to it.
#include <chrono>
#include <cmath>
#include <cstring>
#include <memory>
#include <numeric>
#include <span>
#include <string>
#include <unordered_map>
#include <vector>

#include "phmat/harness.hpp"
#include "phmat/phmatrix.hpp"

using namespace phmat;

namespace {

thread_local std::string g_err;

template <typename F>
int guarded(F&& f) {
  try {
    f();
    return 0;
  } catch (const std::domain_error& e) {
    g_err = e.what();
    return 1;
  } catch (const std::invalid_argument& e) {
    g_err = e.what();
    return 2;
  } catch (const std::logic_error& e) {
    g_err = e.what();
    return 3;
  } catch (const std::exception& e) {
    g_err = e.what();
    return 4;
  }
}

double now_s() {
  return std::chrono::duration<double>(std::chrono::steady_clock::now().time_since_epoch()).count();
}

// Snapshot-mode evaluation: the near tensor A_b[e, k] = f_{theta_k}(r_e) of
// nearfield.cpp:7-48 evaluated by the reference's near_oracle, with an
// evaluation spec / grid that expresses the BASELINE families in the
// reference's own kernels: Gaussian exp(-r^2/(2 l^2))
// = se at lambda = sqrt(2) l; Matern-3/2, -5/2 = mn at nu = 1.5, 2.5; the
// sigma^2 amplitude is an exactly linear extra theta-core.
struct EvalSpec {
  KernelSpec spec;
  ThetaGrids grids;       // nodes passed as theta to kernel_value
  bool amplitude = false;  // theta-dim 1 is sigma^2 (linear)
};

struct RefMatrix {
  PHConfig cfg;
  bool h2 = true;
  std::shared_ptr<ClusterTree> tree;
  BlockClusterTree blocks;
  ThetaGrids grids;
  std::vector<int> far_key, rep;
  std::vector<std::shared_ptr<const CouplingTT>> couplings;
  std::vector<NearBlockTT> near;
  EvalSpec ev;
  bool have_ev = false;
  std::shared_ptr<ParametricHMatrix> ph;
  std::shared_ptr<ParametricH2Matrix> ph2;
  std::shared_ptr<NestedClusterBasis> basis;  // H^2 basis for row probes before finalize
};

struct RefInst {
  std::unique_ptr<InstantiatedHMatrix> ih;
  std::unique_ptr<InstantiatedH2Matrix> ih2;
  const std::vector<Eigen::MatrixXd>& near_d() const { return ih ? ih->near_d : ih2->near_d; }
  const std::vector<Eigen::MatrixXd>& far_h() const { return ih ? ih->far_h : ih2->far_h; }
  const LinearOperator& op() const {
    if (ih) return *ih;
    return *ih2;
  }
};

void classes(const ClusterTree& tree, const BlockClusterTree& bct, std::vector<int>& key_of,
             std::vector<int>& rep) {
  // phmatrix.cpp:29-41, on the reference's public translation_key.
  key_of.assign(bct.far.size(), 0);
  rep.clear();
  std::unordered_map<TranslationKey, int, TranslationKeyHash> seen;
  for (std::size_t i = 0; i < bct.far.size(); ++i) {
    auto [it, fresh] = seen.emplace(translation_key(tree, bct.far[i]), static_cast<int>(rep.size()));
    if (fresh) rep.push_back(static_cast<int>(i));
    key_of[i] = it->second;
  }
}

TTTensor tt_from(int ncores, const std::int64_t* dims, const double* data) {
  TTTensor tt;
  std::int64_t off = 0;
  for (int k = 0; k < ncores; ++k) {
    TTCore c = TTCore::zeros(dims[3 * k], dims[3 * k + 1], dims[3 * k + 2]);
    std::memcpy(c.data.data(), data + off, sizeof(double) * c.size());
    off += c.size();
    tt.cores.push_back(std::move(c));
  }
  tt.validate();
  return tt;
}

NearBlockTT snapshot_tt(const RefMatrix& M, Index b) {
  PHMAT_CHECK(M.have_ev, "snapshot: evaluation spec not set");
  const Block blk = M.blocks.near[b];
  const EvalSpec& ev = M.ev;
  EntryOracle oracle = near_oracle(*M.tree, blk, ev.spec, ev.grids, nullptr);
  const Index ns = M.tree->node(blk.sigma).size(), nt = M.tree->node(blk.tau).size();
  const Index N = ns * nt;
  const Index P = ev.grids.grids[0].p;
  const int d_eval = ev.grids.d_theta();
  // G1 (1, N, P): A_b unfolded; G2 (P, P, 1) identity on the length-scale
  // nodes (SURVEY.md §8(a) "Snapshot mode is exact in the reference's types").
  TTCore g1 = TTCore::zeros(1, N, P);
  std::vector<Index> idx(1 + d_eval, 0);
  for (Index k = 0; k < P; ++k) {
    idx[1] = k;
    for (Index e = 0; e < N; ++e) {
      idx[0] = e;
      g1.at(0, e, k) = oracle(idx.data());
    }
  }
  NearBlockTT nb;
  nb.n_rows = ns;
  nb.n_cols = nt;
  nb.tt.cores.push_back(std::move(g1));
  const int d_theta = M.grids.d_theta();
  TTCore g2 = TTCore::zeros(P, M.grids.grids[0].p, 1);
  PHMAT_CHECK(M.grids.grids[0].p == P, "snapshot: grid size mismatch");
  if (d_theta == 1) {
    for (Index k = 0; k < P; ++k) g2.at(k, k, 0) = 1.0;
    nb.tt.cores.push_back(std::move(g2));
  } else {
    PHMAT_CHECK(d_theta == 2 && ev.amplitude, "snapshot: second theta-dim must be the amplitude");
    for (Index k = 0; k < P; ++k) g2.at(k, k, 0) = 1.0;
    nb.tt.cores.push_back(std::move(g2));
    const ChebGrid1D& g = M.grids.grids[1];
    TTCore g3 = TTCore::zeros(1, g.p, 1);
    for (Index j = 0; j < g.p; ++j) g3.at(0, j, 0) = g.nodes[j];
    nb.tt.cores.push_back(std::move(g3));
  }
  nb.tt.validate();
  return nb;
}

Eigen::MatrixXd near_block_online(const RefMatrix& M, Index b, const std::vector<Eigen::VectorXd>& v) {
  if (b < static_cast<Index>(M.near.size()) && !M.near[b].tt.cores.empty()) return nearfield_online(M.near[b], v);
  return nearfield_online(snapshot_tt(M, b), v);
}

void copy_out(const Eigen::MatrixXd& m, double* out) { std::memcpy(out, m.data(), sizeof(double) * m.size()); }

}  // namespace

extern "C" {

const char* rfd_last_error() { return g_err.c_str(); }

int rfd_generate_points(std::int64_t n, int d, std::uint64_t seed, double* out_rowmajor) {
  return guarded([&] {
    const Eigen::MatrixXd p = generate_points(n, d, seed);
    for (Index i = 0; i < n; ++i)
      for (int k = 0; k < d; ++k) out_rowmajor[i * d + k] = p(i, k);
  });
}

// x ~ N(0,1) by Box-Muller on the reference's Rng (common.hpp:22-33), the
// same stream as the product's generate_normal (host/core.cpp): u1 = 1 - U.
int rfd_generate_normal(std::int64_t n, std::uint64_t seed, double* out) {
  return guarded([&] {
    Rng rng(mix_seed(seed, 0x6e6f726dULL));
    for (Index i = 0; i < n; ++i) {
      const double u1 = 1.0 - rng.uniform();
      const double u2 = rng.uniform();
      out[i] = std::sqrt(-2.0 * std::log(u1)) * std::cos(6.283185307179586476925286766559 * u2);
    }
  });
}

// run_experiment's theta draws (harness.cpp:254-260).
int rfd_theta_draws(double lo, double hi, std::int64_t count, std::uint64_t seed, double* out) {
  return guarded([&] {
    Rng rng(mix_seed(seed, 0x74686574ULL));
    for (Index i = 0; i < count; ++i) out[i] = rng.uniform(lo, hi);
  });
}

double rfd_kernel_value(int family, double r, const double* theta, int d_theta) {
  KernelSpec s;
  s.family = static_cast<KernelFamily>(family);
  s.theta_box.resize(d_theta);
  return kernel_value(s, r, theta);
}

int rfd_lagrange(double lo, double hi, int p, double x, double* out) {
  return guarded([&] {
    const ChebGrid1D g = cheb_grid(lo, hi, p);
    lagrange_eval_all(g, x, out);
  });
}

int rfd_cheb_grid(double lo, double hi, int p, double* nodes, double* weights) {
  return guarded([&] {
    const ChebGrid1D g = cheb_grid(lo, hi, p);
    for (int j = 0; j < p; ++j) {
      nodes[j] = g.nodes[j];
      weights[j] = g.weights[j];
    }
  });
}

int rfd_create(const double* points_rowmajor, std::int64_t n, int d, int l_max, double eta, void** out) {
  return guarded([&] {
    Eigen::MatrixXd pts(n, d);
    for (Index i = 0; i < n; ++i)
      for (int k = 0; k < d; ++k) pts(i, k) = points_rowmajor[i * d + k];
    auto M = std::make_unique<RefMatrix>();
    M->tree = std::make_shared<ClusterTree>(std::move(pts), unit_box(d), l_max);
    M->cfg.l_max = l_max;
    M->cfg.eta = eta;
    M->blocks = build_block_cluster_tree(*M->tree, M->cfg.resolved_eta(d));
    classes(*M->tree, M->blocks, M->far_key, M->rep);
    *out = M.release();
  });
}

void rfd_destroy(void* h) { delete static_cast<RefMatrix*>(h); }

// counts: nodes, leaves, near, far, classes, c_sp, block_count, coverage
int rfd_counts(void* h, std::int64_t* out) {
  return guarded([&] {
    auto& M = *static_cast<RefMatrix*>(h);
    out[0] = M.tree->node_count();
    out[1] = static_cast<std::int64_t>(M.tree->leaves().size());
    out[2] = static_cast<std::int64_t>(M.blocks.near.size());
    out[3] = static_cast<std::int64_t>(M.blocks.far.size());
    out[4] = static_cast<std::int64_t>(M.rep.size());
    out[5] = M.blocks.c_sp;
    out[6] = M.blocks.block_count;
    out[7] = coverage_sum(*M.tree, M.blocks);
  });
}

// Tree-order permutation: leaf index sets concatenated in leaf-id order.
int rfd_perm(void* h, std::int32_t* out) {
  return guarded([&] {
    auto& M = *static_cast<RefMatrix*>(h);
    Index pos = 0;
    for (int leaf : M.tree->leaves())
      for (std::int32_t i : M.tree->node(leaf).indices) out[pos++] = i;
  });
}

int rfd_nodes(void* h, std::int32_t* level, std::int32_t* parent, std::int32_t* first_child, std::int64_t* size,
              std::int64_t* coords) {
  return guarded([&] {
    auto& M = *static_cast<RefMatrix*>(h);
    for (int i = 0; i < M.tree->node_count(); ++i) {
      const ClusterNode& nd = M.tree->node(i);
      level[i] = nd.level;
      parent[i] = nd.parent;
      first_child[i] = nd.first_child;
      size[i] = nd.size();
      for (int k = 0; k < kMaxDim; ++k) coords[3 * i + k] = nd.coords[k];
    }
  });
}

int rfd_blocks(void* h, std::int32_t* near_s, std::int32_t* near_t, std::int32_t* far_s, std::int32_t* far_t,
               std::int32_t* far_key) {
  return guarded([&] {
    auto& M = *static_cast<RefMatrix*>(h);
    for (std::size_t i = 0; i < M.blocks.near.size(); ++i) {
      near_s[i] = M.blocks.near[i].sigma;
      near_t[i] = M.blocks.near[i].tau;
    }
    for (std::size_t i = 0; i < M.blocks.far.size(); ++i) {
      far_s[i] = M.blocks.far[i].sigma;
      far_t[i] = M.blocks.far[i].tau;
      far_key[i] = M.far_key[i];
    }
  });
}

// Parametric configuration: a reference KernelSpec (family id of
// kernels.hpp:21, one interval per theta-dim) whose box defines the theta
// grids (make_theta_grids, one p_theta for every dim as in PHConfig).
int rfd_setup(void* h, int h2, int family, int d_theta, const double* lo, const double* hi, int p_theta, int p_s) {
  return guarded([&] {
    auto& M = *static_cast<RefMatrix*>(h);
    M.h2 = h2 != 0;
    M.cfg.spec.family = static_cast<KernelFamily>(family);
    M.cfg.spec.theta_box.clear();
    for (int k = 0; k < d_theta; ++k) M.cfg.spec.theta_box.push_back({lo[k], hi[k]});
    M.cfg.p_theta = p_theta;
    M.cfg.p_s = p_s;
    M.cfg.near_mode = NearMode::TT;
    M.cfg.translation_cache = true;
    M.grids = make_theta_grids(M.cfg.spec, p_theta);
    M.couplings.assign(M.rep.size(), nullptr);
    M.near.assign(M.blocks.near.size(), NearBlockTT{});
    if (M.h2) M.basis = std::make_shared<NestedClusterBasis>(*M.tree, p_s);
  });
}

int rfd_theta_grid(void* h, int k, double* nodes, double* weights) {
  return guarded([&] {
    auto& M = *static_cast<RefMatrix*>(h);
    const ChebGrid1D& g = M.grids.grids.at(k);
    for (int j = 0; j < g.p; ++j) {
      nodes[j] = g.nodes[j];
      weights[j] = g.weights[j];
    }
  });
}

// Snapshot evaluation spec: reference family + fixed second parameter (nu for
// mn), length-scale multiplier (sqrt(2) for the Gaussian as se), amplitude.
int rfd_set_eval(void* h, int family, double nu, double lam_scale, int amplitude) {
  return guarded([&] {
    auto& M = *static_cast<RefMatrix*>(h);
    EvalSpec ev;
    ev.spec.family = static_cast<KernelFamily>(family);
    ChebGrid1D g = M.grids.grids.at(0);
    for (int j = 0; j < g.p; ++j) g.nodes[j] *= lam_scale;
    g.lo *= lam_scale;
    g.hi *= lam_scale;
    ev.grids.grids.push_back(g);
    ev.spec.theta_box.push_back({g.lo, g.hi});
    if (ev.spec.family == KernelFamily::Matern) {
      ChebGrid1D gn;
      gn.lo = gn.hi = nu;
      gn.p = 1;
      gn.nodes = Eigen::VectorXd::Constant(1, nu);
      gn.weights = Eigen::VectorXd::Constant(1, 1.0);
      ev.grids.grids.push_back(gn);
      ev.spec.theta_box.push_back({nu, nu});
    }
    ev.amplitude = amplitude != 0;
    M.ev = std::move(ev);
    M.have_ev = true;
  });
}

int rfd_set_coupling(void* h, int k, int ncores, const std::int64_t* dims, const double* data) {
  return guarded([&] {
    auto& M = *static_cast<RefMatrix*>(h);
    auto c = std::make_shared<CouplingTT>();
    c->tt = tt_from(ncores, dims, data);
    c->d = M.tree->dim();
    c->d_theta = M.grids.d_theta();
    PHMAT_CHECK(c->tt.order() == 2 * c->d + c->d_theta, "rfd_set_coupling: core count");
    M.couplings.at(k) = std::move(c);
  });
}

int rfd_set_near_tt(void* h, std::int64_t b, int ncores, const std::int64_t* dims, const double* data) {
  return guarded([&] {
    auto& M = *static_cast<RefMatrix*>(h);
    NearBlockTT nb;
    nb.tt = tt_from(ncores, dims, data);
    nb.n_rows = M.tree->node(M.blocks.near.at(b).sigma).size();
    nb.n_cols = M.tree->node(M.blocks.near.at(b).tau).size();
    M.near.at(b) = std::move(nb);
  });
}

// Builds the snapshot TT of every near block (reference near_oracle).
int rfd_make_near_snapshots(void* h, int threads) {
  return guarded([&] {
    auto& M = *static_cast<RefMatrix*>(h);
    parallel_for(
        static_cast<Index>(M.blocks.near.size()), [&](Index b) { M.near[b] = snapshot_tt(M, b); }, threads);
  });
}

// Assembles the reference's ParametricHMatrix / ParametricH2Matrix (H form:
// S_b, T_b by the reference's own pttk_offline, farfield.cpp:126-147).
int rfd_finalize(void* h, int threads) {
  return guarded([&] {
    auto& M = *static_cast<RefMatrix*>(h);
    for (const auto& c : M.couplings) PHMAT_CHECK(c != nullptr, "rfd_finalize: coupling missing");
    for (const auto& nb : M.near) PHMAT_CHECK(!nb.tt.cores.empty(), "rfd_finalize: near block missing");
    M.cfg.threads = threads;
    if (M.h2) {
      auto pm = std::make_shared<ParametricH2Matrix>();
      pm->config = M.cfg;
      pm->tree = M.tree;
      pm->blocks = M.blocks;
      pm->theta_grids = M.grids;
      pm->basis = *M.basis;
      pm->far_key = M.far_key;
      pm->couplings = M.couplings;
      pm->far.resize(M.blocks.far.size());
      for (std::size_t i = 0; i < pm->far.size(); ++i) pm->far[i].coupling = M.couplings[M.far_key[i]];
      pm->near = M.near;
      M.ph2 = std::move(pm);
    } else {
      auto pm = std::make_shared<ParametricHMatrix>();
      pm->config = M.cfg;
      pm->tree = M.tree;
      pm->blocks = M.blocks;
      pm->theta_grids = M.grids;
      pm->far_key = M.far_key;
      pm->couplings = M.couplings;
      pm->far.resize(M.blocks.far.size());
      parallel_for(
          static_cast<Index>(pm->far.size()),
          [&](Index i) {
            pm->far[i] = pttk_offline(*M.tree, M.blocks.far[i], M.cfg.p_s, M.couplings[M.far_key[i]]);
          },
          threads);
      pm->near = M.near;
      M.ph = std::move(pm);
    }
  });
}

int rfd_far_st(void* h, std::int64_t i, double* S, double* T, std::int64_t* shape) {
  return guarded([&] {
    auto& M = *static_cast<RefMatrix*>(h);
    PHMAT_CHECK(M.ph != nullptr, "rfd_far_st: not an H-form matrix");
    const FarBlockH& f = M.ph->far.at(i);
    shape[0] = f.s.rows();
    shape[1] = f.s.cols();
    shape[2] = f.t.rows();
    shape[3] = f.t.cols();
    if (S) copy_out(f.s, S);
    if (T) copy_out(f.t, T);
  });
}

int rfd_instantiate(void* h, const double* theta, void** out, double* seconds) {
  return guarded([&] {
    auto& M = *static_cast<RefMatrix*>(h);
    std::span<const double> th(theta, M.grids.d_theta());
    auto I = std::make_unique<RefInst>();
    const double t0 = now_s();
    if (M.h2) {
      PHMAT_CHECK(M.ph2 != nullptr, "rfd_instantiate: finalize first");
      I->ih2 = std::make_unique<InstantiatedH2Matrix>(instantiate(M.ph2, th));
    } else {
      PHMAT_CHECK(M.ph != nullptr, "rfd_instantiate: finalize first");
      I->ih = std::make_unique<InstantiatedHMatrix>(instantiate(M.ph, th));
    }
    if (seconds) *seconds = now_s() - t0;
    *out = I.release();
  });
}

void rfd_inst_destroy(void* i) { delete static_cast<RefInst*>(i); }

int rfd_inst_near_d(void* i, std::int64_t b, double* out) {
  return guarded([&] { copy_out(static_cast<RefInst*>(i)->near_d().at(b), out); });
}

int rfd_inst_far_h(void* i, std::int64_t b, double* out, std::int64_t* shape) {
  return guarded([&] {
    const Eigen::MatrixXd& m = static_cast<RefInst*>(i)->far_h().at(b);
    shape[0] = m.rows();
    shape[1] = m.cols();
    if (out) copy_out(m, out);
  });
}

// y = K(theta) x for nrhs columns (column loop over the reference's apply,
// which takes one VectorXd, phmatrix.hpp:99).
int rfd_inst_apply(void* i, const double* x, double* y, std::int64_t n, int nrhs, double* seconds) {
  return guarded([&] {
    const LinearOperator& op = static_cast<RefInst*>(i)->op();
    const double t0 = now_s();
    for (int c = 0; c < nrhs; ++c) {
      Eigen::VectorXd xv(n);
      std::memcpy(xv.data(), x + c * n, sizeof(double) * n);
      const Eigen::VectorXd yv = op.apply(xv);
      std::memcpy(y + c * n, yv.data(), sizeof(double) * n);
    }
    if (seconds) *seconds = now_s() - t0;
  });
}

int rfd_inst_to_dense(void* i, double* out, std::int64_t guard) {
  return guarded([&] {
    auto* I = static_cast<RefInst*>(i);
    copy_out(I->ih ? I->ih->to_dense(guard) : I->ih2->to_dense(guard), out);
  });
}

// ---- artifacts: the reference's own offline build, saved / loaded ---------
// offline_h / offline_h2 of the reference itself (its TT-cross for the
// couplings and, in TT near mode, for every near block; phmatrix.cpp:51-164)
// on generate_points(n, d, seed), then save_parametric (serialize.cpp:108-
// 177): the `phmat build --artifact` path (tools/phmat.cpp:155-171).
int rfd_build_save(std::int64_t n, int d, std::uint64_t seed, int h2, int family, int d_theta, const double* lo,
                   const double* hi, int l_max, int p_s, int p_theta, double eps, double eta, int near_tt,
                   const char* path, int threads) {
  return guarded([&] {
    PHConfig cfg;
    cfg.spec.family = static_cast<KernelFamily>(family);
    for (int k = 0; k < d_theta; ++k) cfg.spec.theta_box.push_back({lo[k], hi[k]});
    cfg.l_max = l_max;
    cfg.p_s = p_s;
    cfg.p_theta = p_theta;
    cfg.eps = eps;
    cfg.eta = eta;
    cfg.near_mode = near_tt ? NearMode::TT : NearMode::Direct;
    cfg.threads = threads;
    StageCounters counters;
    const Eigen::MatrixXd pts = generate_points(n, d, seed);
    if (h2)
      save_parametric(offline_h2(pts, cfg, counters), path);
    else
      save_parametric(offline_h(pts, cfg, counters), path);
  });
}

// load_parametric_h / _h2 (serialize.cpp:180-269) into a driver handle
// (instantiate / apply / near_d / far_h through the rfd_inst_* calls).
int rfd_load(const char* path, void** out) {
  return guarded([&] {
    auto M = std::make_unique<RefMatrix>();
    M->h2 = artifact_is_h2(path);
    auto fill = [&](auto& pm) {
      M->cfg = pm->config;
      M->tree = std::const_pointer_cast<ClusterTree>(pm->tree);
      M->blocks = pm->blocks;
      M->grids = pm->theta_grids;
      M->far_key = pm->far_key;
      M->couplings = pm->couplings;
      M->rep.assign(pm->couplings.size(), 0);
      M->near = pm->near;
    };
    if (M->h2) {
      M->ph2 = std::make_shared<ParametricH2Matrix>(load_parametric_h2(path));
      fill(M->ph2);
      M->basis = std::make_shared<NestedClusterBasis>(M->ph2->basis);
    } else {
      M->ph = std::make_shared<ParametricHMatrix>(load_parametric_h(path));
      fill(M->ph);
    }
    *out = M.release();
  });
}

// ---- per-block entry points (full-size sampled parity without a full build)
int rfd_class_h(void* h, int k, const double* theta, double* out, std::int64_t* shape) {
  return guarded([&] {
    auto& M = *static_cast<RefMatrix*>(h);
    const auto v = parametric_vectors(M.grids, std::span<const double>(theta, M.grids.d_theta()));
    const Eigen::MatrixXd H = pttk_online(*M.couplings.at(k), v);
    shape[0] = H.rows();
    shape[1] = H.cols();
    if (out) copy_out(H, out);
  });
}

// C_k = L_k H_k R_k^T (P x P): the explicit coupling coupling_apply applies
// (farfield.cpp:157-212, test_farfield.cpp:310-333).
int rfd_class_c(void* h, int k, const double* theta, double* out) {
  return guarded([&] {
    auto& M = *static_cast<RefMatrix*>(h);
    const auto v = parametric_vectors(M.grids, std::span<const double>(theta, M.grids.d_theta()));
    const CouplingTT& c = *M.couplings.at(k);
    const auto [L, R] = assemble_L_R(c);
    copy_out(L * (pttk_online(c, v) * R.transpose()), out);
  });
}

int rfd_near_online(void* h, std::int64_t b, const double* theta, double* out) {
  return guarded([&] {
    auto& M = *static_cast<RefMatrix*>(h);
    const auto v = parametric_vectors(M.grids, std::span<const double>(theta, M.grids.d_theta()));
    copy_out(near_block_online(M, b, v), out);
  });
}

// Rows J of y = K(theta) x for the H^2 form, composed from the reference's
// own pieces exactly as InstantiatedH2Matrix::apply (phmatrix.cpp:246-269)
// does, restricted to the blocks that reach J: the full forward pass, then
// coupling_apply for every far block whose sigma contains a probe row, the
// backward pass, and nearfield_online + GEMV for the near blocks of the
// probe leaves. Lets full-size configs (C3: 100 GB of snapshots) be checked
// against the reference without instantiating every block.
int rfd_apply_rows(void* h, const double* theta, const double* x, int nrhs, const std::int64_t* rows,
                   std::int64_t nrows, double* out, int threads) {
  return guarded([&] {
    auto& M = *static_cast<RefMatrix*>(h);
    PHMAT_CHECK(M.h2 && M.basis, "rfd_apply_rows: H^2 form only");
    const ClusterTree& T = *M.tree;
    const Index n = T.n_points();
    const auto v = parametric_vectors(M.grids, std::span<const double>(theta, M.grids.d_theta()));
    // leaf of each point, and the set of nodes on the probe rows' paths
    std::vector<int> leaf_of(n, -1);
    for (int leaf : T.leaves())
      for (std::int32_t i : T.node(leaf).indices) leaf_of[i] = leaf;
    std::vector<char> on_path(T.node_count(), 0), probe_leaf(T.node_count(), 0);
    for (Index r = 0; r < nrows; ++r) {
      int id = leaf_of.at(rows[r]);
      probe_leaf[id] = 1;
      for (; id >= 0; id = T.node(id).parent) on_path[id] = 1;
    }
    std::vector<Eigen::MatrixXd> class_h(M.couplings.size());
    std::vector<char> need(M.couplings.size(), 0);
    for (std::size_t i = 0; i < M.blocks.far.size(); ++i)
      if (on_path[M.blocks.far[i].sigma]) need[M.far_key[i]] = 1;
    parallel_for(
        static_cast<Index>(M.couplings.size()),
        [&](Index k) {
          if (need[k]) class_h[k] = pttk_online(*M.couplings[k], v);
        },
        threads);
    std::vector<Index> near_idx;
    for (std::size_t i = 0; i < M.blocks.near.size(); ++i)
      if (probe_leaf[M.blocks.near[i].sigma]) near_idx.push_back(static_cast<Index>(i));
    std::vector<Eigen::MatrixXd> D(near_idx.size());
    parallel_for(
        static_cast<Index>(near_idx.size()), [&](Index j) { D[j] = near_block_online(M, near_idx[j], v); },
        threads);
    for (int c = 0; c < nrhs; ++c) {
      Eigen::VectorXd xv(n);
      std::memcpy(xv.data(), x + static_cast<Index>(c) * n, sizeof(double) * n);
      const std::vector<Eigen::VectorXd> xhat = M.basis->forward(T, xv);
      std::vector<Eigen::VectorXd> yhat(T.node_count());
      for (std::size_t i = 0; i < M.blocks.far.size(); ++i) {
        const Block b = M.blocks.far[i];
        if (!on_path[b.sigma]) continue;
        Eigen::VectorXd z = coupling_apply(*M.couplings[M.far_key[i]], class_h[M.far_key[i]], xhat[b.tau]);
        if (yhat[b.sigma].size() == 0)
          yhat[b.sigma] = std::move(z);
        else
          yhat[b.sigma] += z;
      }
      Eigen::VectorXd y = Eigen::VectorXd::Zero(n);
      for (std::size_t j = 0; j < near_idx.size(); ++j) {
        const Block b = M.blocks.near[near_idx[j]];
        const auto& ti = T.node(b.tau).indices;
        const auto& si = T.node(b.sigma).indices;
        Eigen::VectorXd xt(static_cast<Index>(ti.size()));
        for (std::size_t q = 0; q < ti.size(); ++q) xt[static_cast<Index>(q)] = xv[ti[q]];
        const Eigen::VectorXd z = D[j] * xt;
        for (std::size_t q = 0; q < si.size(); ++q) y[si[q]] += z[static_cast<Index>(q)];
      }
      M.basis->backward(T, yhat, y);
      for (Index r = 0; r < nrows; ++r) out[static_cast<Index>(c) * nrows + r] = y[rows[r]];
    }
  });
}

}  // extern "C"

namespace {
// ---- reference CPU arm for bench.py (no product code involved) ------------
// Builds the reference's own parametric matrix: offline_h / offline_h2 in
// Direct near mode gives the tree, blocks, classes and coupling TTs by the
// reference's TT-cross (phmatrix.cpp:51-164, farfield.cpp:102-124) and, for
// the H form, S_b / T_b by pttk_offline; the near field is the snapshot-mode
// TT (near_oracle) of a seeded 1/stride sample of near blocks. Two parametric
// matrices share that data: `sample` (every class, the sampled near and far
// blocks) and `fixed` (every class, one far block per sigma so the basis
// passes run in full, no near blocks). The per-step cost is timed on both
// through the reference's own instantiate + apply, so the whole-theta cost
// is fixed + (sample - fixed) * stride.
struct RefBenchBase {
  virtual ~RefBenchBase() = default;
  double near_frac = 0, far_frac = 0, build_s = 0;
  Index n = 0, near_blocks = 0, far_blocks = 0;
  int d_theta = 1;
  virtual void step(int which, const double* theta, const double* x, int nrhs, double* y, double* times) = 0;
};

template <typename PM, typename Inst>
struct RefBenchT : RefBenchBase {
  std::shared_ptr<PM> sample, fixed;
  void step(int which, const double* theta, const double* x, int nrhs, double* y, double* times) override {
    auto pm = which == 0 ? sample : fixed;
    const double t0 = now_s();
    Inst inst = instantiate(std::shared_ptr<const PM>(pm), std::span<const double>(theta, d_theta));
    const double t1 = now_s();
    Eigen::VectorXd xv(n);
    for (int c = 0; c < nrhs; ++c) {
      std::memcpy(xv.data(), x + static_cast<Index>(c) * n, sizeof(double) * n);
      const Eigen::VectorXd yv = inst.apply(xv);
      std::memcpy(y, yv.data(), sizeof(double) * n);
    }
    const double t2 = now_s();
    times[0] = t1 - t0;
    times[1] = t2 - t1;
  }
};

template <typename PM, typename Inst>
RefBenchBase* bench_build(PM full, const EvalSpec& ev, std::uint64_t seed, Index stride, int threads) {
  auto B = std::make_unique<RefBenchT<PM, Inst>>();
  B->n = full.tree->n_points();
  B->d_theta = full.theta_grids.d_theta();
  auto make = [&](bool sampled) {
    auto pm = std::make_shared<PM>();
    pm->config = full.config;
    pm->config.near_mode = NearMode::TT;
    pm->tree = full.tree;
    pm->theta_grids = full.theta_grids;
    if constexpr (std::is_same_v<PM, ParametricH2Matrix>) pm->basis = full.basis;
    pm->couplings = full.couplings;
    pm->blocks.c_sp = full.blocks.c_sp;
    pm->blocks.eta = full.blocks.eta;
    auto take_far = [&](std::size_t i) {
      pm->blocks.far.push_back(full.blocks.far[i]);
      pm->far_key.push_back(full.far_key[i]);
      pm->far.push_back(full.far[i]);
    };
    if (!sampled) {
      // one far block per sigma, so the fixed-cost matrix runs the full
      // basis passes (phmatrix.cpp:251, 266) as the sampled one does
      std::vector<char> seen(full.tree->node_count(), 0);
      for (std::size_t i = 0; i < full.blocks.far.size(); ++i)
        if (!seen[full.blocks.far[i].sigma]) {
          seen[full.blocks.far[i].sigma] = 1;
          take_far(i);
        }
      return pm;
    }
    Rng rng(mix_seed(seed, 0x62656e63ULL));
    const Index off_near = static_cast<Index>(rng.integer(stride)), off_far = static_cast<Index>(rng.integer(stride));
    double near_e = 0, near_all = 0;
    for (std::size_t i = 0; i < full.blocks.near.size(); ++i) {
      const Block b = full.blocks.near[i];
      const double e = double(full.tree->node(b.sigma).size()) * double(full.tree->node(b.tau).size());
      near_all += e;
      if (static_cast<Index>(i) % stride == off_near) {
        pm->blocks.near.push_back(b);
        near_e += e;
      }
    }
    for (std::size_t i = 0; i < full.blocks.far.size(); ++i)
      if (static_cast<Index>(i) % stride == off_far) take_far(i);
    B->near_frac = near_e / near_all;
    B->far_frac = double(pm->blocks.far.size()) / double(full.blocks.far.size());
    B->near_blocks = static_cast<Index>(pm->blocks.near.size());
    B->far_blocks = static_cast<Index>(pm->blocks.far.size());
    RefMatrix M;
    M.tree = std::const_pointer_cast<ClusterTree>(full.tree);
    M.blocks = pm->blocks;
    M.grids = full.theta_grids;
    M.ev = ev;
    M.have_ev = true;
    pm->near.resize(pm->blocks.near.size());
    parallel_for(
        static_cast<Index>(pm->near.size()), [&](Index b) { pm->near[b] = snapshot_tt(M, b); }, threads);
    return pm;
  };
  B->sample = make(true);
  B->fixed = make(false);
  return B.release();
}

}  // namespace

extern "C" {

// family: reference KernelFamily of the parametric spec (the grids); eval_*:
// the snapshot evaluation (rfd_set_eval's conventions). h2: format.
int rfd_bench_create(std::int64_t n, int d, std::uint64_t seed, int h2, int family, int d_theta, const double* lo,
                     const double* hi, int l_max, int p_s, int p_theta, double eta, double eps, int eval_family,
                     double eval_nu, double eval_lam_scale, std::int64_t stride, int threads, void** out) {
  return guarded([&] {
    const double t0 = now_s();
    PHConfig cfg;
    cfg.spec.family = static_cast<KernelFamily>(family);
    for (int k = 0; k < d_theta; ++k) cfg.spec.theta_box.push_back({lo[k], hi[k]});
    cfg.l_max = l_max;
    cfg.p_s = p_s;
    cfg.p_theta = p_theta;
    cfg.eps = eps;
    cfg.eta = eta;
    cfg.seed = 0;
    cfg.near_mode = NearMode::Direct;
    cfg.threads = threads;
    StageCounters counters;
    const Eigen::MatrixXd pts = generate_points(n, d, seed);
    EvalSpec ev;
    ev.spec.family = static_cast<KernelFamily>(eval_family);
    ChebGrid1D g = make_theta_grids(cfg.spec, p_theta).grids[0];
    for (int j = 0; j < g.p; ++j) g.nodes[j] *= eval_lam_scale;
    ev.grids.grids.push_back(g);
    ev.spec.theta_box.push_back({g.lo * eval_lam_scale, g.hi * eval_lam_scale});
    if (ev.spec.family == KernelFamily::Matern) {
      ChebGrid1D gn;
      gn.lo = gn.hi = eval_nu;
      gn.p = 1;
      gn.nodes = Eigen::VectorXd::Constant(1, eval_nu);
      gn.weights = Eigen::VectorXd::Constant(1, 1.0);
      ev.grids.grids.push_back(gn);
      ev.spec.theta_box.push_back({eval_nu, eval_nu});
    }
    RefBenchBase* B = nullptr;
    if (h2)
      B = bench_build<ParametricH2Matrix, InstantiatedH2Matrix>(offline_h2(pts, cfg, counters), ev, seed, stride,
                                                                 threads);
    else
      B = bench_build<ParametricHMatrix, InstantiatedHMatrix>(offline_h(pts, cfg, counters), ev, seed, stride,
                                                               threads);
    B->build_s = now_s() - t0;
    *out = B;
  });
}

void rfd_bench_destroy(void* h) { delete static_cast<RefBenchBase*>(h); }

// info: near_frac, far_frac, build_s, near blocks sampled, far blocks sampled
int rfd_bench_info(void* h, double* info) {
  return guarded([&] {
    auto& B = *static_cast<RefBenchBase*>(h);
    info[0] = B.near_frac;
    info[1] = B.far_frac;
    info[2] = B.build_s;
    info[3] = static_cast<double>(B.near_blocks);
    info[4] = static_cast<double>(B.far_blocks);
  });
}

// One reference step (instantiate + nrhs applies) on the sampled matrix
// (which = 0) or the fixed-cost matrix (which = 1). times: instantiate s,
// apply s. y receives the last apply's output (kept live).
int rfd_bench_step(void* h, int which, const double* theta, const double* x, int nrhs, double* y, double* times) {
  return guarded([&] { static_cast<RefBenchBase*>(h)->step(which, theta, x, nrhs, y, times); });
}

}  // extern "C"
