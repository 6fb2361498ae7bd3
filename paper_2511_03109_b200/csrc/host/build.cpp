// Offline orchestration on the host (proj/src/phmatrix.cpp:51-164 with the
// far-field producers of proj/src/farfield.cpp:41-184 and the TT near-field
// producer of proj/src/nearfield.cpp:7-69). Produces a HostMatrix; the
// device layer uploads it once. Snapshot-mode near data is generated on the
// GPU (device.cu, K11) and never exists on the host.
#include <algorithm>
#include <chrono>
#include <cmath>
#include <map>

#include "phm.hpp"

namespace phm {

namespace {

double now_s() {
  return std::chrono::duration<double>(std::chrono::steady_clock::now().time_since_epoch()).count();
}

// In-box Chebyshev node offsets for one level (farfield.cpp:43-52): equal for
// every box of the level, so translated blocks see identical differences.
std::vector<double> node_offsets(double side, int p) {
  constexpr double kPi = 3.141592653589793238462643383279502884;
  std::vector<double> u(p);
  for (int k = 0; k < p; ++k) {
    const double c = std::cos((2.0 * k + 1.0) * kPi / (2.0 * p));
    u[p - 1 - k] = 0.5 * (c + 1.0) * side;
  }
  return u;
}

// Coupling tensor M_b over (sigma nodes)^d x theta nodes x (tau nodes)^d
// (farfield.cpp:56-100).
EntryFn coupling_entries(const Tree& t, Block b, const KernelSpec& spec, int ps, const ThetaGrids& g,
                         EvalCounter* counter, EvalCounter* audit) {
  const int d = t.d, dt = g.d_theta();
  const TreeNode& s = t.nodes[b.sigma];
  const TreeNode& u = t.nodes[b.tau];
  PHM_CHECK(s.level == u.level, "coupling_oracle: blocks must pair same-level boxes");
  EntryFn f;
  for (int k = 0; k < d; ++k) f.dims.push_back(ps);
  for (int k = 0; k < dt; ++k) f.dims.push_back(g.grids[k].p);
  for (int k = 0; k < d; ++k) f.dims.push_back(ps);
  struct Ctx {
    int d, dt;
    std::array<double, kMaxDim> delta;
    std::vector<std::vector<double>> off;
    std::vector<std::vector<double>> th;
    KernelSpec spec;
  };
  auto ctx = std::make_shared<Ctx>();
  ctx->d = d;
  ctx->dt = dt;
  ctx->spec = spec;
  for (int k = 0; k < d; ++k) {
    const double side = t.level_side(s.level, k);
    ctx->delta[k] = static_cast<double>(s.coords[k] - u.coords[k]) * side;
    ctx->off.push_back(node_offsets(side, ps));
  }
  for (int k = 0; k < dt; ++k) ctx->th.push_back(g.grids[k].nodes);
  f.fn = [ctx](const Index* idx) {
    double r2 = 0.0;
    for (int k = 0; k < ctx->d; ++k) {
      const double dl = ctx->delta[k] + (ctx->off[k][idx[k]] - ctx->off[k][idx[ctx->d + ctx->dt + k]]);
      r2 += dl * dl;
    }
    double th[3];
    for (int k = 0; k < ctx->dt; ++k) th[k] = ctx->th[k][idx[ctx->d + k]];
    return kernel_value(ctx->spec, std::sqrt(r2), th);
  };
  f.counter = counter;
  f.audit = audit;
  return f;
}

// Near tensor A_b[i + j n_sigma, k...] (nearfield.cpp:7-48).
EntryFn near_entries(const Tree& t, Block b, const KernelSpec& spec, const ThetaGrids& g, EvalCounter* counter,
                     EvalCounter* audit) {
  const TreeNode& s = t.nodes[b.sigma];
  const TreeNode& u = t.nodes[b.tau];
  PHM_CHECK(s.count > 0 && u.count > 0, "near_oracle: empty block");
  EntryFn f;
  f.dims.push_back(s.count * u.count);
  for (int k = 0; k < g.d_theta(); ++k) f.dims.push_back(g.grids[k].p);
  const Tree* tp = &t;
  const Index ns = s.count, sb = s.begin, ub = u.begin;
  const int d = t.d, dt = g.d_theta();
  auto th_nodes = std::make_shared<std::vector<std::vector<double>>>();
  for (int k = 0; k < dt; ++k) th_nodes->push_back(g.grids[k].nodes);
  f.fn = [tp, ns, sb, ub, d, dt, spec, th_nodes](const Index* idx) {
    const Index i = idx[0] % ns, j = idx[0] / ns;
    const Index oi = tp->perm[sb + i], oj = tp->perm[ub + j];
    double r2 = 0.0;
    for (int k = 0; k < d; ++k) {
      const double dl = tp->coord(oi, k) - tp->coord(oj, k);
      r2 += dl * dl;
    }
    double th[3];
    for (int k = 0; k < dt; ++k) th[k] = (*th_nodes)[k][idx[1 + k]];
    return kernel_value(spec, std::sqrt(r2), th);
  };
  f.counter = counter;
  f.audit = audit;
  return f;
}

// Leaf-style cluster basis factor U_{node,k}: rows = the node's points in
// tree order, columns = cardinals of the node box grid (chebyshev.cpp:71-86).
Mat basis_factor(const Tree& t, int id, int k, int ps) {
  const TreeNode& nd = t.nodes[id];
  const Grid1D g = cheb_grid(nd.box.lo[k], nd.box.hi[k], ps);
  Mat f(nd.count, ps);
  std::vector<double> row(ps);
  for (Index i = 0; i < nd.count; ++i) {
    lagrange_all(g, t.coord(t.perm[nd.begin + i], k), row.data());
    for (int j = 0; j < ps; ++j) f(i, j) = row[j];
  }
  return f;
}

// Row-wise Kronecker product: column j * b.cols + k = a_j .* b_k.
Mat face_split(const Mat& a, const Mat& b) {
  Mat o(a.rows, a.cols * b.cols);
  for (Index j = 0; j < a.cols; ++j)
    for (Index k = 0; k < b.cols; ++k) {
      double* oc = &o.a[(j * b.cols + k) * o.rows];
      for (Index i = 0; i < a.rows; ++i) oc[i] = a(i, j) * b(i, k);
    }
  return o;
}

// Column-wise Kronecker product: row i * b.rows + k = a(i, j) b(k, j).
Mat face_split_cols(const Mat& a, const Mat& b) {
  Mat o(a.rows * b.rows, a.cols);
  for (Index j = 0; j < a.cols; ++j)
    for (Index i = 0; i < a.rows; ++i)
      for (Index k = 0; k < b.rows; ++k) o(i * b.rows + k, j) = a(i, j) * b(k, j);
  return o;
}

// Phase 3 of the parametric H build (farfield.cpp:126-147): S_b = U_sigma L_b
// and T_b = U_tau R_b through interleaved face-splitting products.
void pttk_offline(const Tree& t, Block b, int ps, const Coupling& cp, Mat& S, Mat& T) {
  const int d = t.d;
  const auto& cores = cp.tt.cores;
  S = basis_factor(t, b.sigma, 0, ps) * cores[0].right();
  for (int i = 1; i < d; ++i) S = face_split(basis_factor(t, b.sigma, i, ps), S) * cores[i].right();
  const int last = cp.tt.order() - 1;
  Mat tt = cores[last].left() * transpose(basis_factor(t, b.tau, d - 1, ps));
  for (int i = 1; i < d; ++i)
    tt = cores[last - i].left() * face_split_cols(tt, transpose(basis_factor(t, b.tau, d - 1 - i, ps)));
  T = transpose(tt);
}

// Explicit L (P x r_d) and R (P x r_{d+dt}), farfield.cpp:157-184.
void assemble_lr(const Coupling& cp, Mat& L, Mat& R) {
  const int d = cp.d;
  const auto& cores = cp.tt.cores;
  L = cores[0].right();
  for (int k = 1; k < d; ++k) {
    Mat tmp = L * cores[k].left();
    Mat nl(tmp.rows * cores[k].m, cores[k].r1);
    nl.a = std::move(tmp.a);
    L = std::move(nl);
  }
  const int last = cp.tt.order() - 1;
  Mat q = cores[last].left();
  for (int k = last - 1; k >= d + cp.d_theta; --k) {
    const TTCore& c = cores[k];
    Mat nx(c.r0, c.m * q.cols);
    for (Index cc = 0; cc < q.cols; ++cc)
      for (Index j = 0; j < c.m; ++j)
        for (Index a = 0; a < c.r0; ++a) {
          double s = 0.0;
          for (Index y = 0; y < c.r1; ++y) s += c.at(a, j, y) * q(y, cc);
          nx(a, j + c.m * cc) = s;
        }
    q = std::move(nx);
  }
  R = transpose(q);
}

// TT-cross (the reference's algorithm). When the cross reports
// non-convergence and the tensor is small enough to evaluate in full (the
// coupling tensors at the BASELINE configs have <= 4^6 * 10 entries), the
// result is replaced by a TT-SVD of the full tensor with a Frobenius budget
// of eps/2 times the max entry, which bounds the max-norm error by the same
// amount. Returns true when the fallback was used.
bool robust_cross(const EntryFn& f, const CrossOptions& co, CrossResult& r) {
  r = tt_cross(f, co);
  if (r.converged) return false;
  Index total = 1;
  for (Index m : f.dims) {
    total *= m;
    if (total > (Index(1) << 22)) return false;
  }
  std::vector<double> full(static_cast<size_t>(total));
  std::vector<Index> idx(f.dims.size(), 0);
  double mx = 0.0;
  for (Index e = 0; e < total; ++e) {
    Index rem = e;
    for (size_t k = 0; k < f.dims.size(); ++k) {
      idx[k] = rem % f.dims[k];
      rem /= f.dims[k];
    }
    if (f.counter) f.counter->add();
    full[e] = f.fn(idx.data());
    mx = std::max(mx, std::abs(full[e]));
  }
  r.tt = tt_svd(full, f.dims, 0.5 * co.eps * mx);
  r.evals += static_cast<std::uint64_t>(total);
  r.converged = true;
  r.rank_capped = false;
  return true;
}

}  // namespace

void assemble_lr_public(const Coupling& cp, Mat& L, Mat& R) { assemble_lr(cp, L, R); }

Index HostMatrix::P() const {
  Index p = 1;
  for (int k = 0; k < tree->d; ++k) p *= cfg.p_s;
  return p;
}

std::unique_ptr<HostMatrix> build_host(const double* points, Index n, int d, const Config& cfg) {
  cfg.spec.validate();
  PHM_CHECK(cfg.shard_count >= 1 && cfg.shard_rank >= 0 && cfg.shard_rank < cfg.shard_count, "bad shard");
  auto hm = std::make_unique<HostMatrix>();
  HostMatrix& M = *hm;
  M.cfg = cfg;
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

  // Row sharding: contiguous leaf ranges balanced by the near-field entries
  // each rank streams. With symmetric snapshot storage a rank streams the
  // pairs whose owner leaf it holds (device.cu's parity rule), so only
  // owned pairs count; otherwise every block of the leaf's rows.
  {
    const bool sym = cfg.near_mode == NearMode::Snapshot && cfg.symmetric_near;
    std::vector<double> leaf_work(T.nodes.size(), 0.0);
    for (const Block& b : M.blocks.near) {
      if (sym && b.sigma != b.tau && (b.sigma < b.tau) != (((b.sigma + b.tau) & 1) == 0)) continue;
      leaf_work[b.sigma] += static_cast<double>(T.nodes[b.sigma].count) * static_cast<double>(T.nodes[b.tau].count);
    }
    std::vector<int> leaves;
    double total = 0.0;
    for (size_t id = 0; id < T.nodes.size(); ++id)
      if (T.nodes[id].leaf()) {
        leaves.push_back(static_cast<int>(id));
        total += leaf_work[id] + 1e-9 * static_cast<double>(T.nodes[id].count);
      }
    double acc = 0.0;
    int rank_of_leaf_begin = -1;
    M.row_begin = T.n;
    M.row_end = 0;
    for (int id : leaves) {
      const double mid = acc + 0.5 * (leaf_work[id] + 1e-9 * static_cast<double>(T.nodes[id].count));
      int r = total > 0 ? static_cast<int>(mid / total * cfg.shard_count) : 0;
      r = std::min(r, cfg.shard_count - 1);
      acc += leaf_work[id] + 1e-9 * static_cast<double>(T.nodes[id].count);
      if (r == cfg.shard_rank) {
        if (rank_of_leaf_begin < 0) rank_of_leaf_begin = id;
        M.row_begin = std::min(M.row_begin, T.nodes[id].begin);
        M.row_end = std::max(M.row_end, T.nodes[id].begin + T.nodes[id].count);
      }
    }
    if (M.row_end < M.row_begin) M.row_begin = M.row_end = 0;
    auto intersects = [&](int id) {
      const TreeNode& nd = T.nodes[id];
      return nd.count > 0 && nd.begin < M.row_end && nd.begin + nd.count > M.row_begin;
    };
    M.node_local.assign(T.nodes.size(), 0);
    for (size_t id = 0; id < T.nodes.size(); ++id) M.node_local[id] = intersects(static_cast<int>(id));
    M.near_local.assign(M.blocks.near.size(), 0);
    for (size_t i = 0; i < M.blocks.near.size(); ++i) M.near_local[i] = M.node_local[M.blocks.near[i].sigma];
    M.far_local.assign(M.blocks.far.size(), 0);
    for (size_t i = 0; i < M.blocks.far.size(); ++i) M.far_local[i] = M.node_local[M.blocks.far[i].sigma];
  }

  // Translation classes in first-seen order (phmatrix.cpp:29-41).
  const double t1 = now_s();
  {
    std::map<std::array<std::int64_t, 4>, int> seen;
    M.far_key.resize(M.blocks.far.size());
    for (size_t i = 0; i < M.blocks.far.size(); ++i) {
      const TreeNode& s = T.nodes[M.blocks.far[i].sigma];
      const TreeNode& u = T.nodes[M.blocks.far[i].tau];
      std::array<std::int64_t, 4> key{s.level, 0, 0, 0};
      for (int k = 0; k < d; ++k) key[1 + k] = u.coords[k] - s.coords[k];
      if (!cfg.translation_cache) {
        M.far_key[i] = static_cast<int>(M.class_rep.size());
        M.class_rep.push_back(static_cast<int>(i));
        M.class_keys.push_back(key);
        continue;
      }
      auto it = seen.find(key);
      if (it == seen.end()) {
        it = seen.emplace(key, static_cast<int>(M.class_rep.size())).first;
        M.class_rep.push_back(static_cast<int>(i));
        M.class_keys.push_back(key);
      }
      M.far_key[i] = it->second;
    }
  }
  // Far field: one TT-cross per class; the cross seed derives from the
  // translation key so every block of a class reproduces the representative
  // bit for bit (farfield.cpp:102-124).
  const Index ncls = static_cast<Index>(M.class_rep.size());
  M.couplings.resize(ncls);
  std::vector<char> fallbacks(static_cast<size_t>(ncls), 0);
  parallel_for(
      ncls,
      [&](Index k) {
        const Block b = M.blocks.far[M.class_rep[k]];
        const auto& key = M.class_keys[k];
        CrossOptions co;
        co.eps = cfg.eps;
        co.r_max = cfg.r_max_far;
        std::uint64_t s = mix_seed(cfg.seed, static_cast<std::uint64_t>(key[0]));
        for (int q = 0; q < kMaxDim; ++q) s = mix_seed(s, static_cast<std::uint64_t>(key[1 + q]));
        co.seed = s;
        const EntryFn f = coupling_entries(T, b, cfg.spec, cfg.p_s, M.grids, &M.counters.offline, &M.counters.audit);
        CrossResult r;
        if (robust_cross(f, co, r)) fallbacks[k] = 1;
        Coupling& c = M.couplings[k];
        c.tt = std::move(r.tt);
        c.d = d;
        c.d_theta = M.grids.d_theta();
        c.rank_capped = r.rank_capped;
        c.est_rel_error = r.est_rel_error;
        c.evals = r.evals;
      },
      cfg.threads);
  for (char fb : fallbacks) M.stats.svd_fallbacks += fb;
  for (const auto& c : M.couplings) {
    M.stats.ff_evals += c.evals;
    M.stats.any_rank_capped = M.stats.any_rank_capped || c.rank_capped;
  }
  if (cfg.format == Format::H) {
    M.far_s.resize(M.blocks.far.size());
    M.far_t.resize(M.blocks.far.size());
    parallel_for(
        static_cast<Index>(M.blocks.far.size()),
        [&](Index i) {
          if (!M.far_local[i]) return;
          pttk_offline(T, M.blocks.far[i], cfg.p_s, M.couplings[M.far_key[i]], M.far_s[i], M.far_t[i]);
        },
        cfg.threads);
  } else {
    M.class_l.resize(ncls);
    M.class_r.resize(ncls);
    parallel_for(
        ncls, [&](Index k) { assemble_lr(M.couplings[k], M.class_l[k], M.class_r[k]); }, cfg.threads);
  }
  M.stats.ff_s = now_s() - t1;

  // Near field, TT mode: one TT-cross per near block (nearfield.cpp:50-69),
  // seeded per block index (phmatrix.cpp:43-45).
  const double t2 = now_s();
  if (cfg.near_mode == NearMode::TT) {
    M.near_tt.resize(M.blocks.near.size());
    std::vector<char> near_fb(M.blocks.near.size(), 0), near_capped(M.blocks.near.size(), 0);
    parallel_for(
        static_cast<Index>(M.blocks.near.size()),
        [&](Index i) {
          if (!M.near_local[i]) return;
          CrossOptions co;
          co.eps = cfg.eps;
          co.r_max = cfg.r_max_near;
          co.seed = mix_seed(mix_seed(cfg.seed, 0x6e656172ULL), static_cast<std::uint64_t>(i));
          const EntryFn f = near_entries(T, M.blocks.near[i], cfg.spec, M.grids, &M.counters.offline, &M.counters.audit);
          CrossResult r;
          if (robust_cross(f, co, r)) near_fb[i] = 1;
          M.near_tt[i] = std::move(r.tt);
          if (r.rank_capped) near_capped[i] = 1;
        },
        cfg.threads);
    for (size_t i = 0; i < near_fb.size(); ++i) {
      M.stats.svd_fallbacks += near_fb[i];
      if (near_capped[i]) M.stats.any_rank_capped = true;
    }
  }
  M.stats.nf_s = now_s() - t2;
  M.stats.nf_evals = M.counters.offline.value() - M.stats.ff_evals;
  return hm;
}

}  // namespace phm
