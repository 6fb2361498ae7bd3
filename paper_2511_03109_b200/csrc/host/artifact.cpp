// "HMAT" v1 artifact, byte-compatible with the reference's
// save_parametric / load_parametric_{h,h2} (proj/src/serialize.cpp:14-269):
// little-endian PODs; config, points (Eigen column-major), far / near block
// lists (validated against the rebuilt tree on load), translation keys,
// coupling TTs, H-form S/T matrices, near-field TTs. This makes the
// reference's offline `phmat build --artifact` output loadable straight into
// the GPU instantiate, and lets this build write
// artifacts the reference can read.
#include <cstring>
#include <fstream>
#include <map>

#include "phm.hpp"

namespace phm {

namespace {

constexpr std::uint32_t kMagic = 0x54414d48;  // "HMAT"
constexpr std::uint32_t kVersion = 1;

struct Out {
  std::ofstream f;
  explicit Out(const std::string& p) : f(p, std::ios::binary) {
    if (!f) throw std::runtime_error("cannot open artifact for writing: " + p);
  }
  template <typename T>
  void put(const T& v) {
    f.write(reinterpret_cast<const char*>(&v), sizeof(T));
  }
  void put_doubles(const double* p, Index n) { f.write(reinterpret_cast<const char*>(p), n * sizeof(double)); }
};

struct In {
  std::ifstream f;
  explicit In(const std::string& p) : f(p, std::ios::binary) {
    if (!f) throw std::runtime_error("cannot open artifact: " + p);
  }
  template <typename T>
  T get() {
    T v;
    f.read(reinterpret_cast<char*>(&v), sizeof(T));
    if (!f) throw std::runtime_error("truncated artifact");
    return v;
  }
  void get_doubles(double* p, Index n) {
    f.read(reinterpret_cast<char*>(p), n * sizeof(double));
    if (!f) throw std::runtime_error("truncated artifact");
  }
};

void put_tt(Out& o, const TTTensor& tt) {
  o.put<std::uint8_t>(static_cast<std::uint8_t>(tt.order()));
  for (const TTCore& c : tt.cores) {
    o.put<Index>(c.r0);
    o.put<Index>(c.m);
    o.put<Index>(c.r1);
    o.put_doubles(c.data.data(), c.size());
  }
}

TTTensor get_tt(In& in) {
  TTTensor tt;
  const int q = in.get<std::uint8_t>();
  for (int k = 0; k < q; ++k) {
    TTCore c;
    c.r0 = in.get<Index>();
    c.m = in.get<Index>();
    c.r1 = in.get<Index>();
    if (c.r0 < 1 || c.m < 1 || c.r1 < 1 || c.r0 * c.m * c.r1 > (Index(1) << 34))
      throw std::runtime_error("artifact: bad TT core shape");
    c.data.resize(static_cast<size_t>(c.size()));
    in.get_doubles(c.data.data(), c.size());
    tt.cores.push_back(std::move(c));
  }
  if (tt.cores.empty() || tt.cores.front().r0 != 1 || tt.cores.back().r1 != 1)
    throw std::logic_error("phmat: TTTensor: boundary ranks must be 1");
  for (int k = 0; k + 1 < q; ++k)
    if (tt.cores[k].r1 != tt.cores[k + 1].r0) throw std::logic_error("phmat: TTTensor: rank chain mismatch");
  return tt;
}

void put_mat(Out& o, const Mat& m) {
  o.put<Index>(m.rows);
  o.put<Index>(m.cols);
  o.put_doubles(m.a.data(), m.rows * m.cols);
}

Mat get_mat(In& in) {
  const Index r = in.get<Index>(), c = in.get<Index>();
  Mat m(r, c);
  in.get_doubles(m.a.data(), r * c);
  return m;
}

}  // namespace

bool artifact_is_h2(const std::string& path) {
  In in(path);
  if (in.get<std::uint32_t>() != kMagic) throw std::runtime_error("not a phmat artifact: " + path);
  if (in.get<std::uint32_t>() != kVersion) throw std::runtime_error("unsupported artifact version");
  return in.get<std::uint8_t>() != 0;
}

void write_artifact(const HostMatrix& M, const std::string& path, const std::function<TTTensor(Index)>& near_tt) {
  const Config& cfg = M.cfg;
  if (cfg.spec.family > kMatern || cfg.spec.amplitude)
    throw std::invalid_argument("HMAT v1 stores only the reference's kernel families (e, tps, se, mc, mn)");
  for (int p : cfg.p_theta)
    if (p != cfg.p_theta[0]) throw std::invalid_argument("HMAT v1 stores one p_theta for every parameter");
  if (cfg.shard_count != 1) throw std::invalid_argument("cannot save a row shard");
  const Tree& T = *M.tree;
  Out o(path);
  o.put(kMagic);
  o.put(kVersion);
  o.put<std::uint8_t>(cfg.format == Format::H2 ? 1 : 0);
  o.put<std::uint8_t>(static_cast<std::uint8_t>(cfg.spec.family));
  o.put<std::int32_t>(cfg.spec.d_theta());
  for (const Interval& iv : cfg.spec.box) {
    o.put<double>(iv.lo);
    o.put<double>(iv.hi);
  }
  o.put<std::int32_t>(cfg.l_max);
  o.put<std::int32_t>(cfg.p_s);
  o.put<std::int32_t>(cfg.p_theta[0]);
  o.put<double>(cfg.eps);
  o.put<double>(cfg.eta);
  o.put<Index>(cfg.r_max_far);
  o.put<Index>(cfg.r_max_near);
  o.put<std::uint64_t>(cfg.seed);
  o.put<std::uint8_t>(cfg.near_mode == NearMode::Direct ? 1 : 0);  // snapshots are full-rank TTs
  o.put<std::uint8_t>(cfg.translation_cache ? 1 : 0);
  o.put<std::int32_t>(T.d);
  o.put<Index>(T.n);
  for (int k = 0; k < T.d; ++k) {
    o.put<double>(T.nodes[0].box.lo[k]);
    o.put<double>(T.nodes[0].box.hi[k]);
  }
  for (int k = 0; k < T.d; ++k)  // Eigen column-major n x d
    for (Index i = 0; i < T.n; ++i) o.put<double>(T.points[i * T.d + k]);
  o.put<Index>(static_cast<Index>(M.blocks.far.size()));
  for (const Block& b : M.blocks.far) {
    o.put<std::int32_t>(b.sigma);
    o.put<std::int32_t>(b.tau);
  }
  o.put<Index>(static_cast<Index>(M.blocks.near.size()));
  for (const Block& b : M.blocks.near) {
    o.put<std::int32_t>(b.sigma);
    o.put<std::int32_t>(b.tau);
  }
  // far_key: the translation-class id per far block (phmatrix.cpp:62-65)
  std::vector<int> key_of(M.blocks.far.size());
  {
    std::map<std::array<std::int64_t, 4>, int> seen;
    for (size_t i = 0; i < M.blocks.far.size(); ++i) {
      const TreeNode& s = T.nodes[M.blocks.far[i].sigma];
      const TreeNode& u = T.nodes[M.blocks.far[i].tau];
      std::array<std::int64_t, 4> key{s.level, 0, 0, 0};
      for (int k = 0; k < T.d; ++k) key[1 + k] = u.coords[k] - s.coords[k];
      auto it = seen.emplace(key, static_cast<int>(seen.size())).first;
      key_of[i] = it->second;
    }
  }
  o.put<Index>(static_cast<Index>(key_of.size()));
  for (int k : key_of) o.put<std::int32_t>(k);
  o.put<Index>(static_cast<Index>(M.couplings.size()));
  for (const Coupling& c : M.couplings) {
    o.put<std::int32_t>(c.d);
    o.put<std::int32_t>(c.d_theta);
    o.put<std::uint8_t>(c.rank_capped ? 1 : 0);
    o.put<double>(c.est_rel_error);
    o.put<std::uint64_t>(c.evals);
    put_tt(o, c.tt);
  }
  if (cfg.format == Format::H)
    for (size_t i = 0; i < M.blocks.far.size(); ++i) {
      put_mat(o, M.far_s[i]);
      put_mat(o, M.far_t[i]);
    }
  const Index nnear = cfg.near_mode == NearMode::Direct ? 0 : static_cast<Index>(M.blocks.near.size());
  o.put<Index>(nnear);
  for (Index b = 0; b < nnear; ++b) {
    const Block blk = M.blocks.near[b];
    o.put<Index>(T.nodes[blk.sigma].count);
    o.put<Index>(T.nodes[blk.tau].count);
    o.put<std::uint8_t>(0);
    o.put<double>(0.0);
    o.put<std::uint64_t>(0);
    put_tt(o, near_tt(b));
  }
  if (!o.f) throw std::runtime_error("failed writing artifact: " + path);
}

std::unique_ptr<HostMatrix> read_artifact(const std::string& path, int threads) {
  In in(path);
  if (in.get<std::uint32_t>() != kMagic) throw std::runtime_error("not a phmat artifact: " + path);
  if (in.get<std::uint32_t>() != kVersion) throw std::runtime_error("unsupported artifact version");
  auto hm = std::make_unique<HostMatrix>();
  HostMatrix& M = *hm;
  Config& cfg = M.cfg;
  cfg.format = in.get<std::uint8_t>() != 0 ? Format::H2 : Format::H;
  cfg.spec.family = in.get<std::uint8_t>();
  const int dt = in.get<std::int32_t>();
  if (dt < 1 || dt > 3) throw std::runtime_error("artifact: bad theta dimension");
  cfg.spec.box.resize(dt);
  for (Interval& iv : cfg.spec.box) {
    iv.lo = in.get<double>();
    iv.hi = in.get<double>();
  }
  cfg.l_max = in.get<std::int32_t>();
  cfg.p_s = in.get<std::int32_t>();
  cfg.p_theta.assign(1, in.get<std::int32_t>());
  cfg.eps = in.get<double>();
  cfg.eta = in.get<double>();
  cfg.r_max_far = in.get<Index>();
  cfg.r_max_near = in.get<Index>();
  cfg.seed = in.get<std::uint64_t>();
  cfg.near_mode = in.get<std::uint8_t>() == 0 ? NearMode::TT : NearMode::Direct;
  cfg.translation_cache = in.get<std::uint8_t>() != 0;
  cfg.threads = threads;
  cfg.spec.validate();
  const int d = in.get<std::int32_t>();
  const Index n = in.get<Index>();
  if (d < 1 || d > kMaxDim || n < 1) throw std::runtime_error("artifact: bad point set header");
  Box root;
  root.d = d;
  for (int k = 0; k < d; ++k) {
    root.lo[k] = in.get<double>();
    root.hi[k] = in.get<double>();
  }
  std::vector<double> colmajor(static_cast<size_t>(n * d)), pts(static_cast<size_t>(n * d));
  in.get_doubles(colmajor.data(), n * d);
  for (Index i = 0; i < n; ++i)
    for (int k = 0; k < d; ++k) pts[i * d + k] = colmajor[i + k * n];
  // rebuild and validate the structure (serialize.cpp:215-232)
  M.tree = std::make_unique<Tree>(pts.data(), n, d, root, cfg.l_max);
  const Tree& T = *M.tree;
  M.blocks = build_blocks(T, cfg.resolved_eta(d));
  M.grids = make_theta_grids(cfg.spec, cfg.p_theta);
  auto check = [&](const std::vector<Block>& rebuilt) {
    const Index count = in.get<Index>();
    if (count != static_cast<Index>(rebuilt.size()))
      throw std::runtime_error("artifact block topology does not match the rebuilt tree");
    for (const Block& b : rebuilt)
      if (in.get<std::int32_t>() != b.sigma || in.get<std::int32_t>() != b.tau)
        throw std::runtime_error("artifact block topology does not match the rebuilt tree");
  };
  check(M.blocks.far);
  check(M.blocks.near);
  const Index nkeys = in.get<Index>();
  if (nkeys != static_cast<Index>(M.blocks.far.size())) throw std::runtime_error("artifact: key count mismatch");
  std::vector<int> key(static_cast<size_t>(nkeys));
  for (Index i = 0; i < nkeys; ++i) key[i] = in.get<std::int32_t>();
  const Index ncpl = in.get<Index>();
  std::vector<Coupling> cpl(static_cast<size_t>(ncpl));
  for (Coupling& c : cpl) {
    c.d = in.get<std::int32_t>();
    c.d_theta = in.get<std::int32_t>();
    c.rank_capped = in.get<std::uint8_t>() != 0;
    c.est_rel_error = in.get<double>();
    c.evals = in.get<std::uint64_t>();
    c.tt = get_tt(in);
    if (c.d != d || c.d_theta != dt || c.tt.order() != 2 * d + dt)
      throw std::runtime_error("artifact: coupling shape does not match the config");
  }
  // classes: with the cache on, couplings are per key (first-seen order);
  // with it off, per far block.
  if (cfg.translation_cache) {
    for (Index i = 0; i < nkeys; ++i)
      if (key[i] < 0 || key[i] >= ncpl) throw std::runtime_error("artifact: far key out of range");
    M.far_key = key;
    M.couplings = std::move(cpl);
  } else {
    if (ncpl != nkeys) throw std::runtime_error("artifact: coupling count mismatch");
    M.far_key.resize(static_cast<size_t>(nkeys));
    for (Index i = 0; i < nkeys; ++i) M.far_key[i] = static_cast<int>(i);
    M.couplings = std::move(cpl);
  }
  M.class_rep.assign(M.couplings.size(), -1);
  M.class_keys.resize(M.couplings.size());
  for (size_t i = 0; i < M.blocks.far.size(); ++i) {
    const int k = M.far_key[i];
    if (M.class_rep[k] >= 0) continue;
    M.class_rep[k] = static_cast<int>(i);
    const TreeNode& s = T.nodes[M.blocks.far[i].sigma];
    const TreeNode& u = T.nodes[M.blocks.far[i].tau];
    M.class_keys[k] = {s.level, 0, 0, 0};
    for (int q = 0; q < d; ++q) M.class_keys[k][1 + q] = u.coords[q] - s.coords[q];
  }
  if (cfg.format == Format::H) {
    M.far_s.resize(M.blocks.far.size());
    M.far_t.resize(M.blocks.far.size());
    for (size_t i = 0; i < M.blocks.far.size(); ++i) {
      M.far_s[i] = get_mat(in);
      M.far_t[i] = get_mat(in);
    }
  } else {
    M.class_l.resize(M.couplings.size());
    M.class_r.resize(M.couplings.size());
    parallel_for(
        static_cast<Index>(M.couplings.size()),
        [&](Index k) { assemble_lr_public(M.couplings[k], M.class_l[k], M.class_r[k]); }, threads);
  }
  const Index nnear = in.get<Index>();
  if (cfg.near_mode == NearMode::TT) {
    if (nnear != static_cast<Index>(M.blocks.near.size())) throw std::runtime_error("artifact: near count mismatch");
    M.near_tt.resize(static_cast<size_t>(nnear));
    for (Index b = 0; b < nnear; ++b) {
      const Block blk = M.blocks.near[b];
      const Index rows = in.get<Index>(), cols = in.get<Index>();
      in.get<std::uint8_t>();
      in.get<double>();
      in.get<std::uint64_t>();
      M.near_tt[b] = get_tt(in);
      if (rows != T.nodes[blk.sigma].count || cols != T.nodes[blk.tau].count ||
          M.near_tt[b].cores[0].m != rows * cols || M.near_tt[b].order() != 1 + dt)
        throw std::runtime_error("artifact: near block shape mismatch");
    }
  } else if (nnear != 0) {
    throw std::runtime_error("artifact: direct near mode with stored near blocks");
  }
  // whole matrix on one device
  M.row_begin = 0;
  M.row_end = T.n;
  M.node_local.assign(T.nodes.size(), 0);
  for (size_t id = 0; id < T.nodes.size(); ++id) M.node_local[id] = T.nodes[id].count > 0;
  M.near_local.assign(M.blocks.near.size(), 1);
  M.far_local.assign(M.blocks.far.size(), 1);
  return hm;
}

}  // namespace phm
