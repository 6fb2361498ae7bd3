// Host structure: RNG, kernels, cluster tree, block lists, Chebyshev grids.
// Bit-exact with the reference where the reference pins the arithmetic
// (proj/src/geometry.cpp, proj/src/chebyshev.cpp:10-69).
#include <algorithm>
#include <cmath>
#include <cstdlib>
#include <limits>
#include <mutex>
#include <thread>

#include "phm.hpp"

namespace phm {

// ------------------------------------------------------------------ common
double Rng::normal() {
  // Box-Muller on (0,1]: u1 = 1 - uniform() avoids log(0).
  const double u1 = 1.0 - uniform();
  const double u2 = uniform();
  return std::sqrt(-2.0 * std::log(u1)) * std::cos(6.283185307179586476925286766559 * u2);
}

std::uint64_t mix_seed(std::uint64_t a, std::uint64_t b) {
  std::uint64_t z = a + 0x9e3779b97f4a7c15ULL * (b + 1);
  z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
  z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
  return z ^ (z >> 31);
}

int max_threads() {
  if (const char* env = std::getenv("PHMAT_THREADS")) {
    const int t = std::atoi(env);
    if (t >= 1) return t;
  }
  const unsigned hw = std::thread::hardware_concurrency();
  return hw ? static_cast<int>(hw) : 1;
}

void parallel_for(Index n, const std::function<void(Index)>& fn, int threads) {
  if (threads <= 0) threads = max_threads();
  threads = static_cast<int>(std::min<Index>(threads, n));
  if (threads <= 1) {
    for (Index i = 0; i < n; ++i) fn(i);
    return;
  }
  std::atomic<Index> next{0};
  std::exception_ptr err;
  std::mutex mu;
  auto work = [&] {
    for (;;) {
      const Index i = next.fetch_add(1, std::memory_order_relaxed);
      if (i >= n) return;
      try {
        fn(i);
      } catch (...) {
        std::lock_guard<std::mutex> lk(mu);
        if (!err) err = std::current_exception();
        return;
      }
    }
  };
  std::vector<std::thread> pool;
  pool.reserve(threads - 1);
  for (int t = 1; t < threads; ++t) pool.emplace_back(work);
  work();
  for (auto& th : pool) th.join();
  if (err) std::rethrow_exception(err);
}

// ----------------------------------------------------------------- kernels
void KernelSpec::validate() const {
  if (family < kExp || family > kMatern52) throw std::invalid_argument("unknown kernel family");
  const int expected = shape_params() + (amplitude ? 1 : 0);
  if (d_theta() != expected)
    throw std::invalid_argument("kernel expects " + std::to_string(expected) + " parameter(s)");
  for (const Interval& iv : box)
    if (!(iv.lo <= iv.hi)) throw std::invalid_argument("empty theta interval");
  if (!(box[0].lo > 0.0)) throw std::invalid_argument("length scale lower bound must be positive");
  if (family == kMatern && !(box[1].lo >= 0.5))
    throw std::invalid_argument("matern smoothness lower bound must be >= 0.5");
}

double kernel_value(const KernelSpec& spec, double r, const double* th) {
  const double l = th[0];
  double v;
  switch (spec.family) {
    case kExp: v = std::exp(-r / l); break;
    case kTps: {
      if (r == 0.0) {
        v = 0.0;
        break;
      }
      const double s = r / l;
      v = s * s * std::log(s);
      break;
    }
    case kSe: {
      const double s = r / l;
      v = std::exp(-s * s);
      break;
    }
    case kMc: {
      const double s = r / l;
      v = std::sqrt(1.0 + s * s);
      break;
    }
    case kMatern: {
      const double nu = th[1];
      if (r == 0.0) {
        v = 1.0;
        break;
      }
      const double z = std::sqrt(2.0 * nu) * r / l;
      v = std::pow(2.0, 1.0 - nu) / std::tgamma(nu) * std::pow(z, nu) * std::cyl_bessel_k(nu, z);
      break;
    }
    case kGauss: {
      const double s = r / l;
      v = std::exp(-0.5 * s * s);
      break;
    }
    case kMatern32: {
      const double s = std::sqrt(3.0) * r / l;
      v = (1.0 + s) * std::exp(-s);
      break;
    }
    case kMatern52: {
      const double s = std::sqrt(5.0) * r / l;
      v = (1.0 + s + s * s / 3.0) * std::exp(-s);
      break;
    }
    default: throw std::invalid_argument("unknown kernel family");
  }
  if (spec.amplitude) v *= th[spec.shape_params()];
  return v;
}

// ---------------------------------------------------------------- geometry
double Box::diam() const {
  double s = 0.0;
  for (int k = 0; k < d; ++k) {
    const double w = hi[k] - lo[k];
    s += w * w;
  }
  return std::sqrt(s);
}

double box_dist(const Box& a, const Box& b) {
  PHM_CHECK(a.d == b.d, "dist: dimension mismatch");
  double s = 0.0;
  for (int k = 0; k < a.d; ++k) {
    const double below = std::max(0.0, a.lo[k] - b.hi[k]);
    const double above = std::max(0.0, b.lo[k] - a.hi[k]);
    s += below * below + above * above;
  }
  return std::sqrt(s);
}

bool admissible(const Box& a, const Box& b, double eta) {
  PHM_CHECK(eta > 0.0, "is_admissible: eta must be positive");
  return std::max(a.diam(), b.diam()) <= eta * box_dist(a, b);
}

double Tree::level_side(int level, int k) const {
  return (nodes[0].box.hi[k] - nodes[0].box.lo[k]) * std::ldexp(1.0, -level);
}

namespace {

// Allocates the node skeleton in the reference's id order: a node's 2^d
// children get consecutive ids at split time, then each child is split in
// turn (depth first), geometry.cpp:71-108.
void grow(std::vector<TreeNode>& nodes, int id, int d, int l_max) {
  if (nodes[id].level >= l_max) return;
  const int nc = 1 << d;
  const TreeNode par = nodes[id];
  std::array<double, kMaxDim> mid{};
  for (int k = 0; k < d; ++k) mid[k] = 0.5 * (par.box.lo[k] + par.box.hi[k]);
  const int first = static_cast<int>(nodes.size());
  nodes[id].first_child = first;
  for (int c = 0; c < nc; ++c) {
    TreeNode ch;
    ch.box.d = d;
    ch.level = par.level + 1;
    ch.parent = id;
    for (int k = 0; k < d; ++k) {
      const bool up = (c >> k) & 1;
      ch.box.lo[k] = up ? mid[k] : par.box.lo[k];
      ch.box.hi[k] = up ? par.box.hi[k] : mid[k];
      ch.coords[k] = 2 * par.coords[k] + (up ? 1 : 0);
    }
    nodes.push_back(ch);
  }
  for (int c = 0; c < nc; ++c) grow(nodes, first + c, d, l_max);
}

}  // namespace

Tree::Tree(const double* pts, Index n_, int d_, const Box& root, int lmax) : d(d_), l_max(lmax), n(n_) {
  PHM_CHECK(d >= 1 && d <= kMaxDim, "ClusterTree: dimension out of range");
  PHM_CHECK(root.d == d, "ClusterTree: point dimension mismatch");
  PHM_CHECK(l_max >= 0, "ClusterTree: l_max must be >= 0");
  points.assign(pts, pts + n * d);
  for (Index i = 0; i < n; ++i)
    for (int k = 0; k < d; ++k)
      if (points[i * d + k] < root.lo[k] || points[i * d + k] > root.hi[k])
        throw std::invalid_argument("ClusterTree: point outside the root box");

  TreeNode r;
  r.box = root;
  nodes.push_back(r);
  grow(nodes, 0, d, l_max);

  // Route every point to its leaf by the same midpoint comparisons the
  // reference's recursive split makes (coord > mid -> upper child).
  std::vector<int> leaf_of(static_cast<size_t>(n));
  parallel_for(
      (n + 4095) / 4096,
      [&](Index chunk) {
        const Index hi = std::min(n, (chunk + 1) * 4096);
        for (Index i = chunk * 4096; i < hi; ++i) {
          int id = 0;
          while (!nodes[id].leaf()) {
            const TreeNode& nd = nodes[id];
            int c = 0;
            for (int k = 0; k < d; ++k) {
              const double mid = 0.5 * (nd.box.lo[k] + nd.box.hi[k]);
              if (points[i * d + k] > mid) c |= 1 << k;
            }
            id = nd.first_child + c;
          }
          leaf_of[i] = id;
        }
      },
      0);

  // Stable counting sort by leaf id: leaves in id order, original index
  // ascending inside a leaf (the reference's sorted index sets).
  const int nn = static_cast<int>(nodes.size());
  std::vector<Index> cnt(nn + 1, 0);
  for (Index i = 0; i < n; ++i) ++cnt[leaf_of[i] + 1];
  for (int id = 0; id < nn; ++id) cnt[id + 1] += cnt[id];
  perm.assign(static_cast<size_t>(n), 0);
  {
    std::vector<Index> pos(cnt.begin(), cnt.end() - 1);
    for (Index i = 0; i < n; ++i) perm[pos[leaf_of[i]]++] = static_cast<std::int32_t>(i);
  }
  // Node ranges: leaves from the counting sort; internal nodes span their
  // children (descendants occupy one contiguous id range, children first).
  for (int id = nn - 1; id >= 0; --id) {
    TreeNode& nd = nodes[id];
    if (nd.leaf()) {
      nd.begin = cnt[id];
      nd.count = cnt[id + 1] - cnt[id];
    } else {
      const int nc = 1 << d;
      nd.begin = nodes[nd.first_child].begin;
      nd.count = 0;
      for (int c = 0; c < nc; ++c) nd.count += nodes[nd.first_child + c].count;
    }
  }
}

namespace {

struct BlockWalker {
  const Tree& t;
  double eta;
  BlockLists& out;
  std::vector<int>& row_pairs;
  void visit(int s, int u) {
    ++out.constructed;
    ++row_pairs[s];
    const TreeNode& a = t.nodes[s];
    const TreeNode& b = t.nodes[u];
    const bool adm = admissible(a.box, b.box, eta);
    if (!adm && !a.leaf() && !b.leaf()) {
      const int nc = 1 << t.d;
      for (int i = 0; i < nc; ++i)
        for (int j = 0; j < nc; ++j) visit(a.first_child + i, b.first_child + j);
      return;
    }
    if (a.count == 0 || b.count == 0) return;  // pruned after the decision
    (adm ? out.far : out.near).push_back({s, u});
  }
};

}  // namespace

BlockLists build_blocks(const Tree& tree, double eta) {
  BlockLists bl;
  bl.eta = eta;
  std::vector<int> row_pairs(tree.nodes.size(), 0);
  BlockWalker w{tree, eta, bl, row_pairs};
  w.visit(0, 0);
  for (int c : row_pairs) bl.c_sp = std::max(bl.c_sp, c);
  return bl;
}

// --------------------------------------------------------------- chebyshev
Grid1D cheb_grid(double lo, double hi, int p) {
  if (p < 1) throw std::invalid_argument("cheb_grid: p must be >= 1");
  PHM_CHECK(lo <= hi, "cheb_grid: empty interval");
  const double eps = std::numeric_limits<double>::epsilon();
  if (hi - lo < 16 * eps * std::max(1.0, std::abs(lo))) {
    const double pad = 8 * eps * std::max(1.0, std::abs(lo));
    lo -= pad;
    hi += pad;
  }
  Grid1D g;
  g.lo = lo;
  g.hi = hi;
  g.p = p;
  g.nodes.resize(p);
  g.weights.resize(p);
  constexpr double kPi = 3.141592653589793238462643383279502884;
  for (int k = 0; k < p; ++k) {
    const double c = std::cos((2.0 * k + 1.0) * kPi / (2.0 * p));
    g.nodes[p - 1 - k] = lo + 0.5 * (c + 1.0) * (hi - lo);
  }
  double wmax = 0.0;
  for (int k = 0; k < p; ++k) {
    double w = 1.0;
    for (int j = 0; j < p; ++j)
      if (j != k) w /= (g.nodes[k] - g.nodes[j]);
    g.weights[k] = w;
    wmax = std::max(wmax, std::abs(w));
  }
  for (double& w : g.weights) w /= wmax;
  return g;
}

void lagrange_all(const Grid1D& g, double x, double* out) {
  double den = 0.0;
  for (int j = 0; j < g.p; ++j) {
    const double diff = x - g.nodes[j];
    if (diff == 0.0) {
      for (int k = 0; k < g.p; ++k) out[k] = (k == j) ? 1.0 : 0.0;
      return;
    }
    out[j] = g.weights[j] / diff;
    den += out[j];
  }
  for (int k = 0; k < g.p; ++k) out[k] /= den;
}

ThetaGrids make_theta_grids(const KernelSpec& spec, const std::vector<int>& p_theta) {
  spec.validate();
  ThetaGrids g;
  for (int k = 0; k < spec.d_theta(); ++k) {
    const int p = p_theta.size() == 1 ? p_theta[0] : p_theta.at(k);
    g.grids.push_back(cheb_grid(spec.box[k].lo, spec.box[k].hi, p));
  }
  return g;
}

std::vector<std::vector<double>> parametric_vectors(const ThetaGrids& g, const double* theta, int n_theta) {
  PHM_CHECK(n_theta == g.d_theta(), "parametric_vectors: theta dimension mismatch");
  std::vector<std::vector<double>> v(g.d_theta());
  for (int k = 0; k < g.d_theta(); ++k) {
    const Grid1D& gr = g.grids[k];
    if (!(theta[k] >= gr.lo && theta[k] <= gr.hi))
      throw std::domain_error("parametric_vectors: theta outside the parameter box");
    v[k].resize(gr.p);
    lagrange_all(gr, theta[k], v[k].data());
  }
  return v;
}

// -------------------------------------------------------------- generators
void generate_points(Index n, int d, std::uint64_t seed, double* out) {
  PHM_CHECK(n >= 1, "generate_points: n must be >= 1");
  Rng rng(mix_seed(seed, 0x706f696eULL));
  for (Index i = 0; i < n; ++i)
    for (int k = 0; k < d; ++k) out[i * d + k] = rng.uniform();
}

// Mixture of `clusters` isotropic Gaussians (std sigma) with centres uniform
// in the unit cube, clipped to [0,1]^d (BASELINE.json config 4).
void generate_mixture_points(Index n, int d, int clusters, double sigma, std::uint64_t seed, double* out) {
  Rng rng(mix_seed(seed, 0x6d697874ULL));
  std::vector<double> centres(static_cast<size_t>(clusters * d));
  for (double& c : centres) c = rng.uniform();
  for (Index i = 0; i < n; ++i) {
    const std::uint64_t c = rng.integer(static_cast<std::uint64_t>(clusters));
    for (int k = 0; k < d; ++k) {
      const double v = centres[c * d + k] + sigma * rng.normal();
      out[i * d + k] = std::min(1.0, std::max(0.0, v));
    }
  }
}

void generate_normal(Index n, std::uint64_t seed, double* out) {
  Rng rng(mix_seed(seed, 0x6e6f726dULL));
  for (Index i = 0; i < n; ++i) out[i] = rng.normal();
}

}  // namespace phm
