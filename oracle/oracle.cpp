// ORACLE — test infrastructure only. NOT part of the product.
//
// Eigen-free CPU restatement of the reference's online path for parametric
// H / H^2 matrices (arXiv 2511.03109, reference at /root/reference/proj).
// Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
// --impl reference legs may load this library, and only as the checker or
// as the timed CPU baseline. The product (paper_2511_03109_b200/) never
// links or calls it.
//
// Parity pinning: the reference itself cannot be compiled here (hard Eigen3
// dependency, proj/CMakeLists.txt:13-18; vendored doctest/CLI11/json absent),
// so this restatement is pinned against the reference's own known-answer
// tests (ported in tests/test_oracle_pins.py) rather than against reference
// binaries. See DESIGN.md "Oracle".
//
// Every function cites the reference file:line it follows. Arithmetic order
// follows the reference wherever the reference pins it (tree boxes,
// admissibility, point ordering, barycentric weights, kron-row construction);
// where the reference delegates to Eigen (GEMV/GEMM summation order), sums
// run in ascending index order.
//
// Build: see oracle/Makefile (g++ -O2 -ffp-contract=off, no -march, like the
// reference's Release build, proj/CMakeLists.txt:6-8).

#include <algorithm>
#include <array>
#include <atomic>
#include <chrono>
#include <limits>
#include <cmath>
#include <cstdint>
#include <cstring>
#include <functional>
#include <map>
#include <memory>
#include <random>
#include <stdexcept>
#include <string>
#include <thread>
#include <unordered_map>
#include <vector>

namespace orc {

using i64 = std::int64_t;

// ---------------------------------------------------------------- common
// proj/include/phmat/common.hpp:22-33
struct Rng {
  std::mt19937_64 g;
  explicit Rng(std::uint64_t s) : g(s) {}
  double uniform() { return static_cast<double>(g() >> 11) * 0x1.0p-53; }
  double uniform(double a, double b) { return a + (b - a) * uniform(); }
  std::uint64_t integer(std::uint64_t n) { return n ? g() % n : 0; }
};

// proj/include/phmat/common.hpp:36-41 (splitmix64 step)
inline std::uint64_t mix_seed(std::uint64_t a, std::uint64_t b) {
  std::uint64_t z = a + 0x9e3779b97f4a7c15ULL * (b + 1);
  z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
  z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
  return z ^ (z >> 31);
}

// proj/src/common.cpp:10-48 — work-counter parallel_for; each index writes
// only its own outputs so results are schedule-independent.
int g_threads = 0;
int max_threads() {
  if (g_threads > 0) return g_threads;
  if (const char* env = std::getenv("PHMAT_THREADS")) {
    int t = std::atoi(env);
    if (t >= 1) return t;
  }
  unsigned hw = std::thread::hardware_concurrency();
  return hw ? static_cast<int>(hw) : 1;
}
void parallel_for(i64 n, const std::function<void(i64)>& fn) {
  int threads = static_cast<int>(std::min<i64>(max_threads(), n));
  if (threads <= 1) {
    for (i64 i = 0; i < n; ++i) fn(i);
    return;
  }
  std::atomic<i64> next{0};
  auto worker = [&]() {
    for (;;) {
      i64 i = next.fetch_add(1, std::memory_order_relaxed);
      if (i >= n) return;
      fn(i);
    }
  };
  std::vector<std::thread> pool;
  for (int t = 1; t < threads; ++t) pool.emplace_back(worker);
  worker();
  for (auto& th : pool) th.join();
}

// Column-major dense matrix (stands in for Eigen::MatrixXd).
struct Mat {
  i64 r = 0, c = 0;
  std::vector<double> a;
  Mat() = default;
  Mat(i64 rows, i64 cols) : r(rows), c(cols), a(static_cast<size_t>(rows * cols), 0.0) {}
  double& operator()(i64 i, i64 j) { return a[i + j * r]; }
  double operator()(i64 i, i64 j) const { return a[i + j * r]; }
};

Mat matmul(const Mat& A, const Mat& B) {
  if (A.c != B.r) throw std::logic_error("oracle matmul: shape");
  Mat C(A.r, B.c);
  for (i64 j = 0; j < B.c; ++j)
    for (i64 i = 0; i < A.r; ++i) {
      double s = 0.0;
      for (i64 k = 0; k < A.c; ++k) s += A(i, k) * B(k, j);
      C(i, j) = s;
    }
  return C;
}
Mat transpose(const Mat& A) {
  Mat T(A.c, A.r);
  for (i64 j = 0; j < A.c; ++j)
    for (i64 i = 0; i < A.r; ++i) T(j, i) = A(i, j);
  return T;
}
Mat identity(i64 n) {
  Mat I(n, n);
  for (i64 i = 0; i < n; ++i) I(i, i) = 1.0;
  return I;
}

// --------------------------------------------------------------- kernels
// proj/src/kernels.cpp:49-78, plus the single-parameter families and the
// amplitude parameter BASELINE.json's configs need.
enum Family { E = 0, TPS = 1, SE = 2, MC = 3, MN = 4, GAUSS = 5, M32 = 6, M52 = 7 };

int base_params(int fam) { return fam == MN ? 2 : 1; }

double kernel_value(int fam, bool amp, double r, const double* th) {
  const double lambda = th[0];
  double v = 0.0;
  switch (fam) {
    case E: v = std::exp(-r / lambda); break;
    case TPS: {
      if (r == 0.0) { v = 0.0; break; }
      const double s = r / lambda;
      v = s * s * std::log(s);
      break;
    }
    case SE: {
      const double s = r / lambda;
      v = std::exp(-s * s);
      break;
    }
    case MC: {
      const double s = r / lambda;
      v = std::sqrt(1.0 + s * s);
      break;
    }
    case MN: {
      const double nu = th[1];
      if (r == 0.0) { v = 1.0; break; }
      const double z = std::sqrt(2.0 * nu) * r / lambda;
      v = std::pow(2.0, 1.0 - nu) / std::tgamma(nu) * std::pow(z, nu) * std::cyl_bessel_k(nu, z);
      break;
    }
    case GAUSS: {
      const double s = r / lambda;
      v = std::exp(-0.5 * s * s);
      break;
    }
    case M32: {
      const double s = std::sqrt(3.0) * r / lambda;
      v = (1.0 + s) * std::exp(-s);
      break;
    }
    case M52: {
      const double s = std::sqrt(5.0) * r / lambda;
      v = (1.0 + s + s * s / 3.0) * std::exp(-s);
      break;
    }
    default: throw std::invalid_argument("oracle: unknown kernel family");
  }
  if (amp) v *= th[base_params(fam)];
  return v;
}

// -------------------------------------------------------------- geometry
// proj/include/phmat/geometry.hpp:15-47, proj/src/geometry.cpp:10-108
struct Box {
  int d = 0;
  double lo[3] = {0, 0, 0}, hi[3] = {0, 0, 0};
  double diam() const {  // geometry.cpp:10-17
    double s = 0.0;
    for (int k = 0; k < d; ++k) {
      const double w = hi[k] - lo[k];
      s += w * w;
    }
    return std::sqrt(s);
  }
};
double dist(const Box& a, const Box& b) {  // geometry.cpp:19-28
  double s = 0.0;
  for (int k = 0; k < a.d; ++k) {
    const double gl = std::max(0.0, a.lo[k] - b.hi[k]);
    const double gh = std::max(0.0, b.lo[k] - a.hi[k]);
    s += gl * gl + gh * gh;
  }
  return std::sqrt(s);
}
bool admissible(const Box& a, const Box& b, double eta) {  // geometry.cpp:30-33
  return std::max(a.diam(), b.diam()) <= eta * dist(a, b);
}

struct Node {
  Box box;
  i64 coords[3] = {0, 0, 0};
  int level = 0, parent = -1, first_child = -1;
  std::vector<std::int32_t> idx;
  bool leaf() const { return first_child < 0; }
  i64 size() const { return static_cast<i64>(idx.size()); }
};

struct Tree {
  int d = 0, l_max = 0;
  i64 n = 0;
  std::vector<double> pts;  // n x d row-major
  std::vector<Node> nodes;
  double pt(i64 i, int k) const { return pts[i * d + k]; }
  double side(int level, int k) const {  // geometry.cpp:67-69
    return (nodes[0].box.hi[k] - nodes[0].box.lo[k]) * std::ldexp(1.0, -level);
  }

  // geometry.cpp:71-108: midpoint split, coord > mid goes to the upper
  // child, child bit k = upper half in dim k, ids parent-before-children
  // (all 2^d children allocated, then each recursed in order).
  void split(int id) {
    if (nodes[id].level >= l_max) return;
    const int nc = 1 << d;
    const Node parent = nodes[id];
    double mid[3] = {0, 0, 0};
    for (int k = 0; k < d; ++k) mid[k] = 0.5 * (parent.box.lo[k] + parent.box.hi[k]);
    std::vector<std::vector<std::int32_t>> ci(nc);
    for (std::int32_t p : parent.idx) {
      int c = 0;
      for (int k = 0; k < d; ++k)
        if (pt(p, k) > mid[k]) c |= 1 << k;
      ci[c].push_back(p);
    }
    const int first = static_cast<int>(nodes.size());
    nodes[id].first_child = first;
    for (int c = 0; c < nc; ++c) {
      Node ch;
      ch.box.d = d;
      ch.level = parent.level + 1;
      ch.parent = id;
      for (int k = 0; k < d; ++k) {
        const bool up = (c >> k) & 1;
        ch.box.lo[k] = up ? mid[k] : parent.box.lo[k];
        ch.box.hi[k] = up ? parent.box.hi[k] : mid[k];
        ch.coords[k] = 2 * parent.coords[k] + (up ? 1 : 0);
      }
      ch.idx = std::move(ci[c]);
      nodes.push_back(std::move(ch));
    }
    for (int c = 0; c < nc; ++c) split(first + c);
  }

  void build(const double* p, i64 n_, int d_, const Box& root, int lmax) {
    d = d_;
    n = n_;
    l_max = lmax;
    pts.assign(p, p + n * d);
    for (i64 i = 0; i < n; ++i)
      for (int k = 0; k < d; ++k)
        if (pt(i, k) < root.lo[k] || pt(i, k) > root.hi[k])
          throw std::invalid_argument("ClusterTree: point outside the root box");
    Node r;
    r.box = root;
    r.idx.resize(n);
    for (i64 i = 0; i < n; ++i) r.idx[i] = static_cast<std::int32_t>(i);
    nodes.clear();
    nodes.push_back(std::move(r));
    split(0);
  }
};

struct BlockTree {
  std::vector<std::pair<int, int>> far, nearb;
  int c_sp = 0;
  i64 block_count = 0;
};

// geometry.cpp:124-157: DFS over pairs, sigma-child outer / tau-child inner;
// empty sides pruned after the split decision; c_sp counts every constructed
// pair per row cluster.
void recurse(const Tree& t, int s, int u, double eta, BlockTree& bt, std::unordered_map<int, int>& rc) {
  ++bt.block_count;
  ++rc[s];
  const Node& a = t.nodes[s];
  const Node& b = t.nodes[u];
  const bool adm = admissible(a.box, b.box, eta);
  if (!adm && !a.leaf() && !b.leaf()) {
    const int nc = 1 << t.d;
    for (int i = 0; i < nc; ++i)
      for (int j = 0; j < nc; ++j) recurse(t, a.first_child + i, b.first_child + j, eta, bt, rc);
    return;
  }
  if (a.size() == 0 || b.size() == 0) return;
  if (adm)
    bt.far.push_back({s, u});
  else
    bt.nearb.push_back({s, u});
}

// ------------------------------------------------------------- chebyshev
// proj/src/chebyshev.cpp:10-43
struct Grid {
  double lo = -1, hi = 1;
  int p = 1;
  std::vector<double> x, w;
};
Grid cheb_grid(double lo, double hi, int p) {
  const double eps = std::numeric_limits<double>::epsilon();
  if (hi - lo < 16 * eps * std::max(1.0, std::abs(lo))) {
    const double pad = 8 * eps * std::max(1.0, std::abs(lo));
    lo -= pad;
    hi += pad;
  }
  Grid g;
  g.lo = lo;
  g.hi = hi;
  g.p = p;
  g.x.assign(p, 0.0);
  g.w.assign(p, 0.0);
  const double pi = 3.141592653589793238462643383279502884;
  for (int k = 0; k < p; ++k) {
    const double c = std::cos((2.0 * k + 1.0) * pi / (2.0 * p));
    g.x[p - 1 - k] = lo + 0.5 * (c + 1.0) * (hi - lo);
  }
  double mx = 0.0;
  for (int k = 0; k < p; ++k) {
    double w = 1.0;
    for (int j = 0; j < p; ++j)
      if (j != k) w /= (g.x[k] - g.x[j]);
    g.w[k] = w;
    mx = std::max(mx, std::abs(w));
  }
  for (int k = 0; k < p; ++k) g.w[k] /= mx;
  return g;
}

// chebyshev.cpp:56-69 (exact-node short-circuit gives a unit vector)
void lagrange_all(const Grid& g, double x, double* out) {
  double den = 0.0;
  for (int j = 0; j < g.p; ++j) {
    const double diff = x - g.x[j];
    if (diff == 0.0) {
      for (int k = 0; k < g.p; ++k) out[k] = (k == j) ? 1.0 : 0.0;
      return;
    }
    out[j] = g.w[j] / diff;
    den += out[j];
  }
  for (int k = 0; k < g.p; ++k) out[k] /= den;
}

// chebyshev.cpp:71-86: U_{sigma,k}(i, j) = cardinal j of the box grid at point i.
std::vector<Mat> basis_factors(const Tree& t, int id, int ps) {
  const Node& nd = t.nodes[id];
  std::vector<Mat> f(t.d);
  std::vector<double> row(ps);
  for (int k = 0; k < t.d; ++k) {
    const Grid g = cheb_grid(nd.box.lo[k], nd.box.hi[k], ps);
    f[k] = Mat(nd.size(), ps);
    for (i64 i = 0; i < nd.size(); ++i) {
      lagrange_all(g, t.pt(nd.idx[i], k), row.data());
      for (int j = 0; j < ps; ++j) f[k](i, j) = row[j];
    }
  }
  return f;
}

// chebyshev.cpp:88-106: E_k(i, j) = parent cardinal j at child node i.
std::vector<Mat> transfer_factors(const Tree& t, int parent, int child, int ps) {
  std::vector<Mat> f(t.d);
  std::vector<double> row(ps);
  for (int k = 0; k < t.d; ++k) {
    const Grid pg = cheb_grid(t.nodes[parent].box.lo[k], t.nodes[parent].box.hi[k], ps);
    const Grid cg = cheb_grid(t.nodes[child].box.lo[k], t.nodes[child].box.hi[k], ps);
    f[k] = Mat(ps, ps);
    for (int i = 0; i < ps; ++i) {
      lagrange_all(pg, cg.x[i], row.data());
      for (int j = 0; j < ps; ++j) f[k](i, j) = row[j];
    }
  }
  return f;
}

// chebyshev.cpp:108-139: face-splitting products and the assembled basis.
Mat face_split(const Mat& a, const Mat& b) {
  Mat o(a.r, a.c * b.c);
  for (i64 j = 0; j < a.c; ++j)
    for (i64 k = 0; k < b.c; ++k)
      for (i64 i = 0; i < a.r; ++i) o(i, j * b.c + k) = a(i, j) * b(i, k);
  return o;
}
Mat face_split_cols(const Mat& a, const Mat& b) {
  Mat o(a.r * b.r, a.c);
  for (i64 j = 0; j < a.c; ++j)
    for (i64 i = 0; i < a.r; ++i)
      for (i64 k = 0; k < b.r; ++k) o(i * b.r + k, j) = a(i, j) * b(k, j);
  return o;
}
Mat assemble_basis(const std::vector<Mat>& f) {
  Mat u = f[0];
  for (size_t k = 1; k < f.size(); ++k) u = face_split(f[k], u);
  return u;
}

// chebyshev.cpp:152-193: d sequential mode contractions.
std::vector<double> kron_apply(const std::vector<Mat>& f, const std::vector<double>& x, bool transposed) {
  std::vector<double> z = x;
  i64 lead = 1;
  for (size_t k = 0; k < f.size(); ++k) {
    const Mat& A = f[k];
    const i64 in_k = transposed ? A.r : A.c;
    const i64 out_k = transposed ? A.c : A.r;
    const i64 trail = static_cast<i64>(z.size()) / (lead * in_k);
    std::vector<double> nx(static_cast<size_t>(lead * out_k * trail), 0.0);
    for (i64 t = 0; t < trail; ++t) {
      const double* zin = z.data() + t * lead * in_k;
      double* zo = nx.data() + t * lead * out_k;
      for (i64 o = 0; o < out_k; ++o)
        for (i64 a = 0; a < lead; ++a) {
          double s = 0.0;
          for (i64 i = 0; i < in_k; ++i) s += zin[a + i * lead] * (transposed ? A(i, o) : A(o, i));
          zo[a + o * lead] = s;
        }
    }
    z.swap(nx);
    lead *= out_k;
  }
  return z;
}

// -------------------------------------------------------------------- tt
// proj/include/phmat/tt.hpp:19-43: core (r0, m, r1), entry (a,j,c) at
// a + j*r0 + c*r0*m.
struct Core {
  i64 r0 = 1, m = 1, r1 = 1;
  std::vector<double> a;
  double at(i64 x, i64 j, i64 c) const { return a[x + j * r0 + c * r0 * m]; }
  Mat right() const {  // (r0*m) x r1 view
    Mat o(r0 * m, r1);
    o.a = a;
    return o;
  }
  Mat left() const {  // r0 x (m*r1) view
    Mat o(r0, m * r1);
    o.a = a;
    return o;
  }
  // tt.cpp:31-37: sum_j v_j G(:, j, :), zero coefficients skipped.
  Mat contract(const std::vector<double>& v) const {
    Mat o(r0, r1);
    for (i64 j = 0; j < m; ++j) {
      if (v[j] == 0.0) continue;
      for (i64 c = 0; c < r1; ++c)
        for (i64 x = 0; x < r0; ++x) o(x, c) += v[j] * at(x, j, c);
    }
    return o;
  }
};

// ------------------------------------------------------------- parametric
struct Spec {
  int fam = SE;
  bool amp = false;
  std::vector<double> lo, hi;  // one interval per parameter
  int dtheta() const { return static_cast<int>(lo.size()); }
};

// farfield.cpp:16-29 (with per-dimension p_theta, Appendix A)
std::vector<std::vector<double>> parametric_vectors(const std::vector<Grid>& grids, const double* theta) {
  std::vector<std::vector<double>> v(grids.size());
  for (size_t k = 0; k < grids.size(); ++k) {
    const Grid& g = grids[k];
    if (theta[k] < g.lo || theta[k] > g.hi)
      throw std::domain_error("parametric_vectors: theta outside the parameter box");
    v[k].assign(g.p, 0.0);
    lagrange_all(g, theta[k], v[k].data());
  }
  return v;
}

struct Coupling {  // farfield.hpp:41-55
  std::vector<Core> cores;
  int d = 0, dt = 0;
  i64 rank_left() const { return cores[d].r0; }
  i64 rank_right() const { return cores[d + dt - 1].r1; }
};

// farfield.cpp:149-155
Mat pttk_online(const Coupling& c, const std::vector<std::vector<double>>& v) {
  Mat h = identity(c.rank_left());
  for (int i = 0; i < c.dt; ++i) h = matmul(h, c.cores[c.d + i].contract(v[i]));
  return h;
}

// farfield.cpp:157-184
std::pair<Mat, Mat> assemble_LR(const Coupling& cp) {
  const int d = cp.d;
  const auto& cores = cp.cores;
  Mat l = cores[0].right();
  for (int k = 1; k < d; ++k) {
    Mat tmp = matmul(l, cores[k].left());
    Mat nl(tmp.r * cores[k].m, cores[k].r1);
    nl.a = tmp.a;
    l = nl;
  }
  const int last = static_cast<int>(cores.size()) - 1;
  Mat q = cores[last].left();
  for (int k = last - 1; k >= d + cp.dt; --k) {
    const Core& c = cores[k];
    Mat nx(c.r0, c.m * q.c);
    for (i64 cc = 0; cc < q.c; ++cc)
      for (i64 j = 0; j < c.m; ++j)
        for (i64 x = 0; x < c.r0; ++x) {
          double s = 0.0;
          for (i64 y = 0; y < c.r1; ++y) s += c.at(x, j, y) * q(y, cc);
          nx(x, j + c.m * cc) = s;
        }
    q = nx;
  }
  return {l, transpose(q)};
}

// farfield.cpp:186-212 (vec-kron chain; equals L H R^T xhat)
std::vector<double> coupling_apply(const Coupling& cp, const Mat& h, const std::vector<double>& xhat) {
  const int d = cp.d;
  const auto& cores = cp.cores;
  const int q = static_cast<int>(cores.size());
  std::vector<double> z = xhat;
  for (int i = 0; i < d; ++i) {
    const Core& c = cores[q - 1 - i];
    const i64 lead = static_cast<i64>(z.size()) / (c.m * c.r1);
    std::vector<double> out(static_cast<size_t>(lead * c.r0), 0.0);
    // out(lead x r0) = zin(lead x m r1) * left()^T, left() is r0 x (m r1)
    for (i64 x = 0; x < c.r0; ++x)
      for (i64 a = 0; a < lead; ++a) {
        double s = 0.0;
        for (i64 col = 0; col < c.m * c.r1; ++col) s += z[a + col * lead] * c.a[x + col * c.r0];
        out[a + x * lead] = s;
      }
    z.swap(out);
  }
  {
    std::vector<double> hz(static_cast<size_t>(h.r), 0.0);
    for (i64 i = 0; i < h.r; ++i) {
      double s = 0.0;
      for (i64 k = 0; k < h.c; ++k) s += h(i, k) * z[k];
      hz[i] = s;
    }
    z.swap(hz);
  }
  for (int i = 0; i < d; ++i) {
    const Core& c = cores[d - 1 - i];
    const i64 trail = static_cast<i64>(z.size()) / c.r1;
    const i64 rows = c.r0 * c.m;
    std::vector<double> out(static_cast<size_t>(rows * trail), 0.0);
    for (i64 t = 0; t < trail; ++t)
      for (i64 rr = 0; rr < rows; ++rr) {
        double s = 0.0;
        for (i64 k = 0; k < c.r1; ++k) s += c.a[rr + k * rows] * z[k + t * c.r1];
        out[rr + t * rows] = s;
      }
    z.swap(out);
  }
  return z;
}

struct NearTT {  // nearfield.hpp:15-24
  std::vector<Core> cores;
  i64 rows = 0, cols = 0;
};

// nearfield.cpp:71-80: w = I * prod contract(G_{i+1}, v_i); a = G1.right() w
Mat nearfield_online(const NearTT& nb, const std::vector<std::vector<double>>& v) {
  const auto& cores = nb.cores;
  Mat w = identity(cores[0].r1);
  for (size_t i = 0; i < v.size(); ++i) w = matmul(w, cores[i + 1].contract(v[i]));
  const i64 N = cores[0].m;
  const i64 R = cores[0].r1;
  Mat D(nb.rows, nb.cols);
  for (i64 e = 0; e < N; ++e) {
    double s = 0.0;
    for (i64 k = 0; k < R; ++k) s += cores[0].a[e + k * N] * w(k, 0);
    D.a[e] = s;
  }
  return D;
}

// ------------------------------------------------------------ the matrix
struct Matrix {
  bool h2 = true;
  Tree tree;
  BlockTree bt;
  double eta = 1.0;
  int ps = 4;
  Spec spec;
  std::vector<int> ptheta;
  std::vector<Grid> grids;
  std::vector<int> far_key, rep;
  std::vector<std::array<i64, 4>> keys;  // level, offset[3]
  std::vector<Coupling> couplings;
  std::vector<NearTT> nearblk;
  // H form (farfield.cpp:126-147) and H^2 basis (chebyshev.cpp:195-203)
  std::vector<Mat> far_s, far_t;
  std::vector<std::vector<Mat>> leaf_f, transfer;
  std::vector<Mat> class_L, class_R;
};

struct Inst {
  const Matrix* m = nullptr;
  std::vector<double> theta;
  std::vector<Mat> class_h;  // H_k(theta) per class (far_h[i] = class_h[far_key[i]])
  std::vector<Mat> near_d;
};

// phmatrix.cpp:29-41: classes in first-seen order over the far list, key =
// (level, tau.coords - sigma.coords), farfield.cpp:31-39.
void make_classes(Matrix& M) {
  std::map<std::array<i64, 4>, int> seen;
  M.far_key.assign(M.bt.far.size(), -1);
  M.rep.clear();
  M.keys.clear();
  for (size_t i = 0; i < M.bt.far.size(); ++i) {
    const Node& s = M.tree.nodes[M.bt.far[i].first];
    const Node& t = M.tree.nodes[M.bt.far[i].second];
    std::array<i64, 4> key{s.level, 0, 0, 0};
    for (int k = 0; k < M.tree.d; ++k) key[1 + k] = t.coords[k] - s.coords[k];
    auto it = seen.find(key);
    if (it == seen.end()) {
      it = seen.emplace(key, static_cast<int>(M.rep.size())).first;
      M.rep.push_back(static_cast<int>(i));
      M.keys.push_back(key);
    }
    M.far_key[i] = it->second;
  }
}

// dense_kernel_block (nearfield.cpp:82-97): kernel at theta for one block.
Mat direct_block(const Matrix& M, size_t b, const double* theta) {
  const Tree& t = M.tree;
  const Node& s = t.nodes[M.bt.nearb[b].first];
  const Node& u = t.nodes[M.bt.nearb[b].second];
  Mat D(s.size(), u.size());
  for (i64 j = 0; j < u.size(); ++j)
    for (i64 i = 0; i < s.size(); ++i) {
      double r2 = 0.0;
      for (int c = 0; c < t.d; ++c) {
        const double dl = t.pt(s.idx[i], c) - t.pt(u.idx[j], c);
        r2 += dl * dl;
      }
      D(i, j) = kernel_value(M.spec.fam, M.spec.amp, std::sqrt(r2), theta);
    }
  return D;
}

// instantiate_common, phmatrix.cpp:168-209 (TT near mode; the snapshot mode
// is a full-rank NearBlockTT)
Inst instantiate(const Matrix& M, const double* theta) {
  Inst I;
  I.m = &M;
  I.theta.assign(theta, theta + M.spec.dtheta());
  const auto v = parametric_vectors(M.grids, theta);
  I.class_h.resize(M.couplings.size());
  parallel_for(static_cast<i64>(M.couplings.size()), [&](i64 k) { I.class_h[k] = pttk_online(M.couplings[k], v); });
  I.near_d.resize(M.bt.nearb.size());
  parallel_for(static_cast<i64>(M.bt.nearb.size()), [&](i64 b) {
    if (M.nearblk[b].cores.empty())
      I.near_d[b] = direct_block(M, b, theta);  // NearMode::Direct, phmatrix.cpp:200-207
    else
      I.near_d[b] = nearfield_online(M.nearblk[b], v);
  });
  return I;
}

// NestedClusterBasis::forward, chebyshev.cpp:223-263
std::vector<std::vector<double>> forward(const Matrix& M, const double* x) {
  const Tree& t = M.tree;
  const int d = t.d, ps = M.ps;
  i64 P = 1;
  for (int k = 0; k < d; ++k) P *= ps;
  std::vector<std::vector<double>> xh(t.nodes.size());
  std::vector<double> row(static_cast<size_t>(P));
  for (int id = static_cast<int>(t.nodes.size()) - 1; id >= 0; --id) {
    const Node& nd = t.nodes[id];
    if (nd.size() == 0) continue;
    xh[id].assign(static_cast<size_t>(P), 0.0);
    if (nd.leaf()) {
      const auto& f = M.leaf_f[id];
      for (i64 i = 0; i < nd.size(); ++i) {
        const double xi = x[nd.idx[i]];
        if (xi == 0.0) continue;
        i64 len = ps;
        for (int j = 0; j < ps; ++j) row[j] = xi * f[0](i, j);
        for (int k = 1; k < d; ++k) {
          for (i64 j = ps - 1; j >= 0; --j)
            for (i64 q = 0; q < len; ++q) row[j * len + q] = f[k](i, j) * row[q];
          len *= ps;
        }
        for (i64 q = 0; q < P; ++q) xh[id][q] += row[q];
      }
    } else {
      for (int c = 0; c < (1 << d); ++c) {
        const int cid = nd.first_child + c;
        if (t.nodes[cid].size() == 0) continue;
        const auto z = kron_apply(M.transfer[cid], xh[cid], true);
        for (i64 q = 0; q < P; ++q) xh[id][q] += z[q];
      }
    }
  }
  return xh;
}

// NestedClusterBasis::backward, chebyshev.cpp:265-298
void backward(const Matrix& M, std::vector<std::vector<double>>& yh, double* y) {
  const Tree& t = M.tree;
  const int d = t.d, ps = M.ps;
  for (size_t id = 0; id < t.nodes.size(); ++id) {
    const Node& nd = t.nodes[id];
    if (nd.size() == 0 || yh[id].empty()) continue;
    if (nd.leaf()) {
      const auto& f = M.leaf_f[id];
      for (i64 i = 0; i < nd.size(); ++i) {
        std::vector<double> fold = yh[id];
        i64 len = static_cast<i64>(fold.size());
        for (int k = d - 1; k >= 1; --k) {
          len /= ps;
          std::vector<double> nx(static_cast<size_t>(len), 0.0);
          for (i64 a = 0; a < len; ++a) {
            double s = 0.0;
            for (int j = 0; j < ps; ++j) s += fold[a + j * len] * f[k](i, j);
            nx[a] = s;
          }
          for (i64 a = 0; a < len; ++a) fold[a] = nx[a];
        }
        double s = 0.0;
        for (int j = 0; j < ps; ++j) s += f[0](i, j) * fold[j];
        y[nd.idx[i]] += s;
      }
    } else {
      for (int c = 0; c < (1 << d); ++c) {
        const int cid = nd.first_child + c;
        if (t.nodes[cid].size() == 0) continue;
        const auto down = kron_apply(M.transfer[cid], yh[id], false);
        if (yh[cid].empty())
          yh[cid] = down;
        else
          for (size_t q = 0; q < down.size(); ++q) yh[cid][q] += down[q];
      }
    }
  }
}

// InstantiatedHMatrix::apply / InstantiatedH2Matrix::apply, phmatrix.cpp:227-269
void apply(const Inst& I, const double* x, double* y) {
  const Matrix& M = *I.m;
  const Tree& t = M.tree;
  std::fill(y, y + t.n, 0.0);
  if (M.h2) {
    auto xh = forward(M, x);
    std::vector<std::vector<double>> yh(t.nodes.size());
    for (size_t i = 0; i < M.bt.far.size(); ++i) {
      const int s = M.bt.far[i].first, u = M.bt.far[i].second;
      const auto z = coupling_apply(M.couplings[M.far_key[i]], I.class_h[M.far_key[i]], xh[u]);
      if (yh[s].empty())
        yh[s] = z;
      else
        for (size_t q = 0; q < z.size(); ++q) yh[s][q] += z[q];
    }
    for (size_t b = 0; b < M.bt.nearb.size(); ++b) {
      const Node& s = t.nodes[M.bt.nearb[b].first];
      const Node& u = t.nodes[M.bt.nearb[b].second];
      const Mat& D = I.near_d[b];
      for (i64 i = 0; i < s.size(); ++i) {
        double acc = 0.0;
        for (i64 j = 0; j < u.size(); ++j) acc += D(i, j) * x[u.idx[j]];
        y[s.idx[i]] += acc;
      }
    }
    backward(M, yh, y);
  } else {
    for (size_t i = 0; i < M.bt.far.size(); ++i) {
      const Node& s = t.nodes[M.bt.far[i].first];
      const Node& u = t.nodes[M.bt.far[i].second];
      const Mat& S = M.far_s[i];
      const Mat& T = M.far_t[i];
      const Mat& H = I.class_h[M.far_key[i]];
      std::vector<double> a(static_cast<size_t>(T.c), 0.0), b(static_cast<size_t>(H.r), 0.0);
      for (i64 k = 0; k < T.c; ++k) {
        double acc = 0.0;
        for (i64 j = 0; j < u.size(); ++j) acc += T(j, k) * x[u.idx[j]];
        a[k] = acc;
      }
      for (i64 r = 0; r < H.r; ++r) {
        double acc = 0.0;
        for (i64 k = 0; k < H.c; ++k) acc += H(r, k) * a[k];
        b[r] = acc;
      }
      for (i64 r = 0; r < s.size(); ++r) {
        double acc = 0.0;
        for (i64 k = 0; k < S.c; ++k) acc += S(r, k) * b[k];
        y[s.idx[r]] += acc;
      }
    }
    for (size_t b = 0; b < M.bt.nearb.size(); ++b) {
      const Node& s = t.nodes[M.bt.nearb[b].first];
      const Node& u = t.nodes[M.bt.nearb[b].second];
      const Mat& D = I.near_d[b];
      for (i64 i = 0; i < s.size(); ++i) {
        double acc = 0.0;
        for (i64 j = 0; j < u.size(); ++j) acc += D(i, j) * x[u.idx[j]];
        y[s.idx[i]] += acc;
      }
    }
  }
}

// farfield.cpp:126-147 (H form phase 3)
void pttk_offline(Matrix& M) {
  const Tree& t = M.tree;
  const int d = t.d;
  M.far_s.resize(M.bt.far.size());
  M.far_t.resize(M.bt.far.size());
  parallel_for(static_cast<i64>(M.bt.far.size()), [&](i64 i) {
    const Coupling& cp = M.couplings[M.far_key[i]];
    const auto us = basis_factors(t, M.bt.far[i].first, M.ps);
    const auto ut = basis_factors(t, M.bt.far[i].second, M.ps);
    Mat s = matmul(us[0], cp.cores[0].right());
    for (int k = 1; k < d; ++k) s = matmul(face_split(us[k], s), cp.cores[k].right());
    const int last = static_cast<int>(cp.cores.size()) - 1;
    Mat tt = matmul(cp.cores[last].left(), transpose(ut[d - 1]));
    for (int k = 1; k < d; ++k) tt = matmul(cp.cores[last - k].left(), face_split_cols(tt, transpose(ut[d - 1 - k])));
    M.far_s[i] = s;
    M.far_t[i] = transpose(tt);
  });
}

// nearfield.cpp:7-48: A_b[i + j n_sigma, k...] with r accumulated over dims
// in order; the full-rank NearBlockTT that snapshot mode stores.
NearTT snapshot_block(const Matrix& M, int s, int u) {
  const Tree& t = M.tree;
  const Node& a = t.nodes[s];
  const Node& b = t.nodes[u];
  const int dt = M.spec.dtheta();
  const int nb = base_params(M.spec.fam);  // non-amplitude parameters
  NearTT nt;
  nt.rows = a.size();
  nt.cols = b.size();
  const i64 N = a.size() * b.size();
  i64 R = 1;
  for (int k = 0; k < nb; ++k) R *= M.ptheta[k];
  Core g1;
  g1.r0 = 1;
  g1.m = N;
  g1.r1 = R;
  g1.a.assign(static_cast<size_t>(N * R), 0.0);
  double th[3] = {0, 0, 0};
  if (M.spec.amp) th[nb] = 1.0;
  for (i64 kap = 0; kap < R; ++kap) {
    i64 rem = kap;
    for (int k = 0; k < nb; ++k) {
      th[k] = M.grids[k].x[rem % M.ptheta[k]];
      rem /= M.ptheta[k];
    }
    for (i64 j = 0; j < b.size(); ++j)
      for (i64 i = 0; i < a.size(); ++i) {
        double r2 = 0.0;
        for (int c = 0; c < t.d; ++c) {
          const double dl = t.pt(a.idx[i], c) - t.pt(b.idx[j], c);
          r2 += dl * dl;
        }
        g1.a[i + j * a.size() + kap * N] = kernel_value(M.spec.fam, false, std::sqrt(r2), th);
      }
  }
  nt.cores.push_back(std::move(g1));
  // theta cores: for the non-amplitude modes the identity chain that makes
  // w = v_1 (x) v_2 (k_1 fastest); for an amplitude mode the rank-1 core of
  // the grid's node values (sigma^2 enters linearly).
  i64 rin = R;
  i64 stride = 1;
  for (int k = 0; k < nb; ++k) {
    const i64 p = M.ptheta[k];
    Core g;
    g.r0 = rin;
    g.m = p;
    g.r1 = rin / p;
    g.a.assign(static_cast<size_t>(g.r0 * g.m * g.r1), 0.0);
    // rows (k_k + p * rest) -> column rest
    for (i64 rest = 0; rest < g.r1; ++rest)
      for (i64 j = 0; j < p; ++j) g.a[(j + p * rest) + j * g.r0 + rest * g.r0 * g.m] = 1.0;
    nt.cores.push_back(std::move(g));
    rin /= p;
    stride *= p;
  }
  if (M.spec.amp) {
    Core g;
    g.r0 = 1;
    g.m = M.ptheta[nb];
    g.r1 = 1;
    g.a = M.grids[nb].x;
    nt.cores.push_back(std::move(g));
  }
  (void)dt;
  return nt;
}

}  // namespace orc

// =================================================================== C ABI
// ctypes surface for tests/ and bench.py (checker / CPU baseline only).
using namespace orc;

namespace {
thread_local std::string g_err;
template <typename F>
int guard(F&& f) {
  try {
    f();
    return 0;
  } catch (const std::domain_error& e) {
    g_err = e.what();
    return 2;
  } catch (const std::invalid_argument& e) {
    g_err = e.what();
    return 3;
  } catch (const std::logic_error& e) {
    g_err = e.what();
    return 4;
  } catch (const std::exception& e) {
    g_err = e.what();
    return 1;
  }
}
}  // namespace

extern "C" {

const char* orc_last_error() { return g_err.c_str(); }
void orc_set_threads(int t) { g_threads = t; }

// harness.cpp:174-181
void orc_generate_points(std::int64_t n, int d, std::uint64_t seed, double* out) {
  Rng rng(mix_seed(seed, 0x706f696eULL));
  for (i64 i = 0; i < n; ++i)
    for (int k = 0; k < d; ++k) out[i * d + k] = rng.uniform();
}
std::uint64_t orc_mix_seed(std::uint64_t a, std::uint64_t b) { return mix_seed(a, b); }
void orc_rng_uniform(std::uint64_t seed, std::int64_t count, double* out) {
  Rng r(seed);
  for (i64 i = 0; i < count; ++i) out[i] = r.uniform();
}
double orc_kernel_value(int fam, int amp, double r, const double* theta) {
  return kernel_value(fam, amp != 0, r, theta);
}
void orc_cheb_grid(double lo, double hi, int p, double* nodes, double* weights, double* lohi) {
  Grid g = cheb_grid(lo, hi, p);
  for (int k = 0; k < p; ++k) {
    nodes[k] = g.x[k];
    weights[k] = g.w[k];
  }
  lohi[0] = g.lo;
  lohi[1] = g.hi;
}
int orc_lagrange_all(double lo, double hi, int p, double x, double* out) {
  return guard([&] { lagrange_all(cheb_grid(lo, hi, p), x, out); });
}
int orc_box_admissible(int d, const double* alo, const double* ahi, const double* blo, const double* bhi, double eta,
                       double* diam_a, double* distance) {
  Box a, b;
  a.d = b.d = d;
  for (int k = 0; k < d; ++k) {
    a.lo[k] = alo[k];
    a.hi[k] = ahi[k];
    b.lo[k] = blo[k];
    b.hi[k] = bhi[k];
  }
  *diam_a = a.diam();
  *distance = dist(a, b);
  return admissible(a, b, eta) ? 1 : 0;
}
// fast_kron / fast_kron_transposed with d square p x p factors (row-major
// factor k at f + k*p*p, entry (i,j) at i*p + j).
void orc_fast_kron(int d, int p, const double* f, const double* x, int transposed, double* out) {
  std::vector<Mat> fs(d);
  for (int k = 0; k < d; ++k) {
    fs[k] = Mat(p, p);
    for (int i = 0; i < p; ++i)
      for (int j = 0; j < p; ++j) fs[k](i, j) = f[k * p * p + i * p + j];
  }
  i64 P = 1;
  for (int k = 0; k < d; ++k) P *= p;
  std::vector<double> xv(x, x + P);
  auto z = kron_apply(fs, xv, transposed != 0);
  std::copy(z.begin(), z.end(), out);
}

// Matrix creation: tree, blocks, classes, grids (and H^2 basis).
// family/amp/theta box/p_theta per parameter; form 0 = H, 1 = H^2.
int orc_matrix_create(const double* pts, std::int64_t n, int d, int l_max, double eta, int ps, int fam, int amp,
                      int dtheta, const double* tlo, const double* thi, const int* ptheta, int form, void** out) {
  return guard([&] {
    auto M = std::make_unique<Matrix>();
    M->h2 = form == 1;
    Box root;
    root.d = d;
    for (int k = 0; k < d; ++k) {
      root.lo[k] = 0.0;
      root.hi[k] = 1.0;
    }
    M->tree.build(pts, n, d, root, l_max);
    M->eta = eta > 0 ? eta : std::sqrt(static_cast<double>(d));
    std::unordered_map<int, int> rc;
    recurse(M->tree, 0, 0, M->eta, M->bt, rc);
    for (auto& kv : rc) M->bt.c_sp = std::max(M->bt.c_sp, kv.second);
    M->ps = ps;
    M->spec.fam = fam;
    M->spec.amp = amp != 0;
    M->spec.lo.assign(tlo, tlo + dtheta);
    M->spec.hi.assign(thi, thi + dtheta);
    M->ptheta.assign(ptheta, ptheta + dtheta);
    for (int k = 0; k < dtheta; ++k) M->grids.push_back(cheb_grid(tlo[k], thi[k], ptheta[k]));
    make_classes(*M);
    M->couplings.resize(M->rep.size());
    M->nearblk.resize(M->bt.nearb.size());
    if (M->h2) {
      const Tree& t = M->tree;
      M->leaf_f.resize(t.nodes.size());
      M->transfer.resize(t.nodes.size());
      for (size_t id = 0; id < t.nodes.size(); ++id) {
        const Node& nd = t.nodes[id];
        if (nd.leaf() && nd.size() > 0) M->leaf_f[id] = basis_factors(t, static_cast<int>(id), ps);
        if (nd.parent >= 0) M->transfer[id] = transfer_factors(t, nd.parent, static_cast<int>(id), ps);
      }
    }
    *out = M.release();
  });
}
void orc_matrix_destroy(void* m) { delete static_cast<Matrix*>(m); }

// counts[0..7] = n, d, nodes, n_near, n_far, n_classes, c_sp, block_count
void orc_matrix_counts(void* m, std::int64_t* counts) {
  const Matrix& M = *static_cast<Matrix*>(m);
  counts[0] = M.tree.n;
  counts[1] = M.tree.d;
  counts[2] = static_cast<i64>(M.tree.nodes.size());
  counts[3] = static_cast<i64>(M.bt.nearb.size());
  counts[4] = static_cast<i64>(M.bt.far.size());
  counts[5] = static_cast<i64>(M.rep.size());
  counts[6] = M.bt.c_sp;
  counts[7] = M.bt.block_count;
}
// per node: level, parent, first_child, size, coords[3]; boxes lo[3], hi[3]
void orc_matrix_nodes(void* m, std::int32_t* ints /*7 per node*/, double* boxes /*6 per node*/) {
  const Matrix& M = *static_cast<Matrix*>(m);
  for (size_t i = 0; i < M.tree.nodes.size(); ++i) {
    const Node& nd = M.tree.nodes[i];
    ints[7 * i + 0] = nd.level;
    ints[7 * i + 1] = nd.parent;
    ints[7 * i + 2] = nd.first_child;
    ints[7 * i + 3] = static_cast<std::int32_t>(nd.size());
    for (int k = 0; k < 3; ++k) ints[7 * i + 4 + k] = static_cast<std::int32_t>(nd.coords[k]);
    for (int k = 0; k < 3; ++k) {
      boxes[6 * i + k] = nd.box.lo[k];
      boxes[6 * i + 3 + k] = nd.box.hi[k];
    }
  }
}
// Tree-order permutation: concatenated leaf index sets in leaf-id order.
void orc_matrix_perm(void* m, std::int32_t* perm) {
  const Matrix& M = *static_cast<Matrix*>(m);
  i64 p = 0;
  for (const Node& nd : M.tree.nodes)
    if (nd.leaf())
      for (auto i : nd.idx) perm[p++] = i;
}
void orc_matrix_blocks(void* m, std::int32_t* nearb /*2 per*/, std::int32_t* farb /*2 per*/, std::int32_t* far_key) {
  const Matrix& M = *static_cast<Matrix*>(m);
  for (size_t i = 0; i < M.bt.nearb.size(); ++i) {
    nearb[2 * i] = M.bt.nearb[i].first;
    nearb[2 * i + 1] = M.bt.nearb[i].second;
  }
  for (size_t i = 0; i < M.bt.far.size(); ++i) {
    farb[2 * i] = M.bt.far[i].first;
    farb[2 * i + 1] = M.bt.far[i].second;
    far_key[i] = M.far_key[i];
  }
}
void orc_matrix_class_keys(void* m, std::int64_t* keys /*4 per class*/) {
  const Matrix& M = *static_cast<Matrix*>(m);
  for (size_t k = 0; k < M.keys.size(); ++k)
    for (int q = 0; q < 4; ++q) keys[4 * k + q] = M.keys[k][q];
}
void orc_matrix_theta_grid(void* m, int k, double* nodes) {
  const Matrix& M = *static_cast<Matrix*>(m);
  for (int j = 0; j < M.grids[k].p; ++j) nodes[j] = M.grids[k].x[j];
}

// Offline data handed over by the product (TT cores are offline outputs;
// parity is on the online path given identical offline data).
// cores: ncores entries of (r0, m, r1) in dims[3*i..], data concatenated.
static std::vector<Core> read_cores(int ncores, const std::int64_t* dims, const double* data) {
  std::vector<Core> cs(ncores);
  i64 off = 0;
  for (int i = 0; i < ncores; ++i) {
    cs[i].r0 = dims[3 * i];
    cs[i].m = dims[3 * i + 1];
    cs[i].r1 = dims[3 * i + 2];
    const i64 sz = cs[i].r0 * cs[i].m * cs[i].r1;
    cs[i].a.assign(data + off, data + off + sz);
    off += sz;
  }
  return cs;
}
int orc_set_coupling(void* m, int k, int ncores, const std::int64_t* dims, const double* data) {
  return guard([&] {
    Matrix& M = *static_cast<Matrix*>(m);
    M.couplings.at(k).cores = read_cores(ncores, dims, data);
    M.couplings[k].d = M.tree.d;
    M.couplings[k].dt = M.spec.dtheta();
    if (ncores != M.tree.d * 2 + M.spec.dtheta()) throw std::invalid_argument("coupling core count");
  });
}
int orc_set_near_tt(void* m, std::int64_t b, int ncores, const std::int64_t* dims, const double* data) {
  return guard([&] {
    Matrix& M = *static_cast<Matrix*>(m);
    NearTT& nt = M.nearblk.at(b);
    nt.cores = read_cores(ncores, dims, data);
    nt.rows = M.tree.nodes[M.bt.nearb[b].first].size();
    nt.cols = M.tree.nodes[M.bt.nearb[b].second].size();
    if (nt.cores[0].m != nt.rows * nt.cols) throw std::invalid_argument("near core size");
  });
}
// Snapshot mode: oracle evaluates the full-rank near tensors itself
// (near_oracle entries, nearfield.cpp:35-46). Only blocks with mask != 0
// (or all when mask == NULL) are built.
int orc_make_near_snapshots(void* m, const std::uint8_t* mask) {
  return guard([&] {
    Matrix& M = *static_cast<Matrix*>(m);
    parallel_for(static_cast<i64>(M.bt.nearb.size()), [&](i64 b) {
      if (mask && !mask[b]) return;
      M.nearblk[b] = snapshot_block(M, M.bt.nearb[b].first, M.bt.nearb[b].second);
    });
  });
}
// Snapshot column kap of near block b (length n_sigma n_tau), for K11 parity.
int orc_near_snapshot_column(void* m, std::int64_t b, std::int64_t kap, double* out) {
  return guard([&] {
    Matrix& M = *static_cast<Matrix*>(m);
    const Core& g = M.nearblk.at(b).cores.at(0);
    std::copy(g.a.begin() + kap * g.m, g.a.begin() + (kap + 1) * g.m, out);
  });
}
int orc_finalize(void* m) {
  return guard([&] {
    Matrix& M = *static_cast<Matrix*>(m);
    if (!M.h2) pttk_offline(M);
    M.class_L.resize(M.couplings.size());
    M.class_R.resize(M.couplings.size());
    for (size_t k = 0; k < M.couplings.size(); ++k) {
      auto lr = assemble_LR(M.couplings[k]);
      M.class_L[k] = lr.first;
      M.class_R[k] = lr.second;
    }
  });
}
int orc_far_st(void* m, std::int64_t i, double* s, double* t) {
  return guard([&] {
    Matrix& M = *static_cast<Matrix*>(m);
    std::copy(M.far_s.at(i).a.begin(), M.far_s[i].a.end(), s);
    std::copy(M.far_t.at(i).a.begin(), M.far_t[i].a.end(), t);
  });
}
int orc_class_LR(void* m, int k, double* L, double* R, std::int64_t* dims) {
  return guard([&] {
    Matrix& M = *static_cast<Matrix*>(m);
    dims[0] = M.class_L.at(k).r;
    dims[1] = M.class_L[k].c;
    dims[2] = M.class_R[k].r;
    dims[3] = M.class_R[k].c;
    if (L) std::copy(M.class_L[k].a.begin(), M.class_L[k].a.end(), L);
    if (R) std::copy(M.class_R[k].a.begin(), M.class_R[k].a.end(), R);
  });
}

int orc_instantiate(void* m, const double* theta, void** out) {
  return guard([&] {
    auto I = std::make_unique<Inst>(instantiate(*static_cast<Matrix*>(m), theta));
    *out = I.release();
  });
}
// Instantiate only the near blocks in mask (bounded CPU-baseline sample)
// and every class; returns wall seconds for (classes, near) separately.
int orc_instantiate_timed(void* m, const double* theta, const std::uint8_t* mask, double* secs, void** out) {
  return guard([&] {
    Matrix& M = *static_cast<Matrix*>(m);
    auto I = std::make_unique<Inst>();
    I->m = &M;
    I->theta.assign(theta, theta + M.spec.dtheta());
    auto t0 = std::chrono::steady_clock::now();
    const auto v = parametric_vectors(M.grids, theta);
    I->class_h.resize(M.couplings.size());
    parallel_for(static_cast<i64>(M.couplings.size()), [&](i64 k) { I->class_h[k] = pttk_online(M.couplings[k], v); });
    auto t1 = std::chrono::steady_clock::now();
    I->near_d.resize(M.bt.nearb.size());
    parallel_for(static_cast<i64>(M.bt.nearb.size()), [&](i64 b) {
      if (mask && !mask[b]) return;
      I->near_d[b] = nearfield_online(M.nearblk[b], v);
    });
    auto t2 = std::chrono::steady_clock::now();
    secs[0] = std::chrono::duration<double>(t1 - t0).count();
    secs[1] = std::chrono::duration<double>(t2 - t1).count();
    *out = I.release();
  });
}
void orc_inst_destroy(void* i) { delete static_cast<Inst*>(i); }
int orc_inst_class_h(void* i, int k, double* out, std::int64_t* rc) {
  return guard([&] {
    const Mat& h = static_cast<Inst*>(i)->class_h.at(k);
    rc[0] = h.r;
    rc[1] = h.c;
    if (out) std::copy(h.a.begin(), h.a.end(), out);
  });
}
int orc_inst_near(void* i, std::int64_t b, double* out) {
  return guard([&] {
    const Mat& D = static_cast<Inst*>(i)->near_d.at(b);
    std::copy(D.a.begin(), D.a.end(), out);
  });
}
// C_k = L_k H_k R_k^T (p_s^d x p_s^d, column-major)
int orc_inst_class_c(void* i, int k, double* out) {
  return guard([&] {
    Inst& I = *static_cast<Inst*>(i);
    const Matrix& M = *I.m;
    Mat c = matmul(matmul(M.class_L.at(k), I.class_h.at(k)), transpose(M.class_R.at(k)));
    std::copy(c.a.begin(), c.a.end(), out);
  });
}
// x, y length n (original point order); m right-hand sides column-major.
int orc_apply(void* i, const double* x, double* y, std::int64_t m_rhs) {
  return guard([&] {
    Inst& I = *static_cast<Inst*>(i);
    const i64 n = I.m->tree.n;
    for (i64 c = 0; c < m_rhs; ++c) apply(I, x + c * n, y + c * n);
  });
}
// Near-field-only / far-field-only partial applies restricted to a block
// mask (bounded CPU-baseline sample). part: 0 near, 1 far (coupling only).
int orc_apply_sample(void* i, const double* x, double* y, const std::uint8_t* near_mask, const std::uint8_t* far_mask,
                     double* secs) {
  return guard([&] {
    Inst& I = *static_cast<Inst*>(i);
    const Matrix& M = *I.m;
    const Tree& t = M.tree;
    std::fill(y, y + t.n, 0.0);
    auto t0 = std::chrono::steady_clock::now();
    std::vector<std::vector<double>> xh;
    if (M.h2) xh = forward(M, x);
    auto t1 = std::chrono::steady_clock::now();
    std::vector<std::vector<double>> yh(t.nodes.size());
    for (size_t f = 0; f < M.bt.far.size(); ++f) {
      if (far_mask && !far_mask[f]) continue;
      const int s = M.bt.far[f].first, u = M.bt.far[f].second;
      if (M.h2) {
        const auto z = coupling_apply(M.couplings[M.far_key[f]], I.class_h[M.far_key[f]], xh[u]);
        if (yh[s].empty())
          yh[s] = z;
        else
          for (size_t q = 0; q < z.size(); ++q) yh[s][q] += z[q];
      }
    }
    auto t2 = std::chrono::steady_clock::now();
    for (size_t b = 0; b < M.bt.nearb.size(); ++b) {
      if (near_mask && !near_mask[b]) continue;
      const Node& s = t.nodes[M.bt.nearb[b].first];
      const Node& u = t.nodes[M.bt.nearb[b].second];
      const Mat& D = I.near_d[b];
      for (i64 r = 0; r < s.size(); ++r) {
        double acc = 0.0;
        for (i64 j = 0; j < u.size(); ++j) acc += D(r, j) * x[u.idx[j]];
        y[s.idx[r]] += acc;
      }
    }
    auto t3 = std::chrono::steady_clock::now();
    if (M.h2) backward(M, yh, y);
    auto t4 = std::chrono::steady_clock::now();
    secs[0] = std::chrono::duration<double>((t1 - t0) + (t4 - t3)).count();
    secs[1] = std::chrono::duration<double>(t2 - t1).count();
    secs[2] = std::chrono::duration<double>(t3 - t2).count();
  });
}
// Induced dense matrix (phmatrix.cpp:273-317), n <= guard.
int orc_to_dense(void* i, double* out, std::int64_t guard_n) {
  return guard([&] {
    Inst& I = *static_cast<Inst*>(i);
    const Matrix& M = *I.m;
    const Tree& t = M.tree;
    const i64 n = t.n;
    if (n > guard_n) throw std::runtime_error("to_dense: matrix exceeds the size guard");
    std::fill(out, out + n * n, 0.0);
    for (size_t f = 0; f < M.bt.far.size(); ++f) {
      const Node& s = t.nodes[M.bt.far[f].first];
      const Node& u = t.nodes[M.bt.far[f].second];
      const Mat& H = I.class_h[M.far_key[f]];
      Mat blk;
      if (M.h2) {
        const Mat us = assemble_basis(basis_factors(t, M.bt.far[f].first, M.ps));
        const Mat ut = assemble_basis(basis_factors(t, M.bt.far[f].second, M.ps));
        const Mat C = matmul(matmul(M.class_L[M.far_key[f]], H), transpose(M.class_R[M.far_key[f]]));
        blk = matmul(matmul(us, C), transpose(ut));
      } else {
        blk = matmul(matmul(M.far_s[f], H), transpose(M.far_t[f]));
      }
      for (i64 c = 0; c < u.size(); ++c)
        for (i64 r = 0; r < s.size(); ++r) out[s.idx[r] + u.idx[c] * n] = blk(r, c);
    }
    for (size_t b = 0; b < M.bt.nearb.size(); ++b) {
      const Node& s = t.nodes[M.bt.nearb[b].first];
      const Node& u = t.nodes[M.bt.nearb[b].second];
      for (i64 c = 0; c < u.size(); ++c)
        for (i64 r = 0; r < s.size(); ++r) out[s.idx[r] + u.idx[c] * n] = I.near_d[b](r, c);
    }
  });
}
// Exact dense kernel matrix K(x_i, x_j; theta) (test oracle, n small).
void orc_dense_kernel(const double* pts, std::int64_t n, int d, int fam, int amp, const double* theta, double* out) {
  for (i64 j = 0; j < n; ++j)
    for (i64 i = 0; i < n; ++i) {
      double r2 = 0.0;
      for (int c = 0; c < d; ++c) {
        const double dl = pts[i * d + c] - pts[j * d + c];
        r2 += dl * dl;
      }
      out[i + j * n] = kernel_value(fam, amp != 0, std::sqrt(r2), theta);
    }
}
// Kernel entries of the coupling tensor at Chebyshev node triples
// (farfield.cpp:41-100; bitwise-translation-invariant construction).
int orc_coupling_entry(void* m, std::int64_t far_index, const std::int64_t* idx, double* out) {
  return guard([&] {
    Matrix& M = *static_cast<Matrix*>(m);
    const Tree& t = M.tree;
    const Node& s = t.nodes[M.bt.far.at(far_index).first];
    const Node& u = t.nodes[M.bt.far[far_index].second];
    const int d = t.d, dt = M.spec.dtheta();
    const double pi = 3.141592653589793238462643383279502884;
    double r2 = 0.0;
    for (int k = 0; k < d; ++k) {
      const double side = t.side(s.level, k);
      std::vector<double> off(M.ps);
      for (int q = 0; q < M.ps; ++q) {
        const double c = std::cos((2.0 * q + 1.0) * pi / (2.0 * M.ps));
        off[M.ps - 1 - q] = 0.5 * (c + 1.0) * side;
      }
      const double bd = static_cast<double>(s.coords[k] - u.coords[k]) * side;
      const double dl = bd + (off[idx[k]] - off[idx[d + dt + k]]);
      r2 += dl * dl;
    }
    double th[3];
    for (int k = 0; k < dt; ++k) th[k] = M.grids[k].x[idx[d + k]];
    *out = kernel_value(M.spec.fam, M.spec.amp, std::sqrt(r2), th);
  });
}

}  // extern "C"
