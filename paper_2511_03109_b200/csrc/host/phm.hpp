// Host-side C++ of the B200 parametric H / H^2 engine.
//
// This is the product's host layer: it builds the cluster tree, the block
// cluster tree, the translation classes and the offline far-field / near-field
// data exactly as the reference does (proj/src/{geometry,chebyshev,tt,
// farfield,nearfield,phmatrix}.cpp), then hands flat arrays to the device
// layer (device.cu). Nothing here runs on the online (instantiate / apply)
// path; that path is CUDA only.
#pragma once

#include <array>
#include <atomic>
#include <cmath>
#include <cstdint>
#include <functional>
#include <memory>
#include <random>
#include <stdexcept>
#include <string>
#include <vector>

namespace phm {

using Index = std::int64_t;
constexpr int kMaxDim = 3;

// ----------------------------------------------------------------- common
// Same generator contract as proj/include/phmat/common.hpp:22-33: raw
// mt19937_64 words, uniform = (g >> 11) * 2^-53.
class Rng {
 public:
  explicit Rng(std::uint64_t seed) : gen_(seed) {}
  double uniform() { return static_cast<double>(gen_() >> 11) * 0x1.0p-53; }
  double uniform(double a, double b) { return a + (b - a) * uniform(); }
  std::uint64_t integer(std::uint64_t n) { return n ? gen_() % n : 0; }
  std::uint64_t raw() { return gen_(); }
  // N(0,1) by the Box-Muller transform on two uniforms (defined here once so
  // the host, the oracle and bench draw the same x; std::normal_distribution
  // is not portable across standard libraries).
  double normal();

 private:
  std::mt19937_64 gen_;
};

// splitmix64 step (proj/include/phmat/common.hpp:36-41).
std::uint64_t mix_seed(std::uint64_t a, std::uint64_t b);

int max_threads();  // PHMAT_THREADS caps it (proj/src/common.cpp:10-17)
// Atomic work counter over [0, n); first worker exception rethrown
// (proj/src/common.cpp:19-48).
void parallel_for(Index n, const std::function<void(Index)>& fn, int threads = 0);

#define PHM_CHECK(cond, msg)                                          \
  do {                                                                \
    if (!(cond)) throw std::logic_error(std::string("phmat: ") + (msg)); \
  } while (0)

// ---------------------------------------------------------------- kernels
// Families of proj/src/kernels.cpp:49-78 plus the single-parameter
// Gaussian / Matern-3/2 / Matern-5/2 and an optional trailing amplitude
// parameter sigma^2.
enum Family : int { kExp = 0, kTps = 1, kSe = 2, kMc = 3, kMatern = 4, kGauss = 5, kMatern32 = 6, kMatern52 = 7 };

struct Interval {
  double lo = 0.0, hi = 0.0;
  bool contains(double x) const { return x >= lo && x <= hi; }
};

struct KernelSpec {
  int family = kSe;
  bool amplitude = false;  // trailing theta component multiplies the kernel
  std::vector<Interval> box;
  int d_theta() const { return static_cast<int>(box.size()); }
  int shape_params() const { return family == kMatern ? 2 : 1; }
  void validate() const;  // std::invalid_argument, cf. kernels.cpp:28-39
};

double kernel_value(const KernelSpec& spec, double r, const double* theta);

class EvalCounter {
 public:
  void add(std::uint64_t k = 1) { n_.fetch_add(k, std::memory_order_relaxed); }
  std::uint64_t value() const { return n_.load(std::memory_order_relaxed); }
  void reset() { n_.store(0); }

 private:
  std::atomic<std::uint64_t> n_{0};
};

struct StageCounters {
  EvalCounter offline, online, audit;
};

// --------------------------------------------------------------- geometry
struct Box {
  int d = 0;
  std::array<double, kMaxDim> lo{}, hi{};
  double diam() const;
};
double box_dist(const Box& a, const Box& b);
bool admissible(const Box& a, const Box& b, double eta);

struct TreeNode {
  Box box;
  std::array<std::int64_t, kMaxDim> coords{};
  int level = 0;
  int parent = -1;
  int first_child = -1;
  Index begin = 0;  // tree-order point range [begin, begin + count)
  Index count = 0;
  bool leaf() const { return first_child < 0; }
};

// Uniform 2^d-way tree to l_max with the reference's exact node numbering
// and point assignment (geometry.cpp:46-108). Points are held in tree order:
// perm[p] is the original index of the p-th point in tree order, and every
// node owns the contiguous range [begin, begin + count). Within a node the
// original indices ascend, as the reference's sorted index sets do.
class Tree {
 public:
  Tree(const double* points, Index n, int d, const Box& root, int l_max);
  int d = 0, l_max = 0;
  Index n = 0;
  std::vector<double> points;        // n x d row-major, original order
  std::vector<std::int32_t> perm;    // tree order -> original index
  std::vector<TreeNode> nodes;
  double level_side(int level, int k) const;
  double coord(Index original, int k) const { return points[original * d + k]; }
};

struct Block {
  int sigma = -1, tau = -1;
};

struct BlockLists {
  std::vector<Block> far, near;
  int c_sp = 0;
  Index constructed = 0;
  double eta = 0.0;
};

// DFS block recursion (geometry.cpp:124-157).
BlockLists build_blocks(const Tree& tree, double eta);

// -------------------------------------------------------------- chebyshev
struct Grid1D {
  double lo = -1, hi = 1;
  int p = 1;
  std::vector<double> nodes, weights;
};
Grid1D cheb_grid(double lo, double hi, int p);          // chebyshev.cpp:10-43
void lagrange_all(const Grid1D& g, double x, double* out);  // chebyshev.cpp:56-69

// --------------------------------------------------------------- dense LA
// Column-major dense matrix, only what the offline stage needs.
struct Mat {
  Index rows = 0, cols = 0;
  std::vector<double> a;
  Mat() = default;
  Mat(Index r, Index c) : rows(r), cols(c), a(static_cast<size_t>(r * c), 0.0) {}
  double& operator()(Index i, Index j) { return a[i + j * rows]; }
  double operator()(Index i, Index j) const { return a[i + j * rows]; }
  static Mat identity(Index n);
};
Mat operator*(const Mat& A, const Mat& B);
Mat transpose(const Mat& A);
double frob(const Mat& A);
// Thin Householder QR: A (m x n) = Q (m x t) R (t x n), t = min(m, n).
void qr_thin(const Mat& A, Mat& Q, Mat& R);
// Thin SVD by one-sided Jacobi: A = U diag(s) V^T, s descending.
void svd_thin(const Mat& A, Mat& U, std::vector<double>& s, Mat& V);
// Minimum-norm least-squares solve A X = B through a rank-revealing
// column-pivoted QR with relative threshold (complete orthogonal
// decomposition, cf. Eigen::CompleteOrthogonalDecomposition used at
// tt.cpp:410-412).
Mat cod_solve(const Mat& A, const Mat& B, double threshold);

// --------------------------------------------------------------------- TT
struct TTCore {  // (r0, m, r1), entry (a, j, c) at a + j r0 + c r0 m (tt.hpp:19-43)
  Index r0 = 1, m = 1, r1 = 1;
  std::vector<double> data;
  static TTCore zeros(Index r0, Index m, Index r1);
  Index size() const { return r0 * m * r1; }
  double at(Index a, Index j, Index c) const { return data[a + j * r0 + c * r0 * m]; }
  Mat left() const;   // r0 x (m r1)
  Mat right() const;  // (r0 m) x r1
  Mat slice(Index j) const;
  Mat contract(const std::vector<double>& v) const;  // tt.cpp:31-37
};

struct TTTensor {
  std::vector<TTCore> cores;
  int order() const { return static_cast<int>(cores.size()); }
  Index rank(int i) const { return i == 0 ? cores.front().r0 : cores[i - 1].r1; }
  Index max_rank() const;
  Index storage() const;
  double entry(const Index* idx) const;
};

// Entry function over a tensor shape; counted (offline) or audit evaluation.
struct EntryFn {
  std::vector<Index> dims;
  std::function<double(const Index*)> fn;
  EvalCounter* counter = nullptr;
  EvalCounter* audit = nullptr;
};

struct CrossOptions {
  double eps = 1e-5;
  Index r_max = 120;
  int min_sweeps = 2;
  int max_sweeps = 12;
  int error_samples = 1000;
  std::uint64_t seed = 0;
  bool round_after = true;
};

struct CrossResult {
  TTTensor tt;
  bool rank_capped = false;
  bool converged = true;
  double est_rel_error = 0.0;
  double max_aca_resid = 0.0;
  std::uint64_t evals = 0;
  int sweeps = 0;
};

// TT-cross with warm-started partially pivoted ACA over supercores and a
// final absolute-budget TT-rounding (tt.cpp:269-480, aca_impl.hpp:34-173).
CrossResult tt_cross(const EntryFn& f, const CrossOptions& opt);
TTTensor tt_round(const TTTensor& tt, double eps, double abs_budget);  // tt.cpp:159-224
TTTensor tt_svd(const std::vector<double>& full, const std::vector<Index>& dims, double abs_budget);

// ------------------------------------------------------------- parametric
struct ThetaGrids {
  std::vector<Grid1D> grids;
  int d_theta() const { return static_cast<int>(grids.size()); }
};
ThetaGrids make_theta_grids(const KernelSpec& spec, const std::vector<int>& p_theta);
// farfield.cpp:16-29; std::domain_error outside the box.
std::vector<std::vector<double>> parametric_vectors(const ThetaGrids& g, const double* theta, int n_theta);

struct Coupling {
  TTTensor tt;
  int d = 0, d_theta = 0;
  bool rank_capped = false;
  double est_rel_error = 0.0;
  std::uint64_t evals = 0;
  Index rank_left() const { return tt.rank(d); }
  Index rank_right() const { return tt.rank(d + d_theta); }
};

// ----------------------------------------------------------------- matrix
enum class Format : int { H = 0, H2 = 1 };
enum class NearMode : int { TT = 0, Direct = 1, Snapshot = 2 };

struct Config {
  KernelSpec spec;
  Format format = Format::H2;
  int l_max = 2;
  int p_s = 15;
  std::vector<int> p_theta{27};  // per parameter dimension
  double eps = 1e-5;
  double eta = 0.0;  // <= 0 selects sqrt(d)
  Index r_max_far = 120;
  Index r_max_near = 150;
  std::uint64_t seed = 0;
  NearMode near_mode = NearMode::TT;
  bool translation_cache = true;
  int threads = 0;
  int shard_rank = 0;   // leaf row-cluster sharding (multi-GPU); 0 / 1 = whole
  int shard_count = 1;
  bool symmetric_near = true;  // snapshot mode: store sigma <= tau near blocks only
  double resolved_eta(int d) const { return eta > 0.0 ? eta : std::sqrt(double(d)); }
};

struct BuildStats {
  std::uint64_t ff_evals = 0, nf_evals = 0;
  double tree_s = 0, ff_s = 0, nf_s = 0, upload_s = 0;
  bool any_rank_capped = false;
  int svd_fallbacks = 0;  // non-converged crosses redone by full TT-SVD
};

enum class Baseline : int { None = 0, HAca = 1, H2Hca = 2 };
struct BaselineData {
  Baseline method = Baseline::None;
  std::vector<double> theta;
  std::vector<int> rank;           // per class (H-ACA: per far block): ACA rank t
  std::vector<std::int64_t> h_off; // per class: offset of its t x t identity in fixed_h
  std::vector<double> fixed_h;     // H_b = I_t per class, column-major
  std::vector<double> fixed_c;     // H^2-HCA: C_k = V_k Y_k^T, P x P per class
  double far_s = 0.0, mean_far_rank = 0.0, coupling_ratio = 0.0;
  std::uint64_t far_evals = 0, near_evals = 0;
  bool any_capped = false;
};

// Everything the offline stage produces on the host, in the reference's
// representation. The device layer flattens it (device.cu).
struct HostMatrix {
  Config cfg;
  std::unique_ptr<Tree> tree;
  BlockLists blocks;
  ThetaGrids grids;
  std::vector<int> far_key;        // class per far block
  std::vector<int> class_rep;      // representative far block per class
  std::vector<std::array<std::int64_t, 4>> class_keys;  // level, offset
  std::vector<Coupling> couplings; // per class
  // H form: S_b (n_sigma x r_d), T_b (n_tau x r_{d+dt}) per far block.
  std::vector<Mat> far_s, far_t;
  // H^2 form: explicit L_k (P x r_d), R_k (P x r_{d+dt}) per class.
  std::vector<Mat> class_l, class_r;
  // TT near mode: per near block TT (G1 is (1, N_b, R_b)).
  std::vector<TTTensor> near_tt;
  // Sharding: leaf range owned, and which blocks are local.
  Index row_begin = 0, row_end = 0;  // tree-order rows
  std::vector<char> near_local, far_local, node_local;
  BuildStats stats;
  StageCounters counters;
  // Non-parametric baselines (baselines.hpp): the far field is fixed at one
  // theta, so instantiate copies it instead of contracting theta-cores.
  BaselineData baseline;
  int d() const { return tree->d; }
  Index n() const { return tree->n; }
  Index P() const;  // p_s^d
};

// Partially pivoted ACA (aca_impl.hpp:34-173) as the baselines use it:
// A ~ V Y^T with V m x t, Y n x t (baselines.cpp:30-50).
struct LowRank {
  Mat v, y;
  bool capped = false;
  Index rank() const { return v.cols; }
};
LowRank aca_partial(const std::function<double(Index, Index)>& entry, Index m, Index n, double eps, Index r_max,
                    std::uint64_t seed);
LowRank aca_partial_rng(const std::function<double(Index, Index)>& entry, Index m, Index n, double eps, Index r_max,
                        Rng& rng);

// Offline build on the host (everything except GPU snapshot generation).
std::unique_ptr<HostMatrix> build_host(const double* points, Index n, int d, const Config& cfg);
// Explicit L (P x r_d) and R (P x r_{d+dt}) of a coupling (farfield.cpp:157-184).
void assemble_lr_public(const Coupling& cp, Mat& L, Mat& R);

// Baselines at a fixed theta (baselines.cpp:52-100 H-ACA, :133-219 H^2-HCA):
// tree and blocks as the parametric build, ACA factors on the host, dense
// near blocks evaluated on the device at instantiate (Direct near mode).
std::unique_ptr<HostMatrix> build_baseline_host(const double* points, Index n, int d, const Config& cfg,
                                                Baseline method, const double* theta, int n_theta, double eps,
                                                Index r_max);

// HMAT v1 artifacts, byte-compatible with proj/src/serialize.cpp.
bool artifact_is_h2(const std::string& path);
void write_artifact(const HostMatrix& M, const std::string& path, const std::function<TTTensor(Index)>& near_tt);
std::unique_ptr<HostMatrix> read_artifact(const std::string& path, int threads);

// Seeded generators (harness.cpp:174-181 and the new mixture generator).
void generate_points(Index n, int d, std::uint64_t seed, double* out);
void generate_mixture_points(Index n, int d, int clusters, double sigma, std::uint64_t seed, double* out);
void generate_normal(Index n, std::uint64_t seed, double* out);

}  // namespace phm
