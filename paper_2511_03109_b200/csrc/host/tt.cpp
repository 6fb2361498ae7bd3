// Offline tensor-train machinery on the host: small dense linear algebra,
// partially pivoted ACA, TT-cross and TT-rounding. Restates the algorithms of
// proj/src/tt.cpp:137-480 and proj/src/aca_impl.hpp:34-173 without Eigen.
// None of this is on the online path; it produces the far-field coupling
// cores (and TT near blocks) that the device instantiates.
#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <limits>
#include <map>
#include <numeric>
#include <unordered_map>

#include "phm.hpp"

namespace phm {

// ------------------------------------------------------------- dense LA
Mat Mat::identity(Index n) {
  Mat I(n, n);
  for (Index i = 0; i < n; ++i) I(i, i) = 1.0;
  return I;
}

Mat operator*(const Mat& A, const Mat& B) {
  PHM_CHECK(A.cols == B.rows, "matmul: shape mismatch");
  Mat C(A.rows, B.cols);
  for (Index j = 0; j < B.cols; ++j)
    for (Index k = 0; k < A.cols; ++k) {
      const double b = B(k, j);
      if (b == 0.0) continue;
      const double* a = &A.a[k * A.rows];
      double* c = &C.a[j * C.rows];
      for (Index i = 0; i < A.rows; ++i) c[i] += a[i] * b;
    }
  return C;
}

Mat transpose(const Mat& A) {
  Mat T(A.cols, A.rows);
  for (Index j = 0; j < A.cols; ++j)
    for (Index i = 0; i < A.rows; ++i) T(j, i) = A(i, j);
  return T;
}

double frob(const Mat& A) {
  double s = 0.0;
  for (double v : A.a) s += v * v;
  return std::sqrt(s);
}

namespace {

// Householder reflector for x (length len): returns beta, overwrites x with
// v (v[0] = 1) and gives the new leading entry.
double householder(double* x, Index len, double& alpha_out) {
  double sigma = 0.0;
  for (Index i = 1; i < len; ++i) sigma += x[i] * x[i];
  const double x0 = x[0];
  if (sigma == 0.0) {
    alpha_out = x0;
    x[0] = 1.0;
    return 0.0;
  }
  const double mu = std::sqrt(x0 * x0 + sigma);
  const double alpha = x0 <= 0.0 ? mu : -mu;  // new diagonal entry
  const double v0 = x0 - alpha;
  const double beta = -v0 / alpha;  // = 2 v0^2 / (sigma + v0^2)
  for (Index i = 1; i < len; ++i) x[i] /= v0;
  x[0] = 1.0;
  alpha_out = alpha;
  return beta;
}

// In-place Householder QR with optional column pivoting. On exit the upper
// triangle of W holds R, the strict lower part the reflectors.
void householder_qr(Mat& W, std::vector<double>& betas, std::vector<Index>* piv) {
  const Index m = W.rows, n = W.cols, t = std::min(m, n);
  betas.assign(t, 0.0);
  std::vector<double> norms;
  if (piv) {
    piv->resize(n);
    std::iota(piv->begin(), piv->end(), 0);
    norms.resize(n);
    for (Index j = 0; j < n; ++j) {
      double s = 0.0;
      for (Index i = 0; i < m; ++i) s += W(i, j) * W(i, j);
      norms[j] = s;
    }
  }
  for (Index j = 0; j < t; ++j) {
    if (piv) {
      Index best = j;
      for (Index c = j + 1; c < n; ++c)
        if (norms[c] > norms[best]) best = c;
      if (best != j) {
        for (Index i = 0; i < m; ++i) std::swap(W(i, j), W(i, best));
        std::swap(norms[j], norms[best]);
        std::swap((*piv)[j], (*piv)[best]);
      }
    }
    double alpha;
    double* col = &W.a[j + j * m];
    const double beta = householder(col, m - j, alpha);
    betas[j] = beta;
    // apply (I - beta v v^T) to the trailing columns
    for (Index c = j + 1; c < n; ++c) {
      double* wc = &W.a[j + c * m];
      double s = 0.0;
      for (Index i = 0; i < m - j; ++i) s += col[i] * wc[i];
      s *= beta;
      for (Index i = 0; i < m - j; ++i) wc[i] -= s * col[i];
    }
    // store alpha on the diagonal; reflector (without its unit head) below
    col[0] = alpha;
    if (piv) {
      for (Index c = j + 1; c < n; ++c) {
        // exact downdate keeps pivoting robust for the small matrices here
        double s = 0.0;
        for (Index i = j + 1; i < m; ++i) s += W(i, c) * W(i, c);
        norms[c] = s;
      }
    }
  }
}

// Q (m x t) from the stored reflectors.
Mat form_q(const Mat& W, const std::vector<double>& betas) {
  const Index m = W.rows, t = static_cast<Index>(betas.size());
  Mat Q(m, t);
  for (Index i = 0; i < t; ++i) Q(i, i) = 1.0;
  std::vector<double> v(static_cast<size_t>(m));
  for (Index j = t - 1; j >= 0; --j) {
    if (betas[j] == 0.0) continue;
    v[j] = 1.0;
    for (Index i = j + 1; i < m; ++i) v[i] = W(i, j);
    for (Index c = 0; c < t; ++c) {
      double s = 0.0;
      for (Index i = j; i < m; ++i) s += v[i] * Q(i, c);
      s *= betas[j];
      for (Index i = j; i < m; ++i) Q(i, c) -= s * v[i];
    }
  }
  return Q;
}

// Q^T B using the stored reflectors (B has W.rows rows).
void apply_qt(const Mat& W, const std::vector<double>& betas, Mat& B) {
  const Index m = W.rows, t = static_cast<Index>(betas.size());
  std::vector<double> v(static_cast<size_t>(m));
  for (Index j = 0; j < t; ++j) {
    if (betas[j] == 0.0) continue;
    v[j] = 1.0;
    for (Index i = j + 1; i < m; ++i) v[i] = W(i, j);
    for (Index c = 0; c < B.cols; ++c) {
      double s = 0.0;
      for (Index i = j; i < m; ++i) s += v[i] * B(i, c);
      s *= betas[j];
      for (Index i = j; i < m; ++i) B(i, c) -= s * v[i];
    }
  }
}

// One-sided Jacobi SVD of a square-ish matrix with rows >= cols.
void jacobi_svd(const Mat& A, Mat& U, std::vector<double>& s, Mat& V) {
  const Index m = A.rows, n = A.cols;
  U = A;
  V = Mat::identity(n);
  const double tol = 1e-15;
  for (int sweep = 0; sweep < 60; ++sweep) {
    bool rotated = false;
    for (Index p = 0; p + 1 < n; ++p)
      for (Index q = p + 1; q < n; ++q) {
        double alpha = 0.0, beta = 0.0, gamma = 0.0;
        const double* up = &U.a[p * m];
        const double* uq = &U.a[q * m];
        for (Index i = 0; i < m; ++i) {
          alpha += up[i] * up[i];
          beta += uq[i] * uq[i];
          gamma += up[i] * uq[i];
        }
        if (gamma == 0.0 || std::abs(gamma) <= tol * std::sqrt(alpha * beta)) continue;
        rotated = true;
        const double zeta = (beta - alpha) / (2.0 * gamma);
        const double t = (zeta >= 0 ? 1.0 : -1.0) / (std::abs(zeta) + std::sqrt(1.0 + zeta * zeta));
        const double c = 1.0 / std::sqrt(1.0 + t * t);
        const double sn = c * t;
        double* Up = &U.a[p * m];
        double* Uq = &U.a[q * m];
        for (Index i = 0; i < m; ++i) {
          const double a = Up[i], b = Uq[i];
          Up[i] = c * a - sn * b;
          Uq[i] = sn * a + c * b;
        }
        double* Vp = &V.a[p * n];
        double* Vq = &V.a[q * n];
        for (Index i = 0; i < n; ++i) {
          const double a = Vp[i], b = Vq[i];
          Vp[i] = c * a - sn * b;
          Vq[i] = sn * a + c * b;
        }
      }
    if (!rotated) break;
  }
  s.assign(n, 0.0);
  for (Index j = 0; j < n; ++j) {
    double nrm = 0.0;
    for (Index i = 0; i < m; ++i) nrm += U(i, j) * U(i, j);
    nrm = std::sqrt(nrm);
    s[j] = nrm;
    if (nrm > 0.0)
      for (Index i = 0; i < m; ++i) U(i, j) /= nrm;
  }
  // sort descending
  std::vector<Index> ord(n);
  std::iota(ord.begin(), ord.end(), 0);
  std::stable_sort(ord.begin(), ord.end(), [&](Index a, Index b) { return s[a] > s[b]; });
  Mat U2(m, n), V2(n, n);
  std::vector<double> s2(n);
  for (Index j = 0; j < n; ++j) {
    s2[j] = s[ord[j]];
    for (Index i = 0; i < m; ++i) U2(i, j) = U(i, ord[j]);
    for (Index i = 0; i < n; ++i) V2(i, j) = V(i, ord[j]);
  }
  U = std::move(U2);
  V = std::move(V2);
  s = std::move(s2);
}

}  // namespace

void qr_thin(const Mat& A, Mat& Q, Mat& R) {
  Mat W = A;
  std::vector<double> betas;
  householder_qr(W, betas, nullptr);
  const Index t = std::min(A.rows, A.cols);
  R = Mat(t, A.cols);
  for (Index j = 0; j < A.cols; ++j)
    for (Index i = 0; i <= std::min(j, t - 1); ++i) R(i, j) = W(i, j);
  Q = form_q(W, betas);
}

void svd_thin(const Mat& A, Mat& U, std::vector<double>& s, Mat& V) {
  if (A.rows < A.cols) {
    svd_thin(transpose(A), V, s, U);
    return;
  }
  // QR first, then Jacobi on the small triangular factor.
  Mat Q, R;
  qr_thin(A, Q, R);
  Mat Ur;
  jacobi_svd(R, Ur, s, V);
  U = Q * Ur;
}

Mat cod_solve(const Mat& A, const Mat& B, double threshold) {
  PHM_CHECK(A.rows == B.rows, "cod_solve: shape mismatch");
  const Index m = A.rows, n = A.cols;
  Mat W = A;
  std::vector<double> betas;
  std::vector<Index> piv;
  householder_qr(W, betas, &piv);
  const Index t = std::min(m, n);
  double maxpiv = 0.0;
  for (Index i = 0; i < t; ++i) maxpiv = std::max(maxpiv, std::abs(W(i, i)));
  Index rank = 0;
  for (Index i = 0; i < t; ++i)
    if (std::abs(W(i, i)) > threshold * maxpiv) ++rank;
  Mat C = B;
  apply_qt(W, betas, C);
  Mat X(n, B.cols);
  if (rank == 0) return X;
  // min-norm solve of [R11 R12] y = c_top via a thin QR of the transpose
  Mat Wt(n, rank);
  for (Index i = 0; i < rank; ++i)
    for (Index j = i; j < n; ++j) Wt(j, i) = W(i, j);
  Mat Q2, R2;
  qr_thin(Wt, Q2, R2);  // Wt = Q2 R2, R2 rank x rank upper
  for (Index c = 0; c < B.cols; ++c) {
    std::vector<double> u(static_cast<size_t>(rank));
    for (Index i = 0; i < rank; ++i) {  // R2^T u = c_top (forward)
      double s = C(i, c);
      for (Index k = 0; k < i; ++k) s -= R2(k, i) * u[k];
      u[i] = s / R2(i, i);
    }
    for (Index j = 0; j < n; ++j) {
      double y = 0.0;
      for (Index i = 0; i < rank; ++i) y += Q2(j, i) * u[i];
      X(piv[j], c) = y;
    }
  }
  return X;
}

// --------------------------------------------------------------- TT core
TTCore TTCore::zeros(Index r0, Index m, Index r1) {
  TTCore c;
  c.r0 = r0;
  c.m = m;
  c.r1 = r1;
  c.data.assign(static_cast<size_t>(r0 * m * r1), 0.0);
  return c;
}
Mat TTCore::left() const {
  Mat o(r0, m * r1);
  o.a = data;
  return o;
}
Mat TTCore::right() const {
  Mat o(r0 * m, r1);
  o.a = data;
  return o;
}
Mat TTCore::slice(Index j) const {
  Mat o(r0, r1);
  for (Index c = 0; c < r1; ++c)
    for (Index a = 0; a < r0; ++a) o(a, c) = at(a, j, c);
  return o;
}
Mat TTCore::contract(const std::vector<double>& v) const {
  PHM_CHECK(static_cast<Index>(v.size()) == m, "contract_mode2: length mismatch");
  Mat o(r0, r1);
  for (Index j = 0; j < m; ++j) {
    if (v[j] == 0.0) continue;
    for (Index c = 0; c < r1; ++c)
      for (Index a = 0; a < r0; ++a) o(a, c) += v[j] * at(a, j, c);
  }
  return o;
}
Index TTTensor::max_rank() const {
  Index r = 1;
  for (const auto& c : cores) r = std::max({r, c.r0, c.r1});
  return r;
}
Index TTTensor::storage() const {
  Index s = 0;
  for (const auto& c : cores) s += c.size();
  return s;
}
double TTTensor::entry(const Index* idx) const {
  std::vector<double> w(static_cast<size_t>(cores[0].r1));
  for (Index c = 0; c < cores[0].r1; ++c) w[c] = cores[0].at(0, idx[0], c);
  for (int k = 1; k < order(); ++k) {
    const TTCore& g = cores[k];
    std::vector<double> nw(static_cast<size_t>(g.r1), 0.0);
    for (Index c = 0; c < g.r1; ++c) {
      double s = 0.0;
      for (Index a = 0; a < g.r0; ++a) s += g.at(a, idx[k], c) * w[a];
      nw[c] = s;
    }
    w.swap(nw);
  }
  return w[0];
}

// ------------------------------------------------------------- rounding
TTTensor tt_round(const TTTensor& in, double eps, double abs_budget) {
  TTTensor tt = in;
  const int q = tt.order();
  if (q == 1) return tt;
  // right-to-left orthogonalization (tt.cpp:167-185)
  for (int k = q - 1; k >= 1; --k) {
    TTCore& c = tt.cores[k];
    const Mat at = transpose(c.left());  // (m r1) x r0
    Mat Q, R;
    qr_thin(at, Q, R);  // Q: (m r1) x t, R: t x r0
    const Index t = Q.cols;
    TTCore fresh = TTCore::zeros(t, c.m, c.r1);
    const Mat qt = transpose(Q);  // t x (m r1)
    fresh.data = qt.a;
    TTCore& prev = tt.cores[k - 1];
    const Mat carried = prev.right() * transpose(R);  // (r0 m) x t
    TTCore pf = TTCore::zeros(prev.r0, prev.m, t);
    pf.data = carried.a;
    tt.cores[k] = std::move(fresh);
    tt.cores[k - 1] = std::move(pf);
  }
  double norm = 0.0;
  for (double v : tt.cores[0].data) norm += v * v;
  norm = std::sqrt(norm);
  const double total = abs_budget >= 0.0 ? abs_budget : (norm == 0.0 ? 0.0 : eps * norm);
  const double delta = total / std::sqrt(static_cast<double>(q - 1));
  // left-to-right truncated SVD (tt.cpp:191-215)
  for (int k = 0; k + 1 < q; ++k) {
    TTCore& c = tt.cores[k];
    Mat U, V;
    std::vector<double> s;
    svd_thin(c.right(), U, s, V);
    Index r = static_cast<Index>(s.size());
    double tail = 0.0;
    while (r > 1 && tail + s[r - 1] * s[r - 1] <= delta * delta) {
      tail += s[r - 1] * s[r - 1];
      --r;
    }
    TTCore fresh = TTCore::zeros(c.r0, c.m, r);
    for (Index j = 0; j < r; ++j)
      for (Index i = 0; i < U.rows; ++i) fresh.data[i + j * U.rows] = U(i, j);
    Mat carry(r, V.rows);
    for (Index i = 0; i < r; ++i)
      for (Index j = 0; j < V.rows; ++j) carry(i, j) = s[i] * V(j, i);
    TTCore& nx = tt.cores[k + 1];
    const Mat nl = carry * nx.left();
    TTCore nf = TTCore::zeros(r, nx.m, nx.r1);
    nf.data = nl.a;
    tt.cores[k] = std::move(fresh);
    tt.cores[k + 1] = std::move(nf);
  }
  return tt;
}

// TT-SVD of a fully evaluated tensor (first index fastest) with an absolute
// Frobenius budget split evenly over the q-1 bonds. Used only as the
// robustness fallback when TT-cross reports non-convergence on a tensor
// small enough to evaluate in full.
TTTensor tt_svd(const std::vector<double>& full, const std::vector<Index>& dims, double abs_budget) {
  const int q = static_cast<int>(dims.size());
  TTTensor tt;
  const double delta = q > 1 ? abs_budget / std::sqrt(static_cast<double>(q - 1)) : 0.0;
  Index rest = 1;
  for (Index m : dims) rest *= m;
  Mat C(dims[0], rest / dims[0]);
  C.a = full;
  Index r_prev = 1;
  for (int k = 0; k + 1 < q; ++k) {
    // C is (r_prev * m_k) x rest_k
    Mat U, V;
    std::vector<double> s;
    svd_thin(C, U, s, V);
    Index r = static_cast<Index>(s.size());
    double tail = 0.0;
    while (r > 1 && tail + s[r - 1] * s[r - 1] <= delta * delta) {
      tail += s[r - 1] * s[r - 1];
      --r;
    }
    TTCore core = TTCore::zeros(r_prev, dims[k], r);
    for (Index j = 0; j < r; ++j)
      for (Index i = 0; i < U.rows; ++i) core.data[i + j * U.rows] = U(i, j);
    tt.cores.push_back(std::move(core));
    // next C = diag(s) V^T reshaped to (r * m_{k+1}) x rest_{k+1}
    const Index cols = V.rows;
    Mat SV(r, cols);
    for (Index j = 0; j < cols; ++j)
      for (Index i = 0; i < r; ++i) SV(i, j) = s[i] * V(j, i);
    const Index m1 = dims[k + 1];
    Mat nc(r * m1, cols / m1);
    nc.a = std::move(SV.a);
    C = std::move(nc);
    r_prev = r;
  }
  TTCore last = TTCore::zeros(r_prev, dims[q - 1], 1);
  last.data = C.a;
  tt.cores.push_back(std::move(last));
  return tt;
}

// ------------------------------------------------------------------ ACA
namespace {

struct AcaSeed {
  std::vector<Index> rows, cols;
};

struct AcaOut {
  std::vector<Index> rows, cols;
  std::vector<std::vector<double>> us, vs;
  double final_ratio = 0.0;
  bool capped = false;
  Index rank() const { return static_cast<Index>(us.size()); }
};

double dot(const std::vector<double>& a, const std::vector<double>& b) {
  double s = 0.0;
  for (size_t i = 0; i < a.size(); ++i) s += a[i] * b[i];
  return s;
}
double sqnorm(const std::vector<double>& a) { return dot(a, a); }

// Partially pivoted ACA with warm-start replay, two-hit stopping and random
// residual probes (aca_impl.hpp:34-173).
template <typename Entry>
AcaOut aca(const Entry& entry, Index m, Index n, double eps, Index r_max, Rng& rng, const AcaSeed* seed) {
  AcaOut out;
  std::vector<char> row_used(m, 0), col_used(n, 0);
  std::vector<double> ratios;
  double frob2 = 0.0;
  size_t replay = 0;
  Index i_star = seed && !seed->rows.empty() ? seed->rows[0] : static_cast<Index>(rng.integer(m));
  const Index t_limit = std::min({m, n, r_max});
  int dead_rows = 0, hits = 0, restarts = 0;

  while (out.rank() < t_limit) {
    const bool replaying = seed && replay < seed->rows.size();
    if (replaying) i_star = seed->rows[replay];
    std::vector<double> rho(n);
    for (Index j = 0; j < n; ++j) rho[j] = entry(i_star, j);
    for (size_t l = 0; l < out.us.size(); ++l) {
      const double ul = out.us[l][i_star];
      const auto& vl = out.vs[l];
      for (Index j = 0; j < n; ++j) rho[j] -= ul * vl[j];
    }
    row_used[i_star] = 1;

    Index j_star = -1;
    double best = -1.0;
    if (replaying) {
      j_star = seed->cols[replay];
      ++replay;
      best = std::abs(rho[j_star]);
      if (col_used[j_star] || best <= 1e-15 * std::sqrt(std::max(frob2, 1.0))) {
        if (replay >= seed->rows.size() && out.rank() == 0) i_star = static_cast<Index>(rng.integer(m));
        continue;
      }
    } else {
      for (Index j = 0; j < n; ++j)
        if (!col_used[j] && std::abs(rho[j]) > best) {
          best = std::abs(rho[j]);
          j_star = j;
        }
      if (j_star < 0) break;
      if (best == 0.0) {
        if (++dead_rows > 3) break;
        Index next = -1;
        for (Index i = 0; i < m; ++i)
          if (!row_used[i]) {
            next = i;
            break;
          }
        if (next < 0) break;
        i_star = next;
        continue;
      }
      dead_rows = 0;
    }

    std::vector<double> gamma(m);
    for (Index i = 0; i < m; ++i) gamma[i] = entry(i, j_star);
    for (size_t l = 0; l < out.us.size(); ++l) {
      const double vl = out.vs[l][j_star];
      const auto& ul = out.us[l];
      for (Index i = 0; i < m; ++i) gamma[i] -= vl * ul[i];
    }
    col_used[j_star] = 1;

    std::vector<double> u = std::move(gamma);
    std::vector<double> v(n);
    const double piv = rho[j_star];
    for (Index j = 0; j < n; ++j) v[j] = rho[j] / piv;
    double cross = 0.0;
    for (size_t l = 0; l < out.us.size(); ++l) cross += dot(out.us[l], u) * dot(out.vs[l], v);
    const double un2 = sqnorm(u), vn2 = sqnorm(v);
    frob2 += un2 * vn2 + 2.0 * cross;
    frob2 = std::max(frob2, 0.0);
    out.rows.push_back(i_star);
    out.cols.push_back(j_star);
    out.us.push_back(std::move(u));
    out.vs.push_back(std::move(v));

    const double term = std::sqrt(un2) * std::sqrt(vn2);
    out.final_ratio = frob2 > 0.0 ? term / std::sqrt(frob2) : 0.0;
    ratios.push_back(out.final_ratio);
    hits = !replaying && out.final_ratio <= eps ? hits + 1 : 0;
    if (hits >= 2) {
      const double fr = std::sqrt(frob2);
      double worst = 0.0;
      Index worst_row = -1;
      const int probes = static_cast<int>(std::min<Index>(64, m));
      for (int s = 0; s < probes; ++s) {
        const Index i = static_cast<Index>(rng.integer(m));
        const Index j = static_cast<Index>(rng.integer(n));
        double res = entry(i, j);
        for (size_t l = 0; l < out.us.size(); ++l) res -= out.us[l][i] * out.vs[l][j];
        if (std::abs(res) > worst) {
          worst = std::abs(res);
          worst_row = i;
        }
      }
      if (worst > eps * fr && restarts < 4) {
        ++restarts;
        hits = 0;
        i_star = worst_row;
        row_used[i_star] = 0;
        continue;
      }
      while (out.rank() > 1 && ratios.back() <= 1e-3 * eps) {
        out.rows.pop_back();
        out.cols.pop_back();
        out.us.pop_back();
        out.vs.pop_back();
        ratios.pop_back();
      }
      return out;
    }
    if (out.rank() >= t_limit) {
      if (out.rank() >= std::min(m, n))
        out.final_ratio = 0.0;
      else if (hits == 0)
        out.capped = true;
      return out;
    }
    Index next = -1;
    best = -1.0;
    const auto& ub = out.us.back();
    for (Index i = 0; i < m; ++i)
      if (!row_used[i] && std::abs(ub[i]) > best) {
        best = std::abs(ub[i]);
        next = i;
      }
    if (next < 0) break;
    i_star = next;
  }
  return out;
}

// Memoised, counted entry access for one tt_cross call. Dense table when the
// tensor is small enough (the coupling tensors are 4^6 * 8 entries), hash
// map otherwise.
class Memo {
 public:
  explicit Memo(const EntryFn& f) : f_(f) {
    strides_.resize(f.dims.size());
    Index s = 1;
    bool dense_ok = true;
    for (size_t k = 0; k < strides_.size(); ++k) {
      strides_[k] = s;
      if (s > (Index(1) << 40) / std::max<Index>(1, f.dims[k])) dense_ok = false;
      s *= f.dims[k];
    }
    if (dense_ok && s <= (Index(1) << 22)) {
      dense_.assign(static_cast<size_t>(s), std::numeric_limits<double>::quiet_NaN());
      have_.assign(static_cast<size_t>(s), 0);
    }
  }
  double operator()(const Index* idx) {
    Index key = 0;
    for (size_t k = 0; k < strides_.size(); ++k) key += idx[k] * strides_[k];
    if (!dense_.empty()) {
      if (have_[key]) return dense_[key];
      const double v = eval(idx);
      dense_[key] = v;
      have_[key] = 1;
      return v;
    }
    auto it = map_.find(key);
    if (it != map_.end()) return it->second;
    const double v = eval(idx);
    map_.emplace(key, v);
    return v;
  }
  std::uint64_t fresh() const { return fresh_; }

 private:
  double eval(const Index* idx) {
    ++fresh_;
    if (f_.counter) f_.counter->add();
    return f_.fn(idx);
  }
  const EntryFn& f_;
  std::vector<Index> strides_;
  std::vector<double> dense_;
  std::vector<char> have_;
  std::unordered_map<Index, double> map_;
  std::uint64_t fresh_ = 0;
};

using IndexList = std::vector<std::vector<Index>>;

}  // namespace

CrossResult tt_cross(const EntryFn& f, const CrossOptions& opt) {
  PHM_CHECK(opt.eps > 0.0, "tt_cross: eps must be positive");
  PHM_CHECK(opt.r_max >= 1, "tt_cross: r_max must be >= 1");
  const int q = static_cast<int>(f.dims.size());
  const std::vector<Index>& dims = f.dims;
  PHM_CHECK(q >= 1, "tt_cross: empty shape");
  Memo memo(f);
  Rng rng(opt.seed);
  CrossResult res;

  if (q == 1) {
    TTCore core = TTCore::zeros(1, dims[0], 1);
    for (Index j = 0; j < dims[0]; ++j) core.data[j] = memo(&j);
    res.tt.cores.push_back(std::move(core));
    res.evals = memo.fresh();
    return res;
  }

  std::vector<Index> z(q);
  for (int k = 0; k < q; ++k) z[k] = static_cast<Index>(rng.integer(dims[k]));
  std::vector<IndexList> left(q), right(q + 1);
  left[0] = {{}};
  right[q] = {{}};
  for (int k = 1; k < q; ++k) {
    left[k] = {std::vector<Index>(z.begin(), z.begin() + k)};
    right[k] = {std::vector<Index>(z.begin() + k, z.end())};
  }
  std::vector<double> bond_ratio(q - 1, 1.0);
  std::vector<Index> scratch(q);
  double eps_aca = 0.5 * opt.eps;

  auto run_supercore = [&](int k) {
    const IndexList& lk = left[k];
    const IndexList& rk2 = right[k + 2];
    const Index nl = static_cast<Index>(lk.size());
    const Index nr = static_cast<Index>(rk2.size());
    const Index m = nl * dims[k];
    const Index n = dims[k + 1] * nr;
    AcaSeed seed;
    {
      std::map<std::vector<Index>, Index> lpos, rpos;
      for (Index a = 0; a < nl; ++a) lpos.emplace(lk[a], a);
      for (Index b = 0; b < nr; ++b) rpos.emplace(rk2[b], b);
      const IndexList& l1 = left[k + 1];
      const IndexList& r1 = right[k + 1];
      for (size_t t = 0; t < l1.size() && t < r1.size(); ++t) {
        std::vector<Index> prefix(l1[t].begin(), l1[t].end() - 1);
        std::vector<Index> suffix(r1[t].begin() + 1, r1[t].end());
        const auto lp = lpos.find(prefix);
        const auto rp = rpos.find(suffix);
        if (lp == lpos.end() || rp == rpos.end()) continue;
        seed.rows.push_back(lp->second + l1[t].back() * nl);
        seed.cols.push_back(r1[t].front() + rp->second * dims[k + 1]);
      }
    }
    auto entry = [&](Index row, Index col) {
      const Index alpha = row % nl, ik = row / nl;
      const Index ik1 = col % dims[k + 1], beta = col / dims[k + 1];
      int pos = 0;
      for (Index v : lk[alpha]) scratch[pos++] = v;
      scratch[pos++] = ik;
      scratch[pos++] = ik1;
      for (Index v : rk2[beta]) scratch[pos++] = v;
      return memo(scratch.data());
    };
    AcaOut a = aca(entry, m, n, eps_aca, opt.r_max, rng, &seed);
    if (a.rows.empty()) return;
    IndexList nlft(a.rows.size()), nrgt(a.cols.size());
    for (size_t t = 0; t < a.rows.size(); ++t) {
      const Index alpha = a.rows[t] % nl, ik = a.rows[t] / nl;
      nlft[t] = lk[alpha];
      nlft[t].push_back(ik);
      const Index ik1 = a.cols[t] % dims[k + 1], beta = a.cols[t] / dims[k + 1];
      nrgt[t] = {ik1};
      nrgt[t].insert(nrgt[t].end(), rk2[beta].begin(), rk2[beta].end());
    }
    left[k + 1] = std::move(nlft);
    right[k + 1] = std::move(nrgt);
    bond_ratio[k] = a.final_ratio;
    res.rank_capped = res.rank_capped || a.capped;
  };

  auto assemble = [&]() {
    TTTensor tt;
    for (int k = 0; k < q; ++k) {
      const IndexList& lk = left[k];
      const IndexList& rk1 = right[k + 1];
      const Index rl = static_cast<Index>(lk.size()), rr = static_cast<Index>(rk1.size());
      Mat a(rl * dims[k], rr);
      for (Index beta = 0; beta < rr; ++beta)
        for (Index j = 0; j < dims[k]; ++j)
          for (Index alpha = 0; alpha < rl; ++alpha) {
            int pos = 0;
            for (Index v : lk[alpha]) scratch[pos++] = v;
            scratch[pos++] = j;
            for (Index v : rk1[beta]) scratch[pos++] = v;
            a(alpha + j * rl, beta) = memo(scratch.data());
          }
      if (k + 1 < q) {
        const IndexList& l1 = left[k + 1];
        const Index r = static_cast<Index>(l1.size());
        Mat cross(r, r);
        for (Index alpha = 0; alpha < r; ++alpha)
          for (Index beta = 0; beta < r; ++beta) {
            int pos = 0;
            for (Index v : l1[alpha]) scratch[pos++] = v;
            for (Index v : rk1[beta]) scratch[pos++] = v;
            cross(alpha, beta) = memo(scratch.data());
          }
        // a <- a cross^{-1} as the minimum-norm solve cross^T X = a^T
        a = transpose(cod_solve(transpose(cross), transpose(a), 1e-13));
      }
      TTCore core = TTCore::zeros(rl, dims[k], a.cols);
      core.data = a.a;
      tt.cores.push_back(std::move(core));
    }
    return tt;
  };

  double max_abs_seen = 0.0;
  auto estimate = [&](const TTTensor& tt, int samples) {
    double max_diff = 0.0;
    std::vector<Index> idx(q);
    for (int s = 0; s < samples; ++s) {
      for (int k = 0; k < q; ++k) idx[k] = static_cast<Index>(rng.integer(dims[k]));
      if (f.audit) f.audit->add();
      const double exact = f.fn(idx.data());
      const double approx = tt.entry(idx.data());
      max_abs_seen = std::max(max_abs_seen, std::abs(exact));
      max_diff = std::max(max_diff, std::abs(exact - approx));
    }
    return max_abs_seen > 0.0 ? max_diff / max_abs_seen : max_diff;
  };

  const int min_sweeps = q == 2 ? 1 : opt.min_sweeps;
  TTTensor best_tt;
  double best_est = std::numeric_limits<double>::infinity();
  for (int sweep = 0; sweep < opt.max_sweeps; ++sweep) {
    if (sweep % 2 == 0)
      for (int k = 0; k <= q - 2; ++k) run_supercore(k);
    else
      for (int k = q - 2; k >= 0; --k) run_supercore(k);
    res.sweeps = sweep + 1;
    if (sweep + 1 >= min_sweeps) {
      TTTensor cand = assemble();
      const double est = estimate(cand, opt.error_samples);
      if (std::getenv("PHMAT_CROSS_DEBUG")) {
        std::fprintf(stderr, "[cross] sweep=%d eps_aca=%.2e est=%.2e ranks:", sweep + 1, eps_aca, est);
        for (int i = 0; i <= cand.order(); ++i) std::fprintf(stderr, " %lld", static_cast<long long>(cand.rank(i)));
        std::fprintf(stderr, "\n");
      }
      if (est < best_est) {
        best_est = est;
        res.est_rel_error = est;
        best_tt = std::move(cand);
      }
      if (best_est <= 0.9 * opt.eps || res.rank_capped) break;
      const double factor = std::clamp(0.45 * opt.eps / best_est, 0.05, 0.8);
      eps_aca = std::max(eps_aca * factor, 0.005 * opt.eps);
    }
  }
  if (best_tt.cores.empty()) best_tt = assemble();
  if (opt.round_after) {
    best_tt = tt_round(best_tt, 0.0, 0.1 * opt.eps * max_abs_seen);
    res.est_rel_error = estimate(best_tt, opt.error_samples);
    if (std::getenv("PHMAT_CROSS_DEBUG")) {
      std::fprintf(stderr, "[cross] rounded est=%.2e ranks:", res.est_rel_error);
      for (int i = 0; i <= best_tt.order(); ++i) std::fprintf(stderr, " %lld", static_cast<long long>(best_tt.rank(i)));
      std::fprintf(stderr, "\n");
    }
  }
  res.converged = res.est_rel_error <= opt.eps;
  res.tt = std::move(best_tt);
  res.max_aca_resid = *std::max_element(bond_ratio.begin(), bond_ratio.end());
  res.evals = memo.fresh();
  return res;
}

// aca_partial (baselines.cpp:45-50): Rng(seed), the ACA engine, and the
// rank-1 terms as the columns of V (m x t) and Y (n x t).
LowRank aca_partial_rng(const std::function<double(Index, Index)>& entry, Index m, Index n, double eps, Index r_max,
                        Rng& rng) {
  PHM_CHECK(eps > 0.0, "aca_partial: eps must be positive");
  AcaOut a = aca(entry, m, n, eps, r_max, rng, nullptr);
  LowRank f;
  f.capped = a.capped;
  const Index t = a.rank();
  f.v = Mat(m, t);
  f.y = Mat(n, t);
  for (Index l = 0; l < t; ++l) {
    std::copy(a.us[l].begin(), a.us[l].end(), f.v.a.begin() + l * m);
    std::copy(a.vs[l].begin(), a.vs[l].end(), f.y.a.begin() + l * n);
  }
  return f;
}
LowRank aca_partial(const std::function<double(Index, Index)>& entry, Index m, Index n, double eps, Index r_max,
                    std::uint64_t seed) {
  Rng rng(seed);
  return aca_partial_rng(entry, m, n, eps, r_max, rng);
}

}  // namespace phm
