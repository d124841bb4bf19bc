// cqr_oracle.cpp — CPU restatement of the reference hot path (test
// infrastructure only; see cqr_oracle.h). Every function cites the reference
// file:line it restates (paths relative to /root/reference/proj).
//
// Compiled with -ffp-contract=off: the only fused multiply-adds are the
// explicit std::fma calls, so vectorisation cannot change a result and the
// fixed summation orders below are exactly what executes.

#include "cqr_oracle.h"

#include <algorithm>
#include <atomic>
#include <chrono>
#include <cmath>
#include <cstring>
#include <functional>
#include <limits>
#include <numbers>
#include <stdexcept>
#include <string>
#include <thread>
#include <unordered_set>
#include <vector>

namespace {

using Index = int64_t;
constexpr double kU = std::numeric_limits<double>::epsilon();  // types.hpp:31

// ---- errors (errors.hpp:18-33, 84-93) -------------------------------------
struct CholeskyBreakdown {
  Index pivot;
};
struct SingularTriangular {
  Index index;
};
struct InvalidArgument {
  std::string what;
};
struct NoConvergence {};

void require(bool c, const char* msg) {
  if (!c) throw InvalidArgument{msg};
}

// ---- dense row-major matrix --------------------------------------------------
struct Mat {
  Index rows = 0, cols = 0;
  std::vector<double> v;
  Mat() = default;
  Mat(Index r, Index c) : rows(r), cols(c), v(static_cast<size_t>(r * c), 0.0) {}
  double& operator()(Index i, Index j) { return v[static_cast<size_t>(i * cols + j)]; }
  double operator()(Index i, Index j) const { return v[static_cast<size_t>(i * cols + j)]; }
  double* row(Index i) { return v.data() + i * cols; }
  const double* row(Index i) const { return v.data() + i * cols; }
  size_t size() const { return v.size(); }
};

Mat from_strided(const double* a, Index m, Index n, Index lda) {
  Mat out(m, n);
  for (Index i = 0; i < m; ++i) std::memcpy(out.row(i), a + i * lda, sizeof(double) * n);
  return out;
}

// ---- rng (rng.hpp:18-92), bit-exact restatement --------------------------
constexpr uint64_t kGolden = 0x9E3779B97F4A7C15ull;
constexpr uint64_t kMix1 = 0xBF58476D1CE4E5B9ull;
constexpr uint64_t kMix2 = 0x94D049BB133111EBull;

inline uint64_t mix64(uint64_t z) {  // rng.hpp:22-26
  z = (z ^ (z >> 30)) * kMix1;
  z = (z ^ (z >> 27)) * kMix2;
  return z ^ (z >> 31);
}
inline uint64_t bits_at(uint64_t seed, uint64_t k) { return mix64(seed + (k + 1) * kGolden); }
inline uint64_t derive(uint64_t seed, uint64_t salt) {  // rng.hpp:35-37
  return mix64(seed ^ mix64(salt + 0x51ED270B8A5EC473ull));
}
inline double unit_at(uint64_t seed, uint64_t k) {  // rng.hpp:40-42
  return static_cast<double>(bits_at(seed, k) >> 11) * 0x1.0p-53;
}
inline double gaussian_at(uint64_t seed, uint64_t k) {  // rng.hpp:47-55
  const uint64_t pair = k / 2;
  const double u1 = static_cast<double>((bits_at(seed, 2 * pair) >> 11) + 1) * 0x1.0p-53;
  const double u2 = unit_at(seed, 2 * pair + 1);
  const double r = std::sqrt(-2.0 * std::log(u1));
  const double a = 2.0 * std::numbers::pi * u2;
  return (k % 2 == 0) ? r * std::cos(a) : r * std::sin(a);
}

struct Stream {  // rng.hpp:58-82
  uint64_t seed, pos;
  Index next_index(Index bound) {
    const double u = unit_at(seed, pos++);
    return static_cast<Index>(u * static_cast<double>(bound));
  }
};

Mat gaussian_matrix(Index rows, Index cols, uint64_t seed) {  // rng.hpp:86-92
  Mat g(rows, cols);
  for (Index i = 0; i < rows; ++i)
    for (Index j = 0; j < cols; ++j) g(i, j) = gaussian_at(seed, static_cast<uint64_t>(i * cols + j));
  return g;
}

// ---- workers (engine.cpp:12-22) ---------------------------------------------
void run_on_workers(int workers, const std::function<void(int)>& fn) {
  if (workers <= 1) {
    fn(0);
    return;
  }
  std::vector<std::thread> pool;
  for (int w = 1; w < workers; ++w) pool.emplace_back(fn, w);
  fn(0);
  for (auto& t : pool) t.join();
}

// Row-block offsets ceil(b*m/p) (parexec.cpp:9-18).
Index block_offset(Index m, int p, int b) {
  if (b <= 0) return 0;
  if (b >= p) return m;
  return (static_cast<Index>(b) * m + p - 1) / p;
}

// ---- sketch (sketch.cpp:20-127) ---------------------------------------------
Index resolved_size(const cqr_sketch_cfg& cfg, Index m, Index n) {  // sketch.cpp:20-23
  Index l = cfg.size > 0 ? cfg.size : static_cast<Index>(std::ceil(cfg.rate * static_cast<double>(n)));
  return std::clamp(l, n, m);
}

std::vector<Index> draw_indices(Index m, Index l, bool without, Stream& s) {  // sketch.cpp:27-40
  std::vector<Index> idx;
  idx.reserve(static_cast<size_t>(l));
  if (!without) {
    for (Index k = 0; k < l; ++k) idx.push_back(s.next_index(m));
  } else {
    std::unordered_set<Index> seen;
    while (static_cast<Index>(idx.size()) < l) {
      const Index i = s.next_index(m);
      if (seen.insert(i).second) idx.push_back(i);
    }
  }
  return idx;
}

Mat sample_rows_uniform(const Mat& a, Index l, bool without, Stream& s, std::vector<Index>* out_idx) {
  // sketch.cpp:45-55
  std::vector<Index> idx = draw_indices(a.rows, l, without, s);
  Mat a1(l, a.cols);
  for (Index k = 0; k < l; ++k) std::memcpy(a1.row(k), a.row(idx[static_cast<size_t>(k)]), sizeof(double) * a.cols);
  if (out_idx) *out_idx = std::move(idx);
  return a1;
}

// sketch.cpp:94-116. Omega(i, j) = gaussian_at(seed, i*m + j), generated in
// 2048-column chunks; fixed order: for each chunk, t(i,c) = fma-chain over the
// chunk's rows in ascending order starting from 0, then a1(i,c) += t(i,c).
// Test-harness knob (orc_set_test_threads): the reference's sketch is serial
// (sketch.cpp:94-116) and so is this one by default (bench.py's CPU arm keeps it
// so); the parity tests may split the sketch rows i, and the diagnostics' Gram
// leaves and residual panels, over threads. Each a1(i, :) is computed by one thread
// with exactly the serial arithmetic (chunks ascending, rows ascending inside a
// chunk), so the result is bitwise the same for any thread count.
std::atomic<int> g_test_threads{1};

Mat sketch_gaussian(const Mat& a, Index l, uint64_t seed, Index m_global = -1, Index row0 = 0) {
  // m_global/row0: a row block of a larger matrix (counters use global rows,
  // the decomposition the multi-GPU path relies on)
  const Index m = a.rows, n = a.cols;
  const Index mg = m_global < 0 ? m : m_global;
  Mat a1(l, n);
  constexpr Index kChunk = 2048;
  const int workers = static_cast<int>(std::max<Index>(1, std::min<Index>(g_test_threads.load(), l)));
  run_on_workers(workers, [&](int w) {
    std::vector<double> omega(static_cast<size_t>(std::min(m, kChunk)));
    std::vector<double> t(static_cast<size_t>(n));
    const Index i0 = l * w / workers, i1 = l * (w + 1) / workers;
    for (Index i = i0; i < i1; ++i) {
      double* out = a1.row(i);
      for (Index j0 = 0; j0 < m; j0 += kChunk) {
        const Index len = std::min(m - j0, kChunk);
        for (Index jj = 0; jj < len; ++jj)
          omega[static_cast<size_t>(jj)] = gaussian_at(seed, static_cast<uint64_t>(i * mg + row0 + j0 + jj));
        std::fill(t.begin(), t.end(), 0.0);
        for (Index jj = 0; jj < len; ++jj) {
          const double wv = omega[static_cast<size_t>(jj)];
          const double* ar = a.row(j0 + jj);
          for (Index c = 0; c < n; ++c) t[c] = std::fma(wv, ar[c], t[c]);
        }
        for (Index c = 0; c < n; ++c) out[c] += t[c];
      }
    }
  });
  return a1;
}

Mat make_sketch(const Mat& a, const cqr_sketch_cfg& cfg, Index l, Stream& s) {  // sketch.cpp:118-127
  switch (cfg.strategy) {
    case CQR_UNIFORM: return sample_rows_uniform(a, l, cfg.without_replacement != 0, s, nullptr);
    case CQR_GAUSSIAN: return sketch_gaussian(a, l, s.seed);
    case CQR_LEVERAGE:
      throw InvalidArgument{"leverage sampling needs an oracle Q; call sample_rows_leverage directly"};
  }
  throw InvalidArgument{"unknown sketch strategy"};
}

// ---- kernels (kernels.hpp) ----------------------------------------------------
constexpr Index kGramLeafRows = 1024;  // kernels.hpp:20

// One leaf's upper triangle: fixed order g(i,j) = fma-chain over the leaf's rows
// in ascending order starting from +0 (restates the Eigen rankUpdate of
// kernels.hpp:36 with a pinned order).
void gram_leaf(const double* x, Index ldx, Index rows, Index n, double* g) {
  std::fill(g, g + n * n, 0.0);
  for (Index k = 0; k < rows; ++k) {
    const double* xr = x + k * ldx;
    for (Index i = 0; i < n; ++i) {
      const double xi = xr[i];
      double* gr = g + i * n;
      for (Index j = i; j < n; ++j) gr[j] = std::fma(xi, xr[j], gr[j]);
    }
  }
}

// kernels.hpp:42-57: pairwise tree (0+1)+(2+3)+...; an odd trailing slot is
// carried up unchanged. Slots are `count` arrays of `len` doubles, consumed.
void gram_tree_combine(std::vector<double>& slots, Index count, Index len) {
  Index cur = count;
  while (cur > 1) {
    const Index pairs = cur / 2;
    for (Index i = 0; i < pairs; ++i) {
      double* d = slots.data() + i * len;
      const double* a = slots.data() + (2 * i) * len;
      const double* b = slots.data() + (2 * i + 1) * len;
      for (Index e = 0; e < len; ++e) d[e] = a[e] + b[e];
    }
    if (cur % 2 == 1) {
      if (pairs != cur - 1)
        std::memmove(slots.data() + pairs * len, slots.data() + (cur - 1) * len, sizeof(double) * len);
      cur = pairs + 1;
    } else {
      cur = pairs;
    }
  }
}

void mirror_upper(double* g, Index n) {  // kernels.hpp:69
  for (Index i = 0; i < n; ++i)
    for (Index j = 0; j < i; ++j) g[i * n + j] = g[j * n + i];
}

// kernels.hpp:64-71 + engine.cpp:24-39 (leaves split over workers; bitwise
// independent of the worker count).
Mat gram(const double* x, Index m, Index n, Index ldx, int workers) {
  require(m >= n, "gram: matrix must have rows >= cols");
  const Index leaves = (m + kGramLeafRows - 1) / kGramLeafRows;
  const Index len = n * n;
  std::vector<double> slots(static_cast<size_t>(std::max<Index>(leaves, 1) * len), 0.0);
  auto work = [&](Index lo, Index hi) {
    for (Index leaf = lo; leaf < hi; ++leaf) {
      const Index r0 = leaf * kGramLeafRows;
      const Index rows = std::min(m - r0, kGramLeafRows);
      gram_leaf(x + r0 * ldx, ldx, rows, n, slots.data() + leaf * len);
    }
  };
  if (workers <= 1) {
    work(0, leaves);
  } else {
    run_on_workers(workers, [&](int w) { work(leaves * w / workers, leaves * (w + 1) / workers); });
  }
  gram_tree_combine(slots, leaves, len);
  Mat g(n, n);
  std::memcpy(g.v.data(), slots.data(), sizeof(double) * len);
  mirror_upper(g.v.data(), n);
  return g;
}

// kernels.hpp:76-90. Fixed order (right-looking restatement of the dot /
// squaredNorm reductions): s(i,j) = g(i,j); for k < i: s = fma(-r(k,i), r(k,j), s);
// diagonal: !(s > 0) -> CholeskyBreakdown(i), r(i,i) = sqrt(s); off-diagonal:
// r(i,j) = s / r(i,i).
Mat cholesky_upper(const Mat& g) {
  require(g.rows == g.cols, "cholesky_upper: matrix must be square");
  const Index n = g.rows;
  Mat s = g;  // trailing working copy (upper triangle used)
  Mat r(n, n);
  for (Index i = 0; i < n; ++i) {
    const double sii = s(i, i);
    if (!(sii > 0.0)) throw CholeskyBreakdown{i};
    const double d = std::sqrt(sii);
    r(i, i) = d;
    for (Index j = i + 1; j < n; ++j) r(i, j) = s(i, j) / d;
    // trailing update, element order k ascending by construction
    for (Index a = i + 1; a < n; ++a) {
      const double ria = r(i, a);
      for (Index b = a; b < n; ++b) s(a, b) = std::fma(-ria, r(i, b), s(a, b));
    }
  }
  return r;
}

// kernels.hpp:94-127: exact restatement (256-row panels, column-major panel
// copy, y_j = fma(-r_kj, x_k, y_j) for k < j skipping r_kj == 0, y_j /= r_jj).
constexpr Index kTrisolvePanelRows = 256;

void right_trisolve_block(double* x, Index rows, Index n, Index ldx, const Mat& rc_colmajor) {
  std::vector<double> w(static_cast<size_t>(kTrisolvePanelRows * n));
  for (Index p0 = 0; p0 < rows; p0 += kTrisolvePanelRows) {
    const Index pr = std::min(rows - p0, kTrisolvePanelRows);
    for (Index i = 0; i < pr; ++i)
      for (Index j = 0; j < n; ++j) w[static_cast<size_t>(j * kTrisolvePanelRows + i)] = x[(p0 + i) * ldx + j];
    for (Index j = 0; j < n; ++j) {
      double* yj = w.data() + j * kTrisolvePanelRows;
      for (Index k = 0; k < j; ++k) {
        const double c = rc_colmajor.v[static_cast<size_t>(j * n + k)];  // R(k, j)
        if (c == 0.0) continue;
        const double* xk = w.data() + k * kTrisolvePanelRows;
        for (Index i = 0; i < pr; ++i) yj[i] = std::fma(-c, xk[i], yj[i]);
      }
      const double d = rc_colmajor.v[static_cast<size_t>(j * n + j)];
      for (Index i = 0; i < pr; ++i) yj[i] /= d;
    }
    for (Index i = 0; i < pr; ++i)
      for (Index j = 0; j < n; ++j) x[(p0 + i) * ldx + j] = w[static_cast<size_t>(j * kTrisolvePanelRows + i)];
  }
}

void check_diag(const Mat& r) {  // kernels.hpp:106-107, engine.cpp:124-125
  for (Index j = 0; j < r.rows; ++j)
    if (r(j, j) == 0.0) throw SingularTriangular{j};
}

// engine.cpp:60-67 / parexec.cpp:30-38: each worker solves its row block.
void trisolve_inplace(double* x, Index m, Index n, Index ldx, const Mat& r, int workers) {
  require(r.rows == n && r.cols == n, "right_trisolve: dimension mismatch");
  check_diag(r);
  Mat rc(n, n);  // column-major copy: rc.v[j*n + k] = R(k, j)
  for (Index k = 0; k < n; ++k)
    for (Index j = 0; j < n; ++j) rc.v[static_cast<size_t>(j * n + k)] = r(k, j);
  const int p = static_cast<int>(std::max<Index>(1, std::min<Index>(workers, m)));
  run_on_workers(p, [&](int w) {
    const Index lo = block_offset(m, p, w), hi = block_offset(m, p, w + 1);
    if (hi > lo) right_trisolve_block(x + lo * ldx, hi - lo, n, ldx, rc);
  });
}

// Householder reflector (the published algorithm behind Eigen's
// makeHouseholder): beta = -sign(c0) * sqrt(c0^2 + ||tail||^2),
// tau = (beta - c0) / beta, v = tail / (c0 - beta); a tail with squared norm
// <= (smallest normal)^2 gives tau = 0. Fixed orders: ||tail||^2 and the
// w = v^T A products are fma chains in ascending row order.
struct HouseholderQr {
  Mat w;                    // column-major working copy, w.v[c*l + i]
  std::vector<double> tau;  // per column
  Index l = 0, n = 0;
};

HouseholderQr householder(const Mat& a) {
  HouseholderQr h;
  h.l = a.rows;
  h.n = a.cols;
  const Index l = h.l, n = h.n;
  h.w = Mat(n, l);  // used as column-major l x n
  for (Index i = 0; i < l; ++i)
    for (Index c = 0; c < n; ++c) h.w.v[static_cast<size_t>(c * l + i)] = a(i, c);
  h.tau.assign(static_cast<size_t>(n), 0.0);
  const double tol = std::numeric_limits<double>::min() * std::numeric_limits<double>::min();
  for (Index j = 0; j < n; ++j) {
    double* col = h.w.v.data() + j * l;
    const double c0 = col[j];
    double tail = 0.0;
    for (Index i = j + 1; i < l; ++i) tail = std::fma(col[i], col[i], tail);
    double tau, beta;
    if (tail <= tol) {
      tau = 0.0;
      beta = c0;
      for (Index i = j + 1; i < l; ++i) col[i] = 0.0;
    } else {
      beta = std::sqrt(c0 * c0 + tail);
      if (c0 >= 0.0) beta = -beta;
      const double denom = c0 - beta;
      for (Index i = j + 1; i < l; ++i) col[i] = col[i] / denom;
      tau = (beta - c0) / beta;
    }
    col[j] = beta;
    h.tau[static_cast<size_t>(j)] = tau;
    if (tau != 0.0) {
      for (Index c = j + 1; c < n; ++c) {
        double* cc = h.w.v.data() + c * l;
        double s = cc[j];
        for (Index i = j + 1; i < l; ++i) s = std::fma(col[i], cc[i], s);
        const double ts = tau * s;
        cc[j] -= ts;
        for (Index i = j + 1; i < l; ++i) cc[i] = std::fma(-ts, col[i], cc[i]);
      }
    }
  }
  return h;
}

void normalize_r_sign(Mat& r) {  // kernels.hpp:165-168
  for (Index i = 0; i < r.rows; ++i)
    if (r(i, i) < 0.0)
      for (Index j = i; j < r.cols; ++j) r(i, j) = -r(i, j);
}

Mat qr_r_factor(const Mat& a1) {  // kernels.hpp:175-184
  require(a1.rows >= a1.cols, "qr_r_factor: need rows >= cols");
  HouseholderQr h = householder(a1);
  const Index n = a1.cols, l = a1.rows;
  Mat r(n, n);
  for (Index i = 0; i < n; ++i)
    for (Index j = i; j < n; ++j) r(i, j) = h.w.v[static_cast<size_t>(j * l + i)];
  normalize_r_sign(r);
  return r;
}

// Thin Q = H_0 ... H_{n-1} I(m x n) (kernels.hpp:192-209, matgen.cpp:12-19).
Mat householder_q(const HouseholderQr& h) {
  const Index l = h.l, n = h.n;
  std::vector<double> q(static_cast<size_t>(n * l), 0.0);  // column-major l x n
  for (Index c = 0; c < n; ++c) q[static_cast<size_t>(c * l + c)] = 1.0;
  for (Index j = n - 1; j >= 0; --j) {
    const double tau = h.tau[static_cast<size_t>(j)];
    if (tau == 0.0) continue;
    const double* v = h.w.v.data() + j * l;  // v[j] = 1 implicit, v[i>j] stored
    for (Index c = j; c < n; ++c) {
      double* qc = q.data() + c * l;
      double s = qc[j];
      for (Index i = j + 1; i < l; ++i) s = std::fma(v[i], qc[i], s);
      const double ts = tau * s;
      qc[j] -= ts;
      for (Index i = j + 1; i < l; ++i) qc[i] = std::fma(-ts, v[i], qc[i]);
    }
  }
  Mat out(l, n);
  for (Index i = 0; i < l; ++i)
    for (Index c = 0; c < n; ++c) out(i, c) = q[static_cast<size_t>(c * l + i)];
  return out;
}

struct ThinQr {
  Mat q, r;
};

ThinQr householder_qr_thin(const Mat& a) {  // kernels.hpp:192-209
  require(a.rows >= a.cols, "householder_qr_thin: need rows >= cols");
  HouseholderQr h = householder(a);
  ThinQr out;
  const Index n = a.cols, l = a.rows;
  out.r = Mat(n, n);
  for (Index i = 0; i < n; ++i)
    for (Index j = i; j < n; ++j) out.r(i, j) = h.w.v[static_cast<size_t>(j * l + i)];
  out.q = householder_q(h);
  for (Index i = 0; i < n; ++i) {
    if (out.r(i, i) < 0.0) {
      for (Index j = i; j < n; ++j) out.r(i, j) = -out.r(i, j);
      for (Index k = 0; k < l; ++k) out.q(k, i) = -out.q(k, i);
    }
  }
  return out;
}

// kernels.hpp:211-248: row-partially-pivoted LU; strict '>' keeps the first
// maximum; exactly-zero pivot -> SingularTriangular(j). Fixed order: the
// trailing update is w(i,k) = fma(-mult, w(j,k), w(i,k)), skipped when mult == 0.
struct Lu {
  Mat packed;
  std::vector<Index> perm;
};

Lu lu_decompose(const Mat& a1) {
  require(a1.rows >= a1.cols, "lu_decompose: need rows >= cols");
  const Index l = a1.rows, n = a1.cols;
  Lu f;
  f.packed = a1;
  f.perm.resize(static_cast<size_t>(l));
  for (Index i = 0; i < l; ++i) f.perm[static_cast<size_t>(i)] = i;
  Mat& w = f.packed;
  for (Index j = 0; j < n; ++j) {
    Index piv = j;
    double best = std::abs(w(j, j));
    for (Index i = j + 1; i < l; ++i) {
      const double v = std::abs(w(i, j));
      if (v > best) {
        best = v;
        piv = i;
      }
    }
    if (w(piv, j) == 0.0) throw SingularTriangular{j};
    if (piv != j) {
      for (Index c = 0; c < n; ++c) std::swap(w(j, c), w(piv, c));
      std::swap(f.perm[static_cast<size_t>(j)], f.perm[static_cast<size_t>(piv)]);
    }
    const double d = w(j, j);
    const double* pr = w.row(j);
    for (Index i = j + 1; i < l; ++i) {
      double* ri = w.row(i);
      const double mult = ri[j] / d;
      ri[j] = mult;
      if (mult != 0.0)
        for (Index c = j + 1; c < n; ++c) ri[c] = std::fma(-mult, pr[c], ri[c]);
    }
  }
  return f;
}

Mat lu_u_factor(const Mat& a1) {  // kernels.hpp:251-257
  Lu f = lu_decompose(a1);
  const Index n = a1.cols;
  Mat u(n, n);
  for (Index i = 0; i < n; ++i)
    for (Index j = i; j < n; ++j) u(i, j) = f.packed(i, j);
  return u;
}

// kernels.hpp:272-310: one-sided Jacobi singular values (restated loops).
std::vector<double> svd_values(const Mat& m_in) {
  constexpr int kMaxSweeps = 100;
  const bool tall = m_in.rows >= m_in.cols;
  const Index rows = tall ? m_in.rows : m_in.cols;
  const Index c = tall ? m_in.cols : m_in.rows;
  std::vector<double> w(static_cast<size_t>(rows * c));  // column-major rows x c
  for (Index i = 0; i < rows; ++i)
    for (Index j = 0; j < c; ++j)
      w[static_cast<size_t>(j * rows + i)] = tall ? m_in(i, j) : m_in(j, i);
  const double tol = 10.0 * kU * std::sqrt(static_cast<double>(rows));
  auto dot = [&](Index p, Index q) {
    const double* a = w.data() + p * rows;
    const double* b = w.data() + q * rows;
    double s = 0.0;
    for (Index i = 0; i < rows; ++i) s = std::fma(a[i], b[i], s);
    return s;
  };
  bool converged = (c <= 1);
  for (int sweep = 0; sweep < kMaxSweeps && !converged; ++sweep) {
    converged = true;
    for (Index p = 0; p < c - 1; ++p) {
      for (Index q = p + 1; q < c; ++q) {
        const double alpha = dot(p, p), beta = dot(q, q), gamma = dot(p, q);
        if (std::abs(gamma) <= tol * std::sqrt(alpha * beta)) continue;
        converged = false;
        const double zeta = (beta - alpha) / (2.0 * gamma);
        const double t = ((zeta >= 0.0) ? 1.0 : -1.0) / (std::abs(zeta) + std::sqrt(1.0 + zeta * zeta));
        const double cs = 1.0 / std::sqrt(1.0 + t * t);
        const double sn = cs * t;
        double* wp = w.data() + p * rows;
        double* wq = w.data() + q * rows;
        for (Index i = 0; i < rows; ++i) {
          const double a = wp[i], b = wq[i];
          wp[i] = cs * a - sn * b;
          wq[i] = sn * a + cs * b;
        }
      }
    }
  }
  if (!converged) throw NoConvergence{};
  std::vector<double> sv(static_cast<size_t>(c));
  for (Index j = 0; j < c; ++j) sv[static_cast<size_t>(j)] = std::sqrt(dot(j, j));
  std::sort(sv.begin(), sv.end(), std::greater<double>());
  return sv;
}

// engine.cpp:103-107: dense L*R with the strict lower part zeroed. Fixed order:
// fma chain over k ascending from +0 (zero terms of the triangles included).
Mat triangular_product(const Mat& left, const Mat& right) {
  const Index n = left.rows;
  Mat out(n, n);
  for (Index i = 0; i < n; ++i)
    for (Index j = 0; j < n; ++j) {
      if (j < i) continue;
      double s = 0.0;
      for (Index k = 0; k < n; ++k) s = std::fma(left(i, k), right(k, j), s);
      out(i, j) = s;
    }
  return out;
}

// ---- engine (engine.cpp:78-305) -----------------------------------------------
struct Clock {
  double ms[CQR_STAGE_COUNT] = {0};
  void add(int s, double v) { ms[s] += v; }
};
struct Scoped {
  Clock& c;
  int s;
  std::chrono::steady_clock::time_point t0 = std::chrono::steady_clock::now();
  Scoped(Clock& c_, int s_) : c(c_), s(s_) {}
  ~Scoped() {
    c.add(s, std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count());
  }
};

struct StageRec {
  int stage;
  bool has_cond = false;
  double cond = 0;
  bool has_shift = false;
  double shift = 0;
  int retries = 0;
};

struct Fact {
  Mat q, r;
  bool has_r = false;
  std::vector<StageRec> stages;
  Index sketch_rows = 0;
};

struct Engine {  // engine.cpp:45-74: owns a copy of A mutated in place A->X->Q
  Mat work;
  int p;
  Clock& clock;
  Engine(const Mat& a, int p_, Clock& c) : work(a), p(p_), clock(c) {}
  Mat gram_() {
    Scoped t(clock, CQR_STAGE_GRAM);
    return gram(work.v.data(), work.rows, work.cols, work.cols, p);
  }
  void trisolve(const Mat& r) {
    Scoped t(clock, CQR_STAGE_TRISOLVE);
    trisolve_inplace(work.v.data(), work.rows, work.cols, work.cols, r, p);
  }
};

// engine.cpp:78-92 with the shift of cholqr.cpp:21-26 already resolved by the
// caller (engine.cpp:270 resolves the theory shift from a.squaredNorm() before
// the first pass).
struct ShiftSpec {
  bool enabled = false;
  double value = 0;
};

// Eigen's a.squaredNorm() (engine.cpp:270): the sum of the squared entries.
// Eigen does not pin the order; this restatement sums row-major, sequentially.
// (The B200 engine takes trace(G1) of the first Gram instead -- the same number
// in exact arithmetic, without the extra pass over A -- so the sCholQR3-theory
// parity test is a tolerance test.)
double squared_norm(const Mat& a) {
  double s = 0.0;
  for (const double v : a.v) s += v * v;
  return s;
}

double theory_shift(Index m, Index n, double fro2) {  // cholqr.cpp:21-26
  const double mn = static_cast<double>(m) * static_cast<double>(n);
  const double nn = static_cast<double>(n) * static_cast<double>(n + 1);
  return 11.0 * (mn + nn) * kU * fro2;
}

Mat cholesky_pass(Engine& eng, Fact& f, ShiftSpec shift = {}) {
  Mat g = eng.gram_();
  f.stages.push_back({CQR_STAGE_GRAM});
  Mat r;
  double applied = 0;
  {
    Scoped t(eng.clock, CQR_STAGE_CHOLESKY);
    if (shift.enabled) {
      applied = shift.value;
      for (Index j = 0; j < g.rows; ++j) g(j, j) += applied;
    }
    r = cholesky_upper(g);
  }
  StageRec ch{CQR_STAGE_CHOLESKY};
  if (shift.enabled) {
    ch.has_shift = true;
    ch.shift = applied;
  }
  f.stages.push_back(ch);
  eng.trisolve(r);
  f.stages.push_back({CQR_STAGE_TRISOLVE});
  return r;
}

double cond_estimate(const Mat& x) {  // engine.cpp:94-100
  const Mat r = qr_r_factor(x);
  const std::vector<double> sv = svd_values(r);
  const double smin = sv.back();
  if (smin <= 0.0) return std::numeric_limits<double>::infinity();
  return sv.front() / smin;
}

void normalize_sign(Fact& f) {  // engine.cpp:109-116
  for (Index i = 0; i < f.r.rows; ++i) {
    if (f.r(i, i) < 0.0) {
      for (Index j = i; j < f.r.cols; ++j) f.r(i, j) = -f.r(i, j);
      for (Index k = 0; k < f.q.rows; ++k) f.q(k, i) = -f.q(k, i);
    }
  }
}

bool degenerate_diagonal(const Mat& r, Index& where) {  // engine.cpp:118-127
  for (Index i = 0; i < r.rows; ++i) {
    const double d = r(i, i);
    if (d == 0.0 || !std::isfinite(d)) {
      where = i;
      return true;
    }
  }
  return false;
}

using Precond = std::function<Mat(const Mat&)>;

// engine.cpp:137-209
Fact run_precond_impl(const Mat& a, const Precond& precond, const cqr_sketch_cfg& cfg, int p,
                      bool diagnostics, bool r_less, Clock& clock) {
  const Index base_l = resolved_size(cfg, a.rows, a.cols);
  for (int attempt = 0;; ++attempt) {
    cqr_sketch_cfg try_cfg = cfg;
    try_cfg.size = std::min<Index>(
        a.rows, static_cast<Index>(std::llround(static_cast<double>(base_l) * std::pow(cfg.retry_growth, attempt))));
    Stream stream{attempt == 0 ? cfg.seed : derive(cfg.seed, static_cast<uint64_t>(attempt)), 0};
    const bool last = attempt >= cfg.max_retries;
    const Index l = resolved_size(try_cfg, a.rows, a.cols);

    Fact fact;
    Mat a1;
    {
      Scoped t(clock, CQR_STAGE_SKETCH);
      a1 = make_sketch(a, try_cfg, l, stream);
    }
    Mat rt;
    {
      Scoped t(clock, CQR_STAGE_PRECONDITION);
      Index bad = 0;
      try {
        rt = precond(a1);
        if (degenerate_diagonal(rt, bad)) throw SingularTriangular{bad};
      } catch (const SingularTriangular&) {
        if (last) throw;
        continue;
      }
    }
    fact.stages.push_back({CQR_STAGE_SKETCH, false, 0, false, 0, attempt});
    try {
      Engine eng(a, p, clock);
      eng.trisolve(rt);
      StageRec pre{CQR_STAGE_PRECONDITION};
      if (diagnostics) {
        pre.has_cond = true;
        try {
          pre.cond = cond_estimate(eng.work);
        } catch (const NoConvergence&) {
          pre.cond = std::numeric_limits<double>::quiet_NaN();
        } catch (const InvalidArgument&) {
          pre.cond = std::numeric_limits<double>::quiet_NaN();
        }
      }
      fact.stages.push_back(pre);
      const Mat rhat = cholesky_pass(eng, fact);
      fact.q = std::move(eng.work);
      fact.sketch_rows = l;
      if (!r_less) {
        Scoped t(clock, CQR_STAGE_RECOVER);
        fact.r = triangular_product(rhat, rt);
        fact.has_r = true;
        normalize_sign(fact);
        fact.stages.push_back({CQR_STAGE_RECOVER});
      }
      return fact;
    } catch (const CholeskyBreakdown&) {
      if (last) throw;
    } catch (const SingularTriangular&) {
      if (last) throw;
    }
  }
}

void require_finite(const Mat& a) {
  for (double v : a.v)
    if (!std::isfinite(v)) throw InvalidArgument{"A has non-finite entries"};
}

Fact run_method(int method, const Mat& a, int p, const cqr_sketch_cfg& sk, const cqr_options& o,
                Clock& clock) {
  require_finite(a);
  require(a.rows >= a.cols && a.cols >= 1, "need m >= n >= 1");
  require(p >= 1 && p <= a.rows, "worker count must be in [1, m]");
  const bool r_less = o.r_less != 0;
  switch (method) {
    case CQR_HOUSEHOLDER: {  // engine.cpp:227-239
      Fact f;
      {
        Scoped t(clock, CQR_STAGE_HOUSEHOLDER);
        ThinQr qr = householder_qr_thin(a);
        f.q = std::move(qr.q);
        if (!r_less) {
          f.r = std::move(qr.r);
          f.has_r = true;
        }
      }
      f.stages.push_back({CQR_STAGE_HOUSEHOLDER});
      return f;
    }
    case CQR_CHOLQR: {  // engine.cpp:241-250
      Engine eng(a, p, clock);
      Fact f;
      Mat r1 = cholesky_pass(eng, f);
      f.q = std::move(eng.work);
      if (!r_less) {
        f.r = std::move(r1);
        f.has_r = true;
      }
      return f;
    }
    case CQR_CHOLQR2: {  // engine.cpp:252-266
      Engine eng(a, p, clock);
      Fact f;
      const Mat r1 = cholesky_pass(eng, f);
      const Mat r2 = cholesky_pass(eng, f);
      f.q = std::move(eng.work);
      if (!r_less) {
        Scoped t(clock, CQR_STAGE_RECOVER);
        f.r = triangular_product(r2, r1);
        f.has_r = true;
        f.stages.push_back({CQR_STAGE_RECOVER});
      }
      return f;
    }
    case CQR_SCHOLQR3: {  // engine.cpp:268-284
      ShiftSpec sh;
      sh.enabled = true;
      sh.value = o.shift_kind == CQR_SHIFT_THEORY ? theory_shift(a.rows, a.cols, squared_norm(a)) : o.shift_value;
      Engine eng(a, p, clock);
      Fact f;
      const Mat r1 = cholesky_pass(eng, f, sh);
      const Mat r2 = cholesky_pass(eng, f);
      const Mat r3 = cholesky_pass(eng, f);
      f.q = std::move(eng.work);
      if (!r_less) {
        Scoped t(clock, CQR_STAGE_RECOVER);
        f.r = triangular_product(r3, triangular_product(r2, r1));
        f.has_r = true;
        f.stages.push_back({CQR_STAGE_RECOVER});
      }
      return f;
    }
    case CQR_RQR:
      return run_precond_impl(a, [](const Mat& a1) { return qr_r_factor(a1); }, sk, p, o.diagnostics != 0,
                              r_less, clock);
    case CQR_RLU:
      return run_precond_impl(a, [](const Mat& a1) { return lu_u_factor(a1); }, sk, p, o.diagnostics != 0,
                              r_less, clock);
    case CQR_RQR_GAUSSIAN: {
      cqr_sketch_cfg g = sk;
      g.strategy = CQR_GAUSSIAN;
      return run_precond_impl(a, [](const Mat& a1) { return qr_r_factor(a1); }, g, p, o.diagnostics != 0,
                              r_less, clock);
    }
  }
  throw InvalidArgument{"unknown method"};
}

void comm_model(int method, int p, Index n, Index l, int* rmin, int* rmax, double* vmin, double* vmax) {
  const double pn2 = static_cast<double>(p) * static_cast<double>(n) * static_cast<double>(n);
  const double nl = static_cast<double>(n) * static_cast<double>(l);
  int a = 0, b = 0;
  double c = 0, d = 0;
  switch (method) {  // parexec.cpp:44-62
    case CQR_CHOLQR: a = 2; b = 2; c = pn2; d = pn2; break;
    case CQR_CHOLQR2: a = 4; b = 4; c = 2 * pn2; d = 2 * pn2; break;
    case CQR_SCHOLQR3: a = 6; b = 6; c = 3 * pn2; d = 3 * pn2; break;
    case CQR_RLU:
    case CQR_RQR:
    case CQR_RQR_GAUSSIAN: a = 3; b = 4; c = 1.5 * pn2; d = 1.5 * pn2 + nl; break;
    default: break;
  }
  if (rmin) *rmin = a;
  if (rmax) *rmax = b;
  if (vmin) *vmin = c;
  if (vmax) *vmax = d;
}

void fill_report(cqr_report* rep, const Fact* f, const Clock& clock, int status, Index index, bool r_less,
                 int method, int p, Index n, Index l) {
  if (!rep) return;
  std::memset(rep, 0, sizeof(*rep));
  rep->status = status;
  rep->index = index;
  rep->r_less = r_less ? 1 : 0;
  double tot = 0;
  for (int s = 0; s < CQR_STAGE_COUNT; ++s) {
    rep->stage_ms[s] = clock.ms[s];
    tot += clock.ms[s];
  }
  rep->total_ms = tot;
  if (f) {
    rep->n_stages = static_cast<int32_t>(std::min<size_t>(f->stages.size(), CQR_MAX_STAGE_INFOS));
    for (int i = 0; i < rep->n_stages; ++i) {
      const StageRec& s = f->stages[static_cast<size_t>(i)];
      rep->stages[i].stage = s.stage;
      rep->stages[i].has_cond_x = s.has_cond;
      rep->stages[i].cond_x = s.cond;
      rep->stages[i].has_shift = s.has_shift;
      rep->stages[i].shift = s.shift;
      rep->stages[i].retries = s.retries;
    }
    rep->sketch_rows = f->sketch_rows;
  }
  double vmax = 0;
  int rmax = 0;
  comm_model(method, p, n, l, nullptr, &rmax, nullptr, &vmax);
  rep->comm_rounds = rmax;
  rep->comm_volume = vmax;
}

template <typename F>
int guarded(F&& f, int64_t* index = nullptr) {
  try {
    f();
    if (index) *index = -1;
    return CQR_OK;
  } catch (const CholeskyBreakdown& e) {
    if (index) *index = e.pivot;
    return CQR_CHOLESKY_BREAKDOWN;
  } catch (const SingularTriangular& e) {
    if (index) *index = e.index;
    return CQR_SINGULAR_TRIANGULAR;
  } catch (const InvalidArgument&) {
    return CQR_INVALID_ARGUMENT;
  } catch (const NoConvergence&) {
    return 8;
  }
}

void store(const Mat& m, double* out) { std::memcpy(out, m.v.data(), sizeof(double) * m.size()); }

cqr_sketch_cfg default_cfg() {
  cqr_sketch_cfg c{};
  c.strategy = CQR_UNIFORM;
  c.size = 0;
  c.rate = 2.0;
  c.seed = 0;
  c.max_retries = 2;
  c.retry_growth = 2.0;
  c.without_replacement = 0;
  return c;
}

int factor_common(int method, const double* a, Index m, Index n, Index lda, const cqr_sketch_cfg* cfg,
                  const cqr_options* opts, int workers, double* q, double* r, cqr_report* report,
                  const Precond* custom) {
  const cqr_sketch_cfg sk = cfg ? *cfg : default_cfg();
  cqr_options o{};
  o.shift_kind = CQR_SHIFT_THEORY;
  if (opts) o = *opts;
  Clock clock;
  Fact f;
  Index index = -1;
  Index l = (m >= n && n >= 1) ? resolved_size(sk, m, n) : 0;
  const int st = guarded(
      [&] {
        require(m >= 1 && n >= 1 && lda >= n, "bad shape");
        Mat A = from_strided(a, m, n, lda);
        if (custom) {
          require_finite(A);
          require(A.rows >= A.cols && A.cols >= 1, "need m >= n >= 1");
          require(workers >= 1 && workers <= A.rows, "worker count must be in [1, m]");
          f = run_precond_impl(A, *custom, sk, workers, o.diagnostics != 0, o.r_less != 0, clock);
        } else {
          f = run_method(method, A, workers, sk, o, clock);
        }
      },
      &index);
  if (st == CQR_OK) {
    store(f.q, q);
    if (f.has_r && r) store(f.r, r);
  }
  fill_report(report, st == CQR_OK ? &f : nullptr, clock, st, index, o.r_less != 0, method, workers, n, l);
  return st;
}

}  // namespace

// ============================ C ABI ==========================================
extern "C" {

uint64_t orc_mix64(uint64_t z) { return mix64(z); }
uint64_t orc_bits_at(uint64_t seed, uint64_t k) { return bits_at(seed, k); }
uint64_t orc_derive(uint64_t seed, uint64_t salt) { return derive(seed, salt); }
double orc_unit_at(uint64_t seed, uint64_t k) { return unit_at(seed, k); }
double orc_gaussian_at(uint64_t seed, uint64_t k) { return gaussian_at(seed, k); }
void orc_bits_fill(uint64_t seed, uint64_t k0, int64_t count, uint64_t* out) {
  for (int64_t i = 0; i < count; ++i) out[i] = bits_at(seed, k0 + static_cast<uint64_t>(i));
}
void orc_gaussian_fill(uint64_t seed, uint64_t k0, int64_t count, double* out) {
  for (int64_t i = 0; i < count; ++i) out[i] = gaussian_at(seed, k0 + static_cast<uint64_t>(i));
}
void orc_gaussian_matrix(int64_t rows, int64_t cols, uint64_t seed, double* out) {
  store(gaussian_matrix(rows, cols, seed), out);
}
void orc_stream_indices(uint64_t seed, uint64_t start, int64_t bound, int64_t count, int64_t* out) {
  Stream s{seed, start};
  for (int64_t i = 0; i < count; ++i) out[i] = s.next_index(bound);
}

int64_t orc_resolved_size(const cqr_sketch_cfg* cfg, int64_t m, int64_t n) { return resolved_size(*cfg, m, n); }

int orc_sample_rows_uniform(const double* a, int64_t m, int64_t n, int64_t lda, int64_t l, uint64_t seed,
                            int without_replacement, double* a1, int64_t* idx) {
  return guarded([&] {
    Mat A = from_strided(a, m, n, lda);
    Stream s{seed, 0};
    std::vector<Index> ix;
    Mat out = sample_rows_uniform(A, l, without_replacement != 0, s, &ix);
    store(out, a1);
    if (idx) std::memcpy(idx, ix.data(), sizeof(int64_t) * static_cast<size_t>(l));
  });
}

void orc_set_test_threads(int w) { g_test_threads.store(w < 1 ? 1 : w); }

int orc_sketch_gaussian(const double* a, int64_t m, int64_t n, int64_t lda, int64_t l, uint64_t seed,
                        double* a1) {
  return guarded([&] { store(sketch_gaussian(from_strided(a, m, n, lda), l, seed), a1); });
}

int orc_sketch_gaussian_shard(const double* a, int64_t m_local, int64_t m_global, int64_t row0, int64_t n,
                              int64_t l, uint64_t seed, double* a1) {
  return guarded([&] { store(sketch_gaussian(from_strided(a, m_local, n, n), l, seed, m_global, row0), a1); });
}

int orc_gram(const double* x, int64_t m, int64_t n, int64_t ldx, int workers, double* g) {
  return guarded([&] { store(gram(x, m, n, ldx, workers), g); });
}

// One leaf chain continued over `rows` rows from init (n x n, upper used; NULL = +0):
// the part of a 1024-row leaf (kernels.hpp:28-38) that one row block holds.
void orc_gram_chain(const double* x, int64_t ldx, int64_t rows, int64_t n, const double* init, double* out) {
  if (init)
    std::memcpy(out, init, sizeof(double) * static_cast<size_t>(n * n));
  else
    std::fill(out, out + n * n, 0.0);
  for (int64_t k = 0; k < rows; ++k) {
    const double* xr = x + k * ldx;
    for (int64_t i = 0; i < n; ++i)
      for (int64_t j = i; j < n; ++j) out[i * n + j] = std::fma(xr[i], xr[j], out[i * n + j]);
  }
}

void orc_gram_tree_combine(double* slots, int64_t count, int64_t len, double* out) {
  std::vector<double> s(slots, slots + count * len);
  gram_tree_combine(s, count, len);
  std::memcpy(out, s.data(), sizeof(double) * static_cast<size_t>(len));
}

// The streaming form used by the B200 Gram reduction: leaves are scanned left to
// right, equal-size subtrees merged (binary counter), and the remaining stack
// folded right-to-left, s0 + (s1 + (s2 + ...)). Identical to the level-by-level
// tree of kernels.hpp:42-57 (tests/test_oracle.py checks it bitwise).
void orc_gram_stack_combine(const double* slots, int64_t count, int64_t len, double* out) {
  for (int64_t e = 0; e < len; ++e) {
    double val[64];
    int64_t size[64];
    int top = 0;
    for (int64_t i = 0; i < count; ++i) {
      double v = slots[i * len + e];
      int64_t sz = 1;
      while (top > 0 && size[top - 1] == sz) {
        v = val[top - 1] + v;
        sz *= 2;
        --top;
      }
      val[top] = v;
      size[top] = sz;
      ++top;
    }
    double acc = val[top - 1];
    for (int t = top - 2; t >= 0; --t) acc = val[t] + acc;
    out[e] = acc;
  }
}

int orc_cholesky_upper(const double* g, int64_t n, double* r, int64_t* pivot) {
  return guarded([&] { store(cholesky_upper(from_strided(g, n, n, n)), r); }, pivot);
}

int orc_trisolve_inplace(double* x, int64_t m, int64_t n, int64_t ldx, const double* r, int workers,
                         int64_t* index) {
  return guarded([&] { trisolve_inplace(x, m, n, ldx, from_strided(r, n, n, n), workers); }, index);
}

int orc_qr_r_factor(const double* a1, int64_t l, int64_t n, double* r) {
  return guarded([&] { store(qr_r_factor(from_strided(a1, l, n, n)), r); });
}

int orc_lu_decompose(const double* a1, int64_t l, int64_t n, double* packed, int64_t* perm, int64_t* index) {
  return guarded(
      [&] {
        Lu f = lu_decompose(from_strided(a1, l, n, n));
        store(f.packed, packed);
        std::memcpy(perm, f.perm.data(), sizeof(int64_t) * static_cast<size_t>(l));
      },
      index);
}

int orc_lu_u_factor(const double* a1, int64_t l, int64_t n, double* u, int64_t* index) {
  return guarded([&] { store(lu_u_factor(from_strided(a1, l, n, n)), u); }, index);
}

int orc_householder_qr_thin(const double* a, int64_t m, int64_t n, double* q, double* r) {
  return guarded([&] {
    ThinQr t = householder_qr_thin(from_strided(a, m, n, n));
    store(t.q, q);
    store(t.r, r);
  });
}

int orc_svd_values(const double* a, int64_t rows, int64_t cols, double* sv) {
  return guarded([&] {
    std::vector<double> s = svd_values(from_strided(a, rows, cols, cols));
    std::memcpy(sv, s.data(), sizeof(double) * s.size());
  });
}

void orc_triangular_product(const double* left, const double* right, int64_t n, double* out) {
  store(triangular_product(from_strided(left, n, n, n), from_strided(right, n, n, n)), out);
}

int orc_factor(int method, const double* a, int64_t m, int64_t n, int64_t lda, const cqr_sketch_cfg* cfg,
               const cqr_options* opts, int workers, double* q, double* r, cqr_report* report) {
  return factor_common(method, a, m, n, lda, cfg, opts, workers, q, r, report, nullptr);
}

int orc_precond_factor(const double* a, int64_t m, int64_t n, int64_t lda, cqr_precond_fn fn, void* user,
                       const cqr_sketch_cfg* cfg, const cqr_options* opts, int workers, double* q, double* r,
                       cqr_report* report) {
  Precond pc = [fn, user](const Mat& a1) {
    Mat out(a1.cols, a1.cols);
    int64_t idx = -1;
    const int st = fn(user, a1.v.data(), a1.rows, a1.cols, out.v.data(), &idx);
    if (st == CQR_SINGULAR_TRIANGULAR) throw SingularTriangular{idx};
    if (st != CQR_OK) throw InvalidArgument{"preconditioner failed"};
    return out;
  };
  return factor_common(CQR_RQR, a, m, n, lda, cfg, opts, workers, q, r, report, &pc);
}

double orc_orthogonality_error(const double* q, int64_t m, int64_t n) {  // diagnostics.cpp:10-14
  Mat g = gram(q, m, n, n, g_test_threads.load());  // leaves over threads: bitwise the same G
  double s = 0.0;
  for (Index i = 0; i < n; ++i)
    for (Index j = 0; j < n; ++j) {
      const double v = g(i, j) - (i == j ? 1.0 : 0.0);
      s = std::fma(v, v, s);
    }
  return std::sqrt(s);
}

double orc_residual_error(const double* a, const double* q, const double* r, int64_t m, int64_t n) {
  // diagnostics.cpp:16-28 (panels of 4096 rows; ||A||_F over all entries)
  double na = 0.0;
  for (int64_t e = 0; e < m * n; ++e) na = std::fma(a[e], a[e], na);
  na = std::sqrt(na);
  if (na == 0.0) return std::numeric_limits<double>::quiet_NaN();
  constexpr int64_t kPanel = 4096;
  const int64_t panels = (m + kPanel - 1) / kPanel;
  std::vector<double> ps(static_cast<size_t>(panels));
  // panel sums in parallel (test-harness threads), accumulated in panel order: the same bits
  const int workers = static_cast<int>(std::max<int64_t>(1, std::min<int64_t>(g_test_threads.load(), panels)));
  run_on_workers(workers, [&](int w) {
    for (int64_t pi = panels * w / workers; pi < panels * (w + 1) / workers; ++pi) {
      const int64_t p0 = pi * kPanel, len = std::min(m - p0, kPanel);
      double s = 0.0;
      for (int64_t i = p0; i < p0 + len; ++i)
        for (int64_t j = 0; j < n; ++j) {
          double qr = 0.0;
          for (int64_t k = 0; k < n; ++k) qr = std::fma(q[i * n + k], r[k * n + j], qr);
          const double d = a[i * n + j] - qr;
          s = std::fma(d, d, s);
        }
      ps[static_cast<size_t>(pi)] = s;
    }
  });
  double acc = 0.0;
  for (const double s : ps) acc += s;
  return std::sqrt(acc) / na;
}

int orc_random_orthogonal(int64_t rows, int64_t cols, uint64_t seed, double* out) {  // matgen.cpp:12-19
  return guarded([&] {
    require(rows >= cols && cols >= 1, "random_orthogonal: need rows >= cols >= 1");
    HouseholderQr h = householder(gaussian_matrix(rows, cols, seed));
    store(householder_q(h), out);
  });
}

int orc_synthesize_sigma(int64_t m, int64_t n, const double* sigma, uint64_t seed, double* out) {
  // matgen.cpp:21-46: A = U diag(sigma) V^T, U = Q(gaussian(m,n,derive(seed,0))),
  // V = Q(gaussian(n,n,derive(seed,1))), built in 4096-row panels.
  return guarded([&] {
    require(m >= n && n >= 1, "synthesize: need m >= n >= 1");
    Mat v = householder_q(householder(gaussian_matrix(n, n, derive(seed, 1))));
    Mat svt(n, n);
    for (Index i = 0; i < n; ++i)
      for (Index j = 0; j < n; ++j) svt(i, j) = sigma[i] * v(j, i);
    Mat u = householder_q(householder(gaussian_matrix(m, n, derive(seed, 0))));
    for (Index i = 0; i < m; ++i) {
      const double* ur = u.row(i);
      for (Index j = 0; j < n; ++j) {
        double s = 0.0;
        for (Index k = 0; k < n; ++k) s = std::fma(ur[k], svt(k, j), s);
        out[i * n + j] = s;
      }
    }
  });
}

int orc_synthesize(int64_t m, int64_t n, double kappa, uint64_t seed, double* out) {
  if (!(kappa >= 1.0) || m < n || n < 1 || (n < 2 && kappa != 1.0)) return CQR_INVALID_ARGUMENT;
  std::vector<double> sigma(static_cast<size_t>(n));
  sigma[0] = 1.0;
  const double lk = std::log(kappa);
  for (int64_t i = 1; i < n; ++i)
    sigma[static_cast<size_t>(i)] = std::exp(-lk * static_cast<double>(i) / static_cast<double>(n - 1));
  return orc_synthesize_sigma(m, n, sigma.data(), seed, out);
}

int orc_embedded_identity(int64_t m, int64_t n, uint64_t seed, double* out) {  // matgen.cpp:48-54
  if (m < n || n < 1) return CQR_INVALID_ARGUMENT;
  std::fill(out, out + m * n, 0.0);
  for (int64_t i = 0; i < n; ++i) out[i * n + i] = 1.0;
  if (m > n) {
    Mat g = gaussian_matrix(m - n, n, seed);
    for (int64_t i = 0; i < (m - n) * n; ++i) out[n * n + i] = 1e-8 * g.v[static_cast<size_t>(i)];
  }
  return CQR_OK;
}

int64_t orc_block_offset(int64_t m, int p, int b) { return block_offset(m, p, b); }

void orc_comm_model(int method, int p, int64_t n, int64_t l, int* rmin, int* rmax, double* vmin, double* vmax) {
  comm_model(method, p, n, l, rmin, rmax, vmin, vmax);
}

}  // extern "C"
