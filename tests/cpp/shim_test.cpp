// Exercises include/cholqr_b200.hpp the way the reference's own doctest cases
// exercise cholqr.hpp (test_cholqr.cpp:26-33, :52-55, :113-121, :258-262).
// Built and run by tests/test_cpp_shim.py (GPU).
#include <algorithm>
#include <cmath>
#include <cstdio>
#include <random>

#include "cholqr_b200.hpp"

using namespace cholqr::b200;

static int fails = 0;
#define CHECK(c)                                                   \
  do {                                                             \
    if (!(c)) {                                                    \
      std::printf("CHECK failed line %d: %s\n", __LINE__, #c);     \
      ++fails;                                                     \
    }                                                              \
  } while (0)

int main() {
  const Index m = 4000, n = 24;
  std::mt19937_64 g(7);
  std::normal_distribution<double> nd;
  Matrix a(m, n);
  for (auto& v : a.data) v = nd(g);
  const QRFactorization f = cholesky_qr2(a);
  // contract: positive diagonal, zero strict lower part, small residual
  double res = 0, na = 0, lower = 0;
  bool pos = true;
  for (Index i = 0; i < n; ++i) {
    pos = pos && f.r(i, i) > 0;
    for (Index j = 0; j < i; ++j) lower += std::abs(f.r(i, j));
  }
  for (Index i = 0; i < m; ++i)
    for (Index j = 0; j < n; ++j) {
      double s = 0;
      for (Index k = 0; k < n; ++k) s += f.q(i, k) * f.r(k, j);
      res += (a(i, j) - s) * (a(i, j) - s);
      na += a(i, j) * a(i, j);
    }
  CHECK(pos);
  CHECK(lower == 0.0);
  CHECK(std::sqrt(res / na) <= 1e-14);
  // identity preconditioner == cholesky_qr bitwise (test_cholqr.cpp:113-121)
  SketchConfig cfg;
  cfg.size = 2 * n;
  cfg.seed = 13;
  const QRFactorization base = cholesky_qr(a);
  const QRFactorization pc = precond_cholesky_qr(
      a, [](const Matrix& a1) {
        Matrix e(a1.cols, a1.cols);
        for (Index i = 0; i < a1.cols; ++i) e(i, i) = 1.0;
        return e;
      },
      cfg);
  CHECK(pc.q.data == base.q.data && pc.r.data == base.r.data);
  // rQR with the Gaussian sketch; report carries the stages
  cfg.strategy = Strategy::Gaussian;
  const QRFactorization fr = rqr_cholesky_qr(a, cfg);
  CHECK(!fr.report.stages.empty() && fr.report.stages.front().stage == Stage::Sketch);
  // breakdown raises CholeskyBreakdown (test_cholqr.cpp:52-55): rank-deficient input
  Matrix d(100, 3);
  for (Index i = 0; i < 100; ++i) {
    d(i, 0) = nd(g);
    d(i, 1) = d(i, 0);
    d(i, 2) = nd(g);
  }
  bool threw = false;
  try {
    (void)cholesky_qr(d);
  } catch (const CholeskyBreakdown& e) {
    threw = e.pivot_index == 1;
  }
  CHECK(threw);
  // non-finite input -> std::invalid_argument (test_cholqr.cpp:258-262)
  Matrix bad(8, 2);
  for (auto& v : bad.data) v = 1.0;
  bad(3, 1) = std::nan("");
  threw = false;
  try {
    (void)cholesky_qr(bad);
  } catch (const std::invalid_argument&) {
    threw = true;
  }
  CHECK(threw);
  // kernels
  Matrix e3(3, 3);
  for (Index i = 0; i < 3; ++i) e3(i, i) = 1.0;
  CHECK(kernels::gram(e3).data == e3.data);
  Matrix g2(2, 2);
  g2.data = {4, 2, 2, 2};
  CHECK((kernels::cholesky_upper(g2).data == std::vector<double>{2, 1, 0, 1}));
  Matrix lu(2, 2);
  lu.data = {2, 1, 4, 3};
  CHECK((kernels::lu_u_factor(lu).data == std::vector<double>{4, 3, 0, -0.5}));
  // the RSVD caller's orthogonalizer: Q of Y equals the r_less factorization with the derived seed
  {
    Matrix y(400, 6);
    for (Index i = 0; i < y.rows; ++i)
      for (Index j = 0; j < y.cols; ++j) y(i, j) = std::sin(0.37 * (double)(i * 7 + j * 13 + 1)) + (i == j ? 3.0 : 0.0);
    Matrix q1 = orthonormalize(y, Orth::RqrCholeskyQr, 99, 2);
    SketchConfig cfg;
    cfg.seed = derive(99, 0xA110 + 2);
    Options o;
    o.r_less = true;
    CHECK(q1.data == rqr_cholesky_qr(y, cfg, o).q.data);
    CHECK(orthonormalize(y, Orth::CholeskyQr2, 99, 0).data == cholesky_qr2(y, o).q.data);
    // HouseholderQr (apps.cpp:171-172) is householder_qr_thin(y).q on the device: orthonormal columns
    Matrix qh = orthonormalize(y, Orth::HouseholderQr, 99, 0);
    double orth = 0.0;
    for (Index i = 0; i < qh.cols; ++i)
      for (Index j = 0; j < qh.cols; ++j) {
        double s = 0.0;
        for (Index k = 0; k < qh.rows; ++k) s += qh(k, i) * qh(k, j);
        orth = std::max(orth, std::abs(s - (i == j ? 1.0 : 0.0)));
      }
    CHECK(orth < 1e-13);
    CHECK(kernels::householder_qr_thin(y).q.data == qh.data);
  }
  std::printf("shim_test %s (%d failures)\n", fails ? "FAILED" : "ok", fails);
  return fails ? 1 : 0;
}
