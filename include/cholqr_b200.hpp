// cholqr_b200.hpp — C++ host API over the C-ABI (include/cqr.h), mirroring the
// reference's public C++ interface so a caller of
// /root/reference/proj/include/cholqr/cholqr.hpp can switch by changing the
// namespace and the matrix type:
//
//   reference (Eigen, CPU)                         this header (B200)
//   cholqr::cholesky_qr(a, opts)        :82   ->   cholqr::b200::cholesky_qr(a, opts)
//   cholqr::cholesky_qr2(a, opts)       :85   ->   cholqr::b200::cholesky_qr2(a, opts)
//   cholqr::shifted_cholesky_qr3(...)   :89   ->   cholqr::b200::shifted_cholesky_qr3(...)
//   cholqr::precond_cholesky_qr(...)    :100  ->   cholqr::b200::precond_cholesky_qr(...)
//   cholqr::rqr_cholesky_qr(a, cfg, o)  :104  ->   cholqr::b200::rqr_cholesky_qr(a, cfg, o)
//   cholqr::rlu_cholesky_qr(a, cfg, o)  :108  ->   cholqr::b200::rlu_cholesky_qr(a, cfg, o)
//   cholqr::parexec::run_parallel       parexec.hpp:89 -> cholqr::b200::run_parallel
//   cholqr::kernels::{gram, cholesky_upper, right_trisolve_in_place, qr_r_factor,
//                     lu_u_factor}      kernels.hpp   -> cholqr::b200::kernels::...
//
// Matrices are plain row-major views (MatrixView / Matrix below) instead of
// Eigen::Ref<const RowMajor>; the same failures raise the same exception
// classes (CholeskyBreakdown{pivot_index}, SingularTriangular{index},
// std::invalid_argument; errors.hpp:18-33, 84-93). Header-only; link libcqr.so.
#pragma once

#include <cstdint>
#include <functional>
#include <optional>
#include <stdexcept>
#include <string>
#include <vector>

#include "cqr.h"

namespace cholqr::b200 {

using Index = std::int64_t;

class Error : public std::runtime_error {
 public:
  explicit Error(const std::string& w) : std::runtime_error(w) {}
};
class CholeskyBreakdown : public Error {
 public:
  explicit CholeskyBreakdown(Index p) : Error("cholesky breakdown at pivot " + std::to_string(p)), pivot_index(p) {}
  Index pivot_index;
};
class SingularTriangular : public Error {
 public:
  explicit SingularTriangular(Index i)
      : Error("singular triangular factor, zero diagonal at " + std::to_string(i)), index(i) {}
  Index index;
};
class DeviceError : public Error {
 public:
  using Error::Error;
};

struct Matrix {  // owning, row-major
  Index rows = 0, cols = 0;
  std::vector<double> data;
  Matrix() = default;
  Matrix(Index r, Index c) : rows(r), cols(c), data(static_cast<size_t>(r * c), 0.0) {}
  double& operator()(Index i, Index j) { return data[static_cast<size_t>(i * cols + j)]; }
  double operator()(Index i, Index j) const { return data[static_cast<size_t>(i * cols + j)]; }
  Index size() const { return rows * cols; }
};

struct MatrixView {  // non-owning row-major view with a row stride (Eigen::Ref with outer stride)
  const double* data;
  Index rows, cols, stride;
  MatrixView(const Matrix& m) : data(m.data.data()), rows(m.rows), cols(m.cols), stride(m.cols) {}  // NOLINT
  MatrixView(const double* d, Index r, Index c, Index s) : data(d), rows(r), cols(c), stride(s) {}
};

enum class Stage { Sketch, Precondition, Gram, Cholesky, Trisolve, Recover, Householder };  // cholqr.hpp:12-20
enum class Method { HouseholderQr, CholeskyQr, CholeskyQr2, ShiftedCholeskyQr3, RluCholeskyQr, RqrCholeskyQr,
                    RqrCholeskyQrGaussian };  // types.hpp:35-43
enum class Strategy { Uniform, Leverage, Gaussian };  // sketch.hpp:14

struct SketchConfig {  // sketch.hpp:16-33
  Strategy strategy = Strategy::Uniform;
  Index size = 0;
  double rate = 2.0;
  std::uint64_t seed = 0;
  int max_retries = 2;
  double retry_growth = 2.0;
  bool without_replacement = false;
  Index resolved_size(Index m, Index n) const {
    cqr_sketch_cfg c = to_c();
    return cqr_resolved_size(&c, m, n);
  }
  cqr_sketch_cfg to_c() const {
    cqr_sketch_cfg c{};
    c.strategy = static_cast<int32_t>(strategy);
    c.size = size;
    c.rate = rate;
    c.seed = seed;
    c.max_retries = max_retries;
    c.retry_growth = retry_growth;
    c.without_replacement = without_replacement ? 1 : 0;
    return c;
  }
};

struct ShiftMode {  // cholqr.hpp:48-59
  enum class Kind { TheoryFormula, Fixed };
  Kind kind = Kind::TheoryFormula;
  double value = 0.0;
  static ShiftMode theory() { return {Kind::TheoryFormula, 0.0}; }
  static ShiftMode fixed(double eps) { return {Kind::Fixed, eps}; }
};

struct Options {  // cholqr.hpp:61-70
  bool diagnostics = false;
  bool r_less = false;
  int workers = 1;
};

struct MethodConfig {  // cholqr.hpp:73-78
  SketchConfig sketch{};
  ShiftMode shift = ShiftMode::theory();
  bool diagnostics = false;
  bool r_less = false;
};

struct StageInfo {  // cholqr.hpp:25-34
  Stage stage;
  std::optional<double> cond_x;
  std::optional<double> shift;
  int retries = 0;
};
struct StageReport {
  std::vector<StageInfo> stages;
  bool r_less = false;
};
struct QRFactorization {  // cholqr.hpp:41-45
  Matrix q;
  Matrix r;  // empty in r_less mode
  StageReport report;
};
struct TimingBreakdown {  // parexec.hpp:73-79
  double stage_ms[CQR_STAGE_COUNT] = {0};
  double total_ms = 0.0;
  int comm_rounds = 0;
  double comm_volume = 0.0;
};
struct ParallelRun {
  QRFactorization factorization;
  TimingBreakdown timing;
};

using Preconditioner = std::function<Matrix(const Matrix& a1)>;  // cholqr.hpp:94

namespace detail {

class Context {
 public:
  static Context& get() {
    thread_local Context ctx;
    return ctx;
  }
  cqr_ctx* h = nullptr;
  ~Context() {
    if (h) cqr_destroy(h);
  }

 private:
  Context() {
    if (cqr_create(&h, 0) != CQR_OK) throw DeviceError("cqr_create failed (no B200 / libcqr.so?)");
  }
};

inline void raise(int st, Index index) {
  switch (st) {
    case CQR_OK: return;
    case CQR_CHOLESKY_BREAKDOWN: throw CholeskyBreakdown(index);
    case CQR_SINGULAR_TRIANGULAR: throw SingularTriangular(index);
    case CQR_INVALID_ARGUMENT: throw std::invalid_argument(cqr_last_error(Context::get().h));
    case CQR_UNSUPPORTED: throw std::invalid_argument(cqr_last_error(Context::get().h));
    default: throw DeviceError(std::string("cqr status ") + std::to_string(st) + ": " + cqr_last_error(Context::get().h));
  }
}

inline cqr_options options(bool diag, bool r_less, ShiftMode sh, int workers) {
  cqr_options o{};
  o.diagnostics = diag ? 1 : 0;
  o.r_less = r_less ? 1 : 0;
  o.shift_kind = sh.kind == ShiftMode::Kind::Fixed ? CQR_SHIFT_FIXED : CQR_SHIFT_THEORY;
  o.shift_value = sh.value;
  o.workers = workers;
  return o;
}

inline QRFactorization to_fact(Matrix q, Matrix r, const cqr_report& rep) {
  QRFactorization f;
  f.q = std::move(q);
  if (!rep.r_less) f.r = std::move(r);
  f.report.r_less = rep.r_less != 0;
  for (int i = 0; i < rep.n_stages; ++i) {
    const cqr_stage_info& s = rep.stages[i];
    StageInfo si{static_cast<Stage>(s.stage), std::nullopt, std::nullopt, s.retries};
    if (s.has_cond_x) si.cond_x = s.cond_x;
    if (s.has_shift) si.shift = s.shift;
    f.report.stages.push_back(si);
  }
  return f;
}

inline QRFactorization run(Method m, const MatrixView& a, const SketchConfig& cfg, const cqr_options& o,
                           cqr_report* rep_out = nullptr) {
  Matrix q(a.rows, a.cols), r(a.cols, a.cols);
  cqr_report rep{};
  const cqr_sketch_cfg c = cfg.to_c();
  const int st = cqr_factor(Context::get().h, static_cast<int>(m), a.data, a.rows, a.cols, a.stride, &c, &o,
                            q.data.data(), a.cols, r.data.data(), a.cols, &rep);
  raise(st, rep.index);
  if (rep_out) *rep_out = rep;
  return to_fact(std::move(q), std::move(r), rep);
}

}  // namespace detail

inline QRFactorization cholesky_qr(const MatrixView& a, const Options& o = {}) {
  return detail::run(Method::CholeskyQr, a, {}, detail::options(o.diagnostics, o.r_less, {}, o.workers));
}
inline QRFactorization cholesky_qr2(const MatrixView& a, const Options& o = {}) {
  return detail::run(Method::CholeskyQr2, a, {}, detail::options(o.diagnostics, o.r_less, {}, o.workers));
}
inline QRFactorization shifted_cholesky_qr3(const MatrixView& a, ShiftMode shift, const Options& o = {}) {
  return detail::run(Method::ShiftedCholeskyQr3, a, {}, detail::options(o.diagnostics, o.r_less, shift, o.workers));
}
inline QRFactorization shifted_cholesky_qr3(const MatrixView& a, const Options& o = {}) {
  return shifted_cholesky_qr3(a, ShiftMode::theory(), o);
}
inline QRFactorization rqr_cholesky_qr(const MatrixView& a, const SketchConfig& cfg, const Options& o = {}) {
  return detail::run(Method::RqrCholeskyQr, a, cfg, detail::options(o.diagnostics, o.r_less, {}, o.workers));
}
inline QRFactorization rlu_cholesky_qr(const MatrixView& a, const SketchConfig& cfg, const Options& o = {}) {
  return detail::run(Method::RluCholeskyQr, a, cfg, detail::options(o.diagnostics, o.r_less, {}, o.workers));
}

inline QRFactorization precond_cholesky_qr(const MatrixView& a, const Preconditioner& precond,
                                           const SketchConfig& cfg, const Options& o = {}) {
  struct Thunk {
    const Preconditioner* p;
    static int call(void* user, const double* a1, int64_t l, int64_t n, double* r, int64_t* index) {
      Matrix m(l, n);
      std::copy(a1, a1 + l * n, m.data.begin());
      try {
        const Matrix out = (*static_cast<Thunk*>(user)->p)(m);
        std::copy(out.data.begin(), out.data.end(), r);
      } catch (const SingularTriangular& e) {
        *index = e.index;
        return CQR_SINGULAR_TRIANGULAR;
      }
      return CQR_OK;
    }
  } thunk{&precond};
  Matrix q(a.rows, a.cols), r(a.cols, a.cols);
  cqr_report rep{};
  const cqr_sketch_cfg c = cfg.to_c();
  const cqr_options opt = detail::options(o.diagnostics, o.r_less, {}, o.workers);
  const int st = cqr_precond_factor(detail::Context::get().h, a.data, a.rows, a.cols, a.stride, &Thunk::call,
                                    &thunk, &c, &opt, q.data.data(), a.cols, r.data.data(), a.cols, &rep);
  detail::raise(st, rep.index);
  return detail::to_fact(std::move(q), std::move(r), rep);
}

inline ParallelRun run_parallel(Method m, const MatrixView& a, int p, const MethodConfig& cfg = {}) {
  if (p < 1 || p > a.rows) throw std::invalid_argument("worker count must be in [1, m]");
  cqr_report rep{};
  ParallelRun run;
  run.factorization =
      detail::run(m, a, cfg.sketch, detail::options(cfg.diagnostics, cfg.r_less, cfg.shift, p), &rep);
  for (int s = 0; s < CQR_STAGE_COUNT; ++s) run.timing.stage_ms[s] = rep.stage_ms[s];
  run.timing.total_ms = rep.total_ms;
  run.timing.comm_rounds = rep.comm_rounds;
  run.timing.comm_volume = rep.comm_volume;
  return run;
}

// rng::derive (rng.hpp:36-38)
inline uint64_t mix64(uint64_t z) {
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}
inline uint64_t derive(uint64_t seed, uint64_t salt) { return mix64(seed ^ mix64(salt + 0x51ED270B8A5EC473ull)); }

// The RSVD caller's orthogonalizer (apps.hpp:48, apps.cpp:166-196): Q only (r_less);
// rQR draws a fresh uniform sketch per call, seed derive(seed, 0xA110 + call_counter).
enum class Orth { HouseholderQr, RqrCholeskyQr, CholeskyQr2 };
inline Matrix orthonormalize(const MatrixView& y, Orth orth, uint64_t seed, int call_counter, int workers = 1) {
  Options o;
  o.r_less = true;
  o.workers = workers;
  switch (orth) {
    case Orth::RqrCholeskyQr: {
      SketchConfig cfg;
      cfg.rate = 2.0;
      cfg.seed = derive(seed, 0xA110 + static_cast<uint64_t>(call_counter));
      return rqr_cholesky_qr(y, cfg, o).q;
    }
    case Orth::CholeskyQr2:
      return cholesky_qr2(y, o).q;
    case Orth::HouseholderQr:  // apps.cpp:171-172: householder_qr_thin(y).q, on the device
      return detail::run(Method::HouseholderQr, y, {}, detail::options(false, true, {}, workers)).q;
    default:
      throw std::invalid_argument("orthonormalize: unknown orthogonalizer");
  }
}

namespace kernels {  // kernels.hpp

inline Matrix gram(const MatrixView& x) {
  if (x.rows < x.cols) throw std::invalid_argument("gram: matrix must have rows >= cols");
  Matrix g(x.cols, x.cols);
  detail::raise(cqr_gram(detail::Context::get().h, x.data, x.rows, x.cols, x.stride, g.data.data()), -1);
  return g;
}
inline Matrix cholesky_upper(const Matrix& g) {
  if (g.rows != g.cols) throw std::invalid_argument("cholesky_upper: matrix must be square");
  Matrix r(g.rows, g.rows);
  int64_t piv = -1;
  detail::raise(cqr_cholesky_upper(detail::Context::get().h, g.data.data(), g.rows, r.data.data(), &piv), piv);
  return r;
}
inline void right_trisolve_in_place(Matrix& x, const Matrix& r) {
  if (r.rows != r.cols || x.cols != r.rows) throw std::invalid_argument("right_trisolve: dimension mismatch");
  int64_t idx = -1;
  detail::raise(cqr_trisolve_inplace(detail::Context::get().h, x.data.data(), x.rows, x.cols, x.cols, r.data.data(),
                                     &idx),
                idx);
}
inline Matrix right_trisolve(const Matrix& a, const Matrix& r) {
  Matrix x = a;
  right_trisolve_in_place(x, r);
  return x;
}
struct ThinQr {  // kernels.hpp:186-189
  Matrix q;
  Matrix r;
};
// kernels.hpp:192-209: thin Householder QR with the R diagonal non-negative (Q adjusted), on the device
inline ThinQr householder_qr_thin(const MatrixView& a) {
  if (a.rows < a.cols) throw std::invalid_argument("householder_qr_thin: need rows >= cols");
  QRFactorization f = detail::run(Method::HouseholderQr, a, {}, detail::options(false, false, {}, 1));
  return ThinQr{std::move(f.q), std::move(f.r)};
}
inline Matrix qr_r_factor(const Matrix& a1) {
  if (a1.rows < a1.cols) throw std::invalid_argument("qr_r_factor: need rows >= cols");
  Matrix r(a1.cols, a1.cols);
  detail::raise(cqr_qr_r_factor(detail::Context::get().h, a1.data.data(), a1.rows, a1.cols, r.data.data()), -1);
  return r;
}
inline Matrix lu_u_factor(const Matrix& a1) {
  if (a1.rows < a1.cols) throw std::invalid_argument("lu_decompose: need rows >= cols");
  Matrix u(a1.cols, a1.cols);
  int64_t idx = -1;
  detail::raise(cqr_lu_u_factor(detail::Context::get().h, a1.data.data(), a1.rows, a1.cols, u.data.data(), &idx),
                idx);
  return u;
}

}  // namespace kernels
}  // namespace cholqr::b200
