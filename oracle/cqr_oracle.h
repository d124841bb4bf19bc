/*
 * cqr_oracle.h — CPU restatement of the reference's rQR/rLU-CholeskyQR hot
 * path, used ONLY as test infrastructure: the parity checker of tests/, the
 * checker of __graft_entry__.smoke() and the cpu_baseline / --impl reference
 * leg of bench.py. Nothing in the product (paper_2111_11148_b200/, include/)
 * links or calls it.
 *
 * The reference (/root/reference/proj, C++20 + Eigen3) cannot be compiled in
 * this image (Eigen, doctest and CLI11 are absent), so this is
 * a line-by-line restatement of its algorithms without Eigen. Wherever the
 * reference delegates an inner reduction to Eigen (rankUpdate, dot,
 * squaredNorm, GEMM), whose summation order the reference does not pin, the
 * oracle fixes one order and documents it next to the function ("fixed
 * order"). The B200 kernels follow the same fixed orders, which is what makes
 * the Gram, Cholesky, trisolve, LU and recover steps bitwise comparable.
 *
 * Pinning: tests/test_oracle.py replays every known-answer and property
 * assertion of proj/tests/test_{kernels,sketch,cholqr,parexec}.cpp against
 * this library, plus numpy/LAPACK cross-checks and committed golden RNG
 * vectors (tests/golden/). There are no reference-produced golden vectors
 * (the reference cannot run here), so parity is pinned by those tests.
 */
#ifndef CQR_ORACLE_H_
#define CQR_ORACLE_H_

#include <stdint.h>

#include "../include/cqr.h"

#ifdef __cplusplus
extern "C" {
#endif

/* rng.hpp:22-92 */
uint64_t orc_mix64(uint64_t z);
uint64_t orc_bits_at(uint64_t seed, uint64_t k);
uint64_t orc_derive(uint64_t seed, uint64_t salt);
double orc_unit_at(uint64_t seed, uint64_t k);
double orc_gaussian_at(uint64_t seed, uint64_t k);
void orc_bits_fill(uint64_t seed, uint64_t k0, int64_t count, uint64_t* out);
void orc_gaussian_fill(uint64_t seed, uint64_t k0, int64_t count, double* out);
void orc_gaussian_matrix(int64_t rows, int64_t cols, uint64_t seed, double* out);
/* Stream(seed, start).next_index(bound) repeated `count` times (rng.hpp:69-71). */
void orc_stream_indices(uint64_t seed, uint64_t start, int64_t bound, int64_t count, int64_t* out);

/* sketch.cpp */
int64_t orc_resolved_size(const cqr_sketch_cfg* cfg, int64_t m, int64_t n);
int orc_sample_rows_uniform(const double* a, int64_t m, int64_t n, int64_t lda, int64_t l,
                            uint64_t seed, int without_replacement, double* a1, int64_t* idx);
/* test-harness knob: split the Gaussian sketch's rows and the diagnostics over w threads
   (bitwise the same results) */
void orc_set_test_threads(int w);
int orc_sketch_gaussian(const double* a, int64_t m, int64_t n, int64_t lda, int64_t l,
                        uint64_t seed, double* a1);
/* the same for rows [row0, row0+m_local) of an m_global-row matrix (global counters) */
int orc_sketch_gaussian_shard(const double* a, int64_t m_local, int64_t m_global, int64_t row0, int64_t n,
                              int64_t l, uint64_t seed, double* a1);

/* kernels.hpp (status codes as cqr_status) */
int orc_gram(const double* x, int64_t m, int64_t n, int64_t ldx, int workers, double* g);
/* Leaf partials + tree, exposed so the tree rule can be tested alone. */
void orc_gram_tree_combine(double* slots, int64_t count, int64_t len, double* out);
void orc_gram_chain(const double* x, int64_t ldx, int64_t rows, int64_t n, const double* init, double* out);
void orc_gram_stack_combine(const double* slots, int64_t count, int64_t len, double* out);
int orc_cholesky_upper(const double* g, int64_t n, double* r, int64_t* pivot);
int orc_trisolve_inplace(double* x, int64_t m, int64_t n, int64_t ldx, const double* r,
                         int workers, int64_t* index);
int orc_qr_r_factor(const double* a1, int64_t l, int64_t n, double* r);
int orc_lu_decompose(const double* a1, int64_t l, int64_t n, double* packed, int64_t* perm,
                     int64_t* index);
int orc_lu_u_factor(const double* a1, int64_t l, int64_t n, double* u, int64_t* index);
int orc_householder_qr_thin(const double* a, int64_t m, int64_t n, double* q, double* r);
/* returns 0, or 8 (NoConvergence) */
int orc_svd_values(const double* a, int64_t rows, int64_t cols, double* sv);
/* engine.cpp:103-107 */
void orc_triangular_product(const double* left, const double* right, int64_t n, double* out);

/* engine.cpp:221-305 / parexec::run_parallel; workers = p. */
int orc_factor(int method, const double* a, int64_t m, int64_t n, int64_t lda,
               const cqr_sketch_cfg* cfg, const cqr_options* opts, int workers, double* q,
               double* r, cqr_report* report);
int orc_precond_factor(const double* a, int64_t m, int64_t n, int64_t lda, cqr_precond_fn fn,
                       void* user, const cqr_sketch_cfg* cfg, const cqr_options* opts,
                       int workers, double* q, double* r, cqr_report* report);

/* diagnostics.cpp:10-28 */
double orc_orthogonality_error(const double* q, int64_t m, int64_t n);
double orc_residual_error(const double* a, const double* q, const double* r, int64_t m, int64_t n);

/* matgen.cpp:12-54; sigma may be NULL (geometric 1..1/kappa) */
int orc_random_orthogonal(int64_t rows, int64_t cols, uint64_t seed, double* out);
int orc_synthesize(int64_t m, int64_t n, double kappa, uint64_t seed, double* out);
int orc_synthesize_sigma(int64_t m, int64_t n, const double* sigma, uint64_t seed, double* out);
int orc_embedded_identity(int64_t m, int64_t n, uint64_t seed, double* out);

/* parexec.cpp:9-62 */
int64_t orc_block_offset(int64_t m, int p, int b);
void orc_comm_model(int method, int p, int64_t n, int64_t l, int* rmin, int* rmax, double* vmin,
                    double* vmax);

#ifdef __cplusplus
}
#endif

#endif
