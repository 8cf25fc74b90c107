/* TEST INFRASTRUCTURE ONLY — the CPU checker, never the product.
 *
 * Plain-C restatement of the reference PARS predictor hot path
 * (/root/reference/proj/src/{features,scorer,pairs,train,scheduler,metrics}.cpp
 * and include/pars/{rng,pairs}.hpp). Every function cites the reference
 * file:line it restates. Only tests/, __graft_entry__.smoke() and bench.py's
 * cpu_baseline / --impl reference legs may load liboracle.so.
 *
 * Parity pinning: tests/test_oracle.py checks every function here against
 * (a) the golden fixtures in tests/golden/ produced by running the reference
 * library itself (oracle/_ref, built from /root/reference by oracle/Makefile,
 * fixtures written by tests/golden/make_golden.py) and (b) the golden values
 * of SURVEY.md Appendix B. Build flags: -ffp-contract=off (the reference
 * objects are compiled without FMA).
 */
#ifndef PARS_ORACLE_H
#define PARS_ORACLE_H
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* mt19937_64 + the reference's samplers (rng.hpp:10-75). */
typedef struct {
  uint64_t mt[312];
  int mti;
} po_rng;
void po_rng_seed(po_rng* r, uint64_t seed);
uint64_t po_rng_u64(po_rng* r);
uint64_t po_rng_below(po_rng* r, uint64_t n);
uint64_t po_splitmix64(uint64_t x);
uint64_t po_derive_seed(uint64_t seed, uint64_t stream);

/* Same layout as pars_extractor (include/pars_cuda.h). */
typedef struct {
  int32_t kind; /* 0 hashed text, 1 precomputed embedding */
  uint32_t dim;
  int32_t norm; /* 0 none, 1 l2 */
  int32_t n_word;
  int32_t n_char;
  int32_t word[8];
  int32_t chr[8];
} po_extractor;

const char* po_last_error(void);

/* extract_features (features.cpp:62-122). Returns nnz (entries written up to
 * cap) or -1 on error. */
int64_t po_extract(const po_extractor* ex, const char* text, int64_t len,
                   const double* emb, int64_t emb_len, uint32_t* idx,
                   double* val, int64_t cap);
/* extract_all over a text arena: row_ptr[n+1]; returns total nnz or -1. */
int64_t po_extract_all(const po_extractor* ex, const char* text,
                       const int64_t* offs, int64_t n, int64_t* row_ptr,
                       uint32_t* idx, double* val, int64_t cap);
/* LinearScorer::score over a text arena (scorer.cpp:9-42, features.hpp:31-35).
 * nthreads > 1 splits prompts across OpenMP threads (each prompt serial). */
int po_score_batch(const po_extractor* ex, const char* text,
                   const int64_t* offs, int64_t n, const double* w,
                   double bias, double* out, int nthreads);
/* Dense embedding rows (features.cpp:67-76 + score). */
int po_score_dense(const po_extractor* ex, const double* X, int64_t n,
                   const double* w, double bias, double* out);

/* pairs.hpp:21-31 */
double po_rel_diff(int64_t a, int64_t b);
double po_margin_loss(double sa, double sb, int y, double margin);
/* dmin[m] = min{d >= 1 : !(rel_diff(m, m-d) < delta)} (or INT32_MAX). */
void po_dmin_table(double delta, int64_t max_len, int32_t* table);
/* build_pairs (pairs.cpp:8-36). Returns count or -1 (error message set). */
int64_t po_build_pairs(const int64_t* lens, int64_t n, double delta,
                       uint64_t max_pairs, uint64_t seed, uint32_t* a,
                       uint32_t* b, int32_t* y, double* rel);

/* train(), pairwise objective (train.cpp:122-166, :34-44, :141-151,
 * :212-216) over precomputed CSR features. loss_trace has `epochs` slots. */
int po_train_pairwise(const int64_t* row_ptr, const uint32_t* idx,
                      const double* val, const int64_t* lens, int64_t n,
                      uint32_t dim, double delta, double margin, int epochs,
                      int batch, double lr, uint64_t seed,
                      uint64_t pairs_per_epoch, double* w_out,
                      double* bias_out, double* loss_trace);
/* One SGD epoch over explicit pairs (the inner loop of train, :154-166). */
int po_sgd_epoch(const int64_t* row_ptr, const uint32_t* idx,
                 const double* val, uint32_t dim, const uint32_t* a,
                 const uint32_t* b, const int32_t* y, int64_t npairs,
                 int batch, double lr, double margin, double* w,
                 double bias, double* epoch_loss, uint64_t* active);

/* All-pairs variant over unordered i<j: Eq. 1 mask,
 * hinge, integer coefficient c (grad = X^T c), loss sum. O(n^2). */
int po_allpairs(const double* s, const int64_t* lens, int64_t n,
                double delta, double margin, int32_t* coeff,
                uint64_t* kept, uint64_t* active, double* loss_sum,
                int nthreads);
/* grad[d] = sum_i c_i * x_i[d] in row order (fp64, sequential). */
void po_xt_c(const int64_t* row_ptr, const uint32_t* idx, const double* val,
             int64_t n, const int32_t* coeff, uint32_t dim, double* grad);

/* select_batch total order (scheduler.cpp:33-60) over all n requests. ids:
 * arena + offsets (byte strings). Returns -1 if some arrival > now. */
int po_select_order(int64_t n, const double* arrival, const char* ids,
                    const int64_t* id_offs, const double* score,
                    const uint8_t* boosted, double now, int64_t* order);

/* kendall_tau_b_serial (metrics.cpp:66-86, finish_tau :13-32).
 * counts = {n_c, n_d, n0, n1, n2}; returns -1 on degenerate input. */
int po_kendall(const double* x, const double* y, int64_t n, uint64_t* counts,
               double* tau, int nthreads);

#ifdef __cplusplus
}
#endif
#endif
