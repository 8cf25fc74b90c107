/*
 * pars_cuda.h — C ABI of the B200-native PARS predictor hot path
 * (libpars_cuda.so, sm_100a).
 *
 * This is the drop-in boundary underneath the reference's C++ predictor and
 * scheduler API (/root/reference/proj/include/pars/ headers). The C++ host shim
 * (paper_2510_03243_b200/host/ sources, compiled against those unmodified
 * headers) and the Python bindings (paper_2510_03243_b200/_lib.py) both call
 * only the functions below. Plain pointers and sizes, no C++ or torch types.
 *
 * Conventions
 *   - Every function returns PARS_OK (0) or a negative PARS_ERR_* code; the
 *     message (verbatim the reference's pars::Error text where one exists) is
 *     available from pars_last_error() on the calling thread.
 *   - pars_* functions take HOST buffers (caller-owned) and do the
 *     host<->device copies themselves; pars_dev_* functions take DEVICE
 *     pointers plus a cudaStream_t (passed as void*, NULL = the ctx stream)
 *     and are asynchronous on that stream.
 *   - A pars_ctx binds one CUDA device and owns its scratch memory; calls on
 *     one ctx are serialised by an internal mutex (the reference's Scorer is
 *     called concurrently from OpenMP threads, scorer.cpp:13-21).
 *   - There is no CPU fallback: without a usable sm_100 device every
 *     compute entry point fails with PARS_ERR_CUDA.
 */
#ifndef PARS_CUDA_H
#define PARS_CUDA_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define PARS_OK 0
#define PARS_ERR_INVALID (-1)     /* contract violation (reference: pars::Error) */
#define PARS_ERR_CUDA (-2)        /* CUDA runtime / no device */
#define PARS_ERR_OOM (-3)         /* device or host allocation failed */
#define PARS_ERR_UNSUPPORTED (-4) /* shape outside the implemented envelope */

/* Arithmetic modes for scoring. */
#define PARS_MODE_EXACT_F64 0 /* bit-identical to the reference (fp64, sequential
                                 ascending-index dot, no FMA) */
#define PARS_MODE_FAST_F32 1  /* fp32 weights/products, tree reduction; within
                                 1e-5 of sum|w_i v_i| */

typedef struct pars_ctx pars_ctx;
typedef struct pars_features pars_features; /* device-resident CSR */

/* pars::FeatureExtractor (features.hpp:17-25) as a C POD.
 * kind: 0 HashedText, 1 PrecomputedEmbedding; norm: 0 None, 1 L2. */
typedef struct {
  int32_t kind;
  uint32_t dim;
  int32_t norm;
  int32_t n_word;
  int32_t n_char;
  int32_t word[8];
  int32_t chr[8];
} pars_extractor;

/* ---- library / context ---------------------------------------------- */
const char* pars_last_error(void);
const char* pars_version(void);
int pars_device_count(int* count);
int pars_ctx_create(int device, pars_ctx** out);
void pars_ctx_destroy(pars_ctx* ctx);
int pars_ctx_synchronize(pars_ctx* ctx);
/* Number of kernel launches this ctx has issued (telemetry for bench.py). */
uint64_t pars_ctx_launches(const pars_ctx* ctx);
/* Pinned host memory for fast host<->device copies (optional). */
int pars_host_alloc(size_t bytes, void** out);
void pars_host_free(void* p);

/* ---- featurize + score ----------------------------------------------
 * Replaces Scorer::score_batch / LinearScorer::score(const PromptRecord&)
 * (scorer.cpp:9-24, :36-42) fused with extract_features' HashedText branch
 * (features.cpp:62-122): whitespace tokenizer, FNV-1a word/char n-grams,
 * sign hashing, merge, zero erase, L2, dot in ascending index order, +bias.
 * text: concatenated prompt bytes; offsets[n+1] (int64, offsets[0] may be
 * nonzero). weights: dim doubles. */
int pars_score_text(pars_ctx* ctx, const pars_extractor* ex, const char* text,
                    const int64_t* offsets, int64_t n, const double* weights,
                    double bias, int mode, double* scores);
/* Scorer::score_batch over records held as separate host strings (the
 * reference's Dataset of std::string, scorer.cpp:9-24): texts[i] points at
 * lens[i] bytes. Host threads gather ~64 MB chunks straight into pinned
 * staging (no packing pass), overlapped with the uploads and the kernels.
 * Bit-identical to pars_score_text over the concatenation. */
int pars_score_records(pars_ctx* ctx, const pars_extractor* ex,
                       const char* const* texts, const int64_t* lens, int64_t n,
                       const double* weights, double bias, int mode,
                       double* scores);
int pars_dev_score_text(pars_ctx* ctx, const pars_extractor* ex,
                        const char* d_text, const int64_t* d_offsets,
                        int64_t n, const double* d_weights, double bias,
                        int mode, double* d_scores, void* stream);
/* enqueue + select_batch in one call (scheduler.cpp:17-31 scores every
 * waiting request, scheduler.cpp:33-60 orders them): score the prompts and
 * return both the scores and the full priority order (order[k] = index of
 * the k-th request to admit; truncate to the free slots). The scores stay on
 * the device between the two steps; one synchronisation. boosted may be
 * NULL. tie_rank as for pars_priority_order. */
int pars_score_order(pars_ctx* ctx, const pars_extractor* ex, const char* text,
                     const int64_t* offsets, int64_t n, const double* weights,
                     double bias, int mode, const uint32_t* tie_rank,
                     const uint8_t* boosted, double* scores, int64_t* order);
/* PrecomputedEmbedding branch (features.cpp:67-76): X is n x dim row-major. */
int pars_score_embeddings(pars_ctx* ctx, const pars_extractor* ex,
                          const double* X, int64_t n, const double* weights,
                          double bias, int mode, double* scores);
/* Same, device-resident X / weights / scores, asynchronous on `stream`
 * (NULL: the context's stream). */
int pars_dev_score_embeddings(pars_ctx* ctx, const pars_extractor* ex,
                              const double* d_X, int64_t n,
                              const double* d_weights, double bias, int mode,
                              double* d_scores, void* stream);

/* ---- dataset ingestion (load_dataset, dataset.cpp:73-173) ------------ */
/* The records of a JSONL dataset file parsed and validated ON THE GPU into a
 * device-resident prompt arena + int64 offsets (what pars_dev_score_text
 * reads), ids, output_len and prompt_len (given, or the whitespace token
 * count). Same acceptance and the reference's error text ("<path>: line N:
 * ..."), limit < 0 = no limit. Records carrying an 'embedding' array are
 * rejected with PARS_ERR_UNSUPPORTED (the GPU loader does not parse them). */
typedef struct pars_dataset pars_dataset;
int pars_load_dataset(pars_ctx* ctx, const char* path, int64_t limit,
                      pars_dataset** out);
int pars_load_dataset_bytes(pars_ctx* ctx, const char* path_for_messages,
                            const char* bytes, int64_t nbytes, int64_t limit,
                            pars_dataset** out);
int64_t pars_dataset_size(const pars_dataset* d);
int64_t pars_dataset_text_bytes(const pars_dataset* d);
int64_t pars_dataset_id_bytes(const pars_dataset* d);
int64_t pars_dataset_embedding_dim(const pars_dataset* d);
const char* pars_dataset_dev_text(const pars_dataset* d);        /* device */
const int64_t* pars_dataset_dev_offsets(const pars_dataset* d);  /* device, [n+1] */
const int64_t* pars_dataset_dev_output_len(const pars_dataset* d);
/* host copies (any pointer may be NULL) */
int pars_dataset_export(const pars_dataset* d, char* text, int64_t* offsets,
                        int64_t* output_len, int64_t* prompt_len, char* ids,
                        int64_t* id_offsets);
/* output_len_samples of record i; returns the count (-1 if > cap or i is
 * out of range) */
int64_t pars_dataset_samples(const pars_dataset* d, int64_t i, int64_t* out,
                             int64_t cap);
void pars_dataset_free(pars_dataset* d);

/* ---- features (extract_all, features.cpp:124-150) -------------------- */
int pars_extract(pars_ctx* ctx, const pars_extractor* ex, const char* text,
                 const int64_t* offsets, int64_t n, const double* embeddings,
                 pars_features** out);
/* Upload caller FeatureVecs (sorted unique idx per row) as a CSR. */
int pars_features_upload(pars_ctx* ctx, uint32_t dim, int64_t rows,
                         const int64_t* row_ptr, const uint32_t* idx,
                         const double* val, pars_features** out);
int64_t pars_features_rows(const pars_features* f);
int64_t pars_features_nnz(const pars_features* f);
int64_t pars_features_dim(const pars_features* f);
/* Copies the CSR back to the host: row_ptr[rows+1], idx[nnz], val[nnz]. */
int pars_features_download(pars_ctx* ctx, const pars_features* f,
                           int64_t* row_ptr, uint32_t* idx, double* val);
void pars_features_free(pars_features* f);
/* LinearScorer::score(const FeatureVec&) for every row (scorer.cpp:40-42). */
int pars_features_score(pars_ctx* ctx, const pars_features* f,
                        const double* weights, double bias, double* scores);
/* Same on the device: rows [row_begin, row_end) of f scored with device
 * weights into d_scores[row_begin, row_end), asynchronous on `stream` (NULL:
 * the context's stream). The scoring step of a data-parallel training step. */
int pars_dev_features_score(pars_ctx* ctx, const pars_features* f,
                            int64_t row_begin, int64_t row_end,
                            const double* d_weights, double bias,
                            double* d_scores, void* stream);

/* ---- pair construction / loss (pairs.hpp, pairs.cpp, train.cpp) ------
 * build_pairs (pairs.cpp:8-36): seeded sampler; host (the mt19937_64 stream
 * is sequential), bit-identical to the reference. Returns the pair count
 * (>0) or a negative error ("no informative pairs"). */
int64_t pars_build_pairs(const int64_t* lengths, int64_t n, double delta,
                         uint64_t max_pairs, uint64_t seed, uint32_t* a,
                         uint32_t* b, int32_t* y, double* rel_diff);
/* dmin[m] = min{d>=1 : !(relative_length_difference(m, m-d) < delta)}
 * (INT32_MAX if none) for m in [0, max_len]: the integer form of Eq. 1. */
int pars_length_gap_table(double delta, int64_t max_len, int32_t* dmin);

/* All-pairs margin ranking loss over unordered pairs i<j:
 * keep = L_i != L_j && |L_i-L_j| >= dmin[max]; y = sign(L_i-L_j);
 * hinge = max(0, -y(s_i-s_j) + margin) (pairs.hpp:27-31). Outputs the
 * integer gradient coefficients c (grad = X^T c, c_a -= y, c_b += y on active
 * pairs), kept/active counts and the loss sum. */
int pars_allpairs(pars_ctx* ctx, const double* scores, const int64_t* lengths,
                  int64_t n, double delta, double margin, int32_t* coeff,
                  uint64_t* kept, uint64_t* active, double* loss_sum);
/* Same, choosing the kernel: PARS_ALLPAIRS_SORTED (length-sorted plan, the
 * default) or PARS_ALLPAIRS_GENERAL (unsorted tiles, per-pair table mask).
 * Identical masks, coefficients and counts; the loss sums differ only in
 * rounding order. */
#define PARS_ALLPAIRS_SORTED 0
#define PARS_ALLPAIRS_GENERAL 1
int pars_allpairs_algo(pars_ctx* ctx, const double* scores,
                       const int64_t* lengths, int64_t n, double delta,
                       double margin, int algo, int32_t* coeff, uint64_t* kept,
                       uint64_t* active, double* loss_sum);
/* Device form over a slice [tile_begin, tile_end) of the upper-triangle tile
 * list (tile count from pars_allpairs_tiles); coeff/counters are ACCUMULATED
 * (int32 c[n]; uint64 counters[2] = kept, active; double loss partials[]
 * one per tile in the slice, summed in a fixed order by the caller).
 * d_lengths are int32; every length must be <= max_len. */
int64_t pars_allpairs_tiles(int64_t n);
int pars_dev_allpairs(pars_ctx* ctx, const double* d_scores,
                      const int32_t* d_lengths, int64_t n, double delta,
                      double margin, int64_t max_len, int64_t tile_begin,
                      int64_t tile_end, int32_t* d_coeff,
                      unsigned long long* d_counters, double* d_loss_partials,
                      void* stream);
/* Per-dataset plan for the length-sorted kernel (lengths are fixed across
 * training steps): stable length order, per-row first kept column, exact
 * kept-pair count. Sharded callers pass [tile_begin, tile_end) slices as
 * for pars_dev_allpairs; outputs are in input order and accumulated. */
typedef struct pars_pair_plan pars_pair_plan;
int pars_pair_plan_create(pars_ctx* ctx, const int64_t* lengths, int64_t n,
                          double delta, pars_pair_plan** out);
uint64_t pars_pair_plan_kept(const pars_pair_plan* plan);
int pars_pair_plan_sorted(const pars_pair_plan* plan);
void pars_pair_plan_free(pars_pair_plan* plan);
int pars_dev_allpairs_plan(pars_ctx* ctx, const pars_pair_plan* plan,
                           const double* d_scores, double margin,
                           int64_t tile_begin, int64_t tile_end,
                           int32_t* d_coeff, unsigned long long* d_counters,
                           double* d_loss_partials, void* stream);
/* grad[d] = sum_i c_i x_i[d] (fp64) for rows [row_begin,row_end) of f. */
int pars_dev_xt_c(pars_ctx* ctx, const pars_features* f, const int32_t* d_coeff,
                  int64_t row_begin, int64_t row_end, double* d_grad,
                  void* stream);

/* ---- training (train.cpp:122-216, pairwise objective) ----------------
 * One SGD epoch over explicit pairs (train.cpp:154-166 with apply
 * :141-151): bit-identical weights and loss to the reference. w is in/out. */
int pars_sgd_epoch(pars_ctx* ctx, const pars_features* f, const uint32_t* a,
                   const uint32_t* b, const int32_t* y, int64_t npairs,
                   int32_t batch, double lr, double margin, double* w,
                   double bias, double* epoch_loss, uint64_t* active);
/* Same, choosing the kernel: PARS_SGD_AUTO (cluster kernel when the
 * features allow it), PARS_SGD_CLUSTER (8-CTA cluster, compact rows staged in
 * shared memory; hashed features, dim <= 65536), PARS_SGD_SINGLE_CTA (one
 * persistent CTA, any features). All are bit-identical to the reference. */
#define PARS_SGD_AUTO 0
#define PARS_SGD_CLUSTER 1
#define PARS_SGD_SINGLE_CTA 2
int pars_sgd_epoch_algo(pars_ctx* ctx, const pars_features* f,
                        const uint32_t* a, const uint32_t* b, const int32_t* y,
                        int64_t npairs, int32_t batch, double lr, double margin,
                        double* w, double bias, double* epoch_loss,
                        uint64_t* active, int algo);
/* train() for Objective::Pairwise from all-zero weights: extract_all on the
 * GPU, per-epoch build_pairs with derive_seed(seed, 0x10000+e), SGD epochs.
 * loss_trace has `epochs` slots. */
int pars_train_pairwise(pars_ctx* ctx, const pars_extractor* ex,
                        const char* text, const int64_t* offsets,
                        const int64_t* lengths, int64_t n, double delta,
                        double margin, int32_t epochs, int32_t batch,
                        double lr, uint64_t seed, uint64_t pairs_per_epoch,
                        double* w_out, double* bias_out, double* loss_trace);

/* ---- comparison objectives (train.cpp:46-94, :168-205) -----------------
 * The paper's baselines on the same engine. */
#define PARS_OBJ_PAIRWISE 0
#define PARS_OBJ_POINTWISE_L1 1
#define PARS_OBJ_LISTMLE 2
/* One PointwiseL1 epoch (train.cpp:168-183 with pointwise_l1_loss_grad
 * :46-54 and apply :141-151): samples order[0..n) (rows of f), `batch` per
 * step; target[f->rows] = pointwise_target(output_len) per row. w[dim] and
 * *bias in/out; *epoch_loss = the sum of |r| (the caller divides by n).
 * Bit-identical to the reference. */
int pars_pointwise_epoch(pars_ctx* ctx, const pars_features* f,
                         const uint32_t* order, int64_t n, const double* target,
                         int32_t batch, double lr, double* w, double* bias,
                         double* epoch_loss);
/* One ListwiseListMLE epoch (train.cpp:185-205 with listmle_loss_grad
 * :66-94): lists[nlists*k] rows, each list already longest-first
 * (pars_listmle_lists), `batch` lists per step; bias is read, not trained.
 * exp/log1p run in the CUDA libm (<= 1 ulp from glibc), so weights and loss
 * match the reference to rounding (tests: 1e-12 relative), not bits. */
int pars_listmle_epoch(pars_ctx* ctx, const pars_features* f,
                       const uint32_t* lists, int64_t nlists, int32_t k,
                       int32_t batch, double lr, double* w, double bias,
                       double* epoch_loss);
/* Host samplers (bit-identical): the PointwiseL1 epoch order (Rng(seed)
 * shuffle of 0..n-1, train.cpp:169-172) and the ListMLE epoch lists
 * (persistent-pool partial Fisher-Yates + sort_by_true_order,
 * train.cpp:110-118, :186-200); lists[nlists * min(list_size, n)]. */
int pars_pointwise_order(int64_t n, uint64_t seed, uint32_t* order);
int pars_listmle_lists(const int64_t* output_len, const char* ids,
                       const int64_t* id_offsets, int64_t n, int64_t nlists,
                       int32_t list_size, uint64_t seed, uint32_t* lists);
/* train() for PARS_OBJ_POINTWISE_L1 / PARS_OBJ_LISTMLE from all-zero
 * weights: GPU extract_all, per-epoch derive_seed(seed, 0x10000+e) order or
 * lists, GPU epochs. ids: arena + id_offsets[n+1] (ListMLE tiebreak). */
int pars_train_baseline(pars_ctx* ctx, const pars_extractor* ex,
                        const char* text, const int64_t* offsets,
                        const int64_t* lengths, const char* ids,
                        const int64_t* id_offsets, int64_t n, int32_t objective,
                        int32_t epochs, int32_t batch, double lr, uint64_t seed,
                        uint64_t lists_per_epoch, int32_t list_size,
                        double* w_out, double* bias_out, double* loss_trace);

/* ---- priority ordering (scheduler.cpp:33-60) --------------------------
 * Full select_batch order: boosted first by tie_rank; the rest ascending by
 * score then tie_rank; equal keys keep input order (stable LSD radix).
 * tie_rank = rank of (arrival_time, prompt_id bytes) — see
 * pars_tie_ranks. order[n] receives indices into the input. */
int pars_priority_order(pars_ctx* ctx, const double* scores,
                        const uint8_t* boosted, const uint32_t* tie_rank,
                        int64_t n, int64_t* order);
int pars_dev_priority_order(pars_ctx* ctx, const double* d_scores,
                            const uint8_t* d_boosted,
                            const uint32_t* d_tie_rank, int64_t n,
                            uint32_t* d_order, void* stream);
/* The global order from shard orders: prompts [run_offsets[r],
 * run_offsets[r+1]) form shard r, d_run_orders holds each shard's
 * pars_dev_priority_order result (indices relative to the shard start),
 * concatenated; d_scores / d_boosted / d_tie cover all n = run_offsets[nruns]
 * prompts. d_order[n] receives what pars_dev_priority_order over all n would
 * (bit-identical), by merging the runs (one level: each element's place is
 * its position in its run plus one binary search per other run; at most 64
 * runs). run_offsets is a host array (read before the call returns); the
 * merge is asynchronous on `stream`. */
int pars_dev_merge_orders(pars_ctx* ctx, const double* d_scores,
                          const uint8_t* d_boosted, const uint32_t* d_tie,
                          const uint32_t* d_run_orders, const int64_t* run_offsets,
                          int nruns, uint32_t* d_order, void* stream);
/* The same placement for the elements of ONE run only (run in [0, nruns)):
 * d_order[p] is written for exactly the positions p that run's elements take
 * in the merged order; other positions are untouched. Disjoint across runs,
 * so data-parallel ranks each place their own shard and combine by a sum
 * (pars_dp_score_order). */
int pars_dev_merge_rank(pars_ctx* ctx, const double* d_scores,
                        const uint8_t* d_boosted, const uint32_t* d_tie,
                        const uint32_t* d_run_orders, const int64_t* run_offsets,
                        int nruns, int run, uint32_t* d_order, void* stream);
/* Host helper: dense ranks of (arrival, id) with equal keys sharing a rank.
 * ids: arena + offsets[n+1] (raw bytes, compared unsigned). */
int pars_tie_ranks(const double* arrival, const char* ids,
                   const int64_t* id_offsets, int64_t n, uint32_t* rank);

/* ---- Kendall tau-b counts (metrics.cpp:42-64) -------------------------
 * counts[5] = {n_c, n_d, n0, n1, n2}; tau_b finished on the host exactly
 * as finish_tau (metrics.cpp:13-32). Degenerate input -> PARS_ERR_INVALID
 * with the reference's message. */
int pars_kendall_tau(pars_ctx* ctx, const double* x, const double* y,
                     int64_t n, uint64_t* counts, double* tau_b);
/* Choosing the algorithm: PARS_TAU_SORTED counts by sorting (two stable
 * radix sorts + a merge-sort inversion count, O(n log n); finite inputs
 * only), PARS_TAU_PAIRS runs the all-pairs tiles, PARS_TAU_AUTO (what
 * pars_kendall_tau does) sorts unless an input is inf/NaN. All give the
 * reference's exact integers. */
#define PARS_TAU_AUTO 0
#define PARS_TAU_SORTED 1
#define PARS_TAU_PAIRS 2
int pars_kendall_tau_algo(pars_ctx* ctx, const double* x, const double* y,
                          int64_t n, uint64_t* counts, double* tau_b, int algo);
/* pars_kendall_tau on device arrays (stream-ordered; returns after the
 * counts are on the host). */
int pars_dev_kendall_tau(pars_ctx* ctx, const double* d_x, const double* d_y,
                         int64_t n, uint64_t* counts, double* tau_b,
                         void* stream);
/* The same counts split over upper-triangle tiles (the all-pairs tiling):
 * {n_c, n_d, n1, n2} of tiles [tile_begin, tile_end) ACCUMULATED into
 * d_counts[4] on the device (for data-parallel ranks: sum the counts, an
 * exact integer all-reduce), then pars_kendall_finish on the totals. */
int64_t pars_kendall_tiles(int64_t n);
int pars_dev_kendall_counts(pars_ctx* ctx, const double* d_x, const double* d_y,
                            int64_t n, int64_t tile_begin, int64_t tile_end,
                            unsigned long long* d_counts, void* stream);
/* finish_tau (metrics.cpp:13-32): counts5 = {n_c, n_d, n0, n1, n2}. */
int pars_kendall_finish(const uint64_t* counts4, int64_t n, uint64_t* counts5,
                        double* tau_b);


/* ---- data-parallel ranks over NCCL ---------------------
 * One process per GPU. A pars_dp binds a pars_ctx to an NCCL communicator
 * (libnccl is bound at run time; an already-loaded copy, e.g. torch's, is
 * reused; PARS_NCCL_LIB overrides the path). Prompt shards are contiguous:
 * rank r owns [r*per, min(n, (r+1)*per)), per = ceil(n / world)
 * (pars_dp_shard). All pars_dp_* calls are collective: every rank calls them
 * in the same order. They are asynchronous on `stream` unless noted. */
typedef struct pars_dp pars_dp;
#define PARS_NCCL_UNIQUE_ID_BYTES 128
/* ncclGetUniqueId on one rank; the caller broadcasts the 128 bytes. */
int pars_nccl_get_unique_id(uint8_t* id);
/* ncclCommInitRank(world, id, rank) on ctx's device (owned by the dp). */
int pars_dp_create(pars_ctx* ctx, const uint8_t* id, int world, int rank,
                   pars_dp** out);
/* Wrap a caller-owned ncclComm_t (passed as void*; not destroyed). */
int pars_dp_create_from_comm(pars_ctx* ctx, void* nccl_comm, pars_dp** out);
int pars_dp_rank(const pars_dp* dp);
int pars_dp_world(const pars_dp* dp);
void pars_dp_destroy(pars_dp* dp);
void pars_dp_shard(int64_t n, int world, int rank, int64_t* begin,
                   int64_t* end);
/* Sharded Scorer::score_batch (scorer.cpp:9-24) + select_batch
 * (scheduler.cpp:33-60) of all n_total prompts: d_text/d_offsets hold THIS
 * rank's shard (offsets[m+1], relative to d_text); d_boosted_all/d_tie_all
 * (optional) cover all n_total prompts. Every rank receives all n_total
 * scores and the global order (indices into all prompts), bit-identical to
 * pars_dev_score_text + pars_dev_priority_order on one GPU: shard scores and
 * shard orders are all-gathered, each rank places its own run
 * (pars_dev_merge_rank) and the placements are summed (uint32 all-reduce). */
int pars_dp_score_order(pars_dp* dp, const pars_extractor* ex,
                        const char* d_text, const int64_t* d_offsets,
                        int64_t n_total, const double* d_w, double bias,
                        int mode, const uint8_t* d_boosted_all,
                        const uint32_t* d_tie_all, double* d_scores_all,
                        uint32_t* d_order_all, void* stream);
/* One full-batch data-parallel step of all-pairs margin-ranking training
 * over the plan's n prompts (pairs.hpp:21-31; train.cpp:34-44 in
 * coefficient form; apply train.cpp:141-151 with batch_n = kept pairs):
 * scores of this rank's rows (exact CSR dot), all-gathered; this rank's
 * cost-balanced slice of the pair tiles (pars_pair_plan_tile_split);
 * int32 coefficients and u64 {kept, active} all-reduced (exact for any rank
 * count); grad = X^T c over the row shard, fp64 all-reduce;
 * w -= (lr / kept) * grad where grad != 0. f holds all n rows on every rank.
 * Outputs (device): d_scores_all[n] (optional), d_coeff[n],
 * d_counters[2] (optional), d_loss (optional: the loss sum, per-tile partials
 * summed in tile order — identical for every rank count). */
int pars_dp_train_step(pars_dp* dp, const pars_features* f,
                       const pars_pair_plan* plan, double* d_w, double margin,
                       double lr, double* d_scores_all, int32_t* d_coeff,
                       unsigned long long* d_counters, double* d_loss,
                       void* stream);
/* kendall_tau_b (metrics.cpp:42-64) with the pair tiles split evenly across
 * ranks and one exact all-reduce of the integer counts; counts[5] and tau on
 * the host of every rank (synchronises `stream`). */
int pars_dp_kendall_tau(pars_dp* dp, const double* d_x, const double* d_y,
                        int64_t n, uint64_t* counts, double* tau_b,
                        void* stream);
/* Host-only helpers (no device): a contiguous split of weighted items with
 * equal weight per rank (bounds[world+1]); the tile weights of a pair plan
 * (fully or partly kept tiles cost 64, empty ones 1) split that way. */
int pars_split_weighted(const int64_t* weights, int64_t n, int world,
                        int64_t* bounds);
int pars_pair_plan_tile_split(const pars_pair_plan* plan, int world,
                              int64_t* bounds);

#ifdef __cplusplus
}
#endif
#endif /* PARS_CUDA_H */
