#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include <vector>

#include "common.cuh"

namespace pars_b200 {

int64_t allpairs_tile_count(int64_t n);
int launch_allpairs(pars_ctx* ctx, const double* s, const int32_t* L, const int32_t* dmin,
                    int64_t n, double margin, int64_t t0, int64_t t1, int32_t* coeff,
                    unsigned long long* counters, double* loss_part, cudaStream_t st);
int launch_sum_partials(pars_ctx* ctx, const double* p, int64_t n, double* out, cudaStream_t st);
// Kendall counts {n_c, n_d, n1, n2} of the upper-triangle tiles [t0, t1)
// (t1 < 0: all), accumulated into out[4]
int launch_tau(pars_ctx* ctx, const double* x, const double* y, int64_t n,
               unsigned long long* out, cudaStream_t st, int64_t t0 = 0, int64_t t1 = -1);
// Column-major copy of a CSR feature set (stable: rows ascending within a
// column) and the per-step gradient X[r0:r1]^T c over it.
size_t csc_scratch_bytes(int64_t rows, uint32_t dim);
int build_csc(pars_ctx* ctx, const int64_t* rp, const uint32_t* idx, const double* val,
              int64_t rows, uint32_t dim, void* scratch, int64_t* ptr, uint32_t* crow,
              double* cval, cudaStream_t st);
int launch_xtc_csc(pars_ctx* ctx, const void* tasks, int64_t ntasks, const int64_t* col_task,
                   const uint32_t* crow, const double* cval, const int32_t* c, int64_t r0,
                   int64_t r1, uint32_t dim, double* part, double* grad, cudaStream_t st);
size_t csc_task_bytes();
int64_t make_csc_tasks(const int64_t* ptr, uint32_t dim, int64_t chunk, std::vector<char>& tasks,
                       std::vector<int64_t>& col_task);
// length-sorted all-pairs plan (pairs_sorted.cu)
struct PairPlanDev {
  int64_t n = 0;
  uint32_t* perm = nullptr;  // sorted position -> input index (stable by length)
  int32_t* Ls = nullptr;     // sorted lengths
  int32_t* f = nullptr;      // first kept column of each sorted row
  double* ss = nullptr;      // per call: sorted scores
  double* T = nullptr;       // per call: hinge thresholds
  int32_t* cs = nullptr;     // per call: coefficients in sorted order
  double* srtS = nullptr;    // per call: each 256-tile's scores, sorted
  double* srtT = nullptr;    // per call: each 256-tile's thresholds, sorted
  int* nanflag = nullptr;    // per call: tile holds a NaN score / threshold
  unsigned long long kept = 0;
  bool monotone = true;  // g_j = L_j - dmin[L_j] non-decreasing (suffix masks valid)
};
size_t pair_plan_scratch_bytes(int64_t n);
int build_pair_plan(pars_ctx* ctx, const int32_t* d_L, const int32_t* d_dmin, int64_t n,
                    PairPlanDev* p, void* scratch, cudaStream_t st);
int launch_allpairs_sorted(pars_ctx* ctx, const PairPlanDev& p, const double* d_scores,
                           double margin, int64_t t0, int64_t t1, int32_t* d_coeff,
                           unsigned long long* d_counters, double* d_loss_part, cudaStream_t st);

// priority sort (sort.cu)
struct SortBuffers {
  uint64_t* khi[2];
  uint32_t* klo[2];
  uint32_t* val[2];
  uint32_t* hist;       // [256][blocks]
  uint32_t* digit_hist; // [12][256] all-digit histogram
};
size_t sort_scratch_bytes(int64_t n);
int launch_priority_sort(pars_ctx* ctx, const double* scores, const uint8_t* boosted,
                         const uint32_t* tie, int64_t n, uint32_t* order, void* scratch,
                         cudaStream_t st);

// SGD epoch (sgd.cu)
struct SgdPlan {
  int64_t npairs;
  int32_t batch;
  int64_t nbatches;
  uint32_t dim;
};
size_t sgd_scratch_bytes(int64_t nbatches, int32_t batch, uint32_t dim, int64_t max_entries);
int launch_sgd_epoch(pars_ctx* ctx, const int64_t* rp, const uint32_t* idx, const double* val,
                     uint32_t dim, const uint32_t* a, const uint32_t* b, const int32_t* y,
                     int64_t npairs, int32_t batch, double lr, double margin, double bias,
                     double* w, double* loss_out, unsigned long long* active_out,
                     int64_t total_entries, void* scratch, size_t scratch_bytes,
                     cudaStream_t st);

// Merge of per-shard select_batch orders into the global one (sort.cu).
constexpr int kMaxRuns = 64;  // shards (ranks) a merge accepts
struct RunOffsets {  // by value in kernel parameters: no upload, capturable
  int64_t off[kMaxRuns + 1];
  int nruns;
};
size_t merge_runs_scratch_bytes(int64_t n, int nruns);
// Places the elements of run `run` (all runs when run < 0) at their merged
// positions in order[] (other positions untouched). h_off: host [nruns+1].
int launch_merge_rank(pars_ctx* ctx, const double* score, const uint8_t* boosted, const uint32_t* tie,
                      const uint32_t* run_order, const int64_t* h_off, int nruns, int run,
                      uint32_t* order, void* scratch, cudaStream_t st);
int launch_merge_runs(pars_ctx* ctx, const double* score, const uint8_t* boosted, const uint32_t* tie,
                      const uint32_t* run_order, const int64_t* h_off, int nruns, int64_t n,
                      uint32_t* order, void* scratch, cudaStream_t st);

// Kendall tau-b counts by sorting (tau_sorted.cu); counts4 on the host.
size_t tau_sorted_scratch_bytes(int64_t n);
int launch_tau_sorted(pars_ctx* ctx, const double* x, const double* y, int64_t n,
                      uint64_t* counts4, void* scratch, cudaStream_t st);
// the same as two halves: every device step on `st` (no host synchronisation,
// capturable into a CUDA graph), then the read-back and finish
int enqueue_tau_sorted(pars_ctx* ctx, const double* x, const double* y, int64_t n, void* scratch,
                       cudaStream_t st);
int finish_tau_sorted(int64_t n, uint64_t* counts4, void* scratch, cudaStream_t st);

// PointwiseL1 / ListMLE epochs (baselines.cu). kind 0 = pointwise, 1 = ListMLE.
size_t baseline_smem_bytes(uint32_t dim, int64_t max_slots);
size_t baseline_scratch_bytes(int64_t nbatches, int64_t nslots, uint32_t dim, int64_t entries);
int launch_baseline_epoch(pars_ctx* ctx, int kind, const int64_t* rp, const uint32_t* idx,
                          const double* val, uint32_t dim, const uint32_t* h_srow,
                          const int64_t* h_soff, int64_t nb, int32_t k, const double* d_target,
                          double lr, double bias, int64_t max_slots, const int64_t* h_ent_off,
                          double* d_w, double* d_bias_out, double* d_loss_out, void* scratch,
                          cudaStream_t st);

}  // namespace pars_b200
