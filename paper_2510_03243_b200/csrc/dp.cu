// Data-parallel ranks over NCCL: one process per GPU, each
// with a pars_ctx and a pars_dp holding an NCCL communicator. The entry
// points are the sharded forms of the reference calls that shard:
//
//   pars_dp_score_order   Scorer::score_batch (scorer.cpp:9-24) over this
//                         rank's contiguous prompt shard + select_batch
//                         (scheduler.cpp:33-60) of ALL prompts: shard scores
//                         and shard orders are all-gathered, each rank places
//                         only its own run's elements in the global order
//                         (one binary search per other run, sort.cu
//                         merge_rank_kernel) and the disjoint placements are
//                         combined by one integer all-reduce — no rank does a
//                         pass over all N, and the result is bit-identical to
//                         one sort of all N.
//   pars_dp_train_step    one full-batch step of all-pairs margin-ranking
//                         training (pairs.hpp:21-31, train.cpp:34-44 in
//                         coefficient form, apply train.cpp:141-151): shard
//                         scores -> all-gather; this rank's cost-balanced
//                         slice of the pair tiles -> integer coefficients +
//                         counts, all-reduced exactly; X^T c on the row shard
//                         -> gradient all-reduce; the update as a kernel.
//   pars_dp_kendall_tau   kendall_tau_b (metrics.cpp:42-64) with the
//                         upper-triangle tiles split across ranks and one
//                         exact all-reduce of the four integer counts.
//
// NCCL is bound at run time (dlopen; the process's already-loaded libnccl —
// e.g. torch's — is reused), so the library has no link-time NCCL
// dependency and single-GPU users never load it.
#include <cuda_runtime.h>
#include <dlfcn.h>
#include <nccl.h>

#include <algorithm>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <string>
#include <type_traits>
#include <vector>

#include "common.cuh"
#include "pairs.cuh"

using namespace pars_b200;

namespace {

struct NcclApi {
  bool ok = false;
  ncclResult_t (*GetUniqueId)(ncclUniqueId*) = nullptr;
  ncclResult_t (*CommInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
  ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
  ncclResult_t (*CommCount)(const ncclComm_t, int*) = nullptr;
  ncclResult_t (*CommUserRank)(const ncclComm_t, int*) = nullptr;
  ncclResult_t (*AllGather)(const void*, void*, size_t, ncclDataType_t, ncclComm_t,
                            cudaStream_t) = nullptr;
  ncclResult_t (*AllReduce)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t,
                            cudaStream_t) = nullptr;
  ncclResult_t (*GroupStart)() = nullptr;
  ncclResult_t (*GroupEnd)() = nullptr;
  const char* (*GetErrorString)(ncclResult_t) = nullptr;
  std::string why;
};

const NcclApi& nccl() {
  static NcclApi api;
  static std::once_flag once;
  std::call_once(once, [] {
    const char* env = std::getenv("PARS_NCCL_LIB");
    void* h = nullptr;
    if (env && *env) {
      h = dlopen(env, RTLD_NOW | RTLD_GLOBAL);
    } else {
      // prefer the copy the process already has (torch's), else the system's
      h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_NOLOAD);
      if (!h) h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
      if (!h) h = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
    }
    if (!h) {
      const char* e = dlerror();
      api.why = std::string("cannot load NCCL (libnccl.so.2): ") + (e ? e : "?");
      return;
    }
    bool all = true;
    auto sym = [&](auto& fp, const char* name) {
      fp = reinterpret_cast<std::remove_reference_t<decltype(fp)>>(dlsym(h, name));
      if (!fp) {
        all = false;
        api.why = std::string("NCCL symbol missing: ") + name;
      }
    };
    sym(api.GetUniqueId, "ncclGetUniqueId");
    sym(api.CommInitRank, "ncclCommInitRank");
    sym(api.CommDestroy, "ncclCommDestroy");
    sym(api.CommCount, "ncclCommCount");
    sym(api.CommUserRank, "ncclCommUserRank");
    sym(api.AllGather, "ncclAllGather");
    sym(api.AllReduce, "ncclAllReduce");
    sym(api.GroupStart, "ncclGroupStart");
    sym(api.GroupEnd, "ncclGroupEnd");
    sym(api.GetErrorString, "ncclGetErrorString");
    api.ok = all;
  });
  return api;
}

#define PARS_NCCL_CHECK(expr)                                                          \
  do {                                                                                 \
    ncclResult_t _r = (expr);                                                          \
    if (_r != ncclSuccess) {                                                           \
      set_error("NCCL error %d at %s:%d: %s", (int)_r, __FILE__, __LINE__,             \
                nccl().GetErrorString ? nccl().GetErrorString(_r) : "?");              \
      return PARS_ERR_CUDA;                                                            \
    }                                                                                  \
  } while (0)

int need_nccl() {
  if (!nccl().ok) {
    set_error("%s", nccl().why.c_str());
    return PARS_ERR_UNSUPPORTED;
  }
  return PARS_OK;
}

struct Buf {
  void* p = nullptr;
  size_t cap = 0;
};

int grow(Buf& b, size_t bytes) {
  if (bytes <= b.cap) return PARS_OK;
  if (b.p) cudaFree(b.p);
  b.p = nullptr;
  b.cap = 0;
  if (cudaMalloc(&b.p, std::max<size_t>(bytes, 256)) != cudaSuccess) {
    cudaGetLastError();
    set_error("device allocation of %zu bytes failed (dp scratch)", bytes);
    return PARS_ERR_OOM;
  }
  b.cap = std::max<size_t>(bytes, 256);
  return PARS_OK;
}

// ---- kernels ----------------------------------------------------------------

// apply (train.cpp:141-151) for the full batch: scale = lr / batch_n with
// batch_n = the kept pairs, w[d] -= scale * grad[d] where grad[d] != 0.
__global__ void sgd_apply_kernel(double* __restrict__ w, const double* __restrict__ g, uint32_t dim,
                                 double scale) {
  const uint32_t d = blockIdx.x * blockDim.x + threadIdx.x;
  if (d < dim && g[d] != 0.0) w[d] = __dsub_rn(w[d], __dmul_rn(scale, g[d]));
}

// Per-tile loss partials gathered as [world][width] -> tile order.
__global__ void compact_partials_kernel(const double* __restrict__ in, int64_t width,
                                        const RunOffsets b, double* __restrict__ out) {
  const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= b.off[b.nruns]) return;
  int r = 0;
  while (r + 1 < b.nruns && b.off[r + 1] <= t) ++r;
  out[t] = in[(int64_t)r * width + (t - b.off[r])];
}

}  // namespace

struct pars_dp {
  pars_ctx* ctx = nullptr;
  int device = 0;
  ncclComm_t comm = nullptr;
  bool owns = false;
  int rank = 0, world = 1;
  std::mutex mu;
  Buf scores, orders, part, part_all, counters, grad, merge, tau;
  // tile split of the last plan used (cost-balanced), recomputed per plan
  const pars_pair_plan* split_plan = nullptr;
  std::vector<int64_t> split;
};

// pars_ctx internals this file needs are reached through the public ABI
// plus these accessors (capi.cu)
namespace pars_b200 {
int ctx_device(pars_ctx* ctx);
cudaStream_t ctx_stream(pars_ctx* ctx, void* s);
int ctx_merge_rank(pars_ctx* ctx, const double* d_scores, const uint8_t* d_boosted,
                   const uint32_t* d_tie, const uint32_t* d_run_orders, const int64_t* run_offsets,
                   int nruns, int run, uint32_t* d_order, void* stream);
int plan_tile_weights(const pars_pair_plan* plan, std::vector<int64_t>* weights);
int64_t plan_size(const pars_pair_plan* plan);
}  // namespace pars_b200

namespace {

int check_dp(pars_dp* dp) {
  if (!dp || !dp->comm) {
    set_error("null pars_dp");
    return PARS_ERR_INVALID;
  }
  return need_nccl();
}

ncclDataType_t u64_type() { return ncclUint64; }

}  // namespace

extern "C" {

int pars_nccl_get_unique_id(uint8_t* id) {
  PARS_TRY(need_nccl());
  ncclUniqueId u;
  PARS_NCCL_CHECK(nccl().GetUniqueId(&u));
  static_assert(sizeof(u) == PARS_NCCL_UNIQUE_ID_BYTES, "ncclUniqueId size");
  std::memcpy(id, &u, sizeof u);
  return PARS_OK;
}

int pars_dp_create(pars_ctx* ctx, const uint8_t* id, int world, int rank, pars_dp** out) {
  *out = nullptr;
  if (!ctx) {
    set_error("null pars_ctx");
    return PARS_ERR_INVALID;
  }
  if (world < 1 || rank < 0 || rank >= world) {
    set_error("dp: rank %d outside world %d", rank, world);
    return PARS_ERR_INVALID;
  }
  PARS_TRY(need_nccl());
  ncclUniqueId u;
  std::memcpy(&u, id, sizeof u);
  cudaSetDevice(ctx_device(ctx));
  ncclComm_t comm = nullptr;
  PARS_NCCL_CHECK(nccl().CommInitRank(&comm, world, u, rank));
  auto* dp = new pars_dp();
  dp->ctx = ctx;
  dp->device = ctx_device(ctx);
  dp->comm = comm;
  dp->owns = true;
  dp->rank = rank;
  dp->world = world;
  *out = dp;
  return PARS_OK;
}

int pars_dp_create_from_comm(pars_ctx* ctx, void* comm, pars_dp** out) {
  *out = nullptr;
  if (!ctx || !comm) {
    set_error("dp: null ctx or communicator");
    return PARS_ERR_INVALID;
  }
  PARS_TRY(need_nccl());
  auto* dp = new pars_dp();
  dp->ctx = ctx;
  dp->device = ctx_device(ctx);
  dp->comm = static_cast<ncclComm_t>(comm);
  dp->owns = false;
  if (nccl().CommCount(dp->comm, &dp->world) != ncclSuccess ||
      nccl().CommUserRank(dp->comm, &dp->rank) != ncclSuccess) {
    delete dp;
    set_error("dp: cannot query the communicator");
    return PARS_ERR_INVALID;
  }
  *out = dp;
  return PARS_OK;
}

int pars_dp_rank(const pars_dp* dp) { return dp ? dp->rank : -1; }
int pars_dp_world(const pars_dp* dp) { return dp ? dp->world : 0; }

void pars_dp_destroy(pars_dp* dp) {
  if (!dp) return;
  cudaSetDevice(dp->device);
  cudaDeviceSynchronize();
  if (dp->owns && dp->comm && nccl().ok) nccl().CommDestroy(dp->comm);
  for (Buf* b : {&dp->scores, &dp->orders, &dp->part, &dp->part_all, &dp->counters, &dp->grad,
                 &dp->merge, &dp->tau})
    if (b->p) cudaFree(b->p);
  cudaGetLastError();
  delete dp;
}

void pars_dp_shard(int64_t n, int world, int rank, int64_t* begin, int64_t* end) {
  const int64_t per = world > 0 ? (n + world - 1) / world : n;
  *begin = std::min<int64_t>(n, (int64_t)rank * per);
  *end = std::min<int64_t>(n, (int64_t)(rank + 1) * per);
}

// Cost-balanced contiguous split of weighted items: bounds[world+1], rank r
// takes [bounds[r], bounds[r+1]); every boundary is the first item whose
// weight prefix reaches r/world of the total.
int pars_split_weighted(const int64_t* weights, int64_t n, int world, int64_t* bounds) {
  if (world < 1 || n < 0) {
    set_error("split: world %d, n %lld", world, (long long)n);
    return PARS_ERR_INVALID;
  }
  long double total = 0;
  for (int64_t t = 0; t < n; ++t) {
    if (weights[t] < 0) {
      set_error("split: negative weight at %lld", (long long)t);
      return PARS_ERR_INVALID;
    }
    total += (long double)weights[t];
  }
  bounds[0] = 0;
  long double acc = 0;
  int64_t t = 0;
  for (int r = 1; r < world; ++r) {
    const long double target = total * r / world;
    while (t < n && acc + (long double)weights[t] / 2 < target) acc += (long double)weights[t++];
    bounds[r] = t;
  }
  bounds[world] = n;
  return PARS_OK;
}

int pars_pair_plan_tile_split(const pars_pair_plan* plan, int world, int64_t* bounds) {
  std::vector<int64_t> w;
  PARS_TRY(plan_tile_weights(plan, &w));
  return pars_split_weighted(w.data(), (int64_t)w.size(), world, bounds);
}

int pars_dev_merge_rank(pars_ctx* ctx, const double* d_scores, const uint8_t* d_boosted,
                        const uint32_t* d_tie, const uint32_t* d_run_orders, const int64_t* run_offsets,
                        int nruns, int run, uint32_t* d_order, void* stream) {
  if (!ctx) {
    set_error("null pars_ctx");
    return PARS_ERR_INVALID;
  }
  if (nruns < 1 || run_offsets[0] != 0 || run >= nruns) {
    set_error("merge_rank: need >= 1 run starting at offset 0 and run < nruns");
    return PARS_ERR_INVALID;
  }
  for (int r = 0; r < nruns; ++r)
    if (run_offsets[r + 1] < run_offsets[r]) {
      set_error("merge_orders: run offsets must be non-decreasing");
      return PARS_ERR_INVALID;
    }
  return ctx_merge_rank(ctx, d_scores, d_boosted, d_tie, d_run_orders, run_offsets, nruns, run,
                        d_order, stream);
}

int pars_dp_score_order(pars_dp* dp, const pars_extractor* ex, const char* d_text,
                        const int64_t* d_offsets, int64_t n_total, const double* d_w, double bias,
                        int mode, const uint8_t* d_boosted_all, const uint32_t* d_tie_all,
                        double* d_scores_all, uint32_t* d_order_all, void* stream) {
  PARS_TRY(check_dp(dp));
  if (n_total < 0 || n_total > 0x7fffffffLL) {
    set_error("dp_score_order: n=%lld outside [0, 2^31-1]", (long long)n_total);
    return PARS_ERR_UNSUPPORTED;
  }
  if (dp->world > kMaxRuns) {
    set_error("dp_score_order: world %d above %d", dp->world, kMaxRuns);
    return PARS_ERR_UNSUPPORTED;
  }
  std::lock_guard<std::mutex> lk(dp->mu);
  cudaSetDevice(dp->device);
  pars_ctx* ctx = dp->ctx;
  cudaStream_t st = ctx_stream(ctx, stream);
  const int W = dp->world, R = dp->rank;
  const int64_t per = (n_total + W - 1) / std::max(W, 1);
  int64_t b, e;
  pars_dp_shard(n_total, W, R, &b, &e);
  const int64_t m = e - b;
  PARS_TRY(grow(dp->scores, (size_t)std::max<int64_t>(per * W, 1) * 8));
  PARS_TRY(grow(dp->orders, (size_t)std::max<int64_t>(per * W, 1) * 4));
  double* S = static_cast<double*>(dp->scores.p);
  uint32_t* O = static_cast<uint32_t*>(dp->orders.p);
  // 1. this rank's shard: scores into its slot of the gather buffer, then
  //    its select_batch order (indices relative to the shard)
  if (m > 0) {
    PARS_TRY(pars_dev_score_text(ctx, ex, d_text, d_offsets, m, d_w, bias, mode, S + R * per, st));
    PARS_TRY(pars_dev_priority_order(ctx, S + R * per, d_boosted_all ? d_boosted_all + b : nullptr,
                                     d_tie_all ? d_tie_all + b : nullptr, m, O + R * per, st));
  }
  // 2. all-gather scores and shard orders (in place: rank r's slot is its
  //    own send buffer). Shards are [r*per, min(n, (r+1)*per)), so the first
  //    n entries of the gathered buffers are the global scores and the runs
  //    back to back.
  if (per > 0) {
    PARS_NCCL_CHECK(nccl().GroupStart());
    PARS_NCCL_CHECK(nccl().AllGather(S + R * per, S, (size_t)per, ncclFloat64, dp->comm, st));
    PARS_NCCL_CHECK(nccl().AllGather(O + R * per, O, (size_t)per, ncclUint32, dp->comm, st));
    PARS_NCCL_CHECK(nccl().GroupEnd());
  }
  if (d_scores_all && n_total > 0)
    PARS_CUDA_CHECK(cudaMemcpyAsync(d_scores_all, S, (size_t)n_total * 8, cudaMemcpyDeviceToDevice, st));
  if (!d_order_all || n_total == 0) return PARS_OK;
  // 3. place this rank's run in the global order; the other positions stay 0
  //    and the ranks' disjoint placements add up in one exact all-reduce
  std::vector<int64_t> off((size_t)W + 1);
  for (int r = 0; r <= W; ++r) off[r] = std::min<int64_t>(n_total, (int64_t)r * per);
  PARS_CUDA_CHECK(cudaMemsetAsync(d_order_all, 0, (size_t)n_total * 4, st));
  PARS_TRY(grow(dp->merge, merge_runs_scratch_bytes(n_total, W)));
  PARS_TRY(launch_merge_rank(ctx, S, d_boosted_all, d_tie_all, O, off.data(), W, R, d_order_all,
                             dp->merge.p, st));
  if (W > 1)
    PARS_NCCL_CHECK(nccl().AllReduce(d_order_all, d_order_all, (size_t)n_total, ncclUint32, ncclSum,
                                     dp->comm, st));
  return PARS_OK;
}

int pars_dp_train_step(pars_dp* dp, const pars_features* f, const pars_pair_plan* plan, double* d_w,
                       double margin, double lr, double* d_scores_all, int32_t* d_coeff,
                       unsigned long long* d_counters, double* d_loss, void* stream) {
  PARS_TRY(check_dp(dp));
  if (!f || !plan) {
    set_error("dp_train_step: null features or pair plan");
    return PARS_ERR_INVALID;
  }
  const int64_t n = plan_size(plan);
  if (pars_features_rows(f) != n) {
    set_error("dp_train_step: %lld feature rows for a %lld-prompt pair plan",
              (long long)pars_features_rows(f), (long long)n);
    return PARS_ERR_INVALID;
  }
  const uint64_t kept = pars_pair_plan_kept(plan);
  if (kept == 0) {
    set_error("no informative pairs");
    return PARS_ERR_INVALID;
  }
  std::lock_guard<std::mutex> lk(dp->mu);
  cudaSetDevice(dp->device);
  pars_ctx* ctx = dp->ctx;
  cudaStream_t st = ctx_stream(ctx, stream);
  const int W = dp->world, R = dp->rank;
  const uint32_t dim = (uint32_t)pars_features_dim(f);
  const int64_t per = (n + W - 1) / W;
  int64_t r0, r1;
  pars_dp_shard(n, W, R, &r0, &r1);
  if (dp->split_plan != plan) {
    dp->split.assign((size_t)W + 1, 0);
    PARS_TRY(pars_pair_plan_tile_split(plan, W, dp->split.data()));
    dp->split_plan = plan;
  }
  const int64_t t0 = dp->split[R], t1 = dp->split[R + 1];
  int64_t width = 1;
  for (int r = 0; r < W; ++r) width = std::max<int64_t>(width, dp->split[r + 1] - dp->split[r]);
  const int64_t tiles = dp->split[W];
  PARS_TRY(grow(dp->scores, (size_t)per * W * 8));
  PARS_TRY(grow(dp->part, (size_t)width * W * 8 + (size_t)tiles * 8 + 64));
  PARS_TRY(grow(dp->counters, 64));
  PARS_TRY(grow(dp->grad, (size_t)dim * 8));
  double* S = static_cast<double*>(dp->scores.p);
  double* part = static_cast<double*>(dp->part.p);  // [W][width] gathered, then [tiles]
  double* tile_loss = part + width * W;
  double* mine = part + width * R;
  unsigned long long* cnt = d_counters ? d_counters : static_cast<unsigned long long*>(dp->counters.p);
  double* g = static_cast<double*>(dp->grad.p);
  // 1. scores of this rank's rows (the kernel writes out[row]: aim it so
  //    row r0 lands in this rank's gather slot), all-gathered
  if (r1 > r0) PARS_TRY(pars_dev_features_score(ctx, f, r0, r1, d_w, 0.0, S + R * per - r0, st));
  if (W > 1)
    PARS_NCCL_CHECK(nccl().AllGather(S + R * per, S, (size_t)per, ncclFloat64, dp->comm, st));
  if (d_scores_all)
    PARS_CUDA_CHECK(cudaMemcpyAsync(d_scores_all, S, (size_t)n * 8, cudaMemcpyDeviceToDevice, st));
  // 2. this rank's tiles: integer coefficients, counts, per-tile loss
  PARS_CUDA_CHECK(cudaMemsetAsync(d_coeff, 0, (size_t)n * 4, st));
  PARS_CUDA_CHECK(cudaMemsetAsync(cnt, 0, 16, st));
  PARS_CUDA_CHECK(cudaMemsetAsync(part, 0, (size_t)width * W * 8, st));
  PARS_TRY(pars_dev_allpairs_plan(ctx, plan, S, margin, t0, t1, d_coeff, cnt, mine, st));
  // 3. exact integer exchange + the per-tile partials in tile order
  if (W > 1) {
    PARS_NCCL_CHECK(nccl().GroupStart());
    PARS_NCCL_CHECK(nccl().AllReduce(d_coeff, d_coeff, (size_t)n, ncclInt32, ncclSum, dp->comm, st));
    PARS_NCCL_CHECK(nccl().AllReduce(cnt, cnt, 2, u64_type(), ncclSum, dp->comm, st));
    PARS_NCCL_CHECK(nccl().AllGather(mine, part, (size_t)width, ncclFloat64, dp->comm, st));
    PARS_NCCL_CHECK(nccl().GroupEnd());
  }
  if (d_loss && tiles > 0) {
    RunOffsets b{};
    b.nruns = W;
    for (int r = 0; r <= W; ++r) b.off[r] = dp->split[r];
    compact_partials_kernel<<<(unsigned)ceil_div(tiles, 256), 256, 0, st>>>(part, width, b, tile_loss);
    count_launch(ctx);
    PARS_TRY(launch_sum_partials(ctx, tile_loss, tiles, d_loss, st));
  }
  // 4. grad = X^T c over this rank's rows, summed across ranks; the update
  PARS_TRY(pars_dev_xt_c(ctx, f, d_coeff, r0, r1, g, st));
  if (W > 1)
    PARS_NCCL_CHECK(nccl().AllReduce(g, g, dim, ncclFloat64, ncclSum, dp->comm, st));
  const double scale = lr / (double)kept;
  sgd_apply_kernel<<<(unsigned)ceil_div(dim, 256), 256, 0, st>>>(d_w, g, dim, scale);
  count_launch(ctx);
  PARS_CUDA_CHECK(cudaGetLastError());
  return PARS_OK;
}

int pars_dp_kendall_tau(pars_dp* dp, const double* d_x, const double* d_y, int64_t n, uint64_t* counts,
                        double* tau_b, void* stream) {
  PARS_TRY(check_dp(dp));
  std::lock_guard<std::mutex> lk(dp->mu);
  cudaSetDevice(dp->device);
  cudaStream_t st = ctx_stream(dp->ctx, stream);
  const int64_t tiles = pars_kendall_tiles(n);
  int64_t t0, t1;
  pars_dp_shard(tiles, dp->world, dp->rank, &t0, &t1);
  PARS_TRY(grow(dp->tau, 64));
  auto* c = static_cast<unsigned long long*>(dp->tau.p);
  PARS_CUDA_CHECK(cudaMemsetAsync(c, 0, 32, st));
  if (t1 > t0) PARS_TRY(pars_dev_kendall_counts(dp->ctx, d_x, d_y, n, t0, t1, c, st));
  if (dp->world > 1)
    PARS_NCCL_CHECK(nccl().AllReduce(c, c, 4, u64_type(), ncclSum, dp->comm, st));
  uint64_t h[4];
  PARS_CUDA_CHECK(cudaMemcpyAsync(h, c, 32, cudaMemcpyDeviceToHost, st));
  PARS_CUDA_CHECK(cudaStreamSynchronize(st));
  return pars_kendall_finish(h, n, counts, tau_b);
}

}  // extern "C"
