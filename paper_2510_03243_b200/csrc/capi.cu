// C ABI (include/pars_cuda.h): context, device memory, host<->device staging
// and orchestration of the kernels in featurize.cu / pairs.cu / sort.cu /
// sgd.cu. Each entry cites the reference function it replaces.
#include <cuda_runtime.h>

#include <algorithm>
#include <atomic>
#include <cmath>
#include <cstdarg>
#include <cstdio>
#include <cstring>
#include <condition_variable>
#include <functional>
#include <memory>
#include <mutex>
#include <string>
#include <thread>
#include <vector>

#include "common.cuh"
#include "featurize.cuh"
#include "pairs.cuh"
#include "ingest.cuh"
#include "ingest_host.hpp"
#include "sgd_cluster.cuh"
#include "tiles.cuh"

namespace pars_b200 {

namespace {
thread_local std::string g_error;
}

void set_error(const char* fmt, ...) {
  char buf[1024];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof buf, fmt, ap);
  va_end(ap);
  g_error = buf;
}
const char* get_error() { return g_error.c_str(); }

}  // namespace pars_b200

using namespace pars_b200;

struct DevBuf {
  void* p = nullptr;
  size_t cap = 0;
};

// pinned host staging (grow-only): lets the chunked host-buffer calls keep
// every copy asynchronous, so chunk k+1's upload overlaps chunk k's kernel
struct HostBuf {
  void* p = nullptr;
  size_t cap = 0;
};

// Fork-join pool of host threads for the gathering copy of pageable records
// into pinned staging (pars_score_records): workers wait on a generation
// counter; run(k, fn) calls fn(0..k-1) across them and the caller.
class CopyPool {
 public:
  explicit CopyPool(int workers) {
    for (int i = 0; i < workers; ++i) th_.emplace_back([this, i] { loop(i + 1); });
  }
  ~CopyPool() {
    {
      std::lock_guard<std::mutex> lk(mu_);
      stop_ = true;
      ++gen_;
    }
    cv_.notify_all();
    for (auto& t : th_) t.join();
  }
  int size() const { return (int)th_.size() + 1; }
  void run(const std::function<void(int)>& fn) {
    {
      std::lock_guard<std::mutex> lk(mu_);
      fn_ = &fn;
      pending_ = (int)th_.size();
      ++gen_;
    }
    cv_.notify_all();
    fn(0);
    std::unique_lock<std::mutex> lk(mu_);
    done_.wait(lk, [this] { return pending_ == 0; });
    fn_ = nullptr;
  }

 private:
  void loop(int id) {
    uint64_t seen = 0;
    for (;;) {
      const std::function<void(int)>* f;
      {
        std::unique_lock<std::mutex> lk(mu_);
        cv_.wait(lk, [&] { return gen_ != seen; });
        seen = gen_;
        if (stop_) return;
        f = fn_;
      }
      (*f)(id);
      std::lock_guard<std::mutex> lk(mu_);
      if (--pending_ == 0) done_.notify_one();
    }
  }
  std::vector<std::thread> th_;
  std::mutex mu_;
  std::condition_variable cv_, done_;
  const std::function<void(int)>* fn_ = nullptr;
  uint64_t gen_ = 0;
  int pending_ = 0;
  bool stop_ = false;
};

struct pars_ctx {
  int device = 0;
  cudaStream_t stream = nullptr;
  cudaStream_t copy_stream = nullptr;
  std::mutex mu;
  std::atomic<uint64_t> launches{0};
  // grow-only scratch
  DevBuf text[2], offs[2], scores[2], w64, w32, misc, misc2, longl, sort, sgd, pairs_in, dmin_buf,
      gscratch, lists, plan_buf, baseline, tau;
  HostBuf h_offs[2], h_scores, h_text[2];
  std::unique_ptr<CopyPool> pool;  // created on the first pars_score_records
  std::vector<cudaEvent_t> ev_chunk;  // per-chunk score hand-off (grow-only)
  // the ctx's device scratch is shared by calls on any stream: each call's
  // work is ordered after the previous call's (event recorded on the stream
  // it used), except inside a stream capture (one stream, ordered already)
  cudaEvent_t scratch_ev = nullptr;
  cudaStream_t scratch_stream = nullptr;  // where scratch_ev was last recorded
  cudaStream_t cur_stream = nullptr;      // the stream the current call uses
  cudaEvent_t ev_copy[2] = {nullptr, nullptr};
  cudaEvent_t ev_done[2] = {nullptr, nullptr};
  double dmin_delta = -1.0;
  int64_t dmin_max = -1;
  // host copy of the weights last uploaded into w64 (and converted into w32):
  // a serving loop that scores with unchanged weights skips the upload
  std::vector<double> w_shadow;
  bool w64_valid = false, w32_valid = false;
  // the sorted Kendall tau's ~30 dependent launches as one CUDA graph,
  // re-instantiated when its inputs, size or scratch change
  cudaGraphExec_t tau_exec = nullptr;
  const void* tau_key[3] = {nullptr, nullptr, nullptr};
  int64_t tau_key_n = -1;
  uint64_t tau_launches = 0;
};

struct pars_features {
  pars_ctx* ctx = nullptr;
  int device = 0;
  uint32_t dim = 0;
  int64_t rows = 0, nnz = 0;
  int64_t* d_rp = nullptr;
  uint32_t* d_idx = nullptr;
  double* d_val = nullptr;
  std::vector<int64_t> h_rp;  // host mirror of the row pointers
  // hashed features only: integer bucket counts and per-row L2 factors
  // (val = count * inv exactly) — the compact form the SGD cluster kernel reads
  int32_t* d_cnt = nullptr;
  double* d_inv = nullptr;
  uint32_t* d_cpk = nullptr;      // rows of (idx << 16 | count + 2^15), 4-entry aligned
  uint32_t* d_cpk_off = nullptr;  // row offsets into d_cpk (entries)
  std::vector<uint32_t> h_cpk_off;
  int cpk_state = 0;  // 0 not built, 1 built, -1 not representable
  // column-major copy for X^T c (built on first use)
  int64_t* d_csc_ptr = nullptr;
  uint32_t* d_csc_row = nullptr;
  double* d_csc_val = nullptr;
  void* d_csc_tasks = nullptr;       // column chunks (one warp each)
  int64_t* d_csc_col_task = nullptr;  // [dim+1] first task of each column
  double* d_csc_part = nullptr;       // per-task partial sums
  int64_t csc_ntasks = 0;
};

namespace pars_b200 {
void count_launch(pars_ctx* ctx, uint64_t k) {
  if (ctx) ctx->launches.fetch_add(k, std::memory_order_relaxed);
}
}  // namespace pars_b200

namespace pars_b200 {
namespace capi_detail {

int ensure(DevBuf& b, size_t bytes) {
  if (bytes <= b.cap) return PARS_OK;
  if (b.p) cudaFree(b.p);
  b.p = nullptr;
  b.cap = 0;
  size_t want = std::max<size_t>(bytes, 256);
  want = want + want / 4;  // headroom for growth
  if (cudaMalloc(&b.p, want) != cudaSuccess) {
    cudaGetLastError();
    if (cudaMalloc(&b.p, bytes) != cudaSuccess) {
      cudaGetLastError();
      set_error("device allocation of %zu bytes failed", bytes);
      return PARS_ERR_OOM;
    }
    want = bytes;
  }
  b.cap = want;
  return PARS_OK;
}

int ensure_host(HostBuf& b, size_t bytes) {
  if (bytes <= b.cap) return PARS_OK;
  if (b.p) cudaFreeHost(b.p);
  b.p = nullptr;
  b.cap = 0;
  const size_t want = std::max<size_t>(bytes + bytes / 4, 4096);
  if (cudaHostAlloc(&b.p, want, cudaHostAllocDefault) != cudaSuccess) {
    cudaGetLastError();
    set_error("pinned host allocation of %zu bytes failed", want);
    return PARS_ERR_OOM;
  }
  b.cap = want;
  return PARS_OK;
}

// Per-object device memory (features, pair plans) comes from the device's
// stream-ordered pool on the context stream: after warm-up an allocation or
// release costs a few microseconds instead of cudaMalloc/cudaFree's
// milliseconds (cudaFree synchronises the device and unmaps).
bool pool_alloc(pars_ctx* ctx, void** p, size_t bytes) {
  if (cudaMallocAsync(p, std::max<size_t>(bytes, 16), ctx->stream) != cudaSuccess) {
    cudaGetLastError();
    *p = nullptr;
    return false;
  }
  return true;
}
void pool_free(pars_ctx* ctx, void* p) {
  if (p) cudaFreeAsync(p, ctx->stream);
}
// Releasing an object may happen after its context is gone (language
// bindings free in any order): wait for the device, then return the blocks
// to the pool through the legacy stream. No context dereference.
void pool_release(int device, void* const* ptrs, int k) {
  cudaSetDevice(device);
  cudaDeviceSynchronize();
  for (int i = 0; i < k; ++i)
    if (ptrs[i]) cudaFreeAsync(ptrs[i], 0);
  cudaGetLastError();
}

bool capturing(cudaStream_t st) {
  cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
  if (cudaStreamIsCapturing(st, &cs) != cudaSuccess) {
    cudaGetLastError();
    return false;
  }
  return cs != cudaStreamCaptureStatusNone;
}

// Orders `st` after the previous call's use of the ctx scratch.
void order_on(pars_ctx* ctx, cudaStream_t st) {
  if (ctx->scratch_stream && ctx->scratch_stream != st && !capturing(st))
    cudaStreamWaitEvent(st, ctx->scratch_ev, 0);
  ctx->cur_stream = st;
}

struct Guard {
  pars_ctx* c;
  std::lock_guard<std::mutex> lk;
  explicit Guard(pars_ctx* ctx) : c(ctx), lk(ctx->mu) {
    cudaSetDevice(ctx->device);
    order_on(ctx, ctx->stream);
  }
  ~Guard() {
    cudaStream_t st = c->cur_stream ? c->cur_stream : c->stream;
    if (c->scratch_ev && !capturing(st)) {
      cudaEventRecord(c->scratch_ev, st);
      c->scratch_stream = st;
    }
    c->cur_stream = nullptr;
  }
};

cudaStream_t pick(pars_ctx* ctx, void* s) {
  cudaStream_t st = s ? static_cast<cudaStream_t>(s) : ctx->stream;
  order_on(ctx, st);
  return st;
}

int check_ctx(pars_ctx* ctx) {
  if (!ctx) {
    set_error("null pars_ctx");
    return PARS_ERR_INVALID;
  }
  return PARS_OK;
}

__global__ void u32_to_i64_kernel(const uint32_t* in, int64_t* out, int64_t n) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) out[i] = in[i];
}

// true when p is page-locked host memory the device can DMA into directly
bool is_pinned(const void* p) {
  cudaPointerAttributes a;
  if (cudaPointerGetAttributes(&a, p) != cudaSuccess) {
    cudaGetLastError();
    return false;
  }
  return a.type == cudaMemoryTypeHost;
}

__global__ void f64_to_f32_kernel(const double* in, float* out, int64_t n) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) out[i] = (float)in[i];
}

// Sequential fp64 dot per CSR row (features.hpp:31-35 + scorer.cpp:40-42).
__global__ void csr_score_kernel(const int64_t* __restrict__ rp, const uint32_t* __restrict__ idx,
                                 const double* __restrict__ val, int64_t rows,
                                 const double* __restrict__ w, double bias,
                                 double* __restrict__ out) {
  const int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (r >= rows) return;
  double s = 0.0;
  for (int64_t e = rp[r]; e < rp[r + 1]; ++e) s = __dadd_rn(s, __dmul_rn(w[idx[e]], val[e]));
  out[r] = __dadd_rn(s, bias);
}

// Same dot over the compact rows (idx << 16 | count + 2^15, 4-entry aligned):
// v = count * inv_row is recomputed with the very __dmul_rn that produced the
// CSR value, so the products and the sequential sum are identical; 4 bytes
// per entry instead of 12, read 16 bytes at a time.
__global__ void cpk_score_kernel(const int64_t* __restrict__ rp, const uint32_t* __restrict__ cpk,
                                 const uint32_t* __restrict__ off, const double* __restrict__ inv_row,
                                 int64_t rows, const double* __restrict__ w, double bias,
                                 double* __restrict__ out) {
  const int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (r >= rows) return;
  const int64_t len = rp[r + 1] - rp[r];
  const uint32_t* row = cpk + off[r];
  const double inv = inv_row[r];
  double s = 0.0;
  int64_t k = 0;
  for (; k + 4 <= len; k += 4) {
    const uint4 q = *reinterpret_cast<const uint4*>(row + k);
    const uint32_t e[4] = {q.x, q.y, q.z, q.w};
#pragma unroll
    for (int j = 0; j < 4; ++j)
      s = __dadd_rn(s, __dmul_rn(w[e[j] >> 16], __dmul_rn(biased16_to_f64(e[j]), inv)));
  }
  for (; k < len; ++k)
    s = __dadd_rn(s, __dmul_rn(w[row[k] >> 16], __dmul_rn(biased16_to_f64(row[k]), inv)));
  out[r] = __dadd_rn(s, bias);
}

// The same dot with cooperative staging (repeated scoring of many rows, the
// HBM-bound case): a CTA owns kCpkRows consecutive rows, one thread per row
// running its sequential chain; the rows' entries arrive in chunks of kCpkW
// entries per row by 16-byte cp.async copies issued so that a warp covers
// four rows' 128-byte segments (full sectors, instead of 32 rows' scattered
// 16-byte loads); the chains read their row from shared memory (a 16-byte pad
// per row keeps the 16-byte reads conflict-free). One 36 KB stage per CTA:
// six CTAs per SM overlap each other's copies, and L1 keeps room for the
// weights the chains gather (1 M C4 rows: 0.476 -> 0.412 ms; 2 / 3 stages
// 0.48 / 0.60 ms, 16- / 64-entry chunks 0.43 / 0.48 ms).
#ifndef PARS_CPK_STAGES
#define PARS_CPK_STAGES 1
#endif
#ifndef PARS_CPK_W
#define PARS_CPK_W 32
#endif
constexpr int kCpkRows = 256, kCpkW = PARS_CPK_W, kCpkStages = PARS_CPK_STAGES;
constexpr int kCpkPitch = kCpkW + 4;  // entries per staged row (+16 B pad)
constexpr size_t kCpkSmem = (size_t)kCpkStages * kCpkRows * kCpkPitch * 4;

__global__ void __launch_bounds__(kCpkRows) cpk_score_coop_kernel(
    const int64_t* __restrict__ rp, const uint32_t* __restrict__ cpk, const uint32_t* __restrict__ off,
    const double* __restrict__ inv_row, int64_t rows, const double* __restrict__ w, double bias,
    double* __restrict__ out) {
  extern __shared__ __align__(16) uint32_t cst[];
  __shared__ uint32_t s_off[kCpkRows], s_len[kCpkRows];
  __shared__ int s_max;
  const int t = threadIdx.x;
  const int64_t r0 = (int64_t)blockIdx.x * kCpkRows;
  const int64_t r = r0 + t;
  const bool ok = r < rows;
  const uint32_t len = ok ? (uint32_t)(rp[r + 1] - rp[r]) : 0u;
  s_off[t] = ok ? off[r] : 0u;
  s_len[t] = len;
  if (t == 0) s_max = 0;
  __syncthreads();
  atomicMax(&s_max, (int)len);
  __syncthreads();
  const int nch = (s_max + kCpkW - 1) / kCpkW;
  // chunk k -> stage k % kCpkStages: thread t copies 16-byte part t % kParts
  // of rows t / kParts + kRowsPer i, i < kParts
  constexpr int kParts = kCpkW / 4, kRowsPer = kCpkRows / kParts;
  auto issue = [&](int k) {
    uint32_t* stg = cst + (size_t)(k % kCpkStages) * kCpkRows * kCpkPitch;
    const uint32_t e0 = (uint32_t)k * kCpkW + 4u * (uint32_t)(t % kParts);
#pragma unroll
    for (int i = 0; i < kParts; ++i) {
      const int rr = t / kParts + kRowsPer * i;
      if (e0 < s_len[rr]) {
        const uint32_t d = (uint32_t)__cvta_generic_to_shared(stg + rr * kCpkPitch + 4 * (t % kParts));
        asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(d), "l"(cpk + s_off[rr] + e0));
      }
    }
    asm volatile("cp.async.commit_group;");
  };
#pragma unroll
  for (int k = 0; k < kCpkStages - 1; ++k) {
    if (k < nch) issue(k);
    else asm volatile("cp.async.commit_group;");
  }
  const double inv = ok ? inv_row[r] : 0.0;
  double s = 0.0;
  for (int k = 0; k < nch; ++k) {
    if (k + kCpkStages - 1 < nch) issue(k + kCpkStages - 1);
    else asm volatile("cp.async.commit_group;");
    asm volatile("cp.async.wait_group %0;" ::"n"(kCpkStages - 1));
    __syncthreads();
    const uint32_t* row = cst + (size_t)(k % kCpkStages) * kCpkRows * kCpkPitch + t * kCpkPitch;
    const int e0 = k * kCpkW;
    const int n = min(kCpkW, (int)len - e0);
    if (n == kCpkW) {
#pragma unroll
      for (int q = 0; q < kCpkW; q += 4) {
        const uint4 v4 = *reinterpret_cast<const uint4*>(row + q);
        const uint32_t e[4] = {v4.x, v4.y, v4.z, v4.w};
#pragma unroll
        for (int j = 0; j < 4; ++j)
          s = __dadd_rn(s, __dmul_rn(__ldg(w + (e[j] >> 16)), __dmul_rn(biased16_to_f64(e[j]), inv)));
      }
    } else {
      for (int q = 0; q < n; ++q) {
        const uint32_t e = row[q];
        s = __dadd_rn(s, __dmul_rn(__ldg(w + (e >> 16)), __dmul_rn(biased16_to_f64(e), inv)));
      }
    }
    __syncthreads();  // the stage is refilled next iteration
  }
  asm volatile("cp.async.wait_all;" ::: "memory");
  if (ok) out[r] = __dadd_rn(s, bias);
}

// Compact per-prompt slots into a CSR.
__global__ void compact_kernel(const int64_t* __restrict__ slot, const int64_t* __restrict__ rp,
                               int64_t n, const uint32_t* __restrict__ sidx,
                               const double* __restrict__ sval, const int32_t* __restrict__ scnt,
                               uint32_t* __restrict__ idx, double* __restrict__ val,
                               int32_t* __restrict__ cnt) {
  const int64_t i = blockIdx.x;
  if (i >= n) return;
  const int64_t s = slot[i], b = rp[i], e = rp[i + 1];
  for (int64_t k = threadIdx.x; k < e - b; k += blockDim.x) {
    idx[b + k] = sidx[s + k];
    val[b + k] = sval[s + k];
    cnt[b + k] = scnt[s + k];
  }
}

// Dense embeddings -> CSR rows with every index (features.cpp:67-76, zeros
// kept), L2 with the reference's sequential sum of squares.
__global__ void dense_csr_kernel(const double* __restrict__ X, int64_t n, uint32_t dim, int norm,
                                 uint32_t* __restrict__ idx, double* __restrict__ val) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const double* x = X + i * (int64_t)dim;
  double inv = 1.0;
  bool scale = false;
  if (norm) {
    double sq = 0.0;
    for (uint32_t k = 0; k < dim; ++k) sq = __dadd_rn(sq, __dmul_rn(x[k], x[k]));
    if (sq > 0.0) {
      inv = __ddiv_rn(1.0, __dsqrt_rn(sq));
      scale = true;
    }
  }
  for (uint32_t k = 0; k < dim; ++k) {
    idx[i * (int64_t)dim + k] = k;
    val[i * (int64_t)dim + k] = scale ? __dmul_rn(x[k], inv) : x[k];
  }
}

int upload_weights(pars_ctx* ctx, const FeatConfig& cfg, const double* w, int mode,
                   cudaStream_t st) {
  const size_t bytes = (size_t)cfg.dim * 8;
  const bool same = ctx->w64_valid && ctx->w_shadow.size() == cfg.dim &&
                    std::memcmp(ctx->w_shadow.data(), w, bytes) == 0;
  if (!same) {
    PARS_TRY(ensure(ctx->w64, bytes));
    PARS_CUDA_CHECK(cudaMemcpyAsync(ctx->w64.p, w, bytes, cudaMemcpyHostToDevice, st));
    ctx->w_shadow.assign(w, w + cfg.dim);
    ctx->w64_valid = true;
    ctx->w32_valid = false;
  }
  if (mode == PARS_MODE_FAST_F32 && !ctx->w32_valid) {
    PARS_TRY(ensure(ctx->w32, (size_t)cfg.dim * 4));
    f64_to_f32_kernel<<<(unsigned)ceil_div(cfg.dim, 256), 256, 0, st>>>(
        (const double*)ctx->w64.p, (float*)ctx->w32.p, cfg.dim);
    count_launch(ctx);
    ctx->w32_valid = true;
  }
  return PARS_OK;
}

int attach_scratch(pars_ctx* ctx, const FeatConfig& cfg, int fmode, int64_t n, FeatArgs* a) {
  size_t gs = 0, ls = 0;
  PARS_TRY(feat_scratch_bytes(cfg, fmode, n, &gs, &ls));
  a->gscratch = nullptr;
  a->gscratch_bytes = 0;
  a->lists = nullptr;
  a->lists_bytes = 0;
  a->list_cap = feat_list_cap_words(cfg);
  if (gs) {
    PARS_TRY(ensure(ctx->gscratch, gs));
    a->gscratch = static_cast<unsigned char*>(ctx->gscratch.p);
    a->gscratch_bytes = ctx->gscratch.cap;
  }
  if (ls) {
    PARS_TRY(ensure(ctx->lists, ls));
    a->lists = static_cast<uint32_t*>(ctx->lists.p);
    a->lists_bytes = ctx->lists.cap;
  }
  return PARS_OK;
}

int check_mode(int mode) {
  if (mode != PARS_MODE_EXACT_F64 && mode != PARS_MODE_FAST_F32) {
    set_error("unknown scoring mode %d", mode);
    return PARS_ERR_INVALID;
  }
  return PARS_OK;
}

// Scores [i0, i1) whose text and offsets are already on the device.
int score_chunk(pars_ctx* ctx, const FeatConfig& cfg, int mode, const uint8_t* d_text_base,
                const int64_t* d_offs, int64_t n, double bias, double* d_scores, cudaStream_t st) {
  PARS_TRY(ensure(ctx->longl, (size_t)std::max<int64_t>(n, 1) * 4 + 16));
  FeatArgs a{};
  a.text = d_text_base;
  a.offsets = d_offs;
  a.n = n;
  a.w64 = (const double*)ctx->w64.p;
  a.w32 = (const float*)ctx->w32.p;
  a.bias = bias;
  a.scores = d_scores;
  a.long_count = (int32_t*)ctx->longl.p;
  a.long_list = (int32_t*)ctx->longl.p + 4;
  const int fm = mode == PARS_MODE_EXACT_F64 ? kFeatScoreExact : kFeatScoreFast;
  PARS_TRY(attach_scratch(ctx, cfg, fm, n, &a));
  return launch_featurize(ctx, cfg, fm, a, st);
}

int ensure_dmin(pars_ctx* ctx, double delta, int64_t max_len, cudaStream_t st) {
  if (ctx->dmin_delta == delta && ctx->dmin_max >= max_len && ctx->dmin_buf.p) return PARS_OK;
  std::vector<int32_t> t((size_t)max_len + 1);
  PARS_TRY(pars_length_gap_table(delta, max_len, t.data()));
  PARS_TRY(ensure(ctx->dmin_buf, t.size() * 4));
  PARS_CUDA_CHECK(cudaMemcpyAsync(ctx->dmin_buf.p, t.data(), t.size() * 4, cudaMemcpyHostToDevice, st));
  PARS_CUDA_CHECK(cudaStreamSynchronize(st));
  ctx->dmin_delta = delta;
  ctx->dmin_max = max_len;
  return PARS_OK;
}

constexpr int64_t kMaxLengthTable = 1ll << 26;

}  // namespace capi_detail
}  // namespace pars_b200
using namespace pars_b200::capi_detail;

extern "C" {

const char* pars_last_error(void) { return get_error(); }
const char* pars_version(void) { return "pars-b200 0.1 (sm_100a)"; }

int pars_device_count(int* count) {
  int n = 0;
  cudaError_t e = cudaGetDeviceCount(&n);
  if (e != cudaSuccess) {
    cudaGetLastError();
    *count = 0;
    set_error("no CUDA device: %s", cudaGetErrorString(e));
    return PARS_ERR_CUDA;
  }
  *count = n;
  return PARS_OK;
}

int pars_ctx_create(int device, pars_ctx** out) {
  *out = nullptr;
  int n = 0;
  PARS_TRY(pars_device_count(&n));
  if (device < 0 || device >= n) {
    set_error("device %d out of range (%d devices)", device, n);
    return PARS_ERR_INVALID;
  }
  cudaDeviceProp prop;
  PARS_CUDA_CHECK(cudaGetDeviceProperties(&prop, device));
  if (prop.major != 10) {
    set_error("libpars_cuda is built for sm_100a (B200); device %d is sm_%d%d", device,
              prop.major, prop.minor);
    return PARS_ERR_CUDA;
  }
  PARS_CUDA_CHECK(cudaSetDevice(device));
  auto* c = new pars_ctx();
  c->device = device;
  PARS_CUDA_CHECK(cudaStreamCreateWithFlags(&c->stream, cudaStreamNonBlocking));
  PARS_CUDA_CHECK(cudaStreamCreateWithFlags(&c->copy_stream, cudaStreamNonBlocking));
  PARS_CUDA_CHECK(cudaEventCreateWithFlags(&c->scratch_ev, cudaEventDisableTiming));
  {
    // keep released pool memory cached (features / plans are re-created per call)
    cudaMemPool_t pool;
    if (cudaDeviceGetDefaultMemPool(&pool, device) == cudaSuccess) {
      uint64_t keep = UINT64_MAX;
      cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &keep);
    }
    cudaGetLastError();
  }
  for (int k = 0; k < 2; ++k) {
    PARS_CUDA_CHECK(cudaEventCreateWithFlags(&c->ev_copy[k], cudaEventDisableTiming));
    PARS_CUDA_CHECK(cudaEventCreateWithFlags(&c->ev_done[k], cudaEventDisableTiming));
  }
  *out = c;
  return PARS_OK;
}

void pars_ctx_destroy(pars_ctx* c) {
  if (!c) return;
  cudaSetDevice(c->device);
  cudaStreamSynchronize(c->stream);
  cudaStreamSynchronize(c->copy_stream);
  DevBuf* bufs[] = {&c->text[0], &c->text[1], &c->offs[0], &c->offs[1], &c->scores[0],
                    &c->scores[1], &c->w64, &c->w32, &c->misc, &c->misc2, &c->longl,
                    &c->sort, &c->sgd, &c->pairs_in, &c->dmin_buf, &c->gscratch, &c->lists, &c->plan_buf,
                    &c->baseline, &c->tau};
  for (DevBuf* b : bufs)
    if (b->p) cudaFree(b->p);
  for (HostBuf* b : {&c->h_offs[0], &c->h_offs[1], &c->h_scores, &c->h_text[0], &c->h_text[1]})
    if (b->p) cudaFreeHost(b->p);
  c->pool.reset();
  if (c->tau_exec) cudaGraphExecDestroy(c->tau_exec);
  for (cudaEvent_t e : c->ev_chunk) cudaEventDestroy(e);
  if (c->scratch_ev) cudaEventDestroy(c->scratch_ev);
  for (int k = 0; k < 2; ++k) {
    cudaEventDestroy(c->ev_copy[k]);
    cudaEventDestroy(c->ev_done[k]);
  }
  cudaStreamDestroy(c->stream);
  cudaStreamDestroy(c->copy_stream);
  delete c;
}

int pars_ctx_synchronize(pars_ctx* ctx) {
  PARS_TRY(check_ctx(ctx));
  cudaSetDevice(ctx->device);
  PARS_CUDA_CHECK(cudaStreamSynchronize(ctx->stream));
  return PARS_OK;
}

uint64_t pars_ctx_launches(const pars_ctx* ctx) { return ctx ? ctx->launches.load() : 0; }

int pars_host_alloc(size_t bytes, void** out) {
  PARS_CUDA_CHECK(cudaHostAlloc(out, std::max<size_t>(bytes, 1), cudaHostAllocDefault));
  return PARS_OK;
}
void pars_host_free(void* p) {
  if (p) cudaFreeHost(p);
}

// ---- scoring -------------------------------------------------------------

// Scorer::score_batch fused with extract_features (scorer.cpp:9-24,
// features.cpp:62-122). Host buffers; the text is streamed to the device in
// chunks on a copy stream, overlapped with the kernel of the previous chunk.
namespace {
// The chunked host-buffer scoring pipeline behind pars_score_text and
// pars_score_order: text and offsets stream to the device in ~64 MB chunks on
// the copy stream, overlapped with the previous chunk's kernel; scores go
// either to pinned host staging (h_out) or stay on the device (d_out).
int score_text_pipeline(pars_ctx* ctx, const FeatConfig& cfg, const char* text,
                        const int64_t* offsets, int64_t n, const double* weights, double bias,
                        int mode, double* d_out, double* h_out, std::vector<int64_t>* chunks) {
  cudaStream_t st = ctx->stream, cs = ctx->copy_stream;
  PARS_TRY(upload_weights(ctx, cfg, weights, mode, st));
  // chunk sizes ramp 4 MB -> 64 MB so the first kernel starts after a short
  // first upload (the pipeline fills in ~0.1 ms instead of a full 64 MB copy)
  const int64_t kChunkPrompts = 1 << 18;
  int64_t chunk_bytes = 4ll << 20;
  std::vector<int64_t> starts;
  for (int64_t i = 0; i < n;) {
    starts.push_back(i);
    int64_t j = i + 1;
    while (j < n && j - i < kChunkPrompts && offsets[j + 1] - offsets[i] <= chunk_bytes) ++j;
    i = j;
    chunk_bytes = std::min<int64_t>(chunk_bytes * 2, 64ll << 20);
  }
  starts.push_back(n);
  const int nchunks = (int)starts.size() - 1;
  while ((int)ctx->ev_chunk.size() < nchunks) {
    cudaEvent_t e;
    PARS_CUDA_CHECK(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
    ctx->ev_chunk.push_back(e);
  }
  int64_t max_bytes = 0, max_n = 0;
  for (int k = 0; k < nchunks; ++k) {
    max_bytes = std::max(max_bytes, offsets[starts[k + 1]] - offsets[starts[k]]);
    max_n = std::max(max_n, starts[k + 1] - starts[k]);
  }
  for (int b = 0; b < 2; ++b) {
    PARS_TRY(ensure(ctx->text[b], (size_t)max_bytes + 16));
    PARS_TRY(ensure(ctx->offs[b], (size_t)(max_n + 1) * 8));
    if (!d_out) PARS_TRY(ensure(ctx->scores[b], (size_t)max_n * 8));
    PARS_TRY(ensure_host(ctx->h_offs[b], (size_t)(max_n + 1) * 8));
  }
  // Every copy stays asynchronous (offsets through pinned staging, scores into
  // pinned staging or device memory), so the host never blocks inside the loop.
  for (int k = 0; k < nchunks; ++k) {
    const int b = k & 1;
    const int64_t i0 = starts[k], i1 = starts[k + 1], m = i1 - i0;
    const int64_t t0 = offsets[i0], tb = offsets[i1] - t0;
    if (k >= 2) {
      PARS_CUDA_CHECK(cudaStreamWaitEvent(cs, ctx->ev_done[b], 0));
      PARS_CUDA_CHECK(cudaEventSynchronize(ctx->ev_copy[b]));  // staging b is free again
    }
    std::memcpy(ctx->h_offs[b].p, offsets + i0, (size_t)(m + 1) * 8);
    PARS_CUDA_CHECK(cudaMemcpyAsync(ctx->text[b].p, text + t0, (size_t)tb, cudaMemcpyHostToDevice, cs));
    PARS_CUDA_CHECK(cudaMemcpyAsync(ctx->offs[b].p, ctx->h_offs[b].p, (size_t)(m + 1) * 8,
                                    cudaMemcpyHostToDevice, cs));
    PARS_CUDA_CHECK(cudaEventRecord(ctx->ev_copy[b], cs));
    PARS_CUDA_CHECK(cudaStreamWaitEvent(st, ctx->ev_copy[b], 0));
    // offsets are absolute: shift the device text base so text[offsets[i]] is valid
    const uint8_t* base = static_cast<const uint8_t*>(ctx->text[b].p) - t0;
    double* dst = d_out ? d_out + i0 : (double*)ctx->scores[b].p;
    PARS_TRY(score_chunk(ctx, cfg, mode, base, (const int64_t*)ctx->offs[b].p, m, bias, dst, st));
    if (h_out) {
      PARS_CUDA_CHECK(cudaMemcpyAsync(h_out + i0, dst, (size_t)m * 8, cudaMemcpyDeviceToHost, st));
      PARS_CUDA_CHECK(cudaEventRecord(ctx->ev_chunk[k], st));
    }
    PARS_CUDA_CHECK(cudaEventRecord(ctx->ev_done[b], st));
  }
  *chunks = std::move(starts);
  return PARS_OK;
}

// Hands each chunk's scores from pinned staging to the caller's buffer as
// soon as its copy lands, while later chunks (and the sort) still run.
int drain_scores(pars_ctx* ctx, const std::vector<int64_t>& chunks, const double* h_stage,
                 double* out) {
  for (size_t k = 0; k + 1 < chunks.size(); ++k) {
    PARS_CUDA_CHECK(cudaEventSynchronize(ctx->ev_chunk[k]));
    std::memcpy(out + chunks[k], h_stage + chunks[k], (size_t)(chunks[k + 1] - chunks[k]) * 8);
  }
  return PARS_OK;
}

int check_text_call(const pars_extractor* ex, int64_t n, FeatConfig* cfg, const char* fn) {
  if (!build_feat_config(ex, cfg)) return PARS_ERR_INVALID;
  if (ex->kind != 0) {
    set_error("%s: extractor kind is precomputed_embedding; use pars_score_embeddings", fn);
    return PARS_ERR_INVALID;
  }
  if (n < 0) {
    set_error("negative prompt count");
    return PARS_ERR_INVALID;
  }
  return PARS_OK;
}
}  // namespace

// Scorer::score_batch fused with extract_features (scorer.cpp:9-24,
// features.cpp:62-122). Host buffers.
int pars_score_text(pars_ctx* ctx, const pars_extractor* ex, const char* text,
                    const int64_t* offsets, int64_t n, const double* weights, double bias, int mode,
                    double* scores) {
  PARS_TRY(check_ctx(ctx));
  PARS_TRY(check_mode(mode));
  FeatConfig cfg;
  PARS_TRY(check_text_call(ex, n, &cfg, "pars_score_text"));
  if (n == 0) return PARS_OK;
  Guard g(ctx);
  // a page-locked result buffer takes the per-chunk score copies directly
  const bool pin = is_pinned(scores);
  double* h_sc = scores;
  if (!pin) {
    PARS_TRY(ensure_host(ctx->h_scores, (size_t)n * 8));
    h_sc = static_cast<double*>(ctx->h_scores.p);
  }
  std::vector<int64_t> chunks;
  PARS_TRY(score_text_pipeline(ctx, cfg, text, offsets, n, weights, bias, mode, nullptr, h_sc, &chunks));
  if (!pin) PARS_TRY(drain_scores(ctx, chunks, h_sc, scores));
  PARS_CUDA_CHECK(cudaStreamSynchronize(ctx->stream));
  return PARS_OK;
}

// Scorer::score_batch over records that live in separate (pageable) host
// strings — the reference's Dataset of std::string (scorer.cpp:9-24). Each
// ~64 MB chunk of records is gathered by a pool of host threads straight
// into pinned staging (one host copy, no packing pass), then streams to the
// device while the next chunk is gathered and the previous one is scored.
int pars_score_records(pars_ctx* ctx, const pars_extractor* ex, const char* const* texts,
                       const int64_t* lens, int64_t n, const double* weights, double bias, int mode,
                       double* scores) {
  PARS_TRY(check_ctx(ctx));
  PARS_TRY(check_mode(mode));
  FeatConfig cfg;
  PARS_TRY(check_text_call(ex, n, &cfg, "pars_score_records"));
  if (n == 0) return PARS_OK;
  for (int64_t i = 0; i < n; ++i)
    if (lens[i] < 0 || (lens[i] > 0 && !texts[i])) {
      set_error("pars_score_records: record %lld has no text", (long long)i);
      return PARS_ERR_INVALID;
    }
  Guard g(ctx);
  if (!ctx->pool) {
    const unsigned hc = std::thread::hardware_concurrency();
    ctx->pool.reset(new CopyPool((int)std::max(1u, std::min(hc ? hc : 1u, 16u)) - 1));
  }
  cudaStream_t st = ctx->stream, cs = ctx->copy_stream;
  PARS_TRY(upload_weights(ctx, cfg, weights, mode, st));
  const bool pin = is_pinned(scores);
  double* h_sc = scores;
  if (!pin) {
    PARS_TRY(ensure_host(ctx->h_scores, (size_t)n * 8));
    h_sc = static_cast<double*>(ctx->h_scores.p);
  }
  // chunks: <= 2^18 records and <= 64 MB (ramping from 4 MB)
  const int64_t kChunkPrompts = 1 << 18;
  int64_t chunk_bytes = 4ll << 20;
  std::vector<int64_t> starts;
  int64_t max_bytes = 0, max_n = 0;
  for (int64_t i = 0; i < n;) {
    starts.push_back(i);
    int64_t j = i, bytes = 0;
    while (j < n && j - i < kChunkPrompts && (j == i || bytes + lens[j] <= chunk_bytes)) bytes += lens[j++];
    max_bytes = std::max(max_bytes, bytes);
    max_n = std::max(max_n, j - i);
    i = j;
    chunk_bytes = std::min<int64_t>(chunk_bytes * 2, 64ll << 20);
  }
  starts.push_back(n);
  const int nchunks = (int)starts.size() - 1;
  while ((int)ctx->ev_chunk.size() < nchunks) {
    cudaEvent_t e;
    PARS_CUDA_CHECK(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
    ctx->ev_chunk.push_back(e);
  }
  for (int b = 0; b < 2; ++b) {
    PARS_TRY(ensure(ctx->text[b], (size_t)max_bytes + 16));
    PARS_TRY(ensure(ctx->offs[b], (size_t)(max_n + 1) * 8));
    PARS_TRY(ensure(ctx->scores[b], (size_t)max_n * 8));
    PARS_TRY(ensure_host(ctx->h_offs[b], (size_t)(max_n + 1) * 8));
    PARS_TRY(ensure_host(ctx->h_text[b], (size_t)max_bytes + 16));
  }
  CopyPool& pool = *ctx->pool;
  const int workers = pool.size();
  for (int k = 0; k < nchunks; ++k) {
    const int b = k & 1;
    const int64_t i0 = starts[k], i1 = starts[k + 1], m = i1 - i0;
    if (k >= 2) PARS_CUDA_CHECK(cudaEventSynchronize(ctx->ev_copy[b]));  // staging b is free again
    int64_t* ho = static_cast<int64_t*>(ctx->h_offs[b].p);
    ho[0] = 0;
    for (int64_t i = 0; i < m; ++i) ho[i + 1] = ho[i] + lens[i0 + i];
    char* ht = static_cast<char*>(ctx->h_text[b].p);
    // byte-balanced split of the chunk's records over the pool
    const int64_t tb = ho[m];
    pool.run([&](int w) {
      int64_t a = 0, e = m;
      {  // first record whose start is >= w/workers of the bytes
        const int64_t lo = tb * w / workers, hi = tb * (w + 1) / workers;
        a = std::lower_bound(ho, ho + m, lo) - ho;
        e = std::lower_bound(ho, ho + m, hi) - ho;
        if (w == workers - 1) e = m;
      }
      for (int64_t i = a; i < e; ++i)
        if (lens[i0 + i]) std::memcpy(ht + ho[i], texts[i0 + i], (size_t)lens[i0 + i]);
    });
    if (k >= 2) PARS_CUDA_CHECK(cudaStreamWaitEvent(cs, ctx->ev_done[b], 0));
    PARS_CUDA_CHECK(cudaMemcpyAsync(ctx->text[b].p, ht, (size_t)tb, cudaMemcpyHostToDevice, cs));
    PARS_CUDA_CHECK(cudaMemcpyAsync(ctx->offs[b].p, ho, (size_t)(m + 1) * 8, cudaMemcpyHostToDevice, cs));
    PARS_CUDA_CHECK(cudaEventRecord(ctx->ev_copy[b], cs));
    PARS_CUDA_CHECK(cudaStreamWaitEvent(st, ctx->ev_copy[b], 0));
    double* dst = (double*)ctx->scores[b].p;
    PARS_TRY(score_chunk(ctx, cfg, mode, static_cast<const uint8_t*>(ctx->text[b].p),
                         (const int64_t*)ctx->offs[b].p, m, bias, dst, st));
    PARS_CUDA_CHECK(cudaMemcpyAsync(h_sc + i0, dst, (size_t)m * 8, cudaMemcpyDeviceToHost, st));
    PARS_CUDA_CHECK(cudaEventRecord(ctx->ev_chunk[k], st));
    PARS_CUDA_CHECK(cudaEventRecord(ctx->ev_done[b], st));
  }
  if (!pin) PARS_TRY(drain_scores(ctx, starts, h_sc, scores));
  PARS_CUDA_CHECK(cudaStreamSynchronize(st));
  return PARS_OK;
}

// enqueue (scheduler.cpp:17-31: score every waiting request) + select_batch
// (scheduler.cpp:33-60: full priority order) in one call: the scores never
// leave the device between the two, and both results come back with one
// synchronisation. Host buffers; boosted may be NULL.
int pars_score_order(pars_ctx* ctx, const pars_extractor* ex, const char* text,
                     const int64_t* offsets, int64_t n, const double* weights, double bias,
                     int mode, const uint32_t* tie_rank, const uint8_t* boosted, double* scores,
                     int64_t* order) {
  PARS_TRY(check_ctx(ctx));
  PARS_TRY(check_mode(mode));
  FeatConfig cfg;
  PARS_TRY(check_text_call(ex, n, &cfg, "pars_score_order"));
  if (n == 0) return PARS_OK;
  if (n > 0x7fffffffLL) {
    set_error("priority order: n=%lld exceeds 2^31-1", (long long)n);
    return PARS_ERR_UNSUPPORTED;
  }
  Guard g(ctx);
  cudaStream_t st = ctx->stream;
  // device layout: scores[n] | order64[n] | tie[n] | order[n] | boosted[n]
  PARS_TRY(ensure(ctx->pairs_in, (size_t)n * (8 + 8 + 4 + 4 + 1) + 64));
  double* d_s = (double*)ctx->pairs_in.p;
  int64_t* d_o64 = (int64_t*)(d_s + n);
  uint32_t* d_t = (uint32_t*)(d_o64 + n);
  uint32_t* d_o = d_t + n;
  uint8_t* d_b = (uint8_t*)(d_o + n);
  // page-locked result buffers (a serving loop's, reused across calls) take
  // the device->host copies directly: no staging, no host-side widening
  const bool pin_s = is_pinned(scores), pin_o = is_pinned(order);
  PARS_TRY(ensure(ctx->sort, sort_scratch_bytes(n) + 4096));
  // pinned staging: scores[n] | order[n] (u32) | tie[n] (u32) | boosted[n]
  PARS_TRY(ensure_host(ctx->h_scores, (size_t)n * 17 + 64));
  double* h_sc = static_cast<double*>(ctx->h_scores.p);
  uint32_t* h_o = reinterpret_cast<uint32_t*>(h_sc + n);
  uint32_t* h_t = h_o + n;
  uint8_t* h_b = reinterpret_cast<uint8_t*>(h_t + n);
  std::vector<int64_t> chunks;
  PARS_TRY(score_text_pipeline(ctx, cfg, text, offsets, n, weights, bias, mode, d_s,
                               pin_s ? scores : h_sc, &chunks));
  // the sort keys' tie ranks (and boost flags) follow the text on the copy
  // stream, staged while the last chunks are scored, so the first text chunk
  // is not queued behind them
  cudaStream_t cs = ctx->copy_stream;
  std::memcpy(h_t, tie_rank, (size_t)n * 4);
  PARS_CUDA_CHECK(cudaMemcpyAsync(d_t, h_t, (size_t)n * 4, cudaMemcpyHostToDevice, cs));
  if (boosted) {
    std::memcpy(h_b, boosted, (size_t)n);
    PARS_CUDA_CHECK(cudaMemcpyAsync(d_b, h_b, (size_t)n, cudaMemcpyHostToDevice, cs));
  }
  PARS_CUDA_CHECK(cudaEventRecord(ctx->ev_copy[0], cs));
  PARS_CUDA_CHECK(cudaStreamWaitEvent(st, ctx->ev_copy[0], 0));
  PARS_TRY(launch_priority_sort(ctx, d_s, boosted ? d_b : nullptr, d_t, n, d_o, ctx->sort.p, st));
  if (pin_o) {
    u32_to_i64_kernel<<<(unsigned)ceil_div(n, 256), 256, 0, st>>>(d_o, d_o64, n);
    count_launch(ctx);
    PARS_CUDA_CHECK(cudaMemcpyAsync(order, d_o64, (size_t)n * 8, cudaMemcpyDeviceToHost, st));
  } else {
    PARS_CUDA_CHECK(cudaMemcpyAsync(h_o, d_o, (size_t)n * 4, cudaMemcpyDeviceToHost, st));
  }
  if (!pin_s) PARS_TRY(drain_scores(ctx, chunks, h_sc, scores));  // overlaps the sort
  PARS_CUDA_CHECK(cudaStreamSynchronize(st));
  if (!pin_o)
    for (int64_t i = 0; i < n; ++i) order[i] = h_o[i];
  return PARS_OK;
}

int pars_dev_score_text(pars_ctx* ctx, const pars_extractor* ex, const char* d_text,
                        const int64_t* d_offsets, int64_t n, const double* d_weights, double bias,
                        int mode, double* d_scores, void* stream) {
  PARS_TRY(check_ctx(ctx));
  PARS_TRY(check_mode(mode));
  FeatConfig cfg;
  if (!build_feat_config(ex, &cfg)) return PARS_ERR_INVALID;
  if (n <= 0) return PARS_OK;
  Guard g(ctx);
  cudaStream_t st = pick(ctx, stream);
  PARS_TRY(ensure(ctx->longl, (size_t)n * 4 + 16));
  FeatArgs a{};
  a.text = reinterpret_cast<const uint8_t*>(d_text);
  a.offsets = d_offsets;
  a.n = n;
  a.w64 = d_weights;
  if (mode == PARS_MODE_FAST_F32) {
    PARS_TRY(ensure(ctx->w32, (size_t)cfg.dim * 4));
    ctx->w32_valid = false;  // overwritten with the caller's device weights
    f64_to_f32_kernel<<<(unsigned)ceil_div(cfg.dim, 256), 256, 0, st>>>(d_weights,
                                                                        (float*)ctx->w32.p, cfg.dim);
    count_launch(ctx);
    a.w32 = (const float*)ctx->w32.p;
  }
  a.bias = bias;
  a.scores = d_scores;
  a.long_count = (int32_t*)ctx->longl.p;
  a.long_list = (int32_t*)ctx->longl.p + 4;
  const int fm = mode == PARS_MODE_EXACT_F64 ? kFeatScoreExact : kFeatScoreFast;
  PARS_TRY(attach_scratch(ctx, cfg, fm, n, &a));
  return launch_featurize(ctx, cfg, fm, a, st);
}

int pars_score_embeddings(pars_ctx* ctx, const pars_extractor* ex, const double* X, int64_t n,
                          const double* weights, double bias, int mode, double* scores) {
  PARS_TRY(check_ctx(ctx));
  PARS_TRY(check_mode(mode));
  FeatConfig cfg;
  if (!build_feat_config(ex, &cfg)) return PARS_ERR_INVALID;
  if (n <= 0) return PARS_OK;
  Guard g(ctx);
  cudaStream_t st = ctx->stream;
  PARS_TRY(upload_weights(ctx, cfg, weights, mode, st));
  PARS_TRY(ensure(ctx->misc, (size_t)n * cfg.dim * 8));
  PARS_TRY(ensure(ctx->scores[0], (size_t)n * 8));
  PARS_CUDA_CHECK(cudaMemcpyAsync(ctx->misc.p, X, (size_t)n * cfg.dim * 8, cudaMemcpyHostToDevice, st));
  PARS_TRY(launch_score_dense(ctx, cfg, mode, (const double*)ctx->misc.p, n,
                              (const double*)ctx->w64.p, (const float*)ctx->w32.p, bias,
                              (double*)ctx->scores[0].p, st));
  PARS_CUDA_CHECK(cudaMemcpyAsync(scores, ctx->scores[0].p, (size_t)n * 8, cudaMemcpyDeviceToHost, st));
  PARS_CUDA_CHECK(cudaStreamSynchronize(st));
  return PARS_OK;
}

int pars_dev_score_embeddings(pars_ctx* ctx, const pars_extractor* ex, const double* d_X, int64_t n,
                              const double* d_weights, double bias, int mode, double* d_scores,
                              void* stream) {
  PARS_TRY(check_ctx(ctx));
  PARS_TRY(check_mode(mode));
  FeatConfig cfg;
  if (!build_feat_config(ex, &cfg)) return PARS_ERR_INVALID;
  if (n <= 0) return PARS_OK;
  Guard g(ctx);
  cudaStream_t st = stream ? static_cast<cudaStream_t>(stream) : ctx->stream;
  const float* w32 = nullptr;
  if (mode == PARS_MODE_FAST_F32) {
    PARS_TRY(ensure(ctx->w32, (size_t)cfg.dim * 4));
    ctx->w32_valid = false;  // overwritten with the caller's device weights
    f64_to_f32_kernel<<<(unsigned)ceil_div(cfg.dim, 256), 256, 0, st>>>(d_weights, (float*)ctx->w32.p,
                                                                         cfg.dim);
    count_launch(ctx);
    w32 = (const float*)ctx->w32.p;
  }
  return launch_score_dense(ctx, cfg, mode, d_X, n, d_weights, w32, bias, d_scores, st);
}

// ---- features ------------------------------------------------------------

// extract_all (features.cpp:124-141) into a device-resident CSR.
int pars_extract(pars_ctx* ctx, const pars_extractor* ex, const char* text, const int64_t* offsets,
                 int64_t n, const double* emb, pars_features** out) {
  *out = nullptr;
  PARS_TRY(check_ctx(ctx));
  FeatConfig cfg;
  if (!build_feat_config(ex, &cfg)) return PARS_ERR_INVALID;
  if (n < 0) {
    set_error("negative prompt count");
    return PARS_ERR_INVALID;
  }
  Guard g(ctx);
  cudaStream_t st = ctx->stream;
  auto* f = new pars_features();
  f->ctx = ctx;
  f->device = ctx->device;
  f->dim = cfg.dim;
  f->rows = n;
  f->h_rp.assign((size_t)n + 1, 0);
  auto fail_free = [&](int rc) {
    pars_features_free(f);
    return rc;
  };
  if (ex->kind == 1) {
    if (n > 0 && !emb) {
      set_error("prompt '%s' has no embedding but extractor kind is precomputed_embedding", "?");
      return fail_free(PARS_ERR_INVALID);
    }
    const int64_t nnz = n * (int64_t)cfg.dim;
    for (int64_t i = 0; i <= n; ++i) f->h_rp[i] = i * (int64_t)cfg.dim;
    f->nnz = nnz;
    if (!pool_alloc(ctx, (void**)&f->d_rp, (size_t)(n + 1) * 8) ||
        !pool_alloc(ctx, (void**)&f->d_idx, (size_t)std::max<int64_t>(nnz, 1) * 4) ||
        !pool_alloc(ctx, (void**)&f->d_val, (size_t)std::max<int64_t>(nnz, 1) * 8)) {
      cudaGetLastError();
      set_error("device allocation failed (extract, embeddings)");
      return fail_free(PARS_ERR_OOM);
    }
    if (ensure(ctx->misc, (size_t)std::max<int64_t>(nnz, 1) * 8) != PARS_OK) return fail_free(PARS_ERR_OOM);
    cudaMemcpyAsync(f->d_rp, f->h_rp.data(), (size_t)(n + 1) * 8, cudaMemcpyHostToDevice, st);
    if (n > 0) {
      cudaMemcpyAsync(ctx->misc.p, emb, (size_t)nnz * 8, cudaMemcpyHostToDevice, st);
      dense_csr_kernel<<<(unsigned)ceil_div(n, 128), 128, 0, st>>>(
          (const double*)ctx->misc.p, n, cfg.dim, cfg.norm, f->d_idx, f->d_val);
      count_launch(ctx);
    }
    if (cudaStreamSynchronize(st) != cudaSuccess) {
      set_error("CUDA error in extract (embeddings): %s", cudaGetErrorString(cudaGetLastError()));
      return fail_free(PARS_ERR_CUDA);
    }
    *out = f;
    return PARS_OK;
  }
  // hashed text: per-prompt slots sized by the feature upper bound
  std::vector<int64_t> slot((size_t)n + 1, 0);
  for (int64_t i = 0; i < n; ++i) slot[i + 1] = slot[i] + feat_cap(cfg, offsets[i + 1] - offsets[i]);
  const int64_t cap_total = slot[n];
  const int64_t t0 = n > 0 ? offsets[0] : 0, tb = n > 0 ? offsets[n] - t0 : 0;
  int rc = PARS_OK;
  if ((rc = ensure(ctx->text[0], (size_t)tb + 16)) != PARS_OK ||
      (rc = ensure(ctx->offs[0], (size_t)(n + 1) * 8)) != PARS_OK ||
      (rc = ensure(ctx->misc, (size_t)std::max<int64_t>(cap_total, 1) * 16 + (size_t)(n + 1) * 8 * 2 + 1024)) != PARS_OK ||
      (rc = ensure(ctx->longl, (size_t)std::max<int64_t>(n, 1) * 4 + 16)) != PARS_OK ||
      (rc = ensure(ctx->scores[0], (size_t)std::max<int64_t>(n, 1) * 8)) != PARS_OK)
    return fail_free(rc);
  char* mp = (char*)ctx->misc.p;
  int64_t* d_slot = (int64_t*)mp;
  int64_t* d_rp_tmp = d_slot + (n + 1);
  uint32_t* s_idx = (uint32_t*)(d_rp_tmp + (n + 1));
  double* s_val = (double*)(((uintptr_t)(s_idx + cap_total) + 15) & ~(uintptr_t)15);
  int32_t* s_cnt = (int32_t*)(s_val + cap_total);
  int32_t* d_nnz = (int32_t*)ctx->scores[0].p;
  if (!pool_alloc(ctx, (void**)&f->d_inv, (size_t)std::max<int64_t>(n, 1) * 8)) {
    cudaGetLastError();
    set_error("device allocation failed (extract)");
    return fail_free(PARS_ERR_OOM);
  }
  if (n > 0) {
    cudaMemcpyAsync(ctx->text[0].p, text + t0, (size_t)tb, cudaMemcpyHostToDevice, st);
    cudaMemcpyAsync(ctx->offs[0].p, offsets, (size_t)(n + 1) * 8, cudaMemcpyHostToDevice, st);
    cudaMemcpyAsync(d_slot, slot.data(), (size_t)(n + 1) * 8, cudaMemcpyHostToDevice, st);
    FeatArgs a{};
    a.text = static_cast<const uint8_t*>(ctx->text[0].p) - t0;
    a.offsets = (const int64_t*)ctx->offs[0].p;
    a.n = n;
    a.slot_base = d_slot;
    a.out_idx = s_idx;
    a.out_val = s_val;
    a.out_nnz = d_nnz;
    a.out_cnt = s_cnt;
    a.out_inv = f->d_inv;
    a.long_count = (int32_t*)ctx->longl.p;
    a.long_list = (int32_t*)ctx->longl.p + 4;
    if ((rc = attach_scratch(ctx, cfg, kFeatCsr, n, &a)) != PARS_OK) return fail_free(rc);
    if ((rc = launch_featurize(ctx, cfg, kFeatCsr, a, st)) != PARS_OK) return fail_free(rc);
    std::vector<int32_t> nnz((size_t)n);
    cudaMemcpyAsync(nnz.data(), d_nnz, (size_t)n * 4, cudaMemcpyDeviceToHost, st);
    if (cudaStreamSynchronize(st) != cudaSuccess) {
      set_error("CUDA error in extract: %s", cudaGetErrorString(cudaGetLastError()));
      return fail_free(PARS_ERR_CUDA);
    }
    for (int64_t i = 0; i < n; ++i) f->h_rp[i + 1] = f->h_rp[i] + nnz[i];
  }
  f->nnz = f->h_rp[n];
  if (!pool_alloc(ctx, (void**)&f->d_rp, (size_t)(n + 1) * 8) ||
      !pool_alloc(ctx, (void**)&f->d_idx, (size_t)std::max<int64_t>(f->nnz, 1) * 4) ||
      !pool_alloc(ctx, (void**)&f->d_val, (size_t)std::max<int64_t>(f->nnz, 1) * 8) ||
      !pool_alloc(ctx, (void**)&f->d_cnt, (size_t)std::max<int64_t>(f->nnz, 1) * 4)) {
    cudaGetLastError();
    set_error("device allocation failed (extract)");
    return fail_free(PARS_ERR_OOM);
  }
  cudaMemcpyAsync(f->d_rp, f->h_rp.data(), (size_t)(n + 1) * 8, cudaMemcpyHostToDevice, st);
  if (n > 0) {
    compact_kernel<<<(unsigned)n, 128, 0, st>>>(d_slot, f->d_rp, n, s_idx, s_val, s_cnt, f->d_idx,
                                                f->d_val, f->d_cnt);
    count_launch(ctx);
  }
  if (cudaStreamSynchronize(st) != cudaSuccess) {
    set_error("CUDA error in extract (compact): %s", cudaGetErrorString(cudaGetLastError()));
    return fail_free(PARS_ERR_CUDA);
  }
  *out = f;
  return PARS_OK;
}

int pars_features_upload(pars_ctx* ctx, uint32_t dim, int64_t rows, const int64_t* row_ptr,
                         const uint32_t* idx, const double* val, pars_features** out) {
  *out = nullptr;
  PARS_TRY(check_ctx(ctx));
  Guard g(ctx);
  auto* f = new pars_features();
  f->ctx = ctx;
  f->device = ctx->device;
  f->dim = dim;
  f->rows = rows;
  f->h_rp.assign(row_ptr, row_ptr + rows + 1);
  const int64_t base = row_ptr[0];
  for (auto& r : f->h_rp) r -= base;
  f->nnz = f->h_rp[rows];
  for (int64_t k = 0; k < f->nnz; ++k)
    if (idx[k] >= dim) {
      set_error("feature index %u outside dimension %u", idx[k], dim);
      delete f;
      return PARS_ERR_INVALID;
    }
  if (!pool_alloc(ctx, (void**)&f->d_rp, (size_t)(rows + 1) * 8) ||
      !pool_alloc(ctx, (void**)&f->d_idx, (size_t)std::max<int64_t>(f->nnz, 1) * 4) ||
      !pool_alloc(ctx, (void**)&f->d_val, (size_t)std::max<int64_t>(f->nnz, 1) * 8)) {
    cudaGetLastError();
    set_error("device allocation failed (features upload)");
    delete f;
    return PARS_ERR_OOM;
  }
  cudaMemcpyAsync(f->d_rp, f->h_rp.data(), (size_t)(rows + 1) * 8, cudaMemcpyHostToDevice, ctx->stream);
  cudaMemcpyAsync(f->d_idx, idx, (size_t)f->nnz * 4, cudaMemcpyHostToDevice, ctx->stream);
  cudaMemcpyAsync(f->d_val, val, (size_t)f->nnz * 8, cudaMemcpyHostToDevice, ctx->stream);
  PARS_CUDA_CHECK(cudaStreamSynchronize(ctx->stream));
  *out = f;
  return PARS_OK;
}

int64_t pars_features_rows(const pars_features* f) { return f ? f->rows : -1; }
int64_t pars_features_nnz(const pars_features* f) { return f ? f->nnz : -1; }
int64_t pars_features_dim(const pars_features* f) { return f ? (int64_t)f->dim : -1; }

int pars_features_download(pars_ctx* ctx, const pars_features* f, int64_t* row_ptr, uint32_t* idx,
                           double* val) {
  PARS_TRY(check_ctx(ctx));
  Guard g(ctx);
  std::memcpy(row_ptr, f->h_rp.data(), (size_t)(f->rows + 1) * 8);
  if (f->nnz > 0) {
    PARS_CUDA_CHECK(cudaMemcpyAsync(idx, f->d_idx, (size_t)f->nnz * 4, cudaMemcpyDeviceToHost, ctx->stream));
    PARS_CUDA_CHECK(cudaMemcpyAsync(val, f->d_val, (size_t)f->nnz * 8, cudaMemcpyDeviceToHost, ctx->stream));
  }
  PARS_CUDA_CHECK(cudaStreamSynchronize(ctx->stream));
  return PARS_OK;
}

void pars_features_free(pars_features* f) {
  if (!f) return;
  void* ptrs[] = {f->d_rp,      f->d_idx,     f->d_val,     f->d_cnt,       f->d_inv,
                  f->d_cpk,     f->d_cpk_off, f->d_csc_ptr, f->d_csc_row,   f->d_csc_val,
                  f->d_csc_tasks, f->d_csc_col_task, f->d_csc_part};
  pool_release(f->device, ptrs, 13);
  delete f;
}

int pars_features_score(pars_ctx* ctx, const pars_features* f, const double* weights, double bias,
                        double* scores) {
  PARS_TRY(check_ctx(ctx));
  if (f->rows == 0) return PARS_OK;
  Guard g(ctx);
  cudaStream_t st = ctx->stream;
  PARS_TRY(ensure(ctx->w64, (size_t)f->dim * 8));
  ctx->w64_valid = ctx->w32_valid = false;  // overwritten below
  PARS_TRY(ensure(ctx->scores[0], (size_t)f->rows * 8));
  PARS_CUDA_CHECK(cudaMemcpyAsync(ctx->w64.p, weights, (size_t)f->dim * 8, cudaMemcpyHostToDevice, st));
  csr_score_kernel<<<(unsigned)ceil_div(f->rows, 128), 128, 0, st>>>(
      f->d_rp, f->d_idx, f->d_val, f->rows, (const double*)ctx->w64.p, bias,
      (double*)ctx->scores[0].p);
  count_launch(ctx);
  PARS_CUDA_CHECK(cudaGetLastError());
  PARS_CUDA_CHECK(cudaMemcpyAsync(scores, ctx->scores[0].p, (size_t)f->rows * 8, cudaMemcpyDeviceToHost, st));
  PARS_CUDA_CHECK(cudaStreamSynchronize(st));
  return PARS_OK;
}

// ---- all-pairs -----------------------------------------------------------

int64_t pars_allpairs_tiles(int64_t n) { return allpairs_tile_count(n); }

int pars_allpairs(pars_ctx* ctx, const double* scores, const int64_t* lengths, int64_t n,
                  double delta, double margin, int32_t* coeff, uint64_t* kept, uint64_t* active,
                  double* loss_sum) {
  return pars_allpairs_algo(ctx, scores, lengths, n, delta, margin, PARS_ALLPAIRS_SORTED, coeff,
                            kept, active, loss_sum);
}

int pars_allpairs_algo(pars_ctx* ctx, const double* scores, const int64_t* lengths, int64_t n,
                       double delta, double margin, int algo, int32_t* coeff, uint64_t* kept,
                       uint64_t* active, double* loss_sum) {
  PARS_TRY(check_ctx(ctx));
  if (algo != PARS_ALLPAIRS_SORTED && algo != PARS_ALLPAIRS_GENERAL) {
    set_error("all-pairs: unknown algorithm %d", algo);
    return PARS_ERR_INVALID;
  }
  if (delta < 0.0 || delta >= 1.0) {
    set_error("all-pairs: delta %g outside [0, 1)", delta);
    return PARS_ERR_INVALID;
  }
  *kept = *active = 0;
  *loss_sum = 0.0;
  if (n < 2) {
    if (n == 1) coeff[0] = 0;
    return PARS_OK;
  }
  int64_t max_len = 0;
  std::vector<int32_t> L((size_t)n);
  for (int64_t i = 0; i < n; ++i) {
    if (lengths[i] < 0 || lengths[i] > kMaxLengthTable) {
      set_error("all-pairs: length %lld outside [0, %lld]", (long long)lengths[i],
                (long long)kMaxLengthTable);
      return PARS_ERR_UNSUPPORTED;
    }
    L[i] = (int32_t)lengths[i];
    max_len = std::max<int64_t>(max_len, lengths[i]);
  }
  Guard g(ctx);
  cudaStream_t st = ctx->stream;
  PARS_TRY(ensure_dmin(ctx, delta, max_len, st));
  const int64_t tiles = allpairs_tile_count(n);
  PARS_TRY(ensure(ctx->pairs_in, (size_t)n * 8 + (size_t)n * 4 + (size_t)n * 4 + 64 + (size_t)tiles * 8 + 1024));
  char* p = (char*)ctx->pairs_in.p;
  double* d_s = (double*)p;
  int32_t* d_L = (int32_t*)(d_s + n);
  int32_t* d_c = d_L + n;
  unsigned long long* d_cnt = (unsigned long long*)(((uintptr_t)(d_c + n) + 15) & ~(uintptr_t)15);
  double* d_part = (double*)(d_cnt + 4);
  double* d_loss = d_part + tiles;
  PARS_CUDA_CHECK(cudaMemcpyAsync(d_s, scores, (size_t)n * 8, cudaMemcpyHostToDevice, st));
  PARS_CUDA_CHECK(cudaMemcpyAsync(d_L, L.data(), (size_t)n * 4, cudaMemcpyHostToDevice, st));
  PARS_CUDA_CHECK(cudaMemsetAsync(d_c, 0, (size_t)n * 4, st));
  PARS_CUDA_CHECK(cudaMemsetAsync(d_cnt, 0, 32, st));
  PairPlanDev plan;
  if (algo == PARS_ALLPAIRS_SORTED) {
    PARS_TRY(ensure(ctx->plan_buf, pair_plan_scratch_bytes(n)));
    PARS_TRY(build_pair_plan(ctx, d_L, (const int32_t*)ctx->dmin_buf.p, n, &plan, ctx->plan_buf.p, st));
  }
  if (algo == PARS_ALLPAIRS_SORTED && plan.monotone) {
    PARS_TRY(launch_allpairs_sorted(ctx, plan, d_s, margin, 0, tiles, d_c, d_cnt, d_part, st));
  } else {
    PARS_TRY(launch_allpairs(ctx, d_s, d_L, (const int32_t*)ctx->dmin_buf.p, n, margin, 0, tiles,
                             d_c, d_cnt, d_part, st));
  }
  PARS_TRY(launch_sum_partials(ctx, d_part, tiles, d_loss, st));
  unsigned long long cnt[2];
  PARS_CUDA_CHECK(cudaMemcpyAsync(coeff, d_c, (size_t)n * 4, cudaMemcpyDeviceToHost, st));
  PARS_CUDA_CHECK(cudaMemcpyAsync(cnt, d_cnt, 16, cudaMemcpyDeviceToHost, st));
  PARS_CUDA_CHECK(cudaMemcpyAsync(loss_sum, d_loss, 8, cudaMemcpyDeviceToHost, st));
  PARS_CUDA_CHECK(cudaStreamSynchronize(st));
  *kept = cnt[0];
  *active = cnt[1];
  return PARS_OK;
}

int pars_dev_allpairs(pars_ctx* ctx, const double* d_scores, const int32_t* d_lengths, int64_t n,
                      double delta, double margin, int64_t max_len, int64_t tile_begin,
                      int64_t tile_end, int32_t* d_coeff, unsigned long long* d_counters,
                      double* d_loss_partials, void* stream) {
  PARS_TRY(check_ctx(ctx));
  if (delta < 0.0 || delta >= 1.0) {
    set_error("all-pairs: delta %g outside [0, 1)", delta);
    return PARS_ERR_INVALID;
  }
  if (max_len < 0 || max_len > kMaxLengthTable) {
    set_error("all-pairs: max_len %lld outside [0, %lld]", (long long)max_len,
              (long long)kMaxLengthTable);
    return PARS_ERR_UNSUPPORTED;
  }
  Guard g(ctx);
  cudaStream_t st = pick(ctx, stream);
  PARS_TRY(ensure_dmin(ctx, delta, max_len, st));
  return launch_allpairs(ctx, d_scores, d_lengths, (const int32_t*)ctx->dmin_buf.p, n, margin,
                         tile_begin, tile_end, d_coeff, d_counters, d_loss_partials, st);
}

}  // extern "C"

struct pars_pair_plan {
  pars_ctx* ctx = nullptr;
  int device = 0;
  PairPlanDev dev;
  void* scratch = nullptr;
  int32_t* d_L = nullptr;     // lengths in input order (general-kernel fallback)
  int32_t* d_dmin = nullptr;  // Eq. 1 table for this plan's delta
  int64_t max_len = 0;
  double delta = 0.0;
};

extern "C" {

// Per-dataset plan of the length-sorted all-pairs kernel (lengths do not
// change across training steps; scores do).
int pars_pair_plan_create(pars_ctx* ctx, const int64_t* lengths, int64_t n, double delta,
                          pars_pair_plan** out) {
  *out = nullptr;
  PARS_TRY(check_ctx(ctx));
  if (delta < 0.0 || delta >= 1.0) {
    set_error("all-pairs: delta %g outside [0, 1)", delta);
    return PARS_ERR_INVALID;
  }
  std::vector<int32_t> L((size_t)std::max<int64_t>(n, 1));
  int64_t max_len = 0;
  for (int64_t i = 0; i < n; ++i) {
    if (lengths[i] < 0 || lengths[i] > kMaxLengthTable) {
      set_error("all-pairs: length %lld outside [0, %lld]", (long long)lengths[i],
                (long long)kMaxLengthTable);
      return PARS_ERR_UNSUPPORTED;
    }
    L[i] = (int32_t)lengths[i];
    max_len = std::max<int64_t>(max_len, lengths[i]);
  }
  std::vector<int32_t> table((size_t)max_len + 1);
  PARS_TRY(pars_length_gap_table(delta, max_len, table.data()));
  Guard g(ctx);
  cudaStream_t st = ctx->stream;
  auto* p = new pars_pair_plan();
  p->ctx = ctx;
  p->device = ctx->device;
  p->max_len = max_len;
  p->delta = delta;
  auto fail = [&](int rc) {
    pool_free(ctx, p->scratch);
    pool_free(ctx, p->d_L);
    pool_free(ctx, p->d_dmin);
    delete p;
    return rc;
  };
  if (!pool_alloc(ctx, (void**)&p->scratch, pair_plan_scratch_bytes(n)) ||
      !pool_alloc(ctx, (void**)&p->d_L, L.size() * 4) ||
      !pool_alloc(ctx, (void**)&p->d_dmin, table.size() * 4)) {
    cudaGetLastError();
    set_error("device allocation failed (pair plan)");
    return fail(PARS_ERR_OOM);
  }
  if (cudaMemcpyAsync(p->d_L, L.data(), L.size() * 4, cudaMemcpyHostToDevice, st) != cudaSuccess ||
      cudaMemcpyAsync(p->d_dmin, table.data(), table.size() * 4, cudaMemcpyHostToDevice, st) !=
          cudaSuccess) {
    set_error("CUDA error uploading the pair plan");
    return fail(PARS_ERR_CUDA);
  }
  int rc = build_pair_plan(ctx, p->d_L, p->d_dmin, n, &p->dev, p->scratch, st);
  if (rc != PARS_OK) return fail(rc);
  *out = p;
  return PARS_OK;
}

uint64_t pars_pair_plan_kept(const pars_pair_plan* p) { return p ? p->dev.kept : 0; }
int pars_pair_plan_sorted(const pars_pair_plan* p) { return p && p->dev.monotone ? 1 : 0; }

void pars_pair_plan_free(pars_pair_plan* p) {
  if (!p) return;
  void* ptrs[] = {p->scratch, p->d_L, p->d_dmin};
  pool_release(p->device, ptrs, 3);
  delete p;
}

int pars_dev_allpairs_plan(pars_ctx* ctx, const pars_pair_plan* p, const double* d_scores,
                           double margin, int64_t tile_begin, int64_t tile_end, int32_t* d_coeff,
                           unsigned long long* d_counters, double* d_loss_partials, void* stream) {
  PARS_TRY(check_ctx(ctx));
  if (!p) {
    set_error("null pair plan");
    return PARS_ERR_INVALID;
  }
  Guard g(ctx);
  cudaStream_t st = pick(ctx, stream);
  if (p->dev.monotone)
    return launch_allpairs_sorted(ctx, p->dev, d_scores, margin, tile_begin, tile_end, d_coeff,
                                  d_counters, d_loss_partials, st);
  return launch_allpairs(ctx, d_scores, p->d_L, p->d_dmin, p->dev.n, margin, tile_begin, tile_end,
                         d_coeff, d_counters, d_loss_partials, st);
}

int pars_dev_xt_c(pars_ctx* ctx, const pars_features* f, const int32_t* d_coeff, int64_t row_begin,
                  int64_t row_end, double* d_grad, void* stream) {
  PARS_TRY(check_ctx(ctx));
  Guard g(ctx);
  cudaStream_t st = pick(ctx, stream);
  row_begin = std::max<int64_t>(0, row_begin);
  row_end = std::min<int64_t>(f->rows, row_end);
  if (row_end <= row_begin) {
    PARS_CUDA_CHECK(cudaMemsetAsync(d_grad, 0, (size_t)f->dim * 8, st));
    return PARS_OK;
  }
  if (!f->d_csc_ptr) {  // the transpose, once per feature set
    auto* fm = const_cast<pars_features*>(f);
    if (!pool_alloc(ctx, (void**)&fm->d_csc_ptr, ((size_t)f->dim + 1) * 8) ||
        !pool_alloc(ctx, (void**)&fm->d_csc_row, (size_t)std::max<int64_t>(f->nnz, 1) * 4) ||
        !pool_alloc(ctx, (void**)&fm->d_csc_val, (size_t)std::max<int64_t>(f->nnz, 1) * 8)) {
      set_error("device allocation failed (X^T c transpose)");
      return PARS_ERR_OOM;
    }
    if (st != ctx->stream) PARS_CUDA_CHECK(cudaStreamSynchronize(ctx->stream));  // pool order
    PARS_TRY(ensure(ctx->misc2, csc_scratch_bytes(f->rows, f->dim)));
    PARS_TRY(build_csc(ctx, f->d_rp, f->d_idx, f->d_val, f->rows, f->dim, ctx->misc2.p,
                       fm->d_csc_ptr, fm->d_csc_row, fm->d_csc_val, st));
    // column chunks of <= 1,024 entries: the one-time host table
    std::vector<int64_t> ptr((size_t)f->dim + 1), col_task;
    std::vector<char> tasks;
    PARS_CUDA_CHECK(cudaMemcpyAsync(ptr.data(), fm->d_csc_ptr, ptr.size() * 8, cudaMemcpyDeviceToHost, st));
    PARS_CUDA_CHECK(cudaStreamSynchronize(st));
    fm->csc_ntasks = make_csc_tasks(ptr.data(), f->dim, 1024, tasks, col_task);
    if (!pool_alloc(ctx, &fm->d_csc_tasks, std::max<size_t>(tasks.size(), 16)) ||
        !pool_alloc(ctx, (void**)&fm->d_csc_col_task, col_task.size() * 8) ||
        !pool_alloc(ctx, (void**)&fm->d_csc_part, (size_t)std::max<int64_t>(fm->csc_ntasks, 1) * 8)) {
      set_error("device allocation failed (X^T c tasks)");
      return PARS_ERR_OOM;
    }
    PARS_CUDA_CHECK(cudaMemcpyAsync(fm->d_csc_tasks, tasks.data(), tasks.size(), cudaMemcpyHostToDevice,
                                    ctx->stream));
    PARS_CUDA_CHECK(cudaMemcpyAsync(fm->d_csc_col_task, col_task.data(), col_task.size() * 8,
                                    cudaMemcpyHostToDevice, ctx->stream));
    PARS_CUDA_CHECK(cudaStreamSynchronize(ctx->stream));
  }
  return launch_xtc_csc(ctx, f->d_csc_tasks, f->csc_ntasks, f->d_csc_col_task, f->d_csc_row,
                        f->d_csc_val, d_coeff, row_begin, row_end, f->dim, f->d_csc_part, d_grad, st);
}

}  // extern "C"

// ---- accessors for the data-parallel layer (dp.cu) -------------------------
namespace pars_b200 {
int ctx_device(pars_ctx* ctx) { return ctx->device; }
// (no scratch ordering: dp.cu's own kernels use dp-owned buffers; the ctx
// calls it makes order themselves)
cudaStream_t ctx_stream(pars_ctx* ctx, void* s) { return s ? static_cast<cudaStream_t>(s) : ctx->stream; }
int ctx_merge_rank(pars_ctx* ctx, const double* d_scores, const uint8_t* d_boosted,
                   const uint32_t* d_tie, const uint32_t* d_run_orders, const int64_t* run_offsets,
                   int nruns, int run, uint32_t* d_order, void* stream) {
  capi_detail::Guard g(ctx);
  cudaStream_t st = capi_detail::pick(ctx, stream);
  PARS_TRY(capi_detail::ensure(ctx->sort, merge_runs_scratch_bytes(run_offsets[nruns], nruns) + 4096));
  return launch_merge_rank(ctx, d_scores, d_boosted, d_tie, d_run_orders, run_offsets, nruns, run,
                           d_order, ctx->sort.p, st);
}
int64_t plan_size(const pars_pair_plan* p) { return p ? p->dev.n : 0; }
// Relative cost of each upper-triangle tile for a cost-balanced split: on a
// length-sorted plan a tile whose rows keep no column of it costs a load
// and a reduction (weight 1), any other tile the full column loop (weight
// 64, the measured ratio of instructions); the general kernel's tiles all
// cost the same.
int plan_tile_weights(const pars_pair_plan* p, std::vector<int64_t>* w) {
  if (!p) {
    set_error("null pair plan");
    return PARS_ERR_INVALID;
  }
  const int64_t n = p->dev.n;
  const int64_t T = kPairTile, nt = ceil_div(std::max<int64_t>(n, 0), T);
  w->assign((size_t)(nt * (nt + 1) / 2), 1);
  if (!p->dev.monotone || n == 0) return PARS_OK;
  std::vector<int32_t> f((size_t)n);
  cudaSetDevice(p->device);
  PARS_CUDA_CHECK(cudaMemcpy(f.data(), p->dev.f, (size_t)n * 4, cudaMemcpyDeviceToHost));
  size_t t = 0;
  for (int64_t I = 0; I < nt; ++I) {
    const int64_t fmin = f[(size_t)(I * T)];
    for (int64_t J = I; J < nt; ++J, ++t) {
      const int64_t J0 = J * T, jn = std::min<int64_t>(T, n - J0);
      (*w)[t] = (I == J || fmin < J0 + jn) ? 64 : 1;
    }
  }
  return PARS_OK;
}
}  // namespace pars_b200

extern "C" {

// ---- training ------------------------------------------------------------

namespace pars_b200 {
namespace capi_detail {

// Compact (idx << 16 | count + 2^15) rows for the cluster SGD kernel, built once
// per feature set; -1 when the features are not representable that way.
int ensure_compact(pars_ctx* ctx, pars_features* f, cudaStream_t st) {
  if (f->cpk_state != 0) return PARS_OK;
  f->cpk_state = -1;
  if (!f->d_cnt || !f->d_inv || f->dim > 65536u) return PARS_OK;
  f->h_cpk_off.assign((size_t)f->rows + 1, 0);
  for (int64_t r = 0; r < f->rows; ++r) {
    const int64_t len = f->h_rp[r + 1] - f->h_rp[r];
    const uint64_t next = (uint64_t)f->h_cpk_off[r] + (uint64_t)((len + 3) & ~3ll);
    if (next > 0xffffffffull) return PARS_OK;
    f->h_cpk_off[r + 1] = (uint32_t)next;
  }
  const size_t words = std::max<size_t>(f->h_cpk_off[f->rows], 4);
  if (!pool_alloc(ctx, (void**)&f->d_cpk, words * 4) ||
      !pool_alloc(ctx, (void**)&f->d_cpk_off, f->h_cpk_off.size() * 4 + 16)) {
    cudaGetLastError();
    set_error("device allocation failed (compact rows)");
    return PARS_ERR_OOM;
  }
  int32_t* d_bad = reinterpret_cast<int32_t*>(f->d_cpk_off + f->h_cpk_off.size());
  PARS_CUDA_CHECK(cudaMemcpyAsync(f->d_cpk_off, f->h_cpk_off.data(), f->h_cpk_off.size() * 4,
                                  cudaMemcpyHostToDevice, st));
  PARS_CUDA_CHECK(cudaMemsetAsync(d_bad, 0, 4, st));
  PARS_TRY(build_compact_rows(ctx, f->d_rp, f->d_idx, f->d_cnt, f->rows, f->d_cpk_off, f->d_cpk,
                              d_bad, st));
  int32_t bad = 0;
  PARS_CUDA_CHECK(cudaMemcpyAsync(&bad, d_bad, 4, cudaMemcpyDeviceToHost, st));
  PARS_CUDA_CHECK(cudaStreamSynchronize(st));
  f->cpk_state = bad ? -1 : 1;
  return PARS_OK;
}

int sgd_epoch_impl(pars_ctx* ctx, pars_features* f, const uint32_t* a, const uint32_t* b,
                   const int32_t* y, int64_t npairs, int32_t batch, double lr, double margin,
                   double* d_w, double bias, double* epoch_loss, uint64_t* active,
                   int algo = PARS_SGD_AUTO, double* d_out = nullptr) {
  // d_out (optional, device, 16 bytes): leave {loss, active} there and return
  // without synchronising, so the caller can prepare the next epoch meanwhile
  if (batch < 1 || batch > 32767) {
    set_error("sgd: batch size %d outside [1, 32767]", batch);
    return PARS_ERR_UNSUPPORTED;
  }
  if ((size_t)f->dim * 8 + (size_t)batch * 29 + 64 > 220 * 1024) {
    set_error("sgd: dimension %u too large for the shared-memory weight vector", f->dim);
    return PARS_ERR_UNSUPPORTED;
  }
  cudaStream_t st = ctx->stream;
  *epoch_loss = 0.0;
  *active = 0;
  if (npairs <= 0) {
    if (d_out) PARS_CUDA_CHECK(cudaMemsetAsync(d_out, 0, 16, st));
    return PARS_OK;
  }
  for (int64_t p = 0; p < npairs; ++p)
    if (a[p] >= f->rows || b[p] >= f->rows) {
      set_error("sgd: pair %lld references a row outside [0, %lld)", (long long)p, (long long)f->rows);
      return PARS_ERR_INVALID;
    }
  const int64_t nb = (npairs + batch - 1) / batch;
  std::vector<int64_t> ent_off((size_t)nb + 1, 0);
  for (int64_t q = 0; q < nb; ++q) {
    int64_t s = 0;
    const int64_t p1 = std::min<int64_t>(npairs, (q + 1) * batch);
    for (int64_t p = q * batch; p < p1; ++p)
      s += (f->h_rp[a[p] + 1] - f->h_rp[a[p]]) + (f->h_rp[b[p] + 1] - f->h_rp[b[p]]);
    ent_off[q + 1] = ent_off[q] + s;
  }
  const int64_t total = ent_off[nb];
  PARS_TRY(ensure(ctx->pairs_in, (size_t)npairs * 12 + 64 + 32));
  uint32_t* d_a = (uint32_t*)ctx->pairs_in.p;
  uint32_t* d_b = d_a + npairs;
  int32_t* d_y = (int32_t*)(d_b + npairs);
  double* d_loss = d_out ? d_out : (double*)(((uintptr_t)(d_y + npairs) + 15) & ~(uintptr_t)15);
  unsigned long long* d_act = (unsigned long long*)(d_loss + 1);
  bool cluster = false;
  if (algo != PARS_SGD_SINGLE_CTA && 2 * (int64_t)batch <= 65535 &&
      sgd_cluster_smem(f->dim, batch) <= 227 * 1024) {
    PARS_TRY(ensure_compact(ctx, f, st));
    cluster = f->cpk_state == 1;
  }
  if (algo == PARS_SGD_CLUSTER && !cluster) {
    set_error("sgd: the cluster kernel needs hashed features with dim <= 65536 and batch <= %d",
              32767);
    return PARS_ERR_UNSUPPORTED;
  }
  const size_t sb = (cluster ? sgd_cluster_scratch_bytes(nb, f->dim, total, npairs)
                             : sgd_scratch_bytes(nb, batch, f->dim, total)) + 4096;
  PARS_TRY(ensure(ctx->sgd, sb));
  PARS_CUDA_CHECK(cudaMemcpyAsync(d_a, a, (size_t)npairs * 4, cudaMemcpyHostToDevice, st));
  PARS_CUDA_CHECK(cudaMemcpyAsync(d_b, b, (size_t)npairs * 4, cudaMemcpyHostToDevice, st));
  PARS_CUDA_CHECK(cudaMemcpyAsync(d_y, y, (size_t)npairs * 4, cudaMemcpyHostToDevice, st));
  PARS_CUDA_CHECK(cudaMemcpyAsync(ctx->sgd.p, ent_off.data(), ent_off.size() * 8, cudaMemcpyHostToDevice, st));
  if (cluster) {
    PARS_TRY(launch_sgd_cluster(ctx, f->d_rp, f->d_cpk, f->d_cpk_off, f->d_inv, f->dim, d_a, d_b,
                                d_y, npairs, batch, lr, margin, bias, d_w, d_loss, d_act, total,
                                ctx->sgd.p, st));
  } else {
    PARS_TRY(launch_sgd_epoch(ctx, f->d_rp, f->d_idx, f->d_val, f->dim, d_a, d_b, d_y, npairs,
                              batch, lr, margin, bias, d_w, d_loss, d_act, total, ctx->sgd.p, sb,
                              st));
  }
  if (d_out) return PARS_OK;
  unsigned long long act = 0;
  PARS_CUDA_CHECK(cudaMemcpyAsync(epoch_loss, d_loss, 8, cudaMemcpyDeviceToHost, st));
  PARS_CUDA_CHECK(cudaMemcpyAsync(&act, d_act, 8, cudaMemcpyDeviceToHost, st));
  PARS_CUDA_CHECK(cudaStreamSynchronize(st));
  *active = act;
  return PARS_OK;
}

}  // namespace capi_detail
}  // namespace pars_b200

// Device-resident LinearScorer::score(FeatureVec) over rows [row_begin,
// row_end) of a feature set (features.hpp:31-35 + scorer.cpp:40-42): scores
// land at d_scores[row_begin, row_end). Asynchronous on `stream`.
int pars_dev_features_score(pars_ctx* ctx, const pars_features* f, int64_t row_begin,
                            int64_t row_end, const double* d_weights, double bias, double* d_scores,
                            void* stream) {
  PARS_TRY(check_ctx(ctx));
  row_begin = std::max<int64_t>(0, row_begin);
  row_end = std::min<int64_t>(f->rows, row_end);
  if (row_end <= row_begin) return PARS_OK;
  Guard g(ctx);
  cudaStream_t st = pick(ctx, stream);
  const int64_t m = row_end - row_begin;
  auto* fm = const_cast<pars_features*>(f);
  PARS_TRY(ensure_compact(ctx, fm, st));
  if (f->cpk_state == 1)
  {
    static bool attr = cudaFuncSetAttribute(cpk_score_coop_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                            (int)kCpkSmem) == cudaSuccess;
    if (!attr) {
      set_error("features score: cannot configure the staged score kernel's shared memory");
      return PARS_ERR_CUDA;
    }
    cpk_score_coop_kernel<<<(unsigned)ceil_div(m, kCpkRows), kCpkRows, kCpkSmem, st>>>(
        f->d_rp + row_begin, f->d_cpk, f->d_cpk_off + row_begin, f->d_inv + row_begin, m, d_weights,
        bias, d_scores + row_begin);
  }
  else
    csr_score_kernel<<<(unsigned)ceil_div(m, 128), 128, 0, st>>>(
        f->d_rp + row_begin, f->d_idx, f->d_val, m, d_weights, bias, d_scores + row_begin);
  count_launch(ctx);
  PARS_CUDA_CHECK(cudaGetLastError());
  return PARS_OK;
}


int pars_sgd_epoch(pars_ctx* ctx, const pars_features* f, const uint32_t* a, const uint32_t* b,
                   const int32_t* y, int64_t npairs, int32_t batch, double lr, double margin,
                   double* w, double bias, double* epoch_loss, uint64_t* active) {
  return pars_sgd_epoch_algo(ctx, f, a, b, y, npairs, batch, lr, margin, w, bias, epoch_loss,
                             active, PARS_SGD_AUTO);
}

int pars_sgd_epoch_algo(pars_ctx* ctx, const pars_features* fc, const uint32_t* a,
                        const uint32_t* b, const int32_t* y, int64_t npairs, int32_t batch,
                        double lr, double margin, double* w, double bias, double* epoch_loss,
                        uint64_t* active, int algo) {
  PARS_TRY(check_ctx(ctx));
  if (algo < PARS_SGD_AUTO || algo > PARS_SGD_SINGLE_CTA) {
    set_error("sgd: unknown algorithm %d", algo);
    return PARS_ERR_INVALID;
  }
  pars_features* f = const_cast<pars_features*>(fc);  // compact rows are a lazily built cache
  Guard g(ctx);
  PARS_TRY(ensure(ctx->misc2, (size_t)f->dim * 8));
  double* d_w = (double*)ctx->misc2.p;
  PARS_CUDA_CHECK(cudaMemcpyAsync(d_w, w, (size_t)f->dim * 8, cudaMemcpyHostToDevice, ctx->stream));
  PARS_TRY(sgd_epoch_impl(ctx, f, a, b, y, npairs, batch, lr, margin, d_w, bias, epoch_loss, active,
                          algo));
  PARS_CUDA_CHECK(cudaMemcpyAsync(w, d_w, (size_t)f->dim * 8, cudaMemcpyDeviceToHost, ctx->stream));
  PARS_CUDA_CHECK(cudaStreamSynchronize(ctx->stream));
  return PARS_OK;
}

// train() for Objective::Pairwise (train.cpp:122-166, 212-216).
int pars_train_pairwise(pars_ctx* ctx, const pars_extractor* ex, const char* text,
                        const int64_t* offsets, const int64_t* lengths, int64_t n, double delta,
                        double margin, int32_t epochs, int32_t batch, double lr, uint64_t seed,
                        uint64_t pairs_per_epoch, double* w_out, double* bias_out,
                        double* loss_trace) {
  PARS_TRY(check_ctx(ctx));
  // validate (train.cpp:96-106), same order and messages
  if (epochs < 0) { set_error("train: epochs must be >= 0"); return PARS_ERR_INVALID; }
  if (batch < 1) { set_error("train: batch_size must be >= 1"); return PARS_ERR_INVALID; }
  if (!(lr > 0.0)) { set_error("train: learning_rate must be > 0"); return PARS_ERR_INVALID; }
  if (margin < 0.0) { set_error("train: margin must be >= 0"); return PARS_ERR_INVALID; }
  if (delta < 0.0 || delta >= 1.0) {
    set_error("train: delta %g outside [0, 1)", delta);
    return PARS_ERR_INVALID;
  }
  if (pairs_per_epoch < 1) { set_error("train: pairs_per_epoch must be >= 1"); return PARS_ERR_INVALID; }
  if (n <= 0) { set_error("train: empty dataset"); return PARS_ERR_INVALID; }
  pars_features* f = nullptr;
  PARS_TRY(pars_extract(ctx, ex, text, offsets, n, nullptr, &f));
  const uint32_t dim = ex->dim;
  int rc = PARS_OK;
  {
    Guard g(ctx);
    cudaStream_t st = ctx->stream;
    rc = ensure(ctx->misc2, (size_t)dim * 8);
    double* d_w = (double*)ctx->misc2.p;
    if (rc == PARS_OK) rc = cudaMemsetAsync(d_w, 0, (size_t)dim * 8, st) == cudaSuccess ? PARS_OK : PARS_ERR_CUDA;
    std::vector<uint32_t> pa(pairs_per_epoch), pb(pairs_per_epoch);
    std::vector<int32_t> py(pairs_per_epoch);
    // each epoch is enqueued without a sync; the next epoch's pairs are drawn
    // on the host while it runs. Losses are checked in epoch order at the end
    // (an epoch after a diverged one only costs time: the error is the same)
    std::vector<int64_t> npe((size_t)std::max(epochs, 0), 0);
    double* d_out = nullptr;
    if (rc == PARS_OK && epochs > 0 && !pool_alloc(ctx, (void**)&d_out, (size_t)epochs * 16)) {
      set_error("device allocation failed (loss slots)");
      rc = PARS_ERR_OOM;
    }
    int done_epochs = 0;
    for (int e = 0; e < epochs && rc == PARS_OK; ++e) {
      const uint64_t es = splitmix64(seed ^ splitmix64(0x10000u + (uint64_t)e));  // derive_seed
      const int64_t np = pars_build_pairs(lengths, n, delta, pairs_per_epoch, es, pa.data(),
                                          pb.data(), py.data(), nullptr);
      if (np < 0) {
        rc = (int)np;
        break;
      }
      double el = 0.0;
      uint64_t act = 0;
      rc = sgd_epoch_impl(ctx, f, pa.data(), pb.data(), py.data(), np, batch, lr, margin, d_w, 0.0,
                          &el, &act, PARS_SGD_AUTO, d_out + 2 * e);
      npe[e] = np;
      if (rc == PARS_OK) done_epochs = e + 1;
    }
    if (done_epochs > 0) {
      std::vector<double> out((size_t)done_epochs * 2);
      if (cudaMemcpyAsync(out.data(), d_out, out.size() * 8, cudaMemcpyDeviceToHost, st) != cudaSuccess ||
          cudaStreamSynchronize(st) != cudaSuccess) {
        set_error("CUDA error reading epoch losses");
        rc = PARS_ERR_CUDA;
      } else {
        const int rc_later = rc;  // a failure after the last enqueued epoch
        const std::string err_later = rc_later == PARS_OK ? "" : pars_last_error();
        rc = PARS_OK;
        for (int e = 0; e < done_epochs; ++e) {
          const double mean = out[2 * e] / (double)npe[e];
          if (!std::isfinite(mean)) {
            set_error("training diverged at epoch %d", e);
            rc = PARS_ERR_INVALID;
            break;
          }
          loss_trace[e] = mean;
        }
        if (rc == PARS_OK && rc_later != PARS_OK) {
          set_error("%s", err_later.c_str());
          rc = rc_later;
        }
      }
    }
    if (d_out) pool_free(ctx, d_out);
    if (rc == PARS_OK) {
      if (cudaMemcpyAsync(w_out, d_w, (size_t)dim * 8, cudaMemcpyDeviceToHost, st) != cudaSuccess ||
          cudaStreamSynchronize(st) != cudaSuccess) {
        set_error("CUDA error reading trained weights");
        rc = PARS_ERR_CUDA;
      }
    }
  }
  *bias_out = 0.0;  // pairwise bias gradient cancels (train.hpp:41-43)
  pars_features_free(f);
  return rc;
}

// ---- comparison objectives (train.cpp:46-94, :168-205) ---------------------

namespace pars_b200 {
namespace capi_detail {

// One PointwiseL1 (kind 0) or ListMLE (kind 1) epoch on the device weights
// d_w. rows[s] is the feature row of slot s; a batch is `batch` samples
// (kind 0) or `batch` lists of k consecutive slots (kind 1). *bias in/out.
int baseline_epoch_impl(pars_ctx* ctx, pars_features* f, int kind, const uint32_t* rows,
                        int64_t nslots, int32_t k, int32_t batch, const double* d_target,
                        double lr, double* d_w, double* bias, double* epoch_loss) {
  const char* who = kind ? "listmle" : "pointwise";
  if (batch < 1) {
    set_error("train: batch_size must be >= 1");
    return PARS_ERR_INVALID;
  }
  if (kind && k < 2) {
    set_error("listmle: list needs >= 2 items");
    return PARS_ERR_INVALID;
  }
  *epoch_loss = 0.0;
  if (nslots <= 0) return PARS_OK;
  if (kind && nslots % k) {
    set_error("listmle: %lld rows are not whole lists of %d", (long long)nslots, k);
    return PARS_ERR_INVALID;
  }
  const int64_t spb = (int64_t)batch * (kind ? k : 1);
  if (baseline_smem_bytes(f->dim, std::min<int64_t>(spb, nslots)) > 227 * 1024) {
    set_error("%s: %lld slots per batch at dim %u exceed the shared-memory step state", who,
              (long long)spb, f->dim);
    return PARS_ERR_UNSUPPORTED;
  }
  for (int64_t s = 0; s < nslots; ++s)
    if (rows[s] >= f->rows) {
      set_error("%s: slot %lld references a row outside [0, %lld)", who, (long long)s,
                (long long)f->rows);
      return PARS_ERR_INVALID;
    }
  const int64_t nb = (nslots + spb - 1) / spb;
  std::vector<int64_t> soff((size_t)nb + 1), ent_off((size_t)nb + 1, 0);
  int64_t max_slots = 0;
  for (int64_t q = 0; q <= nb; ++q) soff[q] = std::min(nslots, q * spb);
  for (int64_t q = 0; q < nb; ++q) {
    int64_t e = 0;
    for (int64_t s = soff[q]; s < soff[q + 1]; ++s) e += f->h_rp[rows[s] + 1] - f->h_rp[rows[s]];
    ent_off[q + 1] = ent_off[q] + e;
    max_slots = std::max(max_slots, soff[q + 1] - soff[q]);
  }
  cudaStream_t st = ctx->stream;
  PARS_TRY(ensure(ctx->sgd, baseline_scratch_bytes(nb, nslots, f->dim, ent_off[nb]) + 4096));
  PARS_TRY(ensure(ctx->pairs_in, 64));
  double* d_out = (double*)ctx->pairs_in.p;  // {loss, bias}
  PARS_TRY(launch_baseline_epoch(ctx, kind, f->d_rp, f->d_idx, f->d_val, f->dim, rows, soff.data(),
                                 nb, k, d_target, lr, *bias, max_slots, ent_off.data(), d_w,
                                 d_out + 1, d_out, ctx->sgd.p, st));
  double out[2];
  PARS_CUDA_CHECK(cudaMemcpyAsync(out, d_out, 16, cudaMemcpyDeviceToHost, st));
  PARS_CUDA_CHECK(cudaStreamSynchronize(st));
  *epoch_loss = out[0];
  *bias = out[1];
  return PARS_OK;
}

// target[r] = pointwise_target(output_len[r]) = log1p(len) (train.cpp:30-32),
// evaluated with the host libm the reference uses, onto the device.
int upload_targets(pars_ctx* ctx, const int64_t* lengths, int64_t n, double** d_target) {
  std::vector<double> t((size_t)n);
  for (int64_t i = 0; i < n; ++i) t[i] = std::log1p(static_cast<double>(lengths[i]));
  PARS_TRY(ensure(ctx->baseline, (size_t)n * 8 + 64));
  *d_target = (double*)ctx->baseline.p;
  PARS_CUDA_CHECK(cudaMemcpyAsync(*d_target, t.data(), (size_t)n * 8, cudaMemcpyHostToDevice,
                                  ctx->stream));
  PARS_CUDA_CHECK(cudaStreamSynchronize(ctx->stream));
  return PARS_OK;
}

}  // namespace capi_detail
}  // namespace pars_b200

int pars_pointwise_epoch(pars_ctx* ctx, const pars_features* fc, const uint32_t* order, int64_t n,
                         const double* target, int32_t batch, double lr, double* w, double* bias,
                         double* epoch_loss) {
  PARS_TRY(check_ctx(ctx));
  pars_features* f = const_cast<pars_features*>(fc);
  Guard g(ctx);
  cudaStream_t st = ctx->stream;
  PARS_TRY(ensure(ctx->misc2, (size_t)f->dim * 8));
  PARS_TRY(ensure(ctx->baseline, (size_t)f->rows * 8 + 64));
  double* d_w = (double*)ctx->misc2.p;
  double* d_t = (double*)ctx->baseline.p;
  PARS_CUDA_CHECK(cudaMemcpyAsync(d_w, w, (size_t)f->dim * 8, cudaMemcpyHostToDevice, st));
  PARS_CUDA_CHECK(cudaMemcpyAsync(d_t, target, (size_t)f->rows * 8, cudaMemcpyHostToDevice, st));
  PARS_TRY(baseline_epoch_impl(ctx, f, 0, order, n, 1, batch, d_t, lr, d_w, bias, epoch_loss));
  PARS_CUDA_CHECK(cudaMemcpyAsync(w, d_w, (size_t)f->dim * 8, cudaMemcpyDeviceToHost, st));
  PARS_CUDA_CHECK(cudaStreamSynchronize(st));
  return PARS_OK;
}

int pars_listmle_epoch(pars_ctx* ctx, const pars_features* fc, const uint32_t* lists,
                       int64_t nlists, int32_t k, int32_t batch, double lr, double* w, double bias,
                       double* epoch_loss) {
  PARS_TRY(check_ctx(ctx));
  pars_features* f = const_cast<pars_features*>(fc);
  Guard g(ctx);
  cudaStream_t st = ctx->stream;
  PARS_TRY(ensure(ctx->misc2, (size_t)f->dim * 8));
  double* d_w = (double*)ctx->misc2.p;
  PARS_CUDA_CHECK(cudaMemcpyAsync(d_w, w, (size_t)f->dim * 8, cudaMemcpyHostToDevice, st));
  double b = bias;
  PARS_TRY(baseline_epoch_impl(ctx, f, 1, lists, nlists * k, k, batch, nullptr, lr, d_w, &b,
                               epoch_loss));
  PARS_CUDA_CHECK(cudaMemcpyAsync(w, d_w, (size_t)f->dim * 8, cudaMemcpyDeviceToHost, st));
  PARS_CUDA_CHECK(cudaStreamSynchronize(st));
  return PARS_OK;
}

// train() for Objective::PointwiseL1 / ListwiseListMLE (train.cpp:122-216).
int pars_train_baseline(pars_ctx* ctx, const pars_extractor* ex, const char* text,
                        const int64_t* offsets, const int64_t* lengths, const char* ids,
                        const int64_t* id_offsets, int64_t n, int32_t objective, int32_t epochs,
                        int32_t batch, double lr, uint64_t seed, uint64_t lists_per_epoch,
                        int32_t list_size, double* w_out, double* bias_out, double* loss_trace) {
  PARS_TRY(check_ctx(ctx));
  if (objective != PARS_OBJ_POINTWISE_L1 && objective != PARS_OBJ_LISTMLE) {
    set_error("train_baseline: objective %d is not pointwise_l1 or listwise_listmle", objective);
    return PARS_ERR_INVALID;
  }
  if (epochs < 0) { set_error("train: epochs must be >= 0"); return PARS_ERR_INVALID; }
  if (batch < 1) { set_error("train: batch_size must be >= 1"); return PARS_ERR_INVALID; }
  if (!(lr > 0.0)) { set_error("train: learning_rate must be > 0"); return PARS_ERR_INVALID; }
  if (lists_per_epoch < 1) { set_error("train: lists_per_epoch must be >= 1"); return PARS_ERR_INVALID; }
  if (list_size < 2) { set_error("train: list_size must be >= 2"); return PARS_ERR_INVALID; }
  if (n <= 0) { set_error("train: empty dataset"); return PARS_ERR_INVALID; }
  const bool listwise = objective == PARS_OBJ_LISTMLE;
  if (listwise && n < 2) { set_error("train: listwise needs >= 2 records"); return PARS_ERR_INVALID; }
  pars_features* f = nullptr;
  PARS_TRY(pars_extract(ctx, ex, text, offsets, n, nullptr, &f));
  const uint32_t dim = ex->dim;
  int rc = PARS_OK;
  double bias = 0.0;
  {
    Guard g(ctx);
    cudaStream_t st = ctx->stream;
    rc = ensure(ctx->misc2, (size_t)dim * 8);
    double* d_w = (double*)ctx->misc2.p;
    if (rc == PARS_OK)
      rc = cudaMemsetAsync(d_w, 0, (size_t)dim * 8, st) == cudaSuccess ? PARS_OK : PARS_ERR_CUDA;
    double* d_t = nullptr;
    if (rc == PARS_OK && !listwise) rc = upload_targets(ctx, lengths, n, &d_t);
    const int32_t k = (int32_t)std::min<int64_t>(list_size, n);
    std::vector<uint32_t> rows(listwise ? (size_t)lists_per_epoch * k : (size_t)n);
    for (int e = 0; e < epochs && rc == PARS_OK; ++e) {
      const uint64_t es = splitmix64(seed ^ splitmix64(0x10000u + (uint64_t)e));  // derive_seed
      rc = listwise ? pars_listmle_lists(lengths, ids, id_offsets, n, (int64_t)lists_per_epoch,
                                         list_size, es, rows.data())
                    : pars_pointwise_order(n, es, rows.data());
      if (rc != PARS_OK) break;
      double el = 0.0;
      rc = baseline_epoch_impl(ctx, f, listwise ? 1 : 0, rows.data(), (int64_t)rows.size(), k,
                               batch, d_t, lr, d_w, &bias, &el);
      if (rc != PARS_OK) break;
      const double mean = el / (double)(listwise ? (int64_t)lists_per_epoch : n);
      if (!std::isfinite(mean)) {
        set_error("training diverged at epoch %d", e);
        rc = PARS_ERR_INVALID;
        break;
      }
      loss_trace[e] = mean;
    }
    if (rc == PARS_OK) {
      if (cudaMemcpyAsync(w_out, d_w, (size_t)dim * 8, cudaMemcpyDeviceToHost, st) != cudaSuccess ||
          cudaStreamSynchronize(st) != cudaSuccess) {
        set_error("CUDA error reading trained weights");
        rc = PARS_ERR_CUDA;
      }
    }
  }
  *bias_out = bias;
  pars_features_free(f);
  return rc;
}

// ---- priority ordering (scheduler.cpp:33-60) -------------------------------

int pars_priority_order(pars_ctx* ctx, const double* scores, const uint8_t* boosted,
                        const uint32_t* tie_rank, int64_t n, int64_t* order) {
  PARS_TRY(check_ctx(ctx));
  if (n <= 0) return PARS_OK;
  Guard g(ctx);
  cudaStream_t st = ctx->stream;
  PARS_TRY(ensure(ctx->pairs_in, (size_t)n * (8 + 1 + 4 + 4) + 64));
  double* d_s = (double*)ctx->pairs_in.p;
  uint32_t* d_t = (uint32_t*)(d_s + n);
  uint32_t* d_o = d_t + n;
  uint8_t* d_b = (uint8_t*)(d_o + n);
  PARS_TRY(ensure(ctx->sort, sort_scratch_bytes(n) + 4096));
  PARS_CUDA_CHECK(cudaMemcpyAsync(d_s, scores, (size_t)n * 8, cudaMemcpyHostToDevice, st));
  PARS_CUDA_CHECK(cudaMemcpyAsync(d_t, tie_rank, (size_t)n * 4, cudaMemcpyHostToDevice, st));
  if (boosted) PARS_CUDA_CHECK(cudaMemcpyAsync(d_b, boosted, (size_t)n, cudaMemcpyHostToDevice, st));
  PARS_TRY(launch_priority_sort(ctx, d_s, boosted ? d_b : nullptr, d_t, n, d_o, ctx->sort.p, st));
  std::vector<uint32_t> o((size_t)n);
  PARS_CUDA_CHECK(cudaMemcpyAsync(o.data(), d_o, (size_t)n * 4, cudaMemcpyDeviceToHost, st));
  PARS_CUDA_CHECK(cudaStreamSynchronize(st));
  for (int64_t i = 0; i < n; ++i) order[i] = o[i];
  return PARS_OK;
}

int pars_dev_priority_order(pars_ctx* ctx, const double* d_scores, const uint8_t* d_boosted,
                            const uint32_t* d_tie, int64_t n, uint32_t* d_order, void* stream) {
  PARS_TRY(check_ctx(ctx));
  if (n <= 0) return PARS_OK;
  Guard g(ctx);
  cudaStream_t st = pick(ctx, stream);
  PARS_TRY(ensure(ctx->sort, sort_scratch_bytes(n) + 4096));
  return launch_priority_sort(ctx, d_scores, d_boosted, d_tie, n, d_order, ctx->sort.p, st);
}

// select_batch order of all prompts from the orders of contiguous shards
// (each from pars_dev_priority_order on its own range): the sharded-scoring
// path's global SJF order without re-sorting everything.
int pars_dev_merge_orders(pars_ctx* ctx, const double* d_scores, const uint8_t* d_boosted,
                          const uint32_t* d_tie, const uint32_t* d_run_orders,
                          const int64_t* run_offsets, int nruns, uint32_t* d_order, void* stream) {
  PARS_TRY(check_ctx(ctx));
  if (nruns < 1 || run_offsets[0] != 0) {
    set_error("merge_orders: need >= 1 run starting at offset 0");
    return PARS_ERR_INVALID;
  }
  for (int r = 0; r < nruns; ++r)
    if (run_offsets[r + 1] < run_offsets[r]) {
      set_error("merge_orders: run offsets must be non-decreasing");
      return PARS_ERR_INVALID;
    }
  const int64_t n = run_offsets[nruns];
  if (n <= 0) return PARS_OK;
  Guard g(ctx);
  cudaStream_t st = pick(ctx, stream);
  PARS_TRY(ensure(ctx->sort, std::max(sort_scratch_bytes(n), merge_runs_scratch_bytes(n, nruns)) + 4096));
  return launch_merge_runs(ctx, d_scores, d_boosted, d_tie, d_run_orders, run_offsets, nruns, n,
                           d_order, ctx->sort.p, st);
}

// ---- Kendall tau-b (metrics.cpp:13-64) -----------------------------------

namespace pars_b200 {
namespace capi_detail {

// The sorted counts' device steps replayed from a CUDA graph captured on
// the first call with these inputs and scratch (launch gaps of ~30 dependent
// kernels are most of the call at n <= 10^5), then the one read-back.
int tau_sorted_graph(pars_ctx* ctx, const double* d_x, const double* d_y, int64_t n, uint64_t* c4,
                     cudaStream_t st) {
  void* scr = ctx->tau.p;
  if (!ctx->tau_exec || ctx->tau_key[0] != d_x || ctx->tau_key[1] != d_y ||
      ctx->tau_key[2] != scr || ctx->tau_key_n != n) {
    if (ctx->tau_exec) cudaGraphExecDestroy(ctx->tau_exec);
    ctx->tau_exec = nullptr;
    ctx->tau_key_n = -1;
    const uint64_t before = ctx->launches.load();
    PARS_CUDA_CHECK(cudaStreamBeginCapture(st, cudaStreamCaptureModeThreadLocal));
    const int rc = enqueue_tau_sorted(ctx, d_x, d_y, n, scr, st);
    cudaGraph_t g = nullptr;
    const cudaError_t ce = cudaStreamEndCapture(st, &g);
    if (rc != PARS_OK) {
      if (g) cudaGraphDestroy(g);
      return rc;
    }
    if (ce != cudaSuccess) {
      set_error("kendall_tau_b: graph capture failed: %s", cudaGetErrorString(ce));
      return PARS_ERR_CUDA;
    }
    const cudaError_t ie = cudaGraphInstantiate(&ctx->tau_exec, g, 0);
    cudaGraphDestroy(g);
    if (ie != cudaSuccess) {
      ctx->tau_exec = nullptr;
      set_error("kendall_tau_b: graph instantiation failed: %s", cudaGetErrorString(ie));
      return PARS_ERR_CUDA;
    }
    ctx->tau_launches = ctx->launches.load() - before;  // counted at replay
    ctx->launches.fetch_sub(ctx->tau_launches);
    ctx->tau_key[0] = d_x;
    ctx->tau_key[1] = d_y;
    ctx->tau_key[2] = scr;
    ctx->tau_key_n = n;
  }
  PARS_CUDA_CHECK(cudaGraphLaunch(ctx->tau_exec, st));
  count_launch(ctx, ctx->tau_launches);
  return finish_tau_sorted(n, c4, scr, st);
}

// tau-b of device arrays on `st`: the O(n log n) sorted counts (tau_sorted.cu)
// unless an input is non-finite (or algo asks for it), else the all-pairs
// tiles (pairs.cu). Both give the reference's exact integers.
int kendall_dev_impl(pars_ctx* ctx, const double* d_x, const double* d_y, int64_t n,
                     uint64_t* counts, double* tau_b, int algo, cudaStream_t st) {
  if (n < 2) {
    set_error("kendall_tau_b: need at least 2 items, got %zu", (size_t)n);
    return PARS_ERR_INVALID;
  }
  if (algo < PARS_TAU_AUTO || algo > PARS_TAU_PAIRS) {
    set_error("kendall_tau_b: unknown algorithm %d", algo);
    return PARS_ERR_INVALID;
  }
  uint64_t c4[4] = {0, 0, 0, 0};
  int rc = PARS_ERR_UNSUPPORTED;
  if (algo != PARS_TAU_PAIRS) {
    PARS_TRY(ensure(ctx->tau, tau_sorted_scratch_bytes(n) + 4096));
    rc = capturing(st) ? launch_tau_sorted(ctx, d_x, d_y, n, c4, ctx->tau.p, st)
                       : tau_sorted_graph(ctx, d_x, d_y, n, c4, st);
    if (rc != PARS_OK && rc != PARS_ERR_UNSUPPORTED) return rc;
    if (rc == PARS_ERR_UNSUPPORTED && algo == PARS_TAU_SORTED) {
      set_error("kendall_tau_b: the sorted algorithm needs finite inputs");
      return PARS_ERR_UNSUPPORTED;
    }
  }
  if (rc != PARS_OK) {
    PARS_TRY(ensure(ctx->tau, 64));
    unsigned long long* d_c = (unsigned long long*)ctx->tau.p;
    PARS_CUDA_CHECK(cudaMemsetAsync(d_c, 0, 32, st));
    PARS_TRY(launch_tau(ctx, d_x, d_y, n, d_c, st));
    unsigned long long c[4];
    PARS_CUDA_CHECK(cudaMemcpyAsync(c, d_c, 32, cudaMemcpyDeviceToHost, st));
    PARS_CUDA_CHECK(cudaStreamSynchronize(st));
    for (int k = 0; k < 4; ++k) c4[k] = c[k];
  }
  return pars_kendall_finish(c4, n, counts, tau_b);
}

}  // namespace capi_detail
}  // namespace pars_b200

int pars_kendall_tau(pars_ctx* ctx, const double* x, const double* y, int64_t n, uint64_t* counts,
                     double* tau_b) {
  return pars_kendall_tau_algo(ctx, x, y, n, counts, tau_b, PARS_TAU_AUTO);
}

int pars_kendall_tau_algo(pars_ctx* ctx, const double* x, const double* y, int64_t n,
                          uint64_t* counts, double* tau_b, int algo) {
  PARS_TRY(check_ctx(ctx));
  if (n < 2) {
    set_error("kendall_tau_b: need at least 2 items, got %zu", (size_t)n);
    return PARS_ERR_INVALID;
  }
  Guard g(ctx);
  cudaStream_t st = ctx->stream;
  PARS_TRY(ensure(ctx->pairs_in, (size_t)n * 16 + 64));
  double* d_x = (double*)ctx->pairs_in.p;
  double* d_y = d_x + n;
  PARS_CUDA_CHECK(cudaMemcpyAsync(d_x, x, (size_t)n * 8, cudaMemcpyHostToDevice, st));
  PARS_CUDA_CHECK(cudaMemcpyAsync(d_y, y, (size_t)n * 8, cudaMemcpyHostToDevice, st));
  return kendall_dev_impl(ctx, d_x, d_y, n, counts, tau_b, algo, st);
}

int pars_dev_kendall_tau(pars_ctx* ctx, const double* d_x, const double* d_y, int64_t n,
                         uint64_t* counts, double* tau_b, void* stream) {
  PARS_TRY(check_ctx(ctx));
  Guard g(ctx);
  return kendall_dev_impl(ctx, d_x, d_y, n, counts, tau_b, PARS_TAU_AUTO, pick(ctx, stream));
}

// finish_tau (metrics.cpp:13-32) on counts {n_c, n_d, n1, n2} of all pairs
int pars_kendall_finish(const uint64_t* c, int64_t n, uint64_t* counts, double* tau_b) {
  const uint64_t n0 = (uint64_t)n * (uint64_t)(n - 1) / 2;
  counts[0] = c[0];
  counts[1] = c[1];
  counts[2] = n0;
  counts[3] = c[2];
  counts[4] = c[3];
  if (c[2] == n0) {
    set_error("degenerate ranking: all values tied in first argument");
    return PARS_ERR_INVALID;
  }
  if (c[3] == n0) {
    set_error("degenerate ranking: all values tied in second argument");
    return PARS_ERR_INVALID;
  }
  const double denom = std::sqrt(static_cast<double>(n0 - c[2]) * static_cast<double>(n0 - c[3]));
  const double tau = (static_cast<double>(c[0]) - static_cast<double>(c[1])) / denom;
  *tau_b = std::clamp(tau, -1.0, 1.0);
  return PARS_OK;
}

int64_t pars_kendall_tiles(int64_t n) { return allpairs_tile_count(n); }

int pars_dev_kendall_counts(pars_ctx* ctx, const double* d_x, const double* d_y, int64_t n,
                            int64_t tile_begin, int64_t tile_end, unsigned long long* d_counts,
                            void* stream) {
  PARS_TRY(check_ctx(ctx));
  if (n < 2) return PARS_OK;
  Guard g(ctx);
  return launch_tau(ctx, d_x, d_y, n, d_counts, pick(ctx, stream), tile_begin, tile_end);
}

}  // extern "C"

// ---- dataset ingestion (load_dataset, dataset.cpp:73-173) -----------------

struct pars_dataset {
  pars_ctx* ctx = nullptr;
  int device = 0;
  int64_t n = 0, text_bytes = 0, id_bytes = 0, embedding_dim = 0;
  uint8_t* d_text = nullptr;     // decoded prompts, concatenated
  int64_t* d_offsets = nullptr;  // [n+1]
  uint8_t* d_ids = nullptr;
  int64_t* d_id_offsets = nullptr;
  int64_t* d_output_len = nullptr;
  int64_t* d_prompt_len = nullptr;
  std::vector<int64_t> samples_rp, samples;  // host CSR of output_len_samples
};

namespace {
using namespace pars_b200;

int ds_fail(const char* path, int64_t line, const std::string& msg) {
  set_error("%s: line %lld: %s", path, (long long)line, msg.c_str());
  return PARS_ERR_INVALID;
}
}  // namespace

extern "C" {

int pars_load_dataset_bytes(pars_ctx* ctx, const char* path, const char* bytes, int64_t nbytes,
                            int64_t limit, pars_dataset** out) {
  *out = nullptr;
  PARS_TRY(check_ctx(ctx));
  if (!path) path = "<bytes>";
  if (nbytes <= 0) {
    set_error("%s: empty file, missing header", path);
    return PARS_ERR_INVALID;
  }
  // header line (host): the reference's checks with the same JSON library
  const char* nlp = static_cast<const char*>(std::memchr(bytes, '\n', (size_t)nbytes));
  const int64_t hlen = nlp ? (int64_t)(nlp - bytes) : nbytes;
  int64_t emb_dim = 0;
  const std::string herr = ingest_header_error(std::string(bytes, (size_t)hlen), &emb_dim);
  if (!herr.empty()) return ds_fail(path, 1, herr);
  const char* body = nlp ? nlp + 1 : bytes + nbytes;
  const int64_t nb = nbytes - (int64_t)(body - bytes);
  if (limit < 0) limit = INT64_MAX;
  Guard g(ctx);
  cudaStream_t st = ctx->stream;
  auto* d = new pars_dataset();
  d->ctx = ctx;
  d->device = ctx->device;
  d->embedding_dim = emb_dim;
  std::vector<void*> tmp;  // per-call device scratch, released at the end
  auto talloc = [&](size_t sz) -> void* {
    void* p = nullptr;
    if (!pool_alloc(ctx, &p, std::max<size_t>(sz, 16))) return nullptr;
    tmp.push_back(p);
    return p;
  };
  auto done = [&](int rc) {
    for (void* p : tmp) pool_free(ctx, p);
    if (rc != PARS_OK) {
      pars_dataset_free(d);
    } else {
      *out = d;
    }
    return rc;
  };
  auto oom = [&]() {
    set_error("device allocation failed (dataset loader)");
    return done(PARS_ERR_OOM);
  };
#define DS_CUDA(x)                                                            \
  do {                                                                        \
    cudaError_t e_ = (x);                                                     \
    if (e_ != cudaSuccess) {                                                  \
      set_error("CUDA error in the dataset loader: %s", cudaGetErrorString(e_)); \
      return done(PARS_ERR_CUDA);                                             \
    }                                                                         \
  } while (0)
  // 1. lines of the body
  int64_t nrec = 0, nlines = 0;
  uint8_t* d_body = nullptr;
  int64_t* d_nl = nullptr;
  if (nb > 0) {
    d_body = (uint8_t*)talloc((size_t)nb + 16);  // word reads may pass the last byte
    const int64_t nblk = ingest_block_count(nb);
    uint32_t* d_blk = (uint32_t*)talloc((size_t)(nblk + 1) * 4);
    void* d_scan = talloc(ingest_scan_scratch_bytes(std::max<int64_t>(nblk, nb + 2)));  // >= lines
    if (!d_body || !d_blk || !d_scan) return oom();
    // the bytes go up in 64 MB pieces on the copy stream; each piece's
    // newline blocks are counted as soon as it lands
    {
      const int64_t kPiece = (64ll << 20) / ingest_block_bytes() * ingest_block_bytes();
      const int npieces = (int)((nb + kPiece - 1) / kPiece);
      while ((int)ctx->ev_chunk.size() < npieces) {
        cudaEvent_t e;
        DS_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
        ctx->ev_chunk.push_back(e);
      }
      for (int k = 0; k < npieces; ++k) {
        const int64_t o = (int64_t)k * kPiece, len = std::min<int64_t>(kPiece, nb - o);
        DS_CUDA(cudaMemcpyAsync(d_body + o, body + o, (size_t)len, cudaMemcpyHostToDevice,
                                ctx->copy_stream));
        DS_CUDA(cudaEventRecord(ctx->ev_chunk[k], ctx->copy_stream));
        DS_CUDA(cudaStreamWaitEvent(st, ctx->ev_chunk[k], 0));
        const int64_t b0 = o / ingest_block_bytes();
        const int64_t b1 = std::min<int64_t>(nblk, (o + len + ingest_block_bytes() - 1) / ingest_block_bytes());
        ingest_count_newlines_range(d_body, nb, b0, b1, d_blk, st);
      }
    }
    int64_t nlc = 0;
    if (ingest_scan_newline_blocks(d_blk, nb, &nlc, d_scan, st) != PARS_OK) return done(PARS_ERR_CUDA);
    nlines = nlc + 1;  // the segment after the last '\n' (empty when the file ends with one)
    d_nl = (int64_t*)talloc((size_t)nlines * 8);
    if (!d_nl) return oom();
    ingest_write_newlines(d_body, nb, d_blk, d_nl, st);
    DS_CUDA(cudaMemcpyAsync(d_nl + nlc, &nb, 8, cudaMemcpyHostToDevice, st));
    // 2. non-empty lines, ranked, truncated to `limit`
    uint32_t* d_rank = (uint32_t*)talloc((size_t)(nlines + 1) * 4);
    if (!d_rank) return oom();
    ingest_launch_line_flags(d_nl, nlines, nb, d_rank, st);
    ingest_launch_scan(d_rank, nlines, d_scan, st);
    uint32_t total = 0;
    DS_CUDA(cudaMemcpyAsync(&total, d_rank + nlines, 4, cudaMemcpyDeviceToHost, st));
    DS_CUDA(cudaStreamSynchronize(st));
    nrec = std::min<int64_t>(total, limit);
    if (nrec > 0) {
      int64_t* d_rb = (int64_t*)talloc((size_t)nrec * 8);
      int64_t* d_re = (int64_t*)talloc((size_t)nrec * 8);
      int64_t* d_rl = (int64_t*)talloc((size_t)nrec * 8);
      if (!d_rb || !d_re || !d_rl) return oom();
      ingest_launch_record_lines(d_nl, nlines, nb, d_rank, nrec, d_rb, d_re, d_rl, st);
      // 3. parse + validate every record line
      RecordOut R;
      R.err = (uint32_t*)talloc((size_t)nrec * 4);
      R.flags = (uint32_t*)talloc((size_t)nrec * 4);
      int64_t** i64s[] = {&R.id_b, &R.id_e, &R.id_len, &R.pr_b, &R.pr_e, &R.pr_len, &R.pr_tok,
                          &R.out_len, &R.prompt_len, &R.sm_b, &R.sm_e};
      for (int64_t** q : i64s) {
        *q = (int64_t*)talloc((size_t)nrec * 8);
        if (!*q) return oom();
      }
      R.any_samples = (uint32_t*)talloc(4);
      if (!R.err || !R.flags || !R.any_samples) return oom();
      DS_CUDA(cudaMemsetAsync(R.any_samples, 0, 4, st));
      ingest_launch_parse(d_body, d_rb, d_re, nrec, R, st);
      // 4. arenas: decoded lengths -> offsets
      int64_t* d_pro = nullptr;
      int64_t* d_ido = nullptr;
      if (!pool_alloc(ctx, (void**)&d->d_offsets, (size_t)(nrec + 1) * 8) ||
          !pool_alloc(ctx, (void**)&d->d_id_offsets, (size_t)(nrec + 1) * 8) ||
          !pool_alloc(ctx, (void**)&d->d_output_len, (size_t)nrec * 8) ||
          !pool_alloc(ctx, (void**)&d->d_prompt_len, (size_t)nrec * 8))
        return oom();
      d_pro = d->d_offsets;
      d_ido = d->d_id_offsets;
      ingest_launch_lengths(nrec, R, d_pro, d_ido, st);
      ingest_launch_scan_i64(d_pro, nrec, d_scan, st);
      ingest_launch_scan_i64(d_ido, nrec, d_scan, st);
      int64_t tot[2] = {0, 0};
      DS_CUDA(cudaMemcpyAsync(&tot[0], d_pro + nrec, 8, cudaMemcpyDeviceToHost, st));
      DS_CUDA(cudaMemcpyAsync(&tot[1], d_ido + nrec, 8, cudaMemcpyDeviceToHost, st));
      DS_CUDA(cudaStreamSynchronize(st));
      d->text_bytes = tot[0];
      d->id_bytes = tot[1];
      if (!pool_alloc(ctx, (void**)&d->d_text, (size_t)tot[0] + 16) ||
          !pool_alloc(ctx, (void**)&d->d_ids, (size_t)tot[1] + 16))
        return oom();
      ingest_launch_emit(d_body, nrec, R, d_pro, d->d_text, d_ido, d->d_ids, d->d_prompt_len, st);
      // 5. duplicates, medians, and the first failing record
      uint64_t cap = 1024;
      while (cap < (uint64_t)nrec * 2) cap <<= 1;
      uint64_t* d_hash = (uint64_t*)talloc((size_t)nrec * 8);
      unsigned long long* d_tkey = (unsigned long long*)talloc((size_t)cap * 8);
      unsigned long long* d_tmin = (unsigned long long*)talloc((size_t)cap * 8);
      uint32_t* d_dup = (uint32_t*)talloc((size_t)nrec * 4);
      uint32_t* d_mis = (uint32_t*)talloc((size_t)nrec * 4);
      uint32_t* d_uns = (uint32_t*)talloc((size_t)nrec * 4);
      unsigned long long* d_first = (unsigned long long*)talloc(8);
      if (!d_hash || !d_tkey || !d_tmin || !d_dup || !d_mis || !d_uns || !d_first) return oom();
      DS_CUDA(cudaMemsetAsync(d_tkey, 0, (size_t)cap * 8, st));
      DS_CUDA(cudaMemsetAsync(d_tmin, 0xff, (size_t)cap * 8, st));
      DS_CUDA(cudaMemsetAsync(d_dup, 0, (size_t)nrec * 4, st));
      DS_CUDA(cudaMemsetAsync(d_mis, 0, (size_t)nrec * 4, st));
      DS_CUDA(cudaMemsetAsync(d_uns, 0, (size_t)nrec * 4, st));
      DS_CUDA(cudaMemsetAsync(d_first, 0xff, 8, st));
      ingest_launch_dups(d->d_ids, d_ido, nrec, d_hash, cap, d_tkey, d_tmin, d_dup, st);
      ingest_launch_samples(d_body, nrec, R, d_mis, d_uns, st);
      ingest_launch_first_fail(nrec, R, d_dup, d_mis, d_uns, d->d_prompt_len, d_first, st);
      DS_CUDA(cudaMemcpyAsync(d->d_output_len, R.out_len, (size_t)nrec * 8, cudaMemcpyDeviceToDevice, st));
      unsigned long long first = 0;
      uint32_t any_samples = 0;
      DS_CUDA(cudaMemcpyAsync(&first, d_first, 8, cudaMemcpyDeviceToHost, st));
      DS_CUDA(cudaMemcpyAsync(&any_samples, R.any_samples, 4, cudaMemcpyDeviceToHost, st));
      DS_CUDA(cudaStreamSynchronize(st));
      count_launch(ctx, 14);
      if (first != ~0ull) {
        // the reference stops at this line: its message, re-derived on the host
        int64_t b = 0, e = 0, ln = 0;
        uint32_t dup = 0;
        DS_CUDA(cudaMemcpy(&b, d_rb + first, 8, cudaMemcpyDeviceToHost));
        DS_CUDA(cudaMemcpy(&e, d_re + first, 8, cudaMemcpyDeviceToHost));
        DS_CUDA(cudaMemcpy(&ln, d_rl + first, 8, cudaMemcpyDeviceToHost));
        DS_CUDA(cudaMemcpy(&dup, d_dup + first, 4, cudaMemcpyDeviceToHost));
        bool has_emb = false;
        const std::string msg =
            ingest_record_error(std::string(body + b, (size_t)(e - b)), dup != 0, emb_dim, &has_emb);
        if (!msg.empty()) {
          ds_fail(path, ln + 2, msg);
          return done(PARS_ERR_INVALID);
        }
        set_error("%s: line %lld: the GPU dataset loader does not parse %s", path,
                  (long long)(ln + 2),
                  has_emb ? "'embedding' arrays" : "more than 256 output_len_samples");
        return done(PARS_ERR_UNSUPPORTED);
      }
      // output_len_samples (host CSR, for export): only when some record has
      // them (an empty CSR means "no samples anywhere")
      if (any_samples) {
        d->samples_rp.assign((size_t)nrec + 1, 0);
        std::vector<uint32_t> fl((size_t)nrec);
        DS_CUDA(cudaMemcpy(fl.data(), R.flags, (size_t)nrec * 4, cudaMemcpyDeviceToHost));
        std::vector<int64_t> sb((size_t)nrec), se((size_t)nrec);
        DS_CUDA(cudaMemcpy(sb.data(), R.sm_b, (size_t)nrec * 8, cudaMemcpyDeviceToHost));
        DS_CUDA(cudaMemcpy(se.data(), R.sm_e, (size_t)nrec * 8, cudaMemcpyDeviceToHost));
        for (int64_t r = 0; r < nrec; ++r) {
          if (fl[r] & kIngHasSamples) {
            const std::vector<int64_t> v =
                ingest_parse_samples(std::string(body + sb[r], (size_t)(se[r] - sb[r])));
            d->samples.insert(d->samples.end(), v.begin(), v.end());
          }
          d->samples_rp[r + 1] = (int64_t)d->samples.size();
        }
      }
    }
  }
#undef DS_CUDA
  d->n = nrec;
  if (nrec == 0) {
    if (!pool_alloc(ctx, (void**)&d->d_offsets, 8) || !pool_alloc(ctx, (void**)&d->d_id_offsets, 8))
      return oom();
    cudaMemsetAsync(d->d_offsets, 0, 8, st);
    cudaMemsetAsync(d->d_id_offsets, 0, 8, st);
    d->samples_rp.clear();
  }
  cudaStreamSynchronize(st);
  return done(PARS_OK);
}

int pars_load_dataset(pars_ctx* ctx, const char* path, int64_t limit, pars_dataset** out) {
  *out = nullptr;
  FILE* f = std::fopen(path, "rb");
  if (!f) {
    set_error("cannot open dataset file '%s'", path);
    return PARS_ERR_INVALID;
  }
  std::fseek(f, 0, SEEK_END);
  const long sz = std::ftell(f);
  std::fseek(f, 0, SEEK_SET);
  void* buf = nullptr;
  if (cudaHostAlloc(&buf, (size_t)std::max<long>(sz, 1), cudaHostAllocDefault) != cudaSuccess) {
    cudaGetLastError();
    std::fclose(f);
    set_error("pinned host allocation of %ld bytes failed", sz);
    return PARS_ERR_OOM;
  }
  const size_t got = std::fread(buf, 1, (size_t)std::max<long>(sz, 0), f);
  std::fclose(f);
  const int rc = pars_load_dataset_bytes(ctx, path, static_cast<const char*>(buf), (int64_t)got, limit, out);
  cudaFreeHost(buf);
  return rc;
}

int64_t pars_dataset_size(const pars_dataset* d) { return d ? d->n : 0; }
int64_t pars_dataset_text_bytes(const pars_dataset* d) { return d ? d->text_bytes : 0; }
int64_t pars_dataset_embedding_dim(const pars_dataset* d) { return d ? d->embedding_dim : 0; }
const char* pars_dataset_dev_text(const pars_dataset* d) { return (const char*)d->d_text; }
const int64_t* pars_dataset_dev_offsets(const pars_dataset* d) { return d->d_offsets; }
const int64_t* pars_dataset_dev_output_len(const pars_dataset* d) { return d->d_output_len; }

int pars_dataset_export(const pars_dataset* d, char* text, int64_t* offsets, int64_t* output_len,
                        int64_t* prompt_len, char* ids, int64_t* id_offsets) {
  cudaSetDevice(d->device);
  const int64_t n = d->n;
  if (text && d->text_bytes)
    PARS_CUDA_CHECK(cudaMemcpy(text, d->d_text, (size_t)d->text_bytes, cudaMemcpyDeviceToHost));
  if (offsets) PARS_CUDA_CHECK(cudaMemcpy(offsets, d->d_offsets, (size_t)(n + 1) * 8, cudaMemcpyDeviceToHost));
  if (output_len && n)
    PARS_CUDA_CHECK(cudaMemcpy(output_len, d->d_output_len, (size_t)n * 8, cudaMemcpyDeviceToHost));
  if (prompt_len && n)
    PARS_CUDA_CHECK(cudaMemcpy(prompt_len, d->d_prompt_len, (size_t)n * 8, cudaMemcpyDeviceToHost));
  if (ids && d->id_bytes) PARS_CUDA_CHECK(cudaMemcpy(ids, d->d_ids, (size_t)d->id_bytes, cudaMemcpyDeviceToHost));
  if (id_offsets)
    PARS_CUDA_CHECK(cudaMemcpy(id_offsets, d->d_id_offsets, (size_t)(n + 1) * 8, cudaMemcpyDeviceToHost));
  return PARS_OK;
}

int64_t pars_dataset_id_bytes(const pars_dataset* d) { return d ? d->id_bytes : 0; }

int64_t pars_dataset_samples(const pars_dataset* d, int64_t i, int64_t* out, int64_t cap) {
  if (i < 0 || i >= d->n) return -1;
  if (d->samples_rp.empty()) return 0;  // no record of the file has samples
  const int64_t b = d->samples_rp[i], e = d->samples_rp[i + 1];
  if (e - b > cap) return -1;
  for (int64_t k = b; k < e; ++k) out[k - b] = d->samples[k];
  return e - b;
}

void pars_dataset_free(pars_dataset* d) {
  if (!d) return;
  void* ptrs[] = {d->d_text, d->d_offsets, d->d_ids, d->d_id_offsets, d->d_output_len, d->d_prompt_len};
  pool_release(d->device, ptrs, 6);
  delete d;
}

}  // extern "C"
