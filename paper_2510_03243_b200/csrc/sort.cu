// Priority ordering: stable LSD radix sort over (score, tie_rank) keys.
//
// Reference: select_batch's comparator (scheduler.cpp:43-50) — boosted
// requests first by (arrival, id); the rest ascending by score, ties by
// (arrival_time, prompt_id), then by waiting index. With tie_rank = dense
// rank of (arrival_time, prompt_id) the comparator is the lexicographic
// order of the 96-bit key
//     hi64 = boosted ? 0 : ordered_bits(score)     lo32 = tie_rank
// and the index tiebreak is exactly the stability of an LSD radix sort
// applied in input order. ordered_bits maps doubles to uint64 preserving <,
// with -0.0 canonicalised to +0.0 (they compare equal in the reference).
//
// Kernels (8-bit digits, 12 digit positions):
//   radix_init      keys + all 12 digit histograms in one pass (one D2H read
//                   lets the host skip positions where every key shares the
//                   digit — typically the constant high exponent bytes and the
//                   unused high bytes of tie_rank);
//   radix_hist      per-CTA digit counts of the current order (digit-major);
//   radix_scan_digits  per digit, the exclusive scan of its per-CTA counts
//                   (one warp per digit, global base from the all-digit
//                   histogram); tie-rank digits are skipped when the ranks
//                   are already non-decreasing in input order;
//   radix_scatter   stable rank within the CTA via warp __match_any_sync +
//                   per-warp digit counters; the tile is laid out in digit
//                   order in shared memory and written run by run (coalesced).
#include <cuda_runtime.h>

#include <algorithm>
#include <vector>

#include "common.cuh"
#include "pairs.cuh"

namespace pars_b200 {

namespace {

constexpr int kThreads = 256;
constexpr int kItems = 8;
constexpr int kTileKeys = kThreads * kItems;  // 2048
constexpr unsigned kFull = 0xffffffffu;

__device__ __forceinline__ uint64_t ordered_bits(double x) {
  uint64_t b = (uint64_t)__double_as_longlong(x);
  if ((b << 1) == 0) b = 0;  // -0.0 == +0.0
  return (b >> 63) ? ~b : (b | 0x8000000000000000ull);
}

__device__ __forceinline__ uint32_t digit_of(uint64_t hi, uint32_t lo, int pos) {
  return pos < 4 ? (lo >> (8 * pos)) & 0xffu : (uint32_t)(hi >> (8 * (pos - 4))) & 0xffu;
}

__global__ void radix_init(const double* __restrict__ score, const uint8_t* __restrict__ boosted,
                           const uint32_t* __restrict__ tie, int64_t n, uint64_t* __restrict__ khi,
                           uint32_t* __restrict__ klo, uint32_t* __restrict__ val,
                           uint32_t* __restrict__ dh) {
  __shared__ uint32_t h[12 * 256];
  for (int k = threadIdx.x; k < 12 * 256; k += blockDim.x) h[k] = 0;
  __syncthreads();
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    const bool bst = boosted && boosted[i];
    const uint64_t hi = bst ? 0ull : ordered_bits(score[i]);
    const uint32_t lo = tie ? tie[i] : 0u;  // no tie ranks: order by score, then index
    khi[i] = hi;
    klo[i] = lo;
    val[i] = (uint32_t)i;
    // tie ranks already non-decreasing in input order -> the stable sort
    // by score alone yields the (score, tie, index) order: skip tie digits
    if (tie && i > 0 && tie[i] < tie[i - 1]) dh[12 * 256] = 1u;
#pragma unroll
    for (int p = 0; p < 12; ++p) atomicAdd(&h[p * 256 + digit_of(hi, lo, p)], 1u);
  }
  __syncthreads();
  for (int k = threadIdx.x; k < 12 * 256; k += blockDim.x)
    if (h[k]) atomicAdd(&dh[k], h[k]);
}

__global__ void __launch_bounds__(kThreads) radix_hist(const uint64_t* __restrict__ khi,
                                                       const uint32_t* __restrict__ klo,
                                                       int64_t n, int pos, int nblocks,
                                                       uint32_t* __restrict__ hist) {
  __shared__ uint32_t h[256];
  h[threadIdx.x] = 0;
  __syncthreads();
  const int64_t base = (int64_t)blockIdx.x * kTileKeys;
  for (int k = threadIdx.x; k < kTileKeys; k += kThreads) {
    const int64_t i = base + k;
    if (i < n) atomicAdd(&h[digit_of(khi[i], klo[i], pos)], 1u);
  }
  __syncthreads();
  hist[(int64_t)threadIdx.x * nblocks + blockIdx.x] = h[threadIdx.x];
}

// Exclusive offsets of one digit position: block d (one warp) scans digit
// d's per-CTA counts in CTA order, starting from the digit's global base
// (sum of the all-digit histogram's counts of smaller digits).
__global__ void __launch_bounds__(32) radix_scan_digits(uint32_t* __restrict__ hist, int nblocks,
                                                        const uint32_t* __restrict__ dh_pos) {
  const int d = blockIdx.x, lane = threadIdx.x;
  uint32_t base = 0;
  for (int k = lane; k < d; k += 32) base += dh_pos[k];
  base = __reduce_add_sync(0xffffffffu, base);
  uint32_t* row = hist + (int64_t)d * nblocks;
  for (int b0 = 0; b0 < nblocks; b0 += 32) {
    const int b = b0 + lane;
    const uint32_t v = b < nblocks ? row[b] : 0u;
    uint32_t x = v;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const uint32_t y = __shfl_up_sync(0xffffffffu, x, o);
      if (lane >= o) x += y;
    }
    if (b < nblocks) row[b] = base + x - v;
    base += __shfl_sync(0xffffffffu, x, 31);
  }
}

__global__ void __launch_bounds__(kThreads) radix_scatter(
    const uint64_t* __restrict__ khi_in, const uint32_t* __restrict__ klo_in,
    const uint32_t* __restrict__ val_in, uint64_t* __restrict__ khi_out,
    uint32_t* __restrict__ klo_out, uint32_t* __restrict__ val_out, int64_t n, int pos,
    int nblocks, const uint32_t* __restrict__ offsets) {
  __shared__ uint32_t wcnt[kThreads / 32][256];
  __shared__ uint32_t gbase[256];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  for (int k = threadIdx.x; k < (kThreads / 32) * 256; k += kThreads) (&wcnt[0][0])[k] = 0;
  gbase[threadIdx.x] = offsets[(int64_t)threadIdx.x * nblocks + blockIdx.x];
  __syncthreads();
  const int64_t sub = (int64_t)blockIdx.x * kTileKeys + warp * (32 * kItems);
  const unsigned lt = (1u << lane) - 1u;
  uint64_t hi[kItems];
  uint32_t lo[kItems], vv[kItems], dg[kItems], rk[kItems];
#pragma unroll
  for (int r = 0; r < kItems; ++r) {
    const int64_t i = sub + r * 32 + lane;
    const bool ok = i < n;
    hi[r] = ok ? khi_in[i] : 0ull;
    lo[r] = ok ? klo_in[i] : 0u;
    vv[r] = ok ? val_in[i] : 0u;
    const uint32_t d = ok ? digit_of(hi[r], lo[r], pos) : 256u;
    dg[r] = d;
    const unsigned peers = __match_any_sync(kFull, d);
    const uint32_t before = ok ? wcnt[warp][d] : 0u;
    rk[r] = before + __popc(peers & lt);
    __syncwarp();
    if (ok && (peers & lt) == 0) wcnt[warp][d] = before + __popc(peers);
    __syncwarp();
  }
  __syncthreads();
  __shared__ uint32_t tstart[256];  // the tile's digit runs, exclusive prefix
  __shared__ uint32_t wsum[kThreads / 32];
  {  // thread = digit: each warp's offset inside the digit's run, the run length
    const int d = threadIdx.x;
    uint32_t run = 0;
    for (int w = 0; w < kThreads / 32; ++w) {
      const uint32_t c = wcnt[w][d];
      wcnt[w][d] = run;
      run += c;
    }
    // exclusive scan of the run lengths over the 256 digits
    uint32_t x = run;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const uint32_t y = __shfl_up_sync(kFull, x, o);
      if (lane >= o) x += y;
    }
    if (lane == 31) wsum[warp] = x;
    __syncthreads();
    uint32_t wb = 0;
    for (int w = 0; w < warp; ++w) wb += wsum[w];
    tstart[d] = wb + x - run;
  }
  __syncthreads();
  // the tile in digit order in shared memory, then written out run by run:
  // consecutive threads store consecutive addresses of a digit's run instead
  // of every key landing in its own sector
  __shared__ uint64_t s_hi[kTileKeys];
  __shared__ uint32_t s_lo[kTileKeys], s_val[kTileKeys];
#pragma unroll
  for (int r = 0; r < kItems; ++r) {
    if (dg[r] < 256u) {
      const uint32_t lp = tstart[dg[r]] + wcnt[warp][dg[r]] + rk[r];
      s_hi[lp] = hi[r];
      s_lo[lp] = lo[r];
      s_val[lp] = vv[r];
    }
  }
  __syncthreads();
  const int64_t t0 = (int64_t)blockIdx.x * kTileKeys;
  const int cnt = (int)(n - t0 < kTileKeys ? n - t0 : (int64_t)kTileKeys);
  for (int k = threadIdx.x; k < cnt; k += kThreads) {
    const uint64_t h = s_hi[k];
    const uint32_t l = s_lo[k];
    const uint32_t d = digit_of(h, l, pos);
    const uint32_t p = gbase[d] + (uint32_t)k - tstart[d];
    khi_out[p] = h;
    klo_out[p] = l;
    val_out[p] = s_val[k];
  }
}

// Small queues (n <= kSmallSort): one CTA, one launch, no host round trip.
// The key (ordered score bits or 0 if boosted, tie rank, input index) is
// unique, so ANY correct sort of it yields the stable order the radix path
// produces; a shared-memory bitonic network sorts it (padding keys are all
// ones and sink to the end).
constexpr int kSmallSort = 4096, kSmallThreads = 1024;

__global__ void __launch_bounds__(kSmallThreads) small_sort_kernel(
    const double* __restrict__ score, const uint8_t* __restrict__ boosted,
    const uint32_t* __restrict__ tie, int n, int n2, uint32_t* __restrict__ order) {
  extern __shared__ uint64_t ks[];  // hi[n2], lo[n2] (lo = tie << 32 | index)
  uint64_t* hi = ks;
  uint64_t* lo = ks + n2;
  for (int i = threadIdx.x; i < n2; i += blockDim.x) {
    if (i < n) {
      hi[i] = (boosted && boosted[i]) ? 0ull : ordered_bits(score[i]);
      lo[i] = ((uint64_t)(tie ? tie[i] : 0u) << 32) | (uint32_t)i;
    } else {
      hi[i] = ~0ull;
      lo[i] = ~0ull;
    }
  }
  __syncthreads();
  for (int k = 2; k <= n2; k <<= 1) {
    for (int j = k >> 1; j > 0; j >>= 1) {
      for (int t = threadIdx.x; t < (n2 >> 1); t += blockDim.x) {
        const int i = 2 * t - (t & (j - 1));  // lower index of the pair (bit j clear)
        const int p = i + j;
        const bool up = (i & k) == 0;
        const uint64_t ah = hi[i], al = lo[i], bh = hi[p], bl = lo[p];
        const bool gt = ah > bh || (ah == bh && al > bl);
        if (gt == up) {
          hi[i] = bh;
          lo[i] = bl;
          hi[p] = ah;
          lo[p] = al;
        }
      }
      __syncthreads();
    }
  }
  for (int i = threadIdx.x; i < n; i += blockDim.x) order[i] = (uint32_t)lo[i];
}

}  // namespace

// ---- merging sorted runs (the global order of sharded scoring) -------------
// Runs [off[r], off[r+1]) are each in select_batch order (run-local orders
// from launch_priority_sort on the shard). Every element becomes the 128-bit
// key (hi = boosted ? 0 : ordered_bits(score), lo = tie << 32 | index), a
// total order equal to the global sort's (key, tie, then input index), and
// adjacent runs are merged level by level: each element finds its place in
// the sibling run by binary search (keys are unique, so no tie rule is needed).
namespace {
__global__ void merge_keys_kernel(const double* __restrict__ score, const uint8_t* __restrict__ boosted,
                                  const uint32_t* __restrict__ tie, const uint32_t* __restrict__ run_order,
                                  const int64_t* __restrict__ off, int nruns, int64_t n,
                                  uint64_t* __restrict__ hi, uint64_t* __restrict__ lo) {
  const int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (k >= n) return;
  int r = 0;
  while (r + 1 < nruns && off[r + 1] <= k) ++r;  // nruns is the rank count: small
  const uint32_t i = (uint32_t)(off[r] + run_order[k]);
  hi[k] = (boosted && boosted[i]) ? 0ull : ordered_bits(score[i]);
  lo[k] = ((uint64_t)(tie ? tie[i] : 0u) << 32) | i;
}

__device__ __forceinline__ bool key_less(uint64_t ah, uint64_t al, uint64_t bh, uint64_t bl) {
  return ah < bh || (ah == bh && al < bl);
}

// one level: runs (a, b) = (2m, 2m+1) of the current boundaries merge into
// [off[2m], off[2m+2]); boundaries for the next level are every other one
__global__ void merge_level_kernel(const uint64_t* __restrict__ hi, const uint64_t* __restrict__ lo,
                                   const int64_t* __restrict__ off, int nruns, int64_t n,
                                   uint64_t* __restrict__ ohi, uint64_t* __restrict__ olo) {
  const int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (k >= n) return;
  int r = 0;
  while (r + 1 < nruns && off[r + 1] <= k) ++r;
  const uint64_t h = hi[k], l = lo[k];
  const int sib = r ^ 1;
  if (sib >= nruns) {  // odd run out: copied through
    ohi[k] = h;
    olo[k] = l;
    return;
  }
  const int64_t s0 = off[sib], s1 = off[sib + 1];
  int64_t a = s0, b = s1;  // first sibling element greater than (h, l)
  while (a < b) {
    const int64_t m = (a + b) >> 1;
    if (key_less(hi[m], lo[m], h, l)) a = m + 1; else b = m;
  }
  const int64_t base = off[r & ~1];
  const int64_t pos = base + (k - off[r]) + (a - s0);
  ohi[pos] = h;
  olo[pos] = l;
}

__global__ void merge_out_kernel(const uint64_t* __restrict__ lo, int64_t n, uint32_t* __restrict__ order) {
  const int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (k < n) order[k] = (uint32_t)lo[k];
}

}  // namespace

size_t merge_runs_scratch_bytes(int64_t n, int nruns) {
  return 4 * ((size_t)n * 8 + 256) + 2 * ((size_t)(nruns + 1) * 8 + 256);
}

int launch_merge_runs(pars_ctx* ctx, const double* score, const uint8_t* boosted, const uint32_t* tie,
                      const uint32_t* run_order, const int64_t* h_off, int nruns, int64_t n,
                      uint32_t* order, void* scratch, cudaStream_t st) {
  if (n == 0) return PARS_OK;
  if (n > 0x7fffffffLL) {
    set_error("priority order: n=%lld exceeds 2^31-1", (long long)n);
    return PARS_ERR_UNSUPPORTED;
  }
  char* p = static_cast<char*>(scratch);
  auto take = [&](size_t bytes) {
    char* r = p;
    p += (bytes + 255) & ~(size_t)255;
    return r;
  };
  uint64_t* hi[2] = {(uint64_t*)take(n * 8), (uint64_t*)take(n * 8)};
  uint64_t* lo[2] = {(uint64_t*)take(n * 8), (uint64_t*)take(n * 8)};
  int64_t* d_off[2] = {(int64_t*)take((nruns + 1) * 8), (int64_t*)take((nruns + 1) * 8)};
  const unsigned g = (unsigned)ceil_div(n, 256);
  std::vector<int64_t> off(h_off, h_off + nruns + 1);
  PARS_CUDA_CHECK(cudaMemcpyAsync(d_off[0], off.data(), off.size() * 8, cudaMemcpyHostToDevice, st));
  merge_keys_kernel<<<g, 256, 0, st>>>(score, boosted, tie, run_order, d_off[0], nruns, n, hi[0], lo[0]);
  count_launch(ctx);
  int cur = 0, cb = 0;
  int runs = nruns;
  while (runs > 1) {
    merge_level_kernel<<<g, 256, 0, st>>>(hi[cur], lo[cur], d_off[cb], runs, n, hi[cur ^ 1],
                                          lo[cur ^ 1]);
    count_launch(ctx);
    cur ^= 1;
    std::vector<int64_t> next;
    for (int r = 0; r < runs; r += 2) next.push_back(off[r]);
    next.push_back(off[runs]);
    off.swap(next);
    runs = (int)off.size() - 1;
    cb ^= 1;
    PARS_CUDA_CHECK(cudaMemcpyAsync(d_off[cb], off.data(), off.size() * 8, cudaMemcpyHostToDevice, st));
  }
  merge_out_kernel<<<g, 256, 0, st>>>(lo[cur], n, order);
  count_launch(ctx);
  PARS_CUDA_CHECK(cudaGetLastError());
  // the boundary vectors are pageable host memory read by async copies
  PARS_CUDA_CHECK(cudaStreamSynchronize(st));
  return PARS_OK;
}

size_t sort_scratch_bytes(int64_t n) {
  const int64_t nb = ceil_div(std::max<int64_t>(n, 1), kTileKeys);
  size_t b = 0;
  b += 2 * (size_t)n * 8 + 2 * (size_t)n * 4 + 2 * (size_t)n * 4;
  b += (size_t)nb * 256 * 4 + 12 * 256 * 4 + 1024;
  return b;
}

int launch_priority_sort(pars_ctx* ctx, const double* score, const uint8_t* boosted,
                         const uint32_t* tie, int64_t n, uint32_t* order, void* scratch,
                         cudaStream_t st) {
  if (n == 0) return PARS_OK;
  if (n > 0x7fffffffLL) {
    set_error("priority order: n=%lld exceeds 2^31-1", (long long)n);
    return PARS_ERR_UNSUPPORTED;
  }
  if (n <= kSmallSort) {
    int n2 = 2;
    while (n2 < n) n2 <<= 1;
    const size_t sm = (size_t)n2 * 16;
    PARS_CUDA_CHECK(cudaFuncSetAttribute(small_sort_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         (int)sm));
    small_sort_kernel<<<1, std::min(kSmallThreads, std::max(32, n2 / 2)), sm, st>>>(score, boosted, tie,
                                                                                  (int)n, n2, order);
    count_launch(ctx);
    PARS_CUDA_CHECK(cudaGetLastError());
    return PARS_OK;
  }
  const int nb = (int)ceil_div(n, kTileKeys);
  char* p = static_cast<char*>(scratch);
  auto take = [&](size_t bytes) {
    char* r = p;
    p += (bytes + 255) & ~(size_t)255;
    return r;
  };
  uint64_t* khi[2] = {(uint64_t*)take(n * 8), (uint64_t*)take(n * 8)};
  uint32_t* klo[2] = {(uint32_t*)take(n * 4), (uint32_t*)take(n * 4)};
  uint32_t* val[2] = {(uint32_t*)take(n * 4), (uint32_t*)take(n * 4)};
  uint32_t* hist = (uint32_t*)take((size_t)nb * 256 * 4);
  uint32_t* dh = (uint32_t*)take(12 * 256 * 4 + 16);
  PARS_CUDA_CHECK(cudaMemsetAsync(dh, 0, 12 * 256 * 4 + 16, st));
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const int64_t ig = std::min<int64_t>(ceil_div(n, 256), (int64_t)sms * 4);
  radix_init<<<(unsigned)ig, 256, 0, st>>>(score, boosted, tie, n, khi[0], klo[0], val[0], dh);
  count_launch(ctx);
  PARS_CUDA_CHECK(cudaGetLastError());
  std::vector<uint32_t> hh(12 * 256 + 1);
  PARS_CUDA_CHECK(cudaMemcpyAsync(hh.data(), dh, hh.size() * 4, cudaMemcpyDeviceToHost, st));
  PARS_CUDA_CHECK(cudaStreamSynchronize(st));
  const bool tie_sorted = hh[12 * 256] == 0;
  int cur = 0;
  for (int pos = tie_sorted ? 4 : 0; pos < 12; ++pos) {
    bool trivial = false;
    for (int d = 0; d < 256; ++d)
      if (hh[pos * 256 + d] == (uint32_t)n) trivial = true;
    if (trivial) continue;
    radix_hist<<<nb, kThreads, 0, st>>>(khi[cur], klo[cur], n, pos, nb, hist);
    radix_scan_digits<<<256, 32, 0, st>>>(hist, nb, dh + pos * 256);
    radix_scatter<<<nb, kThreads, 0, st>>>(khi[cur], klo[cur], val[cur], khi[cur ^ 1],
                                           klo[cur ^ 1], val[cur ^ 1], n, pos, nb, hist);
    count_launch(ctx, 3);
    PARS_CUDA_CHECK(cudaGetLastError());
    cur ^= 1;
  }
  PARS_CUDA_CHECK(cudaMemcpyAsync(order, val[cur], (size_t)n * 4, cudaMemcpyDeviceToDevice, st));
  return PARS_OK;
}

}  // namespace pars_b200
