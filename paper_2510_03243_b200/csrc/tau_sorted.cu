// Kendall tau-b counts in O(n log n), exact (Knight's method).
//
// Reference: kendall_tau_b (metrics.cpp:42-64) loops over all n(n-1)/2 pairs
// and counts n1 (dx == 0), n2 (dy == 0), and among the untied pairs n_c
// (same sign) and n_d. For finite inputs dx == 0 iff x_i == x_j and the sign
// of dx is the order of x_i, x_j, so the same integers follow from sorting:
//   n1 = sum over runs of equal x of C(t, 2); n2 likewise for y; n3 = pairs
//   tied in both; sorted by (x, y), every pair (k < l) with X[k] < X[l] and
//   Y[k] > Y[l] is discordant and no other pair is an inversion, so n_d is
//   the inversion count of the y sequence; n_c = n0 - n1 - n2 + n3 - n_d.
// Non-finite values (inf - inf = NaN is "not tied" and "not negative" in the
// reference) break that equivalence: the caller checks for them and runs the
// all-pairs tile kernel instead.
//
// Steps (all on the device, two stable radix sorts from sort.cu):
//   1. y order (radix on y); ry[i] = first position of y_i's run in that
//      order (a rank that preserves < and =), n2 from the same binary search;
//   2. (x, ry) order (radix on x with ry as the tie rank);
//   3. n1 / n3 by binary searches for run starts in the sorted keys;
//   4. n_d: merge sort of the ry sequence, counting for every element of a
//      right run the elements of its left run that are greater. Runs of 2,048
//      are merged inside one CTA's shared memory, longer ones level by level
//      in global memory (one thread per element, one binary search each).
#include <cuda_runtime.h>

#include <algorithm>

#include "common.cuh"
#include "pairs.cuh"

namespace pars_b200 {

namespace {

#ifndef PARS_TAU_TILE_T
#define PARS_TAU_TILE_T 1024
#endif
constexpr int kTileT = PARS_TAU_TILE_T;  // threads per tile CTA
#ifndef PARS_TAU_TILE_PER_T
#define PARS_TAU_TILE_PER_T 2
#endif
constexpr int kTile = PARS_TAU_TILE_PER_T * kTileT;  // elements per tile

__device__ __forceinline__ uint64_t key_of(double v) {
  uint64_t b = (uint64_t)__double_as_longlong(v);
  if ((b << 1) == 0) b = 0;  // -0.0 == +0.0
  return (b >> 63) ? ~b : (b | 0x8000000000000000ull);
}

// warp-wide 64-bit sum, one atomic per warp (all lanes must call)
__device__ __forceinline__ void add_u64(unsigned long long* dst, unsigned long long v) {
#pragma unroll
  for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  if ((threadIdx.x & 31) == 0 && v) atomicAdd(dst, v);
}

// first index in a[0, n) whose value is >= v (lower) or > v (upper)
template <typename T>
__device__ __forceinline__ int64_t lower_idx(const T* a, int64_t n, T v) {
  int64_t lo = 0, hi = n;
  while (lo < hi) {
    const int64_t m = (lo + hi) >> 1;
    if (a[m] < v) lo = m + 1; else hi = m;
  }
  return lo;
}
template <typename T>
__device__ __forceinline__ int64_t upper_idx(const T* a, int64_t n, T v) {
  int64_t lo = 0, hi = n;
  while (lo < hi) {
    const int64_t m = (lo + hi) >> 1;
    if (a[m] <= v) lo = m + 1; else hi = m;
  }
  return lo;
}

// step 1: ky sorted by the y order; ry[i] = start of y_i's run; n2
// (oy and o are permutations, so these two gathers see every y and every x
// once: they also raise the non-finite flag)
__device__ __forceinline__ void flag_nonfinite(bool b, unsigned* bad) {
  if (__any_sync(0xffffffffu, b) && (threadIdx.x & 31) == 0) atomicOr(bad, 1u);
}
__global__ void tau_yrank_kernel(const double* __restrict__ y, const uint32_t* __restrict__ oy,
                                 int64_t n, uint64_t* __restrict__ kys, unsigned* __restrict__ bad) {
  const int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  bool b = false;
  if (k < n) {
    const double v = y[oy[k]];
    kys[k] = key_of(v);
    b = !isfinite(v);
  }
  flag_nonfinite(b, bad);
}
__global__ void tau_yrun_kernel(const uint64_t* __restrict__ kys, const uint32_t* __restrict__ oy,
                                int64_t n, uint32_t* __restrict__ ry,
                                unsigned long long* __restrict__ counts) {
  const int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  unsigned long long t = 0;
  if (k < n) {
    const int64_t s = lower_idx(kys, k, kys[k]);
    ry[oy[k]] = (uint32_t)s;
    t = (unsigned long long)(k - s);
  }
  add_u64(&counts[3], t);  // n2
}

// steps 2-3: X / Y in (x, ry) order; n1 and n3 (pairs tied in both)
__global__ void tau_gather_kernel(const double* __restrict__ x, const uint32_t* __restrict__ ry,
                                  const uint32_t* __restrict__ o, int64_t n,
                                  uint64_t* __restrict__ kx, uint32_t* __restrict__ Y,
                                  unsigned* __restrict__ bad) {
  const int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  bool b = false;
  if (k < n) {
    const uint32_t i = o[k];
    const double v = x[i];
    kx[k] = key_of(v);
    Y[k] = ry[i];
    b = !isfinite(v);
  }
  flag_nonfinite(b, bad);
}
__global__ void tau_xrun_kernel(const uint64_t* __restrict__ kx, const uint32_t* __restrict__ Y,
                                int64_t n, unsigned long long* __restrict__ counts,
                                unsigned long long* __restrict__ n3) {
  const int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  unsigned long long t1 = 0, t3 = 0;
  if (k < n) {
    const uint64_t v = kx[k];
    const int64_t s = lower_idx(kx, k, v);  // start of the x run
    t1 = (unsigned long long)(k - s);
    // within the x run the Y values are sorted: start of the (x, y) run
    const int64_t s3 = s + lower_idx(Y + s, k - s, Y[k]);
    t3 = (unsigned long long)(k - s3);
  }
  add_u64(&counts[2], t1);  // n1
  add_u64(n3, t3);
}

// 32-bit forms for the shared-memory tile (runs shorter than kTile)
__device__ __forceinline__ int lower_idx32(const uint32_t* a, int n, uint32_t v) {
  int lo = 0, hi = n;
  while (lo < hi) {
    const int m = (lo + hi) >> 1;
    if (a[m] < v) lo = m + 1; else hi = m;
  }
  return lo;
}
__device__ __forceinline__ int upper_idx32(const uint32_t* a, int n, uint32_t v) {
  int lo = 0, hi = n;
  while (lo < hi) {
    const int m = (lo + hi) >> 1;
    if (a[m] <= v) lo = m + 1; else hi = m;
  }
  return lo;
}

// step 4a: sort tiles of kTile elements in shared memory, counting the
// inversions inside each tile
__global__ void __launch_bounds__(kTileT) tau_tile_merge_kernel(uint32_t* __restrict__ Y, int64_t n,
                                                                unsigned long long* __restrict__ nd) {
  __shared__ uint32_t buf[2][kTile];
  const int64_t t0 = (int64_t)blockIdx.x * kTile;
  const int len = (int)(n - t0 < kTile ? n - t0 : (int64_t)kTile);
  for (int k = threadIdx.x; k < kTile; k += kTileT) buf[0][k] = k < len ? Y[t0 + k] : 0xffffffffu;
  __syncthreads();
  unsigned long long inv = 0;
  int cur = 0;
  for (int w = 1; w < kTile; w <<= 1) {
    const uint32_t* a = buf[cur];
    uint32_t* b = buf[cur ^ 1];
    for (int k = threadIdx.x; k < kTile; k += kTileT) {
      const int base = k & ~(2 * w - 1);
      const uint32_t v = a[k];
      if (k < base + w) {  // left run element
        const int r = lower_idx32(a + base + w, w, v);
        b[k + r] = v;
      } else {             // right run element: left elements greater than v
        const int u = upper_idx32(a + base, w, v);
        // padding (0xffffffff) sits at the end of the last tile only and is
        // never greater than a real value's left partner: count real ones
        if (k < len) inv += (unsigned long long)(w - u);
        b[k - w + u] = v;
      }
    }
    cur ^= 1;
    __syncthreads();
  }
  for (int k = threadIdx.x; k < len; k += kTileT) Y[t0 + k] = buf[cur][k];
  add_u64(nd, inv);
}

// step 4b: one merge level of runs of width w (>= kTile) in global memory
__global__ void tau_merge_level_kernel(const uint32_t* __restrict__ a, uint32_t* __restrict__ b,
                                       int64_t n, int64_t w, unsigned long long* __restrict__ nd) {
  const int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  unsigned long long inv = 0;
  if (k < n) {
    const int64_t base = k & ~(2 * w - 1);
    const uint32_t v = a[k];
    const int64_t rem = n - base - w;
    const int64_t rl = rem <= 0 ? 0 : (rem < w ? rem : w);  // right run length
    if (k < base + w) {
      b[k + lower_idx(a + base + w, rl, v)] = v;
    } else {
      const int64_t u = upper_idx(a + base, w, v);
      inv = (unsigned long long)(w - u);
      b[k - w + u] = v;
    }
  }
  add_u64(nd, inv);
}

}  // namespace

size_t tau_sorted_scratch_bytes(int64_t n) {
  size_t b = 256 + sort_scratch_bytes(n) + 1024;  // counts block first
  b += 2 * ((size_t)n * 4 + 256);  // oy, o
  b += (size_t)n * 8 + 256;        // kys / kx
  b += 3 * ((size_t)n * 4 + 256);  // ry, Y ping-pong
  b += 256;                        // flags / n3
  return b;
}

// counts4 (host) receives {n_c, n_d, n1, n2}; synchronises `st`. Returns
// PARS_ERR_UNSUPPORTED (nothing written) when x or y holds a non-finite value.
namespace {
// the counts block sits at the front of the scratch (its place does not
// depend on n, so the read-back needs only the scratch pointer)
unsigned long long* tau_aux(void* scratch) { return static_cast<unsigned long long*>(scratch); }
}  // namespace

int launch_tau_sorted(pars_ctx* ctx, const double* x, const double* y, int64_t n,
                      uint64_t* counts4, void* scratch, cudaStream_t st) {
  PARS_TRY(enqueue_tau_sorted(ctx, x, y, n, scratch, st));
  return finish_tau_sorted(n, counts4, scratch, st);
}

int enqueue_tau_sorted(pars_ctx* ctx, const double* x, const double* y, int64_t n, void* scratch,
                       cudaStream_t st) {
  if (n > 0x7fffffffLL) {
    set_error("kendall_tau_b: n=%lld exceeds 2^31-1", (long long)n);
    return PARS_ERR_UNSUPPORTED;
  }
  // aux: [0] non-finite flag, [1] n3, [2..5] {n_c, n_d, n1, n2}
  unsigned long long* aux = tau_aux(scratch);
  char* p = static_cast<char*>(scratch) + 256;
  auto take = [&](size_t bytes) {
    char* r = p;
    p += (bytes + 255) & ~(size_t)255;
    return r;
  };
  void* sort_scr = take(sort_scratch_bytes(n) + 1024);
  uint32_t* oy = (uint32_t*)take((size_t)n * 4);
  uint32_t* o = (uint32_t*)take((size_t)n * 4);
  uint64_t* k64 = (uint64_t*)take((size_t)n * 8);
  uint32_t* ry = (uint32_t*)take((size_t)n * 4);
  uint32_t* Y[2] = {(uint32_t*)take((size_t)n * 4), (uint32_t*)take((size_t)n * 4)};
  unsigned long long* dc = aux + 2;
  PARS_CUDA_CHECK(cudaMemsetAsync(aux, 0, 64, st));
  const unsigned g256 = (unsigned)ceil_div(n, 256);
  // the non-finite flag is raised by the two gathers below and read with the
  // counts at the end (one synchronisation per call): the sorts and searches
  // are safe on any bit patterns, their counts only meaningless then
  // 1. y order and y-run ranks
  PARS_TRY(launch_priority_sort(ctx, y, nullptr, nullptr, n, oy, sort_scr, st));
  tau_yrank_kernel<<<g256, 256, 0, st>>>(y, oy, n, k64, reinterpret_cast<unsigned*>(aux));
  tau_yrun_kernel<<<g256, 256, 0, st>>>(k64, oy, n, ry, dc);
  // 2. (x, ry) order
  PARS_TRY(launch_priority_sort(ctx, x, nullptr, ry, n, o, sort_scr, st));
  // 3. n1, n3
  tau_gather_kernel<<<g256, 256, 0, st>>>(x, ry, o, n, k64, Y[0], reinterpret_cast<unsigned*>(aux));
  tau_xrun_kernel<<<g256, 256, 0, st>>>(k64, Y[0], n, dc, aux + 1);
  // 4. inversions of Y = n_d
  tau_tile_merge_kernel<<<(unsigned)ceil_div(n, kTile), kTileT, 0, st>>>(Y[0], n, dc + 1);
  int cur = 0;
  for (int64_t w = kTile; w < n; w <<= 1) {
    tau_merge_level_kernel<<<g256, 256, 0, st>>>(Y[cur], Y[cur ^ 1], n, w, dc + 1);
    cur ^= 1;
    count_launch(ctx);
  }
  count_launch(ctx, 5);
  PARS_CUDA_CHECK(cudaGetLastError());
  return PARS_OK;
}

int finish_tau_sorted(int64_t n, uint64_t* counts4, void* scratch, cudaStream_t st) {
  // n_c = n0 - n1 - n2 + n3 - n_d, on the host after one read
  unsigned long long a[6];
  PARS_CUDA_CHECK(cudaMemcpyAsync(a, tau_aux(scratch), sizeof a, cudaMemcpyDeviceToHost, st));
  PARS_CUDA_CHECK(cudaStreamSynchronize(st));
  if ((unsigned)a[0]) return PARS_ERR_UNSUPPORTED;
  const uint64_t n0 = (uint64_t)n * (uint64_t)(n - 1) / 2;
  counts4[1] = a[3];
  counts4[2] = a[4];
  counts4[3] = a[5];
  counts4[0] = n0 - a[4] - a[5] + a[1] - a[3];
  return PARS_OK;
}

}  // namespace pars_b200
