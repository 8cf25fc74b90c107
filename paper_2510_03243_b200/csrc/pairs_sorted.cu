// Length-sorted all-pairs margin-ranking loss (config C5 fast path).
//
// Same contract as allpairs_kernel (pairs.cu) — Eq. 1 mask, hinge of
// pairs.hpp:27-31, integer gradient coefficients, kept/active counts,
// per-tile loss partials — but on prompts pre-sorted by length (stable), a
// per-dataset plan:
//   * for i < j in sorted order L_i <= L_j, so a kept pair always has y = -1
//     (the shorter prompt first) and hinge = fl(fl(s_i - s_j) + m);
//   * keep(i, j) <=> L_i <= g_j with g_j = L_j - dmin[L_j]; g is
//     non-decreasing in j (checked when the plan is built), so row i keeps
//     exactly the column suffix [f_i, n): the bit-exact integer Eq. 1 mask
//     becomes one integer compare per pair, and whole tiles are classified as
//     fully kept / partially kept / empty from f at the tile corners;
//   * active <=> fl(s_i - s_j) > -m (the sign of fl(x + m) is the sign of the
//     exact x + m) <=> s_j < T_i, with T_i the smallest double for which
//     fl(s_i - T_i) <= -m, found per row by a binary search over ordered
//     double keys. One fp64 compare per pair decides the hinge bit-exactly;
//   * per column, the warp's active bits are one ballot + popc; rows count in
//     registers; c_i += #active in row, c_j -= #active in column (integers);
//   * the tile's loss is sum_i a_i (s_i + m) - sum_j b_j s_j (a/b the row /
//     column active counts) in fp64, reduced in a fixed order.
// Inner loop (fully kept tile), per column x 32 rows: LDS.64 broadcast,
// DSETP, row-count add, VOTE, POPC, SEL. (Keeping the 32 ballots and one
// popc per lane, or 2-column LDS.128, measured slower: 0.74 vs 0.60 ms.)
#include <cuda_runtime.h>
#include <math_constants.h>

#include <algorithm>
#include <cmath>
#include <vector>

#include "common.cuh"
#include "pairs.cuh"
#include "tiles.cuh"

namespace pars_b200 {

namespace {

constexpr int kT = kPairTile;
constexpr unsigned kFull = 0xffffffffu;

__global__ void plan_gather_kernel(const uint32_t* __restrict__ perm, const int32_t* __restrict__ L,
                                   const int32_t* __restrict__ dmin, int64_t n,
                                   int32_t* __restrict__ Ls, int32_t* __restrict__ g) {
  const int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (k >= n) return;
  const int32_t l = L[perm[k]];
  Ls[k] = l;
  const int64_t d = dmin[l];
  g[k] = (int32_t)max((int64_t)INT32_MIN, (int64_t)l - d);
}

__global__ void plan_check_kernel(const int32_t* __restrict__ g, int64_t n, int32_t* bad) {
  const int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (k > 0 && k < n && g[k] < g[k - 1]) atomicExch(bad, 1);
}

// f_i = first j with g_j >= L_i (binary search on non-decreasing g).
__global__ void plan_first_kernel(const int32_t* __restrict__ g, const int32_t* __restrict__ Ls,
                                  int64_t n, int32_t* __restrict__ f,
                                  unsigned long long* __restrict__ kept) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  unsigned long long k = 0;
  if (i < n) {
    const int32_t li = Ls[i];
    int64_t lo = 0, hi = n;
    while (lo < hi) {
      const int64_t mid = (lo + hi) >> 1;
      if (g[mid] >= li)
        hi = mid;
      else
        lo = mid + 1;
    }
    const int64_t fi = max(lo, i + 1);  // g_j < L_j <= L_i for j <= i
    f[i] = (int32_t)fi;
    k = (unsigned long long)(n - fi);
  }
  for (int o = 16; o; o >>= 1) k += __shfl_down_sync(kFull, k, o);
  if ((threadIdx.x & 31) == 0 && k) atomicAdd(kept, k);
}

// Order-preserving map between doubles and uint64 keys (-inf .. +inf).
__device__ __forceinline__ uint64_t dkey(double x) {
  const uint64_t b = (uint64_t)__double_as_longlong(x);
  return (b >> 63) ? ~b : (b | 0x8000000000000000ull);
}
__device__ __forceinline__ double kdbl(uint64_t k) {
  return __longlong_as_double((long long)((k >> 63) ? (k & 0x7fffffffffffffffull) : ~k));
}

// Smallest double t with fl(s - t) <= -m; s_j is active against row s iff
// s_j < t. fl(s - t) is non-increasing in t (exact difference decreasing,
// rounding monotone), so a binary search over the ordered keys between -inf
// (fl = +inf, active) and +inf (fl = -inf) finds it exactly in 64 steps —
// also where fl(s - t) is flat over many ulps (s + m ~ 0). NaN s -> NaN and
// s = -inf -> -inf: never active, as the reference's NaN/-inf hinge.
__device__ __forceinline__ double hinge_threshold(double s, double m) {
  if (isnan(s) || s == -CUDART_INF) return s;
  uint64_t lo = dkey(-CUDART_INF), hi = dkey(CUDART_INF);
  while (hi - lo > 1) {
    const uint64_t mid = lo + ((hi - lo) >> 1);
    if (__dsub_rn(s, kdbl(mid)) <= -m)
      hi = mid;
    else
      lo = mid;
  }
  return kdbl(hi);
}

__global__ void prep_kernel(const uint32_t* __restrict__ perm, const double* __restrict__ s,
                            int64_t n, double m, double* __restrict__ ss, double* __restrict__ T,
                            int32_t* __restrict__ cs) {
  const int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (k >= n) return;
  const double v = s[perm[k]];
  ss[k] = v;
  T[k] = hinge_threshold(v, m);
  cs[k] = 0;
}

// Per 256-prompt tile of the sorted order: its scores and its hinge
// thresholds each sorted ascending (bitonic in shared memory; padding +inf
// scores, -inf thresholds), and whether any of them is NaN (such a tile keeps
// the pair-by-pair path). In a fully kept tile (I, J) a row's active count is
// then #{s_j < T_i} = lower_bound over tile J's sorted scores, and a column's
// #{T_i > s_j} = 256 - upper_bound over tile I's sorted thresholds: two
// 8-step binary searches per thread instead of 256 compares + ballots.
__global__ void __launch_bounds__(kT) tile_sort_kernel(const double* __restrict__ ss,
                                                       const double* __restrict__ T, int64_t n,
                                                       double* __restrict__ srtS, double* __restrict__ srtT,
                                                       int* __restrict__ nanflag) {
  __shared__ double a[kT], b[kT];
  const int tid = threadIdx.x;
  const int64_t k = (int64_t)blockIdx.x * kT + tid;
  const double x = k < n ? ss[k] : CUDART_INF;
  const double y = k < n ? T[k] : -CUDART_INF;
  const int bad = __syncthreads_or(isnan(x) || isnan(y));
  a[tid] = x;
  b[tid] = y;
  __syncthreads();
  for (int kk = 2; kk <= kT; kk <<= 1) {
    for (int j = kk >> 1; j > 0; j >>= 1) {
      const int partner = tid ^ j;
      if (partner > tid) {
        const bool up = (tid & kk) == 0;
        const double a0 = a[tid], a1 = a[partner], b0 = b[tid], b1 = b[partner];
        if ((a1 < a0) == up) {
          a[tid] = a1;
          a[partner] = a0;
        }
        if ((b1 < b0) == up) {
          b[tid] = b1;
          b[partner] = b0;
        }
      }
      __syncthreads();
    }
  }
  srtS[k] = a[tid];
  srtT[k] = b[tid];
  if (tid == 0) nanflag[blockIdx.x] = bad;
}

// number of entries of the ascending a[0..kT) below x (or <= x)
template <bool LE>
__device__ __forceinline__ int rank_in(const double* a, double x) {
  const double last = a[kT - 1];
  if (LE ? (last <= x) : (last < x)) return kT;  // (the lifting below reaches kT - 1 at most)
  int pos = 0;
#pragma unroll
  for (int step = kT / 2; step; step >>= 1) {
    const double v = a[pos + step - 1];
    if (LE ? (v <= x) : (v < x)) pos += step;
  }
  return pos;
}

template <int KIND>  // 0 fully kept, 1 partially kept, 2 diagonal
__device__ __forceinline__ void tile_columns(const double* sS, double Ti, int64_t fi, int64_t J0,
                                             int tid, int lane, int& cnt, int* sC) {
  for (int jb = 0; jb < kT; jb += 32) {
    int colacc = 0;
#pragma unroll
    for (int jj = 0; jj < 32; ++jj) {
      const int j = jb + jj;
      bool act = sS[j] < Ti;
      if (KIND >= 1) act = act && (J0 + j >= fi);
      if (KIND == 2) act = act && (j > tid);
      cnt += act;
      const int pc = __popc(__ballot_sync(kFull, act));
      colacc = (lane == jj) ? pc : colacc;
    }
    if (colacc) atomicAdd(&sC[jb + lane], colacc);
  }
}

// Tiles are taken in chunks of kChunk consecutive tiles of the enumeration
// (row tile I, columns J, J + 1, ...): the row side — scores, thresholds,
// first kept columns, the row tile's sorted thresholds — is loaded once per
// row of the chunk, and each row's count goes to cs once per row of the
// chunk. Per tile: its columns, the counts, the column atomics and the
// tile's loss part (one per tile, as before: the fixed-order sum is
// independent of the chunking).
constexpr int kChunk = 4;

__global__ void __launch_bounds__(kT) allpairs_sorted_kernel(
    const double* __restrict__ ss, const double* __restrict__ T, const int32_t* __restrict__ f,
    int64_t n, int64_t nt, double m, int64_t t0, int64_t t1, int32_t* __restrict__ cs,
    unsigned long long* __restrict__ counters, double* __restrict__ loss_part,
    const double* __restrict__ srtS, const double* __restrict__ srtT, const int* __restrict__ nanflag) {
  __shared__ __align__(16) double sS[kT];
  __shared__ __align__(16) double sSs[kT], sTs[kT];  // the tiles' sorted scores / thresholds
  __shared__ int sC[kT];
  __shared__ double redd[kT / 32];
  __shared__ unsigned long long redu[kT / 32];
  const int tid = threadIdx.x, lane = tid & 31;
  unsigned long long kept_acc = 0, act_acc = 0;
  const int64_t nchunks = (t1 - t0 + kChunk - 1) / kChunk;
  for (int64_t c = blockIdx.x; c < nchunks; c += gridDim.x) {
    const int64_t tA = t0 + c * kChunk, tB = min(t1, tA + kChunk);
    int64_t I, J;
    tile_of(tA, nt, &I, &J);
    int64_t i = 0, fi = 0, fmin = 0, fmax = 0;
    bool row_ok = false, nanI = false;
    double si = 0.0, Ti = 0.0;
    int rowcnt = 0;
    for (int64_t t = tA; t < tB; ++t, ++J) {
      if (J == nt || t == tA) {  // a new row tile: flush the last one's counts, load its row side
        if (t != tA) {
          if (row_ok && rowcnt) atomicAdd(&cs[i], rowcnt);
          rowcnt = 0;
          ++I;
          J = I;
        }
        i = I * kT + tid;
        row_ok = i < n;
        si = row_ok ? ss[i] : 0.0;
        Ti = row_ok ? T[i] : -CUDART_INF;
        fi = row_ok ? (int64_t)f[i] : INT64_MAX;
        fmin = f[I * kT];
        fmax = f[min(n, (I + 1) * kT) - 1];
        nanI = nanflag[I] != 0;
        sTs[tid] = srtT[I * kT + tid];  // (read only after this tile's first barrier)
      }
      const int64_t J0 = J * kT;
      const int64_t jn = min((int64_t)kT, n - J0);
      const bool diag = I == J;
      // fully kept and NaN-free: counts by rank in the tiles' sorted scores / thresholds
      const bool ranked = !diag && fmax <= J0 && !nanI && !nanflag[J];
      sS[tid] = (tid < jn) ? ss[J0 + tid] : CUDART_NAN;
      if (ranked)
        sSs[tid] = srtS[J0 + tid];
      else
        sC[tid] = 0;
      __syncthreads();
      int cnt = 0;
      if (ranked) {
        cnt = row_ok ? rank_in<false>(sSs, Ti) : 0;
        sC[tid] = kT - rank_in<true>(sTs, sS[tid]);  // (a padding column's count is never read)
      } else if (diag) {
        tile_columns<2>(sS, Ti, fi, J0, tid, lane, cnt, sC);
      } else if (fmax <= J0) {
        tile_columns<0>(sS, Ti, fi, J0, tid, lane, cnt, sC);
      } else if (fmin < J0 + jn) {
        tile_columns<1>(sS, Ti, fi, J0, tid, lane, cnt, sC);
      }
      __syncthreads();
      if (row_ok) {
        const int64_t from = max(max(fi, J0), diag ? i + 1 : (int64_t)0);
        kept_acc += (unsigned long long)max((int64_t)0, J0 + jn - from);
        act_acc += (unsigned)cnt;
        rowcnt += cnt;
      }
      double part = cnt ? __dmul_rn(i32_to_f64(cnt), __dadd_rn(si, m)) : 0.0;
      if (tid < jn && sC[tid]) {
        atomicSub(&cs[J0 + tid], sC[tid]);
        part = __dsub_rn(part, __dmul_rn(i32_to_f64(sC[tid]), sS[tid]));
      }
      // no trailing barrier: red, sS, sSs, sTs and sC are next written
      // before a barrier that every thread reaches after this one
      const double tl = block_sum_fixed<double, false>(part, redd);
      if (tid == 0) loss_part[t - t0] = tl;
    }
    if (row_ok && rowcnt) atomicAdd(&cs[i], rowcnt);
  }
  const unsigned long long k = block_sum_fixed<unsigned long long>(kept_acc, redu);
  const unsigned long long a = block_sum_fixed<unsigned long long>(act_acc, redu);
  if (tid == 0) {
    atomicAdd(&counters[0], k);
    atomicAdd(&counters[1], a);
  }
}

__global__ void scatter_kernel(const uint32_t* __restrict__ perm, const int32_t* __restrict__ cs,
                               int64_t n, int32_t* __restrict__ coeff) {
  const int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (k < n && cs[k]) atomicAdd(&coeff[perm[k]], cs[k]);
}

int sm_count() {
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  return sms;
}

}  // namespace

size_t pair_plan_scratch_bytes(int64_t n) {
  const int64_t np = ceil_div(std::max<int64_t>(n, 1), kT) * kT;  // whole tiles
  return (size_t)n * (4 + 4 + 4 + 4 + 8 + 8 + 4) + (size_t)np * 16 + (size_t)(np / kT) * 4 + 3 * 256 +
         sort_scratch_bytes(n) + 8192;
}

int build_pair_plan(pars_ctx* ctx, const int32_t* d_L, const int32_t* d_dmin, int64_t n,
                    PairPlanDev* p, void* scratch, cudaStream_t st) {
  char* q = static_cast<char*>(scratch);
  auto take = [&](size_t bytes) {
    char* r = q;
    q += (bytes + 255) & ~(size_t)255;
    return r;
  };
  p->n = n;
  p->perm = (uint32_t*)take(n * 4);
  p->Ls = (int32_t*)take(n * 4);
  p->f = (int32_t*)take(n * 4);
  int32_t* g = (int32_t*)take(n * 4);
  p->ss = (double*)take(n * 8);
  p->T = (double*)take(n * 8);
  p->cs = (int32_t*)take(n * 4);
  const int64_t np = ceil_div(std::max<int64_t>(n, 1), kT) * kT;
  p->srtS = (double*)take(np * 8);
  p->srtT = (double*)take(np * 8);
  p->nanflag = (int*)take(np / kT * 4);
  double* zeros = p->ss;  // reuse: all-equal primary keys for the length sort
  int32_t* flag = (int32_t*)take(64);
  unsigned long long* kept = (unsigned long long*)take(64);
  void* sort_scratch = take(sort_scratch_bytes(n));
  if (n <= 0) {
    p->kept = 0;
    p->monotone = true;
    return PARS_OK;
  }
  PARS_CUDA_CHECK(cudaMemsetAsync(zeros, 0, n * 8, st));
  PARS_CUDA_CHECK(cudaMemsetAsync(flag, 0, 4, st));
  PARS_CUDA_CHECK(cudaMemsetAsync(kept, 0, 8, st));
  // stable sort by length (ties keep input order)
  PARS_TRY(launch_priority_sort(ctx, zeros, nullptr, reinterpret_cast<const uint32_t*>(d_L), n,
                                p->perm, sort_scratch, st));
  const unsigned blocks = (unsigned)ceil_div(n, 256);
  plan_gather_kernel<<<blocks, 256, 0, st>>>(p->perm, d_L, d_dmin, n, p->Ls, g);
  plan_check_kernel<<<blocks, 256, 0, st>>>(g, n, flag);
  plan_first_kernel<<<blocks, 256, 0, st>>>(g, p->Ls, n, p->f, kept);
  count_launch(ctx, 3);
  PARS_CUDA_CHECK(cudaGetLastError());
  int32_t bad = 0;
  unsigned long long kk = 0;
  PARS_CUDA_CHECK(cudaMemcpyAsync(&bad, flag, 4, cudaMemcpyDeviceToHost, st));
  PARS_CUDA_CHECK(cudaMemcpyAsync(&kk, kept, 8, cudaMemcpyDeviceToHost, st));
  PARS_CUDA_CHECK(cudaStreamSynchronize(st));
  p->monotone = bad == 0;
  p->kept = kk;
  return PARS_OK;
}

int launch_allpairs_sorted(pars_ctx* ctx, const PairPlanDev& p, const double* d_scores,
                           double margin, int64_t t0, int64_t t1, int32_t* d_coeff,
                           unsigned long long* d_counters, double* d_loss_part, cudaStream_t st) {
  const int64_t n = p.n;
  if (n < 2 || t1 <= t0) return PARS_OK;
  const unsigned blocks = (unsigned)ceil_div(n, 256);
  prep_kernel<<<blocks, 256, 0, st>>>(p.perm, d_scores, n, margin, p.ss, p.T, p.cs);
  const int64_t nt = ceil_div(n, kT);
  tile_sort_kernel<<<(unsigned)nt, kT, 0, st>>>(p.ss, p.T, n, p.srtS, p.srtT, p.nanflag);
  static const int per_sm = [] {  // resident CTAs per SM: one wave of chunk walkers
    int k = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&k, allpairs_sorted_kernel, kT, 0);
    return std::max(k, 1);
  }();
  const int64_t grid = std::min<int64_t>(ceil_div(t1 - t0, kChunk), (int64_t)sm_count() * per_sm);
  allpairs_sorted_kernel<<<(unsigned)grid, kT, 0, st>>>(p.ss, p.T, p.f, n, nt, margin, t0, t1,
                                                        p.cs, d_counters, d_loss_part, p.srtS, p.srtT,
                                                        p.nanflag);
  scatter_kernel<<<blocks, 256, 0, st>>>(p.perm, p.cs, n, d_coeff);
  count_launch(ctx, 4);
  PARS_CUDA_CHECK(cudaGetLastError());
  return PARS_OK;
}

}  // namespace pars_b200
