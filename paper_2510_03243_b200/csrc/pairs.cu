// All-pairs kernels: margin-ranking loss with the Eq. 1 length-gap mask
// (C2 exhaustive / C5), Kendall tau-b pair counts, and the X^T c gradient.
//
// Reference semantics:
//   pairs.hpp:21-24 relative_length_difference, pairs.cpp:28-31 (keep iff
//   la != lb && !(rel < delta), y = la > lb ? +1 : -1), pairs.hpp:27-31
//   margin_ranking_loss, train.cpp:34-44 (grad -= y x_a, += y x_b on the
//   active branch); metrics.cpp:42-64 (tau pair counting).
//
// Design: the upper triangle of the n x n pair matrix is cut into 256 x 256
// tiles; one CTA (256 threads) owns a tile, each thread one row (score,
// length, dmin[length] in registers), the 256 columns (score, length,
// dmin[length]) staged in shared memory and read as broadcasts. The Eq. 1
// mask is the integer test |li - lj| >= dmin[max(li, lj)] where the table
// entry of the longer side is either the row's or the column's — no per-pair
// table gather. Row coefficients accumulate in registers; column coefficients
// are reduced across the warp with one REDUX (__reduce_add_sync) per column
// and across warps in shared memory; integers only, so c is exact and
// order-free. The loss is summed per thread and reduced in a fixed order
// into one partial per tile (deterministic run to run).
#include <cuda_runtime.h>

#include <algorithm>
#include <cstring>
#include <vector>
#include <cmath>

#include "common.cuh"
#include "pairs.cuh"
#include "tiles.cuh"

namespace pars_b200 {

namespace {

constexpr int kTile = kPairTile;
constexpr unsigned kFull = 0xffffffffu;

__global__ void __launch_bounds__(kTile) allpairs_kernel(
    const double* __restrict__ s, const int32_t* __restrict__ L,
    const int32_t* __restrict__ dmin, int64_t n, int64_t nt, double margin,
    int64_t t0, int64_t t1, int32_t* __restrict__ coeff,
    unsigned long long* __restrict__ counters, double* __restrict__ loss_part) {
  __shared__ double sS[kTile];
  __shared__ int32_t sL[kTile];
  __shared__ int32_t sD[kTile];
  __shared__ int32_t sC[kTile];
  __shared__ double redd[kTile / 32];
  __shared__ unsigned long long redu[kTile / 32];
  const int tid = threadIdx.x, lane = tid & 31;
  unsigned long long kept_acc = 0, act_acc = 0;
  int64_t I = 0, J = 0;
  if (t0 + blockIdx.x < t1) tile_of(t0 + blockIdx.x, nt, &I, &J);
  for (int64_t t = t0 + blockIdx.x; t < t1; t += gridDim.x) {
    if (t != t0 + blockIdx.x) tile_advance(gridDim.x, nt, I, J);
    const int64_t gi = I * kTile + tid;
    const bool row_ok = gi < n;
    const double si = row_ok ? s[gi] : 0.0;
    const int32_t li = row_ok ? L[gi] : 0;
    const int32_t dmi = row_ok ? dmin[li] : 0x7fffffff;
    {
      const int64_t gj = J * kTile + tid;
      const bool ok = gj < n;
      sS[tid] = ok ? s[gj] : 0.0;
      const int32_t lj = ok ? L[gj] : 0;
      sL[tid] = lj;
      sD[tid] = ok ? dmin[lj] : 0x7fffffff;
      sC[tid] = 0;
    }
    __syncthreads();
    const bool diag = (I == J);
    const int jmax = (int)imin64(kTile, n - J * kTile);
    int32_t ci = 0, kept = 0, act = 0, colacc = 0;
    double loss = 0.0;
    for (int jb = 0; jb < kTile; jb += 32) {
#pragma unroll 8
      for (int jj = 0; jj < 32; ++jj) {
        const int j = jb + jj;
        const int32_t lj = sL[j];
        const int32_t d = li - lj;
        const bool gt = d > 0;
        const int32_t dm = gt ? dmi : sD[j];
        const int32_t ad = gt ? d : -d;
        bool keep = row_ok && (j < jmax) && (ad >= dm) && (!diag || j > tid);
        const double diff = si - sS[j];
        const double h = __dadd_rn(gt ? -diff : diff, margin);
        const bool a = keep && (h > 0.0);
        kept += keep;
        act += a;
        if (a) loss += h;
        const int32_t y = gt ? 1 : -1;
        if (a) ci -= y;
        const int32_t cj = __reduce_add_sync(kFull, a ? y : 0);
        if (lane == jj) colacc = cj;
      }
      atomicAdd(&sC[jb + lane], colacc);
    }
    __syncthreads();
    if (row_ok && ci != 0) atomicAdd(&coeff[gi], ci);
    {
      const int64_t gj = J * kTile + tid;
      if (gj < n && sC[tid] != 0) atomicAdd(&coeff[gj], sC[tid]);
    }
    kept_acc += (unsigned)kept;
    act_acc += (unsigned)act;
    const double tl = block_sum_fixed<double>(loss, redd);
    if (tid == 0) loss_part[t - t0] = tl;
  }
  const unsigned long long k = block_sum_fixed<unsigned long long>(kept_acc, redu);
  const unsigned long long a = block_sum_fixed<unsigned long long>(act_acc, redu);
  if (tid == 0) {
    atomicAdd(&counters[0], k);
    atomicAdd(&counters[1], a);
  }
}

// Fixed-order reduction of the per-tile loss partials.
__global__ void sum_partials_kernel(const double* __restrict__ p, int64_t n, double* out) {
  __shared__ double red[32];
  double v = 0.0;
  // thread-strided then fixed tree: deterministic for a given n
  for (int64_t i = threadIdx.x; i < n; i += blockDim.x) v += p[i];
  const double r = block_sum_fixed<double>(v, red);
  if (threadIdx.x == 0) *out = r;
}

// Kendall tau-b counts (metrics.cpp:47-62): n_c, n_d, n1 (ties in x), n2.
__global__ void __launch_bounds__(kTile) tau_kernel(const double* __restrict__ x,
                                                    const double* __restrict__ y, int64_t n,
                                                    int64_t nt, int64_t t0, int64_t t1,
                                                    unsigned long long* __restrict__ out) {
  __shared__ double sx[kTile], sy[kTile];
  __shared__ unsigned long long red[kTile / 32];
  const int tid = threadIdx.x;
  unsigned long long nc = 0, nd = 0, n1 = 0, n2 = 0;
  int64_t I = 0, J = 0;
  if (t0 + blockIdx.x < t1) tile_of(t0 + blockIdx.x, nt, &I, &J);
  for (int64_t t = t0 + blockIdx.x; t < t1; t += gridDim.x) {
    if (t != t0 + blockIdx.x) tile_advance(gridDim.x, nt, I, J);
    const int64_t gi = I * kTile + tid;
    const bool row_ok = gi < n;
    const double xi = row_ok ? x[gi] : 0.0, yi = row_ok ? y[gi] : 0.0;
    const int64_t gj0 = J * kTile + tid;
    sx[tid] = gj0 < n ? x[gj0] : 0.0;
    sy[tid] = gj0 < n ? y[gj0] : 0.0;
    __syncthreads();
    const int jmax = (int)imin64(kTile, n - J * kTile);
    const int jmin = (I == J) ? tid + 1 : 0;
    uint32_t c_c = 0, c_d = 0, c_1 = 0, c_2 = 0;
    if (row_ok) {
#pragma unroll 4
      for (int j = jmin; j < jmax; ++j) {
        const double dx = xi - sx[j], dy = yi - sy[j];
        const bool tx = dx == 0.0, ty = dy == 0.0;
        c_1 += tx;
        c_2 += ty;
        const bool both = !tx && !ty;
        const bool conc = (dx > 0.0) == (dy > 0.0);
        c_c += both && conc;
        c_d += both && !conc;
      }
    }
    nc += c_c;
    nd += c_d;
    n1 += c_1;
    n2 += c_2;
    __syncthreads();
  }
  unsigned long long v[4] = {nc, nd, n1, n2};
  for (int k = 0; k < 4; ++k) {
    const unsigned long long r = block_sum_fixed<unsigned long long>(v[k], red);
    if (tid == 0) atomicAdd(&out[k], r);
  }
}

int sms_of_current() {
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  return sms;
}

// ---- X^T c through a column-major (CSC) copy of the features -------------
// The feature matrix is fixed for a whole training run, so its transpose is
// built once (stable: entries of a column in row order) and every step's
// gradient becomes one warp per column: lane-strided partial sums of
// c[row] * val in entry order, then a fixed xor-shuffle tree — deterministic
// for a given row range, with no shared-memory accumulator or per-row
// barrier. Rows [r0, r1) of a shard are found by binary search (each
// column's rows are sorted).
constexpr int kCscRows = 128;  // rows per placement block

__global__ void csc_block_count(const int64_t* __restrict__ rp, const uint32_t* __restrict__ idx,
                                int64_t rows, uint32_t dim, uint32_t* __restrict__ bcnt) {
  extern __shared__ uint32_t h[];
  for (uint32_t d = threadIdx.x; d < dim; d += blockDim.x) h[d] = 0;
  __syncthreads();
  const int64_t r0 = (int64_t)blockIdx.x * kCscRows, r1 = min(rows, r0 + kCscRows);
  for (int64_t k = rp[r0] + threadIdx.x; k < rp[r1]; k += blockDim.x) atomicAdd(&h[idx[k]], 1u);
  __syncthreads();
  for (uint32_t d = threadIdx.x; d < dim; d += blockDim.x) bcnt[(int64_t)blockIdx.x * dim + d] = h[d];
}

// per column: block offsets (exclusive over blocks) and the column total
__global__ void csc_column_scan(uint32_t* __restrict__ bcnt, int nblocks, uint32_t dim,
                                uint32_t* __restrict__ colcnt) {
  const uint32_t d = blockIdx.x * blockDim.x + threadIdx.x;
  if (d >= dim) return;
  uint32_t run = 0;
  for (int b = 0; b < nblocks; ++b) {
    const uint32_t c = bcnt[(int64_t)b * dim + d];
    bcnt[(int64_t)b * dim + d] = run;
    run += c;
  }
  colcnt[d] = run;
}

__global__ void csc_ptr_scan(const uint32_t* __restrict__ colcnt, uint32_t dim,
                             int64_t* __restrict__ ptr) {
  if (threadIdx.x != 0) return;
  int64_t run = 0;
  for (uint32_t d = 0; d < dim; ++d) {
    ptr[d] = run;
    run += colcnt[d];
  }
  ptr[dim] = run;
}

__global__ void csc_place(const int64_t* __restrict__ rp, const uint32_t* __restrict__ idx,
                          const double* __restrict__ val, int64_t rows, uint32_t dim,
                          const uint32_t* __restrict__ boff, const int64_t* __restrict__ ptr,
                          uint32_t* __restrict__ crow, double* __restrict__ cval) {
  extern __shared__ uint32_t cur[];
  for (uint32_t d = threadIdx.x; d < dim; d += blockDim.x)
    cur[d] = boff[(int64_t)blockIdx.x * dim + d];
  __syncthreads();
  const int64_t r0 = (int64_t)blockIdx.x * kCscRows, r1 = min(rows, r0 + kCscRows);
  for (int64_t r = r0; r < r1; ++r) {
    // a row's columns are unique: its entries take distinct cursors
    for (int64_t k = rp[r] + threadIdx.x; k < rp[r + 1]; k += blockDim.x) {
      const uint32_t d = idx[k];
      const int64_t pos = ptr[d] + cur[d];
      cur[d] += 1;
      crow[pos] = (uint32_t)r;
      cval[pos] = val[k];
    }
    __syncthreads();
  }
}

__device__ __forceinline__ int64_t lower_row(const uint32_t* __restrict__ rows, int64_t lo,
                                             int64_t hi, int64_t r) {
  // a task wholly above / below r (every task of a one-rank run, most of a
  // shard's) needs no search
  if (lo >= hi || (int64_t)rows[lo] >= r) return lo;
  if ((int64_t)rows[hi - 1] < r) return hi;
  while (lo < hi) {
    const int64_t mid = (lo + hi) >> 1;
    if ((int64_t)rows[mid] < r)
      lo = mid + 1;
    else
      hi = mid;
  }
  return lo;
}

// One warp per task = a fixed chunk of one column's entries (long columns —
// hot buckets present in most prompts — are split so no warp walks tens of
// thousands of dependent gathers): lane-strided partial sums in entry order,
// then a fixed xor-shuffle tree. The row range [r0, r1) clamps the chunk.
struct CscTask {
  int64_t beg, end;
  int32_t col, pad;
};

__global__ void xtc_csc_kernel(const CscTask* __restrict__ tasks, int64_t ntasks,
                               const uint32_t* __restrict__ crow, const double* __restrict__ cval,
                               const int32_t* __restrict__ c, int64_t r0, int64_t r1,
                               double* __restrict__ part) {
  const int lane = threadIdx.x & 31;
  const int64_t t = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  if (t >= ntasks) return;
  const CscTask tk = tasks[t];
  const int64_t b = lower_row(crow, tk.beg, tk.end, r0);
  const int64_t e = lower_row(crow, b, tk.end, r1);
  double s = 0.0;
  int64_t k = b + lane;
  for (; k + 96 < e; k += 128) {  // four independent gathers in flight
    const uint32_t q0 = crow[k], q1 = crow[k + 32], q2 = crow[k + 64], q3 = crow[k + 96];
    const double v0 = cval[k], v1 = cval[k + 32], v2 = cval[k + 64], v3 = cval[k + 96];
    const double p0 = __dmul_rn(i32_to_f64(c[q0]), v0), p1 = __dmul_rn(i32_to_f64(c[q1]), v1);
    const double p2 = __dmul_rn(i32_to_f64(c[q2]), v2), p3 = __dmul_rn(i32_to_f64(c[q3]), v3);
    s = __dadd_rn(__dadd_rn(__dadd_rn(__dadd_rn(s, p0), p1), p2), p3);
  }
  for (; k < e; k += 32) s = __dadd_rn(s, __dmul_rn(i32_to_f64(c[crow[k]]), cval[k]));
#pragma unroll
  for (int o = 16; o; o >>= 1) s = __dadd_rn(s, __shfl_xor_sync(0xffffffffu, s, o));
  if (lane == 0) part[t] = s;
}

// column d = the sum of its tasks' partials, in task order
__global__ void xtc_task_reduce(const int64_t* __restrict__ col_task, const double* __restrict__ part,
                                uint32_t dim, double* __restrict__ grad) {
  const uint32_t d = blockIdx.x * blockDim.x + threadIdx.x;
  if (d >= dim) return;
  double s = 0.0;
  for (int64_t t = col_task[d]; t < col_task[d + 1]; ++t) s = __dadd_rn(s, part[t]);
  grad[d] = s;
}

}  // namespace

int64_t allpairs_tile_count(int64_t n) {
  const int64_t nt = ceil_div(n, kTile);
  return nt * (nt + 1) / 2;
}

int launch_allpairs(pars_ctx* ctx, const double* s, const int32_t* L, const int32_t* dmin,
                    int64_t n, double margin, int64_t t0, int64_t t1, int32_t* coeff,
                    unsigned long long* counters, double* loss_part, cudaStream_t st) {
  if (t1 <= t0 || n < 2) return PARS_OK;
  const int64_t nt = ceil_div(n, kTile);
  const int64_t tiles = t1 - t0;
  const int64_t grid = std::min<int64_t>(tiles, (int64_t)sms_of_current() * 8);
  allpairs_kernel<<<(unsigned)grid, kTile, 0, st>>>(s, L, dmin, n, nt, margin, t0, t1, coeff,
                                                    counters, loss_part);
  count_launch(ctx);
  PARS_CUDA_CHECK(cudaGetLastError());
  return PARS_OK;
}

int launch_sum_partials(pars_ctx* ctx, const double* p, int64_t n, double* out, cudaStream_t st) {
  sum_partials_kernel<<<1, 1024, 0, st>>>(p, n, out);
  count_launch(ctx);
  PARS_CUDA_CHECK(cudaGetLastError());
  return PARS_OK;
}

int launch_tau(pars_ctx* ctx, const double* x, const double* y, int64_t n,
               unsigned long long* out, cudaStream_t st, int64_t t0, int64_t t1) {
  const int64_t nt = ceil_div(n, kTile);
  const int64_t tiles = nt * (nt + 1) / 2;
  if (t1 < 0 || t1 > tiles) t1 = tiles;
  t0 = std::max<int64_t>(0, t0);
  if (t1 <= t0) return PARS_OK;
  const int64_t grid = std::min<int64_t>(t1 - t0, (int64_t)sms_of_current() * 8);
  tau_kernel<<<(unsigned)grid, kTile, 0, st>>>(x, y, n, nt, t0, t1, out);
  count_launch(ctx);
  PARS_CUDA_CHECK(cudaGetLastError());
  return PARS_OK;
}

size_t csc_scratch_bytes(int64_t rows, uint32_t dim) {
  return (size_t)ceil_div(std::max<int64_t>(rows, 1), kCscRows) * dim * 4 + (size_t)dim * 4 + 256;
}

int build_csc(pars_ctx* ctx, const int64_t* rp, const uint32_t* idx, const double* val,
              int64_t rows, uint32_t dim, void* scratch, int64_t* ptr, uint32_t* crow,
              double* cval, cudaStream_t st) {
  if (rows <= 0) return PARS_OK;
  const int nb = (int)ceil_div(rows, kCscRows);
  uint32_t* bcnt = static_cast<uint32_t*>(scratch);
  uint32_t* colcnt = bcnt + (size_t)nb * dim;
  const size_t sm = (size_t)dim * 4;
  PARS_CUDA_CHECK(cudaFuncSetAttribute(csc_block_count, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm));
  PARS_CUDA_CHECK(cudaFuncSetAttribute(csc_place, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm));
  csc_block_count<<<nb, 256, sm, st>>>(rp, idx, rows, dim, bcnt);
  csc_column_scan<<<(unsigned)ceil_div(dim, 256), 256, 0, st>>>(bcnt, nb, dim, colcnt);
  csc_ptr_scan<<<1, 32, 0, st>>>(colcnt, dim, ptr);
  csc_place<<<nb, 256, sm, st>>>(rp, idx, val, rows, dim, bcnt, ptr, crow, cval);
  count_launch(ctx, 4);
  PARS_CUDA_CHECK(cudaGetLastError());
  return PARS_OK;
}

int launch_xtc_csc(pars_ctx* ctx, const void* tasks, int64_t ntasks, const int64_t* col_task,
                   const uint32_t* crow, const double* cval, const int32_t* c, int64_t r0,
                   int64_t r1, uint32_t dim, double* part, double* grad, cudaStream_t st) {
  xtc_csc_kernel<<<(unsigned)ceil_div(ntasks * 32, 256), 256, 0, st>>>(
      static_cast<const CscTask*>(tasks), ntasks, crow, cval, c, r0, r1, part);
  xtc_task_reduce<<<(unsigned)ceil_div(dim, 256), 256, 0, st>>>(col_task, part, dim, grad);
  count_launch(ctx, 2);
  PARS_CUDA_CHECK(cudaGetLastError());
  return PARS_OK;
}

size_t csc_task_bytes() { return sizeof(CscTask); }

// Host: split every column [ptr[d], ptr[d+1]) into chunks of at most `chunk`
// entries. Fills task records (packed CscTask) and col_task[dim+1].
int64_t make_csc_tasks(const int64_t* ptr, uint32_t dim, int64_t chunk, std::vector<char>& tasks,
                       std::vector<int64_t>& col_task) {
  std::vector<CscTask> t;
  col_task.assign((size_t)dim + 1, 0);
  for (uint32_t d = 0; d < dim; ++d) {
    col_task[d] = (int64_t)t.size();
    for (int64_t b = ptr[d]; b < ptr[d + 1]; b += chunk)
      t.push_back(CscTask{b, std::min(ptr[d + 1], b + chunk), (int32_t)d, 0});
  }
  col_task[dim] = (int64_t)t.size();
  tasks.resize(t.size() * sizeof(CscTask));
  if (!t.empty()) std::memcpy(tasks.data(), t.data(), tasks.size());
  return (int64_t)t.size();
}

}  // namespace pars_b200
