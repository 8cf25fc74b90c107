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
  for (int64_t t = t0 + blockIdx.x; t < t1; t += gridDim.x) {
    int64_t I, J;
    tile_of(t, nt, &I, &J);
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
                                                    int64_t nt, int64_t ntiles,
                                                    unsigned long long* __restrict__ out) {
  __shared__ double sx[kTile], sy[kTile];
  __shared__ unsigned long long red[kTile / 32];
  const int tid = threadIdx.x;
  unsigned long long nc = 0, nd = 0, n1 = 0, n2 = 0;
  for (int64_t t = blockIdx.x; t < ntiles; t += gridDim.x) {
    int64_t I, J;
    tile_of(t, nt, &I, &J);
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

// X^T c over a CSR row range: each CTA walks its rows in order and
// accumulates c_i * v into a shared dense vector (indices within one row are
// unique, so no atomics); per-CTA partials are summed in CTA order by
// xtc_reduce_kernel -> deterministic.
__global__ void xtc_partial_kernel(const int64_t* __restrict__ rp, const uint32_t* __restrict__ idx,
                                   const double* __restrict__ val, const int32_t* __restrict__ c,
                                   int64_t r0, int64_t r1, uint32_t dim,
                                   double* __restrict__ partial) {
  extern __shared__ double g[];
  for (uint32_t d = threadIdx.x; d < dim; d += blockDim.x) g[d] = 0.0;
  __syncthreads();
  const int64_t rows = r1 - r0;
  const int64_t per = (rows + gridDim.x - 1) / gridDim.x;
  const int64_t a = r0 + (int64_t)blockIdx.x * per;
  const int64_t b = min(r1, a + per);
  for (int64_t r = a; r < b; ++r) {
    const int32_t ci = c[r];
    if (ci != 0) {
      const double cd = (double)ci;
      for (int64_t k = rp[r] + threadIdx.x; k < rp[r + 1]; k += blockDim.x)
        g[idx[k]] = __dadd_rn(g[idx[k]], __dmul_rn(cd, val[k]));
    }
    __syncthreads();
  }
  for (uint32_t d = threadIdx.x; d < dim; d += blockDim.x)
    partial[(int64_t)blockIdx.x * dim + d] = g[d];
}

__global__ void xtc_reduce_kernel(const double* __restrict__ partial, int nparts, uint32_t dim,
                                  double* __restrict__ grad) {
  const uint32_t d = blockIdx.x * blockDim.x + threadIdx.x;
  if (d >= dim) return;
  double s = 0.0;
  for (int p = 0; p < nparts; ++p) s = __dadd_rn(s, partial[(int64_t)p * dim + d]);
  grad[d] = s;
}

int sms_of_current() {
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  return sms;
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
               unsigned long long* out, cudaStream_t st) {
  const int64_t nt = ceil_div(n, kTile);
  const int64_t tiles = nt * (nt + 1) / 2;
  const int64_t grid = std::min<int64_t>(tiles, (int64_t)sms_of_current() * 8);
  tau_kernel<<<(unsigned)grid, kTile, 0, st>>>(x, y, n, nt, tiles, out);
  count_launch(ctx);
  PARS_CUDA_CHECK(cudaGetLastError());
  return PARS_OK;
}

int xtc_parts(int64_t rows) {
  return (int)std::max<int64_t>(1, std::min<int64_t>(sms_of_current(), ceil_div(rows, 64)));
}

int launch_xtc(pars_ctx* ctx, const int64_t* rp, const uint32_t* idx, const double* val,
               const int32_t* c, int64_t r0, int64_t r1, uint32_t dim, double* partial,
               double* grad, cudaStream_t st) {
  const int parts = xtc_parts(r1 - r0);
  const size_t smem = (size_t)dim * sizeof(double);
  if (smem > 227 * 1024) {
    set_error("X^T c: dimension %u exceeds the shared-memory accumulator", dim);
    return PARS_ERR_UNSUPPORTED;
  }
  PARS_CUDA_CHECK(cudaFuncSetAttribute(xtc_partial_kernel,
                                       cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  xtc_partial_kernel<<<parts, 256, smem, st>>>(rp, idx, val, c, r0, r1, dim, partial);
  xtc_reduce_kernel<<<(unsigned)ceil_div(dim, 256), 256, 0, st>>>(partial, parts, dim, grad);
  count_launch(ctx, 2);
  PARS_CUDA_CHECK(cudaGetLastError());
  return PARS_OK;
}

}  // namespace pars_b200
