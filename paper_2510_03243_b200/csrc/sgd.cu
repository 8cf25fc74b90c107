// Reference-equivalent pairwise SGD epoch, bit-identical to train.cpp.
//
// Reference (train.cpp): per 128-pair batch (:156-165), pairwise_loss_grad
// (:34-44) scores both prompts with the current weights
// (s = sum_{idx ascending} w[idx]*v, + bias), takes the margin loss, and on
// the active branch does grad[idx] -= y*v (prompt a) then += y*v (prompt b)
// in pair order; apply (:141-151) does w[d] -= (lr/batch_n) * grad[d] for
// grad[d] != 0. epoch_loss sums the per-pair losses in pair order (:160).
//
// Every floating-point operation and its order is reproduced:
//   * scores: one thread per prompt slot runs the sequential __dadd_rn chain
//     over its CSR row (rows are stored in ascending index order);
//   * gradient: the per-index accumulation order is (pair, a-before-b). A
//     per-batch CSC (entries sorted by index, stable in slot order) is built
//     for the whole epoch up front, in parallel over batches
//     (sgd_build_kernel). The step kernel then folds each index's entries in
//     order — one thread per touched index, no atomics, no reordering — and
//     applies the update right away;
//   * the epoch loss is one sequential chain in pair order.
// The 782 dependent steps run inside ONE persistent CTA (sgd_epoch_kernel)
// with the weights resident in shared memory, so a step costs three
// __syncthreads instead of kernel launches.
#include <cuda_runtime.h>

#include <algorithm>
#include <vector>

#include "common.cuh"
#include "pairs.cuh"

namespace pars_b200 {

namespace {

constexpr int kBuildThreads = 256;
constexpr int kStepThreads = 1024;

// One CTA per batch: stable counting sort of the batch's (slot, idx, val)
// entries by idx. Slots are processed in order; within one slot (one CSR row)
// indices are unique, so the cursor updates never collide.
__global__ void __launch_bounds__(kBuildThreads) sgd_build_kernel(
    const int64_t* __restrict__ rp, const uint32_t* __restrict__ idx,
    const double* __restrict__ val, uint32_t dim, const uint32_t* __restrict__ pa,
    const uint32_t* __restrict__ pb, int64_t npairs, int32_t B,
    const int64_t* __restrict__ ent_off, uint16_t* __restrict__ ent_slot,
    double* __restrict__ ent_val, uint32_t* __restrict__ run_d, uint32_t* __restrict__ run_beg,
    uint32_t* __restrict__ nruns) {
  extern __shared__ uint32_t cur[];  // [dim] counts -> cursors
  __shared__ uint32_t part[kBuildThreads];
  __shared__ uint32_t rpart[kBuildThreads];
  const int64_t q = blockIdx.x;
  const int64_t p0 = q * B;
  const int bn = (int)imin64(B, npairs - p0);
  const int S = 2 * bn;
  const int64_t base = ent_off[q];
  for (uint32_t d = threadIdx.x; d < dim; d += kBuildThreads) cur[d] = 0;
  __syncthreads();
  for (int k = 0; k < S; ++k) {
    const uint32_t r = (k & 1) ? pb[p0 + (k >> 1)] : pa[p0 + (k >> 1)];
    for (int64_t e = rp[r] + threadIdx.x; e < rp[r + 1]; e += kBuildThreads)
      atomicAdd(&cur[idx[e]], 1u);
  }
  __syncthreads();
  // exclusive scan of counts over [0, dim) in contiguous chunks
  const uint32_t chunk = (dim + kBuildThreads - 1) / kBuildThreads;
  const uint32_t d0 = min(dim, threadIdx.x * chunk), d1 = min(dim, d0 + chunk);
  uint32_t s = 0, rs = 0;
  for (uint32_t d = d0; d < d1; ++d) {
    s += cur[d];
    rs += cur[d] != 0;
  }
  part[threadIdx.x] = s;
  rpart[threadIdx.x] = rs;
  __syncthreads();
  for (int o = 1; o < kBuildThreads; o <<= 1) {
    uint32_t v = threadIdx.x >= (unsigned)o ? part[threadIdx.x - o] : 0u;
    uint32_t w = threadIdx.x >= (unsigned)o ? rpart[threadIdx.x - o] : 0u;
    __syncthreads();
    part[threadIdx.x] += v;
    rpart[threadIdx.x] += w;
    __syncthreads();
  }
  uint32_t run = part[threadIdx.x] - s, rrun = rpart[threadIdx.x] - rs;
  uint32_t* rd = run_d + q * (int64_t)dim;
  uint32_t* rb = run_beg + q * (int64_t)dim;
  for (uint32_t d = d0; d < d1; ++d) {
    const uint32_t c = cur[d];
    if (c) {
      rd[rrun] = d;
      rb[rrun] = run;
      ++rrun;
    }
    cur[d] = run;
    run += c;
  }
  if (threadIdx.x == kBuildThreads - 1) nruns[q] = rrun;
  __syncthreads();
  for (int k = 0; k < S; ++k) {
    const uint32_t r = (k & 1) ? pb[p0 + (k >> 1)] : pa[p0 + (k >> 1)];
    for (int64_t e = rp[r] + threadIdx.x; e < rp[r + 1]; e += kBuildThreads) {
      const uint32_t d = idx[e];
      const uint32_t pos = cur[d];
      cur[d] = pos + 1;
      ent_slot[base + pos] = (uint16_t)k;
      ent_val[base + pos] = val[e];
    }
    __syncthreads();
  }
}

// The whole epoch in one CTA. Shared: W[dim], score[2B], loss[B], act[B], yb[B].
__global__ void __launch_bounds__(kStepThreads) sgd_epoch_kernel(
    const int64_t* __restrict__ rp, const uint32_t* __restrict__ idx,
    const double* __restrict__ val, uint32_t dim, const uint32_t* __restrict__ pa,
    const uint32_t* __restrict__ pb, const int32_t* __restrict__ py, int64_t npairs, int32_t B,
    double lr, double margin, double bias, const int64_t* __restrict__ ent_off,
    const uint16_t* __restrict__ ent_slot, const double* __restrict__ ent_val,
    const uint32_t* __restrict__ run_d, const uint32_t* __restrict__ run_beg,
    const uint32_t* __restrict__ nruns, double* __restrict__ w_io, double* __restrict__ loss_out,
    unsigned long long* __restrict__ active_out) {
  extern __shared__ __align__(16) unsigned char sm[];
  double* W = reinterpret_cast<double*>(sm);
  double* score = W + dim;
  double* lossb = score + 2 * B;
  int32_t* yb = reinterpret_cast<int32_t*>(lossb + B);
  uint8_t* act = reinterpret_cast<uint8_t*>(yb + B);
  const int tid = threadIdx.x;
  for (uint32_t d = tid; d < dim; d += kStepThreads) W[d] = w_io[d];
  double epoch_loss = 0.0;  // thread kStepThreads-1 only
  unsigned long long active = 0;
  const int64_t nb = (npairs + B - 1) / B;
  __syncthreads();
  for (int64_t q = 0; q < nb; ++q) {
    const int64_t p0 = q * B;
    const int bn = (int)imin64(B, npairs - p0);
    // phase A: scores of both prompts of every pair (scorer.cpp:40-42)
    for (int k = tid; k < 2 * bn; k += kStepThreads) {
      const uint32_t r = (k & 1) ? pb[p0 + (k >> 1)] : pa[p0 + (k >> 1)];
      const int64_t e0 = rp[r], e1 = rp[r + 1];
      double s = 0.0;
      int64_t e = e0;
      for (; e + 4 <= e1; e += 4) {
        const uint32_t i0 = idx[e], i1 = idx[e + 1], i2 = idx[e + 2], i3 = idx[e + 3];
        const double v0 = val[e], v1 = val[e + 1], v2 = val[e + 2], v3 = val[e + 3];
        s = __dadd_rn(s, __dmul_rn(W[i0], v0));
        s = __dadd_rn(s, __dmul_rn(W[i1], v1));
        s = __dadd_rn(s, __dmul_rn(W[i2], v2));
        s = __dadd_rn(s, __dmul_rn(W[i3], v3));
      }
      for (; e < e1; ++e) s = __dadd_rn(s, __dmul_rn(W[idx[e]], val[e]));
      score[k] = __dadd_rn(s, bias);
    }
    __syncthreads();
    // phase B: margin loss per pair (pairs.hpp:27-31)
    for (int p = tid; p < bn; p += kStepThreads) {
      const int32_t y = py[p0 + p];
      const double v = __dadd_rn(__dmul_rn(-(double)y, __dsub_rn(score[2 * p], score[2 * p + 1])),
                                 margin);
      const double l = v > 0.0 ? v : 0.0;
      lossb[p] = l;
      act[p] = l > 0.0;
      yb[p] = y;
    }
    __syncthreads();
    // phase C: epoch loss chain (last thread) || per-index gradient fold +
    // update (apply, train.cpp:141-151)
    if (tid == kStepThreads - 1) {
      for (int p = 0; p < bn; ++p) {
        epoch_loss = __dadd_rn(epoch_loss, lossb[p]);
        active += act[p];
      }
    } else {
      const double scale = __ddiv_rn(lr, (double)bn);
      const uint32_t R = nruns[q];
      const int64_t base = ent_off[q];
      const int64_t tot = ent_off[q + 1] - base;
      const uint32_t* rd = run_d + q * (int64_t)dim;
      const uint32_t* rb = run_beg + q * (int64_t)dim;
      for (uint32_t r = tid; r < R; r += kStepThreads - 1) {
        const uint32_t d = rd[r];
        const int64_t b = rb[r];
        const int64_t e = (r + 1 < R) ? (int64_t)rb[r + 1] : tot;
        double g = 0.0;
        for (int64_t k = b; k < e; ++k) {
          const uint32_t slot = ent_slot[base + k];
          const int p = slot >> 1;
          if (act[p]) {
            const double v = ent_val[base + k];
            const double yv = yb[p] > 0 ? v : -v;  // (double)y * v, exact
            g = (slot & 1) ? __dadd_rn(g, yv) : __dsub_rn(g, yv);
          }
        }
        if (g != 0.0) W[d] = __dsub_rn(W[d], __dmul_rn(scale, g));
      }
    }
    __syncthreads();
  }
  for (uint32_t d = tid; d < dim; d += kStepThreads) w_io[d] = W[d];
  if (tid == kStepThreads - 1) {
    *loss_out = epoch_loss;
    *active_out = active;
  }
}

}  // namespace

size_t sgd_scratch_bytes(int64_t nbatches, int32_t batch, uint32_t dim, int64_t max_entries) {
  (void)batch;
  size_t b = 0;
  b += (size_t)(nbatches + 1) * 8 + 256;
  b += (size_t)max_entries * 2 + 256;
  b += (size_t)max_entries * 8 + 256;
  b += 2 * (size_t)nbatches * dim * 4 + 512;
  b += (size_t)nbatches * 4 + 256;
  return b;
}

int launch_sgd_epoch(pars_ctx* ctx, const int64_t* rp, const uint32_t* idx, const double* val,
                     uint32_t dim, const uint32_t* a, const uint32_t* b, const int32_t* y,
                     int64_t npairs, int32_t B, double lr, double margin, double bias, double* w,
                     double* loss_out, unsigned long long* active_out, int64_t total,
                     void* scratch, size_t scratch_bytes, cudaStream_t st) {
  (void)scratch_bytes;
  // scratch layout: ent_off (filled by caller, first), ent_slot, ent_val, run_d, run_beg, nruns
  const int64_t nb = (npairs + B - 1) / B;
  char* p = static_cast<char*>(scratch);
  auto take = [&](size_t bytes) {
    char* r = p;
    p += (bytes + 255) & ~(size_t)255;
    return r;
  };
  int64_t* ent_off = (int64_t*)take((size_t)(nb + 1) * 8);
  // the caller has uploaded ent_off[nb+1] (per-batch entry offsets, total = ent_off[nb])
  uint16_t* ent_slot = (uint16_t*)take((size_t)total * 2);
  double* ent_val = (double*)take((size_t)total * 8);
  uint32_t* run_d = (uint32_t*)take((size_t)nb * dim * 4);
  uint32_t* run_beg = (uint32_t*)take((size_t)nb * dim * 4);
  uint32_t* nruns = (uint32_t*)take((size_t)nb * 4);
  const size_t build_smem = (size_t)dim * 4;
  PARS_CUDA_CHECK(cudaFuncSetAttribute(sgd_build_kernel,
                                       cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       (int)build_smem));
  sgd_build_kernel<<<(unsigned)nb, kBuildThreads, build_smem, st>>>(
      rp, idx, val, dim, a, b, npairs, B, ent_off, ent_slot, ent_val, run_d, run_beg, nruns);
  const size_t step_smem = (size_t)dim * 8 + (size_t)B * (16 + 8 + 4 + 1) + 64;
  PARS_CUDA_CHECK(cudaFuncSetAttribute(sgd_epoch_kernel,
                                       cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       (int)step_smem));
  sgd_epoch_kernel<<<1, kStepThreads, step_smem, st>>>(rp, idx, val, dim, a, b, y, npairs, B, lr,
                                                       margin, bias, ent_off, ent_slot, ent_val,
                                                       run_d, run_beg, nruns, w, loss_out,
                                                       active_out);
  count_launch(ctx, 2);
  PARS_CUDA_CHECK(cudaGetLastError());
  return PARS_OK;
}

}  // namespace pars_b200
