// The paper's comparison objectives on the GPU engine:
// one SGD epoch of PointwiseL1 or ListwiseListMLE over device features.
//
// Reference (train.cpp):
//   PointwiseL1 (:168-183, pointwise_l1_loss_grad :46-54): samples in the
//     epoch's shuffled order, batch_size per step; r = score(x) - target,
//     sign = sgn(r), grad[idx] += sign*v, bias_grad += sign, loss += |r|;
//     apply(batch_n, bias_grad) (:141-151).
//   ListwiseListMLE (:185-205, listmle_loss_grad :66-94): lists of list_size
//     rows ordered longest-first; suffix log-sum-exp lse[i], loss +=
//     lse[i]-s[i], coef[i] -= 1, coef[j] += exp(s[j]-lse[i]) for j >= i;
//     grad[idx] += coef[j]*v; batch_size lists per step, apply(lists, 0).
//
// Both are the same machine as the pairwise epoch (sgd.cu) with a different
// per-slot coefficient: a "slot" is one (sample) or (list, position); every
// batch owns a contiguous slot range. A build kernel sorts each batch's
// (slot, idx, val) entries by idx, stable in slot order, in parallel over
// batches; one persistent CTA then runs the dependent steps with the weights
// resident in shared memory:
//   A  scores of every slot: the sequential __dadd_rn chain of scorer.cpp:40-42,
//      8 lanes per slot loading and multiplying ahead of the chain;
//   B  coefficients: sgn(r) per sample; for ListMLE one thread per list runs
//      the lse chain and loss, then one thread per slot its coef[j] in the
//      reference's i order;
//   C  the epoch-loss (and bias-gradient) chain in slot order on one thread,
//      while the others fold each touched index's entries in slot order
//      (grad[idx] += coef*v) and apply w[d] -= scale*g for g != 0.
// PointwiseL1 is bit-identical to the reference (its only transcendental,
// pointwise_target = log1p(len), is input data computed by the caller on the
// host with the reference's own libm). ListMLE evaluates exp/log1p with the
// CUDA libm (<= 1 ulp from glibc's), so it matches to rounding, not bits.
#include <cuda_runtime.h>

#include <algorithm>
#include <vector>

#include "common.cuh"
#include "pairs.cuh"

namespace pars_b200 {

namespace {

constexpr int kBuildThreads = 1024;
constexpr int kBuildWarps = kBuildThreads / 32;
constexpr int kStepThreads = 1024;
constexpr int kG = 8;                        // lanes per slot in phase A
constexpr int kD = 4;                        // entries in flight per lane
constexpr int kGroups = kStepThreads / kG;

// One CTA per batch: stable counting sort of slots [soff[q], soff[q+1]) by
// feature index. Within one slot (one CSR row) indices are unique, so cursor
// updates never collide.
__global__ void __launch_bounds__(kBuildThreads) slot_build_kernel(
    const int64_t* __restrict__ rp, const uint32_t* __restrict__ idx,
    const double* __restrict__ val, uint32_t dim, const uint32_t* __restrict__ srow,
    const int64_t* __restrict__ soff, const int64_t* __restrict__ ent_off,
    uint32_t* __restrict__ ent_slot, double* __restrict__ ent_val, uint32_t* __restrict__ run_d,
    uint32_t* __restrict__ run_beg, uint32_t* __restrict__ nruns) {
  extern __shared__ uint32_t cur[];  // [dim] counts -> cursors, then [dim] slot masks
  uint32_t* mask = cur + dim;
  __shared__ uint32_t part[kBuildThreads];
  __shared__ uint32_t rpart[kBuildThreads];
  const int64_t q = blockIdx.x;
  const int64_t s0 = soff[q];
  const int S = (int)(soff[q + 1] - s0);
  const int64_t base = ent_off[q];
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  for (uint32_t d = threadIdx.x; d < dim; d += kBuildThreads) cur[d] = 0, mask[d] = 0;
  __syncthreads();
  for (int k = w; k < S; k += kBuildWarps) {  // one warp per slot
    const uint32_t r = srow[s0 + k];
    const int64_t e0 = rp[r], e1 = rp[r + 1];
    for (int64_t e = e0 + lane; e < e1; e += 32) atomicAdd(&cur[idx[e]], 1u);
  }
  __syncthreads();
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
    const uint32_t v = threadIdx.x >= (unsigned)o ? part[threadIdx.x - o] : 0u;
    const uint32_t w = threadIdx.x >= (unsigned)o ? rpart[threadIdx.x - o] : 0u;
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
  // Stable placement, kBuildWarps slots per round (one warp each): a
  // bucket's entries from the round's slots go in slot order, ranked by the
  // lower warps' bits in the bucket's slot mask (a row holds each bucket once);
  // the lowest warp of each bucket then advances its cursor.
  const uint32_t below = (1u << w) - 1u;
  for (int k0 = 0; k0 < S; k0 += kBuildWarps) {
    const int k = k0 + w;
    int64_t e0 = 0, e1 = 0;
    if (k < S) {
      const uint32_t r = srow[s0 + k];
      e0 = rp[r];
      e1 = rp[r + 1];
    }
    for (int64_t e = e0 + lane; e < e1; e += 32) atomicOr(&mask[idx[e]], 1u << w);
    __syncthreads();
    for (int64_t e = e0 + lane; e < e1; e += 32) {
      const uint32_t d = idx[e];
      const uint32_t pos = cur[d] + __popc(mask[d] & below);
      ent_slot[base + pos] = (uint32_t)k;
      ent_val[base + pos] = val[e];
    }
    __syncthreads();
    for (int64_t e = e0 + lane; e < e1; e += 32) {
      const uint32_t d = idx[e];
      const uint32_t m = mask[d];
      if (m && !(m & below)) {  // the bucket's lowest warp this round
        cur[d] += __popc(m);
        mask[d] = 0;
      }
    }
    __syncthreads();
  }
}

// log_add_exp (train.cpp:58-62): std::max / std::min argument conventions.
__device__ __forceinline__ double log_add_exp(double a, double b) {
  const double hi = a < b ? b : a;
  const double lo = b < a ? b : a;
  return __dadd_rn(hi, log1p(exp(__dsub_rn(lo, hi))));
}

// The whole epoch in one CTA. kind 0 = PointwiseL1, 1 = ListMLE (k = list size).
// Shared: W[dim], score[Smax], coef[Smax], tail[Smax], lossb[Smax], bias.
__global__ void __launch_bounds__(kStepThreads) baseline_epoch_kernel(
    int kind, const int64_t* __restrict__ rp, const uint32_t* __restrict__ idx,
    const double* __restrict__ val, uint32_t dim, const uint32_t* __restrict__ srow,
    const int64_t* __restrict__ soff, int64_t nb, int32_t k, const double* __restrict__ target,
    double lr, double bias0, int32_t smax, const int64_t* __restrict__ ent_off,
    const uint32_t* __restrict__ ent_slot, const double* __restrict__ ent_val,
    const uint32_t* __restrict__ run_d, const uint32_t* __restrict__ run_beg,
    const uint32_t* __restrict__ nruns, double* __restrict__ w_io, double* __restrict__ bias_out,
    double* __restrict__ loss_out) {
  extern __shared__ __align__(16) unsigned char sm[];
  double* W = reinterpret_cast<double*>(sm);
  double* score = W + dim;
  double* coef = score + smax;
  double* tail = coef + smax;
  double* lossb = tail + smax;
  double* bias_sh = lossb + smax;
  const int tid = threadIdx.x;
  const int gl = tid & (kG - 1), grp = tid / kG;
  for (uint32_t d = tid; d < dim; d += kStepThreads) W[d] = w_io[d];
  if (tid == 0) *bias_sh = bias0;
  double epoch_loss = 0.0;  // thread kStepThreads-1 only
  __syncthreads();
  for (int64_t q = 0; q < nb; ++q) {
    const int64_t s0 = soff[q];
    const int S = (int)(soff[q + 1] - s0);
    const double bias = *bias_sh;
    // phase A: slot scores (features.hpp:31-35 + scorer.cpp:40-42). A group
    // of kG lanes per slot loads kG*kD entries at a time (coalesced, kD
    // loads in flight per lane) and forms the products; the sequential
    // __dadd_rn chain then runs over them in entry order via shuffles.
    for (int sb = 0; sb < S; sb += kGroups) {  // warp-uniform trip count
      const int s = sb + grp;
      int64_t e = 0, e1 = 0;
      if (s < S) {
        const uint32_t r = srow[s0 + s];
        e = rp[r];
        e1 = rp[r + 1];
      }
      // Out-of-row lanes contribute +0.0, which leaves the chain unchanged
      // (acc starts at +0.0 and a round-to-nearest sum is never -0.0 unless
      // both operands are), so the adds need no predicate.
      double acc = 0.0;
      int left = (int)(e1 - e);
      while (__any_sync(0xffffffffu, left > 0)) {
        double p[kD];
#pragma unroll
        for (int j = 0; j < kD; ++j) {
          const int x = j * kG + gl;
          p[j] = x < left ? __dmul_rn(W[idx[e + x]], val[e + x]) : 0.0;
        }
#pragma unroll
        for (int j = 0; j < kD; ++j) {
#pragma unroll
          for (int i = 0; i < kG; ++i) acc = __dadd_rn(acc, __shfl_sync(0xffffffffu, p[j], i, kG));
        }
        e += kD * kG;
        left -= kD * kG;
      }
      if (s < S && gl == 0) score[s] = __dadd_rn(acc, bias);
    }
    __syncthreads();
    // phase B: per-slot coefficients and per-sample losses
    int nsamples;
    if (kind == 0) {
      nsamples = S;
      for (int s = tid; s < S; s += kStepThreads) {
        const double r = __dsub_rn(score[s], target[srow[s0 + s]]);
        coef[s] = r > 0.0 ? 1.0 : (r < 0.0 ? -1.0 : 0.0);
        lossb[s] = fabs(r);
      }
    } else {
      nsamples = S / k;
      // suffix log-sum-exp chain and loss per list (train.cpp:75-87) ...
      for (int l = tid; l < nsamples; l += kStepThreads) {
        const double* sl = score + l * k;
        double* tl = tail + l * k;
        tl[k - 1] = sl[k - 1];
        for (int i = k - 1; i-- > 0;) tl[i] = log_add_exp(sl[i], tl[i + 1]);
        double loss = 0.0;
        for (int i = 0; i < k; ++i) loss = __dadd_rn(loss, __dsub_rn(tl[i], sl[i]));
        lossb[l] = loss;
      }
      __syncthreads();
      // ... then coef[j] per slot: the reference's i-loop touches coef[j]
      // for i = 0..j in order (+= exp(s_j - lse_i), with -= 1 before i == j)
      for (int x = tid; x < S; x += kStepThreads) {
        const int l = x / k, j = x - l * k;
        const double sj = score[x];
        const double* tl = tail + l * k;
        double c = 0.0;
        for (int i = 0; i < j; ++i) c = __dadd_rn(c, exp(__dsub_rn(sj, tl[i])));
        c = __dsub_rn(c, 1.0);
        coef[x] = __dadd_rn(c, exp(__dsub_rn(sj, tl[j])));
      }
    }
    __syncthreads();
    // phase C: loss / bias-gradient chain || per-index gradient fold + apply
    const double scale = __ddiv_rn(lr, (double)nsamples);
    if (tid == kStepThreads - 1) {
      double bias_grad = 0.0;
      int p = 0;
      for (; p + 4 <= nsamples; p += 4) {
        const double l0 = lossb[p], l1 = lossb[p + 1], l2 = lossb[p + 2], l3 = lossb[p + 3];
        epoch_loss = __dadd_rn(__dadd_rn(__dadd_rn(__dadd_rn(epoch_loss, l0), l1), l2), l3);
      }
      for (; p < nsamples; ++p) epoch_loss = __dadd_rn(epoch_loss, lossb[p]);
      // sum of signs: small integers, exact in any grouping
      if (kind == 0)
        for (p = 0; p < S; ++p) bias_grad += coef[p];
      *bias_sh = __dsub_rn(bias, __dmul_rn(scale, bias_grad));
    } else {
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
        int64_t x = b;
        for (; x + 4 <= e; x += 4) {
          const uint32_t k0 = ent_slot[base + x], k1 = ent_slot[base + x + 1],
                         k2 = ent_slot[base + x + 2], k3 = ent_slot[base + x + 3];
          const double v0 = ent_val[base + x], v1 = ent_val[base + x + 1],
                       v2 = ent_val[base + x + 2], v3 = ent_val[base + x + 3];
          g = __dadd_rn(g, __dmul_rn(coef[k0], v0));
          g = __dadd_rn(g, __dmul_rn(coef[k1], v1));
          g = __dadd_rn(g, __dmul_rn(coef[k2], v2));
          g = __dadd_rn(g, __dmul_rn(coef[k3], v3));
        }
        for (; x < e; ++x) g = __dadd_rn(g, __dmul_rn(coef[ent_slot[base + x]], ent_val[base + x]));
        if (g != 0.0) W[d] = __dsub_rn(W[d], __dmul_rn(scale, g));
      }
    }
    __syncthreads();
  }
  for (uint32_t d = tid; d < dim; d += kStepThreads) w_io[d] = W[d];
  if (tid == kStepThreads - 1) {
    *loss_out = epoch_loss;
    *bias_out = *bias_sh;
  }
}

}  // namespace

size_t baseline_smem_bytes(uint32_t dim, int64_t max_slots) {
  return (size_t)dim * 8 + (size_t)max_slots * 32 + 64;
}

size_t baseline_scratch_bytes(int64_t nbatches, int64_t nslots, uint32_t dim, int64_t entries) {
  size_t b = 0;
  b += (size_t)(nbatches + 1) * 8 + 256;  // ent_off
  b += (size_t)(nbatches + 1) * 8 + 256;  // soff
  b += (size_t)nslots * 4 + 256;          // srow
  b += (size_t)entries * 4 + 256;         // ent_slot
  b += (size_t)entries * 8 + 256;         // ent_val
  b += 2 * (size_t)nbatches * dim * 4 + 512;
  b += (size_t)nbatches * 4 + 256;
  b += 64;                                // loss, bias
  return b;
}

int launch_baseline_epoch(pars_ctx* ctx, int kind, const int64_t* rp, const uint32_t* idx,
                          const double* val, uint32_t dim, const uint32_t* h_srow,
                          const int64_t* h_soff, int64_t nb, int32_t k, const double* d_target,
                          double lr, double bias, int64_t max_slots, const int64_t* h_ent_off,
                          double* d_w, double* d_bias_out, double* d_loss_out, void* scratch,
                          cudaStream_t st) {
  char* p = static_cast<char*>(scratch);
  auto take = [&](size_t bytes) {
    char* r = p;
    p += (bytes + 255) & ~(size_t)255;
    return r;
  };
  const int64_t nslots = h_soff[nb];
  const int64_t total = h_ent_off[nb];
  int64_t* ent_off = (int64_t*)take((size_t)(nb + 1) * 8);
  int64_t* soff = (int64_t*)take((size_t)(nb + 1) * 8);
  uint32_t* srow = (uint32_t*)take((size_t)nslots * 4);
  uint32_t* ent_slot = (uint32_t*)take((size_t)total * 4);
  double* ent_val = (double*)take((size_t)total * 8);
  uint32_t* run_d = (uint32_t*)take((size_t)nb * dim * 4);
  uint32_t* run_beg = (uint32_t*)take((size_t)nb * dim * 4);
  uint32_t* nruns = (uint32_t*)take((size_t)nb * 4);
  PARS_CUDA_CHECK(cudaMemcpyAsync(ent_off, h_ent_off, (size_t)(nb + 1) * 8,
                                  cudaMemcpyHostToDevice, st));
  PARS_CUDA_CHECK(cudaMemcpyAsync(soff, h_soff, (size_t)(nb + 1) * 8, cudaMemcpyHostToDevice, st));
  PARS_CUDA_CHECK(cudaMemcpyAsync(srow, h_srow, (size_t)nslots * 4, cudaMemcpyHostToDevice, st));
  const size_t build_smem = (size_t)dim * 8;  // cursors + slot masks
  PARS_CUDA_CHECK(cudaFuncSetAttribute(slot_build_kernel,
                                       cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       (int)build_smem));
  slot_build_kernel<<<(unsigned)nb, kBuildThreads, build_smem, st>>>(
      rp, idx, val, dim, srow, soff, ent_off, ent_slot, ent_val, run_d, run_beg, nruns);
  const size_t step_smem = baseline_smem_bytes(dim, max_slots);
  PARS_CUDA_CHECK(cudaFuncSetAttribute(baseline_epoch_kernel,
                                       cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       (int)step_smem));
  baseline_epoch_kernel<<<1, kStepThreads, step_smem, st>>>(
      kind, rp, idx, val, dim, srow, soff, nb, k, d_target, lr, bias, (int32_t)max_slots,
      ent_off, ent_slot, ent_val, run_d, run_beg, nruns, d_w, d_bias_out, d_loss_out);
  count_launch(ctx, 2);
  PARS_CUDA_CHECK(cudaGetLastError());
  return PARS_OK;
}

}  // namespace pars_b200
