// Reference-equivalent pairwise SGD epoch on a thread-block cluster.
//
// Same arithmetic, in the same order, as the single-CTA sgd_epoch_kernel
// (sgd.cu) and the reference (train.cpp:34-44, :141-166) — bit-identical
// weights and loss — but the 782 dependent steps are spread over a cluster
// of 8 CTAs (8 SMs) with the step's data staged in shared memory ahead of
// time:
//   * hashed features are kept in a compact form, one u32 per entry
//     (idx << 16 | count + 2^15), since every value is exactly count * inv_row
//     (features.cpp:113-120); v is rebuilt with __dmul_rn(count, inv), the
//     very product the featurizer stored;
//   * every CTA holds the full weight vector in shared memory; a CTA owns 1/8
//     of each batch's prompt slots (score chains, pair losses) and 1/8 of the
//     buckets (gradient folds + updates); updated weights, active flags and
//     slot L2 factors are broadcast to the other CTAs' shared memory through
//     DSMEM, with two cluster barriers per step;
//   * while warps 0-1 run the step's score chains, warps 2-7 stage the NEXT
//     step's rows, CSC entries and runs into the other half of a double
//     buffer with cp.async, so the dependent chains read shared memory only.
// Steps whose data does not fit the buffers read it from global memory.
#include <cooperative_groups.h>
#include <cuda_pipeline.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdio>
#include <vector>

#include "common.cuh"
#include "sgd_cluster.cuh"

namespace cg = cooperative_groups;

namespace pars_b200 {

namespace {

constexpr int kCL = kSgdCluster;  // CTAs per cluster
#ifndef PARS_SGD_THREADS
#define PARS_SGD_THREADS 256
#endif
constexpr int kThreads = PARS_SGD_THREADS;
#ifndef PARS_SGD_CHAIN_WARPS
#define PARS_SGD_CHAIN_WARPS 3
#endif
constexpr int kChainWarps = PARS_SGD_CHAIN_WARPS;  // warps running the step's score chains
constexpr int kChainThreads = kChainWarps * 32;
constexpr int kBuildThreads = 1024;  // one warp per slot of a placement round
constexpr int kBuildWarps = kBuildThreads / 32;
constexpr int kRegEntries = 12;      // row entries per lane kept in registers

// ---- compact rows ----------------------------------------------------------
__global__ void cpk_build_kernel(const int64_t* __restrict__ rp, const uint32_t* __restrict__ idx,
                                 const int32_t* __restrict__ cnt, int64_t n,
                                 const uint32_t* __restrict__ off, uint32_t* __restrict__ cpk,
                                 int32_t* bad) {
  const int64_t r = blockIdx.x;
  if (r >= n) return;
  const int64_t b = rp[r], e = rp[r + 1];
  uint32_t* out = cpk + off[r];
  for (int64_t k = threadIdx.x; k < e - b; k += blockDim.x) {
    const uint32_t i = idx[b + k];
    const int32_t c = cnt[b + k];
    if (i > 0xffffu || c > 32767 || c < -32768) atomicExch(bad, 1);
    out[k] = (i << 16) | ((uint32_t)(c + 0x8000) & 0xffffu);  // count biased by 2^15
  }
}

// ---- per-batch CSC, compact ---------------------------------------------
// One CTA per batch: stable counting sort of the batch's (slot, idx, count)
// entries by idx, slots in order. Entry = slot << 16 | count + 2^15. Runs are
// (idx, first entry); rb[q][r] = first run of rank r's bucket range.
__global__ void __launch_bounds__(kBuildThreads) csc_build_kernel(
    const int64_t* __restrict__ rp, const uint32_t* __restrict__ cpk,
    const uint32_t* __restrict__ cpk_off, uint32_t dim, const uint32_t* __restrict__ pa,
    const uint32_t* __restrict__ pb, int64_t npairs, int32_t B,
    const int64_t* __restrict__ ent_off, uint32_t* __restrict__ ent, uint2* __restrict__ runs,
    uint32_t* __restrict__ nruns, uint32_t* __restrict__ rb, uint4* __restrict__ desc4,
    const uint4* __restrict__ slots) {
  extern __shared__ uint32_t cur[];  // [dim] counts -> cursors, then [dim] slot masks
  uint32_t* mask = cur + dim;
  __shared__ uint32_t part[kBuildThreads], rpart[kBuildThreads];
  const int64_t q = blockIdx.x;
  const int64_t p0 = q * B;
  const int bn = (int)imin64(B, npairs - p0);
  const int S = 2 * bn;
  const int64_t base = ent_off[q];
  for (uint32_t d = threadIdx.x; d < dim; d += kBuildThreads) cur[d] = 0;
  __syncthreads();
  // slot k's row from the epoch's slot table (slot_table_kernel): one warp
  // per slot, coalesced over the row
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  for (int k = w; k < S; k += kBuildWarps) {
    const uint4 m = slots[2 * p0 + k];
    const uint32_t* row = cpk + m.x;
#pragma unroll 4
    for (int e = lane; e < (int)m.y; e += 32) atomicAdd(&cur[row[e] >> 16], 1u);
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
  uint2* rq = runs + q * (int64_t)dim;
  for (uint32_t d = d0; d < d1; ++d) {
    const uint32_t c = cur[d];
    if (c) rq[rrun++] = make_uint2(d, run);
    cur[d] = run;
    run += c;
  }
  if (threadIdx.x == kBuildThreads - 1) nruns[q] = rrun;
  __syncthreads();
  // rank boundaries: first run whose bucket >= r * ceil(dim / kCL)
  if (threadIdx.x <= kCL) {
    const uint32_t bound = (uint32_t)min((uint64_t)dim, (uint64_t)threadIdx.x * ((dim + kCL - 1) / kCL));
    uint32_t lo = 0, hi = nruns[q];
    while (lo < hi) {
      const uint32_t mid = (lo + hi) >> 1;
      if (rq[mid].x >= bound)
        hi = mid;
      else
        lo = mid + 1;
    }
    rb[q * (kCL + 1) + threadIdx.x] = lo;
  }
  __syncthreads();
  if (threadIdx.x < kCL) {  // per rank: runs [r0, r1), batch entries [e0, e1)
    const uint32_t r0 = rb[q * (kCL + 1) + threadIdx.x], r1 = rb[q * (kCL + 1) + threadIdx.x + 1];
    const uint32_t nr = nruns[q], total = (uint32_t)(ent_off[q + 1] - ent_off[q]);
    desc4[q * kCL + threadIdx.x] =
        make_uint4(r0, r1, r0 < nr ? rq[r0].y : total, r1 < nr ? rq[r1].y : total);
  }
  // Stable placement, one warp per slot, kBuildWarps slots per round: a
  // bucket's entries from the round's slots go in slot order, ranked by the
  // bits of the lower warps in the bucket's slot mask (a row holds each bucket
  // at most once); the lowest warp of each bucket then advances its cursor.
  // A lane keeps its first kRegEntries entries of the row in registers across
  // the three passes (longer rows re-read their tail).
  for (uint32_t d = threadIdx.x; d < dim; d += kBuildThreads) mask[d] = 0;
  __syncthreads();
  const uint32_t below = (1u << w) - 1u;
  for (int k0 = 0; k0 < S; k0 += kBuildWarps) {
    const int k = k0 + w;
    const uint32_t* row = nullptr;
    int len = 0;
    if (k < S) {
      const uint4 m = slots[2 * p0 + k];
      row = cpk + m.x;
      len = (int)m.y;
    }
    uint32_t R[kRegEntries];
#pragma unroll
    for (int j = 0; j < kRegEntries; ++j) {
      const int e = lane + 32 * j;
      R[j] = e < len ? row[e] : 0u;
    }
    auto each = [&](auto&& f) {
#pragma unroll
      for (int j = 0; j < kRegEntries; ++j)
        if (lane + 32 * j < len) f(R[j]);
      for (int e = lane + 32 * kRegEntries; e < len; e += 32) f(row[e]);
    };
    each([&](uint32_t E) { atomicOr(&mask[E >> 16], 1u << w); });
    __syncthreads();
    each([&](uint32_t E) {
      const uint32_t d = E >> 16;
      ent[base + cur[d] + __popc(mask[d] & below)] = ((uint32_t)k << 16) | (E & 0xffffu);
    });
    __syncthreads();
    each([&](uint32_t E) {
      // atomic read / reset: the bucket's other warps read the mask while its
      // lowest warp clears it (their outcome is the same either way, but a
      // plain load racing the store is a data race)
      const uint32_t d = E >> 16;
      const uint32_t m = atomicOr(&mask[d], 0u);
      if (m && !(m & below)) {  // the bucket's lowest warp this round
        cur[d] += __popc(m);
        atomicExch(&mask[d], 0u);
      }
    });
    __syncthreads();
  }
  // Runs re-encoded as (bucket | length << 16, first entry) and, within each
  // rank's range, put longest first (counting sort on min(length, 255)): the
  // fold thread t takes runs t, t + 256, ... so the longest runs land on
  // different threads and a thread's second run is a short one. The order of
  // runs is free (each bucket's fold is independent).
  {
    uint2* tmp = reinterpret_cast<uint2*>(cur);  // cur + mask: dim uint2 >= runs
    uint32_t* hist = part;                        // 256 bins
    const uint32_t nr = nruns[q], total = (uint32_t)(ent_off[q + 1] - ent_off[q]);
    for (uint32_t k = threadIdx.x; k < nr; k += kBuildThreads) {
      const uint2 v = rq[k];
      const uint32_t len = (k + 1 < nr ? rq[k + 1].y : total) - v.y;
      tmp[k] = make_uint2(v.x | (len << 16), v.y);
    }
    __syncthreads();
    for (int r = 0; r < kCL; ++r) {
      const uint32_t r0 = rb[q * (kCL + 1) + r], r1 = rb[q * (kCL + 1) + r + 1];
      if (threadIdx.x < 256) hist[threadIdx.x] = 0;
      __syncthreads();
      for (uint32_t k = r0 + threadIdx.x; k < r1; k += kBuildThreads)
        atomicAdd(&hist[255 - min(tmp[k].x >> 16, 255u)], 1u);
      __syncthreads();
      if (threadIdx.x == 0) {
        uint32_t acc = 0;
        for (int b = 0; b < 256; ++b) {
          const uint32_t c = hist[b];
          hist[b] = acc;
          acc += c;
        }
      }
      __syncthreads();
      for (uint32_t k = r0 + threadIdx.x; k < r1; k += kBuildThreads)
        rq[r0 + atomicAdd(&hist[255 - min(tmp[k].x >> 16, 255u)], 1u)] = tmp[k];
      __syncthreads();
    }
  }
}

// Per epoch slot table: for slot g of the epoch (2 per pair, a then b):
// {compact row offset, length, inv (2 words)} — one 16-byte load per slot
// when a step is staged, instead of a chain of dependent lookups.
__global__ void slot_table_kernel(const uint32_t* __restrict__ pa, const uint32_t* __restrict__ pb,
                                  int64_t npairs, const int64_t* __restrict__ rp,
                                  const uint32_t* __restrict__ cpk_off,
                                  const double* __restrict__ inv_row, uint4* __restrict__ table) {
  const int64_t g = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (g >= 2 * npairs) return;
  const uint32_t r = (g & 1) ? pb[g >> 1] : pa[g >> 1];
  const unsigned long long iv = (unsigned long long)__double_as_longlong(inv_row[r]);
  table[g] = make_uint4(cpk_off[r], (uint32_t)(rp[r + 1] - rp[r]), (uint32_t)iv,
                        (uint32_t)(iv >> 32));
}

// Score chain over a staged (shared-memory) row: the raw entries are read two
// groups of 4 ahead and the weights one group ahead of the __dadd_rn chain,
// so the chain does not wait on the load -> dependent gather latency.
// The entry's signed 16-bit count as a double, exactly, without an I2F.F64
// (a slow conversion pipe on this part): the bits of 2^52 + (c + 2^15), less
// 2^52 + 2^15, in one DADD.
__device__ __forceinline__ double cnt_of(uint32_t E) { return biased16_to_f64(E); }

__device__ __forceinline__ double chain_row_s(const uint32_t* __restrict__ rs, uint32_t len, double inv,
                                              const double* __restrict__ W) {
  double acc = 0.0;
  const uint32_t ng = len >> 2;
  if (ng >= 2) {
    // pipeline: raw entries of group g+2, weights of group g+1, products of
    // group g, adds of group g
    const uint4* r4 = reinterpret_cast<const uint4*>(rs);
    uint4 A = r4[0], B = r4[1];
    double p0 = __dmul_rn(W[A.x >> 16], __dmul_rn(cnt_of(A.x), inv));
    double p1 = __dmul_rn(W[A.y >> 16], __dmul_rn(cnt_of(A.y), inv));
    double p2 = __dmul_rn(W[A.z >> 16], __dmul_rn(cnt_of(A.z), inv));
    double p3 = __dmul_rn(W[A.w >> 16], __dmul_rn(cnt_of(A.w), inv));
    double w0 = W[B.x >> 16], w1 = W[B.y >> 16], w2 = W[B.z >> 16], w3 = W[B.w >> 16];
    for (uint32_t g = 0; g < ng; ++g) {
      const uint4 Cn = g + 2 < ng ? r4[g + 2] : B;
      const double q0 = __dmul_rn(w0, __dmul_rn(cnt_of(B.x), inv));
      const double q1 = __dmul_rn(w1, __dmul_rn(cnt_of(B.y), inv));
      const double q2 = __dmul_rn(w2, __dmul_rn(cnt_of(B.z), inv));
      const double q3 = __dmul_rn(w3, __dmul_rn(cnt_of(B.w), inv));
      w0 = W[Cn.x >> 16], w1 = W[Cn.y >> 16], w2 = W[Cn.z >> 16], w3 = W[Cn.w >> 16];
      acc = __dadd_rn(__dadd_rn(__dadd_rn(__dadd_rn(acc, p0), p1), p2), p3);
      p0 = q0, p1 = q1, p2 = q2, p3 = q3;
      B = Cn;
    }
  }
  for (uint32_t e = ng >= 2 ? ng << 2 : 0; e < len; ++e) {
    const uint32_t E = rs[e];
    acc = __dadd_rn(acc, __dmul_rn(W[E >> 16], __dmul_rn(cnt_of(E), inv)));
  }
  return acc;
}

// Gradient fold of one bucket's run over staged (shared-memory) CSC entries,
// same prefetch scheme: raw entries two groups of 4 ahead, the slots' signed
// L2 factors one group ahead of the add chain.
__device__ __forceinline__ double chain_run_s(const uint32_t* __restrict__ cs, uint32_t b, uint32_t e1,
                                              const double* __restrict__ sinv) {
  double g = 0.0;
  uint32_t e = b;
  const uint32_t ng = (e1 - b) >> 2;
  if (ng >= 2) {
    uint32_t a0 = cs[e], a1 = cs[e + 1], a2 = cs[e + 2], a3 = cs[e + 3];
    uint32_t b0 = cs[e + 4], b1 = cs[e + 5], b2 = cs[e + 6], b3 = cs[e + 7];
    double s0 = sinv[a0 >> 16], s1 = sinv[a1 >> 16], s2 = sinv[a2 >> 16], s3 = sinv[a3 >> 16];
    for (uint32_t k = 0; k < ng; ++k) {
      const uint32_t o = e + 8;
      const bool more = k + 2 < ng;
      const uint32_t c0 = more ? cs[o] : b0, c1 = more ? cs[o + 1] : b1;
      const uint32_t c2 = more ? cs[o + 2] : b2, c3 = more ? cs[o + 3] : b3;
      const double t0 = sinv[b0 >> 16], t1 = sinv[b1 >> 16], t2 = sinv[b2 >> 16], t3 = sinv[b3 >> 16];
      g = __dadd_rn(g, __dmul_rn(cnt_of(a0), s0));
      g = __dadd_rn(g, __dmul_rn(cnt_of(a1), s1));
      g = __dadd_rn(g, __dmul_rn(cnt_of(a2), s2));
      g = __dadd_rn(g, __dmul_rn(cnt_of(a3), s3));
      a0 = b0, a1 = b1, a2 = b2, a3 = b3;
      b0 = c0, b1 = c1, b2 = c2, b3 = c3;
      s0 = t0, s1 = t1, s2 = t2, s3 = t3;
      e += 4;
    }
  }
  for (; e < e1; ++e) {
    const uint32_t E = cs[e];
    g = __dadd_rn(g, __dmul_rn(cnt_of(E), sinv[E >> 16]));
  }
  return g;
}

// ---- the cluster epoch kernel ------------------------------------------------
struct Layout {
  uint32_t dim, B, spc, ppc;  // slots / pairs per CTA
  uint32_t rowcap, csccap, runcap;
  size_t w, rowbuf, slotptr, slotsrc, slotlen, slotinv, pairy, cscbuf, runbuf, desc, sinv,
      loss_all, score, mbar, total;
};

struct StepDesc {
  const uint32_t* csc;  // entries of this CTA's runs (smem or global)
  const uint2* runs;
  uint32_t nruns;
  uint32_t ent_base;  // batch-relative index of csc[0]
  uint32_t ent_end;   // batch-relative end of this CTA's entries
  uint32_t pad;
  uint32_t cshift;    // staged CSC: entry ent_base sits at cscbuf[cshift] (16-byte copies)
  uint32_t rshift;    // staged runs: run pad sits at runbuf[rshift] (16-byte aligned copy)
};

// TMA bulk copy global -> this CTA's shared memory, completing on an mbarrier
__device__ __forceinline__ void bulk_g2s(uint32_t dst, const void* src, uint32_t bytes, uint32_t bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(dst),
      "l"(src), "r"(bytes), "r"(bar)
      : "memory");
}
__device__ __forceinline__ void bar_expect(uint32_t bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(bytes) : "memory");
}
__device__ __forceinline__ void bar_wait(uint32_t bar, uint32_t parity) {
  asm volatile(
      "{\n\t.reg .pred p;\n\tSTAGE_WAIT_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t@!p bra STAGE_WAIT_%=;\n\t}" ::"r"(bar),
      "r"(parity)
      : "memory");
}

__host__ __device__ inline size_t al16(size_t x) { return (x + 15) & ~(size_t)15; }

__host__ __device__ inline Layout make_layout(uint32_t dim, uint32_t B, uint32_t rowcap,
                                              uint32_t csccap, uint32_t runcap) {
  Layout L;
  L.dim = dim;
  L.B = B;
  L.spc = (2 * B + kCL - 1) / kCL;
  L.spc += L.spc & 1;  // whole pairs per CTA
  L.ppc = L.spc / 2;
  L.rowcap = rowcap;
  L.csccap = csccap;
  L.runcap = runcap;
  size_t o = 0;
  L.w = o;
  o = al16(o + (size_t)dim * 8);
  L.rowbuf = o;
  o = al16(o + 2ull * rowcap * 4);
  L.slotptr = o;
  o = al16(o + 2ull * L.spc * 8);
  L.slotsrc = o;
  o = al16(o + 2ull * L.spc * 8);
  L.slotlen = o;
  o = al16(o + 2ull * L.spc * 4);
  L.slotinv = o;
  o = al16(o + 2ull * L.spc * 8);
  L.pairy = o;
  o = al16(o + 2ull * L.ppc * 4);
  L.cscbuf = o;
  o = al16(o + 2ull * csccap * 4);
  L.runbuf = o;
  o = al16(o + 2ull * runcap * 8);
  L.desc = o;
  o = al16(o + 2ull * sizeof(StepDesc));
  L.sinv = o;
  o = al16(o + 2ull * B * 8);
  L.loss_all = o;
  o = al16(o + (size_t)B * 8);
  L.score = o;
  o = al16(o + (size_t)L.spc * 8);
  L.mbar = o;
  o = al16(o + 2 * 8);
  L.total = o;
  return L;
}

struct EpochArgs {
  const int64_t* rp;
  const uint32_t* cpk;
  const uint32_t* cpk_off;
  const double* inv_row;
  const uint32_t* pa;
  const uint32_t* pb;
  const int32_t* py;
  int64_t npairs;
  double lr, margin, bias;
  const int64_t* ent_off;
  const uint32_t* ent;
  const uint2* runs;
  const uint32_t* nruns;
  const uint32_t* rb;
  const uint4* slots;  // slot table (slot_table_kernel)
  const uint4* desc4;  // per (batch, rank): r0, r1, e0, e1
  double* w_io;
  double* loss_out;
  unsigned long long* active_out;
  long long* timing;  // PARS_SGD_TIMING builds only: [5 phases][8 ranks] max over threads
};

// Stage step q's data for CTA `rank` into buffer `buf`; run by the staging
// warps (t = thread index within them, nt = their thread count) while the
// chain warps score step q-1. The rows, the CTA's CSC entries and its runs
// are TMA bulk copies (one per slot row, one for the CSC range, one for the
// runs) completing on the buffer's mbarrier, whose two arrivals (staging
// warp 0's lane 0 and thread 32, each with the bytes its copies carry) are
// made here; stage_wait() waits for the phase.
__device__ void stage_step(const Layout& L, const EpochArgs& a, unsigned char* sm, int64_t q,
                           int buf, int rank, int t, int nt) {
  const int64_t p0 = q * L.B;
  const int bn = (int)imin64(L.B, a.npairs - p0);
  uint32_t* rowbuf = reinterpret_cast<uint32_t*>(sm + L.rowbuf) + (size_t)buf * L.rowcap;
  const uint32_t** slotptr = reinterpret_cast<const uint32_t**>(sm + L.slotptr) + (size_t)buf * L.spc;
  const uint32_t** slotsrc = reinterpret_cast<const uint32_t**>(sm + L.slotsrc) + (size_t)buf * L.spc;
  uint32_t* slotlen = reinterpret_cast<uint32_t*>(sm + L.slotlen) + (size_t)buf * L.spc;
  double* slotinv = reinterpret_cast<double*>(sm + L.slotinv) + (size_t)buf * L.spc;
  int32_t* pairy = reinterpret_cast<int32_t*>(sm + L.pairy) + (size_t)buf * L.ppc;
  uint32_t* cscbuf = reinterpret_cast<uint32_t*>(sm + L.cscbuf) + (size_t)buf * L.csccap;
  uint2* runbuf = reinterpret_cast<uint2*>(sm + L.runbuf) + (size_t)buf * L.runcap;
  StepDesc* desc = reinterpret_cast<StepDesc*>(sm + L.desc) + buf;
  const uint32_t bar = (uint32_t)__cvta_generic_to_shared(sm + L.mbar) + 8u * (uint32_t)buf;
  const int w = t >> 5, lane = t & 31;
  // the buffer's previous contents were read through the generic proxy
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  if (w == 0) {
    // slot metadata, 32 slots at a time; buffer offsets by a warp scan
    uint32_t off = 0, bytes = 0;
    for (uint32_t k0 = 0; k0 < L.spc; k0 += 32) {
      const uint32_t k = k0 + lane;
      const int s = rank * (int)L.spc + (int)k;
      const bool ok = k < L.spc && s < 2 * bn;
      uint4 st = make_uint4(0u, 0u, 0u, 0u);
      if (ok) {
        st = a.slots[2 * p0 + s];
        slotinv[k] = __longlong_as_double((long long)(((unsigned long long)st.w << 32) | st.z));
        if ((s & 1) == 0) pairy[k >> 1] = a.py[p0 + (s >> 1)];
      }
      const uint32_t len = st.y, padded = (len + 3) & ~3u;
      uint32_t x = padded;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const uint32_t y = __shfl_up_sync(0xffffffffu, x, o);
        if (lane >= o) x += y;
      }
      const uint32_t my_off = off + x - padded;
      if (k < L.spc) {
        const uint32_t* src = ok ? a.cpk + st.x : nullptr;
        const bool staged = ok && my_off + padded <= L.rowcap;
        slotlen[k] = len;
        slotsrc[k] = src;
        slotptr[k] = !ok ? nullptr : (staged ? rowbuf + my_off : src);
        if (staged && padded) {
          bulk_g2s((uint32_t)__cvta_generic_to_shared(rowbuf + my_off), src, padded * 4, bar);
          bytes += padded * 4;
        }
      }
      off += __shfl_sync(0xffffffffu, x, 31);
    }
    bytes = __reduce_add_sync(0xffffffffu, bytes);
    if (lane == 0) bar_expect(bar, bytes);
  } else if (t == 32) {
    // this CTA's runs [r0, r1) and batch entries [e0, e1)
    const uint4 q4 = a.desc4[q * kCL + rank];
    StepDesc d;
    d.nruns = q4.y - q4.x;
    d.ent_base = q4.z;
    d.ent_end = q4.w;
    const uint2* rq = a.runs + q * (int64_t)L.dim;
    // runs from the 16-byte aligned entry at or before the first (the runs
    // array has slack after it): run q4.x lands at runbuf[rshift]
    d.rshift = (uint32_t)((reinterpret_cast<uintptr_t>(rq + q4.x) >> 3) & 1u);
    const uint32_t rbytes = ((d.nruns + d.rshift) * 8 + 15) & ~15u;
    const bool runs_staged = d.nruns > 0 && rbytes <= L.runcap * 8;
    d.runs = runs_staged ? runbuf + d.rshift : rq + q4.x;
    const uint32_t* g0 = a.ent + a.ent_off[q] + d.ent_base;
    d.cshift = (uint32_t)((reinterpret_cast<uintptr_t>(g0) >> 2) & 3u);
    const uint32_t cbytes = ((d.ent_end - d.ent_base + d.cshift) * 4 + 15) & ~15u;
    const bool csc_staged = d.ent_end > d.ent_base && d.ent_end - d.ent_base + d.cshift + 3 <= L.csccap;
    d.csc = csc_staged ? cscbuf : g0;
    d.pad = q4.x;
    *desc = d;
    uint32_t bytes = 0;
    if (runs_staged) {
      bulk_g2s((uint32_t)__cvta_generic_to_shared(runbuf), rq + q4.x - d.rshift, rbytes, bar);
      bytes += rbytes;
    }
    if (csc_staged) {
      bulk_g2s((uint32_t)__cvta_generic_to_shared(cscbuf), g0 - d.cshift, cbytes, bar);
      bytes += cbytes;
    }
    bar_expect(bar, bytes);
  }
  (void)nt;
}

// Wait until buffer buf's bulk copies have landed (its u-th use, parity u & 1).
__device__ __forceinline__ void stage_wait(const Layout& L, unsigned char* sm, int buf, int64_t use) {
  bar_wait((uint32_t)__cvta_generic_to_shared(sm + L.mbar) + 8u * (uint32_t)buf, (uint32_t)(use & 1));
}

__global__ void __launch_bounds__(kThreads, 1) sgd_cluster_kernel(const Layout L, const EpochArgs a) {
  extern __shared__ __align__(16) unsigned char sm[];
  // the same bytes as 32-bit words: indexing it makes the staged rows / CSC
  // entries explicit shared-memory loads (the staged-or-global pointers are
  // generic, and generic loads of shared memory are slower)
  extern __shared__ __align__(16) uint32_t smw[];
  cg::cluster_group cluster = cg::this_cluster();
  const int rank = (int)cluster.block_rank();
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  double* W = reinterpret_cast<double*>(sm + L.w);
  // per slot of the batch: +-inv when its pair is active (sign of the
  // gradient term: -y for prompt a, +y for prompt b), 0.0 when inactive
  double* sinv = reinterpret_cast<double*>(sm + L.sinv);
  double* loss_all = reinterpret_cast<double*>(sm + L.loss_all);
  double* score = reinterpret_cast<double*>(sm + L.score);
  for (uint32_t d = tid; d < L.dim; d += kThreads) W[d] = a.w_io[d];
  const int64_t nb = (a.npairs + L.B - 1) / L.B;
  // stage step 0 with every warp but 0, wait, start
  if (tid < 2)
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 2;" ::"r"((uint32_t)__cvta_generic_to_shared(sm + L.mbar) +
                                                                  8u * tid));
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  __syncthreads();
  if (warp >= kChainWarps) stage_step(L, a, sm, 0, 0, rank, tid - kChainThreads, kThreads - kChainThreads);
  if (tid == 0) stage_wait(L, sm, 0, 0);
  __syncthreads();
  cluster.sync();
  double epoch_loss = 0.0;
  unsigned long long active = 0;
#ifdef PARS_SGD_TIMING
  long long tt[6] = {0, 0, 0, 0, 0, 0};  // [0] the chain warps, [5] the staging warps
#endif
  for (int64_t q = 0; q < nb; ++q) {
#ifdef PARS_SGD_TIMING
    long long c0 = clock64();
#endif
    const int buf = (int)(q & 1);
    const int64_t p0 = q * L.B;
    const int bn = (int)imin64(L.B, a.npairs - p0);
    const uint32_t** slotptr = reinterpret_cast<const uint32_t**>(sm + L.slotptr) + (size_t)buf * L.spc;
    const uint32_t* slotlen = reinterpret_cast<const uint32_t*>(sm + L.slotlen) + (size_t)buf * L.spc;
    const double* slotinv = reinterpret_cast<const double*>(sm + L.slotinv) + (size_t)buf * L.spc;
    const int32_t* pairy = reinterpret_cast<const int32_t*>(sm + L.pairy) + (size_t)buf * L.ppc;
    const StepDesc d = reinterpret_cast<const StepDesc*>(sm + L.desc)[buf];
    if (warp < kChainWarps) {
      // phase A: score chains of this CTA's slots (scorer.cpp:40-42), spread
      // over kChainWarps warps (few lanes each: fewer bank conflicts on the
      // weight gathers, one chain warp per scheduler), then the margin loss
      // of its pairs (pairs.hpp:27-31)
      const uint32_t per = (L.spc + kChainWarps - 1) / kChainWarps;
      for (uint32_t j = lane; j < per; j += 32) {
        const uint32_t k = warp * per + j;
        if (k >= L.spc) break;
        const int s = rank * (int)L.spc + (int)k;
        if (s >= 2 * bn) continue;
        const uint32_t* row = slotptr[k];
        const uint32_t len = slotlen[k];
        const double inv = slotinv[k];
        const uint32_t* rbuf = reinterpret_cast<const uint32_t*>(sm + L.rowbuf) + (size_t)buf * L.rowcap;
        double acc = 0.0;
        uint32_t e = 0;
        if (row >= rbuf && row < rbuf + L.rowcap) {  // staged: shared-memory loads
          const uint32_t* rs = smw + (L.rowbuf >> 2) + (size_t)buf * L.rowcap + (uint32_t)(row - rbuf);
          acc = chain_row_s(rs, len, inv, W);
        } else {
#pragma unroll 8
          for (; e < len; ++e) {
            const uint32_t E = row[e];
            acc = __dadd_rn(acc, __dmul_rn(W[E >> 16], __dmul_rn(cnt_of(E), inv)));
          }
        }
        score[k] = __dadd_rn(acc, a.bias);
      }
      asm volatile("bar.sync 2, %0;" ::"r"(kChainThreads));  // chain warps only
      for (uint32_t k = tid; k < L.ppc; k += kChainThreads) {
        const int p = rank * (int)L.ppc + (int)k;
        if (p >= bn) continue;
        const int32_t y = pairy[k];
        const double v =
            __dadd_rn(__dmul_rn(-(double)y, __dsub_rn(score[2 * k], score[2 * k + 1])), a.margin);
        const double l = v > 0.0 ? v : 0.0;
        // grad[idx] -= y*v for a, += y*v for b (train.cpp:38-42); the sign
        // flips and the zero for inactive pairs are exact, so each entry's
        // term is one __dmul_rn(count, sinv[slot])
        const double ia = slotinv[2 * k], ib = slotinv[2 * k + 1];
        const double sa = l > 0.0 ? (y > 0 ? -ia : ia) : 0.0;
        const double sb = l > 0.0 ? (y > 0 ? ib : -ib) : 0.0;
        for (int rr = 0; rr < kCL; ++rr) {
          double* ri = cluster.map_shared_rank(sinv, rr);
          ri[2 * p] = sa;
          ri[2 * p + 1] = sb;
        }
        cluster.map_shared_rank(loss_all, 0)[p] = l;
      }
    } else if (q + 1 < nb) {
      // stage the next step while the chain warps score this one
      stage_step(L, a, sm, q + 1, buf ^ 1, rank, tid - kChainThreads, kThreads - kChainThreads);
    }
#ifdef PARS_SGD_TIMING
    long long c1 = clock64();
#endif
    cluster.sync();
#ifdef PARS_SGD_TIMING
    long long c2 = clock64();
#endif
    // phase C: gradient folds of this CTA's buckets, in (pair, a-before-b)
    // order, and the update w[d] -= (lr/bn) * g[d] (train.cpp:141-151)
    const double scale = __ddiv_rn(a.lr, (double)bn);
    const uint32_t* cbuf = reinterpret_cast<const uint32_t*>(sm + L.cscbuf) + (size_t)buf * L.csccap;
    const bool csc_staged = d.csc == cbuf;
    const bool runs_staged =
        d.runs == reinterpret_cast<const uint2*>(sm + L.runbuf) + (size_t)buf * L.runcap + d.rshift;
    const uint2* runs_s = reinterpret_cast<const uint2*>(smw + (L.runbuf >> 2)) + (size_t)buf * L.runcap + d.rshift;
    for (uint32_t r = tid; r < d.nruns; r += kThreads) {
      const uint2 run = runs_staged ? runs_s[r] : d.runs[r];
      const uint32_t bucket = run.x & 0xffffu, e1 = run.y + (run.x >> 16);  // (bucket | len << 16, first)
      // g starts at +0.0 and is never -0.0 under round-to-nearest, so the
      // +-0.0 terms of inactive pairs leave it unchanged: branch-free fold
      double g = 0.0;
      uint32_t e = run.y;
      if (csc_staged) {  // shared-memory loads
        const uint32_t* cs = smw + (L.cscbuf >> 2) + (size_t)buf * L.csccap + d.cshift - d.ent_base;
        g = chain_run_s(cs, e, e1, sinv);
      } else {
        const uint32_t* csc = d.csc - d.ent_base;
#pragma unroll 8
        for (; e < e1; ++e) {
          const uint32_t E = csc[e];
          g = __dadd_rn(g, __dmul_rn(cnt_of(E), sinv[E >> 16]));
        }
      }
      if (g != 0.0) {
        const double nw = __dsub_rn(W[bucket], __dmul_rn(scale, g));
        for (int rr = 0; rr < kCL; ++rr) cluster.map_shared_rank(W, rr)[bucket] = nw;
      }
    }
    if (rank == 0 && tid == kThreads - 1) {
      for (int p = 0; p < bn; ++p) {
        epoch_loss = __dadd_rn(epoch_loss, loss_all[p]);
        active += loss_all[p] > 0.0;
      }
    }
#ifdef PARS_SGD_TIMING
    long long c3 = clock64();
#endif
    if (tid == 0 && q + 1 < nb) stage_wait(L, sm, buf ^ 1, (q + 1) >> 1);  // next step's staged data
#ifdef PARS_SGD_TIMING
    long long c4 = clock64();
#endif
    __syncthreads();
    cluster.sync();
#ifdef PARS_SGD_TIMING
    long long c5 = clock64();
    tt[warp < kChainWarps ? 0 : 5] += c1 - c0; tt[1] += c2 - c1; tt[2] += c3 - c2; tt[3] += c4 - c3; tt[4] += c5 - c4;
#endif
  }
#ifdef PARS_SGD_TIMING
  if (a.timing) {
    for (int k = 0; k < 6; ++k) atomicMax(&a.timing[k * 8 + rank], tt[k]);
  }
#endif
  if (rank == 0) {
    for (uint32_t dd = tid; dd < L.dim; dd += kThreads) a.w_io[dd] = W[dd];
    if (tid == kThreads - 1) {
      *a.loss_out = epoch_loss;
      *a.active_out = active;
    }
  }
}

}  // namespace

size_t sgd_cluster_smem(uint32_t dim, int32_t B) {
  return make_layout(dim, (uint32_t)B, kSgdRowCap, kSgdCscCap, kSgdRunCap).total;
}

int build_compact_rows(pars_ctx* ctx, const int64_t* d_rp, const uint32_t* d_idx,
                       const int32_t* d_cnt, int64_t rows, const uint32_t* d_off, uint32_t* d_cpk,
                       int32_t* d_bad, cudaStream_t st) {
  if (rows <= 0) return PARS_OK;
  cpk_build_kernel<<<(unsigned)rows, 128, 0, st>>>(d_rp, d_idx, d_cnt, rows, d_off, d_cpk, d_bad);
  count_launch(ctx);
  PARS_CUDA_CHECK(cudaGetLastError());
  return PARS_OK;
}

size_t sgd_cluster_scratch_bytes(int64_t nbatches, uint32_t dim, int64_t total_entries,
                                 int64_t npairs) {
  return (size_t)(nbatches + 1) * 8 + 256 + (size_t)total_entries * 4 + 256 +
         (size_t)nbatches * dim * 8 + 256 + (size_t)nbatches * 4 + 256 +
         (size_t)nbatches * (kCL + 1) * 4 + 256 + (size_t)nbatches * kCL * 16 + 256 +
         (size_t)npairs * 2 * 16 + 256;
}

int launch_sgd_cluster(pars_ctx* ctx, const int64_t* rp, const uint32_t* cpk,
                       const uint32_t* cpk_off, const double* inv_row, uint32_t dim,
                       const uint32_t* a, const uint32_t* b, const int32_t* y, int64_t npairs,
                       int32_t B, double lr, double margin, double bias, double* w,
                       double* loss_out, unsigned long long* active_out, int64_t total,
                       void* scratch, cudaStream_t st) {
  const int64_t nb = (npairs + B - 1) / B;
  char* p = static_cast<char*>(scratch);
  auto take = [&](size_t bytes) {
    char* r = p;
    p += (bytes + 255) & ~(size_t)255;
    return r;
  };
  int64_t* ent_off = (int64_t*)take((size_t)(nb + 1) * 8);  // uploaded by the caller
  uint32_t* ent = (uint32_t*)take((size_t)total * 4);
  uint2* runs = (uint2*)take((size_t)nb * dim * 8);
  uint32_t* nruns = (uint32_t*)take((size_t)nb * 4);
  uint32_t* rb = (uint32_t*)take((size_t)nb * (kCL + 1) * 4);
  uint4* desc4 = (uint4*)take((size_t)nb * kCL * 16);
  uint4* slots = (uint4*)take((size_t)npairs * 2 * 16);
  const size_t build_smem = (size_t)dim * 8;  // cursors + slot masks
  PARS_CUDA_CHECK(cudaFuncSetAttribute(csc_build_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       (int)build_smem));
  slot_table_kernel<<<(unsigned)ceil_div(2 * npairs, 256), 256, 0, st>>>(a, b, npairs, rp, cpk_off,
                                                                         inv_row, slots);
  csc_build_kernel<<<(unsigned)nb, kBuildThreads, build_smem, st>>>(
      rp, cpk, cpk_off, dim, a, b, npairs, B, ent_off, ent, runs, nruns, rb, desc4, slots);
  const Layout L = make_layout(dim, (uint32_t)B, kSgdRowCap, kSgdCscCap, kSgdRunCap);
  PARS_CUDA_CHECK(cudaFuncSetAttribute(sgd_cluster_kernel,
                                       cudaFuncAttributeMaxDynamicSharedMemorySize, (int)L.total));
  PARS_CUDA_CHECK(cudaFuncSetAttribute(sgd_cluster_kernel,
                                       cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
  EpochArgs ea;
  ea.rp = rp;
  ea.cpk = cpk;
  ea.cpk_off = cpk_off;
  ea.inv_row = inv_row;
  ea.pa = a;
  ea.pb = b;
  ea.py = y;
  ea.npairs = npairs;
  ea.lr = lr;
  ea.margin = margin;
  ea.bias = bias;
  ea.ent_off = ent_off;
  ea.ent = ent;
  ea.runs = runs;
  ea.nruns = nruns;
  ea.rb = rb;
  ea.slots = slots;
  ea.desc4 = desc4;
  ea.w_io = w;
  ea.loss_out = loss_out;
  ea.active_out = active_out;
  ea.timing = nullptr;
#ifdef PARS_SGD_TIMING
  static long long* dbg = nullptr;
  if (!dbg) cudaMalloc(&dbg, 64 * 8);
  cudaMemsetAsync(dbg, 0, 64 * 8, st);
  ea.timing = dbg;
#endif
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(kCL, 1, 1);
  cfg.blockDim = dim3(kThreads, 1, 1);
  cfg.dynamicSmemBytes = L.total;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = kCL;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  if (kCL > 8) {
    static const bool np = cudaFuncSetAttribute(sgd_cluster_kernel, cudaFuncAttributeNonPortableClusterSizeAllowed,
                                                1) == cudaSuccess;
    (void)np;
  }
  PARS_CUDA_CHECK(cudaLaunchKernelEx(&cfg, sgd_cluster_kernel, L, ea));
#ifdef PARS_SGD_TIMING
  {
    long long h[64];
    cudaStreamSynchronize(st);
    cudaMemcpy(h, dbg, sizeof h, cudaMemcpyDeviceToHost);
    const char* names[6] = {"chains(w0)", "sync1", "phaseC", "cp.wait", "sync2", "stage(w1-7)"};
    for (int k = 0; k < 6; ++k) {
      fprintf(stderr, "%-14s", names[k]);
      for (int r = 0; r < kCL; ++r) fprintf(stderr, " %8.0f", (double)h[k * 8 + r] / (double)nb);
      fprintf(stderr, "\n");
    }
  }
#endif
  count_launch(ctx, 3);
  PARS_CUDA_CHECK(cudaGetLastError());
  return PARS_OK;
}

}  // namespace pars_b200
