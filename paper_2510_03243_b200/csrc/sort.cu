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
//   radix_scatter   stable rank within the CTA via warp ballots +
//                   per-warp digit counters; the tile is laid out in digit
//                   order in shared memory and written run by run (coalesced).
//
// Speculative high-word sort (when at least two of the low eight positions
// are active): the passes over the key's top 32 bits run first (positions
// 8..11, stable), then radix_fixup orders each run of equal top words by the
// full key with one thread per element (rank = number of smaller keys in the
// run). A run longer than kFixRun sets `redo`, and the full LSD sort — the
// same passes as without speculation, launched behind a device-side gate —
// runs instead. For scores spread over many binades the runs are a few keys
// long and 4 passes replace 8 (12 with tie ranks).
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdlib>
#include <vector>

#include "common.cuh"
#include "pairs.cuh"

namespace pars_b200 {

namespace {

constexpr int kThreads = 256;
constexpr int kItems = 8;
constexpr int kTileKeys = kThreads * kItems;  // 2048
constexpr unsigned kFull = 0xffffffffu;

// Programmatic dependent launch: the sort's kernels after radix_init are
// launched with programmatic stream serialisation, so each is dispatched
// while its predecessor drains; it waits here (predecessor complete, its
// writes visible) before touching any data, and releases its own successor
// at once.
__device__ __forceinline__ void pdl_enter() {
  asm volatile("griddepcontrol.wait;" ::: "memory");
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
}

__device__ __forceinline__ uint64_t ordered_bits(double x) {
  uint64_t b = (uint64_t)__double_as_longlong(x);
  if ((b << 1) == 0) b = 0;  // -0.0 == +0.0
  return (b >> 63) ? ~b : (b | 0x8000000000000000ull);
}

__device__ __forceinline__ uint32_t digit_of(uint64_t hi, uint32_t lo, int pos) {
  return pos < 4 ? (lo >> (8 * pos)) & 0xffu : (uint32_t)(hi >> (8 * (pos - 4))) & 0xffu;
}

// All 12 digit histograms in one pass over the inputs (keys formed on the
// fly), plus whether the tie ranks are already non-decreasing in input
// order (then the stable sort by score alone is the (score, tie, index)
// order and the tie digits are skipped).
__global__ void radix_init(const double* __restrict__ score, const uint8_t* __restrict__ boosted,
                           const uint32_t* __restrict__ tie, int64_t n, uint32_t* __restrict__ dh) {
  __shared__ uint32_t h[12 * 256];
  for (int k = threadIdx.x; k < 12 * 256; k += blockDim.x) h[k] = 0;
  __syncthreads();
  bool unsorted = false;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    const bool bst = boosted && boosted[i];
    const uint64_t hi = bst ? 0ull : ordered_bits(score[i]);
    const uint32_t lo = tie ? tie[i] : 0u;  // no tie ranks: order by score, then index
    if (tie && i > 0 && lo < tie[i - 1]) unsorted = true;
#pragma unroll
    for (int p = 0; p < 12; ++p) {
      if (p < 4 && !tie) continue;  // all-zero tie digits: counted once below
      const uint32_t d = digit_of(hi, lo, p);
      // the high byte positions of each word are shared by most keys (the
      // exponent, the high bytes of the ranks): aggregate them per warp so
      // the shared-memory atomics do not serialise
      if (p == 1 || p == 2 || p == 3 || p == 9 || p == 10 || p == 11) {
        const unsigned peers = __match_any_sync(__activemask(), d);  // (8 ballots measured slower here)
        if ((peers & ((1u << (threadIdx.x & 31)) - 1u)) == 0) atomicAdd(&h[p * 256 + d], __popc(peers));
      } else {
        atomicAdd(&h[p * 256 + d], 1u);
      }
    }
  }
  if (__any_sync(kFull, unsorted) && (threadIdx.x & 31) == 0) dh[12 * 256] = 1u;
  if (!tie && blockIdx.x == 0 && threadIdx.x < 4) h[threadIdx.x * 256] = (uint32_t)n;
  __syncthreads();
  for (int k = threadIdx.x; k < 12 * 256; k += blockDim.x)
    if (h[k]) atomicAdd(&dh[k], h[k]);
}

// The per-position pass plan, decided on the device (no host round trip, so
// the whole sort is stream-ordered and capturable): a position runs when its
// digits are not all equal (and, for tie digits, when the tie ranks are not
// already in input order). For every position: active, which ping-pong
// buffer it reads (or the raw inputs for the first active pass), whether it
// carries the tie ranks (only while tie passes remain), whether it is the
// last (writes the order), and the exclusive digit bases.
struct PassPlan {
  int active, first, last, src, carry_lo, none;
};
// spec: the speculative high-word passes ran (fixup has work); src: the
// ping-pong buffer holding their output; use_lo: the tie ranks order keys;
// redo: run the full LSD passes (no speculation, or a run over kFixRun)
struct FixPlan {
  int spec, src, use_lo, redo;
};
constexpr int kFixRun = 32;
// Speculation from this many keys (PARS_SORT_SPEC_MIN overrides at run
// time). Measured (tools/sort_ab.py, burst tie ranks, stream timing): with /
// without speculation 0.077 / 0.117 ms at 8,192 keys, 0.086 / 0.133 at 131 k,
// 0.122 / 0.169 at 1 M — it pays at every size the radix path serves.
#ifndef PARS_SORT_SPEC_MIN
#define PARS_SORT_SPEC_MIN 0
#endif
constexpr int64_t kSpecMin = PARS_SORT_SPEC_MIN;

__global__ void __launch_bounds__(256) radix_plan(const uint32_t* __restrict__ dh, int64_t n,
                                                  PassPlan* __restrict__ plan, PassPlan* __restrict__ plan_hi,
                                                  FixPlan* __restrict__ fix, uint32_t* __restrict__ dbase) {
  __shared__ int trivial[12];
  __shared__ int act[12];
  __shared__ int plow;
  __shared__ unsigned long long sqw[8];
  pdl_enter();
  const int t = threadIdx.x, lane = t & 31, warp = t >> 5;
  const bool tie_sorted = dh[12 * 256] == 0u;
  if (t < 12) trivial[t] = 0;
  __syncthreads();
  for (int k = t; k < 12 * 256; k += blockDim.x)  // a digit holding every key
    if (dh[k] == (uint32_t)n) trivial[k >> 8] = 1;
  __syncthreads();
  if (t < 12) act[t] = !trivial[t] && !(t < 4 && tie_sorted);
  __syncthreads();
  if (t == 0) {
    plow = -1;
    for (int p = 7; p >= 4; --p)
      if (act[p]) plow = p;
  }
  __syncthreads();
  // duplication probe for the speculation below: the sum of squared digit
  // counts at the lowest active score byte (n distinct, evenly spread low
  // bytes give a variance-to-mean ratio near 1; keys repeated r times, ~r)
  {
    const unsigned long long c = plow >= 0 ? dh[plow * 256 + t] : 0u;
    unsigned long long v = c * c;
#pragma unroll
    for (int o = 16; o; o >>= 1) v += __shfl_down_sync(kFull, v, o);
    if (lane == 0) sqw[warp] = v;
  }
  // exclusive bases of every position, warp w scanning positions w, w+8
  for (int p = warp; p < 12; p += 8) {
    uint32_t base = 0;
    for (int d0 = 0; d0 < 256; d0 += 32) {
      const uint32_t v = dh[p * 256 + d0 + lane];
      uint32_t x = v;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const uint32_t y = __shfl_up_sync(kFull, x, o);
        if (lane >= o) x += y;
      }
      dbase[p * 256 + d0 + lane] = base + x - v;
      base += __shfl_sync(kFull, x, 31);
    }
  }
  __syncthreads();
  if (t == 0) {
    int last = -1, last_tie = -1, cnt = 0;
    for (int p = 0; p < 12; ++p)
      if (act[p]) {
        last = p;
        if (p < 4) last_tie = p;
      }
    for (int p = 0; p < 12; ++p) {
      PassPlan q;
      q.active = act[p];
      q.first = act[p] && cnt == 0;
      q.src = cnt & 1;
      q.last = p == last;
      q.carry_lo = p < last_tie;  // a later tie pass still needs the ranks
      q.none = last < 0;
      plan[p] = q;
      cnt += act[p];
    }
    int low = 0, high = 0, use_lo = 0;
    for (int p = 0; p < 12; ++p) {
      if (p < 8) low += act[p]; else high += act[p];
      if (p < 4) use_lo |= act[p];
    }
    // speculate when it saves passes and the keys do not look repetitive
    // (a wrong guess costs the 4 high-word passes; the result is exact
    // either way)
    const double mean = (double)n / 256.0;
    unsigned long long sq = 0;
    for (int w = 0; w < 8; ++w) sq += sqw[w];
    const double ratio = plow >= 0 ? ((double)sq / 256.0 - mean * mean) / mean : 0.0;
    const int spec = high > 0 && low >= 2 && ratio < 8.0;
    int k = 0;
    for (int p = 0; p < 12; ++p) {
      PassPlan q{};
      q.active = spec && p >= 8 && act[p];
      q.first = q.active && k == 0;
      q.src = k & 1;
      q.carry_lo = use_lo;
      plan_hi[p] = q;  // never `last`: the keys go on to radix_fixup
      k += q.active;
    }
    FixPlan f;
    f.spec = spec;
    f.src = k & 1;  // after k passes the keys sit in buffer k & 1
    f.use_lo = use_lo;
    f.redo = !spec;
    *fix = f;
  }
}

// One thread per element of the high-word order: its run of equal top
// words (bounded scans both ways), and its place in the run by counting the
// run's smaller full keys (hi, tie if it orders, index) — every key is
// distinct, so the places are a permutation of the run.
__global__ void __launch_bounds__(256) radix_fixup(const uint64_t* __restrict__ khi0,
                                                   const uint64_t* __restrict__ khi1,
                                                   const uint32_t* __restrict__ klo0,
                                                   const uint32_t* __restrict__ klo1,
                                                   const uint32_t* __restrict__ val0,
                                                   const uint32_t* __restrict__ val1, int64_t n,
                                                   FixPlan* __restrict__ fix, uint32_t* __restrict__ order) {
  pdl_enter();
  if (!fix->spec) return;  // (uniform)
  const int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int src = fix->src;
  const uint64_t* kh = src ? khi1 : khi0;
  const uint32_t* kl = src ? klo1 : klo0;
  const uint32_t* kv = src ? val1 : val0;
  const bool valid = k < n;
  const uint64_t h = valid ? kh[k] : 0ull;
  const uint32_t top = (uint32_t)(h >> 32);
  // the keys are in top-word order, so k's run is longer than kFixRun iff
  // the key kFixRun places before or after k has the same top word: two
  // loads decide it, and no thread scans a long run
  const bool long_run = valid && ((k >= kFixRun && (uint32_t)(kh[k - kFixRun] >> 32) == top) ||
                                  (k + kFixRun < n && (uint32_t)(kh[k + kFixRun] >> 32) == top));
  if (__syncthreads_or(long_run)) {
    if (threadIdx.x == 0) atomicExch(&fix->redo, 1);
    return;
  }
  if (!valid) return;
  const uint32_t v = kv[k];
  int64_t a = k, b = k + 1;  // the run, at most kFixRun keys
  while (a > 0 && (uint32_t)(kh[a - 1] >> 32) == top) --a;
  while (b < n && (uint32_t)(kh[b] >> 32) == top) ++b;
  if (b - a == 1) {
    order[k] = v;
    return;
  }
  const bool use_lo = fix->use_lo;
  const uint32_t l = use_lo ? kl[k] : 0u;
  int64_t r = a;
  for (int64_t j = a; j < b; ++j) {
    const uint64_t hj = kh[j];
    const uint32_t lj = use_lo ? kl[j] : 0u, vj = kv[j];
    r += hj < h || (hj == h && (lj < l || (lj == l && vj < v)));
  }
  order[r] = v;
}

// One onesweep LSD pass: dynamic tile ids (launch order), per-tile digit
// counts by warp match_any ranking, the tile's global digit offsets by
// decoupled look-back over the previous tiles' (aggregate | inclusive
// prefix) status words, then the tile laid out in digit order in shared
// memory and written run by run (coalesced).
constexpr uint64_t kStAgg = 1ull << 62, kStPre = 2ull << 62, kStMask = (1ull << 62) - 1;

// 512 threads x 14 keys = 7,168-key tiles, one CTA per SM: 1M keys are 140
// tiles, one wave (a pass is latency-bound: two waves cost twice as much)
#ifndef PARS_SWEEP_THREADS
#define PARS_SWEEP_THREADS 512
#endif
constexpr int kSweepThreads = PARS_SWEEP_THREADS;
constexpr int kSweepWarps = kSweepThreads / 32;
#ifndef PARS_SWEEP_ITEMS
#define PARS_SWEEP_ITEMS 14
#endif
constexpr int kSweepItems = PARS_SWEEP_ITEMS;
constexpr int kSweepTile = kSweepThreads * kSweepItems;
constexpr size_t kSweepSmem = (size_t)kSweepWarps * 256 * 4 /* wcnt */ + 256 * 4 * 2 /* gbase, tstart */ +
                              64 /* wsum, tile */ + (size_t)kSweepTile * (8 + 4 + 4);

__device__ __forceinline__ unsigned long long ld_status(const unsigned long long* q) {
  return *reinterpret_cast<const volatile unsigned long long*>(q);
}

__global__ void __launch_bounds__(kSweepThreads) radix_onesweep(
    const double* __restrict__ score, const uint8_t* __restrict__ boosted,
    const uint32_t* __restrict__ tie, uint64_t* __restrict__ khi0, uint64_t* __restrict__ khi1,
    uint32_t* __restrict__ klo0, uint32_t* __restrict__ klo1, uint32_t* __restrict__ val0,
    uint32_t* __restrict__ val1, uint32_t* __restrict__ order, int64_t n, int pos,
    const PassPlan* __restrict__ plans, const uint32_t* __restrict__ dbase,
    unsigned long long* __restrict__ status, unsigned* __restrict__ tile_ctr,
    const FixPlan* __restrict__ gate) {
  pdl_enter();
  if (gate && !gate->redo) return;  // the speculative high-word sort held
  const PassPlan pl = plans[pos];
  if (!pl.active) {
    if (pos == 11 && pl.none)  // every key equal: the stable order is the input order
      for (int64_t i = (int64_t)blockIdx.x * kSweepThreads + threadIdx.x; i < n;
           i += (int64_t)gridDim.x * kSweepThreads)
        order[i] = (uint32_t)i;
    return;
  }
  extern __shared__ __align__(16) unsigned char osm[];
  uint64_t* s_hi = reinterpret_cast<uint64_t*>(osm);
  uint32_t* s_lo = reinterpret_cast<uint32_t*>(s_hi + kSweepTile);
  uint32_t* s_val = s_lo + kSweepTile;
  uint32_t (*wcnt)[256] = reinterpret_cast<uint32_t (*)[256]>(s_val + kSweepTile);
  uint32_t* gbase = &wcnt[kSweepWarps][0];
  uint32_t* tstart = gbase + 256;
  uint32_t* wsum = tstart + 256;  // [8]
  unsigned* s_tile = wsum + 8;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  if (threadIdx.x == 0) *s_tile = atomicAdd(tile_ctr, 1u);
  for (int k = threadIdx.x; k < kSweepWarps * 256; k += kSweepThreads) (&wcnt[0][0])[k] = 0;
  __syncthreads();
  const unsigned tile = *s_tile;
  const uint64_t* khi_in = pl.src ? khi1 : khi0;
  const uint32_t* klo_in = pl.src ? klo1 : klo0;
  const uint32_t* val_in = pl.src ? val1 : val0;
  uint64_t* khi_out = pl.src ? khi0 : khi1;
  uint32_t* klo_out = pl.src ? klo0 : klo1;
  uint32_t* val_out = pl.src ? val0 : val1;
  const bool need_lo = pos < 4 || pl.carry_lo;  // this pass reads the tie digits or carries them
  const int64_t sub = (int64_t)tile * kSweepTile + warp * (32 * kSweepItems);
  const unsigned lt = (1u << lane) - 1u;
  uint64_t hi[kSweepItems];
  uint32_t lo[kSweepItems], vv[kSweepItems], dr[kSweepItems];  // dr = digit << 16 | rank
#pragma unroll
  for (int r = 0; r < kSweepItems; ++r) {
    const int64_t i = sub + r * 32 + lane;
    const bool ok = i < n;
    if (pl.first) {
      hi[r] = ok ? ((boosted && boosted[i]) ? 0ull : ordered_bits(score[i])) : 0ull;
      lo[r] = (ok && tie) ? tie[i] : 0u;
      vv[r] = (uint32_t)i;
    } else {
      hi[r] = ok ? khi_in[i] : 0ull;
      lo[r] = (ok && need_lo) ? klo_in[i] : 0u;
      vv[r] = ok ? val_in[i] : 0u;
    }
  }
#pragma unroll
  for (int r = 0; r < kSweepItems; ++r) {
    const bool ok = sub + r * 32 + lane < n;
    const uint32_t d = ok ? digit_of(hi[r], lo[r], pos) : 256u;
#ifndef PARS_SWEEP_MATCH_RANK
    // the lanes holding the same digit, by 9 ballots (8 digit bits + the
    // out-of-range sentinel bit): on this part MATCH.ANY is slower (1 M keys:
    // 0.205 -> 0.191 ms per sort)
    unsigned peers = kFull;
#pragma unroll
    for (int bit = 0; bit < 9; ++bit) {
      const unsigned bb = __ballot_sync(kFull, (d >> bit) & 1u);
      peers &= ((d >> bit) & 1u) ? bb : ~bb;
    }
#else
    const unsigned peers = __match_any_sync(kFull, d);
#endif
    const uint32_t before = ok ? wcnt[warp][d] : 0u;
    dr[r] = (d << 16) | (before + __popc(peers & lt));
    __syncwarp();
    if (ok && (peers & lt) == 0) wcnt[warp][d] = before + __popc(peers);
    __syncwarp();
  }
  __syncthreads();
  const int d = threadIdx.x;  // threads 0..255: one digit each
  uint32_t run = 0, x = 0;
  if (d < 256) {
    for (int w = 0; w < kSweepWarps; ++w) {
      const uint32_t c = wcnt[w][d];
      wcnt[w][d] = run;
      run += c;
    }
    // decoupled look-back, four predecessors per step: publish the
    // aggregate, add predecessors' counts back to the first inclusive prefix
    unsigned long long* st = status + (size_t)tile * 256 + d;
    uint32_t excl = 0;
    if (tile == 0) {
      __stcg(st, kStPre | run);
    } else {
      __stcg(st, kStAgg | run);
      // kLook predecessors per step, loaded together: the inclusive-prefix
      // front advances kLook tiles per L2 round trip even when every tile
      // starts at once
      constexpr int kLook = 8;
      for (int64_t j = (int64_t)tile - 1;; j -= kLook) {
        const unsigned long long* q = status + (size_t)j * 256 + d;
        unsigned long long v[kLook];
#pragma unroll
        for (int k = 0; k < kLook; ++k) v[k] = j >= k ? ld_status(q - (size_t)k * 256) : kStPre;
        bool done = false;
#pragma unroll
        for (int k = 0; k < kLook; ++k) {
          if (!done) {
            while ((v[k] & ~kStMask) == 0) v[k] = ld_status(q - (size_t)k * 256);
            excl += (uint32_t)(v[k] & kStMask);
            done = (v[k] & ~kStMask) == kStPre;
          }
        }
        if (done) break;
      }
      __stcg(st, kStPre | (excl + run));
    }
    gbase[d] = dbase[pos * 256 + d] + excl;
    // the tile's digit runs: exclusive scan of the run lengths
    x = run;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const uint32_t y = __shfl_up_sync(kFull, x, o);
      if (lane >= o) x += y;
    }
    if (lane == 31) wsum[warp] = x;
  }
  __syncthreads();
  if (d < 256) {
    uint32_t wb = 0;
    for (int w = 0; w < warp; ++w) wb += wsum[w];
    tstart[d] = wb + x - run;
  }
  __syncthreads();
#pragma unroll
  for (int r = 0; r < kSweepItems; ++r) {
    const uint32_t dg = dr[r] >> 16;
    if (dg < 256u) {
      const uint32_t lp = tstart[dg] + wcnt[warp][dg] + (dr[r] & 0xffffu);
      s_hi[lp] = hi[r];
      s_lo[lp] = lo[r];
      s_val[lp] = vv[r];
    }
  }
  __syncthreads();
  const int64_t t0 = (int64_t)tile * kSweepTile;
  const int cnt = (int)(n - t0 < kSweepTile ? n - t0 : (int64_t)kSweepTile);
  for (int k = threadIdx.x; k < cnt; k += kSweepThreads) {
    const uint64_t h = s_hi[k];
    const uint32_t l = s_lo[k];
    const uint32_t dd = digit_of(h, l, pos);
    const uint32_t p = gbase[dd] + (uint32_t)k - tstart[dd];
    if (pl.last) {
      order[p] = s_val[k];
    } else {
      khi_out[p] = h;
      if (pl.carry_lo) klo_out[p] = l;
      val_out[p] = s_val[k];
    }
  }
}

}  // namespace

namespace {
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
// total order equal to the global sort's (key, tie, then input index) with
// no two keys equal. An element's place in the merged order is then its
// position in its own run plus, for every other run, the number of that
// run's keys below it (one binary search per run): one level, any run count,
// and each element's place is independent of every other's — so a data-
// parallel rank can place only its own run's elements (launch_merge_rank
// with run >= 0) and the ranks' disjoint outputs combine by a sum.
namespace {
__global__ void merge_keys_kernel(const double* __restrict__ score, const uint8_t* __restrict__ boosted,
                                  const uint32_t* __restrict__ tie, const uint32_t* __restrict__ run_order,
                                  const RunOffsets off, int64_t n, uint64_t* __restrict__ hi,
                                  uint64_t* __restrict__ lo) {
  const int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (k >= n) return;
  int r = 0;
  while (r + 1 < off.nruns && off.off[r + 1] <= k) ++r;  // nruns is the rank count: small
  const uint32_t i = (uint32_t)(off.off[r] + run_order[k]);
  hi[k] = (boosted && boosted[i]) ? 0ull : ordered_bits(score[i]);
  lo[k] = ((uint64_t)(tie ? tie[i] : 0u) << 32) | i;
}

__device__ __forceinline__ bool key_less(uint64_t ah, uint64_t al, uint64_t bh, uint64_t bl) {
  return ah < bh || (ah == bh && al < bl);
}

// Elements [k0, k1) (one run, or all): order[place] = input index.
__global__ void merge_rank_kernel(const uint64_t* __restrict__ hi, const uint64_t* __restrict__ lo,
                                  const RunOffsets off, int64_t k0, int64_t k1,
                                  uint32_t* __restrict__ order) {
  const int64_t k = k0 + (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (k >= k1) return;
  int r = 0;
  while (r + 1 < off.nruns && off.off[r + 1] <= k) ++r;
  const uint64_t h = hi[k], l = lo[k];
  int64_t pos = k - off.off[r];
  for (int j = 0; j < off.nruns; ++j) {
    if (j == r) continue;
    int64_t a = off.off[j], b = off.off[j + 1];  // first element of run j above (h, l)
    const int64_t s0 = a;
    while (a < b) {
      const int64_t m = (a + b) >> 1;
      if (key_less(hi[m], lo[m], h, l)) a = m + 1; else b = m;
    }
    pos += a - s0;
  }
  order[pos] = (uint32_t)l;
}

}  // namespace

size_t merge_runs_scratch_bytes(int64_t n, int nruns) {
  (void)nruns;
  return 2 * ((size_t)n * 8 + 256);
}

int launch_merge_rank(pars_ctx* ctx, const double* score, const uint8_t* boosted, const uint32_t* tie,
                      const uint32_t* run_order, const int64_t* h_off, int nruns, int run,
                      uint32_t* order, void* scratch, cudaStream_t st) {
  if (nruns < 1 || nruns > kMaxRuns) {
    set_error("merge_orders: %d runs (supported: 1..%d)", nruns, kMaxRuns);
    return PARS_ERR_UNSUPPORTED;
  }
  const int64_t n = h_off[nruns];
  if (n == 0) return PARS_OK;
  if (n > 0x7fffffffLL) {
    set_error("priority order: n=%lld exceeds 2^31-1", (long long)n);
    return PARS_ERR_UNSUPPORTED;
  }
  RunOffsets off{};
  off.nruns = nruns;
  for (int r = 0; r <= nruns; ++r) off.off[r] = h_off[r];
  char* p = static_cast<char*>(scratch);
  uint64_t* hi = (uint64_t*)p;
  uint64_t* lo = (uint64_t*)(p + (((size_t)n * 8 + 255) & ~(size_t)255));
  const int64_t k0 = run < 0 ? 0 : h_off[run], k1 = run < 0 ? n : h_off[run + 1];
  merge_keys_kernel<<<(unsigned)ceil_div(n, 256), 256, 0, st>>>(score, boosted, tie, run_order, off, n,
                                                                 hi, lo);
  count_launch(ctx);
  if (k1 > k0) {
    merge_rank_kernel<<<(unsigned)ceil_div(k1 - k0, 256), 256, 0, st>>>(hi, lo, off, k0, k1, order);
    count_launch(ctx);
  }
  PARS_CUDA_CHECK(cudaGetLastError());
  return PARS_OK;
}

int launch_merge_runs(pars_ctx* ctx, const double* score, const uint8_t* boosted, const uint32_t* tie,
                      const uint32_t* run_order, const int64_t* h_off, int nruns, int64_t n,
                      uint32_t* order, void* scratch, cudaStream_t st) {
  (void)n;
  return launch_merge_rank(ctx, score, boosted, tie, run_order, h_off, nruns, -1, order, scratch, st);
}

size_t sort_scratch_bytes(int64_t n) {
  const int64_t nb = ceil_div(std::max<int64_t>(n, 1), kSweepTile);
  size_t b = 0;
  b += 2 * ((size_t)n * 8 + 256) + 2 * ((size_t)n * 4 + 256) * 2;  // khi, klo, val ping-pong
  b += (size_t)nb * 256 * 8 * 16 + 256;                            // look-back status per pass (4 + 12)
  b += 12 * 256 * 4 * 2 + 1024 + 24 * sizeof(PassPlan) + 256 + 64 * 4;  // histograms, bases, plans, tile ids
  return b + 4096;
}

namespace {
template <typename... KArgs, typename... Args>
cudaError_t launch_pdl(void (*kernel)(KArgs...), unsigned grid, unsigned block, size_t smem, cudaStream_t st,
                       Args... args) {
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(block);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, kernel, static_cast<KArgs>(args)...);
}
}  // namespace

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
  const int nb = (int)ceil_div(n, kSweepTile);
  char* p = static_cast<char*>(scratch);
  auto take = [&](size_t bytes) {
    char* r = p;
    p += (bytes + 255) & ~(size_t)255;
    return r;
  };
  uint64_t* khi[2] = {(uint64_t*)take(n * 8), (uint64_t*)take(n * 8)};
  uint32_t* klo[2] = {(uint32_t*)take(n * 4), (uint32_t*)take(n * 4)};
  uint32_t* val[2] = {(uint32_t*)take(n * 4), (uint32_t*)take(n * 4)};
  // zeroed together: status words, tile counters, histograms + tie flag
  const size_t status_bytes = (size_t)nb * 256 * 8 * 16;  // 4 high-word passes + 12
  char* zero0 = p;
  auto* status = (unsigned long long*)take(status_bytes);
  auto* tile_ctr = (unsigned*)take(64 * 4);
  auto* dh = (uint32_t*)take(12 * 256 * 4 + 16);
  const size_t zero_bytes = (size_t)(p - zero0);
  auto* dbase = (uint32_t*)take(12 * 256 * 4);
  auto* plan = (PassPlan*)take(12 * sizeof(PassPlan));
  auto* plan_hi = (PassPlan*)take(12 * sizeof(PassPlan));
  auto* fix = (FixPlan*)take(sizeof(FixPlan));
  PARS_CUDA_CHECK(cudaMemsetAsync(zero0, 0, zero_bytes, st));
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const int64_t ig = std::min<int64_t>(ceil_div(n, 256), (int64_t)sms * 2);
  radix_init<<<(unsigned)ig, 256, 0, st>>>(score, boosted, tie, n, dh);
  static bool attr = [] {
    return cudaFuncSetAttribute(radix_onesweep, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                (int)kSweepSmem) == cudaSuccess;
  }();
  if (!attr) {
    set_error("priority order: cannot configure the sort kernel's shared memory");
    return PARS_ERR_CUDA;
  }
  PARS_CUDA_CHECK(launch_pdl(radix_plan, 1, 256, 0, st, dh, n, plan, plan_hi, fix, dbase));
  count_launch(ctx, 2);
  const FixPlan* no_gate = nullptr;
  // without speculation the full LSD runs ungated
  static const int64_t spec_min = [] {
    const char* e = std::getenv("PARS_SORT_SPEC_MIN");
    return e ? std::atoll(e) : (int64_t)kSpecMin;
  }();
  const bool speculate = n >= spec_min;
  for (int pos = 8; speculate && pos < 12; ++pos) {  // speculative: the top 32 bits only
    PARS_CUDA_CHECK(launch_pdl(radix_onesweep, (unsigned)nb, kSweepThreads, kSweepSmem, st, score, boosted, tie,
                               khi[0], khi[1], klo[0], klo[1], val[0], val[1], order, n, pos, plan_hi, dbase,
                               status + (size_t)nb * 256 * (pos - 8), tile_ctr + pos, no_gate));
    count_launch(ctx);
  }
  if (speculate) {
    PARS_CUDA_CHECK(launch_pdl(radix_fixup, (unsigned)ceil_div(n, 256), 256, 0, st, khi[0], khi[1], klo[0],
                               klo[1], val[0], val[1], n, fix, order));
    count_launch(ctx);
  }
  // the full LSD sort, gated on fix->redo; without tie ranks the tie digits
  // are all zero: those passes are known trivial on the host and not launched
  for (int pos = tie ? 0 : 4; pos < 12; ++pos) {
    PARS_CUDA_CHECK(launch_pdl(radix_onesweep, (unsigned)nb, kSweepThreads, kSweepSmem, st, score, boosted, tie,
                               khi[0], khi[1], klo[0], klo[1], val[0], val[1], order, n, pos, plan, dbase,
                               status + (size_t)nb * 256 * (4 + pos), tile_ctr + 16 + pos,
                               speculate ? (const FixPlan*)fix : no_gate));
    count_launch(ctx);
  }
  PARS_CUDA_CHECK(cudaGetLastError());
  return PARS_OK;
}

}  // namespace pars_b200
