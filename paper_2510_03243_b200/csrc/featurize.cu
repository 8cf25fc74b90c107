// Fused hashing featurizer + linear score head.
//
// Reference semantics (all in /root/reference/proj/src/features.cpp):
//   split_tokens :36-49 (C-locale isspace), word n-grams :80-92 (FNV-1a over
//   token bytes then "\x1f", seeded by salt(1, order)), char n-grams inside
//   tokens :93-101 (salt(2, order)), add_hashed :29-34 (idx = (h>>1) % dim,
//   sign = h&1 ? +1 : -1), sort+merge :102-109, erase zeros :110,
//   L2 :113-120; scorer.cpp:36-42 + features.hpp:31-35 for the dot + bias.
//
// B200 design (one warp owns one prompt at a time):
//   * tokenise: the prompt streams through the warp in 128-byte windows (one
//     aligned 32-bit load per lane, next window prefetched); whitespace
//     transitions come from lane bit masks, are ranked with 4 ballots and
//     written to a per-warp transition ring in shared memory (transitions
//     strictly alternate start/end, so token t = ring[2t], ring[2t+1]);
//   * hash: lane t hashes token t of a 32-token batch (word n-gram + all char
//     n-grams of that token). For power-of-two dims only the low log2(dim)+1
//     bits of the 64-bit FNV state are observed and FNV is closed mod 2^32,
//     so the hash runs in 32-bit arithmetic (P mod 2^32 = 0x1b3);
//   * histogram: per-warp shared-memory table of biased 16-bit counters, two
//     per word (atomicAdd); prompts with more than 32,767 hashed features are
//     routed to the 32-bit-counter variant (so a counter can never wrap). The
//     atomics' old values give the exact change of sum(count^2) (2cd+1), so
//     the L2 norm needs no extra pass; a bitmap records first touches;
//   * finish (exact fp64 mode): the touched buckets are walked in ascending
//     order into a per-warp list (idx, count) in L2-resident global scratch;
//     after a group of 16 prompts, lane k runs the sequential __dadd_rn chain
//     of prompt k (products w[idx] * (count * inv) with __dmul_rn), so 16
//     bit-exact chains proceed in parallel instead of one lane at a time.
//     Fast fp32 mode reduces lane-parallel products with a warp tree; CSR
//     mode compacts (idx, value) rows.
#include <cuda_pipeline.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdlib>
#include <cstring>

#include "featurize.cuh"

namespace pars_b200 {

namespace {

constexpr unsigned kFull = 0xffffffffu;
constexpr int kRing = 256;                   // transition ring entries per warp
constexpr int kGroup = 16;                   // prompts per exact chain group (one per lane)
constexpr uint32_t kBias2 = 0x80008000u;     // two biased 16-bit zero counters
constexpr int64_t kNarrowMaxFeatures = 32767;  // |count| <= features: 16 bits cannot wrap
constexpr size_t kMaxSmemPerBlock = 200 * 1024;
constexpr size_t kMaxLaneSmem = 227 * 1024;  // per-CTA opt-in maximum on sm_100

struct WarpSmem {
  uint32_t* counts;  // narrow: 2 x u16 biased per word; wide: int32
  uint32_t* bitmap;  // touched buckets
  uint32_t* ring;    // token transitions (relative byte offsets)
};

__host__ __device__ inline uint32_t bitmap_words_padded(uint32_t dim) {
  uint32_t w = (dim + 31) / 32;
  return (w + 7) & ~7u;
}
// Covers every 8-bucket group that can be touched (clears are per group).
__host__ __device__ inline uint32_t count_words(uint32_t dim, bool wide) {
  return wide ? ((dim + 7) / 8) * 8 : ((dim + 7) / 8) * 4;  // multiple of 4 words (16 B)
}
__host__ __device__ inline size_t warp_table_bytes(const FeatConfig& c, bool wide) {
  return (size_t)count_words(c.dim, wide) * 4 + (size_t)bitmap_words_padded(c.dim) * 4 +
         (size_t)kRing * 4;
}
// list entry: packed u32 (idx << 16 | count + 0x8000) for narrow counters and
// dim <= 65536, else two u32 (idx, count)
__host__ __device__ inline uint32_t entry_words(const FeatConfig& c, bool wide) {
  return (!wide && c.dim <= 65536u) ? 1u : 2u;
}
// Per-warp list arena (u32 words), the same stride for the narrow and the
// wide kernel: a full group of typical prompts, and never less than one
// prompt's worst case (dim entries).
__host__ inline uint32_t list_cap_words(const FeatConfig& c) {
  uint32_t cap = 0;
  for (int wide = 0; wide < 2; ++wide) {
    const uint32_t ew = entry_words(c, wide != 0);
    cap = std::max<uint32_t>(cap, std::max<uint32_t>(c.dim * ew, kGroup * 512u * ew) + 4u * ew);
  }
  return (cap + 3u) & ~3u;
}

// One hashed feature: +-1 into its bucket; the first touch of a bucket (old
// count 0) sets its bit in the touched bitmap.
template <bool WIDE>
__device__ __forceinline__ void emit(const WarpSmem& S, uint32_t idx, bool pos) {
  bool first;
  if (WIDE) {
    first = atomicAdd(&S.counts[idx], pos ? 1u : 0xffffffffu) == 0u;
  } else {
    const uint32_t sh = (idx & 1u) << 4;
    const uint32_t d = pos ? (1u << sh) : (0u - (1u << sh));
    first = ((atomicAdd(&S.counts[idx >> 1], d) >> sh) & 0xffffu) == 0x8000u;
  }
  if (first) atomicOr(&S.bitmap[idx >> 5], 1u << (idx & 31));
}

template <bool WIDE>
__device__ __forceinline__ int count_of(const WarpSmem& S, uint32_t idx) {
  if (WIDE) return (int)S.counts[idx];
  return (int)reinterpret_cast<const uint16_t*>(S.counts)[idx] - 0x8000;  // little-endian halves
}

// Reset the 8 counters of buckets [b0, b0+8) (b0 % 8 == 0).
template <bool WIDE>
__device__ __forceinline__ void clear_group(const WarpSmem& S, uint32_t b0) {
  if (WIDE) {
    *reinterpret_cast<uint4*>(S.counts + b0) = make_uint4(0u, 0u, 0u, 0u);
    *reinterpret_cast<uint4*>(S.counts + b0 + 4) = make_uint4(0u, 0u, 0u, 0u);
  } else {
    *reinterpret_cast<uint4*>(S.counts + (b0 >> 1)) = make_uint4(kBias2, kBias2, kBias2, kBias2);
  }
}

template <bool WIDE>
__device__ void clear_all(const WarpSmem& S, const FeatConfig& c, int lane) {
  const uint32_t cw = count_words(c.dim, WIDE);
  for (uint32_t k = lane; k < cw; k += 32) S.counts[k] = WIDE ? 0u : kBias2;
  for (uint32_t k = lane; k < bitmap_words_padded(c.dim); k += 32) S.bitmap[k] = 0u;
  __syncwarp();
}

// Hash state: 32-bit when only the low bits matter (power-of-two dims).
template <bool POW2>
struct H;
template <>
struct H<true> {
  using T = uint32_t;
  __device__ static __forceinline__ T step(T h, uint32_t b) { return (h ^ b) * 0x1b3u; }
  __device__ static __forceinline__ T seed(uint64_t s) { return (uint32_t)s; }
  __device__ static __forceinline__ uint32_t bucket(T h, const FeatConfig& c) {
    return (h >> 1) & c.mask;
  }
};
template <>
struct H<false> {
  using T = uint64_t;
  __device__ static __forceinline__ T step(T h, uint32_t b) { return (h ^ b) * kFnvPrime; }
  __device__ static __forceinline__ T seed(uint64_t s) { return s; }
  __device__ static __forceinline__ uint32_t bucket(T h, const FeatConfig& c) {
    return (uint32_t)((h >> 1) % c.dim);
  }
};

__device__ __forceinline__ uint32_t ld_byte(const uint8_t* p) { return __ldg(p); }

// Hash token `t` (from the transition ring) and every n-gram that starts at
// it: the general path for arbitrary word/char n-gram orders.
template <bool POW2, bool WIDE, bool DEF>
__device__ __forceinline__ void hash_token(const FeatConfig& c, const WarpSmem& S,
                                           const uint8_t* base, uint32_t t, uint32_t ntok) {
  using HT = H<POW2>;
  using T = typename HT::T;
  const uint32_t s = S.ring[(2 * t) & (kRing - 1)], e = S.ring[(2 * t + 1) & (kRing - 1)];
  const uint8_t* tp = base + s;
  const int len = (int)(e - s);
  if (DEF) {
    // word {1} + char {3} in one pass; two bytes per iteration so the two
    // trigram hashes of a step are independent
    T hw = HT::seed(c.word_salt[0]);
    const T hc0 = HT::seed(c.char_salt[0]);
    uint32_t b2 = 0, b1 = 0;
    int i = 0;
    for (; i + 2 <= len; i += 2) {
      const uint32_t x = ld_byte(tp + i), y = ld_byte(tp + i + 1);
      hw = HT::step(HT::step(hw, x), y);
      if (i >= 2) {
        const T h = HT::step(HT::step(HT::step(hc0, b2), b1), x);
        emit<WIDE>(S, HT::bucket(h, c), (h & 1) != 0);
        const T g = HT::step(HT::step(HT::step(hc0, b1), x), y);
        emit<WIDE>(S, HT::bucket(g, c), (g & 1) != 0);
      }
      b2 = x;
      b1 = y;
    }
    if (i < len) {
      const uint32_t x = ld_byte(tp + i);
      hw = HT::step(hw, x);
      if (i >= 2) {
        const T h = HT::step(HT::step(HT::step(hc0, b2), b1), x);
        emit<WIDE>(S, HT::bucket(h, c), (h & 1) != 0);
      }
    }
    hw = HT::step(hw, 0x1fu);
    emit<WIDE>(S, HT::bucket(hw, c), (hw & 1) != 0);
    return;
  }
  for (int k = 0; k < c.n_word; ++k) {
    const int order = c.word[k];
    if (t + (uint32_t)order > ntok) continue;  // n-gram runs past the last token
    T h = HT::seed(c.word_salt[k]);
    for (int j = 0; j < order; ++j) {
      const uint32_t sj = S.ring[(2 * (t + j)) & (kRing - 1)];
      const uint32_t ej = S.ring[(2 * (t + j) + 1) & (kRing - 1)];
      for (uint32_t q = sj; q < ej; ++q) h = HT::step(h, ld_byte(base + q));
      h = HT::step(h, 0x1fu);
    }
    emit<WIDE>(S, HT::bucket(h, c), (h & 1) != 0);
  }
  for (int k = 0; k < c.n_char; ++k) {
    const int order = c.chr[k];
    const T seed = HT::seed(c.char_salt[k]);
    for (int i = 0; i + order <= len; ++i) {
      T h = seed;
      for (int j = 0; j < order; ++j) h = HT::step(h, ld_byte(tp + i + j));
      emit<WIDE>(S, HT::bucket(h, c), (h & 1) != 0);
    }
  }
}

// SWAR: bit k of the result = byte k of w is not C-locale whitespace.
__device__ __forceinline__ uint32_t nonspace_nibble(uint32_t w) {
  const uint32_t x = w ^ 0x20202020u;  // zero byte where ' '
  const uint32_t not_blank = ((x & 0x7f7f7f7fu) + 0x7f7f7f7fu) | x;  // high bit: byte != ' '
  // high bit: byte in [9, 13] (\t \n \v \f \r); bytes >= 0x80 are never spaces
  const uint32_t lo7 = w & 0x7f7f7f7fu;
  const uint32_t ctl = (0x8d8d8d8du - lo7) & ~w & (lo7 + 0x77777777u);
  const uint32_t ns_hi = not_blank & ~ctl & 0x80808080u;
  return ((ns_hi >> 7) * 0x01020408u) >> 24;
}

__device__ __forceinline__ int warp_excl_scan(int v, int lane, int* total) {
  int x = v;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    int y = __shfl_up_sync(kFull, x, o);
    if (lane >= o) x += y;
  }
  *total = __shfl_sync(kFull, x, 31);
  return x - v;
}

// 4 text bytes at base[p .. p+4) (p relative, may be out of range: spaces).
__device__ __forceinline__ uint32_t load_word(const uint8_t* base, int64_t p, int64_t len) {
  if (p >= 0 && p + 4 <= len) return __ldg(reinterpret_cast<const uint32_t*>(base + p));
  uint32_t word = 0x20202020u;
#pragma unroll
  for (int k = 0; k < 4; ++k)
    if (p + k >= 0 && p + k < len)
      word = (word & ~(0xffu << (8 * k))) | ((uint32_t)base[p + k] << (8 * k));
  return word;
}

// Tokeniser + hasher: whitespace transitions (SWAR non-space nibble per
// lane) are ranked with 4 ballots into the per-warp transition ring; lane t
// hashes token t of each complete 32-token batch, so every lane has exactly
// one token per batch whatever the token-length mix.
template <bool POW2, bool WIDE, bool DEF>
__device__ void hash_prompt_ring(const FeatConfig& c, const WarpSmem& S, const uint8_t* base,
                                 int64_t len, int lane) {
  uint32_t n_tr = 0, done = 0;
  uint32_t carry_ns = 0;
  const uint32_t look = c.max_word > 1 ? (uint32_t)c.max_word - 1 : 0;
  const unsigned lt = (1u << lane) - 1u;
  // windows are aligned on the ABSOLUTE address so each lane's 4-byte load
  // is naturally aligned whatever the arena/offset alignment
  const int64_t mis = (int64_t)(reinterpret_cast<uintptr_t>(base) & 3u);
  uint32_t next = load_word(base, -mis + 4 * lane, len);
  for (int64_t wrel = -mis; wrel < len; wrel += 128) {
    const int64_t p = wrel + 4 * lane;  // relative to base; may be negative
    const uint32_t word = next;
    if (wrel + 128 < len) next = load_word(base, p + 128, len);
    const uint32_t ns = nonspace_nibble(word);
    uint32_t prev = __shfl_up_sync(kFull, ns >> 3, 1);
    if (lane == 0) prev = carry_ns;
    const uint32_t trm = (ns ^ ((ns << 1) | prev)) & 0xfu;  // transitions at byte k
    carry_ns = __shfl_sync(kFull, ns >> 3, 31);
    uint32_t rank = 0, tot = 0;
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      const uint32_t b = __ballot_sync(kFull, (trm >> k) & 1u);
      rank += __popc(b & lt);
      tot += __popc(b);
    }
    const uint32_t rel = (uint32_t)p;
    for (uint32_t m = trm; m; m &= m - 1) S.ring[(n_tr + rank++) & (kRing - 1)] = rel + __ffs(m) - 1;
    n_tr += tot;
    __syncwarp();
    while ((n_tr >> 1) - done >= 32 + look) {
      hash_token<POW2, WIDE, DEF>(c, S, base, done + lane, n_tr >> 1);
      done += 32;
      __syncwarp();
    }
  }
  if (carry_ns) {  // the last token runs to the end of the prompt
    if (lane == 0) S.ring[n_tr & (kRing - 1)] = (uint32_t)len;
    ++n_tr;
    __syncwarp();
  }
  const uint32_t ntok = n_tr >> 1;
  while (done < ntok) {
    if (done + lane < ntok) hash_token<POW2, WIDE, DEF>(c, S, base, done + lane, ntok);
    done += 32;
  }
  __syncwarp();
}

__device__ __forceinline__ long long warp_sum_i64(long long v) {
#pragma unroll
  for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(kFull, v, o);
  return v;
}
__device__ __forceinline__ uint32_t warp_sum_u32(uint32_t v) { return __reduce_add_sync(kFull, v); }
__device__ __forceinline__ float warp_sum_f32(float v) {
#pragma unroll
  for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(kFull, v, o);
  return v;
}

// Window = 8 bitmap words (256 buckets); lane l owns byte (l&3) of word
// (l>>2), i.e. buckets [b0, b0+8): lane order is bucket order. A lane's
// rank in the window is the popcount of the window's bits before its own,
// from two broadcast 16-byte loads.
struct Win {
  uint32_t bits, before, total, b0;
  bool empty;
};
__device__ __forceinline__ Win window(const WarpSmem& S, uint32_t wb, int lane) {
  const int sub = lane & 3, wsel = lane >> 2;
  const uint4 q0 = *reinterpret_cast<const uint4*>(S.bitmap + wb);
  const uint4 q1 = *reinterpret_cast<const uint4*>(S.bitmap + wb + 4);
  const uint32_t wv[8] = {q0.x, q0.y, q0.z, q0.w, q1.x, q1.y, q1.z, q1.w};
  Win w;
  w.empty = (q0.x | q0.y | q0.z | q0.w | q1.x | q1.y | q1.z | q1.w) == 0;
  uint32_t before = 0, total = 0, mine = 0;
#pragma unroll
  for (int k = 0; k < 8; ++k) {
    const uint32_t pk = __popc(wv[k]);
    total += pk;
    before += (k < wsel) ? pk : 0u;
    mine = (k == wsel) ? wv[k] : mine;
  }
  w.before = before + __popc(mine & ((1u << (8 * sub)) - 1u));
  w.bits = (mine >> (8 * sub)) & 0xffu;
  w.total = total;
  w.b0 = (wb + wsel) * 32 + 8 * sub;
  return w;
}

// Exact mode: append the prompt's touched buckets, ascending, to `list`
// (zero-count entries included: they add +0.0, a no-op on a chain that
// starts at +0.0 under round-to-nearest) and return the exact integer
// sum(count^2) (features.cpp:113-116). Clears the table.
template <bool WIDE>
__device__ long long walk_to_list(const FeatConfig& c, const WarpSmem& S, uint32_t* list,
                                  bool packed, int lane) {
  long long sq = 0;
  const uint32_t nbw = bitmap_words_padded(c.dim);
  uint32_t run = 0;
  for (uint32_t wb = 0; wb < nbw; wb += 8) {
    const Win w = window(S, wb, lane);
    if (w.empty) continue;
    uint32_t pos = run + w.before;
    for (uint32_t m = w.bits; m; m &= m - 1) {
      const uint32_t idx = w.b0 + __ffs(m) - 1;
      const int cnt = count_of<WIDE>(S, idx);
      sq += (long long)cnt * cnt;
      if (packed) {
        list[pos] = (idx << 16) | (uint32_t)(cnt + 0x8000);
      } else {
        list[2 * pos] = idx;
        list[2 * pos + 1] = (uint32_t)cnt;
      }
      ++pos;
    }
    if (w.bits) clear_group<WIDE>(S, w.b0);
    __syncwarp();
    if ((lane & 3) == 0) S.bitmap[wb + (lane >> 2)] = 0u;
    run += w.total;
  }
  __syncwarp();
  return warp_sum_i64(sq);
}

__device__ __forceinline__ double inv_norm(const FeatConfig& c, long long sq) {
  return (c.norm && sq > 0) ? __ddiv_rn(1.0, __dsqrt_rn((double)sq)) : 1.0;
}

__device__ __forceinline__ uint32_t touched_total(const FeatConfig& c, const WarpSmem& S, int lane) {
  uint32_t t = 0;
  for (uint32_t k = lane; k < bitmap_words_padded(c.dim); k += 32) t += __popc(S.bitmap[k]);
  return warp_sum_u32(t);
}

// Lane k < n: the sequential fp64 dot of group member k (features.hpp:31-35).
__device__ void chain_group(const FeatConfig& c, const FeatArgs& a, const uint32_t* lists,
                            bool packed, int lane, int n, int64_t prompt, uint32_t off,
                            uint32_t cnt_entries, double inv) {
  if (lane < n) {
    double s = 0.0;
    const double* __restrict__ w = a.w64;
    if (packed) {
      const uint32_t* L = lists + off;
      // the whole list into L1 first (it was written long enough ago to have
      // left L1), so the sequential chain below does not wait on L2 per load
      for (uint32_t q = 0; q < cnt_entries; q += 32)
        asm volatile("prefetch.global.L1 [%0];" ::"l"(L + q));
      uint32_t k = 0;
      for (; k + 4 <= cnt_entries; k += 4) {
        const uint4 e = *reinterpret_cast<const uint4*>(L + k);
        const uint32_t ev[4] = {e.x, e.y, e.z, e.w};
        double p[4];
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          const int cn = (int)(ev[j] & 0xffffu) - 0x8000;
          const double v = c.norm ? __dmul_rn((double)cn, inv) : (double)cn;
          p[j] = cn != 0 ? __dmul_rn(__ldg(w + (ev[j] >> 16)), v) : 0.0;
        }
#pragma unroll
        for (int j = 0; j < 4; ++j) s = __dadd_rn(s, p[j]);
      }
      for (; k < cnt_entries; ++k) {
        const uint32_t e = L[k];
        const int cn = (int)(e & 0xffffu) - 0x8000;
        const double v = c.norm ? __dmul_rn((double)cn, inv) : (double)cn;
        s = __dadd_rn(s, cn != 0 ? __dmul_rn(__ldg(w + (e >> 16)), v) : 0.0);
      }
    } else {
      const uint32_t* L = lists + 2 * (size_t)off;
      for (uint32_t k = 0; k < cnt_entries; ++k) {
        const int cn = (int)L[2 * k + 1];
        const double v = c.norm ? __dmul_rn((double)cn, inv) : (double)cn;
        s = __dadd_rn(s, cn != 0 ? __dmul_rn(__ldg(w + L[2 * k]), v) : 0.0);
      }
    }
    a.scores[prompt] = __dadd_rn(s, a.bias);
  }
  __syncwarp();
}

// Fast fp32 mode and CSR mode finish one prompt in place.
template <bool WIDE, int MODE>
__device__ void finish_prompt(const FeatConfig& c, const WarpSmem& S, const FeatArgs& a, int64_t i,
                              int lane) {
  const uint32_t nbw = bitmap_words_padded(c.dim);
  long long sq = 0;
  if (MODE == kFeatCsr && c.norm) {  // values need inv before they are written
    for (uint32_t wb = 0; wb < nbw; wb += 8) {
      const Win w = window(S, wb, lane);
      for (uint32_t m = w.bits; m; m &= m - 1) {
        const int cnt = count_of<WIDE>(S, w.b0 + __ffs(m) - 1);
        sq += (long long)cnt * cnt;
      }
    }
    sq = warp_sum_i64(sq);
  }
  const double inv = inv_norm(c, sq);
  float facc = 0.f;
  int64_t row_pos = 0;
  const int64_t slot = (MODE == kFeatCsr) ? a.slot_base[i] : 0;
  for (uint32_t wb = 0; wb < nbw; wb += 8) {
    const Win w = window(S, wb, lane);
    if (w.empty) continue;
    if (MODE == kFeatScoreFast) {
      for (uint32_t m = w.bits; m; m &= m - 1) {
        const uint32_t idx = w.b0 + __ffs(m) - 1;
        const int cnt = count_of<WIDE>(S, idx);
        sq += (long long)cnt * cnt;
        facc += __ldg(a.w32 + idx) * (float)cnt;
      }
    } else {
      // CSR rows must not contain erased zeros (features.cpp:110): compact
      int cnt[8];
      uint32_t nz = 0;
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        cnt[j] = ((w.bits >> j) & 1u) ? count_of<WIDE>(S, w.b0 + j) : 0;
        nz |= (cnt[j] != 0 ? 1u : 0u) << j;
      }
      int tot;
      const int pos = warp_excl_scan(__popc(nz), lane, &tot);
#pragma unroll
      for (int j = 0; j < 8; ++j)
        if (nz & (1u << j)) {
          const double v = c.norm ? __dmul_rn((double)cnt[j], inv) : (double)cnt[j];
          const int64_t o = slot + row_pos + pos + __popc(nz & ((1u << j) - 1));
          a.out_idx[o] = w.b0 + j;
          a.out_val[o] = v;
          if (a.out_cnt) a.out_cnt[o] = cnt[j];
        }
      row_pos += tot;
    }
    if (w.bits) clear_group<WIDE>(S, w.b0);
    __syncwarp();
    if ((lane & 3) == 0) S.bitmap[wb + (lane >> 2)] = 0u;
  }
  if (MODE == kFeatScoreFast) {
    facc = warp_sum_f32(facc);
    const float finv = (float)inv_norm(c, warp_sum_i64(sq));
    if (lane == 0) a.scores[i] = (double)(facc * finv) + a.bias;
  } else {
    if (lane == 0) {
      a.out_nnz[i] = (int32_t)row_pos;
      if (a.out_inv) a.out_inv[i] = inv;  // v = count * inv, exactly
    }
  }
  __syncwarp();
}

// G: the per-warp tables live in global scratch (dims too large for smem).
template <bool POW2, bool WIDE, bool DEF, int MODE, bool G>
__global__ void __launch_bounds__(256) featurize_kernel(const FeatConfig c, const FeatArgs a) {
  extern __shared__ __align__(16) unsigned char smem[];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int64_t gw = (int64_t)blockIdx.x * (blockDim.x >> 5) + warp;
  const int64_t nw = (int64_t)gridDim.x * (blockDim.x >> 5);
  const size_t per = warp_table_bytes(c, WIDE);
  unsigned char* my = G ? a.gscratch + per * (size_t)gw : smem + per * warp;
  WarpSmem S;
  S.counts = reinterpret_cast<uint32_t*>(my);
  S.bitmap = S.counts + count_words(c.dim, WIDE);
  S.ring = S.bitmap + bitmap_words_padded(c.dim);
  clear_all<WIDE>(S, c, lane);

  const bool packed = entry_words(c, WIDE) == 1;
  uint32_t* lists = (MODE == kFeatScoreExact) ? a.lists + (size_t)gw * a.list_cap : nullptr;
  // exact-mode group state: lane k holds member k
  int gn = 0;
  uint32_t used = 0;
  int64_t g_prompt = 0;
  uint32_t g_off = 0, g_cnt = 0;
  double g_inv = 1.0;

  const int64_t count = WIDE ? (int64_t)*a.long_count : a.n;
  for (int64_t it = gw; it < count; it += nw) {
    const int64_t i = WIDE ? (int64_t)a.long_list[it] : it;
    const int64_t beg = a.offsets[i], end = a.offsets[i + 1];
    const int64_t len = end - beg;
    if (!WIDE) {
      const int64_t feats = (int64_t)c.n_word * ((len + 1) / 2) + (int64_t)c.n_char * len;
      if (feats > kNarrowMaxFeatures) {
        if (lane == 0) a.long_list[atomicAdd(a.long_count, 1)] = (int32_t)i;
        continue;
      }
    }
    hash_prompt_ring<POW2, WIDE, DEF>(c, S, a.text + beg, len, lane);
    if (MODE == kFeatScoreExact) {
      const uint32_t n_ent = touched_total(c, S, lane);
      const uint32_t ew = packed ? 1u : 2u;
      const uint32_t need = ((n_ent + 3) & ~3u) * ew;
      if (gn == kGroup || used + need > a.list_cap) {
        chain_group(c, a, lists, packed, lane, gn, g_prompt, g_off, g_cnt, g_inv);
        gn = 0;
        used = 0;
      }
      const uint32_t off = used / ew;
      const double inv = inv_norm(c, walk_to_list<WIDE>(c, S, lists + used, packed, lane));
      if (lane == gn) {
        g_prompt = i;
        g_off = off;
        g_cnt = n_ent;
        g_inv = inv;
      }
      ++gn;
      used += need;
    } else {
      finish_prompt<WIDE, MODE>(c, S, a, i, lane);
    }
  }
  if (MODE == kFeatScoreExact && gn > 0)
    chain_group(c, a, lists, packed, lane, gn, g_prompt, g_off, g_cnt, g_inv);
}

// ---- sequential-lane front end (word {1} + char {3}, power-of-two dims) ----
//
// The prompt is cut into 32 word-aligned byte ranges, one per lane; lane l
// owns every token that STARTS in its range (features.cpp:36-49 tokens) and
// runs the reference's per-byte loop over it sequentially — word FNV state
// plus the three rolling states whose last one is the char trigram ending at
// the byte (features.cpp:80-101) — reading the text straight from global
// memory 4 bytes at a time. Per 4-byte word the token structure comes from
// bit masks: non-space bits (SWAR), run starts, and token ownership by the
// carry-propagation identity ((ns + starts) ^ ns), which marks each owned run
// plus the space that ends it. Each byte emits at most one feature: the
// trigram ending at it (non-space byte, two non-space predecessors) or the
// word ending just before it (space byte). No shuffles, no ring, no
// per-token divergence beyond a lane's own range.
constexpr uint32_t kSeqMinDim = 1024, kSeqMaxDim = 16384;

// biased u16 counters + touched bitmap + one dummy word per lane (the target
// of lanes without a feature)
__host__ __device__ inline size_t seq_table_bytes(uint32_t dim) {
  return (size_t)dim * 2 + (size_t)dim / 8 + 128;
}

__host__ inline bool use_seq(const FeatConfig& c) {
  return c.default_orders && c.pow2 && c.dim >= kSeqMinDim && c.dim <= kSeqMaxDim;
}

// 4 bytes at aligned position r of the aligned base a0; the prompt occupies
// [lo, hi), bytes outside it read as ' '.
// The 4 bytes at a0 + r (4-aligned) with those outside the prompt [lo, hi)
// read as spaces. A word straddling a prompt edge is still one aligned load
// when it lies inside the buffer's readable range [rlo, rhi); only a word
// crossing the buffer's own ends is assembled byte by byte.
__device__ __forceinline__ uint32_t seq_word(const uint8_t* a0, int r, int lo, int hi, int rlo,
                                             int rhi) {
  if (r >= lo && r + 4 <= hi) return __ldg(reinterpret_cast<const uint32_t*>(a0 + r));
  if (r + 4 <= lo || r >= hi) return 0x20202020u;
  if (r >= rlo && r + 4 <= rhi) {
    const uint32_t w = __ldg(reinterpret_cast<const uint32_t*>(a0 + r));
    const int k0 = lo > r ? lo - r : 0, k1 = hi - r < 4 ? hi - r : 4;  // valid bytes [k0, k1)
    const uint32_t keep = (k1 >= 4 ? 0xffffffffu : ((1u << (8 * k1)) - 1u)) & ~((1u << (8 * k0)) - 1u);
    return (w & keep) | (0x20202020u & ~keep);
  }
  uint32_t w = 0x20202020u;
#pragma unroll
  for (int k = 0; k < 4; ++k)
    if (r + k >= lo && r + k < hi) w = (w & ~(0xffu << (8 * k))) | ((uint32_t)a0[r + k] << (8 * k));
  return w;
}

// One feature into the per-warp table, branch-free: +-1 into the bucket's
// biased 16-bit half (idx = (e >> 1) & mask, sign = e & 1, features.cpp:29-34)
// and its touched bit, both fire-and-forget `red` operations. A lane without
// a feature targets its own dummy word instead (bank = lane, never read), so
// it neither branches nor adds bank conflicts.
__device__ __forceinline__ void seq_emit(uint32_t cbase, uint32_t bbase, uint32_t dummy, uint32_t e,
                                         uint32_t m1, uint32_t m2, bool p) {
  const uint32_t caddr = p ? cbase + (e & m1) : dummy;
  const uint32_t d = ((e & 1u) * 2u - 1u) << ((e << 3) & 16u);  // +-1 in the bucket's half
  const uint32_t baddr = p ? bbase + ((e >> 4) & m2) : dummy;
  const uint32_t bit = 1u << ((e >> 1) & 31u);
  asm volatile("red.shared.add.u32 [%0], %1;\n\tred.shared.or.b32 [%2], %3;" ::"r"(caddr), "r"(d),
               "r"(baddr), "r"(bit)
               : "memory");
}

__device__ __forceinline__ void hash_prompt_seq(const FeatConfig& c, const WarpSmem& S,
                                                const uint8_t* base, int len, int lane,
                                                const uint8_t* buf_lo, const uint8_t* buf_hi) {
  if (len <= 0) return;
  const int mis = (int)(reinterpret_cast<uintptr_t>(base) & 3u);
  const uint8_t* a0 = base - mis;
  const int lo = mis, hi = mis + len;
  // the buffer's readable bytes relative to a0 (clamped to this prompt's
  // neighbourhood; the text of all prompts of the launch is readable)
  const int64_t dlo = buf_lo - a0, dhi = buf_hi - a0;
  const int rlo = dlo > 0 ? (int)dlo : 0;
  const int rhi = dhi < (int64_t)hi + 8 ? (int)dhi : hi + 8;
  const int wpl = (((hi + 3) >> 2) + 31) >> 5;  // words per lane
  const int cs = lane * wpl * 4, ce = cs + wpl * 4;
  if (cs >= hi) return;
  const uint32_t sw = (uint32_t)c.word_salt[0], sc = (uint32_t)c.char_salt[0];
  const uint32_t cbase = (uint32_t)__cvta_generic_to_shared(S.counts);
  const uint32_t bbase = (uint32_t)__cvta_generic_to_shared(S.bitmap);
  const uint32_t dummy = bbase + (c.dim / 8) + 4u * lane;
  const uint32_t m1 = (c.dim / 2 - 1) << 2, m2 = (c.dim / 32 - 1) << 2;
  uint32_t prev2 = cs > 0 ? nonspace_nibble(seq_word(a0, cs - 4, lo, hi, rlo, rhi)) >> 2 : 0u;
  uint32_t hw = sw, A = 0, B = 0, carry = 0;
  // two words (8 bytes) per iteration: the mask logic runs once per 8 bytes
  uint32_t w0 = seq_word(a0, cs, lo, hi, rlo, rhi), w1 = seq_word(a0, cs + 4, lo, hi, rlo, rhi);
  for (int r = cs;; r += 8) {
    const uint32_t n0 = seq_word(a0, r + 8, lo, hi, rlo, rhi), n1 = seq_word(a0, r + 12, lo, hi, rlo, rhi);
    const uint32_t ns = nonspace_nibble(w0) | (nonspace_nibble(w1) << 4);
    const uint32_t E = (ns << 2) | prev2;  // bit k+2: byte r+k is not a space
    const uint32_t start = ns & ~(E >> 1);
    // tokens may start only inside [cs, ce): the second word can lie beyond ce
    const uint32_t inr = r < ce ? (r + 4 < ce ? 0xffu : 0x0fu) : 0u;
    const uint32_t own = (ns + ((start & inr) | carry)) ^ ns;
    carry = own >> 8;
    const uint32_t ev_tri = ns & (E >> 1) & E & own;
    const uint32_t ev = ev_tri | (~ns & (E >> 1) & own & 0xffu);
#pragma unroll
    for (int k = 0; k < 8; ++k) {
      const uint32_t b = ((k < 4 ? w0 : w1) >> (8 * (k & 3))) & 0xffu;
      const uint32_t hin = ((start >> k) & 1u) ? sw : hw;
      const uint32_t wend = (hw ^ 0x1fu) * 0x1b3u;  // the word that ends at this space
      const uint32_t tri = (B ^ b) * 0x1b3u;
      B = (A ^ b) * 0x1b3u;
      A = (sc ^ b) * 0x1b3u;
      hw = (hin ^ b) * 0x1b3u;
      seq_emit(cbase, bbase, dummy, ((ev_tri >> k) & 1u) ? tri : wend, m1, m2, ((ev >> k) & 1u) != 0);
    }
    prev2 = ns >> 6;
    if (!carry && (r + 8 >= ce || r + 8 >= hi)) break;
    w0 = n0;
    w1 = n1;
  }
}

// Lane l owns buckets [l*dim/32, (l+1)*dim/32): bitmap words [l*nb, (l+1)*nb).
template <int MODE>
__global__ void __launch_bounds__(256) featurize_seq_kernel(const FeatConfig c, const FeatArgs a) {
  extern __shared__ __align__(16) unsigned char smem[];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int64_t gw = (int64_t)blockIdx.x * (blockDim.x >> 5) + warp;
  const int64_t nw = (int64_t)gridDim.x * (blockDim.x >> 5);
  WarpSmem S;
  S.counts = reinterpret_cast<uint32_t*>(smem + seq_table_bytes(c.dim) * warp);
  S.bitmap = S.counts + c.dim / 2;
  S.ring = nullptr;
  for (uint32_t k = lane; k < c.dim / 2; k += 32) S.counts[k] = kBias2;
  for (uint32_t k = lane; k < c.dim / 32; k += 32) S.bitmap[k] = 0u;
  __syncwarp();
  const uint32_t nb = c.dim >> 10;
  uint32_t* bm = S.bitmap + lane * nb;
  uint16_t* c16 = reinterpret_cast<uint16_t*>(S.counts);

  uint32_t* lists = (MODE == kFeatScoreExact) ? a.lists + (size_t)gw * a.list_cap : nullptr;
  // readable text of this launch: the bytes of its prompts, offsets[0] .. offsets[n]
  const uint8_t* text_lo = a.text + a.offsets[0];
  const uint8_t* text_hi = a.text + a.offsets[a.n];
  int gn = 0;
  uint32_t used = 0;
  int64_t g_prompt = 0;
  uint32_t g_off = 0, g_cnt = 0;
  double g_inv = 1.0;

  for (int64_t i = gw; i < a.n; i += nw) {
    const int64_t beg = a.offsets[i], len = a.offsets[i + 1] - beg;
    if (((len + 1) / 2) + len > kNarrowMaxFeatures) {  // 16-bit counters could wrap
      if (lane == 0) a.long_list[atomicAdd(a.long_count, 1)] = (int32_t)i;
      continue;
    }
    {
      // the warp's next prompt into L2, so the lanes' sequential word loads
      // do not each expose a DRAM miss (an L1 prefetch of the current prompt
      // measured slower: with 3 x 70 KB of shared memory per SM, L1 keeps
      // less than one prompt per warp)
      if (i + nw < a.n) {
        const int64_t nb = a.offsets[i + nw], ne = a.offsets[i + nw + 1];
        const uintptr_t n0 = reinterpret_cast<uintptr_t>(a.text + nb) & ~(uintptr_t)127;
        for (uintptr_t q = n0 + 128u * lane; q < reinterpret_cast<uintptr_t>(a.text + ne); q += 4096u)
          asm volatile("prefetch.global.L2 [%0];" ::"l"(q));
      }
    }
    hash_prompt_seq(c, S, a.text + beg, (int)len, lane, text_lo, text_hi);
    __syncwarp();
    // pass 1: this lane's entry count (CSR: non-zero counts, and sum(count^2))
    uint32_t mine = 0;
    long long sq = 0;
    for (uint32_t j = 0; j < nb; ++j) {
      const uint32_t m = bm[j];
      if (MODE == kFeatCsr) {
        for (uint32_t t = m; t; t &= t - 1) {
          const int cnt = (int)c16[(lane * nb + j) * 32 + __ffs(t) - 1] - 0x8000;
          mine += cnt != 0;
          sq += (long long)cnt * cnt;
        }
      } else {
        mine += __popc(m);
      }
    }
    int tot;
    const uint32_t off = (uint32_t)warp_excl_scan((int)mine, lane, &tot);
    double inv = 1.0;
    if (MODE == kFeatCsr) inv = inv_norm(c, warp_sum_i64(sq));
    uint32_t* L = nullptr;
    if (MODE == kFeatScoreExact) {
      const uint32_t need = ((uint32_t)tot + 3u) & ~3u;
      if (gn == kGroup || used + need > a.list_cap) {
        chain_group(c, a, lists, true, lane, gn, g_prompt, g_off, g_cnt, g_inv);
        gn = 0;
        used = 0;
      }
      L = lists + used;
    }
    const int64_t slot = (MODE == kFeatCsr) ? a.slot_base[i] : 0;
    // pass 2: ascending entries (lane-major = bucket order); resets the table
    uint32_t pos = off;
    float facc = 0.f;
    for (uint32_t j = 0; j < nb; ++j) {
      const uint32_t m = bm[j];
      if (!m) continue;
      bm[j] = 0u;
      const uint32_t b0 = (lane * nb + j) * 32;
      for (uint32_t t = m; t; t &= t - 1) {
        const uint32_t idx = b0 + __ffs(t) - 1;
        const int cnt = (int)c16[idx] - 0x8000;
        c16[idx] = 0x8000;
        if (MODE == kFeatScoreExact) {
          L[pos++] = (idx << 16) | (uint32_t)(cnt + 0x8000);
          sq += (long long)cnt * cnt;
        } else if (MODE == kFeatScoreFast) {
          facc += __ldg(a.w32 + idx) * (float)cnt;
          sq += (long long)cnt * cnt;
        } else if (cnt != 0) {
          a.out_idx[slot + pos] = idx;
          a.out_val[slot + pos] = c.norm ? __dmul_rn((double)cnt, inv) : (double)cnt;
          if (a.out_cnt) a.out_cnt[slot + pos] = cnt;
          ++pos;
        }
      }
    }
    if (MODE == kFeatScoreExact) {
      inv = inv_norm(c, warp_sum_i64(sq));
      if (lane == gn) {
        g_prompt = i;
        g_off = used;
        g_cnt = (uint32_t)tot;
        g_inv = inv;
      }
      ++gn;
      used += ((uint32_t)tot + 3u) & ~3u;
    } else if (MODE == kFeatScoreFast) {
      facc = warp_sum_f32(facc);
      const float finv = (float)inv_norm(c, warp_sum_i64(sq));
      if (lane == 0) a.scores[i] = (double)(facc * finv) + a.bias;
    } else if (lane == 0) {
      a.out_nnz[i] = tot;
      if (a.out_inv) a.out_inv[i] = inv;
    }
    __syncwarp();
  }
  if (MODE == kFeatScoreExact && gn > 0)
    chain_group(c, a, lists, true, lane, gn, g_prompt, g_off, g_cnt, g_inv);
}

// ---- lane-range front end, v2 (score modes; word {1} + char {3}, pow2 dims) ----
//
// Same per-lane decomposition as featurize_seq_kernel (lane l owns the
// tokens that start in its word-aligned byte range and runs the reference's
// per-byte loop over them, features.cpp:80-101), restructured for fewer
// instructions per byte and for shared-memory text:
//   * the prompt is staged into a per-warp shared buffer by cp.async (16-byte
//     copies, L2 evict-first policy: the text streams through L2 once) while
//     the previous prompt is walked and scored, and the buffer's bytes
//     outside the prompt are overwritten with spaces, so the byte loop has
//     no edge logic and reads 4 bytes per LDS (stride-wpl words per lane,
//     no L1 tag traffic);
//   * spaces are rewritten to 0x1f ('\x1f', the word separator the reference
//     hashes after every word token) in the loaded word, so one expression
//     gives both features a byte can emit: e = ((space ? hw : B) ^ b') * P is
//     the trigram ending at a token byte and the word that ends at a space;
//   * emission is predicated (no dummy target): the counter word address is
//     one OR into the table (tables aligned to their size), the bitmap bit
//     one funnel shift;
// Prompts that do not fit the buffer run the same loop on global loads.
constexpr int kLaneTextCap = 2560;   // prompt bytes staged in shared memory per warp
constexpr int kLaneBuf = kLaneTextCap + 64;  // + 16-byte alignment slack and space padding

__host__ __device__ inline size_t lane_warp_bytes(uint32_t dim) {
  return (size_t)dim * 2 + dim / 8 + 48 /* increment table + staging mbarrier */ + kLaneBuf;
}
// + (fast mode) the fp32 weights in shared memory: the walk gathers w[idx]
// for every entry, and an L2 round trip per gather would serialise it
__host__ inline size_t lane_cta_bytes(uint32_t dim, int warps, int mode) {
  return (size_t)dim * 2 /* alignment slack */ + (size_t)warps * lane_warp_bytes(dim) +
         (mode == 1 ? (size_t)dim * 4 : 0);
}

__device__ __forceinline__ uint32_t lds32(uint32_t a) {
  uint32_t v;
  asm volatile("ld.shared.u32 %0, [%1];" : "=r"(v) : "r"(a));
  return v;
}

// SWAR: 0x80 in every byte of w that is not C-locale whitespace.
__device__ __forceinline__ uint32_t nonspace_hi(uint32_t w) {
  const uint32_t x = w ^ 0x20202020u;
  const uint32_t not_blank = ((x & 0x7f7f7f7fu) + 0x7f7f7f7fu) | x;
  const uint32_t lo7 = w & 0x7f7f7f7fu;
  const uint32_t ctl = (0x8d8d8d8du - lo7) & ~w & (lo7 + 0x77777777u);
  return not_blank & ~ctl & 0x80808080u;
}
__device__ __forceinline__ uint32_t hi_to_nibble(uint32_t h) { return ((h >> 7) * 0x01020408u) >> 24; }
// w with every whitespace byte replaced by 0x1f
__device__ __forceinline__ uint32_t spaces_to_sep(uint32_t w, uint32_t nsh) {
  const uint32_t m = (nsh << 1) - (nsh >> 7);  // 0xff in non-space bytes
  return (w & m) | (0x1f1f1f1fu & ~m);
}

// One feature e (idx = (e >> 1) & mask, sign = e & 1; features.cpp:29-34):
// +-1 into the bucket's biased 16-bit half and its touched bit, both as
// fire-and-forget `red` operations; when ev == 0 both target the lane's own
// dummy word (never read), so there is no branch (ptxas turns predicated
// shared-memory reductions into branches). Right shifts are IMAD.HI and the
// +-1 << (16 * half) product an IMAD, keeping the ALU pipe for the rest.
// One feature e = z * P (idx = (e >> 1) & mask, sign = e & 1;
// features.cpp:29-34): +-1 into the bucket's biased 16-bit half and its
// touched bit, as two fire-and-forget `red` operations issued by every lane
// (ptxas turns predicated shared-memory reductions into branches). A lane
// without a feature at this byte (ev bit clear) adds 0 and ORs 0: the
// increment comes from an 8-entry shared table indexed by (ev bit, e & 3)
// = {0, 0, 0, 0, -1, +1, -1 << 16, +1 << 16} and the bit is ev << bucket.
// Bit extraction and right shifts are multiplies (IMAD / IMAD.HI on the FMA
// pipe), leaving the ALU pipe the xors, selects and address masks.
template <int K>
__device__ __forceinline__ void lane_emit(uint32_t lut, uint32_t cbase, uint32_t bbase,
                                          uint32_t m1, uint32_t m2, uint32_t z, uint32_t ev) {
  asm volatile(
      "{\n\t.reg .u32 t, e, ca, ba, e1, e4, d, bt, k, la;\n\t"
      "mul.lo.u32 k, %5, %6;\n\tmul.hi.u32 k, k, 2;\n\t"          // k = (ev >> K) & 1
      "mul.lo.u32 e, %0, 435;\n\t"                                  // e = z * P
      "mul.lo.u32 t, %0, -1073741824;\n\tmul.hi.u32 t, t, 16;\n\t"  // 4 * (e & 3): (z * (P << 30)) = (e & 3) << 30
      "mad.lo.u32 la, k, 16, %7;\n\tadd.u32 la, la, t;\n\t"
      "ld.shared.u32 d, [la];\n\t"
      "and.b32 t, e, %3;\n\tor.b32 ca, t, %1;\n\t"
      "mul.hi.u32 e1, e, -2147483648;\n\tmul.hi.u32 e4, e, 268435456;\n\t"
      "and.b32 t, e4, %4;\n\tor.b32 ba, t, %2;\n\t"
      "shf.l.wrap.b32 bt, k, k, e1;\n\t"
      "red.shared.add.u32 [ca], d;\n\tred.shared.or.b32 [ba], bt;\n\t}" ::"r"(z),
      "r"(cbase), "r"(bbase), "r"(m1), "r"(m2), "r"(ev), "n"(1u << (31 - K)), "r"(lut));
}

// Byte K of an 8-byte step: the rolling char states A (one byte), B (two
// bytes), the word state hw (reset to the salt at spaces), and the feature
// that ends at this byte (features.cpp:84-90, :96-99).
template <int K>
__device__ __forceinline__ void lane_bytes(uint32_t p, uint32_t ns, uint32_t ev, uint32_t sw,
                                           uint32_t sc, uint32_t& hw, uint32_t& A, uint32_t& B,
                                           uint32_t cbase, uint32_t bbase, uint32_t m1, uint32_t m2,
                                           uint32_t lut) {
  const uint32_t b = __byte_perm(p, 0u, 0x4440u + (K & 3));
  const bool sp = ((ns >> K) & 1u) == 0u;
  const uint32_t An = (sc ^ b) * 0x1b3u;
  const uint32_t Bn = (A ^ b) * 0x1b3u;
  const uint32_t z = (sp ? hw : B) ^ b;  // the feature ending here: e = z * P
  hw = sp ? sw : (hw ^ b) * 0x1b3u;
  A = An;
  B = Bn;
  lane_emit<K>(lut, cbase, bbase, m1, m2, z, ev);
}

// The byte loop over lane l's range of a prompt occupying [lo, hi) of a
// space-padded source: SMEM reads the staged buffer at shared address src;
// otherwise 4-byte global words through seq_word (edges assembled there).
template <bool SMEM>
__device__ __forceinline__ void hash_lane(const FeatConfig& c, uint32_t src, const uint8_t* a0,
                                          int lo, int hi, int rlo, int rhi, int lane, uint32_t cbase,
                                          uint32_t bbase, uint32_t lut) {
  const int wpl = (((hi + 3) >> 2) + 31) >> 5;  // words per lane
  const int cs = lane * wpl * 4, ce = cs + wpl * 4;
  if (cs >= hi) return;
  auto word = [&](int r) -> uint32_t {
    if (SMEM) return lds32(src + (uint32_t)r);
    return seq_word(a0, r, lo, hi, rlo, rhi);
  };
  const uint32_t sw = (uint32_t)c.word_salt[0], sc = (uint32_t)c.char_salt[0];
  const uint32_t m1 = (c.dim / 2 - 1) << 2, m2 = (c.dim / 32 - 1) << 2;
  uint32_t prev2 = cs > 0 ? hi_to_nibble(nonspace_hi(word(cs - 4))) >> 2 : 0u;
  uint32_t hw = sw, A = 0, B = 0, carry = 0;
  uint32_t w0 = word(cs), w1 = word(cs + 4);
  for (int r = cs;; r += 8) {
    const uint32_t n0 = word(r + 8), n1 = word(r + 12);
    const uint32_t h0 = nonspace_hi(w0), h1 = nonspace_hi(w1);
    const uint32_t ns = hi_to_nibble(h0) | (hi_to_nibble(h1) << 4);
    const uint32_t E = (ns << 2) | prev2;  // bit k+2: byte r+k is not a space
    const uint32_t start = ns & ~(E >> 1);
    // tokens may start only inside [cs, ce): the second word can lie beyond ce
    const uint32_t inr = r < ce ? (r + 4 < ce ? 0xffu : 0x0fu) : 0u;
    const uint32_t own = (ns + ((start & inr) | carry)) ^ ns;
    carry = own >> 8;
    const uint32_t ev = ((ns & E) | ~ns) & (E >> 1) & own & 0xffu;  // trigram or word end
    const uint32_t p0 = spaces_to_sep(w0, h0), p1 = spaces_to_sep(w1, h1);
    lane_bytes<0>(p0, ns, ev, sw, sc, hw, A, B, cbase, bbase, m1, m2, lut);
    lane_bytes<1>(p0, ns, ev, sw, sc, hw, A, B, cbase, bbase, m1, m2, lut);
    lane_bytes<2>(p0, ns, ev, sw, sc, hw, A, B, cbase, bbase, m1, m2, lut);
    lane_bytes<3>(p0, ns, ev, sw, sc, hw, A, B, cbase, bbase, m1, m2, lut);
    lane_bytes<4>(p1, ns, ev, sw, sc, hw, A, B, cbase, bbase, m1, m2, lut);
    lane_bytes<5>(p1, ns, ev, sw, sc, hw, A, B, cbase, bbase, m1, m2, lut);
    lane_bytes<6>(p1, ns, ev, sw, sc, hw, A, B, cbase, bbase, m1, m2, lut);
    lane_bytes<7>(p1, ns, ev, sw, sc, hw, A, B, cbase, bbase, m1, m2, lut);
    prev2 = ns >> 6;
    if (!carry && (r + 8 >= ce || r + 8 >= hi)) break;
    w0 = n0;
    w1 = n1;
  }
}

// Stage text[beg, end) into the warp's buffer (shared address buf): the
// 16-byte-aligned chunks covering it, by cp.async with zero fill past the
// launch's readable text; returns the prompt's offset lo inside the buffer.
__device__ __forceinline__ int lane_stage(uint32_t buf, const uint8_t* text, int64_t beg, int64_t end,
                                          const uint8_t* rlo, const uint8_t* rhi, int lane,
                                          uint64_t pol) {
  const uint8_t* p0 = text + beg;
  const uint8_t* a0 = reinterpret_cast<const uint8_t*>(reinterpret_cast<uintptr_t>(p0) & ~(uintptr_t)15);
  const int lo = (int)(p0 - a0);
  const int nch = (lo + (int)(end - beg) + 15) >> 4;
  for (int k = lane; k < nch; k += 32) {
    const uint8_t* s = a0 + 16 * k;
    const uint32_t d = buf + 16u * (uint32_t)k;
    if (s < rlo) {  // chunk starts before the readable text: bytes one by one
      for (int j = 0; j < 16; ++j) {
        const uint32_t v = (s + j >= rlo && s + j < rhi) ? (uint32_t)s[j] : 0x20u;
        asm volatile("st.shared.u8 [%0], %1;" ::"r"(d + j), "r"(v));
      }
    } else {
      const int64_t avail = rhi - s;
      const uint32_t sz = avail >= 16 ? 16u : (uint32_t)avail;
      asm volatile("cp.async.cg.shared.global.L2::cache_hint [%0], [%1], 16, %2, %3;" ::"r"(d),
                   "l"(s), "r"(sz), "l"(pol));
    }
  }
  asm volatile("cp.async.commit_group;");
  return lo;
}

// The same staging as one TMA bulk copy of the 16-byte-aligned chunks
// covering the prompt (lane 0 issues it; completion on the warp's mbarrier),
// when those chunks lie inside the launch's readable text; otherwise the
// per-lane cp.async form above. Returns the prompt's offset in the buffer.
__device__ __forceinline__ int lane_stage_bulk(uint32_t buf, const uint8_t* text, int64_t beg, int64_t end,
                                               const uint8_t* rlo, const uint8_t* rhi, int lane,
                                               uint64_t pol, uint32_t bar, bool& bulk) {
  const uint8_t* p0 = text + beg;
  const uint8_t* a0 = reinterpret_cast<const uint8_t*>(reinterpret_cast<uintptr_t>(p0) & ~(uintptr_t)15);
  const int lo = (int)(p0 - a0);
  const uint32_t nbytes = ((uint32_t)(lo + (end - beg)) + 15u) & ~15u;
  bulk = a0 >= rlo && a0 + nbytes <= rhi && nbytes > 0;
  if (!bulk) return lane_stage(buf, text, beg, end, rlo, rhi, lane, pol);
  if (lane == 0) {
    // the buffer's previous prompt was read through the generic proxy
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(nbytes) : "memory");
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], "
        "%4;" ::"r"(buf),
        "l"(a0), "r"(nbytes), "r"(bar), "l"(pol)
        : "memory");
  }
  return lo;
}

// Wait for a bulk-staged prompt (every lane waits on the phase) and pad it.
__device__ __forceinline__ void lane_stage_finish_bulk(uint32_t buf, int lo, int hi, int lane, uint32_t bar,
                                                       uint32_t& phase) {
  asm volatile(
      "{\n\t.reg .pred p;\n\tLSTAGE_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t@!p bra LSTAGE_%=;\n\t}" ::"r"(bar),
      "r"(phase)
      : "memory");
  phase ^= 1u;
  __syncwarp();
  if (lane < lo) asm volatile("st.shared.u8 [%0], %1;" ::"r"(buf + lane), "r"(0x20u));
  asm volatile("st.shared.u8 [%0], %1;" ::"r"(buf + hi + lane), "r"(0x20u));
  __syncwarp();
}

// Wait for the staged prompt and pad it with spaces: [0, lo) and [hi, hi+32).
__device__ __forceinline__ void lane_stage_finish(uint32_t buf, int lo, int hi, int lane) {
  asm volatile("cp.async.wait_all;" ::: "memory");
  __syncwarp();  // every lane's copies have landed before the padding is written
  if (lane < lo) asm volatile("st.shared.u8 [%0], %1;" ::"r"(buf + lane), "r"(0x20u));
  asm volatile("st.shared.u8 [%0], %1;" ::"r"(buf + hi + lane), "r"(0x20u));
  __syncwarp();
}

// Exact mode: a prompt whose (idx, count) list fits kSlotCap entries writes
// it to its own slot (plus its entry count and L2 factor) for
// chain_slots_kernel; a longer list is chained by the hashing warp itself.
constexpr uint32_t kSlotCap = 512;

__host__ inline size_t lane_slot_bytes(int64_t n) {
  return (size_t)n * kSlotCap * 4 + (size_t)n * 8 + (size_t)n * 4 + 256;
}

// Exact mode, fused (default): the CTA is kFuseH hashing warps plus kFuseC
// chain warps. A hashing warp walks each prompt's touched buckets in
// ascending order into a ring slot (kFuseD slots of kRingCap entries per
// hashing warp, in global memory; for C4 the written part stays L2-resident:
// 148 x 18 x 8 x ~1.2 KB) and publishes it through a shared-memory sequence
// counter; the chain warp runs the sequential fp64 dots of 32 prompts at a
// time, one per lane, with the weights read through L1, and hands the slots
// back. The counters and the slot metadata are shared-memory atomics
// (ordered by __threadfence_block). The (idx, count) lists never travel to
// DRAM and no second kernel runs.
#ifndef PARS_FUSE_H
#define PARS_FUSE_H 18
#endif
#ifndef PARS_FUSE_D
#define PARS_FUSE_D 8
#endif
#ifndef PARS_FUSE_C
#define PARS_FUSE_C 2
#endif
constexpr int kFuseH = PARS_FUSE_H;  // hashing warps per CTA
constexpr int kFuseD = PARS_FUSE_D;  // ring slots per hashing warp
constexpr int kFuseC = PARS_FUSE_C;  // chain warps (round-robin over 32-item rounds)
// Ring slot capacity (entries): a prompt with more touched buckets is chained
// by its hashing warp itself (one lane). 2,048 covers the C4 hard variant
// (random 6-letter words: ~1,520 touched buckets, at most ~1,690); only the
// entries written are touched, so the slot stride costs no L2 for short
// lists (148 CTAs x 18 warps x 8 slots x 8 KB = 170 MB of scratch).
constexpr uint32_t kRingCap = 2048;
#ifndef PARS_FUSE_SPIN_NS
#define PARS_FUSE_SPIN_NS 32  // back-off of a hashing warp waiting for its ring slot
#endif
#ifndef PARS_FUSE_WSMEM
#define PARS_FUSE_WSMEM 0
#endif
constexpr bool kFuseWSmem = PARS_FUSE_WSMEM;  // fp64 weights in shared memory (else through L1)
struct FuseMeta {
  double inv;
  int64_t prompt;
  int32_t nnz;  // entries in the slot; -1: nothing to chain (scored elsewhere)
  int32_t pad;
};
__host__ inline size_t fused_cta_bytes(uint32_t dim) {
  return (size_t)dim * 2 /* table alignment slack */ + (size_t)kFuseH * lane_warp_bytes(dim) +
         (kFuseWSmem ? (size_t)dim * 8 : 0) + (size_t)kFuseH * kFuseD * sizeof(FuseMeta) +
         (kFuseH + kFuseH * kFuseD) * sizeof(int) + 64;
}
__host__ inline size_t fused_ring_bytes(int64_t grid) {
  return (size_t)grid * kFuseH * kFuseD * kRingCap * 4;
}

// Products of one 4-entry chunk (entries past the list's end give +0.0,
// which leaves a sum that started at +0.0 unchanged under round-to-nearest).
__device__ __forceinline__ void chain_products(const FeatConfig& c, const double* sw, uint4 q4,
                                               int lim, double inv, double p[4]) {
  const uint32_t ev[4] = {q4.x, q4.y, q4.z, q4.w};
#pragma unroll
  for (int t = 0; t < 4; ++t) {
    // the biased 16-bit count as a double without an I2F.F64 (a slow pipe):
    // the bits of 2^52 + (cnt + 2^15), less 2^52 + 2^15, exactly, in one DADD
    const uint32_t cb = ev[t] & 0xffffu;
    const double cd = __dsub_rn(__hiloint2double(0x43300000, (int)cb), 4503599627403264.0);
    const double v = c.norm ? __dmul_rn(cd, inv) : cd;
    const double pr = __dmul_rn(sw[(ev[t] >> 16) & c.mask], v);
    p[t] = (t < lim && cb != 0x8000u) ? pr : 0.0;
  }
}

// A chain warp: 32 prompts' sequential dots per round (features.hpp:31-35,
// scorer.cpp:40-42). Round b covers items [32b, 32b + 32) of the sequence
// (generation t, hashing warp h), item = t * kFuseH + h; chain warp cw takes
// rounds cw, cw + kFuseC, ...
__device__ __forceinline__ void fused_chain_warp(const FeatConfig& c, const FeatArgs& a,
                                                 const double* sw, const FuseMeta* meta,
                                                 volatile int* produced, volatile int* free_gen,
                                                 const uint32_t* ring, int64_t nw, int lane, int cw) {
  const int64_t rem0 = a.n - a.first - (int64_t)blockIdx.x * kFuseH;
  const int cnt0 = rem0 > 0 ? (int)((rem0 + nw - 1) / nw) : 0;  // warp 0 has the most prompts
  const int items = cnt0 * kFuseH;
  for (int b = cw; b * 32 < items; b += kFuseC) {
    const int j = b * 32 + lane;
    const int t = j / kFuseH, h = j - t * kFuseH;
    const int64_t rem = a.n - a.first - ((int64_t)blockIdx.x * kFuseH + h);
    const bool valid = j < items && (int64_t)t * nw < rem;
    if (valid)
      while (atomicAdd(const_cast<int*>(&produced[h]), 0) <= t) __nanosleep(64);
    __syncwarp();
    __threadfence_block();
    int m = -1;
    double inv = 1.0;
    int64_t prompt = 0;
    const int slot = t % kFuseD;
    if (valid) {
      const FuseMeta& f = meta[h * kFuseD + slot];
      // hand-off fields read as atomics (ordered by the fences around the
      // sequence counters; atomic so the sanitizer sees no plain race)
      FuseMeta& fm = const_cast<FuseMeta&>(f);
      m = atomicAdd(&fm.nnz, 0);
      inv = __longlong_as_double(
          (long long)atomicAdd(reinterpret_cast<unsigned long long*>(&fm.inv), 0ull));
      prompt = (int64_t)atomicAdd(reinterpret_cast<unsigned long long*>(&fm.prompt), 0ull);
    }
    const uint4* L = reinterpret_cast<const uint4*>(ring + ((size_t)h * kFuseD + slot) * kRingCap);
    const int nq = m > 0 ? (m + 3) >> 2 : 0;
    // software pipeline as in chain_slots_thread_kernel; loads bypass L1 (the
    // slot was rewritten by another warp since this SM last read it)
    constexpr int kAhead = 8;
    const uint4 z4 = make_uint4(0u, 0u, 0u, 0u);
    uint4 r[kAhead];
#pragma unroll
    for (int j = 0; j < kAhead; ++j) r[j] = j < nq ? __ldcg(L + j) : z4;
    double pa[4];
    chain_products(c, sw, r[0], m, inv, pa);
    double s = 0.0;
    for (int q0 = 0; q0 < nq; q0 += kAhead) {
#pragma unroll
      for (int j = 0; j < kAhead; ++j) {
        const int q = q0 + j;
        if (q < nq) {
          r[j] = q + kAhead < nq ? __ldcg(L + q + kAhead) : z4;
          double pb[4];
          chain_products(c, sw, r[(j + 1) % kAhead], m - 4 * (q + 1), inv, pb);
          s = __dadd_rn(s, pa[0]);
          s = __dadd_rn(s, pa[1]);
          s = __dadd_rn(s, pa[2]);
          s = __dadd_rn(s, pa[3]);
#pragma unroll
          for (int u = 0; u < 4; ++u) pa[u] = pb[u];
        }
      }
    }
    if (m >= 0) a.scores[prompt] = __dadd_rn(s, a.bias);
    __threadfence_block();
    __syncwarp();
    if (valid) atomicExch(const_cast<int*>(&free_gen[h * kFuseD + slot]), t + kFuseD);  // the slot's next writer
  }
}

template <int MODE, bool FUSED>
__global__ void __launch_bounds__(FUSED ? (kFuseH + kFuseC) * 32 : 576, 1)
    featurize_lane_kernel(const FeatConfig c, const FeatArgs a) {
  extern __shared__ __align__(16) unsigned char smem[];
  constexpr bool kChain = MODE == kFeatScoreExact;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int nwc = FUSED ? kFuseH : (int)(blockDim.x >> 5);  // hashing warps per CTA
  const int64_t gw = (int64_t)blockIdx.x * nwc + warp;
  const int64_t nw = (int64_t)gridDim.x * nwc;
  // tables aligned to their size, so a counter address is base | offset
  const uint32_t tsz = c.dim * 2;
  const uint32_t s0 = (uint32_t)__cvta_generic_to_shared(smem);
  const uint32_t tb = (s0 + tsz - 1) & ~(tsz - 1);
  // fast mode: the fp32 weights in shared memory after the warps' regions
  // (the walk gathers w[idx] per entry; an L2 round trip each would
  // serialise it)
  float* sw32 = reinterpret_cast<float*>(smem + (tb - s0) + (size_t)nwc * lane_warp_bytes(c.dim));
  if (!kChain) {
    for (uint32_t k = threadIdx.x; k < c.dim; k += blockDim.x) sw32[k] = a.w32[k];
    __syncthreads();
  }
  // fused exact mode: slot metadata and sequence counters (the chain warps
  // gather the fp64 weights through L1: 32 KB, the rest of the SM's
  // on-chip memory after the hashing warps' shared memory)
  double* sw64s = reinterpret_cast<double*>(sw32);
  const double* sw64 = kFuseWSmem ? sw64s : a.w64;
  FuseMeta* meta = reinterpret_cast<FuseMeta*>(sw32 + (kFuseWSmem ? 2 * c.dim : 0));
  volatile int* produced = reinterpret_cast<volatile int*>(meta + kFuseH * kFuseD);
  volatile int* free_gen = produced + kFuseH;  // [kFuseH][kFuseD]: generation allowed to write the slot
  uint32_t* ring = a.slots + (size_t)blockIdx.x * kFuseH * kFuseD * kRingCap;
  if (FUSED) {
    if (kFuseWSmem)
      for (uint32_t k = threadIdx.x; k < c.dim; k += blockDim.x) sw64s[k] = a.w64[k];
    if (threadIdx.x < kFuseH) produced[threadIdx.x] = 0;
    if (threadIdx.x < kFuseH * kFuseD) free_gen[threadIdx.x] = threadIdx.x % kFuseD;
    __syncthreads();
    if (warp >= kFuseH) {
      fused_chain_warp(c, a, sw64, meta, produced, free_gen, ring, (int64_t)gridDim.x * kFuseH, lane,
                       warp - kFuseH);
      return;
    }
  }
  int gen = 0;  // this warp's prompt count so far (its ring sequence number)
  // fused: wait until the chain warp has released slot gen % kFuseD
  auto wait_slot = [&]() {
    if (lane == 0)
      while (atomicAdd(const_cast<int*>(&free_gen[warp * kFuseD + gen % kFuseD]), 0) != gen)
        __nanosleep(PARS_FUSE_SPIN_NS);
    __syncwarp();
  };
  // fused: publish generation gen (its slot's entries written by the lanes)
  auto publish = [&](int nnz, double inv, int64_t prompt) {
    __threadfence_block();
    __syncwarp();
    if (lane == 0) {
      FuseMeta& f = meta[warp * kFuseD + gen % kFuseD];
      atomicExch(reinterpret_cast<unsigned long long*>(&f.inv), (unsigned long long)__double_as_longlong(inv));
      atomicExch(reinterpret_cast<unsigned long long*>(&f.prompt), (unsigned long long)prompt);
      atomicExch(&f.nnz, nnz);
      __threadfence_block();
      atomicExch(const_cast<int*>(&produced[warp]), gen + 1);
    }
    __syncwarp();
    ++gen;
  };
  const uint32_t cbase = tb + (uint32_t)warp * tsz;
  const uint32_t bbase = tb + (uint32_t)nwc * tsz + (uint32_t)warp * (c.dim / 8);
  // increments by (ev bit, half, sign): 0 x4, then -1, +1, -1 << 16, +1 << 16
  const uint32_t lut = tb + (uint32_t)nwc * (tsz + c.dim / 8) + (uint32_t)warp * 48u;
  const uint32_t sbar = lut + 32u;  // the warp's staging mbarrier
  const uint32_t buf = tb + (uint32_t)nwc * (tsz + c.dim / 8 + 48u) + (uint32_t)warp * kLaneBuf;
  if (lane == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(sbar));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  uint32_t sphase = 0;
  bool st_bulk = false;
  if (lane < 8) {
    const uint32_t dv =
        lane < 4 ? 0u : ((lane & 1) ? 1u : 0xffffffffu) << ((lane & 2) ? 16 : 0);
    asm volatile("st.shared.u32 [%0], %1;" ::"r"(lut + 4u * lane), "r"(dv));
  }
  uint32_t* counts = reinterpret_cast<uint32_t*>(smem + (cbase - s0));
  uint32_t* bitmap = reinterpret_cast<uint32_t*>(smem + (bbase - s0));
  for (uint32_t k = lane; k < c.dim / 2; k += 32) counts[k] = kBias2;
  for (uint32_t k = lane; k < c.dim / 32; k += 32) bitmap[k] = 0u;
  __syncwarp();
  const uint32_t nb = c.dim >> 10;
  uint32_t* bm = bitmap + lane * nb;
  uint16_t* c16 = reinterpret_cast<uint16_t*>(counts);
  uint64_t pol;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));

  uint32_t* lists = kChain ? a.lists + (size_t)gw * a.list_cap : nullptr;
  const uint8_t* text_lo = a.text + a.offsets[0];
  const uint8_t* text_hi = a.text + a.offsets[a.n];
  auto fits = [&](int64_t beg, int64_t len) {
    return (int64_t)(reinterpret_cast<uintptr_t>(a.text + beg) & 15u) + len + 32 <= kLaneBuf;
  };
  int st_lo = -1;  // buffer offset of the staged prompt (-1: nothing staged)
  if (a.first + gw < a.n) {
    const int64_t beg = a.offsets[a.first + gw], len = a.offsets[a.first + gw + 1] - beg;
    if (fits(beg, len))
      st_lo = lane_stage_bulk(buf, a.text, beg, beg + len, text_lo, text_hi, lane, pol, sbar, st_bulk);
  }
  for (int64_t i = a.first + gw; i < a.n; i += nw) {
    const int64_t beg = a.offsets[i], len = a.offsets[i + 1] - beg;
    if (((len + 1) / 2) + len > kNarrowMaxFeatures) {  // 16-bit counters could wrap
      if (lane == 0) a.long_list[atomicAdd(a.long_count, 1)] = (int32_t)i;
      st_lo = -1;
    } else if (st_lo >= 0) {
      if (st_bulk) lane_stage_finish_bulk(buf, st_lo, st_lo + (int)len, lane, sbar, sphase);
      else lane_stage_finish(buf, st_lo, st_lo + (int)len, lane);
      hash_lane<true>(c, buf, nullptr, st_lo, st_lo + (int)len, 0, 0, lane, cbase, bbase, lut);
    } else if (len > 0) {
      const uint8_t* base = a.text + beg;
      const int mis = (int)(reinterpret_cast<uintptr_t>(base) & 3u);
      const uint8_t* a0 = base - mis;
      const int lo = mis, hi = mis + (int)len;
      const int64_t dlo = text_lo - a0, dhi = text_hi - a0;
      const int rlo = dlo > 0 ? (int)dlo : 0;
      const int rhi = dhi < (int64_t)hi + 8 ? (int)dhi : hi + 8;
      hash_lane<false>(c, 0, a0, lo, hi, rlo, rhi, lane, cbase, bbase, lut);
    }
    __syncwarp();
    // the next prompt streams into the (now free) buffer while this one is
    // walked and scored
    st_lo = -1;
    if (i + nw < a.n) {
      const int64_t nb2 = a.offsets[i + nw], nl = a.offsets[i + nw + 1] - nb2;
      if (fits(nb2, nl))
        st_lo = lane_stage_bulk(buf, a.text, nb2, nb2 + nl, text_lo, text_hi, lane, pol, sbar, st_bulk);
    }
    if (((len + 1) / 2) + len > kNarrowMaxFeatures) {
      if (FUSED) {
        wait_slot();
        publish(-1, 1.0, i);
      }
      continue;
    }
    // pass 1: this lane's entries (bitmap popcount)
    uint32_t mine = 0;
    for (uint32_t j = 0; j < nb; ++j) mine += __popc(bm[j]);
    int tot;
    const uint32_t off = (uint32_t)warp_excl_scan((int)mine, lane, &tot);
    uint32_t sq = 0;  // sum of count^2 <= features^2 <= 32767^2: exact in 32 bits
    // exact: the prompt's own slot (fused: the warp's next ring slot), or
    // (long lists) the warp's arena
    const bool in_slot = kChain && (uint32_t)tot <= (FUSED ? kRingCap : kSlotCap);
    if (FUSED) wait_slot();
    uint32_t* L = !in_slot ? lists
                  : FUSED  ? ring + ((size_t)warp * kFuseD + gen % kFuseD) * kRingCap
                           : a.slots + (size_t)(i - a.first) * kSlotCap;
    // pass 2: ascending entries (lane-major = bucket order); resets the table
    uint32_t pos = off;
    float facc = 0.f;
    for (uint32_t j = 0; j < nb; ++j) {
      const uint32_t m = bm[j];
      if (!m) continue;
      bm[j] = 0u;
      const uint32_t b0 = (lane * nb + j) * 32;
      for (uint32_t t = m; t; t &= t - 1) {
        const uint32_t idx = b0 + __ffs(t) - 1;
        const int cnt = (int)c16[idx] - 0x8000;
        c16[idx] = 0x8000;
        sq += (uint32_t)(cnt * cnt);
        if (kChain) {
          L[pos++] = (idx << 16) | (uint32_t)(cnt + 0x8000);
        } else {
          facc += sw32[idx] * (float)cnt;
        }
      }
    }
    const double inv = inv_norm(c, (long long)__reduce_add_sync(kFull, sq));
    if (FUSED) {
      if (!in_slot) {
        __syncwarp();
        chain_group(c, a, lists, true, lane, 1, i, 0, (uint32_t)tot, inv);
      }
      publish(in_slot ? tot : -1, inv, i);
    } else if (kChain) {
      if (lane == 0) {
        a.slot_nnz[i - a.first] = in_slot ? tot : -1;
        a.slot_inv[i - a.first] = inv;
      }
      if (!in_slot) {
        __syncwarp();
        chain_group(c, a, lists, true, lane, 1, i, 0, (uint32_t)tot, inv);
      }
    } else {
      facc = warp_sum_f32(facc);
      if (lane == 0) a.scores[i] = (double)(facc * (float)inv) + a.bias;
    }
    __syncwarp();
  }
  asm volatile("cp.async.wait_all;" ::: "memory");
}

// Exact mode, second pass (features.hpp:31-35, scorer.cpp:40-42): thread k
// runs the sequential fp64 dot of the prompt in slot k — s = +0.0, then
// s += w[idx] * (count * inv) in ascending index order, then + bias — with
// 16-byte entry loads issued four ahead and the weights in shared memory.
// It runs right after the hashing kernel on the same chunk of prompts, so
// the slots it reads were written moments ago and are still in L2.
__global__ void __launch_bounds__(256) chain_slots_thread_kernel(const FeatConfig c, const FeatArgs a) {
  extern __shared__ __align__(16) unsigned char csm[];
  double* sw = reinterpret_cast<double*>(csm);
  for (uint32_t k = threadIdx.x; k < c.dim; k += blockDim.x) sw[k] = a.w64[k];
  __syncthreads();
  const int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;  // slot
  if (a.first + k >= a.n) return;
  const int64_t i = a.first + k;
  const int32_t m = a.slot_nnz[k];
  if (m < 0) return;  // chained by the hashing kernel
  const double inv = a.slot_inv[k];
  const uint4* L = reinterpret_cast<const uint4*>(a.slots + (size_t)k * kSlotCap);
  const int nq = (m + 3) >> 2;
  // software pipeline: chunk q's four adds (the only dependent chain) run
  // while chunk q+1's products are formed; entry loads run kAhead chunks
  // ahead (DRAM latency x bandwidth needs many bytes in flight per thread)
  constexpr int kAhead = 8;
  const uint4 z4 = make_uint4(0u, 0u, 0u, 0u);
  uint4 r[kAhead];
#pragma unroll
  for (int j = 0; j < kAhead; ++j) r[j] = j < nq ? __ldcs(L + j) : z4;
  double pa[4];
  chain_products(c, sw, r[0], m, inv, pa);
  double s = 0.0;
  for (int q0 = 0; q0 < nq; q0 += kAhead) {
#pragma unroll
    for (int j = 0; j < kAhead; ++j) {
      const int q = q0 + j;
      if (q < nq) {
        // chunk q's slot r[j] is done: refill it with chunk q + kAhead
        r[j] = q + kAhead < nq ? __ldcs(L + q + kAhead) : z4;
        double pb[4];
        chain_products(c, sw, r[(j + 1) % kAhead], m - 4 * (q + 1), inv, pb);
        s = __dadd_rn(s, pa[0]);
        s = __dadd_rn(s, pa[1]);
        s = __dadd_rn(s, pa[2]);
        s = __dadd_rn(s, pa[3]);
#pragma unroll
        for (int t = 0; t < 4; ++t) pa[t] = pb[t];
      }
    }
  }
  a.scores[i] = __dadd_rn(s, a.bias);
}

struct Plan {
  bool global_tables;
  int warps;
  int64_t grid;
  size_t smem;
};

template <bool POW2, bool WIDE, bool DEF, int MODE>
int plan_one(const FeatConfig& c, int64_t items, Plan* p) {
  const size_t per = warp_table_bytes(c, WIDE);
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  if (per > kMaxSmemPerBlock) {
    p->global_tables = true;
    p->warps = 4;
    p->grid = (int64_t)sms * 4;
    p->smem = 0;
    return PARS_OK;
  }
  p->global_tables = false;
  auto kern = featurize_kernel<POW2, WIDE, DEF, MODE, false>;
  // warps per CTA: the choice that keeps the most warps resident per SM
  // (the per-warp table makes shared memory the occupancy limiter)
  int warps = 1, per_sm = 1, best = 0;
  for (int w : {8, 4, 2, 1}) {
    if (WIDE && w != 1) continue;
    const size_t sm_bytes = per * w;
    if (sm_bytes > kMaxSmemPerBlock) continue;
    if (cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm_bytes) !=
        cudaSuccess)
      continue;
    int b = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&b, kern, w * 32, sm_bytes);
    if (b * w > best) {
      best = b * w;
      warps = w;
      per_sm = b;
    }
  }
  cudaGetLastError();
  if (best == 0) {
    set_error("featurize: no launchable configuration for dimension %u", c.dim);
    return PARS_ERR_UNSUPPORTED;
  }
  p->warps = warps;
  p->smem = per * warps;
  int64_t grid = std::min<int64_t>(ceil_div(std::max<int64_t>(items, 1), warps), (int64_t)sms * per_sm);
  if (WIDE) grid = (int64_t)sms * per_sm;  // count known only on device
  p->grid = std::max<int64_t>(grid, 1);
  return PARS_OK;
}

template <bool POW2, bool WIDE, bool DEF, int MODE>
int launch_one(pars_ctx* ctx, const FeatConfig& c, const FeatArgs& a, cudaStream_t st,
               int64_t items) {
  Plan p;
  PARS_TRY((plan_one<POW2, WIDE, DEF, MODE>(c, items, &p)));
  const size_t total_warps = (size_t)p.grid * p.warps;
  if (p.global_tables && a.gscratch_bytes < warp_table_bytes(c, WIDE) * total_warps) {
    set_error("featurize: global table scratch too small");
    return PARS_ERR_INVALID;
  }
  if (MODE == kFeatScoreExact && a.lists_bytes < (size_t)a.list_cap * 4 * total_warps) {
    set_error("featurize: list scratch too small");
    return PARS_ERR_INVALID;
  }
  if (p.global_tables) {
    featurize_kernel<POW2, WIDE, DEF, MODE, true><<<(unsigned)p.grid, p.warps * 32, 0, st>>>(c, a);
  } else {
    auto kern = featurize_kernel<POW2, WIDE, DEF, MODE, false>;
    PARS_CUDA_CHECK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)p.smem));
    kern<<<(unsigned)p.grid, p.warps * 32, p.smem, st>>>(c, a);
  }
  count_launch(ctx);
  PARS_CUDA_CHECK(cudaGetLastError());
  return PARS_OK;
}

// The score modes run the v2 lane kernel (featurize_lane_kernel) unless
// PARS_FEAT_V1=1 selects the round-1 kernel (kept for A/B measurements);
// CSR mode runs featurize_seq_kernel.
__host__ inline bool use_lane(int mode) {
  static const bool v1 = [] {
    const char* e = std::getenv("PARS_FEAT_V1");
    return e && e[0] == '1';
  }();
  return mode != kFeatCsr && !v1;
}

template <int MODE>
int plan_seq(const FeatConfig& c, int64_t items, Plan* p) {
  const bool lane = use_lane(MODE);
  const size_t per = lane ? lane_warp_bytes(c.dim) : seq_table_bytes(c.dim);
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  auto kern = lane ? featurize_lane_kernel<MODE, false> : featurize_seq_kernel<MODE>;
  int warps = 1, per_sm = 1, best = 0;
  for (int w : {18, 16, 12, 9, 8, 6, 4, 2, 1}) {
    if (!lane && w > 8) continue;
    const size_t sm_bytes = lane ? lane_cta_bytes(c.dim, w, MODE) : per * w;
    if (sm_bytes > kMaxLaneSmem) continue;
    if (cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm_bytes) !=
        cudaSuccess)
      continue;
    int b = 0;
    const int threads = w * 32;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&b, kern, threads, sm_bytes);
    if (b * w > best) {
      best = b * w;
      warps = w;
      per_sm = b;
    }
  }
  cudaGetLastError();
  if (best == 0) {
    set_error("featurize: no launchable configuration for dimension %u", c.dim);
    return PARS_ERR_UNSUPPORTED;
  }
  p->global_tables = false;
  p->warps = warps;
  p->smem = lane ? lane_cta_bytes(c.dim, warps, MODE) : per * warps;
  p->grid = std::max<int64_t>(
      1, std::min<int64_t>(ceil_div(std::max<int64_t>(items, 1), warps), (int64_t)sms * per_sm));
  return PARS_OK;
}

// Exact mode on the lane path runs in chunks of chain_chunk() prompts
// (default 2^20; PARS_CHAIN_CHUNK overrides): the hashing kernel writes each
// prompt's (idx, count) list to its slot, then chain_slots_thread_kernel
// scores the chunk. Measured on C4 (1M prompts): chunks small enough for the
// lists to stay L2-resident (65,536) lose more to the chain kernel's low
// occupancy than they gain from L2 (5.92 vs 5.38 ms), so the default chunk
// is large and bounds the scratch (2 KB per prompt).
// Scratch after the per-warp arenas: chain_chunk() slots of kSlotCap packed
// entries, then each slot's L2 factor and entry count.
static int64_t chain_chunk() {
  static const int64_t v = [] {
    const char* e = std::getenv("PARS_CHAIN_CHUNK");
    return e ? std::max<int64_t>(1024, std::atoll(e)) : (int64_t)1 << 20;
  }();
  return v;
}

// Exact mode runs the fused lane kernel (hashing warps + chain warp) when
// its shared memory fits; PARS_FEAT_UNFUSED=1 selects the two-kernel form
// (lane kernel writing per-prompt slots + chain_slots_thread_kernel) for A/B.
__host__ inline bool use_fused(const FeatConfig& c) {
  static const bool off = [] {
    const char* e = std::getenv("PARS_FEAT_UNFUSED");
    return e && e[0] == '1';
  }();
  return !off && fused_cta_bytes(c.dim) <= kMaxLaneSmem;
}

__host__ inline int64_t fused_grid(int64_t n) {
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  return std::max<int64_t>(1, std::min<int64_t>(sms, ceil_div(std::max<int64_t>(n, 1), kFuseH)));
}

__host__ inline size_t fused_scratch_bytes(const FeatConfig& c, int64_t n) {
  const int64_t g = fused_grid(n);
  return (((size_t)list_cap_words(c) * 4 * (size_t)g * kFuseH + 255) & ~(size_t)255) + fused_ring_bytes(g);
}

int launch_fused(pars_ctx* ctx, const FeatConfig& c, const FeatArgs& a0, cudaStream_t st) {
  auto kern = featurize_lane_kernel<kFeatScoreExact, true>;
  const size_t bytes = fused_cta_bytes(c.dim);
  PARS_CUDA_CHECK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes));
  const int threads = (kFuseH + kFuseC) * 32;
  int b = 0;
  PARS_CUDA_CHECK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&b, kern, threads, bytes));
  if (b < 1) {
    set_error("featurize: fused kernel does not fit an SM (dimension %u)", c.dim);
    return PARS_ERR_UNSUPPORTED;
  }
  const int64_t grid = fused_grid(a0.n);
  const size_t arenas = (((size_t)a0.list_cap * 4 * (size_t)grid * kFuseH) + 255) & ~(size_t)255;
  if (a0.lists_bytes < arenas + fused_ring_bytes(grid)) {
    set_error("featurize: list scratch too small (fused)");
    return PARS_ERR_INVALID;
  }
  FeatArgs a = a0;
  a.slots = reinterpret_cast<uint32_t*>(reinterpret_cast<unsigned char*>(a0.lists) + arenas);
  a.first = 0;
  kern<<<(unsigned)grid, threads, bytes, st>>>(c, a);
  count_launch(ctx);
  PARS_CUDA_CHECK(cudaGetLastError());
  return PARS_OK;
}

template <int MODE>
int launch_seq(pars_ctx* ctx, const FeatConfig& c, const FeatArgs& a0, cudaStream_t st) {
  if (MODE == kFeatScoreExact && use_lane(MODE) && use_fused(c)) return launch_fused(ctx, c, a0, st);
  Plan p;
  PARS_TRY(plan_seq<MODE>(c, a0.n, &p));
  const size_t arenas = (((size_t)a0.list_cap * 4 * (size_t)p.grid * p.warps) + 255) & ~(size_t)255;
  const bool slots = MODE == kFeatScoreExact && use_lane(MODE);
  const int64_t chunk = std::min<int64_t>(a0.n, chain_chunk());
  if (MODE == kFeatScoreExact && a0.lists_bytes < arenas + (slots ? lane_slot_bytes(chunk) : 0)) {
    set_error("featurize: list scratch too small");
    return PARS_ERR_INVALID;
  }
  auto kern = use_lane(MODE) ? featurize_lane_kernel<MODE, false> : featurize_seq_kernel<MODE>;
  PARS_CUDA_CHECK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)p.smem));
  if (!slots) {
    kern<<<(unsigned)p.grid, p.warps * 32, p.smem, st>>>(c, a0);
    count_launch(ctx);
    PARS_CUDA_CHECK(cudaGetLastError());
    return PARS_OK;
  }
  FeatArgs a = a0;
  unsigned char* b = reinterpret_cast<unsigned char*>(a0.lists) + arenas;
  a.slots = reinterpret_cast<uint32_t*>(b);
  b += (size_t)chunk * kSlotCap * 4;
  a.slot_inv = reinterpret_cast<double*>(b);
  b += (size_t)chunk * 8;
  a.slot_nnz = reinterpret_cast<int32_t*>(b);
  const size_t csm = (size_t)c.dim * 8;
  PARS_CUDA_CHECK(cudaFuncSetAttribute(chain_slots_thread_kernel,
                                       cudaFuncAttributeMaxDynamicSharedMemorySize, (int)csm));
  Plan pc;
  PARS_TRY(plan_seq<MODE>(c, chunk, &pc));  // (plan_seq leaves the attribute at its last probe)
  PARS_CUDA_CHECK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)pc.smem));
  for (int64_t f = 0; f < a0.n; f += chunk) {
    a.first = f;
    a.n = std::min<int64_t>(a0.n, f + chunk);
    kern<<<(unsigned)pc.grid, pc.warps * 32, pc.smem, st>>>(c, a);
    chain_slots_thread_kernel<<<(unsigned)ceil_div(a.n - f, 256), 256, csm, st>>>(c, a);
    count_launch(ctx, 2);
    PARS_CUDA_CHECK(cudaGetLastError());
  }
  return PARS_OK;
}

template <bool POW2, bool DEF, int MODE>
int launch_pair(pars_ctx* ctx, const FeatConfig& c, const FeatArgs& a, cudaStream_t st) {
  PARS_CUDA_CHECK(cudaMemsetAsync(a.long_count, 0, sizeof(int32_t), st));
  if (POW2 && DEF && use_seq(c)) {
    PARS_TRY(launch_seq<MODE>(ctx, c, a, st));
  } else {
    PARS_TRY((launch_one<POW2, false, DEF, MODE>(ctx, c, a, st, a.n)));
  }
  return launch_one<POW2, true, DEF, MODE>(ctx, c, a, st, 0);
}

template <bool POW2, bool DEF, int MODE>
int scratch_pair(const FeatConfig& c, int64_t n, size_t* gs, size_t* ls) {
  *gs = 0;
  *ls = 0;
  for (int wide = 0; wide < 2; ++wide) {
    Plan p;
    int rc = wide ? plan_one<POW2, true, DEF, MODE>(c, 0, &p) : plan_one<POW2, false, DEF, MODE>(c, n, &p);
    if (rc != PARS_OK) return rc;
    const size_t tw = (size_t)p.grid * p.warps;
    if (p.global_tables) *gs = std::max(*gs, warp_table_bytes(c, wide != 0) * tw);
    if (MODE == kFeatScoreExact) *ls = std::max(*ls, (size_t)list_cap_words(c) * 4 * tw);
  }
  if (POW2 && DEF && use_seq(c)) {
    Plan p;
    PARS_TRY(plan_seq<MODE>(c, n, &p));
    if (MODE == kFeatScoreExact) {
      *ls = std::max(*ls, (((size_t)list_cap_words(c) * 4 * (size_t)p.grid * p.warps + 255) & ~(size_t)255) +
                              (use_lane(MODE) ? lane_slot_bytes(std::min<int64_t>(n, chain_chunk())) : 0));
      if (use_lane(MODE) && use_fused(c)) *ls = std::max(*ls, fused_scratch_bytes(c, n));
    }
  }
  return PARS_OK;
}

template <int MODE>
int launch_mode(pars_ctx* ctx, const FeatConfig& c, const FeatArgs& a, cudaStream_t st) {
  if (c.pow2) {
    if (c.default_orders) return launch_pair<true, true, MODE>(ctx, c, a, st);
    return launch_pair<true, false, MODE>(ctx, c, a, st);
  }
  return launch_pair<false, false, MODE>(ctx, c, a, st);
}

template <int MODE>
int scratch_mode(const FeatConfig& c, int64_t n, size_t* gs, size_t* ls) {
  if (c.pow2) {
    if (c.default_orders) return scratch_pair<true, true, MODE>(c, n, gs, ls);
    return scratch_pair<true, false, MODE>(c, n, gs, ls);
  }
  return scratch_pair<false, false, MODE>(c, n, gs, ls);
}

// ---- dense embeddings (features.cpp:67-76) -----------------------------
// Exact: the reference's two sequential chains per prompt — sum of squares in
// index order (features.cpp:113-116), then the dot in index order
// (features.hpp:31-35) — one thread per prompt, the rows reaching it through
// shared memory by TMA bulk copies (cp.async.bulk, one 256-byte row segment
// per copy, completion on an mbarrier). A persistent CTA walks blocks of 128
// prompts; its job stream is (block, pass, 32-column tile) and warp 0 keeps
// kDenseStages tiles in flight ahead of the chains, across pass and block
// boundaries. Rows land with a 272-byte pitch so each quarter-warp's 16-byte
// loads hit distinct banks. With L2 normalisation every row is streamed
// twice (the dot needs the norm first). Requires 16-byte aligned rows (even
// dim, aligned base); otherwise dense_exact_simple_kernel runs.
constexpr int kDenseRows = 64, kDenseCols = 64, kDenseStages = 3;
constexpr int kDensePitch = kDenseCols * 8 + 16;  // bytes per row in a stage
constexpr size_t kDenseStageBytes = (size_t)kDenseRows * kDensePitch;
constexpr size_t kDenseSmem = kDenseStages * kDenseStageBytes + 64;

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return (uint32_t)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void mbar_wait(uint32_t bar, uint32_t parity) {
  asm volatile(
      "{\n\t.reg .pred p;\n\tWAIT_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t@!p bra WAIT_%=;\n\t}" ::"r"(bar),
      "r"(parity)
      : "memory");
}

__global__ void __launch_bounds__(kDenseRows) dense_exact_kernel(
    const double* __restrict__ X, int64_t n, uint32_t dim, int norm, const double* __restrict__ w,
    double bias, double* __restrict__ out) {
  extern __shared__ __align__(128) unsigned char dsm[];
  uint64_t* full = reinterpret_cast<uint64_t*>(dsm + kDenseStages * kDenseStageBytes);
  const int t = threadIdx.x, lane = t & 31, warp = t >> 5;
  const uint32_t ntiles = (dim + kDenseCols - 1) / kDenseCols;
  const int npass = norm ? 2 : 1;
  const int64_t nblocks = (n + kDenseRows - 1) / kDenseRows;
  const int64_t my_blocks = blockIdx.x < nblocks ? (nblocks - 1 - blockIdx.x) / gridDim.x + 1 : 0;
  const int64_t njobs = my_blocks * npass * ntiles;
  if (t == 0) {
    for (int st = 0; st < kDenseStages; ++st)
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(full + st)));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  // job j -> (block, tile); warp 0 copies it into stage j % kDenseStages
  auto issue = [&](int64_t j) {
    const int64_t b = blockIdx.x + (j / (npass * ntiles)) * (int64_t)gridDim.x;
    const uint32_t kt = (uint32_t)(j % ntiles);
    const int64_t r0 = b * kDenseRows;
    const int rows = (int)imin64(kDenseRows, n - r0);
    const uint32_t k0 = kt * kDenseCols;
    const uint32_t seg = min((uint32_t)kDenseCols, dim - k0) * 8u;
    const int st = (int)(j % kDenseStages);
    const uint32_t bar = smem_u32(full + st);
    if (lane == 0)
      asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar),
                   "r"(seg * (uint32_t)rows)
                   : "memory");
    __syncwarp();
    unsigned char* stage = dsm + st * kDenseStageBytes;
    for (int r = lane; r < rows; r += 32)
      asm volatile(
          "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::
              "r"(smem_u32(stage + r * kDensePitch)),
          "l"(X + (r0 + r) * (int64_t)dim + k0), "r"(seg), "r"(bar)
          : "memory");
  };
  if (warp == 0)
    for (int64_t j = 0; j < imin64(njobs, kDenseStages); ++j) issue(j);
  double acc = 0.0, inv = 1.0;
  bool scale = false;
  int64_t j = 0;
  for (int64_t bi = 0; bi < my_blocks; ++bi) {
    const int64_t r0 = (blockIdx.x + bi * (int64_t)gridDim.x) * kDenseRows;
    inv = 1.0;
    scale = false;
    for (int pass = 2 - npass; pass < 2; ++pass) {
      acc = 0.0;
      for (uint32_t kt = 0; kt < ntiles; ++kt, ++j) {
        const int st = (int)(j % kDenseStages);
        mbar_wait(smem_u32(full + st), (uint32_t)((j / kDenseStages) & 1));
        const double* row = reinterpret_cast<const double*>(dsm + st * kDenseStageBytes + t * kDensePitch);
        const uint32_t k0 = kt * kDenseCols;
        if (k0 + kDenseCols <= dim) {
          if (pass == 0) {
#pragma unroll
            for (int k = 0; k < kDenseCols; k += 2) {
              const double2 v = *reinterpret_cast<const double2*>(row + k);
              acc = __dadd_rn(acc, __dmul_rn(v.x, v.x));
              acc = __dadd_rn(acc, __dmul_rn(v.y, v.y));
            }
          } else {
#pragma unroll
            for (int k = 0; k < kDenseCols; k += 2) {
              const double2 v = *reinterpret_cast<const double2*>(row + k);
              const double2 wk = __ldg(reinterpret_cast<const double2*>(w + k0 + k));
              const double a = scale ? __dmul_rn(v.x, inv) : v.x;
              const double b = scale ? __dmul_rn(v.y, inv) : v.y;
              acc = __dadd_rn(acc, __dmul_rn(wk.x, a));
              acc = __dadd_rn(acc, __dmul_rn(wk.y, b));
            }
          }
        } else {
          for (uint32_t k = 0; k < dim - k0; ++k) {
            const double x = row[k];
            if (pass == 0) {
              acc = __dadd_rn(acc, __dmul_rn(x, x));
            } else {
              const double v = scale ? __dmul_rn(x, inv) : x;
              acc = __dadd_rn(acc, __dmul_rn(__ldg(w + k0 + k), v));
            }
          }
        }
        __syncthreads();  // every chain is done with stage st
        if (warp == 0 && j + kDenseStages < njobs) {
          asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
          issue(j + kDenseStages);
        }
      }
      if (pass == 0 && acc > 0.0) {
        inv = __ddiv_rn(1.0, __dsqrt_rn(acc));
        scale = true;
      }
    }
    if (r0 + t < n) out[r0 + t] = __dadd_rn(acc, bias);
  }
}

// Rows that are not 16-byte aligned (odd dim or unaligned base): the same
// two chains straight from global memory, one thread per prompt.
__global__ void dense_exact_simple_kernel(const double* __restrict__ X, int64_t n, uint32_t dim,
                                          int norm, const double* __restrict__ w, double bias,
                                          double* __restrict__ out) {
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
  double s = 0.0;
  for (uint32_t k = 0; k < dim; ++k) {
    const double v = scale ? __dmul_rn(x[k], inv) : x[k];
    s = __dadd_rn(s, __dmul_rn(w[k], v));
  }
  out[i] = __dadd_rn(s, bias);
}

// Fast: one warp per prompt, 16-byte row loads eight deep per lane (4 KB
// of the row in flight per warp), fp32 products, tree reductions.
__global__ void __launch_bounds__(256) dense_fast_kernel(const double* __restrict__ X, int64_t n,
                                                         uint32_t dim, int norm,
                                                         const float* __restrict__ w, double bias,
                                                         double* __restrict__ out) {
  const int lane = threadIdx.x & 31;
  const int64_t i = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  if (i >= n) return;
  const double* x = X + i * (int64_t)dim;
  float sq = 0.f, dot = 0.f;
  if ((dim & 1) == 0 && (reinterpret_cast<uintptr_t>(x) & 15) == 0) {
    const double2* x2 = reinterpret_cast<const double2*>(x);
    const uint32_t n2 = dim >> 1;
    constexpr int kU = 8;
    uint32_t k = lane;
    for (; k + 32 * (kU - 1) < n2; k += 32 * kU) {
      double2 v[kU];
#pragma unroll
      for (int u = 0; u < kU; ++u) v[u] = __ldcs(x2 + k + 32 * u);
#pragma unroll
      for (int u = 0; u < kU; ++u) {
        const float a = (float)v[u].x, b = (float)v[u].y;
        const uint32_t e = 2 * (k + 32 * u);
        sq = fmaf(a, a, fmaf(b, b, sq));
        dot = fmaf(__ldg(w + e), a, fmaf(__ldg(w + e + 1), b, dot));
      }
    }
    for (; k < n2; k += 32) {
      const double2 v = __ldcs(x2 + k);
      const float a = (float)v.x, b = (float)v.y;
      sq = fmaf(a, a, fmaf(b, b, sq));
      dot = fmaf(__ldg(w + 2 * k), a, fmaf(__ldg(w + 2 * k + 1), b, dot));
    }
  } else {
    for (uint32_t k = lane; k < dim; k += 32) {
      const float v = (float)x[k];
      sq = fmaf(v, v, sq);
      dot = fmaf(w[k], v, dot);
    }
  }
  sq = warp_sum_f32(sq);
  dot = warp_sum_f32(dot);
  if (lane == 0) {
    const float inv = (norm && sq > 0.f) ? rsqrtf(sq) : 1.f;
    out[i] = (double)(dot * inv) + bias;
  }
}

// Exact, cooperative staging: a CTA owns blocks of kCoopRows prompts, one
// thread per prompt running the reference's sequential chains (sum of
// squares in index order, features.cpp:113-116, then the dot in index order,
// features.hpp:31-35). All 256 threads stream each 32-column tile of the
// block's rows into shared memory with 16-byte cp.async copies (a warp
// covers two 256-byte row segments: full sectors), kCoopStages tiles in
// flight, the weights' tile alongside; the chains then read their row from
// shared memory (272-byte pitch: conflict-free 16-byte reads). With L2
// normalisation the block is streamed twice (the dot needs the norm first).
constexpr int kCoopRows = 256, kCoopCols = 32, kCoopStages = 3;
constexpr int kCoopPitch = kCoopCols * 8 + 16;
constexpr size_t kCoopStageBytes = (size_t)kCoopRows * kCoopPitch + kCoopCols * 8;
constexpr size_t kCoopSmem = kCoopStages * kCoopStageBytes;

__global__ void __launch_bounds__(kCoopRows, 1) dense_coop_kernel(
    const double* __restrict__ X, int64_t n, uint32_t dim, int norm, const double* __restrict__ w,
    double bias, double* __restrict__ out) {
  extern __shared__ __align__(16) unsigned char csm2[];
  const int t = threadIdx.x;
  const uint32_t ntiles = (dim + kCoopCols - 1) / kCoopCols;
  const int npass = norm ? 2 : 1;
  const int64_t nblocks = (n + kCoopRows - 1) / kCoopRows;
  const int64_t my_blocks = blockIdx.x < nblocks ? (nblocks - 1 - blockIdx.x) / gridDim.x + 1 : 0;
  const int64_t njobs = my_blocks * npass * ntiles;
  // job j -> (block, pass, tile): every thread copies 16 of the stage's
  // 16-byte chunks (+ one weight chunk for threads < 16)
  auto issue = [&](int64_t j) {
    const int64_t b = blockIdx.x + (j / (npass * ntiles)) * (int64_t)gridDim.x;
    const uint32_t kt = (uint32_t)(j % ntiles);
    const int64_t r0 = b * kCoopRows;
    const uint32_t c0 = kt * kCoopCols;
    unsigned char* st = csm2 + (size_t)(j % kCoopStages) * kCoopStageBytes;
#pragma unroll
    for (int q = 0; q < (kCoopRows * kCoopCols / 2) / kCoopRows; ++q) {
      const int c = t + kCoopRows * q;  // chunk: row c / 16, column pair c % 16
      const int r = c >> 4, cp = c & 15;
      const uint32_t col = c0 + 2 * cp;
      const bool ok = r0 + r < n && col < dim;
      const double* src = ok ? X + (r0 + r) * (int64_t)dim + col : X;
      const uint32_t dst = (uint32_t)__cvta_generic_to_shared(st + (size_t)r * kCoopPitch + 16 * cp);
      asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(dst), "l"(src),
                   "r"(ok ? 16 : 0));
    }
    if (t < kCoopCols / 2) {
      const uint32_t col = c0 + 2 * t;
      const uint32_t dst =
          (uint32_t)__cvta_generic_to_shared(st + (size_t)kCoopRows * kCoopPitch + 16 * t);
      asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(dst),
                   "l"(col < dim ? w + col : w), "r"(col < dim ? 16 : 0));
    }
  };
  for (int64_t j = 0; j < kCoopStages - 1; ++j) {
    if (j < njobs) issue(j);
    asm volatile("cp.async.commit_group;");
  }
  double acc = 0.0, inv = 1.0;
  bool scale = false;
  for (int64_t j = 0; j < njobs; ++j) {
    asm volatile("cp.async.wait_group %0;" ::"n"(kCoopStages - 2));
    __syncthreads();  // stage j % S landed for every thread; stage (j-1) % S is free
    if (j + kCoopStages - 1 < njobs) issue(j + kCoopStages - 1);
    asm volatile("cp.async.commit_group;");
    const int64_t b = blockIdx.x + (j / (npass * ntiles)) * (int64_t)gridDim.x;
    const int pass = (int)((j / ntiles) % npass);
    const uint32_t kt = (uint32_t)(j % ntiles);
    const unsigned char* st = csm2 + (size_t)(j % kCoopStages) * kCoopStageBytes;
    const double2* row = reinterpret_cast<const double2*>(st + (size_t)t * kCoopPitch);
    const double2* wt = reinterpret_cast<const double2*>(st + (size_t)kCoopRows * kCoopPitch);
    const uint32_t cols = min((uint32_t)kCoopCols, dim - kt * kCoopCols);
    if (kt == 0) acc = 0.0;
    if (pass == 0 && norm) {
#pragma unroll 4
      for (uint32_t k = 0; k < cols / 2; ++k) {
        const double2 v = row[k];
        acc = __dadd_rn(acc, __dmul_rn(v.x, v.x));
        acc = __dadd_rn(acc, __dmul_rn(v.y, v.y));
      }
      if (kt == ntiles - 1) {
        scale = acc > 0.0;
        inv = scale ? __ddiv_rn(1.0, __dsqrt_rn(acc)) : 1.0;
      }
    } else {
#pragma unroll 4
      for (uint32_t k = 0; k < cols / 2; ++k) {
        const double2 v = row[k], ww = wt[k];
        const double a = scale ? __dmul_rn(v.x, inv) : v.x;
        const double bq = scale ? __dmul_rn(v.y, inv) : v.y;
        acc = __dadd_rn(acc, __dmul_rn(ww.x, a));
        acc = __dadd_rn(acc, __dmul_rn(ww.y, bq));
      }
      if (kt == ntiles - 1) {
        const int64_t i = b * kCoopRows + t;
        if (i < n) out[i] = __dadd_rn(acc, bias);
        scale = false;
        inv = 1.0;
      }
    }
  }
  asm volatile("cp.async.wait_all;" ::: "memory");
}

}  // namespace

bool build_feat_config(const pars_extractor* ex, FeatConfig* c) {
  std::memset(c, 0, sizeof *c);
  if (ex->dim == 0) {
    set_error("feature extractor dimension is 0");
    return false;
  }
  if (ex->n_word < 0 || ex->n_word > 8 || ex->n_char < 0 || ex->n_char > 8) {
    set_error("at most 8 word and 8 char n-gram orders are supported");
    return false;
  }
  c->dim = ex->dim;
  c->pow2 = (ex->dim & (ex->dim - 1)) == 0 ? 1 : 0;
  c->mask = ex->dim - 1;
  c->norm = ex->norm == 1 ? 1 : 0;
  c->n_word = ex->n_word;
  c->n_char = ex->n_char;
  c->max_word = 0;
  for (int k = 0; k < ex->n_word; ++k) {
    if (ex->word[k] < 1) {
      set_error("word n-gram order must be >= 1");
      return false;
    }
    c->word[k] = ex->word[k];
    c->word_salt[k] = ngram_salt(1, (uint64_t)ex->word[k]);
    c->max_word = std::max(c->max_word, ex->word[k]);
  }
  for (int k = 0; k < ex->n_char; ++k) {
    if (ex->chr[k] < 1) {
      set_error("char n-gram order must be >= 1");
      return false;
    }
    c->chr[k] = ex->chr[k];
    c->char_salt[k] = ngram_salt(2, (uint64_t)ex->chr[k]);
  }
  if (c->max_word > 32) {
    set_error("word n-gram order %d exceeds the supported maximum (32)", c->max_word);
    return false;
  }
  c->default_orders = (ex->n_word == 1 && ex->word[0] == 1 && ex->n_char == 1 && ex->chr[0] == 3);
  return true;
}

uint32_t feat_list_cap_words(const FeatConfig& c) { return list_cap_words(c); }

int feat_scratch_bytes(const FeatConfig& c, int mode, int64_t n, size_t* gscratch, size_t* lists) {
  switch (mode) {
    case kFeatScoreExact:
      return scratch_mode<kFeatScoreExact>(c, n, gscratch, lists);
    case kFeatScoreFast:
      return scratch_mode<kFeatScoreFast>(c, n, gscratch, lists);
    case kFeatCsr:
      return scratch_mode<kFeatCsr>(c, n, gscratch, lists);
  }
  set_error("unknown featurize mode %d", mode);
  return PARS_ERR_INVALID;
}

int launch_featurize(pars_ctx* ctx, const FeatConfig& c, int mode, const FeatArgs& a,
                     cudaStream_t st) {
  if (a.n == 0) return PARS_OK;
  switch (mode) {
    case kFeatScoreExact:
      return launch_mode<kFeatScoreExact>(ctx, c, a, st);
    case kFeatScoreFast:
      return launch_mode<kFeatScoreFast>(ctx, c, a, st);
    case kFeatCsr:
      return launch_mode<kFeatCsr>(ctx, c, a, st);
  }
  set_error("unknown featurize mode %d", mode);
  return PARS_ERR_INVALID;
}

// PARS_DENSE_TMA=1 selects the round-1 TMA bulk-copy kernel (A/B)
__host__ inline bool use_dense_tma() {
  static const bool v = [] {
    const char* e = std::getenv("PARS_DENSE_TMA");
    return e && e[0] == '1';
  }();
  return v;
}

int launch_score_dense(pars_ctx* ctx, const FeatConfig& c, int mode, const double* X, int64_t n,
                       const double* w64, const float* w32, double bias, double* scores,
                       cudaStream_t st) {
  if (n == 0) return PARS_OK;
  if (mode == PARS_MODE_EXACT_F64) {
    const bool aligned = (c.dim % 2 == 0) && (reinterpret_cast<uintptr_t>(X) % 16 == 0) &&
                         (reinterpret_cast<uintptr_t>(w64) % 16 == 0);
    if (!aligned) {
      dense_exact_simple_kernel<<<(unsigned)ceil_div(n, 128), 128, 0, st>>>(X, n, c.dim, c.norm, w64,
                                                                           bias, scores);
    } else if (!use_dense_tma()) {
      PARS_CUDA_CHECK(cudaFuncSetAttribute(dense_coop_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                           (int)kCoopSmem));
      int dev = 0, sms = 148;
      cudaGetDevice(&dev);
      cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
      const int64_t grid = std::max<int64_t>(1, std::min<int64_t>(ceil_div(n, kCoopRows), sms));
      dense_coop_kernel<<<(unsigned)grid, kCoopRows, kCoopSmem, st>>>(X, n, c.dim, c.norm, w64, bias,
                                                                    scores);
    } else {
      PARS_CUDA_CHECK(cudaFuncSetAttribute(dense_exact_kernel,
                                           cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kDenseSmem));
      int dev = 0, sms = 148, per_sm = 1;
      cudaGetDevice(&dev);
      cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
      cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, dense_exact_kernel, kDenseRows, kDenseSmem);
      const int64_t blocks = ceil_div(n, kDenseRows);
      const int64_t grid =
          std::max<int64_t>(1, std::min<int64_t>(blocks, (int64_t)sms * std::max(per_sm, 1)));
      dense_exact_kernel<<<(unsigned)grid, kDenseRows, kDenseSmem, st>>>(X, n, c.dim, c.norm, w64,
                                                                       bias, scores);
    }
  } else {
    dense_fast_kernel<<<(unsigned)ceil_div(n * 32, 256), 256, 0, st>>>(X, n, c.dim, c.norm, w32,
                                                                       bias, scores);
  }
  count_launch(ctx);
  PARS_CUDA_CHECK(cudaGetLastError());
  return PARS_OK;
}

}  // namespace pars_b200
