// Fused hashing featurizer + linear score head, one warp per prompt.
//
// Reference semantics (all in /root/reference/proj/src/features.cpp):
//   split_tokens :36-49 (C-locale isspace), word n-grams :80-92 (FNV-1a over
//   token bytes then "\x1f", seeded by salt(1, order)), char n-grams inside
//   tokens :93-101 (salt(2, order)), add_hashed :29-34 (idx = (h>>1) % dim,
//   sign = h&1 ? +1 : -1), sort+merge :102-109, erase zeros :110,
//   L2 :113-120; scorer.cpp:36-42 + features.hpp:31-35 for the dot + bias.
//
// B200 design:
//   * one warp owns one prompt at a time; the text is streamed through the
//     warp 128 bytes per step (one aligned 4-byte load per lane), whitespace
//     transitions are found with lane bitmasks + shuffles and compacted into a
//     per-warp token ring in shared memory;
//   * lane t hashes token t of a 32-token batch (word n-gram + all char
//     n-grams of that token). For power-of-two dims only the low log2(dim)+1
//     bits of the 64-bit FNV state are ever observed, and FNV's xor/multiply
//     are closed mod 2^32, so the hash runs in 32-bit arithmetic
//     (P mod 2^32 = 0x1b3): one LOP3 + one IMAD per byte;
//   * features are histogrammed into a per-warp shared-memory table of
//     16-bit biased counters packed two per word (atomicAdd), with a
//     touched-bucket bitmap set on first touch. Integer sums are exact and
//     order-free, so the merge/erase of the reference needs no sort;
//   * the bitmap is walked in ascending bucket order: L2 from the exact
//     integer sum of squares, products w[idx]*v computed lane-parallel, and
//     the bit-exact fp64 dot is a sequential __dadd_rn chain over the
//     ascending products (exact mode) or a warp tree reduction (fast mode).
#include <cuda_runtime.h>

#include <algorithm>
#include <cstring>

#include "featurize.cuh"

namespace pars_b200 {

namespace {

constexpr unsigned kFull = 0xffffffffu;
constexpr int kRing = 128;       // token ring entries per warp (start,end)
constexpr int kProd = 256;       // exact-mode product buffer (doubles)
constexpr uint32_t kBias2 = 0x80008000u;  // two biased 16-bit zero counters
constexpr int64_t kPackedMaxFeatures = 32767;
constexpr int kGlobalWarps = 1184;  // 148 SMs x 8 warps

struct WarpSmem {
  uint32_t* counts;  // packed (2 x u16 biased) or wide (int32)
  uint32_t* bitmap;  // touched buckets
  uint32_t* tok_s;   // ring: token start (relative to prompt begin)
  uint32_t* tok_e;   // ring: token end (exclusive)
  double* prod;      // exact-mode product buffer
};

__host__ __device__ inline uint32_t bitmap_words_padded(uint32_t dim) {
  uint32_t w = (dim + 31) / 32;
  return (w + 7) & ~7u;
}
// Rounded so that every 8-bucket group read/clear stays inside the table.
__host__ __device__ inline uint32_t count_words(uint32_t dim, bool wide) {
  return wide ? ((dim + 7) & ~7u) : ((((dim + 1) / 2) + 3) & ~3u);
}

template <bool WIDE>
__device__ __forceinline__ void emit(const WarpSmem& S, uint32_t idx, bool pos) {
  uint32_t old;
  bool first;
  if (WIDE) {
    old = atomicAdd(&S.counts[idx], pos ? 1u : 0xffffffffu);
    first = old == 0u;
  } else {
    uint32_t sh = (idx & 1u) << 4;
    uint32_t d = pos ? (1u << sh) : (0u - (1u << sh));
    old = atomicAdd(&S.counts[idx >> 1], d);
    first = ((old >> sh) & 0xffffu) == 0x8000u;
  }
  if (first) atomicOr(&S.bitmap[idx >> 5], 1u << (idx & 31));
}

// Counters of the 8 consecutive buckets [b0, b0+8) (b0 % 8 == 0): one
// 16-byte shared load (packed) or two (wide).
template <bool WIDE>
__device__ __forceinline__ void load_group(const WarpSmem& S, uint32_t b0, int cnt[8]) {
  if (WIDE) {
    const uint4 u0 = *reinterpret_cast<const uint4*>(S.counts + b0);
    const uint4 u1 = *reinterpret_cast<const uint4*>(S.counts + b0 + 4);
    cnt[0] = (int)u0.x; cnt[1] = (int)u0.y; cnt[2] = (int)u0.z; cnt[3] = (int)u0.w;
    cnt[4] = (int)u1.x; cnt[5] = (int)u1.y; cnt[6] = (int)u1.z; cnt[7] = (int)u1.w;
  } else {
    const uint4 u = *reinterpret_cast<const uint4*>(S.counts + (b0 >> 1));
    const uint32_t w[4] = {u.x, u.y, u.z, u.w};
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      cnt[2 * j] = (int)(w[j] & 0xffffu) - 0x8000;
      cnt[2 * j + 1] = (int)(w[j] >> 16) - 0x8000;
    }
  }
}

template <bool WIDE>
__device__ __forceinline__ void clear_group(const WarpSmem& S, uint32_t b0) {
  if (WIDE) {
    *reinterpret_cast<uint4*>(S.counts + b0) = make_uint4(0u, 0u, 0u, 0u);
    *reinterpret_cast<uint4*>(S.counts + b0 + 4) = make_uint4(0u, 0u, 0u, 0u);
  } else {
    *reinterpret_cast<uint4*>(S.counts + (b0 >> 1)) = make_uint4(kBias2, kBias2, kBias2, kBias2);
  }
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

// Hash token `t` (ring index) and everything that starts at it.
template <bool POW2, bool WIDE, bool DEF>
__device__ __forceinline__ void hash_token(const FeatConfig& c, const WarpSmem& S,
                                           const uint8_t* base, int64_t t,
                                           int64_t ntok_avail) {
  using HT = H<POW2>;
  using T = typename HT::T;
  const uint32_t s = S.tok_s[t % kRing], e = S.tok_e[t % kRing];
  const uint8_t* tp = base + s;
  const int len = (int)(e - s);
  if (DEF) {
    // word {1} + char {3} in one pass over the token bytes
    T hw = HT::seed(c.word_salt[0]);
    const T hc0 = HT::seed(c.char_salt[0]);
    uint32_t b2 = 0, b1 = 0;
    for (int i = 0; i < len; ++i) {
      uint32_t b = ld_byte(tp + i);
      hw = HT::step(hw, b);
      if (i >= 2) {
        T h = HT::step(HT::step(HT::step(hc0, b2), b1), b);
        emit<WIDE>(S, HT::bucket(h, c), (h & 1) != 0);
      }
      b2 = b1;
      b1 = b;
    }
    hw = HT::step(hw, 0x1fu);
    emit<WIDE>(S, HT::bucket(hw, c), (hw & 1) != 0);
    return;
  }
  for (int k = 0; k < c.n_word; ++k) {
    const int order = c.word[k];
    if (t + order - 1 >= ntok_avail) continue;  // n-gram runs past the last token
    T h = HT::seed(c.word_salt[k]);
    for (int j = 0; j < order; ++j) {
      const uint32_t sj = S.tok_s[(t + j) % kRing], ej = S.tok_e[(t + j) % kRing];
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

// Tokenise + hash one prompt into the warp's histogram.
template <bool POW2, bool WIDE, bool DEF>
__device__ void hash_prompt(const FeatConfig& c, const WarpSmem& S, const uint8_t* text,
                            int64_t beg, int64_t end, int lane) {
  const uint8_t* base = text + beg;
  int64_t n_start = 0, n_end = 0, done = 0;
  uint32_t carry_ns = 0;
  const int64_t look = c.max_word > 1 ? c.max_word - 1 : 0;
  // windows are aligned on the ABSOLUTE address so every lane's 4-byte load
  // is naturally aligned whatever the arena/offset alignment
  const int64_t len = end - beg;
  const int64_t mis = (int64_t)(reinterpret_cast<uintptr_t>(base) & 3u);
  for (int64_t wrel = -mis; wrel < len; wrel += 128) {
    const int64_t p = wrel + 4 * lane;  // relative to base; may be negative
    uint32_t word;
    if (p >= 0 && p + 4 <= len) {
      word = __ldg(reinterpret_cast<const uint32_t*>(base + p));
    } else {
      word = 0x20202020u;
#pragma unroll
      for (int k = 0; k < 4; ++k)
        if (p + k >= 0 && p + k < len)
          word = (word & ~(0xffu << (8 * k))) | ((uint32_t)base[p + k] << (8 * k));
    }
    uint32_t ns = 0;
#pragma unroll
    for (int k = 0; k < 4; ++k) ns |= (is_space((word >> (8 * k)) & 0xffu) ? 0u : 1u) << k;
    uint32_t prev = __shfl_up_sync(kFull, ns >> 3, 1);
    if (lane == 0) prev = carry_ns;
    const uint32_t nsprev = ((ns << 1) | prev) & 0xfu;
    const uint32_t starts = ns & ~nsprev;
    const uint32_t ends = ~ns & nsprev & 0xfu;  // byte k is the exclusive end
    carry_ns = __shfl_sync(kFull, ns >> 3, 31);
    int tot_s, tot_e;
    int ps = warp_excl_scan(__popc(starts), lane, &tot_s);
    int pe = warp_excl_scan(__popc(ends), lane, &tot_e);
    const uint32_t rel = (uint32_t)p;
    for (uint32_t m = starts; m; m &= m - 1) {
      int k = __ffs(m) - 1;
      S.tok_s[(n_start + ps++) % kRing] = rel + k;
    }
    for (uint32_t m = ends; m; m &= m - 1) {
      int k = __ffs(m) - 1;
      S.tok_e[(n_end + pe++) % kRing] = rel + k;
    }
    n_start += tot_s;
    n_end += tot_e;
    __syncwarp();
    while (n_end - done >= 32 + look) {
      hash_token<POW2, WIDE, DEF>(c, S, base, done + lane, n_end);
      done += 32;
      __syncwarp();
    }
  }
  if (carry_ns) {  // the last token runs to the end of the prompt
    if (lane == 0) S.tok_e[n_end % kRing] = (uint32_t)len;
    ++n_end;
    __syncwarp();
  }
  while (done < n_end) {
    if (done + lane < n_end) hash_token<POW2, WIDE, DEF>(c, S, base, done + lane, n_end);
    done += 32;
  }
  __syncwarp();
}

__device__ __forceinline__ unsigned long long warp_sum_u64(unsigned long long v) {
#pragma unroll
  for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(kFull, v, o);
  return v;
}
__device__ __forceinline__ float warp_sum_f32(float v) {
#pragma unroll
  for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(kFull, v, o);
  return v;
}

// Walk the touched buckets in ascending order and finish the prompt.
// Lane l of an 8-word bitmap window owns buckets [b0, b0+8), so lane order is
// bucket order; entries are compacted with a warp scan.
template <bool WIDE, int MODE>
__device__ void finish_prompt(const FeatConfig& c, const WarpSmem& S, const FeatArgs& a,
                              int64_t i, int lane) {
  const uint32_t nbw = bitmap_words_padded(c.dim);
  const int sub = lane & 3, wsel = lane >> 2;
  // pass A: exact integer sum of squares (features.cpp:113-116)
  unsigned long long sq = 0;
  if (c.norm) {
    for (uint32_t wb = 0; wb < nbw; wb += 8) {
      const uint32_t bits = (S.bitmap[wb + wsel] >> (8 * sub)) & 0xffu;
      if (bits) {
        int cnt[8];
        load_group<WIDE>(S, (wb + wsel) * 32 + 8 * sub, cnt);
#pragma unroll
        for (int j = 0; j < 8; ++j) sq += (unsigned long long)((long long)cnt[j] * cnt[j]);
      }
    }
    sq = warp_sum_u64(sq);
  }
  const double inv = (c.norm && sq > 0) ? __ddiv_rn(1.0, __dsqrt_rn((double)sq)) : 1.0;

  double chain = 0.0;  // lane 0: sequential fp64 dot (exact mode)
  float facc = 0.f;    // fast mode partial
  int64_t row_pos = 0;
  const int64_t slot = (MODE == kFeatCsr) ? a.slot_base[i] : 0;
  for (uint32_t wb = 0; wb < nbw; wb += 8) {
    const uint32_t bits = (S.bitmap[wb + wsel] >> (8 * sub)) & 0xffu;
    if (__ballot_sync(kFull, bits != 0) == 0) continue;
    __syncwarp();
    if (sub == 0) S.bitmap[wb + wsel] = 0u;
    const uint32_t b0 = (wb + wsel) * 32 + 8 * sub;
    int cnt[8];
    uint32_t nz = 0;
    if (bits) {
      load_group<WIDE>(S, b0, cnt);
      clear_group<WIDE>(S, b0);
#pragma unroll
      for (int j = 0; j < 8; ++j) nz |= (cnt[j] != 0 ? 1u : 0u) << j;  // erase zeros (:110)
    }
    int total;
    const int pos = warp_excl_scan(__popc(nz), lane, &total);
    if (total == 0) continue;
    if (MODE == kFeatScoreExact) {
#pragma unroll
      for (int j = 0; j < 8; ++j)
        if (nz & (1u << j)) {
          const double v = c.norm ? __dmul_rn((double)cnt[j], inv) : (double)cnt[j];
          S.prod[pos + __popc(nz & ((1u << j) - 1))] = __dmul_rn(__ldg(a.w64 + b0 + j), v);
        }
      __syncwarp();
      if (lane == 0) {
        int k = 0;
        for (; k + 4 <= total; k += 4) {
          const double2 p01 = *reinterpret_cast<const double2*>(S.prod + k);
          const double2 p23 = *reinterpret_cast<const double2*>(S.prod + k + 2);
          chain = __dadd_rn(chain, p01.x);
          chain = __dadd_rn(chain, p01.y);
          chain = __dadd_rn(chain, p23.x);
          chain = __dadd_rn(chain, p23.y);
        }
        for (; k < total; ++k) chain = __dadd_rn(chain, S.prod[k]);
      }
      __syncwarp();
    } else if (MODE == kFeatScoreFast) {
      const float finv = (float)inv;
#pragma unroll
      for (int j = 0; j < 8; ++j)
        if (nz & (1u << j)) facc += __ldg(a.w32 + b0 + j) * ((float)cnt[j] * finv);
    } else {
#pragma unroll
      for (int j = 0; j < 8; ++j)
        if (nz & (1u << j)) {
          const double v = c.norm ? __dmul_rn((double)cnt[j], inv) : (double)cnt[j];
          const int64_t o = slot + row_pos + pos + __popc(nz & ((1u << j) - 1));
          a.out_idx[o] = b0 + j;
          a.out_val[o] = v;
        }
      row_pos += total;
    }
  }
  if (MODE == kFeatScoreExact) {
    if (lane == 0) a.scores[i] = __dadd_rn(chain, a.bias);
  } else if (MODE == kFeatScoreFast) {
    facc = warp_sum_f32(facc);
    if (lane == 0) a.scores[i] = (double)facc + a.bias;
  } else {
    if (lane == 0) a.out_nnz[i] = (int32_t)row_pos;
  }
  __syncwarp();
}

__host__ __device__ inline size_t warp_smem_bytes(const FeatConfig& c, int mode, bool wide) {
  size_t b = (size_t)count_words(c.dim, wide) * 4 + (size_t)bitmap_words_padded(c.dim) * 4 +
             (size_t)kRing * 8;
  b = (b + 15) & ~(size_t)15;
  if (mode == kFeatScoreExact) b += (size_t)kProd * 8;
  return b;
}

// G: the per-warp table lives in a global-memory scratch region instead of
// shared memory (dimensions whose histogram does not fit on chip).
template <bool POW2, bool WIDE, bool DEF, int MODE, bool G>
__global__ void __launch_bounds__(256) featurize_kernel(const FeatConfig c, const FeatArgs a) {
  extern __shared__ __align__(16) unsigned char smem[];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const size_t per = warp_smem_bytes(c, MODE, WIDE);
  unsigned char* my = G ? a.gscratch + per * ((size_t)blockIdx.x * (blockDim.x >> 5) + warp)
                        : smem + per * warp;
  WarpSmem S;
  S.counts = reinterpret_cast<uint32_t*>(my);
  S.bitmap = S.counts + count_words(c.dim, WIDE);
  S.tok_s = S.bitmap + bitmap_words_padded(c.dim);
  S.tok_e = S.tok_s + kRing;
  S.prod = reinterpret_cast<double*>(my + (((size_t)count_words(c.dim, WIDE) * 4 +
                                            (size_t)bitmap_words_padded(c.dim) * 4 +
                                            (size_t)kRing * 8 + 15) & ~(size_t)15));
  const uint32_t cw = count_words(c.dim, WIDE);
  for (uint32_t k = lane; k < cw; k += 32) S.counts[k] = WIDE ? 0u : kBias2;
  for (uint32_t k = lane; k < bitmap_words_padded(c.dim); k += 32) S.bitmap[k] = 0u;
  __syncwarp();

  const int64_t gw = (int64_t)blockIdx.x * (blockDim.x >> 5) + warp;
  const int64_t nw = (int64_t)gridDim.x * (blockDim.x >> 5);
  const int64_t count = WIDE ? (int64_t)*a.long_count : a.n;
  for (int64_t it = gw; it < count; it += nw) {
    const int64_t i = WIDE ? (int64_t)a.long_list[it] : it;
    const int64_t beg = a.offsets[i], end = a.offsets[i + 1];
    if (!WIDE) {
      const int64_t len = end - beg;
      const int64_t feats = (int64_t)c.n_word * ((len + 1) / 2) + (int64_t)c.n_char * len;
      if (feats > kPackedMaxFeatures) {  // 16-bit counters could overflow
        if (lane == 0) a.long_list[atomicAdd(a.long_count, 1)] = (int32_t)i;
        continue;
      }
    }
    hash_prompt<POW2, WIDE, DEF>(c, S, a.text, beg, end, lane);
    finish_prompt<WIDE, MODE>(c, S, a, i, lane);
  }
}

constexpr size_t kMaxSmemPerBlock = 200 * 1024;

template <bool POW2, bool WIDE, bool DEF, int MODE>
int launch_one(pars_ctx* ctx, const FeatConfig& c, const FeatArgs& a, cudaStream_t st,
               int64_t items_hint) {
  const size_t per = warp_smem_bytes(c, MODE, WIDE);
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  if (per > kMaxSmemPerBlock) {
    // global-memory tables: fixed grid, region per warp provided by the caller
    if (!a.gscratch || a.gscratch_bytes < per * (size_t)kGlobalWarps) {
      set_error("featurize: global scratch missing for dimension %u", c.dim);
      return PARS_ERR_INVALID;
    }
    auto kern = featurize_kernel<POW2, WIDE, DEF, MODE, true>;
    kern<<<kGlobalWarps / 4, 128, 0, st>>>(c, a);
    count_launch(ctx);
    PARS_CUDA_CHECK(cudaGetLastError());
    return PARS_OK;
  }
  int warps = (int)std::max<size_t>(1, std::min<size_t>(8, (96 * 1024) / per));
  if (WIDE) warps = 1;
  const size_t smem = per * warps;
  auto kern = featurize_kernel<POW2, WIDE, DEF, MODE, false>;
  PARS_CUDA_CHECK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  int per_sm = 1;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, warps * 32, smem);
  if (per_sm < 1) per_sm = 1;
  int64_t want = ceil_div(std::max<int64_t>(items_hint, 1), warps);
  int64_t grid = std::min<int64_t>(want, (int64_t)sms * per_sm);
  if (WIDE) grid = (int64_t)sms * per_sm;  // count known only on device
  if (grid < 1) grid = 1;
  kern<<<(unsigned)grid, warps * 32, smem, st>>>(c, a);
  count_launch(ctx);
  PARS_CUDA_CHECK(cudaGetLastError());
  return PARS_OK;
}

template <bool POW2, bool DEF, int MODE>
int launch_pair(pars_ctx* ctx, const FeatConfig& c, const FeatArgs& a, cudaStream_t st) {
  PARS_CUDA_CHECK(cudaMemsetAsync(a.long_count, 0, sizeof(int32_t), st));
  PARS_TRY((launch_one<POW2, false, DEF, MODE>(ctx, c, a, st, a.n)));
  return launch_one<POW2, true, DEF, MODE>(ctx, c, a, st, 0);
}

template <int MODE>
int launch_mode(pars_ctx* ctx, const FeatConfig& c, const FeatArgs& a, cudaStream_t st) {
  if (c.pow2) {
    if (c.default_orders) return launch_pair<true, true, MODE>(ctx, c, a, st);
    return launch_pair<true, false, MODE>(ctx, c, a, st);
  }
  return launch_pair<false, false, MODE>(ctx, c, a, st);
}

// ---- dense embeddings (features.cpp:67-76) -----------------------------
// Exact: one thread per prompt keeps the reference's two sequential chains
// (sum of squares in index order, then the dot in index order).
__global__ void dense_exact_kernel(const double* __restrict__ X, int64_t n, uint32_t dim,
                                   int norm, const double* __restrict__ w, double bias,
                                   double* __restrict__ out) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const double* x = X + i * (int64_t)dim;
  double inv = 1.0;
  bool scale = false;
  if (norm) {
    double sq = 0.0;
    for (uint32_t k = 0; k < dim; ++k) {
      double v = x[k];
      sq = __dadd_rn(sq, __dmul_rn(v, v));
    }
    if (sq > 0.0) {
      inv = __ddiv_rn(1.0, __dsqrt_rn(sq));
      scale = true;
    }
  }
  double s = 0.0;
  for (uint32_t k = 0; k < dim; ++k) {
    double v = scale ? __dmul_rn(x[k], inv) : x[k];
    s = __dadd_rn(s, __dmul_rn(w[k], v));
  }
  out[i] = __dadd_rn(s, bias);
}

// Fast: one warp per prompt, coalesced row reads, fp32 tree reductions.
__global__ void dense_fast_kernel(const double* __restrict__ X, int64_t n, uint32_t dim,
                                  int norm, const float* __restrict__ w, double bias,
                                  double* __restrict__ out) {
  const int lane = threadIdx.x & 31;
  const int64_t i = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  if (i >= n) return;
  const double* x = X + i * (int64_t)dim;
  float sq = 0.f, dot = 0.f;
  for (uint32_t k = lane; k < dim; k += 32) {
    float v = (float)x[k];
    sq += v * v;
    dot += w[k] * v;
  }
  sq = warp_sum_f32(sq);
  dot = warp_sum_f32(dot);
  if (lane == 0) {
    float inv = (norm && sq > 0.f) ? rsqrtf(sq) : 1.f;
    out[i] = (double)(dot * inv) + bias;
  }
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

size_t feat_warp_smem(const FeatConfig& cfg, int mode, bool wide) {
  return warp_smem_bytes(cfg, mode, wide);
}

size_t feat_global_scratch_bytes(const FeatConfig& cfg, int mode) {
  size_t need = 0;
  for (int wide = 0; wide < 2; ++wide) {
    const size_t per = warp_smem_bytes(cfg, mode, wide != 0);
    if (per > kMaxSmemPerBlock) need = std::max(need, per * (size_t)kGlobalWarps);
  }
  return need;
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

int launch_score_dense(pars_ctx* ctx, const FeatConfig& c, int mode, const double* X, int64_t n,
                       const double* w64, const float* w32, double bias, double* scores,
                       cudaStream_t st) {
  if (n == 0) return PARS_OK;
  if (mode == PARS_MODE_EXACT_F64) {
    dense_exact_kernel<<<(unsigned)ceil_div(n, 128), 128, 0, st>>>(X, n, c.dim, c.norm, w64, bias,
                                                                   scores);
  } else {
    dense_fast_kernel<<<(unsigned)ceil_div(n * 32, 256), 256, 0, st>>>(X, n, c.dim, c.norm, w32,
                                                                       bias, scores);
  }
  count_launch(ctx);
  PARS_CUDA_CHECK(cudaGetLastError());
  return PARS_OK;
}

}  // namespace pars_b200
