// Dataset ingestion on the GPU: load_dataset (dataset.cpp:73-173) for the
// records of a JSONL dataset file, so prompt texts reach HBM as the arena +
// offsets the featurizer reads without ever becoming std::string records
// (SURVEY §8(f).2).
//
//   1. line split: '\n' counts per 16 KB block (16-byte loads, a SWAR
//      per-byte test), one scan, newline positions;
//   2. non-empty lines in file order, truncated to `limit` records
//      (dataset.cpp:98-100: empty lines are skipped, the limit is checked
//      before a line is parsed);
//   3. one thread per record line validates it with JSON's grammar exactly as
//      nlohmann::json::parse does (strings: UTF-8, escapes, surrogate pairs,
//      no raw control characters; numbers: JSON grammar, integers vs floats;
//      literals; nesting; last duplicate key wins) and the record checks of
//      dataset.cpp:107-168 (id non-empty string, prompt string, positive
//      integer output_len / prompt_len / samples, output_len == median of the
//      samples), recording the spans of id and prompt and the integer fields;
//   4. duplicate ids through a device hash table keyed by the ids' FNV-1a
//      hash: every line whose id appeared on an earlier line is a duplicate;
//   5. decoded lengths, scans, and a warp per record writes the decoded
//      prompt (and id) bytes into the arenas; prompt_len defaults to the
//      whitespace token count (dataset.cpp:32-44).
// Errors: the first failing line in file order is what the reference
// reports; the host re-derives that one line's message (capi.cu).
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdint>

#include "common.cuh"
#include "ingest.cuh"

namespace pars_b200 {

namespace {

constexpr int kLineThreads = 256;
constexpr int kLineVec = 4;                                // 16-byte loads per thread
constexpr int kBlockBytes = kLineThreads * kLineVec * 16;  // bytes per line-split block (16 KB)
constexpr int kScanThreads = 256;
constexpr int kScanItems = 8;
constexpr int kScanTile = kScanThreads * kScanItems;

// 16-bit mask of the '\n' bytes among the 16 at p0 (zeros past n); the
// per-byte zero test ((b & 0x7f) + 0x7f) | b has no cross-byte carries
__device__ __forceinline__ uint32_t nl_mask16(const uint8_t* __restrict__ b, int64_t p0, int64_t n) {
  uint32_t w[4];
  if (p0 + 16 <= n) {
    const uint4 v = __ldg(reinterpret_cast<const uint4*>(b + p0));
    w[0] = v.x; w[1] = v.y; w[2] = v.z; w[3] = v.w;
  } else {
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      uint32_t x = 0;
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        const int64_t q = p0 + 4 * k + j;
        x |= (uint32_t)(q < n ? b[q] : 0u) << (8 * j);
      }
      w[k] = x;
    }
  }
  uint32_t m = 0;
#pragma unroll
  for (int k = 0; k < 4; ++k) {
    const uint32_t t = w[k] ^ 0x0a0a0a0au;
    const uint32_t z = ~(((t & 0x7f7f7f7fu) + 0x7f7f7f7fu) | t) & 0x80808080u;  // bit 7 per '\n'
    // gather bits 7, 15, 23, 31 into 4 consecutive bits
    m |= (((z >> 7) * 0x204081u) >> 21 & 0xfu) << (4 * k);
  }
  return p0 < n ? m : 0u;
}

__global__ void __launch_bounds__(kLineThreads) nl_count_kernel(const uint8_t* __restrict__ b,
                                                                int64_t n, uint32_t* __restrict__ cnt) {
  const int64_t p0 = (int64_t)blockIdx.x * kBlockBytes + threadIdx.x * 16;
  uint32_t c = 0;
#pragma unroll
  for (int v = 0; v < kLineVec; ++v) c += __popc(nl_mask16(b, p0 + (int64_t)v * kLineThreads * 16, n));
  c = __reduce_add_sync(0xffffffffu, c);
  __shared__ uint32_t ws[kLineThreads / 32];
  if ((threadIdx.x & 31) == 0) ws[threadIdx.x >> 5] = c;
  __syncthreads();
  if (threadIdx.x == 0) {
    uint32_t t = 0;
    for (int w = 0; w < kLineThreads / 32; ++w) t += ws[w];
    cnt[blockIdx.x] = t;
  }
}

// newline positions in file order: the block's 16-byte groups are visited
// group-major (v, then thread), which is byte order within the block
__global__ void __launch_bounds__(kLineThreads) nl_write_kernel(const uint8_t* __restrict__ b,
                                                                int64_t n,
                                                                const uint32_t* __restrict__ boff,
                                                                int64_t* __restrict__ nl) {
  __shared__ uint32_t warp_tot[kLineThreads / 32];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  uint32_t base = boff[blockIdx.x];
#pragma unroll
  for (int v = 0; v < kLineVec; ++v) {
    const int64_t p0 = (int64_t)blockIdx.x * kBlockBytes + ((int64_t)v * kLineThreads + threadIdx.x) * 16;
    uint32_t m = nl_mask16(b, p0, n);
    const uint32_t c = __popc(m);
    uint32_t x = c;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const uint32_t y = __shfl_up_sync(0xffffffffu, x, o);
      if (lane >= o) x += y;
    }
    if (lane == 31) warp_tot[warp] = x;
    __syncthreads();
    uint32_t pos = base + x - c, tot = 0;
    for (int w = 0; w < kLineThreads / 32; ++w) {
      const uint32_t t = warp_tot[w];
      if (w < warp) pos += t;
      tot += t;
    }
    for (; m; m &= m - 1) nl[pos++] = p0 + __ffs(m) - 1;
    base += tot;
    __syncthreads();
  }
}

// Exclusive scan in three passes (tile sums, one CTA over the sums, tiles
// with their offsets); the total lands at v[n].
template <typename T>
__global__ void __launch_bounds__(kScanThreads) scan_tile_sum_kernel(const T* __restrict__ v, int64_t n,
                                                                     T* __restrict__ part) {
  __shared__ T ws[kScanThreads / 32];
  const int64_t base = (int64_t)blockIdx.x * kScanTile;
  T s = 0;
#pragma unroll
  for (int k = 0; k < kScanItems; ++k) {
    const int64_t i = base + k * kScanThreads + threadIdx.x;
    if (i < n) s += v[i];
  }
#pragma unroll
  for (int o = 16; o; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
  if ((threadIdx.x & 31) == 0) ws[threadIdx.x >> 5] = s;
  __syncthreads();
  if (threadIdx.x == 0) {
    T t = 0;
    for (int w = 0; w < kScanThreads / 32; ++w) t += ws[w];
    part[blockIdx.x] = t;
  }
}

template <typename T>
__global__ void __launch_bounds__(1024) scan_parts_kernel(T* __restrict__ part, int64_t nb,
                                                          T* __restrict__ total) {
  __shared__ T sh[1024];
  const int t = threadIdx.x;
  const int64_t per = (nb + 1023) / 1024;
  const int64_t a = t * per, e = a + per < nb ? a + per : nb;
  T s = 0;
  for (int64_t k = a; k < e; ++k) s += part[k];
  sh[t] = s;
  __syncthreads();
  for (int o = 1; o < 1024; o <<= 1) {
    const T x = t >= o ? sh[t - o] : (T)0;
    __syncthreads();
    sh[t] += x;
    __syncthreads();
  }
  T run = sh[t] - s;
  for (int64_t k = a; k < e; ++k) {
    const T c = part[k];
    part[k] = run;
    run += c;
  }
  if (t == 1023) *total = sh[1023];
}

template <typename T>
__global__ void __launch_bounds__(kScanThreads) scan_tile_apply_kernel(T* __restrict__ v, int64_t n,
                                                                       const T* __restrict__ part) {
  __shared__ T sh[kScanTile];
  __shared__ T ws[kScanThreads / 32];
  const int64_t base = (int64_t)blockIdx.x * kScanTile;
#pragma unroll
  for (int k = 0; k < kScanItems; ++k) {
    const int j = k * kScanThreads + threadIdx.x;
    sh[j] = base + j < n ? v[base + j] : (T)0;
  }
  __syncthreads();
  T loc[kScanItems];
  T s = 0;
#pragma unroll
  for (int k = 0; k < kScanItems; ++k) {
    loc[k] = s;
    s += sh[threadIdx.x * kScanItems + k];
  }
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  T x = s;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const T y = __shfl_up_sync(0xffffffffu, x, o);
    if (lane >= o) x += y;
  }
  if (lane == 31) ws[warp] = x;
  __syncthreads();
  T off = part[blockIdx.x] + x - s;
  for (int w = 0; w < warp; ++w) off += ws[w];
#pragma unroll
  for (int k = 0; k < kScanItems; ++k) sh[threadIdx.x * kScanItems + k] = off + loc[k];
  __syncthreads();
#pragma unroll
  for (int k = 0; k < kScanItems; ++k) {
    const int j = k * kScanThreads + threadIdx.x;
    if (base + j < n) v[base + j] = sh[j];
  }
}

template <typename T>
void launch_scan(T* v, int64_t n, void* scratch, cudaStream_t st) {
  const int64_t nb = std::max<int64_t>(1, ceil_div(n, kScanTile));
  T* part = static_cast<T*>(scratch);
  scan_tile_sum_kernel<T><<<(unsigned)nb, kScanThreads, 0, st>>>(v, n, part);
  scan_parts_kernel<T><<<1, 1024, 0, st>>>(part, nb, v + n);
  scan_tile_apply_kernel<T><<<(unsigned)nb, kScanThreads, 0, st>>>(v, n, part);
}

// line i = [start, end): start = nl[i-1] + 1 (0 for i = 0), end = nl[i] (n for
// the last line when the file does not end with '\n'); flag non-empty lines
__global__ void line_flags_kernel(const int64_t* __restrict__ nl, int64_t nlines, int64_t n,
                                  uint32_t* __restrict__ nonempty) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= nlines) return;
  const int64_t s = i == 0 ? 0 : nl[i - 1] + 1;
  const int64_t e = nl[i] < n ? nl[i] : n;
  nonempty[i] = e > s ? 1u : 0u;
}

__global__ void record_lines_kernel(const int64_t* __restrict__ nl, int64_t nlines, int64_t n,
                                    const uint32_t* __restrict__ rank, int64_t limit,
                                    int64_t* __restrict__ rb, int64_t* __restrict__ re,
                                    int64_t* __restrict__ rline) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= nlines) return;
  const int64_t s = i == 0 ? 0 : nl[i - 1] + 1;
  const int64_t e = nl[i] < n ? nl[i] : n;
  if (e <= s) return;
  const int64_t r = rank[i];
  if (r >= limit) return;
  rb[r] = s;
  re[r] = e;
  rline[r] = i;
}

// ---- JSON scanning (nlohmann::json::parse semantics) ----------------------
struct Cur {
  const uint8_t* p;
  int64_t i, e;
  __device__ int peek() const { return i < e ? (int)p[i] : -1; }
};

__device__ __forceinline__ void skip_ws(Cur& c) {
  while (c.i < c.e) {
    const uint8_t ch = c.p[c.i];
    if (ch == ' ' || ch == '\t' || ch == '\n' || ch == '\r')
      ++c.i;
    else
      break;
  }
}

__device__ __forceinline__ int hexval(int ch) {
  if (ch >= '0' && ch <= '9') return ch - '0';
  if (ch >= 'a' && ch <= 'f') return ch - 'a' + 10;
  if (ch >= 'A' && ch <= 'F') return ch - 'A' + 10;
  return -1;
}

__device__ __forceinline__ int read_u4(Cur& c) {  // after "\u"
  if (c.i + 4 > c.e) return -1;
  int v = 0;
  for (int k = 0; k < 4; ++k) {
    const int h = hexval(c.p[c.i + k]);
    if (h < 0) return -1;
    v = (v << 4) | h;
  }
  c.i += 4;
  return v;
}

// A string starting at the opening quote. On success: [sb, se) is the raw
// content, esc = it contains escapes, dlen = decoded byte length.
// With `tok`, also the whitespace-token count of the DECODED string
// (whitespace_token_count, dataset.cpp:32-44: C-locale isspace bytes).
__device__ bool scan_string(Cur& c, int64_t& sb, int64_t& se, bool& esc, int64_t& dlen,
                            int64_t* tok = nullptr) {
  if (c.peek() != '"') return false;
  ++c.i;
  sb = c.i;
  esc = false;
  dlen = 0;
  int64_t tk = 0;
  bool prev_sp = true;
  auto note = [&](uint32_t d) {  // one decoded byte
    const bool sp = d == 0x20u || (d >= 9u && d <= 13u);
    tk += (!sp && prev_sp) ? 1 : 0;
    prev_sp = sp;
  };
  while (c.i < c.e) {
    // fast path: 8 bytes at a time while they are plain ASCII (no quote,
    // backslash, control character or byte >= 0x80); the first special byte
    // (exact: the lowest flagged byte of the haszero tests) goes the slow way
    if (c.i + 16 <= c.e) {
      const uintptr_t addr = reinterpret_cast<uintptr_t>(c.p + c.i);
      const uint64_t* a = reinterpret_cast<const uint64_t*>(addr & ~(uintptr_t)7);
      const unsigned off = (unsigned)(addr & 7) * 8;
      const uint64_t lo = a[0], hi = a[1];
      const uint64_t x = off ? (lo >> off) | (hi << (64 - off)) : lo;
      constexpr uint64_t k01 = 0x0101010101010101ull, k80 = 0x8080808080808080ull;
      const uint64_t q = x ^ (k01 * '"'), bs = x ^ (k01 * '\\');
      const uint64_t special = (((x - k01 * 0x20) & ~x) | ((q - k01) & ~q) | ((bs - k01) & ~bs) |
                                x) & k80;
      const int plain = special == 0 ? 8 : __ffsll((long long)special) / 8 - 1;
      if (tok && plain) {
        // plain bytes hold no control characters: the only whitespace is ' '
        constexpr uint64_t k7f = 0x7f7f7f7f7f7f7f7full;
        const uint64_t t = x ^ (k01 * 0x20);
        const uint64_t ns = (((t & k7f) + k7f) | t) & k80;  // bit 7: byte != ' '
        const uint64_t lim = plain == 8 ? ~0ull : ((1ull << (8 * plain)) - 1);
        const uint64_t prev = (ns << 8) | (prev_sp ? 0ull : 0x80ull);
        tk += __popcll(ns & ~prev & lim);
        prev_sp = ((ns >> (8 * plain - 1)) & 1ull) == 0;
      }
      c.i += plain;
      dlen += plain;
      if (special == 0) continue;
    }
    const uint32_t ch = c.p[c.i];
    if (ch == '"') {
      se = c.i;
      ++c.i;
      if (tok) *tok = tk;
      return true;
    }
    if (ch < 0x20) return false;  // control characters must be escaped
    if (ch == '\\') {
      esc = true;
      ++c.i;
      if (c.i >= c.e) return false;
      const uint32_t x = c.p[c.i++];
      if (x == '"' || x == '\\' || x == '/' || x == 'b' || x == 'f' || x == 'n' || x == 'r' ||
          x == 't') {
        dlen += 1;
        note(x == 'b' ? 8u : x == 'f' ? 12u : x == 'n' ? 10u : x == 'r' ? 13u : x == 't' ? 9u : x);
      } else if (x == 'u') {
        int cp = read_u4(c);
        if (cp < 0) return false;
        if (cp >= 0xD800 && cp <= 0xDBFF) {  // high surrogate: a low one must follow
          if (c.i + 2 > c.e || c.p[c.i] != '\\' || c.p[c.i + 1] != 'u') return false;
          c.i += 2;
          const int lo = read_u4(c);
          if (lo < 0xDC00 || lo > 0xDFFF) return false;
          dlen += 4;
          note(0x80u);
        } else if (cp >= 0xDC00 && cp <= 0xDFFF) {
          return false;
        } else {
          dlen += cp < 0x80 ? 1 : (cp < 0x800 ? 2 : 3);
          note(cp < 0x80 ? (uint32_t)cp : 0x80u);
        }
      } else {
        return false;
      }
      continue;
    }
    // UTF-8 (the ranges nlohmann's lexer accepts)
    int more = 0;
    uint32_t lo = 0x80, hi = 0xBF;
    if (ch < 0x80) {
      more = 0;
    } else if (ch >= 0xC2 && ch <= 0xDF) {
      more = 1;
    } else if (ch == 0xE0) {
      more = 2;
      lo = 0xA0;
    } else if ((ch >= 0xE1 && ch <= 0xEC) || ch == 0xEE || ch == 0xEF) {
      more = 2;
    } else if (ch == 0xED) {
      more = 2;
      hi = 0x9F;
    } else if (ch == 0xF0) {
      more = 3;
      lo = 0x90;
    } else if (ch >= 0xF1 && ch <= 0xF3) {
      more = 3;
    } else if (ch == 0xF4) {
      more = 3;
      hi = 0x8F;
    } else {
      return false;
    }
    ++c.i;
    for (int k = 0; k < more; ++k) {
      if (c.i >= c.e) return false;
      const uint32_t cc = c.p[c.i];
      const uint32_t l = k == 0 ? lo : 0x80, h = k == 0 ? hi : 0xBF;
      if (cc < l || cc > h) return false;
      ++c.i;
    }
    dlen += 1 + more;
    note(more ? 0x80u : ch);
  }
  return false;  // unterminated
}

// A number per JSON's grammar. is_int: no fraction/exponent (nlohmann's
// number_integer/unsigned); val: its value when it is an integer in
// [-2^63, 2^63-1], with `big` set when it is beyond int64's range.
__device__ bool scan_number(Cur& c, bool& is_int, int64_t& val, bool& big) {
  bool neg = false;
  if (c.peek() == '-') {
    neg = true;
    ++c.i;
  }
  const int d0 = c.peek();
  if (d0 < '0' || d0 > '9') return false;
  is_int = true;
  big = false;
  uint64_t u = 0;
  if (d0 == '0') {
    ++c.i;
  } else {
    while (c.i < c.e && c.p[c.i] >= '0' && c.p[c.i] <= '9') {
      const uint64_t dgt = c.p[c.i] - '0';
      if (u > (0xffffffffffffffffull - dgt) / 10ull) big = true;
      u = u * 10ull + dgt;
      ++c.i;
    }
  }
  if (c.peek() == '.') {
    is_int = false;
    ++c.i;
    const int d = c.peek();
    if (d < '0' || d > '9') return false;
    while (c.i < c.e && c.p[c.i] >= '0' && c.p[c.i] <= '9') ++c.i;
  }
  if (c.peek() == 'e' || c.peek() == 'E') {
    is_int = false;
    ++c.i;
    if (c.peek() == '+' || c.peek() == '-') ++c.i;
    const int d = c.peek();
    if (d < '0' || d > '9') return false;
    while (c.i < c.e && c.p[c.i] >= '0' && c.p[c.i] <= '9') ++c.i;
  }
  if (is_int) {
    if (!big && (neg ? u > 0x8000000000000000ull : u > 0x7fffffffffffffffull)) big = true;
    val = big ? 0 : (neg ? (int64_t)(0 - u) : (int64_t)u);
  }
  return true;
}

__device__ bool scan_literal(Cur& c, const char* w, int len) {
  if (c.i + len > c.e) return false;
  for (int k = 0; k < len; ++k)
    if (c.p[c.i + k] != (uint8_t)w[k]) return false;
  c.i += len;
  return true;
}

// Any JSON value (validated, skipped); containers by an explicit bit stack.
__device__ bool skip_value(Cur& c) {
  uint64_t stack = 0;  // bit d: container at depth d is an array
  int depth = 0;
  bool expect_value = true;
  for (;;) {
    skip_ws(c);
    if (expect_value) {
      const int ch = c.peek();
      if (ch == '{') {
        if (depth == 64) return false;
        ++c.i;
        stack &= ~(1ull << depth);
        ++depth;
        skip_ws(c);
        if (c.peek() == '}') {
          ++c.i;
          --depth;
          expect_value = false;
        } else {
          int64_t sb, se, dl;
          bool esc;
          if (!scan_string(c, sb, se, esc, dl)) return false;
          skip_ws(c);
          if (c.peek() != ':') return false;
          ++c.i;
          continue;  // a value follows
        }
      } else if (ch == '[') {
        if (depth == 64) return false;
        ++c.i;
        stack |= 1ull << depth;
        ++depth;
        skip_ws(c);
        if (c.peek() == ']') {
          ++c.i;
          --depth;
          expect_value = false;
        } else {
          continue;
        }
      } else if (ch == '"') {
        int64_t sb, se, dl;
        bool esc;
        if (!scan_string(c, sb, se, esc, dl)) return false;
        expect_value = false;
      } else if (ch == 't') {
        if (!scan_literal(c, "true", 4)) return false;
        expect_value = false;
      } else if (ch == 'f') {
        if (!scan_literal(c, "false", 5)) return false;
        expect_value = false;
      } else if (ch == 'n') {
        if (!scan_literal(c, "null", 4)) return false;
        expect_value = false;
      } else {
        bool ii, big;
        int64_t v;
        if (!scan_number(c, ii, v, big)) return false;
        expect_value = false;
      }
    }
    if (depth == 0) return true;
    // after a value inside a container: ',' or the closer
    skip_ws(c);
    const bool arr = (stack >> (depth - 1)) & 1ull;
    const int ch = c.peek();
    if (ch == ',') {
      ++c.i;
      if (!arr) {  // object: next key
        skip_ws(c);
        int64_t sb, se, dl;
        bool esc;
        if (!scan_string(c, sb, se, esc, dl)) return false;
        skip_ws(c);
        if (c.peek() != ':') return false;
        ++c.i;
      }
      expect_value = true;
    } else if (ch == (arr ? ']' : '}')) {
      ++c.i;
      --depth;
      expect_value = false;
      if (depth == 0) return true;
    } else {
      return false;
    }
  }
}

__device__ __forceinline__ bool key_is(const Cur& c, int64_t sb, int64_t se, bool esc, const char* k,
                                       int len) {
  if (esc || se - sb != len) return false;  // field names never need escapes
  for (int j = 0; j < len; ++j)
    if (c.p[sb + j] != (uint8_t)k[j]) return false;
  return true;
}

}  // namespace

__global__ void parse_records_kernel(const uint8_t* __restrict__ text, const int64_t* __restrict__ rb,
                                     const int64_t* __restrict__ re, int64_t nrec, RecordOut out) {
  const int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (r >= nrec) return;
  Cur c{text, rb[r], re[r]};
  uint32_t err = kIngOk;
  int64_t id_b = 0, id_e = 0, pr_b = 0, pr_e = 0, id_dl = 0, pr_dl = 0, pr_tk = 0, ol = -1, pl = -1;
  int64_t sm_b = -1, sm_e = -1;
  uint32_t flags = 0;
  // which fields are present, and whether each is well-typed
  bool has_id = false, id_ok = false, has_pr = false, pr_ok = false, has_ol = false, ol_ok = false;
  bool has_pl = false, pl_ok = false, has_sm = false, sm_ok = false, has_emb = false;
  skip_ws(c);
  if (c.peek() != '{') {
    // valid JSON but not an object, or malformed
    Cur d = c;
    err = (skip_value(d) && (skip_ws(d), d.i == d.e)) ? kIngNotObject : kIngMalformed;
  } else {
    ++c.i;
    skip_ws(c);
    bool ok = true;
    if (c.peek() == '}') {
      ++c.i;
    } else {
      for (;;) {
        skip_ws(c);
        int64_t kb, ke, kd;
        bool kesc;
        if (!scan_string(c, kb, ke, kesc, kd)) {
          ok = false;
          break;
        }
        skip_ws(c);
        if (c.peek() != ':') {
          ok = false;
          break;
        }
        ++c.i;
        skip_ws(c);
        const int64_t v0 = c.i;
        // the value, validated; typed capture for the fields we read (a later
        // duplicate key replaces an earlier one, as in nlohmann)
        const int ch = c.peek();
        if (key_is(c, kb, ke, kesc, "id", 2) || key_is(c, kb, ke, kesc, "prompt", 6)) {
          const bool is_id = ke - kb == 2;
          bool typed = false;
          if (ch == '"') {
            int64_t sb, se, dl, tk = 0;
            bool esc;
            if (!scan_string(c, sb, se, esc, dl, is_id ? nullptr : &tk)) {
              ok = false;
              break;
            }
            typed = true;
            if (is_id) {
              id_b = sb, id_e = se, id_dl = dl;
              flags = esc ? (flags | kIngIdEsc) : (flags & ~kIngIdEsc);
            } else {
              pr_b = sb, pr_e = se, pr_dl = dl, pr_tk = tk;
              flags = esc ? (flags | kIngPromptEsc) : (flags & ~kIngPromptEsc);
            }
          } else if (!skip_value(c)) {
            ok = false;
            break;
          }
          if (is_id) {
            has_id = true;
            id_ok = typed && id_dl > 0;
          } else {
            has_pr = true;
            pr_ok = typed;
          }
        } else if (key_is(c, kb, ke, kesc, "output_len", 10) ||
                   key_is(c, kb, ke, kesc, "prompt_len", 10)) {
          const bool is_ol = c.p[kb] == 'o';
          bool good = false;
          int64_t v = 0;
          if (ch == '-' || (ch >= '0' && ch <= '9')) {
            bool ii, big;
            if (!scan_number(c, ii, v, big)) {
              ok = false;
              break;
            }
            good = ii && !big && v >= 1;
          } else if (!skip_value(c)) {
            ok = false;
            break;
          }
          if (is_ol) {
            has_ol = true, ol_ok = good, ol = v;
          } else {
            has_pl = true, pl_ok = good, pl = v;
          }
        } else if (key_is(c, kb, ke, kesc, "output_len_samples", 18)) {
          has_sm = true;
          sm_ok = false;
          if (ch == '[') {
            // a non-empty array of positive integers
            Cur d = c;
            ++d.i;
            skip_ws(d);
            bool good = d.peek() != ']';
            bool fine = true;
            while (good) {
              skip_ws(d);
              const int x = d.peek();
              if (x == '-' || (x >= '0' && x <= '9')) {
                bool ii, big;
                int64_t v;
                if (!scan_number(d, ii, v, big)) {
                  fine = false;
                  break;
                }
                if (!(ii && !big && v >= 1)) good = false;
              } else {
                good = false;
                break;
              }
              skip_ws(d);
              if (d.peek() == ',') {
                ++d.i;
                continue;
              }
              if (d.peek() == ']') break;
              good = false;
            }
            (void)fine;
            // validate (and skip) the whole array with the generic scanner
            if (!skip_value(c)) {
              ok = false;
              break;
            }
            sm_ok = good;
            sm_b = v0;
            sm_e = c.i;
          } else if (!skip_value(c)) {
            ok = false;
            break;
          }
        } else if (key_is(c, kb, ke, kesc, "embedding", 9)) {
          has_emb = true;
          if (!skip_value(c)) {
            ok = false;
            break;
          }
        } else if (!skip_value(c)) {
          ok = false;
          break;
        }
        skip_ws(c);
        if (c.peek() == ',') {
          ++c.i;
          continue;
        }
        if (c.peek() == '}') {
          ++c.i;
          break;
        }
        ok = false;
        break;
      }
    }
    if (ok) {
      skip_ws(c);
      if (c.i != c.e) ok = false;  // trailing characters
    }
    if (!ok) {
      err = kIngMalformed;
    } else if (!(has_id && id_ok)) {
      err = kIngBadId;
    } else if (!(has_pr && pr_ok)) {
      err = kIngBadPrompt;
    } else if (has_sm && !sm_ok) {
      err = kIngBadSamples;
    } else if (has_ol && !ol_ok) {
      err = kIngBadOutputLen;
    } else if (!has_ol && !has_sm) {
      err = kIngMissingOutputLen;
    } else if (has_emb) {
      err = kIngEmbedding;  // the GPU loader does not parse embedding arrays
    } else if (has_pl && !pl_ok) {
      err = kIngBadPromptLen;
    }
  }
  out.err[r] = err;
  out.flags[r] = flags | (has_sm ? kIngHasSamples : 0u) | (has_ol ? kIngHasOutputLen : 0u);
  if (has_sm && out.any_samples) atomicOr(out.any_samples, 1u);  // the host exports them
  out.id_b[r] = id_b;
  out.id_e[r] = id_e;
  out.id_len[r] = id_dl;
  out.pr_b[r] = pr_b;
  out.pr_e[r] = pr_e;
  out.pr_len[r] = pr_dl;
  out.pr_tok[r] = pr_tk;
  out.out_len[r] = ol;
  out.prompt_len[r] = pl;
  out.sm_b[r] = sm_b;
  out.sm_e[r] = sm_e;
}

namespace {

// Decoded string bytes of a raw span (escapes resolved, UTF-8 for \u).
__device__ void decode_string(const uint8_t* __restrict__ p, int64_t b, int64_t e, uint8_t* __restrict__ o) {
  int64_t w = 0;
  for (int64_t i = b; i < e;) {
    const uint8_t ch = p[i];
    if (ch != '\\') {
      o[w++] = ch;
      ++i;
      continue;
    }
    const uint8_t x = p[i + 1];
    i += 2;
    switch (x) {
      case 'b': o[w++] = '\b'; break;
      case 'f': o[w++] = '\f'; break;
      case 'n': o[w++] = '\n'; break;
      case 'r': o[w++] = '\r'; break;
      case 't': o[w++] = '\t'; break;
      case 'u': {
        uint32_t cp = 0;
        for (int k = 0; k < 4; ++k) cp = (cp << 4) | (uint32_t)hexval(p[i + k]);
        i += 4;
        if (cp >= 0xD800 && cp <= 0xDBFF) {
          uint32_t lo = 0;
          for (int k = 0; k < 4; ++k) lo = (lo << 4) | (uint32_t)hexval(p[i + 2 + k]);
          i += 6;
          cp = 0x10000 + ((cp - 0xD800) << 10) + (lo - 0xDC00);
        }
        if (cp < 0x80) {
          o[w++] = (uint8_t)cp;
        } else if (cp < 0x800) {
          o[w++] = (uint8_t)(0xC0 | (cp >> 6));
          o[w++] = (uint8_t)(0x80 | (cp & 0x3F));
        } else if (cp < 0x10000) {
          o[w++] = (uint8_t)(0xE0 | (cp >> 12));
          o[w++] = (uint8_t)(0x80 | ((cp >> 6) & 0x3F));
          o[w++] = (uint8_t)(0x80 | (cp & 0x3F));
        } else {
          o[w++] = (uint8_t)(0xF0 | (cp >> 18));
          o[w++] = (uint8_t)(0x80 | ((cp >> 12) & 0x3F));
          o[w++] = (uint8_t)(0x80 | ((cp >> 6) & 0x3F));
          o[w++] = (uint8_t)(0x80 | (cp & 0x3F));
        }
        break;
      }
      default: o[w++] = x; break;  // " \ /
    }
  }
}

}  // namespace

// Warp copy of len raw bytes to an arbitrarily aligned destination: byte
// head up to 4-byte alignment of dst, then one 4-byte store per lane per
// step (each assembled from two aligned source words with a funnel shift;
// the source buffer is padded so the second word may pass its end), then
// the byte tail.
__device__ __forceinline__ void warp_copy(const uint8_t* __restrict__ src, uint8_t* __restrict__ dst,
                                          int64_t len, int lane) {
  const int64_t h4 = (int64_t)((4u - ((uint32_t)(uintptr_t)dst & 3u)) & 3u);
  const int64_t head = len < h4 ? len : h4;
  if (lane < head) dst[lane] = src[lane];
  const int64_t nw = (len - head) >> 2;
  const uint8_t* s0 = src + head;
  uint32_t* d0 = reinterpret_cast<uint32_t*>(dst + head);
  const uint32_t sh = ((uint32_t)(uintptr_t)s0 & 3u) * 8u;
  const uint32_t* a0 = reinterpret_cast<const uint32_t*>((uintptr_t)s0 & ~(uintptr_t)3);
  for (int64_t q = lane; q < nw; q += 32) {
    const uint32_t lo = a0[q], hi = a0[q + 1];
    d0[q] = sh ? __funnelshift_r(lo, hi, sh) : lo;
  }
  for (int64_t k = head + nw * 4 + lane; k < len; k += 32) dst[k] = src[k];
}

// One warp per record: copy (or decode) the prompt and the id into their
// arenas; prompt_len defaults to the whitespace token count of the decoded
// prompt (dataset.cpp:32-44), counted by the parser.
__global__ void emit_records_kernel(const uint8_t* __restrict__ text, int64_t nrec, RecordOut rec,
                                    const int64_t* __restrict__ pr_off, uint8_t* __restrict__ arena,
                                    const int64_t* __restrict__ id_off, uint8_t* __restrict__ ids,
                                    int64_t* __restrict__ tokens) {
  const int lane = threadIdx.x & 31;
  const int64_t r = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  if (r >= nrec) return;
  const uint32_t fl = rec.flags[r];
  uint8_t* dst = arena + pr_off[r];
  const int64_t len = pr_off[r + 1] - pr_off[r];
  if (len == 0) {
    // nothing to copy (an empty prompt, or a record that failed before it)
  } else if (fl & kIngPromptEsc) {
    if (lane == 0) decode_string(text, rec.pr_b[r], rec.pr_e[r], dst);
  } else {
    warp_copy(text + rec.pr_b[r], dst, len, lane);
  }
  uint8_t* idd = ids + id_off[r];
  if (id_off[r + 1] == id_off[r]) {
    // a record whose id did not parse
  } else if (fl & kIngIdEsc) {
    if (lane == 0) decode_string(text, rec.id_b[r], rec.id_e[r], idd);
  } else {
    const uint8_t* src = text + rec.id_b[r];
    for (int64_t k = lane; k < id_off[r + 1] - id_off[r]; k += 32) idd[k] = src[k];
  }
  if (lane == 0) tokens[r] = rec.prompt_len[r] < 0 ? (len ? rec.pr_tok[r] : 0) : rec.prompt_len[r];
}

// Duplicate ids: open addressing on the 64-bit FNV-1a of the decoded id
// bytes; each slot keeps the smallest record index with that hash. A record
// is a duplicate when an EARLIER record has the same id bytes (hash equal,
// then compared byte by byte).
__device__ __forceinline__ uint64_t fnv_bytes(const uint8_t* p, int64_t n) {
  uint64_t h = 0xcbf29ce484222325ull;
  for (int64_t k = 0; k < n; ++k) h = (h ^ p[k]) * 0x100000001b3ull;
  return h;
}

__global__ void id_hash_kernel(const uint8_t* __restrict__ ids, const int64_t* __restrict__ id_off,
                               int64_t nrec, uint64_t* __restrict__ hash) {
  const int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (r < nrec) hash[r] = fnv_bytes(ids + id_off[r], id_off[r + 1] - id_off[r]);
}

__global__ void id_insert_kernel(const uint64_t* __restrict__ hash, int64_t nrec, uint64_t cap,
                                 unsigned long long* __restrict__ tkey, unsigned long long* __restrict__ tmin) {
  const int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (r >= nrec) return;
  const unsigned long long h = hash[r] | 1ull;  // 0 = empty slot
  uint64_t s = (h >> 7) & (cap - 1);
  for (;;) {
    const unsigned long long prev = atomicCAS(&tkey[s], 0ull, h);
    if (prev == 0ull || prev == h) {
      atomicMin(&tmin[s], (unsigned long long)r);
      return;
    }
    s = (s + 1) & (cap - 1);
  }
}

// a record is a duplicate if some earlier record with the same hash has the
// same bytes; the earliest record of a hash is never a duplicate
__global__ void id_dup_kernel(const uint64_t* __restrict__ hash, const uint8_t* __restrict__ ids,
                              const int64_t* __restrict__ id_off, int64_t nrec, uint64_t cap,
                              const unsigned long long* __restrict__ tkey,
                              const unsigned long long* __restrict__ tmin, uint32_t* __restrict__ dup) {
  const int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (r >= nrec) return;
  const unsigned long long h = hash[r] | 1ull;
  uint64_t s = (h >> 7) & (cap - 1);
  while (tkey[s] != h) s = (s + 1) & (cap - 1);
  const int64_t first = (int64_t)tmin[s];
  if (first == r) return;
  // same hash seen earlier: scan earlier records with this hash for equal bytes
  // (hash collisions between different ids are astronomically rare; the scan
  // only runs for records that share a hash)
  const int64_t n = id_off[r + 1] - id_off[r];
  const uint8_t* a = ids + id_off[r];
  for (int64_t q = first; q < r; ++q) {
    if (hash[q] != hash[r] || id_off[q + 1] - id_off[q] != n) continue;
    const uint8_t* b = ids + id_off[q];
    bool eq = true;
    for (int64_t k = 0; k < n && eq; ++k) eq = a[k] == b[k];
    if (eq) {
      dup[r] = 1u;
      return;
    }
  }
}

// median_floor (dataset.cpp:46-52) of each record's samples: the integers
// of the validated array, insertion-sorted in thread-local storage.
constexpr int kMaxSamples = 256;

__global__ void samples_kernel(const uint8_t* __restrict__ text, int64_t nrec, RecordOut rec,
                               uint32_t* __restrict__ mismatch, uint32_t* __restrict__ unsup) {
  const int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (r >= nrec || rec.err[r] != kIngOk || !(rec.flags[r] & kIngHasSamples)) return;
  int64_t v[kMaxSamples];
  int n = 0;
  for (int64_t i = rec.sm_b[r] + 1; i < rec.sm_e[r];) {
    const uint8_t ch = text[i];
    if (ch >= '0' && ch <= '9') {
      int64_t x = 0;
      while (i < rec.sm_e[r] && text[i] >= '0' && text[i] <= '9') x = x * 10 + (text[i++] - '0');
      if (n == kMaxSamples) {
        unsup[r] = 1u;
        return;
      }
      int k = n++;
      while (k > 0 && v[k - 1] > x) {
        v[k] = v[k - 1];
        --k;
      }
      v[k] = x;
    } else {
      ++i;
    }
  }
  const int64_t med = (n & 1) ? v[n / 2] : (v[n / 2 - 1] + v[n / 2]) / 2;
  if (rec.flags[r] & kIngHasOutputLen) {
    if (rec.out_len[r] != med) mismatch[r] = 1u;
  } else {
    rec.out_len[r] = med;
  }
}

void ingest_launch_samples(const uint8_t* text, int64_t nrec, const RecordOut& rec,
                           uint32_t* mismatch, uint32_t* unsup, cudaStream_t st) {
  samples_kernel<<<(unsigned)ceil_div(std::max<int64_t>(nrec, 1), 128), 128, 0, st>>>(
      text, nrec, rec, mismatch, unsup);
}

// exclusive scan of n int64 values (one CTA); total at v[n]
// decoded lengths of the records that parsed (others contribute 0)
__global__ void lengths_kernel(int64_t nrec, RecordOut rec, int64_t* __restrict__ pr_len,
                               int64_t* __restrict__ id_len) {
  const int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (r >= nrec) return;
  const uint32_t e = rec.err[r];
  const bool id_ok = e != kIngMalformed && e != kIngNotObject && e != kIngBadId;
  const bool pr_ok = id_ok && e != kIngBadPrompt;
  id_len[r] = id_ok ? rec.id_len[r] : 0;
  pr_len[r] = pr_ok ? rec.pr_len[r] : 0;
}

// the first record that fails any check (file order)
__global__ void first_fail_kernel(int64_t nrec, RecordOut rec, const uint32_t* __restrict__ dup,
                                  const uint32_t* __restrict__ mismatch, const uint32_t* __restrict__ unsup,
                                  const int64_t* __restrict__ tokens, unsigned long long* __restrict__ first) {
  const int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (r >= nrec) return;
  const bool fail = rec.err[r] != kIngOk || dup[r] || mismatch[r] || unsup[r] || tokens[r] < 1;
  if (fail) atomicMin(first, (unsigned long long)r);
}

size_t ingest_scan_scratch_bytes(int64_t n) {
  return (size_t)std::max<int64_t>(1, ceil_div(n, kScanTile)) * 8 + 256;
}

void ingest_launch_scan_i64(int64_t* v, int64_t n, void* scratch, cudaStream_t st) {
  launch_scan<int64_t>(v, n, scratch, st);
}

void ingest_launch_lengths(int64_t nrec, const RecordOut& rec, int64_t* pr_len, int64_t* id_len,
                           cudaStream_t st) {
  lengths_kernel<<<(unsigned)ceil_div(std::max<int64_t>(nrec, 1), 256), 256, 0, st>>>(nrec, rec, pr_len,
                                                                                      id_len);
}

void ingest_launch_first_fail(int64_t nrec, const RecordOut& rec, const uint32_t* dup,
                              const uint32_t* mismatch, const uint32_t* unsup, const int64_t* tokens,
                              unsigned long long* first, cudaStream_t st) {
  first_fail_kernel<<<(unsigned)ceil_div(std::max<int64_t>(nrec, 1), 256), 256, 0, st>>>(
      nrec, rec, dup, mismatch, unsup, tokens, first);
}

int64_t ingest_block_bytes() { return kBlockBytes; }

void ingest_count_newlines_range(const uint8_t* d_text, int64_t n, int64_t b0, int64_t b1,
                                 uint32_t* d_blk, cudaStream_t st) {
  if (b1 <= b0) return;
  const int64_t off = b0 * kBlockBytes;
  nl_count_kernel<<<(unsigned)(b1 - b0), kLineThreads, 0, st>>>(d_text + off, n - off, d_blk + b0);
}

int ingest_scan_newline_blocks(uint32_t* d_blk, int64_t n, int64_t* total, void* scratch,
                               cudaStream_t st) {
  const int64_t nb = std::max<int64_t>(1, ceil_div(n, kBlockBytes));
  launch_scan<uint32_t>(d_blk, nb, scratch, st);
  uint32_t t = 0;
  PARS_CUDA_CHECK(cudaMemcpyAsync(&t, d_blk + nb, 4, cudaMemcpyDeviceToHost, st));
  PARS_CUDA_CHECK(cudaStreamSynchronize(st));
  *total = t;
  return PARS_OK;
}

int ingest_count_newlines(const uint8_t* d_text, int64_t n, uint32_t* d_blk, int64_t* total,
                          void* scratch, cudaStream_t st) {
  const int64_t nb = std::max<int64_t>(1, ceil_div(n, kBlockBytes));
  nl_count_kernel<<<(unsigned)nb, kLineThreads, 0, st>>>(d_text, n, d_blk);
  launch_scan<uint32_t>(d_blk, nb, scratch, st);
  uint32_t t = 0;
  PARS_CUDA_CHECK(cudaMemcpyAsync(&t, d_blk + nb, 4, cudaMemcpyDeviceToHost, st));
  PARS_CUDA_CHECK(cudaStreamSynchronize(st));
  *total = t;
  return PARS_OK;
}

void ingest_write_newlines(const uint8_t* d_text, int64_t n, const uint32_t* d_blk, int64_t* d_nl,
                           cudaStream_t st) {
  const int64_t nb = std::max<int64_t>(1, ceil_div(n, kBlockBytes));
  nl_write_kernel<<<(unsigned)nb, kLineThreads, 0, st>>>(d_text, n, d_blk, d_nl);
}

int64_t ingest_block_count(int64_t n) { return std::max<int64_t>(1, ceil_div(n, kBlockBytes)); }

void ingest_launch_line_flags(const int64_t* nl, int64_t nlines, int64_t n, uint32_t* nonempty,
                              cudaStream_t st) {
  line_flags_kernel<<<(unsigned)ceil_div(std::max<int64_t>(nlines, 1), 256), 256, 0, st>>>(
      nl, nlines, n, nonempty);
}

void ingest_launch_scan(uint32_t* v, int64_t n, void* scratch, cudaStream_t st) {
  launch_scan<uint32_t>(v, n, scratch, st);
}

void ingest_launch_record_lines(const int64_t* nl, int64_t nlines, int64_t n, const uint32_t* rank,
                                int64_t limit, int64_t* rb, int64_t* re, int64_t* rline,
                                cudaStream_t st) {
  record_lines_kernel<<<(unsigned)ceil_div(std::max<int64_t>(nlines, 1), 256), 256, 0, st>>>(
      nl, nlines, n, rank, limit, rb, re, rline);
}

void ingest_launch_parse(const uint8_t* text, const int64_t* rb, const int64_t* re, int64_t nrec,
                         const RecordOut& out, cudaStream_t st) {
  parse_records_kernel<<<(unsigned)ceil_div(std::max<int64_t>(nrec, 1), 128), 128, 0, st>>>(
      text, rb, re, nrec, out);
}

void ingest_launch_emit(const uint8_t* text, int64_t nrec, const RecordOut& rec, const int64_t* pr_off,
                        uint8_t* arena, const int64_t* id_off, uint8_t* ids, int64_t* tokens,
                        cudaStream_t st) {
  emit_records_kernel<<<(unsigned)ceil_div(std::max<int64_t>(nrec, 1) * 32, 256), 256, 0, st>>>(
      text, nrec, rec, pr_off, arena, id_off, ids, tokens);
}

void ingest_launch_dups(const uint8_t* ids, const int64_t* id_off, int64_t nrec, uint64_t* hash,
                        uint64_t cap, unsigned long long* tkey, unsigned long long* tmin,
                        uint32_t* dup, cudaStream_t st) {
  const unsigned g = (unsigned)ceil_div(std::max<int64_t>(nrec, 1), 256);
  id_hash_kernel<<<g, 256, 0, st>>>(ids, id_off, nrec, hash);
  id_insert_kernel<<<g, 256, 0, st>>>(hash, nrec, cap, tkey, tmin);
  id_dup_kernel<<<g, 256, 0, st>>>(hash, ids, id_off, nrec, cap, tkey, tmin, dup);
}

}  // namespace pars_b200
