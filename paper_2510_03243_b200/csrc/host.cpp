// Host-side parts of the hot path that are sequential by construction:
//   * build_pairs (pairs.cpp:8-36): one mt19937_64 stream, draw by draw;
//   * the integer Eq. 1 table dmin[m] (pairs.hpp:21-24 evaluated on host with
//     the reference's own double division, once per (delta, max_len));
//   * tie ranks for the priority key (scheduler.cpp:44-49 tie_key);
//   * the synthetic workload generator (dataset.cpp:204-297 and the C4
//     padding of SURVEY §8(d)) used to produce inputs; bit-identical text.
// Compiled with -ffp-contract=off (the reference objects contain no FMA).
#include <algorithm>
#include <cmath>
#include <cstdarg>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <numeric>
#include <random>
#include <string>
#include <string_view>
#include <vector>

#include <cuda_runtime.h>

#include "pars_cuda.h"

namespace pars_b200 {
void set_error(const char* fmt, ...);
}
using pars_b200::set_error;

namespace {

// The reference's Rng (rng.hpp:22-75): mt19937_64 + hand-coded samplers.
class Rng {
 public:
  explicit Rng(uint64_t seed) : eng_(seed) {}
  uint64_t u64() { return eng_(); }
  double uniform01() { return static_cast<double>(eng_() >> 11) * 0x1.0p-53; }
  uint64_t below(uint64_t n) {
    return static_cast<uint64_t>((static_cast<unsigned __int128>(eng_()) * n) >> 64);
  }
  double exponential(double rate) { return -std::log1p(-uniform01()) / rate; }
  double normal() {
    if (have_spare_) {
      have_spare_ = false;
      return spare_;
    }
    constexpr double kTwoPi = 6.283185307179586476925286766559;
    double u1 = 1.0 - uniform01();
    double u2 = uniform01();
    double r = std::sqrt(-2.0 * std::log(u1));
    double a = kTwoPi * u2;
    spare_ = r * std::sin(a);
    have_spare_ = true;
    return r * std::cos(a);
  }
  template <class T>
  void shuffle(std::vector<T>& v) {
    for (size_t i = v.size(); i > 1; --i) std::swap(v[i - 1], v[below(i)]);
  }

 private:
  std::mt19937_64 eng_;
  double spare_ = 0.0;
  bool have_spare_ = false;
};

inline double rel_diff(int64_t a, int64_t b) {
  return static_cast<double>(std::llabs(a - b)) / static_cast<double>(std::max(a, b));
}

inline void append_u64(std::string& s, uint64_t v) {
  char buf[24];
  int n = 0;
  do {
    buf[n++] = (char)('0' + v % 10);
    v /= 10;
  } while (v);
  while (n) s.push_back(buf[--n]);
}
inline void append_i64(std::string& s, int64_t v) {
  if (v < 0) {
    s.push_back('-');
    append_u64(s, (uint64_t)(-(v + 1)) + 1);
  } else {
    append_u64(s, (uint64_t)v);
  }
}

}  // namespace

struct pars_workload {
  char* text = nullptr;  // pinned when possible
  bool pinned = false;
  int64_t bytes = 0;
  std::vector<int64_t> offsets, output_len, prompt_len;
};

extern "C" {

int64_t pars_build_pairs(const int64_t* lens, int64_t n, double delta, uint64_t max_pairs,
                         uint64_t seed, uint32_t* a, uint32_t* b, int32_t* y, double* rel) {
  if (n <= 0) {
    set_error("build_pairs: empty dataset");
    return PARS_ERR_INVALID;
  }
  if (delta < 0.0 || delta >= 1.0) {
    set_error("build_pairs: delta %g outside [0, 1)", delta);
    return PARS_ERR_INVALID;
  }
  if (max_pairs == 0) {
    set_error("build_pairs: max_pairs must be >= 1");
    return PARS_ERR_INVALID;
  }
  int64_t cnt = 0;
  if (n >= 2) {
    Rng rng(seed);
    const uint64_t budget = 50ull * max_pairs;  // kSamplingBudgetFactor (pairs.hpp:36)
    for (uint64_t draw = 0; draw < budget && (uint64_t)cnt < max_pairs; ++draw) {
      uint32_t i = static_cast<uint32_t>(rng.below((uint64_t)n));
      uint32_t j = static_cast<uint32_t>(rng.below((uint64_t)n - 1));
      if (j >= i) ++j;
      const int64_t la = lens[i], lb = lens[j];
      if (la == lb) continue;
      const double r = rel_diff(la, lb);
      if (r < delta) continue;
      a[cnt] = i;
      b[cnt] = j;
      y[cnt] = la > lb ? 1 : -1;
      if (rel) rel[cnt] = r;
      ++cnt;
    }
  }
  if (cnt == 0) {
    set_error("no informative pairs");
    return PARS_ERR_INVALID;
  }
  return cnt;
}

// PointwiseL1 epoch order (train.cpp:169-172): iota shuffled by Rng(seed).
int pars_pointwise_order(int64_t n, uint64_t seed, uint32_t* order) {
  if (n < 0) {
    set_error("pointwise_order: negative count");
    return PARS_ERR_INVALID;
  }
  std::vector<uint32_t> v(static_cast<size_t>(n));
  for (int64_t i = 0; i < n; ++i) v[i] = static_cast<uint32_t>(i);
  Rng rng(seed);
  rng.shuffle(v);
  std::copy(v.begin(), v.end(), order);
  return PARS_OK;
}

// ListMLE epoch lists (train.cpp:186-200): partial Fisher-Yates on a pool
// that persists across the epoch's lists, each list then ordered longest
// first with the id (unsigned bytes) as tiebreak (sort_by_true_order,
// train.cpp:110-118). lists[nlists * k], k = min(list_size, n).
int pars_listmle_lists(const int64_t* output_len, const char* ids, const int64_t* id_offsets,
                       int64_t n, int64_t nlists, int32_t list_size, uint64_t seed,
                       uint32_t* lists) {
  if (n < 2) {
    set_error("train: listwise needs >= 2 records");
    return PARS_ERR_INVALID;
  }
  if (list_size < 2) {
    set_error("train: list_size must be >= 2");
    return PARS_ERR_INVALID;
  }
  const size_t k = std::min<size_t>(static_cast<size_t>(list_size), static_cast<size_t>(n));
  Rng rng(seed);
  std::vector<uint32_t> pool(static_cast<size_t>(n));
  for (int64_t i = 0; i < n; ++i) pool[i] = static_cast<uint32_t>(i);
  auto id_of = [&](uint32_t r) {
    return std::string_view(ids + id_offsets[r], static_cast<size_t>(id_offsets[r + 1] - id_offsets[r]));
  };
  for (int64_t l = 0; l < nlists; ++l) {
    for (size_t t = 0; t < k; ++t) std::swap(pool[t], pool[t + rng.below(n - t)]);
    uint32_t* list = lists + l * static_cast<int64_t>(k);
    std::copy(pool.begin(), pool.begin() + k, list);
    std::sort(list, list + k, [&](uint32_t a, uint32_t b) {
      if (output_len[a] != output_len[b]) return output_len[a] > output_len[b];
      return id_of(a) < id_of(b);
    });
  }
  return PARS_OK;
}

int pars_length_gap_table(double delta, int64_t max_len, int32_t* dmin) {
  if (max_len < 0) {
    set_error("length gap table: max_len must be >= 0");
    return PARS_ERR_INVALID;
  }
  dmin[0] = INT32_MAX;
  // fl(d/m) is monotone in d: start next to delta*m and walk to the first d
  // with !(relative_length_difference(m, m-d) < delta), exact double compare.
  for (int64_t m = 1; m <= max_len; ++m) {
    int64_t k = std::max<int64_t>(1, (int64_t)std::floor(delta * (double)m) - 1);
    while (k > 1 && !(rel_diff(m, m - (k - 1)) < delta)) --k;
    while (k <= m && rel_diff(m, m - k) < delta) ++k;
    dmin[m] = k <= m ? (int32_t)std::min<int64_t>(k, INT32_MAX - 1) : INT32_MAX;
  }
  return PARS_OK;
}

int pars_tie_ranks(const double* arrival, const char* ids, const int64_t* offs, int64_t n,
                   uint32_t* rank) {
  std::vector<int64_t> o(n);
  std::iota(o.begin(), o.end(), 0);
  auto cmp_id = [&](int64_t a, int64_t b) {
    const int64_t la = offs[a + 1] - offs[a], lb = offs[b + 1] - offs[b];
    int r = std::memcmp(ids + offs[a], ids + offs[b], (size_t)std::min(la, lb));
    if (r != 0) return r;
    return la < lb ? -1 : (la > lb ? 1 : 0);
  };
  std::stable_sort(o.begin(), o.end(), [&](int64_t a, int64_t b) {
    if (arrival[a] != arrival[b]) return arrival[a] < arrival[b];
    return cmp_id(a, b) < 0;
  });
  uint32_t r = 0;
  for (int64_t k = 0; k < n; ++k) {
    if (k > 0) {
      const int64_t p = o[k - 1], c = o[k];
      if (arrival[p] != arrival[c] || cmp_id(p, c) != 0) ++r;
    }
    rank[o[k]] = r;
  }
  return PARS_OK;
}

int pars_workload_synthesize(uint64_t n, double mu, double sigma, uint64_t seed, int64_t pad_tokens,
                             uint64_t pad_seed, pars_workload** out) {
  *out = nullptr;
  if (n < 1) {
    set_error("synthesize: n must be >= 1");
    return PARS_ERR_INVALID;
  }
  if (sigma <= 0.0) {
    set_error("synthesize: sigma must be > 0 (got %g)", sigma);
    return PARS_ERR_INVALID;
  }
  constexpr double kLatentStep = 0.05;  // dataset.cpp:196
  const int64_t min_len = 1, max_len = 16384;
  auto* w = new pars_workload();
  w->offsets.resize(n + 1);
  w->output_len.resize(n);
  w->prompt_len.resize(n);
  Rng rng(seed);
  std::vector<std::string> texts(n);
  auto clamp_len = [&](double v) {
    int64_t len = static_cast<int64_t>(std::llround(v));
    return std::clamp(len, min_len, max_len);
  };
  const int64_t q_cap =
      static_cast<int64_t>(std::llround(std::log(static_cast<double>(max_len)) / kLatentStep));
  std::vector<std::string> tokens;
  for (uint64_t i = 0; i < n; ++i) {
    (void)rng.uniform01();  // mixture pick (single component, dataset.cpp:229-239)
    const double z = mu + sigma * rng.normal();
    const int64_t q = static_cast<int64_t>(std::llround(z / kLatentStep));
    const int64_t clean = clamp_len(std::exp(kLatentStep * static_cast<double>(q)));
    w->output_len[i] = clean;
    const int64_t q_therm = std::clamp<int64_t>(q, 0, q_cap);
    tokens.clear();
    std::string t = "len";
    append_i64(t, q);
    tokens.push_back(t);
    for (int64_t lvl = 0; lvl <= q_therm; ++lvl) {
      std::string s = "lvl";
      append_i64(s, lvl);
      tokens.push_back(std::move(s));
    }
    const size_t n_filler = 4 + rng.below(21);
    for (size_t f = 0; f < n_filler; ++f) {
      std::string s = "w";
      append_u64(s, rng.below(50));
      tokens.push_back(std::move(s));
    }
    rng.shuffle(tokens);
    std::string& text = texts[i];
    for (const std::string& tok : tokens) {
      if (!text.empty()) text += ' ';
      text += tok;
    }
    w->prompt_len[i] = static_cast<int64_t>(tokens.size());
  }
  if (pad_tokens > 0) {  // " w<k>", k = Rng(pad_seed).below(50)
    Rng pad(pad_seed);
    for (uint64_t i = 0; i < n; ++i) {
      std::string& text = texts[i];
      for (int64_t k = w->prompt_len[i]; k < pad_tokens; ++k) {
        text += " w";
        append_u64(text, pad.below(50));
      }
      w->prompt_len[i] = std::max<int64_t>(w->prompt_len[i], pad_tokens);
    }
  }
  int64_t total = 0;
  for (uint64_t i = 0; i < n; ++i) {
    w->offsets[i] = total;
    total += (int64_t)texts[i].size();
  }
  w->offsets[n] = total;
  w->bytes = total;
  if (cudaHostAlloc(reinterpret_cast<void**>(&w->text), std::max<int64_t>(total, 1),
                    cudaHostAllocDefault) == cudaSuccess) {
    w->pinned = true;
  } else {
    cudaGetLastError();
    w->text = static_cast<char*>(std::malloc(std::max<int64_t>(total, 1)));
    if (!w->text) {
      delete w;
      set_error("synthesize: out of host memory");
      return PARS_ERR_OOM;
    }
  }
  for (uint64_t i = 0; i < n; ++i)
    std::memcpy(w->text + w->offsets[i], texts[i].data(), texts[i].size());
  *out = w;
  return PARS_OK;
}

int64_t pars_workload_count(const pars_workload* w) { return (int64_t)w->output_len.size(); }
int64_t pars_workload_text_bytes(const pars_workload* w) { return w->bytes; }
const char* pars_workload_text(const pars_workload* w) { return w->text; }
const int64_t* pars_workload_offsets(const pars_workload* w) { return w->offsets.data(); }
const int64_t* pars_workload_output_len(const pars_workload* w) { return w->output_len.data(); }
const int64_t* pars_workload_prompt_len(const pars_workload* w) { return w->prompt_len.data(); }
void pars_workload_free(pars_workload* w) {
  if (!w) return;
  if (w->pinned)
    cudaFreeHost(w->text);
  else
    std::free(w->text);
  delete w;
}

}  // extern "C"
