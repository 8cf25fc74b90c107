// Host-side parts of the hot path that are sequential by construction:
//   * build_pairs (pairs.cpp:8-36): one mt19937_64 stream, draw by draw;
//   * the integer Eq. 1 table dmin[m] (pairs.hpp:21-24 evaluated on host with
//     the reference's own double division, once per (delta, max_len));
//   * tie ranks for the priority key (scheduler.cpp:44-49 tie_key).
// (The synthetic workload generator is a tool, tools/workload, not part of
// this library.)
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
#include "rng_host.hpp"

namespace pars_b200 {
void set_error(const char* fmt, ...);
}
using pars_b200::set_error;
using pars_b200::Rng;

namespace {

inline double rel_diff(int64_t a, int64_t b) {
  return static_cast<double>(std::llabs(a - b)) / static_cast<double>(std::max(a, b));
}

}  // namespace

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
  auto cmp_id = [&](int64_t a, int64_t b) {
    const int64_t la = offs[a + 1] - offs[a], lb = offs[b + 1] - offs[b];
    int r = std::memcmp(ids + offs[a], ids + offs[b], (size_t)std::min(la, lb));
    if (r != 0) return r;
    return la < lb ? -1 : (la > lb ? 1 : 0);
  };
  // common case (a trace in arrival order, a burst with ascending ids): the
  // keys are already non-decreasing in input order -> one linear pass
  bool sorted = true;
  for (int64_t k = 1; k < n && sorted; ++k)
    sorted = arrival[k - 1] < arrival[k] || (arrival[k - 1] == arrival[k] && cmp_id(k - 1, k) <= 0);
  if (sorted) {
    uint32_t r = 0;
    for (int64_t k = 0; k < n; ++k) {
      if (k > 0 && (arrival[k - 1] != arrival[k] || cmp_id(k - 1, k) != 0)) ++r;
      rank[k] = r;
    }
    return PARS_OK;
  }
  std::vector<int64_t> o(n);
  std::iota(o.begin(), o.end(), 0);
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

}  // extern "C"
