// Synthetic workload tool (tools/workload/pars_workload.h): the reference's
// synthesize_dataset (proj/src/dataset.cpp:204-297) restated for fast input
// generation, plus the C4 padding. Built into tools/libpars_workload.so by
// tools/workload/Makefile — not part of the product library.
#include <algorithm>
#include <cmath>
#include <cstdint>
#include <cstdlib>
#include <cstring>
#include <string>
#include <vector>

#include <cuda_runtime.h>

#include "pars_workload.h"
#include "rng_host.hpp"

using pars_b200::append_i64;
using pars_b200::append_u64;
using pars_b200::Rng;

namespace {
thread_local std::string g_err;
}

struct pars_workload {
  char* text = nullptr;  // pinned when possible
  bool pinned = false;
  int64_t bytes = 0;
  std::vector<int64_t> offsets, output_len, prompt_len;
};

extern "C" {

const char* pars_workload_last_error(void) { return g_err.c_str(); }

int pars_workload_synthesize(uint64_t n, double mu, double sigma, uint64_t seed, int64_t pad_tokens,
                             uint64_t pad_seed, pars_workload** out) {
  return pars_workload_synthesize_pad(n, mu, sigma, seed, pad_tokens, pad_seed, 0, out);
}

int pars_workload_synthesize_pad(uint64_t n, double mu, double sigma, uint64_t seed, int64_t pad_tokens,
                                 uint64_t pad_seed, int pad_kind, pars_workload** out) {
  *out = nullptr;
  if (n < 1) {
    g_err = "synthesize: n must be >= 1";
    return 2;
  }
  if (sigma <= 0.0) {
    g_err = "synthesize: sigma must be > 0 (got " + std::to_string(sigma) + ")";
    return 2;
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
    Rng pad(pad_seed);     // (pad_kind 1, the hard variant: random 6-letter lowercase words)
    for (uint64_t i = 0; i < n; ++i) {
      std::string& text = texts[i];
      for (int64_t k = w->prompt_len[i]; k < pad_tokens; ++k) {
        if (pad_kind == 1) {
          text += ' ';
          for (int c = 0; c < 6; ++c) text += static_cast<char>('a' + pad.below(26));
        } else {
          text += " w";
          append_u64(text, pad.below(50));
        }
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
      g_err = "synthesize: out of host memory";
      return 3;
    }
  }
  for (uint64_t i = 0; i < n; ++i)
    std::memcpy(w->text + w->offsets[i], texts[i].data(), texts[i].size());
  *out = w;
  return 0;
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

extern "C" int pars_workload_token_stats(const char* text, const int64_t* offsets, int64_t n,
                                         uint64_t* out) {
  uint64_t tok = 0, sum = 0, tri = 0;
  const unsigned char* t = reinterpret_cast<const unsigned char*>(text);
  for (int64_t i = 0; i < n; ++i) {
    int64_t len = 0;
    for (int64_t p = offsets[i]; p < offsets[i + 1]; ++p) {
      const unsigned c = t[p];
      if (c == 32u || (c - 9u) < 5u) {
        if (len) {
          ++tok;
          sum += (uint64_t)len;
          tri += len > 2 ? (uint64_t)(len - 2) : 0;
          len = 0;
        }
      } else {
        ++len;
      }
    }
    if (len) {
      ++tok;
      sum += (uint64_t)len;
      tri += len > 2 ? (uint64_t)(len - 2) : 0;
    }
  }
  out[0] = tok;
  out[1] = sum;
  out[2] = tri;
  out[3] = n > 0 ? (uint64_t)(offsets[n] - offsets[0]) : 0;
  return 0;
}
