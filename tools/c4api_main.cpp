// C4 end to end through the reference's public API (proj/include/pars):
// a program written against the reference headers only —
// Scorer::score_batch (scorer.cpp:9-24) over a Dataset of pageable
// std::string records, then select_batch (scheduler.cpp:33-60) of the burst —
// exactly the reference arm's step (oracle/ref_capi.cpp ref_score_order).
// Linked with the B200 drop-in (libpars_b200 + libpars_cuda) it is
// oracle/_ref/c4api_b200: the user-facing end-to-end number beside the
// pinned C-ABI one.
//
//   inputs:  synthesize_dataset(n, seed 31) padded to 512 whitespace tokens
//            with " w<k>", k = Rng(5).below(50)
//   weights: argv[2] (4096 raw fp64, written by bench.py) or Rng-normal
//   usage:   c4api_b200 N [weights.bin] [steps] [out_prefix]
//            (out_prefix: the last step's scores and order as raw fp64 /
//            int64 files <prefix>.scores, <prefix>.order for the caller's
//            parity check)
// Prints one JSON line: per-step seconds (median), prompts/s, and FNV-1a
// digests of the scores and the order (comparable with bench.py's).
#include <algorithm>
#include <chrono>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <string>
#include <vector>

#include "pars/dataset.hpp"
#include "pars/rng.hpp"
#include "pars/scheduler.hpp"
#include "pars/scorer.hpp"

static uint64_t fnv(const void* p, size_t n, uint64_t h = 0xcbf29ce484222325ull) {
  const unsigned char* b = static_cast<const unsigned char*>(p);
  for (size_t i = 0; i < n; ++i) {
    h ^= b[i];
    h *= 0x100000001b3ull;
  }
  return h;
}

int main(int argc, char** argv) {
  const size_t n = argc > 1 ? std::strtoull(argv[1], nullptr, 10) : 1000000;
  const int steps = argc > 3 ? std::atoi(argv[3]) : 3;
  pars::SynthConfig sc;
  sc.n = n;
  sc.seed = 31;
  pars::Dataset ds = pars::synthesize_dataset(sc);
  pars::Rng pad(5);
  for (pars::PromptRecord& r : ds.records) {
    for (int64_t k = r.prompt_len; k < 512; ++k) {
      r.prompt_text += " w";
      r.prompt_text += std::to_string(pad.below(50));
    }
    r.prompt_len = std::max<int64_t>(r.prompt_len, 512);
  }
  pars::FeatureExtractor ex;  // the reference's default predictor
  std::vector<double> w(ex.dim);
  if (argc > 2) {
    FILE* f = std::fopen(argv[2], "rb");
    if (!f || std::fread(w.data(), 8, w.size(), f) != w.size()) {
      std::fprintf(stderr, "cannot read %s\n", argv[2]);
      return 2;
    }
    std::fclose(f);
  } else {
    pars::Rng r(1234);
    for (double& x : w) x = 0.05 * r.normal();
  }
  const pars::LinearScorer scorer(ex, w, 0.0);
  std::vector<double> s;
  std::vector<size_t> sel;
  auto step = [&] {
    s = scorer.score_batch(ds);
    std::vector<pars::Request> q(ds.records.size());
    for (size_t i = 0; i < q.size(); ++i) {
      q[i].record_idx = static_cast<uint32_t>(i);
      q[i].prompt_id = ds.records[i].id;
      q[i].arrival_time = 0.0;
      q[i].score = s[i];
    }
    pars::PolicyConfig cfg;
    sel = pars::select_batch(q, 0.0, q.size(), cfg);
  };
  step();  // warm-up (device context, scratch, weights)
  std::vector<double> ts;
  std::vector<double> t_score;
  for (int k = 0; k < steps; ++k) {
    const auto t0 = std::chrono::steady_clock::now();
    s = scorer.score_batch(ds);
    const auto t1 = std::chrono::steady_clock::now();
    std::vector<pars::Request> q(ds.records.size());
    for (size_t i = 0; i < q.size(); ++i) {
      q[i].record_idx = static_cast<uint32_t>(i);
      q[i].prompt_id = ds.records[i].id;
      q[i].arrival_time = 0.0;
      q[i].score = s[i];
    }
    pars::PolicyConfig cfg;
    sel = pars::select_batch(q, 0.0, q.size(), cfg);
    const auto t2 = std::chrono::steady_clock::now();
    ts.push_back(std::chrono::duration<double>(t2 - t0).count());
    t_score.push_back(std::chrono::duration<double>(t1 - t0).count());
  }
  std::sort(ts.begin(), ts.end());
  std::sort(t_score.begin(), t_score.end());
  const double med = ts[ts.size() / 2], med_score = t_score[t_score.size() / 2];
  uint64_t text_bytes = 0;
  for (const auto& r : ds.records) text_bytes += r.prompt_text.size();
  std::vector<int64_t> order(sel.begin(), sel.end());
  if (argc > 4) {
    const std::string pre = argv[4];
    FILE* fs = std::fopen((pre + ".scores").c_str(), "wb");
    FILE* fo = std::fopen((pre + ".order").c_str(), "wb");
    if (!fs || !fo || std::fwrite(s.data(), 8, s.size(), fs) != s.size() ||
        std::fwrite(order.data(), 8, order.size(), fo) != order.size()) {
      std::fprintf(stderr, "cannot write %s.*\n", pre.c_str());
      return 2;
    }
    std::fclose(fs);
    std::fclose(fo);
  }
  std::printf("{\"n\": %zu, \"steps\": %d, \"step_s\": %.6f, \"score_batch_s\": %.6f, "
              "\"prompts_per_s\": %.1f, \"text_bytes\": %llu, \"scores_fnv\": \"%016llx\", "
              "\"order_fnv\": \"%016llx\"}\n",
              n, steps, med, med_score, n / med, (unsigned long long)text_bytes,
              (unsigned long long)fnv(s.data(), s.size() * 8),
              (unsigned long long)fnv(order.data(), order.size() * 8));
  return 0;
}
