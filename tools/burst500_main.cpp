// README burst-500 driver (proj/README.md:26-36): a program written against
// the reference's public headers only, run through compare_policies
// (simulator.cpp:226-283). Linked with the reference library it is
// oracle/_ref/burst500_ref; linked with the B200 drop-in (libpars_b200 for
// features/scorer/train/scheduler/metrics/simulator, the reference objects
// for error/dataset/arrivals/model_io) it is oracle/_ref/burst500_b200.
//
//   model:    synthesize(4000, lognormal(5,1.2), seed 21), split(0.2, 21),
//             train(TrainConfig{seed = 21})         (pars gen-workload + train)
//   workload: synthesize(500, seed 22), burst arrivals (seed 0), default
//             SimConfig (continuous, batch 32)      (pars compare --policies
//                                                    fcfs,oracle,pars)
// Prints one JSON line with every policy's mean / p90 per-token latency,
// iterations, simulated seconds and tau_b at full precision, plus the
// completion FNV (prompt id bytes then the 8 bytes of finish_s).
#include <cstdint>
#include <cstdio>
#include <memory>

#include "pars/arrivals.hpp"
#include "pars/dataset.hpp"
#include "pars/scheduler.hpp"
#include "pars/scorer.hpp"
#include "pars/simulator.hpp"
#include "pars/train.hpp"

int main() {
  pars::SynthConfig mc;
  mc.n = 4000;
  mc.seed = 21;
  const pars::Dataset full = pars::synthesize_dataset(mc);
  const auto split = pars::split_dataset(full, 0.2, 21);
  pars::TrainConfig tc;
  tc.seed = 21;
  const pars::TrainedModel model = pars::train(split.first, tc);

  pars::SynthConfig wc;
  wc.n = 500;
  wc.seed = 22;
  const pars::Dataset ds = pars::synthesize_dataset(wc);
  const pars::ArrivalTrace trace = pars::generate_burst_arrivals(ds, 0);

  std::vector<pars::Policy> policies;
  policies.push_back(pars::make_fcfs_policy());
  policies.push_back(pars::make_sjf_policy("oracle", std::make_shared<pars::OracleScorer>(ds)));
  policies.push_back(
      pars::make_sjf_policy("pars", std::make_shared<pars::LinearScorer>(model.scorer)));
  pars::SimConfig base;
  const pars::ComparisonReport rep = pars::compare_policies(trace, ds, base, policies);

  std::printf("{");
  for (size_t k = 0; k < rep.runs.size(); ++k) {
    const auto& r = rep.runs[k];
    uint64_t h = 0xcbf29ce484222325ull;
    auto fnv = [&](const void* p, size_t n) {
      const unsigned char* b = static_cast<const unsigned char*>(p);
      for (size_t i = 0; i < n; ++i) {
        h ^= b[i];
        h *= 0x100000001b3ull;
      }
    };
    for (const auto& q : r.result.requests) {
      fnv(q.prompt_id.data(), q.prompt_id.size());
      fnv(&q.finish_s, 8);
    }
    std::printf(
        "\"%s\": {\"mean_ms\": %.17g, \"p90_ms\": %.17g, \"iterations\": %llu, "
        "\"simulated_s\": %.17g, \"tau_b\": %.17g, \"completion_fnv\": \"%016llx\"}%s",
        r.policy.c_str(), r.latency.mean_per_token_ms, r.latency.p90_per_token_ms,
        (unsigned long long)r.result.iterations, r.result.simulated_seconds,
        r.tau_b ? *r.tau_b : -2.0, (unsigned long long)h, k + 1 < rep.runs.size() ? ", " : "");
  }
  std::printf("}\n");
  return 0;
}
