// C3 driver (BASELINE config 3): a program written against the reference's
// public headers only. Linked with the reference library it is the CPU
// baseline (oracle/_ref/c3_ref); linked with the B200 drop-in (libpars_b200
// for scorer/train/scheduler/metrics/simulator, the reference objects for
// dataset/arrivals) it is the GPU path (oracle/_ref/c3_b200).
//
//   model:    README recipe — synthesize(4000, seed 21), split(0.2, 21),
//             train(TrainConfig{seed = 21})
//   workload: synthesize(100000, seed 23), Poisson arrivals 5 req/s seed 24,
//             default SimConfig (continuous, batch 32, starvation 120 s)
//   runs:     FCFS and PARS (the trained model as the SJF scorer)
// Prints one JSON line: per policy the completion FNV (prompt id bytes then
// the 8 bytes of finish_s, in completion order), iterations, simulated
// seconds, mean/p90 per-token latency and the wall time of run_simulation.
#include <chrono>
#include <cstdint>
#include <cstdio>
#include <cstring>
#include <memory>
#include <string>

#include "pars/arrivals.hpp"
#include "pars/dataset.hpp"
#include "pars/metrics.hpp"
#include "pars/scheduler.hpp"
#include "pars/simulator.hpp"
#include "pars/train.hpp"

namespace {

uint64_t fnv(uint64_t h, const void* p, size_t n) {
  const unsigned char* b = static_cast<const unsigned char*>(p);
  for (size_t i = 0; i < n; ++i) {
    h ^= b[i];
    h *= 0x100000001b3ull;
  }
  return h;
}

double secs_since(std::chrono::steady_clock::time_point t0) {
  return std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
}

void report(const char* name, const pars::SimResult& r, double wall, bool last) {
  uint64_t h = 0xcbf29ce484222325ull;
  for (const auto& q : r.requests) {
    h = fnv(h, q.prompt_id.data(), q.prompt_id.size());
    h = fnv(h, &q.finish_s, 8);
  }
  const pars::LatencySummary s = pars::latency_summary(r);
  std::printf(
      "\"%s\": {\"completion_fnv\": \"%016llx\", \"iterations\": %llu, \"simulated_s\": %.17g, "
      "\"mean_ms\": %.17g, \"p90_ms\": %.17g, \"wall_s\": %.6f}%s",
      name, (unsigned long long)h, (unsigned long long)r.iterations, r.simulated_seconds,
      s.mean_per_token_ms, s.p90_per_token_ms, wall, last ? "" : ", ");
}

}  // namespace

int main(int argc, char** argv) {
  const size_t n = argc > 1 ? std::strtoull(argv[1], nullptr, 10) : 100000;
  pars::SynthConfig mc;
  mc.n = 4000;
  mc.seed = 21;
  const pars::Dataset full = pars::synthesize_dataset(mc);
  const auto split = pars::split_dataset(full, 0.2, 21);
  pars::TrainConfig tc;
  tc.seed = 21;
  auto t0 = std::chrono::steady_clock::now();
  const pars::TrainedModel model = pars::train(split.first, tc);
  const double train_s = secs_since(t0);

  pars::SynthConfig wc;
  wc.n = n;
  wc.seed = 23;
  const pars::Dataset ds = pars::synthesize_dataset(wc);
  const pars::ArrivalTrace trace = pars::generate_poisson_arrivals(ds, 5.0, 24);

  pars::SimConfig fcfs;
  fcfs.policy.policy = pars::make_fcfs_policy();
  t0 = std::chrono::steady_clock::now();
  const pars::SimResult rf = pars::run_simulation(trace, ds, fcfs);
  const double wf = secs_since(t0);

  pars::SimConfig sjf;
  sjf.policy.policy =
      pars::make_sjf_policy("pars", std::make_shared<pars::LinearScorer>(model.scorer));
  // twice: the first run also pays one-time costs (lazy module loading of
  // the kernels it launches, buffer growth); the reported wall is the second
  t0 = std::chrono::steady_clock::now();
  (void)pars::run_simulation(trace, ds, sjf);
  const double wp_first = secs_since(t0);
  t0 = std::chrono::steady_clock::now();
  const pars::SimResult rp = pars::run_simulation(trace, ds, sjf);
  const double wp = secs_since(t0);

  std::printf("{\"n\": %zu, \"train_s\": %.6f, \"pars_first_wall_s\": %.6f, ", n, train_s, wp_first);
  report("fcfs", rf, wf, false);
  report("pars", rp, wp, true);
  std::printf("}\n");
  return 0;
}
