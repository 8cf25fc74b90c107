// scheduler.hpp / metrics.hpp over libpars_cuda (replaces
// proj/src/scheduler.cpp and proj/src/metrics.cpp).
//   select_batch    -> GPU stable radix sort on (score, tie rank) keys
//                      (sort.cu); the index tiebreak is the sort's stability
//   kendall_tau_b   -> GPU all-pairs integer counts (pairs.cu tau_kernel),
//                      finished on the host exactly as finish_tau
//   latency_summary / percentile / relative variance: host bookkeeping
//   (reporting, not the hot path).
#include <algorithm>
#include <cmath>

#include "pars/metrics.hpp"
#include "pars/scheduler.hpp"
#include "pars/simulator.hpp"
#include "shim.hpp"

namespace pars {

Policy make_fcfs_policy() { return Policy{"fcfs", PolicyKind::Fcfs, nullptr}; }

Policy make_sjf_policy(std::string name, std::shared_ptr<const Scorer> scorer) {
  if (!scorer) throw Error("sjf policy needs a scorer");
  return Policy{std::move(name), PolicyKind::Sjf, std::move(scorer)};
}

void enqueue(Request& request, const PolicyConfig& config, const PromptRecord& record) {
  if (request.state != RequestState::Waiting)
    fail("enqueue: request '%s' is not waiting", request.prompt_id.c_str());
  if (config.policy.kind == PolicyKind::Fcfs) {
    request.score = request.arrival_time;
    return;
  }
  try {
    request.score = config.policy.scorer->score(record);
  } catch (const Error& e) {
    fail("enqueue: cannot score request '%s': %s", request.prompt_id.c_str(), e.what());
  }
}

std::vector<size_t> select_batch(std::span<const Request> waiting, double now, size_t free_slots,
                                 const PolicyConfig& config) {
  (void)config;
  const size_t n = waiting.size();
  std::vector<size_t> order(n);
  if (n == 0) return order;
  std::vector<double> score(n), arrival(n);
  std::vector<uint8_t> boosted(n);
  std::string ids;
  std::vector<int64_t> id_offs(n + 1, 0);
  for (size_t i = 0; i < n; ++i) {
    score[i] = waiting[i].score;
    arrival[i] = waiting[i].arrival_time;
    boosted[i] = waiting[i].boosted ? 1 : 0;
    ids += waiting[i].prompt_id;
    id_offs[i + 1] = static_cast<int64_t>(ids.size());
  }
  std::vector<uint32_t> tie(n);
  b200::check(pars_tie_ranks(arrival.data(), ids.data(), id_offs.data(), static_cast<int64_t>(n),
                             tie.data()));
  std::vector<int64_t> perm(n);
  b200::check(pars_priority_order(b200::ctx(), score.data(), boosted.data(), tie.data(),
                                  static_cast<int64_t>(n), perm.data()));
  for (size_t k = 0; k < n; ++k) {
    order[k] = static_cast<size_t>(perm[k]);
    if (waiting[order[k]].arrival_time > now)
      fail("select_batch: request '%s' has not arrived yet", waiting[order[k]].prompt_id.c_str());
  }
  order.resize(std::min(free_slots, n));
  return order;
}

size_t update_boosts(std::span<Request> waiting, double now, double threshold,
                     std::vector<size_t>* newly_boosted) {
  if (threshold <= 0.0) fail("update_boosts: threshold must be > 0");
  size_t count = 0;
  for (size_t i = 0; i < waiting.size(); ++i) {
    Request& r = waiting[i];
    if (r.boosted || !(now - r.arrival_time > threshold)) continue;
    r.boosted = true;
    ++count;
    if (newly_boosted) newly_boosted->push_back(i);
  }
  return count;
}

// ---- metrics ----------------------------------------------------------------

TauResult kendall_tau_b(std::span<const double> x, std::span<const double> y) {
  if (x.size() != y.size())
    fail("kendall_tau_b: size mismatch (%zu vs %zu)", x.size(), y.size());
  if (x.size() < 2) fail("kendall_tau_b: need at least 2 items, got %zu", x.size());
  uint64_t c[5];
  double tau = 0.0;
  b200::check(pars_kendall_tau(b200::ctx(), x.data(), y.data(), static_cast<int64_t>(x.size()), c,
                               &tau));
  TauResult r;
  r.n_c = c[0];
  r.n_d = c[1];
  r.n0 = c[2];
  r.n1 = c[3];
  r.n2 = c[4];
  r.tau_b = tau;
  return r;
}

TauResult kendall_tau_b_serial(std::span<const double> x, std::span<const double> y) {
  return kendall_tau_b(x, y);  // integer counts: identical for any decomposition
}

double percentile_nearest_rank(std::vector<double> values, int pct) {
  if (values.empty()) throw Error("percentile: empty input");
  if (pct < 1 || pct > 100) fail("percentile: pct %d outside [1,100]", pct);
  const size_t rank = (static_cast<size_t>(pct) * values.size() + 99) / 100;  // ceil, integer
  std::nth_element(values.begin(), values.begin() + (rank - 1), values.end());
  return values[rank - 1];
}

LatencySummary latency_summary(std::span<const double> per_token_latency_s) {
  if (per_token_latency_s.empty()) throw Error("latency_summary: no completed requests");
  LatencySummary s;
  s.count = per_token_latency_s.size();
  std::vector<double> ms(per_token_latency_s.size());
  double sum = 0.0;
  for (size_t i = 0; i < ms.size(); ++i) {
    ms[i] = per_token_latency_s[i] * 1000.0;
    sum += ms[i];
  }
  s.mean_per_token_ms = sum / static_cast<double>(s.count);
  s.p90_per_token_ms = percentile_nearest_rank(std::move(ms), 90);
  return s;
}

LatencySummary latency_summary(const SimResult& result) {
  std::vector<double> lat(result.requests.size());
  for (size_t i = 0; i < lat.size(); ++i) lat[i] = result.requests[i].per_token_latency_s;
  return latency_summary(lat);
}

double relative_variance_pct(std::span<const int64_t> samples) {
  if (samples.size() < 2) fail("relative_variance: need >= 2 samples, got %zu", samples.size());
  const auto [lo, hi] = std::minmax_element(samples.begin(), samples.end());
  for (int64_t v : samples)
    if (v < 1) fail("relative_variance: sample %lld < 1", static_cast<long long>(v));
  return (static_cast<double>(*hi) / static_cast<double>(*lo) - 1.0) * 100.0;
}

}  // namespace pars
