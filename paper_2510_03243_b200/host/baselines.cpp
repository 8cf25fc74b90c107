// The paper's comparison objectives (pointwise L1 regression on log length,
// ListMLE) for train.hpp — outside the PARS hot path (SURVEY §2 row 6,
// §8(f).4), kept so the shim is a complete drop-in for train.cpp. Host code
// over GPU-extracted features; every floating-point expression keeps the
// reference's evaluation order (train.cpp:46-94 and :141-151, :168-209), so
// results match the CPU library.
#include <algorithm>
#include <cmath>
#include <span>

#include "pars/rng.hpp"
#include "pars/train.hpp"
#include "shim.hpp"

namespace pars {

namespace {

// Minibatch accumulator: dense gradient + bias gradient, applied as
// w[d] -= (lr / batch) * g[d] for g[d] != 0, then cleared.
struct Minibatch {
  std::vector<double> g;
  double gb = 0.0;
  explicit Minibatch(uint32_t dim) : g(dim, 0.0) {}
  void add(const FeatureVec& x, double coef) {
    for (const auto& [d, v] : x.entries) g[d] += coef * v;
  }
  void step(LinearScorer& s, double lr, size_t batch) {
    const double scale = lr / static_cast<double>(batch);
    std::vector<double>& w = s.weights();
    for (size_t d = 0; d < g.size(); ++d) {
      if (g[d] == 0.0) continue;
      w[d] -= scale * g[d];
      g[d] = 0.0;
    }
    s.bias() -= scale * gb;
    gb = 0.0;
  }
};

double dot_bias(const LinearScorer& s, const FeatureVec& x) {
  return x.dot(s.weights()) + s.bias();
}

double sgn(double v) { return v > 0.0 ? 1.0 : (v < 0.0 ? -1.0 : 0.0); }

// log(exp(a) + exp(b)) evaluated around the larger argument.
double lse2(double a, double b) {
  const double m = a < b ? b : a;
  const double r = a < b ? a : b;
  return m + std::log1p(std::exp(r - m));
}

// ListMLE negative log-likelihood of a list given longest-first, and its
// score gradient dL/ds_j (coef), for scores s[0..k).
double listmle_nll(const std::vector<double>& s, std::vector<double>& coef) {
  const size_t k = s.size();
  std::vector<double> tail(k);  // tail[i] = log sum_{j>=i} exp(s_j)
  tail[k - 1] = s[k - 1];
  for (size_t i = k - 1; i > 0; --i) tail[i - 1] = lse2(s[i - 1], tail[i]);
  coef.assign(k, 0.0);
  double nll = 0.0;
  for (size_t i = 0; i < k; ++i) {
    nll += tail[i] - s[i];
    coef[i] -= 1.0;
    for (size_t j = i; j < k; ++j) coef[j] += std::exp(s[j] - tail[i]);
  }
  return nll;
}

}  // namespace

double pointwise_l1_loss_grad(const LinearScorer& scorer, const FeatureVec& x, double target,
                              std::vector<double>& grad, double& bias_grad) {
  const double r = scorer.score(x) - target;
  const double g = sgn(r);
  for (const auto& [d, v] : x.entries) grad[d] += g * v;
  bias_grad += g;
  return std::fabs(r);
}

double listmle_loss_grad(const LinearScorer& scorer, const std::vector<FeatureVec>& features,
                         std::span<const uint32_t> list_true_order, std::vector<double>& grad) {
  if (list_true_order.size() < 2) throw Error("listmle: list needs >= 2 items");
  std::vector<double> s;
  s.reserve(list_true_order.size());
  for (uint32_t r : list_true_order) s.push_back(scorer.score(features[r]));
  std::vector<double> coef;
  const double nll = listmle_nll(s, coef);
  for (size_t j = 0; j < list_true_order.size(); ++j)
    for (const auto& [d, v] : features[list_true_order[j]].entries) grad[d] += coef[j] * v;
  return nll;
}

namespace b200 {

void train_baseline(const Dataset& ds, const TrainConfig& cfg, const std::vector<FeatureVec>& feats,
                    TrainedModel& model) {
  const size_t n = ds.records.size();
  LinearScorer& sc = model.scorer;
  Minibatch mb(cfg.extractor.dim);
  const bool listwise = cfg.objective == Objective::ListwiseListMLE;
  if (listwise && n < 2) throw Error("train: listwise needs >= 2 records");
  std::vector<uint32_t> idx(n);
  for (size_t i = 0; i < n; ++i) idx[i] = static_cast<uint32_t>(i);
  for (int epoch = 0; epoch < cfg.epochs; ++epoch) {
    Rng rng(derive_seed(cfg.seed, 0x10000u + epoch));
    double total = 0.0;
    size_t samples = 0;
    if (!listwise) {
      // one shuffled pass, batch_size samples per step
      std::vector<uint32_t> perm = idx;
      rng.shuffle(perm);
      for (size_t lo = 0; lo < n; lo += cfg.batch_size) {
        const size_t hi = std::min(n, lo + static_cast<size_t>(cfg.batch_size));
        for (size_t p = lo; p < hi; ++p) {
          const FeatureVec& x = feats[perm[p]];
          const double r = dot_bias(sc, x) - pointwise_target(ds.records[perm[p]].output_len);
          const double g = sgn(r);
          mb.add(x, g);
          mb.gb += g;
          total += std::fabs(r);
        }
        mb.step(sc, cfg.learning_rate, hi - lo);
        samples += hi - lo;
      }
    } else {
      // lists_per_epoch lists of list_size items drawn without replacement
      // (partial Fisher-Yates on a persistent pool), ordered longest-first
      // with id tiebreak; batch_size lists per step
      const size_t k = std::min<size_t>(static_cast<size_t>(cfg.list_size), n);
      std::vector<uint32_t> pool = idx, list(k);
      std::vector<double> s(k), coef;
      size_t pending = 0;
      for (size_t l = 0; l < cfg.lists_per_epoch; ++l) {
        for (size_t t = 0; t < k; ++t) std::swap(pool[t], pool[t + rng.below(n - t)]);
        std::copy(pool.begin(), pool.begin() + k, list.begin());
        std::sort(list.begin(), list.end(), [&](uint32_t a, uint32_t b) {
          const PromptRecord& ra = ds.records[a];
          const PromptRecord& rb = ds.records[b];
          return ra.output_len != rb.output_len ? ra.output_len > rb.output_len : ra.id < rb.id;
        });
        for (size_t t = 0; t < k; ++t) s[t] = dot_bias(sc, feats[list[t]]);
        total += listmle_nll(s, coef);
        for (size_t t = 0; t < k; ++t) mb.add(feats[list[t]], coef[t]);
        ++samples;
        if (++pending == static_cast<size_t>(cfg.batch_size) || l + 1 == cfg.lists_per_epoch) {
          mb.step(sc, cfg.learning_rate, pending);
          pending = 0;
        }
      }
    }
    const double mean = total / static_cast<double>(samples);
    if (!std::isfinite(mean)) fail("training diverged at epoch %d", epoch);
    model.loss_trace.push_back(mean);
  }
}

}  // namespace b200
}  // namespace pars
