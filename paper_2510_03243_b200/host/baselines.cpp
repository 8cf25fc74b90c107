// The paper's comparison objectives (pointwise L1 regression on log length,
// ListMLE) for train.hpp. train() runs them on the GPU
// engine (baselines.cu via pars_pointwise_epoch / pars_listmle_epoch); the
// single-call loss/grad helpers below are host code over host FeatureVecs,
// each floating-point expression in the reference's order
// (train.cpp:46-94), so they match the CPU library.
#include <algorithm>
#include <cmath>
#include <span>

#include "pars/rng.hpp"
#include "pars/train.hpp"
#include "shim.hpp"

namespace pars {

namespace {

double sgn(double v) { return v > 0.0 ? 1.0 : (v < 0.0 ? -1.0 : 0.0); }

// log(exp(a) + exp(b)) evaluated around the larger argument.
double lse2(double a, double b) {
  const double m = a < b ? b : a;  // std::max / std::min (train.cpp:58-62)
  const double r = b < a ? b : a;
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

// train() for the comparison objectives (train.cpp:168-209) on the GPU
// engine: the epoch order / lists come from the reference's Rng on the host
// (pars_pointwise_order / pars_listmle_lists, bit-identical), the epochs run
// in baselines.cu over the device features.
void train_baseline(const Dataset& ds, const TrainConfig& cfg, const DeviceFeatures& dev,
                    TrainedModel& model) {
  const size_t n = ds.records.size();
  const bool listwise = cfg.objective == Objective::ListwiseListMLE;
  if (listwise && n < 2) throw Error("train: listwise needs >= 2 records");
  std::vector<int64_t> lens(n);
  for (size_t i = 0; i < n; ++i) lens[i] = ds.records[i].output_len;
  std::vector<double> target;
  std::string ids;
  std::vector<int64_t> id_offs(n + 1, 0);
  if (listwise) {
    for (size_t i = 0; i < n; ++i) {
      ids += ds.records[i].id;
      id_offs[i + 1] = static_cast<int64_t>(ids.size());
    }
  } else {
    target.resize(n);
    for (size_t i = 0; i < n; ++i) target[i] = pointwise_target(lens[i]);
  }
  const int32_t k = static_cast<int32_t>(std::min<size_t>(static_cast<size_t>(cfg.list_size), n));
  std::vector<uint32_t> rows(listwise ? cfg.lists_per_epoch * k : n);
  std::vector<double>& w = model.scorer.weights();
  for (int epoch = 0; epoch < cfg.epochs; ++epoch) {
    const uint64_t es = derive_seed(cfg.seed, 0x10000u + epoch);
    double total = 0.0;
    if (listwise) {
      check(pars_listmle_lists(lens.data(), ids.data(), id_offs.data(), static_cast<int64_t>(n),
                               static_cast<int64_t>(cfg.lists_per_epoch), cfg.list_size, es,
                               rows.data()));
      check(pars_listmle_epoch(ctx(), dev.f, rows.data(), static_cast<int64_t>(cfg.lists_per_epoch),
                               k, cfg.batch_size, cfg.learning_rate, w.data(),
                               model.scorer.bias(), &total));
    } else {
      check(pars_pointwise_order(static_cast<int64_t>(n), es, rows.data()));
      check(pars_pointwise_epoch(ctx(), dev.f, rows.data(), static_cast<int64_t>(n), target.data(),
                                 cfg.batch_size, cfg.learning_rate, w.data(),
                                 &model.scorer.bias(), &total));
    }
    const double mean =
        total / static_cast<double>(listwise ? cfg.lists_per_epoch : n);
    if (!std::isfinite(mean)) fail("training diverged at epoch %d", epoch);
    model.loss_trace.push_back(mean);
  }
}

}  // namespace b200
}  // namespace pars
