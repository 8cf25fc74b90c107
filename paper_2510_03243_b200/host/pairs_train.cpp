// pairs.hpp / train.hpp over libpars_cuda (replaces proj/src/pairs.cpp and
// proj/src/train.cpp).
//   build_pairs      -> pars_build_pairs (the seeded sampler is one sequential
//                       mt19937_64 stream; host, bit-identical)
//   train, Pairwise  -> GPU extract_all + per-epoch build_pairs + the
//                       persistent SGD-epoch kernel (sgd.cu), bit-identical
//                       weights and loss trace
//   pairwise_loss_grad -> both scores on the GPU, the hinge and the sparse
//                       update of the caller's host gradient as train.cpp:34-44
//   PointwiseL1 / ListwiseListMLE (train.cpp:46-94, :168-209) are the
//   paper's comparison baselines: host-sampled epoch order
//   / lists, GPU epochs (baselines.cu); pointwise bit-identical, ListMLE to
//   rounding (CUDA exp/log1p).
#include <algorithm>
#include <cmath>
#include <span>

#include "pars/pairs.hpp"
#include "pars/rng.hpp"
#include "pars/train.hpp"
#include "shim.hpp"

namespace pars {

namespace b200 {
void train_baseline(const Dataset& ds, const TrainConfig& cfg, const DeviceFeatures& dev,
                    TrainedModel& model);
}
using b200::train_baseline;

std::vector<RankedPair> build_pairs(const Dataset& ds, double delta, size_t max_pairs,
                                    uint64_t seed) {
  if (ds.records.empty()) throw Error("build_pairs: empty dataset");
  if (delta < 0.0 || delta >= 1.0) fail("build_pairs: delta %g outside [0, 1)", delta);
  if (max_pairs == 0) fail("build_pairs: max_pairs must be >= 1");
  std::vector<int64_t> lens(ds.records.size());
  for (size_t i = 0; i < lens.size(); ++i) lens[i] = ds.records[i].output_len;
  std::vector<uint32_t> a(max_pairs), b(max_pairs);
  std::vector<int32_t> y(max_pairs);
  std::vector<double> rel(max_pairs);
  const int64_t n = pars_build_pairs(lens.data(), static_cast<int64_t>(lens.size()), delta,
                                     max_pairs, seed, a.data(), b.data(), y.data(), rel.data());
  b200::check(n);
  std::vector<RankedPair> out(static_cast<size_t>(n));
  for (int64_t i = 0; i < n; ++i) out[i] = RankedPair{a[i], b[i], y[i], rel[i]};
  return out;
}

const char* objective_name(Objective obj) {
  switch (obj) {
    case Objective::Pairwise:
      return "pairwise";
    case Objective::PointwiseL1:
      return "pointwise_l1";
    case Objective::ListwiseListMLE:
      return "listwise_listmle";
  }
  return "?";
}

Objective objective_from_name(const std::string& name) {
  if (name == "pairwise") return Objective::Pairwise;
  if (name == "pointwise_l1") return Objective::PointwiseL1;
  if (name == "listwise_listmle") return Objective::ListwiseListMLE;
  fail("unknown objective '%s'", name.c_str());
}

double pointwise_target(int64_t output_len) { return std::log1p(static_cast<double>(output_len)); }

namespace {

// Both scores of a pair in one GPU launch (exact fp64).
void score_two(const LinearScorer& s, const FeatureVec& a, const FeatureVec& b, double out[2]) {
  b200::DeviceFeatures f;
  b200::upload(s.extractor().dim, {&a, &b}, f);
  b200::check(pars_features_score(b200::ctx(), f.f, s.weights().data(), s.bias(), out));
}

}  // namespace

double pairwise_loss_grad(const LinearScorer& scorer, const FeatureVec& a, const FeatureVec& b,
                          int y, double margin, std::vector<double>& grad) {
  double s[2];
  score_two(scorer, a, b, s);
  const double loss = margin_ranking_loss(s[0], s[1], y, margin);
  if (loss > 0.0) {
    for (const auto& [idx, v] : a.entries) grad[idx] -= y * v;
    for (const auto& [idx, v] : b.entries) grad[idx] += y * v;
  }
  return loss;
}

namespace {

void validate(const TrainConfig& cfg) {
  if (cfg.epochs < 0) fail("train: epochs must be >= 0");
  if (cfg.batch_size < 1) fail("train: batch_size must be >= 1");
  if (cfg.learning_rate <= 0.0) fail("train: learning_rate must be > 0");
  if (cfg.margin < 0.0) fail("train: margin must be >= 0");
  if (cfg.delta < 0.0 || cfg.delta >= 1.0) fail("train: delta %g outside [0, 1)", cfg.delta);
  if (cfg.pairs_per_epoch < 1) fail("train: pairs_per_epoch must be >= 1");
  if (cfg.lists_per_epoch < 1) fail("train: lists_per_epoch must be >= 1");
  if (cfg.list_size < 2) fail("train: list_size must be >= 2");
}

}  // namespace

TrainedModel train(const Dataset& ds, const TrainConfig& cfg) {
  validate(cfg);
  if (ds.records.empty()) throw Error("train: empty dataset");
  b200::DeviceFeatures dev;
  b200::extract_device(cfg.extractor, ds, dev);
  TrainedModel model;
  model.objective = cfg.objective;
  model.config = cfg;
  model.scorer = LinearScorer(cfg.extractor);  // all-zero init
  const size_t n = ds.records.size();

  if (cfg.objective == Objective::Pairwise) {
    std::vector<int64_t> lens(n);
    for (size_t i = 0; i < n; ++i) lens[i] = ds.records[i].output_len;
    std::vector<uint32_t> a(cfg.pairs_per_epoch), b(cfg.pairs_per_epoch);
    std::vector<int32_t> y(cfg.pairs_per_epoch);
    for (int epoch = 0; epoch < cfg.epochs; ++epoch) {
      const uint64_t epoch_seed = derive_seed(cfg.seed, 0x10000u + epoch);
      const int64_t np = pars_build_pairs(lens.data(), static_cast<int64_t>(n), cfg.delta,
                                          cfg.pairs_per_epoch, epoch_seed, a.data(), b.data(),
                                          y.data(), nullptr);
      b200::check(np);
      double epoch_loss = 0.0;
      uint64_t active = 0;
      b200::check(pars_sgd_epoch(b200::ctx(), dev.f, a.data(), b.data(), y.data(), np,
                                 cfg.batch_size, cfg.learning_rate, cfg.margin,
                                 model.scorer.weights().data(), model.scorer.bias(), &epoch_loss,
                                 &active));
      const double mean_loss = epoch_loss / static_cast<double>(np);
      if (!std::isfinite(mean_loss)) fail("training diverged at epoch %d", epoch);
      model.loss_trace.push_back(mean_loss);
    }
    return model;
  }

  // comparison baselines (train.cpp:168-209): GPU epochs (baselines.cu)
  train_baseline(ds, cfg, dev, model);
  return model;
}

}  // namespace pars
