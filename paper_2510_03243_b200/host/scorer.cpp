// scorer.hpp over libpars_cuda (replaces proj/src/scorer.cpp).
// LinearScorer scoring — single prompts, batches and FeatureVecs — runs the
// GPU kernels in exact fp64 mode (bit-identical to features.hpp:31-35 +
// scorer.cpp:40-42). Scorer::score_batch is non-virtual in the reference
// header, so it dispatches on the exact dynamic type: LinearScorer -> one
// fused GPU launch over the whole dataset; any other Scorer (OracleScorer,
// user subclasses of Scorer or of LinearScorer) keeps the per-record virtual
// call, so overrides are honoured as in scorer.cpp:13-21.
#include <exception>
#include <typeinfo>

#include "pars/metrics.hpp"
#include "pars/scorer.hpp"
#include "shim.hpp"

namespace pars {

namespace {

std::vector<double> linear_scores(const LinearScorer& s, const Dataset& ds) {
  const FeatureExtractor& ex = s.extractor();
  if (ex.dim == 0) throw Error("feature extractor dimension is 0");
  std::vector<double> out(ds.records.size());
  if (ds.records.empty()) return out;
  pars_extractor ce = b200::to_c(ex);
  if (ex.kind == FeatureKind::PrecomputedEmbedding) {
    std::vector<double> X;
    X.reserve(ds.records.size() * static_cast<size_t>(ex.dim));
    for (const auto& r : ds.records) {
      b200::check_embedding(ex, r);
      X.insert(X.end(), r.embedding.begin(), r.embedding.end());
    }
    b200::check(pars_score_embeddings(b200::ctx(), &ce, X.data(),
                                      static_cast<int64_t>(ds.records.size()), s.weights().data(),
                                      s.bias(), PARS_MODE_EXACT_F64, out.data()));
    return out;
  }
  // the records' own strings, gathered by the library into pinned staging
  // (no packing pass over the dataset)
  const size_t n = ds.records.size();
  std::vector<const char*> texts(n);
  std::vector<int64_t> lens(n);
  for (size_t i = 0; i < n; ++i) {
    texts[i] = ds.records[i].prompt_text.data();
    lens[i] = static_cast<int64_t>(ds.records[i].prompt_text.size());
  }
  b200::check(pars_score_records(b200::ctx(), &ce, texts.data(), lens.data(), static_cast<int64_t>(n),
                                 s.weights().data(), s.bias(), PARS_MODE_EXACT_F64, out.data()));
  return out;
}

}  // namespace

std::vector<double> Scorer::score_batch(const Dataset& ds) const {
  // exact type, not dynamic_cast: a subclass of LinearScorer may override
  // score(const PromptRecord&), and the reference's loop (scorer.cpp:16)
  // calls that override
  if (typeid(*this) == typeid(LinearScorer))
    return linear_scores(static_cast<const LinearScorer&>(*this), ds);
  std::vector<double> out(ds.records.size());
  for (size_t i = 0; i < ds.records.size(); ++i) out[i] = score(ds.records[i]);
  return out;
}

LinearScorer::LinearScorer(FeatureExtractor extractor, std::vector<double> weights, double bias)
    : extractor_(std::move(extractor)), weights_(std::move(weights)), bias_(bias) {
  if (weights_.size() != extractor_.dim)
    fail("weight vector length %zu != extractor dimension %u", weights_.size(), extractor_.dim);
}

double LinearScorer::score(const PromptRecord& record) const {
  Dataset one;
  one.records.push_back(record);
  return linear_scores(*this, one)[0];
}

double LinearScorer::score(const FeatureVec& features) const {
  b200::DeviceFeatures f;
  b200::upload(extractor_.dim, {&features}, f);
  double s = 0.0;
  b200::check(pars_features_score(b200::ctx(), f.f, weights_.data(), bias_, &s));
  return s;
}

TauResult evaluate_ranking(const Scorer& scorer, const Dataset& ds) {
  std::vector<double> scores = scorer.score_batch(ds);
  std::vector<double> truth(ds.records.size());
  for (size_t i = 0; i < ds.records.size(); ++i)
    truth[i] = static_cast<double>(ds.records[i].output_len);
  return kendall_tau_b(scores, truth);
}

OracleScorer::OracleScorer(const Dataset& ds) {
  lengths_.reserve(ds.records.size());
  for (const PromptRecord& rec : ds.records) lengths_.emplace(rec.id, rec.output_len);
}

double OracleScorer::score(const PromptRecord& record) const {
  auto it = lengths_.find(record.id);
  if (it == lengths_.end()) fail("oracle scorer: unknown prompt id '%s'", record.id.c_str());
  return static_cast<double>(it->second);
}

}  // namespace pars
