// features.hpp over libpars_cuda (replaces proj/src/features.cpp; the
// reference's own error.cpp stays in the program — it is not on the hot path,
// so pars::strf / pars::fail resolve against it at load time).
// extract_features / extract_all run the fused GPU featurizer (featurize.cu, CSR mode); results are bit-identical to the
// reference (tests: the reference's own test_features.cpp, compiled against
// this file — oracle/Makefile `conformance`).
#include <cstdlib>
#include <mutex>

#include "shim.hpp"

namespace pars {

// ---- device context ---------------------------------------------------------
namespace b200 {

pars_ctx* ctx() {
  static std::once_flag once;
  static pars_ctx* c = nullptr;
  static std::string err;
  std::call_once(once, [] {
    const char* d = std::getenv("PARS_DEVICE");
    int dev = d ? std::atoi(d) : 0;
    if (pars_ctx_create(dev, &c) != PARS_OK) {
      err = pars_last_error();
      c = nullptr;
    }
  });
  if (!c) throw Error("libpars_cuda: no usable CUDA device: " + err);
  return c;
}

void check(int64_t rc) {
  if (rc < 0) throw Error(pars_last_error());
}

pars_extractor to_c(const FeatureExtractor& ex) {
  pars_extractor e{};
  e.kind = ex.kind == FeatureKind::HashedText ? 0 : 1;
  e.dim = ex.dim;
  e.norm = ex.norm == Normalization::L2 ? 1 : 0;
  if (ex.word_ngrams.size() > 8 || ex.char_ngrams.size() > 8)
    throw Error("libpars_cuda: at most 8 word and 8 char n-gram orders are supported");
  e.n_word = static_cast<int32_t>(ex.word_ngrams.size());
  e.n_char = static_cast<int32_t>(ex.char_ngrams.size());
  for (size_t k = 0; k < ex.word_ngrams.size(); ++k) e.word[k] = ex.word_ngrams[k];
  for (size_t k = 0; k < ex.char_ngrams.size(); ++k) e.chr[k] = ex.char_ngrams[k];
  return e;
}

Packed pack(const Dataset& ds) {
  Packed p;
  p.offsets.reserve(ds.records.size() + 1);
  size_t total = 0;
  for (const auto& r : ds.records) total += r.prompt_text.size();
  p.text.reserve(total);
  for (const auto& r : ds.records) {
    p.offsets.push_back(static_cast<int64_t>(p.text.size()));
    p.text += r.prompt_text;
  }
  p.offsets.push_back(static_cast<int64_t>(p.text.size()));
  return p;
}

Packed pack(const PromptRecord& rec) {
  Packed p;
  p.text = rec.prompt_text;
  p.offsets = {0, static_cast<int64_t>(p.text.size())};
  return p;
}

void check_embedding(const FeatureExtractor& ex, const PromptRecord& rec) {
  if (rec.embedding.empty())
    fail("prompt '%s' has no embedding but extractor kind is precomputed_embedding",
         rec.id.c_str());
  if (rec.embedding.size() != ex.dim)
    fail("prompt '%s': embedding length %zu != extractor dimension %u", rec.id.c_str(),
         rec.embedding.size(), ex.dim);
}

void extract_device(const FeatureExtractor& ex, const Dataset& ds, DeviceFeatures& out) {
  if (ex.dim == 0) throw Error("feature extractor dimension is 0");
  pars_extractor ce = to_c(ex);
  if (ex.kind == FeatureKind::PrecomputedEmbedding) {
    std::vector<double> X;
    X.reserve(ds.records.size() * static_cast<size_t>(ex.dim));
    for (const auto& r : ds.records) {
      check_embedding(ex, r);
      X.insert(X.end(), r.embedding.begin(), r.embedding.end());
    }
    std::vector<int64_t> offs(ds.records.size() + 1, 0);
    check(pars_extract(ctx(), &ce, "", offs.data(), static_cast<int64_t>(ds.records.size()),
                       X.data(), &out.f));
    return;
  }
  Packed p = pack(ds);
  check(pars_extract(ctx(), &ce, p.text.data(), p.offsets.data(),
                     static_cast<int64_t>(ds.records.size()), nullptr, &out.f));
}

void upload(uint32_t dim, const std::vector<const FeatureVec*>& rows, DeviceFeatures& out) {
  std::vector<int64_t> rp(rows.size() + 1, 0);
  std::vector<uint32_t> idx;
  std::vector<double> val;
  for (size_t i = 0; i < rows.size(); ++i) {
    for (const auto& [k, v] : rows[i]->entries) {
      idx.push_back(k);
      val.push_back(v);
    }
    rp[i + 1] = static_cast<int64_t>(idx.size());
  }
  check(pars_features_upload(ctx(), dim, static_cast<int64_t>(rows.size()), rp.data(), idx.data(),
                             val.data(), &out.f));
}

std::vector<FeatureVec> download(const DeviceFeatures& f) {
  const int64_t rows = pars_features_rows(f.f), nnz = pars_features_nnz(f.f);
  std::vector<int64_t> rp(rows + 1);
  std::vector<uint32_t> idx(std::max<int64_t>(nnz, 1));
  std::vector<double> val(std::max<int64_t>(nnz, 1));
  check(pars_features_download(ctx(), f.f, rp.data(), idx.data(), val.data()));
  std::vector<FeatureVec> out(rows);
  for (int64_t i = 0; i < rows; ++i) {
    out[i].entries.reserve(rp[i + 1] - rp[i]);
    for (int64_t k = rp[i]; k < rp[i + 1]; ++k) out[i].entries.emplace_back(idx[k], val[k]);
  }
  return out;
}

}  // namespace b200

// ---- features.cpp ---------------------------------------------------------
const char* feature_kind_name(FeatureKind kind) {
  return kind == FeatureKind::HashedText ? "hashed_text" : "precomputed_embedding";
}

const char* normalization_name(Normalization norm) {
  return norm == Normalization::L2 ? "l2" : "none";
}

FeatureVec extract_features(const FeatureExtractor& extractor, const PromptRecord& record) {
  Dataset one;
  one.records.push_back(record);
  b200::DeviceFeatures f;
  b200::extract_device(extractor, one, f);
  return std::move(b200::download(f)[0]);
}

std::vector<FeatureVec> extract_all(const FeatureExtractor& extractor, const Dataset& ds) {
  b200::DeviceFeatures f;
  b200::extract_device(extractor, ds, f);
  return b200::download(f);
}

std::vector<FeatureVec> extract_all_serial(const FeatureExtractor& extractor, const Dataset& ds) {
  return extract_all(extractor, ds);  // one deterministic GPU pass either way
}

}  // namespace pars
