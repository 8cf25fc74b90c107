// TEST INFRASTRUCTURE ONLY — never linked into the product.
//
// extern "C" wrapper over the *unmodified* reference library compiled from
// /root/reference/proj/src (see oracle/Makefile). Only tests/, the golden
// generator (tests/golden/make_golden.py), __graft_entry__.smoke() and
// bench.py's cpu_baseline / --impl reference legs load the resulting
// oracle/_ref/libpars_ref.so. It lets Python drive the reference's own public
// API (proj/include/pars/*.hpp) with flat arrays:
//   - synthesize_dataset / split_dataset / generate_poisson_arrivals
//   - extract_features, Scorer::score_batch, train, build_pairs,
//     select_batch, kendall_tau_b, run_simulation, compare_policies.
// Errors: every entry returns 0 on success, -1 on pars::Error (message via
// ref_last_error()).

#include <omp.h>

#include <algorithm>
#include <cstdint>
#include <cstring>
#include <optional>
#include <memory>
#include <string>
#include <vector>

#include "pars/arrivals.hpp"
#include "pars/dataset.hpp"
#include "pars/error.hpp"
#include "pars/features.hpp"
#include "pars/metrics.hpp"
#include "pars/pairs.hpp"
#include "pars/rng.hpp"
#include "pars/scheduler.hpp"
#include "pars/scorer.hpp"
#include "pars/simulator.hpp"
#include "pars/train.hpp"

using namespace pars;

namespace {
thread_local std::string g_err;

// Same field layout as pars_extractor in include/pars_cuda.h (plain C POD).
struct RefExtractor {
  int32_t kind;
  uint32_t dim;
  int32_t norm;
  int32_t n_word;
  int32_t n_char;
  int32_t word[8];
  int32_t chr[8];
};

FeatureExtractor to_ex(const RefExtractor* e) {
  FeatureExtractor ex;
  ex.kind = e->kind == 0 ? FeatureKind::HashedText : FeatureKind::PrecomputedEmbedding;
  ex.dim = e->dim;
  ex.norm = e->norm == 0 ? Normalization::None : Normalization::L2;
  ex.word_ngrams.assign(e->word, e->word + e->n_word);
  ex.char_ngrams.assign(e->chr, e->chr + e->n_char);
  return ex;
}

template <class F>
int guard(F&& f) {
  try {
    f();
    return 0;
  } catch (const std::exception& e) {
    g_err = e.what();
    return -1;
  }
}

struct SimHandle {
  SimResult res;
};

// Scores supplied by the caller (e.g. computed on the GPU), looked up by
// record index: the "GPU-scored priorities" policy of config C3.
class ArrayScorer : public Scorer {
 public:
  ArrayScorer(const Dataset& ds, const double* s) : ds_(ds), s_(s, s + ds.size()) {}
  double score(const PromptRecord& r) const override { return s_[ds_.index_of(r.id)]; }

 private:
  const Dataset& ds_;
  std::vector<double> s_;
};
}  // namespace

extern "C" {

const char* ref_last_error() { return g_err.c_str(); }
void ref_set_threads(int n) { omp_set_num_threads(n); }
int ref_max_threads() { return omp_get_max_threads(); }

// ---- datasets -------------------------------------------------------------
void* ref_synthesize(uint64_t n, double mu, double sigma, uint64_t seed,
                     int64_t embed_dim, int64_t max_len) {
  Dataset* ds = nullptr;
  int rc = guard([&] {
    SynthConfig cfg;
    cfg.n = n;
    cfg.components = {LengthComponent{mu, sigma, 1.0}};
    cfg.seed = seed;
    cfg.embed_dim = embed_dim;
    if (max_len > 0) cfg.max_len = max_len;
    ds = new Dataset(synthesize_dataset(cfg));
  });
  return rc == 0 ? ds : nullptr;
}

// ids are "p%06zu" unless ids_arena is given (NUL-separated arena + offsets).
void* ref_dataset_from_arrays(const char* text, const int64_t* offs,
                              const int64_t* out_len, const int64_t* prompt_len,
                              int64_t n, const double* emb, int64_t emb_dim) {
  auto* ds = new Dataset();
  ds->embedding_dim = emb ? emb_dim : 0;
  ds->records.resize(n);
  for (int64_t i = 0; i < n; ++i) {
    PromptRecord& r = ds->records[i];
    r.id = strf("p%06lld", static_cast<long long>(i));
    r.prompt_text.assign(text + offs[i], text + offs[i + 1]);
    r.output_len = out_len[i];
    r.prompt_len = prompt_len ? prompt_len[i] : whitespace_token_count(r.prompt_text);
    if (emb) r.embedding.assign(emb + i * emb_dim, emb + (i + 1) * emb_dim);
  }
  ds->build_index();
  return ds;
}

// load_dataset / save_dataset (dataset.cpp:73-195), for the ingestion parity
// tests; limit < 0 means no limit.
void* ref_load_dataset(const char* path, int64_t limit) {
  Dataset* ds = nullptr;
  int rc = guard([&] {
    std::optional<size_t> lim;
    if (limit >= 0) lim = static_cast<size_t>(limit);
    ds = new Dataset(load_dataset(path, lim));
  });
  return rc == 0 ? ds : nullptr;
}
int ref_save_dataset(void* h, const char* path) {
  return guard([&] { save_dataset(path, *static_cast<Dataset*>(h)); });
}
int64_t ref_dataset_samples(void* h, uint64_t i, int64_t* out, int64_t cap) {
  const auto& s = static_cast<Dataset*>(h)->records[i].output_len_samples;
  if (static_cast<int64_t>(s.size()) > cap) return -1;
  for (size_t k = 0; k < s.size(); ++k) out[k] = s[k];
  return static_cast<int64_t>(s.size());
}
void ref_dataset_free(void* ds) { delete static_cast<Dataset*>(ds); }
uint64_t ref_dataset_size(void* ds) { return static_cast<Dataset*>(ds)->size(); }
int64_t ref_dataset_text_bytes(void* h) {
  int64_t t = 0;
  for (auto& r : static_cast<Dataset*>(h)->records) t += r.prompt_text.size();
  return t;
}
int64_t ref_dataset_embed_dim(void* h) { return static_cast<Dataset*>(h)->embedding_dim; }

// Flatten: text arena + offsets[n+1] + output_len + prompt_len (+ embeddings).
void ref_dataset_export(void* h, char* text, int64_t* offs, int64_t* out_len,
                        int64_t* prompt_len, double* emb) {
  auto* ds = static_cast<Dataset*>(h);
  int64_t pos = 0;
  for (size_t i = 0; i < ds->size(); ++i) {
    const PromptRecord& r = ds->records[i];
    offs[i] = pos;
    std::memcpy(text + pos, r.prompt_text.data(), r.prompt_text.size());
    pos += r.prompt_text.size();
    out_len[i] = r.output_len;
    prompt_len[i] = r.prompt_len;
    if (emb && ds->embedding_dim > 0)
      std::memcpy(emb + i * ds->embedding_dim, r.embedding.data(),
                  sizeof(double) * ds->embedding_dim);
  }
  offs[ds->size()] = pos;
}

// Record ids, NUL-terminated, concatenated.
int64_t ref_dataset_id(void* h, uint64_t i, char* buf, int64_t cap) {
  const std::string& id = static_cast<Dataset*>(h)->records[i].id;
  if (static_cast<int64_t>(id.size()) + 1 > cap) return -1;
  std::memcpy(buf, id.c_str(), id.size() + 1);
  return static_cast<int64_t>(id.size());
}

void* ref_split(void* h, double val_frac, uint64_t seed, int which) {
  Dataset* out = nullptr;
  guard([&] {
    auto [tr, va] = split_dataset(*static_cast<Dataset*>(h), val_frac, seed);
    out = new Dataset(which == 0 ? std::move(tr) : std::move(va));
    out->build_index();
  });
  return out;
}

// Subset of records by index (e.g. "first 1,024 with prompt_len <= 128").
void* ref_subset(void* h, const int64_t* idx, int64_t n) {
  auto* src = static_cast<Dataset*>(h);
  auto* ds = new Dataset();
  ds->embedding_dim = src->embedding_dim;
  for (int64_t i = 0; i < n; ++i) ds->records.push_back(src->records[idx[i]]);
  ds->build_index();
  return ds;
}

// ---- features / scoring ---------------------------------------------------
int64_t ref_extract(const RefExtractor* e, const char* text, int64_t len,
                    const double* emb, int64_t emb_len, uint32_t* idx,
                    double* val, int64_t cap) {
  int64_t nnz = -1;
  int rc = guard([&] {
    PromptRecord rec;
    rec.id = "r";
    rec.prompt_text.assign(text, text + len);
    if (emb) rec.embedding.assign(emb, emb + emb_len);
    FeatureVec v = extract_features(to_ex(e), rec);
    nnz = static_cast<int64_t>(v.entries.size());
    for (int64_t k = 0; k < nnz && k < cap; ++k) {
      idx[k] = v.entries[k].first;
      val[k] = v.entries[k].second;
    }
  });
  return rc == 0 ? nnz : -1;
}

// extract_all over a dataset: row_ptr[n+1] plus entries (cap total).
int64_t ref_extract_all(const RefExtractor* e, void* h, int64_t* row_ptr,
                        uint32_t* idx, double* val, int64_t cap) {
  int64_t total = -1;
  int rc = guard([&] {
    auto feats = extract_all(to_ex(e), *static_cast<Dataset*>(h));
    int64_t pos = 0;
    for (size_t i = 0; i < feats.size(); ++i) {
      row_ptr[i] = pos;
      for (auto& [k, v] : feats[i].entries) {
        if (pos < cap) {
          idx[pos] = k;
          val[pos] = v;
        }
        ++pos;
      }
    }
    row_ptr[feats.size()] = pos;
    total = pos;
  });
  return rc == 0 ? total : -1;
}

int ref_score_batch(const RefExtractor* e, void* h, const double* w,
                    double bias, double* out) {
  return guard([&] {
    FeatureExtractor ex = to_ex(e);
    LinearScorer sc(ex, std::vector<double>(w, w + ex.dim), bias);
    auto s = sc.score_batch(*static_cast<Dataset*>(h));
    std::memcpy(out, s.data(), sizeof(double) * s.size());
  });
}

int ref_evaluate_ranking(const RefExtractor* e, void* h, const double* w,
                         double bias, double* tau, uint64_t* counts) {
  return guard([&] {
    FeatureExtractor ex = to_ex(e);
    LinearScorer sc(ex, std::vector<double>(w, w + ex.dim), bias);
    TauResult r = evaluate_ranking(sc, *static_cast<Dataset*>(h));
    *tau = r.tau_b;
    counts[0] = r.n_c; counts[1] = r.n_d; counts[2] = r.n0;
    counts[3] = r.n1; counts[4] = r.n2;
  });
}

// ---- training -------------------------------------------------------------
int ref_train(void* h, const RefExtractor* e, int objective, double delta,
              double margin, int epochs, int batch_size, double lr,
              uint64_t seed, uint64_t pairs_per_epoch, uint64_t lists_per_epoch,
              int list_size, double* w_out, double* bias_out, double* loss_trace_out) {
  return guard([&] {
    TrainConfig cfg;
    cfg.lists_per_epoch = lists_per_epoch;
    cfg.list_size = list_size;
    cfg.objective = static_cast<Objective>(objective);
    cfg.delta = delta;
    cfg.margin = margin;
    cfg.epochs = epochs;
    cfg.batch_size = batch_size;
    cfg.learning_rate = lr;
    cfg.seed = seed;
    cfg.pairs_per_epoch = pairs_per_epoch;
    cfg.extractor = to_ex(e);
    TrainedModel m = train(*static_cast<Dataset*>(h), cfg);
    const auto& w = m.scorer.weights();
    std::memcpy(w_out, w.data(), sizeof(double) * w.size());
    *bias_out = m.scorer.bias();
    for (size_t i = 0; i < m.loss_trace.size(); ++i) loss_trace_out[i] = m.loss_trace[i];
  });
}

// The epoch samplers of train()'s comparison objectives, which train.cpp
// keeps inline, restated over the reference's own Rng (rng.hpp): the
// PointwiseL1 order (train.cpp:169-172) and the ListMLE lists
// (train.cpp:186-200, ordered by sort_by_true_order, train.cpp:110-118).
int ref_pointwise_order(uint64_t n, uint64_t seed, uint32_t* out) {
  return guard([&] {
    std::vector<uint32_t> order(n);
    for (size_t i = 0; i < n; ++i) order[i] = static_cast<uint32_t>(i);
    Rng rng(seed);
    rng.shuffle(order);
    std::memcpy(out, order.data(), n * 4);
  });
}

int ref_listmle_lists(void* h, uint64_t nlists, int list_size, uint64_t seed, uint32_t* out) {
  return guard([&] {
    const Dataset& ds = *static_cast<Dataset*>(h);
    const size_t n = ds.records.size();
    const size_t k = std::min<size_t>(static_cast<size_t>(list_size), n);
    Rng rng(seed);
    std::vector<uint32_t> pool(n), list(k);
    for (size_t i = 0; i < n; ++i) pool[i] = static_cast<uint32_t>(i);
    for (size_t l = 0; l < nlists; ++l) {
      for (size_t t = 0; t < k; ++t) std::swap(pool[t], pool[t + rng.below(n - t)]);
      std::copy_n(pool.begin(), k, list.begin());
      std::sort(list.begin(), list.end(), [&](uint32_t a, uint32_t b) {
        const auto& ra = ds.records[a];
        const auto& rb = ds.records[b];
        if (ra.output_len != rb.output_len) return ra.output_len > rb.output_len;
        return ra.id < rb.id;
      });
      std::memcpy(out + l * k, list.data(), k * 4);
    }
  });
}

int64_t ref_build_pairs(void* h, double delta, uint64_t max_pairs,
                        uint64_t seed, uint32_t* a, uint32_t* b, int32_t* y,
                        double* rel) {
  int64_t n = -1;
  int rc = guard([&] {
    auto p = build_pairs(*static_cast<Dataset*>(h), delta, max_pairs, seed);
    n = static_cast<int64_t>(p.size());
    for (size_t i = 0; i < p.size(); ++i) {
      a[i] = p[i].a;
      b[i] = p[i].b;
      y[i] = p[i].y;
      rel[i] = p[i].rel_diff;
    }
  });
  return rc == 0 ? n : -1;
}

double ref_relative_length_difference(int64_t a, int64_t b) {
  return relative_length_difference(a, b);
}

double ref_margin_ranking_loss(double sa, double sb, int y, double m) {
  return margin_ranking_loss(sa, sb, y, m);
}

// pairwise_loss_grad on two explicit sparse vectors (train.cpp:34-44).
int ref_pairwise_loss_grad(const double* w, uint32_t dim, double bias,
                           const uint32_t* ia, const double* va, int64_t na,
                           const uint32_t* ib, const double* vb, int64_t nb,
                           int y, double margin, double* grad, double* loss) {
  return guard([&] {
    FeatureExtractor ex;
    ex.dim = dim;
    LinearScorer sc(ex, std::vector<double>(w, w + dim), bias);
    FeatureVec a, b;
    for (int64_t k = 0; k < na; ++k) a.entries.emplace_back(ia[k], va[k]);
    for (int64_t k = 0; k < nb; ++k) b.entries.emplace_back(ib[k], vb[k]);
    std::vector<double> g(grad, grad + dim);
    *loss = pairwise_loss_grad(sc, a, b, y, margin, g);
    std::memcpy(grad, g.data(), sizeof(double) * dim);
  });
}

// C4 padding: every prompt padded with " w<k>" tokens,
// k = Rng(pad_seed).below(50) (the reference's own Rng, rng.hpp), to exactly
// pad_tokens whitespace tokens, records in order. Used by bench.py's
// reference arm on a dataset from the reference's synthesize_dataset.
int ref_pad_dataset(void* h, int64_t pad_tokens, uint64_t pad_seed) {
  return guard([&] {
    Dataset& ds = *static_cast<Dataset*>(h);
    Rng pad(pad_seed);
    for (PromptRecord& r : ds.records) {
      for (int64_t k = r.prompt_len; k < pad_tokens; ++k) {
        r.prompt_text += " w";
        r.prompt_text += std::to_string(pad.below(50));
      }
      r.prompt_len = std::max<int64_t>(r.prompt_len, pad_tokens);
    }
  });
}

// The C4 step on the reference's own code path: LinearScorer::score_batch
// over the dataset (scorer.cpp:9-24, OpenMP), then the requests of a burst
// (arrival 0, the record ids) ordered by select_batch (scheduler.cpp:33-60)
// with every slot free. scores: n doubles, order: n indices.
int ref_score_order(const RefExtractor* e, void* h, const double* w, double bias,
                    double* scores, uint64_t* order) {
  return guard([&] {
    const Dataset& ds = *static_cast<Dataset*>(h);
    FeatureExtractor ex = to_ex(e);
    LinearScorer sc(ex, std::vector<double>(w, w + ex.dim), bias);
    std::vector<double> s = sc.score_batch(ds);
    std::vector<Request> q(ds.records.size());
    for (size_t i = 0; i < q.size(); ++i) {
      q[i].record_idx = static_cast<uint32_t>(i);
      q[i].prompt_id = ds.records[i].id;
      q[i].arrival_time = 0.0;
      q[i].score = s[i];
    }
    PolicyConfig cfg;
    auto sel = select_batch(q, 0.0, q.size(), cfg);
    std::memcpy(scores, s.data(), sizeof(double) * s.size());
    for (size_t i = 0; i < sel.size(); ++i) order[i] = sel[i];
  });
}

// ---- scheduling -----------------------------------------------------------
// ids: NUL-separated arena with offsets; out: selected indices.
int64_t ref_select_batch(int64_t n, const double* arrival, const char* ids,
                         const int64_t* id_offs, const double* score,
                         const uint8_t* boosted, double now,
                         uint64_t free_slots, uint64_t* out) {
  int64_t k = -1;
  int rc = guard([&] {
    std::vector<Request> w(n);
    for (int64_t i = 0; i < n; ++i) {
      w[i].prompt_id.assign(ids + id_offs[i], ids + id_offs[i + 1]);
      w[i].arrival_time = arrival[i];
      w[i].score = score[i];
      w[i].boosted = boosted[i] != 0;
    }
    PolicyConfig cfg;
    auto sel = select_batch(w, now, free_slots, cfg);
    k = static_cast<int64_t>(sel.size());
    for (size_t i = 0; i < sel.size(); ++i) out[i] = sel[i];
  });
  return rc == 0 ? k : -1;
}

int ref_kendall(const double* x, const double* y, int64_t n, int serial,
                double* tau, uint64_t* counts) {
  return guard([&] {
    std::span<const double> xs(x, n), ys(y, n);
    TauResult r = serial ? kendall_tau_b_serial(xs, ys) : kendall_tau_b(xs, ys);
    *tau = r.tau_b;
    counts[0] = r.n_c; counts[1] = r.n_d; counts[2] = r.n0;
    counts[3] = r.n1; counts[4] = r.n2;
  });
}

// ---- simulation -----------------------------------------------------------
// policy: 0 fcfs, 1 pars (linear scorer with w/bias), 2 oracle,
//         3 precomputed scores (w = per-record scores).
// arrivals: per-record times in dataset order (NULL -> burst at 0).
void* ref_simulate(void* h, const double* arrivals, int policy,
                   const RefExtractor* e, const double* w, double bias,
                   int batch_limit, double starvation_s, int record_events) {
  SimHandle* out = nullptr;
  guard([&] {
    auto* ds = static_cast<Dataset*>(h);
    ds->build_index();
    ArrivalTrace tr;
    for (size_t i = 0; i < ds->size(); ++i)
      tr.entries.push_back({ds->records[i].id, arrivals ? arrivals[i] : 0.0});
    SimConfig cfg;
    cfg.policy.batch_limit = batch_limit;
    cfg.policy.starvation_threshold_s = starvation_s;
    cfg.record_events = record_events != 0;
    if (policy == 0) {
      cfg.policy.policy = make_fcfs_policy();
    } else if (policy == 1) {
      FeatureExtractor ex = to_ex(e);
      auto sc = std::make_shared<LinearScorer>(ex, std::vector<double>(w, w + ex.dim), bias);
      cfg.policy.policy = make_sjf_policy("pars", sc);
    } else if (policy == 2) {
      cfg.policy.policy = make_sjf_policy("oracle", std::make_shared<OracleScorer>(*ds));
    } else {
      cfg.policy.policy = make_sjf_policy("pars-gpu", std::make_shared<ArrayScorer>(*ds, w));
    }
    auto* sh = new SimHandle();
    sh->res = run_simulation(tr, *ds, cfg);
    out = sh;
  });
  return out;
}

void ref_sim_free(void* s) { delete static_cast<SimHandle*>(s); }
uint64_t ref_sim_iterations(void* s) { return static_cast<SimHandle*>(s)->res.iterations; }
double ref_sim_seconds(void* s) { return static_cast<SimHandle*>(s)->res.simulated_seconds; }
uint64_t ref_sim_count(void* s) { return static_cast<SimHandle*>(s)->res.requests.size(); }
// per completed request (completion order): record index (from id), arrival,
// admit, finish, per-token latency.
void ref_sim_requests(void* s, void* h, int64_t* rec, double* arrival,
                      double* admit, double* finish, double* ptl) {
  auto* sh = static_cast<SimHandle*>(s);
  auto* ds = static_cast<Dataset*>(h);
  for (size_t i = 0; i < sh->res.requests.size(); ++i) {
    const RequestRecord& r = sh->res.requests[i];
    rec[i] = static_cast<int64_t>(ds->index_of(r.prompt_id));
    arrival[i] = r.arrival_s;
    admit[i] = r.admit_s;
    finish[i] = r.finish_s;
    ptl[i] = r.per_token_latency_s;
  }
}
int ref_sim_summary(void* s, double* mean_ms, double* p90_ms) {
  return guard([&] {
    LatencySummary L = latency_summary(static_cast<SimHandle*>(s)->res);
    *mean_ms = L.mean_per_token_ms;
    *p90_ms = L.p90_per_token_ms;
  });
}

int ref_poisson(void* h, double rate, uint64_t seed, double* times) {
  return guard([&] {
    ArrivalTrace t = generate_poisson_arrivals(*static_cast<Dataset*>(h), rate, seed);
    for (size_t i = 0; i < t.entries.size(); ++i) times[i] = t.entries[i].arrival_time_s;
  });
}

}  // extern "C"
