/* TEST INFRASTRUCTURE ONLY — see pars_oracle.h for the contract.
 * Plain-C restatement of the reference's predictor hot path; each function
 * cites the reference file:line (paths relative to /root/reference/proj). */
#include "pars_oracle.h"

#include <math.h>
#include <stdarg.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

static __thread char g_err[512];
const char* po_last_error(void) { return g_err; }
static void set_err(const char* fmt, ...) {
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(g_err, sizeof g_err, fmt, ap);
  va_end(ap);
}

/* ---- rng.hpp:10-75 ------------------------------------------------------ */
uint64_t po_splitmix64(uint64_t x) { /* rng.hpp:10-15 */
  x += 0x9e3779b97f4a7c15ull;
  x = (x ^ (x >> 30)) * 0xbf58476d1ce4e5b9ull;
  x = (x ^ (x >> 27)) * 0x94d049bb133111ebull;
  return x ^ (x >> 31);
}
uint64_t po_derive_seed(uint64_t seed, uint64_t stream) { /* rng.hpp:18-20 */
  return po_splitmix64(seed ^ po_splitmix64(stream));
}
/* std::mt19937_64 as specified by [rand.predef] (rng.hpp:73 uses it). */
void po_rng_seed(po_rng* r, uint64_t seed) {
  r->mt[0] = seed;
  for (int i = 1; i < 312; ++i)
    r->mt[i] = 6364136223846793005ull * (r->mt[i - 1] ^ (r->mt[i - 1] >> 62)) + (uint64_t)i;
  r->mti = 312;
}
uint64_t po_rng_u64(po_rng* r) {
  const uint64_t UM = 0xFFFFFFFF80000000ull, LM = 0x7FFFFFFFull;
  const uint64_t A = 0xB5026F5AA96619E9ull;
  if (r->mti >= 312) {
    int i;
    for (i = 0; i < 312 - 156; ++i) {
      uint64_t x = (r->mt[i] & UM) | (r->mt[i + 1] & LM);
      r->mt[i] = r->mt[i + 156] ^ (x >> 1) ^ ((x & 1) ? A : 0);
    }
    for (; i < 311; ++i) {
      uint64_t x = (r->mt[i] & UM) | (r->mt[i + 1] & LM);
      r->mt[i] = r->mt[i + 156 - 312] ^ (x >> 1) ^ ((x & 1) ? A : 0);
    }
    uint64_t x = (r->mt[311] & UM) | (r->mt[0] & LM);
    r->mt[311] = r->mt[155] ^ (x >> 1) ^ ((x & 1) ? A : 0);
    r->mti = 0;
  }
  uint64_t x = r->mt[r->mti++];
  x ^= (x >> 29) & 0x5555555555555555ull;
  x ^= (x << 17) & 0x71D67FFFEDA60000ull;
  x ^= (x << 37) & 0xFFF7EEE000000000ull;
  x ^= x >> 43;
  return x;
}
uint64_t po_rng_below(po_rng* r, uint64_t n) { /* rng.hpp:34-38 (Lemire) */
  return (uint64_t)(((unsigned __int128)po_rng_u64(r) * n) >> 64);
}

/* ---- features.cpp ------------------------------------------------------- */
static uint64_t fnv1a(const unsigned char* d, int64_t len, uint64_t h) { /* :17-23 */
  for (int64_t i = 0; i < len; ++i) {
    h ^= d[i];
    h *= 0x100000001b3ull;
  }
  return h;
}
static uint64_t salt(uint64_t field, uint64_t order) { /* :25-27 */
  return po_splitmix64(0xcbf29ce484222325ull ^ (field << 32) ^ order);
}
static int is_space(unsigned char c) { /* C-locale std::isspace, :40-44 */
  return c == ' ' || c == '\t' || c == '\n' || c == '\v' || c == '\f' || c == '\r';
}

typedef struct {
  uint32_t idx;
  double v;
} entry;

static int cmp_entry(const void* a, const void* b) {
  uint32_t x = ((const entry*)a)->idx, y = ((const entry*)b)->idx;
  return x < y ? -1 : (x > y);
}

/* Returns nnz; entries (malloc'ed) in *out. */
static int64_t extract_one(const po_extractor* ex, const char* text, int64_t len,
                           const double* emb, int64_t emb_len, entry** out) {
  *out = NULL;
  if (ex->dim == 0) { /* :63 */
    set_err("feature extractor dimension is 0");
    return -1;
  }
  entry* raw = NULL;
  int64_t nraw = 0;
  if (ex->kind == 1) { /* :67-76 */
    if (emb == NULL || emb_len == 0) {
      set_err("prompt has no embedding but extractor kind is precomputed_embedding");
      return -1;
    }
    if (emb_len != (int64_t)ex->dim) {
      set_err("embedding length %lld != extractor dimension %u", (long long)emb_len, ex->dim);
      return -1;
    }
    raw = (entry*)malloc(sizeof(entry) * (emb_len ? emb_len : 1));
    for (int64_t i = 0; i < emb_len; ++i) raw[i] = (entry){(uint32_t)i, emb[i]};
    nraw = emb_len;
  } else {
    /* split_tokens :36-49 */
    int64_t ntok = 0;
    int64_t* ts = (int64_t*)malloc(sizeof(int64_t) * (len + 1));
    int64_t* tl = (int64_t*)malloc(sizeof(int64_t) * (len + 1));
    const unsigned char* u = (const unsigned char*)text;
    for (int64_t i = 0; i < len;) {
      while (i < len && is_space(u[i])) ++i;
      int64_t s = i;
      while (i < len && !is_space(u[i])) ++i;
      if (i > s) {
        ts[ntok] = s;
        tl[ntok] = i - s;
        ++ntok;
      }
    }
    int64_t cap = 0;
    for (int k = 0; k < ex->n_word; ++k) cap += ntok;
    for (int k = 0; k < ex->n_char; ++k) cap += len;
    raw = (entry*)malloc(sizeof(entry) * (cap ? cap : 1));
    for (int k = 0; k < ex->n_word; ++k) { /* :80-92 */
      int order = ex->word[k];
      if (order < 1) {
        set_err("word n-gram order must be >= 1");
        free(ts); free(tl); free(raw);
        return -1;
      }
      uint64_t s = salt(1, (uint64_t)order);
      if (ntok < order) continue;
      for (int64_t i = 0; i + order <= ntok; ++i) {
        uint64_t h = s;
        for (int j = 0; j < order; ++j) {
          h = fnv1a(u + ts[i + j], tl[i + j], h);
          h = fnv1a((const unsigned char*)"\x1f", 1, h);
        }
        raw[nraw++] = (entry){(uint32_t)((h >> 1) % ex->dim), (h & 1) ? 1.0 : -1.0}; /* :29-34 */
      }
    }
    for (int k = 0; k < ex->n_char; ++k) { /* :93-101 */
      int order = ex->chr[k];
      if (order < 1) {
        set_err("char n-gram order must be >= 1");
        free(ts); free(tl); free(raw);
        return -1;
      }
      uint64_t s = salt(2, (uint64_t)order);
      for (int64_t t = 0; t < ntok; ++t) {
        if (tl[t] < order) continue;
        for (int64_t i = 0; i + order <= tl[t]; ++i) {
          uint64_t h = fnv1a(u + ts[t] + i, order, s);
          raw[nraw++] = (entry){(uint32_t)((h >> 1) % ex->dim), (h & 1) ? 1.0 : -1.0};
        }
      }
    }
    free(ts);
    free(tl);
    /* sort by idx :102-103, merge :104-109, erase zeros :110 */
    qsort(raw, (size_t)nraw, sizeof(entry), cmp_entry);
    int64_t m = 0;
    for (int64_t i = 0; i < nraw; ++i) {
      if (m > 0 && raw[m - 1].idx == raw[i].idx)
        raw[m - 1].v += raw[i].v;
      else
        raw[m++] = raw[i];
    }
    int64_t z = 0;
    for (int64_t i = 0; i < m; ++i)
      if (raw[i].v != 0.0) raw[z++] = raw[i];
    nraw = z;
  }
  if (ex->norm == 1) { /* :113-120 */
    double sq = 0.0;
    for (int64_t i = 0; i < nraw; ++i) sq += raw[i].v * raw[i].v;
    if (sq > 0.0) {
      double inv = 1.0 / sqrt(sq);
      for (int64_t i = 0; i < nraw; ++i) raw[i].v *= inv;
    }
  }
  *out = raw;
  return nraw;
}

int64_t po_extract(const po_extractor* ex, const char* text, int64_t len,
                   const double* emb, int64_t emb_len, uint32_t* idx,
                   double* val, int64_t cap) {
  entry* e;
  int64_t n = extract_one(ex, text, len, emb, emb_len, &e);
  if (n < 0) return -1;
  for (int64_t i = 0; i < n && i < cap; ++i) {
    idx[i] = e[i].idx;
    val[i] = e[i].v;
  }
  free(e);
  return n;
}

int64_t po_extract_all(const po_extractor* ex, const char* text,
                       const int64_t* offs, int64_t n, int64_t* row_ptr,
                       uint32_t* idx, double* val, int64_t cap) {
  int64_t pos = 0;
  for (int64_t i = 0; i < n; ++i) {
    entry* e;
    int64_t k = extract_one(ex, text + offs[i], offs[i + 1] - offs[i], NULL, 0, &e);
    if (k < 0) return -1;
    row_ptr[i] = pos;
    for (int64_t j = 0; j < k; ++j, ++pos)
      if (pos < cap) {
        idx[pos] = e[j].idx;
        val[pos] = e[j].v;
      }
    free(e);
  }
  row_ptr[n] = pos;
  return pos;
}

/* FeatureVec::dot (features.hpp:31-35) + bias (scorer.cpp:40-42). */
static double dot_bias(const entry* e, int64_t n, const double* w, double bias) {
  double s = 0.0;
  for (int64_t i = 0; i < n; ++i) s += w[e[i].idx] * e[i].v;
  return s + bias;
}

int po_score_batch(const po_extractor* ex, const char* text,
                   const int64_t* offs, int64_t n, const double* w,
                   double bias, double* out, int nthreads) {
  int failed = 0;
#pragma omp parallel for schedule(dynamic, 256) num_threads(nthreads > 0 ? nthreads : 1)
  for (int64_t i = 0; i < n; ++i) {
    entry* e;
    int64_t k = extract_one(ex, text + offs[i], offs[i + 1] - offs[i], NULL, 0, &e);
    if (k < 0) {
      failed = 1;
      continue;
    }
    out[i] = dot_bias(e, k, w, bias);
    free(e);
  }
  return failed ? -1 : 0;
}

int po_score_dense(const po_extractor* ex, const double* X, int64_t n,
                   const double* w, double bias, double* out) {
  for (int64_t i = 0; i < n; ++i) {
    entry* e;
    int64_t k = extract_one(ex, NULL, 0, X + i * (int64_t)ex->dim, ex->dim, &e);
    if (k < 0) return -1;
    out[i] = dot_bias(e, k, w, bias);
    free(e);
  }
  return 0;
}

/* ---- pairs.hpp / pairs.cpp ---------------------------------------------- */
double po_rel_diff(int64_t a, int64_t b) { /* pairs.hpp:21-24 */
  return (double)llabs(a - b) / (double)(a > b ? a : b);
}
double po_margin_loss(double sa, double sb, int y, double margin) { /* :27-31 */
  double v = -(double)y * (sa - sb) + margin;
  return v > 0.0 ? v : 0.0;
}
void po_dmin_table(double delta, int64_t max_len, int32_t* table) {
  table[0] = INT32_MAX;
  for (int64_t m = 1; m <= max_len; ++m) {
    int32_t d = INT32_MAX;
    for (int64_t k = 1; k <= m; ++k)
      if (!(po_rel_diff(m, m - k) < delta)) {
        d = (int32_t)k;
        break;
      }
    table[m] = d;
  }
}

int64_t po_build_pairs(const int64_t* lens, int64_t n, double delta,
                       uint64_t max_pairs, uint64_t seed, uint32_t* a,
                       uint32_t* b, int32_t* y, double* rel) {
  if (n == 0) { set_err("build_pairs: empty dataset"); return -1; }
  if (delta < 0.0 || delta >= 1.0) { set_err("build_pairs: delta %g outside [0, 1)", delta); return -1; }
  if (max_pairs == 0) { set_err("build_pairs: max_pairs must be >= 1"); return -1; }
  int64_t cnt = 0;
  if (n >= 2) {
    po_rng r;
    po_rng_seed(&r, seed);
    uint64_t budget = 50ull * max_pairs; /* kSamplingBudgetFactor, pairs.hpp:36 */
    for (uint64_t draw = 0; draw < budget && (uint64_t)cnt < max_pairs; ++draw) {
      uint32_t i = (uint32_t)po_rng_below(&r, (uint64_t)n);
      uint32_t j = (uint32_t)po_rng_below(&r, (uint64_t)n - 1);
      if (j >= i) ++j;
      int64_t la = lens[i], lb = lens[j];
      if (la == lb) continue;
      double rd = po_rel_diff(la, lb);
      if (rd < delta) continue;
      a[cnt] = i; b[cnt] = j; y[cnt] = la > lb ? 1 : -1; rel[cnt] = rd;
      ++cnt;
    }
  }
  if (cnt == 0) { set_err("no informative pairs"); return -1; }
  return cnt;
}

/* ---- train.cpp ---------------------------------------------------------- */
static double csr_score(const int64_t* rp, const uint32_t* idx, const double* val,
                        int64_t r, const double* w, double bias) {
  double s = 0.0;
  for (int64_t k = rp[r]; k < rp[r + 1]; ++k) s += w[idx[k]] * val[k];
  return s + bias;
}

int po_sgd_epoch(const int64_t* rp, const uint32_t* idx, const double* val,
                 uint32_t dim, const uint32_t* a, const uint32_t* b,
                 const int32_t* y, int64_t npairs, int batch, double lr,
                 double margin, double* w, double bias, double* epoch_loss,
                 uint64_t* active) {
  double* grad = (double*)calloc(dim, sizeof(double));
  double el = *epoch_loss;
  uint64_t act = 0;
  for (int64_t start = 0; start < npairs; start += batch) { /* train.cpp:156-165 */
    int64_t end = start + batch < npairs ? start + batch : npairs;
    for (int64_t p = start; p < end; ++p) { /* pairwise_loss_grad :34-44 */
      double loss = po_margin_loss(csr_score(rp, idx, val, a[p], w, bias),
                                   csr_score(rp, idx, val, b[p], w, bias), y[p], margin);
      if (loss > 0.0) {
        ++act;
        for (int64_t k = rp[a[p]]; k < rp[a[p] + 1]; ++k) grad[idx[k]] -= y[p] * val[k];
        for (int64_t k = rp[b[p]]; k < rp[b[p] + 1]; ++k) grad[idx[k]] += y[p] * val[k];
      }
      el += loss;
    }
    double scale = lr / (double)(end - start); /* apply :141-151 */
    for (uint32_t d = 0; d < dim; ++d)
      if (grad[d] != 0.0) {
        w[d] -= scale * grad[d];
        grad[d] = 0.0;
      }
  }
  free(grad);
  *epoch_loss = el;
  *active = act;
  return 0;
}

int po_train_pairwise(const int64_t* rp, const uint32_t* idx, const double* val,
                      const int64_t* lens, int64_t n, uint32_t dim, double delta,
                      double margin, int epochs, int batch, double lr,
                      uint64_t seed, uint64_t ppe, double* w, double* bias_out,
                      double* loss_trace) {
  memset(w, 0, sizeof(double) * dim);
  double bias = 0.0;
  uint32_t* a = (uint32_t*)malloc(sizeof(uint32_t) * ppe);
  uint32_t* b = (uint32_t*)malloc(sizeof(uint32_t) * ppe);
  int32_t* y = (int32_t*)malloc(sizeof(int32_t) * ppe);
  double* rel = (double*)malloc(sizeof(double) * ppe);
  int rc = 0;
  for (int e = 0; e < epochs; ++e) {
    uint64_t es = po_derive_seed(seed, 0x10000u + (uint64_t)e); /* :137 */
    int64_t np = po_build_pairs(lens, n, delta, ppe, es, a, b, y, rel);
    if (np < 0) { rc = -1; break; }
    double el = 0.0;
    uint64_t act;
    po_sgd_epoch(rp, idx, val, dim, a, b, y, np, batch, lr, margin, w, bias, &el, &act);
    double mean = el / (double)np; /* :212-216 */
    if (!isfinite(mean)) { set_err("training diverged at epoch %d", e); rc = -1; break; }
    loss_trace[e] = mean;
  }
  free(a); free(b); free(y); free(rel);
  *bias_out = bias;
  return rc;
}

/* ---- all-pairs ---------------------------------------- */
int po_allpairs(const double* s, const int64_t* lens, int64_t n, double delta,
                double margin, int32_t* coeff, uint64_t* kept, uint64_t* active,
                double* loss_sum, int nthreads) {
  uint64_t K = 0, A = 0;
  double L = 0.0;
  memset(coeff, 0, sizeof(int32_t) * n);
  /* rows are independent given the symmetric form c_i = sum_j active(i,j)
   * * (-y_ij) with y_ij = sign(L_i - L_j); loss/kept/active count i<j. */
#pragma omp parallel for schedule(dynamic, 64) reduction(+ : K, A, L) num_threads(nthreads > 0 ? nthreads : 1)
  for (int64_t i = 0; i < n; ++i) {
    int32_t ci = 0;
    for (int64_t j = 0; j < n; ++j) {
      if (j == i) continue;
      int64_t la = lens[i], lb = lens[j];
      if (la == lb) continue;
      if (po_rel_diff(la, lb) < delta) continue;
      int y = la > lb ? 1 : -1;
      double h = -(double)y * (s[i] - s[j]) + margin;
      if (j > i) ++K;
      if (h > 0.0) {
        ci -= y;
        if (j > i) {
          ++A;
          L += h;
        }
      }
    }
    coeff[i] = ci;
  }
  *kept = K;
  *active = A;
  *loss_sum = L;
  return 0;
}

void po_xt_c(const int64_t* rp, const uint32_t* idx, const double* val,
             int64_t n, const int32_t* coeff, uint32_t dim, double* grad) {
  memset(grad, 0, sizeof(double) * dim);
  for (int64_t i = 0; i < n; ++i)
    if (coeff[i] != 0)
      for (int64_t k = rp[i]; k < rp[i + 1]; ++k) grad[idx[k]] += (double)coeff[i] * val[k];
}

/* ---- scheduler.cpp:33-60 ------------------------------------------------ */
typedef struct {
  int64_t n;
  const double* arrival;
  const char* ids;
  const int64_t* offs;
  const double* score;
  const uint8_t* boosted;
} sel_ctx;

static int tie_less(const sel_ctx* c, int64_t a, int64_t b, int* equal) {
  *equal = 0;
  if (c->arrival[a] != c->arrival[b]) return c->arrival[a] < c->arrival[b];
  int64_t la = c->offs[a + 1] - c->offs[a], lb = c->offs[b + 1] - c->offs[b];
  int64_t m = la < lb ? la : lb;
  int r = memcmp(c->ids + c->offs[a], c->ids + c->offs[b], (size_t)m); /* unsigned bytes */
  if (r != 0) return r < 0;
  if (la != lb) return la < lb;
  *equal = 1;
  return 0;
}
static int sel_less(const sel_ctx* c, int64_t ia, int64_t ib) {
  int ba = c->boosted[ia] != 0, bb = c->boosted[ib] != 0;
  if (ba != bb) return ba; /* boosted precede all */
  if (!ba && c->score[ia] != c->score[ib]) return c->score[ia] < c->score[ib];
  int eq;
  int lt = tie_less(c, ia, ib, &eq);
  if (!eq) return lt;
  return ia < ib;
}
static void merge_sort(const sel_ctx* c, int64_t* v, int64_t* tmp, int64_t n) {
  if (n < 2) return;
  int64_t h = n / 2;
  merge_sort(c, v, tmp, h);
  merge_sort(c, v + h, tmp, n - h);
  int64_t i = 0, j = h, k = 0;
  while (i < h && j < n) tmp[k++] = sel_less(c, v[j], v[i]) ? v[j++] : v[i++];
  while (i < h) tmp[k++] = v[i++];
  while (j < n) tmp[k++] = v[j++];
  memcpy(v, tmp, sizeof(int64_t) * n);
}
int po_select_order(int64_t n, const double* arrival, const char* ids,
                    const int64_t* id_offs, const double* score,
                    const uint8_t* boosted, double now, int64_t* order) {
  sel_ctx c = {n, arrival, ids, id_offs, score, boosted};
  for (int64_t i = 0; i < n; ++i) order[i] = i;
  int64_t* tmp = (int64_t*)malloc(sizeof(int64_t) * (n ? n : 1));
  merge_sort(&c, order, tmp, n);
  free(tmp);
  for (int64_t i = 0; i < n; ++i)
    if (arrival[order[i]] > now) {
      int64_t k = order[i];
      set_err("select_batch: request '%.*s' has not arrived yet",
              (int)(id_offs[k + 1] - id_offs[k]), ids + id_offs[k]);
      return -1;
    }
  return 0;
}

/* ---- metrics.cpp:13-32, :66-86 ------------------------------------------ */
int po_kendall(const double* x, const double* y, int64_t n, uint64_t* counts,
               double* tau, int nthreads) {
  if (n < 2) { set_err("kendall_tau_b: need at least 2 items, got %lld", (long long)n); return -1; }
  uint64_t nc = 0, nd = 0, n1 = 0, n2 = 0;
#pragma omp parallel for schedule(dynamic, 64) reduction(+ : nc, nd, n1, n2) num_threads(nthreads > 0 ? nthreads : 1)
  for (int64_t i = 0; i < n - 1; ++i)
    for (int64_t j = i + 1; j < n; ++j) {
      double dx = x[i] - x[j], dy = y[i] - y[j];
      if (dx == 0.0) ++n1;
      if (dy == 0.0) ++n2;
      if (dx != 0.0 && dy != 0.0) {
        if ((dx > 0.0) == (dy > 0.0)) ++nc; else ++nd;
      }
    }
  uint64_t n0 = (uint64_t)n * (uint64_t)(n - 1) / 2;
  counts[0] = nc; counts[1] = nd; counts[2] = n0; counts[3] = n1; counts[4] = n2;
  if (n1 == n0) { set_err("degenerate ranking: all values tied in first argument"); return -1; }
  if (n2 == n0) { set_err("degenerate ranking: all values tied in second argument"); return -1; }
  double denom = sqrt((double)(n0 - n1) * (double)(n0 - n2));
  double t = ((double)nc - (double)nd) / denom;
  *tau = t < -1.0 ? -1.0 : (t > 1.0 ? 1.0 : t);
  return 0;
}
