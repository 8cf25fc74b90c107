/* Synthetic workload tool (NOT part of the product library libpars_cuda.so).
 *
 * synthesize_dataset(n, lognormal(mu, sigma), seed) restated from the
 * reference's generator (proj/src/dataset.cpp:204-297; bit-identical text and
 * lengths, pinned by tests/test_abi.py against the reference library), plus
 * the C4 padding of SURVEY §8(d): pad_tokens > 0 pads every prompt with
 * " w<k>" tokens, k = Rng(pad_seed).below(50), to exactly pad_tokens
 * whitespace tokens. The text arena is page-locked when possible (it is the
 * host buffer of the end-to-end benchmark). Used by bench.py (our arm),
 * tools/ and tests/ to produce inputs quickly; the reference arm of bench.py
 * uses the reference's own synthesize_dataset instead. */
#ifndef PARS_WORKLOAD_H
#define PARS_WORKLOAD_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct pars_workload pars_workload;

int pars_workload_synthesize(uint64_t n, double mu, double sigma, uint64_t seed,
                             int64_t pad_tokens, uint64_t pad_seed, pars_workload** out);
/* pad_kind 0: the C4 filler above; 1: the C4 hard variant of SURVEY §8(d),
 * random 6-letter lowercase words (letters from Rng(pad_seed).below(26)). */
int pars_workload_synthesize_pad(uint64_t n, double mu, double sigma, uint64_t seed,
                                 int64_t pad_tokens, uint64_t pad_seed, int pad_kind,
                                 pars_workload** out);
int64_t pars_workload_count(const pars_workload* w);
int64_t pars_workload_text_bytes(const pars_workload* w);
/* Pointers stay valid until pars_workload_free. */
const char* pars_workload_text(const pars_workload* w);
const int64_t* pars_workload_offsets(const pars_workload* w);
const int64_t* pars_workload_output_len(const pars_workload* w);
const int64_t* pars_workload_prompt_len(const pars_workload* w);
void pars_workload_free(pars_workload* w);
/* Token statistics of prompts [0, n) of a text arena (offsets[n+1],
 * absolute), tokens split as features.cpp:36-49 (C-locale isspace):
 * out[0] = tokens, out[1] = sum of token lengths, out[2] = sum of
 * max(0, len - 2) (char trigrams), out[3] = text bytes. Measurement only
 * (the integer-issue roofline of bench.py). */
int pars_workload_token_stats(const char* text, const int64_t* offsets, int64_t n, uint64_t* out);
const char* pars_workload_last_error(void);

#ifdef __cplusplus
}
#endif
#endif /* PARS_WORKLOAD_H */
