// Dataset ingestion on the GPU (ingest.cu) — declarations shared with capi.cu.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include "common.cuh"

namespace pars_b200 {

// per-record status codes of the device parser (first failure in the
// reference's check order; duplicates, the samples median and the token
// count are settled by later kernels)
enum IngestErr : uint32_t {
  kIngOk = 0,
  kIngMalformed = 1,
  kIngNotObject = 2,
  kIngBadId = 3,
  kIngBadPrompt = 4,
  kIngBadSamples = 5,
  kIngBadOutputLen = 6,
  kIngMissingOutputLen = 7,
  kIngEmbedding = 8,  // an "embedding" field: not parsed by the GPU loader
  kIngBadPromptLen = 9,
};
enum IngestFlag : uint32_t {
  kIngIdEsc = 1,
  kIngPromptEsc = 2,
  kIngHasSamples = 4,
  kIngHasOutputLen = 8,
};

// Structure of arrays, one entry per record (device pointers).
struct RecordOut {
  uint32_t* err;
  uint32_t* flags;
  int64_t *id_b, *id_e, *id_len;  // raw span (file offsets) and decoded length
  int64_t *pr_b, *pr_e, *pr_len;
  int64_t* pr_tok;  // whitespace tokens of the decoded prompt
  int64_t* out_len;     // -1 when absent
  int64_t* prompt_len;  // -1 when absent
  int64_t *sm_b, *sm_e;  // the samples array's span ('[' .. ']'), -1 when absent
  uint32_t* any_samples;  // set to 1 when any record has output_len_samples
};

int64_t ingest_block_count(int64_t n);
// '\n' count of n bytes (block counts scanned into d_blk[0..nb], total back
// on the host), then the newline positions in file order
// Scratch for the scans below: ingest_scan_scratch_bytes(n) for n elements.
size_t ingest_scan_scratch_bytes(int64_t n);
int ingest_count_newlines(const uint8_t* d_text, int64_t n, uint32_t* d_blk, int64_t* total,
                          void* scratch, cudaStream_t st);
// The same in pieces: counts of blocks [b0, b1) (as their bytes land), then
// the scan of all block counts with the total back on the host.
int64_t ingest_block_bytes();
void ingest_count_newlines_range(const uint8_t* d_text, int64_t n, int64_t b0, int64_t b1,
                                 uint32_t* d_blk, cudaStream_t st);
int ingest_scan_newline_blocks(uint32_t* d_blk, int64_t n, int64_t* total, void* scratch,
                               cudaStream_t st);
void ingest_write_newlines(const uint8_t* d_text, int64_t n, const uint32_t* d_blk, int64_t* d_nl,
                           cudaStream_t st);
void ingest_launch_line_flags(const int64_t* nl, int64_t nlines, int64_t n, uint32_t* nonempty,
                              cudaStream_t st);
void ingest_launch_scan(uint32_t* v, int64_t n, void* scratch, cudaStream_t st);  // exclusive, total at v[n]
void ingest_launch_record_lines(const int64_t* nl, int64_t nlines, int64_t n, const uint32_t* rank,
                                int64_t limit, int64_t* rb, int64_t* re, int64_t* rline,
                                cudaStream_t st);
void ingest_launch_parse(const uint8_t* text, const int64_t* rb, const int64_t* re, int64_t nrec,
                         const RecordOut& out, cudaStream_t st);
// output_len from / checked against the median of the samples; sets
// mismatch[r] = 1 when output_len != median_floor(samples), unsup[r] = 1
// when a record has more samples than the device path sorts
void ingest_launch_samples(const uint8_t* text, int64_t nrec, const RecordOut& rec,
                           uint32_t* mismatch, uint32_t* unsup, cudaStream_t st);
void ingest_launch_emit(const uint8_t* text, int64_t nrec, const RecordOut& rec, const int64_t* pr_off,
                        uint8_t* arena, const int64_t* id_off, uint8_t* ids, int64_t* tokens,
                        cudaStream_t st);
void ingest_launch_dups(const uint8_t* ids, const int64_t* id_off, int64_t nrec, uint64_t* hash,
                        uint64_t cap, unsigned long long* tkey, unsigned long long* tmin,
                        uint32_t* dup, cudaStream_t st);

void ingest_launch_scan_i64(int64_t* v, int64_t n, void* scratch, cudaStream_t st);  // exclusive, total at v[n]
void ingest_launch_lengths(int64_t nrec, const RecordOut& rec, int64_t* pr_len, int64_t* id_len,
                           cudaStream_t st);
void ingest_launch_first_fail(int64_t nrec, const RecordOut& rec, const uint32_t* dup,
                              const uint32_t* mismatch, const uint32_t* unsup, const int64_t* tokens,
                              unsigned long long* first, cudaStream_t st);

}  // namespace pars_b200
