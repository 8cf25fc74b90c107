// Fused featurize(+score) kernels — declarations shared by capi.cu.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include "common.cuh"

namespace pars_b200 {

// Host-prepared extractor description (features.hpp:17-25 + precomputed salts).
struct FeatConfig {
  uint32_t dim;
  uint32_t mask;  // dim-1 when dim is a power of two
  int32_t pow2;   // 1 -> 32-bit hashing (only the low log2(dim)+1 bits matter)
  int32_t norm;   // 0 none, 1 l2
  int32_t n_word, n_char;
  int32_t word[8], chr[8];
  int32_t max_word;
  int32_t default_orders;  // word {1} + char {3}: single-pass specialisation
  uint64_t word_salt[8], char_salt[8];
};

enum FeatMode : int {
  kFeatScoreExact = 0,  // fp64, sequential ascending-index dot (bit-exact)
  kFeatScoreFast = 1,   // fp32 products + warp tree reduction
  kFeatCsr = 2,         // write (idx, value) rows into per-prompt slots
};

struct FeatArgs {
  const uint8_t* text;
  const int64_t* offsets;  // [n+1], absolute into text
  int64_t n;
  const double* w64;  // exact mode weights
  const float* w32;   // fast mode weights
  double bias;
  double* scores;  // score modes
  // CSR mode: per-prompt slot base (entries) + outputs
  const int64_t* slot_base;
  uint32_t* out_idx;
  double* out_val;
  int32_t* out_nnz;
  int32_t* out_cnt;  // optional: the integer bucket count behind each value
  double* out_inv;   // optional: per prompt, the L2 factor (1.0 without norm)
  // long-prompt hand-off (packed kernel -> wide kernel)
  int32_t* long_list;
  int32_t* long_count;
  // per-warp tables in global memory for dimensions too large for smem
  unsigned char* gscratch;
  size_t gscratch_bytes;
  // exact mode: per-warp (idx, count) list arenas, list_cap u32 words each
  uint32_t* lists;
  size_t lists_bytes;
  uint32_t list_cap;
  // exact mode, lane kernel: per-prompt entry slots for chain_slots_kernel
  // (carved out of the lists scratch by the launcher)
  uint32_t* slots;
  int32_t* slot_nnz;
  double* slot_inv;
  // lane kernel + chain kernel: this launch covers prompts [first, n) (slot
  // k holds prompt first + k); every other kernel requires first == 0
  int64_t first;
};

bool build_feat_config(const pars_extractor* ex, FeatConfig* cfg);

// Scratch a launch over n prompts needs: global per-warp tables (dims too
// large for shared memory) and exact-mode list arenas (bytes each).
int feat_scratch_bytes(const FeatConfig& cfg, int mode, int64_t n, size_t* gscratch,
                       size_t* lists);
uint32_t feat_list_cap_words(const FeatConfig& cfg);

// Launches the packed kernel over all prompts followed by the wide kernel
// over prompts whose feature count may exceed the 16-bit counters.
int launch_featurize(pars_ctx* ctx, const FeatConfig& cfg, int mode,
                     const FeatArgs& args, cudaStream_t stream);

// Upper bound on hashed features of one prompt (CSR slot size).
__host__ __device__ inline int64_t feat_cap(const FeatConfig& c, int64_t len) {
  int64_t cap = (int64_t)c.n_word * ((len + 1) / 2) + (int64_t)c.n_char * len;
  return cap < (int64_t)c.dim ? cap : (int64_t)c.dim;
}

// Dense embedding scoring (features.cpp:67-76 + score).
int launch_score_dense(pars_ctx* ctx, const FeatConfig& cfg, int mode,
                       const double* X, int64_t n, const double* w64,
                       const float* w32, double bias, double* scores,
                       cudaStream_t stream);

}  // namespace pars_b200
