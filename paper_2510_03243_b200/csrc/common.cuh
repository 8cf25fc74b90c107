// Shared device/host helpers for libpars_cuda.so (sm_100a).
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include <string>

#include "pars_cuda.h"

namespace pars_b200 {

// ---- error plumbing (thread-local message, pars_last_error) ---------------
void set_error(const char* fmt, ...) __attribute__((format(printf, 1, 2)));
const char* get_error();

struct Status {
  int code = PARS_OK;
};

#define PARS_CUDA_CHECK(expr)                                                \
  do {                                                                       \
    cudaError_t _e = (expr);                                                 \
    if (_e != cudaSuccess) {                                                 \
      ::pars_b200::set_error("CUDA error %s at %s:%d: %s", cudaGetErrorName(_e), \
                             __FILE__, __LINE__, cudaGetErrorString(_e));    \
      return PARS_ERR_CUDA;                                                  \
    }                                                                        \
  } while (0)

#define PARS_TRY(expr)          \
  do {                          \
    int _rc = (expr);           \
    if (_rc != PARS_OK) return _rc; \
  } while (0)

// ---- FNV-1a / salts (reference features.cpp:17-27, rng.hpp:10-15) ---------
constexpr uint64_t kFnvPrime = 0x100000001b3ull;
constexpr uint64_t kFnvOffset = 0xcbf29ce484222325ull;

__host__ __device__ inline uint64_t splitmix64(uint64_t x) {
  x += 0x9e3779b97f4a7c15ull;
  x = (x ^ (x >> 30)) * 0xbf58476d1ce4e5b9ull;
  x = (x ^ (x >> 27)) * 0x94d049bb133111ebull;
  return x ^ (x >> 31);
}
__host__ __device__ inline uint64_t ngram_salt(uint64_t field, uint64_t order) {
  return splitmix64(kFnvOffset ^ (field << 32) ^ order);
}

__host__ __device__ inline bool is_space(unsigned c) {
  // C-locale std::isspace: ' ' \t \n \v \f \r
  return c == 32u || (c - 9u) < 5u;
}

__host__ __device__ inline int64_t imin64(int64_t a, int64_t b) { return a < b ? a : b; }

// ---- integer divide helpers -------------------------------------------------
__host__ __device__ inline int64_t ceil_div(int64_t a, int64_t b) { return (a + b - 1) / b; }

// ---- exact integer -> double without I2F.F64 ---------------------------------
// The conversion pipe is slow on this part; the bits of 2^52 + u (u < 2^32
// in the low word) are exactly that double, so one DADD removes the bias.
// A 16-bit count stored biased by 2^15 (compact rows: count + 0x8000):
__device__ __forceinline__ double biased16_to_f64(uint32_t e) {
  return __dsub_rn(__hiloint2double(0x43300000, (int)(e & 0xffffu)), 4503599627403264.0);  // 2^52 + 2^15
}
// any int32:
__device__ __forceinline__ double i32_to_f64(int32_t c) {
  return __dsub_rn(__hiloint2double(0x43300000, (int)((uint32_t)c ^ 0x80000000u)), 4503601774854144.0);  // 2^52 + 2^31
}

// ---- launch telemetry -----------------------------------------------------
void count_launch(pars_ctx* ctx, uint64_t k = 1);

}  // namespace pars_b200
