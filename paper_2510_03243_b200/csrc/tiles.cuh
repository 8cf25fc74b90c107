// Upper-triangle tile enumeration + fixed-order block reduction shared by
// the all-pairs kernels.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

namespace pars_b200 {

constexpr int kPairTile = 256;

// Row-major enumeration of the upper triangle (J >= I) of an nt x nt tile
// grid: row I starts at index I*nt - I*(I-1)/2.
__device__ __forceinline__ void tile_of(int64_t t, int64_t nt, int64_t* I, int64_t* J) {
  const double b = 2.0 * (double)nt + 1.0;
  int64_t i = (int64_t)floor((b - sqrt(b * b - 8.0 * (double)t)) / 2.0);
  if (i < 0) i = 0;
  if (i > nt - 1) i = nt - 1;
  auto start = [&](int64_t r) { return r * nt - r * (r - 1) / 2; };
  while (i > 0 && start(i) > t) --i;
  while (i + 1 < nt && start(i + 1) <= t) ++i;
  *I = i;
  *J = i + (t - start(i));
}

// Moves (I, J) forward by `step` tiles in the same enumeration (the target
// must exist): a grid-stride walk pays tile_of's sqrt once per block.
__device__ __forceinline__ void tile_advance(int64_t step, int64_t nt, int64_t& I, int64_t& J) {
  J += step;
  while (J >= nt) {  // spill into the next row, which starts at column I + 1
    J -= nt - (I + 1);
    ++I;
  }
}

// Deterministic (fixed-order) block reduction; result valid in thread 0.
template <typename T, bool TRAIL = true>
__device__ __forceinline__ T block_sum_fixed(T v, T* red) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll
  for (int o = 16; o; o >>= 1) v += __shfl_down_sync(0xffffffffu, v, o);
  if (lane == 0) red[warp] = v;
  __syncthreads();
  T r = 0;
  if (threadIdx.x == 0)
    for (int w = 0; w < (int)(blockDim.x >> 5); ++w) r += red[w];
  if (TRAIL) __syncthreads();  // callers with another barrier before red's next use may skip it
  return r;
}

}  // namespace pars_b200
