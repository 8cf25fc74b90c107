// Microbenchmark: issue throughput (cycles per warp-instruction) of DMUL /
// DADD / I2F.F64 / LDS.64 for ONE warp on an SM sub-partition, with 8
// independent chains so latency is hidden; and for 4 warps per SM (one per
// scheduler). Tells whether a single warp's fp64 chain is pipe-bound.
#include <cstdio>
#include <cuda_runtime.h>

template <int KIND>
__global__ void thr(double* out, long long* cyc, double a, double b, int iters,
                    const double* __restrict__ gw) {
  __shared__ double sh[1024];
  for (int k = threadIdx.x; k < 1024; k += blockDim.x) sh[k] = a + k;
  __syncthreads();
  double x[8];
#pragma unroll
  for (int j = 0; j < 8; ++j) x[j] = a + j;
  int idx = threadIdx.x * 33 & 1023;
  long long t0 = clock64();
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      if (KIND == 0) x[j] = __dmul_rn(x[j], b);
      if (KIND == 1) x[j] = __dadd_rn(x[j], b);
      if (KIND == 2) x[j] = __dadd_rn(x[j], (double)(int)(i + j));
      if (KIND == 3) {
        x[j] = __dadd_rn(x[j], sh[idx]);
        idx = (idx + 97) & 1023;
      }
      if (KIND == 4) x[j] = __dadd_rn(x[j], sh[(idx + 131 * j + 7 * i) & 1023]);  // independent
      if (KIND == 5) x[j] = __dadd_rn(x[j], sh[(threadIdx.x + 32 * j) & 1023]);   // conflict-free
      if (KIND == 6) x[j] = __dadd_rn(x[j], __ldg(gw + ((idx + 131 * j + 7 * i) & 4095)));  // L1 gather
    }
  }
  long long t1 = clock64();
  double s = 0;
#pragma unroll
  for (int j = 0; j < 8; ++j) s += x[j];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}

int main() {
  double* o;
  long long* c;
  cudaMalloc(&o, 1 << 20);
  cudaMallocManaged(&c, 1024 * 8);
  const int iters = 4096;
  const char* names[7] = {"DMUL", "DADD", "DADD+I2F", "DADD+LDS.64 gather (serial idx)",
                          "DADD+LDS.64 gather", "DADD+LDS.64 linear", "DADD+LDG.64 gather (L1)"};
  double* gw;
  cudaMalloc(&gw, 4096 * 8);
  cudaMemset(gw, 0, 4096 * 8);
  for (int warps : {1, 4, 8}) {
    for (int k = 0; k < 7; ++k) {
      auto f = k == 0 ? thr<0> : k == 1 ? thr<1> : k == 2 ? thr<2> : k == 3 ? thr<3>
             : k == 4 ? thr<4> : k == 5 ? thr<5> : thr<6>;
      f<<<1, 32 * warps>>>(o, c, 1.000001, 0.999999, iters, gw);
      cudaDeviceSynchronize();
      f<<<1, 32 * warps>>>(o, c, 1.000001, 0.999999, iters, gw);
      cudaDeviceSynchronize();
      const double per = (double)c[0] / (iters * 8.0);
      printf("%d warp(s)/SM  %-20s %.2f cycles per warp-instruction (per warp)\n", warps, names[k],
             per);
    }
  }
  return 0;
}
