// Microbenchmark: whole-GPU integer issue throughput on this B200, the peak
// that the featurize kernel's integer-issue roofline divides by (SURVEY §8(d):
// "the non-TC issue peak ... measure it with a microbenchmark").
//
// Every thread runs 8 independent FNV-style chains; one "step" of a chain is
//   LOP3 only:        x = x ^ (x >> 7) ^ k            (1 LOP3-class op, ALU pipe)
//   IMAD only:        x = x * P + k                    (1 IMAD, FMA pipe)
//   FNV step:         x = (x ^ b) * P                  (1 LOP3 + 1 IMAD)
//   FNV + select:     x = (c ? x : s) ^ b) * P         (SEL + LOP3 + IMAD)
// Grid = 148 SMs x 4 CTAs x 256 threads (full occupancy of issue slots), the
// kernel timed with CUDA events, best of 5. Output: one JSON line with the
// achieved lane-ops/s per kind (lane-ops = executed thread instructions of
// the measured kind, counted from the loop structure and cross-checked with
// SASS: tools/micro/int_issue.sass.txt).
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o int_issue int_issue.cu
#include <cstdio>
#include <cuda_runtime.h>

constexpr unsigned P = 0x1b3u;

template <int KIND>
__global__ void __launch_bounds__(256) issue(unsigned* out, int iters, unsigned k, unsigned s) {
  unsigned x[8];
#pragma unroll
  for (int j = 0; j < 8; ++j) x[j] = threadIdx.x * 0x9e3779b9u + j;
  unsigned b = threadIdx.x * 7u + blockIdx.x;  // per-thread (not uniform)
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      if (KIND == 0) x[j] = x[j] ^ (x[j] >> 7) ^ k;  // LOP3 with funnel-free shift folded? (SHF + LOP3)
      if (KIND == 1) x[j] = x[j] * P + k;
      if (KIND == 2) x[j] = (x[j] ^ b) * P;
      if (KIND == 3) x[j] = (((b >> j) & 1u ? x[j] : s) ^ b) * P;
      if (KIND == 4) x[j] = x[j] ^ (x[j] << 3) ^ b;  // SHF/IMAD.SHL + LOP3
    }
    b = b * 5u + 1u;
  }
  unsigned r = 0;
#pragma unroll
  for (int j = 0; j < 8; ++j) r ^= x[j];
  out[blockIdx.x * blockDim.x + threadIdx.x] = r;
}

template <int KIND>
float run(unsigned* out, int grid, int iters) {
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  issue<KIND><<<grid, 256>>>(out, 16, 3u, 5u);
  cudaDeviceSynchronize();
  float best = 1e30f;
  for (int r = 0; r < 5; ++r) {
    cudaEventRecord(a);
    issue<KIND><<<grid, 256>>>(out, iters, 3u, 5u);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    if (ms < best) best = ms;
  }
  return best;
}

int main() {
  int dev = 0, sms = 0, clk = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, dev);  // kHz
  const int grid = sms * 4, iters = 4096;
  unsigned* out;
  cudaMalloc(&out, (size_t)grid * 256 * 4);
  const double threads = (double)grid * 256, steps = threads * iters * 8;
  const char* names[5] = {"shift_xor (SHF+LOP3)", "imad", "fnv_step (LOP3+IMAD)",
                          "fnv_select (SEL+LOP3+IMAD)", "shl_xor (IMAD.SHL+LOP3)"};
  const double ops_per_step[5] = {2, 1, 2, 3, 2};
  float ms[5];
  ms[0] = run<0>(out, grid, iters);
  ms[1] = run<1>(out, grid, iters);
  ms[2] = run<2>(out, grid, iters);
  ms[3] = run<3>(out, grid, iters);
  ms[4] = run<4>(out, grid, iters);
  printf("{\"sms\": %d, \"clock_mhz_attr\": %.0f, \"kinds\": {", sms, clk / 1e3);
  for (int k = 0; k < 5; ++k) {
    const double lane_ops = steps * ops_per_step[k] / (ms[k] / 1e3);
    printf("\"%s\": {\"ms\": %.4f, \"lane_ops_per_s\": %.4e, \"warp_inst_per_clk_per_sm\": %.3f}%s",
           names[k], ms[k], lane_ops, lane_ops / 32.0 / sms / (clk * 1e3), k < 4 ? ", " : "");
  }
  printf("}}\n");
  return 0;
}
