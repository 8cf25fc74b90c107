// Microbenchmark: dependent-chain latency (cycles) of DADD / DMUL / DFMA /
// IMAD / LOP3 on this GPU, one thread, clock64 around 4096 dependent ops.
#include <cstdio>
#include <cuda_runtime.h>

__global__ void lat(double* out, long long* cyc, double a, double b, unsigned u) {
  double x = a;
  long long t0 = clock64();
#pragma unroll 64
  for (int i = 0; i < 4096; ++i) x = __dadd_rn(x, b);
  long long t1 = clock64();
  double y = a;
#pragma unroll 64
  for (int i = 0; i < 4096; ++i) y = __dmul_rn(y, b);
  long long t2 = clock64();
  double z = a;
#pragma unroll 64
  for (int i = 0; i < 4096; ++i) z = __fma_rn(z, b, a);
  long long t3 = clock64();
  unsigned h = u;
#pragma unroll 64
  for (int i = 0; i < 4096; ++i) h = (h ^ (unsigned)i) * 0x1b3u;
  long long t4 = clock64();
  out[0] = x + y + z + h;
  cyc[0] = t1 - t0; cyc[1] = t2 - t1; cyc[2] = t3 - t2; cyc[3] = t4 - t3;
}

int main() {
  double* o; long long* c;
  cudaMalloc(&o, 8); cudaMallocManaged(&c, 64);
  for (int r = 0; r < 3; ++r) lat<<<1, 1>>>(o, c, 1.0, 1.0000001, 7u);
  cudaDeviceSynchronize();
  printf("cycles per dependent op: dadd %.2f dmul %.2f dfma %.2f (lop3+imad) %.2f\n",
         c[0] / 4096.0, c[1] / 4096.0, c[2] / 4096.0, c[3] / 4096.0);
  return 0;
}
