// Dependent-chain latency (SM cycles per op, one thread) of FP64 ops on this GPU.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o fp64_lat fp64_lat.cu && ./fp64_lat
#include <cstdio>
__global__ void k(double* out, long long* cyc, double x0, double y0) {
  double x = x0, y = y0;
  long long t0, t1;
  // DFMA chain
  t0 = clock64();
#pragma unroll 1
  for (int i = 0; i < 1024; ++i) x = __fma_rn(x, y, 0.5);
  t1 = clock64();
  cyc[0] = t1 - t0;
  out[0] = x;
  // DADD chain
  x = x0;
  t0 = clock64();
#pragma unroll 1
  for (int i = 0; i < 1024; ++i) x = __dadd_rn(x, y);
  t1 = clock64();
  cyc[1] = t1 - t0;
  out[1] = x;
  // IEEE division chain
  x = x0;
  t0 = clock64();
#pragma unroll 1
  for (int i = 0; i < 256; ++i) x = y / x;
  t1 = clock64();
  cyc[2] = t1 - t0;
  out[2] = x;
  // loop overhead reference: integer chain
  int z = (int)x0;
  t0 = clock64();
#pragma unroll 1
  for (int i = 0; i < 1024; ++i) z = z * 3 + 1;
  t1 = clock64();
  cyc[3] = t1 - t0;
  out[3] = z;
  // DFMA chain unrolled by 8 (loop overhead amortised)
  x = x0;
  t0 = clock64();
#pragma unroll 1
  for (int i = 0; i < 128; ++i) {
#pragma unroll
    for (int u = 0; u < 8; ++u) x = __fma_rn(x, y, 0.5);
  }
  t1 = clock64();
  cyc[4] = t1 - t0;
  out[4] = x;
}
int main() {
  double* o;
  long long* c;
  cudaMallocManaged(&o, 64);
  cudaMallocManaged(&c, 64);
  for (int r = 0; r < 2; ++r) {
    k<<<1, 1>>>(o, c, 1.0000001, 0.999999);
    cudaDeviceSynchronize();
  }
  printf("DFMA %.1f  DADD %.1f  DIV %.1f  IMAD-loop %.1f  DFMA(unroll8) %.1f cycles/op\n", c[0] / 1024.0, c[1] / 1024.0,
         c[2] / 256.0, c[3] / 1024.0, c[4] / 1024.0);
  return 0;
}
