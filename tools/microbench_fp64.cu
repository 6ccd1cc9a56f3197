// FP64 dependent-chain latency and split_c-style scalbn cost on this GPU (clock64):
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/mbf tools/microbench_fp64.cu && /tmp/mbf
#include <cstdio>
__global__ void k(double* out, long long* cyc, double a, double b, int e) {
  double x = a, y = b;
  long long t0 = clock64();
#pragma unroll 1
  for (int i = 0; i < 1000; ++i) { x = __dadd_rn(x, y); }
  long long t1 = clock64();
#pragma unroll 1
  for (int i = 0; i < 1000; ++i) { x = __fma_rn(x, y, a); }
  long long t2 = clock64();
  double s = 0;
#pragma unroll 1
  for (int i = 0; i < 100; ++i) { s += scalbn(x, e + (i & 7)); }
  long long t3 = clock64();
  unsigned long long u = 0;
#pragma unroll 1
  for (int i = 0; i < 1000; ++i) { u = __shfl_xor_sync(0xffffffffu, u + 1, 1); }
  long long t4 = clock64();
  out[threadIdx.x] = x + s + (double)u;
  if (threadIdx.x == 0) { cyc[0] = t1 - t0; cyc[1] = t2 - t1; cyc[2] = t3 - t2; cyc[3] = t4 - t3; }
}
int main() {
  double* o; long long* c; cudaMalloc(&o, 1024 * 8); cudaMallocManaged(&c, 64);
  for (int r = 0; r < 2; ++r) { k<<<1, 32>>>(o, c, 1.0000001, 1e-9, 30); cudaDeviceSynchronize(); }
  printf("DADD chain %.1f cyc/op, DFMA chain %.1f cyc/op, scalbn %.1f cyc/call, SHFL chain %.1f cyc/op\n",
         c[0] / 1000.0, c[1] / 1000.0, c[2] / 100.0, c[3] / 1000.0);
  return 0;
}
