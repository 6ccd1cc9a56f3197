// Legacy-path tensor throughput on this GPU: mma.sync m16n8k32 s8*s8 -> s32 (the INT8 path
// an int8 byte-sliced NTT round could use without tcgen05), register operands only, 4
// independent accumulator chains per warp.  Data point for DESIGN section 16.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/mb_imma tools/microbench_imma.cu
#include <cstdio>
#include <cuda_runtime.h>

__global__ void k_imma(int iters, int* out) {
  unsigned a0 = threadIdx.x * 0x01010101u, a1 = a0 + 1, a2 = a0 + 2, a3 = a0 + 3;
  unsigned b0 = blockIdx.x * 0x01010101u, b1 = b0 + 5;
  int c[4][4] = {};
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int k = 0; k < 4; ++k)
      asm volatile(
          "mma.sync.aligned.m16n8k32.row.col.s32.s8.s8.s32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, "
          "{%0,%1,%2,%3};\n"
          : "+r"(c[k][0]), "+r"(c[k][1]), "+r"(c[k][2]), "+r"(c[k][3])
          : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1));
  }
  int s = 0;
#pragma unroll
  for (int k = 0; k < 4; ++k) s += c[k][0] + c[k][1] + c[k][2] + c[k][3];
  if (s == 0x12345678) out[0] = s;
}

__global__ void k_hmma(int iters, float* out) {
  unsigned a0 = threadIdx.x * 0x3c003c00u, a1 = a0, a2 = a0, a3 = a0;
  unsigned b0 = 0x3c003c00u, b1 = b0;
  float c[4][4] = {};
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int k = 0; k < 4; ++k)
      asm volatile(
          "mma.sync.aligned.m16n8k16.row.col.f32.f16.f16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, "
          "{%0,%1,%2,%3};\n"
          : "+f"(c[k][0]), "+f"(c[k][1]), "+f"(c[k][2]), "+f"(c[k][3])
          : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1));
  }
  float s = 0;
#pragma unroll
  for (int k = 0; k < 4; ++k) s += c[k][0] + c[k][1] + c[k][2] + c[k][3];
  if (s == 1.2345f) out[0] = s;
}

int main() {
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  int* dout;
  cudaMalloc(&dout, 16);
  const int iters = 20000, threads = 256, blocks = sms * 8;
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  for (int rep = 0; rep < 2; ++rep) {
    k_imma<<<blocks, threads>>>(100, dout);
    cudaEventRecord(e0);
    k_imma<<<blocks, threads>>>(iters, dout);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    const double ops = 2.0 * 16 * 8 * 32 * 4 * (double)iters * blocks * (threads / 32);
    printf("mma.sync m16n8k32 s8: %.1f TOPS (%.3f ms)\n", ops / (ms * 1e-3) / 1e12, ms);
    k_hmma<<<blocks, threads>>>(100, reinterpret_cast<float*>(dout));
    cudaEventRecord(e0);
    k_hmma<<<blocks, threads>>>(iters, reinterpret_cast<float*>(dout));
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    cudaEventElapsedTime(&ms, e0, e1);
    const double fops = 2.0 * 16 * 8 * 16 * 4 * (double)iters * blocks * (threads / 32);
    printf("mma.sync m16n8k16 f16: %.1f TFLOP/s (%.3f ms)\n", fops / (ms * 1e-3) / 1e12, ms);
  }
  printf("%s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
