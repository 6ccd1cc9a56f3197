// Step-0 box facts: integer pipe throughput on sm_100a (IMAD, IMAD.HI, IADD3, umin
// (VIADDMNMX), and a full Shoup modular butterfly). Each thread runs 8 independent
// chains so the pipes, not latency, bound the loop. Reports ops/clk/SM and Gops/s.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

#define ITERS 4096
constexpr uint32_t P0 = 2130706433u;

__global__ void k_imad(uint32_t* out, uint32_t a0) {
  uint32_t x[8]; for (int i = 0; i < 8; i++) x[i] = a0 + threadIdx.x + i;
  for (int it = 0; it < ITERS; it++)
#pragma unroll
    for (int i = 0; i < 8; i++) x[i] = x[i] * 0x9E3779B1u + 0x7F4A7C15u;
  uint32_t s = 0; for (int i = 0; i < 8; i++) s ^= x[i]; out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
__global__ void k_imadhi(uint32_t* out, uint32_t a0) {
  uint32_t x[8]; for (int i = 0; i < 8; i++) x[i] = a0 + threadIdx.x + i;
  for (int it = 0; it < ITERS; it++)
#pragma unroll
    for (int i = 0; i < 8; i++) x[i] = __umulhi(x[i], 0x9E3779B1u) ^ x[i];
  uint32_t s = 0; for (int i = 0; i < 8; i++) s ^= x[i]; out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
__global__ void k_iadd(uint32_t* out, uint32_t a0) {
  uint32_t x[8]; for (int i = 0; i < 8; i++) x[i] = a0 + threadIdx.x + i;
  for (int it = 0; it < ITERS; it++)
#pragma unroll
    for (int i = 0; i < 8; i++) x[i] = x[i] + 0x7F4A7C15u + (x[i] >> 3);
  uint32_t s = 0; for (int i = 0; i < 8; i++) s ^= x[i]; out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
__global__ void k_umin(uint32_t* out, uint32_t a0) {
  uint32_t x[8]; for (int i = 0; i < 8; i++) x[i] = a0 + threadIdx.x + i;
  for (int it = 0; it < ITERS; it++)
#pragma unroll
    for (int i = 0; i < 8; i++) { uint32_t s = x[i] + 0x3u; x[i] = min(s, s - P0); }
  uint32_t s = 0; for (int i = 0; i < 8; i++) s ^= x[i]; out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
// DIF butterfly with Shoup twiddle, canonical [0,p)
__global__ void k_bfly(uint32_t* out, uint32_t a0) {
  uint32_t x[8]; for (int i = 0; i < 8; i++) x[i] = (a0 + threadIdx.x * 77 + i * 1234567u) % P0;
  const uint32_t w = 1234567891u % P0; const uint32_t ws = (uint32_t)(((uint64_t)w << 32) / P0);
  for (int it = 0; it < ITERS; it++) {
#pragma unroll
    for (int i = 0; i < 8; i += 2) {
      uint32_t u = x[i], v = x[i + 1];
      uint32_t s = u + v; s = min(s, s - P0);
      uint32_t d = u - v + P0;
      uint32_t q = __umulhi(d, ws);
      uint32_t r = d * w - q * P0; r = min(r, r - P0);
      x[i] = s; x[i + 1] = r;
    }
  }
  uint32_t s = 0; for (int i = 0; i < 8; i++) s ^= x[i]; out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

int main() {
  int dev = 0; cudaDeviceProp prop; cudaGetDeviceProperties(&prop, dev);
  int clk_khz = 0; cudaDeviceGetAttribute(&clk_khz, cudaDevAttrClockRate, dev);
  printf("device %s SMs %d L2 %d B smemPerBlockOptin %zu clock_attr_khz %d\n", prop.name,
         prop.multiProcessorCount, prop.l2CacheSize, prop.sharedMemPerBlockOptin, clk_khz);
  const int threads = 256, blocks = prop.multiProcessorCount * 8;
  uint32_t* out; cudaMalloc(&out, sizeof(uint32_t) * threads * blocks);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  struct { const char* name; void (*k)(uint32_t*, uint32_t); double ops_per_inner; } ks[] = {
      {"imad (x*c+d)", k_imad, 8.0}, {"imad.hi+lop", k_imadhi, 8.0}, {"iadd3+shf", k_iadd, 8.0},
      {"iadd+umin", k_umin, 8.0}, {"dif_bfly_shoup", k_bfly, 4.0}};
  for (auto& kk : ks) {
    for (int rep = 0; rep < 2; rep++) kk.k<<<blocks, threads>>>(out, rep);
    cudaEventRecord(e0);
    const int R = 5;
    for (int rep = 0; rep < R; rep++) kk.k<<<blocks, threads>>>(out, rep);
    cudaEventRecord(e1); cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    double ops = (double)blocks * threads * ITERS * kk.ops_per_inner * R;
    double gops = ops / (ms * 1e-3) / 1e9;
    printf("%-18s %10.1f G(op)/s  per-SM-per-ns %.2f  (%.3f ms/launch)\n", kk.name, gops,
           gops / prop.multiProcessorCount, ms / R);
  }
  printf("err %s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
