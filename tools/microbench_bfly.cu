// Ceiling for the NTT kernels' arithmetic on sm_100a: radix-2 Shoup butterflies in the
// register-resident form the kernels use (16 values per thread, 4 stages of 8 independent
// butterflies, twiddles held in registers, canonical residues mod a 31-bit prime), plus
// single-instruction-class throughputs with 16 independent chains per thread.  No memory
// traffic inside the timed loop.  Prints butterflies (or ops) per SM per clock and G/s.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/microbench_bfly tools/microbench_bfly.cu
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>

constexpr uint32_t P0 = 2130706433u;
#define ITERS 512

__device__ __forceinline__ uint32_t add_mod(uint32_t a, uint32_t b, uint32_t p) {
  const uint32_t s = a + b;
  return min(s, s - p);
}
__device__ __forceinline__ uint32_t sub_mod(uint32_t a, uint32_t b, uint32_t p) {
  const uint32_t d = a + (p - b);
  return min(d, d - p);
}
__device__ __forceinline__ uint32_t mul_shoup(uint32_t a, uint32_t w, uint32_t ws, uint32_t p) {
  const uint32_t q = __umulhi(a, ws);
  const uint32_t r = a * w - q * p;
  return min(r, r - p);
}

// DIF radix-16 network in registers (the kernels' dif_group with S = 4)
__global__ void __launch_bounds__(256) k_dif16(uint32_t* out, uint32_t seed, uint32_t p) {
  uint32_t x[16], w[15], ws[15];
  for (int i = 0; i < 16; ++i) x[i] = (seed * 2654435761u + threadIdx.x * 97u + i * 1234567u) % p;
  for (int i = 0; i < 15; ++i) {
    w[i] = (seed + 77u * i + 5u) % p;
    ws[i] = (uint32_t)(((uint64_t)w[i] << 32) / p);
  }
  for (int it = 0; it < ITERS; ++it) {
#pragma unroll
    for (int st = 3; st >= 0; --st) {
      const int d = 1 << st;
#pragma unroll
      for (int k = 0; k < 16; ++k) {
        if (k & d) continue;
        const int ti = (d - 1) + (k & (d - 1));  // 15 distinct twiddles over the 4 stages
        const uint32_t a = x[k], b = x[k + d];
        x[k] = add_mod(a, b, p);
        x[k + d] = mul_shoup(a + (p - b), w[ti], ws[ti], p);
      }
    }
  }
  uint32_t s = 0;
  for (int i = 0; i < 16; ++i) s ^= x[i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

// DIT radix-16 network with the kernels' lazy intermediate outputs (dit_group, S = 4)
__global__ void __launch_bounds__(256) k_dit16(uint32_t* out, uint32_t seed, uint32_t p) {
  uint32_t x[16], w[15], ws[15];
  for (int i = 0; i < 16; ++i) x[i] = (seed * 2654435761u + threadIdx.x * 97u + i * 1234567u) % p;
  for (int i = 0; i < 15; ++i) {
    w[i] = (seed + 77u * i + 5u) % p;
    ws[i] = (uint32_t)(((uint64_t)w[i] << 32) / p);
  }
  for (int it = 0; it < ITERS; ++it) {
#pragma unroll
    for (int st = 0; st < 4; ++st) {
      const int d = 1 << st;
#pragma unroll
      for (int k = 0; k < 16; ++k) {
        if (k & d) continue;
        const int ti = (d - 1) + (k & (d - 1));
        const uint32_t a = x[k];
        const uint32_t b = mul_shoup(x[k + d], w[ti], ws[ti], p);
        if (st + 1 < 4 && (k & (2 * d))) {
          x[k] = a + b;
          x[k + d] = a + (p - b);
        } else {
          x[k] = add_mod(a, b, p);
          x[k + d] = sub_mod(a, b, p);
        }
      }
    }
    // keep every value canonical for the next iteration's "u" operands
#pragma unroll
    for (int k = 0; k < 16; ++k) x[k] = min(x[k], x[k] - p);
  }
  uint32_t s = 0;
  for (int i = 0; i < 16; ++i) s ^= x[i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

// instruction classes, 16 independent chains per thread
__global__ void __launch_bounds__(256) k_umin(uint32_t* out, uint32_t seed, uint32_t p) {
  uint32_t x[16];
  for (int i = 0; i < 16; ++i) x[i] = seed + threadIdx.x + i;
  for (int it = 0; it < ITERS; ++it)
#pragma unroll
    for (int i = 0; i < 16; ++i) x[i] = min(x[i] + 0x3u, x[i] - p);  // one VIADDMNMX
  uint32_t s = 0;
  for (int i = 0; i < 16; ++i) s ^= x[i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
__global__ void __launch_bounds__(256) k_imadhi(uint32_t* out, uint32_t seed, uint32_t p) {
  uint32_t x[16];
  for (int i = 0; i < 16; ++i) x[i] = seed + threadIdx.x + i;
  for (int it = 0; it < ITERS; ++it)
#pragma unroll
    for (int i = 0; i < 16; ++i) x[i] = __umulhi(x[i], p) + x[(i + 1) & 15];  // IMAD.HI (+acc)
  uint32_t s = 0;
  for (int i = 0; i < 16; ++i) s ^= x[i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
__global__ void __launch_bounds__(256) k_imad(uint32_t* out, uint32_t seed, uint32_t p) {
  uint32_t x[16];
  for (int i = 0; i < 16; ++i) x[i] = seed + threadIdx.x + i;
  for (int it = 0; it < ITERS; ++it)
#pragma unroll
    for (int i = 0; i < 16; ++i) x[i] = x[i] * x[(i + 3) & 15] + p;  // IMAD, not foldable
  uint32_t s = 0;
  for (int i = 0; i < 16; ++i) s ^= x[i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
__global__ void __launch_bounds__(256) k_iadd3(uint32_t* out, uint32_t seed, uint32_t p) {
  uint32_t x[16];
  for (int i = 0; i < 16; ++i) x[i] = seed + threadIdx.x + i;
  for (int it = 0; it < ITERS; ++it)
#pragma unroll
    for (int i = 0; i < 16; ++i) x[i] = x[i] + x[(i + 5) & 15] - p;  // IADD3
  uint32_t s = 0;
  for (int i = 0; i < 16; ++i) s ^= x[i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

// the same networks with p a compile-time immediate (IMAD / VIADDMNMX immediate forms)
__global__ void __launch_bounds__(256) k_dif16_imm(uint32_t* out, uint32_t seed, uint32_t) {
  constexpr uint32_t p = P0;
  uint32_t x[16], w[15], ws[15];
  for (int i = 0; i < 16; ++i) x[i] = (seed * 2654435761u + threadIdx.x * 97u + i * 1234567u) % p;
  for (int i = 0; i < 15; ++i) {
    w[i] = (seed + 77u * i + 5u) % p;
    ws[i] = (uint32_t)(((uint64_t)w[i] << 32) / p);
  }
  for (int it = 0; it < ITERS; ++it) {
#pragma unroll
    for (int st = 3; st >= 0; --st) {
      const int d = 1 << st;
#pragma unroll
      for (int k = 0; k < 16; ++k) {
        if (k & d) continue;
        const int ti = (d - 1) + (k & (d - 1));
        const uint32_t a = x[k], b = x[k + d];
        x[k] = add_mod(a, b, p);
        x[k + d] = mul_shoup(a + (p - b), w[ti], ws[ti], p);
      }
    }
  }
  uint32_t s = 0;
  for (int i = 0; i < 16; ++i) s ^= x[i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
__global__ void __launch_bounds__(256) k_umin_imm(uint32_t* out, uint32_t seed, uint32_t) {
  uint32_t x[16];
  for (int i = 0; i < 16; ++i) x[i] = seed + threadIdx.x + i;
  for (int it = 0; it < ITERS; ++it)
#pragma unroll
    for (int i = 0; i < 16; ++i) x[i] = min(x[i], x[i] - P0);
  uint32_t s = 0;
  for (int i = 0; i < 16; ++i) s ^= x[i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
__global__ void __launch_bounds__(256) k_imad_imm(uint32_t* out, uint32_t seed, uint32_t) {
  uint32_t x[16];
  for (int i = 0; i < 16; ++i) x[i] = seed + threadIdx.x + i;
  for (int it = 0; it < ITERS; ++it)
#pragma unroll
    for (int i = 0; i < 16; ++i) x[i] = x[(i + 3) & 15] - x[i] * P0;  // IMAD with immediate
  uint32_t s = 0;
  for (int i = 0; i < 16; ++i) s ^= x[i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
__global__ void __launch_bounds__(256) k_imadhi_imm(uint32_t* out, uint32_t seed, uint32_t) {
  uint32_t x[16];
  for (int i = 0; i < 16; ++i) x[i] = seed + threadIdx.x + i;
  for (int it = 0; it < ITERS; ++it)
#pragma unroll
    for (int i = 0; i < 16; ++i) x[i] = __umulhi(x[i], 0x9E3779B1u) + x[(i + 1) & 15];
  uint32_t s = 0;
  for (int i = 0; i < 16; ++i) s ^= x[i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

int main() {
  cudaDeviceProp prop;
  cudaGetDeviceProperties(&prop, 0);
  int clk_khz = 0;
  cudaDeviceGetAttribute(&clk_khz, cudaDevAttrClockRate, 0);
  const int sms = prop.multiProcessorCount;
  printf("device %s SMs %d max clock %.0f MHz\n", prop.name, sms, clk_khz / 1e3);
  const int threads = 256;
  uint32_t* out;
  cudaMalloc(&out, sizeof(uint32_t) * threads * sms * 64);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  struct K {
    const char* name;
    void (*k)(uint32_t*, uint32_t, uint32_t);
    double per_iter;  // counted units per thread per iteration
  } ks[] = {{"dif16 butterfly", k_dif16, 32}, {"dit16 butterfly", k_dit16, 32},
            {"viaddmnmx", k_umin, 16},        {"imad.hi", k_imadhi, 16},
            {"imad", k_imad, 16},             {"iadd3", k_iadd3, 16},
            {"dif16 imm-p", k_dif16_imm, 32}, {"viaddmnmx imm", k_umin_imm, 16},
            {"imad imm", k_imad_imm, 16},     {"imad.hi imm", k_imadhi_imm, 16}};
  for (auto& kk : ks) {
    for (int bps : {4, 8}) {  // CTAs per SM (256 threads each)
      const int blocks = sms * bps;
      kk.k<<<blocks, threads>>>(out, 1, P0);
      cudaEventRecord(e0);
      const int R = 5;
      for (int r = 0; r < R; ++r) kk.k<<<blocks, threads>>>(out, r + 2, P0);
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
      float ms;
      cudaEventElapsedTime(&ms, e0, e1);
      const double units = (double)blocks * threads * ITERS * kk.per_iter * R;
      const double gps = units / (ms * 1e-3) / 1e9;
      printf("%-16s %d CTA/SM: %9.1f G/s  %6.2f per SM per clock (at %.0f MHz)\n", kk.name, bps, gps,
             gps * 1e9 / sms / (clk_khz * 1e3), clk_khz / 1e3);
    }
  }
  printf("err %s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
