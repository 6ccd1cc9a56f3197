// kernels.cu -- sm_100a kernels of the ozfft hot path (arXiv 2603.29129).
//
// Default path, per execute of a batch:
//   k_split_max<TS>       a1+a2  chirp premultiply (DD, or TS for f4) + per-level max |hi|
//                                 of the Ozaki split (Alg.6 l.778/786), one launch per level
//   k_split_digits<TS>    a2     int32 digits D = fl(fl(hi+sigma)-sigma) 2^(alpha-E)
//                                 (Alg.6 l.781-785) + the Alg.8 flush schedules
//   k_split_cluster<TS>   a1+a2  n <= 2^15: both of the above in one launch, one thread-block
//                                 cluster per transform (x' in shared memory, DSMEM max)
//   k_col_fwd<R,C,IMG>    a3     residue lift (or digit images, f2) + the first log2 R DIF
//                                 stages of the length-m forward NTT on column tiles
//   k_row_fused<C,2PASS>  a3-a5  last log2 C DIF stages of the slices of one row, pointwise
//                                 products + NTT-domain accumulation per Alg.8 group, first
//                                 log2 C DIT stages of each group's inverse NTT (one-pass
//                                 plans: whole NTTs, groups spread over gridDim.z CTAs)
//   k_col_inv_crt<R,C,PRUNE,TS>  a5-a7  last log2 R DIT stages, Garner CRT, exact 2^-c
//                                 scaling and the DD (TS) sum in flush order per real conv
//   k_finish_dd           a7     rr - ii, ir + ri, post-chirp, fp64 (inverse: conj, 1/n)
// Variants: k_col_inv_crt_img / k_crt_finish_img (complex images, f2), k_crt_finish(_ts)
// (one-pass plans, m <= 4096; one thread per (output, real conv)), k_col_inv + k_crt_finish
// (unit-sharded single transform,
// SURVEY 8(e)), k_w_finalize (plan time), k_tap_permute (test taps).
//
// NTT arithmetic: canonical residues in [0,p), Shoup multiplication by precomputed
// twiddles, branch-free conditional subtraction via unsigned min
// (one VIADDMNMX on sm_100a).  The forward NTT is decimation-in-frequency from
// natural order to bit-reversed order; the inverse is decimation-in-time from
// bit-reversed to natural order, so the pointwise stage needs no permutation.
// m^{-1} of eq:intt is folded into the cached W spectra.  Compile-time tuning knobs
// (OZ_*) default to the measured best (DESIGN.md section 6 lists the rejected ones).
#include <cooperative_groups.h>
#include <cuda_runtime.h>

#include <atomic>
#include <cstdlib>
#include <cstdio>
#include <type_traits>

#include "internal.h"

namespace ozfft {
namespace cg = cooperative_groups;

// ============================================================== modular arithmetic
// (ptxas issues part of the plain adds as IMAD.IADD on the FMA pipe, balancing it against
// the ALU pipe; forcing every add onto the ALU (__viaddmin_u32 forms) measured slower:
// c3 row kernel 1110 vs 1078 us -- the ALU pipe is the busier one)

__device__ __forceinline__ uint32_t add_mod(uint32_t a, uint32_t b, uint32_t p) {
  const uint32_t s = a + b;  // a, b < p < 2^31
  return min(s, s - p);
}
__device__ __forceinline__ uint32_t sub_mod(uint32_t a, uint32_t b, uint32_t p) {
  const uint32_t d = a + (p - b);
  return min(d, d - p);
}
// a * w mod p for any a < 2^32, w = (w, floor(w 2^32 / p)) (Shoup)
__device__ __forceinline__ uint32_t mul_shoup(uint32_t a, uint2 w, uint32_t p) {
  const uint32_t q = __umulhi(a, w.y);
  const uint32_t r = a * w.x - q * p;  // in [0, 2p)
  return min(r, r - p);
}

// T * 2^-32 mod p (canonical) for T < 3 p^2 (a sum of at most three products of residues),
// p < 2^31: fold the high word below p (T < 2p 2^32), then the subtractive Montgomery REDC
// with pinv_pos = +p^{-1} mod 2^32: mq p = tl (mod 2^32), so (T - mq p) / 2^32 = th - hi(mq p)
// exactly, in (-p, p); one conditional add of p makes it canonical.
__device__ __forceinline__ uint32_t redc_lazy2(unsigned long long T, uint32_t p, uint32_t pinv_pos) {
  // T < p 2^32 (at most two products): th < p already
  const uint32_t d = (uint32_t)(T >> 32) - __umulhi((uint32_t)T * pinv_pos, p);
  return min(d, d + p);
}
__device__ __forceinline__ uint32_t redc_lazy3(unsigned long long T, uint32_t p, uint32_t pinv_pos) {
  uint32_t th = (uint32_t)(T >> 32);
  const uint32_t tl = (uint32_t)T;
  th = min(th, th - p);
  const uint32_t mq = tl * pinv_pos;
  const uint32_t d = th - __umulhi(mq, p);
  return min(d, d + p);
}

// ============================================================== async copies (TMA bulk, mbarrier)
// One-shot global -> shared bulk copies (cp.async.bulk, the TMA engine's 1-D form; SASS
// UBLKCP) completing on an mbarrier (transaction bytes), and the waits on it.
__device__ __forceinline__ uint32_t smem_addr(const void* p) {
  return (uint32_t)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void mbar_init(unsigned long long* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_addr(bar)), "r"(count) : "memory");
}
// make the initialised barriers visible to the async proxy (the bulk-copy engine)
__device__ __forceinline__ void mbar_fence_init() {
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
// order this thread's earlier generic-proxy shared-memory accesses before later async-proxy
// writes to the same bytes (a buffer re-filled by a bulk copy after threads used it)
__device__ __forceinline__ void fence_proxy_async_smem() {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}
__device__ __forceinline__ void mbar_expect_tx(unsigned long long* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_addr(bar)), "r"(bytes)
               : "memory");
}
// bytes: multiple of 16; src, dst 16-byte aligned
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes,
                                         unsigned long long* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
          smem_addr(dst)),
      "l"(src), "r"(bytes), "r"(smem_addr(bar))
      : "memory");
}
__device__ __forceinline__ void mbar_wait(unsigned long long* bar, uint32_t parity) {
  asm volatile(
      "{\n .reg .pred p;\n"
      "WAIT_%=:\n mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      " @!p bra WAIT_%=;\n}" ::"r"(smem_addr(bar)),
      "r"(parity)
      : "memory");
}

// ============================================================== double-double (DD)
// Fixed IEEE RN operation sequences (no contraction): must match the oracle bit for bit.
__device__ __forceinline__ void two_prod(double a, double b, double& p, double& e) {
  p = __dmul_rn(a, b);
  e = __fma_rn(a, b, -p);
}
__device__ __forceinline__ void two_sum(double a, double b, double& s, double& e) {
  s = __dadd_rn(a, b);
  const double bb = __dsub_rn(s, a);
  e = __dadd_rn(__dsub_rn(a, __dsub_rn(s, bb)), __dsub_rn(b, bb));
}
// FastTwoSum, Alg.7
__device__ __forceinline__ void fast_two_sum(double a, double b, double& s, double& e) {
  s = __dadd_rn(a, b);
  e = __dsub_rn(b, __dsub_rn(s, a));
}
__device__ __forceinline__ void dd_add(double ah, double al, double bh, double bl, double& rh,
                                       double& rl) {
  double s, e, t, f;
  two_sum(ah, bh, s, e);
  two_sum(al, bl, t, f);
  e = __dadd_rn(e, t);
  fast_two_sum(s, e, s, e);
  e = __dadd_rn(e, f);
  fast_two_sum(s, e, rh, rl);
}
__device__ __forceinline__ void dd_mul_d(double ah, double al, double b, double& rh, double& rl) {
  double p, e;
  two_prod(ah, b, p, e);
  e = __fma_rn(al, b, e);
  fast_two_sum(p, e, rh, rl);
}

#ifndef OZ_CVT32
#define OZ_CVT32 1  // CRT integers to scaled double-doubles through 32-bit conversions
#endif
// (RN(Z) sc, (Z - RN(Z)) sc) for an exact integer Z and a power of two sc (Alg.8 l.975: z' / c
// as a double-double, no rounding beyond RN(Z)).  OZ_CVT32: from the two 32-bit halves,
// a = hi32(Z) 2^32 sc and b = lo32(Z) sc are exact, RN(a + b) = RN(Z) sc and FastTwoSum's
// error term is (Z - RN(Z)) sc exactly (|a| >= |b| or a = 0) -- the same two doubles as the
// 64-bit conversions (I2F.F64.S64, F2I.S64.F64, I2F.F64.S64), with 32-bit conversions.
__device__ __forceinline__ void scaled_split(long long Z, double sc, double& hs, double& ls) {
#if OZ_CVT32
  const double a = __dmul_rn((double)(int)(Z >> 32), __dmul_rn(sc, 4294967296.0));
  const double b = __dmul_rn((double)(unsigned)Z, sc);
  fast_two_sum(a, b, hs, ls);
#else
  const double h = __ll2double_rn(Z);
  const double l = __ll2double_rn(Z - __double2ll_rz(h));
  hs = __dmul_rn(h, sc);
  ls = __dmul_rn(l, sc);
#endif
}

// ============================================================== triple-single (TS, f4)
// x0 + x1 + x2 in fp32 words.  The op sequences are this build's reading of
// TSAdd / TSMul (DESIGN ruling 24) and must match oracle/ozfft_oracle.c op for op.
struct TSv {
  float x0, x1, x2;
};
__device__ __forceinline__ void two_sum_f(float a, float b, float& s, float& e) {
  s = __fadd_rn(a, b);
  const float bb = __fsub_rn(s, a);
  e = __fadd_rn(__fsub_rn(a, __fsub_rn(s, bb)), __fsub_rn(b, bb));
}
__device__ __forceinline__ void fast_two_sum_f(float a, float b, float& s, float& e) {
  s = __fadd_rn(a, b);
  e = __fsub_rn(b, __fsub_rn(s, a));
}
__device__ __forceinline__ void two_prod_f(float a, float b, float& p, float& e) {
  p = __fmul_rn(a, b);
  e = __fmaf_rn(a, b, -p);
}
__device__ __forceinline__ TSv ts_renorm3(float a, float b, float c) {
  float s, t3, s0, t2, s1, s2;
  two_sum_f(b, c, s, t3);
  two_sum_f(a, s, s0, t2);
  two_sum_f(t2, t3, s1, s2);
  fast_two_sum_f(s0, s1, s0, s1);
  fast_two_sum_f(s1, s2, s1, s2);
  return TSv{s0, s1, s2};
}
__device__ __forceinline__ TSv ts_from_double(double d) {
  TSv r;
  r.x0 = __double2float_rn(d);
  double t = __dsub_rn(d, (double)r.x0);
  r.x1 = __double2float_rn(t);
  t = __dsub_rn(t, (double)r.x1);
  r.x2 = __double2float_rn(t);
  return r;
}
__device__ __forceinline__ TSv ts_from_int64(long long v) {
  TSv r;
  r.x0 = __ll2float_rn(v);
  long long t = v - __float2ll_rz(r.x0);
  r.x1 = __ll2float_rn(t);
  t = t - __float2ll_rz(r.x1);
  r.x2 = __ll2float_rn(t);
  return r;
}
__device__ __forceinline__ double ts_to_double(TSv a) {
  return __dadd_rn((double)a.x0, __dadd_rn((double)a.x1, (double)a.x2));
}
__device__ __forceinline__ TSv ts_add(TSv a, TSv b) {
  float s0, e0, s1, e1, t1, f1;
  two_sum_f(a.x0, b.x0, s0, e0);
  two_sum_f(a.x1, b.x1, s1, e1);
  const float s2 = __fadd_rn(a.x2, b.x2);
  two_sum_f(e0, s1, t1, f1);
  const float t2 = __fadd_rn(__fadd_rn(f1, e1), s2);
  return ts_renorm3(s0, t1, t2);
}
__device__ __forceinline__ TSv ts_neg(TSv a) { return TSv{-a.x0, -a.x1, -a.x2}; }
__device__ __forceinline__ TSv ts_mul(TSv a, TSv b) {
  float p0, q0, p1, q1, p2, q2, s1, r1, t1, r2;
  two_prod_f(a.x0, b.x0, p0, q0);
  two_prod_f(a.x0, b.x1, p1, q1);
  two_prod_f(a.x1, b.x0, p2, q2);
  const float c = __fadd_rn(__fadd_rn(__fadd_rn(__fadd_rn(__fmul_rn(a.x0, b.x2), __fmul_rn(a.x1, b.x1)),
                                                __fmul_rn(a.x2, b.x0)), q1), q2);
  two_sum_f(p1, p2, s1, r1);
  two_sum_f(q0, s1, t1, r2);
  const float t2 = __fadd_rn(__fadd_rn(r1, r2), c);
  return ts_renorm3(p0, t1, t2);
}
__device__ __forceinline__ TSv ts_ldexp(TSv a, int e) {
  return TSv{ldexpf(a.x0, e), ldexpf(a.x1, e), ldexpf(a.x2, e)};
}
// TS split step (ruling 25): x = fl32(fl32(r0 + sigma) - sigma), digit x 2^(alpha-E),
// (r0, t) = FastTwoSum(fl32(r0 - x), r1), (r1, r2) = FastTwoSum(t, r2).
// The level constants sigma = 2^(E + rho) and 2^(alpha - E) depend on (part, level) only:
// SplitC holds them, computed once per CTA (or level), not per element.
template <bool TS>
struct SplitC {
  std::conditional_t<TS, float, double> sigma, scale;
};
// 2^e exactly: the exponent field directly in the normal range (scalbn costs ~84 clocks
// of dependent FP64 work on B200, and the small-transform kernel computes these per level)
__device__ __forceinline__ double pow2_exact(int e) {
  if (e >= -1022 && e <= 1023) return __longlong_as_double((long long)(e + 1023) << 52);
  return scalbn(1.0, e);
}
template <bool TS>
__device__ __forceinline__ SplitC<TS> split_c(int E, int alpha, int rho) {
  if constexpr (TS)
    return SplitC<TS>{ldexpf(1.0f, E + rho), ldexpf(1.0f, alpha - E)};
  else
    return SplitC<TS>{pow2_exact(E + rho), pow2_exact(alpha - E)};
}
__device__ __forceinline__ int32_t split_step_ts(TSv& r, SplitC<true> c) {
  const float sigma = c.sigma;
  const float t = __fadd_rn(r.x0, sigma);
  const float x = __fsub_rn(t, sigma);
  const int32_t D = __float2int_rz(__fmul_rn(x, c.scale));
  const float d = __fsub_rn(r.x0, x);
  float a, b;
  fast_two_sum_f(d, r.x1, a, b);
  r.x0 = a;
  fast_two_sum_f(b, r.x2, r.x1, r.x2);
  return D;
}
// x' in TS (Alg.4 TS form): TS(x), TS(omega); mode 1: TS(omega~*).  Also the max-key of
// |r0| (a NaN key when r1 or r2 is not finite, as the oracle's mu).
__device__ __forceinline__ unsigned long long ts_key(const TSv& r) {
  if (!isfinite(r.x1) || !isfinite(r.x2)) return 0x7FF8000000000000ull;
  return (unsigned long long)__double_as_longlong(fabs((double)r.x0));
}

// ceil(log2(mu)) exactly from the bits of a positive finite double (ruling 8)
__device__ __forceinline__ int ceil_log2_bits(unsigned long long u) {
  const int eb = (int)(u >> 52);
  const unsigned long long man = u & ((1ull << 52) - 1);
  if (eb == 0) return (64 - __clzll((long long)(man - 1))) - 1074;  // subnormal
  return man == 0 ? eb - 1023 : eb - 1022;
}

constexpr unsigned long long kInfBits = 0x7FF0000000000000ull;

// ============================================================== split kernels
#ifndef OZ_SPLIT_EPT
#define OZ_SPLIT_EPT 8  // elements per thread of k_split_max / k_split_digits
#endif
#ifndef OZ_SPLIT_ILP
#define OZ_SPLIT_ILP 2  // k_split_max / k_split_digits: elements per thread interleaved
#endif
#ifndef OZ_SPLIT_CL_EPT
#define OZ_SPLIT_CL_EPT 1  // elements per thread per iteration of k_split_cluster
#endif
#ifndef OZ_SPLIT_CL_MAXLEN
#define OZ_SPLIT_CL_MAXLEN (1 << 15)  // longest vector split by k_split_cluster
#endif
#ifndef OZ_SPLIT_CL_CHUNK
#define OZ_SPLIT_CL_CHUNK 256  // target elements per CTA of k_split_cluster
#endif
struct SplitParams {
  const double2* x;       // mode 0: input complex [nb][len]; mode 1: raw DD hi values [len]
  const double2* chirp;   // [len] (C, S)
  int64_t len;            // vector length (n for x', m for omega~*)
  int mode;               // 0: x' = x (.) omega (conj on load if inverse); 1: raw (lo = 0)
  int conj;               // inverse-direction wrapper (ruling 16)
  int K, alpha, rho;
  unsigned long long* mu; // [nb][2][K] max-|hi| bits per level
  int32_t* digits;        // [nb][2][K][len]
  int32_t* stats;         // [nb][stats_stride]
  int32_t* sched;         // [nb][4][sched_stride] (nullptr: no schedule)
  const int32_t* wsplit;  // kw[2], Ew[2][K] of omega~* (for the schedule)
  int L;
  int shared;             // image mode (f2): one exponent per level for both parts
};

__device__ __forceinline__ void load_xprime(const SplitParams& P, int64_t b, int64_t j, double& hr,
                                            double& lr, double& hi, double& li) {
  if (P.mode == 0) {
    const double2 xv = __ldg(&P.x[b * P.len + j]);
    const double2 w = __ldg(&P.chirp[j]);
    const double xr = xv.x, xi = P.conj ? -xv.y : xv.y;
    double p1, e1, p2, e2;
    two_prod(xr, w.x, p1, e1);
    two_prod(xi, w.y, p2, e2);
    dd_add(p1, e1, -p2, -e2, hr, lr);
    two_prod(xr, w.y, p1, e1);
    two_prod(xi, w.x, p2, e2);
    dd_add(p1, e1, p2, e2, hi, li);
  } else {
    const double2 wv = __ldg(&P.x[j]);
    hr = wv.x;
    hi = wv.y;
    lr = 0.0;
    li = 0.0;
  }
}

// x' in TS (Alg.4 TS form, steps 1-2): TS(x), TS(omega); mode 1: TS(omega~*) (f4).
__device__ __forceinline__ void load_xprime_ts(const SplitParams& P, int64_t b, int64_t j, TSv& re,
                                               TSv& im) {
  if (P.mode == 0) {
    const double2 xv = __ldg(&P.x[b * P.len + j]);
    const double2 w = __ldg(&P.chirp[j]);
    const TSv xr = ts_from_double(xv.x), xi = ts_from_double(P.conj ? -xv.y : xv.y);
    const TSv c = ts_from_double(w.x), sn = ts_from_double(w.y);
    re = ts_add(ts_mul(xr, c), ts_neg(ts_mul(xi, sn)));
    im = ts_add(ts_mul(xr, sn), ts_mul(xi, c));
  } else {
    const double2 wv = __ldg(&P.x[j]);
    re = ts_from_double(wv.x);
    im = ts_from_double(wv.y);
  }
}

// One Ozaki extraction step on (h, l) with level exponent E (Alg.6 l.781-783).
__device__ __forceinline__ int32_t split_step(double& h, double& l, SplitC<false> c) {
  const double sigma = c.sigma;
  const double t = __dadd_rn(h, sigma);
  const double d = __dsub_rn(t, sigma);
  const int32_t D = __double2int_rz(__dmul_rn(d, c.scale));
  const double r = __dsub_rn(h, d);
  fast_two_sum(r, l, h, l);
  return D;
}

__device__ __forceinline__ unsigned long long warp_max_u64(unsigned long long v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    const unsigned long long w = __shfl_xor_sync(0xffffffffu, v, o);
    v = w > v ? w : v;
  }
  return v;
}

// Max |hi| over the transform at split level `level` (levels < level applied first).
template <bool TS>
__global__ void __launch_bounds__(256) k_split_max(SplitParams P, int level) {
  const int64_t b = blockIdx.y;
  const unsigned long long* mub = P.mu + b * 2 * P.K;
  int E[2][kMaxK];
  int lv[2] = {level, level};  // levels already extracted (stop at the first mu == 0)
  bool bad = false;
  for (int v = 0; v < 2; ++v)
    for (int k = 0; k < level; ++k) {
      const unsigned long long u = mub[v * P.K + k];
      if (u >= kInfBits) bad = true;
      if (u == 0 && lv[v] == level) lv[v] = k;
      E[v][k] = (u == 0 || u >= kInfBits) ? 0 : ceil_log2_bits(u);
    }
  if (bad) return;  // non-finite transform: nothing more to compute
  __shared__ SplitC<TS> s_c[2][kMaxK];
  if (threadIdx.x < 2 * kMaxK) {
    const int v = threadIdx.x / kMaxK, k = threadIdx.x % kMaxK;
    s_c[v][k] = split_c<TS>(k < lv[v] ? E[v][k] : 0, P.alpha, P.rho);
  }
  __syncthreads();
  unsigned long long m0 = 0, m1 = 0;
  // OZ_SPLIT_ILP elements per thread and iteration as independent chains (a dependent DADD
  // costs ~25 clocks on B200); out-of-range slots redo the thread's first element
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t j0 = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; j0 < P.len; j0 += OZ_SPLIT_ILP * stride) {
    unsigned long long a0[OZ_SPLIT_ILP], a1[OZ_SPLIT_ILP];
    if constexpr (TS) {  // f4: TS words, mu over r0
      TSv r[OZ_SPLIT_ILP][2];
#pragma unroll
      for (int u = 0; u < OZ_SPLIT_ILP; ++u) {
        const int64_t j = j0 + u * stride < P.len ? j0 + u * stride : j0;
        load_xprime_ts(P, b, j, r[u][0], r[u][1]);
      }
#pragma unroll
      for (int v = 0; v < 2; ++v)
        for (int k = 0; k < lv[v]; ++k)
#pragma unroll
          for (int u = 0; u < OZ_SPLIT_ILP; ++u) (void)split_step_ts(r[u][v], s_c[v][k]);
#pragma unroll
      for (int u = 0; u < OZ_SPLIT_ILP; ++u) {
        a0[u] = ts_key(r[u][0]);
        a1[u] = ts_key(r[u][1]);
      }
    } else {
      double h[OZ_SPLIT_ILP][2], l[OZ_SPLIT_ILP][2];
#pragma unroll
      for (int u = 0; u < OZ_SPLIT_ILP; ++u) {
        const int64_t j = j0 + u * stride < P.len ? j0 + u * stride : j0;
        load_xprime(P, b, j, h[u][0], l[u][0], h[u][1], l[u][1]);
      }
#pragma unroll
      for (int v = 0; v < 2; ++v)  // a level with mu == 0 ended this part's split (Alg.6 l.780)
        for (int k = 0; k < lv[v]; ++k)
#pragma unroll
          for (int u = 0; u < OZ_SPLIT_ILP; ++u) (void)split_step(h[u][v], l[u][v], s_c[v][k]);
#pragma unroll
      for (int u = 0; u < OZ_SPLIT_ILP; ++u) {
        a0[u] = (unsigned long long)__double_as_longlong(fabs(h[u][0]));
        a1[u] = (unsigned long long)__double_as_longlong(fabs(h[u][1]));
      }
    }
#pragma unroll
    for (int u = 0; u < OZ_SPLIT_ILP; ++u) {
      m0 = a0[u] > m0 ? a0[u] : m0;  // NaN bits exceed +Inf bits: a NaN sticks
      m1 = a1[u] > m1 ? a1[u] : m1;
    }
  }
  __shared__ unsigned long long red[2][8];
  m0 = warp_max_u64(m0);
  m1 = warp_max_u64(m1);
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (lane == 0) { red[0][w] = m0; red[1][w] = m1; }
  __syncthreads();
  if (threadIdx.x < 32) {
    const int nw = blockDim.x >> 5;
    m0 = lane < nw ? red[0][lane] : 0;
    m1 = lane < nw ? red[1][lane] : 0;
    m0 = warp_max_u64(m0);
    m1 = warp_max_u64(m1);
    if (lane == 0) {
      unsigned long long* dst = P.mu + b * 2 * P.K;
      if (P.shared) m0 = m1 = m0 > m1 ? m0 : m1;  // mu = max over both parts (f2)
      if (m0) atomicMax(&dst[0 * P.K + level], m0);
      if (m1) atomicMax(&dst[1 * P.K + level], m1);
    }
  }
}

// Alg.8 flush schedule for one real convolution; writes the row layout
// [ngroups, (cexp, npairs, s0, t0, ..., s_{L-1}, t_{L-1}) x K*K].
__device__ void alg8_schedule(int kx, const int* sx, int ky, const int* sy, int K, int L,
                              int32_t* row, bool prezeroed = false) {
  const int stride = 1 + K * K * (2 + 2 * L);
  if (!prezeroed)
    for (int i = 0; i < stride; ++i) row[i] = 0;
  if (kx <= 0 || ky <= 0) return;
  int ng = 0;
  int c = sx[kx - 1] + sy[ky - 1];
  int l = 0;
  int32_t* grp = row + 1;
  grp[0] = c;
  for (int k = kx + ky - 2; k >= 0; --k) {
    const int s_lo = max(0, k - ky + 1), s_hi = min(kx - 1, k);
    for (int s = s_lo; s <= s_hi; ++s) {
      const int t = k - s;
      const int e = sx[s] + sy[t];
      if (l >= L || e != c) {  // flush the current group (l.972-979)
        ++ng;
        grp = row + 1 + ng * (2 + 2 * L);
        c = e;
        l = 0;
        grp[0] = c;
      }
      grp[2 + 2 * l] = s;
      grp[3 + 2 * l] = t;
      ++l;
      grp[1] = l;
    }
  }
  row[0] = ng + 1;
}

// Level exponents E, slice counts kv and the non-finite flag of one transform from its
// per-level maxima mu (Alg.6 l.778-780; ruling 8); `lead` threads (thread 0 / threads < 4)
// write the stats row and the four Alg.8 schedules.
__device__ __forceinline__ bool split_exponents(const SplitParams& P, int64_t b,
                                                const unsigned long long* mub, int (&E)[2][kMaxK],
                                                int (&kv)[2], bool lead, bool prezeroed = false) {
  bool bad = false;
  for (int v = 0; v < 2; ++v) {
    kv[v] = P.K;
    for (int k = 0; k < P.K; ++k) {
      const unsigned long long u = mub[v * P.K + k];
      if (u >= kInfBits) bad = true;
      E[v][k] = (u == 0 || u >= kInfBits) ? 0 : ceil_log2_bits(u);
      if (u == 0 && kv[v] == P.K) kv[v] = k;
    }
  }
  // mu of level k is only meaningful while all previous levels were non-zero
  for (int v = 0; v < 2; ++v)
    for (int k = kv[v]; k < P.K; ++k) E[v][k] = 0;
  if (bad) { kv[0] = 0; kv[1] = 0; }
  if (lead && threadIdx.x == 0) {
    int32_t* st = P.stats + b * stats_stride(P.K);
    st[0] = kv[0];
    st[1] = kv[1];
    for (int v = 0; v < 2; ++v)
      for (int k = 0; k < P.K; ++k) st[2 + v * P.K + k] = E[v][k];
    st[2 + 2 * P.K] = bad ? 1 : 0;
  }
  if (P.sched && lead && threadIdx.x < 4) {
    const int cv = threadIdx.x;
    const int a = conv_a(cv), bw = conv_b(cv);
    int sx[kMaxK], sy[kMaxK];
    const int kw = P.wsplit[bw];
    for (int k = 0; k < P.K; ++k) {
      sx[k] = P.alpha - E[a][k];                 // c = (u sigma)^-1 = 2^(alpha - E) (l.785)
      sy[k] = P.alpha - P.wsplit[2 + bw * P.K + k];
    }
    // image mode: one complex schedule in row 0 (both parts share E), rows 1-3 empty
    alg8_schedule(bad || (P.shared && cv > 0) ? 0 : kv[a], sx, kw, sy, P.K, P.L,
                  P.sched + (b * 4 + cv) * sched_stride(P.K, P.L), prezeroed);
  }
  return bad;
}

// Digits for every level, per-transform stats and (block 0) the schedules.
template <bool TS>
__global__ void __launch_bounds__(256) k_split_digits(SplitParams P) {
  const int64_t b = blockIdx.y;
  int E[2][kMaxK];
  int kv[2];
  const bool bad = split_exponents(P, b, P.mu + b * 2 * P.K, E, kv, blockIdx.x == 0);
  if (bad) return;
  __shared__ SplitC<TS> s_c[2][kMaxK];
  if (threadIdx.x < 2 * kMaxK) {
    const int v = threadIdx.x / kMaxK, k = threadIdx.x % kMaxK;
    s_c[v][k] = split_c<TS>(k < P.K ? E[v][k] : 0, P.alpha, P.rho);
  }
  __syncthreads();
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t j0 = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; j0 < P.len; j0 += OZ_SPLIT_ILP * stride) {
    if constexpr (TS) {
      TSv r[OZ_SPLIT_ILP][2];
#pragma unroll
      for (int u = 0; u < OZ_SPLIT_ILP; ++u) {
        const int64_t j = j0 + u * stride < P.len ? j0 + u * stride : j0;
        load_xprime_ts(P, b, j, r[u][0], r[u][1]);
      }
#pragma unroll
      for (int v = 0; v < 2; ++v) {
        int32_t* dv = P.digits + ((b * 2 + v) * P.K) * P.len + j0;
        for (int k = 0; k < P.K; ++k)
#pragma unroll
          for (int u = 0; u < OZ_SPLIT_ILP; ++u) {
            int32_t D = 0;
            if (k < kv[v]) D = split_step_ts(r[u][v], s_c[v][k]);
            if (j0 + u * stride < P.len) dv[k * P.len + u * stride] = D;
          }
      }
    } else {
      double h[OZ_SPLIT_ILP][2], l[OZ_SPLIT_ILP][2];
#pragma unroll
      for (int u = 0; u < OZ_SPLIT_ILP; ++u) {
        const int64_t j = j0 + u * stride < P.len ? j0 + u * stride : j0;
        load_xprime(P, b, j, h[u][0], l[u][0], h[u][1], l[u][1]);
      }
#pragma unroll
      for (int v = 0; v < 2; ++v) {
        int32_t* dv = P.digits + ((b * 2 + v) * P.K) * P.len + j0;
        for (int k = 0; k < P.K; ++k)
#pragma unroll
          for (int u = 0; u < OZ_SPLIT_ILP; ++u) {
            int32_t D = 0;
            if (k < kv[v]) D = split_step(h[u][v], l[u][v], s_c[v][k]);
            if (j0 + u * stride < P.len) dv[k * P.len + u * stride] = D;
          }
      }
    }
  }
}

// ============================================================== fused small-n split
// n <= kSplitClusterMaxLen: a1 + a2 of one transform in ONE launch.  One thread-block
// cluster of CS <= 8 CTAs per transform; each CTA keeps its chunk of x' (DD: hi, lo of both
// parts; TS: the three words of both parts) in shared memory across the K levels, and the
// per-level max |hi| (Alg.6 l.778/786) is a block reduction plus a DSMEM exchange of the
// CS partial maxima (one cluster barrier per level).  Level k's digits are written in the
// pass that computes level k+1's max.  Every element goes through the same operation
// sequence as in k_split_max + k_split_digits and max is exact, so the digits, stats and
// schedules are bitwise those of the multi-launch path (which stays for larger n).
// (For a non-finite transform both leave the digits unused: stats say kv = 0.)
constexpr int kSplitClusterMaxLen = OZ_SPLIT_CL_MAXLEN;
#ifndef OZ_SPLIT_CL_THREADS
#define OZ_SPLIT_CL_THREADS 512
#endif
constexpr int kSplitClusterThreads = OZ_SPLIT_CL_THREADS;

template <bool TS>
__global__ void __launch_bounds__(kSplitClusterThreads) k_split_cluster(SplitParams P, int chunk) {
  extern __shared__ __align__(16) unsigned char split_sm[];
  __shared__ unsigned long long s_part[kMaxK][2];           // this CTA's max per level / part
  __shared__ unsigned long long s_red[2][kSplitClusterThreads / 32];
  __shared__ unsigned long long s_mu[2 * kMaxK];
  cg::cluster_group cl = cg::this_cluster();
  const int rank = (int)cl.block_rank();
  const int cs = (int)cl.num_blocks();
  const int64_t b = blockIdx.y;
  const int K = P.K;
  const int64_t j0 = (int64_t)rank * chunk;
  const int cnt = (int)(P.len - j0 < chunk ? (P.len - j0 > 0 ? P.len - j0 : 0) : chunk);
  double* sh = reinterpret_cast<double*>(split_sm);  // DD: h[2][chunk], l[2][chunk]
  float* sr = reinterpret_cast<float*>(split_sm);    // TS: r[2][3][chunk]
  unsigned long long mu[2][kMaxK];
  int E[2][kMaxK], kv[2] = {K, K};
  for (int v = 0; v < 2; ++v)
    for (int k = 0; k < kMaxK; ++k) { mu[v][k] = 0; E[v][k] = 0; }
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  for (int level = 0; level <= K; ++level) {
    SplitC<TS> lc[2];  // level - 1's constants
#pragma unroll
    for (int v = 0; v < 2; ++v) lc[v] = split_c<TS>(level > 0 ? E[v][level - 1] : 0, P.alpha, P.rho);
    unsigned long long m0 = 0, m1 = 0;
    for (int i0 = threadIdx.x; i0 < cnt; i0 += OZ_SPLIT_CL_EPT * blockDim.x)
#pragma unroll
    for (int u = 0; u < OZ_SPLIT_CL_EPT; ++u) {
      // out-of-range slots recompute element cnt - 1 and store nothing (as in k_split_max)
      const bool ok = i0 + u * (int)blockDim.x < cnt;
      const int i = ok ? i0 + u * (int)blockDim.x : cnt - 1;
      const int64_t j = j0 + i;
      unsigned long long a0, a1;
      if constexpr (TS) {
        TSv r[2];
        if (level == 0) {
          load_xprime_ts(P, b, j, r[0], r[1]);
        } else {
#pragma unroll
          for (int v = 0; v < 2; ++v)
            r[v] = TSv{sr[(v * 3 + 0) * chunk + i], sr[(v * 3 + 1) * chunk + i], sr[(v * 3 + 2) * chunk + i]};
#pragma unroll
          for (int v = 0; v < 2; ++v) {  // level - 1's digits (Alg.6 l.781-785)
            int32_t D = 0;
            if (level - 1 < kv[v]) D = split_step_ts(r[v], lc[v]);
            if (ok) P.digits[((b * 2 + v) * K + level - 1) * P.len + j] = D;
          }
        }
        if (level == K) continue;
#pragma unroll
        for (int v = 0; v < 2 && ok; ++v) {
          sr[(v * 3 + 0) * chunk + i] = r[v].x0;
          sr[(v * 3 + 1) * chunk + i] = r[v].x1;
          sr[(v * 3 + 2) * chunk + i] = r[v].x2;
        }
        a0 = ts_key(r[0]);
        a1 = ts_key(r[1]);
      } else {
        double h[2], l[2];
        if (level == 0) {
          load_xprime(P, b, j, h[0], l[0], h[1], l[1]);
        } else {
#pragma unroll
          for (int v = 0; v < 2; ++v) {
            h[v] = sh[v * chunk + i];
            l[v] = sh[(2 + v) * chunk + i];
          }
#pragma unroll
          for (int v = 0; v < 2; ++v) {
            int32_t D = 0;
            if (level - 1 < kv[v]) D = split_step(h[v], l[v], lc[v]);
            if (ok) P.digits[((b * 2 + v) * K + level - 1) * P.len + j] = D;
          }
        }
        if (level == K) continue;
#pragma unroll
        for (int v = 0; v < 2 && ok; ++v) {
          sh[v * chunk + i] = h[v];
          sh[(2 + v) * chunk + i] = l[v];
        }
        a0 = (unsigned long long)__double_as_longlong(fabs(h[0]));
        a1 = (unsigned long long)__double_as_longlong(fabs(h[1]));
      }
      if (!ok) a0 = a1 = 0;
      m0 = a0 > m0 ? a0 : m0;  // NaN bits exceed +Inf bits: a NaN sticks
      m1 = a1 > m1 ? a1 : m1;
    }
    if (level == K) break;
    m0 = warp_max_u64(m0);
    m1 = warp_max_u64(m1);
    if (lane == 0) { s_red[0][warp] = m0; s_red[1][warp] = m1; }
    __syncthreads();
    if (warp == 0) {
      const int nw = blockDim.x >> 5;
      m0 = lane < nw ? s_red[0][lane] : 0;
      m1 = lane < nw ? s_red[1][lane] : 0;
      m0 = warp_max_u64(m0);
      m1 = warp_max_u64(m1);
      if (lane == 0) { s_part[level][0] = m0; s_part[level][1] = m1; }
    }
    if (cs > 1)
      cl.sync();  // every CTA's partial max of this level is visible cluster-wide
    else
      __syncthreads();
    m0 = m1 = 0;
    for (int r = 0; r < cs; ++r) {
      const unsigned long long* rp = cl.map_shared_rank(&s_part[level][0], r);
      m0 = rp[0] > m0 ? rp[0] : m0;
      m1 = rp[1] > m1 ? rp[1] : m1;
    }
    if (P.shared) m0 = m1 = m0 > m1 ? m0 : m1;  // mu = max over both parts (f2)
    mu[0][level] = m0;
    mu[1][level] = m1;
    // the exponents and slice counts as k_split_max / k_split_digits derive them
    bool bad = false;
    for (int v = 0; v < 2; ++v) {
      const unsigned long long u = mu[v][level];
      if (u >= kInfBits) bad = true;
      E[v][level] = (u == 0 || u >= kInfBits) ? 0 : ceil_log2_bits(u);
      if (u == 0 && kv[v] == K) kv[v] = level;
    }
    if (bad) break;  // k_split_max stops here too: later levels keep mu = 0
  }
  // mu (as the multi-launch path leaves it), stats and schedules: rank 0
  if (rank == 0) {
    if (threadIdx.x < 2 * K) s_mu[threadIdx.x] = mu[threadIdx.x / K][threadIdx.x % K];
    __syncthreads();
    if (threadIdx.x < 2 * K) P.mu[b * 2 * K + threadIdx.x] = s_mu[threadIdx.x];
    int Ef[2][kMaxK], kvf[2];
    (void)split_exponents(P, b, s_mu, Ef, kvf, true);
  }
  if (cs > 1) cl.sync();  // no CTA leaves while another may still read its s_part
}

// ============================================================== NTT building blocks
// twiddle load: read-only global path, or a shared-memory table (generic load)
template <bool SMEM>
__device__ __forceinline__ uint2 tw_load(const uint2* p) {
  if constexpr (SMEM)
    return *p;
  else
    return __ldg(p);
}

// A group of 2^S registers x[k] holding global positions gbase + k*gstep, with
// rmod = gbase mod gstep.  DIF stages h = gstep*2^(S-1) .. gstep (block length 2h):
//   (u, v) -> (u + v, (u - v) * T[h + (pos mod h)]),  T[h + j] = w_{2h}^j.
// x is [NV][E] (E = elements per thread); the group occupies x[v][off .. off + 2^S).
// UNIT: the caller guarantees rmod == 0 and gstep == 1 (the step-1 round of a row), so the
// twiddle index is compile-time and the butterflies with T[h] = w^0 = 1 skip the product.
// ZHI: the upper half of the group's block is zero on entry (zero-padded input, n <= m/2),
// so the first stage is (u, 0) -> (u, u * w).
template <int S, int NV, int E, bool UNIT = false, bool SMEM_T = false, bool ZHI = false>
__device__ __forceinline__ void dif_group(uint32_t (&x)[NV][E], int off, uint32_t rmod,
                                          uint32_t gstep, const uint2* __restrict__ T, uint32_t p) {
  if constexpr (UNIT) {
    rmod = 0u;
    gstep = 1u;
  }
#pragma unroll
  for (int st = S - 1; st >= 0; --st) {
    const int d = 1 << st;
    const uint32_t h = gstep << st;
#pragma unroll
    for (int k = 0; k < (1 << S); ++k) {
      if (k & d) continue;
      if (ZHI && st == S - 1) {
        const uint2 w = tw_load<SMEM_T>(&T[h + rmod + (uint32_t)(k & (d - 1)) * gstep]);
#pragma unroll
        for (int v = 0; v < NV; ++v) x[v][off + k + d] = mul_shoup(x[v][off + k], w, p);
        continue;
      }
      if (UNIT && (k & (d - 1)) == 0) {  // (u - v) * 1
#pragma unroll
        for (int v = 0; v < NV; ++v) {
          const uint32_t a = x[v][off + k], b = x[v][off + k + d];
          x[v][off + k] = add_mod(a, b, p);
          x[v][off + k + d] = sub_mod(a, b, p);
        }
        continue;
      }
      const uint2 w = tw_load<SMEM_T>(&T[h + rmod + (uint32_t)(k & (d - 1)) * gstep]);  // shared by NV
#pragma unroll
      for (int v = 0; v < NV; ++v) {
        const uint32_t a = x[v][off + k], b = x[v][off + k + d];
        x[v][off + k] = add_mod(a, b, p);
        x[v][off + k + d] = mul_shoup(a + (p - b), w, p);
      }
    }
  }
}
// DIT stages h = gstep .. gstep*2^(S-1): v' = v * Tinv[h + (pos mod h)]; (u + v', u - v')
// CANON0: the group's inputs are canonical (< p; the first round of an inverse row item reads
// the pointwise REDC outputs), so the w^0 = 1 butterflies of the first stage skip the
// canonicalising min of v (it only guards the lazy < 2p values of later stages)
// LZ: the last stage leaves its outputs lazy (< 2p): only for outputs that are consumed as
// the v-operand of a Shoup product (two-pass rows of odd index, see k_row_fused)
template <int S, int NV, int E, bool UNIT = false, bool SMEM_T = false, bool CANON0 = false, bool LZ = false>
__device__ __forceinline__ void dit_group(uint32_t (&x)[NV][E], int off, uint32_t rmod,
                                          uint32_t gstep, const uint2* __restrict__ T, uint32_t p) {
  if constexpr (UNIT) {
    rmod = 0u;
    gstep = 1u;
  }
#pragma unroll
  for (int st = 0; st < S; ++st) {
    const int d = 1 << st;
    const uint32_t h = gstep << st;
#pragma unroll
    for (int k = 0; k < (1 << S); ++k) {
      if (k & d) continue;
      const bool one = UNIT && (k & (d - 1)) == 0;  // twiddle w^0 = 1
      const uint2 w =
          one ? make_uint2(1u, 0u) : tw_load<SMEM_T>(&T[h + rmod + (uint32_t)(k & (d - 1)) * gstep]);
#pragma unroll
      for (int v = 0; v < NV; ++v) {
        const uint32_t a = x[v][off + k];  // always canonical: it was a "u" of this stage
        const uint32_t vin = x[v][off + k + d];  // may be lazy (< 2p)
        const uint32_t b = one ? ((CANON0 && st == 0) ? vin : min(vin, vin - p)) : mul_shoup(vin, w, p);
        if ((st + 1 < S && (k & (2 * d))) || (LZ && st + 1 == S)) {
          // both outputs are the "v" operand of the next stage, whose Shoup product
          // accepts any 32-bit input: keep them in [0, 2p), skip the subtractions
          x[v][off + k] = a + b;
          x[v][off + k + d] = a + (p - b);
        } else {
          x[v][off + k] = add_mod(a, b, p);
          x[v][off + k + d] = sub_mod(a, b, p);
        }
      }
    }
  }
}

// Padded shared-memory index: one word of padding per 2^LOGE words.
template <int LOGE>
__device__ __forceinline__ uint32_t pad_idx(uint32_t e) { return e + (e >> LOGE); }

// Round structure of a length-2^LOGN sub-transform with 2^LOGE elements per thread, fixed at
// compile time.  Rounds have LOGE radix-2 stages except a partial round that comes first
// in DIF order (block length 2^LOGN) / last in DIT order, so that the step-1 round always
// has 2^LOGE-element groups (conflict-free padded smem).
template <int LOGN, bool INV, int R, int LOGE = 4>
struct RoundT {
  static constexpr int E = 1 << LOGE;
  static constexpr int nr = (LOGN + LOGE - 1) / LOGE;
  static constexpr int rd = INV ? (nr - 1 - R) : R;  // index in DIF order
  static constexpr int S = rd == 0 ? LOGN - LOGE * (nr - 1) : LOGE;  // stages in the round
  static constexpr int lb = rd == 0 ? LOGN : LOGE * (nr - rd);       // log2 block length
  static constexpr int logstep = lb - S;
  static constexpr int cnt = LOGN >= LOGE ? E : (1 << LOGN);  // elements per thread
  static constexpr int Tv = LOGN >= LOGE ? (1 << (LOGN - LOGE)) : 1;
};

// Element index of register i of thread tv in round R.
template <int LOGN, bool INV, int R, int LOGE = 4>
__device__ __forceinline__ uint32_t round_elem(int tv, int i) {
  using RT = RoundT<LOGN, INV, R, LOGE>;
  const uint32_t g = (uint32_t)(tv + (i >> RT::S) * RT::Tv);
  const uint32_t k = (uint32_t)(i & ((1 << RT::S) - 1));
  return ((g >> RT::logstep) << RT::lb) + (g & ((1u << RT::logstep) - 1)) + (k << RT::logstep);
}

// Shared-memory slot of register i in round R: pad(base_g) + koff(k), where base_g is the
// group's first element and koff(k) = k*step + (k*step >> LOGE) is a compile-time constant
// (valid because every block has length >= 2^LOGE when a round touches smem), so the
// per-element address is a base register plus an immediate offset.
template <int LOGN, bool INV, int R, int CB, int LOGE = 4>
__device__ __forceinline__ uint32_t* round_slot(uint32_t* sm, int tv, int i) {
  using RT = RoundT<LOGN, INV, R, LOGE>;
  const uint32_t g = (uint32_t)(tv + (i >> RT::S) * RT::Tv);
  const uint32_t k = (uint32_t)(i & ((1 << RT::S) - 1));
  const uint32_t base = ((g >> RT::logstep) << RT::lb) + (g & ((1u << RT::logstep) - 1));
  const uint32_t ks = k << RT::logstep;
  return sm + (pad_idx<LOGE>(base) + ks + (ks >> LOGE)) * CB;
}

// Is the exchange between rounds R and R + 1 confined to one warp?  With one group per
// thread in both rounds, the values of a block of the coarser round (larger block length,
// round R in DIF order, R + 1 in DIT order) are read and written only by the 2^logstep * CB
// threads that own it in either round; if they fit in an aligned warp, __syncwarp suffices.
template <int LOGN, bool INV, int R, int CB, int LOGE>
struct RoundSync {
  using A = RoundT<LOGN, INV, R, LOGE>;
  using B = RoundT<LOGN, INV, R + 1, LOGE>;
  static constexpr bool one_group = A::cnt == (1 << A::S) && B::cnt == (1 << B::S);
  static constexpr int coarse_logstep = INV ? B::logstep : A::logstep;
  static constexpr bool warp_local =
      A::Tv * CB <= 32 || (one_group && (1 << coarse_logstep) * CB <= 32);
};

// Staged copy of the step-1 round's twiddles (logstep == 0): in that round every thread
// reads T[h + gb_mod + j * gs] (h = gs 2^st), which depends only on gb_mod; a kernel may
// stage these entries (e.g. per column in shared memory) as T0[(gs0 << st) + gb0 + j gs0].
struct Tw0 {
  const uint2* T;
  uint32_t gb, gs;
};

template <int LOGN, bool INV, int R, int CB, int NV, int LOGE, bool UNIT, bool T0S, bool ZHI,
          bool TGEN, bool LZ, class LoadF, class StoreF>
__device__ __forceinline__ void sub_ntt_round(uint32_t (&x)[NV][1 << LOGE], int tv,
                                              uint32_t* const (&sm)[NV], uint32_t gb_mod,
                                              uint32_t gs, const uint2* __restrict__ T, Tw0 t0,
                                              uint32_t p, LoadF& load_first, StoreF& store_last) {
  using RT = RoundT<LOGN, INV, R, LOGE>;
  constexpr int E = 1 << LOGE;
  constexpr uint32_t step = 1u << RT::logstep;
#pragma unroll
  for (int v = 0; v < NV; ++v)
#pragma unroll
    for (int i = 0; i < RT::cnt; ++i) {
      if constexpr (R == 0)
        x[v][i] = load_first(v, i, round_elem<LOGN, INV, R, LOGE>(tv, i));
      else
        x[v][i] = *round_slot<LOGN, INV, R, CB, LOGE>(sm[v], tv, i);
    }
#pragma unroll
  for (int u = 0; u < (RT::cnt >> RT::S); ++u) {
    const uint32_t g = (uint32_t)(tv + u * RT::Tv);
    const uint32_t rmod = gb_mod + (g & (step - 1)) * gs;
    constexpr bool unit = UNIT && RT::logstep == 0;  // rmod == gb_mod == 0, gstep == gs == 1
    constexpr bool zhi = ZHI && !INV && R == 0;  // first DIF stage of the first round
    if constexpr (T0S && RT::logstep == 0) {  // staged step-1 twiddles
      if constexpr (INV)
        dit_group<RT::S, NV, E, false, true>(x, u * (1 << RT::S), t0.gb, t0.gs, t0.T, p);
      else
        dif_group<RT::S, NV, E, false, true, zhi>(x, u * (1 << RT::S), t0.gb, t0.gs, t0.T, p);
    } else if constexpr (INV) {
      // round 0 reads load_first's values: canonical for every UNIT (row) caller
      dit_group<RT::S, NV, E, unit, TGEN, unit && R == 0, LZ && R == RT::nr - 1>(x, u * (1 << RT::S), rmod,
                                                                            step * gs, T, p);
    } else {
      dif_group<RT::S, NV, E, unit, TGEN, zhi>(x, u * (1 << RT::S), rmod, step * gs, T, p);
    }
  }
#pragma unroll
  for (int v = 0; v < NV; ++v)
#pragma unroll
    for (int i = 0; i < RT::cnt; ++i) {
      if constexpr (R == RT::nr - 1)
        store_last(v, i, round_elem<LOGN, INV, R, LOGE>(tv, i), x[v][i]);
      else
        *round_slot<LOGN, INV, R, CB, LOGE>(sm[v], tv, i) = x[v][i];
    }
  if constexpr (R != RT::nr - 1) {
    if constexpr (RoundSync<LOGN, INV, R, CB, LOGE>::warp_local)
      __syncwarp();  // every value read in round R + 1 was written by the same warp
    else
      __syncthreads();
  }
}

template <int LOGN, bool INV, int R, int CB, int NV, int LOGE, bool UNIT, bool T0S, bool ZHI,
          bool TGEN, bool LZ, class LoadF, class StoreF>
__device__ __forceinline__ void sub_ntt_rounds(uint32_t (&x)[NV][1 << LOGE], int tv,
                                               uint32_t* const (&sm)[NV], uint32_t gb_mod,
                                               uint32_t gs, const uint2* __restrict__ T, Tw0 t0,
                                               uint32_t p, LoadF& load_first, StoreF& store_last) {
  if constexpr (R < RoundT<LOGN, INV, 0, LOGE>::nr) {
    sub_ntt_round<LOGN, INV, R, CB, NV, LOGE, UNIT, T0S, ZHI, TGEN, LZ>(x, tv, sm, gb_mod, gs, T, t0, p,
                                                                   load_first, store_last);
    sub_ntt_rounds<LOGN, INV, R + 1, CB, NV, LOGE, UNIT, T0S, ZHI, TGEN, LZ>(x, tv, sm, gb_mod, gs, T, t0, p,
                                                                        load_first, store_last);
  }
}

// Length-2^LOGN sub-transforms of NV vectors at the same positions, executed cooperatively
// by 2^max(LOGN-LOGE,0) threads (index tv), 2^LOGE elements per thread and vector per round
// in rounds of <= LOGE radix-2 stages; twiddles are loaded once for the NV vectors, and
// shared memory (padded, interleave CB) is used between rounds (one buffer per vector).
//   INV = false: DIF stages len = N .. 2;   INV = true: DIT stages len = 2 .. N.
// Element e has global position gbase_vec + e*gs; gb_mod = gbase_vec mod (gs*step) for
// every step used (0 for rows, the column index for columns).  load_first(v, i, e) gives
// the round-0 input of register i / element e of vector v; store_last(v, i, e, val)
// consumes the final values.  The buffers must be free for writes on entry.  UNIT: the
// caller passes gb_mod == 0 and gs == 1 (rows), enabling the compile-time step-1 round.
template <int LOGN, bool INV, int CB, int NV, int LOGE = 4, bool UNIT = false, bool T0S = false,
          bool ZHI = false, bool TGEN = false, bool LZ = false, class LoadF, class StoreF>
__device__ __forceinline__ void sub_ntt_multi(int tv, uint32_t* const (&sm)[NV], uint32_t gb_mod,
                                              uint32_t gs, const uint2* __restrict__ T, Tw0 t0,
                                              uint32_t p, LoadF&& load_first, StoreF&& store_last) {
  if constexpr (LOGN == 0) {  // N == 1: identity
    if (tv == 0)
#pragma unroll
      for (int v = 0; v < NV; ++v) store_last(v, 0, 0u, load_first(v, 0, 0u));
  } else {
    uint32_t x[NV][1 << LOGE];
    sub_ntt_rounds<LOGN, INV, 0, CB, NV, LOGE, UNIT, T0S, ZHI, TGEN, LZ>(x, tv, sm, gb_mod, gs, T, t0, p,
                                                                    load_first, store_last);
  }
}

// Single-vector form: load_first(i, e), store_last(i, e, val).  TGEN: T may point to shared
// memory (generic loads instead of the read-only global path).
template <int LOGN, bool INV, int CB, int LOGE = 4, bool UNIT = false, bool TGEN = false, bool LZ = false,
          class LoadF, class StoreF>
__device__ __forceinline__ void sub_ntt(int tv, uint32_t* __restrict__ sm, uint32_t gb_mod,
                                        uint32_t gs, const uint2* __restrict__ T, uint32_t p,
                                        LoadF&& load_first, StoreF&& store_last) {
  uint32_t* const sms[1] = {sm};
  sub_ntt_multi<LOGN, INV, CB, 1, LOGE, UNIT, false, false, TGEN, LZ>(
      tv, sms, gb_mod, gs, T, Tw0{nullptr, 0u, 0u}, p,
      [&](int, int i, uint32_t e) { return load_first(i, e); },
      [&](int, int i, uint32_t e, uint32_t v) { store_last(i, e, v); });
}
// ... with the step-1 round's twiddles read from a staged copy (Tw0).
template <int LOGN, bool INV, int CB, int LOGE = 4, bool ZHI = false, class LoadF, class StoreF>
__device__ __forceinline__ void sub_ntt_t0(int tv, uint32_t* __restrict__ sm, uint32_t gb_mod,
                                           uint32_t gs, const uint2* __restrict__ T, Tw0 t0,
                                           uint32_t p, LoadF&& load_first, StoreF&& store_last) {
  uint32_t* const sms[1] = {sm};
  sub_ntt_multi<LOGN, INV, CB, 1, LOGE, false, true, ZHI>(
      tv, sms, gb_mod, gs, T, t0, p, [&](int, int i, uint32_t e) { return load_first(i, e); },
      [&](int, int i, uint32_t e, uint32_t v) { store_last(i, e, v); });
}

// Stage the step-1 round twiddles of the Cb columns [col0, col0 + Cb) of a column pass:
// dst[(Cb << st) + c + j Cb] = T[(C << st) + col0 + c + j C], st < S1, j < 2^st (indices
// 1 .. 2^S1 - 1 in units of Cb; S1 = stages of that round).  All threads of the CTA.
template <int S1, int Cb>
__device__ __forceinline__ void stage_col_tw0(uint2* dst, const uint2* __restrict__ T, uint32_t C,
                                              uint32_t col0) {
  for (int i = threadIdx.x; i < ((1 << S1) - 1) * Cb; i += blockDim.x) {
    const uint32_t r = 1u + (uint32_t)i / Cb, c = (uint32_t)i % Cb;  // r = 2^st + j
    dst[r * Cb + c] = T[r * C + col0 + c];
  }
}

__device__ __forceinline__ uint32_t lift(int32_t D, uint32_t p) {
  return D >= 0 ? (uint32_t)D : (uint32_t)D + p;  // canonical lift (ruling 5)
}

// ============================================================== column passes
struct ColParams {
  int logm, logC, logR, logCb;
  int64_t nb;
  int K, L;
  uint32_t p[2];
  const uint2* tw;        // [2 prime][2 dir][m]
  // forward
  const int32_t* digits;  // [nb][2][K][in_len]
  int64_t in_len;         // n (x') or m (omega~*)
  uint32_t* Y;            // [nb][2 q][2 a][K][m]
  // inverse
  const uint32_t* G;      // [nb][2 q][4 cv][K*K][m]
  uint32_t* res;          // [nb][4 cv][2 q][rg][n]
  int rg;                 // group stride of res (K*K; the schedule's max group count when sharded)
  int64_t n;
  const int32_t* stats;   // [nb][stats_stride]
  const int32_t* sched;   // [nb][4][sched_stride]
  uint32_t unit_mask;
  uint32_t* res_peers[8];  // unit-sharded transform, peer-memory exchange: residues also stored
  int npeers;              // into these buffers (same offsets as res)
  int image;              // f2: the forward vectors are the digit images D_re +- iota D_im
  uint2 io[2][2];         // [q][image] Shoup pair of iota_q (image 0) or p_q - iota_q (1)
};

// Digit image a = 0: D_re + iota D_im, a = 1: D_re - iota D_im (mod p), canonical (f2).
__device__ __forceinline__ uint32_t digit_image(int32_t dre, int32_t dim, uint2 io, uint32_t p) {
  const uint32_t r = dre >= 0 ? (uint32_t)dre : (uint32_t)dre + p;
  const uint32_t i = dim >= 0 ? (uint32_t)dim : (uint32_t)dim + p;
  return add_mod(r, mul_shoup(i, io, p), p);
}

// Elements per thread per round (log2) of the row and column sub-transforms: 32 for the
// one-warp rows of C = 2^10 (two-pass plans) and for columns of R >= 2^9, else 16.
#ifndef OZ_ROW_LOGE11
#define OZ_ROW_LOGE11 4  // elements per thread (log2) of the two-pass rows of C = 2^11
#endif
__host__ __device__ constexpr int row_loge(int logC, bool two_pass) {
  return two_pass && logC == 11 ? OZ_ROW_LOGE11 : (two_pass && logC == 10 ? 5 : 4);
}
#ifndef OZ_COL_E32_MIN_LOGR
#define OZ_COL_E32_MIN_LOGR 9
#endif
__host__ __device__ constexpr int col_loge(int logR) { return logR >= OZ_COL_E32_MIN_LOGR ? 5 : 4; }

#ifndef OZ_CI_CB_SHIFT
#define OZ_CI_CB_SHIFT 0
#endif
#ifndef OZ_CI_CB_SHIFT_FULL
#define OZ_CI_CB_SHIFT_FULL 0
#endif
#ifndef OZ_IMG_CB_SHIFT
#define OZ_IMG_CB_SHIFT 1
#endif
#ifndef OZ_COL_ZHI
#define OZ_COL_ZHI 1  // forward column pass: zero upper half of padded inputs (dif_group ZHI)
#endif
#ifndef OZ_CI_MINB
#define OZ_CI_MINB 3
#endif
#ifndef OZ_CI_SNAKE_MIN  // k_col_inv_crt tile order q0 q1 | q1 q0 | ... for these log2 R
#define OZ_CI_SNAKE_MIN 6  // (measured: R = 2^6 c5 -3.6 %, 2^7 c4 -7 %; 2^4 c2 and 2^8 c3 +1 %)
#endif
#ifndef OZ_CI_SNAKE_MAX
#define OZ_CI_SNAKE_MAX 7
#endif
#ifndef OZ_CI_RACC
#define OZ_CI_RACC 0  // k_col_inv_crt: DD accumulators in registers (<= 8 slots per thread); measured
                      // slower: c3 821 us at 127 registers / 2 CTAs, 931 at 80 / 3 (spills), vs 763
#endif
__host__ __device__ constexpr bool ci_racc(int nh) { return OZ_CI_RACC && nh <= 8; }
#ifndef OZ_CI_GACC
#define OZ_CI_GACC 0  // k_col_inv_crt: DD accumulators read-modify-written in place in the output S
#endif                // (L2-resident, .cg) instead of 32 KB of shared memory per CTA: more L1 for the
                      // column twiddles
__host__ __device__ constexpr bool ci_gacc(int nh) { return OZ_CI_GACC && !ci_racc(nh); }
#ifndef OZ_CI_DB
#define OZ_CI_DB 0  // k_col_inv_crt: double-buffered exchange tile (measured slower: c3 873 vs 763 us,
                    // the larger shared-memory carveout leaves less L1 for the column twiddles)
#endif
#ifndef OZ_CI_T0S
#define OZ_CI_T0S 8  // k_col_inv_crt: step-1 round column twiddles staged in shared memory
#endif  // for log2 R >= this (c3 803 -> 769 us; shorter columns lose: c4 658 -> 715, c2 132 -> 215,
        // wider column blocks make the table large and the snake order already reuses L1)
#ifndef OZ_CI_FETCH_FIRST
#define OZ_CI_FETCH_FIRST 1  // k_col_inv_crt: the first tile's loads issued before the CTA's set-up (c3 176.76 -> 177.18 GFLOP/s)
#endif
#ifndef OZ_CI_ILP
#define OZ_CI_ILP 4  // k_col_inv_crt: CRT + DD chains interleaved per batch
#endif
#ifndef OZ_CF_MINB
#define OZ_CF_MINB 5
#endif
#ifndef OZ_CF_QLOOP
#define OZ_CF_QLOOP 0  // k_col_fwd (real mode): one CTA does both primes of its (part, column block);
                       // measured slower (c3 col_fwd 180.5 vs 175.8 us, c2 44.2 vs 37.3 us): half as
                       // many CTAs, and the first tile load is already hidden behind the twiddle staging
#endif
template <int LOGR>
struct ColCfg {
  static constexpr int min_blocks_fwd = col_loge(LOGR) == 5 ? 1 : OZ_CF_MINB;
  static constexpr int min_blocks_inv_crt = col_loge(LOGR) == 5 ? 1 : OZ_CI_MINB;
};

// Column tile geometry: R x Cb columns with (R / E) * Cb = 256 threads (Cb >= 8 so that each
// row segment is at least one 32-byte sector; the long columns of R = 2^11, 2^12 -- m = 2^23,
// 2^24, the primes' limit -- take Cb = 4, 2 to stay at 256 threads).
__host__ __device__ constexpr int col_log_cb_raw(int logR) {
  return logR >= col_loge(logR) ? 8 - (logR - col_loge(logR)) : 8;
}
__host__ __device__ constexpr int col_log_cb(int logR, int logC) {
  return (col_log_cb_raw(logR) < (logR >= 11 ? 1 : 3) ? (logR >= 11 ? 1 : 3) : col_log_cb_raw(logR)) > logC
             ? logC
             : (col_log_cb_raw(logR) < (logR >= 11 ? 1 : 3) ? (logR >= 11 ? 1 : 3) : col_log_cb_raw(logR));
}

// Stages of the column pass's step-1 round (DIF: the last round; DIT: the first).
__host__ __device__ constexpr int col_s1(int logR) {
  return logR >= col_loge(logR) ? col_loge(logR) : logR;
}

// Forward column pass: global DIF stages len = m .. 2C on columns of the R x C view.
// One CTA per (transform, prime, part, column block) loops over the part's slices; the
// next slice's column tile is loaded while the current one is transformed.
// ZHI: padded plan (n <= m/2): rows >= R/2 of every column are zero, the first DIF stage
// is a plain product (dif_group ZHI).
template <int LOGR, int LOGC, bool IMG, bool ZHI>
__global__ void __launch_bounds__(256, ColCfg<LOGR>::min_blocks_fwd) k_col_fwd(ColParams P) {
  extern __shared__ uint32_t smem[];
  constexpr int LOGCB = col_log_cb(LOGR, LOGC);
  constexpr int LOGE = col_loge(LOGR);
  constexpr int E = 1 << LOGE;
  constexpr int Cb = 1 << LOGCB;
  constexpr uint32_t C = 1u << LOGC;
  constexpr uint32_t m = 1u << (LOGR + LOGC);
  constexpr uint32_t ncb = 1u << (LOGC - LOGCB);
  constexpr int CNT = RoundT<LOGR, false, 0, LOGE>::cnt;
  const uint32_t cb = blockIdx.x % ncb;
  // OZ_CF_QLOOP (real mode): one CTA per (transform, part, column block) transforms the part's
  // slices for BOTH primes in turn -- 2 ka tiles per CTA instead of ka, so only one tile load
  // in 2 ka (not one in ka) has nothing to overlap with; the raw digits are prefetched and
  // lifted (ruling 5) when the tile starts.  Otherwise v = (b * 2 + q) * 2 + a.
  constexpr bool QL = OZ_CF_QLOOP && !IMG;
  uint32_t v = blockIdx.x / ncb;
  const int a = (int)(v & 1); v >>= 1;
  int q0 = 0;
  if constexpr (!QL) { q0 = (int)(v & 1); v >>= 1; }
  const int64_t b = v;
  const int32_t* st = P.stats + b * stats_stride(P.K);
  const int ka = st[a];  // 0 if the transform is non-finite
  // unit (cv, q) needs part a if conv_a(cv) == a
  auto need = [&](int q) {
    return a == 0 ? ((1u << (0 * 2 + q)) | (1u << (3 * 2 + q))) : ((1u << (1 * 2 + q)) | (1u << (2 * 2 + q)));
  };
  int nq = 1;
  if constexpr (QL) {
    const bool n0 = (P.unit_mask & need(0)) != 0, n1 = (P.unit_mask & need(1)) != 0;
    if (!n0 && !n1) return;
    q0 = n0 ? 0 : 1;
    nq = n0 && n1 ? 2 : 1;
  } else {
    if (!(P.unit_mask & need(q0))) return;
  }
  if (ka == 0) return;
  const int c = threadIdx.x & (Cb - 1);
  const int tv = threadIdx.x >> LOGCB;
  const uint32_t col = (cb << LOGCB) + c;
  const uint32_t lim = P.in_len > col ? (uint32_t)(P.in_len - col) : 0u;  // e*C < lim <=> i < in_len
  constexpr int S1 = col_s1(LOGR);
  constexpr uint32_t TILEW = (((1u << LOGR) + (1u << LOGR) / E + 1) * Cb + 1) & ~1u;  // 8-byte aligned
  uint2* tw0 = reinterpret_cast<uint2*>(smem + TILEW);  // [nq][2^S1][Cb] step-1 twiddles
  uint32_t nxt[E];  // IMG: residues of the image; real mode: raw digits (lifted at use)
  auto fetch = [&](int s, int q) {
    if constexpr (IMG) {  // image a of slice s from both parts' digits (f2; P.image)
      const uint2 io = P.io[q][a];
      const uint32_t p = q ? P.p[1] : P.p[0];
      const int32_t* Dr = P.digits + ((b * 2 + 0) * P.K + s) * P.in_len + col;
      const int32_t* Di = P.digits + ((b * 2 + 1) * P.K + s) * P.in_len + col;
#pragma unroll
      for (int i = 0; i < CNT; ++i) {
        const uint32_t e = round_elem<LOGR, false, 0, LOGE>(tv, i);
        nxt[i] = e * C < lim ? digit_image(__ldg(&Dr[e * C]), __ldg(&Di[e * C]), io, p) : 0u;
      }
    } else {
      const int32_t* D = P.digits + ((b * 2 + a) * P.K + s) * P.in_len + col;
#pragma unroll
      for (int i = 0; i < CNT; ++i) {
        const uint32_t e = round_elem<LOGR, false, 0, LOGE>(tv, i);
        nxt[i] = e * C < lim ? (uint32_t)__ldg(&D[e * C]) : 0u;
      }
    }
  };
  fetch(0, q0);  // in flight while the twiddles are staged
  for (int k = 0; k < nq; ++k)
    stage_col_tw0<S1, Cb>(tw0 + k * (Cb << S1), P.tw + (size_t)((q0 + k) * 2 + 0) * m, C, cb << LOGCB);
  __syncthreads();
  const int nit = nq * ka;
  for (int it = 0; it < nit; ++it) {
    const int k = it >= ka ? 1 : 0, s = it - k * ka, q = q0 + k;
    const uint32_t p = q ? P.p[1] : P.p[0];
    const uint2* T = P.tw + (size_t)(q * 2 + 0) * m;
    uint32_t cur[E];
#pragma unroll
    for (int i = 0; i < E; ++i) cur[i] = IMG ? nxt[i] : lift((int32_t)nxt[i], p);
    if (it + 1 < nit) fetch(it + 1 >= ka ? it + 1 - ka : it + 1, it + 1 >= ka ? q0 + 1 : q0);
    if (it > 0) __syncthreads();  // smem tile free
    uint32_t* out = P.Y + (((b * 2 + q) * 2 + a) * P.K + s) * (int64_t)m + col;
    sub_ntt_t0<LOGR, false, Cb, LOGE, ZHI>(
        tv, smem + c, col, C, T, Tw0{tw0 + k * (Cb << S1), (uint32_t)c, (uint32_t)Cb}, p,
        [&](int i, uint32_t) -> uint32_t { return cur[i]; },
        [&](int, uint32_t e, uint32_t val) { out[e * C] = val; });
  }
}

// Inverse column pass: global DIT stages len = 2C .. m; writes rows i < n only.
// One CTA per (transform, prime, conv, column block) loops over the conv's Alg.8 groups
// with the next group's tile prefetched.
template <int LOGR, int LOGC>
__global__ void __launch_bounds__(256) k_col_inv(ColParams P) {
  extern __shared__ uint32_t smem[];
  constexpr int LOGCB = col_log_cb(LOGR, LOGC);
  constexpr int LOGE = col_loge(LOGR);
  constexpr int E = 1 << LOGE;
  constexpr int Cb = 1 << LOGCB;
  constexpr uint32_t C = 1u << LOGC;
  constexpr uint32_t m = 1u << (LOGR + LOGC);
  constexpr uint32_t ncb = 1u << (LOGC - LOGCB);
  constexpr int CNT = RoundT<LOGR, true, 0, LOGE>::cnt;
  const int G = P.K * P.K;
  const uint32_t cb = blockIdx.x % ncb;
  uint32_t v = blockIdx.x / ncb;  // (b * 2 + q) * 4 + cv
  const int cv = (int)(v & 3); v >>= 2;
  const int q = (int)(v & 1); v >>= 1;
  const int64_t b = v;
  if (!(P.unit_mask & (1u << (cv * 2 + q)))) return;
  const int ng = P.sched[(b * 4 + cv) * sched_stride(P.K, P.L)];
  if (ng == 0) return;
  const int c = threadIdx.x & (Cb - 1);
  const int tv = threadIdx.x >> LOGCB;
  const uint32_t p = q ? P.p[1] : P.p[0];
  const uint32_t col = (cb << LOGCB) + c;
  const uint2* T = P.tw + (size_t)(q * 2 + 1) * m;
  const uint32_t lim = P.n > col ? (uint32_t)(P.n - col) : 0u;
  uint32_t nxt[E];
  auto fetch = [&](int g) {
    const uint32_t* in = P.G + (((b * 2 + q) * 4 + cv) * G + g) * (int64_t)m + col;
#pragma unroll
    for (int i = 0; i < CNT; ++i) nxt[i] = __ldcs(&in[round_elem<LOGR, true, 0, LOGE>(tv, i) * C]);
  };
  fetch(0);
  for (int g = 0; g < ng; ++g) {
    uint32_t cur[E];
#pragma unroll
    for (int i = 0; i < E; ++i) cur[i] = nxt[i];
    if (g + 1 < ng) fetch(g + 1);
    if (g > 0) __syncthreads();  // smem tile free
    const int64_t ooff = (((b * 4 + cv) * 2 + q) * P.rg + g) * P.n + col;
    uint32_t* out = P.res + ooff;
    sub_ntt<LOGR, true, Cb, LOGE>(
        tv, smem + c, col, C, T, p, [&](int i, uint32_t) -> uint32_t { return cur[i]; },
        [&](int, uint32_t e, uint32_t val) {
          if (e * C < lim) {
            out[e * C] = val;
            // peer-memory exchange: the same residue into every other rank's buffer
            for (int r = 0; r < P.npeers; ++r)
              if (P.res_peers[r] != P.res) P.res_peers[r][ooff + (int64_t)e * C] = val;
          }
        });
  }
  // peer stores visible system-wide before anything this rank signals afterwards (the
  // barrier / collective the caller orders after the kernel)
  if (P.npeers > 0) __threadfence_system();
}

// ============================================================== fused row kernel
struct RowParams {
  int logm, logC, logR;
  int64_t nb;
  int K, L;
  uint32_t p[2];
  const uint2* tw;        // [2 prime][2 dir][m]
  const int32_t* digits;  // R == 1: [nb][2][K][in_len]
  int64_t in_len;
  const uint32_t* Y;      // R > 1: [nb][2][2][K][m]
  const uint32_t* W;      // [2 q][2 b][K][m] Montgomery form W m^{-1} 2^32 mod p (row_perm)
  uint32_t pinv[2];       // -p^{-1} mod 2^32 (Montgomery)
  uint32_t* G;            // R > 1: [nb][2 q][4][K*K][m]
  uint32_t* res;          // R == 1: [nb][4][2][rg][n]
  int rg;                 // group stride of res
  int64_t n;
  const int32_t* stats;
  const int32_t* sched;
  uint32_t unit_mask;
  uint32_t* res_peers[8];  // as ColParams (one-pass plans write residues in the row kernel)
  int npeers;
  int fwd_only;           // 1: write the forward spectra (internal order) to Xout, stop
  uint32_t* Xout;         // fwd_only or tap: [nb][2 q][2 a][K][m]
  uint32_t* Zout;         // tap: [nb][2 q][4][K*K][m] (internal order, W m^{-1} scaled)
  int image;              // f2: a = image index; one "conv" (the image) per CTA, schedule
                          // row 0, W rows of image a; digits imaged on load (R == 1)
  uint2 io[2][2];         // [q][image] Shoup pair of iota_q / p_q - iota_q
};

#ifndef OZ_ROW_LAZYG
#define OZ_ROW_LAZYG 0  // two-pass rows of odd index store G lazily (< 2p), see k_row_fused; off:
                        // the second inverse instance costs more (c3 row 1102 vs 1026 us) than it saves
#endif
#ifndef OZ_ROW_QMAJOR
#define OZ_ROW_QMAJOR 1
#endif
#ifndef OZ_ROW_NA
#define OZ_ROW_NA 1
#endif
#ifndef OZ_ROW_FWD3
#define OZ_ROW_FWD3 1  // two-pass rows with three slices: the forward NTTs as one NV = 3 pass
#endif
#ifndef OZ_ROW_BULKY
#define OZ_ROW_BULKY 1  // two-pass rows: Y rows bulk-copied (TMA) into shared memory up front
#endif
// streaming read-only load that does not allocate in L1 (keeps the twiddle tables there)
__device__ __forceinline__ uint32_t ldg_stream(const uint32_t* p) {
#if OZ_ROW_NA
  uint32_t v;
  asm("ld.global.nc.L1::no_allocate.u32 %0, [%1];" : "=r"(v) : "l"(p));
  return v;
#else
  return __ldg(p);
#endif
}
template <int LOGC, bool TWO_PASS>
struct RowCfg {
  static constexpr int LOGE = row_loge(LOGC, TWO_PASS);
  static constexpr int E = 1 << LOGE;
  static constexpr int threads = LOGC >= LOGE ? (1 << (LOGC - LOGE)) : 1;
#ifndef OZ_ROW_MINB
#define OZ_ROW_MINB 6  // 80 registers, 6 CTAs/SM (with the 16-byte W/X quads: c3 1031 vs 1037 us at 96 / 5)
#endif
  static constexpr int min_blocks = LOGC == 11 ? OZ_ROW_MINB : (LOGC == 10 && TWO_PASS ? 12 : 1);
  // stages of the first DIT round (= last DIF round): its groups are contiguous blocks
  static constexpr int S0 = LOGC >= LOGE ? LOGE : LOGC;
};

// Row-local storage order used for the X rows in shared memory and for the cached W
// spectra.  In the first DIT round thread t holds the 2^S0 contiguous elements
// e = t 2^S0 + i (internal bit-reversed order).  OZ_ROW_VEC: element e lives at
// (i / 4) (C 4 / 2^S0) + 4 t + (i mod 4), so a thread's registers 4k .. 4k+3 are one 16-byte
// word and a warp's 16-byte loads / stores of quad k cover 512 contiguous bytes (coalesced
// LDG.128, conflict-free LDS/STS.128: a quarter of the W / X load instructions of the
// pointwise stage).  Without it: (e mod 2^S0) (C / 2^S0) + e / 2^S0 (32-bit words, a warp
// touches consecutive words per register).
#ifndef OZ_ROW_VEC
#define OZ_ROW_VEC 1
#endif
__host__ __device__ __forceinline__ uint32_t row_perm_lin(uint32_t e, int logC, int S0) {
  return ((e & ((1u << S0) - 1)) << (logC - S0)) + (e >> S0);
}
__host__ __device__ __forceinline__ uint32_t row_perm(uint32_t e, int logC, int S0) {
#if OZ_ROW_VEC
  if (S0 >= 2) {
    const uint32_t i = e & ((1u << S0) - 1), t = e >> S0;
    return ((i >> 2) << (logC - S0 + 2)) + (t << 2) + (i & 3);
  }
#endif
  return row_perm_lin(e, logC, S0);
}

// row_perm of the element held in register i (< 2^S0) by thread tv in the first DIT round
// (element tv 2^S0 + i): a compile-time offset plus a function of tv.
template <int LOGC, bool TWO_PASS>
__device__ __forceinline__ uint32_t row_slot(int tv, int i) {
  constexpr int S0 = RowCfg<LOGC, TWO_PASS>::S0;
  constexpr int Tv = RowCfg<LOGC, TWO_PASS>::threads;
#if OZ_ROW_VEC
  if constexpr (S0 >= 2)
    return ((uint32_t)(i >> 2) << (LOGC - S0 + 2)) + ((uint32_t)tv << 2) + (uint32_t)(i & 3);
#endif
  return (uint32_t)tv + ((uint32_t)(i & ((1 << S0) - 1)) << (LOGC - S0)) + (uint32_t)(i >> S0) * Tv;
}
// 16-byte quads of row_slot: registers 4k .. 4k+3 of thread tv start at row_quad(tv, k)
template <int LOGC, bool TWO_PASS>
__device__ __forceinline__ uint32_t row_quad(int tv, int k) {
  constexpr int S0 = RowCfg<LOGC, TWO_PASS>::S0;
  return ((uint32_t)k << (LOGC - S0 + 2)) + ((uint32_t)tv << 2);
}
template <int LOGC, bool TWO_PASS>
__host__ __device__ constexpr bool row_vec() {
  return OZ_ROW_VEC && RowCfg<LOGC, TWO_PASS>::S0 >= 2;
}
__device__ __forceinline__ uint4 ldg_stream4(const uint32_t* p) {
  uint4 v;
  asm("ld.global.nc.L1::no_allocate.v4.u32 {%0, %1, %2, %3}, [%4];"
      : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w)
      : "l"(p));
  return v;
}

template <int LOGC, bool TWO_PASS>
__global__ void __launch_bounds__(RowCfg<LOGC, TWO_PASS>::threads, RowCfg<LOGC, TWO_PASS>::min_blocks)
    k_row_fused(RowParams P) {
  extern __shared__ uint32_t smem[];
  __shared__ int s_ng[2];
  const int64_t b = blockIdx.x;
  const int a = blockIdx.y & 1;
#if OZ_ROW_QMAJOR
  // prime-major CTA order: the CTAs resident at any time mostly share one prime, so the
  // L1 holds one prime's twiddle tables
  const uint32_t row = (blockIdx.y >> 1) & ((1u << P.logR) - 1);
  const int q = (int)(blockIdx.y >> (P.logR + 1));
#else
  const int q = (blockIdx.y >> 1) & 1;
  const uint32_t row = blockIdx.y >> 2;
#endif
  constexpr int logC = LOGC;
  constexpr uint32_t C = 1u << logC;
  constexpr int LOGE = RowCfg<LOGC, TWO_PASS>::LOGE;
  constexpr int E = 1 << LOGE;
  constexpr uint32_t padC = C + (C >> LOGE) + 1;
  const int tv = threadIdx.x;
  const int64_t m = 1ll << P.logm;
  const uint32_t p = q ? P.p[1] : P.p[0];
  const int K = P.K, L = P.L, G = K * K;
  const int32_t* st = P.stats + b * stats_stride(K);
  const int ka = st[a];
  // convolutions using part a: a = 0 -> rr (0), ri (3); a = 1 -> ii (1), ir (2)
  // (image mode: the CTA's one "conv" is its image a)
  const int cv0 = P.image ? a : (a == 0 ? 0 : 1), cv1 = a == 0 ? 3 : 2;
  const bool want0 = P.image || ((P.unit_mask >> (cv0 * 2 + q)) & 1u);
  const bool want1 = !P.image && ((P.unit_mask >> (cv1 * 2 + q)) & 1u);
  if (!P.fwd_only && !want0 && !want1) return;
  if (ka == 0 && !P.fwd_only) return;  // no slices: the schedule has no groups here
  // [K][XS] forward spectra rows (row_perm order); two-pass rows are XS = C + C/16 + 4 words
  // apart (the padded exchange layout of the three-slice forward fits in place, 16B-aligned)
  constexpr uint32_t XS = TWO_PASS ? C + (C >> LOGE) + 4 : C;
  uint32_t* Xs = smem;
  // [padC]: inter-round exchange buffer; a CTA barrier before each sub-transform frees it
  // (double buffering, which would drop that barrier, measured slower: more registers)
  uint32_t* work = smem + K * XS;
  // group table for 2 convs x K*K groups: npairs, then (X row offset, W row offset) x L
  uint32_t* tab = work + padC;
  const int tstride = 1 + 2 * L;
  const uint2* Tf = P.tw + (size_t)(q * 2 + 0) * m;
  const uint2* Ti = P.tw + (size_t)(q * 2 + 1) * m;
  const uint32_t rowoff = row << logC;
#if OZ_ROW_BULKY
  // two-pass plans: the ka rows of Y this CTA transforms are bulk-copied into the X area at
  // the start (one mbarrier per slice), so their HBM latency is paid once, overlapped with
  // the earlier slices' NTTs, instead of once per slice behind the sub-transform barriers.
  // Slice s's first round reads Y[s] from there; its last round overwrites it with X[s]
  // (every read of Y[s] precedes the round-0 exchange barrier).
  __shared__ __align__(8) unsigned long long s_ybar[kMaxK];
  if constexpr (TWO_PASS) {
    if (threadIdx.x == 0) {
      for (int s = 0; s < ka; ++s) mbar_init(&s_ybar[s], 1);
      mbar_fence_init();
      for (int s = 0; s < ka; ++s) {
        mbar_expect_tx(&s_ybar[s], C * 4u);
        bulk_g2s(Xs + s * XS, P.Y + (((b * 2 + q) * 2 + a) * K + s) * m + rowoff, C * 4u, &s_ybar[s]);
      }
    }
  }
#endif
  // one (conv, group) entry per thread, every schedule load independent of the others (the
  // whole table costs one L2 latency; a serial walk over the groups cost ~10 dependent ones)
  for (int it = tv; it < 2 * G && !P.fwd_only; it += blockDim.x) {  // blockDim may be 1 (C < 32)
    const int ci = it / G, g = it - (it / G) * G;
    const int cv = ci ? cv1 : cv0;
    const bool want = ci ? want1 : want0;
    const int32_t* srow = P.sched + (b * 4 + (P.image ? 0 : cv)) * sched_stride(K, L);
    const int32_t* grp = srow + 1 + g * (2 + 2 * L);
    const int ng = want ? __ldg(&srow[0]) : 0;
    const int np = __ldg(&grp[1]);
    uint32_t* tg = tab + (ci * G + g) * tstride;
    for (int i = 0; i < L; ++i) {
      const uint32_t sx = (uint32_t)__ldg(&grp[2 + 2 * i]), tw = (uint32_t)__ldg(&grp[3 + 2 * i]);
      if (g < ng && i < np) {
        tg[1 + 2 * i] = sx * XS;
        tg[2 + 2 * i] = tw * (uint32_t)m;  // W row offset
      }
    }
    if (g < ng) tg[0] = (uint32_t)np;
    if (g == 0) s_ng[ci] = ng;
  }
  if constexpr (TWO_PASS && OZ_ROW_BULKY) __syncthreads();  // mbarriers initialised
  // ---- forward: last log2(C) DIF stages of each slice's NTT (Alg.6 l.787)
  int s_begin = 0;
#if OZ_ROW_FWD3
  if constexpr (TWO_PASS && OZ_ROW_BULKY) {
    if (ka == 3) {
      // The three slices together (sub_ntt_multi, NV = 3): one twiddle load per butterfly
      // position serves the three vectors, three independent butterflies per position, and
      // the whole forward takes three CTA barriers instead of six.  The exchange runs in
      // place in each slice's own XS-word row (padded layout): Y[s] is read into registers
      // first (barrier), and X[s] is written in row_perm order after the last round's reads
      // (barrier).
      constexpr int CNT0 = RoundT<LOGC, false, 0, LOGE>::cnt;
      uint32_t yv[3][E];
#pragma unroll
      for (int v = 0; v < 3; ++v) {
        mbar_wait(&s_ybar[v], 0u);
#pragma unroll
        for (int i = 0; i < CNT0; ++i) yv[v][i] = Xs[v * XS + round_elem<LOGC, false, 0, LOGE>(tv, i)];
      }
      __syncthreads();  // every Y read done before the in-place exchange writes
      uint32_t* const sms[3] = {Xs, Xs + XS, Xs + 2 * XS};
      uint32_t* const outX = P.Xout && blockIdx.z == 0 ? P.Xout + (((b * 2 + q) * 2 + a) * K) * m + rowoff
                                                      : nullptr;  // tap / plan-time spectra
      uint32_t xv[3][E];
      sub_ntt_multi<LOGC, false, 1, 3, LOGE, true, false>(
          tv, sms, 0u, 1u, Tf, Tw0{nullptr, 0u, 0u}, p,
          [&](int v, int i, uint32_t) -> uint32_t { return yv[v][i]; },
          [&](int v, int i, uint32_t e, uint32_t val) {
            xv[v][i] = val;
            if (outX) outX[(size_t)v * m + e] = val;
          });
      __syncthreads();  // every last-round read done before X overwrites the rows
#pragma unroll
      for (int v = 0; v < 3; ++v) {
        if constexpr (row_vec<LOGC, TWO_PASS>()) {
#pragma unroll
          for (int k = 0; k < CNT0 / 4; ++k)
            *reinterpret_cast<uint4*>(Xs + v * XS + row_quad<LOGC, TWO_PASS>(tv, k)) =
                make_uint4(xv[v][4 * k], xv[v][4 * k + 1], xv[v][4 * k + 2], xv[v][4 * k + 3]);
        } else {
#pragma unroll
          for (int i = 0; i < CNT0; ++i) Xs[v * XS + row_slot<LOGC, TWO_PASS>(tv, i)] = xv[v][i];
        }
      }
      s_begin = 3;
    }
  }
#endif
  for (int s = s_begin; s < ka; ++s) {
    uint32_t* xs = Xs + s * XS;
    uint32_t* outX = P.Xout && blockIdx.z == 0 ? P.Xout + (((b * 2 + q) * 2 + a) * K + s) * m + rowoff
                                              : nullptr;
    uint32_t* wk = work;
    if (s > s_begin) __syncthreads();  // `work` free (previous last reads done)
    auto store_x = [&](int i, uint32_t e, uint32_t v) {
      xs[row_slot<LOGC, TWO_PASS>(tv, i)] = v;  // == row_perm(e)
      if (outX) outX[e] = v;
    };
    if constexpr (TWO_PASS) {
#if OZ_ROW_BULKY
      mbar_wait(&s_ybar[s], 0u);  // Y[s] landed in xs
      sub_ntt<LOGC, false, 1, LOGE, true>(tv, wk, 0u, 1u, Tf, p,
                           [&](int, uint32_t e) -> uint32_t { return xs[e]; }, store_x);
#else
      const uint32_t* y = P.Y + (((b * 2 + q) * 2 + a) * K + s) * m + rowoff;
      sub_ntt<LOGC, false, 1, LOGE, true>(tv, wk, 0u, 1u, Tf, p,
                           [&](int, uint32_t e) -> uint32_t { return ldg_stream(&y[e]); }, store_x);
#endif
    } else {
      const int32_t* D = P.digits + ((b * 2 + a) * K + s) * P.in_len;
      const uint32_t in_len = (uint32_t)P.in_len;
      if (P.image) {  // digit image a of slice s (f2)
        const int32_t* Dr = P.digits + ((b * 2 + 0) * K + s) * P.in_len;
        const int32_t* Di = P.digits + ((b * 2 + 1) * K + s) * P.in_len;
        const uint2 io = P.io[q][a];
        sub_ntt<LOGC, false, 1, LOGE, true>(
            tv, wk, 0u, 1u, Tf, p,
            [&](int, uint32_t e) -> uint32_t {
              return e < in_len ? digit_image(__ldg(&Dr[e]), __ldg(&Di[e]), io, p) : 0u;
            },
            store_x);
      } else {
        sub_ntt<LOGC, false, 1, LOGE, true>(
            tv, wk, 0u, 1u, Tf, p,
            [&](int, uint32_t e) -> uint32_t { return e < in_len ? lift(__ldg(&D[e]), p) : 0u; },
            store_x);
      }
    }
  }
  if (P.fwd_only) return;
  // ---- per group: Z = sum X_s (.) W_t (Alg.8 l.981-982), then the first log2(C) DIT
  // stages of its inverse NTT (l.973).  The (conv, group) items of both convolutions are
  // processed two at a time: their twiddles are shared and one barrier serves both.
  constexpr int CNT = RoundT<LOGC, true, 0, LOGE>::cnt;
  const uint32_t pinv = 0u - (q ? P.pinv[1] : P.pinv[0]);  // +p^{-1} mod 2^32 (redc_lazy3)
  __syncthreads();  // group table visible
  const int ng0 = s_ng[0], nitems = s_ng[0] + s_ng[1];
  auto item = [&](int it, int& ci, int& g) {
    ci = it < ng0 ? 0 : 1;
    g = it < ng0 ? it : it - ng0;
  };
  // pointwise products for this thread's round-0 elements: 64-bit lazy sums of up to 3
  // products X * W~ (W~ = W m^{-1} 2^32, sums < 3 p^2 < 2^64), one Montgomery reduction each
  auto wld = [&](const uint32_t* w) -> uint32_t { return ldg_stream(w); };
  // this thread's CNT words of a W row / an X row (16-byte quads with OZ_ROW_VEC)
  auto ld_wrow = [&](const uint32_t* wr, uint32_t (&w)[E]) {
    if constexpr (row_vec<LOGC, TWO_PASS>()) {
#pragma unroll
      for (int k = 0; k < CNT / 4; ++k) {
        const uint4 v = ldg_stream4(wr + row_quad<LOGC, TWO_PASS>(tv, k));
        w[4 * k] = v.x; w[4 * k + 1] = v.y; w[4 * k + 2] = v.z; w[4 * k + 3] = v.w;
      }
    } else {
#pragma unroll
      for (int i = 0; i < CNT; ++i) w[i] = wld(&wr[row_slot<LOGC, TWO_PASS>(tv, i)]);
    }
  };
  auto ld_xrow = [&](const uint32_t* xr, uint32_t (&x)[E]) {
    if constexpr (row_vec<LOGC, TWO_PASS>()) {
#pragma unroll
      for (int k = 0; k < CNT / 4; ++k) {
        const uint4 v = *reinterpret_cast<const uint4*>(xr + row_quad<LOGC, TWO_PASS>(tv, k));
        x[4 * k] = v.x; x[4 * k + 1] = v.y; x[4 * k + 2] = v.z; x[4 * k + 3] = v.w;
      }
    } else {
#pragma unroll
      for (int i = 0; i < CNT; ++i) x[i] = xr[row_slot<LOGC, TWO_PASS>(tv, i)];
    }
  };
  auto load_w0 = [&](int ci, int g, uint32_t (&w)[E]) {  // W row of an item's first pair
    const int cv = ci ? cv1 : cv0;
    const uint32_t* wr0 = P.W + (size_t)(q * 2 + (P.image ? a : conv_b(cv))) * K * m + rowoff +
                          tab[(ci * G + g) * tstride + 2];
    ld_wrow(wr0, w);
  };
  auto pointwise = [&](int ci, int g, uint32_t (&z)[E]) {
    const int cv = ci ? cv1 : cv0;
    const uint32_t* Wb = P.W + (size_t)(q * 2 + (P.image ? a : conv_b(cv))) * K * m + rowoff;
    const uint32_t* tg = tab + (ci * G + g) * tstride;
    const int np = (int)tg[0];
    if (np <= 3) {  // (L <= 3 always): the W loads of two pairs in flight ahead of the
                    // products (one L2 latency per group instead of one per pair; loading the
                    // next item's W during this item's NTT measured slower -- registers)
      uint32_t w0[E], w1[E], xv[E];
      load_w0(ci, g, w0);
      if (np > 1) ld_wrow(Wb + tg[4], w1);
      unsigned long long T[E];
      ld_xrow(Xs + tg[1], xv);
#pragma unroll
      for (int i = 0; i < CNT; ++i) T[i] = (unsigned long long)xv[i] * w0[i];
      if (np > 2) ld_wrow(Wb + tg[6], w0);
      if (np > 1) {
        ld_xrow(Xs + tg[3], xv);
#pragma unroll
        for (int i = 0; i < CNT; ++i) T[i] += (unsigned long long)xv[i] * w1[i];
      }
      if (np > 2) {
        ld_xrow(Xs + tg[5], xv);
#pragma unroll
        for (int i = 0; i < CNT; ++i) T[i] += (unsigned long long)xv[i] * w0[i];
      }
      if (np == 3) {
#pragma unroll
        for (int i = 0; i < CNT; ++i) z[i] = redc_lazy3(T[i], p, pinv);
      } else {  // T < 2 p^2 < p 2^32: the high word is already below p
#pragma unroll
        for (int i = 0; i < CNT; ++i) z[i] = redc_lazy2(T[i], p, pinv);
      }
      return;
    }
#pragma unroll
    for (int i = 0; i < E; ++i) z[i] = 0;
    for (int ip0 = 0; ip0 < np; ip0 += 3) {
      unsigned long long T[E];
#pragma unroll
      for (int i = 0; i < E; ++i) T[i] = 0ull;
      const int ipe = min(np, ip0 + 3);
      for (int ip = ip0; ip < ipe; ++ip) {
        const uint32_t* xr = Xs + tg[1 + 2 * ip];
        const uint32_t* wr = Wb + tg[2 + 2 * ip];
#pragma unroll
        for (int i = 0; i < CNT; ++i) {
          const uint32_t pe = row_slot<LOGC, TWO_PASS>(tv, i);  // == row_perm(round-0 element)
          T[i] += (unsigned long long)xr[pe] * wld(&wr[pe]);
        }
      }
#pragma unroll
      for (int i = 0; i < CNT; ++i) {
        const uint32_t r = redc_lazy3(T[i], p, pinv);
        z[i] = ip0 == 0 ? r : add_mod(z[i], r, p);
      }
    }
  };
  auto out_ptr = [&](int ci, int g) -> uint32_t* {
    const int cv = ci ? cv1 : cv0;
    if constexpr (TWO_PASS) return P.G + (((b * 2 + q) * 4 + cv) * G + g) * m + rowoff;
    return P.res + (((b * 4 + cv) * 2 + q) * P.rg + g) * P.n;
  };
  auto ztap_ptr = [&](int ci, int g) -> uint32_t* {
    const int cv = ci ? cv1 : cv0;
    return P.Zout ? P.Zout + (((b * 2 + q) * 4 + cv) * G + g) * m + rowoff : nullptr;
  };
  const uint32_t nlim = TWO_PASS ? C : (uint32_t)P.n;
  // (processing two items at once with sub_ntt_multi<..., 2> shares twiddles and barriers
  // but measured slower on B200 -- fewer resident CTAs -- so items run one at a time)
  // Small one-pass plans spread the items over gridDim.z CTAs (each recomputes the few
  // forward spectra): latency, not throughput, bounds them.
  for (int it = blockIdx.z; it < nitems; it += gridDim.z) {
    uint32_t* wk = work;
    if (it >= (int)gridDim.z) __syncthreads();  // exchange buffer free
    int ci0, g0;
    item(it, ci0, g0);
    uint32_t z[E];
    pointwise(ci0, g0, z);
    uint32_t* const zt = ztap_ptr(ci0, g0);
    uint32_t* const op = out_ptr(ci0, g0);
    auto inverse = [&](auto lz) {
      sub_ntt<LOGC, true, 1, LOGE, true, false, decltype(lz)::value>(
          tv, wk, 0u, 1u, Ti, p,
          [&](int i, uint32_t e) -> uint32_t {
            if (zt) zt[e] = z[i];
            return z[i];
          },
          [&](int, uint32_t e, uint32_t val) {
            if (e < nlim) {
              op[e] = val;
              if constexpr (!TWO_PASS)  // peer-memory exchange (unit-sharded single transform)
                for (int r = 0; r < P.npeers; ++r)
                  if (P.res_peers[r] != P.res) P.res_peers[r][(op - P.res) + e] = val;
            }
          });
    };
    // Two-pass plans: G row `row` of an odd index is, in every column kernel, the v-operand of
    // the first DIT stage (rows 2i, 2i + 1), i.e. the input of a Shoup product, which accepts
    // any 32-bit value -- so odd rows leave the last stage's outputs lazy (< 2p).
    if (TWO_PASS && OZ_ROW_LAZYG && (row & 1u))
      inverse(std::integral_constant<bool, true>{});
    else
      inverse(std::integral_constant<bool, false>{});
  }
  if (!TWO_PASS && P.npeers > 0) __threadfence_system();  // as k_col_inv
}

// ============================================================== CRT + recombination
struct FinishParams {
  int64_t n, nb;
  int K, L;
  uint32_t p0, p1, p0inv, p0inv_sh;  // p0^{-1} mod p1 and its Shoup companion
  uint32_t p1_barrett;               // floor(2^32 / p1)
  unsigned long long P, halfP;       // p0 p1 and (p0 p1 - 1) / 2
  const uint32_t* res;      // [nb][4][2][rg][n]
  int rg;                   // group stride of res
  const int32_t* stats;
  const int32_t* sched;
  const double2* chirp;     // [n]
  double2* out;             // [nb][n]
  int direction;
  int64_t* crt_tap;         // [nb][4][K*K][n] or null
  // image mode (f2): per prime q the Shoup pairs of 2^-1 and (2 iota_q)^-1 mod p_q
  uint2 inv2[2], inv2i[2];
  int ts;                   // f4: TS accumulation (sums stored as float4 (x0, x1, x2, 0))
};

// f4: accumulate z 2^-cexp into a TS sum kept in a 16-byte slot (Alg.8 l.975-976 with TSAdd)
__device__ __forceinline__ double2 ts_accum(double2 slot, long long Z, int cexp) {
  const float4 a = *reinterpret_cast<const float4*>(&slot);
  const TSv r = ts_add(TSv{a.x, a.y, a.z}, ts_ldexp(ts_from_int64(Z), -cexp));
  const float4 o = make_float4(r.x0, r.x1, r.x2, 0.0f);
  return *reinterpret_cast<const double2*>(&o);
}
__device__ __forceinline__ TSv ts_of_slot(double2 slot) {
  const float4 a = *reinterpret_cast<const float4*>(&slot);
  return TSv{a.x, a.y, a.z};
}
// f4: y' = (rr - ii) + i (ir + ri), y = y' (.) omega in TS, fl64 (Alg.4 TS steps 4-5)
__device__ __forceinline__ double2 ts_finish(TSv rr, TSv ii, TSv ir, TSv ri, double2 w) {
  const TSv yr = ts_add(rr, ts_neg(ii)), yi = ts_add(ir, ri);
  const TSv c = ts_from_double(w.x), sn = ts_from_double(w.y);
  const TSv orr = ts_add(ts_mul(yr, c), ts_neg(ts_mul(yi, sn)));
  const TSv oii = ts_add(ts_mul(yr, sn), ts_mul(yi, c));
  return make_double2(ts_to_double(orr), ts_to_double(oii));
}

// f2: (re, im) residues of a complex integer from its two images z+ = re + iota im and
// z- = re - iota im (mod p): re = (z+ + z-)/2, im = (z+ - z-)/(2 iota).
__device__ __forceinline__ void image_pair(uint32_t zp, uint32_t zm, uint2 inv2, uint2 inv2i,
                                           uint32_t p, uint32_t& re, uint32_t& im) {
  re = mul_shoup(add_mod(zp, zm, p), inv2, p);
  im = mul_shoup(sub_mod(zp, zm, p), inv2i, p);
}

// Garner, two primes (Alg.8 l.974): Z' = z0 + p0 ((z1 - z0) p0^{-1} mod p1)
// in [0, p0 p1), then the symmetric representative in [-p0p1/2, p0p1/2) (
// it is unique, so this equals the symmetric-Garner form of the oracle).
__device__ __forceinline__ long long garner2(uint32_t z0, uint32_t z1, const FinishParams& P) {
  // z0 mod p1 for any prime pair: Barrett with c = floor(2^32 / p1) leaves r < 2 p1, one
  // conditional subtraction finishes (for the paper's primes c = 2 and z0 < 2^31, so q = 0)
  const uint32_t q0 = __umulhi(z0, P.p1_barrett);
  uint32_t z0r = z0 - q0 * P.p1;
  z0r = min(z0r, z0r - P.p1);
  const uint32_t d = sub_mod(z1, z0r, P.p1);
  const uint32_t t = mul_shoup(d, make_uint2(P.p0inv, P.p0inv_sh), P.p1);
  const unsigned long long Zp = (unsigned long long)z0 + (unsigned long long)P.p0 * t;
  return Zp > P.halfP ? (long long)(Zp - P.P) : (long long)Zp;
}

// y' = (S_rr - S_ii) + i (S_ir + S_ri) from the four convolutions' DD sums,
// post-chirp y = y' (.) omega (Alg.4 l.480-484), fp64; inverse direction: conj and RN
// division by n (O10).  One operation sequence for every kernel that finishes a transform.
__device__ __forceinline__ double2 dd_combine_postchirp(double2 rr, double2 ii, double2 ir, double2 ri,
                                                        double2 w, int direction, int64_t n) {
  double yrh, yrl, yih, yil;
  dd_add(rr.x, rr.y, -ii.x, -ii.y, yrh, yrl);  // rr - ii
  dd_add(ir.x, ir.y, ri.x, ri.y, yih, yil);    // ir + ri
  double a1h, a1l, a2h, a2l, ore, oim, tmp;
  dd_mul_d(yrh, yrl, w.x, a1h, a1l);
  dd_mul_d(yih, yil, w.y, a2h, a2l);
  dd_add(a1h, a1l, -a2h, -a2l, ore, tmp);
  dd_mul_d(yrh, yrl, w.y, a1h, a1l);
  dd_mul_d(yih, yil, w.x, a2h, a2l);
  dd_add(a1h, a1l, a2h, a2l, oim, tmp);
  if (direction > 0) {
    const double dn = (double)n;
    ore = __ddiv_rn(ore, dn);
    oim = __ddiv_rn(-oim, dn);
  }
  return make_double2(ore, oim);
}

// CTA = 64 outputs x 4 real convolutions: thread (cv, jl) forms conv cv's DD sum of
// output j (Garner + scaled sum in flush order), then the cv = 0 threads combine the four
// sums and post-chirp.  (The four per-conv chains are independent: one thread per conv
// quarters the dependent-latency chain of the small one-pass plans this kernel serves.)
constexpr int kFinishCols = 64;
__global__ void __launch_bounds__(256, 4) k_crt_finish(FinishParams P) {
  const int64_t b = blockIdx.y;
  const int K = P.K, L = P.L, G = K * K;
  // per-transform schedule: group counts and exact scales 2^-cexp (l.975), in smem
  __shared__ int s_ng[4];
  __shared__ double s_sc[4][kMaxK * kMaxK];
  __shared__ double2 s_S[4][kFinishCols];
  if (threadIdx.x < 4) {
    const int cv = threadIdx.x;
    const int32_t* srow = P.sched + (b * 4 + cv) * sched_stride(K, L);
    const int ng = srow[0];
    s_ng[cv] = ng;
    for (int g = 0; g < ng; ++g) s_sc[cv][g] = scalbn(1.0, -srow[1 + g * (2 + 2 * L)]);
  }
  __syncthreads();
  const int cvt = threadIdx.x / kFinishCols, jl = threadIdx.x % kFinishCols;
  const int64_t j = (int64_t)blockIdx.x * kFinishCols + jl;
  const int32_t* st = P.stats + b * stats_stride(K);
  const bool bad = st[2 + 2 * K] & 1;
  if (j < P.n && !bad) {
    const int cv = cvt;
    double sh = 0.0, sl = 0.0;
    const int ng = s_ng[cv];
    const uint32_t* r0 = P.res + (((b * 4 + cv) * 2 + 0) * P.rg) * P.n + j;
    const uint32_t* r1 = P.res + (((b * 4 + cv) * 2 + 1) * P.rg) * P.n + j;
    for (int g0 = 0; g0 < ng; g0 += 9) {
      // issue every residue load of up to 9 groups before the dependent DD chain
      uint32_t z0[9], z1[9];
#pragma unroll
      for (int i = 0; i < 9; ++i) {
        if (g0 + i < ng) {
          z0[i] = __ldcs(&r0[(int64_t)(g0 + i) * P.n]);
          z1[i] = __ldcs(&r1[(int64_t)(g0 + i) * P.n]);
        }
      }
#pragma unroll
      for (int i = 0; i < 9; ++i) {
        if (g0 + i < ng) {
          const int g = g0 + i;
          const long long Z = garner2(z0[i], z1[i], P);
          if (P.crt_tap) P.crt_tap[((b * 4 + cv) * G + g) * P.n + j] = Z;
          double hs, ls;
          scaled_split(Z, s_sc[cv][g], hs, ls);  // z' / c, c an exact power of two (l.975)
          dd_add(sh, sl, hs, ls, sh, sl);          // flush order (l.976)
        }
      }
    }
    s_S[cv][jl] = make_double2(sh, sl);
  }
  __syncthreads();
  if (cvt != 0 || j >= P.n) return;
  double2 o;
  if (bad) {
    o.x = __longlong_as_double(0x7FF8000000000000ll);
    o.y = o.x;
    P.out[b * P.n + j] = o;
    return;
  }
  P.out[b * P.n + j] = dd_combine_postchirp(s_S[0][jl], s_S[1][jl], s_S[2][jl], s_S[3][jl], P.chirp[j],
                                            P.direction, P.n);
}

// f4, single-pass plans: Garner per group, z 2^-cexp accumulated with TSAdd in flush order
// per real conv, TS combine + post-chirp, fl64 (as k_crt_finish, in TS).
__global__ void __launch_bounds__(256, 4) k_crt_finish_ts(FinishParams P) {
  const int64_t b = blockIdx.y;
  const int K = P.K, L = P.L, G = K * K;
  __shared__ int s_ng[4];
  __shared__ int s_ce[4][kMaxK * kMaxK];
  if (threadIdx.x < 4) {
    const int cv = threadIdx.x;
    const int32_t* srow = P.sched + (b * 4 + cv) * sched_stride(K, L);
    const int ng = srow[0];
    s_ng[cv] = ng;
    for (int g = 0; g < ng; ++g) s_ce[cv][g] = srow[1 + g * (2 + 2 * L)];
  }
  __syncthreads();
  const int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (j >= P.n) return;
  double2 o;
  if (P.stats[b * stats_stride(K) + 2 + 2 * K] & 1) {
    o.x = __longlong_as_double(0x7FF8000000000000ll);
    o.y = o.x;
    P.out[b * P.n + j] = o;
    return;
  }
  TSv S[4];
#pragma unroll
  for (int cv = 0; cv < 4; ++cv) {
    TSv acc{0.0f, 0.0f, 0.0f};
    const uint32_t* r0 = P.res + (((b * 4 + cv) * 2 + 0) * P.rg) * P.n + j;
    const uint32_t* r1 = P.res + (((b * 4 + cv) * 2 + 1) * P.rg) * P.n + j;
    for (int g = 0; g < s_ng[cv]; ++g) {
      const long long Z = garner2(__ldcs(&r0[(int64_t)g * P.n]), __ldcs(&r1[(int64_t)g * P.n]), P);
      if (P.crt_tap) P.crt_tap[((b * 4 + cv) * G + g) * P.n + j] = Z;
      acc = ts_add(acc, ts_ldexp(ts_from_int64(Z), -s_ce[cv][g]));
    }
    S[cv] = acc;
  }
  o = ts_finish(S[0], S[1], S[2], S[3], P.chirp[j]);
  if (P.direction > 0) {
    const double dn = (double)P.n;
    o.x = __ddiv_rn(o.x, dn);
    o.y = __ddiv_rn(-o.y, dn);
  }
  P.out[b * P.n + j] = o;
}

// f2, single-pass plans: the residues of both images of each group -> (re, im) per prime
// -> Garner -> DD sums in flush order -> post-chirp (as k_crt_finish; res [nb][img][q][g][n]).
__global__ void __launch_bounds__(256, 4) k_crt_finish_img(FinishParams P) {
  const int64_t b = blockIdx.y;
  const int K = P.K, L = P.L, G = K * K;
  __shared__ int s_ng;
  __shared__ double s_sc[kMaxK * kMaxK];
  if (threadIdx.x == 0) {
    const int32_t* srow = P.sched + (b * 4) * sched_stride(K, L);  // the complex schedule
    s_ng = srow[0];
    for (int g = 0; g < s_ng; ++g) s_sc[g] = scalbn(1.0, -srow[1 + g * (2 + 2 * L)]);
  }
  __syncthreads();
  const int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (j >= P.n) return;
  double2 o;
  if (P.stats[b * stats_stride(K) + 2 + 2 * K] & 1) {
    o.x = __longlong_as_double(0x7FF8000000000000ll);
    o.y = o.x;
    P.out[b * P.n + j] = o;
    return;
  }
  double sh[2] = {0.0, 0.0}, sl[2] = {0.0, 0.0};
  const int ng = s_ng;
  for (int g = 0; g < ng; ++g) {
    uint32_t zr[2], zi[2];
#pragma unroll
    for (int q = 0; q < 2; ++q) {
      const uint32_t p = q ? P.p1 : P.p0;
      const uint32_t zp = __ldcs(&P.res[(((b * 4 + 0) * 2 + q) * P.rg + g) * P.n + j]);
      const uint32_t zm = __ldcs(&P.res[(((b * 4 + 1) * 2 + q) * P.rg + g) * P.n + j]);
      image_pair(zp, zm, P.inv2[q], P.inv2i[q], p, zr[q], zi[q]);
    }
    const double sc = s_sc[g];
#pragma unroll
    for (int part = 0; part < 2; ++part) {
      const long long Z = part ? garner2(zi[0], zi[1], P) : garner2(zr[0], zr[1], P);
      if (P.crt_tap) P.crt_tap[((b * 4 + part) * G + g) * P.n + j] = Z;
      double hs, ls;
      scaled_split(Z, sc, hs, ls);
      dd_add(sh[part], sl[part], hs, ls, sh[part], sl[part]);
    }
  }
  const double2 w = P.chirp[j];
  double a1h, a1l, a2h, a2l, ore, oim, tmp;
  dd_mul_d(sh[0], sl[0], w.x, a1h, a1l);
  dd_mul_d(sh[1], sl[1], w.y, a2h, a2l);
  dd_add(a1h, a1l, -a2h, -a2l, ore, tmp);
  dd_mul_d(sh[0], sl[0], w.y, a1h, a1l);
  dd_mul_d(sh[1], sl[1], w.x, a2h, a2l);
  dd_add(a1h, a1l, a2h, a2l, oim, tmp);
  if (P.direction > 0) {
    const double dn = (double)P.n;
    ore = __ddiv_rn(ore, dn);
    oim = __ddiv_rn(-oim, dn);
  }
  o.x = ore;
  o.y = oim;
  P.out[b * P.n + j] = o;
}

// Garner + scaled DD sums in flush order from gathered residues (the unit-sharded single
// transform after its all-gather; one transform): CTA = (conv, 256 x kCrtDDPer outputs).
// A dependent DADD costs ~25 clocks on B200, so each thread keeps kCrtDDPer independent DD chains and
// the next group's residues in flight.  Same per-value sequence as k_col_inv_crt /
// k_crt_finish (Alg.8 l.974-976); k_finish_dd then combines the four sums and post-chirps.
#ifndef OZ_CRTDD_PER
#define OZ_CRTDD_PER 4
#endif
constexpr int kCrtDDPer = OZ_CRTDD_PER;  // outputs (independent DD chains) per thread
__global__ void __launch_bounds__(256) k_crt_dd(FinishParams P, double2* __restrict__ S) {
  const int cv = blockIdx.y;
  const int K = P.K, L = P.L;
  __shared__ double s_sc[kMaxK * kMaxK];
  const int32_t* srow = P.sched + cv * sched_stride(K, L);
  const int ng = srow[0];
  for (int g = threadIdx.x; g < ng; g += blockDim.x) s_sc[g] = pow2_exact(-srow[1 + g * (2 + 2 * L)]);
  __syncthreads();
  if (P.stats[2 + 2 * K] & 1) return;  // non-finite transform: k_finish_dd writes NaN
  const int64_t n = P.n;
  const int64_t j0 = (int64_t)blockIdx.x * 256 * kCrtDDPer + threadIdx.x;
  const uint32_t* r0 = P.res + (size_t)(cv * 2 + 0) * P.rg * n;
  const uint32_t* r1 = P.res + (size_t)(cv * 2 + 1) * P.rg * n;
  double h[kCrtDDPer], l[kCrtDDPer];
  uint32_t a0[kCrtDDPer], a1[kCrtDDPer];
#pragma unroll
  for (int u = 0; u < kCrtDDPer; ++u) {
    const int64_t j = j0 + u * 256;
    h[u] = 0.0;
    l[u] = 0.0;
    a0[u] = ng > 0 && j < n ? __ldcs(&r0[j]) : 0u;
    a1[u] = ng > 0 && j < n ? __ldcs(&r1[j]) : 0u;
  }
  for (int g = 0; g < ng; ++g) {
    uint32_t c0[kCrtDDPer], c1[kCrtDDPer];
#pragma unroll
    for (int u = 0; u < kCrtDDPer; ++u) {
      c0[u] = a0[u];
      c1[u] = a1[u];
    }
    if (g + 1 < ng) {
#pragma unroll
      for (int u = 0; u < kCrtDDPer; ++u) {
        const int64_t j = j0 + u * 256;
        a0[u] = j < n ? __ldcs(&r0[(int64_t)(g + 1) * n + j]) : 0u;
        a1[u] = j < n ? __ldcs(&r1[(int64_t)(g + 1) * n + j]) : 0u;
      }
    }
    const double sc = s_sc[g];
#pragma unroll
    for (int u = 0; u < kCrtDDPer; ++u) {
      const long long Z = garner2(c0[u], c1[u], P);
      double hs, ls;
      scaled_split(Z, sc, hs, ls);
      dd_add(h[u], l[u], hs, ls, h[u], l[u]);
    }
  }
#pragma unroll
  for (int u = 0; u < kCrtDDPer; ++u) {
    const int64_t j = j0 + u * 256;
    if (j < n) S[cv * n + j] = make_double2(h[u], l[u]);
  }
}

// ============================================================== one-launch small transform
// One-pass plans (R = 1, 2^8 <= m = C <= 2^12), default mode (DD, four real convolutions):
// the whole path of ONE transform -- split (a1, a2), the forward NTTs (a3), pointwise
// products + NTT-domain accumulation (a4), inverse NTTs (a5), Garner (a6) and the scaled DD
// sums + post-chirp (a7) -- in ONE launch.  One thread-block cluster of 4 Z CTAs per
// transform; CTA rank = (q * 2 + a) * Z + z owns prime q, x' part a and every Z-th
// (conv, group) item of the two convolutions that use part a (as the one-pass row kernel's
// gridDim.z split).  Every CTA splits the whole transform itself (n <= 2^11 elements: the
// K + 1 passes need a block reduction each, no cluster barrier), keeps its part's digits,
// the K forward spectra and its items' residues in shared memory; one cluster barrier
// publishes the residues and the Garner + DD sums read the partner prime's residues through
// distributed shared memory.  Every value goes through the operation sequence of the
// multi-kernel path (k_split_cluster, k_row_fused, k_crt_finish), so the output is bitwise
// that path's.  (a fused kernel for the latency-bound small sizes.)
// Latency notes (B200, tools/microbench_fp64.cu): a dependent DADD / DFMA costs ~25 clocks,
// so the split processes up to 4 elements per thread as interleaved chains, and the prime's
// twiddles and the part's W rows are bulk-copied (TMA) into shared memory at the start, where
// they land while the split runs.
struct SmallParams {
  const double2* x;      // [nb][n]
  const double2* chirp;  // [n]
  double2* out;          // [nb][n]
  int64_t n;
  int K, L, alpha, rho, conj, direction;
  uint32_t p[2], pinv[2];
  const uint2* tw;          // [2 prime][2 dir][m]
  const uint32_t* W;        // [2 q][2 b][K][m] Montgomery W m^{-1} 2^32, row_perm(., logC, w_s0)
  int w_s0;
  const int32_t* wsplit;    // kw[2], Ew[2][K]
  FinishParams F;           // Garner constants
  unsigned long long* mu;   // [nb][2][K]  (written by rank 0, as the split kernels leave them)
  int32_t* stats;           // [nb][stats_stride]
  int32_t* sched;           // [nb][4][sched_stride]
  int Z;                    // CTAs per (prime, part)
  int slots;                // residue slots per CTA (>= ceil(items / Z))
  int stage;                // twiddles + W rows staged in shared memory
  int fault;                // test-only residue corruption (as k_fault_inject)
};
constexpr int kSmallLogE = 3;  // 8 elements per thread and round
#ifndef OZ_SMALL_FWD3
#define OZ_SMALL_FWD3 1  // k_small_fused: the three forward spectra as one NV = 3 pass
#endif
#ifndef OZ_SMALL_EPT
#define OZ_SMALL_EPT 4
#endif
constexpr int kSmallEPT = OZ_SMALL_EPT;  // split: elements per thread interleaved
#ifndef OZ_SMALL_TIMING
#define OZ_SMALL_TIMING 0  // tools/: per-phase %globaltimer stamps of every CTA (debug builds)
#endif
#if OZ_SMALL_TIMING
__device__ unsigned long long g_small_t[64][16];
#define SMALL_STAMP(k)                                                               \
  do {                                                                               \
    if (threadIdx.x == 0 && blockIdx.y == 0) {                                       \
      unsigned long long t_;                                                         \
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_));                         \
      g_small_t[cl.block_rank()][k] = t_;                                            \
    }                                                                                \
  } while (0)
#else
#define SMALL_STAMP(k) \
  do {                 \
  } while (0)
#endif
__host__ __device__ constexpr int small_threads(int logC) { return 1 << (logC - kSmallLogE); }
// dynamic shared memory (32-bit words), in order:
//   head: sched [4][SS] | stats | wsplit | digits of part a [K][n]
//   stage (optional): twiddles of prime q [2 dir][m] uint2 | W rows of part a's convs [2 b][K][m]
//   union: x' of the split [4][n] doubles | (X spectra [K][m] | 3 exchange buffers | residues)
__host__ __device__ inline size_t small_head_words(int64_t n, int K, int L) {
  return ((4 * (size_t)sched_stride(K, L) + stats_stride(K) + 2 + 2 * K + (size_t)K * n) + 3) & ~(size_t)3;
}
__host__ __device__ inline size_t small_stage_words(int logC, int K) {
  const size_t m = (size_t)1 << logC;
  return 4 * m + 2 * (size_t)K * m;
}
__host__ __device__ inline size_t small_union_words(int logC, int64_t n, int K, int slots) {
  const size_t m = (size_t)1 << logC;
  const size_t ntt = (size_t)K * m + 3 * (m + (m >> kSmallLogE) + 4) + (size_t)slots * n;
  const size_t split = 8 * (size_t)n;  // four doubles per element
  return ntt > split ? ntt : split;
}

template <int LOGC, bool STAGE>
__global__ void __launch_bounds__(small_threads(LOGC)) k_small_fused(SmallParams P) {
  constexpr int NT = small_threads(LOGC);
  constexpr uint32_t m = 1u << LOGC;
  constexpr uint32_t padm = (m + (m >> kSmallLogE) + 4) & ~3u;
  extern __shared__ __align__(16) uint32_t smem[];
  __shared__ unsigned long long s_red[2][NT / 32];
  __shared__ unsigned long long s_mu[2 * kMaxK];
  __shared__ double s_sc[4][kMaxK * kMaxK];
  __shared__ double2 s_S[4][NT / 4];
  __shared__ __align__(8) unsigned long long s_bar;
  cg::cluster_group cl = cg::this_cluster();
  const int rank = (int)cl.block_rank();
  const int Z = P.Z;
  const int z = rank % Z, a = (rank / Z) & 1, q = rank / (2 * Z);
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int64_t b = blockIdx.y;
  const int K = P.K, L = P.L;
  const int nn = (int)P.n;
  const int SS = sched_stride(K, L);
  SMALL_STAMP(0);
  int32_t* s_sched = reinterpret_cast<int32_t*>(smem);  // [4][SS]
  int32_t* s_stats = s_sched + 4 * SS;
  int32_t* s_wsplit = s_stats + stats_stride(K);         // [2 + 2K]
  int32_t* dig = s_wsplit + 2 + 2 * K;                   // [K][n], part a
  uint32_t* after_head = smem + small_head_words(P.n, K, L);
  uint2* s_tw = reinterpret_cast<uint2*>(after_head);    // stage: [2 dir][m]
  uint32_t* s_W = after_head + 4 * m;                    // stage: [2 b][K][m]
  uint32_t* U = after_head + (STAGE ? small_stage_words(LOGC, K) : 0);
  double* xp = reinterpret_cast<double*>(U);              // split: h[2][n], l[2][n]
  uint32_t* X = U;                                        // [K][m], row_perm_lin(., LOGC, 3)
  uint32_t* work = X + (size_t)K * m;                     // [3][padm]
  uint32_t* res = work + 3 * padm;                        // [slots][n]
  const uint32_t p = P.p[q];
  const uint2* gTf = P.tw + (size_t)(q * 2 + 0) * m;
  const uint2* gTi = P.tw + (size_t)(q * 2 + 1) * m;
  const uint32_t* gW = P.W + (size_t)(q * 2) * K * m;    // [2 b][K][m] of prime q

  // ---- stage the prime's twiddles and W rows (TMA bulk copies; they land during the split)
  if (STAGE && tid == 0) {
    mbar_init(&s_bar, 1);
    mbar_fence_init();
    mbar_expect_tx(&s_bar, (uint32_t)(4 * m + 2 * K * m) * 4u);
    bulk_g2s(s_tw, gTf, m * 8u, &s_bar);
    bulk_g2s(s_tw + m, gTi, m * 8u, &s_bar);
    for (int r = 0; r < 2 * K; ++r) bulk_g2s(s_W + (size_t)r * m, gW + (size_t)r * m, m * 4u, &s_bar);
  }
  for (int i = tid; i < 4 * SS + stats_stride(K); i += NT) s_sched[i] = 0;  // schedules (alg8_schedule
                                                                             // expects them zeroed), stats
  if (tid < 2 + 2 * K) s_wsplit[tid] = __ldg(&P.wsplit[tid]);

  // ---- a1 + a2: split of both parts (the k_split_cluster sequence, one CTA, no DSMEM)
  SplitParams SP{};
  SP.x = P.x; SP.chirp = P.chirp; SP.len = P.n; SP.mode = 0; SP.conj = P.conj;
  SP.K = K; SP.alpha = P.alpha; SP.rho = P.rho; SP.L = L; SP.wsplit = s_wsplit;
  SP.stats = s_stats; SP.sched = s_sched; SP.shared = 0;
  int kv[2] = {K, K};
  int Eprev[2] = {0, 0};
  bool bad = false;
  for (int level = 0; level <= K; ++level) {
    SplitC<false> lc[2];
#pragma unroll
    for (int v = 0; v < 2; ++v) lc[v] = split_c<false>(Eprev[v], P.alpha, P.rho);
    unsigned long long m0 = 0, m1 = 0;
    for (int j0 = tid; j0 < nn; j0 += kSmallEPT * NT) {
      double h[kSmallEPT][2], l[kSmallEPT][2];
#pragma unroll
      for (int u = 0; u < kSmallEPT; ++u) {
        const int j = min(j0 + u * NT, nn - 1);  // out-of-range slots redo element n - 1
        if (level == 0) {
          load_xprime(SP, b, j, h[u][0], l[u][0], h[u][1], l[u][1]);
        } else {
#pragma unroll
          for (int v = 0; v < 2; ++v) {
            h[u][v] = xp[v * nn + j];
            l[u][v] = xp[(2 + v) * nn + j];
          }
        }
      }
      if (level > 0) {
#pragma unroll
        for (int u = 0; u < kSmallEPT; ++u) {
          const int j = j0 + u * NT;
#pragma unroll
          for (int v = 0; v < 2; ++v) {
            int32_t D = 0;
            if (level - 1 < kv[v]) D = split_step(h[u][v], l[u][v], lc[v]);
            if (v == a && j < nn) dig[(level - 1) * nn + j] = D;
          }
        }
      }
      if (level == K) continue;
#pragma unroll
      for (int u = 0; u < kSmallEPT; ++u) {
        const int j = j0 + u * NT;
        if (j >= nn) continue;
#pragma unroll
        for (int v = 0; v < 2; ++v) {
          xp[v * nn + j] = h[u][v];
          xp[(2 + v) * nn + j] = l[u][v];
        }
        const unsigned long long a0 = (unsigned long long)__double_as_longlong(fabs(h[u][0]));
        const unsigned long long a1 = (unsigned long long)__double_as_longlong(fabs(h[u][1]));
        m0 = a0 > m0 ? a0 : m0;  // NaN bits exceed +Inf bits: a NaN sticks
        m1 = a1 > m1 ? a1 : m1;
      }
    }
    if (level == K) break;
    SMALL_STAMP(8 + 2 * level);
    m0 = warp_max_u64(m0);
    m1 = warp_max_u64(m1);
    if (lane == 0) { s_red[0][warp] = m0; s_red[1][warp] = m1; }
    __syncthreads();
    SMALL_STAMP(9 + 2 * level);
    m0 = m1 = 0;
#pragma unroll
    for (int w = 0; w < NT / 32; ++w) {
      m0 = s_red[0][w] > m0 ? s_red[0][w] : m0;
      m1 = s_red[1][w] > m1 ? s_red[1][w] : m1;
    }
    __syncthreads();  // s_red free for the next level
    if (tid == 0) { s_mu[level] = m0; s_mu[K + level] = m1; }
    const unsigned long long mv[2] = {m0, m1};
#pragma unroll
    for (int v = 0; v < 2; ++v) {
      const unsigned long long u = mv[v];
      if (u >= kInfBits) bad = true;
      Eprev[v] = (u == 0 || u >= kInfBits) ? 0 : ceil_log2_bits(u);
      if (u == 0 && kv[v] == K) kv[v] = level;
    }
    if (bad) {  // as k_split_cluster: later levels keep mu = 0
      for (int k = level + 1; k < K; ++k)
        if (tid == 0) { s_mu[k] = 0; s_mu[K + k] = 0; }
      break;
    }
  }
  SMALL_STAMP(14);
  __syncthreads();
  int Ef[2][kMaxK], kvf[2];
  bad = split_exponents(SP, 0, s_mu, Ef, kvf, true, true);  // stats + 4 schedules -> smem
  __syncthreads();
  SMALL_STAMP(15);
  if (rank == 0) {  // the per-transform records the multi-kernel path leaves in the workspace
    if (tid < 2 * K) P.mu[b * 2 * K + tid] = s_mu[tid];
    for (int i = tid; i < stats_stride(K); i += NT) P.stats[b * stats_stride(K) + i] = s_stats[i];
    for (int i = tid; i < 4 * SS; i += NT) P.sched[b * 4 * SS + i] = s_sched[i];
  }
  for (int i = tid; i < 4 * K * K; i += NT) {
    const int cv = i / (K * K), g = i % (K * K);
    if (g < s_sched[cv * SS]) s_sc[cv][g] = pow2_exact(-s_sched[cv * SS + 1 + g * (2 + 2 * L)]);
  }
  const int ng[4] = {s_sched[0], s_sched[SS], s_sched[2 * SS], s_sched[3 * SS]};
  SMALL_STAMP(1);

  // ---- a3: the ka forward spectra of part a, prime q (every z recomputes them)
  if (STAGE) mbar_wait(&s_bar, 0u);
  const uint2* Tf = STAGE ? s_tw : gTf;
  const uint2* Ti = STAGE ? s_tw + m : gTi;
  const uint32_t* Wq = STAGE ? s_W : gW;
  const int ka = bad ? 0 : kvf[a];
  uint32_t* const wk3[3] = {work, work + padm, work + 2 * padm};
  if (OZ_SMALL_FWD3 && ka == 3) {  // the three slices as one NV = 3 pass (shared twiddle loads, 3x ILP)
    __syncthreads();  // xp reads done
    sub_ntt_multi<LOGC, false, 1, 3, kSmallLogE, true, false, false, STAGE>(
        tid, wk3, 0u, 1u, Tf, Tw0{nullptr, 0u, 0u}, p,
        [&](int v, int, uint32_t e) -> uint32_t { return e < (uint32_t)nn ? lift(dig[v * nn + e], p) : 0u; },
        [&](int v, int, uint32_t e, uint32_t val) { X[v * m + row_perm_lin(e, LOGC, kSmallLogE)] = val; });
  } else {
    for (int s = 0; s < ka; ++s) {
      __syncthreads();  // xp reads done (s = 0) / exchange buffer free
      const int32_t* D = dig + s * nn;
      uint32_t* xs = X + s * m;
      sub_ntt<LOGC, false, 1, kSmallLogE, true, STAGE>(
          tid, work, 0u, 1u, Tf, p,
          [&](int, uint32_t e) -> uint32_t { return e < (uint32_t)nn ? lift(D[e], p) : 0u; },
          [&](int, uint32_t e, uint32_t v) { xs[row_perm_lin(e, LOGC, kSmallLogE)] = v; });
    }
  }
  SMALL_STAMP(2);
  // ---- a4 + a5: items (ci, g) = every Z-th of the two convolutions' Alg.8 groups
  const uint32_t pinv = 0u - P.pinv[q];  // +p^{-1} mod 2^32
  const int cvs[2] = {a, a == 0 ? 3 : 2};
  const int nitems = bad ? 0 : ng[cvs[0]] + ng[cvs[1]];
  constexpr int CNT = RoundT<LOGC, true, 0, kSmallLogE>::cnt;
  for (int it = z, slot = 0; it < nitems; it += Z, ++slot) {
    __syncthreads();  // spectra written / exchange buffer free
    const int ci = it < ng[cvs[0]] ? 0 : 1;
    const int g = ci ? it - ng[cvs[0]] : it;
    const int cv = cvs[ci];
    const int32_t* grp = s_sched + cv * SS + 1 + g * (2 + 2 * L);
    const int np = grp[1];
    const uint32_t* Wb = Wq + (size_t)conv_b(cv) * K * m;
    uint32_t zv[CNT];
    for (int ip0 = 0; ip0 < np; ip0 += 3) {  // lazy sums of <= 3 products, one REDC each
      unsigned long long T[CNT];
#pragma unroll
      for (int i = 0; i < CNT; ++i) T[i] = 0ull;
      const int ipe = min(np, ip0 + 3);
      for (int ip = ip0; ip < ipe; ++ip) {
        const uint32_t* xr = X + grp[2 + 2 * ip] * m;
        const uint32_t* wr = Wb + (size_t)grp[3 + 2 * ip] * m;
#pragma unroll
        for (int i = 0; i < CNT; ++i) {
          const uint32_t e = round_elem<LOGC, true, 0, kSmallLogE>(tid, i);
          T[i] += (unsigned long long)xr[row_perm_lin(e, LOGC, kSmallLogE)] * wr[row_perm(e, LOGC, P.w_s0)];
        }
      }
#pragma unroll
      for (int i = 0; i < CNT; ++i) {
        const uint32_t r = redc_lazy3(T[i], p, pinv);
        zv[i] = ip0 == 0 ? r : add_mod(zv[i], r, p);
      }
    }
    uint32_t* rs = res + (size_t)slot * nn;
    const bool flip = P.fault && b == 0 && q == 0 && cv == 0 && g == ng[0] - 1;
    sub_ntt<LOGC, true, 1, kSmallLogE, true, STAGE>(
        tid, work, 0u, 1u, Ti, p, [&](int i, uint32_t) -> uint32_t { return zv[i]; },
        [&](int, uint32_t e, uint32_t val) {
          if (e < (uint32_t)nn) rs[e] = (flip && e == 0) ? val ^ 1u : val;
        });
  }
  SMALL_STAMP(3);
  cl.sync();  // every CTA's residues visible cluster-wide
  SMALL_STAMP(4);

  // ---- a6 + a7: thread (cv, jl) sums conv cv's Garner values 2^-cexp in flush order, then
  // the cv = 0 threads combine the four sums and post-chirp (k_crt_finish's sequence)
  constexpr int NQ = NT / 4;
  const int cvt = tid / NQ, jl = tid % NQ;
  for (int64_t j0 = (int64_t)rank * NQ; j0 < P.n; j0 += (int64_t)4 * Z * NQ) {
    const int64_t j = j0 + jl;
    double2 w = make_double2(0.0, 0.0);
    if (cvt == 0 && j < P.n) w = __ldg(&P.chirp[j]);  // in flight during the DD chain
    if (j < P.n && !bad) {
      const int cv = cvt, ca = conv_a(cv), ci = cv >> 1;  // cv 2, 3 are part a's second conv
      double sh = 0.0, sl = 0.0;
      for (int g0 = 0; g0 < ng[cv]; g0 += 9) {
        uint32_t z0[9], z1[9];
#pragma unroll
        for (int i = 0; i < 9; ++i) {
          if (g0 + i < ng[cv]) {
            const int it = ci ? ng[ca] + g0 + i : g0 + i;
            const int zr = it % Z, sl_ = it / Z;
            const uint32_t* r0 = cl.map_shared_rank(res, (0 * 2 + ca) * Z + zr);
            const uint32_t* r1 = cl.map_shared_rank(res, (1 * 2 + ca) * Z + zr);
            z0[i] = r0[(size_t)sl_ * nn + j];
            z1[i] = r1[(size_t)sl_ * nn + j];
          }
        }
#pragma unroll
        for (int i = 0; i < 9; ++i) {
          if (g0 + i < ng[cv]) {
            const long long Zv = garner2(z0[i], z1[i], P.F);
            double hs, ls;
            scaled_split(Zv, s_sc[cv][g0 + i], hs, ls);
            dd_add(sh, sl, hs, ls, sh, sl);
          }
        }
      }
      s_S[cv][jl] = make_double2(sh, sl);
    }
    __syncthreads();
    if (cvt == 0 && j < P.n) {
      double2 o;
      if (bad) {
        o.x = __longlong_as_double(0x7FF8000000000000ll);
        o.y = o.x;
      } else {
        o = dd_combine_postchirp(s_S[0][jl], s_S[1][jl], s_S[2][jl], s_S[3][jl], w, P.direction, P.n);
      }
      P.out[b * P.n + j] = o;
    }
    __syncthreads();
  }
  SMALL_STAMP(5);
  cl.sync();  // no CTA exits while another may still read its residues
  SMALL_STAMP(6);
}
#if OZ_SMALL_TIMING
extern "C" int ozfft_debug_small_times(unsigned long long* out) {
  return (int)cudaMemcpyFromSymbol(out, g_small_t, sizeof(g_small_t));
}
#endif

// ============================================================== fused inverse column pass + CRT
// For R > 1 the last log2(R) DIT stages, Garner's CRT and the scaled DD accumulation
// of one real convolution run in one kernel: CTA = (transform, conv, column block),
// looping over the conv's Alg.8 groups and both primes (next tile prefetched).  PRUNE
// (padded plans, n <= m/2): only the output rows i1 < R/2 are needed, so the
// upper half of the last stage is pruned; cyclic plans (m = n) keep all rows.  Output: the conv's DD sum S_cv(j) = sum_g Z_g(j) 2^-cexp_g in
// flush order (Alg.8 l.975-976), [nb][4][n] double2 (hi, lo).
struct ColCrtParams {
  int logm, K, L;
  int64_t n, nb;
  FinishParams F;          // CRT constants (p0, p1, p0inv, ...)
  const uint2* tw;         // [2 prime][2 dir][m]
  const uint32_t* G;       // [nb][2 q][4 cv][K*K][m]
  const int32_t* sched;    // [nb][4][sched_stride]
  double2* S;              // [nb][4][n]
  uint32_t* res_tap;       // null, or [nb][4][2][K*K][n] (workspace res layout)
  int64_t* crt_tap;        // null, or [nb][4][K*K][n]
};

// Column block of the fused inverse column kernel (real mode): the real-mode column width,
// narrowed by OZ_CI_CB_SHIFT (pruned plans) / OZ_CI_CB_SHIFT_FULL (unpruned, twice the
// accumulators) down to >= 8 columns.
__host__ __device__ constexpr int col_log_cb_ci(int logR, int logC, bool prune) {
  return col_log_cb(logR, logC) - (prune ? OZ_CI_CB_SHIFT : OZ_CI_CB_SHIFT_FULL) >= 3
             ? col_log_cb(logR, logC) - (prune ? OZ_CI_CB_SHIFT : OZ_CI_CB_SHIFT_FULL)
             : (col_log_cb(logR, logC) < 3 ? col_log_cb(logR, logC) : 3);
}

template <int LOGR, int LOGC, bool PRUNE, bool TS>
__global__ void __launch_bounds__(256, ColCfg<LOGR>::min_blocks_inv_crt) k_col_inv_crt(ColCrtParams P) {
  extern __shared__ uint32_t smem[];
  constexpr int LOGCB = col_log_cb_ci(LOGR, LOGC, PRUNE);
  constexpr int LOGE = col_loge(LOGR);
  constexpr int E = 1 << LOGE;
  constexpr int Cb = 1 << LOGCB;
  constexpr uint32_t C = 1u << LOGC;
  constexpr uint32_t m = 1u << (LOGR + LOGC);
  constexpr uint32_t ncb = 1u << (LOGC - LOGCB);
  constexpr int CNT = RoundT<LOGR, true, 0, LOGE>::cnt;
  constexpr int NR = RoundT<LOGR, true, 0, LOGE>::nr;
  // last DIT round: registers i with (i mod 2^S) < 2^(S-1) hold rows < R/2 (the only rows
  // needed, n <= m/2); they are packed into NH slots by hslot(i)
  constexpr int SL = RoundT<LOGR, true, NR - 1, LOGE>::S;
  constexpr int NH = RoundT<LOGR, true, NR - 1, LOGE>::cnt / (PRUNE ? 2 : 1);
  auto needed = [](int i) { return !PRUNE || (i & ((1 << SL) - 1)) < (1 << (SL - 1)); };
  auto hslot = [](int i) {
    return PRUNE ? ((i >> SL) << (SL - 1)) + (i & ((1 << (SL - 1)) - 1)) : i;
  };
  constexpr int THREADS = RoundT<LOGR, true, 0, LOGE>::Tv << LOGCB;
  constexpr int CNTL = RoundT<LOGR, true, NR - 1, LOGE>::cnt;  // registers of the last round
  const int G = P.K * P.K;
  const uint32_t cb = blockIdx.x % ncb;
  uint32_t v = blockIdx.x / ncb;  // b * 4 + cv
  const int cv = (int)(v & 3);
  const int64_t b = v >> 2;
  const int tid = threadIdx.x;
  const int c = tid & (Cb - 1);
  const int tv = tid >> LOGCB;
  const uint32_t col = (cb << LOGCB) + c;
  __shared__ double s_sc[kMaxK * kMaxK];
  __shared__ int s_ce[kMaxK * kMaxK];
  const int32_t* srow = P.sched + (b * 4 + cv) * sched_stride(P.K, P.L);
  const int ng = srow[0];
  const uint32_t lim = P.n > col ? (uint32_t)(P.n - col) : 0u;
  uint32_t nxt[E];
  // tile t -> (group g, prime q): t = 2 g + (q xor snake(g)).  With OZ_CI_SNAKE the primes
  // alternate q0 q1 | q1 q0 | q0 q1 ..., so each prime's column twiddles serve two tiles in a
  // row (L1 reuse); the group's second tile runs Garner either way.
  constexpr bool SNAKE = LOGR >= OZ_CI_SNAKE_MIN && LOGR <= OZ_CI_SNAKE_MAX;
  auto tile_q = [](int t) { return SNAKE ? ((t & 1) ^ ((t >> 1) & 1)) : (t & 1); };
  auto fetch = [&](int t) {
    const int g = t >> 1, q = tile_q(t);
    const uint32_t* in = P.G + (((b * 2 + q) * 4 + cv) * G + g) * (int64_t)m + col;
#pragma unroll
    for (int i = 0; i < CNT; ++i) nxt[i] = __ldcs(&in[round_elem<LOGR, true, 0, LOGE>(tv, i) * C]);
  };
#if OZ_CI_FETCH_FIRST
  if (ng > 0) fetch(0);  // in flight during the schedule, accumulator and twiddle set-up
#endif
  for (int g = tid; g < ng; g += blockDim.x) {
    s_ce[g] = srow[1 + g * (2 + 2 * P.L)];
    s_sc[g] = scalbn(1.0, -s_ce[g]);
  }
  constexpr uint32_t TILE = ((1u << LOGR) + (1u << LOGR) / E + 1) * Cb;
  constexpr uint32_t TILEW = (TILE + 3) & ~3u;
  // OZ_CI_DB: two exchange tiles used alternately, so a tile's exchange writes never meet
  // the previous tile's reads and the per-tile "tile free" barrier goes (the extra 17 KB
  // keep 3 CTAs per SM: registers bound the occupancy)
  double2* Sacc = reinterpret_cast<double2*>(smem + (OZ_CI_DB ? 2 : 1) * TILEW);  // [NH][THREADS]
  // OZ_CI_RACC: the DD accumulators in registers instead of shared memory (frees 32 KB per
  // CTA for L1, where the column twiddles live)
  constexpr bool kRacc = ci_racc(NH);
  constexpr bool kGacc = ci_gacc(NH);
  double2 racc[kRacc ? NH : 1];
#pragma unroll
  for (int i = 0; i < NH; ++i) {
    if constexpr (kRacc)
      racc[i] = make_double2(0.0, 0.0);
    else if constexpr (!kGacc)
      Sacc[i * THREADS + tid] = make_double2(0.0, 0.0);
  }
  // OZ_CI_GACC: slot h of this thread is output row hrow(h) of its column
  auto islot = [](int h) {
    return PRUNE ? ((h >> (SL - 1)) << SL) + (h & ((1 << (SL - 1)) - 1)) : h;
  };
  // OZ_CI_T0S: for long columns, the step-1 round's column twiddles of both primes (the same
  // for every group of the CTA) are staged in shared memory once, after the accumulators (ncu
  // at c3: the first product of each tile waited on these L2 loads, 13 % of the samples)
  constexpr int S1 = col_s1(LOGR);
  constexpr bool kT0S = OZ_CI_T0S != 0 && LOGR >= OZ_CI_T0S;
  [[maybe_unused]] uint2* tw0 = reinterpret_cast<uint2*>(Sacc + (kRacc || kGacc ? 0 : NH * THREADS));  // [2 q][2^S1][Cb]
  if constexpr (kT0S) {
    for (int q = 0; q < 2; ++q)
      stage_col_tw0<S1, Cb>(tw0 + q * (Cb << S1), P.tw + (size_t)(q * 2 + 1) * m, C, cb << LOGCB);
  }
#if !OZ_CI_FETCH_FIRST
  if (ng > 0) fetch(0);
#endif
  __syncthreads();  // s_sc ready
  uint32_t r0[NH];  // the group's first tile's residues
  double2* const So = P.S + (b * 4 + cv) * P.n + col;
  for (int t = 0; t < 2 * ng; ++t) {
    const int g = t >> 1, q = tile_q(t);
    uint32_t cur[E];
#pragma unroll
    for (int i = 0; i < E; ++i) cur[i] = nxt[i];
    if (t + 1 < 2 * ng) fetch(t + 1);
    if (!OZ_CI_DB && t > 0) __syncthreads();  // smem tile free
    uint32_t* const tb = smem + (OZ_CI_DB ? (uint32_t)(t & 1) * TILEW : 0u);
    const uint32_t p = q ? P.F.p1 : P.F.p0;
    const uint2* T = P.tw + (size_t)(q * 2 + 1) * m;
    uint32_t rr[NH];
    if constexpr (kT0S)
      sub_ntt_t0<LOGR, true, Cb, LOGE>(tv, tb + c, col, C, T, Tw0{tw0 + q * (Cb << S1), (uint32_t)c, (uint32_t)Cb}, p,
                              [&](int i, uint32_t) -> uint32_t { return cur[i]; },
                              [&](int i, uint32_t, uint32_t val) {
                                if (needed(i)) rr[hslot(i)] = val;  // rows >= R/2 never needed
                              });
    else
      sub_ntt<LOGR, true, Cb, LOGE>(tv, tb + c, col, C, T, p,
                              [&](int i, uint32_t) -> uint32_t { return cur[i]; },
                              [&](int i, uint32_t, uint32_t val) {
                                if (needed(i)) rr[hslot(i)] = val;  // rows >= R/2 never needed
                              });
    if (P.res_tap) {
      uint32_t* rt = P.res_tap + (((b * 4 + cv) * 2 + q) * G + g) * P.n + col;
#pragma unroll
      for (int i = 0; i < CNTL; ++i) {
        if (!needed(i)) continue;
        const uint32_t e = round_elem<LOGR, true, NR - 1, LOGE>(tv, i);
        if (e * C < lim) rt[e * C] = rr[hslot(i)];
      }
    }
    if ((t & 1) == 0) {
#pragma unroll
      for (int i = 0; i < NH; ++i) r0[i] = rr[i];
    } else {
      const double sc = s_sc[g];
      if (P.crt_tap) {  // test-only tap: the CRT integers of the rows < n
#pragma unroll
        for (int i = 0; i < CNTL; ++i) {
          if (!needed(i)) continue;
          const uint32_t e = round_elem<LOGR, true, NR - 1, LOGE>(tv, i);
          const int h = hslot(i);
          if (e * C < lim)
            P.crt_tap[((b * 4 + cv) * G + g) * P.n + col + e * C] =
                q ? garner2(r0[h], rr[h], P.F) : garner2(rr[h], r0[h], P.F);
        }
      }
      // Garner (l.974) and the scaled sum in flush order (l.975-976) for every slot, without
      // a per-row branch: rows >= n compute sums that are never stored, and the slots' chains
      // are independent, so batches of OZ_CI_ILP of them interleave (a branch per row
      // serialised them behind the DD add's dependent latency)
#pragma unroll
      for (int h0 = 0; h0 < NH; h0 += OZ_CI_ILP) {
        constexpr int NB = OZ_CI_ILP;
        double2 acc[NB];
        long long Z[NB];
#pragma unroll
        for (int j = 0; j < NB; ++j)
          if (h0 + j < NH) {
            const int h = h0 + j;
            Z[j] = q ? garner2(r0[h], rr[h], P.F) : garner2(rr[h], r0[h], P.F);
            if constexpr (kRacc) {
              acc[j] = racc[h];
            } else if constexpr (kGacc) {
              const uint32_t e = round_elem<LOGR, true, NR - 1, LOGE>(tv, islot(h));
              acc[j] = (g > 0 && e * C < lim) ? __ldcg(&So[e * C]) : make_double2(0.0, 0.0);
            } else {
              acc[j] = Sacc[h * THREADS + tid];
            }
          }
#pragma unroll
        for (int j = 0; j < NB; ++j)
          if (h0 + j < NH) {
            if constexpr (TS) {  // f4: TSAdd of z 2^-cexp (slot holds the TS words)
              acc[j] = ts_accum(acc[j], Z[j], s_ce[g]);
            } else {
              double hs, ls;
              scaled_split(Z[j], sc, hs, ls);
              dd_add(acc[j].x, acc[j].y, hs, ls, acc[j].x, acc[j].y);
            }
          }
#pragma unroll
        for (int j = 0; j < NB; ++j)
          if (h0 + j < NH) {
            if constexpr (kRacc) {
              racc[h0 + j] = acc[j];
            } else if constexpr (kGacc) {
              const uint32_t e = round_elem<LOGR, true, NR - 1, LOGE>(tv, islot(h0 + j));
              if (e * C < lim) __stcg(&So[e * C], acc[j]);
            } else {
              Sacc[(h0 + j) * THREADS + tid] = acc[j];
            }
          }
      }
    }
  }
  if (kGacc && ng > 0) return;  // the sums are already in place
#pragma unroll
  for (int i = 0; i < CNTL; ++i) {
    if (!needed(i)) continue;
    const uint32_t e = round_elem<LOGR, true, NR - 1, LOGE>(tv, i);
    if (e * C < lim) {
      if constexpr (kRacc)
        So[e * C] = racc[hslot(i)];
      else if constexpr (kGacc)
        So[e * C] = make_double2(0.0, 0.0);  // no groups: the zero sum
      else
        So[e * C] = Sacc[hslot(i) * THREADS + tid];
    }
  }
}

// f2 (image mode): the fused inverse column pass + CRT for the complex convolution.  CTA
// = (transform, column block); per Alg.8 group the four tiles (image +, p0), (image -, p0),
// (image +, p1), (image -, p1) are transformed in turn (next tile prefetched); each prime's
// image pair gives (re, im) residues, the primes' pairs give Re and Im by Garner, and the
// DD sums of Re 2^-c and Im 2^-c in flush order go to S[b][0] and S[b][1].
// Column block of the image kernel: half the real-mode width (>= 8 columns, one 32-byte
// sector per row segment) -- its accumulators are twice as many (Re and Im sums), so the
// narrower block keeps more CTAs resident.
__host__ __device__ constexpr int col_log_cb_img(int logR, int logC) {
  return col_log_cb(logR, logC) - OZ_IMG_CB_SHIFT >= 3 ? col_log_cb(logR, logC) - OZ_IMG_CB_SHIFT
                                                        : (col_log_cb(logR, logC) < 3 ? col_log_cb(logR, logC) : 3);
}

template <int LOGR, int LOGC, bool PRUNE>
__global__ void __launch_bounds__(256, 2) k_col_inv_crt_img(ColCrtParams P) {
  extern __shared__ uint32_t smem[];
  constexpr int LOGCB = col_log_cb_img(LOGR, LOGC);
  constexpr int LOGE = col_loge(LOGR);
  constexpr int E = 1 << LOGE;
  constexpr int Cb = 1 << LOGCB;
  constexpr uint32_t C = 1u << LOGC;
  constexpr uint32_t m = 1u << (LOGR + LOGC);
  constexpr uint32_t ncb = 1u << (LOGC - LOGCB);
  constexpr int CNT = RoundT<LOGR, true, 0, LOGE>::cnt;
  constexpr int NR = RoundT<LOGR, true, 0, LOGE>::nr;
  constexpr int SL = RoundT<LOGR, true, NR - 1, LOGE>::S;
  constexpr int NH = RoundT<LOGR, true, NR - 1, LOGE>::cnt / (PRUNE ? 2 : 1);
  auto needed = [](int i) { return !PRUNE || (i & ((1 << SL) - 1)) < (1 << (SL - 1)); };
  auto hslot = [](int i) {
    return PRUNE ? ((i >> SL) << (SL - 1)) + (i & ((1 << (SL - 1)) - 1)) : i;
  };
  constexpr int THREADS = RoundT<LOGR, true, 0, LOGE>::Tv << LOGCB;
  constexpr int CNTL = RoundT<LOGR, true, NR - 1, LOGE>::cnt;
  const int G = P.K * P.K;
  const uint32_t cb = blockIdx.x % ncb;
  const int64_t b = blockIdx.x / ncb;
  const int tid = threadIdx.x;
  const int c = tid & (Cb - 1);
  const int tv = tid >> LOGCB;
  const uint32_t col = (cb << LOGCB) + c;
  __shared__ double s_sc[kMaxK * kMaxK];
  const int32_t* srow = P.sched + (b * 4) * sched_stride(P.K, P.L);  // the complex schedule
  const int ng = srow[0];
  for (int g = tid; g < ng; g += blockDim.x) s_sc[g] = scalbn(1.0, -srow[1 + g * (2 + 2 * P.L)]);
  constexpr uint32_t TILE = ((1u << LOGR) + (1u << LOGR) / E + 1) * Cb;
  double2* Sacc = reinterpret_cast<double2*>(smem + ((TILE + 3) & ~3u));  // [2][NH][THREADS], 16B-aligned
#pragma unroll
  for (int i = 0; i < 2 * NH; ++i) Sacc[i * THREADS + tid] = make_double2(0.0, 0.0);
  const uint32_t lim = P.n > col ? (uint32_t)(P.n - col) : 0u;
  uint32_t nxt[E];
  auto fetch = [&](int t) {  // tile t = 4 g + 2 q + image
    const int g = t >> 2, q = (t >> 1) & 1, img = t & 1;
    const uint32_t* in = P.G + (((b * 2 + q) * 4 + img) * G + g) * (int64_t)m + col;
#pragma unroll
    for (int i = 0; i < CNT; ++i) nxt[i] = __ldcs(&in[round_elem<LOGR, true, 0, LOGE>(tv, i) * C]);
  };
  if (ng > 0) fetch(0);
  __syncthreads();  // s_sc ready
  uint32_t ra[NH], zr0[NH], zi0[NH];
  for (int t = 0; t < 4 * ng; ++t) {
    const int g = t >> 2, q = (t >> 1) & 1, img = t & 1;
    uint32_t cur[E];
#pragma unroll
    for (int i = 0; i < E; ++i) cur[i] = nxt[i];
    if (t + 1 < 4 * ng) fetch(t + 1);
    if (t > 0) __syncthreads();  // smem tile free
    const uint32_t p = q ? P.F.p1 : P.F.p0;
    const uint2* T = P.tw + (size_t)(q * 2 + 1) * m;
    uint32_t rr[NH];
    sub_ntt<LOGR, true, Cb, LOGE>(tv, smem + c, col, C, T, p,
                            [&](int i, uint32_t) -> uint32_t { return cur[i]; },
                            [&](int i, uint32_t, uint32_t val) {
                              if (needed(i)) rr[hslot(i)] = val;
                            });
    if (P.res_tap) {
      uint32_t* rt = P.res_tap + (((b * 4 + img) * 2 + q) * G + g) * P.n + col;
#pragma unroll
      for (int i = 0; i < CNTL; ++i) {
        if (!needed(i)) continue;
        const uint32_t e = round_elem<LOGR, true, NR - 1, LOGE>(tv, i);
        if (e * C < lim) rt[e * C] = rr[hslot(i)];
      }
    }
    if (img == 0) {
#pragma unroll
      for (int i = 0; i < NH; ++i) ra[i] = rr[i];
    } else if (q == 0) {
#pragma unroll
      for (int i = 0; i < NH; ++i) image_pair(ra[i], rr[i], P.F.inv2[0], P.F.inv2i[0], p, zr0[i], zi0[i]);
    } else {
      const double sc = s_sc[g];
#pragma unroll
      for (int i = 0; i < CNTL; ++i) {
        if (!needed(i)) continue;
        const uint32_t e = round_elem<LOGR, true, NR - 1, LOGE>(tv, i);
        const int h = hslot(i);
        if (e * C < lim) {
          uint32_t zr1, zi1;
          image_pair(ra[h], rr[h], P.F.inv2[1], P.F.inv2i[1], p, zr1, zi1);
#pragma unroll
          for (int part = 0; part < 2; ++part) {
            const long long Z = part ? garner2(zi0[h], zi1, P.F) : garner2(zr0[h], zr1, P.F);
            if (P.crt_tap) P.crt_tap[((b * 4 + part) * G + g) * P.n + col + e * C] = Z;
            double hs, ls;
            scaled_split(Z, sc, hs, ls);
            double2 a = Sacc[(part * NH + h) * THREADS + tid];
            dd_add(a.x, a.y, hs, ls, a.x, a.y);
            Sacc[(part * NH + h) * THREADS + tid] = a;
          }
        }
      }
    }
  }
#pragma unroll
  for (int part = 0; part < 2; ++part) {
    double2* So = P.S + (b * 4 + part) * P.n + col;
#pragma unroll
    for (int i = 0; i < CNTL; ++i) {
      if (!needed(i)) continue;
      const uint32_t e = round_elem<LOGR, true, NR - 1, LOGE>(tv, i);
      if (e * C < lim) So[e * C] = Sacc[(part * NH + hslot(i)) * THREADS + tid];
    }
  }
}

// y' = (S_rr - S_ii) + i (S_ir + S_ri), post-chirp y = y' (.) omega
// (Alg.4 l.480-484), fp64 output; inverse direction: conj and RN division by n (O10).
__global__ void __launch_bounds__(256) k_finish_dd(const double2* __restrict__ S,
                                                   const int32_t* __restrict__ stats, int K,
                                                   const double2* __restrict__ chirp,
                                                   double2* __restrict__ out, int64_t n,
                                                   int direction, int image, int ts) {
  const int64_t b = blockIdx.y;
  const int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (j >= n) return;
  double2 o;
  if (stats[b * stats_stride(K) + 2 + 2 * K] & 1) {
    o.x = __longlong_as_double(0x7FF8000000000000ll);
    o.y = o.x;
    out[b * n + j] = o;
    return;
  }
  if (ts) {  // f4: the four sums are TS words
    o = ts_finish(ts_of_slot(__ldcs(&S[(b * 4 + 0) * n + j])), ts_of_slot(__ldcs(&S[(b * 4 + 1) * n + j])),
                  ts_of_slot(__ldcs(&S[(b * 4 + 2) * n + j])), ts_of_slot(__ldcs(&S[(b * 4 + 3) * n + j])),
                  chirp[j]);
    if (direction > 0) {
      const double dn = (double)n;
      o.x = __ddiv_rn(o.x, dn);
      o.y = __ddiv_rn(-o.y, dn);
    }
    out[b * n + j] = o;
    return;
  }
  double yrh, yrl, yih, yil;
  if (image) {  // f2: the DD sums are Re y' and Im y' themselves
    const double2 re = __ldcs(&S[(b * 4 + 0) * n + j]), im = __ldcs(&S[(b * 4 + 1) * n + j]);
    yrh = re.x; yrl = re.y; yih = im.x; yil = im.y;
  } else {
    const double2 rr = __ldcs(&S[(b * 4 + 0) * n + j]), ii = __ldcs(&S[(b * 4 + 1) * n + j]);
    const double2 ir = __ldcs(&S[(b * 4 + 2) * n + j]), ri = __ldcs(&S[(b * 4 + 3) * n + j]);
    dd_add(rr.x, rr.y, -ii.x, -ii.y, yrh, yrl);
    dd_add(ir.x, ir.y, ri.x, ri.y, yih, yil);
  }
  const double2 w = chirp[j];
  double a1h, a1l, a2h, a2l, ore, oim, tmp;
  dd_mul_d(yrh, yrl, w.x, a1h, a1l);
  dd_mul_d(yih, yil, w.y, a2h, a2l);
  dd_add(a1h, a1l, -a2h, -a2l, ore, tmp);
  dd_mul_d(yrh, yrl, w.y, a1h, a1l);
  dd_mul_d(yih, yil, w.x, a2h, a2l);
  dd_add(a1h, a1l, a2h, a2l, oim, tmp);
  if (direction > 0) {
    const double dn = (double)n;
    ore = __ddiv_rn(ore, dn);
    oim = __ddiv_rn(-oim, dn);
  }
  o.x = ore;
  o.y = oim;
  out[b * n + j] = o;
}

static void fill_crt_consts(const Plan& pl, FinishParams& FP) {
  FP.p0 = pl.p[0];
  FP.p1 = pl.p[1];
  FP.p0inv = pl.p0inv_mod_p1;
  FP.p0inv_sh = (uint32_t)(((uint64_t)pl.p0inv_mod_p1 << 32) / pl.p[1]);
  FP.p1_barrett = (uint32_t)((1ull << 32) / pl.p[1]);
  FP.P = (unsigned long long)pl.p[0] * pl.p[1];
  FP.halfP = (FP.P - 1) / 2;
  for (int q = 0; q < 2; ++q) {  // f2: 2^-1 and (2 iota)^-1 = 2^-1 (-iota) (iota^-1 = -iota)
    const uint64_t p = pl.p[q];
    const uint64_t i2 = (p + 1) / 2;
    const uint64_t i2i = pl.image ? i2 * (p - pl.iota[q]) % p : 0;
    FP.inv2[q] = make_uint2((uint32_t)i2, (uint32_t)((i2 << 32) / p));
    FP.inv2i[q] = make_uint2((uint32_t)i2i, (uint32_t)((i2i << 32) / p));
  }
  FP.ts = pl.ts;
}

// f2: Shoup pairs of iota_q (image 0) and p_q - iota_q (image 1)
static void fill_iota(const Plan& pl, uint2 (&io)[2][2]) {
  for (int q = 0; q < 2; ++q)
    for (int img = 0; img < 2; ++img) {
      const uint64_t p = pl.p[q];
      const uint64_t w = pl.image ? (img ? p - pl.iota[q] : pl.iota[q]) : 0;
      io[q][img] = make_uint2((uint32_t)w, (uint32_t)((w << 32) / p));
    }
}

// ============================================================== small utility kernels
// W finalize: W~[q][b][t][row*C + row_perm(e)] = W m^{-1} 2^32 mod p (Montgomery form for the
// pointwise REDC) from the forward spectra X[q][b][t][row*C + e] (internal order).
__global__ void k_w_finalize(const uint32_t* __restrict__ X, uint32_t* __restrict__ Wm, int K,
                             int64_t m, int logC, int S0, uint32_t p0, uint32_t p1, uint32_t minv0,
                             uint32_t minv1) {
  const int64_t total = (int64_t)4 * K * m;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < total;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int q = (int)(i / (2 * K * m));
    const uint32_t p = q ? p1 : p0, mi = q ? minv1 : minv0;
    const uint32_t w = (uint32_t)(((uint64_t)X[i] * mi) % p);
    const int64_t e = i & ((1ll << logC) - 1);
    const int64_t dst = (i - e) + row_perm((uint32_t)e, logC, S0);
    Wm[dst] = (uint32_t)(((uint64_t)w << 32) % p);
  }
}

// Test-only fault injection (Plan::fault, env OZFFT_FAULT_INJECT): flip bit 0 of the first
// word of one NTT-domain group value / residue vector -- the last group in Alg.8 flush order
// (the leading digits, so the error reaches the fp64 output; the first groups hold the
// smallest terms, 2^-144 below) -- so that the parity tests must fail (tests/test_gpu_fault.py).
__global__ void k_fault_inject(uint32_t* base, int64_t gstride, const int32_t* sched) {
  const int g = sched[0] > 0 ? sched[0] - 1 : 0;
  base[g * gstride] ^= 1u;
}

// Tap conversion: internal bit-reversed order (optionally row-permuted, optionally times a
// per-vector constant mod p) -> natural order:  dst[o(v)][k] = src[v][pos(bitrev(k))] * mult[v].
__global__ void k_tap_permute(const uint32_t* __restrict__ src, uint32_t* __restrict__ dst,
                              int64_t nvec, int logm, const int64_t* __restrict__ dst_off,
                              const uint32_t* __restrict__ vec_p,
                              const uint32_t* __restrict__ vec_mult, int logC, int S0) {
  const int64_t m = 1ll << logm;
  const int64_t total = nvec * m;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < total;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t v = i >> logm, k = i & (m - 1);
    int64_t br = logm ? (int64_t)(__brevll((unsigned long long)k) >> (64 - logm)) : 0;
    if (logC >= 0) {  // source stored in row_perm order
      const int64_t e = br & ((1ll << logC) - 1);
      br = (br - e) + row_perm((uint32_t)e, logC, S0);
    }
    uint32_t val = src[v * m + br];
    if (vec_mult) val = (uint32_t)(((uint64_t)val * vec_mult[v]) % vec_p[v]);
    dst[dst_off[v] + k] = val;
  }
}

// ============================================================== launchers
static ozfft_status cuda_check(const char* what) {
  const cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) {
    set_error(std::string(what) + ": " + cudaGetErrorString(e));
    return OZFFT_ERR_CUDA;
  }
  return OZFFT_OK;
}

static int col_logCb(int logR, int logC) { return col_log_cb(logR, logC); }
static size_t col_smem(int logR, int logCb) {
  const size_t R = 1ull << logR;
  return (R + (R >> col_loge(logR)) + 1) * (1ull << logCb) * sizeof(uint32_t);
}
static int col_threads(int logR, int logCb) {
  const int le = col_loge(logR);
  const int Tv = logR >= le ? (1 << (logR - le)) : 1;
  return Tv << logCb;
}
template <class K>
static void set_smem(K kern, size_t bytes) {
  if (bytes > 48 * 1024)
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes);
}

#ifndef OZ_SPLIT_CLUSTER
#define OZ_SPLIT_CLUSTER 1  // fused one-launch split for n <= kSplitClusterMaxLen
#endif
// SM count of the current device (cached per device id; a process may drive several GPUs)
static int sm_count() {
  static std::atomic<int> cache[64] = {};
  int d = 0;
  cudaGetDevice(&d);
  if (d < 0 || d >= 64) d = 0;
  int v = cache[d].load(std::memory_order_relaxed);
  if (v == 0) {
    v = 148;
    cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, d);
    cache[d].store(v, std::memory_order_relaxed);
  }
  return v;
}
#ifndef OZ_ROW_Z_WAVES
#define OZ_ROW_Z_WAVES 0  // two-pass rows: item split when the grid has fewer waves than this
#endif
#ifndef OZ_ROW_ZMAX
#define OZ_ROW_ZMAX 18  // most CTAs one (transform, part, prime) row of a one-pass plan uses
#endif
static ozfft_status launch_split(const Plan& pl, SplitParams SP, int64_t nb, cudaStream_t st) {
  const int threads = 256;
  int64_t blocks_per = (SP.len + threads * OZ_SPLIT_EPT - 1) / (threads * OZ_SPLIT_EPT);
  if (blocks_per < 1) blocks_per = 1;
  if (blocks_per * nb < 4 * sm_count()) {  // small batches: fill the GPU (grid-stride kernels)
    const int64_t want = (4 * sm_count() + nb - 1) / nb, most = (SP.len + threads - 1) / threads;
    blocks_per = want < most ? want : most;
    if (blocks_per < 1) blocks_per = 1;
  }
  if (blocks_per > 65535) blocks_per = 65535;
  dim3 grid((unsigned)blocks_per, (unsigned)nb);
#if OZ_SPLIT_CLUSTER
  const int64_t cl_max = pl.split_cluster_max >= 0 && pl.split_cluster_max < kSplitClusterMaxLen
                            ? pl.split_cluster_max : kSplitClusterMaxLen;
  if (SP.len <= cl_max) {  // one cluster per transform, one launch (a1 + a2)
    int cs = 1;
    while (cs < 8 && (int64_t)cs * OZ_SPLIT_CL_CHUNK < SP.len) cs *= 2;
    const int chunk = (int)((SP.len + cs - 1) / cs);
    int thr = (chunk + OZ_SPLIT_CL_EPT - 1) / OZ_SPLIT_CL_EPT;
    thr = thr < 32 ? 32 : (thr > kSplitClusterThreads ? kSplitClusterThreads : (thr + 31) & ~31);
    const size_t smem = (size_t)chunk * (pl.ts ? 6 * sizeof(float) : 4 * sizeof(double));
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3((unsigned)cs, (unsigned)nb);
    cfg.blockDim = dim3((unsigned)thr);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = st;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = (unsigned)cs;
    at[0].val.clusterDim.y = 1;
    at[0].val.clusterDim.z = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    // static + dynamic shared memory may pass 48 KB: opt in once per device to the largest
    // chunk (function attributes are per device)
    static std::atomic<bool> smem_set[64] = {};
    int dev = 0;
    cudaGetDevice(&dev);
    if (dev < 0 || dev >= 64) dev = 0;
    if (!smem_set[dev].load(std::memory_order_relaxed)) {
      const int mx = 160 * 1024;
      cudaFuncSetAttribute(k_split_cluster<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, mx);
      cudaFuncSetAttribute(k_split_cluster<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, mx);
      smem_set[dev].store(true, std::memory_order_relaxed);
    }
    prof_mark(pl, OZFFT_STAGE_SPLIT_MAX, true, st);
    if (pl.ts)
      cudaLaunchKernelEx(&cfg, k_split_cluster<true>, SP, chunk);
    else
      cudaLaunchKernelEx(&cfg, k_split_cluster<false>, SP, chunk);
    prof_mark(pl, OZFFT_STAGE_SPLIT_MAX, false, st);
    count_launches(1);
    return cuda_check("k_split_cluster");
  }
#endif
  cudaMemsetAsync(SP.mu, 0, sizeof(unsigned long long) * 2 * SP.K * nb, st);
  prof_mark(pl, OZFFT_STAGE_SPLIT_MAX, true, st);
  for (int level = 0; level < SP.K; ++level) {
    if (pl.ts)
      k_split_max<true><<<grid, threads, 0, st>>>(SP, level);
    else
      k_split_max<false><<<grid, threads, 0, st>>>(SP, level);
  }
  prof_mark(pl, OZFFT_STAGE_SPLIT_MAX, false, st);
  prof_mark(pl, OZFFT_STAGE_SPLIT_DIGITS, true, st);
  if (pl.ts)
    k_split_digits<true><<<grid, threads, 0, st>>>(SP);
  else
    k_split_digits<false><<<grid, threads, 0, st>>>(SP);
  prof_mark(pl, OZFFT_STAGE_SPLIT_DIGITS, false, st);
  count_launches(SP.K + 1);
  return cuda_check("split kernels");
}

struct NttLaunch {
  int logCb;
  size_t col_smem;
  size_t col_fwd_smem;  // + staged step-1 twiddles
  int col_threads;
  size_t row_smem;
  int row_threads;
};
static NttLaunch ntt_launch_cfg(const Plan& pl) {
  NttLaunch c;
  c.logCb = col_logCb(pl.logR, pl.logC);
  c.col_smem = col_smem(pl.logR, c.logCb);
  c.col_fwd_smem = ((c.col_smem + 7) & ~(size_t)7) +
                   (OZ_CF_QLOOP && !pl.image ? 2 : 1) * ((size_t)1 << col_s1(pl.logR)) * ((size_t)1 << c.logCb) * 8;
  c.col_threads = col_threads(pl.logR, c.logCb);
  const size_t C = 1ull << pl.logC;
  const int rle = row_loge(pl.logC, pl.logR > 0);
  const size_t padC = C + (C >> rle) + 1;
  const size_t XS = pl.logR > 0 ? C + (C >> rle) + 4 : C;  // X row stride (k_row_fused)
  c.row_smem = ((size_t)pl.K * XS + padC + 2 * pl.K * pl.K * (1 + 2 * pl.L)) * sizeof(uint32_t);
  c.row_threads = pl.logC >= rle ? (1 << (pl.logC - rle)) : 1;  // exactly Tv: every thread active
  return c;
}

// Compile-time dispatch of the log2 sub-transform length (row: 0..12, column: 1..8).
template <int LO, int HI, class F>
static void dispatch_log(int v, F&& f) {
  if constexpr (LO <= HI) {
    if (v == LO)
      f(std::integral_constant<int, LO>{});
    else
      dispatch_log<LO + 1, HI>(v, f);
  }
}

// Compile-time dispatch of the two-pass decompositions this build instantiates (capi.cpp
// picks them): C = 2^11 with R = 2^2 .. 2^8 (m = 2^13 .. 2^19) and C = 2^12 with R = 2^7 ..
// 2^12 (m = 2^19 tuning knob, 2^20 .. 2^24).  f(R, C) receives integral constants.
template <int R, int C, class F>
static void dispatch_rc_(int logR, int logC, F& f) {
  if constexpr (C == 11 && R <= 8) {
    if (logR == R && logC == C) return f(std::integral_constant<int, R>{}, std::integral_constant<int, C>{});
    return dispatch_rc_<R + 1, C>(logR, logC, f);
  } else if constexpr (C == 11) {
    return dispatch_rc_<7, 12>(logR, logC, f);
  } else if constexpr (R <= 12) {
    if (logR == R && logC == C) return f(std::integral_constant<int, R>{}, std::integral_constant<int, C>{});
    return dispatch_rc_<R + 1, C>(logR, logC, f);
  }
}
template <class F>
static void dispatch_rc(int logR, int logC, F&& f) {
  dispatch_rc_<2, 11>(logR, logC, f);
}
bool decomposition_supported(int logR, int logC) {
  return (logC == 11 && logR >= 2 && logR <= 8) || (logC == 12 && logR >= 7 && logR <= 12);
}


static void launch_col_fwd(int logR, int logC, unsigned nblk, const NttLaunch& c, cudaStream_t st,
                           const ColParams& CP, bool zhi = false) {
  if (OZ_CF_QLOOP && !CP.image) nblk /= 2;  // both primes in one CTA
  dispatch_rc(logR, logC, [&](auto I, auto J) {
    if (CP.image && zhi) {
      set_smem(k_col_fwd<I.value, J.value, true, true>, c.col_fwd_smem);
      k_col_fwd<I.value, J.value, true, true><<<nblk, c.col_threads, c.col_fwd_smem, st>>>(CP);
    } else if (CP.image) {
      set_smem(k_col_fwd<I.value, J.value, true, false>, c.col_fwd_smem);
      k_col_fwd<I.value, J.value, true, false><<<nblk, c.col_threads, c.col_fwd_smem, st>>>(CP);
    } else if (zhi) {
      set_smem(k_col_fwd<I.value, J.value, false, true>, c.col_fwd_smem);
      k_col_fwd<I.value, J.value, false, true><<<nblk, c.col_threads, c.col_fwd_smem, st>>>(CP);
    } else {
      set_smem(k_col_fwd<I.value, J.value, false, false>, c.col_fwd_smem);
      k_col_fwd<I.value, J.value, false, false><<<nblk, c.col_threads, c.col_fwd_smem, st>>>(CP);
    }
  });
}
static void launch_col_inv(int logR, int logC, unsigned nblk, const NttLaunch& c, cudaStream_t st,
                           const ColParams& CP) {
  dispatch_rc(logR, logC, [&](auto I, auto J) {
    set_smem(k_col_inv<I.value, J.value>, c.col_smem);
    k_col_inv<I.value, J.value><<<nblk, c.col_threads, c.col_smem, st>>>(CP);
  });
}
static void launch_row(int logC, int logR, dim3 grid, const NttLaunch& c, cudaStream_t st,
                       const RowParams& RP) {
  if (logR > 0) {
    dispatch_log<11, 12>(logC, [&](auto I) {
      set_smem(k_row_fused<I.value, true>, c.row_smem);
      k_row_fused<I.value, true><<<grid, c.row_threads, c.row_smem, st>>>(RP);
    });
  } else {
    dispatch_log<0, 12>(logC, [&](auto I) {
      set_smem(k_row_fused<I.value, false>, c.row_smem);
      k_row_fused<I.value, false><<<grid, c.row_threads, c.row_smem, st>>>(RP);
    });
  }
}
static int row_s0(int logC, bool two_pass) {
  const int le = row_loge(logC, two_pass);
  return logC >= le ? le : logC;
}

// Forward NTT of digit vectors [nb][2][K][in_len] into internal-order spectra Xout
// [nb][2 q][2 a][K][m] (used at plan time for omega~*; the hot path fuses the row part).
static ozfft_status launch_forward_only(const Plan& pl, const int32_t* digits, int64_t in_len,
                                        const int32_t* stats, uint32_t* Y, uint32_t* Xout,
                                        int64_t nb, cudaStream_t st) {
  const NttLaunch c = ntt_launch_cfg(pl);
  const uint2* tw = reinterpret_cast<const uint2*>(pl.pers + pl.poff.tw);
  if (pl.logR > 0) {
    ColParams CP{};
    CP.logm = pl.logm; CP.logC = pl.logC; CP.logR = pl.logR; CP.logCb = c.logCb;
    CP.nb = nb; CP.K = pl.K; CP.L = pl.L; CP.p[0] = pl.p[0]; CP.p[1] = pl.p[1];
    CP.tw = tw; CP.digits = digits; CP.in_len = in_len; CP.Y = Y; CP.stats = stats;
    CP.unit_mask = 0xFF;
    CP.image = pl.image;
    fill_iota(pl, CP.io);
    const int64_t nblk = (1ll << (pl.logC - c.logCb)) * nb * 4;
    launch_col_fwd(pl.logR, pl.logC, (unsigned)nblk, c, st, CP);
  }
  RowParams RP{};
  RP.logm = pl.logm; RP.logC = pl.logC; RP.logR = pl.logR; RP.nb = nb; RP.K = pl.K; RP.L = pl.L;
  RP.p[0] = pl.p[0]; RP.p[1] = pl.p[1]; RP.tw = tw; RP.digits = digits; RP.in_len = in_len;
  RP.Y = Y; RP.stats = stats; RP.unit_mask = 0xFF; RP.fwd_only = 1; RP.Xout = Xout;
  RP.image = pl.image;
  fill_iota(pl, RP.io);
  dim3 grid((unsigned)nb, (unsigned)(4u << pl.logR));
  launch_row(pl.logC, pl.logR, grid, c, st, RP);
  return cuda_check("forward-only NTT");
}

ozfft_status launch_plan_precompute(Plan& pl, void* stream) {
  cudaStream_t st = (cudaStream_t)stream;
  const int64_t m = pl.m;
  const int K = pl.K;
  // scratch (plan time only): carved from the caller's workspace, which is free before the
  // first execute and sized for it (capi.cpp layout(): bind_scratch_bytes)
  uint8_t* sc = pl.ws;
  auto carve = [&](size_t bytes) {
    uint8_t* p = sc;
    sc += (bytes + 255) & ~(size_t)255;
    return p;
  };
  unsigned long long* mu = reinterpret_cast<unsigned long long*>(carve(sizeof(unsigned long long) * 2 * K));
  int32_t* digits = reinterpret_cast<int32_t*>(carve(sizeof(int32_t) * 2 * K * m));
  int32_t* stats = reinterpret_cast<int32_t*>(carve(sizeof(int32_t) * stats_stride(K)));
  uint32_t* Y = reinterpret_cast<uint32_t*>(carve(sizeof(uint32_t) * 4 * K * m));
  uint32_t* X = reinterpret_cast<uint32_t*>(carve(sizeof(uint32_t) * 4 * K * m));
  cudaMemsetAsync(X, 0, sizeof(uint32_t) * 4 * K * m, st);
  SplitParams SP{};
  SP.x = reinterpret_cast<const double2*>(pl.pers + pl.poff.W);  // wstar staged in the W area
  SP.chirp = nullptr;
  SP.len = m;
  SP.mode = 1;
  SP.K = K;
  SP.alpha = pl.alpha;
  SP.rho = pl.rho;
  SP.mu = mu;
  SP.digits = digits;
  SP.stats = stats;
  SP.sched = nullptr;
  SP.L = pl.L;
  SP.shared = pl.image;
  ozfft_status s = launch_split(pl, SP, 1, st);
  if (!s) s = launch_forward_only(pl, digits, m, stats, Y, X, 1, st);
  int32_t hstats[4 + 2 * kMaxK];
  if (!s) {
    cudaMemcpyAsync(hstats, stats, sizeof(int32_t) * stats_stride(K), cudaMemcpyDeviceToHost, st);
    if (cudaStreamSynchronize(st) != cudaSuccess) s = cuda_check("plan precompute");
  }
  if (!s) {
    if (hstats[2 + 2 * K] & 1) {
      set_error("omega~* split produced a non-finite value");
      s = OZFFT_ERR_CUDA;
    }
  }
  if (!s) {
    pl.kw[0] = hstats[0];
    pl.kw[1] = hstats[1];
    int32_t wsplit[2 + 2 * kMaxK] = {0};
    wsplit[0] = pl.kw[0];
    wsplit[1] = pl.kw[1];
    for (int v = 0; v < 2; ++v)
      for (int k = 0; k < K; ++k) {
        pl.Ew[v][k] = hstats[2 + v * K + k];
        wsplit[2 + v * K + k] = pl.Ew[v][k];
      }
    cudaMemcpyAsync(pl.pers + pl.poff.wsplit, wsplit, sizeof(int32_t) * (2 + 2 * K),
                    cudaMemcpyHostToDevice, st);
    k_w_finalize<<<592, 256, 0, st>>>(X, reinterpret_cast<uint32_t*>(pl.pers + pl.poff.W), K, m,
                                      pl.logC, row_s0(pl.logC, pl.logR > 0), pl.p[0], pl.p[1], pl.minv[0],
                                      pl.minv[1]);
    s = cuda_check("W finalize");
    if (!s && cudaStreamSynchronize(st) != cudaSuccess) s = cuda_check("plan precompute sync");
  }
  return s;
}

#ifndef OZ_SMALL_Z
#define OZ_SMALL_Z 4  // CTAs per (prime, part) of k_small_fused: clusters of 4 Z CTAs
#endif
// k_small_fused for one-pass plans in the default mode; OZFFT_ERR_UNSUPPORTED_LENGTH (no
// error recorded) when the plan is outside its range, so the caller takes the multi-kernel path.
static ozfft_status launch_small_fused(const Plan& pl, const ExecArgs& A, int32_t* stats, int32_t* sched,
                                       unsigned long long* mu, const double2* chirp, const uint2* tw,
                                       const uint32_t* W, const int32_t* wsplit, cudaStream_t st) {
  if (!pl.small_fused || pl.logR != 0 || pl.logC < 8 || pl.logC > 12 || pl.image || pl.ts)
    return OZFFT_ERR_UNSUPPORTED_LENGTH;
  const int Z = pl.small_z > 0 ? pl.small_z : OZ_SMALL_Z;
  const int slots = (2 * pl.K * pl.K + Z - 1) / Z;
  const size_t base = 4 * (small_head_words(pl.n, pl.K, pl.L) + small_union_words(pl.logC, pl.n, pl.K, slots));
  const size_t staged = base + 4 * small_stage_words(pl.logC, pl.K);
  const int stage = staged <= 200 * 1024 ? 1 : 0;
  const size_t smem = stage ? staged : base;
  if (smem > 200 * 1024) return OZFFT_ERR_UNSUPPORTED_LENGTH;
  SmallParams P{};
  P.x = reinterpret_cast<const double2*>(A.in);
  P.chirp = chirp;
  P.out = reinterpret_cast<double2*>(A.out);
  P.n = pl.n; P.K = pl.K; P.L = pl.L; P.alpha = pl.alpha; P.rho = pl.rho;
  P.conj = A.direction > 0 ? 1 : 0;
  P.direction = A.direction;
  P.p[0] = pl.p[0]; P.p[1] = pl.p[1]; P.pinv[0] = pl.pinv[0]; P.pinv[1] = pl.pinv[1];
  P.tw = tw; P.W = W; P.w_s0 = row_s0(pl.logC, false); P.wsplit = wsplit;
  fill_crt_consts(pl, P.F);
  P.mu = mu; P.stats = stats; P.sched = sched;
  P.Z = Z; P.slots = slots; P.stage = stage;
  P.fault = pl.fault;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3((unsigned)(4 * Z), (unsigned)A.nb);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = (unsigned)(4 * Z);
  at[0].val.clusterDim.y = 1;
  at[0].val.clusterDim.z = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  cudaError_t e = cudaSuccess;
  prof_mark(pl, OZFFT_STAGE_ROW_FUSED, true, st);
  dispatch_log<8, 12>(pl.logC, [&](auto I) {
    auto kern = stage ? k_small_fused<I.value, true> : k_small_fused<I.value, false>;
    cfg.blockDim = dim3((unsigned)small_threads(I.value));
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (4 * Z > 8) cudaFuncSetAttribute(kern, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
    e = cudaLaunchKernelEx(&cfg, kern, P);
  });
  prof_mark(pl, OZFFT_STAGE_ROW_FUSED, false, st);
  count_launches(1);
  if (e != cudaSuccess) {
    set_error(std::string("k_small_fused: ") + cudaGetErrorString(e));
    cudaGetLastError();
    return OZFFT_ERR_CUDA;
  }
  return cuda_check("k_small_fused");
}

ozfft_status launch_execute(const Plan& pl, const ExecArgs& A, void* stream) {
  cudaStream_t st = (cudaStream_t)stream;
  if (A.nb < 1 || A.ws0 < 0 || A.ws0 + A.nb > pl.chunk) {  // the chunked workspace regions
    set_error("internal: sub-batch does not fit the workspace chunk");
    return OZFFT_ERR_INVALID_ARGUMENT;
  }
  const int K = pl.K, L = pl.L, G = K * K;
  const int64_t nb = A.nb, m = pl.m, n = pl.n;
  uint8_t* ws = pl.ws;
  // per-batch stats and schedules live at the transform's global index
  int32_t* stats = reinterpret_cast<int32_t*>(ws + pl.woff.stats) + A.b0 * stats_stride(K);
  int32_t* sched = reinterpret_cast<int32_t*>(ws + pl.woff.sched) + A.b0 * 4 * sched_stride(K, L);
  // chunked per-transform regions, from workspace slot A.ws0
  const int64_t w0 = A.ws0;
  unsigned long long* mu = reinterpret_cast<unsigned long long*>(ws + pl.woff.mu) + w0 * 2 * K;
  int32_t* digits = reinterpret_cast<int32_t*>(ws + pl.woff.digits) + w0 * 2 * K * n;
  uint32_t* Y = reinterpret_cast<uint32_t*>(ws + pl.woff.Y) + w0 * 4 * K * m;
  uint32_t* Gb = reinterpret_cast<uint32_t*>(ws + pl.woff.G) + w0 * 8 * G * m;
  // residues: the workspace (stride K*K groups) or, for the unit-sharded single transform,
  // the caller's exchange buffer (stride A.res_groups = the schedule's max group count)
  uint32_t* res = A.res_out ? A.res_out : reinterpret_cast<uint32_t*>(ws + pl.woff.res) + w0 * 8 * G * n;
  const int rg = A.res_out ? A.res_groups : G;
  double2* Sdd = reinterpret_cast<double2*>(ws + pl.woff.S) + w0 * 4 * n;
  const uint2* tw = reinterpret_cast<const uint2*>(pl.pers + pl.poff.tw);
  const uint32_t* W = reinterpret_cast<const uint32_t*>(pl.pers + pl.poff.W);
  const double2* chirp = reinterpret_cast<const double2*>(pl.pers + pl.poff.chirp);
  const int32_t* wsplit = reinterpret_cast<const int32_t*>(pl.pers + pl.poff.wsplit);
  const ozfft_taps* taps = A.taps;

  if (A.phase == 0 && !taps && !A.res_out && A.unit_mask == 0xFFu && A.finish) {
    const ozfft_status fs = launch_small_fused(pl, A, stats, sched, mu, chirp, tw, W, wsplit, st);
    if (fs != OZFFT_ERR_UNSUPPORTED_LENGTH) return fs;  // else: the multi-kernel path
  }
  SplitParams SP{};
  SP.x = reinterpret_cast<const double2*>(A.in);
  SP.chirp = chirp;
  SP.len = n;
  SP.mode = 0;
  SP.conj = A.direction > 0 ? 1 : 0;
  SP.K = K;
  SP.alpha = pl.alpha;
  SP.rho = pl.rho;
  SP.mu = mu;
  SP.digits = taps && taps->digits ? reinterpret_cast<int32_t*>(taps->digits) : digits;
  SP.stats = stats;
  SP.sched = sched;
  SP.wsplit = wsplit;
  SP.L = L;
  SP.shared = pl.image;
  ozfft_status s = A.phase == 2 ? OZFFT_OK : launch_split(pl, SP, nb, st);
  if (s || A.phase == 1) return s;
  const NttLaunch c = ntt_launch_cfg(pl);
  uint32_t* Xtap = nullptr;
  uint32_t* Ztap = nullptr;
  if (taps && (taps->X || taps->Z)) {
    if (taps->X && cudaMalloc(&Xtap, sizeof(uint32_t) * nb * 4 * K * m)) return cuda_check("tap alloc");
    if (taps->Z && cudaMalloc(&Ztap, sizeof(uint32_t) * nb * 8 * G * m)) return cuda_check("tap alloc");
    if (Xtap) cudaMemsetAsync(Xtap, 0, sizeof(uint32_t) * nb * 4 * K * m, st);
    if (Ztap) cudaMemsetAsync(Ztap, 0, sizeof(uint32_t) * nb * 8 * G * m, st);
  }
  if (pl.logR > 0) {
    ColParams CP{};
    CP.logm = pl.logm; CP.logC = pl.logC; CP.logR = pl.logR; CP.logCb = c.logCb;
    CP.nb = nb; CP.K = K; CP.L = L; CP.p[0] = pl.p[0]; CP.p[1] = pl.p[1];
    CP.tw = tw; CP.digits = SP.digits; CP.in_len = n; CP.Y = Y; CP.stats = stats;
    CP.sched = sched; CP.G = Gb; CP.res = res; CP.rg = rg; CP.n = n; CP.unit_mask = A.unit_mask;
    CP.image = pl.image;
    CP.npeers = A.npeers;
    for (int r = 0; r < 8; ++r) CP.res_peers[r] = A.res_peers[r];
    fill_iota(pl, CP.io);
    const int64_t nblk = (1ll << (pl.logC - c.logCb)) * nb * 4;
    prof_mark(pl, OZFFT_STAGE_COL_FWD, true, st);
    launch_col_fwd(pl.logR, pl.logC, (unsigned)nblk, c, st, CP, OZ_COL_ZHI && 2 * n <= m);
    prof_mark(pl, OZFFT_STAGE_COL_FWD, false, st);
    count_launches(1);
    s = cuda_check("k_col_fwd");
    if (s) return s;
  }
  RowParams RP{};
  RP.logm = pl.logm; RP.logC = pl.logC; RP.logR = pl.logR; RP.nb = nb; RP.K = K; RP.L = L;
  RP.p[0] = pl.p[0]; RP.p[1] = pl.p[1]; RP.tw = tw; RP.digits = SP.digits; RP.in_len = n;
  RP.Y = Y; RP.W = W; RP.pinv[0] = pl.pinv[0]; RP.pinv[1] = pl.pinv[1]; RP.G = Gb; RP.res = res; RP.rg = rg; RP.n = n; RP.stats = stats; RP.sched = sched;
  RP.unit_mask = A.unit_mask; RP.fwd_only = 0; RP.Xout = Xtap; RP.Zout = Ztap;
  RP.npeers = A.npeers;
  for (int r = 0; r < 8; ++r) RP.res_peers[r] = A.res_peers[r];
  RP.image = pl.image;
  fill_iota(pl, RP.io);
  {
    dim3 grid((unsigned)nb, (unsigned)(4u << pl.logR));
    if (pl.logR == 0) {  // one-pass plan: split the (conv, group) items over gridDim.z
      const int64_t ctas = nb * 4;
      int64_t z = ctas < sm_count() ? sm_count() / ctas : 1;
      z = z > 2 * K * K ? 2 * K * K : (z < 1 ? 1 : z);
      grid.z = (unsigned)(z > OZ_ROW_ZMAX ? OZ_ROW_ZMAX : z);
    } else {
      // small batches of two-pass plans: split each row's (conv, group) items over z CTAs
      // (each recomputes the row's forward spectra) so that the grid fills more waves
      static const int zknob = [] {
        const char* t = std::getenv("OZFFT_ROW_Z");  // tuning knob (tools/)
        return t ? std::atoi(t) : 0;
      }();
      int64_t z = 1;
      if (zknob > 0) {
        z = zknob;
      } else {
        const int64_t ctas = nb * (4ll << pl.logR);
        while (z < 2 && ctas * z < (int64_t)OZ_ROW_Z_WAVES * sm_count() * OZ_ROW_MINB) z *= 2;
      }
      grid.z = (unsigned)(z > 2 * K * K ? 2 * K * K : z);
    }
    prof_mark(pl, OZFFT_STAGE_ROW_FUSED, true, st);
    launch_row(pl.logC, pl.logR, grid, c, st, RP);
    prof_mark(pl, OZFFT_STAGE_ROW_FUSED, false, st);
    count_launches(1);
    s = cuda_check("k_row_fused");
    if (s) return s;
    if (pl.fault && (A.unit_mask & 1u)) {  // test-only: unit (cv 0, prime 0), group 0, first word
      k_fault_inject<<<1, 1, 0, st>>>(pl.logR > 0 ? Gb : res, pl.logR > 0 ? m : n, sched);
      count_launches(1);
    }
  }
  // fused inverse column pass + CRT + DD accumulation (full transforms with R > 1)
  const bool fused = pl.logR > 0 && A.unit_mask == 0xFFu && A.finish;
  if (fused) {
    ColCrtParams XP{};
    XP.logm = pl.logm; XP.K = K; XP.L = L; XP.n = n; XP.nb = nb;
    fill_crt_consts(pl, XP.F);
    XP.tw = tw; XP.G = Gb; XP.sched = sched;
    XP.S = Sdd;
    XP.res_tap = taps && taps->res ? res : nullptr;
    XP.crt_tap = taps ? reinterpret_cast<int64_t*>(taps->crt) : nullptr;
    const int cle = col_loge(pl.logR);
    const int lcb = pl.image ? col_log_cb_img(pl.logR, pl.logC) : col_log_cb_ci(pl.logR, pl.logC, 2 * n <= m);
    const int threads = col_threads(pl.logR, lcb);
    const size_t tile = ((1ull << pl.logR) + ((1ull << pl.logR) >> cle) + 1) * (1ull << lcb);
    const bool prune = 2 * n <= m;  // padded plans; cyclic plans (m = n) need every row
    const int nh = (pl.logR >= cle ? (1 << cle) : (1 << pl.logR)) / (prune ? 2 : 1);
    const size_t smem = ((tile + 3) & ~(size_t)3) * 4 * (!pl.image && OZ_CI_DB ? 2 : 1) +
                        (!pl.image && (ci_racc(nh) || ci_gacc(nh)) ? 0 : (size_t)nh * threads * 16 * (pl.image ? 2 : 1)) +
                        (!pl.image && OZ_CI_T0S && pl.logR >= OZ_CI_T0S
                             ? (size_t)2 * ((size_t)1 << col_s1(pl.logR)) * ((size_t)1 << lcb) * 8 : 0);
    const int64_t nblk = (1ll << (pl.logC - lcb)) * nb * (pl.image ? 1 : 4);
    prof_mark(pl, OZFFT_STAGE_COL_INV, true, st);
    dispatch_rc(pl.logR, pl.logC, [&](auto I, auto J) {
      {
        if (pl.image && prune) {
          set_smem(k_col_inv_crt_img<I.value, J.value, true>, smem);
          k_col_inv_crt_img<I.value, J.value, true><<<(unsigned)nblk, threads, smem, st>>>(XP);
        } else if (pl.image) {
          set_smem(k_col_inv_crt_img<I.value, J.value, false>, smem);
          k_col_inv_crt_img<I.value, J.value, false><<<(unsigned)nblk, threads, smem, st>>>(XP);
        } else if (prune && pl.ts) {
          set_smem(k_col_inv_crt<I.value, J.value, true, true>, smem);
          k_col_inv_crt<I.value, J.value, true, true><<<(unsigned)nblk, threads, smem, st>>>(XP);
        } else if (pl.ts) {
          set_smem(k_col_inv_crt<I.value, J.value, false, true>, smem);
          k_col_inv_crt<I.value, J.value, false, true><<<(unsigned)nblk, threads, smem, st>>>(XP);
        } else if (prune) {
          set_smem(k_col_inv_crt<I.value, J.value, true, false>, smem);
          k_col_inv_crt<I.value, J.value, true, false><<<(unsigned)nblk, threads, smem, st>>>(XP);
        } else {
          set_smem(k_col_inv_crt<I.value, J.value, false, false>, smem);
          k_col_inv_crt<I.value, J.value, false, false><<<(unsigned)nblk, threads, smem, st>>>(XP);
        }
      }
    });
    prof_mark(pl, OZFFT_STAGE_COL_INV, false, st);
    count_launches(1);
    s = cuda_check("k_col_inv_crt");
    if (s) return s;
    dim3 grid((unsigned)((n + 255) / 256), (unsigned)nb);
    prof_mark(pl, OZFFT_STAGE_CRT_FINISH, true, st);
    k_finish_dd<<<grid, 256, 0, st>>>(XP.S, stats, K, chirp, reinterpret_cast<double2*>(A.out), n,
                                      A.direction, pl.image, pl.ts);
    prof_mark(pl, OZFFT_STAGE_CRT_FINISH, false, st);
    count_launches(1);
    s = cuda_check("k_finish_dd");
    if (s) return s;
  }
  if (pl.logR > 0 && !fused) {
    ColParams CP{};
    CP.logm = pl.logm; CP.logC = pl.logC; CP.logR = pl.logR; CP.logCb = c.logCb;
    CP.nb = nb; CP.K = K; CP.L = L; CP.p[0] = pl.p[0]; CP.p[1] = pl.p[1];
    CP.tw = tw; CP.stats = stats; CP.sched = sched; CP.G = Gb; CP.res = res; CP.rg = rg; CP.n = n;
    CP.unit_mask = A.unit_mask;
    CP.npeers = A.npeers;
    for (int r = 0; r < 8; ++r) CP.res_peers[r] = A.res_peers[r];
    const int64_t nblk = (1ll << (pl.logC - c.logCb)) * nb * 8;
    prof_mark(pl, OZFFT_STAGE_COL_INV, true, st);
    launch_col_inv(pl.logR, pl.logC, (unsigned)nblk, c, st, CP);
    prof_mark(pl, OZFFT_STAGE_COL_INV, false, st);
    count_launches(1);
    s = cuda_check("k_col_inv");
    if (s) return s;
  }
  if (A.finish && !fused) {
    FinishParams FP{};
    FP.n = n; FP.nb = nb; FP.K = K; FP.L = L; fill_crt_consts(pl, FP); FP.res = res; FP.rg = rg; FP.stats = stats; FP.sched = sched;
    FP.chirp = chirp; FP.out = reinterpret_cast<double2*>(A.out); FP.direction = A.direction;
    FP.crt_tap = taps ? reinterpret_cast<int64_t*>(taps->crt) : nullptr;
    dim3 grid((unsigned)((n + 255) / 256), (unsigned)nb);
    const dim3 grid4((unsigned)((n + kFinishCols - 1) / kFinishCols), (unsigned)nb);
    prof_mark(pl, OZFFT_STAGE_CRT_FINISH, true, st);
    if (pl.image)
      k_crt_finish_img<<<grid, 256, 0, st>>>(FP);
    else if (pl.ts)
      k_crt_finish_ts<<<grid, 256, 0, st>>>(FP);
    else
      k_crt_finish<<<grid4, 256, 0, st>>>(FP);
    prof_mark(pl, OZFFT_STAGE_CRT_FINISH, false, st);
    count_launches(1);
    s = cuda_check("k_crt_finish");
    if (s) return s;
  }
  // ---- taps (test only): convert internal orders to the oracle's natural layouts
  if (taps) {
    std::vector<int64_t> off;
    std::vector<uint32_t> vp, vm;
    // per-vector constants: m (undo m^-1 folded into W) and m 2^-32 (Montgomery W~)
    uint32_t mconst[2], mmont[2];
    for (int q = 0; q < 2; ++q) {
      const uint64_t pq = pl.p[q];
      mconst[q] = (uint32_t)((uint64_t)m % pq);
      uint64_t inv2_32 = 1;  // 2^-32 mod p = (2^-1)^32
      const uint64_t half = (pq + 1) / 2;
      for (int i = 0; i < 32; ++i) inv2_32 = inv2_32 * half % pq;
      mmont[q] = (uint32_t)((uint64_t)mconst[q] * inv2_32 % pq);
    }
    auto run_perm = [&](const uint32_t* src, void* dst, bool mult, bool rowperm) -> ozfft_status {
      int64_t* doff = nullptr;
      uint32_t *dvp = nullptr, *dvm = nullptr;
      const int64_t nvec = (int64_t)off.size();
      cudaMalloc(&doff, sizeof(int64_t) * nvec);
      cudaMalloc(&dvp, sizeof(uint32_t) * nvec);
      cudaMalloc(&dvm, sizeof(uint32_t) * nvec);
      cudaMemcpyAsync(doff, off.data(), sizeof(int64_t) * nvec, cudaMemcpyHostToDevice, st);
      cudaMemcpyAsync(dvp, vp.data(), sizeof(uint32_t) * nvec, cudaMemcpyHostToDevice, st);
      if (mult) cudaMemcpyAsync(dvm, vm.data(), sizeof(uint32_t) * nvec, cudaMemcpyHostToDevice, st);
      k_tap_permute<<<1184, 256, 0, st>>>(src, reinterpret_cast<uint32_t*>(dst), nvec, pl.logm,
                                          doff, dvp, mult ? dvm : nullptr, rowperm ? pl.logC : -1,
                                          row_s0(pl.logC, pl.logR > 0));
      cudaStreamSynchronize(st);
      cudaFree(doff);
      cudaFree(dvp);
      cudaFree(dvm);
      vm.clear();
      return cuda_check("tap permute");
    };
    if (taps->X) {  // src [b][q][a][s][m] -> dst [b][a][s][q][m]
      off.clear(); vp.clear();
      for (int64_t b = 0; b < nb; ++b)
        for (int q = 0; q < 2; ++q)
          for (int a = 0; a < 2; ++a)
            for (int s2 = 0; s2 < K; ++s2) {
              off.push_back((((b * 2 + a) * K + s2) * 2 + q) * m);
              vp.push_back(pl.p[q]);
            }
      s = run_perm(Xtap, taps->X, false, false);
      if (s) return s;
    }
    if (taps->Z) {  // src [b][q][cv][g][m] (W m^-1 scaled) -> dst [b][cv][g][q][m] (times m)
      off.clear(); vp.clear();
      for (int64_t b = 0; b < nb; ++b)
        for (int q = 0; q < 2; ++q)
          for (int cv = 0; cv < 4; ++cv)
            for (int g = 0; g < G; ++g) {
              off.push_back((((b * 4 + cv) * G + g) * 2 + q) * m);
              vp.push_back(pl.p[q]);
              vm.push_back(mconst[q]);
            }
      s = run_perm(Ztap, taps->Z, true, false);
      if (s) return s;
    }
    if (taps->res) {  // [b][cv][q][g][n] -> [b][cv][g][q][n]
      for (int64_t b = 0; b < nb; ++b)
        for (int cv = 0; cv < 4; ++cv)
          for (int q = 0; q < 2; ++q)
            for (int g = 0; g < G; ++g)
              cudaMemcpyAsync(reinterpret_cast<uint32_t*>(taps->res) + (((b * 4 + cv) * G + g) * 2 + q) * n,
                              res + (((b * 4 + cv) * 2 + q) * G + g) * n, sizeof(uint32_t) * n,
                              cudaMemcpyDeviceToDevice, st);
    }
    if (taps->sched)
      cudaMemcpyAsync(taps->sched, sched, sizeof(int32_t) * nb * 4 * sched_stride(K, L),
                      cudaMemcpyDeviceToDevice, st);
    if (taps->W) {  // src W~ [q][b][t][m] (W m^-1 2^32) -> [b][t][q][m] times m 2^-32
      off.clear(); vp.clear();
      for (int q = 0; q < 2; ++q)
        for (int bw = 0; bw < 2; ++bw)
          for (int t = 0; t < K; ++t) {
            off.push_back(((bw * K + t) * 2 + q) * m);
            vp.push_back(pl.p[q]);
            vm.push_back(mmont[q]);
          }
      s = run_perm(W, taps->W, true, true);
      if (s) return s;
    }
    if (taps->E || taps->kv) {
      std::vector<int32_t> hs((size_t)nb * stats_stride(K));
      cudaMemcpyAsync(hs.data(), stats, sizeof(int32_t) * hs.size(), cudaMemcpyDeviceToHost, st);
      cudaStreamSynchronize(st);
      std::vector<int32_t> hE((size_t)nb * 2 * K), hk((size_t)nb * 2);
      for (int64_t b = 0; b < nb; ++b) {
        const int32_t* r = hs.data() + b * stats_stride(K);
        hk[b * 2] = r[0];
        hk[b * 2 + 1] = r[1];
        for (int i = 0; i < 2 * K; ++i) hE[b * 2 * K + i] = r[2 + i];
      }
      if (taps->E) cudaMemcpyAsync(taps->E, hE.data(), sizeof(int32_t) * hE.size(), cudaMemcpyHostToDevice, st);
      if (taps->kv) cudaMemcpyAsync(taps->kv, hk.data(), sizeof(int32_t) * hk.size(), cudaMemcpyHostToDevice, st);
      cudaStreamSynchronize(st);
    }
    cudaStreamSynchronize(st);
    if (Xtap) cudaFree(Xtap);
    if (Ztap) cudaFree(Ztap);
    s = cuda_check("taps");
  }
  return s;
}

ozfft_status launch_finish_from_residues(const Plan& pl, const uint32_t* res, int groups, double* out,
                                         int direction, void* stream) {
  cudaStream_t st = (cudaStream_t)stream;
  FinishParams FP{};
  FP.n = pl.n; FP.nb = 1; FP.K = pl.K; FP.L = pl.L; fill_crt_consts(pl, FP); FP.res = res; FP.rg = groups;
  FP.stats = reinterpret_cast<const int32_t*>(pl.ws + pl.woff.stats);
  FP.sched = reinterpret_cast<const int32_t*>(pl.ws + pl.woff.sched);
  FP.chirp = reinterpret_cast<const double2*>(pl.pers + pl.poff.chirp);
  FP.out = reinterpret_cast<double2*>(out);
  FP.direction = direction;
  dim3 grid((unsigned)((pl.n + 255) / 256), 1);
  const dim3 grid4((unsigned)((pl.n + kFinishCols - 1) / kFinishCols), 1);
  prof_mark(pl, OZFFT_STAGE_CRT_FINISH, true, st);
  int nl = 1;
  if (pl.ts) {
    k_crt_finish_ts<<<grid, 256, 0, st>>>(FP);
  } else if (pl.logR > 0) {  // long transforms: 8 DD chains per thread, then the combine
    double2* S = reinterpret_cast<double2*>(pl.ws + pl.woff.S);
    const dim3 gdd((unsigned)((pl.n + 256 * kCrtDDPer - 1) / (256 * kCrtDDPer)), 4);
    k_crt_dd<<<gdd, 256, 0, st>>>(FP, S);
    k_finish_dd<<<grid, 256, 0, st>>>(S, FP.stats, pl.K, FP.chirp, FP.out, pl.n, direction, 0, 0);
    nl = 2;
  } else {
    k_crt_finish<<<grid4, 256, 0, st>>>(FP);
  }
  prof_mark(pl, OZFFT_STAGE_CRT_FINISH, false, st);
  count_launches(nl);
  return cuda_check("k_crt_finish (shard)");
}

}  // namespace ozfft
