/*
 * ozfft_oracle.c -- TEST INFRASTRUCTURE ONLY.
 *
 * A plain, slow, obviously-correct CPU implementation of the hot path of
 * arXiv 2603.29129 (Kawakami & Takahashi, "Computing FFTs at Target Precision
 * Using Lower-Precision FFTs"): an fp64 Bluestein DFT whose cyclic convolution
 * is Ozaki-split into integer slices, convolved exactly with two-prime 32-bit
 * NTTs, accumulated in the NTT domain and reconstructed with Garner's CRT.
 *
 * Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / reference
 * leg may load this library.  The product path (paper_2603_29129_b200/) never
 * links, imports or calls it, and this file shares no code, header, table or
 * constant generator with the CUDA path.
 *
 * Citation convention: "P:N" = /root/reference/PAPER.md line N (with section /
 * equation / algorithm), "S:N" = SPEC.md line N, "SURVEY O<k>" / "ruling <k>" =
 * SURVEY.md section 8(c), whose readings are restated in DESIGN.md.
 *
 * Every float step is a fixed sequence of IEEE-754 binary64 round-to-nearest
 * operations (compile with -ffp-contract=off, no fast-math); fma() only where
 * written.  Integers use uint64 "% p" -- no Montgomery, no Shoup, no lazy
 * reduction -- so a reader can check each line against the paper.
 *
 * Parity status of each function (pins live in tests/test_oracle_*.py):
 *   orc_alpha          pinned: paper-printed alpha values
 *   orc_chirp          pinned: mpmath 200-bit correctly-rounded table + closed forms
 *   orc_premul         pinned: exact-rational DD error bound (Fraction)
 *   orc_split          pinned: exact reconstruction, |D| <= 2^alpha, k-bound
 *   orc_ntt            pinned: O(m^2) definition eq:ntt / eq:intt in Python big ints
 *   orc_garner2        pinned: S:183-185 examples, exhaustive (7,11), random big-int CRT
 *   orc_schedule       pinned: paper transform counts 52/64/96
 *   integer core       pinned: brute-force integer cyclic convolution of the digits
 *   orc_execute        pinned: __float128 direct DFT, closed forms, Parseval, linearity
 *   final fp64 bits    the DD op sequence is this build's contract; the
 *                      paper fixes only the [1e-16,1e-15] error band ->
 *                      "parity unpinned" at the bit level, pinned in error band.
 *   cyclic plans (f1)  pinned: brute-force integer cyclic convolution of length n, and
 *                      bitwise equality with the padded plans
 *   orc_split_shared,  pinned: brute-force complex integer convolution, the iota ring
 *   orc_execute_image  homomorphism, the alpha bound, counts 12+20, float128 (f2)
 *   orc_ts_*           pinned: exact rationals -- conversions exact, TSAdd/TSMul relative
 *                      error <= 2^-62 (f4; the algorithms are this build's reading,
 *                      DESIGN ruling 24, so their exact bits are unpinned by the paper)
 *   orc_split_ts       pinned: |D| <= 2^alpha, reconstruction within the last unit
 *   orc_execute (TS)   pinned: float128 error band, 64 NTTs at phi = 0
 */
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#include <math.h>
#include <quadmath.h>

#define ORC_MAXK 8
#define ORC_MAXL 8

typedef __int128 i128;

/* ------------------------------------------------------------------------- */
/* O0. Constants and modular arithmetic (P:142-149 symmetric remainder;      */
/*     P:244-264 NTT over Z_p; values of p0, p1 at P:1046).                  */
/* ------------------------------------------------------------------------- */

/* a mod m with minimum absolute value: a - m*floor(a/m + 1/2) */
int64_t orc_sym_mod(int64_t a, int64_t m) {
  /* floor(a/m + 1/2) = floor((2a + m) / (2m)) computed exactly in 128 bits */
  i128 num = (i128)2 * a + m, den = (i128)2 * m;
  i128 q = num / den;
  if ((num % den != 0) && ((num < 0) != (den < 0))) q -= 1; /* floor */
  return (int64_t)((i128)a - (i128)m * q);
}

static uint32_t mulmod(uint32_t a, uint32_t b, uint32_t p) {
  return (uint32_t)(((uint64_t)a * (uint64_t)b) % p);
}
static uint32_t addmod(uint32_t a, uint32_t b, uint32_t p) {
  return (uint32_t)(((uint64_t)a + (uint64_t)b) % p);
}
uint32_t orc_powmod(uint32_t a, uint64_t e, uint32_t p) {
  uint32_t r = 1 % p;
  a %= p;
  while (e) {
    if (e & 1) r = mulmod(r, a, p);
    a = mulmod(a, a, p);
    e >>= 1;
  }
  return r;
}
/* inverse by Fermat (p prime) */
uint32_t orc_invmod(uint32_t a, uint32_t p) { return orc_powmod(a, (uint64_t)p - 2, p); }

int orc_is_prime(uint64_t p) {
  if (p < 2) return 0;
  for (uint64_t d = 2; d * d <= p; d++)
    if (p % d == 0) return 0;
  return 1;
}

/* smallest primitive root of prime p: g with g^((p-1)/q) != 1 for every prime q | p-1 */
uint32_t orc_primitive_root(uint32_t p) {
  uint64_t f[64];
  int nf = 0;
  uint64_t r = (uint64_t)p - 1;
  for (uint64_t d = 2; d * d <= r; d++)
    if (r % d == 0) {
      f[nf++] = d;
      while (r % d == 0) r /= d;
    }
  if (r > 1) f[nf++] = r;
  for (uint32_t g = 2; g < p; g++) {
    int ok = 1;
    for (int i = 0; i < nf && ok; i++)
      if (orc_powmod(g, ((uint64_t)p - 1) / f[i], p) == 1) ok = 0;
    if (ok) return g;
  }
  return 0;
}

/* primitive m-th root of unity: g^((p-1)/m), m | p-1 (S:62-70 convention) */
uint32_t orc_root_of_unity(uint32_t p, uint64_t m) {
  return orc_powmod(orc_primitive_root(p), ((uint64_t)p - 1) / m, p);
}

/* alpha = floor((log2(p0 p1 / 2) - log2(L n)) / 2)   (accumulation-aware
 * form of eq:ozaki-scheme-conv-ntt-crt-alpha).  Evaluated exactly:
 * the largest integer a with 2*L*n*4^a < p0*p1.  Returns 0 if no a >= 1 works. */
int orc_alpha(int64_t n, int64_t L, uint32_t p0, uint32_t p1) {
  i128 P = (i128)p0 * p1;
  int a = 0;
  while (a < 62) {
    i128 lhs = (i128)2 * L * n;
    int ok = 1;
    for (int i = 0; i < a + 1; i++) {
      lhs *= 4;
      if (lhs >= P) { ok = 0; break; }
    }
    if (!ok) break;
    a++;
  }
  return a;
}

/* Garner's algorithm for two primes (Alg.8), symmetric as in
 * returns the unique v in [-p0p1/2, p0p1/2) with v = z0 mod p0 and
 * v = z1 mod p1.  *fix is set if the final range map changed the value (never
 * expected; ruling 13). */
int64_t orc_garner2(uint32_t z0, uint32_t z1, uint32_t p0, uint32_t p1, int* fix) {
  uint32_t inv = orc_invmod(p0 % p1, p1); /* p0^{-1} mod p1 */
  int64_t z0s = orc_sym_mod((int64_t)z0, (int64_t)p0);
  int64_t d = ((int64_t)z1 - z0s) % (int64_t)p1;
  if (d < 0) d += p1;
  uint32_t t = mulmod((uint32_t)d, inv, p1);
  int64_t ts = orc_sym_mod((int64_t)t, (int64_t)p1);
  i128 v = (i128)z0s + (i128)ts * p0;
  i128 P = (i128)p0 * p1;
  i128 w = v;
  /* unique representative in [-P/2, P/2):  w in [-P/2, P/2) <=> 2w in [-P, P) */
  while (2 * w >= P) w -= P;
  while (2 * w < -P) w += P;
  if (fix) *fix = (w != v);
  return (int64_t)w;
}

/* ------------------------------------------------------------------------- */
/* O5/O7. NTT and inverse NTT (eq:ntt, eq:intt).                  */
/* Plain iterative radix-2 Cooley-Tukey: bit-reverse permutation, then        */
/* butterflies; natural order in and out, canonical residues [0,p).          */
/* ------------------------------------------------------------------------- */
void orc_ntt(uint32_t* a, int64_t m, uint32_t p, int inverse) {
  if (m <= 1) return;
  /* bit-reversal permutation */
  for (int64_t i = 1, j = 0; i < m; i++) {
    int64_t bit = m >> 1;
    for (; j & bit; bit >>= 1) j ^= bit;
    j ^= bit;
    if (i < j) { uint32_t t = a[i]; a[i] = a[j]; a[j] = t; }
  }
  uint32_t w = orc_root_of_unity(p, (uint64_t)m);
  if (inverse) w = orc_invmod(w, p);
  for (int64_t len = 2; len <= m; len <<= 1) {
    uint32_t wlen = orc_powmod(w, (uint64_t)(m / len), p); /* primitive len-th root */
    for (int64_t i = 0; i < m; i += len) {
      uint32_t wj = 1;
      for (int64_t j = 0; j < len / 2; j++) {
        uint32_t u = a[i + j];
        uint32_t v = mulmod(a[i + j + len / 2], wj, p);
        a[i + j] = addmod(u, v, p);
        a[i + j + len / 2] = addmod(u, p - v, p);
        wj = mulmod(wj, wlen, p);
      }
    }
  }
  if (inverse) {
    uint32_t minv = orc_invmod((uint32_t)(m % p), p); /* n^{-1} of eq:intt */
    for (int64_t i = 0; i < m; i++) a[i] = mulmod(a[i], minv, p);
  }
}

/* ------------------------------------------------------------------------- */
/* O1. Chirp omega(j) = omega_{2n}^{j^2} as fp64 (C_j, S_j):          */
/*     C_j = RN(cos(pi r/n)), S_j = RN(-sin(pi r/n)), r = j^2 mod 2n (ruling 3)*/
/* ------------------------------------------------------------------------- */
void orc_chirp(int64_t n, double* C, double* S) {
  for (int64_t j = 0; j < n; j++) {
    int64_t r = (int64_t)(((i128)j * j) % (2 * (i128)n));
    double c, s;
    if (r == 0) { c = 1.0; s = 0.0; }
    else if (2 * r == n) { c = 0.0; s = -1.0; }        /* angle pi/2 */
    else if (r == n) { c = -1.0; s = 0.0; }            /* angle pi   */
    else if (2 * r == 3 * n) { c = 0.0; s = 1.0; }     /* angle 3pi/2 */
    else {
      __float128 th = M_PIq * ((__float128)r / (__float128)n);
      c = (double)cosq(th);
      s = (double)(-sinq(th));
    }
    C[j] = c;
    S[j] = s;
  }
}

/* ------------------------------------------------------------------------- */
/* O3. Double-double error-free transformations.                             */
/*   FastTwoSum: Alg.7 (Dekker 1971).  TwoSum: Knuth.  TwoProd by   */
/*   FMA.  DDAdd is the "accurate" double-double addition (Hida et al. 2001,  */
/*   cited at P:416); TS of the paper is replaced by DD (ruling 1).           */
/* ------------------------------------------------------------------------- */
static void two_prod(double a, double b, double* p, double* e) {
  double pp = a * b;
  *e = fma(a, b, -pp);
  *p = pp;
}
static void two_sum(double a, double b, double* s, double* e) {
  double ss = a + b;
  double bb = ss - a;
  *e = (a - (ss - bb)) + (b - bb);
  *s = ss;
}
static void fast_two_sum(double a, double b, double* s, double* e) {
  double ss = a + b;
  *e = b - (ss - a);
  *s = ss;
}
static void dd_add(double ah, double al, double bh, double bl, double* rh, double* rl) {
  double s, e, t, f;
  two_sum(ah, bh, &s, &e);
  two_sum(al, bl, &t, &f);
  e = e + t;
  fast_two_sum(s, e, &s, &e);
  e = e + f;
  fast_two_sum(s, e, &s, &e);
  *rh = s;
  *rl = e;
}
/* DD times double: (p,e) = TwoProd(A.hi, b); e = fma(A.lo, b, e); FastTwoSum */
static void dd_mul_d(double ah, double al, double b, double* rh, double* rl) {
  double p, e;
  two_prod(ah, b, &p, &e);
  e = fma(al, b, e);
  fast_two_sum(p, e, rh, rl);
}

/* Alg.4 step 2: x' = x (.) omega in DD.
 * conj != 0 conjugates x on load (inverse-direction wrapper, O10). */
void orc_premul(int64_t n, const double* x /* interleaved complex */, const double* C,
                const double* S, int conj, double* hre, double* lre, double* him, double* lim) {
  for (int64_t j = 0; j < n; j++) {
    double xr = x[2 * j], xi = conj ? -x[2 * j + 1] : x[2 * j + 1];
    double p1, e1, p2, e2;
    two_prod(xr, C[j], &p1, &e1);
    two_prod(xi, S[j], &p2, &e2);
    dd_add(p1, e1, -p2, -e2, &hre[j], &lre[j]);
    two_prod(xr, S[j], &p1, &e1);
    two_prod(xi, C[j], &p2, &e2);
    dd_add(p1, e1, p2, e2, &him[j], &lim[j]);
  }
}

/* ------------------------------------------------------------------------- */
/* O4. Ozaki split, Alg.6 SplitTSAndCalcNTT (eqs) with   */
/* u = 2^-53 (DD working precision, ruling 1), rho = 53 - alpha,*/
/* capped at K levels.  Level k:                                  */
/*   mu = max|hi|; stop if 0;  E = ceil(log2 mu) exactly (ruling 8);          */
/*   sigma = 2^(E+rho);  d = fl(fl(hi + sigma) - sigma)      */
/*   D = d * 2^(alpha-E)  (c = (u sigma)^-1)  -> int32 digit           */
/*   (hi, lo) = FastTwoSum(fl(hi - d), lo)      */
/* Returns the number of levels k; -1 if mu is not finite (ruling 18).        */
/* digits is [K][len]; E[k] receives E_k (scale exponent s_k = alpha - E_k).   */
/* ------------------------------------------------------------------------- */
static int ceil_log2_exact(double mu) {
  int e;
  double f = frexp(mu, &e); /* mu = f 2^e, f in [1/2, 1) */
  return (f == 0.5) ? e - 1 : e;
}
int orc_split(int64_t len, double* hi, double* lo, int alpha, int K, int32_t* digits,
              int32_t* E) {
  const int rho = 53 - alpha;
  int k;
  for (k = 0; k < K; k++) {
    double mu = 0.0;
    for (int64_t j = 0; j < len; j++) {
      double a = fabs(hi[j]);
      if (a > mu || a != a) mu = a; /* a NaN sticks in mu */
    }
    if (!isfinite(mu)) return -1;
    if (mu == 0.0) break;
    int Ek = ceil_log2_exact(mu);
    double sigma = ldexp(1.0, Ek + rho);
    double scale = ldexp(1.0, alpha - Ek);
    E[k] = Ek;
    for (int64_t j = 0; j < len; j++) {
      double t = hi[j] + sigma;
      double d = t - sigma;
      digits[(int64_t)k * len + j] = (int32_t)(d * scale);
      double r = hi[j] - d;
      fast_two_sum(r, lo[j], &hi[j], &lo[j]);
    }
  }
  return k;
}

/* ------------------------------------------------------------------------- */
/* O-TS. Triple-single (TS) working precision.  */
/* A TS number is x0 + x1 + x2 with fp32 words, |x_s| <= ulp(x_{s-1})/2.  The  */
/* paper cites TS arithmetic (Fabiano et al.) without giving TSAdd / TSMul;     */
/* the sequences below are this build's reading (DESIGN ruling 24): error-free */
/* TwoSum / FastTwoSum / FMA TwoProd on fp32 words, a fixed rounded tail, then */
/* Renorm3.  Their accuracy (relative error <= 2^-62) is pinned against exact  */
/* rationals in tests/test_oracle_ts.py.  Every op is a single fp32 RN op; the */
/* file is compiled with -ffp-contract=off.                                    */
/* ------------------------------------------------------------------------- */
typedef struct { float x0, x1, x2; } orc_ts;

static void two_sum_f(float a, float b, float* s, float* e) {
  *s = a + b;
  float bb = *s - a;
  *e = (a - (*s - bb)) + (b - bb);
}
static void fast_two_sum_f(float a, float b, float* s, float* e) {
  *s = a + b;
  *e = b - (*s - a);
}
static void two_prod_f(float a, float b, float* p, float* e) {
  *p = a * b;
  *e = fmaf(a, b, -*p);
}
/* Renorm3: (a, b, c) with a the leading term -> non-overlapping triple */
static orc_ts ts_renorm3(float a, float b, float c) {
  float s, t3, s0, t2, s1, s2;
  two_sum_f(b, c, &s, &t3);
  two_sum_f(a, s, &s0, &t2);
  two_sum_f(t2, t3, &s1, &s2);
  fast_two_sum_f(s0, s1, &s0, &s1);
  fast_two_sum_f(s1, s2, &s1, &s2);
  orc_ts r = {s0, s1, s2};
  return r;
}
/* TS(d): exact for finite d inside the normal fp32 range (53 <= 72 bits) */
orc_ts orc_ts_from_double(double d) {
  orc_ts r;
  r.x0 = (float)d;
  double t = d - (double)r.x0;
  r.x1 = (float)t;
  t = t - (double)r.x1;
  r.x2 = (float)t;
  return r;
}
/* TS(v) for |v| < 2^62: exact (24 + 24 + 14 bits) */
orc_ts orc_ts_from_int64(int64_t v) {
  orc_ts r;
  r.x0 = (float)v;
  int64_t t = v - (int64_t)r.x0;
  r.x1 = (float)t;
  t = t - (int64_t)r.x1;
  r.x2 = (float)t;
  return r;
}
/* fl64(x0 + x1 + x2): x1 + x2 is exact in binary64, one rounding at the end */
double orc_ts_to_double(orc_ts a) { return (double)a.x0 + ((double)a.x1 + (double)a.x2); }
orc_ts orc_ts_add(orc_ts a, orc_ts b) {
  float s0, e0, s1, e1, t1, f1;
  two_sum_f(a.x0, b.x0, &s0, &e0);
  two_sum_f(a.x1, b.x1, &s1, &e1);
  const float s2 = a.x2 + b.x2;
  two_sum_f(e0, s1, &t1, &f1);
  const float t2 = (f1 + e1) + s2;
  return ts_renorm3(s0, t1, t2);
}
orc_ts orc_ts_neg(orc_ts a) {
  orc_ts r = {-a.x0, -a.x1, -a.x2};
  return r;
}
orc_ts orc_ts_mul(orc_ts a, orc_ts b) {
  float p0, q0, p1, q1, p2, q2, s1, r1, t1, r2;
  two_prod_f(a.x0, b.x0, &p0, &q0);
  two_prod_f(a.x0, b.x1, &p1, &q1);
  two_prod_f(a.x1, b.x0, &p2, &q2);
  const float c = ((((a.x0 * b.x2) + (a.x1 * b.x1)) + (a.x2 * b.x0)) + q1) + q2;
  two_sum_f(p1, p2, &s1, &r1);
  two_sum_f(q0, s1, &t1, &r2);
  const float t2 = (r1 + r2) + c;
  return ts_renorm3(p0, t1, t2);
}
/* exact scaling by 2^e (no overflow / underflow on this path's ranges) */
static orc_ts ts_ldexp(orc_ts a, int e) {
  orc_ts r = {ldexpf(a.x0, e), ldexpf(a.x1, e), ldexpf(a.x2, e)};
  return r;
}
static int ts_finite(orc_ts a) { return isfinite(a.x0) && isfinite(a.x1) && isfinite(a.x2); }

/* x' = x (.) omega in TS (Alg.4 TS form, P:473-474 with TS ops): TS(x) and
 * TS(omega) from the binary64 values, TSSub / TSAdd of TSMul products. */
void orc_premul_ts(int64_t n, const double* x, const double* C, const double* S, int conj,
                   float* re /* [3][n] */, float* im /* [3][n] */) {
  for (int64_t j = 0; j < n; j++) {
    const orc_ts xr = orc_ts_from_double(x[2 * j]);
    const orc_ts xi = orc_ts_from_double(conj ? -x[2 * j + 1] : x[2 * j + 1]);
    const orc_ts c = orc_ts_from_double(C[j]), sn = orc_ts_from_double(S[j]);
    const orc_ts r = orc_ts_add(orc_ts_mul(xr, c), orc_ts_neg(orc_ts_mul(xi, sn)));
    const orc_ts i = orc_ts_add(orc_ts_mul(xr, sn), orc_ts_mul(xi, c));
    re[j] = r.x0; re[n + j] = r.x1; re[2 * n + j] = r.x2;
    im[j] = i.x0; im[n + j] = i.x1; im[2 * n + j] = i.x2;
  }
}

/* TS split, Alg. SplitTSAndCalcNTT literally: rho = 24 - alpha (u32 = 2^-24),
 * mu = ||r0||_inf, sigma = 2^(ceil(log2 mu) + rho), x = fl32(fl32(r0 + sigma) - sigma),
 * (r0, r1) <- FastTwoSum(fl32(r0 - x), r1), then (r1, r2) <- FastTwoSum(r1, r2) with the
 * r1 just produced (ruling 25), D = x c with c = (u32 sigma)^-1 = 2^(alpha - E).
 * r is [3][len] (r0, r1, r2); digits [K][len]; returns levels, -1 if non-finite. */
int orc_split_ts(int64_t len, float* r, int alpha, int K, int32_t* digits, int32_t* E) {
  const int rho = 24 - alpha;
  float* r0 = r;
  float* r1 = r + len;
  float* r2 = r + 2 * len;
  int k;
  for (k = 0; k < K; k++) {
    double mu = 0.0;
    for (int64_t j = 0; j < len; j++) {
      double a = fabs((double)r0[j]);
      if (a > mu || a != a) mu = a;
    }
    for (int64_t j = 0; j < len; j++)
      if (!isfinite(r1[j]) || !isfinite(r2[j])) mu = NAN;
    if (!isfinite(mu)) return -1;
    if (mu == 0.0) break;
    const int Ek = ceil_log2_exact(mu);
    const float sigma = ldexpf(1.0f, Ek + rho);
    const float scale = ldexpf(1.0f, alpha - Ek);
    E[k] = Ek;
    for (int64_t j = 0; j < len; j++) {
      const float t = r0[j] + sigma;
      const float x = t - sigma;
      digits[(int64_t)k * len + j] = (int32_t)(x * scale);
      const float d = r0[j] - x;
      float a, b;
      fast_two_sum_f(d, r1[j], &a, &b);
      r0[j] = a;
      fast_two_sum_f(b, r2[j], &r1[j], &r2[j]);
    }
  }
  return k;
}

/* Image mode (beyond the paper): Alg.6 applied to the complex vector
 * with ONE exponent per level shared by both parts -- mu = max_j max(|hi_re|, |hi_im|),
 * then the same sigma and scale for both parts, each part stepping exactly as orc_split.
 * digits is [2 parts][K][len]; returns the common level count (or -1, non-finite). */
int orc_split_shared(int64_t len, double* hre, double* lre, double* him, double* lim, int alpha,
                     int K, int32_t* digits, int32_t* E) {
  const int rho = 53 - alpha;
  int k;
  for (k = 0; k < K; k++) {
    double mu = 0.0;
    for (int64_t j = 0; j < len; j++) {
      double a = fabs(hre[j]), b = fabs(him[j]);
      if (a > mu || a != a) mu = a;
      if (b > mu || b != b) mu = b;
    }
    if (!isfinite(mu)) return -1;
    if (mu == 0.0) break;
    int Ek = ceil_log2_exact(mu);
    double sigma = ldexp(1.0, Ek + rho);
    double scale = ldexp(1.0, alpha - Ek);
    E[k] = Ek;
    for (int part = 0; part < 2; part++) {
      double* hi = part ? him : hre;
      double* lo = part ? lim : lre;
      int32_t* D = digits + ((int64_t)part * K + k) * len;
      for (int64_t j = 0; j < len; j++) {
        double t = hi[j] + sigma;
        double d = t - sigma;
        D[j] = (int32_t)(d * scale);
        double r = hi[j] - d;
        fast_two_sum(r, lo[j], &hi[j], &lo[j]);
      }
    }
  }
  return k;
}

/* ------------------------------------------------------------------------- */
/* O6. Alg.8 flush schedule (literally).  For one real convolution  */
/* with kx slices of scale exponents sx[] and ky slices with sy[]:             */
/*   c <- c_x^(kx-1) c_y^(ky-1); l <- 0    */
/*   for k = kx+ky-2 .. 0: for s = max(0,k-ky+1) .. min(kx-1,k): t = k - s    */
/*     if l >= L or c != c_x^(s) c_y^(t): flush group (scale c); reset        */
/*     append (s,t); l++                                                      */
/*   flush last group                                                         */
/* Scales are powers of two c = 2^(sx+sy), so equality compares exponents.    */
/* Output layout (int32): [0] = ngroups; group g at 1 + g*(2+2L):              */
/*   cexp, npairs, s0, t0, s1, t1, ...   (slots for K*K groups)               */
/* ------------------------------------------------------------------------- */
int orc_sched_stride(int K, int L) { return 1 + K * K * (2 + 2 * L); }

int orc_schedule(int kx, const int32_t* sx, int ky, const int32_t* sy, int K, int L,
                 int32_t* out) {
  int stride = orc_sched_stride(K, L);
  for (int i = 0; i < stride; i++) out[i] = 0;
  if (kx <= 0 || ky <= 0) return 0; /* empty vector: the convolution is 0 (ruling 11) */
  int ng = 0;
  int32_t c = sx[kx - 1] + sy[ky - 1];
  int l = 0;
  int32_t* g = out + 1;
  g[0] = c;
  g[1] = 0;
  for (int k = kx + ky - 2; k >= 0; k--) {
    int s0 = k - ky + 1 > 0 ? k - ky + 1 : 0;
    int s1 = kx - 1 < k ? kx - 1 : k;
    for (int s = s0; s <= s1; s++) {
      int t = k - s;
      int32_t e = sx[s] + sy[t];
      if (l >= L || c != e) {
        ng++; /* flush: group closed with scale exponent c */
        g = out + 1 + ng * (2 + 2 * L);
        c = e;
        l = 0;
        g[0] = c;
        g[1] = 0;
      }
      g[2 + 2 * l] = s;
      g[3 + 2 * l] = t;
      g[1] = l + 1;
      l++;
    }
  }
  ng++;
  out[0] = ng;
  return ng;
}

/* ------------------------------------------------------------------------- */
/* Plan: everything that does not depend on the input (P:1038 precompute).    */
/* ------------------------------------------------------------------------- */
typedef struct {
  int64_t n, m;
  int K, L, alpha;
  uint32_t p[2];
  double *C, *S;        /* chirp [n] */
  int32_t* wdig;        /* omega~* digits [2 parts][K][m] */
  int32_t Ew[2][ORC_MAXK];
  int kw[2];
  uint32_t* W;          /* [2 parts][K][2 primes][m], natural order; image mode: [2 images] */
  int status;
  int image;            /* 1: complex-image accumulation, see orc_execute_image */
  int ts;               /* 1: triple-single working precision for a1, a2, a7 */
  uint32_t iota[2];     /* image mode: iota_q = g_q^((p_q - 1)/4), iota^2 = -1 mod p_q */
} orc_plan;

typedef struct {
  int32_t* digits; /* [2][K][n]            split digits of Re x', Im x'          */
  int32_t* E;      /* [2][K]               level exponents E_k                   */
  int32_t* kv;     /* [2]                  levels of Re x', Im x'                */
  uint32_t* X;     /* [2][K][2][m]         forward NTTs, natural order           */
  int32_t* sched;  /* [4][stride]          Alg.8 groups per real conv            */
  uint32_t* Z;     /* [4][K*K][2][m]       NTT-domain accumulated groups         */
  uint32_t* res;   /* [4][K*K][2][n]       inverse NTT outputs j < n             */
  int64_t* crt;    /* [4][K*K][n]          Garner integers                       */
  double* xdd;     /* [4][n]               hi_re, lo_re, hi_im, lo_im of x'      */
  int64_t* counts; /* [3]                  runtime fwd NTTs, inv NTTs, cached    */
  int32_t* flags;  /* [1]                  1 = non-finite input, 2 = CRT fix     */
} orc_taps;

static int64_t pow2_ceil(int64_t v) {
  int64_t m = 1;
  while (m < v) m <<= 1;
  return m;
}

void orc_plan_destroy(orc_plan* pl) {
  if (!pl) return;
  free(pl->C);
  free(pl->S);
  free(pl->wdig);
  free(pl->W);
  free(pl);
}

/* Bluestein length (Alg.4 Require): cyclic == 0 -> m = 2^ceil(log2(2n-1)) >= 2n-1
 * (north star).  cyclic == 1 -> m = n for a power-of-two n: "the convolution in
 * eq:bluestein_convolution becomes a cyclic convolution; therefore, zero-padding is
 * unnecessary and the FFT length N can be kept equal to n".  The ZeroPad_pm
 * formula below then reduces to omega~*(j) = omega*(j), j < n (its two ranges coincide
 * because omega*(n - j) = omega*(j) for even n). */
orc_plan* orc_plan_create_ts(int64_t n, int K, int L, uint32_t p0, uint32_t p1, int cyclic,
                             int image, int ts);
orc_plan* orc_plan_create_ex(int64_t n, int K, int L, uint32_t p0, uint32_t p1, int cyclic,
                             int image) {
  return orc_plan_create_ts(n, K, L, p0, p1, cyclic, image, 0);
}
orc_plan* orc_plan_create_ts(int64_t n, int K, int L, uint32_t p0, uint32_t p1, int cyclic,
                             int image, int ts) {
  if (n < 1 || K < 1 || K > ORC_MAXK || L < 1 || L > ORC_MAXL) return NULL;
  if (ts && image) return NULL; /* TS precision is built for the paper's real mode only */
  if (cyclic && (n & (n - 1))) return NULL;
  if (image && ((p0 & 3u) != 1u || (p1 & 3u) != 1u)) return NULL; /* need iota, p = 1 mod 4 */
  orc_plan* pl = (orc_plan*)calloc(1, sizeof(orc_plan));
  pl->n = n;
  pl->m = cyclic ? n : pow2_ceil(2 * n - 1);
  pl->K = K;
  pl->L = L;
  pl->p[0] = p0;
  pl->p[1] = p1;
  pl->image = image;
  pl->ts = ts;
  /* n = DFT length (ruling 2).  Image mode: a real output of a group sums up to L n
   * complex products, |Re(ab)| <= |ar br| + |ai bi| <= 2 4^alpha, so the bound is
   * 2 L n 4^alpha < P/2, i.e. the real-mode alpha at 2n. */
  pl->alpha = orc_alpha(image ? 2 * n : n, L, p0, p1);
  if (image)
    for (int q = 0; q < 2; q++) pl->iota[q] = orc_root_of_unity(pl->p[q], 4);
  int64_t m = pl->m;
  pl->C = (double*)malloc(sizeof(double) * n);
  pl->S = (double*)malloc(sizeof(double) * n);
  orc_chirp(n, pl->C, pl->S);
  /* omega~* = ZeroPad_pm(omega*, m): omega*(j) = (C_j, -S_j) */
  double* hre = (double*)calloc(m, sizeof(double));
  double* him = (double*)calloc(m, sizeof(double));
  double* lre = (double*)calloc(m, sizeof(double));
  double* lim = (double*)calloc(m, sizeof(double));
  for (int64_t j = 0; j < m; j++) {
    int64_t src = -1;
    if (j < n) src = j;
    else if (j >= m - n + 1) src = m - j;
    if (src >= 0) {
      hre[j] = pl->C[src];
      him[j] = -pl->S[src];
    }
  }
  /* -S of +0.0 is -0.0: zeros compare equal and split identically */
  pl->wdig = (int32_t*)calloc((size_t)2 * K * m, sizeof(int32_t));
  if (image) {
    pl->kw[0] = pl->kw[1] = orc_split_shared(m, hre, lre, him, lim, pl->alpha, K, pl->wdig,
                                             pl->Ew[0]);
    for (int k = 0; k < K; k++) pl->Ew[1][k] = pl->Ew[0][k];
  } else if (ts) { /* TS(omega~*) from the binary64 table (Alg.4 TS form, step 1) */
    float* r = (float*)malloc(sizeof(float) * 3 * m);
    for (int part = 0; part < 2; part++) {
      const double* h = part ? him : hre;
      for (int64_t j = 0; j < m; j++) {
        const orc_ts t = orc_ts_from_double(h[j]);
        r[j] = t.x0; r[m + j] = t.x1; r[2 * m + j] = t.x2;
      }
      pl->kw[part] = orc_split_ts(m, r, pl->alpha, K, pl->wdig + (size_t)part * K * m, pl->Ew[part]);
    }
    free(r);
  } else {
    pl->kw[0] = orc_split(m, hre, lre, pl->alpha, K, pl->wdig, pl->Ew[0]);
    pl->kw[1] = orc_split(m, him, lim, pl->alpha, K, pl->wdig + (size_t)K * m, pl->Ew[1]);
  }
  free(hre); free(him); free(lre); free(lim);
  if (image) { /* W images: NTT(Dre + iota Dim) (b = 0) and NTT(Dre - iota Dim) (b = 1) */
    pl->W = (uint32_t*)calloc((size_t)2 * K * 2 * m, sizeof(uint32_t));
    for (int b = 0; b < 2; b++)
      for (int t = 0; t < pl->kw[0]; t++)
        for (int q = 0; q < 2; q++) {
          const uint32_t p = pl->p[q];
          const uint32_t io = b ? p - pl->iota[q] : pl->iota[q];
          uint32_t* dst = pl->W + (((size_t)b * K + t) * 2 + q) * m;
          const int32_t* Dr = pl->wdig + (size_t)t * m;
          const int32_t* Di = pl->wdig + ((size_t)K + t) * m;
          for (int64_t j = 0; j < m; j++) {
            uint32_t r = Dr[j] >= 0 ? (uint32_t)Dr[j] : (uint32_t)((int64_t)Dr[j] + p);
            uint32_t i = Di[j] >= 0 ? (uint32_t)Di[j] : (uint32_t)((int64_t)Di[j] + p);
            dst[j] = addmod(r, mulmod(io, i, p), p);
          }
          orc_ntt(dst, m, p, 0);
        }
    return pl;
  }
  /* the 4K forward NTTs of the omega~* slices, computed once */
  pl->W = (uint32_t*)calloc((size_t)2 * K * 2 * m, sizeof(uint32_t));
  for (int b = 0; b < 2; b++)
    for (int t = 0; t < pl->kw[b]; t++)
      for (int q = 0; q < 2; q++) {
        uint32_t* dst = pl->W + (((size_t)b * K + t) * 2 + q) * m;
        const int32_t* D = pl->wdig + ((size_t)b * K + t) * m;
        for (int64_t j = 0; j < m; j++) /* canonical lift (ruling 5) */
          dst[j] = D[j] >= 0 ? (uint32_t)D[j] : (uint32_t)((int64_t)D[j] + pl->p[q]);
        orc_ntt(dst, m, pl->p[q], 0);
      }
  return pl;
}

orc_plan* orc_plan_create_conv(int64_t n, int K, int L, uint32_t p0, uint32_t p1, int cyclic) {
  return orc_plan_create_ex(n, K, L, p0, p1, cyclic, 0);
}
orc_plan* orc_plan_create(int64_t n, int K, int L, uint32_t p0, uint32_t p1) {
  return orc_plan_create_ex(n, K, L, p0, p1, 0, 0);
}

int64_t orc_plan_m(const orc_plan* pl) { return pl->m; }
int orc_plan_alpha(const orc_plan* pl) { return pl->alpha; }
void orc_plan_wsplit(const orc_plan* pl, int32_t* kw, int32_t* Ew) {
  kw[0] = pl->kw[0];
  kw[1] = pl->kw[1];
  for (int b = 0; b < 2; b++)
    for (int k = 0; k < pl->K; k++) Ew[b * pl->K + k] = pl->Ew[b][k];
}
void orc_plan_copy(const orc_plan* pl, double* C, double* S, int32_t* wdig, uint32_t* W) {
  int64_t n = pl->n, m = pl->m;
  int K = pl->K;
  if (C) memcpy(C, pl->C, sizeof(double) * n);
  if (S) memcpy(S, pl->S, sizeof(double) * n);
  if (wdig) memcpy(wdig, pl->wdig, sizeof(int32_t) * 2 * K * m);
  if (W) memcpy(W, pl->W, sizeof(uint32_t) * 2 * K * 2 * m);
}

/* ------------------------------------------------------------------------- */
/* One transform: Alg.4 steps with Alg.8 as the convolution.    */
/* dir = -1 forward (omega_n = e^{-2 pi i/n}); +1 inverse = conj(F(conj(y)))/n */
/* (O10, ruling 16).                                                          */
/* Returns 0, or 1 if the input was non-finite (output all NaN, ruling 18).   */
/* ------------------------------------------------------------------------- */
/* ------------------------------------------------------------------------- */
/* Image mode (builds on P:916-938; beyond the  */
/* paper).  The complex digit vectors D = Dre + i Dim (shared exponents, above)   */
/* and Dw of omega~* are convolved as complex integers.  Since iota^2 = -1 mod p, */
/* a -> a+ = ar + iota ai and a -> a- = ar - iota ai are ring homomorphisms of     */
/* Z[i] -> Z_p, so (D (*) Dw)+- = D+- (*) Dw+-: two modular cyclic convolutions    */
/* (images) replace the four real ones.  Per Alg.8 group and image:               */
/*   Z+-_g = sum_(s,t) NTT(D+-_s) (.) W+-_t,  z+-_g = NTT^-1(Z+-_g)               */
/* then per prime  re = (z+ + z-) / 2,  im = (z+ - z-) / (2 iota)  (mod p), Garner */
/* on each across the primes, and the DD sums of re 2^-c and im 2^-c in flush     */
/* order give y' directly.  Forward: 2 images x k slices x 2 primes; inverse:     */
/* 2 images x groups x 2 primes (32 runtime NTTs at (K, L) = (3, 3) vs 52).       */
/* Taps: digits / E / kv as the real mode (E and kv repeated per part); X[img];  */
/* sched row 0 (rows 1-3 zero); Z[img], res[img]; crt row 0 = Re, row 1 = Im.    */
/* ------------------------------------------------------------------------- */
static int orc_execute_image(const orc_plan* pl, const double* x, double* y, int dir,
                             orc_taps* tp) {
  const int64_t n = pl->n, m = pl->m;
  const int K = pl->K, L = pl->L, alpha = pl->alpha;
  const int stride = orc_sched_stride(K, L);
  const int G = K * K;
  int flags = 0;
  int64_t nfwd = 0, ninv = 0;
  double* hr = (double*)malloc(sizeof(double) * n);
  double* lr = (double*)malloc(sizeof(double) * n);
  double* hi = (double*)malloc(sizeof(double) * n);
  double* li = (double*)malloc(sizeof(double) * n);
  orc_premul(n, x, pl->C, pl->S, dir > 0, hr, lr, hi, li);
  if (tp && tp->xdd) {
    memcpy(tp->xdd, hr, sizeof(double) * n);
    memcpy(tp->xdd + n, lr, sizeof(double) * n);
    memcpy(tp->xdd + 2 * n, hi, sizeof(double) * n);
    memcpy(tp->xdd + 3 * n, li, sizeof(double) * n);
  }
  int32_t* dig = (int32_t*)calloc((size_t)2 * K * n, sizeof(int32_t));
  int32_t Ex[ORC_MAXK] = {0};
  const int kx = orc_split_shared(n, hr, lr, hi, li, alpha, K, dig, Ex);
  free(hr); free(lr); free(hi); free(li);
  if (kx < 0) {
    flags |= 1;
    for (int64_t j = 0; j < 2 * n; j++) y[j] = NAN;
    if (tp && tp->flags) tp->flags[0] = flags;
    free(dig);
    return 1;
  }
  if (tp && tp->digits) memcpy(tp->digits, dig, sizeof(int32_t) * 2 * K * n);
  if (tp && tp->E)
    for (int a = 0; a < 2; a++)
      for (int k = 0; k < K; k++) tp->E[a * K + k] = k < kx ? Ex[k] : 0;
  if (tp && tp->kv) { tp->kv[0] = kx; tp->kv[1] = kx; }
  /* forward NTTs of the digit images */
  uint32_t* X = (uint32_t*)calloc((size_t)2 * K * 2 * m, sizeof(uint32_t));
  for (int img = 0; img < 2; img++)
    for (int s = 0; s < kx; s++)
      for (int q = 0; q < 2; q++) {
        const uint32_t p = pl->p[q];
        const uint32_t io = img ? p - pl->iota[q] : pl->iota[q];
        uint32_t* dst = X + (((size_t)img * K + s) * 2 + q) * m;
        const int32_t* Dr = dig + (size_t)s * n;
        const int32_t* Di = dig + ((size_t)K + s) * n;
        for (int64_t j = 0; j < m; j++) {
          int64_t vr = j < n ? Dr[j] : 0, vi = j < n ? Di[j] : 0;
          uint32_t r = vr >= 0 ? (uint32_t)vr : (uint32_t)(vr + p);
          uint32_t i = vi >= 0 ? (uint32_t)vi : (uint32_t)(vi + p);
          dst[j] = addmod(r, mulmod(io, i, p), p);
        }
        orc_ntt(dst, m, p, 0);
        nfwd++;
      }
  free(dig);
  if (tp && tp->X) memcpy(tp->X, X, sizeof(uint32_t) * 2 * K * 2 * m);
  int32_t sx[ORC_MAXK], sw[ORC_MAXK];
  for (int k = 0; k < K; k++) {
    sx[k] = alpha - Ex[k];
    sw[k] = alpha - pl->Ew[0][k];
  }
  int32_t* sched = (int32_t*)malloc(sizeof(int32_t) * stride);
  const int ng = orc_schedule(kx, sx, pl->kw[0], sw, K, L, sched);
  if (tp && tp->sched) {
    memset(tp->sched, 0, sizeof(int32_t) * 4 * stride);
    memcpy(tp->sched, sched, sizeof(int32_t) * stride);
  }
  /* (2 iota)^-1 and 2^-1 per prime */
  uint32_t inv2[2], inv2i[2];
  for (int q = 0; q < 2; q++) {
    inv2[q] = orc_invmod(2, pl->p[q]);
    inv2i[q] = orc_invmod(mulmod(2, pl->iota[q], pl->p[q]), pl->p[q]);
  }
  double* acc = (double*)calloc((size_t)4 * n, sizeof(double)); /* DD re, DD im */
  uint32_t* Zg = (uint32_t*)malloc(sizeof(uint32_t) * 4 * m);    /* [img][q][m] */
  for (int g = 0; g < ng; g++) {
    const int32_t* gr = sched + 1 + g * (2 + 2 * L);
    const int32_t cexp = gr[0], np = gr[1];
    for (int img = 0; img < 2; img++)
      for (int q = 0; q < 2; q++) {
        uint32_t* Zq = Zg + ((size_t)img * 2 + q) * m;
        for (int64_t i = 0; i < m; i++) Zq[i] = 0;
        for (int e = 0; e < np; e++) {
          const int s = gr[2 + 2 * e], t = gr[3 + 2 * e];
          const uint32_t* Xs = X + (((size_t)img * K + s) * 2 + q) * m;
          const uint32_t* Wt = pl->W + (((size_t)img * K + t) * 2 + q) * m;
          for (int64_t i = 0; i < m; i++)
            Zq[i] = addmod(Zq[i], mulmod(Xs[i], Wt[i], pl->p[q]), pl->p[q]);
        }
        if (tp && tp->Z)
          memcpy(tp->Z + (((size_t)img * G + g) * 2 + q) * m, Zq, sizeof(uint32_t) * m);
        orc_ntt(Zq, m, pl->p[q], 1);
        ninv++;
        if (tp && tp->res)
          memcpy(tp->res + (((size_t)img * G + g) * 2 + q) * n, Zq, sizeof(uint32_t) * n);
      }
    const double scale = ldexp(1.0, -cexp);
    for (int64_t j = 0; j < n; j++) {
      uint32_t zr[2], zi[2];
      for (int q = 0; q < 2; q++) {
        const uint32_t p = pl->p[q];
        const uint32_t zp = Zg[((size_t)0 * 2 + q) * m + j], zm = Zg[((size_t)1 * 2 + q) * m + j];
        zr[q] = mulmod(addmod(zp, zm, p), inv2[q], p);
        zi[q] = mulmod(addmod(zp, p - zm, p), inv2i[q], p);
      }
      for (int part = 0; part < 2; part++) {
        int fix = 0;
        const int64_t Zj = part ? orc_garner2(zi[0], zi[1], pl->p[0], pl->p[1], &fix)
                                : orc_garner2(zr[0], zr[1], pl->p[0], pl->p[1], &fix);
        if (fix) flags |= 2;
        if (tp && tp->crt) tp->crt[((size_t)part * G + g) * n + j] = Zj;
        double h = (double)Zj;
        double l = (double)(Zj - (int64_t)h);
        dd_add(acc[(part * 2) * n + j], acc[(part * 2 + 1) * n + j], h * scale, l * scale,
               &acc[(part * 2) * n + j], &acc[(part * 2 + 1) * n + j]);
      }
    }
  }
  free(Zg); free(sched); free(X);
  for (int64_t j = 0; j < n; j++) {
    const double yrh = acc[j], yrl = acc[n + j], yih = acc[2 * n + j], yil = acc[3 * n + j];
    double a1h, a1l, a2h, a2l, o_re, o_im, tmp;
    dd_mul_d(yrh, yrl, pl->C[j], &a1h, &a1l);
    dd_mul_d(yih, yil, pl->S[j], &a2h, &a2l);
    dd_add(a1h, a1l, -a2h, -a2l, &o_re, &tmp);
    dd_mul_d(yrh, yrl, pl->S[j], &a1h, &a1l);
    dd_mul_d(yih, yil, pl->C[j], &a2h, &a2l);
    dd_add(a1h, a1l, a2h, a2l, &o_im, &tmp);
    if (dir > 0) {
      o_re = o_re / (double)n;
      o_im = -o_im / (double)n;
    }
    y[2 * j] = o_re;
    y[2 * j + 1] = o_im;
  }
  free(acc);
  if (tp && tp->counts) {
    tp->counts[0] = nfwd;
    tp->counts[1] = ninv;
    tp->counts[2] = 4 * (int64_t)pl->kw[0];
  }
  if (tp && tp->flags) tp->flags[0] = flags;
  return 0;
}

int orc_execute(const orc_plan* pl, const double* x, double* y, int dir, orc_taps* tp) {
  if (pl->image) return orc_execute_image(pl, x, y, dir, tp);
  const int64_t n = pl->n, m = pl->m;
  const int K = pl->K, L = pl->L, alpha = pl->alpha;
  const int stride = orc_sched_stride(K, L);
  const int G = K * K;
  int flags = 0;
  int64_t nfwd = 0, ninv = 0;

  /* Alg.6 on Re x' and Im x' (split caching) */
  int32_t* dig = (int32_t*)calloc((size_t)2 * K * n, sizeof(int32_t));
  int32_t Ex[2][ORC_MAXK] = {{0}};
  int kx[2];
  if (pl->ts) { /* TS working precision (f4): Alg.4 TS steps 1-2, TS split */
    float* tre = (float*)malloc(sizeof(float) * 3 * n);
    float* tim = (float*)malloc(sizeof(float) * 3 * n);
    orc_premul_ts(n, x, pl->C, pl->S, dir > 0, tre, tim);
    kx[0] = orc_split_ts(n, tre, alpha, K, dig, Ex[0]);
    kx[1] = orc_split_ts(n, tim, alpha, K, dig + (size_t)K * n, Ex[1]);
    free(tre); free(tim);
  } else {
    double* hr = (double*)malloc(sizeof(double) * n);
    double* lr = (double*)malloc(sizeof(double) * n);
    double* hi = (double*)malloc(sizeof(double) * n);
    double* li = (double*)malloc(sizeof(double) * n);
    /* step 2 of Alg.4: x' = x (.) omega */
    orc_premul(n, x, pl->C, pl->S, dir > 0, hr, lr, hi, li);
    if (tp && tp->xdd) {
      memcpy(tp->xdd, hr, sizeof(double) * n);
      memcpy(tp->xdd + n, lr, sizeof(double) * n);
      memcpy(tp->xdd + 2 * n, hi, sizeof(double) * n);
      memcpy(tp->xdd + 3 * n, li, sizeof(double) * n);
    }
    kx[0] = orc_split(n, hr, lr, alpha, K, dig, Ex[0]);
    kx[1] = orc_split(n, hi, li, alpha, K, dig + (size_t)K * n, Ex[1]);
    free(hr); free(lr); free(hi); free(li);
  }
  if (kx[0] < 0 || kx[1] < 0) {
    flags |= 1;
    for (int64_t j = 0; j < 2 * n; j++) y[j] = NAN;
    if (tp && tp->flags) tp->flags[0] = flags;
    free(dig);
    return 1;
  }
  if (tp && tp->digits) memcpy(tp->digits, dig, sizeof(int32_t) * 2 * K * n);
  if (tp && tp->E)
    for (int a = 0; a < 2; a++)
      for (int k = 0; k < K; k++) tp->E[a * K + k] = k < kx[a] ? Ex[a][k] : 0;
  if (tp && tp->kv) { tp->kv[0] = kx[0]; tp->kv[1] = kx[1]; }

  /* forward NTTs of the x' slices under both primes (Alg.6) */
  uint32_t* X = (uint32_t*)calloc((size_t)2 * K * 2 * m, sizeof(uint32_t));
  for (int a = 0; a < 2; a++)
    for (int s = 0; s < kx[a]; s++)
      for (int q = 0; q < 2; q++) {
        uint32_t* dst = X + (((size_t)a * K + s) * 2 + q) * m;
        const int32_t* D = dig + ((size_t)a * K + s) * n;
        for (int64_t j = 0; j < m; j++) { /* ZeroPad(x', m), canonical lift */
          int64_t v = j < n ? D[j] : 0;
          dst[j] = v >= 0 ? (uint32_t)v : (uint32_t)(v + pl->p[q]);
        }
        orc_ntt(dst, m, pl->p[q], 0);
        nfwd++;
      }
  free(dig);
  if (tp && tp->X) memcpy(tp->X, X, sizeof(uint32_t) * 2 * K * 2 * m);

  /* scale exponents s = alpha - E (c = 2^s) */
  int32_t sx[2][ORC_MAXK], sw[2][ORC_MAXK];
  for (int a = 0; a < 2; a++)
    for (int k = 0; k < K; k++) {
      sx[a][k] = alpha - Ex[a][k];
      sw[a][k] = alpha - pl->Ew[a][k];
    }

  /* four real convolutions: rr, ii, ir, ri as (x part, w part) */
  static const int conv_a[4] = {0, 1, 1, 0};
  static const int conv_b[4] = {0, 1, 0, 1};
  double* acc = (double*)calloc((size_t)4 * 2 * n, sizeof(double)); /* DD per conv */
  orc_ts* tacc = pl->ts ? (orc_ts*)calloc((size_t)4 * n, sizeof(orc_ts)) : NULL; /* TS per conv */
  int32_t* sched = (int32_t*)malloc(sizeof(int32_t) * stride);
  uint32_t* Zg = (uint32_t*)malloc(sizeof(uint32_t) * 2 * m);
  for (int cv = 0; cv < 4; cv++) {
    const int a = conv_a[cv], b = conv_b[cv];
    int ng = orc_schedule(kx[a], sx[a], pl->kw[b], sw[b], K, L, sched);
    if (tp && tp->sched) memcpy(tp->sched + cv * stride, sched, sizeof(int32_t) * stride);
    for (int g = 0; g < ng; g++) {
      const int32_t* gr = sched + 1 + g * (2 + 2 * L);
      const int32_t cexp = gr[0], np = gr[1];
      /* Z'_q = sum over the group's pairs of X_q^(s) (.) Y_q^(t) mod p_q (lines 981-982) */
      for (int q = 0; q < 2; q++) {
        uint32_t* Zq = Zg + (size_t)q * m;
        for (int64_t i = 0; i < m; i++) Zq[i] = 0;
        for (int e = 0; e < np; e++) {
          const int s = gr[2 + 2 * e], t = gr[3 + 2 * e];
          const uint32_t* Xs = X + (((size_t)a * K + s) * 2 + q) * m;
          const uint32_t* Wt = pl->W + (((size_t)b * K + t) * 2 + q) * m;
          for (int64_t i = 0; i < m; i++)
            Zq[i] = addmod(Zq[i], mulmod(Xs[i], Wt[i], pl->p[q]), pl->p[q]);
        }
        if (tp && tp->Z)
          memcpy(tp->Z + (((size_t)cv * G + g) * 2 + q) * m, Zq, sizeof(uint32_t) * m);
        orc_ntt(Zq, m, pl->p[q], 1); /* line 973 / 986 */
        ninv++;
        if (tp && tp->res)
          memcpy(tp->res + (((size_t)cv * G + g) * 2 + q) * n, Zq, sizeof(uint32_t) * n);
      }
      /* Garner (line 974) on the first n entries, then z' / c (line 975) and
       * TSAdd -> DDAdd in flush order (line 976). */
      const double scale = ldexp(1.0, -cexp);
      for (int64_t j = 0; j < n; j++) {
        int fix = 0;
        int64_t Zj = orc_garner2(Zg[j], Zg[m + j], pl->p[0], pl->p[1], &fix);
        if (fix) flags |= 2;
        if (tp && tp->crt) tp->crt[((size_t)cv * G + g) * n + j] = Zj;
        if (pl->ts) { /* z / c in TS (exact), TSAdd in flush order (Alg.8 l.975-976) */
          tacc[(size_t)cv * n + j] =
              orc_ts_add(tacc[(size_t)cv * n + j], ts_ldexp(orc_ts_from_int64(Zj), -cexp));
          continue;
        }
        double h = (double)Zj;
        double l = (double)(Zj - (int64_t)h);
        dd_add(acc[(cv * 2) * n + j], acc[(cv * 2 + 1) * n + j], h * scale, l * scale,
               &acc[(cv * 2) * n + j], &acc[(cv * 2 + 1) * n + j]);
      }
    }
  }
  free(Zg); free(sched); free(X);

  if (pl->ts) { /* TS: y' = (rr - ii) + i (ir + ri), y = y' (.) omega in TS, fl64 (Alg.4 TS 4-5) */
    for (int64_t j = 0; j < n; j++) {
      const orc_ts yr = orc_ts_add(tacc[0 * n + j], orc_ts_neg(tacc[1 * n + j]));
      const orc_ts yi = orc_ts_add(tacc[2 * n + j], tacc[3 * n + j]);
      const orc_ts c = orc_ts_from_double(pl->C[j]), sn = orc_ts_from_double(pl->S[j]);
      const orc_ts orr = orc_ts_add(orc_ts_mul(yr, c), orc_ts_neg(orc_ts_mul(yi, sn)));
      const orc_ts oii = orc_ts_add(orc_ts_mul(yr, sn), orc_ts_mul(yi, c));
      double o_re = orc_ts_to_double(orr), o_im = orc_ts_to_double(oii);
      if (!ts_finite(orr) || !ts_finite(oii)) flags |= 1;
      if (dir > 0) {
        o_re = o_re / (double)n;
        o_im = -o_im / (double)n;
      }
      y[2 * j] = o_re;
      y[2 * j + 1] = o_im;
    }
    free(tacc);
  } else
  /* y' = (rr - ii) + i (ir + ri); Alg.4 step 4: y = y' (.) omega; step 5: round to fp64 */
  for (int64_t j = 0; j < n; j++) {
    double yrh, yrl, yih, yil;
    dd_add(acc[0 * n + j], acc[1 * n + j], -acc[2 * n + j], -acc[3 * n + j], &yrh, &yrl);
    dd_add(acc[4 * n + j], acc[5 * n + j], acc[6 * n + j], acc[7 * n + j], &yih, &yil);
    double a1h, a1l, a2h, a2l, o_re, o_im, tmp;
    dd_mul_d(yrh, yrl, pl->C[j], &a1h, &a1l);
    dd_mul_d(yih, yil, pl->S[j], &a2h, &a2l);
    dd_add(a1h, a1l, -a2h, -a2l, &o_re, &tmp);
    dd_mul_d(yrh, yrl, pl->S[j], &a1h, &a1l);
    dd_mul_d(yih, yil, pl->C[j], &a2h, &a2l);
    dd_add(a1h, a1l, a2h, a2l, &o_im, &tmp);
    if (dir > 0) { /* x = conj(F(conj(y))) / n, RN division (O10) */
      o_re = o_re / (double)n;
      o_im = -o_im / (double)n;
    }
    y[2 * j] = o_re;
    y[2 * j + 1] = o_im;
  }
  free(acc);
  if (tp && tp->counts) {
    tp->counts[0] = nfwd;
    tp->counts[1] = ninv;
    tp->counts[2] = 2 * (int64_t)(pl->kw[0] + pl->kw[1]);
  }
  if (tp && tp->flags) tp->flags[0] = flags;
  return 0;
}

/* Batch of independent transforms, parallel over transforms like the paper's
 * "independent loop iterations ... OpenMP".  Returns the threads used. */
#ifdef _OPENMP
#include <omp.h>
#endif
int orc_execute_batch(const orc_plan* pl, int64_t B, const double* x, double* y, int dir,
                      int nthreads) {
  int used = 1;
#ifdef _OPENMP
  if (nthreads > 0) omp_set_num_threads(nthreads);
#pragma omp parallel
  {
#pragma omp single
    used = omp_get_num_threads();
  }
#pragma omp parallel for schedule(dynamic, 1)
#endif
  for (int64_t b = 0; b < B; b++)
    orc_execute(pl, x + 2 * b * pl->n, y + 2 * b * pl->n, dir, NULL);
  (void)nthreads;
  return used;
}

/* ------------------------------------------------------------------------- */
/* Reference DFT in __float128 (eq:dft P:152-156), used only to pin the oracle */
/* and the GPU output; not part of the method.  out = (hi, lo) doubles per     */
/* component: out[4k+0..1] = Re hi, lo; out[4k+2..3] = Im hi, lo.              */
/* bins == NULL evaluates every k < n; else the nb listed bins.                */
/* ------------------------------------------------------------------------- */
void orc_dft_f128(int64_t n, const double* x, int dir, const int64_t* bins, int64_t nb,
                  double* out) {
  __float128* cs = (__float128*)malloc(sizeof(__float128) * n);
  __float128* sn = (__float128*)malloc(sizeof(__float128) * n);
  for (int64_t r = 0; r < n; r++) { /* omega_n^r = cos(2 pi r/n) - i sin(2 pi r/n) */
    __float128 th = 2 * M_PIq * ((__float128)r / (__float128)n);
    cs[r] = cosq(th);
    sn[r] = sinq(th);
  }
  int64_t cnt = bins ? nb : n;
#ifdef _OPENMP
#pragma omp parallel for schedule(dynamic, 4)
#endif
  for (int64_t ii = 0; ii < cnt; ii++) {
    int64_t k = bins ? bins[ii] : ii;
    __float128 sr = 0, si = 0;
    for (int64_t j = 0; j < n; j++) {
      int64_t r = (int64_t)(((i128)j * k) % n);
      __float128 c = cs[r], s = dir > 0 ? sn[r] : -sn[r]; /* w = c + i s */
      __float128 xr = x[2 * j], xi = x[2 * j + 1];
      sr += xr * c - xi * s;
      si += xr * s + xi * c;
    }
    if (dir > 0) { sr /= n; si /= n; }
    double h;
    h = (double)sr; out[4 * ii + 0] = h; out[4 * ii + 1] = (double)(sr - (__float128)h);
    h = (double)si; out[4 * ii + 2] = h; out[4 * ii + 3] = (double)(si - (__float128)h);
  }
  free(cs);
  free(sn);
}
