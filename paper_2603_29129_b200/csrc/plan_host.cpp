// plan_host.cpp -- host-side plan math for ozfft (runs once at plan create).
//
// Everything here is input-independent precomputation (the paper precomputes the
// omega* split and its NTTs offline): the chirp table omega(j) =
// omega_{2n}^{j^2} correctly rounded to binary64 (ruling 3 in DESIGN.md),
// omega~* = ZeroPad_pm(omega*, m), and per-prime NTT twiddle tables
// with Shoup companions (Shoup multiplication).  Written independently of
// oracle/ (shares no code with it).
#include <quadmath.h>

#include <cmath>
#include <cstring>

#include "internal.h"

namespace ozfft {

namespace {

uint32_t pow_mod(uint64_t a, uint64_t e, uint32_t p) {
  uint64_t r = 1 % p;
  a %= p;
  for (; e; e >>= 1) {
    if (e & 1) r = (r * a) % p;
    a = (a * a) % p;
  }
  return (uint32_t)r;
}

// smallest generator of (Z/pZ)^*: g^((p-1)/q) != 1 for all prime factors q of p-1
uint32_t generator(uint32_t p) {
  std::vector<uint64_t> qs;
  uint64_t r = p - 1;
  for (uint64_t d = 2; d * d <= r; ++d) {
    if (r % d == 0) {
      qs.push_back(d);
      while (r % d == 0) r /= d;
    }
  }
  if (r > 1) qs.push_back(r);
  for (uint32_t g = 2; g < p; ++g) {
    bool ok = true;
    for (uint64_t q : qs)
      if (pow_mod(g, (p - 1) / q, p) == 1) { ok = false; break; }
    if (ok) return g;
  }
  return 0;
}

}  // namespace

ozfft_status build_plan_tables(Plan& pl) {
  const int64_t n = pl.n, m = pl.m;
  // ---- chirp omega(j) = exp(-i pi j^2 / n): C = RN(cos(pi r/n)), S = RN(-sin(pi r/n)),
  //      r = j^2 mod 2n, with the four axis angles exact and zeros as +0.0.
  pl.chirp.assign((size_t)2 * n, 0.0);
  for (int64_t j = 0; j < n; ++j) {
    const int64_t r = (int64_t)(((__int128)j * j) % (2 * (__int128)n));
    double c, s;
    if (r == 0) {
      c = 1.0; s = 0.0;
    } else if (2 * r == n) {
      c = 0.0; s = -1.0;
    } else if (r == n) {
      c = -1.0; s = 0.0;
    } else if (2 * r == 3 * n) {
      c = 0.0; s = 1.0;
    } else {
      const __float128 th = M_PIq * ((__float128)r / (__float128)n);
      c = (double)cosq(th);
      s = (double)(-sinq(th));
    }
    pl.chirp[2 * j] = c;
    pl.chirp[2 * j + 1] = s;
  }
  // ---- omega~*(j): omega*(j) for j < n, 0 for n <= j < m-n+1, omega*(m-j) above
  pl.wstar.assign((size_t)2 * m, 0.0);
  for (int64_t j = 0; j < m; ++j) {
    int64_t src = j < n ? j : (j >= m - n + 1 ? m - j : -1);
    if (src >= 0) {
      pl.wstar[2 * j] = pl.chirp[2 * src];
      pl.wstar[2 * j + 1] = -pl.chirp[2 * src + 1];  // conj
    }
  }
  // ---- twiddles: T[h + j] = w_{2h}^{j} (dir 0) or w_{2h}^{-j} (dir 1), h = 1..m/2
  for (int q = 0; q < 2; ++q) {
    const uint32_t p = pl.p[q];
    const uint32_t wm = pow_mod(generator(p), (uint64_t)(p - 1) / (uint64_t)m, p);
    const uint32_t wmi = pow_mod(wm, p - 2, p);
    pl.minv[q] = pow_mod((uint64_t)m % p, p - 2, p);
    uint32_t inv = p;  // p^{-1} mod 2^32 by Newton iteration (p odd)
    for (int i = 0; i < 5; ++i) inv *= 2u - p * inv;
    pl.pinv[q] = 0u - inv;
    for (int dir = 0; dir < 2; ++dir) {
      std::vector<uint32_t>& T = pl.tw[q][dir];
      T.assign((size_t)2 * std::max<int64_t>(m, 2), 0);
      for (int64_t h = 1; h <= m / 2; h <<= 1) {
        const uint32_t w2h = pow_mod(dir ? wmi : wm, (uint64_t)(m / (2 * h)), p);
        uint64_t w = 1;
        for (int64_t j = 0; j < h; ++j) {
          T[2 * (h + j)] = (uint32_t)w;
          T[2 * (h + j) + 1] = (uint32_t)((w << 32) / p);  // Shoup companion floor(w 2^32 / p)
          w = (w * w2h) % p;
        }
      }
    }
  }
  pl.p0inv_mod_p1 = pow_mod(pl.p[0] % pl.p[1], pl.p[1] - 2, pl.p[1]);
  // image mode (f2): iota = g^((p-1)/4), a square root of -1 mod p
  if (pl.image)
    for (int q = 0; q < 2; ++q) pl.iota[q] = pow_mod(generator(pl.p[q]), (pl.p[q] - 1) / 4, pl.p[q]);
  return OZFFT_OK;
}

}  // namespace ozfft
