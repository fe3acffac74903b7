// plan.cpp -- host plan builder.  See plan.h.
//
// psi: primitive 2N-th root of unity mod q, psi^{2N} = 1, psi^i != 1 for
// i < 2N; default = the smallest one (reading C1).
// Tables: psi^{brv_n(i)} and psi^{-brv_n(i)} (the index order of the CT / GS
// loops of Eq. 1), each with Shoup companion floor(w 2^64 / q).
#include "plan.h"

#include <algorithm>
#include <cstring>
#include <set>

namespace rnt {

typedef unsigned __int128 u128;

uint64_t hp_mulmod(uint64_t a, uint64_t b, uint64_t q) { return (uint64_t)((u128)a * b % q); }

uint64_t hp_powmod(uint64_t a, uint64_t e, uint64_t q) {
  uint64_t r = 1 % q;
  a %= q;
  for (; e; e >>= 1) {
    if (e & 1) r = hp_mulmod(r, a, q);
    a = hp_mulmod(a, a, q);
  }
  return r;
}

static bool mr_round(uint64_t n, uint64_t a, uint64_t d, int s) {
  uint64_t x = hp_powmod(a, d, n);
  if (x == 1 || x == n - 1) return true;
  for (int i = 1; i < s; ++i) {
    x = hp_mulmod(x, x, n);
    if (x == n - 1) return true;
  }
  return false;
}

bool hp_is_prime(uint64_t n) {
  if (n < 2) return false;
  static const uint64_t small[] = {2, 3, 5, 7, 11, 13, 17, 19, 23, 29, 31, 37};
  for (uint64_t p : small) {
    if (n % p == 0) return n == p;
  }
  uint64_t d = n - 1;
  int s = 0;
  while (!(d & 1)) {
    d >>= 1;
    ++s;
  }
  for (uint64_t a : small)
    if (!mr_round(n, a, d, s)) return false;
  return true;
}

uint32_t hp_bitrev(uint32_t x, uint32_t bits) {
  uint32_t r = 0;
  for (uint32_t i = 0; i < bits; ++i, x >>= 1) r = (r << 1) | (x & 1);
  return r;
}

uint64_t hp_smallest_psi(uint64_t q, uint32_t logn) {
  const uint64_t n = 1ull << logn;
  const uint64_t order = 2 * n;
  if ((q - 1) % order) return 0;
  uint64_t g = 0;
  for (uint64_t x = 2; x < q && !g; ++x) {
    uint64_t c = hp_powmod(x, (q - 1) / order, q);
    if (hp_powmod(c, n, q) == q - 1) g = c;  // order exactly 2N
  }
  if (!g) return 0;
  // all primitive 2N-th roots: g^k, k odd
  uint64_t g2 = hp_mulmod(g, g, q), cur = g, best = g;
  for (uint64_t k = 1; k < order; k += 2) {
    best = std::min(best, cur);
    cur = hp_mulmod(cur, g2, q);
  }
  return best;
}

static HostTW make_tw(uint64_t w, uint64_t q) {
  HostTW t;
  t.w = w;
  t.wp = (uint64_t)(((u128)w << 64) / q);
  return t;
}

int plan_limbs(uint32_t logn, uint32_t L, const uint64_t* moduli, const uint64_t* psi,
               std::vector<HostLimb>& out) {
  const uint64_t n = 1ull << logn;
  out.assign(L, HostLimb{});
  std::set<uint64_t> seen;
  for (uint32_t l = 0; l < L; ++l) {
    const uint64_t q = moduli[l];
    if (q >= (1ull << 62) || q < 3 || (q - 1) % (2 * n) != 0 || !hp_is_prime(q)) return PLAN_E_MODULUS;
    if (!seen.insert(q).second) return PLAN_E_MODULUS;
    uint64_t p = psi ? psi[l] : hp_smallest_psi(q, logn);
    if (p == 0 || p >= q || hp_powmod(p, n, q) != q - 1) return PLAN_E_ROOT;
    HostLimb& lm = out[l];
    lm.q = q;
    lm.psi = p;
    lm.q2 = 2 * q;
    uint64_t inv = q;  // Newton: q * q == 1 mod 8
    for (int i = 0; i < 6; ++i) inv *= 2 - q * inv;
    lm.qinv = inv;
    const uint64_t R = (uint64_t)(((u128)1 << 64) % q);
    lm.r2 = hp_mulmod(R, R, q);
    const uint64_t ninv = hp_powmod(n % q, q - 2, q);
    const uint64_t psi_inv = hp_powmod(p, q - 2, q);
    const uint64_t w1 = hp_powmod(psi_inv, hp_bitrev(1, logn), q);  // psi^{-brv(1)}
    lm.ninv = make_tw(ninv, q);
    lm.ninv_w1 = make_tw(hp_mulmod(ninv, w1, q), q);
    const uint64_t ninvR = hp_mulmod(ninv, R, q);
    lm.ninvR = make_tw(ninvR, q);
    lm.ninvR_w1 = make_tw(hp_mulmod(ninvR, w1, q), q);
  }
  return PLAN_OK;
}

void plan_powers(const HostLimb& lm, uint32_t logn, bool inverse, uint32_t count, HostTW* tab) {
  const uint64_t q = lm.q;
  const uint64_t n = 1ull << logn;
  const uint64_t base = inverse ? hp_powmod(lm.psi, q - 2, q) : lm.psi;
  std::vector<uint64_t> pw(n);
  uint64_t cur = 1;
  for (uint64_t k = 0; k < n; ++k) {
    pw[k] = cur;
    cur = hp_mulmod(cur, base, q);
  }
  for (uint32_t i = 0; i < count; ++i) tab[i] = make_tw(pw[hp_bitrev(i, logn)], q);
}

void plan_row_layout(const HostTW* nat, uint32_t logn, HostTW* out) {
  const uint32_t n1 = (logn + 1) / 2, n2 = logn / 2, R = 1u << n1, Cn = 1u << n2, T2 = Cn / 16;
  std::memset(out, 0, sizeof(HostTW) * (size_t)R * Cn);
  for (uint32_t r = 0; r < R; ++r) {
    HostTW* row = out + (size_t)r * Cn;
    for (uint32_t v = 0; v < n2; ++v) {
      const uint32_t blk = (1u << v) - 1;
      const uint32_t g = (1u << (n1 + v)) + r * (1u << v);
      if (v < 4) {
        for (uint32_t k = 0; k < (1u << v); ++k) row[blk + k] = nat[g + k];
      } else {
        const uint32_t per = 1u << (v + 4 - n2);
        for (uint32_t m = 0; m < per; ++m)
          for (uint32_t c1 = 0; c1 < T2; ++c1) row[blk + m * T2 + c1] = nat[g + c1 * per + m];
      }
    }
  }
}

}  // namespace rnt

namespace rnt {
void plan_row_natural(const HostTW* nat, uint32_t logn, HostTW* out) {
  const uint32_t n1 = (logn + 1) / 2, n2 = logn / 2, R = 1u << n1, Cn = 1u << n2;
  std::memset(out, 0, sizeof(HostTW) * (size_t)R * Cn);
  for (uint32_t r = 0; r < R; ++r)
    for (uint32_t v = 0; v < n2; ++v)
      for (uint32_t j = 0; j < (1u << v); ++j)
        out[(size_t)r * Cn + (1u << v) + j] = nat[(1u << (n1 + v)) + r * (1u << v) + j];
}
}  // namespace rnt
