// modarith.cuh -- 64-bit modular arithmetic for sm_100a built from 32-bit
// IMAD / IMAD.HI / IMAD.WIDE (no tensor cores; BASELINE.json north_star (b)).
//
// Moduli: q < 2^62 (reading C5), so lazy ranges up to [0, 4q) fit in a word.
//
//   shoup_lazy(y, W)   y * w mod q for any y < 2^64, result in [0, 2q);
//                      W = (w, w' = floor(w 2^64 / q)) precomputed (Shoup).
//   ct_bfly            Cooley-Tukey butterfly of NTT^{CT,psi}_{no->bo}
//                      (Eq. 1): (X, Y) -> (X + wY, X - wY), Harvey's
//                      lazy form: inputs and outputs in [0, 4q).
//   gs_bfly            Gentleman-Sande butterfly of INTT^{GS,psi^-1}_{bo->no}
//                      (Eq. 1): (X, Y) -> (X + Y, (X - Y) w), lazy:
//                      inputs and outputs in [0, 2q).
//   mont_mul           a b 2^{-64} mod q (Montgomery), a < 4q, b < q,
//                      result in (0, 2q); used for the (.) of Eq. 1.
#pragma once
#include <stdint.h>

#include <type_traits>

namespace rnt {

typedef unsigned long long u64;

// Compile-time loop: f(std::integral_constant<int, i>) for i in [B, E).  The
// stage loops below nest loops whose trip counts depend on the stage index;
// forcing them through templates guarantees full unrolling, so the
// coefficient arrays stay in registers (no local-memory stack frame).
template <int B, int E, typename F>
__device__ __forceinline__ void sfor(F&& f) {
  if constexpr (B < E) {
    f(std::integral_constant<int, B>{});
    sfor<B + 1, E>(f);
  }
}

struct __align__(16) TW {
  u64 w;   // twiddle value, canonical
  u64 wp;  // Shoup companion floor(w * 2^64 / q)
};

// Per-limb constants, device resident.
struct __align__(16) LimbC {
  u64 q, q2;     // q, 2q
  u64 qinv;      // q^{-1} mod 2^64 (Montgomery)
  u64 r2;        // 2^128 mod q (Montgomery R^2)
  TW ninv;       // N^{-1}
  TW ninv_w1;    // N^{-1} * psi^{-brv(1)}: last GS stage with N^{-1} folded
  TW ninvR;      // N^{-1} * 2^64: after a Montgomery pointwise product
  TW ninvR_w1;   // N^{-1} * 2^64 * psi^{-brv(1)}
};

__device__ __forceinline__ u64 ldg_u64(const u64* p) { return __ldg(p); }

__device__ __forceinline__ TW ldg_tw(const TW* p) {
  ulonglong2 v = __ldg(reinterpret_cast<const ulonglong2*>(p));
  TW t;
  t.w = v.x;
  t.wp = v.y;
  return t;
}

__device__ __forceinline__ u64 shoup_lazy(u64 y, TW t, u64 q) {
  u64 Q = __umul64hi(y, t.wp);
  return y * t.w - Q * q;
}

// x - m if x >= m else x, for x < 2m and m < 2^63 (every call site: lazy
// bounds 2m at most): the sign of the 64-bit difference decides, one compare
// instead of the unsigned compare pair (ptxas then drops an IMAD.IADD from
// the fmaheavy pipe per butterfly).
__device__ __forceinline__ u64 csub(u64 x, u64 m) {
  const u64 d = x - m;
  return (long long)d < 0 ? x : d;
}

__device__ __forceinline__ void ct_bfly(u64& X, u64& Y, TW t, u64 q, u64 q2) {
  u64 x = csub(X, q2);          // [0, 2q)
  u64 v = shoup_lazy(Y, t, q);  // [0, 2q)
  X = x + v;                    // [0, 4q)
  Y = x + q2 - v;               // (0, 4q)
}

__device__ __forceinline__ void gs_bfly(u64& X, u64& Y, TW t, u64 q, u64 q2) {
  u64 s = csub(X + Y, q2);      // [0, 2q)
  u64 d = X + q2 - Y;           // (0, 4q)
  X = s;
  Y = shoup_lazy(d, t, q);      // [0, 2q)
}

// CT butterfly without the input reduction, for moduli q < 2^60 (16 q < 2^64;
// LZ kernels, plan flag lazy60): X in [0, B q) -> X', Y' in [0, (B + 2) q).
// From canonical input at global stage 0 the bound grows by 2q per stage and
// X is reduced by 8q only when the bound would pass 16q (RED: [0, 16q) ->
// [0, 8q)): stages 7, 11, 15 of a 2^16 transform, only stage 7 at 2^10, so
// 13 of 16 (9 of 10) stages drop the csub of Harvey's butterfly.
__host__ __device__ constexpr int lz_bound_before(int s) {
  int b = 1;
  for (int i = 0; i < s; ++i) b = (b > 14 ? 8 : b) + 2;
  return b;
}
__host__ __device__ constexpr bool lz_red(int s) { return lz_bound_before(s) > 14; }
static_assert(lz_bound_before(7) == 15 && lz_red(7) && !lz_red(6) && lz_red(11) && lz_red(15), "LZ schedule");

template <bool RED>
__device__ __forceinline__ void ct_bfly_lz(u64& X, u64& Y, TW t, u64 q, u64 q2) {
  u64 x = RED ? csub(X, q2 << 2) : X;
  u64 v = shoup_lazy(Y, t, q);  // [0, 2q)
  X = x + v;
  Y = x + q2 - v;
}

// CT butterfly of global stage s: Harvey's [0, 4q) form, or the LZ form.
template <bool LZ, int s>
__device__ __forceinline__ void ct_bfly_at(u64& X, u64& Y, TW t, u64 q, u64 q2) {
  if constexpr (LZ) ct_bfly_lz<lz_red(s)>(X, Y, t, q, q2);
  else ct_bfly(X, Y, t, q, q2);
}

// GS butterflies of the last three inverse stages without the sum reduction
// (LZ, q < 2^60): the final stage multiplies both outputs (N^{-1} folded in),
// and a Shoup product accepts any input below 2^64, so the sum path may grow
// from [0, 2q) at global stage 2 to [0, 8q) into stage 0 (16q < 2^64).
// BY = bound of the Y input in units of q (2, 4, 8 at stages 2, 1, 0).
template <int BY>
__device__ __forceinline__ void gs_bfly_nr(u64& X, u64& Y, TW t, u64 q, u64 q2) {
  const u64 d = X + (q2 * (BY / 2)) - Y;   // (0, (BX + BY) q)
  X = X + Y;                               // [0, (BX + BY) q)
  Y = shoup_lazy(d, t, q);                 // [0, 2q)
}
template <int BY>
__device__ __forceinline__ void gs_bfly_last_nr(u64& X, u64& Y, TW s0, TW s1, u64 q, u64 q2) {
  const u64 s = X + Y;
  const u64 d = X + (q2 * (BY / 2)) - Y;
  X = shoup_lazy(s, s0, q);
  Y = shoup_lazy(d, s1, q);
}

// GS butterfly with a negated twiddle: (X, Y) -> (X + Y, (Y - X) w).  With
// w = psi^{brv(k')} of the mirrored index k' = 3 2^s - 1 - k this equals the GS
// butterfly with psi^{-brv(k)} = -psi^{brv(k')}, so inverse row stages can read
// the forward twiddle table (ntt_large.cuh).
__device__ __forceinline__ void gs_bfly_neg(u64& X, u64& Y, TW t, u64 q, u64 q2) {
  u64 s = csub(X + Y, q2);      // [0, 2q)
  u64 d = Y + q2 - X;           // (0, 4q)
  X = s;
  Y = shoup_lazy(d, t, q);      // [0, 2q)
}

// Last GS stage (t = N/2, twiddle psi^{-brv(1)}) with the N^{-1} scaling of
// S:167 folded in: X' = (X + Y) N^{-1}, Y' = (X - Y) psi^{-brv(1)} N^{-1}.
__device__ __forceinline__ void gs_bfly_last(u64& X, u64& Y, TW s0, TW s1, u64 q, u64 q2) {
  u64 s = X + Y;                // [0, 4q)
  u64 d = X + q2 - Y;           // (0, 4q)
  X = shoup_lazy(s, s0, q);     // [0, 2q)
  Y = shoup_lazy(d, s1, q);
}

// [0, 4q) -> [0, q)
__device__ __forceinline__ u64 canon4(u64 x, u64 q, u64 q2) { return csub(csub(x, q2), q); }
// [0, 16q) -> [0, q) (LZ outputs)
__device__ __forceinline__ u64 canon16(u64 x, u64 q, u64 q2) {
  return csub(csub(csub(csub(x, q2 << 2), q2 << 1), q2), q);
}
// [0, 2q) -> [0, q)
__device__ __forceinline__ u64 canon2(u64 x, u64 q) { return csub(x, q); }

__device__ __forceinline__ u64 mont_mul(u64 a, u64 b, u64 q, u64 qinv) {
  // one 128-bit product (4 IMAD.WIDE) instead of lo and hi separately (5 + 2 IMAD)
  const unsigned __int128 T = (unsigned __int128)a * b;
  u64 lo = (u64)T;
  u64 hi = (u64)(T >> 64);
  u64 m = lo * qinv;            // m q == lo (mod 2^64)
  u64 mh = __umul64hi(m, q);
  return hi - mh + q;           // (a b - m q) / 2^64 + q in (0, 2q)
}

// T 2^{-64} mod q for an exact sum of products T < 15 q 2^64 (Montgomery
// reduction of the whole sum): (T - m q) / 2^64 + q = hi - hi64(m q) + q in
// (0, 16q) with m q == T mod 2^64; three conditional subtractions -> [0, 2q).
// Callers are LZ kernels (q < 2^60, 16q < 2^64).
__device__ __forceinline__ u64 redc_sum(unsigned __int128 T, u64 q, u64 q2, u64 qinv) {
  const u64 lo = (u64)T, hi = (u64)(T >> 64);
  const u64 m = lo * qinv;
  const u64 r = hi - __umul64hi(m, q) + q;   // (0, 16q)
  return csub(csub(csub(r, q2 << 2), q2 << 1), q2);
}

}  // namespace rnt
