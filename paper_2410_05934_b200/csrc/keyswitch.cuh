// keyswitch.cuh -- device kernels of CKKS hybrid key switching (rnt_keyswitch_*,
// "INTT -> BConv (ModUp) -> NTT -> evk inner product -> INTT ->
// ModDown"; P:247-248 name the operators, P:831 the parameters
// (N, L, dnum) = (2^16, 44, 45); readings KS1-KS4 in DESIGN.md).
//
// The transforms are the library's NTT/INTT kernels; this file adds the three
// steps between them:
//   k_modup        digit j: e_j[t] = BConv_{D_j -> t}(x[D_j]) (t outside digit j),
//                  e_j[t] = x[t] (t in digit j); coefficient form, [dnum][L+K][N]
//   k_ks_mac       u_k[t] = sum_j e_j[t] evk[j][k][t] mod m_t, k = 0, 1 (NTT form);
//                  products summed exactly in 128 bits, one reduction per output
//   k_moddown      out_k[i] = (u_k[i] - w_k[i]) P^{-1} mod q_i (+ add0 for k = 0)
#pragma once
#include "modarith.cuh"

namespace rnt {

struct KsMod {
  u64 m, m2;
  u64 qinv;    // m^{-1} mod 2^64 (Montgomery)
  u64 r2;      // 2^128 mod m
  TW one;      // (1, floor(2^64 / m)): Shoup reduction of a word mod m
  TW pinv;     // P^{-1} mod m (Q limbs only, ModDown)
  TW qhatinv;  // (Q_j / q_i)^{-1} mod q_i of the limb's own digit (Q limbs only, ModUp)
};

constexpr int kKsTile = 128;

// grid (ceil(N / kKsTile), dnum); dynamic smem alpha * kKsTile words.
// tab: [dnum][LK][alpha] Shoup pairs of (Q_j / q_i mod m_t).
__global__ void __launch_bounds__(kKsTile)
k_modup(u64* __restrict__ E, const u64* __restrict__ x, const KsMod* __restrict__ km, const TW* __restrict__ tab,
        uint32_t L, uint32_t LK, uint32_t alpha, uint32_t logn) {
  extern __shared__ __align__(16) u64 ys[];
  const uint32_t n = 1u << logn;
  const uint32_t j = blockIdx.y;
  const uint32_t c = blockIdx.x * kKsTile + threadIdx.x;
  if (c >= n) return;
  const uint32_t lo = j * alpha, hi = min(L, lo + alpha);
  for (uint32_t i = lo; i < hi; ++i) {
    const u64 q = km[i].m;
    ys[(i - lo) * kKsTile + threadIdx.x] = csub(shoup_lazy(__ldg(x + ((uint64_t)i << logn) + c), km[i].qhatinv, q), q);
  }
  u64* e = E + ((uint64_t)j * LK << logn) + c;
  const TW* row = tab + (uint64_t)j * LK * alpha;
  for (uint32_t t = 0; t < LK; ++t, row += alpha) {
    u64 v;
    if (t >= lo && t < hi) {
      v = __ldg(x + ((uint64_t)t << logn) + c);
    } else {
      const u64 p = km[t].m, p2 = km[t].m2;
      u64 acc = 0;
      for (uint32_t i = 0; i < hi - lo; ++i) acc = csub(acc + shoup_lazy(ys[i * kKsTile + threadIdx.x], ldg_tw(row + i), p), p2);
      v = csub(acc, p);
    }
    e[(uint64_t)t << logn] = v;
  }
}

// a (< 2^64) times b (< 2^64) added to the 128-bit accumulator (hi, lo).
__device__ __forceinline__ void mac128(u64& hi, u64& lo, u64 a, u64 b) {
  const u64 pl = a * b;
  const u64 ph = __umul64hi(a, b);
  lo += pl;
  hi += ph + (lo < pl);
}

// (hi 2^64 + lo) mod m, canonical, for any hi, lo.
__device__ __forceinline__ u64 reduce128(u64 hi, u64 lo, const KsMod& k) {
  const u64 m = k.m;
  const u64 h = csub(shoup_lazy(hi, k.one, m), m);  // hi mod m
  // Montgomery REDC of h 2^64 + lo (< m 2^64): (h 2^64 + lo) 2^{-64} mod m
  const u64 mq = lo * k.qinv;
  const u64 mh = __umul64hi(mq, m);
  u64 r = h >= mh ? h - mh : h + m - mh;           // [0, m)
  return csub(mont_mul(r, k.r2, m, k.qinv), m);     // times 2^64: back to the plain residue
}

// u: [2][LK][N], E: [dnum][LK][N], evk: [dnum][2][LK][N]; all NTT form.
__global__ void __launch_bounds__(256)
k_ks_mac(u64* __restrict__ u, const u64* __restrict__ E, const u64* __restrict__ evk, const KsMod* __restrict__ km,
         uint32_t dnum, uint32_t LK, uint32_t logn) {
  const uint64_t per = (uint64_t)LK << logn;
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  for (uint64_t e = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; e < per; e += stride) {
    u64 h0 = 0, l0 = 0, h1 = 0, l1 = 0;
    const u64* pe = E + e;
    const u64* pk = evk + e;
#pragma unroll 3
    for (uint32_t j = 0; j < dnum; ++j) {
      const u64 a = __ldcs(pe);
      const u64 b0 = __ldcs(pk);
      const u64 b1 = __ldcs(pk + per);
      mac128(h0, l0, a, b0);
      mac128(h1, l1, a, b1);
      pe += per;
      pk += 2 * per;
    }
    const KsMod k = km[e >> logn];
    u[e] = reduce128(h0, l0, k);
    u[per + e] = reduce128(h1, l1, k);
  }
}

// u = sum of the `parts` partial key products at u + s * total (canonical inputs).
__global__ void __launch_bounds__(256)
k_ks_sum(u64* __restrict__ u, uint32_t parts, const KsMod* __restrict__ km, uint32_t LK, uint32_t logn) {
  const uint64_t per = (uint64_t)LK << logn, total = 2 * per;
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  for (uint64_t e = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; e < total; e += stride) {
    const u64 m = km[(e % per) >> logn].m;
    u64 v = u[e];
    for (uint32_t s = 1; s < parts; ++s) v = csub(v + __ldcs(u + s * total + e), m);
    u[e] = v;
  }
}

// out: [2][L][N], u: [2][LK][N], w: [2][L][N], add0: [L][N] or null.
__global__ void __launch_bounds__(256)
k_moddown(u64* __restrict__ out, const u64* __restrict__ u, const u64* __restrict__ w, const u64* __restrict__ add0,
          const KsMod* __restrict__ km, uint32_t L, uint32_t LK, uint32_t logn) {
  const uint64_t perq = (uint64_t)L << logn, perqp = (uint64_t)LK << logn;
  const uint64_t total = 2 * perq;
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  for (uint64_t e = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; e < total; e += stride) {
    const uint32_t k = e >= perq;
    const uint64_t r = e - k * perq;
    const KsMod m = km[r >> logn];
    const u64 d = __ldg(u + k * perqp + r) + m.m - __ldg(w + e);  // (0, 2m)
    u64 v = csub(shoup_lazy(d, m.pinv, m.m), m.m);
    if (!k && add0) v = csub(v + __ldg(add0 + r), m.m);
    out[e] = v;
  }
}

}  // namespace rnt
