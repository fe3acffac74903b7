// hrf.cuh -- HRF-MatVec, the homomorphic-rotation-free matrix-vector product
// of repack (tab:repack P:393-395: 0 rotations, n_slot scalar
// multiplications, n_slot precomputed rotation ciphertexts):
//
//   out[c][l][k] = add[c][l][k] + sum_{j < n_slot} pt[j][l][k] * ct[j][c][l][k]  mod q_l
//
// pt [n_slot][L][N] (plaintext diagonals, NTT form), ct [n_slot][2][L][N]
// (rotation ciphertexts, NTT form), add [2][L][N] or null, out [2][L][N].
//
// HBM-bound: 24 bytes are read per (j, l, k) and two 64 x 64 -> 128-bit
// products are formed from them.  Every thread owns two consecutive slots k
// of one limb (16-byte loads of pt and of both ct components, coalesced
// across the warp) and keeps four 192-bit sums (lo, hi, top) of exact
// products: no modular reduction inside the j loop, one per output at the
// end (three Montgomery products against 2^64 and 2^128 mod q), so the integer
// pipes carry ~45 % of what the HBM rate needs and loads stay the bottleneck.
#pragma once
#include "modarith.cuh"

namespace rnt {

struct Acc192 {
  u64 lo, hi, top;
};

__device__ __forceinline__ void acc_mul(Acc192& a, u64 x, u64 y) {
  const u64 plo = x * y;
  const u64 phi = __umul64hi(x, y);
  const u64 lo = a.lo + plo;
  const u64 c0 = lo < plo;
  const u64 hi = a.hi + phi + c0;                  // phi < 2^60 (q < 2^62): no overflow of phi + c0
  a.top += (hi < a.hi) ? 1ull : 0ull;
  a.lo = lo;
  a.hi = hi;
}

// x = top 2^128 + hi 2^64 + lo  ->  x mod q, canonical; plus a canonical addend.
// Montgomery products mont(a, b) = a b 2^-64 with b < q accept any a < 2^64;
// every term is made canonical before the modular additions (q < 2^62, so two
// canonical terms never overflow a word).
__device__ __forceinline__ u64 reduce192(const Acc192& a, u64 addv, u64 q, u64 qinv, u64 r2, u64 r1) {
  const u64 t0 = canon2(mont_mul(a.lo, r1, q, qinv), q);                                    // lo
  const u64 t1 = canon2(mont_mul(a.hi, r2, q, qinv), q);                                    // hi 2^64
  const u64 t2 = canon2(mont_mul(canon2(mont_mul(a.top, r2, q, qinv), q), r2, q, qinv), q);  // top 2^128
  return csub(csub(t0 + t1, q) + csub(t2 + addv, q), q);
}

// grid-stride over v in [0, L N / 2): thread owns slots e = 2v, 2v + 1 of limb e >> logn.
template <int UNROLL>
__global__ void __launch_bounds__(256)
k_hrf_matvec(u64* out, const u64* __restrict__ pt, const u64* __restrict__ ct,
             const u64* add, const LimbC* __restrict__ lc, uint32_t n_slot, uint32_t L, uint32_t logn,
             uint64_t nvec) {
  const uint64_t ln = (uint64_t)L << logn;          // elements per [L][N] block
  const ulonglong2* P = reinterpret_cast<const ulonglong2*>(pt);
  const ulonglong2* C = reinterpret_cast<const ulonglong2*>(ct);
  const uint64_t vs = ln / 2;                       // vectors per [L][N] block
  for (uint64_t v = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; v < nvec;
       v += (uint64_t)gridDim.x * blockDim.x) {
    Acc192 a00{0, 0, 0}, a01{0, 0, 0}, a10{0, 0, 0}, a11{0, 0, 0};   // [slot][component]
    uint32_t j = 0;
    for (; j + UNROLL <= n_slot; j += UNROLL) {
      ulonglong2 p[UNROLL], c0[UNROLL], c1[UNROLL];
#pragma unroll
      for (int u = 0; u < UNROLL; ++u) {             // all loads of the group in flight at once
        p[u] = __ldcs(P + (uint64_t)(j + u) * vs + v);
        c0[u] = __ldcs(C + (uint64_t)(2 * (j + u)) * vs + v);
        c1[u] = __ldcs(C + (uint64_t)(2 * (j + u) + 1) * vs + v);
      }
#pragma unroll
      for (int u = 0; u < UNROLL; ++u) {
        acc_mul(a00, p[u].x, c0[u].x);
        acc_mul(a01, p[u].x, c1[u].x);
        acc_mul(a10, p[u].y, c0[u].y);
        acc_mul(a11, p[u].y, c1[u].y);
      }
    }
    for (; j < n_slot; ++j) {
      const ulonglong2 p = __ldcs(P + (uint64_t)j * vs + v);
      const ulonglong2 c0 = __ldcs(C + (uint64_t)(2 * j) * vs + v);
      const ulonglong2 c1 = __ldcs(C + (uint64_t)(2 * j + 1) * vs + v);
      acc_mul(a00, p.x, c0.x);
      acc_mul(a01, p.x, c1.x);
      acc_mul(a10, p.y, c0.y);
      acc_mul(a11, p.y, c1.y);
    }
    const uint32_t l = (uint32_t)((2 * v) >> logn);
    const u64 q = lc[l].q, qinv = lc[l].qinv, r2 = lc[l].r2;
    const u64 r1 = canon2(mont_mul(1ull, r2, q, qinv), q);            // 2^64 mod q
    ulonglong2 d0{0, 0}, d1{0, 0};
    if (add) {
      d0 = reinterpret_cast<const ulonglong2*>(add)[v];
      d1 = reinterpret_cast<const ulonglong2*>(add)[vs + v];
    }
    ulonglong2 o0, o1;
    o0.x = reduce192(a00, d0.x, q, qinv, r2, r1);
    o0.y = reduce192(a10, d0.y, q, qinv, r2, r1);
    o1.x = reduce192(a01, d1.x, q, qinv, r2, r1);
    o1.y = reduce192(a11, d1.y, q, qinv, r2, r1);
    reinterpret_cast<ulonglong2*>(out)[v] = o0;
    reinterpret_cast<ulonglong2*>(out)[vs + v] = o1;
  }
}

}  // namespace rnt
