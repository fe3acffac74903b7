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
// pipes carry about a fifth of what the HBM rate needs and the loads -- their
// latency, with L N / 2 threads in flight -- bound it.
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

__device__ __forceinline__ void acc_add(Acc192& a, const Acc192& b) {
  const u64 lo = a.lo + b.lo;
  const u64 c0 = lo < b.lo;
  const u64 hs = a.hi + b.hi;
  const u64 c1 = hs < b.hi;
  const u64 hi = hs + c0;
  const u64 c2 = hi < c0;
  a.lo = lo;
  a.hi = hi;
  a.top += b.top + c1 + c2;
}

// CTA of 256 threads = JS groups of VB = 256 / JS threads: the groups share the
// CTA's VB slot pairs and split the slots j (group g takes j = g, g + JS, ...), so
// JS times more loads are in flight for the same outputs (the kernel is bound by
// memory latency, not by the integer pipes); the groups' 192-bit sums are added
// through shared memory before the reduction.  Grid-stride over slot-pair blocks.
// Thread v owns slots 2v, 2v + 1 of limb (2v) >> logn.
#ifndef RNT_HRF_MINB
#define RNT_HRF_MINB 4
#endif
template <int UNROLL, int JS>
__global__ void __launch_bounds__(256, RNT_HRF_MINB)
k_hrf_matvec(u64* out, const u64* __restrict__ pt, const u64* __restrict__ ct,
             const u64* add, const LimbC* __restrict__ lc, uint32_t n_slot, uint32_t L, uint32_t logn,
             uint64_t nvec) {
  constexpr int VB = 256 / JS;
  __shared__ Acc192 part[JS > 1 ? JS - 1 : 1][4][VB];
  const ulonglong2* P = reinterpret_cast<const ulonglong2*>(pt);
  const ulonglong2* C = reinterpret_cast<const ulonglong2*>(ct);
  const uint64_t vs = ((uint64_t)L << logn) / 2;    // vectors per [L][N] block
  const int tv = (int)threadIdx.x % VB, jg = (int)threadIdx.x / VB;
  for (uint64_t v0 = (uint64_t)blockIdx.x * VB; v0 < nvec; v0 += (uint64_t)gridDim.x * VB) {
    const uint64_t v = v0 + tv;
    const bool live = v < nvec;
    Acc192 acc[4] = {{0, 0, 0}, {0, 0, 0}, {0, 0, 0}, {0, 0, 0}};   // [slot x / y][component]
    if (live) {
      uint32_t j = (uint32_t)jg;
      for (; j + (UNROLL - 1) * JS < n_slot; j += UNROLL * JS) {
        ulonglong2 p[UNROLL], c0[UNROLL], c1[UNROLL];
#pragma unroll
        for (int u = 0; u < UNROLL; ++u) {             // all loads of the group in flight at once
          const uint64_t jj = j + (uint64_t)u * JS;
          p[u] = __ldcs(P + jj * vs + v);
          c0[u] = __ldcs(C + 2 * jj * vs + v);
          c1[u] = __ldcs(C + (2 * jj + 1) * vs + v);
        }
#pragma unroll
        for (int u = 0; u < UNROLL; ++u) {
          acc_mul(acc[0], p[u].x, c0[u].x);
          acc_mul(acc[1], p[u].x, c1[u].x);
          acc_mul(acc[2], p[u].y, c0[u].y);
          acc_mul(acc[3], p[u].y, c1[u].y);
        }
      }
      for (; j < n_slot; j += JS) {
        const ulonglong2 p = __ldcs(P + (uint64_t)j * vs + v);
        const ulonglong2 c0 = __ldcs(C + (uint64_t)(2 * j) * vs + v);
        const ulonglong2 c1 = __ldcs(C + (uint64_t)(2 * j + 1) * vs + v);
        acc_mul(acc[0], p.x, c0.x);
        acc_mul(acc[1], p.x, c1.x);
        acc_mul(acc[2], p.y, c0.y);
        acc_mul(acc[3], p.y, c1.y);
      }
    }
    if constexpr (JS > 1) {
      if (jg > 0) {
#pragma unroll
        for (int k = 0; k < 4; ++k) part[jg - 1][k][tv] = acc[k];
      }
      __syncthreads();
      if (jg == 0) {
#pragma unroll
        for (int g = 0; g < JS - 1; ++g)
#pragma unroll
          for (int k = 0; k < 4; ++k) acc_add(acc[k], part[g][k][tv]);
      }
      __syncthreads();
    }
    if (jg == 0 && live) {
      const uint32_t l = (uint32_t)((2 * v) >> logn);
      const u64 q = lc[l].q, qinv = lc[l].qinv, r2 = lc[l].r2;
      const u64 r1 = canon2(mont_mul(1ull, r2, q, qinv), q);            // 2^64 mod q
      ulonglong2 d0{0, 0}, d1{0, 0};
      if (add) {
        d0 = reinterpret_cast<const ulonglong2*>(add)[v];
        d1 = reinterpret_cast<const ulonglong2*>(add)[vs + v];
      }
      ulonglong2 o0, o1;
      o0.x = reduce192(acc[0], d0.x, q, qinv, r2, r1);
      o0.y = reduce192(acc[2], d0.y, q, qinv, r2, r1);
      o1.x = reduce192(acc[1], d1.x, q, qinv, r2, r1);
      o1.y = reduce192(acc[3], d1.y, q, qinv, r2, r1);
      reinterpret_cast<ulonglong2*>(out)[v] = o0;
      reinterpret_cast<ulonglong2*>(out)[vs + v] = o1;
    }
  }
}

}  // namespace rnt
