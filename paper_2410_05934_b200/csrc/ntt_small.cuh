// ntt_small.cuh -- one-kernel negacyclic NTT / INTT / fused polymul for
// N = 2^4 .. 2^10 (the TFHE polynomial size), batched over
// (polynomial, limb) units (CMux-level batching).
//
// B200 design (the paper's BD/TA/PCS kernels, are prior art):
//   * one warp owns a 1024-coefficient shared-memory buffer holding 1024/N
//     polynomials; no CTA-wide barrier anywhere, only __syncwarp;
//   * the log2 N stages are grouped into passes of <= 4 stages (N = 2^10:
//     4 + 4 + 2).  In a pass every lane loads radix-2^k groups of
//     coefficients into registers, runs k CT (or GS) stages, stores back;
//   * pass bodies are *looped* (not unrolled) over groups, so the whole
//     kernel is a few kB of SASS and stays resident in the instruction cache
//     (a fully unrolled 32-coefficient-per-lane design measured 2.3 stall
//     cycles per instruction waiting on instruction fetch, profiles/);
//   * the first forward pass reads global memory directly (coalesced, stride
//     layout) and the last pass of each direction writes global memory;
//   * polymul fuses last-forward-pass -> (.) b_hat -> first-inverse-pass in
//     registers (the NTT-domain product never touches shared memory);
//   * shared-memory padding j + (j >> 4) makes all three pass patterns of
//     N = 2^10 conflict-free with immediate-offset addressing (wpad).
// Lazy Harvey ranges (modarith.cuh); outputs are canonical.
#pragma once
#include "modarith.cuh"

namespace rnt {

constexpr int kWarpElems = 1024;          // coefficients per warp buffer
constexpr int kTeamWarps = 4;             // warps per CTA

template <int LOGN>
struct WarpCfg {
  static constexpr int N = 1 << LOGN;
  static constexpr int P = kWarpElems / N;             // polynomials per warp
  static constexpr int K0 = LOGN < 4 ? LOGN : 4;       // stages per pass
  static constexpr int K1 = (LOGN - K0) < 4 ? (LOGN - K0) : 4;
  static constexpr int K2 = LOGN - K0 - K1;
  static constexpr int NPASS = 1 + (K1 > 0) + (K2 > 0);
  static_assert(K2 <= 4, "N <= 2^12");
};

// Shared-memory layout of a warp buffer: one pad word per 16 coefficients,
// phys(j) = j + (j >> 4).  For N = 2^10 every pass pattern (group stride 64,
// 4 and 1) is bank-conflict free, and inside a group the offsets
// phys(base + i LO) - phys(base) are compile-time constants (pad_off), so
// each shared access is one LDS/STS with an immediate offset.
constexpr int kWarpBuf = kWarpElems + kWarpElems / 16;
__device__ __forceinline__ int wpad(int j) { return j + (j >> 4); }
template <int LOGN, int S, int LO>
__host__ __device__ constexpr int pad_off(int i) {
  return ((1 << (LOGN - S)) >= 16) ? i * LO + ((i * LO) >> 4) : i * LO;
}

__device__ __forceinline__ void cp_async8(void* smem, const void* gmem) {
  unsigned s = (unsigned)__cvta_generic_to_shared(smem);
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"(s), "l"(gmem) : "memory");
}
__device__ __forceinline__ void cp_async_wait_all() { asm volatile("cp.async.wait_all;\n" ::: "memory"); }

// Geometry of group G (0 .. 1024/2^K - 1) of a pass covering stages [S, S+K):
// element j = hi 2^{n-S} + lo + i 2^{n-S-K} of polynomial `poly` in the warp.
template <int LOGN, int S, int K>
struct PassGeo {
  static constexpr int N = 1 << LOGN;
  static constexpr int R = 1 << K;
  static constexpr int LO = 1 << (LOGN - S - K);   // element stride inside a group
  static constexpr int GPP = N / R;                // groups per polynomial
  static constexpr int GPL = (kWarpElems / R) / 32;
  int poly, hi, base;                              // base = warp-buffer index of i = 0
  __device__ __forceinline__ PassGeo(int G) {
    poly = G / GPP;
    const int gl = G % GPP;
    hi = gl / LO;
    base = poly * N + hi * (N >> S) + (gl % LO);
  }
};

// K CT stages on x[0 .. 2^K) of one group; twiddle w[2^{S+v} + hi 2^v + blk].
template <int S, int K>
__device__ __forceinline__ void ct_group(u64 (&x)[1 << K], const TW* T, int hi, u64 q, u64 q2) {
  sfor<0, K>([&](auto V_) {
    constexpr int v = decltype(V_)::value;
    constexpr int half = (1 << K) >> (v + 1);
#pragma unroll
    for (int blk = 0; blk < (1 << v); ++blk) {
      TW w = ldg_tw(T + (1 << (S + v)) + hi * (1 << v) + blk);
#pragma unroll
      for (int k = 0; k < half; ++k) ct_bfly(x[blk * 2 * half + k], x[blk * 2 * half + k + half], w, q, q2);
    }
  });
}

// K GS stages (reverse order).  If LAST (S == 0), local stage 0 is the final
// stage of the inverse and carries the N^{-1} (or N^{-1} R) factor.
template <int S, int K, bool LAST>
__device__ __forceinline__ void gs_group(u64 (&x)[1 << K], const TW* T, int hi, TW s0, TW s1, u64 q, u64 q2) {
  sfor<0, K>([&](auto I_) {
    constexpr int v = K - 1 - decltype(I_)::value;
    constexpr int half = (1 << K) >> (v + 1);
    if constexpr (LAST && v == 0) {
#pragma unroll
      for (int k = 0; k < half; ++k) gs_bfly_last(x[k], x[k + half], s0, s1, q, q2);
    } else {
#pragma unroll
      for (int blk = 0; blk < (1 << v); ++blk) {
        TW w = ldg_tw(T + (1 << (S + v)) + hi * (1 << v) + blk);
#pragma unroll
        for (int k = 0; k < half; ++k) gs_bfly(x[blk * 2 * half + k], x[blk * 2 * half + k + half], w, q, q2);
      }
    }
  });
}

// Global view of the polynomials a warp works on: polynomial p of the warp is
// unit (u0 + p) of one limb; element jj of it lives at base + (u0+p)*stride + jj
// (stride = L*N for the [B][L][N] layout; 0 for a broadcast operand).
struct GView {
  const u64* base;
  uint64_t u0, stride, units;
  __device__ __forceinline__ bool live(int p) const { return u0 + p < units; }
  __device__ __forceinline__ const u64* at(int p) const { return base + (u0 + p) * stride; }
};

// Destination kinds of a pass.
constexpr int kToBuf = 0;      // lazy values back into the warp buffer
constexpr int kToGlobal = 1;   // canonical values to global memory
constexpr int kToBufCanon = 2; // canonical values into the warp buffer

// ---- one forward pass (CT) over the warp buffer -----------------------------
template <int LOGN, int S, int K, bool SRC_GLOBAL, int DST>
__device__ __forceinline__ void fwd_pass(u64* buf, GView src, GView dst, int lane, const TW* T, u64 q, u64 q2) {
  using Geo = PassGeo<LOGN, S, K>;
  constexpr int N = 1 << LOGN;
#pragma unroll 1
  for (int gi = 0; gi < Geo::GPL; ++gi) {
    const Geo g(lane + 32 * gi);
    const int jj0 = g.base - g.poly * N;
    const int pb = wpad(g.base);
    u64 x[1 << K];
    if constexpr (SRC_GLOBAL) {
      const bool live = src.live(g.poly);
      const u64* s = src.at(g.poly) + jj0;
#pragma unroll
      for (int i = 0; i < (1 << K); ++i) x[i] = live ? s[i * Geo::LO] : 0ull;
    } else {
#pragma unroll
      for (int i = 0; i < (1 << K); ++i) x[i] = buf[pb + pad_off<LOGN, S, Geo::LO>(i)];
    }
    ct_group<S, K>(x, T, g.hi, q, q2);
    if constexpr (DST == kToGlobal) {
      if (dst.live(g.poly)) {
        u64* d = const_cast<u64*>(dst.at(g.poly)) + jj0;
#pragma unroll
        for (int i = 0; i < (1 << K); ++i) d[i * Geo::LO] = canon4(x[i], q, q2);
      }
    } else {
#pragma unroll
      for (int i = 0; i < (1 << K); ++i)
        buf[pb + pad_off<LOGN, S, Geo::LO>(i)] = DST == kToBufCanon ? canon4(x[i], q, q2) : x[i];
    }
  }
  __syncwarp();
}

template <int LOGN, int S, int K, bool SRC_GLOBAL, bool DST_GLOBAL, bool LAST>
__device__ __forceinline__ void inv_pass(u64* buf, GView src, GView dst, int lane, const TW* T, TW s0, TW s1,
                                         u64 q, u64 q2) {
  using Geo = PassGeo<LOGN, S, K>;
  constexpr int N = 1 << LOGN;
#pragma unroll 1
  for (int gi = 0; gi < Geo::GPL; ++gi) {
    const Geo g(lane + 32 * gi);
    const int jj0 = g.base - g.poly * N;
    const int pb = wpad(g.base);
    u64 x[1 << K];
    if constexpr (SRC_GLOBAL) {
      const bool live = src.live(g.poly);
      const u64* s = src.at(g.poly) + jj0;
#pragma unroll
      for (int i = 0; i < (1 << K); ++i) x[i] = live ? s[i * Geo::LO] : 0ull;
    } else {
#pragma unroll
      for (int i = 0; i < (1 << K); ++i) x[i] = buf[pb + pad_off<LOGN, S, Geo::LO>(i)];
    }
    gs_group<S, K, LAST>(x, T, g.hi, s0, s1, q, q2);
    if constexpr (DST_GLOBAL) {
      if (dst.live(g.poly)) {
        u64* d = const_cast<u64*>(dst.at(g.poly)) + jj0;
#pragma unroll
        for (int i = 0; i < (1 << K); ++i) d[i * Geo::LO] = canon2(x[i], q);
      }
    } else {
#pragma unroll
      for (int i = 0; i < (1 << K); ++i) buf[pb + pad_off<LOGN, S, Geo::LO>(i)] = x[i];
    }
  }
  __syncwarp();
}

// Fused turn-around pass of the polymul: last CT pass -> (.) b_hat -> first
// GS pass, all in registers.  b_hat comes from global memory (bview) or from
// a second warp buffer holding canonical NTT(b) (BSRC_BUF).
template <int LOGN, int S, int K, bool SRC_GLOBAL, bool DST_GLOBAL, bool BSRC_BUF>
__device__ __forceinline__ void turn_pass(u64* buf, GView src, GView dst, GView bview, const u64* bbuf, int lane,
                                          const TW* Tf, const TW* Ti, TW s0, TW s1, u64 q, u64 q2, u64 qinv) {
  using Geo = PassGeo<LOGN, S, K>;
  constexpr int N = 1 << LOGN;
#pragma unroll 1
  for (int gi = 0; gi < Geo::GPL; ++gi) {
    const Geo g(lane + 32 * gi);
    const int jj0 = g.base - g.poly * N;
    const int pb = wpad(g.base);
    u64 x[1 << K];
    if constexpr (SRC_GLOBAL) {
      const bool live = src.live(g.poly);
      const u64* s = src.at(g.poly) + jj0;
#pragma unroll
      for (int i = 0; i < (1 << K); ++i) x[i] = live ? s[i * Geo::LO] : 0ull;
    } else {
#pragma unroll
      for (int i = 0; i < (1 << K); ++i) x[i] = buf[pb + pad_off<LOGN, S, Geo::LO>(i)];
    }
    ct_group<S, K>(x, Tf, g.hi, q, q2);
    if constexpr (BSRC_BUF) {
#pragma unroll
      for (int i = 0; i < (1 << K); ++i) x[i] = mont_mul(x[i], bbuf[pb + pad_off<LOGN, S, Geo::LO>(i)], q, qinv);
    } else {
      const bool live = bview.live(g.poly);
      const u64* b = bview.at(g.poly) + jj0;
#pragma unroll
      for (int i = 0; i < (1 << K); ++i) x[i] = mont_mul(x[i], live ? __ldg(b + i * Geo::LO) : 0ull, q, qinv);
    }
    gs_group<S, K, S == 0>(x, Ti, g.hi, s0, s1, q, q2);
    if constexpr (DST_GLOBAL) {
      if (dst.live(g.poly)) {
        u64* d = const_cast<u64*>(dst.at(g.poly)) + jj0;
#pragma unroll
        for (int i = 0; i < (1 << K); ++i) d[i * Geo::LO] = canon2(x[i], q);
      }
    } else {
#pragma unroll
      for (int i = 0; i < (1 << K); ++i) buf[pb + pad_off<LOGN, S, Geo::LO>(i)] = x[i];
    }
  }
  __syncwarp();
}

// ---- full transforms on one warp buffer ---------------------------------------
template <int LOGN, int DST, bool SYNC = false>
__device__ __forceinline__ void warp_forward(u64* buf, GView src, GView dst, int lane, const TW* T, u64 q, u64 q2) {
  using C = WarpCfg<LOGN>;
  if constexpr (C::NPASS == 1) {
    fwd_pass<LOGN, 0, C::K0, true, DST>(buf, src, dst, lane, T, q, q2);
    if constexpr (SYNC) __syncthreads();
  } else if constexpr (C::NPASS == 2) {
    fwd_pass<LOGN, 0, C::K0, true, kToBuf>(buf, src, dst, lane, T, q, q2);
    if constexpr (SYNC) __syncthreads();
    fwd_pass<LOGN, C::K0, C::K1, false, DST>(buf, src, dst, lane, T, q, q2);
    if constexpr (SYNC) __syncthreads();
  } else {
    fwd_pass<LOGN, 0, C::K0, true, kToBuf>(buf, src, dst, lane, T, q, q2);
    if constexpr (SYNC) __syncthreads();
    fwd_pass<LOGN, C::K0, C::K1, false, kToBuf>(buf, src, dst, lane, T, q, q2);
    if constexpr (SYNC) __syncthreads();
    fwd_pass<LOGN, C::K0 + C::K1, C::K2, false, DST>(buf, src, dst, lane, T, q, q2);
    if constexpr (SYNC) __syncthreads();
  }
}

template <int LOGN, bool SYNC = false>
__device__ __forceinline__ void warp_inverse(u64* buf, GView src, GView dst, int lane, const TW* T, TW s0, TW s1,
                                             u64 q, u64 q2) {
  using C = WarpCfg<LOGN>;
  if constexpr (C::NPASS == 1) {
    inv_pass<LOGN, 0, C::K0, true, true, true>(buf, src, dst, lane, T, s0, s1, q, q2);
    if constexpr (SYNC) __syncthreads();
  } else if constexpr (C::NPASS == 2) {
    inv_pass<LOGN, C::K0, C::K1, true, false, false>(buf, src, dst, lane, T, s0, s1, q, q2);
    if constexpr (SYNC) __syncthreads();
    inv_pass<LOGN, 0, C::K0, false, true, true>(buf, src, dst, lane, T, s0, s1, q, q2);
    if constexpr (SYNC) __syncthreads();
  } else {
    inv_pass<LOGN, C::K0 + C::K1, C::K2, true, false, false>(buf, src, dst, lane, T, s0, s1, q, q2);
    if constexpr (SYNC) __syncthreads();
    inv_pass<LOGN, C::K0, C::K1, false, false, false>(buf, src, dst, lane, T, s0, s1, q, q2);
    if constexpr (SYNC) __syncthreads();
    inv_pass<LOGN, 0, C::K0, false, true, true>(buf, src, dst, lane, T, s0, s1, q, q2);
    if constexpr (SYNC) __syncthreads();
  }
}

template <int LOGN, bool BSRC_BUF, bool SYNC = false>
__device__ __forceinline__ void warp_polymul(u64* buf, GView src, GView dst, GView bview, const u64* bbuf, int lane,
                                             const TW* Tf, const TW* Ti, TW s0, TW s1, u64 q, u64 q2, u64 qinv) {
  using C = WarpCfg<LOGN>;
  if constexpr (C::NPASS == 1) {
    turn_pass<LOGN, 0, C::K0, true, true, BSRC_BUF>(buf, src, dst, bview, bbuf, lane, Tf, Ti, s0, s1, q, q2, qinv);
    if constexpr (SYNC) __syncthreads();
  } else if constexpr (C::NPASS == 2) {
    fwd_pass<LOGN, 0, C::K0, true, kToBuf>(buf, src, dst, lane, Tf, q, q2);
    if constexpr (SYNC) __syncthreads();
    turn_pass<LOGN, C::K0, C::K1, false, false, BSRC_BUF>(buf, src, dst, bview, bbuf, lane, Tf, Ti, s0, s1, q, q2,
                                                          qinv);
                                                          if constexpr (SYNC) __syncthreads();
    inv_pass<LOGN, 0, C::K0, false, true, true>(buf, src, dst, lane, Ti, s0, s1, q, q2);
    if constexpr (SYNC) __syncthreads();
  } else {
    fwd_pass<LOGN, 0, C::K0, true, kToBuf>(buf, src, dst, lane, Tf, q, q2);
    if constexpr (SYNC) __syncthreads();
    fwd_pass<LOGN, C::K0, C::K1, false, kToBuf>(buf, src, dst, lane, Tf, q, q2);
    if constexpr (SYNC) __syncthreads();
    turn_pass<LOGN, C::K0 + C::K1, C::K2, false, false, BSRC_BUF>(buf, src, dst, bview, bbuf, lane, Tf, Ti, s0, s1,
                                                                  q, q2, qinv);
                                                                  if constexpr (SYNC) __syncthreads();
    inv_pass<LOGN, C::K0, C::K1, false, false, false>(buf, src, dst, lane, Ti, s0, s1, q, q2);
    if constexpr (SYNC) __syncthreads();
    inv_pass<LOGN, 0, C::K0, false, true, true>(buf, src, dst, lane, Ti, s0, s1, q, q2);
    if constexpr (SYNC) __syncthreads();
  }
}

// ---- kernel --------------------------------------------------------------------
// grid = (ceil(B / (kTeamWarps * P)), L): CTA (x, l) owns polynomials
// [x * kTeamWarps * P, ...) of limb l; unit (b, l) sits at (b L + l) N
// (layout [B][L][N], reading C10).
// MODE 0: forward, 1: inverse, 2: c = INTT(NTT(a) (.) b_hat), 3: c = INTT(NTT(a) (.) NTT(b)).
template <int LOGN, int MODE, int W = kTeamWarps, int MINB = 1, bool SYNC = false>
__global__ void __launch_bounds__(W * 32, MINB)
k_warp(u64* __restrict__ out, const u64* __restrict__ in, const u64* __restrict__ bop, int b_bcast,
       const TW* __restrict__ tw_fwd, const TW* __restrict__ tw_inv, const LimbC* __restrict__ lc,
       uint32_t L, uint32_t B) {
  using C = WarpCfg<LOGN>;
  constexpr int N = C::N;
  extern __shared__ __align__(16) u64 smem[];
  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  const uint32_t l = blockIdx.y;
  const uint64_t p0 = ((uint64_t)blockIdx.x * W + warp) * C::P;
  if (!SYNC && p0 >= B) return;   // whole warp idle (warp-uniform); with SYNC idle warps run predicated
  u64* buf = smem + (size_t)warp * kWarpBuf * (MODE == 3 ? 2 : 1);
  const u64 q = lc[l].q, q2 = lc[l].q2;
  const uint64_t stride = (uint64_t)L * N;
  const GView src{in + (uint64_t)l * N, p0, stride, B};
  const GView dst{out + (uint64_t)l * N, p0, stride, B};
  const TW* Tf = tw_fwd + (size_t)l * N;
  const TW* Ti = tw_inv + (size_t)l * N;
  if constexpr (MODE == 0) {
    warp_forward<LOGN, kToGlobal, SYNC>(buf, src, dst, lane, Tf, q, q2);
  } else if constexpr (MODE == 1) {
    warp_inverse<LOGN, SYNC>(buf, src, dst, lane, Ti, lc[l].ninv, lc[l].ninv_w1, q, q2);
  } else {
    const GView bview{bop + (uint64_t)l * N, b_bcast ? 0 : p0, b_bcast ? 0 : stride, b_bcast ? ~0ull : B};
    const u64 qinv = lc[l].qinv;
    if constexpr (MODE == 3) {
      u64* bbuf = buf + kWarpBuf;
      // canonical NTT(b) parked in the second warp buffer
      warp_forward<LOGN, kToBufCanon, SYNC>(bbuf, bview, bview, lane, Tf, q, q2);
      warp_polymul<LOGN, true, SYNC>(buf, src, dst, bview, bbuf, lane, Tf, Ti, lc[l].ninvR, lc[l].ninvR_w1, q, q2, qinv);
    } else {
      warp_polymul<LOGN, false, SYNC>(buf, src, dst, bview, nullptr, lane, Tf, Ti, lc[l].ninvR, lc[l].ninvR_w1, q, q2,
                                qinv);
    }
  }
}

template <int LOGN, int MODE, int W = kTeamWarps>
inline size_t warp_smem_bytes() {
  return (size_t)W * kWarpBuf * 8 * (MODE == 3 ? 2 : 1);
}

}  // namespace rnt
