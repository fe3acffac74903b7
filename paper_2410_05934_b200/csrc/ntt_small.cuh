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
// Group-loop unroll of the 4-coefficient (K = 2) passes: 2 groups per iteration give
// each stage 4 independent butterflies instead of 2 (experiment builds:
// -DRNT_K2_UNROLL=n; the 8-coefficient passes stay rolled for the register budget).
#ifndef RNT_K2_UNROLL
#define RNT_K2_UNROLL 1
#endif
constexpr int kK2Unroll = RNT_K2_UNROLL;

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

// A warp buffer is worked on by a team of warps (TEAM = 1: one warp, the
// default).  The team's lanes split every pass's groups; between passes the team
// synchronises with __syncwarp (one warp), __syncthreads (TEAM = 2, 4: the team is
// the whole CTA) or a named barrier (TEAM = -2: teams of 2 warps inside a larger
// CTA, barrier id 1 + warp / 2, 64 threads).
template <int TEAM>
struct Team {
  static constexpr int size = TEAM > 0 ? TEAM : -TEAM;
  static constexpr bool named = TEAM < 0;
};
template <int TEAM>
__device__ __forceinline__ void team_sync() {
  if constexpr (Team<TEAM>::size == 1) {
    __syncwarp();
  } else if constexpr (Team<TEAM>::named) {
    asm volatile("bar.sync %0, %1;" ::"r"(1 + (int)(threadIdx.x >> 5) / Team<TEAM>::size), "n"(32 * Team<TEAM>::size)
                 : "memory");
  } else {
    __syncthreads();
  }
}

// K CT stages on x[0 .. 2^K) of one group; twiddle w[2^{S+v} + hi 2^v + blk].
// LZ: lazy ranges for q < 2^60 (ct_bfly_lz; input canonical at stage 0).
template <int S, int K, bool LZ = false, int S0 = 0>
__device__ __forceinline__ void ct_group(u64 (&x)[1 << K], const TW* T, int hi, u64 q, u64 q2) {
  sfor<0, K>([&](auto V_) {
    constexpr int v = decltype(V_)::value;
    constexpr int half = (1 << K) >> (v + 1);
#pragma unroll
    for (int blk = 0; blk < (1 << v); ++blk) {
      TW w = ldg_tw(T + (1 << (S + v)) + hi * (1 << v) + blk);
#pragma unroll
      for (int k = 0; k < half; ++k) {
        ct_bfly_at<LZ, S0 + S + v>(x[blk * 2 * half + k], x[blk * 2 * half + k + half], w, q, q2);
      }
    }
  });
}

// canonical value of a forward output (lazy bound 4q, or 16q with LZ)
template <bool LZ>
__device__ __forceinline__ u64 canon_fwd(u64 x, u64 q, u64 q2) {
  if constexpr (LZ) return canon16(x, q, q2);
  else return canon4(x, q, q2);
}

// K GS stages (reverse order).  If LAST (S == 0), local stage 0 is the final
// stage of the inverse and carries the N^{-1} (or N^{-1} R) factor.
// LZT: the inverse ends with the scaled stage 0 and q < 2^60: global stages
// 2, 1, 0 skip the sum reduction (gs_bfly_nr / gs_bfly_last_nr).
template <int S, int K, bool LAST, bool MIRROR = false, bool LZT = false>
__device__ __forceinline__ void gs_group(u64 (&x)[1 << K], const TW* T, int hi, TW s0, TW s1, u64 q, u64 q2) {
  static_assert(!(LZT && MIRROR), "LZ tail needs the scaled last stage");
  sfor<0, K>([&](auto I_) {
    constexpr int v = K - 1 - decltype(I_)::value;
    constexpr int half = (1 << K) >> (v + 1);
    if constexpr (LAST && v == 0) {
#pragma unroll
      for (int k = 0; k < half; ++k) {
        if constexpr (LZT && S == 0) gs_bfly_last_nr<8>(x[k], x[k + half], s0, s1, q, q2);
        else gs_bfly_last(x[k], x[k + half], s0, s1, q, q2);
      }
    } else if constexpr (LZT && S + v <= 2) {
#pragma unroll
      for (int blk = 0; blk < (1 << v); ++blk) {
        TW w = ldg_tw(T + (1 << (S + v)) + hi * (1 << v) + blk);
#pragma unroll
        for (int k = 0; k < half; ++k)
          gs_bfly_nr<(2 << (2 - (S + v)))>(x[blk * 2 * half + k], x[blk * 2 * half + k + half], w, q, q2);
      }
    } else {
#pragma unroll
      for (int blk = 0; blk < (1 << v); ++blk) {
        if constexpr (MIRROR) {
          // psi^{-brv(k)} = -psi^{brv(3 2^s - 1 - k)}: read the mirrored forward
          // entry and use the negated-twiddle butterfly (ntt_large.cuh rows)
          TW w = ldg_tw(T + (2 << (S + v)) - 1 - (hi * (1 << v) + blk));
#pragma unroll
          for (int k = 0; k < half; ++k) gs_bfly_neg(x[blk * 2 * half + k], x[blk * 2 * half + k + half], w, q, q2);
        } else {
          TW w = ldg_tw(T + (1 << (S + v)) + hi * (1 << v) + blk);
#pragma unroll
          for (int k = 0; k < half; ++k) gs_bfly(x[blk * 2 * half + k], x[blk * 2 * half + k + half], w, q, q2);
        }
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

// Source kinds of a pass.
constexpr int kFromBuf = 0;     // padded warp buffer
constexpr int kFromGlobal = 1;  // global memory (GView)

// Destination kinds of a pass.
constexpr int kToBuf = 0;      // lazy values back into the warp buffer
constexpr int kToGlobal = 1;   // canonical values to global memory
constexpr int kToBufCanon = 2; // canonical values into the warp buffer

// ---- one forward pass (CT) over the warp buffer -----------------------------
// TWS: twiddle-table stride per polynomial of the warp (0: all polynomials
// share T; 2^{n2}: row r + p of a 2^16 limb uses row table r + p).
// S0: global index of local stage 0 (rows of a 2^16 limb: n1), for the LZ schedule.
template <int LOGN, int S, int K, int SRC, int DST, int TWS = 0, bool LZ = false, int S0 = 0, int TEAM = 1>
__device__ __forceinline__ void fwd_pass(u64* buf, GView src, GView dst, int lane, const TW* T, u64 q, u64 q2) {
  using Geo = PassGeo<LOGN, S, K>;
  constexpr int N = 1 << LOGN;
  constexpr int TS = Team<TEAM>::size;
  static_assert(Geo::GPL % TS == 0, "team splits the groups evenly");
#pragma unroll(K == 2 ? kK2Unroll : 1)
  for (int gi = 0; gi < Geo::GPL / TS; ++gi) {
    const Geo g(lane + 32 * TS * gi);
    const int jj0 = g.base - g.poly * N;
    const int pb = wpad(g.base);
    u64 x[1 << K];
    if constexpr (SRC == kFromGlobal) {
      const bool live = src.live(g.poly);
      const u64* s = src.at(g.poly) + jj0;
#pragma unroll
      for (int i = 0; i < (1 << K); ++i) x[i] = live ? s[i * Geo::LO] : 0ull;
    } else {
#pragma unroll
      for (int i = 0; i < (1 << K); ++i) x[i] = buf[pb + pad_off<LOGN, S, Geo::LO>(i)];
    }
    ct_group<S, K, LZ, S0>(x, T + g.poly * TWS, g.hi, q, q2);
    if constexpr (DST == kToGlobal) {
      if (dst.live(g.poly)) {
        u64* d = const_cast<u64*>(dst.at(g.poly)) + jj0;
#pragma unroll
        for (int i = 0; i < (1 << K); ++i) d[i * Geo::LO] = canon_fwd<LZ>(x[i], q, q2);
      }
    } else {
#pragma unroll
      for (int i = 0; i < (1 << K); ++i)
        buf[pb + pad_off<LOGN, S, Geo::LO>(i)] = DST == kToBufCanon ? canon_fwd<LZ>(x[i], q, q2) : x[i];
    }
  }
  team_sync<TEAM>();
}

template <int LOGN, int S, int K, int SRC, bool DST_GLOBAL, bool LAST, int TWS = 0, bool MIRROR = false,
          bool LZT = false, int TEAM = 1>
__device__ __forceinline__ void inv_pass(u64* buf, GView src, GView dst, int lane, const TW* T, TW s0, TW s1,
                                         u64 q, u64 q2) {
  using Geo = PassGeo<LOGN, S, K>;
  constexpr int N = 1 << LOGN;
  constexpr int TS = Team<TEAM>::size;
  static_assert(Geo::GPL % TS == 0, "team splits the groups evenly");
#pragma unroll(K == 2 ? kK2Unroll : 1)
  for (int gi = 0; gi < Geo::GPL / TS; ++gi) {
    const Geo g(lane + 32 * TS * gi);
    const int jj0 = g.base - g.poly * N;
    const int pb = wpad(g.base);
    u64 x[1 << K];
    if constexpr (SRC == kFromGlobal) {
      const bool live = src.live(g.poly);
      const u64* s = src.at(g.poly) + jj0;
#pragma unroll
      for (int i = 0; i < (1 << K); ++i) x[i] = live ? s[i * Geo::LO] : 0ull;
    } else {
#pragma unroll
      for (int i = 0; i < (1 << K); ++i) x[i] = buf[pb + pad_off<LOGN, S, Geo::LO>(i)];
    }
    gs_group<S, K, LAST, MIRROR, LZT>(x, MIRROR ? T - g.poly * TWS : T + g.poly * TWS, g.hi, s0, s1, q, q2);
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
  team_sync<TEAM>();
}

// Fused turn-around pass of the polymul: last CT pass -> (.) b_hat -> first
// GS pass, all in registers.  b_hat comes from global memory (bview) or from
// a second warp buffer holding canonical NTT(b) (BSRC == kFromBuf).
template <int LOGN, int S, int K, int SRC, bool DST_GLOBAL, int BSRC, bool SCALE = true, int TWS = 0,
          bool MIRROR = false, bool LZ = false, int S0 = 0, int TEAM = 1>
__device__ __forceinline__ void turn_pass(u64* buf, GView src, GView dst, GView bview, const u64* bbuf, int lane,
                                          const TW* Tf, const TW* Ti, TW s0, TW s1, u64 q, u64 q2, u64 qinv) {
  using Geo = PassGeo<LOGN, S, K>;
  constexpr int N = 1 << LOGN;
  constexpr int TS = Team<TEAM>::size;
  static_assert(Geo::GPL % TS == 0, "team splits the groups evenly");
#pragma unroll(K == 2 ? kK2Unroll : 1)
  for (int gi = 0; gi < Geo::GPL / TS; ++gi) {
    const Geo g(lane + 32 * TS * gi);
    const int jj0 = g.base - g.poly * N;
    const int pb = wpad(g.base);
    u64 x[1 << K];
    if constexpr (SRC == kFromGlobal) {
      const bool live = src.live(g.poly);
      const u64* s = src.at(g.poly) + jj0;
#pragma unroll
      for (int i = 0; i < (1 << K); ++i) x[i] = live ? s[i * Geo::LO] : 0ull;
    } else {
#pragma unroll
      for (int i = 0; i < (1 << K); ++i) x[i] = buf[pb + pad_off<LOGN, S, Geo::LO>(i)];
    }
    // b_hat is fetched before the CT stages so its latency hides behind them
    u64 bv[1 << K];
    if constexpr (BSRC == kFromBuf) {
#pragma unroll
      for (int i = 0; i < (1 << K); ++i) bv[i] = bbuf[pb + pad_off<LOGN, S, Geo::LO>(i)];
    } else {
      const bool live = bview.live(g.poly);
      const u64* b = bview.at(g.poly) + jj0;
#pragma unroll
      for (int i = 0; i < (1 << K); ++i) bv[i] = live ? __ldg(b + i * Geo::LO) : 0ull;
    }
    ct_group<S, K, LZ, S0>(x, Tf + g.poly * TWS, g.hi, q, q2);
    // a < 16q (LZ, q < 2^60) or < 4q, b_hat < q: a b < q 2^64, result in (0, 2q)
#pragma unroll
    for (int i = 0; i < (1 << K); ++i) x[i] = mont_mul(x[i], bv[i], q, qinv);
    gs_group<S, K, SCALE && S == 0, MIRROR, LZ && SCALE>(x, MIRROR ? Ti - g.poly * TWS : Ti + g.poly * TWS, g.hi, s0,
                                                         s1, q, q2);
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
  team_sync<TEAM>();
}

// ---- full transforms on one warp buffer ---------------------------------------
// Pass schedule: stages grouped into passes of KM (the last takes the
// remainder), e.g. N = 2^10: KM = 4 -> 4 + 4 + 2, KM = 3 -> 3 + 3 + 3 + 1.
template <int LOGN, int KM>
struct Passes {
  // KM >= 10 encodes radix KM / 10 with a split tail: when LOGN leaves a
  // remainder of 1, the last two passes take (B - 1, 2) stages instead of (B, 1)
  // (N = 2^10, KM = 32: 3 + 3 + 2 + 2), so the fused polymul turn pass holds
  // 4-coefficient groups.
  static constexpr int B = KM >= 10 ? KM / 10 : KM;
  static constexpr int NP = (LOGN + B - 1) / B;
  static constexpr bool SPLIT = KM >= 10 && NP >= 2 && LOGN - B * (NP - 1) == 1 && B >= 3;
  __host__ __device__ static constexpr int k(int p) {
    return SPLIT ? (p < NP - 2 ? B : (p == NP - 2 ? B - 1 : 2)) : (p < NP - 1 ? B : LOGN - B * (NP - 1));
  }
  __host__ __device__ static constexpr int s(int p) { return (SPLIT && p == NP - 1) ? B * (NP - 2) + B - 1 : p * B; }
};
static_assert(Passes<10, 32>::k(2) == 2 && Passes<10, 32>::k(3) == 2 && Passes<10, 32>::s(3) == 8, "split tail");
static_assert(Passes<10, 3>::k(3) == 1 && Passes<10, 3>::s(3) == 9, "radix-8 schedule");

// SRC0: source of the first pass (kFromGlobal, or kFromBuf for data already staged).
template <int LOGN, int KM, int DST, bool SYNC = false, int TWS = 0, bool LZ = false, int S0 = 0,
          int SRC0 = kFromGlobal, int TEAM = 1>
__device__ __forceinline__ void warp_forward(u64* buf, GView src, GView dst, int lane, const TW* T, u64 q, u64 q2) {
  using PS = Passes<LOGN, KM>;
  sfor<0, PS::NP>([&](auto P_) {
    constexpr int p = decltype(P_)::value;
    constexpr int SRC = p == 0 ? SRC0 : kFromBuf;
    constexpr int D = p == PS::NP - 1 ? DST : kToBuf;
    fwd_pass<LOGN, PS::s(p), PS::k(p), SRC, D, TWS, LZ, S0, TEAM>(buf, src, dst, lane, T, q, q2);
    if constexpr (SYNC) __syncthreads();
  });
}

template <int LOGN, int KM, bool SYNC = false, bool SCALE = true, int TWS = 0, bool MIRROR = false, bool LZ = false,
          int SRC0 = kFromGlobal, int TEAM = 1>
__device__ __forceinline__ void warp_inverse(u64* buf, GView src, GView dst, int lane, const TW* T, TW s0, TW s1,
                                             u64 q, u64 q2) {
  using PS = Passes<LOGN, KM>;
  sfor<0, PS::NP>([&](auto I_) {
    constexpr int i = decltype(I_)::value;
    constexpr int p = PS::NP - 1 - i;
    constexpr int SRC = i == 0 ? SRC0 : kFromBuf;
    inv_pass<LOGN, PS::s(p), PS::k(p), SRC, p == 0, SCALE && p == 0, TWS, MIRROR, LZ && SCALE, TEAM>(
        buf, src, dst, lane, T, s0, s1, q, q2);
    if constexpr (SYNC) __syncthreads();
  });
}

template <int LOGN, int KM, int BSRC, bool SYNC = false, bool SCALE = true, int TWS = 0, bool MIRROR = false,
          bool LZ = false, int S0 = 0, int SRC0 = kFromGlobal, int TEAM = 1>
__device__ __forceinline__ void warp_polymul(u64* buf, GView src, GView dst, GView bview, const u64* bbuf, int lane,
                                             const TW* Tf, const TW* Ti, TW s0, TW s1, u64 q, u64 q2, u64 qinv) {
  using PS = Passes<LOGN, KM>;
  constexpr int NP = PS::NP;
  sfor<0, NP - 1>([&](auto P_) {
    constexpr int p = decltype(P_)::value;
    fwd_pass<LOGN, PS::s(p), PS::k(p), p == 0 ? SRC0 : kFromBuf, kToBuf, TWS, LZ, S0, TEAM>(buf, src, dst, lane, Tf,
                                                                                                  q, q2);
    if constexpr (SYNC) __syncthreads();
  });
  turn_pass<LOGN, PS::s(NP - 1), PS::k(NP - 1), NP == 1 ? SRC0 : kFromBuf, NP == 1, BSRC, SCALE, TWS, MIRROR,
            LZ, S0, TEAM>(
      buf, src, dst, bview, bbuf, lane, Tf, Ti, s0, s1, q, q2, qinv);
  if constexpr (SYNC) __syncthreads();
  sfor<0, NP - 1>([&](auto I_) {
    constexpr int p = NP - 2 - decltype(I_)::value;
    inv_pass<LOGN, PS::s(p), PS::k(p), kFromBuf, p == 0, SCALE && p == 0, TWS, MIRROR, LZ && SCALE, TEAM>(
        buf, src, dst, lane, Ti, s0, s1, q, q2);
    if constexpr (SYNC) __syncthreads();
  });
}

// ---- kernel --------------------------------------------------------------------
// grid = (ceil(B / (kTeamWarps * P)), L): CTA (x, l) owns polynomials
// [x * kTeamWarps * P, ...) of limb l; unit (b, l) sits at (b L + l) N
// (layout [B][L][N], reading C10).
// MODE 0: forward, 1: inverse, 2: c = INTT(NTT(a) (.) b_hat), 3: c = INTT(NTT(a) (.) NTT(b)).
// LZ: lazy CT ranges (ct_bfly_lz), valid when every modulus of the plan is < 2^60.
// TEAM warps share one warp buffer (TEAM = 1: every warp owns its polynomials;
// TEAM = 2 / 4: a team of warps splits each pass of one buffer -- more, shorter
// work units, for batches that would leave the last wave of the GPU mostly empty).
template <int LOGN, int MODE, int W = kTeamWarps, int MINB = 1, bool SYNC = false, int KM = 4, bool LZ = false,
          int TEAM = 1>
__global__ void __launch_bounds__(W * 32, MINB)
k_warp(u64* __restrict__ out, const u64* __restrict__ in, const u64* __restrict__ bop, int b_bcast,
       const TW* __restrict__ tw_fwd, const TW* __restrict__ tw_inv, const LimbC* __restrict__ lc,
       uint32_t L, uint32_t B) {
  using C = WarpCfg<LOGN>;
  constexpr int N = C::N;
  static_assert((TEAM == 1 || TEAM == W) && !(SYNC && TEAM > 1), "a team is one warp or the whole CTA");
  extern __shared__ __align__(16) u64 smem[];
  const int team = (int)(threadIdx.x >> 5) / TEAM;
  const int lane = (int)threadIdx.x % (32 * TEAM);   // lane within the team
  const uint32_t l = blockIdx.y;
  const uint64_t p0 = ((uint64_t)blockIdx.x * (W / TEAM) + team) * C::P;
  if (!SYNC && p0 >= B) return;   // whole team idle (team-uniform); with SYNC idle warps run predicated
  u64* buf = smem + (size_t)team * kWarpBuf * (MODE == 3 ? 2 : 1);
  const u64 q = lc[l].q, q2 = lc[l].q2;
  const uint64_t stride = (uint64_t)L * N;
  const GView src{in + (uint64_t)l * N, p0, stride, B};
  const GView dst{out + (uint64_t)l * N, p0, stride, B};
  const TW* Tf = tw_fwd + (size_t)l * N;
  const TW* Ti = tw_inv + (size_t)l * N;
  constexpr int SRC0 = kFromGlobal;
  if constexpr (MODE == 0) {
    warp_forward<LOGN, KM, kToGlobal, SYNC, 0, LZ, 0, SRC0, TEAM>(buf, src, dst, lane, Tf, q, q2);
  } else if constexpr (MODE == 1) {
    warp_inverse<LOGN, KM, SYNC, true, 0, false, LZ, SRC0, TEAM>(buf, src, dst, lane, Ti, lc[l].ninv, lc[l].ninv_w1,
                                                                 q, q2);
  } else {
    const GView bview{bop + (uint64_t)l * N, b_bcast ? 0 : p0, b_bcast ? 0 : stride, b_bcast ? ~0ull : B};
    const u64 qinv = lc[l].qinv;
    if constexpr (MODE == 3) {
      u64* bbuf = buf + kWarpBuf;
      // canonical NTT(b) parked in the second warp buffer
      warp_forward<LOGN, KM, kToBufCanon, SYNC, 0, LZ, 0, kFromGlobal, TEAM>(bbuf, bview, bview, lane, Tf, q, q2);
      warp_polymul<LOGN, KM, kFromBuf, SYNC, true, 0, false, LZ, 0, kFromGlobal, TEAM>(
          buf, src, dst, bview, bbuf, lane, Tf, Ti, lc[l].ninvR, lc[l].ninvR_w1, q, q2, qinv);
    } else {
      warp_polymul<LOGN, KM, kFromGlobal, SYNC, true, 0, false, LZ, 0, SRC0, TEAM>(
          buf, src, dst, bview, nullptr, lane, Tf, Ti, lc[l].ninvR, lc[l].ninvR_w1, q, q2, qinv);
    }
  }
}

// ---- TFHE external product ---------------------------------
// c [n_slot][2][N] (RLWE pairs, one prime), rgsw_hat [2l][2][N] (NTT form, shared
// by all slots -- the CMux-level batching of P:324-332 applies one RGSW key to
// n_slot ciphertexts), out [n_slot][2][N]:
//   out_i = INTT( sum_{t,j} NTT(D_{t,j}) (.) rgsw_hat[t l + j][i] ),
// D_{t,j} = signed gadget digit j of c_t (Decompose).  Per warp: the
// digit is formed while the first pass loads c_t; the last forward pass
// multiplies (Montgomery) and accumulates into two shared-memory accumulators;
// two inverse transforms (N^{-1} 2^64 scale) write the output pair.
// Copy the warp's polynomials (padded layout) into buf with 8-byte cp.async:
// every global load is in flight at once (the external product's warps have
// only long-latency work in their first pass).
template <int LOGN>
__device__ __forceinline__ void warp_stage(u64* buf, const GView& src, int lane) {
  constexpr int N = 1 << LOGN;
#pragma unroll 4
  for (int e = lane; e < kWarpElems; e += 32) {
    const int poly = e >> LOGN;
    if (src.live(poly)) cp_async8(buf + wpad(e), src.at(poly) + (e & (N - 1)));
  }
  cp_async_wait_all();
  __syncwarp();
}

struct DigitSpec {
  uint32_t bg, levels;
  int64_t off;     // sum_{i < l-1} (B/2) B^i
  u64 half_q;      // (q - 1) / 2
};

__device__ __forceinline__ u64 gadget_digit(u64 v, u64 q, const DigitSpec& ds, uint32_t j) {
  const int64_t vc = v > ds.half_q ? (int64_t)v - (int64_t)q : (int64_t)v;   // centred
  const int64_t u = vc + ds.off;
  int64_t d;
  if (j + 1 < ds.levels) {
    const int64_t B = (int64_t)1 << ds.bg;
    d = ((u >> (j * ds.bg)) & (B - 1)) - (B >> 1);   // balanced digit
  } else {
    d = u >> (j * ds.bg);                           // last level: the remainder
  }
  return d >= 0 ? (u64)d : q - (u64)(-d);
}

// first forward pass of digit j of component view `src`
// STAGED: the component was already copied into buf (same padded positions,
// warp_stage); the digit is formed from shared memory instead of global memory.
template <int LOGN, int S, int K, bool LZ = false, bool STAGED = false>
__device__ __forceinline__ void fwd_pass_digit(u64* buf, GView src, int lane, const TW* T, u64 q, u64 q2,
                                               const DigitSpec& ds, uint32_t j) {
  using Geo = PassGeo<LOGN, S, K>;
  constexpr int N = 1 << LOGN;
#pragma unroll 1
  for (int gi = 0; gi < Geo::GPL; ++gi) {
    const Geo g(lane + 32 * gi);
    const int jj0 = g.base - g.poly * N;
    const int pb = wpad(g.base);
    const bool live = src.live(g.poly);
    const u64* sp = src.at(g.poly) + jj0;
    u64 x[1 << K];
#pragma unroll
    for (int i = 0; i < (1 << K); ++i) {
      const u64 v = STAGED ? buf[pb + pad_off<LOGN, S, Geo::LO>(i)] : (live ? sp[i * Geo::LO] : 0ull);
      x[i] = live ? gadget_digit(v, q, ds, j) : 0ull;
    }
    ct_group<S, K, LZ>(x, T, g.hi, q, q2);
#pragma unroll
    for (int i = 0; i < (1 << K); ++i) buf[pb + pad_off<LOGN, S, Geo::LO>(i)] = x[i];
  }
  __syncwarp();
}

// last forward pass: CT stages, then acc_i (+)= x (.) z_i (i = 0, 1), kept in
// [0, 2q).  The accumulators live in the output pair itself (NTT domain; L2-
// resident while the slot is in flight), so a warp needs one shared buffer.
template <int LOGN, int S, int K>
__device__ __forceinline__ void fwd_pass_mac(u64* buf, GView acc0v, GView acc1v, const u64* z0, const u64* z1,
                                             bool first, int lane, const TW* T, u64 q, u64 q2, u64 qinv) {
  using Geo = PassGeo<LOGN, S, K>;
  constexpr int N = 1 << LOGN;
#pragma unroll 1
  for (int gi = 0; gi < Geo::GPL; ++gi) {
    const Geo g(lane + 32 * gi);
    const int jj0 = g.base - g.poly * N;
    const int pb = wpad(g.base);
    u64 x[1 << K];
#pragma unroll
    for (int i = 0; i < (1 << K); ++i) x[i] = buf[pb + pad_off<LOGN, S, Geo::LO>(i)];
    ct_group<S, K>(x, T, g.hi, q, q2);
    if (acc0v.live(g.poly)) {
      u64* a0 = const_cast<u64*>(acc0v.at(g.poly)) + jj0;
      u64* a1 = const_cast<u64*>(acc1v.at(g.poly)) + jj0;
#pragma unroll
      for (int i = 0; i < (1 << K); ++i) {
        const int e = jj0 + i * Geo::LO;
        const u64 m0 = mont_mul(x[i], __ldg(z0 + e), q, qinv);
        const u64 m1 = mont_mul(x[i], __ldg(z1 + e), q, qinv);
        a0[i * Geo::LO] = first ? m0 : csub(a0[i * Geo::LO] + m0, q2);
        a1[i * Geo::LO] = first ? m1 : csub(a1[i * Geo::LO] + m1, q2);
      }
    }
  }
  __syncwarp();
}

template <int LOGN, int KM = 3>
__global__ void __launch_bounds__(2 * 32, 12)
k_extprod(u64* __restrict__ out, const u64* __restrict__ c, const u64* __restrict__ zhat,
          const TW* __restrict__ tw_fwd, const TW* __restrict__ tw_inv, const LimbC* __restrict__ lc,
          uint32_t n_slot, DigitSpec ds) {
  using PS = Passes<LOGN, KM>;
  constexpr int N = 1 << LOGN;
  constexpr int P = kWarpElems / N;
  constexpr int NP = PS::NP;
  static_assert(NP >= 2, "N >= 16");
  extern __shared__ __align__(16) u64 smem[];
  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  const uint64_t s0 = ((uint64_t)blockIdx.x * 2 + warp) * P;
  if (s0 >= n_slot) return;
  u64* buf = smem + (size_t)warp * kWarpBuf;
  const u64 q = lc[0].q, q2 = lc[0].q2, qinv = lc[0].qinv;
  const GView o0{out, s0, 2ull * N, n_slot};
  const GView o1{out + N, s0, 2ull * N, n_slot};
  for (uint32_t t = 0; t < 2; ++t) {
    const GView cv{c + (uint64_t)t * N, s0, 2ull * N, n_slot};
    for (uint32_t j = 0; j < ds.levels; ++j) {
      const uint64_t r = (uint64_t)t * ds.levels + j;
      fwd_pass_digit<LOGN, 0, PS::k(0)>(buf, cv, lane, tw_fwd, q, q2, ds, j);
      sfor<1, NP - 1>([&](auto P_) {
        constexpr int p = decltype(P_)::value;
        fwd_pass<LOGN, PS::s(p), PS::k(p), kFromBuf, kToBuf>(buf, cv, cv, lane, tw_fwd, q, q2);
      });
      fwd_pass_mac<LOGN, PS::s(NP - 1), PS::k(NP - 1)>(buf, o0, o1, zhat + (r * 2 + 0) * N, zhat + (r * 2 + 1) * N,
                                                       r == 0, lane, tw_fwd, q, q2, qinv);
    }
  }
  // INTT of both accumulators in place (N^{-1} 2^64 scale after the Montgomery products)
  warp_inverse<LOGN, KM>(buf, o0, o0, lane, tw_inv, lc[0].ninvR, lc[0].ninvR_w1, q, q2);
  warp_inverse<LOGN, KM>(buf, o1, o1, lane, tw_inv, lc[0].ninvR, lc[0].ninvR_w1, q, q2);
}

// CTA-parallel external product: one CTA per warp-buffer of slots (1024 / N
// slots) and one warp per decomposed polynomial r = t l + j (component t,
// digit j): the 2l forward NTTs run concurrently (k_extprod runs them one after
// another in a single warp), then all threads form
// acc_i[e] = sum_r NTT_r[e] (.) z[r][i][e] (Montgomery, [0, 2q)) in warp buffers
// 0 and 1, and warps 0 / 1 run the two inverse NTTs (N^{-1} 2^64 scale).
// LV = l (digit levels, 1..8); blockDim = 64 l, dynamic shared memory 2 l warp buffers.
// LZ: lazy CT ranges / inverse tail (q < 2^60; the digits are canonical residues).
template <int LOGN, int LV, int KM = 3, bool LZ = false>
__global__ void __launch_bounds__(64 * LV)
k_extprod_cta(u64* __restrict__ out, const u64* __restrict__ c, const u64* __restrict__ zhat,
              const TW* __restrict__ tw_fwd, const TW* __restrict__ tw_inv, const LimbC* __restrict__ lc,
              uint32_t n_slot, DigitSpec ds) {
  using PS = Passes<LOGN, KM>;
  constexpr int N = 1 << LOGN;
  constexpr int P = kWarpElems / N;
  constexpr int NP = PS::NP;
  static_assert(NP >= 2, "N >= 16");
  extern __shared__ __align__(16) u64 smem[];
  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  constexpr int NW = 2 * LV;        // warps = decomposed polynomials (ds.levels == LV)
  const uint64_t s0 = (uint64_t)blockIdx.x * P;
  const u64 q = lc[0].q, q2 = lc[0].q2, qinv = lc[0].qinv;
  u64* buf = smem + (size_t)warp * kWarpBuf;
  {
    const uint32_t t = (uint32_t)warp / LV, j = (uint32_t)warp % LV;
    const GView cv{c + (uint64_t)t * N, s0, 2ull * N, n_slot};
    warp_stage<LOGN>(buf, cv, lane);
    fwd_pass_digit<LOGN, 0, PS::k(0), LZ, true>(buf, cv, lane, tw_fwd, q, q2, ds, j);
    sfor<1, NP>([&](auto P_) {
      constexpr int p = decltype(P_)::value;
      fwd_pass<LOGN, PS::s(p), PS::k(p), kFromBuf, kToBuf, 0, LZ>(buf, cv, cv, lane, tw_fwd, q, q2);
    });
  }
  __syncthreads();
  // element e of every warp buffer: slot s0 + e / N, coefficient e % N; each
  // position is read and rewritten by one thread only
#pragma unroll 1
  for (int e = threadIdx.x; e < kWarpElems; e += 32 * NW) {
    const int k = e & (N - 1);
    const int pe = wpad(e);
    u64 z0[NW], z1[NW], x[NW];
#pragma unroll
    for (int r = 0; r < NW; ++r) {   // all loads first: one latency for the whole sum
      z0[r] = __ldg(zhat + (size_t)(2 * r) * N + k);
      z1[r] = __ldg(zhat + (size_t)(2 * r + 1) * N + k);
      x[r] = smem[(size_t)r * kWarpBuf + pe];   // lazy: [0, 15q) (LZ) or [0, 4q)
    }
    u64 a0 = 0, a1 = 0;
    if constexpr (LZ) {
      // exact 128-bit sums, one Montgomery reduction per output instead of one per
      // product: x < 15q (LZ forward output), z < q, NW <= 16 -> T < 240 q^2 < 15 q 2^64
      unsigned __int128 T0 = 0, T1 = 0;
#pragma unroll
      for (int r = 0; r < NW; ++r) {
        T0 += (unsigned __int128)x[r] * z0[r];
        T1 += (unsigned __int128)x[r] * z1[r];
      }
      a0 = redc_sum(T0, q, q2, qinv);
      a1 = redc_sum(T1, q, q2, qinv);
    } else {
#pragma unroll
      for (int r = 0; r < NW; ++r) {
        a0 = csub(a0 + mont_mul(x[r], z0[r], q, qinv), q2);
        a1 = csub(a1 + mont_mul(x[r], z1[r], q, qinv), q2);
      }
    }
    smem[pe] = a0;
    smem[kWarpBuf + pe] = a1;
  }
  __syncthreads();
  if constexpr (NW >= 4) {
    // the two inverse NTTs on teams of two warps (warps 0-1: component 0, warps 2-3:
    // component 1; named barriers), so the inverse phase takes half as long
    if (warp < 4) {
      const int team = warp >> 1;
      const GView o{out + (uint64_t)team * N, s0, 2ull * N, n_slot};
      sfor<0, NP>([&](auto I_) {
        constexpr int p = NP - 1 - decltype(I_)::value;
        inv_pass<LOGN, PS::s(p), PS::k(p), kFromBuf, p == 0, p == 0, 0, false, LZ, -2>(
            smem + (size_t)team * kWarpBuf, o, o, (int)threadIdx.x & 63, tw_inv, lc[0].ninvR, lc[0].ninvR_w1, q, q2);
      });
    }
  } else if (warp < 2) {
    const GView o{out + (uint64_t)warp * N, s0, 2ull * N, n_slot};
    sfor<0, NP>([&](auto I_) {
      constexpr int p = NP - 1 - decltype(I_)::value;
      inv_pass<LOGN, PS::s(p), PS::k(p), kFromBuf, p == 0, p == 0, 0, false, LZ>(buf, o, o, lane, tw_inv,
                                                                                 lc[0].ninvR, lc[0].ninvR_w1, q, q2);
    });
  }
}

template <int LOGN, int MODE, int W = kTeamWarps, int TEAM = 1>
inline size_t warp_smem_bytes() {
  return (size_t)(W / TEAM) * kWarpBuf * 8 * (MODE == 3 ? 2 : 1);
}

}  // namespace rnt

// ============================ latency engine =================================
// One CTA of N/2 threads per (polynomial, limb) unit, one butterfly per thread
// per stage, the polynomial in shared memory, a CTA barrier between stages:
// the loops of Eq. 1 exactly as written (Longa-Naehrig CT forward, GS inverse,
// P:205-213) with the Shoup butterflies of modarith.cuh.  For latency-bound
// jobs (a handful of units, e.g. cfg1's single polynomial), where the warp
// engine would leave one warp doing all N/2 log N butterflies alone.
// MODE 0 forward, 1 inverse, 2 c = INTT(NTT(a) (.) b_hat), 3 c = INTT(NTT(a) (.) NTT(b)).
namespace rnt {

template <int LOGN>
__device__ __forceinline__ void lat_forward(u64* a, const TW* F, u64 q, u64 q2) {   // F: shared-memory table
  constexpr int N = 1 << LOGN;
  const int b = threadIdx.x;
#pragma unroll 1
  for (int m = 1, lt = LOGN - 1; m < N; m <<= 1, --lt) {   // t = 2^lt = N / (2m)
    const int t = 1 << lt;
    const int i = b >> lt, j = 2 * i * t + (b & (t - 1));
    u64 X = a[j], Y = a[j + t];
    ct_bfly(X, Y, F[m + i], q, q2);
    a[j] = X;
    a[j + t] = Y;
    __syncthreads();
  }
}

template <int LOGN, bool AFTER_MONT>
__device__ __forceinline__ void lat_inverse(u64* a, const TW* I, const LimbC& c, u64 q, u64 q2) {
  constexpr int N = 1 << LOGN;
  const int b = threadIdx.x;
#pragma unroll 1
  for (int h = N / 2, lt = 0; h > 1; h >>= 1, ++lt) {       // t = 2^lt, twiddle inv[h + i]
    const int t = 1 << lt;
    const int i = b >> lt, j = 2 * i * t + (b & (t - 1));
    u64 X = a[j], Y = a[j + t];
    gs_bfly(X, Y, I[h + i], q, q2);
    a[j] = X;
    a[j + t] = Y;
    __syncthreads();
  }
  // last stage (h = 1, t = N/2) with the N^{-1} scale folded in (reading C4 / C15)
  u64 X = a[b], Y = a[b + N / 2];
  gs_bfly_last(X, Y, AFTER_MONT ? c.ninvR : c.ninv, AFTER_MONT ? c.ninvR_w1 : c.ninv_w1, q, q2);
  a[b] = canon2(X, q);
  a[b + N / 2] = canon2(Y, q);
}

template <int LOGN, int MODE>
__global__ void __launch_bounds__((1 << LOGN) / 2)
k_lat(u64* __restrict__ out, const u64* __restrict__ in, const u64* __restrict__ bop, int b_bcast,
      const TW* __restrict__ fwd, const TW* __restrict__ inv, const LimbC* __restrict__ lc, uint32_t L) {
  constexpr int N = 1 << LOGN, H = N / 2;
  __shared__ __align__(16) u64 a[N];
  __shared__ __align__(16) u64 bb[MODE == 3 ? N : 1];
  // twiddle tables staged once in shared memory (every stage then reads shared
  // memory, not L2); MODE 3 reuses the forward table's space for the inverse one
  __shared__ __align__(16) TW F[MODE != 1 ? N : 1];
  __shared__ __align__(16) TW Ibuf[(MODE == 1 || MODE == 2) ? N : 1];
  TW* I = MODE == 3 ? F : Ibuf;
  const uint64_t u = blockIdx.x;
  const uint32_t l = (uint32_t)(u % L);
  const LimbC c = lc[l];
  const u64 q = c.q, q2 = c.q2;
  const int b = threadIdx.x;
  if constexpr (MODE != 1) {
    F[b] = ldg_tw(fwd + ((size_t)l << LOGN) + b);
    F[b + H] = ldg_tw(fwd + ((size_t)l << LOGN) + b + H);
  }
  if constexpr (MODE == 1 || MODE == 2) {
    I[b] = ldg_tw(inv + ((size_t)l << LOGN) + b);
    I[b + H] = ldg_tw(inv + ((size_t)l << LOGN) + b + H);
  }
  const u64* src = in + (u << LOGN);
  a[b] = src[b];
  a[b + H] = src[b + H];
  const u64* bsrc = bop ? bop + ((b_bcast ? (uint64_t)l : u) << LOGN) : nullptr;
  if constexpr (MODE == 3) {
    bb[b] = bsrc[b];
    bb[b + H] = bsrc[b + H];
  }
  __syncthreads();
  if constexpr (MODE != 1) lat_forward<LOGN>(a, F, q, q2);
  if constexpr (MODE == 3) {
    lat_forward<LOGN>(bb, F, q, q2);   // ends with a barrier: F is free
    I[b] = ldg_tw(inv + ((size_t)l << LOGN) + b);
    I[b + H] = ldg_tw(inv + ((size_t)l << LOGN) + b + H);
  }
  u64* dst = out + (u << LOGN);
  if constexpr (MODE == 0) {
    dst[b] = canon4(a[b], q, q2);
    dst[b + H] = canon4(a[b + H], q, q2);
    return;
  } else {
    if constexpr (MODE >= 2) {
      const u64 b0 = MODE == 3 ? canon4(bb[b], q, q2) : __ldg(bsrc + b);
      const u64 b1 = MODE == 3 ? canon4(bb[b + H], q, q2) : __ldg(bsrc + b + H);
      a[b] = mont_mul(a[b], b0, q, c.qinv);
      a[b + H] = mont_mul(a[b + H], b1, q, c.qinv);
      __syncthreads();
    }
    lat_inverse<LOGN, (MODE >= 2)>(a, I, c, q, q2);
    dst[b] = a[b];
    dst[b + H] = a[b + H];
  }
}

}  // namespace rnt
