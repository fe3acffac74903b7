// ntt_small.cuh -- one-kernel negacyclic NTT / INTT / fused polymul for
// N = 2^4 .. 2^10 (the TFHE polynomial size), batched over
// (polynomial, limb) units (CMux-level batching).
//
// Decomposition (B200 design, replaces the paper's BD/TA/PCS kernels,
// P:425-498, as prior art): a *team* of S = 2^G lanes owns one
// polynomial, each lane holding E = 2^e = N/S coefficients in registers
// (G = floor(n/2), e = n - G; N=1024: 32 lanes x 32 coefficients, one warp).
//   pass 1: lane l holds coefficients j = l + S*i (i < E).  The first e CT
//           stages (distance t >= S) pair i with i + t/S inside the lane;
//           their twiddles depend only on i (warp-uniform loads).
//   transpose through a swizzled per-team shared-memory buffer (__syncwarp
//           only, no CTA barrier).
//   pass 2: lane l holds j = E*l + i.  The last G stages (t < S <= E) are
//           lane-local again; twiddles come from a lane-major table layout so
//           each load is one coalesced 16-byte-per-lane access.
// So the whole transform has one intra-warp exchange (the paper's
// "synchronisations", drop to one __syncwarp pair) and all global
// traffic is coalesced.  Lazy Harvey ranges (modarith.cuh); outputs are
// canonicalised in the last stage.
#pragma once
#include "modarith.cuh"

namespace rnt {

template <int LOGN>
struct TeamCfg {
  static constexpr int N = 1 << LOGN;
  static constexpr int G = LOGN / 2;
  static constexpr int S = 1 << G;        // lanes per team
  static constexpr int e = LOGN - G;
  static constexpr int E = 1 << e;        // coefficients per lane
  static constexpr int TEAMS = 32 / S;    // teams per warp
};

constexpr int kTeamWarps = 4;             // warps per CTA

// Swizzle of a team buffer index: conflict-free for both j = l + S*i (pass 1)
// and j = E*l + i (pass 2) access patterns.
template <int LOGN>
__device__ __forceinline__ int team_swz(int j) {
  using C = TeamCfg<LOGN>;
  return j ^ ((j >> C::e) & (C::E - 1));
}

// ---- forward stages ------------------------------------------------------
// Pass 1: CT stages s = 0 .. e-1 on x[i] = a[l + S*i]; twiddle w[2^s + (i >> (e-s))].
template <int LOGN>
__device__ __forceinline__ void team_fwd_pass1(u64 (&x)[TeamCfg<LOGN>::E], const TW* T, u64 q, u64 q2) {
  using C = TeamCfg<LOGN>;
  sfor<0, C::e>([&](auto S_) {
    constexpr int s = decltype(S_)::value;
    constexpr int half = C::E >> (s + 1);
#pragma unroll
    for (int blk = 0; blk < (1 << s); ++blk) {
      TW w = ldg_tw(T + (1 << s) + blk);
#pragma unroll
      for (int k = 0; k < half; ++k) ct_bfly(x[blk * 2 * half + k], x[blk * 2 * half + k + half], w, q, q2);
    }
  });
}

// Pass 2: CT stages s = e .. n-1 on x[i] = a[E*l + i]; twiddle of sub-block m
// is at lane-major position 2^s + m*S + l of the team table.
template <int LOGN>
__device__ __forceinline__ void team_fwd_pass2(u64 (&x)[TeamCfg<LOGN>::E], const TW* T, int lane, u64 q, u64 q2) {
  using C = TeamCfg<LOGN>;
  sfor<C::e, LOGN>([&](auto S_) {
    constexpr int s = decltype(S_)::value;
    constexpr int t = C::N >> (s + 1);
#pragma unroll
    for (int m = 0; m < (1 << (s - C::G)); ++m) {
      TW w = ldg_tw(T + (1 << s) + m * C::S + lane);
#pragma unroll
      for (int k = 0; k < t; ++k) ct_bfly(x[m * 2 * t + k], x[m * 2 * t + k + t], w, q, q2);
    }
  });
}

// ---- inverse stages (mirror) ---------------------------------------------
template <int LOGN>
__device__ __forceinline__ void team_inv_pass2(u64 (&x)[TeamCfg<LOGN>::E], const TW* T, int lane, u64 q, u64 q2) {
  using C = TeamCfg<LOGN>;
  sfor<0, LOGN - C::e>([&](auto I_) {
    constexpr int s = LOGN - 1 - decltype(I_)::value;
    constexpr int t = C::N >> (s + 1);
#pragma unroll
    for (int m = 0; m < (1 << (s - C::G)); ++m) {
      TW w = ldg_tw(T + (1 << s) + m * C::S + lane);
#pragma unroll
      for (int k = 0; k < t; ++k) gs_bfly(x[m * 2 * t + k], x[m * 2 * t + k + t], w, q, q2);
    }
  });
}

// GS stages s = e-1 .. 1, then stage 0 with N^{-1} (times s0/s1) folded in.
template <int LOGN>
__device__ __forceinline__ void team_inv_pass1(u64 (&x)[TeamCfg<LOGN>::E], const TW* T, TW s0, TW s1, u64 q, u64 q2) {
  using C = TeamCfg<LOGN>;
  sfor<0, C::e - 1>([&](auto I_) {
    constexpr int s = C::e - 1 - decltype(I_)::value;
    constexpr int half = C::E >> (s + 1);
#pragma unroll
    for (int blk = 0; blk < (1 << s); ++blk) {
      TW w = ldg_tw(T + (1 << s) + blk);
#pragma unroll
      for (int k = 0; k < half; ++k) gs_bfly(x[blk * 2 * half + k], x[blk * 2 * half + k + half], w, q, q2);
    }
  });
#pragma unroll
  for (int k = 0; k < C::E / 2; ++k) gs_bfly_last(x[k], x[k + C::E / 2], s0, s1, q, q2);
}

// ---- shared-memory transposes -----------------------------------------------
template <int LOGN>
__device__ __forceinline__ void team_p1_to_p2(u64 (&x)[TeamCfg<LOGN>::E], u64* buf, int lane) {
  using C = TeamCfg<LOGN>;
#pragma unroll
  for (int i = 0; i < C::E; ++i) buf[team_swz<LOGN>(lane + C::S * i)] = x[i];
  __syncwarp();
#pragma unroll
  for (int i = 0; i < C::E; ++i) x[i] = buf[team_swz<LOGN>(C::E * lane + i)];
  __syncwarp();
}

template <int LOGN>
__device__ __forceinline__ void team_p2_to_p1(u64 (&x)[TeamCfg<LOGN>::E], u64* buf, int lane) {
  using C = TeamCfg<LOGN>;
#pragma unroll
  for (int i = 0; i < C::E; ++i) buf[team_swz<LOGN>(C::E * lane + i)] = x[i];
  __syncwarp();
#pragma unroll
  for (int i = 0; i < C::E; ++i) x[i] = buf[team_swz<LOGN>(lane + C::S * i)];
  __syncwarp();
}

__device__ __forceinline__ void cp_async8(void* smem, const void* gmem) {
  unsigned s = (unsigned)__cvta_generic_to_shared(smem);
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"(s), "l"(gmem) : "memory");
}
__device__ __forceinline__ void cp_async_wait_all() { asm volatile("cp.async.wait_all;\n" ::: "memory"); }

// ---- kernels ------------------------------------------------------------------
// Work unit u = polynomial * L + limb (layout [B][L][N], reading C10).
// MODE 0: forward, 1: inverse, 2: c = INTT(NTT(a) (.) b_hat) (b_hat eval form),
// 3: c = INTT(NTT(a) (.) NTT(b)) (b coefficient form).
template <int LOGN, int MODE>
__global__ void __launch_bounds__(kTeamWarps * 32)
k_team(u64* __restrict__ out, const u64* __restrict__ in, const u64* __restrict__ bop, int b_bcast,
       const TW* __restrict__ tw_fwd, const TW* __restrict__ tw_inv, const LimbC* __restrict__ lc,
       uint32_t L, uint64_t units) {
  using C = TeamCfg<LOGN>;
  extern __shared__ __align__(16) u64 smem[];
  const int warp = threadIdx.x >> 5;
  const int team = (threadIdx.x & 31) / C::S;
  const int lane = threadIdx.x & (C::S - 1);
  const uint64_t u = ((uint64_t)blockIdx.x * kTeamWarps + warp) * C::TEAMS + team;
  const bool active = u < units;
  const uint64_t uu = active ? u : units - 1;   // inactive teams shadow a valid unit, never store
  const uint32_t l = (uint32_t)(uu % L);
  const u64 q = lc[l].q, q2 = lc[l].q2;
  u64* buf = smem + (size_t)((warp * C::TEAMS + team) * (MODE == 3 ? 2 : 1)) * C::N;
  const u64* src = in + uu * C::N;
  u64 x[C::E];

  if (MODE == 1) {
    // inverse: bit-reversed input -> pass-2 layout
#pragma unroll
    for (int i = 0; i < C::E; ++i) x[i] = src[lane + C::S * i];
    team_p1_to_p2<LOGN>(x, buf, lane);
    const TW* Ti = tw_inv + (size_t)l * C::N;
    team_inv_pass2<LOGN>(x, Ti, lane, q, q2);
    team_p2_to_p1<LOGN>(x, buf, lane);
    team_inv_pass1<LOGN>(x, Ti, lc[l].ninv, lc[l].ninv_w1, q, q2);
#pragma unroll
    for (int i = 0; i < C::E; ++i) x[i] = canon2(x[i], q);
  } else {
    const TW* Tf = tw_fwd + (size_t)l * C::N;
    u64* bbuf = buf + C::N;
    if (MODE == 3) {
      // NTT(b) first, parked in pass-2 layout in the second team buffer.
      const u64* bsrc = bop + (b_bcast ? (uint64_t)l : uu) * C::N;
#pragma unroll
      for (int i = 0; i < C::E; ++i) x[i] = bsrc[lane + C::S * i];
      team_fwd_pass1<LOGN>(x, Tf, q, q2);
      team_p1_to_p2<LOGN>(x, buf, lane);
      team_fwd_pass2<LOGN>(x, Tf, lane, q, q2);
#pragma unroll
      for (int i = 0; i < C::E; ++i) bbuf[team_swz<LOGN>(C::E * lane + i)] = canon4(x[i], q, q2);
    }
#pragma unroll
    for (int i = 0; i < C::E; ++i) x[i] = src[lane + C::S * i];
    team_fwd_pass1<LOGN>(x, Tf, q, q2);
    team_p1_to_p2<LOGN>(x, buf, lane);
    if (MODE == 2) {
      // prefetch b_hat into the (now free) team buffer, overlapping pass 2
      const u64* bsrc = bop + (b_bcast ? (uint64_t)l : uu) * C::N;
#pragma unroll
      for (int i = 0; i < C::E; ++i) cp_async8(buf + team_swz<LOGN>(lane + C::S * i), bsrc + lane + C::S * i);
    }
    team_fwd_pass2<LOGN>(x, Tf, lane, q, q2);
    if (MODE == 0) {
#pragma unroll
      for (int i = 0; i < C::E; ++i) x[i] = canon4(x[i], q, q2);
      team_p2_to_p1<LOGN>(x, buf, lane);
    } else {
      const u64* bb = buf;
      if (MODE == 2) {
        cp_async_wait_all();
        __syncwarp();
      } else {
        bb = bbuf;
      }
      const u64 qinv = lc[l].qinv;
#pragma unroll
      for (int i = 0; i < C::E; ++i) x[i] = mont_mul(x[i], bb[team_swz<LOGN>(C::E * lane + i)], q, qinv);
      __syncwarp();
      const TW* Ti = tw_inv + (size_t)l * C::N;
      team_inv_pass2<LOGN>(x, Ti, lane, q, q2);
      team_p2_to_p1<LOGN>(x, buf, lane);
      team_inv_pass1<LOGN>(x, Ti, lc[l].ninvR, lc[l].ninvR_w1, q, q2);
#pragma unroll
      for (int i = 0; i < C::E; ++i) x[i] = canon2(x[i], q);
    }
  }
  if (active) {
    u64* dst = out + u * C::N;
#pragma unroll
    for (int i = 0; i < C::E; ++i) dst[lane + C::S * i] = x[i];
  }
}

template <int LOGN, int MODE>
inline size_t team_smem_bytes() {
  return (size_t)kTeamWarps * TeamCfg<LOGN>::TEAMS * TeamCfg<LOGN>::N * 8 * (MODE == 3 ? 2 : 1);
}

}  // namespace rnt
