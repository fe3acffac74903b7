// ntt_large.cuh -- two-pass negacyclic NTT / INTT / fused polymul for
// N = 2^11 .. 2^16 (the CKKS polynomial size), batched over
// (polynomial, limb) units (RNS limbs).
//
// View a limb as a 2^{n1} x 2^{n2} row-major matrix M[r][c] = a[r 2^{n2} + c]
// (n1 = ceil(n/2) column stages, n2 = floor(n/2) row stages; 256 x 256 at 2^16).
// CT stage s pairs j with j + N/2^{s+1} and uses twiddle w[2^s + (j >> (n-s))]:
//   * stages 0 .. n1-1 only mix elements of one column c and their twiddle
//     depends only on the row r        -> pass 1 ("columns"),
//   * stages n1 .. n-1 only mix elements of one row r      -> pass 2 ("rows").
// This is the B200 analogue of the paper's coefficient shuffling + switching
// point (prior art): exactly one global exchange (the kernel
// boundary; the 22.5 MiB cfg3 intermediate stays L2-resident, 126 MB L2),
// and every other exchange is a shared-memory transpose inside one CTA
// (pass 1: one __syncthreads) or one half-warp (pass 2: __syncwarp only).
//
// Inside a pass every thread holds E = 16 coefficients in registers:
//   sub-pass A: the 4 stages with distance >= 16 threads (stride layout),
//   sub-pass B: the remaining <= 4 stages (16 contiguous coefficients).
// Global loads/stores are always in the stride layout, i.e. coalesced
// 16 x 8 B = 128 B per half-warp row segment.
#pragma once
#include "modarith.cuh"
#include "ntt_small.cuh"   // cp_async8

namespace rnt {

// Programmatic dependent launch between the kernels of one N >= 2^11 chain (column ->
// row -> column pass, api.cu launch_pdl): the dependent is launched with the programmatic
// serialization attribute, so its launch overlaps the primary's last CTAs (the implicit
// trigger at CTA exit), and it waits for the primary's completion and memory before its
// first read of the primary's output (pdl_wait; a no-op for a launch without the
// attribute).  Measured (profiles/r02/pdl): cfg3 90.8 -> 89.4 us, cfg5 336.6 -> 334.4 us,
// cfg4 745.9 -> 740.8 us, a 23-limb 2^16 polymul (the 8-GPU shard) 65.5 -> 60.0 us.  An
// explicit trigger at kernel entry (RNT_PDL_EARLY=1: dependents resident early, waiting)
// was slower for the two-window chains (cfg3 99-100 us): waiting CTAs hold slots the other
// window needs.
#ifndef RNT_PDL
#define RNT_PDL 1
#endif
#ifndef RNT_PDL_EARLY
#define RNT_PDL_EARLY 0
#endif
__device__ __forceinline__ void pdl_trigger() {
#if RNT_PDL && RNT_PDL_EARLY
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
#endif
}
__device__ __forceinline__ void pdl_wait() {
#if RNT_PDL
  asm volatile("griddepcontrol.wait;" ::: "memory");
#endif
}

constexpr int kEl = 16;       // coefficients per thread
constexpr int kColTile = 16;  // columns per pass-1 CTA (one 128-byte line per row)

template <int LOGN>
struct TwoPass {
  static constexpr int n = LOGN;
  static constexpr int n1 = (LOGN + 1) / 2;   // column stages
  static constexpr int n2 = LOGN / 2;         // row stages
  static constexpr int R = 1 << n1;           // rows
  static constexpr int Cn = 1 << n2;          // columns (row length)
  static constexpr int T1 = R / kEl;          // threads per column
  static constexpr int T2 = Cn / kEl;         // threads per row
  static constexpr int P1_THREADS = kColTile * T1;
  static constexpr int RPC = (256 / T2) < R ? (256 / T2) : R;  // rows per pass-2 CTA
  static constexpr int P2_THREADS = RPC * T2;                   // <= 256
  static constexpr int ROWBUF = Cn + T2;      // padded row buffer (elements)
  static_assert(n1 >= 4 && n1 <= 8 && n2 >= 5 && n2 <= 8, "two-pass covers 2^10..2^16");
};

// Swizzle inside a row buffer: conflict-free for c = c0 + T2*i and c = 16*c1 + i'.
template <int LOGN>
__device__ __forceinline__ int row_swz(int c) {
  return c ^ ((c >> 4) & (TwoPass<LOGN>::T2 - 1));
}

// ============================== pass 1 (columns) ==============================
// (RNT_COL_MINB: experiment knob for the column kernels' min-blocks, like RNT_ROW_MINB.)
#ifdef RNT_COL_MINB
#define RNT_COL_BOUNDS(t) __launch_bounds__(t, RNT_COL_MINB)
#else
#define RNT_COL_BOUNDS(t) __launch_bounds__(t)
#endif
// Forward: CT stages 0..n1-1 on columns [cb*16, cb*16+16) of unit u.
// MODE 0: plain forward (in -> out).
// MODUP (key switching, keyswitch.cuh): unit (poly j, limb t) reads limb j of a
// single L-limb polynomial (one-prime digits, reading KS2 with alpha = 1) and
// lifts it to q_t on load: x mod q_t = x - q_t if x >= q_t (requires q_j < 2 q_t).
// LZ: lazy CT ranges (modarith.cuh ct_bfly_lz, plan flag lazy60); the output
// then carries the LZ bound of stage n1 and must feed an LZ row pass.
// CG = true: data loads bypass L1 (ld.global.cg), for callers that read data another
// CTA of the same launch wrote (a round-2 single-launch dataflow experiment, see
// DESIGN.md KB2); the stand-alone kernels use plain loads.
template <bool CG>
__device__ __forceinline__ u64 ld_data(const u64* p) {
  if constexpr (CG) return __ldcg(p);
  else return *p;
}

// One pass-1 tile: columns [bx CT, bx CT + CT) of unit y (y = limb * B + poly,
// limb-major CTA order); `tile` is R * CT words of shared memory.
template <int LOGN, int CT, bool MODUP, bool LZ, bool CG = false>
__device__ __forceinline__ void col_fwd_tile(u64* __restrict__ out, const u64* __restrict__ in,
                                             const TW* __restrict__ tw_col, const LimbC* __restrict__ lc, uint32_t L,
                                             uint32_t B, uint64_t y, int bx, u64* tile) {
  using P = TwoPass<LOGN>;
  const int c = threadIdx.x % CT;
  const int r0 = threadIdx.x / CT;
  const uint32_t l = (uint32_t)(y / B);
  const uint64_t u = (y % B) * L + l;
  const u64 q = lc[l].q, q2 = lc[l].q2;
  const TW* T = tw_col + (size_t)l * P::R;
  const size_t base = u * (size_t)(P::R * P::Cn) + (size_t)bx * CT + c;
  u64 x[kEl];
  if constexpr (MODUP) {
    const size_t ibase = (y % B) * (size_t)(P::R * P::Cn) + (size_t)bx * CT + c;
#pragma unroll
    for (int i = 0; i < kEl; ++i) x[i] = csub(__ldg(in + ibase + (size_t)(r0 + P::T1 * i) * P::Cn), q);
  } else {
#pragma unroll
    for (int i = 0; i < kEl; ++i) x[i] = ld_data<CG>(in + base + (size_t)(r0 + P::T1 * i) * P::Cn);
  }
  // sub-pass A: stages 0..3, twiddle w[2^s + (i >> (4-s))] (uniform)
  sfor<0, 4>([&](auto S_) {
    constexpr int s = decltype(S_)::value;
    constexpr int half = kEl >> (s + 1);
#pragma unroll
    for (int blk = 0; blk < (1 << s); ++blk) {
      TW w = ldg_tw(T + (1 << s) + blk);
#pragma unroll
      for (int k = 0; k < half; ++k)
        ct_bfly_at<LZ, s>(x[blk * 2 * half + k], x[blk * 2 * half + k + half], w, q, q2);
    }
  });
#pragma unroll
  for (int i = 0; i < kEl; ++i) tile[(r0 + P::T1 * i) * CT + c] = x[i];
  __syncthreads();
  const int r1 = r0;
#pragma unroll
  for (int i = 0; i < kEl; ++i) x[i] = tile[(kEl * r1 + i) * CT + c];
  // sub-pass B: stages 4..n1-1 on rows 16 r1 + i; twiddle w[2^s + ((16 r1 + i) >> (n1 - s))]
  sfor<4, P::n1>([&](auto S_) {
    constexpr int s = decltype(S_)::value;
    constexpr int t = P::R >> (s + 1);
#pragma unroll
    for (int m = 0; m < kEl / (2 * t); ++m) {
      TW w = ldg_tw(T + (1 << s) + ((kEl * r1 + m * 2 * t) >> (P::n1 - s)));
#pragma unroll
      for (int k = 0; k < t; ++k) ct_bfly_at<LZ, s>(x[m * 2 * t + k], x[m * 2 * t + k + t], w, q, q2);
    }
  });
#pragma unroll
  for (int i = 0; i < kEl; ++i) out[base + (size_t)(kEl * r1 + i) * P::Cn] = x[i];
}

template <int LOGN, int CT = kColTile, bool MODUP = false, bool LZ = false>
__global__ void RNT_COL_BOUNDS(CT * TwoPass<LOGN>::T1)
k_col_fwd(u64* __restrict__ out, const u64* __restrict__ in, const TW* __restrict__ tw_col,
          const LimbC* __restrict__ lc, uint32_t L, uint32_t B, uint64_t y0) {
  __shared__ __align__(16) u64 tile[TwoPass<LOGN>::R * CT];
  if constexpr (!MODUP) pdl_trigger();
  col_fwd_tile<LOGN, CT, MODUP, LZ>(out, in, tw_col, lc, L, B, y0 + blockIdx.y, (int)blockIdx.x, tile);
}

// Inverse: GS stages n1-1..0 (+ N^{-1} or N^{-1} R scaling), canonical output.
template <int LOGN, int CT, bool CG = false>
__device__ __forceinline__ void col_inv_tile(u64* __restrict__ out, const u64* __restrict__ in,
                                             const TW* __restrict__ tw_col, const LimbC* __restrict__ lc, uint32_t L,
                                             uint32_t B, uint64_t y, int bx, int after_mont, u64* tile) {
  using P = TwoPass<LOGN>;
  const int c = threadIdx.x % CT;
  const int r1 = threadIdx.x / CT;
  const uint32_t l = (uint32_t)(y / B);
  const uint64_t u = (y % B) * L + l;
  const u64 q = lc[l].q, q2 = lc[l].q2;
  const TW* T = tw_col + (size_t)l * P::R;
  const size_t base = u * (size_t)(P::R * P::Cn) + (size_t)bx * CT + c;
  u64 x[kEl];
#pragma unroll
  for (int i = 0; i < kEl; ++i) x[i] = ld_data<CG>(in + base + (size_t)(kEl * r1 + i) * P::Cn);
  sfor<0, P::n1 - 4>([&](auto I_) {
    constexpr int s = P::n1 - 1 - decltype(I_)::value;
    constexpr int t = P::R >> (s + 1);
#pragma unroll
    for (int m = 0; m < kEl / (2 * t); ++m) {
      TW w = ldg_tw(T + (1 << s) + ((kEl * r1 + m * 2 * t) >> (P::n1 - s)));
#pragma unroll
      for (int k = 0; k < t; ++k) gs_bfly(x[m * 2 * t + k], x[m * 2 * t + k + t], w, q, q2);
    }
  });
#pragma unroll
  for (int i = 0; i < kEl; ++i) tile[(kEl * r1 + i) * CT + c] = x[i];
  __syncthreads();
  const int r0 = r1;
#pragma unroll
  for (int i = 0; i < kEl; ++i) x[i] = tile[(r0 + P::T1 * i) * CT + c];
  sfor<0, 3>([&](auto I_) {
    constexpr int s = 3 - decltype(I_)::value;
    constexpr int half = kEl >> (s + 1);
#pragma unroll
    for (int blk = 0; blk < (1 << s); ++blk) {
      TW w = ldg_tw(T + (1 << s) + blk);
#pragma unroll
      for (int k = 0; k < half; ++k) gs_bfly(x[blk * 2 * half + k], x[blk * 2 * half + k + half], w, q, q2);
    }
  });
  const TW s0 = after_mont ? lc[l].ninvR : lc[l].ninv;
  const TW s1 = after_mont ? lc[l].ninvR_w1 : lc[l].ninv_w1;
#pragma unroll
  for (int k = 0; k < kEl / 2; ++k) gs_bfly_last(x[k], x[k + kEl / 2], s0, s1, q, q2);
#pragma unroll
  for (int i = 0; i < kEl; ++i) out[base + (size_t)(r0 + P::T1 * i) * P::Cn] = canon2(x[i], q);
}

template <int LOGN, int CT = kColTile>
__global__ void RNT_COL_BOUNDS(CT * TwoPass<LOGN>::T1)
k_col_inv(u64* __restrict__ out, const u64* __restrict__ in, const TW* __restrict__ tw_col,
          const LimbC* __restrict__ lc, uint32_t L, uint32_t B, uint64_t y0, int after_mont) {
  __shared__ __align__(16) u64 tile[TwoPass<LOGN>::R * CT];
  pdl_wait();
  col_inv_tile<LOGN, CT>(out, in, tw_col, lc, L, B, y0 + blockIdx.y, (int)blockIdx.x, after_mont, tile);
}

// ============================== pass 2 (rows) =================================
// Row twiddle table (forward only; per limb, per row r, 2^{n2} entries): stage v (global
// stage n1 + v) occupies [2^v - 1, 2^{v+1} - 1); for v < 4 entry k holds
// w[2^{n1+v} + r 2^v + k]; for v >= 4 entry m*T2 + c1 holds
// w[2^{n1+v} + r 2^v + c1 2^{v+4-n2} + m] (lane-major: coalesced loads).

template <int LOGN, bool LZ = false>
__device__ __forceinline__ void row_fwd_A(u64 (&x)[kEl], const TW* Tr, u64 q, u64 q2) {
  sfor<0, 4>([&](auto V_) {
    constexpr int v = decltype(V_)::value;
    constexpr int half = kEl >> (v + 1);
#pragma unroll
    for (int blk = 0; blk < (1 << v); ++blk) {
      TW w = ldg_tw(Tr + (1 << v) - 1 + blk);
#pragma unroll
      for (int k = 0; k < half; ++k)
        ct_bfly_at<LZ, TwoPass<LOGN>::n1 + v>(x[blk * 2 * half + k], x[blk * 2 * half + k + half], w, q, q2);
    }
  });
}

template <int LOGN, bool LZ = false>
__device__ __forceinline__ void row_fwd_B(u64 (&x)[kEl], const TW* Tr, int c1, u64 q, u64 q2) {
  using P = TwoPass<LOGN>;
  sfor<4, P::n2>([&](auto V_) {
    constexpr int v = decltype(V_)::value;
    constexpr int t = P::Cn >> (v + 1);
#pragma unroll
    for (int m = 0; m < kEl / (2 * t); ++m) {
      TW w = ldg_tw(Tr + (1 << v) - 1 + m * P::T2 + c1);
#pragma unroll
      for (int k = 0; k < t; ++k) ct_bfly_at<LZ, P::n1 + v>(x[m * 2 * t + k], x[m * 2 * t + k + t], w, q, q2);
    }
  });
}

// Inverse row stages read the FORWARD row table of the mirrored row R-1-r,
// block-reversed (psi^{-brv(k)} = -psi^{brv(3 2^s - 1 - k)}), with the
// negated-twiddle GS butterfly: no inverse row table exists.
template <int LOGN>
__device__ __forceinline__ void row_inv_B(u64 (&x)[kEl], const TW* Tm, int c1, u64 q, u64 q2) {
  using P = TwoPass<LOGN>;
  sfor<0, P::n2 - 4>([&](auto I_) {
    constexpr int v = P::n2 - 1 - decltype(I_)::value;
    constexpr int t = P::Cn >> (v + 1);
    constexpr int per = kEl / (2 * t);
#pragma unroll
    for (int m = 0; m < per; ++m) {
      TW w = ldg_tw(Tm + (1 << v) - 1 + (per - 1 - m) * P::T2 + (P::T2 - 1 - c1));
#pragma unroll
      for (int k = 0; k < t; ++k) gs_bfly_neg(x[m * 2 * t + k], x[m * 2 * t + k + t], w, q, q2);
    }
  });
}

template <int LOGN>
__device__ __forceinline__ void row_inv_A(u64 (&x)[kEl], const TW* Tm, u64 q, u64 q2) {
  sfor<0, 4>([&](auto I_) {
    constexpr int v = 3 - decltype(I_)::value;
    constexpr int half = kEl >> (v + 1);
#pragma unroll
    for (int blk = 0; blk < (1 << v); ++blk) {
      TW w = ldg_tw(Tm + (1 << v) - 1 + ((1 << v) - 1 - blk));
#pragma unroll
      for (int k = 0; k < half; ++k) gs_bfly_neg(x[blk * 2 * half + k], x[blk * 2 * half + k + half], w, q, q2);
    }
  });
}

// stride layout (c = c0 + T2 i) -> contiguous layout (c = 16 c1 + i)
template <int LOGN>
__device__ __forceinline__ void row_A_to_B(u64 (&x)[kEl], u64* rb, int c0) {
  using P = TwoPass<LOGN>;
#pragma unroll
  for (int i = 0; i < kEl; ++i) rb[row_swz<LOGN>(c0 + P::T2 * i)] = x[i];
  __syncwarp();
#pragma unroll
  for (int i = 0; i < kEl; ++i) x[i] = rb[row_swz<LOGN>(kEl * c0 + i)];
  __syncwarp();
}

template <int LOGN>
__device__ __forceinline__ void row_B_to_A(u64 (&x)[kEl], u64* rb, int c0) {
  using P = TwoPass<LOGN>;
#pragma unroll
  for (int i = 0; i < kEl; ++i) rb[row_swz<LOGN>(kEl * c0 + i)] = x[i];
  __syncwarp();
#pragma unroll
  for (int i = 0; i < kEl; ++i) x[i] = rb[row_swz<LOGN>(c0 + P::T2 * i)];
  __syncwarp();
}

// MODE 0: forward rows (CT stages n1..n-1, canonical output)
// MODE 1: inverse rows (GS stages n-1..n1, lazy [0,2q) output for k_col_inv)
// MODE 2: fused forward rows -> (.) b_hat (Montgomery) -> inverse rows
// (RNT_ROW_MINB: experiment knob; an explicit min-blocks of 1 measured 18 % slower
// than leaving it unspecified, 3 about equal.)
#ifdef RNT_ROW_MINB
#define RNT_ROW_BOUNDS(t) __launch_bounds__(t, RNT_ROW_MINB)
#else
#define RNT_ROW_BOUNDS(t) __launch_bounds__(t)
#endif
// One pass-2 tile: RPC_ rows (block rx) of unit y; `sbuf` is RPC_ ROWBUF words.
template <int LOGN, int MODE, int RPC_, bool LZ, bool CG = false>
__device__ __forceinline__ void row_tile(u64* __restrict__ out, const u64* __restrict__ in, const u64* __restrict__ bop,
                                         int b_bcast, const TW* __restrict__ tw_row_fwd, const LimbC* __restrict__ lc,
                                         uint32_t L, uint32_t B, uint64_t y, int rx, u64* sbuf) {
  using P = TwoPass<LOGN>;
  const int c0 = threadIdx.x % P::T2;
  const int rr = threadIdx.x / P::T2;
  // With 16 threads per row a warp holds two rows: make them r and R-1-r, so
  // the inverse stages of each row read (from L1) the forward twiddles its
  // partner half-warp just loaded.
  int r;
  if constexpr (P::T2 == 16 && RPC_ % 2 == 0) {
    const int pi = rx * (RPC_ / 2) + (rr >> 1);
    r = (rr & 1) ? (P::R - 1 - pi) : pi;
  } else {
    r = rx * RPC_ + rr;
  }
  const uint32_t l = (uint32_t)(y / B);
  const uint64_t u = (y % B) * L + l;
  const u64 q = lc[l].q, q2 = lc[l].q2;
  u64* rb = sbuf + rr * P::ROWBUF;
  const size_t rowoff = u * (size_t)(P::R * P::Cn) + (size_t)r * P::Cn;
  const size_t troff = ((size_t)l * P::R + r) * P::Cn;
  const TW* Tm = tw_row_fwd + ((size_t)l * P::R + (P::R - 1 - r)) * P::Cn;   // mirrored row
  u64 x[kEl];
#pragma unroll
  for (int i = 0; i < kEl; ++i) x[i] = ld_data<CG>(in + rowoff + c0 + P::T2 * i);
  if (MODE == 1) {
    row_A_to_B<LOGN>(x, rb, c0);
    row_inv_B<LOGN>(x, Tm, c0, q, q2);
    row_B_to_A<LOGN>(x, rb, c0);
    row_inv_A<LOGN>(x, Tm, q, q2);
  } else {
    const TW* Tf = tw_row_fwd + troff;
    row_fwd_A<LOGN, LZ>(x, Tf, q, q2);
    row_A_to_B<LOGN>(x, rb, c0);
    if (MODE == 2) {
      const u64* bsrc = bop + (b_bcast ? (size_t)l * P::R * P::Cn : u * (size_t)(P::R * P::Cn)) + (size_t)r * P::Cn;
#pragma unroll
      for (int i = 0; i < kEl; ++i) cp_async8(rb + row_swz<LOGN>(c0 + P::T2 * i), bsrc + c0 + P::T2 * i);
    }
    row_fwd_B<LOGN, LZ>(x, Tf, c0, q, q2);
    if (MODE == 0) {
#pragma unroll
      for (int i = 0; i < kEl; ++i) x[i] = canon_fwd<LZ>(x[i], q, q2);
      row_B_to_A<LOGN>(x, rb, c0);
    } else {
      cp_async_wait_all();
      __syncwarp();
      const u64 qinv = lc[l].qinv;
#pragma unroll
      for (int i = 0; i < kEl; ++i) x[i] = mont_mul(x[i], rb[row_swz<LOGN>(kEl * c0 + i)], q, qinv);
      __syncwarp();
      row_inv_B<LOGN>(x, Tm, c0, q, q2);
      row_B_to_A<LOGN>(x, rb, c0);
      row_inv_A<LOGN>(x, Tm, q, q2);
    }
  }
#pragma unroll
  for (int i = 0; i < kEl; ++i) out[rowoff + c0 + P::T2 * i] = x[i];
}

template <int LOGN, int MODE, int RPC_ = TwoPass<LOGN>::RPC, bool LZ = false>
__global__ void RNT_ROW_BOUNDS(RPC_ * TwoPass<LOGN>::T2)
k_row(u64* __restrict__ out, const u64* __restrict__ in, const u64* __restrict__ bop, int b_bcast,
      const TW* __restrict__ tw_row_fwd, const LimbC* __restrict__ lc, uint32_t L, uint32_t B, uint64_t y0) {
  __shared__ __align__(16) u64 sbuf[RPC_ * TwoPass<LOGN>::ROWBUF];
  pdl_trigger();
  pdl_wait();
  row_tile<LOGN, MODE, RPC_, LZ>(out, in, bop, b_bcast, tw_row_fwd, lc, L, B, y0 + blockIdx.y, (int)blockIdx.x, sbuf);
}

// ============================ pass 2 + key product ============================

// Key switching (keyswitch.cuh, rnt_keyswitch_apply): for the RPC rows r of
// limb t, run the forward row stages of every digit's extended polynomial
// (E: [dnum][LK][N], column pass done) and accumulate the products with the
// key rows in shared memory, u_k[t] = sum_j NTT(e_j)[t] (.) evk[j][k][t]:
// the NTT-form extended polynomials never go back to HBM.  Montgomery
// products, accumulators kept in [0, 2q); u written canonical.
// (min-blocks 2: the LZ variant compiled to 130 registers, one CTA per SM)
// (RNT_ROWMAC_MINB, RNT_ROWMAC_PREFETCH: experiment builds; PREFETCH loads digit
// j + 1's rows of E into registers while digit j's row stages run.)
#ifndef RNT_ROWMAC_MINB
#define RNT_ROWMAC_MINB 2
#endif
#ifndef RNT_ROWMAC_PREFETCH
#define RNT_ROWMAC_PREFETCH 0
#endif
template <int LOGN, int RPC_, bool LZ = false>
__global__ void __launch_bounds__(RPC_ * TwoPass<LOGN>::T2, RNT_ROWMAC_MINB)
k_row_mac(u64* __restrict__ uo, const u64* __restrict__ E, const u64* __restrict__ evk,
          const TW* __restrict__ tw_row_fwd, const LimbC* __restrict__ lc, uint32_t LK, uint32_t dnum,
          uint32_t dsplit) {
  // blockIdx.z = s: digits [s dnum / dsplit, (s+1) dnum / dsplit) into partial sum s
  // (uo + s 2 LK N); dsplit > 1 evens out the last wave, k_ks_sum adds the parts.
  using P = TwoPass<LOGN>;
  constexpr size_t N = (size_t)P::R * P::Cn;
  __shared__ __align__(16) u64 sbuf[RPC_ * P::ROWBUF];
  extern __shared__ __align__(16) u64 acc[];   // [2][RPC_][Cn]
  const int c0 = threadIdx.x % P::T2;
  const int rr = threadIdx.x / P::T2;
  const int r = blockIdx.x * RPC_ + rr;
  const uint32_t t = blockIdx.y;
  const u64 q = lc[t].q, q2 = lc[t].q2, qinv = lc[t].qinv;
  u64* rb = sbuf + rr * P::ROWBUF;
  u64* a0 = acc + (size_t)rr * P::Cn + c0;
  u64* a1 = acc + (size_t)(RPC_ + rr) * P::Cn + c0;
  const TW* Tf = tw_row_fwd + ((size_t)t * P::R + r) * P::Cn;
#pragma unroll
  for (int i = 0; i < kEl; ++i) a0[P::T2 * i] = a1[P::T2 * i] = 0;
  const size_t roff = (size_t)r * P::Cn + c0;
  const uint32_t jb = blockIdx.z * dnum / dsplit, je = (blockIdx.z + 1) * dnum / dsplit;
  uo += (size_t)blockIdx.z * 2 * LK * N;
#if RNT_ROWMAC_PREFETCH
  u64 nx[kEl];
  if (jb < je) {
    const u64* src = E + ((size_t)jb * LK + t) * N + roff;
#pragma unroll
    for (int i = 0; i < kEl; ++i) nx[i] = __ldcs(src + P::T2 * i);
  }
#endif
  for (uint32_t j = jb; j < je; ++j) {
    u64 x[kEl];
#if RNT_ROWMAC_PREFETCH
#pragma unroll
    for (int i = 0; i < kEl; ++i) x[i] = nx[i];
    if (j + 1 < je) {
      const u64* nsrc = E + ((size_t)(j + 1) * LK + t) * N + roff;
#pragma unroll
      for (int i = 0; i < kEl; ++i) nx[i] = __ldcs(nsrc + P::T2 * i);
    }
#else
    const u64* src = E + ((size_t)j * LK + t) * N + roff;
#pragma unroll
    for (int i = 0; i < kEl; ++i) x[i] = __ldcs(src + P::T2 * i);
#endif
    row_fwd_A<LOGN, LZ>(x, Tf, q, q2);
    row_A_to_B<LOGN>(x, rb, c0);
    row_fwd_B<LOGN, LZ>(x, Tf, c0, q, q2);
    row_B_to_A<LOGN>(x, rb, c0);
    const u64* k0 = evk + ((size_t)(2 * j) * LK + t) * N + roff;
    const u64* k1 = k0 + (size_t)LK * N;
#pragma unroll
    for (int i = 0; i < kEl; ++i) {
      const u64 b0 = __ldcs(k0 + P::T2 * i), b1 = __ldcs(k1 + P::T2 * i);
      a0[P::T2 * i] = csub(a0[P::T2 * i] + mont_mul(x[i], b0, q, qinv), q2);
      a1[P::T2 * i] = csub(a1[P::T2 * i] + mont_mul(x[i], b1, q, qinv), q2);
    }
  }
  const u64 r2 = lc[t].r2;
  u64* o0 = uo + (size_t)t * N + roff;
  u64* o1 = uo + ((size_t)LK + t) * N + roff;
#pragma unroll
  for (int i = 0; i < kEl; ++i) {
    o0[P::T2 * i] = canon2(mont_mul(a0[P::T2 * i], r2, q, qinv), q);
    o1[P::T2 * i] = canon2(mont_mul(a1[P::T2 * i], r2, q, qinv), q);
  }
}

// ============================ pass 2, warp engine =============================
// Rows through the warp engine of ntt_small.cuh: a warp owns 1024 / 2^{n2}
// consecutive rows of one limb in a padded shared buffer and runs the row
// stages as radix-8 passes (n2 = 8: 3 + 3 + 2).  Row r uses its own twiddle
// table T_r[2^s + i] = w[2^{n1+s} + r 2^s + i] (natural per-row layout,
// stride 2^{n2}); the inverse stages read the mirrored row R-1-r
// (MIRROR, negated-twiddle GS butterfly) and never apply N^{-1}.
// MODE 0: forward rows, 1: inverse rows, 2: forward rows -> (.) b_hat -> inverse rows.
constexpr int kRowWarps = 2;
constexpr int kRowKM = 3;

#ifndef RNT_ROWS_MINB
#define RNT_ROWS_MINB 12
#endif
template <int LOGN, int MODE, bool LZ = false, int TEAM = 1>
__global__ void __launch_bounds__(kRowWarps * 32, RNT_ROWS_MINB)
k_rows(u64* __restrict__ out, const u64* __restrict__ in, const u64* __restrict__ bop, int b_bcast,
       const TW* __restrict__ tw_rows, const LimbC* __restrict__ lc, uint32_t L, uint32_t B, uint64_t y0) {
  using P = TwoPass<LOGN>;
  constexpr int n2 = P::n2;
  constexpr int N2 = P::Cn;
  constexpr int RPW = kWarpElems / N2;   // rows per warp buffer
  static_assert(TEAM == 1 || TEAM == kRowWarps, "a team is one warp or the whole CTA");
  extern __shared__ __align__(16) u64 smem[];
  pdl_trigger();
  pdl_wait();
  const int team = (int)(threadIdx.x >> 5) / TEAM;
  const int lane = (int)threadIdx.x % (32 * TEAM);
  const uint64_t y = y0 + blockIdx.y;
  const uint32_t l = (uint32_t)(y / B);
  const uint64_t u = (y % B) * L + l;
  const int r0 = (blockIdx.x * (kRowWarps / TEAM) + team) * RPW;
  if (r0 >= P::R) return;
  u64* buf = smem + (size_t)team * kWarpBuf;
  const u64 q = lc[l].q, q2 = lc[l].q2;
  const size_t base = u * (size_t)(P::R * P::Cn);
  const GView src{in + base, (uint64_t)r0, (uint64_t)N2, (uint64_t)P::R};
  const GView dst{out + base, (uint64_t)r0, (uint64_t)N2, (uint64_t)P::R};
  const TW* Tr = tw_rows + (size_t)l * P::R * N2;
  const TW* Tf = Tr + (size_t)r0 * N2;                  // row r0 (+ p * N2)
  const TW* Tm = Tr + (size_t)(P::R - 1 - r0) * N2;     // mirrored row R-1-r0 (- p * N2)
  const TW none{0, 0};
  if constexpr (MODE == 0) {
    warp_forward<n2, kRowKM, kToGlobal, false, N2, LZ, P::n1, kFromGlobal, TEAM>(buf, src, dst, lane, Tf, q, q2);
  } else if constexpr (MODE == 1) {
    warp_inverse<n2, kRowKM, false, false, N2, true, false, kFromGlobal, TEAM>(buf, src, dst, lane, Tm, none, none, q,
                                                                              q2);
  } else {
    const size_t boff = b_bcast ? (size_t)l * P::R * P::Cn : base;
    const GView bview{bop + boff, (uint64_t)r0, (uint64_t)N2, (uint64_t)P::R};
    warp_polymul<n2, kRowKM, kFromGlobal, false, false, N2, true, LZ, P::n1, kFromGlobal, TEAM>(
        buf, src, dst, bview, nullptr, lane, Tf, Tm, none, none, q, q2, lc[l].qinv);
  }
}

}  // namespace rnt
