// ntt_cluster.cuh -- single-launch NTT / INTT / fused polymul of ONE limb of one
// polynomial for N = 2^11 .. 2^16 on a thread-block cluster (SURVEY 8(f) f3:
// "one polynomial ... single launch (cluster/DSMEM for 2^16)"; the paper's
// single-kernel OSSP design, re-done with distributed shared
// memory instead of its global synchronisation).
//
// The limb is the 2^{n1} x 2^{n2} matrix of ntt_large.cuh.  A cluster of C CTAs
// owns it entirely on chip:
//   phase 1 (columns)  CTA k holds columns [k Cn/C, (k+1) Cn/C): the column
//                      stages of k_col_fwd on a tile in its own shared memory;
//   exchange X1        every thread stores its column segment straight into
//                      the receive rows of the owning CTA (st to DSMEM);
//   phase 2 (rows)     CTA k holds rows [k R/C, (k+1) R/C): the row stages of
//                      k_row (forward, fused (.) b_hat + inverse, or inverse);
//   exchange X2        row segments back to the owners of the columns;
//   phase 3 (columns)  inverse column stages of k_col_inv (N^-1 scaling).
// MODE 0 forward = P1 X1 P2; MODE 1 inverse = P2 X2 P3; MODE 2 polymul = all.
// Global memory sees only the input, b_hat and the output (24 B per element
// for the polymul) -- no intermediate round trip, one launch.
#pragma once
#include <cooperative_groups.h>

#include "modarith.cuh"
#include "ntt_large.cuh"
#include "ntt_small.cuh"

namespace rnt {

template <int LOGN, int C>
struct ClusterGeo {
  using P = TwoPass<LOGN>;
  static constexpr int CTc = P::Cn / C;   // columns per CTA (phases 1 and 3)
  static constexpr int RPCc = P::R / C;   // rows per CTA (phase 2)
  static constexpr int THREADS = CTc * P::T1;
  static_assert(CTc >= 1 && RPCc >= 1, "cluster larger than the matrix");
  static_assert(THREADS == RPCc * P::T2, "phase thread counts differ");
  static constexpr int TILE = P::R * CTc;             // phase-1/3 tile (words)
  static constexpr int RECV = RPCc * P::ROWBUF;       // phase-2 rows (words), also the row transposes
  static constexpr size_t SMEM = (size_t)(TILE + RECV) * 8;
};

__device__ __forceinline__ void cluster_arrive_relaxed() {
  asm volatile("barrier.cluster.arrive.relaxed.aligned;\n" ::: "memory");
}
__device__ __forceinline__ void cluster_wait() { asm volatile("barrier.cluster.wait.aligned;\n" ::: "memory"); }
__device__ __forceinline__ void cluster_sync_release_acquire() {
  asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;\n" ::: "memory");
}

// grid.x = units * C (cluster dims C x 1 x 1); unit u = blockIdx.x / C, limb u % L.
template <int LOGN, int C, int MODE>
__global__ void __launch_bounds__(ClusterGeo<LOGN, C>::THREADS)
k_cluster(u64* __restrict__ out, const u64* __restrict__ in, const u64* __restrict__ bop, int b_bcast,
          const TW* __restrict__ tw_col, const TW* __restrict__ tw_col_inv, const TW* __restrict__ tw_row_fwd,
          const LimbC* __restrict__ lc, uint32_t L) {
  using P = TwoPass<LOGN>;
  using G = ClusterGeo<LOGN, C>;
  constexpr int CTc = G::CTc, RPCc = G::RPCc;
  constexpr size_t N = (size_t)P::R * P::Cn;
  extern __shared__ __align__(16) u64 sm[];
  u64* tile = sm;               // [R][CTc]
  u64* recv = sm + G::TILE;     // [RPCc][ROWBUF]
  namespace cg = cooperative_groups;
  cg::cluster_group cluster = cg::this_cluster();
  const int k = (int)cluster.block_rank();
  const uint64_t u = blockIdx.x / C;
  const uint32_t l = (uint32_t)(u % L);
  const u64 q = lc[l].q, q2 = lc[l].q2;
  const size_t ubase = u * N;
  const int tid = threadIdx.x;
  cluster_arrive_relaxed();     // every CTA has started before anyone writes into it (wait below)
  u64 x[kEl];

  if constexpr (MODE != 1) {
    // ---------------- phase 1: forward column stages on columns [k CTc, (k+1) CTc)
    const int c = tid % CTc, r0 = tid / CTc;
    const TW* T = tw_col + (size_t)l * P::R;
    const size_t gcol = ubase + (size_t)k * CTc + c;
#pragma unroll
    for (int i = 0; i < kEl; ++i) x[i] = __ldg(in + gcol + (size_t)(r0 + P::T1 * i) * P::Cn);
    sfor<0, 4>([&](auto S_) {
      constexpr int s = decltype(S_)::value;
      constexpr int half = kEl >> (s + 1);
#pragma unroll
      for (int blk = 0; blk < (1 << s); ++blk) {
        TW w = ldg_tw(T + (1 << s) + blk);
#pragma unroll
        for (int kk = 0; kk < half; ++kk) ct_bfly(x[blk * 2 * half + kk], x[blk * 2 * half + kk + half], w, q, q2);
      }
    });
#pragma unroll
    for (int i = 0; i < kEl; ++i) tile[(r0 + P::T1 * i) * CTc + c] = x[i];
    __syncthreads();
    const int r1 = r0;
#pragma unroll
    for (int i = 0; i < kEl; ++i) x[i] = tile[(kEl * r1 + i) * CTc + c];
    sfor<4, P::n1>([&](auto S_) {
      constexpr int s = decltype(S_)::value;
      constexpr int t = P::R >> (s + 1);
#pragma unroll
      for (int m = 0; m < kEl / (2 * t); ++m) {
        TW w = ldg_tw(T + (1 << s) + ((kEl * r1 + m * 2 * t) >> (P::n1 - s)));
#pragma unroll
        for (int kk = 0; kk < t; ++kk) ct_bfly(x[m * 2 * t + kk], x[m * 2 * t + kk + t], w, q, q2);
      }
    });
    // ---------------- X1: rows 16 r1 + i of column k CTc + c -> receive rows of their owners
    cluster_wait();
#pragma unroll
    for (int i = 0; i < kEl; ++i) {
      const int row = kEl * r1 + i;
      u64* dst = cluster.map_shared_rank(recv, row / RPCc);
      dst[(row % RPCc) * P::ROWBUF + k * CTc + c] = x[i];
    }
    cluster_sync_release_acquire();
  }

  // ---------------- phase 2: row stages on rows [k RPCc, (k+1) RPCc)
  {
    const int c0 = tid % P::T2, rr = tid / P::T2;
    const int r = k * RPCc + rr;
    u64* rb = recv + rr * P::ROWBUF;
    const TW* Tm = tw_row_fwd + ((size_t)l * P::R + (P::R - 1 - r)) * P::Cn;   // mirrored row (inverse)
    if constexpr (MODE == 1) {
#pragma unroll
      for (int i = 0; i < kEl; ++i) x[i] = __ldg(in + ubase + (size_t)r * P::Cn + c0 + P::T2 * i);
      row_A_to_B<LOGN>(x, rb, c0);
      row_inv_B<LOGN>(x, Tm, c0, q, q2);
      row_B_to_A<LOGN>(x, rb, c0);
      row_inv_A<LOGN>(x, Tm, q, q2);
    } else {
#pragma unroll
      for (int i = 0; i < kEl; ++i) x[i] = rb[c0 + P::T2 * i];
      __syncwarp();
      const TW* Tf = tw_row_fwd + ((size_t)l * P::R + r) * P::Cn;
      row_fwd_A<LOGN>(x, Tf, q, q2);
      row_A_to_B<LOGN>(x, rb, c0);
      if constexpr (MODE == 2) {
        const u64* bsrc = bop + (b_bcast ? (size_t)l * N : ubase) + (size_t)r * P::Cn;
#pragma unroll
        for (int i = 0; i < kEl; ++i) cp_async8(rb + row_swz<LOGN>(c0 + P::T2 * i), bsrc + c0 + P::T2 * i);
      }
      row_fwd_B<LOGN>(x, Tf, c0, q, q2);
      if constexpr (MODE == 0) {
#pragma unroll
        for (int i = 0; i < kEl; ++i) x[i] = canon4(x[i], q, q2);
        row_B_to_A<LOGN>(x, rb, c0);
#pragma unroll
        for (int i = 0; i < kEl; ++i) out[ubase + (size_t)r * P::Cn + c0 + P::T2 * i] = x[i];
        // forward done: no DSMEM access after the X1 barrier
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
    // ---------------- X2: row r, columns c0 + T2 i -> tiles of the column owners
    if constexpr (MODE != 0) {
      if constexpr (MODE == 1) cluster_wait();
#pragma unroll
      for (int i = 0; i < kEl; ++i) {
        const int col = c0 + P::T2 * i;
        u64* dst = cluster.map_shared_rank(tile, col / CTc);
        dst[r * CTc + (col % CTc)] = x[i];
      }
      cluster_sync_release_acquire();
    }
  }
  if constexpr (MODE == 0) return;

  // ---------------- phase 3: inverse column stages (+ N^-1, or N^-1 2^64 after the Montgomery (.))
  {
    const int c = tid % CTc, r1 = tid / CTc;
    const TW* T = tw_col_inv + (size_t)l * P::R;
#pragma unroll
    for (int i = 0; i < kEl; ++i) x[i] = tile[(kEl * r1 + i) * CTc + c];
    sfor<0, P::n1 - 4>([&](auto I_) {
      constexpr int s = P::n1 - 1 - decltype(I_)::value;
      constexpr int t = P::R >> (s + 1);
#pragma unroll
      for (int m = 0; m < kEl / (2 * t); ++m) {
        TW w = ldg_tw(T + (1 << s) + ((kEl * r1 + m * 2 * t) >> (P::n1 - s)));
#pragma unroll
        for (int kk = 0; kk < t; ++kk) gs_bfly(x[m * 2 * t + kk], x[m * 2 * t + kk + t], w, q, q2);
      }
    });
#pragma unroll
    for (int i = 0; i < kEl; ++i) tile[(kEl * r1 + i) * CTc + c] = x[i];   // the thread's own read positions
    __syncthreads();
    const int r0 = r1;
#pragma unroll
    for (int i = 0; i < kEl; ++i) x[i] = tile[(r0 + P::T1 * i) * CTc + c];
    sfor<0, 3>([&](auto I_) {
      constexpr int s = 3 - decltype(I_)::value;
      constexpr int half = kEl >> (s + 1);
#pragma unroll
      for (int blk = 0; blk < (1 << s); ++blk) {
        TW w = ldg_tw(T + (1 << s) + blk);
#pragma unroll
        for (int kk = 0; kk < half; ++kk) gs_bfly(x[blk * 2 * half + kk], x[blk * 2 * half + kk + half], w, q, q2);
      }
    });
    const TW s0 = MODE == 2 ? lc[l].ninvR : lc[l].ninv;
    const TW s1 = MODE == 2 ? lc[l].ninvR_w1 : lc[l].ninv_w1;
#pragma unroll
    for (int kk = 0; kk < kEl / 2; ++kk) gs_bfly_last(x[kk], x[kk + kEl / 2], s0, s1, q, q2);
    const size_t gcol = ubase + (size_t)k * CTc + c;
#pragma unroll
    for (int i = 0; i < kEl; ++i) out[gcol + (size_t)(r0 + P::T1 * i) * P::Cn] = canon2(x[i], q);
  }
}

}  // namespace rnt
