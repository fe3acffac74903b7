// ntt_clat.cuh -- latency-oriented single-launch NTT / INTT / fused polymul of
// ONE limb for N = 2^11 .. 2^16 on a thread-block cluster (the
// paper's single-polynomial latency).
//
// Same column/row decomposition and DSMEM exchanges as ntt_cluster.cuh
// (k_cluster), but built for latency instead of throughput: every thread holds
// only E (4 or 8) coefficients, so a 2^12 limb runs on 8 x 128 threads instead
// of 8 x 32, and the stages of a phase are radix-E passes through shared
// memory separated by CTA barriers.  With 16 coefficients per thread the
// k_cluster warps serialise 48 butterflies per stage group on one SMSP; here
// each thread runs E/2 independent butterflies per stage and all four SMSPs of
// every SM of the cluster issue.
//
//   phase A   CTA k owns columns [k CW, (k+1) CW) of the R x Cn matrix (all R
//             rows): CT stages 0 .. n1-1 (column-local, Eq. 1 loop);
//   X1        the last column pass stores its registers straight into the row
//             buffers of the owning CTAs (st to DSMEM), cluster barrier;
//   phase B   CTA k owns rows [k RC, (k+1) RC): CT stages n1 .. n-1; for the
//             polymul the last forward pass, (.) b_hat (Montgomery) and the
//             first GS pass run on the same registers; then GS stages n-1..n1;
//   X2        row registers -> column tiles of the owners, cluster barrier;
//   phase A'  GS stages n1-1 .. 0 with the N^-1 (N^-1 2^64) scale.
// MODE 0 forward = A X1 B; MODE 1 inverse = B' X2 A'; MODE 2 polymul = all.
#pragma once
#include <cooperative_groups.h>

#include "modarith.cuh"
#include "ntt_cluster.cuh"

namespace rnt {

template <int LOGN, int C, int E>
struct Clat {
  static constexpr int N = 1 << LOGN;
  static constexpr int n1 = (LOGN + 1) / 2, n2 = LOGN / 2;
  static constexpr int R = 1 << n1, Cn = 1 << n2;
  static constexpr int CW = Cn / C;   // columns per CTA (phase A)
  static constexpr int RC = R / C;    // rows per CTA (phase B)
  static constexpr int M = N / C;     // coefficients per CTA
  static constexpr int TH = M / E;    // threads per CTA
  static constexpr int KE = E == 4 ? 2 : (E == 8 ? 3 : 4);
  static constexpr int RPAD = Cn + Cn / 32;   // padded row (phase B buffer)
  static_assert(CW >= 1 && RC >= 1 && TH >= 32 && TH <= 1024, "cluster latency geometry");
  static constexpr int NP1 = (n1 + KE - 1) / KE;   // column passes
  static constexpr int NP2 = (n2 + KE - 1) / KE;   // row passes
  static constexpr size_t DATA = (size_t)(R * CW + RC * RPAD) * 8;
  // + twiddles staged at kernel start: column table(s) [R] and the CTA's row
  // table(s) [RC][Cn] (forward rows for MODE != 1, mirrored rows for MODE != 0)
  template <int MODE>
  static constexpr size_t smem() {
    return DATA + (size_t)((MODE != 1) + (MODE != 0)) * (R + RC * Cn) * sizeof(TW);
  }
};

__device__ __forceinline__ void cp_async16(void* smem, const void* gmem) {
  unsigned s = (unsigned)__cvta_generic_to_shared(smem);
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(s), "l"(gmem) : "memory");
}

// stages covered by pass p of an n-stage phase in radix-2^KE passes
__host__ __device__ constexpr int clat_k(int n, int KE, int p) { return n - p * KE < KE ? n - p * KE : KE; }

// Group g (of NG = E >> K per thread) of a pass over stages [S, S+K) of lines of
// length LEN: element u of the group is at position base + u LO of its line.
template <int LEN, int S, int K>
struct CGroup {
  static constexpr int LO = LEN >> (S + K);
  static constexpr int GPL = LEN >> K;   // groups per line
  int line, base;
  // COLMAJOR: consecutive groups walk the lines first (phase A: coalesced columns);
  // else they walk one line first (phase B: coalesced rows).
  template <int NLINES, bool COLMAJOR>
  __device__ __forceinline__ void at(int G) {
    int gr;
    if constexpr (COLMAJOR) { line = G % NLINES; gr = G / NLINES; }
    else { line = G / GPL; gr = G % GPL; }
    base = (gr / LO) * (LEN >> S) + gr % LO;
  }
  __device__ __forceinline__ int pos(int u) const { return base + u * LO; }
};

// CT stages [S, S+K) (global stage S0 + s) on x[g 2^K .. (g+1) 2^K) of a group;
// twiddle of the pair at position j of a line: TWF(s_global, j).
template <int S, int K, int S0, int LEN, typename TWF>
__device__ __forceinline__ void clat_ct(u64* x, const CGroup<LEN, S, K>& gg, TWF twf, u64 q, u64 q2) {
  sfor<0, K>([&](auto L_) {
    constexpr int l = decltype(L_)::value;
    constexpr int half = 1 << (K - 1 - l);
#pragma unroll
    for (int u = 0; u < (1 << K); ++u) {
      if (u & half) continue;
      const TW w = twf(S0 + S + l, gg.pos(u));
      ct_bfly(x[u], x[u + half], w, q, q2);
    }
  });
}

// GS stages S+K-1 .. S; LASTSCALE: global stage 0 carries N^-1 (s0, s1).
template <int S, int K, int S0, int LEN, bool LASTSCALE, bool NEG, typename TWF>
__device__ __forceinline__ void clat_gs(u64* x, const CGroup<LEN, S, K>& gg, TWF twf, TW s0, TW s1, u64 q, u64 q2) {
  sfor<0, K>([&](auto L_) {
    constexpr int l = K - 1 - decltype(L_)::value;
    constexpr int half = 1 << (K - 1 - l);
#pragma unroll
    for (int u = 0; u < (1 << K); ++u) {
      if (u & half) continue;
      if constexpr (LASTSCALE && S0 + S + l == 0) {
        gs_bfly_last(x[u], x[u + half], s0, s1, q, q2);
      } else {
        const TW w = twf(S0 + S + l, gg.pos(u));
        if constexpr (NEG) gs_bfly_neg(x[u], x[u + half], w, q, q2);
        else gs_bfly(x[u], x[u + half], w, q, q2);
      }
    }
  });
}

// Inside a phase every thread stores back exactly the positions it loaded, so a
// pass needs one CTA barrier (between its stores and the next pass's loads).
// grid.x = units * C (cluster C x 1 x 1); unit u = blockIdx.x / C, limb u % L.
// tw_col / tw_col_inv: natural entries psi^{+-brv(i)}, i < R, [L][R];
// tw_rows: natural per-row forward table [L][R][Cn] (plan_row_natural).
template <int LOGN, int C, int E, int MODE>
__global__ void __launch_bounds__(Clat<LOGN, C, E>::TH)
k_clat(u64* __restrict__ out, const u64* __restrict__ in, const u64* __restrict__ bop, int b_bcast,
       const TW* __restrict__ tw_col, const TW* __restrict__ tw_col_inv, const TW* __restrict__ tw_rows,
       const LimbC* __restrict__ lc, uint32_t L) {
  using G = Clat<LOGN, C, E>;
  constexpr int R = G::R, Cn = G::Cn, CW = G::CW, RC = G::RC, KE = G::KE, n1 = G::n1, n2 = G::n2;
  extern __shared__ __align__(16) u64 sm[];
  u64* tile = sm;                  // [R][CW]      phase A / A'
  u64* recv = sm + R * CW;         // [RC][RPAD]   phase B
  namespace cg = cooperative_groups;
  cg::cluster_group cluster = cg::this_cluster();
  const int k = (int)cluster.block_rank();
  const uint64_t unit = blockIdx.x / C;
  const uint32_t l = (uint32_t)(unit % L);
  const u64 q = lc[l].q, q2 = lc[l].q2;
  const size_t ubase = unit * (size_t)G::N;
  const int tid = threadIdx.x;
  cluster_arrive_relaxed();        // all CTAs resident before the first remote store (wait below)
  auto rpos = [](int j) { return j + (j >> 5); };
  u64 x[E];

  // Twiddles this CTA needs, staged into shared memory once with cp.async (one
  // memory round trip instead of one dependent L2 load per pass): the latency
  // path is bound by load latency, not by bandwidth.
  TW* tws = reinterpret_cast<TW*>(sm + G::DATA / 8);
  TW* sTc = tws;                                       // [R]      forward columns
  TW* sTr = sTc + (MODE != 1 ? R : 0);                 // [RC][Cn] forward rows k RC + rr
  TW* sTci = sTr + (MODE != 1 ? RC * Cn : 0);          // [R]      inverse columns
  TW* sTm = sTci + (MODE != 0 ? R : 0);                // [RC][Cn] mirrored rows R-1-(k RC + rr)
  {
    const TW* Trows = tw_rows + (size_t)l * R * Cn;
    if constexpr (MODE != 1) {
      for (int i = tid; i < R; i += G::TH) cp_async16(sTc + i, tw_col + (size_t)l * R + i);
      for (int i = tid; i < RC * Cn; i += G::TH) cp_async16(sTr + i, Trows + (size_t)k * RC * Cn + i);
    }
    if constexpr (MODE != 0) {
      for (int i = tid; i < R; i += G::TH) cp_async16(sTci + i, tw_col_inv + (size_t)l * R + i);
      for (int i = tid; i < RC * Cn; i += G::TH) {
        const int rr = i / Cn, e = i % Cn;
        cp_async16(sTm + i, Trows + (size_t)(R - 1 - (k * RC + rr)) * Cn + e);
      }
    }
    asm volatile("cp.async.commit_group;\n" ::: "memory");
  }
  auto tw_ready = [&] {
    asm volatile("cp.async.wait_all;\n" ::: "memory");
    __syncthreads();
  };
  // column twiddle of CT/GS stage s at row j: w[2^s + (j >> (n1 - s))]
  auto twc = [&](int s, int j) { return sTc[(1 << s) + (j >> (n1 - s))]; };
  auto twci = [&](int s, int j) { return sTci[(1 << s) + (j >> (n1 - s))]; };

  // ---------------- phase A: forward column stages
  if constexpr (MODE != 1) {
    sfor<0, G::NP1>([&](auto P_) {
      constexpr int p = decltype(P_)::value;
      constexpr int S = p * KE, K = clat_k(n1, KE, p), NG = E >> K;
      CGroup<R, S, K> gg[NG];
#pragma unroll
      for (int g = 0; g < NG; ++g) {
        gg[g].template at<CW, true>(tid + G::TH * g);
#pragma unroll
        for (int u = 0; u < (1 << K); ++u) {
          const int j = gg[g].pos(u);
          x[g * (1 << K) + u] =
              p == 0 ? __ldg(in + ubase + (size_t)j * Cn + k * CW + gg[g].line) : tile[j * CW + gg[g].line];
        }
      }
      if constexpr (p == 0) tw_ready();
#pragma unroll
      for (int g = 0; g < NG; ++g) clat_ct<S, K, 0>(x + g * (1 << K), gg[g], twc, q, q2);
      if constexpr (p < G::NP1 - 1) {
#pragma unroll
        for (int g = 0; g < NG; ++g)
#pragma unroll
          for (int u = 0; u < (1 << K); ++u) tile[gg[g].pos(u) * CW + gg[g].line] = x[g * (1 << K) + u];
        __syncthreads();
      } else {
        // X1: row j of column k CW + line -> row buffer of CTA j / RC
        cluster_wait();
#pragma unroll
        for (int g = 0; g < NG; ++g)
#pragma unroll
          for (int u = 0; u < (1 << K); ++u) {
            const int j = gg[g].pos(u);
            u64* dst = cluster.map_shared_rank(recv, j / RC);
            dst[(j % RC) * G::RPAD + rpos(k * CW + gg[g].line)] = x[g * (1 << K) + u];
          }
        cluster_sync_release_acquire();
      }
    });
  }

  // ---------------- phase B: row stages on rows [k RC, (k+1) RC)
  {
    // forward row twiddle of global stage s = n1 + v at column c of row r:
    // w[2^s + r 2^v + (c >> (n2 - v))] = Trows[r Cn + 2^v + (c >> (n2 - v))];
    // inverse: psi^{-brv(2^s + i)} = -w[2^{s+1} - 1 - i] = -(mirrored row R-1-r, entry 2^v + 2^v - 1 - (c >> (n2 - v)))
    int rowline = 0;   // set per group (all groups of a thread share the row when NG == 1)
    auto twr = [&](int s, int c) {
      const int v = s - n1;
      return sTr[rowline * Cn + (1 << v) + (c >> (n2 - v))];
    };
    auto twrm = [&](int s, int c) {
      const int v = s - n1;
      return sTm[rowline * Cn + (2 << v) - 1 - (c >> (n2 - v))];
    };
    if constexpr (MODE != 1) {
      // forward row passes 0 .. NP2-2 (the last one is fused below)
      sfor<0, G::NP2>([&](auto P_) {
        constexpr int p = decltype(P_)::value;
        constexpr int S = p * KE, K = clat_k(n2, KE, p), NG = E >> K;
        CGroup<Cn, S, K> gg[NG];
#pragma unroll
        for (int g = 0; g < NG; ++g) {
          gg[g].template at<RC, false>(tid + G::TH * g);
#pragma unroll
          for (int u = 0; u < (1 << K); ++u)
            x[g * (1 << K) + u] = recv[gg[g].line * G::RPAD + rpos(gg[g].pos(u))];
        }
#pragma unroll
        for (int g = 0; g < NG; ++g) {
          rowline = gg[g].line;
          clat_ct<S, K, n1>(x + g * (1 << K), gg[g], twr, q, q2);
        }
        if constexpr (p < G::NP2 - 1) {
#pragma unroll
          for (int g = 0; g < NG; ++g)
#pragma unroll
            for (int u = 0; u < (1 << K); ++u) recv[gg[g].line * G::RPAD + rpos(gg[g].pos(u))] = x[g * (1 << K) + u];
          __syncthreads();
        } else if constexpr (MODE == 0) {
#pragma unroll
          for (int g = 0; g < NG; ++g)
#pragma unroll
            for (int u = 0; u < (1 << K); ++u)
              out[ubase + (size_t)(k * RC + gg[g].line) * Cn + gg[g].pos(u)] = canon4(x[g * (1 << K) + u], q, q2);
        } else {
          // turn-around: (.) b_hat then the first GS pass (same stages, same registers)
          const u64 qinv = lc[l].qinv;
          const u64* bb = bop + (b_bcast ? (size_t)l * G::N : ubase);
#pragma unroll
          for (int g = 0; g < NG; ++g)
#pragma unroll
            for (int u = 0; u < (1 << K); ++u) {
              const size_t e = (size_t)(k * RC + gg[g].line) * Cn + gg[g].pos(u);
              x[g * (1 << K) + u] = mont_mul(x[g * (1 << K) + u], __ldg(bb + e), q, qinv);
            }
#pragma unroll
          for (int g = 0; g < NG; ++g) {
            rowline = gg[g].line;
            clat_gs<S, K, n1, Cn, false, true>(x + g * (1 << K), gg[g], twrm, TW{}, TW{}, q, q2);
          }
          if constexpr (G::NP2 > 1) {
#pragma unroll
            for (int g = 0; g < NG; ++g)
#pragma unroll
              for (int u = 0; u < (1 << K); ++u)
                recv[gg[g].line * G::RPAD + rpos(gg[g].pos(u))] = x[g * (1 << K) + u];
            __syncthreads();
          }
        }
      });
    }
    if constexpr (MODE != 0) {
      // inverse row passes: MODE 1 all of them (first from global), MODE 2 the rest
      constexpr int FIRST = MODE == 1 ? G::NP2 - 1 : G::NP2 - 2;
      sfor<0, FIRST + 1>([&](auto I_) {
        constexpr int p = FIRST - decltype(I_)::value;
        constexpr int S = p * KE, K = clat_k(n2, KE, p), NG = E >> K;
        CGroup<Cn, S, K> gg[NG];
#pragma unroll
        for (int g = 0; g < NG; ++g) {
          gg[g].template at<RC, false>(tid + G::TH * g);
#pragma unroll
          for (int u = 0; u < (1 << K); ++u)
            x[g * (1 << K) + u] = (MODE == 1 && p == G::NP2 - 1)
                                      ? __ldg(in + ubase + (size_t)(k * RC + gg[g].line) * Cn + gg[g].pos(u))
                                      : recv[gg[g].line * G::RPAD + rpos(gg[g].pos(u))];
        }
        if constexpr (MODE == 1 && p == G::NP2 - 1) tw_ready();
#pragma unroll
        for (int g = 0; g < NG; ++g) {
          rowline = gg[g].line;
          clat_gs<S, K, n1, Cn, false, true>(x + g * (1 << K), gg[g], twrm, TW{}, TW{}, q, q2);
        }
        if constexpr (p > 0) {
#pragma unroll
          for (int g = 0; g < NG; ++g)
#pragma unroll
            for (int u = 0; u < (1 << K); ++u)
              recv[gg[g].line * G::RPAD + rpos(gg[g].pos(u))] = x[g * (1 << K) + u];
          __syncthreads();
        }
      });
      // the thread now holds the row-pass-0 groups; X2: row r, column c -> tile of CTA c / CW
      {
        constexpr int K = clat_k(n2, KE, 0), NG = E >> K;
        if constexpr (MODE == 1) cluster_wait();
#pragma unroll
        for (int g = 0; g < NG; ++g) {
          CGroup<Cn, 0, K> gg;
          gg.template at<RC, false>(tid + G::TH * g);
#pragma unroll
          for (int u = 0; u < (1 << K); ++u) {
            const int c = gg.pos(u);
            u64* dst = cluster.map_shared_rank(tile, c / CW);
            dst[(k * RC + gg.line) * CW + c % CW] = x[g * (1 << K) + u];
          }
        }
        cluster_sync_release_acquire();
      }
    }
  }
  if constexpr (MODE == 0) return;

  // ---------------- phase A': inverse column stages, N^-1 (N^-1 2^64 after the Montgomery (.))
  {
    const TW s0 = MODE == 2 ? lc[l].ninvR : lc[l].ninv;
    const TW s1 = MODE == 2 ? lc[l].ninvR_w1 : lc[l].ninv_w1;
    sfor<0, G::NP1>([&](auto I_) {
      constexpr int p = G::NP1 - 1 - decltype(I_)::value;
      constexpr int S = p * KE, K = clat_k(n1, KE, p), NG = E >> K;
      CGroup<R, S, K> gg[NG];
#pragma unroll
      for (int g = 0; g < NG; ++g) {
        gg[g].template at<CW, true>(tid + G::TH * g);
#pragma unroll
        for (int u = 0; u < (1 << K); ++u) x[g * (1 << K) + u] = tile[gg[g].pos(u) * CW + gg[g].line];
      }
#pragma unroll
      for (int g = 0; g < NG; ++g) clat_gs<S, K, 0, R, true, false>(x + g * (1 << K), gg[g], twci, s0, s1, q, q2);
      if constexpr (p > 0) {
#pragma unroll
        for (int g = 0; g < NG; ++g)
#pragma unroll
          for (int u = 0; u < (1 << K); ++u) tile[gg[g].pos(u) * CW + gg[g].line] = x[g * (1 << K) + u];
        __syncthreads();
      } else {
#pragma unroll
        for (int g = 0; g < NG; ++g)
#pragma unroll
          for (int u = 0; u < (1 << K); ++u)
            out[ubase + (size_t)gg[g].pos(u) * Cn + k * CW + gg[g].line] = canon2(x[g * (1 << K) + u], q);
      }
    });
  }
}

}  // namespace rnt
