// api.cu -- C ABI (include/rnsntt.h) over the sm_100a kernels.
//
// Dispatch (reading C14): N = 2^4 .. 2^10 -> one-kernel warp NTT (ntt_small.cuh);
// N = 2^11 .. 2^16 -> two-pass column/row NTT (ntt_large.cuh).  Every entry
// point validates its arguments on the host before launching anything and
// never synchronises the stream.
#include <cuda_runtime.h>

#include <atomic>
#include <mutex>
#include <cstdio>
#include <algorithm>
#include <cstdlib>
#include <cstring>
#include <new>
#include <vector>

#include "../../include/rnsntt.h"
#include "modarith.cuh"
#include "ntt_large.cuh"
#include "ntt_small.cuh"
#include "keyswitch.cuh"
#include "ntt_cluster.cuh"
#include "ntt_clat.cuh"
#include "hrf.cuh"
#include "plan.h"

using namespace rnt;

struct rnt_plan_s {
  uint32_t logn = 0, L = 0;
  int device = 0;
  std::vector<HostLimb> limbs;
  LimbC* d_lc = nullptr;
  TW* d_fwd = nullptr;      // natural order (n <= 10) or row layout (n >= 11), [L][N]
  TW* d_inv = nullptr;
  TW* d_col_fwd = nullptr;  // n >= 11: natural entries [L][2^{n1}]
  TW* d_col_inv = nullptr;
  TW* d_rowtw = nullptr;    // n >= 11: natural per-row forward table [L][2^{n1}][2^{n2}] (k_rows)
  // rnt_execute_host pipelining: auxiliary streams, created on first use
  std::mutex aux_mu;
  cudaStream_t aux[3] = {nullptr, nullptr, nullptr};   // H2D copy, compute, D2H copy
  std::vector<cudaEvent_t> ev_pool;                    // per-chunk events, reused under aux_mu
  // limb-window split of single-polynomial multi-limb jobs (N >= 2^11)
  std::mutex split_mu;
  cudaStream_t split[4] = {nullptr, nullptr, nullptr, nullptr};
  cudaEvent_t split_ev[5] = {nullptr, nullptr, nullptr, nullptr, nullptr};
  bool is_view = false;     // limb-window view used internally (owns nothing)
  bool lazy60 = false;      // every modulus < 2^60: LZ kernels (ct_bfly_lz, 16q lazy bound) are valid
};

// Shallow limb-window view [l0, l0 + nl) of a plan (for batch == 1 chunking).
static void make_view(const rnt_plan_s* p, uint32_t l0, uint32_t nl, rnt_plan_s* v) {
  v->logn = p->logn;
  v->L = nl;
  v->device = p->device;
  v->d_lc = p->d_lc + l0;
  const size_t n = (size_t)1 << p->logn;
  v->d_fwd = p->d_fwd + l0 * n;
  v->d_inv = p->d_inv ? p->d_inv + l0 * n : nullptr;
  if (p->d_col_fwd) {
    const size_t r = (size_t)1 << ((p->logn + 1) / 2);
    v->d_col_fwd = p->d_col_fwd + l0 * r;
    v->d_col_inv = p->d_col_inv + l0 * r;
    v->d_rowtw = p->d_rowtw + l0 * n;
  }
  v->is_view = true;
  v->lazy60 = p->lazy60;
}

static thread_local int g_last_cuda = 0;
static std::atomic<uint64_t> g_launches{0};

static rnt_status cuda_fail(cudaError_t e) {
  g_last_cuda = (int)e;
  return e == cudaErrorMemoryAllocation ? RNT_E_OOM : RNT_E_CUDA;
}

#define RNT_CUDA(call)                         \
  do {                                         \
    cudaError_t e_ = (call);                   \
    if (e_ != cudaSuccess) return cuda_fail(e_); \
  } while (0)

static rnt_status after_launch() {
  g_launches.fetch_add(1, std::memory_order_relaxed);
  cudaError_t e = cudaGetLastError();
  return e == cudaSuccess ? RNT_OK : cuda_fail(e);
}

// ------------------------------------------------------------------ kernels
// Elementwise (.) of Eq. 1 with canonical output: mont(mont(a, b), R^2) = a b mod q.
__global__ void k_pointwise(u64* __restrict__ c, const u64* __restrict__ a, const u64* __restrict__ b,
                            int b_bcast, const LimbC* __restrict__ lc, uint32_t L, uint32_t logn,
                            uint64_t total2) {
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  for (uint64_t v = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; v < total2; v += stride) {
    const uint64_t e = v * 2;
    const uint64_t u = e >> logn;
    const uint32_t l = (uint32_t)(u % L);
    const uint64_t k = e & ((1ull << logn) - 1);
    const u64 q = lc[l].q, qinv = lc[l].qinv, r2 = lc[l].r2;
    const ulonglong2 av = __ldg(reinterpret_cast<const ulonglong2*>(a) + v);
    const uint64_t bi = b_bcast ? (((uint64_t)l << logn) + k) : e;
    const ulonglong2 bv = __ldg(reinterpret_cast<const ulonglong2*>(b + bi));
    ulonglong2 cv;
    cv.x = canon2(mont_mul(mont_mul(av.x, bv.x, q, qinv), r2, q, qinv), q);
    cv.y = canon2(mont_mul(mont_mul(av.y, bv.y, q, qinv), r2, q, qinv), q);
    reinterpret_cast<ulonglong2*>(c)[v] = cv;
  }
}

// Galois automorphism sigma_g (rnt_automorph).
//   NTT form:  out[k] = in[pi(k)],  2 brv(pi(k)) + 1 = (2 brv(k) + 1) g mod 2N
//   coeff form: out[j] = +-in[j g^{-1} mod 2N] (sign when the source index >= N)
// Scatter formulation (default): a thread reads in[e] (coalesced) and writes it to its
// destination -- pi^{-1} is the same map with g^{-1}, and coefficient i goes to i g mod
// 2N (negated past N) -- so the loads never stall on a gather; the 8-byte scattered
// stores merge into sectors in L2.  RNT_AUTOMORPH_SCATTER=0 (experiment builds) keeps the
// gather form.  One limb is 8N bytes (512 KB at 2^16): L2-resident while it is permuted.
#ifndef RNT_AUTOMORPH_SCATTER
#define RNT_AUTOMORPH_SCATTER 1
#endif
__global__ void k_automorph(u64* __restrict__ out, const u64* __restrict__ in, const LimbC* __restrict__ lc,
                            uint32_t L, uint32_t logn, uint32_t g, uint32_t ginv, int ntt_domain, uint64_t total) {
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  const uint32_t n = 1u << logn, mask2n = 2 * n - 1;
  for (uint64_t e = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; e < total; e += stride) {
    const uint64_t u = e >> logn;
    const uint32_t k = (uint32_t)(e & (n - 1));
#if RNT_AUTOMORPH_SCATTER
    const u64 x = __ldcs(in + e);
    u64* dst = out + (u << logn);
    if (ntt_domain) {
      const uint32_t ek = 2u * (__brev(k) >> (32 - logn)) + 1u;
      const uint32_t es = (uint32_t)(((uint64_t)ek * ginv) & mask2n);
      dst[__brev((es - 1u) >> 1) >> (32 - logn)] = x;
    } else {
      const uint32_t t = (uint32_t)(((uint64_t)k * g) & mask2n);
      if (t < n) {
        dst[t] = x;
      } else {
        const u64 q = lc[u % L].q;
        dst[t - n] = x ? q - x : 0ull;
      }
    }
#else
    const u64* src = in + (u << logn);
    u64 v;
    if (ntt_domain) {
      const uint32_t ek = 2u * (__brev(k) >> (32 - logn)) + 1u;          // odd exponent of slot k
      const uint32_t es = (uint32_t)(((uint64_t)ek * g) & mask2n);       // times g mod 2N (odd)
      const uint32_t kk = __brev((es - 1u) >> 1) >> (32 - logn);
      v = __ldg(src + kk);
    } else {
      const uint32_t i0 = (uint32_t)(((uint64_t)k * ginv) & mask2n);
      if (i0 < n) {
        v = __ldg(src + i0);
      } else {
        const u64 x = __ldg(src + (i0 - n));
        const u64 q = lc[u % L].q;
        v = x ? q - x : 0ull;
      }
    }
    out[e] = v;
#endif
  }
}

// Fast basis conversion (rnt_bconv_apply).  A CTA converts kBcTile coefficient
// positions of one polynomial: phase 1 computes y_i = x_i qhat_i^{-1} mod q_i
// into shared memory, phase 2 accumulates out_j = sum_i y_i (qhat_i mod p_j)
// with Shoup products w.r.t. p_j (lazy [0, 2p_j), one conditional subtraction
// per term), canonical output.
constexpr int kBcTile = 128;
struct BcMod {
  u64 m, m2;
  TW qhatinv;  // only for source limbs
};

__global__ void __launch_bounds__(kBcTile)
k_bconv(u64* __restrict__ out, const u64* __restrict__ in, const BcMod* __restrict__ src, const BcMod* __restrict__ dst,
        const TW* __restrict__ qhat_p, uint32_t L, uint32_t K, uint32_t logn) {
  extern __shared__ __align__(16) u64 ys[];   // [L][kBcTile]
  const uint32_t n = 1u << logn;
  const uint64_t b = blockIdx.y;
  const uint32_t c = blockIdx.x * kBcTile + threadIdx.x;
  const bool live = c < n;
  const u64* x = in + (b * L << logn) + (live ? c : 0);
  for (uint32_t i = 0; i < L; ++i) {
    const u64 q = src[i].m;
    ys[i * kBcTile + threadIdx.x] = csub(shoup_lazy(__ldg(x + ((uint64_t)i << logn)), src[i].qhatinv, q), q);
  }
  __syncthreads();
  if (!live) return;
  u64* o = out + (b * K << logn) + c;
  for (uint32_t j = 0; j < K; ++j) {
    const u64 p = dst[j].m, p2 = dst[j].m2;
    const TW* row = qhat_p + (size_t)j * L;
    u64 acc = 0;
#pragma unroll 4
    for (uint32_t i = 0; i < L; ++i) acc = csub(acc + shoup_lazy(ys[i * kBcTile + threadIdx.x], ldg_tw(row + i), p), p2);
    o[(uint64_t)j << logn] = csub(acc, p);
  }
}

// RNT_DEBUG=1: residue range check of the inputs (reading C6).  Sets *bad
// when some element of limb (u % L) is >= q.
__global__ void k_check_range(const u64* __restrict__ x, const LimbC* __restrict__ lc, uint32_t L, uint32_t logn,
                              uint64_t total, int* __restrict__ bad) {
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  int any = 0;
  for (uint64_t e = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; e < total; e += stride)
    any |= __ldg(x + e) >= lc[(e >> logn) % L].q;
  if (__syncthreads_or(any) && threadIdx.x == 0) atomicOr(bad, 1);
}

static int num_sms() {
  static const int n = [] {
    int d = 0, v = 0;
    cudaGetDevice(&d);
    cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, d);
    return v > 0 ? v : 148;
  }();
  return n;
}

// Integer tuning knob from the environment, read once (thread-safe static init).
static int env_int(const char* name, int dflt) {
  const char* e = getenv(name);
  return e ? atoi(e) : dflt;
}

// One-time (per kernel, per device) function attributes: dynamic shared memory
// above 48 KB and, for 16-CTA clusters, the non-portable cluster size.
template <typename K>
static rnt_status ensure_attr(K kern, size_t smem, std::atomic<uint64_t>& done, bool nonportable = false) {
  int d = 0;
  RNT_CUDA(cudaGetDevice(&d));
  const uint64_t bit = 1ull << (d & 63);
  if (done.load(std::memory_order_acquire) & bit) return RNT_OK;
  RNT_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  if (nonportable) RNT_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
  done.fetch_or(bit, std::memory_order_release);
  return RNT_OK;
}

// Kernels whose shared memory depends on runtime sizes: set it on every call
// above the default 48 KB (host-side, microseconds; not on the NTT hot path).
template <typename K>
static rnt_status set_smem(K kern, size_t smem) {
  if (smem > 48 * 1024) RNT_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  return RNT_OK;
}

// ---------------------------------------------------------------- launchers
template <int LOGN, int MODE, int W, int MINB, bool SYNC, int KM = 4, bool LZ = false, int TEAM = 1>
static rnt_status launch_warp_v(const rnt_plan_s* p, u64* out, const u64* in, const u64* bop,
                                int bcast, uint32_t batch, cudaStream_t st) {
  static std::atomic<uint64_t> attr{0};
  auto kern = k_warp<LOGN, MODE, W, MINB, SYNC, KM, LZ, TEAM>;
  const size_t smem = warp_smem_bytes<LOGN, MODE, W, TEAM>();
  if (rnt_status s = ensure_attr(kern, smem, attr); s != RNT_OK) return s;
  const uint64_t per_cta = (uint64_t)(W / TEAM) * WarpCfg<LOGN>::P;
  const uint64_t gx = (batch + per_cta - 1) / per_cta;
  for (uint32_t l0 = 0; l0 < p->L; l0 += 65535u) {
    const uint32_t nl = p->L - l0 < 65535u ? p->L - l0 : 65535u;
    dim3 grid((unsigned)gx, nl);
    kern<<<grid, W * 32, smem, st>>>(
        out + ((size_t)l0 << LOGN), in + ((size_t)l0 << LOGN), bop ? bop + ((size_t)l0 << LOGN) : nullptr, bcast,
        p->d_fwd + ((size_t)l0 << LOGN), p->d_inv + ((size_t)l0 << LOGN), p->d_lc + l0, p->L, batch);
    rnt_status s = after_launch();
    if (s != RNT_OK) return s;
  }
  return RNT_OK;
}

// Dispatch test hook (documented in rnsntt.h): RNT_LAZY=0 keeps the [0, 4q)
// kernels even when every modulus is below 2^60.
static bool lazy_enabled() {
  static const bool v = env_int("RNT_LAZY", 1) != 0;
  return v;
}

// CTAs per SM the warp engine is compiled for (2 warps each); experiments rebuild
// with RNT_NVCC_EXTRA=-DRNT_WARP_MINB=n (build.py), the shipped value is 12.
#ifndef RNT_WARP_MINB
#define RNT_WARP_MINB 12
#endif
// N = 2^10 units (forward, inverse, polymul) run on teams of 2 warps per polynomial (one
// CTA), compiled for 16 CTAs = 32 warps per SM (<= 64 registers, no spills).  Measured (profiles/r02/teams,
// team2_minb): one warp per polynomial at 24 warps/SM: cfg2 0.0816 ms, cfg5 k_warp 0.2619 ms
// (cfg2's 4096 units are 1.15 waves); 2-warp teams at 24 warps/SM: 0.0764 / 0.2609; at 28 /
// 32 / 36 / 40 / 48 warps/SM: cfg5 0.2594 / 0.2553 / 0.2565 / 0.2573 / 0.2653 ms, cfg2 0.0742
// / 0.0741 / 0.0753 / 0.0766 / 0.0810 ms; teams of 4 warps: cfg2 0.0763, cfg5 0.2673 ms.
// Experiment builds: -DRNT_TEAM2_WAVES=x (one-warp units from x waves up; default: always
// teams), -DRNT_TEAM2_MINB=n.
#ifndef RNT_TEAM2_WAVES
#define RNT_TEAM2_WAVES 1e30
#endif
#ifndef RNT_TEAM2_MINB
#define RNT_TEAM2_MINB 16
#endif
// Jobs below this many waves of 2-warp teams run 4-warp teams (experiment builds:
// -DRNT_TEAM4_WAVES=x).
#ifndef RNT_TEAM4_WAVES
#define RNT_TEAM4_WAVES 3
#endif
// Pass schedule of the LZ warp engine (Passes<LOGN, KM>): 32 = radix-8 with the split
// tail (N = 2^10: 3 + 3 + 2 + 2); experiment builds: -DRNT_WARP_KM=40 (4 + 4 + 2).
#ifndef RNT_WARP_KM
#define RNT_WARP_KM 32
#endif

template <int LOGN, int MODE>
static rnt_status launch_warp(const rnt_plan_s* p, u64* out, const u64* in, const u64* bop,
                              int bcast, uint32_t batch, cudaStream_t st) {
  // radix-8 passes, 2 warps per CTA: one warp per buffer at <= 85 registers (24 warps/SM),
  // or for the N = 2^10 polymul a 2-warp team per buffer at <= 64 registers (32 warps/SM);
  // lazy CT ranges with the split-tail schedule (N = 2^10: 3 + 3 + 2 + 2, the polymul turn
  // pass on 4-coefficient groups) when every modulus is below 2^60; [0, 4q) Harvey ranges
  // with 3 + 3 + 3 + 1 otherwise
  if (p->lazy60 && lazy_enabled()) {
    if constexpr (LOGN == 10) {
      const double waves = (double)batch * p->L / ((double)num_sms() * RNT_WARP_MINB * 2);
      // below 3 waves of 2-warp teams, teams of 4 warps (8 CTAs = 32 warps per SM): a shorter
      // critical path per polynomial beats the coarser wave quantization (round 2, session 3,
      // profiles/r02/t4: 1200 / 2731 / 3000 / 4096 / 6000 polymuls 37.1 / 61.1 / 65.0 / 78.6 /
      // 108.7 -> 34.9 / 57.1 / 61.9 / 77.7 / 107.4 us; 8192 / 16384: 139.5 / 259.1 -> 140.6 /
      // 262.3 us, so larger batches keep the 2-warp teams)
      if ((uint64_t)batch * p->L < (uint64_t)num_sms() * RNT_TEAM2_MINB * RNT_TEAM4_WAVES)
        return launch_warp_v<LOGN, MODE, 4, 8, false, RNT_WARP_KM, true, 4>(p, out, in, bop, bcast, batch, st);
      if (waves < RNT_TEAM2_WAVES)
        return launch_warp_v<LOGN, MODE, 2, RNT_TEAM2_MINB, false, RNT_WARP_KM, true, 2>(p, out, in, bop, bcast, batch,
                                                                                          st);
    }
    return launch_warp_v<LOGN, MODE, 2, RNT_WARP_MINB, false, RNT_WARP_KM, true>(p, out, in, bop, bcast, batch, st);
  }
  return launch_warp_v<LOGN, MODE, 2, RNT_WARP_MINB, false, 3>(p, out, in, bop, bcast, batch, st);
}

// Latency engine (k_lat, ntt_small.cuh) for jobs of at most lat_units()
// (polynomial, limb) units at N <= 2^10 (env RNT_LAT_UNITS; 0 disables).  Default
// 512 (round 1: crossover with the warp engine near 1024 units, 2^10 polymul 18.6 vs
// 24.7 us at 512 units), 256 for the N = 2^10 LZ plans whose warp engine runs 4-warp
// teams on small batches (round 2, profiles/r02/lat: 128 / 256 / 384 / 512 units 16.6 /
// 20.0 / 24.1 / 26.6 us on k_lat, 19.9 / 20.0 / 21.7 / 22.6 us on the warp engine).
static int lat_units(const rnt_plan_s* p) {
  static const int v = env_int("RNT_LAT_UNITS", -1);
  if (v >= 0) return v;
  return (p->logn == 10 && p->lazy60 && lazy_enabled()) ? 256 : 512;
}

template <int LOGN, int MODE>
static rnt_status launch_lat(const rnt_plan_s* p, u64* out, const u64* in, const u64* bop, int bcast, uint32_t batch,
                             cudaStream_t st) {
  const uint64_t units = (uint64_t)batch * p->L;
  k_lat<LOGN, MODE><<<(unsigned)units, (1 << LOGN) / 2, 0, st>>>(out, in, bop, bcast, p->d_fwd, p->d_inv, p->d_lc,
                                                                   p->L);
  return after_launch();
}

template <int MODE>
static rnt_status lat_dispatch(const rnt_plan_s* p, u64* out, const u64* in, const u64* bop, int bcast,
                               uint32_t batch, cudaStream_t st) {
  switch (p->logn) {
    case 4: return launch_lat<4, MODE>(p, out, in, bop, bcast, batch, st);
    case 5: return launch_lat<5, MODE>(p, out, in, bop, bcast, batch, st);
    case 6: return launch_lat<6, MODE>(p, out, in, bop, bcast, batch, st);
    case 7: return launch_lat<7, MODE>(p, out, in, bop, bcast, batch, st);
    case 8: return launch_lat<8, MODE>(p, out, in, bop, bcast, batch, st);
    case 9: return launch_lat<9, MODE>(p, out, in, bop, bcast, batch, st);
    case 10: return launch_lat<10, MODE>(p, out, in, bop, bcast, batch, st);
    default: return RNT_E_UNSUPPORTED_N;
  }
}

static int cluster_units();
static bool clat_enabled();
template <int LOGN>
static rnt_status clat_op(const rnt_plan_s* p, int op, u64* out, const u64* in, const u64* bop, int bcast,
                          uint32_t batch, cudaStream_t st);

template <int MODE>
static rnt_status warp_dispatch(const rnt_plan_s* p, u64* out, const u64* in, const u64* bop, int bcast,
                                uint32_t batch, cudaStream_t st) {
  // single-unit jobs at N = 2^10 (cfg1): the cluster latency kernel spreads the
  // limb over 8 SMs (k_clat, defined below); polymul with coefficient-form b stays on k_lat
  if constexpr (MODE <= 2) {
    if (p->logn == 10 && (uint64_t)batch * p->L <= (uint64_t)cluster_units() && clat_enabled())
      return clat_op<10>(p, MODE, out, in, bop, bcast, batch, st);
  }
  if ((uint64_t)batch * p->L <= (uint64_t)lat_units(p)) return lat_dispatch<MODE>(p, out, in, bop, bcast, batch, st);
  switch (p->logn) {
    case 4: return launch_warp<4, MODE>(p, out, in, bop, bcast, batch, st);
    case 5: return launch_warp<5, MODE>(p, out, in, bop, bcast, batch, st);
    case 6: return launch_warp<6, MODE>(p, out, in, bop, bcast, batch, st);
    case 7: return launch_warp<7, MODE>(p, out, in, bop, bcast, batch, st);
    case 8: return launch_warp<8, MODE>(p, out, in, bop, bcast, batch, st);
    case 9: return launch_warp<9, MODE>(p, out, in, bop, bcast, batch, st);
    case 10: return launch_warp<10, MODE>(p, out, in, bop, bcast, batch, st);
    default: return RNT_E_UNSUPPORTED_N;
  }
}

// CTA order for the two-pass kernels: block b -> (sub-block, poly, limb) with
// the sub-block fastest, then the polynomial, then the limb, so CTAs that
// share a limb's twiddle rows run back to back (L2 reuse across the batch).
// Launch shape chosen per call by large_op: N = 2^16 jobs of >= 192 limb-units
// (cfg4) take 8-column pass-1 tiles and the warp-engine rows (k_rows; cfg4
// 0.827 -> 0.804 ms); smaller jobs the 16-column tiles and k_row (k_rows
// under-fills the GPU for one 45-limb polynomial: cfg3 0.097 -> 0.111 ms).
static thread_local bool g_large_wide = false;   // set by large_op for the current call
static thread_local bool g_rows_warp = false;    // rows through k_rows (wide path or RNT_ROWS_WARP_UNITS)
static thread_local bool g_col8 = false;         // 8-column pass-1 tiles (wide path or RNT_COL8_UNITS)
// Experiment builds: -DRNT_WIDE_UNITS=n (limb-units from which the wide path is taken),
// -DRNT_ROWS_TEAM=2 (k_rows with 2-warp teams).
#ifndef RNT_WIDE_UNITS
#define RNT_WIDE_UNITS 192
#endif
#ifndef RNT_ROWS_TEAM
#define RNT_ROWS_TEAM 1
#endif
#ifndef RNT_ROWS_WARP_UNITS
#define RNT_ROWS_WARP_UNITS RNT_WIDE_UNITS
#endif
#ifndef RNT_COL8_UNITS
#define RNT_COL8_UNITS RNT_WIDE_UNITS
#endif

// Launch with the programmatic-stream-serialization attribute: the kernel may be
// scheduled before its stream predecessor finishes and waits for it in-kernel (pdl_wait,
// ntt_large.cuh).  Used for the dependent kernels of an N >= 2^11 chain.
template <typename... KArgs, typename... Args>
static cudaError_t launch_pdl(void (*kern)(KArgs...), dim3 g, dim3 b, size_t smem, cudaStream_t st, Args... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = g;
  cfg.blockDim = b;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = RNT_PDL;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, kern, static_cast<KArgs>(args)...);
}

template <int LOGN, int CT, bool LZ = false>
static rnt_status launch_col_v(const rnt_plan_s* p, bool inv, int after_mont, u64* out, const u64* in,
                               uint32_t batch, cudaStream_t st) {
  using P = TwoPass<LOGN>;
  const uint64_t units = (uint64_t)batch * p->L;
  for (uint64_t y0 = 0; y0 < units; y0 += 65535u) {
    const uint64_t cnt = units - y0 < 65535u ? units - y0 : 65535u;
    dim3 g(P::Cn / CT, (unsigned)cnt);
    if (inv) {
      RNT_CUDA(launch_pdl(k_col_inv<LOGN, CT>, g, dim3(CT * P::T1), 0, st, out, in, p->d_col_inv, p->d_lc, p->L,
                          batch, y0, after_mont));
    } else
      k_col_fwd<LOGN, CT, false, LZ><<<g, CT * P::T1, 0, st>>>(out, in, p->d_col_fwd, p->d_lc, p->L, batch, y0);
    rnt_status s = after_launch();
    if (s != RNT_OK) return s;
  }
  return RNT_OK;
}

template <int LOGN>
static rnt_status launch_col(const rnt_plan_s* p, bool inv, int after_mont, u64* out, const u64* in,
                             uint32_t batch, cudaStream_t st) {
  // forward columns with lazy CT ranges when the plan allows it; the row pass
  // that consumes them (launch_row) makes the same choice
  if (!inv && p->lazy60 && lazy_enabled()) {
    if (g_col8) return launch_col_v<LOGN, 8, true>(p, inv, after_mont, out, in, batch, st);
    return launch_col_v<LOGN, kColTile, true>(p, inv, after_mont, out, in, batch, st);
  }
  if (g_col8) return launch_col_v<LOGN, 8>(p, inv, after_mont, out, in, batch, st);
  return launch_col_v<LOGN, kColTile>(p, inv, after_mont, out, in, batch, st);
}

// Rows per k_row CTA (experiment builds: -DRNT_ROW_RPC=n with -DRNT_ROW_MINB=m; 8 rows x 4
// CTAs/SM measured within 0.5 % of the default 16 x 2, profiles/r02/README).
#ifndef RNT_ROW_RPC
#define RNT_ROW_RPC 0
#endif
template <int LOGN>
constexpr int kRowRpc() { return RNT_ROW_RPC ? RNT_ROW_RPC : TwoPass<LOGN>::RPC; }

template <int LOGN, int MODE, int RPC_, bool LZ = false>
static rnt_status launch_row_v(const rnt_plan_s* p, u64* out, const u64* in, const u64* bop, int bcast,
                               uint32_t batch, cudaStream_t st) {
  using P = TwoPass<LOGN>;
  const uint64_t units = (uint64_t)batch * p->L;
  for (uint64_t y0 = 0; y0 < units; y0 += 65535u) {
    const uint64_t cnt = units - y0 < 65535u ? units - y0 : 65535u;
    dim3 g(P::R / RPC_, (unsigned)cnt);
    RNT_CUDA(launch_pdl(k_row<LOGN, MODE, RPC_, LZ>, g, dim3(RPC_ * P::T2), 0, st, out, in, bop, bcast, p->d_fwd,
                        p->d_lc, p->L, batch, y0));
    rnt_status s = after_launch();
    if (s != RNT_OK) return s;
  }
  return RNT_OK;
}

template <int LOGN, int MODE, bool LZ = false, int TEAM = 1>
static rnt_status launch_rows_warp(const rnt_plan_s* p, u64* out, const u64* in, const u64* bop, int bcast,
                                   uint32_t batch, cudaStream_t st) {
  using P = TwoPass<LOGN>;
  static std::atomic<uint64_t> attr{0};
  auto kern = k_rows<LOGN, MODE, LZ, TEAM>;
  const size_t smem = (size_t)(kRowWarps / TEAM) * kWarpBuf * 8;
  if (rnt_status s = ensure_attr(kern, smem, attr); s != RNT_OK) return s;
  constexpr int rows_per_cta = (kRowWarps / TEAM) * (kWarpElems / P::Cn);
  const unsigned gx = (unsigned)((P::R + rows_per_cta - 1) / rows_per_cta);
  const uint64_t units = (uint64_t)batch * p->L;
  for (uint64_t y0 = 0; y0 < units; y0 += 65535u) {
    const uint64_t cnt = units - y0 < 65535u ? units - y0 : 65535u;
    dim3 g(gx, (unsigned)cnt);
    RNT_CUDA(launch_pdl(kern, g, dim3(kRowWarps * 32), smem, st, out, in, bop, bcast, p->d_rowtw, p->d_lc, p->L,
                        batch, y0));
    rnt_status s = after_launch();
    if (s != RNT_OK) return s;
  }
  return RNT_OK;
}

template <int LOGN, int MODE>
static rnt_status launch_row(const rnt_plan_s* p, u64* out, const u64* in, const u64* bop, int bcast,
                             uint32_t batch, cudaStream_t st) {
  if constexpr (MODE != 1) {
    // input from an LZ forward column pass (launch_col makes the same choice)
    if (p->lazy60 && lazy_enabled()) {
      if (g_rows_warp) return launch_rows_warp<LOGN, MODE, true, RNT_ROWS_TEAM>(p, out, in, bop, bcast, batch, st);
      return launch_row_v<LOGN, MODE, kRowRpc<LOGN>(), true>(p, out, in, bop, bcast, batch, st);
    }
  }
  if (g_rows_warp) return launch_rows_warp<LOGN, MODE, false, RNT_ROWS_TEAM>(p, out, in, bop, bcast, batch, st);
  return launch_row_v<LOGN, MODE, kRowRpc<LOGN>()>(p, out, in, bop, bcast, batch, st);
}

template <int LOGN>
static rnt_status large_op(const rnt_plan_s* p, int op, u64* out, const u64* in, const u64* bop, int bcast,
                           uint32_t batch, cudaStream_t st) {
  rnt_status s;
  g_large_wide = LOGN == 16 && (uint64_t)batch * p->L >= RNT_WIDE_UNITS;
  g_rows_warp = g_large_wide || (LOGN == 16 && (uint64_t)batch * p->L >= RNT_ROWS_WARP_UNITS);
  g_col8 = g_large_wide || (LOGN == 16 && (uint64_t)batch * p->L >= RNT_COL8_UNITS);
  switch (op) {
    case 0:  // forward
      if ((s = launch_col<LOGN>(p, false, 0, out, in, batch, st)) != RNT_OK) return s;
      return launch_row<LOGN, 0>(p, out, out, nullptr, 0, batch, st);
    case 1:  // inverse
      if ((s = launch_row<LOGN, 1>(p, out, in, nullptr, 0, batch, st)) != RNT_OK) return s;
      return launch_col<LOGN>(p, true, 0, out, out, batch, st);
    case 2:  // c = INTT(NTT(a) . b_hat)
      if ((s = launch_col<LOGN>(p, false, 0, out, in, batch, st)) != RNT_OK) return s;
      if ((s = launch_row<LOGN, 2>(p, out, out, bop, bcast, batch, st)) != RNT_OK) return s;
      return launch_col<LOGN>(p, true, 1, out, out, batch, st);
    default: return RNT_E_INVALID_ARG;
  }
}

// Single-launch cluster path (ntt_cluster.cuh) for latency-bound jobs: a
// cluster of C CTAs owns one limb on chip.  Used when batch * L is at most
// cluster_units() (dispatch test hook RNT_CLUSTER_UNITS; 0 disables).
static int cluster_units() {
  static const int v = env_int("RNT_CLUSTER_UNITS", 2);
  return v;
}

template <int LOGN, int C, int MODE>
static rnt_status launch_cluster_v(const rnt_plan_s* p, u64* out, const u64* in, const u64* bop, int bcast,
                                   uint32_t batch, cudaStream_t st) {
  using G = ClusterGeo<LOGN, C>;
  auto kern = k_cluster<LOGN, C, MODE>;
  static std::atomic<uint64_t> attr{0};
  if (rnt_status s = ensure_attr(kern, G::SMEM, attr, C > 8); s != RNT_OK) return s;
  const uint64_t units = (uint64_t)batch * p->L;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3((unsigned)(units * C), 1, 1);
  cfg.blockDim = dim3(G::THREADS, 1, 1);
  cfg.dynamicSmemBytes = G::SMEM;
  cfg.stream = st;
  cudaLaunchAttribute a[1];
  a[0].id = cudaLaunchAttributeClusterDimension;
  a[0].val.clusterDim.x = C;
  a[0].val.clusterDim.y = 1;
  a[0].val.clusterDim.z = 1;
  cfg.attrs = a;
  cfg.numAttrs = 1;
  const TW* cf = p->d_col_fwd;
  const TW* ci = p->d_col_inv;
  const TW* rf = p->d_fwd;
  const LimbC* lcp = p->d_lc;
  RNT_CUDA(cudaLaunchKernelEx(&cfg, kern, out, in, bop, bcast, cf, ci, rf, lcp, p->L));
  return after_launch();
}

template <int LOGN, int C>
static rnt_status cluster_op_c(const rnt_plan_s* p, int op, u64* out, const u64* in, const u64* bop, int bcast,
                               uint32_t batch, cudaStream_t st) {
  switch (op) {
    case 0: return launch_cluster_v<LOGN, C, 0>(p, out, in, bop, bcast, batch, st);
    case 1: return launch_cluster_v<LOGN, C, 1>(p, out, in, bop, bcast, batch, st);
    case 2: return launch_cluster_v<LOGN, C, 2>(p, out, in, bop, bcast, batch, st);
    default: return RNT_E_INVALID_ARG;
  }
}

// Latency cluster kernel (ntt_clat.cuh): E = 4 coefficients per thread and C CTAs
// per limb (clat_op).
template <int LOGN, int C, int E, int MODE>
static rnt_status launch_clat_v(const rnt_plan_s* p, u64* out, const u64* in, const u64* bop, int bcast,
                                uint32_t batch, cudaStream_t st) {
  using G = Clat<LOGN, C, E>;
  auto kern = k_clat<LOGN, C, E, MODE>;
  static std::atomic<uint64_t> attr{0};
  if (rnt_status s = ensure_attr(kern, G::template smem<MODE>(), attr, C > 8); s != RNT_OK) return s;
  const uint64_t units = (uint64_t)batch * p->L;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3((unsigned)(units * C), 1, 1);
  cfg.blockDim = dim3(G::TH, 1, 1);
  cfg.dynamicSmemBytes = G::template smem<MODE>();
  cfg.stream = st;
  cudaLaunchAttribute a[1];
  a[0].id = cudaLaunchAttributeClusterDimension;
  a[0].val.clusterDim.x = C;
  a[0].val.clusterDim.y = 1;
  a[0].val.clusterDim.z = 1;
  cfg.attrs = a;
  cfg.numAttrs = 1;
  const TW* cf = p->d_col_fwd;
  const TW* ci = p->d_col_inv;
  const TW* rt = p->d_rowtw;
  const LimbC* lcp = p->d_lc;
  RNT_CUDA(cudaLaunchKernelEx(&cfg, kern, out, in, bop, bcast, cf, ci, rt, lcp, p->L));
  return after_launch();
}

template <int LOGN, int C, int E>
static constexpr bool clat_valid() {
  return (1 << LOGN) / C / E >= 32 && (1 << LOGN) / C / E <= 1024 && (1 << (LOGN / 2)) >= C;
}

template <int LOGN, int C, int E>
static rnt_status clat_op_ce(const rnt_plan_s* p, int op, u64* out, const u64* in, const u64* bop, int bcast,
                             uint32_t batch, cudaStream_t st) {
  switch (op) {
    case 0: return launch_clat_v<LOGN, C, E, 0>(p, out, in, bop, bcast, batch, st);
    case 1: return launch_clat_v<LOGN, C, E, 1>(p, out, in, bop, bcast, batch, st);
    case 2: return launch_clat_v<LOGN, C, E, 2>(p, out, in, bop, bcast, batch, st);
    default: return RNT_E_INVALID_ARG;
  }
}

// Defaults (measured, single-polynomial forward latency under CUDA-graph replay;
// E = 8 coefficients per thread measured slower at every N and is not built):
// C = 8 up to 2^12, 16 above; E = 4 (2^12 / 2^13 / 2^14 / 2^15: 3.5 / 3.8 / 5.2 / 8.0 us
// vs 7.5 / 8.1 / 8.2 / 9.4 us for k_cluster).
template <int LOGN>
static rnt_status clat_op(const rnt_plan_s* p, int op, u64* out, const u64* in, const u64* bop, int bcast,
                          uint32_t batch, cudaStream_t st) {
  constexpr int DC = LOGN <= 12 ? 8 : 16, DE = 4;
  static_assert(clat_valid<LOGN, DC, DE>(), "default latency geometry");
  return clat_op_ce<LOGN, DC, DE>(p, op, out, in, bop, bcast, batch, st);
}

static bool clat_enabled() { return true; }

template <int LOGN>
static rnt_status cluster_op(const rnt_plan_s* p, int op, u64* out, const u64* in, const u64* bop, int bcast,
                             uint32_t batch, cudaStream_t st) {
  // k_clat up to 2^15; at 2^16 the 16-CTA cluster is throughput-bound with 4 coefficients per
  // thread (13.9 us vs 11.5 us for k_cluster's 16 per thread, CUDA-graph replay)
  if constexpr (LOGN <= 15) {
    if (clat_enabled()) return clat_op<LOGN>(p, op, out, in, bop, bcast, batch, st);
  }
  // cluster size: 8 CTAs up to 2^14, 16 above (measured, single-polynomial latency)
  if constexpr (LOGN <= 14) return cluster_op_c<LOGN, 8>(p, op, out, in, bop, bcast, batch, st);
  else return cluster_op_c<LOGN, 16>(p, op, out, in, bop, bcast, batch, st);
}

static rnt_status cluster_dispatch(const rnt_plan_s* p, int op, u64* out, const u64* in, const u64* bop, int bcast,
                                   uint32_t batch, cudaStream_t st) {
  switch (p->logn) {
    case 11: return cluster_op<11>(p, op, out, in, bop, bcast, batch, st);
    case 12: return cluster_op<12>(p, op, out, in, bop, bcast, batch, st);
    case 13: return cluster_op<13>(p, op, out, in, bop, bcast, batch, st);
    case 14: return cluster_op<14>(p, op, out, in, bop, bcast, batch, st);
    case 15: return cluster_op<15>(p, op, out, in, bop, bcast, batch, st);
    case 16: return cluster_op<16>(p, op, out, in, bop, bcast, batch, st);
    default: return RNT_E_UNSUPPORTED_N;
  }
}

static rnt_status large_dispatch(const rnt_plan_s* p, int op, u64* out, const u64* in, const u64* bop,
                                 int bcast, uint32_t batch, cudaStream_t st) {
  const uint64_t units = (uint64_t)batch * p->L;
  if (units == 0) return RNT_OK;
  if (units <= (uint64_t)cluster_units()) return cluster_dispatch(p, op, out, in, bop, bcast, batch, st);
  switch (p->logn) {
    case 11: return large_op<11>(p, op, out, in, bop, bcast, batch, st);
    case 12: return large_op<12>(p, op, out, in, bop, bcast, batch, st);
    case 13: return large_op<13>(p, op, out, in, bop, bcast, batch, st);
    case 14: return large_op<14>(p, op, out, in, bop, bcast, batch, st);
    case 15: return large_op<15>(p, op, out, in, bop, bcast, batch, st);
    case 16: return large_op<16>(p, op, out, in, bop, bcast, batch, st);
    default: return RNT_E_UNSUPPORTED_N;
  }
}

// ------------------------------------------------------------------- checks
static bool aligned16(const void* p) { return ((uintptr_t)p & 15u) == 0; }

static rnt_status check_plan_device(const rnt_plan_s* p) {
  int d = -1;
  cudaError_t e = cudaGetDevice(&d);
  if (e != cudaSuccess) return cuda_fail(e);
  return d == p->device ? RNT_OK : RNT_E_PLAN_MISMATCH;
}

static int num_sms();

static bool debug_checks() {
  static const bool on = env_int("RNT_DEBUG", 0) > 0;
  return on;
}

// Debug-only (RNT_DEBUG=1): validate that `batch` polynomials (or, with
// units_override, that many limb vectors) at x are canonical.  Synchronises st.
static rnt_status debug_validate(const rnt_plan_s* p, const void* x, uint64_t units, cudaStream_t st) {
  if (!debug_checks() || !units) return RNT_OK;
  int* bad = nullptr;
  RNT_CUDA(cudaMallocAsync(&bad, sizeof(int), st));
  RNT_CUDA(cudaMemsetAsync(bad, 0, sizeof(int), st));
  const uint64_t total = units << p->logn;
  uint64_t blocks = (total + 255) / 256;
  const uint64_t cap = (uint64_t)num_sms() * 8;
  if (blocks > cap) blocks = cap;
  k_check_range<<<(unsigned)blocks, 256, 0, st>>>(reinterpret_cast<const u64*>(x), p->d_lc, p->L, p->logn, total, bad);
  int h = 0;
  RNT_CUDA(cudaGetLastError());
  RNT_CUDA(cudaMemcpyAsync(&h, bad, sizeof(int), cudaMemcpyDeviceToHost, st));
  RNT_CUDA(cudaFreeAsync(bad, st));
  RNT_CUDA(cudaStreamSynchronize(st));
  return h ? RNT_E_INVALID_ARG : RNT_OK;
}

static rnt_status check_data(const rnt_plan_s* p, const void* a, const void* b, uint32_t batch) {
  if (!p) return RNT_E_INVALID_ARG;
  if (batch == 0) return RNT_OK;
  if (!a || !b || !aligned16(a) || !aligned16(b)) return RNT_E_INVALID_ARG;
  const unsigned __int128 bytes = (unsigned __int128)batch * p->L * (1ull << p->logn) * 8u;
  if (bytes >> 62) return RNT_E_INVALID_ARG;
  return check_plan_device(p);
}

// --------------------------------------------------------------------- ABI
struct rnt_bconv_s {
  int device = 0;
  uint32_t logn = 0, L = 0, K = 0;
  BcMod* d_src = nullptr;
  BcMod* d_dst = nullptr;
  TW* d_qhat_p = nullptr;   // [K][L]: Shoup pair of (Q/q_i mod p_j) w.r.t. p_j
};

template <int LOGN, int LV, int KM, bool LZ>
static rnt_status launch_extprod_cta_v(const rnt_plan_s* p, u64* out, const u64* c, const u64* z, uint32_t n_slot,
                                       DigitSpec ds, cudaStream_t st) {
  static std::atomic<uint64_t> attr{0};
  const size_t smem = (size_t)2 * LV * kWarpBuf * 8;
  if (rnt_status s = ensure_attr(k_extprod_cta<LOGN, LV, KM, LZ>, smem, attr); s != RNT_OK) return s;
  const uint64_t per_cta = kWarpElems >> LOGN;
  const uint64_t grid = (n_slot + per_cta - 1) / per_cta;
  k_extprod_cta<LOGN, LV, KM, LZ><<<(unsigned)grid, 64 * LV, smem, st>>>(out, c, z, p->d_fwd, p->d_inv, p->d_lc,
                                                                          n_slot, ds);
  return after_launch();
}

// LZ kernels (split-tail schedule) when the modulus is below 2^60
template <int LOGN, int LV>
static rnt_status launch_extprod_cta(const rnt_plan_s* p, u64* out, const u64* c, const u64* z, uint32_t n_slot,
                                     DigitSpec ds, cudaStream_t st) {
  if (p->lazy60 && lazy_enabled()) return launch_extprod_cta_v<LOGN, LV, 32, true>(p, out, c, z, n_slot, ds, st);
  return launch_extprod_cta_v<LOGN, LV, 3, false>(p, out, c, z, n_slot, ds, st);
}

// N = 2^10 (the TFHE size): the CTA-parallel kernel, one warp per decomposed
// polynomial (l = 3: 1024 / 4096 / 16384 slots 0.127 / 0.411 / 1.55 ms vs 0.209 /
// 0.537 / 1.73 ms for the single-warp kernel); smaller N: the single-warp k_extprod.
template <int LOGN>
static rnt_status launch_extprod(const rnt_plan_s* p, u64* out, const u64* c, const u64* z, uint32_t n_slot,
                                 DigitSpec ds, cudaStream_t st) {
  if constexpr (LOGN == 10) {
    switch (ds.levels) {
      case 1: return launch_extprod_cta<LOGN, 1>(p, out, c, z, n_slot, ds, st);
      case 2: return launch_extprod_cta<LOGN, 2>(p, out, c, z, n_slot, ds, st);
      case 3: return launch_extprod_cta<LOGN, 3>(p, out, c, z, n_slot, ds, st);
      case 4: return launch_extprod_cta<LOGN, 4>(p, out, c, z, n_slot, ds, st);
      case 5: return launch_extprod_cta<LOGN, 5>(p, out, c, z, n_slot, ds, st);
      case 6: return launch_extprod_cta<LOGN, 6>(p, out, c, z, n_slot, ds, st);
      case 7: return launch_extprod_cta<LOGN, 7>(p, out, c, z, n_slot, ds, st);
      case 8: return launch_extprod_cta<LOGN, 8>(p, out, c, z, n_slot, ds, st);
      default: return RNT_E_INVALID_ARG;
    }
  } else {
    static std::atomic<uint64_t> attr{0};
    const size_t smem = (size_t)2 * kWarpBuf * 8;
    if (rnt_status s = ensure_attr(k_extprod<LOGN>, smem, attr); s != RNT_OK) return s;
    const uint64_t per_cta = 2ull * (kWarpElems >> LOGN);
    const uint64_t grid = (n_slot + per_cta - 1) / per_cta;
    k_extprod<LOGN><<<(unsigned)grid, 64, smem, st>>>(out, c, z, p->d_fwd, p->d_inv, p->d_lc, n_slot, ds);
    return after_launch();
  }
}

// BConv tables from basis {q_i} (L) to {p_j} (K) (reading G3):
// src[i].qhatinv = (Q/q_i)^{-1} mod q_i, qp[j][i] = Q/q_i mod p_j, Shoup pairs.
static void bconv_tables(const uint64_t* q, uint32_t L, const uint64_t* p, uint32_t K, std::vector<BcMod>& src,
                         std::vector<BcMod>& dst, std::vector<TW>& qp) {
  src.assign(L, BcMod{});
  dst.assign(K, BcMod{});
  qp.assign((size_t)K * L, TW{0, 0});
  for (uint32_t i = 0; i < L; ++i) {
    uint64_t h = 1 % q[i];
    for (uint32_t k = 0; k < L; ++k)
      if (k != i) h = hp_mulmod(h, q[k] % q[i], q[i]);
    const uint64_t hinv = hp_powmod(h, q[i] - 2, q[i]);
    src[i].m = q[i];
    src[i].m2 = 2 * q[i];
    src[i].qhatinv = TW{hinv, (uint64_t)(((unsigned __int128)hinv << 64) / q[i])};
  }
  for (uint32_t j = 0; j < K; ++j) {
    dst[j].m = p[j];
    dst[j].m2 = 2 * p[j];
    dst[j].qhatinv = TW{0, 0};
    for (uint32_t i = 0; i < L; ++i) {
      uint64_t h = 1 % p[j];
      for (uint32_t k = 0; k < L; ++k)
        if (k != i) h = hp_mulmod(h, q[k] % p[j], p[j]);
      qp[(size_t)j * L + i] = TW{h, (uint64_t)(((unsigned __int128)h << 64) / p[j])};
    }
  }
}

// Fused ModUp -> NTT -> key product for one-prime digits (keyswitch.cuh):
// column pass with the lift on load (k_col_fwd<.., MODUP>), then the row pass
// with the key multiply-accumulate (k_row_mac).  E: [dnum][LK][N] scratch.
// Digit split of the fused key product (k_row_mac blockIdx.z): dnum digits in
// `split` partial sums, added by k_ks_sum (round 1: 2..5 measured no faster; experiment
// builds: -DRNT_KS_SPLIT=n).
#ifndef RNT_KS_SPLIT
#define RNT_KS_SPLIT 1
#endif
static uint32_t ks_split(uint32_t dnum) { return dnum < RNT_KS_SPLIT ? dnum : RNT_KS_SPLIT; }

template <int LOGN, bool LZ>
static rnt_status ks_fused_launch_v(const rnt_plan_s* qp, u64* u, u64* E, const u64* x, const u64* evk,
                                    uint32_t dnum, uint32_t split, cudaStream_t st) {
  using P = TwoPass<LOGN>;
  const uint32_t LK = qp->L;
  const uint64_t units = (uint64_t)dnum * LK;
  for (uint64_t y0 = 0; y0 < units; y0 += 65535u) {
    const uint64_t cnt = units - y0 < 65535u ? units - y0 : 65535u;
    dim3 g(P::Cn / kColTile, (unsigned)cnt);
    k_col_fwd<LOGN, kColTile, true, LZ><<<g, kColTile * P::T1, 0, st>>>(E, x, qp->d_col_fwd, qp->d_lc, LK, dnum, y0);
    rnt_status s = after_launch();
    if (s != RNT_OK) return s;
  }
  constexpr int RPC = P::RPC;
  const size_t smem = (size_t)2 * RPC * P::Cn * 8;
  static std::atomic<uint64_t> attr{0};
  if (rnt_status s = ensure_attr(k_row_mac<LOGN, RPC, LZ>, smem, attr); s != RNT_OK) return s;
  dim3 g(P::R / RPC, LK, split);
  k_row_mac<LOGN, RPC, LZ><<<g, RPC * P::T2, smem, st>>>(u, E, evk, qp->d_fwd, qp->d_lc, LK, dnum, split);
  return after_launch();
}

// lazy CT ranges (LZ) when every prime of Q u P is below 2^60 (the lifted
// column input is canonical, the Montgomery key product accepts [0, 16q))
template <int LOGN>
static rnt_status ks_fused_launch(const rnt_plan_s* qp, u64* u, u64* E, const u64* x, const u64* evk, uint32_t dnum,
                                  uint32_t split, const KsMod* km, cudaStream_t st) {
  rnt_status s = (qp->lazy60 && lazy_enabled()) ? ks_fused_launch_v<LOGN, true>(qp, u, E, x, evk, dnum, split, st)
                                                : ks_fused_launch_v<LOGN, false>(qp, u, E, x, evk, dnum, split, st);
  if (s != RNT_OK || split == 1) return s;
  const uint32_t LK = qp->L;
  const uint64_t total = 2ull * LK << LOGN;
  uint64_t blocks = (total + 255) / 256;
  const uint64_t cap = (uint64_t)num_sms() * 8;
  if (blocks > cap) blocks = cap;
  k_ks_sum<<<(unsigned)blocks, 256, 0, st>>>(u, split, km, LK, LOGN);
  return after_launch();
}

static rnt_status ks_fused(const rnt_plan_s* qp, u64* u, u64* E, const u64* x, const u64* evk, uint32_t dnum,
                           uint32_t split, const KsMod* km, cudaStream_t st) {
  switch (qp->logn) {
    case 11: return ks_fused_launch<11>(qp, u, E, x, evk, dnum, split, km, st);
    case 12: return ks_fused_launch<12>(qp, u, E, x, evk, dnum, split, km, st);
    case 13: return ks_fused_launch<13>(qp, u, E, x, evk, dnum, split, km, st);
    case 14: return ks_fused_launch<14>(qp, u, E, x, evk, dnum, split, km, st);
    case 15: return ks_fused_launch<15>(qp, u, E, x, evk, dnum, split, km, st);
    case 16: return ks_fused_launch<16>(qp, u, E, x, evk, dnum, split, km, st);
    default: return RNT_E_UNSUPPORTED_N;
  }
}

static inline uint64_t* U(u64* p) { return reinterpret_cast<uint64_t*>(p); }
static inline const uint64_t* U(const u64* p) { return reinterpret_cast<const uint64_t*>(p); }

struct rnt_keyswitch_s {
  int device = 0;
  uint32_t logn = 0, L = 0, K = 0, LK = 0, dnum = 0, alpha = 0;
  rnt_plan_s* qp = nullptr;  // borrowed: extended-basis plan (Q then P)
  rnt_plan_s* q = nullptr;   // borrowed: Q plan
  KsMod* d_km = nullptr;     // [LK]
  TW* d_tab = nullptr;       // [dnum][LK][alpha]
  BcMod* d_bsrc = nullptr;   // ModDown BConv P -> Q
  BcMod* d_bdst = nullptr;
  TW* d_bqp = nullptr;
  u64* d_ws = nullptr;       // x [L][N] | E [dnum][LK][N] | u [2][LK][N] | uP [2][K][N] | w [2][L][N]
  uint32_t split = 1;        // digit split of the fused key product (u region holds `split` partial sums)
  bool fused = false;        // N >= 2^11, one-prime digits: ModUp in the column pass, key product in the row pass
  std::mutex mu;             // one apply at a time per handle (the workspace is shared)
};

extern "C" {

const char* rnt_status_string(rnt_status s) {
  switch (s) {
    case RNT_OK: return "RNT_OK";
    case RNT_E_INVALID_ARG: return "RNT_E_INVALID_ARG: invalid argument";
    case RNT_E_UNSUPPORTED_N: return "RNT_E_UNSUPPORTED_N: log2n outside [4, 16]";
    case RNT_E_MODULUS: return "RNT_E_MODULUS: modulus not prime, not 1 mod 2N, >= 2^62, or duplicated";
    case RNT_E_ROOT: return "RNT_E_ROOT: psi is not a primitive 2N-th root of unity";
    case RNT_E_PLAN_MISMATCH: return "RNT_E_PLAN_MISMATCH: current device differs from the plan's";
    case RNT_E_CUDA: return "RNT_E_CUDA: CUDA runtime error";
    case RNT_E_OOM: return "RNT_E_OOM: out of memory";
  }
  return "unknown rnt_status";
}

int rnt_last_cuda_error(void) { return g_last_cuda; }

uint64_t rnt_launch_count(void) { return g_launches.load(); }

rnt_status rnt_plan_create(rnt_plan* out, uint32_t log2n, uint32_t n_limbs, const uint64_t* moduli,
                           const uint64_t* psi, int device) {
  if (!out || !moduli || n_limbs == 0 || n_limbs > RNT_MAX_LIMBS) return RNT_E_INVALID_ARG;
  *out = nullptr;
  if (log2n < RNT_MIN_LOG2N || log2n > RNT_MAX_LOG2N) return RNT_E_UNSUPPORTED_N;
  std::vector<HostLimb> limbs;
  int pe = plan_limbs(log2n, n_limbs, moduli, psi, limbs);
  if (pe == PLAN_E_MODULUS) return RNT_E_MODULUS;
  if (pe == PLAN_E_ROOT) return RNT_E_ROOT;
  if (pe != PLAN_OK) return RNT_E_INVALID_ARG;

  int ndev = 0;
  cudaError_t ce = cudaGetDeviceCount(&ndev);
  if (ce != cudaSuccess) return cuda_fail(ce);
  if (device < 0 || device >= ndev) return RNT_E_INVALID_ARG;
  int prev = 0;
  RNT_CUDA(cudaGetDevice(&prev));
  RNT_CUDA(cudaSetDevice(device));

  rnt_plan_s* p = new (std::nothrow) rnt_plan_s;
  if (!p) {
    cudaSetDevice(prev);   // leave the caller's current device as it was
    return RNT_E_OOM;
  }
  p->logn = log2n;
  p->L = n_limbs;
  p->device = device;
  p->limbs = limbs;
  const uint32_t n = 1u << log2n;
  const uint32_t n1 = (log2n + 1) / 2;
  const bool large = log2n > 10;

  // The coefficient-form polymul (op 3) takes its NTT(b) temporary from the device's
  // default stream-ordered pool (cudaMallocAsync); keep freed blocks in the pool instead
  // of returning them to the driver at every synchronisation, so repeated calls reuse
  // one allocation (the pool is per device; PyTorch's caching allocator does not use it).
  {
    cudaMemPool_t pool;
    if (cudaDeviceGetDefaultMemPool(&pool, device) == cudaSuccess) {
      uint64_t keep = UINT64_MAX;
      cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &keep);
    }
  }
  p->lazy60 = true;
  for (uint32_t l = 0; l < n_limbs; ++l) p->lazy60 = p->lazy60 && limbs[l].q < (1ull << 60);
  std::vector<LimbC> lc(n_limbs);
  for (uint32_t l = 0; l < n_limbs; ++l) {
    const HostLimb& h = limbs[l];
    lc[l].q = h.q;
    lc[l].q2 = h.q2;
    lc[l].qinv = h.qinv;
    lc[l].r2 = h.r2;
    lc[l].ninv = TW{h.ninv.w, h.ninv.wp};
    lc[l].ninv_w1 = TW{h.ninv_w1.w, h.ninv_w1.wp};
    lc[l].ninvR = TW{h.ninvR.w, h.ninvR.wp};
    lc[l].ninvR_w1 = TW{h.ninvR_w1.w, h.ninvR_w1.wp};
  }
  // large N: the inverse row stages mirror the forward row table (ntt_large.cuh),
  // so only the small column table is kept per direction.
  std::vector<HostTW> nat(n), lay((size_t)n_limbs * n), layi(large ? 0 : (size_t)n_limbs * n);
  std::vector<HostTW> col, coli, rowtw;
  // column / per-row tables: the two-pass kernels (N >= 2^11) and the cluster
  // latency kernel k_clat (N >= 2^10)
  const bool ctabs = log2n >= 10;
  if (ctabs) {
    rowtw.resize((size_t)n_limbs * n);
    col.resize((size_t)n_limbs << n1);
    coli.resize((size_t)n_limbs << n1);
  }
  for (uint32_t l = 0; l < n_limbs; ++l) {
    for (int dir = 0; dir < 2; ++dir) {
      plan_powers(limbs[l], log2n, dir == 1, n, nat.data());
      if (ctabs) {
        if (dir == 0) plan_row_natural(nat.data(), log2n, rowtw.data() + (size_t)l * n);
        std::memcpy((dir ? coli.data() : col.data()) + ((size_t)l << n1), nat.data(), sizeof(HostTW) << n1);
      }
      if (large) {
        if (dir == 0) plan_row_layout(nat.data(), log2n, lay.data() + (size_t)l * n);
      } else {
        HostTW* dst = (dir ? layi.data() : lay.data()) + (size_t)l * n;
        std::memcpy(dst, nat.data(), sizeof(HostTW) * n);  // natural order (ntt_small.cuh)
      }
    }
  }
  auto fail = [&](cudaError_t e) {
    rnt_plan_destroy(p);
    cudaSetDevice(prev);
    return cuda_fail(e);
  };
  cudaError_t e;
  if ((e = cudaMalloc(&p->d_lc, sizeof(LimbC) * n_limbs)) != cudaSuccess) return fail(e);
  if ((e = cudaMalloc(&p->d_fwd, sizeof(TW) * lay.size())) != cudaSuccess) return fail(e);
  if (!large && (e = cudaMalloc(&p->d_inv, sizeof(TW) * layi.size())) != cudaSuccess) return fail(e);
  if ((e = cudaMemcpy(p->d_lc, lc.data(), sizeof(LimbC) * n_limbs, cudaMemcpyHostToDevice)) != cudaSuccess) return fail(e);
  if ((e = cudaMemcpy(p->d_fwd, lay.data(), sizeof(TW) * lay.size(), cudaMemcpyHostToDevice)) != cudaSuccess) return fail(e);
  if (!large && (e = cudaMemcpy(p->d_inv, layi.data(), sizeof(TW) * layi.size(), cudaMemcpyHostToDevice)) != cudaSuccess)
    return fail(e);
  if (ctabs) {
    if ((e = cudaMalloc(&p->d_col_fwd, sizeof(TW) * col.size())) != cudaSuccess) return fail(e);
    if ((e = cudaMalloc(&p->d_col_inv, sizeof(TW) * coli.size())) != cudaSuccess) return fail(e);
    if ((e = cudaMemcpy(p->d_col_fwd, col.data(), sizeof(TW) * col.size(), cudaMemcpyHostToDevice)) != cudaSuccess) return fail(e);
    if ((e = cudaMemcpy(p->d_col_inv, coli.data(), sizeof(TW) * coli.size(), cudaMemcpyHostToDevice)) != cudaSuccess) return fail(e);
    if ((e = cudaMalloc(&p->d_rowtw, sizeof(TW) * rowtw.size())) != cudaSuccess) return fail(e);
    if ((e = cudaMemcpy(p->d_rowtw, rowtw.data(), sizeof(TW) * rowtw.size(), cudaMemcpyHostToDevice)) != cudaSuccess) return fail(e);
  }
  cudaSetDevice(prev);
  *out = p;
  return RNT_OK;
}

rnt_status rnt_plan_destroy(rnt_plan p) {
  if (!p) return RNT_OK;
  int prev = 0;
  cudaGetDevice(&prev);
  cudaSetDevice(p->device);
  cudaFree(p->d_lc);
  cudaFree(p->d_fwd);
  cudaFree(p->d_inv);
  cudaFree(p->d_col_fwd);
  cudaFree(p->d_col_inv);
  cudaFree(p->d_rowtw);
  for (auto& a : p->aux)
    if (a) cudaStreamDestroy(a);
  for (auto e : p->ev_pool) cudaEventDestroy(e);
  for (auto& a : p->split)
    if (a) cudaStreamDestroy(a);
  for (auto& e : p->split_ev)
    if (e) cudaEventDestroy(e);
  cudaSetDevice(prev);
  delete p;
  return RNT_OK;
}

rnt_status rnt_plan_query(rnt_plan p, uint32_t* log2n, uint32_t* n_limbs, uint64_t* psi_out, int* device) {
  if (!p) return RNT_E_INVALID_ARG;
  if (log2n) *log2n = p->logn;
  if (n_limbs) *n_limbs = p->L;
  if (device) *device = p->device;
  if (psi_out)
    for (uint32_t l = 0; l < p->L; ++l) psi_out[l] = p->limbs[l].psi;
  return RNT_OK;
}

// N >= 2^11: op 3 computes NTT(b) into a stream-ordered temporary, then runs
// the fused eval-form path; ops 0..2 go straight to the kernel chain.
static rnt_status run_large(const rnt_plan_s* p, int op, u64* out, const u64* in, const u64* b, int bcast,
                            uint32_t batch, cudaStream_t st) {
  if (op == 3) {
    const uint64_t bunits = (uint64_t)(bcast ? 1u : batch) * p->L;
    const size_t bytes = (size_t)bunits << (p->logn + 3);
    u64* tmp = nullptr;
    RNT_CUDA(cudaMallocAsync(&tmp, bytes, st));
    rnt_status s = large_dispatch(p, 0, tmp, b, nullptr, 0, bcast ? 1u : batch, st);
    if (s == RNT_OK) s = large_dispatch(p, 2, out, in, tmp, bcast, batch, st);
    cudaError_t e = cudaFreeAsync(tmp, st);
    if (s == RNT_OK && e != cudaSuccess) return cuda_fail(e);
    return s;
  }
  return large_dispatch(p, op, out, in, b, bcast, batch, st);
}

static rnt_status run_op(rnt_plan p, int op, uint64_t* out_, const uint64_t* in_, const uint64_t* b_, int bcast,
                         uint32_t batch, cudaStream_t st) {
  u64* out = reinterpret_cast<u64*>(out_);
  const u64* in = reinterpret_cast<const u64*>(in_);
  const u64* b = reinterpret_cast<const u64*>(b_);
  if (p->logn <= 10) {
    switch (op) {
      case 0: return warp_dispatch<0>(p, out, in, nullptr, 0, batch, st);
      case 1: return warp_dispatch<1>(p, out, in, nullptr, 0, batch, st);
      case 2: return warp_dispatch<2>(p, out, in, b, bcast, batch, st);
      case 3: return warp_dispatch<3>(p, out, in, b, bcast, batch, st);
    }
    return RNT_E_INVALID_ARG;
  }
  // A single polynomial with many limbs (cfg3) launches few CTAs per kernel and
  // pays each kernel's ramp and tail three times; running G limb windows as
  // independent kernel chains on G streams lets the windows overlap
  // (measured: 2^16 x 45 limbs polymul 0.103 -> 0.094 ms with G = 2; 3 and 4 no
  // better).  The window streams belong to the plan, so concurrent callers of one
  // plan serialise on them; a stream under CUDA-graph capture skips the split (the
  // plan's streams must not join another thread's capture).
#ifdef RNT_EXPERIMENTS
  static const int split_g = std::min(4, std::max(1, env_int("RNT_SPLIT_G", 2)));   // limb windows
#else
  constexpr int split_g = 2;
#endif
  cudaStreamCaptureStatus cap = cudaStreamCaptureStatusNone;
  RNT_CUDA(cudaStreamIsCapturing(st, &cap));
  if (cap == cudaStreamCaptureStatusNone && batch == 1 && p->L >= (uint32_t)(2 * split_g) && !p->is_view) {
    std::lock_guard<std::mutex> g(p->split_mu);
    for (int i = 0; i < split_g; ++i)
      if (!p->split[i]) RNT_CUDA(cudaStreamCreateWithFlags(&p->split[i], cudaStreamNonBlocking));
    for (int i = 0; i <= split_g; ++i)
      if (!p->split_ev[i]) RNT_CUDA(cudaEventCreateWithFlags(&p->split_ev[i], cudaEventDisableTiming));
    RNT_CUDA(cudaEventRecord(p->split_ev[split_g], st));
    const size_t n = (size_t)1 << p->logn;
    const uint32_t per = (p->L + split_g - 1) / split_g;
    rnt_status s = RNT_OK;
    for (int gi = 0; gi < split_g; ++gi) {
      const uint32_t l0 = gi * per;
      if (l0 >= p->L) break;   // fewer windows than streams (e.g. L = 9, G = 4)
      const uint32_t nl = p->L - l0 < per ? p->L - l0 : per;
      rnt_plan_s view;
      make_view(p, l0, nl, &view);
      RNT_CUDA(cudaStreamWaitEvent(p->split[gi], p->split_ev[split_g], 0));
      if (s == RNT_OK)
        s = run_large(&view, op, out + l0 * n, in + l0 * n, b ? b + l0 * n : nullptr, bcast, 1, p->split[gi]);
      // Always join, so `st` never runs ahead of work already queued.
      RNT_CUDA(cudaEventRecord(p->split_ev[gi], p->split[gi]));
      RNT_CUDA(cudaStreamWaitEvent(st, p->split_ev[gi], 0));
    }
    return s;
  }
  return run_large(p, op, out, in, b, bcast, batch, st);
}

rnt_status rnt_ntt_forward(rnt_plan p, uint64_t* out, const uint64_t* in, uint32_t batch, void* stream) {
  rnt_status s = check_data(p, out, in, batch);
  if (s != RNT_OK || batch == 0) return s;
  if ((s = debug_validate(p, in, (uint64_t)batch * p->L, (cudaStream_t)stream)) != RNT_OK) return s;
  return run_op(p, 0, out, in, nullptr, 0, batch, (cudaStream_t)stream);
}

rnt_status rnt_ntt_inverse(rnt_plan p, uint64_t* out, const uint64_t* in, uint32_t batch, void* stream) {
  rnt_status s = check_data(p, out, in, batch);
  if (s != RNT_OK || batch == 0) return s;
  if ((s = debug_validate(p, in, (uint64_t)batch * p->L, (cudaStream_t)stream)) != RNT_OK) return s;
  return run_op(p, 1, out, in, nullptr, 0, batch, (cudaStream_t)stream);
}

rnt_status rnt_pointwise_mul(rnt_plan p, uint64_t* c, const uint64_t* a_hat, const uint64_t* b_hat, uint32_t batch,
                             int b_broadcast, void* stream) {
  rnt_status s = check_data(p, c, a_hat, batch);
  if (s != RNT_OK || batch == 0) return s;
  if (!b_hat || !aligned16(b_hat)) return RNT_E_INVALID_ARG;
  if ((s = debug_validate(p, a_hat, (uint64_t)batch * p->L, (cudaStream_t)stream)) != RNT_OK ||
      (s = debug_validate(p, b_hat, (uint64_t)(b_broadcast ? 1u : batch) * p->L, (cudaStream_t)stream)) != RNT_OK)
    return s;
  const uint64_t total2 = ((uint64_t)batch * p->L << p->logn) / 2;
  const int threads = 256;
  uint64_t blocks = (total2 + threads - 1) / threads;
  const uint64_t cap = (uint64_t)num_sms() * 16;
  if (blocks > cap) blocks = cap;
  k_pointwise<<<(unsigned)blocks, threads, 0, (cudaStream_t)stream>>>(
      reinterpret_cast<u64*>(c), reinterpret_cast<const u64*>(a_hat), reinterpret_cast<const u64*>(b_hat), b_broadcast ? 1 : 0, p->d_lc,
                                                                      p->L, p->logn, total2);
  return after_launch();
}

rnt_status rnt_automorph(rnt_plan p, uint64_t* out, const uint64_t* in, uint32_t batch, uint32_t galois_elt,
                         int ntt_domain, void* stream) {
  rnt_status s = check_data(p, out, in, batch);
  if (s != RNT_OK || batch == 0) return s;
  const uint32_t two_n = 2u << p->logn;
  if (out == in || (galois_elt & 1u) == 0 || galois_elt >= two_n) return RNT_E_INVALID_ARG;
  if ((s = debug_validate(p, in, (uint64_t)batch * p->L, (cudaStream_t)stream)) != RNT_OK) return s;
  uint32_t ginv = 1;  // g^{-1} mod 2N: g^(N/2 - 1), the group (Z/2N)^* has exponent N/2 (N >= 4)
  {
    uint64_t b = galois_elt, e = (two_n / 4) - 1, r = 1;
    for (; e; e >>= 1, b = b * b % two_n)
      if (e & 1) r = r * b % two_n;
    ginv = (uint32_t)r;
  }
  const uint64_t total = (uint64_t)batch * p->L << p->logn;
  const int threads = 256;
  uint64_t blocks = (total + threads - 1) / threads;
  const uint64_t cap = (uint64_t)num_sms() * 16;
  if (blocks > cap) blocks = cap;
  k_automorph<<<(unsigned)blocks, threads, 0, (cudaStream_t)stream>>>(
      reinterpret_cast<u64*>(out), reinterpret_cast<const u64*>(in), p->d_lc, p->L, p->logn, galois_elt, ginv,
      ntt_domain ? 1 : 0, total);
  return after_launch();
}

// HRF-MatVec (f4): one launch of k_hrf_matvec (hrf.cuh), a grid-stride loop
// over the L N / 2 slot pairs, enough CTAs for every SM.  Experiments rebuild with
// RNT_NVCC_EXTRA=-DRNT_HRF_UNROLL=n / -DRNT_HRF_JS=n / -DRNT_HRF_CTAS_PER_SM=n (build.py).
// Measured (N = 2^16, 4 limbs; fraction of HBM at n_slot 64 / 256 / 1024,
// profiles/r02/hrf): unroll 4, JS 1: 0.51 / 0.57 / 0.59 (31 % warps active, long-scoreboard
// bound); unroll 2, JS 2: 0.71 / 0.86 / 0.90; unroll 1, JS 4: 0.71 / 0.90 / 0.96;
// unroll 2, JS 1, min 4 CTAs/SM (<= 64 registers): 0.79 / 0.92 / 0.95 -- shipped.
#ifndef RNT_HRF_UNROLL
#define RNT_HRF_UNROLL 2
#endif
#ifndef RNT_HRF_JS
#define RNT_HRF_JS 1
#endif
#ifndef RNT_HRF_CTAS_PER_SM
#define RNT_HRF_CTAS_PER_SM 8
#endif
rnt_status rnt_hrf_matvec(rnt_plan p, uint64_t* out, const uint64_t* pt, const uint64_t* ct, uint32_t n_slot,
                          const uint64_t* add, void* stream) {
  if (!p || !out || !aligned16(out) || (add && !aligned16(add))) return RNT_E_INVALID_ARG;
  const uint64_t ln = (uint64_t)p->L << p->logn;
  if (n_slot) {
    if (!pt || !ct || !aligned16(pt) || !aligned16(ct)) return RNT_E_INVALID_ARG;
    const unsigned __int128 bytes = (unsigned __int128)n_slot * 3u * ln * 8u;
    if (bytes >> 62) return RNT_E_INVALID_ARG;
    auto overlap = [](const void* a, uint64_t na, const void* b, uint64_t nb) {
      const uintptr_t x = (uintptr_t)a, y = (uintptr_t)b;
      return x < y + nb && y < x + na;
    };
    const uint64_t ob = 2 * ln * 8;
    if (overlap(out, ob, pt, (uint64_t)n_slot * ln * 8) || overlap(out, ob, ct, (uint64_t)n_slot * 2 * ln * 8))
      return RNT_E_INVALID_ARG;
  }
  rnt_status s = check_plan_device(p);
  if (s != RNT_OK) return s;
  const cudaStream_t st = (cudaStream_t)stream;
  if (n_slot) {
    if ((s = debug_validate(p, pt, n_slot, st)) != RNT_OK) return s;
    if ((s = debug_validate(p, ct, 2ull * n_slot, st)) != RNT_OK) return s;
  }
  if (add && (s = debug_validate(p, add, 2, st)) != RNT_OK) return s;
  const uint64_t nvec = ln / 2;
  constexpr int vb = 256 / RNT_HRF_JS;   // slot pairs per CTA
  uint64_t blocks = (nvec + vb - 1) / vb;
  const uint64_t cap = (uint64_t)num_sms() * RNT_HRF_CTAS_PER_SM;
  if (blocks > cap) blocks = cap;
  k_hrf_matvec<RNT_HRF_UNROLL, RNT_HRF_JS><<<(unsigned)blocks, 256, 0, st>>>(reinterpret_cast<u64*>(out), reinterpret_cast<const u64*>(pt),
                                                        reinterpret_cast<const u64*>(ct), reinterpret_cast<const u64*>(add),
                                                        p->d_lc, n_slot, p->L, p->logn, nvec);
  return after_launch();
}

rnt_status rnt_bconv_create(rnt_bconv* out, rnt_plan from, rnt_plan to) {
  if (!out || !from || !to) return RNT_E_INVALID_ARG;
  *out = nullptr;
  if (from->logn != to->logn || from->device != to->device || from->L > 192) return RNT_E_INVALID_ARG;
  rnt_status s = check_plan_device(from);
  if (s != RNT_OK) return s;
  const uint32_t L = from->L, K = to->L;
  std::vector<uint64_t> fq(L), tq(K);
  for (uint32_t i = 0; i < L; ++i) fq[i] = from->limbs[i].q;
  for (uint32_t j = 0; j < K; ++j) tq[j] = to->limbs[j].q;
  std::vector<BcMod> src, dst;
  std::vector<TW> qp;
  bconv_tables(fq.data(), L, tq.data(), K, src, dst, qp);
  rnt_bconv_s* c = new (std::nothrow) rnt_bconv_s;
  if (!c) return RNT_E_OOM;
  c->device = from->device;
  c->logn = from->logn;
  c->L = L;
  c->K = K;
  cudaError_t e;
  if ((e = cudaMalloc(&c->d_src, sizeof(BcMod) * L)) != cudaSuccess ||
      (e = cudaMalloc(&c->d_dst, sizeof(BcMod) * K)) != cudaSuccess ||
      (e = cudaMalloc(&c->d_qhat_p, sizeof(TW) * qp.size())) != cudaSuccess ||
      (e = cudaMemcpy(c->d_src, src.data(), sizeof(BcMod) * L, cudaMemcpyHostToDevice)) != cudaSuccess ||
      (e = cudaMemcpy(c->d_dst, dst.data(), sizeof(BcMod) * K, cudaMemcpyHostToDevice)) != cudaSuccess ||
      (e = cudaMemcpy(c->d_qhat_p, qp.data(), sizeof(TW) * qp.size(), cudaMemcpyHostToDevice)) != cudaSuccess) {
    rnt_bconv_destroy(c);
    return cuda_fail(e);
  }
  *out = c;
  return RNT_OK;
}

rnt_status rnt_bconv_destroy(rnt_bconv c) {
  if (!c) return RNT_OK;
  cudaFree(c->d_src);
  cudaFree(c->d_dst);
  cudaFree(c->d_qhat_p);
  delete c;
  return RNT_OK;
}

rnt_status rnt_bconv_apply(rnt_bconv c, uint64_t* out, const uint64_t* in, uint32_t batch, void* stream) {
  if (!c) return RNT_E_INVALID_ARG;
  if (batch == 0) return RNT_OK;
  if (!out || !in || out == in || !aligned16(out) || !aligned16(in)) return RNT_E_INVALID_ARG;
  int d = -1;
  cudaError_t e = cudaGetDevice(&d);
  if (e != cudaSuccess) return cuda_fail(e);
  if (d != c->device) return RNT_E_PLAN_MISMATCH;
  const size_t smem = (size_t)c->L * kBcTile * 8;
  if (rnt_status s = set_smem(k_bconv, smem); s != RNT_OK) return s;
  const uint32_t n = 1u << c->logn;
  // grid.y carries the polynomial: chunks of at most 65535 polynomials per launch
  for (uint32_t b0 = 0; b0 < batch; b0 += 65535u) {
    const uint32_t nb = batch - b0 < 65535u ? batch - b0 : 65535u;
    dim3 grid((n + kBcTile - 1) / kBcTile, nb);
    k_bconv<<<grid, kBcTile, smem, (cudaStream_t)stream>>>(
        reinterpret_cast<u64*>(out) + (size_t)b0 * c->K * n, reinterpret_cast<const u64*>(in) + (size_t)b0 * c->L * n,
        c->d_src, c->d_dst, c->d_qhat_p, c->L, c->K, c->logn);
    if (rnt_status st = after_launch(); st != RNT_OK) return st;
  }
  return RNT_OK;
}

rnt_status rnt_keyswitch_destroy(rnt_keyswitch ks) {
  if (!ks) return RNT_OK;
  cudaFree(ks->d_km);
  cudaFree(ks->d_tab);
  cudaFree(ks->d_bsrc);
  cudaFree(ks->d_bdst);
  cudaFree(ks->d_bqp);
  cudaFree(ks->d_ws);
  delete ks;
  return RNT_OK;
}

rnt_status rnt_keyswitch_create(rnt_keyswitch* out, rnt_plan q_plan, rnt_plan qp_plan, uint32_t dnum) {
  if (!out || !q_plan || !qp_plan) return RNT_E_INVALID_ARG;
  *out = nullptr;
  if (q_plan->is_view || qp_plan->is_view) return RNT_E_INVALID_ARG;
  const uint32_t L = q_plan->L, LK = qp_plan->L;
  if (q_plan->logn != qp_plan->logn || q_plan->device != qp_plan->device || LK <= L || LK - L > 192)
    return RNT_E_INVALID_ARG;
  for (uint32_t i = 0; i < L; ++i)
    if (q_plan->limbs[i].q != qp_plan->limbs[i].q || q_plan->limbs[i].psi != qp_plan->limbs[i].psi)
      return RNT_E_INVALID_ARG;
  if (dnum == 0 || dnum > L) return RNT_E_INVALID_ARG;
  const uint32_t alpha = (L + dnum - 1) / dnum;
  if ((dnum - 1) * alpha >= L || alpha > 192) return RNT_E_INVALID_ARG;  // every digit non-empty
  rnt_status s = check_plan_device(q_plan);
  if (s != RNT_OK) return s;
  const uint32_t K = LK - L;
  std::vector<uint64_t> m(LK);
  unsigned __int128 mmax = 0;
  for (uint32_t t = 0; t < LK; ++t) {
    m[t] = qp_plan->limbs[t].q;
    if (m[t] > mmax) mmax = m[t];
  }
  // k_ks_mac sums dnum exact products in 128 bits
  if (mmax * mmax > (~(unsigned __int128)0) / dnum) return RNT_E_INVALID_ARG;
  std::vector<KsMod> km(LK);
  for (uint32_t t = 0; t < LK; ++t) {
    const HostLimb& h = qp_plan->limbs[t];
    km[t].m = h.q;
    km[t].m2 = h.q2;
    km[t].qinv = h.qinv;
    km[t].r2 = h.r2;
    km[t].one = TW{1, (uint64_t)(((unsigned __int128)1 << 64) / h.q)};
    km[t].pinv = TW{0, 0};
    km[t].qhatinv = TW{0, 0};
  }
  for (uint32_t i = 0; i < L; ++i) {
    uint64_t pp = 1;
    for (uint32_t t = L; t < LK; ++t) pp = hp_mulmod(pp, m[t] % m[i], m[i]);
    const uint64_t pinv = hp_powmod(pp, m[i] - 2, m[i]);
    km[i].pinv = TW{pinv, (uint64_t)(((unsigned __int128)pinv << 64) / m[i])};
  }
  // ModUp tables per digit (reading KS2: digit j = limbs [j alpha, min(L, (j+1) alpha)))
  std::vector<TW> tab((size_t)dnum * LK * alpha, TW{0, 0});
  for (uint32_t j = 0; j < dnum; ++j) {
    const uint32_t lo = j * alpha, hi = (lo + alpha < L) ? lo + alpha : L;
    std::vector<BcMod> src, dst;
    std::vector<TW> qp;
    bconv_tables(m.data() + lo, hi - lo, m.data(), LK, src, dst, qp);
    for (uint32_t i = lo; i < hi; ++i) km[i].qhatinv = src[i - lo].qhatinv;
    for (uint32_t t = 0; t < LK; ++t)
      for (uint32_t i = 0; i < hi - lo; ++i) tab[((size_t)j * LK + t) * alpha + i] = qp[(size_t)t * (hi - lo) + i];
  }
  std::vector<BcMod> bsrc, bdst;
  std::vector<TW> bqp;
  bconv_tables(m.data() + L, K, m.data(), L, bsrc, bdst, bqp);

  rnt_keyswitch_s* ks = new (std::nothrow) rnt_keyswitch_s;
  if (!ks) return RNT_E_OOM;
  ks->device = q_plan->device;
  ks->logn = q_plan->logn;
  ks->L = L;
  ks->K = K;
  ks->LK = LK;
  ks->dnum = dnum;
  ks->alpha = alpha;
  ks->q = q_plan;
  ks->qp = qp_plan;
  {
    uint64_t qmax = 0, mmin = ~0ull;
    for (uint32_t i = 0; i < L; ++i) qmax = m[i] > qmax ? m[i] : qmax;
    for (uint32_t t = 0; t < LK; ++t) mmin = m[t] < mmin ? m[t] : mmin;
    static const bool force_unfused = env_int("RNT_KS_UNFUSED", 0) > 0;   // dispatch test hook
    ks->fused = !force_unfused && ks->logn >= 11 && alpha == 1 && qmax / 2 < mmin;
    ks->split = ks->fused ? ks_split(dnum) : 1;
  }
  const size_t n = (size_t)1 << ks->logn;
  const size_t ws =
      n * ((size_t)L + (size_t)dnum * LK + 2 * (size_t)LK * ks->split + 2 * (size_t)K + 2 * (size_t)L);
  cudaError_t e;
  if ((e = cudaMalloc(&ks->d_km, sizeof(KsMod) * LK)) != cudaSuccess ||
      (e = cudaMalloc(&ks->d_tab, sizeof(TW) * tab.size())) != cudaSuccess ||
      (e = cudaMalloc(&ks->d_bsrc, sizeof(BcMod) * K)) != cudaSuccess ||
      (e = cudaMalloc(&ks->d_bdst, sizeof(BcMod) * L)) != cudaSuccess ||
      (e = cudaMalloc(&ks->d_bqp, sizeof(TW) * bqp.size())) != cudaSuccess ||
      (e = cudaMalloc(&ks->d_ws, sizeof(u64) * ws)) != cudaSuccess ||
      (e = cudaMemcpy(ks->d_km, km.data(), sizeof(KsMod) * LK, cudaMemcpyHostToDevice)) != cudaSuccess ||
      (e = cudaMemcpy(ks->d_tab, tab.data(), sizeof(TW) * tab.size(), cudaMemcpyHostToDevice)) != cudaSuccess ||
      (e = cudaMemcpy(ks->d_bsrc, bsrc.data(), sizeof(BcMod) * K, cudaMemcpyHostToDevice)) != cudaSuccess ||
      (e = cudaMemcpy(ks->d_bdst, bdst.data(), sizeof(BcMod) * L, cudaMemcpyHostToDevice)) != cudaSuccess ||
      (e = cudaMemcpy(ks->d_bqp, bqp.data(), sizeof(TW) * bqp.size(), cudaMemcpyHostToDevice)) != cudaSuccess) {
    rnt_keyswitch_destroy(ks);
    return cuda_fail(e);
  }
  *out = ks;
  return RNT_OK;
}

rnt_status rnt_keyswitch_query(rnt_keyswitch ks, uint32_t* alpha, uint64_t* workspace_bytes) {
  if (!ks) return RNT_E_INVALID_ARG;
  const size_t n = (size_t)1 << ks->logn;
  if (alpha) *alpha = ks->alpha;
  if (workspace_bytes)
    *workspace_bytes = 8 * n * ((size_t)ks->L + (size_t)ks->dnum * ks->LK + 2 * (size_t)ks->LK * ks->split +
                                2 * (size_t)ks->K + 2 * (size_t)ks->L);
  return RNT_OK;
}

rnt_status rnt_keyswitch_apply(rnt_keyswitch ks, uint64_t* out_, const uint64_t* d_, const uint64_t* evk_,
                               const uint64_t* add0_, void* stream) {
  if (!ks) return RNT_E_INVALID_ARG;
  if (!out_ || !d_ || !evk_ || !aligned16(out_) || !aligned16(d_) || !aligned16(evk_) ||
      (add0_ && !aligned16(add0_)))
    return RNT_E_INVALID_ARG;
  rnt_status s = check_plan_device(ks->q);
  if (s != RNT_OK) return s;
  if ((s = debug_validate(ks->q, d_, ks->L, (cudaStream_t)stream)) != RNT_OK) return s;
  std::lock_guard<std::mutex> g(ks->mu);
  cudaStream_t st = (cudaStream_t)stream;
  u64* out = reinterpret_cast<u64*>(out_);
  const u64* d = reinterpret_cast<const u64*>(d_);
  const u64* evk = reinterpret_cast<const u64*>(evk_);
  const u64* add0 = reinterpret_cast<const u64*>(add0_);
  const uint32_t L = ks->L, K = ks->K, LK = ks->LK, logn = ks->logn;
  const size_t n = (size_t)1 << logn;
  u64* x = ks->d_ws;
  u64* E = x + (size_t)L * n;
  u64* u = E + (size_t)ks->dnum * LK * n;
  u64* up = u + 2 * (size_t)LK * n * ks->split;
  u64* w = up + 2 * (size_t)K * n;
  // 1. x = INTT_Q(d)
  if ((s = run_op(ks->q, 1, U(x), U(d), nullptr, 0, 1, st)) != RNT_OK) return s;
  // 2-3 fused: lift on load + column pass, row pass + key product
  if (ks->fused) {
    if ((s = ks_fused(ks->qp, u, E, x, evk, ks->dnum, ks->split, ks->d_km, st)) != RNT_OK) return s;
  } else {
  // 2. ModUp every digit, then NTT of the extended polynomials (batch = dnum)
  {
    const size_t smem = (size_t)ks->alpha * kKsTile * 8;
    if ((s = set_smem(k_modup, smem)) != RNT_OK) return s;
    dim3 grid((unsigned)((n + kKsTile - 1) / kKsTile), ks->dnum);
    k_modup<<<grid, kKsTile, smem, st>>>(E, x, ks->d_km, ks->d_tab, L, LK, ks->alpha, logn);
    if ((s = after_launch()) != RNT_OK) return s;
  }
  if ((s = run_op(ks->qp, 0, U(E), U(E), nullptr, 0, ks->dnum, st)) != RNT_OK) return s;
  // 3. key inner product
  {
    const uint64_t per = (uint64_t)LK * n;
    uint64_t blocks = (per + 255) / 256;
    const uint64_t cap = (uint64_t)num_sms() * 8;
    if (blocks > cap) blocks = cap;
    k_ks_mac<<<(unsigned)blocks, 256, 0, st>>>(u, E, evk, ks->d_km, ks->dnum, LK, logn);
    if ((s = after_launch()) != RNT_OK) return s;
  }
  }
  // 4. ModDown: INTT of the P limbs, BConv P -> Q, NTT_Q, (u - w) P^{-1}
  {
    rnt_plan_s pv;
    make_view(ks->qp, L, K, &pv);
    for (int k = 0; k < 2; ++k)
      if ((s = run_op(&pv, 1, U(up + (size_t)k * K * n), U(u + ((size_t)k * LK + L) * n), nullptr, 0, 1, st)) != RNT_OK)
        return s;
    const size_t smem = (size_t)K * kBcTile * 8;
    if ((s = set_smem(k_bconv, smem)) != RNT_OK) return s;
    dim3 grid((unsigned)((n + kBcTile - 1) / kBcTile), 2);
    k_bconv<<<grid, kBcTile, smem, st>>>(w, up, ks->d_bsrc, ks->d_bdst, ks->d_bqp, K, L, logn);
    if ((s = after_launch()) != RNT_OK) return s;
    if ((s = run_op(ks->q, 0, U(w), U(w), nullptr, 0, 2, st)) != RNT_OK) return s;
    const uint64_t total = 2 * (uint64_t)L * n;
    uint64_t blocks = (total + 255) / 256;
    const uint64_t cap = (uint64_t)num_sms() * 8;
    if (blocks > cap) blocks = cap;
    k_moddown<<<(unsigned)blocks, 256, 0, st>>>(out, u, w, add0, ks->d_km, L, LK, logn);
    return after_launch();
  }
}

rnt_status rnt_external_product(rnt_plan p, uint64_t* out, const uint64_t* c, const uint64_t* rgsw_hat,
                                uint32_t n_slot, uint32_t base_log2, uint32_t levels, void* stream) {
  if (!p) return RNT_E_INVALID_ARG;
  if (n_slot == 0) return RNT_OK;
  if (p->L != 1 || p->logn > 10) return RNT_E_INVALID_ARG;
  if (!out || !c || !rgsw_hat || out == c || !aligned16(out) || !aligned16(c) || !aligned16(rgsw_hat))
    return RNT_E_INVALID_ARG;
  if (base_log2 < 1 || base_log2 > 31 || levels < 1 || levels > 8 || base_log2 * (levels - 1) >= 63)
    return RNT_E_INVALID_ARG;
  rnt_status s = check_plan_device(p);
  if (s != RNT_OK) return s;
  DigitSpec ds;
  ds.bg = base_log2;
  ds.levels = levels;
  ds.off = 0;
  for (uint32_t i = 0; i + 1 < levels; ++i) ds.off += ((int64_t)1 << (base_log2 - 1)) << (i * base_log2);
  ds.half_q = (p->limbs[0].q - 1) / 2;
  u64* o = reinterpret_cast<u64*>(out);
  const u64* ci = reinterpret_cast<const u64*>(c);
  const u64* z = reinterpret_cast<const u64*>(rgsw_hat);
  cudaStream_t st = (cudaStream_t)stream;
  switch (p->logn) {
    case 4: return launch_extprod<4>(p, o, ci, z, n_slot, ds, st);
    case 5: return launch_extprod<5>(p, o, ci, z, n_slot, ds, st);
    case 6: return launch_extprod<6>(p, o, ci, z, n_slot, ds, st);
    case 7: return launch_extprod<7>(p, o, ci, z, n_slot, ds, st);
    case 8: return launch_extprod<8>(p, o, ci, z, n_slot, ds, st);
    case 9: return launch_extprod<9>(p, o, ci, z, n_slot, ds, st);
    case 10: return launch_extprod<10>(p, o, ci, z, n_slot, ds, st);
  }
  return RNT_E_UNSUPPORTED_N;
}

rnt_status rnt_polymul(rnt_plan p, uint64_t* c, const uint64_t* a, const uint64_t* b, uint32_t batch, int b_is_eval,
                       int b_broadcast, void* stream) {
  rnt_status s = check_data(p, c, a, batch);
  if (s != RNT_OK || batch == 0) return s;
  if (!b || !aligned16(b) || b == c) return RNT_E_INVALID_ARG;
  if ((s = debug_validate(p, a, (uint64_t)batch * p->L, (cudaStream_t)stream)) != RNT_OK ||
      (s = debug_validate(p, b, (uint64_t)(b_broadcast ? 1u : batch) * p->L, (cudaStream_t)stream)) != RNT_OK)
    return s;
  return run_op(p, b_is_eval ? 2 : 3, c, a, b, b_broadcast ? 1 : 0, batch, (cudaStream_t)stream);
}

rnt_status rnt_execute_host(rnt_plan p, rnt_op op, uint64_t* out_host, const uint64_t* in_host, uint64_t* dev_ws,
                            const uint64_t* b_dev, uint32_t batch, int b_broadcast, void* stream) {
  if (!p || (int)op < 0 || (int)op > 3) return RNT_E_INVALID_ARG;
  if (batch == 0) return RNT_OK;
  if (!out_host || !in_host) return RNT_E_INVALID_ARG;
  rnt_status s = check_data(p, dev_ws, dev_ws, batch);
  if (s != RNT_OK) return s;
  const bool bop = (op == RNT_OP_POLYMUL_EVAL || op == RNT_OP_POLYMUL);
  if (bop && (!b_dev || !aligned16(b_dev) || b_dev == dev_ws)) return RNT_E_INVALID_ARG;
  cudaStream_t st = (cudaStream_t)stream;
  const size_t n = (size_t)1 << p->logn;
  const size_t unit_bytes = n * 8;
  const size_t total_units = (size_t)batch * p->L;
  // Chunking: chunks over polynomials (batch > 1) or limbs (batch == 1),
  // round-robin over three internal streams so H2D copy, kernels and D2H copy
  // of successive chunks overlap.  Fork/join with the caller's stream by events.
  // Chunks of 32 MiB, uniform (round 2 sweep, profiles/r02/e2e: 32 MiB uniform beats the
  // earlier 16 MiB chunks with a ramp by 11 % on cfg5, 16 % on cfg2, 12 % on cfg3 and
  // 23 % on the serial schedule -- in a stream of calls the ramp's small chunks only
  // add per-copy overhead; RNT_EXPERIMENTS builds: RNT_E2E_CHUNK_MB, RNT_E2E_RAMP).
#ifdef RNT_EXPERIMENTS
  const size_t target = (size_t)(getenv("RNT_E2E_CHUNK_MB") ? atoi(getenv("RNT_E2E_CHUNK_MB")) : 32) << 20;
#else
  constexpr size_t target = (size_t)32 << 20;
#endif
  // Granule = one polynomial (batch > 1) or one limb (batch == 1).  Chunks of
  // `target` bytes; with `ramp` the first and last chunks ramp (target/8, /4, /2, ...).
#ifdef RNT_EXPERIMENTS
  const bool ramp = getenv("RNT_E2E_RAMP") != nullptr;
#else
  constexpr bool ramp = false;
#endif
  const size_t gbytes = batch > 1 ? (size_t)p->L * unit_bytes : unit_bytes;
  const size_t G = batch > 1 ? batch : p->L;
  size_t T = target / gbytes;
  if (T < 1) T = 1;
  std::vector<size_t> front, back;
  {
    size_t left = G;
    const size_t r0 = ramp ? (T / 8 ? T / 8 : 1) : T;
    for (size_t sz = r0; left; sz = sz * 2 < T ? sz * 2 : T) {
      const size_t a = sz < left ? sz : left;
      front.push_back(a);
      left -= a;
      if (!left) break;
      const size_t b = sz < left ? sz : left;
      back.push_back(b);
      left -= b;
    }
  }
  std::vector<size_t> csz(front);
  csz.insert(csz.end(), back.rbegin(), back.rend());
  const uint32_t nchunks = (uint32_t)csz.size();
  if (nchunks <= 1) {
    RNT_CUDA(cudaMemcpyAsync(dev_ws, in_host, total_units * unit_bytes, cudaMemcpyHostToDevice, st));
    s = run_op(p, (int)op, dev_ws, dev_ws, b_dev, b_broadcast ? 1 : 0, batch, st);
    if (s != RNT_OK) return s;
    RNT_CUDA(cudaMemcpyAsync(out_host, dev_ws, total_units * unit_bytes, cudaMemcpyDeviceToHost, st));
    return RNT_OK;
  }
  // Three-stage pipeline: aux[0] copies chunks in, aux[1] runs the kernels of
  // chunk c once its copy landed, aux[2] copies chunk c out once computed.
  // Chunks own disjoint parts of dev_ws, so the stages only wait on per-chunk
  // events and both copy engines stay busy.
  std::lock_guard<std::mutex> g(p->aux_mu);
  for (auto& a : p->aux)
    if (!a) RNT_CUDA(cudaStreamCreateWithFlags(&a, cudaStreamNonBlocking));
  while (p->ev_pool.size() < 2 * (size_t)nchunks + 4) {
    cudaEvent_t e;
    RNT_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
    p->ev_pool.push_back(e);
  }
  cudaEvent_t fork = p->ev_pool[0];
  RNT_CUDA(cudaEventRecord(fork, st));
  for (int i = 0; i < 3; ++i) RNT_CUDA(cudaStreamWaitEvent(p->aux[i], fork, 0));
  size_t g0 = 0;
  for (uint32_t c = 0; c < nchunks && s == RNT_OK; g0 += csz[c], ++c) {
    size_t u0, nu;
    const uint64_t* bchunk = b_dev;
    rnt_plan_s view;
    const rnt_plan_s* pp = p;
    uint32_t cb = batch;
    if (batch > 1) {
      cb = (uint32_t)csz[c];
      u0 = g0 * p->L;
      nu = (size_t)cb * p->L;
      if (bop && !b_broadcast) bchunk = b_dev + u0 * n;
    } else {
      const uint32_t l0 = (uint32_t)g0, nl = (uint32_t)csz[c];
      make_view(p, l0, nl, &view);
      pp = &view;
      u0 = l0;
      nu = nl;
      if (bop) bchunk = b_dev + (size_t)l0 * n;
    }
    cudaEvent_t ev_in = p->ev_pool[4 + 2 * c], ev_done = p->ev_pool[5 + 2 * c];
    cudaError_t e = cudaMemcpyAsync(dev_ws + u0 * n, in_host + u0 * n, nu * unit_bytes, cudaMemcpyHostToDevice,
                                    p->aux[0]);
    if (e == cudaSuccess) e = cudaEventRecord(ev_in, p->aux[0]);
    if (e == cudaSuccess) e = cudaStreamWaitEvent(p->aux[1], ev_in, 0);
    if (e != cudaSuccess) { s = cuda_fail(e); break; }
    s = run_op(const_cast<rnt_plan_s*>(pp), (int)op, dev_ws + u0 * n, dev_ws + u0 * n, bchunk,
               b_broadcast ? 1 : 0, cb, p->aux[1]);
    if (s != RNT_OK) break;
    e = cudaEventRecord(ev_done, p->aux[1]);
    if (e == cudaSuccess) e = cudaStreamWaitEvent(p->aux[2], ev_done, 0);
    if (e == cudaSuccess)
      e = cudaMemcpyAsync(out_host + u0 * n, dev_ws + u0 * n, nu * unit_bytes, cudaMemcpyDeviceToHost, p->aux[2]);
    if (e != cudaSuccess) { s = cuda_fail(e); break; }
  }
  for (int i = 0; i < 3; ++i) {
    cudaEventRecord(p->ev_pool[1 + i], p->aux[i]);
    cudaStreamWaitEvent(st, p->ev_pool[1 + i], 0);
  }
  return s;
}

}  // extern "C"
