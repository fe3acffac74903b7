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
// Scatter formulation: a thread reads in[e] (coalesced) and writes it to its destination --
// pi^{-1} is the same map with g^{-1}, and coefficient i goes to i g mod 2N (negated past
// N) -- so the loads never stall on a gather.  In NTT form pi maps every aligned block of
// 32 slots onto one aligned block of 32 slots (the 5 low bits of k are the high bits of
// brv(k), and multiplying by odd g mod 2N permutes high bits among themselves), so a
// warp's 32 scattered 8-byte stores still cover whole 32-byte sectors of one 256-byte run.
// Each thread loads KA pairs of slots with 16-byte loads, all in flight before the
// first store (the one-element grid-stride loop was latency bound on small jobs:
// cfg3 moves 47 MB at 0.43 of HBM).
constexpr int kAutoPairs = 4;
__device__ __forceinline__ void automorph_put(u64* __restrict__ out, const LimbC* __restrict__ lc, uint64_t e, u64 x,
                                              uint32_t L, uint32_t logn, uint32_t g, uint32_t ginv, int ntt_domain) {
  const uint32_t n = 1u << logn, mask2n = 2 * n - 1;
  const uint64_t u = e >> logn;
  const uint32_t k = (uint32_t)(e & (n - 1));
  u64* dst = out + (u << logn);
  if (ntt_domain) {
    const uint32_t ek = 2u * (__brev(k) >> (32 - logn)) + 1u;
    const uint32_t es = (uint32_t)(((uint64_t)ek * ginv) & mask2n);
    __stcs(dst + (__brev((es - 1u) >> 1) >> (32 - logn)), x);
  } else {
    const uint32_t t = (uint32_t)(((uint64_t)k * g) & mask2n);
    if (t < n) {
      __stcs(dst + t, x);
    } else {
      const u64 q = lc[u % L].q;
      __stcs(dst + (t - n), x ? q - x : 0ull);
    }
  }
}

__global__ void __launch_bounds__(256) k_automorph(u64* __restrict__ out, const u64* __restrict__ in,
                                                   const LimbC* __restrict__ lc, uint32_t L, uint32_t logn, uint32_t g,
                                                   uint32_t ginv, int ntt_domain, uint64_t total) {
  const uint64_t npair = total >> 1;   // total = units N, N >= 16: even
  const ulonglong2* in2 = reinterpret_cast<const ulonglong2*>(in);
  const uint64_t step = (uint64_t)gridDim.x * blockDim.x * kAutoPairs;
  for (uint64_t b = (uint64_t)blockIdx.x * blockDim.x * kAutoPairs + threadIdx.x; b < npair; b += step) {
    ulonglong2 v[kAutoPairs];
#pragma unroll
    for (int i = 0; i < kAutoPairs; ++i) {
      const uint64_t p = b + (uint64_t)i * blockDim.x;
      if (p < npair) v[i] = __ldcs(in2 + p);
    }
#pragma unroll
    for (int i = 0; i < kAutoPairs; ++i) {
      const uint64_t p = b + (uint64_t)i * blockDim.x;
      if (p < npair) {
        automorph_put(out, lc, 2 * p, v[i].x, L, logn, g, ginv, ntt_domain);
        automorph_put(out, lc, 2 * p + 1, v[i].y, L, logn, g, ginv, ntt_domain);
      }
    }
  }
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
  uint64_t blocks = (total / 2 + threads * kAutoPairs - 1) / (threads * kAutoPairs);
  const uint64_t cap = (uint64_t)num_sms() * 8;
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
  // chunk bytes: 16 MiB (measured best of 4 .. 64)
  constexpr size_t target = (size_t)16 << 20;
  // Granule = one polynomial (batch > 1) or one limb (batch == 1).  Chunks of
  // `target` bytes, except that the first and last chunks ramp (target/8,
  // /4, /2, ...) so the copy engines start and drain sooner (measured better than uniform).
  constexpr bool ramp = true;
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
