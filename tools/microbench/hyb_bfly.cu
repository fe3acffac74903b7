// Hybrid integer / FP64 Shoup butterfly for sm_100a -- throughput microbenchmark.
//
// The exact Shoup product y w mod q (modarith.cuh) costs 5 IMAD.WIDE + 1 IMAD.HI
// + 4 IMAD on the fmaheavy pipe (~41 fmaheavy cycles per warp-butterfly, the
// binding pipe of every NTT kernel).  Here the quotient is estimated on the
// FP64 pipe (64 DFMA/clk/SM on B200, otherwise idle):
//   y = yh 2^32 + yl,  P = yl w + yh w2  (w2 = w 2^32 mod q, P = y w mod q),
//   x = P / q < 2^33,  b = fma(yh, f2, fma(yl, f, -0.75)) with f = w/q, f2 = w2/q,
//   t = b + 1.5 2^52  ->  bits(t) = C + Q, C = 0x4338000000000000, Q = round(b)
//   in {floor(x) - 1, floor(x)}  (|b - (x - 0.75)| < 2^-18),
//   r = P - Q q = yl w + yh w2 + bits(t) (-q) + C q  (mod 2^64)  in [0, 2q):
// 3 IMAD.WIDE + 4 IMAD, no bit extraction of Q (the double's exponent bits are
// the constant C, cancelled by the per-modulus constant K = C q mod 2^64).
//
//   A   V14 exact Shoup + sign csub (the shipped arithmetic)
//   B   hybrid, conversions by I2F.F64.U32
//   C   hybrid, conversions by the 2^52 magic (hiloint2double + DADD)
//   D   A with the LZ butterfly (no csub)
//   E   B with the LZ butterfly
//
// Build: nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o hyb tools/microbench/hyb_bfly.cu
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <cuda_runtime.h>

typedef unsigned long long u64;
typedef unsigned __int128 u128;

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("CUDA %s at %d\n", cudaGetErrorString(e), __LINE__); exit(1); } } while (0)

__device__ __forceinline__ uint32_t lo32(u64 x) { return (uint32_t)x; }
__device__ __forceinline__ uint32_t hi32(u64 x) { return (uint32_t)(x >> 32); }
__device__ __forceinline__ u64 mwide(uint32_t a, uint32_t b, u64 c) {
  u64 d;
  asm("mad.wide.u32 %0, %1, %2, %3;" : "=l"(d) : "r"(a), "r"(b), "l"(c));
  return d;
}
__device__ __forceinline__ uint32_t mlo(uint32_t a, uint32_t b, uint32_t c) {
  uint32_t d;
  asm("mad.lo.u32 %0, %1, %2, %3;" : "=r"(d) : "r"(a), "r"(b), "r"(c));
  return d;
}
__device__ __forceinline__ u64 pack(uint32_t lo, uint32_t hi) { return ((u64)hi << 32) | lo; }

struct HW {          // hybrid twiddle: 32 bytes
  u64 w, w2;         // w, w 2^32 mod q
  double f, f2;      // w / q, w2 / q
};

template <int CONV>
__device__ __forceinline__ double u2d(uint32_t x) {
  if constexpr (CONV == 0) return __uint2double_rn(x);
  else return __hiloint2double(0x43300000, (int)x) - 4503599627370496.0;
}

template <int CONV>
__device__ __forceinline__ u64 hyb_mul(u64 y, const HW& t, u64 nq, u64 K) {
  const uint32_t yl = lo32(y), yh = hi32(y);
  const double a = fma(u2d<CONV>(yl), t.f, -0.75);
  const double b = fma(u2d<CONV>(yh), t.f2, a);
  const u64 Qb = (u64)__double_as_longlong(__dadd_rn(b, 6755399441055744.0));
  u64 acc = mwide(yl, lo32(t.w), K);
  acc = mwide(yh, lo32(t.w2), acc);
  acc = mwide(lo32(Qb), lo32(nq), acc);
  uint32_t h = hi32(acc);
  h = mlo(yl, hi32(t.w), h);
  h = mlo(yh, hi32(t.w2), h);
  h = mlo(lo32(Qb), hi32(nq), h);
  h = mlo(hi32(Qb), lo32(nq), h);
  return pack(lo32(acc), h);
}

// Reordered: every y-only partial product is formed while the FP64 quotient is in
// flight; after it only lo64(Qb (-q)) = 1 WIDE + 2 IMAD and the adds remain.
// M3: the 1.5 2^52 magic is added inside the first FMA (one DADD less on the
// chain): two roundings at ulp 1 (error <= 1 + 2^-18), offset -2 -> r in [0, 4q).
template <bool M3>
__device__ __forceinline__ u64 hyb_mul2(u64 y, const HW& t, u64 nq, u64 K) {
  const uint32_t yl = lo32(y), yh = hi32(y);
  u64 Qb;
  if constexpr (M3) {
    const double a = fma(__uint2double_rn(yl), t.f, 6755399441055744.0 - 2.0);
    Qb = (u64)__double_as_longlong(fma(__uint2double_rn(yh), t.f2, a));
  } else {
    const double a = fma(__uint2double_rn(yl), t.f, -0.75);
    const double b = fma(__uint2double_rn(yh), t.f2, a);
    Qb = (u64)__double_as_longlong(__dadd_rn(b, 6755399441055744.0));
  }
  u64 acc = mwide(yl, lo32(t.w), K);
  acc = mwide(yh, lo32(t.w2), acc);
  const uint32_t g = yl * hi32(t.w) + yh * hi32(t.w2);
  const u64 pq = (u64)lo32(Qb) * lo32(nq);
  const uint32_t u = lo32(Qb) * hi32(nq) + hi32(Qb) * lo32(nq);
  return acc + pq + ((u64)(g + u) << 32);
}

__device__ __forceinline__ u64 csub(u64 x, u64 m) {
  const u64 d = x - m;
  return (long long)d < 0 ? x : d;
}

__device__ __forceinline__ u64 shoup(u64 y, u64 w, u64 wp, u64 q) {
  u64 Q = __umul64hi(y, wp);
  return y * w - Q * q;
}

constexpr int ITERS = 128;
constexpr int ILPMAX = 8;

struct Par {
  u64 q, q2, nq, K, w, wp;
  HW h;
};

// V: 0 exact (csub), 1 hybrid I2F (csub), 2 hybrid magic (csub), 3 exact LZ, 4 hybrid I2F LZ, 5 hybrid magic LZ
// LZ chains: X never reduced -> values grow; to keep them bounded the LZ variants
// reduce X by csub(X, 8q) every 4th iteration (one reduction per 4 stages).
template <int V, int ILP = 8>
__global__ void __launch_bounds__(256) k_chain(u64* out, const u64* in, Par p, long long* cyc) {
  u64 X[ILP], Y[ILP];
  const int gid = blockIdx.x * blockDim.x + threadIdx.x;
#pragma unroll
  for (int i = 0; i < ILP; ++i) {
    X[i] = in[(gid * 2 * ILP + 2 * i) & ((1 << 20) - 1)];
    Y[i] = in[(gid * 2 * ILP + 2 * i + 1) & ((1 << 20) - 1)];
  }
  const u64 q2 = p.q2;
  // twiddles in registers, as the NTT kernels hold them (loaded from memory)
  Par r;
  r.q = in[(1 << 20) + 0]; r.nq = in[(1 << 20) + 1]; r.K = in[(1 << 20) + 2];
  r.w = in[(1 << 20) + 3]; r.wp = in[(1 << 20) + 4];
  r.h.w = in[(1 << 20) + 5]; r.h.w2 = in[(1 << 20) + 6];
  r.h.f = __longlong_as_double((long long)in[(1 << 20) + 7]); r.h.f2 = __longlong_as_double((long long)in[(1 << 20) + 8]);
  long long t0 = clock64();
  for (int it = 0; it < ITERS; ++it) {
#pragma unroll
    for (int i = 0; i < ILP; ++i) {
      // V 8 / 9: mixed -- pairs i % MIX != 0 exact, i % MIX == 0 hybrid (B)
      constexpr int MIX = V == 8 ? 2 : 4;
      const bool hyb = (V == 8 || V == 9) && (i % MIX == 0);
      const bool lz = V >= 3 && V != 6 && V != 7 && V != 8 && V != 9;
      u64 x = X[i];
      if (V == 7) x = csub(x, q2 << 1);          // [0, 8q) -> [0, 4q)
      else if (!lz) x = csub(x, q2);
      else if ((it & 3) == 3) x = csub(x, q2 << 2);
      u64 v;
      if constexpr (V == 8 || V == 9) v = hyb ? hyb_mul<0>(Y[i], r.h, r.nq, r.K) : shoup(Y[i], r.w, r.wp, r.q);
      else if constexpr (V == 0 || V == 3) v = shoup(Y[i], r.w, r.wp, r.q);
      else if constexpr (V == 1 || V == 4) v = hyb_mul<0>(Y[i], r.h, r.nq, r.K);
      else if constexpr (V == 6) v = hyb_mul2<false>(Y[i], r.h, r.nq, r.K);
      else if constexpr (V == 7) v = hyb_mul2<true>(Y[i], r.h, r.nq, r.K);
      else v = hyb_mul<1>(Y[i], r.h, r.nq, r.K);
      X[i] = x + v;
      Y[i] = x + (V == 7 ? q2 << 1 : q2) - v;
    }
  }
  long long t1 = clock64();
#pragma unroll
  for (int i = 0; i < ILP; ++i) {
    out[gid * 2 * ILP + 2 * i] = X[i];
    out[gid * 2 * ILP + 2 * i + 1] = Y[i];
  }
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}

static u64 mulmod(u64 a, u64 b, u64 q) { return (u64)(((u128)a * b) % q); }

int main(int argc, char** argv) {
  int dev = 0;
  CK(cudaSetDevice(dev));
  int sms;
  CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
  const u64 q = (1ull << 60) - (1ull << 14) + 1;  // reading C2, N = 2^10 prime
  const u64 w = 0x0123456789abcdefull % q;
  Par p;
  p.q = q; p.q2 = 2 * q; p.nq = 0ull - q;
  p.K = (u64)(0x4338000000000000ull * q);
  p.w = w; p.wp = (u64)(((u128)w << 64) / q);
  p.h.w = w; p.h.w2 = (u64)(((u128)w << 32) % q);
  p.h.f = (double)w / (double)q; p.h.f2 = (double)p.h.w2 / (double)q;
  // exact f, f2: round(w / q) computed in long double is close enough; refine with __int128
  {
    // f = w/q to nearest double: use 2^-64 scaled integer quotient
    u128 fq = ((u128)w << 64) / q; long double fl = (long double)fq / 18446744073709551616.0L; p.h.f = (double)fl;
    u128 fq2 = ((u128)p.h.w2 << 64) / q; long double fl2 = (long double)fq2 / 18446744073709551616.0L; p.h.f2 = (double)fl2;
  }
  const int TPB = 256;
  int cps = argc > 1 ? atoi(argv[1]) : 4;
  const int grid = sms * cps, nthr = grid * TPB;
  u64 *din, *dout; long long* cyc;
  CK(cudaMalloc(&din, (size_t)((1 << 20) + 16) * 8));
  CK(cudaMalloc(&dout, (size_t)nthr * 2 * ILPMAX * 8));
  CK(cudaMalloc(&cyc, grid * 8));
  u64* h = (u64*)malloc((size_t)(1 << 20) * 8);
  u64 s = 88172645463325252ull;
  for (int i = 0; i < (1 << 20); ++i) { s ^= s << 13; s ^= s >> 7; s ^= s << 17; h[i] = s % q; }
  CK(cudaMemcpy(din, h, (size_t)(1 << 20) * 8, cudaMemcpyHostToDevice));
  {
    u64 c[9] = {p.q, p.nq, p.K, p.w, p.wp, p.h.w, p.h.w2, 0, 0};
    memcpy(&c[7], &p.h.f, 8); memcpy(&c[8], &p.h.f2, 8);
    CK(cudaMemcpy(din + (1 << 20), c, sizeof c, cudaMemcpyHostToDevice));
  }
  u64* ho = (u64*)malloc((size_t)nthr * 2 * ILPMAX * 8);
  long long* hc = (long long*)malloc(grid * 8);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  auto run = [&](auto kern, const char* name, int ILP = 8) {
    kern<<<grid, TPB>>>(dout, din, p, cyc);
    CK(cudaEventRecord(e0));
    kern<<<grid, TPB>>>(dout, din, p, cyc);
    CK(cudaEventRecord(e1));
    CK(cudaEventSynchronize(e1));
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    CK(cudaMemcpy(hc, cyc, grid * 8, cudaMemcpyDeviceToHost));
    CK(cudaMemcpy(ho, dout, (size_t)nthr * 2 * ILPMAX * 8, cudaMemcpyDeviceToHost));
    long long mx = 0;
    for (int i = 0; i < grid; ++i) if (hc[i] > mx) mx = hc[i];
    int bad = 0;
    for (int t = 0; t < 64; ++t) {
      for (int i = 0; i < ILP; ++i) {
        u64 rX = h[(t * 2 * ILP + 2 * i) & ((1 << 20) - 1)], rY = h[(t * 2 * ILP + 2 * i + 1) & ((1 << 20) - 1)];
        for (int it = 0; it < ITERS; ++it) {
          u64 tt = mulmod(rY, w, q);
          u64 nx = (rX + tt) % q, ny = (rX + q - tt) % q;
          rX = nx; rY = ny;
        }
        if (ho[t * 2 * ILP + 2 * i] % q != rX || ho[t * 2 * ILP + 2 * i + 1] % q != rY) ++bad;
      }
    }
    const double bfly = (double)ITERS * ILP * TPB * cps;
    printf("{\"variant\":\"%s\",\"ilp\":%d,\"cta_per_sm\":%d,\"bfly_per_clk_per_sm\":%.3f,\"ms\":%.4f,\"bad\":%d}\n", name, ILP, cps,
           bfly / mx, ms, bad);
  };
  for (int rep = 0; rep < 2; ++rep) {
    run(k_chain<0>, "A_exact");
    run(k_chain<1>, "B_hyb_i2f");
    run(k_chain<2>, "C_hyb_magic");
    run(k_chain<3>, "D_exact_lz");
    run(k_chain<4>, "E_hyb_i2f_lz");
    run(k_chain<5>, "F_hyb_magic_lz");
    run(k_chain<6>, "G_hyb_reorder");
    run(k_chain<7>, "H_hyb_reorder_3q");
    run(k_chain<8>, "I_mix_1of2");
    run(k_chain<9>, "J_mix_1of4");
    run(k_chain<0, 4>, "A_exact", 4);
    run(k_chain<1, 4>, "B_hyb_i2f", 4);
    run(k_chain<6, 4>, "G_hyb_reorder", 4);
    run(k_chain<7, 4>, "H_hyb_reorder_3q", 4);
  }
  return 0;
}
