// Butterfly arithmetic variants for sm_100a: throughput (bfly/clk/SM) and a
// correctness check (results agree mod q with an exact __int128 host model).
//
//   V0  nvcc default: __umul64hi Shoup + csub            (baseline)
//   V2  hand-split exact Shoup: 1 IMAD.HI + 5 IMAD.WIDE + 4 IMAD, r = YW + Q(-q)
//   V3  V2 with a high-word-only lazy compare (range [0, 4q + 2^32))
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <cuda_runtime.h>

typedef unsigned long long u64;
typedef unsigned __int128 u128;

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("CUDA %s at %d\n", cudaGetErrorString(e), __LINE__); exit(1); } } while (0)

struct TW { u64 w, wp; };

__device__ __forceinline__ uint32_t lo32(u64 x) { return (uint32_t)x; }
__device__ __forceinline__ uint32_t hi32(u64 x) { return (uint32_t)(x >> 32); }
__device__ __forceinline__ u64 mwide(uint32_t a, uint32_t b, u64 c) {
  u64 d;
  asm("mad.wide.u32 %0, %1, %2, %3;" : "=l"(d) : "r"(a), "r"(b), "l"(c));
  return d;
}
__device__ __forceinline__ uint32_t mhi(uint32_t a, uint32_t b) {
  uint32_t d;
  asm("mul.hi.u32 %0, %1, %2;" : "=r"(d) : "r"(a), "r"(b));
  return d;
}
__device__ __forceinline__ uint32_t mlo(uint32_t a, uint32_t b, uint32_t c) {
  uint32_t d;
  asm("mad.lo.u32 %0, %1, %2, %3;" : "=r"(d) : "r"(a), "r"(b), "r"(c));
  return d;
}
__device__ __forceinline__ u64 pack(uint32_t lo, uint32_t hi) { return ((u64)hi << 32) | lo; }

// exact hi64(y * wp) for y < 2^62 (y1 < 2^30)
__device__ __forceinline__ u64 hi64_exact(u64 y, u64 wp) {
  uint32_t y0 = lo32(y), y1 = hi32(y), p0 = lo32(wp), p1 = hi32(wp);
  uint32_t A = mhi(y0, p0);
  u64 B = mwide(y0, p1, (u64)A);            // < 2^64
  u64 C = mwide(y1, p0, (u64)lo32(B));      // < 2^62 + 2^32
  u64 F = (u64)hi32(B) + (u64)hi32(C);      // 64-bit add (ALU)
  return mwide(y1, p1, F);
}

// r = y*w - Q*q (mod 2^64) with nq = -q mod 2^64
__device__ __forceinline__ u64 shoup_r(u64 y, u64 w, u64 Q, u64 nq) {
  uint32_t y0 = lo32(y), y1 = hi32(y), w0 = lo32(w), w1 = hi32(w);
  u64 yw = mwide(y0, w0, 0ull);
  uint32_t h = mlo(y0, w1, hi32(yw));
  h = mlo(y1, w0, h);
  yw = pack(lo32(yw), h);
  uint32_t Q0 = lo32(Q), Q1 = hi32(Q), n0 = lo32(nq), n1 = hi32(nq);
  u64 r = mwide(Q0, n0, yw);
  uint32_t rh = mlo(Q0, n1, hi32(r));
  rh = mlo(Q1, n0, rh);
  return pack(lo32(r), rh);
}

__device__ __forceinline__ void bfly_v0(u64& X, u64& Y, u64 w, u64 wp, u64 q, u64 q2, u64 nq) {
  u64 x = X >= q2 ? X - q2 : X;
  u64 Q = __umul64hi(Y, wp);
  u64 T = Y * w - Q * q;
  X = x + T;
  Y = x - T + q2;
}

// V14: V0 with the kernels' sign-test conditional subtraction (modarith.cuh csub)
__device__ __forceinline__ void bfly_v14(u64& X, u64& Y, u64 w, u64 wp, u64 q, u64 q2, u64 nq) {
  const u64 d = X - q2;
  u64 x = (long long)d < 0 ? X : d;
  u64 Q = __umul64hi(Y, wp);
  u64 T = Y * w - Q * q;
  X = x + T;
  Y = x - T + q2;
}

__device__ __forceinline__ void bfly_v2(u64& X, u64& Y, u64 w, u64 wp, u64 q, u64 q2, u64 nq) {
  u64 x = X >= q2 ? X - q2 : X;
  u64 Q = hi64_exact(Y, wp);
  u64 T = shoup_r(Y, w, Q, nq);
  X = x + T;
  Y = x - T + q2;
}

// high-word lazy compare: X in [0, 4q + 2^32) -> x in [0, 2q + 2^32)
__device__ __forceinline__ void bfly_v3(u64& X, u64& Y, u64 w, u64 wp, u64 q, u64 q2, u64 nq) {
  u64 sub = hi32(X) > hi32(q2) ? q2 : 0ull;
  u64 Q = hi64_exact(Y, wp);
  u64 T = shoup_r(Y, w, Q, nq);
  u64 x = X - sub;
  X = x + T;
  Y = x - T + q2;
}


// V4: whole CT butterfly in one PTX block (32-bit registers, explicit carries)
__device__ __forceinline__ void bfly_v4(u64& X, u64& Y, u64 w, u64 wp, u64 q, u64 q2, u64 nq) {
  uint32_t x0 = lo32(X), x1 = hi32(X), y0 = lo32(Y), y1 = hi32(Y);
  uint32_t X0, X1, Y0, Y1;
  asm("{\n\t"
      ".reg .u32 A, Bl, Bh, Cl, Ch, f0, f1, Q0, Q1, W0, W1, R0, R1, d0, d1, s0, s1, t0, t1;\n\t"
      ".reg .u64 B, C, F, Q, YW, R, A64, Bl64;\n\t"
      ".reg .pred p;\n\t"
      "mul.hi.u32 A, %4, %8;\n\t"
      "mov.b64 A64, {A, 0};\n\t"
      "mad.wide.u32 B, %4, %9, A64;\n\t"
      "mov.b64 {Bl, Bh}, B;\n\t"
      "mov.b64 Bl64, {Bl, 0};\n\t"
      "mad.wide.u32 C, %5, %8, Bl64;\n\t"
      "mov.b64 {Cl, Ch}, C;\n\t"
      "add.cc.u32 f0, Bh, Ch;\n\t"
      "addc.u32 f1, 0, 0;\n\t"
      "mov.b64 F, {f0, f1};\n\t"
      "mad.wide.u32 Q, %5, %9, F;\n\t"
      "mov.b64 {Q0, Q1}, Q;\n\t"
      "mul.wide.u32 YW, %4, %6;\n\t"
      "mov.b64 {W0, W1}, YW;\n\t"
      "mad.lo.u32 W1, %4, %7, W1;\n\t"
      "mad.lo.u32 W1, %5, %6, W1;\n\t"
      "mov.b64 YW, {W0, W1};\n\t"
      "mad.wide.u32 R, Q0, %10, YW;\n\t"
      "mov.b64 {R0, R1}, R;\n\t"
      "mad.lo.u32 R1, Q0, %11, R1;\n\t"
      "mad.lo.u32 R1, Q1, %10, R1;\n\t"
      // x' = X >= 2q ? X - 2q : X   (sign of the 64-bit difference)
      "sub.cc.u32 d0, %14, %12;\n\t"
      "subc.u32 d1, %15, %13;\n\t"
      "setp.lt.s32 p, d1, 0;\n\t"
      "selp.u32 d0, %14, d0, p;\n\t"
      "selp.u32 d1, %15, d1, p;\n\t"
      // X_out = x' + T ; Y_out = x' + 2q - T
      "add.cc.u32 %0, d0, R0;\n\t"
      "addc.u32 %1, d1, R1;\n\t"
      "sub.cc.u32 t0, %12, R0;\n\t"
      "subc.u32 t1, %13, R1;\n\t"
      "add.cc.u32 %2, d0, t0;\n\t"
      "addc.u32 %3, d1, t1;\n\t"
      "}"
      : "=r"(X0), "=r"(X1), "=r"(Y0), "=r"(Y1)
      : "r"(y0), "r"(y1), "r"(lo32(w)), "r"(hi32(w)), "r"(lo32(wp)), "r"(hi32(wp)),
        "r"(lo32(nq)), "r"(hi32(nq)), "r"(lo32(q2)), "r"(hi32(q2)), "r"(x0), "r"(x1));
  X = pack(X0, X1);
  Y = pack(Y0, Y1);
}


// V5: approximate Shoup quotient (lo partials dropped, Q' in [Qe-2, Qe] ->
// r in [0, 4q)), lazy invariant [0, 8q + 2^32), high-word compare.  q < 2^60.
__device__ __forceinline__ void bfly_v5(u64& X, u64& Y, u64 w, u64 wp, u64 q4, u64 nq) {
  const uint32_t y0 = lo32(Y), y1 = hi32(Y);
  const uint32_t p0 = lo32(wp), p1 = hi32(wp), w0 = lo32(w), w1 = hi32(w);
  u64 B, C, S, Q, YW, R;
  asm("mul.wide.u32 %0, %1, %2;" : "=l"(B) : "r"(y0), "r"(p1));
  asm("mul.wide.u32 %0, %1, %2;" : "=l"(C) : "r"(y1), "r"(p0));
  S = (u64)hi32(B) + (u64)hi32(C);
  asm("mad.wide.u32 %0, %1, %2, %3;" : "=l"(Q) : "r"(y1), "r"(p1), "l"(S));
  asm("mul.wide.u32 %0, %1, %2;" : "=l"(YW) : "r"(y0), "r"(w0));
  uint32_t h = hi32(YW);
  asm("mad.lo.u32 %0, %1, %2, %0;" : "+r"(h) : "r"(y0), "r"(w1));
  asm("mad.lo.u32 %0, %1, %2, %0;" : "+r"(h) : "r"(y1), "r"(w0));
  YW = pack(lo32(YW), h);
  const uint32_t Q0 = lo32(Q), Q1 = hi32(Q);
  asm("mad.wide.u32 %0, %1, %2, %3;" : "=l"(R) : "r"(Q0), "r"(lo32(nq)), "l"(YW));
  uint32_t rh = hi32(R);
  asm("mad.lo.u32 %0, %1, %2, %0;" : "+r"(rh) : "r"(Q0), "r"(hi32(nq)));
  asm("mad.lo.u32 %0, %1, %2, %0;" : "+r"(rh) : "r"(Q1), "r"(lo32(nq)));
  const u64 r = pack(lo32(R), rh);
  const bool big = hi32(X) > hi32(q4);
  const u64 sub = big ? q4 : 0ull;
  const u64 add = big ? 0ull : q4;
  const u64 Xin = X;
  X = Xin - sub + r;
  Y = Xin + add - r;
}

// V6: exact Shoup with a 3-input carry sum (IMAD.HI + 3 WIDE + IADD3 chain).
__device__ __forceinline__ void bfly_v6(u64& X, u64& Y, u64 w, u64 wp, u64 q2, u64 nq) {
  const uint32_t y0 = lo32(Y), y1 = hi32(Y);
  const uint32_t p0 = lo32(wp), p1 = hi32(wp), w0 = lo32(w), w1 = hi32(w);
  u64 B, C, D, YW, R;
  uint32_t A, t0, t1, s;
  asm("mul.hi.u32 %0, %1, %2;" : "=r"(A) : "r"(y0), "r"(p0));
  asm("mul.wide.u32 %0, %1, %2;" : "=l"(B) : "r"(y0), "r"(p1));
  asm("mul.wide.u32 %0, %1, %2;" : "=l"(C) : "r"(y1), "r"(p0));
  asm("mul.wide.u32 %0, %1, %2;" : "=l"(D) : "r"(y1), "r"(p1));
  asm("{\n\t"
      "add.cc.u32 %2, %3, %4;\n\t"
      "addc.cc.u32 %0, %5, %6;\n\t"
      "addc.u32 %1, %7, 0;\n\t"
      "add.cc.u32 %2, %2, %8;\n\t"
      "addc.cc.u32 %0, %0, %9;\n\t"
      "addc.u32 %1, %1, 0;\n\t"
      "}"
      : "=r"(t0), "=r"(t1), "=r"(s)
      : "r"(lo32(B)), "r"(lo32(C)), "r"(lo32(D)), "r"(hi32(B)), "r"(hi32(D)), "r"(A), "r"(hi32(C)));
  const uint32_t Q0 = t0, Q1 = t1;
  asm("mul.wide.u32 %0, %1, %2;" : "=l"(YW) : "r"(y0), "r"(w0));
  uint32_t h = hi32(YW);
  asm("mad.lo.u32 %0, %1, %2, %0;" : "+r"(h) : "r"(y0), "r"(w1));
  asm("mad.lo.u32 %0, %1, %2, %0;" : "+r"(h) : "r"(y1), "r"(w0));
  YW = pack(lo32(YW), h);
  asm("mad.wide.u32 %0, %1, %2, %3;" : "=l"(R) : "r"(Q0), "r"(lo32(nq)), "l"(YW));
  uint32_t rh = hi32(R);
  asm("mad.lo.u32 %0, %1, %2, %0;" : "+r"(rh) : "r"(Q0), "r"(hi32(nq)));
  asm("mad.lo.u32 %0, %1, %2, %0;" : "+r"(rh) : "r"(Q1), "r"(lo32(nq)));
  const u64 r = pack(lo32(R), rh);
  const bool big = hi32(X) > hi32(q2);
  const u64 sub = big ? q2 : 0ull;
  const u64 add = big ? 0ull : q2;
  const u64 Xin = X;
  X = Xin - sub + r;
  Y = Xin + add - r;
}


// V7: nvcc-style C, but T = Y*w + Q*(-q) (negation folded into the constant)
//     and a high-word-only lazy compare.
__device__ __forceinline__ void bfly_v7(u64& X, u64& Y, u64 w, u64 wp, u64 q2, u64 nq) {
  const u64 Q = __umul64hi(Y, wp);
  const u64 T = Y * w + Q * nq;
  const bool big = (uint32_t)(X >> 32) > (uint32_t)(q2 >> 32);
  const u64 x = X - (big ? q2 : 0ull);
  X = x + T;
  Y = x + q2 - T;
}
// V8: V7 with the approximate quotient (r in [0,4q)), invariant [0, 8q + 2^32).
__device__ __forceinline__ void bfly_v8(u64& X, u64& Y, u64 w, u64 wp, u64 q4, u64 nq) {
  const uint32_t y0 = (uint32_t)Y, y1 = (uint32_t)(Y >> 32), p0 = (uint32_t)wp, p1 = (uint32_t)(wp >> 32);
  const u64 Q = (u64)y1 * p1 + (((u64)y0 * p1) >> 32) + (((u64)y1 * p0) >> 32);
  const u64 T = Y * w + Q * nq;
  const bool big = (uint32_t)(X >> 32) > (uint32_t)(q4 >> 32);
  const u64 x = X - (big ? q4 : 0ull);
  X = x + T;
  Y = x + q4 - T;
}
// V9: V8 but with __umulhi for the two cross terms.
__device__ __forceinline__ void bfly_v9(u64& X, u64& Y, u64 w, u64 wp, u64 q4, u64 nq) {
  const uint32_t y0 = (uint32_t)Y, y1 = (uint32_t)(Y >> 32), p0 = (uint32_t)wp, p1 = (uint32_t)(wp >> 32);
  const u64 Q = (u64)y1 * p1 + (u64)__umulhi(y0, p1) + (u64)__umulhi(y1, p0);
  const u64 T = Y * w + Q * nq;
  const bool big = (uint32_t)(X >> 32) > (uint32_t)(q4 >> 32);
  const u64 x = X - (big ? q4 : 0ull);
  X = x + T;
  Y = x + q4 - T;
}

constexpr int ITERS = 256;

// V15: V14 for a sparse modulus q = 2^60 - 2^b + 1 (1 <= b < 32): Q q mod 2^64 =
// (Q << 60) - (Q << b) + Q is formed with shifts and adds on the ALU pipe instead of
// one IMAD.WIDE + two IMAD on the fmaheavy pipe.
__device__ __forceinline__ void bfly_v15(u64& X, u64& Y, u64 w, u64 wp, u64 q2, int b) {
  const u64 d = X - q2;
  u64 x = (long long)d < 0 ? X : d;
  u64 Q = __umul64hi(Y, wp);
  const uint32_t Q0 = (uint32_t)Q, Q1 = (uint32_t)(Q >> 32);
  const u64 Qb = ((u64)__funnelshift_l(Q0, Q1, b) << 32) | (uint32_t)(Q0 << b);   // Q << b (b < 32)
  const u64 Q60 = (u64)(Q0 << 28) << 32;                                            // Q << 60 mod 2^64
  u64 T = Y * w - Q - Q60 + Qb;
  X = x + T;
  Y = x - T + q2;
}

// V16: V15 with the correction neg = (Q << b) - Q - (Q << 60) formed first (runtime shift
// counts, so ptxas cannot turn the shifts into IMADs by constants) and folded into the
// addend of the y w product.
__device__ __forceinline__ void bfly_v16(u64& X, u64& Y, u64 w, u64 wp, u64 q2, int b, int s28) {
  const u64 d = X - q2;
  u64 x = (long long)d < 0 ? X : d;
  u64 Q = __umul64hi(Y, wp);
  const uint32_t Q0 = (uint32_t)Q, Q1 = (uint32_t)(Q >> 32);
  uint32_t n0, n1;
  asm("{\n\t.reg .u32 t0, t1, t2;\n\t"
      "shl.b32 t0, %2, %4;\n\t"
      "shf.l.wrap.b32 t1, %2, %3, %4;\n\t"
      "shl.b32 t2, %2, %5;\n\t"
      "sub.cc.u32 %0, t0, %2;\n\t"
      "subc.u32 %1, t1, %3;\n\t"
      "sub.u32 %1, %1, t2;\n\t}"
      : "=r"(n0), "=r"(n1) : "r"(Q0), "r"(Q1), "r"(b), "r"(s28));
  const u64 neg = ((u64)n1 << 32) | n0;
  u64 T = Y * w + neg;
  X = x + T;
  Y = x - T + q2;
}

template <int V>
__global__ void k_bfly(u64* out, const u64* in, u64 w, u64 wp, u64 q, long long* cyc) {
  u64 X[4], Y[4];
  const int gid = blockIdx.x * blockDim.x + threadIdx.x;
  for (int i = 0; i < 4; ++i) { X[i] = in[gid * 8 + 2 * i]; Y[i] = in[gid * 8 + 2 * i + 1]; }
  const u64 q2 = 2 * q, nq = 0ull - q;
  const int sb = __ffsll((long long)((1ull << 60) + 1 - q)) - 1;   // V15: q = 2^60 - 2^sb + 1
  const int s28 = 28 + (int)(q >> 63);                              // V16: runtime 28
  long long t0 = clock64();
  for (int it = 0; it < ITERS; ++it) {
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      if (V == 0) bfly_v0(X[i], Y[i], w, wp, q, q2, nq);
      if (V == 2) bfly_v2(X[i], Y[i], w, wp, q, q2, nq);
      if (V == 3) bfly_v3(X[i], Y[i], w, wp, q, q2, nq);
      if (V == 4) bfly_v4(X[i], Y[i], w, wp, q, q2, nq);
      if (V == 5) bfly_v5(X[i], Y[i], w, wp, 4 * q, nq);
      if (V == 6) bfly_v6(X[i], Y[i], w, wp, q2, nq);
      if (V == 7) bfly_v7(X[i], Y[i], w, wp, q2, nq);
      if (V == 8) bfly_v8(X[i], Y[i], w, wp, 4 * q, nq);
      if (V == 9) bfly_v9(X[i], Y[i], w, wp, 4 * q, nq);
      if (V == 14) bfly_v14(X[i], Y[i], w, wp, q, q2, nq);
      if (V == 15) bfly_v15(X[i], Y[i], w, wp, q2, sb);
      if (V == 16) bfly_v16(X[i], Y[i], w, wp, q2, sb, s28);
    }
  }
  long long t1 = clock64();
  for (int i = 0; i < 4; ++i) { out[gid * 8 + 2 * i] = X[i]; out[gid * 8 + 2 * i + 1] = Y[i]; }
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}


// V10: hybrid integer/FP64 butterfly.  t = Y w mod q with Y = yh 2^32 + yl:
//   P = yl w + yh w2 (w2 = w 2^32 mod q), Q = round(P/q - 0.75) from DFMA with
//   f = w/q, f2 = w2/q (|error| < 2^-18, so Q in {floor(P/q)-1, floor(P/q)}),
//   r = P - Q q computed exactly mod 2^64 in [0, 2q).
__device__ __forceinline__ double u32_to_f64(uint32_t x) {
#ifdef HYB_I2F
  return __uint2double_rn(x);
#else
  return __hiloint2double(0x43300000, (int)x) - 4503599627370496.0;
#endif
}
__device__ __forceinline__ void bfly_v10(u64& X, u64& Y, u64 w, u64 w2, double f, double f2, u64 q2, u64 nq) {
  const uint32_t yl = (uint32_t)Y, yh = (uint32_t)(Y >> 32);
  const double dl = u32_to_f64(yl), dh = u32_to_f64(yh);
  const double qf = fma(dh, f2, fma(dl, f, -0.75));
  const double t = qf + 6755399441055744.0;              // 1.5 * 2^52: low mantissa bits = round(qf)
  const u64 Qb = (u64)__double_as_longlong(t);
  const uint32_t Q0 = (uint32_t)Qb, Q1 = (uint32_t)(Qb >> 32) & 1u;
  u64 r = (u64)yl * w + (u64)yh * w2 + (u64)Q0 * nq + ((u64)(Q1 ? (uint32_t)nq : 0u) << 32);
  const bool big = (uint32_t)(X >> 32) > (uint32_t)(q2 >> 32);
  const u64 x = X - (big ? q2 : 0ull);
  X = x + r;
  Y = x + q2 - r;
}

template <int V, int ILP>
__global__ void k_bfly_h(u64* out, const u64* in, u64 w, u64 w2, double f, double f2, u64 q, long long* cyc) {
  u64 X[ILP], Y[ILP];
  const int gid = blockIdx.x * blockDim.x + threadIdx.x;
  for (int i = 0; i < ILP; ++i) { X[i] = in[(gid * 2 * ILP + 2 * i) % (1 << 20)]; Y[i] = in[(gid * 2 * ILP + 2 * i + 1) % (1 << 20)]; }
  const u64 q2 = 2 * q, nq = 0ull - q;
  const u64 wp = (u64)w2;  // unused for V10
  long long t0 = clock64();
  for (int it = 0; it < 256; ++it) {
#pragma unroll
    for (int i = 0; i < ILP; ++i) {
      if (V == 10) bfly_v10(X[i], Y[i], w, w2, f, f2, q2, nq);
      else bfly_v0(X[i], Y[i], w, (u64)f2 /*wp passed via f2 bits below*/, q, q2, nq);
    }
  }
  long long t1 = clock64();
  for (int i = 0; i < ILP; ++i) { out[gid * 2 * ILP + 2 * i] = X[i]; out[gid * 2 * ILP + 2 * i + 1] = Y[i]; }
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
  (void)wp;
}

__global__ void k_dfma(double* out, double a, double b, long long* cyc) {
  double x[8];
  for (int i = 0; i < 8; ++i) x[i] = threadIdx.x + i;
  long long t0 = clock64();
  for (int it = 0; it < 1024; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i) x[i] = fma(x[i], a, b);
  }
  long long t1 = clock64();
  double s = 0; for (int i = 0; i < 8; ++i) s += x[i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}


// V12: exact Shoup, every product a mul.wide/mul.lo with a zero addend (no
// 64-bit register-pair addends), every sum a 32-bit carry chain.
__device__ __forceinline__ void bfly_v12(uint32_t& x0, uint32_t& x1, uint32_t& y0, uint32_t& y1, uint32_t w0,
                                         uint32_t w1, uint32_t p0, uint32_t p1, uint32_t n0, uint32_t n1,
                                         uint32_t q20, uint32_t q21) {
  uint32_t X0, X1, Y0, Y1;
  asm("{\n\t"
      ".reg .u32 A, Bl, Bh, Cl, Ch, Dl, Dh, s, Q0, Q1, El, Eh, Fl, Fh, t1, t2, r0, r1, s0, s1, a0, a1;\n\t"
      ".reg .u64 B, C, D, E, F;\n\t"
      ".reg .pred big;\n\t"
      "mul.hi.u32 A, %4, %10;\n\t"
      "mul.wide.u32 B, %4, %11;\n\t"
      "mul.wide.u32 C, %5, %10;\n\t"
      "mul.wide.u32 D, %5, %11;\n\t"
      "mov.b64 {Bl, Bh}, B;\n\t"
      "mov.b64 {Cl, Ch}, C;\n\t"
      "mov.b64 {Dl, Dh}, D;\n\t"
      "add.cc.u32 s, A, Bl;\n\t"
      "addc.cc.u32 Q0, Dl, Bh;\n\t"
      "addc.u32 Q1, Dh, 0;\n\t"
      "add.cc.u32 s, s, Cl;\n\t"
      "addc.cc.u32 Q0, Q0, Ch;\n\t"
      "addc.u32 Q1, Q1, 0;\n\t"
      "mul.wide.u32 E, %4, %8;\n\t"
      "mul.wide.u32 F, Q0, %12;\n\t"
      "mov.b64 {El, Eh}, E;\n\t"
      "mov.b64 {Fl, Fh}, F;\n\t"
      "mad.lo.u32 t1, %4, %9, Eh;\n\t"
      "mad.lo.u32 t1, %5, %8, t1;\n\t"
      "mad.lo.u32 t2, Q0, %13, Fh;\n\t"
      "mad.lo.u32 t2, Q1, %12, t2;\n\t"
      "add.cc.u32 r0, El, Fl;\n\t"
      "addc.u32 r1, t1, t2;\n\t"
      "setp.gt.u32 big, %7, %15;\n\t"
      "selp.u32 s0, %14, 0, big;\n\t"
      "selp.u32 s1, %15, 0, big;\n\t"
      "selp.u32 a0, 0, %14, big;\n\t"
      "selp.u32 a1, 0, %15, big;\n\t"
      "sub.cc.u32 %0, %6, s0;\n\t"
      "subc.u32 %1, %7, s1;\n\t"
      "add.cc.u32 %0, %0, r0;\n\t"
      "addc.u32 %1, %1, r1;\n\t"
      "add.cc.u32 %2, %6, a0;\n\t"
      "addc.u32 %3, %7, a1;\n\t"
      "sub.cc.u32 %2, %2, r0;\n\t"
      "subc.u32 %3, %3, r1;\n\t"
      "}"
      : "=r"(X0), "=r"(X1), "=r"(Y0), "=r"(Y1)
      : "r"(y0), "r"(y1), "r"(x0), "r"(x1), "r"(w0), "r"(w1), "r"(p0), "r"(p1), "r"(n0), "r"(n1), "r"(q20),
        "r"(q21));
  x0 = X0; x1 = X1; y0 = Y0; y1 = Y1;
}

__global__ void k_bfly12(u64* out, const u64* in, u64 w, u64 wp, u64 q, long long* cyc) {
  uint32_t x0[4], x1[4], y0[4], y1[4];
  const int gid = blockIdx.x * blockDim.x + threadIdx.x;
  for (int i = 0; i < 4; ++i) {
    u64 X = in[gid * 8 + 2 * i], Y = in[gid * 8 + 2 * i + 1];
    x0[i] = (uint32_t)X; x1[i] = (uint32_t)(X >> 32); y0[i] = (uint32_t)Y; y1[i] = (uint32_t)(Y >> 32);
  }
  const u64 q2 = 2 * q, nq = 0ull - q;
  long long t0 = clock64();
  for (int it = 0; it < ITERS; ++it) {
#pragma unroll
    for (int i = 0; i < 4; ++i)
      bfly_v12(x0[i], x1[i], y0[i], y1[i], (uint32_t)w, (uint32_t)(w >> 32), (uint32_t)wp, (uint32_t)(wp >> 32),
               (uint32_t)nq, (uint32_t)(nq >> 32), (uint32_t)q2, (uint32_t)(q2 >> 32));
  }
  long long t1 = clock64();
  for (int i = 0; i < 4; ++i) {
    out[gid * 8 + 2 * i] = ((u64)x1[i] << 32) | x0[i];
    out[gid * 8 + 2 * i + 1] = ((u64)y1[i] << 32) | y0[i];
  }
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}


// V13: Shoup with W'' = floor(w 2^63 / q) < 2^63: the middle partial-product sum
// cannot overflow 64 bits (y < 2^62), so no carry capture is needed:
//   mid = y0 p1 + y1 p0 + hi(y0 p0);  Q = 2 y1 p1 + (mid >> 31)  (= floor(y W'' / 2^63))
__device__ __forceinline__ void bfly_v13(u64& X, u64& Y, u64 w, u64 wpp, u64 q2, u64 nq) {
  const uint32_t y0 = (uint32_t)Y, y1 = (uint32_t)(Y >> 32), p0 = (uint32_t)wpp, p1 = (uint32_t)(wpp >> 32);
  const u64 mid = (u64)y0 * p1 + (u64)y1 * p0 + __umulhi(y0, p0);
  const u64 Q = (((u64)y1 * p1) << 1) + (mid >> 31);
  const u64 T = Y * w + Q * nq;
  const u64 x = X >= q2 ? X - q2 : X;
  X = x + T;
  Y = x + q2 - T;
}

template <int V>
__global__ void k_bfly13(u64* out, const u64* in, u64 w, u64 wpp, u64 q, long long* cyc) {
  u64 X[4], Y[4];
  const int gid = blockIdx.x * blockDim.x + threadIdx.x;
  for (int i = 0; i < 4; ++i) { X[i] = in[gid * 8 + 2 * i]; Y[i] = in[gid * 8 + 2 * i + 1]; }
  const u64 q2 = 2 * q, nq = 0ull - q;
  long long t0 = clock64();
  for (int it = 0; it < ITERS; ++it) {
#pragma unroll
    for (int i = 0; i < 4; ++i) bfly_v13(X[i], Y[i], w, wpp, q2, nq);
  }
  long long t1 = clock64();
  for (int i = 0; i < 4; ++i) { out[gid * 8 + 2 * i] = X[i]; out[gid * 8 + 2 * i + 1] = Y[i]; }
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}

static u64 mulmod(u64 a, u64 b, u64 q) { return (u64)((u128)a * b % q); }

int main() {
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  const int TPB = 256, CPS = 4, grid = sms * CPS, nthr = grid * TPB;
  const u64 q = 1152921504606584833ull;  // 2^60 - 2^18 + 1
  const u64 w = 987654321987654321ull % q;
  const u64 wp = (u64)(((u128)w << 64) / q);
  u64 *din, *dout;
  long long* cyc;
  CK(cudaMalloc(&din, (size_t)nthr * 8 * 8));
  CK(cudaMalloc(&dout, (size_t)nthr * 8 * 8));
  CK(cudaMalloc(&cyc, grid * 8));
  u64* h = (u64*)malloc((size_t)nthr * 8 * 8);
  u64* ho = (u64*)malloc((size_t)nthr * 8 * 8);
  u64 s = 88172645463325252ull;
  for (size_t i = 0; i < (size_t)nthr * 8; ++i) { s ^= s << 13; s ^= s >> 7; s ^= s << 17; h[i] = s % q; }
  CK(cudaMemcpy(din, h, (size_t)nthr * 64, cudaMemcpyHostToDevice));
  long long* hc = (long long*)malloc(grid * 8);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  // host reference for 8 threads' worth of pairs
  const int NREF = 64;
  u64 refX[NREF], refY[NREF];
  for (int i = 0; i < NREF; ++i) {
    u64 X = h[2 * i], Y = h[2 * i + 1];
    for (int it = 0; it < ITERS; ++it) {
      u64 t = mulmod(Y, w, q);
      u64 nx = (X + t) % q, ny = (X + q - t) % q;
      X = nx; Y = ny;
    }
    refX[i] = X; refY[i] = Y;
  }
  auto run = [&](auto kern, const char* name) {
    kern<<<grid, TPB>>>(dout, din, w, wp, q, cyc);
    cudaEventRecord(e0);
    kern<<<grid, TPB>>>(dout, din, w, wp, q, cyc);
    cudaEventRecord(e1);
    CK(cudaEventSynchronize(e1));
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    CK(cudaMemcpy(hc, cyc, grid * 8, cudaMemcpyDeviceToHost));
    CK(cudaMemcpy(ho, dout, (size_t)nthr * 64, cudaMemcpyDeviceToHost));
    long long mx = 0; double avg = 0;
    for (int i = 0; i < grid; ++i) { if (hc[i] > mx) mx = hc[i]; avg += hc[i]; }
    avg /= grid;
    int bad = 0;
    for (int i = 0; i < NREF; ++i) {
      // thread t = i/4 pair k = i%4 -> positions t*8 + 2k
      int t = i / 4, k = i % 4;
      u64 X = ho[t * 8 + 2 * k] % q, Y = ho[t * 8 + 2 * k + 1] % q;
      u64 hX = h[t * 8 + 2 * k], hY = h[t * 8 + 2 * k + 1];
      u64 rX = hX, rY = hY;
      for (int it = 0; it < ITERS; ++it) { u64 tt = mulmod(rY, w, q); u64 nx = (rX + tt) % q, ny = (rX + q - tt) % q; rX = nx; rY = ny; }
      if (X != rX || Y != rY) ++bad;
    }
    double bfly_sm = (double)ITERS * 4 * TPB * CPS;
    printf("{\"variant\":\"%s\",\"bfly_per_clk_per_sm\":%.3f,\"avg_cyc_basis\":%.3f,\"ms\":%.4f,\"mhz\":%.0f,\"bad\":%d}\n",
           name, bfly_sm / mx, bfly_sm / avg, ms, mx / (ms * 1e3), bad);
  };
  for (int rep = 0; rep < 2; ++rep) {
    run(k_bfly<0>, "V0_nvcc");
    run(k_bfly<14>, "V14_sign_csub");
    run(k_bfly<15>, "V15_sparse_q");
    run(k_bfly<16>, "V16_sparse_q_alu");
    run(k_bfly<2>, "V2_split_exact");
    run(k_bfly<3>, "V3_split_hiword");
    run(k_bfly<4>, "V4_ptx_block");
    run(k_bfly<5>, "V5_approxQ_8q");
    run(k_bfly<6>, "V6_exact_carry3");
    run(k_bfly<7>, "V7_c_nq_hiword");
    run(k_bfly<8>, "V8_c_approx");
    run(k_bfly<9>, "V9_c_approx_umulhi");
    run(k_bfly12, "V12_ptx_noaddend_hiword");
    {
      const u64 wpp = (u64)(((u128)w << 63) / q);
      auto k13 = [&](u64* o, const u64* i, u64 ww, u64 /*wp*/, u64 qq, long long* c) {};
      (void)k13;
      k_bfly13<0><<<grid, TPB>>>(dout, din, w, wpp, q, cyc);
      cudaEventRecord(e0);
      k_bfly13<0><<<grid, TPB>>>(dout, din, w, wpp, q, cyc);
      cudaEventRecord(e1);
      CK(cudaEventSynchronize(e1));
      float ms; cudaEventElapsedTime(&ms, e0, e1);
      CK(cudaMemcpy(hc, cyc, grid * 8, cudaMemcpyDeviceToHost));
      CK(cudaMemcpy(ho, dout, (size_t)nthr * 64, cudaMemcpyDeviceToHost));
      long long mx = 0; for (int i = 0; i < grid; ++i) if (hc[i] > mx) mx = hc[i];
      int bad = 0;
      for (int i = 0; i < NREF; ++i) {
        int t = i / 4, k = i % 4;
        u64 X = ho[t * 8 + 2 * k] % q, Y = ho[t * 8 + 2 * k + 1] % q;
        u64 rX = h[t * 8 + 2 * k], rY = h[t * 8 + 2 * k + 1];
        for (int it = 0; it < ITERS; ++it) { u64 tt = mulmod(rY, w, q); u64 nx = (rX + tt) % q, ny = (rX + q - tt) % q; rX = nx; rY = ny; }
        if (X != rX || Y != rY) ++bad;
      }
      if (rep) printf("{\"variant\":\"V13_half_scale_shoup\",\"bfly_per_clk_per_sm\":%.3f,\"ms\":%.4f,\"bad\":%d}\n", 256.0 * 4 * TPB * CPS / mx, ms, bad);
    }
  }
  {
    // hybrid variant
    const u64 w2 = (u64)(((u128)w << 32) % q);
    const double f = (double)w / (double)q, f2 = (double)w2 / (double)q;
    for (int rep = 0; rep < 2; ++rep) {
      k_bfly_h<10, 4><<<grid, TPB>>>(dout, din, w, w2, f, f2, q, cyc);
      cudaEventRecord(e0);
      k_bfly_h<10, 4><<<grid, TPB>>>(dout, din, w, w2, f, f2, q, cyc);
      cudaEventRecord(e1);
      CK(cudaEventSynchronize(e1));
      float ms; cudaEventElapsedTime(&ms, e0, e1);
      CK(cudaMemcpy(hc, cyc, grid * 8, cudaMemcpyDeviceToHost));
      CK(cudaMemcpy(ho, dout, (size_t)nthr * 64, cudaMemcpyDeviceToHost));
      long long mx = 0; for (int i = 0; i < grid; ++i) if (hc[i] > mx) mx = hc[i];
      int bad = 0;
      for (int i = 0; i < 256; ++i) {
        int t = i / 4, k = i % 4;
        u64 X = ho[t * 8 + 2 * k] % q, Y = ho[t * 8 + 2 * k + 1] % q;
        u64 rX = h[t * 8 + 2 * k], rY = h[t * 8 + 2 * k + 1];
        for (int it = 0; it < 256; ++it) { u64 tt = mulmod(rY, w, q); u64 nx = (rX + tt) % q, ny = (rX + q - tt) % q; rX = nx; rY = ny; }
        if (X != rX || Y != rY) ++bad;
      }
      double bfly_sm = 256.0 * 4 * TPB * CPS;
      if (rep) printf("{\"variant\":\"V10_hybrid_fp64\",\"bfly_per_clk_per_sm\":%.3f,\"ms\":%.4f,\"bad\":%d}\n", bfly_sm / mx, ms, bad);
    }
    // throughput at ILP 8 (no correctness check; 8 pairs per thread, half the CTAs)
    u64* dout2; CK(cudaMalloc(&dout2, (size_t)nthr * 16 * 8));
    auto tp = [&](auto kern, const char* name, double fa) {
      const int g2 = grid / 2;
      for (int rep = 0; rep < 2; ++rep) {
        kern<<<g2, TPB>>>(dout2, din, w, w2, f, fa, q, cyc);
        CK(cudaDeviceSynchronize());
      }
      CK(cudaMemcpy(hc, cyc, g2 * 8, cudaMemcpyDeviceToHost));
      long long mx = 0; for (int i = 0; i < g2; ++i) if (hc[i] > mx) mx = hc[i];
      printf("{\"variant\":\"%s\",\"bfly_per_clk_per_sm\":%.3f}\n", name, 256.0 * 8 * TPB * (CPS / 2) / mx);
    };
    tp(k_bfly_h<10, 8>, "V10_hybrid_ILP8", f2);
    double wpd; { u64 wpv = wp; memcpy(&wpd, &wpv, 8); }
    tp(k_bfly_h<0, 8>, "V0_ILP8(wp garbage ok for tput)", 12345.0);
    double* dd; CK(cudaMalloc(&dd, (size_t)nthr * 8));
    for (int rep = 0; rep < 2; ++rep) {
      k_dfma<<<grid, TPB>>>(dd, 1.0000001, 1e-9, cyc);
      CK(cudaDeviceSynchronize());
      CK(cudaMemcpy(hc, cyc, grid * 8, cudaMemcpyDeviceToHost));
      long long mx = 0; for (int i = 0; i < grid; ++i) if (hc[i] > mx) mx = hc[i];
      if (rep) printf("{\"kernel\":\"DFMA\",\"ops_per_clk_per_sm\":%.2f}\n", 1024.0 * 8 * TPB * CPS / mx);
    }
  }
  (void)refX; (void)refY;
  return 0;
}
