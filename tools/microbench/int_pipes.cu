// Microbenchmark: integer-pipe throughput on sm_100a (B200), used to pin the
// INT32 roofline that bounds the modular butterflies.
//
// Each kernel runs 148*k CTAs of 512 threads; every thread keeps 8 independent
// dependency chains so issue, not latency, is the limit.  Per-CTA cycle counts
// come from clock64(); ops/clk/SM = total ops / (max CTA cycles * CTAs-per-SM) / 148
// is reported together with wall time (CUDA events) so the clock can be inferred.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("CUDA %s at %d\n", cudaGetErrorString(e), __LINE__); return 1; } } while (0)

constexpr int ITERS = 2048;
constexpr int ILP = 8;

__global__ void k_imad(uint32_t* out, uint32_t a, uint32_t b, long long* cyc) {
  uint32_t x[ILP];
  for (int i = 0; i < ILP; ++i) x[i] = threadIdx.x + i;
  long long t0 = clock64();
  for (int it = 0; it < ITERS; ++it) {
#pragma unroll
    for (int i = 0; i < ILP; ++i) asm volatile("mad.lo.u32 %0, %0, %1, %2;" : "+r"(x[i]) : "r"(a), "r"(b));
  }
  long long t1 = clock64();
  uint32_t s = 0; for (int i = 0; i < ILP; ++i) s ^= x[i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}

__global__ void k_imadhi(uint32_t* out, uint32_t a, uint32_t b, long long* cyc) {
  uint32_t x[ILP];
  for (int i = 0; i < ILP; ++i) x[i] = threadIdx.x + i;
  long long t0 = clock64();
  for (int it = 0; it < ITERS; ++it) {
#pragma unroll
    for (int i = 0; i < ILP; ++i) asm volatile("mad.hi.u32 %0, %0, %1, %2;" : "+r"(x[i]) : "r"(a), "r"(b));
  }
  long long t1 = clock64();
  uint32_t s = 0; for (int i = 0; i < ILP; ++i) s ^= x[i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}

__global__ void k_imadwide(uint32_t* out, uint32_t a, uint32_t b, long long* cyc) {
  uint64_t x[ILP];
  for (int i = 0; i < ILP; ++i) x[i] = threadIdx.x + i;
  long long t0 = clock64();
  for (int it = 0; it < ITERS; ++it) {
#pragma unroll
    for (int i = 0; i < ILP; ++i) {
      uint32_t lo = (uint32_t)x[i];
      asm volatile("mad.wide.u32 %0, %1, %2, %0;" : "+l"(x[i]) : "r"(lo), "r"(a));
    }
  }
  long long t1 = clock64();
  uint32_t s = 0; for (int i = 0; i < ILP; ++i) s ^= (uint32_t)(x[i] ^ (x[i] >> 32));
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}

__global__ void k_iadd3(uint32_t* out, uint32_t a, uint32_t b, long long* cyc) {
  uint32_t x[ILP];
  for (int i = 0; i < ILP; ++i) x[i] = threadIdx.x + i;
  long long t0 = clock64();
  for (int it = 0; it < ITERS; ++it) {
#pragma unroll
    for (int i = 0; i < ILP; ++i) asm volatile("add.u32 %0, %0, %1;" : "+r"(x[i]) : "r"(a));
  }
  long long t1 = clock64();
  uint32_t s = 0; for (int i = 0; i < ILP; ++i) s ^= x[i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}

// mixed: one IMAD and one IADD per step on independent chains (dual-pipe issue check)
__global__ void k_mix(uint32_t* out, uint32_t a, uint32_t b, long long* cyc) {
  uint32_t x[ILP], y[ILP];
  for (int i = 0; i < ILP; ++i) { x[i] = threadIdx.x + i; y[i] = i; }
  long long t0 = clock64();
  for (int it = 0; it < ITERS; ++it) {
#pragma unroll
    for (int i = 0; i < ILP; ++i) {
      asm volatile("mad.lo.u32 %0, %0, %1, %2;" : "+r"(x[i]) : "r"(a), "r"(b));
      asm volatile("add.u32 %0, %0, %1;" : "+r"(y[i]) : "r"(a));
    }
  }
  long long t1 = clock64();
  uint32_t s = 0; for (int i = 0; i < ILP; ++i) s ^= x[i] ^ y[i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}

// Lazy Harvey CT butterfly with exact Shoup (umul64hi), values in [0,4q).
__device__ __forceinline__ void bfly_exact(uint64_t& X, uint64_t& Y, uint64_t W, uint64_t Wp, uint64_t q) {
  uint64_t q2 = q << 1;
  uint64_t x = X >= q2 ? X - q2 : X;
  uint64_t Q = __umul64hi(Y, Wp);
  uint64_t T = Y * W - Q * q;
  X = x + T;
  Y = x - T + q2;
}

// Same with an approximate high product (lo*lo partial dropped); T in [0,3q).
__device__ __forceinline__ uint64_t mulhi_approx(uint64_t a, uint64_t b) {
  uint32_t a0 = (uint32_t)a, a1 = (uint32_t)(a >> 32), b0 = (uint32_t)b, b1 = (uint32_t)(b >> 32);
  uint64_t m1 = (uint64_t)a0 * b1;
  uint64_t m2 = (uint64_t)a1 * b0;
  uint64_t hi = (uint64_t)a1 * b1;
  uint64_t mid = (m1 >> 32) + (m2 >> 32) + (((m1 & 0xffffffffu) + (m2 & 0xffffffffu)) >> 32);
  return hi + mid;
}

template <int V>
__global__ void k_bfly(uint64_t* out, uint64_t W, uint64_t Wp, uint64_t q, long long* cyc) {
  uint64_t X[4], Y[4];
  for (int i = 0; i < 4; ++i) { X[i] = threadIdx.x * 977 + i; Y[i] = blockIdx.x * 131 + i * 7; }
  long long t0 = clock64();
  for (int it = 0; it < ITERS / 4; ++it) {
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      if (V == 0) bfly_exact(X[i], Y[i], W, Wp, q);
      else {
        uint64_t q2 = q << 1;
        uint64_t x = X[i] >= q2 ? X[i] - q2 : X[i];
        uint64_t Q = mulhi_approx(Y[i], Wp);
        uint64_t T = Y[i] * W - Q * q;
        T = T >= q2 ? T - q2 : T;
        X[i] = x + T;
        Y[i] = x - T + q2;
      }
    }
  }
  long long t1 = clock64();
  uint64_t s = 0; for (int i = 0; i < 4; ++i) s ^= X[i] ^ Y[i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}

__global__ void k_copy(const uint4* __restrict__ a, uint4* __restrict__ b, size_t n) {
  size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x, st = (size_t)gridDim.x * blockDim.x;
  for (; i < n; i += st) b[i] = a[i];
}

int main() {
  cudaDeviceProp p; CK(cudaGetDeviceProperties(&p, 0));
  int clk = 0; cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  printf("{\"device\":\"%s\",\"sm\":%d,\"cc\":\"%d.%d\",\"l2_bytes\":%d,\"smem_per_sm\":%zu,\"smem_optin\":%zu,\"regs_per_sm\":%d,\"clock_khz\":%d,\"mem_bus_bits\":%d}\n",
         p.name, p.multiProcessorCount, p.major, p.minor, p.l2CacheSize, p.sharedMemPerMultiprocessor,
         p.sharedMemPerBlockOptin, p.regsPerMultiprocessor, clk, p.memoryBusWidth);
  const int SMS = p.multiProcessorCount;
  const int TPB = 512, CPS = 2;  // 2 CTAs of 512 threads per SM = 32 warps
  const int grid = SMS * CPS;
  uint32_t* o32; uint64_t* o64; long long* cyc;
  CK(cudaMalloc(&o32, grid * TPB * 4)); CK(cudaMalloc(&o64, grid * TPB * 8)); CK(cudaMalloc(&cyc, grid * 8));
  long long* hc = new long long[grid];
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  auto report = [&](const char* name, double ops_per_thread, float ms) {
    cudaMemcpy(hc, cyc, grid * 8, cudaMemcpyDeviceToHost);
    long long mx = 0; double avg = 0; for (int i = 0; i < grid; ++i) { if (hc[i] > mx) mx = hc[i]; avg += hc[i]; }
    avg /= grid;
    double ops_sm = ops_per_thread * TPB * CPS;
    printf("{\"kernel\":\"%s\",\"ops_per_clk_per_sm\":%.2f,\"ops_per_clk_per_sm_avgcyc\":%.2f,\"ms\":%.4f,\"implied_mhz\":%.0f}\n",
           name, ops_sm / mx, ops_sm / avg, ms, mx / (ms * 1e3));
  };
  for (int rep = 0; rep < 2; ++rep) {
#define RUN(K, name, ops, ...) { K<<<grid, TPB>>>(__VA_ARGS__); cudaEventRecord(e0); K<<<grid, TPB>>>(__VA_ARGS__); cudaEventRecord(e1); CK(cudaEventSynchronize(e1)); float ms; cudaEventElapsedTime(&ms, e0, e1); if (rep) report(name, ops, ms); }
    RUN(k_imad, "IMAD", (double)ITERS * ILP, o32, 3u, 5u, cyc);
    RUN(k_imadhi, "IMAD.HI", (double)ITERS * ILP, o32, 3u, 5u, cyc);
    RUN(k_imadwide, "IMAD.WIDE", (double)ITERS * ILP, o32, 3u, 5u, cyc);
    RUN(k_iadd3, "IADD", (double)ITERS * ILP, o32, 3u, 5u, cyc);
    RUN(k_mix, "IMAD+IADD(pairs)", (double)ITERS * ILP * 2, o32, 3u, 5u, cyc);
    const uint64_t q = 1152921504606584833ull, W = 123456789012345ull;
    const uint64_t Wp = (uint64_t)(((unsigned __int128)W << 64) / q);
    RUN(k_bfly<0>, "bfly_exact(bfly/clk/SM)", (double)(ITERS / 4) * 4, o64, W, Wp, q, cyc);
    RUN(k_bfly<1>, "bfly_approx(bfly/clk/SM)", (double)(ITERS / 4) * 4, o64, W, Wp, q, cyc);
  }
  // HBM copy
  size_t n = (size_t)1 << 30;  // 1 GiB each
  uint4 *a, *b; CK(cudaMalloc(&a, n)); CK(cudaMalloc(&b, n));
  cudaMemset(a, 1, n);
  float best = 1e9;
  for (int r = 0; r < 6; ++r) {
    cudaEventRecord(e0); k_copy<<<SMS * 8, 512>>>(a, b, n / 16); cudaEventRecord(e1); cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1); if (r && ms < best) best = ms;
  }
  printf("{\"kernel\":\"copy_1GiB\",\"GBps\":%.1f}\n", 2.0 * n / (best * 1e6));
  return 0;
}
