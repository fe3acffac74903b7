// plan.h -- host-side plan builder (prime / root validation, twiddle tables
// with Shoup companions, N^{-1} and Montgomery constants).  Independent
// implementation: shares no code with oracle/ (test infrastructure).
#pragma once
#include <cstdint>
#include <string>
#include <vector>

namespace rnt {

struct HostTW {
  uint64_t w, wp;
};

struct HostLimb {
  uint64_t q = 0, psi = 0;
  uint64_t q2 = 0, qinv = 0, r2 = 0;
  HostTW ninv{}, ninv_w1{}, ninvR{}, ninvR_w1{};
};

// Status codes mirror rnt_status (include/rnsntt.h).
enum PlanErr { PLAN_OK = 0, PLAN_E_ARG = 1, PLAN_E_N = 2, PLAN_E_MODULUS = 3, PLAN_E_ROOT = 4 };

uint64_t hp_mulmod(uint64_t a, uint64_t b, uint64_t q);
uint64_t hp_powmod(uint64_t a, uint64_t e, uint64_t q);
bool hp_is_prime(uint64_t n);
uint64_t hp_smallest_psi(uint64_t q, uint32_t logn);
uint32_t hp_bitrev(uint32_t x, uint32_t bits);

// Validate moduli / psi and fill per-limb constants.
int plan_limbs(uint32_t logn, uint32_t L, const uint64_t* moduli, const uint64_t* psi,
               std::vector<HostLimb>& out);

// Natural-index twiddle powers: tab[i] = (psi or psi^{-1})^{brv_n(i)}, i < count,
// each with its Shoup companion.
void plan_powers(const HostLimb& lm, uint32_t logn, bool inverse, uint32_t count, HostTW* tab);

// Kernel layouts (see ntt_small.cuh / ntt_large.cuh): N <= 2^10 uses the
// natural order; N >= 2^11 uses a lane-major row layout (k_row), a natural
// per-row layout (k_rows) and the first 2^{n1} natural entries (columns).
void plan_row_layout(const HostTW* natural, uint32_t logn, HostTW* out);
// Natural per-row layout for the warp-engine row kernel (k_rows):
// out[r 2^{n2} + 2^v + j] = natural[2^{n1+v} + r 2^v + j].
void plan_row_natural(const HostTW* natural, uint32_t logn, HostTW* out);

}  // namespace rnt
