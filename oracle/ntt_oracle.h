/* ntt_oracle.h -- CPU oracle (TEST INFRASTRUCTURE ONLY; see ntt_oracle.c).
 * Private to oracle/: the product's include/ never includes this file. */
#ifndef NTT_ORACLE_H
#define NTT_ORACLE_H
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

uint64_t or_mulmod(uint64_t a, uint64_t b, uint64_t q);
uint64_t or_addmod(uint64_t a, uint64_t b, uint64_t q);
uint64_t or_submod(uint64_t a, uint64_t b, uint64_t q);
uint64_t or_powmod(uint64_t base, uint64_t e, uint64_t q);
int or_is_prime(uint64_t n);
uint32_t or_brv(uint32_t i, uint32_t logn);
int or_is_primitive_2n_root(uint64_t psi, uint64_t q, uint32_t logn);
uint64_t or_min_psi(uint64_t q, uint32_t logn);
int or_primes(uint32_t logn, uint32_t count, uint64_t* out);
void or_tables(uint64_t q, uint64_t psi, uint32_t logn, uint64_t* fwd, uint64_t* inv, uint64_t* ninv);
void or_ntt_fwd(uint64_t* a, uint32_t logn, uint64_t q, const uint64_t* fwd);
void or_ntt_inv(uint64_t* a, uint32_t logn, uint64_t q, const uint64_t* inv, uint64_t ninv);
void or_pointwise(uint64_t* c, const uint64_t* a, const uint64_t* b, uint64_t n, uint64_t q);
uint64_t or_naive_ntt_at(const uint64_t* a, uint32_t logn, uint64_t q, uint64_t psi, uint32_t k);
void or_naive_ntt(uint64_t* out, const uint64_t* a, uint32_t logn, uint64_t q, uint64_t psi);
uint64_t or_naive_intt_at(const uint64_t* A, uint32_t logn, uint64_t q, uint64_t psi, uint32_t i);
uint64_t or_schoolbook_at(const uint64_t* a, const uint64_t* b, uint32_t logn, uint64_t q, uint32_t k);
void or_schoolbook(uint64_t* c, const uint64_t* a, const uint64_t* b, uint32_t logn, uint64_t q);
void or_automorph(uint64_t* out, const uint64_t* a, uint32_t logn, uint64_t q, uint64_t g);
void or_decompose(uint64_t* digits, uint64_t v, uint64_t q, uint32_t base_log2, uint32_t levels);
void or_external_product(uint64_t* out, const uint64_t* c, const uint64_t* rgsw_hat, uint32_t logn, uint64_t q,
                         uint64_t psi, uint32_t base_log2, uint32_t levels);
void or_hrf_matvec(uint64_t* out, const uint64_t* pt, const uint64_t* ct, const uint64_t* add, uint32_t n_slot,
                   const uint64_t* q, uint32_t L, uint64_t n);
void or_bconv(uint64_t* out, const uint64_t* in, uint64_t n, const uint64_t* q, uint32_t L, const uint64_t* p,
              uint32_t K);
void or_keyswitch(uint64_t* out, const uint64_t* d, const uint64_t* evk, const uint64_t* add0, uint32_t logn,
                  const uint64_t* q, uint32_t L, const uint64_t* p, uint32_t K, uint32_t dnum);
int or_batch(int op, uint64_t* data, const uint64_t* b, int b_bcast, uint32_t batch,
             uint32_t n_limbs, uint32_t logn, const uint64_t* moduli, const uint64_t* psi,
             int n_threads);

#ifdef __cplusplus
}
#endif
#endif
