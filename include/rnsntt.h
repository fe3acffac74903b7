/*
 * rnsntt.h -- C ABI of the B200-native batched negacyclic NTT library
 * (librnsntt.so, package paper_2410_05934_b200).
 *
 * The operation is Eq. 1 of arxiv 2410.05934:
 *
 *     c = INTT^{GS,psi^-1}_{bo->no}( NTT^{CT,psi}_{no->bo}(a) (.) NTT^{CT,psi}_{no->bo}(b) )
 *
 * over R_q = Z_q[x]/(x^N + 1), applied independently to every RNS
 * limb q_l of every polynomial of a batch (RNS representation of the big
 * modulus Q; CMux-level batching of TFHE polynomials).
 *
 * Conventions fixed by DESIGN.md "Readings":
 *   C1  psi_l defaults to the numerically smallest primitive 2N-th root mod q_l.
 *   C3  forward output slot k holds the evaluation of a at psi^{2 brv(k) + 1}
 *       ("no -> bo"); the inverse takes that order back to natural.
 *   C4  the inverse includes the final N^{-1} scaling, so
 *       INTT(NTT(a)) = a.
 *   C5  residues are canonical, 0 <= r < q_l, on input and on output.
 *   C10 data layout is [batch][n_limbs][N] uint64 (limb-major, each limb is a
 *       contiguous 8N-byte vector).
 *
 * Ownership: a plan owns its device tables (allocated on the device current at
 * rnt_plan_create); the caller owns every data buffer and every stream.
 * Errors: argument and plan errors are returned synchronously, before any
 * launch, and nothing is launched.  Asynchronous device faults surface as
 * RNT_E_CUDA from a later call.  No call performs a host synchronisation.
 * No exception crosses this boundary.
 * Thread safety: a plan is immutable after creation and may be used from
 * several host threads and streams concurrently.
 */
#ifndef RNSNTT_H
#define RNSNTT_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct rnt_plan_s* rnt_plan;

typedef enum {
  RNT_OK = 0,
  RNT_E_INVALID_ARG = 1,   /* null pointer, n_limbs == 0, size overflow, pointer not 16-byte aligned */
  RNT_E_UNSUPPORTED_N = 2, /* log2n outside [RNT_MIN_LOG2N, RNT_MAX_LOG2N] */
  RNT_E_MODULUS = 3,       /* q not prime, q != 1 mod 2N, q >= 2^62, or duplicate moduli */
  RNT_E_ROOT = 4,          /* caller-supplied psi is not a primitive 2N-th root of unity mod q */
  RNT_E_PLAN_MISMATCH = 5, /* current device differs from the plan's device */
  RNT_E_CUDA = 6,          /* a CUDA runtime call failed; see rnt_last_cuda_error() */
  RNT_E_OOM = 7            /* device or host allocation failed */
} rnt_status;

/* Residue precondition (reading C6): every input residue of limb l must be
 * canonical, 0 <= r < q_l.  The hot path does not check it (a violation gives
 * undefined output).  With the environment variable RNT_DEBUG=1 set when the
 * library first runs an operation, rnt_ntt_forward / rnt_ntt_inverse /
 * rnt_pointwise_mul / rnt_polymul / rnt_automorph validate their inputs on
 * the device first, synchronise `stream`, and return RNT_E_INVALID_ARG (no
 * output written) if any residue is out of range. */

/* Dispatch test hooks (read once per process; defaults are the shipped
 * behaviour, the hooks exist so tests can reach every kernel instantiation):
 *   RNT_LAT_UNITS=k      N <= 2^10 jobs of <= k (poly, limb) units use the
 *                        latency engine k_lat (default 512; 256 for N = 2^10 with
 *                        every q < 2^60; 0 = never);
 *   RNT_CLUSTER_UNITS=k  jobs of <= k units use the single-launch cluster
 *                        kernels (default 2; 0 = never);
 *   RNT_LAZY=0           keep the [0, 4q) kernels even when every q < 2^60;
 *   RNT_KS_UNFUSED=1     key switching always takes the unfused path;
 *   RNT_DEBUG=1          input range validation (above). */

#define RNT_MIN_LOG2N 4u
#define RNT_MAX_LOG2N 16u
#define RNT_MAX_LIMBS 1024u

/* Build a plan for N = 2^log2n and n_limbs moduli (host array moduli[n_limbs]).
 * psi: host array [n_limbs] of primitive 2N-th roots, or NULL for reading C1.
 * device: CUDA device ordinal that will own the tables (and run the kernels).
 * Validates every modulus (prime, q = 1 mod 2N, q < 2^62, pairwise distinct)
 * and every psi (psi^N = -1 mod q); computes the bit-reversed twiddle
 * tables of psi and psi^{-1} with their Shoup companions, N^{-1} and the
 * Montgomery constants, and uploads them.  Synchronous; not on the hot path. */
rnt_status rnt_plan_create(rnt_plan* out, uint32_t log2n, uint32_t n_limbs,
                           const uint64_t* moduli, const uint64_t* psi, int device);

/* Free the plan's device tables.  The caller must ensure no work using the
 * plan is still in flight.  NULL is accepted (no-op). */
rnt_status rnt_plan_destroy(rnt_plan p);

/* Read back N, the limb count and (optionally, host array [n_limbs]) the psi
 * values the plan uses.  Any output pointer may be NULL. */
rnt_status rnt_plan_query(rnt_plan p, uint32_t* log2n, uint32_t* n_limbs, uint64_t* psi_out,
                          int* device);

/* Forward negacyclic NTT, NTT^{CT,psi}_{no->bo} of Eq. 1, of
 * every limb of `batch` polynomials.  in/out: device pointers to
 * [batch][n_limbs][N] uint64, 16-byte aligned.  out == in (in place) is
 * allowed; any other overlap is undefined.  batch == 0 is a no-op.
 * Asynchronous on `stream` (a cudaStream_t; NULL = legacy default stream). */
rnt_status rnt_ntt_forward(rnt_plan p, uint64_t* out, const uint64_t* in, uint32_t batch,
                           void* stream);

/* Inverse negacyclic NTT, INTT^{GS,psi^-1}_{bo->no} of Eq. 1
 * including the N^{-1} scaling.  Same argument rules as forward. */
rnt_status rnt_ntt_inverse(rnt_plan p, uint64_t* out, const uint64_t* in, uint32_t batch,
                           void* stream);

/* NTT-domain pointwise product, the (.) of Eq. 1 (ModMul):
 * c[b][l][k] = a_hat[b][l][k] * b_hat[b'][l][k] mod q_l, with b' = b, or
 * b' = 0 when b_broadcast != 0 (b_hat is then [n_limbs][N], reused for every
 * polynomial).  c may alias a_hat.  Device pointers, 16-byte aligned. */
rnt_status rnt_pointwise_mul(rnt_plan p, uint64_t* c, const uint64_t* a_hat,
                             const uint64_t* b_hat, uint32_t batch, int b_broadcast,
                             void* stream);

/* Negacyclic product c = a * b mod (x^N + 1) per limb by Eq. 1:
 *   b_is_eval == 0:  c = INTT(NTT(a) (.) NTT(b)), b in coefficient form;
 *   b_is_eval != 0:  c = INTT(NTT(a) (.) b), b already in NTT form (e.g. a
 *                    key held in evaluation form).
 * b may be broadcast ([n_limbs][N]) with b_broadcast != 0.  c may alias a;
 * c must not alias b.  Fused kernels: the NTT-domain intermediate never
 * leaves the SM for N <= 2^10 and never leaves the row tile for N >= 2^11. */
rnt_status rnt_polymul(rnt_plan p, uint64_t* c, const uint64_t* a, const uint64_t* b,
                       uint32_t batch, int b_is_eval, int b_broadcast, void* stream);

/* Galois automorphism sigma_g: a(x) -> a(x^g) mod (x^N + 1), g odd, 0 < g < 2N
 * (the Automorph operator of CKKS key switching / rotation; the
 * rotation-ciphertext bank of HRF-MatVec).
 *   ntt_domain == 0: coefficient form; coefficient i moves to i g mod 2N, negated
 *                    when i g mod 2N >= N.
 *   ntt_domain != 0: NTT form (the order of rnt_ntt_forward, reading C3); a pure
 *                    permutation out[k] = in[pi(k)], 2 brv(pi(k)) + 1 = (2 brv(k) + 1) g mod 2N.
 * out must not alias in (RNT_E_INVALID_ARG).  Layout, alignment, batch == 0 and
 * stream rules as rnt_ntt_forward.  Even g or g >= 2N: RNT_E_INVALID_ARG. */
rnt_status rnt_automorph(rnt_plan p, uint64_t* out, const uint64_t* in, uint32_t batch, uint32_t galois_elt,
                         int ntt_domain, void* stream);

/* TFHE external product, batched over ciphertexts (P:164-166,
 * CMux-level batching P:312-332).  Plan: 2^4 <= N <= 2^10 and n_limbs == 1
 * (one NTT prime, reading C9).  For every slot s:
 *   out[s][i] = INTT( sum_{t<2, j<l} NTT(D_{t,j}(c[s][t])) (.) rgsw_hat[t l + j][i] ),  i = 0, 1,
 * with D_{t,j} the signed gadget digit j (base 2^base_log2, l = levels) of the
 * centred coefficients of c[s][t] (digits j < l-1 balanced in [-B/2, B/2), the
 * last keeps the remainder; exact when B^l >= q, reading G1 of DESIGN.md).
 * c, out: device [n_slot][2][N]; rgsw_hat: device [2 l][2][N] in NTT form
 * (rnt_ntt_forward order), shared by all slots.  out must not alias c.
 * base_log2 in [1, 31], levels in [1, 8], base_log2 * (levels - 1) < 63. */
rnt_status rnt_external_product(rnt_plan p, uint64_t* out, const uint64_t* c, const uint64_t* rgsw_hat,
                                uint32_t n_slot, uint32_t base_log2, uint32_t levels, void* stream);

/* Fast basis conversion BConv (CKKS key switching ModUp / ModDown, P:247-248;
 * SPEC S:82-90) from the basis Q of plan `from` (L limbs) to
 * the basis P of plan `to` (K limbs), same N and device.  Per coefficient:
 *   y_i = x_i (Q/q_i)^{-1} mod q_i,   out_j = sum_i y_i (Q/q_i mod p_j) mod p_j
 * (= X + alpha Q mod p_j with X the CRT value and 0 <= alpha < L).  Coefficient
 * form in and out: in [batch][L][N], out [batch][K][N], device, 16-byte aligned,
 * out must not alias in.  The context owns its device tables; L <= 192. */
typedef struct rnt_bconv_s* rnt_bconv;
rnt_status rnt_bconv_create(rnt_bconv* out, rnt_plan from, rnt_plan to);
rnt_status rnt_bconv_destroy(rnt_bconv c);
rnt_status rnt_bconv_apply(rnt_bconv c, uint64_t* out, const uint64_t* in, uint32_t batch, void* stream);

/* CKKS hybrid key switching: "critical key switching" built
 * from NTT, BConv, ModMul and ModAdd, at the paper's parameters
 * (N, L, dnum) = (2^16, 44, 45) or any other.  Readings KS1-KS4
 * fix the method the paper leaves unstated:
 *   Q = q_plan's moduli (L limbs); qp_plan's moduli = Q followed by the
 *   special primes P (K = n_limbs(qp_plan) - L >= 1), same N, same psi on Q.
 *   Digits: alpha = ceil(L / dnum) primes each, digit j = limbs
 *   [j alpha, min(L, (j+1) alpha)), every digit non-empty.
 *   apply:  x = INTT_Q(d);  for each digit j: e_j = ModUp(x[D_j]) over QP
 *           (BConv from the digit's primes to all other primes of QP),
 *           NTT_QP(e_j);  u_k = sum_j e_j (.) evk[j][k] (k = 0, 1);
 *           out_k = (u_k[Q] - NTT_Q(BConv_{P->Q}(INTT_P(u_k[P])))) P^{-1} mod q_i,
 *           plus add0 on out_0 when add0 != NULL.
 * d:    device [L][N], NTT form over Q (e.g. c_1 of a ciphertext, after an
 *       automorphism for a rotation).
 * evk:  device [dnum][2][L+K][N], NTT form over QP (the switching key rows).
 * add0: device [L][N] NTT form over Q, or NULL (HROT adds sigma(c_0) here).
 * out:  device [2][L][N], NTT form over Q; must not overlap the inputs.
 * The handle borrows both plans (keep them alive) and owns a device workspace
 * of rnt_keyswitch_query(...workspace_bytes) bytes, allocated at create; one
 * apply runs at a time per handle (serialised on the host; calls on different
 * streams are ordered by the caller).  Requires dnum * max(m)^2 < 2^128
 * (exact 128-bit key inner product).  Errors: RNT_E_INVALID_ARG (plans do not
 * match, dnum out of range, null/unaligned pointers), RNT_E_PLAN_MISMATCH,
 * RNT_E_CUDA / RNT_E_OOM. */
typedef struct rnt_keyswitch_s* rnt_keyswitch;
rnt_status rnt_keyswitch_create(rnt_keyswitch* out, rnt_plan q_plan, rnt_plan qp_plan, uint32_t dnum);
rnt_status rnt_keyswitch_destroy(rnt_keyswitch ks);
rnt_status rnt_keyswitch_query(rnt_keyswitch ks, uint32_t* alpha, uint64_t* workspace_bytes);
rnt_status rnt_keyswitch_apply(rnt_keyswitch ks, uint64_t* out, const uint64_t* d, const uint64_t* evk,
                               const uint64_t* add0, void* stream);

/* HRF-MatVec, the homomorphic-rotation-free matrix-vector product of repack
 * (tab:repack P:393-395: 0 rotations, n_slot scalar
 * multiplications over n_slot precomputed rotation ciphertexts).  In the NTT
 * domain, for every component c < 2, limb l and slot k (reading H1):
 *   out[c][l][k] = add[c][l][k] + sum_{j < n_slot} pt[j][l][k] * ct[j][c][l][k]  mod q_l
 * pt:  device [n_slot][n_limbs][N], plaintext diagonals (giant-step automorph
 *      already applied), NTT form, canonical;
 * ct:  device [n_slot][2][n_limbs][N], rotation ciphertexts, NTT form, canonical;
 * add: device [2][n_limbs][N] (the "+ b" of As + b) or NULL (= 0); may equal
 *      out (accumulate in place);
 * out: device [2][n_limbs][N], canonical; must not overlap pt or ct.
 * All pointers 16-byte aligned.  n_slot == 0 writes add (or zeros).  Argument
 * errors (null / unaligned pointers, overlap, size overflow) return
 * RNT_E_INVALID_ARG before any launch.  One launch, asynchronous on `stream`. */
rnt_status rnt_hrf_matvec(rnt_plan p, uint64_t* out, const uint64_t* pt, const uint64_t* ct, uint32_t n_slot,
                          const uint64_t* add, void* stream);

/* Operation codes for rnt_execute_host. */
typedef enum {
  RNT_OP_FORWARD = 0,
  RNT_OP_INVERSE = 1,
  RNT_OP_POLYMUL_EVAL = 2, /* c = INTT(NTT(a) (.) b_dev), b_dev device-resident NTT-form operand */
  RNT_OP_POLYMUL = 3       /* c = INTT(NTT(a) (.) NTT(b_dev)), b_dev device-resident coefficients */
} rnt_op;

/* End-to-end convenience over HOST buffers: copies in_host (pinned host
 * memory recommended) to the device workspace dev_ws, runs `op`, and copies
 * the result to out_host, all asynchronously on `stream`.  dev_ws: caller-
 * owned device buffer of batch*n_limbs*N uint64.  b_dev: device operand for
 * the polymul ops (ignored otherwise).  The caller synchronises the stream
 * before reading out_host. */
rnt_status rnt_execute_host(rnt_plan p, rnt_op op, uint64_t* out_host, const uint64_t* in_host,
                            uint64_t* dev_ws, const uint64_t* b_dev, uint32_t batch,
                            int b_broadcast, void* stream);

/* Human-readable name of a status code (static storage). */
const char* rnt_status_string(rnt_status s);

/* The cudaError_t of the last RNT_E_CUDA / RNT_E_OOM returned on this host thread. */
int rnt_last_cuda_error(void);

/* Number of kernels the library launched since process start (all threads);
 * used by bench.py to report gpu_launches. */
uint64_t rnt_launch_count(void);

#ifdef __cplusplus
}
#endif
#endif /* RNSNTT_H */
