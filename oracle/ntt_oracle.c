/*
 * ntt_oracle.c -- plain, slow, obviously-correct CPU oracle for the batched
 * negacyclic NTT / INTT / pointwise-modmul path of arxiv 2410.05934
 * ("Chameleon"), section II.D, Eq. 1.
 *
 * TEST INFRASTRUCTURE ONLY.  Nothing in the product path (the package
 * paper_2410_05934_b200/, its CUDA kernels or its C ABI) may include, link or
 * call this file.  Only tests/, __graft_entry__.smoke() and bench.py's
 * cpu_baseline / --impl reference legs use it.  It shares no code, header,
 * table or constant generator with the CUDA path.
 *
 * Arithmetic: every modular product is the exact 128-bit product reduced with
 * the C '%' operator (no Barrett, Shoup or Montgomery), every sum is reduced
 * with '%'.  Residues are canonical in [0, q).
 *
 * Citations (P:n = PAPER.md line n, S:n = SPEC.md line n):
 *   - ring and product c(x) = a(x) b(x) mod (x^N + 1) ............ P:194
 *   - NTT^{CT,psi}_{no->bo}, INTT^{GS,psi^-1}_{bo->no}, Eq. 1 ..... P:205-213
 *   - psi: primitive 2N-th root, psi^{2N}=1, psi^i != 1 (i<2N) .... P:213
 *   - INTT includes the final N^{-1} scaling (reading C4) ......... S:165-167
 *   - choice of psi (smallest primitive root, reading C1) and of
 *     the primes (L largest q < 2^60, q = 1 mod 2N, reading C2) ... DESIGN.md
 */
#include "ntt_oracle.h"

#include <pthread.h>
#include <stdlib.h>
#include <string.h>

typedef unsigned __int128 u128;

/* ---------------------------------------------------------------- scalars */

uint64_t or_mulmod(uint64_t a, uint64_t b, uint64_t q) {
  return (uint64_t)(((u128)a * (u128)b) % (u128)q);
}

uint64_t or_addmod(uint64_t a, uint64_t b, uint64_t q) {
  return (uint64_t)(((u128)a + (u128)b) % (u128)q);
}

uint64_t or_submod(uint64_t a, uint64_t b, uint64_t q) {
  return (uint64_t)(((u128)a + (u128)q - (u128)b) % (u128)q);
}

uint64_t or_powmod(uint64_t base, uint64_t e, uint64_t q) {
  uint64_t r = 1 % q, b = base % q;
  while (e) {
    if (e & 1) r = or_mulmod(r, b, q);
    b = or_mulmod(b, b, q);
    e >>= 1;
  }
  return r;
}

/* Deterministic Miller-Rabin; bases 2..37 are exact for all n < 2^64. */
int or_is_prime(uint64_t n) {
  static const uint64_t bases[12] = {2, 3, 5, 7, 11, 13, 17, 19, 23, 29, 31, 37};
  if (n < 2) return 0;
  for (int i = 0; i < 12; ++i) {
    if (n == bases[i]) return 1;
    if (n % bases[i] == 0) return 0;
  }
  uint64_t d = n - 1;
  int s = 0;
  while ((d & 1) == 0) { d >>= 1; ++s; }
  for (int i = 0; i < 12; ++i) {
    uint64_t x = or_powmod(bases[i], d, n);
    if (x == 1 || x == n - 1) continue;
    int composite = 1;
    for (int r = 1; r < s; ++r) {
      x = or_mulmod(x, x, n);
      if (x == n - 1) { composite = 0; break; }
    }
    if (composite) return 0;
  }
  return 1;
}

/* bit reversal of the low logn bits of i */
uint32_t or_brv(uint32_t i, uint32_t logn) {
  uint32_t r = 0;
  for (uint32_t b = 0; b < logn; ++b) r |= ((i >> b) & 1u) << (logn - 1 - b);
  return r;
}

/* psi is a primitive 2N-th root of unity mod q: psi^{2N} = 1 and
 * psi^i != 1 for 0 < i < 2N.  For N a power of two this is psi^N = q - 1. */
int or_is_primitive_2n_root(uint64_t psi, uint64_t q, uint32_t logn) {
  uint64_t n = (uint64_t)1 << logn;
  if (psi == 0 || psi >= q) return 0;
  return or_powmod(psi, n, q) == q - 1;
}

/* Reading C1: the numerically smallest primitive 2N-th root of unity.
 * Step 1: find any primitive root r = x^{(q-1)/2N} with r^N = -1.
 * Step 2: the primitive 2N-th roots are exactly r^{2t+1}, t in [0,N);
 *         enumerate them by repeated multiplication with r^2, keep the min. */
uint64_t or_min_psi(uint64_t q, uint32_t logn) {
  uint64_t n = (uint64_t)1 << logn, two_n = n << 1;
  if ((q - 1) % two_n != 0) return 0;
  uint64_t r = 0;
  for (uint64_t x = 2; x < q; ++x) {
    uint64_t c = or_powmod(x, (q - 1) / two_n, q);
    if (or_powmod(c, n, q) == q - 1) { r = c; break; }
  }
  if (r == 0) return 0;
  uint64_t r2 = or_mulmod(r, r, q), cur = r, best = r;
  for (uint64_t t = 0; t < n; ++t) {
    if (cur < best) best = cur;
    cur = or_mulmod(cur, r2, q);
  }
  return best;
}

/* Reading C2: the L largest primes q < 2^60 with q = 1 (mod 2N), descending. */
int or_primes(uint32_t logn, uint32_t count, uint64_t* out) {
  uint64_t two_n = (uint64_t)2 << logn;
  uint64_t k = (((uint64_t)1 << 60) - 1) / two_n; /* largest k with k*2N+1 < 2^60 */
  uint32_t found = 0;
  while (found < count && k > 0) {
    uint64_t q = k * two_n + 1;
    if (q < ((uint64_t)1 << 60) && or_is_prime(q)) out[found++] = q;
    --k;
  }
  return found == count ? 0 : -1;
}

/* ---------------------------------------------------------------- tables */

/* fwd[i] = psi^{brv(i)}, inv[i] = (psi^{-1})^{brv(i)}, ninv = N^{-1} mod q
 * (the twiddle tables the Longa-Naehrig CT/GS loops below index). */
void or_tables(uint64_t q, uint64_t psi, uint32_t logn, uint64_t* fwd, uint64_t* inv,
               uint64_t* ninv) {
  uint64_t n = (uint64_t)1 << logn;
  uint64_t psi_inv = or_powmod(psi, q - 2, q); /* Fermat: q prime */
  for (uint64_t i = 0; i < n; ++i) {
    uint32_t e = or_brv((uint32_t)i, logn);
    fwd[i] = or_powmod(psi, e, q);
    inv[i] = or_powmod(psi_inv, e, q);
  }
  *ninv = or_powmod(n % q, q - 2, q);
}

/* ------------------------------------------------------------- transforms */

/* NTT^{CT,psi}_{no->bo} (Eq. 1): Cooley-Tukey butterflies,
 * natural-order input, bit-reversed-order output, in place. */
void or_ntt_fwd(uint64_t* a, uint32_t logn, uint64_t q, const uint64_t* fwd) {
  uint64_t n = (uint64_t)1 << logn;
  uint64_t t = n;
  for (uint64_t m = 1; m < n; m <<= 1) {
    t >>= 1;
    for (uint64_t i = 0; i < m; ++i) {
      uint64_t S = fwd[m + i];
      uint64_t j1 = 2 * i * t;
      for (uint64_t j = j1; j < j1 + t; ++j) {
        uint64_t U = a[j];
        uint64_t V = or_mulmod(a[j + t], S, q);
        a[j] = or_addmod(U, V, q);
        a[j + t] = or_submod(U, V, q);
      }
    }
  }
}

/* INTT^{GS,psi^-1}_{bo->no} (Eq. 1): Gentleman-Sande
 * butterflies, bit-reversed input, natural output, then x N^{-1}. */
void or_ntt_inv(uint64_t* a, uint32_t logn, uint64_t q, const uint64_t* inv, uint64_t ninv) {
  uint64_t n = (uint64_t)1 << logn;
  uint64_t t = 1;
  for (uint64_t m = n; m > 1; m >>= 1) {
    uint64_t h = m >> 1, j1 = 0;
    for (uint64_t i = 0; i < h; ++i) {
      uint64_t S = inv[h + i];
      for (uint64_t j = j1; j < j1 + t; ++j) {
        uint64_t U = a[j];
        uint64_t V = a[j + t];
        a[j] = or_addmod(U, V, q);
        a[j + t] = or_mulmod(or_submod(U, V, q), S, q);
      }
      j1 += 2 * t;
    }
    t <<= 1;
  }
  for (uint64_t j = 0; j < n; ++j) a[j] = or_mulmod(a[j], ninv, q);
}

/* The (.) of Eq. 1: c_k = a_k * b_k mod q. */
void or_pointwise(uint64_t* c, const uint64_t* a, const uint64_t* b, uint64_t n, uint64_t q) {
  for (uint64_t k = 0; k < n; ++k) c[k] = or_mulmod(a[k], b[k], q);
}

/* ----------------------------------------------------------- definitions */

/* The plain definition the CT loop computes: output slot k is
 * the evaluation of a at the root psi^{2 brv(k) + 1} of x^N + 1:
 *   NTT(a)[k] = sum_i a_i * psi^{(2 brv(k) + 1) i}  mod q.   O(N) per k. */
uint64_t or_naive_ntt_at(const uint64_t* a, uint32_t logn, uint64_t q, uint64_t psi, uint32_t k) {
  uint64_t n = (uint64_t)1 << logn;
  uint64_t zeta = or_powmod(psi, 2 * (uint64_t)or_brv(k, logn) + 1, q);
  uint64_t acc = 0, pw = 1;
  for (uint64_t i = 0; i < n; ++i) {
    acc = or_addmod(acc, or_mulmod(a[i], pw, q), q);
    pw = or_mulmod(pw, zeta, q);
  }
  return acc;
}

void or_naive_ntt(uint64_t* out, const uint64_t* a, uint32_t logn, uint64_t q, uint64_t psi) {
  uint64_t n = (uint64_t)1 << logn;
  for (uint64_t k = 0; k < n; ++k) out[k] = or_naive_ntt_at(a, logn, q, psi, (uint32_t)k);
}

/* Inverse of the definition above: a_i = N^{-1} sum_k A[k] psi^{-(2 brv(k)+1) i}. */
uint64_t or_naive_intt_at(const uint64_t* A, uint32_t logn, uint64_t q, uint64_t psi, uint32_t i) {
  uint64_t n = (uint64_t)1 << logn;
  uint64_t psi_inv = or_powmod(psi, q - 2, q);
  uint64_t acc = 0;
  for (uint64_t k = 0; k < n; ++k) {
    uint64_t e = ((2 * (uint64_t)or_brv((uint32_t)k, logn) + 1) * (uint64_t)i) % (2 * n);
    acc = or_addmod(acc, or_mulmod(A[k], or_powmod(psi_inv, e, q), q), q);
  }
  return or_mulmod(acc, or_powmod(n % q, q - 2, q), q);
}

/* Schoolbook negacyclic product:
 *   c_k = sum_{i+j=k} a_i b_j - sum_{i+j=k+N} a_i b_j  mod q.   O(N) per k. */
uint64_t or_schoolbook_at(const uint64_t* a, const uint64_t* b, uint32_t logn, uint64_t q, uint32_t k) {
  uint64_t n = (uint64_t)1 << logn;
  uint64_t acc = 0;
  for (uint64_t i = 0; i < n; ++i) {
    if (i <= k) {
      acc = or_addmod(acc, or_mulmod(a[i], b[k - i], q), q);
    } else {
      acc = or_submod(acc, or_mulmod(a[i], b[n + k - i], q), q);
    }
  }
  return acc;
}

void or_schoolbook(uint64_t* c, const uint64_t* a, const uint64_t* b, uint32_t logn, uint64_t q) {
  uint64_t n = (uint64_t)1 << logn;
  for (uint64_t k = 0; k < n; ++k) c[k] = or_schoolbook_at(a, b, logn, q, (uint32_t)k);
}

/* Galois automorphism (Automorph):
 * sigma_g(a)(x) = a(x^g) mod (x^N + 1) for odd g: coefficient i goes to
 * i g mod 2N, negated when that exponent is >= N (x^N = -1). */
void or_automorph(uint64_t* out, const uint64_t* a, uint32_t logn, uint64_t q, uint64_t g) {
  uint64_t n = (uint64_t)1 << logn;
  for (uint64_t i = 0; i < n; ++i) {
    uint64_t t = (i * g) % (2 * n);
    if (t < n) out[t] = a[i] % q;
    else out[t - n] = or_submod(0, a[i] % q, q);
  }
}

/* Signed gadget decomposition (Decompose), reading G1:
 * centre v in (-q/2, q/2]; digits d_0..d_{l-2} balanced in [-B/2, B/2),
 * d_{l-1} takes the rest; sum_j d_j B^j = centred v exactly when B^l >= q.
 * Digits are returned as residues mod q. */
void or_decompose(uint64_t* digits, uint64_t v, uint64_t q, uint32_t base_log2, uint32_t levels) {
  int64_t vc = (v > (q - 1) / 2) ? (int64_t)v - (int64_t)q : (int64_t)v;
  const int64_t B = (int64_t)1 << base_log2;
  for (uint32_t j = 0; j < levels; ++j) {
    int64_t d;
    if (j + 1 < levels) {
      d = vc % B;               /* C remainder has the sign of vc */
      if (d < 0) d += B;        /* mathematical vc mod B, in [0, B) */
      if (d >= B / 2) d -= B;   /* balanced, in [-B/2, B/2) */
      vc = (vc - d) / B;        /* exact division */
    } else {
      d = vc;                   /* last level keeps the remainder */
    }
    digits[j] = d >= 0 ? (uint64_t)d % q : q - (uint64_t)(-d) % q;
  }
}

/* External product of TFHE (CMux building block):
 * c = (c_0, c_1) an RLWE pair, rgsw_hat[r][i] (r < 2l, i < 2) RGSW rows in NTT
 * form (the order of or_ntt_fwd).  D_{t,j} = digit j of c_t; r = t l + j;
 *   out_i = INTT( sum_r NTT(D_r) (.) rgsw_hat[r][i] ),  i = 0, 1.
 * c and out are [2][N]; rgsw_hat is [2l][2][N]. */
void or_external_product(uint64_t* out, const uint64_t* c, const uint64_t* rgsw_hat, uint32_t logn, uint64_t q,
                         uint64_t psi, uint32_t base_log2, uint32_t levels) {
  uint64_t n = (uint64_t)1 << logn;
  uint64_t* fwd = (uint64_t*)malloc(n * sizeof(uint64_t));
  uint64_t* inv = (uint64_t*)malloc(n * sizeof(uint64_t));
  uint64_t ninv;
  or_tables(q, psi, logn, fwd, inv, &ninv);
  uint64_t* acc = (uint64_t*)calloc(2 * n, sizeof(uint64_t));
  uint64_t* dig = (uint64_t*)malloc((size_t)levels * n * sizeof(uint64_t));
  uint64_t* tmp = (uint64_t*)malloc(levels * sizeof(uint64_t));
  for (uint32_t t = 0; t < 2; ++t) {
    for (uint64_t k = 0; k < n; ++k) {
      or_decompose(tmp, c[t * n + k], q, base_log2, levels);
      for (uint32_t j = 0; j < levels; ++j) dig[j * n + k] = tmp[j];
    }
    for (uint32_t j = 0; j < levels; ++j) {
      uint64_t* D = dig + (uint64_t)j * n;
      or_ntt_fwd(D, logn, q, fwd);
      uint64_t r = (uint64_t)t * levels + j;
      for (uint32_t i = 0; i < 2; ++i)
        for (uint64_t k = 0; k < n; ++k)
          acc[i * n + k] = or_addmod(acc[i * n + k], or_mulmod(D[k], rgsw_hat[(r * 2 + i) * n + k], q), q);
    }
  }
  for (uint32_t i = 0; i < 2; ++i) {
    or_ntt_inv(acc + i * n, logn, q, inv, ninv);
    memcpy(out + i * n, acc + i * n, n * sizeof(uint64_t));
  }
  free(fwd); free(inv); free(acc); free(dig); free(tmp);
}

/* HRF-MatVec, the homomorphic-rotation-free matrix-vector product of repack
 * (tab:repack P:393-395, row HRF-MatVec: 0 rotations, n_slot scalar
 * multiplications, n_slot precomputed rotation ciphertexts).
 * With every rotation ciphertext ct_j = rot_j(Enc(s)) precomputed and every
 * plaintext diagonal pt_j (giant-step automorph already applied) in
 * NTT form, the linear transformation is a sum of scalar (plaintext-ciphertext)
 * products, per RNS limb l, component c and NTT slot k (reading H1):
 *   out[c][l][k] = add[c][l][k] + sum_{j < n_slot} pt[j][l][k] * ct[j][c][l][k]  mod q_l
 * pt [n_slot][L][N], ct [n_slot][2][L][N], add [2][L][N] or NULL (the "+ b" of
 * As + b), out [2][L][N]. */
void or_hrf_matvec(uint64_t* out, const uint64_t* pt, const uint64_t* ct, const uint64_t* add, uint32_t n_slot,
                   const uint64_t* q, uint32_t L, uint64_t n) {
  for (uint32_t c = 0; c < 2; ++c)
    for (uint32_t l = 0; l < L; ++l)
      for (uint64_t k = 0; k < n; ++k) {
        uint64_t acc = add ? add[((uint64_t)c * L + l) * n + k] % q[l] : 0;
        for (uint32_t j = 0; j < n_slot; ++j) {
          uint64_t a = pt[((uint64_t)j * L + l) * n + k];
          uint64_t b = ct[(((uint64_t)j * 2 + c) * L + l) * n + k];
          acc = or_addmod(acc, or_mulmod(a, b, q[l]), q[l]);
        }
        out[((uint64_t)c * L + l) * n + k] = acc;
      }
}

/* Fast basis conversion BConv (CKKS key switching ModUp / ModDown, P:247-248;
 * SPEC S:82-90): from basis Q = {q_0..q_{L-1}} to P = {p_0..p_{K-1}},
 * per coefficient (reading G3):
 *   y_i   = x_i * (Q/q_i)^{-1} mod q_i
 *   out_j = sum_i y_i * (Q/q_i mod p_j) mod p_j      (= X + alpha Q mod p_j, 0 <= alpha < L)
 * in: [L][N] residues, out: [K][N]. */
void or_bconv(uint64_t* out, const uint64_t* in, uint64_t n, const uint64_t* q, uint32_t L, const uint64_t* p,
              uint32_t K) {
  uint64_t* qhat_inv = (uint64_t*)malloc(L * sizeof(uint64_t));
  uint64_t* qhat_p = (uint64_t*)malloc((size_t)L * K * sizeof(uint64_t));
  for (uint32_t i = 0; i < L; ++i) {
    uint64_t h = 1 % q[i];
    for (uint32_t k = 0; k < L; ++k)
      if (k != i) h = or_mulmod(h, q[k] % q[i], q[i]);
    qhat_inv[i] = or_powmod(h, q[i] - 2, q[i]);
    for (uint32_t j = 0; j < K; ++j) {
      uint64_t hp = 1 % p[j];
      for (uint32_t k = 0; k < L; ++k)
        if (k != i) hp = or_mulmod(hp, q[k] % p[j], p[j]);
      qhat_p[(size_t)i * K + j] = hp;
    }
  }
  uint64_t* y = (uint64_t*)malloc(L * sizeof(uint64_t));
  for (uint64_t c = 0; c < n; ++c) {
    for (uint32_t i = 0; i < L; ++i) y[i] = or_mulmod(in[(size_t)i * n + c], qhat_inv[i], q[i]);
    for (uint32_t j = 0; j < K; ++j) {
      uint64_t acc = 0;
      for (uint32_t i = 0; i < L; ++i)
        acc = or_addmod(acc, or_mulmod(y[i] % p[j], qhat_p[(size_t)i * K + j], p[j]), p[j]);
      out[(size_t)j * n + c] = acc;
    }
  }
  free(qhat_inv); free(qhat_p); free(y);
}

/* CKKS hybrid key switching ("critical key switching ... NTT,
 * BConv, ModMul, ModAdd, Automorph"; parameters (N, L, dnum) of
 * P:831).  The paper gives no algorithm text; readings KS1-KS4
 * fix the standard hybrid method, which this function follows step by step:
 *   Q = {q_0..q_{L-1}}, P = {p_0..p_{K-1}}, extended basis QP = Q then P.
 *   digits (KS2): alpha = ceil(L / dnum); digit j = limbs [j alpha, min(L, (j+1) alpha)).
 *   1. x = INTT_Q(d)                                  (d in NTT form over Q)
 *   2. for each digit j: ModUp  e_j[t] = BConv_{D_j -> t}(x[D_j]) for t not in D_j,
 *                               e_j[t] = x[t] for t in D_j;  then NTT_t(e_j[t])
 *   3. u_k[t] = sum_j e_j[t] * evk[j][k][t]  (k = 0, 1; NTT form over QP)
 *   4. ModDown (KS3): w = BConv_{P -> Q}(INTT_P(u_k[P])), NTT_Q(w),
 *                     out_k[i] = (u_k[i] - w[i]) * P^{-1} mod q_i   (+ add0 for k = 0)
 * psi of every prime: reading C1 (or_min_psi).  evk: [dnum][2][L+K][N], out: [2][L][N],
 * add0: [L][N] or NULL.  All in NTT form (bit-reversed order, reading C3). */
void or_keyswitch(uint64_t* out, const uint64_t* d, const uint64_t* evk, const uint64_t* add0, uint32_t logn,
                  const uint64_t* q, uint32_t L, const uint64_t* p, uint32_t K, uint32_t dnum) {
  const uint64_t n = (uint64_t)1 << logn;
  const uint32_t LK = L + K, alpha = (L + dnum - 1) / dnum;
  uint64_t* mod = (uint64_t*)malloc(LK * sizeof(uint64_t));
  for (uint32_t t = 0; t < L; ++t) mod[t] = q[t];
  for (uint32_t t = 0; t < K; ++t) mod[L + t] = p[t];
  uint64_t* fwd = (uint64_t*)malloc((size_t)LK * n * sizeof(uint64_t));
  uint64_t* inv = (uint64_t*)malloc((size_t)LK * n * sizeof(uint64_t));
  uint64_t* ninv = (uint64_t*)malloc(LK * sizeof(uint64_t));
  for (uint32_t t = 0; t < LK; ++t)
    or_tables(mod[t], or_min_psi(mod[t], logn), logn, fwd + (size_t)t * n, inv + (size_t)t * n, ninv + t);
  /* 1. coefficient form of d */
  uint64_t* x = (uint64_t*)malloc((size_t)L * n * sizeof(uint64_t));
  memcpy(x, d, (size_t)L * n * sizeof(uint64_t));
  for (uint32_t t = 0; t < L; ++t) or_ntt_inv(x + (size_t)t * n, logn, q[t], inv + (size_t)t * n, ninv[t]);
  /* 2-3. ModUp each digit, NTT, multiply-accumulate with the key */
  uint64_t* u = (uint64_t*)calloc((size_t)2 * LK * n, sizeof(uint64_t));
  uint64_t* e = (uint64_t*)malloc((size_t)LK * n * sizeof(uint64_t));
  for (uint32_t j = 0; j < dnum; ++j) {
    const uint32_t lo = j * alpha, hi = (j + 1) * alpha < L ? (j + 1) * alpha : L;
    for (uint32_t t = 0; t < LK; ++t) {
      uint64_t* et = e + (size_t)t * n;
      if (t >= lo && t < hi)
        memcpy(et, x + (size_t)t * n, n * sizeof(uint64_t));
      else
        or_bconv(et, x + (size_t)lo * n, n, q + lo, hi - lo, mod + t, 1);
      or_ntt_fwd(et, logn, mod[t], fwd + (size_t)t * n);
      for (uint32_t k = 0; k < 2; ++k) {
        const uint64_t* key = evk + (((size_t)j * 2 + k) * LK + t) * n;
        uint64_t* ut = u + ((size_t)k * LK + t) * n;
        for (uint64_t c = 0; c < n; ++c) ut[c] = or_addmod(ut[c], or_mulmod(et[c], key[c], mod[t]), mod[t]);
      }
    }
  }
  /* 4. ModDown */
  uint64_t* pinv = (uint64_t*)malloc(L * sizeof(uint64_t));
  for (uint32_t i = 0; i < L; ++i) {
    uint64_t pp = 1 % q[i];
    for (uint32_t t = 0; t < K; ++t) pp = or_mulmod(pp, p[t] % q[i], q[i]);
    pinv[i] = or_powmod(pp, q[i] - 2, q[i]);
  }
  uint64_t* up = (uint64_t*)malloc((size_t)K * n * sizeof(uint64_t));
  uint64_t* w = (uint64_t*)malloc((size_t)L * n * sizeof(uint64_t));
  for (uint32_t k = 0; k < 2; ++k) {
    memcpy(up, u + ((size_t)k * LK + L) * n, (size_t)K * n * sizeof(uint64_t));
    for (uint32_t t = 0; t < K; ++t) or_ntt_inv(up + (size_t)t * n, logn, p[t], inv + (size_t)(L + t) * n, ninv[L + t]);
    or_bconv(w, up, n, p, K, q, L);
    for (uint32_t i = 0; i < L; ++i) {
      uint64_t* wi = w + (size_t)i * n;
      or_ntt_fwd(wi, logn, q[i], fwd + (size_t)i * n);
      const uint64_t* ui = u + ((size_t)k * LK + i) * n;
      uint64_t* oi = out + ((size_t)k * L + i) * n;
      for (uint64_t c = 0; c < n; ++c) {
        oi[c] = or_mulmod(or_submod(ui[c], wi[c], q[i]), pinv[i], q[i]);
        if (k == 0 && add0) oi[c] = or_addmod(oi[c], add0[(size_t)i * n + c], q[i]);
      }
    }
  }
  free(mod); free(fwd); free(inv); free(ninv); free(x); free(u); free(e); free(pinv); free(up); free(w);
}

/* ---------------------------------------------------------- batch driver */
/* Layout (reading C10): [batch][n_limbs][N], limb l uses moduli[l], psi[l].
 * op: 0 forward, 1 inverse, 2 polymul-with-eval-operand c = INTT(NTT(a) . b_hat),
 *     3 full polymul c = INTT(NTT(a) . NTT(b)).  b is [b_batch][n_limbs][N]
 *     with b_batch in {1, batch} (1 = broadcast). */

typedef struct {
  uint64_t* data;
  const uint64_t* b;
  uint32_t batch, n_limbs, logn, b_bcast;
  const uint64_t* moduli;
  uint64_t** fwd;
  uint64_t** inv;
  const uint64_t* ninv;
  int op;
  uint64_t unit_begin, unit_end;
} or_job;

static void run_unit(const or_job* J, uint64_t u, uint64_t* scratch) {
  uint64_t n = (uint64_t)1 << J->logn;
  uint32_t l = (uint32_t)(u % J->n_limbs);
  uint64_t bidx = u / J->n_limbs;
  uint64_t q = J->moduli[l];
  uint64_t* a = J->data + u * n;
  if (J->op == 0) {
    or_ntt_fwd(a, J->logn, q, J->fwd[l]);
  } else if (J->op == 1) {
    or_ntt_inv(a, J->logn, q, J->inv[l], J->ninv[l]);
  } else {
    const uint64_t* b = J->b + ((J->b_bcast ? 0 : bidx) * J->n_limbs + l) * n;
    or_ntt_fwd(a, J->logn, q, J->fwd[l]);
    if (J->op == 3) {
      memcpy(scratch, b, n * sizeof(uint64_t));
      or_ntt_fwd(scratch, J->logn, q, J->fwd[l]);
      b = scratch;
    }
    or_pointwise(a, a, b, n, q);
    or_ntt_inv(a, J->logn, q, J->inv[l], J->ninv[l]);
  }
}

static void* run_job(void* arg) {
  const or_job* J = (const or_job*)arg;
  uint64_t n = (uint64_t)1 << J->logn;
  uint64_t* scratch = (uint64_t*)malloc(n * sizeof(uint64_t));
  for (uint64_t u = J->unit_begin; u < J->unit_end; ++u) run_unit(J, u, scratch);
  free(scratch);
  return NULL;
}

int or_batch(int op, uint64_t* data, const uint64_t* b, int b_bcast, uint32_t batch,
             uint32_t n_limbs, uint32_t logn, const uint64_t* moduli, const uint64_t* psi,
             int n_threads) {
  uint64_t n = (uint64_t)1 << logn;
  uint64_t units = (uint64_t)batch * n_limbs;
  if (units == 0) return 0;
  uint64_t** fwd = (uint64_t**)calloc(n_limbs, sizeof(uint64_t*));
  uint64_t** inv = (uint64_t**)calloc(n_limbs, sizeof(uint64_t*));
  uint64_t* ninv = (uint64_t*)calloc(n_limbs, sizeof(uint64_t));
  for (uint32_t l = 0; l < n_limbs; ++l) {
    fwd[l] = (uint64_t*)malloc(n * sizeof(uint64_t));
    inv[l] = (uint64_t*)malloc(n * sizeof(uint64_t));
    or_tables(moduli[l], psi[l], logn, fwd[l], inv[l], &ninv[l]);
  }
  if (n_threads < 1) n_threads = 1;
  if ((uint64_t)n_threads > units) n_threads = (int)units;
  pthread_t* th = (pthread_t*)calloc((size_t)n_threads, sizeof(pthread_t));
  or_job* jobs = (or_job*)calloc((size_t)n_threads, sizeof(or_job));
  for (int t = 0; t < n_threads; ++t) {
    or_job J = {data, b, batch, n_limbs, logn, (uint32_t)b_bcast, moduli, fwd, inv, ninv, op,
                units * (uint64_t)t / (uint64_t)n_threads,
                units * (uint64_t)(t + 1) / (uint64_t)n_threads};
    jobs[t] = J;
    pthread_create(&th[t], NULL, run_job, &jobs[t]);
  }
  for (int t = 0; t < n_threads; ++t) pthread_join(th[t], NULL);
  for (uint32_t l = 0; l < n_limbs; ++l) { free(fwd[l]); free(inv[l]); }
  free(fwd); free(inv); free(ninv); free(th); free(jobs);
  return 0;
}
