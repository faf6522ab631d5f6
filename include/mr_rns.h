/*
 * mr_rns.h — C ABI of the B200-native MR-MOD / MR-RSA hot path of Chauvet & Mahé,
 * "Secrets from the GPU" (arXiv:1305.3699).  Citations: PAPER.md line numbers (P:n), section in
 * brackets; readings (R#) where the paper is silent.
 *
 * What the library computes (the paper's MR-MOD layer, §3.1, and the MR-RSA kernels,
 * P:50-56 §3.2-§3.3): batched modular exponentiation x^E mod N where every bignum lives in the
 * Residue Number System over two 32-bit prime bases B, B' plus the extra modulus m_r = 2^32,
 * and every multiply is an RNS Montgomery multiplication with R = M = prod(B) ([Bajard2001])
 * whose two base extensions B -> B' ∪ {m_r} and B' -> B carry all cross-channel work.  The results
 * are exact integers: bit-identical to x^E mod N computed any other way.
 *
 * Conventions shared by every entry point
 *  - Big integers are little-endian arrays of uint32_t limbs, fixed width per call (R16).
 *  - Batch buffers (d_*) are DEVICE pointers owned by the caller (e.g. torch tensors), row-major
 *    [count][limbs], 4-byte aligned (16-byte alignment is faster).  Host pointers are marked HOST.
 *  - Every batch call except mr_rsa_keygen_batch is asynchronous on `stream` (a cudaStream_t passed
 *    as void*; NULL = legacy default stream) and returns after enqueuing.  The return code reports
 *    host-detectable problems only (arguments, capacity, launch failure) and never synchronises the
 *    device.  mr_rsa_keygen_batch is synchronous (its search schedule depends on device results).
 *  - Per-message data errors go to d_status[i] (nullable): MR_OK, or MR_ERR_RANGE when the input is
 *    >= its bound, in which case that output is zero-filled.
 *  - count = 0 is MR_OK and launches nothing.
 *  - Contexts are immutable after creation and may be used concurrently from any host thread or
 *    stream (also several batches of one context at once: the persistent kernels never wait for a CTA
 *    that has not started).  Scratch memory is allocated stream-ordered (cudaMallocAsync)
 *    inside each call.  Exception to "never synchronises": the first call with a new exponent on a
 *    context uploads its ladder program (one small copy on a private stream that the host waits for;
 *    the first 64 programs per context are cached, later ones are uploaded and freed stream-ordered).
 *  - There is no CPU fallback: on a machine without a usable CUDA device every call returns
 *    MR_ERR_CUDA.
 */
#ifndef MR_RNS_H
#define MR_RNS_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct mr_rns_ctx mr_rns_ctx;   /* modulus N + base pair (B, B', m_r) + device constants */
typedef struct mr_rsa_priv mr_rsa_priv; /* RSA private key for CRT decryption (two half contexts) */

enum {
    MR_OK = 0,
    MR_ERR_ARG = 1,          /* null pointer, bad size, unsupported k, exponent/limb count invalid */
    MR_ERR_EVEN_MODULUS = 2, /* N even or N < 3: R = M is odd, so Montgomery needs N odd */
    MR_ERR_NOT_COPRIME = 3,  /* N shares a prime with B ∪ B' (gcd(N, M M') != 1)                  */
    MR_ERR_CAPACITY = 4,     /* N too large for the requested k (bound of DESIGN.md §3, R5)        */
    MR_ERR_RANGE = 5,        /* per-message: input >= bound                                        */
    MR_ERR_CUDA = 6,         /* CUDA runtime error or no device                                    */
    MR_ERR_NOMEM = 7         /* host or device allocation failed                                   */
};

enum { MR_COMPOSITE = 0, MR_PROBABLY_PRIME = 1, MR_FACTOR = 2 }; /* Miller-Rabin verdicts */

/* ------------------------------------------------------------------------------------------
 * mr_rns_ctx_create — precompute and install the RNS/Montgomery constants for modulus N.
 *   "these constants are pre-computed and installed permanently in GPU memory at initialization
 *    time" (§3.1).
 * modulus: HOST, `limbs` limbs, odd, N >= 3.
 * k: channels per base.  0 = auto = the smallest compiled k with 4(k+3)^2 N < M and
 *    4(k+3) N < M' (e.g. 33 for 1024-bit, 65 for 2048-bit, 257 for 8192-bit, 505 for 16,128-bit N).
 *    A nonzero k is rounded up to the next compiled k (see mr_rns_supported_k); below the bound ->
 *    MR_ERR_CAPACITY.  k <= 65: tensor-core base extensions; 97, 129, 257, 505: the wide-operand
 *    channels-on-threads kernel ("keys up to 16,128 bits"; §8(f)).
 * device: CUDA ordinal that will run every batch call on this context.
 * On success *out owns host and device memory until mr_rns_ctx_destroy.
 * Errors: MR_ERR_ARG, MR_ERR_EVEN_MODULUS, MR_ERR_NOT_COPRIME, MR_ERR_CAPACITY, MR_ERR_CUDA,
 *         MR_ERR_NOMEM.  *out is NULL on error.
 * ------------------------------------------------------------------------------------------ */
int mr_rns_ctx_create(mr_rns_ctx **out, const uint32_t *modulus, size_t limbs, int k, int device);
void mr_rns_ctx_destroy(mr_rns_ctx *ctx);

/* k actually used; limbs of N; max_modulus_bits = the largest b such that every odd N < 2^b passes this
 * k's admission test (4 K_B^2 N < M and 4 K_B N < M', DESIGN.md §3 / R5: the enforced capacity, SURVEY
 * §8(b)); bits(N); and the paper's nominal key-size cap k*31 bits for k 32-bit primes ("128 32-bit prime
 * integers, sufficient for RSA keys up to 3,968-bit"; R4, reported for reference only).
 * Any out pointer may be NULL. */
int mr_rns_ctx_info(const mr_rns_ctx *ctx, int *k, size_t *limbs, int *max_modulus_bits, int *modulus_bits,
                    int *paper_cap_bits);

/* Writes up to `cap` compiled channel counts k (ascending) into ks (HOST); returns how many exist. */
int mr_rns_supported_k(int *ks, int cap);

/* ------------------------------------------------------------------------------------------
 * mr_modexp_batch — d_y[i] = d_x[i]^E mod N for i < count (§3.1: "exponentiation,
 * implemented with traditional square-and-multiply algorithms ... chaining Montgomery modular
 * multiplications"; here a sliding window, reading R6).
 * d_x, d_y: DEVICE [count][limbs(N)].  d_x[i] must be < N, else d_status[i] = MR_ERR_RANGE and
 *           d_y[i] = 0.  d_y may alias d_x.
 * exp: HOST, exp_limbs limbs, shared by the whole batch; any length (R7: exponents longer than N
 *      are computed literally); E = 0 gives 1.
 * d_status: DEVICE int32 [count] or NULL.
 * ------------------------------------------------------------------------------------------ */
int mr_modexp_batch(const mr_rns_ctx *ctx, const uint32_t *d_x, uint32_t *d_y, size_t count,
                    const uint32_t *exp, size_t exp_limbs, int32_t *d_status, void *stream);

/* mr_rsa_encrypt_batch — c = m^e mod N (§3.3 "two GPU kernels respectively for encryption
 * and decryption of messages, applying modular exponentiation").  Same contract as
 * mr_modexp_batch with E = e. */
int mr_rsa_encrypt_batch(const mr_rns_ctx *n_ctx, const uint32_t *e, size_t e_limbs, const uint32_t *d_m,
                         uint32_t *d_c, size_t count, int32_t *d_status, void *stream);

/* ------------------------------------------------------------------------------------------
 * mr_rsa_priv_create — private key for CRT decryption (north_star; Garner recombination, HAC 14.71;
 * the paper mentions p/q splitting only in related work).
 * p, q, d_p = d mod (p-1), d_q = d mod (q-1), q_inv = q^-1 mod p: HOST, half_limbs limbs each.
 * The two half contexts share one base pair; k_half = 0 picks it automatically.
 * Ciphertexts and plaintexts of mr_rsa_decrypt_batch have 2*half_limbs limbs and must be < p*q.
 * Errors as mr_rns_ctx_create, plus MR_ERR_ARG if p == q or q_inv*q != 1 mod p.  Halves above ~4,070
 * bits run on the wide kernel with a positional recombination (keys up to 16,128 bits).
 * ------------------------------------------------------------------------------------------ */
int mr_rsa_priv_create(mr_rsa_priv **out, const uint32_t *p, const uint32_t *q, size_t half_limbs,
                       const uint32_t *d_p, const uint32_t *d_q, const uint32_t *q_inv, int k_half, int device);
void mr_rsa_priv_destroy(mr_rsa_priv *priv);

/* mr_rsa_decrypt_batch — d_m[i] = d_c[i]^d mod pq by CRT: m_p = c^d_p mod p, m_q = c^d_q mod q
 * (two half-size RNS ladders in one launch), h = q_inv (m_p - m_q) mod p, m = m_q + q h.
 * d_c, d_m: DEVICE [count][2*half_limbs]; d_c[i] >= pq -> MR_ERR_RANGE.  d_m may alias d_c. */
int mr_rsa_decrypt_batch(const mr_rsa_priv *priv, const uint32_t *d_c, uint32_t *d_m, size_t count,
                         int32_t *d_status, void *stream);

/* ------------------------------------------------------------------------------------------
 * mr_miller_rabin_batch — Miller-Rabin in the Montgomery domain, one candidate per message
 * ("primality testing in the Montgomery domain has been implemented as a dedicated GPU kernel ...
 *  a Miller-Rabin test with a user-parameterized number of iterations", §3.2; HAC 4.24).
 * d_n: DEVICE [count][limbs] candidates; d_bases: DEVICE [count][rounds][limbs], each in [2, n-2]
 *      (bases are inputs, reading R13).
 * k: channels (0 = auto from limbs; candidates up to 504 limbs = 16,128 bits, else MR_ERR_CAPACITY): k <= 65 tensor-core
 *    rounds, 97 / 129 the per-k IMAD kernel, 257 / 505 (4,097 .. 16,128-bit candidates) the channels-on-threads kernels
 *    with a per-candidate setup.
 * d_verdict: DEVICE uint8 [count] = MR_COMPOSITE |
 * MR_PROBABLY_PRIME | MR_FACTOR (n > 2^32 divisible by a prime of B ∪ B', R14).
 * d_witness_round: DEVICE int16 [count] or NULL: first round that proved compositeness, else -1.
 * d_status: DEVICE int32 [count] or NULL: MR_ERR_RANGE if n even, n < 5 or a base outside
 *           [2, n-2]; MR_ERR_NOT_COPRIME if n < 2^32 is itself a base prime.
 * ------------------------------------------------------------------------------------------ */
int mr_miller_rabin_batch(const uint32_t *d_n, size_t limbs, size_t count, const uint32_t *d_bases, int rounds,
                          int k, uint8_t *d_verdict, int16_t *d_witness_round, int32_t *d_status, int device,
                          void *stream);

/* ------------------------------------------------------------------------------------------
 * mr_rsa_keygen_batch — RSA key generation on the GPU ("RSA key generation ... is completely
 * performed on the GPU with only e ... and N being transferred back to the CPU host", §3.3;
 * "small primes testing (up to the first 10,000 primes) combined with Miller-Rabin compositeness
 * tests", §4.3; d, d_p, d_q by Arazi's inversion, §3.1).
 * Key i (global index first_key + i) follows the recipe of DESIGN.md reading R19: attempt a draws
 * start = odd_with_top_bits(bits/2, seed, TAG_KEY, (first_key + i) * 65536 + a) (synth/ SplitMix64
 * stream); its prime is the first probable prime >= start that survives trial division by the odd
 * primes among the first 10,000 and `rounds` Miller-Rabin rounds with bases 2, 3, 5, ... (the first
 * `rounds` primes).  Primes with gcd(e, p - 1) != 1, and a second prime q with |p - q| <= 2^(bits/2-100),
 * are skipped; p is the first accepted prime, q the second.
 * bits: multiple of 64 in [256, 4096]; e: an odd prime < 2^32 (e.g. 65537); rounds in [1, 256].
 * Outputs, DEVICE, little-endian 32-bit limbs: d_n, d_d [count][bits/32] (n = p q, d = e^-1 mod
 * (p-1)(q-1)); d_p, d_q, d_dp, d_dq, d_qinv [count][bits/64] (d_p = d mod (p-1), d_q = d mod (q-1),
 * q_inv = q^-1 mod p).  Synchronous: returns after the keys are in the output buffers (the host
 * schedules the search from per-search flags it reads back; no key material leaves the device).
 * Errors: MR_ERR_ARG (bad bits/e/rounds/count, NULL output), MR_ERR_RANGE (a key needed more than
 * 65,536 prime searches), MR_ERR_CUDA, MR_ERR_NOMEM.
 * WARNING — DETERMINISTIC FIXTURE RECIPE, NOT FOR PRODUCTION KEYS: every prime follows from the 64-bit
 * `seed` through SplitMix64 (not a cryptographic generator) and the Miller-Rabin bases are the fixed
 * primes 2, 3, 5, ...; anyone who knows or guesses the seed can regenerate p, q and d.  It exists so the
 * GPU pipeline can be checked limb for limb against the oracle's fixture keys.  Real keys:
 * mr_rsa_keygen_batch_drbg (below, after the DRBG declarations).
 * ------------------------------------------------------------------------------------------ */
int mr_rsa_keygen_batch(size_t count, int bits, uint32_t e, uint64_t seed, uint64_t first_key, int rounds,
                        uint32_t *d_n, uint32_t *d_p, uint32_t *d_q, uint32_t *d_d, uint32_t *d_dp, uint32_t *d_dq,
                        uint32_t *d_qinv, int device, void *stream);

/* Human-readable name of an MR_* code (static storage). */
/* ------------------------------------------------------------------------------------------
 * DRBG + FIPS 140-2 health tests (the MR-TRNG layer's deterministic half).
 * "The unpredictable stream of bits is seeded as an unguessable input key to an approved deterministic
 *  RBG" (§2); "a self-validating kernel ... streamlines FIPS basic tests right after the generation"
 *  (§4.2).  Entropy harvesting is out of scope: the caller supplies entropy_input and nonce.
 * Reading R20: Hash_DRBG with SHA-256 (NIST SP 800-90A §10.1.1, seedlen 440, no additional input, no
 * prediction resistance), `streams` independent instances; stream s is instantiated with
 * personalization_string = pers || s (4 bytes big-endian).
 *
 * mr_drbg_create: entropy (HOST, >= 32 bytes), nonce (HOST, >= 16 bytes), pers (HOST, may be empty).
 *   Errors: MR_ERR_ARG (short entropy/nonce, streams == 0), MR_ERR_CUDA, MR_ERR_NOMEM.
 * mr_drbg_generate: one Hash_DRBG_Generate request of every stream: d_out DEVICE [streams][nbytes] bytes
 *   (stream s at d_out + s * nbytes), nbytes <= 65,536 (2^19 bits, the per-request maximum); then each
 *   state is updated (V += Hash(0x03 || V) + C + reseed_counter).  nbytes = 0 only updates the states.
 *   Asynchronous on `stream`; successive calls must be stream-ordered.  Errors: MR_ERR_ARG, MR_ERR_CUDA,
 *   MR_ERR_RANGE after 2^48 requests (the reseed interval; reseeding is not provided).
 * mr_fips_health_batch: the FIPS 140-2 §4.9.1 tests on d_blocks DEVICE [nblocks][2500] bytes (20,000
 *   bits each, most significant bit of each byte first); d_stats DEVICE uint32 [nblocks][16]: ones,
 *   poker S = sum of the squared nibble counts, runs of ones of length 1..5, 6+, runs of zeros of length
 *   1..5, 6+, long-run flag (a run >= 26 exists), verdict bits (1 monobit, 2 poker, 4 runs, 8 long run;
 *   set = pass).  Thresholds: 9,725 < ones < 10,275; 2.16 < 16 S / 5000 - 5000 < 46.17; runs within
 *   [2315,2685] [1114,1386] [527,723] [240,384] [103,209] [103,209]; no run >= 26 (reading R21).
 * ------------------------------------------------------------------------------------------ */
typedef struct mr_drbg mr_drbg;
int mr_drbg_create(mr_drbg **out, const uint8_t *entropy, size_t entropy_len, const uint8_t *nonce, size_t nonce_len,
                   const uint8_t *pers, size_t pers_len, uint32_t streams, int device);
int mr_drbg_generate(mr_drbg *d, uint8_t *d_out, size_t nbytes, void *stream);
void mr_drbg_destroy(mr_drbg *d);
int mr_fips_health_batch(const uint8_t *d_blocks, size_t nblocks, uint32_t *d_stats, void *stream);

/* ------------------------------------------------------------------------------------------
 * mr_rsa_keygen_batch_drbg — production form of mr_rsa_keygen_batch: the same GPU pipeline (sieve by the
 * first 10,000 primes, Miller-Rabin in the RNS Montgomery domain, Arazi inversion)
 * with every random choice drawn from the caller's Hash_DRBG `rng` (§2 "an approved deterministic
 * RBG", seeded by the caller with >= 256 bits of entropy):
 *   - each prime search starts at bits/2 DRBG bits with the top two bits and bit 0 set (FIPS 186-4 B.3.3);
 *   - each of the `rounds` Miller-Rabin rounds of a candidate w uses its own base b = 2 + (c mod (w - 3)),
 *     c = bits/2 + 64 DRBG bits (uniform in [2, w - 2] up to 2^-62: FIPS 186-4 C.3.1 with the
 *     "extra random bits" method of B.5.1).  FIPS 186-4 Table C.2 asks for 5 (bits = 2048) / 4 (3072)
 *     rounds after trial division; more are allowed.
 * The acceptance rules (gcd(e, p - 1) = 1, |p - q| > 2^(bits/2 - 100)) and outputs are those of
 * mr_rsa_keygen_batch; rng must live on `device`; the call advances rng (its requests are ordered on
 * `stream`).  Synchronous.  Same errors as mr_rsa_keygen_batch, plus MR_ERR_ARG for rng == NULL.
 * ------------------------------------------------------------------------------------------ */
int mr_rsa_keygen_batch_drbg(mr_drbg *rng, size_t count, int bits, uint32_t e, int rounds, uint32_t *d_n,
                             uint32_t *d_p, uint32_t *d_q, uint32_t *d_d, uint32_t *d_dp, uint32_t *d_dq,
                             uint32_t *d_qinv, int device, void *stream);

const char *mr_strerror(int code);

#ifdef __cplusplus
}
#endif
#endif /* MR_RNS_H */
