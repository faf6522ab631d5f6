/*
 * oracle.c — plain, slow, obviously-correct CPU oracle for the MR-MOD / MR-RSA hot path of
 * Chauvet & Mahé, "Secrets from the GPU" (arXiv:1305.3699).
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
 * --impl reference leg may load this library.  The product path (paper_1305_3699_b200/) never
 * links, imports or executes anything under oracle/, and this file shares no code, header, table
 * or constant generator with it.
 *
 * What it computes is the *plain definition* of each result the GPU path produces, never an RNS
 * re-implementation: the RNS/Montgomery machinery of the paper (PAPER.md:38-48,
 * §3.1) reaches exactly x^E mod N, a value with a plain definition, so the oracle is that definition
 * written out with positional radix-2^32 bignums:
 *
 *   O1 representation   little-endian uint32 limbs, (ptr, len), normalised = no high zero limbs
 *   O2 cmp / add / sub  limb loops with 64-bit carry / borrow
 *   O3 multiply         schoolbook, 64-bit accumulation            ("schoolbook")
 *   O4 divmod           Knuth TAOCP vol.2 §4.3.1 Algorithm D       (paper cites [TheArt])
 *                        + an independent bit-by-bit shift-subtract division used only as a pin
 *   O5 modexp           left-to-right binary square-and-multiply   ("traditional
 *                        square-and-multiply algorithms" [HAC 14.79]); reduce after every product
 *   O6 inverse          extended Euclid, coefficients kept in [0, m)  (P:54 d = e^-1 mod (p-1)(q-1))
 *   O7 CRT decrypt      Garner: m_p = c^dp mod p, m_q = c^dq mod q, h = qinv (m_p - m_q) mod p,
 *                        m = m_q + q h                               (north_star; HAC 14.71)
 *   O8 Miller-Rabin     HAC Alg. 4.24 with explicit bases          ("Miller-Rabin test with a
 *                        user-parameterized number of iterations"); FACTOR verdict when n > 2^32
 *                        shares a prime with the 2k-prime RNS base pair (reading R14)
 *   O9 small primes     sieve of Eratosthenes                       ("first 10,000 primes")
 *   O10 next prime      trial division + deterministic MR bases 2,3,5,... (fixture key generation)
 *   O12 batch drivers   pthreads over message indices (static interleave) for the CPU baseline
 *
 * Parity status: every function above is pinned by tests/test_oracle_*.py (textbook RSA,
 * Fermat on Mersenne primes, closed forms 2^E mod 2^n±1, brute force on tiny moduli, Carmichael
 * numbers, strong pseudoprimes A014233, the 10,000th prime, shift-subtract vs Knuth D, CPython pow
 * and sympy as independent libraries).  No function is "parity unpinned".
 */
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#include <pthread.h>

typedef uint32_t u32;
typedef uint64_t u64;
typedef int64_t i64;

#define ORC_EXPORT __attribute__((visibility("default")))

/* ------------------------------------------------------------------ O1 / O2 */

static int nrm(const u32 *a, int n) {
    while (n > 0 && a[n - 1] == 0) n--;
    return n;
}

ORC_EXPORT int orc_cmp(const u32 *a, int na, const u32 *b, int nb) {
    na = nrm(a, na);
    nb = nrm(b, nb);
    if (na != nb) return na < nb ? -1 : 1;
    for (int i = na - 1; i >= 0; i--)
        if (a[i] != b[i]) return a[i] < b[i] ? -1 : 1;
    return 0;
}

/* r has room for max(na, nb) + 1 limbs; r may alias a or b. Returns normalised length. */
ORC_EXPORT int orc_add(u32 *r, const u32 *a, int na, const u32 *b, int nb) {
    int n = na > nb ? na : nb;
    u64 carry = 0;
    for (int i = 0; i < n; i++) {
        u64 s = carry;
        if (i < na) s += a[i];
        if (i < nb) s += b[i];
        r[i] = (u32)s;
        carry = s >> 32;
    }
    r[n] = (u32)carry;
    return nrm(r, n + 1);
}

/* r = a - b, requires a >= b (returns -1 otherwise); r has room for na limbs; may alias a. */
ORC_EXPORT int orc_sub(u32 *r, const u32 *a, int na, const u32 *b, int nb) {
    if (orc_cmp(a, na, b, nb) < 0) return -1;
    na = nrm(a, na);
    u64 borrow = 0;
    for (int i = 0; i < na; i++) {
        u64 ai = a[i];
        u64 bi = (i < nb ? (u64)b[i] : 0) + borrow;
        r[i] = (u32)(ai - bi);
        borrow = ai < bi;
    }
    return nrm(r, na);
}

/* ------------------------------------------------------------------ O3 */

/* r = a * b, schoolbook; r has room for na + nb limbs and must not alias a or b. */
ORC_EXPORT int orc_mul(u32 *r, const u32 *a, int na, const u32 *b, int nb) {
    na = nrm(a, na);
    nb = nrm(b, nb);
    for (int i = 0; i < na + nb; i++) r[i] = 0;
    for (int i = 0; i < na; i++) {
        u64 carry = 0;
        for (int j = 0; j < nb; j++) {
            /* (2^32-1)^2 + 2 (2^32-1) = 2^64 - 1: never overflows */
            u64 t = (u64)a[i] * b[j] + r[i + j] + carry;
            r[i + j] = (u32)t;
            carry = t >> 32;
        }
        r[i + nb] = (u32)carry;
    }
    return nrm(r, na + nb);
}

/* ------------------------------------------------------------------ O4 */

/*
 * Knuth, TAOCP vol. 2, §4.3.1, Algorithm D (base b = 2^32).
 * a = q*m + r, 0 <= r < m.  q has room for na - nm + 1 limbs (may be NULL), r for nm limbs.
 * Returns 0, or -1 when m = 0.  Neither q nor r may alias a or m.
 */
ORC_EXPORT int orc_divmod(u32 *q, int *nq, u32 *r, int *nr, const u32 *a, int na, const u32 *m, int nm) {
    na = nrm(a, na);
    nm = nrm(m, nm);
    if (nm == 0) return -1;
    if (orc_cmp(a, na, m, nm) < 0) {            /* quotient 0, remainder a */
        for (int i = 0; i < na; i++) r[i] = a[i];
        *nr = na;
        if (nq) *nq = 0;
        return 0;
    }
    if (nm == 1) {                                /* short division by one limb */
        u64 rem = 0;
        for (int i = na - 1; i >= 0; i--) {
            u64 cur = (rem << 32) | a[i];
            if (q) q[i] = (u32)(cur / m[0]);
            rem = cur % m[0];
        }
        r[0] = (u32)rem;
        *nr = nrm(r, 1);
        if (nq) *nq = nrm(q, na);
        return 0;
    }
    /* D1: normalise so the top limb of the divisor has its high bit set */
    int s = __builtin_clz(m[nm - 1]);
    u32 *v = (u32 *)malloc(sizeof(u32) * nm);
    u32 *u = (u32 *)malloc(sizeof(u32) * (na + 1));
    for (int i = nm - 1; i > 0; i--) v[i] = s ? (m[i] << s) | (m[i - 1] >> (32 - s)) : m[i];
    v[0] = m[0] << s;
    u[na] = s ? a[na - 1] >> (32 - s) : 0;
    for (int i = na - 1; i > 0; i--) u[i] = s ? (a[i] << s) | (a[i - 1] >> (32 - s)) : a[i];
    u[0] = a[0] << s;
    /* D2..D7: one quotient limb per step, from the top */
    for (int j = na - nm; j >= 0; j--) {
        /* D3: estimate qhat from the top two limbs of the current remainder */
        u64 num = ((u64)u[j + nm] << 32) | u[j + nm - 1];
        u64 qhat = num / v[nm - 1];
        u64 rhat = num % v[nm - 1];
        while (qhat >> 32 || qhat * v[nm - 2] > ((rhat << 32) | u[j + nm - 2])) {
            qhat--;
            rhat += v[nm - 1];
            if (rhat >> 32) break;
        }
        /* D4: u[j .. j+nm] -= qhat * v */
        u64 mulcarry = 0;
        u64 borrow = 0;
        for (int i = 0; i < nm; i++) {
            u64 p = qhat * v[i] + mulcarry;
            mulcarry = p >> 32;
            u64 sub = (u64)(u32)p + borrow;
            borrow = (u64)u[i + j] < sub;
            u[i + j] = (u32)((u64)u[i + j] - sub);
        }
        u64 sub = mulcarry + borrow;
        int negative = (u64)u[j + nm] < sub;
        u[j + nm] = (u32)((u64)u[j + nm] - sub);
        /* D5/D6: if the remainder went negative, qhat was one too large: add v back */
        if (negative) {
            qhat--;
            u64 c = 0;
            for (int i = 0; i < nm; i++) {
                u64 t = (u64)u[i + j] + v[i] + c;
                u[i + j] = (u32)t;
                c = t >> 32;
            }
            u[j + nm] = (u32)((u64)u[j + nm] + c);   /* the final carry cancels the borrow */
        }
        if (q) q[j] = (u32)qhat;
    }
    /* D8: un-normalise the remainder */
    for (int i = 0; i < nm; i++) r[i] = s ? (u[i] >> s) | (u[i + 1] << (32 - s)) : u[i];
    *nr = nrm(r, nm);
    if (nq) *nq = nrm(q, na - nm + 1);
    free(u);
    free(v);
    return 0;
}

/*
 * Independent long division, one bit at a time (restoring shift-subtract).  Used only by the
 * tests as a second algorithm that pins orc_divmod (SURVEY.md §8(c) "O4 ... cross-checked").
 */
ORC_EXPORT int orc_divmod_bitwise(u32 *q, int *nq, u32 *r, int *nr, const u32 *a, int na, const u32 *m, int nm) {
    na = nrm(a, na);
    nm = nrm(m, nm);
    if (nm == 0) return -1;
    int rl = nm + 1;
    u32 *rem = (u32 *)calloc((size_t)(rl > 0 ? rl : 1), sizeof(u32));
    for (int i = 0; i < na; i++) q[i] = 0;
    for (int bit = na * 32 - 1; bit >= 0; bit--) {
        /* rem = 2 rem + bit */
        u32 in = (a[bit / 32] >> (bit % 32)) & 1u;
        for (int i = rl - 1; i > 0; i--) rem[i] = (rem[i] << 1) | (rem[i - 1] >> 31);
        rem[0] = (rem[0] << 1) | in;
        if (orc_cmp(rem, rl, m, nm) >= 0) {
            orc_sub(rem, rem, rl, m, nm);
            q[bit / 32] |= 1u << (bit % 32);
        }
    }
    for (int i = 0; i < nm; i++) r[i] = rem[i];
    *nr = nrm(r, nm);
    *nq = nrm(q, na);
    free(rem);
    return 0;
}

/* r = a mod m (r has room for nm limbs) */
static int modred(u32 *r, const u32 *a, int na, const u32 *m, int nm) {
    int nr;
    int nqcap = na - nm + 1 > 1 ? na - nm + 1 : 1;
    u32 *q = (u32 *)malloc(sizeof(u32) * nqcap);
    int nq;
    orc_divmod(q, &nq, r, &nr, a, na, m, nm);
    free(q);
    return nr;
}

/* ------------------------------------------------------------------ O5 */

/*
 * y = x^E mod n, left-to-right binary square-and-multiply (HAC Alg. 14.79).
 * x may be >= n (it is reduced first).  E = 0 gives 1 (also for x = 0), and n = 1 gives 0.
 * y has room for nn limbs.  Returns the normalised length of y, or -1 if n = 0.
 */
ORC_EXPORT int orc_modexp(u32 *y, const u32 *x, int nx, const u32 *e, int ne, const u32 *n, int nn) {
    nn = nrm(n, nn);
    if (nn == 0) return -1;
    nx = nrm(x, nx);
    ne = nrm(e, ne);
    u32 *acc = (u32 *)calloc(nn, sizeof(u32));
    u32 *base = (u32 *)calloc(nn, sizeof(u32));
    u32 *prod = (u32 *)calloc(2 * nn, sizeof(u32));
    u32 one = 1;
    int nacc = modred(acc, &one, 1, n, nn);            /* acc = 1 mod n */
    int nbase = modred(base, x, nx, n, nn);            /* base = x mod n */
    for (int bit = ne * 32 - 1; bit >= 0; bit--) {
        int np = orc_mul(prod, acc, nacc, acc, nacc);  /* square */
        nacc = modred(acc, prod, np, n, nn);
        if ((e[bit / 32] >> (bit % 32)) & 1u) {        /* multiply */
            np = orc_mul(prod, acc, nacc, base, nbase);
            nacc = modred(acc, prod, np, n, nn);
        }
    }
    for (int i = 0; i < nn; i++) y[i] = i < nacc ? acc[i] : 0;
    free(acc);
    free(base);
    free(prod);
    return nacc;
}

/* ------------------------------------------------------------------ O6 */

/*
 * inv = a^-1 mod m by the extended Euclidean algorithm.  The Bezout coefficient of a is carried
 * modulo m, so it never goes negative: t_{i+1} = (t_{i-1} - q_i t_i) mod m.
 * Returns the normalised length of inv, or -1 when gcd(a, m) != 1 (or m < 2).
 * inv has room for nm limbs.
 */
ORC_EXPORT int orc_modinv(u32 *inv, const u32 *a, int na, const u32 *m, int nm) {
    nm = nrm(m, nm);
    if (nm == 0 || (nm == 1 && m[0] < 2)) return -1;
    int cap = nm + 2;
    u32 *r0 = calloc(cap, 4), *r1 = calloc(cap, 4), *r2 = calloc(cap, 4);
    u32 *t0 = calloc(cap, 4), *t1 = calloc(cap, 4), *t2 = calloc(cap, 4);
    u32 *q = calloc(cap, 4), *qt = calloc(2 * cap, 4), *tmp = calloc(cap, 4);
    int n0, n1, n2, nt0, nt1, nt2, nq, ntmp;
    for (int i = 0; i < nm; i++) r0[i] = m[i];
    n0 = nm;
    n1 = modred(r1, a, nrm(a, na), m, nm);            /* r1 = a mod m */
    nt0 = 0;                                          /* t0 = 0 */
    t1[0] = 1;
    nt1 = 1;                                          /* t1 = 1 */
    while (n1 > 0) {
        orc_divmod(q, &nq, r2, &n2, r0, n0, r1, n1);  /* r0 = q r1 + r2 */
        int nqt = orc_mul(qt, q, nq, t1, nt1);        /* t2 = (t0 - q t1) mod m */
        ntmp = modred(tmp, qt, nqt, m, nm);
        if (orc_cmp(t0, nt0, tmp, ntmp) >= 0) {
            nt2 = orc_sub(t2, t0, nt0, tmp, ntmp);
        } else {
            u32 *s = calloc(cap + 1, 4);
            int ns = orc_add(s, t0, nt0, m, nm);
            nt2 = orc_sub(t2, s, ns, tmp, ntmp);
            free(s);
        }
        /* shift (r0, r1) <- (r1, r2), (t0, t1) <- (t1, t2) */
        memcpy(r0, r1, 4 * cap); n0 = n1;
        memcpy(r1, r2, 4 * cap); n1 = n2;
        memset(r2, 0, 4 * cap);
        memcpy(t0, t1, 4 * cap); nt0 = nt1;
        memcpy(t1, t2, 4 * cap); nt1 = nt2;
        memset(t2, 0, 4 * cap);
    }
    int ok = (n0 == 1 && r0[0] == 1);                 /* gcd = r0 */
    int nres = -1;
    if (ok) {
        for (int i = 0; i < nm; i++) inv[i] = i < nt0 ? t0[i] : 0;
        nres = nt0;
    }
    free(r0); free(r1); free(r2); free(t0); free(t1); free(t2); free(q); free(qt); free(tmp);
    return nres;
}

/* ------------------------------------------------------------------ O7 */

/*
 * RSA decryption by the Chinese Remainder Theorem, Garner's recombination (HAC Note 14.75):
 *   m_p = c^dp mod p,  m_q = c^dq mod q,  h = qinv (m_p - m_q) mod p,  m = m_q + q h.
 * p, q, dp, dq, qinv have nh limbs; c and m have 2 nh limbs.  Returns 0.
 */
ORC_EXPORT int orc_crt_decrypt(u32 *m, const u32 *c, const u32 *p, const u32 *q, const u32 *dp,
                               const u32 *dq, const u32 *qinv, int nh) {
    int nc = 2 * nh;
    u32 *mp = calloc(nh, 4), *mq = calloc(nh, 4), *mqp = calloc(nh, 4);
    u32 *diff = calloc(nh + 1, 4), *prod = calloc(2 * nh + 1, 4), *h = calloc(nh, 4);
    u32 *qh = calloc(2 * nh + 1, 4);
    int nmp = orc_modexp(mp, c, nc, dp, nh, p, nh);
    int nmq = orc_modexp(mq, c, nc, dq, nh, q, nh);
    int nmqp = modred(mqp, mq, nmq, p, nh);            /* m_q mod p */
    int nd;
    if (orc_cmp(mp, nmp, mqp, nmqp) >= 0) {
        nd = orc_sub(diff, mp, nmp, mqp, nmqp);
    } else {
        u32 *s = calloc(nh + 1, 4);
        int ns = orc_add(s, mp, nmp, p, nh);
        nd = orc_sub(diff, s, ns, mqp, nmqp);
        free(s);
    }
    int nprod = orc_mul(prod, qinv, nh, diff, nd);
    int nhh = modred(h, prod, nprod, p, nh);
    int nqh = orc_mul(qh, q, nh, h, nhh);
    u32 *res = calloc(2 * nh + 2, 4);
    int nres = orc_add(res, qh, nqh, mq, nmq);
    for (int i = 0; i < nc; i++) m[i] = i < nres ? res[i] : 0;
    free(mp); free(mq); free(mqp); free(diff); free(prod); free(h); free(qh); free(res);
    return 0;
}

/* ------------------------------------------------------------------ O9 */

/* the first `count` primes, ascending, by the sieve of Eratosthenes; returns how many were written */
ORC_EXPORT int orc_small_primes(u32 *out, int count) {
    if (count <= 0) return 0;
    u32 limit = 16;
    for (;;) {
        char *comp = calloc(limit + 1, 1);
        int found = 0;
        for (u32 i = 2; i <= limit && found < count; i++) {
            if (comp[i]) continue;
            out[found++] = i;
            for (u64 j = (u64)i * i; j <= limit; j += i) comp[j] = 1;
        }
        free(comp);
        if (found == count) return found;
        limit *= 2;
    }
}

/* is the 32-bit word w prime?  trial division by every odd d <= sqrt(w) */
static int word_is_prime(u32 w) {
    if (w < 2) return 0;
    if (w % 2 == 0) return w == 2;
    for (u64 d = 3; d * d <= w; d += 2)
        if (w % d == 0) return 0;
    return 1;
}

/*
 * The RNS base pair of the GPU library (reading R1): B = the k largest primes below
 * 2^32, B' = the next k, where for k <= 65 (2k <= 130) only primes congruent to 3 mod 4 are
 * taken.  The oracle derives them on its own (trial division on words) and uses them only to
 * define the MR "FACTOR" verdict (reading R14).  out receives 2k primes, descending.
 */
ORC_EXPORT int orc_base_primes(u32 *out, int two_k) {
    int found = 0;
    const int only_3mod4 = two_k <= 130;
    for (u64 w = 0xFFFFFFFFull; found < two_k && w > 1; w--)
        if ((!only_3mod4 || (w & 3u) == 3u) && word_is_prime((u32)w)) out[found++] = (u32)w;
    return found;
}

/* ------------------------------------------------------------------ O8 */

enum { ORC_COMPOSITE = 0, ORC_PROBABLY_PRIME = 1, ORC_FACTOR = 2, ORC_BAD_INPUT = -1 };

/*
 * Miller-Rabin, HAC Algorithm 4.24, with the bases given explicitly (reading R13):
 *   write n - 1 = 2^s d, d odd; for each round r: y = a_r^d mod n; if y not in {1, n-1}:
 *   repeat up to s-1 times { y = y^2 mod n; if y = 1 -> COMPOSITE; if y = n-1 -> next round };
 *   if y never reached n-1 -> COMPOSITE (witness round r).  After all rounds: PROBABLY_PRIME.
 * Before round 0, when n > 2^32 and some prime of the supplied list divides n -> FACTOR
 * (the RNS base cannot represent n^-1; reading R14).  Input rules: n odd, n >= 5, every base in
 * [2, n-2], else ORC_BAD_INPUT.  bases is [rounds][nn] limbs.  *witness = first witnessing round
 * or -1.
 */
ORC_EXPORT int orc_miller_rabin(const u32 *n, int nn, const u32 *bases, int rounds,
                                const u32 *factor_primes, int nfp, int *witness) {
    *witness = -1;
    int nnn = nrm(n, nn);
    if (nnn == 0 || (n[0] & 1u) == 0) return ORC_BAD_INPUT;
    if (nnn == 1 && n[0] < 5) return ORC_BAD_INPUT;
    u32 *nm1 = calloc(nn, 4), *nm2 = calloc(nn, 4), *d = calloc(nn, 4), *y = calloc(nn, 4);
    u32 *prod = calloc(2 * nn, 4), *two = calloc(nn, 4);
    u32 one = 1;
    int nnm1 = orc_sub(nm1, n, nnn, &one, 1);
    u32 twov = 2;
    int nnm2 = orc_sub(nm2, n, nnn, &twov, 1);
    int verdict = ORC_PROBABLY_PRIME;
    for (int r = 0; r < rounds; r++) {                 /* base range check */
        const u32 *a = bases + (size_t)r * nn;
        if (orc_cmp(a, nn, &twov, 1) < 0 || orc_cmp(a, nn, nm2, nnm2) > 0) { verdict = ORC_BAD_INPUT; goto out; }
    }
    if (nnn > 1) {                                     /* n > 2^32: FACTOR check against the base */
        for (int i = 0; i < nfp; i++) {
            u32 rem[1];
            int nrem = modred(rem, n, nnn, &factor_primes[i], 1);
            if (nrem == 0) { verdict = ORC_FACTOR; goto out; }
        }
    }
    /* n - 1 = 2^s d */
    int s = 0;
    while (((nm1[s / 32] >> (s % 32)) & 1u) == 0) s++;
    for (int i = 0; i < nn; i++) {
        int w = i + s / 32, b = s % 32;
        u32 lo = w < nn ? nm1[w] : 0, hi = w + 1 < nn ? nm1[w + 1] : 0;
        d[i] = b ? (lo >> b) | (hi << (32 - b)) : lo;
    }
    int nd = nrm(d, nn);
    for (int r = 0; r < rounds; r++) {
        const u32 *a = bases + (size_t)r * nn;
        int ny = orc_modexp(y, a, nn, d, nd, n, nnn);
        if ((ny == 1 && y[0] == 1) || orc_cmp(y, ny, nm1, nnm1) == 0) continue;
        int reached = 0;
        for (int j = 1; j < s; j++) {
            int np = orc_mul(prod, y, ny, y, ny);
            ny = modred(y, prod, np, n, nnn);
            if (orc_cmp(y, ny, nm1, nnm1) == 0) { reached = 1; break; }
            if (ny == 1 && y[0] == 1) break;
        }
        if (!reached) { verdict = ORC_COMPOSITE; *witness = r; goto out; }
    }
out:
    free(nm1); free(nm2); free(d); free(y); free(prod); free(two);
    return verdict;
}

/* ------------------------------------------------------------------ O10 */

/*
 * p = the first probable prime >= start (start forced odd), stepping by 2: trial division by the
 * first 10,000 primes, then Miller-Rabin with the deterministic prime bases 2, 3, 5, ...
 * (`rounds` of them).  Used only to generate committed key fixtures.  Returns the number of
 * candidates examined, or -1 if none was found within max_steps.
 */
ORC_EXPORT int orc_next_prime(u32 *p, const u32 *start, int n, int rounds, int max_steps) {
    static u32 sp[10000];
    static int have = 0;
    if (!have) { orc_small_primes(sp, 10000); have = 1; }
    u32 *cand = calloc(n + 1, 4), *bases = calloc((size_t)rounds * n, 4);
    memcpy(cand, start, 4 * n);
    cand[0] |= 1u;
    for (int r = 0; r < rounds; r++) bases[(size_t)r * n] = sp[r];
    for (int step = 0; step < max_steps; step++) {
        int composite = 0;
        for (int i = 1; i < 10000 && !composite; i++) {       /* odd small primes */
            u32 rem[1];
            int nr = modred(rem, cand, n, &sp[i], 1);
            if (nr == 0 && orc_cmp(cand, n, &sp[i], 1) != 0) composite = 1;
        }
        if (!composite) {
            int w;
            int v = orc_miller_rabin(cand, n, bases, rounds, NULL, 0, &w);
            if (v == ORC_PROBABLY_PRIME) {
                memcpy(p, cand, 4 * n);
                free(cand); free(bases);
                return step + 1;
            }
        }
        u32 two = 2;
        int nc = orc_add(cand, cand, n, &two, 1);
        (void)nc;
        if (cand[n] != 0) break;                               /* ran past n limbs */
    }
    free(cand); free(bases);
    return -1;
}

/* ------------------------------------------------------------------ O12: threaded batch drivers */

typedef struct {
    int kind;                 /* 0 modexp, 1 crt, 2 mr */
    int tid, nthreads, count;
    const u32 *x; int lx; u32 *y; int ly;
    const u32 *e; int ne; const u32 *n; int nn;
    const u32 *p, *q, *dp, *dq, *qinv; int nh;
    const u32 *bases; int rounds; const u32 *fp; int nfp; int *verdict; int *witness;
} job_t;

static void *worker(void *arg) {
    job_t *j = (job_t *)arg;
    for (int i = j->tid; i < j->count; i += j->nthreads) {   /* static interleave over messages */
        if (j->kind == 0) {
            orc_modexp(j->y + (size_t)i * j->ly, j->x + (size_t)i * j->lx, j->lx, j->e, j->ne, j->n, j->nn);
        } else if (j->kind == 1) {
            orc_crt_decrypt(j->y + (size_t)i * 2 * j->nh, j->x + (size_t)i * 2 * j->nh, j->p, j->q, j->dp,
                            j->dq, j->qinv, j->nh);
        } else {
            j->verdict[i] = orc_miller_rabin(j->x + (size_t)i * j->lx, j->lx,
                                             j->bases + (size_t)i * j->rounds * j->lx, j->rounds, j->fp,
                                             j->nfp, &j->witness[i]);
        }
    }
    return NULL;
}

static int run_jobs(job_t proto, int threads) {
    if (threads < 1) threads = 1;
    pthread_t *th = malloc(sizeof(pthread_t) * threads);
    job_t *jobs = malloc(sizeof(job_t) * threads);
    for (int t = 0; t < threads; t++) {
        jobs[t] = proto;
        jobs[t].tid = t;
        jobs[t].nthreads = threads;
        pthread_create(&th[t], NULL, worker, &jobs[t]);
    }
    for (int t = 0; t < threads; t++) pthread_join(th[t], NULL);
    free(th);
    free(jobs);
    return 0;
}

/* y[i] = x[i]^e mod n for i < count; x is [count][lx], y is [count][nn] */
ORC_EXPORT int orc_modexp_batch(const u32 *x, int lx, int count, const u32 *e, int ne, const u32 *n, int nn,
                                u32 *y, int threads) {
    job_t j;
    memset(&j, 0, sizeof j);
    j.kind = 0; j.count = count; j.x = x; j.lx = lx; j.y = y; j.ly = nn; j.e = e; j.ne = ne; j.n = n; j.nn = nn;
    return run_jobs(j, threads);
}

/* m[i] = CRT-decrypt(c[i]); c, m are [count][2 nh] */
ORC_EXPORT int orc_crt_decrypt_batch(const u32 *c, int count, const u32 *p, const u32 *q, const u32 *dp,
                                     const u32 *dq, const u32 *qinv, int nh, u32 *m, int threads) {
    job_t j;
    memset(&j, 0, sizeof j);
    j.kind = 1; j.count = count; j.x = c; j.y = m; j.p = p; j.q = q; j.dp = dp; j.dq = dq; j.qinv = qinv; j.nh = nh;
    return run_jobs(j, threads);
}

/* verdict[i], witness[i] = MR(n[i], bases[i][0..rounds)); n is [count][nn], bases [count][rounds][nn] */
ORC_EXPORT int orc_miller_rabin_batch(const u32 *n, int nn, int count, const u32 *bases, int rounds,
                                      const u32 *factor_primes, int nfp, int *verdict, int *witness,
                                      int threads) {
    job_t j;
    memset(&j, 0, sizeof j);
    j.kind = 2; j.count = count; j.x = n; j.lx = nn; j.bases = bases; j.rounds = rounds; j.fp = factor_primes;
    j.nfp = nfp; j.verdict = verdict; j.witness = witness;
    return run_jobs(j, threads);
}
