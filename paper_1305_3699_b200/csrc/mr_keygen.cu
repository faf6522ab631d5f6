// mr_keygen.cu — device kernels of the GPU RSA key-generation pipeline (
// the paper's MR-RSA lower tier: "RSA key generation ... is completely performed on the GPU with only
// e ... and N being transferred back to the CPU host", §3.3; "small primes testing (up to the
// first 10,000 primes) combined with Miller-Rabin compositeness tests", §4.3; Arazi inversion,
// P:46 §3.1).  The Miller-Rabin step itself is the library's mr_miller_rabin batch (RNS Montgomery
// domain); these kernels generate the candidates, sieve them, pick the first probable prime of
// every search in candidate order, and assemble N, d, d_p, d_q, q^-1 on the device.
#include <cuda_runtime.h>

#include <cstdint>

#include "mr_internal.h"

namespace mr {
namespace {

constexpr int KG_MAXL = 64;        // limbs of a prime (up to 2048-bit primes, RSA-4096)
constexpr u64 GOLDEN = 0x9E3779B97F4A7C15ull, IDX_MUL = 0xD1B54A32D192ED03ull;

__device__ __forceinline__ u64 splitmix64(u64 &s) {
    s += GOLDEN;
    u64 z = s;
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    return z ^ (z >> 31);
}

// start of search s: synth.odd_with_top_bits(32 L, seed, TAG_KEY, index[s]) — the same SplitMix64
// stream as synth/ (state0 = seed ^ tag*GOLDEN ^ index*IDX_MUL, limbs = low/high halves of successive
// outputs), top two bits and bit 0 forced; index[s] = key * 65536 + attempt (reading R19)
__global__ void k_kg_start(u64 seed, const u64 *index, u32 nslots, u32 L, u32 *starts) {
    const u32 s = blockIdx.x * blockDim.x + threadIdx.x;
    if (s >= nslots) return;
    u64 st = seed ^ (1ull * GOLDEN) ^ (index[s] * IDX_MUL);      // tag KEY = 1
    u32 *o = starts + (size_t)s * L;
    for (u32 l = 0; l < L; l += 2) {
        const u64 z = splitmix64(st);
        o[l] = (u32)z;
        if (l + 1 < L) o[l + 1] = (u32)(z >> 32);
    }
    o[L - 1] |= 0xC0000000u;
    o[0] |= 1u;
}

// DRBG-seeded variant (mr_rsa_keygen_batch_drbg): start of search s = L words of Hash_DRBG output with the
// top two bits and bit 0 forced (FIPS 186-4 B.3.3 draws the candidate from an approved RBG)
__global__ void k_kg_start_rand(const u32 *rnd, u32 nslots, u32 L, u32 *starts) {
    const u32 s = blockIdx.x * blockDim.x + threadIdx.x;
    if (s >= nslots) return;
    u32 *o = starts + (size_t)s * L;
    for (u32 l = 0; l < L; l++) o[l] = rnd[(size_t)s * L + l];
    o[L - 1] |= 0xC0000000u;
    o[0] |= 1u;
}

// Random Miller-Rabin bases for the DRBG-seeded variant: FIPS 186-4 C.3.1 step 4.3 wants b uniform in
// [2, w - 2]; the "extra random bits" method of FIPS 186-4 B.5.1 gives b = 2 + (c mod (w - 3)) with c of
// 32 (L + 2) DRBG bits (statistical distance from uniform < 2^-62).  w has its top two bits set, so
// m = w - 3 > 2^(32 L - 1): the top L words of c are < 2m (one conditional subtraction), then the low 64
// bits enter one at a time (r = 2 r + bit, minus m when it reaches m).  One thread per item.
__global__ void k_kg_rand_bases(const u32 *cand, const u32 *rnd, u32 items, u32 L, u32 *base) {
    const u32 it = blockIdx.x * blockDim.x + threadIdx.x;
    if (it >= items) return;
    const u32 *w = cand + (size_t)it * L, *c = rnd + (size_t)it * (L + 2);
    u32 m[KG_MAXL], r[KG_MAXL];
    u64 br = 3;
    for (u32 l = 0; l < L; l++) {                 // m = w - 3
        const u64 v = (u64)w[l] - (br & 0xFFFFFFFFull);
        m[l] = (u32)v;
        br = (br >> 32) + ((v >> 63) & 1);
        r[l] = c[l + 2];
    }
    auto ge = [&](u32 top) {                      // (top, r) >= m
        if (top) return true;
        for (int l = (int)L - 1; l >= 0; l--)
            if (r[l] != m[l]) return r[l] > m[l];
        return true;
    };
    auto subm = [&]() {
        u64 b = 0;
        for (u32 l = 0; l < L; l++) {
            const u64 v = (u64)r[l] - m[l] - b;
            r[l] = (u32)v;
            b = (v >> 63) & 1;
        }
    };
    if (ge(0)) subm();
    for (int bit = 63; bit >= 0; bit--) {
        const u32 in = (bit >= 32 ? c[1] >> (bit - 32) : c[0] >> bit) & 1u;
        u32 carry = in;
        for (u32 l = 0; l < L; l++) {
            const u32 nv = (r[l] << 1) | carry;
            carry = r[l] >> 31;
            r[l] = nv;
        }
        if (ge(carry)) subm();
    }
    u64 cy = 2;
    u32 *o = base + (size_t)it * L;
    for (u32 l = 0; l < L; l++) {                 // b = r + 2 <= w - 2
        const u64 v = (u64)r[l] + cy;
        o[l] = (u32)v;
        cy = v >> 32;
    }
}

// powers for the sieve: pw[l][i] = 2^(32 l) mod p_i, mu[i] = floor((2^64 - 1) / p_i)
__global__ void k_kg_pow(const u32 *small, u32 nsmall, u32 L, u32 *pw, u64 *mu) {
    const u32 i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= nsmall) return;
    const u32 p = small[i];
    u64 v = 1 % p;
    for (u32 l = 0; l < L; l++) {
        pw[(size_t)l * nsmall + i] = (u32)v;
        v = (v << 32) % p;
    }
    mu[i] = ~0ull / p;
}

__global__ void k_kg_zero(const u32 *list, u32 W, u32 *bitmap) {
    const u32 s = list[blockIdx.x];
    for (u32 w = threadIdx.x; w < W / 32; w += blockDim.x) bitmap[(size_t)s * (W / 32) + w] = 0;
}

// trial division of window w of search s (candidates start + 2 (W w + t), t < W) by the odd primes
// among the first 10,000: bit t of the bitmap is set when a small prime divides the candidate
// (the candidates exceed 2^31 > 104,729, so "divides" means "composite").
// CTA (x, y): KG_SB listed searches x KG_SB.. x 256 primes y*256..; thread = one prime.  The residue of
// a start is the contraction sum_l limb_l * (2^(32 l) mod p) (< 2^56 for L <= 64), reduced once by
// Barrett with mu = floor(2^64/p); the marks t = (p - r)(p + 1)/2 + j p < W go to the global bitmap.
constexpr u32 KG_SB = 16;
__global__ void __launch_bounds__(256) k_kg_sieve(const u32 *starts, const u32 *window, const u32 *list, u32 nlist,
                                                  u32 L, const u32 *small, const u32 *pw, const u64 *mu, u32 nsmall,
                                                  u32 W, u32 *bitmap) {
    __shared__ u32 limbs[KG_SB][KG_MAXL];
    __shared__ u64 off[KG_SB];
    const u32 s0 = blockIdx.x * KG_SB;
    const u32 ns = min(KG_SB, nlist - s0);
    for (u32 x = threadIdx.x; x < KG_SB * L; x += blockDim.x) {
        const u32 j = x / L, l = x % L;
        limbs[j][l] = j < ns ? starts[(size_t)list[s0 + j] * L + l] : 0u;
    }
    if (threadIdx.x < KG_SB) off[threadIdx.x] = threadIdx.x < ns ? 2ull * W * window[list[s0 + threadIdx.x]] : 0ull;
    __syncthreads();
    const u32 i = blockIdx.y * blockDim.x + threadIdx.x;
    if (i >= nsmall) return;
    const u32 p = small[i];
    const u64 m = mu[i];
    u64 acc[KG_SB];
#pragma unroll
    for (u32 j = 0; j < KG_SB; j++) acc[j] = off[j];
    for (u32 l = 0; l < L; l++) {
        const u32 w = pw[(size_t)l * nsmall + i];
#pragma unroll
        for (u32 j = 0; j < KG_SB; j++) acc[j] += (u64)w * limbs[j][l];
    }
    const u32 half = (p + 1) / 2;
#pragma unroll
    for (u32 j = 0; j < KG_SB; j++) {
        if (j >= ns) break;
        const u64 x = acc[j];
        u64 r = x - __umul64hi(x, m) * p;
        while (r >= p) r -= p;
        // (r + 2t) = 0 (mod p)  <=>  t = (p - r) (p + 1)/2 (mod p)
        const u64 y = (u64)(r ? p - (u32)r : 0u) * half;
        u64 t = y - __umul64hi(y, m) * p;
        while (t >= p) t -= p;
        u32 *bm = bitmap + (size_t)list[s0 + j] * (W / 32);
        for (; t < W; t += p) atomicOr(&bm[t / 32], 1u << (t % 32));
    }
}

// Miller-Rabin items are (candidate, base) pairs run as one-round tests in a single batch (reading
// R19: the verdict of a candidate is the AND over its rounds, so rounds may run as separate items).
// Phase-A items: for every listed search a (search act[a]) the next G sieve survivors in candidate
// order, after the tested[s] already consumed, as rows cand[a G + g] with base 2; ncand[a] = how many
// (< G: the window is exhausted after them).  Unused rows repeat the start (odd, never chosen).
__global__ void k_kg_pick(const u32 *starts, const u32 *window, const u32 *bitmap, const u32 *tested, const u32 *act,
                          u32 nact, u32 L, u32 W, u32 G, u32 *cand, u32 *base, u32 *ncand) {
    const u32 a = blockIdx.x * blockDim.x + threadIdx.x;
    if (a >= nact) return;
    const u32 s = act[a];
    const u32 *st = starts + (size_t)s * L;
    const u32 *bm = bitmap + (size_t)s * (W / 32);
    u32 skip = tested[s], n = 0;
    for (u32 wd = 0; wd < W / 32 && n < G; wd++) {
        u32 live = ~bm[wd];
        while (live && n < G) {
            const u32 b = __ffs(live) - 1;
            live &= live - 1;
            if (skip) { skip--; continue; }
            const u64 add = 2ull * ((u64)W * window[s] + 32u * wd + b);
            u32 *c = cand + ((size_t)a * G + n) * L;
            u64 carry = add;
            for (u32 l = 0; l < L; l++) {
                const u64 v = (u64)st[l] + (carry & 0xFFFFFFFFull);
                c[l] = (u32)v;
                carry = (carry >> 32) + (v >> 32);
            }
            n++;
        }
    }
    ncand[a] = n;
    for (u32 g = n; g < G; g++) {
        u32 *c = cand + ((size_t)a * G + g) * L;
        for (u32 l = 0; l < L; l++) c[l] = st[l];
    }
    for (u32 g = 0; g < G; g++) {
        u32 *bs = base + ((size_t)a * G + g) * L;
        for (u32 l = 0; l < L; l++) bs[l] = l ? 0u : 2u;
    }
}

// Verification items: rounds 2..R of the search's pending candidate vcand[s] (bases 3, 5, 7, ... = the
// 2nd..R-th primes), rows (v (R-1) + r) of cand/base for listed search v (search vl[v]).
__global__ void k_kg_vitems(const u32 *vl, u32 nv, const u32 *vcand, const u32 *small_all, u32 R, u32 L, u32 *cand,
                            u32 *base) {
    const u32 item = blockIdx.x * blockDim.x + threadIdx.x;
    if (item >= nv * (R - 1)) return;
    const u32 v = item / (R - 1), r = item % (R - 1);
    const u32 *src = vcand + (size_t)vl[v] * L;
    u32 *c = cand + (size_t)item * L, *bs = base + (size_t)item * L;
    for (u32 l = 0; l < L; l++) {
        c[l] = src[l];
        bs[l] = l ? 0u : small_all[r + 1];
    }
}

// dst[dst_row[i]] = src[src_row[i]] (rows of L words)
__global__ void k_kg_copy_rows(const u32 *src, const u32 *src_row, u32 *dst, const u32 *dst_row, u32 cnt, u32 L) {
    const u32 i = blockIdx.x;
    if (i >= cnt) return;
    for (u32 l = threadIdx.x; l < L; l += blockDim.x)
        dst[(size_t)dst_row[i] * L + l] = src[(size_t)src_row[i] * L + l];
}

// ---------------------------------------------------------------- per-key assembly

__device__ __forceinline__ u32 inv_mod_word(u32 a, u32 m) {   // a^-1 mod m (gcd = 1), extended Euclid
    long long t0 = 0, t1 = 1;
    u64 r0 = m, r1 = a % m;
    while (r1) {
        const u64 q = r0 / r1;
        const u64 r2 = r0 - q * r1;
        const long long t2 = t0 - (long long)q * t1;
        r0 = r1; r1 = r2; t0 = t1; t1 = t2;
    }
    if (t0 < 0) t0 += m;
    return (u32)t0;
}

__device__ __forceinline__ u32 mod_word(const u32 *a, u32 n, u32 m) {
    u64 r = 0;
    for (int l = (int)n - 1; l >= 0; l--) r = ((r << 32) | a[l]) % m;
    return (u32)r;
}

// Arazi inversion: d = (1 + f (-f^-1 mod e)) / e, the inverse of e modulo f for small e.
// f has n limbs; d has n limbs.  Requires gcd(e, f) = 1.
__device__ void arazi(const u32 *f, u32 n, u32 e, u32 *d) {
    const u32 fe = mod_word(f, n, e);
    const u32 x = (e - inv_mod_word(fe, e)) % e;          // -f^-1 mod e
    u32 t[2 * KG_MAXL + 1];
    u64 carry = 1;                                          // 1 + f x
    for (u32 l = 0; l < n; l++) {
        const u64 v = (u64)f[l] * x + carry;
        t[l] = (u32)v;
        carry = v >> 32;
    }
    t[n] = (u32)carry;
    u64 rem = 0;                                            // exact division by e
    for (int l = (int)n; l >= 0; l--) {
        const u64 cur = (rem << 32) | t[l];
        if (l < (int)n) d[l] = (u32)(cur / e);
        rem = cur % e;
    }
}

// q^-1 mod p (p odd prime, 0 < q mod p): binary inversion, HAC Alg. 14.61 shape
__device__ void inv_binary(const u32 *qin, const u32 *p, u32 n, u32 *out) {
    u32 u[KG_MAXL], v[KG_MAXL], x1[KG_MAXL + 1], x2[KG_MAXL + 1];
    // u = q mod p (q < 2^(32n) and p has its top two bits set: q < 2p suffices after one subtraction)
    {
        u64 br = 0;
        u32 tmp[KG_MAXL];
        for (u32 l = 0; l < n; l++) {
            const u64 t = (u64)qin[l] - p[l] - br;
            tmp[l] = (u32)t;
            br = (u32)(t >> 63);
        }
        for (u32 l = 0; l < n; l++) u[l] = br ? qin[l] : tmp[l];
    }
    for (u32 l = 0; l < n; l++) { v[l] = p[l]; x1[l] = l ? 0u : 1u; x2[l] = 0; }
    x1[n] = x2[n] = 0;
    auto is_one = [&](const u32 *a) {
        u32 z = a[0] ^ 1u;
        for (u32 l = 1; l < n; l++) z |= a[l];
        return z == 0;
    };
    auto halve = [&](u32 *a, u32 len) {
        for (u32 l = 0; l + 1 < len; l++) a[l] = (a[l] >> 1) | (a[l + 1] << 31);
        a[len - 1] >>= 1;
    };
    auto half_mod = [&](u32 *x) {        // x = x / 2 mod p   (x < p)
        if (x[0] & 1u) {
            u64 c = 0;
            for (u32 l = 0; l < n; l++) {
                const u64 t = (u64)x[l] + p[l] + c;
                x[l] = (u32)t;
                c = t >> 32;
            }
            x[n] = (u32)c;
        }
        halve(x, n + 1);
    };
    auto ge = [&](const u32 *a, const u32 *b) {
        for (int l = (int)n - 1; l >= 0; l--)
            if (a[l] != b[l]) return a[l] > b[l];
        return true;
    };
    auto sub_mod = [&](u32 *a, const u32 *b) {   // a = a - b mod p  (a, b < p)
        u64 br = 0;
        for (u32 l = 0; l < n; l++) {
            const u64 t = (u64)a[l] - b[l] - br;
            a[l] = (u32)t;
            br = (u32)(t >> 63);
        }
        if (br) {
            u64 c = 0;
            for (u32 l = 0; l < n; l++) {
                const u64 t = (u64)a[l] + p[l] + c;
                a[l] = (u32)t;
                c = t >> 32;
            }
        }
    };
    auto sub = [&](u32 *a, const u32 *b) {
        u64 br = 0;
        for (u32 l = 0; l < n; l++) {
            const u64 t = (u64)a[l] - b[l] - br;
            a[l] = (u32)t;
            br = (u32)(t >> 63);
        }
    };
    while (!is_one(u) && !is_one(v)) {
        while (!(u[0] & 1u)) { halve(u, n); half_mod(x1); }
        while (!(v[0] & 1u)) { halve(v, n); half_mod(x2); }
        if (ge(u, v)) { sub(u, v); sub_mod(x1, x2); }
        else { sub(v, u); sub_mod(x2, x1); }
    }
    const u32 *r = is_one(u) ? x1 : x2;
    for (u32 l = 0; l < n; l++) out[l] = r[l];
}

// one thread per key: N = p q, d = e^-1 mod (p-1)(q-1) (Arazi), d_p, d_q (Arazi), q^-1 mod p
__global__ void k_kg_assemble(const u32 *prime, const u32 *key_slot, u32 nkeys, u32 n, u32 e, u32 *N, u32 *P, u32 *Q,
                              u32 *D, u32 *DP, u32 *DQ, u32 *QINV) {
    const u32 k = blockIdx.x * blockDim.x + threadIdx.x;
    if (k >= nkeys) return;
    const u32 *p = prime + (size_t)key_slot[2 * k] * n;
    const u32 *q = prime + (size_t)key_slot[2 * k + 1] * n;
    u32 pm1[KG_MAXL], qm1[KG_MAXL], phi[2 * KG_MAXL];
    for (u32 l = 0; l < n; l++) {
        pm1[l] = p[l];
        qm1[l] = q[l];
    }
    pm1[0] -= 1u;                      // p, q odd: no borrow
    qm1[0] -= 1u;
    u32 *Nk = N + (size_t)k * 2 * n;
    for (u32 l = 0; l < 2 * n; l++) { Nk[l] = 0; phi[l] = 0; }
    for (u32 i = 0; i < n; i++) {      // schoolbook products N = p q, phi = (p-1)(q-1)
        u64 c1 = 0, c2 = 0;
        for (u32 j = 0; j < n; j++) {
            const u64 v1 = (u64)p[i] * q[j] + Nk[i + j] + c1;
            Nk[i + j] = (u32)v1;
            c1 = v1 >> 32;
            const u64 v2 = (u64)pm1[i] * qm1[j] + phi[i + j] + c2;
            phi[i + j] = (u32)v2;
            c2 = v2 >> 32;
        }
        Nk[i + n] = (u32)c1;
        phi[i + n] = (u32)c2;
    }
    arazi(phi, 2 * n, e, D + (size_t)k * 2 * n);
    arazi(pm1, n, e, DP + (size_t)k * n);
    arazi(qm1, n, e, DQ + (size_t)k * n);
    inv_binary(q, p, n, QINV + (size_t)k * n);
    for (u32 l = 0; l < n; l++) {
        P[(size_t)k * n + l] = p[l];
        Q[(size_t)k * n + l] = q[l];
    }
}

// acceptance tests of the fixture recipe for the primes listed: ok[i] bit 0 = gcd(e, p - 1) = 1
// (e prime: e does not divide p - 1), bit 1 = |p - q| > 2^(32 n - 100) against pool row first[i]
// (bit 1 set when first[i] = ~0).
__global__ void k_kg_check(const u32 *pool, u32 n, u32 e, const u32 *which, const u32 *first, u32 cnt, u32 *ok) {
    const u32 i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= cnt) return;
    const u32 *p = pool + (size_t)which[i] * n;
    u32 r = (mod_word(p, n, e) + e - 1) % e;
    u32 flags = r != 0 ? 1u : 0u;
    const u32 f = first[i];
    if (f == 0xFFFFFFFFu) {
        flags |= 2u;
    } else {
        const u32 *q = pool + (size_t)f * n;
        bool p_ge = true;
        for (int l = (int)n - 1; l >= 0; l--)
            if (p[l] != q[l]) { p_ge = p[l] > q[l]; break; }
        const u32 *x = p_ge ? p : q, *y = p_ge ? q : p;
        u32 diff[KG_MAXL];
        u64 br = 0;
        for (u32 l = 0; l < n; l++) {
            const u64 t = (u64)x[l] - y[l] - br;
            diff[l] = (u32)t;
            br = (u32)(t >> 63);
        }
        int bits = 0;
        for (int l = (int)n - 1; l >= 0; l--)
            if (diff[l]) { bits = 32 * l + 32 - __clz(diff[l]); break; }
        if (bits > (int)(32 * n) - 100) flags |= 2u;
    }
    ok[i] = flags;
}

}  // namespace

// ---------------------------------------------------------------- launchers (called by mr_host.cpp)
static int kg_err() { return cudaGetLastError() == cudaSuccess ? 0 : 6; }

int kg_launch_start(u64 seed, const u64 *index, u32 nslots, u32 L, u32 *starts, void *st) {
    if (!nslots) return 0;
    k_kg_start<<<(nslots + 127) / 128, 128, 0, (cudaStream_t)st>>>(seed, index, nslots, L, starts);
    return kg_err();
}
int kg_launch_pow(const u32 *small, u32 nsmall, u32 L, u32 *pw, u64 *mu, void *st) {
    k_kg_pow<<<(nsmall + 127) / 128, 128, 0, (cudaStream_t)st>>>(small, nsmall, L, pw, mu);
    return kg_err();
}
int kg_launch_sieve(const u32 *starts, const u32 *window, const u32 *list, u32 nlist, u32 L, const u32 *small,
                    const u32 *pw, const u64 *mu, u32 nsmall, u32 W, u32 *bitmap, void *st) {
    if (!nlist) return 0;
    k_kg_zero<<<nlist, 128, 0, (cudaStream_t)st>>>(list, W, bitmap);
    dim3 grid((nlist + KG_SB - 1) / KG_SB, (nsmall + 255) / 256);
    k_kg_sieve<<<grid, 256, 0, (cudaStream_t)st>>>(starts, window, list, nlist, L, small, pw, mu, nsmall, W, bitmap);
    return kg_err();
}
int kg_launch_pick(const u32 *starts, const u32 *window, const u32 *bitmap, const u32 *tested, const u32 *act, u32 nact,
                   u32 L, u32 W, u32 G, u32 *cand, u32 *base, u32 *ncand, void *st) {
    if (!nact) return 0;
    k_kg_pick<<<(nact + 63) / 64, 64, 0, (cudaStream_t)st>>>(starts, window, bitmap, tested, act, nact, L, W, G, cand,
                                                             base, ncand);
    return kg_err();
}
int kg_launch_vitems(const u32 *vl, u32 nv, const u32 *vcand, const u32 *small_all, u32 R, u32 L, u32 *cand, u32 *base,
                     void *st) {
    if (!nv || R < 2) return 0;
    const u32 n = nv * (R - 1);
    k_kg_vitems<<<(n + 127) / 128, 128, 0, (cudaStream_t)st>>>(vl, nv, vcand, small_all, R, L, cand, base);
    return kg_err();
}
int kg_launch_start_rand(const u32 *rnd, u32 nslots, u32 L, u32 *starts, void *st) {
    if (!nslots) return 0;
    k_kg_start_rand<<<(nslots + 127) / 128, 128, 0, (cudaStream_t)st>>>(rnd, nslots, L, starts);
    return kg_err();
}
int kg_launch_rand_bases(const u32 *cand, const u32 *rnd, u32 items, u32 L, u32 *base, void *st) {
    if (!items) return 0;
    k_kg_rand_bases<<<(items + 127) / 128, 128, 0, (cudaStream_t)st>>>(cand, rnd, items, L, base);
    return kg_err();
}
int kg_launch_copy_rows(const u32 *src, const u32 *src_row, u32 *dst, const u32 *dst_row, u32 cnt, u32 L, void *st) {
    if (!cnt) return 0;
    k_kg_copy_rows<<<cnt, 64, 0, (cudaStream_t)st>>>(src, src_row, dst, dst_row, cnt, L);
    return kg_err();
}
int kg_launch_check(const u32 *pool, u32 n, u32 e, const u32 *which, const u32 *first, u32 cnt, u32 *ok, void *st) {
    if (!cnt) return 0;
    k_kg_check<<<(cnt + 127) / 128, 128, 0, (cudaStream_t)st>>>(pool, n, e, which, first, cnt, ok);
    return kg_err();
}
int kg_launch_assemble(const u32 *prime, const u32 *key_slot, u32 nkeys, u32 n, u32 e, u32 *N, u32 *P, u32 *Q, u32 *D,
                       u32 *DP, u32 *DQ, u32 *QINV, void *st) {
    if (!nkeys) return 0;
    k_kg_assemble<<<(nkeys + 63) / 64, 64, 0, (cudaStream_t)st>>>(prime, key_slot, nkeys, n, e, N, P, Q, D, DP, DQ,
                                                                  QINV);
    return kg_err();
}

}  // namespace mr
