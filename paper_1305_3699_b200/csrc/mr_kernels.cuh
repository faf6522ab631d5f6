// mr_kernels.cuh — sm_100a device code of the MR-MOD / MR-RSA hot path (arXiv:1305.3699 §3.1-§3.3).
//
// Included once per channel count by mr_k<K>.cu with MR_K defined.  Each translation unit is its
// own CUDA module, so the __constant__ base tables below are private to that K.
//
// Mapping: thread-per-message.  A thread keeps the 2K+1 residues of its message in
// registers for the whole exponentiation; the two base extensions (92-97% of the word products,
// SURVEY §8(a6)) run as fully-unrolled 96-bit multiply-accumulate chains whose constant operands
// come from the __constant__ bank (warp-uniform, no load instruction), CH output accumulators at a
// time for ILP.  Every residue reduction uses the pseudo-Mersenne form m = 2^32 - c, c < 2^13.
// Residues are kept lazily in [0, 2^32) (congruent, not necessarily < m); DESIGN.md §3 shows the
// value bound r < (K+3)N still holds, and the exit conversion canonicalises.
#pragma once
#include <cuda_runtime.h>
#include <cstdint>
#include "mr_internal.h"

#ifndef MR_K
#error "define MR_K before including mr_kernels.cuh"
#endif

namespace mr {
namespace {  // everything below is private to this K's translation unit

constexpr int K = MR_K;
constexpr int NCH = 2 * K + 1;                // residues per value: B, B', m_r
constexpr int CH = 8;                         // base-extension outputs per register tile
constexpr int THREADS = 128;
constexpr int MINB = K <= 9 ? 6 : (K <= 33 ? 4 : 2);
constexpr int SMAX = (K + 3 <= 2) ? 0 : (32 - __builtin_clz((unsigned)(K + 3 - 1))) - 1;  // N·2^s, s ≤ SMAX

constexpr BaseLayout BL = base_layout(K);
constexpr u32 O_C = BL.c, O_C2 = BL.c2, O_A1 = BL.A1, O_A1R = BL.A1r, O_A2 = BL.A2, O_A2R = BL.A2r;
constexpr u32 O_C1 = BL.C1, O_PIN = BL.pin, O_MISC = BL.misc, O_MPL = BL.MpL, O_NMP = BL.NMp;
constexpr u32 BASE_WORDS = BL.words;
constexpr u32 CXW = cx_words(K);

__constant__ u32 g_base[BASE_WORDS];

// ------------------------------------------------------------------ word arithmetic

// 96-bit multiply-accumulate (lo, mid, hi) += x * y; lowers to IMAD.WIDE.U32 with carry-out + IADD3.X
__device__ __forceinline__ void mac96(u32 &lo, u32 &mid, u32 &hi, u32 x, u32 y) {
    asm("mad.lo.cc.u32 %0, %3, %4, %0;\n\t"
        "madc.hi.cc.u32 %1, %3, %4, %1;\n\t"
        "addc.u32 %2, %2, 0;"
        : "+r"(lo), "+r"(mid), "+r"(hi)
        : "r"(x), "r"(y));
}

// h·2^32 + l  ->  congruent value in [0, 2^32) modulo m = 2^32 - c  (c < 2^13)
__device__ __forceinline__ u32 red64(u32 h, u32 l, u32 c) {
    u64 u = (u64)h * c + l;                   // < 2^32 (c + 1)
    u64 v = (u64)(u32)(u >> 32) * c + (u32)u; // < 2^32 + c^2
    u32 vl = (u32)v;
    return (v >> 32) ? vl + c : vl;           // 2^32 ≡ c; vl < c^2 then, so no wrap
}

// hi·2^64 + mid·2^32 + lo -> congruent value in [0, 2^32), hi < 2^7, c2 = c^2
__device__ __forceinline__ u32 red96(u32 hi, u32 mid, u32 lo, u32 c, u32 c2) {
    u64 u = (u64)mid * c + lo;                // < 2^45 + 2^32
    u = (u64)hi * c2 + u;                     // + < 2^33
    u64 v = (u64)(u32)(u >> 32) * c + (u32)u; // < 2^27 + 2^32
    u32 vl = (u32)v;
    return (v >> 32) ? vl + c : vl;
}

__device__ __forceinline__ u32 mulmod(u32 a, u32 b, u32 c) {
    u64 p = (u64)a * b;
    return red64((u32)(p >> 32), (u32)p, c);
}

__device__ __forceinline__ u32 canon(u32 x, u32 c) {  // lazy residue -> [0, m)
    u32 m = 0u - c;
    return x >= m ? x - m : x;
}

#define CC(ch) g_base[O_C + (ch)]
#define CC2(ch) g_base[O_C2 + (ch)]

// ------------------------------------------------------------------ RNS Montgomery multiplication
//
// a <- a · b · M^-1 (mod N), SURVEY §8(a6) / DESIGN.md §3, values < (K+3)N throughout.
//   6.1/6.2  B:   ξ_i = (a_i b_i mod m_i) σ_i mod m_i,      σ_i = |-N^-1 M_i^-1|_{m_i}
//            B':  t*_j = a*_j b*_j mod m'_j  (ξ-form operands)
//            m_r: t_r = a_r b_r mod 2^32
//   6.3  BE1 (approximate): q̂_j = Σ_i ξ_i |M_i|_{m'_j},  q̂_r = Σ_i ξ_i |M_i|_{2^32}
//   6.4/6.5  ξ'_j = t*_j |M^-1 λ_j^-1| + q̂_j |N M^-1 λ_j|  (= r_j λ_j, the ξ-form of r),
//            r_r = (t_r + q̂_r N) M^-1 mod 2^32
//   6.6  BE2 (exact, Shenoy-Kumaresan through m_r = 2^32): S_i = Σ_j ξ'_j |M'_j|_{m_i},
//        α' = (Σ_j ξ'_j |M'_j|_{2^32} - r_r) M'^-1 mod 2^32,  r_i = S_i - α'|M'|_{m_i}
// b is either a itself (square) or the vector at bp[c * bstride] (global window table or the
// global context block).  cx = this CTA's context block in shared memory.
__device__ __forceinline__ void mont_mul(u32 (&a)[NCH], const u32 *__restrict__ bp, u32 bstride, bool sq,
                                         const u32 *__restrict__ cx) {
    // ---- 6.1 / 6.2: channel products, q-digits
#pragma unroll
    for (int i = 0; i < K; i++) {
        u32 b = sq ? a[i] : bp[(size_t)i * bstride];
        u32 t = mulmod(a[i], b, CC(i));
        a[i] = mulmod(t, cx[cx_sigma(K) + i], CC(i));
    }
#pragma unroll
    for (int j = 0; j < K; j++) {
        u32 b = sq ? a[K + j] : bp[(size_t)(K + j) * bstride];
        a[K + j] = mulmod(a[K + j], b, CC(K + j));
    }
    const u32 tr = a[2 * K] * (sq ? a[2 * K] : bp[(size_t)(2 * K) * bstride]);

    // ---- 6.3 BE1, m_r column and r_r
    u32 qr = 0;
#pragma unroll
    for (int i = 0; i < K; i++) qr += a[i] * g_base[O_A1R + i];
    const u32 rr = tr * g_base[O_MISC + 0] + qr * cx[CX_NMINV_R];

    // ---- 6.3 BE1 main [1 x K]·[K x K] contraction, CH outputs per pass; 6.4/6.5 fused in the epilogue
#pragma unroll
    for (int j0 = 0; j0 < K; j0 += CH) {
        u32 lo[CH], mi[CH], hi[CH];
#pragma unroll
        for (int jj = 0; jj < CH; jj++) lo[jj] = mi[jj] = hi[jj] = 0;
#pragma unroll
        for (int i = 0; i < K; i++) {
#pragma unroll
            for (int jj = 0; jj < CH; jj++)
                if (j0 + jj < K) mac96(lo[jj], mi[jj], hi[jj], a[i], g_base[O_A1 + i * K + j0 + jj]);
        }
#pragma unroll
        for (int jj = 0; jj < CH; jj++) {
            const int j = j0 + jj;
            if (j < K) {
                const u32 c = CC(K + j), c2 = CC2(K + j);
                const u32 q = red96(hi[jj], mi[jj], lo[jj], c, c2);
                u64 p = (u64)a[K + j] * g_base[O_C1 + j];
                u32 l2 = (u32)p, m2 = (u32)(p >> 32), h2 = 0;
                mac96(l2, m2, h2, q, cx[cx_c2(K) + j]);
                a[K + j] = red96(h2, m2, l2, c, c2);
            }
        }
    }
    a[2 * K] = rr;

    // ---- 6.6 BE2 [1 x K]·[K x K] contraction, exact via the extra modulus
    u32 sr = 0;
#pragma unroll
    for (int j = 0; j < K; j++) sr += a[K + j] * g_base[O_A2R + j];
    const u32 alpha = (sr - rr) * g_base[O_MISC + 1];
#pragma unroll
    for (int i0 = 0; i0 < K; i0 += CH) {
        u32 lo[CH], mi[CH], hi[CH];
#pragma unroll
        for (int ii = 0; ii < CH; ii++) {
            if (i0 + ii < K) {
                u64 p = (u64)alpha * g_base[O_PIN + i0 + ii];
                lo[ii] = (u32)p;
                mi[ii] = (u32)(p >> 32);
                hi[ii] = 0;
            }
        }
#pragma unroll
        for (int j = 0; j < K; j++) {
#pragma unroll
            for (int ii = 0; ii < CH; ii++)
                if (i0 + ii < K) mac96(lo[ii], mi[ii], hi[ii], a[K + j], g_base[O_A2 + j * K + i0 + ii]);
        }
#pragma unroll
        for (int ii = 0; ii < CH; ii++) {
            const int i = i0 + ii;
            if (i < K) a[i] = red96(hi[ii], mi[ii], lo[ii], CC(i), CC2(i));
        }
    }
}

// ------------------------------------------------------------------ positional -> RNS (a2)
// a_c = Σ_l x_l |2^(32 l)|_{m_c} (B' entries of pow_tab already carry λ_j: ξ-form), a_r = x_0.
// Limbs are masked to zero when `ok` is false (out-of-range inputs run on x = 0).
__device__ __forceinline__ void to_rns(u32 (&a)[NCH], const u32 *__restrict__ x, u32 nl, bool ok,
                                       const u32 *__restrict__ pow_tab) {
    const u32 mask = ok ? 0xFFFFFFFFu : 0u;
#pragma unroll
    for (int c0 = 0; c0 < 2 * K; c0 += CH) {
        u32 lo[CH], mi[CH], hi[CH];
#pragma unroll
        for (int jj = 0; jj < CH; jj++) lo[jj] = mi[jj] = hi[jj] = 0;
#pragma unroll 1
        for (u32 l = 0; l < nl; l++) {
            const u32 xl = x[l] & mask;
            const u32 *pr = pow_tab + (size_t)l * (2 * K) + c0;
#pragma unroll
            for (int jj = 0; jj < CH; jj++)
                if (c0 + jj < 2 * K) mac96(lo[jj], mi[jj], hi[jj], xl, __ldg(pr + jj));
        }
#pragma unroll
        for (int jj = 0; jj < CH; jj++)
            if (c0 + jj < 2 * K) a[c0 + jj] = red96(hi[jj], mi[jj], lo[jj], CC(c0 + jj), CC2(c0 + jj));
    }
    a[2 * K] = x[0] & mask;
}

// ------------------------------------------------------------------ RNS -> positional, canonical (a7)
// z on B' ∪ {m_r}, z < (K+3)N < M': α' = (Σ ξ'_j |M'_j|_{2^32} - z_r) M'^-1 mod 2^32 (exact, P:42
// "provided an extra modulus"), X = Σ_j ξ'_j M'_j + α'(2^(32(K+1)) - M') mod 2^(32(K+1)) = z, then
// X mod N by conditional subtraction of N·2^s, s = SMAX..0.  Writes X[0..K].
__device__ __forceinline__ void from_rns(const u32 (&a)[NCH], const u32 *__restrict__ nlimbs, u32 (&X)[K + 1]) {
    u32 sr = 0;
#pragma unroll
    for (int j = 0; j < K; j++) sr += a[K + j] * g_base[O_A2R + j];
    const u32 alpha = (sr - a[2 * K]) * g_base[O_MISC + 1];
    u32 clo = 0, cmi = 0;
#pragma unroll
    for (int l = 0; l <= K; l++) {
        u32 lo = clo, mi = cmi, hi = 0;
#pragma unroll
        for (int j = 0; j < K; j++) mac96(lo, mi, hi, a[K + j], g_base[O_MPL + j * (K + 1) + l]);
        mac96(lo, mi, hi, alpha, g_base[O_NMP + l]);
        X[l] = lo;
        clo = mi;
        cmi = hi;
    }
    // X < 2^(SMAX+1) N  ->  X mod N
#pragma unroll 1
    for (int s = SMAX; s >= 0; s--) {
        u32 Y[K + 1];
        u32 borrow = 0;
#pragma unroll
        for (int l = 0; l <= K; l++) {
            const u32 cur = nlimbs[l];
            const u32 prev = l ? nlimbs[l - 1] : 0u;
            const u32 nsh = s ? ((cur << s) | (prev >> (32 - s))) : cur;
            const u64 t = (u64)X[l] - nsh - borrow;
            Y[l] = (u32)t;
            borrow = (u32)(t >> 63);
        }
        if (!borrow) {
#pragma unroll
            for (int l = 0; l <= K; l++) X[l] = Y[l];
        }
    }
}

// x (nl limbs) < bound (nl limbs)?
__device__ __forceinline__ bool less_than(const u32 *__restrict__ x, const u32 *__restrict__ bound, u32 nl) {
    int res = 0;  // -1 less, 1 greater, 0 equal so far (scan from the top)
#pragma unroll 1
    for (int l = (int)nl - 1; l >= 0 && res == 0; l--) {
        const u32 xv = x[l], bv = bound[l];
        res = xv < bv ? -1 : (xv > bv ? 1 : 0);
    }
    return res < 0;
}

// ------------------------------------------------------------------ modexp interpreter kernel (a2-a7, a8 ladders)
__global__ void __launch_bounds__(THREADS, MINB) k_modexp(const ModexpParams P) {
    __shared__ u32 s_cx[CXW];
    const u32 sel = blockIdx.x >= P.ctas0 ? 1u : 0u;
    const u32 *gcx = sel ? P.ctx[1] : P.ctx[0];
    for (u32 w = threadIdx.x; w < CXW; w += blockDim.x) s_cx[w] = gcx[w];
    __syncthreads();
    const u32 jl = (blockIdx.x - sel * P.ctas0) * blockDim.x + threadIdx.x;
    if (jl >= P.count) return;
    const u32 slot = sel * P.ctas0 * blockDim.x + jl;
    const size_t tstride = P.jobs_total;
    const size_t entry = (size_t)NCH * tstride;
    const u32 *xrow = P.x + (size_t)jl * P.in_limbs;
    const bool ok = less_than(xrow, s_cx + cx_inb(K), P.in_limbs);
    if (sel == 0 && P.status) P.status[jl] = ok ? 0 : 5 /* MR_ERR_RANGE */;

    const u64 *prog = sel ? P.prog[1] : P.prog[0];
    const u32 nops = sel ? P.nops[1] : P.nops[0];
    u32 a[NCH];
#pragma unroll
    for (int c = 0; c < NCH; c++) a[c] = 0;

#pragma unroll 1
    for (u32 s = 0; s < nops; s++) {
        const u64 op = __ldg(prog + s);
        const u32 fl = (u32)op & 0xFF, opnd = (u32)(op >> 8) & 0xFF, ld = (u32)(op >> 16) & 0xFF;
        const u32 ad = (u32)(op >> 24) & 0xFF, st = (u32)(op >> 32) & 0xFF;
        if (fl & (OPF_TORNS_ALL | OPF_TORNS_LO | OPF_TORNS_HI)) {
            const u32 off = (fl & OPF_TORNS_HI) ? P.half : 0u;
            const u32 nl = (fl & OPF_TORNS_ALL) ? P.in_limbs : P.half;
            to_rns(a, xrow + off, nl, ok, P.pow_tab);
        }
        if (fl & OPF_LOAD) {
            const u32 *src;
            size_t str;
            if (ld >= 0xF0) { src = gcx + cx_r2(K) + (ld - 0xF0) * NCH; str = 1; }
            else { src = P.table + ld * entry + slot; str = tstride; }
#pragma unroll
            for (int c = 0; c < NCH; c++) a[c] = src[c * str];
        }
        if (!(fl & OPF_NOMUL)) {
            const bool sq = opnd == OPND_SQ;
            const u32 *bp;
            u32 bs;
            if (sq) { bp = gcx; bs = 0; }
            else if (opnd >= 0xF0) { bp = gcx + cx_r2(K) + (opnd - 0xF0) * NCH; bs = 1; }
            else { bp = P.table + opnd * entry + slot; bs = (u32)tstride; }
            mont_mul(a, bp, bs, sq, s_cx);
        }
        if (fl & OPF_ADD) {  // channel-wise modular addition (CRT entry, a3)
            const u32 *src = P.table + ad * entry + slot;
#pragma unroll
            for (int c = 0; c < 2 * K; c++) {
                const u32 b = src[c * tstride];
                const u32 s2 = a[c] + b;
                a[c] = red64(s2 < b ? 1u : 0u, s2, CC(c));
            }
            a[2 * K] += src[(2 * K) * tstride];
        }
        if (fl & OPF_STORE) {
            u32 *dst = P.table + st * entry + slot;
#pragma unroll
            for (int c = 0; c < NCH; c++) dst[c * tstride] = a[c];
        }
    }
    u32 X[K + 1];
    from_rns(a, s_cx + cx_n(K), X);
    u32 *yrow = P.y + sel * P.out_stride + (size_t)jl * P.out_limbs;
#pragma unroll
    for (int l = 0; l <= K; l++)
        if ((u32)l < P.out_limbs) yrow[l] = ok ? X[l] : 0u;
}

// ------------------------------------------------------------------ CRT recombination (a8)
// m = m_q + q · h,  h = (m_p - m_q mod p) · qinv mod p computed as one RNS Montgomery
// multiplication by qinv·R mod p followed by the canonical exit.
__global__ void __launch_bounds__(THREADS, MINB) k_combine(const CombineParams P) {
    __shared__ u32 s_cx[CXW];
    for (u32 w = threadIdx.x; w < CXW; w += blockDim.x) s_cx[w] = P.ctx_p[w];
    __syncthreads();
    const u32 i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= P.count) return;
    const u32 H = P.half;
    const u32 *mp = P.mpq + (size_t)i * H;
    const u32 *mq = P.mpq + ((size_t)P.count + i) * H;
    const u32 *pl = s_cx + cx_n(K);
    // t = m_q mod p  (m_q < q < 2^(32H) ≤ 2^32 p): conditional subtraction of p·2^s, s = 32..0
    u32 t[K + 1];
#pragma unroll
    for (int l = 0; l <= K; l++) t[l] = (u32)l < H ? mq[l] : 0u;
#pragma unroll 1
    for (int s = 32; s >= 0; s--) {
        u32 Y[K + 1];
        u32 borrow = 0;
#pragma unroll
        for (int l = 0; l <= K; l++) {
            u32 nsh;
            if (s == 32) nsh = l ? pl[l - 1] : 0u;
            else {
                const u32 prev = l ? pl[l - 1] : 0u;
                nsh = s ? ((pl[l] << s) | (prev >> (32 - s))) : pl[l];
            }
            const u64 d = (u64)t[l] - nsh - borrow;
            Y[l] = (u32)d;
            borrow = (u32)(d >> 63);
        }
        if (!borrow) {
#pragma unroll
            for (int l = 0; l <= K; l++) t[l] = Y[l];
        }
    }
    // diff = m_p - t mod p  (both < p)
    u32 diff[K + 1];
    u32 borrow = 0;
#pragma unroll
    for (int l = 0; l <= K; l++) {
        const u64 d = (u64)((u32)l < H ? mp[l] : 0u) - t[l] - borrow;
        diff[l] = (u32)d;
        borrow = (u32)(d >> 63);
    }
    if (borrow) {
        u32 carry = 0;
#pragma unroll
        for (int l = 0; l <= K; l++) {
            const u64 s2 = (u64)diff[l] + pl[l] + carry;
            diff[l] = (u32)s2;
            carry = (u32)(s2 >> 32);
        }
    }
    // h = diff · qinv mod p in RNS:  mm(diff, qinv R mod p) = diff qinv (mod p)
    u32 a[NCH];
    {
        // to_rns of a register-resident number: reuse the table contraction on a local copy
        const u32 mask = 0xFFFFFFFFu;
#pragma unroll
        for (int c0 = 0; c0 < 2 * K; c0 += CH) {
            u32 lo[CH], mi[CH], hi[CH];
#pragma unroll
            for (int jj = 0; jj < CH; jj++) lo[jj] = mi[jj] = hi[jj] = 0;
#pragma unroll
            for (int l = 0; l <= K; l++) {
                if ((u32)l < H) {
                    const u32 *pr = P.pow_tab + (size_t)l * (2 * K) + c0;
#pragma unroll
                    for (int jj = 0; jj < CH; jj++)
                        if (c0 + jj < 2 * K) mac96(lo[jj], mi[jj], hi[jj], diff[l] & mask, __ldg(pr + jj));
                }
            }
#pragma unroll
            for (int jj = 0; jj < CH; jj++)
                if (c0 + jj < 2 * K) a[c0 + jj] = red96(hi[jj], mi[jj], lo[jj], CC(c0 + jj), CC2(c0 + jj));
        }
        a[2 * K] = diff[0];
    }
    mont_mul(a, P.ctx_p + cx_qinvr(K), 1, false, s_cx);
    u32 h[K + 1];
    from_rns(a, pl, h);
    // m = m_q + q · h  (schoolbook, H x H limbs)
    u32 *mrow = P.m + (size_t)i * 2 * H;
#pragma unroll 1
    for (u32 l = 0; l < 2 * H; l++) mrow[l] = l < H ? mq[l] : 0u;
#pragma unroll 1
    for (u32 r = 0; r < H; r++) {
        const u32 qr = P.q[r];
        u32 carry = 0;
#pragma unroll
        for (int l = 0; l < K; l++) {
            if ((u32)l < H) {
                const u64 v = (u64)qr * h[l] + mrow[r + l] + carry;
                mrow[r + l] = (u32)v;
                carry = (u32)(v >> 32);
            }
        }
        for (u32 l = r + H; l < 2 * H && carry; l++) {
            const u64 v = (u64)mrow[l] + carry;
            mrow[l] = (u32)v;
            carry = (u32)(v >> 32);
        }
    }
    if (P.status && P.status[i] != 0) {
        for (u32 l = 0; l < 2 * H; l++) mrow[l] = 0;
    }
}

// ------------------------------------------------------------------ host-side launchers

int upload_base(const u32 *flat, int device) {
    if (cudaSetDevice(device) != cudaSuccess) return 6;
    if (cudaMemcpyToSymbol(g_base, flat, sizeof(u32) * BASE_WORDS) != cudaSuccess) return 6;
    return 0;
}

int launch_modexp(const ModexpParams &p, u32 ctas, void *stream) {
    k_modexp<<<ctas, THREADS, 0, (cudaStream_t)stream>>>(p);
    return cudaGetLastError() == cudaSuccess ? 0 : 6;
}

int launch_combine(const CombineParams &p, void *stream) {
    const u32 ctas = (p.count + THREADS - 1) / THREADS;
    k_combine<<<ctas, THREADS, 0, (cudaStream_t)stream>>>(p);
    return cudaGetLastError() == cudaSuccess ? 0 : 6;
}

int launch_mr(const MrParams &, void *) { return 1; }

}  // namespace
}  // namespace mr
