// mr_wide.cu — wide-operand RNS Montgomery modexp (8192-bit moduli, keys up to
// 16,128 bits; "up to 16,128-bit long").  DESIGN.md §4h.
//
// For k = 257 and 505 channels per base the per-message state (2k+1 words) and the base-extension matrices
// (k² words each: 264 KB / 1 MB) no longer fit the thread-per-message kernels, so this kernel maps
// CHANNELS to threads ("channels-on-lanes", the paper's own mapping) and register-blocks MB = 16
// messages per CTA: every thread owns output channels and accumulates them for the CTA's 16 messages at
// once, so each constant-matrix word read from L2 serves 16 multiply-accumulates.
//   state   st[ch][msg] in shared memory (2k+1 rows of 16 words)
//   BE1     q̂_j = Σ_i ξ_i A1'[i][j]   thread per output j, A1' row-major in HBM (coalesced over j),
//                                     ξ_i broadcast from shared memory (LDS.128)
//   BE2     r_i = Σ_j ξ'_j A2[j][i] + α' (m_i - |M'|_{m_i})   same shape
// Every channel product and every 96-bit column sum is reduced with a word Montgomery reduction; the
// resulting 2^-32 factors are absorbed into the host-built constants (A1' and A2 × 2^32, σ and C1 × 2^64,
// powers × 2^32), so any odd 32-bit modulus works (no bound on c = 2^32 mod m).  Runtime k: one kernel
// for every wide k.  Plain (unscaled) residues; the exit is the same CRT-with-extra-modulus reconstruction
// as mr_kernels.cuh from_rns, done cooperatively (column sums by thread, carries by one thread per message).
#include <cuda_runtime.h>
#include <cstdint>
#include <cstdlib>

#include "mr_internal.h"

namespace mr {
namespace {

constexpr int MB = 16;                 // messages per CTA (register-blocked)
constexpr int NTMAX = 512;             // threads per CTA (runtime: 32 * ceil((k+1)/32), <= 512)

__device__ __forceinline__ void mac96(u32 &lo, u32 &mid, u32 &hi, u32 x, u32 y) {
    asm("mad.lo.cc.u32 %0, %3, %4, %0;\n\t"
        "madc.hi.cc.u32 %1, %3, %4, %1;\n\t"
        "addc.u32 %2, %2, 0;"
        : "+r"(lo), "+r"(mid), "+r"(hi)
        : "r"(x), "r"(y));
}

// T = thi 2^32 + tlo -> T 2^-32 mod m, lazy in [0, 2^32) (as mr_kernels.cuh mont_red; valid for any odd m)
__device__ __forceinline__ u32 mont_red(u32 tlo, u32 thi, u32 m, u32 minv) {
    const u32 q = tlo * minv;
    [[maybe_unused]] u32 ulo;
    u32 uhi, cy;
    asm("mad.lo.cc.u32 %0, %3, %4, %5;\n\tmadc.hi.cc.u32 %1, %3, %4, %6;\n\taddc.u32 %2, 0, 0;"
        : "=r"(ulo), "=r"(uhi), "=r"(cy)
        : "r"(q), "r"(m), "r"(tlo), "r"(thi));
    return cy ? uhi - m : uhi;
}
// lazy a + b mod m (a, b < 2^32): each 2^32 carried out is worth r32 = 2^32 mod m; after one fold the value
// is < 2^32 + r32, and a second carry leaves a low word < r32, so the last add cannot wrap
__device__ __forceinline__ u32 addmod_lazy(u32 a, u32 b, u32 r32) {
    const u64 s = (u64)a + b;
    const u64 t = (u64)(u32)s + (s >> 32) * r32;
    return (u32)t + (u32)(t >> 32) * r32;
}
// (hi 2^64 + mid 2^32 + lo) 2^-32 mod m, hi < 2^9:  mont(mid:lo) + hi r32  (hi r32 < 2^9 2^16)
__device__ __forceinline__ u32 red96_mont(u32 hi, u32 mid, u32 lo, u32 m, u32 minv, u32 r32) {
    const u32 r = mont_red(lo, mid, m, minv);
    const u32 t = hi * r32;
    const u32 s = r + t;
    return s < r ? s + r32 : s;
}

struct WideArgs {
    const u32 *tab;                    // per-k wide table (mr_internal.h wide_*)
    u32 k;
    u32 nt;                            // threads per CTA
    u32 cxw;                           // word offset of the wide section in the context block
};

__device__ __forceinline__ u32 &ST(u32 *st, u32 ch, u32 msg) { return st[ch * MB + msg]; }

// acc[q] += Σ_{i < n} xs[i * MB + q] · A[i][j]  for the CTA's MB messages (96-bit accumulators); A is a
// chunked [R][ncols] matrix (mr_internal.h wch_at, R >= n): the thread's 8 coefficients of a row group are
// two 16-byte loads, issued one group ahead so their L2 latency overlaps the previous group's 128
// multiply-accumulates.  Rows i >= n of the last group are skipped (the xs rows there may be anything).
template <bool PP>
__device__ __forceinline__ void dot_mb(const u32 *__restrict__ mat, u32 ncols, u32 j, const u32 *xs, u32 n,
                                       u32 (&lo)[MB], u32 (&mi)[MB], u32 (&hi)[MB]) {
    const uint4 *cp = reinterpret_cast<const uint4 *>(mat + (size_t)j * 8);
    const u32 gs = 2 * ncols;                         // uint4 per row group
    const u32 ng = (n + 7) / 8;
    uint4 c0 = __ldg(cp), c1 = __ldg(cp + 1);
    auto group = [&](const u32 *xg, const uint4 &a, const uint4 &b, u32 rows) {
        const u32 c[8] = {a.x, a.y, a.z, a.w, b.x, b.y, b.z, b.w};
#pragma unroll
        for (int p = 0; p < 8; p++) {
            if ((u32)p < rows) {
                const uint4 *x = reinterpret_cast<const uint4 *>(xg + p * MB);
#pragma unroll
                for (int v4 = 0; v4 < MB / 4; v4++) {
                    const uint4 xv = x[v4];
                    mac96(lo[4 * v4 + 0], mi[4 * v4 + 0], hi[4 * v4 + 0], xv.x, c[p]);
                    mac96(lo[4 * v4 + 1], mi[4 * v4 + 1], hi[4 * v4 + 1], xv.y, c[p]);
                    mac96(lo[4 * v4 + 2], mi[4 * v4 + 2], hi[4 * v4 + 2], xv.z, c[p]);
                    mac96(lo[4 * v4 + 3], mi[4 * v4 + 3], hi[4 * v4 + 3], xv.w, c[p]);
                }
            }
        }
    };
if constexpr (PP) {
    // two groups per iteration with ping-pong coefficient registers (no copies between the buffers)
    u32 g = 0;
#pragma unroll 1
    for (; g + 2 < ng; g += 2) {
        const uint4 *np = cp + (size_t)(g + 1) * gs;
        const uint4 n0 = __ldg(np), n1 = __ldg(np + 1);
        group(xs + g * 8 * MB, c0, c1, 8);
        c0 = __ldg(np + gs);
        c1 = __ldg(np + gs + 1);
        group(xs + (g + 1) * 8 * MB, n0, n1, 8);
    }
    if (g + 1 < ng) {
        const uint4 *np = cp + (size_t)(g + 1) * gs;
        const uint4 n0 = __ldg(np), n1 = __ldg(np + 1);
        group(xs + g * 8 * MB, c0, c1, 8);
        group(xs + (g + 1) * 8 * MB, n0, n1, n - (g + 1) * 8);
    } else if (g < ng) {
        group(xs + g * 8 * MB, c0, c1, n - g * 8);
    }
    } else {
#pragma unroll 1
    for (u32 g = 0; g + 1 < ng; g++) {                // whole groups, the next one prefetched
        const uint4 *np = cp + (size_t)(g + 1) * gs;
        const uint4 n0 = __ldg(np), n1 = __ldg(np + 1);
        group(xs + g * 8 * MB, c0, c1, 8);
        c0 = n0;
        c1 = n1;
    }
    if (ng) group(xs + (ng - 1) * 8 * MB, c0, c1, n - (ng - 1) * 8);
    }
}

// block-wide Σ over threads of v[msg] (MB values): warp shuffles, then one partial per warp in red[w][msg];
// the caller syncs and reads the partials
__device__ __forceinline__ void block_partials(u32 (&v)[MB], u32 *red) {
#pragma unroll
    for (int q = 0; q < MB; q++) {
        u32 x = v[q];
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) x += __shfl_xor_sync(0xFFFFFFFFu, x, o);
        v[q] = x;
    }
    if ((threadIdx.x & 31) == 0) {
#pragma unroll
        for (int q = 0; q < MB; q++) red[(threadIdx.x >> 5) * MB + q] = v[q];
    }
}

// Warp-cooperative version for an output column left over when k + 1 exceeds the CTA's threads by a few:
// lane l sums the inputs i ≡ l (mod 32), then a butterfly of 96-bit adds leaves the total in every lane.
__device__ __forceinline__ void dot_mb_warp(const u32 *__restrict__ mat, u32 ncols, u32 j, const u32 *xs, u32 n,
                                            u32 (&lo)[MB], u32 (&mi)[MB], u32 (&hi)[MB]) {
    const u32 lane = threadIdx.x & 31;
    for (u32 i = lane; i < n; i += 32) {
        const u32 c = __ldg(mat + wch_at(i, j, ncols));
#pragma unroll
        for (int q = 0; q < MB; q++) mac96(lo[q], mi[q], hi[q], xs[i * MB + q], c);
    }
#pragma unroll
    for (int q = 0; q < MB; q++) {
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
            const u32 l2 = __shfl_xor_sync(0xFFFFFFFFu, lo[q], o), m2 = __shfl_xor_sync(0xFFFFFFFFu, mi[q], o);
            const u32 h2 = __shfl_xor_sync(0xFFFFFFFFu, hi[q], o);
            asm("add.cc.u32 %0, %0, %3;\n\taddc.cc.u32 %1, %1, %4;\n\taddc.u32 %2, %2, %5;"
                : "+r"(lo[q]), "+r"(mi[q]), "+r"(hi[q])
                : "r"(l2), "r"(m2), "r"(h2));
        }
    }
}



// Miller-Rabin: per-candidate constants of the CTA's MB candidates (k_mr_rounds_wide)
struct MrCand {
    const u32 *pcw;                    // per-candidate rows (mr_internal.h wmr_*), row r of candidate i at pcw[r cnt + i]
    size_t cnt;
    const u32 *cand;                   // [MB] candidate index of message q (shared memory)
    const u32 *const *mp;              // [MB] multiplicand of message q: channel ch at mp[q][ch mstr] (shared memory)
    u32 mstr;
    __device__ u32 row(u32 r, int q) const { return __ldcg(pcw + (size_t)r * cnt + cand[q]); }
};

template <bool PP>   // PP: dot_mb with ping-pong coefficient groups (faster at k >= 257, slower at 129)
struct Wide {
    const WideArgs &W;
    const u32 *cx;                     // context block (HBM) of this CTA's modulus
    u32 *st;                           // [2k+1][MB]
    u32 *red;                          // [NW][MB] warp partials
    u32 *aux;                          // [4][MB]: t_r, r_r, α', ok
    u32 k, nch, nw;

    __device__ const u32 *T(u32 off) const { return W.tab + off; }

    // st <- st · b · M^-1 (mod N) for the CTA's MB messages; b at bp[ch * bstride + msg * mstride]
    // MRC (Miller-Rabin): every message q has its own modulus n_q; σ, c2, n M^-1 come from mc, b from mc->mp[q], and
    // BE1 is the unmerged per-k contraction (a1w) followed by × c2_j per candidate (6.4)
    template <bool COOP, bool MRC = false>   // COOP: the CTA has fewer threads than k + 1 outputs (leftovers by warps)
    __device__ void mont_mul(const u32 *bp, size_t bstride, u32 mstride, bool sq, const MrCand *mc = nullptr) {
        const WideLayout L = wide_layout(k);
        const u32 tid = threadIdx.x, nt = blockDim.x;
        const u32 *sigw = MRC ? nullptr : cx + W.cxw + wide_cx_sig(k);
        auto mul_b = [&](u32 ch, int q) -> u32 {
            if constexpr (MRC) return __ldcg(mc->mp[q] + (size_t)ch * mc->mstr);
            else return __ldcg(bp + ch * bstride + (size_t)q * mstride);
        };
        // ---- channel products: B: ξ_i = mont(mont(a b) σ_i 2^64) = a b σ_i;  B': t*_j = a* b* 2^-32
        for (u32 ch = tid; ch < 2 * k; ch += nt) {
            const u32 m = __ldg(T(L.mm) + ch), mi = __ldg(T(L.minv) + ch);
            const u32 s = (!MRC && ch < k) ? __ldg(sigw + ch) : 0u;
#pragma unroll 4
            for (int q = 0; q < MB; q++) {
                const u32 a = ST(st, ch, q);
                const u32 b = sq ? a : mul_b(ch, q);
                const u64 pr = (u64)a * b;
                u32 t = mont_red((u32)pr, (u32)(pr >> 32), m, mi);
                if (ch < k) {
                    const u64 ps = (u64)t * (MRC ? mc->row(wmr_sig(k) + ch, q) : s);
                    t = mont_red((u32)ps, (u32)(ps >> 32), m, mi);
                }
                ST(st, ch, q) = t;
            }
        }
        if (tid < MB) {   // m_r: t_r = a_r b_r mod 2^32
            const u32 a = ST(st, 2 * k, tid);
            const u32 b = sq ? a : mul_b(2 * k, (int)tid);
            aux[0 * MB + tid] = a * b;
        }
        __syncthreads();
        // ---- BE1 (approximate, merged with 6.4): thread per output j of B' ∪ {m_r}
        const u32 *A1w = MRC ? T(L.a1w) : cx + W.cxw + wide_cx_a1(k);
        u32 part[MB];
#pragma unroll
        for (int q = 0; q < MB; q++) part[q] = 0;
        // outputs j = 0 .. k (j = k: the m_r column); one per thread for j < nt, and the few left over
        // (k + 1 > nt, e.g. 258 on 256 threads) cooperatively by one warp each
        const u32 lane = tid & 31, warp = tid >> 5;
        auto be1_out = [&](u32 j, bool coop) {
            if (j < k) {
                u32 lo[MB], mi[MB], hi[MB];
#pragma unroll
                for (int q = 0; q < MB; q++) lo[q] = mi[q] = hi[q] = 0;
                if (COOP && coop) dot_mb_warp(A1w, k, j, st, k, lo, mi, hi);
                else dot_mb<PP>(A1w, k, j, st, k, lo, mi, hi);
                const u32 ch = k + j;
                const u32 m = __ldg(T(L.mm) + ch), mv = __ldg(T(L.minv) + ch), r32 = __ldg(T(L.r32) + ch);
                const u32 X = __ldg(T(L.xw) + j), a2r = __ldg(T(L.a2r) + j);
#pragma unroll
                for (int q = 0; q < MB; q++) {
                    if (coop && lane != (u32)q) continue;                              // lane q finishes message q
                    u32 v = red96_mont(hi[q], mi[q], lo[q], m, mv, r32);              // Σ ξ A1'  (mod m'_j)
                    if constexpr (MRC) {                                                // unmerged: × |n M^-1 λ_j| 2^32
                        const u64 pv = (u64)v * mc->row(wmr_c2(k) + j, q);
                        v = mont_red((u32)pv, (u32)(pv >> 32), m, mv);
                    }
                    const u64 p = (u64)ST(st, ch, q) * X;                              // t* C1 2^64
                    const u32 xp = addmod_lazy(mont_red((u32)p, (u32)(p >> 32), m, mv), v, r32);
                    ST(st, ch, q) = xp;                                                // ξ'_j (lazy)
                    part[q] += xp * a2r;                                               // Σ ξ'_j |M'_j|_{2^32}
                }
            } else {   // m_r column: q̂_r = Σ ξ_i |M_i|_{2^32},  r_r = (t_r + q̂_r N) M^-1 mod 2^32
                u32 qr[MB];
#pragma unroll
                for (int q = 0; q < MB; q++) qr[q] = 0;
                for (u32 i = coop ? lane : 0u; i < k; i += coop ? 32u : 1u) {
                    const u32 a1r = __ldg(T(L.a1r) + i);
#pragma unroll
                    for (int q = 0; q < MB; q++) qr[q] += ST(st, i, q) * a1r;
                }
                if (coop) {
#pragma unroll
                    for (int q = 0; q < MB; q++)
#pragma unroll
                        for (int o = 16; o > 0; o >>= 1) qr[q] += __shfl_xor_sync(0xFFFFFFFFu, qr[q], o);
                }
                const u32 minv32 = __ldg(T(L.misc) + 0), nminv = MRC ? 0u : cx[CX_NMINV_R];
                if (!coop || lane == 0) {
#pragma unroll
                    for (int q = 0; q < MB; q++)
                        aux[1 * MB + q] = aux[0 * MB + q] * minv32 + qr[q] * (MRC ? mc->row(wmr_nminv(k), q) : nminv);
                }
            }
        };
        for (u32 j = tid; j <= k && j < nt; j += nt) be1_out(j, false);
        if constexpr (COOP)
            if (k + 1 > nt && nt + warp <= k) be1_out(nt + warp, true);   // leftover outputs, one warp each
        block_partials(part, red);
        __syncthreads();
        if (tid < MB) {   // α' = (Σ ξ'_j |M'_j|_{2^32} - r_r) M'^-1 mod 2^32, exact (Shenoy-Kumaresan)
            u32 sr = 0;
            for (u32 w = 0; w < nw; w++) sr += red[w * MB + tid];
            aux[2 * MB + tid] = (sr - aux[1 * MB + tid]) * __ldg(T(L.misc) + 1);
        }
        __syncthreads();
        // ---- BE2 (exact): thread per output i of B; the m_r slot takes r_r
        const u32 *A2w = T(L.a2w);
        auto be2_out = [&](u32 i, bool coop) {
            const u32 pinw = __ldg(T(L.pinw) + i);
            u32 lo[MB], mi[MB], hi[MB];
#pragma unroll
            for (int q = 0; q < MB; q++) {   // α' (m_i - |M'|_{m_i}) 2^32 (the warp-cooperative sum adds it at the end)
                const u64 p = (COOP && coop) ? 0ull : (u64)aux[2 * MB + q] * pinw;
                lo[q] = (u32)p;
                mi[q] = (u32)(p >> 32);
                hi[q] = 0;
            }
            if (COOP && coop) dot_mb_warp(A2w, k, i, st + k * MB, k, lo, mi, hi);
            else dot_mb<PP>(A2w, k, i, st + k * MB, k, lo, mi, hi);
            const u32 m = __ldg(T(L.mm) + i), mv = __ldg(T(L.minv) + i), r32 = __ldg(T(L.r32) + i);
#pragma unroll
            for (int q = 0; q < MB; q++) {
                if (coop && lane != (u32)q) continue;
                if (COOP && coop) mac96(lo[q], mi[q], hi[q], aux[2 * MB + q], pinw);
                ST(st, i, q) = red96_mont(hi[q], mi[q], lo[q], m, mv, r32);
            }
        };
        for (u32 i = tid; i < k && i < nt; i += nt) be2_out(i, false);
        if constexpr (COOP)
            if (k > nt && nt + warp < k) be2_out(nt + warp, true);
        if (tid < MB) ST(st, 2 * k, tid) = aux[1 * MB + tid];
        __syncthreads();
    }

    // positional -> RNS of x (nl limbs per message, rows xs[l * MB + msg] in shared memory): channel c =
    // Σ_l x_l |2^(32 l)|_{m_c} (B' in ξ-form; the table carries × 2^32 for the Montgomery fold), m_r = x_0
    __device__ void to_rns(const u32 *xs, u32 nl) {
        const WideLayout L = wide_layout(k);
        const u32 tid = threadIdx.x, nt = blockDim.x;
        for (u32 ch = tid; ch < 2 * k; ch += nt) {
            u32 lo[MB], mi[MB], hi[MB];
#pragma unroll
            for (int q = 0; q < MB; q++) lo[q] = mi[q] = hi[q] = 0;
            dot_mb<PP>(T(L.pow), 2 * k, ch, xs, nl, lo, mi, hi);
            const u32 m = __ldg(T(L.mm) + ch), mv = __ldg(T(L.minv) + ch), r32 = __ldg(T(L.r32) + ch);
#pragma unroll
            for (int q = 0; q < MB; q++) ST(st, ch, q) = red96_mont(hi[q], mi[q], lo[q], m, mv, r32);
        }
        if (tid < MB) ST(st, 2 * k, tid) = xs[tid];
        __syncthreads();
    }
};

// Exit (a7): z on B' ∪ {m_r} -> canonical X mod N, written to y rows.  Column sums of
// X = Σ_j ξ'_j M'_j + α'(2^(32(k+1)) - M') go to the scratch rows (3 words per column and message), one
// thread per message then propagates carries and conditionally subtracts N 2^s, s = SMAX..0.
template <bool COOP, bool PP>
__device__ void wide_exit(Wide<PP> &w, u32 *scratch, size_t sstride, const u32 *sslot, u32 *yrow[MB], const bool *okv,
                          u32 out_limbs) {
    const u32 k = w.k, tid = threadIdx.x, nt = blockDim.x;
    const WideLayout L = wide_layout(k);
    u32 part[MB];
#pragma unroll
    for (int q = 0; q < MB; q++) part[q] = 0;
    for (u32 j = tid; j < k; j += nt) {
        const u32 a2r = __ldg(w.T(L.a2r) + j);
#pragma unroll
        for (int q = 0; q < MB; q++) part[q] += ST(w.st, k + j, q) * a2r;
    }
    block_partials(part, w.red);
    __syncthreads();
    if (tid < MB) {
        u32 sr = 0;
        for (u32 v = 0; v < w.nw; v++) sr += w.red[v * MB + tid];
        w.aux[2 * MB + tid] = (sr - ST(w.st, 2 * k, tid)) * __ldg(w.T(L.misc) + 1);
    }
    __syncthreads();
    const u32 lane = tid & 31, warp = tid >> 5;
    auto column = [&](u32 l, bool coop) {
        u32 lo[MB], mi[MB], hi[MB];
        const u32 nmp = __ldg(w.T(L.nmp) + l);
#pragma unroll
        for (int q = 0; q < MB; q++) {
            const u64 p = (COOP && coop) ? 0ull : (u64)w.aux[2 * MB + q] * nmp;
            lo[q] = (u32)p;
            mi[q] = (u32)(p >> 32);
            hi[q] = 0;
        }
        if (COOP && coop) dot_mb_warp(w.T(L.mpl), k + 1, l, w.st + k * MB, k, lo, mi, hi);
        else dot_mb<PP>(w.T(L.mpl), k + 1, l, w.st + k * MB, k, lo, mi, hi);
#pragma unroll
        for (int q = 0; q < MB; q++) {
            if (coop && lane != (u32)q) continue;
            if (COOP && coop) mac96(lo[q], mi[q], hi[q], w.aux[2 * MB + q], nmp);   // + α' (2^(32(k+1)) - M')
            u32 *col = scratch + (size_t)(3 * l) * sstride + sslot[q];
            col[0] = lo[q];
            col[sstride] = mi[q];
            col[2 * sstride] = hi[q];
        }
    };
    for (u32 l = tid; l <= k && l < nt; l += nt) column(l, false);
    if constexpr (COOP)
        if (k + 1 > nt && nt + warp <= k) column(nt + warp, true);   // leftover columns, one warp each
    __threadfence_block();
    __syncthreads();
    if (tid < MB) {   // carries, then X mod N by conditional subtraction of N 2^s
        const u32 q = tid;
        u64 carry = 0;   // < 2^42
        for (u32 l = 0; l <= k; l++) {
            const u32 *col = scratch + (size_t)(3 * l) * sstride + sslot[q];
            const u32 lo = col[0], mi = col[sstride], hi = col[2 * sstride];
            const u64 s = (u64)lo + (u32)carry;                    // limb l of X
            ST(w.st, l, q) = (u32)s;
            carry = (carry >> 32) + mi + ((u64)hi << 32) + (s >> 32);
        }
        const u32 *nl = w.cx + cx_n(k);
        const int smax = (int)(32 - __clz(k + 2)) - 1;   // X < (k+3) N <= 2^(smax+1) N (as mr_kernels.cuh SMAX)
        for (int s = smax; s >= 0; s--) {
            for (int pass = 0; pass < 2; pass++) {
                u32 br = 0;
                for (u32 l = 0; l <= k; l++) {
                    const u32 nlo = l ? nl[l - 1] : 0u, nhi = l < k ? nl[l] : 0u;
                    const u32 nsh = s ? __funnelshift_l(nlo, nhi, s) : nhi;
                    const u64 t = (u64)ST(w.st, l, q) - nsh - br;
                    if (pass) ST(w.st, l, q) = (u32)t;
                    br = (u32)(t >> 63);
                }
                if (br) break;
            }
        }
        if (yrow[q])
            for (u32 l = 0; l < out_limbs; l++) yrow[q][l] = okv[q] ? ST(w.st, l, q) : 0u;
    }
    __syncthreads();
}

// modexp interpreter (same op programs as k_modexp, mr_internal.h make_op), CTA = MB messages of one context
// NTB/MINB: register budget — 512 threads x 1 CTA (k = 505) or 256 threads x 2 CTAs per SM (k <= 257)
template <int NTB, int MINB, bool COOP, bool PP>
__global__ void __launch_bounds__(NTB, MINB) k_modexp_wide(const ModexpParams P, const WideArgs W) {
    extern __shared__ __align__(16) u32 smem[];
    const u32 k = W.k, nch = 2 * k + 1, nw = blockDim.x / 32, tid = threadIdx.x;
    u32 *st = smem;                                   // [nch][MB]
    u32 *xs = st + nch * MB;                          // [k][MB] staged input limbs
    u32 *red = xs + k * MB;                           // [16][MB]
    u32 *aux = red + 16 * MB;                         // [4][MB]
    __shared__ bool okv[MB];
    __shared__ u32 sslot[MB];
    const u32 sel = blockIdx.x >= P.ctas0 ? 1u : 0u;
    const u32 *cx = sel ? P.ctx[1] : P.ctx[0];
    const u32 j0 = (blockIdx.x - sel * P.ctas0) * MB;
    Wide<PP> w{W, cx, st, red, aux, k, nch, nw};
    if (tid < MB) {
        const u32 jl = j0 + tid;
        const bool valid = jl < P.count;
        bool ok = false;
        if (valid) {   // x < input bound (little-endian limbs, most significant first)
            const u32 *xr = P.x + (size_t)jl * P.in_limbs, *bnd = cx + cx_inb(k);
            int res = 0;
            for (int l = (int)P.in_limbs - 1; l >= 0 && res == 0; l--) res = xr[l] < bnd[l] ? -1 : (xr[l] > bnd[l] ? 1 : 0);
            ok = res < 0;
            if (sel == 0 && P.status) P.status[jl] = ok ? 0 : 5 /* MR_ERR_RANGE */;
        }
        okv[tid] = ok;
        sslot[tid] = sel * P.ctas0 * MB + jl;
    }
    __syncthreads();
    const u64 *prog = sel ? P.prog[1] : P.prog[0];
    const u32 nops = sel ? P.nops[1] : P.nops[0];
    const size_t tstride = P.jobs_total, entry = (size_t)nch * tstride;
    const u32 slot0 = sel * P.ctas0 * MB + j0;
    for (u32 s = 0; s < nops; s++) {
        const u64 op = __ldg(prog + s);
        const u32 fl = (u32)op & 0xFF, opnd = (u32)(op >> 8) & 0xFF, ld = (u32)(op >> 16) & 0xFF;
        const u32 ad = (u32)(op >> 24) & 0xFF, sto = (u32)(op >> 32) & 0xFF;
        if (fl & (OPF_TORNS_ALL | OPF_TORNS_LO | OPF_TORNS_HI)) {
            const u32 off = (fl & OPF_TORNS_HI) ? P.half : 0u;
            const u32 nl = (fl & OPF_TORNS_ALL) ? P.in_limbs : P.half;
            for (u32 e = tid; e < nl * MB; e += blockDim.x) {
                const u32 l = e / MB, q = e % MB, jl = j0 + q;
                xs[l * MB + q] = okv[q] ? P.x[(size_t)jl * P.in_limbs + off + l] : 0u;
            }
            __syncthreads();
            w.to_rns(xs, nl);
        }
        if (fl & OPF_LOAD) {
            for (u32 e = tid; e < nch * MB; e += blockDim.x) {
                const u32 ch = e / MB, q = e % MB;
                st[e] = ld >= 0xF0 ? cx[cx_r2(k) + (ld - 0xF0) * nch + ch] : P.table[ld * entry + ch * tstride + slot0 + q];
            }
            __syncthreads();
        }
        if (!(fl & OPF_NOMUL)) {
            if (opnd == OPND_SQ) w.template mont_mul<COOP>(nullptr, 0, 0, true);
            else if (opnd >= 0xF0) w.template mont_mul<COOP>(cx + cx_r2(k) + (opnd - 0xF0) * nch, 1, 0, false);
            else w.template mont_mul<COOP>(P.table + opnd * entry + slot0, tstride, 1, false);
        }
        if (fl & OPF_ADD) {   // channel-wise lazy modular addition (CRT entry)
            const WideLayout L = wide_layout(k);
            for (u32 e = tid; e < nch * MB; e += blockDim.x) {
                const u32 ch = e / MB, q = e % MB;
                const u32 b = P.table[ad * entry + ch * tstride + slot0 + q];
                st[e] = ch < 2 * k ? addmod_lazy(st[e], b, __ldg(W.tab + L.r32 + ch)) : st[e] + b;
            }
            __syncthreads();
        }
        if (fl & OPF_STORE) {
            for (u32 e = tid; e < nch * MB; e += blockDim.x) {
                const u32 ch = e / MB, q = e % MB;
                P.table[sto * entry + ch * tstride + slot0 + q] = st[e];
            }
            __syncthreads();
        }
    }
    u32 *yrow[MB];
#pragma unroll
    for (int q = 0; q < MB; q++) {
        const u32 jl = j0 + q;
        yrow[q] = jl < P.count ? P.y + sel * P.out_stride + (size_t)jl * P.out_limbs : nullptr;
    }
    // column scratch: the window table (no longer needed) — 3(k+1) rows <= table_slots(w) (2k+1) rows
    wide_exit<COOP, PP>(w, P.table, tstride, sslot, yrow, okv, P.out_limbs);
}

}  // namespace

size_t wide_smem_bytes(u32 k) {
    return 4 * ((size_t)(2 * k + 1) * MB + (size_t)k * MB + 16 * MB + 4 * MB);
}
int wide_messages_per_cta() { return MB; }

int launch_modexp_wide(const ModexpParams &p, u32 ctas, const u32 *d_wide_tab, u32 k, u32 cxw, void *stream) {
    WideArgs W{d_wide_tab, k, 0, cxw};
    // threads: one per base-extension output (k + 1 with the m_r column), rounded to whole warps — except
    // when k + 1 overshoots a multiple of 32 by at most 4 (k = 257: 258 -> 256 threads, the two extra
    // outputs done by one warp each), which keeps the warps a multiple of the 4 SM sub-partitions
    const u32 up = 32 * ((k + 1 + 31) / 32), down = 32 * ((k + 1) / 32);
    const u32 nt32 = (k + 1) - down <= 4 && down >= 64 ? down : up, nt = nt32 < (u32)NTMAX ? nt32 : (u32)NTMAX;
    W.nt = nt;
    const size_t smem = wide_smem_bytes(k);
    // ping-pong coefficient groups: A/B +8 % at k = 257, +5 % at 505, -13 % at 129 (tools/ab_w.sh)
    static const u32 pp_min = [] { const char *e = getenv("MR_WIDE_PP_MIN"); return e ? (u32)atoi(e) : 257u; }();
    const bool pp = k >= pp_min;
    // k = 97 (96 threads): a 168-register budget (no accumulator-pair shuffling) beats the 128-register
    // one by 5-8 %; at k = 129 (128 threads) the 4th resident CTA is worth more (tools/ab_k129.py)
    const void *kern = nt > 256 ? (const void *)k_modexp_wide<NTMAX, 1, false, true>
                       : pp     ? (const void *)k_modexp_wide<256, 2, true, true>
                       : nt <= 96 ? (const void *)k_modexp_wide<128, 3, true, false>
                                : (const void *)k_modexp_wide<256, 2, true, false>;
    if (cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) != cudaSuccess) return 6;
    void *args[] = {const_cast<ModexpParams *>(&p), &W};
    return cudaLaunchKernel(kern, dim3(ctas), dim3(nt), args, smem, (cudaStream_t)stream) == cudaSuccess ? 0 : 6;
}

}  // namespace mr

// ------------------------------------------------------------------ CRT recombination for wide halves (a8)
// One thread per message, positional (O(H²) word operations, negligible next to the two ladders):
//   t = m_q mod p;  d = (m_p - t) mod p;  h = d·q_inv mod p (schoolbook product, Knuth Algorithm D
//   remainder, TAOCP 4.3.1);  m = m_q + q·h  (Garner, HAC 14.71).  scratch: [count][2H + 2] words.
namespace mr {
namespace {

// u[0, ulen) mod v[0, n) in place (remainder left in u[0, n)); v top limb non-zero; u needs ulen + 1 words
__device__ void rem_knuth_row(u32 *u, u32 ulen, const u32 *v, u32 n) {
    const u32 sh = __clz(v[n - 1]);
    auto vn = [&](u32 l) -> u32 { return sh ? (v[l] << sh) | (l ? v[l - 1] >> (32 - sh) : 0u) : v[l]; };
    if (sh) {
        u[ulen] = u[ulen - 1] >> (32 - sh);
        for (int l = (int)ulen - 1; l > 0; l--) u[l] = (u[l] << sh) | (u[l - 1] >> (32 - sh));
        u[0] <<= sh;
    } else {
        u[ulen] = 0;
    }
    if (ulen >= n) {
        const u32 vt = vn(n - 1), vs = n > 1 ? vn(n - 2) : 0u;
        for (int j = (int)(ulen - n); j >= 0; j--) {
            const u64 num = ((u64)u[j + n] << 32) | u[j + n - 1];
            u64 qh = num / vt, rh = num - qh * vt;
            while (qh >> 32 || (n > 1 && qh * vs > ((rh << 32) | u[j + n - 2]))) {
                qh--;
                rh += vt;
                if (rh >> 32) break;
            }
            u64 carry = 0;
            long long br = 0;
            for (u32 i = 0; i < n; i++) {
                const u64 pr = qh * vn(i) + carry;
                carry = pr >> 32;
                const long long t = (long long)u[i + j] - (long long)(u32)pr + br;
                u[i + j] = (u32)t;
                br = t >> 32;
            }
            const long long t = (long long)u[j + n] - (long long)carry + br;
            u[j + n] = (u32)t;
            if (t < 0) {   // add back (probability ~2/2^32)
                u64 c = 0;
                for (u32 i = 0; i < n; i++) {
                    const u64 s2 = (u64)u[i + j] + vn(i) + c;
                    u[i + j] = (u32)s2;
                    c = s2 >> 32;
                }
                u[j + n] += (u32)c;
            }
        }
    }
    if (sh)
        for (u32 l = 0; l < n; l++) u[l] = (u[l] >> sh) | (l + 1 < n ? u[l + 1] << (32 - sh) : 0u);
}

__global__ void k_combine_wide(const CombineParams P, const u32 *qinv, u32 *scr, u32 k) {
    const u32 i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= P.count) return;
    const u32 H = P.half;
    const u32 *mp = P.mpq + (size_t)i * H, *mq = P.mpq + ((size_t)P.count + i) * H;
    const u32 *pl = P.ctx_p + cx_n(k);
    u32 *mrow = P.m + (size_t)i * 2 * H;
    u32 *t = scr + (size_t)i * (2 * H + 2);
    u32 n = H;
    while (n > 1 && pl[n - 1] == 0) n--;
    // t = m_q mod p
    for (u32 l = 0; l < H; l++) t[l] = mq[l];
    rem_knuth_row(t, H, pl, n);
    // d = m_p - t (mod p) -> mrow[0, H)
    u32 br = 0;
    for (u32 l = 0; l < H; l++) {
        const u64 d = (u64)mp[l] - (l < n ? t[l] : 0u) - br;
        mrow[l] = (u32)d;
        br = (u32)(d >> 63);
    }
    if (br) {
        u32 c = 0;
        for (u32 l = 0; l < H; l++) {
            const u64 s2 = (u64)mrow[l] + (l < n ? pl[l] : 0u) + c;
            mrow[l] = (u32)s2;
            c = (u32)(s2 >> 32);
        }
    }
    // h = d q_inv mod p: product into t[0, 2H), remainder -> t[0, n)
    for (u32 l = 0; l < 2 * H; l++) t[l] = 0;
    for (u32 a = 0; a < H; a++) {
        const u32 da = mrow[a];
        u64 c = 0;
        for (u32 b = 0; b < H; b++) {
            const u64 v = (u64)da * qinv[b] + t[a + b] + c;
            t[a + b] = (u32)v;
            c = v >> 32;
        }
        t[a + H] = (u32)c;
    }
    rem_knuth_row(t, 2 * H, pl, n);
    // m = m_q + q h  (product scanning)
    const bool bad = P.status && P.status[i] != 0;
    u32 lo = 0, mi = 0, hi = 0;
    for (u32 col = 0; col < 2 * H; col++) {
        if (col < H) mac96(lo, mi, hi, mq[col], 1u);
        const u32 r0 = col >= H ? col - H + 1 : 0u, r1 = col < H ? col : H - 1;
        for (u32 r = r0; r <= r1; r++)
            if (col - r < n) mac96(lo, mi, hi, P.q[r], t[col - r]);
        mrow[col] = bad ? 0u : lo;
        lo = mi;
        mi = hi;
        hi = 0;
    }
}

}  // namespace

int launch_combine_wide(const CombineParams &p, const u32 *d_qinv, u32 *d_scratch, u32 k, void *stream) {
    const u32 nt = 128;
    void *args[] = {const_cast<CombineParams *>(&p), const_cast<u32 **>(&d_qinv), &d_scratch, &k};
    return cudaLaunchKernel((const void *)k_combine_wide, dim3((p.count + nt - 1) / nt), dim3(nt), args, 0,
                            (cudaStream_t)stream) == cudaSuccess
               ? 0
               : 6;
}

}  // namespace mr

// ------------------------------------------------------------------ Miller-Rabin on wide candidates (k = 257, 505)
// P:50 §3.2 ("Miller-Rabin tests ... in the Montgomery domain"), HAC 4.24, for candidates of 4,097 .. 16,128 bits
// (keys up to 16,128 bits).  Every candidate has its own modulus n, so the 6.4 step cannot be merged into a
// per-context BE1 matrix as in the modexp kernel: BE1 contracts with the per-k |M_i|_{m'_j} 2^32 (wide table a1w) and
// the epilogue multiplies by the candidate's c2_j = |n M^-1 λ_j| 2^32; σ_i, c2_j, n M^-1 mod 2^32, the RNS image of
// M^2 mod n, s and d come from a per-candidate setup kernel (rows wmr_* of mr_internal.h).  Same channels-on-threads
// mapping as k_modexp_wide: MB = 16 candidates per CTA, one thread per output channel.
namespace mr {
namespace {

__host__ __device__ constexpr u32 wmr_scr_words(u32 k) { return 3 * k + 4; }

struct WmrArgs {
    const u32 *tab;          // wide table (wide_layout)
    u32 k, nt;
    u32 *pcw;                // [wmr_words(k)][count] per-candidate rows
    u32 *scr;                // [count][wmr_scr_words(k)] setup scratch (positional M^2 mod n)
    const u32 *n;            // [count][limbs]
    const u32 *bases;        // [count][rounds][limbs]
    u32 count, limbs, rounds, window, forced;
    u32 *table;              // [E + 3 slots][2k + 1][count]: window table, stash, exit column scratch (2 slots)
    uint8_t *verdict;
    int16_t *witness;
    int32_t *status;
};

__device__ __forceinline__ u32 wmr_mulm(u32 a, u32 b, u32 m) { return (u32)((u64)a * b % m); }
__device__ u32 wmr_powm(u32 a, u32 e, u32 m) {
    u32 r = 1;
    while (e) {
        if (e & 1) r = wmr_mulm(r, a, m);
        a = wmr_mulm(a, a, m);
        e >>= 1;
    }
    return r;
}

// per-candidate constants (thread per candidate): input rules, residues of n (factor test, reading R14), σ, c2,
// n M^-1 mod 2^32, s and d (n - 1 = 2^s d), and the RNS image of R^2 mod n (R = M) by Knuth remainders
__global__ void k_mr_setup_wide(const WmrArgs A) {
    const u32 i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= A.count) return;
    const u32 k = A.k, L = A.limbs;
    const size_t cnt = A.count;
    const WideLayout W = wide_layout(k);
    u32 *pc = A.pcw + i;
    auto row = [&](u32 r) -> u32 & { return pc[(size_t)r * cnt]; };
    const u32 *nrow = A.n + (size_t)i * L;
    for (u32 l = 0; l <= k; l++) row(wmr_n(k) + l) = l < L ? nrow[l] : 0u;
    u32 nz = 0;
    for (u32 l = 1; l < L; l++) nz |= nrow[l];
    const bool small = nz == 0;
    int32_t status = 0;
    u32 live = 1, verdict = 0 /* composite */;
    if (!(nrow[0] & 1u) || (small && nrow[0] < 5u)) { status = 5; live = 0; }
    if (live) {
        // residues of n in every channel: Horner over the limbs (one 64-bit remainder per limb and channel)
        bool factor = false;
        for (u32 c = 0; c < 2 * k && !factor; c++) {
            const u32 m = __ldg(A.tab + W.mm + c);
            u32 r = 0;
            for (int l = (int)L - 1; l >= 0; l--) r = (u32)((((u64)r << 32) | nrow[l]) % m);
            if (r == 0) { factor = true; break; }
            const u32 r32 = __ldg(A.tab + W.r32 + c);
            if (c < k) {   // σ_i = -(n M_i)^-1 mod m_i, stored × 2^64
                const u32 x = wmr_mulm(r, __ldg(A.tab + W.mis + c), m);
                const u32 sg = (m - wmr_powm(x, m - 2, m)) % m;
                row(wmr_sig(k) + c) = wmr_mulm(wmr_mulm(sg, r32, m), r32, m);
            } else {       // c2_j = |n M^-1 λ_j|, stored × 2^32
                const u32 j = c - k;
                const u32 c2 = wmr_mulm(wmr_mulm(r, __ldg(A.tab + W.lam + j), m), __ldg(A.tab + W.mu + j), m);
                row(wmr_c2(k) + j) = wmr_mulm(c2, r32, m);
            }
        }
        if (factor) {
            live = 0;
            if (small) { status = 3; verdict = 1; }   // n is itself a base prime (MR_ERR_NOT_COPRIME)
            else verdict = 2;                          // MR_FACTOR (reading R14)
        }
    }
    if (live) {
        row(wmr_nminv(k)) = nrow[0] * __ldg(A.tab + W.misc + 0);
        u32 l0 = 0, w0 = nrow[0] & ~1u;
        while (w0 == 0 && l0 + 1 < L) w0 = nrow[++l0];
        const u32 s = 32 * l0 + __ffs(w0) - 1, ls = s / 32, bs = s % 32;
        for (u32 l = 0; l < k; l++) {
            const u32 a0 = l + ls < L ? nrow[l + ls] : 0u, a1 = l + ls + 1 < L ? nrow[l + ls + 1] : 0u;
            row(wmr_d(k) + l) = __funnelshift_r(l + ls == 0 ? (a0 & ~1u) : a0, a1, bs);
        }
        row(wmr_s(k)) = s;
        // R^2 mod n, positional: rho = M mod n, then rho^2 mod n (Knuth Algorithm D remainders)
        u32 Ln = L;
        while (Ln > 1 && nrow[Ln - 1] == 0) Ln--;
        u32 *u = A.scr + (size_t)i * wmr_scr_words(k);    // [2k + 2] remainders, then [k] rho
        for (u32 l = 0; l <= k; l++) u[l] = __ldg(A.tab + W.ml + l);
        rem_knuth_row(u, k + 1, nrow, Ln);
        u32 *t = u + 2 * k + 2;
        for (u32 l = 0; l < Ln; l++) t[l] = u[l];          // rho (Ln <= k - 1 words)
        for (u32 l = 0; l < 2 * Ln + 1; l++) u[l] = 0;
        for (u32 a = 0; a < Ln; a++) {
            u64 c = 0;
            for (u32 b = 0; b < Ln; b++) {
                const u64 v = (u64)t[a] * t[b] + u[a + b] + c;
                u[a + b] = (u32)v;
                c = v >> 32;
            }
            u[a + Ln] = (u32)c;
        }
        rem_knuth_row(u, 2 * Ln, nrow, Ln);
        // RNS image: B plain, B' in ξ-form (× λ_j), m_r = low limb
        for (u32 c = 0; c < 2 * k; c++) {
            const u32 m = __ldg(A.tab + W.mm + c);
            u32 r = 0;
            for (int l = (int)Ln - 1; l >= 0; l--) r = (u32)((((u64)r << 32) | u[l]) % m);
            row(wmr_r2(k) + c) = c < k ? r : wmr_mulm(r, __ldg(A.tab + W.lam + (c - k)), m);
        }
        row(wmr_r2(k) + 2 * k) = u[0];
    }
    row(wmr_live(k)) = live;
    A.verdict[i] = (uint8_t)verdict;
    if (A.witness) A.witness[i] = -1;
    if (A.status) A.status[i] = status;
}

// exit of the CTA's MB candidates (as wide_exit, with the candidate's own n): X mod n_q in st rows 0..k
template <bool COOP, bool PP>
__device__ void wmr_exit(Wide<PP> &w, const MrCand &mc, u32 *scratch, size_t sstride, const u32 *sslot) {
    const u32 k = w.k, tid = threadIdx.x, nt = blockDim.x;
    const WideLayout L = wide_layout(k);
    u32 part[MB];
#pragma unroll
    for (int q = 0; q < MB; q++) part[q] = 0;
    for (u32 j = tid; j < k; j += nt) {
        const u32 a2r = __ldg(w.T(L.a2r) + j);
#pragma unroll
        for (int q = 0; q < MB; q++) part[q] += ST(w.st, k + j, q) * a2r;
    }
    block_partials(part, w.red);
    __syncthreads();
    if (tid < MB) {
        u32 sr = 0;
        for (u32 v = 0; v < w.nw; v++) sr += w.red[v * MB + tid];
        w.aux[2 * MB + tid] = (sr - ST(w.st, 2 * k, tid)) * __ldg(w.T(L.misc) + 1);
    }
    __syncthreads();
    const u32 lane = tid & 31, warp = tid >> 5;
    auto column = [&](u32 l, bool coop) {
        u32 lo[MB], mi[MB], hi[MB];
        const u32 nmp = __ldg(w.T(L.nmp) + l);
#pragma unroll
        for (int q = 0; q < MB; q++) {
            const u64 p = (COOP && coop) ? 0ull : (u64)w.aux[2 * MB + q] * nmp;
            lo[q] = (u32)p;
            mi[q] = (u32)(p >> 32);
            hi[q] = 0;
        }
        if (COOP && coop) dot_mb_warp(w.T(L.mpl), k + 1, l, w.st + k * MB, k, lo, mi, hi);
        else dot_mb<PP>(w.T(L.mpl), k + 1, l, w.st + k * MB, k, lo, mi, hi);
#pragma unroll
        for (int q = 0; q < MB; q++) {
            if (coop && lane != (u32)q) continue;
            if (COOP && coop) mac96(lo[q], mi[q], hi[q], w.aux[2 * MB + q], nmp);
            u32 *col = scratch + (size_t)(3 * l) * sstride + sslot[q];
            col[0] = lo[q];
            col[sstride] = mi[q];
            col[2 * sstride] = hi[q];
        }
    };
    for (u32 l = tid; l <= k && l < nt; l += nt) column(l, false);
    if constexpr (COOP)
        if (k + 1 > nt && nt + warp <= k) column(nt + warp, true);
    __threadfence_block();
    __syncthreads();
    if (tid < MB) {
        const u32 q = tid;
        u64 carry = 0;
        for (u32 l = 0; l <= k; l++) {
            const u32 *col = scratch + (size_t)(3 * l) * sstride + sslot[q];
            const u64 s = (u64)col[0] + (u32)carry;
            ST(w.st, l, q) = (u32)s;
            carry = (carry >> 32) + col[sstride] + ((u64)col[2 * sstride] << 32) + (s >> 32);
        }
        const int smax = (int)(32 - __clz(k + 2)) - 1;
        for (int s = smax; s >= 0; s--) {
            for (int pass = 0; pass < 2; pass++) {
                u32 br = 0;
                for (u32 l = 0; l <= k; l++) {
                    const u32 nlo = l ? mc.row(wmr_n(k) + l - 1, q) : 0u, nhi = mc.row(wmr_n(k) + l, q);
                    const u32 nsh = s ? __funnelshift_l(nlo, nhi, s) : nhi;
                    const u64 t = (u64)ST(w.st, l, q) - nsh - br;
                    if (pass) ST(w.st, l, q) = (u32)t;
                    br = (u32)(t >> 63);
                }
                if (br) break;
            }
        }
    }
    __syncthreads();
}

// HAC 4.24 for MB candidates per CTA, every round r with the caller's base a_{i,r}: fixed-window a^d (window w, the
// table T[e] = a^e R for e < 2^w per candidate), then up to s - 1 squarings looking for n - 1; the CTA skips a round
// when none of its candidates is pending (early exit; forced: every live candidate runs every round).
template <int NTB, int MINB, bool COOP, bool PP>
__global__ void __launch_bounds__(NTB, MINB) k_mr_rounds_wide(const WmrArgs A) {
    extern __shared__ __align__(16) u32 smem[];
    const u32 k = A.k, nch = 2 * k + 1, nw = blockDim.x / 32, tid = threadIdx.x, L = A.limbs;
    u32 *st = smem;
    u32 *xs = st + nch * MB;
    u32 *red = xs + k * MB;
    u32 *aux = red + 16 * MB;
    __shared__ u32 cand[MB], sslot[MB], dig[MB];
    __shared__ const u32 *mp[MB];
    __shared__ u32 live_s[MB], pend[MB], need[MB], pass_s[MB], jj_s[MB], verd[MB], anyf;
    __shared__ int wit[MB];
    const size_t cnt = A.count, tstride = A.count, entry = (size_t)nch * tstride;
    const u32 j0 = blockIdx.x * MB;
    const u32 E = 1u << A.window, ndig = (32 * L + A.window - 1) / A.window;
    WideArgs WA{A.tab, k, blockDim.x, 0};
    Wide<PP> w{WA, nullptr, st, red, aux, k, nch, nw};
    MrCand mc{A.pcw, cnt, cand, mp, 0};
    if (tid < MB) {
        const u32 i = j0 + tid < A.count ? j0 + tid : A.count - 1;   // tail lanes shadow the last candidate
        cand[tid] = i;
        sslot[tid] = i;
        live_s[tid] = j0 + tid < A.count ? A.pcw[(size_t)wmr_live(k) * cnt + i] : 0u;
        verd[tid] = 1;
        wit[tid] = -1;
        if (live_s[tid]) {   // base rule for every round first (HAC 4.24 input): 2 <= a <= n - 2
            const u32 *nrow = A.n + (size_t)i * L;
            bool bad = false;
            for (u32 r = 0; r < A.rounds && !bad; r++) {
                const u32 *a = A.bases + ((size_t)i * A.rounds + r) * L;
                u32 br = 0, dhi = 0, ahi = 0, d0 = 0;
                for (u32 l = 0; l < L; l++) {
                    const u64 t = (u64)nrow[l] - a[l] - br;
                    br = (u32)(t >> 63);
                    if (l) { dhi |= (u32)t; ahi |= a[l]; } else d0 = (u32)t;
                }
                bad = !(ahi || a[0] >= 2u) || !(!br && (dhi || d0 >= 2u));
            }
            if (bad) {
                if (A.status) A.status[i] = 5;
                verd[tid] = 0;          // composite, no witness round (as k_mr_rounds)
                live_s[tid] = 0;
            }
        }
        pend[tid] = live_s[tid];
    }
    __syncthreads();
    const u32 *tab0 = A.table;
#pragma unroll 1
    for (u32 r = 0; r < A.rounds; r++) {
        if (tid == 0) {
            u32 a = 0;
            for (int q = 0; q < MB; q++) a |= pend[q] | (A.forced ? live_s[q] : 0u);
            anyf = a;
        }
        __syncthreads();
        if (!anyf) break;
        // uniform part: T0 = mm(R^2, 1) = R, T1 = mm(a, R^2) = a R, T[e] = T[e-1] T1; the ladder starts at T0
        for (u32 u = 0; u < E + ndig * (A.window + 1); u++) {
            bool sq = false;
            if (u == 0) {
                for (u32 e = tid; e < nch * MB; e += blockDim.x) {
                    const u32 ch = e / MB, q = e % MB;
                    st[e] = A.pcw[(size_t)(wmr_r2(k) + ch) * cnt + cand[q]];
                }
                if (tid < MB) mp[tid] = A.tab + wide_layout(k).one;
                mc.mstr = 1;
            } else if (u == 1) {
                for (u32 e = tid; e < L * MB; e += blockDim.x) {
                    const u32 l = e / MB, q = e % MB;
                    xs[l * MB + q] = A.bases[((size_t)cand[q] * A.rounds + r) * L + l];
                }
                __syncthreads();
                w.to_rns(xs, L);
                if (tid < MB) mp[tid] = A.pcw + (size_t)wmr_r2(k) * cnt + cand[tid];
                mc.mstr = (u32)cnt;
            } else if (u < E) {
                if (tid < MB) mp[tid] = tab0 + entry + cand[tid];
                mc.mstr = (u32)tstride;
            } else {
                const u32 qq = u - E, dg = ndig - 1 - qq / (A.window + 1), sub = qq % (A.window + 1);
                if (qq == 0) {
                    for (u32 e = tid; e < nch * MB; e += blockDim.x) {
                        const u32 ch = e / MB, q = e % MB;
                        st[e] = tab0[ch * tstride + cand[q]];
                    }
                }
                if (sub < A.window) {
                    sq = true;
                } else {
                    if (tid < MB) {
                        const u32 b0 = dg * A.window, lw = b0 / 32, bw = b0 % 32;
                        const u32 *dl = A.pcw + (size_t)wmr_d(k) * cnt + cand[tid];
                        const u32 lo = lw < k ? dl[(size_t)lw * cnt] : 0u, hi = lw + 1 < k ? dl[(size_t)(lw + 1) * cnt] : 0u;
                        mp[tid] = tab0 + (size_t)(__funnelshift_r(lo, hi, bw) & (E - 1)) * entry + cand[tid];
                    }
                    mc.mstr = (u32)tstride;
                }
            }
            __syncthreads();
            w.template mont_mul<COOP, true>(nullptr, 0, 0, sq, &mc);

            if (u < E) {
                for (u32 e = tid; e < nch * MB; e += blockDim.x) {
                    const u32 ch = e / MB, q = e % MB;
                    A.table[u * entry + ch * tstride + cand[q]] = st[e];
                }
                __syncthreads();
            }
        }
        // checks: even steps leave the Montgomery domain (× 1) and compare with 1 and n - 1, odd steps square
        if (tid < MB) {
            need[tid] = pend[tid] | (A.forced ? live_s[tid] : 0u);
            pass_s[tid] = 0;
            jj_s[tid] = 0;
        }
        __syncthreads();
        u32 *stash = A.table + (size_t)E * entry;
        for (u32 v = 0;; v++) {
            const bool check = (v % 2) == 0;
            if (check) {
                for (u32 e = tid; e < nch * MB; e += blockDim.x) {
                    const u32 ch = e / MB, q = e % MB;
                    stash[ch * tstride + cand[q]] = st[e];
                }
                if (tid < MB) mp[tid] = A.tab + wide_layout(k).one;
                mc.mstr = 1;
            }
            __syncthreads();
            w.template mont_mul<COOP, true>(nullptr, 0, 0, !check, &mc);
            if (check) {
                wmr_exit<COOP, PP>(w, mc, A.table + (size_t)(E + 1) * entry, tstride, sslot);
                if (tid < MB) {
                    const u32 q = tid;
                    u32 one = ST(st, 0, q) ^ 1u, nm1 = ST(st, 0, q) ^ (mc.row(wmr_n(k), q) - 1u);
                    for (u32 l = 1; l <= k; l++) {
                        one |= ST(st, l, q);
                        nm1 |= ST(st, l, q) ^ mc.row(wmr_n(k) + l, q);
                    }
                    if (need[q]) {
                        const u32 s = mc.row(wmr_s(k), q);
                        if (nm1 == 0) { pass_s[q] = 1; need[q] = 0; }
                        else if (one == 0) { pass_s[q] = jj_s[q] == 0; need[q] = 0; }
                        else if (jj_s[q] + 1 >= s) need[q] = 0;
                    }
                    jj_s[q]++;
                }
                __syncthreads();   // the comparisons read st rows 0..k: restore the state only after them
                for (u32 e = tid; e < nch * MB; e += blockDim.x) {
                    const u32 ch = e / MB, q = e % MB;
                    st[e] = stash[ch * tstride + cand[q]];
                }
                if (tid == 0) {
                    u32 a = 0;
                    for (int q = 0; q < MB; q++) a |= need[q];
                    anyf = a;
                }
                __syncthreads();
                if (!anyf) break;
            }
        }
        if (tid < MB) {
            const u32 q = tid;
            if (pend[q] && !pass_s[q]) {
                if (verd[q] == 1) { verd[q] = 0; wit[q] = (int)r; }
                if (!A.forced) pend[q] = 0;
            }
        }
        __syncthreads();
    }
    if (tid < MB && j0 + tid < A.count && A.pcw[(size_t)wmr_live(k) * cnt + cand[tid]]) {
        const u32 i = cand[tid];
        A.verdict[i] = (uint8_t)verd[tid];
        if (A.witness) A.witness[i] = (int16_t)wit[tid];
    }
}

}  // namespace

// Miller-Rabin for wide candidates (k = 257, 505): setup (thread per candidate), then the rounds (16 per CTA)
int launch_mr_wide(const u32 *d_wide_tab, u32 k, u32 *d_pcw, u32 *d_scr, const u32 *d_n, const u32 *d_bases, u32 count,
                   u32 limbs, u32 rounds, u32 window, u32 forced, u32 *d_table, uint8_t *d_verdict, int16_t *d_witness,
                   int32_t *d_status, void *stream) {
    WmrArgs A{d_wide_tab, k, 0, d_pcw, d_scr, d_n, d_bases, count, limbs, rounds, window, forced, d_table, d_verdict,
              d_witness, d_status};
    cudaStream_t st = (cudaStream_t)stream;
    {
        void *args[] = {&A};
        if (cudaLaunchKernel((const void *)k_mr_setup_wide, dim3((count + 63) / 64), dim3(64), args, 0, st) != cudaSuccess)
            return 6;
    }
    const u32 up = 32 * ((k + 1 + 31) / 32), down = 32 * ((k + 1) / 32);
    const u32 nt32 = (k + 1) - down <= 4 && down >= 64 ? down : up, nt = nt32 < (u32)NTMAX ? nt32 : (u32)NTMAX;
    A.nt = nt;
    const size_t smem = wide_smem_bytes(k);
    const void *kern = nt > 256 ? (const void *)k_mr_rounds_wide<NTMAX, 1, false, true>
                                : (const void *)k_mr_rounds_wide<256, 2, true, true>;
    if (cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) != cudaSuccess) return 6;
    void *args[] = {&A};
    return cudaLaunchKernel(kern, dim3((count + MB - 1) / MB), dim3(nt), args, smem, st) == cudaSuccess ? 0 : 6;
}
// test hook: the per-candidate setup alone (rows wmr_* into d_pcw)
int launch_mr_wide_setup(const u32 *d_wide_tab, u32 k, u32 *d_pcw, u32 *d_scr, const u32 *d_n, u32 count, u32 limbs,
                         uint8_t *d_verdict, void *stream) {
    WmrArgs A{d_wide_tab, k, 0, d_pcw, d_scr, d_n, nullptr, count, limbs, 0, 1, 0, nullptr, d_verdict, nullptr, nullptr};
    void *args[] = {&A};
    return cudaLaunchKernel((const void *)k_mr_setup_wide, dim3((count + 63) / 64), dim3(64), args, 0,
                            (cudaStream_t)stream) == cudaSuccess
               ? 0
               : 6;
}
size_t mr_wide_table_words(u32 k, u32 window, u32 count) { return (size_t)((1u << window) + 3) * (2 * k + 1) * count; }
size_t mr_wide_pcw_words(u32 k, u32 count) { return (size_t)wmr_words(k) * count; }
size_t mr_wide_scr_words(u32 k, u32 count) { return (size_t)wmr_scr_words(k) * count; }

}  // namespace mr
