// mr_kernels.cuh — sm_100a device code of the MR-MOD / MR-RSA hot path (arXiv:1305.3699 §3.1-§3.3).
//
// Included once per channel count by mr_k<K>.cu with MR_K defined.  Each translation unit is its
// own CUDA module, so the __constant__ base tables below are private to that K.
//
// Mapping: thread-per-message.  A CTA of T = 128 threads owns 128 messages; the
// 2K+1 residues of every message live in shared memory in [channel][thread] layout (conflict-free),
// and each phase of the RNS Montgomery multiplication pulls its input vector into registers:
//   phase 1  channel products -> ξ (registers) and t*_B' (smem)
//   BE1      ξ[K] (registers) x |M_i|_{m'_j} (constant bank)  -> ξ'_j (smem), CH outputs per pass
//   BE2      ξ'[K] (registers) x |M'_j|_{m_i} (constant bank) -> r_i  (smem)
// The base-extension contractions (92-97% of the word products) are 96-bit
// multiply-accumulate chains (IMAD.WIDE.U32 with carry-out + IADD3.X), CH independent accumulators
// per pass for ILP, the inner loop over the K inputs fully unrolled and the outer loop over output
// tiles rolled, so the kernel body stays small enough for the instruction cache.
// Every residue reduction uses the pseudo-Mersenne form m = 2^32 - c, c < 2^13.  Residues are kept
// lazily in [0, 2^32) (congruent, not necessarily < m); DESIGN.md §3 shows the value bound
// r < (K+3)N still holds, and the exit conversion canonicalises.
#pragma once
#include <cuda_runtime.h>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include "mr_internal.h"

#ifndef MR_K
#error "define MR_K before including mr_kernels.cuh"
#endif

namespace mr {
namespace {  // everything below is private to this K's translation unit

constexpr int K = MR_K;
constexpr int NCH = 2 * K + 1;                // residues per value: B, B', m_r
constexpr int T = K > 97 ? 64 : 128;          // threads (messages) per CTA of the IMAD-path kernels (k = 129: smem)
constexpr int CH = be_ch(K);                  // base-extension outputs per register tile
constexpr int KF = (K / CH) * CH;             // outputs covered by full tiles
constexpr int KT = K - KF;                    // tail tile
constexpr u32 BEW = be_words(K);              // base-extension image words (smem)
constexpr u32 BEH = be_half_words(K);         // BE1 part; BE2 follows
constexpr int MINB = K <= 33 ? 4 : (K <= 65 ? 3 : 2);   // CTAs per SM the register budget targets
// X < KB N <= 2^(SMAX+1) N; KB = 2K+3 for K <= 65 (sign-folded digits of the tensor path, §4e), else K+3
constexpr int KB = K <= 65 ? 2 * K + 3 : K + 3;
constexpr int SMAX = (KB <= 2) ? 0 : (32 - __builtin_clz((unsigned)(KB - 1))) - 1;
enum : u32 { MR_COMPOSITE_V = 0, MR_PROBABLY_PRIME_V = 1, MR_FACTOR_V = 2 };

constexpr BaseLayout BL = base_layout(K);
constexpr u32 O_C = BL.c, O_C2 = BL.c2, O_A1R = BL.A1r, O_A2R = BL.A2r;
constexpr u32 O_C1 = BL.C1, O_PIN = BL.pin, O_MISC = BL.misc, O_NMP = BL.NMp;
constexpr u32 O_MIS = BL.MiS, O_MU = BL.MU, O_ONE = BL.ONE, O_ML = BL.ML, O_MM = BL.MM, O_MINV = BL.MINV, O_XW = BL.XW;
constexpr u32 O_A2C = BL.A2C;
constexpr u32 BASE_WORDS = BL.const_words;          // __constant__ prefix of the base table
constexpr u32 CXW = cx_words(K);
constexpr u32 SMEM_STATE = NCH * T;           // words of per-CTA residue state
constexpr size_t SMEM_BYTES = 4 * (size_t)(SMEM_STATE + BEW + CXW);   // state | BE image | context

__constant__ u32 g_base[BASE_WORDS];

#define GB(off) g_base[(off)]

// ------------------------------------------------------------------ word arithmetic
#ifndef MR_ABL_NOMMA
#define MR_ABL_NOMMA 0
#endif
#ifndef MR_SQ_SPLIT
#define MR_SQ_SPLIT 1
#endif
#ifndef MR_RED_VARIANT
#define MR_RED_VARIANT 2
#endif
#ifndef MR_EPI_UNROLL
#define MR_EPI_UNROLL 1     // fully unrolled tensor epilogues with constant-bank operands (+6 % over LDS-fed rolled loops)
#endif
#ifndef MR_BP_LATE
#define MR_BP_LATE 0        // A/B hook: B' products after the BE1 MMA issue (overlap the MMA); measured 0.8 % slower
#endif
#ifndef MR_CHAN_FUSE
#define MR_CHAN_FUSE 0      // A/B hook: interleave the B' channel products with the B chunks
#endif
#ifndef MR_PF_L1
#define MR_PF_L1 0          // A/B hook: prefetch the next window-table operand into L1 instead of L2
#endif
#ifndef MR_WAIT_HINT
#define MR_WAIT_HINT 0      // 1: MMA-completion waits with a suspend-time hint (measured 0.4 % slower on C2 / C5)
#endif
#ifndef MR_TAB_PF
#define MR_TAB_PF 1         // Miller-Rabin: prefetch each window digit's table entry into L2 at its first squaring
#endif
#ifndef MR_MR_EPI_UNROLL
#define MR_MR_EPI_UNROLL 0  // 1: Miller-Rabin tensor epilogues unrolled with constant-bank operands (A/B: 5 % slower, spills)
#endif
#ifndef MR_EPI_NOFOLD
#define MR_EPI_NOFOLD 1     // 1: the scaled BE1 epilogue adds V (< 2^48.1) unfolded (one IMAD fewer per output)
#endif
#ifndef MR_FRAC_ALPHA
// 1: the tensor kernels take the BE2 / exit overflow count α' = floor(Σ_j ξ'_j / m'_j) from the top bits of the ξ'_j
// (Kawamura's fractional base extension: the value r being extended is < (2k+3)N, so r / M' < 0.11 and the sum is
// within 2^-13.9 below an integer plus r / M'), instead of through the extra modulus m_r = 2^32, which then needs no
// upkeep at all (no m_r product, no Σ ξ_i |M_i|_{2^32} and Σ ξ'_j |M'_j|_{2^32} IMAD chains).  DESIGN.md §4e, reading R5.
#define MR_FRAC_ALPHA 1
#endif
// α' = floor(Σ_j ξ'_j / m'_j) from s = Σ_j (ξ'_j >> 8): ξ'_j / m'_j exceeds ξ'_j / 2^32 by < c'_j / m'_j <= 2^-20 and the
// shift drops < 2^-24, so s / 2^24 is below the sum by < k (2^-20 + 2^-24) <= 2^-13.9 (k <= 65); adding 2^-10 and
// truncating gives α' exactly while r / M' + 2^-10 < 1
__device__ __forceinline__ u32 frac_alpha(u32 s) { return (s + (1u << 14)) >> 24; }
#ifndef MR_SIG_PF
#define MR_SIG_PF 8         // Miller-Rabin: per-candidate σ_i / c2_j loaded this many channels / outputs ahead
#endif

// 96-bit multiply-accumulate (lo, mid, hi) += x * y; lowers to IMAD.WIDE.U32 with carry-out + IADD3.X
__device__ __forceinline__ void mac96(u32 &lo, u32 &mid, u32 &hi, u32 x, u32 y) {
    asm("mad.lo.cc.u32 %0, %3, %4, %0;\n\t"
        "madc.hi.cc.u32 %1, %3, %4, %1;\n\t"
        "addc.u32 %2, %2, 0;"
        : "+r"(lo), "+r"(mid), "+r"(hi)
        : "r"(x), "r"(y));
}

// p = h·2^32 + l  ->  congruent value in [0, 2^32) modulo m = 2^32 - c  (c < 2^13).
// h·2^32 + l ≡ h·c + l = uh·2^32 + ul (uh <= c) ≡ uh·c + ul = cy·2^32 + vl (cy <= 1) ≡ vl + cy·c, and when
// cy = 1, vl < 2^26 so vl + c does not wrap.  Both products take the previous 64-bit value as their
// addend pair, so each is one IMAD.WIDE with no register moves: u = h c + p has high word uh + h
// (mod 2^32), v = uh c + u has high word cy + uh + h; the differences recover uh and cy.
#if MR_RED_VARIANT == 2
// u = h c (IMAD.WIDE, no addend pair to build) + l with an ALU carry chain; then v = uh c + ul (uh < 2^13:
// one 32-bit IMAD), a wrap adds c (v < 2^26 then)
__device__ __forceinline__ u32 red64p(u64 p, u32 c) {
    const u64 hc = (u64)(u32)(p >> 32) * c;
    u32 ul, uh;
    asm("add.cc.u32 %0, %2, %3;\n\taddc.u32 %1, %4, 0;" : "=r"(ul), "=r"(uh) : "r"((u32)hc), "r"((u32)p), "r"((u32)(hc >> 32)));
    const u32 vl = uh * c + ul;
    return vl < ul ? vl + c : vl;
}
#elif MR_RED_VARIANT == 1
__device__ __forceinline__ u32 red64p(u64 p, u32 c) {
    const u64 u = (u64)(u32)(p >> 32) * c + (u32)p;
    const u32 uh = (u32)(u >> 32), ul = (u32)u;
    const u32 vl = uh * c + ul;
    return vl < ul ? vl + c : vl;
}
#else
__device__ __forceinline__ u32 red64p(u64 p, u32 c) {
    const u32 h = (u32)(p >> 32);
    const u64 u = (u64)h * c + p;
    const u32 uh = (u32)(u >> 32) - h;
    const u64 v = (u64)uh * c + u;
    const u32 cy = (u32)(v >> 32) - (u32)(u >> 32);
    return (u32)v + cy * c;
}
#endif
__device__ __forceinline__ u32 red64(u32 h, u32 l, u32 c) { return red64p(((u64)h << 32) | l, c); }

// hi·2^64 + mid·2^32 + lo -> congruent value in [0, 2^32), hi < 2^7
// hi·2^64 ≡ hi·c·2^32, so V ≡ W·2^32 + lo with W = mid + hi·c (may carry once: wc), then
// W·2^32 ≡ w·c + wc·c·2^32 and one more fold.
__device__ __forceinline__ u32 red96(u32 hi, u32 mid, u32 lo, u32 c, u32 c2) {
    (void)c2;
    const u32 w = mid + hi * c;                          // hi c < 2^20
    const u32 wc = w < mid ? c : 0u;                     // carry out of W, as its weight c at 2^32
    const u64 u = (u64)w * c + lo;                       // < 2^45 + 2^32
    const u32 uh = (u32)(u >> 32) + wc, ul = (u32)u;     // uh < 2^14
    const u32 vl = uh * c + ul;                          // uh c < 2^27: wraps at most once
    return vl < ul ? vl + c : vl;
}

__device__ __forceinline__ u32 mulmod(u32 a, u32 b, u32 c) { return red64p((u64)a * b, c); }

// Word Montgomery reduction (tensor path): T = thi·2^32 + tlo < 2^64 -> R ≡ T·2^-32 (mod m),
// R in [0, 2^32) (lazy).  q = tlo·(-m^-1) makes q·m + T ≡ 0 mod 2^32; U = (q·m + T) / 2^32 < 2^32 + m;
// a carry out of the 64-bit sum means U ≥ 2^32, and U - 2^32 + c ≡ U with no wrap (U - 2^32 < m).
// Three instructions (IMAD, IMAD.WIDE with carry, predicated add) instead of the ~8 of red64p.
__device__ __forceinline__ u32 mont_red(u32 tlo, u32 thi, u32 m, u32 minv) {
    const u32 q = tlo * minv;
    [[maybe_unused]] u32 ulo;
    u32 uhi, cy;
    asm("mad.lo.cc.u32 %0, %3, %4, %5;\n\tmadc.hi.cc.u32 %1, %3, %4, %6;\n\taddc.u32 %2, 0, 0;"
        : "=r"(ulo), "=r"(uhi), "=r"(cy)
        : "r"(q), "r"(m), "r"(tlo), "r"(thi));
    return cy ? uhi - m : uhi;             // - m ≡ + c (mod 2^32)
}

__device__ __forceinline__ u32 canon(u32 x, u32 c) {  // lazy residue -> [0, m)
    const u32 m = 0u - c;
    return x >= m ? x - m : x;
}

__device__ __forceinline__ u32 &S(u32 *st, int ch) { return st[ch * T + threadIdx.x]; }

// Tensor-core tiles keep the B channels of a value inside the tile's A operand (the message's row of
// the core-matrix layout, where the base extension reads them) and B' ∪ {m_r} in [channel][lane] rows.
struct StTile {
    uint8_t *arow;                    // this message's row in the A tile: (m/8)*SBO + (m%8)*16
    u32 *rows;                        // rows[(ch - K) * 128] = channel ch >= K of this message
};
__device__ __forceinline__ u32 &S(const StTile &s, int ch) {
    return ch < K ? *reinterpret_cast<u32 *>(s.arow + (ch >> 2) * 128 + 4 * (ch & 3)) : s.rows[(ch - K) * 128];
}

// ------------------------------------------------------------------ per-modulus constant sources

struct CtxSmem {                      // one modulus per CTA (encrypt / decrypt): context block in smem
    static constexpr bool kMerged = true;   // BE1 image carries |N M^-1 λ_j| (per-context image)
    static constexpr bool kScaled = false;  // B residues stored plainly; q-digits via σ_i
    static constexpr bool kMont = false;    // word-Montgomery reductions in the tensor multiplication (§4g)
    const u32 *cx;
    __device__ u32 sigma(int i) const { return cx[cx_sigma(K) + i]; }
    __device__ u32 c2(int j) const { return cx[cx_c2(K) + j]; }
    __device__ u32 nminv() const { return cx[CX_NMINV_R]; }
    __device__ u32 nlimb(int l) const { return cx[cx_n(K) + l]; }        // l in [0, K]
};

struct CtxThread {                    // one modulus per thread (Miller-Rabin): per-candidate rows
    static constexpr bool kMerged = false;
    static constexpr bool kScaled = false;
    static constexpr bool kMont = false;
    const u32 *pc;
    u32 stride;
    __device__ u32 sigma(int i) const { return pc[(size_t)(pc_sigma(K) + i) * stride]; }
    __device__ u32 c2(int j) const { return pc[(size_t)(pc_c2(K) + j) * stride]; }
    __device__ u32 nminv() const { return pc[(size_t)pc_nminv(K) * stride]; }
    // n limbs from the candidate-major pc rows (coalesced across the warp; the caller's [count][limbs]
    // rows would cost one sector per thread and limb in the exit's conditional subtractions)
    __device__ u32 nlimb(int l) const { return pc[(size_t)(pc_n(K) + l) * stride]; }   // l in [0, K]
};

// Tensor-core modexp contexts: B residues stored ρ-scaled (s_i = x_i ρ_i, ρ_i² = ε_i σ_i),
// so the q-digit step is one product, ε_i ξ_i = s_a s_b mod m_i; the signs are folded into the
// per-context BE1 image (offset column) and the vectors below, the scales into the BE2 image.
struct CtxTc : CtxSmem {
    static constexpr bool kScaled = true;
    static constexpr bool kMont = true;
    __device__ uint2 a1x(int i) const { return reinterpret_cast<const uint2 *>(cx + cx_a1x(K))[i]; }
    __device__ u32 qr_off() const { return cx[cx_scv(K) + 0]; }
    __device__ u32 c1_off() const { return cx[cx_scv(K) + 1]; }
    __device__ u32 rho_nc() const { return cx[cx_scv(K) + 2]; }
    __device__ u32 c1nc() const { return cx[cx_scv(K) + 3]; }
    __device__ uint4 ep1(int j) const { return reinterpret_cast<const uint4 *>(cx + cx_ep1(K))[j]; }
    __device__ uint2 ep2(int i) const { return reinterpret_cast<const uint2 *>(cx + cx_ep2(K))[i]; }
};

// ------------------------------------------------------------------ RNS Montgomery multiplication
//
// st <- st · b · M^-1 (mod N), SURVEY §8(a6) / DESIGN.md §3, values < (K+3)N throughout.
//   6.1/6.2  B:   ξ_i = (a_i b_i mod m_i) σ_i mod m_i,      σ_i = |-N^-1 M_i^-1|_{m_i}
//            B':  t*_j = a*_j b*_j mod m'_j  (ξ-form operands)
//            m_r: t_r = a_r b_r mod 2^32
//   6.3  BE1 (approximate): q̂_j = Σ_i ξ_i |M_i|_{m'_j},  q̂_r = Σ_i ξ_i |M_i|_{2^32}
//   6.4/6.5  ξ'_j = t*_j |M^-1 λ_j^-1| + q̂_j |N M^-1 λ_j|  (= r_j λ_j, the ξ-form of r),
//            r_r = (t_r + q̂_r N) M^-1 mod 2^32
//   6.6  BE2 (exact, Shenoy-Kumaresan through m_r = 2^32): S_i = Σ_j ξ'_j |M'_j|_{m_i},
//        α' = (Σ_j ξ'_j |M'_j|_{2^32} - r_r) M'^-1 mod 2^32,  r_i = S_i - α'|M'|_{m_i}
// b is st itself (square) or the vector at bp[c * bstride] (global window table or a constant
// vector in shared memory).

// Register tile of the base-extension contraction: W outputs as 96-bit accumulators; the K inputs
// are read from shared-memory rows xr .. xr+K-1 of the state (one LDS per W MACs), the constants
// from the tile's shared-memory image via 16-byte broadcast loads.  The loop over the inputs is
// rolled (unrolled by UI) so the whole multiplication stays resident in the instruction cache.
constexpr int UI = (K % 3 == 0) ? 3 : ((K % 5 == 0) ? 5 : ((K % 7 == 0) ? 7 : 4));
template <int W>
__device__ __forceinline__ void be_tile_acc(const u32 *st, int xr, const u32 *tile, u32 (&lo)[W], u32 (&mi)[W],
                                            u32 (&hi)[W]) {
    constexpr int Q = (W + 3) / 4;
    const uint4 *tb = reinterpret_cast<const uint4 *>(tile);
#pragma unroll UI
    for (int i = 0; i < K; i++) {
        const u32 xi = st[(xr + i) * T + threadIdx.x];
#pragma unroll
        for (int q = 0; q < Q; q++) {
            const uint4 v = tb[i * Q + q];
            if (4 * q + 0 < W) mac96(lo[(4 * q + 0) % W], mi[(4 * q + 0) % W], hi[(4 * q + 0) % W], xi, v.x);
            if (4 * q + 1 < W) mac96(lo[(4 * q + 1) % W], mi[(4 * q + 1) % W], hi[(4 * q + 1) % W], xi, v.y);
            if (4 * q + 2 < W) mac96(lo[(4 * q + 2) % W], mi[(4 * q + 2) % W], hi[(4 * q + 2) % W], xi, v.z);
            if (4 * q + 3 < W) mac96(lo[(4 * q + 3) % W], mi[(4 * q + 3) % W], hi[(4 * q + 3) % W], xi, v.w);
        }
    }
}

// BE1 tile: for j in [j0, j0+W) produce ξ'_j (6.3-6.5) into row K+j and accumulate the m_r column of
// BE2, sr += ξ'_j |M'_j|_{2^32}.  MERGED (one modulus per CTA): the tile image holds
// A1'[i][j] = |M_i|_{m'_j}|N M^-1 λ_j|, so ξ'_j = red(t*_j |M^-1 λ_j^-1| + Σ_i ξ_i A1'[i][j]).
// Otherwise (one modulus per thread, Miller-Rabin): q̂_j = red(Σ_i ξ_i |M_i|_{m'_j}) first.
template <int W, bool MERGED, class CS>
__device__ __forceinline__ void be1_tile(int j0, const u32 *tile, u32 *st, const u32 *s_be, const CS &cs, u32 &sr) {
    u32 lo[W], mi[W], hi[W];
#pragma unroll
    for (int jj = 0; jj < W; jj++) {
        if (MERGED) {
            const u64 p = (u64)S(st, K + j0 + jj) * s_be[bev_C1(K) + j0 + jj];
            lo[jj] = (u32)p;
            mi[jj] = (u32)(p >> 32);
        } else {
            lo[jj] = mi[jj] = 0;
        }
        hi[jj] = 0;
    }
    be_tile_acc<W>(st, 0, tile, lo, mi, hi);
#pragma unroll
    for (int jj = 0; jj < W; jj++) {
        const int j = j0 + jj;
        const u32 c = s_be[bev_c(K) + K + j];
        u32 xp;
        if (MERGED) {
            xp = red96(hi[jj], mi[jj], lo[jj], c, 0);
        } else {
            const u32 q = red96(hi[jj], mi[jj], lo[jj], c, 0);
            const u64 p = (u64)S(st, K + j) * s_be[bev_C1(K) + j];
            u32 l2 = (u32)p, m2 = (u32)(p >> 32), h2 = 0;
            mac96(l2, m2, h2, q, cs.c2(j));
            xp = red96(h2, m2, l2, c, 0);
        }
        S(st, K + j) = xp;
        sr += xp * s_be[bev_A2r(K) + j];
    }
}

// BE2 tile: r_i for i in [i0, i0+W) into row i (the inputs ξ' are rows K..2K-1).
template <int W>
__device__ __forceinline__ void be2_tile(int i0, const u32 *tile, u32 alpha, u32 *st, const u32 *s_be) {
    u32 lo[W], mi[W], hi[W];
#pragma unroll
    for (int ii = 0; ii < W; ii++) {
        const u64 p = (u64)alpha * s_be[bev_pin(K) + i0 + ii];
        lo[ii] = (u32)p;
        mi[ii] = (u32)(p >> 32);
        hi[ii] = 0;
    }
    be_tile_acc<W>(st, K, tile, lo, mi, hi);
#pragma unroll
    for (int ii = 0; ii < W; ii++) {
        const int i = i0 + ii;
        S(st, i) = red96(hi[ii], mi[ii], lo[ii], s_be[bev_c(K) + i], s_be[bev_c2(K) + i]);
    }
}

template <class CS>
__device__ __forceinline__ void mont_mul(u32 *st, const u32 *__restrict__ bp, u32 bstride, bool sq, const CS &cs,
                                         const u32 *s_be) {
    constexpr bool MERGED = CS::kMerged;
    // ---- 6.1 / 6.2: channel products; q-digits ξ_i overwrite a_i; m_r column of BE1 on the fly
    u32 qr = 0;
#pragma unroll 3
    for (int i = 0; i < K; i++) {
        const u32 a = S(st, i);
        const u32 b = sq ? a : bp[(size_t)i * bstride];
        const u32 c = s_be[bev_c(K) + i];
        const u32 xi = mulmod(mulmod(a, b, c), cs.sigma(i), c);
        S(st, i) = xi;
        qr += xi * s_be[bev_A1r(K) + i];
    }
#pragma unroll 3
    for (int j = 0; j < K; j++) {
        const u32 a = S(st, K + j);
        const u32 b = sq ? a : bp[(size_t)(K + j) * bstride];
        S(st, K + j) = mulmod(a, b, s_be[bev_c(K) + K + j]);
    }
    const u32 ar = S(st, 2 * K);
    const u32 tr = ar * (sq ? ar : bp[(size_t)(2 * K) * bstride]);
    const u32 rr = tr * GB(O_MISC + 0) + qr * cs.nminv();       // 6.4 on m_r
    // ---- 6.3-6.5 BE1 [1 x K]·[K x K] contraction, CH outputs per tile, ξ' epilogue
    u32 sr = 0;
#pragma unroll 1
    for (int t = 0; t < KF / CH; t++) be1_tile<CH, MERGED>(t * CH, s_be + t * K * pad4(CH), st, s_be, cs, sr);
    if (KT) be1_tile<KT ? KT : 1, MERGED>(KF, s_be + (KF / CH) * K * pad4(CH), st, s_be, cs, sr);
    // ---- 6.6 BE2 [1 x K]·[K x K] contraction, exact through the extra modulus
    const u32 alpha = (sr - rr) * GB(O_MISC + 1);
    S(st, 2 * K) = rr;
#pragma unroll 1
    for (int t = 0; t < KF / CH; t++) be2_tile<CH>(t * CH, s_be + BEH + t * K * pad4(CH), alpha, st, s_be);
    if (KT) be2_tile<KT ? KT : 1>(KF, s_be + BEH + (KF / CH) * K * pad4(CH), alpha, st, s_be);
}

// ------------------------------------------------------------------ positional -> RNS (a2)
// st_c = Σ_l x_l |2^(32 l)|_{m_c} (B' entries of pow_tab carry λ_j: ξ-form), st_r = x_0.
// x is read at x[l * xstride]; limbs are masked to zero when `ok` is false.
template <class STT>
__device__ __forceinline__ void to_rns(STT st, const u32 *__restrict__ x, u32 xstride, u32 nl, bool ok,
                                       const u32 *__restrict__ pow_tab) {
    const u32 mask = ok ? 0xFFFFFFFFu : 0u;
    constexpr int W = 8;
#pragma unroll 1
    for (int c0 = 0; c0 < 2 * K; c0 += W) {
        u32 lo[W], mi[W], hi[W];
#pragma unroll
        for (int jj = 0; jj < W; jj++) lo[jj] = mi[jj] = hi[jj] = 0;
#pragma unroll 1
        for (u32 l = 0; l < nl; l++) {
            const u32 xl = x[(size_t)l * xstride] & mask;
            const u32 *pr = pow_tab + (size_t)l * (2 * K) + c0;
#pragma unroll
            for (int jj = 0; jj < W; jj++)
                if (c0 + jj < 2 * K) mac96(lo[jj], mi[jj], hi[jj], xl, __ldg(pr + jj));
        }
#pragma unroll
        for (int jj = 0; jj < W; jj++)
            if (c0 + jj < 2 * K) S(st, c0 + jj) = red96(hi[jj], mi[jj], lo[jj], GB(O_C + c0 + jj), GB(O_C2 + c0 + jj));
    }
    S(st, 2 * K) = x[0] & mask;
}

// ------------------------------------------------------------------ RNS -> positional, canonical (a7)
// z on B' ∪ {m_r}, z < (K+3)N < M': α' = (Σ ξ'_j |M'_j|_{2^32} - z_r) M'^-1 mod 2^32 (exact, P:42
// "provided an extra modulus"), X = Σ_j ξ'_j M'_j + α'(2^(32(K+1)) - M') mod 2^(32(K+1)) = z, then
// X mod N by conditional subtraction of N·2^s, s = SMAX..0.  Leaves X in st[0..K] (limb l in row l).
template <class STT, class CS>
__device__ __forceinline__ void from_rns(STT st, const CS &cs, const u32 *__restrict__ mpl) {
    u32 x[K];
#pragma unroll
    for (int j = 0; j < K; j++) x[j] = S(st, K + j);
    u32 sr = 0, alpha;
    if constexpr (MR_FRAC_ALPHA && CS::kMont) {   // tensor kernels: no m_r channel (frac_alpha; z / M' < 0.11)
#pragma unroll
        for (int j = 0; j < K; j++) sr += x[j] >> 8;
        alpha = frac_alpha(sr);
    } else {
#pragma unroll
        for (int j = 0; j < K; j++) sr += x[j] * GB(O_A2R + j);
        alpha = (sr - S(st, 2 * K)) * GB(O_MISC + 1);
    }
    u32 clo = 0, cmi = 0;
#pragma unroll 1
    for (int l = 0; l <= K; l++) {
        u32 lo = clo, mi = cmi, hi = 0;
#pragma unroll
        for (int j = 0; j < K; j++) mac96(lo, mi, hi, x[j], __ldg(mpl + j * (K + 1) + l));
        mac96(lo, mi, hi, alpha, GB(O_NMP + l));
        S(st, l) = lo;
        clo = mi;
        cmi = hi;
    }
#pragma unroll 1
    for (int s = SMAX; s >= 0; s--) {
        // X >= N·2^s ?  compared from the most significant limb down (the first difference decides, usually at
        // once), then one subtraction pass; same decisions as a full borrow pass
        int cmp = 0;
#pragma unroll 1
        for (int l = K; l >= 0 && cmp == 0; l--) {
            const u32 nsh = __funnelshift_l(l ? cs.nlimb(l - 1) : 0u, cs.nlimb(l), s), xv = S(st, l);
            cmp = xv > nsh ? 1 : (xv < nsh ? -1 : 0);
        }
        if (cmp < 0) continue;
        u32 br = 0;
#pragma unroll 1
        for (int l = 0; l <= K; l++) {
            const u32 nsh = __funnelshift_l(l ? cs.nlimb(l - 1) : 0u, cs.nlimb(l), s);
            const u64 t = (u64)S(st, l) - nsh - br;
            S(st, l) = (u32)t;
            br = (u32)(t >> 63);
        }
    }
}

// x (nl limbs) < bound (nl limbs)?
__device__ __forceinline__ bool less_than(const u32 *__restrict__ x, const u32 *__restrict__ bound, u32 nl) {
    int res = 0;
#pragma unroll 1
    for (int l = (int)nl - 1; l >= 0 && res == 0; l--) {
        const u32 xv = x[l], bv = bound[l];
        res = xv < bv ? -1 : (xv > bv ? 1 : 0);
    }
    return res < 0;
}

// stage the per-CTA constants: context block, its merged BE1 image (stored right after the block),
// and the per-k BE2 image + vectors
__device__ __forceinline__ void stage_smem(u32 *s_be, u32 *s_cx, const u32 *gcx, const u32 *be_tab) {
    for (u32 w = threadIdx.x; w < CXW; w += T) s_cx[w] = gcx[w];
    const uint4 *be1 = reinterpret_cast<const uint4 *>(gcx + CXW);
    for (u32 w = threadIdx.x; w < BEH / 4; w += T) reinterpret_cast<uint4 *>(s_be)[w] = __ldg(be1 + w);
    for (u32 w = BEH / 4 + threadIdx.x; w < BEW / 4; w += T)
        reinterpret_cast<uint4 *>(s_be)[w] = __ldg(reinterpret_cast<const uint4 *>(be_tab) + w);
    __syncthreads();
}

// ------------------------------------------------------------------ modexp interpreter kernel (a2-a7, a8 ladders)
// The exponentiation program of one message (one thread): entry, window table, ladder, exit
// multiply, canonical exit, store.  MM is the Montgomery multiplication (IMAD tiles or tensor core);
// `valid` = false runs the program on zeros without storing (tail threads of a tensor-core tile
// must still take part in the tile's barriers).
// Ops [o_begin, o_end) of the program (split schedule, §4f): o_begin > 0 resumes from the handoff slot
// (loaded by the caller), o_end < nops stops before the exit and leaves the state in st.
template <class STT, class MM, class CS = CtxSmem>
__device__ __forceinline__ void run_program(const ModexpParams &P, u32 sel, u32 jl, u32 slot, bool valid, STT st,
                                            const u32 *s_cx, MM &mm, u32 o_begin = 0, u32 o_end = 0xFFFFFFFFu) {
    const CS cs{s_cx};
    // constant operands / accumulators (0xF0 + i): plain vectors at cx_r2; the ρ-scaled path (§4e) uses
    // cx_sc: operands right after to_rns twice-scaled (R2, KHI), ONE scaled, the loaded R2 scaled
    const u32 *cvec = s_cx + (CS::kScaled ? cx_sc(K) : cx_r2(K));
    // the scaled (tensor) path reads every multiplicand from global memory (window table, or the constant
    // vectors of the context block in HBM), so its operand loads are explicit ld.global (mulop_ld)
    const u32 *gcvec = (sel ? P.ctx[1] : P.ctx[0]) + cx_sc(K);
    const size_t tstride = P.jobs_total;
    const size_t entry = (size_t)NCH * tstride;
    const u32 *xrow = P.x + (size_t)(valid ? jl : 0) * P.in_limbs;
    const bool ok = valid && less_than(xrow, s_cx + cx_inb(K), P.in_limbs);
    if (valid && sel == 0 && P.status && o_begin == 0) P.status[jl] = ok ? 0 : 5 /* MR_ERR_RANGE */;

    const u64 *prog = sel ? P.prog[1] : P.prog[0];
    const u32 nops_all = sel ? P.nops[1] : P.nops[0];
    const u32 nops = o_end < nops_all ? o_end : nops_all;
#pragma unroll 1
    for (u32 s = o_begin; s < nops; s++) {
        const u64 op = __ldg(prog + s);
        if (s + 1 < nops) {   // next multiplicand from the window table: pull it from HBM into L2 now
            const u64 nx = __ldg(prog + s + 1);
            const u32 nopnd = (u32)(nx >> 8) & 0xFF;
            if (!(nx & OPF_NOMUL) && nopnd < 0xF0) {
                // the warp's 32 consecutive slots of channel c form one 128-byte line: lane l prefetches the
                // lines of channels l, l + 32, ... (3 instructions per lane instead of 2k+1)
                const u32 lane = threadIdx.x & 31;
                const u32 *np = P.table + nopnd * entry + (slot - lane);
#pragma unroll 1
                for (u32 c = lane; c < (u32)NCH; c += 32) {
#if MR_PF_L1
                    asm volatile("prefetch.global.L1 [%0];" ::"l"(np + c * tstride));
#else
                    asm volatile("prefetch.global.L2 [%0];" ::"l"(np + c * tstride));
#endif
                }
            }
        }
        const u32 fl = (u32)op & 0xFF, opnd = (u32)(op >> 8) & 0xFF, ld = (u32)(op >> 16) & 0xFF;
        const u32 ad = (u32)(op >> 24) & 0xFF, sto = (u32)(op >> 32) & 0xFF;
        if (fl & (OPF_TORNS_ALL | OPF_TORNS_LO | OPF_TORNS_HI)) {
            const u32 off = (fl & OPF_TORNS_HI) ? P.half : 0u;
            const u32 nl = (fl & OPF_TORNS_ALL) ? P.in_limbs : P.half;
            to_rns(st, xrow + off, 1, nl, ok, P.pow_tab);
        }
        if (fl & OPF_LOAD) {
            const u32 *src;
            size_t str;
            if (ld >= 0xF0) { src = cvec + (CS::kScaled && ld == OPND_R2 ? 3u : ld - 0xF0) * NCH; str = 1; }
            else { src = P.table + ld * entry + slot; str = tstride; }
#pragma unroll 1
            for (int c = 0; c < NCH; c++) S(st, c) = src[c * str];
        }
        if (!(fl & OPF_NOMUL)) {
            const bool sq = opnd == OPND_SQ;
            const u32 *bp;
            u32 bs;
            if (sq) { bp = s_cx; bs = 0; }
            else if (opnd >= 0xF0) { bp = (CS::kScaled ? gcvec : cvec) + (opnd - 0xF0) * NCH; bs = 1; }
            else { bp = P.table + opnd * entry + slot; bs = (u32)tstride; }
            mm(st, bp, bs, sq, cs);
        }
        if (fl & OPF_ADD) {  // channel-wise modular addition (CRT entry, a3)
            const u32 *src = P.table + ad * entry + slot;
#pragma unroll 1
            for (int c = 0; c < 2 * K; c++) {
                const u32 b = src[c * tstride];
                const u32 s2 = S(st, c) + b;
                S(st, c) = red64(s2 < b ? 1u : 0u, s2, GB(O_C + c));
            }
            S(st, 2 * K) += src[(2 * K) * tstride];
        }
        if (fl & OPF_STORE) {
            u32 *dst = P.table + sto * entry + slot;
#pragma unroll 1
            for (int c = 0; c < NCH; c++) dst[c * tstride] = S(st, c);
        }
    }
    if (nops < nops_all) return;        // first part of a split job: the caller hands the state over
    from_rns(st, cs, P.mpl);
    if (valid) {
        u32 *yrow = P.y + sel * P.out_stride + (size_t)jl * P.out_limbs;
#pragma unroll 1
        for (u32 l = 0; l < P.out_limbs; l++) yrow[l] = ok ? S(st, l) : 0u;
    }
}

struct MulImad {                      // IMAD-pipe Montgomery multiplication (register-tiled contraction)
    const u32 *s_be;
    __device__ __forceinline__ void operator()(u32 *st, const u32 *bp, u32 bs, bool sq, const CtxSmem &cs) {
        mont_mul(st, bp, bs, sq, cs, s_be);
    }
};

__global__ void __launch_bounds__(T, MINB) k_modexp(const ModexpParams P) {
    extern __shared__ __align__(1024) u32 smem[];
    u32 *st = smem;
    u32 *s_be = smem + SMEM_STATE;
    u32 *s_cx = s_be + BEW;
    const u32 sel = blockIdx.x >= P.ctas0 ? 1u : 0u;
    const u32 *gcx = sel ? P.ctx[1] : P.ctx[0];
    stage_smem(s_be, s_cx, gcx, P.be_tab);
    const u32 jl = (blockIdx.x - sel * P.ctas0) * T + threadIdx.x;
    if (jl >= P.count) return;
    MulImad mm{s_be};
    run_program(P, sel, jl, sel * P.ctas0 * T + jl, true, st, s_cx, mm);
}

#if MR_K * 4 <= 256 || MR_K == 65
// ------------------------------------------------------------------ tensor-core Montgomery multiplication
// DESIGN.md §4b.  Both base extensions run on the 5th-generation tensor cores as u8 x u8 -> s32
// contractions (tcgen05.mma.kind::i8): with x_i = Σ_a byte_a(x_i) 2^(8a) and the pre-shifted
// constants C^(a)_ij = 2^(8a) A_ij mod m_j split into bytes b,
//     D[m][(j, b)] = Σ_(i, a) byte_a(x_{m,i}) · byte_b(C^(a)_ij),   Σ_i x_i A_ij ≡ Σ_b 2^(8b) D[m][(j, b)].
// One tile = 128 messages = 128 threads = the 128 TMEM lanes of an M = 128 MMA.  A CTA runs TCT
// independent tiles; each tile keeps its q-digits as the A operand in shared memory (core-matrix
// layout), its accumulator in TCNP TMEM columns, and synchronises with a named barrier and an
// mbarrier signalled by tcgen05.commit.  Elementwise steps and the m_r column stay on the CUDA cores.
constexpr u32 TCKP = tc_kp(K), TCNP = tc_np(K), TCSBO = tc_sbo(K);
// CTA-pair mode (k = 65): a 2-CTA cluster issues M = 256 MMAs (cta_group::2); each CTA
// holds 128 of the B image's NP rows and receives all NP accumulator columns for its own 128 messages
constexpr bool PAIR = tc_pair(K);
constexpr u32 TC_BB = PAIR ? tc_bbytes(K) / 2 : tc_bbytes(K);   // B image bytes resident per CTA
static_assert(!PAIR || TCNP == 256, "pair mode splits N = 256 into two CTA halves of 128 rows");
constexpr int TCNT = tc_nt(K);                                  // outputs per base extension on the tensor core
constexpr int TCNC = K - TCNT;                                  // outputs on the CUDA cores (k = 33: the last one)
static_assert(TCNC <= 1, "at most one CUDA-core output per base extension");
static_assert(TCNC == 0 || (TCNT + 1 == K && TCNT % 4 == 0), "α' word K sits right after the CUDA-core output");
static_assert(TCNT % 4 == 0 || TCNC == 0, "tensor outputs must fill whole 16-column groups when split");
// the Miller-Rabin kernel's split (mr_internal.h tc_nt_mr)
constexpr int TCNT_MR = tc_nt_mr(K), TCNC_MR = K - TCNT_MR;
constexpr u32 TCNP_MR = tc_np_mr(K);
static_assert(TCNC_MR <= 1 && (TCNC_MR == 0 || (TCNT_MR + 1 == K && TCNT_MR % 4 == 0)), "Miller-Rabin output split");
constexpr u32 BEV_ = BEW - bev_c(K);
constexpr u32 TC_ROWS = (K + 1) * 128;                          // B' and m_r rows of a tile (words)
constexpr u32 TC_CVEC = 2 * pad4(K);                            // CUDA-core output columns: A1' col, A2 col
constexpr size_t tc_smem_for(int tiles) {
    return 4 * (size_t)(tiles * TC_ROWS + BEV_ + CXW + TC_CVEC) + (size_t)tiles * tc_abytes(K) +
           2 * (size_t)TC_BB + 128;
}
#ifndef MR_TC_SLOTS
// 1: when the tiles' accumulators exceed the 512 TMEM columns (k = 33 with all 33 outputs on the tensor core: 4 x 144),
// the tiles of a CTA share 512 / NP accumulator slots, each taken from BE1's MMA issue to the end of BE2's epilogue
// (the channel products, a third of a multiplication, need none), so all four tiles still fit
#define MR_TC_SLOTS 1
#endif
constexpr bool tc_fits(int tiles) {
    return tc_smem_for(tiles) <= 232448 && ((u32)tiles * TCNP <= 512 || (MR_TC_SLOTS && !PAIR && tiles <= 4));
}
// tiles per CTA: as many as fit the 227 KB of shared memory and the 512 TMEM columns (at most 4)
#ifndef MR_TCT_MAX
#define MR_TCT_MAX 4        // A/B hook: cap on the tiles per CTA of the modexp tensor kernel
#endif
constexpr int TCT = (MR_TCT_MAX >= 4 && tc_fits(4)) ? 4 : ((MR_TCT_MAX >= 3 && tc_fits(3)) ? 3 : (tc_fits(2) ? 2 : 1));
static_assert(tc_smem_for(TCT) <= 232448, "tensor-core tile does not fit shared memory");
constexpr u32 TC_M = PAIR ? 256u : 128u;
constexpr u32 TC_IDESC = (2u << 4) | ((TCNP >> 3) << 17) | ((TC_M >> 4) << 24);  // s32 = u8 x u8, K-major
constexpr u32 tmem_cols_for(u32 n) { return n <= 32 ? 32 : n <= 64 ? 64 : n <= 128 ? 128 : n <= 256 ? 256 : 512; }
// shared accumulator slots per CTA (0: every tile owns its accumulator)
constexpr u32 TC_NSLOT = (u32)TCT * TCNP <= 512 ? 0u : 512u / TCNP;
constexpr u32 TC_TMEM_COLS = tmem_cols_for(TC_NSLOT ? TC_NSLOT * TCNP : TCT * TCNP);   // power of two >= 32
constexpr u32 BEV = BEV_;                                      // the per-channel vectors of the BE image
constexpr size_t TC_SMEM = tc_smem_for(TCT);

__device__ __forceinline__ u32 smem_u32(const void *p) { return (u32)__cvta_generic_to_shared(p); }
__device__ __forceinline__ u64 globaltimer_ns() {
    u64 t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}

// word index of (input row i, output column j) inside one half of the IMAD-path tile image (be_*)
__device__ __forceinline__ u32 be_img_index(u32 i, u32 j) {
    const u32 t = j / CH;
    if (t < (u32)(KF / CH)) return t * K * pad4(CH) + i * pad4(CH) + (j - t * CH);
    return (KF / CH) * K * pad4(CH) + i * pad4(KT ? KT : 1) + (j - KF);
}

__device__ __forceinline__ u64 umma_desc(u32 saddr) {
    return (u64)((saddr >> 4) & 0x3FFF) | ((u64)(128u >> 4) << 16) | ((u64)(TCSBO >> 4) << 32) | ((u64)1 << 46);
}

struct TcTile {
    uint8_t *a;                       // A operand tile (128 x TCKP bytes)
    const uint8_t *b1, *b2;           // B images: BE1 (this context), BE2 (this k)
    u32 tmem;                         // TMEM address of this tile's accumulator (lane 0, first column)
    u32 mbar;                         // shared address of this tile's mbarrier
    u32 phase;                        // mbarrier phase parity
    int bar;                          // named barrier id (1 + tile)
    bool leader;                      // thread 0 of the tile issues the MMAs
    u32 m;                            // message (= TMEM lane) index inside the tile
    // pair mode: the tile's A operand is complete in both CTAs when rank 0's "ready" mbarrier (count 2)
    // has one arrival from each CTA's tile leader; only rank 0's leader issues
    u32 rbar;                         // cluster-window address of rank 0's ready mbarrier for this tile
    u32 rphase;                       // its phase parity (rank 0 leader)
    bool issuer;                      // leader && (rank 0 || !PAIR)
    // shared accumulator slots (TC_NSLOT / TC_MR_NSLOT != 0): free-slot mask of the CTA, this tile's slot word
    u32 *pool = nullptr;
    u32 *myslot = nullptr;
    u32 tbase = 0;                    // TMEM base of the CTA's allocation
    u32 idesc = TC_IDESC;             // MMA instruction descriptor (N of this kernel's images)
    u32 *relcnt = nullptr;            // warps of the tile done with the slot (MR_TC_RELWARP)
};

// Shared accumulator slots: the tile leader takes a free slot before BE1's MMA issue (the tile barrier inside tc_issue
// then publishes it to the tile), the tile gives it back once every thread's TMEM reads of BE2 are done.  A tile holds
// at most one slot and never waits while holding one, so the pool cannot deadlock.
__device__ __forceinline__ void acc_acquire(TcTile &t, u32 np) {
    if (!t.pool || !t.leader) return;
    u32 sl = 0;
#pragma unroll 1
    for (u32 spin = 0;; spin++) {
        const u32 f = *reinterpret_cast<volatile u32 *>(t.pool);
        if (f) {
            sl = __ffs(f) - 1;
            if (atomicAnd(t.pool, ~(1u << sl)) & (1u << sl)) break;
        } else {
            __nanosleep(32);
        }
        if (spin > (1u << 28)) __trap();
    }
    __threadfence_block();
    *reinterpret_cast<volatile u32 *>(t.myslot) = sl;
    t.tmem = t.tbase + sl * np;
}
__device__ __forceinline__ void acc_bind(TcTile &t, u32 np) {   // after tc_issue's tile barrier
    if (t.pool && !t.leader) t.tmem = t.tbase + *reinterpret_cast<volatile u32 *>(t.myslot) * np;
}
__device__ __forceinline__ void acc_release(TcTile &t, u32 np);

__device__ __forceinline__ void tile_sync(const TcTile &t) { asm volatile("bar.sync %0, 128;" ::"r"(t.bar) : "memory"); }
#ifndef MR_TC_RELWARP
#define MR_TC_RELWARP 0     // 1: each warp counts itself out of the slot, the last one frees it, no tile barrier (A/B: 1 % slower on C2)
#endif
__device__ __forceinline__ void acc_release(TcTile &t, u32 np) {   // after tcgen05.fence::before_thread_sync
    if (!t.pool) return;
    const u32 bit = 1u << (((t.tmem & 0xFFFFu) - (t.tbase & 0xFFFFu)) / np);
    if (MR_TC_RELWARP && t.relcnt) {
        __syncwarp();
        if ((t.m & 31) == 0) {
            __threadfence_block();
            if (atomicAdd(t.relcnt, 1u) == 3u) {   // the tile's fourth warp: every TMEM read of the slot is done
                *reinterpret_cast<volatile u32 *>(t.relcnt) = 0u;
                __threadfence_block();
                atomicOr(t.pool, bit);
            }
        }
        return;
    }
    tile_sync(t);
    if (t.leader) {
        __threadfence_block();
        atomicOr(t.pool, bit);
    }
}

// issue the K-steps of one base extension (tile leader) after the A tile is complete
__device__ __forceinline__ void tc_issue(TcTile &t, const uint8_t *bimg) {
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");     // A tile written by the generic proxy
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    tile_sync(t);
#if MR_ABL_NOMMA
    return;
#endif
    if (PAIR && t.leader)   // this CTA's half of the M = 256 operand is complete
        asm volatile("mbarrier.arrive.release.cluster.shared::cluster.b64 _, [%0];" ::"r"(t.rbar) : "memory");
    if (t.issuer) {
        if (PAIR) {         // wait for the peer CTA's half (bounded: a lost arrival traps)
            u32 done = 0;
#pragma unroll 1
            for (u32 spin = 0; !done; spin++) {
                asm volatile(
                    "{\n\t.reg .pred P1;\n\tmbarrier.try_wait.parity.acquire.cluster.shared::cta.b64 P1, [%1], %2;\n\t"
                    "selp.u32 %0, 1, 0, P1;\n\t}"
                    : "=r"(done)
                    : "r"(t.mbar + 8 * TCT), "r"(t.rphase)   // own ready barrier, shared::cta address
                    : "memory");
                if (spin > (1u << 26)) __trap();
            }
            t.rphase ^= 1u;
        }
        asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
        const u32 sa = smem_u32(t.a), sb = smem_u32(bimg);
#pragma unroll
        for (u32 ks = 0; ks < TCKP / 32; ks++) {
            const u64 da = umma_desc(sa + ks * 256), db = umma_desc(sb + ks * 256);
            if (PAIR)
                asm volatile(
                    "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                    "tcgen05.mma.cta_group::2.kind::i8 [%0], %1, %2, %3, p;\n\t}" ::"r"(t.tmem),
                    "l"(da), "l"(db), "r"(t.idesc), "r"(ks) : "memory");
            else
                asm volatile(
                    "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                    "tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n\t}" ::"r"(t.tmem),
                    "l"(da), "l"(db), "r"(t.idesc), "r"(ks) : "memory");
        }
        if (PAIR)           // completion to the same mbarrier offset in both CTAs
            asm volatile(
                "tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;" ::"r"(
                    t.mbar), "h"((unsigned short)3) : "memory");
        else
            asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(t.mbar)
                         : "memory");
    }
}

// wait for the tile's MMA chain (bounded: a lost completion traps instead of hanging the GPU)
__device__ __forceinline__ void tc_wait(TcTile &t) {
#if MR_ABL_NOMMA
    return;
#endif
    u32 done = 0;
#if MR_WAIT_HINT
    // with a suspend-time hint the thread sleeps in hardware until the phase completes instead of re-issuing the
    // test (the spin loop was ~4 % of the issued instructions); a wait beyond 30 s traps instead of hanging
    u64 t0 = 0;
#pragma unroll 1
    for (u32 spin = 0; !done; spin++) {
        asm volatile(
            "{\n\t.reg .pred P1;\n\tmbarrier.try_wait.parity.shared::cta.b64 P1, [%1], %2, %3;\n\t"
            "selp.u32 %0, 1, 0, P1;\n\t}"
            : "=r"(done)
            : "r"(t.mbar), "r"(t.phase), "r"(1000000u)
            : "memory");
        if (!done && (spin & 255) == 255) {
            const u64 tt = globaltimer_ns();
            if (!t0) t0 = tt;
            else if (tt - t0 > 30000000000ull) __trap();
        }
    }
#else
#pragma unroll 1
    for (u32 spin = 0; !done; spin++) {
        asm volatile(
            "{\n\t.reg .pred P1;\n\tmbarrier.try_wait.parity.shared::cta.b64 P1, [%1], %2;\n\t"
            "selp.u32 %0, 1, 0, P1;\n\t}"
            : "=r"(done)
            : "r"(t.mbar), "r"(t.phase)
            : "memory");
        if (spin > (1u << 26)) __trap();
    }
#endif
    t.phase ^= 1u;
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
}

__device__ __forceinline__ void tmem_ld16_nowait(u32 taddr, u32 (&v)[16]) {
    // no memory clobber: volatile keeps it after tc_wait, tmem_wait_ld_regs orders the uses of v
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
                 : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]),
                   "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15])
                 : "r"(taddr));
}
// 32 consecutive accumulator columns in one load (two 16-column groups), no memory clobber (see above)
__device__ __forceinline__ void tmem_ld32_nowait(u32 taddr, u32 (&v)[2][16]) {
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
                 "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
                 : "=r"(v[0][0]), "=r"(v[0][1]), "=r"(v[0][2]), "=r"(v[0][3]), "=r"(v[0][4]), "=r"(v[0][5]),
                   "=r"(v[0][6]), "=r"(v[0][7]), "=r"(v[0][8]), "=r"(v[0][9]), "=r"(v[0][10]), "=r"(v[0][11]),
                   "=r"(v[0][12]), "=r"(v[0][13]), "=r"(v[0][14]), "=r"(v[0][15]), "=r"(v[1][0]), "=r"(v[1][1]),
                   "=r"(v[1][2]), "=r"(v[1][3]), "=r"(v[1][4]), "=r"(v[1][5]), "=r"(v[1][6]), "=r"(v[1][7]),
                   "=r"(v[1][8]), "=r"(v[1][9]), "=r"(v[1][10]), "=r"(v[1][11]), "=r"(v[1][12]), "=r"(v[1][13]),
                   "=r"(v[1][14]), "=r"(v[1][15])
                 : "r"(taddr));
}
#ifndef MR_TMEM_X32
#define MR_TMEM_X32 1
#endif
__device__ __forceinline__ void tmem_ld_pair(u32 taddr, bool two, u32 (&v)[2][16]) {
#if MR_TMEM_X32
    if (two) {
        tmem_ld32_nowait(taddr, v);
        return;
    }
#endif
    tmem_ld16_nowait(taddr, v[0]);
    if (two) tmem_ld16_nowait(taddr + 16, v[1]);
}
__device__ __forceinline__ void tmem_wait_ld() { asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory"); }
// wait for the TMEM loads of vv with the loaded registers as in/out operands instead of a memory clobber: the
// uses of vv stay after the wait, and independent shared-memory loads (epilogue constants, B' state) may be
// scheduled above it
#ifndef MR_TMEM_WAIT_REGS
#define MR_TMEM_WAIT_REGS 1
#endif
__device__ __forceinline__ void tmem_wait_ld_regs(u32 (&v)[2][16]) {
#if MR_TMEM_WAIT_REGS
    asm volatile("tcgen05.wait::ld.sync.aligned;"
                 : "+r"(v[0][0]), "+r"(v[0][1]), "+r"(v[0][2]), "+r"(v[0][3]), "+r"(v[0][4]), "+r"(v[0][5]), "+r"(v[0][6]),
                   "+r"(v[0][7]), "+r"(v[0][8]), "+r"(v[0][9]), "+r"(v[0][10]), "+r"(v[0][11]), "+r"(v[0][12]),
                   "+r"(v[0][13]), "+r"(v[0][14]), "+r"(v[0][15]), "+r"(v[1][0]), "+r"(v[1][1]), "+r"(v[1][2]),
                   "+r"(v[1][3]), "+r"(v[1][4]), "+r"(v[1][5]), "+r"(v[1][6]), "+r"(v[1][7]), "+r"(v[1][8]),
                   "+r"(v[1][9]), "+r"(v[1][10]), "+r"(v[1][11]), "+r"(v[1][12]), "+r"(v[1][13]), "+r"(v[1][14]),
                   "+r"(v[1][15]));
#else
    (void)v;
    tmem_wait_ld();
#endif
}
__device__ __forceinline__ void tmem_ld16(u32 taddr, u32 (&v)[16]) {
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
                 : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]),
                   "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15])
                 : "r"(taddr)
                 : "memory");
    asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
}

// Byte-column combine of a tensor-core output: V = Σ_b 2^(8b) d_b = hi·2^32 + lo, formed with shifts and
// one carry chain (ALU pipe, no IMAD).  k <= 64: d_b < 4k·255² < 2^24, so x = d0 + 2^8 d1 and
// y = d2 + 2^8 d3 fit 32 bits and V = x + 2^16 y; k = 65: d_b < 2^24.02, every term is split.
// hi < 2^16.1 (V < 2^48.1, plus the α·pin byte column of BE2, < 2^15).
#ifndef MR_COMBINE_ALU
#define MR_COMBINE_ALU 0
#endif
__device__ __forceinline__ void tc_split(u32 d0, u32 d1, u32 d2, u32 d3, u32 &lo, u32 &hi) {
    if (4ull * K * 255 * 255 < (1ull << 24)) {
#if MR_COMBINE_ALU
        // the same sums as funnel shifts and integer adds (ALU pipe): ptxas otherwise forms x with an IMAD and
        // y·2^16 + x with an IMAD.WIDE, 6 of the FMA-heavy pipe's cycles per output (profiles/r2_c2_pipe_floor.md)
        u32 x, y, yl, yh;
        asm("shf.l.clamp.b32 %0, 0, %1, 8;" : "=r"(x) : "r"(d1));
        asm("shf.l.clamp.b32 %0, 0, %1, 8;" : "=r"(y) : "r"(d3));
        x += d0;
        y += d2;
        asm("shf.l.clamp.b32 %0, 0, %1, 16;" : "=r"(yl) : "r"(y));
        asm("shf.r.clamp.b32 %0, %1, 0, 16;" : "=r"(yh) : "r"(y));
        asm("add.cc.u32 %0, %2, %3;\n\taddc.u32 %1, %4, 0;" : "=r"(lo), "=r"(hi) : "r"(x), "r"(yl), "r"(yh));
#else
        const u32 x = d0 + (d1 << 8), y = d2 + (d3 << 8);
        asm("add.cc.u32 %0, %2, %3;\n\taddc.u32 %1, %4, 0;" : "=r"(lo), "=r"(hi) : "r"(x), "r"(y << 16), "r"(y >> 16));
#endif
    } else {
        asm("add.cc.u32 %0, %2, %3;\n\taddc.u32 %1, %4, 0;\n\t"
            "add.cc.u32 %0, %0, %5;\n\taddc.u32 %1, %1, %6;\n\t"
            "add.cc.u32 %0, %0, %7;\n\taddc.u32 %1, %1, %8;"
            : "=r"(lo), "=r"(hi)
            : "r"(d0), "r"(d1 << 8), "r"(d1 >> 24), "r"(d2 << 16), "r"(d2 >> 16), "r"(d3 << 24), "r"(d3 >> 8));
    }
}
// hi·2^32 + lo ≡ lo + hi·c (mod 2^32 - c) = cw·2^32 + w with cw <= 1 (hi c < 2^29.1): one 32-bit IMAD
__device__ __forceinline__ void fold_hi(u32 lo, u32 hi, u32 c, u32 &w, u32 &cw) {
    asm("mad.lo.cc.u32 %0, %2, %3, %4;\n\taddc.u32 %1, 0, 0;" : "=r"(w), "=r"(cw) : "r"(hi), "r"(c), "r"(lo));
}
// ... and to a word: cw·2^32 + w ≡ w + cw·c, no wrap (cw = 1 leaves w < 2^29.1)
__device__ __forceinline__ u32 fold_word(u32 lo, u32 hi, u32 c) {
    u32 w, cw;
    fold_hi(lo, hi, c, w, cw);
    return cw ? w + c : w;
}

// multiplicand load: global-only on the scaled modexp path (no aliasing with the A-tile stores, so the
// compiler may issue the loads early), generic otherwise (Miller-Rabin passes shared-memory constants)
template <class CS>
__device__ __forceinline__ u32 mulop_ld(const u32 *p) {
    // Miller-Rabin (per-candidate exponent, so per-thread window entries): each candidate's entry is
    // contiguous and read through L1, one 32-byte sector serving 8 consecutive channel loads
    if constexpr (!CS::kMerged && CS::kMont) return __ldca(p);
    else if constexpr (CS::kScaled || CS::kMont) return __ldcg(p);
    else return *p;
}

// NT_ = outputs of each base extension on the tensor core (the rest, at most one, on the CUDA cores); the member
// constants below shadow the modexp kernel's namespace-level ones inside the body
template <int NT_>
struct MulTcT {
    static constexpr int TCNT = NT_;
    static constexpr int TCNC = K - NT_;
    static constexpr u32 TCNP = tc_np_of(NT_);
    const u32 *s_be;
    const u32 *s_a1c;                 // CUDA-core output column of BE1: A1'[i][TCNT] (this context)
    const u32 *s_a2c;                 // CUDA-core output column of BE2: A2[j][TCNT]
    TcTile t;
    // 6.1/6.2 channel products: ξ_i overwrite a_i in place in the A tile (4 channels per 16-byte chunk),
    // t*_j (B') -> rows, m_r column of BE1 (qr), CUDA-core BE1 output accumulated on the fly; returns the
    // m_r product.  SQ: the multiplicand is the state itself (no operand loads, no pointer walk).
    template <bool SQ, class CS>
    __device__ __forceinline__ u32 chan(const StTile &st, const u32 *bp, u32 bs, const CS &cs, u32 &qr, u32 &c1lo,
                                        u32 &c1mi, u32 &c1hi, bool sq = SQ) {
        uint8_t *arow = st.arow;
        const u32 *bq = bp;                          // multiplicand channel pointer, advanced by bs
        // per-thread σ_i (Miller-Rabin: candidate-major rows in L1 / L2) loaded MR_SIG_PF channels ahead, so their
        // latency runs under the products of the channels before (the loop is unrolled: the ring is registers)
        constexpr int PF = (!CS::kMerged && CS::kMont) ? MR_SIG_PF : 0;
        u32 sring[PF > 0 ? PF : 1];
#pragma unroll
        for (int t = 0; t < PF; t++) sring[t] = t < K ? cs.sigma(t) : 0u;
#pragma unroll
        for (int c = 0; c < (K + 3) / 4; c++) {
            uint4 *chunk = reinterpret_cast<uint4 *>(arow + c * 128);
            const uint4 av = *chunk;
            const u32 aw[4] = {av.x, av.y, av.z, av.w};
            u32 w[4];
#pragma unroll
            for (int q = 0; q < 4; q++) {
                const int i = 4 * c + q;
                w[q] = (CS::kScaled && i == K) ? 0x100u : 0u;   // scaled: the BE1 offset column holds 1
                if (i < K) {
                    const u32 a = aw[q];
                    u32 b = a;
                    if (!SQ) {
                        b = sq ? a : mulop_ld<CS>(bq);
                        bq += bs;
                    }
                    const u32 cc = GB(O_C + i);       // unrolled: constant-bank operands
                    u32 xi;
                    if constexpr (CS::kScaled) {      // ε_i ξ_i = s_a s_b 2^-32, lazy (signed digit 2 m_i - xi)
                        const u64 pr = (u64)a * b;
                        xi = mont_red((u32)pr, (u32)(pr >> 32), GB(O_MM + i), GB(O_MINV + i));
                        const uint2 ax = cs.a1x(i);
                        if (!MR_FRAC_ALPHA) qr += xi * ax.x;
                        if (TCNC) mac96(c1lo, c1mi, c1hi, xi, ax.y);
                    } else if constexpr (CS::kMont) {   // ξ_i = mont(mont(a b) σ_i 2^64) = a b σ_i
                        const u64 pr = (u64)a * b;
                        const u32 t = mont_red((u32)pr, (u32)(pr >> 32), GB(O_MM + i), GB(O_MINV + i));
                        u32 sg;
                        if constexpr (PF > 0) {
                            sg = sring[i % (PF > 0 ? PF : 1)];
                            if (i + PF < K) sring[i % (PF > 0 ? PF : 1)] = cs.sigma(i + PF);
                        } else {
                            sg = cs.sigma(i);
                        }
                        const u64 ps = (u64)t * sg;
                        xi = mont_red((u32)ps, (u32)(ps >> 32), GB(O_MM + i), GB(O_MINV + i));   // lazy digit < 2^32
                        if (!MR_FRAC_ALPHA) qr += xi * GB(O_A1R + i);
                        if (TCNC) mac96(c1lo, c1mi, c1hi, xi, s_a1c[i]);
                    } else {
                        xi = mulmod(mulmod(a, b, cc), cs.sigma(i), cc);
                        qr += xi * GB(O_A1R + i);
                        if (TCNC) mac96(c1lo, c1mi, c1hi, xi, s_a1c[i]);
                    }
                    w[q] = xi;
                }
            }
            *chunk = make_uint4(w[0], w[1], w[2], w[3]);
#if MR_CHAN_FUSE
            // B' channels of the same index range, interleaved with the B chunk (more independent chains)
#pragma unroll
            for (int q = 0; q < 4; q++) {
                const int j = 4 * c + q;
                if (j < K) {
                    const u32 a = S(st, K + j);
                    u32 b = a;
                    if (!SQ) b = sq ? a : mulop_ld<CS>(bp + (size_t)(K + j) * bs);
                    if constexpr (CS::kMont) {
                        const u64 pr = (u64)a * b;
                        S(st, K + j) = mont_red((u32)pr, (u32)(pr >> 32), GB(O_MM + K + j), GB(O_MINV + K + j));
                    } else {
                        S(st, K + j) = mulmod(a, b, GB(O_C + K + j));
                    }
                }
            }
#endif
        }
#if MR_CHAN_FUSE || MR_BP_LATE
        bq = bp + (size_t)(2 * K) * bs;
#pragma unroll
        for (int j = 0; j < 0; j++) {
#else
#pragma unroll
        for (int j = 0; j < K; j++) {
#endif
            const u32 a = S(st, K + j);
            u32 b = a;
            if (!SQ) {
                b = sq ? a : mulop_ld<CS>(bq);
                bq += bs;
            }
            if constexpr (CS::kMont) {                // t*_j 2^-32 (the epilogue constants carry the 2^32s)
                const u64 pr = (u64)a * b;
                S(st, K + j) = mont_red((u32)pr, (u32)(pr >> 32), GB(O_MM + K + j), GB(O_MINV + K + j));
            } else {
                S(st, K + j) = mulmod(a, b, GB(O_C + K + j));
            }
        }
#if MR_BP_LATE
        return 0;
#else
        if constexpr (MR_FRAC_ALPHA && CS::kMont) return 0u;   // no m_r channel
        const u32 ar = S(st, 2 * K);
        return ar * (SQ || sq ? ar : mulop_ld<CS>(bq));
#endif
    }

    // B' channel products t*_j and the m_r product (returned); with MR_BP_LATE they run after the BE1 MMA
    // issue, overlapping the tensor-core latency
    template <bool SQ, class CS>
    __device__ __forceinline__ u32 chan_bp(const StTile &st, const u32 *bp, u32 bs, bool sq = SQ) {
#pragma unroll
        for (int j = 0; j < K; j++) {
            const u32 a = S(st, K + j);
            u32 b = a;
            if (!SQ) b = sq ? a : mulop_ld<CS>(bp + (size_t)(K + j) * bs);
            if constexpr (CS::kMont) {
                const u64 pr = (u64)a * b;
                S(st, K + j) = mont_red((u32)pr, (u32)(pr >> 32), GB(O_MM + K + j), GB(O_MINV + K + j));
            } else {
                S(st, K + j) = mulmod(a, b, GB(O_C + K + j));
            }
        }
        if constexpr (MR_FRAC_ALPHA && CS::kMont) return 0u;
        const u32 ar = S(st, 2 * K);
        return ar * (SQ || sq ? ar : mulop_ld<CS>(bp + (size_t)(2 * K) * bs));
    }

    template <class CS>
    __device__ __forceinline__ void operator()(const StTile &st, const u32 *bp, u32 bs, bool sq, const CS &cs) {
        constexpr bool MERGED = CS::kMerged;      // false: per-thread modulus (Miller-Rabin), unmerged BE1
        constexpr u32 ONECOL = CS::kScaled ? 0x100u : 0u;   // byte 1 of A word K: the BE1 offset column
        constexpr bool FRAC = MR_FRAC_ALPHA && CS::kMont;   // α' from the top bits of ξ' (no m_r channel)
        const u32 lane_base = (u32)(t.m & ~31u) << 16;
        uint8_t *arow = st.arow;
        // ---- 6.1/6.2: q-digits ξ_i overwrite a_i in place in the A tile (4 channels per 16-byte chunk);
        //      t*_j (B') -> rows; m_r column of BE1; CUDA-core BE1 output accumulated on the fly
        u32 qr = 0, tr;
        u32 c1lo = 0, c1mi = 0, c1hi = 0;
        if constexpr (CS::kScaled) {      // constant offsets of the sign-folded digits
            if (!FRAC) qr = cs.qr_off();
            if (TCNC) c1lo = cs.c1_off();
        }
#if MR_SQ_SPLIT
        if (sq) tr = chan<true>(st, bp, bs, cs, qr, c1lo, c1mi, c1hi);
        else tr = chan<false>(st, bp, bs, cs, qr, c1lo, c1mi, c1hi);
#else
        tr = chan<false>(st, bp, bs, cs, qr, c1lo, c1mi, c1hi, sq);
#endif
#if MR_BP_LATE
        // ---- 6.3-6.5 BE1 on the tensor core (merged image: ξ'_j = t*_j C1_j + Σ_i ξ_i A1'_ij); the B'
        //      channel products and the m_r product run while the MMA does
        tc_issue(t, t.b1);
        tr = sq ? chan_bp<true, CS>(st, bp, bs) : chan_bp<false, CS>(st, bp, bs);
        const u32 rr = FRAC ? 0u : tr * GB(O_MISC + 0) + qr * cs.nminv();
#else
        const u32 rr = FRAC ? 0u : tr * GB(O_MISC + 0) + qr * cs.nminv();
        // ---- 6.3-6.5 BE1 on the tensor core (merged image: ξ'_j = t*_j C1_j + Σ_i ξ_i A1'_ij)
        acc_acquire(t, TCNP);
        tc_issue(t, t.b1);
        acc_bind(t, TCNP);
#endif
        u32 xp_c = 0;
        if (TCNC) {   // the CUDA-core output overlaps the MMA
            const int j = TCNT;
            const u32 cj = s_be[bev_c(K) + K + j];
            u32 c1j;
            if constexpr (CS::kScaled) c1j = cs.c1nc();     // t* carries 2^-32: C1 c'
            else if constexpr (CS::kMont) c1j = cs.c1c[j];
            else c1j = s_be[bev_C1(K) + j];
            const u64 p = (u64)S(st, K + j) * c1j;
            if (MERGED) {
                mac96(c1lo, c1mi, c1hi, (u32)p, 1u);
                u32 hi2 = c1hi;
                asm("add.cc.u32 %0, %0, %2;\n\taddc.u32 %1, %1, 0;" : "+r"(c1mi), "+r"(hi2) : "r"((u32)(p >> 32)));
                xp_c = red96(hi2, c1mi, c1lo, cj, 0);
            } else {
                const u32 q = red96(c1hi, c1mi, c1lo, cj, 0);
                u32 l2 = (u32)p, m2 = (u32)(p >> 32), h2 = 0;
                mac96(l2, m2, h2, q, cs.c2(j));
                xp_c = red96(h2, m2, l2, cj, 0);
            }
        }
        tc_wait(t);
        u32 sr = 0;
        u32 c2lo = 0, c2mi = 0, c2hi = 0;
        constexpr int NG = TCNT / 4 + (TCNT % 4 ? 1 : 0);
        auto epi1 = [&](int g0) {
          // Miller-Rabin: the 8 per-candidate c2_j of these outputs load while the TMEM loads are in flight
          constexpr bool C2PF = !MERGED && CS::kMont && MR_SIG_PF > 0;
          u32 c2v[C2PF ? 8 : 1];
          if constexpr (C2PF) {
#pragma unroll
            for (int o = 0; o < 8; o++) c2v[o] = 4 * g0 + o < TCNT ? cs.c2(4 * g0 + o) : 0u;
          }
          u32 vv[2][16];                              // two TMEM loads in flight, one wait
          tmem_ld_pair(t.tmem + lane_base + 16 * g0, g0 + 1 < NG, vv);
          tmem_wait_ld_regs(vv);
#pragma unroll
          for (int h = 0; h < 2; h++) {
            const int g = g0 + h;
            if (g >= NG) break;
            const u32 (&v)[16] = vv[h];
            u32 w[4];
#pragma unroll
            for (int o = 0; o < 4; o++) {
                const int j = 4 * g + o;
                w[o] = 0;
                if (j < TCNT) {
                    u32 lo, hi, w33 = 0, c33 = 0;
                    tc_split(v[4 * o], v[4 * o + 1], v[4 * o + 2], v[4 * o + 3], lo, hi);
                    u32 xp;
                    if constexpr (CS::kScaled) {   // ξ'_j = mont(t*_j C1_j c'^2 + V'_j): (m', -m'^-1, C1 c'^2, A2r)
#if MR_EPI_UNROLL
                        const uint4 e = make_uint4(GB(O_MM + K + j), GB(O_MINV + K + j), GB(O_XW + j), GB(O_A2R + j));
                        if (!MR_EPI_NOFOLD) fold_hi(lo, hi, GB(O_C + K + j), w33, c33);
#else
                        const uint4 e = cs.ep1(j);
                        if (!MR_EPI_NOFOLD) fold_hi(lo, hi, 0u - e.x, w33, c33);
#endif
                        // NOFOLD: t*_j (C1 c'^2)_j + V_j in one 64-bit multiply-add: every per-k constant (C1 c'^2)_j is below
                        // 0.998 2^32 and V < 2^48.1, so the sum stays below 2^64 (pinned: test_abi_host.py
                        // ::test_scaled_be1_epilogue_sum_fits_64_bits)
                        const u64 p = MR_EPI_NOFOLD ? (u64)S(st, K + j) * e.z + (((u64)hi << 32) | lo)
                                                    : (u64)S(st, K + j) * e.z + (((u64)c33 << 32) | w33);
                        xp = mont_red((u32)p, (u32)(p >> 32), e.x, e.y);
                        S(st, K + j) = xp;
                        sr += FRAC ? xp >> 8 : xp * e.w;
                        if (TCNC) mac96(c2lo, c2mi, c2hi, xp, GB(O_A2C + j));   // unscaled column, × ρ at the end
                        w[o] = xp;
                        continue;
                    }
                    const u32 c = (MR_MR_EPI_UNROLL && CS::kMont) ? GB(O_C + K + j) : s_be[bev_c(K) + K + j];
                    fold_hi(lo, hi, c, w33, c33);                  // q̂_j (merged: + Σ term) as w33 + c33·2^32
                    if constexpr (MERGED) {   // t*_j C1_j + (w33 + c33 2^32) <= (2^32-1)(2^32-6) + 2^33 < 2^64: no carry
                        const u64 p = (u64)S(st, K + j) * s_be[bev_C1(K) + j] + (((u64)c33 << 32) | w33);
                        xp = red64p(p, c);
                    } else {   // ξ'_j = t*_j C1_j + q̂_j |n M^-1 λ_j|  (6.4 with a per-thread modulus)
                        const u32 q = c33 ? w33 + c : w33;
                        u32 c1j;
                        if constexpr (CS::kMont) c1j = cs.c1c[j];   // t* carries 2^-32
                        else c1j = s_be[bev_C1(K) + j];
                        const u64 p = (u64)S(st, K + j) * c1j;
                        u32 l2 = (u32)p, m2 = (u32)(p >> 32), h2 = 0;
                        u32 c2j;
                        if constexpr (C2PF) c2j = c2v[4 * h + o];
                        else c2j = cs.c2(j);
                        mac96(l2, m2, h2, q, c2j);
                        xp = red96(h2, m2, l2, c, 0);
                    }
                    S(st, K + j) = xp;
                    sr += FRAC ? xp >> 8 : xp * ((MR_MR_EPI_UNROLL && CS::kMont) ? GB(O_A2R + j) : s_be[bev_A2r(K) + j]);
                    if (TCNC) mac96(c2lo, c2mi, c2hi, xp, s_a2c[j]);
                    w[o] = xp;
                }
            }
            *reinterpret_cast<uint4 *>(arow + g * 128) = make_uint4(w[0], w[1], w[2], w[3]);   // BE2 operand
          }
        };
        if constexpr ((CS::kScaled || (MR_MR_EPI_UNROLL && CS::kMont)) && MR_EPI_UNROLL) {   // constant-bank operands need the unrolled loop
#pragma unroll
            for (int g0 = 0; g0 < NG; g0 += 2) epi1(g0);
        } else {
#pragma unroll 1
            for (int g0 = 0; g0 < NG; g0 += 2) epi1(g0);
        }
        // α' (6.6, exact through the extra modulus) goes into the A row at word K, the K-byte column where
        // the BE2 image holds the bytes of m_i - |M'|_{m_i}: the MMA adds α'·(m_i - |M'|_{m_i}) itself
        u32 alpha;
        if constexpr (TCNC != 0) {   // CUDA-core output of BE1 completes the BE2 operand and its own BE2 term
            const int j = TCNT;
            S(st, K + j) = xp_c;
            sr += FRAC ? xp_c >> 8 : xp_c * s_be[bev_A2r(K) + j];
            if constexpr (CS::kScaled) mac96(c2lo, c2mi, c2hi, xp_c, GB(O_A2C + j));
            else mac96(c2lo, c2mi, c2hi, xp_c, s_a2c[j]);
            alpha = FRAC ? frac_alpha(sr) : (sr - rr) * GB(O_MISC + 1);
            *reinterpret_cast<uint4 *>(arow + (j / 4) * 128) = make_uint4(xp_c, alpha | ONECOL, 0u, 0u);
        } else {
            alpha = FRAC ? frac_alpha(sr) : (sr - rr) * GB(O_MISC + 1);
            *reinterpret_cast<u32 *>(arow + (K / 4) * 128 + 4 * (K % 4)) = alpha | ONECOL;
        }
        // ---- 6.6 BE2 on the tensor core; r_i back into the A tile
        asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");   // TMEM reads done before reuse
        tc_issue(t, t.b2);
        if (!FRAC) S(st, 2 * K) = rr;
        u32 r_c = 0;
        if (TCNC) {
            const int i = TCNT;
            mac96(c2lo, c2mi, c2hi, alpha, CS::kScaled ? GB(O_PIN + i) : s_be[bev_pin(K) + i]);
            r_c = red96(c2hi, c2mi, c2lo, s_be[bev_c(K) + i], 0);
            if constexpr (CS::kScaled) r_c = mulmod(r_c, cs.rho_nc(), s_be[bev_c(K) + i]);   // stored B residues carry ρ
        }
        tc_wait(t);
        auto epi2 = [&](int g0) {
          u32 vv[2][16];
          tmem_ld_pair(t.tmem + lane_base + 16 * g0, g0 + 1 < NG, vv);
          tmem_wait_ld_regs(vv);
#pragma unroll
          for (int h = 0; h < 2; h++) {
            const int g = g0 + h;
            if (g >= NG) break;
            const u32 (&v)[16] = vv[h];
            u32 w[4];
#pragma unroll
            for (int o = 0; o < 4; o++) {
                const int i = 4 * g + o;
                w[o] = 0;
                if (i < TCNT) {   // V = S_i + α'(m_i - |M'|_{m_i}) < 2^48.1
                    u32 lo, hi;
                    tc_split(v[4 * o], v[4 * o + 1], v[4 * o + 2], v[4 * o + 3], lo, hi);
                    if constexpr (CS::kScaled) {   // s_i = mont(V_i) (the image carries × c_i)
#if MR_EPI_UNROLL
                        const uint2 e = make_uint2(GB(O_MM + i), GB(O_MINV + i));
#else
                        const uint2 e = cs.ep2(i);
#endif
                        w[o] = mont_red(lo, hi, e.x, e.y);
                    } else {
                        w[o] = fold_word(lo, hi, (MR_MR_EPI_UNROLL && CS::kMont) ? GB(O_C + i) : s_be[bev_c(K) + i]);
                    }
                }
            }
            *reinterpret_cast<uint4 *>(arow + g * 128) = make_uint4(w[0], w[1], w[2], w[3]);
          }
        };
        if constexpr ((CS::kScaled || (MR_MR_EPI_UNROLL && CS::kMont)) && MR_EPI_UNROLL) {   // constant-bank operands need the unrolled loop
#pragma unroll
            for (int g0 = 0; g0 < NG; g0 += 2) epi2(g0);
        } else {
#pragma unroll 1
            for (int g0 = 0; g0 < NG; g0 += 2) epi2(g0);
        }
        if (TCNC) *reinterpret_cast<uint4 *>(arow + (TCNT / 4) * 128) = make_uint4(r_c, 0u, 0u, 0u);
        asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
        acc_release(t, TCNP);
    }
};
using MulTc = MulTcT<TCNT>;        // modexp kernel
using MulTcMr = MulTcT<TCNT_MR>;   // Miller-Rabin kernel

__global__ void __launch_bounds__(TCT * 128, 1) k_modexp_tc(const ModexpParams P) {
    extern __shared__ __align__(1024) u32 smem[];
    // layout: [B1 image | B2 image | A tiles | states | BE image | ctx | mbarriers + TMEM slot]
    uint8_t *s_b1 = reinterpret_cast<uint8_t *>(smem);
    uint8_t *s_b2 = s_b1 + TC_BB;
    uint8_t *s_a = s_b2 + TC_BB;
    u32 *st_all = reinterpret_cast<u32 *>(s_a + TCT * tc_abytes(K));
    u32 *s_vec = st_all + TCT * TC_ROWS;             // vectors only: s_be[bev_*(K) + i] = s_vec[...]
    u32 *s_be = s_vec - bev_c(K);
    u32 *s_cx = s_vec + BEV;
    u32 *s_a1c = s_cx + CXW;                         // CUDA-core output columns (k = 33)
    u32 *s_a2c = s_a1c + pad4(K);
    u64 *mbar = reinterpret_cast<u64 *>(s_a2c + pad4(K));      // [TCT] MMA done, pair mode: + [TCT] ready
    u32 *tslot = reinterpret_cast<u32 *>(mbar + (PAIR ? 2 : 1) * TCT);
    u32 rank = 0;                                               // CTA rank in the pair (pair mode)
    if (PAIR) asm("mov.u32 %0, %%cluster_ctarank;" : "=r"(rank));
    const u32 tid = threadIdx.x, tile = tid / 128, m = tid % 128;
    // Unit = CTA (or CTA pair).  Split schedule: units are numbered in START order by a ticket, so a unit
    // that waits for a hand-over (below) only ever waits for a unit that has already started, i.e. is
    // resident or finished: no deadlock whatever part of the grid is resident (concurrent kernels on other
    // streams, MPS SM limits).  Whole-job round robin has no inter-CTA waits and uses blockIdx.
    u32 unit = PAIR ? blockIdx.x / 2 : blockIdx.x;
    if (P.flags) {
        __shared__ u32 s_ticket;
        const u32 njobs_ = PAIR ? P.ctas0 / 2 : P.ctas0;
        if (tid == 0 && rank == 0) s_ticket = atomicAdd(P.flags + (size_t)4 * njobs_, 1u);
        if (PAIR) {
            asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
            u32 ra;
            asm("mapa.shared::cluster.u32 %0, %1, 0;" : "=r"(ra) : "r"(smem_u32(&s_ticket)));
            asm volatile("ld.shared::cluster.u32 %0, [%1];" : "=r"(unit) : "r"(ra) : "memory");
        } else {
            __syncthreads();
            unit = s_ticket;
        }
    }
    const u32 sel = unit >= P.tc_gc ? 1u : 0u;
    const u32 *gcx = sel ? P.ctx[1] : P.ctx[0];
    // stage constants: context block, IMAD-path BE image words, tensor images
    for (u32 w = tid; w < CXW; w += blockDim.x) s_cx[w] = gcx[w];
    for (u32 w = tid; w < BEV; w += blockDim.x) s_vec[w] = __ldg(P.be_tab + bev_c(K) + w);
    // B images (pair mode: this CTA's 128 of the NP rows, a contiguous byte range of the core-matrix layout)
    const uint4 *g_b1 = reinterpret_cast<const uint4 *>(gcx + P.tc_be1_off) + rank * (TC_BB / 16);
    const uint4 *g_b2 = reinterpret_cast<const uint4 *>(gcx + P.tc_be2_off) + rank * (TC_BB / 16);   // ρ-scaled, per context
    for (u32 w = tid; w < TC_BB / 16; w += blockDim.x) {
        reinterpret_cast<uint4 *>(s_b1)[w] = __ldg(g_b1 + w);
        reinterpret_cast<uint4 *>(s_b2)[w] = __ldg(g_b2 + w);
    }
    __shared__ u32 s_pool, s_myslot[TCT], s_relcnt[TCT];   // shared accumulator slots (TC_NSLOT != 0)
    if (tid == 0) s_pool = (1u << TC_NSLOT) - 1u;
    if (tid < (u32)TCT) s_relcnt[tid] = 0u;
    if (tid < (u32)TCT) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(mbar + tid)));
    if (PAIR && tid < (u32)TCT) asm volatile("mbarrier.init.shared::cta.b64 [%0], 2;" ::"r"(smem_u32(mbar + TCT + tid)));
    if (tid < 32) {
        if (PAIR) {
            asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tslot)),
                         "r"(TC_TMEM_COLS));
            asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;");
        } else {
            asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tslot)),
                         "r"(TC_TMEM_COLS));
            asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
        }
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    if (PAIR)   // both CTAs' mbarriers initialised before any remote arrive
        asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    const u32 tmem_base = *tslot;
    u32 rbar = 0;
    if (PAIR) asm("mapa.shared::cluster.u32 %0, %1, 0;" : "=r"(rbar) : "r"(smem_u32(mbar + TCT + tile)));

    // CUDA-core output columns of the scaled path come from the context block (cx_a1x via CtxTc, cx_a2s)
    MulTc mm{s_be, s_a1c, s_cx + cx_a2s(K), TcTile{s_a + tile * tc_abytes(K), s_b1, s_b2, tmem_base + tile * TCNP,
                                                 smem_u32(mbar + tile), 0u, 1 + (int)tile, m == 0, m, rbar, 0u,
                                                 m == 0 && rank == 0, TC_NSLOT ? &s_pool : nullptr,
                                                 s_myslot + tile, tmem_base, TC_IDESC, s_relcnt + tile}};
    // per-message state: B channels in the A tile row, B' and m_r in the tile's rows
    uint8_t *tile_a = s_a + tile * tc_abytes(K);
    const StTile st{tile_a + (m / 8) * TCSBO + (m % 8) * 16, st_all + tile * TC_ROWS + m};
    // Persistent, balanced schedule.  The CTAs form one group per context (so the
    // shared-memory constants of a CTA serve all its tiles); the tile-jobs t of a group (128
    // messages each) go round-robin, t -> CTA t % Gc, slot (t / Gc) % TCT: every CTA gets
    // floor(ctas0/Gc) or one more job, and a final partial round runs one tile per SM instead of
    // leaving a whole wave of tile slots idle.
    // Pair mode: the unit is a CTA pair and a job is 256 messages (128 per CTA); both CTAs walk the same
    // job list, so every M = 256 MMA finds both halves of its operand (host: ctas0 even).
    const u32 Gc = P.tc_gc, cta = unit - sel * Gc;
    const u32 njobs = PAIR ? P.ctas0 / 2 : P.ctas0;
    // Whole jobs round-robin (no flags), or the split (McNaughton wrap-around) schedule of DESIGN.md §4f: the
    // group's njobs x L op-units are laid out linearly and slot s = NS - 1 - (cta * TCT + tile) takes units
    // [s C, (s+1) C), C = max(L, ceil(njobs L / NS)).  A job straddling the boundary of slots s and s+1 runs
    // its EARLY ops at the start of slot s+1 and its LATE ops at the end of slot s (C >= L keeps the two
    // parts apart in time); the state passes through table slot hslot and a release/acquire flag.  The
    // reversed numbering puts slot s+1 in an earlier-started unit (or an earlier tile of the same CTA), and
    // an early part is the first thing its slot runs, so every wait is for work that is already running.
    // One loop, one inlined copy of run_program (the multiplication code is large: instruction cache).
    const bool split = P.flags != nullptr;
    const u32 L = sel ? P.nops[1] : P.nops[0], NS = Gc * TCT;
    const u64 W = (u64)njobs * L;
    const u64 C = (W + NS - 1) / NS > L ? (W + NS - 1) / NS : (u64)L;
    const u64 s0 = (u64)(NS - 1 - (cta * TCT + tile)) * C;
    const u64 s1 = s0 + C < W ? s0 + C : W;
    const size_t hoff = (size_t)P.hslot * NCH * P.jobs_total;
    u32 *flag_base = split ? P.flags + (size_t)sel * njobs * 2 + rank : nullptr;
    u64 u = s0;
    u32 trr = cta + Gc * tile;
#pragma unroll 1
    while (true) {
        u32 t, ob, oe;
        if (split) {
            if (u >= s1) break;
            t = (u32)(u / L);
            const u32 o = (u32)(u % L);
            if (o) { ob = 0; oe = L - o; }                          // early part of a job shared with slot s-1
            else if (u + L <= s1) { ob = 0; oe = L; }               // whole job
            else { ob = L - (u32)(s1 - u); oe = L; }                // late part of a job shared with slot s+1
        } else {
            if (trr >= njobs) break;
            t = trr;
            trr += Gc * TCT;
            ob = 0;
            oe = L;
        }
        const u32 jl = (PAIR ? t * 256 + rank * 128 : t * 128) + m;
        const u32 col = sel * P.ctas0 * 128 + jl;
        u32 *flag = split ? flag_base + (size_t)t * 2 : nullptr;
        if (ob) {   // wait for the early part, then resume from the handed-over state
            if (m == 0) {
                u32 v = 0;
                const u64 t0 = globaltimer_ns();
#pragma unroll 1
                while (true) {
                    asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(flag) : "memory");
                    if (v) break;
                    if (globaltimer_ns() - t0 > 120000000000ull) __trap();   // 120 s: a lost hand-over
                }
            }
            tile_sync(mm.t);
            const u32 *src = P.table + hoff + col;
#pragma unroll 1
            for (int c = 0; c < NCH; c++) S(st, c) = __ldcg(src + (size_t)c * P.jobs_total);
        }
        run_program<StTile, MulTc, CtxTc>(P, sel, jl, col, jl < P.count, st, s_cx, mm, ob, oe);
        if (oe < L) {   // hand the state over to the slot that runs the late part
            u32 *dst = P.table + hoff + col;
#pragma unroll 1
            for (int c = 0; c < NCH; c++) __stcg(dst + (size_t)c * P.jobs_total, S(st, c));
            __threadfence();
            tile_sync(mm.t);
            if (m == 0) asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(flag), "r"(1u) : "memory");
        }
        u += oe - ob;
    }

    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    if (PAIR) {
        asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
        if (tid < 32)
            asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(tmem_base), "r"(TC_TMEM_COLS));
    } else if (tid < 32) {
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem_base), "r"(TC_TMEM_COLS));
    }
}
#endif

// ------------------------------------------------------------------ CRT recombination (a8)
// m = m_q + q · h,  h = (m_p - m_q mod p) · qinv mod p computed as one RNS Montgomery
// multiplication by qinv·R mod p followed by the canonical exit.  The output row doubles as
// positional scratch (it is overwritten by m at the end).
__global__ void __launch_bounds__(T, MINB) k_combine(const CombineParams P) {
    extern __shared__ __align__(1024) u32 smem[];
    u32 *st = smem;
    u32 *s_be = smem + SMEM_STATE;
    u32 *s_cx = s_be + BEW;
    stage_smem(s_be, s_cx, P.ctx_p, P.be_tab);
    const u32 i = blockIdx.x * T + threadIdx.x;
    if (i >= P.count) return;
    const CtxSmem cs{s_cx};
    const u32 H = P.half;
    const u32 *mp = P.mpq + (size_t)i * H;
    const u32 *mq = P.mpq + ((size_t)P.count + i) * H;
    u32 *mrow = P.m + (size_t)i * 2 * H;
    // t = m_q mod p in st rows [0, H]:  m_q < 2^(32H) <= 2^32 p, subtract p·2^s for s = s0..0 where
    // s0 = bits(m_q) - bits(p) (p·2^s > m_q beyond it; for RSA keys s0 <= 1, so one or two passes)
    int bt = 0, bp = 0;
#pragma unroll 1
    for (u32 l = 0; l <= H; l++) S(st, l) = l < H ? mq[l] : 0u;
#pragma unroll 1
    for (int l = (int)H - 1; l >= 0 && !(bt && bp); l--) {
        if (!bt && mq[l]) bt = 32 * l + 32 - __clz(mq[l]);
        if (!bp && cs.nlimb(l)) bp = 32 * l + 32 - __clz(cs.nlimb(l));
    }
    const int s0 = bt > bp ? (bt - bp < 32 ? bt - bp : 32) : 0;
#pragma unroll 1
    for (int s = s0; s >= 0; s--) {
#pragma unroll 1
        for (int pass = 0; pass < 2; pass++) {
            u32 br = 0;
#pragma unroll 1
            for (u32 l = 0; l <= H; l++) {
                u32 nsh;
                if (s == 32) nsh = l ? cs.nlimb(l - 1) : 0u;
                else nsh = __funnelshift_l(l ? cs.nlimb(l - 1) : 0u, cs.nlimb(l), s);
                const u64 t = (u64)S(st, l) - nsh - br;
                if (pass) S(st, l) = (u32)t;
                br = (u32)(t >> 63);
            }
            if (br) break;   // pass 0 found t < p·2^s: skip the subtraction
        }
    }
    // diff = m_p - t mod p -> mrow[0, H)
    u32 br = 0;
#pragma unroll 1
    for (u32 l = 0; l < H; l++) {
        const u64 d = (u64)mp[l] - S(st, l) - br;
        mrow[l] = (u32)d;
        br = (u32)(d >> 63);
    }
    if (br) {
        u32 carry = 0;
#pragma unroll 1
        for (u32 l = 0; l < H; l++) {
            const u64 s2 = (u64)mrow[l] + cs.nlimb(l) + carry;
            mrow[l] = (u32)s2;
            carry = (u32)(s2 >> 32);
        }
    }
    // h = diff · qinv mod p in RNS:  mm(diff, qinv R mod p) ≡ diff qinv (mod p), then canonical
    to_rns(st, mrow, 1, H, true, P.pow_tab);
    mont_mul(st, s_cx + cx_qinvr(K), 1, false, cs, s_be);
    from_rns(st, cs, P.mpl);
    // m = m_q + q · h  (schoolbook by product scanning: column sums in a 96-bit register accumulator, q
    // broadcast through L1, h in shared-memory rows; each output limb is stored once)
    const bool bad = P.status && P.status[i] != 0;
    u32 lo = 0, mi = 0, hi = 0;
#pragma unroll 1
    for (u32 col = 0; col < 2 * H; col++) {
        if (col < H) mac96(lo, mi, hi, mq[col], 1u);
        const u32 r0 = col >= H ? col - H + 1 : 0u, r1 = col < H ? col : H - 1;
#pragma unroll 4
        for (u32 r = r0; r <= r1; r++) mac96(lo, mi, hi, __ldg(P.q + r), S(st, col - r));
        mrow[col] = bad ? 0u : lo;
        lo = mi;
        mi = hi;
        hi = 0;
    }
}

// ------------------------------------------------------------------ Miller-Rabin (a9)
// Per candidate n (one thread), §3.2 "primality testing in the Montgomery domain ... a
// Miller-Rabin test with a user-parameterized number of iterations", HAC Alg. 4.24.

// word inverse modulo the prime m = 2^32 - c by Fermat: x^(m-2)  (per-channel inversion)
__device__ __forceinline__ u32 inv_word(u32 x, u32 c) {
    const u32 e = 0u - c - 2u;
    u32 r = 1, b = x;
#pragma unroll 1
    for (int bit = 0; bit < 32; bit++) {
        if ((e >> bit) & 1u) r = mulmod(r, b, c);
        b = mulmod(b, b, c);
    }
    return canon(r, c);
}

// smem-row positional helpers for the setup kernel (row l of a value at v[l * T + tid])
__device__ __forceinline__ u32 &R(u32 *v, u32 l) { return v[l * T + threadIdx.x]; }

// remainder of the positional value u (smem rows [0, ulen)) modulo n (global limbs, Ln significant,
// top limb nonzero), Knuth Algorithm D with the divisor normalised on the fly (TAOCP 4.3.1): the
// remainder is left in rows [0, Ln); rows [0, ulen] are clobbered (ulen + 1 rows needed).
__device__ __forceinline__ u32 vnorm(const u32 *n, u32 l, u32 sh) {
    return sh ? (n[l] << sh) | (l ? n[l - 1] >> (32 - sh) : 0u) : n[l];
}
__device__ void rem_knuth(u32 *u, u32 ulen, const u32 *n, u32 Ln) {
    const u32 sh = __clz(n[Ln - 1]);
    if (sh) {                                        // normalise u into ulen + 1 rows
        R(u, ulen) = R(u, ulen - 1) >> (32 - sh);
#pragma unroll 1
        for (int l = (int)ulen - 1; l > 0; l--) R(u, l) = (R(u, l) << sh) | (R(u, l - 1) >> (32 - sh));
        R(u, 0) <<= sh;
    } else {
        R(u, ulen) = 0;
    }
    if (ulen < Ln) return;
    const u32 vt = vnorm(n, Ln - 1, sh), vs = Ln > 1 ? vnorm(n, Ln - 2, sh) : 0u;
#pragma unroll 1
    for (int j = (int)(ulen - Ln); j >= 0; j--) {
        const u64 num = ((u64)R(u, j + Ln) << 32) | R(u, j + Ln - 1);
        u64 qh = num / vt, rh = num - qh * vt;
        while (qh >> 32 || (Ln > 1 && qh * vs > ((rh << 32) | R(u, j + Ln - 2)))) {
            qh--;
            rh += vt;
            if (rh >> 32) break;
        }
        u64 carry = 0;
        long long br = 0;
#pragma unroll 1
        for (u32 i = 0; i < Ln; i++) {
            const u64 pr = qh * vnorm(n, i, sh) + carry;
            carry = pr >> 32;
            const long long t = (long long)R(u, i + j) - (long long)(u32)pr + br;
            R(u, i + j) = (u32)t;
            br = t >> 32;
        }
        const long long t = (long long)R(u, j + Ln) - (long long)carry + br;
        R(u, j + Ln) = (u32)t;
        if (t < 0) {                                 // add back (probability ~2/2^32)
            u64 c = 0;
#pragma unroll 1
            for (u32 i = 0; i < Ln; i++) {
                const u64 s2 = (u64)R(u, i + j) + vnorm(n, i, sh) + c;
                R(u, i + j) = (u32)s2;
                c = s2 >> 32;
            }
            R(u, j + Ln) += (u32)c;
        }
    }
    if (sh) {                                        // unnormalise the remainder
#pragma unroll 1
        for (u32 l = 0; l < Ln; l++) R(u, l) = (R(u, l) >> sh) | (l + 1 < Ln ? R(u, l + 1) << (32 - sh) : 0u);
    }
}

// setup: residues of n, FACTOR check, σ_i, |n M^-1 λ_j|, n M^-1 mod 2^32, s, d, R^2 = M^2 mod n
__global__ void __launch_bounds__(T) k_mr_setup(const MrParams P) {
    extern __shared__ __align__(1024) u32 smem[];
    u32 *st = smem;
    const u32 i = blockIdx.x * T + threadIdx.x;
    if (i >= P.count) return;
    const u32 L = P.limbs;
    const u32 *nrow = P.n + (size_t)i * L;
    u32 *pc = P.pc + i;
    const size_t cs = P.count;
#pragma unroll 1
    for (u32 l = 0; l <= (u32)K; l++) pc[(size_t)(pc_n(K) + l) * cs] = l < L ? nrow[l] : 0u;   // column copy of n
    int32_t status = 0;
    u32 live = 1;
    u32 verdict = MR_COMPOSITE_V;
    u32 nz = 0;                                    // input rules: n odd, n >= 5
    for (u32 l = 1; l < L; l++) nz |= nrow[l];
    const bool small = nz == 0;                    // n < 2^32
    if (!(nrow[0] & 1u) || (small && nrow[0] < 5u)) { status = 5; live = 0; }
    if (live) {
        to_rns(st, nrow, 1, L, true, P.pow_tab);
        bool factor = false;
#pragma unroll 1
        for (int c = 0; c < 2 * K; c++) factor |= canon(S(st, c), GB(O_C + c)) == 0u;
        if (factor) {
            live = 0;
            if (small) { status = 3; verdict = MR_PROBABLY_PRIME_V; }   // n is itself a base prime
            else verdict = MR_FACTOR_V;                                 // reading R14
        }
    }
    if (live) {
#pragma unroll 1
        for (int j = 0; j < K; j++) {              // |n M^-1 λ_j| = (n λ_j) μ_j  (ξ-form residue)
            const u32 c = GB(O_C + K + j);
            pc[(size_t)(pc_c2(K) + j) * cs] = canon(mulmod(S(st, K + j), GB(O_MU + j), c), c);
        }
        pc[(size_t)pc_nminv(K) * cs] = S(st, 2 * K) * GB(O_MISC + 0);
#pragma unroll 1
        for (int k = 0; k < K; k++) {              // σ_i = -(n M_i)^-1 mod m_i
            const u32 c = GB(O_C + k);
            const u32 v = inv_word(canon(mulmod(S(st, k), GB(O_MIS + k), c), c), c);
            const u32 sg = v ? (0u - c) - v : 0u;
            pc[(size_t)(pc_sigma(K) + k) * cs] = sg;
            // σ_i 2^64 ≡ σ_i c_i^2 (mod m_i): the word-Montgomery form the tensor rounds kernel streams
            pc[(size_t)(pc_sig64(K) + k) * cs] = canon(mulmod(mulmod(sg, c, c), c, c), c);
        }
        // s, d with n - 1 = 2^s d
        u32 l0 = 0, w0 = nrow[0] & ~1u;
        while (w0 == 0 && l0 + 1 < L) w0 = nrow[++l0];
        const u32 s = 32 * l0 + __ffs(w0) - 1;
        const u32 ls = s / 32, bs = s % 32;
#pragma unroll 1
        for (u32 l = 0; l < (u32)K; l++) {
            const u32 a0 = l + ls < L ? nrow[l + ls] : 0u;
            const u32 a1 = l + ls + 1 < L ? nrow[l + ls + 1] : 0u;
            pc[(size_t)(pc_d(K) + l) * cs] = __funnelshift_r(l + ls == 0 ? (a0 & ~1u) : a0, a1, bs);
        }
        pc[(size_t)pc_s(K) * cs] = s;
        // R^2 = M^2 mod n, positional: rho = M mod n and rho^2 mod n by Knuth D remainders in smem rows
        // (rho parked in the pc R^2 rows, which are scratch until the RNS image is written)
        u32 Ln = L;
        while (Ln > 1 && nrow[Ln - 1] == 0) Ln--;
        u32 *u = st;
        u32 *r2 = pc + (size_t)pc_r2(K) * cs;
#pragma unroll 1
        for (u32 l = 0; l <= (u32)K; l++) R(u, l) = GB(O_ML + l);
        rem_knuth(u, K + 1, nrow, Ln);                      // rows [0, K + 2)
#pragma unroll 1
        for (u32 l = 0; l < Ln; l++) r2[l * cs] = R(u, l);
#pragma unroll 1
        for (u32 l = 0; l < 2 * Ln; l++) R(u, l) = 0;
#pragma unroll 1
        for (u32 a = 0; a < Ln; a++) {                     // rho^2, schoolbook
            const u32 ra = r2[a * cs];
            u64 c = 0;
#pragma unroll 1
            for (u32 b = 0; b < Ln; b++) {
                const u64 t = (u64)ra * r2[b * cs] + R(u, a + b) + c;
                R(u, a + b) = (u32)t;
                c = t >> 32;
            }
            R(u, a + Ln) = (u32)c;
        }
        rem_knuth(u, 2 * Ln, nrow, Ln);                     // rows [0, 2 Ln + 1)
#pragma unroll 1
        for (u32 l = 0; l < L; l++) r2[l * cs] = l < Ln ? R(u, l) : 0u;
        to_rns(st, r2, (u32)cs, L, true, P.pow_tab);
#pragma unroll 1
        for (int c = 0; c < NCH; c++) r2[c * cs] = S(st, c);
    }
    pc[(size_t)pc_live(K) * cs] = live;
    P.verdict[i] = (uint8_t)verdict;
    if (P.witness) P.witness[i] = -1;
    if (P.status) P.status[i] = status;
}

// canonical X in st rows [0, K] vs 1 and n - 1
__device__ __forceinline__ bool x_is_one(u32 *st) {
    u32 nz = S(st, 0) ^ 1u;
#pragma unroll 1
    for (int l = 1; l <= K; l++) nz |= S(st, l);
    return nz == 0;
}
template <class CS>
__device__ __forceinline__ bool x_is_nm1(u32 *st, const CS &cs) {
    u32 diff = S(st, 0) ^ (cs.nlimb(0) - 1u);      // n odd: n - 1 only changes limb 0
#pragma unroll 1
    for (u32 l = 1; l <= (u32)K; l++) diff |= S(st, l) ^ cs.nlimb(l);
    return diff == 0;
}

// one thread per candidate, all rounds; early exit per candidate unless P.forced
__global__ void __launch_bounds__(T) k_mr_rounds(const MrParams P) {
    extern __shared__ __align__(1024) u32 smem[];
    u32 *st = smem;
    u32 *s_be = smem + SMEM_STATE;
    u32 *s_one = s_be + BEW;
    for (u32 w = threadIdx.x; w < (u32)NCH; w += T) s_one[w] = GB(O_ONE + w);
    for (u32 w = threadIdx.x; w < BEW / 4; w += T)
        reinterpret_cast<uint4 *>(s_be)[w] = __ldg(reinterpret_cast<const uint4 *>(P.be_tab) + w);
    __syncthreads();
    const u32 i = blockIdx.x * T + threadIdx.x;
    if (i >= P.count) return;
    const size_t cnt = P.count;
    const u32 *pcol = P.pc + i;
    if (!pcol[(size_t)pc_live(K) * cnt]) return;
    const u32 L = P.limbs;
    const u32 *nrow = P.n + (size_t)i * L;
    const CtxThread cs{pcol, (u32)cnt};
    const u32 w = P.window, E = 1u << w;
    // window table: the candidate's E entries (+ stash) contiguous, pad4(NCH) words apart (per-candidate
    // window digits: a column layout would scatter every warp load over up to 2^w entries)
    const size_t entry = pad4(NCH);
    u32 *tab = P.table + (size_t)i * (E + 1) * entry;   // slot e at tab + e * entry, channel c at + c
    u32 *stash = tab + E * entry;
    const u32 *r2 = pcol + (size_t)pc_r2(K) * cnt;
    const u32 s = pcol[(size_t)pc_s(K) * cnt];
    const u32 *dl = pcol + (size_t)pc_d(K) * cnt;
    u32 verdict = MR_PROBABLY_PRIME_V;
    int witness = -1;
    int32_t status = 0;
    const u32 ndig = (32 * L + w - 1) / w;        // fixed-window schedule over a padded exponent
    // base rule for every round first: 2 <= a <= n - 2, i.e. a >= 2 and d = n - a >= 2 without borrow
#pragma unroll 1
    for (u32 r = 0; r < P.rounds && !status; r++) {
        const u32 *a = P.bases + ((size_t)i * P.rounds + r) * L;
        u32 br = 0, dhi = 0, ahi = 0, d0 = 0;
#pragma unroll 1
        for (u32 l = 0; l < L; l++) {
            const u64 t = (u64)nrow[l] - a[l] - br;
            br = (u32)(t >> 63);
            if (l) { dhi |= (u32)t; ahi |= a[l]; } else d0 = (u32)t;
        }
        const bool a_ge2 = ahi || a[0] >= 2u;
        const bool d_ge2 = !br && (dhi || d0 >= 2u);
        if (!a_ge2 || !d_ge2) status = 5;
    }
    if (status) {
        P.verdict[i] = (uint8_t)MR_COMPOSITE_V;
        if (P.status) P.status[i] = status;
        return;
    }
#pragma unroll 1
    for (u32 r = 0; r < P.rounds; r++) {
        const u32 *a = P.bases + ((size_t)i * P.rounds + r) * L;
        // table: T[0] = 1~ = mm(R^2, 1), T[1] = ã = mm(a, R^2), T[e] = T[e-1] ã
#pragma unroll 1
        for (int c = 0; c < NCH; c++) S(st, c) = r2[(size_t)c * cnt];
        mont_mul(st, s_one, 1, false, cs, s_be);
#pragma unroll 1
        for (int c = 0; c < NCH; c++) tab[c] = S(st, c);
        to_rns(st, a, 1, L, true, P.pow_tab);
        mont_mul(st, r2, (u32)cnt, false, cs, s_be);
#pragma unroll 1
        for (int c = 0; c < NCH; c++) tab[entry + c] = S(st, c);
#pragma unroll 1
        for (u32 e = 2; e < E; e++) {
            mont_mul(st, tab + entry, 1u, false, cs, s_be);
#pragma unroll 1
            for (int c = 0; c < NCH; c++) tab[e * entry + c] = S(st, c);
        }
        // y = a^d: fixed window from the top digit; acc starts at 1~
#pragma unroll 1
        for (int c = 0; c < NCH; c++) S(st, c) = tab[c];
#pragma unroll 1
        for (int dg = (int)ndig - 1; dg >= 0; dg--) {
            const u32 b0 = dg * w;
            const u32 lw = b0 / 32, bw = b0 % 32;
            const u32 lo = lw < (u32)K ? dl[(size_t)lw * cnt] : 0u;
            const u32 hi = lw + 1 < (u32)K ? dl[(size_t)(lw + 1) * cnt] : 0u;
            const u32 digit = __funnelshift_r(lo, hi, bw) & (E - 1);
#pragma unroll 1
            for (u32 q = 0; q < w; q++) mont_mul(st, s_one, 0, true, cs, s_be);
            mont_mul(st, tab + digit * entry, 1u, false, cs, s_be);
        }
        // HAC 4.24 steps 2.3-2.6: y in {1, n-1} passes; else up to s-1 squarings looking for n-1
        bool pass = false, decided = false;
#pragma unroll 1
        for (u32 j = 0; j < s && !decided; j++) {
            if (j) mont_mul(st, s_one, 0, true, cs, s_be);           // y = y^2
#pragma unroll 1
            for (int c = 0; c < NCH; c++) stash[c] = S(st, c);
            mont_mul(st, s_one, 1, false, cs, s_be);                 // leave the Montgomery domain
            from_rns(st, cs, P.mpl);
            const bool one = x_is_one(st), nm1 = x_is_nm1(st, cs);
            if (nm1) { pass = true; decided = true; }
            else if (one) { pass = (j == 0); decided = true; }  // y = 1 first: pass; later: composite
#pragma unroll 1
            for (int c = 0; c < NCH; c++) S(st, c) = stash[c];
        }
        if (!pass) {
            if (verdict == MR_PROBABLY_PRIME_V) { verdict = MR_COMPOSITE_V; witness = (int)r; }
            if (!P.forced) break;
        }
    }
    P.verdict[i] = (uint8_t)verdict;
    if (P.witness) P.witness[i] = (int16_t)witness;
    if (P.status && status) P.status[i] = status;
}

#if MR_K * 4 <= 256
// ------------------------------------------------------------------ Miller-Rabin rounds on the tensor cores
// Same tiles as k_modexp_tc (128 candidates = 128 TMEM lanes, up to TCT tiles per CTA, persistent
// round-robin tile-jobs), with a per-candidate modulus: the BE1 image is the unmerged per-k one and
// 6.4 multiplies by |n M^-1 λ_j| per thread (CtxMr).  Every thread of a tile takes part in every
// Montgomery multiplication of the tile (the MMA is collective); a thread that is already decided,
// past the end of the batch, or not live (setup verdict) computes on its stale state and its results
// are ignored.  Early exit is per tile: a round is skipped when no candidate of the tile is pending.
struct CtxMr {                        // per-candidate constants of one thread
    static constexpr bool kMerged = false;
    static constexpr bool kScaled = false;
    static constexpr bool kMont = true;   // word-Montgomery reductions: σ_i held as σ_i 2^64, C1 as C1 2^32
    // σ_i 2^64 and c2_j = |n M^-1 λ_j|_{m'_j} stream from the candidate-major pc block in L2 (coalesced
    // across the tile: lane m reads column i + m) instead of occupying 33 registers and 17 KB of shared
    // memory per tile: that is what lets four tiles (16 warps) fit an SM within 128 registers per thread
    const u32 *sigcol;                // pc + pc_sig64 rows: σ_i 2^64 at sigcol[i * nstride]
    const u32 *c1c;                   // shared memory: |M^-1 λ_j^-1| 2^32 mod m'_j (per k)
    const u32 *c2col;                 // pc + pc_c2 rows: c2_j at c2col[j * nstride]
    u32 nmv;                          // n M^-1 mod 2^32
    const u32 *ncol;                  // pcol + pc_n rows: n limb l at ncol[l * nstride] (coalesced)
    u32 nstride;
    // through L1 (ld.global.ca): a tile's σ and c2 columns (34 KB) stay in L1 when few tiles share the SM
    // (the early-exit items phase runs one tile per SM and is latency-bound)
    __device__ u32 sigma(int i) const { return __ldca(sigcol + (size_t)i * nstride); }
    __device__ u32 c2(int j) const { return __ldca(c2col + (size_t)j * nstride); }
    __device__ u32 nminv() const { return nmv; }
    __device__ u32 nlimb(int l) const { return ncol[(size_t)l * nstride]; }   // l in [0, K]
};

__device__ __forceinline__ bool tile_any(const TcTile &t, bool v) {
    u32 r;
    asm volatile("{\n\t.reg .pred p, q;\n\tsetp.ne.u32 p, %1, 0;\n\t"
                 "bar.red.or.pred q, %2, 128, p;\n\tselp.u32 %0, 1, 0, q;\n\t}"
                 : "=r"(r) : "r"((u32)v), "r"(t.bar) : "memory");
    return r != 0;
}

__device__ __forceinline__ bool x_is_one_t(const StTile &st) {
    u32 nz = S(st, 0) ^ 1u;
#pragma unroll 1
    for (int l = 1; l <= K; l++) nz |= S(st, l);
    return nz == 0;
}
__device__ __forceinline__ bool x_is_nm1_t(const StTile &st, const CtxMr &cs) {
    u32 diff = S(st, 0) ^ (cs.nlimb(0) - 1u);
#pragma unroll 1
    for (u32 l = 1; l <= (u32)K; l++) diff |= S(st, l) ^ cs.nlimb(l);
    return diff == 0;
}

constexpr size_t tc_mr_smem_for(int tiles) {
    return 4 * (size_t)(tiles * TC_ROWS + BEV + pad4(NCH) + 3 * pad4(K)) +
           (size_t)tiles * tc_abytes(K) + 2 * (size_t)tc_bbytes_mr(K) + 64;
}
constexpr bool tc_mr_fits(int tiles) {
    return tc_mr_smem_for(tiles) <= 232448 && ((u32)tiles * TCNP_MR <= 512 || (MR_TC_SLOTS && !PAIR && tiles <= 4));
}
constexpr int TCM = tc_mr_fits(4) ? 4 : (tc_mr_fits(3) ? 3 : (tc_mr_fits(2) ? 2 : 1));   // MR tiles per CTA
constexpr u32 TC_MR_NSLOT = (u32)TCM * TCNP_MR <= 512 ? 0u : 512u / TCNP_MR;   // shared accumulator slots (0: per tile)
constexpr u32 TC_MR_TMEM = tmem_cols_for(TC_MR_NSLOT ? TC_MR_NSLOT * TCNP_MR : TCM * TCNP_MR);

__global__ void __launch_bounds__(TCM * 128, 1) k_mr_rounds_tc(const MrParams P) {
    extern __shared__ __align__(1024) u32 smem[];
    // layout: [B1 (unmerged, per k) | B2 | A tiles | state rows | vectors | ONE | a1c | a2c | mbar]
    uint8_t *s_b1 = reinterpret_cast<uint8_t *>(smem);
    uint8_t *s_b2 = s_b1 + tc_bbytes_mr(K);
    uint8_t *s_a = s_b2 + tc_bbytes_mr(K);
    u32 *st_all = reinterpret_cast<u32 *>(s_a + TCM * tc_abytes(K));
    u32 *s_vec = st_all + TCM * TC_ROWS;
    u32 *s_be = s_vec - bev_c(K);
    u32 *s_one = s_vec + BEV;
    u32 *s_a1c = s_one + pad4(NCH);
    u32 *s_a2c = s_a1c + pad4(K);
    u32 *s_c1c = s_a2c + pad4(K);                          // |M^-1 λ_j^-1| 2^32 (word-Montgomery t*, §4g)
    u64 *mbar = reinterpret_cast<u64 *>(s_c1c + pad4(K));
    u32 *tslot = reinterpret_cast<u32 *>(mbar + TCM);
    const u32 tid = threadIdx.x, tile = tid / 128, m = tid % 128;
    for (u32 w = tid; w < BEV; w += blockDim.x) s_vec[w] = __ldg(P.be_tab + bev_c(K) + w);
    for (u32 w = tid; w < (u32)NCH; w += blockDim.x) s_one[w] = GB(O_ONE + w);
    __syncthreads();   // s_vec complete
    for (u32 j = tid; j < (u32)K; j += blockDim.x) {
        const u32 c = s_be[bev_c(K) + K + j];
        s_c1c[j] = canon(mulmod(s_be[bev_C1(K) + j], c, c), c);
    }
    if (TCNC_MR)
        for (u32 i = tid; i < (u32)K; i += blockDim.x) {
            s_a1c[i] = __ldg(P.be_tab + be_img_index(i, TCNT_MR));
            s_a2c[i] = __ldg(P.be_tab + BEH + be_img_index(i, TCNT_MR));
        }
    for (u32 w = tid; w < tc_bbytes_mr(K) / 16; w += blockDim.x) {
        reinterpret_cast<uint4 *>(s_b1)[w] = __ldg(reinterpret_cast<const uint4 *>(P.tc_b1) + w);
        reinterpret_cast<uint4 *>(s_b2)[w] = __ldg(reinterpret_cast<const uint4 *>(P.tc_b2) + w);
    }
    __shared__ u32 s_pool, s_myslot[TCM], s_relcnt[TCM];   // shared accumulator slots (TC_MR_NSLOT != 0)
    if (tid == 0) s_pool = (1u << TC_MR_NSLOT) - 1u;
    if (tid < (u32)TCM) s_relcnt[tid] = 0u;
    if (tid < (u32)TCM) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(mbar + tid)));
    if (tid < 32) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tslot)),
                     "r"(TC_MR_TMEM));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    const u32 tmem_base = *tslot;

    MulTcMr mm{s_be, s_a1c, s_a2c, TcTile{s_a + tile * tc_abytes(K), s_b1, s_b2, tmem_base + tile * TCNP_MR,
                                        smem_u32(mbar + tile), 0u, 1 + (int)tile, m == 0, m, 0u, 0u, m == 0,
                                        TC_MR_NSLOT ? &s_pool : nullptr, s_myslot + tile, tmem_base,
                                        (2u << 4) | ((TCNP_MR >> 3) << 17) | ((128u >> 4) << 24), s_relcnt + tile}};
    uint8_t *tile_a = s_a + tile * tc_abytes(K);
    const StTile st{tile_a + (m / 8) * TCSBO + (m % 8) * 16, st_all + tile * TC_ROWS + m};
    const size_t cnt = P.count;
    const u32 L = P.limbs, w = P.window, E = 1u << w, R = P.rounds;
    // window table: each candidate slot's E entries (+ the check stash) contiguous, NCHP words apart,
    // channel stride 1 (the window digit differs per candidate: a column layout would scatter every
    // warp load over up to 32 entries; here a 32-byte sector serves 8 channel loads)
    constexpr u32 NCHP = pad4(NCH);
    const size_t entry = NCHP;
    const u32 ndig = (32 * L + w - 1) / w;
    const u32 items = P.mode == 2 ? *P.nlive * (R - 1) : 0u;
    const u32 jobs = P.mode == 2 ? (items + 127) / 128 : (P.count + 127) / 128, G = gridDim.x;
#pragma unroll 1
    for (u32 job = blockIdx.x + G * tile; job < jobs; job += G * TCM) {
        u32 i, r_first = 0, r_count = P.mode == 1 ? 1u : R;
        bool pending;
        if (P.mode == 2) {                                          // item = (live candidate, round >= 1)
            const u32 q = job * 128 + m, qq = q < items ? q : items - 1;
            i = P.live[qq / (R - 1)];
            r_first = 1 + qq % (R - 1);
            r_count = 1;
            pending = q < items;
        } else {
            const u32 i0 = job * 128 + m;
            i = i0 < P.count ? i0 : P.count - 1;                    // tail lanes shadow the last candidate
            pending = i0 < P.count && P.pc[i + (size_t)pc_live(K) * cnt] != 0;
        }
        const u32 *pcol = P.pc + i;
        const u32 *nrow = P.n + (size_t)i * L;
        // base rule for every round (HAC 4.24 input), as in k_mr_rounds (items were checked in mode 1)
        int32_t status = 0;
#pragma unroll 1
        for (u32 r = 0; r < P.rounds && pending && !status && P.mode != 2; r++) {
            const u32 *a = P.bases + ((size_t)i * P.rounds + r) * L;
            u32 br = 0, dhi = 0, ahi = 0, d0 = 0;
#pragma unroll 1
            for (u32 l = 0; l < L; l++) {
                const u64 tt = (u64)nrow[l] - a[l] - br;
                br = (u32)(tt >> 63);
                if (l) { dhi |= (u32)tt; ahi |= a[l]; } else d0 = (u32)tt;
            }
            if (!(ahi || a[0] >= 2u) || !(!br && (dhi || d0 >= 2u))) status = 5;
        }
        if (pending && status) {
            P.verdict[i] = (uint8_t)MR_COMPOSITE_V;
            if (P.status) P.status[i] = status;
            pending = false;
        }
        CtxMr cs;
        cs.sigcol = pcol + (size_t)pc_sig64(K) * cnt;
        cs.c1c = s_c1c;
        cs.c2col = pcol + (size_t)pc_c2(K) * cnt;
        cs.nmv = pcol[(size_t)pc_nminv(K) * cnt];
        cs.ncol = pcol + (size_t)pc_n(K) * cnt;
        cs.nstride = (u32)cnt;
        const u32 *r2 = pcol + (size_t)pc_r2(K) * cnt;
        const u32 s = pcol[(size_t)pc_s(K) * cnt];
        const u32 *dl = pcol + (size_t)pc_d(K) * cnt;
        u32 *tab = P.table + (P.mode == 2 ? (size_t)(blockIdx.x * TCM + tile) * 128 + m : (size_t)i) * (E + 1) * NCHP;
        u32 *stash = tab + E * entry;
        u32 verdict = MR_PROBABLY_PRIME_V;
        int witness = -1;
        const bool was_live = pending;
#pragma unroll 1
        for (u32 r = r_first; r < r_first + r_count; r++) {
            if (!tile_any(mm.t, pending || (P.forced && was_live))) break;
            const u32 *a = P.bases + ((size_t)i * P.rounds + r) * L;
            // uniform part: T0 = mm(R^2, 1), T1 = mm(a, R^2), T[e] = T[e-1] T1, then the fixed-window ladder
            const u32 nuni = E + ndig * (w + 1);
#pragma unroll 1
            for (u32 u = 0; u < nuni; u++) {
                const u32 *bp;
                u32 bs;
                bool sq = false;
                if (u == 0) {
#pragma unroll 1
                    for (int c = 0; c < NCH; c++) S(st, c) = r2[(size_t)c * cnt];
                    bp = P.one_g; bs = 1;
                } else if (u == 1) {
                    to_rns(st, a, 1, L, true, P.pow_tab);
                    bp = r2; bs = (u32)cnt;
                } else if (u < E) {
                    bp = tab + entry; bs = 1;
                } else {
                    const u32 q = u - E, dg = ndig - 1 - q / (w + 1), sub = q % (w + 1);
                    if (q == 0) {
#pragma unroll 1
                        for (int c = 0; c < NCH; c++) S(st, c) = tab[c];
                    }
                    if (sub < w) {
                        sq = true; bp = s_one; bs = 0;
                        if (sub == 0 && MR_TAB_PF) {   // this digit's table entry (HBM: the tables exceed L2) -> L2,
                            const u32 b0 = dg * w, lw = b0 / 32, bw = b0 % 32;   // under the w squarings before its use
                            const u32 lo = lw < (u32)K ? dl[(size_t)lw * cnt] : 0u;
                            const u32 hi = lw + 1 < (u32)K ? dl[(size_t)(lw + 1) * cnt] : 0u;
                            const u32 *ent = tab + (size_t)(__funnelshift_r(lo, hi, bw) & (E - 1)) * entry;
#pragma unroll
                            for (u32 l = 0; l < (NCHP * 4 + 127) / 128; l++)
                                asm volatile("prefetch.global.L2 [%0];" ::"l"(ent + 32 * l));
                        }
                    } else {
                        const u32 b0 = dg * w, lw = b0 / 32, bw = b0 % 32;
                        const u32 lo = lw < (u32)K ? dl[(size_t)lw * cnt] : 0u;
                        const u32 hi = lw + 1 < (u32)K ? dl[(size_t)(lw + 1) * cnt] : 0u;
                        bp = tab + (size_t)(__funnelshift_r(lo, hi, bw) & (E - 1)) * entry;
                        bs = 1;
                    }
                }
                mm(st, bp, bs, sq, cs);
                if (u < E) {
                    u32 *dst = tab + (size_t)u * entry;
#pragma unroll 1
                    for (int c = 0; c < NCH; c++) dst[c] = S(st, c);
                }
            }
            // checks (HAC 4.24): even steps leave the Montgomery domain and compare, odd steps square
            // lanes without a live candidate (setup verdict, tail lanes) take no part in the checks: their s is not
            // set (a stale s once kept a whole tile squaring forever)
            bool need = pending || (P.forced && was_live), pass = false;
            u32 jj = 0;
#pragma unroll 1
            for (u32 v = 0;; v++) {
                const bool check = (v % 2) == 0;
                if (check) {
#pragma unroll 1
                    for (int c = 0; c < NCH; c++) stash[c] = S(st, c);
                }
                mm(st, P.one_g, check ? 1u : 0u, !check, cs);
                if (check) {
                    from_rns(st, cs, P.mpl);
                    const bool one = x_is_one_t(st), nm1 = x_is_nm1_t(st, cs);
                    if (need) {
                        if (nm1) { pass = true; need = false; }
                        else if (one) { pass = (jj == 0); need = false; }
                        else if (jj + 1 >= s) need = false;
                    }
                    jj++;
#pragma unroll 1
                    for (int c = 0; c < NCH; c++) S(st, c) = stash[c];
                    if (!tile_any(mm.t, need)) break;
                }
            }
            if (pending && !pass) {
                if (verdict == MR_PROBABLY_PRIME_V) { verdict = MR_COMPOSITE_V; witness = (int)r; }
                if (!P.forced) pending = false;
            }
        }
        if (P.mode == 2) {
            if (was_live && verdict != MR_PROBABLY_PRIME_V) atomicMin(P.wit32 + i, (u32)witness);
        } else if (was_live) {
            P.verdict[i] = (uint8_t)verdict;
            if (P.witness) P.witness[i] = (int16_t)witness;
            if (P.mode == 1 && verdict == MR_PROBABLY_PRIME_V && R > 1) {   // survivor of round 0
                P.wit32[i] = 0xFFFFFFFFu;
                P.live[atomicAdd(P.nlive, 1u)] = i;
            }
        }
    }
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    if (tid < 32) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem_base), "r"(TC_MR_TMEM));
}
constexpr size_t TC_MR_SMEM = tc_mr_smem_for(TCM);
static_assert(TC_MR_SMEM <= 232448, "Miller-Rabin tensor tiles do not fit shared memory");

// fold the items' first failing rounds into the verdicts of the round-0 survivors
__global__ void k_mr_final(const MrParams P) {
    const u32 q = blockIdx.x * blockDim.x + threadIdx.x;
    if (q >= *P.nlive) return;
    const u32 i = P.live[q], wr = P.wit32[i];
    if (wr != 0xFFFFFFFFu) {
        P.verdict[i] = (uint8_t)MR_COMPOSITE_V;
        if (P.witness) P.witness[i] = (int16_t)wr;
    }
}
constexpr int MR_TC_TILES = TCM;
#else
constexpr int MR_TC_TILES = 0;
#endif

#include "mr_tcw.cuh"   // tensor-core wide kernel (k = 97, 129)

// ------------------------------------------------------------------ host-side launchers

template <class Prm>
int launch(void (*kern)(Prm), u32 ctas, const Prm &params, void *stream) {
    void *args[] = {const_cast<Prm *>(&params)};
    return cudaLaunchKernel((const void *)kern, dim3(ctas), dim3(T), args, SMEM_BYTES, (cudaStream_t)stream) ==
                   cudaSuccess
               ? 0
               : 6;
}

int upload_base(const u32 *flat, int device) {
    if (cudaSetDevice(device) != cudaSuccess) return 6;
    if (cudaMemcpyToSymbol(g_base, flat, sizeof(u32) * BASE_WORDS) != cudaSuccess) return 6;
    const void *kerns[] = {(const void *)k_modexp, (const void *)k_combine, (const void *)k_mr_setup,
                           (const void *)k_mr_rounds};
    for (const void *k : kerns)
        if (cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)SMEM_BYTES) != cudaSuccess)
            return 6;
#if MR_K * 4 <= 256 || MR_K == 65
    if (cudaFuncSetAttribute((const void *)k_modexp_tc, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)TC_SMEM) !=
        cudaSuccess)
        return 6;
#endif
#if MR_K * 4 <= 256
    if (cudaFuncSetAttribute((const void *)k_mr_rounds_tc, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             (int)TC_MR_SMEM) != cudaSuccess)
        return 6;
#endif
    return 0;
}

int launch_modexp(const ModexpParams &p, u32 ctas, void *stream) { return launch(k_modexp, ctas, p, stream); }

#if MR_K * 4 <= 256 || MR_K == 65
// ctas = persistent CTAs (pair mode: 2 x the CTA pairs; the cluster dimension is set here)
int launch_modexp_tc(const ModexpParams &p, u32 ctas, void *stream) {
    void *args[] = {const_cast<ModexpParams *>(&p)};
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(ctas);
    cfg.blockDim = dim3(TCT * 128);
    cfg.dynamicSmemBytes = TC_SMEM;
    cfg.stream = (cudaStream_t)stream;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = PAIR ? 2 : 1;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    cfg.attrs = attr;
    cfg.numAttrs = PAIR ? 1 : 0;
    return cudaLaunchKernelExC(&cfg, (const void *)k_modexp_tc, args) == cudaSuccess ? 0 : 6;
}
constexpr int TC_TILES = TCT;
#else
constexpr int (*launch_modexp_tc)(const ModexpParams &, u32, void *) = nullptr;
constexpr int TC_TILES = 0;
#endif

#if MR_K == 97 || MR_K == 129
// ctas = persistent CTAs (one per SM); tab = wide table, kimg = per-k images, cxw / be1w = context offsets (words)
int launch_modexp_tcw(const ModexpParams &p, u32 ctas, const u32 *tab, const void *kimg, u32 cxw, u32 be1w, u32 jobs,
                      void *trace, void *stream) {
    return tcw_launch(p, ctas, TcwArgs{tab, reinterpret_cast<const uint8_t *>(kimg), cxw, be1w, jobs,
                                       reinterpret_cast<unsigned long long *>(trace)}, stream);
}
#else
constexpr int (*launch_modexp_tcw)(const ModexpParams &, u32, const u32 *, const void *, u32, u32, u32, void *,
                                   void *) = nullptr;
#endif

int launch_combine(const CombineParams &p, void *stream) { return launch(k_combine, (p.count + T - 1) / T, p, stream); }

int launch_mr(const MrParams &p, void *stream) {
    const u32 ctas = (p.count + T - 1) / T;
    int rc = launch(k_mr_setup, ctas, p, stream);
    if (rc) return rc;
#if MR_K * 4 <= 256
    if (p.tc_b1 && p.tc_gc) {
        auto run = [&](u32 mode) {
            MrParams q = p;
            q.mode = mode;
            void *args[] = {&q};
            return cudaLaunchKernel((const void *)k_mr_rounds_tc, dim3(p.tc_gc), dim3(TCM * 128), args, TC_MR_SMEM,
                                    (cudaStream_t)stream) == cudaSuccess;
        };
        if (p.live && !p.forced && p.rounds > 1) {          // round 0 for all, then compacted items
            if (cudaMemsetAsync(p.nlive, 0, 4, (cudaStream_t)stream) != cudaSuccess || !run(1) || !run(2)) return 6;
            MrParams q = p;
            void *args[] = {&q};
            return cudaLaunchKernel((const void *)k_mr_final, dim3((p.count + 255) / 256), dim3(256), args, 0,
                                    (cudaStream_t)stream) == cudaSuccess
                       ? 0
                       : 6;
        }
        return run(0) ? 0 : 6;
    }
#endif
    return launch(k_mr_rounds, ctas, p, stream);
}

}  // namespace
}  // namespace mr
