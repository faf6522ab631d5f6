// mr_internal.h — layouts shared by the host runtime (mr_host.cpp) and the per-k CUDA
// translation units (mr_k*.cu).  Not part of the public ABI (include/mr_rns.h is).
#pragma once
#include <cstddef>
#include <cstdint>

namespace mr {

typedef uint32_t u32;
typedef uint64_t u64;

// ---------------------------------------------------------------------------------------------
// Per-context constant block (device global memory, copied to shared memory by every CTA).
// Offsets are constexpr functions of k so the host (runtime k) and device (template K) agree.
// B' residues are stored in "ξ-form" x*_j = x_j · λ_j mod m'_j (λ_j = |M'_j^-1|_{m'_j}), so the
// second base extension reads its CRT digits directly (DESIGN.md §4 "ξ-form").
// ---------------------------------------------------------------------------------------------
enum : u32 {
    CX_K = 0,        // k
    CX_LIMBS,        // limbs of N (canonical output width)
    CX_INLIMBS,      // limbs of the input bound (N, or p·q for CRT halves)
    CX_SMAX,         // largest s with N·2^s used by the exit reduction
    CX_NMINV_R,      // N · M^-1 mod 2^32
    CX_HDR = 8       // header words
};
__host__ __device__ constexpr u32 cx_sigma(u32 k) { return CX_HDR; }                 // [k]  |-N^-1 M_i^-1|_{m_i}
__host__ __device__ constexpr u32 cx_c2(u32 k) { return cx_sigma(k) + k; }           // [k]  |N M^-1 λ_j|_{m'_j}
__host__ __device__ constexpr u32 cx_r2(u32 k) { return cx_c2(k) + k; }              // [2k+1] R^2 mod N
__host__ __device__ constexpr u32 cx_one(u32 k) { return cx_r2(k) + 2 * k + 1; }     // [2k+1] 1
__host__ __device__ constexpr u32 cx_khi(u32 k) { return cx_one(k) + 2 * k + 1; }    // [2k+1] 2^(32 Lh) R^2 mod p
__host__ __device__ constexpr u32 cx_qinvr(u32 k) { return cx_khi(k) + 2 * k + 1; }  // [2k+1] qinv R mod p
__host__ __device__ constexpr u32 cx_n(u32 k) { return cx_qinvr(k) + 2 * k + 1; }    // [k+1] N limbs
__host__ __device__ constexpr u32 cx_inb(u32 k) { return cx_n(k) + k + 1; }          // [2k+2] input bound limbs
// Tensor-core path only: B residues are stored ρ-scaled, s_i = x_i ρ_i with ρ_i² = ε_i σ_i 2^32 (ε_i = ±1; the
// B primes are ≡ 3 mod 4 for k <= 65, so one of ±σ_i is a square), which turns the q-digit step
// ξ_i = σ_i a_i b_i into ε_i ξ_i = s_a s_b mod m_i; the signs ε_i and the scales ρ_i live in the
// per-context constants below and in the per-context tensor images.
__host__ __device__ constexpr u32 cx_sc(u32 k) { return cx_inb(k) + 2 * k + 2; }     // [4][2k+1] R2ρ², ONEρ, KHIρ², R2ρ
__host__ __device__ constexpr u32 cx_a1x(u32 k) { return (cx_sc(k) + 4 * (2 * k + 1) + 1) & ~1u; }  // [k][2] (ε_i|M_i|_{2^32}, ε_i A1'[i][TCNT])
__host__ __device__ constexpr u32 cx_a2s(u32 k) { return cx_a1x(k) + 2 * k; }        // [k]  A2[j][TCNT] ρ_TCNT
__host__ __device__ constexpr u32 cx_scv(u32 k) { return cx_a2s(k) + k; }            // [4]  q̂_r offset, BE1-TCNT offset, ρ_TCNT, C1_TCNT R32
// epilogue constants of the word-Montgomery reductions (§4g): BE1 output j: (m'_j, -m'_j^-1, C1_j R32², |M'_j|_{2^32});
// BE2 output i: (m_i, -m_i^-1)
__host__ __device__ constexpr u32 cx_ep1(u32 k) { return (cx_scv(k) + 4 + 3) & ~3u; }   // [k][4]
__host__ __device__ constexpr u32 cx_ep2(u32 k) { return cx_ep1(k) + 4 * k; }          // [k][2]
__host__ __device__ constexpr u32 cx_words(u32 k) { return (cx_ep2(k) + 2 * k + 3) & ~3u; }

// ---------------------------------------------------------------------------------------------
// Per-k base tables (N-independent).  The CUDA TU for k keeps the hot ones in __constant__ memory
// and the to_rns powers in global memory.  Flat layout produced by the host:
// ---------------------------------------------------------------------------------------------
struct BaseLayout {
    u32 k;
    u32 c, c2, A1r, A2r, C1, pin, misc, NMp, MiS, MU, ONE, ML, MM, MINV, XW, A2C;   // device constant bank (prefix)
    u32 const_words;                                              // words uploaded to __constant__
    u32 MpL, A1, A2, words;                                       // host-side / global-memory tables
};
__host__ __device__ constexpr BaseLayout base_layout(u32 k) {
    BaseLayout b{};
    b.k = k;
    b.c = 0;                        // [2k]     c = 2^32 - m (B then B')
    b.c2 = b.c + 2 * k;             // [2k]     c^2
    b.A1r = b.c2 + 2 * k;           // [k]      |M_i|_{2^32}
    b.A2r = b.A1r + k;              // [k]      |M'_j|_{2^32}
    b.C1 = b.A2r + k;               // [k]      |M^-1 λ_j^-1|_{m'_j}
    b.pin = b.C1 + k;               // [k]      m_i - |M'|_{m_i}
    b.misc = b.pin + k;             // [4]      M^-1 mod 2^32, M'^-1 mod 2^32
    b.NMp = b.misc + 4;             // [k+1]    2^(32(k+1)) - M' limbs
    b.MiS = b.NMp + k + 1;          // [k]      |M_i|_{m_i}           (Miller-Rabin setup)
    b.MU = b.MiS + k;               // [k]      |M^-1|_{m'_j}         (Miller-Rabin setup)
    b.ONE = b.MU + k;               // [2k+1]   RNS image of 1 (B' in ξ-form)
    b.ML = b.ONE + 2 * k + 1;       // [k+1]    M positional limbs    (Miller-Rabin setup)
    b.MM = b.ML + k + 1;            // [2k]     m (B then B')         (word Montgomery reduction, §4g)
    b.MINV = b.MM + 2 * k;          // [2k]     -m^-1 mod 2^32
    b.XW = b.MINV + 2 * k;          // [k]      |M^-1 λ_j^-1| 2^64 mod m'_j (tensor-path BE1 epilogue, §4g)
    b.A2C = b.XW + k;               // [k]      |M'_j|_{m_TCNT}: the CUDA-core BE2 output column (tensor path)
    b.const_words = b.A2C + k;
    b.MpL = b.const_words;          // [k][k+1] M'_j positional limbs (global memory, exit conversion)
    b.A1 = b.MpL + k * (k + 1);     // [k][k]   |M_i|_{m'_j}  (row i, column j; source of the BE images)
    b.A2 = b.A1 + k * k;            // [k][k]   |M'_j|_{m_i}  (row j, column i)
    b.words = b.A2 + k * k;
    return b;
}

// ---------------------------------------------------------------------------------------------
// Base-extension constant image staged in shared memory (read with 16-byte broadcast loads).
// Outputs are processed in tiles of be_ch(k) columns; tile t holds, for every input row i, the
// tile's columns padded to a multiple of 4 words.  Image = BE1 tiles (A1[i][j]) then BE2 tiles
// (A2[j][i]).  Full tiles first, then the tail tile (k mod be_ch(k) columns) if any.
// ---------------------------------------------------------------------------------------------
__host__ __device__ constexpr u32 be_ch(u32 k) {
    for (u32 c = 13; c >= 6; c--)
        if (k % c == 0) return c;
    return k <= 13 ? k : 8;
}
__host__ __device__ constexpr u32 pad4(u32 x) { return (x + 3) & ~3u; }
__host__ __device__ constexpr u32 be_nfull(u32 k) { return k / be_ch(k); }
__host__ __device__ constexpr u32 be_tail(u32 k) { return k - be_nfull(k) * be_ch(k); }
__host__ __device__ constexpr u32 be_half_words(u32 k) {
    return be_nfull(k) * k * pad4(be_ch(k)) + (be_tail(k) ? k * pad4(be_tail(k)) : 0);
}
// per-channel vectors after the two matrices (each padded to a multiple of 4 words)
__host__ __device__ constexpr u32 bev_c(u32 k) { return 2 * be_half_words(k); }          // [2k] c = 2^32 - m
__host__ __device__ constexpr u32 bev_c2(u32 k) { return bev_c(k) + pad4(2 * k); }       // [2k] c^2
__host__ __device__ constexpr u32 bev_C1(u32 k) { return bev_c2(k) + pad4(2 * k); }      // [k]  |M^-1 λ_j^-1|_{m'_j}
__host__ __device__ constexpr u32 bev_pin(u32 k) { return bev_C1(k) + pad4(k); }         // [k]  m_i - |M'|_{m_i}
__host__ __device__ constexpr u32 bev_A1r(u32 k) { return bev_pin(k) + pad4(k); }        // [k]  |M_i|_{2^32}
__host__ __device__ constexpr u32 bev_A2r(u32 k) { return bev_A1r(k) + pad4(k); }        // [k]  |M'_j|_{2^32}
__host__ __device__ constexpr u32 be_words(u32 k) { return bev_A2r(k) + pad4(k); }

// ---------------------------------------------------------------------------------------------
// Tensor-core base extension (tcgen05.mma.kind::i8).  Byte-split contraction:
//   Σ_i x_i A_ij ≡ Σ_b 2^(8b) Σ_(i,a) byte_a(x_i) · byte_b(2^(8a) A_ij mod m_j)   (mod m_j)
// A operand: [128 messages x KP bytes] (row m = the message's K words, little-endian);
// B operand: [NP rows (j, b) x KP bytes (i, a)]; both K-major, SWIZZLE_NONE core-matrix layout:
// byte (r, kb) at (r / 8) * SBO + (kb / 16) * 128 + (r % 8) * 16 + kb % 16, SBO = (KP / 16) * 128.
// D = [128 x NP] s32 in TMEM; every D value < 4k·255² (< 2^24 for k <= 64, < 2^24.02 at k = 65).
// ---------------------------------------------------------------------------------------------
__host__ __device__ constexpr u32 tc_kp(u32 k) { return (4 * k + 31) & ~31u; }     // K bytes, multiple of 32
// outputs of each base extension computed on the tensor core; for k = 33 the 33rd output runs on the
// CUDA cores so that N = 128 columns and four 128-message tiles fit the 512 TMEM columns of an SM;
// for k = 65 the 65th, so that N = 256 (the largest MMA N) covers the other 64
// k = 33, modexp kernel: all 33 outputs on the tensor core (N = 144; four tiles share three TMEM accumulator slots,
// mr_kernels.cuh MR_TC_SLOTS) — 32 is the A/B alternative with the 33rd output on the CUDA cores (N = 128, a fixed
// accumulator per tile).  The Miller-Rabin kernel keeps 32 (MR_TC_NT33_MR): with per-candidate constants its 4-tile
// build spills heavily at N = 144 and 3 tiles are 36 % slower (profiles/r2r/ab.log).
#ifndef MR_TC_NT33
#define MR_TC_NT33 33
#endif
#ifndef MR_TC_NT33_MR
#define MR_TC_NT33_MR 32
#endif
__host__ __device__ constexpr u32 tc_nt_for(u32 k, u32 nt33) {
    return (4 * k > 128 && 4 * k <= 136) ? nt33 : ((4 * k > 256 && 4 * k <= 264) ? 64 : k);
}
__host__ __device__ constexpr u32 tc_nt(u32 k) { return tc_nt_for(k, MR_TC_NT33); }         // modexp kernel
__host__ __device__ constexpr u32 tc_nt_mr(u32 k) { return tc_nt_for(k, MR_TC_NT33_MR); }   // Miller-Rabin kernel
__host__ __device__ constexpr u32 tc_np_of(u32 nt) { return (4 * nt + 15) & ~15u; }          // N rows, multiple of 16
__host__ __device__ constexpr u32 tc_np(u32 k) { return tc_np_of(tc_nt(k)); }
__host__ __device__ constexpr u32 tc_np_mr(u32 k) { return tc_np_of(tc_nt_mr(k)); }
// CTA-pair mode: the two B images of k = 65 (2 x 72 KB) do not fit one CTA next to two
// tiles, so a 2-CTA cluster runs M = 256 MMAs (tcgen05 cta_group::2) and each CTA holds half of the
// B rows (N/2 = 128 of the (j, b) columns); each CTA's TMEM still receives all N columns of its rows.
__host__ __device__ constexpr bool tc_pair(u32 k) { return 4 * k > 256; }
__host__ __device__ constexpr bool tc_ok(u32 k) { return 4 * k <= 256 || tc_nt(k) == 64; }
__host__ __device__ constexpr u32 tc_sbo(u32 k) { return (tc_kp(k) / 16) * 128; }
__host__ __device__ constexpr u32 tc_off(u32 k, u32 r, u32 kb) {
    return (r / 8) * tc_sbo(k) + (kb / 16) * 128 + (r % 8) * 16 + kb % 16;
}
__host__ __device__ constexpr u32 tc_bbytes(u32 k) { return tc_np(k) * tc_kp(k); }   // one B image
__host__ __device__ constexpr u32 tc_bbytes_mr(u32 k) { return tc_np_mr(k) * tc_kp(k); }   // ... of the Miller-Rabin kernel
__host__ __device__ constexpr u32 tc_abytes(u32 k) { return 128 * tc_kp(k); }        // one A tile

// ---------------------------------------------------------------------------------------------
// Wide-operand kernel (mr_wide.cu, k > 129: channels on threads, 16 messages per CTA).
// Per-k table in HBM (word Montgomery reductions: the 2^-32 factors are folded into the constants):
// ---------------------------------------------------------------------------------------------
// The four contraction matrices ([R][C], row = input channel / limb, column = output) are stored CHUNKED:
// rows in groups of 8, element (i, j) at ((i / 8) C + j) 8 + i % 8, rows padded with zeros to a multiple
// of 8, so the thread of column j loads a group's 8 coefficients as two 16-byte words (coalesced across
// the warp: 32 columns = 1 KB contiguous).  Offsets are multiples of 4 words (16-byte aligned).
__host__ __device__ constexpr u32 wch_rows(u32 r) { return (r + 7) & ~7u; }
__host__ __device__ constexpr u32 wch_words(u32 r, u32 c) { return wch_rows(r) * c; }
__host__ __device__ constexpr u32 wch_at(u32 i, u32 j, u32 c) { return ((i >> 3) * c + j) * 8 + (i & 7); }
struct WideLayout {
    u32 mm, minv, r32;        // [2k] m, -m^-1 mod 2^32, 2^32 mod m   (B then B')
    u32 xw;                   // [k]  |M^-1 λ_j^-1| 2^64 mod m'_j       (t*_j carries 2^-32 twice)
    u32 a1r, a2r;             // [k]  |M_i|_{2^32}, |M'_j|_{2^32}
    u32 pinw;                 // [k]  (m_i - |M'|_{m_i}) 2^32 mod m_i
    u32 misc;                 // [4]  M^-1 mod 2^32, M'^-1 mod 2^32
    u32 a2w;                  // chunked [k][k] row j, column i: |M'_j|_{m_i} 2^32 mod m_i
    u32 pow;                  // chunked [k][2k] |2^(32 l) 2^32|_{m_c} (B' × λ_j)
    u32 mpl;                  // chunked [k][k+1] M'_j limbs
    u32 nmp;                  // [k+1] 2^(32(k+1)) - M' limbs
    // Miller-Rabin (per-candidate moduli, unmerged BE1; mr_wide.cu k_mr_*_wide):
    u32 a1w;                  // chunked [k][k] row i, column j: |M_i|_{m'_j} 2^32 mod m'_j
    u32 lam, mu, mis;         // [k] λ_j = |M'_j^-1|_{m'_j}, μ_j = |M^-1|_{m'_j}, |M_i|_{m_i}
    u32 ml;                   // [k+1] M limbs
    u32 one;                  // [2k+1] RNS image of 1 (B' in ξ-form)
    u32 words;
};
__host__ __device__ constexpr WideLayout wide_layout(u32 k) {
    WideLayout w{};
    w.mm = 0;
    w.minv = w.mm + 2 * k;
    w.r32 = w.minv + 2 * k;
    w.xw = w.r32 + 2 * k;
    w.a1r = w.xw + k;
    w.a2r = w.a1r + k;
    w.pinw = w.a2r + k;
    w.misc = w.pinw + k;
    w.a2w = (w.misc + 4 + 3) & ~3u;
    w.pow = w.a2w + wch_words(k, k);
    w.mpl = w.pow + wch_words(k, 2 * k);
    w.nmp = w.mpl + wch_words(k, k + 1);
    w.a1w = (w.nmp + k + 1 + 3) & ~3u;
    w.lam = w.a1w + wch_words(k, k);
    w.mu = w.lam + k;
    w.mis = w.mu + k;
    w.ml = w.mis + k;
    w.one = w.ml + k + 1;
    w.words = w.one + 2 * k + 1;
    return w;
}
// per-context wide section, after the cx block: σ_i 2^64 mod m_i [k], then A1'[i][j] 2^32 mod m'_j chunked
// [k][k] (A1' = |M_i|_{m'_j} |N M^-1 λ_j|)
__host__ __device__ constexpr u32 wide_cx_sig(u32 k) { return 0; }
__host__ __device__ constexpr u32 wide_cx_a1(u32 k) { return (k + 3) & ~3u; }
__host__ __device__ constexpr u32 wide_cx_words(u32 k) { return wide_cx_a1(k) + wch_words(k, k); }
__host__ __device__ constexpr bool is_wide(u32 k) { return k > 129; }
// Per-candidate rows of the wide Miller-Rabin kernels (row r of candidate i at pcw[r * count + i]):
__host__ __device__ constexpr u32 wmr_sig(u32 k) { return 0; }            // [k]    σ_i 2^64 mod m_i
__host__ __device__ constexpr u32 wmr_c2(u32 k) { return k; }             // [k]    |n M^-1 λ_j| 2^32 mod m'_j
__host__ __device__ constexpr u32 wmr_r2(u32 k) { return 2 * k; }         // [2k+1] RNS image of M^2 mod n
__host__ __device__ constexpr u32 wmr_nminv(u32 k) { return 4 * k + 1; }  // [1]    n M^-1 mod 2^32
__host__ __device__ constexpr u32 wmr_s(u32 k) { return 4 * k + 2; }      // [1]    s with n - 1 = 2^s d
__host__ __device__ constexpr u32 wmr_live(u32 k) { return 4 * k + 3; }   // [1]    1 = run the rounds
__host__ __device__ constexpr u32 wmr_d(u32 k) { return 4 * k + 4; }      // [k]    d limbs
__host__ __device__ constexpr u32 wmr_n(u32 k) { return 5 * k + 4; }      // [k+1]  n limbs (0 above the input's)
__host__ __device__ constexpr u32 wmr_scr(u32 k) { return 6 * k + 5; }    // [2k+4] setup scratch (positional M^2 mod n)
__host__ __device__ constexpr u32 wmr_words(u32 k) { return 8 * k + 9; }

// ---------------------------------------------------------------------------------------------
// Tensor-core wide kernel (mr_tcw.cuh, k = 97 and 129: 3072- / 4096-bit moduli and the CRT halves of
// 6144- / 8192-bit keys).  The byte-split contraction of tc_* above, but the B images
// (k² words × 16 bytes) no longer fit shared memory, so they are STREAMED from L2 by the bulk-copy
// (TMA) engine, one [chunk rows × 128 K-bytes] slab per pipeline stage.  Four contraction types share
// the machinery ("extensions" e):
//   TCW_BE1  BE1 merged with 6.4: outputs j < k (B') and j = k (the m_r column q̂_r)     k+1 outputs
//   TCW_BE2  BE2 with the α' column                                                       k outputs
//   TCW_TRN  positional -> RNS (to_rns): outputs = the 2k channels                       2k outputs
//   TCW_EXT  RNS -> positional (exit): outputs = the k+1 limbs of X (4 byte positions)   k+1 outputs
// Each output owns 4 accumulator columns (byte b of the constant; for TCW_EXT byte position 4L+b).
// A CTA runs TCW_TILES = 2 independent 128-message tiles; each tile owns, in TMEM, the B residues of its
// state (round4(k) columns) and one accumulator buffer; outputs are cut into chunks (multiples of 4
// outputs) whose 4·outputs columns, rounded to 16, fit that buffer: 2·(round4(k) + NCMAX) <= 512.
// K: every extension reads the whole A row of tcw_kp(k) bytes (zero-padded): 13 K-steps of 32 bytes at
// k = 97, 17 at k = 129, grouped in slabs of 4 steps (the last slab shorter).
// Global image of an extension: the blocks (chunk c, slab s) back to back, each NC_c × 32·steps_s
// bytes in the K-major SWIZZLE_NONE core-matrix layout with SBO = steps_s·256 (LBO = 128).
// ---------------------------------------------------------------------------------------------
enum : u32 { TCW_BE1 = 0, TCW_BE2 = 1, TCW_TRN = 2, TCW_EXT = 3 };
__host__ __device__ constexpr bool tcw_k(u32 k) { return k == 97 || k == 129 || k == 257 || k == 505; }
// messages per tile: at k = 505 a 128-row A tile (2,048-byte rows) would be 256 KB, so the tile is 64 messages and the
// MMAs are M = 64 (the accumulator then sits in TMEM lanes 16q .. 16q + 15 of each lane quadrant q)
__host__ __device__ constexpr u32 tcw_m(u32 k) { return k > 257 ? 64u : 128u; }
// B residues in TMEM (k <= 257) or in an L2-resident global scratch slot (k = 505: they would take 508 columns)
__host__ __device__ constexpr bool tcw_bres_tmem(u32 k) { return k <= 257; }
__host__ __device__ constexpr u32 tcw_kp(u32 k) { return (4 * k + 4 + 31) & ~31u; }     // A row bytes (α' word k)
__host__ __device__ constexpr u32 tcw_ks(u32 k) { return tcw_kp(k) / 32; }               // K-steps
__host__ __device__ constexpr u32 tcw_nslab(u32 k) { return (tcw_ks(k) + 3) / 4; }
__host__ __device__ constexpr u32 tcw_steps(u32 k, u32 s) { return s + 1 < tcw_nslab(k) ? 4u : tcw_ks(k) - 4 * s; }
__host__ __device__ constexpr u32 tcw_bsw(u32 k) { return tcw_bres_tmem(k) ? (k + 3) & ~3u : 0u; }   // TMEM columns of B residues
__host__ __device__ constexpr u32 tcw_nout(u32 k, u32 e) {
    return e == TCW_BE1 ? k + 1 : e == TCW_BE2 ? k : e == TCW_TRN ? 2 * k : k + 1;
}
constexpr u32 TCW_TILES = 2;
// tiles per CTA at channel count k: at k = 257 one 128-message A tile is 135 KB of shared memory and its B residues
// take 260 TMEM columns, so a CTA runs a single tile (with two compute warps per lane quadrant, tcw_halves)
__host__ __device__ constexpr u32 tcw_tiles(u32 k) { return k > 129 ? 1u : TCW_TILES; }
// MR_TCW_LOCK = 1: the two tiles of a CTA run jobs of the same context in lockstep and share ONE stream of B slabs
// (each slab feeds both tiles' MMAs: half the L2 traffic); 0: independent tiles, one stream each
#ifndef MR_TCW_LOCK
#define MR_TCW_LOCK 0
#endif
constexpr bool TCW_LOCK = MR_TCW_LOCK != 0;
// MR_TCW_PAIR = 1: CTA pairs (2-CTA clusters) issue M = 256 MMAs (tcgen05 cta_group::2) over the two CTAs' 128-message
// tiles, and each CTA streams only HALF of every B slab (its N/2 rows): the slab copies run at the chip's L2 -> SM
// bandwidth cap, so halving the bytes each SM ingests per multiplication halves the MMA phases
#ifndef MR_TCW_PAIR
#define MR_TCW_PAIR 0
#endif
constexpr bool TCW_PAIR = MR_TCW_PAIR != 0 && !TCW_LOCK;
// largest outputs per chunk (multiple of 4) whose columns fit a tile's accumulator buffer (MR_TCW_OCCAP: a smaller cap
// trades MMA width for epilogue registers; host and device must be built with the same value)
#ifndef MR_TCW_OCCAP
#define MR_TCW_OCCAP 64
#endif
__host__ __device__ constexpr u32 tcw_ocmax(u32 k) {
    return (((512 / tcw_tiles(k) - tcw_bsw(k)) & ~15u) / 4 & ~3u) < MR_TCW_OCCAP
               ? (((512 / tcw_tiles(k) - tcw_bsw(k)) & ~15u) / 4 & ~3u)
               : MR_TCW_OCCAP;
}
__host__ __device__ constexpr u32 tcw_nchunks(u32 k, u32 e) { return (tcw_nout(k, e) + tcw_ocmax(k) - 1) / tcw_ocmax(k); }
__host__ __device__ constexpr u32 tcw_oc(u32 k, u32 e) {                                 // outputs per chunk (last: rest)
    return ((tcw_nout(k, e) + tcw_nchunks(k, e) - 1) / tcw_nchunks(k, e) + 3) & ~3u;
}
__host__ __device__ constexpr u32 tcw_out0(u32 k, u32 e, u32 c) { return c * tcw_oc(k, e); }
__host__ __device__ constexpr u32 tcw_outn(u32 k, u32 e, u32 c) {
    return tcw_out0(k, e, c) + tcw_oc(k, e) <= tcw_nout(k, e) ? tcw_oc(k, e) : tcw_nout(k, e) - tcw_out0(k, e, c);
}
__host__ __device__ constexpr u32 tcw_nc(u32 k, u32 e, u32 c) { return (4 * tcw_outn(k, e, c) + 15) & ~15u; }  // MMA N
__host__ __device__ constexpr u32 tcw_ncmax(u32 k) {
    u32 m = 0;
    for (u32 e = 0; e < 4; e++)
        for (u32 c = 0; c < tcw_nchunks(k, e); c++) m = tcw_nc(k, e, c) > m ? tcw_nc(k, e, c) : m;
    return m;
}
__host__ __device__ constexpr u32 tcw_stage_bytes(u32 k) { return tcw_ncmax(k) * 128; }
__host__ __device__ constexpr u32 tcw_blk_bytes(u32 k, u32 e, u32 c, u32 s) { return tcw_nc(k, e, c) * 32 * tcw_steps(k, s); }
__host__ __device__ constexpr u32 tcw_blk_off(u32 k, u32 e, u32 c, u32 s) {              // bytes from the image start
    u32 o = 0;
    for (u32 cc = 0; cc < c; cc++) o += tcw_nc(k, e, cc) * tcw_kp(k);
    for (u32 ss = 0; ss < s; ss++) o += tcw_blk_bytes(k, e, c, ss);
    return o;
}
__host__ __device__ constexpr u32 tcw_img_bytes(u32 k, u32 e) { return tcw_blk_off(k, e, tcw_nchunks(k, e), 0); }
// byte (row r of chunk c, K byte kb) of an extension image
__host__ __device__ constexpr u32 tcw_at(u32 k, u32 e, u32 c, u32 r, u32 kb) {
    const u32 s = kb / 128, kl = kb % 128;
    return tcw_blk_off(k, e, c, s) + (r / 8) * (tcw_steps(k, s) * 256) + (kl / 16) * 128 + (r % 8) * 16 + kl % 16;
}
// per-k image buffer: BE2 | TRN | EXT (each 16-byte aligned; BE1 is per context, after the wide section)
__host__ __device__ constexpr u32 tcw_img_off(u32 k, u32 e) {
    return e == TCW_BE2 ? 0u : e == TCW_TRN ? tcw_img_bytes(k, TCW_BE2) : tcw_img_bytes(k, TCW_BE2) + tcw_img_bytes(k, TCW_TRN);
}
__host__ __device__ constexpr u32 tcw_kimg_bytes(u32 k) { return tcw_img_off(k, TCW_EXT) + tcw_img_bytes(k, TCW_EXT); }
// per-context words after the wide section: the BE1 image
__host__ __device__ constexpr u32 tcw_cx_words(u32 k) { return tcw_img_bytes(k, TCW_BE1) / 4; }

// ---------------------------------------------------------------------------------------------
// Exponentiation "program": one u64 op per Montgomery multiplication step, executed by a single
// inlined mont_mul inside the kernel's interpreter loop (keeps one copy of the unrolled code).
// ---------------------------------------------------------------------------------------------
enum : u32 {
    OPF_TORNS_ALL = 1u,   // before: acc = to_rns(input limbs [0, in_limbs))
    OPF_TORNS_LO = 2u,    // before: acc = to_rns(input limbs [0, half))
    OPF_TORNS_HI = 4u,    // before: acc = to_rns(input limbs [half, 2 half))
    OPF_LOAD = 8u,        // before: acc = operand(load)
    OPF_NOMUL = 16u,      // skip the Montgomery multiplication
    OPF_ADD = 32u,        // after: acc = acc + table[add]  (channel-wise)
    OPF_STORE = 64u,      // after: table[store] = acc
};
enum : u32 { OPND_SQ = 0xFF, OPND_R2 = 0xF0, OPND_ONE = 0xF1, OPND_KHI = 0xF2, OPND_QINVR = 0xF3 };
__host__ __device__ constexpr u64 make_op(u32 flags, u32 opnd, u32 load = 0, u32 add = 0, u32 store = 0) {
    return (u64)(flags & 0xFF) | ((u64)(opnd & 0xFF) << 8) | ((u64)(load & 0xFF) << 16) |
           ((u64)(add & 0xFF) << 24) | ((u64)(store & 0xFF) << 32);
}

// ---------------------------------------------------------------------------------------------
// Kernel launch parameter blocks (plain structs passed by value).
// ---------------------------------------------------------------------------------------------
struct ModexpParams {
    const u32 *ctx[2];        // device context blocks; CTA b uses ctx[b >= ctas0]
    const u64 *prog[2];       // device programs
    u32 nops[2];
    u32 ctas0;                // CTAs of the first context
    u32 count;                // messages per context
    const u32 *x;             // [count][in_limbs]
    u32 in_limbs;             // limbs per input row
    u32 half;                 // CRT: limbs per half (inputs split at `half`)
    u32 *y;                   // [count][out_limbs] per context: y + ctxsel * out_stride
    u32 out_limbs;
    size_t out_stride;        // words between the two contexts' outputs
    int32_t *status;          // nullable
    u32 *table;               // window table [slot][2k+1][jobs_total]
    u32 jobs_total;           // = 2 * ctas0 * blockDim (or ctas0 * blockDim)
    const u32 *pow_tab;       // to_rns powers [k][2k]
    const u32 *be_tab;        // base-extension image (be_words(k))
    const u32 *tc_b2;         // tensor-core BE2 image (tc_bbytes(k)); BE1 image follows each ctx block
    const u32 *mpl;           // M'_j limbs [k][k+1] (global; exit conversion)
    u32 tc_be1_off;           // word offset of the BE1 tensor image inside a context buffer
    u32 tc_be2_off;           // word offset of the (ρ-scaled, per-context) BE2 tensor image
    u32 tc_gc;                // tensor kernel: persistent CTAs (CTA pairs in pair mode) per context group
    // tensor kernel, split schedule: a job whose ops straddle two tile slots hands its
    // state over through table slot `hslot` and a per-(job, rank) flag (zeroed before the launch)
    u32 hslot;                // handoff slot index in the window table (= table_slots(w))
    u32 *flags;               // [2 contexts][jobs][2 ranks] + 1 start ticket; null = no split schedule
};

struct CombineParams {          // CRT recombination m = m_q + q ((m_p - m_q) qinv mod p)
    const u32 *ctx_p;
    const u32 *q;               // [half] limbs of q
    const u32 *mpq;             // [2][count][half]: m_p rows then m_q rows
    u32 count, half;
    u32 *m;                     // [count][2 half]
    int32_t *status;            // nullable (range flag already written by the ladder kernel)
    const u32 *pow_tab;
    const u32 *be_tab;
    const u32 *mpl;
};

struct MrParams {               // Miller-Rabin (§3.2; HAC 4.24)
    const u32 *n;               // [count][limbs] candidates
    const u32 *bases;           // [count][rounds][limbs]
    u32 count, limbs, rounds, window;
    u32 forced;                 // 1: run every round for every candidate (benchmark mode)
    u32 *pc;                    // per-candidate constants [pc_words(k)][count] (structure of arrays)
    u32 *table;                 // [2^w + 1][2k+1][count] window table + stash slot
    uint8_t *verdict;
    int16_t *witness;
    int32_t *status;
    const u32 *pow_tab;
    const u32 *be_tab;
    const u32 *mpl;
    const u32 *tc_b1;           // tensor path: unmerged BE1 image (per k); null = IMAD path
    const u32 *tc_b2;           // tensor path: BE2 image
    u32 tc_gc;                  // tensor path: persistent CTAs
    const u32 *one_g;           // tensor path: RNS image of 1 (per k) in global memory (multiplicand loads are ld.global)
    // tensor path, early-exit compaction: mode 0 = every round in one tile-job (forced, or a
    // single round); mode 1 = round 0 for every candidate, survivors appended to live[] (count *nlive);
    // mode 2 = items (live candidate, round r >= 1) as independent one-round jobs, the first failing
    // round min-reduced into wit32[]; k_mr_final folds wit32 into verdict/witness.
    u32 mode;
    u32 *live;                  // [count]
    u32 *nlive;                 // device counter
    u32 *wit32;                 // [count]
    u32 tstride;                // window-table stride: count (modes 0, 1) or persistent slots (mode 2)
};

// per-candidate constant rows for Miller-Rabin (row r at pc + r * count)
__host__ __device__ constexpr u32 pc_sigma(u32 k) { return 0; }                 // [k]  |-n^-1 M_i^-1|_{m_i}
__host__ __device__ constexpr u32 pc_c2(u32 k) { return k; }                    // [k]  |n M^-1 λ_j|_{m'_j}
__host__ __device__ constexpr u32 pc_r2(u32 k) { return 2 * k; }                // [2k+1] M^2 mod n (RNS)
__host__ __device__ constexpr u32 pc_nminv(u32 k) { return 4 * k + 1; }         // [1]  n M^-1 mod 2^32
__host__ __device__ constexpr u32 pc_s(u32 k) { return 4 * k + 2; }             // [1]  s with n - 1 = 2^s d
__host__ __device__ constexpr u32 pc_live(u32 k) { return 4 * k + 3; }          // [1]  1 = run the rounds
__host__ __device__ constexpr u32 pc_d(u32 k) { return 4 * k + 4; }             // [k]  d limbs
__host__ __device__ constexpr u32 pc_n(u32 k) { return 5 * k + 4; }             // [k+1] n limbs (0 above limbs),
                                                                                  // column layout: coalesced reads
__host__ __device__ constexpr u32 pc_sig64(u32 k) { return 6 * k + 5; }         // [k]  σ_i 2^64 mod m_i (canonical)
__host__ __device__ constexpr u32 pc_words(u32 k) { return 7 * k + 5; }

// ---------------------------------------------------------------------------------------------
// Per-k entry points exported by each mr_k<K>.cu translation unit.
// ---------------------------------------------------------------------------------------------
struct KernelSet {
    int k;
    int (*upload_base)(const u32 *flat, int device);     // fills __constant__ tables on `device`
    int (*launch_modexp)(const ModexpParams &p, u32 ctas, void *stream);
    int (*launch_combine)(const CombineParams &p, void *stream);
    int (*launch_mr)(const MrParams &p, void *stream);
    int (*launch_modexp_tc)(const ModexpParams &p, u32 ctas, void *stream);   // null when unsupported
    int tc_tiles;                                         // 128-message tiles per CTA of the TC kernel
    int threads;                                          // CTA size used by launch_modexp
    int mr_tiles;                                         // 128-candidate tiles per CTA of k_mr_rounds_tc
    // tensor-core wide kernel (k = 97, 129; mr_tcw.cuh), null elsewhere: tab = wide table, kimg = per-k images
    int (*launch_modexp_tcw)(const ModexpParams &p, u32 ctas, const u32 *tab, const void *kimg, u32 cxw, u32 be1w,
                             u32 jobs, void *trace, void *stream);
};

}  // namespace mr
