// mr_tcw.cuh — tensor-core modexp for wide operands, k = 97 and 129 (3072- / 4096-bit moduli, CRT halves of
// 6144- / 8192-bit keys): SURVEY §8(f) rows 2-3, DESIGN.md §4k.  Included by mr_kernels.cuh inside its
// per-k anonymous namespace (MR_K = 97 or 129), or by mr_tcw257.cu (MR_K = 257: one tile per CTA), so K, NCH, SMAX,
// mont_red(), less_than() are this TU's.
//
// The arithmetic is the RNS Montgomery multiplication of mr_kernels.cuh (§3.1) in the plain
// word-Montgomery form of the wide kernel (mr_wide.cu: every product reduced by mont_red, the 2^-32 factors
// absorbed into host constants, any odd 32-bit modulus), with ALL FOUR contractions on the tensor cores as
// u8 x u8 -> s32 byte-split MMAs (tcgen05.mma.kind::i8):
//   BE1 (6.3-6.5, merged)    D ≡ Σ_i ξ_i A1'_ij 2^64 (mod m'_j), plus the m_r column q̂_r = Σ_i ξ_i |M_i|_{2^32}
//   BE2 (6.6, α' column)     D ≡ (Σ_j ξ'_j A2_ji + α'(m_i - |M'|_{m_i})) 2^32 (mod m_i)
//   TRN (a2, to_rns)         D ≡ Σ_l x_l |2^(32l)|_{m_c} 2^32 (mod m_c)   (B' entries × λ_j: ξ-form)
//   EXT (a7, exit)           D[p] = Σ byte_a(ξ'_j) byte_{p-a}(M'_j) + α' bytes × (2^(32(k+1)) - M'): the byte
//                            convolution of X = Σ_j ξ'_j M'_j + α'(2^(32(k+1)) - M'), carried into limbs per thread
// The B images (16k² bytes per extension: 150 KB at k = 97) exceed shared memory, so they are STREAMED from L2
// by the bulk-copy (TMA) engine through a ring of stages, one [chunk rows x 128 K-bytes] slab per stage.
//
// A CTA runs W_TILES = 2 (k = 257: 1) independent tiles of 128 messages (one message per thread, the 128 TMEM lanes), each
// with its own producer thread (stage ring), MMA-issuer thread, accumulator buffer and four compute warps, so one
// tile's CUDA-core phases (channel products, epilogues) run under the other tile's MMAs.
// State of a message (the shared memory of two tiles holds only their A tiles and stages):
//   B residues   TMEM columns [BS, BS + k) of the tile, lane = message
//   B' (ξ-form)  its A row, words 0 .. k-1 — exactly the BE2 / exit input, so no copy after BE2
//   m_r          its A row, word k+1 (the images are zero in those K columns)
// The A row is also each contraction's input; an extension whose outputs would overwrite inputs still needed by
// later chunks parks them in TMEM (BE1: ξ'_j in place of t*_j in the B columns) or in HBM (to_rns: the B' outputs
// in the window table's spare slot), and the A row is written once all chunks are done.
#pragma once

#if MR_K == 97 || MR_K == 129 || MR_K == 257 || MR_K == 505

constexpr u32 W_TILES = tcw_tiles(K);                 // independent 128-message tiles per CTA (k = 257: one)

constexpr u32 W_M = tcw_m(K);                         // messages per tile (k = 505: 64, M = 64 MMAs)
constexpr bool W_BT = tcw_bres_tmem(K);               // B residues in TMEM (else the global scratch slot)
constexpr u32 W_KP = tcw_kp(K);                       // A row bytes
constexpr u32 W_KC = W_KP / 16;                       // K-cores (4 words) per A row
constexpr u32 W_SBOA = (W_KP / 16) * 128;             // A tile: bytes between 8-row groups
constexpr u32 W_NCMAX = tcw_ncmax(K);                 // TMEM columns of a tile's accumulator buffer
constexpr u32 W_BSW = tcw_bsw(K);
constexpr u32 W_TCOLS = W_NCMAX + W_BSW;              // TMEM columns per tile: [acc | B residues]
static_assert(W_TILES * W_TCOLS <= 512, "tiles x (accumulator + B residues) exceed the 512 TMEM columns");
static_assert(W_KC * 4 >= K + 2, "A row must hold B' (k words), α' (word k) and m_r (word k+1)");
constexpr bool W_PAIR = TCW_PAIR && W_M == 128;                     // CTA pairs: M = 256 MMAs, each CTA streams half of every slab
constexpr u32 W_STG = tcw_stage_bytes(K) / (W_PAIR ? 2u : 1u);   // bytes of one stage (pair: the CTA's N/2 rows)
constexpr u32 W_ABYTES = W_M * W_KP;
constexpr size_t W_FIXED = (size_t)W_TILES * W_ABYTES + 16 * K + 8 * K + 8 * K + 512 + W_TILES * 2048;
constexpr u32 W_RINGS = TCW_LOCK ? 1 : W_TILES;       // streams of B slabs per CTA
constexpr u32 W_NST_FIT = (u32)((232448 - W_FIXED) / (W_RINGS * W_STG));
constexpr u32 W_NST = W_NST_FIT > 8 ? 8 : W_NST_FIT;  // pipeline stages per stream
static_assert(W_NST >= 2, "tensor wide kernel: fewer than two B stages per tile fit shared memory");
constexpr size_t W_SMEM = W_FIXED + (size_t)W_RINGS * W_NST * W_STG;
constexpr u32 W_SUB = TCW_LOCK ? W_TILES : 1;         // tiles served by one stream (one producer, one MMA issuer)
#ifndef MR_TCW_HALVES
#define MR_TCW_HALVES 1       // compute warps per TMEM lane quadrant and tile (2: each takes alternate channel groups)
#endif
constexpr u32 W_HV = K > 129 ? 2u : (u32)MR_TCW_HALVES;   // k = 257: 8 compute warps for the single tile
#ifndef MR_TCW_CHAN_PIPE
#define MR_TCW_CHAN_PIPE 0    // 1: next group's operand loads under the current group's products (A/B: 9 % slower, spills)
#endif
constexpr u32 W_CW = 4 * W_HV * W_TILES;              // compute warps
constexpr u32 W_THREADS = 32 * (W_CW + 2 * W_TILES);     // + per tile a producer warp and an MMA warp (one lane each:
                                                         // two roles in one warp would sleep on each other's waits)
constexpr u32 W_NBAR = 2 * W_NST + 3;
#ifndef MR_TCW_CMPTOP
#define MR_TCW_CMPTOP 1 // exit: compare X with N 2^s from the top limb (usually one limb) before a full subtraction pass
#endif
#ifndef MR_TCW_VEC
#define MR_TCW_VEC 1    // 16-byte loads of the input rows in to_rns and 16-byte stores of the output rows
#endif
#ifndef MR_TCW_FRAC
#define MR_TCW_FRAC 1   // α' from the top bits of the ξ'_j (reading R2b) instead of the m_r channel
#endif
// s = Σ_j (ξ'_j >> W_FSH) stays below 2^32 (k < 2^W_FSH) and α' = (s + 2^(26 - W_FSH)) >> (32 - W_FSH): the shift drops
// < k 2^(W_FSH - 32) and ξ'_j / 2^32 undercuts ξ'_j / m'_j by < k max c'_j / m'_j, together < 2^-6 for every tensor-wide
// k (2^-9.5 at k = 505), while r / M' < 2^-20; pinned by tests/test_abi_host.py::test_fractional_alpha_bound_wide
constexpr u32 W_FSH = K <= 129 ? 8u : (K <= 257 ? 9u : 10u);
// with the m_r channel (MR_TCW_FRAC = 0) the thread that forms r_r reads A-row word k+1, which at k = 505 the other half
// of the tile writes (16-word group 31) with no barrier in between: that variant is only valid up to k = 257
static_assert(MR_TCW_FRAC || K <= 257, "k = 505 needs the fractional α' (MR_TCW_FRAC = 1)");
__device__ __forceinline__ u32 w_frac_alpha(u32 s) { return (s + (1u << (26 - W_FSH))) >> (32 - W_FSH); }                 // per tile: full[NST] empty[NST] accf acce aready

struct TcwArgs {
    const u32 *wtab;          // per-k wide table (mr_internal.h wide_layout): m, -m^-1, C1 2^64, |M'_j|_{2^32}
    const uint8_t *kimg;      // per-k images: BE2 | TRN | EXT (tcw_img_off)
    u32 cxw;                  // word offset of the wide section (σ_i 2^64) in a context block
    u32 be1w;                 // word offset of the context's BE1 image in its context block
    u32 jobs;                 // 128-message tile-jobs over all contexts (ctas0 per context)
    unsigned long long *trace;   // debug timeline (MR_TCW_TRACE, CTA 0 only): [0] = count, then (clock << 16 | code)
};
// code = tile << 12 | role << 8 | event (role 0 compute thread 0, 1 MMA issuer, 2 producer); each (tile, role) writes
// its own region of W_TRN entries with plain stores (no atomics: the trace must not perturb the timeline)
constexpr u32 W_TRN = 2700;
struct WTrace {
    unsigned long long *p = nullptr;
    u32 n = 0, code = 0;
    __device__ void init(unsigned long long *tr, u32 tile, u32 role) {
        if (tr && blockIdx.x == 0) {
            p = tr + 1 + (tile * 3 + role) * W_TRN;
            code = tile << 12 | role << 8;
        }
    }
    __device__ void operator()(u32 ev) {
        if (p && n < W_TRN) {
            long long c;
            asm volatile("mov.u64 %0, %%clock64;" : "=l"(c));
            p[n++] = ((unsigned long long)c << 16) | code | ev;
        }
    }
};
__device__ __forceinline__ u64 mulw(u32 a, u32 b) {   // one IMAD.WIDE.U32
    u64 r;
    asm("mul.wide.u32 %0, %1, %2;" : "=l"(r) : "r"(a), "r"(b));
    return r;
}
__device__ __forceinline__ u64 madw(u32 a, u32 b, u64 c) {
    u64 r;
    asm("mad.wide.u32 %0, %1, %2, %3;" : "=l"(r) : "r"(a), "r"(b), "l"(c));
    return r;
}

__device__ __forceinline__ u32 smem_u32(const void *p) { return (u32)__cvta_generic_to_shared(p); }
// byte-column combine V = d0 + 2^8 d1 + 2^16 d2 + 2^24 d3 (< 2^49.2 for d_b < 2^25.1) as three wide multiply-adds
// (3 IMAD.WIDE instead of 6 shifts + 6 carry adds)
__device__ __forceinline__ u64 tc_comb(u32 d0, u32 d1, u32 d2, u32 d3) {
    u64 v;
    asm("mad.wide.u32 %0, %1, 256, %2;\n\t"
        "mad.wide.u32 %0, %3, 65536, %0;\n\t"
        "mad.wide.u32 %0, %4, 16777216, %0;"
        : "=l"(v)
        : "r"(d1), "l"((u64)d0), "r"(d2), "r"(d3));
    return v;
}
// the same sum as hi 2^32 + lo with shifts and one carry chain (ALU pipe; the FMA-heavy pipe is the contended one)
__device__ __forceinline__ void tc_split(u32 d0, u32 d1, u32 d2, u32 d3, u32 &lo, u32 &hi) {
    asm("add.cc.u32 %0, %2, %3;\n\taddc.u32 %1, %4, 0;\n\t"
        "add.cc.u32 %0, %0, %5;\n\taddc.u32 %1, %1, %6;\n\t"
        "add.cc.u32 %0, %0, %7;\n\taddc.u32 %1, %1, %8;"
        : "=r"(lo), "=r"(hi)
        : "r"(d0), "r"(d1 << 8), "r"(d1 >> 24), "r"(d2 << 16), "r"(d2 >> 16), "r"(d3 << 24), "r"(d3 >> 8));
}
__device__ __forceinline__ void w_mbar_init(u32 a, u32 n) { asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(a), "r"(n)); }
__device__ __forceinline__ u64 w_gtimer() {
    u64 t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}
// wait for phase `par` of an mbarrier; try_wait with a suspend-time hint parks the thread in hardware until the phase
// completes (instead of re-issuing the test); a wait longer than 30 s traps instead of hanging the GPU
template <bool CL = false>   // CL: acquire at cluster scope (the barrier also counts arrivals of the peer CTA)
__device__ __forceinline__ void w_mbar_wait(u32 a, u32 par) {
    u32 done = 0;
    u64 t0 = 0;
#pragma unroll 1
    for (u32 spin = 0; !done; spin++) {
        if constexpr (CL)
            asm volatile("{\n\t.reg .pred P1;\n\tmbarrier.try_wait.parity.acquire.cluster.shared::cta.b64 P1, [%1], %2, %3;\n\t"
                         "selp.u32 %0, 1, 0, P1;\n\t}"
                         : "=r"(done)
                         : "r"(a), "r"(par), "r"(1000000u)
                         : "memory");
        else
            asm volatile("{\n\t.reg .pred P1;\n\tmbarrier.try_wait.parity.shared::cta.b64 P1, [%1], %2, %3;\n\tselp.u32 %0, 1, 0, P1;\n\t}"
                         : "=r"(done)
                         : "r"(a), "r"(par), "r"(1000000u)
                         : "memory");
        if (!done && (spin & 255) == 255) {
            const u64 t = w_gtimer();
            if (!t0) t0 = t;
            else if (t - t0 > 30000000000ull) __trap();
        }
    }
}
__device__ __forceinline__ void w_mbar_arrive(u32 a) { asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(a) : "memory"); }
// arrive on a barrier of another CTA of the cluster (cluster-window address), releasing this thread's prior writes
__device__ __forceinline__ void w_mbar_arrive_cl(u32 ca) {
    asm volatile("mbarrier.arrive.release.cluster.shared::cluster.b64 _, [%0];" ::"r"(ca) : "memory");
}
// cluster-window address of the same shared-memory offset in the pair's leader CTA (rank 0)
__device__ __forceinline__ u32 w_lead(u32 a) {
    u32 r;
    asm("mapa.shared::cluster.u32 %0, %1, 0;" : "=r"(r) : "r"(a));
    return r;
}
__device__ __forceinline__ void w_mbar_expect_tx(u32 a, u32 bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(a), "r"(bytes) : "memory");
}
// bulk copy global -> shared (the TMA engine, SASS UBLKCP), completion counted in bytes on the stage's mbarrier;
// the images are re-read by every SM for every multiplication: keep them in L2 (evict_last)
__device__ __forceinline__ void w_bulk_g2s(u32 dst, const void *src, u32 bytes, u32 bar, u64 pol) {
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], %4;"
                 ::"r"(dst), "l"(src), "r"(bytes), "r"(bar), "l"(pol) : "memory");
}
__device__ __forceinline__ u64 w_desc(u32 saddr, u32 sbo) {
    return (u64)((saddr >> 4) & 0x3FFF) | ((u64)(128u >> 4) << 16) | ((u64)(sbo >> 4) << 32) | ((u64)1 << 46);
}
// TMEM loads without a memory clobber: w_tmem_wait(v) orders the uses of the loaded registers, so independent loads
// (shared memory, the window table) can be issued while the TMEM load is in flight
__device__ __forceinline__ void w_tmem_ld16(u32 taddr, u32 (&v)[16]) {
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
                 : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]),
                   "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15])
                 : "r"(taddr));
}
__device__ __forceinline__ void w_tmem_ld8(u32 taddr, u32 (&v)[8]) {
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                 : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7])
                 : "r"(taddr));
}
__device__ __forceinline__ void w_tmem_ld4(u32 taddr, u32 (&v)[4]) {
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x4.b32 {%0,%1,%2,%3}, [%4];"
                 : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3])
                 : "r"(taddr));
}
template <int N>
__device__ __forceinline__ void w_tmem_wait(u32 (&v)[N]) {
    asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
    for (int i = 0; i < N; i++) asm volatile("" : "+r"(v[i]));   // the loaded registers are used after the wait
}
__device__ __forceinline__ void w_tmem_st4(u32 taddr, u32 a, u32 b, u32 c, u32 d) {
    asm volatile("tcgen05.st.sync.aligned.32x32b.x4.b32 [%0], {%1,%2,%3,%4};" ::"r"(taddr), "r"(a), "r"(b), "r"(c), "r"(d)
                 : "memory");
}
__device__ __forceinline__ void w_tmem_st16(u32 taddr, const u32 (&v)[16]) {
    asm volatile("tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16};"
                 ::"r"(taddr), "r"(v[0]), "r"(v[1]), "r"(v[2]), "r"(v[3]), "r"(v[4]), "r"(v[5]), "r"(v[6]), "r"(v[7]),
                 "r"(v[8]), "r"(v[9]), "r"(v[10]), "r"(v[11]), "r"(v[12]), "r"(v[13]), "r"(v[14]), "r"(v[15])
                 : "memory");
}
__device__ __forceinline__ void w_tmem_wait_st() { asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory"); }
// lazy a + b mod m (a, b < 2^32), r32 = 2^32 mod m (as mr_wide.cu)
__device__ __forceinline__ u32 w_addmod(u32 a, u32 b, u32 r32) {
    const u64 s = (u64)a + b;
    const u64 t = (u64)(u32)s + (s >> 32) * r32;
    return (u32)t + (u32)(t >> 32) * r32;
}

// chunk geometry of extension e (runtime e, compile-time K)
__device__ __forceinline__ u32 w_nchunks(u32 e) {
    return e == TCW_BE1 ? tcw_nchunks(K, TCW_BE1) : e == TCW_BE2 ? tcw_nchunks(K, TCW_BE2)
                        : e == TCW_TRN ? tcw_nchunks(K, TCW_TRN) : tcw_nchunks(K, TCW_EXT);
}
__device__ __forceinline__ u32 w_oc(u32 e) {
    return e == TCW_BE1 ? tcw_oc(K, TCW_BE1) : e == TCW_BE2 ? tcw_oc(K, TCW_BE2) : e == TCW_TRN ? tcw_oc(K, TCW_TRN)
                                                                                                : tcw_oc(K, TCW_EXT);
}
__device__ __forceinline__ u32 w_outn(u32 e, u32 c) {
    const u32 o0 = c * w_oc(e), n = tcw_nout(K, e);
    return o0 + w_oc(e) <= n ? w_oc(e) : n - o0;
}
__device__ __forceinline__ u32 w_nc(u32 e, u32 c) { return (4 * w_outn(e, c) + 15) & ~15u; }

struct TcwTile {               // one tile's shared memory and barriers
    uint8_t *a;                // A tile [128 x W_KP] core-matrix layout
    u32 stage0;                // shared address of its stage 0
    u32 bar;                   // shared address of its barriers: full[NST] empty[NST] accf acce aready
    u32 tacc;                  // TMEM column of its accumulator buffer (lane 0)
    u32 rank = 0;              // pair mode: CTA rank in the cluster (rank 0 issues the pair's MMAs)
    __device__ u32 full(u32 s) const { return bar + 8 * s; }
    __device__ u32 empty(u32 s) const { return bar + 8 * (W_NST + s); }
    __device__ u32 accf() const { return bar + 8 * (2 * W_NST); }
    __device__ u32 acce() const { return bar + 8 * (2 * W_NST + 1); }
    __device__ u32 aready() const { return bar + 8 * (2 * W_NST + 2); }
};

// ---------------------------------------------------------------- producer: stream the B slabs of an extension
struct TcwProducer {
    u32 st = 0, ph = 0;
    u64 pol;
    WTrace tr;
    __device__ void ext(const TcwTile &T, u32 e, const uint8_t *img) {
        u32 off = 0;
#pragma unroll 1
        for (u32 c = 0; c < w_nchunks(e); c++) {
            const u32 nc = w_nc(e, c);
#pragma unroll 1
            for (u32 s = 0; s < tcw_nslab(K); s++) {
                const u32 bytes = nc * 32 * tcw_steps(K, s);
                // pair mode: this CTA's N/2 rows = the first / second half of the block (row groups are outermost)
                const u32 hb = W_PAIR ? bytes / 2 : bytes;
                w_mbar_wait(T.empty(st), ph ^ 1u);
                tr((e << 4) | (s == 0 ? 1 : 2));
                w_mbar_expect_tx(T.full(st), hb);
                w_bulk_g2s(T.stage0 + st * W_STG, img + off + T.rank * hb, hb, T.full(st), pol);
                off += bytes;
                if (++st == W_NST) { st = 0; ph ^= 1u; }
            }
        }
    }
};

// ---------------------------------------------------------------- MMA issuer: one thread per tile
struct TcwMma {
    u32 st = 0, fph = 0, aph = 0, eph = 0;
    u32 tmem;
    WTrace tr;
    u32 sa1 = 0, td1 = 0;                  // lockstep: the second tile's A tile and accumulator
    // completion of the MMAs issued so far -> an mbarrier (pair: the same offset in both CTAs)
    __device__ static void commit(u32 bar) {
        if constexpr (W_PAIR)
            asm volatile("tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;"
                         ::"r"(bar), "h"((unsigned short)3) : "memory");
        else
            asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(bar) : "memory");
    }
    // pair mode, rank 1: forward each landed half-slab to the leader's full barrier (the bulk copy can only signal an
    // mbarrier of its own CTA); walks the same (extension, chunk, slab) sequence as the leader's issuer
    __device__ void relay(const TcwTile &T, u32 e) {
#pragma unroll 1
        for (u32 c = 0; c < w_nchunks(e); c++) {
#pragma unroll 1
            for (u32 s = 0; s < tcw_nslab(K); s++) {
                w_mbar_wait(T.full(st), fph);
                w_mbar_arrive_cl(w_lead(T.full(st)));
                if (++st == W_NST) { st = 0; fph ^= 1u; }
            }
        }
    }
    __device__ void ext(const TcwTile &T, u32 e) {
        w_mbar_wait<W_PAIR>(T.aready(), aph);  // the A rows of all 128 (pair: 256) messages are written (and proxy-fenced)
        aph ^= 1u;
        tr(e << 4);
        asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
        const u32 sa = smem_u32(T.a), td = tmem + T.tacc;
#pragma unroll 1
        for (u32 c = 0; c < w_nchunks(e); c++) {
            const u32 nc = w_nc(e, c);
            w_mbar_wait<W_PAIR>(T.acce(), eph ^ 1u);   // the epilogue (pair: of both CTAs) has read the previous chunk
            eph ^= 1u;
            tr((e << 4) | 1);
            asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
            // s32 = u8 x u8, K-major, M = 128 (pair: M = 256 over the two CTAs' tiles, N = nc with N/2 B rows per CTA)
            const u32 idesc = (2u << 4) | ((nc >> 3) << 17) | (((W_PAIR ? 256u : W_M) >> 4) << 24);
#pragma unroll 1
            for (u32 s = 0; s < tcw_nslab(K); s++) {
                const u32 steps = tcw_steps(K, s);
                w_mbar_wait<W_PAIR>(T.full(st), fph);   // pair: own half landed + the peer's relayed arrival
                tr((e << 4) | 3);
                asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
                const u32 sb = T.stage0 + st * W_STG;
#pragma unroll
                for (u32 u = 0; u < W_SUB; u++) {
#pragma unroll 1
                    for (u32 j = 0; j < steps; j++) {
                        const u64 da = w_desc((u ? sa1 : sa) + (4 * s + j) * 256, W_SBOA), db = w_desc(sb + j * 256, steps * 256);
                        const u32 accum = (s | j) ? 1u : 0u;
                        if constexpr (W_PAIR)
                            asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                                         "tcgen05.mma.cta_group::2.kind::i8 [%0], %1, %2, %3, p;\n\t}" ::"r"(td),
                                         "l"(da), "l"(db), "r"(idesc), "r"(accum)
                                         : "memory");
                        else
                            asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                                         "tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n\t}" ::"r"(u ? td1 : td),
                                         "l"(da), "l"(db), "r"(idesc), "r"(accum)
                                         : "memory");
                    }
                }
                commit(T.empty(st));           // stage free (pair: in both CTAs)
                if (++st == W_NST) { st = 0; fph ^= 1u; }
            }
            commit(T.accf());                  // chunk accumulated (pair: both CTAs' epilogues start)
            tr((e << 4) | 2);
        }
    }
};

// ---------------------------------------------------------------- compute warps
// A tile's 128 messages are served by 8 warps: warp (quadrant q, half h) owns messages 32q .. 32q+31 (its TMEM lane
// quadrant) and, of every group of 16 channels / 4 extension outputs, the groups whose index is ≡ h (mod 2).  The two
// halves meet at a named barrier where a step needs the other half's results (α', the B residues before the next
// multiplication, the parked to_rns outputs, the exit).
struct TcwCompute {
    const TcwTile &T;
    const uint4 *ep1;         // [K] (m'_j, -m'_j^-1, C1_j 2^64, |M'_j|_{2^32})
    const uint2 *ep2;         // [K] (m_i, -m_i^-1)
    const u32 *sig;           // [2][K] σ_i 2^64 mod m_i per context
    u32 tmem;                 // TMEM base + this warp's lane quadrant
    u32 bs;                   // TMEM column of the tile's B residues
    u32 m;                    // message = TMEM lane
    u32 h;                    // half: the groups ≡ h (mod 2)
    uint8_t *arow;            // this message's A row
    uint2 *xch;               // [2][128] per-half partial sums (α')
    u32 bar_id;               // named barrier of the tile's 256 compute threads
    u32 fph = 0;
    WTrace tr;                // trace (thread 0 of the tile only)
    __device__ void trace(u32 ev) { if (m == 0 && h == 0) tr(ev); }
    u32 minv_r = 0, mpinv_r = 0;   // M^-1 and M'^-1 mod 2^32 (the m_r channel, wide table misc)
    u32 sel = 0;              // context of the current job
    const u32 *cx = nullptr;  // its context block (HBM)

    __device__ u32 &aw(u32 i) const { return *reinterpret_cast<u32 *>(arow + (i >> 2) * 128 + 4 * (i & 3)); }
    __device__ uint4 &ac(u32 c) const { return *reinterpret_cast<uint4 *>(arow + c * 128); }   // K-core c: words 4c..4c+3
    __device__ u32 tb(u32 col) const { return tmem + col; }
    // lane 0 of the warp (M = 64: m no longer tells, lanes 16..31 shadow 0..15)
    __device__ bool lane0() const { return (W_M == 128 ? (m & 31) : (threadIdx.x & 31)) == 0; }
    // B residues / parked values: TMEM columns bs + c of this message's lane (k <= 257), or rows c of the job's global
    // scratch slot (k = 505, bres / bstr set per job); bld issues, bwait completes (TMEM loads are asynchronous)
    u32 *bres = nullptr;
    size_t bstr = 0;
    template <int N>
    __device__ __forceinline__ void bld(u32 c, u32 (&v)[N]) const {
        if constexpr (W_BT) {
            if constexpr (N == 16) w_tmem_ld16(tb(bs + c), v);
            else if constexpr (N == 8) w_tmem_ld8(tb(bs + c), v);
            else w_tmem_ld4(tb(bs + c), v);
        } else {
#pragma unroll
            for (int i = 0; i < N; i++) v[i] = bres[(size_t)(c + i) * bstr];
        }
    }
    template <int N>
    __device__ __forceinline__ void bwait(u32 (&v)[N]) const {
        if constexpr (W_BT) w_tmem_wait(v);
    }
    __device__ __forceinline__ void bst4(u32 c, u32 a, u32 b, u32 d, u32 e) const {
        if constexpr (W_BT) {
            w_tmem_st4(tb(bs + c), a, b, d, e);
        } else {
            bres[(size_t)c * bstr] = a;
            bres[(size_t)(c + 1) * bstr] = b;
            bres[(size_t)(c + 2) * bstr] = d;
            bres[(size_t)(c + 3) * bstr] = e;
        }
    }
    // M = 64 tiles: the accumulator rows of message m sit in lane 32q + (m % 16) of quadrant q, so the upper 16 lanes of a
    // warp load nothing useful; they take their partner's values and shadow its work (identical stores, no divergence)
    template <int N>
    __device__ __forceinline__ void dshare(u32 (&v)[N]) const {
        if constexpr (W_M == 64) {
#pragma unroll
            for (int i = 0; i < N; i++) v[i] = __shfl_sync(0xFFFFFFFFu, v[i], threadIdx.x & 15);
        }
    }
    __device__ bool mine16(u32 g) const { return W_HV == 1 || (g & 1u) == h; }   // 16-word / 16-channel group g
    static constexpr u32 GW = (K + 16) / 16;                               // 16-word groups covering words 0 .. K+1
    // both halves of the tile: TMEM stores done, shared / global writes visible
    __device__ void sync() const {
        w_tmem_wait_st();
        if (W_HV == 1) return;
        asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
        asm volatile("bar.sync %0, %1;" ::"r"(bar_id), "r"(128 * W_HV) : "memory");
        asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    }
    // 16 B columns 16g.. of the tile (the last group stops at W_BSW: the next columns are the other tile's)
    __device__ void st_b16(u32 g, const u32 (&v)[16]) const {
        if constexpr (!W_BT) {
#pragma unroll
            for (int q = 0; q < 4; q++) bst4(16 * g + 4 * q, v[4 * q], v[4 * q + 1], v[4 * q + 2], v[4 * q + 3]);
            return;
        }
        if (16 * g + 16 <= W_BSW) {
            w_tmem_st16(tb(bs + 16 * g), v);
        } else {
#pragma unroll
            for (int q = 0; q < 4; q++)
                if (16 * g + 4 * q < W_BSW) w_tmem_st4(tb(bs + 16 * g + 4 * q), v[4 * q], v[4 * q + 1], v[4 * q + 2], v[4 * q + 3]);
        }
    }
    __device__ void a_done() {
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");   // generic-proxy A writes -> async proxy (MMA)
        if (!W_PAIR || T.rank == 0) {
            w_mbar_arrive(T.aready());
        } else {                                                       // one arrival per warp on the leader's barrier
            __syncwarp();
            if (lane0()) w_mbar_arrive_cl(w_lead(T.aready()));
        }
        trace(0x0F);
    }
    // the accumulator buffer is read (one arrival per warp; pair: on the leader's barrier)
    __device__ void acc_free() const {
        asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
        __syncwarp();
        if (lane0()) {
            if (!W_PAIR || T.rank == 0) w_mbar_arrive(T.acce());
            else w_mbar_arrive_cl(w_lead(T.acce()));
        }
    }
    // Chunks of extension E: wait for the accumulator, combine the four byte columns of every output of this half's
    // groups into V (64-bit registers), release the buffer at once (the next chunk's MMAs run under the rest of the
    // epilogue), then f(o0, n4, Vl, Vh): group g = W_HV gi + h of the chunk has outputs o0 + 4g .. +3, V = Vh 2^32 + Vl
    // at [4 gi ..].
    template <u32 E>
    __host__ __device__ static constexpr u32 nloc() { return (tcw_oc(K, E) / 4 + W_HV - 1) / W_HV; }
    template <u32 E, class F>
    __device__ void chunks(F &&f) {
        constexpr u32 OC = tcw_oc(K, E), LG = nloc<E>();
#pragma unroll 1
        for (u32 c = 0; c < tcw_nchunks(K, E); c++) {
            w_mbar_wait(T.accf(), fph);
            fph ^= 1u;
            trace((E << 4) | 1);
            asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
            const u32 n4 = (w_outn(E, c) + 3) / 4;
            u32 Vl[4 * LG], Vh[4 * LG];
            {
#pragma unroll
                for (u32 gi = 0; gi < LG; gi += 2) {
                    const u32 g0 = W_HV * gi + h, g1 = W_HV * (gi + 1) + h;
                    if (g0 < n4) {
                        u32 v[16], w[16];
                        w_tmem_ld16(tb(T.tacc + 16 * g0), v);
                        if (gi + 1 < LG && g1 < n4) w_tmem_ld16(tb(T.tacc + 16 * g1), w);
                        w_tmem_wait(v);
                        if (gi + 1 < LG && g1 < n4) w_tmem_wait(w);
                        dshare(v);
                        if (gi + 1 < LG && g1 < n4) dshare(w);
#pragma unroll
                        for (int t = 0; t < 4; t++) {
                            tc_split(v[4 * t], v[4 * t + 1], v[4 * t + 2], v[4 * t + 3], Vl[4 * gi + t], Vh[4 * gi + t]);
                            if (gi + 1 < LG)
                                tc_split(w[4 * t], w[4 * t + 1], w[4 * t + 2], w[4 * t + 3], Vl[4 * gi + 4 + t], Vh[4 * gi + 4 + t]);
                        }
                    }
                }
            }
            acc_free();
            trace((E << 4) | 2);
            f(c * OC, n4, Vl, Vh);
            trace((E << 4) | 3);
        }
    }

    // a2: positional -> RNS of nl limbs at x (masked to zero when !ok); B -> TMEM, B' -> the A row (parked in the
    // window table's spare slot `park` while the chunks still read the limbs), m_r = x_0 -> word k+1
    __device__ void to_rns(const u32 *x, u32 nl, bool ok, u32 *park, size_t tstride) {
        const bool vec = (nl & 3u) == 0 && (reinterpret_cast<uintptr_t>(x) & 15u) == 0;   // row of whole uint4 groups
#pragma unroll 1
        for (u32 w = 0; w < W_KC; w++) {
            if (!mine16(w / 4)) continue;
            if (MR_TCW_VEC && vec) {                  // whole 16-byte limb groups: one vector load each
                ac(w) = (ok && 4 * w < nl) ? __ldg(reinterpret_cast<const uint4 *>(x) + w) : make_uint4(0u, 0u, 0u, 0u);
                continue;
            }
            u32 q[4];
#pragma unroll
            for (int t = 0; t < 4; t++) q[t] = (ok && 4 * w + t < nl) ? __ldg(x + 4 * w + t) : 0u;
            ac(w) = make_uint4(q[0], q[1], q[2], q[3]);
        }
        const u32 x0 = ok ? __ldg(x) : 0u;
        a_done();
        constexpr u32 LG = nloc<TCW_TRN>();
        chunks<TCW_TRN>([&](u32 o0, u32 n4, const u32 (&Vl)[4 * LG], const u32 (&Vh)[4 * LG]) {
#pragma unroll
            for (u32 gi = 0; gi < LG; gi++) {
                const u32 g = W_HV * gi + h;
                if (g < n4) {
                    const u32 o = o0 + 4 * g;
                    u32 r[4];
#pragma unroll
                    for (int t = 0; t < 4; t++) {
                        const u32 ch = o + t;
                        const u32 j = ch - K < K ? ch - K : 0u;
                        const uint2 mm = ch < K ? ep2[ch] : make_uint2(ep1[j].x, ep1[j].y);
                        r[t] = mont_red(Vl[4 * gi + t], Vh[4 * gi + t], mm.x, mm.y);
                        if (ch >= K && ch < 2 * K) park[(size_t)(ch - K) * tstride] = r[t];
                    }
                    if (o < K) bst4(o, r[0], r[1], r[2], r[3]);   // straddling group: B' lanes -> padding
                }
            }
        });
        sync();                                           // both halves' parked B' outputs and B residues written
#pragma unroll 4
        for (u32 w = 0; w < W_KC; w++) {
            if (!mine16(w / 4)) continue;
            u32 q[4];
#pragma unroll
            for (int t = 0; t < 4; t++) {
                const u32 j = 4 * w + t;
                q[t] = j < K ? park[(size_t)j * tstride] : (j == K + 1 ? x0 : 0u);
            }
            ac(w) = make_uint4(q[0], q[1], q[2], q[3]);
        }
    }

    // 6.1 / 6.2 for channels c0 .. c0 + N - 1 (N <= 16, c0 a multiple of 8): ξ_i = mont(mont(a_i b_i) σ_i 2^64) (B, into
    // the A row over the B' words it consumed) and t*_j = mont(a*_j b*_j) (B', into the TMEM columns of the B residues
    // it consumed)
    template <bool SQ, u32 N>
    __device__ __forceinline__ void chan_group(u32 c0, const u32 *bp, u32 bs_, const u32 *sg) {
        constexpr u32 NW = N > 8 ? 16 : 8;
        const uint2 *e2 = ep2 + c0;
        const uint4 *e1 = ep1 + c0;
        const u32 *sgg = sg + c0;
        u32 r[NW], xa[NW], b1[N], b2[N];
        bld(c0, r);
#pragma unroll
        for (u32 q = 0; q < (N + 3) / 4; q++) {
            const uint4 v = ac(c0 / 4 + q);
            xa[4 * q] = v.x; xa[4 * q + 1] = v.y; xa[4 * q + 2] = v.z; xa[4 * q + 3] = v.w;
        }
        if (!SQ) {
            const u32 *b = bp + (size_t)c0 * bs_;
#pragma unroll
            for (u32 t = 0; t < N; t++) {
                b1[t] = __ldcg(b + (size_t)t * bs_);
                b2[t] = __ldcg(b + (size_t)(K + t) * bs_);
            }
        }
        bwait(r);
        u32 xi[NW], ts[NW];
#pragma unroll
        for (u32 t = 0; t < NW; t++) xi[t] = ts[t] = 0u;
#pragma unroll
        for (u32 t = 0; t < N; t++) {
            const uint2 mm = e2[t];
            const u64 pr = mulw(r[t], SQ ? r[t] : b1[t]);
            const u32 tt = mont_red((u32)pr, (u32)(pr >> 32), mm.x, mm.y);
            const u64 ps = mulw(tt, sgg[t]);
            xi[t] = mont_red((u32)ps, (u32)(ps >> 32), mm.x, mm.y);
            const uint4 c1 = e1[t];
            const u64 pp = mulw(xa[t], SQ ? xa[t] : b2[t]);
            ts[t] = mont_red((u32)pp, (u32)(pp >> 32), c1.x, c1.y);
        }
#pragma unroll
        for (u32 q = 0; q < (N + 3) / 4; q++) bst4(c0 + 4 * q, ts[4 * q], ts[4 * q + 1], ts[4 * q + 2], ts[4 * q + 3]);
#pragma unroll
        for (u32 q = 0; q < (N + 3) / 4; q++) ac(c0 / 4 + q) = make_uint4(xi[4 * q], xi[4 * q + 1], xi[4 * q + 2], xi[4 * q + 3]);
    }

    // 6.1 / 6.2 over the full 16-channel groups with the TMEM and A-row loads of group g+1 issued under the products of
    // group g (one warp per lane quadrant: W_HV = 1)
    template <bool SQ>
    __device__ __forceinline__ void chan_pipe(const u32 *bp, u32 bs_, const u32 *sg) {
        u32 r[16], xa[16];
        auto load_xa = [&](u32 g) {
#pragma unroll
            for (u32 q = 0; q < 4; q++) {
                const uint4 v = ac(4 * g + q);
                xa[4 * q] = v.x; xa[4 * q + 1] = v.y; xa[4 * q + 2] = v.z; xa[4 * q + 3] = v.w;
            }
        };
        w_tmem_ld16(tb(bs), r);
        load_xa(0);
#pragma unroll 1
        for (u32 g = 0; g < K / 16; g++) {
            w_tmem_wait(r);
            u32 u[16], v[16];                        // this group's B residues and B' words (then ξ, t*)
#pragma unroll
            for (u32 t = 0; t < 16; t++) { u[t] = r[t]; v[t] = xa[t]; }
            u32 b1[16], b2[16];
            if (!SQ) {
                const u32 *b = bp + (size_t)(16 * g) * bs_;
#pragma unroll
                for (u32 t = 0; t < 16; t++) {
                    b1[t] = __ldcg(b + (size_t)t * bs_);
                    b2[t] = __ldcg(b + (size_t)(K + t) * bs_);
                }
            }
            if (g + 1 < K / 16) {                    // next group's operands in flight
                w_tmem_ld16(tb(bs + 16 * (g + 1)), r);
                load_xa(g + 1);
            }
            const uint2 *e2 = ep2 + 16 * g;
            const uint4 *e1 = ep1 + 16 * g;
            const u32 *sgg = sg + 16 * g;
#pragma unroll
            for (u32 t = 0; t < 16; t++) {
                const uint2 mm = e2[t];
                const u64 pr = mulw(u[t], SQ ? u[t] : b1[t]);
                const u32 tt = mont_red((u32)pr, (u32)(pr >> 32), mm.x, mm.y);
                const u64 ps = mulw(tt, sgg[t]);
                u[t] = mont_red((u32)ps, (u32)(ps >> 32), mm.x, mm.y);            // ξ_i
                const uint4 c1 = e1[t];
                const u64 pp = mulw(v[t], SQ ? v[t] : b2[t]);
                v[t] = mont_red((u32)pp, (u32)(pp >> 32), c1.x, c1.y);            // t*_j
            }
            w_tmem_st16(tb(bs + 16 * g), v);
#pragma unroll
            for (u32 q = 0; q < 4; q++) ac(4 * g + q) = make_uint4(u[4 * q], u[4 * q + 1], u[4 * q + 2], u[4 * q + 3]);
        }
    }

    // α' and r_r from both halves' partial sums (Σ ξ'_j |M'_j|_{2^32} over each half's outputs; r_r from its owner)
    __device__ uint2 exchange(u32 sr, u32 rr) {
        if (W_HV == 1) { sync(); return make_uint2(sr, rr); }
        xch[h * 128 + m] = make_uint2(sr, rr);
        sync();
        const uint2 o = xch[(h ^ 1u) * 128 + m];
        return make_uint2(sr + o.x, rr + o.y);
    }

    // 6.1-6.6: st <- st · b · M^-1 (mod N); b at bp[c · bs_] (window table column or constant vector), or st (SQ)
    template <bool SQ>
    __device__ void mont_mul(const u32 *bp, u32 bs_) {
        trace(0x0E);
        const u32 *sg = sig + sel * K;
        u32 br = 0;
        const u32 ar = aw(K + 1);
        if (!SQ) br = __ldcg(bp + (size_t)(2 * K) * bs_);
        // ---- 6.1 / 6.2: this half's 16-channel groups
        if (W_HV == 1 && MR_TCW_CHAN_PIPE) {
            chan_pipe<SQ>(bp, bs_, sg);
        } else {
#pragma unroll 1
            for (u32 g = h; g < K / 16; g += W_HV) {
                if (W_HV == 1) {
                    chan_group<SQ, 16>(16 * g, bp, bs_, sg);
                } else {
                    chan_group<SQ, 8>(16 * g, bp, bs_, sg);
                    chan_group<SQ, 8>(16 * g + 8, bp, bs_, sg);
                }
            }
        }
        static_assert(K % 16 <= 8 || !W_BT, "tail channels fit one 8-channel group (TMEM columns of the tile)");
        if (K % 16 && mine16(K / 16)) chan_group<SQ, K % 16>(16 * (K / 16), bp, bs_, sg);
        const u32 trm = ar * (SQ ? ar : br);
        w_tmem_wait_st();
        if constexpr (!W_BT) sync();   // t*_j (global) of both halves written before either half's BE1 epilogue
        a_done();
        // ---- 6.3-6.5 BE1 epilogue: ξ'_j = mont(t*_j C1_j 2^64 + D_j) over t*_j in TMEM; m_r column -> r_r
        u32 sr = 0, rr = 0;
        const u32 nminv = cx[CX_NMINV_R];
        constexpr u32 LG1 = nloc<TCW_BE1>();
        chunks<TCW_BE1>([&](u32 o0, u32 n4, const u32 (&Vl)[4 * LG1], const u32 (&Vh)[4 * LG1]) {
#pragma unroll
            for (u32 gi = 0; gi < LG1; gi += 2) {
                const u32 g0 = W_HV * gi + h, g1 = g0 + W_HV;
                if (g0 < n4) {
                    const u32 oa = o0 + 4 * g0, ob = o0 + 4 * g1;
                    u32 ta[4], tc[4];
                    bld(oa < K ? oa : 0, ta);
                    if (gi + 1 < LG1 && g1 < n4) bld(ob < K ? ob : 0, tc);
                    bwait(ta);
                    if (gi + 1 < LG1 && g1 < n4) bwait(tc);
#pragma unroll
                    for (u32 u = 0; u < 2; u++) {
                        if (gi + u < LG1 && (u == 0 || g1 < n4)) {
                            const u32 oh = u ? ob : oa;
                            u32 xp[4];
#pragma unroll
                            for (int t = 0; t < 4; t++) {
                                const u32 j = oh + t, q = 4 * (gi + u) + t;
                                const uint4 e1 = ep1[j < K ? j : 0];
                                // ξ'_j = mont(t*_j C1_j 2^64 + V_j): t* < 2^32 and V <= 4k 255^2 (1 + 2^8 + 2^16 + 2^24)
                                // < 2^50.1, and every per-k constant C1_j 2^64 mod m'_j is below 0.9985 2^32, so the sum
                                // fits 64 bits (pinned per k by test_tcw_host.py::test_be1_epilogue_sum_fits_64_bits)
                                const u64 p = madw(u ? tc[t] : ta[t], e1.z, ((u64)Vh[q] << 32) | Vl[q]);
                                xp[t] = mont_red((u32)p, (u32)(p >> 32), e1.x, e1.y);
                                if (j < K) sr += MR_TCW_FRAC ? xp[t] >> W_FSH : xp[t] * e1.w;
                                if (!MR_TCW_FRAC && j == K) rr = trm * minv_r + Vl[q] * nminv;   // q̂_r = Σ ξ_i |M_i|_{2^32}
                            }
                            if (oh < K) bst4(oh, xp[0], xp[1], xp[2], xp[3]);   // ξ'_j in place of t*_j
                        }
                    }
                }
            }
        });
        // ---- 6.6 BE2: A row = (ξ'_0 .. ξ'_{k-1}, α', r_r), α' = (Σ ξ'_j |M'_j|_{2^32} - r_r) M'^-1 exact
        const uint2 tot = exchange(sr, rr);              // (also: every ξ'_j of both halves is in TMEM)
        const u32 alpha = MR_TCW_FRAC ? w_frac_alpha(tot.x) : (tot.x - tot.y) * mpinv_r;
        rr = tot.y;
#pragma unroll 1
        for (u32 g = h; g < GW; g += W_HV) {
            u32 v[16];
            bld(16 * g, v);
            bwait(v);
#pragma unroll
            for (int q = 0; q < 4; q++) {
                if (4 * g + q < W_KC) {
                    u32 w4[4];
#pragma unroll
                    for (int t = 0; t < 4; t++) {
                        const u32 j = 16 * g + 4 * q + t;
                        w4[t] = j < K ? v[4 * q + t] : (j == K ? alpha : (j == K + 1 ? rr : 0u));
                    }
                    ac(4 * g + q) = make_uint4(w4[0], w4[1], w4[2], w4[3]);
                }
            }
        }
        a_done();
        constexpr u32 LG2 = nloc<TCW_BE2>();
        chunks<TCW_BE2>([&](u32 o0, u32 n4, const u32 (&Vl)[4 * LG2], const u32 (&Vh)[4 * LG2]) {
#pragma unroll
            for (u32 gi = 0; gi < LG2; gi++) {
                const u32 g = W_HV * gi + h;
                if (g < n4) {
                    const u32 o = o0 + 4 * g;
                    u32 r[4];
#pragma unroll
                    for (int t = 0; t < 4; t++) {
                        const uint2 mm = ep2[o + t < K ? o + t : K - 1];
                        r[t] = mont_red(Vl[4 * gi + t], Vh[4 * gi + t], mm.x, mm.y);
                    }
                    bst4(o, r[0], r[1], r[2], r[3]);
                }
            }
        });
        sync();                                           // every r_i in TMEM before the next multiplication reads them
    }

    // a7: X = Σ ξ'_j M'_j + α'(2^(32(K+1)) - M') on the tensor core (byte convolution); half 0 carries the limbs (parked
    // in the TMEM B columns, then A row words 0..K) and reduces X mod N by conditional subtraction of N 2^s,
    // s = SMAX..0 (X < (K+3) N); returns with the limbs in the A row of half 0's thread
    __device__ void from_rns() {
        u32 sr = 0;
#pragma unroll 1
        for (u32 g = h; g < GW; g += W_HV) {
#pragma unroll
            for (u32 t = 0; t < 16; t++)
                if (16 * g + t < K) sr += MR_TCW_FRAC ? aw(16 * g + t) >> W_FSH : aw(16 * g + t) * ep1[16 * g + t].w;
        }
        const uint2 tot = exchange(sr, 0u);
        if (mine16(K / 16)) aw(K) = MR_TCW_FRAC ? w_frac_alpha(tot.x) : (tot.x - aw(K + 1)) * mpinv_r;
        a_done();
        // half 0 carries the byte-position sums into limbs group by group (the buffer is released after the chunk)
        u64 carry = 0;
#pragma unroll 1
        for (u32 c = 0; c < tcw_nchunks(K, TCW_EXT); c++) {
            w_mbar_wait(T.accf(), fph);
            fph ^= 1u;
            asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
            if (h == 0) {
                const u32 n4 = (w_outn(TCW_EXT, c) + 3) / 4, o0 = c * tcw_oc(K, TCW_EXT);
#pragma unroll 1
                for (u32 g = 0; g < n4; g++) {
                    u32 v[16];
                    w_tmem_ld16(tb(T.tacc + 16 * g), v);
                    w_tmem_wait(v);
                    dshare(v);
                    u32 l4[4];
#pragma unroll
                    for (int t = 0; t < 4; t++) {
                        const u64 s = carry + tc_comb(v[4 * t], v[4 * t + 1], v[4 * t + 2], v[4 * t + 3]);
                        l4[t] = (u32)s;
                        carry = s >> 32;
                    }
                    bst4(o0 + 4 * g, l4[0], l4[1], l4[2], l4[3]);   // limbs (columns < round4(K+1))
                }
            }
            acc_free();
        }
        if (h) return;
        w_tmem_wait_st();
#pragma unroll 1
        for (u32 g = 0; g < GW; g++) {
            u32 v[16];
            bld(16 * g, v);
            bwait(v);
#pragma unroll
            for (int q = 0; q < 4; q++)
                if (4 * g + q < W_KC) ac(4 * g + q) = make_uint4(v[4 * q], v[4 * q + 1], v[4 * q + 2], v[4 * q + 3]);
        }
        const u32 *nl = cx + cx_n(K);
#pragma unroll 1
        for (int s = SMAX; s >= 0; s--) {
            if (MR_TCW_CMPTOP) {   // X >= N 2^s ? from the most significant limb down: the first difference decides
                int cmp = 0;
#pragma unroll 1
                for (int l = K; l >= 0 && cmp == 0; l--) {
                    const u32 nsh = __funnelshift_l(l ? __ldg(nl + l - 1) : 0u, __ldg(nl + l), s), xv = aw(l);
                    cmp = xv > nsh ? 1 : (xv < nsh ? -1 : 0);
                }
                if (cmp < 0) continue;
                u32 brw = 0;
#pragma unroll 4
                for (u32 l = 0; l <= K; l++) {
                    const u32 nsh = __funnelshift_l(l ? __ldg(nl + l - 1) : 0u, __ldg(nl + l), s);
                    const u64 t = (u64)aw(l) - nsh - brw;
                    aw(l) = (u32)t;
                    brw = (u32)(t >> 63);
                }
                continue;
            }
#pragma unroll 1
            for (int pass = 0; pass < 2; pass++) {   // pass 0: borrow of X - N 2^s; pass 1: subtract
                u32 brw = 0;
#pragma unroll 4
                for (u32 l = 0; l <= K; l++) {
                    const u32 nsh = __funnelshift_l(l ? __ldg(nl + l - 1) : 0u, __ldg(nl + l), s);
                    const u64 t = (u64)aw(l) - nsh - brw;
                    if (pass) aw(l) = (u32)t;
                    brw = (u32)(t >> 63);
                }
                if (brw) break;
            }
        }
    }

    // the op program of one 128-message job (same ops as run_program in mr_kernels.cuh)
    __device__ void job(const ModexpParams &P, u32 jl, bool valid) {
        const u32 *xrow = P.x + (size_t)(valid ? jl : 0) * P.in_limbs;
        const bool ok = valid && less_than(xrow, cx + cx_inb(K), P.in_limbs);
        if (valid && h == 0 && sel == 0 && P.status) P.status[jl] = ok ? 0 : 5 /* MR_ERR_RANGE */;
        const size_t tstride = P.jobs_total, entry = (size_t)NCH * tstride;
        const u32 col = sel * P.ctas0 * W_M + jl;     // window-table column (tail lanes too: jl < ctas0 * W_M)
        if constexpr (!W_BT) {                         // B residues: the slot after to_rns's parking slot
            bres = P.table + (size_t)(P.hslot + 1) * entry + col;
            bstr = tstride;
        }
        const u64 *prog = sel ? P.prog[1] : P.prog[0];
        const u32 nops = sel ? P.nops[1] : P.nops[0];
        u64 nop = __ldg(prog);
#pragma unroll 1
        for (u32 s = 0; s < nops; s++) {
            const u64 op = nop;
            if (s + 1 < nops) nop = __ldg(prog + s + 1);   // next op under this one (the program lives in L2)
            const u32 fl = (u32)op & 0xFF, opnd = (u32)(op >> 8) & 0xFF, ld = (u32)(op >> 16) & 0xFF;
            const u32 ad = (u32)(op >> 24) & 0xFF, sto = (u32)(op >> 32) & 0xFF;
            if (fl & (OPF_TORNS_ALL | OPF_TORNS_LO | OPF_TORNS_HI)) {
                const u32 off = (fl & OPF_TORNS_HI) ? P.half : 0u;
                to_rns(xrow + off, (fl & OPF_TORNS_ALL) ? P.in_limbs : P.half, ok, P.table + P.hslot * entry + col,
                       tstride);
            }
            if (fl & OPF_LOAD) {
                const u32 *src;
                size_t str;
                if (ld >= 0xF0) { src = cx + cx_r2(K) + (ld - 0xF0) * NCH; str = 1; }
                else { src = P.table + ld * entry + col; str = tstride; }
#pragma unroll 1
                for (u32 g = h; g < GW; g += W_HV) {
#pragma unroll
                    for (u32 q = 0; q < 4; q++) {
                        const u32 w = 4 * g + q;
                        if (w < (W_BT ? W_BSW : (K + 3) & ~3u) / 4) {   // B residues: TMEM columns / global rows
                            u32 b4[4];
#pragma unroll
                            for (int t = 0; t < 4; t++) b4[t] = 4 * w + t < K ? src[(4 * w + t) * str] : 0u;
                            bst4(4 * w, b4[0], b4[1], b4[2], b4[3]);
                        }
                        if (w < W_KC) {
                            u32 a4[4];
#pragma unroll
                            for (int t = 0; t < 4; t++) {
                                const u32 j = 4 * w + t;
                                a4[t] = j < K ? src[(K + j) * str] : (j == K + 1 ? src[2 * K * str] : 0u);
                            }
                            ac(w) = make_uint4(a4[0], a4[1], a4[2], a4[3]);
                        }
                    }
                }
                w_tmem_wait_st();
            }
            if (!(fl & OPF_NOMUL)) {
                if (opnd == OPND_SQ) mont_mul<true>(nullptr, 0);
                else if (opnd >= 0xF0) mont_mul<false>(cx + cx_r2(K) + (opnd - 0xF0) * NCH, 1);
                else mont_mul<false>(P.table + opnd * entry + col, (u32)tstride);
            }
            if (fl & OPF_ADD) {   // channel-wise modular addition (CRT entry, a3)
                const u32 *src = P.table + ad * entry + col;
#pragma unroll 1
                for (u32 g = h; g < GW; g += W_HV) {
                    u32 a[16];
                    bld(16 * g, a);
                    bwait(a);
#pragma unroll
                    for (int t = 0; t < 16; t++) {
                        const u32 i = 16 * g + t;
                        if (i < K) a[t] = w_addmod(a[t], src[i * tstride], 0u - ep2[i].x);
                        if (i < K) aw(i) = w_addmod(aw(i), src[(K + i) * tstride], 0u - ep1[i].x);
                        if (i == K + 1) aw(K + 1) += src[2 * K * tstride];
                    }
                    st_b16(g, a);
                }
                w_tmem_wait_st();
            }
            if (fl & OPF_STORE) {
                u32 *dst = P.table + sto * entry + col;
#pragma unroll 1
                for (u32 g = h; g < GW; g += W_HV) {
                    u32 a[16];
                    bld(16 * g, a);
                    bwait(a);
#pragma unroll
                    for (int t = 0; t < 16; t++) {
                        const u32 i = 16 * g + t;
                        if (i < K) dst[i * tstride] = a[t];
                        if (i < K) dst[(K + i) * tstride] = aw(i);
                        if (i == K + 1) dst[2 * K * tstride] = aw(K + 1);
                    }
                }
            }
        }
        from_rns();
        if (valid && h == 0) {
            u32 *yrow = P.y + sel * P.out_stride + (size_t)jl * P.out_limbs;
#pragma unroll 1
            if (MR_TCW_VEC && (P.out_limbs & 3u) == 0 && (reinterpret_cast<uintptr_t>(yrow) & 15u) == 0) {
#pragma unroll 1
                for (u32 w = 0; w < P.out_limbs / 4; w++)   // the A row's K-core w holds limbs 4w .. 4w+3
                    reinterpret_cast<uint4 *>(yrow)[w] = ok ? ac(w) : make_uint4(0u, 0u, 0u, 0u);
            } else {
                for (u32 l = 0; l < P.out_limbs; l++) yrow[l] = ok ? aw(l) : 0u;
            }
        }
        sync();                                           // the A row is free for the next job
    }
};

// Persistent kernel, one CTA per SM, W_TILES independent tiles per CTA: tile u of CTA b takes the tile-jobs
// t = b·TILES + u, + gridDim.x·TILES, ...; job t runs context sel = t / ctas0.  The producer, the MMA issuer and
// the compute warps of a tile walk the same job list and op programs, so they meet on the same sequence of
// (extension, chunk, slab).
__global__ void __launch_bounds__(W_THREADS, 1) k_modexp_tcw(const ModexpParams P, const TcwArgs A) {
    extern __shared__ __align__(1024) uint8_t wsm[];
    __shared__ u32 tslot;
    const u32 tid = threadIdx.x, warp = tid / 32;
    u32 rank = 0;                                     // pair mode: CTA rank in the 2-CTA cluster
    if constexpr (W_PAIR) asm("mov.u32 %0, %%cluster_ctarank;" : "=r"(rank));
    uint8_t *stages = wsm + (size_t)W_TILES * W_ABYTES;
    uint4 *ep1 = reinterpret_cast<uint4 *>(stages + (size_t)W_RINGS * W_NST * W_STG);
    uint2 *ep2 = reinterpret_cast<uint2 *>(ep1 + K);
    u32 *sig = reinterpret_cast<u32 *>(ep2 + K);
    u64 *bars = reinterpret_cast<u64 *>(((uintptr_t)(sig + 2 * K) + 7) & ~(uintptr_t)7);
    // role: compute warps 0 .. W_CW-1 (tile = warp / (4 W_HV), half = (warp / 4) % W_HV; the warp's TMEM lane quadrant
    // is warp % 4), then per tile a producer warp and an MMA warp (lane 0 works; pair mode: rank 1's MMA warp relays)
    const u32 tile = warp < W_CW ? warp / (4 * W_HV) : (warp - W_CW) % W_TILES;
    TcwTile T;
    const u32 ring = TCW_LOCK ? 0u : tile;
    T.a = wsm + (size_t)tile * W_ABYTES;
    T.stage0 = smem_u32(stages + (size_t)ring * W_NST * W_STG);
    T.bar = smem_u32(bars + ring * W_NBAR);
    T.tacc = tile * W_TCOLS;
    T.rank = rank;
    const WideLayout WL = wide_layout(K);
    for (u32 j = tid; j < K; j += W_THREADS) {
        ep1[j] = make_uint4(__ldg(A.wtab + WL.mm + K + j), __ldg(A.wtab + WL.minv + K + j), __ldg(A.wtab + WL.xw + j),
                            __ldg(A.wtab + WL.a2r + j));
        ep2[j] = make_uint2(__ldg(A.wtab + WL.mm + j), __ldg(A.wtab + WL.minv + j));
        sig[j] = __ldg(P.ctx[0] + A.cxw + wide_cx_sig(K) + j);
        sig[K + j] = __ldg(P.ctx[1] + A.cxw + wide_cx_sig(K) + j);
    }
    if (tid < W_RINGS) {
        TcwTile U;
        U.bar = smem_u32(bars + tid * W_NBAR);
        const bool lead = W_PAIR && rank == 0;        // the leader's barriers also count the peer's arrivals
        for (u32 s = 0; s < W_NST; s++) {
            w_mbar_init(U.full(s), lead ? 2 : 1);     // pair leader: own expect_tx + the peer's relay
            w_mbar_init(U.empty(s), 1);
        }
        w_mbar_init(U.accf(), 1);
        w_mbar_init(U.acce(), 4 * W_HV * W_SUB + (lead ? 4 * W_HV : 0));
        w_mbar_init(U.aready(), 128 * W_HV * W_SUB + (lead ? 4 * W_HV : 0));
    }
    if (warp == 0) {
        if constexpr (W_PAIR) {
            asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(&tslot)), "r"(512));
            asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;");
        } else {
            asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(&tslot)), "r"(512));
            asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
        }
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    if constexpr (W_PAIR)   // both CTAs' barriers initialised before any remote arrival
        asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    const u32 tmem = tslot;
    // independent tiles: tile u of CTA b walks jobs b TILES + u + i gridDim.x TILES; lockstep: the producer and the
    // MMA issuer walk the job PAIRS (jobs 2p, 2p + 1 share a context: the host pads ctas0 to even) and tile u takes 2p + u;
    // CTA pairs: tile u of cluster c walks the pair-jobs q = c TILES + u + i (clusters) TILES and CTA r takes job 2q + r
    // (the two jobs of a pair share a context: the host pads ctas0 to even)
    const u32 cl = W_PAIR ? blockIdx.x / 2 : blockIdx.x, ncl = W_PAIR ? gridDim.x / 2 : gridDim.x;
    const u32 J = W_PAIR ? A.jobs / 2 : A.jobs, stride = ncl * W_TILES;
    const u32 first = cl * W_TILES + tile;
    auto job_of = [&](u32 q) { return W_PAIR ? 2 * q + rank : q; };
    const bool role_on = !TCW_LOCK || tile == 0 || warp < W_CW;   // lockstep: tile 1's producer / MMA warps idle

    if (warp >= W_CW && warp < W_CW + W_TILES) {    // ---- producer of `tile`
        if ((tid & 31) == 0 && role_on) {
            TcwProducer pr;
            asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(pr.pol));
            pr.tr.init(A.trace, tile, 2);
#pragma unroll 1
            for (u32 q = first; q < J; q += stride) {
                const u32 t = job_of(q);
                const u32 sel = t / P.ctas0;
                const uint8_t *be1 = reinterpret_cast<const uint8_t *>((sel ? P.ctx[1] : P.ctx[0]) + A.be1w);
                const u64 *prog = sel ? P.prog[1] : P.prog[0];
                const u32 nops = sel ? P.nops[1] : P.nops[0];
#pragma unroll 1
                for (u32 s = 0; s < nops; s++) {
                    const u32 fl = (u32)__ldg(prog + s) & 0xFF;
                    if (fl & (OPF_TORNS_ALL | OPF_TORNS_LO | OPF_TORNS_HI)) pr.ext(T, TCW_TRN, A.kimg + tcw_img_off(K, TCW_TRN));
                    if (!(fl & OPF_NOMUL)) {
                        pr.ext(T, TCW_BE1, be1);
                        pr.ext(T, TCW_BE2, A.kimg + tcw_img_off(K, TCW_BE2));
                    }
                }
                pr.ext(T, TCW_EXT, A.kimg + tcw_img_off(K, TCW_EXT));
            }
        }
    } else if (warp >= W_CW + W_TILES) {            // ---- MMA issuer of `tile` (pair mode, rank 1: relay)
        if ((tid & 31) == 0 && role_on) {
            TcwMma mm;
            mm.tmem = tmem;
            mm.sa1 = smem_u32(wsm + W_ABYTES);
            mm.td1 = tmem + W_TCOLS;
            mm.tr.init(A.trace, tile, 1);
#pragma unroll 1
            for (u32 q = first; q < J; q += stride) {
                const u32 sel = job_of(q) / P.ctas0;
                const u64 *prog = sel ? P.prog[1] : P.prog[0];
                const u32 nops = sel ? P.nops[1] : P.nops[0];
                auto ext = [&](u32 e) {
                    if (W_PAIR && rank) mm.relay(T, e);
                    else mm.ext(T, e);
                };
#pragma unroll 1
                for (u32 s = 0; s < nops; s++) {
                    const u32 fl = (u32)__ldg(prog + s) & 0xFF;
                    if (fl & (OPF_TORNS_ALL | OPF_TORNS_LO | OPF_TORNS_HI)) ext(TCW_TRN);
                    if (!(fl & OPF_NOMUL)) {
                        ext(TCW_BE1);
                        ext(TCW_BE2);
                    }
                }
                ext(TCW_EXT);
            }
        }
    } else {                                          // ---- compute warps of `tile`
        const u32 m = (warp % 4) * (W_M / 4) + (tid & 31) % (W_M / 4), h = (warp / 4) % W_HV;   // M = 64: lanes 16..31
                                                                                               // shadow lanes 0..15
        uint2 *xch = reinterpret_cast<uint2 *>(bars + W_TILES * W_NBAR) + tile * 256;
        TcwCompute cw{T, ep1, ep2, sig, tmem + ((warp % 4) * 32u << 16), T.tacc + W_NCMAX, m, h,
                      T.a + (m / 8) * W_SBOA + (m % 8) * 16, xch, 1 + tile};
        cw.tr.init(A.trace, tile, 0);
        cw.minv_r = __ldg(A.wtab + WL.misc);
        cw.mpinv_r = __ldg(A.wtab + WL.misc + 1);
#pragma unroll 1
        for (u32 q = first; q < J; q += stride) {
            const u32 t = job_of(q);
            cw.sel = t / P.ctas0;
            cw.cx = cw.sel ? P.ctx[1] : P.ctx[0];
            const u32 jl = (t - cw.sel * P.ctas0) * W_M + m;
            cw.job(P, jl, jl < P.count);
        }
    }
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    if constexpr (W_PAIR) {   // the peer's MMAs / remote arrivals are done before either CTA frees TMEM or exits
        asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
        if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(512));
    } else {
        if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(512));
    }
}

// host side of one launch (both the per-k TUs and mr_tcw257.cu): shared-memory attribute once per process, 2-CTA
// clusters in pair mode (ctas even)
int tcw_launch(const ModexpParams &p, u32 ctas, const TcwArgs &a, void *stream) {
    static bool attr[64] = {};                        // the attribute is per device: set once on each
    int dev = 0;
    if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= 64) return 6;
    if (!attr[dev]) {
        const cudaError_t e = cudaFuncSetAttribute((const void *)k_modexp_tcw, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                                   (int)W_SMEM);
        if (e != cudaSuccess) {
            if (getenv("MR_RNS_DEBUG")) fprintf(stderr, "k_modexp_tcw<%d> smem %zu: %s\n", K, (size_t)W_SMEM, cudaGetErrorString(e));
            return 6;
        }
        attr[dev] = true;
    }
    TcwArgs aa = a;
    ModexpParams pp = p;
    void *args[] = {&pp, &aa};
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(ctas);
    cfg.blockDim = dim3(W_THREADS);
    cfg.dynamicSmemBytes = W_SMEM;
    cfg.stream = (cudaStream_t)stream;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = W_PAIR ? 2 : 1;
    at[0].val.clusterDim.y = 1;
    at[0].val.clusterDim.z = 1;
    cfg.attrs = at;
    cfg.numAttrs = W_PAIR ? 1 : 0;
    const cudaError_t e = cudaLaunchKernelExC(&cfg, (const void *)k_modexp_tcw, args);
    if (e != cudaSuccess && getenv("MR_RNS_DEBUG")) fprintf(stderr, "k_modexp_tcw<%d> launch: %s\n", K, cudaGetErrorString(e));
    return e == cudaSuccess ? 0 : 6;
}

#endif  // MR_K == 97 || MR_K == 129 || MR_K == 257 || MR_K == 505
