// mr_tcw.cuh — tensor-core modexp for wide operands, k = 97 and 129 (3072- / 4096-bit moduli, CRT halves of
// 6144- / 8192-bit keys): SURVEY §8(f) rows 2-3, DESIGN.md §4k.  Included by mr_kernels.cuh inside its
// per-k anonymous namespace (MR_K = 97 or 129), so K, NCH, SMAX, GB(), mont_red(), less_than() are this TU's.
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
// The B images (16k² bytes per extension: 150 KB at k = 97) exceed shared memory next to a 128-message tile, so a
// producer warp streams them from L2 with the bulk-copy (TMA) engine through a ring of stages, one
// [chunk rows x 128 K-bytes] slab per stage; an MMA warp issues the K-steps of each slab into one of two TMEM
// accumulator buffers; the four compute warps (one message per thread, 128 messages = the 128 TMEM lanes) run the
// channel products and the epilogues, the epilogue of chunk c overlapping the MMAs of chunk c+1.
// State of a message: B residues in TMEM (columns W_BS.., one lane per message), B' and m_r in shared-memory rows,
// the A row (its K-major operand bytes) as scratch for the current contraction's inputs.
#pragma once

#if MR_K == 97 || MR_K == 129

constexpr u32 W_KP = tcw_kp(K);                       // A row bytes
constexpr u32 W_SBOA = (W_KP / 16) * 128;             // A tile: bytes between 8-row groups
constexpr u32 W_NCMAX = tcw_ncmax(K);                 // TMEM columns of one accumulator buffer
constexpr u32 W_BS = 2 * W_NCMAX;                     // first TMEM column of the B residues
static_assert(W_BS + tcw_bsw(K) <= 512, "accumulator buffers + B residues exceed the 512 TMEM columns");
constexpr u32 W_STG = tcw_stage_bytes(K);
constexpr u32 W_ROWS = (K + 1) * 128;                 // B' and m_r rows (words)
constexpr size_t W_FIXED = (size_t)128 * W_KP + 4 * (size_t)W_ROWS + 16 * K + 8 * K + 8 * K + 256;
constexpr u32 W_NST_FIT = (u32)((232448 - W_FIXED) / W_STG);
constexpr u32 W_NST = W_NST_FIT > 8 ? 8 : W_NST_FIT;  // pipeline stages
static_assert(W_NST >= 2, "tensor wide kernel: fewer than two B stages fit shared memory");
constexpr size_t W_SMEM = W_FIXED + (size_t)W_NST * W_STG;
constexpr u32 W_THREADS = 192;                        // warps 0-3 compute, 4 producer (TMA), 5 MMA issuer

struct TcwArgs {
    const u32 *wtab;          // per-k wide table (mr_internal.h wide_layout): m, -m^-1, C1 2^64, |M'_j|_{2^32}
    const uint8_t *kimg;      // per-k images: BE2 | TRN | EXT (tcw_img_off)
    u32 cxw;                  // word offset of the wide section (σ_i 2^64) in a context block
    u32 be1w;                 // word offset of the context's BE1 image in its context block
    u32 jobs;                 // 128-message tile-jobs over all contexts (ctas0 per context)
};

__device__ __forceinline__ u32 smem_u32(const void *p) { return (u32)__cvta_generic_to_shared(p); }
// byte-column combine V = d0 + 2^8 d1 + 2^16 d2 + 2^24 d3 = hi 2^32 + lo for d_b < 2^31 (one carry chain)
__device__ __forceinline__ void tc_split(u32 d0, u32 d1, u32 d2, u32 d3, u32 &lo, u32 &hi) {
    asm("add.cc.u32 %0, %2, %3;\n\taddc.u32 %1, %4, 0;\n\t"
        "add.cc.u32 %0, %0, %5;\n\taddc.u32 %1, %1, %6;\n\t"
        "add.cc.u32 %0, %0, %7;\n\taddc.u32 %1, %1, %8;"
        : "=r"(lo), "=r"(hi)
        : "r"(d0), "r"(d1 << 8), "r"(d1 >> 24), "r"(d2 << 16), "r"(d2 >> 16), "r"(d3 << 24), "r"(d3 >> 8));
}
__device__ __forceinline__ void w_mbar_init(u32 a, u32 n) { asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(a), "r"(n)); }
__device__ __forceinline__ void w_mbar_wait(u32 a, u32 par) {
    u32 done = 0;
#pragma unroll 1
    for (u32 spin = 0; !done; spin++) {
        asm volatile("{\n\t.reg .pred P1;\n\tmbarrier.try_wait.parity.shared::cta.b64 P1, [%1], %2;\n\tselp.u32 %0, 1, 0, P1;\n\t}"
                     : "=r"(done)
                     : "r"(a), "r"(par)
                     : "memory");
        if (spin > (1u << 26)) __trap();   // a lost arrival traps instead of hanging the GPU
    }
}
__device__ __forceinline__ void w_mbar_arrive(u32 a) { asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(a) : "memory"); }
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
__device__ __forceinline__ void w_tmem_ld16(u32 taddr, u32 (&v)[16]) {
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];\n\t"
                 "tcgen05.wait::ld.sync.aligned;"
                 : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]),
                   "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15])
                 : "r"(taddr)
                 : "memory");
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

// the extensions of one program op, in the order every role walks them (TRN, then BE1 + BE2)
__device__ __forceinline__ u32 w_nchunks(u32 e) {
    return e == TCW_BE1 ? tcw_nchunks(K, TCW_BE1) : e == TCW_BE2 ? tcw_nchunks(K, TCW_BE2)
                        : e == TCW_TRN ? tcw_nchunks(K, TCW_TRN) : tcw_nchunks(K, TCW_EXT);
}
__device__ __forceinline__ u32 w_oc(u32 e) {
    return e == TCW_BE1 ? tcw_oc(K, TCW_BE1) : e == TCW_BE2 ? tcw_oc(K, TCW_BE2) : e == TCW_TRN ? tcw_oc(K, TCW_TRN)
                                                                                                : tcw_oc(K, TCW_EXT);
}
__device__ __forceinline__ u32 w_nout(u32 e) { return tcw_nout(K, e); }
__device__ __forceinline__ u32 w_outn(u32 e, u32 c) {
    const u32 o0 = c * w_oc(e), n = w_nout(e);
    return o0 + w_oc(e) <= n ? w_oc(e) : n - o0;
}
__device__ __forceinline__ u32 w_nc(u32 e, u32 c) { return (4 * w_outn(e, c) + 15) & ~15u; }

struct TcwSm {                 // shared-memory carve-up and barrier addresses
    uint8_t *a;                // A tile [128 x W_KP] core-matrix layout
    u32 stage0;                // shared address of stage 0
    u32 *rows;                 // [(K+1)][128]: B' (ξ-form) and m_r
    const uint4 *ep1;          // [K] (m'_j, -m'_j^-1, C1_j 2^64, |M'_j|_{2^32})
    const uint2 *ep2;          // [K] (m_i, -m_i^-1)
    const u32 *sig;            // [2][K] σ_i 2^64 mod m_i per context
    u32 bar;                   // shared address of the barrier block: full[NST] empty[NST] accf[2] acce[2] aready
    __device__ u32 full(u32 s) const { return bar + 8 * s; }
    __device__ u32 empty(u32 s) const { return bar + 8 * (W_NST + s); }
    __device__ u32 accf(u32 b) const { return bar + 8 * (2 * W_NST + b); }
    __device__ u32 acce(u32 b) const { return bar + 8 * (2 * W_NST + 2 + b); }
    __device__ u32 aready() const { return bar + 8 * (2 * W_NST + 4); }
};

// ---------------------------------------------------------------- producer: stream the B slabs of an extension
struct TcwProducer {
    u32 st = 0, ph = 0;
    u64 pol;
    __device__ void ext(const TcwSm &S, u32 e, const uint8_t *img) {
        u32 off = 0;
#pragma unroll 1
        for (u32 c = 0; c < w_nchunks(e); c++) {
            const u32 nc = w_nc(e, c);
#pragma unroll 1
            for (u32 s = 0; s < tcw_nslab(K); s++) {
                const u32 bytes = nc * 32 * tcw_steps(K, s);
                w_mbar_wait(S.empty(st), ph ^ 1u);
                w_mbar_expect_tx(S.full(st), bytes);
                w_bulk_g2s(S.stage0 + st * W_STG, img + off, bytes, S.full(st), pol);
                off += bytes;
                if (++st == W_NST) { st = 0; ph ^= 1u; }
            }
        }
    }
};

// ---------------------------------------------------------------- MMA issuer: one thread
struct TcwMma {
    u32 st = 0, fph = 0, aph = 0, acc = 0, eph[2] = {0, 0};
    u32 tmem;
    __device__ void ext(const TcwSm &S, u32 e) {
        w_mbar_wait(S.aready(), aph);          // the A rows of all 128 messages are written (and proxy-fenced)
        aph ^= 1u;
        asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
        const u32 sa = smem_u32(S.a);
#pragma unroll 1
        for (u32 c = 0; c < w_nchunks(e); c++) {
            const u32 b = acc, nc = w_nc(e, c);
            w_mbar_wait(S.acce(b), eph[b] ^ 1u);   // the epilogue has read this buffer's previous chunk
            eph[b] ^= 1u;
            asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
            const u32 idesc = (2u << 4) | ((nc >> 3) << 17) | ((128u >> 4) << 24);   // s32 = u8 x u8, K-major, M = 128
            const u32 td = tmem + b * W_NCMAX;
#pragma unroll 1
            for (u32 s = 0; s < tcw_nslab(K); s++) {
                const u32 steps = tcw_steps(K, s);
                w_mbar_wait(S.full(st), fph);
                asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
                const u32 sb = S.stage0 + st * W_STG;
#pragma unroll 1
                for (u32 j = 0; j < steps; j++) {
                    const u64 da = w_desc(sa + (4 * s + j) * 256, W_SBOA), db = w_desc(sb + j * 256, steps * 256);
                    const u32 accum = (s | j) ? 1u : 0u;
                    asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                                 "tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n\t}" ::"r"(td),
                                 "l"(da), "l"(db), "r"(idesc), "r"(accum)
                                 : "memory");
                }
                asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(S.empty(st))
                             : "memory");
                if (++st == W_NST) { st = 0; fph ^= 1u; }
            }
            asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(S.accf(b))
                         : "memory");
            acc ^= 1u;
        }
    }
};

// ---------------------------------------------------------------- compute warps: one message per thread
struct TcwCompute {
    const TcwSm &S;
    u32 tmem;                 // TMEM base
    u32 lane_base;            // (warp's first lane) << 16
    u32 m;                    // message = TMEM lane
    uint8_t *arow;            // this message's A row
    u32 acc = 0, fph[2] = {0, 0};
    u32 sel = 0;              // context of the current job
    const u32 *cx = nullptr;  // its context block (HBM)

    __device__ u32 &row(u32 j) const { return S.rows[j * 128 + m]; }
    __device__ u32 tb(u32 col) const { return tmem + lane_base + col; }
    __device__ void put_a(u32 w, const uint4 &v) const { *reinterpret_cast<uint4 *>(arow + w * 128) = v; }   // words 4w..4w+3 (K-core w)
    __device__ void a_done() const {
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");   // generic-proxy A writes -> async proxy (MMA)
        w_mbar_arrive(S.aready());
    }
    // chunk c of an extension: wait for its accumulator, hand each 16-column group (4 outputs) to f, release
    template <class F>
    __device__ void chunks(u32 e, F &&f) {
#pragma unroll 1
        for (u32 c = 0; c < w_nchunks(e); c++) {
            const u32 b = acc;
            w_mbar_wait(S.accf(b), fph[b]);
            fph[b] ^= 1u;
            asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
            const u32 n4 = (w_outn(e, c) + 3) / 4, o0 = c * w_oc(e);
#pragma unroll 1
            for (u32 g = 0; g < n4; g++) {
                u32 v[16];
                w_tmem_ld16(tb(b * W_NCMAX + 16 * g), v);
                f(o0 + 4 * g, v);
            }
            asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
            __syncwarp();
            if ((m & 31) == 0) w_mbar_arrive(S.acce(b));
            acc ^= 1u;
        }
    }

    // a2: positional -> RNS of nl limbs at x (masked to zero when !ok); m_r = x_0
    __device__ void to_rns(const u32 *x, u32 nl, bool ok) {
#pragma unroll 1
        for (u32 w = 0; w < W_KP / 16; w++) {
            u32 q[4];
#pragma unroll
            for (int t = 0; t < 4; t++) q[t] = (ok && 4 * w + t < nl) ? x[4 * w + t] : 0u;
            put_a(w, make_uint4(q[0], q[1], q[2], q[3]));
        }
        a_done();
        row(K) = ok ? x[0] : 0u;
        chunks(TCW_TRN, [&](u32 o, const u32 (&v)[16]) {
            u32 r[4];
#pragma unroll
            for (int t = 0; t < 4; t++) {
                const u32 ch = o + t;
                u32 lo, hi;
                tc_split(v[4 * t], v[4 * t + 1], v[4 * t + 2], v[4 * t + 3], lo, hi);
                const uint2 mm = ch < K ? S.ep2[ch] : make_uint2(S.ep1[ch - K < K ? ch - K : 0].x, S.ep1[ch - K < K ? ch - K : 0].y);
                r[t] = mont_red(lo, hi, mm.x, mm.y);
                if (ch >= K && ch < 2 * K) row(ch - K) = r[t];
            }
            if (o < K) w_tmem_st4(tb(W_BS + o), r[0], r[1], r[2], r[3]);   // straddling group: B' lanes land in padding
        });
        w_tmem_wait_st();
    }

    // 6.1-6.6: st <- st · b · M^-1 (mod N); b at bp[c · bs] (window table column or constant vector), or st (sq)
    __device__ void mont_mul(const u32 *bp, u32 bs, bool sq) {
        const u32 *sig = S.sig + sel * K;
        // ---- 6.1 B channels: ξ_i = mont(mont(a b) σ_i 2^64) = a b σ_i, into the A row (BE1 input)
#pragma unroll 1
        for (u32 g = 0; g < (K + 15) / 16; g++) {
            u32 a[16];
            w_tmem_ld16(tb(W_BS + 16 * g), a);
            u32 xi[16];
#pragma unroll
            for (int t = 0; t < 16; t++) {
                const u32 i = 16 * g + t;
                xi[t] = 0;
                if (i < K) {
                    const u32 b = sq ? a[t] : __ldcg(bp + (size_t)i * bs);
                    const uint2 mm = S.ep2[i];
                    const u64 pr = (u64)a[t] * b;
                    const u32 tt = mont_red((u32)pr, (u32)(pr >> 32), mm.x, mm.y);
                    const u64 ps = (u64)tt * sig[i];
                    xi[t] = mont_red((u32)ps, (u32)(ps >> 32), mm.x, mm.y);
                }
            }
#pragma unroll
            for (int q = 0; q < 4; q++)   // (the last group may reach past the row's W_KP / 16 K-cores)
                if (4 * g + q < W_KP / 16) put_a(4 * g + q, make_uint4(xi[4 * q], xi[4 * q + 1], xi[4 * q + 2], xi[4 * q + 3]));
        }
        a_done();
        // ---- 6.2 B' channels t*_j = a*_j b*_j 2^-32 and the m_r product, under the BE1 MMAs
#pragma unroll 4
        for (u32 j = 0; j < K; j++) {
            const u32 a = row(j);
            const u32 b = sq ? a : __ldcg(bp + (size_t)(K + j) * bs);
            const uint4 e1 = S.ep1[j];
            const u64 pr = (u64)a * b;
            row(j) = mont_red((u32)pr, (u32)(pr >> 32), e1.x, e1.y);
        }
        const u32 ar = row(K);
        const u32 tr = ar * (sq ? ar : __ldcg(bp + (size_t)(2 * K) * bs));
        // ---- 6.3-6.5 BE1 epilogue: ξ'_j = mont(t*_j C1_j 2^64 + mont(D_j)); m_r column -> r_r
        u32 sr = 0, rr = 0;
        const u32 nminv = cx[CX_NMINV_R];
        chunks(TCW_BE1, [&](u32 o, const u32 (&v)[16]) {
#pragma unroll
            for (int t = 0; t < 4; t++) {
                const u32 j = o + t;
                u32 lo, hi;
                tc_split(v[4 * t], v[4 * t + 1], v[4 * t + 2], v[4 * t + 3], lo, hi);
                if (j < K) {
                    const uint4 e1 = S.ep1[j];
                    const u32 x1 = mont_red(lo, hi, e1.x, e1.y);
                    const u64 p = (u64)row(j) * e1.z + x1;
                    const u32 xp = mont_red((u32)p, (u32)(p >> 32), e1.x, e1.y);
                    row(j) = xp;
                    sr += xp * e1.w;
                } else if (j == K) {   // q̂_r = Σ ξ_i |M_i|_{2^32} mod 2^32;  r_r = (t_r + q̂_r N) M^-1
                    rr = tr * GB(O_MISC + 0) + lo * nminv;
                }
            }
        });
        // ---- 6.6 BE2: A row = (ξ'_0 .. ξ'_{k-1}, α'), α' = (Σ ξ'_j |M'_j|_{2^32} - r_r) M'^-1 exact
        const u32 alpha = (sr - rr) * GB(O_MISC + 1);
        fill_a_from_rows(alpha);
        a_done();
        row(K) = rr;
        chunks(TCW_BE2, [&](u32 o, const u32 (&v)[16]) {
            u32 r[4];
#pragma unroll
            for (int t = 0; t < 4; t++) {
                const u32 i = o + t < K ? o + t : K - 1;
                u32 lo, hi;
                tc_split(v[4 * t], v[4 * t + 1], v[4 * t + 2], v[4 * t + 3], lo, hi);
                const uint2 mm = S.ep2[i];
                r[t] = mont_red(lo, hi, mm.x, mm.y);
            }
            w_tmem_st4(tb(W_BS + o), r[0], r[1], r[2], r[3]);
        });
        w_tmem_wait_st();
    }

    // A row words 0..K-1 <- B' rows, word K <- extra (α'), the rest zero
    __device__ void fill_a_from_rows(u32 extra) {
#pragma unroll 1
        for (u32 w = 0; w < W_KP / 16; w++) {
            u32 q[4];
#pragma unroll
            for (int t = 0; t < 4; t++) {
                const u32 j = 4 * w + t;
                q[t] = j < K ? row(j) : (j == K ? extra : 0u);
            }
            put_a(w, make_uint4(q[0], q[1], q[2], q[3]));
        }
    }

    // a7: X = Σ ξ'_j M'_j + α'(2^(32(K+1)) - M') on the tensor core (byte convolution), limbs into rows 0..K,
    // then X mod N by conditional subtraction of N 2^s, s = SMAX..0 (X < (K+3) N)
    __device__ void from_rns() {
        u32 sr = 0;
#pragma unroll 4
        for (u32 j = 0; j < K; j++) sr += row(j) * S.ep1[j].w;
        const u32 alpha = (sr - row(K)) * GB(O_MISC + 1);
        fill_a_from_rows(alpha);
        a_done();
        u64 carry = 0;
        chunks(TCW_EXT, [&](u32 o, const u32 (&v)[16]) {
#pragma unroll
            for (int t = 0; t < 4; t++) {
                const u32 l = o + t;
                if (l <= K) {
                    const u64 s = carry + v[4 * t] + ((u64)v[4 * t + 1] << 8) + ((u64)v[4 * t + 2] << 16) + ((u64)v[4 * t + 3] << 24);
                    row(l) = (u32)s;
                    carry = s >> 32;
                }
            }
        });
        const u32 *nl = cx + cx_n(K);
#pragma unroll 1
        for (int s = SMAX; s >= 0; s--) {
#pragma unroll 1
            for (int pass = 0; pass < 2; pass++) {   // pass 0: borrow of X - N 2^s; pass 1: subtract
                u32 br = 0;
#pragma unroll 4
                for (u32 l = 0; l <= K; l++) {
                    const u32 nsh = __funnelshift_l(l ? __ldg(nl + l - 1) : 0u, __ldg(nl + l), s);
                    const u64 t = (u64)row(l) - nsh - br;
                    if (pass) row(l) = (u32)t;
                    br = (u32)(t >> 63);
                }
                if (br) break;
            }
        }
    }

    // the op program of one 128-message job (same ops as run_program in mr_kernels.cuh)
    __device__ void job(const ModexpParams &P, u32 jl, bool valid) {
        const u32 *xrow = P.x + (size_t)(valid ? jl : 0) * P.in_limbs;
        const bool ok = valid && less_than(xrow, cx + cx_inb(K), P.in_limbs);
        if (valid && sel == 0 && P.status) P.status[jl] = ok ? 0 : 5 /* MR_ERR_RANGE */;
        const size_t tstride = P.jobs_total, entry = (size_t)NCH * tstride;
        const u32 col = sel * P.ctas0 * 128 + jl;     // window-table column (tail lanes too: jl < ctas0 * 128)
        const u64 *prog = sel ? P.prog[1] : P.prog[0];
        const u32 nops = sel ? P.nops[1] : P.nops[0];
#pragma unroll 1
        for (u32 s = 0; s < nops; s++) {
            const u64 op = __ldg(prog + s);
            const u32 fl = (u32)op & 0xFF, opnd = (u32)(op >> 8) & 0xFF, ld = (u32)(op >> 16) & 0xFF;
            const u32 ad = (u32)(op >> 24) & 0xFF, sto = (u32)(op >> 32) & 0xFF;
            if (fl & (OPF_TORNS_ALL | OPF_TORNS_LO | OPF_TORNS_HI)) {
                const u32 off = (fl & OPF_TORNS_HI) ? P.half : 0u;
                to_rns(xrow + off, (fl & OPF_TORNS_ALL) ? P.in_limbs : P.half, ok);
            }
            if (fl & OPF_LOAD) {
                const u32 *src;
                size_t str;
                if (ld >= 0xF0) { src = cx + cx_r2(K) + (ld - 0xF0) * NCH; str = 1; }
                else { src = P.table + ld * entry + col; str = tstride; }
#pragma unroll 1
                for (u32 g = 0; g < tcw_bsw(K) / 4; g++) {
                    u32 q[4];
#pragma unroll
                    for (int t = 0; t < 4; t++) q[t] = 4 * g + t < K ? src[(4 * g + t) * str] : 0u;
                    w_tmem_st4(tb(W_BS + 4 * g), q[0], q[1], q[2], q[3]);
                }
#pragma unroll 4
                for (u32 j = 0; j <= K; j++) row(j) = src[(K + j) * str];
                w_tmem_wait_st();
            }
            if (!(fl & OPF_NOMUL)) {
                const bool sq = opnd == OPND_SQ;
                const u32 *bp = sq ? nullptr : (opnd >= 0xF0 ? cx + cx_r2(K) + (opnd - 0xF0) * NCH : P.table + opnd * entry + col);
                mont_mul(bp, sq ? 0u : (opnd >= 0xF0 ? 1u : (u32)tstride), sq);
            }
            if (fl & OPF_ADD) {   // channel-wise modular addition (CRT entry, a3)
                const u32 *src = P.table + ad * entry + col;
#pragma unroll 1
                for (u32 g = 0; g < (K + 15) / 16; g++) {
                    u32 a[16];
                    w_tmem_ld16(tb(W_BS + 16 * g), a);
#pragma unroll
                    for (int t = 0; t < 16; t++) {
                        const u32 i = 16 * g + t;
                        if (i < K) a[t] = w_addmod(a[t], src[i * tstride], 0u - S.ep2[i].x);
                    }
                    w_tmem_st16(tb(W_BS + 16 * g), a);
                }
#pragma unroll 4
                for (u32 j = 0; j < K; j++) row(j) = w_addmod(row(j), src[(K + j) * tstride], 0u - S.ep1[j].x);
                row(K) += src[2 * K * tstride];
                w_tmem_wait_st();
            }
            if (fl & OPF_STORE) {
                u32 *dst = P.table + sto * entry + col;
#pragma unroll 1
                for (u32 g = 0; g < (K + 15) / 16; g++) {
                    u32 a[16];
                    w_tmem_ld16(tb(W_BS + 16 * g), a);
#pragma unroll
                    for (int t = 0; t < 16; t++)
                        if (16 * g + t < K) dst[(16 * g + t) * tstride] = a[t];
                }
#pragma unroll 4
                for (u32 j = 0; j <= K; j++) dst[(K + j) * tstride] = row(j);
            }
        }
        from_rns();
        if (valid) {
            u32 *yrow = P.y + sel * P.out_stride + (size_t)jl * P.out_limbs;
#pragma unroll 1
            for (u32 l = 0; l < P.out_limbs; l++) yrow[l] = ok ? row(l) : 0u;
        }
    }
};

// Persistent kernel, one CTA per SM: tile-jobs t = blockIdx.x, blockIdx.x + gridDim.x, ... of 128 messages;
// job t runs context sel = t / ctas0.  Every role walks the same job list and op programs, so the producer,
// the MMA issuer and the epilogues meet on the same sequence of (extension, chunk, slab).
__global__ void __launch_bounds__(W_THREADS, 1) k_modexp_tcw(const ModexpParams P, const TcwArgs A) {
    extern __shared__ __align__(1024) uint8_t wsm[];
    TcwSm S;
    S.a = wsm;
    S.stage0 = smem_u32(wsm + (size_t)128 * W_KP);
    S.rows = reinterpret_cast<u32 *>(wsm + (size_t)128 * W_KP + (size_t)W_NST * W_STG);
    uint4 *ep1 = reinterpret_cast<uint4 *>(S.rows + W_ROWS);
    uint2 *ep2 = reinterpret_cast<uint2 *>(ep1 + K);
    u32 *sig = reinterpret_cast<u32 *>(ep2 + K);
    S.ep1 = ep1;
    S.ep2 = ep2;
    S.sig = sig;
    u64 *bars = reinterpret_cast<u64 *>(((uintptr_t)(sig + 2 * K) + 7) & ~(uintptr_t)7);
    u32 *tslot = reinterpret_cast<u32 *>(bars + 2 * W_NST + 5);
    S.bar = smem_u32(bars);
    const u32 tid = threadIdx.x, warp = tid / 32;
    const WideLayout WL = wide_layout(K);
    for (u32 j = tid; j < K; j += W_THREADS) {
        ep1[j] = make_uint4(__ldg(A.wtab + WL.mm + K + j), __ldg(A.wtab + WL.minv + K + j), __ldg(A.wtab + WL.xw + j),
                            __ldg(A.wtab + WL.a2r + j));
        ep2[j] = make_uint2(__ldg(A.wtab + WL.mm + j), __ldg(A.wtab + WL.minv + j));
        sig[j] = __ldg(P.ctx[0] + A.cxw + wide_cx_sig(K) + j);
        sig[K + j] = __ldg(P.ctx[1] + A.cxw + wide_cx_sig(K) + j);
    }
    if (tid == 0) {
        for (u32 s = 0; s < W_NST; s++) {
            w_mbar_init(S.full(s), 1);
            w_mbar_init(S.empty(s), 1);
        }
        for (u32 b = 0; b < 2; b++) {
            w_mbar_init(S.accf(b), 1);
            w_mbar_init(S.acce(b), 4);
        }
        w_mbar_init(S.aready(), 128);
    }
    if (warp == 5) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tslot)), "r"(512));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    const u32 tmem = *tslot;
    const u32 J = A.jobs;

    if (warp == 4) {                                  // ---- producer
        if ((tid & 31) == 0) {
            TcwProducer pr;
            asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(pr.pol));
#pragma unroll 1
            for (u32 t = blockIdx.x; t < J; t += gridDim.x) {
                const u32 sel = t / P.ctas0;
                const uint8_t *be1 = reinterpret_cast<const uint8_t *>((sel ? P.ctx[1] : P.ctx[0]) + A.be1w);
                const u64 *prog = sel ? P.prog[1] : P.prog[0];
                const u32 nops = sel ? P.nops[1] : P.nops[0];
#pragma unroll 1
                for (u32 s = 0; s < nops; s++) {
                    const u32 fl = (u32)__ldg(prog + s) & 0xFF;
                    if (fl & (OPF_TORNS_ALL | OPF_TORNS_LO | OPF_TORNS_HI)) pr.ext(S, TCW_TRN, A.kimg + tcw_img_off(K, TCW_TRN));
                    if (!(fl & OPF_NOMUL)) {
                        pr.ext(S, TCW_BE1, be1);
                        pr.ext(S, TCW_BE2, A.kimg + tcw_img_off(K, TCW_BE2));
                    }
                }
                pr.ext(S, TCW_EXT, A.kimg + tcw_img_off(K, TCW_EXT));
            }
        }
    } else if (warp == 5) {                           // ---- MMA issuer
        if ((tid & 31) == 0) {
            TcwMma mm;
            mm.tmem = tmem;
#pragma unroll 1
            for (u32 t = blockIdx.x; t < J; t += gridDim.x) {
                const u32 sel = t / P.ctas0;
                const u64 *prog = sel ? P.prog[1] : P.prog[0];
                const u32 nops = sel ? P.nops[1] : P.nops[0];
#pragma unroll 1
                for (u32 s = 0; s < nops; s++) {
                    const u32 fl = (u32)__ldg(prog + s) & 0xFF;
                    if (fl & (OPF_TORNS_ALL | OPF_TORNS_LO | OPF_TORNS_HI)) mm.ext(S, TCW_TRN);
                    if (!(fl & OPF_NOMUL)) {
                        mm.ext(S, TCW_BE1);
                        mm.ext(S, TCW_BE2);
                    }
                }
                mm.ext(S, TCW_EXT);
            }
        }
    } else {                                          // ---- compute warps
        TcwCompute cw{S, tmem, (tid & ~31u) << 16, tid, S.a + (tid / 8) * W_SBOA + (tid % 8) * 16};
#pragma unroll 1
        for (u32 t = blockIdx.x; t < J; t += gridDim.x) {
            cw.sel = t / P.ctas0;
            cw.cx = cw.sel ? P.ctx[1] : P.ctx[0];
            const u32 jl = (t - cw.sel * P.ctas0) * 128 + tid;
            cw.job(P, jl, jl < P.count);
        }
    }
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    if (warp == 5) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(512));
}

#endif  // MR_K == 97 || MR_K == 129
