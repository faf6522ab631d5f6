// mr_lanes.cu — small-batch ladder kernel for the narrow channel counts (k = 17, 33, 49, 65), DESIGN.md §4j.
//
// A batch of a few hundred messages fills two or three 128-message tensor tiles, i.e. two or three SMs, and
// each tile then runs at the latency of one Montgomery multiplication chain (~3.3 µs per multiplication).
// This kernel maps ONE message to a CTA and its RNS channels to threads — the paper's own mapping ("channels
// are directly mapped onto threads", §3.1) — so a 256-message batch occupies 256 CTAs, and splits every
// base-extension output over MR_LANES_LPO = 4 lanes (each lane sums every LPO-th input, log2(LPO) 96-bit shuffle adds combine
// them), so the critical path of a multiplication is ~k/4 multiply-accumulates instead of k:
//   channel products   thread per channel (2k+1 <= threads)
//   BE1 (6.3-6.5)      output j in B' ∪ {m_r}: lanes 4j..4j+3 of the CTA, Σ_i ξ_i A1'[j][i]
//   BE2 (6.6)          output i in B: lanes 4i..4i+3, Σ_j ξ'_j A2[i][j] + α' (m_i - |M'|_{m_i})
// The constant matrices (8.7 KB at k = 33, 33 KB at k = 65) are staged once per CTA in shared memory, rows
// per output so the four lanes of an output read interleaved words.  Arithmetic is the wide kernel's
// (mr_wide.cu): word Montgomery reductions with the 2^-32 factors folded into the per-k wide table and the
// per-context wide section (σ 2^64, A1' 2^32, A2 2^32, powers 2^32), plain B residues, B' in ξ-form, the same op
// programs (sliding window, CRT entry) and the same exit (CRT with the extra modulus m_r = 2^32, then
// conditional subtraction of N 2^s).  Results are bit-identical to every other path (tests/test_gpu_paths.py).
#include <cuda_runtime.h>

#include <cstdint>

#include "mr_internal.h"

namespace mr {
namespace {

__device__ __forceinline__ void mac96(u32 &lo, u32 &mid, u32 &hi, u32 x, u32 y) {
    asm("mad.lo.cc.u32 %0, %3, %4, %0;\n\t"
        "madc.hi.cc.u32 %1, %3, %4, %1;\n\t"
        "addc.u32 %2, %2, 0;"
        : "+r"(lo), "+r"(mid), "+r"(hi)
        : "r"(x), "r"(y));
}
__device__ __forceinline__ void add96(u32 &lo, u32 &mi, u32 &hi, u32 l2, u32 m2, u32 h2) {
    asm("add.cc.u32 %0, %0, %3;\n\taddc.cc.u32 %1, %1, %4;\n\taddc.u32 %2, %2, %5;"
        : "+r"(lo), "+r"(mi), "+r"(hi)
        : "r"(l2), "r"(m2), "r"(h2));
}
// T = thi 2^32 + tlo -> T 2^-32 mod m, lazy in [0, 2^32) (any odd m)
__device__ __forceinline__ u32 mont_red(u32 tlo, u32 thi, u32 m, u32 minv) {
    const u32 q = tlo * minv;
    [[maybe_unused]] u32 ulo;
    u32 uhi, cy;
    asm("mad.lo.cc.u32 %0, %3, %4, %5;\n\tmadc.hi.cc.u32 %1, %3, %4, %6;\n\taddc.u32 %2, 0, 0;"
        : "=r"(ulo), "=r"(uhi), "=r"(cy)
        : "r"(q), "r"(m), "r"(tlo), "r"(thi));
    return cy ? uhi - m : uhi;
}
__device__ __forceinline__ u32 addmod_lazy(u32 a, u32 b, u32 r32) {
    const u64 s = (u64)a + b;
    const u64 t = (u64)(u32)s + (s >> 32) * r32;
    return (u32)t + (u32)(t >> 32) * r32;
}
__device__ __forceinline__ u32 red96_mont(u32 hi, u32 mid, u32 lo, u32 m, u32 minv, u32 r32) {
    const u32 r = mont_red(lo, mid, m, minv);
    const u32 t = hi * r32;
    const u32 s = r + t;
    return s < r ? s + r32 : s;
}
#ifndef MR_LANES_LPO
#define MR_LANES_LPO 4      // lanes per base-extension output (4 or 8; A/B: 8 is 15 % slower on C1, profiles/r2aj)
#endif
// 96-bit sum over the MR_LANES_LPO lanes of an output group (lanes LPO g .. LPO g + LPO - 1 of a warp)
__device__ __forceinline__ void quad_sum(u32 &lo, u32 &mi, u32 &hi) {
#pragma unroll
    for (int o = 1; o < MR_LANES_LPO; o <<= 1) {
        const u32 l2 = __shfl_xor_sync(0xFFFFFFFFu, lo, o), m2 = __shfl_xor_sync(0xFFFFFFFFu, mi, o);
        const u32 h2 = __shfl_xor_sync(0xFFFFFFFFu, hi, o);
        add96(lo, mi, hi, l2, m2, h2);
    }
}

#ifndef MR_LANES_CREG
#define MR_LANES_CREG 1     // 1: each lane keeps its 2 x ceil(k/4) base-extension coefficients in registers
#endif
#ifndef MR_LANES_FRAC
// 1: α' of BE2 and of the exit from the top bits of the ξ'_j (reading R2b, as the tensor kernels), so the
// m_r = 2^32 channel needs no upkeep: no m_r column in BE1 (a divergent branch of one output group), no
// Σ ξ'_j |M'_j|_{2^32} products, no r_r round trip through shared memory
#define MR_LANES_FRAC 1
#endif
// α' = floor(Σ_j ξ'_j / m'_j) from s = Σ_j (ξ'_j >> 8) (exact for k <= 65 and r / M' < 0.11: reading R2b)
__device__ __forceinline__ u32 frac_alpha(u32 s) { return (s + (1u << 14)) >> 24; }

template <int K>
struct LaneCfg {
    static constexpr int NCH = 2 * K + 1;
    static constexpr int LPO = MR_LANES_LPO;          // lanes per output
    static constexpr int OPW = 32 / LPO;              // outputs per warp
    static constexpr int W = (K + 1 + OPW - 1) / OPW; // warps
    static constexpr int NT = 32 * W;
    static constexpr int Q = (K + LPO - 1) / LPO;     // inputs per lane (the last lanes may have one fewer)
    static_assert(NT >= NCH, "one thread per channel");
};

// shared memory layout (words)
template <int K>
struct LaneSmem {
    static constexpr u32 st = 0;                             // [2k+1] state
    static constexpr u32 a1 = (2 * K + 1 + 3) & ~3;          // [k+1][k] BE1 rows: A1'[j][i] 2^32, row k: |M_i|_{2^32}
    static constexpr u32 a2 = a1 + (K + 1) * K;              // [k][k] BE2 rows: A2[i][j] 2^32 (|M'_j|_{m_i})
    static constexpr u32 mm = a2 + K * K;                    // [2k] m
    static constexpr u32 minv = mm + 2 * K;                  // [2k] -m^-1
    static constexpr u32 r32 = minv + 2 * K;                 // [2k] 2^32 mod m
    static constexpr u32 sig = r32 + 2 * K;                  // [k]  σ_i 2^64
    static constexpr u32 xw = sig + K;                       // [k]  |M^-1 λ_j^-1| 2^64
    static constexpr u32 a2r = xw + K;                       // [k]  |M'_j|_{2^32}
    static constexpr u32 pinw = a2r + K;                     // [k]  (m_i - |M'|_{m_i}) 2^32
    static constexpr u32 red = pinw + K;                     // [W]  warp partials
    static constexpr u32 aux = red + 32;                     // [4]  r_r, α', misc
    static constexpr u32 xs = aux + 4;                       // [2k+2] staged input limbs / exit scratch
    static constexpr u32 words = xs + 3 * (K + 1) + 4;       // exit: 3 words per column
};

template <int K>
__global__ void __launch_bounds__(LaneCfg<K>::NT) k_modexp_lane(const ModexpParams P, const u32 *__restrict__ tab,
                                                                const u32 cxw) {
    using C = LaneCfg<K>;
    using S = LaneSmem<K>;
    extern __shared__ __align__(16) u32 sm[];
    constexpr int NCH = C::NCH;
    const u32 tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const u32 sel = blockIdx.x >= P.ctas0 ? 1u : 0u;
    const u32 *cx = sel ? P.ctx[1] : P.ctx[0];
    const u32 jl = blockIdx.x - sel * P.ctas0;               // message index in the context
    const WideLayout L = wide_layout(K);
    u32 *st = sm + S::st;
    // ---- stage the constants (per context: A1' and σ from the wide section; per k: the rest)
    const u32 *a1w = cx + cxw + wide_cx_a1(K), *sigw = cx + cxw + wide_cx_sig(K);
    for (u32 e = tid; e < (u32)(K * K); e += C::NT) {
        const u32 j = e / K, i = e % K;
        sm[S::a1 + e] = __ldg(a1w + wch_at(i, j, K));         // row j (output), column i (input)
        sm[S::a2 + e] = __ldg(tab + L.a2w + wch_at(i, j, K)); // row j here = output i of BE2, column = input
    }
    for (u32 i = tid; i < (u32)K; i += C::NT) {
        sm[S::a1 + K * K + i] = __ldg(tab + L.a1r + i);
        sm[S::sig + i] = __ldg(sigw + i);
        sm[S::xw + i] = __ldg(tab + L.xw + i);
        sm[S::a2r + i] = __ldg(tab + L.a2r + i);
        sm[S::pinw + i] = __ldg(tab + L.pinw + i);
    }
    for (u32 c = tid; c < (u32)(2 * K); c += C::NT) {
        sm[S::mm + c] = __ldg(tab + L.mm + c);
        sm[S::minv + c] = __ldg(tab + L.minv + c);
        sm[S::r32 + c] = __ldg(tab + L.r32 + c);
    }
    __shared__ bool ok_s;
    if (tid == 0) {   // x < input bound (little-endian limbs, most significant first)
        bool ok = false;
        if (jl < P.count) {
            const u32 *xr = P.x + (size_t)jl * P.in_limbs, *bnd = cx + cx_inb(K);
            int res = 0;
            for (int l = (int)P.in_limbs - 1; l >= 0 && res == 0; l--) res = xr[l] < bnd[l] ? -1 : (xr[l] > bnd[l] ? 1 : 0);
            ok = res < 0;
            if (sel == 0 && P.status) P.status[jl] = ok ? 0 : 5 /* MR_ERR_RANGE */;
        }
        ok_s = ok;
    }
    __syncthreads();
    const bool ok = ok_s;
    const u32 minv32 = __ldg(tab + L.misc + 0), minvp = __ldg(tab + L.misc + 1), nminv = cx[CX_NMINV_R];
    const u32 g = lane / C::LPO, sub = lane % C::LPO, o = warp * C::OPW + g;   // this lane's output and share
    const u32 *a1row = sm + S::a1 + o * K, *a2row = sm + S::a2 + o * K;
    // this lane's base-extension coefficients (inputs sub + LPO t of its output) in registers for the whole ladder
    // (MR_LANES_CREG): the multiply-accumulate loops then read only the state from shared memory
    u32 c1r[C::Q], c2r[C::Q];
#pragma unroll
    for (int t = 0; t < C::Q; t++) {
        const u32 i = sub + C::LPO * t;
        const bool in = MR_LANES_CREG && o < (u32)K && i < (u32)K;
        c1r[t] = in ? a1row[i] : 0u;
        c2r[t] = in ? a2row[i] : 0u;
    }
    // ... and the per-channel / per-output moduli and constants (shared-memory reads otherwise, every multiplication)
    const u32 chm = tid < (u32)(2 * K) ? sm[S::mm + tid] : 1u, chmi = tid < (u32)(2 * K) ? sm[S::minv + tid] : 0u;
    const u32 chsig = tid < (u32)K ? sm[S::sig + tid] : 0u;
    const u32 oc = o < (u32)K ? o : 0u;
    const u32 e1m = sm[S::mm + K + oc], e1mv = sm[S::minv + K + oc], e1r = sm[S::r32 + K + oc], e1xw = sm[S::xw + oc];
    const u32 e2m = sm[S::mm + oc], e2mv = sm[S::minv + oc], e2r = sm[S::r32 + oc], e2pin = sm[S::pinw + oc];

    // st <- st · b · M^-1 (mod N); b at bp[ch * bstride] or the state itself (sq)
    auto mont_mul = [&](const u32 *bp, size_t bstride, bool sq) {
        // channel products: B: ξ_i = mont(mont(a b) σ_i 2^64); B': t*_j = mont(a* b*); m_r: a_r b_r
        if (tid < (u32)(2 * K)) {
            const u32 a = st[tid], b = sq ? a : __ldcg(bp + tid * bstride);
            const u32 m = MR_LANES_CREG ? chm : sm[S::mm + tid], mi = MR_LANES_CREG ? chmi : sm[S::minv + tid];
            const u64 pr = (u64)a * b;
            u32 t = mont_red((u32)pr, (u32)(pr >> 32), m, mi);
            if (tid < (u32)K) {
                const u64 ps = (u64)t * (MR_LANES_CREG ? chsig : sm[S::sig + tid]);
                t = mont_red((u32)ps, (u32)(ps >> 32), m, mi);
            }
            st[tid] = t;
        } else if (!MR_LANES_FRAC && tid == (u32)(2 * K)) {
            const u32 a = st[tid];
            st[tid] = a * (sq ? a : __ldcg(bp + tid * bstride));
        }
        __syncthreads();
        // BE1: output o (o < K: B' channel; o = K: the m_r column), lanes split the inputs i = sub + LPO t over two
        // accumulator chains.  The shuffles run on every lane (groups past the last output sum zeros), so they
        // stay convergent.
        {
            u32 lo = 0, mi = 0, hi = 0, l1 = 0, m1 = 0, h1 = 0, qr = 0;
            if (o < (u32)K) {
#pragma unroll
                for (int t = 0; t < C::Q; t++) {
                    const u32 i = sub + C::LPO * t;
                    if (C::LPO * t + C::LPO - 1 < K || i < (u32)K) {
                        const u32 cf = MR_LANES_CREG ? c1r[t] : a1row[i];
                        if (t & 1) mac96(l1, m1, h1, st[i], cf);
                        else mac96(lo, mi, hi, st[i], cf);
                    }
                }
                add96(lo, mi, hi, l1, m1, h1);
            } else if (!MR_LANES_FRAC && o == (u32)K) {
#pragma unroll
                for (int t = 0; t < C::Q; t++) {
                    const u32 i = sub + C::LPO * t;
                    if (C::LPO * t + C::LPO - 1 < K || i < (u32)K) qr += st[i] * a1row[i];
                }
            }
            quad_sum(lo, mi, hi);
            if (!MR_LANES_FRAC) {
#pragma unroll
                for (int sh = 1; sh < C::LPO; sh <<= 1) qr += __shfl_xor_sync(0xFFFFFFFFu, qr, sh);
            }
            if (sub == 0 && o < (u32)K) {
                const u32 ch = K + o;
                const u32 m = MR_LANES_CREG ? e1m : sm[S::mm + ch], mv = MR_LANES_CREG ? e1mv : sm[S::minv + ch];
                const u32 r32 = MR_LANES_CREG ? e1r : sm[S::r32 + ch];
                const u32 v = red96_mont(hi, mi, lo, m, mv, r32);          // Σ ξ A1'  (mod m'_j)
                const u64 p = (u64)st[ch] * (MR_LANES_CREG ? e1xw : sm[S::xw + o]);   // t* C1 2^64
                st[ch] = addmod_lazy(mont_red((u32)p, (u32)(p >> 32), m, mv), v, r32);   // ξ'_j (lazy)
            } else if (!MR_LANES_FRAC && sub == 0 && o == (u32)K) {
                sm[S::aux + 0] = st[2 * K] * minv32 + qr * nminv;          // r_r = (t_r + q̂_r N) M^-1
            }
        }
        __syncthreads();
        // BE2: output o < K of B, lanes split the inputs j = sub + LPO t.  Every group also sums its share of
        // Σ_j ξ'_j |M'_j|_{2^32} over the same j, so each group forms α' = (that sum - r_r) M'^-1 mod 2^32
        // (exact: Shenoy-Kumaresan through m_r) itself — no block reduction and no extra barrier — and adds
        // α' (m_i - |M'|_{m_i}) after the contraction.
        const u32 rr = MR_LANES_FRAC ? 0u : sm[S::aux + 0];
        {
            u32 lo = 0, mi = 0, hi = 0, l1 = 0, m1 = 0, h1 = 0, sa = 0;
            if (o < (u32)K) {
#pragma unroll
                for (int t = 0; t < C::Q; t++) {
                    const u32 j = sub + C::LPO * t;
                    if (C::LPO * t + C::LPO - 1 < K || j < (u32)K) {
                        const u32 x = st[K + j];
                        const u32 cf = MR_LANES_CREG ? c2r[t] : a2row[j];
                        if (t & 1) mac96(l1, m1, h1, x, cf);
                        else mac96(lo, mi, hi, x, cf);
                        sa += MR_LANES_FRAC ? x >> 8 : x * sm[S::a2r + j];
                    }
                }
                add96(lo, mi, hi, l1, m1, h1);
            }
            quad_sum(lo, mi, hi);
#pragma unroll
            for (int sh = 1; sh < C::LPO; sh <<= 1) sa += __shfl_xor_sync(0xFFFFFFFFu, sa, sh);
            if (sub == 0 && o < (u32)K) {
                const u32 alpha = MR_LANES_FRAC ? frac_alpha(sa) : (sa - rr) * minvp;
                mac96(lo, mi, hi, alpha, MR_LANES_CREG ? e2pin : sm[S::pinw + o]);
                st[o] = MR_LANES_CREG ? red96_mont(hi, mi, lo, e2m, e2mv, e2r)
                                      : red96_mont(hi, mi, lo, sm[S::mm + o], sm[S::minv + o], sm[S::r32 + o]);
            }
        }
        if (!MR_LANES_FRAC && tid == 0) st[2 * K] = rr;
        __syncthreads();
    };

    const u64 *prog = sel ? P.prog[1] : P.prog[0];
    const u32 nops = sel ? P.nops[1] : P.nops[0];
    const size_t tstride = P.jobs_total, entry = (size_t)NCH * tstride;
    const u32 slot0 = sel * P.ctas0 + jl;
    u32 *xs = sm + S::xs;
    for (u32 s = 0; s < nops; s++) {
        const u64 op = __ldg(prog + s);
        const u32 fl = (u32)op & 0xFF, opnd = (u32)(op >> 8) & 0xFF, ld = (u32)(op >> 16) & 0xFF;
        const u32 ad = (u32)(op >> 24) & 0xFF, sto = (u32)(op >> 32) & 0xFF;
        if (fl & (OPF_TORNS_ALL | OPF_TORNS_LO | OPF_TORNS_HI)) {   // positional -> RNS (a2)
            const u32 off = (fl & OPF_TORNS_HI) ? P.half : 0u;
            const u32 nl = (fl & OPF_TORNS_ALL) ? P.in_limbs : P.half;
            for (u32 l = tid; l < nl; l += C::NT) xs[l] = ok ? P.x[(size_t)jl * P.in_limbs + off + l] : 0u;
            __syncthreads();
            if (tid < (u32)(2 * K)) {   // channel c = Σ_l x_l |2^(32 l) 2^32|_{m_c}, one Montgomery fold
                u32 lo = 0, mi = 0, hi = 0;
                for (u32 l = 0; l < nl; l++) mac96(lo, mi, hi, xs[l], __ldg(tab + L.pow + wch_at(l, tid, 2 * K)));
                st[tid] = red96_mont(hi, mi, lo, sm[S::mm + tid], sm[S::minv + tid], sm[S::r32 + tid]);
            } else if (tid == (u32)(2 * K)) {
                st[tid] = xs[0];
            }
            __syncthreads();
        }
        if (fl & OPF_LOAD) {
            if (tid < (u32)NCH)
                st[tid] = ld >= 0xF0 ? cx[cx_r2(K) + (ld - 0xF0) * NCH + tid] : P.table[ld * entry + tid * tstride + slot0];
            __syncthreads();
        }
        if (!(fl & OPF_NOMUL)) {
            if (opnd == OPND_SQ) mont_mul(nullptr, 0, true);
            else if (opnd >= 0xF0) mont_mul(cx + cx_r2(K) + (opnd - 0xF0) * NCH, 1, false);
            else mont_mul(P.table + opnd * entry + slot0, tstride, false);
        }
        if (fl & OPF_ADD) {   // channel-wise lazy modular addition (CRT entry)
            if (tid < (u32)NCH) {
                const u32 b = P.table[ad * entry + tid * tstride + slot0];
                st[tid] = tid < (u32)(2 * K) ? addmod_lazy(st[tid], b, sm[S::r32 + tid]) : st[tid] + b;
            }
            __syncthreads();
        }
        if (fl & OPF_STORE) {
            if (tid < (u32)NCH) P.table[sto * entry + tid * tstride + slot0] = st[tid];
            __syncthreads();
        }
    }

    // ---- exit (a7): X = Σ_j ξ'_j M'_j + α'(2^(32(k+1)) - M') (column sums), then X mod N
    {
        u32 part = 0;
        if (tid < (u32)K) part = MR_LANES_FRAC ? st[K + tid] >> 8 : st[K + tid] * sm[S::a2r + tid];
#pragma unroll
        for (int s = 16; s > 0; s >>= 1) part += __shfl_xor_sync(0xFFFFFFFFu, part, s);
        if (lane == 0) sm[S::red + warp] = part;
        __syncthreads();
        u32 sr = 0;
#pragma unroll
        for (int w = 0; w < C::W; w++) sr += sm[S::red + w];
        const u32 alpha = MR_LANES_FRAC ? frac_alpha(sr) : (sr - st[2 * K]) * minvp;
        if (tid <= (u32)K) {   // column l = tid
            const u32 l = tid;
            u32 lo = 0, mi = 0, hi = 0;
            mac96(lo, mi, hi, alpha, __ldg(tab + L.nmp + l));
            for (u32 j = 0; j < (u32)K; j++) mac96(lo, mi, hi, st[K + j], __ldg(tab + L.mpl + wch_at(j, l, K + 1)));
            xs[3 * l] = lo;
            xs[3 * l + 1] = mi;
            xs[3 * l + 2] = hi;
        }
        __syncthreads();
        if (tid == 0) {   // carries, then conditional subtraction of N 2^s, s = smax .. 0
            u32 *X = st;   // the state is no longer needed: X limbs [0, k]
            u64 carry = 0;
            for (u32 l = 0; l <= (u32)K; l++) {
                const u64 s2 = (u64)xs[3 * l] + (u32)carry;
                X[l] = (u32)s2;
                carry = (carry >> 32) + xs[3 * l + 1] + ((u64)xs[3 * l + 2] << 32) + (s2 >> 32);
            }
            const u32 *nl = cx + cx_n(K);
            const int smax = (int)(32 - __clz(K + 2)) - 1;   // X < (k+3) N <= 2^(smax+1) N
            for (int s = smax; s >= 0; s--) {
                int cmp = 0;   // X >= N 2^s ? from the top limb down, then one subtraction pass
                for (int l = K; l >= 0 && cmp == 0; l--) {
                    const u32 nlo = l ? nl[l - 1] : 0u, nhi = l < K ? nl[l] : 0u;
                    const u32 nsh = s ? __funnelshift_l(nlo, nhi, s) : nhi;
                    cmp = X[l] > nsh ? 1 : (X[l] < nsh ? -1 : 0);
                }
                if (cmp < 0) continue;
                u32 br = 0;
                for (u32 l = 0; l <= (u32)K; l++) {
                    const u32 nlo = l ? nl[l - 1] : 0u, nhi = l < (u32)K ? nl[l] : 0u;
                    const u32 nsh = s ? __funnelshift_l(nlo, nhi, s) : nhi;
                    const u64 t = (u64)X[l] - nsh - br;
                    X[l] = (u32)t;
                    br = (u32)(t >> 63);
                }
            }
        }
        __syncthreads();
        if (jl < P.count) {
            u32 *y = P.y + sel * P.out_stride + (size_t)jl * P.out_limbs;
            for (u32 l = tid; l < P.out_limbs; l += C::NT) y[l] = ok ? st[l] : 0u;
        }
    }
}

template <int K>
int launch_k(const ModexpParams &p, u32 ctas, const u32 *tab, u32 cxw, void *stream) {
    const size_t smem = 4 * (size_t)LaneSmem<K>::words;
    if (cudaFuncSetAttribute((const void *)k_modexp_lane<K>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) !=
        cudaSuccess)
        return 6;
    void *args[] = {const_cast<ModexpParams *>(&p), const_cast<u32 **>(&tab), &cxw};
    return cudaLaunchKernel((const void *)k_modexp_lane<K>, dim3(ctas), dim3(LaneCfg<K>::NT), args, smem,
                            (cudaStream_t)stream) == cudaSuccess
               ? 0
               : 6;
}

}  // namespace

int wide_messages_per_cta_lanes() { return 1; }

// one CTA per message and context; k in {17, 33, 49, 65} (host: small_ok)
int launch_modexp_wide_lanes(const ModexpParams &p, u32 ctas, const u32 *d_wide_tab, u32 k, u32 cxw, void *stream) {
    switch (k) {
        case 17: return launch_k<17>(p, ctas, d_wide_tab, cxw, stream);
        case 33: return launch_k<33>(p, ctas, d_wide_tab, cxw, stream);
        case 49: return launch_k<49>(p, ctas, d_wide_tab, cxw, stream);
        case 65: return launch_k<65>(p, ctas, d_wide_tab, cxw, stream);
        default: return 6;
    }
}

}  // namespace mr
