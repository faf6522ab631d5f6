// mr_host.cpp — host runtime of the C ABI (include/mr_rns.h): base construction, constant
// precomputation ("pre-computed and installed permanently in GPU memory at initialization time",
// P:48 §3.1), exponent recoding into kernel programs (sliding window, reading R6), scratch
// management and launches.  All bignum work here is library-internal positional helpers used only
// for precomputation; it shares no code with oracle/.
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdlib>
#include <cstdio>
#include <cstring>
#include <map>
#include <mutex>
#include <new>
#include <vector>

#include "../../include/mr_rns.h"
#include "mr_internal.h"

namespace mr {
#define MR_DECLARE_K(k) KernelSet kernels_k##k();
MR_DECLARE_K(1)
MR_DECLARE_K(2)
MR_DECLARE_K(3)
MR_DECLARE_K(5)
MR_DECLARE_K(9)
MR_DECLARE_K(17)
MR_DECLARE_K(33)
MR_DECLARE_K(49)
MR_DECLARE_K(65)
MR_DECLARE_K(97)
MR_DECLARE_K(129)

size_t wide_smem_bytes(u32 k);
int wide_messages_per_cta();
int launch_modexp_wide(const ModexpParams &p, u32 ctas, const u32 *d_wide_tab, u32 k, u32 cxw, void *stream);
// the tensor-core wide kernel at k = 257 (mr_tcw257.cu; k = 97 / 129 come with their per-k kernel sets)
int launch_modexp_tcw_k257(const ModexpParams &p, u32 ctas, const u32 *tab, const void *kimg, u32 cxw, u32 be1w, u32 jobs,
                           void *trace, void *stream);
int launch_modexp_tcw_k505(const ModexpParams &p, u32 ctas, const u32 *tab, const void *kimg, u32 cxw, u32 be1w, u32 jobs,
                           void *trace, void *stream);
int wide_messages_per_cta_lanes();
int launch_modexp_wide_lanes(const ModexpParams &p, u32 ctas, const u32 *d_wide_tab, u32 k, u32 cxw, void *stream);
int launch_combine_wide(const CombineParams &p, const u32 *d_qinv, u32 *d_scratch, u32 k, void *stream);
int launch_mr_wide(const u32 *d_wide_tab, u32 k, u32 *d_pcw, u32 *d_scr, const u32 *d_n, const u32 *d_bases, u32 count,
                   u32 limbs, u32 rounds, u32 window, u32 forced, u32 *d_table, uint8_t *d_verdict, int16_t *d_witness,
                   int32_t *d_status, void *stream);
size_t mr_wide_table_words(u32 k, u32 window, u32 count);
int launch_mr_wide_setup(const u32 *d_wide_tab, u32 k, u32 *d_pcw, u32 *d_scr, const u32 *d_n, u32 count, u32 limbs,
                         uint8_t *d_verdict, void *stream);
size_t mr_wide_pcw_words(u32 k, u32 count);
size_t mr_wide_scr_words(u32 k, u32 count);

static const KernelSet &kernel_set_for(int k) {
    static std::vector<KernelSet> sets = {kernels_k1(),  kernels_k2(),  kernels_k3(),  kernels_k5(), kernels_k9(),
                                          kernels_k17(), kernels_k33(), kernels_k49(), kernels_k65(),
                                          kernels_k97(), kernels_k129()};
    for (const auto &s : sets)
        if (s.k == k) return s;
    return sets[0];
}
// k >= 97: the wide-operand kernel (mr_wide.cu, runtime k): 3072- (97), 4096- (129), 8192- (257), 16,128-bit (505)
// moduli (k = 97 / 129 keep their per-k kernel sets for Miller-Rabin)
static const int kSupportedK[] = {1, 2, 3, 5, 9, 17, 33, 49, 65, 97, 129, 257, 505};
static const int kNumK = sizeof(kSupportedK) / sizeof(kSupportedK[0]);

// ------------------------------------------------------------------ host positional helpers
typedef std::vector<u32> Big;  // little-endian limbs, trimmed (no high zero limbs)

static void trim(Big &a) {
    while (!a.empty() && a.back() == 0) a.pop_back();
}
static Big big_of(const u32 *p, size_t n) {
    Big a(p, p + n);
    trim(a);
    return a;
}
static int cmp(const Big &a, const Big &b) {
    if (a.size() != b.size()) return a.size() < b.size() ? -1 : 1;
    for (size_t i = a.size(); i-- > 0;)
        if (a[i] != b[i]) return a[i] < b[i] ? -1 : 1;
    return 0;
}
static Big add(const Big &a, const Big &b) {
    Big r(std::max(a.size(), b.size()) + 1, 0);
    u64 c = 0;
    for (size_t i = 0; i + 1 < r.size(); i++) {
        u64 s = c + (i < a.size() ? a[i] : 0) + (i < b.size() ? b[i] : 0);
        r[i] = (u32)s;
        c = s >> 32;
    }
    r.back() = (u32)c;
    trim(r);
    return r;
}
static Big sub(const Big &a, const Big &b) {  // a >= b
    Big r(a.size(), 0);
    u64 br = 0;
    for (size_t i = 0; i < a.size(); i++) {
        u64 bi = (i < b.size() ? b[i] : 0) + br;
        r[i] = (u32)((u64)a[i] - bi);
        br = (u64)a[i] < bi;
    }
    trim(r);
    return r;
}
static Big mul(const Big &a, const Big &b) {
    if (a.empty() || b.empty()) return Big();
    Big r(a.size() + b.size(), 0);
    for (size_t i = 0; i < a.size(); i++) {
        u64 c = 0;
        for (size_t j = 0; j < b.size(); j++) {
            u64 t = (u64)a[i] * b[j] + r[i + j] + c;
            r[i + j] = (u32)t;
            c = t >> 32;
        }
        r[i + b.size()] = (u32)c;
    }
    trim(r);
    return r;
}
static Big mul_word(const Big &a, u32 w) { return mul(a, Big{w}); }
static int bits(const Big &a) { return a.empty() ? 0 : 32 * (int)(a.size() - 1) + (32 - __builtin_clz(a.back())); }
static int bit(const Big &a, int i) { return (a[i / 32] >> (i % 32)) & 1; }
static Big mod(const Big &a, const Big &n) {  // bit-serial restoring reduction
    Big r;
    for (int i = bits(a) - 1; i >= 0; i--) {
        r = add(r, r);
        if (bit(a, i)) r = add(r, Big{1});
        if (cmp(r, n) >= 0) r = sub(r, n);
    }
    return r;
}
static u32 mod_word(const Big &a, u32 m) {
    u64 r = 0;
    for (size_t i = a.size(); i-- > 0;) r = ((r << 32) | a[i]) % m;
    return (u32)r;
}
static Big pow2(int e) {
    Big r(e / 32 + 1, 0);
    r[e / 32] = 1u << (e % 32);
    return r;
}

// ------------------------------------------------------------------ word arithmetic
static u32 mulm(u32 a, u32 b, u32 m) { return (u32)((u64)a * b % m); }
static u32 powm(u32 a, u64 e, u32 m) {
    u64 r = 1 % m, x = a % m;
    while (e) {
        if (e & 1) r = r * x % m;
        x = x * x % m;
        e >>= 1;
    }
    return (u32)r;
}
static u32 invp(u32 a, u32 p) { return powm(a % p, p - 2, p); }  // p prime (Fermat)
static u32 inv32(u32 a) {                                        // a odd: a^-1 mod 2^32 (Newton)
    u32 x = a;                                                   // correct to 3 bits
    for (int i = 0; i < 5; i++) x *= 2 - a * x;
    return x;
}
static bool is_prime32(u32 n) {  // deterministic Miller-Rabin for n < 2^32: bases 2, 7, 61
    if (n < 2) return false;
    for (u32 p : {2u, 3u, 5u, 7u, 11u, 13u, 61u})
        if (n % p == 0) return n == p;
    u32 d = n - 1;
    int s = 0;
    while (!(d & 1)) d >>= 1, s++;
    for (u32 a : {2u, 7u, 61u}) {
        u64 x = powm(a, d, n);
        if (x == 1 || x == n - 1) continue;
        bool comp = true;
        for (int r = 1; r < s; r++) {
            x = x * x % n;
            if (x == n - 1) { comp = false; break; }
        }
        if (comp) return false;
    }
    return true;
}

// reading R1: B = the k largest primes below 2^32 (descending), B' = the next k; for k <= 65 only primes
// m ≡ 3 (mod 4) are taken (-1 is then a non-residue, which the ρ-scaled tensor path needs, §4e)
static std::mutex g_mu;
static std::vector<u32> g_primes[2];   // [0] all primes, [1] primes ≡ 3 mod 4; descending from 2^32
static bool base_3mod4(int k) { return k <= 65; }
static const std::vector<u32> &primes_desc(size_t n, bool three_mod_four) {
    std::vector<u32> &g = g_primes[three_mod_four ? 1 : 0];
    if (g.size() < n) {
        u32 w = g.empty() ? 0xFFFFFFFFu : g.back() - 1;
        while (g.size() < n) {
            if ((!three_mod_four || (w & 3u) == 3u) && is_prime32(w)) g.push_back(w);
            w--;
        }
    }
    return g;
}

// ------------------------------------------------------------------ per-k base data
struct Base {
    int k = 0;
    std::vector<u32> B, Bp;        // moduli
    std::vector<u32> lambda;       // |M'_j^-1|_{m'_j}
    std::vector<u32> mu;           // |M^-1|_{m'_j}
    std::vector<u32> Mi_self;      // |M_i|_{m_i}
    u32 M_r = 0, Mp_r = 0;         // M, M' mod 2^32
    Big M, Mp;                     // products
    std::vector<u32> flat;         // constant-bank image (BaseLayout)
    std::vector<u32> pow;          // to_rns powers [k][2k]
    std::vector<u32> be;           // base-extension shared-memory image (mr_internal.h be_*)
};
static std::map<int, Base> g_bases;

static const Base &base_for(int k) {
    auto it = g_bases.find(k);
    if (it != g_bases.end()) return it->second;
    Base b;
    b.k = k;
    const std::vector<u32> &pr = primes_desc(2 * k, base_3mod4(k));
    b.B.assign(pr.begin(), pr.begin() + k);
    b.Bp.assign(pr.begin() + k, pr.begin() + 2 * k);
    b.M = Big{1};
    b.Mp = Big{1};
    for (u32 m : b.B) b.M = mul_word(b.M, m);
    for (u32 m : b.Bp) b.Mp = mul_word(b.Mp, m);
    b.M_r = b.M.empty() ? 0 : b.M[0];
    b.Mp_r = b.Mp[0];
    const BaseLayout L = base_layout(k);
    b.flat.assign(L.words, 0);
    u32 *f = b.flat.data();
    for (int i = 0; i < k; i++) {
        f[L.c + i] = 0u - b.B[i];
        f[L.c + k + i] = 0u - b.Bp[i];
    }
    for (int ch = 0; ch < 2 * k; ch++) f[L.c2 + ch] = f[L.c + ch] * f[L.c + ch];
    std::vector<u32> M_bp(k), Mp_b(k);
    for (int j = 0; j < k; j++) M_bp[j] = mod_word(b.M, b.Bp[j]);
    for (int i = 0; i < k; i++) Mp_b[i] = mod_word(b.Mp, b.B[i]);
    b.lambda.resize(k);
    b.mu.resize(k);
    b.Mi_self.resize(k);
    for (int j = 0; j < k; j++) {
        u32 Mpj = 1;
        for (int l = 0; l < k; l++)
            if (l != j) Mpj = mulm(Mpj, b.Bp[l] % b.Bp[j], b.Bp[j]);
        b.lambda[j] = invp(Mpj, b.Bp[j]);
        b.mu[j] = invp(M_bp[j], b.Bp[j]);
    }
    for (int i = 0; i < k; i++) {
        u32 Mi = 1;
        for (int l = 0; l < k; l++)
            if (l != i) Mi = mulm(Mi, b.B[l] % b.B[i], b.B[i]);
        b.Mi_self[i] = Mi;
    }
    for (int i = 0; i < k; i++) {
        for (int j = 0; j < k; j++) f[L.A1 + i * k + j] = mulm(M_bp[j], invp(b.B[i] % b.Bp[j], b.Bp[j]), b.Bp[j]);
        f[L.A1r + i] = b.M_r * inv32(b.B[i]);
    }
    for (int j = 0; j < k; j++) {
        for (int i = 0; i < k; i++) f[L.A2 + j * k + i] = mulm(Mp_b[i], invp(b.Bp[j] % b.B[i], b.B[i]), b.B[i]);
        f[L.A2r + j] = b.Mp_r * inv32(b.Bp[j]);
    }
    for (int j = 0; j < k; j++) f[L.C1 + j] = mulm(b.mu[j], invp(b.lambda[j], b.Bp[j]), b.Bp[j]);
    for (int i = 0; i < k; i++) f[L.pin + i] = (b.B[i] - Mp_b[i]) % b.B[i];
    f[L.misc + 0] = inv32(b.M_r);
    f[L.misc + 1] = inv32(b.Mp_r);
    for (int j = 0; j < k; j++) {
        Big Mpj{1};
        for (int l = 0; l < k; l++)
            if (l != j) Mpj = mul_word(Mpj, b.Bp[l]);
        for (int l = 0; l <= k; l++) f[L.MpL + j * (k + 1) + l] = l < (int)Mpj.size() ? Mpj[l] : 0;
    }
    {
        Big NMp = sub(pow2(32 * (k + 1)), b.Mp);
        for (int l = 0; l <= k; l++) f[L.NMp + l] = l < (int)NMp.size() ? NMp[l] : 0;
    }
    for (int i = 0; i < k; i++) f[L.MiS + i] = b.Mi_self[i];
    for (int j = 0; j < k; j++) f[L.MU + j] = b.mu[j];
    for (int i = 0; i < k; i++) f[L.ONE + i] = 1;
    for (int j = 0; j < k; j++) f[L.ONE + k + j] = b.lambda[j];
    f[L.ONE + 2 * k] = 1;
    for (int l = 0; l <= k; l++) f[L.ML + l] = l < (int)b.M.size() ? b.M[l] : 0;
    for (int ch = 0; ch < 2 * k; ch++) {
        const u32 m = ch < k ? b.B[ch] : b.Bp[ch - k];
        f[L.MM + ch] = m;
        f[L.MINV + ch] = 0u - inv32(m);
    }
    for (int j = 0; j < k; j++) {   // C1_j 2^64 mod m'_j  (2^32 ≡ c'_j = -m'_j mod 2^32)
        const u32 m = b.Bp[j], c = 0u - m;
        f[L.XW + j] = mulm(mulm(f[L.C1 + j], c, m), c, m);
    }
    if (tc_nt_mr(k) < (u32)k)   // the CUDA-core output column of the Miller-Rabin kernel's BE2
        for (int j = 0; j < k; j++) f[L.A2C + j] = f[L.A2 + j * k + tc_nt_mr(k)];   // |M'_j|_{m_TCNT}
    b.pow.assign((size_t)k * 2 * k, 0);
    for (int l = 0; l < k; l++) {
        Big p2 = pow2(32 * l);
        for (int i = 0; i < k; i++) b.pow[(size_t)l * 2 * k + i] = mod_word(p2, b.B[i]);
        for (int j = 0; j < k; j++)
            b.pow[(size_t)l * 2 * k + k + j] = mulm(mod_word(p2, b.Bp[j]), b.lambda[j], b.Bp[j]);
    }
    // base-extension image: BE1 tiles of A1[i][j] (columns j), then BE2 tiles of A2[j][i] (columns i)
    b.be.assign(be_words(k), 0);
    for (int half = 0; half < 2; half++) {
        const u32 *tab = f + (half ? L.A2 : L.A1);
        u32 *out = b.be.data() + half * be_half_words(k);
        const u32 ch = be_ch(k), nt = be_nfull(k) + (be_tail(k) ? 1 : 0);
        u32 off = 0;
        for (u32 t = 0; t < nt; t++) {
            const u32 w = t < be_nfull(k) ? ch : be_tail(k), pw = pad4(w);
            for (int i = 0; i < k; i++)
                for (u32 jj = 0; jj < w; jj++) out[off + i * pw + jj] = tab[i * k + t * ch + jj];
            off += k * pw;
        }
    }
    {
        u32 *v = b.be.data();
        for (int ch = 0; ch < 2 * k; ch++) {
            v[bev_c(k) + ch] = f[L.c + ch];
            v[bev_c2(k) + ch] = f[L.c2 + ch];
        }
        for (int i = 0; i < k; i++) {
            v[bev_C1(k) + i] = f[L.C1 + i];
            v[bev_pin(k) + i] = f[L.pin + i];
            v[bev_A1r(k) + i] = f[L.A1r + i];
            v[bev_A2r(k) + i] = f[L.A2r + i];
        }
    }
    return g_bases.emplace(k, std::move(b)).first->second;
}

// RNS image of a positional value x (B, B' in ξ-form, m_r)
static void to_rns_host(const Base &b, const Big &x, u32 *out) {
    const int k = b.k;
    for (int i = 0; i < k; i++) out[i] = mod_word(x, b.B[i]);
    for (int j = 0; j < k; j++) out[k + j] = mulm(mod_word(x, b.Bp[j]), b.lambda[j], b.Bp[j]);
    out[2 * k] = x.empty() ? 0 : x[0];
}

// Tensor-core B image (mr_internal.h tc_*): row (j, b), k byte (i, a) holds byte b of
// 2^(8a) A[i][j] mod m_j, where A[i][j] is the contraction constant of input i for output j.
// col0 (BE2): row (j, b), k byte 4k holds byte b of col0[j] = m_j - |M'|_{m_j} (times ρ_j on the scaled
// path); the kernel puts α' (< 2^7) in that A column, so the MMA adds the Shenoy-Kumaresan term.
// col1 (scaled BE1): k byte 4k + 1 holds byte b of col1[j], the constant offset of the sign-folded digits;
// the kernel keeps a 1 in that A column.
static void fill_tc_image(int k, int nt, const u32 *A /* [k][k], row i, column j */, const std::vector<u32> &mods,
                          uint8_t *out, const u32 *col0 = nullptr, const u32 *col1 = nullptr) {
    static_assert(tc_kp(33) >= 4 * 33 + 4 && tc_kp(65) >= 4 * 65 + 4, "a spare K byte column for α'");
    memset(out, 0, (size_t)tc_np_of((u32)nt) * tc_kp(k));
    for (int j = 0; j < nt; j++) {
        for (int i = 0; i < k; i++)
            for (int a = 0; a < 4; a++) {
                const u32 v = (u32)(((u64)A[i * k + j] << (8 * a)) % mods[j]);
                for (int b = 0; b < 4; b++) out[tc_off(k, 4 * j + b, 4 * i + a)] = (uint8_t)(v >> (8 * b));
            }
        if (col0)
            for (int b = 0; b < 4; b++) out[tc_off(k, 4 * j + b, 4 * k)] = (uint8_t)(col0[j] >> (8 * b));
        if (col1)
            for (int b = 0; b < 4; b++) out[tc_off(k, 4 * j + b, 4 * k + 1)] = (uint8_t)(col1[j] >> (8 * b));
    }
}

// device residency of per-k tables
struct DevBase {
    u32 *d_pow = nullptr;
    u32 *d_be = nullptr;
    u32 *d_mpl = nullptr;      // M'_j limbs [k][k+1] for the exit conversion
    u32 *d_tcb2 = nullptr;     // tensor-core BE2 image (k <= 64, and k = 65 in CTA-pair mode)
    u32 *d_tcb1u = nullptr;    // tensor-core unmerged BE1 image (Miller-Rabin, per-thread modulus)
    u32 *d_one = nullptr;      // RNS image of 1 (2k+1 words; Miller-Rabin tensor path multiplicand)
    u32 *d_wide = nullptr;     // wide-operand table (wide_path(k), mr_internal.h wide_layout)
    void *d_tcw = nullptr;     // tensor-core wide images (k = 97, 129: mr_internal.h tcw_*)
};

// per-k table of the wide kernel (mr_internal.h WideLayout): word-Montgomery constants with their 2^32
// factors folded in
static std::vector<u32> build_wide_table(const Base &b) {
    const int k = b.k;
    const BaseLayout L = base_layout(k);
    const WideLayout W = wide_layout(k);
    const u32 *f = b.flat.data();
    std::vector<u32> t(W.words, 0);
    for (int ch = 0; ch < 2 * k; ch++) {
        const u32 m = ch < k ? b.B[ch] : b.Bp[ch - k];
        t[W.mm + ch] = m;
        t[W.minv + ch] = 0u - inv32(m);
        t[W.r32 + ch] = (u32)((1ull << 32) % m);
    }
    for (int j = 0; j < k; j++) {
        const u32 m = b.Bp[j], r = t[W.r32 + k + j];
        t[W.xw + j] = mulm(mulm(f[L.C1 + j], r, m), r, m);
        t[W.a2r + j] = f[L.A2r + j];
    }
    for (int i = 0; i < k; i++) {
        t[W.a1r + i] = f[L.A1r + i];
        t[W.pinw + i] = mulm(f[L.pin + i], t[W.r32 + i], b.B[i]);
    }
    t[W.misc + 0] = f[L.misc + 0];
    t[W.misc + 1] = f[L.misc + 1];
    for (int j = 0; j < k; j++)
        for (int i = 0; i < k; i++) t[W.a2w + wch_at(j, i, k)] = mulm(f[L.A2 + j * k + i], t[W.r32 + i], b.B[i]);
    for (int l = 0; l < k; l++)
        for (int ch = 0; ch < 2 * k; ch++) {
            const u32 m = ch < k ? b.B[ch] : b.Bp[ch - k];
            t[W.pow + wch_at(l, ch, 2 * k)] = mulm(b.pow[(size_t)l * 2 * k + ch], t[W.r32 + ch], m);
        }
    for (int j = 0; j < k; j++)
        for (int l = 0; l <= k; l++) t[W.mpl + wch_at(j, l, k + 1)] = f[L.MpL + j * (k + 1) + l];
    for (int l = 0; l <= k; l++) t[W.nmp + l] = f[L.NMp + l];
    // Miller-Rabin (per-candidate n): unmerged BE1, the per-k vectors the setup needs, M limbs, the image of 1
    for (int i = 0; i < k; i++)
        for (int j = 0; j < k; j++) t[W.a1w + wch_at(i, j, k)] = mulm(f[L.A1 + i * k + j], t[W.r32 + k + j], b.Bp[j]);
    for (int j = 0; j < k; j++) {
        t[W.lam + j] = b.lambda[j];
        t[W.mu + j] = b.mu[j];
    }
    for (int i = 0; i < k; i++) t[W.mis + i] = b.Mi_self[i];
    for (int l = 0; l <= k; l++) t[W.ml + l] = f[L.ML + l];
    for (int c = 0; c < 2 * k + 1; c++) t[W.one + c] = f[L.ONE + c];
    return t;
}
static std::map<std::pair<int, int>, DevBase> g_devbases;

// modexp / CRT contexts that run on the wide-operand kernel (mr_wide.cu): every k >= 97.  At k = 97 / 129
// the per-k IMAD kernel fits only 128 / 64 messages (4 / 2 warps per SM) next to its 75 / 136 KB shared-
// memory base-extension image; the wide kernel runs 16 warps per SM with the images streamed from L2
// (A/B in DESIGN.md §4h).  Miller-Rabin at k = 97 / 129 keeps the per-k kernel (is_wide stays k > 129).
// MR_RNS_WIDE_MIN=k' moves the threshold (A/B hook; 999 = per-k kernels up to 129).
static bool wide_path(int k) {
    if (is_wide((u32)k)) return true;
    static const int kmin = [] { const char *e = getenv("MR_RNS_WIDE_MIN"); return e ? atoi(e) : 97; }();
    return k >= 97 && k >= kmin;
}

// Small-batch path: narrow k whose contexts also carry the wide section, so a batch too small
// to fill the SMs with 128-message tensor tiles runs on the channels-on-threads kernel with one message per
// CTA (mr_lanes.cu).  MR_RNS_SMALL_MAX = the largest count x contexts that takes it (0 disables it).
static bool small_ok(int k) { return k >= 17 && k <= 65; }
static long g_small_override = -1;   // mr_internal_set_small_max (tests: both paths at the same batch size)
static size_t small_max() {
    static const size_t v = [] { const char *e = getenv("MR_RNS_SMALL_MAX"); return e ? (size_t)atol(e) : (size_t)1024; }();
    return g_small_override >= 0 ? (size_t)g_small_override : v;
}

static std::vector<uint8_t> build_tcw_images(const Base &b);

static int ensure_device_base(int k, int device, const u32 **d_pow, const u32 **d_be) {
    auto key = std::make_pair(device, k);
    auto it = g_devbases.find(key);
    if (it != g_devbases.end()) {
        *d_pow = it->second.d_pow;
        *d_be = it->second.d_be;
        return MR_OK;
    }
    const Base &b = base_for(k);
    if (cudaSetDevice(device) != cudaSuccess) return MR_ERR_CUDA;
    {   // scratch (window tables, CRT halves) is stream-ordered: keep freed blocks in the device's
        // default pool instead of returning them to the OS at every synchronisation
        cudaMemPool_t pool;
        if (cudaDeviceGetDefaultMemPool(&pool, device) == cudaSuccess) {
            uint64_t keep = UINT64_MAX;
            cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &keep);
        }
    }
    DevBase db;
    if (wide_path(k) || small_ok(k)) {   // wide-operand / small-batch kernel: one table in HBM
        const std::vector<u32> t = build_wide_table(b);
        if (cudaMalloc(&db.d_wide, t.size() * 4) != cudaSuccess) return MR_ERR_NOMEM;
        if (cudaMemcpy(db.d_wide, t.data(), t.size() * 4, cudaMemcpyHostToDevice) != cudaSuccess) return MR_ERR_CUDA;
    }
    if (wide_path(k) && tcw_k((u32)k)) {
        const std::vector<uint8_t> im = build_tcw_images(b);
        if (cudaMalloc(&db.d_tcw, im.size()) != cudaSuccess) return MR_ERR_NOMEM;
        if (cudaMemcpy(db.d_tcw, im.data(), im.size(), cudaMemcpyHostToDevice) != cudaSuccess) return MR_ERR_CUDA;
    }
    if (is_wide((u32)k)) {   // no per-k kernel set
        g_devbases[key] = db;
        *d_pow = nullptr;
        *d_be = nullptr;
        return MR_OK;
    }
    const KernelSet &ks = kernel_set_for(k);
    if (ks.upload_base(b.flat.data(), device) != 0) return MR_ERR_CUDA;
    if (cudaMalloc(&db.d_pow, b.pow.size() * 4) != cudaSuccess) return MR_ERR_NOMEM;
    if (cudaMemcpy(db.d_pow, b.pow.data(), b.pow.size() * 4, cudaMemcpyHostToDevice) != cudaSuccess)
        return MR_ERR_CUDA;
    {
        const BaseLayout L = base_layout(k);
        const size_t n = (size_t)k * (k + 1);
        if (cudaMalloc(&db.d_mpl, n * 4) != cudaSuccess) return MR_ERR_NOMEM;
        if (cudaMemcpy(db.d_mpl, b.flat.data() + L.MpL, n * 4, cudaMemcpyHostToDevice) != cudaSuccess) return MR_ERR_CUDA;
    }
    if (cudaMalloc(&db.d_one, (2 * (size_t)k + 1) * 4) != cudaSuccess) return MR_ERR_NOMEM;
    if (cudaMemcpy(db.d_one, b.flat.data() + base_layout(k).ONE, (2 * (size_t)k + 1) * 4, cudaMemcpyHostToDevice) !=
        cudaSuccess)
        return MR_ERR_CUDA;
    if (cudaMalloc(&db.d_be, b.be.size() * 4) != cudaSuccess) return MR_ERR_NOMEM;
    if (cudaMemcpy(db.d_be, b.be.data(), b.be.size() * 4, cudaMemcpyHostToDevice) != cudaSuccess)
        return MR_ERR_CUDA;
    if (tc_ok(k)) {   // tensor BE2 image of A2 as [input j][output i]
        const u32 *A2 = b.flat.data() + base_layout(k).A2;   // row j, column i
        std::vector<uint8_t> img(tc_bbytes_mr(k));   // the per-k images serve the Miller-Rabin kernel
        if (4 * k + 4 > (int)tc_kp(k)) return MR_ERR_ARG;   // no spare K column for α' (not a supported k)
        fill_tc_image(k, (int)tc_nt_mr(k), A2, b.B, img.data(), b.flat.data() + base_layout(k).pin);
        if (cudaMalloc(&db.d_tcb2, img.size()) != cudaSuccess) return MR_ERR_NOMEM;
        if (cudaMemcpy(db.d_tcb2, img.data(), img.size(), cudaMemcpyHostToDevice) != cudaSuccess) return MR_ERR_CUDA;
        fill_tc_image(k, (int)tc_nt_mr(k), b.flat.data() + base_layout(k).A1, b.Bp, img.data());
        if (cudaMalloc(&db.d_tcb1u, img.size()) != cudaSuccess) return MR_ERR_NOMEM;
        if (cudaMemcpy(db.d_tcb1u, img.data(), img.size(), cudaMemcpyHostToDevice) != cudaSuccess) return MR_ERR_CUDA;
    }
    g_devbases[key] = db;
    *d_pow = db.d_pow;
    *d_be = db.d_be;
    return MR_OK;
}

// capacity: 4 (k+3)^2 N < M and 4 (k+3) N < M'; for k <= 65 (tensor path: sign-folded
// digits up to 2 m_i, §4e) values stay below (2k+3) N, so the bound uses 2k+3
static bool fits(const Base &b, const Big &N) {
    const u32 kk = b.k <= 65 ? 2 * (u32)b.k + 3 : (u32)b.k + 3;
    Big lhs = mul_word(mul_word(N, 4 * kk), kk);
    Big lhs2 = mul_word(N, 4 * kk);
    return cmp(lhs, b.M) < 0 && cmp(lhs2, b.Mp) < 0;
}

// largest b such that every modulus below 2^b passes fits() for this base (mr_rns_ctx_info)
static int max_modulus_bits(const Base &b) {
    for (int nb = 32 * b.k; nb > 1; nb--) {
        Big t((size_t)(nb + 31) / 32, 0xFFFFFFFFu);
        if (nb % 32) t.back() = (1u << (nb % 32)) - 1u;
        if (fits(b, t)) return nb;
    }
    return 1;
}

static int auto_k(const Big &N, int min_k) {
    for (int i = 0; i < kNumK; i++) {
        int k = kSupportedK[i];
        if (k < min_k) continue;
        if (fits(base_for(k), N)) return k;
    }
    return -1;
}

}  // namespace mr

using namespace mr;

struct DevProg {
    u64 *d_ops = nullptr;
    u32 nops = 0;
    int w = 1;
    bool transient = false;    // not cached: stream-ordered allocation, freed by release_prog after the launch
};

struct mr_rns_ctx {
    int k = 0, device = 0;
    size_t limbs = 0;
    int bits = 0;
    int max_bits = 0;          // capacity of this k's base pair (admission test of DESIGN.md §3)
    Big N;
    u32 *d_cx = nullptr;       // device context block
    const u32 *d_pow = nullptr;
    const u32 *d_be = nullptr;
    const u32 *d_tcb2 = nullptr;
    const u32 *d_mpl = nullptr;
    const u32 *d_wide = nullptr;   // wide-operand table of this k (wide_path(k) or small_ok(k))
    u32 cxw = 0;                   // word offset of the wide section in the context block (0: none)
    u32 be1w = 0;                  // word offset of the tensor-core wide BE1 image (k = 97 / 129; 0: none)
    const void *d_tcw = nullptr;   // per-k tensor-core wide images (BE2 | TRN | EXT)
    std::vector<u32> h_cx;
    std::mutex mu;             // guards the program cache
    std::map<std::pair<Big, bool>, DevProg> progs;  // (exponent, crt) -> uploaded program (<= kProgCache)
    cudaStream_t upload = nullptr;                   // private stream for program uploads
};

struct mr_rsa_priv {
    mr_rns_ctx *cp = nullptr, *cq = nullptr;
    size_t half = 0;
    Big dp, dq;
    u32 *d_q = nullptr;        // q limbs on device
    u32 *d_qinv = nullptr;     // q^-1 mod p limbs on device (wide halves: positional recombination)
};

// the per-context constant block of DESIGN.md §3 (layout cx_* in mr_internal.h)
static void fill_ctx_block(const Base &b, const Big &N, size_t limbs, const Big &in_bound, size_t in_limbs,
                           const Big *khi_half, const Big *qinv, u32 *x) {
    const int k = b.k;
    x[CX_K] = k;
    x[CX_LIMBS] = (u32)limbs;
    x[CX_INLIMBS] = (u32)in_limbs;
    x[CX_NMINV_R] = N[0] * inv32(b.M_r);                        // N M^-1 mod 2^32
    for (int i = 0; i < k; i++) {                               // σ_i = |-N^-1 M_i^-1|_{m_i}
        u32 Ni = mod_word(N, b.B[i]);
        u32 inv = invp(mulm(Ni, b.Mi_self[i], b.B[i]), b.B[i]);
        x[cx_sigma(k) + i] = (b.B[i] - inv) % b.B[i];
    }
    for (int j = 0; j < k; j++) {                               // |N M^-1 λ_j|_{m'_j}
        u32 Nj = mod_word(N, b.Bp[j]);
        x[cx_c2(k) + j] = mulm(mulm(Nj, b.mu[j], b.Bp[j]), b.lambda[j], b.Bp[j]);
    }
    Big Rm = mod(b.M, N);                                       // R = M ("By choosing R = M")
    Big R2 = mod(mul(Rm, Rm), N);
    to_rns_host(b, R2, x + cx_r2(k));
    to_rns_host(b, Big{1}, x + cx_one(k));
    if (khi_half) {  // 2^(32 half) R^2 mod N: enters the high half of a CRT ciphertext (a3)
        int half = (int)(*khi_half)[0];
        to_rns_host(b, mod(mul(pow2(32 * half), R2), N), x + cx_khi(k));
    }
    if (qinv) to_rns_host(b, mod(mul(*qinv, Rm), N), x + cx_qinvr(k));  // mm(diff, .) = diff qinv mod p
    for (int l = 0; l <= k && l < (int)N.size(); l++) x[cx_n(k) + l] = N[l];
    for (int l = 0; l < 2 * k + 2 && l < (int)in_bound.size(); l++) x[cx_inb(k) + l] = in_bound[l];
}

// Per-context BE1 image with 6.4 merged into the contraction: the tile layout of
// mr_internal.h be_* holding A1'[i][j] = |M_i|_{m'_j} · |N M^-1 λ_j|_{m'_j} mod m'_j, so that
// ξ'_j = t*_j |M^-1 λ_j^-1| + Σ_i ξ_i A1'[i][j] needs one reduction.
static void fill_merged_be1(const Base &b, u32 *out, const u32 *cx) {
    const int k = b.k;
    const BaseLayout L = base_layout(k);
    const u32 *A1 = b.flat.data() + L.A1;
    const u32 ch = be_ch(k), nt = be_nfull(k) + (be_tail(k) ? 1 : 0);
    u32 off = 0;
    for (u32 t = 0; t < nt; t++) {
        const u32 w = t < be_nfull(k) ? ch : be_tail(k), pw = pad4(w);
        for (int i = 0; i < k; i++)
            for (u32 jj = 0; jj < w; jj++) {
                const u32 j = t * ch + jj;
                out[off + i * pw + jj] = mulm(A1[i * k + j], cx[cx_c2(k) + j], b.Bp[j]);
            }
        off += k * pw;
    }
}

// Tensor-core (ρ-scaled) part of a context, after fill_ctx_block and fill_merged_be1.
// The tensor path reduces channel products with word Montgomery reductions (result T·2^-32 mod m), so
// the constants absorb R32 = 2^32 mod m = c: ε_i = Legendre(σ_i c_i | m_i), ρ_i = (ε_i σ_i c_i)^((m_i+1)/4)
// (m_i ≡ 3 mod 4, so ρ_i² = ε_i σ_i c_i); the scaled constant vectors, the sign-folded BE1 image (× c'_j)
// with its offset column, the ρ-scaled BE2 image (× c_i) with the α' column, the CUDA-core output
// column vectors (plain red96, no R32) and the epilogue constants.
static bool fill_tc_scaled(const Base &b, u32 *x) {
    const int k = b.k;
    const BaseLayout L = base_layout(k);
    const u32 *A1 = b.flat.data() + L.A1, *A2 = b.flat.data() + L.A2, *pin = b.flat.data() + L.pin;
    const int nt = (int)tc_nt(k);
    std::vector<u32> rho(k), v(k);
    std::vector<int> neg(k);
    for (int i = 0; i < k; i++) {
        const u32 m = b.B[i], s = mulm(x[cx_sigma(k) + i], 0u - m, m);   // σ_i c_i, c_i = 2^32 mod m_i
        neg[i] = powm(s, (m - 1) / 2, m) != 1;                  // σ_i c_i a non-residue: use -σ_i c_i
        v[i] = neg[i] ? (m - s) % m : s;                         // v_i = ε_i σ_i c_i = ρ_i²
        rho[i] = powm(v[i], ((u64)m + 1) / 4, m);
        if ((m & 3u) != 3u || mulm(rho[i], rho[i], m) != v[i]) return false;
    }
    // constants: [0] R2 twice-scaled (operand right after to_rns), [1] ONE scaled, [2] KHI twice-scaled,
    // [3] R2 scaled (loaded as an accumulator); B' and m_r channels unchanged
    const u32 srcs[4] = {cx_r2(k), cx_one(k), cx_khi(k), cx_r2(k)};
    for (int t = 0; t < 4; t++) {
        u32 *dst = x + cx_sc(k) + t * (2 * k + 1);
        const u32 *src = x + srcs[t];
        for (int ch = 0; ch <= 2 * k; ch++) dst[ch] = src[ch];
        for (int i = 0; i < k; i++) dst[i] = mulm(src[i] % b.B[i], (t == 1 || t == 3) ? rho[i] : v[i], b.B[i]);
    }
    // merged BE1 constants A1'[i][j] = |M_i|_{m'_j} |N M^-1 λ_j|, signed by ε_i; offsets Σ_{ε_i = -1} m_i A1'[i][j]
    std::vector<u32> A1s((size_t)k * k), off(k, 0);
    const u32 *c2 = x + cx_c2(k);
    u32 qr_off = 0;
    for (int i = 0; i < k; i++) {
        for (int j = 0; j < k; j++) {
            const u32 mj = b.Bp[j], a = mulm(A1[i * k + j], c2[j], mj);
            A1s[(size_t)i * k + j] = neg[i] ? (mj - a) % mj : a;
            // ε_i = -1: the digit is 2 m_i - ξ̂_i (lazy ξ̂_i < 2^32 keeps it positive): offset 2 m_i A1'[i][j]
            if (neg[i]) off[j] = (u32)(((u64)off[j] + mulm((u32)(2ull * b.B[i] % mj), a, mj)) % mj);
        }
        const u32 a1r = b.flat[L.A1r + i];
        x[cx_a1x(k) + 2 * i] = neg[i] ? 0u - a1r : a1r;
        if (neg[i]) qr_off += 2u * b.B[i] * a1r;
        if (nt < k) x[cx_a1x(k) + 2 * i + 1] = A1s[(size_t)i * k + nt];
    }
    x[cx_scv(k) + 0] = qr_off;
    if (nt < k) {   // CUDA-core output (plain red96): its t* carries 2^-32, so C1 is taken times c'
        x[cx_scv(k) + 1] = off[nt];
        x[cx_scv(k) + 2] = rho[nt];   // the CUDA-core BE2 output is formed unscaled, then × ρ_TCNT
        x[cx_scv(k) + 3] = mulm(b.flat[L.C1 + nt], 0u - b.Bp[nt], b.Bp[nt]);
        for (int j = 0; j < k; j++) x[cx_a2s(k) + j] = mulm(A2[j * k + nt], rho[nt], b.B[nt]);
    }
    for (int j = 0; j < k; j++) {   // BE1 epilogue: ξ'_j = mont(t*_j · C1_j c'^2 + V'_j), V' carries × c'
        const u32 mj = b.Bp[j], cj = 0u - mj;
        x[cx_ep1(k) + 4 * j + 0] = mj;
        x[cx_ep1(k) + 4 * j + 1] = 0u - inv32(mj);
        x[cx_ep1(k) + 4 * j + 2] = mulm(mulm(b.flat[L.C1 + j], cj, mj), cj, mj);
        x[cx_ep1(k) + 4 * j + 3] = b.flat[L.A2r + j];
    }
    for (int i = 0; i < k; i++) {   // BE2 epilogue: s_i = mont(V_i), V carries × c_i
        x[cx_ep2(k) + 2 * i + 0] = b.B[i];
        x[cx_ep2(k) + 2 * i + 1] = 0u - inv32(b.B[i]);
    }
    const size_t tcw = tc_bbytes(k) / 4;
    uint8_t *img1 = reinterpret_cast<uint8_t *>(x + cx_words(k) + be_half_words(k));
    std::vector<u32> A1t((size_t)k * k), offt(k);   // tensor copies × c'_j (the Montgomery factor)
    for (int j = 0; j < k; j++) {
        const u32 mj = b.Bp[j], cj = 0u - mj;
        for (int i = 0; i < k; i++) A1t[(size_t)i * k + j] = mulm(A1s[(size_t)i * k + j], cj, mj);
        offt[j] = mulm(off[j], cj, mj);
    }
    fill_tc_image(k, nt, A1t.data(), b.Bp, img1, nullptr, offt.data());
    // BE2: |M'_j|_{m_i} ρ_i c_i (row j, column i) and the α' column (m_i - |M'|_{m_i}) ρ_i c_i
    std::vector<u32> A2s((size_t)k * k), pins(k);
    for (int j = 0; j < k; j++)
        for (int i = 0; i < k; i++)
            A2s[(size_t)j * k + i] = mulm(mulm(A2[j * k + i], rho[i], b.B[i]), 0u - b.B[i], b.B[i]);
    for (int i = 0; i < k; i++) pins[i] = mulm(mulm(pin[i], rho[i], b.B[i]), 0u - b.B[i], b.B[i]);
    fill_tc_image(k, nt, A2s.data(), b.B, reinterpret_cast<uint8_t *>(x + cx_words(k) + be_half_words(k) + tcw),
                  pins.data());
    return true;
}

// per-context part of the wide kernel's constants (mr_internal.h wide_cx_*): σ_i 2^64 mod m_i and
// A1'[i][j] 2^32 mod m'_j, A1' = |M_i|_{m'_j} |N M^-1 λ_j| (6.4 merged into BE1, row-major)
static void fill_wide_ctx(const Base &b, u32 *x, u32 cxw) {
    const int k = b.k;
    const u32 *A1 = b.flat.data() + base_layout(k).A1;
    u32 *w = x + cxw;
    for (int i = 0; i < k; i++) {
        const u32 m = b.B[i], r = (u32)((1ull << 32) % m);
        w[wide_cx_sig(k) + i] = mulm(mulm(x[cx_sigma(k) + i], r, m), r, m);
    }
    for (int j = 0; j < k; j++) {
        const u32 m = b.Bp[j], r = (u32)((1ull << 32) % m), nu = mulm(x[cx_c2(k) + j], r, m);
        for (int i = 0; i < k; i++) w[wide_cx_a1(k) + wch_at(i, j, k)] = mulm(A1[i * k + j], nu, m);
    }
}

// ------------------------------------------------------------------ tensor-core wide kernel images (§4k)
namespace mr {
// Byte-split image of a modular contraction (mr_internal.h tcw_*): row (output o, byte b), K byte (input word i,
// byte a) holds byte b of C(i, a, o) = 2^(8a) A(i, o) mod m_o, so Σ_b 2^(8b) D[(o, b)] ≡ Σ_i x_i A(i, o) (mod m_o).
// `coef(i, o)` returns A(i, o) already reduced (< m_o), `mod(o)` m_o (0 = 2^32: the m_r column), `nin` inputs.
template <class Coef, class Mod>
static void fill_tcw_modular(int k, u32 e, int nin, Coef &&coef, Mod &&modo, uint8_t *img) {
    memset(img, 0, tcw_img_bytes(k, e));
    const u32 nout = tcw_nout(k, e), oc = tcw_oc(k, e);
    for (u32 o = 0; o < nout; o++) {
        const u32 c = o / oc, rl = 4 * (o - c * oc);
        const u64 m = modo(o);
        for (int i = 0; i < nin; i++) {
            const u64 A = coef(i, o);
            for (u32 a = 0; a < 4; a++) {
                const u32 v = m ? (u32)((A << (8 * a)) % m) : (u32)(A << (8 * a));
                for (u32 b = 0; b < 4; b++) img[tcw_at(k, e, c, rl + b, 4 * i + a)] = (uint8_t)(v >> (8 * b));
            }
        }
    }
}
static u32 r32_of(u32 m) { return (u32)((1ull << 32) % m); }
// per-context BE1: A(i, j) = A1'_ij 2^32 mod m'_j (6.4 merged; the epilogue folds t*_j C1_j 2^64 + D_j with one
// Montgomery reduction), and the m_r column A(i, k) = |M_i|_{2^32}
static void fill_tcw_be1(const Base &b, const u32 *cx, uint8_t *img) {
    const int k = b.k;
    const u32 *A1 = b.flat.data() + base_layout(k).A1, *A1r = b.flat.data() + base_layout(k).A1r;
    fill_tcw_modular(k, TCW_BE1, k,
        [&](int i, u32 j) -> u64 {
            if ((int)j == k) return A1r[i];
            const u32 m = b.Bp[j], r = r32_of(m);
            return mulm(mulm(A1[i * k + j], cx[cx_c2(k) + j], m), r, m);
        },
        [&](u32 j) -> u64 { return (int)j == k ? 0 : b.Bp[j]; }, img);
}
// per-k BE2 (A2_ji 2^32, α' column (m_i - |M'|_{m_i}) 2^32 at input word k), TRN (|2^(32l)|_{m_c} 2^32, B' × λ_j),
// EXT (byte convolution with M'_j and 2^(32(k+1)) - M')
static std::vector<uint8_t> build_tcw_images(const Base &b) {
    const int k = b.k;
    const BaseLayout L = base_layout(k);
    const u32 *f = b.flat.data();
    std::vector<uint8_t> img(tcw_kimg_bytes(k), 0);
    fill_tcw_modular(k, TCW_BE2, k + 1,
        [&](int j, u32 i) -> u64 {
            const u32 m = b.B[i], r = r32_of(m);
            return j < k ? mulm(f[L.A2 + j * k + i], r, m) : mulm(f[L.pin + i], r, m);
        },
        [&](u32 i) -> u64 { return b.B[i]; }, img.data() + tcw_img_off(k, TCW_BE2));
    fill_tcw_modular(k, TCW_TRN, k,
        [&](int l, u32 c) -> u64 {
            const u32 m = (int)c < k ? b.B[c] : b.Bp[c - k];
            return mulm(b.pow[(size_t)l * 2 * k + c], r32_of(m), m);
        },
        [&](u32 c) -> u64 { return (int)c < k ? b.B[c] : b.Bp[c - k]; }, img.data() + tcw_img_off(k, TCW_TRN));
    {   // EXT: row p = byte position of X (4 per limb), K byte (j, a): byte p - a of M'_j (j < k) or of 2^(32(k+1)) - M'
        uint8_t *x = img.data() + tcw_img_off(k, TCW_EXT);
        const u32 oc = tcw_oc(k, TCW_EXT);
        auto byte_of = [&](int j, int q) -> uint8_t {   // byte q of M'_j (j < k) / of NMp (j = k)
            if (q < 0 || q >= 4 * (k + 1)) return 0;
            const u32 w = j < k ? f[L.MpL + j * (k + 1) + q / 4] : f[L.NMp + q / 4];
            return (uint8_t)(w >> (8 * (q % 4)));
        };
        for (u32 l = 0; l <= (u32)k; l++) {
            const u32 c = l / oc, rl = 4 * (l - c * oc);
            for (u32 bb = 0; bb < 4; bb++) {
                const int p = 4 * (int)l + (int)bb;
                for (int j = 0; j <= k; j++)
                    for (int a = 0; a < 4; a++) x[tcw_at(k, TCW_EXT, c, rl + bb, 4 * j + a)] = byte_of(j, p - a);
            }
        }
    }
    return img;
}
}  // namespace mr

static int build_ctx(mr_rns_ctx **out, const Big &N, size_t limbs, int k_req, int device, const Big &in_bound,
                     size_t in_limbs, const Big *khi_shift_limbs_half /* CRT: half limbs */, const Big *qinv) {
    *out = nullptr;
    if (N.empty() || !(N[0] & 1) || (N.size() == 1 && N[0] < 3)) return MR_ERR_EVEN_MODULUS;
    int k;
    {
        std::lock_guard<std::mutex> lk(g_mu);
        int kmin = 1;
        if (k_req > 0) {
            kmin = -1;
            for (int i = 0; i < kNumK; i++)
                if (kSupportedK[i] >= k_req) { kmin = kSupportedK[i]; break; }
            if (kmin < 0) return MR_ERR_ARG;
            if (!fits(base_for(kmin), N)) return MR_ERR_CAPACITY;
        }
        k = auto_k(N, kmin);
        if (k < 0) return MR_ERR_CAPACITY;
    }
    if (limbs > (size_t)k || in_limbs > (size_t)(2 * k + 2)) return MR_ERR_CAPACITY;
    std::lock_guard<std::mutex> lk(g_mu);
    const Base &b = base_for(k);
    for (u32 m : b.B)
        if (mod_word(N, m) == 0) return MR_ERR_NOT_COPRIME;
    for (u32 m : b.Bp)
        if (mod_word(N, m) == 0) return MR_ERR_NOT_COPRIME;
    mr_rns_ctx *c = new (std::nothrow) mr_rns_ctx;
    if (!c) return MR_ERR_NOMEM;
    c->k = k;
    c->device = device;
    c->limbs = limbs;
    c->bits = bits(N);
    c->max_bits = max_modulus_bits(b);
    c->N = N;
    const size_t tc_words = tc_ok(k) ? tc_bbytes(k) / 4 : 0;
    int rc = MR_OK;
    if (wide_path(k)) {   // cx block + wide section (σ 2^64, A1' 2^32 row-major) [+ tensor BE1 image, k = 97 / 129]
        const size_t tcw = tcw_k((u32)k) ? tcw_cx_words((u32)k) : 0;
        c->h_cx.assign(cx_words(k) + wide_cx_words(k) + tcw, 0);
        fill_ctx_block(b, N, limbs, in_bound, in_limbs, khi_shift_limbs_half, qinv, c->h_cx.data());
        c->cxw = cx_words(k);
        fill_wide_ctx(b, c->h_cx.data(), c->cxw);
        if (tcw) {
            c->be1w = cx_words(k) + wide_cx_words(k);
            fill_tcw_be1(b, c->h_cx.data(), reinterpret_cast<uint8_t *>(c->h_cx.data() + c->be1w));
        }
    } else {   // narrow layout; small-batch k append the wide section after the tensor images
        const size_t narrow = cx_words(k) + be_half_words(k) + 2 * tc_words;
        c->h_cx.assign(narrow + (small_ok(k) ? wide_cx_words(k) : 0), 0);
        fill_ctx_block(b, N, limbs, in_bound, in_limbs, khi_shift_limbs_half, qinv, c->h_cx.data());
        fill_merged_be1(b, c->h_cx.data() + cx_words(k), c->h_cx.data());
        if (small_ok(k)) {
            c->cxw = (u32)narrow;
            fill_wide_ctx(b, c->h_cx.data(), c->cxw);
        }
    }
    if (tc_ok(k) && !fill_tc_scaled(b, c->h_cx.data())) rc = MR_ERR_ARG;   // not reachable for the R1 bases
    if (rc == MR_OK) rc = ensure_device_base(k, device, &c->d_pow, &c->d_be);
    if (rc == MR_OK) {
        c->d_tcb2 = g_devbases[std::make_pair(device, k)].d_tcb2;
        c->d_mpl = g_devbases[std::make_pair(device, k)].d_mpl;
        c->d_wide = g_devbases[std::make_pair(device, k)].d_wide;
        c->d_tcw = g_devbases[std::make_pair(device, k)].d_tcw;
    }
    if (rc != MR_OK) { delete c; return rc; }
    if (cudaSetDevice(device) != cudaSuccess) { delete c; return MR_ERR_CUDA; }
    if (cudaMalloc(&c->d_cx, c->h_cx.size() * 4) != cudaSuccess) { delete c; return MR_ERR_NOMEM; }
    if (cudaMemcpy(c->d_cx, c->h_cx.data(), c->h_cx.size() * 4, cudaMemcpyHostToDevice) != cudaSuccess) {
        cudaFree(c->d_cx);
        delete c;
        return MR_ERR_CUDA;
    }
    *out = c;
    return MR_OK;
}

// ------------------------------------------------------------------ optional per-launch CUDA-event timing
// (bench hook: records an event pair around each kernel on the stream it is launched on)
namespace mr {
struct EvPair {
    cudaEvent_t a, b;
    int kind;  // 0 ladder (k_modexp), 1 combine, 2 Miller-Rabin (setup + rounds)
};
static std::mutex g_tmu;
static int g_timing = 0;
static std::vector<EvPair> g_events;
static double g_last_mr_ms = 0;
static int g_last_mr_n = 0;

template <class F>
static int timed_launch(int kind, cudaStream_t st, F &&launch) {
    int on;
    {
        std::lock_guard<std::mutex> lk(g_tmu);
        on = g_timing;
    }
    if (!on) return launch();
    EvPair e;
    e.kind = kind;
    cudaEventCreate(&e.a);
    cudaEventCreate(&e.b);
    cudaEventRecord(e.a, st);
    int rc = launch();
    cudaEventRecord(e.b, st);
    std::lock_guard<std::mutex> lk(g_tmu);
    g_events.push_back(e);
    return rc;
}
}  // namespace mr

// ------------------------------------------------------------------ exponent -> program (R6)
namespace mr {
struct Ladder {
    int w = 1;
    std::vector<u64> ops;
};

// sliding-window recoding of E (HAC Alg. 14.85 shape), window w: appends ladder ops that start
// with acc = x̃^(first window) loaded from the table; table slot i holds x̃^(2i+1).
static int sliding_ops(const Big &E, int w, std::vector<u64> *ops) {
    int n = 0;
    bool first = true;
    int i = bits(E) - 1;
    while (i >= 0) {
        if (!bit(E, i)) {
            if (ops) ops->push_back(make_op(0, OPND_SQ));
            n++;
            i--;
            continue;
        }
        int l = std::max(i - w + 1, 0);
        while (!bit(E, l)) l++;
        u32 v = 0;
        for (int t = i; t >= l; t--) v = (v << 1) | (u32)bit(E, t);
        if (first) {
            if (ops) ops->push_back(make_op(OPF_LOAD | OPF_NOMUL, 0, (v - 1) / 2));
            first = false;
        } else {
            for (int t = i; t >= l; t--) {
                if (ops) ops->push_back(make_op(0, OPND_SQ));
                n++;
            }
            if (ops) ops->push_back(make_op(0, (v - 1) / 2));
            n++;
        }
        i = l - 1;
    }
    return n;
}

static int table_cost(int w) { return w > 1 ? (1 << (w - 1)) : 0; }

static int best_window(const Big &E) {
    int best = 1, bestc = 1 << 30;
    // MR_RNS_WMAX=w: cap the sliding window (A/B hook: a smaller window table stays in L2 longer)
    static const int wmax = [] { const char *e = getenv("MR_RNS_WMAX"); const int v = e ? atoi(e) : 7; return v < 1 ? 1 : (v > 7 ? 7 : v); }();
    for (int w = 1; w <= wmax; w++) {
        int c = table_cost(w) + sliding_ops(E, w, nullptr);
        if (c < bestc) bestc = c, best = w;
    }
    return best;
}

// full program: entry (plain or CRT), table, ladder, exit multiply by 1
static Ladder build_program(const Big &E, bool crt) {
    Ladder L;
    if (E.empty()) {  // x^0 = 1: acc = R^2 · 1 / M = R (Montgomery one), then the exit multiply
        L.w = 1;
        L.ops.push_back(make_op(OPF_LOAD | OPF_NOMUL, 0, OPND_R2));
        L.ops.push_back(make_op(0, OPND_ONE));
        L.ops.push_back(make_op(0, OPND_ONE));
        return L;
    }
    L.w = best_window(E);
    const u32 S = 1u << (L.w - 1);  // scratch slot (x̃^2, CRT high half)
    if (crt) {
        L.ops.push_back(make_op(OPF_TORNS_HI | OPF_STORE, OPND_KHI, 0, 0, S));
        L.ops.push_back(make_op(OPF_TORNS_LO | OPF_ADD | OPF_STORE, OPND_R2, 0, S, 0));
    } else {
        L.ops.push_back(make_op(OPF_TORNS_ALL | OPF_STORE, OPND_R2, 0, 0, 0));
    }
    if (L.w > 1) {
        L.ops.push_back(make_op(OPF_STORE, OPND_SQ, 0, 0, S));
        for (u32 i = 1; i < S; i++) L.ops.push_back(make_op(OPF_STORE | (i == 1 ? OPF_LOAD : 0), S, 0, 0, i));
    }
    sliding_ops(E, L.w, &L.ops);
    L.ops.push_back(make_op(0, OPND_ONE));
    return L;
}
static u32 table_slots(int w) { return (1u << (w - 1)) + 1; }
}  // namespace mr

// Program for exponent E on ctx.  The first kProgCache distinct (exponent, crt) programs of a context are
// built, uploaded once (cudaMalloc + a copy on a private stream that the host waits for: no device-wide
// synchronisation) and cached until the context is destroyed; cached programs are never evicted, so a pointer
// handed to one thread can never be freed under another thread's launch.  Past the bound, a program is
// TRANSIENT: allocated and copied stream-ordered on the caller's stream and released with cudaFreeAsync on the
// same stream after the launch (release_prog), so an unbounded stream of distinct exponents costs one small
// H2D copy per call and no memory growth.
static constexpr size_t kProgCache = 64;

static int get_prog(mr_rns_ctx *c, const Big &E, bool crt, DevProg *out, void *stream) {
    std::lock_guard<std::mutex> lk(c->mu);
    auto key = std::make_pair(E, crt);
    auto it = c->progs.find(key);
    if (it != c->progs.end()) {
        *out = it->second;
        return MR_OK;
    }
    Ladder L = build_program(E, crt);
    DevProg dp;
    dp.nops = (u32)L.ops.size();
    dp.w = L.w;
    if (cudaSetDevice(c->device) != cudaSuccess) return MR_ERR_CUDA;
    const size_t bytes = L.ops.size() * 8;
    if (c->progs.size() >= kProgCache) {
        cudaStream_t st = (cudaStream_t)stream;
        if (cudaMallocAsync(&dp.d_ops, bytes, st) != cudaSuccess) return MR_ERR_NOMEM;
        // pageable source: staged before the call returns, so L may go out of scope
        if (cudaMemcpyAsync(dp.d_ops, L.ops.data(), bytes, cudaMemcpyHostToDevice, st) != cudaSuccess) {
            cudaFreeAsync(dp.d_ops, st);
            return MR_ERR_CUDA;
        }
        dp.transient = true;
        *out = dp;
        return MR_OK;
    }
    if (!c->upload) {
        if (cudaStreamCreateWithFlags(&c->upload, cudaStreamNonBlocking) != cudaSuccess) return MR_ERR_CUDA;
    }
    if (cudaMalloc(&dp.d_ops, bytes) != cudaSuccess) return MR_ERR_NOMEM;
    if (cudaMemcpyAsync(dp.d_ops, L.ops.data(), bytes, cudaMemcpyHostToDevice, c->upload) != cudaSuccess ||
        cudaStreamSynchronize(c->upload) != cudaSuccess) {
        cudaFree(dp.d_ops);
        return MR_ERR_CUDA;
    }
    c->progs.emplace(key, dp);
    *out = dp;
    return MR_OK;
}

static void release_prog(const DevProg &dp, void *stream) {
    if (dp.transient) cudaFreeAsync(dp.d_ops, (cudaStream_t)stream);
}

// ------------------------------------------------------------------ C ABI

#pragma GCC visibility push(default)
extern "C" {
int mr_internal_miller_rabin(const uint32_t *d_n, size_t limbs, size_t count, const uint32_t *d_bases, int rounds,
                             int k, uint8_t *d_verdict, int16_t *d_witness_round, int32_t *d_status, int device,
                             void *stream, int forced, int window);

const char *mr_strerror(int code) {
    switch (code) {
        case MR_OK: return "ok";
        case MR_ERR_ARG: return "invalid argument";
        case MR_ERR_EVEN_MODULUS: return "modulus must be odd and >= 3";
        case MR_ERR_NOT_COPRIME: return "modulus shares a prime with the RNS base";
        case MR_ERR_CAPACITY: return "modulus too large for the RNS base";
        case MR_ERR_RANGE: return "input out of range";
        case MR_ERR_CUDA: return "CUDA error";
        case MR_ERR_NOMEM: return "out of memory";
        default: return "unknown error";
    }
}

int mr_rns_supported_k(int *ks, int cap) {
    for (int i = 0; i < kNumK && i < cap; i++) ks[i] = kSupportedK[i];
    return kNumK;
}

int mr_rns_ctx_create(mr_rns_ctx **out, const uint32_t *modulus, size_t limbs, int k, int device) {
    if (!out) return MR_ERR_ARG;
    *out = nullptr;
    if (!modulus || limbs == 0 || k < 0) return MR_ERR_ARG;
    Big N = big_of(modulus, limbs);
    return build_ctx(out, N, limbs, k, device, N, limbs, nullptr, nullptr);
}

void mr_rns_ctx_destroy(mr_rns_ctx *ctx) {
    if (!ctx) return;
    cudaSetDevice(ctx->device);
    if (ctx->d_cx) cudaFree(ctx->d_cx);
    for (auto &kv : ctx->progs) cudaFree(kv.second.d_ops);
    if (ctx->upload) cudaStreamDestroy(ctx->upload);
    delete ctx;
}

int mr_rns_ctx_info(const mr_rns_ctx *ctx, int *k, size_t *limbs, int *max_modulus_bits, int *modulus_bits,
                    int *paper_cap_bits) {
    if (!ctx) return MR_ERR_ARG;
    if (k) *k = ctx->k;
    if (limbs) *limbs = ctx->limbs;
    if (max_modulus_bits) *max_modulus_bits = ctx->max_bits;
    if (modulus_bits) *modulus_bits = ctx->bits;
    if (paper_cap_bits) *paper_cap_bits = ctx->k * 31;  // P:48 "128 32-bit primes ... 3,968-bit" = 128 x 31 (R4)
    return MR_OK;
}

// The tensor-core base extension (k <= 64) is the default; MR_RNS_IMAD_ONLY=1 selects the IMAD-pipe
// kernel (same results; kept for comparison and parity testing) — see mr_internal_set_path.
static int g_path_override = -1;   // -1: environment, 0: IMAD only, 1: tensor allowed
static bool tensor_path_enabled() {
    if (g_path_override >= 0) return g_path_override == 1;
    const char *e = getenv("MR_RNS_IMAD_ONLY");
    return !(e && e[0] == '1');
}

// tensor-core wide kernel (k = 97, 129; §4k): MR_RNS_TCW=0 (or the IMAD-only path) keeps the IMAD wide kernel
static int g_tcw_override = -1;
static bool tcw_enabled() {
    if (!tensor_path_enabled()) return false;
    if (g_tcw_override >= 0) return g_tcw_override == 1;
    static const bool on = [] { const char *e = getenv("MR_RNS_TCW"); return !(e && e[0] == '0'); }();
    return on;
}

// 128-message tile-jobs (ctas0 per context) on one persistent CTA per SM
static int launch_ladders_tcw(mr_rns_ctx *const *ctxs, const DevProg *progs, int nctx, const u32 *d_x, size_t in_limbs,
                              size_t half, u32 *d_y, size_t out_limbs, size_t count, int32_t *d_status, void *stream,
                              int (*launch_tcw)(const ModexpParams &, u32, const u32 *, const void *, u32, u32, u32, void *,
                                                void *)) {
    const mr_rns_ctx *c0 = ctxs[0];
    cudaStream_t st = (cudaStream_t)stream;
    const u32 tm = tcw_m((u32)c0->k);                // messages per tile-job (k = 505: 64)
    u32 ctas0 = (u32)((count + tm - 1) / tm);
    if (TCW_LOCK || (TCW_PAIR && tm == 128)) ctas0 += ctas0 & 1u;   // lockstep tiles / CTA pairs: job pairs of one context
    const u32 jobs = ctas0 * (u32)nctx;
    const u32 jobs_total = ctas0 * tm * (u32)nctx;
    int sms = 148;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, c0->device);
    static const int max_sms = [] { const char *e = getenv("MR_RNS_MAX_SMS"); return e ? atoi(e) : 0; }();
    if (max_sms > 0) sms = std::min(sms, std::max(1, max_sms));
    const u32 tiles = tcw_tiles((u32)c0->k);
    // CTA pairs (2-CTA clusters): each cluster runs `tiles` pair-jobs (256 messages each) at a time
    const u32 grid = (TCW_PAIR && tm == 128) ? 2 * std::min<u32>(std::max(1, sms / 2), (jobs / 2 + tiles - 1) / tiles)
                              : std::min<u32>((u32)sms, (jobs + tiles - 1) / tiles);
    int w = 1;
    for (int i = 0; i < nctx; i++) w = std::max(w, progs[i].w);
    const size_t nch = 2 * (size_t)c0->k + 1;
    u32 *d_table = nullptr;
    // window table + one spare slot (to_rns parks its B' outputs there, mr_tcw.cuh) [+ the B-residue slot, k = 505]
    const size_t slots = (size_t)table_slots(w) + 1 + (tcw_bres_tmem((u32)c0->k) ? 0 : 1);
    if (cudaMallocAsync(&d_table, slots * nch * jobs_total * 4, st) != cudaSuccess) return MR_ERR_NOMEM;
    ModexpParams P;
    memset(&P, 0, sizeof P);
    for (int i = 0; i < 2; i++) {
        const int s = i < nctx ? i : nctx - 1;
        P.ctx[i] = ctxs[s]->d_cx;
        P.prog[i] = progs[s].d_ops;
        P.nops[i] = progs[s].nops;
    }
    P.ctas0 = ctas0;
    P.count = (u32)count;
    P.x = d_x;
    P.in_limbs = (u32)in_limbs;
    P.half = (u32)half;
    P.y = d_y;
    P.out_limbs = (u32)out_limbs;
    P.out_stride = count * out_limbs;
    P.status = d_status;
    P.table = d_table;
    P.jobs_total = jobs_total;
    P.hslot = table_slots(w);
    // MR_TCW_TRACE=file: debug timeline of CTA 0 (phase timestamps, mr_tcw.cuh w_trace) appended to `file`
    static const char *trace_file = getenv("MR_TCW_TRACE");
    unsigned long long *d_trace = nullptr;
    if (trace_file && cudaMallocAsync(&d_trace, 16384 * 8, st) == cudaSuccess) cudaMemsetAsync(d_trace, 0, 16384 * 8, st);
    int rc = timed_launch(0, st, [&] {
                 return launch_tcw(P, grid, c0->d_wide, c0->d_tcw, c0->cxw, c0->be1w, jobs, d_trace, stream);
             }) == 0
                 ? MR_OK
                 : MR_ERR_CUDA;
    if (d_trace) {
        std::vector<unsigned long long> h(16384);
        if (cudaMemcpyAsync(h.data(), d_trace, h.size() * 8, cudaMemcpyDeviceToHost, st) == cudaSuccess &&
            cudaStreamSynchronize(st) == cudaSuccess) {
            if (FILE *f = fopen(trace_file, "ab")) {
                fwrite(h.data(), 8, h.size(), f);
                fclose(f);
            }
        }
        cudaFreeAsync(d_trace, st);
    }
    cudaFreeAsync(d_table, st);
    return rc;
}

// wide-operand ladders (wide_path(k)): 16 messages per CTA, one CTA per 16 messages and context
static int launch_ladders_wide(mr_rns_ctx *const *ctxs, const DevProg *progs, int nctx, const u32 *d_x,
                               size_t in_limbs, size_t half, u32 *d_y, size_t out_limbs, size_t count, int32_t *d_status,
                               void *stream, bool lanes) {
    const mr_rns_ctx *c0 = ctxs[0];
    cudaStream_t st = (cudaStream_t)stream;
    if (!lanes && c0->d_tcw && c0->be1w && tcw_enabled()) {
        auto launch_tcw = c0->k == 505   ? launch_modexp_tcw_k505
                          : c0->k == 257 ? launch_modexp_tcw_k257
                                         : kernel_set_for(c0->k).launch_modexp_tcw;
        if (launch_tcw)
            return launch_ladders_tcw(ctxs, progs, nctx, d_x, in_limbs, half, d_y, out_limbs, count, d_status, stream,
                                      launch_tcw);
    }
    const u32 MBm = (u32)(lanes ? wide_messages_per_cta_lanes() : wide_messages_per_cta());
    const u32 ctas0 = (u32)((count + MBm - 1) / MBm);
    const u32 jobs_total = ctas0 * MBm * nctx;
    int w = 1;
    for (int i = 0; i < nctx; i++) w = std::max(w, progs[i].w);
    const size_t nch = 2 * (size_t)c0->k + 1;
    const size_t rows = std::max<size_t>((size_t)table_slots(w) * nch, 3 * ((size_t)c0->k + 1));   // + exit scratch
    u32 *d_table = nullptr;
    if (cudaMallocAsync(&d_table, rows * jobs_total * 4, st) != cudaSuccess) return MR_ERR_NOMEM;
    ModexpParams P;
    memset(&P, 0, sizeof P);
    for (int i = 0; i < 2; i++) {
        const int s = i < nctx ? i : nctx - 1;
        P.ctx[i] = ctxs[s]->d_cx;
        P.prog[i] = progs[s].d_ops;
        P.nops[i] = progs[s].nops;
    }
    P.ctas0 = ctas0;
    P.count = (u32)count;
    P.x = d_x;
    P.in_limbs = (u32)in_limbs;
    P.half = (u32)half;
    P.y = d_y;
    P.out_limbs = (u32)out_limbs;
    P.out_stride = count * out_limbs;
    P.status = d_status;
    P.table = d_table;
    P.jobs_total = jobs_total;
    int rc = timed_launch(0, st, [&] {
                 return lanes ? launch_modexp_wide_lanes(P, ctas0 * nctx, c0->d_wide, (u32)c0->k, c0->cxw, stream)
                              : launch_modexp_wide(P, ctas0 * nctx, c0->d_wide, (u32)c0->k, c0->cxw, stream);
             }) == 0
                 ? MR_OK
                 : MR_ERR_CUDA;
    cudaFreeAsync(d_table, st);
    return rc;
}

static int launch_ladders(mr_rns_ctx *const *ctxs, const DevProg *progs, int nctx, const u32 *d_x, size_t in_limbs,
                          size_t half, u32 *d_y, size_t out_limbs, size_t count, int32_t *d_status, void *stream) {
    const mr_rns_ctx *c0 = ctxs[0];
    const KernelSet &ks = kernel_set_for(c0->k);
    if (cudaSetDevice(c0->device) != cudaSuccess) return MR_ERR_CUDA;
    cudaStream_t st = (cudaStream_t)stream;
    if (wide_path(c0->k)) return launch_ladders_wide(ctxs, progs, nctx, d_x, in_limbs, half, d_y, out_limbs, count,
                                                        d_status, stream, false);
    if (c0->cxw && c0->d_wide && tensor_path_enabled() && count * (size_t)nctx <= small_max())   // small batch (§4j)
        return launch_ladders_wide(ctxs, progs, nctx, d_x, in_limbs, half, d_y, out_limbs, count, d_status, stream, true);
    const bool use_tc = ks.launch_modexp_tc && c0->d_tcb2 && tensor_path_enabled();
    // IMAD path: one CTA per T messages; tensor path: ctas0 = 128-message tile-jobs per context,
    // run by Gc persistent CTAs per context (one per SM share)
    const u32 T = use_tc ? 128u : (u32)ks.threads;
    const bool pair = use_tc && tc_pair((u32)c0->k);   // CTA-pair tensor kernel: 256-message jobs
    u32 ctas0 = (u32)((count + T - 1) / T);
    if (pair) ctas0 += ctas0 & 1u;
    const u32 jobs_total = ctas0 * T * nctx;
    u32 gc = 0, grid = 0;
    if (use_tc) {
        int sms = 148;
        cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, c0->device);
        // MR_RNS_MAX_SMS=n: size the persistent grid as if only n SMs existed (tests and sanitizer runs reach
        // the split schedule with small batches this way; results do not depend on it)
        static const int max_sms = [] { const char *e = getenv("MR_RNS_MAX_SMS"); return e ? atoi(e) : 0; }();
        if (max_sms > 0) sms = std::min(sms, std::max(2, max_sms));
        if (pair) {   // gc = CTA pairs per context
            gc = std::max<u32>(1u, std::min<u32>((u32)(sms / 2) / (u32)nctx, ctas0 / 2));
            grid = 2 * gc * nctx;
        } else {
            gc = std::min<u32>((u32)((sms + nctx - 1) / nctx), ctas0);
            grid = gc * nctx;
        }
    }
    int w = 1;
    for (int i = 0; i < nctx; i++) w = std::max(w, progs[i].w);
    const size_t nch = 2 * (size_t)c0->k + 1;
    // split schedule when jobs do not divide evenly over the tile slots: one more table
    // slot for the handed-over states, and one flag per (context, job, rank)
    const u32 njobs = pair ? ctas0 / 2 : ctas0;
    const u32 slots_per_group = gc * (u32)ks.tc_tiles;
    const char *ns = getenv("MR_RNS_NO_SPLIT");
    const bool split = use_tc && !(ns && ns[0] == '1') && njobs > slots_per_group && njobs % slots_per_group != 0;
    const size_t table_words = (size_t)(table_slots(w) + (split ? 1 : 0)) * nch * jobs_total;
    const size_t flag_words = split ? (size_t)2 * njobs * 2 + 1 : 0;   // + the start-order ticket
    u32 *d_table = nullptr;
    if (cudaMallocAsync(&d_table, (table_words + flag_words) * 4, st) != cudaSuccess) return MR_ERR_NOMEM;
    if (split && cudaMemsetAsync(d_table + table_words, 0, flag_words * 4, st) != cudaSuccess) {
        cudaFreeAsync(d_table, st);
        return MR_ERR_CUDA;
    }
    ModexpParams P;
    memset(&P, 0, sizeof P);
    for (int i = 0; i < 2; i++) {
        const int s = i < nctx ? i : nctx - 1;
        P.ctx[i] = ctxs[s]->d_cx;
        P.prog[i] = progs[s].d_ops;
        P.nops[i] = progs[s].nops;
    }
    P.ctas0 = ctas0;
    P.count = (u32)count;
    P.x = d_x;
    P.in_limbs = (u32)in_limbs;
    P.half = (u32)half;
    P.y = d_y;
    P.out_limbs = (u32)out_limbs;
    P.out_stride = count * out_limbs;
    P.status = d_status;
    P.table = d_table;
    P.jobs_total = jobs_total;
    P.pow_tab = c0->d_pow;
    P.be_tab = c0->d_be;
    P.tc_b2 = c0->d_tcb2;
    P.mpl = c0->d_mpl;
    P.tc_be1_off = cx_words(c0->k) + be_half_words(c0->k);
    P.tc_be2_off = P.tc_be1_off + tc_bbytes(c0->k) / 4;
    P.tc_gc = gc;
    P.hslot = table_slots(w);
    P.flags = split ? d_table + table_words : nullptr;
    int rc = timed_launch(0, st, [&] {
                 return use_tc ? ks.launch_modexp_tc(P, grid, stream) : ks.launch_modexp(P, ctas0 * nctx, stream);
             }) == 0
                 ? MR_OK
                 : MR_ERR_CUDA;
    cudaFreeAsync(d_table, st);
    return rc;
}

int mr_modexp_batch(const mr_rns_ctx *ctx, const uint32_t *d_x, uint32_t *d_y, size_t count, const uint32_t *exp,
                    size_t exp_limbs, int32_t *d_status, void *stream) {
    if (!ctx || (count && (!d_x || !d_y)) || (exp_limbs && !exp)) return MR_ERR_ARG;
    if (count == 0) return MR_OK;
    if (count > 0x7FFFFFFFu / 2) return MR_ERR_ARG;
    Big E = exp_limbs ? big_of(exp, exp_limbs) : Big();
    mr_rns_ctx *c = const_cast<mr_rns_ctx *>(ctx);
    DevProg dp;
    int rc = get_prog(c, E, false, &dp, stream);
    if (rc != MR_OK) return rc;
    rc = launch_ladders(&c, &dp, 1, d_x, ctx->limbs, 0, d_y, ctx->limbs, count, d_status, stream);
    release_prog(dp, stream);
    return rc;
}

int mr_rsa_encrypt_batch(const mr_rns_ctx *n_ctx, const uint32_t *e, size_t e_limbs, const uint32_t *d_m,
                         uint32_t *d_c, size_t count, int32_t *d_status, void *stream) {
    return mr_modexp_batch(n_ctx, d_m, d_c, count, e, e_limbs, d_status, stream);
}

int mr_rsa_priv_create(mr_rsa_priv **out, const uint32_t *p, const uint32_t *q, size_t half_limbs, const uint32_t *d_p,
                       const uint32_t *d_q, const uint32_t *q_inv, int k_half, int device) {
    if (!out) return MR_ERR_ARG;
    *out = nullptr;
    if (!p || !q || !d_p || !d_q || !q_inv || half_limbs == 0 || k_half < 0) return MR_ERR_ARG;
    Big P = big_of(p, half_limbs), Q = big_of(q, half_limbs), QI = big_of(q_inv, half_limbs);
    if (P.empty() || Q.empty() || cmp(P, Q) == 0) return MR_ERR_ARG;
    if (cmp(mod(mul(QI, Q), P), Big{1}) != 0) return MR_ERR_ARG;
    Big N = mul(P, Q);
    // both halves share one base pair: pick k that fits the larger prime
    int k;
    {
        std::lock_guard<std::mutex> lk(g_mu);
        const Big &big = cmp(P, Q) > 0 ? P : Q;
        int kmin = 1;
        if (k_half > 0) {
            kmin = -1;
            for (int i = 0; i < kNumK; i++)
                if (kSupportedK[i] >= k_half) { kmin = kSupportedK[i]; break; }
            if (kmin < 0) return MR_ERR_ARG;
        }
        k = auto_k(big, kmin);
        if (k < 0) return MR_ERR_CAPACITY;
    }
    Big hl{(u32)half_limbs};
    mr_rsa_priv *pr = new (std::nothrow) mr_rsa_priv;
    if (!pr) return MR_ERR_NOMEM;
    pr->half = half_limbs;
    pr->dp = big_of(d_p, half_limbs);
    pr->dq = big_of(d_q, half_limbs);
    int rc = build_ctx(&pr->cp, P, half_limbs, k, device, N, 2 * half_limbs, &hl, &QI);
    if (rc == MR_OK) rc = build_ctx(&pr->cq, Q, half_limbs, k, device, N, 2 * half_limbs, &hl, nullptr);
    if (rc == MR_OK && pr->cp->k != pr->cq->k) rc = MR_ERR_CAPACITY;
    if (rc == MR_OK) {
        if (cudaMalloc(&pr->d_q, half_limbs * 4) != cudaSuccess) rc = MR_ERR_NOMEM;
        else if (cudaMemcpy(pr->d_q, q, half_limbs * 4, cudaMemcpyHostToDevice) != cudaSuccess) rc = MR_ERR_CUDA;
    }
    if (rc == MR_OK && wide_path(k)) {
        if (cudaMalloc(&pr->d_qinv, half_limbs * 4) != cudaSuccess) rc = MR_ERR_NOMEM;
        else if (cudaMemcpy(pr->d_qinv, q_inv, half_limbs * 4, cudaMemcpyHostToDevice) != cudaSuccess) rc = MR_ERR_CUDA;
    }
    if (rc != MR_OK) {
        mr_rsa_priv_destroy(pr);
        return rc;
    }
    *out = pr;
    return MR_OK;
}

void mr_rsa_priv_destroy(mr_rsa_priv *priv) {
    if (!priv) return;
    mr_rns_ctx_destroy(priv->cp);
    mr_rns_ctx_destroy(priv->cq);
    if (priv->d_q) cudaFree(priv->d_q);
    if (priv->d_qinv) cudaFree(priv->d_qinv);
    delete priv;
}

int mr_rsa_decrypt_batch(const mr_rsa_priv *priv, const uint32_t *d_c, uint32_t *d_m, size_t count, int32_t *d_status,
                         void *stream) {
    if (!priv || (count && (!d_c || !d_m))) return MR_ERR_ARG;
    if (count == 0) return MR_OK;
    if (count > 0x7FFFFFFFu / 2) return MR_ERR_ARG;
    const size_t H = priv->half;
    mr_rns_ctx *cs[2] = {priv->cp, priv->cq};
    DevProg L[2];
    int rc0 = get_prog(priv->cp, priv->dp, true, &L[0], stream);
    if (rc0 == MR_OK) rc0 = get_prog(priv->cq, priv->dq, true, &L[1], stream);
    if (rc0 != MR_OK) {
        release_prog(L[0], stream);
        return rc0;
    }
    if (cudaSetDevice(priv->cp->device) != cudaSuccess) return MR_ERR_CUDA;
    cudaStream_t st = (cudaStream_t)stream;
    u32 *d_mpq = nullptr;
    int32_t *d_st = d_status;
    int32_t *d_tmpst = nullptr;
    if (cudaMallocAsync(&d_mpq, 2 * count * H * 4, st) != cudaSuccess) {
        release_prog(L[0], stream);
        release_prog(L[1], stream);
        return MR_ERR_NOMEM;
    }
    if (!d_st) {
        if (cudaMallocAsync(&d_tmpst, count * 4, st) != cudaSuccess) {
            cudaFreeAsync(d_mpq, st);
            release_prog(L[0], stream);
            release_prog(L[1], stream);
            return MR_ERR_NOMEM;
        }
        d_st = d_tmpst;
    }
    int rc = launch_ladders(cs, L, 2, d_c, 2 * H, H, d_mpq, H, count, d_st, stream);
    if (rc == MR_OK) {
        CombineParams C;
        memset(&C, 0, sizeof C);
        C.ctx_p = priv->cp->d_cx;
        C.q = priv->d_q;
        C.mpq = d_mpq;
        C.count = (u32)count;
        C.half = (u32)H;
        C.m = d_m;
        C.status = d_st;
        C.pow_tab = priv->cp->d_pow;
        C.be_tab = priv->cp->d_be;
        C.mpl = priv->cp->d_mpl;
        if (wide_path(priv->cp->k)) {   // positional recombination (mr_wide.cu k_combine_wide)
            u32 *d_scr = nullptr;
            if (cudaMallocAsync(&d_scr, count * (2 * H + 2) * 4, st) != cudaSuccess) {
                rc = MR_ERR_NOMEM;
            } else {
                rc = timed_launch(1, st, [&] {
                         return launch_combine_wide(C, priv->d_qinv, d_scr, (u32)priv->cp->k, stream);
                     }) == 0
                         ? MR_OK
                         : MR_ERR_CUDA;
                cudaFreeAsync(d_scr, st);
            }
        } else {
            const KernelSet &ks = kernel_set_for(priv->cp->k);
            rc = timed_launch(1, st, [&] { return ks.launch_combine(C, stream); }) == 0 ? MR_OK : MR_ERR_CUDA;
        }
    }
    cudaFreeAsync(d_mpq, st);
    if (d_tmpst) cudaFreeAsync(d_tmpst, st);
    release_prog(L[0], stream);
    release_prog(L[1], stream);
    return rc;
}

// fixed window of the a^d ladder: w = 5 above 768-bit candidates (1024-bit C5: +2.7 % over w = 4; w = 6 and
// w = 3 slower), else 4 (a 2^w-entry table per candidate)
int mr_internal_mr_window(size_t limbs) { return limbs * 32 > 768 ? 5 : 4; }

int mr_miller_rabin_batch(const uint32_t *d_n, size_t limbs, size_t count, const uint32_t *d_bases, int rounds, int k,
                          uint8_t *d_verdict, int16_t *d_witness_round, int32_t *d_status, int device, void *stream) {
    return mr_internal_miller_rabin(d_n, limbs, count, d_bases, rounds, k, d_verdict, d_witness_round, d_status,
                                    device, stream, 0, mr_internal_mr_window(limbs));
}

// Miller-Rabin with benchmark controls: forced = 1 runs every round for every candidate (MR-rounds/s),
// window = fixed-window width of the a^d ladder.
int mr_internal_miller_rabin(const uint32_t *d_n, size_t limbs, size_t count, const uint32_t *d_bases, int rounds,
                             int k, uint8_t *d_verdict, int16_t *d_witness_round, int32_t *d_status, int device,
                             void *stream, int forced, int window) {
    if ((count && (!d_n || !d_verdict || (rounds > 0 && !d_bases))) || limbs == 0 || rounds < 0 || k < 0 ||
        window < 1 || window > 6)
        return MR_ERR_ARG;
    if (count == 0) return MR_OK;
    if (count > 0x7FFFFFFFu) return MR_ERR_ARG;
    int kk;
    const u32 *d_pow = nullptr, *d_be = nullptr;
    DevBase db;
    {
        std::lock_guard<std::mutex> lk(g_mu);
        Big top = sub(pow2(32 * (int)limbs), Big{1});   // capacity for any n < 2^(32 limbs)
        int kmin = 1;
        if (k > 0) {
            kmin = -1;
            for (int i = 0; i < kNumK; i++)
                if (kSupportedK[i] >= k) { kmin = kSupportedK[i]; break; }
            if (kmin < 0) return MR_ERR_ARG;
        }
        kk = auto_k(top, kmin);
        if (kk < 0) return MR_ERR_CAPACITY;
        if ((int)limbs > kk - 1) return MR_ERR_CAPACITY;
        int rc = ensure_device_base(kk, device, &d_pow, &d_be);
        if (rc != MR_OK) return rc;
        db = g_devbases[std::make_pair(device, kk)];
    }
    if (cudaSetDevice(device) != cudaSuccess) return MR_ERR_CUDA;
    cudaStream_t st = (cudaStream_t)stream;
    if (is_wide((u32)kk)) {   // 4,097 .. 16,128-bit candidates: channels-on-threads kernels (mr_wide.cu)
        u32 *d_pcw = nullptr, *d_scr = nullptr, *d_wt = nullptr;
        const u32 c = (u32)count, kw = (u32)kk;
        if (cudaMallocAsync(&d_pcw, mr_wide_pcw_words(kw, c) * 4, st) != cudaSuccess) return MR_ERR_NOMEM;
        if (cudaMallocAsync(&d_scr, mr_wide_scr_words(kw, c) * 4, st) != cudaSuccess ||
            cudaMallocAsync(&d_wt, mr_wide_table_words(kw, (u32)window, c) * 4, st) != cudaSuccess) {
            cudaFreeAsync(d_pcw, st);
            if (d_scr) cudaFreeAsync(d_scr, st);
            return MR_ERR_NOMEM;
        }
        int rc = timed_launch(2, st, [&] {
                     return launch_mr_wide(db.d_wide, kw, d_pcw, d_scr, d_n, d_bases, c, (u32)limbs, (u32)rounds,
                                           (u32)window, (u32)forced, d_wt, d_verdict, d_witness_round, d_status, stream);
                 }) == 0
                     ? MR_OK
                     : MR_ERR_CUDA;
        cudaFreeAsync(d_pcw, st);
        cudaFreeAsync(d_scr, st);
        cudaFreeAsync(d_wt, st);
        return rc;
    }
    const size_t nch = 2 * (size_t)kk + 1;
    const KernelSet &ks = kernel_set_for(kk);
    const bool tc = db.d_tcb1u && ks.launch_modexp_tc && ks.mr_tiles > 0 && tensor_path_enabled();
    u32 gc = 0;
    if (tc) {
        int sms = 148;
        cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device);
        gc = std::min<u32>((u32)sms, (u32)((count + 127) / 128));
    }
    // early-exit compaction on the tensor path (round 0 for all, then (survivor, round) items)
    const bool compact = tc && !forced && rounds > 1;
    const size_t slots = compact ? (size_t)gc * ks.mr_tiles * 128 : 0;
    const size_t tcols = std::max<size_t>(count, slots);
    u32 *d_pc = nullptr, *d_tab = nullptr, *d_aux = nullptr;
    if (cudaMallocAsync(&d_pc, (size_t)pc_words(kk) * count * 4, st) != cudaSuccess) return MR_ERR_NOMEM;
    // window tables: (2^w + 1) entries per candidate slot; the tensor kernel pads entries to pad4(nch)
    if (cudaMallocAsync(&d_tab, ((size_t)(1u << window) + 1) * ((nch + 3) & ~(size_t)3) * tcols * 4, st) != cudaSuccess) {
        cudaFreeAsync(d_pc, st);
        return MR_ERR_NOMEM;
    }
    if (compact && cudaMallocAsync(&d_aux, (2 * count + 4) * 4, st) != cudaSuccess) {
        cudaFreeAsync(d_pc, st);
        cudaFreeAsync(d_tab, st);
        return MR_ERR_NOMEM;
    }
    MrParams P;
    memset(&P, 0, sizeof P);
    P.n = d_n;
    P.bases = d_bases;
    P.count = (u32)count;
    P.limbs = (u32)limbs;
    P.rounds = (u32)rounds;
    P.window = (u32)window;
    P.forced = (u32)forced;
    P.pc = d_pc;
    P.table = d_tab;
    P.verdict = d_verdict;
    P.witness = d_witness_round;
    P.status = d_status;
    P.pow_tab = d_pow;
    P.be_tab = d_be;
    P.mpl = db.d_mpl;
    if (tc) {
        P.tc_b1 = db.d_tcb1u;
        P.tc_b2 = db.d_tcb2;
        P.tc_gc = gc;
        P.one_g = db.d_one;
    }
    if (compact) {
        P.live = d_aux;
        P.wit32 = d_aux + count;
        P.nlive = d_aux + 2 * count;
        P.tstride = (u32)slots;
    }
    int rc = timed_launch(2, st, [&] { return ks.launch_mr(P, stream); }) == 0 ? MR_OK : MR_ERR_CUDA;
    cudaFreeAsync(d_pc, st);
    cudaFreeAsync(d_tab, st);
    if (d_aux) cudaFreeAsync(d_aux, st);
    return rc;
}

// ---- test hooks (not part of include/mr_rns.h): host images of the precomputed tables, so the
// CPU test suite can check the identities of DESIGN.md §3 without a GPU.
int mr_internal_base_table(int k, uint32_t *out, size_t cap, uint32_t *primes_out) {
    bool ok = false;
    for (int i = 0; i < kNumK; i++) ok |= kSupportedK[i] == k;
    if (!ok) return -1;
    std::lock_guard<std::mutex> lk(g_mu);
    const Base &b = base_for(k);
    if (out) memcpy(out, b.flat.data(), std::min(cap, b.flat.size()) * 4);
    if (primes_out) {
        memcpy(primes_out, b.B.data(), 4 * k);
        memcpy(primes_out + k, b.Bp.data(), 4 * k);
    }
    return (int)b.flat.size();
}

int mr_internal_pow_table(int k, uint32_t *out, size_t cap) {
    std::lock_guard<std::mutex> lk(g_mu);
    const Base &b = base_for(k);
    if (out) memcpy(out, b.pow.data(), std::min(cap, b.pow.size()) * 4);
    return (int)b.pow.size();
}

// builds the context block of modulus N for a given k (no device work); returns its word count or
// a negative MR_* error code
// test hook: the wide-operand per-k table (mr_internal.h WideLayout) without a device
int mr_internal_wide_table(int k, uint32_t *out, size_t cap) {
    if (k < 97) return -MR_ERR_ARG;
    bool ok = false;
    for (int i = 0; i < kNumK; i++) ok |= kSupportedK[i] == k;
    if (!ok) return -MR_ERR_ARG;
    std::lock_guard<std::mutex> lk(g_mu);
    const std::vector<u32> t = build_wide_table(base_for(k));
    if (out) memcpy(out, t.data(), std::min(cap, t.size()) * 4);
    return (int)t.size();
}

// test hook (CPU): byte image of tensor-core wide extension e (mr_internal.h TCW_*) for k = 97 / 129; e = TCW_BE1 is
// per context and needs the modulus (limbs words), the others are per k.  Returns the byte count, < 0 on error.
int mr_internal_tcw_image(int k, int e, const uint32_t *modulus, size_t limbs, uint8_t *out, size_t cap) {
    if (!tcw_k((u32)k) || e < 0 || e > 3) return -MR_ERR_ARG;
    std::lock_guard<std::mutex> lk(g_mu);
    const Base &b = base_for(k);
    std::vector<uint8_t> img;
    if (e == TCW_BE1) {
        Big N = big_of(modulus, limbs);
        if (N.empty() || !(N[0] & 1)) return -MR_ERR_EVEN_MODULUS;
        if (!fits(b, N)) return -MR_ERR_CAPACITY;
        std::vector<u32> x(cx_words(k), 0);
        fill_ctx_block(b, N, limbs, N, limbs, nullptr, nullptr, x.data());
        img.resize(tcw_img_bytes(k, TCW_BE1));
        fill_tcw_be1(b, x.data(), img.data());
    } else {
        const std::vector<uint8_t> all = build_tcw_images(b);
        const u32 o = tcw_img_off(k, e);
        img.assign(all.begin() + o, all.begin() + o + tcw_img_bytes(k, e));
    }
    if (out) memcpy(out, img.data(), std::min(cap, img.size()));
    return (int)img.size();
}

// test hook: the wide Miller-Rabin setup alone (k = 257 / 505): per-candidate rows wmr_* into d_pcw
// (DEVICE, mr_wide_pcw_words), for checking σ, c2, R^2, s, d against their definitions
int mr_internal_mr_wide_setup(const uint32_t *d_n, size_t limbs, size_t count, int k, uint32_t *d_pcw, uint8_t *d_verdict,
                              int device) {
    if (!is_wide((u32)k) || !d_n || !d_pcw || !d_verdict) return MR_ERR_ARG;
    const u32 *d_pow = nullptr, *d_be = nullptr;
    DevBase db;
    {
        std::lock_guard<std::mutex> lk(g_mu);
        int rc = ensure_device_base(k, device, &d_pow, &d_be);
        if (rc != MR_OK) return rc;
        db = g_devbases[std::make_pair(device, k)];
    }
    u32 *d_scr = nullptr;
    if (cudaMalloc(&d_scr, mr_wide_scr_words((u32)k, (u32)count) * 4) != cudaSuccess) return MR_ERR_NOMEM;
    const int rc = launch_mr_wide_setup(db.d_wide, (u32)k, d_pcw, d_scr, d_n, (u32)count, (u32)limbs, d_verdict, nullptr);
    cudaDeviceSynchronize();
    cudaFree(d_scr);
    return rc == 0 ? MR_OK : MR_ERR_CUDA;
}

// test hook: the tensor-core wide kernel for k = 97 / 129 (§4k): 1 = on (default), 0 = the IMAD wide kernel,
// -1 = follow MR_RNS_TCW
int mr_internal_set_tcw(int on) {
    g_tcw_override = on;
    return MR_OK;
}

int mr_internal_ctx_table(const uint32_t *modulus, size_t limbs, int k, uint32_t *out, size_t cap) {
    Big N = big_of(modulus, limbs);
    if (N.empty() || !(N[0] & 1)) return -MR_ERR_EVEN_MODULUS;
    std::lock_guard<std::mutex> lk(g_mu);
    const Base &b = base_for(k);
    if (!fits(b, N)) return -MR_ERR_CAPACITY;
    for (u32 m : b.B)
        if (mod_word(N, m) == 0) return -MR_ERR_NOT_COPRIME;
    for (u32 m : b.Bp)
        if (mod_word(N, m) == 0) return -MR_ERR_NOT_COPRIME;
    const size_t tc_words = tc_ok(k) ? tc_bbytes(k) / 4 : 0;
    std::vector<u32> x(cx_words(k) + be_half_words(k) + 2 * tc_words, 0);   // the device context buffer
    fill_ctx_block(b, N, limbs, N, limbs, nullptr, nullptr, x.data());
    fill_merged_be1(b, x.data() + cx_words(k), x.data());
    if (tc_ok(k) && !fill_tc_scaled(b, x.data())) return -MR_ERR_ARG;
    if (out) memcpy(out, x.data(), std::min(cap, x.size()) * 4);
    return (int)x.size();
}

// bench hook: enable/disable event timing of every launch; mr_internal_timing_collect waits for the
// recorded events and returns the summed milliseconds and launch counts per kernel kind.
// Miller-Rabin launch time collected by the last mr_internal_timing_collect
int mr_internal_timing_mr(double *ms, int *n) {
    if (ms) *ms = g_last_mr_ms;
    if (n) *n = g_last_mr_n;
    return MR_OK;
}

// select the Montgomery-multiplication kernel: 0 = IMAD pipe only, 1 = tensor core where compiled,
// -1 = follow MR_RNS_IMAD_ONLY
int mr_internal_set_path(int path) {
    g_path_override = path;
    return MR_OK;
}

// test hook: largest count x contexts routed to the small-batch kernel (§4j); -1 restores the default
int mr_internal_set_small_max(long n) {
    g_small_override = n;
    return MR_OK;
}

int mr_internal_timing(int enable) {
    std::lock_guard<std::mutex> lk(g_tmu);
    g_timing = enable;
    return MR_OK;
}

int mr_internal_timing_collect(double *ms_ladder, int *n_ladder, double *ms_combine, int *n_combine) {
    std::vector<EvPair> ev;
    {
        std::lock_guard<std::mutex> lk(g_tmu);
        ev.swap(g_events);
    }
    double t[3] = {0, 0, 0};
    int n[3] = {0, 0, 0};
    int rc = MR_OK;
    for (auto &e : ev) {
        float ms = 0;
        if (cudaEventSynchronize(e.b) != cudaSuccess || cudaEventElapsedTime(&ms, e.a, e.b) != cudaSuccess) rc = MR_ERR_CUDA;
        t[e.kind] += ms;
        n[e.kind]++;
        cudaEventDestroy(e.a);
        cudaEventDestroy(e.b);
    }
    if (ms_ladder) *ms_ladder = t[0];
    if (n_ladder) *n_ladder = n[0];
    if (ms_combine) *ms_combine = t[1];
    if (n_combine) *n_combine = n[1];
    g_last_mr_ms = t[2];
    g_last_mr_n = n[2];
    return rc;
}

}  // extern "C"
#pragma GCC visibility pop
