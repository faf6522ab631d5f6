// mr_keygen_host.cpp — host orchestration of mr_rsa_keygen_batch (include/mr_rns.h; SURVEY §8(f)
// NEXT-1; §3.3 "RSA key generation ... completely performed on the GPU", §4.3 small-prime
// sieve + Miller-Rabin, §3.1 Arazi inversion).
//
// The host only schedules: which searches run, how many candidates each hands to Miller-Rabin, and the
// acceptance bookkeeping of the key recipe (reading R19).  It reads back flags and candidate indices,
// never a prime or a private exponent: all number arithmetic runs in the kernels of mr_keygen.cu and
// in the library's Miller-Rabin batch (RNS Montgomery domain, tensor-core base extensions).
//
// Search s of key i, attempt a: start_s = odd_with_top_bits(bits/2, seed, TAG_KEY, i * 65536 + a);
// its prime is the first probable prime in start_s, start_s + 2, ... that survives trial division by the
// odd primes among the first 10,000 and passes `rounds` Miller-Rabin rounds with bases 2, 3, 5, ...
// Each Miller-Rabin stage is two batches: round 1 (base 2) over up to G sieve survivors per search, then
// all rounds for the first survivor that passed — exact, because a candidate passing every round passes
// round 1, and a failed verification resumes the search just after that survivor.
#include <cuda_runtime.h>

#include <algorithm>
#include <cstring>
#include <deque>
#include <vector>

#include "../../include/mr_rns.h"
#include "mr_internal.h"

extern "C" int mr_internal_miller_rabin(const uint32_t *d_n, size_t limbs, size_t count, const uint32_t *d_bases,
                                        int rounds, int k, uint8_t *d_verdict, int16_t *d_witness_round,
                                        int32_t *d_status, int device, void *stream, int forced, int window);

extern "C" uint32_t mr_internal_drbg_streams(const mr_drbg *d);

namespace mr {
int kg_launch_start(u64 seed, const u64 *index, u32 nslots, u32 L, u32 *starts, void *st);
int kg_launch_start_rand(const u32 *rnd, u32 nslots, u32 L, u32 *starts, void *st);
int kg_launch_rand_bases(const u32 *cand, const u32 *rnd, u32 items, u32 L, u32 *base, void *st);
int kg_launch_pow(const u32 *small, u32 nsmall, u32 L, u32 *pw, u64 *mu, void *st);
int kg_launch_sieve(const u32 *starts, const u32 *window, const u32 *list, u32 nlist, u32 L, const u32 *small,
                    const u32 *pw, const u64 *mu, u32 nsmall, u32 W, u32 *bitmap, void *st);
int kg_launch_pick(const u32 *starts, const u32 *window, const u32 *bitmap, const u32 *tested, const u32 *act, u32 nact,
                   u32 L, u32 W, u32 G, u32 *cand, u32 *base, u32 *ncand, void *st);
int kg_launch_vitems(const u32 *vl, u32 nv, const u32 *vcand, const u32 *small_all, u32 R, u32 L, u32 *cand, u32 *base,
                     void *st);
int kg_launch_copy_rows(const u32 *src, const u32 *src_row, u32 *dst, const u32 *dst_row, u32 cnt, u32 L, void *st);
int kg_launch_check(const u32 *pool, u32 n, u32 e, const u32 *which, const u32 *first, u32 cnt, u32 *ok, void *st);
int kg_launch_assemble(const u32 *prime, const u32 *key_slot, u32 nkeys, u32 n, u32 e, u32 *N, u32 *P, u32 *Q, u32 *D,
                       u32 *DP, u32 *DQ, u32 *QINV, void *st);

namespace {

constexpr u32 kNumSmall = 10000;       // "up to the first 10,000 primes"
constexpr u32 kWindow = 4096;          // odd candidates per sieve window
constexpr u32 kTarget = 4 * 148 * 128; // phase-A items per Miller-Rabin batch (4 tiles per SM)
constexpr u32 kMaxG = 256;             // survivors per search per batch: a small tail batch costs one
                                       // round of latency whatever its size, so it takes more survivors

const std::vector<u32> &small_primes() {
    static std::vector<u32> sp = [] {
        std::vector<u32> v;
        const u32 lim = 105000;                      // p_10000 = 104,729
        std::vector<bool> comp(lim + 1, false);
        for (u32 i = 2; i <= lim && v.size() < kNumSmall; i++) {
            if (comp[i]) continue;
            v.push_back(i);
            for (u64 j = (u64)i * i; j <= lim; j += i) comp[j] = true;
        }
        return v;
    }();
    return sp;
}

bool is_prime_u32(u32 e) {
    if (e < 2) return false;
    for (u64 d = 2; d * d <= e; d++)
        if (e % d == 0) return false;
    return true;
}

// device scratch owned by one call
struct Dev {
    std::vector<void *> ptrs;
    cudaStream_t st;
    explicit Dev(cudaStream_t s) : st(s) {}
    template <class T>
    T *get(size_t n) {
        void *p = nullptr;
        if (cudaMallocAsync(&p, std::max<size_t>(n, 1) * sizeof(T), st) != cudaSuccess) return nullptr;
        ptrs.push_back(p);
        return (T *)p;
    }
    void release(void *p) {
        for (auto &q : ptrs)
            if (q == p) {
                cudaFreeAsync(q, st);
                q = nullptr;
            }
    }
    ~Dev() {
        for (void *p : ptrs)
            if (p) cudaFreeAsync(p, st);
    }
};

template <class T>
int up(T *d, const std::vector<T> &h, cudaStream_t st) {
    if (h.empty()) return 0;
    return cudaMemcpyAsync(d, h.data(), h.size() * sizeof(T), cudaMemcpyHostToDevice, st) == cudaSuccess ? 0 : 1;
}
template <class T>
int down(std::vector<T> &h, const T *d, size_t n, cudaStream_t st) {
    h.resize(n);
    if (!n) return 0;
    if (cudaMemcpyAsync(h.data(), d, n * sizeof(T), cudaMemcpyDeviceToHost, st) != cudaSuccess) return 1;
    return cudaStreamSynchronize(st) == cudaSuccess ? 0 : 1;
}

#define KG_TRY(x)                              \
    do {                                       \
        if ((x) != 0) return MR_ERR_CUDA;      \
    } while (0)
#define KG_NEW(var, T, n)                      \
    T *var = dev.get<T>(n);                    \
    if (!var) return MR_ERR_NOMEM

// `words` fresh 32-bit words of Hash_DRBG output into a new scratch buffer of dev (rng's streams each
// contribute one request of <= 2^16 bytes per generate call; several calls if more is needed)
u32 *draw(Dev &dev, mr_drbg *rng, size_t words, cudaStream_t st) {
    const size_t S = mr_internal_drbg_streams(rng);
    const size_t per = std::min<size_t>(65536, ((words * 4 + S - 1) / S + 3) / 4 * 4);
    const size_t chunk = S * per, calls = (words * 4 + chunk - 1) / chunk;
    u32 *buf = dev.get<u32>(calls * chunk / 4);
    if (!buf) return nullptr;
    for (size_t i = 0; i < calls; i++)
        if (mr_drbg_generate(rng, reinterpret_cast<uint8_t *>(buf) + i * chunk, per, st) != MR_OK) return nullptr;
    return buf;
}

// Runs searches (one per entry of `index`) to completion; prime of search s -> pool row row0 + s.
// rng != NULL (mr_rsa_keygen_batch_drbg): starts and every Miller-Rabin base come from the DRBG instead
// of the seeded recipe (index is then only a count).
// Every iteration is ONE Miller-Rabin launch of one-round items: phase-A items (the next G sieve
// survivors of each search in phase A, base 2) and verification items (rounds 2..R of the candidate
// each search in phase V found in the previous iteration).
int run_searches(Dev &dev, cudaStream_t st, const std::vector<u64> &index, u32 L, int rounds, u64 seed,
                 const u32 *d_small, const u32 *d_pw, const u64 *d_mu, u32 *pool, u32 row0, int device,
                 mr_drbg *rng) {
    const u32 S = (u32)index.size();
    const u32 W = kWindow, R = (u32)rounds;
    KG_NEW(d_index, u64, S);
    KG_NEW(d_starts, u32, (size_t)S * L);
    KG_NEW(d_window, u32, S);
    KG_NEW(d_tested, u32, S);
    KG_NEW(d_bitmap, u32, (size_t)S * (W / 32));
    KG_NEW(d_list, u32, S);
    KG_NEW(d_vlist, u32, S);
    KG_NEW(d_ncand, u32, S);
    KG_NEW(d_vcand, u32, (size_t)S * L);
    // items: phase A <= max(8 S, kTarget + S); verification <= S (R - 1)
    const size_t capA = std::max<size_t>((size_t)S * 8, (size_t)kTarget + S);
    const size_t cap = capA + (size_t)S * (R - 1);
    KG_NEW(d_cand, u32, cap * L);
    KG_NEW(d_base, u32, cap * L);
    KG_NEW(d_verd, uint8_t, cap);
    KG_NEW(d_rows, u32, 2 * (size_t)S);
    if (rng) {
        const u32 *rnd = draw(dev, rng, (size_t)S * L, st);
        if (!rnd) return MR_ERR_CUDA;
        KG_TRY(kg_launch_start_rand(rnd, S, L, d_starts, st));
    } else {
        KG_TRY(up(d_index, index, st));
        KG_TRY(kg_launch_start(seed, d_index, S, L, d_starts, st));
    }

    std::vector<u32> window(S, 0), tested(S, 0), pend_first(S, 0), resieve(S), ncand;
    std::vector<uint8_t> verd;
    std::vector<char> found(S, 0), verify(S, 0);
    std::vector<u32> act(S);
    for (u32 s = 0; s < S; s++) resieve[s] = act[s] = s;
    int guard = 0;
    while (!act.empty()) {
        if (++guard > 1000000) return MR_ERR_CUDA;
        std::vector<u32> A, V;
        for (u32 s : act) (verify[s] ? V : A).push_back(s);
        KG_TRY(up(d_window, window, st));
        KG_TRY(up(d_tested, tested, st));
        if (!resieve.empty()) {
            KG_TRY(up(d_list, resieve, st));
            KG_TRY(kg_launch_sieve(d_starts, d_window, d_list, (u32)resieve.size(), L, d_small + 1, d_pw, d_mu,
                                   kNumSmall - 1, W, d_bitmap, st));
            resieve.clear();
        }
        const u32 nA = (u32)A.size(), nV = (u32)V.size();
        const u32 G = nA ? std::min<u32>(kMaxG, std::max<u32>(8, (kTarget + nA - 1) / nA)) : 0;
        const size_t itemsA = (size_t)nA * G, items = itemsA + (size_t)nV * (R - 1);
        KG_TRY(up(d_list, A, st));
        KG_TRY(up(d_vlist, V, st));
        KG_TRY(kg_launch_pick(d_starts, d_window, d_bitmap, d_tested, d_list, nA, L, W, G, d_cand, d_base, d_ncand,
                              st));
        KG_TRY(kg_launch_vitems(d_vlist, nV, d_vcand, d_small, R, L, d_cand + itemsA * L, d_base + itemsA * L, st));
        if (rng && items) {   // every item (candidate, round) gets its own random base
            Dev rscratch(st);
            const u32 *rnd = draw(rscratch, rng, items * (L + 2), st);
            if (!rnd) return MR_ERR_CUDA;
            KG_TRY(kg_launch_rand_bases(d_cand, rnd, (u32)items, L, d_base, st));
        }
        if (items) {
            int rc = mr_internal_miller_rabin(d_cand, L, items, d_base, 1, 0, d_verd, nullptr, nullptr, device, st, 0,
                                              4);   // w = 5 measured slower here (KG 64 rounds: 14.6 k -> 11.8 k keys/s)
            if (rc != MR_OK) return rc;
        }
        KG_TRY(down(ncand, d_ncand, nA, st));
        KG_TRY(down(verd, d_verd, items, st));
        std::vector<u32> to_v_src, to_v_dst, to_p_src, to_p_dst, vc_src, vc_dst;
        for (u32 a = 0; a < nA; a++) {
            const u32 s = A[a];
            int f = -1;
            for (u32 g = 0; g < ncand[a]; g++)
                if (verd[(size_t)a * G + g] == MR_PROBABLY_PRIME) { f = (int)g; break; }
            if (f >= 0) {
                if (R == 1) {                        // one round: the first passer is the prime
                    found[s] = 1;
                    to_p_src.push_back(a * G + (u32)f);
                    to_p_dst.push_back(row0 + s);
                } else {
                    verify[s] = 1;
                    pend_first[s] = (u32)f;
                    to_v_src.push_back(a * G + (u32)f);
                    to_v_dst.push_back(s);
                }
            } else {
                tested[s] += ncand[a];
                if (ncand[a] < G) {                  // window exhausted: next window
                    window[s]++;
                    tested[s] = 0;
                    resieve.push_back(s);
                }
            }
        }
        for (u32 v = 0; v < nV; v++) {
            const u32 s = V[v];
            bool ok = true;
            for (u32 r = 0; r + 1 < R; r++) ok &= verd[itemsA + (size_t)v * (R - 1) + r] == MR_PROBABLY_PRIME;
            verify[s] = 0;
            if (ok) {
                found[s] = 1;
                vc_src.push_back(s);
                vc_dst.push_back(row0 + s);
            } else {
                tested[s] += pend_first[s] + 1;      // resume after the failed candidate
            }
        }
        auto copy = [&](const u32 *src, std::vector<u32> &sr, u32 *dst, std::vector<u32> &dr) {
            if (sr.empty()) return 0;
            if (up(d_rows, sr, st) || up(d_rows + S, dr, st)) return 1;
            return kg_launch_copy_rows(src, d_rows, dst, d_rows + S, (u32)sr.size(), L, st);
        };
        // d_rows is reused by the three copies: the uploads and kernels are ordered on one stream, and
        // pageable uploads are staged before cudaMemcpyAsync returns, so the host vectors may go away
        KG_TRY(copy(d_cand, to_p_src, pool, to_p_dst));
        KG_TRY(copy(d_cand, to_v_src, d_vcand, to_v_dst));
        KG_TRY(copy(d_vcand, vc_src, pool, vc_dst));
        std::vector<u32> next;
        for (u32 s : act)
            if (!found[s]) next.push_back(s);
        act.swap(next);
    }
    return cudaStreamSynchronize(st) == cudaSuccess ? MR_OK : MR_ERR_CUDA;
}

}  // namespace
}  // namespace mr

using namespace mr;

static int keygen_impl(mr_drbg *rng, size_t count, int bits, uint32_t e, uint64_t seed, uint64_t first_key, int rounds,
                       uint32_t *d_n, uint32_t *d_p, uint32_t *d_q, uint32_t *d_d, uint32_t *d_dp, uint32_t *d_dq,
                       uint32_t *d_qinv, int device, void *stream) {
    if (bits < 256 || bits > 4096 || bits % 64 != 0 || e < 3 || !is_prime_u32(e) || rounds < 1 || rounds > 256 ||
        count > (1u << 24))
        return MR_ERR_ARG;
    if (count && (!d_n || !d_p || !d_q || !d_d || !d_dp || !d_dq || !d_qinv)) return MR_ERR_ARG;
    if ((first_key + count) > (UINT64_MAX >> 16)) return MR_ERR_ARG;
    if (count == 0) return MR_OK;
    if (cudaSetDevice(device) != cudaSuccess) return MR_ERR_CUDA;
    cudaStream_t st = (cudaStream_t)stream;
    const u32 L = (u32)bits / 64;                      // limbs of a prime
    Dev dev(st);
    const std::vector<u32> &sp = small_primes();
    KG_NEW(d_small, u32, kNumSmall);
    KG_TRY(up(d_small, sp, st));
    KG_NEW(d_pw, u32, (size_t)L * (kNumSmall - 1));
    KG_NEW(d_mu, u64, kNumSmall - 1);
    KG_TRY(kg_launch_pow(d_small + 1, kNumSmall - 1, L, d_pw, d_mu, st));      // odd primes

    // prime pool: every prime found, in search order; grows as keys need more attempts
    u32 cap = (u32)(2 * count + 64), npool = 0;
    u32 *pool = dev.get<u32>((size_t)cap * L);
    if (!pool) return MR_ERR_NOMEM;

    struct Row {
        u32 row, first_used, flags;
    };
    std::vector<int> kp(count, -1), kq(count, -1);
    std::vector<u32> attempt(count, 0);
    std::vector<std::deque<Row>> pend(count);
    size_t remaining = count;
    while (remaining) {
        std::vector<u64> index;
        std::vector<u32> owner;
        for (size_t i = 0; i < count; i++) {
            if (kq[i] >= 0) continue;
            const int need = (kp[i] < 0 ? 2 : 1) - (int)pend[i].size();
            for (int j = 0; j < need; j++) {
                if (attempt[i] >= 65536) return MR_ERR_RANGE;
                index.push_back((first_key + i) * 65536ull + attempt[i]++);
                owner.push_back((u32)i);
            }
        }
        const u32 S = (u32)index.size();
        if (npool + S > cap) {                         // grow the pool
            const u32 ncap = std::max<u32>(cap * 2, npool + S);
            u32 *np = dev.get<u32>((size_t)ncap * L);
            if (!np) return MR_ERR_NOMEM;
            if (npool && cudaMemcpyAsync(np, pool, (size_t)npool * L * 4, cudaMemcpyDeviceToDevice, st) != cudaSuccess)
                return MR_ERR_CUDA;
            dev.release(pool);
            pool = np;
            cap = ncap;
        }
        {
            Dev scratch(st);
            int rc = run_searches(scratch, st, index, L, rounds, seed, d_small, d_pw, d_mu, pool, npool, device, rng);
            if (rc != MR_OK) return rc;
        }
        for (u32 s = 0; s < S; s++) pend[owner[s]].push_back(Row{npool + s, 0xFFFFFFFEu, 0});
        npool += S;
        // acceptance in attempt order: gcd(e, p - 1) = 1 for both; |p - q| > 2^(bits/2 - 100) for q
        for (int pass = 0; pass < 4; pass++) {
            std::vector<u32> which, firsts;
            std::vector<std::pair<u32, u32>> where;
            for (size_t i = 0; i < count; i++) {
                if (kq[i] >= 0) continue;
                const u32 want = kp[i] < 0 ? 0xFFFFFFFFu : (u32)kp[i];
                for (size_t r = 0; r < pend[i].size(); r++)
                    if (pend[i][r].first_used != want) {
                        which.push_back(pend[i][r].row);
                        firsts.push_back(want);
                        where.push_back({(u32)i, (u32)r});
                    }
            }
            if (which.empty()) break;
            Dev scratch(st);
            KG_NEW(d_which, u32, which.size());
            KG_NEW(d_firsts, u32, which.size());
            KG_NEW(d_ok, u32, which.size());
            KG_TRY(up(d_which, which, st));
            KG_TRY(up(d_firsts, firsts, st));
            KG_TRY(kg_launch_check(pool, L, e, d_which, d_firsts, (u32)which.size(), d_ok, st));
            std::vector<u32> ok;
            KG_TRY(down(ok, d_ok, which.size(), st));
            for (size_t w = 0; w < which.size(); w++) {
                Row &r = pend[where[w].first][where[w].second];
                r.first_used = firsts[w];
                r.flags = ok[w];
            }
            for (size_t i = 0; i < count; i++) {
                while (kq[i] < 0 && !pend[i].empty()) {
                    const Row r = pend[i].front();
                    if (!(r.flags & 1u) && r.first_used != 0xFFFFFFFEu) { pend[i].pop_front(); continue; }
                    if (r.first_used == 0xFFFFFFFEu) break;
                    if (kp[i] < 0) {
                        kp[i] = (int)r.row;
                        pend[i].pop_front();
                        continue;                   // later rows were tested against no p: recheck
                    }
                    if (r.first_used != (u32)kp[i]) break;
                    pend[i].pop_front();
                    if (r.flags & 2u) {
                        kq[i] = (int)r.row;
                        pend[i].clear();
                        remaining--;
                    }
                }
            }
        }
    }
    std::vector<u32> ks(2 * count);
    for (size_t i = 0; i < count; i++) {
        ks[2 * i] = (u32)kp[i];
        ks[2 * i + 1] = (u32)kq[i];
    }
    KG_NEW(d_ks, u32, ks.size());
    KG_TRY(up(d_ks, ks, st));
    KG_TRY(kg_launch_assemble(pool, d_ks, (u32)count, L, e, d_n, d_p, d_q, d_d, d_dp, d_dq, d_qinv, st));
    return cudaStreamSynchronize(st) == cudaSuccess ? MR_OK : MR_ERR_CUDA;
}

#pragma GCC visibility push(default)
extern "C" int mr_rsa_keygen_batch(size_t count, int bits, uint32_t e, uint64_t seed, uint64_t first_key, int rounds,
                                   uint32_t *d_n, uint32_t *d_p, uint32_t *d_q, uint32_t *d_d, uint32_t *d_dp,
                                   uint32_t *d_dq, uint32_t *d_qinv, int device, void *stream) {
    return keygen_impl(nullptr, count, bits, e, seed, first_key, rounds, d_n, d_p, d_q, d_d, d_dp, d_dq, d_qinv,
                       device, stream);
}

extern "C" int mr_rsa_keygen_batch_drbg(mr_drbg *rng, size_t count, int bits, uint32_t e, int rounds, uint32_t *d_n,
                                        uint32_t *d_p, uint32_t *d_q, uint32_t *d_d, uint32_t *d_dp, uint32_t *d_dq,
                                        uint32_t *d_qinv, int device, void *stream) {
    if (!rng) return MR_ERR_ARG;
    return keygen_impl(rng, count, bits, e, 0, 0, rounds, d_n, d_p, d_q, d_d, d_dp, d_dq, d_qinv, device, stream);
}
#pragma GCC visibility pop
