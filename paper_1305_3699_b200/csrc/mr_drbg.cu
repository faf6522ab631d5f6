// mr_drbg.cu — the DRBG and FIPS 140-2 health-test kernels of the MR-TRNG layer (
// DESIGN.md §4i).  The paper seeds "an approved deterministic RBG" from GPU entropy (§2) and runs "a
// self-validating kernel [that] streamlines FIPS basic tests right after the generation" (§4.2);
// entropy harvesting itself is out of scope — the caller supplies entropy_input and nonce.
//
// Readings (R20-R22): Hash_DRBG with SHA-256 (NIST SP 800-90A §10.1.1, seedlen = 440, no
// additional input, no prediction resistance); `streams` independent instances, stream s personalised with
// pers || be32(s); the FIPS 140-2 §4.9.1 monobit / poker / runs / long-run tests on 20,000-bit blocks.
//
// B200 mapping: Hashgen is counter mode over V (data = V + i), so every 32-byte output block is one
// SHA-256 compression of a 55-byte message — one thread per output block, the whole request in one
// launch (integer-ALU bound: 64 rounds of 32-bit adds, rotates and logic).  The state update
// (V += Hash(0x03 || V) + C + reseed_counter) is one thread per stream.  The health test runs one CTA per
// block with bit-parallel run counting: for each bit value b and run length l, the run starts p (bit p = b,
// bit p-1 != b) whose next l bits are all b are counted with shifted-AND masks and popcounts, so no
// sequential bit walk is needed.
#include <cuda_runtime.h>

#include <cstdint>
#include <cstring>
#include <new>
#include <vector>

#include "../../include/mr_rns.h"

namespace mr {
namespace {

typedef uint32_t u32;
typedef uint64_t u64;

constexpr u32 VW = 14;                 // V, C: 440-bit integers as 14 big-endian u32 limbs (limb 0 < 2^24)

__host__ __device__ inline u32 rotr(u32 x, int n) { return (x >> n) | (x << (32 - n)); }

__constant__ u32 K256[64] = {
    0x428a2f98, 0x71374491, 0xb5c0fbcf, 0xe9b5dba5, 0x3956c25b, 0x59f111f1, 0x923f82a4, 0xab1c5ed5, 0xd807aa98,
    0x12835b01, 0x243185be, 0x550c7dc3, 0x72be5d74, 0x80deb1fe, 0x9bdc06a7, 0xc19bf174, 0xe49b69c1, 0xefbe4786,
    0x0fc19dc6, 0x240ca1cc, 0x2de92c6f, 0x4a7484aa, 0x5cb0a9dc, 0x76f988da, 0x983e5152, 0xa831c66d, 0xb00327c8,
    0xbf597fc7, 0xc6e00bf3, 0xd5a79147, 0x06ca6351, 0x14292967, 0x27b70a85, 0x2e1b2138, 0x4d2c6dfc, 0x53380d13,
    0x650a7354, 0x766a0abb, 0x81c2c92e, 0x92722c85, 0xa2bfe8a1, 0xa81a664b, 0xc24b8b70, 0xc76c51a3, 0xd192e819,
    0xd6990624, 0xf40e3585, 0x106aa070, 0x19a4c116, 0x1e376c08, 0x2748774c, 0x34b0bcb5, 0x391c0cb3, 0x4ed8aa4a,
    0x5b9cca4f, 0x682e6ff3, 0x748f82ee, 0x78a5636f, 0x84c87814, 0x8cc70208, 0x90befffa, 0xa4506ceb, 0xbef9a3f7,
    0xc67178f2};
static const u32 K256_HOST[64] = {
    0x428a2f98, 0x71374491, 0xb5c0fbcf, 0xe9b5dba5, 0x3956c25b, 0x59f111f1, 0x923f82a4, 0xab1c5ed5, 0xd807aa98,
    0x12835b01, 0x243185be, 0x550c7dc3, 0x72be5d74, 0x80deb1fe, 0x9bdc06a7, 0xc19bf174, 0xe49b69c1, 0xefbe4786,
    0x0fc19dc6, 0x240ca1cc, 0x2de92c6f, 0x4a7484aa, 0x5cb0a9dc, 0x76f988da, 0x983e5152, 0xa831c66d, 0xb00327c8,
    0xbf597fc7, 0xc6e00bf3, 0xd5a79147, 0x06ca6351, 0x14292967, 0x27b70a85, 0x2e1b2138, 0x4d2c6dfc, 0x53380d13,
    0x650a7354, 0x766a0abb, 0x81c2c92e, 0x92722c85, 0xa2bfe8a1, 0xa81a664b, 0xc24b8b70, 0xc76c51a3, 0xd192e819,
    0xd6990624, 0xf40e3585, 0x106aa070, 0x19a4c116, 0x1e376c08, 0x2748774c, 0x34b0bcb5, 0x391c0cb3, 0x4ed8aa4a,
    0x5b9cca4f, 0x682e6ff3, 0x748f82ee, 0x78a5636f, 0x84c87814, 0x8cc70208, 0x90befffa, 0xa4506ceb, 0xbef9a3f7,
    0xc67178f2};
static const u32 IV256[8] = {0x6a09e667, 0xbb67ae85, 0x3c6ef372, 0xa54ff53a,
                             0x510e527f, 0x9b05688c, 0x1f83d9ab, 0x5be0cd19};

// FIPS 180-2 SHA-256 compression of one 16-word (big-endian) message block into h
__device__ __forceinline__ void sha256_block(u32 (&h)[8], const u32 (&m)[16]) {
    u32 w[16];
#pragma unroll
    for (int t = 0; t < 16; t++) w[t] = m[t];
    u32 a = h[0], b = h[1], c = h[2], d = h[3], e = h[4], f = h[5], g = h[6], hh = h[7];
#pragma unroll
    for (int t = 0; t < 64; t++) {
        if (t >= 16) {
            const u32 x = w[(t - 15) & 15], y = w[(t - 2) & 15];
            const u32 s0 = rotr(x, 7) ^ rotr(x, 18) ^ (x >> 3), s1 = rotr(y, 17) ^ rotr(y, 19) ^ (y >> 10);
            w[t & 15] += s0 + w[(t - 7) & 15] + s1;
        }
        const u32 S1 = rotr(e, 6) ^ rotr(e, 11) ^ rotr(e, 25);
        const u32 ch = (e & f) ^ (~e & g);
        const u32 t1 = hh + S1 + ch + K256[t] + w[t & 15];
        const u32 S0 = rotr(a, 2) ^ rotr(a, 13) ^ rotr(a, 22);
        const u32 mj = (a & b) ^ (a & c) ^ (b & c);
        const u32 t2 = S0 + mj;
        hh = g;
        g = f;
        f = e;
        e = d + t1;
        d = c;
        c = b;
        b = a;
        a = t1 + t2;
    }
    h[0] += a; h[1] += b; h[2] += c; h[3] += d; h[4] += e; h[5] += f; h[6] += g; h[7] += hh;
}

// V + i (i < 2^32) in place, mod 2^440
__device__ __forceinline__ void add_small(u32 (&v)[VW], u32 i) {
    u64 c = i;
#pragma unroll
    for (int l = VW - 1; l >= 0; l--) {
        const u64 s = (u64)v[l] + c;
        v[l] = (u32)s;
        c = s >> 32;
    }
    v[0] &= 0x00FFFFFFu;
}

// Hashgen block i of every stream: out[s][32 i .. 32 i + 31] = SHA-256((V_s + i) as 55 bytes)
__global__ void k_drbg_generate(const u32 *__restrict__ V, uint8_t *__restrict__ out, u32 streams, u32 nblk,
                                u32 nbytes) {
    const u64 t = (u64)blockIdx.x * blockDim.x + threadIdx.x;
    if (t >= (u64)streams * nblk) return;
    const u32 s = (u32)(t / nblk), i = (u32)(t % nblk);
    u32 v[VW];
#pragma unroll
    for (int l = 0; l < (int)VW; l++) v[l] = __ldg(V + (size_t)s * VW + l);
    add_small(v, i);
    u32 m[16];   // 55 message bytes || 0x80, bit length 440
#pragma unroll
    for (int w = 0; w < 13; w++) m[w] = (v[w] << 8) | (v[w + 1] >> 24);
    m[13] = (v[13] << 8) | 0x80u;
    m[14] = 0;
    m[15] = 440;
    u32 h[8] = {0x6a09e667, 0xbb67ae85, 0x3c6ef372, 0xa54ff53a, 0x510e527f, 0x9b05688c, 0x1f83d9ab, 0x5be0cd19};
    sha256_block(h, m);
    uint8_t *o = out + (size_t)s * nbytes + (size_t)i * 32;
    const u32 rem = nbytes - i * 32;
    if (rem >= 32 && (((uintptr_t)o) & 15) == 0) {
        uint4 *o4 = reinterpret_cast<uint4 *>(o);
        o4[0] = make_uint4(__byte_perm(h[0], 0, 0x0123), __byte_perm(h[1], 0, 0x0123), __byte_perm(h[2], 0, 0x0123),
                           __byte_perm(h[3], 0, 0x0123));
        o4[1] = make_uint4(__byte_perm(h[4], 0, 0x0123), __byte_perm(h[5], 0, 0x0123), __byte_perm(h[6], 0, 0x0123),
                           __byte_perm(h[7], 0, 0x0123));
    } else {
        for (u32 b = 0; b < 32 && b < rem; b++) o[b] = (uint8_t)(h[b >> 2] >> (24 - 8 * (b & 3)));
    }
}

// V = (V + Hash(0x03 || V) + C + reseed_counter) mod 2^440; reseed_counter += 1  (SP 800-90A §10.1.1.4)
__global__ void k_drbg_update(u32 *__restrict__ V, const u32 *__restrict__ C, u64 *__restrict__ rc, u32 streams) {
    const u32 s = blockIdx.x * blockDim.x + threadIdx.x;
    if (s >= streams) return;
    u32 v[VW];
    for (int l = 0; l < (int)VW; l++) v[l] = V[(size_t)s * VW + l];
    u32 m[16];   // block 1: 0x03 || V (56 bytes) || 0x80 || 0...; block 2: zeros || bit length 448
    m[0] = (3u << 24) | v[0];
    for (int w = 1; w < 14; w++) m[w] = v[w];
    m[14] = 0x80000000u;
    m[15] = 0;
    u32 h[8] = {0x6a09e667, 0xbb67ae85, 0x3c6ef372, 0xa54ff53a, 0x510e527f, 0x9b05688c, 0x1f83d9ab, 0x5be0cd19};
    sha256_block(h, m);
    for (int w = 0; w < 15; w++) m[w] = 0;
    m[15] = 448;
    sha256_block(h, m);
    const u64 r = rc[s];
    u64 c = 0;
    for (int l = VW - 1; l >= 0; l--) {
        u64 sum = (u64)v[l] + C[(size_t)s * VW + l] + c;
        if (l >= (int)VW - 8) sum += h[l - (VW - 8)];
        if (l == VW - 1) sum += (u32)r;
        if (l == VW - 2) sum += (u32)(r >> 32);
        v[l] = (u32)sum;
        c = sum >> 32;
    }
    v[0] &= 0x00FFFFFFu;
    for (int l = 0; l < (int)VW; l++) V[(size_t)s * VW + l] = v[l];
    rc[s] = r + 1;
}

// FIPS 140-2 §4.9.1 on 20,000-bit blocks (2,500 bytes, bits most significant first within each byte).
// stats[16] per block: ones, poker S = Σ f_i², runs of ones of length 1..5, 6+, runs of zeros 1..5, 6+,
// long-run flag (a run >= 26 exists), verdict bits (1 monobit, 2 poker, 4 runs, 8 long run: set = pass).
constexpr u32 HB_WORDS = 625;
__global__ void __launch_bounds__(128) k_fips_health(const uint8_t *__restrict__ blocks, u32 *__restrict__ stats) {
    __shared__ u32 acc[2 + 12 + 1 + 16];   // ones, (unused), runs[2][6], long flag, nibble counts
    const u32 tid = threadIdx.x;
    for (u32 q = tid; q < 31; q += blockDim.x) acc[q] = 0;
    __syncthreads();
    const u32 *wb = reinterpret_cast<const u32 *>(blocks + (size_t)blockIdx.x * 2500);
    u32 ones = 0, runs[2][6] = {{0}}, longf = 0, nib[16];
#pragma unroll
    for (int q = 0; q < 16; q++) nib[q] = 0;
    for (u32 wi = tid; wi < HB_WORDS; wi += blockDim.x) {
        // stream-order words: byte 0 of the word is the most significant byte (bits MSB first)
        const u32 cur = __byte_perm(__ldg(wb + wi), 0, 0x0123);
        const u32 prev = wi ? __byte_perm(__ldg(wb + wi - 1), 0, 0x0123) : 0u;
        const u32 next = wi + 1 < HB_WORDS ? __byte_perm(__ldg(wb + wi + 1), 0, 0x0123) : 0u;
        ones += __popc(cur);
        // nibble histogram without data-dependent indexing: for each value v, the nibbles of cur ^ (v * 0x11111111)
        // that are zero are the nibbles equal to v
#pragma unroll
        for (int v = 0; v < 16; v++) {
            const u32 z = cur ^ (0x11111111u * (u32)v);
            const u32 nz = (z | (z >> 1) | (z >> 2) | (z >> 3)) & 0x11111111u;
            nib[v] += 8 - __popc(nz);
        }
#pragma unroll
        for (int b = 0; b < 2; b++) {
            // y: 1 where the stream bit equals b; outside the block y = 0 (runs end at the block edges)
            const u32 yc = b ? cur : ~cur;
            const u32 yp = wi ? (b ? prev : ~prev) : 0u;
            const u32 yn = wi + 1 < HB_WORDS ? (b ? next : ~next) : 0u;
            const u32 start = yc & ~((yc >> 1) | (yp << 31));       // position j starts a run of b
            const u64 W = ((u64)yc << 32) | yn;                      // positions j .. j + 31 of the window
            u32 all = yc;                                            // y[j .. j + l - 1] all 1
            u32 ge[7];
            ge[0] = __popc(start & all);                             // runs of length >= 1
#pragma unroll
            for (int l = 1; l < 6; l++) {
                all &= (u32)((W << l) >> 32);
                ge[l] = __popc(start & all);                         // >= l + 1
            }
#pragma unroll
            for (int l = 6; l < 26; l++) all &= (u32)((W << l) >> 32);
            ge[6] = __popc(start & all);                             // >= 26
#pragma unroll
            for (int l = 0; l < 5; l++) runs[b][l] += ge[l] - ge[l + 1];
            runs[b][5] += ge[5];
            longf |= ge[6];
        }
    }
    atomicAdd(&acc[0], ones);
    for (int b = 0; b < 2; b++)
        for (int l = 0; l < 6; l++) atomicAdd(&acc[2 + 6 * (1 - b) + l], runs[b][l]);   // ones first, then zeros
    if (longf) atomicOr(&acc[14], 1u);
#pragma unroll
    for (int q = 0; q < 16; q++) {
        u32 x = nib[q];
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) x += __shfl_xor_sync(0xFFFFFFFFu, x, o);
        if ((tid & 31) == 0 && x) atomicAdd(&acc[15 + q], x);
    }
    __syncthreads();
    if (tid == 0) {
        u32 *o = stats + (size_t)blockIdx.x * 16;
        u64 s2 = 0;
        for (int q = 0; q < 16; q++) s2 += (u64)acc[15 + q] * acc[15 + q];
        const u32 one = acc[0];
        static const u32 lo[6] = {2315, 1114, 527, 240, 103, 103}, hi[6] = {2685, 1386, 723, 384, 209, 209};
        bool runs_ok = true;
        for (int l = 0; l < 12; l++) runs_ok &= acc[2 + l] >= lo[l % 6] && acc[2 + l] <= hi[l % 6];
        u32 verdict = 0;
        if (one > 9725 && one < 10275) verdict |= 1;
        if (16 * s2 > 25010800ull && 16 * s2 < 25230850ull) verdict |= 2;   // 2.16 < 16 S / 5000 - 5000 < 46.17
        if (runs_ok) verdict |= 4;
        if (!acc[14]) verdict |= 8;
        o[0] = one;
        o[1] = (u32)s2;
        for (int l = 0; l < 12; l++) o[2 + l] = acc[2 + l];
        o[14] = acc[14];
        o[15] = verdict;
    }
}

// ---------------------------------------------------------------- host: SHA-256, Hash_df, instantiate
struct Sha256 {
    u32 h[8];
    std::vector<uint8_t> buf;
    u64 len = 0;
    Sha256() { memcpy(h, IV256, sizeof h); }
    void block(const uint8_t *p) {
        u32 w[64];
        for (int t = 0; t < 16; t++) w[t] = (u32)p[4 * t] << 24 | (u32)p[4 * t + 1] << 16 | (u32)p[4 * t + 2] << 8 | p[4 * t + 3];
        for (int t = 16; t < 64; t++) {
            const u32 s0 = rotr(w[t - 15], 7) ^ rotr(w[t - 15], 18) ^ (w[t - 15] >> 3);
            const u32 s1 = rotr(w[t - 2], 17) ^ rotr(w[t - 2], 19) ^ (w[t - 2] >> 10);
            w[t] = w[t - 16] + s0 + w[t - 7] + s1;
        }
        u32 a = h[0], b = h[1], c = h[2], d = h[3], e = h[4], f = h[5], g = h[6], hh = h[7];
        for (int t = 0; t < 64; t++) {
            const u32 t1 = hh + (rotr(e, 6) ^ rotr(e, 11) ^ rotr(e, 25)) + ((e & f) ^ (~e & g)) + K256_HOST[t] + w[t];
            const u32 t2 = (rotr(a, 2) ^ rotr(a, 13) ^ rotr(a, 22)) + ((a & b) ^ (a & c) ^ (b & c));
            hh = g; g = f; f = e; e = d + t1; d = c; c = b; b = a; a = t1 + t2;
        }
        h[0] += a; h[1] += b; h[2] += c; h[3] += d; h[4] += e; h[5] += f; h[6] += g; h[7] += hh;
    }
    void update(const uint8_t *p, size_t n) {
        len += n;
        buf.insert(buf.end(), p, p + n);
        size_t off = 0;
        for (; off + 64 <= buf.size(); off += 64) block(buf.data() + off);
        buf.erase(buf.begin(), buf.begin() + off);
    }
    void digest(uint8_t out[32]) {
        const u64 bits = len * 8;
        buf.push_back(0x80);
        while (buf.size() % 64 != 56) buf.push_back(0);
        for (int q = 7; q >= 0; q--) buf.push_back((uint8_t)(bits >> (8 * q)));
        for (size_t off = 0; off < buf.size(); off += 64) block(buf.data() + off);
        for (int q = 0; q < 8; q++)
            for (int b = 0; b < 4; b++) out[4 * q + b] = (uint8_t)(h[q] >> (24 - 8 * b));
    }
};

// SP 800-90A §10.3.1 Hash_df(input, 440) -> 55 bytes
static void hash_df440(const std::vector<uint8_t> &in, uint8_t out[55]) {
    uint8_t t[64];
    for (int ctr = 1; ctr <= 2; ctr++) {
        Sha256 s;
        const uint8_t hdr[5] = {(uint8_t)ctr, 0, 0, 0x01, 0xB8};   // counter, no_of_bits = 440 (big-endian)
        s.update(hdr, 5);
        s.update(in.data(), in.size());
        s.digest(t + 32 * (ctr - 1));
    }
    memcpy(out, t, 55);
}

static void bytes_to_limbs(const uint8_t b[55], u32 v[VW]) {   // 55 big-endian bytes -> 14 limbs
    v[0] = (u32)b[0] << 16 | (u32)b[1] << 8 | b[2];
    for (int l = 1; l < (int)VW; l++)
        v[l] = (u32)b[3 + 4 * (l - 1)] << 24 | (u32)b[4 + 4 * (l - 1)] << 16 | (u32)b[5 + 4 * (l - 1)] << 8 | b[6 + 4 * (l - 1)];
}

}  // namespace
}  // namespace mr

struct mr_drbg {
    uint32_t streams = 0;
    int device = 0;
    uint32_t *d_V = nullptr, *d_C = nullptr;
    uint64_t *d_rc = nullptr;
    uint64_t reseed_counter = 1;   // host mirror (all streams advance together)
};

extern "C" {

uint32_t mr_internal_drbg_streams(const mr_drbg *d) { return d ? d->streams : 0; }

int mr_drbg_create(mr_drbg **out, const uint8_t *entropy, size_t entropy_len, const uint8_t *nonce, size_t nonce_len,
                   const uint8_t *pers, size_t pers_len, uint32_t streams, int device) {
    using namespace mr;
    if (!out) return MR_ERR_ARG;
    *out = nullptr;
    if (!entropy || entropy_len < 32 || !nonce || nonce_len < 16 || (pers_len && !pers) || streams == 0)
        return MR_ERR_ARG;   // SP 800-90A: entropy >= security strength (256 bits), nonce >= 128 bits
    std::vector<u32> V((size_t)streams * VW), C((size_t)streams * VW);
    std::vector<uint8_t> material(entropy, entropy + entropy_len);
    material.insert(material.end(), nonce, nonce + nonce_len);
    material.insert(material.end(), pers, pers + pers_len);
    const size_t base = material.size();
    material.resize(base + 4);
    for (uint32_t s = 0; s < streams; s++) {   // personalization = pers || be32(s)
        for (int b = 0; b < 4; b++) material[base + b] = (uint8_t)(s >> (24 - 8 * b));
        uint8_t seed[55], c[55];
        hash_df440(material, seed);
        std::vector<uint8_t> cin(1, 0x00);
        cin.insert(cin.end(), seed, seed + 55);
        hash_df440(cin, c);
        bytes_to_limbs(seed, V.data() + (size_t)s * VW);
        bytes_to_limbs(c, C.data() + (size_t)s * VW);
    }
    mr_drbg *d = new (std::nothrow) mr_drbg;
    if (!d) return MR_ERR_NOMEM;
    d->streams = streams;
    d->device = device;
    std::vector<uint64_t> rc(streams, 1);
    if (cudaSetDevice(device) != cudaSuccess || cudaMalloc(&d->d_V, V.size() * 4) != cudaSuccess ||
        cudaMalloc(&d->d_C, C.size() * 4) != cudaSuccess || cudaMalloc(&d->d_rc, rc.size() * 8) != cudaSuccess ||
        cudaMemcpy(d->d_V, V.data(), V.size() * 4, cudaMemcpyHostToDevice) != cudaSuccess ||
        cudaMemcpy(d->d_C, C.data(), C.size() * 4, cudaMemcpyHostToDevice) != cudaSuccess ||
        cudaMemcpy(d->d_rc, rc.data(), rc.size() * 8, cudaMemcpyHostToDevice) != cudaSuccess) {
        if (d->d_V) cudaFree(d->d_V);
        if (d->d_C) cudaFree(d->d_C);
        if (d->d_rc) cudaFree(d->d_rc);
        delete d;
        return MR_ERR_CUDA;
    }
    *out = d;
    return MR_OK;
}

void mr_drbg_destroy(mr_drbg *d) {
    if (!d) return;
    cudaFree(d->d_V);
    cudaFree(d->d_C);
    cudaFree(d->d_rc);
    delete d;
}

int mr_drbg_generate(mr_drbg *d, uint8_t *d_out, size_t nbytes, void *stream) {
    using namespace mr;
    if (!d || (nbytes && !d_out) || nbytes > (1u << 19) / 8) return MR_ERR_ARG;   // <= 2^19 bits per request
    if (d->reseed_counter > (1ull << 48)) return MR_ERR_RANGE;                    // reseed_interval (never reached)
    if (cudaSetDevice(d->device) != cudaSuccess) return MR_ERR_CUDA;
    cudaStream_t st = (cudaStream_t)stream;
    const u32 nblk = (u32)((nbytes + 31) / 32);
    const u64 threads = (u64)d->streams * nblk;
    if (threads) {
        k_drbg_generate<<<(unsigned)((threads + 255) / 256), 256, 0, st>>>(d->d_V, d_out, d->streams, nblk, (u32)nbytes);
        if (cudaGetLastError() != cudaSuccess) return MR_ERR_CUDA;
    }
    k_drbg_update<<<(d->streams + 127) / 128, 128, 0, st>>>(d->d_V, d->d_C, d->d_rc, d->streams);
    if (cudaGetLastError() != cudaSuccess) return MR_ERR_CUDA;
    d->reseed_counter++;
    return MR_OK;
}

int mr_fips_health_batch(const uint8_t *d_blocks, size_t nblocks, uint32_t *d_stats, void *stream) {
    using namespace mr;
    if (nblocks && (!d_blocks || !d_stats)) return MR_ERR_ARG;
    if (nblocks == 0) return MR_OK;
    if (nblocks > 0x7FFFFFFFu) return MR_ERR_ARG;
    k_fips_health<<<(unsigned)nblocks, 128, 0, (cudaStream_t)stream>>>(d_blocks, d_stats);
    return cudaGetLastError() == cudaSuccess ? MR_OK : MR_ERR_CUDA;
}

}  // extern "C"
