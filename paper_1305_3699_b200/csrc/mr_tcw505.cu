// mr_tcw505.cu — the tensor-core wide modexp kernel (mr_tcw.cuh) at k = 505: 16,128-bit moduli (P:48
// §3.1 "up to 16,128-bit long RSA keys").  A 128-message A tile would be 256 KB (2,048-byte rows) and the B residues
// alone 508 TMEM columns, so this instantiation runs 64-message tiles (M = 64 MMAs: the accumulator sits in lanes
// 16q .. 16q + 15 of each quadrant, the upper lanes of a warp shadow the lower ones) and keeps the B residues in an
// L2-resident global scratch slot; the A tile (128 KB) holds the whole row, so no contraction is split along K.
#include <cuda_runtime.h>
#include <cstdint>
#include <cstdio>
#include <cstdlib>

#include "mr_internal.h"

#define MR_K 505

namespace mr {
namespace {

constexpr int K = MR_K;
constexpr int NCH = 2 * K + 1;                // residues per value: B, B', m_r
// exit: X < (K+3) N <= 2^(SMAX+1) N (plain lazy digits, as mr_kernels.cuh for K > 65)
constexpr int KB = K + 3;
constexpr int SMAX = (32 - __builtin_clz((unsigned)(KB - 1))) - 1;

// T = thi 2^32 + tlo -> T 2^-32 mod m, lazy in [0, 2^32) (word Montgomery reduction, as mr_kernels.cuh)
__device__ __forceinline__ u32 mont_red(u32 tlo, u32 thi, u32 m, u32 minv) {
    const u32 q = tlo * minv;
    [[maybe_unused]] u32 ulo;
    u32 uhi, cy;
    asm("mad.lo.cc.u32 %0, %3, %4, %5;\n\tmadc.hi.cc.u32 %1, %3, %4, %6;\n\taddc.u32 %2, 0, 0;"
        : "=r"(ulo), "=r"(uhi), "=r"(cy)
        : "r"(q), "r"(m), "r"(tlo), "r"(thi));
    return cy ? uhi - m : uhi;
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

#include "mr_tcw.cuh"

}  // namespace

// ctas = persistent CTAs (one per SM); same contract as the per-k launch_modexp_tcw of mr_kernels.cuh
int launch_modexp_tcw_k505(const ModexpParams &p, u32 ctas, const u32 *tab, const void *kimg, u32 cxw, u32 be1w, u32 jobs,
                           void *trace, void *stream) {
    return tcw_launch(p, ctas, TcwArgs{tab, reinterpret_cast<const uint8_t *>(kimg), cxw, be1w, jobs,
                                       reinterpret_cast<unsigned long long *>(trace)}, stream);
}

}  // namespace mr
