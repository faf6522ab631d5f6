// tc_i8_test.cu — standalone check of the tcgen05 kind::i8 building blocks used by the tensor-core
// base extension: K-major SWIZZLE_NONE shared-memory operands, UMMA descriptors, TMEM alloc,
// tcgen05.mma (u8 x u8 -> s32), commit to an mbarrier, tcgen05.ld.32x32b readback.
// One CTA of 128 threads computes D[128 x N] = A[128 x KB] · B[N x KB]^T and compares with the CPU.
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cuda_runtime.h>

typedef uint32_t u32;
typedef uint64_t u64;

constexpr int M = 128, N = 144, KB = 160;        // KB bytes of K (5 MMA steps of 32)
constexpr int SBO_A = (KB / 16) * 128;            // bytes between 8-row groups
constexpr int LBO = 128;                          // bytes between adjacent 16-byte K chunks

__device__ __forceinline__ u32 smem_u32(const void *p) { return (u32)__cvta_generic_to_shared(p); }

// core-matrix layout offset of (row r, k byte kb)
__host__ __device__ constexpr int off(int r, int kb) { return (r / 8) * SBO_A + (kb / 16) * LBO + (r % 8) * 16 + kb % 16; }

__device__ __forceinline__ u64 sdesc(u32 saddr, u32 lbo, u32 sbo) {
    u64 d = 0;
    d |= (u64)((saddr >> 4) & 0x3FFF);
    d |= (u64)((lbo >> 4) & 0x3FFF) << 16;
    d |= (u64)((sbo >> 4) & 0x3FFF) << 32;
    d |= (u64)1 << 46;                       // version = 1 (sm100)
    // base_offset 0, lbo_mode 0, layout SWIZZLE_NONE (0) in bits 61..63
    return d;
}

__global__ void k_test(const uint8_t *gA, const uint8_t *gB, int32_t *gD, u32 idesc) {
    extern __shared__ __align__(1024) uint8_t sm[];
    uint8_t *sA = sm;
    uint8_t *sB = sm + M * KB;
    u64 *mbar = (u64 *)(sB + N * KB);
    u32 *tslot = (u32 *)(mbar + 1);
    const int t = threadIdx.x, w = t / 32;
    for (int i = t; i < M * KB; i += blockDim.x) sA[off(i / KB, i % KB)] = gA[i];
    for (int i = t; i < N * KB; i += blockDim.x) sB[off(i / KB, i % KB)] = gB[i];
    if (t == 0) {
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(mbar)));
        asm volatile("fence.mbarrier_init.release.cluster;");
    }
    if (w == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 256;" ::"r"(smem_u32(tslot)));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    asm volatile("fence.proxy.async.shared::cta;");      // generic-proxy smem writes -> async proxy
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;");
    const u32 tmem = *tslot;
    if (t == 0) {
        for (int ks = 0; ks < KB / 32; ks++) {
            const u64 da = sdesc(smem_u32(sA) + ks * 2 * LBO, LBO, SBO_A);
            const u64 db = sdesc(smem_u32(sB) + ks * 2 * LBO, LBO, SBO_A);
            const u32 acc = ks > 0;
            asm volatile(
                "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                "tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem),
                "l"(da), "l"(db), "r"(idesc), "r"(acc));
        }
        asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(mbar))
                     : "memory");
    }
    // wait for the MMA chain (phase 0)
    asm volatile(
        "{\n\t.reg .pred P1;\n\tWAIT:\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], 0;\n\t"
        "@!P1 bra WAIT;\n\t}" ::"r"(smem_u32(mbar)) : "memory");
    asm volatile("tcgen05.fence::after_thread_sync;");
    for (int c0 = 0; c0 < N; c0 += 16) {
        u32 v[16];
        const u32 taddr = tmem + ((u32)(w * 32) << 16) + c0;
        asm volatile("tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
                     : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]),
                       "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15])
                     : "r"(taddr));
        asm volatile("tcgen05.wait::ld.sync.aligned;");
        for (int j = 0; j < 16; j++) gD[t * N + c0 + j] = (int32_t)v[j];
    }
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    if (w == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 256;" ::"r"(tmem));
}

int main() {
    uint8_t *hA = (uint8_t *)malloc(M * KB), *hB = (uint8_t *)malloc(N * KB);
    srand(1);
    for (int i = 0; i < M * KB; i++) hA[i] = rand() & 255;
    for (int i = 0; i < N * KB; i++) hB[i] = rand() & 255;
    uint8_t *dA, *dB;
    int32_t *dD;
    cudaMalloc(&dA, M * KB);
    cudaMalloc(&dB, N * KB);
    cudaMalloc(&dD, M * N * 4);
    cudaMemcpy(dA, hA, M * KB, cudaMemcpyHostToDevice);
    cudaMemcpy(dB, hB, N * KB, cudaMemcpyHostToDevice);
    // instruction descriptor: c_format S32 (2) at [4,6), a/b u8 (0), K-major both, N>>3 at [17,23), M>>4 at [24,29)
    const u32 idesc = (2u << 4) | ((u32)(N >> 3) << 17) | ((u32)(M >> 4) << 24);
    const int smem = M * KB + N * KB + 64;
    cudaFuncSetAttribute(k_test, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    k_test<<<1, 128, smem>>>(dA, dB, dD, idesc);
    cudaError_t e = cudaDeviceSynchronize();
    printf("kernel: %s\n", cudaGetErrorString(e));
    int32_t *hD = (int32_t *)malloc(M * N * 4);
    cudaMemcpy(hD, dD, M * N * 4, cudaMemcpyDeviceToHost);
    long bad = 0;
    for (int m = 0; m < M; m++)
        for (int n = 0; n < N; n++) {
            int64_t s = 0;
            for (int k = 0; k < KB; k++) s += (int64_t)hA[m * KB + k] * hB[n * KB + k];
            if (s != hD[m * N + n]) {
                if (bad < 5) printf("mismatch m=%d n=%d got %d want %lld\n", m, n, hD[m * N + n], (long long)s);
                bad++;
            }
        }
    printf("{\"tc_i8_test\": \"%s\", \"mismatches\": %ld}\n", bad ? "FAIL" : "PASS", bad);
    return bad ? 1 : 0;
}
