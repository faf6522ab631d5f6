// tc2_i8_test.cu — standalone check of the CTA-pair (cta_group::2) tcgen05 kind::i8 building blocks
// used by the k = 65 tensor-core base extension:
//   * a 2-CTA cluster; each CTA holds 128 rows of A (its messages) and HALF of the B rows (N/2);
//   * TMEM allocated with tcgen05.alloc.cta_group::2 by one warp of each CTA;
//   * CTA 1 signals "my A tile is written" by a remote mbarrier arrive (release.cluster) on CTA 0;
//   * the rank-0 leader issues tcgen05.mma.cta_group::2 (M = 256, N = 256) and commits with a
//     multicast arrive on both CTAs' mbarriers; every thread reads its own lane's N columns.
// ITER iterations with fresh A contents exercise the mbarrier phases.  D is checked against the CPU.
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cuda_runtime.h>

typedef uint32_t u32;
typedef uint64_t u64;

constexpr int M = 256, N = 256, KB = 288, ITER = 3;   // KB bytes of K (9 MMA steps of 32)
constexpr int SBO = (KB / 16) * 128;
constexpr int LBO = 128;

__device__ __forceinline__ u32 smem_u32(const void *p) { return (u32)__cvta_generic_to_shared(p); }
__host__ __device__ constexpr int off(int r, int kb) { return (r / 8) * SBO + (kb / 16) * LBO + (r % 8) * 16 + kb % 16; }

__device__ __forceinline__ u64 sdesc(u32 saddr) {
    return (u64)((saddr >> 4) & 0x3FFF) | ((u64)(LBO >> 4) << 16) | ((u64)(SBO >> 4) << 32) | ((u64)1 << 46);
}

__device__ __forceinline__ void wait_parity(u32 mbar, u32 ph, bool cluster_acq) {
    u32 done = 0;
    for (u32 spin = 0; !done; spin++) {
        if (cluster_acq)
            asm volatile("{\n\t.reg .pred P1;\n\tmbarrier.try_wait.parity.acquire.cluster.shared::cta.b64 P1, [%1], %2;\n\t"
                         "selp.u32 %0, 1, 0, P1;\n\t}" : "=r"(done) : "r"(mbar), "r"(ph) : "memory");
        else
            asm volatile("{\n\t.reg .pred P1;\n\tmbarrier.try_wait.parity.shared::cta.b64 P1, [%1], %2;\n\t"
                         "selp.u32 %0, 1, 0, P1;\n\t}" : "=r"(done) : "r"(mbar), "r"(ph) : "memory");
        if (spin > (1u << 24)) __trap();
    }
}

__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(128, 1)
k_test2(const uint8_t *gA /* [ITER][M][KB] */, const uint8_t *gB /* [N][KB] */, int32_t *gD /* [ITER][M][N] */,
        u32 idesc, long long *cycles) {
    extern __shared__ __align__(1024) uint8_t sm[];
    uint8_t *sA = sm;                       // 128 rows
    uint8_t *sB = sm + 128 * KB;            // N/2 rows
    u64 *mbar = (u64 *)(sB + (N / 2) * KB); // [0] ready (rank 0 only, count 2), [1] done (count 1)
    u32 *tslot = (u32 *)(mbar + 2);
    u32 rank;
    asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(rank));
    const int t = threadIdx.x, w = t / 32;
    for (int i = t; i < (N / 2) * KB; i += blockDim.x) sB[off(i / KB, i % KB)] = gB[(size_t)rank * (N / 2) * KB + i];
    if (t == 0) {
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 2;" ::"r"(smem_u32(mbar + 0)));
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(mbar + 1)));
        asm volatile("fence.mbarrier_init.release.cluster;");
    }
    if (w == 0) {
        asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], 256;" ::"r"(smem_u32(tslot)));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;");
    }
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
    asm volatile("tcgen05.fence::after_thread_sync;");
    const u32 tmem = *tslot;
    u32 rmbar;                               // rank 0's ready barrier, in the cluster window
    asm volatile("mapa.shared::cluster.u32 %0, %1, 0;" : "=r"(rmbar) : "r"(smem_u32(mbar + 0)));
    long long t0 = 0, t1 = 0;
    for (int it = 0; it < ITER; it++) {
        const u32 ph = it & 1;
        for (int i = t; i < 128 * KB; i += blockDim.x)
            sA[off(i / KB, i % KB)] = gA[((size_t)it * M + rank * 128) * KB + i];
        if (rank == 1 && it == 1) __nanosleep(20000);      // the peer is late: rank 0 must wait for it
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
        __syncthreads();
        if (t == 0) asm volatile("mbarrier.arrive.release.cluster.shared::cluster.b64 _, [%0];" ::"r"(rmbar) : "memory");
        if (rank == 0 && t == 0) {
            wait_parity(smem_u32(mbar + 0), ph, true);
            asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
            t0 = clock64();
            for (int ks = 0; ks < KB / 32; ks++) {
                const u64 da = sdesc(smem_u32(sA) + ks * 256), db = sdesc(smem_u32(sB) + ks * 256);
                asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                             "tcgen05.mma.cta_group::2.kind::i8 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem),
                             "l"(da), "l"(db), "r"(idesc), "r"((u32)ks) : "memory");
            }
            asm volatile("tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;"
                         ::"r"(smem_u32(mbar + 1)), "h"((unsigned short)3) : "memory");
        }
        wait_parity(smem_u32(mbar + 1), ph, false);
        if (rank == 0 && t == 0) t1 = clock64();
        asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
        for (int c0 = 0; c0 < N; c0 += 16) {
            u32 v[16];
            const u32 taddr = tmem + ((u32)(w * 32) << 16) + c0;
            asm volatile("tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
                         : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]),
                           "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15])
                         : "r"(taddr));
            asm volatile("tcgen05.wait::ld.sync.aligned;");
            for (int j = 0; j < 16; j++) gD[((size_t)it * M + rank * 128 + t) * N + c0 + j] = (int32_t)v[j];
        }
        if (rank == 0 && t == 0) cycles[it] = t1 - t0;
    }
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
    if (w == 0) asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, 256;" ::"r"(tmem));
}

int main() {
    const size_t na = (size_t)ITER * M * KB, nb = (size_t)N * KB, nd = (size_t)ITER * M * N;
    uint8_t *hA = (uint8_t *)malloc(na), *hB = (uint8_t *)malloc(nb);
    srand(7);
    for (size_t i = 0; i < na; i++) hA[i] = rand() & 255;
    for (size_t i = 0; i < nb; i++) hB[i] = rand() & 255;
    uint8_t *dA, *dB;
    int32_t *dD;
    long long *dc;
    cudaMalloc(&dA, na);
    cudaMalloc(&dB, nb);
    cudaMalloc(&dD, nd * 4);
    cudaMalloc(&dc, ITER * 8);
    cudaMemset(dD, 0xFF, nd * 4);
    cudaMemcpy(dA, hA, na, cudaMemcpyHostToDevice);
    cudaMemcpy(dB, hB, nb, cudaMemcpyHostToDevice);
    const u32 idesc = (2u << 4) | ((u32)(N >> 3) << 17) | ((u32)(M >> 4) << 24);
    const int smem = 128 * KB + (N / 2) * KB + 64;
    cudaFuncSetAttribute(k_test2, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    k_test2<<<2, 128, smem>>>(dA, dB, dD, idesc, dc);
    cudaError_t e = cudaDeviceSynchronize();
    printf("kernel: %s\n", cudaGetErrorString(e));
    int32_t *hD = (int32_t *)malloc(nd * 4);
    long long hc[ITER];
    cudaMemcpy(hD, dD, nd * 4, cudaMemcpyDeviceToHost);
    cudaMemcpy(hc, dc, sizeof hc, cudaMemcpyDeviceToHost);
    long bad = 0;
    for (int it = 0; it < ITER; it++)
        for (int m = 0; m < M; m++)
            for (int n = 0; n < N; n++) {
                int64_t s = 0;
                for (int k = 0; k < KB; k++) s += (int64_t)hA[((size_t)it * M + m) * KB + k] * hB[(size_t)n * KB + k];
                const int32_t g = hD[((size_t)it * M + m) * N + n];
                if (s != g) {
                    if (bad < 8) printf("mismatch it=%d m=%d n=%d got %d want %lld\n", it, m, n, g, (long long)s);
                    bad++;
                }
            }
    printf("{\"tc2_i8_test\": \"%s\", \"mismatches\": %ld, \"mma_chain_cycles\": [%lld, %lld, %lld]}\n",
           bad ? "FAIL" : "PASS", bad, hc[0], hc[1], hc[2]);
    return bad ? 1 : 0;
}
