// tc_i8_peak.cu — measured peak of the int8 tensor cores on sm_100a (tcgen05.mma.kind::i8, u8 x u8 -> s32),
// the denominator of roofline.tensor_i8 in bench.py (VERDICT r1 "do this" #4).
//
// One persistent CTA per SM (grid = SM count; 2-CTA clusters for cta_group::2).  Operands are random bytes
// staged once in shared memory (K-major SWIZZLE_NONE core-matrix layout, the layout the base-extension
// kernels use); the elected thread 0 (rank 0 of the pair) issues ITERS x KSTEPS back-to-back MMAs into one
// TMEM accumulator and commits once at the end, so the tensor pipe never waits on anything but itself.
// Shapes:
//   g1 M=128 N=256   cta_group::1  (the largest single-CTA MMA)
//   g1 M=128 N=128   cta_group::1  (k = 33 base-extension shape: 128 messages x 32 outputs x 4 byte columns)
//   g1 M=128 N=144   cta_group::1  (k = 33 with all 33 outputs on the tensor core)
//   g2 M=256 N=256   cta_group::2  (k = 65 CTA-pair shape)
// Ops counted: 2 * M * N * 32 per MMA instruction (K = 32 bytes).  Time: cudaEvents around the launch,
// best of REPS; also the median per-CTA clock64 span of the issue loop.  Output: one JSON object per shape.
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cuda_runtime.h>
#include <vector>
#include <algorithm>

typedef uint32_t u32;
typedef uint64_t u64;

constexpr int KB = 128;                      // K bytes staged (4 MMA k-steps of 32)
constexpr int KSTEPS = KB / 32;
constexpr int SBO = (KB / 16) * 128;
constexpr int LBO = 128;

__device__ __forceinline__ u32 smem_u32(const void *p) { return (u32)__cvta_generic_to_shared(p); }
__host__ __device__ constexpr int off(int r, int kb) { return (r / 8) * SBO + (kb / 16) * LBO + (r % 8) * 16 + kb % 16; }
__device__ __forceinline__ u64 sdesc(u32 saddr) {
    return (u64)((saddr >> 4) & 0x3FFF) | ((u64)(LBO >> 4) << 16) | ((u64)(SBO >> 4) << 32) | ((u64)1 << 46);
}
__device__ __forceinline__ void wait_parity(u32 mbar, u32 ph) {
    u32 done = 0;
    while (!done)
        asm volatile("{\n\t.reg .pred P1;\n\tmbarrier.try_wait.parity.acquire.cluster.shared::cta.b64 P1, [%1], %2;\n\t"
                     "selp.u32 %0, 1, 0, P1;\n\t}" : "=r"(done) : "r"(mbar), "r"(ph) : "memory");
}

// G = 1 or 2 (cta_group); NB = B rows held by this CTA (N for G=1, N/2 for G=2)
template <int G>
__global__ void __launch_bounds__(128, 1) k_peak(const uint8_t *gA, const uint8_t *gB, int NB, u32 idesc, int iters,
                                                 long long *cyc, u32 *sink) {
    extern __shared__ __align__(1024) uint8_t sm[];
    uint8_t *sA = sm;
    uint8_t *sB = sm + 128 * KB;
    u64 *mbar = (u64 *)(sB + 256 * KB);
    u32 *tslot = (u32 *)(mbar + 2);
    u32 rank = 0;
    if (G == 2) asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(rank));
    const int t = threadIdx.x, w = t / 32;
    for (int i = t; i < 128 * KB; i += blockDim.x) sA[off(i / KB, i % KB)] = gA[i];
    for (int i = t; i < NB * KB; i += blockDim.x) sB[off(i / KB, i % KB)] = gB[i];
    if (t == 0) {
        asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(mbar + 0)), "r"(G));
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(mbar + 1)));
        asm volatile("fence.mbarrier_init.release.cluster;");
    }
    if (w == 0) {
        if (G == 1) {
            asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 256;" ::"r"(smem_u32(tslot)));
            asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
        } else {
            asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], 256;" ::"r"(smem_u32(tslot)));
            asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;");
        }
    }
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    if (G == 2) asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    const u32 tmem = *tslot;
    long long t0 = clock64();
    if (rank == 0 && t == 0) {
        const u32 a0 = smem_u32(sA), b0 = smem_u32(sB);
        for (int it = 0; it < iters; it++) {
#pragma unroll
            for (int ks = 0; ks < KSTEPS; ks++) {
                const u64 da = sdesc(a0 + ks * 256), db = sdesc(b0 + ks * 256);
                const u32 acc = (it | ks) != 0;
                if (G == 1)
                    asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                                 "tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem),
                                 "l"(da), "l"(db), "r"(idesc), "r"(acc) : "memory");
                else
                    asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                                 "tcgen05.mma.cta_group::2.kind::i8 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem),
                                 "l"(da), "l"(db), "r"(idesc), "r"(acc) : "memory");
            }
        }
        if (G == 1)
            asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];"
                         ::"r"(smem_u32(mbar + 1)) : "memory");
        else
            asm volatile("tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;"
                         ::"r"(smem_u32(mbar + 1)), "h"((unsigned short)3) : "memory");
    }
    wait_parity(smem_u32(mbar + 1), 0);
    long long t1 = clock64();
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    u32 v;
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x1.b32 {%0}, [%1];" : "=r"(v) : "r"(tmem + ((u32)(w * 32) << 16)));
    asm volatile("tcgen05.wait::ld.sync.aligned;");
    atomicXor(sink, v);
    if (t == 0) cyc[blockIdx.x] = t1 - t0;
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    if (G == 2) asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
    if (w == 0) {
        if (G == 1) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 256;" ::"r"(tmem));
        else asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, 256;" ::"r"(tmem));
    }
}

static void run(int G, int M, int N, int iters, int reps, const cudaDeviceProp &p) {
    const int sms = p.multiProcessorCount;
    const int grid = G == 2 ? sms / 2 * 2 : sms;
    const int NB = G == 2 ? N / 2 : N;
    std::vector<uint8_t> hA(128 * KB), hB(256 * KB);
    srand(11);
    for (auto &x : hA) x = rand() & 255;
    for (auto &x : hB) x = rand() & 255;
    uint8_t *dA, *dB;
    long long *dc;
    u32 *sink;
    cudaMalloc(&dA, hA.size());
    cudaMalloc(&dB, hB.size());
    cudaMalloc(&dc, grid * sizeof(long long));
    cudaMalloc(&sink, 4);
    cudaMemcpy(dA, hA.data(), hA.size(), cudaMemcpyHostToDevice);
    cudaMemcpy(dB, hB.data(), hB.size(), cudaMemcpyHostToDevice);
    const u32 idesc = (2u << 4) | ((u32)(N >> 3) << 17) | ((u32)(M >> 4) << 24);
    const int smem = 128 * KB + 256 * KB + 64;
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    float best = 1e30f;
    std::vector<long long> cyc(grid);
    for (int r = 0; r < reps + 1; r++) {
        cudaEventRecord(e0);
        if (G == 1) {
            cudaFuncSetAttribute(k_peak<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
            k_peak<1><<<grid, 128, smem>>>(dA, dB, NB, idesc, iters, dc, sink);
        } else {
            cudaFuncSetAttribute(k_peak<2>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
            cudaLaunchConfig_t cfg = {};
            cudaLaunchAttribute at[1];
            at[0].id = cudaLaunchAttributeClusterDimension;
            at[0].val.clusterDim.x = 2;
            at[0].val.clusterDim.y = 1;
            at[0].val.clusterDim.z = 1;
            cfg.gridDim = dim3(grid);
            cfg.blockDim = dim3(128);
            cfg.dynamicSmemBytes = smem;
            cfg.attrs = at;
            cfg.numAttrs = 1;
            cudaLaunchKernelEx(&cfg, k_peak<2>, (const uint8_t *)dA, (const uint8_t *)dB, NB, idesc, iters, dc, sink);
        }
        cudaEventRecord(e1);
        cudaError_t err = cudaEventSynchronize(e1);
        if (err != cudaSuccess || cudaGetLastError() != cudaSuccess) {
            printf("{\"error\": \"%s\"}\n", cudaGetErrorString(err));
            exit(1);
        }
        float ms;
        cudaEventElapsedTime(&ms, e0, e1);
        if (r > 0) best = std::min(best, ms);
    }
    cudaMemcpy(cyc.data(), dc, grid * sizeof(long long), cudaMemcpyDeviceToHost);
    std::sort(cyc.begin(), cyc.end());
    const double mmas = (double)(G == 2 ? grid / 2 : grid) * iters * KSTEPS;
    const double ops = mmas * 2.0 * M * N * 32;
    const double per_clk_sm = 2.0 * M * N * 32 * iters * KSTEPS / (double)cyc[grid / 2] / G;
    printf("{\"shape\": \"cta_group::%d M=%d N=%d K=32 kind::i8\", \"sms\": %d, \"grid\": %d, \"mmas\": %.0f, "
           "\"ms_best\": %.4f, \"tops\": %.1f, \"ops_per_clk_per_sm\": %.1f, \"cyc_median\": %lld, \"cyc_max\": %lld}\n",
           G, M, N, sms, grid, mmas, best, ops / best / 1e9, per_clk_sm, cyc[grid / 2], cyc[grid - 1]);
    cudaFree(dA);
    cudaFree(dB);
    cudaFree(dc);
    cudaFree(sink);
}

int main(int argc, char **argv) {
    const int iters = argc > 1 ? atoi(argv[1]) : 8192;
    cudaDeviceProp p;
    cudaGetDeviceProperties(&p, 0);
    printf("{\"device\": \"%s\", \"sms\": %d, \"cc\": \"%d.%d\", \"iters\": %d, \"ksteps\": %d}\n", p.name,
           p.multiProcessorCount, p.major, p.minor, iters, KSTEPS);
    run(1, 128, 256, iters, 5, p);
    run(1, 128, 128, iters, 5, p);
    run(1, 128, 144, iters, 5, p);
    run(2, 256, 256, iters, 5, p);
    return 0;
}
