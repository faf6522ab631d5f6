// N9 — integer-multiply pipe peak microbenchmark for sm_100a (SURVEY.md §7 step 0, §8(d) "Denominator").
// Measures warp-instruction throughput of independent streams of:
//   imad      : 32-bit  mad.lo.u32          (IMAD)
//   imad_wide : 32x32+64 mad.wide.u32        (IMAD.WIDE.U32)
//   mac96     : mad.lo.cc / madc.hi.cc / addc (the 96-bit MAC of the base extension)
//   imad_hi   : mul.hi.u32                   (IMAD.HI.U32)
//   dfma      : fp64 fma                      (DFMA)
//   imad_c    : IMAD.WIDE with a __constant__ operand (constant-bank operand)
// Output: thread-ops per clock per SM, using the SM clock measured with clock64 over the same region.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

#define U 8
#define ITERS 4096

__constant__ uint32_t cst[64];

__global__ void k_imad(uint32_t *out, uint32_t y, uint32_t z, unsigned long long *cyc) {
  uint32_t x[U];
  #pragma unroll
  for (int j = 0; j < U; j++) x[j] = threadIdx.x + j;
  unsigned long long t0 = clock64();
  for (int it = 0; it < ITERS; it++) {
    #pragma unroll
    for (int j = 0; j < U; j++) x[j] = x[j] * y + z;
  }
  unsigned long long t1 = clock64();
  uint32_t s = 0;
  #pragma unroll
  for (int j = 0; j < U; j++) s ^= x[j];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}

__global__ void k_imad_wide(uint32_t *out, uint32_t y, uint32_t z, unsigned long long *cyc) {
  uint64_t a[U]; uint32_t x[U];
  #pragma unroll
  for (int j = 0; j < U; j++) { a[j] = threadIdx.x + j; x[j] = threadIdx.x * 7 + j; }
  unsigned long long t0 = clock64();
  for (int it = 0; it < ITERS; it++) {
    #pragma unroll
    for (int j = 0; j < U; j++) a[j] = (uint64_t)x[j] * y + a[j];
    #pragma unroll
    for (int j = 0; j < U; j++) x[j] ^= (uint32_t)(a[j] >> 32);
  }
  unsigned long long t1 = clock64();
  uint32_t s = 0;
  #pragma unroll
  for (int j = 0; j < U; j++) s ^= (uint32_t)a[j] ^ x[j];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}

// pure IMAD.WIDE accumulate chains, multiplier fixed per chain (no xor feedback)
__global__ void k_imad_wide2(uint32_t *out, uint32_t y, uint32_t z, unsigned long long *cyc) {
  uint64_t a[U]; uint32_t x[U];
  #pragma unroll
  for (int j = 0; j < U; j++) { a[j] = threadIdx.x + j; x[j] = threadIdx.x * 7 + j + z; }
  unsigned long long t0 = clock64();
  for (int it = 0; it < ITERS; it++) {
    #pragma unroll
    for (int j = 0; j < U; j++) a[j] = (uint64_t)x[j] * (y + it) + a[j];
  }
  unsigned long long t1 = clock64();
  uint32_t s = 0;
  #pragma unroll
  for (int j = 0; j < U; j++) s ^= (uint32_t)a[j] ^ (uint32_t)(a[j] >> 32);
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}

__device__ __forceinline__ void mac96(uint32_t &lo, uint32_t &mid, uint32_t &hi, uint32_t x, uint32_t c) {
  asm("mad.lo.cc.u32 %0, %3, %4, %0;\n\t"
      "madc.hi.cc.u32 %1, %3, %4, %1;\n\t"
      "addc.u32 %2, %2, 0;" : "+r"(lo), "+r"(mid), "+r"(hi) : "r"(x), "r"(c));
}

__global__ void k_mac96(uint32_t *out, uint32_t y, uint32_t z, unsigned long long *cyc) {
  uint32_t lo[U], mid[U], hi[U], x[U];
  #pragma unroll
  for (int j = 0; j < U; j++) { lo[j] = threadIdx.x + j; mid[j] = 0; hi[j] = 0; x[j] = threadIdx.x * 13 + j + z; }
  unsigned long long t0 = clock64();
  for (int it = 0; it < ITERS; it++) {
    uint32_t c = y + it;
    #pragma unroll
    for (int j = 0; j < U; j++) mac96(lo[j], mid[j], hi[j], x[j], c);
  }
  unsigned long long t1 = clock64();
  uint32_t s = 0;
  #pragma unroll
  for (int j = 0; j < U; j++) s ^= lo[j] ^ mid[j] ^ hi[j];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}

// 96-bit MAC with constant-bank operand, like the base-extension inner loop
__global__ void k_mac96_c(uint32_t *out, uint32_t y, uint32_t z, unsigned long long *cyc) {
  uint32_t lo[U], mid[U], hi[U], x[U];
  #pragma unroll
  for (int j = 0; j < U; j++) { lo[j] = threadIdx.x + j; mid[j] = 0; hi[j] = 0; x[j] = threadIdx.x * 13 + j + z; }
  unsigned long long t0 = clock64();
  for (int it = 0; it < ITERS / 8; it++) {
    #pragma unroll
    for (int i = 0; i < 8; i++) {
      #pragma unroll
      for (int j = 0; j < U; j++) mac96(lo[j], mid[j], hi[j], x[i], cst[i * U + j]);
    }
    #pragma unroll
    for (int j = 0; j < U; j++) x[j] += lo[j];
  }
  unsigned long long t1 = clock64();
  uint32_t s = 0;
  #pragma unroll
  for (int j = 0; j < U; j++) s ^= lo[j] ^ mid[j] ^ hi[j];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}

__global__ void k_imad_hi(uint32_t *out, uint32_t y, uint32_t z, unsigned long long *cyc) {
  uint32_t x[U];
  #pragma unroll
  for (int j = 0; j < U; j++) x[j] = threadIdx.x + j + z;
  unsigned long long t0 = clock64();
  for (int it = 0; it < ITERS; it++) {
    #pragma unroll
    for (int j = 0; j < U; j++) x[j] = __umulhi(x[j], y) + x[j];
  }
  unsigned long long t1 = clock64();
  uint32_t s = 0;
  #pragma unroll
  for (int j = 0; j < U; j++) s ^= x[j];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}

__global__ void k_dfma(uint32_t *out, uint32_t y, uint32_t z, unsigned long long *cyc) {
  double x[U]; double yy = 1.0000001 + y * 1e-12, zz = 1e-9 * z;
  #pragma unroll
  for (int j = 0; j < U; j++) x[j] = threadIdx.x + j;
  unsigned long long t0 = clock64();
  for (int it = 0; it < ITERS; it++) {
    #pragma unroll
    for (int j = 0; j < U; j++) x[j] = fma(x[j], yy, zz);
  }
  unsigned long long t1 = clock64();
  double s = 0;
  #pragma unroll
  for (int j = 0; j < U; j++) s += x[j];
  out[blockIdx.x * blockDim.x + threadIdx.x] = (uint32_t)s;
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}

typedef void (*kfn)(uint32_t *, uint32_t, uint32_t, unsigned long long *);

static void run(const char *name, kfn f, double ops_per_iter_per_thread, int sms, int bpsm, int threads) {
  int blocks = sms * bpsm;
  uint32_t *out; unsigned long long *cyc;
  cudaMalloc(&out, (size_t)blocks * threads * 4);
  cudaMalloc(&cyc, blocks * 8);
  f<<<blocks, threads>>>(out, 3, 5, cyc);  // warm-up
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  cudaEventRecord(e0);
  f<<<blocks, threads>>>(out, 3, 5, cyc);
  cudaEventRecord(e1); cudaEventSynchronize(e1);
  float ms; cudaEventElapsedTime(&ms, e0, e1);
  unsigned long long *h = new unsigned long long[blocks];
  cudaMemcpy(h, cyc, blocks * 8, cudaMemcpyDeviceToHost);
  unsigned long long mx = 0; double avg = 0;
  for (int i = 0; i < blocks; i++) { if (h[i] > mx) mx = h[i]; avg += h[i]; }
  avg /= blocks;
  double ops = (double)blocks * threads * ITERS * ops_per_iter_per_thread;
  // every block resident at once (bpsm*threads <= 2048): ops per SM per clock over the block's own window
  double per_sm_clk = ops / sms / (double)mx;
  double f_mhz = mx / (ms * 1e3);
  printf("{\"op\": \"%s\", \"threads_per_sm\": %d, \"ops_per_clk_per_sm\": %.2f, \"ops_per_s\": %.4e, \"sm_mhz_est\": %.0f, \"ms\": %.3f, \"cyc_max\": %llu, \"cyc_avg\": %.0f}\n",
         name, bpsm * threads, per_sm_clk, ops / (ms * 1e-3), f_mhz, ms, mx, avg);
  cudaError_t err = cudaGetLastError();
  if (err != cudaSuccess) printf("error %s\n", cudaGetErrorString(err));
  delete[] h; cudaFree(out); cudaFree(cyc);
}

int main() {
  cudaDeviceProp p; cudaGetDeviceProperties(&p, 0);
  printf("{\"device\": \"%s\", \"sms\": %d, \"cc\": \"%d.%d\", \"clock_khz\": %d}\n", p.name, p.multiProcessorCount, p.major, p.minor, p.clockRate);
  uint32_t hc[64]; for (int i = 0; i < 64; i++) hc[i] = 0x9E3779B9u * (i + 1);
  cudaMemcpyToSymbol(cst, hc, sizeof(hc));
  int sms = p.multiProcessorCount;
  for (int bpsm : {2, 4, 8}) {
    run("imad", k_imad, U, sms, bpsm, 256);
    run("imad_wide_xor", k_imad_wide, U, sms, bpsm, 256);
    run("imad_wide", k_imad_wide2, U, sms, bpsm, 256);
    run("mac96", k_mac96, U, sms, bpsm, 256);
    run("mac96_const", k_mac96_c, U, sms, bpsm, 256);
    run("imad_hi", k_imad_hi, U, sms, bpsm, 256);
    run("dfma", k_dfma, U, sms, bpsm, 256);
  }
  return 0;
}
