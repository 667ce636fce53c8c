// Integer-pipe microbenchmark for the B200 POPC/LOP3 roofline denominator.
// One CTA of 1024 threads per SM; each thread runs 16 independent chains so
// the measured rate is throughput-bound, not latency-bound. Rates are per SM
// per SM-clock (clock64 deltas), so they do not depend on the clock the GPU
// happens to run at.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

#define CHAINS 16
#define ITERS 4096

__device__ __forceinline__ uint32_t popc_asm(uint32_t x) {
  uint32_t r; asm volatile("popc.b32 %0, %1;" : "=r"(r) : "r"(x)); return r;
}
__device__ __forceinline__ uint32_t lop3_xor3(uint32_t a, uint32_t b, uint32_t c) {
  uint32_t r; asm volatile("lop3.b32 %0, %1, %2, %3, 0x96;" : "=r"(r) : "r"(a), "r"(b), "r"(c)); return r;
}
__device__ __forceinline__ uint32_t and_asm(uint32_t a, uint32_t b) {
  uint32_t r; asm volatile("and.b32 %0, %1, %2;" : "=r"(r) : "r"(a), "r"(b)); return r;
}

// mode 0: popc only (v = popc(v) chains; each popc depends on the previous of
// its chain, CHAINS independent chains per thread)
// mode 1: lop3 only
// mode 2: the search inner step: t = p & z ; acc += popc(t)  (and + popc + add)
// mode 3: dadd only (fp64 add)
__global__ void bench(int mode, uint32_t seed, uint32_t* out, long long* cyc) {
  uint32_t v[CHAINS], acc[CHAINS];
  for (int c = 0; c < CHAINS; ++c) { v[c] = seed * (threadIdx.x + 1) + c * 0x9e3779b9u; acc[c] = 0; }
  double d[CHAINS];
  for (int c = 0; c < CHAINS; ++c) d[c] = 1.0 + 1e-9 * (threadIdx.x + c);
  __syncthreads();
  long long t0 = clock64();
  if (mode == 0) {
    for (int it = 0; it < ITERS; ++it)
#pragma unroll
      for (int c = 0; c < CHAINS; ++c) v[c] = popc_asm(v[c] + it);  // popc + iadd
  } else if (mode == 1) {
    for (int it = 0; it < ITERS; ++it)
#pragma unroll
      for (int c = 0; c < CHAINS; ++c) v[c] = lop3_xor3(v[c], v[(c + 1) % CHAINS], seed);
  } else if (mode == 2) {
    for (int it = 0; it < ITERS; ++it)
#pragma unroll
      for (int c = 0; c < CHAINS; ++c) acc[c] += popc_asm(and_asm(v[c], it ^ seed));
  } else if (mode == 4) {
    // popc only, feeding from an independent value (no add on the chain)
    for (int it = 0; it < ITERS; ++it)
#pragma unroll
      for (int c = 0; c < CHAINS; ++c) acc[c] ^= popc_asm(v[c] ^ it);
  } else {
    for (int it = 0; it < ITERS; ++it)
#pragma unroll
      for (int c = 0; c < CHAINS; ++c) d[c] = d[c] + d[(c + 3) % CHAINS];
  }
  __syncthreads();
  long long t1 = clock64();
  uint32_t s = 0;
  for (int c = 0; c < CHAINS; ++c) s += v[c] + acc[c] + (uint32_t)(d[c] > 3.0);
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}

int main() {
  int dev = 0; cudaDeviceProp p; cudaGetDeviceProperties(&p, dev);
  int nsm = p.multiProcessorCount;
  printf("device %s SMs %d\n", p.name, nsm);
  uint32_t* out; long long* cyc;
  cudaMalloc(&out, sizeof(uint32_t) * nsm * 1024);
  cudaMalloc(&cyc, sizeof(long long) * nsm);
  long long* h = new long long[nsm];
  const char* names[] = {"popc(+iadd)", "lop3", "and+popc+iadd", "dadd", "popc(+lop)"};
  for (int mode : {0, 1, 2, 3, 4}) {
    for (int threads : {256, 512, 1024}) {
      cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
      bench<<<nsm, threads>>>(mode, 12345, out, cyc);
      cudaEventRecord(e0);
      bench<<<nsm, threads>>>(mode, 12345, out, cyc);
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
      float ms; cudaEventElapsedTime(&ms, e0, e1);
      cudaMemcpy(h, cyc, sizeof(long long) * nsm, cudaMemcpyDeviceToHost);
      double mean = 0; for (int i = 0; i < nsm; ++i) mean += h[i]; mean /= nsm;
      double ops = double(threads) * ITERS * CHAINS;  // per SM
      printf("mode %-16s threads %4d: %.2f ops/clk/SM (cycles %.0f, %.3f ms, implied SM clock %.0f MHz)\n",
             names[mode], threads, ops / mean, mean, ms, mean / (ms * 1e3));
    }
  }
  cudaError_t err = cudaGetLastError();
  printf("err: %s\n", cudaGetErrorString(err));
  return 0;
}
