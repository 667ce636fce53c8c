// umma_probe.cu — feasibility probe for the tensor-core contingency path:
// tcgen05.mma.cta_group::1.kind::i8 with K-major, no-swizzle smem operands
// (8x16B core matrices), D in TMEM read back with tcgen05.ld.32x32b.
// Checks D == A*B^T exactly (0/1 bytes, s32 accumulate) and times the
// MMA issue loop (M=128, N=256, K=32 per instruction).
#include <cstdio>
#include <cstdint>
#include <cstdlib>
#include <vector>
#include <cuda_runtime.h>

constexpr int M = 128, N = 256, KC = 128;  // K bytes per smem chunk
constexpr int NCHUNK = 4;                  // K total = 512
constexpr int THREADS = 128;

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

// K-major INTERLEAVE layout for a (rows x 128 B) chunk: core matrix (8 rows x 16 B)
// at ((r/8)*8 + k/16) * 128 B; row r%8 at +16 B.
__device__ __forceinline__ uint32_t off_of(int r, int kslab) {
  return ((r >> 3) * 8 + kslab) * 128 + (r & 7) * 16;
}

__device__ __forceinline__ uint64_t make_desc(uint32_t saddr, uint32_t lbo, uint32_t sbo) {
  uint64_t d = 0;
  d |= uint64_t((saddr >> 4) & 0x3fff);
  d |= uint64_t((lbo >> 4) & 0x3fff) << 16;
  d |= uint64_t((sbo >> 4) & 0x3fff) << 32;
  d |= uint64_t(1) << 46;  // version = 1 (sm100)
  // base_offset 0, lbo_mode 0, layout_type 0 (SWIZZLE_NONE)
  return d;
}

__global__ void __launch_bounds__(THREADS, 1)
probe(const uint8_t* A, const uint8_t* B, int32_t* D, int iters, long long* cycles) {
  extern __shared__ __align__(1024) uint8_t smem[];
  uint8_t* sA = smem;                          // NCHUNK * M * KC
  uint8_t* sB = smem + NCHUNK * M * KC;        // NCHUNK * N * KC
  __shared__ uint64_t mbar;
  __shared__ uint32_t tmem_base;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;

  // stage operands: A[r][k] global row-major (K total = NCHUNK*KC)
  for (int idx = threadIdx.x; idx < NCHUNK * M * (KC / 16); idx += THREADS) {
    const int c = idx / (M * (KC / 16)), rem = idx % (M * (KC / 16));
    const int r = rem / (KC / 16), ks = rem % (KC / 16);
    const uint4 v = *reinterpret_cast<const uint4*>(A + size_t(r) * NCHUNK * KC + c * KC + ks * 16);
    *reinterpret_cast<uint4*>(sA + c * M * KC + off_of(r, ks)) = v;
  }
  for (int idx = threadIdx.x; idx < NCHUNK * N * (KC / 16); idx += THREADS) {
    const int c = idx / (N * (KC / 16)), rem = idx % (N * (KC / 16));
    const int r = rem / (KC / 16), ks = rem % (KC / 16);
    const uint4 v = *reinterpret_cast<const uint4*>(B + size_t(r) * NCHUNK * KC + c * KC + ks * 16);
    *reinterpret_cast<uint4*>(sB + c * N * KC + off_of(r, ks)) = v;
  }
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&mbar)));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 256;" ::"r"(smem_u32(&tmem_base)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t tmem = tmem_base;

  // instruction descriptor: D s32, A/B u8, K-major, N=256, M=128
  const uint32_t idesc = (2u << 4) | (uint32_t(N >> 3) << 17) | (uint32_t(M >> 4) << 24);
  long long t0 = 0, t1 = 0;
  if (threadIdx.x == 0) {
    t0 = clock64();
    uint32_t phase = 0;
    for (int it = 0; it < iters; ++it) {
      for (int c = 0; c < NCHUNK; ++c)
        for (int kk = 0; kk < KC / 32; ++kk) {
          const uint64_t ad = make_desc(smem_u32(sA + c * M * KC + kk * 2 * 128), 128, 1024);
          const uint64_t bd = make_desc(smem_u32(sB + c * N * KC + kk * 2 * 128), 128, 1024);
          const uint32_t acc = (c | kk) ? 1u : 0u;
          asm volatile(
              "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
              "tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n\t}\n"
              ::"r"(tmem), "l"(ad), "l"(bd), "r"(idesc), "r"(acc));
        }
      asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];"
                   ::"r"(smem_u32(&mbar)));
      // wait for completion of this pass
      asm volatile(
          "{\n\t.reg .pred P1;\n\tWAIT_%=:\n\t"
          "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n\t"
          "@!P1 bra WAIT_%=;\n\t}\n" ::"r"(smem_u32(&mbar)), "r"(phase));
      phase ^= 1;
    }
    t1 = clock64();
    *cycles = t1 - t0;
  }
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  // epilogue: warp w reads TMEM lanes 32w..32w+31, 8 columns at a time
  for (int c0 = 0; c0 < N; c0 += 8) {
    uint32_t v[8];
    const uint32_t addr = tmem + (uint32_t(warp * 32) << 16) + c0;
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                 : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]),
                   "=r"(v[6]), "=r"(v[7])
                 : "r"(addr));
    asm volatile("tcgen05.wait::ld.sync.aligned;");
    for (int x = 0; x < 8; ++x) D[(warp * 32 + lane) * N + c0 + x] = int32_t(v[x]);
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 256;" ::"r"(tmem));
}

int main() {
  const int K = NCHUNK * KC;
  std::vector<uint8_t> hA(M * K), hB(N * K);
  uint32_t s = 12345;
  auto rnd = [&]() { s = s * 1664525u + 1013904223u; return (s >> 16) & 1u; };
  for (auto& x : hA) x = uint8_t(rnd());
  for (auto& x : hB) x = uint8_t(rnd());
  uint8_t *dA, *dB; int32_t* dD; long long* dc;
  cudaMalloc(&dA, hA.size()); cudaMalloc(&dB, hB.size());
  cudaMalloc(&dD, sizeof(int32_t) * M * N); cudaMalloc(&dc, sizeof(long long));
  cudaMemcpy(dA, hA.data(), hA.size(), cudaMemcpyHostToDevice);
  cudaMemcpy(dB, hB.data(), hB.size(), cudaMemcpyHostToDevice);
  const size_t smem = size_t(NCHUNK) * (M + N) * KC;
  cudaFuncSetAttribute(probe, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem));
  for (int iters : {1, 2000}) {
    cudaMemset(dD, 0xff, sizeof(int32_t) * M * N);
    probe<<<1, THREADS, smem>>>(dA, dB, dD, iters, dc);
    cudaError_t e = cudaDeviceSynchronize();
    if (e != cudaSuccess) { printf("CUDA error: %s\n", cudaGetErrorString(e)); return 1; }
    std::vector<int32_t> hD(M * N);
    long long cyc = 0;
    cudaMemcpy(hD.data(), dD, sizeof(int32_t) * M * N, cudaMemcpyDeviceToHost);
    cudaMemcpy(&cyc, dc, sizeof(long long), cudaMemcpyDeviceToHost);
    long bad = 0;
    for (int r = 0; r < M; ++r)
      for (int c = 0; c < N; ++c) {
        int32_t ref = 0;
        for (int k = 0; k < K; ++k) ref += hA[r * K + k] * hB[c * K + k];
        if (ref != hD[r * N + c]) { if (bad < 5) printf("mismatch r=%d c=%d got %d want %d\n", r, c, hD[r * N + c], ref); ++bad; }
      }
    const double mmas = double(iters) * NCHUNK * (KC / 32);
    printf("iters %d: mismatches %ld; %.1f cycles per MMA (M128 N256 K32 = %.0f MAC/clk)\n", iters, bad,
           cyc / mmas, double(M) * N * 32 / (cyc / mmas));
  }
  return 0;
}
