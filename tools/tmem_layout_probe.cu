// tmem_layout_probe.cu — which (TMEM lane, column) each thread of a warp
// receives from tcgen05.ld.16x256b (and .16x64b): every cell of lanes 0-31,
// columns 0-15 is written with lane * 256 + column through the 32x32b shape
// (thread t = lane t), then read back with the other shapes; prints the map.
// nvcc -gencode arch=compute_100a,code=sm_100a -o tools/tmem_layout_probe tools/tmem_layout_probe.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__global__ void probe(uint32_t* out) {
  __shared__ uint32_t tbase;
  const int lane = threadIdx.x & 31;
  asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 32;" ::"r"(
      uint32_t(__cvta_generic_to_shared(&tbase))));
  asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncwarp();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t t = tbase;
  uint32_t v[16];
  for (int c = 0; c < 16; ++c) v[c] = uint32_t(lane) * 256u + uint32_t(c);
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16};"
      ::"r"(t), "r"(v[0]), "r"(v[1]), "r"(v[2]), "r"(v[3]), "r"(v[4]), "r"(v[5]), "r"(v[6]), "r"(v[7]),
      "r"(v[8]), "r"(v[9]), "r"(v[10]), "r"(v[11]), "r"(v[12]), "r"(v[13]), "r"(v[14]), "r"(v[15]));
  asm volatile("tcgen05.wait::st.sync.aligned;");
  uint32_t a[4], b[8];
  // lanes 0-15 and 16-31 (lane base in address bits 16+)
  asm volatile("tcgen05.ld.sync.aligned.16x256b.x1.b32 {%0,%1,%2,%3}, [%4];"
               : "=r"(a[0]), "=r"(a[1]), "=r"(a[2]), "=r"(a[3]) : "r"(t));
  asm volatile("tcgen05.ld.sync.aligned.16x256b.x2.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
               : "=r"(b[0]), "=r"(b[1]), "=r"(b[2]), "=r"(b[3]), "=r"(b[4]), "=r"(b[5]), "=r"(b[6]),
                 "=r"(b[7])
               : "r"(t + (16u << 16)));
  asm volatile("tcgen05.wait::ld.sync.aligned;");
  for (int k = 0; k < 4; ++k) out[lane * 12 + k] = a[k];
  for (int k = 0; k < 8; ++k) out[lane * 12 + 4 + k] = b[k];
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncwarp();
  asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 32;" ::"r"(t));
}

int main() {
  uint32_t* d;
  cudaMalloc(&d, 32 * 12 * 4);
  probe<<<1, 32>>>(d);
  cudaError_t e = cudaDeviceSynchronize();
  if (e != cudaSuccess) { printf("error %s\n", cudaGetErrorString(e)); return 1; }
  uint32_t h[32 * 12];
  cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
  printf("thread: 16x256b.x1 @lane0 (lane.col) | 16x256b.x2 @lane16\n");
  for (int t = 0; t < 32; ++t) {
    printf("%2d:", t);
    for (int k = 0; k < 12; ++k) printf(" %2u.%-2u", h[t * 12 + k] / 256, h[t * 12 + k] % 256);
    printf("\n");
  }
  return 0;
}
