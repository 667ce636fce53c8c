// pairs_tc.cuh — the marginal pair index as a tensor-core Gram matrix
// (included by engine.cu after search_syrk.cuh; reuses its fp4 helpers).
//
// pair[c][x*M + y] = {popc(X0^x & X0^y), popc(X0^x & X1^y), popc(X1^x & X0^y),
// popc(X1^x & X1^y)} over class c, for x < y, mirrored at [y*M + x]. With the
// plane rows (snp, g) as operand rows this is G_c = X_c X_c^T: per tile of
// 64 x-SNPs by 64 y-SNPs (x-block <= y-block) and class, one 128 x 128 f32
// accumulator over the class's samples, issued as tcgen05.mma kind::mxf4 on
// E2M1 0/1 nibbles (exact: counts < 2^23). Replaces the POPC pairs_kernel
// (15.6 ms at 8192 x 16384) in dataset creation.
//
// Warp roles: warp 0 issues the MMAs (per tile: class 0 then class 1 into a
// 3-slot TMEM ring), warps 1-4 expand plane quads into the fp4 stages (thread
// r owns A row r and B row r), warps 5-8 drain both classes of a tile
// together and write the index (class-packed in narrow mode).

namespace pairs_tc {

using namespace tc;
using syrk::kSChunk;
using syrk::kSRowBytes;
using syrk::kSfCol;

// A + B operand stages in shared memory (A-from-TMEM, as in the SYRK kernel,
// measured 9% slower here: 3 stages instead of 4 plus the tcgen05.st issue)
constexpr int kStagesP = 4;
constexpr int kSStageBytes = 2 * kRows * kSRowBytes;  // 32 KiB
constexpr int kProd = 4, kDrain = 4;
constexpr int kThreadsP = 32 * (1 + kProd + kDrain);
constexpr int kBlk = 64;  // SNPs per block -> 128 operand rows

struct PArgs {
  uint32_t M, nb;           // SNPs, 64-SNP blocks
  uint32_t wq[2];           // word-quads per class
  const uint4* planes[2];   // [wq + 1][M][2]
  uint4* pair[2];           // [M * M] wide (u32) counts
  uint4* pairp;             // [M * M] narrow class-packed mirror (c0 | c1 << 16), every N_c < 2^16
  uint64_t tiles;           // nb (nb + 1) / 2 tiles; each = two units (class 0, class 1)
  uint32_t shift;           // narrow: packed counts scaled by 1 << shift
};

// tile -> (x-block, y-block), row-major triangle xb <= yb
struct PWalker {
  uint32_t xb, yb, nb;
  __device__ void start(const PArgs& p, uint64_t t) {
    nb = p.nb;
    xb = 0;
    while (t >= uint64_t(nb - xb)) { t -= nb - xb; ++xb; }
    yb = xb + uint32_t(t);
  }
  __device__ void next() {
    if (++yb == nb) {
      ++xb;
      yb = xb;
    }
  }
};

constexpr int kRing = 3;  // TMEM accumulators (128 columns each) + scale factors at kSfCol

// kNarrow: only the SYRK engine's class-packed mirrored index is written (the
// wide index of a narrow dataset is built by a later <false> launch on first
// use); else the wide per-class index, upper triangle + mirror.
template <bool kNarrow>
__global__ void __launch_bounds__(kThreadsP, 1) pairs_tc_kernel(const PArgs p) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* stages = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                               ~uintptr_t(1023));
  __shared__ uint64_t full_bar[kStagesP], empty_bar[kStagesP];
  __shared__ uint64_t tfull_bar[kRing], tempty_bar[kRing];
  __shared__ uint32_t tmem_base_sh;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint64_t t0 = p.tiles * blockIdx.x / gridDim.x;
  const uint64_t t1 = p.tiles * (blockIdx.x + 1) / gridDim.x;

  if (threadIdx.x == 0) {
    for (int st = 0; st < kStagesP; ++st) {
      mbar_init(&full_bar[st], kProd);
      mbar_init(&empty_bar[st], 1);
    }
    for (int b = 0; b < kRing; ++b) {
      mbar_init(&tfull_bar[b], 1);
      mbar_init(&tempty_bar[b], 32 * kDrain);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                     smem_u32(&tmem_base_sh)), "n"(kTmemCols));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  fence_before();
  __syncthreads();
  fence_after();
  const uint32_t tmem = tmem_base_sh;
  if (warp > kProd)  // block scale factors (syrk::expand_stage_f4), one warp per TMEM lane quarter
    syrk::init_scale_factors(tmem + (uint32_t((warp & 3) * 32) << 16) + kSfCol);
  fence_before();
  __syncthreads();
  fence_after();

  if (warp == 0) {
    if (lane == 0 && t0 < t1) {
      uint32_t n = 0, u = 0;
      const uint32_t tsf = tmem + kSfCol;
      for (uint64_t t = t0; t < t1; ++t) {
#pragma unroll
        for (uint32_t c = 0; c < 2; ++c, ++u) {
          const uint32_t slot = u % kRing;
          mbar_wait(&tempty_bar[slot], ((u / kRing) & 1) ^ 1);
          fence_after();
          const uint32_t nch = (p.wq[c] + 1) / 2;
          const uint32_t dcol = tmem + slot * 128;
          for (uint32_t ch = 0; ch < nch; ++ch, ++n) {
            const uint32_t st = n % kStagesP;
            mbar_wait_spin(&full_bar[st], (n / kStagesP) & 1);
            fence_after();
            const uint32_t abase = smem_u32(stages + st * kSStageBytes);
            const uint32_t bbase = abase + kRows * kSRowBytes;
#pragma unroll
            for (int kk = 0; kk < kSRowBytes / 32; ++kk)
              syrk::mma_f4(dcol, syrk::f4_desc(abase + kk * 256), syrk::f4_desc(bbase + kk * 256),
                           tsf + syrk::sf_col(kk), (ch != 0 || kk != 0) ? 1u : 0u);
            mma_commit(&empty_bar[st]);
          }
          mma_commit(&tfull_bar[slot]);
        }
      }
    }
    __syncwarp();
  } else if (warp <= kProd) {
    const int r = threadIdx.x - 32;  // 0..127
    const uint32_t row_off = (r >> 3) * (kSRowBytes / 16) * 128 + (r & 7) * 16;
    const uint32_t stage_a = smem_u32(stages) + row_off, stage_b = stage_a + kRows * kSRowBytes;
    if (t0 < t1) {
      PWalker wk;
      wk.start(p, t0);
      uint32_t st = 0, ph = 0;
      const uint32_t rmax = 2 * p.M - 1;
      const size_t row = size_t(p.M) * 2;
      for (uint64_t t = t0; t < t1; ++t) {
#pragma unroll 1
        for (uint32_t c = 0; c < 2; ++c) {
          const uint4* pl = p.planes[c];
          const uint4* Ya = pl + min(2 * kBlk * wk.xb + r, rmax);
          const uint4* Yb = pl + min(2 * kBlk * wk.yb + r, rmax);
          const uint32_t nq = (p.wq[c] + 1) / 2 * 2;  // zero quad pads an odd count
          // plane quads of the next kAhead stages in flight (L2 latency)
          constexpr uint32_t kAhead = 2;
          uint4 pa[kAhead][2], pb[kAhead][2];
#pragma unroll
          for (uint32_t x = 0; x < kAhead; ++x)
            if (2 * x < nq) {
              pa[x][0] = __ldg(Ya + size_t(2 * x) * row); pa[x][1] = __ldg(Ya + size_t(2 * x + 1) * row);
              pb[x][0] = __ldg(Yb + size_t(2 * x) * row); pb[x][1] = __ldg(Yb + size_t(2 * x + 1) * row);
            }
          for (uint32_t q = 0; q < nq; q += 2) {
            const uint4 ca0 = pa[0][0], ca1 = pa[0][1], cb0 = pb[0][0], cb1 = pb[0][1];
#pragma unroll
            for (uint32_t x = 0; x + 1 < kAhead; ++x) {
              pa[x][0] = pa[x + 1][0]; pa[x][1] = pa[x + 1][1];
              pb[x][0] = pb[x + 1][0]; pb[x][1] = pb[x + 1][1];
            }
            if (q + 2 * kAhead < nq) {
              const size_t o = size_t(q + 2 * kAhead) * row;
              pa[kAhead - 1][0] = __ldg(Ya + o); pa[kAhead - 1][1] = __ldg(Ya + o + row);
              pb[kAhead - 1][0] = __ldg(Yb + o); pb[kAhead - 1][1] = __ldg(Yb + o + row);
            }
            mbar_wait(&empty_bar[st], ph ^ 1);
            const uint32_t so = st * kSStageBytes;
            syrk::expand_stage_f4(stage_a + so, ca0, ca1);
            syrk::expand_stage_f4(stage_b + so, cb0, cb1);
            asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
            __syncwarp();
            if (lane == 0) mbar_arrive(&full_bar[st]);
            if (++st == kStagesP) { st = 0; ph ^= 1; }
          }
        }
        wk.next();
      }
    }
  } else {
    // drain both classes of a tile together: lane = row (x, a), columns (y, b)
    // -> wide uint2 {b=0, b=1} at component offset 2a of pair[c][x*M + y] and
    // its mirror, or (narrow) the class-packed uint2 at offset 2a of
    // pairp[x*M + y] and pairp[y*M + x]
    const int quarter = warp & 3;
    const int row = quarter * 32 + lane;
    const int a = row & 1;
    if (t0 < t1) {
      PWalker wk;
      wk.start(p, t0);
      uint32_t u = 0;
      const bool e0 = p.wq[0] == 0, e1 = p.wq[1] == 0;
      for (uint64_t t = t0; t < t1; ++t, u += 2) {
        const uint32_t s0 = u % kRing, s1 = (u + 1) % kRing;
        mbar_wait(&tfull_bar[s0], (u / kRing) & 1);
        mbar_wait(&tfull_bar[s1], ((u + 1) / kRing) & 1);
        fence_after();
        const uint32_t x = wk.xb * kBlk + (row >> 1);
        const uint32_t tb = tmem + (uint32_t(quarter * 32) << 16);
#pragma unroll 1
        for (int c16 = 0; c16 < 128; c16 += 16) {
          uint32_t v0[16], v1[16];
          syrk::tmem_ld16(tb + s0 * 128 + c16, v0);
          syrk::tmem_ld16(tb + s1 * 128 + c16, v1);
          tmem_wait_ld();
#pragma unroll
          for (int e = 0; e < 8; ++e) {
            const uint32_t y = wk.yb * kBlk + (c16 >> 1) + e;
            if (x < y && y < p.M) {
              const uint2 w0 = e0 ? make_uint2(0u, 0u)
                                  : make_uint2(syrk::f32_count(v0[2 * e]), syrk::f32_count(v0[2 * e + 1]));
              const uint2 w1 = e1 ? make_uint2(0u, 0u)
                                  : make_uint2(syrk::f32_count(v1[2 * e]), syrk::f32_count(v1[2 * e + 1]));
              const size_t up = size_t(x) * p.M + y, lo = size_t(y) * p.M + x;
              if (kNarrow) {
                const uint32_t sh = p.shift;
                const uint2 pk = make_uint2((w0.x << sh) | (w1.x << (16 + sh)),
                                            (w0.y << sh) | (w1.y << (16 + sh)));
                *reinterpret_cast<uint2*>(reinterpret_cast<uint32_t*>(p.pairp + up) + 2 * a) = pk;
                *reinterpret_cast<uint2*>(reinterpret_cast<uint32_t*>(p.pairp + lo) + 2 * a) = pk;
              } else {
                *reinterpret_cast<uint2*>(reinterpret_cast<uint32_t*>(p.pair[0] + up) + 2 * a) = w0;
                *reinterpret_cast<uint2*>(reinterpret_cast<uint32_t*>(p.pair[1] + up) + 2 * a) = w1;
                *reinterpret_cast<uint2*>(reinterpret_cast<uint32_t*>(p.pair[0] + lo) + 2 * a) = w0;
                *reinterpret_cast<uint2*>(reinterpret_cast<uint32_t*>(p.pair[1] + lo) + 2 * a) = w1;
              }
            }
          }
        }
        fence_before();
        mbar_arrive(&tempty_bar[s0]);
        mbar_arrive(&tempty_bar[s1]);
        wk.next();
      }
    }
  }
  fence_before();
  __syncthreads();
  if (warp == 0) {
    fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "n"(kTmemCols));
  }
}

inline size_t smem_bytes() { return 1024 + size_t(kStagesP) * kSStageBytes; }

}  // namespace pairs_tc
