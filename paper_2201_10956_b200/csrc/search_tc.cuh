// search_tc.cuh — the tensor-core contingency kernel (included by engine.cu).
//
// The 8 counted cells of a triple are a GEMM over the sample axis:
//   T_c[a][b][g](i,j,k) = sum_{s in class c} (X_a^i & X_b^j)[s] * X_g^k[s]
// A CTA tile fixes i, a block of 32 j's and a block of 64 k's:
//   A (M=128 rows)  = pair products (j, a, b) as 0/1 bytes, K-major
//   B (N=128 rows)  = single planes (k, g) as 0/1 bytes, K-major
//   D_c (TMEM, s32) = A . B^T per class, 128 lanes x 128 columns
// issued as tcgen05.mma.cta_group::1.kind::i8 (M128 N128 K32) by one thread.
// Bit planes stay bit-packed in HBM/L2; producer warps expand each 128-sample
// word-quad to bytes directly into the canonical no-swizzle K-major smem
// layout (8-row x 16-byte core matrices). Epilogue warps read D with
// tcgen05.ld, transpose within 4-lane groups so each thread owns one triple,
// and run the same exact marginal derivation, K2 and top-k as the POPC kernel.
// Pipelines: smem stages (full/empty mbarriers, producers <-> MMA) and two
// TMEM accumulator buffers (tmem_full/tmem_empty, MMA <-> epilogue), so the
// epilogue of tile t overlaps the MMAs of tile t+1.

namespace tc {

constexpr int kJT = 32;                  // j per tile  -> A rows = 4 * 32 = 128
constexpr int kKT = 64;                  // k per tile  -> B rows = 2 * 64 = 128
constexpr int kRows = 128;
constexpr int kChunk = 256;              // samples per smem stage (two word-quads)
constexpr int kSlabs = kChunk / 16;      // 16-byte K slabs per row per stage
constexpr int kStages = 3;
constexpr int kStageBytes = 2 * kRows * kChunk;   // A + B = 64 KiB
constexpr int kProducerWarps = 8;        // warps 1..8
constexpr int kEpilogueWarps = 8;        // warps 9..16: two warpgroups split the k columns
constexpr int kThreads = 32 * (1 + kProducerWarps + kEpilogueWarps);
constexpr int kTmemCols = 512;           // 2 buffers x 2 classes x 128 columns
constexpr uint32_t kIdesc = (2u << 4)                 // D format s32
                          | (uint32_t(128 >> 3) << 17)  // N = 128
                          | (uint32_t(128 >> 4) << 24); // M = 128; A/B u8, K-major

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("{\n\t.reg .b64 st;\n\tmbarrier.arrive.shared::cta.b64 st, [%0];\n\t}" ::"r"(smem_u32(bar))
               : "memory");
}
// try_wait with a suspend-time hint: the waiting thread is parked by the
// hardware until the phase completes instead of spinning on issue slots.
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n\t.reg .pred P1;\n\tWAIT_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1, %2;\n\t"
      "@!P1 bra WAIT_%=;\n\t}" ::"r"(smem_u32(bar)), "r"(parity), "r"(0x100000)
      : "memory");
}
// Waiters that may block for a whole tile back off so their spinning does not
// steal issue slots from the producer warps on the same SM sub-partition.
__device__ __forceinline__ void mbar_wait_sleep(uint64_t* bar, uint32_t parity) {
  uint32_t done = 0, ns = 32;
  while (true) {
    asm volatile(
        "{\n\t.reg .pred P1;\n\tmbarrier.try_wait.parity.shared::cta.b64 P1, [%1], %2;\n\t"
        "selp.u32 %0, 1, 0, P1;\n\t}"
        : "=r"(done)
        : "r"(smem_u32(bar)), "r"(parity)
        : "memory");
    if (done) break;
    __nanosleep(ns);
    if (ns < 1024) ns <<= 1;
  }
}
// Tight spin (no suspend hint) for the single MMA-issuing thread: it must
// react to a filled stage within a few cycles.
__device__ __forceinline__ void mbar_wait_spin(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n\t.reg .pred P1;\n\tWAIT_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n\t"
      "@!P1 bra WAIT_%=;\n\t}" ::"r"(smem_u32(bar)), "r"(parity)
      : "memory");
}
// The same waits/arrivals on a precomputed shared-memory address (the hot
// loops of the SYRK kernel hoist the generic->shared conversions).
__device__ __forceinline__ void mbar_wait_a(uint32_t addr, uint32_t parity) {
  asm volatile(
      "{\n\t.reg .pred P1;\n\tWAIT_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1, %2;\n\t"
      "@!P1 bra WAIT_%=;\n\t}" ::"r"(addr), "r"(parity), "r"(0x100000)
      : "memory");
}
__device__ __forceinline__ void mbar_wait_spin_a(uint32_t addr, uint32_t parity) {
  asm volatile(
      "{\n\t.reg .pred P1;\n\tWAIT_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n\t"
      "@!P1 bra WAIT_%=;\n\t}" ::"r"(addr), "r"(parity)
      : "memory");
}
__device__ __forceinline__ void mbar_arrive_a(uint32_t addr) {
  asm volatile("{\n\t.reg .b64 st;\n\tmbarrier.arrive.shared::cta.b64 st, [%0];\n\t}" ::"r"(addr)
               : "memory");
}
__device__ __forceinline__ void mma_commit_a(uint32_t addr) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
      addr) : "memory");
}
__device__ __forceinline__ void sts_u32(uint32_t addr, uint32_t v) {
  asm volatile("st.shared.u32 [%0], %1;" ::"r"(addr), "r"(v) : "memory");
}
__device__ __forceinline__ uint32_t lds_u32(uint32_t addr) {
  uint32_t v;
  asm volatile("ld.shared.u32 %0, [%1];" : "=r"(v) : "r"(addr) : "memory");
  return v;
}
__device__ __forceinline__ void fence_before() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void fence_after() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }

// Shared-memory matrix descriptor: K-major, no swizzle, version 1 (sm_100).
__device__ __forceinline__ uint64_t smem_desc(uint32_t saddr) {
  constexpr uint32_t kLbo = 128;   // next 16-byte K slab
  constexpr uint32_t kSbo = kSlabs * 128;  // next 8-row core-matrix group
  return uint64_t((saddr >> 4) & 0x3fff) | (uint64_t(kLbo >> 4) << 16) |
         (uint64_t(kSbo >> 4) << 32) | (uint64_t(1) << 46);
}

__device__ __forceinline__ void mma_i8(uint32_t tmem_d, uint64_t adesc, uint64_t bdesc,
                                       uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem_d),
      "l"(adesc), "l"(bdesc), "r"(kIdesc), "r"(accumulate));
}
__device__ __forceinline__ void mma_commit(uint64_t* bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
      smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void tmem_ld8(uint32_t taddr, uint32_t (&v)[8]) {
  asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
               : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]),
                 "=r"(v[6]), "=r"(v[7])
               : "r"(taddr));
}
__device__ __forceinline__ void tmem_wait_ld() { asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory"); }

// 4 sample bits -> 4 bytes of 0/1 (bit t -> byte t); the partial products of
// 0x00204081 land on distinct bit positions, so no carries.
__device__ __forceinline__ uint32_t spread4(uint32_t nib) { return (nib * 0x00204081u) & 0x01010101u; }

// Expands one 128-sample quad (4 words) into slabs [8h, 8h+8) of row r in
// the canonical layout (16-byte slab s holds samples 16s..16s+15 of the stage).
__device__ __forceinline__ void expand_quad(uint32_t stage_saddr, int r, int h, uint4 q) {
  const uint32_t w[4] = {q.x, q.y, q.z, q.w};
  const uint32_t rowa = stage_saddr + (r >> 3) * (kSlabs * 128) + (r & 7) * 16 + h * 8 * 128;
#pragma unroll
  for (int s = 0; s < 8; ++s) {
    const uint32_t bits = w[s >> 1] >> (16 * (s & 1));
    const uint32_t o0 = spread4(bits & 0xF), o1 = spread4((bits >> 4) & 0xF);
    const uint32_t o2 = spread4((bits >> 8) & 0xF), o3 = spread4((bits >> 12) & 0xF);
    asm volatile("st.shared.v4.b32 [%0], {%1, %2, %3, %4};" ::"r"(rowa + s * 128), "r"(o0),
                 "r"(o1), "r"(o2), "r"(o3)
                 : "memory");
  }
}

// Item walk: (i, a = 32-j unit, b = 64-k tile) with b >= a/2, i-major.
struct Walker {
  uint32_t M, i, a, b, nu, nk;
  __device__ void set_i(uint32_t ii) {
    i = ii;
    const uint32_t L = M - 1 - i;
    nu = (L + kJT - 1) / kJT;
    nk = (L + kKT - 1) / kKT;
  }
  __device__ void start(uint32_t MM, const uint64_t* off, uint32_t i_hi, uint64_t item) {
    M = MM;
    uint32_t lo = 0, hi = i_hi;
    while (lo < hi) {
      const uint32_t mid = (lo + hi + 1) >> 1;
      if (off[mid] <= item) lo = mid; else hi = mid - 1;
    }
    set_i(lo);
    uint64_t u = item - off[lo];
    a = 0;
    // rows a have (nk - a/2) tiles; walk (nu <= 2^16)
    while (u >= uint64_t(nk - a / 2)) { u -= nk - a / 2; ++a; }
    b = a / 2 + uint32_t(u);
  }
  __device__ void next() {
    if (++b == nk) {
      if (++a == nu) { set_i(i + 1); a = 0; }
      b = a / 2;
    }
  }
};

struct TcArgs {
  uint64_t item_begin, item_count;
  uint64_t rank_begin, rank_end;
  uint32_t top_k;
  uint64_t* gthr;
  ulonglong2* out_lists;   // [grid * kEpilogueWarps][top_k]
  uint32_t* out_counts;
  const uint64_t* itemoff; // [M-1]
  unsigned long long* evals;  // triples evaluated (device counter, add_evals)
  Collect col;               // large top_k, second pass (offer)
};

template <bool kRanged>
__global__ void __launch_bounds__(kThreads, 1) search_tc_kernel(const DevData d, const TcArgs a) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  // 1 KiB alignment for the operand stages
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                             ~uintptr_t(1023));
  uint8_t* stages = smem;                                        // kStages x 32 KiB
  uint64_t* lists = reinterpret_cast<uint64_t*>(smem + kStages * kStageBytes);  // 4 x 2K u64
  __shared__ uint64_t full_bar[kStages], empty_bar[kStages];
  __shared__ uint64_t tfull_bar[2], tempty_bar[2];
  __shared__ uint32_t tmem_base_sh;

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint32_t M = d.M;
  const uint32_t K = a.top_k;
  const uint64_t it0 = a.item_begin + a.item_count * blockIdx.x / gridDim.x;
  const uint64_t it1 = a.item_begin + a.item_count * (blockIdx.x + 1) / gridDim.x;

  if (threadIdx.x == 0) {
    for (int s = 0; s < kStages; ++s) {
      mbar_init(&full_bar[s], kProducerWarps);
      mbar_init(&empty_bar[s], 1);
    }
    for (int b = 0; b < 2; ++b) {
      mbar_init(&tfull_bar[b], 1);
      mbar_init(&tempty_bar[b], 32 * kEpilogueWarps);
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
  const uint32_t nch0 = (d.wq[0] + 1) / 2;   // stages of class 0 (two quads each)
  const uint32_t nchunks = nch0 + (d.wq[1] + 1) / 2;

  if (it0 < it1) {
    if (warp == 0) {
      // ===================== MMA issuer (one thread) =====================
      if (lane == 0) {
        uint32_t n = 0;  // global chunk counter (stage ring)
        uint32_t t = 0;  // tile counter (TMEM ring)
        for (uint64_t it = it0; it < it1; ++it, ++t) {
          const uint32_t buf = t & 1;
          mbar_wait(&tempty_bar[buf], ((t >> 1) & 1) ^ 1);
          fence_after();
          for (uint32_t ch = 0; ch < nchunks; ++ch, ++n) {
            const uint32_t s = n % kStages;
            mbar_wait(&full_bar[s], (n / kStages) & 1);
            fence_after();
            const uint32_t cls = ch < nch0 ? 0 : 1;
            const uint32_t first = cls == 0 ? 0 : nch0;
            const uint32_t dcol = tmem + buf * 256 + cls * 128;
            const uint32_t abase = smem_u32(stages + s * kStageBytes);
            const uint32_t bbase = abase + kRows * kChunk;
#pragma unroll
            for (int kk = 0; kk < kChunk / 32; ++kk)
              mma_i8(dcol, smem_desc(abase + kk * 256), smem_desc(bbase + kk * 256),  // 2 slabs
                     (ch != first || kk != 0) ? 1u : 0u);
            mma_commit(&empty_bar[s]);
          }
          mma_commit(&tfull_bar[buf]);
        }
      }
      __syncwarp();
    } else if (warp <= kProducerWarps) {
      // ===================== producers: bits -> bytes =====================
      // Each thread owns one operand row; the plane words of the next stage
      // are fetched (not yet combined) while the current stage is expanded.
      const int pt = threadIdx.x - 32;           // 0..255
      const bool is_a = pt < kRows;
      const int r = is_a ? pt : pt - kRows;
      const uint32_t stage0 = smem_u32(stages) + (is_a ? 0 : kRows * kChunk);
      struct Cursor {
        Walker wk;
        uint32_t ch;
      };
      struct Words {
        uint4 x[2], y[2];
      };
      Cursor pf;
      pf.wk.start(M, a.itemoff, M - 3, it0);
      pf.ch = 0;
      auto fetch = [&](const Cursor& c, Words& o) {
        const uint32_t i = c.wk.i;
        const uint32_t cls = c.ch < nch0 ? 0 : 1;
        const uint32_t q = 2 * (cls == 0 ? c.ch : c.ch - nch0);
        const size_t row = size_t(M) * 2;
        const uint4* pl = (cls ? d.planes[1] : d.planes[0]) + size_t(q) * row;
        if (is_a) {  // row = j_local*4 + a*2 + b
          const uint32_t j = min(i + 1 + c.wk.a * kJT + (r >> 2), M - 1);
          const uint32_t xo = 2 * i + ((r >> 1) & 1), yo = 2 * j + (r & 1);
          o.x[0] = __ldg(pl + xo); o.x[1] = __ldg(pl + row + xo);
          o.y[0] = __ldg(pl + yo); o.y[1] = __ldg(pl + row + yo);
        } else {     // row = k_local*2 + g
          const uint32_t k = min(i + 1 + c.wk.b * kKT + (r >> 1), M - 1);
          const uint32_t xo = 2 * k + (r & 1);
          o.x[0] = __ldg(pl + xo); o.x[1] = __ldg(pl + row + xo);
        }
      };
      auto advance = [&](Cursor& c) {
        if (++c.ch == nchunks) {
          c.ch = 0;
          c.wk.next();
        }
      };
      const uint64_t total_chunks = (it1 - it0) * nchunks;
      Words cur, nxt;
      fetch(pf, cur);
      advance(pf);
      for (uint64_t n = 0; n < total_chunks; ++n) {
        if (n + 1 < total_chunks) {
          fetch(pf, nxt);
          advance(pf);
        }
        const uint32_t s = uint32_t(n % kStages);
        mbar_wait(&empty_bar[s], uint32_t((n / kStages) & 1) ^ 1);
        const uint32_t sb = stage0 + s * kStageBytes;
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          uint4 v = cur.x[h];
          if (is_a) {
            v.x &= cur.y[h].x; v.y &= cur.y[h].y; v.z &= cur.y[h].z; v.w &= cur.y[h].w;
          }
          expand_quad(sb, r, h, v);
        }
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        __syncwarp();
        if (lane == 0) mbar_arrive(&full_bar[s]);
        cur = nxt;
      }
    } else {
      // ===================== epilogue: TMEM -> K2 -> top-k =====================
      const int ew = warp - 1 - kProducerWarps;      // 0..7
      const int half = ew >> 2;                      // which 32 k's of the tile
      const int quarter = warp & 3;                  // TMEM lane quarter this warp may access
      uint64_t* ls = lists + size_t(ew) * 2 * K;
      uint64_t* lt = ls + K;
      uint32_t nlist = 0;
      uint32_t nevals = 0;
      const int jl = quarter * 8 + (lane >> 2);      // j_local 0..31
      const int ab = lane & 3;                       // this thread's (a,b) row and k phase
      Walker wk;
      wk.start(M, a.itemoff, M - 3, it0);
      uint32_t t = 0;
      for (uint64_t it = it0; it < it1; ++it, ++t) {
        const uint32_t buf = t & 1;
        mbar_wait_sleep(&tfull_bar[buf], (t >> 1) & 1);
        fence_after();
        const uint32_t i = wk.i;
        const uint32_t j = i + 1 + wk.a * kJT + jl;
        const uint32_t jc = min(j, M - 1);
        const uint64_t gth = *reinterpret_cast<volatile uint64_t*>(a.gthr);
        uint64_t rank_ij = 0;
        if (kRanged) {
          const uint64_t Mi = M - i, Mj = M - jc;
          rank_ij = (uint64_t(M) * (M - 1) * (M - 2) - Mi * (Mi - 1) * (Mi - 2)) / 6 +
                    (uint64_t(Mi - 1) * (Mi - 2)) / 2 - Mj * (Mj - 1) / 2;
        }
        const uint4 pij0 = __ldg(d.pair[0] + size_t(i) * M + jc);
        const uint4 pij1 = __ldg(d.pair[1] + size_t(i) * M + jc);
        const uint2 si0 = __ldg(d.single[0] + i), si1 = __ldg(d.single[1] + i);
        const uint2 sj0 = __ldg(d.single[0] + jc), sj1 = __ldg(d.single[1] + jc);
        for (int m = half * (kKT / 8); m < (half + 1) * (kKT / 8); ++m) {
          uint32_t v0[8], v1[8];
          const uint32_t taddr = tmem + (uint32_t(quarter * 32) << 16) + buf * 256 + 8 * m;
          tmem_ld8(taddr, v0);
          tmem_ld8(taddr + 128, v1);
          tmem_wait_ld();
          if (d.wq[0] == 0) for (int x = 0; x < 8; ++x) v0[x] = 0;
          if (d.wq[1] == 0) for (int x = 0; x < 8; ++x) v1[x] = 0;
          // 4x4 transpose in the lane quad: thread ab gets k = 4m + ab for all (a,b)
          uint32_t T0[8], T1[8];
#pragma unroll
          for (int dd = 0; dd < 4; ++dd) {
            const int src = ab ^ dd;  // partner; it sends its values for our k
            const int want = ab;      // our k phase
            // value the partner must send = partner's v[2*want + g]; every thread
            // sends v[2*(ab^dd) + g], which for the partner equals v[2*ab + g].
            const int sidx = 2 * (ab ^ dd);
            uint32_t s00 = v0[0], s01 = v0[1], s10 = v1[0], s11 = v1[1];
#pragma unroll
            for (int x = 1; x < 4; ++x)
              if (sidx == 2 * x) { s00 = v0[2 * x]; s01 = v0[2 * x + 1]; s10 = v1[2 * x]; s11 = v1[2 * x + 1]; }
            const int srcl = (lane & ~3) | src;
            const uint32_t r00 = __shfl_sync(0xffffffffu, s00, srcl);
            const uint32_t r01 = __shfl_sync(0xffffffffu, s01, srcl);
            const uint32_t r10 = __shfl_sync(0xffffffffu, s10, srcl);
            const uint32_t r11 = __shfl_sync(0xffffffffu, s11, srcl);
            // partner's row is (a,b) = src -> T index src*2 + g
            (void)want;
#pragma unroll
            for (int x = 0; x < 4; ++x)
              if (src == x) { T0[2 * x] = r00; T0[2 * x + 1] = r01; T1[2 * x] = r10; T1[2 * x + 1] = r11; }
          }
          const uint32_t k = i + 1 + wk.b * kKT + 4 * m + ab;
          const uint32_t kc = min(k, M - 1);
          bool valid = j < k && k < M;
          if (kRanged && valid) {
            const uint64_t r = rank_ij + (k - j - 1);
            valid = r >= a.rank_begin && r < a.rank_end;
          }
          uint64_t sk = ~0ull, tk = ~0ull;
          nevals += valid;
          if (valid) {
            uint32_t n0[27], n1[27];
            derive_cells(T0, pij0, __ldg(d.pair[0] + size_t(i) * M + kc),
                         __ldg(d.pair[0] + size_t(jc) * M + kc), si0, sj0,
                         __ldg(d.single[0] + kc), d.n[0], n0);
            derive_cells(T1, pij1, __ldg(d.pair[1] + size_t(i) * M + kc),
                         __ldg(d.pair[1] + size_t(jc) * M + kc), si1, sj1,
                         __ldg(d.single[1] + kc), d.n[1], n1);
            sk = score_key(k2_device(n0, n1, d.logp));
            tk = triple_key(i, j, k);
          }
          offer(valid, sk, tk, gth, ls, lt, nlist, K, lane, a.gthr, a.col);
        }
        fence_before();
        mbar_arrive(&tempty_bar[buf]);
        wk.next();
      }
      const size_t list = size_t(blockIdx.x) * kEpilogueWarps + ew;
      for (uint32_t e = lane; e < nlist; e += 32)
        a.out_lists[list * K + e] = make_ulonglong2(ls[e], lt[e]);
      if (lane == 0) a.out_counts[list] = nlist;
      add_evals(a.evals, nevals);
    }
  } else if (warp > kProducerWarps) {
    const int ew = warp - 1 - kProducerWarps;
    if (lane == 0) a.out_counts[size_t(blockIdx.x) * kEpilogueWarps + ew] = 0;
  }
  fence_before();
  __syncthreads();
  if (warp == 0) {
    fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "n"(kTmemCols));
  }
}

inline size_t smem_bytes(uint32_t top_k) {
  return 1024 + size_t(kStages) * kStageBytes + size_t(kEpilogueWarps) * 2 * top_k * sizeof(uint64_t);
}

// Items of i: sum over j-units a < nu of (nk - floor(a/2)).
inline uint64_t items_of(uint64_t M, uint64_t i) {
  const uint64_t L = M - 1 - i;
  const uint64_t nu = (L + kJT - 1) / kJT, nk = (L + kKT - 1) / kKT;
  const uint64_t s = ((nu - 1) / 2) * (nu / 2);  // sum_{a<nu} floor(a/2)
  return nu * nk - s;
}

}  // namespace tc
