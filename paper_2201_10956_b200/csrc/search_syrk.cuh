// search_syrk.cuh — compacted tensor-core engine (included by engine.cu after
// search_tc.cuh; reuses its tcgen05/mbarrier helpers).
//
// For a fixed first SNP i and genotype a in {0,1}, the counted cells are a
// Gram matrix over the samples where SNP i has genotype a:
//   T_c[a][b][g](i,j,k) = sum_{s in S_{i,a,c}} X_b^j[s] * X_g^k[s],
//   S_{i,a,c} = { s in class c : X_a^i[s] = 1 }.
// Compacting the sample axis to S_{i,a,c} (|S_0| + |S_1| ~ 0.91 N at maf 0.3)
// makes every MMA byte useful: 4 (b,g) MACs per compacted sample instead of
// the masked formulation's 8 over all samples (2.2x less MMA and operand
// expansion per triplet x sample). Per batch of i's:
//   compact_pext_kernel       Y_{i,a}[quad][row=(j,b)] = X_b^j at S_{i,a,*}
//                             (bit compression by the mask words of SNP i)
//                             (bit-packed, class 0 quads then class 1 quads,
//                             each class padded to 256 samples)
//   search_syrk_kernel        tiles (i, 64-j block, 64-k block), j-block <=
//                             k-block; phase a=0 then a=1 per tile, each into
//                             its own TMEM buffer (2 classes x 128 columns),
//                             so the epilogue of one phase overlaps the MMAs
//                             of the other. The a=0 counts go to a per-CTA
//                             scratch tile; the a=1 phase completes the 8
//                             counted cells and runs the exact derivation,
//                             K2 and top-k of the other engines.

namespace syrk {

using namespace tc;

constexpr int kJB = 64;           // SNPs per j / k block -> 128 operand rows each
// Operands are packed E2M1 (fp4, two samples per byte; a one is a single-bit
// nibble whose value the UE8M0 block scale brings back to 1.0, see
// expand_stage_regs), multiplied by tcgen05.mma kind::mxf4 with f32
// accumulation, which is exact for counts < 2^24 (host requires N_c < 2^23).
constexpr int kSChunk = 256;                           // samples per stage
constexpr int kSRowBytes = kSChunk / 2;                // 128 B per operand row
// SYRK operand stages: A (the j rows) lives in TMEM — tcgen05.mma reads it
// from there ("[a-tmem]"), so neither the producers' stores nor the tensor
// core's operand reads of A touch shared memory (measured M128 N128 K64:
// 83.5 cycles vs 127.6 with both operands in shared memory,
// tools/mxf4_ts_probe.cu) — and B (the k rows) in shared memory.
constexpr int kSyrkStages = 3;                          // a launch uses s.nst of them
constexpr int kSBStageBytes = kRows * kSRowBytes;      // B only = 16 KiB
constexpr uint32_t kAStageCols = kSRowBytes / 4;       // 32 TMEM columns per A stage
constexpr uint32_t kACol = 416;                        // A stages: columns [416, 512)
constexpr int kUnits = 3;          // TMEM ring of (tile, a, c) accumulators, 128 columns each
constexpr uint32_t kSfCol = 384;   // scale-factor columns (init_scale_factors)
static_assert(kACol >= kSfCol + 32 && kACol + kSyrkStages * kAStageCols <= 512, "TMEM columns");
// E3_PAIR: CTA pairs (cta_group::2). The pair's two CTAs take j blocks 2p
// and 2p + 1 of the same (i, k block): one M256 N128 MMA per K step (issued by
// the leader, A from each CTA's TMEM, B split over the pair's shared memory:
// each CTA expands 64 of the 128 B rows), so each SM expands half the B
// operand and the tensor core runs at 64 instead of 83.5 cycles per
// M128-equivalent K64 MMA (tools/mxf4_2cta_probe.cu).
#ifndef E3_PAIR
#define E3_PAIR 0
#endif
constexpr bool kPair = E3_PAIR != 0;
constexpr uint32_t kIdescF4 = (1u << 7) | (1u << 10)          // A, B = E2M1
                            | (uint32_t(128 >> 3) << 17)      // N = 128
                            | (1u << 23)                      // scale type UE8M0
                            | (uint32_t(128 >> 4) << 24);     // M = 128, K = 64

// the pair MMA: M = 256 (each CTA's 128 A rows)
constexpr uint32_t kIdescPair = (kIdescF4 & ~(0x1Fu << 24)) | (uint32_t(256 >> 4) << 24);
// K-major no-swizzle descriptor for a 128-byte stage row (8 16-byte slabs).
__device__ __forceinline__ uint64_t f4_desc(uint32_t saddr) {
  return uint64_t((saddr >> 4) & 0x3fff) | (uint64_t(128 >> 4) << 16) |
         (uint64_t((kSRowBytes / 16) * 128 >> 4) << 32) | (uint64_t(1) << 46);
}
__device__ __forceinline__ void mma_f4(uint32_t tmem_d, uint64_t adesc, uint64_t bdesc,
                                       uint32_t tsf, uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::mxf4.block_scale.block32 [%0], %1, %2, %3, [%5], [%5], p;\n\t}"
      ::"r"(tmem_d), "l"(adesc), "l"(bdesc), "r"(kIdescF4), "r"(accumulate), "r"(tsf));
}
// A from TMEM (lane = row, column c = row bytes [4c, 4c+4)), B from shared memory.
__device__ __forceinline__ void mma_f4_ts(uint32_t tmem_d, uint32_t tmem_a, uint64_t bdesc,
                                          uint32_t tsf, uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::mxf4.block_scale.block32 [%0], [%1], %2, %3, [%5], [%5], p;\n\t}"
      ::"r"(tmem_d), "r"(tmem_a), "l"(bdesc), "r"(kIdescF4), "r"(accumulate), "r"(tsf));
}
// One stage's four MMAs (K = 4 x 64) and the commit of its operand stage, in
// one asm block issued by one elected lane of a converged warp: the warp's
// operands are uniform, so no per-instruction single-lane waterfall is needed.
__device__ __forceinline__ void mma_stage_f4_elect(uint32_t tmem_d, uint32_t tmem_a, uint64_t bdesc,
                                                   uint32_t tsf, uint32_t accumulate, uint32_t bar) {
  asm volatile(
      "{\n\t.reg .pred e, p, t;\n\t"
      "elect.sync _|e, 0xffffffff;\n\t"
      "setp.ne.b32 p, %3, 0;\n\t"
      "setp.eq.b32 t, 0, 0;\n\t"
      ".reg .b32 a1, a2, a3, s1, s2;\n\t.reg .b64 b1, b2, b3;\n\t"
      "add.u32 a1, %1, 8;\n\tadd.u32 a2, %1, 16;\n\tadd.u32 a3, %1, 24;\n\t"
      "add.u64 b1, %2, 16;\n\tadd.u64 b2, %2, 32;\n\tadd.u64 b3, %2, 48;\n\t"
      "add.u32 s1, %4, 8;\n\tadd.u32 s2, %4, 16;\n\t"
      "@e tcgen05.mma.cta_group::1.kind::mxf4.block_scale.block32 [%0], [%1], %2, %5, [%4], [%4], p;\n\t"
      "@e tcgen05.mma.cta_group::1.kind::mxf4.block_scale.block32 [%0], [a1], b1, %5, [s1], [s1], t;\n\t"
      "@e tcgen05.mma.cta_group::1.kind::mxf4.block_scale.block32 [%0], [a2], b2, %5, [s2], [s2], t;\n\t"
      "@e tcgen05.mma.cta_group::1.kind::mxf4.block_scale.block32 [%0], [a3], b3, %5, [s2], [s2], t;\n\t"
      "@e tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%6];\n\t}"
      ::"r"(tmem_d), "r"(tmem_a), "l"(bdesc), "r"(accumulate), "r"(tsf), "r"(kIdescF4), "r"(bar)
      : "memory");
}
// the pair's stage: four M256 MMAs (leader CTA), commit multicast to both CTAs
__device__ __forceinline__ void mma_stage_pair_elect(uint32_t tmem_d, uint32_t tmem_a, uint64_t bdesc,
                                                     uint32_t tsf, uint32_t accumulate, uint32_t bar) {
  asm volatile(
      "{\n\t.reg .pred e, p, t;\n\t"
      "elect.sync _|e, 0xffffffff;\n\t"
      "setp.ne.b32 p, %3, 0;\n\t"
      "setp.eq.b32 t, 0, 0;\n\t"
      ".reg .b32 a1, a2, a3, s1, s2;\n\t.reg .b64 b1, b2, b3;\n\t"
      "add.u32 a1, %1, 8;\n\tadd.u32 a2, %1, 16;\n\tadd.u32 a3, %1, 24;\n\t"
      "add.u64 b1, %2, 16;\n\tadd.u64 b2, %2, 32;\n\tadd.u64 b3, %2, 48;\n\t"
      "add.u32 s1, %4, 8;\n\tadd.u32 s2, %4, 16;\n\t"
      "@e tcgen05.mma.cta_group::2.kind::mxf4.block_scale.block32 [%0], [%1], %2, %5, [%4], [%4], p;\n\t"
      "@e tcgen05.mma.cta_group::2.kind::mxf4.block_scale.block32 [%0], [a1], b1, %5, [s1], [s1], t;\n\t"
      "@e tcgen05.mma.cta_group::2.kind::mxf4.block_scale.block32 [%0], [a2], b2, %5, [s2], [s2], t;\n\t"
      "@e tcgen05.mma.cta_group::2.kind::mxf4.block_scale.block32 [%0], [a3], b3, %5, [s2], [s2], t;\n\t"
      "@e tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%6], %7;\n\t}"
      ::"r"(tmem_d), "r"(tmem_a), "l"(bdesc), "r"(accumulate), "r"(tsf), "r"(kIdescPair), "r"(bar),
        "h"((unsigned short)3)
      : "memory");
}
__device__ __forceinline__ void commit_pair_elect(uint32_t bar) {
  asm volatile(
      "{\n\t.reg .pred e;\n\telect.sync _|e, 0xffffffff;\n\t"
      "@e tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;\n\t}"
      ::"r"(bar), "h"((unsigned short)3) : "memory");
}
// arrive on the pair leader's (rank 0) copy of a barrier at CTA-local address
// `bar` (release at cluster scope: the data written before it is visible)
__device__ __forceinline__ void mbar_arrive_leader(uint32_t bar) {
  uint32_t remote;
  asm volatile("mapa.shared::cluster.u32 %0, %1, 0;" : "=r"(remote) : "r"(bar));
  asm volatile("mbarrier.arrive.release.cluster.shared::cluster.b64 _, [%0];" ::"r"(remote) : "memory");
}
__device__ __forceinline__ void cluster_sync() {
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}
__device__ __forceinline__ void commit_elect(uint32_t bar) {
  asm volatile(
      "{\n\t.reg .pred e;\n\telect.sync _|e, 0xffffffff;\n\t"
      "@e tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n\t}"
      ::"r"(bar) : "memory");
}
// One 256-sample stage of an operand row (two 128-sample quads q0, q1) as
// E2M1 nibbles: eight 16-byte slabs (32 samples = one block-scale K block
// each). Slab 2t+h holds "part t" of the four words of quad h: the samples
// at bit 4n+t of each word, kept in place as nibble bit t (t = 0, 1, 2:
// values 0.5, 1.0, 2.0 — a single AND) or, for t = 3 (bit 3 is the E2M1
// sign), moved to nibble bit 2 (2.0). MMA kk (two slabs, K = 64) then sees
// one encoding, undone exactly by its UE8M0 block scales (2, 1, 1/2, 1/2 on
// both A and B, kSfCol groups), so every product of two ones is 1.0: 5 ALU
// ops per 32 samples instead of 7. The sample permutation is the same for A
// and B, so every dot product is unchanged.
__device__ __forceinline__ uint32_t f4_part(uint32_t v, int t) {
  return t == 0 ? (v & 0x11111111u)
       : t == 1 ? (v & 0x22222222u)
       : t == 2 ? (v & 0x44444444u)
                : ((v >> 1) & 0x44444444u);
}
// Half `hf` of the stage (slabs 4hf .. 4hf+3, i.e. parts t = 2hf, 2hf+1) as
// 16 registers in row-byte order (register 4s + x = word x of slab s).
__device__ __forceinline__ void expand_stage_regs(uint32_t* out, uint4 q0, uint4 q1, int hf) {
  const uint32_t w[2][4] = {{q0.x, q0.y, q0.z, q0.w}, {q1.x, q1.y, q1.z, q1.w}};
#pragma unroll
  for (int tt = 0; tt < 2; ++tt)
#pragma unroll
    for (int h = 0; h < 2; ++h)
#pragma unroll
      for (int x = 0; x < 4; ++x) out[4 * (2 * tt + h) + x] = f4_part(w[h][x], 2 * hf + tt);
}
__device__ __forceinline__ void tmem_st32(uint32_t taddr, const uint32_t* v) {
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x32.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,"
      "%15,%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31,%32};" ::"r"(taddr),
      "r"(v[0]), "r"(v[1]), "r"(v[2]), "r"(v[3]), "r"(v[4]), "r"(v[5]), "r"(v[6]), "r"(v[7]),
      "r"(v[8]), "r"(v[9]), "r"(v[10]), "r"(v[11]), "r"(v[12]), "r"(v[13]), "r"(v[14]), "r"(v[15]),
      "r"(v[16]), "r"(v[17]), "r"(v[18]), "r"(v[19]), "r"(v[20]), "r"(v[21]), "r"(v[22]), "r"(v[23]),
      "r"(v[24]), "r"(v[25]), "r"(v[26]), "r"(v[27]), "r"(v[28]), "r"(v[29]), "r"(v[30]), "r"(v[31])
      : "memory");
}
__device__ __forceinline__ void tmem_st16(uint32_t taddr, const uint32_t* v) {
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,"
      "%15,%16};" ::"r"(taddr),
      "r"(v[0]), "r"(v[1]), "r"(v[2]), "r"(v[3]), "r"(v[4]), "r"(v[5]), "r"(v[6]), "r"(v[7]),
      "r"(v[8]), "r"(v[9]), "r"(v[10]), "r"(v[11]), "r"(v[12]), "r"(v[13]), "r"(v[14]), "r"(v[15])
      : "memory");
}
__device__ __forceinline__ void tmem_ld16(uint32_t taddr, uint32_t (&v)[16]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
      : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]),
        "=r"(v[7]), "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]),
        "=r"(v[14]), "=r"(v[15])
      : "r"(taddr));
}
// Exact f32 count (< 2^23) -> u32: adding 2^23 puts the integer in the mantissa.
__device__ __forceinline__ uint32_t f32_count(uint32_t bits) {
  return __float_as_uint(__uint_as_float(bits) + 8388608.f) - 0x4B000000u;
}
// Block scale factors of the encodings above, written by one warp per TMEM
// lane quarter: every byte of columns kSfCol + [0, 8) is UE8M0 2^1, of
// [8, 16) 2^0 and of [16, 32) 2^-1, so MMA kk of a stage reads its uniform
// scale at sf_col(kk) whatever the per-lane byte layout of the SF operand.
__device__ __forceinline__ void init_scale_factors(uint32_t tmem_quarter_sf) {
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x32.b32 [%0], {%1,%1,%1,%1,%1,%1,%1,%1,%2,%2,%2,%2,%2,%2,%2,%2,"
      "%3,%3,%3,%3,%3,%3,%3,%3,%3,%3,%3,%3,%3,%3,%3,%3};" ::"r"(tmem_quarter_sf),
      "r"(0x80808080u), "r"(0x7F7F7F7Fu), "r"(0x7E7E7E7Eu)
      : "memory");
  asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
}
__host__ __device__ constexpr uint32_t sf_col(int kk) {
  return kk == 0 ? 0u : kk == 1 ? 8u : 16u;
}
// The same stage of a B row into shared memory: slab s at row_saddr + 128 s
// (canonical no-swizzle K-major layout).
__device__ __forceinline__ void expand_stage_f4(uint32_t row_saddr, uint4 q0, uint4 q1) {
  const uint32_t w[2][4] = {{q0.x, q0.y, q0.z, q0.w}, {q1.x, q1.y, q1.z, q1.w}};
#pragma unroll
  for (int t = 0; t < 4; ++t)
#pragma unroll
    for (int h = 0; h < 2; ++h)
      asm volatile("st.shared.v4.b32 [%0], {%1, %2, %3, %4};" ::"r"(row_saddr + (2 * t + h) * 128),
                   "r"(f4_part(w[h][0], t)), "r"(f4_part(w[h][1], t)), "r"(f4_part(w[h][2], t)),
                   "r"(f4_part(w[h][3], t))
                   : "memory");
}
constexpr int kRounds = 8;        // 4-column rounds per epilogue warpgroup (32 k)
constexpr int kScratchPerThread = kRounds * 32;  // u32: 8 values x 2 classes x 2 phases per round
constexpr int kSmemScratchBytes = kRounds * 16 * 256 * 4;  // narrow: class-packed, 128 KiB
// 16 warps = four warpgroups: WG0 (warps 0-3) expand operands (thread r owns
// A row r — TMEM lane r, so each warp writes its own lane quarter — and B row
// r), WG1-2 (warps 4-11) run the epilogue, WG3 warp 12 issues the MMAs (13-15
// idle). setmaxnreg moves registers to the epilogue: per SM sub-partition
// (one warp of WG0 and of WG3, two of WG1-2) 120 + 2 * 168 + 56 = 512 = the
// 16K-register file / 32 lanes (13 uniform warps were capped at 128 each).
// narrow epilogue: per warp, pair(i, k) and single(k) of its 32 k of the tile
// staged in shared memory (loaded a tile ahead into registers), so the rounds
// read them with broadcast LDS instead of global loads that miss the small L1
constexpr int kKStageBytes = 32 * 16 + 32 * 8;
constexpr int kKStageTotal = kKStageBytes * 8;   // kEpilogueWarps warps
__device__ __forceinline__ uint4 lds_u128(uint32_t a) {
  uint4 v;
  asm volatile("ld.shared.v4.u32 {%0, %1, %2, %3}, [%4];" : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "r"(a));
  return v;
}
__device__ __forceinline__ uint2 lds_u64(uint32_t a) {
  uint2 v;
  asm volatile("ld.shared.v2.u32 {%0, %1}, [%2];" : "=r"(v.x), "=r"(v.y) : "r"(a));
  return v;
}
// Y staging ring (when shared memory is free: no screening table / global
// scratch, e.g. cfg4): warp 13 streams each operand stage's bit-packed Y rows
// (A quads q, q+1 and B quads q, q+1: four 2 KiB bulk copies, 128 rows x 16 B
// each, contiguous in the quad-major Y layout) into a slot ahead of the
// producers, who then read their row with one conflict-free LDS.128 each.
constexpr int kMaxYSlots = 16;
constexpr int kYSlotBytes = 4 * 128 * 16;
constexpr int kSyrkProducerWarps = 4;
constexpr int kSyrkThreads = 32 * 16;
#ifndef E3_REG_PROD
#define E3_REG_PROD 120
#define E3_REG_EPI 168
#endif
#ifndef E3_REG_MMA
#define E3_REG_MMA 56
#endif
constexpr int kRegProducer = E3_REG_PROD, kRegEpilogue = E3_REG_EPI, kRegMma = E3_REG_MMA;
#ifndef E3_PJK_LATE
#define E3_PJK_LATE 1  // mode 3 rounds (with E3_W_INPLACE): next pair(j,k) rows loaded after derive_cells
#endif
#ifndef E3_W_INPLACE
#define E3_W_INPLACE 1  // narrow rounds: next-round scratch words loaded in place after T
#endif
#ifndef E3_ROUND_UNROLL
#define E3_ROUND_UNROLL 1
#endif
constexpr int kRoundUnroll = E3_ROUND_UNROLL;  // narrow epilogue: unroll of the round loop
// code size matters (the SM's instruction cache is shared by three warp
// roles): unroll factors of the MMA issuer's unit (a, c) and stage loops and
// of the narrow drain's slot loop
#ifndef E3_MMA_WARP
#define E3_MMA_WARP 1  // MMA issuer as a converged warp (elect inside the asm)
#endif
#ifndef E3_PROD_DEPTH
#define E3_PROD_DEPTH 0  // producers: operand stages of Y words in flight (2 or 3 register sets;
                         // 0 = per kernel mode, see kProdDepth; 4 measured slower)
#endif
#ifndef E3_MMA_AC_UNROLL
#define E3_MMA_AC_UNROLL 1
#define E3_MMA_CH_UNROLL 1
#define E3_DRAIN_UNROLL 2
#endif
constexpr int kMmaAcUnroll = E3_MMA_AC_UNROLL, kMmaChUnroll = E3_MMA_CH_UNROLL,
              kDrainUnroll = E3_DRAIN_UNROLL;
static_assert(kRegProducer + 2 * kRegEpilogue + kRegMma <= 512 && kRegProducer % 8 == 0 &&
              kRegEpilogue % 8 == 0, "setmaxnreg budgets");
constexpr int kEpiWarp0 = 4, kMmaWarp = 12;

// Per-i layout of the compacted operands (one record per i of the batch).
struct IInfo {
  // Per class c only two of the three genotype phases of SNP i are computed
  // ("slots" p = 0, 1: phases lo < hi); the largest phase drop[c] follows
  // exactly from the pair index: T_drop[b][g] = P_jk[b][g] - T_lo - T_hi.
  uint64_t y_off[2];     // uint4 offset of Y_{i,p} (slot p, both classes) in the batch buffer
  uint32_t n[2][2];      // |S_{i,phase(p,c),c}|
  uint32_t q[2][2];      // quads of class c in Y_{i,p} (even: 256-sample stages)
  uint32_t R;            // rows = 2 (M - 1 - i)
  uint32_t nb;           // 64-SNP blocks above i
  uint32_t drop[2];      // dropped phase per class (slots hold the other two, ascending)
};

struct SyrkArgs {
  uint64_t item_begin, item_count;   // items of this batch (tile index space)
  uint64_t rank_begin, rank_end;
  uint32_t top_k;
  uint32_t i_lo, n_i;                // batch = [i_lo, i_lo + n_i)
  uint64_t* gthr;
  ulonglong2* lists;                 // [grid * kEpilogueWarps][top_k], persistent
  uint32_t* counts;
  const IInfo* info;                 // [n_i]
  const uint64_t* itemoff;           // [n_i + 1] tile prefix within the batch
  const uint4* Y;
  uint32_t* scratch;                 // [grid][kRounds * 16][256]
  unsigned long long* evals;         // triples evaluated (device counter, add_evals)
  Collect col;                       // large top_k, second pass (offer)
  uint32_t debug_skip;               // profiling only (E3_DEBUG_SKIP): 1 = no scoring, 2 = no
                                     // operand expansion, 4 = derivation without the screen,
                                     // 8 = no MMAs (barrier protocol only), 16 = conflict-
                                     // free screen lookups (scaled path)
  uint32_t screen;                   // 1: K2 screening table in shared memory (d.ktab)
  uint32_t nst;                      // operand stages in use (2..kSyrkStages)
  uint32_t ktab_n;                   // screening-table entries staged in shared memory
  uint32_t ny;                       // Y staging slots in shared memory (0: register prefetch)
};

// Profiling-only variants (E3_DEBUG_SKIP) exist only in a library built with
// -DE3_PROFILE_SKIP=1 (build.py build_profile_variant); the product build
// compiles every check below away.
#ifndef E3_PROFILE_SKIP
#define E3_PROFILE_SKIP 0
#endif
// E3_TIMELINE=1 (profiling builds only): per-role cycle counters printed by
// the first CTAs at kernel end (waits on each barrier, drain, rounds)
#ifndef E3_TIMELINE
#define E3_TIMELINE 0
#endif
__device__ __forceinline__ long long tl_clock() {
  if constexpr (E3_TIMELINE) return clock64();
  else return 0;
}
__device__ __forceinline__ uint32_t dbg_skip(const SyrkArgs& s) {
  return E3_PROFILE_SKIP ? s.debug_skip : 0u;
}

// Y_{i,p} by bit compression: for slot p (phase a) and class c, every
// operand row (j, b) keeps the bits of X_b^j at the samples where SNP i has
// genotype a, in sample order (= positions ascending). The mask word of i is
// shared by all rows of the block, so the five shift masks of the parallel
// compress (Hacker's Delight 7-4) are computed once per word into shared
// memory; each row then compresses a source word in 16 ALU ops and appends
// popc(mask) bits to a 64-bit accumulator that emits 128-bit output quads.
// Block = 128 rows of one (i, p, c); rows read/write coalesced uint4s.
// Long sample axes are split into `nseg` segments of kPextSeg source words
// (grid z = i x segment): a segment starts at the output bit offset given by
// the popcount of the mask before it, owns its interior output words (plain
// stores) and ORs its two partial boundary words into a pre-zeroed Y.
constexpr uint32_t kPextSeg = 256;  // source words (8192 samples) per segment
__global__ void __launch_bounds__(128) compact_pext_kernel(const DevData d, const SyrkArgs s,
                                                           uint4* __restrict__ Y, uint32_t nseg) {
  const uint32_t ii = blockIdx.z / nseg, seg = blockIdx.z % nseg;
  const uint32_t p = blockIdx.y >> 1, c = blockIdx.y & 1;
  const IInfo* inf = s.info + ii;
  const uint32_t i = s.i_lo + ii;
  const uint32_t R = inf->R;
  if (blockIdx.x * 128 >= R) return;
  const uint32_t drop = inf->drop[c];
  const uint32_t a = (p == 0) ? (drop == 0 ? 1u : 0u) : (drop == 2 ? 1u : 2u);
  const uint32_t qout = inf->q[p][c];
  const uint32_t row = blockIdx.x * 128 + threadIdx.x;
  const bool active = row < R;
  const uint32_t snp = min(i + 1 + (row >> 1), d.M - 1), g = row & 1;
  const uint32_t ncls = d.n[c];
  const uint32_t nw = (ncls + 31) / 32;  // source words of the class
  const uint32_t wbeg = seg * kPextSeg, wend = min(nw, wbeg + kPextSeg);
  if (nseg > 1 && wbeg >= nw) return;
  const size_t rstride = size_t(d.M) * 2;
  const uint4* pl = c ? d.planes[1] : d.planes[0];
  uint4* dst = Y + inf->y_off[p] + size_t(c ? inf->q[p][0] : 0) * R + row;
  __shared__ uint32_t smv[5][128], smask[128], sred[4];
  auto mask_word = [&](uint32_t w) -> uint32_t {
    const uint4 q0 = __ldg(pl + size_t(w >> 2) * rstride + 2 * i);
    const uint4 q1 = __ldg(pl + size_t(w >> 2) * rstride + 2 * i + 1);
    const uint32_t c0[4] = {q0.x, q0.y, q0.z, q0.w}, c1[4] = {q1.x, q1.y, q1.z, q1.w};
    if (a == 0) return c0[w & 3];
    if (a == 1) return c1[w & 3];
    const uint32_t lo = w * 32;
    const uint32_t valid = ncls - lo >= 32 ? ~0u : ((1u << (ncls - lo)) - 1u);
    return ~(c0[w & 3] | c1[w & 3]) & valid;
  };
  uint64_t acc = 0;
  uint32_t nacc = 0, nq = 0, ne = 0;
  uint32_t o0 = 0, o1 = 0, o2 = 0, o3 = 0;
  uint32_t kw = 0;       // segmented: output word index of the next emitted word
  bool first = false;    // segmented: the next emitted word is the shared first word
  if (nseg > 1) {
    // output bit offset of this segment = popcount of the mask before it
    uint32_t cnt = 0;
    for (uint32_t w = threadIdx.x; w < wbeg; w += 128) cnt += __popc(mask_word(w));
#pragma unroll
    for (int o = 16; o; o >>= 1) cnt += __shfl_xor_sync(0xffffffffu, cnt, o);
    if ((threadIdx.x & 31) == 0) sred[threadIdx.x >> 5] = cnt;
    __syncthreads();
    const uint32_t off = sred[0] + sred[1] + sred[2] + sred[3];
    kw = off >> 5;
    nacc = off & 31;
    first = nacc != 0;
  }
  auto emit = [&](uint32_t w) {  // uniform across the block: counts depend on the mask only
    if (nseg > 1) {
      uint32_t* wp = reinterpret_cast<uint32_t*>(dst + size_t(kw >> 2) * R) + (kw & 3);
      if (active) {
        if (first) atomicOr(wp, w);
        else *wp = w;
      }
      first = false;
      ++kw;
      return;
    }
    o0 = o1; o1 = o2; o2 = o3; o3 = w;
    if (++ne == 4) {
      if (active) dst[size_t(nq) * R] = make_uint4(o0, o1, o2, o3);
      ++nq;
      ne = 0;
    }
  };
  for (uint32_t w0 = wbeg; w0 < wend; w0 += 128) {
    {
      const uint32_t w = w0 + threadIdx.x;
      uint32_t m = w < wend ? mask_word(w) : 0u;
      smask[threadIdx.x] = m;
      uint32_t mk = ~m << 1;
#pragma unroll
      for (int k = 0; k < 5; ++k) {
        uint32_t mp = mk ^ (mk << 1);
        mp ^= mp << 2;
        mp ^= mp << 4;
        mp ^= mp << 8;
        mp ^= mp << 16;
        const uint32_t mv = mp & m;
        smv[k][threadIdx.x] = mv;
        m = (m ^ mv) | (mv >> (1 << k));
        mk &= ~mp;
      }
    }
    __syncthreads();
    const uint32_t wn = min(128u, wend - w0);
    for (uint32_t x = 0; x < wn; x += 4) {
      const uint4 src = __ldg(pl + size_t((w0 + x) >> 2) * rstride + 2 * snp + g);
      const uint32_t sw[4] = {src.x, src.y, src.z, src.w};
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        if (x + e >= wn) break;
        const uint32_t m = smask[x + e];
        if (m == 0) continue;
        uint32_t v = sw[e] & m;
#pragma unroll
        for (int k = 0; k < 5; ++k) {
          const uint32_t t = v & smv[k][x + e];
          v = (v ^ t) | (t >> (1 << k));
        }
        acc |= uint64_t(v) << nacc;
        nacc += __popc(m);
        if (nacc >= 32) {
          emit(uint32_t(acc));
          acc >>= 32;
          nacc -= 32;
        }
      }
    }
    __syncthreads();
  }
  if (nseg > 1) {
    // the last partial word is shared with the next segment; padding is pre-zeroed
    if (nacc > 0) {
      first = true;
      emit(uint32_t(acc));
    }
    return;
  }
  // flush and zero-pad to the slot's quad count (256-sample stages)
  if (nacc > 0) emit(uint32_t(acc));
  while (nq < qout) emit(0u);
}

// Tile walk within a batch: (i, jb, kb) with jb <= kb < nb(i).
// Tile walk within a batch: (i, jb, kb), kb >= kb_first(jb); with kPair jb
// indexes pairs of j blocks (2 jb, 2 jb + 1) whose tiles share the k block.
__host__ __device__ constexpr uint32_t n_jb(uint32_t nb) { return kPair ? (nb + 1) / 2 : nb; }
__host__ __device__ constexpr uint32_t kb_first(uint32_t jb) { return kPair ? 2 * jb : jb; }
struct SWalker {
  uint32_t ii, jb, kb, nb;
  __device__ void start(const SyrkArgs& s, uint64_t item) {
    uint32_t lo = 0, hi = s.n_i - 1;
    while (lo < hi) {
      const uint32_t mid = (lo + hi + 1) >> 1;
      if (s.itemoff[mid] <= item) lo = mid; else hi = mid - 1;
    }
    ii = lo;
    nb = s.info[ii].nb;
    uint64_t u = item - s.itemoff[ii];
    jb = 0;
    while (u >= uint64_t(nb - kb_first(jb))) { u -= nb - kb_first(jb); ++jb; }
    kb = kb_first(jb) + uint32_t(u);
  }
  __device__ void next(const SyrkArgs& s) {
    if (++kb == nb) {
      if (++jb == n_jb(nb)) {
        ++ii;
        jb = 0;
        if (ii < s.n_i) nb = s.info[ii].nb;
      }
      kb = kb_first(jb);
    }
  }
};

// The rare tail of a narrow round, out of line so the hot round loop stays
// compact in the instruction cache: the exact K2 of the triples whose screen
// passed, then the warp's top-k offers (warp-synchronous; called by whole
// warps). Inputs by value (no addressable register arrays on the hot path).
struct RareIn {
  uint32_t T[2][8];
  uint4 pij, pik[2], pjk[2];
  uint2 sip, sjp, skp[2];
  uint32_t i, j, kk[2];
  bool pass[2], valid[2];
};
struct RareState {
  uint32_t nlist;
  uint64_t lastS, lastT;
};
template <uint32_t kSh>
__device__ __noinline__ RareState syrk_rare(const RareIn in, const double* __restrict__ logp,
                                            uint32_t npk, uint64_t gth, uint64_t* ls, uint64_t* lt,
                                            RareState st, uint32_t K, uint64_t* gthr, const Collect col) {
  const int lane = threadIdx.x & 31;
  uint64_t sk[2] = {~0ull, ~0ull}, tk[2] = {~0ull, ~0ull};
#pragma unroll 1
  for (int h = 0; h < 2; ++h) {
    if (in.pass[h]) {
      uint32_t n[27], n0[27], n1[27];
      derive_cells(in.T[h], in.pij, in.pik[h], in.pjk[h], in.sip, in.sjp, in.skp[h], npk, n);
#pragma unroll
      for (int c = 0; c < 27; ++c) {
        n0[c] = (n[c] & 0xffffu) >> kSh;
        n1[c] = n[c] >> (16 + kSh);
      }
      sk[h] = score_key(k2_device(n0, n1, logp));
      tk[h] = triple_key(in.i, in.j, in.kk[h]);
    }
  }
#pragma unroll 1
  for (int h = 0; h < 2; ++h)
    offer_cached(in.valid[h], sk[h], tk[h], gth, ls, lt, st.nlist, K, lane, gthr, col, st.lastS, st.lastT);
  return st;
}

// kNarrow: every class has < 2^16 samples, so counts are carried as
// class-packed u16 pairs (class0 | class1 << 16) — scratch, pair index,
// singles — and the dropped-phase recovery and the table derivation run on
// both classes at once (every intermediate is a true count, so the packed
// 32-bit arithmetic never carries or borrows across the halves).
// kMode: 0 = wide, 1 = narrow, 2 = narrow with counts scaled by 4 (every
// class < 2^14 samples): a packed word then holds the byte offsets of its two
// counts in the screening table, which saves the index arithmetic per lookup;
// 3 = as 2 with the screen's pooled term from Stirling's bound (the table in
// shared memory then ends at max(N0, N1)).
// kSS (narrow only): the epilogue's thread-private scratch lives in shared
// memory (after the B stages) instead of per-CTA global memory.
#if E3_PAIR
#define E3_SYRK_CLUSTER __cluster_dims__(2, 1, 1)
#else
#define E3_SYRK_CLUSTER
#endif
template <bool kRanged, int kMode, bool kSS = false>
__global__ void E3_SYRK_CLUSTER __launch_bounds__(kSyrkThreads, 1)
search_syrk_kernel(const DevData d, const SyrkArgs s) {
  constexpr bool kNarrow = kMode >= 1;
  static_assert(kNarrow || !kSS, "shared-memory scratch is narrow-only");
  constexpr uint32_t kSh = kMode >= 2 ? 2u : 0u;  // count scale shift of packed words
  // producer prefetch depth: 3 where the operands stream (cfg4 +9%, cfg5 +1.3%,
  // cfg2 +1.5%); 2 for the Stirling-scaled path (cfg3), where the larger loop
  // cost 0.3% on the same box
  constexpr int kProdDepth = E3_PROD_DEPTH == 0 ? (kMode == 3 ? 2 : 3) : E3_PROD_DEPTH;
  // measured: cfg3 (mode 3) +0.5%, cfg2 (mode 2) -1.6%
  constexpr bool kPjkLate = E3_PJK_LATE && E3_W_INPLACE && kMode == 3;
  // no-swizzle K-major operand tiles need 16-byte alignment only
  extern __shared__ __align__(128) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 127) &
                                             ~uintptr_t(127));
  uint8_t* stages = smem;
  const uint32_t nst = s.nst;  // operand stages in use (fewer frees room for the K2 table)
  uint32_t* const sscr = reinterpret_cast<uint32_t*>(smem + nst * kSBStageBytes);
  uint64_t* lists = reinterpret_cast<uint64_t*>(smem + nst * kSBStageBytes +
                                                (kSS ? kSmemScratchBytes : 0));
  float* ktab = reinterpret_cast<float*>(lists + size_t(kEpilogueWarps) * 2 * s.top_k);
  // narrow: per-warp k staging (kKStageTotal bytes) after the screening table
  uint8_t* kstage = reinterpret_cast<uint8_t*>(ktab) + (s.screen ? size_t(s.ktab_n) * 4 : 0);
  uint8_t* yring = reinterpret_cast<uint8_t*>(
      (reinterpret_cast<uintptr_t>(kstage + (kNarrow ? kKStageTotal : 0)) + 127) & ~uintptr_t(127));
  __shared__ uint64_t yfull_bar[kMaxYSlots], yempty_bar[kMaxYSlots];
  __shared__ uint64_t full_bar[kSyrkStages], empty_bar[kSyrkStages];
  __shared__ uint64_t tfull_bar[kUnits], tempty_bar[kUnits];
  __shared__ uint32_t tmem_base_sh;

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint32_t M = d.M;
  const uint32_t K = s.top_k;
  // kPair: the two CTAs of a cluster walk the same items (crank = which j block)
  uint32_t crank = 0;
  if constexpr (kPair) asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(crank));
  const uint32_t nclus = kPair ? gridDim.x / 2 : gridDim.x, cidx = kPair ? blockIdx.x / 2 : blockIdx.x;
  const uint64_t it0 = s.item_begin + s.item_count * cidx / nclus;
  const uint64_t it1 = s.item_begin + s.item_count * (cidx + 1) / nclus;

  if (threadIdx.x == 0) {
    for (int st = 0; st < kSyrkStages; ++st) {
      // kPair: the leader's barriers also count one forwarded arrival from the peer
      mbar_init(&full_bar[st], kSyrkProducerWarps + (kPair && crank == 0 ? 1 : 0));
      mbar_init(&empty_bar[st], 1);
    }
    for (uint32_t y = 0; y < s.ny; ++y) {
      mbar_init(&yfull_bar[y], 1);
      mbar_init(&yempty_bar[y], kSyrkProducerWarps);
    }
    for (int b = 0; b < kUnits; ++b) {
      mbar_init(&tfull_bar[b], 1);
      mbar_init(&tempty_bar[b], kPair ? kEpilogueWarps + (crank == 0 ? 1 : 0) : 32 * kEpilogueWarps);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 0) {
    if constexpr (kPair) {
      asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                       smem_u32(&tmem_base_sh)), "n"(kTmemCols));
      asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;");
    } else {
      asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                       smem_u32(&tmem_base_sh)), "n"(kTmemCols));
      asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
  }
  if (s.screen) {  // K2 screening table -> shared memory
    const float4* src = reinterpret_cast<const float4*>(d.ktab);
    float4* dst = reinterpret_cast<float4*>(ktab);
    for (uint32_t x = threadIdx.x; x < s.ktab_n / 4; x += blockDim.x) dst[x] = __ldg(src + x);
  }
  fence_before();
  if constexpr (kPair) cluster_sync();  // the peer's barriers exist before any remote arrival
  else __syncthreads();
  fence_after();
  const uint32_t tmem = tmem_base_sh;
  uint32_t ktab_s = smem_u32(ktab);
  asm volatile("" : "+r"(ktab_s));  // keep in a register (see scr_s)
  // shared addresses of the barriers, hoisted out of the hot loops
  uint32_t full_s = smem_u32(full_bar), empty_s = smem_u32(empty_bar);
  uint32_t tfull_s = smem_u32(tfull_bar), tempty_s = smem_u32(tempty_bar);
  // opaque: the compiler would recompute generic->shared conversions (S2UR
  // SR_CgaCtaId + address arithmetic) inside the loops
  asm volatile("" : "+r"(full_s), "+r"(empty_s), "+r"(tfull_s), "+r"(tempty_s));
  // Block scale factors (expand_stage_regs) in columns [kSfCol, kSfCol+32) of
  // all 128 lanes: one epilogue warp per TMEM lane quarter writes them.
  if (warp >= kEpiWarp0 && warp < kEpiWarp0 + 4)
    init_scale_factors(tmem + (uint32_t((warp & 3) * 32) << 16) + kSfCol);
  fence_before();
  __syncthreads();
  fence_after();

  if (warp >= kMmaWarp) {
    asm volatile("setmaxnreg.dec.sync.aligned.u32 %0;" ::"n"(kRegMma));
  }
  if (warp == kMmaWarp) {
    // ===================== MMA issuer (one thread) =====================
    // Units (tile, a, c) in order; unit u accumulates into ring slot u % kUnits.
    // kPair: the peer CTA's warp 12 forwards its producers' and epilogue's
    // local barrier completions to the leader, one cluster-scope arrival each
    // (producer warps arriving remotely themselves paid a cluster release per
    // stage that waited for their in-flight prefetch loads: 44% slower)
    if ((E3_MMA_WARP || lane == 0) && it0 < it1) {
      SWalker wk;
      wk.start(s, it0);
      // one thread (or a converged warp with E3_MMA_WARP, electing the issuing
      // lane inside the asm), so every dependent instruction's latency is exposed:
      // stage / slot indices and phases advance incrementally (no division by
      // the runtime stage count) and the B descriptors are base + offsets
      // (the 14-bit address field cannot carry: shared addresses < 256 KiB)
      uint32_t st = 0, ph = 0, slot = 0, sph = 1;
      uint32_t fwd_units = 0;  // kPair forwarder: units seen
      const uint32_t tsf = tmem + kSfCol;
      const uint64_t bdesc0 = f4_desc(smem_u32(stages));
      long long tl_t0 = tl_clock(), tl_we = 0, tl_wf = 0;
      for (uint64_t it = it0; it < it1; ++it) {
        const IInfo& inf = s.info[wk.ii];
#pragma unroll kMmaAcUnroll
        for (uint32_t a = 0; a < 2; ++a) {
#pragma unroll kMmaAcUnroll
          for (uint32_t c = 0; c < 2; ++c) {
            long long tl_a = tl_clock();
            mbar_wait_a(tempty_s + 8 * slot, sph);
            tl_we += tl_clock() - tl_a;
            fence_after();
            const uint32_t nch = inf.q[a][c] / 2;
            if (kPair && crank != 0) {  // forwarder: the unit's release, then its stages
              // (the first kUnits waits pass on the initially free slots: nothing to forward)
              if (lane == 0 && fwd_units >= uint32_t(kUnits)) mbar_arrive_leader(tempty_s + 8 * slot);
              ++fwd_units;
              for (uint32_t ch = 0; ch < nch; ++ch) {
                mbar_wait_spin_a(full_s + 8 * st, ph);
                if (lane == 0) mbar_arrive_leader(full_s + 8 * st);
                if (++st == nst) { st = 0; ph ^= 1; }
              }
              if (++slot == kUnits) { slot = 0; sph ^= 1; }
              continue;
            }
            const uint32_t dcol = tmem + slot * 128;
#pragma unroll kMmaChUnroll
            for (uint32_t ch = 0; ch < nch; ++ch) {
              long long tl_b = tl_clock();
              mbar_wait_spin_a(full_s + 8 * st, ph);
              tl_wf += tl_clock() - tl_b;
              fence_after();
              const uint32_t acol = tmem + kACol + st * kAStageCols;
              const uint64_t bd = bdesc0 + st * uint32_t(kSBStageBytes >> 4);
              static_assert(kSRowBytes / 32 == 4 && sf_col(1) == 8 && sf_col(2) == 16 && sf_col(3) == 16,
                            "mma_stage_f4_elect layout");
              if (kPair) {
                mma_stage_pair_elect(dcol, acol, bd, tsf, ch != 0 ? 1u : 0u, empty_s + 8 * st);
              } else if (E3_MMA_WARP) {
                mma_stage_f4_elect(dcol, acol, bd, tsf, ch != 0 ? 1u : 0u, empty_s + 8 * st);
              } else {
                if (!(dbg_skip(s) & 8)) {
#pragma unroll
                  for (int kk = 0; kk < kSRowBytes / 32; ++kk)
                    mma_f4_ts(dcol, acol + kk * 8, bd + kk * (256 >> 4), tsf + sf_col(kk),
                              (ch != 0 || kk != 0) ? 1u : 0u);
                }
                mma_commit_a(empty_s + 8 * st);
              }
              if (++st == nst) { st = 0; ph ^= 1; }
            }
            if (kPair) commit_pair_elect(tfull_s + 8 * slot);
            else if (E3_MMA_WARP) commit_elect(tfull_s + 8 * slot);
            else mma_commit_a(tfull_s + 8 * slot);
            if (++slot == kUnits) { slot = 0; sph ^= 1; }
          }
        }
        wk.next(s);
      }
      if (E3_TIMELINE && blockIdx.x < 3 && lane == 0)
        printf("TL cta %d mma: total %lld wait_tempty %lld wait_full %lld tiles %llu\n", blockIdx.x,
               tl_clock() - tl_t0, tl_we, tl_wf, (unsigned long long)(it1 - it0));
    }
    __syncwarp();
  } else if (warp < kSyrkProducerWarps) {
    asm volatile("setmaxnreg.dec.sync.aligned.u32 %0;" ::"n"(kRegProducer));
    // ===================== producers: compacted bits -> E2M1 nibbles =====================
    // Each thread owns A row r (TMEM lane r: a warp reaches only its own lane
    // quarter, hence r = 32 (warp & 3) + lane) and B row r (shared memory); the
    // Y words of the next kAhead stages are prefetched into registers.
    const int r = (warp & 3) * 32 + lane;       // 0..127
    const uint32_t row_off = (r >> 3) * (kSRowBytes / 16) * 128 + (r & 7) * 16;
    const uint32_t stage_b = smem_u32(stages) + row_off;
    const uint32_t tmem_a = tmem + (uint32_t((warp & 3) * 32) << 16) + kACol;
    const bool has_b = !kPair || r < 64;        // kPair: each CTA expands 64 B rows (warp-uniform)
    if (it0 < it1 && s.ny > 0) {
      // Y words from the staging ring (warp 13 streams them ahead)
      SWalker wk;
      wk.start(s, it0);
      uint32_t st = 0, ph = 0, ys = 0, yph = 0;
      const uint32_t ring_s = smem_u32(yring) + r * 16;
      const uint32_t yfull_s = smem_u32(yfull_bar), yempty_s = smem_u32(yempty_bar);
      for (uint64_t it = it0; it < it1; ++it) {
        const IInfo inf = s.info[wk.ii];
#pragma unroll 1
        for (uint32_t a = 0; a < 2; ++a) {
          const uint32_t nsu = (inf.q[a][0] + inf.q[a][1]) / 2;
          for (uint32_t u = 0; u < nsu; ++u) {
            mbar_wait_a(yfull_s + 8 * ys, yph);
            const uint32_t yb = ring_s + ys * kYSlotBytes;
            const uint4 x0 = lds_u128(yb), x1 = lds_u128(yb + 2048);
            const uint4 y0 = lds_u128(yb + 4096), y1 = lds_u128(yb + 6144);
            // generic-proxy reads of the slot before the loader's next bulk copy
            // (async proxy) overwrites it: without this proxy fence the copy
            // could land first (cfg4: 4 of 150 searches differed)
            asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
            __syncwarp();
            if (lane == 0) mbar_arrive_a(yempty_s + 8 * ys);
            if (++ys == s.ny) { ys = 0; yph ^= 1; }
            mbar_wait_a(empty_s + 8 * st, ph ^ 1);
            fence_after();  // the MMAs that read this stage have completed
#pragma unroll
            for (int hf = 0; hf < 2; ++hf) {
              uint32_t av[16];
              expand_stage_regs(av, x0, x1, hf);
              tmem_st16(tmem_a + st * kAStageCols + 16 * hf, av);
            }
            expand_stage_f4(stage_b + st * kSBStageBytes, y0, y1);
            asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
            fence_before();
            asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
            __syncwarp();
            if (lane == 0) mbar_arrive_a(full_s + 8 * st);
            if (++st == nst) { st = 0; ph ^= 1; }
          }
        }
        wk.next(s);
      }
    } else if (it0 < it1) {
      SWalker wk;
      wk.start(s, it0);
      uint32_t st = 0, ph = 0;
      long long tl_t0 = tl_clock(), tl_w = 0;
      for (uint64_t it = it0; it < it1; ++it) {
        const IInfo inf = s.info[wk.ii];
        // kPair: this CTA's j block of the pair; its half (64 rows) of the B rows
        const uint32_t jbx = kPair ? 2 * wk.jb + crank : wk.jb;
        const uint32_t row_a = min(jbx * 2 * kJB + r, inf.R - 1);
        const uint32_t row_b = min(wk.kb * 2 * kJB + (kPair ? 64 * crank : 0u) + r, inf.R - 1);
#pragma unroll 1
        for (uint32_t a = 0; a < 2; ++a) {
          const uint4* __restrict__ Ya = s.Y + inf.y_off[a] + row_a;
          const uint4* __restrict__ Yb = s.Y + inf.y_off[a] + row_b;
          const uint32_t R = inf.R;
          const uint32_t qtot = inf.q[a][0] + inf.q[a][1];  // even: 256-sample stages
          // Y quads of the next E3_PROD_DEPTH stages in flight (L2 / HBM
          // latency): that many named register sets, the loop unrolled over
          // them so the load of stage q + depth refills the set stage q just
          // consumed (register rotation would wait for the in-flight loads one
          // stage early; indexed register arrays compiled badly), with running
          // row pointers (no per-load 64-bit index arithmetic)
          const uint32_t nsu = qtot / 2;  // stages of this unit
          const size_t R2 = size_t(2) * R;
          uint4 a00, a01, b00, b01, a10, a11, b10, b11;
          auto load = [&](uint4& x0, uint4& x1, uint4& y0, uint4& y1) {
            x0 = __ldg(Ya); x1 = __ldg(Ya + R);
            if (has_b) {
              y0 = __ldg(Yb); y1 = __ldg(Yb + R);
            }
            Ya += R2;
            Yb += R2;
          };
          auto stage = [&](uint4 x0, uint4 x1, uint4 y0, uint4 y1) {
            long long tl_a = tl_clock();
            mbar_wait_a(empty_s + 8 * st, ph ^ 1);
            tl_w += tl_clock() - tl_a;
            fence_after();  // the MMAs that read this A stage have completed
            if (!(dbg_skip(s) & 2)) {
#pragma unroll
              for (int hf = 0; hf < 2; ++hf) {  // A: two 16-column halves (register pressure)
                uint32_t av[16];
                expand_stage_regs(av, x0, x1, hf);
                tmem_st16(tmem_a + st * kAStageCols + 16 * hf, av);
              }
              if (has_b) expand_stage_f4(stage_b + st * kSBStageBytes, y0, y1);
              asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
            }
            fence_before();
            asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
            __syncwarp();
            if (lane == 0) mbar_arrive_a(full_s + 8 * st);
            if (++st == nst) { st = 0; ph ^= 1; }
          };
          if constexpr (kProdDepth == 3) {
          // three register sets: the load of stage q + 3 refills the set stage q used
          uint4 a20, a21, b20, b21;
          if (nsu > 0) load(a00, a01, b00, b01);
          if (nsu > 1) load(a10, a11, b10, b11);
          if (nsu > 2) load(a20, a21, b20, b21);
          for (uint32_t u3 = 0; u3 < nsu; u3 += 3) {
            stage(a00, a01, b00, b01);
            if (u3 + 3 < nsu) load(a00, a01, b00, b01);
            if (u3 + 1 < nsu) {
              stage(a10, a11, b10, b11);
              if (u3 + 4 < nsu) load(a10, a11, b10, b11);
            }
            if (u3 + 2 < nsu) {
              stage(a20, a21, b20, b21);
              if (u3 + 5 < nsu) load(a20, a21, b20, b21);
            }
          }
          } else {
          if (nsu > 0) load(a00, a01, b00, b01);
          if (nsu > 1) load(a10, a11, b10, b11);
          for (uint32_t u2 = 0; u2 < nsu; u2 += 2) {
            stage(a00, a01, b00, b01);
            if (u2 + 2 < nsu) load(a00, a01, b00, b01);
            if (u2 + 1 < nsu) {
              stage(a10, a11, b10, b11);
              if (u2 + 3 < nsu) load(a10, a11, b10, b11);
            }
          }
          }
        }
        wk.next(s);
      }
      if (E3_TIMELINE && blockIdx.x < 3 && lane == 0)
        printf("TL cta %d producer warp %d: total %lld wait_empty %lld\n", blockIdx.x, warp,
               tl_clock() - tl_t0, tl_w);
    }
  } else if (warp == kMmaWarp + 1) {
    // ===================== Y loader (staging ring, one thread) =====================
    if (!kPair && s.ny > 0 && lane == 0 && it0 < it1) {
      SWalker wk;
      wk.start(s, it0);
      uint32_t ys = 0, yph = 0;
      const uint32_t ring = smem_u32(yring);
      const uint32_t yfull_s = smem_u32(yfull_bar), yempty_s = smem_u32(yempty_bar);
      for (uint64_t it = it0; it < it1; ++it) {
        const IInfo inf = s.info[wk.ii];
        const uint32_t R = inf.R;
#pragma unroll 1
        for (uint32_t a = 0; a < 2; ++a) {
          // rows [128 jb, +128) and [128 kb, +128) of quads 2u, 2u + 1 (rows past
          // R are garbage of the next quad: they only feed invalid triples)
          const uint4* pa = s.Y + inf.y_off[a] + size_t(wk.jb) * 2 * kJB;
          const uint4* pb = s.Y + inf.y_off[a] + size_t(wk.kb) * 2 * kJB;
          const uint32_t nsu = (inf.q[a][0] + inf.q[a][1]) / 2;
          for (uint32_t u = 0; u < nsu; ++u) {
            mbar_wait_a(yempty_s + 8 * ys, yph ^ 1);
            const uint32_t bar = yfull_s + 8 * ys, dst = ring + ys * kYSlotBytes;
            asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar),
                         "r"(uint32_t(kYSlotBytes)) : "memory");
            const uint4* src[4] = {pa, pa + R, pb, pb + R};
#pragma unroll
            for (int x = 0; x < 4; ++x)
              asm volatile(
                  "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                  ::"r"(dst + x * 2048), "l"(src[x]), "r"(2048u), "r"(bar) : "memory");
            pa += size_t(2) * R;
            pb += size_t(2) * R;
            if (++ys == s.ny) { ys = 0; yph ^= 1; }
          }
        }
        wk.next(s);
      }
    }
    __syncwarp();
  } else if (warp < kMmaWarp) {
    asm volatile("setmaxnreg.inc.sync.aligned.u32 %0;" ::"n"(kRegEpilogue));
    // ===================== epilogue =====================
    const int ew = warp - kEpiWarp0;            // 0..7
    const int half = ew >> 2;                   // k columns [32*half, 32*half+32)
    const int quarter = warp & 3;               // TMEM lane quarter
    const int et = ew * 32 + lane;              // 0..255 scratch slot
    uint64_t* ls = lists + size_t(ew) * 2 * K;
    uint64_t* lt = ls + K;
    const size_t list = size_t(blockIdx.x) * kEpilogueWarps + ew;
    uint32_t nlist = s.counts[list];
    for (uint32_t e = lane; e < nlist; e += 32) {
      const ulonglong2 v = s.lists[list * K + e];
      ls[e] = v.x;
      lt[e] = v.y;
    }
    __syncwarp();
    uint64_t lastS = ~0ull, lastT = ~0ull;  // the list's last key once full (offer_cached)
    if (nlist == K) {
      lastS = ls[K - 1];
      lastT = lt[K - 1];
    }
    const int jl = quarter * 16 + (lane >> 1);  // row = 2*j_local + b
    const int bsel = lane & 1;
    uint32_t* scr = kSS ? sscr + et : s.scratch + size_t(blockIdx.x) * kScratchPerThread * 256 + et;
    // narrow scratch word x of this thread (x-major, thread-minor): explicit
    // shared-memory accesses when it lives there (no generic LD/ST)
    uint32_t scr_s = kSS ? smem_u32(sscr + et) : 0u;
    // opaque to the compiler: otherwise it rematerialises the aligned
    // dynamic-shared-memory base (≈15 uniform instructions) every round
    asm volatile("" : "+r"(scr_s));
    auto scr_st = [&](uint32_t x, uint32_t v) {
      if constexpr (kSS) sts_u32(scr_s + x * 1024u, v);
      else scr[x * 256] = v;
    };
    auto scr_ld = [&](uint32_t x) -> uint32_t {
      if constexpr (kSS) return lds_u32(scr_s + x * 1024u);
      else return scr[x * 256];
    };
    uint64_t nevals = 0;
    long long tl_t0 = tl_clock(), tl_w[2] = {0, 0}, tl_dr = 0, tl_rd = 0;
    uint32_t kst_s = smem_u32(kstage + ew * kKStageBytes);
    asm volatile("" : "+r"(kst_s));
    // next tile's pair(i, k) / single(k) for k = this warp's 32 k, lane = k
    uint4 npik = make_uint4(0, 0, 0, 0);
    uint2 nskp = make_uint2(0, 0);
    auto load_k = [&](const SWalker& w) {
      const uint32_t i_ = s.i_lo + w.ii;
      const uint32_t k_ = min(i_ + 1 + w.kb * kJB + 32 * half + lane, M - 1);
      npik = __ldg(d.pairp + size_t(i_) * M + k_);
      nskp = __ldg(d.singlep + k_);
    };
    if (it0 < it1) {
      SWalker wk;
      wk.start(s, it0);
      uint32_t u = 0;
      if constexpr (kNarrow) load_k(wk);
      for (uint64_t it = it0; it < it1; ++it) {
        const IInfo inf = s.info[wk.ii];
        if constexpr (kNarrow) {
          __syncwarp();  // the previous tile's rounds are done with the staging
          asm volatile("st.shared.v4.u32 [%0], {%1, %2, %3, %4};" ::"r"(kst_s + lane * 16), "r"(npik.x),
                       "r"(npik.y), "r"(npik.z), "r"(npik.w) : "memory");
          asm volatile("st.shared.v2.u32 [%0], {%1, %2};" ::"r"(kst_s + 512 + lane * 8), "r"(nskp.x),
                       "r"(nskp.y) : "memory");
          __syncwarp();
          if (it + 1 < it1) {
            SWalker nw = wk;
            nw.next(s);
            load_k(nw);
          }
        }
        const uint32_t i = s.i_lo + wk.ii;
        const uint32_t j = i + 1 + (kPair ? 2 * wk.jb + crank : wk.jb) * kJB + jl;
        const uint32_t jc = min(j, M - 1);
        const uint32_t kbase = i + 1 + wk.kb * kJB + 4 * half * kRounds + 2 * bsel;
        // narrow: the tile's marginals and round 0's pair(j,k) entries are
        // requested before the drain waits for the MMAs (DRAM latency hidden)
        uint4 pij = make_uint4(0, 0, 0, 0), pjn[2];
        uint2 sip = make_uint2(0, 0), sjp = make_uint2(0, 0);
        auto fetch_pairs = [&](int mm) {
#pragma unroll
          for (int h = 0; h < 2; ++h)
            pjn[h] = __ldg(d.pairp + size_t(min(kbase + 4 * mm + h, M - 1)) * M + jc);
        };
        if constexpr (kNarrow) {
          pij = __ldg(d.pairp + size_t(i) * M + jc);
          sip = __ldg(d.singlep + i);
          sjp = __ldg(d.singlep + jc);
          fetch_pairs(0);
        }
        const long long tl_d0 = tl_clock();
        // ---- drain the four units (a, c) of this tile: TMEM (f32 counts) ->
        // scratch, releasing each ring slot as soon as it is copied, so the MMAs
        // of the next units overlap the scoring below.
        if constexpr (kNarrow) {
          // the two classes of slot a are drained together into class-packed
          // words (a, m, t, g) = class0 | class1 << 16
#pragma unroll kDrainUnroll
          for (uint32_t a = 0; a < 2; ++a, u += 2) {
            const uint32_t s0 = u % kUnits, s1 = (u + 1) % kUnits;
            const long long tl_a = tl_clock();
            mbar_wait_a(tfull_s + 8 * s0, (u / kUnits) & 1);
            mbar_wait_a(tfull_s + 8 * s1, ((u + 1) / kUnits) & 1);
            tl_w[a] += tl_clock() - tl_a;
            fence_after();
            // count c (f32, exact) -> 2^23 + c * 2^kSh by one FFMA (c * 2^kSh < 2^16),
            // then one PRMT joins the low halves of both classes; a class with
            // no samples in this slot has an unwritten accumulator -> constant 0
            const bool e0 = inf.q[a][0] == 0, e1 = inf.q[a][1] == 0;
            const uint64_t scl2 = f2_splat(float(1u << kSh)), k23 = f2_splat(8388608.f);
            const uint32_t tbase = tmem + (uint32_t(quarter * 32) << 16) + half * 8 * kRounds;
            auto drain = [&](auto empty) {
              constexpr bool kEmpty = decltype(empty)::value;
#pragma unroll
              for (int m2 = 0; m2 < kRounds; m2 += 2) {
                uint32_t v0[16], v1[16];
                tmem_ld16(tbase + s0 * 128 + 8 * m2, v0);
                tmem_ld16(tbase + s1 * 128 + 8 * m2, v1);
                tmem_wait_ld();
                uint32_t w0[16], w1[16];  // 2^23 + c * 2^kSh, two counts per FFMA2
#pragma unroll
                for (int x = 0; x < 16; x += 2) {
                  const uint64_t p0 = f2_fma(f2_pack(__uint_as_float(v0[x]), __uint_as_float(v0[x + 1])),
                                             scl2, k23);
                  const uint64_t p1 = f2_fma(f2_pack(__uint_as_float(v1[x]), __uint_as_float(v1[x + 1])),
                                             scl2, k23);
                  w0[x] = uint32_t(p0); w0[x + 1] = uint32_t(p0 >> 32);
                  w1[x] = uint32_t(p1); w1[x + 1] = uint32_t(p1 >> 32);
                }
#pragma unroll
                for (int x = 0; x < 16; ++x) {
                  const int m = m2 + (x >> 3), tg = x & 7;
                  uint32_t b0 = w0[x], b1 = w1[x];
                  if constexpr (kEmpty) {
                    if (e0) b0 = 0x4B000000u;
                    if (e1) b1 = 0x4B000000u;
                  }
                  scr_st(a * kRounds * 8 + m * 8 + tg, __byte_perm(b0, b1, 0x5410));
                }
              }
            };
            // (tile-uniform branch: the selects only for the rare empty slot)
            if (e0 || e1) drain(std::true_type{});
            else drain(std::false_type{});
            fence_before();
            if constexpr (kPair) {  // one arrival per warp (the peer forwards its own)
              __syncwarp();
              if (lane == 0) {
                mbar_arrive_a(tempty_s + 8 * s0);
                mbar_arrive_a(tempty_s + 8 * s1);
              }
            } else {
              mbar_arrive_a(tempty_s + 8 * s0);
              mbar_arrive_a(tempty_s + 8 * s1);
            }
          }
        } else {
#pragma unroll
        for (uint32_t a = 0; a < 2; ++a)
#pragma unroll
          for (uint32_t c = 0; c < 2; ++c, ++u) {
            const uint32_t slot = u % kUnits;
            mbar_wait_sleep(&tfull_bar[slot], (u / kUnits) & 1);
            fence_after();
            const bool nonempty = inf.q[a][c] != 0;
            const uint32_t taddr =
                tmem + (uint32_t(quarter * 32) << 16) + slot * 128 + half * 8 * kRounds;
#pragma unroll
            for (int m2 = 0; m2 < kRounds; m2 += 2) {
              uint32_t v[16];
              tmem_ld16(taddr + 8 * m2, v);
              tmem_wait_ld();
#pragma unroll
              for (int x = 0; x < 16; ++x) {
                const int m = m2 + (x >> 3);
                scr[(a * kRounds * 16 + m * 16 + c * 8 + (x & 7)) * 256] =
                    nonempty ? f32_count(v[x]) : 0u;
              }
            }
            fence_before();
            if constexpr (kPair) {
              __syncwarp();
              if (lane == 0) mbar_arrive_a(tempty_s + 8 * slot);
            } else {
              mbar_arrive_a(tempty_s + 8 * slot);
            }
          }
        }
        const long long tl_d1 = tl_clock();
        tl_dr += tl_d1 - tl_d0;
        const uint64_t gth = *reinterpret_cast<volatile uint64_t*>(s.gthr);
        // screening bound: a triple whose fp32 screen exceeds thr_f cannot reach
        // the threshold (margin proven on the host, k2_screen_margin)
        const float thr_f = gth == ~0ull ? __int_as_float(0x7f800000)
                                         : __double2float_ru(key_score(gth) + (kMode == 3 ? d.kshift_st
                                                                                                        : d.kshift));
        uint64_t rank_ij = 0;
        if (kRanged) {
          const uint64_t Mi = M - i, Mj = M - jc;
          rank_ij = (uint64_t(M) * (M - 1) * (M - 2) - Mi * (Mi - 1) * (Mi - 2)) / 6 +
                    (uint64_t(Mi - 1) * (Mi - 2)) / 2 - Mj * (Mj - 1) / 2;
        }
        if constexpr (kNarrow) {
          // class-packed words (class0 | class1 << 16) throughout
          // per-half masks of the dropped phase (slots hold the other two, ascending)
          const uint32_t mk0 = (inf.drop[0] == 0 ? 0xffffu : 0u) | (inf.drop[1] == 0 ? 0xffff0000u : 0u);
          const uint32_t mk1 = (inf.drop[0] == 1 ? 0xffffu : 0u) | (inf.drop[1] == 1 ? 0xffff0000u : 0u);
          const uint32_t mk2 = ~(mk0 | mk1);
          // the next round's pair(j,k) entries and scratch words are fetched one
          // round ahead (software pipelining across rounds)
#if E3_W_INPLACE
          // W[a][t][g]: this row (j, b=bsel), unit slot a, k phase t, genotype g;
          // the next round's words are loaded into W itself once T is built
          // (they land during the screen; no register copies)
          uint32_t W[2][4][2];
          auto load_w = [&](int mm) {
#pragma unroll
            for (int a = 0; a < 2; ++a)
#pragma unroll
              for (int t = 0; t < 4; ++t)
#pragma unroll
                for (int g = 0; g < 2; ++g)
                  W[a][t][g] = scr_ld(a * kRounds * 8 + mm * 8 + t * 2 + g);
          };
          load_w(0);
#pragma unroll kRoundUnroll
          for (int m = 0; m < kRounds; ++m) {
            // kPjkLate: this round's pair(j,k) rows are pjn itself, the next
            // round's are loaded into it once derive_cells has used them
            // (during the screens) and the rare tail reloads its own copy;
            // otherwise they are copied and the next ones fetched here
            uint4 pjk_copy[2];
            if constexpr (!kPjkLate) {
#pragma unroll
              for (int h = 0; h < 2; ++h) pjk_copy[h] = pjn[h];
              if (m + 1 < kRounds) fetch_pairs(m + 1);
            }
            uint4 (&pjk)[2] = kPjkLate ? pjn : pjk_copy;
            const int mnext = min(m + 1, kRounds - 1);
#else
          uint32_t Wn[2][4][2];
          auto fetch_round = [&](int mm) {
            if (mm > 0) fetch_pairs(mm);
#pragma unroll
            for (int a = 0; a < 2; ++a)
#pragma unroll
              for (int t = 0; t < 4; ++t)
#pragma unroll
                for (int g = 0; g < 2; ++g)
                  Wn[a][t][g] = scr_ld(a * kRounds * 8 + mm * 8 + t * 2 + g);
          };
          fetch_round(0);
#pragma unroll kRoundUnroll
          for (int m = 0; m < kRounds; ++m) {
            uint4 pjk[2];
            // W[a][t][g]: this row (j, b=bsel), unit slot a, k phase t, genotype g
            uint32_t W[2][4][2];
#pragma unroll
            for (int h = 0; h < 2; ++h) pjk[h] = pjn[h];
#pragma unroll
            for (int a = 0; a < 2; ++a)
#pragma unroll
              for (int t = 0; t < 4; ++t)
#pragma unroll
                for (int g = 0; g < 2; ++g) W[a][t][g] = Wn[a][t][g];
            if (m + 1 < kRounds) fetch_round(m + 1);
#endif
            // the partner row (j, b^1) sends its words for this thread's phases 2*bsel + h
            uint32_t rcv[2][2][2];
#pragma unroll
            for (int a = 0; a < 2; ++a)
#pragma unroll
              for (int h = 0; h < 2; ++h)
#pragma unroll
                for (int g = 0; g < 2; ++g)
                  rcv[a][h][g] = __shfl_xor_sync(0xffffffffu, bsel ? W[a][h][g] : W[a][2 + h][g], 1);
            uint32_t kk[2];
            bool valid[2];
#pragma unroll
            for (int h = 0; h < 2; ++h) {
              kk[h] = kbase + 4 * m + h;
              valid[h] = j < kk[h] && kk[h] < M && !(dbg_skip(s) & 1);
              if (kRanged && valid[h]) {
                const uint64_t rr = rank_ij + (kk[h] - j - 1);
                valid[h] = rr >= s.rank_begin && rr < s.rank_end;
              }
            }
            nevals += uint32_t(valid[0]) + uint32_t(valid[1]);
            if (__any_sync(0xffffffffu, valid[0] || valid[1])) {
              uint32_t T[2][8];  // [h][a*4 + b*2 + g], class-packed
              uint4 pik[2];
              uint2 skp[2];
#pragma unroll
              for (int h = 0; h < 2; ++h) {
                // this warp's staged k index 4m + 2 bsel + h (clamped like kk)
                const uint32_t kx = 4 * m + 2 * bsel + h;
                pik[h] = lds_u128(kst_s + kx * 16);
                skp[h] = lds_u64(kst_s + 512 + kx * 8);
                const uint32_t P[4] = {pjk[h].x, pjk[h].y, pjk[h].z, pjk[h].w};
#pragma unroll
                for (int b = 0; b < 2; ++b)
#pragma unroll
                  for (int g = 0; g < 2; ++g) {
                    const uint32_t own0 = bsel ? W[0][2 + h][g] : W[0][h][g];
                    const uint32_t own1 = bsel ? W[1][2 + h][g] : W[1][h][g];
                    const uint32_t s0 = (b == bsel) ? own0 : rcv[0][h][g];
                    const uint32_t s1 = (b == bsel) ? own1 : rcv[1][h][g];
                    // slots -> phases 0 and 1; the dropped phase from the pair index
                    const uint32_t X = P[b * 2 + g] - s0 - s1;
                    T[h][b * 2 + g] = (X & mk0) | (s0 & ~mk0);
                    T[h][4 + b * 2 + g] = (s1 & mk2) | (X & mk1) | (s0 & mk0);
                  }
              }
#if E3_W_INPLACE
              load_w(mnext);
#endif
              bool pass[2];
#pragma unroll
              for (int h = 0; h < 2; ++h) {
                uint32_t n[27];
                derive_cells(T[h], pij, pik[h], pjk[h], sip, sjp, skp[h], d.npk, n);
                if constexpr (kPjkLate)
                  if (m + 1 < kRounds) pjn[h] = __ldg(d.pairp + size_t(min(kbase + 4 * (m + 1) + h, M - 1)) * M + jc);
                if (dbg_skip(s) & 2) {  // profiling: operands not expanded -> keep lookups in range
#pragma unroll
                  for (int c = 0; c < 27; ++c) n[c] &= 0x0ffc0ffcu;
                }
                if (dbg_skip(s) & 16) {  // profiling: screen lookups within 32 entries (no bank conflicts)
#pragma unroll
                  for (int c = 0; c < 27; ++c) n[c] &= 0x007c007cu;
                }
                if (dbg_skip(s) & 4)
                  pass[h] = n[26] == 0x7fffffffu;  // profiling: derivation only
                else
                  pass[h] = valid[h] && (!s.screen || (kSh ? k2_screen_scaled<kMode == 3>(n, ktab_s, d.st_c1)
                                                              : k2_screen_packed(n, ktab_s, d.st_c1)) <= thr_f) &&
                            !(dbg_skip(s) & 18);
              }
              // rare once the threshold has settled: exact K2 + offers out of
              // line (a warp none of whose triples passed offers nothing: its
              // score keys would all be ~0, never inserted or collected)
              if (__any_sync(0xffffffffu, pass[0] || pass[1])) {
                RareIn in;
#pragma unroll
                for (int h = 0; h < 2; ++h) {
#pragma unroll
                  for (int x = 0; x < 8; ++x) in.T[h][x] = T[h][x];
                  in.pik[h] = pik[h];
                  in.pjk[h] = kPjkLate ? __ldg(d.pairp + size_t(min(kk[h], M - 1)) * M + jc) : pjk[h];
                  in.skp[h] = skp[h];
                  in.kk[h] = kk[h];
                  in.pass[h] = pass[h];
                  in.valid[h] = valid[h];
                }
                in.pij = pij;
                in.sip = sip;
                in.sjp = sjp;
                in.i = i;
                in.j = j;
                const RareState r = syrk_rare<kSh>(in, d.logp, d.npk, gth, ls, lt,
                                                   RareState{nlist, lastS, lastT}, K, s.gthr, s.col);
                nlist = r.nlist;
                lastS = r.lastS;
                lastT = r.lastT;
              }
            }
#if E3_W_INPLACE
            else {
              load_w(mnext);
              if constexpr (kPjkLate)
                if (m + 1 < kRounds) fetch_pairs(m + 1);
            }
#endif
          }
        } else {
          const uint4 pij0 = __ldg(d.pair[0] + size_t(i) * M + jc);
          const uint4 pij1 = __ldg(d.pair[1] + size_t(i) * M + jc);
          const uint2 si0 = __ldg(d.single[0] + i), si1 = __ldg(d.single[1] + i);
          const uint2 sj0 = __ldg(d.single[0] + jc), sj1 = __ldg(d.single[1] + jc);
          for (int m = 0; m < kRounds; ++m) {
            // pair(j,k) rows first: their L2 latency overlaps the scratch loads
            // and the lane-pair exchange below
            uint4 pjk[2][2];
  #pragma unroll
            for (int h = 0; h < 2; ++h) {
              const size_t o = size_t(min(kbase + 4 * m + h, M - 1)) * M + jc;
              pjk[h][0] = __ldg(d.pair[0] + o);
              pjk[h][1] = __ldg(d.pair[1] + o);
            }
            uint32_t T[2][2][8];  // [h][class][a*4 + b*2 + g]
            {
            uint32_t v0[8], v1[8], u0[8], u1[8];
  #pragma unroll
            for (int x = 0; x < 8; ++x) {
              u0[x] = scr[(m * 16 + x) * 256];
              u1[x] = scr[(m * 16 + 8 + x) * 256];
              v0[x] = scr[(kRounds * 16 + m * 16 + x) * 256];
              v1[x] = scr[(kRounds * 16 + m * 16 + 8 + x) * 256];
            }
            // This thread holds T_a[b=bsel][g] for k phases t=0..3 (index 2t+g),
            // a=0 in u, a=1 in v. Thread b owns phases 2b, 2b+1; it sends the
            // partner (b^1) its values for the partner's phases.
            uint32_t snd[16], rcv[16];
  #pragma unroll
            for (int x = 0; x < 4; ++x) {
              const int h = x >> 1, g = x & 1;
              const int i_b0 = 2 * (2 + h) + g;  // partner phases when bsel == 0: 2, 3
              const int i_b1 = 2 * h + g;        // partner phases when bsel == 1: 0, 1
              snd[x] = bsel ? u0[i_b1] : u0[i_b0];
              snd[4 + x] = bsel ? u1[i_b1] : u1[i_b0];
              snd[8 + x] = bsel ? v0[i_b1] : v0[i_b0];
              snd[12 + x] = bsel ? v1[i_b1] : v1[i_b0];
            }
  #pragma unroll
            for (int x = 0; x < 16; ++x) rcv[x] = __shfl_xor_sync(0xffffffffu, snd[x], 1);
  #pragma unroll
            for (int h = 0; h < 2; ++h) {
  #pragma unroll
              for (int g = 0; g < 2; ++g) {
                const int o0 = 2 * h + g, o1 = 2 * (2 + h) + g;  // own index for bsel 0 / 1
                const uint32_t own_u0 = bsel ? u0[o1] : u0[o0], own_u1 = bsel ? u1[o1] : u1[o0];
                const uint32_t own_v0 = bsel ? v0[o1] : v0[o0], own_v1 = bsel ? v1[o1] : v1[o0];
                const int px = h * 2 + g;
  #pragma unroll
                for (int bb = 0; bb < 2; ++bb) {
                  const bool mine = bb == bsel;
                  T[h][0][0 * 4 + bb * 2 + g] = mine ? own_u0 : rcv[px];
                  T[h][1][0 * 4 + bb * 2 + g] = mine ? own_u1 : rcv[4 + px];
                  T[h][0][1 * 4 + bb * 2 + g] = mine ? own_v0 : rcv[8 + px];
                  T[h][1][1 * 4 + bb * 2 + g] = mine ? own_v1 : rcv[12 + px];
                }
              }
            }
            }
            uint32_t kk[2];
            bool valid[2];
  #pragma unroll
            for (int h = 0; h < 2; ++h) {
              kk[h] = i + 1 + wk.kb * kJB + 4 * (half * kRounds + m) + 2 * bsel + h;
              valid[h] = j < kk[h] && kk[h] < M && !(dbg_skip(s) & 1);
              if (kRanged && valid[h]) {
                const uint64_t rr = rank_ij + (kk[h] - j - 1);
                valid[h] = rr >= s.rank_begin && rr < s.rank_end;
              }
            }
            nevals += uint32_t(valid[0]) + uint32_t(valid[1]);
            uint64_t sk[2] = {~0ull, ~0ull}, tk[2] = {~0ull, ~0ull};
            if (valid[0] || valid[1]) {
              uint4 pik[2][2];
              uint2 skc[2][2];
  #pragma unroll
              for (int h = 0; h < 2; ++h) {
                const uint32_t kc = min(kk[h], M - 1);
  #pragma unroll
                for (int c = 0; c < 2; ++c) {
                  pik[h][c] = __ldg(d.pair[c] + size_t(i) * M + kc);
                  skc[h][c] = __ldg(d.single[c] + kc);
                }
                // slots -> phases 0 and 1; the dropped phase from the pair index
  #pragma unroll
                for (int c = 0; c < 2; ++c) {
                  const uint32_t P[4] = {pjk[h][c].x, pjk[h][c].y, pjk[h][c].z, pjk[h][c].w};
                  uint32_t* t = T[h][c];
                  if (inf.drop[c] == 1) {
  #pragma unroll
                    for (int x = 0; x < 4; ++x) t[4 + x] = P[x] - t[x] - t[4 + x];
                  } else if (inf.drop[c] == 0) {
  #pragma unroll
                    for (int x = 0; x < 4; ++x) {
                      const uint32_t t1 = t[x];
                      t[x] = P[x] - t[x] - t[4 + x];
                      t[4 + x] = t1;
                    }
                  }
                }
              }
              bool pass[2];
  #pragma unroll
              for (int h = 0; h < 2; ++h) {
                uint32_t n0[27], n1[27];
                derive_cells(T[h][0], pij0, pik[h][0], pjk[h][0], si0, sj0, skc[h][0], d.n[0], n0);
                derive_cells(T[h][1], pij1, pik[h][1], pjk[h][1], si1, sj1, skc[h][1], d.n[1], n1);
                if (dbg_skip(s) & 4)
                  pass[h] = n0[26] == 0x7fffffffu;  // profiling: derivation only
                else
                  pass[h] = valid[h] && (!s.screen || k2_screen(n0, n1, ktab_s) <= thr_f);
              }
  #pragma unroll
              for (int h = 0; h < 2; ++h) {
                if (pass[h]) {  // rare once the threshold has settled: score exactly
                  uint32_t n0[27], n1[27];
                  derive_cells(T[h][0], pij0, pik[h][0], pjk[h][0], si0, sj0, skc[h][0], d.n[0], n0);
                  derive_cells(T[h][1], pij1, pik[h][1], pjk[h][1], si1, sj1, skc[h][1], d.n[1], n1);
                  sk[h] = score_key(k2_device(n0, n1, d.logp));
                  tk[h] = triple_key(i, j, kk[h]);
                }
              }
            }
  #pragma unroll
            for (int h = 0; h < 2; ++h) {
              offer_cached(valid[h], sk[h], tk[h], gth, ls, lt, nlist, K, lane, s.gthr, s.col, lastS, lastT);
            }
          }
        }
        tl_rd += tl_clock() - tl_d1;
        wk.next(s);
      }
    }
    if (E3_TIMELINE && blockIdx.x < 3 && lane == 0)
      printf("TL cta %d epilogue warp %d: total %lld drain %lld (wait a0 %lld a1 %lld) rounds %lld\n",
             blockIdx.x, warp, tl_clock() - tl_t0, tl_dr, tl_w[0], tl_w[1], tl_rd);
    for (uint32_t e = lane; e < nlist; e += 32) s.lists[list * K + e] = make_ulonglong2(ls[e], lt[e]);
    if (lane == 0) s.counts[list] = nlist;
    add_evals(s.evals, nevals);
  }
  fence_before();
  if constexpr (kPair) cluster_sync();  // the leader's last commits reached the peer
  else __syncthreads();
  if (warp == 0) {
    fence_after();
    if constexpr (kPair)
      asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(tmem), "n"(kTmemCols));
    else
      asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "n"(kTmemCols));
  }
}

inline uint64_t tiles_of(uint64_t M, uint64_t i) {
  const uint64_t nb = (M - 1 - i + kJB - 1) / kJB;
  if (!kPair) return nb * (nb + 1) / 2;
  uint64_t t = 0;  // pairs of j blocks: (nb - 2 p) k blocks each
  for (uint64_t p = 0; p < n_jb(uint32_t(nb)); ++p) t += nb - 2 * p;
  return t;
}

}  // namespace syrk
