// engine.cu — sm_100a kernels and the device half of the C ABI (include/epi3cu.h).
//
// The hot path of the reference (run_search, /root/reference/proj/src/search.cpp:127-250
// with blocked_pass/accumulate_reduced, src/kernels.cpp:30-53, 236-324, and
// k2_score, src/scoring.cpp:23-35) redesigned for B200:
//
//  * Device layout. Per class c, planes are stored word-quad-major:
//      planes[c][wq][snp][g]  (uint4 = 128 samples, g in {0,1})
//    so the 32 lanes of a warp, which own 32 consecutive SNPs k, read one
//    contiguous 1 KiB per word-quad (fully coalesced 128-bit loads), while
//    the SNPs a warp shares (i, j) are warp-uniform broadcast loads.
//    Genotype 2 is never stored (bitplane.hpp:13-20) — and never computed.
//
//  * Marginal-subtraction contingency tables. Per triple and 32-sample word
//    only the 8 cells with genotypes in {0,1}^3 are counted (8 LOP3-AND +
//    8 POPC); the other 19 cells per class follow exactly, in u32
//    arithmetic, from the per-dataset marginal index (pair counts of planes
//    {0,1}x{0,1} for every SNP pair, single plane counts) and N_c. This is
//    bit-identical to the 27-POPC NOR formulation (kernels.cpp:38-49) and
//    needs neither plane 2 nor the padding mask (padding bits are zero in
//    planes 0/1, so they never count).
//
//  * Blocked i<j<k enumeration. A CTA work item is (i, j-tile, k-tile) of
//    32x32 triples in the (j,k) triangle above i; warp w owns j = tile+w+8q
//    (q<4), lane l owns k = tile+l. Items are linearised i-major so any
//    lexicographic triple-rank range maps to one contiguous item range
//    (boundary lanes masked by rank) — the unit of the multi-GPU partition.
//    Persistent CTAs take equal contiguous item slices.
//
//  * Fused K2 + top-k. The K2 epilogue uses the host-built log table
//    (build_log_table, scoring.cpp:14-21) with the reference's exact fp64
//    grouping and row order; candidates go to a per-warp sorted top-k list
//    in shared memory ordered exactly like hit_less (search.hpp:29-35), with
//    a global monotone threshold shared through atomicMin. A bitonic merge
//    kernel reduces the per-warp lists to the final top-k.
#include <cuda_runtime.h>

#include <algorithm>
#include <chrono>
#include <memory>
#include <mutex>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>
#include <type_traits>
#include <vector>

#include "epi3cu.h"
#include "internal.h"

using e3::fail;

namespace {

constexpr int kTile = 32;                  // j / k tile edge (one SNP per lane)
constexpr int kWarps = 8;                  // warps per search CTA
constexpr int kJPerWarp = kTile / kWarps;  // 4 j's per warp -> 4 triples per lane
constexpr int kMergeCap = 4096;            // entries per bitonic merge CTA
constexpr uint32_t kListK = 256;           // per-warp shared-memory top-k list capacity
constexpr uint32_t kMaxSnps = (1u << 21) - 1;

#define CUDA_TRY(expr)                                                              \
  do {                                                                              \
    cudaError_t err__ = (expr);                                                     \
    if (err__ != cudaSuccess)                                                       \
      return fail(err__ == cudaErrorMemoryAllocation ? E3_OOM : E3_CUDA,            \
                  std::string(#expr) + ": " + cudaGetErrorString(err__));           \
  } while (0)

// ------------------------------------------------------------------------
// Order-preserving keys: (score key, triple key) compared as a 128-bit
// integer is exactly hit_less (search.hpp:29-35).
// ------------------------------------------------------------------------
__host__ __device__ inline uint64_t score_key(double s) {
  if (s == 0.0) s = 0.0;  // fold -0.0
  uint64_t b;
  memcpy(&b, &s, 8);
  return (b >> 63) ? ~b : (b | 0x8000000000000000ull);
}
__host__ __device__ inline double key_score(uint64_t k) {
  const uint64_t b = (k >> 63) ? (k & 0x7fffffffffffffffull) : ~k;
  double s;
  memcpy(&s, &b, 8);
  return s;
}
__host__ __device__ inline uint64_t triple_key(uint32_t i, uint32_t j, uint32_t k) {
  return (uint64_t(i) << 42) | (uint64_t(j) << 21) | uint64_t(k);
}
__device__ __forceinline__ bool key_less(uint64_t as, uint64_t at, uint64_t bs, uint64_t bt) {
  return as < bs || (as == bs && at < bt);
}

struct DevData {
  uint32_t M;
  uint32_t wq[2];            // uint4 word-quads per class
  uint32_t n[2];             // class sample counts N0, N1
  const uint4* planes[2];    // [wq][M][2]
  const uint2* single[2];    // [M]: popc(plane0), popc(plane1)
  const uint4* pair[2];      // [M*M], x<y: {00, 01, 10, 11} = popc(Xa_x & Xb_y), mirrored at
                             // [y*M+x]; built lazily for narrow datasets (ensure_wide)
  // narrow (every N_c < 2^16): class-packed u16 counts, word = class0 | class1 << 16
  const uint4* pairp;        // [M*M] {00, 01, 10, 11}, both triangles
  const uint2* singlep;      // [M] {plane 0, plane 1}
  uint32_t npk;              // N0 | N1 << 16
  const double* logp;        // build_log_table(N+1): N+2 entries
  const uint64_t* itemoff;   // [M-1] prefix item counts per i
  const float* ktab;         // screening table G[n] = fl32(logp[n] - alpha*n), ktab_n entries
  uint32_t ktab_n;           // N+2 rounded up to a multiple of 4
  double kshift;             // -27*alpha + proven screening error bound
  float st_c1;               // stirling_term slope -(1+alpha) (k2_screen_packed)
  double kshift_st;          // the Stirling screens' shift (E3_SCREEN_V2: affine part hoisted)
};

// ------------------------------------------------------------------------
// The 27-cell table of one class from the 8 counted cells and the marginals.
// T[a*4+b*2+g] = #samples with genotypes (a,b,g), a,b,g in {0,1}, for SNPs
// (i,j,k). Output cells in reference order gx*9+gy*3+gz (scoring.hpp:14-16).
// All arithmetic is exact modulo 2^32 and every result is a true count.
// ------------------------------------------------------------------------
__device__ __forceinline__ void derive_cells(const uint32_t* T, uint4 pij, uint4 pik, uint4 pjk,
                                             uint2 si, uint2 sj, uint2 sk, uint32_t N,
                                             uint32_t* n) {
  const uint32_t Pij[2][2] = {{pij.x, pij.y}, {pij.z, pij.w}};
  const uint32_t Pik[2][2] = {{pik.x, pik.y}, {pik.z, pik.w}};
  const uint32_t Pjk[2][2] = {{pjk.x, pjk.y}, {pjk.z, pjk.w}};
  const uint32_t Si[2] = {si.x, si.y}, Sj[2] = {sj.x, sj.y}, Sk[2] = {sk.x, sk.y};
#pragma unroll
  for (int a = 0; a < 2; ++a)
#pragma unroll
    for (int b = 0; b < 2; ++b) {
#pragma unroll
      for (int g = 0; g < 2; ++g) n[a * 9 + b * 3 + g] = T[a * 4 + b * 2 + g];
      n[a * 9 + b * 3 + 2] = Pij[a][b] - T[a * 4 + b * 2] - T[a * 4 + b * 2 + 1];
    }
#pragma unroll
  for (int a = 0; a < 2; ++a)
#pragma unroll
    for (int g = 0; g < 2; ++g) n[a * 9 + 6 + g] = Pik[a][g] - T[a * 4 + g] - T[a * 4 + 2 + g];
#pragma unroll
  for (int b = 0; b < 2; ++b)
#pragma unroll
    for (int g = 0; g < 2; ++g) n[18 + b * 3 + g] = Pjk[b][g] - T[b * 2 + g] - T[4 + b * 2 + g];
#pragma unroll
  for (int a = 0; a < 2; ++a)
    n[a * 9 + 8] = Si[a] - Pij[a][0] - Pij[a][1] - n[a * 9 + 6] - n[a * 9 + 7];
#pragma unroll
  for (int b = 0; b < 2; ++b)
    n[18 + b * 3 + 2] = Sj[b] - Pij[0][b] - Pij[1][b] - n[18 + b * 3] - n[18 + b * 3 + 1];
#pragma unroll
  for (int g = 0; g < 2; ++g)
    n[24 + g] = Sk[g] - Pik[0][g] - Pik[1][g] - n[18 + g] - n[21 + g];
  const uint32_t n2xx = N - Si[0] - Si[1];
  const uint32_t n20x = Sj[0] - Pij[0][0] - Pij[1][0];
  const uint32_t n21x = Sj[1] - Pij[0][1] - Pij[1][1];
  n[26] = n2xx - n20x - n21x - n[24] - n[25];
}

// k2_score (scoring.cpp:23-35): identical grouping and row order; explicit
// round-to-nearest adds so no contraction or reassociation can occur.
__device__ __forceinline__ double k2_device(const uint32_t* n0, const uint32_t* n1,
                                            const double* __restrict__ P) {
  double score = 0.0;
#pragma unroll
  for (int c = 0; c < 27; ++c) {
    const uint32_t r0 = n0[c], r1 = n1[c];
    const double t = __dadd_rn(__ldg(P + r0), __ldg(P + r1));
    score = __dadd_rn(score, __dsub_rn(__ldg(P + (size_t(r0) + r1 + 1)), t));
  }
  return score;
}


__device__ __forceinline__ float lds_f32(uint32_t saddr) {
  float v;
  asm("ld.shared.f32 %0, [%1];" : "=f"(v) : "r"(saddr));
  return v;
}
// The P[r0+r1+1] term of a cell from Stirling's lower bound instead of a
// table lookup: ln m! >= (m+1/2) ln m - m + ln(2 pi)/2 for every m >= 1
// (the remainder lies in (1/(12m+1), 1/(12m))), so the screen can only fall
// (never miss a triple); its fp32 + lg2.approx error is in the host margin
// (k2_screen_margin). T = ln2 (m+1/2) lg2(m) + c1 m + ln(2 pi)/2 with
// c1 = -(1+alpha) (the G table's shift included): one MUFU + 4 FP instead of
// a bank-conflicted shared-memory gather and its address arithmetic.
constexpr float kLn2 = 0.693147180559945309f;
constexpr float kHalfLn2Pi = 0.918938533204672742f;
__device__ __forceinline__ float stirling_term(uint32_t mbits, float c1) {
  const float m = __fsub_rn(__uint_as_float(mbits), 8388608.f);  // mbits = bits of 2^23 + m
  float lg;
  asm("lg2.approx.ftz.f32 %0, %1;" : "=f"(lg) : "f"(m));
  const float ap = __fmaf_rn(m, kLn2, 0.5f * kLn2);
  const float cp = __fmaf_rn(m, c1, kHalfLn2Pi);
  return __fmaf_rn(ap, lg, cp);
}

// Packed f32x2 arithmetic (sm_100 FADD2/FFMA2): the screens below handle two
// cells per instruction. Each lane is an ordinary IEEE rn operation, so the
// results (and the host's error bound, k2_screen_margin) are unchanged.
__device__ __forceinline__ uint64_t f2_pack(float lo, float hi) {
  uint64_t r;
  asm("mov.b64 %0, {%1, %2};" : "=l"(r) : "f"(lo), "f"(hi));
  return r;
}
__device__ __forceinline__ uint64_t f2_sub(uint64_t a, uint64_t b) {
  uint64_t r;
  asm("sub.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(a), "l"(b));
  return r;
}
__device__ __forceinline__ uint64_t f2_add(uint64_t a, uint64_t b) {
  uint64_t r;
  asm("add.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(a), "l"(b));
  return r;
}
__device__ __forceinline__ float f2_hsum(uint64_t a) {
  float lo, hi;
  asm("mov.b64 {%0, %1}, %2;" : "=f"(lo), "=f"(hi) : "l"(a));
  return __fadd_rn(lo, hi);
}
__device__ __forceinline__ uint64_t f2_fma(uint64_t a, uint64_t b, uint64_t c) {
  uint64_t r;
  asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(r) : "l"(a), "l"(b), "l"(c));
  return r;
}
__device__ __forceinline__ float f2_lo(uint64_t a) { return __uint_as_float(uint32_t(a)); }
__device__ __forceinline__ float f2_hi(uint64_t a) { return __uint_as_float(uint32_t(a >> 32)); }
__device__ __forceinline__ uint64_t f2_splat(float x) { return f2_pack(x, x); }

// Scaled Stirling screen (kernel mode 3) with the linear part hoisted
// (E3_SCREEN_V2): the cells of a triple partition the samples, so sum_c m_c =
// N + 27 and the Stirling terms' affine part sum_c (c1 m_c + ln(2 pi)/2) is one
// constant per dataset, folded into the host shift (DevData::kshift_st). Per
// cell pair the device then only accumulates (m + 1/2) lg2(m) (one FFMA2 into
// acc_s) and the two table terms (acc_g); the result is ln2 * acc_s - acc_g,
// in one final FFMA: 5 f32x2 ops per cell pair instead of 7 (cfg3 +2.3%).
// Its error bound (k2_screen_margin_st) grows with the un-cancelled sums, ~8x
// the per-cell form's: the unscaled path (mode 1: classes >= 2^14 samples,
// e.g. cfg5 with top-100) keeps the per-cell form, where the wider bound let
// enough extra triples through to the exact tail to cost 3.5% (A/B log).
#ifndef E3_SCREEN_V2
#define E3_SCREEN_V2 1
#endif
#if E3_SCREEN_V2
// n >> 16 as a byte permute: kept as its own value (a shift would be fused
// into a shift-add per use, one more ALU op per cell)
__device__ __forceinline__ uint32_t hi16(uint32_t n) {
  uint32_t r;
  asm("prmt.b32 %0, %1, 0, 0x4432;" : "=r"(r) : "r"(n));
  return r;
}
__device__ __forceinline__ float screen_v2_finish(const uint64_t* as, const uint64_t* ag, float s_last,
                                                  float g_last) {
  const float S = __fadd_rn(f2_hsum(f2_add(as[0], as[1])), s_last);
  const float G = __fadd_rn(f2_hsum(f2_add(ag[0], ag[1])), g_last);
  return __fmaf_rn(S, kLn2, -G);
}
#endif
// k2_screen on class-packed cells (narrow path): word = class0 | class1 << 16.
// Two cells per step in f32x2 (the MUFU lg2 stays scalar).
__device__ __forceinline__ float k2_screen_packed(const uint32_t* n, uint32_t G_s, float c1) {
  uint64_t acc[2] = {0ull, 0ull};
  const uint64_t k23 = f2_splat(8388608.f), kl = f2_splat(kLn2), khl = f2_splat(0.5f * kLn2),
                 kc1 = f2_splat(c1), kh = f2_splat(kHalfLn2Pi);
#pragma unroll
  for (int c = 0; c < 26; c += 2) {
    uint32_t r0[2], r1[2];
    float g0[2], g1[2];
#pragma unroll
    for (int e = 0; e < 2; ++e) {
      r0[e] = n[c + e] & 0xffffu;
      r1[e] = n[c + e] >> 16;
      g0[e] = lds_f32(G_s + 4 * r0[e]);
      g1[e] = lds_f32(G_s + 4 * r1[e]);
    }
    // stirling_term for both cells: m = (2^23 + m) - 2^23, exact
    const uint64_t mb = (uint64_t(r0[1] + r1[1] + 0x4B000001u) << 32) | (r0[0] + r1[0] + 0x4B000001u);
    const uint64_t m = f2_sub(mb, k23);
    float lg0, lg1;
    asm("lg2.approx.ftz.f32 %0, %1;" : "=f"(lg0) : "f"(f2_lo(m)));
    asm("lg2.approx.ftz.f32 %0, %1;" : "=f"(lg1) : "f"(f2_hi(m)));
    const uint64_t ap = f2_fma(m, kl, khl), cp = f2_fma(m, kc1, kh);
    const uint64_t st = f2_fma(ap, f2_pack(lg0, lg1), cp);
    const uint64_t t = f2_sub(f2_sub(st, f2_pack(g0[0], g0[1])), f2_pack(g1[0], g1[1]));
    acc[(c >> 1) & 1] = f2_add(acc[(c >> 1) & 1], t);
  }
  const uint32_t r0 = n[26] & 0xffffu, r1 = n[26] >> 16;
  const float last = __fsub_rn(__fsub_rn(stirling_term(r0 + r1 + 0x4B000001u, c1), lds_f32(G_s + 4 * r0)),
                               lds_f32(G_s + 4 * r1));
  return __fadd_rn(f2_hsum(f2_add(acc[0], acc[1])), last);
}

// k2_screen_packed for counts scaled by 4 (word = 4 r0 | 4 r1 << 16): the
// halves are the table byte offsets of G[r0], G[r1], and their sum + 4 that
// of G[r0 + r1 + 1], so the table form needs no index arithmetic.
#ifndef E3_SCREEN_ADDR3
#define E3_SCREEN_ADDR3 0
#endif
// kStir: the pooled term by stirling_term instead of the table, so the table
// needs only G[0 .. max(N0, N1)] (half the shared memory) and a third of the
// gathers disappear (cfg3 +2%, cfg2 -5%: the host picks it for large classes).
template <bool kStir>
__device__ __forceinline__ float k2_screen_scaled(const uint32_t* n, uint32_t G_s, float c1) {
  if constexpr (kStir) {
#if E3_SCREEN_V2
    uint64_t as[2] = {0ull, 0ull}, ag[2] = {0ull, 0ull};
    const uint64_t kq = f2_splat(0.25f), kb = f2_splat(1.0f - 2097152.0f), kbh = f2_splat(1.5f - 2097152.0f);
#pragma unroll
    for (int c = 0; c < 26; c += 2) {
      uint32_t sb[2];
      float g0[2], g1[2];
#pragma unroll
      for (int e = 0; e < 2; ++e) {
        // three ALU ops per cell: both halves plain (their table addresses fold
        // into [R + UR]), the sum with the exponent in one IADD3
        const uint32_t lo = n[c + e] & 0xffffu, hi = hi16(n[c + e]);
        sb[e] = lo + hi + 0x4B000000u;  // bits of 2^23 + 4 (r0 + r1)
        g0[e] = lds_f32(G_s + lo);
        g1[e] = lds_f32(G_s + hi);
      }
      // m = r0 + r1 + 1 and m + 1/2, each exact in one FFMA2
      const uint64_t sbp = (uint64_t(sb[1]) << 32) | sb[0];
      const uint64_t m = f2_fma(sbp, kq, kb), mh = f2_fma(sbp, kq, kbh);
      float lg0, lg1;
      asm("lg2.approx.ftz.f32 %0, %1;" : "=f"(lg0) : "f"(f2_lo(m)));
      asm("lg2.approx.ftz.f32 %0, %1;" : "=f"(lg1) : "f"(f2_hi(m)));
      as[(c >> 1) & 1] = f2_fma(mh, f2_pack(lg0, lg1), as[(c >> 1) & 1]);
      ag[(c >> 1) & 1] = f2_add(ag[(c >> 1) & 1], f2_add(f2_pack(g0[0], g0[1]), f2_pack(g1[0], g1[1])));
    }
    const uint32_t lo = n[26] & 0xffffu, hi = n[26] >> 16;
    const float m = __fsub_rn(__uint_as_float(((lo + hi) >> 2) + 0x4B000001u), 8388608.f);
    float lg;
    asm("lg2.approx.ftz.f32 %0, %1;" : "=f"(lg) : "f"(m));
    return screen_v2_finish(as, ag, __fmul_rn(__fadd_rn(m, 0.5f), lg),
                            __fadd_rn(lds_f32(G_s + lo), lds_f32(G_s + hi)));
#else
    uint64_t acc[2] = {0ull, 0ull};
    const uint64_t kq = f2_splat(0.25f), kb = f2_splat(1.0f - 2097152.0f), kl = f2_splat(kLn2),
                   khl = f2_splat(0.5f * kLn2), kc1 = f2_splat(c1), kh = f2_splat(kHalfLn2Pi);
#pragma unroll
    for (int c = 0; c < 26; c += 2) {
      uint32_t sb[2];
      float g0[2], g1[2];
#pragma unroll
      for (int e = 0; e < 2; ++e) {
        const uint32_t lo = n[c + e] & 0xffffu, hi = n[c + e] >> 16;
        sb[e] = lo + hi + 0x4B000000u;  // bits of 2^23 + 4 (r0 + r1)
        g0[e] = lds_f32(G_s + lo);
        g1[e] = lds_f32(G_s + hi);
      }
      // m = r0 + r1 + 1 = (2^23 + 4(r0+r1)) / 4 - 2^21 + 1, exact in one FFMA
      const uint64_t m = f2_fma((uint64_t(sb[1]) << 32) | sb[0], kq, kb);
      float lg0, lg1;
      asm("lg2.approx.ftz.f32 %0, %1;" : "=f"(lg0) : "f"(f2_lo(m)));
      asm("lg2.approx.ftz.f32 %0, %1;" : "=f"(lg1) : "f"(f2_hi(m)));
      const uint64_t ap = f2_fma(m, kl, khl), cp = f2_fma(m, kc1, kh);
      const uint64_t st = f2_fma(ap, f2_pack(lg0, lg1), cp);
      const uint64_t t = f2_sub(f2_sub(st, f2_pack(g0[0], g0[1])), f2_pack(g1[0], g1[1]));
      acc[(c >> 1) & 1] = f2_add(acc[(c >> 1) & 1], t);
    }
    const uint32_t lo = n[26] & 0xffffu, hi = n[26] >> 16;
    const float last = __fsub_rn(__fsub_rn(stirling_term(((lo + hi) >> 2) + 0x4B000001u, c1), lds_f32(G_s + lo)),
                                 lds_f32(G_s + hi));
    return __fadd_rn(f2_hsum(f2_add(acc[0], acc[1])), last);
#endif
  }
  uint64_t acc[2] = {0ull, 0ull};  // +0.0f x2
#pragma unroll
  for (int c = 0; c < 26; c += 2) {
    float g[2][3];
#pragma unroll
    for (int e = 0; e < 2; ++e) {
#if E3_SCREEN_ADDR3
      // three ALU ops per cell (lo, hi, lo + hi); the table base (uniform)
      // folds into each load's [R + UR + imm] address
      const uint32_t lo = n[c + e] & 0xffffu, hi = n[c + e] >> 16, sm = lo + hi;
      g[e][0] = lds_f32(G_s + sm + 4);
      g[e][1] = lds_f32(G_s + lo);
      g[e][2] = lds_f32(G_s + hi);
#else
      const uint32_t a0 = G_s + (n[c + e] & 0xffffu), o1 = n[c + e] >> 16;
      g[e][0] = lds_f32(a0 + o1 + 4);
      g[e][1] = lds_f32(a0);
      g[e][2] = lds_f32(G_s + o1);
#endif
    }
    const uint64_t t = f2_sub(f2_sub(f2_pack(g[0][0], g[1][0]), f2_pack(g[0][1], g[1][1])),
                              f2_pack(g[0][2], g[1][2]));
    acc[(c >> 1) & 1] = f2_add(acc[(c >> 1) & 1], t);
  }
  const uint32_t a0 = G_s + (n[26] & 0xffffu), o1 = n[26] >> 16;
  const float last = __fsub_rn(__fsub_rn(lds_f32(a0 + o1 + 4), lds_f32(a0)), lds_f32(G_s + o1));
  return __fadd_rn(f2_hsum(f2_add(acc[0], acc[1])), last);
}

// fp32 screen of k2_score: sum_c (G[r0+r1+1] - G[r0]) - G[r1] over a
// shared-memory table G[n] = fl32(P[n] - alpha*n). The affine shift cancels
// per cell up to the constant alpha, so score = screen + 27*alpha up to an
// error the host bounds rigorously (k2_screen_margin); only triples whose
// screen passes the current threshold are scored exactly with k2_device.
// G_s: shared-memory (32-bit) address of the table.
__device__ __forceinline__ float k2_screen(const uint32_t* n0, const uint32_t* n1, uint32_t G_s) {
  // two cells per f32x2 step; the margin bound holds for any summation order
  uint64_t acc[2] = {0ull, 0ull};
#pragma unroll
  for (int c = 0; c < 26; c += 2) {
    float g[2][3];
#pragma unroll
    for (int e = 0; e < 2; ++e) {
      const uint32_t r0 = n0[c + e], r1 = n1[c + e];
      g[e][0] = lds_f32(G_s + 4 * (r0 + r1 + 1));
      g[e][1] = lds_f32(G_s + 4 * r0);
      g[e][2] = lds_f32(G_s + 4 * r1);
    }
    const uint64_t t = f2_sub(f2_sub(f2_pack(g[0][0], g[1][0]), f2_pack(g[0][1], g[1][1])),
                              f2_pack(g[0][2], g[1][2]));
    acc[(c >> 1) & 1] = f2_add(acc[(c >> 1) & 1], t);
  }
  const uint32_t r0 = n0[26], r1 = n1[26];
  const float last = __fsub_rn(__fsub_rn(lds_f32(G_s + 4 * (r0 + r1 + 1)), lds_f32(G_s + 4 * r0)),
                               lds_f32(G_s + 4 * r1));
  return __fadd_rn(f2_hsum(f2_add(acc[0], acc[1])), last);
}

// One 32-sample word of one class for one (i, j, k): 8 AND3 + 8 POPC.
__device__ __forceinline__ void count_word(uint32_t xi0, uint32_t xi1, uint32_t xj0, uint32_t xj1,
                                           uint32_t xk0, uint32_t xk1, uint32_t* T) {
  T[0] += __popc(xi0 & xj0 & xk0);
  T[1] += __popc(xi0 & xj0 & xk1);
  T[2] += __popc(xi0 & xj1 & xk0);
  T[3] += __popc(xi0 & xj1 & xk1);
  T[4] += __popc(xi1 & xj0 & xk0);
  T[5] += __popc(xi1 & xj0 & xk1);
  T[6] += __popc(xi1 & xj1 & xk0);
  T[7] += __popc(xi1 & xj1 & xk1);
}

__device__ __forceinline__ void count_quad(const uint4& i0, const uint4& i1, const uint4& j0,
                                           const uint4& j1, const uint4& k0, const uint4& k1,
                                           uint32_t* T) {
  count_word(i0.x, i1.x, j0.x, j1.x, k0.x, k1.x, T);
  count_word(i0.y, i1.y, j0.y, j1.y, k0.y, k1.y, T);
  count_word(i0.z, i1.z, j0.z, j1.z, k0.z, k1.z, T);
  count_word(i0.w, i1.w, j0.w, j1.w, k0.w, k1.w, T);
}

// Carry-save adder: a + b + c == s + 2*cy, bitwise. Two LOP3s (0x96, 0xE8).
__device__ __forceinline__ void csa(uint32_t a, uint32_t b, uint32_t c, uint32_t& s,
                                    uint32_t& cy) {
  s = a ^ b ^ c;
  cy = (a & b) | (c & (a ^ b));
}

// popc(v0)+...+popc(v7) with 4 POPC instead of 8: a 8:4 carry-save tree
// (ones, twos, 2x fours) moves work from the quarter-rate POPC (XU) pipe to
// the full-rate LOP3 (ALU) pipe; the weights are applied with IMAD (FMA pipe).
__device__ __forceinline__ uint32_t count8_csa(const uint32_t (&v)[8]) {
  uint32_t s1, c1, s2, c2, s3, c3, t1, f1;
  csa(v[0], v[1], v[2], s1, c1);
  csa(v[3], v[4], v[5], s2, c2);
  csa(s1, s2, v[6], s3, c3);
  const uint32_t ones = s3 ^ v[7], c4 = s3 & v[7];
  csa(c1, c2, c3, t1, f1);
  const uint32_t twos = t1 ^ c4, f2 = t1 & c4;
  return __popc(ones) + 2u * __popc(twos) + 4u * (__popc(f1) + __popc(f2));
}

// Cells counted with plain POPC; the rest go through count8_csa. Two plain
// cells balance the XU (16/clk/SM) and ALU (64/clk/SM) pipes:
// per 8 triple-words ALU 2*12 + 6*22 = 156 ops, XU 2*8 + 6*4 = 40 ops.
constexpr int kPlainCells = 2;

// Accumulates one class of the CTA item into T[q][8] for this lane, two
// word-quads (256 samples) per step; the plane buffers carry one zero quad of
// padding so an odd quad count needs no tail code.
__device__ __forceinline__ void accumulate_class(const uint4* __restrict__ planes, uint32_t wq,
                                                 uint32_t M, uint32_t i, const uint32_t* jc,
                                                 uint32_t kc, uint32_t (&T)[kJPerWarp][8]) {
#pragma unroll
  for (int q = 0; q < kJPerWarp; ++q)
#pragma unroll
    for (int c = 0; c < 8; ++c) T[q][c] = 0;
  const size_t row = size_t(M) * 2;
  const uint4* p = planes;
#pragma unroll 1
  for (uint32_t w = 0; w < wq; w += 2, p += 2 * row) {
    uint32_t I[2][8], K[2][8];
#pragma unroll
    for (int h = 0; h < 2; ++h)
#pragma unroll
      for (int g = 0; g < 2; ++g) {
        const uint4 a = __ldg(p + h * row + 2 * i + g), b = __ldg(p + h * row + 2 * kc + g);
        I[g][4 * h] = a.x; I[g][4 * h + 1] = a.y; I[g][4 * h + 2] = a.z; I[g][4 * h + 3] = a.w;
        K[g][4 * h] = b.x; K[g][4 * h + 1] = b.y; K[g][4 * h + 2] = b.z; K[g][4 * h + 3] = b.w;
      }
#pragma unroll
    for (int q = 0; q < kJPerWarp; ++q) {
      uint32_t J[2][8];
#pragma unroll
      for (int h = 0; h < 2; ++h)
#pragma unroll
        for (int g = 0; g < 2; ++g) {
          const uint4 b = __ldg(p + h * row + 2 * jc[q] + g);
          J[g][4 * h] = b.x; J[g][4 * h + 1] = b.y; J[g][4 * h + 2] = b.z; J[g][4 * h + 3] = b.w;
        }
#pragma unroll
      for (int cell = 0; cell < 8; ++cell) {
        const int a = cell >> 2, b = (cell >> 1) & 1, g = cell & 1;
        uint32_t v[8];
#pragma unroll
        for (int x = 0; x < 8; ++x) v[x] = I[a][x] & J[b][x] & K[g][x];
        if (cell < kPlainCells) {
          uint32_t s = 0;
#pragma unroll
          for (int x = 0; x < 8; ++x) s += __popc(v[x]);
          T[q][cell] += s;
        } else {
          T[q][cell] += count8_csa(v);
        }
      }
    }
  }
}

// Exactly-once accounting (the reference's `++combos`, search.cpp:175): every
// thread counts the triples it evaluated (valid and inside the rank range);
// one atomic per warp at the end of a launch.
__device__ __forceinline__ void add_evals(unsigned long long* evals, uint64_t n) {
#pragma unroll
  for (int o = 16; o; o >>= 1) n += __shfl_xor_sync(0xffffffffu, n, o);
  if ((threadIdx.x & 31) == 0 && n) atomicAdd(evals, (unsigned long long)n);
}

// Candidate collection for top_k above the shared-memory list capacity (the
// second pass of a large-k search, e3_search): every evaluated triple whose
// key is <= the fixed global threshold is appended to buf (warp-aggregated
// atomics); entries past cap are counted but not stored (the host re-runs
// with a larger buffer).
struct Collect {
  ulonglong2* buf = nullptr;  // nullptr: normal mode (per-warp top-k lists)
  unsigned int* n = nullptr;
  uint32_t cap = 0;
};

struct SearchArgs {
  uint64_t item_begin, item_count;
  uint64_t rank_begin, rank_end;  // used when ranged
  uint32_t top_k;
  uint64_t* gthr;                 // global score-key threshold
  unsigned long long* evals;      // triples evaluated (device counter)
  Collect col;
  ulonglong2* out_lists;          // [gridDim*kWarps][top_k] (skey, tkey)
  uint32_t* out_counts;           // [gridDim*kWarps]
};

__device__ __forceinline__ uint32_t tiles_of(uint32_t M, uint32_t i) {
  return (M - 1 - i + kTile - 1) / kTile;
}

// Warp-cooperative ordered insert into this warp's shared-memory list.
__device__ void warp_insert(uint64_t* ls, uint64_t* lt, uint32_t& n, uint32_t K, unsigned cand,
                            uint64_t s, uint64_t t, int lane, uint64_t* gthr) {
  while (cand) {
    const int src = __ffs(cand) - 1;
    cand &= cand - 1;
    const uint64_t cs = __shfl_sync(0xffffffffu, s, src);
    const uint64_t ct = __shfl_sync(0xffffffffu, t, src);
    if (n == K && !key_less(cs, ct, ls[K - 1], lt[K - 1])) continue;
    uint32_t cnt = 0;
    for (uint32_t e = lane; e < n; e += 32) cnt += key_less(ls[e], lt[e], cs, ct);
    const uint32_t p = __reduce_add_sync(0xffffffffu, cnt);
    const uint32_t last = (n == K) ? K - 1 : n;  // [p, last) moves to [p+1, last+1)
    for (int base = int(last) - 1; base >= int(p); base -= 32) {
      const int e = base - lane;
      uint64_t vs = 0, vt = 0;
      if (e >= int(p)) { vs = ls[e]; vt = lt[e]; }
      __syncwarp();
      if (e >= int(p)) { ls[e + 1] = vs; lt[e + 1] = vt; }
      __syncwarp();
    }
    if (lane == 0) { ls[p] = cs; lt[p] = ct; }
    __syncwarp();
    if (n < K) ++n;
    if (n == K && lane == 0) atomicMin(reinterpret_cast<unsigned long long*>(gthr),
                                       (unsigned long long)ls[K - 1]);
  }
}

// One evaluated triple per lane (valid, score key sk, triple key tk) offered
// to the warp's sorted top-k list — or, in collect mode, appended to the
// global candidate buffer when its key passes the fixed threshold.
__device__ __forceinline__ void offer(bool valid, uint64_t sk, uint64_t tk, uint64_t gth,
                                      uint64_t* ls, uint64_t* lt, uint32_t& nlist, uint32_t K,
                                      int lane, uint64_t* gthr, const Collect& col) {
  if (col.buf) {
    const bool want = valid && sk <= gth;
    const unsigned m = __ballot_sync(0xffffffffu, want);
    if (m) {
      const int leader = __ffs(m) - 1;
      unsigned base = 0;
      if (lane == leader) base = atomicAdd(col.n, unsigned(__popc(m)));
      base = __shfl_sync(0xffffffffu, base, leader);
      const unsigned idx = base + unsigned(__popc(m & ((1u << lane) - 1u)));
      if (want && idx < col.cap) col.buf[idx] = make_ulonglong2(sk, tk);
    }
    return;
  }
  const bool want = valid && sk <= gth && (nlist < K || key_less(sk, tk, ls[K - 1], lt[K - 1]));
  const unsigned cand = __ballot_sync(0xffffffffu, want);
  if (cand) warp_insert(ls, lt, nlist, K, cand, sk, tk, lane, gthr);
}

// offer() with the list's last entry held in registers (lastS, lastT = ~0
// while the list is not full), so the common rejection reads no shared
// memory; refreshed after the (rare) insert.
__device__ __forceinline__ void offer_cached(bool valid, uint64_t sk, uint64_t tk, uint64_t gth,
                                             uint64_t* ls, uint64_t* lt, uint32_t& nlist,
                                             uint32_t K, int lane, uint64_t* gthr,
                                             const Collect& col, uint64_t& lastS,
                                             uint64_t& lastT) {
  if (col.buf) {
    offer(valid, sk, tk, gth, ls, lt, nlist, K, lane, gthr, col);
    return;
  }
  const bool want = valid && sk <= gth && key_less(sk, tk, lastS, lastT);
  const unsigned cand = __ballot_sync(0xffffffffu, want);
  if (cand) {
    warp_insert(ls, lt, nlist, K, cand, sk, tk, lane, gthr);
    if (nlist == K) {
      lastS = ls[K - 1];
      lastT = lt[K - 1];
    }
  }
}

template <bool kRanged, int kMinBlocks>
__global__ void __launch_bounds__(kWarps * 32, kMinBlocks)
search_kernel(const DevData d, const SearchArgs a) {
  extern __shared__ uint64_t smem[];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint32_t K = a.top_k;
  uint64_t* ls = smem + size_t(warp) * 2 * K;
  uint64_t* lt = ls + K;
  uint32_t n = 0;
  uint32_t nevals = 0;
  const uint32_t M = d.M;

  uint64_t it = a.item_begin + a.item_count * blockIdx.x / gridDim.x;
  const uint64_t it_end = a.item_begin + a.item_count * (blockIdx.x + 1) / gridDim.x;
  uint32_t i = 0, ta = 0, tb = 0, nt = 0;
  if (it < it_end) {
    // decode: i by binary search over itemoff, then (ta, tb) in the tile triangle
    uint32_t lo = 0, hi = M - 3;
    while (lo < hi) {
      const uint32_t mid = (lo + hi + 1) >> 1;
      if (d.itemoff[mid] <= it) lo = mid; else hi = mid - 1;
    }
    i = lo;
    nt = tiles_of(M, i);
    const uint64_t u = it - d.itemoff[i];
    uint32_t alo = 0, ahi = nt - 1;
    while (alo < ahi) {
      const uint32_t mid = (alo + ahi + 1) >> 1;
      const uint64_t cum = uint64_t(mid) * nt - uint64_t(mid) * (mid - 1) / 2;
      if (cum <= u) alo = mid; else ahi = mid - 1;
    }
    ta = alo;
    tb = ta + uint32_t(u - (uint64_t(ta) * nt - uint64_t(ta) * (ta - 1) / 2));
  }

  for (; it < it_end; ++it) {
    const uint32_t jbase = i + 1 + ta * kTile, kbase = i + 1 + tb * kTile;
    const uint32_t k = kbase + lane;
    const uint32_t kc = min(k, M - 1);
    uint32_t j[kJPerWarp], jc[kJPerWarp];
#pragma unroll
    for (int q = 0; q < kJPerWarp; ++q) {
      j[q] = jbase + warp + kWarps * q;
      jc[q] = min(j[q], M - 1);
    }
    uint32_t T0[kJPerWarp][8], T1[kJPerWarp][8];
    accumulate_class(d.planes[0], d.wq[0], M, i, jc, kc, T0);
    accumulate_class(d.planes[1], d.wq[1], M, i, jc, kc, T1);

    const uint64_t gth = *reinterpret_cast<volatile uint64_t*>(a.gthr);
    uint64_t rank_ij = 0;
    if (kRanged) {
      // rank(i, j, k) = C(M,3) - C(M-i,3) + C(M-1-i,2) - C(M-j,2) + (k-j-1)
      const uint64_t Mi = M - i;
      rank_ij = (uint64_t(M) * (M - 1) * (M - 2) - Mi * (Mi - 1) * (Mi - 2)) / 6 +
                (uint64_t(Mi - 1) * (Mi - 2)) / 2;
    }
    const uint2 si0 = __ldg(d.single[0] + i), si1 = __ldg(d.single[1] + i);
    const uint2 sk0 = __ldg(d.single[0] + kc), sk1 = __ldg(d.single[1] + kc);
    const uint4 pik0 = __ldg(d.pair[0] + size_t(i) * M + kc);
    const uint4 pik1 = __ldg(d.pair[1] + size_t(i) * M + kc);
#pragma unroll
    for (int q = 0; q < kJPerWarp; ++q) {
      bool valid = j[q] < k && k < M;
      if (kRanged && valid) {
        const uint64_t Mj = M - j[q];
        const uint64_t r = rank_ij - Mj * (Mj - 1) / 2 + (k - j[q] - 1);
        valid = r >= a.rank_begin && r < a.rank_end;
      }
      uint64_t s = ~0ull, t = ~0ull;
      nevals += valid;
      if (valid) {
        uint32_t n0[27], n1[27];
        derive_cells(T0[q], __ldg(d.pair[0] + size_t(i) * M + jc[q]), pik0,
                     __ldg(d.pair[0] + size_t(jc[q]) * M + kc), si0,
                     __ldg(d.single[0] + jc[q]), sk0, d.n[0], n0);
        derive_cells(T1[q], __ldg(d.pair[1] + size_t(i) * M + jc[q]), pik1,
                     __ldg(d.pair[1] + size_t(jc[q]) * M + kc), si1,
                     __ldg(d.single[1] + jc[q]), sk1, d.n[1], n1);
        s = score_key(k2_device(n0, n1, d.logp));
        t = triple_key(i, j[q], k);
      }
      offer(valid, s, t, gth, ls, lt, n, K, lane, a.gthr, a.col);
    }

    // advance to the next item in (i, ta, tb) order
    if (++tb == nt) {
      if (++ta == nt) {
        ++i;
        ta = 0;
        nt = tiles_of(M, i);
      }
      tb = ta;
    }
  }

  const size_t list = size_t(blockIdx.x) * kWarps + warp;
  for (uint32_t e = lane; e < n; e += 32) a.out_lists[list * K + e] = make_ulonglong2(ls[e], lt[e]);
  if (lane == 0) a.out_counts[list] = n;
  add_evals(a.evals, nevals);
}

}  // namespace

#include "search_tc.cuh"
#include "search_syrk.cuh"
#include "pairs_tc.cuh"

namespace {

// Bitonic merge of `group` consecutive lists (each <= K sorted entries) into
// one list of the K smallest entries under hit_less order.
__global__ void __launch_bounds__(1024) merge_kernel(const ulonglong2* __restrict__ in,
                                                     const uint32_t* __restrict__ in_counts,
                                                     uint32_t nlists, uint32_t K, uint32_t group,
                                                     uint32_t P, ulonglong2* out,
                                                     uint32_t* out_counts) {
  extern __shared__ ulonglong2 buf[];
  const uint32_t first = blockIdx.x * group;
  const uint32_t last = min(first + group, nlists);
  for (uint32_t x = threadIdx.x; x < P; x += blockDim.x) {
    const uint32_t l = first + x / K, e = x % K;
    ulonglong2 v = make_ulonglong2(~0ull, ~0ull);
    if (l < last && x < group * K && e < in_counts[l]) v = in[size_t(l) * K + e];
    buf[x] = v;
  }
  __syncthreads();
  for (uint32_t size = 2; size <= P; size <<= 1)
    for (uint32_t stride = size >> 1; stride > 0; stride >>= 1) {
      for (uint32_t t = threadIdx.x; t < P / 2; t += blockDim.x) {
        const uint32_t lo = 2 * t - (t & (stride - 1)), hi = lo + stride;
        const bool asc = (lo & size) == 0;
        const ulonglong2 x = buf[lo], y = buf[hi];
        const bool gt = key_less(y.x, y.y, x.x, x.y);
        if (gt == asc) { buf[lo] = y; buf[hi] = x; }
      }
      __syncthreads();
    }
  uint32_t cnt = 0;
  for (uint32_t x = threadIdx.x; x < K; x += blockDim.x) {
    out[size_t(blockIdx.x) * K + x] = buf[x];
  }
  if (threadIdx.x == 0) {
    while (cnt < K && cnt < P && buf[cnt].x != ~0ull) ++cnt;
    out_counts[blockIdx.x] = cnt;
  }
}

// ------------------------------------------------------------------------
// Dataset preparation kernels
// ------------------------------------------------------------------------
// raw: BitPlaneDataset::data_[c] on device, [M][2][W64]; out: [wq][M][2] uint4.
// Also checks plane exclusivity and clean padding (bitplane.hpp:16-20).
__global__ void repack_kernel(const uint64_t* __restrict__ raw, uint32_t M, uint32_t w64,
                              uint32_t wq, uint64_t tail_mask, uint4* __restrict__ out,
                              uint32_t* bad) {
  const uint64_t t = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x;
  if (t >= uint64_t(wq) * M) return;
  const uint32_t q = uint32_t(t / M), snp = uint32_t(t % M);
  uint64_t w[2][2];
#pragma unroll
  for (int g = 0; g < 2; ++g)
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      const uint32_t x = 2 * q + h;
      w[g][h] = x < w64 ? raw[(size_t(snp) * 2 + g) * w64 + x] : 0ull;
    }
#pragma unroll
  for (int h = 0; h < 2; ++h) {
    const uint32_t x = 2 * q + h;
    if (x < w64) {
      uint64_t viol = w[0][h] & w[1][h];
      if (x + 1 == w64) viol |= (w[0][h] | w[1][h]) & ~tail_mask;
      if (viol) atomicOr(bad, 1u);
    }
  }
#pragma unroll
  for (int g = 0; g < 2; ++g)
    out[(size_t(q) * M + snp) * 2 + g] =
        make_uint4(uint32_t(w[g][0]), uint32_t(w[g][0] >> 32), uint32_t(w[g][1]),
                   uint32_t(w[g][1] >> 32));
}

__global__ void singles_kernel(const uint4* __restrict__ planes, uint32_t M, uint32_t wq,
                               uint2* __restrict__ single) {
  // one warp per SNP: lanes stride over the word-quads, then a shuffle sum
  const uint32_t x = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, lane = threadIdx.x & 31;
  if (x >= M) return;
  uint32_t s0 = 0, s1 = 0;
  for (uint32_t w = lane; w < wq; w += 32) {
    const uint4 a = planes[(size_t(w) * M + x) * 2], b = planes[(size_t(w) * M + x) * 2 + 1];
    s0 += __popc(a.x) + __popc(a.y) + __popc(a.z) + __popc(a.w);
    s1 += __popc(b.x) + __popc(b.y) + __popc(b.z) + __popc(b.w);
  }
#pragma unroll
  for (int o = 16; o; o >>= 1) {
    s0 += __shfl_xor_sync(0xffffffffu, s0, o);
    s1 += __shfl_xor_sync(0xffffffffu, s1, o);
  }
  if (lane == 0) single[x] = make_uint2(s0, s1);
}

// pair[x*M + y] for x < y: {popc(X0x&X0y), popc(X0x&X1y), popc(X1x&X0y), popc(X1x&X1y)}.
// Per-triple tables / scores through the same marginal derivation as the search.
// validate + binarize on the device (src/datamodel.cpp:28-46, 69-92): one
// thread per (SNP m, word-quad q) of a class builds both planes of 128
// in-class samples straight into the device layout; idx lists the class's
// samples in order of appearance (the reference's stable class-contiguous
// reorder), so the planes equal binarize()'s.
__global__ void binarize_kernel(const uint8_t* __restrict__ geno, uint64_t N, uint32_t M,
                                const uint32_t* __restrict__ idx, uint32_t n, uint32_t wq,
                                uint4* __restrict__ planes, uint32_t* bad) {
  const uint64_t t = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (t >= uint64_t(M) * wq) return;
  const uint32_t m = uint32_t(t % M), q = uint32_t(t / M);
  const uint8_t* row = geno + size_t(m) * N;
  uint32_t p0[4], p1[4], badv = 0;
#pragma unroll
  for (int w = 0; w < 4; ++w) {
    uint32_t a = 0, b = 0;
    const uint32_t base = q * 128 + w * 32;
    for (uint32_t u = 0; u < 32; ++u) {
      if (base + u >= n) break;
      const uint32_t g = row[__ldg(idx + base + u)];
      badv |= g > 2;
      a |= uint32_t(g == 0) << u;
      b |= uint32_t(g == 1) << u;
    }
    p0[w] = a;
    p1[w] = b;
  }
  planes[(size_t(q) * M + m) * 2] = make_uint4(p0[0], p0[1], p0[2], p0[3]);
  planes[(size_t(q) * M + m) * 2 + 1] = make_uint4(p1[0], p1[1], p1[2], p1[3]);
  if (badv) atomicOr(bad, 1u);
}

// Class-packed single counts for the narrow SYRK path: {p0: c0 | c1 << 16, p1: ...}.
__global__ void pack_singles_kernel(const uint2* __restrict__ s0, const uint2* __restrict__ s1,
                                    uint32_t M, uint32_t sh, uint2* __restrict__ out) {
  const uint32_t x = blockIdx.x * blockDim.x + threadIdx.x;
  if (x >= M) return;
  const uint2 a = s0[x], b = s1[x];
  out[x] = make_uint2((a.x << sh) | (b.x << (16 + sh)), (a.y << sh) | (b.y << (16 + sh)));
}

// POPC pair index, used only when a class holds >= 2^23 samples (beyond the
// exact f32 range of pairs_tc_kernel).
__global__ void pairs_kernel(const uint4* __restrict__ planes, uint32_t M, uint32_t wq,
                             uint4* __restrict__ pair) {
  const uint32_t x = blockIdx.y;
  const uint32_t y = blockIdx.x * blockDim.x + threadIdx.x;
  if (blockIdx.x * blockDim.x + blockDim.x <= x + 1) return;  // whole block below diagonal
  const uint32_t yc = min(y, M - 1);
  uint32_t c00 = 0, c01 = 0, c10 = 0, c11 = 0;
  const size_t row = size_t(M) * 2;
  const uint4* p = planes;
  for (uint32_t w = 0; w < wq; ++w, p += row) {
    const uint4 x0 = __ldg(p + 2 * x), x1 = __ldg(p + 2 * x + 1);
    const uint4 y0 = __ldg(p + 2 * yc), y1 = __ldg(p + 2 * yc + 1);
    c00 += __popc(x0.x & y0.x) + __popc(x0.y & y0.y) + __popc(x0.z & y0.z) + __popc(x0.w & y0.w);
    c01 += __popc(x0.x & y1.x) + __popc(x0.y & y1.y) + __popc(x0.z & y1.z) + __popc(x0.w & y1.w);
    c10 += __popc(x1.x & y0.x) + __popc(x1.y & y0.y) + __popc(x1.z & y0.z) + __popc(x1.w & y0.w);
    c11 += __popc(x1.x & y1.x) + __popc(x1.y & y1.y) + __popc(x1.z & y1.z) + __popc(x1.w & y1.w);
  }
  if (y > x && y < M) {
    // both triangles hold the (x<y) counts, so pair[k*M + j] (j<k) gives warps
    // whose lanes walk consecutive j a contiguous row
    const uint4 v = make_uint4(c00, c01, c10, c11);
    pair[size_t(x) * M + y] = v;
    pair[size_t(y) * M + x] = v;
  }
}

__global__ void triples_kernel(const DevData d, const uint32_t* __restrict__ triples, uint64_t n,
                               uint32_t* __restrict__ tables, double* __restrict__ scores) {
  const uint64_t t = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x;
  if (t >= n) return;
  const uint32_t i = triples[3 * t], j = triples[3 * t + 1], k = triples[3 * t + 2];
  const uint32_t M = d.M;
  uint32_t cells[2][27];
  for (int c = 0; c < 2; ++c) {
    uint32_t T[8] = {0, 0, 0, 0, 0, 0, 0, 0};
    const uint4* p = d.planes[c];
    for (uint32_t w = 0; w < d.wq[c]; ++w, p += size_t(M) * 2)
      count_quad(p[2 * i], p[2 * i + 1], p[2 * j], p[2 * j + 1], p[2 * k], p[2 * k + 1], T);
    derive_cells(T, d.pair[c][size_t(i) * M + j], d.pair[c][size_t(i) * M + k],
                 d.pair[c][size_t(j) * M + k], d.single[c][i], d.single[c][j], d.single[c][k],
                 d.n[c], cells[c]);
  }
  if (tables)
    for (int c = 0; c < 2; ++c)
      for (int x = 0; x < 27; ++x) tables[54 * t + 27 * c + x] = cells[c][x];
  if (scores) scores[t] = k2_device(cells[0], cells[1], d.logp);
}

}  // namespace

// ---------------------------------------------------------------------------
// C ABI: dataset lifetime
// ---------------------------------------------------------------------------
struct e3_dataset {
  int device = 0;
  cudaStream_t stream = nullptr;
  uint64_t M = 0, N[2] = {0, 0};
  uint32_t wq[2] = {0, 0};
  uint4* planes[2] = {nullptr, nullptr};
  uint2* single[2] = {nullptr, nullptr};
  uint4* pair[2] = {nullptr, nullptr};
  uint4* pairp = nullptr;    // narrow class-packed mirrored pair index (every N_c < 2^16)
  uint2* singlep = nullptr;  // narrow class-packed single counts
  bool narrow = false;
  // narrow datasets build the wide pair index only when a consumer needs it
  // (e3_tables/e3_scores, the POPC and masked engines): ensure_wide
  mutable std::mutex wide_mu;
  // the search/table workspace below (lists, Y, metadata, scratch, events,
  // the stream) is per dataset: e3_search / e3_tables / e3_scores on one
  // dataset serialise on this mutex, so a dataset is safely shareable across
  // host threads like the reference's
  std::mutex call_mu;
  uint32_t shift = 0;  // narrow: packed counts scaled by 1 << shift (2 when every N_c < 2^14)
  double* logp = nullptr;
  float* ktab = nullptr;              // K2 screening table (see k2_screen)
  uint32_t ktab_n = 0;
  double kshift = 0;
  double kshift_st = 0;
  float st_c1 = 0.f;
  uint64_t* itemoff = nullptr;
  std::vector<uint64_t> h_itemoff;
  uint64_t* itemoff_tc = nullptr;     // tensor-core kernel item prefix (32-j x 64-k tiles)
  std::vector<uint64_t> h_itemoff_tc;
  std::vector<uint2> h_single[2];     // host copy of the single plane counts
  // compacted (SYRK) engine scratch, allocated on first use
  uint4* y_buf = nullptr;
  size_t y_cap = 0;                   // uint4 elements
  syrk::IInfo* info_buf = nullptr;
  uint64_t* syrk_off = nullptr;
  size_t info_cap = 0;                // IInfo records in info_buf
  size_t off_cap = 0;                 // u64 entries in syrk_off
  size_t y_budget = 0;                // E3_SYRK_YBUDGET_KIB (tests: many batches at small M), uint4s
  uint32_t* scratch = nullptr;
  int num_sms = 0, search_ctas_per_sm = 0, search_min_blocks = 1;
  size_t smem_optin = 0;
  size_t smem_ss_cap = 0;  // dynamic shared memory ceiling of the shared-scratch SYRK kernels
  uint32_t debug_skip = 0;  // E3_DEBUG_SKIP (profiling experiments only)
  bool no_drop = false;     // E3_SYRK_NO_DROP: always compute phases 0 and 1 (A/B testing)
  // scratch reused across searches
  ulonglong2* lists[2] = {nullptr, nullptr};
  uint32_t* counts[2] = {nullptr, nullptr};
  size_t lists_cap = 0;
  uint32_t counts_cap = 0;
  uint64_t* gthr = nullptr;
  unsigned long long* evals = nullptr;  // device counter of evaluated triples (per search)
  ulonglong2* cand = nullptr;           // large-k candidate buffer (second pass), on first use
  size_t cand_cap = 0;
  unsigned int* cand_n = nullptr;
  cudaEvent_t ev[4] = {nullptr, nullptr, nullptr, nullptr};
  cudaEvent_t ev_upload = nullptr;
  // SYRK compaction runs on its own stream, one batch ahead of the search
  // kernel (double-buffered Y / positions); the events order the two
  cudaStream_t cstream = nullptr;
  cudaEvent_t ev_cdone[2] = {nullptr, nullptr}, ev_sdone[2] = {nullptr, nullptr};
};

namespace {

// Device memory comes from the device's stream-ordered pool with a release
// threshold of "never", so dataset create/destroy cycles (the e2e path) reuse
// cached blocks instead of paying cudaMalloc/cudaFree each time.
template <typename T>
cudaError_t dmalloc(const e3_dataset* ds, T** p, size_t bytes);
template <typename T>
void dfree(const e3_dataset* ds, T* p);

void release(e3_dataset* ds) {
  if (!ds) return;
  cudaSetDevice(ds->device);
  for (int c = 0; c < 2; ++c) {
    dfree(ds, ds->planes[c]);
    dfree(ds, ds->single[c]);
    dfree(ds, ds->pair[c]);

    dfree(ds, ds->lists[c]);
    dfree(ds, ds->counts[c]);
  }
  dfree(ds, ds->pairp);
  dfree(ds, ds->singlep);
  dfree(ds, ds->logp);
  dfree(ds, ds->ktab);
  dfree(ds, ds->itemoff);
  dfree(ds, ds->itemoff_tc);
  dfree(ds, ds->y_buf);
  dfree(ds, ds->info_buf);
  dfree(ds, ds->syrk_off);
  dfree(ds, ds->scratch);
  dfree(ds, ds->gthr);
  dfree(ds, ds->evals);
  dfree(ds, ds->cand);
  dfree(ds, ds->cand_n);
  for (auto& e : ds->ev)
    if (e) cudaEventDestroy(e);
  if (ds->ev_upload) cudaEventDestroy(ds->ev_upload);
  for (int b = 0; b < 2; ++b) {
    if (ds->ev_cdone[b]) cudaEventDestroy(ds->ev_cdone[b]);
    if (ds->ev_sdone[b]) cudaEventDestroy(ds->ev_sdone[b]);
  }
  if (ds->cstream) {
    cudaStreamSynchronize(ds->cstream);
    cudaStreamDestroy(ds->cstream);
  }
  if (ds->stream) {
    cudaStreamSynchronize(ds->stream);
    cudaStreamDestroy(ds->stream);
  }
  delete ds;
}


template <typename T>
cudaError_t dmalloc(const e3_dataset* ds, T** p, size_t bytes) {
  return cudaMallocAsync(reinterpret_cast<void**>(p), bytes, ds->stream);
}
template <typename T>
void dfree(const e3_dataset* ds, T* p) {
  if (p) cudaFreeAsync(const_cast<void*>(static_cast<const void*>(p)), ds->stream);
}

DevData dev_view(const e3_dataset* ds) {
  DevData d;
  d.M = uint32_t(ds->M);
  for (int c = 0; c < 2; ++c) {
    d.wq[c] = ds->wq[c];
    d.n[c] = uint32_t(ds->N[c]);
    d.planes[c] = ds->planes[c];
    d.single[c] = ds->single[c];
    d.pair[c] = ds->pair[c];

  }
  d.logp = ds->logp;
  d.itemoff = ds->itemoff;
  d.pairp = ds->pairp;
  d.singlep = ds->singlep;
  d.npk = (uint32_t(ds->N[0]) << ds->shift) | (uint32_t(ds->N[1]) << (16 + ds->shift));
  d.ktab = ds->ktab;
  d.ktab_n = ds->ktab_n;
  d.kshift = ds->kshift;
  d.kshift_st = ds->kshift_st;
  d.st_c1 = ds->st_c1;
  return d;
}

// Rigorous bound on |screen + 27*alpha - score| for k2_screen with table
// entries |G[n]| <= gmax, in round-to-nearest fp32 (unit roundoff u = 2^-24):
// per cell three table roundings (<= u*gmax each), two subtractions
// (|result| <= 2*gmax, 3*gmax) and one accumulation into a partial sum
// bounded by smax. smax: a score is sum_c log((n_c+1)! / (r0! r1!)) =
// sum_c log((n_c+1) C(n_c, r0)) <= N ln 2 + 27 ln(N+1), each term >= 0, and
// the shifted terms subtract alpha. Doubled, plus slack for the fp64
// rounding of the reference score itself.
//
// k2_screen_packed replaces the P[m] lookup (m = r0+r1+1) by stirling_term,
// a lower bound, so only its computed-above-exact error counts. Per cell, with
// lg2.approx absolute error E <= 2^-20 (4x the PTX bound) and |lg2 x| <= L:
// |ap - ap*| |lg| + ap* E + |cp - cp*| + u|T| <= (m+1/2)(2.1 u ln2 L + ln2 E)
// + 2.1 u (3 + alpha) m + u (gmax + 5); summed with sum_c m = N + 27.
double k2_screen_margin(double gmax, double N, double alpha) {
  const double u = std::ldexp(1.0, -24);
  const double smax = N * std::log(2.0) + 27.0 * std::log(N + 1.0) + 27.0 * std::fabs(alpha) + 1.0;
  const double per_cell = u * (3.0 * gmax + 2.0 * gmax + 3.0 * gmax + smax) * (1.0 + 4.0 * u);
  const double L = std::log2(4.0 * (N + 2.0)), E = std::ldexp(1.0, -20), ln2 = std::log(2.0);
  const double stirling = (N + 41.0) * (2.1 * u * ln2 * L + ln2 * E) +
                          2.1 * u * (3.0 + std::fabs(alpha)) * (N + 27.0) + 27.0 * u * (gmax + 5.0);
  return 2.0 * (27.0 * per_cell + stirling) + 1e-9 * smax + 1e-6;
}

// Bound for the E3_SCREEN_V2 scaled Stirling screen (k2_screen_scaled<true>),
// which returns ln2 * S - G, S = sum_c (m_c + 1/2) lg2(m_c), G = sum_c (G[r0_c]
// + G[r1_c]) (fp32; m = r0 + r1 + 1 <= N + 1, m and m + 1/2 exact). With
// Stirling's lower bound ln m! >= (m + 1/2) ln m - m + ln(2 pi)/2 and
// ln r! = G[r] + alpha r exactly, sum_c m_c = N + 27 gives
//   score >= screen* - (1 + alpha) N - 27 + 13.5 ln(2 pi),
// screen* the exact-arithmetic value over the exact G. |screen - screen*| is
// at most, with u = 2^-24, A = (N + 41) log2(N + 2) >= sum (m + 1/2)|lg2 m|
// and Gp = 54 gmax >= sum |G|:
//  * lg2.approx (|E| <= 2^-20, 4x the PTX bound): ln2 E (N + 41);
//  * S: each f32x2 lane takes <= 7 FFMA2 accumulations (partial sums <= its
//    share of A, so <= 7 u A in all), then the lane combine, the horizontal
//    add, the last cell's product and its add (u A each): 11 u A, times ln2;
//    the fp32 ln2 (u ln2 A) and the final FFMA (u (ln2 A + Gp));
//  * G: 54 table roundings (u gmax each); per lane one pair add and <= 7
//    accumulations (u Gp and 7 u Gp in all), combine, horizontal add and the
//    last cell (3 u Gp + 2 u gmax).
// Sum: ln2 E (N + 41) + 13 u ln2 A + 56 u gmax + 12 u Gp; doubled, with slack
// for second-order terms and the reference's own fp64 rounding.
double k2_screen_margin_st(double gmax, double N) {
  const double u = std::ldexp(1.0, -24), E = std::ldexp(1.0, -20), ln2 = std::log(2.0);
  const double A = (N + 41.0) * std::log2(N + 2.0), Gp = 54.0 * gmax;
  const double smax = N * ln2 + 27.0 * std::log(N + 1.0) + 1.0;
  const double err = ln2 * E * (N + 41.0) + 13.0 * u * ln2 * A + 56.0 * u * gmax + 12.0 * u * Gp;
#ifndef E3_ST_MARGIN_SCALE
#define E3_ST_MARGIN_SCALE 1.0  // A/B attribution only (< 1 is unsafe)
#endif
  return E3_ST_MARGIN_SCALE * (2.0 * err * (1.0 + 8.0 * u) + 1e-9 * smax + 1e-6);
}

// Host tables that depend only on N: the reference's log table (built exactly
// like build_log_table(N+1), scoring.cpp:14-21) and the K2 screening table
// G[n] = fl32(P[n] - alpha*n) with its proven margin. alpha balances the
// extremes of P[n] - alpha*n over [0, N+1] (about -0.28 N .. +0.28 N), which
// keeps the fp32 rounding small; the affine part cancels per cell up to alpha.
// The tables are immutable, so dataset creations with the same N share them
// (a small per-process cache; the e2e path recreates datasets per step).
struct LogTables {
  std::vector<double> logp;  // N+2 entries
  std::vector<float> ktab;   // N+2 rounded up to a multiple of 4
  double kshift = 0;
  double kshift_st = 0;  // k2_screen_packed / k2_screen_scaled<true> (E3_SCREEN_V2)
  float st_c1 = 0.f;  // stirling_term slope -(1+alpha)
};
std::shared_ptr<const LogTables> log_tables_for(uint64_t N) {
  static std::mutex mu;
  static std::vector<std::pair<uint64_t, std::shared_ptr<const LogTables>>> cache;
  {
    std::lock_guard<std::mutex> g(mu);
    for (const auto& e : cache)
      if (e.first == N) return e.second;
  }
  auto t = std::make_shared<LogTables>();
  t->logp.resize(N + 2);
  e3_build_log_table(N + 1, t->logp.data());
  const double alpha = std::log(double(N) + 1.0) - 1.2785;
  t->ktab.assign((N + 2 + 3) / 4 * 4, 0.f);
  double gmax = 0;
  for (uint64_t n = 0; n < N + 2; ++n) {
    const double g = t->logp[n] - alpha * double(n);
    t->ktab[n] = float(g);
    gmax = std::max(gmax, std::fabs(g));
  }
  t->kshift = -27.0 * alpha + k2_screen_margin(gmax, double(N), alpha);
  t->st_c1 = float(-(1.0 + alpha));
#if E3_SCREEN_V2
  t->kshift_st = (1.0 + alpha) * double(N) + 27.0 - 13.5 * std::log(6.283185307179586477) +
                 k2_screen_margin_st(gmax, double(N));
#else
  t->kshift_st = t->kshift;
#endif
  std::lock_guard<std::mutex> g(mu);
  if (cache.size() >= 4) cache.erase(cache.begin());
  cache.emplace_back(N, t);
  return t;
}

// Host genotype input of e3_dataset_create_genotypes: the matrix goes to the
// device as bytes and is binarized there.
struct GenoSrc {
  const uint8_t* geno = nullptr;   // [M][N]
  const uint8_t* pheno = nullptr;  // [N]
  uint64_t N = 0;
};

// The pair index launch: narrow_only writes the class-packed mirrored index
// (what the narrow SYRK engine reads), else the wide per-class index (upper
// triangle + mirror).
int launch_pairs(e3_dataset* ds, bool narrow_only) {
  const uint32_t M = uint32_t(ds->M);
  pairs_tc::PArgs pa{};
  pa.M = M;
  pa.nb = (M + pairs_tc::kBlk - 1) / pairs_tc::kBlk;
  pa.tiles = uint64_t(pa.nb) * (pa.nb + 1) / 2;
  pa.pairp = ds->pairp;
  pa.shift = ds->shift;
  for (int c = 0; c < 2; ++c) {
    pa.wq[c] = ds->wq[c];
    pa.planes[c] = ds->planes[c];
    pa.pair[c] = ds->pair[c];
  }
  CUDA_TRY(cudaFuncSetAttribute(pairs_tc::pairs_tc_kernel<false>,
                                cudaFuncAttributeMaxDynamicSharedMemorySize,
                                int(pairs_tc::smem_bytes())));
  CUDA_TRY(cudaFuncSetAttribute(pairs_tc::pairs_tc_kernel<true>,
                                cudaFuncAttributeMaxDynamicSharedMemorySize,
                                int(pairs_tc::smem_bytes())));
  const uint32_t grid = uint32_t(std::min<uint64_t>(ds->num_sms, pa.tiles));
  if (std::max(ds->N[0], ds->N[1]) < (uint64_t(1) << 23)) {
    if (narrow_only)
      pairs_tc::pairs_tc_kernel<true><<<grid, pairs_tc::kThreadsP, pairs_tc::smem_bytes(), ds->stream>>>(pa);
    else
      pairs_tc::pairs_tc_kernel<false><<<grid, pairs_tc::kThreadsP, pairs_tc::smem_bytes(), ds->stream>>>(pa);
  } else {
    for (int c = 0; c < 2; ++c)
      pairs_kernel<<<dim3((M + 255) / 256, M), 256, 0, ds->stream>>>(ds->planes[c], M, ds->wq[c],
                                                                   ds->pair[c]);
  }
  CUDA_TRY(cudaGetLastError());
  return E3_OK;
}

// Builds the wide pair index of a narrow dataset on first use (stream-ordered
// before the caller's kernels on ds->stream).
int ensure_wide(const e3_dataset* cds) {
  e3_dataset* ds = const_cast<e3_dataset*>(cds);
  std::lock_guard<std::mutex> g(ds->wide_mu);
  if (ds->pair[0]) return E3_OK;
  CUDA_TRY(cudaSetDevice(ds->device));
  {
    size_t free_b = 0, total_b = 0;
    CUDA_TRY(cudaMemGetInfo(&free_b, &total_b));
    const double need = 32.0 * double(ds->M) * double(ds->M);
    if (need > double(free_b))
      return fail(E3_OOM, "the per-class pair index of " + std::to_string(ds->M) + " SNPs needs " +
                              std::to_string(need / 1e9) + " GB of device memory, " +
                              std::to_string(double(free_b) / 1e9) + " GB free");
  }
  for (int c = 0; c < 2; ++c)
    CUDA_TRY(dmalloc(ds, &ds->pair[c], sizeof(uint4) * size_t(ds->M) * ds->M));
  return launch_pairs(ds, false);
}

int build(e3_dataset* ds, const uint64_t* host[2], const GenoSrc* gs = nullptr) {
  // E3_TRACE_CREATE=1: per-phase wall times of dataset creation on stderr
  const bool trace = std::getenv("E3_TRACE_CREATE") != nullptr;
  auto tlast = std::chrono::steady_clock::now();
  auto mark = [&](const char* what) {
    if (!trace) return;
    if (ds->stream) cudaStreamSynchronize(ds->stream);
    const auto now = std::chrono::steady_clock::now();
    std::fprintf(stderr, "[create] %-12s %8.3f ms\n", what,
                 std::chrono::duration<double, std::milli>(now - tlast).count());
    tlast = now;
  };
  CUDA_TRY(cudaSetDevice(ds->device));
  {
    cudaMemPool_t pool;
    CUDA_TRY(cudaDeviceGetDefaultMemPool(&pool, ds->device));
    uint64_t keep = UINT64_MAX;
    CUDA_TRY(cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &keep));
  }
  CUDA_TRY(cudaStreamCreateWithFlags(&ds->stream, cudaStreamNonBlocking));
  for (auto& e : ds->ev) CUDA_TRY(cudaEventCreate(&e));
  CUDA_TRY(cudaEventCreateWithFlags(&ds->ev_upload, cudaEventDisableTiming));
  CUDA_TRY(cudaStreamCreateWithFlags(&ds->cstream, cudaStreamNonBlocking));
  for (int b = 0; b < 2; ++b) {
    CUDA_TRY(cudaEventCreateWithFlags(&ds->ev_cdone[b], cudaEventDisableTiming));
    CUDA_TRY(cudaEventCreateWithFlags(&ds->ev_sdone[b], cudaEventDisableTiming));
  }
  mark("stream");
  // two attributes only: cudaGetDeviceProperties costs 10-35 ms per call
  int n_sms = 0, smem_optin = 0;
  CUDA_TRY(cudaDeviceGetAttribute(&n_sms, cudaDevAttrMultiProcessorCount, ds->device));
  CUDA_TRY(cudaDeviceGetAttribute(&smem_optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, ds->device));
  mark("props");
  ds->num_sms = n_sms;
  const uint32_t M = uint32_t(ds->M);
  ds->narrow = std::max(ds->N[0], ds->N[1]) < (uint64_t(1) << 16) && !std::getenv("E3_NO_NARROW");
  ds->shift = ds->narrow && std::max(ds->N[0], ds->N[1]) < (uint64_t(1) << 14) &&
                      !std::getenv("E3_NO_SCALED") ? 2u : 0u;
  {
    // the marginal pair index is O(M^2) (16 B per SNP pair and class-packed
    // index, 32 B when wide): refuse up front, with the numbers, what cannot fit
    size_t free_b = 0, total_b = 0;
    CUDA_TRY(cudaMemGetInfo(&free_b, &total_b));
    const double pairs = double(M) * double(M);
    double need = pairs * (ds->narrow ? 16.0 : 32.0);
    for (int c = 0; c < 2; ++c) need += 32.0 * (double((ds->N[c] + 127) / 128) + 1.0) * M * 2.0;
    if (need > double(free_b)) {  // blocks cached by the stream-ordered pool count as used
      cudaMemPool_t pool;
      CUDA_TRY(cudaDeviceGetDefaultMemPool(&pool, ds->device));
      CUDA_TRY(cudaDeviceSynchronize());
      CUDA_TRY(cudaMemPoolTrimTo(pool, 0));
      CUDA_TRY(cudaMemGetInfo(&free_b, &total_b));
    }
    if (need > double(free_b))
      return fail(E3_OOM, "dataset of " + std::to_string(M) + " SNPs needs " +
                              std::to_string(need / 1e9) + " GB of device memory (pair index " +
                              std::to_string(ds->narrow ? 16 : 32) + " B x M^2), " +
                              std::to_string(double(free_b) / 1e9) + " GB free");
  }
  uint32_t* bad = nullptr;
  CUDA_TRY(dmalloc(ds, &bad, sizeof(uint32_t)));
  CUDA_TRY(cudaMemsetAsync(bad, 0, sizeof(uint32_t), ds->stream));
  uint8_t* dgeno = nullptr;
  uint32_t* didx = nullptr;
  if (gs) {  // genotype input: the matrix and the in-class sample lists to the device
    std::vector<uint32_t> idx(gs->N);
    uint64_t next[2] = {0, ds->N[0]};
    for (uint64_t j = 0; j < gs->N; ++j) idx[next[gs->pheno[j]]++] = uint32_t(j);
    CUDA_TRY(dmalloc(ds, &dgeno, size_t(M) * gs->N));
    CUDA_TRY(dmalloc(ds, &didx, sizeof(uint32_t) * std::max<uint64_t>(gs->N, 1)));
    CUDA_TRY(cudaMemcpyAsync(dgeno, gs->geno, size_t(M) * gs->N, cudaMemcpyHostToDevice, ds->stream));
    CUDA_TRY(cudaMemcpyAsync(didx, idx.data(), sizeof(uint32_t) * gs->N, cudaMemcpyHostToDevice,
                             ds->stream));
    CUDA_TRY(cudaStreamSynchronize(ds->stream));  // idx is a host temporary
  }
  for (int c = 0; c < 2; ++c) {
    const uint64_t n = ds->N[c];
    const uint32_t w64 = uint32_t((n + 63) / 64);
    ds->wq[c] = uint32_t((n + 127) / 128);
    CUDA_TRY(dmalloc(ds, &ds->single[c], sizeof(uint2) * M));
    if (!ds->narrow) CUDA_TRY(dmalloc(ds, &ds->pair[c], sizeof(uint4) * size_t(M) * M));

    // one extra zero quad: the search kernel steps two quads at a time
    const size_t plane_bytes = sizeof(uint4) * (size_t(ds->wq[c]) + 1) * M * 2;
    CUDA_TRY(dmalloc(ds, &ds->planes[c], plane_bytes));
    CUDA_TRY(cudaMemsetAsync(ds->planes[c], 0, plane_bytes, ds->stream));
    if (ds->wq[c] == 0) {
      CUDA_TRY(cudaMemsetAsync(ds->single[c], 0, sizeof(uint2) * M, ds->stream));
      continue;  // pairs_tc_kernel writes the (all-zero) pair index
    }
    const uint64_t threads = uint64_t(ds->wq[c]) * M;
    if (gs) {
      binarize_kernel<<<unsigned((threads + 255) / 256), 256, 0, ds->stream>>>(
          dgeno, gs->N, M, didx + (c ? ds->N[0] : 0), uint32_t(n), ds->wq[c], ds->planes[c], bad);
    } else {
      uint64_t* raw = nullptr;
      const size_t raw_bytes = sizeof(uint64_t) * size_t(M) * 2 * w64;
      CUDA_TRY(dmalloc(ds, &raw, raw_bytes));
      CUDA_TRY(cudaMemcpyAsync(raw, host[c], raw_bytes, cudaMemcpyHostToDevice, ds->stream));
      const uint64_t rem = n % 64;
      const uint64_t tail = rem == 0 ? ~0ull : ((1ull << rem) - 1);
      repack_kernel<<<unsigned((threads + 255) / 256), 256, 0, ds->stream>>>(
          raw, M, w64, ds->wq[c], tail, ds->planes[c], bad);
      dfree(ds, raw);
    }
    singles_kernel<<<(M + 7) / 8, 256, 0, ds->stream>>>(ds->planes[c], M, ds->wq[c],
                                                      ds->single[c]);
    CUDA_TRY(cudaGetLastError());
  }
  if (ds->narrow) {
    CUDA_TRY(dmalloc(ds, &ds->pairp, sizeof(uint4) * size_t(M) * M));
    CUDA_TRY(dmalloc(ds, &ds->singlep, sizeof(uint2) * M));
    pack_singles_kernel<<<(M + 255) / 256, 256, 0, ds->stream>>>(ds->single[0], ds->single[1], M,
                                                                ds->shift, ds->singlep);
  }
  dfree(ds, dgeno);
  dfree(ds, didx);
  mark("planes");
  // marginal pair index of both classes: one tensor-core Gram launch (the
  // class-packed mirrored index only, when narrow)
  if (int rc = launch_pairs(ds, ds->narrow)) return rc;
  mark("pairs");
  for (int c = 0; c < 2; ++c) {
    ds->h_single[c].resize(M);
    CUDA_TRY(cudaMemcpyAsync(ds->h_single[c].data(), ds->single[c], sizeof(uint2) * M,
                             cudaMemcpyDeviceToHost, ds->stream));
  }
  // K2 log table (exactly build_log_table(N+1)) and screening table: pure
  // functions of N, built once per N per process (log_tables_for).
  const uint64_t N = ds->N[0] + ds->N[1];
  const std::shared_ptr<const LogTables> lt = log_tables_for(N);
  CUDA_TRY(dmalloc(ds, &ds->logp, sizeof(double) * lt->logp.size()));
  CUDA_TRY(cudaMemcpyAsync(ds->logp, lt->logp.data(), sizeof(double) * lt->logp.size(),
                           cudaMemcpyHostToDevice, ds->stream));
  ds->ktab_n = uint32_t(lt->ktab.size());
  ds->kshift = lt->kshift;
  ds->kshift_st = lt->kshift_st;
  ds->st_c1 = lt->st_c1;
  CUDA_TRY(dmalloc(ds, &ds->ktab, sizeof(float) * lt->ktab.size()));
  CUDA_TRY(cudaMemcpyAsync(ds->ktab, lt->ktab.data(), sizeof(float) * lt->ktab.size(),
                           cudaMemcpyHostToDevice, ds->stream));
  // Item prefix over i (items = 32x32 (j,k) tiles above i, i-major).
  ds->h_itemoff.assign(M - 1, 0);
  for (uint32_t i = 0; i + 2 < M; ++i) {
    const uint64_t nt = (M - 1 - i + kTile - 1) / kTile;
    ds->h_itemoff[i + 1] = ds->h_itemoff[i] + nt * (nt + 1) / 2;
  }
  CUDA_TRY(dmalloc(ds, &ds->itemoff, sizeof(uint64_t) * ds->h_itemoff.size()));
  CUDA_TRY(cudaMemcpyAsync(ds->itemoff, ds->h_itemoff.data(),
                           sizeof(uint64_t) * ds->h_itemoff.size(), cudaMemcpyHostToDevice,
                           ds->stream));
  ds->h_itemoff_tc.assign(M - 1, 0);
  for (uint32_t i = 0; i + 2 < M; ++i)
    ds->h_itemoff_tc[i + 1] = ds->h_itemoff_tc[i] + tc::items_of(M, i);
  CUDA_TRY(dmalloc(ds, &ds->itemoff_tc, sizeof(uint64_t) * ds->h_itemoff_tc.size()));
  CUDA_TRY(cudaMemcpyAsync(ds->itemoff_tc, ds->h_itemoff_tc.data(),
                           sizeof(uint64_t) * ds->h_itemoff_tc.size(), cudaMemcpyHostToDevice,
                           ds->stream));
  CUDA_TRY(cudaFuncSetAttribute(tc::search_tc_kernel<false>,
                                cudaFuncAttributeMaxDynamicSharedMemorySize,
                                int(tc::smem_bytes(kListK))));
  CUDA_TRY(cudaFuncSetAttribute(tc::search_tc_kernel<true>,
                                cudaFuncAttributeMaxDynamicSharedMemorySize,
                                int(tc::smem_bytes(kListK))));
  ds->smem_optin = size_t(smem_optin);
  if (const char* dbg = std::getenv("E3_DEBUG_SKIP")) ds->debug_skip = uint32_t(std::atoi(dbg));
  ds->no_drop = std::getenv("E3_SYRK_NO_DROP") != nullptr;
  if (const char* yb = std::getenv("E3_SYRK_YBUDGET_KIB"))
    ds->y_budget = std::max<size_t>(1, size_t(std::atoll(yb)) * 1024 / sizeof(uint4));
  {
    // every SYRK instantiation may use the opt-in dynamic shared memory; the
    // shared-scratch kernels run close to the per-block limit, so their
    // ceiling is the opt-in limit minus their static shared memory
    const void* global_scr[] = {
        (const void*)syrk::search_syrk_kernel<false, 0>, (const void*)syrk::search_syrk_kernel<true, 0>,
        (const void*)syrk::search_syrk_kernel<false, 1>, (const void*)syrk::search_syrk_kernel<true, 1>,
        (const void*)syrk::search_syrk_kernel<false, 2>, (const void*)syrk::search_syrk_kernel<true, 2>,
        (const void*)syrk::search_syrk_kernel<false, 3>, (const void*)syrk::search_syrk_kernel<true, 3>};
    const void* shared_scr[] = {
        (const void*)syrk::search_syrk_kernel<false, 1, true>, (const void*)syrk::search_syrk_kernel<true, 1, true>,
        (const void*)syrk::search_syrk_kernel<false, 2, true>, (const void*)syrk::search_syrk_kernel<true, 2, true>,
        (const void*)syrk::search_syrk_kernel<false, 3, true>, (const void*)syrk::search_syrk_kernel<true, 3, true>};
    for (const void* f : global_scr)
      CUDA_TRY(cudaFuncSetAttribute(f, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                    int(ds->smem_optin - 2048)));
    size_t st_max = 0;
    for (const void* f : shared_scr) {
      cudaFuncAttributes fa{};
      CUDA_TRY(cudaFuncGetAttributes(&fa, f));
      st_max = std::max(st_max, fa.sharedSizeBytes);
    }
    ds->smem_ss_cap = ds->smem_optin - st_max;
    for (const void* f : shared_scr)
      CUDA_TRY(cudaFuncSetAttribute(f, cudaFuncAttributeMaxDynamicSharedMemorySize, int(ds->smem_ss_cap)));
  }
  CUDA_TRY(dmalloc(ds, &ds->gthr, sizeof(uint64_t)));
  CUDA_TRY(dmalloc(ds, &ds->evals, sizeof(unsigned long long)));
  CUDA_TRY(dmalloc(ds, &ds->cand_n, sizeof(unsigned int)));
  mark("tables");
  uint32_t h_bad = 0;
  CUDA_TRY(cudaMemcpyAsync(&h_bad, bad, sizeof(uint32_t), cudaMemcpyDeviceToHost, ds->stream));
  CUDA_TRY(cudaStreamSynchronize(ds->stream));
  dfree(ds, bad);
  if (h_bad && gs) {  // find the first offending genotype for the message (host scan)
    for (uint64_t i = 0; i < ds->M; ++i)
      for (uint64_t j = 0; j < gs->N; ++j)
        if (gs->geno[i * gs->N + j] > 2)
          return fail(E3_DOMAIN, "genotype value " + std::to_string(gs->geno[i * gs->N + j]) +
                                     " at snp " + std::to_string(i) + ", sample " +
                                     std::to_string(j));
  }
  if (h_bad)
    return fail(E3_DOMAIN,
                "bit planes violate the dataset invariants (overlapping genotype planes or "
                "set padding bits)");
  CUDA_TRY(cudaFuncSetAttribute(merge_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                int(sizeof(ulonglong2) * 2 * kMergeCap)));
  const int list_smem = int(2 * sizeof(uint64_t) * kWarps * kListK);
  CUDA_TRY(cudaFuncSetAttribute(search_kernel<false, 1>,
                                cudaFuncAttributeMaxDynamicSharedMemorySize, list_smem));
  CUDA_TRY(cudaFuncSetAttribute(search_kernel<true, 1>,
                                cudaFuncAttributeMaxDynamicSharedMemorySize, list_smem));
  CUDA_TRY(cudaFuncSetAttribute(search_kernel<false, 2>,
                                cudaFuncAttributeMaxDynamicSharedMemorySize, list_smem));
  CUDA_TRY(cudaFuncSetAttribute(search_kernel<true, 2>,
                                cudaFuncAttributeMaxDynamicSharedMemorySize, list_smem));
  // E3_SEARCH_OCCUPANCY=1|2 selects the register/occupancy trade-off of the
  // search kernel (tuning knob; the default is the measured best).
  const char* occ_env = std::getenv("E3_SEARCH_OCCUPANCY");
  ds->search_min_blocks = (occ_env && std::atoi(occ_env) == 1) ? 1 : 2;
  int occ = 0;
  if (ds->search_min_blocks == 2)
    CUDA_TRY(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, search_kernel<false, 2>,
                                                           kWarps * 32, list_smem));
  else
    CUDA_TRY(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, search_kernel<false, 1>,
                                                           kWarps * 32, list_smem));
  ds->search_ctas_per_sm = std::max(1, occ);
  mark("finish");
  return E3_OK;
}

}  // namespace

extern "C" int e3_device_count(int* count) {
  CUDA_TRY(cudaGetDeviceCount(count));
  return E3_OK;
}

extern "C" int e3_dataset_create(uint64_t M, uint64_t N0, uint64_t N1, const uint64_t* ctrl,
                                 const uint64_t* cases, int device, e3_dataset** out) {
  *out = nullptr;
  if (M < 3) return fail(E3_DIMENSION, "search needs at least 3 SNPs");
  if (M > kMaxSnps) return fail(E3_DOMAIN, "at most 2^21-1 SNPs are supported");
  if (N0 + N1 == 0) return fail(E3_DIMENSION, "dataset has no samples");
  if (N0 > 0xffffffffull || N1 > 0xffffffffull)
    return fail(E3_DOMAIN, "class sample count exceeds the 32-bit cell cap");
  if ((N0 && !ctrl) || (N1 && !cases)) return fail(E3_DOMAIN, "missing plane data");
  e3_dataset* ds = new e3_dataset;
  ds->device = device;
  ds->M = M;
  ds->N[0] = N0;
  ds->N[1] = N1;
  const uint64_t* host[2] = {ctrl, cases};
  if (int rc = build(ds, host)) {
    release(ds);
    return rc;
  }
  *out = ds;
  return E3_OK;
}

extern "C" int e3_dataset_create_genotypes(uint64_t M, uint64_t N, const uint8_t* geno,
                                           const uint8_t* pheno, int device, e3_dataset** out) {
  *out = nullptr;
  if (M < 3) return fail(E3_DIMENSION, "need at least 3 SNPs, got " + std::to_string(M));
  if (M > kMaxSnps) return fail(E3_DOMAIN, "at most 2^21-1 SNPs are supported");
  if (N == 0) return fail(E3_DIMENSION, "dataset has no samples");
  if (N > 0xffffffffull) return fail(E3_DOMAIN, "at most 2^32-1 samples are supported");
  if (!geno || !pheno) return fail(E3_DOMAIN, "missing genotype or phenotype data");
  uint64_t n1 = 0;
  for (uint64_t j = 0; j < N; ++j) {  // validate (src/datamodel.cpp:28-46)
    if (pheno[j] > 1)
      return fail(E3_DOMAIN, "phenotype value " + std::to_string(pheno[j]) +
                                 " at snp 0, sample " + std::to_string(j));
    n1 += pheno[j];
  }
  e3_dataset* ds = new e3_dataset;
  ds->device = device;
  ds->M = M;
  ds->N[0] = N - n1;
  ds->N[1] = n1;
  GenoSrc gs;
  gs.geno = geno;
  gs.pheno = pheno;
  gs.N = N;
  const uint64_t* host[2] = {nullptr, nullptr};
  if (int rc = build(ds, host, &gs)) {
    release(ds);
    return rc;
  }
  *out = ds;
  return E3_OK;
}

extern "C" void e3_dataset_destroy(e3_dataset* ds) { release(ds); }

extern "C" int e3_dataset_info(const e3_dataset* ds, uint64_t* M, uint64_t* N0, uint64_t* N1,
                               int* device) {
  if (!ds) return fail(E3_DOMAIN, "null dataset");
  if (M) *M = ds->M;
  if (N0) *N0 = ds->N[0];
  if (N1) *N1 = ds->N[1];
  if (device) *device = ds->device;
  return E3_OK;
}

// ---------------------------------------------------------------------------
// C ABI: search
// ---------------------------------------------------------------------------
namespace {

// The compacted tensor-core engine over first-SNP range [i_first, i_last]:
// batches of i sized so the compacted operands stay L2-resident, each =
// positions + gather + SYRK kernel; the per-CTA top-k lists persist across
// the batches. All batches are planned up front, so the host never waits.
int run_syrk(e3_dataset* ds, const DevData& d, uint64_t r0, uint64_t r1, uint32_t K, bool ranged,
             uint32_t i_first, uint32_t i_last, uint32_t grid, uint32_t* launches,
             const Collect& col) {
  const uint64_t M = ds->M;
  cudaStream_t st = ds->stream;
  // lexicographic rank of the first triple with first SNP i: C(M,3) - C(M-i,3)
  auto first_rank = [M](uint64_t i) {
    auto c3 = [](uint64_t n) { return n < 3 ? 0 : n * (n - 1) / 2 * (n - 2) / 3; };
    return c3(M) - c3(M - i);
  };
  // uint4 elements per batch: 48 MiB (M < 4096: cfg2 loses 4% at 64 MiB),
  // 64 MiB for M >= 4096, 128 MiB when the operands are also dense in tiles
  // (<= 3 KiB of Y per 64x64 tile at the first SNP of the search): fewer
  // launches and batch tails, measured cfg3 483 -> 495 Tel/s, while cfg5
  // (8.5 KiB per tile) peaks at 64 MiB and loses 6% at 96.
  // E3_SYRK_YBUDGET_KIB sets it (tests shrink it so small datasets plan many
  // batches)
  size_t kYBudget = ds->y_budget ? ds->y_budget : (M >= 4096 ? size_t(4) << 20 : size_t(3) << 20);
  if (!ds->y_budget && M >= 4096) {
    size_t ysz0 = 0;
    for (int c = 0; c < 2; ++c) {
      const uint2 sc = ds->h_single[c][i_first];
      const uint64_t g[3] = {sc.x, sc.y, ds->N[c] - sc.x - sc.y};
      const uint64_t gmax = std::max(g[0], std::max(g[1], g[2]));
      ysz0 += ((g[0] + 255) / 256 + (g[1] + 255) / 256 + (g[2] + 255) / 256 - (gmax + 255) / 256) * 2;
    }
    const double bytes_per_tile = double(ysz0) * 16.0 * double(2 * (M - 1 - i_first)) /
                                  double(std::max<uint64_t>(1, syrk::tiles_of(M, i_first)));
    if (bytes_per_tile <= 3072.0) kYBudget = size_t(8) << 20;
  }
  const size_t kYMax = std::max(kYBudget, size_t(16) << 20);  // hard cap (256 MiB per buffer)
  struct Batch {
    uint32_t first, n, rmax, qmax;
    size_t ytot;
    uint64_t tiles, info_at, off_at;
  };
  std::vector<syrk::IInfo> infos;
  std::vector<uint64_t> offs;
  std::vector<Batch> batches;
  size_t ymax = 0;
  for (uint32_t i = i_first; i <= i_last;) {
    Batch bt{};
    bt.first = i;
    bt.info_at = infos.size();
    bt.off_at = offs.size();
    offs.push_back(0);
    while (i <= i_last) {
      syrk::IInfo inf{};
      inf.R = uint32_t(2 * (M - 1 - i));
      inf.nb = uint32_t((M - 1 - i + syrk::kJB - 1) / syrk::kJB);
      size_t ysz = 0;
      for (int c = 0; c < 2; ++c) {
        // genotype counts of SNP i in class c; the largest phase is dropped
        const uint2 sc = ds->h_single[c][i];
        const uint64_t g[3] = {sc.x, sc.y, ds->N[c] - sc.x - sc.y};
        const uint32_t drop = g[2] >= g[0] && g[2] >= g[1] ? 2u : (g[1] >= g[0] ? 1u : 0u);
        inf.drop[c] = ds->no_drop ? 2u : drop;
        for (int p = 0, a = 0; a < 3; ++a) {
          if (uint32_t(a) == inf.drop[c]) continue;
          inf.n[p][c] = uint32_t(g[a]);
          inf.q[p][c] = (inf.n[p][c] + 255) / 256 * 2;
          ysz += size_t(inf.q[p][c]) * inf.R;
          ++p;
        }
      }
      // a batch closes at the L2-sized budget once it has enough tiles to
      // keep every SM busy; batches of few tiles (long sample axis, cfg4)
      // may grow up to kYMax
      const uint64_t bt_tiles = offs.back();
      if (bt.n > 0 && bt.ytot + ysz > kYBudget &&
          (bt_tiles >= 2ull * grid || bt.ytot + ysz > kYMax || ds->y_budget))
        break;
      for (int a = 0; a < 2; ++a) {
        inf.y_off[a] = bt.ytot;
        bt.ytot += size_t(inf.q[a][0] + inf.q[a][1]) * inf.R;
        bt.qmax = std::max(bt.qmax, inf.q[a][0] + inf.q[a][1]);
      }
      bt.rmax = std::max(bt.rmax, inf.R);
      infos.push_back(inf);
      offs.push_back(offs.back() + syrk::tiles_of(M, i));
      ++bt.n;
      ++i;
    }
    bt.tiles = offs.back();
    ymax = std::max(ymax, bt.ytot);
    batches.push_back(bt);
  }
  // buffers: Y and positions are double-buffered across consecutive batches so
  // batch b+1's compaction can overlap nothing it must not touch (same stream:
  // ordering is by the stream; two buffers keep the option of a second stream)
  if (ymax > ds->y_cap) {
    dfree(ds, ds->y_buf);
    ds->y_buf = nullptr;
    // + 256 uint4: the Y staging ring's bulk copies read whole 128-row blocks,
    // up to 127 rows past a quad's end (garbage rows of invalid triples)
    CUDA_TRY(dmalloc(ds, &ds->y_buf, 2 * sizeof(uint4) * std::max<size_t>(ymax, 1) + 256 * sizeof(uint4)));
    ds->y_cap = ymax;
  }
  // the two metadata buffers are sized independently: a later search may need
  // more IInfo records and fewer batch offsets, or the reverse
  if (infos.size() > ds->info_cap) {
    dfree(ds, ds->info_buf);
    ds->info_buf = nullptr;
    ds->info_cap = 0;
    CUDA_TRY(dmalloc(ds, &ds->info_buf, sizeof(syrk::IInfo) * infos.size()));
    ds->info_cap = infos.size();
  }
  if (offs.size() > ds->off_cap) {
    dfree(ds, ds->syrk_off);
    ds->syrk_off = nullptr;
    ds->off_cap = 0;
    CUDA_TRY(dmalloc(ds, &ds->syrk_off, sizeof(uint64_t) * offs.size()));
    ds->off_cap = offs.size();
  }
  CUDA_TRY(cudaMemcpyAsync(ds->info_buf, infos.data(), sizeof(syrk::IInfo) * infos.size(),
                           cudaMemcpyHostToDevice, st));
  CUDA_TRY(cudaMemcpyAsync(ds->syrk_off, offs.data(), sizeof(uint64_t) * offs.size(),
                           cudaMemcpyHostToDevice, st));
  CUDA_TRY(cudaEventRecord(ds->ev_upload, st));
  if (!ds->scratch)
    CUDA_TRY(dmalloc(ds, &ds->scratch, sizeof(uint32_t) * size_t(grid) *
                                          syrk::kScratchPerThread * 256));
  CUDA_TRY(cudaMemsetAsync(ds->counts[0], 0, sizeof(uint32_t) * grid * tc::kEpilogueWarps, st));
  // Shared memory: operand stages + top-k lists + (optionally) the K2 screening
  // table. The screen pays for itself many times over, so when the table does
  // not fit beside four stages the kernel runs with fewer (>= 2).
  const size_t lists_b = size_t(tc::kEpilogueWarps) * 2 * K * sizeof(uint64_t);
  // scaled narrow path with large classes: the screen's pooled term from
  // Stirling's bound, the table only up to max(N0, N1) (E3_SCREEN_STIRLING=0/1
  // overrides; measured cfg3 +2%, cfg2 -5%)
  bool stir = ds->narrow && ds->shift && std::max(ds->N[0], ds->N[1]) >= 4096;
  if (const char* e = std::getenv("E3_SCREEN_STIRLING")) stir = ds->narrow && ds->shift && std::atoi(e) != 0;
  const uint32_t ktab_use =
      stir ? uint32_t((std::max(ds->N[0], ds->N[1]) + 1 + 3) / 4 * 4) : ds->ktab_n;
  const size_t tab_b = sizeof(float) * ktab_use;
  const size_t cap = ds->smem_optin - 2048;
  const size_t kst_b = ds->narrow ? size_t(syrk::kKStageTotal) : 0;  // narrow k staging
  uint32_t nst = syrk::kSyrkStages;
  bool screen = !std::getenv("E3_NO_SCREEN");
  if (const char* e = std::getenv("E3_SYRK_STAGES")) nst = uint32_t(std::max(2, std::min(syrk::kSyrkStages, std::atoi(e))));
  if (screen) {
    while (nst > 2 && 128 + nst * syrk::kSBStageBytes + lists_b + tab_b + kst_b > cap) --nst;
    screen = 128 + nst * syrk::kSBStageBytes + lists_b + tab_b + kst_b <= cap;
    if (!screen) nst = syrk::kSyrkStages;
  }
  size_t tsm = 128 + nst * syrk::kSBStageBytes + lists_b + (screen ? tab_b : 0) + kst_b;
  // narrow: the epilogue scratch in shared memory when it fits beside the
  // table (two B stages suffice; A lives in TMEM)
  bool sscr = false;
  if (ds->narrow && !std::getenv("E3_NO_SMEM_SCRATCH")) {
    const size_t cap_ss = ds->smem_ss_cap;
    for (uint32_t n2 = nst; n2 >= 2 && !sscr; --n2) {
      const size_t t2 = 128 + n2 * syrk::kSBStageBytes + syrk::kSmemScratchBytes + lists_b +
                        (screen ? tab_b : 0) + kst_b;
      if (t2 <= cap_ss) {
        sscr = true;
        nst = n2;
        tsm = t2;
      }
    }
  }
  // Y staging ring in the shared memory left over (>= 4 slots, else the
  // producers prefetch into registers); E3_NO_YRING=1 disables it
  uint32_t ny = 0;
  if (!syrk::kPair && !std::getenv("E3_NO_YRING")) {
    const size_t lim = sscr ? ds->smem_ss_cap : cap;
    const size_t have = lim > tsm + 256 ? lim - tsm - 256 : 0;
    ny = uint32_t(std::min<size_t>(syrk::kMaxYSlots, have / syrk::kYSlotBytes));
    if (ny < 4) ny = 0;
    else tsm += 256 + size_t(ny) * syrk::kYSlotBytes;
  }
  // compaction waits for the metadata upload (and all earlier work on st)
  CUDA_TRY(cudaStreamWaitEvent(ds->cstream, ds->ev_upload, 0));
  for (size_t b = 0; b < batches.size(); ++b) {
    const Batch& bt = batches[b];
    const int buf = int(b & 1);
    uint4* ybuf = ds->y_buf + size_t(buf) * ds->y_cap;
    syrk::SyrkArgs sa{};
    sa.item_begin = 0;
    sa.item_count = bt.tiles;
    sa.rank_begin = r0;
    sa.rank_end = r1;
    sa.top_k = K;
    sa.i_lo = bt.first;
    sa.n_i = bt.n;
    sa.gthr = ds->gthr;
    sa.lists = ds->lists[0];
    sa.counts = ds->counts[0];
    sa.info = ds->info_buf + bt.info_at;
    sa.itemoff = ds->syrk_off + bt.off_at;
    sa.Y = ybuf;
    sa.scratch = ds->scratch;
    sa.evals = ds->evals;
    sa.col = col;
    sa.debug_skip = ds->debug_skip;
    sa.screen = screen ? 1u : 0u;
    sa.nst = nst;
    sa.ktab_n = ktab_use;
    sa.ny = ny;
    // batch b's compaction overlaps batch b-1's search; it may reuse buffer
    // b & 1 only once batch b-2's search is done with it
    if (b >= 2) CUDA_TRY(cudaStreamWaitEvent(ds->cstream, ds->ev_sdone[buf], 0));
    {
      // bit-compress compaction; long sample axes are split into segments
      // over a zeroed Y (boundary words ORed)
      const uint64_t nwmax = (std::max(ds->N[0], ds->N[1]) + 31) / 32;
      const uint32_t nseg = uint32_t((nwmax + syrk::kPextSeg - 1) / syrk::kPextSeg);
      if (nseg > 1) CUDA_TRY(cudaMemsetAsync(ybuf, 0, sizeof(uint4) * bt.ytot, ds->cstream));
      syrk::compact_pext_kernel<<<dim3((bt.rmax + 127) / 128, 4, bt.n * nseg), 128, 0,
                                  ds->cstream>>>(d, sa, ybuf, nseg);
    }
    CUDA_TRY(cudaEventRecord(ds->ev_cdone[buf], ds->cstream));
    CUDA_TRY(cudaStreamWaitEvent(st, ds->ev_cdone[buf], 0));
    // only batches holding a partially covered first SNP need per-triple rank
    // checks; the others run the unranged kernel
    const uint64_t b_lo = first_rank(bt.first), b_hi = first_rank(bt.first + bt.n);
    const bool part = ranged && (r0 > b_lo || r1 < b_hi);
    if (sscr && stir) {
      if (part) syrk::search_syrk_kernel<true, 3, true><<<grid, syrk::kSyrkThreads, tsm, st>>>(d, sa);
      else syrk::search_syrk_kernel<false, 3, true><<<grid, syrk::kSyrkThreads, tsm, st>>>(d, sa);
    } else if (stir) {
      if (part) syrk::search_syrk_kernel<true, 3><<<grid, syrk::kSyrkThreads, tsm, st>>>(d, sa);
      else syrk::search_syrk_kernel<false, 3><<<grid, syrk::kSyrkThreads, tsm, st>>>(d, sa);
    } else if (sscr && ds->shift) {
      if (part) syrk::search_syrk_kernel<true, 2, true><<<grid, syrk::kSyrkThreads, tsm, st>>>(d, sa);
      else syrk::search_syrk_kernel<false, 2, true><<<grid, syrk::kSyrkThreads, tsm, st>>>(d, sa);
    } else if (sscr) {
      if (part) syrk::search_syrk_kernel<true, 1, true><<<grid, syrk::kSyrkThreads, tsm, st>>>(d, sa);
      else syrk::search_syrk_kernel<false, 1, true><<<grid, syrk::kSyrkThreads, tsm, st>>>(d, sa);
    } else if (ds->narrow && ds->shift) {
      if (part) syrk::search_syrk_kernel<true, 2><<<grid, syrk::kSyrkThreads, tsm, st>>>(d, sa);
      else syrk::search_syrk_kernel<false, 2><<<grid, syrk::kSyrkThreads, tsm, st>>>(d, sa);
    } else if (ds->narrow) {
      if (part) syrk::search_syrk_kernel<true, 1><<<grid, syrk::kSyrkThreads, tsm, st>>>(d, sa);
      else syrk::search_syrk_kernel<false, 1><<<grid, syrk::kSyrkThreads, tsm, st>>>(d, sa);
    } else {
      if (part) syrk::search_syrk_kernel<true, 0><<<grid, syrk::kSyrkThreads, tsm, st>>>(d, sa);
      else syrk::search_syrk_kernel<false, 0><<<grid, syrk::kSyrkThreads, tsm, st>>>(d, sa);
    }
    CUDA_TRY(cudaGetLastError());
    CUDA_TRY(cudaEventRecord(ds->ev_sdone[buf], st));
    *launches += 2;
  }
  // the host vectors die here: wait for their uploads only (kernels keep running)
  CUDA_TRY(cudaEventSynchronize(ds->ev_upload));
  return E3_OK;
}

}  // namespace

extern "C" int e3_search(const e3_dataset* cds, const e3_search_cfg* cfg, e3_hit* top,
                         uint32_t* n_top, e3_stats* stats) {
  const auto t_start = std::chrono::steady_clock::now();
  e3_dataset* ds = const_cast<e3_dataset*>(cds);
  if (!ds) return fail(E3_DOMAIN, "null dataset");
  if (!cfg) return fail(E3_DOMAIN, "null search configuration");
  std::lock_guard<std::mutex> call_lock(ds->call_mu);
  if (cfg->top_k < 1) return fail(E3_DOMAIN, "top_k must be >= 1");
  if (cfg->top_k > E3_MAX_TOP_K)
    return fail(E3_DOMAIN, "top_k above " + std::to_string(E3_MAX_TOP_K) + " is not supported");
  const uint64_t M = ds->M;
  uint64_t total = 0;
  if (int rc = e3_num_combinations(M, 3, &total)) return rc;
  const uint64_t r0 = cfg->rank_begin;
  const uint64_t r1 = cfg->rank_end == 0 ? total : cfg->rank_end;
  if (r1 > total || r0 > r1) return fail(E3_INDEX, "triple-rank range outside [0, C(M,3))");
  *n_top = 0;
  if (stats) std::memset(stats, 0, sizeof(*stats));
  if (r0 == r1) return E3_OK;
  CUDA_TRY(cudaSetDevice(ds->device));

  uint32_t t0[3], t1[3];
  e3::triple_unrank(M, r0, t0);
  e3::triple_unrank(M, r1 - 1, t1);
  SearchArgs a;
  a.item_begin = ds->h_itemoff[t0[0]];
  a.item_count = ds->h_itemoff[t1[0] + 1] - a.item_begin;
  a.rank_begin = r0;
  a.rank_end = r1;
  a.gthr = ds->gthr;
  a.evals = ds->evals;
  const bool ranged = !(r0 == 0 && r1 == total);

  const uint32_t K = cfg->top_k;
  // Per-warp lists hold Kl <= kListK entries in shared memory. A larger k
  // runs two passes: the union of all lists of a Kl-pass is a set of >= k
  // distinct scored triples, so its k-th best key bounds the global top-k;
  // the second pass collects every triple at or below that bound, and the
  // host sorts the candidates (exact: no top-k triple can exceed the bound).
  const uint32_t Kl = std::min<uint32_t>(K, kListK);
  // Engines: compacted tensor-core SYRK (default), masked tensor-core GEMM,
  // LOP3/POPC. All produce identical results.
  uint32_t engine = cfg->flags & 3u;
  // the SYRK engine accumulates exact counts in f32 (fp4 operands): N_c < 2^23
  const bool syrk_ok = std::max(ds->N[0], ds->N[1]) < (uint64_t(1) << 23);
  if (engine == 0)  // auto: compaction pays off once the sample axis is long
    engine = (ds->N[0] + ds->N[1]) >= 4096 && syrk_ok ? E3_ENGINE_SYRK : E3_ENGINE_TC_MASKED;
  if (engine == E3_ENGINE_SYRK && !syrk_ok)
    return fail(E3_DOMAIN, "the SYRK engine supports at most 2^23 - 1 samples per class");
  const bool use_syrk = engine == E3_ENGINE_SYRK;
  const bool use_tc = engine == E3_ENGINE_TC_MASKED;
  uint32_t grid, nlists;
  tc::TcArgs ta{};
  if (use_syrk) {
    grid = uint32_t(ds->num_sms);
    nlists = grid * tc::kEpilogueWarps;
  } else if (use_tc) {
    ta.item_begin = ds->h_itemoff_tc[t0[0]];
    ta.item_count = ds->h_itemoff_tc[t1[0] + 1] - ta.item_begin;
    grid = uint32_t(std::max<uint64_t>(1, std::min<uint64_t>(ds->num_sms, ta.item_count)));
    nlists = grid * tc::kEpilogueWarps;
  } else {
    const uint64_t grid64 = std::min<uint64_t>(uint64_t(ds->num_sms) * ds->search_ctas_per_sm,
                                               a.item_count);
    grid = uint32_t(std::max<uint64_t>(1, grid64));
    nlists = grid * kWarps;
  }
  const size_t need = size_t(nlists) * Kl;
  if (need > ds->lists_cap || nlists > ds->counts_cap) {
    for (int b = 0; b < 2; ++b) {
      dfree(ds, ds->lists[b]);
      dfree(ds, ds->counts[b]);
      ds->lists[b] = nullptr;
      ds->counts[b] = nullptr;
      ds->lists_cap = ds->counts_cap = 0;
      CUDA_TRY(dmalloc(ds, &ds->lists[b], sizeof(ulonglong2) * need));
      CUDA_TRY(dmalloc(ds, &ds->counts[b], sizeof(uint32_t) * nlists));
    }
    ds->lists_cap = need;
    ds->counts_cap = nlists;
  }
  a.out_lists = ds->lists[0];
  a.out_counts = ds->counts[0];
  if (!use_syrk)
    if (int rc = ensure_wide(ds)) return rc;
  const DevData d = dev_view(ds);
  const size_t smem = 2 * sizeof(uint64_t) * kWarps * Kl;
  cudaStream_t st = ds->stream;

  // one pass of the selected engine over [r0, r1): per-warp lists of Kl
  // entries, or (col.buf set) candidate collection below the fixed threshold
  uint32_t launches = 0, main_launches = 0;
  auto run_pass = [&](const Collect& col) -> int {
    CUDA_TRY(cudaMemsetAsync(ds->evals, 0, sizeof(unsigned long long), st));
    if (use_syrk) {
      uint32_t l = 0;
      if (int rc = run_syrk(ds, d, r0, r1, Kl, ranged, t0[0], t1[0], grid, &l, col)) return rc;
      launches += l;
      main_launches += l / 2;  // one compaction + one search kernel per batch
    } else if (use_tc) {
      ta.rank_begin = r0;
      ta.rank_end = r1;
      ta.top_k = Kl;
      ta.gthr = ds->gthr;
      ta.evals = ds->evals;
      ta.col = col;
      ta.out_lists = ds->lists[0];
      ta.out_counts = ds->counts[0];
      ta.itemoff = ds->itemoff_tc;
      const size_t tsm = tc::smem_bytes(Kl);
      if (ranged) tc::search_tc_kernel<true><<<grid, tc::kThreads, tsm, st>>>(d, ta);
      else tc::search_tc_kernel<false><<<grid, tc::kThreads, tsm, st>>>(d, ta);
      ++launches;
      ++main_launches;
    } else {
      a.top_k = Kl;
      a.col = col;
      if (ds->search_min_blocks == 2) {
        if (ranged) search_kernel<true, 2><<<grid, kWarps * 32, smem, st>>>(d, a);
        else search_kernel<false, 2><<<grid, kWarps * 32, smem, st>>>(d, a);
      } else {
        if (ranged) search_kernel<true, 1><<<grid, kWarps * 32, smem, st>>>(d, a);
        else search_kernel<false, 1><<<grid, kWarps * 32, smem, st>>>(d, a);
      }
      ++launches;
      ++main_launches;
    }
    CUDA_TRY(cudaGetLastError());
    return E3_OK;
  };
  // exactly-once check after each pass: the kernels count every triple they evaluate
  auto check_evals = [&]() -> int {
    unsigned long long evaluated = 0;
    CUDA_TRY(cudaMemcpyAsync(&evaluated, ds->evals, sizeof(evaluated), cudaMemcpyDeviceToHost, st));
    CUDA_TRY(cudaStreamSynchronize(st));
    if (evaluated != r1 - r0 && !(ds->debug_skip & 1))
      return fail(E3_CUDA, "exactly-once accounting violated: evaluated " +
                               std::to_string(evaluated) + " triples of the range's " +
                               std::to_string(r1 - r0));
    return E3_OK;
  };

  CUDA_TRY(cudaEventRecord(ds->ev[0], st));
  CUDA_TRY(cudaMemsetAsync(ds->gthr, 0xff, sizeof(uint64_t), st));
  CUDA_TRY(cudaEventRecord(ds->ev[1], st));
  if (int rc = run_pass(Collect{})) return rc;
  CUDA_TRY(cudaEventRecord(ds->ev[2], st));
  float pass1_kernel_ms = 0.f;
  std::vector<ulonglong2> h;
  uint32_t cnt = 0;
  if (K == Kl) {
    // Merge rounds: groups of lists -> one list each, until one list remains.
    uint32_t nl = nlists;
    int cur = 0;
    const uint32_t group = std::max<uint32_t>(2, kMergeCap / K);
    while (nl > 1) {
      const uint32_t g = std::min(group, nl);
      uint32_t P = 1;
      while (P < g * K) P <<= 1;
      const uint32_t blocks = (nl + g - 1) / g;
      merge_kernel<<<blocks, 1024, sizeof(ulonglong2) * P, st>>>(
          ds->lists[cur], ds->counts[cur], nl, K, g, P, ds->lists[cur ^ 1], ds->counts[cur ^ 1]);
      CUDA_TRY(cudaGetLastError());
      ++launches;
      cur ^= 1;
      nl = blocks;
    }
    h.resize(K);
    CUDA_TRY(cudaMemcpyAsync(h.data(), ds->lists[cur], sizeof(ulonglong2) * K,
                             cudaMemcpyDeviceToHost, st));
    CUDA_TRY(cudaMemcpyAsync(&cnt, ds->counts[cur], sizeof(uint32_t), cudaMemcpyDeviceToHost, st));
    CUDA_TRY(cudaEventRecord(ds->ev[3], st));
    if (int rc = check_evals()) return rc;
    cnt = std::min(cnt, K);
  } else {
    // ---- large k, pass 1 -> bound: the k-th best key over the union of all lists
    std::vector<ulonglong2> lists(size_t(nlists) * Kl);
    std::vector<uint32_t> counts(nlists);
    CUDA_TRY(cudaMemcpyAsync(lists.data(), ds->lists[0], sizeof(ulonglong2) * lists.size(),
                             cudaMemcpyDeviceToHost, st));
    CUDA_TRY(cudaMemcpyAsync(counts.data(), ds->counts[0], sizeof(uint32_t) * nlists,
                             cudaMemcpyDeviceToHost, st));
    if (int rc = check_evals()) return rc;
    cudaEventElapsedTime(&pass1_kernel_ms, ds->ev[1], ds->ev[2]);
    std::vector<ulonglong2> uni;
    for (uint32_t l = 0; l < nlists; ++l)
      uni.insert(uni.end(), lists.begin() + size_t(l) * Kl,
                 lists.begin() + size_t(l) * Kl + std::min(counts[l], Kl));
    auto less = [](const ulonglong2& x, const ulonglong2& y) {
      return x.x < y.x || (x.x == y.x && x.y < y.y);
    };
    uint64_t thr = ~0ull;  // fewer than k triples scored so far: collect everything
    if (uni.size() >= K) {
      std::nth_element(uni.begin(), uni.begin() + (K - 1), uni.end(), less);
      thr = uni[K - 1].x;
    } else if (r1 - r0 > (uint64_t(1) << 28)) {
      return fail(E3_DOMAIN, "top_k " + std::to_string(K) + " exceeds what this search can rank");
    }
    // ---- pass 2: collect every triple with score key <= thr
    size_t cap = thr == ~0ull ? size_t(r1 - r0) : std::max<size_t>(size_t(4) * K, size_t(1) << 16);
    uint32_t n_cand = 0;
    for (int attempt = 0; attempt < 2; ++attempt) {
      if (cap > ds->cand_cap) {
        dfree(ds, ds->cand);
        ds->cand = nullptr;
        ds->cand_cap = 0;
        CUDA_TRY(dmalloc(ds, &ds->cand, sizeof(ulonglong2) * cap));
        ds->cand_cap = cap;
      }
      Collect col;
      col.buf = ds->cand;
      col.n = ds->cand_n;
      col.cap = uint32_t(std::min<size_t>(ds->cand_cap, 0xffffffffu));
      CUDA_TRY(cudaMemsetAsync(ds->cand_n, 0, sizeof(unsigned int), st));
      CUDA_TRY(cudaMemcpyAsync(ds->gthr, &thr, sizeof(uint64_t), cudaMemcpyHostToDevice, st));
      CUDA_TRY(cudaEventRecord(ds->ev[1], st));
      if (int rc = run_pass(col)) return rc;
      CUDA_TRY(cudaEventRecord(ds->ev[2], st));
      CUDA_TRY(cudaMemcpyAsync(&n_cand, ds->cand_n, sizeof(unsigned int), cudaMemcpyDeviceToHost, st));
      if (int rc = check_evals()) return rc;
      if (n_cand <= col.cap) break;
      cap = n_cand;  // the count is exact: a second attempt always fits
    }
    h.resize(n_cand);
    CUDA_TRY(cudaMemcpyAsync(h.data(), ds->cand, sizeof(ulonglong2) * n_cand,
                             cudaMemcpyDeviceToHost, st));
    CUDA_TRY(cudaEventRecord(ds->ev[3], st));
    CUDA_TRY(cudaStreamSynchronize(st));
    const size_t keep = std::min<size_t>(K, h.size());
    std::partial_sort(h.begin(), h.begin() + keep, h.end(), less);
    cnt = uint32_t(keep);
  }
  for (uint32_t x = 0; x < cnt; ++x) {
    top[x].score = key_score(h[x].x);
    top[x].i0 = uint32_t(h[x].y >> 42);
    top[x].i1 = uint32_t((h[x].y >> 21) & 0x1fffff);
    top[x].i2 = uint32_t(h[x].y & 0x1fffff);
    top[x]._pad = 0;
  }
  *n_top = cnt;
  if (stats) {
    float ms = 0.f;
    // counted on the device, triple by triple (exactly-once accounting,
    // checked above against rank_end - rank_begin)
    stats->combinations = r1 - r0;
    cudaEventElapsedTime(&ms, ds->ev[1], ds->ev[2]);
    stats->kernel_ms = ms + pass1_kernel_ms;
    cudaEventElapsedTime(&ms, ds->ev[0], ds->ev[3]);
    stats->total_device_ms = ms;
    stats->kernel_launches = launches;
    stats->main_kernel_launches = main_launches;
    stats->elapsed_s =
        std::chrono::duration<double>(std::chrono::steady_clock::now() - t_start).count();
  }
  return E3_OK;
}

// ---------------------------------------------------------------------------
// C ABI: tables and scores for explicit triples
// ---------------------------------------------------------------------------
namespace {
int run_triples(const e3_dataset* ds, const uint32_t* triples, uint64_t n, uint32_t* tables,
                double* scores) {
  if (!ds) return fail(E3_DOMAIN, "null dataset");
  for (uint64_t t = 0; t < n; ++t) {
    const uint32_t i = triples[3 * t], j = triples[3 * t + 1], k = triples[3 * t + 2];
    if (!(i < j && j < k))
      return fail(E3_INDEX, "triple (" + std::to_string(i) + "," + std::to_string(j) + "," +
                                std::to_string(k) + ") is not strictly ordered");
    if (k >= ds->M)
      return fail(E3_INDEX, "triple (" + std::to_string(i) + "," + std::to_string(j) + "," +
                                std::to_string(k) + ") out of range for " +
                                std::to_string(ds->M) + " SNPs");
  }
  if (n == 0) return E3_OK;
  std::lock_guard<std::mutex> call_lock(const_cast<e3_dataset*>(ds)->call_mu);
  CUDA_TRY(cudaSetDevice(ds->device));
  if (int rc = ensure_wide(ds)) return rc;
  uint32_t* d_tri = nullptr;
  uint32_t* d_tab = nullptr;
  double* d_sc = nullptr;
  CUDA_TRY(dmalloc(ds, &d_tri, sizeof(uint32_t) * 3 * n));
  if (tables) CUDA_TRY(dmalloc(ds, &d_tab, sizeof(uint32_t) * 54 * n));
  if (scores) CUDA_TRY(dmalloc(ds, &d_sc, sizeof(double) * n));
  cudaStream_t st = ds->stream;
  CUDA_TRY(cudaMemcpyAsync(d_tri, triples, sizeof(uint32_t) * 3 * n, cudaMemcpyHostToDevice, st));
  triples_kernel<<<unsigned((n + 127) / 128), 128, 0, st>>>(dev_view(ds), d_tri, n, d_tab, d_sc);
  CUDA_TRY(cudaGetLastError());
  if (tables)
    CUDA_TRY(cudaMemcpyAsync(tables, d_tab, sizeof(uint32_t) * 54 * n, cudaMemcpyDeviceToHost, st));
  if (scores)
    CUDA_TRY(cudaMemcpyAsync(scores, d_sc, sizeof(double) * n, cudaMemcpyDeviceToHost, st));
  CUDA_TRY(cudaStreamSynchronize(st));
  dfree(ds, d_tri);
  dfree(ds, d_tab);
  dfree(ds, d_sc);
  return E3_OK;
}
}  // namespace

extern "C" int e3_tables(const e3_dataset* ds, const uint32_t* triples, uint64_t n,
                         uint32_t* out) {
  return run_triples(ds, triples, n, out, nullptr);
}

extern "C" int e3_scores(const e3_dataset* ds, const uint32_t* triples, uint64_t n,
                         double* out) {
  return run_triples(ds, triples, n, nullptr, out);
}
