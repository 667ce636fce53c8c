// host.cpp — host-side entry points of the C ABI (include/epi3cu.h) that do no
// device work: dataset load/format, synthetic inputs, the K2 log table, rank
// arithmetic, the partitioner and the top-k merge. Fresh implementations of
// the reference behaviour cited per function (/root/reference/proj/...).
#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <random>
#include <string>
#include <vector>

#include "epi3cu.h"
#include "internal.h"

namespace e3 {

thread_local std::string g_last_error;

int fail(int code, const std::string& msg) {
  g_last_error = msg;
  return code;
}

}  // namespace e3

using e3::fail;
using u128 = unsigned __int128;

extern "C" const char* e3_last_error(void) { return e3::g_last_error.c_str(); }

// ---------------------------------------------------------------------------
// combinatorics: num_combinations (src/search.cpp:48-59) and the rank space
// ---------------------------------------------------------------------------
extern "C" int e3_num_combinations(uint64_t m, uint64_t k, uint64_t* out) {
  if (m < k)
    return fail(E3_DOMAIN, "cannot choose " + std::to_string(k) + " from " + std::to_string(m));
  u128 r = 1;
  for (uint64_t i = 1; i <= k; ++i) {
    r = r * (m - k + i) / i;
    if (r > (u128)UINT64_MAX) return fail(E3_DOMAIN, "binomial coefficient exceeds 64 bits");
  }
  *out = (uint64_t)r;
  return E3_OK;
}

namespace {
u128 c3(uint64_t n) { return n < 3 ? 0 : (u128)n * (n - 1) * (n - 2) / 6; }
u128 c2(uint64_t n) { return n < 2 ? 0 : (u128)n * (n - 1) / 2; }
}  // namespace

namespace e3 {
uint64_t triple_rank(uint64_t M, uint64_t i0, uint64_t i1, uint64_t i2) {
  return (uint64_t)(c3(M) - c3(M - i0) + c2(M - 1 - i0) - c2(M - i1) + (i2 - i1 - 1));
}
void triple_unrank(uint64_t M, uint64_t r, uint32_t* t) {
  uint64_t lo = 0, hi = M - 3;
  while (lo < hi) {
    const uint64_t mid = (lo + hi + 1) / 2;
    if (c3(M) - c3(M - mid) <= r) lo = mid; else hi = mid - 1;
  }
  const uint64_t a = lo;
  const uint64_t rest = r - (uint64_t)(c3(M) - c3(M - a));
  lo = a + 1;
  hi = M - 2;
  while (lo < hi) {
    const uint64_t mid = (lo + hi + 1) / 2;
    if (c2(M - 1 - a) - c2(M - mid) <= rest) lo = mid; else hi = mid - 1;
  }
  const uint64_t b = lo;
  t[0] = uint32_t(a);
  t[1] = uint32_t(b);
  t[2] = uint32_t(b + 1 + rest - (uint64_t)(c2(M - 1 - a) - c2(M - b)));
}
}  // namespace e3

extern "C" int e3_triple_rank(uint64_t M, uint32_t i0, uint32_t i1, uint32_t i2,
                              uint64_t* rank) {
  if (!(i0 < i1 && i1 < i2) || i2 >= M)
    return fail(E3_INDEX, "triple (" + std::to_string(i0) + "," + std::to_string(i1) + "," +
                              std::to_string(i2) + ") is not an ordered triple below M");
  *rank = e3::triple_rank(M, i0, i1, i2);
  return E3_OK;
}

extern "C" int e3_triple_unrank(uint64_t M, uint64_t rank, uint32_t* t) {
  if (M < 3 || (u128)rank >= c3(M)) return fail(E3_INDEX, "triple rank out of range");
  e3::triple_unrank(M, rank, t);
  return E3_OK;
}

// Equal-work split of the lexicographic rank space. Every triple costs the
// same (27 cells x the class words), so equal counts are equal work; this is
// the GPU analogue of the reference's shared work counter (search.cpp:155,
// 179-185), fixed ahead of time because ranks are independent.
extern "C" int e3_partition(uint64_t M, uint32_t parts, uint64_t* bounds) {
  if (parts < 1) return fail(E3_DOMAIN, "parts must be >= 1");
  if (M < 3) return fail(E3_DIMENSION, "search needs at least 3 SNPs");
  const u128 total = c3(M);
  for (uint32_t p = 0; p <= parts; ++p) bounds[p] = (uint64_t)(total * p / parts);
  return E3_OK;
}

// Cost-balanced partition for the multi-GPU split: the SYRK engine's device
// time over a range is, to ~1-3%, a fixed cost per 64x64 (j,k) tile plus a
// per-first-SNP cost (compaction, batch boundaries) of about kTilesPerSnp
// tiles (64: refitted to the 8 equal-cost ranges of the final cfg3 kernel,
// profiles/r02e_bench_cfg3_driver_cmd.json partition_balance; the earlier
// kernel fitted 16, profiles/r02_partition_model.json). Ranges hold equal shares of that cost; inside a first SNP the cost
// is taken as proportional to its triples (j-major order covers tile rows).
extern "C" int e3_partition_balanced(uint64_t M, uint32_t parts, uint64_t* bounds) {
  if (parts < 1) return fail(E3_DOMAIN, "parts must be >= 1");
  if (M < 3) return fail(E3_DIMENSION, "search needs at least 3 SNPs");
  constexpr double kTilesPerSnp = 64.0;
  constexpr uint64_t kEdge = 64;
  std::vector<double> cw(M - 1, 0.0);  // cumulative cost before first SNP i
  for (uint64_t i = 0; i + 2 < M; ++i) {
    const uint64_t nb = (M - 1 - i + kEdge - 1) / kEdge;
    cw[i + 1] = cw[i] + double(nb * (nb + 1) / 2) + kTilesPerSnp;
  }
  const double total_cost = cw[M - 2];
  const uint64_t total = (uint64_t)c3(M);
  bounds[0] = 0;
  uint64_t i = 0;
  for (uint32_t p = 1; p < parts; ++p) {
    const double target = total_cost * p / parts;
    while (i + 3 < M && cw[i + 1] <= target) ++i;
    const uint64_t first = total - (uint64_t)c3(M - i);  // rank of (i, i+1, i+2)
    const uint64_t tri = (M - 1 - i) * (M - 2 - i) / 2;
    const double frac = std::min(1.0, std::max(0.0, (target - cw[i]) / (cw[i + 1] - cw[i])));
    bounds[p] = std::max(bounds[p - 1], first + uint64_t(std::llround(frac * double(tri))));
  }
  bounds[parts] = total;
  return E3_OK;
}

// ---------------------------------------------------------------------------
// K2 scoring on the host: build_log_table / k2_score (src/scoring.cpp:14-35)
// ---------------------------------------------------------------------------
extern "C" int e3_build_log_table(uint64_t n_max, double* prefix) {
  prefix[0] = 0.0;
  for (uint64_t n = 1; n <= n_max; ++n) prefix[n] = prefix[n - 1] + std::log(double(n));
  return E3_OK;
}

extern "C" double e3_k2_score(const uint32_t* t, const double* P) {
  double score = 0.0;
  for (int c = 0; c < 27; ++c) {
    const uint32_t r0 = t[c], r1 = t[27 + c];
    const uint64_t r = uint64_t(r0) + r1;
    score += P[r + 1] - (P[r0] + P[r1]);
  }
  return score;
}

// hit_less (include/epi3/search.hpp:29-35)
static bool hit_less(const e3_hit& a, const e3_hit& b) {
  if (a.score != b.score) return a.score < b.score;
  if (a.i0 != b.i0) return a.i0 < b.i0;
  if (a.i1 != b.i1) return a.i1 < b.i1;
  return a.i2 < b.i2;
}

// reduce_results' list merge (search.cpp:119-123)
extern "C" int e3_merge_hits(const e3_hit* hits, uint64_t n, uint32_t top_k, e3_hit* out,
                             uint32_t* n_out) {
  std::vector<e3_hit> v(hits, hits + n);
  std::sort(v.begin(), v.end(), hit_less);
  auto same = [](const e3_hit& a, const e3_hit& b) {
    return a.score == b.score && a.i0 == b.i0 && a.i1 == b.i1 && a.i2 == b.i2;
  };
  v.erase(std::unique(v.begin(), v.end(), same), v.end());
  if (v.size() > top_k) v.resize(top_k);
  std::copy(v.begin(), v.end(), out);
  *n_out = uint32_t(v.size());
  return E3_OK;
}

// ---------------------------------------------------------------------------
// validate + binarize (src/datamodel.cpp:28-46, 69-92)
// ---------------------------------------------------------------------------
extern "C" int e3_binarize(uint64_t M, uint64_t N, const uint8_t* geno, const uint8_t* pheno,
                           uint64_t* N0, uint64_t* N1, uint64_t* ctrl, uint64_t* cases) {
  if (M < 3) return fail(E3_DIMENSION, "need at least 3 SNPs, got " + std::to_string(M));
  if (N == 0) return fail(E3_DIMENSION, "dataset has no samples");
  uint64_t n1 = 0;
  for (uint64_t j = 0; j < N; ++j) {
    if (pheno[j] > 1)
      return fail(E3_DOMAIN, "phenotype value " + std::to_string(pheno[j]) +
                                 " at snp 0, sample " + std::to_string(j));
    n1 += pheno[j];
  }
  const uint64_t n0 = N - n1;
  if (n0 > 0xffffffffull || n1 > 0xffffffffull)
    return fail(E3_DOMAIN, "class sample count exceeds the 32-bit cell cap");
  *N0 = n0;
  *N1 = n1;
  if (!ctrl || !cases) return E3_OK;
  for (uint64_t i = 0; i < M; ++i)
    for (uint64_t j = 0; j < N; ++j)
      if (geno[i * N + j] > 2)
        return fail(E3_DOMAIN, "genotype value " + std::to_string(geno[i * N + j]) +
                                   " at snp " + std::to_string(i) + ", sample " +
                                   std::to_string(j));
  const uint64_t w[2] = {(n0 + 63) / 64, (n1 + 63) / 64};
  std::memset(ctrl, 0, M * 2 * w[0] * sizeof(uint64_t));
  std::memset(cases, 0, M * 2 * w[1] * sizeof(uint64_t));
  // In-class positions, stable in order of appearance (datamodel.cpp:75-79).
  std::vector<uint64_t> pos(N);
  uint64_t next[2] = {0, 0};
  for (uint64_t j = 0; j < N; ++j) pos[j] = next[pheno[j]]++;
  uint64_t* data[2] = {ctrl, cases};
  for (uint64_t i = 0; i < M; ++i) {
    const uint8_t* row = geno + i * N;
    for (uint64_t j = 0; j < N; ++j) {
      const uint8_t g = row[j];
      if (g < 2) {
        const int c = pheno[j];
        data[c][(i * 2 + g) * w[c] + (pos[j] >> 6)] |= 1ull << (pos[j] & 63);
      }
    }
  }
  return E3_OK;
}

// ---------------------------------------------------------------------------
// generate_synthetic (src/datamodel.cpp:169-227) + exact class counts
// ---------------------------------------------------------------------------
extern "C" int e3_generate_synthetic(uint64_t M, uint64_t N, double maf, uint64_t seed,
                                     const e3_plant* plant, int64_t exact_cases,
                                     uint8_t* geno, uint8_t* pheno) {
  if (!(maf > 0.0 && maf <= 0.5))
    return fail(E3_DOMAIN, "maf must be in (0, 0.5], got " + std::to_string(maf));
  if (M < 3) return fail(E3_DOMAIN, "need at least 3 SNPs");
  if (N == 0) return fail(E3_DOMAIN, "need at least 1 sample");
  if (exact_cases > (int64_t)N) return fail(E3_DOMAIN, "exact_cases exceeds the sample count");
  if (plant) {
    const e3_plant& p = *plant;
    if (p.i0 == p.i1 || p.i0 == p.i2 || p.i1 == p.i2)
      return fail(E3_DOMAIN, "plant SNP indices must be distinct");
    if (p.i0 >= M || p.i1 >= M || p.i2 >= M) return fail(E3_DOMAIN, "plant SNP index out of range");
    for (int k = 0; k < 3; ++k)
      if (p.target[k] > 2) return fail(E3_DOMAIN, "plant target genotype out of range");
    if (!(p.p_case_match >= 0.0 && p.p_case_match <= 1.0 && p.p_case_other >= 0.0 &&
          p.p_case_other <= 1.0))
      return fail(E3_DOMAIN, "plant probabilities must be in [0, 1]");
    if (!(p.p_case_match > p.p_case_other))
      return fail(E3_DOMAIN, "plant needs p_case_match > p_case_other");
  }
  const double p0 = (1.0 - maf) * (1.0 - maf);
  const double p01 = p0 + 2.0 * maf * (1.0 - maf);
  std::mt19937_64 rng(seed);
  // Uniform in [0,1) from the top 53 bits (datamodel.cpp:173-175).
  auto unit = [&]() { return double(rng() >> 11) * 0x1.0p-53; };
  for (uint64_t i = 0; i < M; ++i)
    for (uint64_t j = 0; j < N; ++j) {
      const double u = unit();
      geno[i * N + j] = u < p0 ? 0 : (u < p01 ? 1 : 2);
    }
  std::vector<uint8_t> match(N, 0);
  for (uint64_t j = 0; j < N; ++j) {
    double p_case = 0.5;
    if (plant) {
      match[j] = geno[plant->i0 * N + j] == plant->target[0] &&
                 geno[plant->i1 * N + j] == plant->target[1] &&
                 geno[plant->i2 * N + j] == plant->target[2];
      p_case = match[j] ? plant->p_case_match : plant->p_case_other;
    }
    pheno[j] = unit() < p_case ? 1 : 0;
  }
  if (exact_cases >= 0) {
    int64_t cases = 0;
    for (uint64_t j = 0; j < N; ++j) cases += pheno[j];
    // Flip surplus labels of non-matching samples first (lowest index first),
    // then matching ones only if that was not enough.
    for (int pass = 0; pass < 2 && cases != exact_cases; ++pass)
      for (uint64_t j = 0; j < N && cases != exact_cases; ++j) {
        if (match[j] != (pass == 1)) continue;
        if (cases > exact_cases && pheno[j] == 1) { pheno[j] = 0; --cases; }
        else if (cases < exact_cases && pheno[j] == 0) { pheno[j] = 1; ++cases; }
      }
  }
  return E3_OK;
}

// ---------------------------------------------------------------------------
// Packed EPI3 v1 (include/epi3/io.hpp:20-25; src/io.cpp:117-203)
// ---------------------------------------------------------------------------
namespace {
constexpr size_t kHeader = 32;
uint64_t le64(const unsigned char* p) {
  uint64_t v = 0;
  for (int i = 0; i < 8; ++i) v |= uint64_t(p[i]) << (8 * i);
  return v;
}

struct File {
  FILE* f = nullptr;
  ~File() { if (f) std::fclose(f); }
};

int read_header(FILE* f, const char* path, uint64_t* M, uint64_t* N0, uint64_t* N1,
                uint64_t* payload_bytes) {
  unsigned char h[kHeader];
  if (std::fread(h, 1, kHeader, f) != kHeader)
    return fail(E3_TRUNCATED, "file shorter than the packed header");
  if (std::memcmp(h, "EPI3", 4) != 0) return fail(E3_MAGIC, "not a packed genotype file (bad magic)");
  const uint32_t ver = uint32_t(h[4]) | uint32_t(h[5]) << 8 | uint32_t(h[6]) << 16 |
                       uint32_t(h[7]) << 24;
  if (ver != 1) return fail(E3_PARSE, "unsupported packed version " + std::to_string(ver) + " (at 4)");
  *M = le64(h + 8);
  *N0 = le64(h + 16);
  *N1 = le64(h + 24);
  if (*N0 > 0xffffffffull || *N1 > 0xffffffffull)
    return fail(E3_PARSE, "class sample count exceeds the 32-bit cell cap (at 16)");
  // Size arithmetic verified against the file before any allocation (io.cpp:134-149).
  const u128 words = (u128)(*M) * 2 * ((*N0 + 63) / 64 + (*N1 + 63) / 64);
  const u128 expected = kHeader + words * 8;
  if (std::fseek(f, 0, SEEK_END) != 0) return fail(E3_IO, std::string("cannot seek ") + path);
  const long size = std::ftell(f);
  if (size < 0) return fail(E3_IO, std::string("cannot size ") + path);
  if (expected > (u128)size) return fail(E3_TRUNCATED, "packed file shorter than its header promises");
  if (expected < (u128)size)
    return fail(E3_PARSE, "trailing bytes after packed payload (at " +
                              std::to_string((uint64_t)expected) + ")");
  std::fseek(f, long(kHeader), SEEK_SET);
  *payload_bytes = uint64_t(words * 8);
  return E3_OK;
}
}  // namespace

extern "C" int e3_packed_header(const char* path, uint64_t* M, uint64_t* N0, uint64_t* N1) {
  File fh;
  fh.f = std::fopen(path, "rb");
  if (!fh.f) return fail(E3_IO, std::string("cannot open ") + path);
  uint64_t payload = 0;
  return read_header(fh.f, path, M, N0, N1, &payload);
}

extern "C" int e3_read_packed(const char* path, uint64_t M, uint64_t N0, uint64_t N1,
                              uint64_t* ctrl, uint64_t* cases) {
  File fh;
  fh.f = std::fopen(path, "rb");
  if (!fh.f) return fail(E3_IO, std::string("cannot open ") + path);
  uint64_t m, n0, n1, payload;
  if (int rc = read_header(fh.f, path, &m, &n0, &n1, &payload)) return rc;
  if (m != M || n0 != N0 || n1 != N1)
    return fail(E3_DIMENSION, "packed header does not match the caller's dimensions");
  const uint64_t w[2] = {(N0 + 63) / 64, (N1 + 63) / 64};
  uint64_t* data[2] = {ctrl, cases};
  std::vector<unsigned char> buf;
  for (uint64_t i = 0; i < M; ++i)
    for (int c = 0; c < 2; ++c) {
      if (w[c] == 0) continue;
      buf.resize(2 * w[c] * 8);
      if (std::fread(buf.data(), 1, buf.size(), fh.f) != buf.size())
        return fail(E3_TRUNCATED, "packed payload ended early");
      uint64_t* dst = data[c] + i * 2 * w[c];
      for (uint64_t x = 0; x < 2 * w[c]; ++x) dst[x] = le64(buf.data() + 8 * x);
    }
  return E3_OK;
}

extern "C" int e3_write_packed(const char* path, uint64_t M, uint64_t N0, uint64_t N1,
                               const uint64_t* ctrl, const uint64_t* cases) {
  File fh;
  fh.f = std::fopen(path, "wb");
  if (!fh.f) return fail(E3_IO, std::string("cannot open ") + path + " for writing");
  unsigned char h[kHeader];
  std::memcpy(h, "EPI3", 4);
  h[4] = 1; h[5] = h[6] = h[7] = 0;
  const uint64_t v[3] = {M, N0, N1};
  for (int k = 0; k < 3; ++k)
    for (int i = 0; i < 8; ++i) h[8 + 8 * k + i] = (unsigned char)(v[k] >> (8 * i));
  std::fwrite(h, 1, kHeader, fh.f);
  const uint64_t w[2] = {(N0 + 63) / 64, (N1 + 63) / 64};
  const uint64_t* data[2] = {ctrl, cases};
  std::vector<unsigned char> buf;
  for (uint64_t i = 0; i < M; ++i)
    for (int c = 0; c < 2; ++c) {
      if (w[c] == 0) continue;
      buf.resize(2 * w[c] * 8);
      const uint64_t* src = data[c] + i * 2 * w[c];
      for (uint64_t x = 0; x < 2 * w[c]; ++x)
        for (int b = 0; b < 8; ++b) buf[8 * x + b] = (unsigned char)(src[x] >> (8 * b));
      std::fwrite(buf.data(), 1, buf.size(), fh.f);
    }
  if (std::ferror(fh.f)) return fail(E3_IO, "write failed");
  return E3_OK;
}
