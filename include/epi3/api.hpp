// epi3/api.hpp — the C++ drop-in surface of the B200 engine.
//
// Same namespace, names and semantics as the reference library's public API
// (/root/reference/proj/include/epi3/*.hpp): a program written against the
// reference's dataset load, run_search, best/top-k and K2 output recompiles
// against this header and links libepi3.so instead of libepi3.a. Everything
// that computes goes through the C ABI in epi3cu.h into sm_100a CUDA; there
// is no CPU search path. CPU-tiling knobs of the reference (KernelVariant,
// BlockParams, CacheSpec, lanes, chunk) have no meaning on the GPU and are
// not part of this surface. Reference file:line for each item below.
#pragma once

#include <array>
#include <compare>
#include <cstddef>
#include <cstdint>
#include <filesystem>
#include <optional>
#include <span>
#include <stdexcept>
#include <string>
#include <vector>

struct e3_dataset;

namespace epi3 {

// ---- core types (common.hpp:13-29) -----------------------------------------
using word = std::uint64_t;
inline constexpr std::size_t kWordBits = 64;
using snp_index = std::uint32_t;
inline constexpr int kControls = 0;
inline constexpr int kCases = 1;

struct Triple {
  snp_index i0 = 0, i1 = 0, i2 = 0;
  friend auto operator<=>(const Triple&, const Triple&) = default;
};
std::string to_string(const Triple& t);

// ---- errors (common.hpp:36-105), one per C-ABI status --------------------------
struct Error : std::runtime_error { using std::runtime_error::runtime_error; };
struct DomainError : Error { using Error::Error; };
struct DimensionError : Error { using Error::Error; };
struct IndexError : Error { using Error::Error; };
struct ParseError : Error { using Error::Error; };
struct MagicMismatch : Error { using Error::Error; };
struct TruncatedFile : Error { using Error::Error; };
struct InfeasibleCache : Error { using Error::Error; };  // common.hpp:97-100
struct CapExceeded : Error { using Error::Error; };      // common.hpp:102-105
struct DeviceError : Error { using Error::Error; };  // CUDA/NCCL/OOM: no reference analogue

// ---- raw data (genotype.hpp:14-33) --------------------------------------------
struct GenotypeMatrix {
  std::size_t num_snps = 0, num_samples = 0;
  std::vector<std::uint8_t> genotypes;  // SNP-major M*N
  std::vector<std::uint8_t> phenotype;  // N
  std::uint8_t geno(std::size_t i, std::size_t j) const { return genotypes[i * num_samples + j]; }
  std::uint8_t& geno(std::size_t i, std::size_t j) { return genotypes[i * num_samples + j]; }
  friend bool operator==(const GenotypeMatrix&, const GenotypeMatrix&) = default;
};
const GenotypeMatrix& validate(const GenotypeMatrix& m);  // datamodel.cpp:28-46

// ---- bit planes (bitplane.hpp:16-72) --------------------------------------------
constexpr word infer_plane2(word w0, word w1, word mask) { return ~(w0 | w1) & mask; }

class BitPlaneDataset {
 public:
  BitPlaneDataset() = default;
  BitPlaneDataset(std::size_t num_snps, std::size_t num_controls, std::size_t num_cases);
  std::size_t num_snps() const { return m_; }
  std::size_t num_controls() const { return n_[0]; }
  std::size_t num_cases() const { return n_[1]; }
  std::size_t num_samples() const { return n_[0] + n_[1]; }
  std::size_t class_count(int cls) const { return n_[cls]; }
  std::size_t words(int cls) const { return w_[cls]; }
  word pad_mask(int cls) const;
  const word* plane(int cls, snp_index snp, int g) const { return data_[cls].data() + (std::size_t(snp) * 2 + g) * w_[cls]; }
  word* plane(int cls, snp_index snp, int g) { return data_[cls].data() + (std::size_t(snp) * 2 + g) * w_[cls]; }
  std::uint8_t geno_at(int cls, snp_index snp, std::size_t pos) const;
  const std::vector<word>& data(int cls) const { return data_[cls]; }  // [snp][g][word]
  std::vector<word>& data(int cls) { return data_[cls]; }
  friend bool operator==(const BitPlaneDataset&, const BitPlaneDataset&) = default;

 private:
  std::size_t m_ = 0, n_[2] = {0, 0}, w_[2] = {0, 0};
  std::vector<word> data_[2];
};
BitPlaneDataset binarize(const GenotypeMatrix& m);  // datamodel.cpp:69-92
GenotypeMatrix decode(const BitPlaneDataset& ds);   // datamodel.cpp:94-109

// ---- synthetic inputs (synthetic.hpp:15-26) ---------------------------------------
struct PlantSpec {
  Triple triple;
  std::array<std::uint8_t, 3> target = {1, 1, 1};
  double p_case_match = 0.9;
  double p_case_other = 0.1;
};
// exact_cases >= 0: exact class counts (see epi3cu.h); -1 = reference behaviour.
GenotypeMatrix generate_synthetic(std::size_t num_snps, std::size_t num_samples, double maf,
                                  std::uint64_t seed, const std::optional<PlantSpec>& plant = {},
                                  std::int64_t exact_cases = -1);

// ---- formats (io.hpp:11-32) ---------------------------------------------------------
GenotypeMatrix read_text(const std::filesystem::path& path);
void write_text(const std::filesystem::path& path, const GenotypeMatrix& m);
BitPlaneDataset read_packed(const std::filesystem::path& path);
void write_packed(const std::filesystem::path& path, const BitPlaneDataset& ds);
bool is_packed_file(const std::filesystem::path& path);

// ---- scoring (scoring.hpp:11-59) ------------------------------------------------------
inline constexpr int kNumCombos = 27;
inline constexpr int kNumClasses = 2;
constexpr int combo_index(int gx, int gy, int gz) { return gx * 9 + gy * 3 + gz; }
struct FrequencyTable {
  std::array<std::uint32_t, 54> counts{};  // [cls][combo]
  std::uint32_t at(int combo, int cls) const { return counts[std::size_t(cls) * 27 + combo]; }
  std::uint32_t& at(int combo, int cls) { return counts[std::size_t(cls) * 27 + combo]; }
  std::uint32_t row_total(int combo) const { return at(combo, 0) + at(combo, 1); }
  std::uint64_t class_total(int cls) const;
  friend bool operator==(const FrequencyTable&, const FrequencyTable&) = default;
};
struct LogSumTable {
  std::vector<double> prefix;
  double log_factorial(std::size_t n) const { return prefix[n]; }
  std::size_t max_n() const { return prefix.size() - 1; }
};
LogSumTable build_log_table(std::size_t n_max);
double k2_score(const FrequencyTable& ft, const LogSumTable& logs);

// ---- kernel variants and CPU tiling knobs (kernels.hpp:17-67) ------------------------
// Accepted for source compatibility; all variants give identical results on
// the reference and the GPU engine ignores them.
enum class KernelVariant {
  NaivePhenotype,        // v1
  ReducedSplit,          // v2
  Blocked,               // v3
  BlockedWide,           // v4
  ThreadPerCombination,  // tpc
};
const char* variant_name(KernelVariant v);                 // kernels.cpp:107-116
KernelVariant variant_from_name(const std::string& name);  // kernels.cpp:118-125, DomainError
struct CacheSpec {
  std::size_t l1_bytes = 48 * 1024;
  std::uint32_t l1_ways = 12;
  std::uint32_t ft_ways = 7;
  std::uint32_t block_ways = 4;
  std::uint32_t count_bytes = 4;
};
struct BlockParams {
  std::uint32_t block_snps = 1;
  std::uint32_t block_samples = 1;
  std::uint32_t sched_edge = 256;
};
// kernels.cpp:136-169: the same sizing (and InfeasibleCache) as the reference,
// so reports print the same block=<B_S,B_P>.
BlockParams derive_block_params(const CacheSpec& cs, std::uint32_t lane_samples);
struct InstructionModel {
  std::uint32_t ops_per_element = 0;
  double relative_memory = 1.0;
};
InstructionModel instruction_count_model(KernelVariant v);  // kernels.cpp:127-134

// ---- search (search.hpp:13-89) ----------------------------------------------------------
struct SearchConfig {
  KernelVariant variant = KernelVariant::BlockedWide;  // accepted, no effect on the GPU
  BlockParams block;                                   // validated (search.cpp:133-135)
  unsigned threads = 1;                                // validated (search.cpp:130)
  std::uint32_t top_k = 10;
  std::uint64_t chunk = 1;                             // validated (search.cpp:132)
  int lanes = 8;                                       // accepted, no effect on the GPU
  std::vector<int> devices = {0};   // GPUs; the triple space is split in equal-work ranges
  std::uint64_t rank_begin = 0;     // lexicographic triple-rank range; [0, 0) = all triples
  std::uint64_t rank_end = 0;
};
struct Hit {
  double score = 0.0;
  Triple triple;
  friend bool operator==(const Hit&, const Hit&) = default;
};
inline bool hit_less(const Hit& a, const Hit& b) {
  if (a.score != b.score) return a.score < b.score;
  return a.triple < b.triple;
}
struct SearchStats {
  std::uint64_t combinations_evaluated = 0;
  double elapsed_seconds = 0.0;
  std::vector<std::uint64_t> per_thread_work;  // triples per GPU
  double kernel_ms = 0.0;                      // device time of the search kernels
};
struct SearchResult {
  Hit best{};
  std::vector<Hit> top;
  std::uint32_t top_k = 1;
  SearchStats stats;
};
bool same_outcome(const SearchResult& a, const SearchResult& b);
std::uint64_t num_combinations(std::uint64_t m, std::uint64_t k);
SearchResult run_search(const BitPlaneDataset& ds, const SearchConfig& cfg);
// Same search starting from a genotype matrix: validate + binarize run on each
// device (e3_dataset_create_genotypes) instead of the host.
SearchResult run_search(const GenotypeMatrix& m, const SearchConfig& cfg);
SearchResult reduce_results(std::span<const SearchResult> partials);

// ---- throughput report (bench.hpp:12-57; bench.cpp:10-107) ------------------------------
// elements = C(M,3) * N; the minimum over repeats; the same eleven fields.
struct BenchReport {
  KernelVariant variant = KernelVariant::BlockedWide;
  std::uint64_t num_snps = 0;
  std::uint64_t num_samples = 0;
  unsigned threads = 1;
  double elapsed_seconds = 0.0;
  std::uint64_t elements = 0;
  double elements_per_second = 0.0;
  double elements_per_second_per_thread = 0.0;
  std::uint32_t model_ops_per_element = 0;
  double model_bytes_per_element = 0.0;
  double arithmetic_intensity = 0.0;
  std::vector<double> repeat_seconds;
};
inline constexpr double kNaiveBytesPerElement = 9.0 / 8.0;
BenchReport make_report(KernelVariant variant, std::uint64_t num_snps, std::uint64_t num_samples,
                        unsigned threads, std::vector<double> repeat_seconds);
BenchReport measure(const BitPlaneDataset& ds, const SearchConfig& cfg, unsigned repeats);
enum class ReportFormat { csv, json };
std::string emit_report(const BenchReport& report, ReportFormat format);

// ---- per-triple tables (kernels.hpp:75) -----------------------------------------------
FrequencyTable freq_table_reduced(const BitPlaneDataset& ds, Triple t);

// A dataset resident on one GPU, for repeated searches/table queries.
class DeviceDataset {
 public:
  explicit DeviceDataset(const BitPlaneDataset& ds, int device = 0);
  // validate + binarize on the device (same dataset as from binarize(m))
  explicit DeviceDataset(const GenotypeMatrix& m, int device = 0);
  ~DeviceDataset();
  DeviceDataset(const DeviceDataset&) = delete;
  DeviceDataset& operator=(const DeviceDataset&) = delete;
  // engine: 0 auto, else E3_ENGINE_POPC / _TC_MASKED / _SYRK (identical results)
  SearchResult search(std::uint32_t top_k, std::uint64_t rank_begin = 0,
                      std::uint64_t rank_end = 0, int engine = 0) const;
  std::vector<FrequencyTable> tables(std::span<const Triple> triples) const;
  std::vector<double> scores(std::span<const Triple> triples) const;
  std::size_t num_snps() const { return m_; }

 private:
  e3_dataset* h_ = nullptr;
  std::size_t m_ = 0;
};

int device_count();

}  // namespace epi3
