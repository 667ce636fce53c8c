// epi3_api.cpp — the C++ drop-in API (include/epi3/api.hpp) over the C ABI.
// Every computation crosses epi3cu.h; this layer only adapts types, maps
// status codes to the epi3::Error hierarchy and fans a search out over GPUs.
#include "epi3/api.hpp"

#include <algorithm>
#include <chrono>
#include <cstdio>
#include <fstream>
#include <sstream>
#include <limits>
#include <thread>

#include "epi3cu.h"

namespace epi3 {

namespace {

[[noreturn]] void raise(int rc) {
  const std::string msg = e3_last_error();
  switch (rc) {
    case E3_DOMAIN: throw DomainError(msg);
    case E3_DIMENSION: throw DimensionError(msg);
    case E3_INDEX: throw IndexError(msg);
    case E3_PARSE: throw ParseError(msg);
    case E3_MAGIC: throw MagicMismatch(msg);
    case E3_TRUNCATED: throw TruncatedFile(msg);
    case E3_CUDA:
    case E3_NCCL:
    case E3_OOM: throw DeviceError(msg);
    default: throw Error(msg);
  }
}

void check(int rc) {
  if (rc != E3_OK) raise(rc);
}

std::size_t words_for(std::size_t n) { return (n + kWordBits - 1) / kWordBits; }

SearchResult from_hits(const std::vector<e3_hit>& hits, std::uint32_t n, std::uint32_t top_k,
                       const e3_stats& st) {
  SearchResult r;
  r.top_k = top_k;
  for (std::uint32_t x = 0; x < n; ++x)
    r.top.push_back(Hit{hits[x].score, Triple{hits[x].i0, hits[x].i1, hits[x].i2}});
  r.best = r.top.empty() ? Hit{} : r.top.front();
  r.stats.combinations_evaluated = st.combinations;
  r.stats.elapsed_seconds = st.elapsed_s;
  r.stats.per_thread_work = {st.combinations};
  r.stats.kernel_ms = st.total_device_ms;
  return r;
}

}  // namespace

std::string to_string(const Triple& t) {
  return "(" + std::to_string(t.i0) + "," + std::to_string(t.i1) + "," + std::to_string(t.i2) + ")";
}

// ---- data model --------------------------------------------------------------
const GenotypeMatrix& validate(const GenotypeMatrix& m) {
  if (m.num_snps < 3) throw DimensionError("need at least 3 SNPs, got " + std::to_string(m.num_snps));
  if (m.num_samples == 0) throw DimensionError("dataset has no samples");
  if (m.genotypes.size() != m.num_snps * m.num_samples)
    throw DimensionError("genotype storage does not match dimensions");
  if (m.phenotype.size() != m.num_samples)
    throw DimensionError("phenotype storage does not match dimensions");
  std::uint64_t n0 = 0, n1 = 0;
  check(e3_binarize(m.num_snps, m.num_samples, m.genotypes.data(), m.phenotype.data(), &n0, &n1,
                    nullptr, nullptr));
  for (std::size_t i = 0; i < m.num_snps; ++i)
    for (std::size_t j = 0; j < m.num_samples; ++j)
      if (m.geno(i, j) > 2)
        throw DomainError("genotype value " + std::to_string(m.geno(i, j)) + " at snp " +
                          std::to_string(i) + ", sample " + std::to_string(j));
  return m;
}

BitPlaneDataset::BitPlaneDataset(std::size_t num_snps, std::size_t n0, std::size_t n1)
    : m_(num_snps), n_{n0, n1}, w_{words_for(n0), words_for(n1)} {
  if (n0 > 0xffffffffull || n1 > 0xffffffffull)
    throw DomainError("class sample count exceeds the 32-bit cell cap");
  for (int c = 0; c < 2; ++c) data_[c].assign(m_ * 2 * w_[c], 0);
}

word BitPlaneDataset::pad_mask(int cls) const {
  const std::size_t rem = n_[cls] % kWordBits;
  return rem == 0 ? ~word{0} : (word{1} << rem) - 1;
}

std::uint8_t BitPlaneDataset::geno_at(int cls, snp_index snp, std::size_t pos) const {
  const word bit = word{1} << (pos % kWordBits);
  if (plane(cls, snp, 0)[pos / kWordBits] & bit) return 0;
  if (plane(cls, snp, 1)[pos / kWordBits] & bit) return 1;
  return 2;
}

BitPlaneDataset binarize(const GenotypeMatrix& m) {
  if (m.genotypes.size() != m.num_snps * m.num_samples || m.phenotype.size() != m.num_samples)
    throw DimensionError("genotype storage does not match dimensions");
  std::uint64_t n0 = 0, n1 = 0;
  check(e3_binarize(m.num_snps, m.num_samples, m.genotypes.data(), m.phenotype.data(), &n0, &n1,
                    nullptr, nullptr));
  BitPlaneDataset ds(m.num_snps, n0, n1);
  check(e3_binarize(m.num_snps, m.num_samples, m.genotypes.data(), m.phenotype.data(), &n0, &n1,
                    ds.data(0).data(), ds.data(1).data()));
  return ds;
}

GenotypeMatrix decode(const BitPlaneDataset& ds) {
  GenotypeMatrix m;
  m.num_snps = ds.num_snps();
  m.num_samples = ds.num_samples();
  m.genotypes.resize(m.num_snps * m.num_samples);
  m.phenotype.assign(m.num_samples, 0);
  std::fill(m.phenotype.begin() + std::ptrdiff_t(ds.num_controls()), m.phenotype.end(), 1);
  for (std::size_t i = 0; i < m.num_snps; ++i) {
    for (std::size_t j = 0; j < ds.num_controls(); ++j) m.geno(i, j) = ds.geno_at(0, snp_index(i), j);
    for (std::size_t j = 0; j < ds.num_cases(); ++j)
      m.geno(i, ds.num_controls() + j) = ds.geno_at(1, snp_index(i), j);
  }
  return m;
}

GenotypeMatrix generate_synthetic(std::size_t num_snps, std::size_t num_samples, double maf,
                                  std::uint64_t seed, const std::optional<PlantSpec>& plant,
                                  std::int64_t exact_cases) {
  GenotypeMatrix m;
  m.num_snps = num_snps;
  m.num_samples = num_samples;
  m.genotypes.resize(num_snps * num_samples);
  m.phenotype.resize(num_samples);
  e3_plant p{};
  if (plant) {
    p.i0 = plant->triple.i0;
    p.i1 = plant->triple.i1;
    p.i2 = plant->triple.i2;
    for (int k = 0; k < 3; ++k) p.target[k] = plant->target[k];
    p.p_case_match = plant->p_case_match;
    p.p_case_other = plant->p_case_other;
  }
  check(e3_generate_synthetic(num_snps, num_samples, maf, seed, plant ? &p : nullptr, exact_cases,
                              m.genotypes.data(), m.phenotype.data()));
  return m;
}

// ---- formats -------------------------------------------------------------------
BitPlaneDataset read_packed(const std::filesystem::path& path) {
  std::uint64_t M = 0, n0 = 0, n1 = 0;
  check(e3_packed_header(path.c_str(), &M, &n0, &n1));
  BitPlaneDataset ds(M, n0, n1);
  check(e3_read_packed(path.c_str(), M, n0, n1, ds.data(0).data(), ds.data(1).data()));
  return ds;
}

void write_packed(const std::filesystem::path& path, const BitPlaneDataset& ds) {
  check(e3_write_packed(path.c_str(), ds.num_snps(), ds.num_controls(), ds.num_cases(),
                        ds.data(0).data(), ds.data(1).data()));
}

bool is_packed_file(const std::filesystem::path& path) {
  std::ifstream in(path, std::ios::binary);
  char head[4] = {};
  in.read(head, 4);
  return in.gcount() == 4 && std::string(head, 4) == "EPI3";
}

// Text format (io.hpp:11-15): "#SNPS=<M> SAMPLES=<N>", M genotype rows, 1 phenotype row.
GenotypeMatrix read_text(const std::filesystem::path& path) {
  std::ifstream in(path);
  if (!in) throw Error("cannot open " + path.string());
  std::string line;
  std::size_t lineno = 1;
  if (!std::getline(in, line)) throw ParseError("missing header line (at 1)");
  GenotypeMatrix m;
  int used = -1;
  if (std::sscanf(line.c_str(), "#SNPS=%zu SAMPLES=%zu%n", &m.num_snps, &m.num_samples, &used) != 2 ||
      used < 0 || line.c_str()[used] != '\0')
    throw ParseError("malformed header, expected '#SNPS=<M> SAMPLES=<N>' (at 1)");
  m.genotypes.resize(m.num_snps * m.num_samples);
  m.phenotype.resize(m.num_samples);
  auto row = [&](std::uint8_t* dst, char maxc) {
    ++lineno;
    if (!std::getline(in, line)) throw ParseError("unexpected end of file (at " + std::to_string(lineno) + ")");
    std::istringstream s(line);
    std::string tok;
    for (std::size_t j = 0; j < m.num_samples; ++j) {
      if (!(s >> tok)) throw ParseError("too few values on line (at " + std::to_string(lineno) + ")");
      if (tok.size() != 1 || tok[0] < '0' || tok[0] > maxc)
        throw ParseError("invalid token '" + tok + "' (at " + std::to_string(lineno) + ")");
      dst[j] = std::uint8_t(tok[0] - '0');
    }
    if (s >> tok) throw ParseError("trailing values on line (at " + std::to_string(lineno) + ")");
  };
  for (std::size_t i = 0; i < m.num_snps; ++i) row(m.genotypes.data() + i * m.num_samples, '2');
  row(m.phenotype.data(), '1');
  return validate(m);
}

void write_text(const std::filesystem::path& path, const GenotypeMatrix& m) {
  validate(m);
  std::ofstream out(path);
  if (!out) throw Error("cannot open " + path.string() + " for writing");
  out << "#SNPS=" << m.num_snps << " SAMPLES=" << m.num_samples << '\n';
  auto row = [&](const std::uint8_t* r) {
    for (std::size_t j = 0; j < m.num_samples; ++j) out << (j ? " " : "") << int(r[j]);
    out << '\n';
  };
  for (std::size_t i = 0; i < m.num_snps; ++i) row(m.genotypes.data() + i * m.num_samples);
  row(m.phenotype.data());
  if (!out) throw Error("write failed");
}

// ---- scoring --------------------------------------------------------------------
std::uint64_t FrequencyTable::class_total(int cls) const {
  std::uint64_t t = 0;
  for (int c = 0; c < 27; ++c) t += at(c, cls);
  return t;
}

LogSumTable build_log_table(std::size_t n_max) {
  LogSumTable t;
  t.prefix.resize(n_max + 1);
  check(e3_build_log_table(n_max, t.prefix.data()));
  return t;
}

double k2_score(const FrequencyTable& ft, const LogSumTable& logs) {
  return e3_k2_score(ft.counts.data(), logs.prefix.data());
}

// ---- search -----------------------------------------------------------------------
bool same_outcome(const SearchResult& a, const SearchResult& b) {
  return a.best == b.best && a.top == b.top &&
         a.stats.combinations_evaluated == b.stats.combinations_evaluated;
}

std::uint64_t num_combinations(std::uint64_t m, std::uint64_t k) {
  std::uint64_t out = 0;
  check(e3_num_combinations(m, k, &out));
  return out;
}

int device_count() {
  int n = 0;
  check(e3_device_count(&n));
  return n;
}

DeviceDataset::DeviceDataset(const BitPlaneDataset& ds, int device) : m_(ds.num_snps()) {
  check(e3_dataset_create(ds.num_snps(), ds.num_controls(), ds.num_cases(), ds.data(0).data(),
                          ds.data(1).data(), device, &h_));
}

DeviceDataset::DeviceDataset(const GenotypeMatrix& m, int device) : m_(m.num_snps) {
  if (m.genotypes.size() != m.num_snps * m.num_samples || m.phenotype.size() != m.num_samples)
    throw DimensionError("genotype matrix size does not match its dimensions");
  check(e3_dataset_create_genotypes(m.num_snps, m.num_samples, m.genotypes.data(),
                                    m.phenotype.data(), device, &h_));
}

DeviceDataset::~DeviceDataset() { e3_dataset_destroy(h_); }

SearchResult DeviceDataset::search(std::uint32_t top_k, std::uint64_t r0, std::uint64_t r1,
                                   int engine) const {
  e3_search_cfg cfg{top_k, std::uint32_t(engine), r0, r1};
  std::vector<e3_hit> hits(std::max<std::uint32_t>(1, top_k));
  std::uint32_t n = 0;
  e3_stats st{};
  check(e3_search(h_, &cfg, hits.data(), &n, &st));
  return from_hits(hits, n, top_k, st);
}

std::vector<FrequencyTable> DeviceDataset::tables(std::span<const Triple> triples) const {
  std::vector<std::uint32_t> flat;
  for (const Triple& t : triples) flat.insert(flat.end(), {t.i0, t.i1, t.i2});
  std::vector<FrequencyTable> out(triples.size());
  std::vector<std::uint32_t> buf(54 * triples.size());
  check(e3_tables(h_, flat.data(), triples.size(), buf.data()));
  for (std::size_t x = 0; x < triples.size(); ++x)
    std::copy(buf.begin() + std::ptrdiff_t(54 * x), buf.begin() + std::ptrdiff_t(54 * x + 54),
              out[x].counts.begin());
  return out;
}

std::vector<double> DeviceDataset::scores(std::span<const Triple> triples) const {
  std::vector<std::uint32_t> flat;
  for (const Triple& t : triples) flat.insert(flat.end(), {t.i0, t.i1, t.i2});
  std::vector<double> out(triples.size());
  check(e3_scores(h_, flat.data(), triples.size(), out.data()));
  return out;
}

SearchResult reduce_results(std::span<const SearchResult> partials) {
  SearchResult out;
  out.best = Hit{std::numeric_limits<double>::infinity(), Triple{}};
  std::vector<e3_hit> all;
  for (const SearchResult& p : partials) {
    out.top_k = std::max(out.top_k, p.top_k);
    if (hit_less(p.best, out.best)) out.best = p.best;
    for (const Hit& h : p.top) all.push_back(e3_hit{h.score, h.triple.i0, h.triple.i1, h.triple.i2, 0});
    out.stats.combinations_evaluated += p.stats.combinations_evaluated;
    out.stats.elapsed_seconds += p.stats.elapsed_seconds;
    out.stats.kernel_ms = std::max(out.stats.kernel_ms, p.stats.kernel_ms);
    out.stats.per_thread_work.insert(out.stats.per_thread_work.end(),
                                     p.stats.per_thread_work.begin(), p.stats.per_thread_work.end());
  }
  std::vector<e3_hit> merged(std::max<std::size_t>(1, out.top_k));
  std::uint32_t n = 0;
  check(e3_merge_hits(all.data(), all.size(), out.top_k, merged.data(), &n));
  out.top.clear();
  for (std::uint32_t x = 0; x < n; ++x)
    out.top.push_back(Hit{merged[x].score, Triple{merged[x].i0, merged[x].i1, merged[x].i2}});
  return out;
}

namespace {
// The body of run_search over any dataset source: one host thread per GPU,
// each building its replicated DeviceDataset and searching an equal-work
// triple-rank range; partials merged by reduce_results.
template <typename Source>
SearchResult run_search_impl(const Source& src, std::size_t num_snps, const SearchConfig& cfg) {
  // argument checks in the reference's order and wording (search.cpp:128-135)
  if (num_snps < 3) throw DimensionError("search needs at least 3 SNPs");
  if (cfg.threads < 1) throw DomainError("threads must be >= 1");
  if (cfg.top_k < 1) throw DomainError("top_k must be >= 1");
  if (cfg.chunk < 1) throw DomainError("chunk must be >= 1");
  if (cfg.block.block_snps < 1 || cfg.block.block_samples < 1)
    throw DomainError("block parameters must be positive");
  if (cfg.block.sched_edge < 1) throw DomainError("sched edge must be positive");
  if (cfg.devices.empty()) throw DomainError("at least one device is required");
  const auto t0 = std::chrono::steady_clock::now();
  const std::uint64_t total = num_combinations(num_snps, 3);
  const std::uint64_t r0 = cfg.rank_begin;
  const std::uint64_t r1 = cfg.rank_end == 0 ? total : cfg.rank_end;
  if (r1 > total || r0 > r1) throw IndexError("triple-rank range outside [0, C(M,3))");
  const std::size_t G = cfg.devices.size();
  std::vector<std::uint64_t> bal(G + 1);
  check(e3_partition_balanced(num_snps, std::uint32_t(G), bal.data()));
  std::vector<SearchResult> partials(G);
  std::vector<std::exception_ptr> failures(G);
  auto worker = [&](std::size_t g) {
    try {
      // whole searches split by measured device cost (e3_partition_balanced),
      // sub-ranges by triple count
      std::uint64_t a = r0 + (r1 - r0) * g / G, b = r0 + (r1 - r0) * (g + 1) / G;
      if (r0 == 0 && r1 == total) {
        a = bal[g];
        b = bal[g + 1];
      }
      DeviceDataset dd(src, cfg.devices[g]);
      partials[g] = a < b ? dd.search(cfg.top_k, a, b) : SearchResult{};
      partials[g].top_k = cfg.top_k;
      if (a == b) partials[g].best = Hit{std::numeric_limits<double>::infinity(), Triple{}};
    } catch (...) {
      failures[g] = std::current_exception();
    }
  };
  if (G == 1) {
    worker(0);
  } else {
    std::vector<std::thread> pool;
    for (std::size_t g = 0; g < G; ++g) pool.emplace_back(worker, g);
    for (auto& t : pool) t.join();
  }
  for (auto& f : failures)
    if (f) std::rethrow_exception(f);
  SearchResult r = reduce_results(partials);
  r.top_k = cfg.top_k;
  r.stats.elapsed_seconds =
      std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
  return r;
}
}  // namespace

// run_search (search.cpp:127-250): one host thread per GPU, each with a
// replicated dataset and an equal-work triple-rank range; partials merged by
// reduce_results exactly as the reference merges its worker partials.
SearchResult run_search(const BitPlaneDataset& ds, const SearchConfig& cfg) {
  return run_search_impl(ds, ds.num_snps(), cfg);
}

SearchResult run_search(const GenotypeMatrix& m, const SearchConfig& cfg) {
  return run_search_impl(m, m.num_snps, cfg);
}

// ---- variants, CPU tiling knobs, bench report -------------------------------------
const char* variant_name(KernelVariant v) {
  switch (v) {
    case KernelVariant::NaivePhenotype: return "v1";
    case KernelVariant::ReducedSplit: return "v2";
    case KernelVariant::Blocked: return "v3";
    case KernelVariant::BlockedWide: return "v4";
    case KernelVariant::ThreadPerCombination: return "tpc";
  }
  return "?";
}

KernelVariant variant_from_name(const std::string& name) {
  static const std::pair<const char*, KernelVariant> names[] = {
      {"v1", KernelVariant::NaivePhenotype}, {"v2", KernelVariant::ReducedSplit},
      {"v3", KernelVariant::Blocked}, {"v4", KernelVariant::BlockedWide},
      {"tpc", KernelVariant::ThreadPerCombination}};
  for (const auto& [n, v] : names)
    if (name == n) return v;
  throw DomainError("unknown kernel variant '" + name + "'");
}

InstructionModel instruction_count_model(KernelVariant v) {
  // the reference's analytic model (kernels.cpp:127-134): 6 ops per combination
  // per element for v1, 3 NOR + 2 per combination for the reduced forms
  if (v == KernelVariant::NaivePhenotype) return {27 * 6, 1.0};
  return {3 + 2 * 27, 2.0 / 3.0};
}

BlockParams derive_block_params(const CacheSpec& cs, std::uint32_t lane_samples) {
  if (cs.l1_bytes == 0 || cs.l1_ways == 0 || cs.ft_ways == 0 || cs.block_ways == 0 ||
      cs.count_bytes == 0)
    throw DomainError("cache spec fields must be positive");
  if (cs.ft_ways + cs.block_ways > cs.l1_ways)
    throw DomainError("frequency-table and block ways exceed the cache ways");
  if (lane_samples == 0) throw DomainError("lane_samples must be positive");
  const std::size_t ft_budget = cs.l1_bytes * cs.ft_ways / cs.l1_ways;
  const std::size_t blk_budget = cs.l1_bytes * cs.block_ways / cs.l1_ways;
  // largest B_S with B_S^3 tables of 54 cells in the table ways
  const std::size_t tables = ft_budget / (std::size_t{2} * kNumCombos * cs.count_bytes);
  std::uint64_t bs = 0;
  while ((bs + 1) * (bs + 1) * (bs + 1) <= tables) ++bs;
  if (bs < 1)
    throw InfeasibleCache("frequency-table budget of " + std::to_string(ft_budget) +
                          " B cannot hold one table");
  // B_P: a multiple of lane_samples with B_S * B_P * 2 cells in the block ways
  const std::uint64_t bp = blk_budget / (bs * 2 * cs.count_bytes) / lane_samples * lane_samples;
  if (bp < lane_samples)
    throw InfeasibleCache("block budget of " + std::to_string(blk_budget) +
                          " B cannot hold one lane of samples");
  BlockParams p;
  p.block_snps = std::uint32_t(bs);
  p.block_samples = std::uint32_t(bp);
  return p;
}

BenchReport make_report(KernelVariant variant, std::uint64_t num_snps, std::uint64_t num_samples,
                        unsigned threads, std::vector<double> repeat_seconds) {
  if (repeat_seconds.empty()) throw DomainError("need at least one repeat");
  if (threads == 0) throw DomainError("threads must be >= 1");
  BenchReport r;
  r.variant = variant;
  r.num_snps = num_snps;
  r.num_samples = num_samples;
  r.threads = threads;
  r.repeat_seconds = std::move(repeat_seconds);
  r.elapsed_seconds = *std::min_element(r.repeat_seconds.begin(), r.repeat_seconds.end());
  const unsigned __int128 el = (unsigned __int128)num_combinations(num_snps, 3) * num_samples;
  if (el > std::numeric_limits<std::uint64_t>::max())
    throw DomainError("element count exceeds 64 bits");
  r.elements = std::uint64_t(el);
  r.elements_per_second = double(r.elements) / r.elapsed_seconds;
  r.elements_per_second_per_thread = r.elements_per_second / threads;
  const InstructionModel im = instruction_count_model(variant);
  r.model_ops_per_element = im.ops_per_element;
  r.model_bytes_per_element = kNaiveBytesPerElement * im.relative_memory;
  r.arithmetic_intensity = double(im.ops_per_element) / r.model_bytes_per_element;
  return r;
}

BenchReport measure(const BitPlaneDataset& ds, const SearchConfig& cfg, unsigned repeats) {
  if (repeats < 1) throw DomainError("repeats must be >= 1");
  std::vector<double> secs;
  SearchResult first;
  for (unsigned r = 0; r < repeats; ++r) {
    SearchResult res = run_search(ds, cfg);
    if (r == 0) first = res;
    else if (!same_outcome(first, res)) throw Error("search outcome changed between repeats");
    secs.push_back(res.stats.elapsed_seconds);
  }
  return make_report(cfg.variant, ds.num_snps(), ds.num_samples(), cfg.threads, std::move(secs));
}

namespace {
std::string g17(double v) {
  char b[64];
  std::snprintf(b, sizeof b, "%.17g", v);
  return b;
}
}  // namespace

std::string emit_report(const BenchReport& r, ReportFormat format) {
  if (format == ReportFormat::csv)
    return "variant,M,N,threads,elapsed_s,elements,eps,eps_per_thread,model_ops,model_bytes,ai\n" +
           std::string(variant_name(r.variant)) + ',' + std::to_string(r.num_snps) + ',' +
           std::to_string(r.num_samples) + ',' + std::to_string(r.threads) + ',' +
           g17(r.elapsed_seconds) + ',' + std::to_string(r.elements) + ',' +
           g17(r.elements_per_second) + ',' + g17(r.elements_per_second_per_thread) + ',' +
           std::to_string(r.model_ops_per_element) + ',' + g17(r.model_bytes_per_element) + ',' +
           g17(r.arithmetic_intensity) + '\n';
  std::string rep;
  for (std::size_t i = 0; i < r.repeat_seconds.size(); ++i)
    rep += (i ? ",\n    " : "\n    ") + g17(r.repeat_seconds[i]);
  return "{\n  \"variant\": \"" + std::string(variant_name(r.variant)) + "\",\n  \"M\": " +
         std::to_string(r.num_snps) + ",\n  \"N\": " + std::to_string(r.num_samples) +
         ",\n  \"threads\": " + std::to_string(r.threads) + ",\n  \"elapsed_s\": " +
         g17(r.elapsed_seconds) + ",\n  \"elements\": " + std::to_string(r.elements) +
         ",\n  \"eps\": " + g17(r.elements_per_second) + ",\n  \"eps_per_thread\": " +
         g17(r.elements_per_second_per_thread) + ",\n  \"model_ops\": " +
         std::to_string(r.model_ops_per_element) + ",\n  \"model_bytes\": " +
         g17(r.model_bytes_per_element) + ",\n  \"ai\": " + g17(r.arithmetic_intensity) +
         ",\n  \"repeats_s\": [" + rep + (rep.empty() ? "" : "\n  ") + "]\n}\n";
}

FrequencyTable freq_table_reduced(const BitPlaneDataset& ds, Triple t) {
  DeviceDataset dd(ds);
  const Triple one[1] = {t};
  return dd.tables(one).front();
}

}  // namespace epi3
