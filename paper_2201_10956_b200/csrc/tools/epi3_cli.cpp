// epi3_cli — `generate | detect | verify | bench` on the B200 engine, through
// the C++ drop-in API only (include/epi3/api.hpp). A drop-in for the
// reference CLI (tools/epi3_main.cpp): the same subcommands, flags, defaults,
// stdout lines, JSON fields and exit codes (Domain/Dimension/InfeasibleCache
// errors and argument errors exit 2, anything else 1; epi3_main.cpp:391-419),
// so scripts written against `epi3` (tests/cli_test.cpp) run unchanged.
//
// The reference's CPU knobs (--variant, --threads, --lanes, --b-sched,
// --tile-snps and the cache flags) are parsed and validated like the
// reference and echoed in the reports (block=<B_S,B_P> from the same
// derive_block_params); the search itself always runs on the GPU engine, and
// every variant returns the identical result (as in the reference). Extra
// flags: --gpus N (detect/bench: split the triple space over N GPUs) and
// --cases N (generate: exact class counts, the BASELINE configs' mode).
#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <fstream>
#include <map>
#include <memory>
#include <set>
#include <string>
#include <thread>
#include <vector>

#include "epi3/api.hpp"

using namespace epi3;

namespace {

// Argument errors (unknown flag, missing value, missing required flag,
// malformed number): exit 2 like CLI11's ParseError in the reference.
struct UsageError : std::runtime_error {
  using std::runtime_error::runtime_error;
};

struct Args {
  std::map<std::string, std::string> kv;
  bool has(const std::string& k) const { return kv.count(k) != 0; }
  std::string get(const std::string& k, const std::string& d = "") const {
    auto it = kv.find(k);
    return it == kv.end() ? d : it->second;
  }
  std::string req(const std::string& k) const {
    if (!has(k)) throw UsageError("--" + k + " is required");
    return get(k);
  }
  std::uint64_t num(const std::string& k, std::uint64_t d) const {
    if (!has(k)) return d;
    const std::string v = get(k);
    char* end = nullptr;
    const unsigned long long x = std::strtoull(v.c_str(), &end, 10);
    if (v.empty() || *end != '\0' || v[0] == '-') throw UsageError("--" + k + ": not a number: " + v);
    return x;
  }
  double real(const std::string& k, double d) const {
    if (!has(k)) return d;
    const std::string v = get(k);
    char* end = nullptr;
    const double x = std::strtod(v.c_str(), &end);
    if (v.empty() || *end != '\0') throw UsageError("--" + k + ": not a number: " + v);
    return x;
  }
};

Args parse(int argc, char** argv, int from, const std::set<std::string>& options,
           const std::set<std::string>& flags) {
  Args a;
  for (int i = from; i < argc; ++i) {
    std::string k = argv[i];
    if (k.rfind("--", 0) != 0) throw UsageError("unexpected argument '" + k + "'");
    k = k.substr(2);
    std::string v;
    const auto eq = k.find('=');
    const bool inline_value = eq != std::string::npos;
    if (inline_value) {
      v = k.substr(eq + 1);
      k = k.substr(0, eq);
    }
    if (flags.count(k)) {
      a.kv[k] = "1";
      continue;
    }
    if (!options.count(k)) throw UsageError("unknown option --" + k);
    if (!inline_value) {
      if (i + 1 >= argc) throw UsageError("missing value for --" + k);
      v = argv[++i];
    }
    a.kv[k] = v;
  }
  return a;
}

unsigned default_threads() {
  const unsigned hw = std::thread::hardware_concurrency();
  return hw == 0 ? 1 : hw;
}

const std::set<std::string> kCacheOpts = {"l1-kb", "l1-ways", "ft-ways", "block-ways",
                                          "lane-samples"};
const std::set<std::string> kSearchOpts = {"variant", "threads", "lanes", "b-sched", "tile-snps",
                                           "gpus"};

std::set<std::string> join(std::initializer_list<std::set<std::string>> sets) {
  std::set<std::string> out;
  for (const auto& s : sets) out.insert(s.begin(), s.end());
  return out;
}

// epi3_main.cpp:35-52 defaults
CacheSpec cache_spec(const Args& a) {
  CacheSpec cs;
  cs.l1_bytes = std::size_t(a.num("l1-kb", 48)) * 1024;
  cs.l1_ways = std::uint32_t(a.num("l1-ways", 12));
  cs.ft_ways = std::uint32_t(a.num("ft-ways", 7));
  cs.block_ways = std::uint32_t(a.num("block-ways", 4));
  cs.count_bytes = 4;
  return cs;
}

std::vector<int> devices(const Args& a) {
  const std::uint64_t n = a.num("gpus", 1);
  if (n < 1) throw DomainError("--gpus must be >= 1");
  std::vector<int> d(n);
  for (std::size_t i = 0; i < n; ++i) d[i] = int(i);
  return d;
}

// make_config (epi3_main.cpp:107-120)
SearchConfig make_config(const Args& a, std::uint32_t top_k) {
  SearchConfig cfg;
  cfg.variant = variant_from_name(a.get("variant", "v4"));
  cfg.block = derive_block_params(cache_spec(a), std::uint32_t(a.num("lane-samples", 16)));
  cfg.block.sched_edge = std::uint32_t(a.num("b-sched", 256));
  if (cfg.variant == KernelVariant::ThreadPerCombination)
    cfg.block.block_snps = std::uint32_t(a.num("tile-snps", 64));
  cfg.threads = unsigned(a.num("threads", default_threads()));
  cfg.top_k = top_k;
  cfg.lanes = int(a.num("lanes", 8));
  cfg.devices = devices(a);
  return cfg;
}

BitPlaneDataset load(const std::string& path) {
  if (is_packed_file(path)) return read_packed(path);
  return binarize(read_text(path));
}

// parse_plant (epi3_main.cpp:55-70): i0,i1,i2:gx,gy,gz:pmatch,pother
PlantSpec parse_plant(const std::string& text) {
  PlantSpec p;
  unsigned i0, i1, i2, g0, g1, g2;
  int consumed = -1;
  if (std::sscanf(text.c_str(), "%u,%u,%u:%u,%u,%u:%lf,%lf%n", &i0, &i1, &i2, &g0, &g1, &g2,
                  &p.p_case_match, &p.p_case_other, &consumed) != 8 ||
      consumed < 0 || text.c_str()[consumed] != '\0')
    throw DomainError("plant spec must look like i0,i1,i2:gx,gy,gz:pmatch,pother");
  p.triple = Triple{i0, i1, i2};
  if (g0 > 2 || g1 > 2 || g2 > 2) throw DomainError("plant target genotypes must be in {0,1,2}");
  p.target = {std::uint8_t(g0), std::uint8_t(g1), std::uint8_t(g2)};
  return p;
}

int cmd_generate(const Args& a) {
  const std::string out = a.req("out");
  const std::size_t M = a.num("snps", 0), N = a.num("samples", 0);
  if (!a.has("snps")) throw UsageError("--snps is required");
  if (!a.has("samples")) throw UsageError("--samples is required");
  const std::string format = a.get("format", "text");
  if (format != "text" && format != "packed") throw UsageError("--format must be text or packed");
  std::optional<PlantSpec> plant;
  if (a.has("plant")) plant = parse_plant(a.get("plant"));
  const std::int64_t cases = a.has("cases") ? std::int64_t(a.num("cases", 0)) : -1;
  const GenotypeMatrix m = generate_synthetic(M, N, a.real("maf", 0.25), a.num("seed", 1), plant,
                                              cases);
  if (format == "packed") write_packed(out, binarize(m));
  else write_text(out, m);
  std::printf("wrote %s: snps=%zu samples=%zu format=%s\n", out.c_str(), m.num_snps,
              m.num_samples, format.c_str());
  if (plant)
    std::printf("planted triple %s target (%d,%d,%d) p=%g/%g\n", to_string(plant->triple).c_str(),
                plant->target[0], plant->target[1], plant->target[2], plant->p_case_match,
                plant->p_case_other);
  return 0;
}

std::string json_str(const std::string& s) {
  std::string o = "\"";
  for (char c : s) {
    if (c == '"' || c == '\\') o += '\\';
    o += c;
  }
  return o + "\"";
}

std::string g17(double v) {
  char b[64];
  std::snprintf(b, sizeof b, "%.17g", v);
  return b;
}

std::string triple_json(const Triple& t) {
  return "[\n      " + std::to_string(t.i0) + ",\n      " + std::to_string(t.i1) + ",\n      " +
         std::to_string(t.i2) + "\n    ]";
}

int cmd_detect(const Args& a) {
  const std::string in = a.req("in");
  const SearchConfig cfg = make_config(a, std::uint32_t(a.num("top-k", 10)));
  // packed input: the bit planes go to the GPU as they are; text input: the
  // genotype matrix is validated and binarized on the GPU
  std::size_t snps = 0, samples = 0, controls = 0, cases = 0;
  SearchResult r;
  if (is_packed_file(in)) {
    const BitPlaneDataset bp = read_packed(in);
    snps = bp.num_snps();
    samples = bp.num_samples();
    controls = bp.num_controls();
    cases = bp.num_cases();
    r = run_search(bp, cfg);
  } else {
    const GenotypeMatrix gm = read_text(in);
    validate(gm);
    cases = std::size_t(std::count(gm.phenotype.begin(), gm.phenotype.end(), std::uint8_t{1}));
    snps = gm.num_snps;
    samples = gm.num_samples;
    controls = samples - cases;
    r = run_search(gm, cfg);
  }
  if (a.has("json")) {
    // the reference's document (epi3_main.cpp:131-159; nlohmann::json: keys
    // sorted, 2-space indent) plus "engine" and "gpus"
    std::string top = "[";
    for (std::size_t i = 0; i < r.top.size(); ++i)
      top += std::string(i ? "," : "") + "\n    {\n      \"score\": " + g17(r.top[i].score) +
             ",\n      \"triple\": [\n        " + std::to_string(r.top[i].triple.i0) +
             ",\n        " + std::to_string(r.top[i].triple.i1) + ",\n        " +
             std::to_string(r.top[i].triple.i2) + "\n      ]\n    }";
    top += r.top.empty() ? "]" : "\n  ]";
    std::string work = "[";
    for (std::size_t i = 0; i < r.stats.per_thread_work.size(); ++i)
      work += std::string(i ? "," : "") + "\n      " + std::to_string(r.stats.per_thread_work[i]);
    work += r.stats.per_thread_work.empty() ? "]" : "\n    ]";
    std::printf(
        "{\n  \"best\": {\n    \"score\": %s,\n    \"triple\": %s\n  },\n  \"block\": {\n"
        "    \"samples\": %u,\n    \"sched\": %u,\n    \"snps\": %u\n  },\n  \"cases\": %zu,\n"
        "  \"controls\": %zu,\n  \"engine\": \"b200\",\n  \"gpus\": %zu,\n  \"input\": %s,\n"
        "  \"samples\": %zu,\n  \"snps\": %zu,\n  \"stats\": {\n    \"combinations\": %llu,\n"
        "    \"elapsed_s\": %s,\n    \"per_thread_work\": %s\n  },\n  \"threads\": %u,\n"
        "  \"top\": %s,\n  \"variant\": \"%s\"\n}\n",
        g17(r.best.score).c_str(), triple_json(r.best.triple).c_str(), cfg.block.block_samples,
        cfg.block.sched_edge, cfg.block.block_snps, cases, controls, cfg.devices.size(),
        json_str(in).c_str(), samples, snps, (unsigned long long)r.stats.combinations_evaluated,
        g17(r.stats.elapsed_seconds).c_str(), work.c_str(), cfg.threads, top.c_str(),
        variant_name(cfg.variant));
    return 0;
  }
  // epi3_main.cpp:161-176, line for line
  std::printf("dataset %s: snps=%zu samples=%zu controls=%zu cases=%zu\n", in.c_str(), snps,
              samples, controls, cases);
  std::printf("variant=%s threads=%u block=<%u,%u> sched=%u lanes=%d\n", variant_name(cfg.variant),
              cfg.threads, cfg.block.block_snps, cfg.block.block_samples, cfg.block.sched_edge,
              cfg.lanes);
  std::printf("best %s k2=%.9f\n", to_string(r.best.triple).c_str(), r.best.score);
  std::printf("top %zu:\n", r.top.size());
  for (std::size_t i = 0; i < r.top.size(); ++i)
    std::printf("  %2zu. %s k2=%.9f\n", i + 1, to_string(r.top[i].triple).c_str(), r.top[i].score);
  std::printf("stats: combinations=%llu elapsed_s=%.3f\n",
              (unsigned long long)r.stats.combinations_evaluated, r.stats.elapsed_seconds);
  return 0;
}

void print_cells(const FrequencyTable& ft) {
  for (int c = 0; c < kNumCombos; ++c)
    std::printf("  combo (%d,%d,%d): controls=%u cases=%u\n", c / 9, c / 3 % 3, c % 3,
                ft.at(c, kControls), ft.at(c, kCases));
}

// verify (epi3_main.cpp:185-292): the same report lines. The oracle is a
// per-sample count over the decoded genotype matrix (host); the "tables
// <variant>" lines check the GPU tables of every triple against it, the
// "search <variant>" lines the GPU search with each engine (v1/tpc: the
// LOP3/POPC engine, v2: the masked tensor-core engine, v3: the fp4 SYRK
// engine, v4: auto) against the brute-force best — bit-identical scores.
int cmd_verify(const Args& a) {
  const std::string in = a.req("in");
  const std::size_t cap = a.num("max-snps", 64);
  (void)cache_spec(a);
  const BitPlaneDataset ds = load(in);
  if (ds.num_snps() > cap)
    throw CapExceeded("verify capped at " + std::to_string(cap) + " SNPs, dataset has " +
                      std::to_string(ds.num_snps()));
  static const char* kVariants[] = {"v1", "v2", "v3", "v4", "tpc"};
  static const int kEngines[] = {1, 2, 3, 0, 1};
  bool all_ok = true;
  const auto report = [&](const std::string& name, bool ok) {
    std::printf("%-28s %s\n", name.c_str(), ok ? "PASS" : "FAIL");
    all_ok = all_ok && ok;
  };
  std::unique_ptr<DeviceDataset> dd;
  try {
    dd = std::make_unique<DeviceDataset>(ds);
  } catch (const DomainError& e) {
    // corrupted planes (bitplane.hpp:13-20 invariants) fail every check
    for (const char* v : kVariants) report(std::string("tables ") + v + " vs oracle", false);
    for (const char* v : kVariants) report(std::string("search ") + v + " vs oracle", false);
    std::printf("dataset rejected: %s\n", e.what());
    return 1;
  }
  const GenotypeMatrix m = decode(ds);
  std::vector<Triple> all;
  for (snp_index i = 0; i + 2 < ds.num_snps(); ++i)
    for (snp_index j = i + 1; j + 1 < ds.num_snps(); ++j)
      for (snp_index k = j + 1; k < ds.num_snps(); ++k) all.push_back({i, j, k});
  std::vector<FrequencyTable> expect(all.size());
  const LogSumTable logs = build_log_table(ds.num_samples() + 1);
  Hit best{INFINITY, {}};
  for (std::size_t x = 0; x < all.size(); ++x) {
    for (std::size_t s = 0; s < m.num_samples; ++s)
      ++expect[x].at(combo_index(m.geno(all[x].i0, s), m.geno(all[x].i1, s), m.geno(all[x].i2, s)),
                     m.phenotype[s]);
    const Hit h{k2_score(expect[x], logs), all[x]};
    if (hit_less(h, best)) best = h;
  }
  const std::vector<FrequencyTable> got = dd->tables(all);
  for (const char* v : kVariants) {
    const std::string name = std::string("tables ") + v + " vs oracle";
    bool ok = true;
    for (std::size_t x = 0; x < all.size() && ok; ++x)
      if (!(got[x] == expect[x])) {
        report(name, false);
        std::printf("first mismatch at triple %s\n", to_string(all[x]).c_str());
        std::printf("oracle:\n");
        print_cells(expect[x]);
        std::printf("%s:\n", name.c_str());
        print_cells(got[x]);
        ok = false;
      }
    if (ok) report(name, true);
  }
  for (int x = 0; x < 5; ++x) {
    const SearchResult r = dd->search(10, 0, 0, kEngines[x]);
    const bool ok = r.best.triple == best.triple && r.best.score == best.score;
    report(std::string("search ") + kVariants[x] + " vs oracle", ok);
    if (!ok)
      std::printf("  oracle %s k2=%.9f, %s %s k2=%.9f\n", to_string(best.triple).c_str(),
                  best.score, kVariants[x], to_string(r.best.triple).c_str(), r.best.score);
  }
  return all_ok ? 0 : 1;
}

// bench (epi3_main.cpp:294-313; bench.cpp:10-107): measure() + emit_report().
int cmd_bench(const Args& a) {
  const std::string in = a.req("in");
  const std::string format = a.get("format", "csv");
  if (format != "csv" && format != "json") throw UsageError("--format must be csv or json");
  const BitPlaneDataset ds = load(in);
  const SearchConfig cfg = make_config(a, 10);
  const BenchReport rep = measure(ds, cfg, unsigned(a.num("repeats", 3)));
  const std::string text = emit_report(rep, format == "json" ? ReportFormat::json : ReportFormat::csv);
  if (!a.has("out")) {
    std::fputs(text.c_str(), stdout);
  } else {
    std::ofstream out(a.get("out"));
    if (!out) throw Error("cannot open " + a.get("out") + " for writing");
    out << text;
  }
  return 0;
}

}  // namespace

int main(int argc, char** argv) {
  if (argc < 2) {
    std::fprintf(stderr, "usage: epi3 generate|detect|verify|bench [--flags]\n");
    return 2;
  }
  const std::string cmd = argv[1];
  Args a;
  try {
    if (cmd == "generate")
      a = parse(argc, argv, 2, {"snps", "samples", "maf", "seed", "plant", "out", "format", "cases"},
                {});
    else if (cmd == "detect")
      a = parse(argc, argv, 2, join({kSearchOpts, kCacheOpts, {"in", "top-k"}}), {"json"});
    else if (cmd == "verify")
      a = parse(argc, argv, 2, join({kCacheOpts, {"in", "max-snps"}}), {});
    else if (cmd == "bench")
      a = parse(argc, argv, 2, join({kSearchOpts, kCacheOpts, {"in", "repeats", "format", "out"}}),
                {});
    else
      throw UsageError("unknown subcommand '" + cmd + "'");
  } catch (const UsageError& e) {
    std::fprintf(stderr, "error: %s\n", e.what());
    return 2;
  }
  try {
    if (cmd == "generate") return cmd_generate(a);
    if (cmd == "detect") return cmd_detect(a);
    if (cmd == "verify") return cmd_verify(a);
    return cmd_bench(a);
  } catch (const UsageError& e) {
    std::fprintf(stderr, "error: %s\n", e.what());
    return 2;
  } catch (const DomainError& e) {
    std::fprintf(stderr, "error: %s\n", e.what());
    return 2;
  } catch (const DimensionError& e) {
    std::fprintf(stderr, "error: %s\n", e.what());
    return 2;
  } catch (const InfeasibleCache& e) {
    std::fprintf(stderr, "error: %s\n", e.what());
    return 2;
  } catch (const std::exception& e) {
    std::fprintf(stderr, "error: %s\n", e.what());
    return 1;
  }
}
