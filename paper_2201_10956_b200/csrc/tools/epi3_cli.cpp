// epi3_cli — `generate | detect | verify | bench` on the B200 engine, through
// the C++ drop-in API only (include/epi3/api.hpp). Output lines and exit codes
// follow the reference CLI (tools/epi3_main.cpp): detect prints
// "best (i,j,k) k2=%.9f" and the top list (161-176); Domain/Dimension errors
// exit 2, anything else 1 (407-419).
#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <map>
#include <string>
#include <vector>

#include "epi3/api.hpp"

using namespace epi3;

namespace {

struct Args {
  std::map<std::string, std::string> kv;
  bool has(const std::string& k) const { return kv.count(k) != 0; }
  std::string get(const std::string& k, const std::string& d = "") const {
    auto it = kv.find(k);
    return it == kv.end() ? d : it->second;
  }
  std::uint64_t num(const std::string& k, std::uint64_t d) const {
    return has(k) ? std::strtoull(get(k).c_str(), nullptr, 10) : d;
  }
};

Args parse(int argc, char** argv, int from) {
  Args a;
  for (int i = from; i < argc; ++i) {
    std::string k = argv[i];
    if (k.rfind("--", 0) != 0) throw DomainError("unexpected argument '" + k + "'");
    k = k.substr(2);
    if (k == "json") { a.kv[k] = "1"; continue; }
    if (i + 1 >= argc) throw DomainError("missing value for --" + k);
    a.kv[k] = argv[++i];
  }
  return a;
}

std::vector<int> devices(const Args& a) {
  const int n = int(a.num("gpus", 1));
  if (n < 1) throw DomainError("--gpus must be >= 1");
  std::vector<int> d(n);
  for (int i = 0; i < n; ++i) d[i] = i;
  return d;
}

BitPlaneDataset load(const std::string& path) {
  if (is_packed_file(path)) return read_packed(path);
  return binarize(read_text(path));
}

int cmd_generate(const Args& a) {
  const std::size_t M = a.num("snps", 0), N = a.num("samples", 0);
  const double maf = std::strtod(a.get("maf", "0.3").c_str(), nullptr);
  std::optional<PlantSpec> plant;
  if (a.has("plant")) {
    PlantSpec p;
    if (std::sscanf(a.get("plant").c_str(), "%u,%u,%u", &p.triple.i0, &p.triple.i1,
                    &p.triple.i2) != 3)
      throw DomainError("--plant expects i,j,k");
    p.p_case_other = std::strtod(a.get("p-other", "0.1").c_str(), nullptr);
    plant = p;
  }
  const std::int64_t cases = a.has("cases") ? std::int64_t(a.num("cases", 0)) : -1;
  const GenotypeMatrix m = generate_synthetic(M, N, maf, a.num("seed", 1), plant, cases);
  if (a.get("format", "packed") == "text") write_text(a.get("out"), m);
  else write_packed(a.get("out"), binarize(m));
  const auto n1 = std::count(m.phenotype.begin(), m.phenotype.end(), std::uint8_t{1});
  std::printf("wrote %s: snps=%zu samples=%zu controls=%zu cases=%zu\n", a.get("out").c_str(), M,
              N, std::size_t(N - n1), std::size_t(n1));
  return 0;
}

int cmd_detect(const Args& a) {
  // packed input: the bit planes go to the GPU as they are; text input: the
  // genotype matrix is validated and binarized on the GPU
  SearchConfig cfg;
  cfg.top_k = std::uint32_t(a.num("top-k", 10));
  cfg.devices = devices(a);
  struct Dims {
    std::size_t snps, samples, controls, cases;
    std::size_t num_snps() const { return snps; }
    std::size_t num_samples() const { return samples; }
    std::size_t num_controls() const { return controls; }
    std::size_t num_cases() const { return cases; }
  } ds{};
  SearchResult r;
  if (is_packed_file(a.get("in"))) {
    const BitPlaneDataset bp = read_packed(a.get("in"));
    ds = {bp.num_snps(), bp.num_samples(), bp.num_controls(), bp.num_cases()};
    r = run_search(bp, cfg);
  } else {
    const GenotypeMatrix gm = read_text(a.get("in"));
    validate(gm);
    const auto n1 = std::size_t(std::count(gm.phenotype.begin(), gm.phenotype.end(), std::uint8_t{1}));
    ds = {gm.num_snps, gm.num_samples, gm.num_samples - n1, n1};
    r = run_search(gm, cfg);
  }
  if (a.has("json")) {
    std::printf("{\"input\": \"%s\", \"snps\": %zu, \"samples\": %zu, \"controls\": %zu, "
                "\"cases\": %zu, \"engine\": \"b200\", \"gpus\": %zu, \"best\": {\"score\": %.17g, "
                "\"triple\": [%u, %u, %u]}, \"top\": [",
                a.get("in").c_str(), ds.num_snps(), ds.num_samples(), ds.num_controls(),
                ds.num_cases(), cfg.devices.size(), r.best.score, r.best.triple.i0,
                r.best.triple.i1, r.best.triple.i2);
    for (std::size_t i = 0; i < r.top.size(); ++i)
      std::printf("%s{\"score\": %.17g, \"triple\": [%u, %u, %u]}", i ? ", " : "", r.top[i].score,
                  r.top[i].triple.i0, r.top[i].triple.i1, r.top[i].triple.i2);
    std::printf("], \"stats\": {\"combinations\": %llu, \"elapsed_s\": %.6f}}\n",
                (unsigned long long)r.stats.combinations_evaluated, r.stats.elapsed_seconds);
    return 0;
  }
  std::printf("dataset %s: snps=%zu samples=%zu controls=%zu cases=%zu\n", a.get("in").c_str(),
              ds.num_snps(), ds.num_samples(), ds.num_controls(), ds.num_cases());
  std::printf("engine=b200 gpus=%zu\n", cfg.devices.size());
  std::printf("best %s k2=%.9f\n", to_string(r.best.triple).c_str(), r.best.score);
  std::printf("top %zu:\n", r.top.size());
  for (std::size_t i = 0; i < r.top.size(); ++i)
    std::printf("  %2zu. %s k2=%.9f\n", i + 1, to_string(r.top[i].triple).c_str(), r.top[i].score);
  std::printf("stats: combinations=%llu elapsed_s=%.3f\n",
              (unsigned long long)r.stats.combinations_evaluated, r.stats.elapsed_seconds);
  return 0;
}

// verify (epi3_main.cpp:185-292): GPU tables for every triple against a
// per-sample count written here, and the GPU best against a brute-force
// host search over those counts (capped like the reference oracle).
int cmd_verify(const Args& a) {
  const std::size_t cap = a.num("cap", 64);
  const BitPlaneDataset ds = load(a.get("in"));
  if (ds.num_snps() > cap)
    throw DomainError("verify is capped at " + std::to_string(cap) + " SNPs");
  const GenotypeMatrix m = decode(ds);
  std::vector<Triple> all;
  for (snp_index i = 0; i < ds.num_snps(); ++i)
    for (snp_index j = i + 1; j < ds.num_snps(); ++j)
      for (snp_index k = j + 1; k < ds.num_snps(); ++k) all.push_back({i, j, k});
  DeviceDataset dd(ds);
  const auto tables = dd.tables(all);
  const LogSumTable logs = build_log_table(ds.num_samples() + 1);
  bool tables_ok = true;
  Hit best{INFINITY, {}};
  for (std::size_t x = 0; x < all.size(); ++x) {
    FrequencyTable ft;
    for (std::size_t s = 0; s < m.num_samples; ++s)
      ++ft.at(combo_index(m.geno(all[x].i0, s), m.geno(all[x].i1, s), m.geno(all[x].i2, s)),
              m.phenotype[s]);
    if (!(ft == tables[x])) {
      if (tables_ok) std::printf("first mismatch at triple %s\n", to_string(all[x]).c_str());
      tables_ok = false;
    }
    const Hit h{k2_score(ft, logs), all[x]};
    if (hit_less(h, best)) best = h;
  }
  std::printf("%-28s %s\n", "b200 tables", tables_ok ? "PASS" : "FAIL");
  const SearchResult r = dd.search(1);
  const bool search_ok = r.best.triple == best.triple && r.best.score == best.score;
  std::printf("%-28s %s\n", "b200 search", search_ok ? "PASS" : "FAIL");
  if (!search_ok)
    std::printf("  host %s k2=%.9f, b200 %s k2=%.9f\n", to_string(best.triple).c_str(), best.score,
                to_string(r.best.triple).c_str(), r.best.score);
  return tables_ok && search_ok ? 0 : 1;
}

// bench (bench.cpp:10-107): elements = C(M,3)*N, minimum over repeats.
int cmd_bench(const Args& a) {
  const BitPlaneDataset ds = load(a.get("in"));
  const unsigned repeats = unsigned(a.num("repeats", 3));
  if (repeats < 1) throw DomainError("repeats must be >= 1");
  SearchConfig cfg;
  cfg.devices = devices(a);
  std::vector<double> secs;
  SearchResult first;
  for (unsigned r = 0; r < repeats; ++r) {
    const SearchResult res = run_search(ds, cfg);
    if (r == 0) first = res;
    else if (!same_outcome(first, res)) throw Error("search outcome changed between repeats");
    secs.push_back(res.stats.elapsed_seconds);
  }
  const double best = *std::min_element(secs.begin(), secs.end());
  const double elements = double(num_combinations(ds.num_snps(), 3)) * double(ds.num_samples());
  const double eps = elements / best;
  if (a.get("format", "csv") == "json") {
    std::printf("{\"variant\": \"b200\", \"M\": %zu, \"N\": %zu, \"gpus\": %zu, \"elapsed_s\": %.17g, "
                "\"elements\": %.17g, \"eps\": %.17g, \"eps_per_gpu\": %.17g, \"repeats_s\": [",
                ds.num_snps(), ds.num_samples(), cfg.devices.size(), best, elements, eps,
                eps / double(cfg.devices.size()));
    for (std::size_t i = 0; i < secs.size(); ++i) std::printf("%s%.17g", i ? ", " : "", secs[i]);
    std::printf("]}\n");
  } else {
    std::printf("variant,M,N,gpus,elapsed_s,elements,eps,eps_per_gpu\n");
    std::printf("b200,%zu,%zu,%zu,%.17g,%.17g,%.17g,%.17g\n", ds.num_snps(), ds.num_samples(),
                cfg.devices.size(), best, elements, eps, eps / double(cfg.devices.size()));
  }
  return 0;
}

}  // namespace

int main(int argc, char** argv) {
  if (argc < 2) {
    std::fprintf(stderr, "usage: epi3 generate|detect|verify|bench [--flags]\n");
    return 2;
  }
  try {
    const std::string cmd = argv[1];
    const Args a = parse(argc, argv, 2);
    if (cmd == "generate") return cmd_generate(a);
    if (cmd == "detect") return cmd_detect(a);
    if (cmd == "verify") return cmd_verify(a);
    if (cmd == "bench") return cmd_bench(a);
    std::fprintf(stderr, "unknown subcommand '%s'\n", cmd.c_str());
    return 2;
  } catch (const DomainError& e) {
    std::fprintf(stderr, "error: %s\n", e.what());
    return 2;
  } catch (const DimensionError& e) {
    std::fprintf(stderr, "error: %s\n", e.what());
    return 2;
  } catch (const std::exception& e) {
    std::fprintf(stderr, "error: %s\n", e.what());
    return 1;
  }
}
