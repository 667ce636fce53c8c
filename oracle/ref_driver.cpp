// ref_driver.cpp — our driver over the UNMODIFIED reference library.
//
// TEST INFRASTRUCTURE ONLY. oracle/Makefile compiles the reference sources in
// place (/root/reference/proj/src/*.cpp, never copied) together with this
// file into oracle/_ref/epi3_ref. It is the reference arm of bench.py
// (`--impl reference`) and the generator of tests/golden/ fixtures.
//
// Subcommands (all output is one JSON document on stdout):
//   gen    M N maf seed out.epi3 [i0 i1 i2 t0 t1 t2 p_match p_other]
//          generate_synthetic (src/datamodel.cpp:179) -> binarize (69) ->
//          write_packed (src/io.cpp:176)
//   search file.epi3 variant threads top_k repeats
//          read_packed (src/io.cpp:117) -> run_search (src/search.cpp:127)
//          with make_config's block params (tools/epi3_main.cpp:107-120)
//   tables file.epi3 i0 i1 i2 [i0 i1 i2 ...]
//          freq_table_reduced (src/kernels.cpp:200)
//   logk2  n_max  c0..c53
//          build_log_table + k2_score (src/scoring.cpp:14-35)
#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <string>
#include <vector>

#include "epi3/bitplane.hpp"
#include "epi3/io.hpp"
#include "epi3/kernels.hpp"
#include "epi3/scoring.hpp"
#include "epi3/search.hpp"
#include "epi3/synthetic.hpp"

using namespace epi3;

namespace {

void print_hit(const Hit& h) {
  std::printf("{\"score\": %.17g, \"hex\": \"%a\", \"triple\": [%u, %u, %u]}", h.score,
              h.score, h.triple.i0, h.triple.i1, h.triple.i2);
}

int cmd_gen(int argc, char** argv) {
  if (argc != 7 && argc != 15) return 2;
  const std::size_t M = std::strtoull(argv[2], nullptr, 10);
  const std::size_t N = std::strtoull(argv[3], nullptr, 10);
  const double maf = std::strtod(argv[4], nullptr);
  const std::uint64_t seed = std::strtoull(argv[5], nullptr, 10);
  std::optional<PlantSpec> plant;
  if (argc == 15) {
    PlantSpec p;
    p.triple = {snp_index(std::atoi(argv[7])), snp_index(std::atoi(argv[8])),
                snp_index(std::atoi(argv[9]))};
    p.target = {std::uint8_t(std::atoi(argv[10])), std::uint8_t(std::atoi(argv[11])),
                std::uint8_t(std::atoi(argv[12]))};
    p.p_case_match = std::strtod(argv[13], nullptr);
    p.p_case_other = std::strtod(argv[14], nullptr);
    plant = p;
  }
  const GenotypeMatrix m = generate_synthetic(M, N, maf, seed, plant);
  const BitPlaneDataset ds = binarize(m);
  write_packed(argv[6], ds);
  std::printf("{\"snps\": %zu, \"controls\": %zu, \"cases\": %zu}\n", ds.num_snps(),
              ds.num_controls(), ds.num_cases());
  return 0;
}

int cmd_search(int argc, char** argv) {
  if (argc != 7) return 2;
  const BitPlaneDataset ds = read_packed(argv[2]);
  SearchConfig cfg;
  cfg.variant = variant_from_name(argv[3]);
  cfg.block = derive_block_params(CacheSpec{}, 16);
  cfg.block.sched_edge = 256;
  if (cfg.variant == KernelVariant::ThreadPerCombination) cfg.block.block_snps = 64;
  cfg.threads = unsigned(std::atoi(argv[4]));
  cfg.top_k = std::uint32_t(std::atoi(argv[5]));
  cfg.lanes = 8;
  const int repeats = std::max(1, std::atoi(argv[6]));
  std::vector<double> secs;
  SearchResult first;
  for (int r = 0; r < repeats; ++r) {
    SearchResult res = run_search(ds, cfg);
    if (r == 0) first = res;
    else if (!same_outcome(first, res)) {
      std::fprintf(stderr, "outcome changed between repeats\n");
      return 1;
    }
    secs.push_back(res.stats.elapsed_seconds);
  }
  std::printf("{\"snps\": %zu, \"controls\": %zu, \"cases\": %zu, \"variant\": \"%s\", "
              "\"threads\": %u, \"block\": [%u, %u], \"combinations\": %llu, \"best\": ",
              ds.num_snps(), ds.num_controls(), ds.num_cases(), variant_name(cfg.variant),
              cfg.threads, cfg.block.block_snps, cfg.block.block_samples,
              (unsigned long long)first.stats.combinations_evaluated);
  print_hit(first.best);
  std::printf(", \"top\": [");
  for (std::size_t i = 0; i < first.top.size(); ++i) {
    if (i) std::printf(", ");
    print_hit(first.top[i]);
  }
  std::printf("], \"elapsed_s\": [");
  for (std::size_t i = 0; i < secs.size(); ++i) std::printf("%s%.9g", i ? ", " : "", secs[i]);
  std::printf("]}\n");
  return 0;
}

int cmd_tables(int argc, char** argv) {
  if (argc < 6 || (argc - 3) % 3 != 0) return 2;
  const BitPlaneDataset ds = read_packed(argv[2]);
  std::printf("{\"tables\": [");
  for (int a = 3; a < argc; a += 3) {
    const Triple t{snp_index(std::atoi(argv[a])), snp_index(std::atoi(argv[a + 1])),
                   snp_index(std::atoi(argv[a + 2]))};
    const FrequencyTable ft = freq_table_reduced(ds, t);
    std::printf("%s[", a > 3 ? ", " : "");
    for (std::size_t c = 0; c < ft.counts.size(); ++c)
      std::printf("%s%u", c ? ", " : "", ft.counts[c]);
    std::printf("]");
  }
  std::printf("]}\n");
  return 0;
}

int cmd_logk2(int argc, char** argv) {
  if (argc != 3 + 54) return 2;
  const LogSumTable logs = build_log_table(std::strtoull(argv[2], nullptr, 10));
  FrequencyTable ft;
  for (int c = 0; c < 54; ++c) ft.counts[c] = std::uint32_t(std::strtoul(argv[3 + c], nullptr, 10));
  const double s = k2_score(ft, logs);
  std::printf("{\"k2\": %.17g, \"hex\": \"%a\", \"prefix_last\": \"%a\"}\n", s, s,
              logs.prefix.back());
  return 0;
}

}  // namespace

int main(int argc, char** argv) {
  if (argc < 2) {
    std::fprintf(stderr, "usage: epi3_ref gen|search|tables|logk2 ...\n");
    return 2;
  }
  try {
    const std::string cmd = argv[1];
    int rc = 2;
    if (cmd == "gen") rc = cmd_gen(argc, argv);
    else if (cmd == "search") rc = cmd_search(argc, argv);
    else if (cmd == "tables") rc = cmd_tables(argc, argv);
    else if (cmd == "logk2") rc = cmd_logk2(argc, argv);
    if (rc == 2) std::fprintf(stderr, "bad arguments for %s\n", cmd.c_str());
    return rc;
  } catch (const std::exception& e) {
    std::fprintf(stderr, "error: %s\n", e.what());
    return 1;
  }
}
