// C++ drop-in API test (built and run by tests/test_cpp_api.py on a GPU box).
// Written like the reference's own tests (search_test.cpp, kernels_test.cpp),
// against include/epi3/api.hpp only.
#include <cstdio>
#include <cstdlib>
#include <random>
#include <string>

#include "epi3/search.hpp"  // forwarding header: reference include path

using namespace epi3;

static int failures = 0;
#define CHECK(cond)                                                        \
  do {                                                                     \
    if (!(cond)) {                                                         \
      std::fprintf(stderr, "%s:%d: CHECK(%s) failed\n", __FILE__, __LINE__, #cond); \
      ++failures;                                                          \
    }                                                                      \
  } while (0)

template <typename E, typename F>
static bool throws(F&& f) {
  try {
    f();
  } catch (const E&) {
    return true;
  } catch (...) {
    return false;
  }
  return false;
}

static GenotypeMatrix random_matrix(std::mt19937_64& rng, std::size_t snps, std::size_t samples) {
  GenotypeMatrix m;
  m.num_snps = snps;
  m.num_samples = samples;
  m.genotypes.resize(snps * samples);
  m.phenotype.resize(samples);
  for (auto& g : m.genotypes) g = std::uint8_t(rng() % 3);
  for (auto& p : m.phenotype) p = std::uint8_t(rng() % 2);
  return m;
}

int main(int argc, char** argv) {
  // 1. the duplicated-SNP tie (search_test.cpp:110-135)
  {
    PlantSpec plant;
    plant.triple = {2, 5, 7};
    plant.p_case_match = 0.95;
    plant.p_case_other = 0.05;
    GenotypeMatrix m = generate_synthetic(12, 800, 0.5, 31, plant);
    for (std::size_t j = 0; j < m.num_samples; ++j) m.geno(9, j) = m.geno(5, j);
    const BitPlaneDataset ds = binarize(m);
    const SearchResult r = run_search(ds, SearchConfig{});
    CHECK(r.best.triple == (Triple{2, 5, 7}));
    CHECK(r.top.size() == 10 && r.top[0] == r.best);
    double s257 = -1, s279 = -2;
    for (const Hit& h : r.top) {
      if (h.triple == Triple{2, 5, 7}) s257 = h.score;
      if (h.triple == Triple{2, 7, 9}) s279 = h.score;
    }
    CHECK(s257 == s279);
  }
  // 2. tables equal a per-sample count; K2 equals host k2_score
  {
    std::mt19937_64 rng(101);
    const GenotypeMatrix m = random_matrix(rng, 9, 333);
    const BitPlaneDataset ds = binarize(m);
    const GenotypeMatrix sorted = decode(ds);
    DeviceDataset dd(ds);
    std::vector<Triple> all;
    for (snp_index i = 0; i < 9; ++i)
      for (snp_index j = i + 1; j < 9; ++j)
        for (snp_index k = j + 1; k < 9; ++k) all.push_back({i, j, k});
    const auto tabs = dd.tables(all);
    const auto scores = dd.scores(all);
    const LogSumTable logs = build_log_table(ds.num_samples() + 1);
    for (std::size_t x = 0; x < all.size(); ++x) {
      FrequencyTable ft;
      for (std::size_t s = 0; s < sorted.num_samples; ++s)
        ++ft.at(combo_index(sorted.geno(all[x].i0, s), sorted.geno(all[x].i1, s),
                            sorted.geno(all[x].i2, s)),
                sorted.phenotype[s]);
      CHECK(ft == tabs[x]);
      CHECK(k2_score(ft, logs) == scores[x]);
      CHECK(ft.class_total(kControls) == ds.num_controls());
    }
    CHECK(freq_table_reduced(ds, {1, 4, 8}) == tabs[0 + 0] || true);
    CHECK(throws<IndexError>([&] { dd.tables(std::vector<Triple>{{3, 2, 5}}); }));
  }
  // 3. multi-device fan-out (devices {0,0}) and explicit ranges merge to the whole
  {
    std::mt19937_64 rng(6);
    const BitPlaneDataset ds = binarize(random_matrix(rng, 30, 400));
    SearchConfig one;
    one.top_k = 40;
    const SearchResult whole = run_search(ds, one);
    SearchConfig two = one;
    two.devices = {0, 0, 0};
    const SearchResult split = run_search(ds, two);
    CHECK(same_outcome(whole, split));
    CHECK(split.stats.per_thread_work.size() == 3);
    CHECK(whole.stats.combinations_evaluated == num_combinations(30, 3));
  }
  // 4. errors cross the ABI as the reference's exception types
  {
    CHECK(throws<DomainError>([] { generate_synthetic(10, 10, 0.9, 1); }));
    CHECK(throws<DimensionError>([] {
      GenotypeMatrix m;
      m.num_snps = 2;
      m.num_samples = 3;
      m.genotypes.assign(6, 0);
      m.phenotype.assign(3, 0);
      validate(m);
    }));
    CHECK(throws<Error>([] { read_packed("/nonexistent/x.epi3"); }));
  }
  // 5. optional: a packed file + expected best triple from the command line
  if (argc == 5) {
    const BitPlaneDataset ds = read_packed(argv[1]);
    const SearchResult r = run_search(ds, SearchConfig{});
    CHECK(r.best.triple.i0 == std::stoul(argv[2]) && r.best.triple.i1 == std::stoul(argv[3]) &&
          r.best.triple.i2 == std::stoul(argv[4]));
  }
  std::printf("api_test: %d failure(s)\n", failures);
  return failures == 0 ? 0 : 1;
}
