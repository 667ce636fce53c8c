/*
 * epi3_oracle.h — CPU restatement of the reference epi3 hot path.
 *
 * TEST INFRASTRUCTURE ONLY. This library is the parity checker for the CUDA
 * engine in paper_2201_10956_b200/. Only tests/, __graft_entry__.smoke() and
 * bench.py's cpu_baseline / --impl reference legs may load it, and only as
 * the checker or the timed CPU baseline — never as the thing measured or
 * shipped. The product path never links or calls it.
 *
 * Parity is pinned two ways:
 *   1. against the reference itself, compiled from /root/reference/proj/src
 *      into oracle/_ref/epi3_ref by oracle/Makefile (tests/golden/ fixtures
 *      are its outputs, made by tests/golden/make_golden.py);
 *   2. against the known-answer values the reference tests hold
 *      (scoring_test.cpp:29-67, kernels_test.cpp:131-194,
 *      search_test.cpp:32-41, 110-135, bench_test.cpp:17-27).
 *
 * Every function cites the reference file:line it restates
 * (paths relative to /root/reference/proj).
 */
#ifndef EPI3_ORACLE_H
#define EPI3_ORACLE_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* std::mt19937_64 (C++ [rand.predef]) — the generator the reference uses in
 * generate_synthetic (src/datamodel.cpp:210). */
typedef struct { uint64_t mt[312]; int idx; } eo_mt64;
void eo_mt64_seed(eo_mt64* g, uint64_t seed);
uint64_t eo_mt64_next(eo_mt64* g);

/* generate_synthetic (src/datamodel.cpp:179-227). geno is M*N SNP-major,
 * pheno is N. plant may be NULL (Bernoulli(0.5) phenotype). plant layout:
 * {i0,i1,i2,t0,t1,t2} plus probabilities. Returns 0 or -1 on a domain error. */
int eo_generate_synthetic(uint64_t M, uint64_t N, double maf, uint64_t seed,
                          const uint32_t* plant_triple, const uint8_t* plant_target,
                          double p_case_match, double p_case_other,
                          uint8_t* geno, uint8_t* pheno);

/* binarize (src/datamodel.cpp:69-92): class-contiguous stable reorder,
 * controls first; planes per class laid out [snp][plane g<2][word64]
 * (include/epi3/bitplane.hpp:58-66). ctrl must hold M*2*ceil(N0/64) words and
 * cases M*2*ceil(N1/64); both zeroed by this call. */
void eo_binarize(uint64_t M, uint64_t N, const uint8_t* geno, const uint8_t* pheno,
                 uint64_t N0, uint64_t N1, uint64_t* ctrl, uint64_t* cases);

/* freq_table_reduced (src/kernels.cpp:200-212) via accumulate_reduced
 * (src/kernels.cpp:30-53): per class, genotype-2 word inferred by NOR under
 * the final-word mask, 27 AND+POPCOUNT per word. out[54] = [cls][gx*9+gy*3+gz]. */
void eo_freq_table(uint64_t M, uint64_t N0, uint64_t N1, const uint64_t* ctrl,
                   const uint64_t* cases, uint32_t i0, uint32_t i1, uint32_t i2,
                   uint32_t* out);

/* build_log_table (src/scoring.cpp:14-21): prefix[n] = prefix[n-1] + log(n). */
void eo_build_log_table(uint64_t n_max, double* prefix /* n_max+1 */);

/* k2_score (src/scoring.cpp:23-35), exact grouping and order. */
double eo_k2_score(const uint32_t* table54, const double* prefix);

/* Hit ordering: hit_less (include/epi3/search.hpp:29-35). */
typedef struct { double score; uint32_t i0, i1, i2, pad; } eo_hit;
int eo_hit_less(const eo_hit* a, const eo_hit* b);

/* num_combinations(m,3) (src/search.cpp:48-59); 0 on overflow/m<3. */
uint64_t eo_num_triples(uint64_t m);
/* Lexicographic triple rank <-> triple over i0<i1<i2<M (our range contract;
 * the reference's run_search covers rank range [0, C(M,3)). */
uint64_t eo_triple_rank(uint64_t M, uint32_t i0, uint32_t i1, uint32_t i2);
void eo_triple_unrank(uint64_t M, uint64_t rank, uint32_t* t /* 3 */);

/* Exhaustive search over triple ranks [r0, r1): run_search semantics
 * (src/search.cpp:127-250) with TopBuffer (24-39) and reduce_results
 * (108-125): top is ascending under hit_less, at most top_k entries,
 * best == top[0]. threads <= 0 means all cores. Returns number of hits. */
uint32_t eo_search_range(uint64_t M, uint64_t N0, uint64_t N1, const uint64_t* ctrl,
                         const uint64_t* cases, uint64_t r0, uint64_t r1,
                         uint32_t top_k, int threads, eo_hit* top);

/* reduce_results (src/search.cpp:108-125) for top lists: concat, sort with
 * hit_less, unique, truncate. Returns the merged count written to out. */
uint32_t eo_merge_tops(const eo_hit* hits, uint32_t n, uint32_t top_k, eo_hit* out);

/* Packed EPI3 v1 format (src/io.cpp:117-169, 176-203; include/epi3/io.hpp:20-25). */
int eo_write_packed(const char* path, uint64_t M, uint64_t N0, uint64_t N1,
                    const uint64_t* ctrl, const uint64_t* cases);

#ifdef __cplusplus
}
#endif
#endif
