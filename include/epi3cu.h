/*
 * epi3cu.h — C ABI of the B200-native exhaustive 3-way K2 epistasis engine.
 *
 * This is the drop-in boundary for the reference's hot path
 * (/root/reference/proj, paths below relative to it). Plain pointers and
 * sizes only; no CUDA or torch types cross it; exceptions never cross it —
 * every entry point returns an e3_status and e3_last_error() holds the
 * thread-local message, mirroring the epi3::Error hierarchy
 * (include/epi3/common.hpp:36-105). The C++ mirror of the reference API
 * (include/epi3/api.hpp in this repo) is implemented on top of these calls.
 *
 * Threading: calls on distinct datasets are independent and may run
 * concurrently; calls on one dataset (e3_search, e3_tables, e3_scores) are
 * serialised by a per-dataset mutex, so a dataset may be shared by host
 * threads like the reference's (immutable, shareable: SPEC.md:126-127).
 */
#ifndef EPI3CU_H
#define EPI3CU_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* Status codes, one per epi3::Error subclass (common.hpp:36-105). */
typedef enum {
  E3_OK = 0,
  E3_DOMAIN = 1,     /* DomainError     (common.hpp:43-61)  */
  E3_DIMENSION = 2,  /* DimensionError  (common.hpp:63-66)  */
  E3_INDEX = 3,      /* IndexError      (common.hpp:68-71)  */
  E3_PARSE = 4,      /* ParseError      (common.hpp:75-85)  */
  E3_MAGIC = 5,      /* MagicMismatch   (common.hpp:87-90)  */
  E3_TRUNCATED = 6,  /* TruncatedFile   (common.hpp:92-95)  */
  E3_IO = 7,         /* plain Error on open/write failure (src/io.cpp:37-47, 109, 199) */
  E3_CUDA = 10,      /* device error (no reference analogue: the reference has no device) */
  E3_NCCL = 11,
  E3_OOM = 12
} e3_status;

/* Opaque device-resident dataset: the BitPlaneDataset (include/epi3/bitplane.hpp:25-67)
 * repacked for the GPU plus its per-dataset marginal index (single and pair
 * plane counts). Immutable after creation. */
typedef struct e3_dataset e3_dataset;

/* One search hit == epi3::Hit (include/epi3/search.hpp:22-27); ordered by
 * hit_less (search.hpp:29-35): score ascending, then (i0,i1,i2). */
typedef struct {
  double score;
  uint32_t i0, i1, i2, _pad;
} e3_hit;

/* Search configuration. Replaces SearchConfig (search.hpp:13-20): variant,
 * block params, threads, chunk and lanes are CPU-tiling knobs with no GPU
 * meaning; top_k keeps its meaning (search.hpp:17). The triple-rank range is
 * new: the lexicographic rank of i0<i1<i2 within [0, C(M,3)); [0, C(M,3)) —
 * or rank_end == 0 — is the full search run_search performs (search.cpp:127). */
typedef struct {
  uint32_t top_k;       /* >= 1, <= E3_MAX_TOP_K */
  uint32_t flags;       /* engine: 0 = auto, else one of E3_ENGINE_* */
  uint64_t rank_begin;
  uint64_t rank_end;    /* 0 = C(M,3) */
} e3_search_cfg;

/* top_k <= 256 runs one pass (per-warp top-k lists in shared memory); a larger
 * top_k runs a second, collecting pass below a bound taken from the first
 * (exact; about twice the search time). */
#define E3_MAX_TOP_K 1048576u
/* Engine selection (e3_search_cfg.flags). All engines produce identical
 * results; 0 = auto (E3_ENGINE_SYRK for N >= 4096 samples with every class
 * < 2^23 samples, else E3_ENGINE_TC_MASKED).
 *   E3_ENGINE_POPC       LOP3/POPC kernel (marginal subtraction + carry-save)
 *   E3_ENGINE_TC_MASKED  tcgen05 kind::i8 GEMM: pair products x singles
 *   E3_ENGINE_SYRK       per-first-SNP sample compaction (two smaller genotype
 *                        phases) + tcgen05 kind::mxf4 SYRK on packed 0/1 E2M1
 *                        operands, fp32 K2 screen + exact fp64 K2; E3_DOMAIN
 *                        when a class holds >= 2^23 samples */
#define E3_ENGINE_POPC 1u
#define E3_ENGINE_TC_MASKED 2u
#define E3_ENGINE_SYRK 3u

/* Replaces SearchStats (search.hpp:37-41). */
typedef struct {
  uint64_t combinations;   /* triples evaluated, counted on the device triple by triple
                              (search.cpp:175 `++combos`); the call fails (E3_CUDA) unless
                              it equals rank_end - rank_begin */
  double elapsed_s;        /* host wall time of the call (SearchStats::elapsed_seconds) */
  double kernel_ms;        /* device time of the contingency+K2 kernel (CUDA events) */
  double total_device_ms;  /* device time of all kernels of the search */
  uint32_t kernel_launches;       /* all kernels of the search */
  uint32_t main_kernel_launches;  /* launches of the contingency+K2 kernel (SYRK: one per batch) */
} e3_stats;

/* ---- dataset load (replaces BitPlaneDataset construction: bitplane.hpp:30-31,
 *      read_packed io.hpp:27, binarize bitplane.hpp:72) ---------------------- */

/* ctrl: [M][2][ceil(N0/64)] u64 and cases: [M][2][ceil(N1/64)] u64 — exactly
 * BitPlaneDataset::data_[0] / data_[1] (bitplane.hpp:58-66); padding bits must
 * be zero and planes mutually exclusive (bitplane.hpp:13-20; checked, E3_DOMAIN).
 * Copies to `device` and builds the marginal index; caller keeps ownership. */
int e3_dataset_create(uint64_t M, uint64_t N0, uint64_t N1, const uint64_t* ctrl,
                      const uint64_t* cases, int device, e3_dataset** out);
/* validate (src/datamodel.cpp:28-46) + binarize (src/datamodel.cpp:69-92) on
 * the device: geno [M][N] u8 SNP-major in {0,1,2}, pheno [N] in {0,1}. Samples
 * are taken class-contiguous and stable (controls first) exactly like
 * binarize(), so the dataset equals e3_dataset_create over e3_binarize's
 * planes; E3_DOMAIN on an out-of-range genotype or phenotype. */
int e3_dataset_create_genotypes(uint64_t M, uint64_t N, const uint8_t* geno,
                                const uint8_t* pheno, int device, e3_dataset** out);
void e3_dataset_destroy(e3_dataset* ds);
int e3_dataset_info(const e3_dataset* ds, uint64_t* M, uint64_t* N0, uint64_t* N1,
                    int* device);

/* ---- search (replaces run_search, search.hpp:85 / search.cpp:127-250) ------ */
/* top: capacity cfg->top_k; *n_top = entries written (ascending, best == top[0]). */
int e3_search(const e3_dataset* ds, const e3_search_cfg* cfg, e3_hit* top,
              uint32_t* n_top, e3_stats* stats);

/* ---- per-triple tables and scores (replace freq_table_reduced,
 *      kernels.hpp:75 / kernels.cpp:200-212, and k2_score, scoring.hpp:59) --- */
/* triples: 3n u32, each i0<i1<i2<M (else E3_INDEX, kernels.cpp:12-18);
 * out: 54n u32, per triple [cls][gx*9+gy*3+gz] == FrequencyTable::counts. */
int e3_tables(const e3_dataset* ds, const uint32_t* triples, uint64_t n, uint32_t* out);
/* out: n doubles, bit-identical to k2_score(freq_table_reduced(t), build_log_table(N+1)). */
int e3_scores(const e3_dataset* ds, const uint32_t* triples, uint64_t n, double* out);

/* ---- host helpers on the same path (no device work) ------------------------ */
const char* e3_last_error(void);
int e3_device_count(int* count);
/* num_combinations (search.cpp:48-59); E3_DOMAIN when m<k or overflow. */
int e3_num_combinations(uint64_t m, uint64_t k, uint64_t* out);
/* Lexicographic triple rank <-> triple. */
int e3_triple_rank(uint64_t M, uint32_t i0, uint32_t i1, uint32_t i2, uint64_t* rank);
int e3_triple_unrank(uint64_t M, uint64_t rank, uint32_t* triple3);
/* Equal-work partition of [0, C(M,3)) into `parts` contiguous rank ranges
 * (the multi-GPU partitioner): bounds has parts+1 entries. */
int e3_partition(uint64_t M, uint32_t parts, uint64_t* bounds);
/* The same split balanced by measured device cost instead of triple count
 * (SYRK engine: a cost per 64x64 (j,k) tile plus a per-first-SNP cost): the
 * ranges the multi-GPU search uses (bench.py, run_search over devices). */
int e3_partition_balanced(uint64_t M, uint32_t parts, uint64_t* bounds);
/* build_log_table (scoring.cpp:14-21): prefix has n_max+1 doubles. */
int e3_build_log_table(uint64_t n_max, double* prefix);
/* k2_score (scoring.cpp:23-35) on the host, same grouping and order. */
double e3_k2_score(const uint32_t* table54, const double* prefix);
/* reduce_results' top merge (search.cpp:108-125): sort by hit_less, unique,
 * truncate to top_k. Returns the merged count in *n_out. */
int e3_merge_hits(const e3_hit* hits, uint64_t n, uint32_t top_k, e3_hit* out,
                  uint32_t* n_out);

/* validate (src/datamodel.cpp:28-46) + binarize (src/datamodel.cpp:69-92):
 * geno M*N SNP-major, pheno N. Call with ctrl/cases NULL to get N0/N1 first. */
int e3_binarize(uint64_t M, uint64_t N, const uint8_t* geno, const uint8_t* pheno,
                uint64_t* N0, uint64_t* N1, uint64_t* ctrl, uint64_t* cases);
/* generate_synthetic (src/datamodel.cpp:179-227) with the same mt19937_64
 * stream; plant may be NULL. exact_cases >= 0 additionally flips the labels
 * of non-matching samples (lowest index first) until exactly exact_cases
 * samples are cases — the exact-class-count mode the BASELINE configs need
 * (SURVEY.md §8(d)); -1 keeps the reference behaviour. */
typedef struct {
  uint32_t i0, i1, i2;
  uint8_t target[3];
  uint8_t _pad;
  double p_case_match, p_case_other;
} e3_plant;
int e3_generate_synthetic(uint64_t M, uint64_t N, double maf, uint64_t seed,
                          const e3_plant* plant, int64_t exact_cases, uint8_t* geno,
                          uint8_t* pheno);

/* Packed EPI3 v1 (include/epi3/io.hpp:20-25; src/io.cpp:117-203). */
int e3_packed_header(const char* path, uint64_t* M, uint64_t* N0, uint64_t* N1);
int e3_read_packed(const char* path, uint64_t M, uint64_t N0, uint64_t N1, uint64_t* ctrl,
                   uint64_t* cases);
int e3_write_packed(const char* path, uint64_t M, uint64_t N0, uint64_t N1,
                    const uint64_t* ctrl, const uint64_t* cases);

#ifdef __cplusplus
}
#endif
#endif /* EPI3CU_H */
