/*
 * epi3_oracle.c — CPU restatement of the reference epi3 hot path.
 *
 * TEST INFRASTRUCTURE ONLY (see epi3_oracle.h): the parity checker and the
 * "port" CPU baseline. The product (paper_2201_10956_b200/) never links it.
 * Parity of this restatement is pinned against the reference build in
 * oracle/_ref and the reference tests' known answers (tests/test_oracle.py).
 *
 * Citations are to /root/reference/proj.
 */
#include "epi3_oracle.h"

#include <math.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>
#include <pthread.h>
#include <unistd.h>

typedef unsigned __int128 u128;

/* ---- std::mt19937_64 (the standard's parameterisation) ------------------ */
#define MT_N 312
#define MT_M 156
#define MT_UPPER 0xFFFFFFFF80000000ULL
#define MT_LOWER 0x000000007FFFFFFFULL

void eo_mt64_seed(eo_mt64* g, uint64_t seed) {
  g->mt[0] = seed;
  for (int i = 1; i < MT_N; ++i)
    g->mt[i] = 6364136223846793005ULL * (g->mt[i - 1] ^ (g->mt[i - 1] >> 62)) + (uint64_t)i;
  g->idx = MT_N;
}

uint64_t eo_mt64_next(eo_mt64* g) {
  if (g->idx >= MT_N) {
    for (int i = 0; i < MT_N; ++i) {
      uint64_t x = (g->mt[i] & MT_UPPER) | (g->mt[(i + 1) % MT_N] & MT_LOWER);
      uint64_t xa = x >> 1;
      if (x & 1ULL) xa ^= 0xB5026F5AA96619E9ULL;
      g->mt[i] = g->mt[(i + MT_M) % MT_N] ^ xa;
    }
    g->idx = 0;
  }
  uint64_t y = g->mt[g->idx++];
  y ^= (y >> 29) & 0x5555555555555555ULL;
  y ^= (y << 17) & 0x71D67FFFEDA60000ULL;
  y ^= (y << 37) & 0xFFF7EEE000000000ULL;
  y ^= y >> 43;
  return y;
}

/* next_unit: src/datamodel.cpp:173-175 */
static double next_unit(eo_mt64* g) { return (double)(eo_mt64_next(g) >> 11) * 0x1.0p-53; }

/* generate_synthetic: src/datamodel.cpp:179-227 */
int eo_generate_synthetic(uint64_t M, uint64_t N, double maf, uint64_t seed,
                          const uint32_t* pt, const uint8_t* ptg, double pm, double po,
                          uint8_t* geno, uint8_t* pheno) {
  if (!(maf > 0.0 && maf <= 0.5) || M < 3 || N == 0) return -1;
  if (pt) {
    if (pt[0] == pt[1] || pt[0] == pt[2] || pt[1] == pt[2]) return -1;
    if (pt[0] >= M || pt[1] >= M || pt[2] >= M) return -1;
    if (ptg[0] > 2 || ptg[1] > 2 || ptg[2] > 2) return -1;
    if (!(pm >= 0.0 && pm <= 1.0 && po >= 0.0 && po <= 1.0) || !(pm > po)) return -1;
  }
  const double p0 = (1.0 - maf) * (1.0 - maf);
  const double p01 = p0 + 2.0 * maf * (1.0 - maf);
  eo_mt64 g;
  eo_mt64_seed(&g, seed);
  for (uint64_t i = 0; i < M; ++i)
    for (uint64_t j = 0; j < N; ++j) {
      const double u = next_unit(&g);
      geno[i * N + j] = u < p0 ? 0 : (u < p01 ? 1 : 2);
    }
  for (uint64_t j = 0; j < N; ++j) {
    double p_case = 0.5;
    if (pt) {
      const int match = geno[pt[0] * N + j] == ptg[0] && geno[pt[1] * N + j] == ptg[1] &&
                        geno[pt[2] * N + j] == ptg[2];
      p_case = match ? pm : po;
    }
    pheno[j] = next_unit(&g) < p_case ? 1 : 0;
  }
  return 0;
}

/* binarize: src/datamodel.cpp:69-92 (positions: 75-79; set bit: 22-24, 86-89) */
void eo_binarize(uint64_t M, uint64_t N, const uint8_t* geno, const uint8_t* pheno,
                 uint64_t N0, uint64_t N1, uint64_t* ctrl, uint64_t* cases) {
  const uint64_t w[2] = {(N0 + 63) / 64, (N1 + 63) / 64};
  memset(ctrl, 0, M * 2 * w[0] * 8);
  memset(cases, 0, M * 2 * w[1] * 8);
  uint64_t* data[2] = {ctrl, cases};
  uint64_t* pos = (uint64_t*)malloc(N * sizeof(uint64_t));
  uint64_t next[2] = {0, 0};
  for (uint64_t j = 0; j < N; ++j) pos[j] = next[pheno[j]]++;
  for (uint64_t i = 0; i < M; ++i)
    for (uint64_t j = 0; j < N; ++j) {
      const uint8_t gv = geno[i * N + j];
      const int c = pheno[j];
      if (gv < 2) data[c][(i * 2 + gv) * w[c] + pos[j] / 64] |= 1ULL << (pos[j] % 64);
    }
  free(pos);
}

/* accumulate_reduced: src/kernels.cpp:30-53 (full range, final-word mask) */
static void accumulate_reduced(const uint64_t* x0, const uint64_t* x1, const uint64_t* y0,
                               const uint64_t* y1, const uint64_t* z0, const uint64_t* z1,
                               uint64_t nw, uint64_t mask, uint32_t* acc) {
  for (uint64_t w = 0; w < nw; ++w) {
    const uint64_t m = (w + 1 == nw) ? mask : ~0ULL;
    const uint64_t xs[3] = {x0[w], x1[w], ~(x0[w] | x1[w]) & m};
    const uint64_t ys[3] = {y0[w], y1[w], ~(y0[w] | y1[w]) & m};
    const uint64_t zs[3] = {z0[w], z1[w], ~(z0[w] | z1[w]) & m};
    int c = 0;
    for (int gx = 0; gx < 3; ++gx)
      for (int gy = 0; gy < 3; ++gy) {
        const uint64_t xy = xs[gx] & ys[gy];
        for (int gz = 0; gz < 3; ++gz) acc[c++] += (uint32_t)__builtin_popcountll(xy & zs[gz]);
      }
  }
}

/* words_for / tail_mask: src/datamodel.cpp:13-20 */
static uint64_t tail_mask(uint64_t n) {
  const uint64_t rem = n % 64;
  return rem == 0 ? ~0ULL : ((1ULL << rem) - 1);
}

/* freq_table_reduced: src/kernels.cpp:200-212 */
void eo_freq_table(uint64_t M, uint64_t N0, uint64_t N1, const uint64_t* ctrl,
                   const uint64_t* cases, uint32_t i0, uint32_t i1, uint32_t i2, uint32_t* out) {
  (void)M;
  memset(out, 0, 54 * sizeof(uint32_t));
  const uint64_t n[2] = {N0, N1};
  const uint64_t* data[2] = {ctrl, cases};
  for (int c = 0; c < 2; ++c) {
    const uint64_t nw = (n[c] + 63) / 64;
    if (nw == 0) continue;
    const uint64_t* d = data[c];
    accumulate_reduced(d + (i0 * 2ULL + 0) * nw, d + (i0 * 2ULL + 1) * nw,
                       d + (i1 * 2ULL + 0) * nw, d + (i1 * 2ULL + 1) * nw,
                       d + (i2 * 2ULL + 0) * nw, d + (i2 * 2ULL + 1) * nw, nw,
                       tail_mask(n[c]), out + 27 * c);
  }
}

/* build_log_table: src/scoring.cpp:14-21 */
void eo_build_log_table(uint64_t n_max, double* prefix) {
  prefix[0] = 0.0;
  for (uint64_t n = 1; n <= n_max; ++n) prefix[n] = prefix[n - 1] + log((double)n);
}

/* k2_score: src/scoring.cpp:23-35 */
double eo_k2_score(const uint32_t* t, const double* P) {
  double score = 0.0;
  for (int c = 0; c < 27; ++c) {
    const uint32_t r0 = t[c], r1 = t[27 + c];
    const uint64_t r = (uint64_t)r0 + r1;
    score += P[r + 1] - (P[r0] + P[r1]);
  }
  return score;
}

/* hit_less: include/epi3/search.hpp:29-35 (score, then Triple <=>, common.hpp:23-29) */
int eo_hit_less(const eo_hit* a, const eo_hit* b) {
  if (a->score != b->score) return a->score < b->score;
  if (a->i0 != b->i0) return a->i0 < b->i0;
  if (a->i1 != b->i1) return a->i1 < b->i1;
  return a->i2 < b->i2;
}

/* num_combinations(m, 3): src/search.cpp:48-59 */
uint64_t eo_num_triples(uint64_t m) {
  if (m < 3) return 0;
  const u128 r = (u128)m * (m - 1) * (m - 2) / 6;
  if (r > (u128)UINT64_MAX) return 0;
  return (uint64_t)r;
}

static u128 c3(uint64_t n) { return n < 3 ? 0 : (u128)n * (n - 1) * (n - 2) / 6; }
static u128 c2(uint64_t n) { return n < 2 ? 0 : (u128)n * (n - 1) / 2; }

uint64_t eo_triple_rank(uint64_t M, uint32_t i0, uint32_t i1, uint32_t i2) {
  return (uint64_t)(c3(M) - c3(M - i0) + c2(M - 1 - i0) - c2(M - i1) + (i2 - i1 - 1));
}

void eo_triple_unrank(uint64_t M, uint64_t r, uint32_t* t) {
  uint64_t lo = 0, hi = M - 3;  /* largest a with C(M,3)-C(M-a,3) <= r */
  while (lo < hi) {
    const uint64_t mid = (lo + hi + 1) / 2;
    if (c3(M) - c3(M - mid) <= r) lo = mid; else hi = mid - 1;
  }
  const uint64_t a = lo;
  const uint64_t rest = r - (uint64_t)(c3(M) - c3(M - a));
  lo = a + 1; hi = M - 2;      /* largest b with C(M-1-a,2)-C(M-b,2) <= rest */
  while (lo < hi) {
    const uint64_t mid = (lo + hi + 1) / 2;
    if (c2(M - 1 - a) - c2(M - mid) <= rest) lo = mid; else hi = mid - 1;
  }
  const uint64_t b = lo;
  t[0] = (uint32_t)a;
  t[1] = (uint32_t)b;
  t[2] = (uint32_t)(b + 1 + rest - (uint64_t)(c2(M - 1 - a) - c2(M - b)));
}

/* TopBuffer::push: src/search.cpp:28-32 */
static void top_push(eo_hit* buf, uint32_t* n, uint32_t k, const eo_hit* h) {
  if (*n == k && !eo_hit_less(h, &buf[k - 1])) return;
  uint32_t p = *n;  /* upper_bound: first element e with hit_less(h, e) */
  while (p > 0 && eo_hit_less(h, &buf[p - 1])) --p;
  const uint32_t last = (*n == k) ? k - 1 : *n;
  memmove(buf + p + 1, buf + p, (last - p) * sizeof(eo_hit));
  buf[p] = *h;
  if (*n < k) ++*n;
}

static int cmp_hit(const void* a, const void* b) {
  if (eo_hit_less((const eo_hit*)a, (const eo_hit*)b)) return -1;
  if (eo_hit_less((const eo_hit*)b, (const eo_hit*)a)) return 1;
  return 0;
}

/* reduce_results top merge: src/search.cpp:119-123 (sort, unique, truncate) */
uint32_t eo_merge_tops(const eo_hit* hits, uint32_t n, uint32_t top_k, eo_hit* out) {
  eo_hit* tmp = (eo_hit*)malloc((n ? n : 1) * sizeof(eo_hit));
  memcpy(tmp, hits, n * sizeof(eo_hit));
  qsort(tmp, n, sizeof(eo_hit), cmp_hit);
  uint32_t m = 0;
  for (uint32_t i = 0; i < n; ++i)
    if (m == 0 || cmp_hit(&tmp[m - 1], &tmp[i]) != 0) tmp[m++] = tmp[i];
  if (m > top_k) m = top_k;
  memcpy(out, tmp, m * sizeof(eo_hit));
  free(tmp);
  return m;
}

/* run_search over a triple-rank range: src/search.cpp:127-250. The worker
 * loop (163-224) scores every triple with freq_table_reduced + k2_score and
 * keeps a per-thread TopBuffer; workers claim work from a shared atomic
 * counter (here: one i0 row per claim, search.cpp:179-184) and the partials
 * are merged by reduce_results (108-125). */
typedef struct {
  uint64_t M, N0, N1, r0, r1;
  const uint64_t *ctrl, *cases;
  const double* P;
  uint32_t top_k, a_first, a_last;
  uint64_t next;      /* shared row counter */
  eo_hit* buf;        /* per-thread top buffer */
  uint32_t count;
  void* shared;
} search_ctx;

static void* search_worker(void* arg) {
  search_ctx* w = (search_ctx*)arg;
  search_ctx* s = (search_ctx*)w->shared;
  const uint64_t M = s->M;
  uint32_t table[54];
  for (;;) {
    const uint64_t a = s->a_first + __atomic_fetch_add(&s->next, 1, __ATOMIC_RELAXED);
    if (a > s->a_last) break;
    for (uint64_t b = a + 1; b + 1 < M; ++b) {
      const uint64_t base = eo_triple_rank(M, (uint32_t)a, (uint32_t)b, (uint32_t)b + 1);
      if (base >= s->r1) break;
      if (base + (M - 1 - b) <= s->r0) continue;
      for (uint64_t c = b + 1; c < M; ++c) {
        const uint64_t r = base + (c - b - 1);
        if (r < s->r0) continue;
        if (r >= s->r1) break;
        eo_freq_table(M, s->N0, s->N1, s->ctrl, s->cases, (uint32_t)a, (uint32_t)b,
                      (uint32_t)c, table);
        eo_hit h = {eo_k2_score(table, s->P), (uint32_t)a, (uint32_t)b, (uint32_t)c, 0};
        top_push(w->buf, &w->count, s->top_k, &h);
      }
    }
  }
  return NULL;
}

uint32_t eo_search_range(uint64_t M, uint64_t N0, uint64_t N1, const uint64_t* ctrl,
                         const uint64_t* cases, uint64_t r0, uint64_t r1, uint32_t top_k,
                         int threads, eo_hit* top) {
  const uint64_t total = eo_num_triples(M);
  if (r1 > total) r1 = total;
  if (r0 >= r1 || top_k == 0) return 0;
  double* P = (double*)malloc((N0 + N1 + 2) * sizeof(double));
  eo_build_log_table(N0 + N1 + 1, P);
  uint32_t t0[3], t1[3];
  eo_triple_unrank(M, r0, t0);
  eo_triple_unrank(M, r1 - 1, t1);
  int nth = threads > 0 ? threads : (int)sysconf(_SC_NPROCESSORS_ONLN);
  if (nth < 1) nth = 1;
  search_ctx shared = {M, N0, N1, r0, r1, ctrl, cases, P, top_k, t0[0], t1[0], 0, NULL, 0, NULL};
  search_ctx* ws = (search_ctx*)calloc((size_t)nth, sizeof(search_ctx));
  eo_hit* bufs = (eo_hit*)malloc((size_t)nth * top_k * sizeof(eo_hit));
  pthread_t* tids = (pthread_t*)malloc((size_t)nth * sizeof(pthread_t));
  for (int t = 0; t < nth; ++t) {
    ws[t].buf = bufs + (size_t)t * top_k;
    ws[t].shared = &shared;
    if (nth == 1) search_worker(&ws[t]);
    else pthread_create(&tids[t], NULL, search_worker, &ws[t]);
  }
  if (nth > 1)
    for (int t = 0; t < nth; ++t) pthread_join(tids[t], NULL);
  uint32_t n = 0;
  eo_hit* all = (eo_hit*)malloc((size_t)nth * top_k * sizeof(eo_hit) + sizeof(eo_hit));
  for (int t = 0; t < nth; ++t) {
    memcpy(all + n, ws[t].buf, ws[t].count * sizeof(eo_hit));
    n += ws[t].count;
  }
  const uint32_t m = eo_merge_tops(all, n, top_k, top);
  free(all);
  free(bufs);
  free(ws);
  free(tids);
  free(P);
  return m;
}

/* write_packed: src/io.cpp:176-203, format include/epi3/io.hpp:20-25 */
int eo_write_packed(const char* path, uint64_t M, uint64_t N0, uint64_t N1,
                    const uint64_t* ctrl, const uint64_t* cases) {
  FILE* f = fopen(path, "wb");
  if (!f) return -1;
  unsigned char h[32];
  memcpy(h, "EPI3", 4);
  const uint32_t ver = 1;
  for (int i = 0; i < 4; ++i) h[4 + i] = (unsigned char)(ver >> (8 * i));
  const uint64_t v[3] = {M, N0, N1};
  for (int k = 0; k < 3; ++k)
    for (int i = 0; i < 8; ++i) h[8 + 8 * k + i] = (unsigned char)(v[k] >> (8 * i));
  fwrite(h, 1, 32, f);
  const uint64_t w[2] = {(N0 + 63) / 64, (N1 + 63) / 64};
  const uint64_t* d[2] = {ctrl, cases};
  for (uint64_t i = 0; i < M; ++i)
    for (int c = 0; c < 2; ++c) {
      if (w[c] == 0) continue;
      for (uint64_t x = 0; x < 2 * w[c]; ++x) {
        const uint64_t word = d[c][i * 2 * w[c] + x];
        unsigned char b[8];
        for (int k = 0; k < 8; ++k) b[k] = (unsigned char)(word >> (8 * k));
        fwrite(b, 1, 8, f);
      }
    }
  const int ok = ferror(f) == 0;
  fclose(f);
  return ok ? 0 : -1;
}
