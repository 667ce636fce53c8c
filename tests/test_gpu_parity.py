"""Parity of the CUDA path (called through the C ABI) with the reference:
bit-exact tables, identical best/top-k triples and bit-identical K2 scores,
against golden outputs of the reference itself and against the oracle on
seeded inputs. Full-size configs are checked through size-independent
properties: random triple-rank ranges vs the oracle, oracle re-scoring of the
GPU top-k, the planted triple, and partition+merge == whole."""
import numpy as np
import pytest

import py_oracle as po
from helpers import assert_hits_identical, hits_of, product_dataset, ref_hits
from paper_2201_10956_b200 import epi3

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module", autouse=True)
def _device():
    assert epi3.device_count() >= 1, "no CUDA device: the product has no CPU fallback"


def _random_ds(M, n0, n1, seed):
    rng = np.random.default_rng(seed)
    geno = rng.integers(0, 3, (M, n0 + n1), dtype=np.uint8)
    pheno = np.array([0] * n0 + [1] * n1, dtype=np.uint8)
    rng.shuffle(pheno)
    return epi3.binarize(geno, pheno)


def test_tables_bit_exact_vs_reference(golden):
    n = 0
    for case in golden["cases"]:
        if "tables" not in case:
            continue
        with epi3.DeviceDataset(product_dataset(case)) as dd:
            got = dd.tables(case["triples"])
        assert got.tolist() == case["tables"], case["name"]
        n += len(case["triples"])
    assert n > 500


@pytest.mark.parametrize("M,n0,n1,seed", [(9, 1, 1, 1), (12, 31, 33, 2), (16, 200, 57, 3),
                                          (10, 0, 77, 4), (10, 129, 0, 5), (40, 513, 511, 6)])
def test_all_tables_and_scores_vs_oracle(M, n0, n1, seed):
    ds = _random_ds(M, n0, n1, seed)
    od = po.OracleDataset.of(ds)
    P = od.log_table()
    triples = [(a, b, c) for a in range(M) for b in range(a + 1, M) for c in range(b + 1, M)]
    with epi3.DeviceDataset(ds) as dd:
        tabs = dd.tables(triples)
        scores = dd.scores(triples)
    for t, tab, s in zip(triples, tabs, scores):
        expect = od.table(t)
        assert (tab == expect).all(), t
        assert float(s).hex() == po.k2_score(expect, P).hex(), t


@pytest.mark.parametrize("engine", ["syrk", "tc_masked", "popc"])
def test_search_matches_reference_golden(golden, engine):
    for case in golden["cases"]:
        expect = ref_hits(case["search"])
        with epi3.DeviceDataset(product_dataset(case)) as dd:
            res = dd.search(epi3.SearchConfig(top_k=len(expect), engine=engine))
        assert_hits_identical(hits_of(res), expect)
        assert res.best.triple == tuple(case["search"]["best"]["triple"]), case["name"]
        assert res.stats.combinations_evaluated == case["search"]["combinations"]


def test_tie_breaks_to_lexicographically_smallest(golden_cases):
    case = golden_cases["tie_dup_snp"]
    res = epi3.run_search(product_dataset(case), epi3.SearchConfig(top_k=10))
    assert res.best.triple == (2, 5, 7)
    s = {h.triple: h.score for h in res.top}
    assert s[(2, 5, 7)] == s[(2, 7, 9)]


def test_planted_recovery(golden):
    # acceptance.cpp:212-229: >= 19/20 recovered, and identical to the reference
    plant = [c for c in golden["cases"] if c["name"].startswith("plant_seed")]
    assert len(plant) == 20
    hit = sum(epi3.run_search(product_dataset(c), epi3.SearchConfig(top_k=1)).best.triple
              == (4, 13, 27) for c in plant)
    assert hit >= 19


@pytest.mark.parametrize("engine", ["syrk", "tc_masked", "popc"])
@pytest.mark.parametrize("top_k", [1, 2, 17, 100, 256])
def test_top_k_sizes_vs_oracle(top_k, engine):
    ds = _random_ds(40, 300, 211, 11)
    od = po.OracleDataset.of(ds)
    res = epi3.run_search(ds, epi3.SearchConfig(top_k=top_k, engine=engine))
    assert_hits_identical(hits_of(res), od.search(top_k=top_k))
    assert res.top[0] == res.best


@pytest.mark.parametrize("engine", ["syrk", "tc_masked", "popc"])
def test_ranged_searches_vs_oracle(engine):
    ds = _random_ds(90, 700, 300, 12)
    od = po.OracleDataset.of(ds)
    total = epi3.num_combinations(90, 3)
    rng = np.random.default_rng(13)
    with epi3.DeviceDataset(ds) as dd:
        for _ in range(12):
            a, b = sorted(int(x) for x in rng.integers(0, total + 1, 2))
            res = dd.search(epi3.SearchConfig(top_k=7, rank_begin=a, rank_end=b, engine=engine))
            assert res.stats.combinations_evaluated == b - a
            assert_hits_identical(hits_of(res), od.search(top_k=7, r0=a, r1=b))


@pytest.mark.parametrize("engine", ["syrk", "tc_masked", "popc"])
@pytest.mark.parametrize("G", [1, 2, 4, 8])
def test_partition_then_merge_equals_whole(G, engine):
    # the multi-GPU contract: equal-work ranges searched independently and
    # merged with reduce_results == one full search (search_test.cpp:212-242)
    ds = _random_ds(120, 600, 600, 14)
    with epi3.DeviceDataset(ds) as dd:
        whole = dd.search(epi3.SearchConfig(top_k=25, engine=engine))
        parts = [dd.search(epi3.SearchConfig(top_k=25, rank_begin=a, rank_end=b, engine=engine))
                 for a, b in epi3.partition(120, G)]
    merged = epi3.reduce_results(parts)
    assert merged.best == whole.best and merged.top == whole.top
    assert merged.stats.combinations_evaluated == epi3.num_combinations(120, 3)


def test_deterministic_repeats():
    ds = _random_ds(64, 400, 400, 15)
    with epi3.DeviceDataset(ds) as dd:
        a = dd.search(epi3.SearchConfig(top_k=50))
        for _ in range(3):
            assert epi3.same_outcome(a, dd.search(epi3.SearchConfig(top_k=50)))


def test_errors_are_loud():
    ds = _random_ds(10, 20, 20, 16)
    with epi3.DeviceDataset(ds) as dd:
        with pytest.raises(epi3.IndexError):
            dd.tables([(3, 2, 5)])
        with pytest.raises(epi3.IndexError):
            dd.tables([(0, 1, 10)])
        with pytest.raises(epi3.DomainError):
            dd.search(epi3.SearchConfig(top_k=0))
        with pytest.raises(epi3.DomainError):
            dd.search(epi3.SearchConfig(top_k=epi3.MAX_TOP_K + 1))
        with pytest.raises(epi3.IndexError):
            dd.search(epi3.SearchConfig(rank_begin=5, rank_end=1000))
    bad = _random_ds(5, 70, 0, 17)
    bad.ctrl[0, 1] |= bad.ctrl[0, 0]  # overlapping planes
    with pytest.raises(epi3.DomainError):
        epi3.DeviceDataset(bad)
    bad = _random_ds(5, 70, 0, 18)
    bad.ctrl[2, 0, -1] |= np.uint64(1) << np.uint64(63)  # dirty padding
    with pytest.raises(epi3.DomainError):
        epi3.DeviceDataset(bad)


def _config_dataset(M, N, n1, seed):
    plant = epi3.PlantSpec((M // 8, M // 2, 7 * M // 8), (1, 1, 1), 0.9,
                           0.468 if 2 * n1 == N else 0.198)
    geno, pheno = epi3.generate_synthetic(M, N, 0.3, seed, plant, exact_cases=n1)
    return epi3.binarize(geno, pheno), plant.triple


@pytest.mark.parametrize("engine", ["syrk", "tc_masked", "popc"])
@pytest.mark.parametrize("name,M,N,n1,top_k,ranges", [
    ("cfg3", 8192, 16384, 8192, 10, 3),
    ("cfg4", 1024, 262144, 131072, 10, 2),
    ("cfg5", 4096, 32768, 8192, 100, 3),
])
def test_full_size_configs_by_ranges(name, M, N, n1, top_k, ranges, engine):
    """BASELINE configs 3-5 at full size: random triple-rank windows vs the
    oracle (identical top-k, bit-identical scores) plus oracle re-scoring."""
    ds, planted = _config_dataset(M, N, n1, {"cfg3": 1003, "cfg4": 1004, "cfg5": 1005}[name])
    od = po.OracleDataset.of(ds)
    P = od.log_table()
    total = epi3.num_combinations(M, 3)
    rng = np.random.default_rng(M)
    window = 200_000 if N <= 32768 else 20_000
    with epi3.DeviceDataset(ds) as dd:
        r_pl = epi3.triple_rank(M, planted)
        starts = [max(0, r_pl - window // 2)] + [int(x) for x in rng.integers(0, total - window, ranges)]
        for a in starts:
            res = dd.search(epi3.SearchConfig(top_k=top_k, rank_begin=a, rank_end=a + window,
                                              engine=engine))
            assert_hits_identical(hits_of(res), od.search(top_k=top_k, r0=a, r1=a + window))
        got = dd.scores([h.triple for h in res.top])
        for h, s in zip(res.top, got):
            assert s.hex() == h.score.hex() == po.k2_score(od.table(h.triple), P).hex()


def test_engines_agree_on_random_inputs():
    rng = np.random.default_rng(99)
    for rep in range(6):
        M = int(rng.integers(3, 150))
        n0, n1 = int(rng.integers(0, 700)), int(rng.integers(1, 700))
        ds = _random_ds(M, n0, n1, 100 + rep)
        with epi3.DeviceDataset(ds) as dd:
            a = dd.search(epi3.SearchConfig(top_k=33, engine="syrk"))
            b = dd.search(epi3.SearchConfig(top_k=33, engine="popc"))
            c = dd.search(epi3.SearchConfig(top_k=33, engine="tc_masked"))
        assert epi3.same_outcome(a, b) and epi3.same_outcome(a, c), (M, n0, n1)


def test_class_beyond_exact_f32_range():
    """A class of >= 2^23 samples: the pair index falls back to POPC, auto
    picks the s32-accumulating masked engine, and SYRK refuses loudly."""
    n0, n1, M = (1 << 23) + 3, 64, 5
    rng = np.random.default_rng(11)
    geno = rng.integers(0, 3, (M, n0 + n1), dtype=np.uint8)
    pheno = np.zeros(n0 + n1, dtype=np.uint8)
    pheno[rng.choice(n0 + n1, n1, replace=False)] = 1
    ds = epi3.binarize(geno, pheno)
    od = po.OracleDataset.of(ds)
    triples = [(a, b, c) for a in range(M) for b in range(a + 1, M) for c in range(b + 1, M)]
    with epi3.DeviceDataset(ds) as dd:
        tabs = dd.tables(triples)
        got = hits_of(dd.search(epi3.SearchConfig(top_k=4)))
        with pytest.raises(epi3.DomainError):
            dd.search(epi3.SearchConfig(top_k=4, engine="syrk"))
    for t, tab in zip(triples, tabs):
        assert (tab == od.table(t)).all(), t
    assert_hits_identical(got, od.search(top_k=4))


@pytest.mark.parametrize("env", [{}, {"E3_NO_NARROW": "1"}, {"E3_NO_SCREEN": "1"}, {"E3_NO_SCALED": "1"},
                                 {"E3_SYRK_STAGES": "2"}, {"E3_SYRK_NO_DROP": "1"},
                                 {"E3_NO_SMEM_SCRATCH": "1"}, {"E3_NO_SCALED": "1", "E3_NO_SMEM_SCRATCH": "1"},
                                 {"E3_NO_NARROW": "1", "E3_NO_SCREEN": "1"},
                                 {"E3_SCREEN_STIRLING": "1"}, {"E3_SCREEN_STIRLING": "0"}])
@pytest.mark.parametrize("M,n0,n1,seed", [(48, 700, 333, 21), (20, 20000, 9000, 22),
                                          (40, 5000, 4200, 23)])
def test_syrk_code_paths_match_oracle(monkeypatch, env, M, n0, n1, seed):
    """Every SYRK code path (narrow class-packed / wide, screened / exact,
    the scaled screen's pooled term from the table or from Stirling's bound
    (automatic for classes >= 4096 samples: the 5000/4200 set), fewer operand
    stages, no dropped phase, epilogue scratch in shared or global memory;
    segmented compaction for the 20000-sample class) returns the oracle's
    top-k bit for bit."""
    for k, v in env.items():
        monkeypatch.setenv(k, v)
    ds = _random_ds(M, n0, n1, seed)
    with epi3.DeviceDataset(ds) as dd:
        got = hits_of(dd.search(epi3.SearchConfig(top_k=12, engine="syrk")))
    assert_hits_identical(got, po.OracleDataset.of(ds).search(top_k=12))


@pytest.mark.parametrize("M,n0,n1,seed", [(30, 517, 260, 31), (12, 0, 300, 32), (9, 20001, 3, 33)])
def test_device_binarize_matches_host(M, n0, n1, seed):
    """e3_dataset_create_genotypes (binarize on the device) builds the same
    dataset as host binarize + e3_dataset_create: identical tables and top-k."""
    rng = np.random.default_rng(seed)
    geno = rng.integers(0, 3, (M, n0 + n1), dtype=np.uint8)
    pheno = np.array([0] * n0 + [1] * n1, dtype=np.uint8)
    rng.shuffle(pheno)
    ds = epi3.binarize(geno, pheno)
    triples = [(a, b, c) for a in range(M) for b in range(a + 1, M) for c in range(b + 1, M)]
    with epi3.DeviceDataset(ds) as host_built, epi3.DeviceDataset.from_genotypes(geno, pheno) as dev_built:
        assert (dev_built.tables(triples) == host_built.tables(triples)).all()
        assert_hits_identical(hits_of(dev_built.search(epi3.SearchConfig(top_k=8))),
                              hits_of(host_built.search(epi3.SearchConfig(top_k=8))))
    assert_hits_identical(hits_of(epi3.DeviceDataset.from_genotypes(geno, pheno).search(
        epi3.SearchConfig(top_k=8))), po.OracleDataset.of(ds).search(top_k=8))


def test_device_binarize_rejects_bad_values():
    geno = np.zeros((4, 10), dtype=np.uint8)
    pheno = np.array([0, 1] * 5, dtype=np.uint8)
    geno[2, 7] = 3
    with pytest.raises(epi3.DomainError, match="snp 2, sample 7"):
        epi3.DeviceDataset.from_genotypes(geno, pheno)
    geno[2, 7] = 1
    pheno[4] = 2
    with pytest.raises(epi3.DomainError):
        epi3.DeviceDataset.from_genotypes(geno, pheno)


@pytest.mark.parametrize("engine", ["syrk", "tc_masked", "popc"])
@pytest.mark.parametrize("M", [3, 4, 65, 66, 130])
def test_snp_block_edges(engine, M):
    """Smallest searches and SNP counts around the 64-SNP tile blocks."""
    ds = _random_ds(M, 301, 257, 40 + M)
    with epi3.DeviceDataset(ds) as dd:
        got = hits_of(dd.search(epi3.SearchConfig(top_k=7, engine=engine)))
    assert_hits_identical(got, po.OracleDataset.of(ds).search(top_k=7))


@pytest.mark.parametrize("order", ["search_first", "tables_first", "engines_alternate"])
def test_lazy_wide_pair_index(order):
    """A narrow dataset (every class < 2^16) builds only the class-packed pair
    index at creation; the wide index appears on the first call that reads it
    (tables/scores, the masked and POPC engines). Every call order gives the
    oracle's answers on ONE dataset."""
    ds = _random_ds(40, 700, 333, 41)
    od = po.OracleDataset.of(ds)
    P = od.log_table()
    expect = od.search(top_k=25)
    triples = [(0, 1, 2), (3, 17, 39), (5, 6, 38), (20, 21, 22)]
    want_tabs = [od.table(t) for t in triples]

    def check_tables(dd):
        tabs, scores = dd.tables(triples), dd.scores(triples)
        for t, tab, w, s in zip(triples, tabs, want_tabs, scores):
            assert (tab == w).all(), t
            assert float(s).hex() == po.k2_score(w, P).hex(), t

    def check_search(dd, engine):
        assert_hits_identical(hits_of(dd.search(epi3.SearchConfig(top_k=25, engine=engine))), expect)

    with epi3.DeviceDataset(ds) as dd:
        if order == "search_first":
            check_search(dd, "syrk")
            check_tables(dd)
            check_search(dd, "syrk")
        elif order == "tables_first":
            check_tables(dd)
            check_search(dd, "syrk")
        else:
            for engine in ["syrk", "tc_masked", "syrk", "popc", "syrk"]:
                check_search(dd, engine)
            check_tables(dd)
