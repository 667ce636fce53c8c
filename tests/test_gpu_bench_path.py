"""The path bench.py takes: many successive ranged searches on ONE
DeviceDataset, each planned as several SYRK batches (boundary batches with
per-triple rank checks, interior batches unranged, double-buffered compacted
operands across batches). Round 1's driver bench crashed here (the batch
metadata buffers were sized from one shared capacity), so this is checked
slice by slice against the oracle and, at the BASELINE sizes, against the
reference's own cfg2 search (golden) and by oracle re-scoring at cfg3.

E3_SYRK_YBUDGET_KIB shrinks the per-batch operand budget so that small
datasets plan dozens of batches per search."""
import numpy as np
import pytest

import py_oracle as po
from helpers import assert_hits_identical, hits_of, product_dataset, ref_hits
from paper_2201_10956_b200 import epi3

pytestmark = pytest.mark.gpu


def _random_ds(M, n0, n1, seed):
    rng = np.random.default_rng(seed)
    geno = rng.integers(0, 3, (M, n0 + n1), dtype=np.uint8)
    pheno = np.array([0] * n0 + [1] * n1, dtype=np.uint8)
    rng.shuffle(pheno)
    return epi3.binarize(geno, pheno)


@pytest.mark.parametrize("env", [{"E3_SYRK_YBUDGET_KIB": "16"}, {"E3_SYRK_YBUDGET_KIB": "48"},
                                 {"E3_SYRK_YBUDGET_KIB": "16", "E3_NO_NARROW": "1"},
                                 {"E3_SYRK_YBUDGET_KIB": "24", "E3_NO_SMEM_SCRATCH": "1"}])
def test_successive_multibatch_slices_vs_oracle(monkeypatch, env):
    """Walk every slice of the triple-rank space through one dataset, in
    bench order, each slice a many-batch ranged search; each slice equals the
    oracle over the same range, the device counts every triple exactly once,
    and the merged slices equal one full search."""
    for k, v in env.items():
        monkeypatch.setenv(k, v)
    M = 150
    ds = _random_ds(M, 700, 650, 61)
    od = po.OracleDataset.of(ds)
    slices = epi3.partition(M, 24)
    parts = []
    with epi3.DeviceDataset(ds) as dd:
        for rep in range(2):  # a second walk reuses every buffer at its grown size
            for a, b in slices:
                res = dd.search(epi3.SearchConfig(top_k=9, rank_begin=a, rank_end=b, engine="syrk"))
                assert res.stats.combinations_evaluated == b - a
                if rep == 0:
                    assert_hits_identical(hits_of(res), od.search(top_k=9, r0=a, r1=b))
                    parts.append(res)
        whole = dd.search(epi3.SearchConfig(top_k=9, engine="syrk"))
    merged = epi3.reduce_results(parts)
    assert merged.top == whole.top
    assert_hits_identical(hits_of(whole), od.search(top_k=9))


def test_alternating_slice_sizes_reuse_buffers(monkeypatch):
    """Searches whose batch plans alternate between many small batches and a
    few large ones (the record-count split that overflowed in round 1)."""
    monkeypatch.setenv("E3_SYRK_YBUDGET_KIB", "20")
    M = 140
    ds = _random_ds(M, 400, 900, 62)
    od = po.OracleDataset.of(ds)
    total = epi3.num_combinations(M, 3)
    rng = np.random.default_rng(5)
    with epi3.DeviceDataset(ds) as dd:
        for _ in range(16):
            a, b = sorted(int(x) for x in rng.integers(0, total + 1, 2))
            if a == b:
                continue
            res = dd.search(epi3.SearchConfig(top_k=5, rank_begin=a, rank_end=b, engine="syrk"))
            assert res.stats.combinations_evaluated == b - a
            assert_hits_identical(hits_of(res), od.search(top_k=5, r0=a, r1=b))


@pytest.mark.parametrize("budget", [None, "256"])
def test_cfg2_slices_merge_to_reference(golden_cases, monkeypatch, budget):
    """cfg2 (2048 x 4096) as bench.py walks it: 64 slices on one dataset; each
    slice's top-k re-scores bit-identically with the oracle, and the merged
    slices are the reference's own full search (golden, bit-identical)."""
    if budget:
        monkeypatch.setenv("E3_SYRK_YBUDGET_KIB", budget)
    case = golden_cases["cfg2"]
    ds = product_dataset(case)
    od = po.OracleDataset.of(ds)
    P = od.log_table()
    parts = []
    with epi3.DeviceDataset(ds) as dd:
        for a, b in epi3.partition(ds.num_snps, 64):
            r = dd.search(epi3.SearchConfig(top_k=10, rank_begin=a, rank_end=b, engine="syrk"))
            assert r.stats.combinations_evaluated == b - a
            for h in r.top[:3]:
                assert h.score.hex() == po.k2_score(od.table(h.triple), P).hex()
            parts.append(r)
    merged = epi3.reduce_results(parts)
    assert_hits_identical(hits_of(merged), ref_hits(case["search"]))
    assert merged.stats.combinations_evaluated == case["search"]["combinations"]


def test_cfg3_full_walk_planted_and_rescored():
    """cfg3 (8192 x 16384) searched completely as 64 successive slices on one
    dataset (the bench's unit of work): the planted triple is the global best,
    every slice's top-k re-scores bit-identically with the oracle, and the
    device counted C(M,3) evaluations in total."""
    M, N, n1 = 8192, 16384, 8192
    plant = epi3.PlantSpec((M // 8, M // 2, 7 * M // 8), (1, 1, 1), 0.9, 0.468)
    geno, pheno = epi3.generate_synthetic(M, N, 0.3, 1003, plant, exact_cases=n1)
    ds = epi3.binarize(geno, pheno)
    del geno
    od = po.OracleDataset.of(ds)
    P = od.log_table()
    parts = []
    with epi3.DeviceDataset(ds) as dd:
        for a, b in epi3.partition(M, 64):
            r = dd.search(epi3.SearchConfig(top_k=10, rank_begin=a, rank_end=b))
            assert r.stats.combinations_evaluated == b - a
            for h in r.top[:2]:
                assert h.score.hex() == po.k2_score(od.table(h.triple), P).hex()
            parts.append(r)
        whole = dd.search(epi3.SearchConfig(top_k=10))
    merged = epi3.reduce_results(parts)
    assert merged.best.triple == plant.triple
    assert merged.top == whole.top
    assert merged.stats.combinations_evaluated == epi3.num_combinations(M, 3)
    for h in whole.top:
        assert h.score.hex() == po.k2_score(od.table(h.triple), P).hex()


def test_concurrent_searches_on_one_dataset():
    """Datasets are shareable across host threads: calls on
    one dataset serialise on its mutex and each returns the oracle's answer."""
    import threading
    ds = _random_ds(70, 500, 500, 63)
    od = po.OracleDataset.of(ds)
    total = epi3.num_combinations(70, 3)
    ranges = [(0, total), (0, total // 3), (total // 3, total), (1000, 20000)] * 3
    expect = {r: od.search(top_k=6, r0=r[0], r1=r[1]) for r in set(ranges)}
    errors = []
    with epi3.DeviceDataset(ds) as dd:
        def work(r):
            try:
                got = dd.search(epi3.SearchConfig(top_k=6, rank_begin=r[0], rank_end=r[1],
                                                  engine="syrk"))
                assert_hits_identical(hits_of(got), expect[r])
                tabs = dd.tables([(0, 1, 2), (3, 30, 69)])
                assert (tabs[1] == od.table((3, 30, 69))).all()
            except Exception as e:  # noqa: BLE001 - re-raised below
                errors.append(e)
        threads = [threading.Thread(target=work, args=(r,)) for r in ranges]
        for t in threads:
            t.start()
        for t in threads:
            t.join()
    assert not errors, errors


@pytest.mark.parametrize("engine", ["syrk", "tc_masked", "popc"])
@pytest.mark.parametrize("M,top_k,ranged", [(40, 300, False), (40, 9880, False), (110, 3000, False),
                                            (110, 1500, True)])
def test_top_k_beyond_list_capacity_vs_oracle(engine, M, top_k, ranged):
    """top_k above the 256-entry shared-memory lists (the reference's top_k is
    any u32, search.hpp:17): two passes, identical to the oracle's top-k —
    including k = C(40,3) (every triple ranked)."""
    ds = _random_ds(M, 400, 380, 64 + M)
    od = po.OracleDataset.of(ds)
    total = epi3.num_combinations(M, 3)
    a, b = (total // 5, total - total // 7) if ranged else (0, total)
    with epi3.DeviceDataset(ds) as dd:
        res = dd.search(epi3.SearchConfig(top_k=top_k, rank_begin=a, rank_end=b, engine=engine))
    assert res.stats.combinations_evaluated == b - a
    expect = od.search(top_k=top_k, r0=a, r1=b)
    assert len(expect) == min(top_k, b - a)
    assert_hits_identical(hits_of(res), expect)


def test_large_m_fits_or_fails_cleanly():
    """The paper's largest shape (40,000 SNPs) fits one
    B200 (class-packed pair index 16 B x M^2 = 25.6 GB): a ranged search
    around the planted triple matches the oracle. A dataset whose pair index
    cannot fit is refused up front with E3_OOM and a message, not a crash."""
    M, N = 40000, 6400
    plant = epi3.PlantSpec((5000, 20000, 35000), (1, 1, 1), 0.9, 0.468)
    geno, pheno = epi3.generate_synthetic(M, N, 0.3, 7, plant, exact_cases=N // 2)
    ds = epi3.binarize(geno, pheno)
    del geno
    od = po.OracleDataset.of(ds)
    r_pl = epi3.triple_rank(M, plant.triple)
    with epi3.DeviceDataset(ds) as dd:
        res = dd.search(epi3.SearchConfig(top_k=5, rank_begin=r_pl - 50_000, rank_end=r_pl + 50_000))
        assert_hits_identical(hits_of(res), od.search(top_k=5, r0=r_pl - 50_000, r1=r_pl + 50_000))
        assert res.best.triple == plant.triple
    big = epi3.BitPlaneDataset(150_000, 64, 64, np.zeros((150_000, 2, 1), dtype=np.uint64),
                               np.zeros((150_000, 2, 1), dtype=np.uint64))
    with pytest.raises(epi3.DeviceError, match="needs .* GB of device memory"):
        epi3.DeviceDataset(big)


@pytest.mark.gpu
def test_y_staging_ring_repeats_identically():
    """A wide, long-sample dataset (no screening table: the shared memory goes
    to the Y staging ring) searched 60 times on one resident dataset returns
    the identical outcome every time; a missing generic->async proxy fence
    in the ring once let 3% of cfg4 searches read a half-overwritten slot."""
    import os
    assert "E3_NO_YRING" not in os.environ
    geno, pheno = epi3.generate_synthetic(260, 140_000, 0.3, 77,
                                          epi3.PlantSpec((3, 100, 250), (1, 1, 1), 0.9, 0.3),
                                          exact_cases=70_000)
    ds = epi3.binarize(geno, pheno)
    od = po.OracleDataset.of(ds)
    with epi3.DeviceDataset(ds) as dd:
        first = dd.search(epi3.SearchConfig(top_k=10))
        for h in first.top:
            assert od.score(h.triple).hex() == h.score.hex(), h
        for _ in range(60):
            assert epi3.same_outcome(first, dd.search(epi3.SearchConfig(top_k=10)))
