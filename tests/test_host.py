"""CPU tests of the product's host layer and the C ABI surface (no device
compute): generator, binarize, packed I/O, combinatorics, partitioner, the
top-k merge and the exported symbol set."""
import re
import tempfile
from pathlib import Path

import numpy as np
import pytest

import py_oracle as po
from helpers import packed_sha, product_dataset
from paper_2201_10956_b200 import epi3

ROOT = Path(__file__).resolve().parents[1]


def test_abi_exports_every_declared_symbol():
    header = (ROOT / "include" / "epi3cu.h").read_text()
    declared = set(re.findall(r"\b(e3_[a-z0-9_]+)\s*\(", header))
    assert len(declared) >= 20
    for name in declared:
        assert hasattr(epi3.lib, name), name
    assert declared == set(epi3.SIGNATURES), declared ^ set(epi3.SIGNATURES)


def test_cpp_api_library_built():
    from paper_2201_10956_b200 import build
    assert build.LIB_CPP.exists() and build.CLI.exists()


def test_inputs_hash_like_reference(golden):
    # generator + binarize + write_packed reproduce the reference's bytes
    for case in golden["cases"]:
        assert packed_sha(product_dataset(case)) == case["sha256"], case["name"]


def test_generator_matches_oracle_and_exact_counts():
    plant = epi3.PlantSpec((3, 9, 14), (1, 1, 1), 0.9, 0.468)
    g1, p1 = epi3.generate_synthetic(20, 999, 0.3, 5, plant)
    g2, p2 = po.generate_synthetic(20, 999, 0.3, 5, plant)
    assert (g1 == g2).all() and (p1 == p2).all()
    for target in (0, 1, 333, 500, 998, 999):
        g3, p3 = epi3.generate_synthetic(20, 999, 0.3, 5, plant, exact_cases=target)
        assert (g3 == g1).all() and int(p3.sum()) == target
    with pytest.raises(epi3.DomainError):
        epi3.generate_synthetic(20, 10, 0.7, 1)
    with pytest.raises(epi3.DomainError):
        epi3.generate_synthetic(20, 10, 0.3, 1, epi3.PlantSpec((1, 1, 2)))


def test_binarize_matches_oracle_and_validates():
    rng = np.random.default_rng(3)
    for M, N in [(3, 1), (5, 64), (7, 65), (4, 129), (9, 333)]:
        geno = rng.integers(0, 3, (M, N), dtype=np.uint8)
        pheno = rng.integers(0, 2, N, dtype=np.uint8)
        ds = epi3.binarize(geno, pheno)
        n0, n1, ctrl, cases = po.binarize(geno, pheno)
        assert (ds.num_controls, ds.num_cases) == (n0, n1)
        assert (ds.ctrl == ctrl).all() and (ds.cases == cases).all()
    geno = np.zeros((3, 4), np.uint8)
    geno[1, 2] = 3
    with pytest.raises(epi3.DomainError, match="snp 1, sample 2"):
        epi3.binarize(geno, np.array([0, 0, 1, 1], np.uint8))
    with pytest.raises(epi3.DimensionError):
        epi3.binarize(np.zeros((2, 4), np.uint8), np.zeros(4, np.uint8))
    with pytest.raises(epi3.DomainError):
        epi3.binarize(np.zeros((3, 4), np.uint8), np.array([0, 2, 0, 0], np.uint8))


def test_binarize_known_layout():
    # datamodel_test: one sample per genotype -> plane0=0b001, plane1=0b010
    ds = epi3.binarize(np.array([[0, 1, 2]] * 3, np.uint8), np.zeros(3, np.uint8))
    assert ds.ctrl[0, 0, 0] == 0b001 and ds.ctrl[0, 1, 0] == 0b010
    assert ds.cases.shape == (3, 2, 0)


def test_packed_round_trip_and_corruption():
    rng = np.random.default_rng(29)
    with tempfile.TemporaryDirectory() as d:
        f = Path(d) / "x.epi3"
        for N in (64, 65, 128, 127, 1):
            geno = rng.integers(0, 3, (5, N), dtype=np.uint8)
            pheno = rng.integers(0, 2, N, dtype=np.uint8)
            ds = epi3.binarize(geno, pheno)
            epi3.write_packed(f, ds)
            back = epi3.read_packed(f)
            assert (back.num_snps, back.num_controls, back.num_cases) == \
                (ds.num_snps, ds.num_controls, ds.num_cases)
            assert (back.ctrl == ds.ctrl).all() and (back.cases == ds.cases).all()
        good = f.read_bytes()

        def check(data, exc):
            f.write_bytes(data)
            with pytest.raises(exc):
                epi3.read_packed(f)

        check(b"X" + good[1:], epi3.MagicMismatch)             # io_test.cpp:100-105
        check(good[:4] + bytes([9]) + good[5:], epi3.ParseError)  # version
        check(good[:-5], epi3.TruncatedFile)                    # truncated payload
        check(good[:10], epi3.TruncatedFile)                    # truncated header
        check(good + b"zz", epi3.ParseError)                    # trailing bytes
        check(good[:8] + bytes([0xff]) + good[9:], epi3.TruncatedFile)  # absurd M
        with pytest.raises(epi3.Error):
            epi3.read_packed(Path(d) / "missing.epi3")


def test_combinatorics_and_partition():
    assert epi3.num_combinations(2048, 3) == 1429559296
    assert epi3.num_combinations(5, 0) == 1
    with pytest.raises(epi3.DomainError):
        epi3.num_combinations(2, 3)
    M = 64
    for r in [0, 1, 5000, epi3.num_combinations(M, 3) - 1]:
        t = epi3.triple_unrank(M, r)
        assert epi3.triple_rank(M, t) == r == po.triple_rank(M, t)
    with pytest.raises(epi3.IndexError):
        epi3.triple_rank(M, (3, 2, 5))
    for G in (1, 2, 4, 8):
        parts = epi3.partition(8192, G)
        assert parts[0][0] == 0 and parts[-1][1] == epi3.num_combinations(8192, 3)
        sizes = [b - a for a, b in parts]
        assert max(sizes) - min(sizes) <= 1
        assert all(parts[i][1] == parts[i + 1][0] for i in range(G - 1))


def test_host_k2_known_answers():
    P = epi3.build_log_table(16)
    assert P[0] == 0.0 and abs(P[10] - 15.104412573075516) < 1e-12
    t = np.zeros(54, np.uint32)
    assert epi3.k2_score(t, P) == 0.0
    t[5] = 1
    assert abs(epi3.k2_score(t, P) - 0.6931471805599453) < 1e-9
    rng = np.random.default_rng(11)
    P2 = epi3.build_log_table(54 * 64 + 2)
    for _ in range(20):
        t = rng.integers(0, 64, 54).astype(np.uint32)
        assert epi3.k2_score(t, P2).hex() == po.k2_score(t, P2).hex()
        swapped = np.concatenate([t[27:], t[:27]])
        assert epi3.k2_score(swapped, P2) == epi3.k2_score(t, P2)


def _res(best, top, k, n=0):
    return epi3.SearchResult(epi3.Hit(*best), [epi3.Hit(*h) for h in top], k,
                             epi3.SearchStats(n, 0.0, [n]))


def test_reduce_results_semantics():
    # search_test.cpp:180-210
    p = _res((1.5, (0, 2, 4)), [(1.5, (0, 2, 4)), (2.0, (1, 2, 3))], 5, 7)
    r = epi3.reduce_results([p])
    assert r.best == p.best and r.top == p.top and r.stats.combinations_evaluated == 7
    a = _res((3.25, (1, 2, 3)), [(3.25, (1, 2, 3))], 4)
    b = _res((3.25, (0, 4, 5)), [(3.25, (0, 4, 5))], 4)
    m = epi3.reduce_results([a, b])
    assert m.best.triple == (0, 4, 5) and [h.triple for h in m.top] == [(0, 4, 5), (1, 2, 3)]
    # duplicates collapse (search.cpp:121)
    m2 = epi3.reduce_results([a, a])
    assert len(m2.top) == 1


def test_merge_matches_oracle_merge():
    rng = np.random.default_rng(8)
    hits = [(float(rng.integers(0, 5)) / 4, tuple(sorted(rng.choice(50, 3, replace=False).tolist())))
            for _ in range(200)]
    got = epi3.merge_hits([epi3.Hit(s, t) for s, t in hits], 17)
    assert [(h.score, h.triple) for h in got] == po.merge_tops(hits, 17)


def test_oracle_built_bench_sample_equals_product_input():
    """bench.py's CPU legs build the reference's input with the oracle alone
    (no product library in the reference arm): it must be byte-identical to
    the product's workload (generator + exact class counts + binarize)."""
    import hashlib
    import tempfile
    import py_oracle as po
    for M, N, n1, seed, p_other, m in [(256, 1024, 512, 1001, 0.468, 256),
                                       (600, 4000, 1000, 77, 0.198, 100)]:
        plant = epi3.PlantSpec((M // 8, M // 2, 7 * M // 8), (1, 1, 1), 0.9, p_other)
        g, p = epi3.generate_synthetic(M, N, 0.3, seed, plant, exact_cases=n1)
        with tempfile.TemporaryDirectory() as d:
            epi3.write_packed(d + "/a.epi3", epi3.binarize(g[:m], p))
            po.workload_sample(d + "/b.epi3", M, N, n1, 0.3, seed, plant.triple, p_other, m)
            a = hashlib.sha256(open(d + "/a.epi3", "rb").read()).hexdigest()
            b = hashlib.sha256(open(d + "/b.epi3", "rb").read()).hexdigest()
        assert a == b, (M, N)


@pytest.mark.parametrize("M", [3, 4, 5, 64, 65, 300, 2048, 8192])
@pytest.mark.parametrize("parts", [1, 2, 3, 4, 8, 16])
def test_partition_balanced_tiles_the_rank_space(M, parts):
    """e3_partition_balanced: contiguous, ordered ranges covering [0, C(M,3))
    exactly; on large M the per-range cost model (64x64 tiles + 64 per first
    SNP) is equal to within a fraction of a first SNP."""
    import numpy as np
    b = epi3.partition_balanced(M, parts)
    total = epi3.num_combinations(M, 3)
    assert b[0][0] == 0 and b[-1][1] == total
    assert all(x[1] == y[0] for x, y in zip(b, b[1:]))
    assert all(x[0] <= x[1] for x in b)
    if M >= 2048:
        i = np.arange(M - 2)
        nb = (M - 1 - i + 63) // 64
        w = nb * (nb + 1) / 2 + 64.0
        tri = (M - 1 - i) * (M - 2 - i) / 2
        ctri = np.concatenate([[0], np.cumsum(tri)])
        costs = []
        for a, e in b:
            c = 0.0
            lo = np.searchsorted(ctri, a, side="right") - 1
            hi = min(np.searchsorted(ctri, e, side="right") - 1, M - 3)
            for ii in range(lo, hi + 1):
                s_, e_ = max(a, ctri[ii]), min(e, ctri[ii + 1])
                if e_ > s_:
                    c += w[ii] * (e_ - s_) / tri[ii]
            costs.append(c)
        assert max(costs) / (sum(costs) / parts) < 1.002
