"""Pins the plain-C oracle (oracle/epi3_oracle.c) before anything trusts it:
against outputs of the reference itself (tests/golden/golden.json, made by
oracle/_ref) and the known answers in the reference's own tests."""
import hashlib
import tempfile
from pathlib import Path

import numpy as np
import pytest

import py_oracle as po
from helpers import ref_hits


def oracle_dataset(case):
    g, kind = case["gen"], case["kind"]
    if kind in ("refgen", "refgen_dup"):
        plant = None
        if "plant" in g:
            p = g["plant"]
            plant = type("P", (), dict(triple=p[:3], target=p[3:6], p_case_match=p[6],
                                       p_case_other=p[7]))
        geno, pheno = po.generate_synthetic(g["M"], g["N"], g["maf"], g["seed"], plant)
        n0, n1, ctrl, cases = po.binarize(geno, pheno)
        if "dup" in g:
            a, b = g["dup"]
            ctrl[a] = ctrl[b]
            cases[a] = cases[b]
        return po.OracleDataset(g["M"], n0, n1, ctrl, cases)
    if kind == "numpy_uniform":
        rng = np.random.default_rng(g["seed"])
        M, n0, n1 = g["M"], g["N0"], g["N1"]
        geno = rng.integers(0, 3, size=(M, n0 + n1), dtype=np.uint8)
        pheno = np.array([0] * n0 + [1] * n1, dtype=np.uint8)
        return po.OracleDataset(M, *po.binarize(geno, pheno))
    return None


def sha_of(od):
    with tempfile.TemporaryDirectory() as d:
        f = Path(d) / "x.epi3"
        po.lib.eo_write_packed(str(f).encode(), od.M, od.N0, od.N1, po._ptr(od.ctrl),
                               po._ptr(od.cases))
        return hashlib.sha256(f.read_bytes()).hexdigest()


def test_mt19937_64_known_answer():
    # C++ [rand.predef]: the 10000th output of default-seeded mt19937_64
    assert po.mt64_stream(5489, 10000)[-1] == 9981545732273789042


def test_log_table_known_answers():
    # scoring_test.cpp:29-37
    P = po.build_log_table(16)
    assert P[0] == 0.0 and P[1] == 0.0
    assert abs(P[2] - 0.6931471805599453) <= 1e-15
    assert abs(P[10] - 15.104412573075516) < 1e-12


def test_k2_known_answers(golden):
    # scoring_test.cpp:48-67 / acceptance.cpp:155-176, bit-identical to the reference
    for kat in golden["k2_kat"]:
        P = po.build_log_table(kat["n_max"])
        assert P[-1].hex() == float.fromhex(kat["prefix_last_hex"]).hex()
        assert po.k2_score(np.array(kat["table"], dtype=np.uint32), P).hex() == \
            float.fromhex(kat["k2_hex"]).hex()
    P = po.build_log_table(8)
    one = np.zeros(54, np.uint32)
    one[5] = 1
    assert abs(po.k2_score(one, P) - 0.6931471805599453) < 1e-9
    mixed = np.zeros(54, np.uint32)
    mixed[19], mixed[27 + 19] = 2, 1
    assert abs(po.k2_score(mixed, P) - 2.4849066497880004) < 1e-9


def test_num_triples_and_ranks():
    # search_test.cpp:32-41
    assert po.num_triples(3) == 1 and po.num_triples(10) == 120
    assert po.num_triples(2048) == 1429559296
    assert po.num_triples(1000000) == 1000000 * 999999 * 999998 // 6
    M = 23
    r = 0
    for a in range(M):
        for b in range(a + 1, M):
            for c in range(b + 1, M):
                assert po.triple_rank(M, (a, b, c)) == r
                assert po.triple_unrank(M, r) == (a, b, c)
                r += 1
    assert r == po.num_triples(M)


def test_oracle_inputs_hash_like_reference(golden):
    for case in golden["cases"]:
        od = oracle_dataset(case)
        if od is not None:
            assert sha_of(od) == case["sha256"], case["name"]


def test_oracle_tables_match_reference(golden):
    n = 0
    for case in golden["cases"]:
        if "tables" not in case:
            continue
        od = oracle_dataset(case)
        for t, expect in zip(case["triples"], case["tables"]):
            tab = od.table(t)
            assert tab.tolist() == expect, (case["name"], t)
            assert int(tab[:27].sum()) == od.N0 and int(tab[27:].sum()) == od.N1
            n += 1
    assert n > 500


@pytest.mark.parametrize("threads", [1, 3])
def test_oracle_search_matches_reference(golden, threads):
    for case in golden["cases"]:
        od = oracle_dataset(case)
        if od is None or case["gen"].get("N", 0) > 4096:
            continue
        k = len(case["search"]["top"])
        got = od.search(top_k=k, threads=threads)
        expect = ref_hits(case["search"])
        assert [t for _, t in got] == [t for _, t in expect], case["name"]
        assert [s.hex() for s, _ in got] == [s.hex() for s, _ in expect], case["name"]


def test_oracle_tie_breaks_lexicographically(golden_cases):
    # search_test.cpp:110-135: (2,7,9) ties (2,5,7); the smaller triple wins
    case = golden_cases["tie_dup_snp"]
    od = oracle_dataset(case)
    top = od.search(top_k=10)
    assert top[0][1] == (2, 5, 7)
    scores = dict((t, s) for s, t in top)
    assert scores[(2, 5, 7)] == scores[(2, 7, 9)]


def test_oracle_range_searches_merge_to_full():
    # reduce_results over a random partition == full search (search_test.cpp:212-242)
    geno, pheno = po.generate_synthetic(30, 300, 0.3, 77)
    od = po.OracleDataset(30, *po.binarize(geno, pheno))
    full = od.search(top_k=20)
    total = po.num_triples(30)
    rng = np.random.default_rng(5)
    cuts = sorted(set([0, total] + [int(x) for x in rng.integers(1, total, 6)]))
    parts = []
    for a, b in zip(cuts[:-1], cuts[1:]):
        parts += od.search(top_k=20, r0=a, r1=b)
    assert po.merge_tops(parts, 20) == full
