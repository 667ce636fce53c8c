"""Generates tests/golden/golden.json from the REFERENCE ITSELF.

Every expected value in the fixture comes from oracle/_ref/epi3_ref — the
unmodified reference library (/root/reference/proj/src, compiled in place by
oracle/Makefile) driven by oracle/ref_driver.cpp. Inputs are either made by
the reference generator (`epi3_ref gen`) or by our generator and written in
the reference's packed format; each case records the sha256 of the packed
file so a test can regenerate the identical input without the fixture
carrying binary data.

Run here (where /root/reference exists):  python tests/golden/make_golden.py
"""
from __future__ import annotations

import hashlib
import json
import sys
import tempfile
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[2]
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "oracle"))

import py_oracle as po  # noqa: E402
from paper_2201_10956_b200 import epi3  # noqa: E402

OUT = Path(__file__).resolve().parent / "golden.json"


def sha(path: Path) -> str:
    return hashlib.sha256(path.read_bytes()).hexdigest()


def ref_search(path, top_k=10, variant="v3"):
    r = po.ref_run("search", path, variant, 8, top_k, 1)
    return {"best": r["best"], "top": r["top"], "combinations": r["combinations"],
            "controls": r["controls"], "cases": r["cases"]}


def ref_tables(path, triples):
    flat = [x for t in triples for x in t]
    return po.ref_run("tables", path, *flat)["tables"]


def sample_triples(M, n, rng):
    out = set()
    while len(out) < n:
        t = tuple(sorted(int(x) for x in rng.choice(M, 3, replace=False)))
        out.add(t)
    return sorted(out)


def main() -> None:
    assert po.ref_available(), "build oracle/_ref first (make -f oracle/Makefile)"
    tmp = Path(tempfile.mkdtemp())
    rng = np.random.default_rng(20260101)
    cases = []

    # 1. acceptance criterion 1 datasets (tests/acceptance.cpp:124-133), made
    #    by the reference generator; full search + tables for sampled triples.
    snp_grid, sample_grid = (10, 20, 64), (33, 257, 1024)
    for s in range(20):
        M, N = snp_grid[s % 3], sample_grid[(s // 3) % 3]
        f = tmp / f"crit1_{s}.epi3"
        po.ref_run("gen", M, N, 0.3, 9000 + s, f)
        triples = sample_triples(M, 24, rng) + [(0, 1, 2), (M - 3, M - 2, M - 1)]
        cases.append({"name": f"crit1_seed{s}", "kind": "refgen",
                      "gen": {"M": M, "N": N, "maf": 0.3, "seed": 9000 + s},
                      "sha256": sha(f), "search": ref_search(f, 10),
                      "triples": triples, "tables": ref_tables(f, triples)})

    # 2. planted recovery (acceptance.cpp:212-229): M=32 N=4096 maf .5, seeds 500..519
    for s in range(20):
        f = tmp / f"plant_{s}.epi3"
        po.ref_run("gen", 32, 4096, 0.5, 500 + s, f, 4, 13, 27, 1, 1, 1, 0.9, 0.1)
        cases.append({"name": f"plant_seed{500 + s}", "kind": "refgen",
                      "gen": {"M": 32, "N": 4096, "maf": 0.5, "seed": 500 + s,
                              "plant": [4, 13, 27, 1, 1, 1, 0.9, 0.1]},
                      "sha256": sha(f), "search": ref_search(f, 10)})

    # 3. duplicated-SNP tie (search_test.cpp:110-135): SNP 9 := SNP 5
    f = tmp / "tie.epi3"
    po.ref_run("gen", 12, 800, 0.5, 31, f, 2, 5, 7, 1, 1, 1, 0.95, 0.05)
    ds = epi3.read_packed(f)
    ds.ctrl[9] = ds.ctrl[5]
    ds.cases[9] = ds.cases[5]
    epi3.write_packed(f, ds)
    cases.append({"name": "tie_dup_snp", "kind": "refgen_dup",
                  "gen": {"M": 12, "N": 800, "maf": 0.5, "seed": 31,
                          "plant": [2, 5, 7, 1, 1, 1, 0.95, 0.05], "dup": [9, 5]},
                  "sha256": sha(f), "search": ref_search(f, 10)})

    # 4. padding / empty-class tables (kernels_test.cpp:170-194): uniform random
    #    matrices from numpy PCG64 with explicit class layouts.
    for n0, extra, seed in [(64, 40, 1), (65, 40, 2), (128, 40, 3), (129, 40, 4), (1, 40, 5),
                            (50, 0, 6), (0, 37, 7), (31, 33, 8), (127, 129, 9)]:
        g = np.random.default_rng(seed)
        M, N = 7, n0 + extra
        geno = g.integers(0, 3, size=(M, N), dtype=np.uint8)
        pheno = np.array([0] * n0 + [1] * extra, dtype=np.uint8)
        ds = epi3.binarize(geno, pheno)
        f = tmp / f"pad_{n0}_{extra}.epi3"
        epi3.write_packed(f, ds)
        triples = [(a, b, c) for a in range(M) for b in range(a + 1, M) for c in range(b + 1, M)]
        cases.append({"name": f"padding_n0_{n0}_n1_{extra}", "kind": "numpy_uniform",
                      "gen": {"M": M, "N0": n0, "N1": extra, "seed": seed},
                      "sha256": sha(f), "search": ref_search(f, 5),
                      "triples": triples, "tables": ref_tables(f, triples)})

    # 5. BASELINE configs 1 and 2 with our exact-class-count generator
    #    (SURVEY.md §8(d)): the reference searches them in full here.
    for name, M, N, n1, seed, top_k in [("cfg1", 256, 1024, 512, 1001, 10),
                                        ("cfg2", 2048, 4096, 2048, 1002, 10)]:
        plant = epi3.PlantSpec((M // 8, M // 2, 7 * M // 8), (1, 1, 1), 0.9, 0.468)
        geno, pheno = epi3.generate_synthetic(M, N, 0.3, seed, plant, exact_cases=n1)
        ds = epi3.binarize(geno, pheno)
        f = tmp / f"{name}.epi3"
        epi3.write_packed(f, ds)
        print(f"reference search {name} ...", flush=True)
        cases.append({"name": name, "kind": "ours_exact",
                      "gen": {"M": M, "N": N, "maf": 0.3, "seed": seed, "cases": n1,
                              "plant": [M // 8, M // 2, 7 * M // 8, 1, 1, 1, 0.9, 0.468]},
                      "sha256": sha(f), "search": ref_search(f, top_k)})

    # 6. K2 known answers through the reference scoring (scoring_test.cpp:48-67)
    kat = []
    for cells, n_max in [({}, 8), ({(5, 0): 1}, 8), ({(19, 0): 2, (19, 1): 1}, 8),
                         ({(13, 0): 2, (13, 1): 1}, 16)]:
        t = [0] * 54
        for (combo, cls), v in cells.items():
            t[cls * 27 + combo] = v
        r = po.ref_run("logk2", n_max, *t)
        kat.append({"table": t, "n_max": n_max, "k2_hex": r["hex"], "prefix_last_hex": r["prefix_last"]})

    OUT.write_text(json.dumps({"generator": "tests/golden/make_golden.py",
                               "reference": "oracle/_ref/epi3_ref (unmodified /root/reference/proj/src)",
                               "cases": cases, "k2_kat": kat}, indent=1))
    print(f"wrote {OUT} ({OUT.stat().st_size} bytes, {len(cases)} cases)")


if __name__ == "__main__":
    main()
