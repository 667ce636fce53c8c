"""Shared test helpers: rebuild golden inputs and compare hits."""
from __future__ import annotations

import hashlib
import tempfile
from pathlib import Path

import numpy as np

from paper_2201_10956_b200 import epi3


def _plant(g):
    if "plant" not in g:
        return None
    p = g["plant"]
    return epi3.PlantSpec((p[0], p[1], p[2]), (p[3], p[4], p[5]), p[6], p[7])


def product_dataset(case) -> epi3.BitPlaneDataset:
    """Regenerates a golden input with the product's host code (generator,
    binarize) — its packed bytes must hash to the reference's."""
    g, kind = case["gen"], case["kind"]
    if kind in ("refgen", "refgen_dup", "ours_exact"):
        geno, pheno = epi3.generate_synthetic(g["M"], g["N"], g["maf"], g["seed"], _plant(g),
                                              exact_cases=g.get("cases", -1))
        ds = epi3.binarize(geno, pheno)
        if "dup" in g:
            a, b = g["dup"]
            ds.ctrl[a] = ds.ctrl[b]
            ds.cases[a] = ds.cases[b]
        return ds
    if kind == "numpy_uniform":
        rng = np.random.default_rng(g["seed"])
        M, n0, n1 = g["M"], g["N0"], g["N1"]
        geno = rng.integers(0, 3, size=(M, n0 + n1), dtype=np.uint8)
        pheno = np.array([0] * n0 + [1] * n1, dtype=np.uint8)
        return epi3.binarize(geno, pheno)
    raise ValueError(kind)


def packed_sha(ds: epi3.BitPlaneDataset) -> str:
    with tempfile.TemporaryDirectory() as d:
        f = Path(d) / "x.epi3"
        epi3.write_packed(f, ds)
        return hashlib.sha256(f.read_bytes()).hexdigest()


def ref_hits(search_json):
    """Reference hits as (score, (i0,i1,i2)) with the exact double."""
    return [(float.fromhex(h["hex"]), tuple(h["triple"])) for h in search_json["top"]]


def hits_of(result: epi3.SearchResult):
    return [(h.score, tuple(h.triple)) for h in result.top]


def assert_hits_identical(got, expect):
    """Same triples in the same order and bit-identical scores."""
    assert len(got) == len(expect), (got, expect)
    for (gs, gt), (es, et) in zip(got, expect):
        assert gt == et, (got, expect)
        assert gs.hex() == es.hex(), (gt, gs.hex(), es.hex())
