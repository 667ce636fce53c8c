"""ctypes binding of the plain-C oracle (oracle/epi3_oracle.c) and a runner
for the reference build (oracle/_ref/epi3_ref).

TEST INFRASTRUCTURE ONLY: imported by tests/, __graft_entry__.smoke() and
bench.py's CPU-baseline legs, as the checker — never by the product package.
"""
from __future__ import annotations

import ctypes as C
import json
import subprocess
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
LIB_PATH = HERE / "_build" / "libepi3_oracle.so"
REF_BIN = HERE / "_ref" / "epi3_ref"


class eo_hit(C.Structure):
    _fields_ = [("score", C.c_double), ("i0", C.c_uint32), ("i1", C.c_uint32),
                ("i2", C.c_uint32), ("pad", C.c_uint32)]


class eo_mt64(C.Structure):
    _fields_ = [("mt", C.c_uint64 * 312), ("idx", C.c_int)]


_P = C.c_void_p
_U64 = C.c_uint64
_U32 = C.c_uint32


def _load():
    if not LIB_PATH.exists():
        raise ImportError(f"{LIB_PATH} missing; build with `make -f oracle/Makefile`")
    lib = C.CDLL(str(LIB_PATH))
    sig = {
        "eo_mt64_seed": (None, [C.POINTER(eo_mt64), _U64]),
        "eo_mt64_next": (_U64, [C.POINTER(eo_mt64)]),
        "eo_generate_synthetic": (C.c_int, [_U64, _U64, C.c_double, _U64, _P, _P, C.c_double,
                                            C.c_double, _P, _P]),
        "eo_binarize": (None, [_U64, _U64, _P, _P, _U64, _U64, _P, _P]),
        "eo_freq_table": (None, [_U64, _U64, _U64, _P, _P, _U32, _U32, _U32, _P]),
        "eo_build_log_table": (None, [_U64, _P]),
        "eo_k2_score": (C.c_double, [_P, _P]),
        "eo_num_triples": (_U64, [_U64]),
        "eo_triple_rank": (_U64, [_U64, _U32, _U32, _U32]),
        "eo_triple_unrank": (None, [_U64, _U64, _P]),
        "eo_search_range": (_U32, [_U64, _U64, _U64, _P, _P, _U64, _U64, _U32, C.c_int, _P]),
        "eo_merge_tops": (_U32, [_P, _U32, _U32, _P]),
        "eo_write_packed": (C.c_int, [C.c_char_p, _U64, _U64, _U64, _P, _P]),
    }
    for name, (res, args) in sig.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    return lib


lib = _load()


def _ptr(a):
    return None if a is None else a.ctypes.data_as(C.c_void_p)


def mt64_stream(seed: int, n: int) -> list:
    g = eo_mt64()
    lib.eo_mt64_seed(C.byref(g), seed)
    return [lib.eo_mt64_next(C.byref(g)) for _ in range(n)]


def generate_synthetic(M, N, maf, seed, plant=None):
    geno = np.empty((M, N), dtype=np.uint8)
    pheno = np.empty(N, dtype=np.uint8)
    pt = ptg = None
    pm = po = 0.0
    if plant is not None:
        pt = np.asarray(plant.triple, dtype=np.uint32)
        ptg = np.asarray(plant.target, dtype=np.uint8)
        pm, po = plant.p_case_match, plant.p_case_other
    rc = lib.eo_generate_synthetic(M, N, maf, seed, _ptr(pt), _ptr(ptg), pm, po, _ptr(geno),
                                   _ptr(pheno))
    if rc != 0:
        raise ValueError("oracle generate_synthetic: domain error")
    return geno, pheno


def binarize(geno, pheno):
    geno = np.ascontiguousarray(geno, dtype=np.uint8)
    pheno = np.ascontiguousarray(pheno, dtype=np.uint8)
    M, N = geno.shape
    n1 = int(pheno.sum())
    n0 = N - n1
    ctrl = np.zeros((M, 2, (n0 + 63) // 64), dtype=np.uint64)
    cases = np.zeros((M, 2, (n1 + 63) // 64), dtype=np.uint64)
    lib.eo_binarize(M, N, _ptr(geno), _ptr(pheno), n0, n1, _ptr(ctrl), _ptr(cases))
    return n0, n1, ctrl, cases


class OracleDataset:
    def __init__(self, M, N0, N1, ctrl, cases):
        self.M, self.N0, self.N1 = M, N0, N1
        self.ctrl = np.ascontiguousarray(ctrl, dtype=np.uint64)
        self.cases = np.ascontiguousarray(cases, dtype=np.uint64)

    @classmethod
    def of(cls, ds):
        """From a paper_2201_10956_b200.epi3.BitPlaneDataset (same layout)."""
        return cls(ds.num_snps, ds.num_controls, ds.num_cases, ds.ctrl, ds.cases)

    def table(self, t) -> np.ndarray:
        out = np.zeros(54, dtype=np.uint32)
        lib.eo_freq_table(self.M, self.N0, self.N1, _ptr(self.ctrl), _ptr(self.cases),
                          int(t[0]), int(t[1]), int(t[2]), _ptr(out))
        return out

    def log_table(self):
        P = np.empty(self.N0 + self.N1 + 2, dtype=np.float64)
        lib.eo_build_log_table(self.N0 + self.N1 + 1, _ptr(P))
        return P

    def score(self, t, P=None) -> float:
        P = self.log_table() if P is None else P
        return lib.eo_k2_score(_ptr(self.table(t)), _ptr(P))

    def search(self, top_k=10, r0=0, r1=None, threads=0):
        """run_search over triple ranks [r0, r1) -> list of (score, (i0,i1,i2))."""
        if r1 is None:
            r1 = lib.eo_num_triples(self.M)
        out = (eo_hit * top_k)()
        n = lib.eo_search_range(self.M, self.N0, self.N1, _ptr(self.ctrl), _ptr(self.cases),
                                r0, r1, top_k, threads, out)
        return [(out[x].score, (out[x].i0, out[x].i1, out[x].i2)) for x in range(n)]


def build_log_table(n_max):
    P = np.empty(n_max + 1, dtype=np.float64)
    lib.eo_build_log_table(n_max, _ptr(P))
    return P


def k2_score(table54, P):
    t = np.ascontiguousarray(table54, dtype=np.uint32)
    return lib.eo_k2_score(_ptr(t), _ptr(np.ascontiguousarray(P, dtype=np.float64)))


def num_triples(M):
    return lib.eo_num_triples(M)


def triple_rank(M, t):
    return lib.eo_triple_rank(M, *[int(x) for x in t])


def triple_unrank(M, r):
    out = np.zeros(3, dtype=np.uint32)
    lib.eo_triple_unrank(M, r, _ptr(out))
    return tuple(int(x) for x in out)


def merge_tops(hits, top_k):
    arr = (eo_hit * max(1, len(hits)))()
    for x, (s, t) in enumerate(hits):
        arr[x].score = s
        arr[x].i0, arr[x].i1, arr[x].i2 = t
    out = (eo_hit * max(1, top_k))()
    n = lib.eo_merge_tops(arr, len(hits), top_k, out)
    return [(out[x].score, (out[x].i0, out[x].i1, out[x].i2)) for x in range(n)]


# --------------------------------------------------------------------------
# the reference build (oracle/_ref/epi3_ref)
# --------------------------------------------------------------------------


def ref_available() -> bool:
    return REF_BIN.exists()


def ref_run(*args, timeout=3600) -> dict:
    out = subprocess.run([str(REF_BIN), *[str(a) for a in args]], capture_output=True,
                         text=True, timeout=timeout)
    if out.returncode != 0:
        raise RuntimeError(f"epi3_ref {args[0]} failed: {out.stderr.strip()}")
    return json.loads(out.stdout)


# --------------------------------------------------------------------------
# bench.py's CPU legs: the workload's input built with the oracle alone, so
# the reference arm never loads the product library
# --------------------------------------------------------------------------


class _Plant:
    def __init__(self, triple, target, p_case_match, p_case_other):
        self.triple, self.target = triple, target
        self.p_case_match, self.p_case_other = p_case_match, p_case_other


def exact_class_fixup(geno, pheno, plant, exact_cases):
    """The exact-class-count fix-up of e3_generate_synthetic (include/epi3cu.h):
    flip surplus labels of samples that do not match the plant first, lowest
    index first, then matching ones only if that was not enough."""
    pheno = pheno.copy()
    match = np.ones(pheno.shape[0], dtype=bool)
    for s, g in zip(plant.triple, plant.target):
        match &= geno[s] == g
    cases = int(pheno.sum())
    for want_match in (False, True):
        if cases == exact_cases:
            break
        idx = np.nonzero(match == want_match)[0]
        if cases > exact_cases:
            cand = idx[pheno[idx] == 1][: cases - exact_cases]
            pheno[cand] = 0
            cases -= cand.size
        else:
            cand = idx[pheno[idx] == 0][: exact_cases - cases]
            pheno[cand] = 1
            cases += cand.size
    return pheno


def workload_sample(path, M, N, n1, maf, seed, plant_triple, p_other, m_sub, p_match=0.9):
    """Writes the first m_sub SNPs x all N samples of a bench workload (the
    reference generator + exact class counts, identical to the product's
    generate_synthetic(..., exact_cases=n1)) as an EPI3 file; returns
    (path, N0, N1)."""
    plant = _Plant(tuple(plant_triple), (1, 1, 1), p_match, p_other)
    geno, pheno = generate_synthetic(M, N, maf, seed, plant)
    pheno = exact_class_fixup(geno, pheno, plant, n1)
    n0, n1_, ctrl, cases = binarize(geno[:m_sub], pheno)
    rc = lib.eo_write_packed(str(path).encode(), m_sub, n0, n1_, _ptr(ctrl), _ptr(cases))
    if rc != 0:
        raise OSError(f"eo_write_packed {path} failed")
    return path, n0, n1_
