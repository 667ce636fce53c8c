"""Python mirror of the reference epi3 API over the C ABI (include/epi3cu.h).

Names, argument meaning and error behaviour follow the reference C++ API
(/root/reference/proj/include/epi3/*.hpp) so parity tests read like the
reference's own tests:

  generate_synthetic (synthetic.hpp:23-26)   binarize (bitplane.hpp:72)
  read_packed / write_packed (io.hpp:27-30)  build_log_table / k2_score (scoring.hpp:53-59)
  num_combinations (search.hpp:55)           hit_less (search.hpp:29-35)
  run_search (search.hpp:85)                 reduce_results (search.hpp:89)
  freq_table_reduced (kernels.hpp:75)

The compute path is the CUDA library libepi3cu.so; there is no CPU fallback:
importing this module on a machine without the built library raises, and
every device call fails loudly when no GPU is present.
"""
from __future__ import annotations

import builtins
import ctypes as C
import os
from dataclasses import dataclass, field
from pathlib import Path
from typing import Iterable, Optional, Sequence

import numpy as np

# E3_LIBCU: path of an alternative build of the same library (A/B experiments)
_LIB_PATH = Path(os.environ.get("E3_LIBCU") or Path(__file__).resolve().parent / "libepi3cu.so")

# ---------------------------------------------------------------------------
# errors: the epi3::Error hierarchy (common.hpp:36-105)
# ---------------------------------------------------------------------------


class Error(RuntimeError):
    """epi3::Error"""


class DomainError(Error, ValueError):
    pass


class DimensionError(Error, ValueError):
    pass


class IndexError(Error, builtins.IndexError):  # noqa: A001 - mirrors epi3::IndexError
    pass


class ParseError(Error):
    pass


class MagicMismatch(Error):
    pass


class TruncatedFile(Error):
    pass


class DeviceError(Error):
    """CUDA/NCCL failure (no reference analogue: the reference has no device)."""


_ERRORS = {1: DomainError, 2: DimensionError, 3: IndexError, 4: ParseError, 5: MagicMismatch,
           6: TruncatedFile, 7: Error, 10: DeviceError, 11: DeviceError, 12: DeviceError}

# ---------------------------------------------------------------------------
# library
# ---------------------------------------------------------------------------


class e3_hit(C.Structure):
    _fields_ = [("score", C.c_double), ("i0", C.c_uint32), ("i1", C.c_uint32),
                ("i2", C.c_uint32), ("_pad", C.c_uint32)]


class e3_search_cfg(C.Structure):
    _fields_ = [("top_k", C.c_uint32), ("flags", C.c_uint32), ("rank_begin", C.c_uint64),
                ("rank_end", C.c_uint64)]


class e3_stats(C.Structure):
    _fields_ = [("combinations", C.c_uint64), ("elapsed_s", C.c_double),
                ("kernel_ms", C.c_double), ("total_device_ms", C.c_double),
                ("kernel_launches", C.c_uint32), ("main_kernel_launches", C.c_uint32)]


class e3_plant(C.Structure):
    _fields_ = [("i0", C.c_uint32), ("i1", C.c_uint32), ("i2", C.c_uint32),
                ("target", C.c_uint8 * 3), ("_pad", C.c_uint8),
                ("p_case_match", C.c_double), ("p_case_other", C.c_double)]


MAX_TOP_K = 1048576  # E3_MAX_TOP_K; above 256 a search runs two passes
# e3_search_cfg.flags: 0 = auto, E3_ENGINE_POPC = 1, E3_ENGINE_TC_MASKED = 2,
# E3_ENGINE_SYRK = 3
ENGINES = {"auto": 0, "popc": 1, "tc_masked": 2, "syrk": 3}
_P = C.c_void_p
_U64 = C.c_uint64
_U32 = C.c_uint32

# name -> (restype, argtypes); every symbol declared in include/epi3cu.h
SIGNATURES = {
    "e3_dataset_create": (C.c_int, [_U64, _U64, _U64, _P, _P, C.c_int, C.POINTER(_P)]),
    "e3_dataset_create_genotypes": (C.c_int, [_U64, _U64, _P, _P, C.c_int, C.POINTER(_P)]),
    "e3_dataset_destroy": (None, [_P]),
    "e3_dataset_info": (C.c_int, [_P, _P, _P, _P, _P]),
    "e3_search": (C.c_int, [_P, C.POINTER(e3_search_cfg), _P, C.POINTER(_U32),
                            C.POINTER(e3_stats)]),
    "e3_tables": (C.c_int, [_P, _P, _U64, _P]),
    "e3_scores": (C.c_int, [_P, _P, _U64, _P]),
    "e3_last_error": (C.c_char_p, []),
    "e3_device_count": (C.c_int, [C.POINTER(C.c_int)]),
    "e3_num_combinations": (C.c_int, [_U64, _U64, C.POINTER(_U64)]),
    "e3_triple_rank": (C.c_int, [_U64, _U32, _U32, _U32, C.POINTER(_U64)]),
    "e3_triple_unrank": (C.c_int, [_U64, _U64, _P]),
    "e3_partition": (C.c_int, [_U64, _U32, _P]),
    "e3_partition_balanced": (C.c_int, [_U64, _U32, _P]),
    "e3_build_log_table": (C.c_int, [_U64, _P]),
    "e3_k2_score": (C.c_double, [_P, _P]),
    "e3_merge_hits": (C.c_int, [_P, _U64, _U32, _P, C.POINTER(_U32)]),
    "e3_binarize": (C.c_int, [_U64, _U64, _P, _P, C.POINTER(_U64), C.POINTER(_U64), _P, _P]),
    "e3_generate_synthetic": (C.c_int, [_U64, _U64, C.c_double, _U64, C.POINTER(e3_plant),
                                        C.c_int64, _P, _P]),
    "e3_packed_header": (C.c_int, [C.c_char_p, C.POINTER(_U64), C.POINTER(_U64),
                                   C.POINTER(_U64)]),
    "e3_read_packed": (C.c_int, [C.c_char_p, _U64, _U64, _U64, _P, _P]),
    "e3_write_packed": (C.c_int, [C.c_char_p, _U64, _U64, _U64, _P, _P]),
}


def _load() -> C.CDLL:
    if not _LIB_PATH.exists():
        raise ImportError(f"{_LIB_PATH} is not built; run `python __graft_entry__.py` "
                          "(build()) first — there is no CPU fallback")
    lib = C.CDLL(str(_LIB_PATH))
    for name, (res, args) in SIGNATURES.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    return lib


lib = _load()


def _check(rc: int) -> None:
    if rc != 0:
        msg = lib.e3_last_error().decode()
        raise _ERRORS.get(rc, Error)(msg)


def _ptr(a: Optional[np.ndarray]):
    return None if a is None else a.ctypes.data_as(C.c_void_p)


# ---------------------------------------------------------------------------
# data model
# ---------------------------------------------------------------------------


@dataclass
class Triple:
    i0: int
    i1: int
    i2: int

    def astuple(self):
        return (self.i0, self.i1, self.i2)


@dataclass
class PlantSpec:
    """synthetic.hpp:15-20"""
    triple: tuple = (0, 1, 2)
    target: tuple = (1, 1, 1)
    p_case_match: float = 0.9
    p_case_other: float = 0.1


@dataclass
class BitPlaneDataset:
    """bitplane.hpp:25-67: per class, [snp][plane g<2][word64] little-endian
    words, controls = class 0, padding bits zero."""
    num_snps: int
    num_controls: int
    num_cases: int
    ctrl: np.ndarray   # uint64 [M, 2, ceil(N0/64)]
    cases: np.ndarray  # uint64 [M, 2, ceil(N1/64)]

    @property
    def num_samples(self) -> int:
        return self.num_controls + self.num_cases

    def words(self, cls: int) -> int:
        return (self.ctrl if cls == 0 else self.cases).shape[2]


def generate_synthetic(num_snps: int, num_samples: int, maf: float, seed: int,
                       plant: Optional[PlantSpec] = None, exact_cases: int = -1):
    """generate_synthetic (src/datamodel.cpp:179-227) -> (geno uint8 [M,N], pheno uint8 [N]).
    exact_cases >= 0 enables the exact-class-count fix-up (see include/epi3cu.h)."""
    geno = np.empty((num_snps, num_samples), dtype=np.uint8)
    pheno = np.empty(num_samples, dtype=np.uint8)
    p = None
    if plant is not None:
        p = e3_plant(plant.triple[0], plant.triple[1], plant.triple[2],
                     (C.c_uint8 * 3)(*plant.target), 0, plant.p_case_match, plant.p_case_other)
    _check(lib.e3_generate_synthetic(num_snps, num_samples, maf, seed,
                                     C.byref(p) if p is not None else None, exact_cases,
                                     _ptr(geno), _ptr(pheno)))
    return geno, pheno


def binarize(geno: np.ndarray, pheno: np.ndarray) -> BitPlaneDataset:
    """validate + binarize (src/datamodel.cpp:28-46, 69-92)."""
    geno = np.ascontiguousarray(geno, dtype=np.uint8)
    pheno = np.ascontiguousarray(pheno, dtype=np.uint8)
    M, N = geno.shape
    n0, n1 = _U64(), _U64()
    _check(lib.e3_binarize(M, N, _ptr(geno), _ptr(pheno), C.byref(n0), C.byref(n1), None, None))
    ctrl = np.zeros((M, 2, (n0.value + 63) // 64), dtype=np.uint64)
    cases = np.zeros((M, 2, (n1.value + 63) // 64), dtype=np.uint64)
    _check(lib.e3_binarize(M, N, _ptr(geno), _ptr(pheno), C.byref(n0), C.byref(n1),
                           _ptr(ctrl), _ptr(cases)))
    return BitPlaneDataset(M, n0.value, n1.value, ctrl, cases)


def read_packed(path) -> BitPlaneDataset:
    """read_packed (src/io.cpp:117-169)."""
    M, n0, n1 = _U64(), _U64(), _U64()
    p = os.fsencode(str(path))
    _check(lib.e3_packed_header(p, C.byref(M), C.byref(n0), C.byref(n1)))
    ctrl = np.zeros((M.value, 2, (n0.value + 63) // 64), dtype=np.uint64)
    cases = np.zeros((M.value, 2, (n1.value + 63) // 64), dtype=np.uint64)
    _check(lib.e3_read_packed(p, M.value, n0.value, n1.value, _ptr(ctrl), _ptr(cases)))
    return BitPlaneDataset(M.value, n0.value, n1.value, ctrl, cases)


def write_packed(path, ds: BitPlaneDataset) -> None:
    """write_packed (src/io.cpp:176-203)."""
    _check(lib.e3_write_packed(os.fsencode(str(path)), ds.num_snps, ds.num_controls,
                               ds.num_cases, _ptr(np.ascontiguousarray(ds.ctrl)),
                               _ptr(np.ascontiguousarray(ds.cases))))


# ---------------------------------------------------------------------------
# scoring / combinatorics (host)
# ---------------------------------------------------------------------------


def build_log_table(n_max: int) -> np.ndarray:
    """build_log_table (scoring.cpp:14-21): prefix[n] = sum_{b<=n} ln b."""
    out = np.empty(n_max + 1, dtype=np.float64)
    _check(lib.e3_build_log_table(n_max, _ptr(out)))
    return out


def k2_score(table54, prefix: np.ndarray) -> float:
    """k2_score (scoring.cpp:23-35), host fp64 with the reference grouping."""
    t = np.ascontiguousarray(table54, dtype=np.uint32).reshape(54)
    return lib.e3_k2_score(_ptr(t), _ptr(np.ascontiguousarray(prefix, dtype=np.float64)))


def num_combinations(m: int, k: int) -> int:
    out = _U64()
    _check(lib.e3_num_combinations(m, k, C.byref(out)))
    return out.value


def triple_rank(M: int, t) -> int:
    out = _U64()
    _check(lib.e3_triple_rank(M, t[0], t[1], t[2], C.byref(out)))
    return out.value


def triple_unrank(M: int, rank: int) -> tuple:
    out = np.zeros(3, dtype=np.uint32)
    _check(lib.e3_triple_unrank(M, rank, _ptr(out)))
    return tuple(int(x) for x in out)


def partition(M: int, parts: int) -> list:
    """Contiguous triple-rank ranges of equal triple counts."""
    b = np.zeros(parts + 1, dtype=np.uint64)
    _check(lib.e3_partition(M, parts, _ptr(b)))
    return [(int(b[p]), int(b[p + 1])) for p in range(parts)]


def partition_balanced(M: int, parts: int) -> list:
    """Contiguous triple-rank ranges of equal measured device cost (the
    multi-GPU split: e3_partition_balanced)."""
    b = np.zeros(parts + 1, dtype=np.uint64)
    _check(lib.e3_partition_balanced(M, parts, _ptr(b)))
    return [(int(b[p]), int(b[p + 1])) for p in range(parts)]


@dataclass(frozen=True, order=False)
class Hit:
    """search.hpp:22-27"""
    score: float
    triple: tuple

    def key(self):
        return (self.score, self.triple)


def hit_less(a: Hit, b: Hit) -> bool:
    """search.hpp:29-35: exact double compare, then lexicographic triple."""
    if a.score != b.score:
        return a.score < b.score
    return a.triple < b.triple


@dataclass
class SearchStats:
    combinations_evaluated: int = 0
    elapsed_seconds: float = 0.0
    per_thread_work: list = field(default_factory=list)  # per-GPU triples here
    kernel_ms: float = 0.0
    total_device_ms: float = 0.0
    kernel_launches: int = 0
    main_kernel_launches: int = 0


@dataclass
class SearchResult:
    """search.hpp:43-48"""
    best: Hit
    top: list
    top_k: int
    stats: SearchStats


@dataclass
class SearchConfig:
    """search.hpp:13-20 reduced to what a GPU search needs: top_k, plus the
    triple-rank range (default: the full space, as run_search)."""
    top_k: int = 10
    rank_begin: int = 0
    rank_end: int = 0  # 0 = C(M,3)
    engine: str = "auto"  # "auto" | "syrk" | "tc_masked" | "popc" — identical results


def same_outcome(a: SearchResult, b: SearchResult) -> bool:
    """search.cpp:43-46"""
    return (a.best == b.best and a.top == b.top and
            a.stats.combinations_evaluated == b.stats.combinations_evaluated)


def _hits_to_array(hits: Sequence[Hit]):
    arr = (e3_hit * max(1, len(hits)))()
    for x, h in enumerate(hits):
        arr[x].score = h.score
        arr[x].i0, arr[x].i1, arr[x].i2 = h.triple
    return arr


def _hits_from_array(arr, n: int) -> list:
    return [Hit(arr[x].score, (arr[x].i0, arr[x].i1, arr[x].i2)) for x in range(n)]


def merge_hits(hits: Sequence[Hit], top_k: int) -> list:
    arr = _hits_to_array(hits)
    out = (e3_hit * max(1, top_k))()
    n = _U32()
    _check(lib.e3_merge_hits(arr, len(hits), top_k, out, C.byref(n)))
    return _hits_from_array(out, n.value)


def reduce_results(partials: Iterable[SearchResult]) -> SearchResult:
    """reduce_results (search.cpp:108-125)."""
    partials = list(partials)
    top_k = max([1] + [p.top_k for p in partials])
    stats = SearchStats()
    allhits = []
    best = Hit(float("inf"), (0, 0, 0))
    for p in partials:
        if hit_less(p.best, best):
            best = p.best
        allhits.extend(p.top)
        stats.combinations_evaluated += p.stats.combinations_evaluated
        stats.elapsed_seconds += p.stats.elapsed_seconds
        stats.per_thread_work.extend(p.stats.per_thread_work)
    return SearchResult(best, merge_hits(allhits, top_k), top_k, stats)


# ---------------------------------------------------------------------------
# device dataset + search
# ---------------------------------------------------------------------------


def device_count() -> int:
    n = C.c_int(0)
    _check(lib.e3_device_count(C.byref(n)))
    return n.value


class DeviceDataset:
    """A BitPlaneDataset resident on one GPU (planes + marginal index)."""

    def __init__(self, ds: BitPlaneDataset, device: int = 0, ctrl_ptr=None, cases_ptr=None):
        self.num_snps = ds.num_snps
        self.num_controls = ds.num_controls
        self.num_cases = ds.num_cases
        self.device = device
        h = C.c_void_p()
        ctrl = ctrl_ptr if ctrl_ptr is not None else _ptr(np.ascontiguousarray(ds.ctrl))
        cases = cases_ptr if cases_ptr is not None else _ptr(np.ascontiguousarray(ds.cases))
        _check(lib.e3_dataset_create(ds.num_snps, ds.num_controls, ds.num_cases, ctrl, cases,
                                     device, C.byref(h)))
        self._h = h

    @classmethod
    def from_genotypes(cls, geno: np.ndarray, pheno: np.ndarray, device: int = 0) -> "DeviceDataset":
        """validate + binarize (src/datamodel.cpp:28-46, 69-92) on the device
        from a [M, N] uint8 genotype matrix and [N] phenotypes; equal to
        DeviceDataset(binarize(geno, pheno))."""
        geno = np.ascontiguousarray(geno, dtype=np.uint8)
        pheno = np.ascontiguousarray(pheno, dtype=np.uint8)
        M, N = geno.shape
        if pheno.shape != (N,):
            raise DimensionError(f"phenotype length {pheno.shape} != {N} samples")
        h = C.c_void_p()
        _check(lib.e3_dataset_create_genotypes(M, N, _ptr(geno), _ptr(pheno), device, C.byref(h)))
        self = cls.__new__(cls)
        self.num_snps = M
        self.num_cases = int(pheno.sum())
        self.num_controls = N - self.num_cases
        self.device = device
        self._h = h
        return self

    @property
    def handle(self):
        return self._h

    def close(self) -> None:
        # at interpreter exit the module global `lib` may already be gone
        if getattr(self, "_h", None) and lib is not None:
            lib.e3_dataset_destroy(self._h)
            self._h = None

    def __del__(self):
        self.close()

    def __enter__(self):
        return self

    def __exit__(self, *exc):
        self.close()

    def search(self, cfg: SearchConfig = SearchConfig()) -> SearchResult:
        if cfg.engine not in ENGINES:
            raise DomainError(f"unknown engine {cfg.engine!r}")
        c = e3_search_cfg(cfg.top_k, ENGINES[cfg.engine], cfg.rank_begin, cfg.rank_end)
        top = (e3_hit * max(1, cfg.top_k))()
        n = _U32()
        st = e3_stats()
        _check(lib.e3_search(self._h, C.byref(c), top, C.byref(n), C.byref(st)))
        hits = _hits_from_array(top, n.value)
        stats = SearchStats(st.combinations, st.elapsed_s, [st.combinations], st.kernel_ms,
                            st.total_device_ms, st.kernel_launches, st.main_kernel_launches)
        best = hits[0] if hits else Hit(float("inf"), (0, 0, 0))
        return SearchResult(best, hits, cfg.top_k, stats)

    def tables(self, triples) -> np.ndarray:
        """freq_table_reduced for each triple -> uint32 [n, 54] ([cls][combo])."""
        t = np.ascontiguousarray(np.asarray(triples, dtype=np.uint32).reshape(-1, 3))
        out = np.zeros((t.shape[0], 54), dtype=np.uint32)
        _check(lib.e3_tables(self._h, _ptr(t), t.shape[0], _ptr(out)))
        return out

    def scores(self, triples) -> np.ndarray:
        t = np.ascontiguousarray(np.asarray(triples, dtype=np.uint32).reshape(-1, 3))
        out = np.zeros(t.shape[0], dtype=np.float64)
        _check(lib.e3_scores(self._h, _ptr(t), t.shape[0], _ptr(out)))
        return out


def run_search(ds, cfg: SearchConfig = SearchConfig(), device: int = 0) -> SearchResult:
    """run_search (search.cpp:127-250) on one GPU. `ds` is a BitPlaneDataset
    (uploaded for this call) or a resident DeviceDataset."""
    if isinstance(ds, DeviceDataset):
        return ds.search(cfg)
    if ds.num_snps < 3:
        raise DimensionError("search needs at least 3 SNPs")
    with DeviceDataset(ds, device) as dd:
        return dd.search(cfg)


def freq_table_reduced(dd: DeviceDataset, t) -> np.ndarray:
    """kernels.hpp:75 for one triple -> uint32[54]."""
    return dd.tables([tuple(t)])[0]
