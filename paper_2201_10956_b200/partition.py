"""Multi-GPU plumbing: one process per GPU, equal-work triple-rank ranges,
genotype planes replicated, and ONE collective — an all-gather of each
rank's top-k (score, i0, i1, i2) records — followed by the reduce_results
merge (/root/reference/proj/src/search.cpp:108-125) on every rank.

The reference has no distributed layer (its only cross-worker exchange is the
post-join host merge, search.cpp:244); this is that merge lifted across
processes. torch.distributed provides the transport (NCCL over NVLink on the
GPU box, gloo on CPU for the tests); the search itself is the C ABI.
"""
from __future__ import annotations

from typing import Callable, Sequence

import torch
import torch.distributed as dist

from . import epi3


def rank_range(M: int, rank: int, world: int) -> tuple:
    """This rank's contiguous slice of [0, C(M,3)) (equal triple counts)."""
    return epi3.partition(M, world)[rank]


def _pack(hits: Sequence[epi3.Hit], top_k: int, device) -> torch.Tensor:
    t = torch.full((top_k, 4), float("inf"), dtype=torch.float64)
    for x, h in enumerate(hits[:top_k]):
        t[x, 0] = h.score
        t[x, 1:] = torch.tensor(h.triple, dtype=torch.float64)
    return t.to(device)


def _unpack(t: torch.Tensor) -> list:
    out = []
    for row in t.cpu().tolist():
        if row[0] == float("inf"):
            continue
        out.append(epi3.Hit(row[0], (int(row[1]), int(row[2]), int(row[3]))))
    return out


def allgather_merge(local: epi3.SearchResult, top_k: int, group=None,
                    device=None) -> epi3.SearchResult:
    """The single collective of a multi-GPU search: all-gather every rank's
    top-k (k x 32 B) and merge with hit_less + dedup + truncate."""
    world = dist.get_world_size(group)
    device = device if device is not None else (
        torch.device("cuda", torch.cuda.current_device())
        if dist.get_backend(group) == "nccl" else torch.device("cpu"))
    mine = _pack(local.top, top_k, device)
    gathered = torch.empty((world * top_k, 4), dtype=torch.float64, device=device)
    dist.all_gather_into_tensor(gathered, mine, group=group)
    work = torch.tensor([local.stats.combinations_evaluated], dtype=torch.int64, device=device)
    works = torch.empty(world, dtype=torch.int64, device=device)
    dist.all_gather_into_tensor(works, work, group=group)
    merged = epi3.merge_hits(_unpack(gathered), top_k)
    best = merged[0] if merged else epi3.Hit(float("inf"), (0, 0, 0))
    stats = epi3.SearchStats(int(works.sum().item()), local.stats.elapsed_seconds,
                             [int(x) for x in works.cpu().tolist()])
    return epi3.SearchResult(best, merged, top_k, stats)


def distributed_search(search_range: Callable[[int, int], epi3.SearchResult], M: int,
                       top_k: int, group=None, device=None) -> epi3.SearchResult:
    """run_search across the process group: this rank searches its equal-work
    range with `search_range(rank_begin, rank_end)` and the ranks merge."""
    rank, world = dist.get_rank(group), dist.get_world_size(group)
    a, b = rank_range(M, rank, world)
    return allgather_merge(search_range(a, b), top_k, group, device)
