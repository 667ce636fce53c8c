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
    """This rank's contiguous slice of [0, C(M,3)) (equal measured device cost,
    e3_partition_balanced)."""
    return epi3.partition_balanced(M, world)[rank]


def _pack(local: epi3.SearchResult, top_k: int, device) -> torch.Tensor:
    """This rank's contribution as ONE f64 tensor [top_k + 1, 4]: rows 0..k-1
    are the top-k hits (score, i0, i1, i2; +inf marks an empty row), the last
    row carries the rank's work (triples evaluated, elapsed seconds). Counts
    below 2^53 and SNP indices are exact in f64."""
    t = torch.full((top_k + 1, 4), float("inf"), dtype=torch.float64)
    for x, h in enumerate(local.top[:top_k]):
        t[x, 0] = h.score
        t[x, 1:] = torch.tensor(h.triple, dtype=torch.float64)
    t[top_k, 0] = float(local.stats.combinations_evaluated)
    t[top_k, 1] = float(local.stats.elapsed_seconds)
    t[top_k, 2:] = 0.0
    return t.to(device)


def _unpack(t: torch.Tensor, world: int, top_k: int):
    rows = t.cpu().view(world, top_k + 1, 4).tolist()
    hits, work, elapsed = [], [], []
    for r in rows:
        for row in r[:top_k]:
            if row[0] == float("inf"):
                continue
            hits.append(epi3.Hit(row[0], (int(row[1]), int(row[2]), int(row[3]))))
        work.append(int(r[top_k][0]))
        elapsed.append(r[top_k][1])
    return hits, work, elapsed


def allgather_merge(local: epi3.SearchResult, top_k: int, group=None,
                    device=None) -> epi3.SearchResult:
    """The single collective of a multi-GPU search: one all-gather of every
    rank's top-k plus its work count ((k+1) x 32 B per rank), then the
    reduce_results merge (hit_less + dedup + truncate) on every rank."""
    world = dist.get_world_size(group)
    device = device if device is not None else (
        torch.device("cuda", torch.cuda.current_device())
        if dist.get_backend(group) == "nccl" else torch.device("cpu"))
    mine = _pack(local, top_k, device)
    gathered = torch.empty((world * (top_k + 1), 4), dtype=torch.float64, device=device)
    dist.all_gather_into_tensor(gathered, mine, group=group)
    hits, work, elapsed = _unpack(gathered, world, top_k)
    merged = epi3.merge_hits(hits, top_k)
    best = merged[0] if merged else epi3.Hit(float("inf"), (0, 0, 0))
    # reduce_results sums elapsed seconds (search.cpp:108-125); a parallel
    # search's wall time is the slowest rank's
    stats = epi3.SearchStats(sum(work), max(elapsed), work)
    return epi3.SearchResult(best, merged, top_k, stats)


def distributed_search(search_range: Callable[[int, int], epi3.SearchResult], M: int,
                       top_k: int, group=None, device=None) -> epi3.SearchResult:
    """run_search across the process group: this rank searches its equal-work
    range with `search_range(rank_begin, rank_end)` and the ranks merge."""
    rank, world = dist.get_rank(group), dist.get_world_size(group)
    a, b = rank_range(M, rank, world)
    return allgather_merge(search_range(a, b), top_k, group, device)
