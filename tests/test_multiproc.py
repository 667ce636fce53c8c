"""World-size-2 (and 3) CPU coverage of the multi-GPU path: partitioner ->
per-rank range search -> the single all-gather -> merge, over gloo. The
per-rank compute here is the oracle (no GPU in this container); on the GPU
box the same plumbing wraps the C-ABI search (bench.py, test_gpu_parity)."""
import os
import socket

import numpy as np
import pytest
import torch.distributed as dist
import torch.multiprocessing as mp


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, M, top_k, q):
    import sys
    from pathlib import Path
    root = Path(__file__).resolve().parents[1]
    sys.path.insert(0, str(root))
    sys.path.insert(0, str(root / "oracle"))
    import py_oracle as po
    from paper_2201_10956_b200 import epi3, partition

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        geno, pheno = epi3.generate_synthetic(M, 400, 0.3, 42)
        od = po.OracleDataset.of(epi3.binarize(geno, pheno))

        def search_range(a, b):
            hits = [epi3.Hit(s, t) for s, t in od.search(top_k=top_k, r0=a, r1=b, threads=1)]
            best = hits[0] if hits else epi3.Hit(float("inf"), (0, 0, 0))
            return epi3.SearchResult(best, hits, top_k, epi3.SearchStats(b - a, 0.0, [b - a]))

        res = partition.distributed_search(search_range, M, top_k)
        q.put((rank, [(h.score, h.triple) for h in res.top], res.stats.combinations_evaluated,
               res.stats.per_thread_work))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_gloo_partition_allgather_merge(world):
    import py_oracle as po
    from paper_2201_10956_b200 import epi3
    M, top_k = 24, 15
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, M, top_k, q)) for r in range(world)]
    for p in procs:
        p.start()
    out = [q.get(timeout=300) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    geno, pheno = epi3.generate_synthetic(M, 400, 0.3, 42)
    whole = po.OracleDataset.of(epi3.binarize(geno, pheno)).search(top_k=top_k)
    for rank, top, combos, work in out:
        assert top == whole  # every rank holds the identical merged result
        assert combos == epi3.num_combinations(M, 3)
        # the cost-balanced ranges tile [0, C(M,3)) exactly, one per rank
        assert work == [b - a for a, b in epi3.partition_balanced(M, world)]
