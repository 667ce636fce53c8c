#!/usr/bin/env python
"""Time the reference CPU search (oracle/_ref/epi3_ref = the unmodified
reference run_search, all host threads) on COMPLETE BASELINE workloads, not
the bounded 512-SNP sample bench.py uses, so the GPU/CPU ratio of the small
configs rests on full searches. cfg3/cfg5 would take
hours on the host and stay sampled.

  python tools/cpu_full.py cfg1 cfg2 cfg4 > gpurun_out/cpu_full.json

Input built by the oracle alone (the product library is not loaded).
"""
import json
import os
import sys
import tempfile
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "oracle"))
import bench  # noqa: E402  (workload table only; no product import at module level)
import py_oracle as po  # noqa: E402

out = []
for name in sys.argv[1:] or ["cfg1", "cfg2"]:
    M, N, n1, seed, top_k = bench.WORKLOADS[name]
    triple, p_other = bench.plant_of(name)
    threads = os.cpu_count() or 1
    with tempfile.TemporaryDirectory() as d:
        f = Path(d) / f"{name}_full.epi3"
        t0 = time.time()
        po.workload_sample(f, M, N, n1, bench.MAF, seed, triple, p_other, M)
        gen_s = time.time() - t0
        per = {}
        for v in ("v3", "v4") if M > 256 else bench.REF_VARIANTS:
            r = po.ref_run("search", f, v, threads, top_k, 1)
            per[v] = {"seconds": min(r["elapsed_s"]), "best": r["best"]}
    elements = bench.c3(M) * N
    best_v = min(per, key=lambda v: per[v]["seconds"])
    line = {"workload": name, "M": M, "N": N, "elements": elements, "threads": threads,
            "variant": best_v, "seconds": per[best_v]["seconds"],
            "value_Tel_s": elements / per[best_v]["seconds"] / 1e12,
            "variants": {v: {"seconds": per[v]["seconds"],
                             "value_Tel_s": elements / per[v]["seconds"] / 1e12} for v in per},
            "best": per[best_v]["best"], "input_generation_s": gen_s}
    out.append(line)
    print(json.dumps(line), flush=True)
