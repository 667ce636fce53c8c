#!/usr/bin/env python
"""Repeat one workload's full search R times on one resident dataset and
report any outcome that differs from the first (nondeterminism hunt).
  python tools/repeat_check.py cfg4 40"""
import sys
from pathlib import Path
ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
import bench  # noqa: E402
from paper_2201_10956_b200 import epi3  # noqa: E402
W = sys.argv[1] if len(sys.argv) > 1 else "cfg4"
R = int(sys.argv[2]) if len(sys.argv) > 2 else 20
ds, top_k, planted = bench.make_dataset(W)
bad = 0
with epi3.DeviceDataset(ds) as dd:
    cfg = epi3.SearchConfig(top_k=top_k)
    first = dd.search(cfg)
    for k in range(R):
        r = dd.search(cfg)
        if not epi3.same_outcome(first, r):
            bad += 1
            print("differs at", k, "best", r.best, "vs", first.best, "evals", r.stats.combinations_evaluated,
                  first.stats.combinations_evaluated,
                  [(h.triple, h.score) for h in r.top if h not in first.top][:3], flush=True)
print(W, "repeats", R, "differing", bad)
