#!/usr/bin/env python
"""Create the dataset anew (H2D, repack, tensor-core pair index) and search it
R times; report outcomes that differ from the first (nondeterminism hunt on
the e2e path).   python tools/repeat_create_check.py cfg2 50 [engine]"""
import sys
from pathlib import Path
ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
import bench  # noqa: E402
from paper_2201_10956_b200 import epi3  # noqa: E402
W = sys.argv[1] if len(sys.argv) > 1 else "cfg2"
R = int(sys.argv[2]) if len(sys.argv) > 2 else 20
eng = sys.argv[3] if len(sys.argv) > 3 else "auto"
ds, top_k, planted = bench.make_dataset(W)
first, bad = None, 0
for k in range(R):
    with epi3.DeviceDataset(ds) as dd:
        r = dd.search(epi3.SearchConfig(top_k=top_k, engine=eng))
    if first is None:
        first = r
    elif not epi3.same_outcome(first, r):
        bad += 1
        print("differs at", k, r.best, first.best, flush=True)
print(W, eng, "create+search repeats", R, "differing", bad)
