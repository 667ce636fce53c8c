"""compute-sanitizer target: successive multi-batch ranged SYRK searches on
one dataset (the path bench.py walks), tiny operand budget so every search
plans many batches. Run:
  E3_SYRK_YBUDGET_KIB=16 compute-sanitizer --tool memcheck python tools/sanitize_multibatch.py
"""
import sys
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
from paper_2201_10956_b200 import epi3  # noqa: E402

rng = np.random.default_rng(3)
M, n0, n1 = 120, 600, 500
geno = rng.integers(0, 3, (M, n0 + n1), dtype=np.uint8)
pheno = np.array([0] * n0 + [1] * n1, dtype=np.uint8)
ds = epi3.binarize(geno, pheno)
with epi3.DeviceDataset(ds) as dd:
    for rep in range(2):
        for a, b in epi3.partition(M, 12):
            r = dd.search(epi3.SearchConfig(top_k=5, rank_begin=a, rank_end=b, engine="syrk"))
            assert r.stats.combinations_evaluated == b - a
    whole = dd.search(epi3.SearchConfig(top_k=5, engine="syrk"))
    for eng in ("tc_masked", "popc"):
        assert epi3.same_outcome(whole, dd.search(epi3.SearchConfig(top_k=5, engine=eng)))
print("sanitize target ok:", whole.best)
