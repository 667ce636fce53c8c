"""Throughput sanity check on an arbitrary shape (random genotypes, device
binarize): full search per engine, device time from the C ABI stats.
usage: python tools/shape_check.py M N [engines...]"""
import sys
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
import numpy as np  # noqa: E402
from paper_2201_10956_b200 import epi3  # noqa: E402

M, N = int(sys.argv[1]), int(sys.argv[2])
engines = sys.argv[3:] or ["syrk", "tc_masked"]
rng = np.random.default_rng(1)
geno = (rng.random((M, N)) < 0.3).astype(np.uint8) + (rng.random((M, N)) < 0.3).astype(np.uint8)
pheno = (rng.random(N) < 0.5).astype(np.uint8)
with epi3.DeviceDataset.from_genotypes(geno, pheno) as dd:
    for e in engines:
        dd.search(epi3.SearchConfig(top_k=10, engine=e))
        r = dd.search(epi3.SearchConfig(top_k=10, engine=e))
        el = epi3.num_combinations(M, 3) * N
        print(f"{M}x{N} {e}: {r.stats.total_device_ms:.2f} ms, {el / r.stats.total_device_ms / 1e9:.1f} Tel/s, "
              f"best {r.best.triple} {r.best.score:.6f}")
