"""Host binarize + dataset create vs. device binarize (e3_dataset_create_genotypes)
at a BASELINE shape; prints wall times (warm, median of 3)."""
import statistics
import sys
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
import numpy as np  # noqa: E402
from paper_2201_10956_b200 import epi3  # noqa: E402

M, N = (int(x) for x in (sys.argv[1:3] if len(sys.argv) > 2 else (1024, 262144)))
rng = np.random.default_rng(5)
geno = rng.integers(0, 3, (M, N), dtype=np.uint8)
pheno = np.zeros(N, dtype=np.uint8)
pheno[rng.choice(N, N // 2, replace=False)] = 1
th, td = [], []
for _ in range(4):
    t0 = time.perf_counter()
    ds = epi3.binarize(geno, pheno)
    dd = epi3.DeviceDataset(ds)
    t1 = time.perf_counter()
    dd.close()
    t2 = time.perf_counter()
    dg = epi3.DeviceDataset.from_genotypes(geno, pheno)
    t3 = time.perf_counter()
    dg.close()
    th.append(t1 - t0)
    td.append(t3 - t2)
print(f"{M}x{N}: host binarize + create {1e3 * statistics.median(th[1:]):.1f} ms, "
      f"device binarize create {1e3 * statistics.median(td[1:]):.1f} ms")
