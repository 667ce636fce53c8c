#!/usr/bin/env python
"""Memory scaling check at the paper's SNP count (PAPER.md: 40,000 SNPs):
create a 40000-SNP x N dataset on one B200 (narrow pair index: 16 B x M^2 =
25.6 GB), search windows of the triple-rank space and re-score every returned
hit with the oracle (bit-identical K2), and show that a size that cannot fit
is rejected up front with E3_OOM instead of failing mid-search.

  python tools/large_m_check.py [M] [N] > gpurun_out/large_m.json
"""
import json
import sys
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "oracle"))
import py_oracle as po  # noqa: E402  (the checker)
from paper_2201_10956_b200 import epi3  # noqa: E402

M = int(sys.argv[1]) if len(sys.argv) > 1 else 40000
N = int(sys.argv[2]) if len(sys.argv) > 2 else 2048
plant = epi3.PlantSpec((7, 19_000, 38_000), (1, 1, 1), 0.9, 0.3)
t0 = time.time()
geno, pheno = epi3.generate_synthetic(M, N, 0.3, 4000, plant, exact_cases=N // 2)
ds = epi3.binarize(geno, pheno)
gen_s = time.time() - t0
od = po.OracleDataset.of(ds)
total = epi3.num_combinations(M, 3)
out = {"M": M, "N": N, "triples": total, "host_generate_binarize_s": round(gen_s, 2)}
t0 = time.time()
with epi3.DeviceDataset(ds) as dd:
    out["dataset_create_s"] = round(time.time() - t0, 3)
    windows = []
    planted = po.triple_rank(M, (7, 19_000, 38_000))
    for a, b in ((0, 20_000_000), (total // 2, total // 2 + 20_000_000),
                 (max(0, planted - 5_000_000), planted + 5_000_000)):
        r = dd.search(epi3.SearchConfig(top_k=10, rank_begin=a, rank_end=b))
        ok = all(po.OracleDataset.score(od, h.triple).hex() == h.score.hex() for h in r.top)
        windows.append({"rank_begin": a, "rank_end": b, "kernel_ms": round(r.stats.kernel_ms, 2),
                        "evaluated": r.stats.combinations_evaluated, "best": list(r.best.triple),
                        "k2": r.best.score, "top10_rescored_bit_identical": ok})
    out["windows"] = windows
# a dataset whose pair index cannot fit is refused before any search
try:
    big = 120_000  # 16 B x M^2 = 230 GB > 180 GB of HBM
    g2, p2 = epi3.generate_synthetic(big, 64, 0.3, 1, None, exact_cases=32)
    with epi3.DeviceDataset(epi3.binarize(g2, p2)):
        out["oom_check"] = "unexpectedly created"
except Exception as e:  # noqa: BLE001
    out["oom_check"] = f"{type(e).__name__}: {e}"
print(json.dumps(out))
