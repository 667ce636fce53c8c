"""Quick A/B timing of one engine on a BASELINE workload (not the bench
contract: no L2 flush, no e2e). Searches the fraction [lo, hi) of the
triple-rank space R times after one warm-up and prints device Tel/s.

  python tools/syrk_time.py --workload cfg3 --lo 0.25 --hi 0.375 --reps 3
  E3_LIBCU=/path/alt.so python tools/syrk_time.py ...   (A/B of two builds)
"""
import argparse
import sys
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
import bench  # noqa: E402
from paper_2201_10956_b200 import epi3  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--workload", default="cfg3")
ap.add_argument("--lo", type=float, default=0.25)
ap.add_argument("--hi", type=float, default=0.375)
ap.add_argument("--reps", type=int, default=3)
ap.add_argument("--engine", default="auto")
ap.add_argument("--tag", default="")
ap.add_argument("--slices", type=int, default=0,
                help="instead: time each of S equal-triple slices of the full space (cost profile)")
args = ap.parse_args()
ds, top_k, planted = bench.make_dataset(args.workload)
M, N = ds.num_snps, ds.num_samples
total = epi3.num_combinations(M, 3)
if args.slices:
    import json
    with epi3.DeviceDataset(ds) as dd:
        out = []
        for a, b in epi3.partition(M, args.slices):
            cfg = epi3.SearchConfig(top_k=top_k, rank_begin=a, rank_end=b, engine=args.engine)
            dd.search(cfg)
            r = min((dd.search(cfg) for _ in range(args.reps)), key=lambda r: r.stats.kernel_ms)
            out.append({"a": a, "b": b, "ms": r.stats.kernel_ms, "total_ms": r.stats.total_device_ms,
                        "batches": r.stats.main_kernel_launches})
    print(json.dumps({"workload": args.workload, "M": M, "N": N, "slices": out}))
    sys.exit(0)
a, b = int(total * args.lo), int(total * args.hi)
cfg = epi3.SearchConfig(top_k=top_k, rank_begin=a, rank_end=b, engine=args.engine)
with epi3.DeviceDataset(ds) as dd:
    first = dd.search(cfg)
    ms = []
    for _ in range(args.reps):
        r = dd.search(cfg)
        assert epi3.same_outcome(first, r)
        ms.append(r.stats.kernel_ms)
best = min(ms)
print(f"{args.tag} {args.workload} [{args.lo},{args.hi}) {(b - a) * N / (best / 1e3) / 1e12:.2f} Tel/s "
      f"kernel {best:.2f} ms (all {[round(x, 2) for x in ms]}) best {first.best.triple}", flush=True)
