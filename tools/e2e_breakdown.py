"""Times the e2e building blocks on cuda:0 exactly as bench.py's e2e loop
runs them: dataset create (H2D + repack + marginal index), one search slice,
destroy — per step, for a workload and a range of slices."""
import ctypes
import sys
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
import torch  # noqa: E402
import bench  # noqa: E402
from paper_2201_10956_b200 import epi3  # noqa: E402

w = sys.argv[1] if len(sys.argv) > 1 else "cfg3"
first = int(sys.argv[2]) if len(sys.argv) > 2 else 0
ds, top_k, _ = bench.make_dataset(w)
pin_c = torch.from_numpy(ds.ctrl.view("int64")).pin_memory()
pin_k = torch.from_numpy(ds.cases.view("int64")).pin_memory()
slices = epi3.partition(ds.num_snps, 64)
keep = epi3.DeviceDataset(ds, 0) if "--keep" in sys.argv else None  # as bench.py: value dataset alive
tot = [0.0, 0.0, 0.0]
for rep in range(first, first + 4):
    t0 = time.perf_counter()
    dd = epi3.DeviceDataset(ds, 0, ctypes.c_void_p(pin_c.data_ptr()), ctypes.c_void_p(pin_k.data_ptr()))
    t1 = time.perf_counter()
    r = dd.search(epi3.SearchConfig(top_k=top_k, rank_begin=slices[rep][0], rank_end=slices[rep][1]))
    t2 = time.perf_counter()
    dd.close()
    t3 = time.perf_counter()
    if rep > first:
        tot = [tot[0] + t1 - t0, tot[1] + t2 - t1, tot[2] + t3 - t2]
    print(f"{w} slice {rep}: create {1e3*(t1-t0):.2f} ms, search {1e3*(t2-t1):.2f} ms "
          f"(device {r.stats.total_device_ms:.2f} ms, {r.stats.kernel_launches} launches), "
          f"destroy {1e3*(t3-t2):.2f} ms")
print(f"{w} mean of last 3: create {tot[0]/3e-3:.2f} search {tot[1]/3e-3:.2f} destroy {tot[2]/3e-3:.2f} ms")
