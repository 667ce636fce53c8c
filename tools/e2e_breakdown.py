"""Times the e2e building blocks on cuda:0: dataset create (H2D + repack +
marginal index) and destroy, and one search slice, for a workload."""
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
ds, desc, top_k = bench.make_dataset(w)
pin_c = torch.from_numpy(ds.ctrl.view("int64")).pin_memory()
pin_k = torch.from_numpy(ds.cases.view("int64")).pin_memory()
slices = epi3.partition(ds.num_snps, 64)
for rep in range(4):
    t0 = time.perf_counter()
    dd = epi3.DeviceDataset(ds, 0, ctypes.c_void_p(pin_c.data_ptr()), ctypes.c_void_p(pin_k.data_ptr()))
    t1 = time.perf_counter()
    r = dd.search(epi3.SearchConfig(top_k=top_k, rank_begin=slices[rep][0], rank_end=slices[rep][1]))
    t2 = time.perf_counter()
    dd.close()
    t3 = time.perf_counter()
    print(f"{w} rep {rep}: create {1e3*(t1-t0):.1f} ms, search {1e3*(t2-t1):.1f} ms "
          f"(device {r.stats.total_device_ms:.1f} ms), destroy {1e3*(t3-t2):.1f} ms")
