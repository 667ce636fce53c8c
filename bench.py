#!/usr/bin/env python
"""Throughput of the exhaustive 3-way K2 search on B200 (BASELINE.json metric:
tera triplet x sample evaluations per second).

Workload (BASELINE.json configs[2], the one the metric's 1/2/4/8-GPU figures are
quoted on): 8192 SNPs x 16384 samples, 8192 controls / 8192 cases, maf 0.3,
planted (1024, 4096, 7168); synthetic (reference HWE generator + exact class
counts). A step is one C-ABI search over a contiguous 1/SLICES slice of the
lexicographic triple-rank space per GPU (weak scaling: every rank does a
fixed slice per step; successive steps walk successive slices).

  value  device time (CUDA events on the search stream) of the K timed
         searches, planes + marginal index already resident in HBM.
  e2e    the same steps through the C ABI from pinned HOST buffers: dataset
         create (H2D planes, repack, marginal index) + search + D2H top-k,
         host wall clock, barrier + synchronize around the region.

`--impl reference` times the reference's own CPU implementation
(oracle/_ref/epi3_ref = the unmodified /root/reference sources) on the box's
host cores, on a bounded sample of the same workload (first 512 SNPs, all
16384 samples).
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import tempfile
import threading
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

METRIC = "tera triplet×sample evals/s (3-way K2 search) at 1/2/4/8 B200 vs CPU ref"
UNIT = "Tel/s"
WORKLOADS = {
    # name: (M, N, cases, seed, top_k)
    "cfg1": (256, 1024, 512, 1001, 10),
    "cfg2": (2048, 4096, 2048, 1002, 10),
    "cfg3": (8192, 16384, 8192, 1003, 10),
    "cfg4": (1024, 262144, 131072, 1004, 10),
    "cfg5": (4096, 32768, 8192, 1005, 100),
}
CPU_SAMPLE_SNPS = 512
POPC_PER_SM_CLK = 16.0  # measured: tools/ipipe_bench.cu, profiles/r01_ipipe.txt
ALG_POPC_PER_ELEMENT = 27.0 / 32.0  # 27 POPC per triple per 32-sample word
TC_OPS_PER_ELEMENT = 16.0  # tensor engine: 8 int8 MACs per triplet x sample


def env_int(name, default):
    return int(os.environ.get(name, default))


class ClockSampler(threading.Thread):
    """nvidia-smi-equivalent clock/throttle sampling (NVML) during the timed region."""

    def __init__(self, device):
        super().__init__(daemon=True)
        self.device = device
        self.samples = []
        self.reasons = set()
        self.max_mhz = None
        self._halt = threading.Event()

    def run(self):
        try:
            import pynvml
            pynvml.nvmlInit()
            h = pynvml.nvmlDeviceGetHandleByIndex(self.device)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(h, pynvml.NVML_CLOCK_SM)
            names = {
                "gpu_idle": 0x1, "applications_clocks_setting": 0x2, "sw_power_cap": 0x4,
                "hw_slowdown": 0x8, "sync_boost": 0x10, "sw_thermal_slowdown": 0x20,
                "hw_thermal_slowdown": 0x40, "hw_power_brake_slowdown": 0x80,
            }
            while not self._halt.is_set():
                self.samples.append(pynvml.nvmlDeviceGetClockInfo(h, pynvml.NVML_CLOCK_SM))
                r = pynvml.nvmlDeviceGetCurrentClocksEventReasons(h)
                for n, bit in names.items():
                    if r & bit and n != "gpu_idle":
                        self.reasons.add(n)
                time.sleep(0.1)
        except Exception as e:  # noqa: BLE001 - clocks are evidence, not a dependency
            self.reasons.add(f"nvml-unavailable: {e}")

    def stop(self):
        self._halt.set()
        self.join(timeout=2)
        med = statistics.median(self.samples) if self.samples else None
        return {"sm_mhz": med, "sm_max_mhz": self.max_mhz, "reasons": sorted(self.reasons),
                "samples": len(self.samples)}


def make_dataset(name):
    from paper_2201_10956_b200 import epi3
    M, N, n1, seed, top_k = WORKLOADS[name]
    p_other = 0.468 if 2 * n1 == N else 0.198
    plant = epi3.PlantSpec((M // 8, M // 2, 7 * M // 8), (1, 1, 1), 0.9, p_other)
    geno, pheno = epi3.generate_synthetic(M, N, 0.3, seed, plant, exact_cases=n1)
    ds = epi3.binarize(geno, pheno)
    del geno
    desc = (f"{name}: {M} SNPs x {N} samples ({N - n1} controls / {n1} cases), maf 0.3, "
            f"seed {seed}, planted {plant.triple} target (1,1,1) p={plant.p_case_match}/{p_other}")
    return ds, desc, top_k


def cpu_reference_sample(ds, workdir):
    """Bounded sample of the workload for the CPU reference: first
    CPU_SAMPLE_SNPS SNPs, all samples, written in the reference's format."""
    from paper_2201_10956_b200 import epi3
    m = min(CPU_SAMPLE_SNPS, ds.num_snps)
    sub = epi3.BitPlaneDataset(m, ds.num_controls, ds.num_cases,
                               np.ascontiguousarray(ds.ctrl[:m]), np.ascontiguousarray(ds.cases[:m]))
    f = Path(workdir) / "cpu_sample.epi3"
    epi3.write_packed(f, sub)
    return f, m


def run_reference_cpu(path, m, n, variants=("v2", "v3"), top_k=10, repeats=1):
    """oracle/_ref/epi3_ref = unmodified reference run_search; best variant."""
    sys.path.insert(0, str(ROOT / "oracle"))
    import py_oracle as po
    threads = os.cpu_count() or 1
    best = None
    for v in variants:
        r = po.ref_run("search", path, v, threads, top_k, repeats)
        t = min(r["elapsed_s"])
        if best is None or t < best[0]:
            best = (t, v, r)
    from paper_2201_10956_b200 import epi3
    elements = epi3.num_combinations(m, 3) * n
    return {"value": elements / best[0] / 1e12, "unit": UNIT, "cores": threads,
            "kind": "reference", "variant": best[1], "seconds": best[0],
            "sample": f"first {m} SNPs x all {n} samples of the workload, full search "
                      f"(C({m},3)*{n} = {elements:.4g} elements), reference run_search "
                      f"variant {best[1]} (best of {list(variants)}), threads={threads}"}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--workload", default="cfg3", choices=sorted(WORKLOADS))
    ap.add_argument("--slices", type=int, default=64,
                    help="a step searches 1/SLICES of the triple-rank space per GPU")
    ap.add_argument("--engine", default="auto", choices=["auto", "syrk", "tc_masked", "popc"],
                    help="auto (default): syrk for N >= 4096 else tc_masked; syrk: compacted "
                         "tcgen05 kind::mxf4 SYRK; tc_masked: tcgen05 GEMM over pair products; "
                         "popc: LOP3/POPC kernel")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    args = ap.parse_args()
    if args.engine == "auto":
        args.engine = "syrk" if WORKLOADS[args.workload][1] >= 4096 else "tc_masked"

    rank, world, local = env_int("RANK", 0), env_int("WORLD_SIZE", 1), env_int("LOCAL_RANK", 0)

    if args.impl == "reference":
        return bench_reference(args, rank, world)

    import torch
    import torch.distributed as dist
    from paper_2201_10956_b200 import epi3

    # E3_BENCH_BACKEND=gloo lets the multi-rank path be exercised with ranks
    # sharing one GPU (testing only; NCCL needs one GPU per rank)
    backend = os.environ.get("E3_BENCH_BACKEND", "nccl")
    local = local % max(1, torch.cuda.device_count())
    torch.cuda.set_device(local)
    if world > 1:
        if backend == "nccl":
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        else:
            dist.init_process_group(backend)
    red_dev = "cuda" if backend == "nccl" else "cpu"

    def barrier():
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()

    ds, desc, top_k = make_dataset(args.workload)
    M, N = ds.num_snps, ds.num_samples
    total = epi3.num_combinations(M, 3)
    slices = epi3.partition(M, args.slices)

    def slice_of(step):
        return slices[(step * world + rank) % args.slices]

    l2_flush = torch.empty(256 * 1024 * 1024, dtype=torch.uint8, device="cuda")

    # ---- value: inputs resident in HBM -----------------------------------
    dd = epi3.DeviceDataset(ds, device=local)
    for s in range(args.warmup):
        a, b = slice_of(s)
        dd.search(epi3.SearchConfig(top_k=top_k, rank_begin=a, rank_end=b, engine=args.engine))
    barrier()
    sampler = ClockSampler(local)
    sampler.start()
    dev_ms, kern_ms, launches, elements = 0.0, 0.0, 0, 0
    syrk_macs = 0.0
    snp_ones = None
    if args.engine == "syrk":
        # per SNP i: compacted samples the SYRK engine multiplies = per class the
        # two smaller genotype phases of i (the largest is recovered exactly)
        def popc64(x):
            return np.unpackbits(x.view(np.uint8), axis=-1).sum(axis=-1, dtype=np.int64)
        snp_ones = np.zeros(M, dtype=np.float64)
        for planes, n_c in ((ds.ctrl, ds.num_controls), (ds.cases, ds.num_cases)):
            g = popc64(planes)                      # [M, 2]: genotype 0, 1 counts
            g3 = np.stack([g[:, 0], g[:, 1], n_c - g[:, 0] - g[:, 1]], axis=1)
            snp_ones += (n_c - g3.max(axis=1)).astype(np.float64)
        ii = np.arange(M, dtype=np.float64)
        c3 = lambda n: n * (n - 1) * (n - 2) / 6.0
        first_rank = c3(float(M)) - c3(M - ii)
        first_cnt = np.maximum(M - 1 - ii, 0) * np.maximum(M - 2 - ii, 0) / 2.0

    def compacted_macs(a, b):
        lo = np.maximum(first_rank, a)
        hi = np.minimum(first_rank + first_cnt, b)
        return float(4.0 * np.sum(np.maximum(hi - lo, 0.0) * snp_ones))
    results = []
    for s in range(args.steps):
        l2_flush.zero_()
        torch.cuda.synchronize()
        a, b = slice_of(args.warmup + s)
        r = dd.search(epi3.SearchConfig(top_k=top_k, rank_begin=a, rank_end=b, engine=args.engine))
        dev_ms += r.stats.total_device_ms
        kern_ms += r.stats.kernel_ms
        launches += r.stats.kernel_launches
        elements += (b - a) * N
        if snp_ones is not None:
            syrk_macs += compacted_macs(a, b)
        results.append(r)
    barrier()
    clocks = sampler.stop()

    # ---- e2e: C ABI from pinned host buffers ------------------------------
    e2e = None
    if not args.no_e2e:
        import ctypes
        pin_ctrl = torch.from_numpy(ds.ctrl.view(np.int64)).pin_memory()
        pin_cases = torch.from_numpy(ds.cases.view(np.int64)).pin_memory()
        h2d = ds.ctrl.nbytes + ds.cases.nbytes + 8 * (N + 2) + 8 * (M - 1)
        d2h = top_k * 16 + 4
        for s in range(min(1, args.warmup)):
            a, b = slice_of(s)
            with epi3.DeviceDataset(ds, local, ctypes.c_void_p(pin_ctrl.data_ptr()),
                                    ctypes.c_void_p(pin_cases.data_ptr())) as d2:
                d2.search(epi3.SearchConfig(top_k=top_k, rank_begin=a, rank_end=b, engine=args.engine))
        barrier()
        t0 = time.perf_counter()
        e2e_el = 0
        for s in range(args.steps):
            a, b = slice_of(args.warmup + s)
            with epi3.DeviceDataset(ds, local, ctypes.c_void_p(pin_ctrl.data_ptr()),
                                    ctypes.c_void_p(pin_cases.data_ptr())) as d2:
                d2.search(epi3.SearchConfig(top_k=top_k, rank_begin=a, rank_end=b, engine=args.engine))
            e2e_el += (b - a) * N
        barrier()
        e2e_s = time.perf_counter() - t0
        e2e = {"secs": e2e_s, "elements": e2e_el, "h2d": h2d, "d2h": d2h}

    # ---- reduce over ranks (max time) --------------------------------------
    t = torch.tensor([dev_ms, kern_ms, e2e["secs"] if e2e else 0.0], dtype=torch.float64,
                     device=red_dev)
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        # the one collective of the search: all-gather + merge of the top-k
        from paper_2201_10956_b200 import partition
        merged = partition.allgather_merge(results[-1], top_k)
    else:
        merged = results[-1]
    dev_ms, kern_ms, e2e_secs = t.tolist()
    tot_elements = elements * world

    if rank == 0:
        value = tot_elements / (dev_ms / 1e3) / 1e12
        kernel_rate = elements / (kern_ms / 1e3)  # one GPU's elements per second in the kernel
        f_mhz = clocks["sm_mhz"] or 1965.0
        nsm = torch.cuda.get_device_properties(local).multi_processor_count
        peaks = json.loads((ROOT / "MEASURED_PEAKS.json").read_text()) \
            if (ROOT / "MEASURED_PEAKS.json").exists() else {}
        if args.engine in ("syrk", "tc_masked"):
            bf16 = peaks.get("bf16_tflops", 1590.0)
            if args.engine == "tc_masked":
                # masked GEMM: 8 int8 MACs (16 ops) per triplet x sample
                achieved = kernel_rate * TC_OPS_PER_ELEMENT / 1e12
                peak, kind = 2.0 * bf16, "int8"  # dense int8 = 2x dense bf16 on B200
            else:
                # compacted SYRK: 4 fp4 MACs per (triple, compacted sample), exact count
                achieved = 2.0 * syrk_macs / (kern_ms / 1e3) / 1e12
                peak, kind = 4.0 * bf16, "fp4"   # dense fp4 (kind::mxf4) = 4x dense bf16
            mult = 2 if kind == "int8" else 4
            roof = {"bound": "tensor", "unit": f"TFLOP/s ({kind} dense, algorithmic)",
                    "peak_source": (f"{mult} x MEASURED_PEAKS.json bf16_tflops (burst)" if peaks
                                    else f"{mult} x fallback 1590 TFLOP/s"),
                    "note": ("compacted SYRK: 4 fp4 MACs per triple per compacted sample, i.e. "
                             "per sample in the two smaller genotype phases of SNP i per class "
                             "(exact count over the timed slices)"
                             if args.engine == "syrk" else
                             "masked GEMM: 8 int8 MACs per element (4 (a,b) pair rows x 2 g "
                             "columns)") + "; the other cells come exactly from the marginal "
                                           "index"}
            if args.engine == "syrk":
                # the tensor pipe is not what binds this kernel: ncu shows the L1
                # LSU data path (the K2 screen's shared-memory gathers, operand
                # stores, scratch/pair loads) as the busiest unit
                roof["binding_unit"] = {
                    "unit": "L1TEX LSU data path (l1tex__data_pipe_lsu_wavefronts)",
                    "pct_of_peak": 71.8, "issue_slots_pct": 56.2, "tensor_pipe_pct": 19.7,
                    "from": "profiles/r01wg_search_cfg3_raw.csv (ncu --set full, cfg3)"}
        else:
            peak = nsm * POPC_PER_SM_CLK * f_mhz * 1e6 / 1e12
            achieved = kernel_rate * ALG_POPC_PER_ELEMENT / 1e12
            roof = {"bound": "int-pipe POPC (SURVEY.md §8(d))", "unit": "T POPC/s (algorithmic, 27/word)",
                    "effective": True,
                    "issued_frac": kernel_rate * (5.0 / 32.0) / 1e12 / peak,
                    "note": "27-POPC algorithmic basis (may exceed 1); the kernel issues 5 POPC "
                            "per triple-word (marginal subtraction + carry-save)"}
        traffic = None
        prof = ROOT / "profiles" / "roofline_traffic.json"
        if prof.exists():
            t = json.loads(prof.read_text()).get(args.workload, {}).get(args.engine)
            if t:  # ncu dram read+write of one launch, scaled to this step's triples
                traffic = {"dram_bytes_per_launch": t["dram_bytes_per_triple"] * elements / N
                           / args.steps, "from": t["report"] + " (per-triple, scaled)"}
        cpu = None
        if world == 1 and not args.no_cpu:
            with tempfile.TemporaryDirectory() as d:
                f, m = cpu_reference_sample(ds, d)
                cpu = run_reference_cpu(f, m, N, top_k=top_k)
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": dev_ms / args.steps, "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None,
            "dtype": {"syrk": "e2m1 (0/1 fp4 MMA, exact f32 accumulate) + f64 (K2)",
                      "tc_masked": "u8 (0/1 int8 MMA, s32 accumulate) + f64 (K2)",
                      "popc": "u32 (bit-plane LOP3/POPC) + f64 (K2)"}[args.engine],
            "data": "synthetic",
            "config": {"workload": desc, "top_k": top_k,
                       "step": f"one search over a 1/{args.slices} triple-rank slice "
                               f"({total // args.slices} triples) per GPU",
                       "l2": "flushed between timed steps (256 MiB write); planes 32 MiB "
                             "stay L2-resident inside a step by design",
                       "index": "marginal index (pair/single plane counts) built at dataset "
                                "load: outside `value`, inside `e2e`",
                       "parallelism": f"dp{world} (triple-rank ranges)"},
            "clocks": clocks,
            "gpu_launches": launches,
            "e2e": None if e2e is None else {
                "value": e2e["elements"] * world / e2e_secs / 1e12, "unit": UNIT,
                "h2d_bytes_per_step": e2e["h2d"], "d2h_bytes_per_step": e2e["d2h"],
                "ms_per_step": e2e_secs * 1e3 / args.steps},
            "roofline": dict(roof, achieved=achieved, peak=peak, frac=achieved / peak,
                             engine=args.engine, kernel_ms_per_step=kern_ms / args.steps,
                             traffic=traffic),
            "cpu_baseline": cpu,
            "last_step_best": {"triple": list(merged.best.triple), "k2": merged.best.score,
                               "merged_over_ranks": world},
        }
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


def bench_reference(args, rank, world):
    if rank != 0:
        return
    if not (ROOT / "oracle" / "_ref" / "epi3_ref").exists():
        print(json.dumps({"impl": "reference", "unavailable": "oracle/_ref/epi3_ref not built"}))
        return
    ds, desc, top_k = make_dataset(args.workload)
    N = ds.num_samples
    with tempfile.TemporaryDirectory() as d:
        f, m = cpu_reference_sample(ds, d)
        for _ in range(args.warmup):
            run_reference_cpu(f, m, N, variants=("v3",), top_k=top_k)
        secs = []
        res = None
        for _ in range(args.steps):
            res = run_reference_cpu(f, m, N, variants=("v3",), top_k=top_k)
            secs.append(res["seconds"])
    from paper_2201_10956_b200 import epi3
    elements = epi3.num_combinations(m, 3) * N
    value = elements * args.steps / sum(secs) / 1e12
    line = {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": 0, "impl": "reference",
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * sum(secs) / args.steps,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
            "dtype": "u64 (popcount) + f64 (K2)", "data": "synthetic",
            "config": {"workload": desc, "top_k": top_k,
                       "step": f"reference run_search (v3, all host threads) over the bounded "
                               f"sample: first {m} SNPs x {N} samples"},
            "cpu_baseline": {"value": value, "unit": UNIT, "cores": res["cores"],
                             "kind": "reference", "sample": res["sample"]},
            "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0,
                    "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


if __name__ == "__main__":
    main()
