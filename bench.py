#!/usr/bin/env python
"""Throughput of the exhaustive 3-way K2 search on B200 (BASELINE.json metric:
tera triplet x sample evaluations per second, elements = C(M,3) * N,
/root/reference/proj/src/bench.cpp:26-30).

Workload (default: BASELINE.json configs[2], the config the metric's
1/2/4/8-GPU figures are quoted on): 8192 SNPs x 16384 samples, 8192 controls /
8192 cases, maf 0.3, planted (1024, 4096, 7168); synthetic (the reference HWE
generator + exact class counts). A STEP IS ONE COMPLETE SEARCH of the workload
(all C(M,3) triples, top-k), split across the N ranks into contiguous
triple-rank ranges (strong scaling: total work is fixed, each rank searches
1/N of it; planes replicated; one all-gather merges the top-k).

  value  C(M,3)*N*K / max over ranks of the device time (CUDA events on the
         search stream) of the K timed searches; planes + marginal index
         resident in HBM, L2 flushed (256 MiB write) before every step.
  e2e    the same K steps through the C ABI from pinned HOST buffers: dataset
         create (H2D planes, repack, marginal index), search, D2H top-k and
         (N > 1) the all-gather merge; barrier + synchronize around the region,
         max over ranks.

Self-check (after the timed region, fails the run loudly): every step returns
the identical outcome; the top-k re-scores bit-identically through
e3_scores (a separate kernel); the device counted C(M,3) evaluations.

`--impl reference` times the reference's own CPU implementation
(oracle/_ref/epi3_ref = the unmodified /root/reference sources) on the box's
host cores, on a bounded sample of the same workload (first 512 SNPs, all
samples), input built by the oracle alone (no product library).

`--gpus N` without a torchrun environment re-launches itself under
torch.distributed.run with N ranks.
"""
from __future__ import annotations

import argparse
import json
import os
import socket
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
MAF = 0.3
CPU_SAMPLE_SNPS = 512
REF_VARIANTS = ("v2", "v3", "v4")  # v4 = the reference default (epi3_main.cpp:350)
POPC_PER_SM_CLK = 16.0  # measured: tools/ipipe_bench.cu, profiles/r01_ipipe.txt
ALG_POPC_PER_ELEMENT = 27.0 / 32.0  # 27 POPC per triple per 32-sample word
TC_OPS_PER_ELEMENT = 16.0  # masked tensor engine: 8 int8 MACs per triplet x sample
# ncu evidence for the SYRK kernel's binding unit (NOT measured by this run)
SYRK_PROFILE = ROOT / "profiles" / "syrk_profile.json"


def env_int(name, default):
    return int(os.environ.get(name, default))


def plant_of(name):
    M, N, n1, seed, top_k = WORKLOADS[name]
    p_other = 0.468 if 2 * n1 == N else 0.198
    return (M // 8, M // 2, 7 * M // 8), p_other


def describe(name):
    M, N, n1, seed, top_k = WORKLOADS[name]
    triple, p_other = plant_of(name)
    return (f"{name}: {M} SNPs x {N} samples ({N - n1} controls / {n1} cases), maf {MAF}, "
            f"seed {seed}, planted {triple} target (1,1,1) p={0.9}/{p_other}")


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


# ---------------------------------------------------------------------------
# CPU legs (the only places bench.py runs oracle/ code: input for, and
# timing of, the reference's own CPU implementation)
# ---------------------------------------------------------------------------


def cpu_sample(name, workdir):
    """First CPU_SAMPLE_SNPS SNPs x all samples of the workload as an EPI3
    file, built with the oracle (reference generator + exact class counts);
    byte-identical to the product's input (tests/test_oracle.py)."""
    sys.path.insert(0, str(ROOT / "oracle"))
    import py_oracle as po
    M, N, n1, seed, top_k = WORKLOADS[name]
    triple, p_other = plant_of(name)
    m = min(CPU_SAMPLE_SNPS, M)
    f = Path(workdir) / f"{name}_cpu_sample.epi3"
    po.workload_sample(f, M, N, n1, MAF, seed, triple, p_other, m)
    return f, m, N


def c3(m):
    return m * (m - 1) * (m - 2) // 6


def run_reference_cpu(path, m, n, variants=REF_VARIANTS, top_k=10, repeats=1):
    """oracle/_ref/epi3_ref = the unmodified reference run_search, all host
    threads; min over repeats per variant (bench.cpp:22-24)."""
    sys.path.insert(0, str(ROOT / "oracle"))
    import py_oracle as po
    threads = os.cpu_count() or 1
    per = {}
    for v in variants:
        r = po.ref_run("search", path, v, threads, top_k, repeats)
        per[v] = {"seconds": min(r["elapsed_s"]), "best": r["best"]["triple"]}
    elements = c3(m) * n
    for v in per:
        per[v]["value"] = elements / per[v]["seconds"] / 1e12
    best_v = min(per, key=lambda v: per[v]["seconds"])
    return {"value": per[best_v]["value"], "unit": UNIT, "cores": threads, "kind": "reference",
            "variant": best_v, "seconds": per[best_v]["seconds"],
            "variants": {v: round(per[v]["value"], 6) for v in per},
            "default_variant_v4": per.get("v4", {}).get("value"),
            "sample": f"first {m} SNPs x all {n} samples of the workload, full search "
                      f"(C({m},3)*{n} = {elements:.4g} elements), reference run_search, "
                      f"best of variants {list(variants)} ({best_v}), threads={threads}, "
                      f"min of {repeats} repeat(s)"}


def bench_reference(args, rank, world):
    if rank != 0:
        return
    if not (ROOT / "oracle" / "_ref" / "epi3_ref").exists():
        print(json.dumps({"impl": "reference", "unavailable": "oracle/_ref/epi3_ref not built"}))
        return
    top_k = WORKLOADS[args.workload][4]
    with tempfile.TemporaryDirectory() as d:
        f, m, N = cpu_sample(args.workload, d)
        # warm-up: every variant once; the steps then time the fastest one
        probe = run_reference_cpu(f, m, N, top_k=top_k)
        for _ in range(max(0, args.warmup - 1)):
            run_reference_cpu(f, m, N, variants=(probe["variant"],), top_k=top_k)
        secs = []
        for _ in range(args.steps):
            r = run_reference_cpu(f, m, N, variants=(probe["variant"],), top_k=top_k)
            secs.append(r["seconds"])
    elements = c3(m) * N
    value = elements * args.steps / sum(secs) / 1e12
    line = {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": 0, "impl": "reference",
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * sum(secs) / args.steps,
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None,
            "dtype": "u64 (popcount) + f64 (K2)", "data": "synthetic",
            "config": {"workload": describe(args.workload), "top_k": top_k,
                       "step": f"reference run_search ({probe['variant']}, the fastest of "
                               f"{list(REF_VARIANTS)} in warm-up; all host threads) over the "
                               f"bounded sample: first {m} SNPs x {N} samples"},
            "cpu_baseline": {"value": value, "unit": UNIT, "cores": probe["cores"],
                             "kind": "reference", "sample": probe["sample"],
                             "variants": probe["variants"]},
            "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0,
                    "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


# ---------------------------------------------------------------------------
# multi-rank launch
# ---------------------------------------------------------------------------


def relaunch_under_torchrun(args):
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
           f"--nproc-per-node={args.gpus}", "--master-addr", "127.0.0.1",
           "--master-port", str(port), str(Path(__file__).resolve())] + sys.argv[1:]
    return subprocess.call(cmd)


# ---------------------------------------------------------------------------
# the product arm
# ---------------------------------------------------------------------------


def make_dataset(name):
    from paper_2201_10956_b200 import epi3
    M, N, n1, seed, top_k = WORKLOADS[name]
    triple, p_other = plant_of(name)
    plant = epi3.PlantSpec(triple, (1, 1, 1), 0.9, p_other)
    geno, pheno = epi3.generate_synthetic(M, N, MAF, seed, plant, exact_cases=n1)
    ds = epi3.binarize(geno, pheno)
    return ds, top_k, triple


def syrk_macs_model(ds):
    """Exact count of the SYRK engine's fp4 MACs: per triple with first SNP i,
    4 (b,g) MACs per compacted sample, i.e. per sample in the two smaller
    genotype phases of SNP i per class (the largest is recovered exactly)."""
    M = ds.num_snps

    def popc64(x):
        return np.unpackbits(x.view(np.uint8), axis=-1).sum(axis=-1, dtype=np.int64)
    snp_ones = np.zeros(M, dtype=np.float64)
    for planes, n_c in ((ds.ctrl, ds.num_controls), (ds.cases, ds.num_cases)):
        g = popc64(planes)                      # [M, 2]: genotype 0, 1 counts
        g3 = np.stack([g[:, 0], g[:, 1], n_c - g[:, 0] - g[:, 1]], axis=1)
        snp_ones += (n_c - g3.max(axis=1)).astype(np.float64)
    ii = np.arange(M, dtype=np.float64)
    first_rank = c3(float(M)) - (M - ii) * (M - ii - 1) * (M - ii - 2) / 6.0
    first_cnt = np.maximum(M - 1 - ii, 0) * np.maximum(M - 2 - ii, 0) / 2.0

    def macs(a, b):
        lo = np.maximum(first_rank, a)
        hi = np.minimum(first_rank + first_cnt, b)
        return float(4.0 * np.sum(np.maximum(hi - lo, 0.0) * snp_ones))
    return macs


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--workload", default="cfg3", choices=sorted(WORKLOADS))
    ap.add_argument("--engine", default="auto", choices=["auto", "syrk", "tc_masked", "popc"],
                    help="auto (default): syrk for N >= 4096 else tc_masked; syrk: compacted "
                         "tcgen05 kind::mxf4 SYRK; tc_masked: tcgen05 GEMM over pair products; "
                         "popc: LOP3/POPC kernel")
    ap.add_argument("--balance-parts", type=int, default=8,
                    help="N=1 only: after the timed region, time the P ranges of the P-GPU "
                         "split (e3_partition_balanced) one by one (max/mean bounds the P-GPU "
                         "efficiency); 0 = off")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    args = ap.parse_args()
    if args.engine == "auto":
        args.engine = "syrk" if WORKLOADS[args.workload][1] >= 4096 else "tc_masked"
    if args.warmup < 3 and args.impl == "ours":
        print(f"warning: --warmup {args.warmup} < 3 (timing rules need >= 3)", file=sys.stderr)

    if "WORLD_SIZE" not in os.environ and args.gpus > 1:
        sys.exit(relaunch_under_torchrun(args))
    rank, world, local = env_int("RANK", 0), env_int("WORLD_SIZE", 1), env_int("LOCAL_RANK", 0)
    if args.impl == "reference":
        return bench_reference(args, rank, world)
    if world != args.gpus:
        raise SystemExit(f"--gpus {args.gpus} but WORLD_SIZE={world}: launch one rank per GPU")

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
    red_dev = torch.device("cuda", local) if backend == "nccl" else torch.device("cpu")

    def barrier():
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()

    ds, top_k, planted = make_dataset(args.workload)
    M, N = ds.num_snps, ds.num_samples
    total = epi3.num_combinations(M, 3)
    my_a, my_b = epi3.partition_balanced(M, world)[rank]
    cfg = epi3.SearchConfig(top_k=top_k, rank_begin=my_a, rank_end=my_b, engine=args.engine)
    l2_flush = torch.empty(256 * 1024 * 1024, dtype=torch.uint8, device="cuda")

    # ---- value: inputs resident in HBM -----------------------------------
    dd = epi3.DeviceDataset(ds, device=local)
    for _ in range(args.warmup):
        dd.search(cfg)
    barrier()
    sampler = ClockSampler(local)
    sampler.start()
    dev_ms, kern_ms, launches, main_launches = 0.0, 0.0, 0, 0
    results = []
    t_wall = time.perf_counter()
    for _ in range(args.steps):
        l2_flush.zero_()
        torch.cuda.synchronize()
        r = dd.search(cfg)
        dev_ms += r.stats.total_device_ms
        kern_ms += r.stats.kernel_ms
        launches += r.stats.kernel_launches
        main_launches += r.stats.main_kernel_launches
        results.append(r)
    barrier()
    wall_s = time.perf_counter() - t_wall
    clocks = sampler.stop()

    # ---- self-check (outside the timed region) ------------------------------
    for r in results[1:]:
        if not epi3.same_outcome(results[0], r):
            raise SystemExit("self-check failed: outcome changed between steps")
    mine = results[0]
    if mine.stats.combinations_evaluated != my_b - my_a:
        raise SystemExit("self-check failed: device evaluation count != range length")
    rescored = dd.scores([h.triple for h in mine.top]) if mine.top else []
    for h, s in zip(mine.top, rescored):
        if float(s).hex() != h.score.hex():
            raise SystemExit(f"self-check failed: {h.triple} scored {h.score.hex()} in the "
                             f"search but {float(s).hex()} by e3_scores")

    # ---- partition balance on one GPU (bounds the P-GPU efficiency) --------
    balance = None
    if world == 1 and args.balance_parts > 1:
        # each range twice, L2 flushed before each, min kept: a single search's
        # device time occasionally includes a host-side stall between its
        # batch launches (one range at ~2x in r02k), which is not range cost
        times, runs = [], []
        for a, b in epi3.partition_balanced(M, args.balance_parts):
            rc = epi3.SearchConfig(top_k=top_k, rank_begin=a, rank_end=b, engine=args.engine)
            ms = []
            for _ in range(2):
                l2_flush.zero_()
                torch.cuda.synchronize()
                ms.append(dd.search(rc).stats.total_device_ms)
            runs.append([round(t, 3) for t in ms])
            times.append(min(ms))
        balance = {"parts": args.balance_parts, "ms": [round(t, 3) for t in times], "runs_ms": runs,
                   "max_over_mean": max(times) / (sum(times) / len(times)),
                   "efficiency_bound": (sum(times) / len(times)) / max(times)}
    dd.close()

    # ---- e2e: C ABI from pinned host buffers ------------------------------
    e2e = None
    merged = None
    if not args.no_e2e:
        import ctypes
        from paper_2201_10956_b200 import partition
        pin_ctrl = torch.from_numpy(ds.ctrl.view(np.int64)).pin_memory()
        pin_cases = torch.from_numpy(ds.cases.view(np.int64)).pin_memory()
        # planes + the host-built log table (f64) and screening table (f32)
        h2d = ds.ctrl.nbytes + ds.cases.nbytes + 12 * (N + 2)
        d2h = top_k * 16 + 12

        def e2e_step():
            with epi3.DeviceDataset(ds, local, ctypes.c_void_p(pin_ctrl.data_ptr()),
                                    ctypes.c_void_p(pin_cases.data_ptr())) as d2:
                r = d2.search(cfg)
            return partition.allgather_merge(r, top_k, device=red_dev) if world > 1 else r
        e2e_step()
        barrier()
        t0 = time.perf_counter()
        for _ in range(args.steps):
            merged = e2e_step()
        barrier()
        e2e = {"secs": time.perf_counter() - t0, "h2d": h2d, "d2h": d2h}
    if merged is None:
        from paper_2201_10956_b200 import partition
        merged = partition.allgather_merge(mine, top_k, device=red_dev) if world > 1 else mine
    if merged.stats.combinations_evaluated != total:
        raise SystemExit("self-check failed: ranks did not evaluate C(M,3) triples in total")

    # ---- reduce timings over ranks (max) ------------------------------------
    t = torch.tensor([dev_ms, kern_ms, e2e["secs"] if e2e else 0.0, wall_s],
                     dtype=torch.float64, device=red_dev)
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    dev_ms, kern_ms, e2e_secs, wall_s = t.tolist()

    if rank == 0:
        elements = total * N * args.steps  # whole job: every rank's share of K searches
        value = elements / (dev_ms / 1e3) / 1e12
        my_elements = (my_b - my_a) * N * args.steps
        f_mhz = clocks["sm_mhz"] or 1965.0
        nsm = torch.cuda.get_device_properties(local).multi_processor_count
        peaks = json.loads((ROOT / "MEASURED_PEAKS.json").read_text()) \
            if (ROOT / "MEASURED_PEAKS.json").exists() else {}
        prof = json.loads(SYRK_PROFILE.read_text()) if SYRK_PROFILE.exists() else {}
        if args.engine in ("syrk", "tc_masked"):
            bf16 = peaks.get("bf16_tflops", 1590.0)
            if args.engine == "tc_masked":
                achieved = my_elements / (kern_ms / 1e3) * TC_OPS_PER_ELEMENT / 1e12
                peak, kind, mult = 2.0 * bf16, "int8", 2
            else:
                macs = syrk_macs_model(ds)(my_a, my_b) * args.steps
                achieved = 2.0 * macs / (kern_ms / 1e3) / 1e12
                peak, kind, mult = 4.0 * bf16, "fp4", 4
            roof = {"bound": "tensor", "unit": "TFLOP/s",
                    "kind": f"{kind} dense, algorithmic",
                    "peak_source": (f"{mult} x MEASURED_PEAKS.json bf16_tflops (burst)" if peaks
                                    else f"{mult} x fallback 1590 TFLOP/s"),
                    "note": ("compacted SYRK: 4 fp4 MACs per triple per compacted sample (the "
                             "two smaller genotype phases of SNP i per class), exact count "
                             "over the timed searches / device time of the search kernels"
                             if args.engine == "syrk" else
                             "masked GEMM: 8 int8 MACs per element")}
            if args.engine == "syrk" and prof.get(args.workload):
                p = prof[args.workload]
                roof["binding_unit_from_profile"] = dict(p.get("binding_unit", {}),
                                                         source=p.get("source"))
        else:
            peak = nsm * POPC_PER_SM_CLK * f_mhz * 1e6 / 1e12
            achieved = my_elements / (kern_ms / 1e3) * ALG_POPC_PER_ELEMENT / 1e12
            roof = {"bound": "int-pipe POPC (SURVEY.md §8(d))", "unit": "T POPC/s",
                    "effective": True,
                    "note": "27-POPC algorithmic basis (may exceed 1); the kernel issues 5 POPC "
                            "per triple-word (marginal subtraction + carry-save)"}
        traffic = None
        if args.engine == "syrk" and prof.get(args.workload, {}).get("dram_bytes_per_triple"):
            p = prof[args.workload]
            # ncu DRAM read+write per triple (one --set full capture) x this
            # run's triples per search-kernel launch: profile-derived, not live
            traffic = p["dram_bytes_per_triple"] * (my_b - my_a) * args.steps / max(1, main_launches)
        # the POPC-roofline view SURVEY.md §8(d) asks for (effective: the
        # engines count 8 of 27 cells, on tensor cores)
        popc_roof = 148 * POPC_PER_SM_CLK * f_mhz * 1e6 * 32.0 / 27.0 / 1e12
        cpu = None
        if world == 1 and not args.no_cpu:
            with tempfile.TemporaryDirectory() as d:
                f, m, n = cpu_sample(args.workload, d)
                cpu = run_reference_cpu(f, m, n, top_k=top_k)
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": dev_ms / args.steps, "higher_is_better": True, "scaling": "strong",
            "vs_baseline": None,
            "dtype": {"syrk": "e2m1 (0/1 fp4 MMA, exact f32 accumulate) + f64 (K2)",
                      "tc_masked": "u8 (0/1 int8 MMA, s32 accumulate) + f64 (K2)",
                      "popc": "u32 (bit-plane LOP3/POPC) + f64 (K2)"}[args.engine],
            "data": "synthetic",
            "config": {"workload": describe(args.workload), "top_k": top_k,
                       "step": f"one complete search (C({M},3) = {total} triples x {N} samples) "
                               f"split into {world} contiguous triple-rank range(s), one per GPU",
                       "l2": "flushed between timed steps (256 MiB write); planes stay "
                             "L2-resident inside a step by design",
                       "index": "marginal index (pair/single plane counts) built at dataset "
                                "load: outside `value`, inside `e2e`",
                       "parallelism": f"dp{world} (triple-rank ranges, planes replicated)"},
            "clocks": clocks,
            "gpu_launches": launches,
            "wall_ms_per_step": wall_s * 1e3 / args.steps,
            "e2e": None if e2e is None else {
                "value": elements / e2e_secs / 1e12, "unit": UNIT,
                "h2d_bytes_per_step": e2e["h2d"], "d2h_bytes_per_step": e2e["d2h"],
                "ms_per_step": e2e_secs * 1e3 / args.steps},
            "roofline": dict(roof, achieved=achieved, peak=peak, frac=achieved / peak,
                             engine=args.engine, kernel_ms_per_step=kern_ms / args.steps,
                             kernel_launches_per_step=main_launches / args.steps,
                             traffic=traffic,
                             traffic_note="ncu dram read+write per triple from "
                                          "profiles/syrk_profile.json x triples per launch"
                                          if traffic else None),
            "popc_roofline_effective": {"achieved": value / world, "peak": popc_roof,
                                        "unit": "Tel/s per GPU",
                                        "frac": value / world / popc_roof,
                                        "note": "SURVEY.md §8(d): 27 POPC per triple-word at "
                                                "16 POPC/clk/SM x 148 SMs x the sampled clock"},
            "cpu_baseline": cpu,
            "partition_balance": balance,
            "self_check": {"steps_identical": True, "rescored_bit_identical": len(rescored),
                           "combinations": merged.stats.combinations_evaluated,
                           "planted": list(planted),
                           "planted_is_best": tuple(merged.best.triple) == tuple(planted)},
            "best": {"triple": list(merged.best.triple), "k2": merged.best.score,
                     "merged_over_ranks": world},
        }
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
