#!/usr/bin/env python
"""Summarise ncu captures brought back in gpurun_out/ into profiles/.

usage: python tools/ncu_summary.py TAG
  reads  gpurun_out/TAG_launches.csv, gpurun_out/TAG_*.ncu-rep
  writes profiles/TAG_launches.csv (copied), profiles/TAG_<kernel>_raw.csv,
         profiles/TAG_ncu_summary.md
"""
import csv
import io
import shutil
import subprocess
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
OUT, PROF = ROOT / "gpurun_out", ROOT / "profiles"

KEYS = [
    ("gpu__time_duration.sum", "duration"),
    ("sm__cycles_elapsed.avg.per_second", "SM clock"),
    ("sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active", "XU pipe (POPC) % of peak"),
    ("sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active", "ALU pipe (LOP3/IADD3) % of peak"),
    ("sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active", "FMA pipe % of peak"),
    ("sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active", "LSU pipe % of peak"),
    ("sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active", "tensor pipe % of peak"),
    ("smsp__issue_active.avg.pct_of_peak_sustained_active", "issue slots busy %"),
    ("sm__warps_active.avg.pct_of_peak_sustained_active", "achieved occupancy %"),
    ("launch__registers_per_thread", "registers/thread"),
    ("launch__grid_size", "grid"),
    ("dram__bytes_read.sum", "DRAM read"),
    ("dram__bytes_write.sum", "DRAM write"),
    ("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "DRAM % of peak"),
    ("l1tex__t_sector_hit_rate.pct", "L1 hit rate"),
    ("lts__t_sector_hit_rate.pct", "L2 hit rate"),
    ("l1tex__data_pipe_lsu_wavefronts_mem_shared.sum", "shared-memory wavefronts"),
    ("l1tex__data_pipe_tc_wavefronts_mem_shared.sum", "tensor-core shared-memory wavefronts"),
    ("l1tex__throughput.avg.pct_of_peak_sustained_active", "L1TEX throughput % of peak"),
    ("sm__pipe_tensor_subpipe_hmma_cycles_active.avg.pct_of_peak_sustained_active",
     "tensor (hmma/fp4) subpipe % of peak"),
    ("smsp__inst_executed.sum", "warp instructions"),
]


def raw(rep: Path):
    txt = subprocess.run(["ncu", "-i", str(rep), "--page", "raw", "--csv"], capture_output=True,
                         text=True, check=True).stdout
    rows = list(csv.reader(io.StringIO(txt)))
    return txt, rows[0], rows[1], rows[2:]


def main(tag: str) -> None:
    PROF.mkdir(exist_ok=True)
    md = [f"# ncu summary {tag}", ""]
    launches = OUT / f"{tag}_launches.csv"
    if launches.exists():
        shutil.copy(launches, PROF / launches.name)
        rows = [r for r in csv.reader(open(launches)) if len(r) > 10]
        hdr = rows[0]
        tot = {}
        for r in rows[1:]:
            d = dict(zip(hdr, r))
            name = d["Kernel Name"].split("(")[0].replace("<unnamed>::", "")
            tot[name] = tot.get(name, 0.0) + float(d["Metric Value"].replace(",", ""))
        allns = sum(tot.values())
        md += ["## Launch list (gpu__time_duration, cold, serialised: read the SHARES)", "",
               "| kernel | total ms | share |", "|---|---|---|"]
        for k, v in sorted(tot.items(), key=lambda kv: -kv[1]):
            md.append(f"| {k} | {v / 1e6:.3f} | {100 * v / allns:.2f}% |")
        md.append("")
    for rep in sorted(OUT.glob(f"{tag}_*.ncu-rep")):
        txt, hdr, units, vals = raw(rep)
        (PROF / f"{rep.stem}_raw.csv").write_text(txt)
        for v in vals:
            d = dict(zip(hdr, v))
            u = dict(zip(hdr, units))
            md += [f"## {rep.stem}: `{d.get('Kernel Name', '?')[:90]}`", "",
                   "| metric | value |", "|---|---|"]
            for key, label in KEYS:
                if key in d:
                    md.append(f"| {label} (`{key}`) | {d[key]} {u.get(key, '')} |")
            md.append("")
    (PROF / f"{tag}_ncu_summary.md").write_text("\n".join(md) + "\n")
    print("\n".join(md))


if __name__ == "__main__":
    main(sys.argv[1] if len(sys.argv) > 1 else "r01")
