"""Per-source-line stall samples and instruction counts from
`ncu -i REP --page source --csv --print-source cuda,sass` output.
usage: python tools/ncu_lines.py FILE.csv [N]"""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
n = int(sys.argv[2]) if len(sys.argv) > 2 else 40
cur_file = "?"
lines = {}
hdr = None
for r in rows:
    if not r:
        continue
    if r[0] in ("File Path", "File Name"):
        cur_file = r[1].split("/")[-1]
        continue
    if r[0] == "Line No":
        hdr = {h: i for i, h in enumerate(r)}
        continue
    if hdr is None or r[0] in ("Function Name",):
        continue
    if r[0]:  # a source line row: aggregated metrics
        key = (cur_file, int(r[0]))
        def num(h):
            try:
                return float(r[hdr[h]])
            except (ValueError, IndexError):
                return 0.0
        S = num("Warp Stall Sampling (All Samples)")
        I = num("Instructions Executed")
        lines[key] = [S, I, r[1]]
tot = sum(v[0] for v in lines.values()) or 1
toti = sum(v[1] for v in lines.values()) or 1
print(f"total samples {tot:.0f}, warp instructions {toti:.3g}")
for k, v in sorted(lines.items(), key=lambda kv: -kv[1][0])[:n]:
    print(f"{k[0][:14]:14} {k[1]:5d} {v[0] / tot * 100:5.1f}% samp {v[1] / toti * 100:5.1f}% inst | {v[2].strip()[:90]}")
