#!/usr/bin/env python
"""Per-warp-role totals from `ncu --page source --csv --print-source sass`:
stall samples, warp instructions executed and shared wavefronts between the
USETMAXREG markers (MMA / producer / epilogue regions), plus the hottest
instructions of one region.   usage: sass_regions.py FILE.csv [region] [N]"""
import csv, sys
rows = list(csv.reader(open(sys.argv[1])))
hdr, data = rows[1], rows[2:]
ix = {h: i for i, h in enumerate(hdr)}
def num(r, h):
    v = r[ix[h]].replace(",", "")
    try: return float(v)
    except ValueError: return 0.0
marks = [0]
for k, r in enumerate(data):
    if "USETMAXREG" in r[ix["Source"]]: marks.append(k)
marks.append(len(data))
names = ["setup", "mma", "producer", "epilogue"] + [f"r{i}" for i in range(10)]
stalls = [h for h in hdr if h.startswith("stall_") or "Stall" in h]
regions = []
for n, (a, b) in enumerate(zip(marks[:-1], marks[1:])):
    seg = data[a:b]
    s = sum(num(r, "Warp Stall Sampling (All Samples)") for r in seg)
    ni = sum(num(r, "Warp Stall Sampling (Not-issued Samples)") for r in seg)
    ie = sum(num(r, "Instructions Executed") for r in seg)
    wf = sum(num(r, "L1 Wavefronts Shared") for r in seg)
    wi = sum(num(r, "L1 Wavefronts Shared Ideal") for r in seg)
    print(f"{names[n]:9s} [{a:5d},{b:5d}) samples {s:9.0f} not-issued {ni:9.0f} inst {ie:12.0f} smem wf {wf:11.0f} ideal {wi:11.0f}")
    regions.append(seg)
if len(sys.argv) > 2:
    seg = regions[names.index(sys.argv[2])]
    N = int(sys.argv[3]) if len(sys.argv) > 3 else 40
    # opcode histogram weighted by executions
    from collections import Counter
    h = Counter(); hs = Counter()
    for r in seg:
        op = r[ix["Source"]].strip().split()
        if not op: continue
        o = op[0] if not op[0].startswith("@") else op[1]
        o = o.split(".")[0]
        h[o] += num(r, "Instructions Executed")
        hs[o] += num(r, "Warp Stall Sampling (All Samples)")
    tot = sum(h.values())
    print("opcode mix (warp inst executed):")
    for o, c in h.most_common(30):
        print(f"  {o:10s} {c:12.0f} {100*c/tot:5.1f}%  samples {hs[o]:8.0f}")
    print("hottest:")
    for r in sorted(seg, key=lambda r: -num(r, "Warp Stall Sampling (All Samples)"))[:N]:
        print(r[ix["Address"]][-5:], f'{num(r,"Warp Stall Sampling (All Samples)"):7.0f}', f'{num(r,"Instructions Executed"):10.0f}', r[ix["Source"]].strip()[:70])
# stall-reason totals per region (all samples), EXIT excluded
st = [h for h in hdr if h.startswith("stall_") and "Not Issued" not in h]
print("stall reasons per region (samples, EXIT excluded):")
for n, seg in enumerate(regions):
    tot = {h: sum(num(r, h) for r in seg if "EXIT" not in r[ix["Source"]]) for h in st}
    s = sum(tot.values()) or 1
    print(f"  {names[n]:9s}", " ".join(f"{h[6:]}={100*v/s:.0f}%" for h, v in sorted(tot.items(), key=lambda x: -x[1]) if v > 0.01 * s))
