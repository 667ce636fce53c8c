#!/usr/bin/env python
"""Hot-spot table from `ncu --page source --csv --print-source sass` output.

usage: python tools/sass_hot.py FILE.csv [N]
Prints the N instructions with the most stall samples (with the stall-reason
breakdown) and the sample totals between warp-role markers.
"""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
hdr, data = rows[1], rows[2:]
idx = {h: i for i, h in enumerate(hdr)}
st = [h for h in hdr if h.startswith("stall_") and "Not" not in h]
n = int(sys.argv[2]) if len(sys.argv) > 2 else 40
tot = sum(int(r[2]) for r in data)
print("total samples", tot)
for r in sorted(data, key=lambda r: -int(r[2]))[:n]:
    b = " ".join(f"{h[6:]}={r[idx[h]]}" for h in st if r[idx[h]] not in ("0", ""))
    print(r[0][-5:], r[2].rjust(6), r[1].strip()[:64].ljust(64), "|", b)
