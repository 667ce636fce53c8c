#!/usr/bin/env python
"""Opcode mix of the narrow epilogue's round loop (the innermost backward
branch attributed to the round-loop source lines) of one search_syrk_kernel
instantiation.  usage: sass_loop.py LIB.so [Lb0ELi3ELb1E]"""
import collections, os, re, subprocess, sys, tempfile
lib = os.path.abspath(sys.argv[1]); inst = sys.argv[2] if len(sys.argv) > 2 else "Lb0ELi3ELb1E"
d = tempfile.mkdtemp()
subprocess.run(["cuobjdump", "-xelf", "all", lib], cwd=d, capture_output=True)
txt = subprocess.run(["nvdisasm", "-g", "engine.sm_100a.cubin"], cwd=d, capture_output=True, text=True).stdout
sec = None
for part in txt.split("//--------------------- .text."):
    if part.startswith("_ZN4syrk18search_syrk_kernelI" + inst):
        sec = part
        break
lines = sec.split("\n")
fl, ins, labels = None, [], {}
for l in lines:
    m = re.search(r'//## File "([^"]+)", line (\d+)', l)
    if m:
        fl = (m.group(1).split("/")[-1], int(m.group(2)))
        continue
    m = re.match(r"^(\.L_x_\d+):", l)
    if m:
        labels[m.group(1)] = len(ins)
        continue
    m = re.match(r"\s*/\*([0-9a-f]{4,})\*/\s+(.*?);", l)
    if m:
        ins.append((fl, m.group(2)))
# the round loop: the smallest backward branch around both screens (>= 54 MUFU)
best = None
for k, (fl, t) in enumerate(ins):
    m = re.search(r"BRA `\((\.L_x_\d+)\)", t)
    if m and m.group(1) in labels and labels[m.group(1)] < k and fl and fl[0] == "search_syrk.cuh":
        a = labels[m.group(1)]
        nm = sum(1 for _, t2 in ins[a:k] if "MUFU" in t2)
        if nm >= 54 and (best is None or k - a < best[1] - best[0]):
            best = (a, k)
a, b = best
c = collections.Counter()
for fl, t in ins[a:b + 1]:
    op = t.split()[1] if t.startswith("@") else t.split()[0]
    c[op.split(".")[0]] += 1
print(inst, "loop", b - a + 1, "instructions")
print(" ".join(f"{k}:{v}" for k, v in c.most_common()))
