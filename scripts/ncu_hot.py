#!/usr/bin/env python
"""Top stall-sample instructions per kernel from `ncu -i rep --page source --csv` output.
Usage: ncu_hot.py <source.csv> [N] [kernel-substring]"""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
N = int(sys.argv[2]) if len(sys.argv) > 2 else 40
want = sys.argv[3] if len(sys.argv) > 3 else ""
# split into per-kernel sections
sections, cur = [], None
for r in rows:
    if r and r[0] == "Kernel Name":
        cur = {"name": r[1], "rows": []}
        sections.append(cur)
    elif cur is not None:
        cur["rows"].append(r)
for sec in sections:
    if want not in sec["name"]:
        continue
    hdr = sec["rows"][0]
    ix = {h: i for i, h in enumerate(hdr)}
    data = [r for r in sec["rows"][1:] if len(r) == len(hdr)]
    tot = sum(int(r[ix["# Samples"]]) for r in data) or 1
    print("==", sec["name"][:100], "| samples", tot, "| instructions", len(data))
    top = sorted(range(len(data)), key=lambda i: -int(data[i][ix["# Samples"]]))[:N]
    stalls = [h for h in hdr if h.startswith("stall_") and "Not Issued" not in h]
    for i in sorted(top):
        r = data[i]
        s = int(r[ix["# Samples"]])
        st = {h[6:]: int(r[ix[h]]) for h in stalls if int(r[ix[h]]) > 0}
        st = sorted(st.items(), key=lambda kv: -kv[1])[:3]
        print(f"{i:5d} {100 * s / tot:5.1f}% exec={r[ix['Instructions Executed']]:>10s} {r[ix['Source']].strip()[:64]:64s} {st}")
