#!/usr/bin/env python
"""Stall samples aggregated per CUDA source line from
`ncu -i rep --page source --csv --print-source cuda,sass`. Usage: ncu_lines.py <csv> <kernel-substring> [N]"""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
want = sys.argv[2]
N = int(sys.argv[3]) if len(sys.argv) > 3 else 40
i = 0
agg = {}
total = 0
fname, func = None, None
hdr = None
while i < len(rows):
    r = rows[i]
    if r and r[0] == "File Path":
        fname = r[1].split("/")[-1]
        func = rows[i + 1][1]
        hdr = rows[i + 2]
        ix = {h: j for j, h in enumerate(hdr)}
        i += 3
        continue
    if hdr and want in (func or "") and len(r) == len(hdr) and r[0] not in ("", "Line No"):
        s = int(r[6])
        key = (fname, int(r[0]), r[1].strip()[:90])
        st = agg.setdefault(key, {"s": 0, "exec": 0, "stalls": {}})
        st["s"] += s
        st["exec"] += int(r[7])
        for h, j in ix.items():
            if h.startswith("stall_") and "Not Issued" not in h and int(r[j]) > 0:
                st["stalls"][h[6:]] = st["stalls"].get(h[6:], 0) + int(r[j])
        total += s
    i += 1
print("total samples", total)
for key, st in sorted(agg.items(), key=lambda kv: -kv[1]["s"])[:N]:
    top = sorted(st["stalls"].items(), key=lambda kv: -kv[1])[:3]
    print(f"{100 * st['s'] / max(total, 1):5.1f}% {key[0]}:{key[1]:<4d} exec={st['exec']:>11d} {key[2][:70]:70s} {top}")
