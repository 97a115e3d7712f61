#!/usr/bin/env python
"""Per-kernel counts of the Blackwell-only SASS mnemonics in the shipped library (cuobjdump -sass on the in-tree .so):
UTCHMMA / UTCQMMA = tcgen05.mma kind::f16 / kind::f8f6f4, LDTM = tcgen05.ld, UTCBAR = tcgen05.commit, UTMALDG = TMA tensor
load, UBLKCP = cp.async.bulk, SYNCS = mbarrier ops, HMMA = mma.sync, REDUX / ATOMS / RED. Writes profiles/sass_summary.txt.
Usage: python scripts/sass_summary.py"""
import collections
import os
import re
import subprocess

root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
so = os.path.join(root, "paper_2603_28458_b200", "_lib", "libhisa_b200.so")
MNEMONICS = ["UTCHMMA", "UTCQMMA", "UTCBAR", "LDTM", "UTMALDG", "UBLKCP", "UTMAPF", "SYNCS", "HMMA", "LDSM", "REDUX", "ATOMS",
             "RED", "FFMA2", "FMNMX", "DADD", "LDGSTS", "BAR"]
sass = subprocess.run(["cuobjdump", "-sass", so], capture_output=True, text=True, check=True).stdout
arch = sorted(set(re.findall(r"arch = (sm_\w+)", sass)))
counts, order, cur = {}, [], None
for line in sass.splitlines():
    m = re.match(r"\s*Function : (\S+)", line)
    if m:
        cur = m.group(1)
        counts[cur] = collections.Counter()
        order.append(cur)
        continue
    m = re.match(r"\s*/\*[0-9a-f]{4,}\*/\s+(?:@!?U?P\d+\s+)?([A-Z0-9_]+)", line)
    if m and cur:
        op = m.group(1)
        counts[cur]["_total"] += 1
        if op in MNEMONICS:
            counts[cur][op] += 1
demangled = subprocess.run(["c++filt"], input="\n".join(order), capture_output=True, text=True).stdout.splitlines()
cols = [m for m in MNEMONICS if any(counts[f][m] for f in order)]
with open(os.path.join(root, "profiles", "sass_summary.txt"), "w") as f:
    f.write(f"cuobjdump -sass paper_2603_28458_b200/_lib/libhisa_b200.so  (arch: {', '.join(arch)}); instruction counts per kernel\n")
    f.write("UTCHMMA/UTCQMMA = tcgen05.mma (bf16 / e4m3), LDTM = tcgen05.ld, UTCBAR = tcgen05.commit, UTMALDG = TMA tensor load,\n"
            "UBLKCP = cp.async.bulk, SYNCS = mbarrier, HMMA/LDSM = mma.sync/ldmatrix (consumer kernel only)\n\n")
    f.write(f"{'kernel':78s} {'instrs':>7s} " + " ".join(f"{c:>7s}" for c in cols) + "\n")
    tot = collections.Counter()
    for fn, dn in zip(order, demangled):
        name = re.sub(r"^void hisa_dev::(\(anonymous namespace\)::)?", "", dn)
        name = re.sub(r"\((hisa_dev::|CUtensorMap|unsigned|float|void|int|__nv|double|long|const|uint).*$", "", name)
        f.write(f"{name[:78]:78s} {counts[fn]['_total']:7d} " + " ".join(f"{counts[fn][c]:7d}" for c in cols) + "\n")
        tot.update(counts[fn])
    f.write(f"{'TOTAL':78s} {tot['_total']:7d} " + " ".join(f"{tot[c]:7d}" for c in cols) + "\n")
print(open(os.path.join(root, "profiles", "sass_summary.txt")).read())
