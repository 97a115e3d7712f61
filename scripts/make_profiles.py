#!/usr/bin/env python
"""Builds the committed profile summaries under profiles/ from the scratch captures in gpurun_out/.
Usage: python scripts/make_profiles.py r01"""
import csv
import json
import os
import subprocess
import sys

tag = sys.argv[1] if len(sys.argv) > 1 else "r01"
root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
out = os.path.join(root, "profiles")
os.makedirs(out, exist_ok=True)

# 1. launch list: per-kernel share of one bench step (cold-cache, serialised: shares, not absolutes)
rows = [r for r in csv.reader(open(os.path.join(root, "gpurun_out", "launches.csv"))) if len(r) > 5]
hdr = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
ix = {h: i for i, h in enumerate(rows[hdr])}
agg, order = {}, []
for r in rows[hdr + 1:]:
    if len(r) != len(rows[hdr]) or r[ix["Metric Name"]] != "gpu__time_duration.sum":
        continue
    name = r[ix["Kernel Name"]]
    val = float(r[ix["Metric Value"]].replace(",", ""))
    unit = r[ix["Metric Unit"]]
    ms = val / 1e6 if unit in ("ns", "nsecond") else val / 1e3 if unit in ("us", "usecond") else val
    if name not in agg:
        agg[name] = [0, 0.0]
        order.append(name)
    agg[name][0] += 1
    agg[name][1] += ms
total = sum(v[1] for v in agg.values())
with open(os.path.join(out, f"{tag}_launches_summary.txt"), "w") as f:
    f.write("ncu --metrics gpu__time_duration.sum --clock-control none : python bench.py --steps 2 --warmup 1 --flat-steps 1\n")
    f.write("(6 hisa_select calls: 1 warm-up + 2 timed + 2 of the instrumented stall-statistics pass, whose scorer is the <..., 1> instantiation, + 1 feeding the consumer; 2 dsa_select calls; 3 sparse_attend calls of the consumer leg; C3, L=Q=65536; times are cold-cache and serialised)\n\n")
    f.write(f"{'kernel':70s} {'launches':>8s} {'total ms':>10s} {'share':>7s}\n")
    for name in sorted(agg, key=lambda n: -agg[n][1]):
        f.write(f"{name[:70]:70s} {agg[name][0]:8d} {agg[name][1]:10.3f} {100 * agg[name][1] / total:6.1f}%\n")
subprocess.run(["cp", os.path.join(root, "gpurun_out", "launches.csv"), os.path.join(out, f"{tag}_launches.csv")], check=True)

# 2. full captures -> short counter tables
for rep, name in (("prof_score_tc.ncu-rep", "score_tc"), ("prof_score_tc_fp8.ncu-rep", "score_tc_fp8"),
                  ("prof_select.ncu-rep", "select"), ("prof_pool.ncu-rep", "pool")):
    path = os.path.join(root, "gpurun_out", rep)
    if not os.path.exists(path):
        continue
    txt = subprocess.run([sys.executable, os.path.join(root, "scripts", "ncu_summary.py"), path],
                         capture_output=True, text=True).stdout
    with open(os.path.join(out, f"{tag}_{name}_ncu_full_summary.txt"), "w") as f:
        f.write(f"ncu --set full --clock-control none --import-source on ({rep}; scripts/profile.sh: python bench.py "
                f"{'--dtype fp8 ' if 'fp8' in rep else ''}--steps 1 --warmup 1; launch 0 = first stage, launch 1 = second stage)\n\n")
        f.write(txt)

# 3. DRAM traffic of the stage-2 scorer launch (the second captured launch) -> bench.py's roofline.traffic
for rep, key, summ in (("prof_score_tc.ncu-rep", "traffic_score_tc_stage2.json", "score_tc"),
                       ("prof_score_tc_fp8.ncu-rep", "traffic_score_tc_stage2_fp8.json", "score_tc_fp8")):
    path = os.path.join(root, "gpurun_out", rep)
    if not os.path.exists(path):
        continue
    raw = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rr = list(csv.reader(raw.splitlines()))
    h, units = rr[0], rr[1]
    d = dict(zip(h, rr[3]))

    def gb(k):
        v = float(d[k].replace(",", ""))
        u = units[h.index(k)]
        return v * {"Gbyte": 1e9, "Mbyte": 1e6, "Kbyte": 1e3, "byte": 1}[u]
    rd, wr = gb("dram__bytes_read.sum"), gb("dram__bytes_write.sum")
    json.dump({"kernel": d["Kernel Name"], "dram_bytes_read": rd, "dram_bytes_write": wr,
               "dram_bytes_per_launch": rd + wr, "source": f"profiles/{tag}_{summ}_ncu_full_summary.txt"},
              open(os.path.join(out, key), "w"), indent=1)
    print(rep, "stage-2 DRAM traffic per launch: %.3f GB" % ((rd + wr) / 1e9))
# 4. racecheck over the selection kernels alone (no TMA / tcgen05 kernel in the process)
rc = os.path.join(root, "gpurun_out", "racecheck_select_only.log")
if os.path.exists(rc):
    with open(os.path.join(out, f"{tag}_racecheck_select_only.txt"), "w") as f:
        f.write("compute-sanitizer --tool racecheck --racecheck-report analysis python -m pytest tests/test_gpu_parity.py -m gpu "
                "-k 'top_k_on_given_scores or select_blocks_on_given'  (scripts/profile.sh; only select_* kernels launch)\n\n")
        f.write(open(rc).read())
print(open(os.path.join(out, f"{tag}_launches_summary.txt")).read())
