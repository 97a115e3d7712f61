timeout 900 python -m pytest tests -m gpu -q -x --timeout 300 -p no:cacheprovider 2>&1 | tail -2
ncu --metrics gpu__time_duration.sum --clock-control none -k regex:select_tok --csv --log-file gpurun_out/tok.csv python bench.py --steps 2 --warmup 1 --flat-steps 0 --e2e-steps 0 --no-cpu-baseline --no-configs --attend-steps 0 > /dev/null 2>&1
python - <<PY
import csv
rows=[r for r in csv.reader(open("gpurun_out/tok.csv")) if len(r)>5]
h=next(i for i,r in enumerate(rows) if "Kernel Name" in r); ix={k:i for i,k in enumerate(rows[h])}
v=[float(r[ix["Metric Value"]].replace(",","")) for r in rows[h+1:] if len(r)==len(rows[h])]
print("select_tok us:", [round(x/1e3,1) for x in v])
PY
