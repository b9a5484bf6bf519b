#!/bin/bash
# launch list (ncu, duration only) of one nonlinear pass: nl2, 2 steps (Newton per step)
mkdir -p gpurun_out
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 2000 --csv --log-file gpurun_out/launches_nl2.csv python tools/one_pass.py nl2 2 > gpurun_out/ncu_nl2.log 2>&1; echo rc=$? >> gpurun_out/ncu_nl2.log
python - <<'PY' >> gpurun_out/ncu_nl2.log
import csv, collections
tot = collections.defaultdict(float); cnt = collections.Counter()
for row in csv.DictReader(l for l in open("gpurun_out/launches_nl2.csv") if l.startswith('"')):
    if row.get("Metric Name") == "gpu__time_duration.sum":
        k = row["Kernel Name"].split("(")[0]; tot[k] += float(row["Metric Value"]) / 1e6; cnt[k] += 1
for k, v in sorted(tot.items(), key=lambda x: -x[1]): print(f"{k:40s} {cnt[k]:6d} {v:10.3f} ms")
PY
S=$(date +%s); python tools/one_pass.py nl2 50 >> gpurun_out/ncu_nl2.log 2>&1; echo "plain nl2 50 steps wall $(( $(date +%s) - S )) s" >> gpurun_out/ncu_nl2.log
