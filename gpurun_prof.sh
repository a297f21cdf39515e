#!/bin/bash
mkdir -p gpurun_out
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/sra_launches.csv python scripts/sra_emul_profile.py 8 > gpurun_out/sra_prof.log 2>&1
python - <<'PY'
import csv, collections
rows = [r for r in csv.DictReader(open("gpurun_out/sra_launches.csv")) if r.get("Metric Name") == "gpu__time_duration.sum"]
half = rows[len(rows)//2:]  # second allreduce call
agg = collections.defaultdict(lambda: [0, 0.0])
for r in half:
    k = r["Kernel Name"].split("(")[0][-60:]
    agg[k][0] += 1; agg[k][1] += float(r["Metric Value"])
for k, (c, t) in sorted(agg.items(), key=lambda x: -x[1][1]):
    print(f"{k:60s} {c:4d} launches {t/1e3:9.1f} us")
PY
cat gpurun_out/sra_prof.log | tail -2
