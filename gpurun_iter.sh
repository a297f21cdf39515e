#!/bin/bash
# GPU call for one build->measure iteration: parity suite, bench line, launch list
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -x --timeout=300 > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 400 python bench.py --steps 20 --warmup 5 > gpurun_out/bench.json 2> gpurun_out/bench.err
timeout 400 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv python bench.py --steps 2 --warmup 3 > /dev/null 2>&1
for k in ${NCU_KERNELS:-}; do
  timeout 400 ncu --set full --clock-control none --import-source on -k regex:$k -s 2 -c 1 -o gpurun_out/c1_$k python bench.py --steps 2 --warmup 3 > gpurun_out/ncu_c1_$k.log 2>&1
done
tail -15 gpurun_out/pytest_gpu.log
python - <<'PY'
import json
d=json.load(open("gpurun_out/bench.json")); c=d["config"]
print("value", d["value"], "ms", d["ms_per_step"], "q_ms", c["quantize_ms"], "dq_ms", c["dequantize_ms"], "e2e", d["e2e"]["value"], "clk", d["clocks"])
PY
python - <<'PY'
import csv, collections
rows=list(csv.reader(open("gpurun_out/launches.csv")))
for i,r in enumerate(rows):
    if r and r[0]=="ID": hdr=r; start=i; break
data=[dict(zip(hdr,r)) for r in rows[start+1:] if len(r)==len(hdr)]
agg=collections.defaultdict(lambda:[0,0.0])
for d in data:
    k=d["Kernel Name"].split("(")[0][-40:]; agg[k][0]+=1; agg[k][1]+=float(d["Metric Value"])
for k,(c,t) in sorted(agg.items(), key=lambda x:-x[1][1]): print(f"{k:40s} {c:3d} {t/c/1e3:9.1f} us avg")
PY
