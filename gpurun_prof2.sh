#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -x --timeout=240 --timeout-method=thread > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/sra_launches.csv python scripts/sra_emul_profile.py 8 > gpurun_out/sra_prof.log 2>&1
for k in k_fold k_norms k_quant k_decode; do
  timeout 400 ncu --set full --clock-control none --import-source on -k regex:$k -s 4 -c 1 -o gpurun_out/sra_$k python scripts/sra_emul_profile.py 8 > gpurun_out/ncu_sra_$k.log 2>&1
done
timeout 200 python bench.py --steps 20 --warmup 5 > gpurun_out/bench.json 2> gpurun_out/bench.err
tail -3 gpurun_out/pytest_gpu.log
python -c "import json; d=json.load(open('gpurun_out/bench.json')); print(d['value'], d['config']['quantize_ms'], d['config']['dequantize_ms'])"
python - <<'PY'
import csv, collections
rows=list(csv.reader(open("gpurun_out/sra_launches.csv")))
for i,r in enumerate(rows):
    if r and r[0]=="ID": hdr=r; start=i; break
data=[dict(zip(hdr,r)) for r in rows[start+1:] if len(r)==len(hdr)]
half=data[len(data)//2:]
agg=collections.defaultdict(lambda:[0,0.0])
for d in half:
    k=d["Kernel Name"].split("(")[0][-40:]; agg[k][0]+=1; agg[k][1]+=float(d["Metric Value"])
for k,(c,t) in sorted(agg.items(), key=lambda x:-x[1][1]): print(f"{k:40s} {c:3d} {t/1e3:9.1f} us")
PY
