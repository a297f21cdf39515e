#!/bin/bash
# GPU call: SRA emulation timings (all ranks on one GPU) + launch list of one N=8 step
mkdir -p gpurun_out
timeout 600 python scripts/sra_emul_bench.py > gpurun_out/sra_emul.log 2>&1
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/sra_launches.csv python scripts/sra_emul_profile.py 8 > gpurun_out/sra_prof.log 2>&1
for k in ${NCU_KERNELS:-}; do
  timeout 400 ncu --set full --clock-control none --import-source on -k regex:$k -s ${NCU_SKIP:-8} -c 1 -o gpurun_out/sra_$k python scripts/sra_emul_profile.py 8 > gpurun_out/ncu_sra_$k.log 2>&1
done
cat gpurun_out/sra_emul.log
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
for k,(c,t) in sorted(agg.items(), key=lambda x:-x[1][1]): print(f"{k:40s} {c:3d} {t/1e3:9.1f} us total")
PY
