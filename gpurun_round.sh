#!/bin/bash
# GPU call: parity suite, smoke, bench line (ours + reference arm), launch
# list, ncu captures of the two C1 kernels (K1 k_span, K3 k_dspan), the
# per-kernel launch list of one emulated N = 8 SRA step, and the emulated
# per-rank SRA times of BASELINE configs C2-C4
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/gpu.txt 2>&1
nproc > gpurun_out/nproc.txt; lscpu | head -20 >> gpurun_out/nproc.txt
timeout 1500 python -m pytest tests -m gpu -q -x --timeout=300 --durations=10 > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke.log
timeout 400 python bench.py --steps 20 --warmup 5 > gpurun_out/bench.json 2> gpurun_out/bench.err
timeout 400 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err
timeout 400 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv python bench.py --steps 2 --warmup 3 > /dev/null 2>&1
# full captures stay on the box (a K1 .ncu-rep is ~50 MB; gpurun merges <= 64 MiB):
# their summaries come back
mkdir -p /tmp/ncu
timeout 400 ncu --set full --clock-control none --import-source on -k regex:k_span -s 2 -c 1 -o /tmp/ncu/c1_k_span python bench.py --steps 2 --warmup 3 > /dev/null 2>&1
timeout 400 ncu --set full --clock-control none --import-source on -k regex:k_dspan -s 2 -c 1 -o /tmp/ncu/c1_k_dspan python bench.py --steps 2 --warmup 3 > /dev/null 2>&1
python scripts/ncu_summary.py /tmp/ncu/c1_k_span.ncu-rep round2_c1_k_span gpurun_out > /dev/null
python scripts/ncu_summary.py /tmp/ncu/c1_k_dspan.ncu-rep round2_c1_k_dspan gpurun_out > /dev/null
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/sra8_launches.csv python scripts/sra_emul_profile.py 8 > /dev/null 2>&1
timeout 600 python scripts/sra_emul_configs.py > gpurun_out/sra_emul_configs.log 2>&1
tail -4 gpurun_out/pytest_gpu.log; tail -2 gpurun_out/smoke.log; cat gpurun_out/bench.json; tail -3 gpurun_out/bench.err; cat gpurun_out/bench_ref.json; tail -12 gpurun_out/sra_emul_configs.log; ls gpurun_out
