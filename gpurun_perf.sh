#!/bin/bash
# GPU call: tests + bench + launch list + ncu captures of K1/K3
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu.log 2>&1
echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 300 python bench.py --steps 20 --warmup 5 > gpurun_out/bench.json 2> gpurun_out/bench.err
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv python bench.py --steps 2 --warmup 3 > /dev/null 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_quantize_pipe -s 3 -c 1 -o gpurun_out/k1 python bench.py --steps 2 --warmup 3 > gpurun_out/ncu_k1.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_decode -s 3 -c 1 -o gpurun_out/k3 python bench.py --steps 2 --warmup 3 > gpurun_out/ncu_k3.log 2>&1
tail -5 gpurun_out/pytest_gpu.log; cat gpurun_out/bench.json; tail -3 gpurun_out/bench.err
