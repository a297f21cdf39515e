#!/bin/bash
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
./scripts/piperate > gpurun_out/piperate.log 2>&1
timeout 600 python scripts/sra_emul_bench.py > gpurun_out/sra_emul.log 2>&1
timeout 300 python bench.py --steps 20 --warmup 5 > gpurun_out/bench.json 2> gpurun_out/bench.err
tail -4 gpurun_out/pytest_gpu.log; cat gpurun_out/piperate.log gpurun_out/sra_emul.log; python -c "import json; d=json.load(open('gpurun_out/bench.json')); print(d['config']['quantize_ms'], d['config']['dequantize_ms'])"
