#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -x --timeout=240 --timeout-method=thread > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 120 ./scripts/piperate > gpurun_out/piperate.log 2>&1
timeout 300 python scripts/variant_bench.py > gpurun_out/variants.log 2>&1
timeout 300 python scripts/sra_emul_bench.py > gpurun_out/sra_emul.log 2>&1
timeout 200 python bench.py --steps 20 --warmup 5 > gpurun_out/bench.json 2> gpurun_out/bench.err
tail -4 gpurun_out/pytest_gpu.log; cat gpurun_out/variants.log gpurun_out/sra_emul.log; python -c "import json; d=json.load(open('gpurun_out/bench.json')); print(d['config']['hash_only_ms'], d['config']['quantize_ms'], d['config']['dequantize_ms'])"
