#!/bin/bash
mkdir -p gpurun_out
timeout 600 python scripts/variant_bench.py > gpurun_out/variants.log 2>&1
timeout 300 python bench.py --steps 20 --warmup 5 > gpurun_out/bench.json 2> gpurun_out/bench.err
cat gpurun_out/variants.log; cat gpurun_out/bench.json | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['config']['hash_only_ms'], d['config']['quantize_ms'], d['config']['dequantize_ms'])"
