#!/bin/bash
# GPU call: full -m gpu suite + smoke
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -q -x --durations=15 > gpurun_out/pytest_gpu.log 2>&1
echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1
tail -40 gpurun_out/pytest_gpu.log; tail -3 gpurun_out/smoke.log
