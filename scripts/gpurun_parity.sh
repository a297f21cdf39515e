mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_loopback.py tests/test_gpu_ddp.py -q --timeout=600 --durations=10 > gpurun_out/pytest_loop.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_loop.log
timeout 900 python -m pytest tests -m gpu -q --timeout=600 --durations=10 --deselect tests/test_gpu_loopback.py > gpurun_out/pytest_gpu.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_gpu.log
timeout 400 python bench.py --steps 20 --warmup 5 > gpurun_out/bench.json 2> gpurun_out/bench.err
tail -30 gpurun_out/pytest_loop.log; tail -30 gpurun_out/pytest_gpu.log; cat gpurun_out/bench.json | head -c 600; tail -5 gpurun_out/bench.err
