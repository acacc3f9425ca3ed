#!/bin/bash
# Round 2: device serving tests + the config-5 line (engine restatement, measured compress).
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_serving.py tests/test_gpu_atomic.py -m gpu -q -x > gpurun_out/pytest_serving.log 2>&1; echo "pytest rc=$?"
tail -5 gpurun_out/pytest_serving.log
timeout 1200 python bench.py --config c5 --no-cpu-baseline > gpurun_out/bench_c5.json 2> gpurun_out/bench_c5.err; echo "bench c5 rc=$?"
tail -3 gpurun_out/bench_c5.err
