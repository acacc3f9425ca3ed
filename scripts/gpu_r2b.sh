#!/bin/bash
# Round 2: BASELINE-scale parity tests + the default bench line (c2 + c3/c4w legs).
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_scale.py -m gpu -q -rs > gpurun_out/pytest_scale.log 2>&1; echo "pytest rc=$?"
tail -5 gpurun_out/pytest_scale.log
timeout 900 python bench.py > gpurun_out/bench_default.json 2> gpurun_out/bench_default.err; echo "bench rc=$?"
tail -3 gpurun_out/bench_default.err
