#!/bin/bash
# Round-2 re-entry check: full GPU suite, default bench line, then the round-2 profile captures.
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/r2e_pytest.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/r2e_pytest.log
timeout 900 python bench.py > gpurun_out/r2e_bench.json 2> gpurun_out/r2e_bench.err; echo "bench rc=$?"; tail -c 600 gpurun_out/r2e_bench.json
bash scripts/gpu_prof_r2.sh
