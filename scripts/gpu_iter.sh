#!/bin/bash
# One build->measure iteration on the B200: tests (optional filter), bench line, ncu capture.
#   bash scripts/gpu_iter.sh <config> [pytest -k filter] [tag]
CFG=${1:-c2}; FILTER=${2:-}; TAG=${3:-$CFG}
mkdir -p gpurun_out
if [ -n "$FILTER" ]; then
  timeout 900 python -m pytest tests -m gpu -x -q -k "$FILTER" 2>&1 | tail -5
fi
python bench.py --config $CFG --steps 10 --warmup 3 --e2e-steps 0 --no-cpu-baseline > gpurun_out/bench_$TAG.json 2> gpurun_out/bench_$TAG.err
tail -3 gpurun_out/bench_$TAG.err; cat gpurun_out/bench_$TAG.json
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"press_kernel|snapkv_tc" -s 3 -c 1 \
  -o gpurun_out/prof_$TAG -f python bench.py --config $CFG --steps 1 --warmup 3 --e2e-steps 0 --no-cpu-baseline > gpurun_out/ncu_$TAG.log 2>&1
tail -2 gpurun_out/ncu_$TAG.log
