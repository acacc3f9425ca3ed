#!/bin/bash
# ncu digests of the SnapKV GQA-unit and two-pass (long segment) paths.
mkdir -p gpurun_out
for c in c3g c3l; do
  timeout 900 ncu --set full --clock-control none -k regex:"snapkv_tc" -s 1 -c 1 \
    -o gpurun_out/prof_$c -f python bench.py --config $c --steps 1 --warmup 3 --e2e-steps 0 --no-cpu-baseline > gpurun_out/ncu_$c.log 2>&1
  tail -1 gpurun_out/ncu_$c.log
done
