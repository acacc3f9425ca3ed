#!/bin/bash
# Round-1 (session 2) profile refresh: ncu captures of c3/c4w and bench lines for c2..c4.
mkdir -p gpurun_out
for c in c3 c4w; do
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:"snapkv_tc|ea_tc" -s 1 -c 1 \
    -o gpurun_out/prof_$c -f python bench.py --config $c --steps 1 --warmup 3 --e2e-steps 0 --no-cpu-baseline > gpurun_out/ncu_$c.log 2>&1
  tail -1 gpurun_out/ncu_$c.log
done
for c in c2 c3 c4; do
  timeout 900 python bench.py --config $c --steps 5 --warmup 3 > gpurun_out/bench_$c.json 2> gpurun_out/bench_$c.err
  python -c "import json; d=json.load(open('gpurun_out/bench_$c.json')); print('$c', d['value'], d['ms_per_step'], d['roofline']['frac'], d.get('e2e',{}).get('value'))"
done
