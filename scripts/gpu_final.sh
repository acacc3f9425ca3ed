#!/bin/bash
# End-of-session validation: every GPU test, smoke(), ncu of the SnapKV kernel, and bench lines.
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -q 2>&1 | tail -1
python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"snapkv_tc" -s 1 -c 1 \
  -o gpurun_out/prof_c3 -f python bench.py --config c3 --steps 1 --warmup 3 --e2e-steps 0 --no-cpu-baseline > gpurun_out/ncu_c3.log 2>&1
tail -1 gpurun_out/ncu_c3.log
for c in c2 c3 c4 c5 c2d c2p; do
  timeout 900 python bench.py --config $c --steps 5 --warmup 3 > gpurun_out/final_$c.json 2> gpurun_out/final_$c.err
  python -c "import json; d=json.load(open('gpurun_out/final_$c.json')); r=d.get('roofline',{}); print('$c', d['value'], d['ms_per_step'], r.get('frac'), d.get('e2e',{}).get('value'), d.get('cpu_baseline',{}).get('value'), d.get('ttft_p50_s'))"
done
