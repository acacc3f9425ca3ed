#!/bin/bash
# Round-2 refresh after the pass-3 / GQA changes: GPU suite, smoke, default line, c3g / c4g /
# c3l lines, ncu captures of the SnapKV kernel at c3 and c3g.
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -q > gpurun_out/r02u_pytest.log 2>&1; tail -1 gpurun_out/r02u_pytest.log
python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" 2>&1 | tail -1
timeout 900 python bench.py > gpurun_out/r02u_default.json 2> gpurun_out/r02u_default.err
python -c "import json; d=json.load(open('gpurun_out/r02u_default.json')); print('default', d['value'], d['roofline']['frac'], d['e2e']['value'], {k: (v['roofline']['frac'], v['parity']['mismatches']) for k, v in d['legs'].items()})"
for c in c3g c4g c3l; do
  timeout 900 python bench.py --config $c --legs "" --steps 5 --warmup 3 > gpurun_out/r02u_$c.json 2> gpurun_out/r02u_$c.err
  python -c "import json; d=json.load(open('gpurun_out/r02u_$c.json')); r=d.get('roofline',{}); print('$c', d['value'], round(d['ms_per_step'],3), r.get('frac'), d.get('clocks',{}).get('sm_mhz'), d.get('clocks',{}).get('reasons'), d.get('parity',{}).get('mismatches'))"
done
for c in c3 c3g; do
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:"snapkv_tc" -s 3 -c 1 \
    -o /tmp/prof_r02u_$c -f python bench.py --config $c --legs "" --steps 1 --warmup 3 --e2e-steps 0 \
    --no-cpu-baseline --parity-segments 0 > gpurun_out/ncu_r02u_$c.log 2>&1
  ncu -i /tmp/prof_r02u_$c.ncu-rep --page raw --csv > gpurun_out/prof_r02u_$c.raw.csv 2>/dev/null
done
