#!/bin/bash
# TMA prefill ingest: full GPU suite, smoke, the c2p bench line, an ncu capture of
# write_prefill_tma_kernel and the c2p launch list.
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -q 2>&1 | tail -3
python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" 2>&1 | tail -1
timeout 600 python bench.py --config c2p --legs "" --steps 5 --warmup 3 > gpurun_out/r02_bench_c2p.json 2> gpurun_out/r02_bench_c2p.err
python -c "import json; d=json.load(open('gpurun_out/r02_bench_c2p.json')); print('c2p', round(d['ms_per_step'],3), d['roofline']['frac'], d['clocks'], d.get('e2e',{}).get('value'))"
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"write_prefill" -s 40 -c 1 \
  -o gpurun_out/prof_r02_c2p -f python bench.py --config c2p --legs "" --steps 1 --warmup 3 --e2e-steps 0 --no-cpu-baseline > gpurun_out/ncu_r02_c2p.log 2>&1
ncu -i gpurun_out/prof_r02_c2p.ncu-rep --page raw --csv > gpurun_out/prof_r02_c2p.raw.csv 2>/dev/null
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_r02_c2p.csv \
  python bench.py --config c2p --legs "" --steps 1 --warmup 3 --e2e-steps 0 --no-cpu-baseline > /dev/null 2>&1
ls gpurun_out | tail -5
