#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_host.py -x -q > gpurun_out/pytest_host.log 2>&1; echo "host tests rc=$?"
tail -30 gpurun_out/pytest_host.log
for c in c2 c3; do
timeout 900 python bench.py --config $c --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/bench_e2e_$c.json 2> gpurun_out/bench_e2e_$c.err; echo "bench $c rc=$?"
tail -3 gpurun_out/bench_e2e_$c.err
python -c "import json; d=json.load(open('gpurun_out/bench_e2e_$c.json')); print('$c', d['value'], d['roofline']['frac'], d['e2e'])"
done
