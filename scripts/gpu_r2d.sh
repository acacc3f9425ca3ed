#!/bin/bash
# Round 2: full GPU suite after the tensor-core spill variants, then c3, c3l, c4w, c3g, c4g timing.
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"
tail -4 gpurun_out/pytest_gpu.log
for c in c3 c3l c4w c3g c4g; do
  timeout 600 python bench.py --config $c --steps 5 --warmup 3 --e2e-steps 0 --no-cpu-baseline --parity-segments 16 > gpurun_out/b_$c.json 2> gpurun_out/b_$c.err
  python -c "import json; d=json.load(open('gpurun_out/b_$c.json')); print('$c', round(d['ms_per_step'],3), round(d['roofline']['frac'],3), d['parity']['mismatches'], d['paths'], d['clocks']['sm_mhz'])" || tail -3 gpurun_out/b_$c.err
done
