#!/bin/bash
# Round-2 end-of-round validation on one B200: GPU suite + smoke, the default bench line, one
# line per other config (each with its clocks record), ncu captures of the GQA presses, and
# compute-sanitizer memcheck over the select / long-segment paths.
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -q 2>&1 | tail -1
python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" 2>&1 | tail -1
timeout 900 python bench.py > gpurun_out/r02f_default.json 2> gpurun_out/r02f_default.err
python -c "import json; d=json.load(open('gpurun_out/r02f_default.json')); print('default', d['value'], d['roofline']['frac'], d['e2e']['value'], {k: (v['roofline']['frac'], v['parity']['mismatches']) for k, v in d['legs'].items()})"
for c in c3g c4g c3l c2m c2d c2p c4 c5; do
  timeout 900 python bench.py --config $c --legs "" --steps 5 --warmup 3 > gpurun_out/r02f_$c.json 2> gpurun_out/r02f_$c.err
  python -c "import json; d=json.load(open('gpurun_out/r02f_$c.json')); r=d.get('roofline',{}); print('$c', d['value'], round(d['ms_per_step'],3), r.get('frac'), d.get('clocks',{}).get('sm_mhz'), d.get('clocks',{}).get('reasons'), d.get('parity',{}).get('mismatches'), d.get('ttft_p50_s'))"
done
for c in c3g c4g; do
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:"snapkv_tc|ea_tc" -s 3 -c 1 \
    -o /tmp/prof_r02_$c -f python bench.py --config $c --legs "" --steps 1 --warmup 3 --e2e-steps 0 \
    --no-cpu-baseline --parity-segments 0 > gpurun_out/ncu_r02_$c.log 2>&1
  ncu -i /tmp/prof_r02_$c.ncu-rep --page raw --csv > gpurun_out/prof_r02_$c.raw.csv 2>/dev/null
done
PYTORCH_NO_CUDA_MEMORY_CACHING=1 timeout 1500 compute-sanitizer --tool memcheck --error-exitcode 9 \
  python -m pytest -q -x -m gpu tests/test_gpu_long.py tests/test_gpu_press.py tests/test_gpu_edges.py \
  > gpurun_out/r02f_memcheck.log 2>&1; echo "memcheck rc=$?"; tail -2 gpurun_out/r02f_memcheck.log
