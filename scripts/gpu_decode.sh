#!/bin/bash
mkdir -p gpurun_out
timeout 600 python bench.py --config c2d --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/bench_c2d.json 2> gpurun_out/bench_c2d.err; echo "bench rc=$?"
tail -3 gpurun_out/bench_c2d.err; cat gpurun_out/bench_c2d.json
timeout 600 ncu --set full --clock-control none --import-source on -k regex:decode_attn -s 200 -c 1 \
  -o gpurun_out/prof_c2d -f python bench.py --config c2d --steps 1 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_c2d.log 2>&1
tail -2 gpurun_out/ncu_c2d.log
