#!/bin/bash
# ncu captures of the decode attention and prefill ingest kernels (c2d / c2p).
mkdir -p gpurun_out
timeout 600 ncu --set full --clock-control none --import-source on -k regex:decode_attn -s 200 -c 1 \
  -o gpurun_out/prof_c2d -f python bench.py --config c2d --steps 1 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_c2d.log 2>&1
tail -1 gpurun_out/ncu_c2d.log
timeout 600 ncu --set full --clock-control none --import-source on -k regex:write_prefill -s 40 -c 1 \
  -o gpurun_out/prof_c2p -f python bench.py --config c2p --steps 1 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_c2p.log 2>&1
tail -1 gpurun_out/ncu_c2p.log
