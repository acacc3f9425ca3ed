#!/bin/bash
# Round 2 profiling: per-role SnapKV timelines (trace build) for c3 and c3g, and an ncu
# source-level capture of the c3g SnapKV kernel (warp-stall samples per line).
mkdir -p gpurun_out
L=$PWD/paper_2503_08461_b200/_lib
for c in c3 c3g; do
  echo "== trace $c"; FASTCACHE_LIB=$L/libfastcache_trace.so timeout 300 python scripts/trace_press.py $c sub 2>&1 | tail -8
done
timeout 900 ncu --set full --import-source on --clock-control none -k regex:"snapkv_tc" -s 1 -c 1 \
  -o gpurun_out/prof_c3g_r2 -f python bench.py --config c3g --steps 1 --warmup 3 --e2e-steps 0 --no-cpu-baseline --parity-segments 0 > gpurun_out/ncu_c3g_r2.log 2>&1
tail -2 gpurun_out/ncu_c3g_r2.log
python scripts/ncu_lines.py gpurun_out/prof_c3g_r2.ncu-rep 40 > gpurun_out/ncu_c3g_lines.txt 2>&1
head -45 gpurun_out/ncu_c3g_lines.txt
