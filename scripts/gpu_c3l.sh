#!/bin/bash
# c3l (long SnapKV) diagnosis: per-role trace, then an ncu capture of the press kernel.
mkdir -p gpurun_out
L=$PWD/paper_2503_08461_b200/_lib
FASTCACHE_LIB=$L/libfastcache_trace.so timeout 300 python scripts/trace_press.py c3l 2>&1 | tail -6
timeout 900 ncu --set full --clock-control none -k regex:"snapkv_tc" -s 3 -c 1 -o /tmp/prof_c3l -f \
  python bench.py --config c3l --legs "" --steps 1 --warmup 3 --e2e-steps 0 --no-cpu-baseline --parity-segments 0 > gpurun_out/ncu_c3l.log 2>&1
ncu -i /tmp/prof_c3l.ncu-rep --page raw --csv > gpurun_out/prof_c3l.raw.csv 2>/dev/null
python scripts/ncu_stalls.py /tmp/prof_c3l.ncu-rep fc_snapkv_tc.cu 199-263 264-299 300-323 324-452 453-524 525-560 561-595 596-640 > gpurun_out/prof_c3l_stalls.txt 2>&1; cat gpurun_out/prof_c3l_stalls.txt | head -60; python scripts/ncu_summary.py gpurun_out/prof_c3l.raw.csv c3l_r2b 2>&1 | head -5
