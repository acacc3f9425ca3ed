#!/bin/bash
# Round 2 profile captures: ncu --set full of each press kernel at its bench config (exported
# on the box to raw CSV + per-region stall digests; the .ncu-rep files are too large to ship
# back), the launch list of the default bench command, and compute-sanitizer memcheck over
# the spill / atomicity paths.
mkdir -p gpurun_out
for c in c2 c3 c4w c2m c3l; do
  timeout 900 ncu --set full --clock-control none --import-source on \
    -k regex:"press_kernel|snapkv_tc|ea_tc|chunk_pool" -s 3 -c 1 \
    -o /tmp/prof_r02_$c -f python bench.py --config $c --steps 1 --warmup 3 --e2e-steps 0 \
    --no-cpu-baseline --parity-segments 0 --legs "" > gpurun_out/ncu_r02_$c.log 2>&1
  tail -1 gpurun_out/ncu_r02_$c.log
  ncu -i /tmp/prof_r02_$c.ncu-rep --page raw --csv > gpurun_out/prof_r02_$c.raw.csv 2>/dev/null
  python scripts/ncu_lines.py /tmp/prof_r02_$c.ncu-rep 25 > gpurun_out/prof_r02_${c}_lines.txt 2>&1
done
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
  --log-file gpurun_out/r02_launches_default.csv python bench.py --steps 2 --warmup 3 \
  --parity-segments 8 --no-cpu-baseline > gpurun_out/r02_launches_default.out 2>&1
wc -l gpurun_out/r02_launches_default.csv
timeout 1200 compute-sanitizer --tool memcheck --error-exitcode 9 python -m pytest -q -x -m gpu \
  tests/test_gpu_long.py tests/test_gpu_atomic.py -k "spill or refused or exhaustion or decode" \
  > gpurun_out/r02_memcheck.log 2>&1; echo "memcheck rc=$?"; tail -3 gpurun_out/r02_memcheck.log
du -sh gpurun_out
