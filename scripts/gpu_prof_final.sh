#!/bin/bash
# Final profile capture of the round: ncu --set full of the three press kernels and the c2 launch list.
mkdir -p gpurun_out
for c in c2 c3 c4w; do
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:"press_kernel|snapkv_tc|ea_tc" -s 3 -c 1 \
    -o gpurun_out/prof_$c -f python bench.py --config $c --steps 1 --warmup 3 --e2e-steps 0 --no-cpu-baseline > gpurun_out/ncu_$c.log 2>&1
  tail -1 gpurun_out/ncu_$c.log
done
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_c2.csv \
  python bench.py --steps 2 --warmup 3 --e2e-steps 0 --no-cpu-baseline > /dev/null 2>&1
ls -la gpurun_out/launches_c2.csv
