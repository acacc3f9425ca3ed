#!/bin/bash
# Full GPU validation + the round's profile captures (run under gpurun).
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -q 2>&1 | tail -3
python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
for c in c2 c3; do
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:"press_kernel|snapkv_tc|ea_tc" -s 3 -c 1 \
    -o gpurun_out/prof_$c -f python bench.py --config $c --steps 1 --warmup 3 --e2e-steps 0 --no-cpu-baseline > gpurun_out/ncu_$c.log 2>&1
done
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"ea_tc" -s 1 -c 1 \
  -o gpurun_out/prof_c4w -f python bench.py --config c4w --steps 1 --warmup 3 --e2e-steps 0 --no-cpu-baseline > gpurun_out/ncu_c4w.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_c2.csv \
  python bench.py --steps 2 --warmup 3 --e2e-steps 0 --no-cpu-baseline > /dev/null 2>&1
ls gpurun_out
