#!/bin/bash
L=$PWD/paper_2503_08461_b200/_lib
for lib in libfastcache.so libfc_r32_b3.so libfc_r32_b5.so libfc_r64_b3.so libfc_r16_b8.so; do
FASTCACHE_LIB=$L/$lib timeout 300 python bench.py --config c3 --steps 5 --warmup 3 --e2e-steps 0 --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.load(sys.stdin); print('$lib c3', d['ms_per_step'], d['roofline']['frac'])"
done
