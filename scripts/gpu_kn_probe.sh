#!/bin/bash
L=$PWD/paper_2503_08461_b200/_lib
for lib in ${LIBS:-libfastcache.so}; do
FASTCACHE_LIB=$L/$lib timeout 300 python bench.py --config c2 --steps 10 --warmup 3 --e2e-steps 0 --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.load(sys.stdin); print('$lib c2', round(d['ms_per_step'],4), round(d['roofline']['frac'],4))"
done
