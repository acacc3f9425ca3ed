#!/bin/bash
L=$PWD/paper_2503_08461_b200/_lib
for lib in libfastcache.so libfc_pf0.so libfc_pf4.so libfc_pf6.so; do
for c in c2 c3; do
FASTCACHE_LIB=$L/$lib timeout 300 python bench.py --config $c --steps 5 --warmup 3 --e2e-steps 0 --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.load(sys.stdin); print('$lib $c', d['ms_per_step'], d['roofline']['frac'])"
done; done
