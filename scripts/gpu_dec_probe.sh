#!/bin/bash
L=$PWD/paper_2503_08461_b200/_lib
for lib in ${LIBS:-libfastcache.so}; do
FASTCACHE_LIB=$L/$lib timeout 300 python bench.py --config c2d --steps 2 --warmup 3 --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.load(sys.stdin); r=d['roofline']; print('$lib', 'dev_us', round(r['attn_us_per_layer'],2), 'frac', round(r['frac'],4))"
done
