#!/bin/bash
for lib in libfastcache.so libfastcache_alt.so; do
for i in 1 2; do
FASTCACHE_LIB=$PWD/paper_2503_08461_b200/_lib/$lib timeout 600 python bench.py --config c2d --steps 2 --warmup 3 --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.load(sys.stdin); print('$lib', 'attn_us', d['roofline']['attn_us_per_layer'], 'frac', d['roofline']['frac'], 'tpot', d['tpot_ms'])"
done; done
