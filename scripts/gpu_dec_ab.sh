#!/bin/bash
L=$PWD/paper_2503_08461_b200/_lib
timeout 300 python -m pytest tests/test_gpu_decode.py -q -x 2>&1 | tail -1
for lib in libfastcache.so libfc_olddec.so; do
FASTCACHE_LIB=$L/$lib timeout 300 python bench.py --config c2d --steps 3 --warmup 3 --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.load(sys.stdin); r=d['roofline']; print('$lib', 'dev_us', r['attn_us_per_layer'], 'in_step_us', r['attn_us_per_layer_in_step'], 'frac', r['frac'], 'tpot', d['tpot_ms'])"
done
