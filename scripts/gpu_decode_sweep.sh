#!/bin/bash
for w in 1 2 4 8 16; do
FC_DECODE_WAVES=$w timeout 600 python bench.py --config c2d --steps 2 --warmup 3 --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.load(sys.stdin); print('waves', $w, 'attn_us', d['roofline']['attn_us_per_layer'], 'frac', d['roofline']['frac'], 'tpot', d['tpot_ms'])"
done
