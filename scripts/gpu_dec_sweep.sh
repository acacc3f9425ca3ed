#!/bin/bash
timeout 300 python -m pytest tests/test_gpu_decode.py -q 2>&1 | tail -1
for i in 1 2 3; do
timeout 300 python bench.py --config c2d --steps 2 --warmup 3 --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.load(sys.stdin); r=d['roofline']; print('dev_us', round(r['attn_us_per_layer'],2), 'frac', round(r['frac'],4), 'tpot', round(d['tpot_ms'],3))"
done
