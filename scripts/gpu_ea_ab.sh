#!/bin/bash
L=$PWD/paper_2503_08461_b200/_lib
timeout 300 python -m pytest tests/test_gpu_press.py tests/test_gpu_host.py -q -k "expected_attention or host" 2>&1 | tail -1
for lib in libfastcache.so libfc_vring.so; do
FASTCACHE_LIB=$L/$lib timeout 300 python bench.py --config c4w --steps 5 --warmup 3 --e2e-steps 0 --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.load(sys.stdin); print('$lib', d['ms_per_step'], d['roofline']['frac'])"
done
FASTCACHE_LIB=$L/libfastcache_trace.so timeout 300 python scripts/trace_ea.py 2>&1 | tail -3
