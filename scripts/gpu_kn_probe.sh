#!/bin/bash
L=$PWD/paper_2503_08461_b200/_lib
timeout 600 python -m pytest tests/test_gpu_press.py tests/test_gpu_edges.py -q -k "knorm or legacy or append" 2>&1 | tail -1
for lib in libfastcache.so libfc_kreg.so libfastcache.so libfc_kreg.so; do
FASTCACHE_LIB=$L/$lib timeout 300 python bench.py --config c2 --steps 10 --warmup 3 --e2e-steps 0 --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.load(sys.stdin); print('$lib c2', d['ms_per_step'], d['roofline']['frac'])"
done
