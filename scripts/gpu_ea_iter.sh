#!/bin/bash
# EA iteration: parity of the EA paths, then c4w timing.
timeout 600 python -m pytest tests/test_gpu_press.py tests/test_gpu_edges.py tests/test_gpu_host.py -q -k "expected_attention" 2>&1 | tail -1
L=$PWD/paper_2503_08461_b200/_lib
for lib in ${LIBS:-libfastcache.so}; do
FASTCACHE_LIB=$L/$lib timeout 300 python bench.py --config c4w --steps 3 --warmup 3 --e2e-steps 0 --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.load(sys.stdin); print('$lib c4w', d['ms_per_step'], d['roofline']['frac'])"
done
