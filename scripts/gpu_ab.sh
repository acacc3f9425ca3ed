#!/bin/bash
# A/B one kernel change: parity of the press suites, then timing of CONFIGS for LIBS
# (default: the shipped library and the `make alt ALTFLAGS=...` build).
mkdir -p gpurun_out
timeout 900 python -m pytest ${TESTS:-tests/test_gpu_press.py tests/test_gpu_long.py tests/test_gpu_edges.py tests/test_gpu_scale.py} -q -x 2>&1 | tail -2
L=$PWD/paper_2503_08461_b200/_lib
for c in ${CONFIGS:-c3g c3}; do
for lib in ${LIBS:-libfastcache.so libfastcache_alt.so}; do
FASTCACHE_LIB=$L/$lib timeout 300 python bench.py --config $c --legs "" --steps 5 --warmup 3 --e2e-steps 0 --no-cpu-baseline $EXTRA 2>/dev/null | python -c "import json,sys; d=json.load(sys.stdin); print('$lib $c', round(d['ms_per_step'],3), round(d['roofline']['frac'],4), d.get('parity',{}).get('mismatches'), d.get('clocks',{}).get('sm_mhz'))"
done; done
