#!/bin/bash
for lib in libfastcache.so libfc_FC_EA_SLEEP.so libfc_FC_EA_PROXY_FENCE.so libfc_FC_EA_IDS_AFTER.so; do
echo "$lib: $(FASTCACHE_LIB=$PWD/paper_2503_08461_b200/_lib/$lib timeout 300 python -m pytest tests/test_gpu_press.py -q -k expected_attention 2>&1 | tail -1)"
done
FASTCACHE_LIB=$PWD/paper_2503_08461_b200/_lib/libfastcache.so timeout 300 python -m pytest tests/test_gpu_press.py -q -k expected_attention 2>&1 | grep -B2 "Error" | head -30
