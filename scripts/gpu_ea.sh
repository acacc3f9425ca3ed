#!/bin/bash
timeout 600 python -m pytest tests/test_gpu_press.py -x -q -k "expected_attention" 2>&1 | tail -2
timeout 600 python bench.py --config c4w --steps 5 --warmup 3 --e2e-steps 0 --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.load(sys.stdin); print('c4w ms', d['ms_per_step'], 'frac', d['roofline']['frac'])"
