#!/bin/bash
# compute-sanitizer over the GPU suite. PYTORCH_NO_CUDA_MEMORY_CACHING=1 gives every torch tensor
# its own cudaMalloc, so memcheck sees exact bounds (the caching allocator hides small overruns).
PYTORCH_NO_CUDA_MEMORY_CACHING=1 timeout 2000 compute-sanitizer --tool memcheck --print-limit 10 \
  python -m pytest tests -m gpu -q 2>&1 | tail -3
timeout 900 compute-sanitizer --tool racecheck --racecheck-report hazard --print-limit 10 \
  python -m pytest tests/test_gpu_press.py -q -x \
  -k "knorm_parity and float16 or snapkv_parity and specs0 or expected_attention_parity and specs0" 2>&1 | tail -2
timeout 600 compute-sanitizer --tool synccheck --print-limit 10 \
  python -m pytest tests/test_gpu_press.py -q -x -k "snapkv_parity and specs0" 2>&1 | tail -2
