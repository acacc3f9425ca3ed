#!/bin/bash
# Round 2: full GPU suite, the default bench line (c2 + c3/c4w legs + sampled parity),
# and the self-launched 2-rank path on a 1-GPU box.
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,memory.total --format=csv > gpurun_out/gpu.txt
timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"
tail -5 gpurun_out/pytest_gpu.log
timeout 900 python bench.py > gpurun_out/bench_default.json 2> gpurun_out/bench_default.err; echo "bench rc=$?"
tail -3 gpurun_out/bench_default.err
timeout 600 python bench.py --gpus 2 --steps 5 --warmup 3 --legs "" --e2e-steps 0 --parity-segments 8 \
  > gpurun_out/bench_n2.json 2> gpurun_out/bench_n2.err; echo "bench n2 rc=$?"
tail -3 gpurun_out/bench_n2.err
