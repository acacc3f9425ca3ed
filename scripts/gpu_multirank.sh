#!/bin/bash
# Two ranks sharing the one GPU (gloo backend) exercise bench.py's N>1 path.
export FASTCACHE_DIST_BACKEND=gloo
for c in c2 c3; do
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29511 bench.py --gpus 2 --config $c --steps 3 --warmup 3 --e2e-steps 1 2>gpurun_out/mr_$c.err | tail -1 | python -c "import json,sys; d=json.load(sys.stdin); print('$c', d['n_gpus'], d['value'], d['scaling'], d.get('e2e',{}).get('value'))"
tail -2 gpurun_out/mr_$c.err
done
timeout 900 python -m pytest tests -m gpu -q 2>&1 | tail -2
