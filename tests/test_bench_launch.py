"""bench.py's launch contract on CPU: ``--gpus N`` without a torchrun environment re-execs
itself as N ranks (torch.distributed.run, 127.0.0.1) and rank 0 alone prints one JSON line;
a WORLD_SIZE that disagrees with --gpus is refused. Uses the CPU reference arm on config 1,
so no GPU is needed (the driver's N>1 launches)."""

import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
BENCH = os.path.join(ROOT, "bench.py")


def _env(**kw):
    env = {k: v for k, v in os.environ.items()
           if k not in ("WORLD_SIZE", "RANK", "LOCAL_RANK", "MASTER_ADDR", "MASTER_PORT")}
    env.update(kw)
    return env


def test_gpus_two_self_launches_two_ranks_and_prints_once():
    out = subprocess.run([sys.executable, BENCH, "--gpus", "2", "--impl", "reference",
                          "--config", "c1", "--steps", "1", "--warmup", "3"],
                         capture_output=True, text=True, timeout=600, env=_env())
    assert out.returncode == 0, out.stderr[-2000:]
    lines = [ln for ln in out.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1, out.stdout
    rec = json.loads(lines[0])
    assert rec["impl"] == "reference" and rec["ranks"] == 2


def test_world_size_mismatch_is_refused():
    out = subprocess.run([sys.executable, BENCH, "--gpus", "2", "--impl", "reference",
                          "--config", "c1", "--steps", "1", "--warmup", "3"],
                         capture_output=True, text=True, timeout=120,
                         env=_env(WORLD_SIZE="3", RANK="0", LOCAL_RANK="0"))
    assert out.returncode != 0 and "WORLD_SIZE=3" in out.stderr
