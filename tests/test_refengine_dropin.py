"""The drop-in on the reference engine (CPU only).

1. The repo's engine restatement (``paper_2503_08461_b200.engine`` + ``scheduling`` +
   ``workload``, cost-model compress stage, ledger-only pool) replays the reference
   engine bit for bit: every request record, the pool ledger, the memory trace and the
   stage intervals hash identically to runs of the reference itself on the config-5
   trace (highload @ 40 req/s, 2000 requests, dynamic policy -- BASELINE.md §5's
   2.306 s p50 TTFT), its 2/4/8-way shards, a tight legacy-zombie pool, static / FCFS /
   coupled runs and attention mode. Pinned by tests/golden/engine_golden.json, generated
   from the reference by ``tests/refdrop/engine_runs.py``.
2. With ``/root/reference`` present: the reference package's own test suites
   (test_pool.py, test_engine.py, test_scheduling.py, test_kv.py minus the
   compress_tensor cases, which need the GPU) run with ``kvservesim.kv``, ``.pool``,
   ``.scheduling`` and ``.engine`` replaced by this repo's modules; the only failures are
   the reference's two known test bugs. And the unmodified reference
   engine, running on the repo's pool, produces the same fingerprints.
"""

import json
import os
import subprocess
import sys
import types

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
REF_SRC = "/root/reference/pkg/src"
REF_TESTS = "/root/reference/pkg/tests"
sys.path.insert(0, os.path.join(ROOT, "tests", "refdrop"))

import engine_runs  # noqa: E402

from paper_2503_08461_b200 import engine, kv, pool, scheduling, workload  # noqa: E402

GOLDEN = os.path.join(ROOT, "tests", "golden", "engine_golden.json")
KNOWN_REFERENCE_TEST_BUGS = {
    "test_engine.py::test_oversized_request_is_rejected_up_front",
    "test_scheduling.py::test_dynamic_formation_delegates_to_packing",
}


def _ours():
    return types.SimpleNamespace(engine=engine, kv=kv, pool=pool, scheduling=scheduling,
                                 workload=workload)


def test_engine_restatement_replays_reference_runs():
    with open(GOLDEN) as f:
        want = json.load(f)
    got = engine_runs.run_all(_ours())
    assert set(got) == set(want)
    for name in want:
        assert got[name] == want[name], name
    assert want["c5_g1"]["ttft_p50_s"] == pytest.approx(2.306, abs=5e-4)


def test_workload_generator_matches_reference_draws():
    with open(GOLDEN) as f:
        want = json.load(f)
    from dataclasses import replace

    reqs = workload.generate(replace(workload.WORKLOAD_PRESETS["highload"], rate_req_per_s=40.0))
    assert len(reqs) == want["c5_g1"]["requests"] == 2000
    mile = workload.generate(replace(workload.WORKLOAD_PRESETS["milebench-like"], num_requests=50))
    assert all(r.image_tokens % 576 == 0 and r.text_tokens >= 1 for r in mile)


def _env():
    env = dict(os.environ)
    env["PYTHONPATH"] = os.pathsep.join([REF_SRC, os.path.join(ROOT, "tests", "refdrop"), ROOT])
    env["PYTHONDONTWRITEBYTECODE"] = "1"
    return env


@pytest.mark.skipif(not os.path.isdir(REF_SRC), reason="/root/reference not present")
def test_reference_suites_pass_on_the_dropin_modules():
    out = subprocess.run(
        [sys.executable, "-m", "pytest", REF_TESTS, "-q", "-p", "no:cacheprovider",
         "-p", "alias_kvservesim", "-k", "not compress_tensor and not meanpool and not seeded_linear",
         "-rf"], capture_output=True, text=True, timeout=600, env=_env(), cwd="/tmp")
    failed = {ln.split()[1].split("tests/")[-1] for ln in out.stdout.splitlines()
              if ln.startswith("FAILED")}
    assert failed == KNOWN_REFERENCE_TEST_BUGS, out.stdout[-3000:]
    assert " passed" in out.stdout


@pytest.mark.skipif(not os.path.isdir(REF_SRC), reason="/root/reference not present")
def test_unmodified_reference_engine_on_the_dropin_pool():
    """kvservesim.engine is the reference's own; only kv / pool / scheduling are ours."""
    env = _env()
    env["FC_ALIAS_ENGINE"] = "0"
    code = ("import alias_kvservesim, json, sys, types, engine_runs\n"
            "import kvservesim.engine as e, kvservesim.workload as w, kvservesim.kv as k, "
            "kvservesim.pool as p, kvservesim.scheduling as s\n"
            "assert e.__file__.startswith('/root/reference')\n"
            "assert p.__name__ == 'paper_2503_08461_b200.pool'\n"
            "json.dump(engine_runs.run_all(types.SimpleNamespace(engine=e, kv=k, pool=p, "
            "scheduling=s, workload=w)), sys.stdout)\n")
    out = subprocess.run([sys.executable, "-c", code], capture_output=True, text=True,
                         timeout=600, env=env, cwd="/tmp")
    assert out.returncode == 0, out.stderr[-3000:]
    with open(GOLDEN) as f:
        assert json.loads(out.stdout) == json.load(f)
