"""pytest plugin (-p alias_kvservesim): make ``kvservesim.kv`` and ``kvservesim.pool`` the
repo's modules before the reference package is imported, so the reference engine,
metrics, experiment harness and the reference's own tests run unmodified on top of the
drop-in (tests/test_refengine_dropin.py)."""

import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

from paper_2503_08461_b200 import kv as _kv  # noqa: E402
from paper_2503_08461_b200 import pool as _pool  # noqa: E402
from paper_2503_08461_b200 import scheduling as _sched  # noqa: E402
from paper_2503_08461_b200 import engine as _eng  # noqa: E402

sys.modules["kvservesim.kv"] = _kv
sys.modules["kvservesim.pool"] = _pool
sys.modules["kvservesim.scheduling"] = _sched
if os.environ.get("FC_ALIAS_ENGINE", "1") == "1":
    sys.modules["kvservesim.engine"] = _eng

import kvservesim  # noqa: E402

kvservesim.kv, kvservesim.pool, kvservesim.scheduling = _kv, _pool, _sched   # not bound by import
kvservesim.engine = sys.modules["kvservesim.engine"]
assert kvservesim.KVCachePool is _pool.KVCachePool and kvservesim.compressed_spec is _kv.compressed_spec
from kvservesim import engine as _engine  # noqa: E402

assert _engine.KVCachePool is _pool.KVCachePool, "the reference engine must use the drop-in pool"
