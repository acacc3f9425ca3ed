"""CPU oracle for the FastCache compression-stage hot path.

TEST INFRASTRUCTURE ONLY. Only ``tests/``, ``__graft_entry__.smoke()`` and
``bench.py``'s CPU-baseline / ``--impl reference`` legs may import anything
under ``oracle/``, and only as the checker (or as the timed CPU reference
arm) -- never as a product path. The product package
(``paper_2503_08461_b200``) never imports this package.

Contents
--------
* ``synth``  -- the counter-based KV generator (bit-identical to the K8 CUDA
  kernel), so any sampled segment can be regenerated without materialising
  the device pool.
* ``press``  -- Knorm / SnapKV / ExpectedAttention scores, the (score desc,
  index asc) top-k and the ascending gather (the press
  math follows NVIDIA kvpress, which is NOT in /root/reference, has no pinned
  version and no call site there -- **parity for the presses is unpinned by
  the reference**; KATs in tests/ pin it).
* ``chunk``  -- restatement of the reference ``compress_tensor`` /
  ``chunk_weights`` (reference pkg/src/kvservesim/kv.py:197-239); pinned by
  the golden vectors generated from the reference itself
  (tests/golden/make_golden.py).
* ``blocks`` -- the deterministic block-allocator model (LIFO stack,
  batch-order pops, request-order pushes) the device allocator must match
  bit for bit.
* ``ledger`` -- restatement of the reference ``KVCachePool`` ledger
  (reference pool.py:87-257), pinned by golden traces from the reference.
"""
