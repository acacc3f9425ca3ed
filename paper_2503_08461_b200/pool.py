"""Centralised KV-cache pool: the reference ledger plus a paged device arena.

Drop-in for ``kvservesim.pool`` (reference pkg/src/kvservesim/pool.py). With
no ``device`` the pool is exactly the reference: a byte ledger of cache
lifetimes with no payload (pool.py:1-9). With ``device="cuda:N"`` it also
owns the KV payload in HBM through the C ABI (include/fastcache.h):

* ``allocate``/``allocate_batch`` pop paged blocks from a device-resident
  free stack and fill the handle's device block table;
* ``compress_batch`` runs one batched press pass over many requests
  (Knorm / SnapKV / ExpectedAttention / the reference chunk fold), compacts
  the kept K/V rows in place inside each request's own blocks and frees the
  tail blocks in the same stream step -- then applies the reference ledger
  transitions in batch order with one ``now`` (engine.py:501-510);
* ``transition_compressed`` keeps the reference signature and compresses one
  handle with the pool's configured compressor;
* ``append_decode_tokens`` / ``release`` grow / free blocks on the device.

The ledger (trace, ledger entries, peak, zombie counters) is kept on the host
with Python ints exactly as the reference does, so ``memory_trace`` and
``ledger`` tuples are identical to ``kvservesim.KVCachePool`` for the same
call sequence.
"""

from __future__ import annotations

import ctypes
from dataclasses import dataclass, field, replace
from enum import Enum
from typing import NamedTuple, Sequence

from . import _native as nat
from .kv import (
    CompressorSpec,
    KVCacheSpec,
    MapKind,
    ModelConfig,
    PressKind,
    chunk_weights,
    compressed_spec,
    kv_bytes,
)


class HandleState(str, Enum):
    """pool.py:20-23."""

    RAW = "raw"
    COMPRESSED = "compressed"
    FREED = "freed"


class PoolMode(str, Enum):
    """pool.py:26-28."""

    POOLED = "pooled"
    LEGACY_ZOMBIE = "legacy"


class CapacityExceeded(RuntimeError):
    """An operation would push current bytes past pool capacity (pool.py:31-39)."""

    def __init__(self, requested: int, available: int):
        super().__init__(f"requested {requested} bytes but only {available} available")
        self.requested = requested
        self.available = available


class InvalidState(RuntimeError):
    """Operation applied to a handle in the wrong lifecycle state (pool.py:42-43)."""


class DoubleFree(RuntimeError):
    """A handle was released twice (pool.py:46-47)."""


class DeviceError(RuntimeError):
    """A CUDA call or a device-side invariant check failed."""


@dataclass
class CacheHandle:
    """One request's cache entry; identity is stable across compression (pool.py:50-60).

    ``block_table`` / ``n_blocks`` are device-pool extensions (None / 0 for a
    ledger-only pool).
    """

    handle_id: int
    request_id: int
    state: HandleState
    spec: KVCacheSpec
    bytes: int
    created_at: float
    retained_raw_bytes: int = 0
    _pool: object = field(default=None, repr=False, compare=False)

    @property
    def n_blocks(self) -> int:
        pool = self._pool
        if pool is None or pool._native is None or self.state is HandleState.FREED:
            return 0
        return pool._native.block_row(self.handle_id)[1]

    @property
    def block_table(self):
        """Device int32 tensor view of the handle's live block ids (device pools only)."""
        pool = self._pool
        if pool is None or pool._native is None or self.state is HandleState.FREED:
            return None
        return pool._native.block_table_view(self.handle_id)


@dataclass(frozen=True)
class PoolStats:
    """pool.py:63-70."""

    current_bytes: int
    peak_bytes: int
    capacity_bytes: int
    live_handles: int
    zombie_bytes_reclaimed: int
    allocation_count: int


class MemorySample(NamedTuple):
    time_s: float
    current_bytes: int
    peak_bytes: int
    live_handles: int


class LedgerEntry(NamedTuple):
    time_s: float
    op: str
    handle_id: int
    delta_bytes: int


@dataclass(frozen=True)
class BlockStats:
    """Device arena occupancy (new; no reference counterpart)."""

    num_blocks: int
    free_blocks: int
    used_blocks: int
    block_bytes: int
    live_token_bytes: int
    fragmentation: float


@dataclass
class CompressResult:
    """Optional per-request outputs of ``compress_batch`` (device tensors)."""

    kept_idx: list  # per request: int32 [L][H][K_r]
    scores: list    # per request: float32 [L][H][T_r]


_TORCH_DTYPES = {"float16": nat.F16, "bfloat16": nat.BF16, "float32": nat.F32, "uint8": nat.U8}


def _default_kv_dtype(bpe: int) -> str:
    return {1: "uint8", 2: "float16", 4: "float32"}[bpe]


class _CudaArray:
    """Minimal __cuda_array_interface__ wrapper to view a raw device pointer in torch."""

    def __init__(self, ptr: int, shape, typestr: str):
        self.__cuda_array_interface__ = {
            "shape": tuple(shape), "typestr": typestr, "data": (ptr, False), "version": 3,
            "strides": None,
        }


class _NativePool:
    """Owns one fc_pool (C ABI) plus its torch-allocated arena."""

    def __init__(self, config: ModelConfig, capacity_bytes: int, mode: PoolMode, device,
                 block_size: int, max_handles: int, max_tokens_per_handle: int,
                 num_blocks: int | None, kv_dtype: str):
        import torch

        nat.require_cuda(device)
        self.lib = nat.load()
        self.torch = torch
        self.device = torch.device(device)
        if self.device.type != "cuda":
            raise ValueError("device must be a CUDA device")
        if self.device.index is None:
            self.device = torch.device("cuda", torch.cuda.current_device())
        if kv_dtype not in _TORCH_DTYPES:
            raise ValueError(f"kv_dtype must be one of {sorted(_TORCH_DTYPES)}")
        if kv_dtype == "uint8":
            # The presses score K as floats; a 1-byte pool has no compiled press kernel,
            # so it is refused here rather than on its first compress call.
            raise NotImplementedError("device pools need a float KV dtype (float16, bfloat16, "
                                      "float32); bytes_per_element=1 pools are ledger-only")
        self.kv_dtype = kv_dtype
        self.torch_dtype = getattr(torch, kv_dtype)
        self.config = config
        self.block_size = block_size
        self.max_blocks = -(-max_tokens_per_handle // block_size)
        block_bytes = config.bytes_per_token * block_size
        if num_blocks is None:
            # One partial block per live handle (two in legacy mode: the retained raw row
            # and the live row), so byte admission implies block availability.
            partial = 2 if mode is PoolMode.LEGACY_ZOMBIE else 1
            num_blocks = capacity_bytes // block_bytes + partial * max_handles
        self.num_blocks = int(num_blocks)
        self.arena = torch.empty(self.num_blocks * block_bytes, dtype=torch.uint8,
                                 device=self.device)
        cfg = nat.ModelConfigC(config.num_layers, config.num_kv_heads, config.head_dim,
                               config.bytes_per_element, _TORCH_DTYPES[kv_dtype])
        opts = nat.PoolOptionsC(block_size, max_handles, self.max_blocks,
                                nat.POOLED if mode is PoolMode.POOLED else nat.LEGACY_ZOMBIE,
                                self.num_blocks, self.arena.data_ptr(), self.arena.numel(),
                                self.device.index, 0)
        handle = ctypes.c_void_p()
        cap = min(int(capacity_bytes), 2 ** 64 - 1)
        with torch.cuda.device(self.device):
            self._check(self.lib.fc_pool_create(ctypes.byref(cfg), cap, ctypes.byref(opts),
                                                ctypes.byref(handle)))
        self.ptr = handle

    def __del__(self):
        ptr = getattr(self, "ptr", None)
        if ptr is not None and getattr(self, "lib", None) is not None:
            try:
                self.lib.fc_pool_destroy(ptr)
            except Exception:  # noqa: BLE001 -- interpreter shutdown
                pass
            self.ptr = None

    # -- helpers ---------------------------------------------------------------
    def stream(self):
        return ctypes.c_void_p(self.torch.cuda.current_stream(self.device).cuda_stream)

    def _check(self, st: int, requested=None, available=None) -> None:
        if st == nat.OK:
            return
        msg = nat.last_error()
        if st == nat.ERR_CAPACITY:
            if requested is not None:
                raise CapacityExceeded(int(requested.value), int(available.value))
            raise CapacityExceeded(-1, -1)
        if st == nat.ERR_INVALID_STATE:
            raise InvalidState(msg)
        if st == nat.ERR_DOUBLE_FREE:
            raise DoubleFree(msg)
        if st in (nat.ERR_INVALID_ARG, nat.ERR_EMPTY_INPUT, nat.ERR_ALREADY_COMPRESSED):
            raise ValueError(msg)
        if st == nat.ERR_UNSUPPORTED:
            raise NotImplementedError(msg)
        raise DeviceError(msg)

    # -- operations ------------------------------------------------------------
    def alloc(self, request_ids: Sequence[int], tokens: Sequence[int]) -> list[int]:
        n = len(tokens)
        out = (ctypes.c_int64 * max(1, n))()
        req, avail = ctypes.c_uint64(), ctypes.c_uint64()
        self._check(self.lib.fc_pool_alloc_batch(self.ptr, n, nat.i64_array(request_ids),
                                                 nat.i64_array(tokens), out, ctypes.byref(req),
                                                 ctypes.byref(avail), self.stream()),
                    req, avail)
        return [int(out[i]) for i in range(n)]

    def compress(self, handle_ids, seg_tokens, comp: CompressorSpec, num_q_heads: int,
                 inputs, kept_out, scores_out, host_kv=None) -> None:
        kind = {
            PressKind.KNORM: nat.PRESS_KNORM,
            PressKind.SNAPKV: nat.PRESS_SNAPKV,
            PressKind.EXPECTED_ATTENTION: nat.PRESS_EXPECTED_ATTENTION,
        }.get(comp.press)
        weights = None
        if kind is None:
            kind = nat.PRESS_MEANPOOL if comp.map_kind is MapKind.MEAN_POOL else nat.PRESS_SEEDEDLINEAR
            if kind == nat.PRESS_SEEDEDLINEAR:
                w = chunk_weights(comp)
                weights = (ctypes.c_double * len(w))(*[float(x) for x in w])
        cfg = nat.PressConfigC(kind, comp.factor, comp.window, comp.pool_kernel, comp.n_sink,
                               num_q_heads, 1 if comp.per_segment else 0, 0,
                               ctypes.cast(weights, ctypes.POINTER(ctypes.c_double))
                               if weights is not None else None)
        q, mu, cov = inputs
        ins = nat.PressInputsC(q, mu, cov)
        outs = nat.PressOutputsC(kept_out, scores_out)
        segs = [int(x) for pair in seg_tokens for x in pair]
        req, avail = ctypes.c_uint64(), ctypes.c_uint64()
        if host_kv is None:
            self._check(self.lib.fc_pool_compress_batch(
                self.ptr, len(handle_ids), nat.i64_array(handle_ids), nat.i64_array(segs),
                ctypes.byref(cfg), ctypes.byref(ins), ctypes.byref(outs), ctypes.byref(req),
                ctypes.byref(avail), self.stream()), req, avail)
            return
        ptrs = (ctypes.c_void_p * max(1, len(host_kv)))(*[int(p) for p in host_kv])
        self._check(self.lib.fc_pool_compress_host_batch(
            self.ptr, len(handle_ids), nat.i64_array(handle_ids), nat.i64_array(segs),
            ctypes.byref(cfg), ctypes.byref(ins), ctypes.byref(outs), ptrs, ctypes.byref(req),
            ctypes.byref(avail), self.stream()), req, avail)

    def append(self, handle_ids, tokens) -> None:
        req, avail = ctypes.c_uint64(), ctypes.c_uint64()
        self._check(self.lib.fc_pool_append(self.ptr, len(handle_ids), nat.i64_array(handle_ids),
                                            nat.i64_array(tokens), ctypes.byref(req),
                                            ctypes.byref(avail), self.stream()), req, avail)

    def write_kv(self, layer: int, handle_ids, positions, k, v) -> None:
        pos = nat.i64_array(positions) if positions is not None else None
        self._check(self.lib.fc_pool_write_kv(self.ptr, layer, len(handle_ids),
                                              nat.i64_array(handle_ids), pos,
                                              ctypes.c_void_p(k.data_ptr()),
                                              ctypes.c_void_p(v.data_ptr()), self.stream()))

    def write_prefill(self, layer: int, handle_ids, cu_seqlens, tok_begin, k, v) -> None:
        tb = nat.i64_array(tok_begin) if tok_begin is not None else None
        self._check(self.lib.fc_pool_write_prefill_kv(
            self.ptr, layer, len(handle_ids), nat.i64_array(handle_ids), nat.i64_array(cu_seqlens),
            tb, ctypes.c_void_p(k.data_ptr()), ctypes.c_void_p(v.data_ptr()), self.stream()))

    def decode_attention(self, layer: int, handle_ids, num_q_heads: int, scale: float, q,
                         out) -> None:
        self._check(self.lib.fc_pool_decode_attention(
            self.ptr, layer, len(handle_ids), nat.i64_array(handle_ids), num_q_heads, scale,
            ctypes.c_void_p(q.data_ptr()), ctypes.c_void_p(out.data_ptr()), self.stream()))

    def release(self, handle_ids) -> None:
        self._check(self.lib.fc_pool_release_batch(self.ptr, len(handle_ids),
                                                   nat.i64_array(handle_ids), self.stream()))

    def stats(self) -> nat.PoolStatsC:
        st = nat.PoolStatsC()
        self._check(self.lib.fc_pool_get_stats(self.ptr, ctypes.byref(st)))
        return st

    def block_row(self, handle_id: int):
        ptr, nb, nt = ctypes.c_void_p(), ctypes.c_int32(), ctypes.c_int64()
        self._check(self.lib.fc_pool_block_table(self.ptr, handle_id, ctypes.byref(ptr),
                                                 ctypes.byref(nb), ctypes.byref(nt)))
        return int(ptr.value or 0), int(nb.value), int(nt.value)

    def block_table_view(self, handle_id: int):
        ptr, nb, _ = self.block_row(handle_id)
        if nb == 0:
            return self.torch.empty(0, dtype=self.torch.int32, device=self.device)
        return self.torch.as_tensor(_CudaArray(ptr, (nb,), "<i4"), device=self.device)

    def synth_fill(self, handle_ids, keys, seed: int, dist: int) -> None:
        self._check(self.lib.fc_synth_fill(self.ptr, len(handle_ids), nat.i64_array(handle_ids),
                                           nat.i64_array(keys), seed & (2 ** 64 - 1), dist,
                                           self.stream()))

    def store(self, handle_id: int, tok_begin: int, dense) -> None:
        n_tok = dense.shape[3]
        self._check(self.lib.fc_pool_store_tokens(self.ptr, handle_id, tok_begin, n_tok,
                                                  ctypes.c_void_p(dense.data_ptr()), self.stream()))

    def load(self, handle_id: int, tok_begin: int, n_tok: int):
        cfg = self.config
        out = self.torch.empty((cfg.num_layers, 2, cfg.num_kv_heads, n_tok, cfg.head_dim),
                               dtype=self.torch_dtype, device=self.device)
        if n_tok:
            self._check(self.lib.fc_pool_load_tokens(self.ptr, handle_id, tok_begin, n_tok,
                                                     ctypes.c_void_p(out.data_ptr()), self.stream()))
        return out


class KVCachePool:
    """Byte-exact cache accounting with strict admission (pool.py:87-257).

    Extra keyword arguments (all optional) turn on the device pool:

    * ``device`` -- e.g. ``"cuda:0"``: allocate the paged KV arena in HBM.
    * ``block_size`` -- tokens per block (default 16).
    * ``max_handles`` -- live handles the device block tables hold.
    * ``max_tokens_per_handle`` -- longest cache a handle may reach.
    * ``num_blocks`` -- arena blocks (default ``capacity // block_bytes +
      max_handles``, twice ``max_handles`` in legacy mode, so byte admission
      implies block availability).
    * ``kv_dtype`` -- element type the presses interpret ("float16",
      "bfloat16", "float32"; default from ``bytes_per_element``).
    * ``compressor`` -- the ``CompressorSpec`` ``transition_compressed`` uses.
    * ``num_q_heads`` -- query heads for SnapKV / ExpectedAttention inputs.
    """

    def __init__(
        self,
        config: ModelConfig,
        capacity_bytes: int,
        mode: PoolMode = PoolMode.POOLED,
        *,
        device=None,
        block_size: int = 16,
        max_handles: int = 1024,
        max_tokens_per_handle: int = 32768,
        num_blocks: int | None = None,
        kv_dtype: str | None = None,
        compressor: CompressorSpec | None = None,
        num_q_heads: int | None = None,
    ):
        if capacity_bytes < 1:
            raise ValueError("capacity_bytes must be >= 1")
        self.config = config
        self.capacity_bytes = capacity_bytes
        self.mode = mode
        self.handles: dict[int, CacheHandle] = {}
        self.memory_trace: list[MemorySample] = []
        self.ledger: list[LedgerEntry] = []
        self._current = 0
        self._peak = 0
        self._live = 0
        self._zombie_reclaimed = 0
        self._alloc_count = 0
        self._retained_handles = 0
        self._next_id = 0
        self.zombie_coexistence_observed = False
        self._deferred: set[int] = set()     # device-compressed, ledger transition pending
        self.compressor = compressor or CompressorSpec()
        self.num_q_heads = num_q_heads or config.num_kv_heads
        self._native: _NativePool | None = None
        if device is not None:
            self._native = _NativePool(config, capacity_bytes, mode, device, block_size,
                                       max_handles, max_tokens_per_handle, num_blocks,
                                       kv_dtype or _default_kv_dtype(config.bytes_per_element))

    # -- accounting internals (pool.py:119-143) ---------------------------------
    @property
    def current_bytes(self) -> int:
        return self._current

    @property
    def peak_bytes(self) -> int:
        return self._peak

    @property
    def available_bytes(self) -> int:
        return self.capacity_bytes - self._current

    @property
    def device(self):
        return None if self._native is None else self._native.device

    def _apply(self, now: float, op: str, handle_id: int, delta: int) -> None:
        self._current += delta
        assert 0 <= self._current <= self.capacity_bytes, "pool accounting broke"
        if self._current > self._peak:
            self._peak = self._current
        if self._retained_handles > 0:
            self.zombie_coexistence_observed = True
        self.ledger.append(LedgerEntry(now, op, handle_id, delta))
        self.memory_trace.append(MemorySample(now, self._current, self._peak, self._live))

    # -- operations --------------------------------------------------------------
    def allocate(self, request_id: int, spec: KVCacheSpec, now: float) -> CacheHandle:
        """Admit a raw cache; strict: the full footprint must fit now (pool.py:147-165)."""
        return self.allocate_batch([request_id], [spec], now)[0]

    def allocate_batch(self, request_ids: Sequence[int], specs: Sequence[KVCacheSpec],
                       now: float) -> list[CacheHandle]:
        """Batched ``allocate`` (atomic: all admitted in order, or none).

        Raises ``CapacityExceeded`` for the first member that would not fit
        after its predecessors were admitted.
        """
        if len(request_ids) != len(specs):
            raise ValueError("request_ids and specs differ in length")
        needs = [kv_bytes(self.config, s.total_tokens) for s in specs]
        avail = self.available_bytes
        for need in needs:
            if need > avail:
                raise CapacityExceeded(need, avail)
            avail -= need
        ids = None
        if self._native is not None:
            ids = self._native.alloc(request_ids, [s.total_tokens for s in specs])
        out = []
        for i, (rid, spec, need) in enumerate(zip(request_ids, specs, needs)):
            handle = CacheHandle(handle_id=self._next_id, request_id=rid, state=HandleState.RAW,
                                 spec=spec, bytes=need, created_at=now, _pool=self)
            assert ids is None or ids[i] == handle.handle_id, "device handle ids diverged"
            self._next_id += 1
            self.handles[handle.handle_id] = handle
            self._live += 1
            self._alloc_count += 1
            self._apply(now, "allocate", handle.handle_id, need)
            out.append(handle)
        return out

    def transition_compressed(self, handle: CacheHandle, new_spec: KVCacheSpec,
                              now: float) -> CacheHandle:
        """Swap a raw cache for its compressed form in one accounting step (pool.py:167-192).

        On a device pool this also compresses the payload with the pool's
        ``compressor``; ``new_spec`` must then be its ``compressed_spec``.
        """
        if handle.state is not HandleState.RAW:
            raise InvalidState(f"transition requires a raw handle, got {handle.state}")
        if self._native is not None:
            expect = compressed_spec(handle.spec, self.compressor)
            if [s.token_count for s in expect.segments] != [s.token_count for s in new_spec.segments]:
                raise ValueError("new_spec does not match the pool compressor's compressed_spec")
            self.compress_batch([handle], self.compressor, now, new_specs=[new_spec])
            return handle
        self._transition_ledger(handle, new_spec, now)
        return handle

    def commit_compressed(self, handles: Sequence[CacheHandle], new_specs: Sequence[KVCacheSpec],
                          now: float) -> None:
        """Ledger half of a ``compress_batch(..., defer_ledger=True)``: the reference
        per-member transitions (pool.py:167-192), in the given order, at ``now``."""
        handles, new_specs = list(handles), list(new_specs)
        for h in handles:
            if h.handle_id not in self._deferred:
                raise InvalidState(f"handle {h.handle_id} has no deferred compression")
        for h, spec in zip(handles, new_specs):
            self._transition_ledger(h, spec, now)
            self._deferred.discard(h.handle_id)

    def _transition_ledger(self, handle: CacheHandle, new_spec: KVCacheSpec, now: float) -> None:
        compressed = kv_bytes(self.config, new_spec.total_tokens)
        if self.mode is PoolMode.POOLED:
            delta = compressed - handle.bytes
            self._zombie_reclaimed += handle.bytes - compressed
        else:
            delta = compressed
            if delta > self.available_bytes:
                raise CapacityExceeded(delta, self.available_bytes)
            handle.retained_raw_bytes = handle.bytes
            self._retained_handles += 1
        handle.spec = new_spec
        handle.bytes = compressed
        handle.state = HandleState.COMPRESSED
        self._apply(now, "transition", handle.handle_id, delta)

    def compress_batch(self, handles: Sequence[CacheHandle], comp: CompressorSpec | None = None,
                       now: float = 0.0, *, q_window=None, mean_q=None, cov_q=None,
                       return_indices: bool = False, return_scores: bool = False,
                       new_specs: Sequence[KVCacheSpec] | None = None, host_kv=None,
                       defer_ledger: bool = False):
        """Compress many RAW handles in one batched device pass, then transition them.

        ``comp.press`` picks the scorer; every member keeps exactly
        ``compressed_spec(handle.spec, comp).total_tokens`` rows per (layer,
        kv-head) (reference ceil rule, kv.py:173-194). SnapKV needs
        ``q_window`` [n, L, Hq, w, D] (pool dtype, CUDA); ExpectedAttention
        needs ``mean_q`` [n, L, Hq, D] and ``cov_q`` [n, L, Hq, D, D] (fp32).
        The batch is atomic: every check runs before any mutation. Ledger
        transitions follow in batch order with the same ``now``
        (engine.py:501-510). Returns ``CompressResult`` when indices/scores
        are requested, else the handles.

        ``host_kv`` (optional): one pinned CPU tensor [L, 2, H, T_r, D] per
        handle holding its raw KV (the prefill output not yet in the pool).
        The library moves it into the handle's blocks as part of the call;
        for pooled Knorm / SnapKV only the K planes and the kept V rows cross
        PCIe (``fc_pool_compress_host_batch``). The tensors must stay alive
        until the pool's stream has run this call.

        ``defer_ledger=True`` (device pools): run the device pass now but leave the
        host ledger transitions to a later ``commit_compressed(handles, specs, now)``
        -- a serving engine charges the measured press time and transitions at the
        stage's completion time, as the reference does (engine.py:501-510). Returns
        the new specs (and the ``CompressResult`` as ``(specs, result)`` when
        indices/scores are requested).
        """
        comp = comp or self.compressor
        handles = list(handles)
        seen = set()
        for h in handles:
            if h.state is not HandleState.RAW or h.handle_id in self._deferred:
                raise InvalidState(f"transition requires a raw handle, got {h.state}")
            if h.handle_id in seen:
                raise ValueError("handle repeated in batch")
            seen.add(h.handle_id)
        expect = [compressed_spec(h.spec, comp) for h in handles]
        if new_specs is None:
            new_specs = expect
        new_specs = list(new_specs)
        if len(new_specs) != len(handles):
            raise ValueError("new_specs needs one spec per handle")
        if self._native is not None:
            # The device keeps exactly compressed_spec(h.spec, comp) rows per segment;
            # a different caller spec would desynchronise the ledger from the payload.
            for h, want, got in zip(handles, expect, new_specs):
                if [s.token_count for s in want.segments] != [s.token_count for s in got.segments]:
                    raise ValueError(f"new_spec of handle {h.handle_id} does not match "
                                     "compressed_spec(handle.spec, comp)")
        if self.mode is PoolMode.LEGACY_ZOMBIE:
            avail = self.available_bytes
            for spec in new_specs:
                need = kv_bytes(self.config, spec.total_tokens)
                if need > avail:
                    raise CapacityExceeded(need, avail)
                avail -= need
        result = None
        if self._native is not None and handles:
            result = self._device_compress(handles, new_specs, comp, q_window, mean_q, cov_q,
                                           return_indices, return_scores, host_kv)
        elif host_kv is not None:
            raise nat.NativeUnavailable("host_kv needs a device pool (pass device=...)")
        if defer_ledger:
            if self._native is None:
                raise ValueError("defer_ledger needs a device pool")
            self._deferred.update(h.handle_id for h in handles)
            return (new_specs, result) if (return_indices or return_scores) else new_specs
        for h, spec in zip(handles, new_specs):
            self._transition_ledger(h, spec, now)
        if return_indices or return_scores:
            return result
        return handles

    def _device_compress(self, handles, new_specs, comp, q_window, mean_q, cov_q,
                         return_indices, return_scores, host_kv=None):
        torch = self._native.torch
        cfg = self.config
        host_ptrs = None
        if host_kv is not None:
            host_kv = list(host_kv)
            if len(host_kv) != len(handles):
                raise ValueError("host_kv needs one tensor per handle")
            host_ptrs = []
            for h, t in zip(handles, host_kv):
                want = (cfg.num_layers, 2, cfg.num_kv_heads, h.spec.total_tokens, cfg.head_dim)
                if tuple(t.shape) != want or t.dtype != self._native.torch_dtype \
                        or t.device.type != "cpu" or not t.is_pinned() or not t.is_contiguous():
                    raise ValueError(f"host_kv tensors must be contiguous pinned CPU "
                                     f"{self._native.kv_dtype} tensors of shape {want}")
                host_ptrs.append(t.data_ptr())
        lh = cfg.num_layers * cfg.num_kv_heads
        n = len(handles)
        segs = []
        for h in handles:
            counts = [s.token_count for s in h.spec.segments]
            mods = [s.modality.value for s in h.spec.segments]
            if len(counts) == 1:
                segs.append((counts[0], 0) if mods[0] == "image" else (0, counts[0]))
            else:
                segs.append((counts[0], counts[1]))
        inputs = [None, None, None]
        dev = self._native.device
        hq = self.num_q_heads
        if comp.press is PressKind.SNAPKV:
            if q_window is None:
                raise ValueError("SnapKV needs q_window [n, L, Hq, w, D]")
            want = (n, cfg.num_layers, hq, comp.window, cfg.head_dim)
            if tuple(q_window.shape) != want or q_window.dtype != self._native.torch_dtype \
                    or q_window.device != dev or not q_window.is_contiguous():
                raise ValueError(f"q_window must be a contiguous {self._native.kv_dtype} CUDA "
                                 f"tensor of shape {want}")
            inputs[0] = q_window.data_ptr()
        elif comp.press is PressKind.EXPECTED_ATTENTION:
            if mean_q is None or cov_q is None:
                raise ValueError("ExpectedAttention needs mean_q and cov_q")
            want_m = (n, cfg.num_layers, hq, cfg.head_dim)
            want_c = want_m + (cfg.head_dim,)
            for t, want in ((mean_q, want_m), (cov_q, want_c)):
                if tuple(t.shape) != want or t.dtype != torch.float32 or t.device != dev \
                        or not t.is_contiguous():
                    raise ValueError(f"EA inputs must be contiguous fp32 CUDA tensors {want}")
            inputs[1], inputs[2] = mean_q.data_ptr(), cov_q.data_ptr()
        kept = [s.total_tokens for s in new_specs]
        raw = [h.spec.total_tokens for h in handles]
        kept_t = scores_t = None
        if return_indices:
            kept_t = torch.empty(sum(kept) * lh, dtype=torch.int32, device=dev)
        if return_scores:
            scores_t = torch.empty(sum(raw) * lh, dtype=torch.float32, device=dev)
        self._native.compress([h.handle_id for h in handles], segs, comp, hq, inputs,
                              kept_t.data_ptr() if kept_t is not None else None,
                              scores_t.data_ptr() if scores_t is not None else None,
                              host_ptrs)
        if not (return_indices or return_scores):
            return None
        res = CompressResult(kept_idx=[], scores=[])
        ko = so = 0
        for k, t in zip(kept, raw):
            if kept_t is not None:
                res.kept_idx.append(kept_t[ko:ko + k * lh].view(cfg.num_layers, cfg.num_kv_heads, k))
            if scores_t is not None:
                res.scores.append(scores_t[so:so + t * lh].view(cfg.num_layers, cfg.num_kv_heads, t))
            ko += k * lh
            so += t * lh
        return res

    def append_decode_tokens(self, handle: CacheHandle, token_count: int,
                             now: float) -> CacheHandle:
        """Grow a compressed cache by freshly decoded tokens (pool.py:194-211)."""
        if handle.state is not HandleState.COMPRESSED:
            raise InvalidState(f"append requires a compressed handle, got {handle.state}")
        if token_count < 1:
            raise ValueError("token_count must be >= 1")
        needed = kv_bytes(self.config, token_count)
        if needed > self.available_bytes:
            raise CapacityExceeded(needed, self.available_bytes)
        if self._native is not None:
            self._native.append([handle.handle_id], [token_count])
        handle.spec = replace(handle.spec,
                              decode_appended_tokens=handle.spec.decode_appended_tokens + token_count)
        handle.bytes += needed
        self._apply(now, "append", handle.handle_id, needed)
        return handle

    def append_decode_batch(self, handles: Sequence[CacheHandle], token_count: int,
                            now: float) -> list[CacheHandle]:
        """``append_decode_tokens(h, token_count, now)`` for every member, in order, as one
        device call (the per-step loop of engine.py:514-521). Atomic: every member is
        checked against the remaining capacity before any mutation."""
        handles = list(handles)
        if token_count < 1:
            raise ValueError("token_count must be >= 1")
        needed = kv_bytes(self.config, token_count)
        avail = self.available_bytes
        for h in handles:
            if h.state is not HandleState.COMPRESSED:
                raise InvalidState(f"append requires a compressed handle, got {h.state}")
            if needed > avail:
                raise CapacityExceeded(needed, avail)
            avail -= needed
        if self._native is not None and handles:
            self._native.append([h.handle_id for h in handles], [token_count] * len(handles))
        for h in handles:
            h.spec = replace(h.spec, decode_appended_tokens=h.spec.decode_appended_tokens + token_count)
            h.bytes += needed
            self._apply(now, "append", h.handle_id, needed)
        return handles

    def write_prefill_kv(self, handles: Sequence[CacheHandle], layer: int, k, v,
                         seq_lens: Sequence[int] | None = None,
                         tok_begin: Sequence[int] | None = None) -> None:
        """P.Store: one layer of the prefill's K and V for a batch, varlen
        layout ``k``, ``v`` = [sum_i n_i, Hkv, D] (pool dtype, CUDA) with request i's rows
        after request i-1's; ``seq_lens[i]`` rows (default: the handle's tokens) land at
        tokens ``tok_begin[i]`` + j (default 0) -- chunked prefill passes the chunk."""
        nv = self._need_native()
        cfg = self.config
        handles = list(handles)
        lens = [h.spec.total_tokens for h in handles] if seq_lens is None else [int(x) for x in seq_lens]
        if len(lens) != len(handles):
            raise ValueError("seq_lens needs one entry per handle")
        rows = sum(lens)
        want = (rows, cfg.num_kv_heads, cfg.head_dim)
        for t in (k, v):
            if tuple(t.shape) != want or t.dtype != nv.torch_dtype or t.device != nv.device \
                    or not t.is_contiguous():
                raise ValueError(f"k and v must be contiguous {nv.kv_dtype} CUDA tensors {want}")
        if tok_begin is not None:
            tok_begin = [int(x) for x in tok_begin]
            if len(tok_begin) != len(handles):
                raise ValueError("tok_begin needs one entry per handle")
        cu = [0]
        for n in lens:
            cu.append(cu[-1] + n)
        if handles:
            nv.write_prefill(layer, [h.handle_id for h in handles], cu, tok_begin, k, v)

    def write_decode_kv(self, handles: Sequence[CacheHandle], layer: int, k, v,
                        positions: Sequence[int] | None = None) -> None:
        """Write one token's K and V ([n, Hkv, D] each, pool dtype, CUDA) per handle into
        layer ``layer`` of its blocks at ``positions`` (default: its last token, the slot
        ``append_decode_batch`` just added) -- the UpdateKVCache of PAPER.md:255-261."""
        nv = self._need_native()
        cfg = self.config
        want = (len(handles), cfg.num_kv_heads, cfg.head_dim)
        for t in (k, v):
            if tuple(t.shape) != want or t.dtype != nv.torch_dtype or t.device != nv.device \
                    or not t.is_contiguous():
                raise ValueError(f"k and v must be contiguous {nv.kv_dtype} CUDA tensors {want}")
        if positions is not None:
            positions = [int(x) for x in positions]
            if len(positions) != len(handles):
                raise ValueError("positions needs one entry per handle")
        if handles:
            nv.write_kv(layer, [h.handle_id for h in handles], positions, k, v)

    def decode_attention(self, handles: Sequence[CacheHandle], layer: int, q, out=None,
                         scale: float | None = None):
        """softmax(scale * q K^T) V of one query token per handle over every live token of
        its (compressed + decoded) cache in layer ``layer``: q [n, Hq, D] (pool dtype,
        CUDA) -> out [n, Hq, D]. Hq = ``num_q_heads``; scale defaults to 1/sqrt(D)."""
        nv = self._need_native()
        cfg = self.config
        want = (len(handles), self.num_q_heads, cfg.head_dim)
        if tuple(q.shape) != want or q.dtype != nv.torch_dtype or q.device != nv.device \
                or not q.is_contiguous():
            raise ValueError(f"q must be a contiguous {nv.kv_dtype} CUDA tensor {want}")
        if out is None:
            out = nv.torch.empty_like(q)
        elif tuple(out.shape) != want or out.dtype != q.dtype or not out.is_contiguous():
            raise ValueError(f"out must be a contiguous {nv.kv_dtype} tensor {want}")
        if handles:
            nv.decode_attention(layer, [h.handle_id for h in handles], self.num_q_heads,
                                0.0 if scale is None else float(scale), q, out)
        return out

    def release(self, handle: CacheHandle, now: float) -> None:
        """Free a cache; legacy mode also drops the retained raw bytes (pool.py:213-224)."""
        self.release_batch([handle], now)

    def release_batch(self, handles: Sequence[CacheHandle], now: float) -> None:
        """Batched ``release`` in order (one device push for all members)."""
        seen = set()
        for h in handles:
            if h.state is HandleState.FREED or h.handle_id in seen:
                raise DoubleFree(f"handle {h.handle_id} already freed")
            seen.add(h.handle_id)
        if self._native is not None and handles:
            self._native.release([h.handle_id for h in handles])
        for handle in handles:
            delta = -(handle.bytes + handle.retained_raw_bytes)
            if handle.retained_raw_bytes > 0:
                self._retained_handles -= 1
                handle.retained_raw_bytes = 0
            handle.state = HandleState.FREED
            self._live -= 1
            self._apply(now, "release", handle.handle_id, delta)
            handle.bytes = 0

    # -- payload helpers (device pools) ------------------------------------------
    def _need_native(self) -> _NativePool:
        if self._native is None:
            raise nat.NativeUnavailable("this pool has no device arena (pass device=...)")
        return self._native

    def synth_fill(self, handles: Sequence[CacheHandle], seed: int = 0, keys=None,
                   dist: str = "scaled") -> None:
        """Fill the handles' raw KV with the deterministic generator (K8, bench input)."""
        nv = self._need_native()
        keys = [h.request_id for h in handles] if keys is None else list(keys)
        nv.synth_fill([h.handle_id for h in handles], keys, seed,
                      nat.SYNTH_SCALED if dist == "scaled" else nat.SYNTH_PLAIN)

    def store_tokens(self, handle: CacheHandle, kv, tok_begin: int = 0) -> None:
        """Write dense KV [L, 2, H, n, D] (CUDA, pool dtype) into the handle's blocks."""
        nv = self._need_native()
        cfg = self.config
        if kv.dim() != 5 or tuple(kv.shape[:3]) != (cfg.num_layers, 2, cfg.num_kv_heads) \
                or kv.shape[4] != cfg.head_dim or kv.dtype != nv.torch_dtype or kv.device != nv.device:
            raise ValueError("kv must be [L, 2, H, n, D] in the pool dtype on the pool device")
        nv.store(handle.handle_id, tok_begin, kv.contiguous())

    def load_tokens(self, handle: CacheHandle, tok_begin: int = 0, n_tok: int | None = None):
        """Gather the handle's tokens into a dense [L, 2, H, n, D] tensor."""
        nv = self._need_native()
        total = nv.block_row(handle.handle_id)[2]
        n_tok = total - tok_begin if n_tok is None else n_tok
        return nv.load(handle.handle_id, tok_begin, n_tok)

    def kv_cache(self, layer: int):
        """Device view of one layer's paged cache: [num_blocks, 2, H, block_size, D]."""
        nv = self._need_native()
        cfg = self.config
        bs = nv.block_size
        per_layer = nv.num_blocks * bs * cfg.bytes_per_token // cfg.num_layers
        raw = nv.arena[layer * per_layer:(layer + 1) * per_layer]
        return raw.view(nv.torch_dtype).view(nv.num_blocks, 2, cfg.num_kv_heads, bs, cfg.head_dim)

    def block_stats(self) -> BlockStats:
        nv = self._need_native()
        st = nv.stats()
        return BlockStats(st.num_blocks, st.free_blocks, st.used_blocks, st.block_bytes,
                          st.live_token_bytes, st.fragmentation)

    def set_profiling(self, enable: bool = True) -> None:
        """Record CUDA events around the press kernels of every compress call."""
        nv = self._need_native()
        nv._check(nv.lib.fc_pool_set_profiling(nv.ptr, 1 if enable else 0))

    def last_profile(self) -> dict:
        """Device timings (ms) of the most recent compress call (synchronising)."""
        nv = self._need_native()
        prof = nat.ProfileC()
        nv._check(nv.lib.fc_pool_last_profile(nv.ptr, ctypes.byref(prof)))
        return {"press_ms": prof.press_ms, "free_ms": prof.free_ms, "total_ms": prof.total_ms,
                "press_launches": prof.press_launches, "total_launches": prof.total_launches}

    def last_paths(self) -> dict:
        """Press launches of the most recent compress call per implementation:
        ``{"tc": tcgen05 kernels, "simt": SIMT press kernels, "chunk": chunk fold}``."""
        nv = self._need_native()
        out = (ctypes.c_int64 * 3)()
        nv._check(nv.lib.fc_pool_last_paths(nv.ptr, out))
        return {"tc": int(out[0]), "simt": int(out[1]), "chunk": int(out[2])}

    def last_prefill_path(self) -> str:
        """Kernel of the most recent ``write_prefill_kv``: ``"tma"`` (TMA head-group tiles,
        whole-chunk bulk stores), ``"copy"`` (register-copy kernel) or ``"none"``."""
        nv = self._need_native()
        out = ctypes.c_int32(-1)
        nv._check(nv.lib.fc_pool_last_prefill_path(nv.ptr, ctypes.byref(out)))
        return {1: "tma", 0: "copy"}.get(out.value, "none")

    def synchronize(self) -> None:
        if self._native is not None:
            self._native._check(self._native.lib.fc_pool_synchronize(self._native.ptr))

    # -- observation (pool.py:228-257) ---------------------------------------------
    def stats(self) -> PoolStats:
        return PoolStats(
            current_bytes=self._current,
            peak_bytes=self._peak,
            capacity_bytes=self.capacity_bytes,
            live_handles=self._live,
            zombie_bytes_reclaimed=self._zombie_reclaimed,
            allocation_count=self._alloc_count,
        )

    def snapshot(self, now: float) -> PoolStats:
        self.memory_trace.append(MemorySample(now, self._current, self._peak, self._live))
        return self.stats()

    def verify_conservation(self) -> None:
        """Replay-check the ledger (pool.py:245-257); device pools also check blocks."""
        live_total = sum(h.bytes + h.retained_raw_bytes for h in self.handles.values()
                         if h.state is not HandleState.FREED)
        ledger_total = sum(e.delta_bytes for e in self.ledger)
        if live_total != self._current or ledger_total != self._current:
            raise AssertionError(
                "conservation violated: "
                f"live={live_total} ledger={ledger_total} current={self._current}")
        if self._native is not None:
            st = self._native.stats()
            if st.current_bytes != self._current or st.live_handles != self._live:
                raise AssertionError(
                    f"device ledger diverged: device current={st.current_bytes} "
                    f"host={self._current}")
            bs = self._native.block_size
            want = 0
            for h in self.handles.values():
                if h.state is HandleState.FREED:
                    continue
                want += -(-h.spec.total_tokens // bs)
                if h.retained_raw_bytes:
                    raw_tokens = h.retained_raw_bytes // self.config.bytes_per_token
                    want += -(-raw_tokens // bs)
            if st.used_blocks != want:
                raise AssertionError(f"block accounting broke: used={st.used_blocks} want={want}")
