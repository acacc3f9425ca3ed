"""ctypes binding of the C ABI in include/fastcache.h (libfastcache.so).

The library is built in-tree by ``__graft_entry__.build()`` (or
``make -C paper_2503_08461_b200/csrc``) into ``paper_2503_08461_b200/_lib/``.
There is no fallback: every device operation of the package goes through this
library, and a missing library or GPU raises ``NativeUnavailable``.
"""

from __future__ import annotations

import ctypes
import os

# FASTCACHE_LIB (non-empty) points at another build of the library, e.g. an A/B variant
LIB_PATH = os.environ.get("FASTCACHE_LIB") or os.path.join(
    os.path.dirname(os.path.abspath(__file__)), "_lib", "libfastcache.so")

# fc_status
OK = 0
ERR_CAPACITY = 1
ERR_INVALID_STATE = 2
ERR_DOUBLE_FREE = 3
ERR_INVALID_ARG = 4
ERR_CUDA = 5
ERR_DEVICE = 6
ERR_UNSUPPORTED = 7
ERR_ALREADY_COMPRESSED = 8
ERR_EMPTY_INPUT = 9

# fc_dtype
F16, BF16, F32, U8, F64 = 0, 1, 2, 3, 4
# fc_press_kind
PRESS_KNORM, PRESS_SNAPKV, PRESS_EXPECTED_ATTENTION, PRESS_MEANPOOL, PRESS_SEEDEDLINEAR = range(5)
# fc_pool_mode
POOLED, LEGACY_ZOMBIE = 0, 1
# fc_synth_dist
SYNTH_SCALED, SYNTH_PLAIN = 0, 1

# every symbol include/fastcache.h declares (checked by tests/test_native_abi.py)
EXPORTS = (
    "fc_abi_version", "fc_last_error", "fc_launch_count", "fc_pool_create", "fc_pool_destroy",
    "fc_pool_arena", "fc_pool_alloc_batch", "fc_pool_compress_batch", "fc_pool_append",
    "fc_pool_release_batch", "fc_pool_get_stats", "fc_pool_synchronize", "fc_pool_block_table",
    "fc_pool_store_tokens", "fc_pool_load_tokens", "fc_synth_fill", "fc_compress_tensor",
    "fc_pool_set_profiling", "fc_pool_last_profile", "fc_pool_compress_host_batch",
    "fc_pool_write_kv", "fc_pool_decode_attention", "fc_pool_write_prefill_kv",
    "fc_pool_last_paths",
    "fc_pool_last_prefill_path",
)


class NativeUnavailable(RuntimeError):
    """The CUDA library (or a GPU) is missing; the package has no CPU fallback."""


class ModelConfigC(ctypes.Structure):
    _fields_ = [("num_layers", ctypes.c_int32), ("num_kv_heads", ctypes.c_int32),
                ("head_dim", ctypes.c_int32), ("bytes_per_element", ctypes.c_int32),
                ("dtype", ctypes.c_int32)]


class PoolOptionsC(ctypes.Structure):
    _fields_ = [("block_size", ctypes.c_int32), ("max_handles", ctypes.c_int32),
                ("max_blocks_per_handle", ctypes.c_int32), ("mode", ctypes.c_int32),
                ("num_blocks", ctypes.c_int64), ("arena", ctypes.c_void_p),
                ("arena_bytes", ctypes.c_uint64), ("device", ctypes.c_int32),
                ("reserved", ctypes.c_int32)]


class PressConfigC(ctypes.Structure):
    _fields_ = [("kind", ctypes.c_int32), ("factor", ctypes.c_int32), ("window", ctypes.c_int32),
                ("pool_kernel", ctypes.c_int32), ("n_sink", ctypes.c_int32),
                ("num_q_heads", ctypes.c_int32), ("per_segment", ctypes.c_int32),
                ("reserved", ctypes.c_int32), ("chunk_weights", ctypes.POINTER(ctypes.c_double))]


class PressInputsC(ctypes.Structure):
    _fields_ = [("q_window", ctypes.c_void_p), ("mean_q", ctypes.c_void_p),
                ("cov_q", ctypes.c_void_p)]


class PressOutputsC(ctypes.Structure):
    _fields_ = [("kept_idx", ctypes.c_void_p), ("scores", ctypes.c_void_p)]


class PoolStatsC(ctypes.Structure):
    _fields_ = [("current_bytes", ctypes.c_uint64), ("peak_bytes", ctypes.c_uint64),
                ("capacity_bytes", ctypes.c_uint64), ("live_handles", ctypes.c_int64),
                ("zombie_bytes_reclaimed", ctypes.c_uint64), ("allocation_count", ctypes.c_int64),
                ("num_blocks", ctypes.c_int64), ("free_blocks", ctypes.c_int64),
                ("used_blocks", ctypes.c_int64), ("block_bytes", ctypes.c_uint64),
                ("live_token_bytes", ctypes.c_uint64), ("fragmentation", ctypes.c_double),
                ("device_error", ctypes.c_int32), ("reserved", ctypes.c_int32)]


class ProfileC(ctypes.Structure):
    _fields_ = [("press_ms", ctypes.c_double), ("free_ms", ctypes.c_double),
                ("total_ms", ctypes.c_double), ("press_launches", ctypes.c_int64),
                ("total_launches", ctypes.c_int64)]


_P = ctypes.c_void_p
_I32 = ctypes.c_int32
_I64 = ctypes.c_int64
_U64 = ctypes.c_uint64
_PI64 = ctypes.POINTER(ctypes.c_int64)
_PU64 = ctypes.POINTER(ctypes.c_uint64)

_SIGS = {
    "fc_abi_version": (_I32, []),
    "fc_last_error": (ctypes.c_char_p, []),
    "fc_launch_count": (_I64, []),
    "fc_pool_create": (_I32, [ctypes.POINTER(ModelConfigC), _U64, ctypes.POINTER(PoolOptionsC),
                              ctypes.POINTER(_P)]),
    "fc_pool_destroy": (_I32, [_P]),
    "fc_pool_arena": (_I32, [_P, ctypes.POINTER(_P), _PU64, _PI64, _PU64]),
    "fc_pool_alloc_batch": (_I32, [_P, _I32, _PI64, _PI64, _PI64, _PU64, _PU64, _P]),
    "fc_pool_compress_batch": (_I32, [_P, _I32, _PI64, _PI64, ctypes.POINTER(PressConfigC),
                                      ctypes.POINTER(PressInputsC), ctypes.POINTER(PressOutputsC),
                                      _PU64, _PU64, _P]),
    "fc_pool_compress_host_batch": (_I32, [_P, _I32, _PI64, _PI64, ctypes.POINTER(PressConfigC),
                                           ctypes.POINTER(PressInputsC),
                                           ctypes.POINTER(PressOutputsC), ctypes.POINTER(_P),
                                           _PU64, _PU64, _P]),
    "fc_pool_append": (_I32, [_P, _I32, _PI64, _PI64, _PU64, _PU64, _P]),
    "fc_pool_write_kv": (_I32, [_P, _I32, _I32, _PI64, _PI64, _P, _P, _P]),
    "fc_pool_write_prefill_kv": (_I32, [_P, _I32, _I32, _PI64, _PI64, _PI64, _P, _P, _P]),
    "fc_pool_decode_attention": (_I32, [_P, _I32, _I32, _PI64, _I32, ctypes.c_float, _P, _P, _P]),
    "fc_pool_release_batch": (_I32, [_P, _I32, _PI64, _P]),
    "fc_pool_get_stats": (_I32, [_P, ctypes.POINTER(PoolStatsC)]),
    "fc_pool_synchronize": (_I32, [_P]),
    "fc_pool_block_table": (_I32, [_P, _I64, ctypes.POINTER(_P), ctypes.POINTER(_I32), _PI64]),
    "fc_pool_store_tokens": (_I32, [_P, _I64, _I64, _I64, _P, _P]),
    "fc_pool_load_tokens": (_I32, [_P, _I64, _I64, _I64, _P, _P]),
    "fc_synth_fill": (_I32, [_P, _I32, _PI64, _PI64, _U64, _I32, _P]),
    "fc_compress_tensor": (_I32, [_P, _I64, _I64, _I32, ctypes.POINTER(PressConfigC), _P, _P]),
    "fc_pool_set_profiling": (_I32, [_P, _I32]),
    "fc_pool_last_profile": (_I32, [_P, ctypes.POINTER(ProfileC)]),
    "fc_pool_last_paths": (_I32, [_P, _PI64]),
    "fc_pool_last_prefill_path": (_I32, [_P, ctypes.POINTER(ctypes.c_int32)]),
}

_lib = None


def load(path: str = LIB_PATH) -> ctypes.CDLL:
    """Load (once) and type the library; raises NativeUnavailable if it is not built."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(path):
        raise NativeUnavailable(
            f"{path} is missing: build it with `python -c 'import __graft_entry__ as g; g.build()'` "
            "(there is no CPU fallback)")
    lib = ctypes.CDLL(path)
    for name, (res, args) in _SIGS.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    _lib = lib
    return lib


def last_error() -> str:
    return load().fc_last_error().decode(errors="replace")


def launch_count() -> int:
    return int(load().fc_launch_count())


def i64_array(values) -> ctypes.Array:
    vals = [int(v) for v in values]
    return (ctypes.c_int64 * max(1, len(vals)))(*vals)


def require_cuda(device) -> None:
    import torch

    if not torch.cuda.is_available():
        raise NativeUnavailable("no CUDA device: the FastCache pool has no CPU fallback")
    load()
