"""B200-native FastCache compression-stage hot path (arXiv 2503.08461).

Drop-in for the reference ``kvservesim`` compressor / pool API
(``kvservesim.kv``, ``kvservesim.pool``; re-exports follow the reference
``__init__.py:26-37,50``), extended with batched device presses and a paged
device pool. See DESIGN.md.
"""

from .kv import (
    AlreadyCompressed,
    CompressorSpec,
    EmptyInput,
    EmptyRequest,
    KVCacheSpec,
    KVSegment,
    MapKind,
    Modality,
    ModelConfig,
    PressKind,
    chunk_weights,
    compress_tensor,
    compressed_spec,
    kv_bytes,
    split_modalities,
)
from .pool import (
    BlockStats,
    CacheHandle,
    CapacityExceeded,
    CompressResult,
    DeviceError,
    DoubleFree,
    HandleState,
    InvalidState,
    KVCachePool,
    LedgerEntry,
    MemorySample,
    PoolMode,
    PoolStats,
)

__version__ = "0.1.0"

__all__ = [
    "AlreadyCompressed",
    "BlockStats",
    "CacheHandle",
    "CapacityExceeded",
    "CompressResult",
    "CompressorSpec",
    "DeviceError",
    "DoubleFree",
    "EmptyInput",
    "EmptyRequest",
    "HandleState",
    "InvalidState",
    "KVCachePool",
    "KVCacheSpec",
    "KVSegment",
    "LedgerEntry",
    "MapKind",
    "MemorySample",
    "Modality",
    "ModelConfig",
    "PoolMode",
    "PoolStats",
    "PressKind",
    "chunk_weights",
    "compress_tensor",
    "compressed_spec",
    "kv_bytes",
    "split_modalities",
]
