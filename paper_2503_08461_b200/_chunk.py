"""Device implementation of the reference ``compress_tensor`` (kv.py:211-239) via K7."""

from __future__ import annotations

import ctypes

import numpy as np

from . import _native as nat
from .kv import CompressorSpec, EmptyInput, MapKind, chunk_weights

_NP_TO_FC = {np.dtype(np.float16): nat.F16, np.dtype(np.float32): nat.F32,
             np.dtype(np.float64): nat.F64}


def compress_tensor(values, comp: CompressorSpec):
    import torch

    is_torch = isinstance(values, torch.Tensor)
    if is_torch:
        if values.dim() != 2:
            raise ValueError("values must be a 2-D (tokens, dim) array")
        fc_dtype = {torch.float16: nat.F16, torch.bfloat16: nat.BF16, torch.float32: nat.F32,
                    torch.float64: nat.F64}.get(values.dtype)
    else:
        values = np.asarray(values)
        if values.ndim != 2:
            raise ValueError("values must be a 2-D (tokens, dim) array")
        fc_dtype = _NP_TO_FC.get(values.dtype)
    n = values.shape[0]
    if n == 0:
        raise EmptyInput("cannot compress an empty token sequence")
    if fc_dtype is None:
        raise TypeError(f"compress_tensor on the GPU supports float16/bfloat16/float32/float64, "
                        f"got {values.dtype}")
    nat.require_cuda(None)
    lib = nat.load()
    dev = values.device if is_torch and values.is_cuda else torch.device("cuda", torch.cuda.current_device())
    src = values.contiguous() if is_torch else torch.from_numpy(np.ascontiguousarray(values))
    src = src.to(dev, non_blocking=False)
    rows = -(-n // comp.factor)
    seeded = comp.map_kind is MapKind.SEEDED_LINEAR
    out = torch.empty((rows, values.shape[1]), dtype=torch.float64 if seeded else src.dtype,
                      device=dev)
    weights = None
    if seeded:
        w = chunk_weights(comp)
        weights = (ctypes.c_double * len(w))(*[float(x) for x in w])
    cfg = nat.PressConfigC(nat.PRESS_SEEDEDLINEAR if seeded else nat.PRESS_MEANPOOL, comp.factor,
                           0, 1, 0, 0, 0, 0,
                           ctypes.cast(weights, ctypes.POINTER(ctypes.c_double)) if weights else None)
    stream = ctypes.c_void_p(torch.cuda.current_stream(dev).cuda_stream)
    with torch.cuda.device(dev):
        st = lib.fc_compress_tensor(ctypes.c_void_p(src.data_ptr()), n, values.shape[1], fc_dtype,
                                    ctypes.byref(cfg), ctypes.c_void_p(out.data_ptr()), stream)
    if st != nat.OK:
        msg = nat.last_error()
        if st == nat.ERR_EMPTY_INPUT:
            raise EmptyInput(msg)
        if st == nat.ERR_INVALID_ARG:
            raise ValueError(msg)
        raise RuntimeError(msg)
    if is_torch:
        return out
    return out.cpu().numpy()
