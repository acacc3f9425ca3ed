"""The C-ABI library loads without a GPU and exports exactly what the header declares.

No compute calls: struct layouts are checked against a tiny C program
compiled with gcc from include/fastcache.h.
"""

import ctypes
import os
import re
import shutil
import subprocess
import tempfile

import pytest

from paper_2503_08461_b200 import _native as nat

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "fastcache.h")


def declared_symbols():
    with open(HEADER) as f:
        text = f.read()
    return sorted(set(re.findall(r"FC_API\s+[\w\s\*]+?\b(fc_\w+)\s*\(", text)))


def test_header_and_binding_agree():
    assert declared_symbols() == sorted(nat.EXPORTS)


def test_library_loads_and_exports_every_symbol():
    if not os.path.exists(nat.LIB_PATH):
        pytest.skip("library not built (run __graft_entry__.build())")
    lib = nat.load()
    for name in declared_symbols():
        assert hasattr(lib, name), name
    assert lib.fc_abi_version() == 1
    out = subprocess.run(["nm", "-D", "--defined-only", nat.LIB_PATH], capture_output=True,
                         text=True, check=True).stdout
    exported = {ln.split()[-1] for ln in out.splitlines() if " T " in ln}
    assert set(declared_symbols()) <= exported
    # nothing but the C ABI leaks out of the library
    assert {s for s in exported if s.startswith("fc_")} == set(declared_symbols())


def test_struct_layouts_match_ctypes():
    if shutil.which("gcc") is None:
        pytest.skip("gcc missing")
    structs = {
        "fc_model_config": nat.ModelConfigC, "fc_pool_options": nat.PoolOptionsC,
        "fc_press_config": nat.PressConfigC, "fc_press_inputs": nat.PressInputsC,
        "fc_press_outputs": nat.PressOutputsC, "fc_pool_stats": nat.PoolStatsC,
        "fc_profile": nat.ProfileC,
    }
    src = ["#include <stdio.h>", "#include <stddef.h>", f'#include "{HEADER}"', "int main(void){"]
    for cname, cls in structs.items():
        src.append(f'printf("{cname} %zu\\n", sizeof({cname}));')
        for fname, _ in cls._fields_:
            src.append(f'printf("{cname}.{fname} %zu\\n", offsetof({cname}, {fname}));')
    src.append("return 0;}")
    with tempfile.TemporaryDirectory() as d:
        c = os.path.join(d, "layout.c")
        exe = os.path.join(d, "layout")
        with open(c, "w") as f:
            f.write("\n".join(src))
        subprocess.run(["gcc", "-std=c99", "-Wall", "-Werror", c, "-o", exe], check=True)
        got = dict(ln.rsplit(" ", 1) for ln in subprocess.run([exe], capture_output=True, text=True,
                                                              check=True).stdout.splitlines())
    for cname, cls in structs.items():
        assert int(got[cname]) == ctypes.sizeof(cls), cname
        for fname, _ in cls._fields_:
            assert int(got[f"{cname}.{fname}"]) == getattr(cls, fname).offset, f"{cname}.{fname}"


def test_missing_library_fails_loudly(tmp_path):
    with pytest.raises(nat.NativeUnavailable):
        nat.load.__wrapped__(str(tmp_path / "nope.so")) if hasattr(nat.load, "__wrapped__") else \
            _load_fresh(str(tmp_path / "nope.so"))


def _load_fresh(path):
    saved = nat._lib
    nat._lib = None
    try:
        return nat.load(path)
    finally:
        nat._lib = saved


def test_device_pool_without_gpu_raises():
    import torch

    if torch.cuda.is_available():
        pytest.skip("has a GPU")
    from paper_2503_08461_b200 import KVCachePool, ModelConfig

    with pytest.raises(nat.NativeUnavailable):
        KVCachePool(ModelConfig("tiny", 4, 8, 64, 4), 1 << 30, device="cuda:0")


def test_device_only_calls_on_a_ledger_pool_fail_loudly():
    """The payload calls (host-resident compress, P.Store, decode) have no CPU fallback:
    on a ledger-only pool they raise instead of silently doing nothing."""
    import torch

    from paper_2503_08461_b200 import (
        CompressorSpec,
        KVCachePool,
        ModelConfig,
        PressKind,
        split_modalities,
    )

    cfg = ModelConfig("tiny", 2, 2, 64, 2)
    pool = KVCachePool(cfg, 1 << 30)
    h = pool.allocate(0, split_modalities(0, 8), 0.0)
    host = torch.zeros((2, 2, 2, 8, 64), dtype=torch.float16)
    with pytest.raises(nat.NativeUnavailable):
        pool.compress_batch([h], CompressorSpec(factor=2, press=PressKind.KNORM), 1.0,
                            host_kv=[host])
    assert h.spec.total_tokens == 8          # nothing was transitioned
    kv = torch.zeros((8, 2, 64), dtype=torch.float16)
    with pytest.raises(nat.NativeUnavailable):
        pool.write_prefill_kv([h], 0, kv, kv)
    with pytest.raises(nat.NativeUnavailable):
        pool.decode_attention([h], 0, torch.zeros((1, 2, 64), dtype=torch.float16))
    with pytest.raises(nat.NativeUnavailable):
        pool.write_decode_kv([h], 0, kv[:1], kv[:1])
    pool.compress_batch([h], CompressorSpec(factor=2, press=PressKind.KNORM), 1.0)
    pool.append_decode_batch([h], 1, 2.0)   # the ledger part works without a device
    assert h.spec.total_tokens == 5
    pool.verify_conservation()
