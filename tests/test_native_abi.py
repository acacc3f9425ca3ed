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
