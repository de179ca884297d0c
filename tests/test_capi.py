"""The C-ABI library loads and exports every symbol include/fjg.h declares;
error categories (error.hpp:9-33) map to status codes and Python exceptions.
No device calls (CPU suite)."""
import ctypes as C
import os
import re

import pytest

from paper_2301_10841_b200 import _capi, plan as P

HEADER = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "include", "fjg.h")


def declared():
    src = open(HEADER).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(fjg_[a-z_0-9]+)\s*\(", src)))


def test_header_symbols_exported():
    lib = C.CDLL(_capi.LIB_PATH)
    names = declared()
    assert len(names) >= 20
    for n in names:
        assert hasattr(lib, n), n
    assert sorted(_capi.EXPORTED) == names


def test_struct_sizes_match_header():
    # fjg_result / fjg_exec_options layouts are mirrored in _capi.py
    assert C.sizeof(_capi.ExecOptions) == 32
    assert C.sizeof(_capi.Predicate) == 24
    assert C.sizeof(_capi.Result) == 8 * 3 + 8 + 4 + 4 + 8 * 3 + 8 * 32 * 3 + 8 * 4 + 8 * 3 + 8 * 2 + 8 + 8 * 4 + 8 * 16 + 4 * 16 + 4 * 2
    assert C.sizeof(_capi.MultiInfo) == 8 * 5 + 8 * 16 + 4 * 2 + 8 * 2


def test_error_codes():
    assert _capi.lib.fjg_abi_version() == 5
    with pytest.raises(_capi.ParseError):
        P.compile_plan("{not json", "free")
    with pytest.raises(_capi.ValidationError):
        P.compile_plan([{"rel": "R", "vars": ["x", "x"]}], "free")
    with pytest.raises(_capi.ValidationError):
        P.covers([[("R", ["x"])]], [{"rel": "R", "vars": ["x"]}], 5)
    assert "json" in _capi.lib.fjg_last_error().decode() or _capi.lib.fjg_last_error()


def test_no_device_without_gpu():
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    from paper_2301_10841_b200 import Engine
    with pytest.raises(_capi.Error):
        Engine(0)
