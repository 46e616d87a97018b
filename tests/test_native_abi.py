"""The C-ABI library loads and exports every symbol include/splbm_b200.h declares; without a GPU
the engine fails loudly (no CPU fallback)."""
import ctypes
import os
import re

import numpy as np
import pytest

import paper_1703_08015_b200 as P
from paper_1703_08015_b200 import _native

HEADER = os.path.join(os.path.dirname(os.path.dirname(__file__)), "include", "splbm_b200.h")


def declared_functions():
    src = open(HEADER).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(splbm_[a-z0-9_]+)\s*\(", src)))


def test_every_declared_symbol_is_exported_and_bound():
    L = _native.lib()
    assert L.missing_symbols == []
    names = declared_functions()
    assert len(names) >= 30
    for n in names:
        assert hasattr(L, n), n
        assert n in _native.SIGNATURES, n


def test_info_struct_layout_matches_the_library():
    """The library's sizeof(splbm_dev_info) equals the Python mirror's (a stale build against an
    older header would otherwise write past the caller's struct)."""
    for L in (_native.lib(), _native.lib("fma")):
        assert L.splbm_dev_info_size() == ctypes.sizeof(_native.DevInfo)
    src = re.sub(r"/\*.*?\*/", "", open(HEADER).read(), flags=re.S)
    body = re.search(r"typedef struct \{([^}]*)\} splbm_dev_info;", src).group(1)
    fields = re.findall(r"\b([a-z_0-9]+)(?:\[\d+\])?\s*[;,]", body)
    assert [f for f, _ in _native.DevInfo._fields_] == fields


def test_tolerance_mode_library_exports_the_same_abi():
    """libsplbm_b200_fma.so (arithmetic="fma") is the same sources with SPLBM_FMA=1."""
    L = _native.lib("fma")
    assert L.missing_symbols == []
    assert L is not _native.lib()
    with pytest.raises(P.ConfigError):
        _native.lib("fast")
    with pytest.raises(P.ConfigError):
        P.TileEngineT2C(P.Geometry.filled(2, (16, 16, 1)), 4, P.FluidModel(tau=0.4),
                        arithmetic="fma")


def test_library_is_sm100a():
    data = open(_native.LIB_PATH, "rb").read()
    assert b"sm_100a" in data or b"sm_100" in data


def test_no_gpu_fails_loudly():
    try:
        import torch
        if torch.cuda.is_available():
            pytest.skip("GPU present")
    except ImportError:
        pass
    g = P.Geometry.filled(2, (16, 16, 1))
    with pytest.raises(P.CudaError):
        P.TileEngineT2C(g, 4, P.FluidModel(tau=0.8))


def test_config_errors_before_device():
    g = P.Geometry.filled(2, (16, 16, 1))
    with pytest.raises(P.ConfigError):
        P.TileEngineT2C(g, 4, P.FluidModel(tau=0.4))
    with pytest.raises(P.ConfigError):
        P.TileEngineT2C(g, 4, P.FluidModel(tau=0.8, collision=P.CollisionKind.MRT, mrt_rates=[1.0] * 5))


def test_status_mapping():
    assert isinstance(P.errors.from_status(3, "x", 7), P.NumericalError)
    assert P.errors.from_status(3, "x", 7).step == 7
    assert isinstance(P.errors.from_status(5, "x"), P.ParseError)
