"""The C-ABI library loads, exports every symbol include/bflybfs.h declares,
and behaves on host-only calls (no GPU needed)."""

import ctypes
import os
import re

import pytest

from paper_2103_13577_b200 import _lib

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def declared_symbols():
    text = open(os.path.join(ROOT, "include", "bflybfs.h")).read()
    return sorted(set(re.findall(r"\b(bfb_[a-z0-9_]+)\s*\(", text)))


def test_header_symbols_exported():
    lib = ctypes.CDLL(_lib.LIB_PATH)
    names = declared_symbols()
    assert len(names) >= 20
    for name in names:
        assert hasattr(lib, name), name
    assert set(names) == set(_lib.EXPORTED)


def test_version_and_library_is_sm100a():
    assert b"sm_100a" in _lib.load().bfb_version()
    data = open(_lib.LIB_PATH, "rb").read()
    assert b"sm_100a" in data or b"sm_100" in data


def test_error_mapping():
    with pytest.raises(ValueError):
        _lib.check(_lib.ERR_ROOT)
    with pytest.raises(RuntimeError):
        _lib.check(_lib.ERR_CUDA)
    with pytest.raises(MemoryError):
        _lib.check(_lib.ERR_OOM)


def test_no_gpu_fails_loudly():
    if _lib.device_count() > 0:
        pytest.skip("GPU present")
    from paper_2103_13577_b200.device import DeviceGraph

    with pytest.raises(RuntimeError):
        DeviceGraph(0)


def test_product_never_imports_oracle():
    pkg = os.path.join(ROOT, "paper_2103_13577_b200")
    for dirpath, _, files in os.walk(pkg):
        for f in files:
            if f.endswith((".py", ".cu", ".cuh", ".h")):
                txt = open(os.path.join(dirpath, f)).read()
                assert "import oracle" not in txt and "from oracle" not in txt, f


def test_levels_readout_bytes():
    """bench.py's e2e d2h accounting mirrors csrc/host_out.cu read_levels:
    4 bits per vertex up to 15 levels (15 = UNREACHED), 8 up to 255, else 32."""
    from paper_2103_13577_b200.device import levels_readout_bytes

    assert levels_readout_bytes(1 << 29, 8) == 1 << 28
    assert levels_readout_bytes(7, 15) == 4
    assert levels_readout_bytes(7, 16) == 7
    assert levels_readout_bytes(1000, 255) == 1000
    assert levels_readout_bytes(1000, 256) == 4000
