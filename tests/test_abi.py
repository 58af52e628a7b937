"""The C-ABI boundary (include/tio.h) without a GPU: the library loads, every
declared entry point is exported, and compute paths fail loudly (no CPU
fallback) when no CUDA device is visible."""

from __future__ import annotations

import ctypes
import os
import re

import pytest

from conftest import ROOT
from paper_2506_06472_b200 import _native

HEADER = os.path.join(ROOT, "include", "tio.h")


def declared_symbols() -> list[str]:
    text = open(HEADER).read()
    return sorted(set(re.findall(r"^\s*int\s+(tio_\w+)\s*\(", text, re.M)))


def test_header_declares_the_boundary():
    syms = declared_symbols()
    for must in ("tio_trace_create", "tio_lifetime", "tio_plan_create", "tio_plan_write",
                 "tio_last_error"):
        assert must in syms, must
    assert set(syms) == set(_native.EXPORTS), "ctypes binding and header disagree"


def test_library_exports_every_declared_symbol():
    lib = _native.load()
    for name in declared_symbols():
        assert hasattr(lib, name), name
    assert lib.tio_abi_version() == 1


def test_no_torch_types_in_header():
    text = open(HEADER).read()
    assert "torch" not in text.replace("no torch types", "")
    assert "at::" not in text and "c10" not in text


def test_transfer_duration_is_exact_host_arithmetic():
    # bandwidth.py:75-84 known answers (reference test_bandwidth.py:12-26)
    assert _native.transfer_duration(20_000.0, 100_000_000) == 5_000
    assert _native.transfer_duration(6_500.0, 100_000_000) == 15_385
    assert _native.transfer_duration(2.0, 5) == 3
    assert _native.transfer_duration(0.5, 3) == 6
    assert _native.transfer_duration(1e9, 0) == 0
    with pytest.raises(_native.TioError):
        _native.transfer_duration(0.0, 10)


def test_last_error_round_trip():
    lib = _native.load()
    assert lib.tio_transfer_duration(ctypes.c_double(-1.0), ctypes.c_int64(1),
                                     ctypes.byref(ctypes.c_int64())) == _native.TIO_ERR_CHANNEL_CONFIG
    assert "rate" in _native.last_error()


def test_compute_fails_loudly_without_device():
    import torch
    if torch.cuda.is_available():
        pytest.skip("a GPU is visible")
    from paper_2506_06472_b200 import gen_random_trace, plan_migrations, ChannelRates
    tr = gen_random_trace(1, 8, 4)
    with pytest.raises(_native.NativeUnavailable):
        plan_migrations(tr, 10**9, ChannelRates.symmetric(1000))
