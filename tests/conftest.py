"""Shared fixtures.  `gpu` marks tests that need a CUDA device (libtio)."""

from __future__ import annotations

import gzip
import json
import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
GOLDEN = os.path.join(ROOT, "tests", "golden")
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

from paper_2506_06472_b200 import (  # noqa: E402
    ChannelRates, KernelRecord, TensorKind, TensorRecord, make_trace)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (runs the sm_100a libtio path)")
    config.addinivalue_line("markers", "slow: long-running case")


def load_golden(name: str):
    path = os.path.join(GOLDEN, f"{name}.json.gz")
    if not os.path.exists(path):
        pytest.skip(f"golden fixture {name} not generated (tests/golden/make_golden.py)")
    with gzip.open(path, "rt", encoding="utf-8") as f:
        return json.load(f)


def mk_trace(durations, tensors, meta=None):
    """Same helper as reference pkg/tests/conftest.py:6-15:
    tensors = iterable of (id, size, kind, accesses[, layer])."""
    kernels = [KernelRecord(i, f"k{i}", d) for i, d in enumerate(durations)]
    recs = []
    for spec in tensors:
        tid, size, kind, acc = spec[:4]
        layer = spec[4] if len(spec) > 4 else None
        recs.append(TensorRecord(tid, size, TensorKind(kind), tuple(acc), layer))
    return make_trace(kernels, recs, meta or {})


@pytest.fixture
def ex1():
    """EX1 (reference conftest.py:18-25): five 10 ms kernels; A (100 MB) at
    k0 and k4, B (100 MB) at k2."""
    return mk_trace([10_000] * 5, [(0, 100_000_000, "intermediate", [0, 4]),
                                   (1, 100_000_000, "intermediate", [2])])


@pytest.fixture
def rates20k():
    return ChannelRates.symmetric(20_000)


def rates_of(rec) -> ChannelRates:
    so, sp, ho, hp = rec["rates"]
    return ChannelRates(so, sp, ho, hp)


def regen(rec):
    """Rebuild a golden case's trace with this repo's generator and check it
    against the reference's write_trace hash."""
    import hashlib
    from paper_2506_06472_b200 import gen_random_trace, write_trace
    g = rec["gen"]
    tr = gen_random_trace(g["seed"], g["num_kernels"], g["num_tensors"],
                          size_range=tuple(g["size_range"]), duration_range=tuple(g["duration_range"]),
                          global_fraction=g.get("global_fraction", 0.3))
    assert hashlib.sha256(write_trace(tr)).hexdigest() == rec["trace_sha256"]
    return tr
