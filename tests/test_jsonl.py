"""Trace ingest (reference trace.py:160-311): the multi-threaded C++ parser
(libtio csrc/jsonl.cu) must produce exactly the columns of the exact
parser, round-trip byte-identically through write_trace, and hand every
malformed file to the exact parser so errors keep the reference's messages.
Host-only."""

from __future__ import annotations

import hashlib

import pytest

from conftest import load_golden
from paper_2506_06472_b200 import (
    TraceParseError, TraceValidationError, TransformerGenConfig, gen_llama_trace, gen_random_trace,
    gen_transformer_trace, LlamaTraceConfig, parse_trace, write_trace)
from paper_2506_06472_b200 import trace as T


@pytest.mark.parametrize("make", [
    lambda: gen_random_trace(3, 50, 40),
    lambda: gen_transformer_trace(TransformerGenConfig(num_layers=2, hidden_dim=64, num_heads=4, batch=2,
                                                       seq_len=16, bytes_per_element=2, compute_rate=10**6,
                                                       seed=1)),
    lambda: gen_llama_trace(LlamaTraceConfig(microbatches=2)),
])
def test_fast_parse_equals_exact_parse(make):
    raw = write_trace(make())
    fast = T._fast_parse(raw)
    assert fast is not None
    exact = T._parse_exact(raw)
    assert fast[0].equals(exact.arrays())
    assert fast[1] == exact.meta
    assert write_trace(parse_trace(raw)) == raw


def test_golden_traces_round_trip():
    for rec in load_golden("c1")[:1]:
        tr = gen_transformer_trace(TransformerGenConfig(num_layers=12, hidden_dim=768, num_heads=12, batch=8,
                                                        seq_len=1024, bytes_per_element=4,
                                                        compute_rate=rec["gen"]["compute_rate"], seed=0))
        raw = write_trace(tr)
        assert hashlib.sha256(write_trace(parse_trace(raw))).hexdigest() == rec["trace_sha256"]


def test_escaped_names_and_meta():
    raw = (b'{"version": 1, "meta": {"a": [1, {"b": "x\\"y"}]}}\n'
           b'{"kernel": {"index": 0, "name": "k\\u00e9\\"q", "duration_us": 5, "stage": 1, "layer": null}}\n'
           b'{"kernel": {"name": "plain", "index": 1, "duration_us": 7}}\n'
           b'{"tensor": {"id": -3, "size_bytes": 9, "kind": "global", "accesses": [1], "layer": 2}}\n')
    fast = T._fast_parse(raw)
    assert fast is not None
    exact = T._parse_exact(raw)
    assert fast[0].equals(exact.arrays()) and fast[1] == exact.meta


@pytest.mark.parametrize("raw, line", [
    (b'{"version": 1}\n{"kernel": {"index": 0, "name": "k", "duration_us": true}}\n', 2),
    (b'{"version": 1}\n{"kernel": {"index": 0, "name": "k", "duration_us": 5, "bogus": 1}}\n', 2),
    (b'{"version": 1}\n{"tensor": {"id": 0, "size_bytes": 5, "kind": "weird", "accesses": []}}\n', 2),
    (b'{"version": 2}\n', 1),
    (b'{"version": 1}\n{"kernel": {"index": 0, "name": "k", "duration_us": 5}}\n'
     b'{"tensor": {"id": 0, "size_bytes": 5, "kind": "global", "accesses": [0]}}\n'
     b'{"kernel": {"index": 1, "name": "k", "duration_us": 5}}\n', 4),
    (b'{"version": 1}\n{"kernel": {"index": 0, "name": "k", "duration_us": 1.5}}\n', 2),
    (b'{"version": 1}\n{"kernel": {"index": 0, "name": "k", "duration_us": 99999999999999999999999}}\n', None),
])
def test_malformed_files_get_the_reference_errors(raw, line):
    assert T._fast_parse(raw) is None
    with pytest.raises((TraceParseError, TraceValidationError, ValueError)) as ei:
        parse_trace(raw)
    with pytest.raises(type(ei.value)) as ej:
        T._parse_exact(raw)
    assert str(ei.value) == str(ej.value)
    if line is not None and isinstance(ei.value, TraceParseError):
        assert ei.value.line == line


def test_validation_errors_from_fast_path():
    raw = (b'{"version": 1, "meta": {}}\n'
           b'{"kernel": {"index": 0, "name": "k", "duration_us": 5, "stage": null, "layer": null}}\n'
           b'{"tensor": {"id": 0, "size_bytes": 5, "kind": "global", "accesses": [3], "layer": null}}\n')
    assert T._fast_parse(raw) is not None
    with pytest.raises(TraceValidationError) as ei:
        parse_trace(raw)
    with pytest.raises(TraceValidationError) as ej:
        T._parse_exact(raw)
    assert str(ei.value) == str(ej.value)
