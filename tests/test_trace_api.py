"""Trace model API (reference trace.py): the reference's test_trace.py known
answers restated against this package (parse, validate, round trip, start
times, mutated streams).  Host-only."""

from __future__ import annotations

import random

import pytest

from paper_2506_06472_b200 import (KernelRecord, TensorKind, TensorRecord, Trace, TraceParseError,
                                   TraceValidationError, gen_random_trace, parse_trace, validate_trace, write_trace)

EX1 = "\n".join(
    ['{"version": 1, "meta": {"model": "ex1"}}'] +
    [f'{{"kernel": {{"index": {i}, "name": "k{i}", "duration_us": 10000, "stage": null, "layer": null}}}}'
     for i in range(5)] +
    ['{"tensor": {"id": 0, "size_bytes": 100000000, "kind": "intermediate", "accesses": [0, 4], "layer": null}}',
     '{"tensor": {"id": 1, "size_bytes": 100000000, "kind": "intermediate", "accesses": [2], "layer": null}}']) + "\n"


def test_parse_known_answers():
    empty = parse_trace('{"version": 1, "meta": {}}\n')
    assert empty.num_kernels == 0 and empty.tensors == []
    tr = parse_trace(EX1)
    assert tr.kernel_start_times() == [0, 10_000, 20_000, 30_000, 40_000]
    assert tr.iteration_length() == 50_000 and tr.meta == {"model": "ex1"}


def test_parse_errors():
    with pytest.raises(TraceValidationError, match="tensor 1"):
        parse_trace(EX1.replace('"accesses": [2]', '"accesses": [7]'))
    with pytest.raises(TraceParseError, match="line 4"):
        parse_trace(EX1.replace('{"kernel": {"index": 2,', '{"kernel": {index: 2,'))
    with pytest.raises(TraceParseError, match="unknown kernel keys"):
        parse_trace(EX1.replace('"layer": null}}', '"layer": null, "color": 3}}', 1))
    lines = EX1.strip().splitlines()
    with pytest.raises(TraceParseError, match="kernel record after tensor"):
        parse_trace("\n".join([lines[0]] + lines[6:] + lines[1:6]))
    with pytest.raises(TraceParseError, match="version"):
        parse_trace('{"version": 9, "meta": {}}\n')


def test_validate(ex1):
    assert validate_trace(ex1).ok
    tr = Trace(kernels=[KernelRecord(i, f"k{i}", 10) for i in range(4)],
               tensors=[TensorRecord(0, 5, TensorKind.INTERMEDIATE, (3, 1))])
    rep = validate_trace(tr)
    assert len(rep.violations) == 1 and "not strictly increasing" in rep.violations[0]
    ex1.tensors.append(ex1.tensors[0])
    assert any("duplicate" in v for v in validate_trace(ex1).violations)


def test_round_trips():
    tr = parse_trace(EX1)
    assert parse_trace(write_trace(tr)) == tr
    empty = parse_trace('{"version": 1, "meta": {}}\n')
    data = write_trace(empty)
    assert data.decode("utf-8").count("\n") == 1 and parse_trace(data) == empty
    assert parse_trace('{"version": 1, "meta": {"x": 1, "y": 2}}\n') == \
        parse_trace('{"version": 1, "meta": {"y": 2, "x": 1}}\n')
    rng = random.Random(1)
    for _ in range(60):
        t = gen_random_trace(rng.randint(0, 10**6), rng.randint(0, 10), rng.randint(0, 8), size_range=(1, 10**9),
                             duration_range=(1, 10**5))
        assert validate_trace(t).ok and parse_trace(write_trace(t)) == t
    for _ in range(40):
        d = [rng.randint(1, 10**6) for _ in range(rng.randint(0, 12))]
        assert Trace([KernelRecord(i, "k", x) for i, x in enumerate(d)], []).kernel_start_times() == \
            [sum(d[:i]) for i in range(len(d))]


@pytest.mark.parametrize("mutant", [
    EX1.replace('"duration_us": 10000', '"duration_us": 0', 1),
    EX1.replace('"index": 3', '"index": 9'),
    EX1.replace('"size_bytes": 100000000', '"size_bytes": 0', 1),
    EX1.replace('"accesses": [0, 4]', '"accesses": []'),
    EX1.replace('"id": 1,', '"id": 0,'),
])
def test_mutated_traces_fail_validation(mutant):
    with pytest.raises(TraceValidationError):
        parse_trace(mutant)


def test_record_edits_invalidate_columns_and_device_cache():
    """edits to the record lists rebuild the columns and drop every
    device-side cache entry (the planner would otherwise plan a stale trace)."""
    tr = parse_trace(EX1)
    ks, ts = list(tr.kernels), list(tr.tensors)
    tr2 = Trace(ks, ts, {})
    a0 = tr2.arrays()
    assert tr2.arrays() is a0                      # unchanged lists: cached
    tr2.device_cache["lifetime"] = "stale"
    tr2.tensors.append(TensorRecord(9, 50_000_000, TensorKind.INTERMEDIATE, (1, 2), None))
    a1 = tr2.arrays()
    assert a1 is not a0 and a1.num_tensors == 3 and "lifetime" not in tr2.device_cache
    # replacing one kernel record twice (ids of dropped records may be reused)
    for d in (20_000, 30_000):
        tr2.kernels[1] = KernelRecord(1, "k1", d, None, None)
        assert tr2.iteration_length() == 40_000 + d
        assert tr2.kernel_start_times()[2] == 10_000 + d


def test_fast_parser_bad_meta_raises_reference_error():
    bad = EX1.replace('{"version": 1, "meta": {"model": "ex1"}}', '{"version": 1, "meta": {"model": "ex1",}}')
    with pytest.raises(TraceParseError, match="line 1"):
        parse_trace(bad)
