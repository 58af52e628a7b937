"""Pin the CPU oracle (oracle/tio_oracle.c) to the reference's own outputs.

The oracle is the checker of the GPU parity tests at sizes where the Python
reference cannot run (C2/C3).  Before it is trusted it must reproduce, bit
for bit, every golden vector the reference produced in tests/golden/
(make_golden.py): the criterion-2 and criterion-3 fuzz corpora of
test_acceptance.py:64-131 and the C1 plans of SURVEY §8d.  CPU only.
"""

from __future__ import annotations

import hashlib

import numpy as np
import pytest

from conftest import load_golden, regen
from oracle import oracle as O
from paper_2506_06472_b200 import TransformerGenConfig, gen_transformer_trace, write_trace


def _check_lifetime(arrays, rec):
    periods, timeline, active = O.lifetime(arrays)
    got = [[int(t), int(s), int(a), int(b), int(w)] for t, s, a, b, w in
           zip(periods["tensor_id"], periods["size"], periods["start"], periods["end"], periods["wraps"])]
    assert got == rec["periods"]
    assert timeline.tolist() == rec["timeline"]
    assert active.tolist() == rec["active"]
    return periods, timeline, active


def _check_plan(arrays, rec, lo=None):
    so, sp, ho, hp = rec["rates"]
    if "unsat_kernel" in rec:
        with pytest.raises(O.OracleUnsatisfiable) as ei:
            O.plan(arrays, rec["capacity"], so, sp, ho, hp, rec["host_cap"], lifetime_out=lo)
        assert ei.value.kernel == rec["unsat_kernel"]
        return
    p = O.plan(arrays, rec["capacity"], so, sp, ho, hp, rec["host_cap"], lifetime_out=lo)
    assert p["plan_bytes"].decode() == rec["plan"]
    assert p["residual"].tolist() == rec["residual"]
    got = []
    for c in p["committed"]:
        rel = [k for lo_, hi_ in c[9] for k in range(lo_, hi_ + 1)]
        got.append([c[0], c[1], c[2], int(c[3]), c[4], list(c[5]), list(c[6]), str(c[7]), c[8], rel])
    assert got == rec["committed"]


@pytest.mark.parametrize("corpus", ["crit2", "crit3", "extreme"])
def test_oracle_matches_reference_fuzz_corpus(corpus):
    cases = load_golden(corpus)
    assert len(cases) >= {"crit2": 1000, "crit3": 3000, "extreme": 300}[corpus]
    for rec in cases:
        tr = regen(rec)
        a = tr.arrays()
        lo = _check_lifetime(a, rec)
        _check_plan(a, rec, lo)


def test_oracle_matches_reference_c1():
    for rec in load_golden("c1"):
        cfg = TransformerGenConfig(num_layers=12, hidden_dim=768, num_heads=12, batch=8, seq_len=1024,
                                   bytes_per_element=4, compute_rate=rec["gen"]["compute_rate"], seed=0)
        tr = gen_transformer_trace(cfg)
        assert hashlib.sha256(write_trace(tr)).hexdigest() == rec["trace_sha256"]
        a = tr.arrays()
        lo = _check_lifetime(a, rec)
        _check_plan(a, rec, lo)
        # the SURVEY App. C fingerprints of the same plans
        assert hashlib.sha256(rec["plan"].encode()).hexdigest() == rec["plan_sha256"]


def test_c1_fingerprints_match_survey():
    want = {"ed841d86", "b5a35595", "4d1ff45f", "27c8b0f8"}
    assert {r["plan_sha256"][:8] for r in load_golden("c1")} == want


def test_oracle_matches_reference_llama1():
    from paper_2506_06472_b200 import LlamaTraceConfig, gen_llama_trace
    recs = load_golden("llama1")
    tr = gen_llama_trace(LlamaTraceConfig(microbatches=1))
    assert hashlib.sha256(write_trace(tr)).hexdigest() == recs[0]["trace_sha256"]
    a = tr.arrays()
    lo = _check_lifetime(a, recs[0])
    _check_plan(a, recs[0], lo)


def test_oracle_timeline_matches_bruteforce_residency():
    """Property of test_analysis.py:105-125 on the oracle's difference array."""
    from paper_2506_06472_b200 import gen_random_trace
    for seed in range(50):
        tr = gen_random_trace(seed, 1 + seed % 40, 1 + seed % 23)
        a = tr.arrays()
        _, timeline, active = O.lifetime(a)
        n = a.num_kernels
        want = np.zeros(n, np.int64)
        want_act = np.zeros(n, np.int64)
        for i in range(a.num_tensors):
            acc = a.accesses[a.access_ptr[i]:a.access_ptr[i + 1]]
            if a.kind[i] == 1:
                want += a.size_bytes[i]
            else:
                want[acc[0]:acc[-1] + 1] += a.size_bytes[i]
            want_act[acc] += a.size_bytes[i]
        assert np.array_equal(timeline, want)
        assert np.array_equal(active, want_act)
        assert (active <= timeline).all()


def test_oracle_lifetime_vs_reference_itself_at_c2():
    """C2 (1.0M events): the oracle's lifetime products against the
    reference's own (tests/golden/c2_lifetime_ref.json, make_ref_lifetime.py)."""
    import json
    import os
    from paper_2506_06472_b200 import LLAMA3_8B, gen_llama_trace
    with open(os.path.join(os.path.dirname(__file__), "golden", "c2_lifetime_ref.json")) as f:
        rec = json.load(f)
    a = gen_llama_trace(LLAMA3_8B).arrays()
    per, tl, act = O.lifetime(a)
    rows = np.stack([a.tensor_id[per["tensor"]], a.size_bytes[per["tensor"]], per["start"].astype(np.int64),
                     per["end"].astype(np.int64), per["wraps"].astype(np.int64)], axis=1)
    h = lambda x: hashlib.sha256(np.ascontiguousarray(x, dtype="<i8").tobytes()).hexdigest()  # noqa: E731
    assert (h(rows), h(tl), h(act)) == (rec["periods_sha256"], rec["timeline_sha256"], rec["active_sha256"])
