"""bench.py keeps the driver's JSON-line contract: the reference arm on CPU
(the oracle port, config C1) and our arm on the GPU (small configs, no
migration leg)."""

from __future__ import annotations

import json
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
BASE_KEYS = {"metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better",
             "scaling", "vs_baseline", "dtype", "data", "config"}


def _run(args, timeout=600):
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), *args], capture_output=True, text=True,
                         timeout=timeout, cwd=ROOT)
    assert out.returncode == 0, out.stderr[-2000:]
    lines = [ln for ln in out.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1, out.stdout
    return json.loads(lines[0])


def test_reference_arm_line_on_cpu():
    d = _run(["--impl", "reference", "--config", "c1", "--steps", "1", "--warmup", "0"])
    assert BASE_KEYS <= set(d)
    assert d["impl"] == "reference" and d["value"] > 0 and d["higher_is_better"] is True
    assert d["cpu_baseline"]["kind"] == "port" and d["cpu_baseline"]["cores"] >= 1
    assert d["e2e"]["h2d_bytes_per_step"] == 0 and d["e2e"]["value"] == d["value"]


@pytest.mark.gpu
def test_our_arm_line_on_gpu():
    d = _run(["--config", "llama1", "--secondary", "c1", "--steps", "3", "--warmup", "3", "--no-migration"])
    assert BASE_KEYS <= set(d)
    assert d["value"] > 0 and d["n_gpus"] == 1 and d["dtype"] == "int64"
    r = d["roofline"]
    assert r["bound"] == "hbm" and r["unit"] == "GB/s" and 0 < r["frac"] == pytest.approx(r["achieved"] / r["peak"])
    assert d["e2e"]["h2d_bytes_per_step"] > 0 and d["e2e"]["d2h_bytes_per_step"] > 0
    assert d["gpu_launches"] > 0 and d["clocks"]["samples"] >= 0
    assert d["cpu_baseline"]["kind"] == "port"
    assert d["c1"]["value"] > 0 and d["c1"]["cpu_baseline"]["value"] > 0
    # the 1-microbatch Llama plan is the reference's (tests/golden/llama1.json.gz,
    # recorded from the reference planner with capacity = peak // 2, SSD 16,000 B/us)
    import gzip
    import hashlib
    with gzip.open(os.path.join(ROOT, "tests", "golden", "llama1.json.gz"), "rt") as f:
        rec = json.load(f)[0]
    if rec.get("capacity") == d["config"]["capacity"]:
        assert d["config"]["plan_sha256"] == hashlib.sha256(rec["plan"].encode()).hexdigest()
