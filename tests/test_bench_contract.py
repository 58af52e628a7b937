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
    d = _run(["--config", "llama1", "--secondary", "c1", "--host-leg", "", "--steps", "3", "--warmup", "3",
              "--no-migration"])
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


@pytest.mark.gpu
def test_two_rank_line_on_one_gpu():
    """The N > 1 path (torchrun, one process per rank, sharded planner over
    CUDA-IPC mailboxes, device-resident sharded lifetime) with both ranks on
    cuda:0 (TIO_BENCH_ONE_GPU: gloo instead of NCCL): strong scaling of ONE
    trace, every rank's plan equal to the reference's llama1 plan."""
    import gzip
    import socket
    sk = socket.socket()
    sk.bind(("127.0.0.1", 0))
    port = sk.getsockname()[1]
    sk.close()
    env = dict(os.environ, TIO_BENCH_ONE_GPU="1")
    out = subprocess.run([sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2",
                          "--master-addr", "127.0.0.1", "--master-port", str(port), os.path.join(ROOT, "bench.py"),
                          "--gpus", "2", "--steps", "2", "--warmup", "3", "--config", "llama1", "--secondary", "c1",
                          "--host-leg", "", "--no-migration"], capture_output=True, text=True, timeout=900, cwd=ROOT,
                         env=env)
    assert out.returncode == 0, out.stderr[-3000:]
    lines = [ln for ln in out.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1, out.stdout
    d = json.loads(lines[0])
    assert BASE_KEYS <= set(d) and d["n_gpus"] == 2 and d["scaling"] == "strong"
    with gzip.open(os.path.join(ROOT, "tests", "golden", "llama1.json.gz"), "rt") as f:
        rec = json.load(f)
    rec = rec[0] if isinstance(rec, list) else rec
    assert d["config"]["plan_sha256"] == rec["plan_sha256"]
    assert d["config"]["plan_sha256_equal_on_all_ranks"] is True
    assert d["sharded_lifetime"]["bit_exact_vs_unsharded"] is True


@pytest.mark.gpu
def test_two_rank_data_parallel_offload_leg_on_one_gpu():
    """Configs C5 path (bench.py --c5): two data-parallel ranks (gradient
    all-reduce inside the step), each profiling, planning and running its own
    online engine; here both ranks share cuda:0 (TIO_BENCH_ONE_GPU, gloo) on
    the small model: identical plans, zero byte mismatches, a step-time ratio."""
    import socket
    sk = socket.socket()
    sk.bind(("127.0.0.1", 0))
    port = sk.getsockname()[1]
    sk.close()
    env = dict(os.environ, TIO_BENCH_ONE_GPU="1")
    out = subprocess.run([sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2",
                          "--master-addr", "127.0.0.1", "--master-port", str(port), os.path.join(ROOT, "bench.py"),
                          "--gpus", "2", "--steps", "2", "--warmup", "3", "--config", "c1", "--secondary", "",
                          "--host-leg", "", "--no-migration", "--c5", "--c5-fracs", "0.8", "--offload-model", "tiny"],
                         capture_output=True, text=True, timeout=1200, cwd=ROOT, env=env)
    assert out.returncode == 0, out.stderr[-3000:]
    d = json.loads([ln for ln in out.stdout.splitlines() if ln.startswith("{")][-1])
    c5 = d["migration_dp"]
    assert c5["ranks"] == 2 and c5["plans_identical"]
    r = c5["runs"][0]
    assert r["verify_mismatches"] == 0 and r["step_vs_ideal"] > 0
