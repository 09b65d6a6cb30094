"""bench.py's output contract (the driver parses one JSON line per arm):
the reference arm on the host cores (CPU, runs here) and our arm on cuda:0
(GPU), each with the keys and units the driver and the judge read."""

import json
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _run(args, timeout):
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py")] + args, cwd=ROOT,
                         capture_output=True, text=True, timeout=timeout)
    assert out.returncode == 0, out.stderr[-2000:]
    lines = [l for l in out.stdout.splitlines() if l.strip().startswith("{")]
    assert len(lines) == 1, out.stdout[-2000:]
    return json.loads(lines[0])


def _common(d):
    for k in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step",
              "higher_is_better", "scaling", "vs_baseline", "dtype", "data", "config", "e2e",
              "cpu_baseline"):
        assert k in d, k
    assert d["metric"] == "requests/sec" and d["unit"] == "req/s"
    assert d["higher_is_better"] is True and d["scaling"] == "weak"
    assert d["value"] > 0 and d["ms_per_step"] > 0
    assert "workload" in d["config"]
    e = d["e2e"]
    for k in ("value", "unit", "h2d_bytes_per_step", "d2h_bytes_per_step"):
        assert k in e, k
    assert e["unit"] == d["unit"]


def test_reference_arm_contract():
    """`bench.py --impl reference`: the oracle port on the host cores, same
    metric / unit / config as our arm, e2e = the line's own value."""
    d = _run(["--impl", "reference", "--config", "c2", "--steps", "1", "--warmup", "1"],
             timeout=600)
    _common(d)
    assert d["impl"] == "reference"
    cb = d["cpu_baseline"]
    assert cb["kind"] in ("port", "reference") and cb["cores"] >= 1 and cb["sample"]
    assert cb["value"] == d["value"]
    assert d["e2e"]["value"] == d["value"]
    assert d["e2e"]["h2d_bytes_per_step"] == 0 and d["e2e"]["d2h_bytes_per_step"] == 0


@pytest.mark.gpu
def test_our_arm_contract():
    """Our arm on cuda:0 (C2, short run): roofline, clocks, e2e with host
    copies, launch count of our own kernels."""
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    d = _run(["--config", "c2", "--steps", "3", "--warmup", "3", "--no-cpu-baseline"],
             timeout=600)
    _common(d)
    r = d["roofline"]
    for k in ("bound", "achieved", "peak", "unit", "frac", "traffic"):
        assert k in r, k
    assert r["bound"] in ("hbm", "tensor") and 0 < r["frac"] < 1
    assert abs(r["achieved"] / r["peak"] - r["frac"]) < 1e-6
    assert d["e2e"]["value"] > 0
    assert d["e2e"]["h2d_bytes_per_step"] > 0 and d["e2e"]["d2h_bytes_per_step"] > 0
    assert d["gpu_launches"] > 0
    c = d["clocks"]
    assert "sm_mhz" in c and "reasons" in c
