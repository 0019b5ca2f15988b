"""bench.py keeps the driver contract: one JSON line with the keys the driver and the judge read.

CPU: the reference arm (`--impl reference`, the oracle on a bounded sample) and the `--gpus N`
refusal without N visible GPUs.  GPU: the product arm on the small config 1 (the same code path
as the default R-MAT line, seconds instead of a minute)."""
import json
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
BASE_KEYS = ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better", "scaling",
             "vs_baseline", "dtype", "data", "config", "cpu_baseline", "e2e")


def _run(args, timeout=600):
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py")] + args, capture_output=True, text=True,
                       timeout=timeout, cwd=ROOT)
    return r


def test_reference_arm_line():
    r = _run(["--impl", "reference", "--config", "random1k", "--steps", "2", "--warmup", "1"])
    assert r.returncode == 0, r.stderr[-2000:]
    d = json.loads(r.stdout.strip().splitlines()[-1])
    for k in BASE_KEYS:
        assert k in d, k
    assert d["impl"] == "reference" and d["steps"] == 2 and d["warmup"] == 1 and d["value"] > 0
    assert d["cpu_baseline"]["kind"] == "oracle" and d["cpu_baseline"]["cores"] >= 1
    assert d["e2e"]["h2d_bytes_per_step"] == 0 and d["e2e"]["d2h_bytes_per_step"] == 0
    assert d["config"]["workload"].startswith("random1k_csr_f64")


def test_gpus_n_refused_without_gpus():
    """--gpus N with fewer than N visible GPUs exits 2 with a message (no CPU fallback, no fewer ranks)."""
    import torch
    n = max(2, torch.cuda.device_count() + 1)
    r = _run(["--gpus", str(n), "--steps", "1", "--warmup", "1"], timeout=300)
    assert r.returncode == 2 and f"needs {n} visible GPUs" in (r.stdout + r.stderr)
    if torch.cuda.device_count() == 0:   # and one rank with no GPU at all says so, too
        r = _run(["--steps", "1", "--warmup", "1"], timeout=300)
        assert r.returncode == 2 and "needs CUDA device 0" in (r.stdout + r.stderr)


@pytest.mark.gpu
def test_product_arm_line():
    r = _run(["--config", "random1k", "--steps", "20", "--warmup", "5", "--e2e-steps", "5", "--cpu-seconds", "1"])
    assert r.returncode == 0, r.stderr[-3000:]
    d = json.loads(r.stdout.strip().splitlines()[-1])
    for k in BASE_KEYS + ("roofline", "gpu_launches", "clocks", "per_call_median_ms"):
        assert k in d, k
    assert d["n_gpus"] == 1 and d["steps"] == 20 and d["warmup"] == 5 and d["value"] > 0
    rf = d["roofline"]
    assert rf["bound"] == "hbm" and rf["peak"] > 0 and rf["achieved"] > 0 and rf["kernel"] == "rows_kernel"
    assert abs(rf["frac"] - rf["achieved"] / rf["peak"]) < 1e-9
    assert d["gpu_launches"] >= 20 and d["e2e"]["h2d_bytes_per_step"] > 0 and d["e2e"]["d2h_bytes_per_step"] > 0
    assert d["cpu_baseline"]["kind"] == "oracle" and "sm_mhz" in d["clocks"]
