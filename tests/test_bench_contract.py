"""bench.py's driver contract on the CPU: the reference arm prints one JSON line with the
required keys, and the GPU arm fails loudly (no CPU fallback) when there is no GPU."""

import json
import os
import subprocess
import sys

import pytest
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _run(*args, timeout=600):
    return subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), *args], cwd=ROOT, capture_output=True,
                          text=True, timeout=timeout)


def test_reference_arm_json_line():
    r = _run("--impl", "reference", "--steps", "1", "--warmup", "0")
    assert r.returncode == 0, r.stderr[-2000:]
    lines = [ln for ln in r.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1
    d = json.loads(lines[0])
    for k in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better", "scaling",
              "vs_baseline", "dtype", "data", "config", "impl", "cpu_baseline", "e2e"):
        assert k in d, k
    assert d["impl"] == "reference" and d["value"] > 0 and d["higher_is_better"] is True
    assert d["config"]["workload"] == "alexnet_b256_synthetic_227"
    cb = d["cpu_baseline"]
    assert cb["kind"] in ("port", "reference") and cb["cores"] >= 1 and cb["value"] == d["value"] and cb["sample"]
    assert d["e2e"] == {"value": d["value"], "unit": d["unit"], "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}


@pytest.mark.skipif(torch.cuda.is_available(), reason="checks the no-GPU behaviour")
def test_gpu_arm_refuses_without_a_gpu():
    r = _run("--steps", "1", "--warmup", "1", timeout=300)
    assert not any(ln.startswith("{") and '"value"' in ln for ln in r.stdout.splitlines()), \
        "the GPU arm must not print a number without a GPU"
    assert r.returncode != 0


def test_reference_arm_times_the_reference_engine_for_configs0():
    """configs[0] (LeNet, 2 ranks): the reference arm measures full steps and the reference's
    own PipelinedRank exchange (baseline/_ref) beside the C port — no extrapolated samples."""
    if not os.path.isdir(os.path.join(ROOT, "baseline", "_ref", "pipesgd")):
        pytest.skip("reference not installed in baseline/_ref")
    r = _run("--impl", "reference", "--workload", "lenet", "--gpus", "2", "--steps", "2", "--warmup", "1")
    assert r.returncode == 0, r.stderr[-2000:]
    d = json.loads([ln for ln in r.stdout.splitlines() if ln.startswith("{")][-1])
    cb = d["cpu_baseline"]
    assert d["n_gpus"] == 2 and cb["steps_measured"] == 2
    assert d["config"]["workload"] == "lenet5_b64_synthetic_28" and d["config"]["global_batch"] == 64
    ref = cb["reference_engine_exchange"]
    assert ref["ms"] > 0 and ref["iterations"] == 2
    assert abs(d["ms_per_step"] - (1e3 * 64 / d["value"])) < 1e-6 * d["ms_per_step"]
