"""bench.py keeps the driver's JSON-line contract: the reference arm here on the CPU, the
B200 arm (short run) on the GPU."""
import json
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _run(*args, timeout=600):
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), *args], cwd=ROOT,
                         capture_output=True, text=True, timeout=timeout)
    assert out.returncode == 0, out.stderr[-2000:]
    lines = [l for l in out.stdout.strip().splitlines() if l.startswith("{")]
    assert len(lines) == 1, out.stdout[-2000:]
    return json.loads(lines[0])


BASE_KEYS = {"metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step",
             "higher_is_better", "scaling", "vs_baseline", "dtype", "data", "config", "e2e"}


def _check_common(d):
    assert BASE_KEYS <= set(d), BASE_KEYS - set(d)
    assert d["metric"].startswith("e-prop train samples")
    assert d["unit"] == "samples*timesteps/s" and d["higher_is_better"] is True
    assert d["value"] > 0 and d["scaling"] in ("weak", "strong") and d["data"] == "synthetic"
    assert {"workload", "seq_len", "n_hidden", "n_inputs", "n_classes"} <= set(d["config"])
    e = d["e2e"]
    assert {"value", "unit", "h2d_bytes_per_step", "d2h_bytes_per_step"} <= set(e)
    assert e["unit"] == d["unit"] and e["value"] > 0


def test_reference_arm_contract():
    d = _run("--impl", "reference", "--config", "c2", "--steps", "1", "--warmup", "0")
    _check_common(d)
    assert d["impl"] == "reference"
    cb = d["cpu_baseline"]
    sys.path.insert(0, ROOT)
    from oracle.cpu_bench import reference_available
    # the reference's own engine when baseline/_ref holds it, else the labelled port
    assert cb["kind"] == ("reference" if reference_available() else "port")
    assert cb["cores"] >= 1 and cb["value"] == d["value"] and cb["cpu_model"]
    assert d["e2e"]["h2d_bytes_per_step"] == 0 and d["e2e"]["d2h_bytes_per_step"] == 0
    assert d["scaling"] == "weak"


def test_reference_arm_strong_scaling_config():
    """--global-batch: the fixed global batch of north_star's C4 curve (1024 split over
    the ranks); the config keys are the ones the B200 arm prints."""
    d = _run("--impl", "reference", "--config", "c4", "--global-batch", "1024",
             "--steps", "1", "--warmup", "0")
    _check_common(d)
    assert d["scaling"] == "strong"
    c = d["config"]
    assert c["global_batch"] == 1024 and c["batch_per_gpu"] == 1024 and c["n_hidden"] == 2048
    assert set(c) == {"workload", "batch_per_gpu", "global_batch", "seq_len", "n_hidden",
                      "n_inputs", "n_classes", "chunk", "parallelism"}


@pytest.mark.gpu
def test_gpu_arm_contract():
    d = _run("--config", "c2", "--steps", "4", "--warmup", "3", "--no-cpu")
    _check_common(d)
    assert "impl" not in d or d["impl"] != "reference"
    assert d["n_gpus"] == 1 and d["steps"] == 4 and d["warmup"] == 3
    assert d["gpu_launches"] > 0
    r = d["roofline"]
    assert {"bound", "achieved", "peak", "unit", "frac", "traffic"} <= set(r)
    assert r["bound"] in ("hbm", "tensor") and 0 < r["frac"] < 2
    assert d["e2e"]["h2d_bytes_per_step"] > 0 and d["e2e"]["d2h_bytes_per_step"] > 0
    c = d["clocks"]
    assert {"sm_mhz", "sm_max_mhz", "reasons"} <= set(c)
    assert set(d["config"]) == {"workload", "batch_per_gpu", "global_batch", "seq_len",
                                "n_hidden", "n_inputs", "n_classes", "chunk", "parallelism"}
    p = d["parity"]
    assert p["checked"] and p["pass"] and p["spike_flips"] == 0
    dp = d["e2e_dropin"]
    assert dp["value"] > 0 and dp["packed"]["value"] > 0
