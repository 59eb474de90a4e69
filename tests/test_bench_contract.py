"""bench.py's JSON line contract (the driver parses it): the reference arm on
the CPU, and our arm on the GPU with a short workload."""
import json
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
BASE_KEYS = {"metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step",
             "higher_is_better", "scaling", "vs_baseline", "dtype", "data", "config", "e2e"}


def _run(args, timeout):
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), *args], cwd=ROOT,
                         capture_output=True, text=True, timeout=timeout)
    assert out.returncode == 0, out.stderr[-3000:]
    lines = [l for l in out.stdout.strip().splitlines() if l.startswith("{")]
    assert len(lines) == 1, out.stdout[-2000:]
    return json.loads(lines[0])


def test_reference_arm_line():
    """--impl reference: the reference's CPU path (dszip from baseline/_ref, or
    the oracle port) timed on the host; one JSON line, e2e equal to value."""
    d = _run(["--impl", "reference", "--steps", "1", "--warmup", "1"], 600)
    assert BASE_KEYS <= set(d)
    assert d["impl"] == "reference" and d["value"] > 0 and d["higher_is_better"] is True
    assert d["e2e"]["value"] == d["value"]
    assert d["e2e"]["h2d_bytes_per_step"] == 0 and d["e2e"]["d2h_bytes_per_step"] == 0
    assert d["cpu_baseline"]["kind"] in ("reference", "port")


@pytest.mark.gpu
def test_our_arm_line():
    """Our arm on a short workload: the base contract keys plus roofline,
    clocks, gpu_launches, the steady-state window and the early window."""
    d = _run(["--steps", "2", "--warmup", "3", "--size", "4000000", "--no-sweep",
              "--no-cpu-baseline", "--e2e-bytes", str(1 << 20), "--skip", "1024"], 900)
    assert BASE_KEYS <= set(d)
    assert {"roofline", "clocks", "gpu_launches"} <= set(d)
    assert d["value"] > 0 and d["n_gpus"] == 1 and d["steps"] == 2 and d["warmup"] == 3
    r = d["roofline"]
    assert {"bound", "achieved", "peak", "unit", "frac", "traffic"} <= set(r)
    assert 0 < r["frac"] < 1.5
    e = d["e2e"]
    assert e["value"] > 0 and e["h2d_bytes_per_step"] > 0 and e["d2h_bytes_per_step"] > 0
    assert d["gpu_launches"] > 0
    c = d["config"]
    assert c["timed_after_timesteps"] >= 1024 and c["early_window_value"] > 0
