"""GPU: bench.py's JSON line keeps the driver's contract (keys, types, consistency), on the
small C1 config so the run takes seconds: metric / value / unit, steps / warmup (>= 3),
roofline with achieved / peak / frac, cpu_baseline from the oracle, e2e with the copied bytes,
clocks sampled during the timed region, gpu_launches, and the sampled parity within tolerance.
The reference arm prints its own line with impl = reference."""
import json
import subprocess
import sys

import pytest

from fmm_testutil import ROOT

pytestmark = pytest.mark.gpu


def run(*args):
    r = subprocess.run([sys.executable, str(ROOT / "bench.py"), *args], capture_output=True,
                       text=True, cwd=str(ROOT), timeout=600)
    assert r.returncode == 0, r.stderr[-2000:]
    lines = [l for l in r.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1, r.stdout
    return json.loads(lines[0])


def test_fmm_line():
    d = run("--config", "C1", "--steps", "3", "--warmup", "1", "--cpu-seconds", "1")
    for k in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step",
              "higher_is_better", "scaling", "vs_baseline", "dtype", "data", "config", "roofline",
              "cpu_baseline", "e2e", "clocks", "gpu_launches", "parity"):
        assert k in d, k
    assert d["n_gpus"] == 1 and d["steps"] == 3 and d["warmup"] >= 3 and d["dtype"] == "f64"
    assert d["value"] > 0 and abs(d["value"] - 2 * 512 ** 3 / (d["ms_per_step"] * 1e-3) / 1e9) < 1e-6 * d["value"]
    rf = d["roofline"]
    assert rf["bound"] == "tensor" and 0 < rf["frac"] <= 1.0 and abs(rf["frac"] - rf["achieved"] / rf["peak"]) < 1e-9
    assert d["cpu_baseline"]["kind"] == "oracle" and d["cpu_baseline"]["cores"] >= 1
    e = d["e2e"]
    assert e["h2d_bytes_per_step"] == 2 * 512 * 512 * 8 and e["d2h_bytes_per_step"] == 512 * 512 * 8
    assert d["clocks"] is not None and d["clocks"]["samples"] >= 1
    assert d["gpu_launches"] > 0
    assert d["parity"]["pass"] and d["parity"]["value"] <= 1e-13
    assert "C1" in d["config"]["workload"]


def test_reference_line():
    d = run("--impl", "reference", "--config", "C1", "--steps", "1", "--warmup", "0")
    assert d["impl"] == "reference" and d["value"] > 0
    assert d["e2e"]["h2d_bytes_per_step"] == 0 and d["cpu_baseline"]["kind"] == "oracle"
