"""The bench.py contract on the GPU: one JSON line with the driver's keys, a roofline object
for the dominant kernel, the oracle baseline, the end-to-end (host buffers) number, sampled
clocks and a positive launch count; and the reference arm's line.  Short runs (a few steps)
so the whole file stays within a minute."""
import json
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def run(*args, timeout=600):
    r = subprocess.run([sys.executable, "bench.py", *args], cwd=ROOT, capture_output=True,
                       text=True, timeout=timeout)
    assert r.returncode == 0, r.stderr[-2000:]
    lines = [ln for ln in r.stdout.splitlines() if ln.strip().startswith("{")]
    assert len(lines) == 1, r.stdout
    return json.loads(lines[0])


def test_bench_line_contract():
    d = run("--steps", "5", "--warmup", "3", "--cpu-seconds", "1", "--e2e-steps", "2")
    for k in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step",
              "higher_is_better", "scaling", "vs_baseline", "dtype", "data", "config", "roofline",
              "cpu_baseline", "e2e", "gpu_launches", "clocks"):
        assert k in d, k
    assert d["n_gpus"] == 1 and d["steps"] == 5 and d["warmup"] == 3 and d["value"] > 0
    assert d["config"]["workload"].startswith("C2")
    r = d["roofline"]
    assert r["bound"] in ("hbm", "tensor", "alu") and 0 < r["frac"] <= 1.05
    assert abs(r["frac"] - r["achieved"] / r["peak"]) < 1e-6
    assert d["cpu_baseline"]["kind"] == "oracle" and d["cpu_baseline"]["cores"] >= 1
    e = d["e2e"]
    assert e["value"] > 0 and e["h2d_bytes_per_step"] > 0 and e["d2h_bytes_per_step"] > 0
    assert d["gpu_launches"] >= d["steps"]
    assert d["clocks"]["sm_max_mhz"] > 0
    assert d["parity"]["pass"]
    assert d["ms_per_step_min"] <= d["ms_per_step_median"] and len(d["inputs_sha256"]) == 64
    assert d["roofline"]["same_run_copy_gbs"] > 0


def test_bench_reference_arm():
    d = run("--impl", "reference", "--steps", "1", "--warmup", "3")
    assert d["impl"] == "reference" and d["value"] > 0
    assert d["cpu_baseline"]["kind"] == "oracle"
    assert d["e2e"]["h2d_bytes_per_step"] == 0


@pytest.mark.parametrize("wl", ["C3", "KNN", "SHF"])
def test_bench_other_workloads(wl):
    d = run("--workload", wl, "--steps", "3", "--warmup", "3", "--no-e2e", "--no-cpu-baseline")
    assert d["value"] > 0 and d["parity"]["pass"] and d["gpu_launches"] > 0
    assert d["roofline"]["bound"] in (("alu",) if wl == "SHF" else ("hbm", "tensor"))
