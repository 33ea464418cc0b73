"""bench.py's JSON line keeps the driver's contract (run on the GPU box): one line on stdout with
the required keys and types, a roofline object for the dominant kernel, clocks sampled during
the timed region, the e2e object with the copied bytes, and a positive launch count."""
import json
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _run(*args):
    r = subprocess.run([sys.executable, "bench.py", *args], cwd=ROOT, capture_output=True, text=True, timeout=900)
    assert r.returncode == 0, r.stderr[-3000:]
    lines = [l for l in r.stdout.splitlines() if l.strip().startswith("{")]
    assert len(lines) == 1, r.stdout
    return json.loads(lines[0])


def test_default_bench_line():
    d = _run("--steps", "3", "--warmup", "3")
    for k, t in (("metric", str), ("value", float), ("unit", str), ("n_gpus", int), ("steps", int), ("warmup", int),
                 ("ms_per_step", float), ("higher_is_better", bool), ("scaling", str), ("dtype", str),
                 ("data", str), ("config", dict), ("roofline", dict), ("clocks", dict), ("e2e", dict),
                 ("gpu_launches", int)):
        assert isinstance(d[k], t), (k, d.get(k))
    assert d["n_gpus"] == 1 and d["steps"] == 3 and d["warmup"] == 3 and d["value"] > 0
    assert d["scaling"] == "weak" and d["vs_baseline"] is None and d["dtype"] == "f64"
    assert "configs[3]" in d["config"]["workload"] and d["config"]["global"] == [512, 512, 512]
    r = d["roofline"]
    assert r["bound"] == "alu" and r["unit"] == "TFLOP/s" and 0 < r["frac"] < 1
    assert abs(r["frac"] - r["achieved"] / r["peak"]) < 1e-9
    assert [st["stage"] for st in r["per_stage"]] == [1, 2] and all(st["launches"] == 3 for st in r["per_stage"])
    if r["ncu"]:  # a committed capture of this workload: per-launch dram bytes, averaged over the stages
        assert r["traffic"] > 0
    c = d["clocks"]
    assert c["samples"] > 0 and c["sm_mhz"] > 0 and isinstance(c["reasons"], list)
    e = d["e2e"]
    assert e["value"] > 0 and e["h2d_bytes_per_step"] > 0 and e["d2h_bytes_per_step"] > 0
    assert d["gpu_launches"] == 3 * 4  # per step: k_dt, the dt store, two k_stage launches
    cb = d["cpu_baseline"]
    assert cb["kind"] == "oracle" and cb["value"] > 0 and cb["per_core_value"] > 0 and cb["cores"] >= 1


def test_strong_and_roofline_configs():
    d = _run("--steps", "2", "--warmup", "3", "--no-cpu", "--no-e2e", "--workload", "ot3d", "--n", "256")
    assert "configs[2]" in d["config"]["workload"] and d["value"] > 0


def test_scheme_bench_lines():
    for scheme, per_step in (("wenoz-rk3", 2 + 3 * 5), ("ct-plm-rk2", 2 + 2 * 5)):
        d = _run("--steps", "2", "--warmup", "3", "--no-cpu", "--no-e2e", "--scheme", scheme)
        assert d["value"] > 0 and d["gpu_launches"] == 2 * per_step, (scheme, d["gpu_launches"])
