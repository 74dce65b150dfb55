"""bench.py's one-JSON-line contract: the keys the driver reads, on both arms.

The reference arm (the oracle port on the host cores) needs no GPU; the product arm runs
config 2 (0.5 GB of output) with every leg on: device-timed value, roofline, e2e through
swdft2d_forward_host with host buffers, the fresh-output call, the CPU baseline.
"""
import json
import os
import subprocess
import sys

import pytest

from conftest import ROOT

BASE_KEYS = {"metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step",
             "higher_is_better", "scaling", "vs_baseline", "dtype", "data", "config"}


def run_bench(*args, timeout=900):
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), *args],
                       capture_output=True, text=True, timeout=timeout, cwd=ROOT)
    lines = [l for l in r.stdout.splitlines() if l.startswith("{")]
    assert r.returncode == 0 and len(lines) == 1, r.stdout[-2000:] + r.stderr[-2000:]
    return json.loads(lines[0])


def test_reference_arm_line():
    d = run_bench("--impl", "reference", "--config", "c1", "--steps", "2", "--warmup", "1")
    assert BASE_KEYS <= set(d) and d["impl"] == "reference"
    assert d["unit"] == "coef/s" and d["higher_is_better"] is True and d["value"] > 0
    assert d["steps"] == 2 and d["warmup"] == 1 and d["config"]["workload"] == "c1"
    cb = d["cpu_baseline"]
    assert cb["kind"] == "port" and cb["cores"] >= 1 and cb["value"] == d["value"] and cb["sample"]
    assert d["e2e"] == {"value": d["value"], "unit": d["unit"], "h2d_bytes_per_step": 0,
                        "d2h_bytes_per_step": 0}


@pytest.mark.gpu
def test_product_arm_line():
    d = run_bench("--config", "c2", "--steps", "4", "--warmup", "3", "--no-others")
    assert BASE_KEYS <= set(d) and "impl" not in d or d.get("impl") == "ours"
    assert d["n_gpus"] == 1 and d["steps"] == 4 and d["warmup"] == 3
    assert d["unit"] == "coef/s" and d["dtype"] == "f32" and d["vs_baseline"] is None
    assert d["config"]["workload"] == "c2" and "model" not in d["config"]
    assert d["gpu_launches"] == 4
    assert abs(d["value"] - 63234304 / (d["ms_per_step"] / 1e3)) / d["value"] < 1e-6
    rf = d["roofline"]
    assert rf["bound"] == "hbm" and rf["unit"] == "GB/s" and rf["peak"] > 1000
    assert abs(rf["frac"] - rf["achieved"] / rf["peak"]) < 1e-9
    assert abs(rf["achieved"] - 506923008 / (d["ms_per_step"] / 1e3) / 1e9) / rf["achieved"] < 1e-6
    assert 0.5 < rf["achieved"] / 1e3 < 8.0                      # TB/s, a B200
    cb = d["cpu_baseline"]
    assert cb["kind"] == "port" and cb["cores"] >= 1 and cb["value"] > 0 and "c2" in cb["sample"]
    e = d["e2e"]
    assert e["unit"] == "coef/s" and 0 < e["value"] < d["value"]
    assert e["h2d_bytes_per_step"] == 512 * 512 * 4
    assert e["d2h_bytes_per_step"] == 63234304 * 8
    assert "swdft2d_forward_host" in e["path"]
    assert e["fresh_output"]["value"] > 0 and e["resident"]["value"] > e["value"]
    ck = d["clocks"]
    assert ck["sm_max_mhz"] >= ck["sm_mhz"] > 0 and isinstance(ck["reasons"], list)
