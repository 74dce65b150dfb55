"""Randomised parity (scripts/fuzz_parity.py): windows 1..1024, every input dtype, padded
row strides, window-row sub-ranges and normalizations; fp64 bitwise against the C oracle,
fp32 within BASELINE's window-relative 1e-4.  A short fixed-seed run here; the round's
long runs are in profiles/fuzz_parity_r01.jsonl."""
import json
import os
import subprocess
import sys

import pytest

from conftest import ROOT


@pytest.mark.gpu
@pytest.mark.parametrize("seed", [11, 12])
def test_fuzz_parity(seed):
    r = subprocess.run([sys.executable, os.path.join(ROOT, "scripts", "fuzz_parity.py"),
                        "--cases", "60", "--seed", str(seed)],
                       capture_output=True, text=True, timeout=600)
    lines = [l for l in r.stdout.splitlines() if l.startswith("{")]
    assert lines, r.stdout + r.stderr
    summary = json.loads(lines[-1])
    assert r.returncode == 0 and summary["fails"] == 0, "\n".join(lines)


@pytest.mark.gpu
@pytest.mark.parametrize("args", [("--seed", "21"), ("--seed", "22", "--exp", "6.5", "7.5")])
def test_fuzz_host_entry(args):
    """scripts/fuzz_host.py: swdft2d_forward_host / swdft2d_download against the device
    path on random shapes, strips, destinations and staging settings (a short run; the
    second one sized so that pageable outputs go through the staging workers)."""
    r = subprocess.run([sys.executable, os.path.join(ROOT, "scripts", "fuzz_host.py"),
                        "--cases", "60", *args], capture_output=True, text=True, timeout=600)
    lines = [l for l in r.stdout.splitlines() if l.startswith("{")]
    assert lines, r.stdout + r.stderr
    summary = json.loads(lines[-1])
    assert r.returncode == 0 and summary["fails"] == 0, "\n".join(lines)
