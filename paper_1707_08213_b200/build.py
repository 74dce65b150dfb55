"""Build libswdft2d.so in-tree for sm_100a (nvcc, no torch extension machinery).

    python -m paper_1707_08213_b200.build [-v]

Objects go to paper_1707_08213_b200/_build/, the library to
paper_1707_08213_b200/libswdft2d.so (git-ignored; it travels to the GPU box
with the gpurun snapshot).  cudart is linked statically; the library talks to
whatever CUDA context is current on the calling thread (torch's).
"""
from __future__ import annotations

import argparse
import concurrent.futures as cf
import os
import subprocess
import sys

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
BUILD = os.path.join(PKG, "_build")
LIB = os.path.join(PKG, "libswdft2d.so")
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
K1_MAX_M = 6   # K1 windows up to 64 x 64; k1_m0_7 adds 128-row windows of n1 <= 16 (fp32)

ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
CFLAGS = ARCH + ["-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC,-O2",
                 "-I", os.path.join(ROOT, "include"), "-I", CSRC]


def _units():
    units = [("abi.cu", [], "abi.o"), ("k0_window.cu", [], "k0_window.o"), ("k2_push.cu", [], "k2_push.o"),
             ("kr_rows.cu", [], "kr_rows.o"), ("kc_cols.cu", [], "kc_cols.o"),
             ("host_pipe.cu", [], "host_pipe.o")]
    for m0 in range(K1_MAX_M + 4):
        units.append(("k1_inst.cu", [f"-DK1_M0={m0}"], f"k1_m0_{m0}.o"))
    return units


def _deps():
    return [os.path.join(CSRC, f) for f in os.listdir(CSRC)] + [
        os.path.join(ROOT, "include", "swdft2d.h"), os.path.abspath(__file__)]


def _stale(target: str, deps) -> bool:
    if not os.path.exists(target):
        return True
    t = os.path.getmtime(target)
    return any(os.path.getmtime(d) > t for d in deps)


def _compile(src: str, defs, obj: str, verbose: bool) -> str:
    # ptxas -v always: its per-kernel register / stack-frame lines are kept next to the
    # object (_build/<obj>.ptxas) for tests/test_host.py's local-memory check
    cmd = [NVCC] + CFLAGS + defs + ["-Xptxas", "-v"] + [
        "-c", os.path.join(CSRC, src), "-o", os.path.join(BUILD, obj)]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError(f"nvcc failed for {src} {defs}:\n{r.stdout}\n{r.stderr}")
    with open(os.path.join(BUILD, obj + ".ptxas"), "w") as f:
        f.write(r.stderr)
    return r.stderr if verbose else ""


def kernel_resources(build_dir: str = BUILD) -> dict:
    """{mangled kernel: (registers, stack_frame_bytes, spill_store_bytes)} from the
    ptxas -v logs of the last build (empty if there are none)."""
    import glob
    import re
    res = {}
    for log in glob.glob(os.path.join(build_dir, "*.ptxas")):
        fn = None
        stack = spill = 0
        for line in open(log):
            m = re.search(r"Compiling entry function '([^']+)'", line)
            if m:
                fn = m.group(1)
                continue
            m = re.search(r"(\d+) bytes stack frame, (\d+) bytes spill stores", line)
            if m and fn:
                stack, spill = int(m.group(1)), int(m.group(2))
                continue
            m = re.search(r"Used (\d+) registers", line)
            if m and fn:
                res[fn] = (int(m.group(1)), stack, spill)
                fn = None
    return res


def build(force: bool = False, verbose: bool = False, jobs: int | None = None) -> str:
    os.makedirs(BUILD, exist_ok=True)
    deps = _deps()
    units = _units()
    todo = [u for u in units if force or _stale(os.path.join(BUILD, u[2]), deps)]
    if todo:
        jobs = jobs or min(len(todo), os.cpu_count() or 4)
        with cf.ThreadPoolExecutor(jobs) as ex:
            logs = list(ex.map(lambda u: _compile(u[0], u[1], u[2], verbose), todo))
        if verbose:
            for log in logs:
                sys.stderr.write(log)
    objs = [os.path.join(BUILD, u[2]) for u in units]
    if force or todo or _stale(LIB, objs):
        tmp = LIB + ".tmp"
        cmd = [NVCC] + ARCH + ["-shared", "-cudart", "static", "-Xlinker",
               "--version-script=" + os.path.join(CSRC, "exports.map"), "-o", tmp] + objs
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            raise RuntimeError(f"link failed:\n{r.stdout}\n{r.stderr}")
        os.replace(tmp, LIB)
    return LIB


if __name__ == "__main__":
    ap = argparse.ArgumentParser()
    ap.add_argument("-f", "--force", action="store_true")
    ap.add_argument("-v", "--verbose", action="store_true")
    a = ap.parse_args()
    print(build(force=a.force, verbose=a.verbose))
