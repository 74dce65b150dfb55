"""SWDF container / transform throughput on the GPU box: write_swdf of a device
coefficient array (widen to complex128 on device, pinned double buffer, D2H overlapped
with the file write) and transform_file end to end (SWDF input -> GPU tree -> SWDF out),
against the numpy write of the same array.  Files go to a scratch directory and are
removed; rates are file bytes per second (page cache included)."""
import json
import os
import sys
import tempfile
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_1707_08213_b200 import WindowSpec, container, tree_swdft_2d  # noqa: E402
from paper_1707_08213_b200.workloads import CONFIGS  # noqa: E402

cfg = CONFIGS["c2"]
x = cfg.generate()
root = sys.argv[1] if len(sys.argv) > 1 else None
d = tempfile.mkdtemp(prefix="swdf_bench_", dir=root)
try:
    res = tree_swdft_2d(x, WindowSpec((cfg.m0, cfg.m1)), precision="fp64", budget=1 << 40)
    torch.cuda.synchronize()
    nbytes = res.values.numel() * 16
    out = os.path.join(d, "c.swdf")
    container.write_swdf(out, res.values)  # warm
    os.remove(out)  # every timed write goes to a fresh file (truncating an existing 1 GB
    # file inside the timed region cost ~40 % on an ext4/overlay /tmp)
    t0 = time.perf_counter()
    container.write_swdf(out, res.values)
    t_dev = time.perf_counter() - t0
    host = res.values.cpu().numpy()
    os.remove(out)
    t0 = time.perf_counter()
    container.write_swdf(out, host)
    t_np = time.perf_counter() - t0
    inp = os.path.join(d, "x.swdf")
    container.write_swdf(inp, x.astype(np.float64))
    container.transform_file(inp, out, (cfg.n0, cfg.n1), budget=1 << 40)  # warm
    os.remove(out)
    t0 = time.perf_counter()
    container.transform_file(inp, out, (cfg.n0, cfg.n1), budget=1 << 40)
    t_tr = time.perf_counter() - t0
    raw = np.ones(nbytes // 8)
    t0 = time.perf_counter()
    with open(os.path.join(d, "raw.bin"), "wb") as f:  # the file system's own ceiling
        f.write(memoryview(raw).cast("B"))
    t_raw = time.perf_counter() - t0
    print(json.dumps({"config": cfg.name, "dir": d, "file_bytes": nbytes,
                      "plain_write_GBps": nbytes / t_raw / 1e9,
                      "write_swdf_device_GBps": nbytes / t_dev / 1e9,
                      "write_swdf_numpy_host_GBps": nbytes / t_np / 1e9,
                      "transform_file_s": t_tr, "transform_file_GBps": nbytes / t_tr / 1e9}))
finally:
    for f in os.listdir(d):
        os.remove(os.path.join(d, f))
    os.rmdir(d)
