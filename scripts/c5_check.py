"""Config-5 K1 launch timed three ways on one process: CUDA events around a direct launch,
around a CUDA-graph replay, and host wall clock with a synchronize (cross-check of the
one-shot grid's bench number against ncu's serialized duration)."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_1707_08213_b200.tree2d import _OUT_DTYPES, forward_into  # noqa: E402
from paper_1707_08213_b200.workloads import CONFIGS  # noqa: E402

cfg = CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "c5"]
dev = torch.device("cuda", 0)
s = torch.cuda.current_stream(dev)
x = torch.from_numpy(cfg.generate()).to(dev)
out = torch.empty((cfg.P0, cfg.P1, cfg.n0, cfg.n1), dtype=_OUT_DTYPES[0], device=dev)
call = lambda st: forward_into(x, cfg.m0, cfg.m1, out, prec=0, stream=st)  # noqa: E731
call(s)
torch.cuda.synchronize()
for rep in range(3):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    e0.record(s)
    call(s)
    e1.record(s)
    torch.cuda.synchronize()
    wall = time.perf_counter() - t0
    print(f"{cfg.name} direct: events {e0.elapsed_time(e1):.3f} ms, wall {wall * 1e3:.3f} ms", flush=True)
