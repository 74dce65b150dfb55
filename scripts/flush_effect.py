"""How the L2 flush between timed steps affects K1's event-timed step, per config.

    python scripts/flush_effect.py c2 c3 c4

Flush variants ahead of the start event (never inside the timed interval):
  write  — fill a 256 MiB buffer (bench.py's flush): L2 is left holding up to ~126 MB of
           DIRTY flush lines, which K1's first output stores must write back to HBM;
  write+read — the same fill, then a sum over a second 256 MiB buffer: the input is
           evicted all the same, and L2 starts the step clean;
  none   — back-to-back graph replays (L2 holds the previous step's dirty tail).
Graph replay of the one K1 launch, CUDA events, median of 9.
"""
import json
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_1707_08213_b200.tree2d import _OUT_DTYPES, _precision_code, forward_into  # noqa: E402
from paper_1707_08213_b200.workloads import CONFIGS  # noqa: E402


def main():
    dev = torch.device("cuda", 0)
    a = torch.empty(64 << 20, dtype=torch.float32, device=dev)
    b = torch.ones(64 << 20, dtype=torch.float32, device=dev)
    for name in sys.argv[1:] or ["c2"]:
        c = CONFIGS[name]
        prec = _precision_code(c.precision, None)
        x = torch.from_numpy(c.generate()).to(dev)
        out = torch.empty((c.P0, c.P1, c.n0, c.n1), dtype=_OUT_DTYPES[prec], device=dev)
        st = torch.cuda.current_stream(dev)
        for _ in range(3):
            forward_into(x, c.m0, c.m1, out, prec=prec)
        g = torch.cuda.CUDAGraph()
        cap = torch.cuda.Stream(dev)
        cap.wait_stream(st)
        with torch.cuda.graph(g, stream=cap):
            forward_into(x, c.m0, c.m1, out, prec=prec, stream=cap)
        st.wait_stream(cap)
        res = {"config": name}
        for mode in ("write", "write+read", "none"):
            ts = []
            for _ in range(9):
                torch.cuda.synchronize()
                if mode != "none":
                    a.fill_(1.0)
                if mode == "write+read":
                    b.sum()
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record()
                g.replay()
                e1.record()
                torch.cuda.synchronize()
                ts.append(e0.elapsed_time(e1))
            t = statistics.median(ts)
            res[mode] = {"ms": t, "write_tbs": out.numel() * out.element_size() / t / 1e9}
        print(json.dumps(res), flush=True)
        del g, x, out
        torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
