"""Why config 2's event-timed step moves between 0.086 and 0.107 ms from box to box.

    python scripts/c2_timing_probe.py [c2 ...]

Every sample of four timing arrangements (graph replay of the one K1 launch, CUDA events):
  bench   — bench.py's: synchronize, L2 flush (write 256 MiB + read 256 MiB), events;
  sleep   — the same with a ~0.3 ms device-side spin queued between the flush and the start
            event, so the host has certainly submitted the replay before the device gets
            to it (rules out host submission latency inside the interval);
  idle    — synchronize, 20 ms of host sleep (device idle), then flush + events (rules
            clock ramp-down in or out);
  b2b     — 20 replays inside one event pair, no flush (steady state, L2 warm).
SM / memory clocks are read through NVML before each arrangement.
"""
import json
import os
import statistics
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_1707_08213_b200.tree2d import _OUT_DTYPES, _precision_code, forward_into  # noqa: E402
from paper_1707_08213_b200.workloads import CONFIGS  # noqa: E402


def clocks():
    try:
        import pynvml

        pynvml.nvmlInit()
        h = pynvml.nvmlDeviceGetHandleByIndex(0)
        return {"sm": pynvml.nvmlDeviceGetClockInfo(h, pynvml.NVML_CLOCK_SM),
                "mem": pynvml.nvmlDeviceGetClockInfo(h, pynvml.NVML_CLOCK_MEM),
                "w": pynvml.nvmlDeviceGetPowerUsage(h) / 1e3}
    except Exception as e:  # noqa: BLE001
        return {"err": str(e)}


def main():
    dev = torch.device("cuda", 0)
    a = torch.empty(64 << 20, dtype=torch.float32, device=dev)
    b = torch.ones(64 << 20, dtype=torch.float32, device=dev)
    reps = int(os.environ.get("REPS", "25"))
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
        g.replay()
        for mode in ("bench", "sleep", "idle", "bench", "b2b"):
            ck = clocks()
            ts = []
            for _ in range(reps):
                torch.cuda.synchronize()
                if mode == "idle":
                    time.sleep(0.02)
                if mode != "b2b":
                    a.fill_(1.0)
                    b.sum()
                if mode == "sleep":
                    torch.cuda._sleep(600000)
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record()
                n = 20 if mode == "b2b" else 1
                for _ in range(n):
                    g.replay()
                e1.record()
                torch.cuda.synchronize()
                ts.append(e0.elapsed_time(e1) / n)
            print(json.dumps({"config": name, "mode": mode, "median_ms": statistics.median(ts),
                              "min_ms": min(ts), "max_ms": max(ts),
                              "samples": [round(t, 4) for t in ts], "clocks_before": ck}), flush=True)
        del g, x, out
        torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
