import json, numpy as np, torch, sys
sys.path.insert(0, '.')
from paper_1707_08213_b200.tree2d import _OUT_DTYPES, forward_into
dev = torch.device("cuda", 0)
flush = torch.empty(64 << 20, dtype=torch.float32, device=dev)
for prec in (0, 1):
    for m in (2, 4, 5, 6):
        n = 1 << m
        for L in (1024, 4096):
            R = (1 << 20) // L
            x = torch.randn((R, L + n - 1), dtype=torch.float64, device=dev)
            out = torch.empty((R, L, 1, n), dtype=_OUT_DTYPES[prec], device=dev)
            s = torch.cuda.Stream(dev)
            forward_into(x, 0, m, out, prec=prec, stream=s)
            torch.cuda.synchronize()
            g = torch.cuda.CUDAGraph()
            with torch.cuda.graph(g, stream=s):
                forward_into(x, 0, m, out, prec=prec, stream=s)
            ts = []
            for _ in range(5):
                torch.cuda.synchronize(); flush.fill_(1.0)
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record(); g.replay(); e1.record(); torch.cuda.synchronize()
                ts.append(e0.elapsed_time(e1) / 1e3)
            t = float(np.median(ts))
            print(json.dumps({"n": n, "L": L, "R": R, "prec": prec, "gcoef_s": R * L * n / t / 1e9, "tbs": R * L * n * (16 if prec else 8) / t / 1e12}), flush=True)
