import sys, time, torch
sys.path.insert(0, '.')
from paper_1707_08213_b200 import WindowSpec, _lib
from paper_1707_08213_b200.stream import SlidingRowStream2D
from paper_1707_08213_b200.workloads import CONFIGS
from paper_1707_08213_b200.tree2d import _OUT_DTYPES
cfg = CONFIGS['c4']
x = torch.from_numpy(cfg.generate(rows=400)).cuda()
st = SlidingRowStream2D(WindowSpec((cfg.m0, cfg.m1)), cfg.N1, precision='fp32')
for r in range(64): st.push_row(x[r])
torch.cuda.synchronize()
N = 200
t0 = time.perf_counter()
for r in range(64, 64 + N): st.push_row(x[r])
t_host = (time.perf_counter() - t0) / N
torch.cuda.synchronize()
t_all = (time.perf_counter() - t0) / N
# components
t0 = time.perf_counter()
for _ in range(N): torch.empty((st.P1, st.n0, st.n1), dtype=_OUT_DTYPES[0], device='cuda')
t_empty = (time.perf_counter() - t0) / N
t0 = time.perf_counter()
for _ in range(N): torch.cuda.current_device()
t_cd = (time.perf_counter() - t0) / N
t0 = time.perf_counter()
for _ in range(N): _lib.raw_stream(0)
t_rs = (time.perf_counter() - t0) / N
print(f"push host {t_host*1e6:.1f} us, incl sync {t_all*1e6:.1f} us; torch.empty {t_empty*1e6:.1f}, current_device {t_cd*1e6:.2f}, raw_stream {t_rs*1e6:.2f}")
