"""A fresh process whose first libswdft2d call is captured into a CUDA graph (used by
tests/test_gpu_parity.py::test_first_call_inside_graph_capture)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_1707_08213_b200.tree2d import _OUT_DTYPES, forward_into
dev = torch.device('cuda', 0)
x = torch.from_numpy(np.random.default_rng(0).standard_normal((64, 64)).astype(np.float32)).to(dev)
out = torch.empty((49, 49, 16, 16), dtype=_OUT_DTYPES[0], device=dev)
g = torch.cuda.CUDAGraph()
s = torch.cuda.Stream(dev)
torch.cuda.synchronize()
with torch.cuda.graph(g, stream=s):
    forward_into(x, 4, 4, out, prec=0, stream=s)
g.replay(); torch.cuda.synchronize()
ref = torch.empty_like(out); forward_into(x, 4, 4, ref, prec=0); torch.cuda.synchronize()
print("first-call capture ok", bool(torch.equal(out, ref)))
