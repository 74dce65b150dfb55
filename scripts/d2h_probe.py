"""PCIe D2H throughput for the e2e path: one big pinned copy vs chunked copies on 1-4 streams."""
import time
import torch

n = 34108540928 // 8  # config-4 output, complex64 elements
dev = torch.device("cuda", 0)
src = torch.empty(n, dtype=torch.complex64, device=dev)
src.real.fill_(1.0)
dst = torch.empty(n, dtype=torch.complex64, pin_memory=True)
print("pinned alloc done", flush=True)
for streams in (1, 2, 4):
    for chunks in (1, 8, 64):
        if chunks < streams:
            continue
        ss = [torch.cuda.Stream(dev) for _ in range(streams)]
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        per = (n + chunks - 1) // chunks
        for c in range(chunks):
            a, b = c * per, min(n, (c + 1) * per)
            with torch.cuda.stream(ss[c % streams]):
                dst[a:b].copy_(src[a:b], non_blocking=True)
        torch.cuda.synchronize()
        dt = time.perf_counter() - t0
        print(f"streams={streams} chunks={chunks} {n * 8 / dt / 1e9:.1f} GB/s", flush=True)
