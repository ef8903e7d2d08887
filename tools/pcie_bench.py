"""Host<->device copy rates on the GPU box (diagnostics for the e2e path)."""
import time
import torch

n = 10 * 1024**3 // 4  # 10 GiB fp32
h = torch.empty(n, dtype=torch.float32, pin_memory=True)
h.fill_(1.0)
d = torch.empty(n, dtype=torch.float32, device="cuda")
for name in ("single", "chunked2", "chunked4"):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    if name == "single":
        d.copy_(h, non_blocking=True)
    else:
        ns = int(name[-1])
        streams = [torch.cuda.Stream() for _ in range(ns)]
        ch = 256 * 1024**2 // 4
        for i, o in enumerate(range(0, n, ch)):
            with torch.cuda.stream(streams[i % ns]):
                d[o:o + ch].copy_(h[o:o + ch], non_blocking=True)
    torch.cuda.synchronize()
    dt = time.perf_counter() - t0
    print(f"H2D {name}: {n * 4 / dt / 1e9:.1f} GB/s")
m = 1470 * 1024**2 // 8
src = torch.empty(m, dtype=torch.float64, device="cuda")
for pinned in (False, True):
    dst = torch.empty(m, dtype=torch.float64, pin_memory=pinned)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    dst.copy_(src)
    torch.cuda.synchronize()
    dt = time.perf_counter() - t0
    print(f"D2H 1.47 GB pinned={pinned}: {m * 8 / dt / 1e9:.1f} GB/s")
