"""Pinned host -> device copy bandwidth (PCIe) for the e2e path."""
import time
import torch

dev = torch.device("cuda", 0)
for mb in (64, 256, 1024, 4096):
    n = mb << 20
    h = torch.empty(n, dtype=torch.uint8).pin_memory()
    d = torch.empty(n, dtype=torch.uint8, device=dev)
    for streams in (1, 2, 4):
        ss = [torch.cuda.Stream(dev) for _ in range(streams)]
        part = n // streams
        d.copy_(h, non_blocking=True)
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        reps = max(2, 8192 // mb)
        for _ in range(reps):
            for i, st in enumerate(ss):
                with torch.cuda.stream(st):
                    d[i * part:(i + 1) * part].copy_(h[i * part:(i + 1) * part], non_blocking=True)
        torch.cuda.synchronize()
        dt = time.perf_counter() - t0
        print(f"{mb:5d} MiB x{reps} streams={streams}: {reps * n / dt / 1e9:.1f} GB/s")
