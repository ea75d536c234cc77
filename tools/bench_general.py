"""Quick device timing of the general path at config 4 (B=1024, N=2^20,
K=128, 20 dB) with per-signal shift seeds; prints signals/s."""
import math
import sys
import time

import torch

sys.path.insert(0, ".")
import paper_1407_8315_b200 as P  # noqa: E402


def gen(B, n, k, snr_db, seed, dev):
    g = torch.Generator(device=dev)
    g.manual_seed(seed)
    X = torch.empty((B, n), dtype=torch.complex128, device=dev)
    for lo in range(0, B, 128):
        hi = min(B, lo + 128)
        idx = torch.topk(torch.rand((hi - lo, n), generator=g, device=dev), k, dim=1).indices
        ph = 2 * math.pi * torch.rand((hi - lo, k), generator=g, device=dev, dtype=torch.float64)
        dense = torch.zeros((hi - lo, n), dtype=torch.complex128, device=dev)
        dense.scatter_(1, idx, torch.polar(torch.ones_like(ph), ph))
        clean = torch.fft.ifft(dense, dim=1) * n
        p_sig = (clean.abs() ** 2).mean(dim=1, keepdim=True)
        sigma = torch.sqrt(p_sig / 10 ** (snr_db / 10) / 2)
        noise = torch.complex(torch.randn((hi - lo, n), generator=g, device=dev, dtype=torch.float64),
                              torch.randn((hi - lo, n), generator=g, device=dev, dtype=torch.float64))
        X[lo:hi] = clean + sigma * noise
    return X


if __name__ == "__main__":
    B = int(sys.argv[1]) if len(sys.argv) > 1 else 1024
    n, k = 1 << 20, 128
    dev = torch.device("cuda", 0)
    X = gen(B, n, k, 20.0, 1, dev)
    cfg = P.GeneralConfig(n=n, k=k)
    plan = P.GeneralPlan(cfg, B, [(9, b) for b in range(B)], dev)
    for _ in range(2):
        r = P.solve_general_batch(X, cfg, device=dev, plan=plan)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    steps = 5
    e0.record()
    for _ in range(steps):
        r = P.solve_general_batch(X, cfg, device=dev, plan=plan)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / steps
    print(f"general cfg4 B={B}: {ms:.3f} ms/step  {B / ms * 1e3:.1f} signals/s  launches={r.kernel_launches}")
