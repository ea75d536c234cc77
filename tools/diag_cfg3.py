import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_1407_8315_b200 as P
from oracle import solvers as OS
from tests.synth import device_exact_batch
n, k, mu, b = 1 << 24, 4096, 1, 3
X, _, _ = device_exact_batch(8, n, k, 304, torch.device("cuda"), values="unit")
x = X[b].cpu().numpy()
np.save("/tmp/cfg3_sig.npy", x)
cfg = P.ExactConfig(n=n, k=k, mu=mu)
res = P.exact_batch(X[b:b+1], cfg, True)
got, tr = res.spectrum(0).entries, res.trace(0)
bins = [1504]
for kern in ("port", "numpy"):
    want, wtr = OS.exact_iterative(x, k, mu, kernels=kern)
    print(kern, "entries", len(want), "full", wtr["full_success"], "unres", wtr["unresolved_bins"][:20])
    print("  iterations", wtr["iterations"])
    for s in sorted(want):
        if s % 4096 in bins: print("   ", kern, s, want[s])
print("gpu entries", len(got), "full", tr.full_success, "unres", tr.unresolved_bins[:20])
print("  iterations", [vars(i) for i in tr.iterations])
for s in sorted(got):
    if s % 4096 in bins: print("    gpu", s, got[s])
