"""Config-1 latency over many signals: collision histogram of each signal's
bins and the CUDA-graph replay time per decode_coop mode (CUDA events over
`reps` replays per signal).  python tools/cfg1_latency.py [nsig]"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_1407_8315_b200 as P
from tests.synth import device_exact_batch

nsig = int(sys.argv[1]) if len(sys.argv) > 1 else 16
dev = torch.device("cuda")
n, k = 1 << 16, 64
cfg = P.ExactConfig(n=n, k=k)
L = n // cfg.resolved_d()
X, sup, _ = device_exact_batch(nsig, n, k, 2024, dev, values="unit")
hist = np.zeros((nsig, 8), int)
for b in range(nsig):
    c = np.bincount(np.bincount(sup[b] % L, minlength=L), minlength=8)
    hist[b] = c[:8]
modes = [0, 1, 2, 3]
graphs = {}
for m in modes:
    with P.tuning(decode_coop=m):
        graphs[m] = P.SolveGraph(cfg, batch=1)
res = np.zeros((nsig, len(modes)))
reps = 50
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
for b in range(nsig):
    for i, m in enumerate(modes):
        g = graphs[m]
        g.solve(X[b:b + 1])
        for _ in range(5):
            g.graph.replay()
        torch.cuda.synchronize()
        e0.record()
        for _ in range(reps):
            g.graph.replay()
        e1.record()
        torch.cuda.synchronize()
        res[b, i] = e0.elapsed_time(e1) * 1e3 / reps
    print(f"sig {b:2d} bins by collisions a=1..5: {hist[b][1:6]}  us per replay by mode {modes}: "
          + " ".join(f"{v:6.1f}" for v in res[b]))
print("mean us per replay by mode", modes, " ".join(f"{v:6.1f}" for v in res.mean(0)))
