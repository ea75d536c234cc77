"""Small solves of every path for `compute-sanitizer --tool racecheck` /
`--tool memcheck` (shared-memory hazards / out-of-bounds accesses):

    compute-sanitizer --tool racecheck python tools/racecheck.py
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

import paper_1407_8315_b200 as P  # noqa: E402
from tests.synth import device_exact_batch, device_general_batch  # noqa: E402

dev = torch.device("cuda")
X, _, _ = device_exact_batch(2, 1 << 16, 64, 3, dev, values="unit")
cfg = P.ExactConfig(n=1 << 16, k=64)
for it in (False, True):
    P.exact_batch(X, cfg, it).to_host()
# large-view path (L > 8192): N=2^18, K=4 -> d=16384? use initial_d for L=16384
P.exact_batch(device_exact_batch(1, 1 << 18, 16, 4, dev, values="unit")[0],
              P.ExactConfig(n=1 << 18, k=16, initial_d=16), False).to_host()
G = device_general_batch(2, 1 << 14, 16, 20.0, 5, dev)
P.solve_general_batch(G, P.GeneralConfig(n=1 << 14, k=16)).to_host()
P.solve_general_batch(G, P.GeneralConfig(n=1 << 14, k=16, prune=False)).to_host()
pipe = P.SolvePipeline(cfg, batch=1, depth=3)
Xh = X.cpu().pin_memory()
for r in pipe.solve_stream([Xh[0:1], Xh[1:2], Xh[0:1], Xh[1:2]]):
    r.spectrum(0)
torch.cuda.synchronize()
print("racecheck workload done")
