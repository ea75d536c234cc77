import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_1407_8315_b200 as P
from tests.synth import device_exact_batch
count = 256
X, _, _ = device_exact_batch(count, 1 << 16, 64, 11, torch.device("cuda"), values="unit")
cfg = P.ExactConfig(n=1 << 16, k=64)
want = P.exact_batch(X, cfg, False).to_host()
def cmp(h, b, tag):
    lo, hi = h["entry_offsets"][0], h["entry_offsets"][1]
    wl, wh = want["entry_offsets"][b], want["entry_offsets"][b + 1]
    out = []
    if not np.array_equal(h["locs"][lo:hi], want["locs"][wl:wh]): out.append(f"locs {hi-lo} vs {wh-wl}")
    elif not np.array_equal(h["vals"][lo:hi], want["vals"][wl:wh]):
        out.append("vals maxdiff %.3g" % np.max(np.abs(h["vals"][lo:hi]-want["vals"][wl:wh])))
    if not np.array_equal(h["stats"][0], want["stats"][b]):
        out.append(f"stats {h['stats'][0][:8]} vs {want['stats'][b][:8]}")
    if out: print(tag, b, out)
    return not out
# 1. standalone single-signal exact_batch
bad1 = [b for b in range(count) if not cmp(P.exact_batch(X[b:b+1], cfg, False).to_host(), b, "single")]
print("single-signal exact_batch mismatches:", len(bad1))
# 2. SolveGraph one at a time
g = P.SolveGraph(cfg, batch=1)
bad2 = [b for b in range(count) if not cmp(g.solve(X[b:b+1]).to_host(), b, "graph")]
print("graph mismatches:", len(bad2))
# 3. host-io graph one at a time
gh = P.SolveGraph(cfg, batch=1, host_io=True)
Xh = X.cpu().pin_memory()
bad3 = [b for b in range(count) if not cmp(gh.solve_host(Xh[b:b+1])._host, b, "hostio")]
print("host-io graph mismatches:", len(bad3))
for depth in (1, 2, 4):
    pipe = P.SolvePipeline(cfg, batch=1, depth=depth)
    bad = [b for b, r in enumerate(pipe.solve_stream(Xh[b:b + 1] for b in range(count))) if not cmp(r._host, b, f"pipe{depth}")]
    print("pipeline depth", depth, "mismatches:", len(bad))
