"""Per-item cycle histogram of the general-path pursuit (k_gen_bins) at cfg4."""
import ctypes
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
import bench  # noqa: E402
import paper_1407_8315_b200 as P  # noqa: E402
from paper_1407_8315_b200 import _lib  # noqa: E402

sys.argv = ["bench.py", "--config", "cfg4"]
a = bench.parse()
dev = torch.device("cuda", 0)
X = bench.gen_batch(a, dev, a.seed)
cfg = P.GeneralConfig(n=a.n, k=a.k)
plan = P.GeneralPlan(cfg, a.batch, [(a.seed, 0, b) for b in range(a.batch)], dev)
lib = _lib.load()
f = lib.sfdt_debug_cycles
f.argtypes = [ctypes.c_int, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int64, ctypes.c_void_p]
P.solve_general_batch(X, cfg, device=dev, plan=plan)
torch.cuda.synchronize()
f(1, None, None, 0, None)
P.solve_general_batch(X, cfg, device=dev, plan=plan)
torch.cuda.synchronize()
cyc = np.zeros(16384, np.int64)
tag = np.zeros(16384, np.int32)
cnt = ctypes.c_int64()
f(-1, cyc.ctypes.data, tag.ctypes.data, 16384, ctypes.byref(cnt))
f(0, None, None, 0, None)
n = cnt.value
cyc, tag = cyc[:n], tag[:n]
print("items", n, "cycles: mean", cyc.mean(), "p50", np.median(cyc), "p99", np.percentile(cyc, 99), "max", cyc.max())
for t in sorted(set(tag.tolist())):
    m = tag == t
    print(f"a={t // 100} ncols={t % 100}: {m.sum():6d} items, mean {cyc[m].mean():10.0f}  max {cyc[m].max():10d}")
