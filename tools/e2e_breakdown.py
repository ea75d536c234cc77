"""Where the config-1 end-to-end time goes (SolveGraph host_io, one signal):
H2D copy alone, graph replay alone (solve + D2H), and the full solve_host,
each host-timed over many repetitions with a sync per repetition."""
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1407_8315_b200 as P  # noqa: E402
from tests.synth import exact_signal  # noqa: E402

dev = torch.device("cuda", 0)
n, k = 1 << 16, 64
x = exact_signal(n, k, 0, "unit")[0]
xp = torch.from_numpy(x[None]).pin_memory()
g = P.SolveGraph(P.ExactConfig(n=n, k=k), batch=1, host_io=True)
s = torch.cuda.current_stream(dev)


def t(f, reps=2000):
    for _ in range(50):
        f()
    t0 = time.perf_counter()
    for _ in range(reps):
        f()
    return (time.perf_counter() - t0) / reps * 1e6


print("h2d 1 MiB + sync      %.1f us" % t(lambda: (g.X.copy_(xp, non_blocking=True), s.synchronize())))
print("graph replay + sync   %.1f us" % t(lambda: (g.graph.replay(), s.synchronize())))
print("h2d + replay + sync   %.1f us" % t(lambda: (g.X.copy_(xp, non_blocking=True), g.graph.replay(), s.synchronize())))
print("solve_host(pinned)    %.1f us" % t(lambda: g.solve_host(xp)))
print("empty sync            %.1f us" % t(lambda: s.synchronize()))
print("d2h nodes:", len(g._host_out), sum(v.nbytes for v in g._host_out.values()), "bytes")
