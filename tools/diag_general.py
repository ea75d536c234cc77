import sys, math, torch, numpy as np
sys.path.insert(0, '.')
import bench, paper_1407_8315_b200 as P
sys.argv = ['bench.py', '--config', 'cfg4']
a = bench.parse()
dev = torch.device('cuda', 0)
X = bench.gen_batch(a, dev, a.seed)
cfg = P.GeneralConfig(n=a.n, k=a.k)
seeds = [(a.seed, 0, b) for b in range(a.batch)]
plan = P.GeneralPlan(cfg, a.batch, seeds, dev)
r = P.solve_general_batch(X, cfg, device=dev, plan=plan)
st = r.to_host()['stats']
from paper_1407_8315_b200 import _lib
h = st[:, _lib.SFDT_GS_HIST0:_lib.SFDT_GS_HIST0 + 5].sum(0)
print('hist', h.tolist(), 'rankdef', st[:, _lib.SFDT_GS_RANKDEF].sum())
