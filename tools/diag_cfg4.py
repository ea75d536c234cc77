import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_1407_8315_b200 as P
from oracle import solvers as OS
from tests.synth import device_general_batch
from tests import oracle_pool
n, k, B, snr = 1 << 20, 128, 1024, 20.0
X = device_general_batch(B, n, k, snr, 4020, torch.device("cuda"))
cfg = P.GeneralConfig(n=n, k=k)
seeds = [(4020, b) for b in range(B)]
res = P.solve_general_batch(X, cfg, seeds=seeds)
h = res.to_host()
idx = list(range(0, B, 4))
host = {b: X[b].cpu().numpy() for b in idx}
out = oracle_pool.run(host, [(b, "general", dict(k=k, rng_seed=seeds[b])) for b in idx])
L = n // cfg.resolved_d()
for b, _, locs, vals, wtr in out:
    lo, hi = h["entry_offsets"][b], h["entry_offsets"][b + 1]
    gl, gv = h["locs"][lo:hi], h["vals"][lo:hi]
    if set(gl.tolist()) != set(locs.tolist()):
        print("signal", b, "shifts", wtr["shifts"], "hist", wtr["collision_histogram"])
        extra = sorted(set(gl.tolist()) - set(locs.tolist())); missing = sorted(set(locs.tolist()) - set(gl.tolist()))
        print(" extra", extra[:40]); print(" missing", missing[:40])
        print(" extra bins", sorted({s % L for s in extra})); print(" missing bins", sorted({s % L for s in missing}))
        np.save("/tmp/sig.npy", host[b])
        want, tr = OS.general(host[b], k, rng_seed=seeds[b], return_internals=True)
        for kb in sorted({s % L for s in extra + missing})[:5]:
            print("  bin", kb, "vote", tr["votes"][kb], "kept", tr["kept"].get(kb))
            print("   oracle", [(s, want[s]) for s in want if s % L == kb])
            print("   gpu   ", [(int(s), complex(v)) for s, v in zip(gl, gv) if s % L == kb])
        print(" rank_deficient", tr["rank_deficient"][:5])
