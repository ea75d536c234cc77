"""Run the CPU oracle (oracle/solvers.py) over many signals on every host
core -- test infrastructure for the sampled parity checks at BASELINE
sizes.

Signals are published in a module-level store BEFORE the fork pool starts,
so the workers inherit them copy-on-write (no pickling of 16-256 MiB rows);
only (job index -> entries, trace) travel back.  Workers run numpy + the
oracle's C kernels only; they never touch CUDA.
"""

from __future__ import annotations

import multiprocessing as mp
import os

import numpy as np

_STORE: dict = {}


def _run(job):
    from oracle import solvers as OS
    key, fn, kwargs = job
    x = _STORE[key]
    if fn == "general":
        want, tr = OS.general(x, **kwargs)
    elif fn == "noniterative":
        want, tr = OS.exact_noniterative(x, **kwargs)
    elif fn == "iterative":
        want, tr = OS.exact_iterative(x, **kwargs)
    else:
        raise ValueError(fn)
    # plain picklable data back to the parent
    tr = {k: (v.tolist() if isinstance(v, np.ndarray) and k != "votes" else v)
          for k, v in tr.items() if k not in ("consecutive", "random_views", "singular_values")}
    locs = np.fromiter(want.keys(), dtype=np.int64, count=len(want))
    vals = np.fromiter(want.values(), dtype=np.complex128, count=len(want))
    return key, fn, locs, vals, tr


def run(signals: dict, jobs: list, procs: int | None = None) -> list:
    """signals: {key: 1-D complex ndarray}; jobs: [(key, fn, kwargs)] with
    fn in {"noniterative", "iterative", "general"}.  Returns one
    (key, fn, locs, vals, trace) per job, in job order."""
    _STORE.clear()
    _STORE.update(signals)
    procs = procs or max(1, min(len(jobs), os.cpu_count() or 1))
    os.environ.setdefault("OPENBLAS_NUM_THREADS", "1")
    try:
        if procs == 1:
            return [_run(j) for j in jobs]
        with mp.get_context("fork").Pool(procs) as pool:
            return pool.map(_run, jobs, chunksize=1)
    finally:
        _STORE.clear()
