"""Generate tests/golden/ fixtures by running the REAL reference package.

Run in the build container (needs /root/reference):

    python tests/golden/make_golden.py

It stages /root/reference/pkg into a scratch directory under /tmp, builds the
reference's Cython extension there (compiled backend), imports `sfft_dt` and
records, for every case in cases.py, the reference solver outputs plus the
sha256 of the input bytes.  Kernel-level vectors (fft_radix2, hankel_solve,
poly_roots, vandermonde_solve, prune_eval, hankel_singular_values) are
recorded with their inputs.  Nothing from the reference is copied into the
repository -- only its outputs.
"""

from __future__ import annotations

import hashlib
import json
import os
import shutil
import subprocess
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)
sys.path.insert(0, HERE)

from cases import EXACT_CASES, GENERAL_CASES, NUMPY_BACKEND_CASES, NUMPY_BACKEND_GENERAL  # noqa: E402
from tests.synth import exact_signal, general_signal  # noqa: E402

SCRATCH = "/tmp/sfdt_ref_golden"


def import_reference(backend="compiled"):
    if not os.path.isdir(os.path.join(SCRATCH, "src")):
        shutil.rmtree(SCRATCH, ignore_errors=True)
        shutil.copytree("/root/reference/pkg", SCRATCH)
        subprocess.run([sys.executable, "setup.py", "build_ext", "--inplace"], cwd=SCRATCH,
                       check=True, capture_output=True)
    sys.path.insert(0, os.path.join(SCRATCH, "src"))
    import sfft_dt
    assert sfft_dt.BACKEND == backend, sfft_dt.BACKEND
    return sfft_dt


def numpy_backend_main():
    """Child process with SFFT_DT_PURE_PYTHON=1: the reference's numpy
    backend on the kernel inputs of golden.npz and on NUMPY_BACKEND_CASES
    -> golden_numpy.npz / .json."""
    ref = import_reference("python")
    from sfft_dt import _kernels as K
    g = np.load(os.path.join(HERE, "golden.npz"))
    arrays, meta = {}, {"exact": {}, "general": {}}
    for n in (1, 2, 4, 8, 16, 64, 256, 512, 1024, 2048):
        x = g[f"kern/fft/{n}/in"]
        arrays[f"kern/fft/{n}/fwd"] = K.fft_radix2(x, inverse=False)
        arrays[f"kern/fft/{n}/inv"] = K.fft_radix2(x, inverse=True)
    for a in (1, 2, 3, 4):
        m, kb = g[f"kern/a{a}/m"], g[f"kern/a{a}/k"]
        c, cd = K.hankel_solve(m, a)
        z = K.poly_roots(c)
        p, pd = K.vandermonde_solve(z, m)
        arrays.update({f"kern/a{a}/c": c, f"kern/a{a}/cd": cd, f"kern/a{a}/z": z,
                       f"kern/a{a}/p": p, f"kern/a{a}/pd": pd,
                       f"kern/a{a}/prune": K.prune_eval(c, kb, 1 << 12, 64),
                       f"kern/a{a}/sv": K.hankel_singular_values(m, a)})
    for name, n, k, mu, a_max, values, seed, synth in EXACT_CASES:
        if name not in NUMPY_BACKEND_CASES:
            continue
        x, _ = exact_signal(n, k, seed, values, synth)
        cfg = ref.ExactConfig(n=n, k=k, mu=mu, a_max=a_max)
        rec = {}
        for solver in ("noniterative", "iterative"):
            spec, tr = getattr(ref, f"solve_{solver}")(x, cfg)
            arrays[f"{name}/{solver}/locs"], arrays[f"{name}/{solver}/vals"] = pack_entries(spec.entries)
            rec[solver] = {"full_success": tr.full_success, "warnings": tr.warnings,
                           "unresolved_bins": [int(b) for b in tr.unresolved_bins]}
        meta["exact"][name] = rec
    for name, n, k, snr_db, seed, prune in GENERAL_CASES:
        if name not in NUMPY_BACKEND_GENERAL:
            continue
        x, _ = general_signal(n, k, snr_db, seed)
        spec, tr = ref.solve_general(x, ref.GeneralConfig(n=n, k=k, rng_seed=seed, prune=prune))
        arrays[f"{name}/general/locs"], arrays[f"{name}/general/vals"] = pack_entries(spec.entries)
        meta["general"][name] = {"collision_histogram": {str(a): c for a, c in
                                                         tr.collision_histogram.items()}}
    np.savez_compressed(os.path.join(HERE, "golden_numpy.npz"), **arrays)
    with open(os.path.join(HERE, "golden_numpy.json"), "w") as fh:
        json.dump(meta, fh, indent=1, sort_keys=True)
    print("wrote", os.path.join(HERE, "golden_numpy.npz"))


def sha(x):
    return hashlib.sha256(np.ascontiguousarray(x, dtype=np.complex128).tobytes()).hexdigest()


def pack_entries(entries):
    locs = np.fromiter(entries.keys(), dtype=np.int64, count=len(entries))
    vals = np.fromiter(entries.values(), dtype=np.complex128, count=len(entries))
    return locs, vals


def main():
    ref = import_reference()
    arrays, meta = {}, {"exact": {}, "general": {}, "numpy": np.__version__}

    for name, n, k, mu, a_max, values, seed, synth in EXACT_CASES:
        x, _ = exact_signal(n, k, seed, values, synth)
        cfg = ref.ExactConfig(n=n, k=k, mu=mu, a_max=a_max)
        rec = {"sha256": sha(x)}
        for solver in ("noniterative", "iterative"):
            spec, tr = getattr(ref, f"solve_{solver}")(x, cfg)
            locs, vals = pack_entries(spec.entries)
            arrays[f"{name}/{solver}/locs"] = locs
            arrays[f"{name}/{solver}/vals"] = vals
            rec[solver] = {
                "full_success": tr.full_success, "fft_samples": tr.fft_samples,
                "syndromes_computed": tr.syndromes_computed,
                "unresolved_bins": [int(b) for b in tr.unresolved_bins],
                "warnings": tr.warnings,
                "iterations": [dict(vars(it)) for it in tr.iterations],
            }
        if n <= 16384:
            est = ref.estimate_sparsity_and_solve(x, mu=mu, a_max=a_max)
            locs, vals = pack_entries(est.spectrum.entries)
            arrays[f"{name}/estimate/locs"] = locs
            arrays[f"{name}/estimate/vals"] = vals
            rec["estimate"] = {"k_hat": est.k_hat, "final_d": est.final_d,
                               "fft_samples": est.fft_samples,
                               "fft_samples_final_run": est.fft_samples_final_run,
                               "dense_fallback": est.dense_fallback,
                               "stages": [[int(d), bool(s)] for d, s in est.stages]}
        meta["exact"][name] = rec
        print(name, {s: len(arrays[f"{name}/{s}/locs"]) for s in ("noniterative", "iterative")})

    for name, n, k, snr_db, seed, prune in GENERAL_CASES:
        x, _ = general_signal(n, k, snr_db, seed)
        cfg = ref.GeneralConfig(n=n, k=k, rng_seed=seed, prune=prune)
        spec, tr = ref.solve_general(x, cfg)
        locs, vals = pack_entries(spec.entries)
        arrays[f"{name}/general/locs"] = locs
        arrays[f"{name}/general/vals"] = vals
        meta["general"][name] = {"sha256": sha(x), "d": tr.d, "r": tr.r, "shifts": tr.shifts,
                                 "fft_samples": tr.fft_samples,
                                 "collision_histogram": {str(a): c for a, c in
                                                         tr.collision_histogram.items()}}
        print(name, len(locs))

    # kernel-level vectors, inputs stored alongside
    from sfft_dt import _kernels as K
    rng = np.random.default_rng(0x5F0)
    for n in (1, 2, 4, 8, 16, 64, 256, 512, 1024, 2048):
        x = rng.standard_normal(n) + 1j * rng.standard_normal(n)
        arrays[f"kern/fft/{n}/in"] = x
        arrays[f"kern/fft/{n}/fwd"] = K.fft_radix2(x, inverse=False)
        arrays[f"kern/fft/{n}/inv"] = K.fft_radix2(x, inverse=True)
    for a in (1, 2, 3, 4):
        # half random syndromes, half true a-sparse syndromes on the unit circle
        rnd = rng.standard_normal((32, 8)) + 1j * rng.standard_normal((32, 8))
        roots = np.exp(2j * np.pi * rng.random((32, a)))
        vals = rng.standard_normal((32, a)) + 1j * rng.standard_normal((32, a))
        tru = np.stack([np.sum(vals * roots ** l, axis=1) for l in range(8)], axis=1)
        m = np.concatenate([rnd, tru])
        c, cd = K.hankel_solve(m, a)
        z = K.poly_roots(c)
        p, pd = K.vandermonde_solve(z, m)
        kb = rng.integers(0, 1 << 6, size=m.shape[0]).astype(np.int64)
        arrays[f"kern/a{a}/m"] = m
        arrays[f"kern/a{a}/c"] = c
        arrays[f"kern/a{a}/cd"] = cd
        arrays[f"kern/a{a}/z"] = z
        arrays[f"kern/a{a}/p"] = p
        arrays[f"kern/a{a}/pd"] = pd
        arrays[f"kern/a{a}/k"] = kb
        arrays[f"kern/a{a}/prune"] = K.prune_eval(c, kb, 1 << 12, 64)
        arrays[f"kern/a{a}/sv"] = K.hankel_singular_values(m, a)

    np.savez_compressed(os.path.join(HERE, "golden.npz"), **arrays)
    with open(os.path.join(HERE, "golden.json"), "w") as fh:
        json.dump(meta, fh, indent=1, sort_keys=True)
    print("wrote", os.path.join(HERE, "golden.npz"))
    # the reference's second (pure-numpy) backend, in a child process: the
    # backend is chosen once at import (_kernels/__init__.py:11-17)
    subprocess.run([sys.executable, os.path.abspath(__file__), "--numpy-backend"], check=True,
                   env=dict(os.environ, SFFT_DT_PURE_PYTHON="1"))


if __name__ == "__main__":
    if "--numpy-backend" in sys.argv:
        numpy_backend_main()
    else:
        main()
