"""Pin the CPU oracle (oracle/) before trusting it as the parity checker.

* the C restatement of the kernels is bit-identical to the golden vectors the
  real reference produced (tests/golden/make_golden.py) and, when built, to
  the reference's own compiled _core (oracle/_ref);
* the restated solver drivers reproduce every golden solver output exactly
  (supports, values, traces);
* the reference's own known-answer tests for the kernels
  (/root/reference/pkg/tests/test_spectral.py, test_syndrome.py) hold.
"""

import hashlib

import numpy as np
import pytest

from oracle import kernels as OK
from oracle import solvers as OS
from tests.golden.cases import EXACT_CASES, GENERAL_CASES
from tests.synth import exact_signal, general_signal


def bits_equal(a, b):
    a, b = np.asarray(a), np.asarray(b)
    return a.shape == b.shape and a.dtype == b.dtype and np.array_equal(
        a.view(np.uint8), b.view(np.uint8))


def sha(x):
    return hashlib.sha256(np.ascontiguousarray(x, dtype=np.complex128).tobytes()).hexdigest()


# ---------------------------------------------------------------- kernels
def test_fft_golden_bitexact(golden):
    arrays, _ = golden
    for n in (1, 2, 4, 8, 16, 64, 256, 512, 1024, 2048):
        x = arrays[f"kern/fft/{n}/in"]
        assert bits_equal(OK.fft_radix2(x, False), arrays[f"kern/fft/{n}/fwd"])
        assert bits_equal(OK.fft_radix2(x, True), arrays[f"kern/fft/{n}/inv"])


@pytest.mark.parametrize("a", [1, 2, 3, 4])
def test_decode_kernels_golden_bitexact(golden, a):
    arrays, _ = golden
    m = arrays[f"kern/a{a}/m"]
    c, cd = OK.hankel_solve(m, a)
    assert bits_equal(c, arrays[f"kern/a{a}/c"]) and bits_equal(cd, arrays[f"kern/a{a}/cd"])
    z = OK.poly_roots(c)
    assert bits_equal(z, arrays[f"kern/a{a}/z"])
    p, pd = OK.vandermonde_solve(z, m)
    assert bits_equal(p, arrays[f"kern/a{a}/p"]) and bits_equal(pd, arrays[f"kern/a{a}/pd"])
    assert bits_equal(OK.prune_eval(c, arrays[f"kern/a{a}/k"], 1 << 12, 64),
                      arrays[f"kern/a{a}/prune"])
    assert bits_equal(OK.hankel_singular_values(m, a), arrays[f"kern/a{a}/sv"])


def test_port_matches_reference_core():
    if OK.reference_core_path() is None:
        pytest.skip("oracle/_ref not built (needs /root/reference)")
    P, R = OK.backend("port"), OK.backend("reference")
    rng = np.random.default_rng(7)
    for n in (2, 32, 1024, 1 << 14):
        x = rng.standard_normal(n) + 1j * rng.standard_normal(n)
        assert bits_equal(P.fft_radix2(x, False), R.fft_radix2(x, False))
    for a in (1, 2, 3, 4):
        m = rng.standard_normal((300, 8)) + 1j * rng.standard_normal((300, 8))
        c, cd = P.hankel_solve(m, a)
        c2, cd2 = R.hankel_solve(m, a)
        assert bits_equal(c, c2) and bits_equal(cd, cd2)
        z = P.poly_roots(c)
        assert bits_equal(z, R.poly_roots(c))
        assert all(bits_equal(u, v) for u, v in zip(P.vandermonde_solve(z, m),
                                                     R.vandermonde_solve(z, m)))
        k = rng.integers(0, 1 << 10, 300)
        assert bits_equal(P.prune_eval(c, k, 1 << 16, 700), R.prune_eval(c, k, 1 << 16, 700))
        assert bits_equal(P.hankel_singular_values(m, a), R.hankel_singular_values(m, a))


def test_kernel_argument_errors():
    with pytest.raises(ValueError):
        OK.fft_radix2(np.zeros(12))
    with pytest.raises(ValueError):
        OK.fft_radix2(np.zeros(0))
    with pytest.raises(ValueError):
        OK.hankel_solve(np.zeros((2, 3), complex), 2)
    with pytest.raises(ValueError):
        OK.hankel_solve(np.zeros((2, 10), complex), 5)
    with pytest.raises(ValueError):
        OK.poly_roots(np.zeros((2, 5), complex))
    with pytest.raises(ValueError):
        OK.hankel_singular_values(np.zeros((2, 4), complex), 3)


# ------------------------------------------- reference known-answer tests
def test_known_answers_spectral():
    # pkg/tests/test_spectral.py:21-28, 37-44, 79-82, 117-121
    n = 8
    x = np.fft.ifft(np.where(np.arange(n) == 5, 2.0, 0.0)) * n
    m0 = OS.shifted_view(OK, x, 4, 0)[1]
    m1 = OS.shifted_view(OK, x, 4, 1)[1]
    assert abs(m0 - 2.0) < 1e-12 and abs(m1 - 2.0 * np.exp(1.25j * np.pi)) < 1e-12
    assert np.allclose(OK.fft_radix2(np.array([1.0, 0, 0, 0])), np.ones(4), atol=1e-14)
    assert np.allclose(OK.fft_radix2(np.exp(2j * np.pi * np.arange(4) / 4)), [0, 4, 0, 0],
                       atol=1e-12)
    idx = (4 * np.arange(2) + 7) % 8
    assert np.array_equal(np.arange(8)[idx], [7, 3])
    x = np.fft.ifft(np.where((np.arange(8) == 1) | (np.arange(8) == 5), 1.0, 0.0)) * 8
    assert abs(OS.shifted_view(OK, x, 2, 0)[1] - 2.0) < 1e-12


def test_known_answers_fft_vs_numpy(rng):
    # pkg/tests/test_spectral.py:46-50 (<= 1e-10 relative vs direct DFT)
    x = rng.normal(size=256) + 1j * rng.normal(size=256)
    ours = OK.fft_radix2(x) / 256
    ref = np.fft.fft(x) / 256
    assert np.max(np.abs(ours - ref)) <= 1e-10 * np.max(np.abs(ref))


def test_known_answers_syndrome():
    # pkg/tests/test_syndrome.py:74-84, 97-105, 137-151
    m = np.array([[2, 0, 2, 0]], dtype=complex)
    c, cd = OK.hankel_solve(m, 2)
    assert np.allclose(c, [[-1.0, 0.0]], atol=1e-14)
    c, cd = OK.hankel_solve(np.array([[2, 2, 2, 2]], dtype=complex), 2)
    assert abs(cd[0]) <= 1e-10 * 2.0 ** 2          # NearSingular
    z = OK.poly_roots(np.array([[1j, -(1 + 1j)]]))
    assert sorted(np.round(z[0], 12), key=lambda t: (t.real, t.imag)) == [1j, 1.0]
    p, pd = OK.vandermonde_solve(np.array([[1.0, -1.0]], dtype=complex), m)
    assert np.allclose(p, [[1.0, 1.0]], atol=1e-14)
    p, pd = OK.vandermonde_solve(np.array([[1.0, 1.0]], dtype=complex),
                                 np.array([[2, 2, 2, 2]], dtype=complex))
    assert abs(pd[0]) <= 1e-10                      # IllConditioned


def test_known_answers_roots_residual(rng):
    # pkg/tests/test_syndrome.py:109-128 (residual bound 1e-8 max(1, |c|))
    for a in (2, 3, 4):
        roots = np.exp(2j * np.pi * rng.random((200, a)))
        c = np.stack([np.poly(r)[1:][::-1] for r in roots])
        z = OK.poly_roots(c)
        res = OS._residuals(c, z)
        assert np.all(res.max(axis=1) <= 1e-8 * np.maximum(1.0, np.abs(c).max(axis=1)))


# ------------------------------------------------------------ solvers
def _check_entries(entries, arrays, key):
    locs, vals = arrays[f"{key}/locs"], arrays[f"{key}/vals"]
    assert list(entries.keys()) == locs.tolist()          # same insertion order
    got = np.fromiter(entries.values(), dtype=np.complex128, count=len(entries))
    assert bits_equal(got, vals)


@pytest.mark.parametrize("case", EXACT_CASES, ids=[c[0] for c in EXACT_CASES])
def test_exact_solvers_match_reference(golden, case):
    arrays, meta = golden
    name, n, k, mu, a_max, values, seed, synth = case
    x, _ = exact_signal(n, k, seed, values, synth)
    rec = meta["exact"][name]
    assert sha(x) == rec["sha256"], "input generator drifted"
    for solver, fn in (("noniterative", OS.exact_noniterative),
                       ("iterative", OS.exact_iterative)):
        entries, tr = fn(x, k, mu, a_max)
        _check_entries(entries, arrays, f"{name}/{solver}")
        want = rec[solver]
        for key in ("full_success", "fft_samples", "syndromes_computed", "unresolved_bins",
                    "warnings", "iterations"):
            assert tr[key] == want[key], (solver, key)
    if "estimate" in rec:
        est = OS.exact_estimate(x, mu, a_max)
        _check_entries(est["entries"], arrays, f"{name}/estimate")
        for key in ("k_hat", "final_d", "fft_samples", "fft_samples_final_run",
                    "dense_fallback"):
            assert est[key] == rec["estimate"][key]
        assert [list(s) for s in est["stages"]] == rec["estimate"]["stages"]


@pytest.mark.parametrize("case", GENERAL_CASES, ids=[c[0] for c in GENERAL_CASES])
def test_general_solver_matches_reference(golden, case):
    arrays, meta = golden
    name, n, k, snr_db, seed, prune = case
    x, _ = general_signal(n, k, snr_db, seed)
    rec = meta["general"][name]
    assert sha(x) == rec["sha256"]
    entries, tr = OS.general(x, k, rng_seed=seed, prune=prune)
    _check_entries(entries, arrays, f"{name}/general")
    assert tr["shifts"] == rec["shifts"] and tr["d"] == rec["d"] and tr["r"] == rec["r"]
    assert {str(a): c for a, c in tr["collision_histogram"].items()} == \
        rec["collision_histogram"]


# ------------------------------------------ the reference's numpy backend
# oracle/numpy_kernels.py restates the reference's second backend
# (_kernels/_reference.py); the parity tests use it for the reference's own
# numerical envelope, so it is pinned bit-exact to that backend's outputs
# (tests/golden/golden_numpy.npz, written by make_golden.py with
# SFFT_DT_PURE_PYTHON=1).
@pytest.fixture(scope="module")
def golden_numpy():
    import json
    import os
    from tests.conftest import GOLDEN_DIR
    arrays = np.load(os.path.join(GOLDEN_DIR, "golden_numpy.npz"))
    with open(os.path.join(GOLDEN_DIR, "golden_numpy.json")) as fh:
        return arrays, json.load(fh)


def test_numpy_backend_kernels_bitexact(golden, golden_numpy):
    arrays, _ = golden
    want, _ = golden_numpy
    NK = OK.backend("numpy")
    for n in (1, 2, 4, 8, 16, 64, 256, 512, 1024, 2048):
        x = arrays[f"kern/fft/{n}/in"]
        assert bits_equal(NK.fft_radix2(x, False), want[f"kern/fft/{n}/fwd"])
        assert bits_equal(NK.fft_radix2(x, True), want[f"kern/fft/{n}/inv"])
    for a in (1, 2, 3, 4):
        m, kb = arrays[f"kern/a{a}/m"], arrays[f"kern/a{a}/k"]
        c, cd = NK.hankel_solve(m, a)
        assert bits_equal(c, want[f"kern/a{a}/c"]) and bits_equal(cd, want[f"kern/a{a}/cd"])
        z = NK.poly_roots(c)
        assert bits_equal(z, want[f"kern/a{a}/z"])
        p, pd = NK.vandermonde_solve(z, m)
        assert bits_equal(p, want[f"kern/a{a}/p"]) and bits_equal(pd, want[f"kern/a{a}/pd"])
        assert bits_equal(NK.prune_eval(c, kb, 1 << 12, 64), want[f"kern/a{a}/prune"])
        assert bits_equal(NK.hankel_singular_values(m, a), want[f"kern/a{a}/sv"])


def test_numpy_backend_solvers_bitexact(golden_numpy):
    from tests.golden.cases import NUMPY_BACKEND_CASES, NUMPY_BACKEND_GENERAL
    arrays, meta = golden_numpy
    for name, n, k, mu, a_max, values, seed, synth in EXACT_CASES:
        if name not in NUMPY_BACKEND_CASES:
            continue
        x, _ = exact_signal(n, k, seed, values, synth)
        for solver, fn in (("noniterative", OS.exact_noniterative),
                           ("iterative", OS.exact_iterative)):
            entries, tr = fn(x, k, mu, a_max, kernels="numpy")
            _check_entries(entries, arrays, f"{name}/{solver}")
            for key in ("full_success", "warnings", "unresolved_bins"):
                assert tr[key] == meta["exact"][name][solver][key], (name, solver, key)
    for name, n, k, snr_db, seed, prune in GENERAL_CASES:
        if name not in NUMPY_BACKEND_GENERAL:
            continue
        x, _ = general_signal(n, k, snr_db, seed)
        entries, tr = OS.general(x, k, rng_seed=seed, prune=prune, kernels="numpy")
        _check_entries(entries, arrays, f"{name}/general")


def test_duplicate_overwrite_cases_present(golden):
    """The golden set holds iterative cases where the real reference warned
    'duplicate location' (exact.py:152-158): the overwrite path is pinned."""
    _, meta = golden
    dups = [n for n, rec in meta["exact"].items() if rec["iterative"]["warnings"]]
    assert len(dups) >= 3, dups
