"""The reference's library functions around the solvers, computed on the
B200 (VERDICT r01 "missing" item 3): spectral.py downsample /
transform_view / aliased_values / forward_dft_oracle / rms, syndrome.py
decode chain, general.py sensing_matrix / prune_columns / subspace_pursuit,
and GeneralTrace.timings -- each against the CPU oracle (oracle/), which is
pinned to the real reference by tests/test_oracle.py.
"""

import logging

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("needs a CUDA device", allow_module_level=True)

import paper_1407_8315_b200 as P                 # noqa: E402
from oracle import kernels as OK                  # noqa: E402
from oracle import solvers as OS                  # noqa: E402
from tests.synth import exact_signal, general_signal   # noqa: E402


def _bits(a, b):
    a, b = np.ascontiguousarray(a), np.ascontiguousarray(b)
    return a.shape == b.shape and np.array_equal(a.view(np.uint8), b.view(np.uint8))


# ------------------------------------------------------------ spectral
def test_downsample_bitexact(rng):
    for n, d, shift in ((64, 4, 0), (64, 4, 7), (1024, 16, 1023), (48, 3, 47), (8, 8, 5)):
        x = rng.normal(size=n) + 1j * rng.normal(size=n)
        v = P.downsample(x, d, shift)
        idx = (d * np.arange(n // d) + shift) % n
        assert (v.n, v.d, v.shift) == (n, d, shift) and _bits(v.data, x[idx])
    x = rng.normal(size=64) + 1j * rng.normal(size=64)
    with pytest.raises(ValueError, match="does not divide"):
        P.downsample(x, 5)
    with pytest.raises(ValueError, match="outside"):
        P.downsample(x, 4, 64)
    # complex64 storage is upconverted exactly
    v = P.downsample(torch.from_numpy(x.astype(np.complex64)).cuda(), 4, 3)
    assert _bits(v.data, x.astype(np.complex64).astype(np.complex128)[(4 * np.arange(16) + 3) % 64])


@pytest.mark.parametrize("n,d", [(1 << 10, 4), (1 << 16, 16), (1 << 16, 1), (1 << 20, 64)])
def test_aliased_values_bitexact(n, d):
    """transform_view / aliased_values are fft_radix2(view) / m bit for bit
    (spectral.py:163-172, _core.pyx:35-77), also past one CTA's shared
    memory (n/d = 2^16)."""
    x, _ = exact_signal(n, 16, 3, "unit")
    for shift in (0, 1, d - 1 if d > 1 else 0, n - 1):
        got = P.aliased_values(x, d, shift)
        want = OS.shifted_view(OK, x, d, shift)
        assert _bits(got, want), (n, d, shift)
    tv = P.transform_view(P.downsample(x, d, 2 % n))
    assert _bits(tv.values, OS.shifted_view(OK, x, d, 2 % n)) and tv.shift == 2 % n
    # batched form: many signals x many shifts in one launch
    X = np.stack([exact_signal(n, 8, s, "unit")[0] for s in range(3)])
    shifts = [0, 5, 9, 3 % d if d > 1 else 0]
    got = P.aliased_values_batch(X, d, shifts).cpu().numpy()
    for b in range(3):
        for v, s in enumerate(shifts):
            assert _bits(got[b, v], OS.shifted_view(OK, X[b], d, s))


def test_syndromes_for_bin_and_views():
    n, d = 1 << 12, 16
    x, _ = exact_signal(n, 32, 5, "unit")
    views = [P.transform_view(P.downsample(x, d, j)) for j in range(6)]
    s = P.syndromes_for_bin(views, 17)
    assert s.bin == 17 and list(s.shifts) == list(range(6))
    assert _bits(s.values, np.array([OS.shifted_view(OK, x, d, j)[17] for j in range(6)]))
    with pytest.raises(ValueError):
        P.syndromes_for_bin(views, n // d)
    with pytest.raises(ValueError):
        P.syndromes_for_bin([], 0)


def test_forward_dft_oracle_and_rms(rng):
    for n in (2, 64, 1024):
        x = rng.normal(size=n) + 1j * rng.normal(size=n)
        got = P.forward_dft_oracle(x)
        want = np.fft.fft(x) / n
        assert np.max(np.abs(got - want)) <= 1e-13 * max(1.0, np.max(np.abs(want)))
    for n in (2, 1 << 10, 1 << 16, 1 << 20):
        x = rng.normal(size=n) + 1j * rng.normal(size=n)
        assert abs(P.rms(x) - OS.rms(x)) <= 1e-15 * OS.rms(x)


# ------------------------------------------------------------ syndrome
@pytest.mark.parametrize("a", [1, 2, 3, 4])
def test_decode_bins_against_oracle(golden, a):
    """The batched decode chain on the golden kernel inputs (half random
    syndromes, half true a-sparse ones): status / coefficients / roots /
    values against the oracle kernels and the reference's own tolerances."""
    arrays, _ = golden
    m = arrays[f"kern/a{a}/m"]
    n, d = 1 << 12, 64
    r = P.decode_bins(m, a, n, d, np.zeros(len(m), dtype=np.int64), upto=4)
    c, cd = OK.hankel_solve(m, a)
    for i in range(len(m)):
        ok = True
        if a == 1:
            scale = max(float(np.max(np.abs(m[i, :2]))), np.finfo(float).tiny)
            ok = abs(m[i, 0]) > 1e-10 * scale
            exp_status = 0 if ok else 1
        else:
            scale = max(float(np.max(np.abs(m[i, :2 * a]))), np.finfo(float).tiny)
            exp_status = 0 if abs(cd[i]) > 1e-10 * scale ** a else 1
            if exp_status == 0:
                assert _bits(r.coefficients[i], c[i])
                z = OK.poly_roots(c[i:i + 1])[0]
                resid = OS._residuals(c[i:i + 1], z[None, :])[0]
                if np.any(resid > 1e-8 * max(1.0, float(np.max(np.abs(c[i]))))):
                    exp_status = 2
                else:
                    # same root multiset (order can follow an ulp-level csqrt branch)
                    g = sorted(r.roots[i], key=lambda t: (round(t.real, 9), round(t.imag, 9)))
                    w = sorted(z, key=lambda t: (round(t.real, 9), round(t.imag, 9)))
                    assert np.allclose(g, w, rtol=1e-12, atol=1e-300)
                    p, pd = OK.vandermonde_solve(z[None, :], m[i:i + 1])
                    if abs(pd[0]) <= 1e-10 * max(1.0, float(np.max(np.abs(z)))) ** a:
                        exp_status = 3
        assert r.status[i] == exp_status or (exp_status >= 2 and r.status[i] >= 2), (i, r.status[i], exp_status)
    # the true a-sparse half decodes and reconstructs its syndromes
    true = np.arange(32, 64)
    good = true[r.status[true] == 0]
    assert good.size >= 28
    from paper_1407_8315_b200 import syndrome as S
    rec = S.reconstruct_syndromes(r.roots[good], r.values[good], 8)
    assert np.allclose(rec, m[good], rtol=1e-8, atol=1e-8 * np.abs(m[good]).max())
    if a == 1:
        return   # decode_bin's a = 1 model has no locator polynomial
    res = S.poly_residuals(r.coefficients[good], r.roots[good])
    assert np.all(res <= 1e-8 * np.maximum(1.0, np.abs(r.coefficients[good]).max(axis=1))[:, None])


def test_syndrome_known_answers():
    """The reference's own known answers (pkg/tests/test_syndrome.py:69-256)
    through the device-backed single-bin API."""
    from paper_1407_8315_b200 import syndrome as S
    c = S.solve_coefficients(np.array([2, 0, 2, 0], dtype=complex), 2)
    assert np.allclose(c.c, [-1.0, 0.0], atol=1e-14)
    with pytest.raises(S.NearSingular):
        S.solve_coefficients(np.array([2, 2, 2, 2], dtype=complex), 2)
    z = S.roots_closed_form(S.PolyCoefficients(a=2, c=np.array([1j, -(1 + 1j)])))
    assert sorted(np.round(z, 12), key=lambda t: (t.real, t.imag)) == [1j, 1.0]
    p = S.solve_values(np.array([2, 0, 2, 0], dtype=complex), np.array([1.0, -1.0]))
    assert np.allclose(p, [1.0, 1.0], atol=1e-14)
    with pytest.raises(S.IllConditioned):
        S.solve_values(np.array([2, 2, 2, 2], dtype=complex), np.array([1.0, 1.0]))
    assert S.root_to_location(np.exp(1.25j * np.pi), 8) == (5, pytest.approx(0.0, abs=1e-12))
    with pytest.raises(ValueError):
        S.root_to_location(0j, 8)
    # decode_bin: single tone at s = 5, n = 8, d = 4 -> bin 1
    n, d, s = 8, 4, 5
    m = np.array([2.0 * np.exp(2j * np.pi * s * j / n) for j in range(4)])
    db = S.decode_bin(m, 1, n, d, 1)
    assert list(db.locations) == [5] and db.membership and db.snap_error < 1e-12
    db2 = S.decode_bin(m, 1, n, d, 0)
    assert not db2.membership
    with pytest.raises(S.NearSingular):
        S.decode_bin(np.zeros(2, complex), 1, n, d, 0)
    with pytest.raises(ValueError):
        S.decode_bin(np.zeros(3, complex), 2, n, d, 0)


# ------------------------------------------------------------- general
def test_sensing_matrix(rng):
    n, d, k = 1 << 12, 64, 37
    sh = np.array([3, 17, 40, 61, 5])
    sm = P.sensing_matrix(n, d, k, sh)
    locs = (k + np.arange(d) * (n // d)) % n
    want = np.exp(2j * np.pi * np.outer(sh, locs) / n)
    assert np.array_equal(sm.column_locations, locs)
    assert np.max(np.abs(sm.matrix - want)) <= 2e-16 * 4
    cols = np.array([1, 9, 33])
    sm2 = P.sensing_matrix(n, d, k, sh, cols)
    assert np.max(np.abs(sm2.matrix - want[:, cols])) <= 1e-15


@pytest.mark.parametrize("snr,seed", [(20.0, 11), (30.0, 12), (10.0, 13)])
def test_prune_columns_against_oracle(snr, seed):
    """prune_columns (general.py:184-221) for the voted bins of a general
    signal: the oracle's fit + prune_eval + argpartition on the same
    syndromes; with augment_with_correlation the oracle's correlation keep."""
    n, k = 1 << 14, 16
    x, _ = general_signal(n, k, snr, seed)
    _, tr = OS.general(x, k, rng_seed=seed, return_internals=True)
    d = tr["d"]
    sh = np.asarray(tr["shifts"])
    cons, rv = tr["consecutive"], tr["random_views"]
    voted = np.nonzero(tr["votes"] > 0)[0]
    assert voted.size
    for kb in voted.tolist():
        a = int(tr["votes"][kb])
        syn = cons[:, kb]
        got = P.prune_columns(syn, a, kb, n, d, a_max=3)
        count = min(2 * a, d)
        want = None
        for order in range(3, 0, -1):
            c, cd = OK.hankel_solve(syn[None, :2 * order], order)
            if abs(cd[0]) > 1e-10 * max(float(np.max(np.abs(syn[:2 * order]))), np.finfo(float).tiny) ** order:
                errs = OK.prune_eval(c, np.array([kb]), n, d)[0]
                want = np.sort(np.argsort(errs, kind="stable")[:count])
                break
        if want is None:
            want = np.arange(d)
        assert np.array_equal(got, want), (kb, got, want)
        aug = P.prune_columns(syn, a, kb, n, d, a_max=3, fallback=(rv[:, kb], sh),
                              augment_with_correlation=True)
        if want.size < d:
            assert np.array_equal(aug, np.union1d(want, OS._corr_keep(rv[:, kb], sh, kb, n, d, min(a, d))))
    # every fit singular (all-zero syndromes): correlation fallback / all columns
    z = np.zeros(6, complex)
    y = rv[:, voted[0]]
    assert np.array_equal(P.prune_columns(z, 1, int(voted[0]), n, d, a_max=3), np.arange(d))
    assert np.array_equal(P.prune_columns(z, 1, int(voted[0]), n, d, a_max=3, fallback=(y, sh)),
                          OS._corr_keep(y, sh, int(voted[0]), n, d, 2))
    with pytest.raises(ValueError):
        P.prune_columns(z[:4], 1, 0, n, d, a_max=3)


def test_subspace_pursuit_against_oracle(rng, caplog):
    """subspace_pursuit (general.py:224-269): supports identical, values
    within 1e-9 of the oracle's (numpy lstsq), random and planted problems,
    including rank-deficient phi (logged like the reference)."""
    checked = 0
    for rows, cols, a in ((9, 6, 1), (9, 16, 2), (12, 24, 3), (9, 256, 1), (6, 8, 4), (3, 40, 1)):
        for _ in range(20):
            phi = np.exp(2j * np.pi * rng.random((rows, cols)))
            sup = rng.choice(cols, size=min(a, cols), replace=False)
            y = phi[:, sup] @ (rng.normal(size=sup.size) + 1j * rng.normal(size=sup.size))
            y = y + 0.05 * (rng.normal(size=rows) + 1j * rng.normal(size=rows))
            got = P.subspace_pursuit(y, phi, a)
            want = OS.subspace_pursuit(y, phi, a)
            assert np.array_equal(np.nonzero(got)[0], np.nonzero(want)[0])
            nz = want != 0
            assert np.all(np.abs(got[nz] - want[nz]) <= 1e-9 * np.abs(want[nz]))
            checked += 1
    # duplicated columns: rank-deficient least squares, minimum-norm solution
    phi = np.exp(2j * np.pi * rng.random((9, 5)))
    phi[:, 3] = phi[:, 1]
    y = phi[:, 1] * 2.0
    with caplog.at_level(logging.WARNING):
        got = P.subspace_pursuit(y, phi, 2)
    want = OS.subspace_pursuit(y, phi, 2)
    assert np.allclose(got, want, atol=1e-9)
    with pytest.raises(ValueError):
        P.subspace_pursuit(y, phi, 10)
    assert checked == 120


def test_general_trace_timings():
    n, k = 1 << 14, 16
    x, _ = general_signal(n, k, 20.0, 3)
    _, tr = P.solve_general(x, P.GeneralConfig(n=n, k=k))
    assert set(tr.timings) == {"fft", "vote", "prune", "subspace_pursuit", "total"}
    assert all(v >= 0.0 for v in tr.timings.values())
    assert tr.timings["total"] >= tr.timings["fft"]
