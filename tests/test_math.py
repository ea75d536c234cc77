"""The device math (paper_1407_8315_b200/csrc/cx.cuh) compiled for the host
must round exactly like the reference: gcc C99 complex ops, libgcc
__divdc3, glibc csqrt/cpow, numpy's complex multiply/divide, and the
composite Hankel / closed-form root / Vandermonde kernels of _core.pyx.

On the host every transcendental is glibc, so equality is bit-for-bit; on the
B200 the same source uses CUDA libm for hypot/atan2/log/exp/sincos (ulp-level
differences, covered by the GPU parity tolerances)."""

import ctypes
import os
import subprocess

import numpy as np
import pytest

from oracle import kernels as OK

HERE = os.path.dirname(os.path.abspath(__file__))
BUILD = os.path.join(HERE, "native", "_build")


@pytest.fixture(scope="module")
def libs():
    os.makedirs(BUILD, exist_ok=True)
    hm = os.path.join(BUILD, "hostmath.so")
    hr = os.path.join(BUILD, "hostref.so")
    subprocess.run(["g++", "-O2", "-fPIC", "-shared", "-ffp-contract=off", "-o", hm,
                    os.path.join(HERE, "native", "hostmath.cpp"), "-lm"], check=True)
    subprocess.run(["gcc", "-O3", "-fPIC", "-shared", "-ffp-contract=off", "-o", hr,
                    os.path.join(HERE, "native", "hostref.c"), "-lm"], check=True)
    return ctypes.CDLL(hm), ctypes.CDLL(hr)


def _p(a):
    return a.ctypes.data_as(ctypes.c_void_p)


def _call(f, n, *args):
    out = np.empty(n, np.complex128)
    f(*[_p(a) for a in args], _p(out), ctypes.c_int64(n))
    return out


def _same(x, y):
    return np.array_equal(np.ascontiguousarray(x).view(np.uint64),
                          np.ascontiguousarray(y).view(np.uint64))


def _rand(rng, n, span):
    z = (rng.standard_normal(n) + 1j * rng.standard_normal(n)) * np.exp(rng.uniform(-span, span, n))
    z[: n // 20] = z[: n // 20].real
    z[n // 20: n // 10] = 1j * z[n // 20: n // 10].imag
    z[n // 10: n // 5] = np.exp(1j * rng.uniform(-4, 4, n // 10)) * (1 + rng.uniform(-1e-3, 1e-3, n // 10))
    return z


def test_primitives_bitexact(libs):
    hm, hr = libs
    rng = np.random.default_rng(11)
    n = 200_000
    a, b = _rand(rng, n, 40), _rand(rng, n, 40)
    with np.errstate(all="ignore"):
        assert _same(_call(hm.hm_gmul, n, a, b), _call(hr.hr_mul, n, a, b))
        assert _same(_call(hm.hm_gdiv, n, a, b), _call(hr.hr_div, n, a, b))
        assert _same(_call(hm.hm_nmul, n, a, b), a * b)
        assert _same(_call(hm.hm_ndiv, n, a, b), a / b)
        assert _same(_call(hm.hm_gsqrt, n, a), _call(hr.hr_sqrt, n, a))
        c = _rand(rng, n, 3)
        assert _same(_call(hm.hm_gcbrt, n, c), _call(hr.hr_cbrt, n, c))


@pytest.mark.parametrize("a", [1, 2, 3, 4])
def test_decode_composites_bitexact(libs, a):
    hm, _ = libs
    rng = np.random.default_rng(100 + a)
    nb = 4000
    rnd = rng.standard_normal((nb, 8)) + 1j * rng.standard_normal((nb, 8))
    roots = np.exp(2j * np.pi * rng.integers(0, 4096, (nb, a)) / 4096)
    vals = rng.standard_normal((nb, a)) + 1j * rng.standard_normal((nb, a))
    tru = np.stack([np.sum(vals * roots ** l, axis=1) for l in range(8)], axis=1)
    m = np.ascontiguousarray(np.concatenate([rnd, tru]))
    nb = m.shape[0]
    c, cd = np.zeros((nb, a), complex), np.zeros(nb, complex)
    hm.hm_hankel(_p(m), ctypes.c_int64(nb), ctypes.c_int64(8), ctypes.c_int(a), _p(c), _p(cd))
    c2, cd2 = OK.hankel_solve(m, a)
    assert _same(c, c2) and _same(cd, cd2)
    z = np.zeros((nb, a), complex)
    hm.hm_roots(_p(c), ctypes.c_int64(nb), ctypes.c_int(a), _p(z))
    assert _same(z, OK.poly_roots(c))
    p, pd = np.zeros((nb, a), complex), np.zeros(nb, complex)
    hm.hm_vand(_p(z), _p(m), ctypes.c_int64(nb), ctypes.c_int(a), ctypes.c_int64(8), _p(p), _p(pd))
    p2, pd2 = OK.vandermonde_solve(z, m)
    assert _same(p, p2) and _same(pd, pd2)
