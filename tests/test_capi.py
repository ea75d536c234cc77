"""CPU checks of the drop-in boundary (no GPU needed):

* libsfdt_b200.so builds for sm_100a, loads, and exports every symbol
  include/sfdt.h declares;
* the host twiddle table replays the reference's radix-2 recurrence: a
  radix-2 DIT evaluated with that table and gcc rounding (no FMA) is
  bit-identical to the reference FFT (oracle) -- the arithmetic the GPU FFT
  kernel performs;
* the Python mirror validates arguments exactly like the reference.
"""

import os
import re

import numpy as np
import pytest

from oracle import kernels as OK
from paper_1407_8315_b200 import _lib
from paper_1407_8315_b200.build import build
from paper_1407_8315_b200.exact import ExactConfig
from paper_1407_8315_b200.spectral import SparseSpectrum, as_signal

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def lib():
    build()
    return _lib.load()


def test_exports_every_header_symbol(lib):
    with open(os.path.join(ROOT, "include", "sfdt.h")) as fh:
        hdr = fh.read()
    declared = set(re.findall(r"\b(sfdt_[a-z0-9_]+)\s*\(", hdr))
    assert declared, "no declarations parsed"
    assert declared == set(_lib.EXPORTS), declared ^ set(_lib.EXPORTS)
    for name in declared:
        assert hasattr(lib, name), name
    assert lib.sfdt_version() >= 10000
    assert lib.sfdt_strerror(-1) == b"invalid argument"


def _twiddles(lib, n, inverse=False):
    out = np.empty(2 * (n - 1), dtype=np.float64)
    assert lib.sfdt_fft_twiddles(n, int(inverse), out.ctypes.data_as(_lib._vp)) == 0
    return out[0::2] + 1j * out[1::2]


def _fft_with_table(x, tw):
    """Radix-2 DIT exactly as k_fft_views runs it, in numpy float64 scalar
    ops (each product rounded separately = gcc complex multiply)."""
    n = x.size
    logn = n.bit_length() - 1
    rev = np.array([int(format(j, f"0{logn}b")[::-1], 2) if logn else 0 for j in range(n)])
    a = np.empty(n, dtype=np.complex128)
    a[rev] = x
    re, im = a.real.copy(), a.imag.copy()
    h = 1
    while h < n:
        w = tw[h - 1: 2 * h - 1]
        idx = np.arange(n // 2)
        k = idx & (h - 1)
        i0 = ((idx >> (h.bit_length() - 1)) << h.bit_length()) + k
        i1 = i0 + h
        wr, wi = w.real[k], w.imag[k]
        tr = re[i1] * wr - im[i1] * wi
        ti = re[i1] * wi + im[i1] * wr
        ur, ui = re[i0].copy(), im[i0].copy()
        re[i0], im[i0] = ur + tr, ui + ti
        re[i1], im[i1] = ur - tr, ui - ti
        h *= 2
    return re + 1j * im


@pytest.mark.parametrize("n", [2, 4, 16, 256, 512, 1024, 4096])
def test_twiddle_table_reproduces_reference_fft(lib, n):
    rng = np.random.default_rng(n)
    x = rng.standard_normal(n) + 1j * rng.standard_normal(n)
    for inverse in (False, True):
        tw = _twiddles(lib, 8192, inverse)        # one table serves every n <= n_max
        got = _fft_with_table(x, tw)
        want = OK.fft_radix2(x, inverse)
        assert np.array_equal(got.view(np.uint64), want.view(np.uint64))


def test_config_validation_mirrors_reference():
    with pytest.raises(ValueError, match="power of two"):
        ExactConfig(n=12, k=2)
    with pytest.raises(ValueError, match="a_max"):
        ExactConfig(n=16, k=2, a_max=5)
    with pytest.raises(ValueError, match="mu"):
        ExactConfig(n=16, k=2, mu=3)
    with pytest.raises(ValueError, match="either k or initial_d"):
        ExactConfig(n=16)
    with pytest.raises(ValueError, match="must divide"):
        ExactConfig(n=16, initial_d=3)
    assert ExactConfig(n=1 << 20, k=256).resolved_d() == 1024
    assert ExactConfig(n=1 << 16, k=64).resolved_d() == 256
    assert ExactConfig(n=64, k=64).resolved_d() == 1
    assert ExactConfig(n=1 << 24, k=4096, mu=1).resolved_d() == 4096
    with pytest.raises(ValueError):
        as_signal(np.zeros((2, 4)))
    with pytest.raises(ValueError):
        as_signal(np.zeros(6))
    with pytest.raises(ValueError):
        SparseSpectrum(4, {7: 1.0})


def test_exact_workspace_query(lib):
    a = _lib.ExactArgs()
    a.batch, a.n, a.d, a.a_max, a.iterative, a.x_dtype = 16, 1 << 16, 256, 4, 0, 0
    assert lib.sfdt_exact_workspace_bytes(a) > 16 * 256 * 8 * 16
    a.d = 3
    assert lib.sfdt_exact_workspace_bytes(a) == 0


def test_tuning_struct_and_validation():
    """Design switches arrive as an sfdt_tuning (no environment reads in the
    library): the library's defaults equal the Python mirror's, unknown keys
    are rejected, and invalid values fail the plan before any launch."""
    import ctypes
    from paper_1407_8315_b200 import _lib
    lib = _lib.load()
    t = _lib.Tuning()
    lib.sfdt_default_tuning(ctypes.byref(t))
    for name, _ in _lib.Tuning._fields_:
        assert getattr(t, name) == _lib.TUNING_DEFAULTS[name], name
    with pytest.raises(KeyError):
        with _lib.tuning(no_such_switch=1):
            pass
    with _lib.tuning(gen_deal=3):
        assert _lib.current_tuning()["gen_deal"] == 3
    assert _lib.current_tuning()["gen_deal"] == _lib.TUNING_DEFAULTS["gen_deal"]
    a = _lib.GeneralArgs()
    a.batch, a.n, a.k, a.d, a.a_max, a.r_eff, a.keep_per_collision = 1, 1 << 12, 8, 16, 3, 9, 2
    cap = _lib._i64()
    assert lib.sfdt_general_caps(ctypes.byref(a), ctypes.byref(cap)) == 0
    bad = _lib.tuning_struct(dict(_lib.TUNING_DEFAULTS, gen_mf_list=5))
    a.tuning = ctypes.addressof(bad)
    assert lib.sfdt_general_caps(ctypes.byref(a), ctypes.byref(cap)) == -1


def test_library_reads_no_environment():
    """the product library reads no environment variables."""
    import glob
    import os
    root = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "paper_1407_8315_b200", "csrc")
    for path in glob.glob(os.path.join(root, "*")):
        with open(path) as fh:
            assert "getenv" not in fh.read(), path
