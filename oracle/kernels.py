"""TEST INFRASTRUCTURE ONLY -- numpy-facing wrapper of the oracle C kernels.

Same six functions and signatures as the reference's backend seam
(/root/reference/pkg/src/sfft_dt/_kernels/__init__.py:19-24):

    fft_radix2(x, inverse=False)          _core.pyx:35-77
    hankel_solve(m, a) -> (c, cd)         _core.pyx:127-162
    poly_roots(c)                         _core.pyx:238-266
    vandermonde_solve(z, m) -> (p, pd)    _core.pyx:273-312
    prune_eval(c, k, n, d)                _core.pyx:319-346
    hankel_singular_values(m, a_max)      _core.pyx:409-433

`backend("port")` returns these; `backend("reference")` returns the
reference's own compiled `_core` built into oracle/_ref by `make ref`
(used to pin the port and as the CPU baseline when present).
Only tests/, __graft_entry__.smoke() and bench.py's CPU legs import this.
"""

from __future__ import annotations

import ctypes
import glob
import importlib.util
import os
import subprocess
import types

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB_PATH = os.path.join(_HERE, "_build", "liboracle_kernels.so")
_lib = None

_c128p = np.ctypeslib.ndpointer(np.complex128, flags="C_CONTIGUOUS")
_f64p = np.ctypeslib.ndpointer(np.float64, flags="C_CONTIGUOUS")
_i64p = np.ctypeslib.ndpointer(np.int64, flags="C_CONTIGUOUS")
_i64 = ctypes.c_int64
_int = ctypes.c_int


def build(force: bool = False) -> str:
    """Compile kernels.c with the reference's arithmetic flags (make)."""
    if force or not os.path.exists(_LIB_PATH) or (
            os.path.getmtime(_LIB_PATH) < os.path.getmtime(os.path.join(_HERE, "kernels.c"))):
        subprocess.run(["make", "-s", "-C", _HERE, "all"], check=True)
    return _LIB_PATH


def _load():
    global _lib
    if _lib is None:
        lib = ctypes.CDLL(build())
        lib.orc_fft_radix2.argtypes = [_c128p, _c128p, _i64, _int]
        lib.orc_fft_radix2.restype = _int
        lib.orc_hankel_solve.argtypes = [_c128p, _i64, _i64, _int, _c128p, _c128p]
        lib.orc_poly_roots.argtypes = [_c128p, _i64, _int, _c128p]
        lib.orc_vandermonde_solve.argtypes = [_c128p, _c128p, _i64, _int, _i64, _c128p, _c128p]
        lib.orc_prune_eval.argtypes = [_c128p, _i64p, _i64, _int, _i64, _i64, _f64p]
        lib.orc_hankel_singular_values.argtypes = [_c128p, _i64, _i64, _int, _f64p]
        for f in (lib.orc_hankel_solve, lib.orc_poly_roots, lib.orc_vandermonde_solve,
                  lib.orc_prune_eval, lib.orc_hankel_singular_values):
            f.restype = None
        _lib = lib
    return _lib


def fft_radix2(x, inverse: bool = False) -> np.ndarray:
    x = np.array(x, dtype=np.complex128, copy=True, order="C").ravel()
    out = np.empty_like(x)
    if x.size == 0 or _load().orc_fft_radix2(x, out, x.size, int(bool(inverse))) != 0:
        raise ValueError(f"length must be a power of two, got {x.size}")
    return out


def hankel_solve(m, a: int):
    m = np.ascontiguousarray(m, dtype=np.complex128)
    if not 1 <= a <= 4:
        raise ValueError(f"collision count must be 1..4, got {a}")
    if m.shape[1] < 2 * a:
        raise ValueError(f"need at least {2 * a} syndromes, got {m.shape[1]}")
    nb = m.shape[0]
    c = np.zeros((nb, a), dtype=np.complex128)
    cd = np.empty(nb, dtype=np.complex128)
    if nb:
        _load().orc_hankel_solve(m, nb, m.shape[1], a, c, cd)
    return c, cd


def poly_roots(c) -> np.ndarray:
    c = np.ascontiguousarray(c, dtype=np.complex128)
    a = c.shape[1]
    if not 1 <= a <= 4:
        raise ValueError(f"degree must be 1..4, got {a}")
    z = np.empty_like(c)
    if c.shape[0]:
        _load().orc_poly_roots(c, c.shape[0], a, z)
    return z


def vandermonde_solve(z, m):
    z = np.ascontiguousarray(z, dtype=np.complex128)
    m = np.ascontiguousarray(m, dtype=np.complex128)
    nb, a = z.shape
    p = np.zeros((nb, a), dtype=np.complex128)
    pd = np.empty(nb, dtype=np.complex128)
    if nb:
        _load().orc_vandermonde_solve(z, m, nb, a, m.shape[1], p, pd)
    return p, pd


def prune_eval(c, k, n: int, d: int) -> np.ndarray:
    c = np.ascontiguousarray(c, dtype=np.complex128)
    k = np.ascontiguousarray(k, dtype=np.int64)
    out = np.empty((c.shape[0], d), dtype=np.float64)
    if c.shape[0]:
        _load().orc_prune_eval(c, k, c.shape[0], c.shape[1], int(n), int(d), out)
    return out


def hankel_singular_values(m, a_max: int) -> np.ndarray:
    m = np.ascontiguousarray(m, dtype=np.complex128)
    if m.shape[1] < 2 * a_max - 1:
        raise ValueError(f"need {2 * a_max - 1} syndromes, got {m.shape[1]}")
    if not 1 <= a_max <= 4:
        raise ValueError(f"a_max must be 1..4, got {a_max}")
    out = np.empty((m.shape[0], a_max), dtype=np.float64)
    if m.shape[0]:
        _load().orc_hankel_singular_values(m, m.shape[0], m.shape[1], a_max, out)
    return out


_PORT = types.SimpleNamespace(
    name="port", fft_radix2=fft_radix2, hankel_solve=hankel_solve, poly_roots=poly_roots,
    vandermonde_solve=vandermonde_solve, prune_eval=prune_eval,
    hankel_singular_values=hankel_singular_values)


def reference_core_path() -> str | None:
    hits = sorted(glob.glob(os.path.join(_HERE, "_ref", "_core*.so")))
    return hits[0] if hits else None


def build_reference() -> str | None:
    """`make ref` when /root/reference is present; returns the .so or None."""
    if os.path.isdir("/root/reference/pkg"):
        subprocess.run(["make", "-s", "-C", _HERE, "ref"], check=True)
    return reference_core_path()


_REF = None


def backend(kind: str = "port"):
    """Kernel namespace: "port" (oracle/kernels.c), "reference" (the
    reference's own compiled _core from oracle/_ref) or "numpy" (the
    restated pure-numpy backend, oracle/numpy_kernels.py: the reference's
    second backend, used to measure its own numerical envelope)."""
    global _REF
    if kind == "port":
        return _PORT
    if kind == "numpy":
        from .numpy_kernels import BACKEND
        return BACKEND
    if kind != "reference":
        raise ValueError(kind)
    if _REF is None:
        path = reference_core_path()
        if path is None:
            raise FileNotFoundError("oracle/_ref/_core*.so not built (make -C oracle ref)")
        spec = importlib.util.spec_from_file_location("_core", path)
        mod = importlib.util.module_from_spec(spec)
        spec.loader.exec_module(mod)
        mod.name = "reference"
        _REF = mod
    return _REF
