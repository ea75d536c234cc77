"""The reference's kernel seam (`sfft_dt._kernels`, _kernels/__init__.py:19-24)
backed by the B200 library: same six functions, numpy in / numpy out, same
argument errors.  Each call moves its arrays to the GPU, runs one batched
sm_100a kernel and copies the result back -- the fine-grained seam the
reference dispatches through; the solver-level entry
points keep data in HBM and are the fast path.

    fft_radix2(x, inverse=False)          _core.pyx:35-77   bit-identical
    hankel_solve(m, a) -> (c, cd)         _core.pyx:127-162 bit-identical
    poly_roots(c)                         _core.pyx:238-266 (CUDA libm ulps)
    vandermonde_solve(z, m) -> (p, pd)    _core.pyx:273-312 bit-identical
    prune_eval(c, k, n, d)                _core.pyx:319-346 (CUDA sincos ulps)
    hankel_singular_values(m, a_max)      _core.pyx:409-433 (CUDA hypot ulps)
"""

from __future__ import annotations

import numpy as np
import torch

from . import _lib
from .device import require_cuda, stream_handle, twiddles

COMPILED = True


def _dev():
    return require_cuda()


def _c128(a, dev):
    return torch.from_numpy(np.ascontiguousarray(a, dtype=np.complex128)).to(dev)


def _host_c(t):
    return t.cpu().numpy()


def fft_radix2(x, inverse: bool = False) -> np.ndarray:
    x = np.array(x, dtype=np.complex128, copy=True, order="C").ravel()
    n = x.size
    if n == 0 or n & (n - 1):
        raise ValueError(f"length must be a power of two, got {n}")
    dev = _dev()
    xd = _c128(x, dev)
    out = torch.empty_like(xd)
    _lib.check(_lib.load().sfdt_fft_radix2(xd.data_ptr(), out.data_ptr(), 1, n, int(bool(inverse)),
                                           twiddles(max(n, 2), dev, inverse).data_ptr(),
                                           stream_handle(dev)), "fft_radix2")
    return _host_c(out)


def hankel_solve(m, a: int):
    m = np.ascontiguousarray(m, dtype=np.complex128)
    if not 1 <= a <= 4:
        raise ValueError(f"collision count must be 1..4, got {a}")
    if m.shape[1] < 2 * a:
        raise ValueError(f"need at least {2 * a} syndromes, got {m.shape[1]}")
    nb = m.shape[0]
    dev = _dev()
    md = _c128(m, dev)
    c = torch.zeros((nb, a), dtype=torch.complex128, device=dev)
    cd = torch.empty(nb, dtype=torch.complex128, device=dev)
    if nb:
        _lib.check(_lib.load().sfdt_hankel_solve(md.data_ptr(), nb, m.shape[1], a, c.data_ptr(),
                                                 cd.data_ptr(), stream_handle(dev)), "hankel_solve")
    return _host_c(c), _host_c(cd)


def poly_roots(c) -> np.ndarray:
    c = np.ascontiguousarray(c, dtype=np.complex128)
    a = c.shape[1]
    if not 1 <= a <= 4:
        raise ValueError(f"degree must be 1..4, got {a}")
    dev = _dev()
    cd = _c128(c, dev)
    z = torch.empty_like(cd)
    if c.shape[0]:
        _lib.check(_lib.load().sfdt_poly_roots(cd.data_ptr(), c.shape[0], a, z.data_ptr(),
                                               stream_handle(dev)), "poly_roots")
    return _host_c(z)


def vandermonde_solve(z, m):
    z = np.ascontiguousarray(z, dtype=np.complex128)
    m = np.ascontiguousarray(m, dtype=np.complex128)
    nb, a = z.shape
    dev = _dev()
    zd, md = _c128(z, dev), _c128(m, dev)
    p = torch.zeros((nb, a), dtype=torch.complex128, device=dev)
    pd = torch.empty(nb, dtype=torch.complex128, device=dev)
    if nb:
        _lib.check(_lib.load().sfdt_vandermonde_solve(zd.data_ptr(), md.data_ptr(), nb, a, m.shape[1],
                                                      p.data_ptr(), pd.data_ptr(), stream_handle(dev)),
                   "vandermonde_solve")
    return _host_c(p), _host_c(pd)


def prune_eval(c, k, n: int, d: int) -> np.ndarray:
    c = np.ascontiguousarray(c, dtype=np.complex128)
    k = np.ascontiguousarray(k, dtype=np.int64)
    nb = c.shape[0]
    dev = _dev()
    cd = _c128(c, dev)
    kd = torch.from_numpy(k).to(dev)
    out = torch.empty((nb, d), dtype=torch.float64, device=dev)
    if nb:
        _lib.check(_lib.load().sfdt_prune_eval(cd.data_ptr(), kd.data_ptr(), nb, c.shape[1], int(n),
                                               int(d), out.data_ptr(), stream_handle(dev)),
                   "prune_eval")
    return out.cpu().numpy()


def hankel_singular_values(m, a_max: int) -> np.ndarray:
    m = np.ascontiguousarray(m, dtype=np.complex128)
    if m.shape[1] < 2 * a_max - 1:
        raise ValueError(f"need {2 * a_max - 1} syndromes, got {m.shape[1]}")
    if not 1 <= a_max <= 4:
        raise ValueError(f"a_max must be 1..4, got {a_max}")
    nb = m.shape[0]
    dev = _dev()
    md = _c128(m, dev)
    out = torch.empty((nb, a_max), dtype=torch.float64, device=dev)
    if nb:
        _lib.check(_lib.load().sfdt_hankel_singular_values(md.data_ptr(), nb, m.shape[1], a_max,
                                                           out.data_ptr(), stream_handle(dev)),
                   "hankel_singular_values")
    return out.cpu().numpy()
