"""TEST INFRASTRUCTURE ONLY -- restatement of the reference's pure-numpy
kernel backend (/root/reference/pkg/src/sfft_dt/_kernels/_reference.py),
the second CPU backend the reference ships (selected there by
SFFT_DT_PURE_PYTHON=1, _kernels/__init__.py:11-17).

It computes the same six functions as the compiled `_core` with different
roundoff (table twiddles instead of the recurrence, LU determinants instead
of cofactors, numpy power instead of repeated products, LAPACK SVD instead of
Jacobi).  The parity tests use `backend("numpy")` to measure the reference's
OWN numerical envelope on an input (rule 3's per-entry bound
max(1e-9, 100 x |compiled - numpy backend|)): how far the two reference
backends already disagree on a value is the scale at which a third
implementation (the B200 kernels) may differ from the oracle.

Never imported by the product package.
"""

from __future__ import annotations

import types

import numpy as np

_CUBE_W = (-0.5 + 0.5j * np.sqrt(3.0), -0.5 - 0.5j * np.sqrt(3.0))   # _reference.py:21-22


def _bitrev(n: int) -> np.ndarray:
    bits = n.bit_length() - 1
    idx = np.arange(n)
    rev = np.zeros(n, dtype=np.intp)
    for b in range(bits):
        rev |= ((idx >> b) & 1) << (bits - 1 - b)
    return rev


def fft_radix2(x, inverse: bool = False) -> np.ndarray:
    """_reference.py:47-65: bit reversal, then per stage a twiddle TABLE
    exp(sign 2 pi i j / m), butterflies (u + w v, u - w v) vectorised over
    the blocks."""
    x = np.ascontiguousarray(x, dtype=np.complex128).ravel()
    n = x.size
    if n == 0 or n & (n - 1):
        raise ValueError(f"length must be a power of two, got {n}")
    if n == 1:
        return x.copy()
    sign = 1.0 if inverse else -1.0
    y = x[_bitrev(n)]
    half = 1
    while half < n:
        m = 2 * half
        w = np.exp(sign * 2j * np.pi * np.arange(half) / m)
        blocks = y.reshape(n // m, m)
        u = blocks[:, :half].copy()
        v = blocks[:, half:] * w
        blocks[:, :half] = u + v
        blocks[:, half:] = u - v
        half = m
    return y


def _cramer(mat: np.ndarray, rhs: np.ndarray, det: np.ndarray) -> np.ndarray:
    """Column-replacement determinants over LU (np.linalg.det), divided by
    det, zero rows where det == 0 (_reference.py:86-103, 221-233)."""
    nb, a, _ = mat.shape
    num = np.empty((nb, a), dtype=np.complex128)
    for j in range(a):
        mj = mat.copy()
        mj[:, :, j] = rhs
        num[:, j] = np.linalg.det(mj)
    out = num / np.where(det == 0, 1.0, det)[:, None]
    out[det == 0] = 0.0
    return out


def hankel_solve(m, a: int):
    """_reference.py:71-103: H_ij = m_{i+j}, rhs -m_{a..2a-1}, Cramer by LU."""
    m = np.asarray(m, dtype=np.complex128)
    if not 1 <= a <= 4:
        raise ValueError(f"collision count must be 1..4, got {a}")
    if m.shape[1] < 2 * a:
        raise ValueError(f"need at least {2 * a} syndromes, got {m.shape[1]}")
    h = m[:, np.arange(a)[:, None] + np.arange(a)[None, :]]
    cd = np.linalg.det(h)
    return _cramer(h, -m[:, a:2 * a], cd), cd


def _stable_pair(b, c):
    """Roots of z^2 + b z + c with the cancellation-free branch
    (_reference.py:112-121, 152-158)."""
    disc = np.sqrt(b * b - 4.0 * c)
    disc = np.where(np.real(np.conj(b) * disc) < 0.0, -disc, disc)
    q = -0.5 * (b + disc)
    other = np.where(q == 0, -0.5 * (b - disc), c / np.where(q == 0, 1.0, q))
    return q, other


def _cbrt_pair(g, h):
    """_reference.py:124-134: A = cbrt of the larger of g -/+ sqrt(g^2+h^3)
    (numpy principal power), B = -h/A (0 when A = 0)."""
    r = np.sqrt(g * g + h ** 3)
    lo, hi = g - r, g + r
    big = np.where(np.abs(lo) >= np.abs(hi), lo, hi)
    A = big ** (1.0 / 3.0)
    B = np.where(A == 0, 0.0, -h / np.where(A == 0, 1.0, A))
    return A, B


def poly_roots(c) -> np.ndarray:
    """_reference.py:188-206 (degree 1..4: negation, stable quadratic,
    Cardano, Ferrari with the A/B reconditioning of 160-185)."""
    c = np.asarray(c, dtype=np.complex128)
    a = c.shape[1]
    if a == 1:
        return -c
    if a == 2:
        return np.stack(_stable_pair(c[:, 1], c[:, 0]), axis=1)
    if a == 3:
        c0, c1, c2 = c[:, 0], c[:, 1], c[:, 2]
        g = c0 / 2.0 - c1 * c2 / 6.0 + c2 ** 3 / 27.0
        h = c1 / 3.0 - c2 ** 2 / 9.0
        A, B = _cbrt_pair(g, h)
        s = -c2 / 3.0
        w1, w2 = _CUBE_W
        return np.stack([s - A - B, s - w1 * A - w2 * B, s - w2 * A - w1 * B], axis=1)
    if a == 4:
        c0, c1, c2, c3 = c[:, 0], c[:, 1], c[:, 2], c[:, 3]
        g = (72.0 * c0 * c2 + 9.0 * c1 * c2 * c3 - 27.0 * c1 ** 2
             - 27.0 * c0 * c3 ** 2 - 2.0 * c2 ** 3) / 432.0
        h = (3.0 * c1 * c3 - 12.0 * c0 - c2 ** 2) / 36.0
        C, D = _cbrt_pair(g, h)
        y = c2 / 6.0 - C - D
        aa = np.sqrt(c3 * c3 / 4.0 - c2 + 2.0 * y)
        num = c3 * y - c1
        sa = 1.0 + np.abs(c3) ** 2 / 4.0 + np.abs(c2) + 2.0 * np.abs(y)
        sb = 1.0 + np.abs(y) ** 2 + np.abs(c0)
        a_ok = np.abs(aa) > 1e-6 * np.sqrt(sa)
        bs = np.sqrt(y * y - c0)
        b_ok = np.abs(bs) > 1e-6 * np.sqrt(sb)
        bb = np.where(a_ok, num / (2.0 * np.where(a_ok, aa, 1.0)), np.where(b_ok, bs, 0.0))
        aa = np.where(a_ok, aa, np.where(b_ok, num / (2.0 * np.where(b_ok, bs, 1.0)), 0.0))
        z0, z1 = _stable_pair(c3 / 2.0 + aa, y + bb)
        z2, z3 = _stable_pair(c3 / 2.0 - aa, y - bb)
        return np.stack([z0, z1, z2, z3], axis=1)
    raise ValueError(f"degree must be 1..4, got {a}")


def vandermonde_solve(z, m):
    """_reference.py:213-233: pd = prod_{i<j}(z_j - z_i) in loop order,
    V_ij = z_j ** i (numpy power), Cramer by LU."""
    z = np.asarray(z, dtype=np.complex128)
    m = np.asarray(m, dtype=np.complex128)
    nb, a = z.shape
    pd = np.ones(nb, dtype=np.complex128)
    for i in range(a):
        for j in range(i + 1, a):
            pd *= z[:, j] - z[:, i]
    v = z[:, None, :] ** np.arange(a)[None, :, None]
    return _cramer(v, m[:, :a], pd), pd


def prune_eval(c, k, n: int, d: int) -> np.ndarray:
    """_reference.py:240-251: |P(z_t)| at z_t = e^{2 pi i k/n} e^{2 pi i t/d}
    (table phases), Horner from the leading coefficient."""
    c = np.asarray(c, dtype=np.complex128)
    k = np.asarray(k)
    z = np.exp(2j * np.pi * (k.astype(np.float64) / n))[:, None] * \
        np.exp(2j * np.pi * np.arange(d) / d)[None, :]
    acc = np.ones_like(z)
    for j in range(c.shape[1] - 1, -1, -1):
        acc = acc * z + c[:, j, None]
    return np.abs(acc)


def hankel_singular_values(m, a_max: int) -> np.ndarray:
    """_reference.py:258-265: LAPACK singular values, descending."""
    m = np.asarray(m, dtype=np.complex128)
    if m.shape[1] < 2 * a_max - 1:
        raise ValueError(f"need {2 * a_max - 1} syndromes, got {m.shape[1]}")
    idx = np.arange(a_max)[:, None] + np.arange(a_max)[None, :]
    return np.linalg.svd(m[:, idx], compute_uv=False)


BACKEND = types.SimpleNamespace(
    name="numpy", fft_radix2=fft_radix2, hankel_solve=hankel_solve, poly_roots=poly_roots,
    vandermonde_solve=vandermonde_solve, prune_eval=prune_eval,
    hankel_singular_values=hankel_singular_values)
