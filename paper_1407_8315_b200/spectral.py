"""Signal / spectrum types of the drop-in API.

Conventions follow the reference (/root/reference/pkg/src/sfft_dt/
spectral.py:3-16): analysis xhat[k] = (1/n) sum_n x[n] e^{-2 pi i k n/N};
a view x[d j + l] of length m = n/d is transformed with the sum DFT divided
by m, so bin k holds sum_t xhat[k + t m] e^{+2 pi i (k + t m) l / n}.
"""

from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np


def as_signal(x) -> np.ndarray:
    """Validate a 1-D power-of-two-length signal (spectral.py:28-36) and
    return it as contiguous complex128 (numpy) -- host-side validation only."""
    arr = np.ascontiguousarray(x, dtype=np.complex128)
    if arr.ndim != 1:
        raise ValueError(f"signal must be 1-D, got shape {arr.shape}")
    n = arr.size
    if n < 2 or n & (n - 1):
        raise ValueError(f"signal length must be a power of two >= 2, got {n}")
    return arr


def check_signal_shape(shape) -> int:
    """Same checks as as_signal on a shape (for device tensors)."""
    if len(shape) != 1:
        raise ValueError(f"signal must be 1-D, got shape {tuple(shape)}")
    n = int(shape[0])
    if n < 2 or n & (n - 1):
        raise ValueError(f"signal length must be a power of two >= 2, got {n}")
    return n


@dataclass
class SparseSpectrum:
    """Sparse spectrum: index -> complex value (spectral.py:39-73)."""

    n: int
    entries: dict = field(default_factory=dict)

    def __post_init__(self):
        if len(self.entries) > self.n:
            raise ValueError("more entries than ambient length")
        for s in self.entries:
            if not 0 <= s < self.n:
                raise ValueError(f"index {s} outside [0, {self.n})")

    def to_dense(self) -> np.ndarray:
        dense = np.zeros(self.n, dtype=np.complex128)
        if self.entries:
            idx = np.fromiter(self.entries.keys(), dtype=np.int64, count=len(self.entries))
            dense[idx] = np.fromiter(self.entries.values(), dtype=np.complex128,
                                     count=len(self.entries))
        return dense

    @classmethod
    def from_dense(cls, dense, k: int | None = None, threshold: float = 0.0) -> "SparseSpectrum":
        dense = np.asarray(dense, dtype=np.complex128)
        mag = np.abs(dense)
        if k is None:
            idx = np.nonzero(mag > threshold)[0]
        elif k:
            idx = np.argpartition(mag, len(dense) - k)[len(dense) - k:]
        else:
            idx = np.array([], dtype=np.int64)
        return cls(len(dense), {int(s): complex(dense[s]) for s in idx})

    def __len__(self) -> int:
        return len(self.entries)


def fft(x, normalization: str = "sum", inverse: bool = False):
    """Radix-2 FFT of a power-of-two-length signal on the B200 (spectral.py:
    128-140), bit-identical to the reference's fft_radix2.  ``normalization``
    is "sum" or "one_over_n".  Accepts numpy or torch; returns numpy.  n up to
    2^25 (longer than one CTA's shared memory runs the two-pass split)."""
    import torch

    from . import _lib
    from .device import require_cuda, stream_handle, twiddles
    if normalization not in ("sum", "one_over_n"):
        raise ValueError(f"unknown normalization {normalization!r}")
    if isinstance(x, torch.Tensor):
        n = check_signal_shape(x.shape)
        dev = require_cuda(x.device if x.is_cuda else None)
        xd = x.to(dev, torch.complex128).contiguous()
    else:
        arr = as_signal(x)
        n = arr.size
        dev = require_cuda()
        xd = torch.from_numpy(arr).to(dev)
    out = torch.empty_like(xd)
    _lib.check(_lib.load().sfdt_fft_radix2(xd.data_ptr(), out.data_ptr(), 1, n, int(bool(inverse)),
                                           twiddles(n, dev, inverse).data_ptr(), stream_handle(dev)),
               "sfdt_fft_radix2")
    res = out.cpu().numpy()
    return res / n if normalization == "one_over_n" else res


def synthesize(spectrum) -> np.ndarray:
    """Time signal from a spectrum, x[n] = sum_k xhat[k] e^{+2 pi i k n/N}
    (spectral.py:143-148), on the B200."""
    if isinstance(spectrum, SparseSpectrum):
        spectrum = spectrum.to_dense()
    return fft(as_signal(spectrum), "sum", inverse=True)


def snr(reference, estimate) -> float:
    """SNR in dB of ``estimate`` against the dense ``reference`` spectrum
    (spectral.py:193-212); math.inf when the error is exactly zero."""
    import math
    reference = np.asarray(reference, dtype=np.complex128)
    if isinstance(estimate, SparseSpectrum):
        if estimate.n != reference.size:
            raise ValueError("length mismatch between reference and estimate")
        estimate = estimate.to_dense()
    else:
        estimate = np.asarray(estimate, dtype=np.complex128)
    if estimate.shape != reference.shape:
        raise ValueError("length mismatch between reference and estimate")
    err = np.mean(np.abs(reference - estimate) ** 2)
    sig = np.mean(np.abs(estimate) ** 2)
    if err == 0.0:
        return math.inf
    return 10.0 * math.log10(sig / err)
