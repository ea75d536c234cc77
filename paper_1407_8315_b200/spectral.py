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


@dataclass(frozen=True)
class DownsampleView:
    """Time-domain view data[j] = parent[(d*j + shift) mod n] (spectral.py:77-84)."""

    n: int
    d: int
    shift: int
    data: np.ndarray


@dataclass(frozen=True)
class AliasedSpectrum:
    """Scaled DFT of a downsampled view (spectral.py:87-95): bin k holds
    sum_t xhat[k + t m] e^{+2 pi i (k + t m) shift / n}, no 1/d factor."""

    n: int
    d: int
    shift: int
    values: np.ndarray


@dataclass(frozen=True)
class SyndromeSet:
    """One bin's shifted-view values m_j and the shifts used (spectral.py:98-107)."""

    bin: int
    values: np.ndarray
    shifts: np.ndarray

    def __post_init__(self):
        if len(self.values) != len(self.shifts):
            raise ValueError("values and shifts must have equal length")


def _device_signal(x, allow_c64=True):
    """(tensor on the GPU, n, dtype code) for a 1-D signal, without copying a
    complex128/complex64 CUDA tensor."""
    import torch

    from . import _lib
    from .device import require_cuda
    if isinstance(x, torch.Tensor):
        dev = require_cuda(x.device if x.is_cuda else None)
        t = x if x.dtype in (torch.complex128, torch.complex64) and allow_c64 else x.to(torch.complex128)
        t = t.to(dev).contiguous()
    else:
        arr = np.ascontiguousarray(x, dtype=np.complex128)
        dev = require_cuda()
        t = torch.from_numpy(arr).to(dev)
    code = _lib.SFDT_C64 if t.dtype == torch.complex64 else _lib.SFDT_C128
    return t, dev, code


def downsample(x, d: int, shift: int = 0) -> DownsampleView:
    """Time-domain downsample by factor d with shift l, indices mod n
    (spectral.py:151-160): one sfdt_downsample gather on the GPU."""
    import torch

    from . import _lib
    from .device import stream_handle
    t, dev, code = _device_signal(x)
    t = t.reshape(-1)
    n = t.numel()
    if d < 1 or n % d:
        raise ValueError(f"downsampling factor {d} does not divide {n}")
    if not 0 <= shift < n:
        raise ValueError(f"shift {shift} outside [0, {n})")
    out = torch.empty((n // d, 2), dtype=torch.float64, device=dev)
    sh = torch.tensor([int(shift)], dtype=torch.int64, device=dev)
    _lib.check(_lib.load().sfdt_downsample(t.data_ptr(), code, 1, n, int(d), sh.data_ptr(), 1, out.data_ptr(),
                                           stream_handle(dev)), "sfdt_downsample")
    return DownsampleView(n=n, d=int(d), shift=int(shift), data=out.cpu().numpy().view(np.complex128).ravel())


def aliased_values_batch(X, d: int, shifts):
    """Batched aliased spectra: out[b, v, :] = fft_radix2(x_b[(d j + s_v) mod n])
    / (n/d) for a (B, n) batch and a list of shifts -- the solvers' fused
    gather + FFT kernel (bit-identical to the reference's transform_view).
    Returns a (B, len(shifts), n/d) complex128 CUDA tensor."""
    import torch

    from . import _lib
    from .device import resolve_workspace, stream_handle, twiddles
    t, dev, code = _device_signal(X)
    if t.dim() == 1:
        t = t.unsqueeze(0)
    B, n = t.shape
    check_signal_shape((n,))
    if d < 1 or n % d:
        raise ValueError(f"downsampling factor {d} does not divide {n}")
    shifts = [int(s) for s in shifts]
    if any(not 0 <= s < n for s in shifts):
        raise ValueError(f"shift outside [0, {n})")
    L = n // d
    out = torch.empty((B, len(shifts), L), dtype=torch.complex128, device=dev)
    if not shifts or B == 0:
        return out
    lib = _lib.load()
    sh = torch.tensor(shifts, dtype=torch.int64, device=dev)
    ws = resolve_workspace(None, lib.sfdt_aliased_values_workspace_bytes(B, n, d, len(shifts)), dev)
    _lib.check(lib.sfdt_aliased_values(t.data_ptr(), code, B, n, int(d), sh.data_ptr(), len(shifts),
                                       twiddles(L, dev).data_ptr(), out.data_ptr(), ws.data_ptr(), ws.numel(),
                                       stream_handle(dev)), "sfdt_aliased_values")
    return out


def transform_view(view: DownsampleView) -> AliasedSpectrum:
    """Scaled DFT of a view, fft_radix2(view) / m (spectral.py:163-167), on
    the GPU (bit-identical to the reference)."""
    m = view.data.size
    if m == 0 or m & (m - 1):
        raise ValueError(f"length must be a power of two, got {m}")
    vals = aliased_values_batch(np.asarray(view.data), 1, [0])[0, 0].cpu().numpy()
    return AliasedSpectrum(n=view.n, d=view.d, shift=view.shift, values=vals)


def aliased_values(x, d: int, shift: int) -> np.ndarray:
    """Scaled DFT of the (d, shift) view of x (spectral.py:170-172): one
    fused gather + FFT launch."""
    n = int(np.shape(x)[-1]) if not hasattr(x, "numel") else int(x.numel())
    if d < 1 or n % d:
        raise ValueError(f"downsampling factor {d} does not divide {n}")
    if not 0 <= shift < n:
        raise ValueError(f"shift {shift} outside [0, {n})")
    m = n // d
    if m == 0 or m & (m - 1):
        raise ValueError(f"length must be a power of two, got {m}")
    if n & (n - 1):   # a non-power-of-two parent: gather, then transform the view
        return transform_view(downsample(x, d, shift)).values
    return aliased_values_batch(x, d, [shift])[0, 0].cpu().numpy()


def syndromes_for_bin(views, k: int) -> SyndromeSet:
    """One bin's syndromes from transformed views sharing a factor d
    (spectral.py:175-190)."""
    views = list(views)
    if not views:
        raise ValueError("need at least one transformed view")
    d = views[0].d
    m = views[0].values.size
    if any(v.d != d for v in views):
        raise ValueError("views must share the downsampling factor")
    if not 0 <= k < m:
        raise ValueError(f"bin {k} outside [0, {m})")
    return SyndromeSet(bin=k, values=np.array([v.values[k] for v in views], dtype=np.complex128),
                       shifts=np.array([v.shift for v in views], dtype=np.int64))


def forward_dft_oracle(x) -> np.ndarray:
    """O(n^2) direct-summation analysis DFT with 1/n (spectral.py:110-125):
    the reference's validation oracle, one warp per output bin on the GPU
    over the same root table exp(-2j pi q / n)."""
    import torch

    from . import _lib
    from .device import stream_handle
    arr = as_signal(x)
    n = arr.size
    t, dev, _ = _device_signal(arr, allow_c64=False)
    roots = torch.empty(2 * n, dtype=torch.float64, device=dev)
    out = torch.empty_like(t)
    _lib.check(_lib.load().sfdt_direct_dft(t.data_ptr(), 1, n, roots.data_ptr(), out.data_ptr(),
                                           stream_handle(dev)), "sfdt_direct_dft")
    return out.cpu().numpy()


def rms(x) -> float:
    """Root mean square magnitude of a time signal (spectral.py:215-218),
    by the solvers' own HBM pass (k_sumsq): the value they threshold with."""
    import torch

    from . import _lib
    from .device import resolve_workspace, stream_handle
    t, dev, code = _device_signal(x)
    t = t.reshape(-1)
    n = check_signal_shape(t.shape)
    out = torch.empty(1, dtype=torch.float64, device=dev)
    lib = _lib.load()
    ws = resolve_workspace(None, lib.sfdt_rms_workspace_bytes(1, n), dev)
    _lib.check(lib.sfdt_rms(t.data_ptr(), code, 1, n, out.data_ptr(), ws.data_ptr(), ws.numel(),
                            stream_handle(dev)), "sfdt_rms")
    return float(out.item())


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
