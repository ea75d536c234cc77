"""Host-resident signals streamed through the GPU (the end-to-end API).

solve_host_batch copies chunk i+1 host->device on a side stream while chunk i
is solved on the current stream, then reads every chunk's compacted results
back to the host.  Works for ExactConfig (solve_noniterative/iterative) and
GeneralConfig (solve_general).
"""

from __future__ import annotations

import numpy as np
import torch

from .device import require_cuda
from .exact import exact_batch
from .general import GeneralConfig, solve_general_batch
from .spectral import SparseSpectrum, check_signal_shape


class HostBatchResult:
    """Host-side results of solve_host_batch: the per-chunk batch results
    (ExactBatch or GeneralBatch) with global signal indexing."""

    def __init__(self, n, iterative, chunks, chunk_size, itemsize=16, zero_copy=False):
        self.n, self.iterative, self.chunks, self.chunk_size = n, iterative, chunks, chunk_size
        self.itemsize, self.zero_copy = itemsize, zero_copy

    def _loc(self, b):
        for ch in self.chunks:   # chunks may be split where a cycled pool wraps
            if b < ch.batch:
                return ch, b
            b -= ch.batch
        raise IndexError("signal index out of range")

    @property
    def h2d_bytes(self) -> int:
        """Signal bytes that crossed PCIe: whole rows, or for zero-copy the
        gathered view samples (sector-granular on the wire)."""
        tot = 0
        for ch in self.chunks:
            if self.zero_copy:
                L = self.n // ch.d
                tot += ch.batch * (2 * ch.cfg.a_max + ch.r_eff) * L * self.itemsize
            else:
                tot += ch.batch * self.n * self.itemsize
        return tot

    def spectrum(self, b) -> SparseSpectrum:
        ch, i = self._loc(b)
        return ch.spectrum(i)

    def trace(self, b):
        ch, i = self._loc(b)
        return ch.trace(i)

    @property
    def d2h_bytes(self) -> int:
        tot = 0
        for ch in self.chunks:
            tot += sum(v.nbytes for v in ch.to_host().values())
        return tot


def solve_host_batch(X_host, cfg, iterative: bool = False, chunk: int = 256,
                     device=None, n_signals: int | None = None,
                     zero_copy: bool | None = None) -> HostBatchResult:
    """Solve signals that live in HOST memory, streaming them through the GPU:
    chunk i+1 is copied host->device on a side stream while chunk i is
    solved, and every chunk's compacted results are read back to host.

    X_host: (B, n) torch tensor (pinned for full PCIe overlap) or numpy.
    n_signals: process this many signals, cycling over X_host's rows
    (synthetic benchmarking of large batches from a smaller host pool).
    zero_copy (GeneralConfig only; default: on when X_host is pinned and the
    downsampling factor d is >= 128, or >= 64 with 4096-point views): the
    general solver touches only (2*a_max + r_eff)*L samples per signal, so
    its view gather reads them from the pinned host rows directly over PCIe
    and the other N - 15*L samples never cross the bus.  The exact solvers
    need every sample (rms, exact.py:176), so they always stream whole rows."""
    dev = require_cuda(device)
    if not isinstance(X_host, torch.Tensor):
        X_host = torch.from_numpy(np.ascontiguousarray(X_host, dtype=np.complex128))
    if X_host.dim() != 2:
        raise ValueError(f"expected (B, n) signals, got shape {tuple(X_host.shape)}")
    H, n = X_host.shape
    check_signal_shape((n,))
    total = H if n_signals is None else int(n_signals)
    chunk = max(1, min(chunk, total))
    if zero_copy is None:
        # zero-copy pays while the views touch a small part of the signal: the
        # link then carries ~(1 + r_eff) read requests per d-block (window-ring
        # gather, 4096-point views; 2*a_max + r_eff otherwise) at the measured
        # ~650 M requests/s, against 16*d bytes per d-block at 55 GB/s for whole
        # rows -- the crossover is d ~ 64 (ring) / 128
        zero_copy = False
        if isinstance(cfg, GeneralConfig) and X_host.is_pinned():
            d = cfg.resolved_d()
            zero_copy = d >= 128 or (d >= 64 and n // d == 4096)
    if zero_copy:
        if not isinstance(cfg, GeneralConfig):
            raise ValueError("zero_copy applies to the general solver only (the exact "
                             "solvers read every sample)")
        results = []
        for lo in range(0, total, chunk):
            rows = min(chunk, total - lo)
            src_lo = lo % H
            if src_lo + rows <= H:
                results.append(solve_general_batch(X_host[src_lo:src_lo + rows], cfg, device=dev,
                                                   zero_copy=True))
            else:   # the cycle wraps: two solves
                k1 = H - src_lo
                results.append(solve_general_batch(X_host[src_lo:], cfg, device=dev, zero_copy=True))
                results.append(solve_general_batch(X_host[:rows - k1], cfg, device=dev,
                                                   zero_copy=True))
        for r in results:
            r.to_host()
        return HostBatchResult(n, False, results, chunk, X_host.element_size(), zero_copy=True)
    compute = torch.cuda.current_stream(dev)
    copy = torch.cuda.Stream(dev)
    bufs = [torch.empty((chunk, n), dtype=X_host.dtype, device=dev) for _ in range(2)]
    free = [torch.cuda.Event() for _ in range(2)]
    ready = [torch.cuda.Event() for _ in range(2)]
    for e in free:
        e.record(compute)
    results = []
    nchunks = (total + chunk - 1) // chunk
    for c in range(nchunks):
        i = c & 1
        lo = c * chunk
        rows = min(chunk, total - lo)
        with torch.cuda.stream(copy):
            copy.wait_event(free[i])
            src_lo = lo % H
            if src_lo + rows <= H:
                bufs[i][:rows].copy_(X_host[src_lo:src_lo + rows], non_blocking=True)
            else:
                k1 = H - src_lo
                bufs[i][:k1].copy_(X_host[src_lo:], non_blocking=True)
                bufs[i][k1:rows].copy_(X_host[:rows - k1], non_blocking=True)
            ready[i].record(copy)
        compute.wait_event(ready[i])
        if isinstance(cfg, GeneralConfig):
            results.append(solve_general_batch(bufs[i][:rows], cfg, device=dev))
        else:
            results.append(exact_batch(bufs[i][:rows], cfg, iterative, dev))
        free[i].record(compute)
    for r in results:
        r.to_host()
    return HostBatchResult(n, bool(iterative), results, chunk, X_host.element_size())

