"""Exactly-K-sparse solvers on the B200 (drop-in for sfft_dt.exact).

Same public names, parameters, validation and results as the reference
(/root/reference/pkg/src/sfft_dt/exact.py):

    ExactConfig, IterationStats, SolverTrace, EstimateResult,
    solve_noniterative(x, cfg)  -> (SparseSpectrum, SolverTrace)   exact.py:161
    solve_iterative(x, cfg)     -> (SparseSpectrum, SolverTrace)   exact.py:203
    estimate_sparsity_and_solve(x, mu, a_max, zero_threshold)      exact.py:307

plus batched forms that keep B signals resident in HBM:

    solve_noniterative_batch(X, cfg) / solve_iterative_batch(X, cfg)
        -> ExactBatch (device results; .spectra(), .traces(), .to_host())

All arithmetic runs in libsfdt_b200.so (one HBM pass over x, shared-memory
FFTs, thread-per-bin decoding); see DESIGN.md.
"""

from __future__ import annotations

import ctypes
import logging
import time
from dataclasses import dataclass, field

import numpy as np
import torch

from . import _lib
from .device import (resolve_workspace, host_copy, as_device_signals, aux_stream, ptr, require_cuda, stream_handle,
                     twiddles)
from .spectral import SparseSpectrum, check_signal_shape

logger = logging.getLogger(__name__)

CONSISTENCY_RTOL = 1e-6
SNAP_TOL = 0.25
UNIT_MODULUS_TOL = 1e-6


@dataclass
class ExactConfig:
    """Exactly-sparse solver parameters (exact.py:31-71).

    d = n/(mu*k) rounded down to a power of two (>= 1) unless initial_d is
    given; syndromes below zero_threshold * rms(x) * d count as zero."""

    n: int
    k: int | None = None
    mu: int = 4
    a_max: int = 4
    zero_threshold: float = 1e-9
    tau: float = 0.01
    initial_d: int | None = None

    def __post_init__(self):
        if self.n < 2 or self.n & (self.n - 1):
            raise ValueError(f"n must be a power of two >= 2, got {self.n}")
        if not 1 <= self.a_max <= 4:
            raise ValueError(f"a_max must be in 1..4, got {self.a_max}")
        if self.mu < 1 or self.mu & (self.mu - 1):
            raise ValueError(f"mu must be a power of two >= 1, got {self.mu}")
        if self.k is None and self.initial_d is None:
            raise ValueError("either k or initial_d is required")
        if self.k is not None and self.k < 1:
            raise ValueError(f"k must be >= 1, got {self.k}")
        if self.initial_d is not None and (self.initial_d < 1 or self.n % self.initial_d):
            raise ValueError(f"initial_d {self.initial_d} must divide n={self.n}")

    def resolved_d(self) -> int:
        if self.initial_d is not None:
            return self.initial_d
        raw = self.n // (self.mu * self.k)
        return 1 if raw < 1 else 1 << (raw.bit_length() - 1)


@dataclass
class IterationStats:
    d: int
    bins_attempted: int
    bins_solved: int
    bins_deferred: int
    syndromes_computed: int
    fft_samples: int


@dataclass
class SolverTrace:
    solver: str
    iterations: list = field(default_factory=list)
    fft_samples: int = 0
    syndromes_computed: int = 0
    full_success: bool = False
    unresolved_bins: list = field(default_factory=list)
    warnings: list = field(default_factory=list)
    elapsed_s: float = 0.0


@dataclass
class EstimateResult:
    spectrum: SparseSpectrum
    k_hat: int
    final_d: int
    fft_samples: int
    fft_samples_final_run: int
    dense_fallback: bool
    stages: list
    trace: SolverTrace


class ExactBatch:
    """Device-resident results of one batched exact solve.

    entry_offsets (B+1) int64, locs int64, vals complex128, unres_offsets,
    unres_bins int32, dup_offsets/dup_locs (iterative), stats (B, 32) int64,
    rms (B,) float64 -- all CUDA tensors, compacted per signal in the
    reference's dictionary insertion order."""

    def __init__(self, n, iterative, tensors, elapsed_s):
        self.n = n
        self.iterative = iterative
        self.t = tensors
        self.elapsed_s = elapsed_s
        self._host = None

    @property
    def batch(self) -> int:
        return self.t["stats"].shape[0]

    def to_host(self) -> dict:
        """Copy the compacted results to host numpy arrays: the fixed-size
        fields, then the used prefix of the variable-size lists (two
        stream syncs, pinned staging)."""
        if self._host is None:
            t = self.t
            fixed = ["entry_offsets", "unres_offsets", "stats", "rms"]
            if t.get("dup_offsets") is not None:
                fixed.append("dup_offsets")
            h = host_copy({k: t[k] for k in fixed})
            total, utotal = int(h["entry_offsets"][-1]), int(h["unres_offsets"][-1])
            var = {"locs": t["locs"][:total], "vals": t["vals"][:total],
                   "unres_bins": t["unres_bins"][:utotal]}
            if "dup_offsets" in h:
                var["dup_locs"] = t["dup_locs"][:int(h["dup_offsets"][-1])]
            h.update(host_copy(var))
            h["vals"] = h["vals"].view(np.complex128).reshape(-1)
            self._host = h
        return self._host

    def spectrum(self, b: int) -> SparseSpectrum:
        h = self.to_host()
        lo, hi = h["entry_offsets"][b], h["entry_offsets"][b + 1]
        return SparseSpectrum(self.n, dict(zip(h["locs"][lo:hi].tolist(), h["vals"][lo:hi].tolist())))

    def spectra(self) -> list:
        return [self.spectrum(b) for b in range(self.batch)]

    def trace(self, b: int) -> SolverTrace:
        h = self.to_host()
        st = h["stats"][b]
        niter = int(st[_lib.SFDT_ST_NITER])
        its = []
        for p in range(niter):
            f = st[_lib.SFDT_ST_ITER0 + 6 * p: _lib.SFDT_ST_ITER0 + 6 * p + 6]
            its.append(IterationStats(int(f[0]), int(f[1]), int(f[2]), int(f[3]), int(f[4]),
                                      int(f[5])))
        lo, hi = h["unres_offsets"][b], h["unres_offsets"][b + 1]
        warnings = []
        if "dup_offsets" in h:
            dl, dh = h["dup_offsets"][b], h["dup_offsets"][b + 1]
            warnings = [f"duplicate location {int(s)}: overwriting earlier value"
                        for s in h["dup_locs"][dl:dh]]
        return SolverTrace(
            solver="iterative" if self.iterative else "non_iterative", iterations=its,
            fft_samples=int(st[_lib.SFDT_ST_FFT_SAMPLES]),
            syndromes_computed=int(st[_lib.SFDT_ST_SYNDROMES]),
            full_success=bool(st[_lib.SFDT_ST_FULL_SUCCESS]),
            unresolved_bins=[int(v) for v in h["unres_bins"][lo:hi]], warnings=warnings,
            elapsed_s=self.elapsed_s)

    def traces(self) -> list:
        return [self.trace(b) for b in range(self.batch)]


def _outputs(caps, B, device, iterative):
    """Fresh output tensors (the caching allocator recycles them cheaply);
    each ExactBatch owns its results."""
    ecap, ucap, dcap = caps
    return {
            "entry_offsets": torch.empty(B + 1, dtype=torch.int64, device=device),
            "locs": torch.empty(ecap, dtype=torch.int64, device=device),
            "vals": torch.empty((ecap, 2), dtype=torch.float64, device=device),
            "unres_offsets": torch.empty(B + 1, dtype=torch.int64, device=device),
            "unres_bins": torch.empty(ucap, dtype=torch.int32, device=device),
            "stats": torch.empty((B, _lib.SFDT_ST_PER_SIGNAL), dtype=torch.int64, device=device),
            "rms": torch.empty(B, dtype=torch.float64, device=device),
            "dup_offsets": torch.empty(B + 1, dtype=torch.int64, device=device) if iterative else None,
            "dup_locs": torch.empty(max(dcap, 1), dtype=torch.int64, device=device) if iterative else None,
    }


def exact_batch(X, cfg: ExactConfig, iterative: bool, device=None,
                stream_events=None, pipeline: int = 0, rms=None, workspace=None) -> ExactBatch:
    """Batched exact solve of X (B, n) (or (n,)) -- the device entry point.

    stream_events: optional (begin, end) torch.cuda.Event pair recorded around
    the HBM stream kernel (roofline instrumentation; events must have been
    recorded once so their handles exist).  rms: optional (B,) float64 CUDA
    tensor of rms(x) from an earlier solve of the same signals -- the HBM
    pass over x is then skipped (rms is a pure function of x).  workspace:
    a device.Workspace to use instead of the (device, stream) default (a
    captured graph keeps its own)."""
    t0 = time.perf_counter()
    dev = require_cuda(device if device is not None else
                       (X.device if isinstance(X, torch.Tensor) and X.is_cuda else None))
    X = as_device_signals(X, dev)
    if X.dim() == 1:
        X = X.unsqueeze(0)
    if X.dim() != 2:
        raise ValueError(f"signal must be 1-D, got shape {tuple(X.shape)}")
    B = X.shape[0]
    n = check_signal_shape(X.shape[1:])
    if n != cfg.n:
        raise ValueError(f"signal length {n} != configured n {cfg.n}")
    d = cfg.resolved_d()
    lib = _lib.load()
    args = _lib.ExactArgs()
    args.x = X.data_ptr()
    args.x_dtype = _lib.SFDT_C64 if X.dtype == torch.complex64 else _lib.SFDT_C128
    args.batch, args.n, args.d = B, n, d
    args.a_max, args.iterative = cfg.a_max, int(bool(iterative))
    args.zero_threshold = float(cfg.zero_threshold)
    caps = [_lib._i64(), _lib._i64(), _lib._i64()]
    _lib.check(lib.sfdt_exact_caps(args, *[ctypes.byref(c) for c in caps]), "sfdt_exact_caps")
    caps = tuple(c.value for c in caps)
    tw = twiddles(n // d, dev)
    args.twiddles = tw.data_ptr()
    o = _outputs(caps, B, dev, iterative)
    args.entry_offsets, args.locs, args.vals = ptr(o["entry_offsets"]), ptr(o["locs"]), ptr(o["vals"])
    args.entry_cap = caps[0]
    args.unres_offsets, args.unres_bins, args.unres_cap = ptr(o["unres_offsets"]), ptr(o["unres_bins"]), caps[1]
    args.dup_offsets = ptr(o["dup_offsets"])
    args.dup_locs = ptr(o["dup_locs"])
    args.dup_cap = caps[2] if iterative else 0
    args.stats, args.rms = ptr(o["stats"]), ptr(o["rms"])
    if rms is not None:
        rms = rms.to(dev, torch.float64).contiguous()
        if rms.numel() != B:
            raise ValueError("rms must have one entry per signal")
        args.rms_in = rms.data_ptr()
    if pipeline and not iterative:
        # overlap the view gather + FFT + decode (aux stream) with the HBM
        # stream pass (current stream), in chunks of `pipeline` signals
        args.aux_stream = aux_stream(dev).cuda_stream
        args.chunk_signals = int(pipeline)
    if stream_events is not None:
        args.ev_stream_begin = stream_events[0].cuda_event
        args.ev_stream_end = stream_events[1].cuda_event
    tn = _lib.tuning_struct()
    args.tuning = ctypes.addressof(tn)
    nbytes = lib.sfdt_exact_workspace_bytes(args)
    ws = resolve_workspace(workspace, nbytes, dev)
    _lib.check(lib.sfdt_exact_solve(args, ws.data_ptr(), ws.numel(), stream_handle(dev)),
               "sfdt_exact_solve")
    if rms is not None:
        o["_rms_in"] = rms
    res = ExactBatch(n, bool(iterative), dict(o), time.perf_counter() - t0)
    res.kernel_launches = int(args.kernel_launches)
    res.workspace_bytes = int(nbytes)
    return res


def solve_noniterative_batch(X, cfg: ExactConfig, device=None) -> ExactBatch:
    return exact_batch(X, cfg, False, device)


def solve_iterative_batch(X, cfg: ExactConfig, device=None) -> ExactBatch:
    return exact_batch(X, cfg, True, device)


def _single(x, cfg, iterative):
    t0 = time.perf_counter()
    if isinstance(x, torch.Tensor):
        check_signal_shape(x.shape)
    else:
        x = np.asarray(x)
        check_signal_shape(x.shape)
    res = exact_batch(x, cfg, iterative)
    spec = res.spectrum(0)
    trace = res.trace(0)
    for w in trace.warnings:
        logger.warning(w)
    trace.elapsed_s = time.perf_counter() - t0
    return spec, trace


def solve_noniterative(x, cfg: ExactConfig):
    """Fixed-d solver (exact.py:161-200): 2*a_max shifted views, per-bin
    decode with ascending collision count, first validated model wins."""
    return _single(x, cfg, False)


def solve_iterative(x, cfg: ExactConfig):
    """Iterative solver (exact.py:203-292): d doubles per pass, previous
    views fold, solved frequencies are subtracted, a = l+1 .. 1 with
    singular-only retry and deferral."""
    return _single(x, cfg, True)


def estimate_sparsity_and_solve(x, mu: int = 4, a_max: int = 4,
                                zero_threshold: float = 1e-9) -> EstimateResult:
    """Bottom-up sparsity estimation (exact.py:307-340): non-iterative solves
    at d = n, n/2, ... until every active bin decodes or d = 1.  The signal
    is uploaded once and stays resident; rms(x) -- the only O(N) read -- is
    computed once by the first stage and reused, so later stages only gather
    their 2*a_max*(n/d) view samples."""
    if isinstance(x, torch.Tensor):
        n = check_signal_shape(x.shape)
    else:
        x = np.asarray(x)
        n = check_signal_shape(x.shape)
    dev = require_cuda(x.device if isinstance(x, torch.Tensor) and x.is_cuda else None)
    xd = as_device_signals(x, dev)
    d, total, stages = n, 0, []
    rms = None   # rms(x) is computed by the first stage's HBM pass and reused
    while True:
        t0 = time.perf_counter()
        cfg = ExactConfig(n=n, k=None, mu=mu, a_max=a_max, zero_threshold=zero_threshold,
                          initial_d=d)
        res = exact_batch(xd, cfg, False, dev, rms=rms)
        if rms is None:
            rms = res.t["rms"]
        spectrum, trace = res.spectrum(0), res.trace(0)
        for w in trace.warnings:
            logger.warning(w)
        trace.elapsed_s = time.perf_counter() - t0
        total += trace.fft_samples
        stages.append((d, trace.full_success))
        if trace.full_success or d == 1:
            return EstimateResult(spectrum=spectrum, k_hat=len(spectrum), final_d=d,
                                  fft_samples=total, fft_samples_final_run=trace.fft_samples,
                                  dense_fallback=not trace.full_success, stages=stages, trace=trace)
        d //= 2
