"""Generally-K-sparse recovery on the B200 (drop-in for sfft_dt.general).

Same public names, parameters and results as the reference
(/root/reference/pkg/src/sfft_dt/general.py):

    GeneralConfig, GeneralTrace, CollisionEstimate, draw_shifts,
    solve_general(x, cfg) -> (SparseSpectrum, GeneralTrace)      general.py:272

plus solve_general_batch(X, cfg, seeds=None) for B signals in HBM.  The
shift draw stays on the host with numpy's Generator (bit-identical shifts);
everything else -- views, singular values, the top-K vote, pruning,
matched filter and subspace pursuit -- runs in libsfdt_b200.so.
"""

from __future__ import annotations

import ctypes
import logging
import time
from dataclasses import dataclass, field

import numpy as np
import torch

from . import _lib
from .device import (as_device_signals, aux_stream, host_copy, ptr, require_cuda, resolve_workspace,
                     stream_handle, twiddles)
from .spectral import SparseSpectrum, check_signal_shape

logger = logging.getLogger(__name__)


@dataclass
class GeneralConfig:
    """Generally-sparse solver parameters (general.py:28-70)."""

    n: int
    k: int
    a_max: int = 3
    d: int | None = None
    rng_seed: int | tuple = 0
    keep_per_collision: int = 2
    prune: bool = True
    zero_vote_rtol: float = 1e-9

    def __post_init__(self):
        if self.n < 2 or self.n & (self.n - 1):
            raise ValueError(f"n must be a power of two >= 2, got {self.n}")
        if not 1 <= self.k <= self.n:
            raise ValueError(f"k must be in [1, n], got {self.k}")
        if not 1 <= self.a_max <= 4:
            raise ValueError(f"a_max must be 1..4, got {self.a_max}")
        if 2 * self.a_max > self.n:
            raise ValueError("n too small for 2*a_max consecutive shifts")
        if self.keep_per_collision < 1:
            raise ValueError("keep_per_collision must be >= 1")
        if self.d is not None and (self.d < 1 or self.n % self.d):
            raise ValueError(f"d={self.d} must divide n={self.n}")

    def resolved_d(self) -> int:
        if self.d is not None:
            return self.d
        raw = self.n // (32 * self.k)
        return 1 if raw < 1 else 1 << (raw.bit_length() - 1)

    @property
    def r(self) -> int:
        return 3 * self.a_max


@dataclass(frozen=True)
class SensingMatrix:
    """Partial-Fourier sensing matrix of one bin (general.py:73-80): rows are
    shifted views, columns candidate frequency locations."""

    matrix: np.ndarray
    shifts: np.ndarray
    column_locations: np.ndarray


@dataclass(frozen=True)
class CollisionEstimate:
    a: np.ndarray
    singular_values: np.ndarray


@dataclass
class GeneralTrace:
    d: int = 0
    r: int = 0
    shifts: list = field(default_factory=list)
    fft_samples: int = 0
    collision_histogram: dict = field(default_factory=dict)
    timings: dict = field(default_factory=dict)
    pruned: bool = True
    warnings: list = field(default_factory=list)


def draw_shifts(d: int, r: int, seed) -> np.ndarray:
    """r distinct shifts drawn uniformly from [0, d-1] (general.py:101-106)."""
    if r > d:
        raise ValueError(f"cannot draw {r} distinct shifts from [0, {d})")
    return np.random.default_rng(seed).choice(d, size=r, replace=False).astype(np.int64)


def base_phi_table(shifts: np.ndarray, d: int) -> np.ndarray:
    """exp(2 pi i shifts_j t / d), evaluated exactly as general.py:309 does."""
    return np.exp(2j * np.pi * np.outer(shifts, np.arange(d)) / d)


class GeneralBatch:
    def __init__(self, n, cfg, d, r_eff, shifts, tensors, elapsed_s, kernel_launches):
        self.n, self.cfg, self.d, self.r_eff = n, cfg, d, r_eff
        self.shifts = shifts          # (B, r_eff) host int64
        self.t = tensors
        self.elapsed_s = elapsed_s
        self.kernel_launches = kernel_launches
        self._host = None

    @property
    def batch(self) -> int:
        return self.t["stats"].shape[0]

    def to_host(self) -> dict:
        """Compacted results to host numpy arrays (two stream syncs)."""
        if self._host is None:
            t = self.t
            h = host_copy({"entry_offsets": t["entry_offsets"], "stats": t["stats"]})
            total = int(h["entry_offsets"][-1])
            h.update(host_copy({"locs": t["locs"][:total], "vals": t["vals"][:total]}))
            h["vals"] = h["vals"].view(np.complex128).reshape(-1)
            self._host = h
        return self._host

    def spectrum(self, b: int) -> SparseSpectrum:
        h = self.to_host()
        lo, hi = h["entry_offsets"][b], h["entry_offsets"][b + 1]
        return SparseSpectrum(self.n, dict(zip(h["locs"][lo:hi].tolist(), h["vals"][lo:hi].tolist())))

    def spectra(self) -> list:
        return [self.spectrum(b) for b in range(self.batch)]

    def trace(self, b: int) -> GeneralTrace:
        h = self.to_host()
        st = h["stats"][b]
        a_max = self.cfg.a_max
        hist = {a: int(st[_lib.SFDT_GS_HIST0 + a]) for a in range(a_max + 1)}
        return GeneralTrace(d=self.d, r=self.r_eff, shifts=self.shifts[b].tolist(),
                            fft_samples=(2 * a_max + self.r_eff) * (self.n // self.d),
                            collision_histogram=hist, timings={"total": self.elapsed_s},
                            pruned=self.cfg.prune, warnings=[])

    def votes(self) -> np.ndarray:
        return self.t["votes"].cpu().numpy()

    def singular_values(self) -> np.ndarray:
        return self.t["singular_values"].cpu().numpy()


class GeneralPlan:
    """Per-(config, batch, seeds) constants on the device: the drawn shifts
    and the base_phi tables (built on the host exactly as general.py:101-106,
    309 build them).  Reusable across batches with the same seeds."""

    def __init__(self, cfg: GeneralConfig, batch: int, seeds=None, device=None):
        dev = require_cuda(device)
        d = cfg.resolved_d()
        r_eff = min(cfg.r, d)
        if seeds is None:
            sh = draw_shifts(d, r_eff, cfg.rng_seed)[None, :]
            phi = base_phi_table(sh[0], d)[None]
            self.stride_s, self.stride_p = 0, 0
            self.sh = np.broadcast_to(sh, (batch, r_eff))
        else:
            if len(seeds) != batch:
                raise ValueError("need one seed per signal")
            sh = np.stack([draw_shifts(d, r_eff, s) for s in seeds])
            phi = np.stack([base_phi_table(s, d) for s in sh])
            self.stride_s, self.stride_p = r_eff, r_eff * d
            self.sh = sh
        self.cfg, self.batch = cfg, batch
        self.sh_d = torch.from_numpy(np.ascontiguousarray(sh)).to(dev)
        self.phi_d = torch.from_numpy(np.ascontiguousarray(phi)).to(dev)


def solve_general_batch(X, cfg: GeneralConfig, seeds=None, device=None,
                        plan: GeneralPlan | None = None, zero_copy: bool = False,
                        fft_events=None, workspace=None, phase_events=None) -> GeneralBatch:
    """Batched solve_general.  seeds: None (cfg.rng_seed for every signal) or
    one rng_seed per signal (per-signal shift draws); plan: precomputed
    GeneralPlan for repeated batches.

    zero_copy: X is a pinned (page-locked) HOST tensor and stays there.  The
    general path reads only the (2*a_max + r_eff)*L view samples of each
    signal (general.py:288-294), so the view gather loads them
    straight from mapped host memory over PCIe (UVA) instead of copying all
    N samples to HBM first."""
    t0 = time.perf_counter()
    dev = require_cuda(device if device is not None else
                       (X.device if isinstance(X, torch.Tensor) and X.is_cuda else None))
    if zero_copy:
        if not (isinstance(X, torch.Tensor) and X.device.type == "cpu" and X.is_pinned()):
            raise ValueError("zero_copy needs a pinned host tensor (tensor.pin_memory())")
        if X.dtype not in (torch.complex128, torch.complex64) or not X.is_contiguous():
            raise ValueError("zero_copy needs a contiguous complex128/complex64 tensor")
    else:
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
    r_eff = min(cfg.r, d)
    if plan is None:
        plan = GeneralPlan(cfg, B, seeds, dev)
    elif plan.batch != B or plan.cfg != cfg:
        raise ValueError("plan was built for a different batch/config")
    sh, sh_d, phi_d, stride_s, stride_p = plan.sh, plan.sh_d, plan.phi_d, plan.stride_s, plan.stride_p
    lib = _lib.load()
    a = _lib.GeneralArgs()
    a.x = X.data_ptr()
    a.x_dtype = _lib.SFDT_C64 if X.dtype == torch.complex64 else _lib.SFDT_C128
    a.batch, a.n, a.k, a.d = B, n, cfg.k, d
    a.a_max, a.r_eff = cfg.a_max, r_eff
    a.keep_per_collision, a.prune = cfg.keep_per_collision, int(bool(cfg.prune))
    a.zero_vote_rtol = float(cfg.zero_vote_rtol)
    a.shifts, a.shift_stride = sh_d.data_ptr(), stride_s
    a.base_phi, a.phi_stride = phi_d.data_ptr(), stride_p
    tw = twiddles(n // d, dev)
    a.twiddles = tw.data_ptr()
    cap = _lib._i64()
    _lib.check(lib.sfdt_general_caps(a, ctypes.byref(cap)), "sfdt_general_caps")
    L = n // d
    o = {
        "entry_offsets": torch.empty(B + 1, dtype=torch.int64, device=dev),
        "locs": torch.empty(cap.value, dtype=torch.int64, device=dev),
        "vals": torch.empty((cap.value, 2), dtype=torch.float64, device=dev),
        "stats": torch.zeros((B, _lib.SFDT_GS_PER_SIGNAL), dtype=torch.int64, device=dev),
        "votes": torch.empty((B, L), dtype=torch.int32, device=dev),
        "singular_values": torch.empty((B, L, cfg.a_max), dtype=torch.float64, device=dev),
    }
    a.entry_offsets, a.locs, a.vals, a.entry_cap = ptr(o["entry_offsets"]), ptr(o["locs"]), \
        ptr(o["vals"]), cap.value
    a.stats, a.votes, a.singular_values = ptr(o["stats"]), ptr(o["votes"]), ptr(o["singular_values"])
    if fft_events is not None:   # (begin, end) around the view gather + FFT (roofline timing)
        a.ev_fft_begin, a.ev_fft_end = fft_events[0].cuda_event, fft_events[1].cuda_event
    if phase_events is not None:   # 5 events: fft begin / end, vote, prune, pursuit ends
        e = [ev.cuda_event for ev in phase_events]
        a.ev_fft_begin, a.ev_fft_end, a.ev_vote_end, a.ev_prune_end, a.ev_pursuit_end = e
    t = _lib.current_tuning()
    tn = _lib.tuning_struct(t)
    a.tuning = ctypes.addressof(tn)
    if t["gen_overlap"]:
        # the multi-collision pursuit forks onto the device's aux stream
        a.aux_stream = aux_stream(dev).cuda_stream
    nbytes = lib.sfdt_general_workspace_bytes(a)
    ws = resolve_workspace(workspace, nbytes, dev)
    _lib.check(lib.sfdt_general_solve(a, ws.data_ptr(), ws.numel(), stream_handle(dev)),
               "sfdt_general_solve")
    o["_keep"] = (sh_d, phi_d, tw, X)   # X: a zero-copy host source stays alive with the results
    return GeneralBatch(n, cfg, d, r_eff, sh, o, time.perf_counter() - t0, int(a.kernel_launches))


def solve_general(x, cfg: GeneralConfig):
    """Full pipeline (general.py:272-372): shifted-view FFTs, collision vote,
    pruning, per-bin subspace pursuit; returns (spectrum, trace).
    trace.timings carries the reference's phases -- fft, vote, prune,
    subspace_pursuit (device time between CUDA events at the phase
    boundaries) and total (wall clock of the call)."""
    t0 = time.perf_counter()
    if isinstance(x, torch.Tensor):
        check_signal_shape(x.shape)
    else:
        x = np.asarray(x)
        check_signal_shape(x.shape)
    dev = require_cuda(x.device if isinstance(x, torch.Tensor) and x.is_cuda else None)
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(5)]
    for e in ev:   # materialise the handles
        e.record(torch.cuda.current_stream(dev))
    res = solve_general_batch(x, cfg, device=dev, phase_events=ev)
    spec = res.spectrum(0)
    tr = res.trace(0)
    ms = [ev[i].elapsed_time(ev[i + 1]) / 1e3 for i in range(4)]
    tr.timings = {"fft": ms[0], "vote": ms[1], "prune": ms[2], "subspace_pursuit": ms[3],
                  "total": time.perf_counter() - t0}
    nrd = int(res.to_host()["stats"][0][_lib.SFDT_GS_RANKDEF])
    if nrd:
        # general.py:243-244 logs one warning per rank-deficient least
        # squares; the device counts them per signal
        logger.warning("rank-deficient least squares on %d pursuit support(s)", nrd)
    return spec, tr


def sensing_matrix(n: int, d: int, k: int, shifts, columns=None) -> SensingMatrix:
    """Phi[j, t] = exp(2i pi (k + t n/d) shifts[j] / n) over the selected
    candidate columns, all d when columns is None (general.py:109-121), built
    on the GPU with numpy's phase evaluation."""
    shifts = np.ascontiguousarray(shifts, dtype=np.int64)
    m = n // d
    cols = np.arange(d, dtype=np.int64) if columns is None else np.ascontiguousarray(columns, dtype=np.int64)
    locs = (k + cols * m) % n
    dev = require_cuda()
    out = torch.empty((shifts.size, cols.size, 2), dtype=torch.float64, device=dev)
    if shifts.size and cols.size:
        sh = torch.from_numpy(shifts).to(dev)
        cd = torch.from_numpy(cols).to(dev)
        _lib.check(_lib.load().sfdt_sensing_matrix(int(n), int(d), int(k), sh.data_ptr(), shifts.size,
                                                   cd.data_ptr(), cols.size, out.data_ptr(), stream_handle(dev)),
                   "sfdt_sensing_matrix")
    phi = out.cpu().numpy().view(np.complex128).reshape(shifts.size, cols.size)
    return SensingMatrix(matrix=phi, shifts=shifts, column_locations=locs)


PRUNE_MAX_KEEP = 64   # keep_per_collision * a of the device mirror


def prune_columns(m, a: int, k: int, n: int, d: int, a_max: int | None = None,
                  keep_per_collision: int = 2, fallback=None,
                  augment_with_correlation: bool = False) -> np.ndarray:
    """Candidate columns of one bin surviving the locator-polynomial test
    (general.py:184-221), on the GPU: Hankel fit of order a_max descending
    past singular fits, |P(z)| over the d candidate roots (the reference's
    recurrence), the keep_per_collision * a smallest, sorted.  All fits
    singular: the correlation fallback when fallback=(y, shifts), else every
    column.  augment_with_correlation unions the top-a correlation columns."""
    m = np.ascontiguousarray(m, dtype=np.complex128)
    if a < 1:
        raise ValueError("a must be >= 1")
    if a_max is None:
        a_max = max(a, min(len(m) // 2, 4))
    if not 1 <= a_max <= 4:
        raise ValueError(f"collision count must be 1..4, got {a_max}")
    if len(m) < 2 * a_max:
        raise ValueError(f"need at least {2 * a_max} syndromes, got {len(m)}")
    if keep_per_collision * a > PRUNE_MAX_KEEP:
        raise ValueError(f"keep_per_collision * a = {keep_per_collision * a} exceeds the device "
                         f"mirror's {PRUNE_MAX_KEEP}")
    dev = require_cuda()
    lib = _lib.load()
    md = torch.from_numpy(m[:2 * a_max].view(np.float64).copy()).to(dev)
    kd = torch.tensor([int(k)], dtype=torch.int64, device=dev)
    yd = shd = None
    r = 0
    if fallback is not None:
        y, sh = fallback
        y = np.ascontiguousarray(y, dtype=np.complex128).ravel()
        sh = np.ascontiguousarray(sh, dtype=np.int64).ravel()
        r = y.size
        if r != sh.size or not 1 <= r <= 12:
            raise ValueError("fallback (y, shifts) must pair 1..12 views")
        yd = torch.from_numpy(y.view(np.float64)).to(dev)
        shd = torch.from_numpy(sh).to(dev)
    cap = keep_per_collision * a + a
    kept = torch.empty(cap, dtype=torch.int64, device=dev)
    nk = torch.empty(1, dtype=torch.int32, device=dev)
    _lib.check(lib.sfdt_prune_columns(md.data_ptr(), 1, 2 * a_max, kd.data_ptr(), int(a), int(a_max), int(n),
                                      int(d), int(keep_per_collision), ptr(yd), r, ptr(shd), r,
                                      int(bool(augment_with_correlation)), kept.data_ptr(), nk.data_ptr(), cap,
                                      stream_handle(dev)), "sfdt_prune_columns")
    count = int(nk.item())
    if count < 0:
        return np.arange(d, dtype=np.int64)
    return kept[:count].cpu().numpy()


def subspace_pursuit(y, phi, a: int, max_iter: int = 10) -> np.ndarray:
    """Greedy a-sparse solve of y ~ phi @ coef (general.py:224-269) on the
    GPU: top-a correlation start, then merge / least squares (gelsd
    semantics: Householder QR, minimum-norm SVD when rank deficient) /
    keep top-a / least squares until the residual stops shrinking by 1e-12
    or max_iter.  Returns the dense coefficient vector over phi's columns.
    Shapes of the solver: rows <= 12, min(a, cols) <= 4."""
    y = np.ascontiguousarray(y, dtype=np.complex128).ravel()
    phi = np.ascontiguousarray(phi, dtype=np.complex128)
    rows, cols = phi.shape
    if a < 1 or a > rows:
        raise ValueError(f"sparsity {a} outside [1, rows={rows}]")
    if rows > 12 or min(a, cols) > 4:
        raise ValueError(f"the device pursuit takes rows <= 12 and min(a, cols) <= 4, got rows={rows}, "
                         f"a={a}, cols={cols}")
    dev = require_cuda()
    yd = torch.from_numpy(y.view(np.float64)).to(dev)
    pd = torch.from_numpy(phi.view(np.float64)).to(dev)
    coef = torch.empty((cols, 2), dtype=torch.float64, device=dev)
    rd = torch.zeros(1, dtype=torch.int32, device=dev)
    _lib.check(_lib.load().sfdt_subspace_pursuit(yd.data_ptr(), pd.data_ptr(), 1, rows, cols, int(a),
                                                 int(max_iter), coef.data_ptr(), rd.data_ptr(),
                                                 stream_handle(dev)), "sfdt_subspace_pursuit")
    nrd = int(rd.item())
    if nrd:
        logger.warning("rank-deficient least squares in %d pursuit step(s)", nrd)
    return coef.cpu().numpy().view(np.complex128).ravel()


def estimate_collisions(syndromes, k: int, a_max: int, d: int,
                        zero_vote_rtol: float = 1e-9) -> CollisionEstimate:
    """Per-bin collision counts via the top-k singular-value vote
    (general.py:131-155), computed by the device kernels (Jacobi singular
    values with the reference's threshold, exact radix-select vote)."""
    syndromes = np.ascontiguousarray(syndromes, dtype=np.complex128)
    nb, ld = syndromes.shape
    dev = require_cuda()
    lib = _lib.load()
    sd = torch.from_numpy(syndromes).to(dev)
    votes = torch.empty(nb, dtype=torch.int32, device=dev)
    sv = torch.empty((nb, a_max), dtype=torch.float64, device=dev)
    ws = resolve_workspace(None, lib.sfdt_estimate_collisions_workspace_bytes(nb), dev)
    _lib.check(lib.sfdt_estimate_collisions(sd.data_ptr(), nb, ld, int(k), int(a_max), int(d),
                                            float(zero_vote_rtol), votes.data_ptr(), sv.data_ptr(),
                                            ws.data_ptr(), ws.numel(), stream_handle(dev)),
               "sfdt_estimate_collisions")
    return CollisionEstimate(a=votes.cpu().numpy().astype(np.int64), singular_values=sv.cpu().numpy())
