"""Device plumbing: CUDA tensors, streams, twiddle tables, workspaces.

PyTorch is used only for device memory and streams; every computation on
the hot path is a kernel of libsfdt_b200.so.
"""

from __future__ import annotations

import numpy as np
import torch

from . import _lib

_twiddle_cache: dict = {}


def require_cuda(device=None) -> torch.device:
    if not torch.cuda.is_available():
        raise RuntimeError("paper_1407_8315_b200 needs a CUDA device (B200, sm_100a); "
                           "there is no CPU fallback")
    dev = torch.device(device) if device is not None else torch.device("cuda", torch.cuda.current_device())
    if dev.type != "cuda":
        raise ValueError(f"expected a CUDA device, got {dev}")
    return dev


def ptr(t: torch.Tensor | None) -> int | None:
    return None if t is None else t.data_ptr()


def stream_handle(device: torch.device) -> int:
    return torch.cuda.current_stream(device).cuda_stream


_aux_streams: dict = {}


def aux_stream(device: torch.device) -> torch.cuda.Stream:
    """Second stream per device for the library's overlap of latency-bound
    kernels with the HBM stream; high priority so its CTAs are dispatched as
    soon as SM resources free up."""
    st = _aux_streams.get(device)
    if st is None:
        st = torch.cuda.Stream(device, priority=-1)
        _aux_streams[device] = st
    return st


def twiddles(n_max: int, device: torch.device, inverse: bool = False) -> torch.Tensor:
    """Device copy of the reference-recurrence twiddle table (sfdt_fft_twiddles).
    Built once per (n_max, sign, device) on the host, cached."""
    n_max = max(int(n_max), 2)
    key = (n_max, bool(inverse), device)
    t = _twiddle_cache.get(key)
    if t is None:
        # the largest cached table of the same sign serves any smaller n
        for (n2, inv2, dev2), t2 in _twiddle_cache.items():
            if inv2 == bool(inverse) and dev2 == device and n2 >= n_max:
                return t2
        host = np.empty(2 * (n_max - 1), dtype=np.float64)
        _lib.check(_lib.load().sfdt_fft_twiddles(n_max, int(bool(inverse)),
                                                 host.ctypes.data_as(_lib._vp)), "sfdt_fft_twiddles")
        t = torch.from_numpy(host).to(device)
        _twiddle_cache[key] = t
    return t


class Workspace:
    """Grow-only byte workspace (the library never allocates).

    A solve writes its views, worklists and counters into the workspace it
    is given, so two solves may share one only if they are ordered on the
    device.  The default workspace of a solve is therefore keyed by
    (device, stream): solves on one stream are serialised by the stream, and
    solves on different streams get different buffers.  A captured CUDA
    graph bakes the workspace pointer in, so SolveGraph owns a private
    Workspace instance for its whole lifetime (pass ``workspace=`` to
    exact_batch / solve_general_batch), frozen once captured.  A superseded
    buffer goes back to PyTorch's caching allocator, which hands it out again
    only in stream order on the stream it was allocated on -- the stream
    whose solves used it -- so it is never reused under a running kernel."""

    _shared: dict = {}

    def __init__(self, device=None):
        self.device = device
        self.buf = None
        self.frozen = False

    def get(self, nbytes: int, device: torch.device) -> torch.Tensor:
        nbytes = max(int(nbytes), 256)
        if self.buf is None or self.buf.numel() < nbytes:
            if self.frozen:
                raise RuntimeError(f"workspace is frozen at {0 if self.buf is None else self.buf.numel()} "
                                   f"bytes (captured graph) but this solve needs {nbytes}")
            self.buf = torch.empty(nbytes, dtype=torch.uint8, device=device)
        return self.buf

    def freeze(self):
        """No further growth (a graph captured the buffer's address)."""
        self.frozen = True
        return self

    @classmethod
    def for_stream(cls, device: torch.device) -> "Workspace":
        st = torch.cuda.current_stream(device)
        key = (device, st.cuda_stream)
        ws = cls._shared.get(key)
        if ws is None:
            ws = cls(device)
            cls._shared[key] = ws
        return ws

    @classmethod
    def release(cls):
        for ws in cls._shared.values():
            ws.buf = None
        cls._shared.clear()


def resolve_workspace(workspace, nbytes: int, device: torch.device) -> torch.Tensor:
    """The workspace tensor for one solve: the caller's Workspace, or the
    (device, current stream) default."""
    ws = workspace if workspace is not None else Workspace.for_stream(device)
    return ws.get(nbytes, device)


def as_device_signals(x, device: torch.device, allow_c64: bool = True):
    """(B, N) complex tensor on `device` (no copy when already there).
    complex64 input stays complex64 (storage mode, upconverted in-kernel)."""
    if isinstance(x, torch.Tensor):
        t = x
    else:
        arr = np.asarray(x)
        if arr.dtype != np.complex64 or not allow_c64:
            arr = np.ascontiguousarray(arr, dtype=np.complex128)
        t = torch.from_numpy(np.ascontiguousarray(arr))
    if t.dtype not in (torch.complex128, torch.complex64) or (t.dtype == torch.complex64 and not allow_c64):
        t = t.to(torch.complex128)
    if t.device != device:
        t = t.to(device, non_blocking=True)
    return t.contiguous()


_staging: dict = {}


def _pinned_staging(nbytes: int) -> torch.Tensor:
    """Grow-only pinned host buffer (one cudaHostAlloc per growth, never per
    call: a fresh pinned allocation is a synchronous, slow driver call)."""
    buf = _staging.get("buf")
    if buf is None or buf.numel() < nbytes:
        size = 1 << max(20, (int(nbytes) - 1).bit_length())
        buf = torch.empty(size, dtype=torch.uint8, pin_memory=True)
        _staging["buf"] = buf
    return buf


def host_copy(tensors: dict) -> dict:
    """Device tensors -> host numpy arrays with ONE stream sync: every copy is
    issued non-blocking into a reused pinned staging buffer on the current
    stream, the stream is synchronised once, and the arrays are copied out
    (instead of a sync per .cpu())."""
    items, total, stream = [], 0, None
    for k, t in tensors.items():
        if t.is_cuda:
            stream = torch.cuda.current_stream(t.device)
            nb = t.numel() * t.element_size()
            items.append((k, t, total, nb))
            total += (nb + 255) & ~255
    out = {k: t.numpy() for k, t in tensors.items() if not t.is_cuda}
    if not items:
        return out
    buf = _pinned_staging(total)
    views = {}
    for k, t, off, nb in items:
        v = buf[off:off + nb].view(t.dtype).view(t.shape)
        v.copy_(t, non_blocking=True)
        views[k] = v
    stream.synchronize()
    for k, v in views.items():
        out[k] = v.numpy().copy()
    return out
