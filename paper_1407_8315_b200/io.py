"""SFDT signal files straight to the device, and JSON spectra (SURVEY 8(f)
row 2; format of /root/reference/pkg/src/sfft_dt/io.py:1-70).

Binary signal: little-endian header {magic "SFDT", version u32, n u64}
followed by n interleaved (re, im) float64 samples.  read_signal_device()
reads the payload straight into pinned host memory and copies it to HBM
without an intermediate numpy copy; read_signals_device() stacks many files
into one (B, n) device batch.
"""

from __future__ import annotations

import json
import os
import struct
from pathlib import Path

import numpy as np
import torch

from .spectral import SparseSpectrum

MAGIC = b"SFDT"
VERSION = 1
_HEADER = struct.Struct("<4sIQ")


class FormatError(ValueError):
    """Malformed or truncated signal/spectrum file."""


def _check_header(path, head: bytes, size: int) -> int:
    if len(head) < _HEADER.size:
        raise FormatError(f"{path}: truncated header")
    magic, version, n = _HEADER.unpack_from(head)
    if magic != MAGIC:
        raise FormatError(f"{path}: bad magic {magic!r}")
    if version != VERSION:
        raise FormatError(f"{path}: unsupported version {version}")
    expected = _HEADER.size + 16 * n
    if size != expected:
        raise FormatError(f"{path}: expected {expected} bytes for n={n}, got {size}")
    if n < 2 or n & (n - 1):
        raise FormatError(f"{path}: length {n} is not a power of two >= 2")
    return n


def write_signal(path, x) -> None:
    x = np.ascontiguousarray(x, dtype=np.complex128)
    with open(path, "wb") as fh:
        fh.write(_HEADER.pack(MAGIC, VERSION, x.size))
        fh.write(x.astype("<c16").tobytes())


def read_signal(path) -> np.ndarray:
    """Host read with the reference's validation and messages."""
    raw = Path(path).read_bytes()
    n = _check_header(path, raw[:_HEADER.size], len(raw))
    return np.frombuffer(raw, dtype="<c16", offset=_HEADER.size).astype(np.complex128)


def read_signals_device(paths, device=None) -> torch.Tensor:
    """Read SFDT files into one (B, n) complex128 CUDA tensor: payloads are
    read (os.readv) directly into a pinned staging buffer, then one H2D copy."""
    from .device import require_cuda
    dev = require_cuda(device)
    paths = list(paths)
    ns = []
    for p in paths:
        with open(p, "rb") as fh:
            head = fh.read(_HEADER.size)
        ns.append(_check_header(p, head, os.path.getsize(p)))
    if len(set(ns)) != 1:
        raise FormatError(f"signals of different lengths: {sorted(set(ns))}")
    n = ns[0]
    host = torch.empty((len(paths), n), dtype=torch.complex128).pin_memory()
    buf = host.numpy().view(np.uint8).reshape(len(paths), n * 16)
    for i, p in enumerate(paths):
        with open(p, "rb") as fh:
            fh.seek(_HEADER.size)
            got = fh.readinto(memoryview(buf[i]))
            if got != n * 16:
                raise FormatError(f"{p}: short read")
    return host.to(dev, non_blocking=True)


def read_signal_device(path, device=None) -> torch.Tensor:
    return read_signals_device([path], device)[0]


def write_spectrum(path, spectrum: SparseSpectrum) -> None:
    rows = [{"index": int(s), "re": float(v.real), "im": float(v.imag)}
            for s, v in sorted(spectrum.entries.items())]
    Path(path).write_text(json.dumps(rows, indent=1) + "\n")


def read_spectrum(path, n: int) -> SparseSpectrum:
    try:
        rows = json.loads(Path(path).read_text())
    except json.JSONDecodeError as exc:
        raise FormatError(f"{path}: invalid JSON: {exc}") from exc
    return SparseSpectrum(n, {int(r["index"]): complex(r["re"], r["im"]) for r in rows})
