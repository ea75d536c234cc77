"""Seeded synthetic workloads for the BASELINE.json configs (test/bench setup,
not the hot path).

No public dataset is involved: every input is a seeded synthetic signal with
the shapes and value distributions BASELINE.json names.

* ``exact_signal(n, k, seed, values)`` -- exactly K-sparse spectrum on a
  uniform support; ``values`` is "unit" (|v| = 1, uniform phase; configs 1,
  3, 5), "mag1_10" (|v| ~ U[1, 10], uniform phase; config 2) or "gauss".
  With ``synth="radix2"`` the time signal is the reference's own radix-2
  inverse (oracle restatement, bit-identical to `gen_exact`,
  /root/reference/pkg/src/sfft_dt/signals.py:61-72); otherwise N*ifft.
* ``general_signal(n, k, snr_db, seed)`` -- K unit-magnitude random-phase
  tones plus time-domain circular Gaussian noise at the given SNR
  (configs 4 and 5-general).
"""

from __future__ import annotations

import numpy as np


def _support_values(rng, n, k, values):
    support = rng.choice(n, size=k, replace=False)
    if values == "unit":
        vals = np.exp(2j * np.pi * rng.random(k))
    elif values == "mag1_10":
        mag = rng.uniform(1.0, 10.0, k)
        vals = mag * np.exp(2j * np.pi * rng.random(k))
    elif values == "logmag":
        # magnitudes spread over 8 decades: a tone ~1e-7 of its bin partner
        # passes the a = 1 consistency test (1e-6), so the iterative solver
        # later re-decodes the leftover at the same location (the
        # duplicate-overwrite path, exact.py:152-158)
        mag = 10.0 ** rng.uniform(-8.0, 0.0, k)
        vals = mag * np.exp(2j * np.pi * rng.random(k))
    elif values == "gauss":
        vals = (rng.standard_normal(k) + 1j * rng.standard_normal(k)) / np.sqrt(2.0)
    else:
        raise ValueError(values)
    return support, vals


def exact_signal(n, k, seed=0, values="unit", synth="numpy"):
    """Returns (x, truth dict)."""
    rng = np.random.default_rng(seed)
    support, vals = _support_values(rng, n, k, values)
    dense = np.zeros(n, dtype=np.complex128)
    dense[support] = vals
    if synth == "radix2":
        from oracle.kernels import fft_radix2
        x = fft_radix2(dense, inverse=True)
    else:
        x = np.fft.ifft(dense) * n
    return x, {int(s): complex(v) for s, v in zip(support, vals)}


def general_signal(n, k, snr_db, seed=0):
    """K unit tones + circular Gaussian noise with sigma^2 = P_sig / 10^(snr/10)."""
    rng = np.random.default_rng(seed)
    support, vals = _support_values(rng, n, k, "unit")
    dense = np.zeros(n, dtype=np.complex128)
    dense[support] = vals
    clean = np.fft.ifft(dense) * n
    p_sig = float(np.mean(np.abs(clean) ** 2))
    sigma2 = p_sig / 10.0 ** (snr_db / 10.0)
    noise = np.sqrt(sigma2 / 2.0) * (rng.standard_normal(n) + 1j * rng.standard_normal(n))
    return clean + noise, {int(s): complex(v) for s, v in zip(support, vals)}


def device_exact_batch(batch, n, k, seed, device, values="mag1_10"):
    """Config-2-sized batches generated on the GPU (the host generator would
    take minutes for 64 GiB): per signal a uniform K-subset support (top-K of
    uniform keys), |v| ~ U[1, 10] (or 1) with uniform phase, x = N * ifft.
    Returns (X (B, n) complex128 on `device`, support (B, K) int64 numpy,
    values (B, K) complex128 numpy).  Setup only -- cuFFT synthesizes the
    inputs; the solver under test never calls it."""
    import math

    import torch
    X = torch.empty((batch, n), dtype=torch.complex128, device=device)
    g = torch.Generator(device=device)
    g.manual_seed(seed)
    sup = np.empty((batch, k), np.int64)
    val = np.empty((batch, k), np.complex128)
    ch = max(1, min(128, (1 << 27) // n))
    for lo in range(0, batch, ch):
        hi = min(batch, lo + ch)
        r = torch.rand((hi - lo, n), generator=g, device=device, dtype=torch.float32)
        idx = torch.topk(r, k, dim=1).indices
        del r
        if values == "mag1_10":
            mag = 1.0 + 9.0 * torch.rand((hi - lo, k), generator=g, device=device, dtype=torch.float64)
        else:
            mag = torch.ones((hi - lo, k), device=device, dtype=torch.float64)
        ph = 2 * math.pi * torch.rand((hi - lo, k), generator=g, device=device, dtype=torch.float64)
        v = torch.polar(mag, ph)
        dense = torch.zeros((hi - lo, n), dtype=torch.complex128, device=device)
        dense.scatter_(1, idx, v)
        X[lo:hi] = torch.fft.ifft(dense, dim=1) * n
        del dense
        sup[lo:hi] = idx.cpu().numpy()
        val[lo:hi] = v.cpu().numpy()
    return X, sup, val


def device_general_batch(batch, n, k, snr_db, seed, device):
    """Config-4-sized noisy batches generated on the GPU: K unit tones with
    uniform phase + time-domain circular Gaussian noise at snr_db (the
    config-4 model of SURVEY.md 8(d)).  Returns X (B, n) complex128."""
    import math

    import torch
    X = torch.empty((batch, n), dtype=torch.complex128, device=device)
    g = torch.Generator(device=device)
    g.manual_seed(seed)
    ch = max(1, min(128, (1 << 27) // n))
    for lo in range(0, batch, ch):
        hi = min(batch, lo + ch)
        r = torch.rand((hi - lo, n), generator=g, device=device, dtype=torch.float32)
        idx = torch.topk(r, k, dim=1).indices
        del r
        ph = 2 * math.pi * torch.rand((hi - lo, k), generator=g, device=device, dtype=torch.float64)
        dense = torch.zeros((hi - lo, n), dtype=torch.complex128, device=device)
        dense.scatter_(1, idx, torch.polar(torch.ones_like(ph), ph))
        x = torch.fft.ifft(dense, dim=1) * n
        del dense
        p_sig = (x.real ** 2 + x.imag ** 2).mean(dim=1, keepdim=True)
        sigma = torch.sqrt(p_sig / 10 ** (snr_db / 10) / 2)
        nr = torch.randn((hi - lo, n), generator=g, device=device, dtype=torch.float64)
        ni = torch.randn((hi - lo, n), generator=g, device=device, dtype=torch.float64)
        X[lo:hi] = x + sigma * torch.complex(nr, ni)
        del x, nr, ni
    return X
