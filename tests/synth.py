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
