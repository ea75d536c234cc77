"""Experiment grids on the GPU (mirror of
/root/reference/pkg/src/sfft_dt/experiments.py:81-216).

Trials of one grid cell are generated on the host with the reference's
generators (seeded numpy, synthesis by the bit-identical device radix-2
inverse) and solved as ONE batch on the B200, instead of one signal per
GIL-bound thread.  Rows carry the same fields and seed tuples as the
reference's, so any cell replays exactly; `elapsed_s` is the batch time
divided by the trials.
"""

from __future__ import annotations

import csv
import json
import math
import time
from dataclasses import dataclass, field

import numpy as np

from .exact import ExactConfig, exact_batch
from .general import GeneralConfig, solve_general_batch
from .spectral import SparseSpectrum, snr, synthesize


@dataclass
class ExperimentReport:
    name: str
    meta: dict = field(default_factory=dict)
    rows: list = field(default_factory=list)

    def write_csv(self, path) -> None:
        if not self.rows:
            raise ValueError("no rows to write")
        with open(path, "w", newline="") as fh:
            w = csv.DictWriter(fh, fieldnames=list(self.rows[0].keys()))
            w.writeheader()
            w.writerows(self.rows)

    def write_json(self, path) -> None:
        with open(path, "w") as fh:
            json.dump({"name": self.name, "meta": self.meta, "rows": self.rows}, fh, indent=1)


def lemma_collision_bound(n: int, d: int, k: int, a_max: int) -> float:
    """P(some bin holds > a_max frequencies) <= (n/d)(d e k/(n(a_max+1)))^(a_max+1)."""
    return (n / d) * (d * math.e * k / (n * (a_max + 1))) ** (a_max + 1)


def partial_recovery_floor(n: int, d: int, k: int, a_max: int, tau: float, mu: int):
    frac_bad = tau / mu - 1.0 / (mu * k)
    inner = (d * k / n) ** a_max * math.e ** (a_max + 2) / (tau * (a_max + 1) ** (a_max + 1))
    return (1.0 - frac_bad) * n, 1.0 - inner ** (tau * k)


def gen_exact(n: int, k: int, seed, values: str = "unit_phase"):
    """signals.py:61-72: uniform support, unit-phase (or circular normal)
    values, time signal by the radix-2 inverse; returns (x, truth)."""
    rng = np.random.default_rng(seed)
    support = rng.choice(n, size=k, replace=False)
    if values == "unit_phase":
        vals = np.exp(2j * np.pi * rng.random(k))
    else:
        vals = (rng.standard_normal(k) + 1j * rng.standard_normal(k)) / np.sqrt(2.0)
    truth = SparseSpectrum(n, {int(s): complex(v) for s, v in zip(support, vals)})
    return synthesize(truth.to_dense()), truth


def gen_mixture(n: int, k: int, sigma_on: float, sigma_off: float, seed):
    """signals.py:75-85: two-component circular Gaussian mixture spectrum;
    returns (x, significant top-k part, full spectrum)."""
    rng = np.random.default_rng(seed)
    on = rng.random(n) < k / n
    sigma = np.where(on, sigma_on, sigma_off)
    full = sigma * ((1.0 / np.sqrt(2.0)) * (rng.standard_normal(n) + 1j * rng.standard_normal(n)))
    order = np.argpartition(np.abs(full), n - k)[n - k:]
    significant = SparseSpectrum(n, {int(s): complex(full[s]) for s in order})
    return synthesize(full), significant, full


def sigma_off_for_snr(n: int, k: int, snr_db: float, sigma_on: float = 1.0) -> float:
    if not 0 < k < n:
        raise ValueError("need 0 < k < n")
    return sigma_on * np.sqrt(k / ((n - k) * 10.0 ** (snr_db / 10.0)))


def run_exact_grid(n: int, k_values, trials: int = 100, mu: int = 4, a_max: int = 4,
                   solver: str = "iterative", seed: int = 0, device=None) -> ExperimentReport:
    """experiments.py:118-141: per k, `trials` exactly sparse signals solved
    as one GPU batch; perfect / recovered_fraction / full_success rows."""
    report = ExperimentReport("exact_grid", {"n": n, "k_values": list(k_values), "trials": trials,
                                             "mu": mu, "a_max": a_max, "solver": solver,
                                             "seed": seed})
    for k in k_values:
        sigs = [gen_exact(n, k, (seed, k, t)) for t in range(trials)]
        X = np.stack([s[0] for s in sigs])
        cfg = ExactConfig(n=n, k=k, mu=mu, a_max=a_max)
        t0 = time.perf_counter()
        res = exact_batch(X, cfg, solver == "iterative", device)
        res.to_host()
        elapsed = (time.perf_counter() - t0) / trials
        for t, (_, truth) in enumerate(sigs):
            spec, tr = res.spectrum(t), res.trace(t)
            correct = sum(1 for s, v in truth.entries.items()
                          if s in spec.entries and abs(spec.entries[s] - v) <= 1e-7 * abs(v))
            spurious = len(set(spec.entries) - set(truth.entries))
            report.rows.append({
                "n": n, "k": k, "mu": mu, "a_max": a_max, "solver": solver,
                "seed": str((seed, k, t)), "perfect": int(correct == k and spurious == 0),
                "recovered_fraction": (n - (k - correct) - spurious) / n,
                "full_success": int(tr.full_success), "fft_samples": tr.fft_samples,
                "elapsed_s": elapsed})
    return report


def run_general_grid(n: int, n_over_k_values, snr_db_values, trials: int = 50, a_max: int = 3,
                     compare_pruning: bool = True, seed: int = 0, device=None) -> ExperimentReport:
    """experiments.py:144-216: per (N/K, SNR) cell, `trials` mixture signals
    solved as one GPU batch with and without pruning (paired shift seeds)."""
    report = ExperimentReport("general_grid", {
        "n": n, "n_over_k_values": list(n_over_k_values), "snr_db_values": list(snr_db_values),
        "trials": trials, "a_max": a_max, "seed": seed, "compare_pruning": compare_pruning})
    for nk in n_over_k_values:
        k = n // nk
        for snr_db in snr_db_values:
            seeds = [(seed, nk, snr_db, t) for t in range(trials)]
            sigs = [gen_mixture(n, k, 1.0, sigma_off_for_snr(n, k, snr_db), s) for s in seeds]
            X = np.stack([s[0] for s in sigs])
            rows = []
            for (_, significant, full), s in zip(sigs, seeds):
                noise = float(np.linalg.norm(full - significant.to_dense()))
                rows.append({"n": n, "n_over_k": nk, "k": k, "snr_target_db": snr_db, "a_max": a_max,
                             "seed": str(s), "snr_significant_db": snr(full, significant),
                             "noise_norm": noise})
            variants = [("prune", True)] + ([("noprune", False)] if compare_pruning else [])
            for label, prune in variants:
                cfg = GeneralConfig(n=n, k=k, a_max=a_max, prune=prune)
                t0 = time.perf_counter()
                res = solve_general_batch(X, cfg, seeds=seeds, device=device)
                res.to_host()
                elapsed = (time.perf_counter() - t0) / trials
                for t, row in enumerate(rows):
                    full = sigs[t][2]
                    spec = res.spectrum(t)
                    err = float(np.linalg.norm(full - spec.to_dense()))
                    row[f"snr_out_db_{label}"] = snr(full, spec)
                    row[f"error_ratio_{label}"] = err / row["noise_norm"] if row["noise_norm"] else math.inf
                    row[f"elapsed_s_{label}"] = elapsed
                    row[f"d_{label}"] = res.d
            report.rows.extend(rows)
    return report


def summarize_general(report: ExperimentReport) -> list:
    """experiments.py:219-233: per (N/K, SNR) cell, the mean of every snr_* /
    error_ratio* / elapsed* column over the cell's finite values."""
    cells = {}
    for row in report.rows:
        cells.setdefault((row["n_over_k"], row["snr_target_db"]), []).append(row)
    out = []
    for (n_over_k, snr_db), rows in sorted(cells.items()):
        entry = {"n_over_k": n_over_k, "snr_target_db": snr_db, "trials": len(rows)}
        for key in rows[0]:
            if key.startswith(("snr_", "error_ratio", "elapsed")):
                vals = [r[key] for r in rows if math.isfinite(r[key])]
                entry[f"mean_{key}"] = float(np.mean(vals)) if vals else math.inf
        out.append(entry)
    return out


def run_collision_census(n: int, k: int, n_plus_values, trials: int = 1000, seed: int = 0,
                         a_cap: int = 4) -> dict:
    """experiments.py:81-111: empirical per-bin collision histograms (host
    integer counting; no solve involved)."""
    results = {}
    for idx, n_plus in enumerate(n_plus_values):
        dk = n // n_plus
        if dk * n_plus != n or dk % k:
            raise ValueError(f"n_plus={n_plus} incompatible with n={n}, k={k}")
        d = dk // k
        m = n // d
        hist = np.zeros(min(k, d) + 1, dtype=np.int64)
        over = 0
        for t in range(trials):
            support = np.random.default_rng((seed, idx, t)).choice(n, size=k, replace=False)
            counts = np.bincount(support % m, minlength=m)
            hist[: counts.max() + 1] += np.bincount(counts)
            over += int(counts.max() > a_cap)
        prob = hist / (trials * m)
        results[n_plus] = {"d": d, "per_bin_probability": prob,
                           "p_bin_over": float(prob[a_cap + 1:].sum()),
                           "p_signal_over": over / trials,
                           "bound_signal_over": lemma_collision_bound(n, d, k, a_cap),
                           "trials": trials}
    return results
