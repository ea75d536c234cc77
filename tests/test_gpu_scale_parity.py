"""Departures from the reference's arithmetic, counted at scale (VERDICT r01
"Next round" item 3).

The general path replaces three LAPACK calls of the reference with device
code: closed-form 3x3 singular values where they are accurate, a Jacobi
that stops at eps-level convergence instead of 60 sweeps at 1e-17
(_core.pyx:353-406), and a Householder-QR least squares instead of gelsd
(general.py:241).  Each moves values by roundoff only, but a singular value
within roundoff of the K-th largest could flip a vote, and a flipped vote
changes a support.  These tests run the oracle over hundreds of signals on
every host core and count vote, support and value mismatches -- the bar is
zero of each (values within 1e-9), except where the reference's own choice
is a roundoff tie (matched_filter_ties below: counted and reported).

The exact path is counted the same way at config 2 (64 signals, both
solvers; SURVEY 8(c) rules 2-3 as in test_gpu_configs.py).
"""

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = [pytest.mark.gpu, pytest.mark.slow]

if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("needs a CUDA device", allow_module_level=True)

import paper_1407_8315_b200 as P                                   # noqa: E402
from tests import oracle_pool                                       # noqa: E402
from tests.synth import device_exact_batch, device_general_batch   # noqa: E402
from tests.test_gpu_configs import _envelope, _exact_compare       # noqa: E402


def _SCALE(default, full):
    """Signals compared per test: `default`, or every signal of the batch with
    SFDT_SCALE_FULL=1 (a one-off campaign, results under profiles/)."""
    import os
    return full if os.environ.get("SFDT_SCALE_FULL") == "1" else default
from tests.test_gpu_parity import VAL_RTOL, _m_levels              # noqa: E402

DEV = torch.device("cuda", 0)
TIE_RTOL = 1e-12


def matched_filter_ties(gl, gv, locs, vals, wtr, n, L):
    """Support differences of one signal that are roundoff ties of the
    reference itself: in every differing bin, each column only one side
    picked scores within TIE_RTOL of a column only the other side picked in
    the oracle's own matched filter (|base_phi^H w|, general.py:345-351 --
    numpy/BLAS summation order decides such a tie), and the values agree in
    magnitude.  Happens when every random shift is odd: column c and
    c + d/2 then have phi columns that are exact negatives, so the data
    cannot tell loc from loc + n/2.  Returns the number of such bins, or
    raises AssertionError for a difference that is not a tie."""
    go = {int(s): complex(v) for s, v in zip(gl, gv)}
    wo = {int(s): complex(v) for s, v in zip(locs, vals)}
    diff_bins = sorted({s % L for s in set(go) ^ set(wo)})
    for kb in diff_bins:
        sc = np.asarray(wtr["mf_scores"][kb])
        cg = {((s - kb) % n) // L: v for s, v in go.items() if s % L == kb}
        co = {((s - kb) % n) // L: v for s, v in wo.items() if s % L == kb}
        only_g, only_o = set(cg) - set(co), set(co) - set(cg)
        assert len(only_g) == len(only_o), (kb, cg, co)
        for c in only_g:
            partner = [o for o in only_o if abs(sc[c] - sc[o]) <= TIE_RTOL * sc[o]]
            assert partner, f"bin {kb}: column {c} (score {sc[c]!r}) ties none of {only_o}"
            assert abs(abs(cg[c]) - abs(co[partner[0]])) <= VAL_RTOL * abs(co[partner[0]])
    return len(diff_bins)


@pytest.mark.parametrize("snr", [20.0, 10.0])
def test_general_cfg4_256_signals(snr):
    """Config 4 (N=2^20, K=128, per-signal shift seeds): 256 signals of one
    1024-signal batch against the oracle -- vote flips, support differences,
    dict-order differences and values over 1e-9 counted (all must be 0)."""
    n, k, B, S = 1 << 20, 128, 1024, _SCALE(256, 1024)
    X = device_general_batch(B, n, k, snr, 4000 + int(snr), DEV)
    cfg = P.GeneralConfig(n=n, k=k)
    seeds = [(4000 + int(snr), b) for b in range(B)]
    res = P.solve_general_batch(X, cfg, seeds=seeds)
    votes = res.votes()
    h = res.to_host()
    idx = list(range(0, B, B // S))
    host = {b: X[b].cpu().numpy() for b in idx}
    del X
    torch.cuda.empty_cache()
    out = oracle_pool.run(host, [(b, "general", dict(k=k, rng_seed=seeds[b], return_internals=True))
                                 for b in idx])
    vote_flips = sup_diff = order_diff = val_over = entries = tie_bins = tie_signals = 0
    worst = 0.0
    L = n // cfg.resolved_d()
    for b, _, locs, vals, wtr in out:
        vote_flips += int(np.count_nonzero(votes[b] != np.asarray(wtr["votes"])))
        lo, hi = h["entry_offsets"][b], h["entry_offsets"][b + 1]
        gl, gv = h["locs"][lo:hi], h["vals"][lo:hi]
        if set(gl.tolist()) != set(locs.tolist()):
            tie_bins += matched_filter_ties(gl, gv, locs, vals, wtr, n, L)
            tie_signals += 1
            continue
        sup_diff += len(set(gl.tolist()) ^ set(locs.tolist()))
        if np.array_equal(gl, locs):
            rel = np.abs(gv - vals) / np.abs(vals)
            val_over += int(np.count_nonzero(rel > VAL_RTOL))
            worst = max(worst, float(rel.max()) if rel.size else 0.0)
        else:
            order_diff += 1
        entries += len(locs)
    print(f"cfg4 {snr:.0f} dB: {len(idx)} signals, {entries} entries, {len(idx) * votes.shape[1]} votes: "
          f"vote flips {vote_flips}, support differences {sup_diff}, order differences {order_diff}, "
          f"values > 1e-9: {val_over} (max rel {worst:.2e}); matched-filter roundoff ties of the "
          f"reference itself: {tie_bins} bins in {tie_signals} signals")
    assert vote_flips == 0 and sup_diff == 0 and order_diff == 0 and val_over == 0


@pytest.mark.parametrize("solver", ["noniterative", "iterative"])
def test_exact_cfg2_64_signals(solver):
    """Config 2 (N=2^20, K=256, |v| in [1,10]): 64 signals of a 512-signal
    batch against the oracle (with the reference's numpy-backend envelope)."""
    n, k, B, S = 1 << 20, 256, 512, _SCALE(64, 512)
    X, _, _ = device_exact_batch(B, n, k, 2200, DEV, values="mag1_10")
    cfg = P.ExactConfig(n=n, k=k)
    res = P.exact_batch(X, cfg, solver == "iterative")
    idx = list(range(0, B, B // S))
    host = {b: X[b].cpu().numpy() for b in idx}
    del X
    torch.cuda.empty_cache()
    out = oracle_pool.run(host, [(b, solver, dict(k=k, kernels=kern)) for kern in ("port", "numpy")
                                 for b in idx])
    half = len(out) // 2
    numpy_runs = {b: (locs, vals) for b, _, locs, vals, _ in out[half:]}
    levels = _m_levels(n, cfg.resolved_d(), 4, solver == "iterative")
    sym = tot = 0
    worst1 = worst_m = 0.0
    for b, _, locs, vals, wtr in out[:half]:
        env = _envelope(locs, vals, *numpy_runs[b])
        c, t, r1, rm = _exact_compare(res.spectrum(b), res.trace(b), locs, vals, wtr, env,
                                      numpy_runs[b][0], n, levels, f"cfg2 {solver} b={b}")
        sym, tot, worst1, worst_m = sym + c, tot + t, max(worst1, r1), max(worst_m, rm)
    print(f"cfg2 {solver}: {len(idx)} signals, {tot} entries, symmetric difference {sym}, "
          f"single-frequency max rel {worst1:.2e}, multi-frequency max rel/bound {worst_m:.2e}")
    assert sym == 0
