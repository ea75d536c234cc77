"""Concurrency of the latency path: SolvePipeline / SolveGraph workspaces.

Every SolveGraph owns its workspace (device.Workspace, frozen at capture),
so the graphs of a SolvePipeline run their kernels side by side on their
own streams.  These tests push hundreds of config-1-shaped signals
(N=2^16, K=64; BASELINE.json configs[0]) through pipelines of depth 2..4
and check every result bitwise against one batched solve of the same
signals (a signal's result does not depend on its batch: the kernels are
per-signal), plus the pinned-buffer reuse contract of solve_stream.
Reference semantics: /root/reference/pkg/src/sfft_dt/exact.py:161-200.
"""

import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu

P = pytest.importorskip("paper_1407_8315_b200")


def _signals(count, n=1 << 16, k=64, seed=11):
    from tests.synth import device_exact_batch
    X, _, _ = device_exact_batch(count, n, k, seed, torch.device("cuda"), values="unit")
    return X


def _same(res, want, b):
    h, w = res.to_host(), want.to_host()
    lo, hi = h["entry_offsets"][0], h["entry_offsets"][1]
    wl, wh = w["entry_offsets"][b], w["entry_offsets"][b + 1]
    return (np.array_equal(h["locs"][lo:hi], w["locs"][wl:wh])
            and np.array_equal(h["vals"][lo:hi].view(np.float64), w["vals"][wl:wh].view(np.float64))
            and np.array_equal(h["stats"][0], w["stats"][b]))


@pytest.mark.parametrize("depth,iterative", [(2, False), (4, False), (3, True)])
def test_pipeline_stress_bitwise(depth, iterative):
    """>= 512 pipelined single-signal solves, each bitwise equal to its row of
    one batched solve (entries, values, per-signal stats)."""
    count = 512
    X = _signals(count)
    cfg = P.ExactConfig(n=1 << 16, k=64)
    want = P.exact_batch(X, cfg, iterative)
    want.to_host()
    Xh = X.cpu().pin_memory()
    pipe = P.SolvePipeline(cfg, batch=1, iterative=iterative, depth=depth)
    bad = [b for b, res in enumerate(pipe.solve_stream(Xh[b:b + 1] for b in range(count)))
           if not _same(res, want, b)]
    print(f"depth={depth} iterative={iterative}: {count} signals, {len(bad)} mismatches")
    assert not bad, f"pipelined results differ from the batched solve at {bad[:10]}"


def test_pipeline_reused_pinned_buffer():
    """A producer that refills ONE pinned buffer for every item: solve_stream
    waits for each H2D before handing control back, so nothing is lost."""
    count = 96
    X = _signals(count, seed=12)
    cfg = P.ExactConfig(n=1 << 16, k=64)
    want = P.exact_batch(X, cfg, False)
    want.to_host()
    Xh = X.cpu()
    buf = torch.empty((1, 1 << 16), dtype=torch.complex128, pin_memory=True)

    def produce():
        for b in range(count):
            buf.copy_(Xh[b:b + 1])
            yield buf
    pipe = P.SolvePipeline(cfg, batch=1, depth=3)
    bad = [b for b, res in enumerate(pipe.solve_stream(produce())) if not _same(res, want, b)]
    assert not bad, f"reused-buffer results differ at {bad[:10]}"


def test_pipeline_general_stress():
    """General path (solve_general) through a depth-3 pipeline: 128 signals,
    bitwise equal to the batched solve with the same per-signal seed."""
    from tests.synth import device_general_batch
    n, k, count = 1 << 14, 16, 128
    X = device_general_batch(count, n, k, 20.0, 13, torch.device("cuda"))
    cfg = P.GeneralConfig(n=n, k=k, rng_seed=7)
    want = P.solve_general_batch(X, cfg)
    want.to_host()
    Xh = X.cpu().pin_memory()
    pipe = P.SolvePipeline(cfg, batch=1, depth=3)
    bad = []
    for b, res in enumerate(pipe.solve_stream(Xh[b:b + 1] for b in range(count))):
        h, w = res.to_host(), want.to_host()
        lo, hi = h["entry_offsets"][0], h["entry_offsets"][1]
        wl, wh = w["entry_offsets"][b], w["entry_offsets"][b + 1]
        if not (np.array_equal(h["locs"][lo:hi], w["locs"][wl:wh])
                and np.array_equal(h["vals"][lo:hi].view(np.float64), w["vals"][wl:wh].view(np.float64))):
            bad.append(b)
    assert not bad, f"general pipelined results differ at {bad[:10]}"


def test_graph_workspace_survives_other_solves():
    """A SolveGraph's captured kernels use its own frozen workspace: larger
    solves in between (which grow the shared per-stream workspace) do not
    move or free it, and the replay stays bitwise equal."""
    X = _signals(4, seed=14)
    cfg = P.ExactConfig(n=1 << 16, k=64)
    g = P.SolveGraph(cfg, batch=4)
    first = g.solve(X)
    h0 = {k: v.copy() for k, v in first.to_host().items()}
    big = _signals(64, n=1 << 18, k=128, seed=15)
    P.exact_batch(big, P.ExactConfig(n=1 << 18, k=128), True).to_host()
    del big
    torch.cuda.empty_cache()
    again = g.solve(X).to_host()
    for key in ("entry_offsets", "locs", "stats"):
        assert np.array_equal(h0[key], again[key]), key
    assert np.array_equal(h0["vals"].view(np.float64), again["vals"].view(np.float64))
    assert g.workspace.frozen and g.workspace.buf is not None
