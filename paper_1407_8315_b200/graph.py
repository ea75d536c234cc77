"""CUDA-graph replay of a batched solve (latency path for small batches).

A single-signal solve (config 1: N=2^16) is a dozen short kernels; launched
one by one from Python it is bound by host launch overhead, not by the GPU.
SolveGraph captures one complete solve -- exact (solve_noniterative /
solve_iterative) or general (solve_general) -- for a fixed (config, batch,
dtype) into a CUDA graph and replays it:

    g = SolveGraph(ExactConfig(n=1 << 16, k=64), batch=1)
    res = g.solve(x)            # x: (B, n) or (n,) device / host tensor or numpy
    res.spectrum(0), res.trace(0)

    g = SolveGraph(cfg, batch=1, host_io=True)
    g.host_input[0] = x          # pinned staging buffer (or pass x to solve_host)
    res = g.solve_host()         # one H2D copy, then one graph: solve + D2H of the results
    res = g.solve_host(xp)       # xp pinned (B, n): copied to the GPU directly, no staging

The captured kernels are exactly those of exact_batch / solve_general_batch
(same arguments, same library entry points); only their launch is replayed.
Results live in the graph's static buffers: a result is valid until the next
solve() / solve_host() of the same SolveGraph (call .clone() to keep one).
"""

from __future__ import annotations

import numpy as np
import torch

from . import _lib
from .device import Workspace, require_cuda
from .exact import ExactBatch, ExactConfig, exact_batch
from .general import GeneralBatch, GeneralConfig, GeneralPlan, solve_general_batch
from .spectral import check_signal_shape


class SolveGraph:
    def __init__(self, cfg, batch: int = 1, iterative: bool = False,
                 dtype=torch.complex128, device=None, seeds=None, host_io: bool = False):
        if not isinstance(cfg, (ExactConfig, GeneralConfig)):
            raise TypeError("cfg must be an ExactConfig or a GeneralConfig")
        if dtype not in (torch.complex128, torch.complex64):
            raise ValueError("dtype must be torch.complex128 or torch.complex64")
        dev = require_cuda(device)
        n = check_signal_shape((cfg.n,))
        self.cfg, self.batch, self.n, self.device = cfg, int(batch), n, dev
        self.iterative = bool(iterative)
        self.general = isinstance(cfg, GeneralConfig)
        self.plan = GeneralPlan(cfg, self.batch, seeds, dev) if self.general else None
        self.X = torch.zeros((self.batch, n), dtype=dtype, device=dev)
        self.host_io = bool(host_io)
        self.host_input = torch.zeros((self.batch, n), dtype=dtype, pin_memory=True) if host_io else None
        # the graph's own workspace: sized by the warm-up solve, frozen for
        # the capture and referenced for the graph's lifetime (the captured
        # kernels hold its address)
        self.workspace = Workspace(dev)

        # warm-up on a side stream: twiddle tables, the workspace, output
        # capacities and kernel attributes are set up outside the capture
        cur = torch.cuda.current_stream(dev)
        side = torch.cuda.Stream(dev)
        side.wait_stream(cur)
        with torch.cuda.stream(side):
            self._launch()
        cur.wait_stream(side)
        torch.cuda.synchronize(dev)
        self.workspace.freeze()

        self.graph = torch.cuda.CUDAGraph()
        with torch.cuda.graph(self.graph):
            # host_io: the H2D is issued before each replay (from the caller's
            # pinned tensor directly, or from host_input), not captured, so a
            # pinned batch is never staged through a host-side memcpy
            proto = self._launch()
            self.t = proto.t
            self.kernel_launches = proto.kernel_launches
            if host_io:
                # results back into one pinned buffer (whole capacity; the
                # offsets say how much of each list is used): the result
                # tensors are packed on the device into one byte buffer and
                # read back by ONE copy (seven small D2H copies cost ~4 us
                # each).  Widest element types first keep every segment
                # aligned for its dtype view.
                keys = sorted((k for k, v in self.t.items()
                               if isinstance(v, torch.Tensor) and not k.startswith("_")),
                              key=lambda k: -self.t[k].element_size())
                flat = [self.t[k].contiguous().reshape(-1).view(torch.uint8) for k in keys]
                self._dev_pack = torch.cat(flat)
                self._host_pack = torch.empty(self._dev_pack.numel(), dtype=torch.uint8, pin_memory=True)
                self._host_pack.copy_(self._dev_pack, non_blocking=True)
                self._host_out, off = {}, 0
                for k, f in zip(keys, flat):
                    v = self.t[k]
                    self._host_out[k] = self._host_pack[off:off + f.numel()].view(v.dtype).reshape(v.shape)
                    off += f.numel()
                self._host_np = {k: v.numpy() for k, v in self._host_out.items()}
        torch.cuda.synchronize(dev)

    def _launch(self):
        if self.general:
            return solve_general_batch(self.X, self.cfg, device=self.device, plan=self.plan,
                                       workspace=self.workspace)
        return exact_batch(self.X, self.cfg, self.iterative, self.device, workspace=self.workspace)

    def _wrap(self):
        if self.general:
            res = GeneralBatch(self.n, self.cfg, self.cfg.resolved_d(), min(self.cfg.r, self.cfg.resolved_d()),
                               self.plan.sh, self.t, 0.0, self.kernel_launches)
        else:
            res = ExactBatch(self.n, self.iterative, self.t, 0.0)
            res.kernel_launches = self.kernel_launches
        return res

    def solve(self, X=None):
        """Replay on the current stream; X (optional) is copied into the
        graph's input buffer first (device-to-device, or host-to-device).
        Returns device-resident results (ExactBatch / GeneralBatch)."""
        if X is not None:
            if not isinstance(X, torch.Tensor):
                X = torch.from_numpy(np.ascontiguousarray(X))
            self.X.copy_(X.reshape(self.X.shape), non_blocking=True)
        self.graph.replay()
        return self._wrap()

    def solve_host(self, x=None):
        """host_io graphs: H2D of host_input, the solve and the D2H of every
        result buffer as ONE graph replay, then one stream sync.  x (optional)
        is first copied into the pinned host_input."""
        if not self.host_io:
            raise ValueError("SolveGraph was built without host_io=True")
        src = self.host_input
        if x is not None:
            if not isinstance(x, torch.Tensor):
                x = torch.from_numpy(np.ascontiguousarray(x))
            if (x.device.type == "cpu" and x.is_pinned() and x.dtype == self.host_input.dtype
                    and x.is_contiguous() and x.numel() == self.host_input.numel()):
                src = x.reshape(self.host_input.shape)   # H2D straight from the caller's pinned rows
            else:
                self.host_input.copy_(x.reshape(self.host_input.shape))
        self.X.copy_(src, non_blocking=True)
        self.graph.replay()
        torch.cuda.current_stream(self.device).synchronize()
        res = self._wrap()
        res._host = _host_view(self._host_np, self.general)
        return res

    @property
    def h2d_bytes(self) -> int:
        return self.X.numel() * self.X.element_size()


class SolvePipeline:
    """A stream of small solves through `depth` host-IO SolveGraphs, each on
    its own CUDA stream and with its own workspace, so the H2D of one batch
    and the kernels of the previous ones run side by side (the copy engine
    and the SMs work concurrently, and independent solves share the SMs).

        pipe = SolvePipeline(ExactConfig(n=1 << 16, k=64), batch=1)
        for res in pipe.solve_stream(xs):   # xs: iterable of (B, n) inputs
            res.spectrum(0)                 # valid until the next result is drawn

    Results come back in submission order; each is the same as
    SolveGraph.solve_host on that input.  A pinned contiguous input is copied
    to the GPU straight from the caller's memory; solve_stream waits for that
    copy to finish before it hands control back to the caller, so a producer
    may refill one pinned buffer for every item.  hold_inputs=True skips that
    wait: the caller then guarantees each input stays unchanged until its
    result has been drawn."""

    def __init__(self, cfg, batch: int = 1, iterative: bool = False,
                 dtype=torch.complex128, device=None, seeds=None, depth: int = 2):
        if depth < 1:
            raise ValueError("depth must be >= 1")
        self.graphs = [SolveGraph(cfg, batch, iterative, dtype, device, seeds, host_io=True)
                       for _ in range(depth)]
        dev = self.graphs[0].device
        self.streams = [torch.cuda.Stream(dev) for _ in range(depth)]
        self.h2d_done = [torch.cuda.Event() for _ in range(depth)]
        self.done = [torch.cuda.Event() for _ in range(depth)]
        for st, e1, e2 in zip(self.streams, self.h2d_done, self.done):
            e1.record(st)   # materialise the event handles
            e2.record(st)
        torch.cuda.synchronize(dev)
        # raw handles for sfdt_graph_submit: H2D + event + graph launch +
        # event in one native call per item
        self._raw = [(g.X.data_ptr(), g.X.numel() * g.X.element_size(), g.graph.raw_cuda_graph_exec(),
                      st.cuda_stream, e1.cuda_event, e2.cuda_event)
                     for g, st, e1, e2 in zip(self.graphs, self.streams, self.h2d_done, self.done)]
        self._lib = _lib.load()

    def _submit(self, slot: int, x):
        g = self.graphs[slot]
        if not isinstance(x, torch.Tensor):
            x = torch.from_numpy(np.ascontiguousarray(x))
        if not (x.device.type == "cpu" and x.dtype == g.host_input.dtype and x.is_contiguous()
                and x.numel() == g.host_input.numel() and x.is_pinned()):
            g.host_input.copy_(x.reshape(g.host_input.shape))
            x = g.host_input
        dst, nbytes, gexec, st, e1, e2 = self._raw[slot]
        _lib.check(self._lib.sfdt_graph_submit(x.data_ptr(), dst, nbytes, gexec, st, e1, e2),
                   "sfdt_graph_submit")

    def _collect(self, slot: int):
        self.done[slot].synchronize()
        g = self.graphs[slot]
        res = g._wrap()
        res._host = _host_view(g._host_np, g.general)
        return res

    def solve_stream(self, xs, hold_inputs: bool = False):
        depth = len(self.graphs)
        pending = []   # slots in submission order
        for i, x in enumerate(xs):
            slot = i % depth
            if len(pending) == depth:   # the slot's previous result is drawn first
                yield self._collect(pending.pop(0))
            self._submit(slot, x)
            pending.append(slot)
            if not hold_inputs:
                # the caller regains control (next item / next result) only
                # once x has been read
                self.h2d_done[slot].synchronize()
        while pending:
            yield self._collect(pending.pop(0))


def _host_view(full: dict, general: bool) -> dict:
    """Slice whole-capacity host copies down to the used prefixes (the layout
    ExactBatch.to_host / GeneralBatch.to_host produce)."""
    h = {"entry_offsets": full["entry_offsets"], "stats": full["stats"]}
    total = int(full["entry_offsets"][-1])
    h["locs"] = full["locs"][:total]
    h["vals"] = full["vals"][:total].reshape(-1, 2).view(np.complex128).reshape(-1)
    if general:
        return h
    h["unres_offsets"] = full["unres_offsets"]
    h["unres_bins"] = full["unres_bins"][:int(full["unres_offsets"][-1])]
    h["rms"] = full["rms"]
    if full.get("dup_offsets") is not None:
        h["dup_offsets"] = full["dup_offsets"]
        h["dup_locs"] = full["dup_locs"][:int(full["dup_offsets"][-1])]
    return h
