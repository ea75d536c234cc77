"""Host/GPU timing of SolvePipeline internals at config 1 (diagnostic)."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_1407_8315_b200 as P
from tests.synth import device_exact_batch
X, _, _ = device_exact_batch(64, 1 << 16, 64, 11, torch.device("cuda"), values="unit")
cfg = P.ExactConfig(n=1 << 16, k=64)
Xh = X.cpu().pin_memory()
for depth in (1, 2, 4):
    pipe = P.SolvePipeline(cfg, batch=1, depth=depth)
    for r in pipe.solve_stream(Xh[b:b+1] for b in range(16)): pass
    torch.cuda.synchronize()
    # host cost of each piece
    g, st = pipe.graphs[0], pipe.streams[0]
    t0 = time.perf_counter(); 
    for i in range(200): Xh[i % 64:i % 64 + 1].is_pinned()
    t1 = time.perf_counter()
    for i in range(200):
        with torch.cuda.stream(st): g.X.copy_(Xh[i % 64:i % 64+1], non_blocking=True)
    t2 = time.perf_counter(); torch.cuda.synchronize()
    t3 = time.perf_counter()
    for i in range(200):
        with torch.cuda.stream(st): g.graph.replay()
    t4 = time.perf_counter(); torch.cuda.synchronize(); t5 = time.perf_counter()
    for i in range(200): pipe._submit(i % depth, Xh[i % 64:i % 64 + 1]); 
    t6 = time.perf_counter(); torch.cuda.synchronize(); t7 = time.perf_counter()
    for i in range(200): pipe._collect(i % depth)
    t8 = time.perf_counter()
    print(f"depth {depth}: is_pinned {(t1-t0)/200*1e6:.1f} us, h2d issue {(t2-t1)/200*1e6:.1f} us, replay issue {(t4-t3)/200*1e6:.1f} us (gpu {(t5-t3)/200*1e6:.1f} us/replay serial), submit {(t6-t5)/200*1e6:.1f} us (all done {(t7-t5)/200*1e6:.1f} us/item), collect {(t8-t7)/200*1e6:.1f} us")
    # GPU overlap: timed events around replays on different streams
    evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(depth)]
    torch.cuda.synchronize()
    for s in range(depth):
        with torch.cuda.stream(pipe.streams[s]):
            evs[s][0].record(); pipe.graphs[s].graph.replay(); evs[s][1].record()
    torch.cuda.synchronize()
    print("   replay intervals (ms rel. to slot 0 start):", [(round(evs[0][0].elapsed_time(a), 4), round(evs[0][0].elapsed_time(b), 4)) for a, b in evs])
    for hold in (False, True):
        t0 = time.perf_counter(); n = 0
        for r in pipe.solve_stream((Xh[b % 64:b % 64 + 1] for b in range(2000)), hold_inputs=hold): n += 1
        dt = time.perf_counter() - t0
        print(f"   solve_stream hold={hold}: {n/dt:.0f} signals/s ({dt/n*1e6:.1f} us/signal)")
