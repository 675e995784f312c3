"""Device timing of one operator call for the sweeps: `reps` calls captured
into a CUDA graph (the engine replays its steps the same way, engine.py), the
graph replayed `trials` times, median ms per call by CUDA events. Without the
graph a Python wrapper's launch cost (tens of us) would be timed instead of
the kernels whenever a call is shorter than it (GEMMs at high sparsity, S=4096,
FLUX attention)."""

import numpy as np
import torch


def graph_time(fn, reps=10, trials=5, warm=3):
    for _ in range(warm):
        fn()
    torch.cuda.synchronize()
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    g = torch.cuda.CUDAGraph()
    with torch.cuda.stream(s):
        fn()  # warm on the capture stream (first-use allocations)
        s.synchronize()
        with torch.cuda.graph(g, stream=s):
            for _ in range(reps):
                fn()
    torch.cuda.synchronize()
    g.replay()
    torch.cuda.synchronize()
    res = []
    for _ in range(trials):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        g.replay()
        e1.record()
        torch.cuda.synchronize()
        res.append(e0.elapsed_time(e1) / reps)
    del g
    return float(np.median(res))


def eager_time(fn, reps=10, trials=5, warm=3):
    for _ in range(warm):
        fn()
    torch.cuda.synchronize()
    res = []
    for _ in range(trials):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(reps):
            fn()
        e1.record()
        torch.cuda.synchronize()
        res.append(e0.elapsed_time(e1) / reps)
    return float(np.median(res))
