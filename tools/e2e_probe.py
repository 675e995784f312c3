"""Where the e2e step's time goes: dispatch_step on resident inputs, the
HostStepper (pinned H2D + D2H overlapped), and the copies alone (C4 bench
workload, 1 GPU)."""
import sys
import time

import numpy as np
import torch

sys.path.insert(0, ".")
import paper_2509_25401_b200 as fo  # noqa: E402
from bench import random_masks  # noqa: E402

T, S, H, dm = 128, 33024, 24, 3072
t = S // T
dev = torch.device("cuda", 0)
rng = np.random.default_rng(0)
cb, sb = random_masks(rng, H, t, 0.25, 0.5)
g = torch.Generator(device=dev).manual_seed(0)
rn = lambda *s, scale=1.0: torch.randn(*s, device=dev, generator=g) * scale  # noqa: E731
params = fo.LayerParams.from_reference(rn(H, dm, T, scale=dm ** -0.5), rn(H, dm, T, scale=dm ** -0.5),
                                       rn(H, dm, T, scale=dm ** -0.5), 1 + 0.05 * rn(H, T),
                                       1 + 0.05 * rn(H, T), rn(H, T, dm, scale=T ** -0.5))
x = rn(S, dm).bfloat16()
sym = fo.encode_symbols(cb, sb, 1)
cache = fo.FeatureCache(H, t, 1, seq=S)
for _ in range(2):
    cache.push(rn(S, H, T).bfloat16())
_, bias = fo.project_out_update(rn(S, H, T).bfloat16(), params.w_out, sym, cache, 1)
state = fo.LayerState(params=params, cache=cache, symbols=sym, bias=bias)
K = 20


def timeit(fn, label):
    for _ in range(3):
        fn(0)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    c0 = time.perf_counter()
    e0.record()
    for k in range(K):
        fn(k)
    cpu = (time.perf_counter() - c0) * 1e3 / K
    e1.record()
    torch.cuda.synchronize()
    print(f"{label}: {e0.elapsed_time(e1) / K:.3f} ms/step (host enqueue {cpu:.3f} ms/step)")


bufs = {n: torch.empty(S, H, T, dtype=torch.bfloat16, device=dev) for n in ("q", "k", "v", "o")}
bufs["out"] = torch.empty(S, dm, dtype=torch.bfloat16, device=dev)
timeit(lambda k: fo.dispatch_step(state, x, 2, 6, 1, check=False, bufs=bufs), "dispatch_step resident")
xh = [x.cpu().pin_memory() for _ in range(2)]
oh = [torch.empty(S, dm, dtype=torch.bfloat16).pin_memory() for _ in range(2)]
stepper = fo.HostStepper(state, S, dm, device=dev)
timeit(lambda k: stepper.step(xh[k & 1], oh[k & 1], 2, 6, 1), "HostStepper (default-stream events)")
xd = torch.empty(S, dm, dtype=torch.bfloat16, device=dev)
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()


def copies(k):
    with torch.cuda.stream(s1):
        xd.copy_(xh[k & 1], non_blocking=True)
    with torch.cuda.stream(s2):
        oh[k & 1].copy_(bufs["out"], non_blocking=True)
    torch.cuda.current_stream().wait_stream(s1)
    torch.cuda.current_stream().wait_stream(s2)


timeit(copies, "H2D + D2H concurrently")
