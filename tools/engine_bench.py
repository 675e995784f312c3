"""Update-Dispatch scheduler (engine.run) at C4 on one B200: per-phase device
time of the GPU run() loop (policy-derived symbols, CUDA-graph dispatch).

    python tools/engine_bench.py [--layers 1] [--steps 13] [--tau-q 0.3] [--tau-kv 0.5]
"""

import argparse
import json
import pathlib
import sys
import time

import numpy as np
import torch

ROOT = pathlib.Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))

from paper_2509_25401_b200 import _lib  # noqa: E402
from paper_2509_25401_b200.engine import Engine, EngineConfig  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--layers", type=int, default=1)
    ap.add_argument("--steps", type=int, default=13)
    ap.add_argument("--interval", type=int, default=6)
    ap.add_argument("--tau-q", type=float, default=0.3)
    ap.add_argument("--tau-kv", type=float, default=0.5)
    ap.add_argument("--graphs", type=int, default=1)
    a = ap.parse_args()
    cfg = EngineConfig(n_text=256, n_vision=32768, d_model=3072, heads=24, tau_q=a.tau_q,
                       tau_kv=a.tau_kv, interval_n=a.interval, order_d=1, steps=a.steps,
                       layers=a.layers, workload="drift")
    t0 = time.time()
    eng = Engine(cfg, graphs=bool(a.graphs))
    setup_s = time.time() - t0
    # warm one full window (captures the dispatch graphs), then time a second
    for t in range(cfg.interval_n):
        eng.step(t)
    torch.cuda.synchronize()
    eng.check("warm-up")
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(cfg.interval_n + 1)]
    _lib.reset_launch_count()
    ev[0].record()
    for k in range(cfg.interval_n):
        eng.step(cfg.interval_n + k)
        ev[k + 1].record()
    torch.cuda.synchronize()
    eng.check("timed window")
    launches = _lib.launch_count()
    ms = [ev[k].elapsed_time(ev[k + 1]) for k in range(cfg.interval_n)]
    # the window's sparsity from the device counters of one more dispatch step
    for layer in eng.layers:
        layer.pairs.zero_()
    eng.step(2 * cfg.interval_n + 1)
    pairs = sum(int(layer.pairs.sum()) for layer in eng.layers)
    total = cfg.layers * cfg.heads * cfg.t_q * cfg.t_kv
    # components: synthetic input generation vs the captured dispatch chain
    e0, e1, e2 = (torch.cuda.Event(enable_timing=True) for _ in range(3))
    e0.record()
    for _ in range(5):
        eng.workload.x_device(7, out=eng.x_buf)
    e1.record()
    for _ in range(5):
        x = eng.x_buf
        for li in range(len(eng.layers)):
            x = eng._dispatch_layer(li, x, 1)
    e2.record()
    torch.cuda.synchronize()
    xgen_ms, chain_ms = e0.elapsed_time(e1) / 5, e1.elapsed_time(e2) / 5
    print(json.dumps({
        "config": {"seq": cfg.n_tokens, "heads": cfg.heads, "d_model": cfg.d_model,
                   "layers": cfg.layers, "interval_n": cfg.interval_n, "tau_q": cfg.tau_q,
                   "tau_kv": cfg.tau_kv, "graphs": bool(a.graphs)},
        "update_ms": round(ms[0], 3), "dispatch_ms": [round(x, 3) for x in ms[1:]],
        "window_ms": round(sum(ms), 3), "avg_step_ms": round(sum(ms) / len(ms), 3),
        "pair_sparsity": round(1 - pairs / total, 4), "x_gen_ms": round(xgen_ms, 3),
        "dispatch_chain_ms": round(chain_ms, 3), "launches_per_window": launches,
        "setup_s": round(setup_s, 1)}))


if __name__ == "__main__":
    main()
