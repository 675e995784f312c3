"""Materialize-mode attention at C4: fused OP_reuse (one launch, K2r) vs
bias-mode attention followed by the standalone forecast kernel.

    python tools/materialize_ab.py [--cached 0.25] [--skip 0.5] [--order 1]
"""

import argparse
import ctypes
import json
import pathlib
import sys

import numpy as np
import torch

ROOT = pathlib.Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))

import paper_2509_25401_b200 as fo  # noqa: E402
from paper_2509_25401_b200 import _lib  # noqa: E402
from paper_2509_25401_b200.attention import ctypes_floats, forecast_coefficients  # noqa: E402
from bench import random_masks  # noqa: E402
from tools.sweep import timeit  # noqa: E402

T = 128


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--seq", type=int, default=33024)
    ap.add_argument("--heads", type=int, default=24)
    ap.add_argument("--cached", type=float, default=0.25)
    ap.add_argument("--skip", type=float, default=0.5)
    ap.add_argument("--order", type=int, default=1)
    a = ap.parse_args()
    S, H = a.seq, a.heads
    t = -(-S // T)
    torch.manual_seed(0)
    q, k, v = (torch.randn(S, H, T, device="cuda").bfloat16() for _ in range(3))
    fc = fo.FeatureCache(H, t, a.order, seq=S)
    for _ in range(a.order + 1):
        fc.push(torch.randn(S, H, T, device="cuda").bfloat16())
    cb, sb = random_masks(np.random.default_rng(0), H, t, a.cached, a.skip)
    sym = fo.encode_symbols(cb, sb, 1)
    out = torch.zeros(S, H, T, dtype=torch.bfloat16, device="cuda")
    plan = sym.plan(valid=fc.valid, valid_version=fc.version, order_d=a.order)
    coef = ctypes_floats(forecast_coefficients(1, 6, a.order + 1))

    def fused():
        fo.sparse_attention(q, k, v, sym, fc, None, 1, 6, a.order, mode="materialize", out=out,
                            check=False)

    def bias_only():
        fo.sparse_attention(q, k, v, sym, fc, None, 1, 6, a.order, mode="bias", out=out,
                            check=False)

    def forecast_only():
        _lib.call("fo_forecast_materialize", fc.stacks.data_ptr(), S, H, T, t, a.order,
                  plan.ptr(), fc.valid.data_ptr(), ctypes.addressof(coef), out.data_ptr(), None)

    def separate():
        bias_only()
        forecast_only()

    import time

    res = {}
    for rep in range(3):
        for name, fn in (("fused", fused), ("separate", separate), ("bias_only", bias_only),
                         ("forecast_only", forecast_only)):
            time.sleep(1.0)  # same thermal / power state for every variant
            res.setdefault(name, []).append(timeit(fn, warm=2, reps=10))
    ms = {k: round(float(np.median(v)), 4) for k, v in res.items()}
    n_cached = int((~cb.astype(bool)).sum())
    fbytes = n_cached * T * T * 2 * (a.order + 2)
    ms["forecast_GBps"] = round(fbytes / ms["forecast_only"] / 1e6, 1)
    ms["config"] = dict(seq=S, heads=H, cached=a.cached, skip=a.skip, order=a.order)
    print(json.dumps(ms))


if __name__ == "__main__":
    main()
