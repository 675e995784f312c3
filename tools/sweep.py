"""Speedup-vs-sparsity sweeps on one B200.

    python tools/sweep.py [--out gpurun_out/sweep.json] [--quick]

attention (C4 HunyuanVideo 33K, C2 FLUX 4608): FC-only, BSS-only and combined
sparsity; GEMM-Q / GEMM-O (C3, d_model 3072, S in {4096, 33024}): cached-tile
ratio 0..0.9, plus the amortized GEMM-O speedup over an update cycle of N
steps, N/(1+(N-1)(1-s)) ideal (costs.py:32-42), measured as
N*T_dense / (T_update + (N-1)*T_dispatch). Every speedup is against the same
engine run with all-active symbols; 'frac' = speedup / ideal.
"""

import argparse
import json
import pathlib
import sys

import numpy as np
import torch

ROOT = pathlib.Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))

import paper_2509_25401_b200 as fo  # noqa: E402
from bench import random_masks  # noqa: E402

T = 128


EAGER = False


def timeit(fn, warm=2, reps=5):
    """median ms per call: a CUDA graph of `reps` calls (tools/timing.py)"""
    from tools.timing import eager_time, graph_time

    return (eager_time if EAGER else graph_time)(fn, reps=reps, trials=5, warm=warm)


def attention_sweep(S, H, points, seed=0):
    t = -(-S // T)
    g = torch.Generator(device="cuda").manual_seed(seed)
    q, k, v = (torch.randn(S, H, T, device="cuda", generator=g).bfloat16() for _ in range(3))
    fc = fo.FeatureCache(H, t, 0, seq=S)
    fc.push(v)
    out = torch.empty_like(q)
    dense = fo.encode_symbols(np.ones((H, t), bool), np.ones((H, t, t), bool), 1)
    t_dense = timeit(lambda: fo.sparse_attention(q, k, v, dense, fc, None, 1, 2, 0, mode="bias",
                                                 out=out, check=False))
    res = []
    for kind, cached, skip in points:
        rng = np.random.default_rng(seed)
        cb, sb = random_masks(rng, H, t, cached, skip)
        sym = fo.encode_symbols(cb, sb, 1)
        ms = timeit(lambda: fo.sparse_attention(q, k, v, sym, fc, None, 1, 2, 0, mode="bias",
                                                out=out, check=False))
        pairs = int(sum(sb[h][cb[h]].sum() for h in range(H)))
        s = 1 - pairs / (H * t * t)
        sp = t_dense / ms
        res.append({"kind": kind, "cached_ratio": cached, "kv_skip_ratio": skip,
                    "sparsity": round(s, 4), "ms": round(ms, 4), "dense_ms": round(t_dense, 4),
                    "speedup": round(sp, 3), "ideal": round(1 / (1 - s), 3),
                    "frac": round(sp * (1 - s), 3),
                    "tflops_effective": round(4.0 * T ** 3 * pairs / (ms * 1e-3) / 1e12, 1),
                    "tops_dense_equivalent": round(4.0 * T ** 3 * H * t * t / (ms * 1e-3) / 1e12, 1)})
    fo._runtime.Status.default().check("attention sweep")
    return res


def gemm_sweep(S, H, dm, ratios, order=1, intervals=(4, 6, 8), seed=0):
    t = -(-S // T)
    g = torch.Generator(device="cuda").manual_seed(seed)
    x = torch.randn(S, dm, device="cuda", generator=g).bfloat16()
    wq = fo.pack_w_q(torch.randn(H, dm, T, device="cuda", generator=g) * dm ** -0.5)
    norm = torch.ones(H, T, device="cuda")
    wo = fo.pack_w_out(torch.randn(H, T, dm, device="cuda", generator=g) * T ** -0.5)
    o = torch.randn(S, H, T, device="cuda", generator=g).bfloat16()
    fc = fo.FeatureCache(H, t, order, seq=S)
    for _ in range(order + 1):
        fc.push(torch.randn(S, H, T, device="cuda", generator=g).bfloat16())
    qo = torch.empty(S, H, T, dtype=torch.bfloat16, device="cuda")
    out = torch.empty(S, dm, dtype=torch.bfloat16, device="cuda")
    full = np.ones((H, t, t), bool)

    def syms(active):
        return fo.encode_symbols(active, full, 1)

    dense = syms(np.ones((H, t), bool))
    tq_dense = timeit(lambda: fo.project_q(x, wq, norm, dense, "dispatch", out=qo, fill=None, check=False))
    _, bias_dense = fo.project_out_update(o, wo, dense, fc, order)
    to_dense = timeit(lambda: fo.project_out_dispatch(o, wo, dense, bias_dense, 1, 6, order, out=out,
                                                      check=False))
    res = []
    for r in ratios:
        rng = np.random.default_rng(seed)
        active = rng.random((H, t)) >= r
        sym = syms(active)
        s = 1 - active.sum() / active.size
        tq = timeit(lambda: fo.project_q(x, wq, norm, sym, "dispatch", out=qo, fill=None, check=False))
        tu = timeit(lambda: fo.project_out_update(o, wo, sym, fc, order, out=out, check=False), 1, 3)
        _, bias = fo.project_out_update(o, wo, sym, fc, order)
        td = timeit(lambda: fo.project_out_dispatch(o, wo, sym, bias, 1, 6, order, out=out, check=False))
        ent = {"S": S, "cached_ratio": r, "sparsity": round(float(s), 4),
               "gemm_q_ms": round(tq, 4), "gemm_q_dense_ms": round(tq_dense, 4),
               "gemm_q_speedup": round(tq_dense / tq, 3), "gemm_q_ideal": round(1 / max(1 - s, 1e-9), 3),
               "gemm_o_dispatch_ms": round(td, 4), "gemm_o_dense_ms": round(to_dense, 4),
               "gemm_o_update_ms": round(tu, 4),
               "gemm_o_dispatch_speedup": round(to_dense / td, 3),
               "gemm_o_amortized": {}}
        for n in intervals:
            meas = n * to_dense / (tu + (n - 1) * td)
            ideal = n / (1 + (n - 1) * (1 - s))
            ent["gemm_o_amortized"][str(n)] = {"measured": round(meas, 3), "ideal": round(ideal, 3),
                                               "frac": round(meas / ideal, 3)}
        res.append(ent)
    fo._runtime.Status.default().check("gemm sweep")
    return res


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--out", default=None)
    ap.add_argument("--quick", action="store_true")
    ap.add_argument("--parts", default="attn,flux,gemm", help="subset of attn,flux,gemm")
    ap.add_argument("--eager", action="store_true", help="time Python calls, not CUDA graphs")
    a = ap.parse_args()
    global EAGER
    EAGER = a.eager
    parts = set(a.parts.split(","))
    pts = [("dense", 0.0, 0.0)]
    pts += [("FC", c, 0.0) for c in (0.1, 0.3, 0.5, 0.8)]
    pts += [("BSS", 0.0, s) for s in (0.1, 0.3, 0.5, 0.8)]
    pts += [("FC+BSS", c, s) for c, s in ((0.25, 0.5), (0.5, 0.6), (0.5, 0.8))]
    res = {"device": torch.cuda.get_device_name(),
           "timing": "eager Python calls" if EAGER else "CUDA graph of 5 calls, median of 5 replays"}
    if "attn" in parts:
        res["attention_c4"] = attention_sweep(33024, 24, pts)
    flux = [("BSS", 0.0, s) for s in (0.0, 0.1, 0.3, 0.5, 0.7, 0.9)]
    if "flux" in parts:
        res["attention_c2_flux"] = attention_sweep(4608, 24, flux)
    ratios = (0.0, 0.25, 0.5, 0.75, 0.9)
    if "gemm" in parts:
        res["gemm_c3_s4096_D1"] = gemm_sweep(4096, 24, 3072, ratios, order=1)
    if "gemm" in parts and not a.quick:
        res["gemm_c3_s33024_D1"] = gemm_sweep(33024, 24, 3072, ratios, order=1)
        res["gemm_c3_s33024_D0"] = gemm_sweep(33024, 24, 3072, ratios, order=0)
    txt = json.dumps(res, indent=1)
    print(txt)
    if a.out:
        pathlib.Path(a.out).write_text(txt)


if __name__ == "__main__":
    main()
