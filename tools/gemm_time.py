"""Median-of-trials timing of GEMM-Q, GEMM-O dispatch and GEMM-O update at C3
(S=33024, d_model 3072, 24 heads) for A/B runs of library variants:
    python tools/gemm_time.py [--ratios 0.25,0.75,0.9] [--orders 0,1]
Prints one JSON object {"<op>@<ratio>/D<order>": ms, ...}."""
import argparse
import json
import pathlib
import sys

import numpy as np
import torch

sys.path.insert(0, str(pathlib.Path(__file__).resolve().parents[1]))
import paper_2509_25401_b200 as fo  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--ratios", default="0.0,0.25,0.75,0.9")
ap.add_argument("--orders", default="0,1")
ap.add_argument("--ops", default="q,disp,upd")
ap.add_argument("--seq", type=int, default=33024)
ap.add_argument("--eager", action="store_true", help="time Python calls, not a CUDA graph")
a = ap.parse_args()
S, H, dm, T = a.seq, 24, 3072, 128
t = S // T
ops = set(a.ops.split(","))


from tools.timing import eager_time, graph_time  # noqa: E402


def timeit(fn, reps=10, trials=5):
    return (eager_time if a.eager else graph_time)(fn, reps=reps, trials=trials)


g = torch.Generator(device="cuda").manual_seed(0)
x = torch.randn(S, dm, device="cuda", generator=g).bfloat16()
wq = fo.pack_w_q(torch.randn(H, dm, T, device="cuda", generator=g) * dm ** -0.5)
norm = torch.ones(H, T, device="cuda")
wo = fo.pack_w_out(torch.randn(H, T, dm, device="cuda", generator=g) * T ** -0.5)
o = torch.randn(S, H, T, device="cuda", generator=g).bfloat16()
qo = torch.empty(S, H, T, dtype=torch.bfloat16, device="cuda")
out = torch.empty(S, dm, dtype=torch.bfloat16, device="cuda")
full = np.ones((H, t, t), bool)
if "qkv" in ops:
    wraw = [torch.randn(H, dm, T, device="cuda", generator=g) * dm ** -0.5 for _ in range(3)]
    wqkv, wk = fo.pack_w_qkv(*wraw), fo.pack_w_q(wraw[1])
    ko, vo = torch.empty_like(qo), torch.empty_like(qo)
    dsym = fo.encode_symbols(np.ones((H, t), bool), full, 1)
res = {}
for order in [int(v) for v in a.orders.split(",")]:
    fc = fo.FeatureCache(H, t, order, seq=S)
    for _ in range(order + 1):
        fc.push(torch.randn(S, H, T, device="cuda", generator=g).bfloat16())
    for r in [float(v) for v in a.ratios.split(",")]:
        active = np.random.default_rng(0).random((H, t)) >= r
        sym = fo.encode_symbols(active, full, 1)
        if "q" in ops and order == int(a.orders.split(",")[0]):
            res[f"q@{r}"] = round(timeit(lambda: fo.project_q(x, wq, norm, sym, "dispatch", out=qo,
                                                              fill=None, check=False)), 4)
        if "qkv" in ops and order == int(a.orders.split(",")[0]):
            # the dispatch step's projections: one fused launch vs Q + K + V launches
            res[f"qkv@{r}"] = round(timeit(lambda: fo.project_qkv(
                x, wqkv, norm, norm, sym, "dispatch", q_out=qo, k_out=ko, v_out=vo,
                check=False)), 4)
            res[f"q+k+v@{r}"] = round(timeit(lambda: (
                fo.project_q(x, wq, norm, sym, "dispatch", out=qo, fill=None, check=False),
                fo.project_q(x, wk, norm, dsym, "dispatch", out=ko, fill=None, check=False),
                fo.project_q(x, wk, None, dsym, "dispatch", out=vo, fill=None, rope=False,
                             check=False))), 4)
        _, bias = fo.project_out_update(o, wo, sym, fc, order)
        if "disp" in ops:
            res[f"disp@{r}/D{order}"] = round(timeit(lambda: fo.project_out_dispatch(
                o, wo, sym, bias, 1, 6, order, out=out, check=False)), 4)
        if "upd" in ops:
            res[f"upd@{r}/D{order}"] = round(timeit(lambda: fo.project_out_update(
                o, wo, sym, fc, order, out=out, bias=bias, check=False), reps=5, trials=3), 4)
fo._runtime.Status.default().check("gemm_time")
print(json.dumps(res))
