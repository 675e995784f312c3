"""GEMM-O dispatch with every head cached (pure bias stream: out = c0 * B_c[0])
against torch copies of the same bytes, to bound the epilogue's streaming rate."""
import json
import pathlib
import sys

import numpy as np
import torch

sys.path.insert(0, str(pathlib.Path(__file__).resolve().parents[1]))
import paper_2509_25401_b200 as fo  # noqa: E402
from tools.timing import graph_time  # noqa: E402

S, H, dm, T = 33024, 24, 3072, 128
t = S // T
res = {}
g = torch.Generator(device="cuda").manual_seed(0)
wo = fo.pack_w_out(torch.randn(H, T, dm, device="cuda", generator=g) * T ** -0.5)
o = torch.randn(S, H, T, device="cuda", generator=g).bfloat16()
out = torch.empty(S, dm, dtype=torch.bfloat16, device="cuda")
for order in [int(v) for v in (sys.argv[1] if len(sys.argv) > 1 else "0,1").split(",")]:
    fc = fo.FeatureCache(H, t, order, seq=S)
    for _ in range(order + 1):
        fc.push(torch.randn(S, H, T, device="cuda", generator=g).bfloat16())
    for r in (1.0, 0.9):
        active = np.random.default_rng(0).random((H, t)) >= r
        sym = fo.encode_symbols(active, np.ones((H, t, t), bool), 1)
        _, bias = fo.project_out_update(o, wo, sym, fc, order)
        res[f"disp@{r}/D{order}"] = round(graph_time(lambda: fo.project_out_dispatch(
            o, wo, sym, bias, 1, 6, order, out=out, check=False)), 4)
a = torch.empty(S, dm, dtype=torch.bfloat16, device="cuda")
b = torch.empty_like(a)
res["copy_203MB"] = round(graph_time(lambda: b.copy_(a)), 4)
a2 = torch.empty(2, S, dm, dtype=torch.bfloat16, device="cuda")
res["add_2x203MB_to_203MB"] = round(graph_time(lambda: torch.add(a2[0], a2[1], out=b)), 4)
print(json.dumps(res))
