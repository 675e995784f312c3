"""GEMM-Q at C4 (S=33024, d_model 3072, 24 heads) with a given cached ratio, for ncu.
    python tools/gemm_q_prof.py [cached_ratio]   (0 = dense update phase)"""
import pathlib
import sys

import numpy as np
import torch

sys.path.insert(0, str(pathlib.Path(__file__).resolve().parents[1]))
import paper_2509_25401_b200 as fo  # noqa: E402

r = float(sys.argv[1]) if len(sys.argv) > 1 else 0.25
S, H, dm, T = 33024, 24, 3072, 128
t = S // T
x = torch.randn(S, dm, device="cuda").bfloat16()
wq = fo.pack_w_q(torch.randn(H, dm, T, device="cuda") * dm ** -0.5)
nw = torch.ones(H, T, device="cuda")
active = np.random.default_rng(0).random((H, t)) >= r
sym = fo.encode_symbols(active, np.ones((H, t, t), bool), 1)
q = torch.empty(S, H, T, dtype=torch.bfloat16, device="cuda")
phase = "update" if r == 0 else "dispatch"
for _ in range(3):
    fo.project_q(x, wq, nw, sym, phase, out=q, check=False)
torch.cuda.synchronize()
