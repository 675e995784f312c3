"""GEMM-O dispatch at C3 (S=33024) with a given cached ratio, for ncu."""
import sys, pathlib
import numpy as np, torch
sys.path.insert(0, str(pathlib.Path(__file__).resolve().parents[1]))
import paper_2509_25401_b200 as fo
r = float(sys.argv[1]) if len(sys.argv) > 1 else 0.9
S, H, dm, T, order = 33024, 24, 3072, 128, 1
t = S // T
wo = fo.pack_w_out(torch.randn(H, T, dm, device="cuda") * T ** -0.5)
o = torch.randn(S, H, T, device="cuda").bfloat16()
fc = fo.FeatureCache(H, t, order, seq=S)
for _ in range(2):
    fc.push(torch.randn(S, H, T, device="cuda").bfloat16())
active = np.random.default_rng(0).random((H, t)) >= r
sym = fo.encode_symbols(active, np.ones((H, t, t), bool), 1)
_, bias = fo.project_out_update(o, wo, sym, fc, order)
out = torch.empty(S, dm, dtype=torch.bfloat16, device="cuda")
for _ in range(3):
    fo.project_out_dispatch(o, wo, sym, bias, 1, 6, order, out=out, check=False)
torch.cuda.synchronize()
