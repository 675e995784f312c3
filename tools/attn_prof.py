"""Sparse attention alone at C4 (S=33024, H=24, 25% cached / 50% KV skip), for ncu.
FO_ATTN_IMPL selects the kernel."""
import pathlib
import sys

import numpy as np
import torch

sys.path.insert(0, str(pathlib.Path(__file__).resolve().parents[1]))
import paper_2509_25401_b200 as fo  # noqa: E402
from bench import random_masks  # noqa: E402

S, H, T = 33024, 24, 128
t = S // T
cb, sb = random_masks(np.random.default_rng(0), H, t, 0.25, 0.5)
q, k, v = (torch.randn(S, H, T, device="cuda").bfloat16() for _ in range(3))
sym = fo.encode_symbols(cb, sb, 1)
fc = fo.FeatureCache(H, t, 0, seq=S)
fc.push(v)
out = torch.empty_like(q)
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
for it in range(4):
    e0.record()
    fo.sparse_attention(q, k, v, sym, fc, None, 1, 2, 0, mode="bias", out=out, check=False)
    e1.record()
    torch.cuda.synchronize()
    print(f"attention {e0.elapsed_time(e1):.3f} ms")
