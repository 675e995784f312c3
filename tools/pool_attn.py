"""Sparse attention at C4 (33,024 tokens, 24 heads) with POOLED symbols
(pool_n = 2: query blocks 2c, 2c+1 share a skip row; the CTA-pair kernel with
K/V multicast runs them), against the same engine on all-active symbols:
    python tools/pool_attn.py [pool_n]
Prints one JSON object {"<cached>/<skip>": [ms, speedup, ideal, frac], "dense": ms}."""
import json
import pathlib
import sys

import numpy as np
import torch

sys.path.insert(0, str(pathlib.Path(__file__).resolve().parents[1]))
import paper_2509_25401_b200 as fo  # noqa: E402
from bench import random_masks  # noqa: E402
from tools.timing import graph_time  # noqa: E402

pool = int(sys.argv[1]) if len(sys.argv) > 1 else 2
S, H, T = 33024, 24, 128
t = S // T
tc = -(-t // pool)
g = torch.Generator(device="cuda").manual_seed(0)
q, k, v = (torch.randn(S, H, T, device="cuda", generator=g).bfloat16() for _ in range(3))
fc = fo.FeatureCache(H, t, 0, seq=S)
fc.push(v)
out = torch.empty_like(q)
dense = fo.encode_symbols(np.ones((H, t), bool), np.ones((H, t, t), bool), 1)
t_dense = graph_time(lambda: fo.sparse_attention(q, k, v, dense, fc, None, 1, 2, 0, mode="bias",
                                                 out=out, check=False), reps=3)
res = {"pool_n": pool, "dense_ms": round(t_dense, 4)}
for cached, skip in ((0.0, 0.0), (0.25, 0.5), (0.5, 0.8)):
    cbc, sbc = random_masks(np.random.default_rng(0), H, tc, cached, skip)  # compressed grid
    cb = np.repeat(cbc, pool, axis=1)[:, :t]
    sb = np.repeat(np.repeat(sbc, pool, axis=1), pool, axis=2)[:, :t, :t]
    sym = fo.encode_symbols(cb, sb, pool)
    ms = graph_time(lambda: fo.sparse_attention(q, k, v, sym, fc, None, 1, 2, 0, mode="bias",
                                                out=out, check=False), reps=3)
    s_ = 1 - sum(sb[h][cb[h]].sum() for h in range(H)) / (H * t * t)
    res[f"{cached}/{skip}"] = [round(ms, 4), round(t_dense / ms, 3), round(1 / (1 - s_), 3),
                               round(t_dense / ms * (1 - s_), 3)]
fo._runtime.Status.default().check("pool_attn")
print(json.dumps(res))
