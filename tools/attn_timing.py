"""Per-phase cycle breakdown of the attention kernel (FO_ATTN_TIMING build)."""
import ctypes, sys, pathlib, shutil
import numpy as np
ROOT = pathlib.Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
so = sys.argv[1]
shutil.copy(so, ROOT / "paper_2509_25401_b200" / "_fo_b200.so")
import torch
import paper_2509_25401_b200 as fo
from bench import random_masks
S, H, T = 33024, 24, 128
t = S // T
rng = np.random.default_rng(0)
cb, sb = random_masks(rng, H, t, 0.25, 0.5)
q, k, v = (torch.randn(S, H, T, device="cuda").bfloat16() for _ in range(3))
sym = fo.encode_symbols(cb, sb, 1)
fc = fo.FeatureCache(H, t, 0, seq=S); fc.push(v)
out = torch.empty_like(q)
for _ in range(3):
    fo.sparse_attention(q, k, v, sym, fc, None, 1, 2, 0, mode="bias", out=out)
lib = fo._lib.load()
lib.fo_debug_timing.argtypes = [ctypes.c_void_p]
buf = np.zeros(148 * 32, np.int64)
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record(); fo.sparse_attention(q, k, v, sym, fc, None, 1, 2, 0, mode="bias", out=out); e1.record()
torch.cuda.synchronize()
lib.fo_debug_timing(buf.ctypes.data)
b = buf.reshape(148, 32).astype(np.float64)
pairs = int(sum(sb[h][cb[h]].sum() for h in range(H)))
tiles_per_cta = pairs / 148
names = {0: "sm:wait S", 1: "sm:LDTM+wait", 2: "sm:max", 3: "sm:exp", 4: "sm:STTM+wait", 5: "sm:o_done+rescale",
         6: "sm:arrive", 7: "sm:loop/epilogue", 16 + 8: "mma:after PV->wait P", 16 + 9: "mma:wait P",
         16 + 10: "mma:wait K", 16 + 11: "mma:QK issue (pre-wait)", 16 + 12: "mma:after P->V wait", 16 + 13: "mma:wait V"}
ms = e0.elapsed_time(e1)
print(f"kernel {ms:.3f} ms, tiles/CTA {tiles_per_cta:.0f}, cycles/tile {ms*1e-3*1.965e9/tiles_per_cta:.0f}")
for kk, nm in names.items():
    print(f"{nm:28s} {b[:, kk].mean() / tiles_per_cta:8.1f} cycles/tile")
